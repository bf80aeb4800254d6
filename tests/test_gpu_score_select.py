"""GPU parity of spc_score_select (one persistent launch: LOGITS + NORM + GROUP + top-k +
INDEXED elastic diff, O1..O8) against the separate ABI calls (spc_score(ALL) + spc_topk +
spc_elastic_diff) and the CPU oracle: logits, head maxima, fixed-point sums, group scores,
selections, diffs and evictions bit-exact, over consecutive steps; adversarial score
patterns (ties, flat rows, huge threshold buckets, wide ranges) built through one-hot
queries, whose logits are exactly the keys' first coordinate (O1 with q = e_0, scale 1)."""
import numpy as np
import pytest
import torch

from paper_2512_00722_b200 import spc, synth

pytestmark = pytest.mark.gpu
DEV = "cuda"
f32, i32 = torch.float32, torch.int32


def z(*s, dt=f32, fill=0):
    return torch.full(s, fill, dtype=dt, device=DEV)


def separate(q, kr, seq, k, scale, prev, force):
    B, G, S, D = kr.shape
    Hq = q.shape[1]
    lg, hm, F, gs = z(B, Hq, S), z(B, Hq), z(B, Hq, dt=torch.int64), z(B, G, S)
    ws = spc.alloc_workspace(spc.score_workspace(B, Hq, S), DEV)
    wt = spc.alloc_workspace(spc.topk_workspace(B, G, S, k), DEV)
    spc.score(q, kr, seq, G, scale, lg, hm, F, gs, ws, phases=spc.SCORE_ALL)
    idx, cnt = z(B, G, k, dt=i32), z(B, G, dt=i32)
    spc.topk(gs, seq, k, idx, cnt, wt, force_last=force)
    lt, nl, et, ne = z(B, G, k, dt=i32), z(B, G, dt=i32), z(B, G, k, dt=i32), z(B, G, dt=i32)
    spc.elastic_diff(prev[0], prev[1], idx, cnt, lt, nl, evict_tok=et, n_evict=ne)
    return dict(logits=lg, head_max=hm, F=F, gs=gs, idx=idx, cnt=cnt, lt=lt, nl=nl, et=et, ne=ne)


def fused(q, kr, seq, k, scale, prev, force, ws):
    B, G, S, D = kr.shape
    Hq = q.shape[1]
    # outputs pre-filled with junk: the kernel must write every element it owns
    lg = z(B, Hq, S, fill=-7.0)
    hm, F, gs = z(B, Hq, fill=3.0), z(B, Hq, dt=torch.int64, fill=-5), z(B, G, S, fill=-1.0)
    idx, cnt = z(B, G, k, dt=i32, fill=-9), z(B, G, dt=i32, fill=-9)
    lt, nl, et, ne = (z(B, G, k, dt=i32, fill=-3), z(B, G, dt=i32, fill=-3),
                      z(B, G, k, dt=i32, fill=-3), z(B, G, dt=i32, fill=-3))
    spc.score_select(q, kr, seq, scale, k, hm, F, gs, idx, cnt, prev[0], prev[1], lt, nl, ws,
                     logits=lg, evict_tok=et, n_evict=ne, force_last=force)
    return dict(logits=lg, head_max=hm, F=F, gs=gs, idx=idx, cnt=cnt, lt=lt, nl=nl, et=et, ne=ne)


def compare(a, b, seq):
    torch.cuda.synchronize()
    B, Hq, S = a["logits"].shape
    for b_ in range(B):  # logits are defined below seq_len only
        n = min(int(seq[b_]), S)
        assert torch.equal(a["logits"][b_, :, :n].view(i32), b["logits"][b_, :, :n].view(i32))
    for key in ("head_max", "gs"):
        assert torch.equal(a[key].view(i32), b[key].view(i32)), key
    for key in ("F", "idx", "cnt", "lt", "nl", "et", "ne"):
        assert torch.equal(a[key], b[key]), key


def run_steps(q_steps, kr, seq, k, scale=0.088, force=True, oracle=None):
    B, G, S, D = kr.shape
    Hq = q_steps.shape[2]
    assert spc.score_select_supported(B, Hq, G, D, S, k)
    ws = spc.alloc_workspace(spc.score_select_workspace(B, Hq, G, S), DEV)
    prev_a = (z(B, G, k, dt=i32, fill=-1), z(B, G, dt=i32))
    prev_b = (prev_a[0].clone(), prev_a[1].clone())
    for step in range(q_steps.shape[0]):
        a = separate(q_steps[step], kr, seq, k, scale, prev_a, force)
        b = fused(q_steps[step], kr, seq, k, scale, prev_b, force, ws)
        compare(a, b, seq.tolist())
        if oracle is not None:
            oidx, _, ocnt, _ = oracle.topk(a["gs"].cpu().numpy(), seq.tolist(), k, force_last=force)
            assert np.array_equal(b["idx"].cpu().numpy(), oidx)
            assert np.array_equal(b["cnt"].cpu().numpy(), ocnt)
        prev_a, prev_b = (a["idx"], a["cnt"]), (b["idx"], b["cnt"])
    torch.cuda.synchronize()  # three launches on one workspace: its counters were restored
    return b


@pytest.mark.parametrize("B,alpha,G,D,S,k,lens", [
    (1, 4, 8, 128, 32768, 2048, None),        # config B
    (2, 4, 2, 128, 5000, 700, [5000, 1667]),  # ragged batch
    (1, 8, 1, 128, 300, 512, None),           # k > S: no cut
    (2, 1, 4, 64, 20000, 64, [20000, 20000]),
    (1, 2, 3, 64, 9000, 1000, None),
    (1, 4, 1, 64, 4096, 256, None),           # config A
])
def test_score_select_equals_separate_calls(oracle, B, alpha, G, D, S, k, lens):
    Hq = alpha * G
    kr = synth.retrieval_keys(B, G, S, D, seed=S + alpha, device=DEV)
    qs = synth.retrieval_queries(3, B, Hq, G, D, seed=S + alpha, device=DEV)
    seq = torch.tensor(lens if lens else [S] * B, dtype=i32, device=DEV)
    run_steps(qs, kr, seq, k, oracle=oracle)


def onehot_case(kind, B, G, S, seed):
    """Key rows whose first coordinate is the wanted logit (bf16), the rest zero."""
    g = torch.Generator(device="cpu").manual_seed(seed)
    if kind == "flat":
        v = torch.zeros((B, G, S))
    elif kind == "two_level":
        v = torch.zeros((B, G, S))
        v[:, :, torch.randperm(S, generator=g)[:S // 50]] = 3.0
    elif kind == "quantised":
        v = torch.randint(0, 17, (B, G, S), generator=g).float() * 0.25
    elif kind == "wide":
        v = -torch.rand((B, G, S), generator=g) * 80.0
        v[:, :, 0] = 0.0
    else:
        v = torch.randn((B, G, S), generator=g) * 2.0
    kr = torch.zeros((B, G, S, 64), dtype=torch.bfloat16)
    kr[..., 0] = v.to(torch.bfloat16)
    return kr.to(DEV)


@pytest.mark.parametrize("kind", ["flat", "two_level", "quantised", "wide", "randn"])
@pytest.mark.parametrize("force", [True, False])
def test_score_select_adversarial(oracle, kind, force):
    B, G, alpha, S, k = 2, 2, 4, 8192, 1024
    Hq = alpha * G
    kr = onehot_case(kind, B, G, S, seed=hash(kind) % 1000)
    q = torch.zeros((2, B, Hq, 64), dtype=torch.bfloat16, device=DEV)
    q[..., 0] = 1.0
    q[1, :, 1::2, 0] = 0.5  # second step: other weights per head
    seq = torch.tensor([S, 3001], dtype=i32, device=DEV)
    run_steps(q, kr, seq, k, scale=1.0, force=force, oracle=oracle)


def test_score_select_rejects_unsupported():
    # 16 rows x 256 tiles = 4096 tiles over <= 148 SMs: > 16 tiles per SM
    assert not spc.score_select_supported(2, 32, 8, 128, 32768, 2048)
    assert not spc.score_select_supported(1, 12, 4, 128, 4096, 256)  # alpha 3
    assert spc.score_select_supported(1, 32, 8, 128, 32768, 2048)
    B, G, Hq, D, S, k = 2, 8, 32, 128, 32768, 2048
    ws = spc.alloc_workspace(spc.score_select_workspace(B, Hq, G, S), DEV)
    with pytest.raises(spc.SpcError):
        spc.score_select(z(B, Hq, D, dt=torch.bfloat16), z(B, G, S, D, dt=torch.bfloat16),
                         z(B, dt=i32, fill=S), 0.1, k, z(B, Hq), z(B, Hq, dt=torch.int64),
                         z(B, G, S), z(B, G, k, dt=i32), z(B, G, dt=i32), z(B, G, k, dt=i32),
                         z(B, G, dt=i32), z(B, G, k, dt=i32), z(B, G, dt=i32), ws)


def test_decode_step_one_launch_equals_default():
    """DecodeStep(one_launch=True) (spc_score_select) reproduces the default step (spc_score +
    spc_select) bit for bit over three graph-replayed config-B steps, attention included."""
    from paper_2512_00722_b200.pipeline import DecodeStep
    c = synth.CONFIGS["B"]
    B, G, Hq, D, S, L, k = c["B"], c["G"], c["Hq"], c["D"], c["S"], 4, c["k"]
    kr = synth.retrieval_keys(B, G, S, D, seed=77, device=DEV)
    kc, vc = synth.llm_kv(L, B, G, S, D, seed=77, device=DEV)
    qr = synth.retrieval_queries(3, B, Hq, G, D, seed=77, device=DEV)
    ql = synth.llm_queries(1, L, B, Hq, D, seed=77, device=DEV)[0]
    seq = torch.full((B,), S, dtype=i32, device=DEV)
    a = DecodeStep(kr, [kc[l] for l in range(L)], [vc[l] for l in range(L)], seq, L, Hq, k)
    b = DecodeStep(kr, [kc[l] for l in range(L)], [vc[l] for l in range(L)], seq, L, Hq, k,
                   one_launch=True)
    assert b.one_launch and not a.one_launch
    for s in range(3):
        ia, ca = a.step(qr[s], ql, use_graph=True)
        ib, cb = b.step(qr[s], ql, use_graph=True)
        torch.cuda.synchronize()
        assert torch.equal(ia, ib) and torch.equal(ca, cb)
        assert torch.equal(a.n_load, b.n_load) and torch.equal(a.load_tok, b.load_tok)
        assert torch.equal(a.out, b.out) and torch.equal(a.lse, b.lse)
