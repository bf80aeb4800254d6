"""GPU parity of spc_score (O1..O6) against the CPU oracle: BIT-EXACT logits, head maxima,
int64 normalisers and group scores, on seeded synthetic inputs of the paper's shapes
(config A; every head dim x alpha the library supports; ragged seq_len; a tail that is
not a multiple of the 256-row tile; config B at full size)."""
import math

import numpy as np
import pytest
import torch

from paper_2512_00722_b200 import spc, synth

pytestmark = pytest.mark.gpu


def run_score(q, kr, seq, G, scale):
    dev = kr.device
    B, Hq, D = q.shape
    Smax = kr.shape[2]
    lg = torch.zeros((B, Hq, Smax), dtype=torch.float32, device=dev)
    hm = torch.zeros((B, Hq), dtype=torch.float32, device=dev)
    F = torch.zeros((B, Hq), dtype=torch.int64, device=dev)
    gs = torch.zeros((B, G, Smax), dtype=torch.float32, device=dev)
    ws = spc.alloc_workspace(spc.score_workspace(B, Hq, Smax), dev)
    spc.score(q, kr, seq, G, scale, lg, hm, F, gs, ws)
    torch.cuda.synchronize()
    return lg.cpu().numpy(), hm.cpu().numpy(), F.cpu().numpy(), gs.cpu().numpy()


def check(oracle, q, kr, seq_list, G, scale):
    dev = torch.device("cuda")
    seq = torch.tensor(seq_list, dtype=torch.int32, device=dev)
    lg, hm, F, gs = run_score(q.to(dev), kr.to(dev), seq, G, scale)
    olg, ohm, oF, ogs = oracle.score(synth.bf16_bits(q), synth.bf16_bits(kr), seq_list, G, scale)
    for b, S in enumerate(seq_list):
        assert np.array_equal(lg[b, :, :S].view(np.uint32), olg[b, :, :S].view(np.uint32)), b
    assert np.array_equal(hm.view(np.uint32), ohm.view(np.uint32))
    assert np.array_equal(F, oF)
    assert np.array_equal(gs.view(np.uint32), ogs.view(np.uint32))
    return gs


def f32(x):
    return float(np.float32(x))


def test_score_config_a(oracle):
    c = synth.CONFIGS["A"]
    kr = synth.retrieval_keys(1, c["G"], c["S"], c["D"], seed=synth.BASE_SEED)
    q = synth.retrieval_queries(2, 1, c["Hq"], c["G"], c["D"], seed=synth.BASE_SEED)
    for s in range(2):
        check(oracle, q[s], kr, [c["S"]], c["G"], f32(1 / math.sqrt(c["D"])))


@pytest.mark.parametrize("D", [64, 128])
@pytest.mark.parametrize("alpha,G", [(1, 3), (2, 2), (4, 2), (8, 1)])
def test_score_shapes_ragged(oracle, D, alpha, G):
    B, Smax = 3, 1000  # 1000 = 3 full 256-row tiles + a ragged tail
    Hq = alpha * G
    kr = synth.retrieval_keys(B, G, Smax, D, seed=D + alpha)
    q = synth.retrieval_queries(1, B, Hq, G, D, seed=D + alpha)[0]
    check(oracle, q, kr, [1000, 1, 517], G, f32(1 / math.sqrt(D)))


def test_score_extreme_logits_and_ties(oracle):
    """Large query scale (logits ~1e3, most weights underflow to 0 in O3) and duplicated keys."""
    B, G, Hq, D, S = 1, 2, 8, 128, 700
    kr = synth.duplicate_rows(synth.retrieval_keys(B, G, S, D, seed=5), 200, seed=5)
    q = (synth.retrieval_queries(1, B, Hq, G, D, seed=5)[0].float() * 40).to(torch.bfloat16)
    check(oracle, q, kr, [S], G, 0.3)


def test_score_config_b_full_size(oracle):
    """Config B (8B shape, 32K context) at full size, bit-exact against the oracle."""
    c = synth.CONFIGS["B"]
    kr = synth.retrieval_keys(1, c["G"], c["S"], c["D"], seed=synth.BASE_SEED + 1,
                              device="cuda")
    q = synth.retrieval_queries(1, 1, c["Hq"], c["G"], c["D"], seed=synth.BASE_SEED + 1,
                                device="cuda")[0]
    check(oracle, q.cpu(), kr.cpu(), [c["S"]], c["G"], f32(1 / math.sqrt(c["D"])))


def test_exp_and_fixpoint_sweep_through_norm_group(oracle):
    """O3/O4 on a sweep of the whole exp domain: every 256th float32 in [-87.5, 0] plus the
    edge values, as one head's logits with head max 0.  The group score of a single-head
    group is e * r per token, so every exp value is checked bit-exactly (NORM and GROUP
    of spc_score, and the fused spc_select), and the int64 normaliser checks every
    fixed-point conversion's sum."""
    hi = np.frombuffer(np.float32(-87.5).tobytes(), np.uint32)[0]
    bits = np.arange(0x80000000, hi + 1, 256, dtype=np.uint64).astype(np.uint32)
    edge = np.array([0.0, -0.0, -87.0, np.nextafter(np.float32(-87), np.float32(0)),
                     np.nextafter(np.float32(-87), np.float32(-100)), -1e-45, -1e-38, -0.5,
                     -0.6931472, -1.0, -2.0, -86.99], np.float32)
    x = np.concatenate([bits.view(np.float32), edge])
    S = (len(x) + 3) // 4 * 4
    lg = np.full((1, 1, S), -100.0, np.float32)
    lg[0, 0, :len(x)] = x
    n = len(x)
    hm = np.zeros((1, 1), np.float32)
    oF = oracle.norm(lg, hm, [n])
    ogs = oracle.group(lg, hm, oF, [n], 1)
    dev = torch.device("cuda")
    lg_d, hm_d = torch.from_numpy(lg).to(dev), torch.from_numpy(hm).to(dev)
    seq = torch.tensor([n], dtype=torch.int32, device=dev)
    F = torch.zeros((1, 1), dtype=torch.int64, device=dev)
    gs = torch.zeros((1, 1, S), dtype=torch.float32, device=dev)
    ws = spc.alloc_workspace(spc.score_workspace(1, 1, S), dev)
    q = torch.zeros((1, 1, 64), dtype=torch.bfloat16, device=dev)
    kr = torch.zeros((1, 1, S, 64), dtype=torch.bfloat16, device=dev)
    spc.score(q, kr, seq, 1, 1.0, lg_d, hm_d, F, gs, ws, phases=spc.SCORE_NORM | spc.SCORE_GROUP)
    torch.cuda.synchronize()
    assert np.array_equal(F.cpu().numpy(), oF)
    assert np.array_equal(gs.cpu().numpy().view(np.uint32), ogs.view(np.uint32))


def test_exp_sweep_through_fused_select(oracle):
    """The same exp/fixed-point check through spc_select's register-cached NORM/GROUP."""
    S = 131072
    rng = np.random.default_rng(11)
    x = -rng.random(S).astype(np.float32) * 88.0
    x[:64] = np.array([0.0, -0.0, -87.0, -1e-45, -1e-38, -0.5, -86.999] + [-1.0] * 57, np.float32)
    lg = x.reshape(1, 1, S).copy()
    hm = np.zeros((1, 1), np.float32)
    oF = oracle.norm(lg, hm, [S])
    ogs = oracle.group(lg, hm, oF, [S], 1)
    dev = torch.device("cuda")
    z = lambda *s, dt=torch.int32: torch.zeros(s, dtype=dt, device=dev)  # noqa: E731
    F, gs = z(1, 1, dt=torch.int64), z(1, 1, S, dt=torch.float32)
    k = 2048
    spc.select(torch.from_numpy(lg).to(dev), torch.from_numpy(hm).to(dev),
               torch.tensor([S], dtype=torch.int32, device=dev), 1, k, F, gs, z(1, 1, k),
               z(1, 1), torch.full((1, 1, k), -1, dtype=torch.int32, device=dev), z(1, 1),
               z(1, 1, k), z(1, 1))
    torch.cuda.synchronize()
    assert np.array_equal(F.cpu().numpy(), oF)
    assert np.array_equal(gs.cpu().numpy().view(np.uint32), ogs.view(np.uint32))


@pytest.mark.parametrize("Smax,lens", [(1001, [1001, 3, 999]), (20001, [20001, 7777, 1])])
def test_score_smax_not_multiple_of_4(oracle, Smax, lens):
    """NORM's scalar path (rows not float4-aligned), single- and multi-block per head."""
    B, G, alpha, D = len(lens), 2, 4, 128
    kr = synth.retrieval_keys(B, G, Smax, D, seed=Smax)
    q = synth.retrieval_queries(1, B, alpha * G, G, D, seed=Smax)[0]
    check(oracle, q, kr, lens, G, f32(1 / math.sqrt(D)))


@pytest.mark.parametrize("Hq,G,Smax,seq_list", [(32, 8, 32768, [32768]), (8, 2, 1000, [1000, 513, 1]),
                                                (4, 4, 3001, [3001, 17]), (64, 8, 2000, [2000])])
def test_batch_level_score_and_topk(oracle, Hq, G, Smax, seq_list):
    """SPC_SCORE_BATCH (NEXT-3): the batch-level score (sum of all heads' weights, O6b) is
    bit-identical to the oracle on every group row, and the per-row top-k selects the
    oracle's set in every group."""
    dev = torch.device("cuda")
    B, D, k = len(seq_list), 128, 256
    kr = synth.retrieval_keys(B, G, Smax, D, seed=Hq + Smax)
    q = synth.retrieval_queries(1, B, Hq, G, D, seed=Hq + Smax)[0]
    scale = f32(1 / math.sqrt(D))
    seq = torch.tensor(seq_list, dtype=torch.int32, device=dev)
    lg = torch.zeros((B, Hq, Smax), dtype=torch.float32, device=dev)
    hm = torch.zeros((B, Hq), dtype=torch.float32, device=dev)
    F = torch.zeros((B, Hq), dtype=torch.int64, device=dev)
    gs = torch.full((B, G, Smax), -1.0, dtype=torch.float32, device=dev)
    ws = spc.alloc_workspace(spc.score_workspace(B, Hq, Smax), dev)
    spc.score(q.to(dev), kr.to(dev), seq, G, scale, lg, hm, F, gs, ws,
              phases=spc.SCORE_ALL | spc.SCORE_BATCH)
    idx = torch.zeros((B, G, k), dtype=torch.int32, device=dev)
    cnt = torch.zeros((B, G), dtype=torch.int32, device=dev)
    wt = spc.alloc_workspace(spc.topk_workspace(B, G, Smax, k), dev)
    spc.topk(gs, seq, k, idx, cnt, wt, force_last=True)
    torch.cuda.synchronize()
    olg, ohm, oF, _ = oracle.score(synth.bf16_bits(q), synth.bf16_bits(kr), seq_list, G, scale)
    obs = oracle.batch_score(olg, ohm, oF, seq_list)
    g = gs.cpu().numpy()
    for gg in range(G):
        assert np.array_equal(g[:, gg].view(np.uint32), obs.view(np.uint32)), gg
    oidx, _, ocnt, _ = oracle.topk(obs[:, None, :], seq_list, k, force_last=True)
    for gg in range(G):
        assert np.array_equal(idx[:, gg].cpu().numpy(), oidx[:, 0])
        assert np.array_equal(cnt[:, gg].cpu().numpy(), ocnt[:, 0])


def test_exp_exhaustive_bit_identity(oracle):
    """O3 exhaustively: every float32 in [-87.5, -0] (1,118,765,057 values) through the device
    exp -- scalar spc_exp_dev and the packed f32x2 form the NORM / GROUP / select kernels run
    -- is bit-identical to the oracle's spcref_exp."""
    import ctypes
    L = spc.lib()
    L.spc_debug_exp.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int,
                                ctypes.c_void_p]
    dev = torch.device("cuda")
    lo = 0x80000000
    hi = int(np.frombuffer(np.float32(-87.5).tobytes(), np.uint32)[0])
    chunk = 1 << 24
    x_d = torch.empty(chunk, dtype=torch.float32, device=dev)
    y1 = torch.empty(chunk, dtype=torch.float32, device=dev)
    y2 = torch.empty(chunk, dtype=torch.float32, device=dev)
    total = 0
    for start in range(lo, hi + 1, chunk):
        n = min(chunk, hi + 1 - start)
        xb = np.arange(start, start + n, dtype=np.uint64).astype(np.uint32)
        x = xb.view(np.float32)
        x_d[:n].copy_(torch.from_numpy(x))
        for packed, y in ((0, y1), (1, y2)):
            assert L.spc_debug_exp(x_d.data_ptr(), y.data_ptr(), n, packed, None) == 0
        want = oracle.exp_array(x).view(np.uint32)
        torch.cuda.synchronize()
        assert np.array_equal(y1[:n].cpu().numpy().view(np.uint32), want), hex(start)
        assert np.array_equal(y2[:n].cpu().numpy().view(np.uint32), want), hex(start)
        total += n
    assert total == hi - lo + 1 == 1118765057
