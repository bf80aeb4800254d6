"""NEXT-4: the LLM decode step around the hot path (paper_2512_00722_b200/llm.py,
csrc/llm.cu).  Each spc_llm_* kernel against a plain PyTorch fp32/fp64 CPU reference of the
same operation (bit-exact where the operation is a rounding or an argmax, else within a
bound derived from its arithmetic), then whole decode steps of a small Llama-style model --
resident KV, offloaded KV with and without the prefetch stream, eager and CUDA-graph --
against a CPU reference forward that takes the selection from the oracle: the selection
bit-exact, the appended K/V rows, logits and next tokens within tolerance."""
import numpy as np
import pytest
import torch

from paper_2512_00722_b200 import rope, spc, synth
from paper_2512_00722_b200.llm import LlmDecoder

pytestmark = pytest.mark.gpu
DEV = "cuda"


def bf(x):
    """round to bf16 (RN-even) and back to f32"""
    return x.to(torch.bfloat16).to(torch.float32)


def ref_rmsnorm(h, w, eps):
    """HF Llama RMSNorm: bf16(w * bf16(h * r)), r = 1/sqrt(mean(h^2) + eps); h f32."""
    r = 1.0 / torch.sqrt((h.double() ** 2).mean(-1, keepdim=True) + eps)
    return bf(w.float() * bf((h.double() * r).float()))


def ref_rope(x, p, inv):
    """rotate_half RoPE of x [n][D] (f32) at position p, angle fl32(p * inv_freq)."""
    D = x.shape[-1]
    a = (torch.tensor(float(p), dtype=torch.float32) * inv).double()
    c, s = torch.cos(a), torch.sin(a)
    u, v = x[..., :D // 2].double(), x[..., D // 2:].double()
    return bf(torch.cat([u * c - v * s, v * c + u * s], -1).float())


# ------------------------------------------------------------------ kernels one by one
def test_llm_embed_and_add_rmsnorm():
    B, V, H = 3, 50, 4096 + 64
    emb = synth.normal_bf16((V, H), 1, device=DEV)
    tok = torch.tensor([7, 0, V - 1], dtype=torch.int32, device=DEV)
    h = torch.empty((B, H), dtype=torch.float32, device=DEV)
    spc.llm_embed(tok, emb, h)
    w = (1 + 0.05 * synth.normal_bf16((H,), 2, device=DEV, dtype=torch.float32)).to(torch.bfloat16)
    d = synth.normal_bf16((B, H), 3, device=DEV)
    xn = torch.empty((B, H), dtype=torch.bfloat16, device=DEV)
    spc.llm_add_rmsnorm(h, d, w, 1e-5, xn)
    torch.cuda.synchronize()
    h0 = emb.cpu().float()[tok.cpu().long()]
    h_ref = h0 + d.cpu().float()
    assert torch.equal(h.cpu(), h_ref)  # the residual add is one fp32 add: exact
    ref = ref_rmsnorm(h_ref, w.cpu(), 1e-5)
    # r differs from the fp64 reference by a few fp32 ulps (block-sum order, rsqrtf): the
    # bf16 outputs agree except at rounding boundaries, by at most one bf16 ulp
    got = xn.cpu().float()
    ulp = torch.abs(ref) * 2.0 ** -7
    assert (torch.abs(got - ref) <= ulp + 1e-30).all()
    assert (got != ref).float().mean() < 0.01
    spc.llm_add_rmsnorm(h, None, w, 1e-5, xn)  # delta NULL: h unchanged
    torch.cuda.synchronize()
    assert torch.equal(h.cpu(), h_ref)


def test_llm_embed_out_of_range_token_gives_zeros():
    emb = synth.normal_bf16((10, 64), 1, device=DEV)
    h = torch.full((2, 64), 5.0, device=DEV)
    spc.llm_embed(torch.tensor([3, 10], dtype=torch.int32, device=DEV), emb, h)
    torch.cuda.synchronize()
    assert torch.equal(h[0].cpu(), emb[3].cpu().float()) and (h[1] == 0).all()


def test_llm_f32_to_bf16_is_rn_even():
    g = torch.Generator().manual_seed(4)
    x = torch.randn(100003, generator=g) * 10.0 ** torch.randint(-30, 30, (100003,), generator=g)
    # exact halfway cases, both parities, and signed zeros / infinities
    halves = torch.tensor([0x3F808000, 0x3F818000, 0xBF808000, 0x7F7F8000 - 0x10000, 0x80000000,
                           0x7F800000, 0xFF800000, 0x7FFFFFFF, 0x7F800001], dtype=torch.int64).to(torch.int32).view(torch.float32)
    x = torch.cat([x, halves])
    y = torch.empty(x.numel(), dtype=torch.bfloat16, device=DEV)
    spc.llm_f32_to_bf16(x.to(DEV), y)
    torch.cuda.synchronize()
    got, ref = y.cpu().view(torch.int16), x.to(torch.bfloat16).view(torch.int16)
    nan = torch.isnan(x)
    assert torch.equal(got[~nan], ref[~nan]) and torch.isnan(y.cpu()[nan].float()).all()


def test_llm_swiglu():
    B, F = 2, 14336 + 40
    gu = synth.normal_bf16((B, 2 * F), 5, device=DEV).mul_(3.0)
    y = torch.empty((B, F), dtype=torch.bfloat16, device=DEV)
    spc.llm_swiglu(gu, y)
    torch.cuda.synchronize()
    g, u = gu.cpu().double()[:, :F], gu.cpu().double()[:, F:]
    ref = (g / (1 + torch.exp(-g)) * u)
    got = y.cpu().double()
    # __expf and the fp32 division: a few fp32 ulps before the bf16 rounding
    assert (torch.abs(got - ref) <= torch.abs(ref) * 2.0 ** -7 + 1e-6).all()


@pytest.mark.parametrize("slots", [False, True])
def test_llm_rope_append(slots):
    B, Hq, G, D, rows, k = 2, 8, 2, 128, 300, 16
    inv, _ = rope.yarn_inv_freq(D)
    inv_d = torch.from_numpy(inv).to(DEV)
    qkv = synth.normal_bf16((B, (Hq + 2 * G) * D), 6, device=DEV)
    seq = torch.tensor([1, 299], dtype=torch.int32, device=DEV)  # positions 0 and 298
    q = torch.zeros((B, Hq, D), dtype=torch.bfloat16, device=DEV)
    kc = torch.zeros((B, G, rows, D), dtype=torch.bfloat16, device=DEV)
    vc = torch.zeros_like(kc)
    kw = {}
    if slots:
        st = torch.full((B, G, k), -1, dtype=torch.int32, device=DEV)
        st[0, 0, 5] = 0     # token 0 in slot 5 of (0, 0)
        st[1, 1, 15] = 298  # token 298 in slot 15 of (1, 1); the other groups: not resident
        st[1, 0, 3] = 297
        kb = torch.zeros((B, G, k, D), dtype=torch.bfloat16, device=DEV)
        vb = torch.zeros_like(kb)
        kw = dict(slot_tok=st, k_buf=kb, v_buf=vb)
    spc.llm_rope_append(qkv, inv_d, seq, Hq, G, q, kc, vc, **kw)
    torch.cuda.synchronize()
    x = qkv.cpu().float().view(B, Hq + 2 * G, D)
    invc = torch.from_numpy(inv)
    for b, p in enumerate([0, 298]):
        qr = ref_rope(x[b, :Hq], p, invc)
        kr = ref_rope(x[b, Hq:Hq + G], p, invc)
        # sincosf / fp32 products vs fp64: at most one bf16 ulp at rounding boundaries
        for got, ref in ((q[b].cpu().float(), qr), (kc[b, :, p].cpu().float(), kr)):
            assert (torch.abs(got - ref) <= torch.abs(ref) * 2.0 ** -7 + 1e-6).all()
        assert torch.equal(vc[b, :, p].cpu().float(), x[b, Hq + G:])  # copied
        assert kc[b, :, :p].abs().sum() == 0 and kc[b, :, p + 1:].abs().sum() == 0
    if slots:
        assert torch.equal(kb[0, 0, 5], kc[0, 0, 0]) and torch.equal(vb[0, 0, 5], vc[0, 0, 0])
        assert torch.equal(kb[1, 1, 15], kc[1, 1, 298]) and torch.equal(vb[1, 1, 15], vc[1, 1, 298])
        kb[0, 0, 5] = 0
        kb[1, 1, 15] = 0
        vb[0, 0, 5] = 0
        vb[1, 1, 15] = 0
        assert kb.abs().sum() == 0 and vb.abs().sum() == 0  # nothing else written


def test_llm_argmax_lowest_index_on_ties_and_advances_seq_len():
    B, V = 4, 128256
    lg = synth.normal_bf16((B, V), 7, device=DEV)
    lg[1, 1000] = 30.0
    lg[1, 77] = 30.0  # tie: the lowest index wins
    lg[2, :] = -5.0  # all equal: index 0
    lg[3, :] = float("nan")
    lg[3, V - 1] = -100.0  # NaN never wins
    tok = torch.zeros(B, dtype=torch.int32, device=DEV)
    seq = torch.tensor([5, 6, 7, 8], dtype=torch.int32, device=DEV)
    spc.llm_argmax(lg, tok, seq)
    torch.cuda.synchronize()
    x = lg.cpu().float()
    ref = []
    for b in range(B):
        m = torch.nan_to_num(x[b], nan=-float("inf")).max()
        ref.append(int(torch.nonzero(x[b] == m)[0]))
    assert tok.cpu().tolist() == ref and ref[1] == 77 and ref[2] == 0 and ref[3] == V - 1
    assert seq.cpu().tolist() == [6, 7, 8, 9]


# ------------------------------------------------------------------ whole decode steps
CFG = dict(L=2, H=256, Hq=4, G=2, D=64, F=512, V=1000, rope_base=500000.0, eps=1e-5)


class RefLlm:
    """Plain PyTorch CPU reference of the decoder forward of llm.py (fp32 GEMMs, fp64
    softmax), with the same bf16 rounding points; its own copies of the K/V caches."""

    def __init__(self, w, kc, vc):
        self.w = {k: ([t.cpu().float() for t in v] if isinstance(v, list) else v.cpu().float())
                  for k, v in w.items()}
        self.K = [t.cpu().float().clone() for t in kc]
        self.V = [t.cpu().float().clone() for t in vc]

    def step(self, tok, pos, idx, cnt, inv, scale):
        c, w = CFG, self.w
        Hq, G, D = c["Hq"], c["G"], c["D"]
        B = len(tok)
        h = w["emb"][torch.tensor(tok).long()].clone()
        q_all = []
        for l in range(c["L"]):
            xn = ref_rmsnorm(h, w["ln1"][l], c["eps"])
            qkv = bf(xn @ w["w_qkv"][l].T).view(B, Hq + 2 * G, D)
            a = torch.zeros(B, Hq, D)
            for b in range(B):
                p = pos[b]
                q = ref_rope(qkv[b, :Hq], p, inv)
                self.K[l][b, :, p] = ref_rope(qkv[b, Hq:Hq + G], p, inv)
                self.V[l][b, :, p] = qkv[b, Hq + G:]
                for hh in range(Hq):
                    g = hh // (Hq // G)
                    J = torch.from_numpy(idx[b, g, :cnt[b, g]].astype(np.int64))
                    Kj, Vj = self.K[l][b, g, J].double(), self.V[l][b, g, J].double()
                    z = scale * (Kj @ q[hh].double())
                    pr = torch.softmax(z, 0)
                    a[b, hh] = (pr @ Vj).float()
                q_all.append(q)
            o = bf(bf(a.view(B, Hq * D)) @ w["w_o"][l].T)
            h = h + o
            xn = ref_rmsnorm(h, w["ln2"][l], c["eps"])
            gu = bf(xn @ w["w_gu"][l].T)
            F = c["F"]
            gg, uu = gu[:, :F].double(), gu[:, F:].double()
            y = bf((gg / (1 + torch.exp(-gg)) * uu).float())
            h = h + bf(y @ w["w_down"][l].T)
        xn = ref_rmsnorm(h, w["norm"], c["eps"])
        return bf(xn @ w["lm_head"].T)


def make_model(B, Smax, S0, kv, seed):
    c = CFG
    L, H, Hq, G, D, F, V = (c[x] for x in ("L", "H", "Hq", "G", "D", "F", "V"))
    w = synth.llm_weights(L, H, Hq, G, D, F, V, seed, device=DEV)
    _, nw, w_qk = synth.retrieval_head_weights(V, H, Hq, G, D, seed, device=DEV)
    inv_r, ms = rope.yarn_inv_freq(D, factor=8.0)
    ret = dict(emb=w["emb"], norm_w=nw, w_qk=w_qk, inv_freq=torch.from_numpy(inv_r).to(DEV),
               mscale=ms)
    kr = synth.retrieval_keys(B, G, Smax, D, seed=seed, device=DEV)
    kc, vc = synth.llm_kv(L, B, G, Smax, D, seed=seed, device=DEV)
    kc[:, :, :, S0:] = 0
    vc[:, :, :, S0:] = 0
    kr[:, :, S0:] = 0
    if kv == "offload":
        kc, vc = kc.cpu().pin_memory(), vc.cpu().pin_memory()
    return w, ret, kr, kc, vc


@pytest.mark.parametrize("kv,prefetch,graph", [("resident", True, False), ("resident", True, True),
                                               ("offload", False, False), ("offload", True, True)])
def test_llm_decode_steps_match_reference(oracle, kv, prefetch, graph):
    B, Smax, k, steps = 2, 640, 64, 4
    S0 = [500, 333]
    w, ret, kr, kc, vc = make_model(B, Smax, max(S0), kv, seed=41)
    seq = torch.tensor([s + 1 for s in S0], dtype=torch.int32, device=DEV)
    dec = LlmDecoder(w, CFG, ret, kr, [kc[l] for l in range(CFG["L"])],
                     [vc[l] for l in range(CFG["L"])], seq, k, kv=kv, prefetch=prefetch)
    ref = RefLlm(w, [kc[l] for l in range(CFG["L"])], [vc[l] for l in range(CFG["L"])])
    tok = synth.tokens(1, B, CFG["V"], 41)[0]
    dec.reset(tok.to(DEV), seq.clone())
    inv = torch.from_numpy(rope.yarn_inv_freq(CFG["D"])[0])
    cur = tok.tolist()
    compared = 0
    for s in range(steps):
        pos = [S0[b] + s for b in range(B)]
        p = dec.parity
        if graph and s == 1:
            dec.capture()
        out_tok = dec.step(use_graph=graph and s >= 1)
        torch.cuda.synchronize()
        st = dec.st
        assert dec.seq_len.cpu().tolist() == [x + 2 for x in pos]
        # the selection: the oracle's on the GPU-appended retrieval cache (its front-end is
        # checked in test_gpu_rethead); then the reference forward with the oracle's sets
        lens = [x + 1 for x in pos]
        _, _, _, gs = oracle.score(synth.bf16_bits(st.q_rets[p]), synth.bf16_bits(st.kr), lens,
                                   CFG["G"], st.scale)
        oidx, _, ocnt, _ = oracle.topk(gs, lens, k, force_last=True)
        assert np.array_equal(st.idx[p].cpu().numpy(), oidx)
        assert np.array_equal(st.cnt[p].cpu().numpy(), ocnt)
        lg_ref = ref.step(cur, pos, oidx, ocnt, inv, dec.scale)
        lg = dec.logits.cpu().float()
        scale_ = lg_ref.abs().max().item()
        assert (lg - lg_ref).abs().max().item() <= 3e-2 * scale_, s
        for l in range(CFG["L"]):  # the appended rows
            for b in range(B):
                for cache, rc in ((dec.k_cache[l], ref.K[l]), (dec.v_cache[l], ref.V[l])):
                    got = cache[b, :, pos[b]].cpu().float()
                    r = rc[b, :, pos[b]]
                    assert (got - r).abs().max() <= 3e-2 * r.abs().max() + 1e-3
        if kv == "offload":  # the new token's rows are in its budget slot
            slot_tok = st.slot_tok.cpu()
            for l in range(CFG["L"]):
                for b in range(B):
                    for g in range(CFG["G"]):
                        sl = int(torch.nonzero(slot_tok[b, g] == pos[b])[0])
                        assert torch.equal(dec.kb[l, b, g, sl].cpu(), dec.k_cache[l][b, g, pos[b]])
                        assert torch.equal(dec.vb[l, b, g, sl].cpu(), dec.v_cache[l][b, g, pos[b]])
        top2 = torch.topk(lg_ref, 2, dim=-1).values
        nxt = out_tok.cpu().tolist()
        ref_nxt = lg_ref.argmax(-1).tolist()
        # the GPU logits are within e of the reference: the argmax is determined wherever the
        # reference's top-2 margin exceeds 2e; below that the sequences may legitimately split
        e = (lg - lg_ref).abs().max().item()
        if ((top2[:, 0] - top2[:, 1]) <= 2 * e).any():
            break
        assert nxt == ref_nxt, s
        # and the device argmax of its own logits, exactly
        assert nxt == [int(torch.nonzero(lg[b] == lg[b].max())[0]) for b in range(B)]
        cur = nxt
        compared += 1
    assert compared >= 2
