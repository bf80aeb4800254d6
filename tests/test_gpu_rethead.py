"""GPU parity of spc_rethead_qk (NEXT-1: embedding -> RMSNorm -> Q/K projection -> RoPE ->
K append) against the CPU oracle, end to end from the token ids.  The normalised input xn
equals the oracle's bit for bit (reading R22: the sum of squares is an exact fixed-point
integer sum on both sides); q and the appended key row are checked against the oracle's
fp64 projection + rotation of the ORACLE's xn, within a rigorous bound: bf16 output rounding
(2^-8 |ref|) + fp32 accumulation over H terms ((H + 16) 2^-24 mscale (sum|W_u x| +
sum|W_v x|)), times 4 for the tensor-core path of B > 4 (fp32 MMA accumulation: exact
products, sums within ~2 ulps)."""
import numpy as np
import pytest
import torch

import oracle
from paper_2512_00722_b200 import rope, spc, synth

pytestmark = pytest.mark.gpu
DEV = "cuda"


def run(B, H, Hq, G, D, V, Smax, pos, factor=1.0, seed=1, norm=True):
    emb, norm_w, w_qk = synth.retrieval_head_weights(V, H, Hq, G, D, seed, device=DEV)
    inv, m = rope.yarn_inv_freq(D, factor=factor, orig_ctx=2048)
    inv_d = torch.from_numpy(inv).to(DEV)
    tok = synth.tokens(1, B, V, seed, device=DEV)[0].contiguous()
    pos_d = torch.tensor(pos, dtype=torch.int32, device=DEV)
    q = torch.full((B, Hq, D), -7.0, dtype=torch.bfloat16, device=DEV)
    kr = torch.full((B, G, Smax, D), 3.0, dtype=torch.bfloat16, device=DEV)
    sl = torch.zeros(B, dtype=torch.int32, device=DEV)
    xo = torch.zeros((B, H), dtype=torch.bfloat16, device=DEV)
    spc.rethead_qk(tok, emb, norm_w if norm else None, 1e-5, w_qk, inv_d, m, pos_d, Hq, G, q, kr,
                   seq_len_out=sl, x_out=xo)
    torch.cuda.synchronize()
    return emb, norm_w if norm else None, w_qk, inv, m, tok, q, kr, sl, xo


@pytest.mark.parametrize("B,H,Hq,G,D,V,Smax,pos,factor", [
    (1, 4096, 32, 8, 128, 1000, 64, [37], 1.0),             # config-B retrieval-head shape
    (3, 512, 8, 2, 64, 300, 50, [0, 49, 7], 4.0),           # D = 64, pos 0 and Smax-1
    (16, 1024, 4, 1, 128, 64, 40, list(range(0, 40, 40 // 16 + 1))[:16] + [39] * 0, 32.0),
    (2, 2048, 16, 2, 128, 50, 1 << 20, [1_000_000, 1], 64.0),  # 1M positions (config E)
    (8, 4096, 32, 8, 128, 300, 64, [63, 0, 5, 9, 11, 2, 40, 41], 64.0),  # tensor-core path
    (12, 4096, 16, 4, 64, 300, 128, list(range(3, 120, 10)), 8.0),      # two n-tiles, D = 64
])
def test_rethead_matches_oracle(B, H, Hq, G, D, V, Smax, pos, factor):
    pos = (pos + [5] * B)[:B]
    emb, nw, w_qk, inv, m, tok, q, kr, sl, xo = run(B, H, Hq, G, D, V, Smax, pos, factor)
    # xn: the normalisation step
    x_rows = synth.bf16_bits(emb)[tok.cpu().numpy()]
    xn_ref = oracle.rmsnorm_bf16(x_rows, None if nw is None else synth.bf16_bits(nw), 1e-5)
    assert np.array_equal(synth.bf16_bits(xo), xn_ref)  # R22: bit-exact
    # projection + RoPE from the oracle's xn (token -> q / k end to end)
    out, bound = oracle.rethead_qk(synth.bf16_bits(w_qk), xn_ref, inv, pos, D, mscale=m)
    half = D // 2
    bnd = bound.reshape(B, Hq + G, 2, half)
    pair = np.concatenate([bnd.sum(2, keepdims=True)] * 2, axis=2).reshape(B, -1)
    acc = 4.0 if B > 4 else 1.0
    tol = 2.0 ** -8 * np.abs(out) + acc * (H + 16) * 2.0 ** -24 * m * pair
    got_q = q.float().cpu().numpy().reshape(B, Hq * D)
    got_k = np.stack([kr[b, :, pos[b]].float().cpu().numpy().reshape(-1) for b in range(B)])
    got = np.concatenate([got_q, got_k], axis=1)
    err = np.abs(got - out)
    assert np.all(err <= tol), f"max err {err.max():.3e}, worst excess {(err - tol).max():.3e}"
    assert np.median(err / np.maximum(np.abs(out), 1e-30)) < 2.0 ** -9
    # only row pos[b] of the key cache changed; seq_len_out = pos + 1
    for b in range(B):
        changed = (kr[b] != 3.0).any(dim=2).any(dim=0).nonzero().flatten().cpu().tolist()
        assert set(changed) <= {pos[b]}
    assert sl.cpu().tolist() == [p + 1 for p in pos]


def test_rethead_unit_norm_weight_and_errors():
    """norm_w = NULL is the unit weight; host-side argument errors come back before launch."""
    B, H, Hq, G, D, V = 2, 256, 4, 2, 64, 20
    emb, _, w_qk, inv, m, tok, q, kr, sl, xo = run(B, H, Hq, G, D, V, 8, [1, 2], norm=False)
    xn_ref = oracle.rmsnorm_bf16(synth.bf16_bits(emb)[tok.cpu().numpy()], None, 1e-5)
    assert np.array_equal(synth.bf16_bits(xo), xn_ref)
    with pytest.raises(spc.SpcError):  # B > 16
        spc.rethead_qk(torch.zeros(17, dtype=torch.int32, device=DEV), emb, None, 1e-5, w_qk,
                       torch.from_numpy(inv).to(DEV), m, torch.zeros(17, dtype=torch.int32,
                                                                      device=DEV),
                       Hq, G, torch.zeros((17, Hq, D), dtype=torch.bfloat16, device=DEV),
                       torch.zeros((17, G, 8, D), dtype=torch.bfloat16, device=DEV))
