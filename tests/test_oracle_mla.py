"""NEXT-3 MLA select-then-expand oracle pins (Fig. 5(e)): against the O10 attention
oracle when the up-projections just pick latent dimensions, closed forms for one row and
equal rows, and linearity in W_UV.  CPU only."""
import numpy as np

import oracle

DC, DR = 512, 64


def bf(x):
    x = np.asarray(x, np.float32)
    u = ((x.view(np.uint32) + 0x8000) & 0xFFFF0000).astype(np.uint32)
    return (u >> 16).astype(np.uint16)


def vals(b):
    return (np.asarray(b, np.uint32) << 16).view(np.float32)


def test_selector_projections_reduce_to_plain_attention():
    """W_UK = W_UV = [I | 0] (keep the first DN latent dims) and q_pe = 0: MLA over the selected
    rows equals O10's attention with K = V = c[:, :DN] (an independent oracle function)."""
    rng = np.random.default_rng(0)
    S, DN = 300, 64
    cache = bf(rng.standard_normal((S, DC + DR)))
    eye = np.zeros((DN, DC), np.float32)
    eye[np.arange(DN), np.arange(DN)] = 1.0
    q = np.concatenate([rng.standard_normal(DN), np.zeros(DR)]).astype(np.float32)
    rows = np.sort(rng.choice(S, 40, replace=False)).astype(np.int32)
    o, lse = oracle.mla_head(bf(q), cache, bf(eye), bf(eye), rows, DC, DR, 0.125)
    kv = np.ascontiguousarray(cache[:, :DN])
    o2, lse2 = oracle.attn_head(bf(q)[:DN], kv, kv, rows, 0.125)
    assert np.allclose(o, o2, rtol=1e-12, atol=1e-12) and abs(lse - lse2) < 1e-12


def test_one_row_and_equal_rows():
    """One selected row: o = W_UV c_j, lse = its score; identical rows: o = W_UV c (mean)."""
    rng = np.random.default_rng(1)
    S, DN, DV = 10, 32, 48
    cache = bf(rng.standard_normal((S, DC + DR)) * 0.5)
    wuk, wuv = bf(rng.standard_normal((DN, DC)) * 0.05), bf(rng.standard_normal((DV, DC)) * 0.05)
    q = bf(rng.standard_normal(DN + DR))
    o, lse = oracle.mla_head(q, cache, wuk, wuv, [7], DC, DR, 0.1)
    c = vals(cache[7]).astype(np.float64)
    want = vals(wuv).astype(np.float64) @ c[:DC]
    score = 0.1 * (vals(q)[:DN] @ (vals(wuk).astype(np.float64) @ c[:DC]) + vals(q)[DN:] @ c[DC:])
    assert np.allclose(o, want, rtol=1e-12) and abs(lse - score) < 1e-9
    same = cache.copy()
    same[:] = cache[3]
    o3, _ = oracle.mla_head(q, same, wuk, wuv, [0, 4, 9], DC, DR, 0.1)
    want3 = vals(wuv).astype(np.float64) @ vals(cache[3]).astype(np.float64)[:DC]
    assert np.allclose(o3, want3, rtol=1e-12)
    o4, _ = oracle.mla_head(q, cache, wuk, wuv, [], DC, DR, 0.1)
    assert np.all(o4 == 0)


def test_linear_in_w_uv():
    rng = np.random.default_rng(2)
    S, DN, DV = 50, 64, 64
    cache = bf(rng.standard_normal((S, DC + DR)))
    wuk, wuv = bf(rng.standard_normal((DN, DC)) * 0.04), bf(rng.standard_normal((DV, DC)) * 0.04)
    q = bf(rng.standard_normal(DN + DR))
    rows = np.arange(0, S, 3, dtype=np.int32)
    o, l1 = oracle.mla_head(q, cache, wuk, wuv, rows, DC, DR, 0.07)
    o2, l2 = oracle.mla_head(q, cache, wuk, bf(2 * vals(wuv)), rows, DC, DR, 0.07)
    assert np.array_equal(o2, 2 * o) and l1 == l2
