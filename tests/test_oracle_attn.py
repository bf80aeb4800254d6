"""Pins for O10 (sparse attention), O11 (dense) and O12 (LSE merge).

Eq.1 restricted to the selected rows, renormalised over them
(reading R15).  Pins: torch's fp64 scaled_dot_product_attention (a library
routine) on the gathered rows; k = S equals dense bit-for-bit; S = 1 gives
V_0; equal keys give the mean of V_J; a dominant logit gives V_j*; merging the
attention of disjoint parts equals attention over the union; an empty part is
neutral.
"""
import numpy as np
import torch

from paper_2512_00722_b200 import synth


def case(S, D, seed, dtype=torch.bfloat16):
    g = torch.Generator().manual_seed(seed)
    q = torch.randn(D, generator=g).to(dtype)
    k = torch.randn(S, D, generator=g).to(dtype)
    v = torch.randn(S, D, generator=g).to(dtype)
    return q, k, v


def bits(t):
    return synth.bf16_bits(t) if t.dtype == torch.bfloat16 else t.numpy()


def test_attn_vs_torch_sdpa(oracle):
    for dt in (torch.bfloat16, torch.float32):
        q, k, v = case(500, 128, 1, dt)
        rows = np.sort(np.random.default_rng(0).choice(500, 77, replace=False)).astype(np.int32)
        out, lse = oracle.attn_head(bits(q), bits(k), bits(v), rows, 0.125)
        qd, kd, vd = q.double(), k.double()[rows], v.double()[rows]
        ref = torch.nn.functional.scaled_dot_product_attention(
            qd[None, None, None], kd[None, None], vd[None, None], scale=0.125)[0, 0, 0]
        assert np.allclose(out, ref.numpy(), atol=1e-12, rtol=0)
        z = (kd @ qd) * 0.125
        assert abs(lse - torch.logsumexp(z, 0).item()) < 1e-12


def test_full_budget_equals_dense_bitwise(oracle):
    q, k, v = case(300, 64, 2)
    dense, l1 = oracle.attn_head(bits(q), bits(k), bits(v), np.arange(300, dtype=np.int32), 0.125)
    sparse, l2 = oracle.attn_head(bits(q), bits(k), bits(v), np.arange(300, dtype=np.int32), 0.125)
    assert np.array_equal(dense, sparse) and l1 == l2


def test_single_row_equal_keys_dominant(oracle):
    q, k, v = case(10, 64, 3)
    vb = bits(v)
    vf = (vb.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    out, _ = oracle.attn_head(bits(q), bits(k), vb, np.array([4], np.int32), 0.125)
    assert np.array_equal(out, vf[4])  # S = 1 -> V_0
    keq = bits(k[:1].repeat(10, 1))
    out, lse = oracle.attn_head(bits(q), keq, vb, np.arange(10, dtype=np.int32), 0.125)
    assert np.allclose(out, vf.mean(axis=0), atol=1e-14)
    kdom = k.clone()
    kdom[7] = q * 100
    out, _ = oracle.attn_head(bits(q), bits(kdom), vb, np.arange(10, dtype=np.int32), 0.125)
    assert np.allclose(out, vf[7], atol=1e-12)


def test_empty_selection(oracle):
    q, k, v = case(5, 64, 4)
    out, lse = oracle.attn_head(bits(q), bits(k), bits(v), np.zeros(0, np.int32), 0.125)
    assert lse == -np.inf and not out.any()


def test_merge_of_disjoint_parts_equals_union(oracle):
    q, k, v = case(400, 128, 5)
    rng = np.random.default_rng(6)
    J = np.sort(rng.choice(400, 200, replace=False)).astype(np.int32)
    full, lfull = oracle.attn_head(bits(q), bits(k), bits(v), J, 0.088)
    for P in (1, 2, 3, 8):
        owner = rng.integers(0, P, len(J))
        owner[:1] = 0
        parts = [oracle.attn_head(bits(q), bits(k), bits(v), J[owner == p], 0.088) for p in range(P)]
        o = np.stack([p[0] for p in parts])[:, None]
        l = np.array([p[1] for p in parts])[:, None]
        out, lse = oracle.attn_merge(o, l)
        assert np.allclose(out[0], full, atol=1e-12), P
        assert abs(lse[0] - lfull) < 1e-12
    # all parts empty
    out, lse = oracle.attn_merge(np.zeros((2, 1, 4)), np.full((2, 1), -np.inf))
    assert lse[0] == -np.inf and not out.any()
