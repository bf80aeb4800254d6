"""GPU parity of spc_sparse_decode_attn (O10) and spc_attn_merge (O12) against the fp64 CPU
oracle: max-abs error <= 2e-3 for bf16 inputs and <= 1e-5 for fp32 inputs (north star);
INDEXED and SLOTS modes; ragged / empty / full selections; k = S equals dense attention."""
import math

import numpy as np
import pytest
import torch

from paper_2512_00722_b200 import spc, synth

pytestmark = pytest.mark.gpu
DEV = "cuda"
TOL = {torch.bfloat16: 2e-3, torch.float32: 1e-5}


def host_bits(t):
    return synth.bf16_bits(t) if t.dtype == torch.bfloat16 else t.cpu().numpy()


def run_attn(q, kc, vc, idx, cnt, k, scale, mode=spc.KV_INDEXED, layers=None, impl="ptr"):
    """impl "ptr": spc_sparse_decode_attn (pointer tables, cp.async gathers); "tma":
    spc_sparse_decode_attn_kv (TMA descriptors, tile::gather4), bf16 only."""
    L, B, Hq, D = q.shape
    G = kc.shape[2]
    rows = kc.shape[3]
    out = torch.zeros((L, B, Hq, D), dtype=torch.float32, device=DEV)
    lse = torch.zeros((L, B, Hq), dtype=torch.float32, device=DEV)
    ws = spc.alloc_workspace(spc.attn_workspace(L, B, Hq, D, k), DEV)
    kd, vd = kc.to(DEV), vc.to(DEV)
    lb, le = (0, L) if layers is None else layers
    idx_d = None if idx is None else torch.as_tensor(idx).to(DEV)
    if impl == "tma":
        desc = spc.KvDesc([kd[l] for l in range(L)], [vd[l] for l in range(L)])
        spc.sparse_decode_attn_kv(desc, q.to(DEV), mode, idx_d, torch.as_tensor(cnt).to(DEV), k,
                                  scale, out, lse, ws, layer_begin=lb, layer_end=le)
    else:
        spc.sparse_decode_attn(q.to(DEV), spc.ptr_table([kd[l] for l in range(L)], DEV),
                               spc.ptr_table([vd[l] for l in range(L)], DEV), mode, idx_d,
                               torch.as_tensor(cnt).to(DEV), rows, k, scale, out, lse, ws, G,
                               layer_begin=lb, layer_end=le)
    torch.cuda.synchronize()
    return out.cpu().numpy(), lse.cpu().numpy()


def oracle_attn(oracle, q, kc, vc, idx, cnt, scale, layers=None):
    L = q.shape[0]
    qh = host_bits(q)
    kh, vh = host_bits(kc), host_bits(vc)
    return oracle.sparse_attn(qh, [kh[l] for l in range(L)], [vh[l] for l in range(L)], idx, cnt,
                              scale, layers=layers)


def random_selection(rng, B, G, rows, k, full=False):
    idx = np.full((B, G, k), -1, np.int32)
    cnt = np.zeros((B, G), np.int32)
    for b in range(B):
        for g in range(G):
            n = min(k, rows) if full else int(rng.integers(0, min(k, rows) + 1))
            if (b + g) == 0:
                n = min(k, rows)
            idx[b, g, :n] = np.sort(rng.choice(rows, n, replace=False))
            cnt[b, g] = n
    return idx, cnt


@pytest.mark.parametrize("dtype,impl", [(torch.bfloat16, "ptr"), (torch.float32, "ptr"),
                                        (torch.bfloat16, "tma")])
@pytest.mark.parametrize("D,alpha,G", [(128, 4, 2), (64, 4, 1), (128, 1, 3), (64, 8, 1), (128, 2, 2),
                                       (128, 8, 1)])
def test_attn_indexed_parity(oracle, dtype, impl, D, alpha, G):
    rng = np.random.default_rng(D * alpha + G)
    L, B, rows, k = 2, 2, 1500, 300  # 3 CTA chunks per (l, b, g), ragged last one
    Hq = alpha * G
    kc, vc = synth.llm_kv(L, B, G, rows, D, seed=D + alpha, dtype=dtype)
    q = synth.llm_queries(1, L, B, Hq, D, seed=D + alpha, dtype=dtype)[0]
    idx, cnt = random_selection(rng, B, G, rows, k)
    scale = 1.0 / math.sqrt(D)
    out, lse = run_attn(q, kc, vc, idx, cnt, k, scale, impl=impl)
    oo, ol = oracle_attn(oracle, q, kc, vc, idx, cnt, scale)
    err = np.abs(out - oo).max()
    assert err <= TOL[dtype], err
    fin = np.isfinite(ol)
    assert np.array_equal(fin, np.isfinite(lse))
    assert np.abs(lse[fin] - ol[fin]).max() <= 1e-4
    assert np.all(out[~np.broadcast_to(fin[..., None], out.shape)] == 0)  # empty selection


IMPLS = pytest.mark.parametrize("impl", ["ptr", "tma"])


@IMPLS
def test_attn_full_budget_equals_dense(oracle, impl):
    """k = S: sparse attention over every row equals dense attention (north-star invariant)."""
    L, B, G, Hq, D, S = 1, 1, 2, 8, 128, 777
    kc, vc = synth.llm_kv(L, B, G, S, D, seed=1)
    q = synth.llm_queries(1, L, B, Hq, D, seed=1)[0]
    idx = np.broadcast_to(np.arange(S, dtype=np.int32), (B, G, S)).copy()
    cnt = np.full((B, G), S, np.int32)
    out, lse = run_attn(q, kc, vc, idx, cnt, S, 0.088, impl=impl)
    dense = []
    qh, kh, vh = host_bits(q), host_bits(kc), host_bits(vc)
    for h in range(Hq):
        o, l = oracle.attn_head(qh[0, 0, h], kh[0, 0, h // 4], vh[0, 0, h // 4],
                                np.arange(S, dtype=np.int32), 0.088)
        dense.append(o)
    assert np.abs(out[0, 0] - np.stack(dense)).max() <= 2e-3


@IMPLS
def test_attn_slots_mode_and_layer_range(oracle, impl):
    L, B, G, Hq, D, k = 4, 1, 2, 8, 128, 256
    kb, vb = synth.llm_kv(L, B, G, k, D, seed=2)
    q = synth.llm_queries(1, L, B, Hq, D, seed=2)[0]
    cnt = np.array([[256, 100]], np.int32)
    idx = np.broadcast_to(np.arange(k, dtype=np.int32), (B, G, k)).copy()
    out, lse = run_attn(q, kb, vb, None, cnt, k, 0.1, mode=spc.KV_SLOTS, layers=(1, 3), impl=impl)
    oo, ol = oracle_attn(oracle, q, kb, vb, idx, cnt, 0.1, layers=range(1, 3))
    assert np.abs(out[1:3] - oo[1:3]).max() <= 2e-3
    assert np.abs(lse[1:3] - ol[1:3]).max() <= 1e-4
    assert np.all(out[0] == 0) and np.all(out[3] == 0)  # untouched layers


@IMPLS
def test_attn_concentrated_weights(oracle, impl):
    """One dominant key (p ~ 1): the bf16 hi/lo split of P keeps the error far below 2e-3."""
    L, B, G, Hq, D, S, k = 1, 1, 1, 4, 128, 600, 512
    kc, vc = synth.llm_kv(L, B, G, S, D, seed=3)
    q = synth.llm_queries(1, L, B, Hq, D, seed=3)[0]
    kc[0, 0, 0, 37] = (q[0, 0, 0].float() * 3).to(torch.bfloat16)
    vc = (vc.float() * 4).to(torch.bfloat16)
    idx = np.sort(np.random.default_rng(0).choice(S, k, replace=False)).astype(np.int32)
    idx[0] = 37
    idx = np.sort(idx)[None, None]
    cnt = np.array([[k]], np.int32)
    out, lse = run_attn(q, kc, vc, idx, cnt, k, 1.0, impl=impl)
    oo, ol = oracle_attn(oracle, q, kc, vc, idx, cnt, 1.0)
    assert np.abs(out - oo).max() <= 2e-3
    assert np.abs(lse - ol).max() <= 1e-4


def test_attn_merge_parity(oracle):
    rng = np.random.default_rng(5)
    P, n, D = 4, 37, 128
    o = rng.standard_normal((P, n, D)).astype(np.float32)
    l = (rng.standard_normal((P, n)) * 5).astype(np.float32)
    l[1, :5] = -np.inf
    l[:, 7] = -np.inf
    out = torch.zeros((n, D), dtype=torch.float32, device=DEV)
    lse = torch.zeros(n, dtype=torch.float32, device=DEV)
    spc.attn_merge(torch.from_numpy(o).to(DEV), torch.from_numpy(l).to(DEV), out, lse)
    torch.cuda.synchronize()
    oo, ol = oracle.attn_merge(o.astype(np.float64), l.astype(np.float64))
    assert np.abs(out.cpu().numpy() - oo).max() <= 1e-5
    fin = np.isfinite(ol)
    assert np.array_equal(np.isfinite(lse.cpu().numpy()), fin)
    assert np.abs(lse.cpu().numpy()[fin] - ol[fin]).max() <= 1e-5


@IMPLS
def test_attn_maximum_budget(oracle, impl):
    """k = SPC_MAX_K (4096) selected rows per (layer, b, g) out of 50,000, ragged counts
    (full / partial / one row), within the bf16 tolerance of the fp64 oracle."""
    rng = np.random.default_rng(4096)
    L, B, G, Hq, D, rows, k = 2, 1, 3, 12, 128, 50000, spc.MAX_K
    kc, vc = synth.llm_kv(L, B, G, rows, D, seed=40)
    q = synth.llm_queries(1, L, B, Hq, D, seed=40)[0]
    idx = np.full((B, G, k), -1, np.int32)
    cnt = np.array([[k, 2345, 1]], np.int32)
    for g in range(G):
        idx[0, g, :cnt[0, g]] = np.sort(rng.choice(rows, cnt[0, g], replace=False))
    out, lse = run_attn(q, kc, vc, idx, cnt, k, 1.0 / math.sqrt(D), impl=impl)
    oo, ol = oracle_attn(oracle, q, kc, vc, idx, cnt, 1.0 / math.sqrt(D))
    assert np.abs(out - oo).max() <= TOL[torch.bfloat16]
    assert np.abs(lse - ol).max() <= 1e-4
