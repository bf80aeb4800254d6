"""CPU oracle for the SpeContext hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product package
``paper_2512_00722_b200`` never imports it and shares no code with it.

This module is a thin ctypes loader over ``spcref.c`` (plain C, see its header
for the paper citations and DESIGN.md §3 for the contract O1..O13) plus numpy
marshalling.  No arithmetic of the method lives in Python here except the
row loops that call the C functions.

Parity pins (what ties each function to something other than itself) are in
``tests/test_oracle_*.py``; every function here is pinned.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "spcref.c")
_LIB = os.path.join(_HERE, "libspcref.so")
CFLAGS = ["-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math",
          "-fno-unsafe-math-optimizations", "-Wall"]


def build(force: bool = False) -> str:
    """Compile spcref.c with gcc (no contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "spcref.h"))):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i32, i64, f32, f64, u32 = (ctypes.c_int, ctypes.c_int64, ctypes.c_float, ctypes.c_double,
                                   ctypes.c_uint32)
        L.spcref_exp.argtypes = [f32]
        L.spcref_exp.restype = f32
        L.spcref_exp_array.argtypes = [P, P, ctypes.c_longlong]
        L.spcref_exp_max_ulp.argtypes = [u32, u32, P]
        L.spcref_exp_max_ulp.restype = f64
        L.spcref_logits.argtypes = [P, P, P, i32, i32, i32, i32, i32, f32, P, P]
        L.spcref_norm.argtypes = [P, P, P, i32, i32, i32, P]
        L.spcref_group.argtypes = [P, P, P, P, i32, i32, i32, i32, P]
        L.spcref_group_score_f64.argtypes = [P, P, P, i32, i32, i32, i32, i32, f64, P]
        L.spcref_topk_row.argtypes = [P, P, i32, i32, i32, i32, i32, P, P, P]
        L.spcref_topk_row.restype = i32
        L.spcref_rmsnorm_bf16.argtypes = [P, P, i32, f64, P]
        L.spcref_rethead_qk.argtypes = [P, i32, i32, P, P, i32, i32, f64, P, P]
        L.spcref_plan_mem.argtypes = [i64, f64, i32, i32, i32, i32, i32, i64, i32, i64, i32]
        L.spcref_plan_mem.restype = i64
        L.spcref_plan_thresholds_search.argtypes = [i64, i64, f64, i32, i32, i32, i32, i32, i64, i32,
                                                    i64, P]
        L.spcref_plan_max_resident.argtypes = [i64, i64, f64, i32, i32, i32, i32, i32, i64, i32, i64]
        L.spcref_plan_max_resident.restype = i32
        L.spcref_plan_step.argtypes = [P, i32, i64, i32, P, P]
        L.spcref_plan_step.restype = i32
        L.spcref_batch_score.argtypes = [P, P, P, P, i32, i32, i32, P]
        L.spcref_mla_head.argtypes = [P, P, P, P, P, i32, i32, i32, i32, i32, f64, P]
        L.spcref_mla_head.restype = f64
        L.spcref_composite.argtypes = [f32, ctypes.c_int32]
        L.spcref_composite.restype = ctypes.c_uint64
        L.spcref_elastic_diff_row.argtypes = [P, i32, P, i32, i32, P, P, P, P, P, P]
        L.spcref_elastic_diff_row.restype = i32
        L.spcref_attn_head.argtypes = [P, P, P, i32, P, i32, i32, f64, P]
        L.spcref_attn_head.restype = f64
        L.spcref_attn_merge_row.argtypes = [P, P, i32, i32, P]
        L.spcref_attn_merge_row.restype = f64
        del i64
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "oracle inputs must be C-contiguous"
    return a.ctypes.data_as(ctypes.c_void_p)


def _bf16_bits(a) -> np.ndarray:
    a = np.asarray(a)
    if a.dtype == np.uint16:
        return np.ascontiguousarray(a)
    if a.dtype == np.int16:
        return np.ascontiguousarray(a.view(np.uint16))
    raise TypeError("bf16 tensors are passed to the oracle as uint16 bit patterns")


# ---------------------------------------------------------------- O3
def spc_exp(x: float) -> float:
    return float(lib().spcref_exp(ctypes.c_float(x)))


def exp_array(x):
    """O3 over a float32 array (spcref_exp elementwise)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    y = np.empty_like(x)
    lib().spcref_exp_array(_p(x), _p(y), x.size)
    return y


def exp_max_ulp(lo_bits: int, hi_bits: int):
    n_sub = ctypes.c_uint64(0)
    worst = lib().spcref_exp_max_ulp(lo_bits, hi_bits, ctypes.byref(n_sub))
    return float(worst), int(n_sub.value)


# ---------------------------------------------------------------- O1..O6
def logits(q, kr, seq_len, G: int, scale: float):
    """Phase LOGITS: returns (logits [B][Hq][Smax] f32, head_max [B][Hq] f32)."""
    q, kr = _bf16_bits(q), _bf16_bits(kr)
    B, Hq, D = q.shape
    Smax = kr.shape[2]
    assert kr.shape == (B, G, Smax, D)
    sl = np.ascontiguousarray(seq_len, dtype=np.int32)
    lg = np.zeros((B, Hq, Smax), np.float32)
    hm = np.zeros((B, Hq), np.float32)
    lib().spcref_logits(_p(q), _p(kr), _p(sl), B, Hq, G, D, Smax, ctypes.c_float(scale), _p(lg),
                        _p(hm))
    return lg, hm


def norm(lg, hm, seq_len):
    """Phase NORM: returns head_sumfix [B][Hq] int64."""
    B, Hq, Smax = lg.shape
    sl = np.ascontiguousarray(seq_len, dtype=np.int32)
    F = np.zeros((B, Hq), np.int64)
    lib().spcref_norm(_p(np.ascontiguousarray(lg)), _p(np.ascontiguousarray(hm)), _p(sl), B, Hq,
                      Smax, _p(F))
    return F


def group(lg, hm, F, seq_len, G: int):
    """Phase GROUP: returns group_score [B][G][Smax] f32."""
    B, Hq, Smax = lg.shape
    sl = np.ascontiguousarray(seq_len, dtype=np.int32)
    gs = np.zeros((B, G, Smax), np.float32)
    lib().spcref_group(_p(np.ascontiguousarray(lg)), _p(np.ascontiguousarray(hm)),
                       _p(np.ascontiguousarray(F, dtype=np.int64)), _p(sl), B, Hq, G, Smax, _p(gs))
    return gs


def score(q, kr, seq_len, G: int, scale: float):
    """O1..O6 end to end: (logits, head_max, head_sumfix, group_score)."""
    lg, hm = logits(q, kr, seq_len, G, scale)
    F = norm(lg, hm, seq_len)
    gs = group(lg, hm, F, seq_len, G)
    return lg, hm, F, gs


def group_score_f64(q, kr, seq_len, G: int, scale: float):
    q, kr = _bf16_bits(q), _bf16_bits(kr)
    B, Hq, D = q.shape
    Smax = kr.shape[2]
    sl = np.ascontiguousarray(seq_len, dtype=np.int32)
    gs = np.zeros((B, G, Smax), np.float64)
    lib().spcref_group_score_f64(_p(q), _p(kr), _p(sl), B, Hq, G, D, Smax, ctypes.c_double(scale),
                                 _p(gs))
    return gs


# ---------------------------------------------------------------- O7
def composite(value: float, gid: int) -> int:
    return int(lib().spcref_composite(ctypes.c_float(value), ctypes.c_int32(gid)))


def topk_row(val, k: int, force_pos: int = -1, id_stride: int = 1, id_offset: int = 0,
             cand_id=None):
    """Returns (positions ascending int32[cnt], values f32[cnt], thresh uint64)."""
    val = np.ascontiguousarray(val, dtype=np.float32)
    n = val.shape[0]
    pos = np.full(max(k, 1), -1, np.int32)
    out_val = np.zeros(max(k, 1), np.float32)
    th = ctypes.c_uint64(0)
    cid = None if cand_id is None else np.ascontiguousarray(cand_id, dtype=np.int32)
    cnt = lib().spcref_topk_row(_p(val), None if cid is None else _p(cid), n, k, force_pos,
                                id_stride, id_offset, _p(pos), _p(out_val), ctypes.byref(th))
    return pos[:cnt].copy(), out_val[:cnt].copy(), int(th.value)


def topk(gs, seq_len, k: int, force_last: bool = False, id_stride: int = 1, id_offset: int = 0):
    """Dense rows [B][G][n]: returns (idx [B][G][k] -1 padded, val [B][G][k], count [B][G],
    thresh [B][G] uint64)."""
    B, G, n = gs.shape
    idx = np.full((B, G, k), -1, np.int32)
    val = np.zeros((B, G, k), np.float32)
    cnt = np.zeros((B, G), np.int32)
    th = np.zeros((B, G), np.uint64)
    for b in range(B):
        ln = min(int(seq_len[b]), n)
        for g in range(G):
            p, v, t = topk_row(gs[b, g, :ln], k, ln - 1 if force_last else -1, id_stride, id_offset)
            idx[b, g, :len(p)] = p
            val[b, g, :len(p)] = v
            cnt[b, g] = len(p)
            th[b, g] = t
    return idx, val, cnt, th


# ---------------------------------------------------------------- O8
def elastic_diff_row(prev, cur, k: int, slot_tok=None):
    """Returns dict(load_tok, load_slot, evict_tok, n_load, n_evict, slot_tok, status)."""
    prev = np.ascontiguousarray(prev, dtype=np.int32)
    cur = np.ascontiguousarray(cur, dtype=np.int32)
    lt = np.full(k, -1, np.int32)
    ls = np.full(k, -1, np.int32)
    et = np.full(k, -1, np.int32)
    nl, ne = ctypes.c_int(0), ctypes.c_int(0)
    st = None if slot_tok is None else np.ascontiguousarray(slot_tok, dtype=np.int32).copy()
    rc = lib().spcref_elastic_diff_row(_p(prev) if len(prev) else None, len(prev),
                                       _p(cur) if len(cur) else None, len(cur), k,
                                       None if st is None else _p(st), _p(lt),
                                       None if st is None else _p(ls), ctypes.byref(nl), _p(et),
                                       ctypes.byref(ne))
    return dict(load_tok=lt, load_slot=ls if st is not None else None, evict_tok=et,
                n_load=nl.value, n_evict=ne.value, slot_tok=st, status=rc)


# ---------------------------------------------------------------- O10..O12
def attn_head(q, k, v, rows, scale: float):
    """One query head over rows of a [N][D] K/V block, fp64. Returns (out [D] f64, lse)."""
    q = np.asarray(q)
    is_bf16 = q.dtype in (np.uint16, np.int16)
    if is_bf16:
        q, k, v = _bf16_bits(q), _bf16_bits(k), _bf16_bits(v)
    else:
        q, k, v = (np.ascontiguousarray(a, dtype=np.float32) for a in (q, k, v))
    D = q.shape[-1]
    rows = np.ascontiguousarray(rows, dtype=np.int32)
    out = np.zeros(D, np.float64)
    lse = lib().spcref_attn_head(_p(q), _p(k), _p(v), int(is_bf16),
                                 _p(rows) if len(rows) else None, len(rows), D,
                                 ctypes.c_double(scale), _p(out))
    return out, float(lse)


def sparse_attn(q, k_layers, v_layers, idx, count, scale: float, layers=None):
    """O10 over every (l, b, h): q [L][B][Hq][D], k_layers/v_layers: list of [B][G][rows][D]
    arrays, idx [B][G][k] (rows to use; for SLOTS pass arange), count [B][G].
    Returns (out [L][B][Hq][D] f64, lse [L][B][Hq] f64)."""
    L, B, Hq, D = q.shape
    G = k_layers[0].shape[1]
    alpha = Hq // G
    layers = range(L) if layers is None else layers
    out = np.zeros((L, B, Hq, D), np.float64)
    lse = np.full((L, B, Hq), -np.inf, np.float64)
    for l in layers:
        for b in range(B):
            for h in range(Hq):
                g = h // alpha
                n = int(count[b, g])
                o, s = attn_head(q[l, b, h], k_layers[l][b, g], v_layers[l][b, g], idx[b, g, :n],
                                 scale)
                out[l, b, h] = o
                lse[l, b, h] = s
    return out, lse


def attn_merge(o_parts, lse_parts):
    """o_parts [P][n][D], lse_parts [P][n] -> (out [n][D] f64, lse [n] f64)."""
    o_parts = np.asarray(o_parts, np.float64)
    lse_parts = np.asarray(lse_parts, np.float64)
    P, n, D = o_parts.shape
    out = np.zeros((n, D), np.float64)
    lse = np.zeros(n, np.float64)
    for i in range(n):
        o = np.ascontiguousarray(o_parts[:, i, :])
        s = np.ascontiguousarray(lse_parts[:, i])
        r = np.zeros(D, np.float64)
        lse[i] = lib().spcref_attn_merge_row(_p(o), _p(s), P, D, _p(r))
        out[i] = r
    return out, lse


# ---------------------------------------------------------------- NEXT-1 front-end
def rmsnorm_bf16(x, w, eps: float):
    """x [B][H] bf16 bits (uint16); w [H] bits or None -> xn [B][H] bf16 bits (spcref_rmsnorm_bf16)."""
    x = np.ascontiguousarray(_bf16_bits(x))
    B, H = x.shape
    wb = None if w is None else np.ascontiguousarray(_bf16_bits(w))
    out = np.zeros((B, H), np.uint16)
    for b in range(B):
        lib().spcref_rmsnorm_bf16(_p(x[b]), None if wb is None else _p(wb), H, float(eps), _p(out[b]))
    return out


def rethead_qk(W, xn, inv_freq, pos, D: int, mscale: float = 1.0):
    """W [N][H] bits, xn [B][H] bits, inv_freq [D/2] f32, pos [B] -> (out [B][N] f64 rotated
    projections, bound [B][N] f64 = sum |W x|) (spcref_rethead_qk)."""
    W = np.ascontiguousarray(_bf16_bits(W))
    xn = np.ascontiguousarray(_bf16_bits(xn))
    inv = np.ascontiguousarray(np.asarray(inv_freq, np.float32))
    N, H = W.shape
    B = xn.shape[0]
    out = np.zeros((B, N), np.float64)
    bound = np.zeros((B, N), np.float64)
    for b in range(B):
        lib().spcref_rethead_qk(_p(W), N, H, _p(xn[b]), _p(inv), D, int(pos[b]), float(mscale),
                                _p(out[b]), _p(bound[b]))
    return out, bound


# ---------------------------------------------------------------- NEXT-2 planner
def _plan_args(c):
    return (int(c["model_bytes"]), float(c.get("runtime_factor", 1.3)), int(c["L"]), int(c["H"]),
            int(c["D"]), int(c["extra_layers"]), int(c["R"]), int(c["B"]),
            int(c.get("bytes_per_elem", 2)))


def plan_mem(c, S: int, l_gpu: int) -> int:
    """Eq. 7 (Eq. 6 at l_gpu = L) for a planner config dict c."""
    return int(lib().spcref_plan_mem(*_plan_args(c), int(S), int(l_gpu)))


def plan_thresholds_search(c, s_cap: int = 1 << 40):
    th = np.zeros(int(c["L"]) + 1, np.int64)
    lib().spcref_plan_thresholds_search(int(c["mem_gpu"]), *_plan_args(c), int(s_cap), _p(th))
    return th


def plan_max_resident(c, S: int) -> int:
    return int(lib().spcref_plan_max_resident(int(c["mem_gpu"]), *_plan_args(c), int(S)))


def plan_step(th, L: int, S: int, l_cpu: int):
    th = np.ascontiguousarray(np.asarray(th, np.int64))
    out = np.zeros(L, np.int32)
    n = np.zeros(1, np.int32)
    lc = int(lib().spcref_plan_step(_p(th), L, int(S), int(l_cpu), _p(out), _p(n)))
    return lc, out[:int(n[0])].tolist()


# ---------------------------------------------------------------- NEXT-3 batch-level
def batch_score(lg, hm, F, seq_len):
    """Batch-level score [B][Smax] (spcref_batch_score, O6b) from logits [B][Hq][Smax],
    head_max [B][Hq], head_sumfix [B][Hq]."""
    lg = np.ascontiguousarray(lg, np.float32)
    B, Hq, Smax = lg.shape
    out = np.zeros((B, Smax), np.float32)
    lib().spcref_batch_score(_p(lg), _p(np.ascontiguousarray(hm, np.float32)),
                             _p(np.ascontiguousarray(F, np.int64)),
                             _p(np.ascontiguousarray(seq_len, np.int32)), B, Hq, Smax, _p(out))
    return out


# ---------------------------------------------------------------- NEXT-3 MLA
def mla_head(q, cache, w_uk, w_uv, rows, DC: int, DR: int, scale: float):
    """One head: select-then-expand MLA attention (spcref_mla_head) -> (o [DV] f64, lse)."""
    q = np.ascontiguousarray(_bf16_bits(q))
    cache = np.ascontiguousarray(_bf16_bits(cache))
    w_uk = np.ascontiguousarray(_bf16_bits(w_uk))
    w_uv = np.ascontiguousarray(_bf16_bits(w_uv))
    rows = np.ascontiguousarray(np.asarray(rows, np.int32))
    DN, DV = w_uk.shape[0], w_uv.shape[0]
    out = np.zeros(DV, np.float64)
    lse = lib().spcref_mla_head(_p(q), _p(cache), _p(w_uk), _p(w_uv), _p(rows), len(rows), DC, DR,
                                DN, DV, float(scale), _p(out))
    return out, lse
