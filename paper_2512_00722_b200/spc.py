"""ctypes binding of libspc.so (include/spc.h) — argument marshalling only.

Every function has the name of the C entry point without the ``spc_`` prefix
and takes torch tensors (device memory) plus plain ints/floats; it passes
their data pointers and the current CUDA stream to the library and raises
``SpcError`` on a non-OK status.  No arithmetic of the method happens here.
There is no CPU fallback: if libspc.so is missing or CUDA is unavailable,
``lib()`` raises.
"""
from __future__ import annotations

import ctypes
import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libspc.so")
DEBUG_LIB_PATH = os.path.join(HERE, "libspc_debug.so")  # SPC_DEBUG: device contract checks

BF16, F32 = 0, 1
SCORE_LOGITS, SCORE_NORM, SCORE_GROUP, SCORE_ALL, SCORE_BATCH = 1, 2, 4, 7, 16
KV_INDEXED, KV_SLOTS = 0, 1
MAX_K = 4096

EXPORTS = [
    "spc_status_string", "spc_last_cuda_error", "spc_version", "spc_launch_count",
    "spc_score_workspace", "spc_score", "spc_topk_workspace", "spc_topk",
    "spc_topk_merge_workspace", "spc_topk_merge", "spc_topk_filter", "spc_elastic_diff",
    "spc_gather_kv", "spc_gather_kv_strided", "spc_attn_workspace", "spc_sparse_decode_attn",
    "spc_attn_merge", "spc_select", "spc_rethead_qk", "spc_plan_mem_part",
    "spc_plan_thresholds", "spc_plan_max_resident", "spc_plan_step", "spc_mla_workspace",
    "spc_mla_sparse_attn", "spc_decode_step_workspace", "spc_decode_step",
    "spc_kv_desc_bytes", "spc_kv_desc_init", "spc_sparse_decode_attn_kv",
    "spc_score_select_supported", "spc_score_select_workspace", "spc_score_select",
    "spc_debug_build", "spc_check_device_errors", "spc_llm_embed", "spc_llm_add_rmsnorm",
    "spc_llm_rope_append", "spc_llm_swiglu", "spc_llm_f32_to_bf16", "spc_llm_argmax",
]


class SpcError(RuntimeError):
    pass


class StepArgs(ctypes.Structure):
    """spc_step_args (include/spc.h): every buffer of one spc_decode_step call."""
    _fields_ = [(n, ctypes.c_int) for n in ("L", "B", "Hq", "G", "D", "Smax", "rows", "k",
                                            "force_last")] + \
        [("scale", ctypes.c_float)] + \
        [(n, ctypes.c_void_p) for n in ("q_ret", "kr", "seq_len", "q_llm", "k_layers", "v_layers",
                                        "logits", "head_max", "head_sumfix", "group_score",
                                        "prev_idx", "prev_count", "cur_idx", "cur_count",
                                        "load_tok", "n_load", "out", "lse", "ws")] + \
        [("ws_bytes", ctypes.c_size_t), ("kv_desc", ctypes.c_void_p)]


class PlanCfg(ctypes.Structure):
    """spc_plan_cfg (include/spc.h): inputs of the adaptive memory planner (Eq. 6-8)."""
    _fields_ = [("mem_gpu", ctypes.c_int64), ("model_bytes", ctypes.c_int64),
                ("runtime_factor", ctypes.c_double), ("L", ctypes.c_int), ("H", ctypes.c_int),
                ("D", ctypes.c_int), ("extra_layers", ctypes.c_int), ("R", ctypes.c_int),
                ("B", ctypes.c_int64), ("bytes_per_elem", ctypes.c_int)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libspc.so and declare signatures (works without a GPU)."""
    if not os.path.exists(path):
        raise SpcError(f"{path} not found: build it with `python -m paper_2512_00722_b200.build` "
                       "(there is no CPU fallback)")
    L = ctypes.CDLL(path)
    P, i32, f32, sz, u64 = (ctypes.c_void_p, ctypes.c_int, ctypes.c_float, ctypes.c_size_t,
                            ctypes.c_uint64)
    L.spc_status_string.argtypes = [i32]
    L.spc_status_string.restype = ctypes.c_char_p
    L.spc_last_cuda_error.restype = ctypes.c_char_p
    L.spc_version.restype = i32
    L.spc_launch_count.restype = u64
    L.spc_score_workspace.argtypes = [i32, i32, i32]
    L.spc_score_workspace.restype = sz
    L.spc_score.argtypes = [i32, P, P, P, i32, i32, i32, i32, i32, f32, i32, P, P, P, P, P, sz, P]
    L.spc_topk_workspace.argtypes = [i32, i32, i32, i32]
    L.spc_topk_workspace.restype = sz
    L.spc_topk.argtypes = [P, P, i32, i32, i32, i32, i32, i32, i32, P, P, P, P, P, sz, P]
    L.spc_topk_merge_workspace.argtypes = [i32, i32, i32]
    L.spc_topk_merge_workspace.restype = sz
    L.spc_topk_merge.argtypes = [P, P, P, i32, i32, i32, P, P, sz, P]
    L.spc_topk_filter.argtypes = [P, P, P, P, i32, i32, i32, i32, P]
    L.spc_elastic_diff.argtypes = [P, P, P, P, i32, i32, i32, P, P, P, P, P, P, P]
    L.spc_gather_kv.argtypes = [i32, P, P, i32, i32, i32, i32, i32, i32, i32, i32, P, P, P, P, P,
                                P]
    L.spc_gather_kv_strided.argtypes = [i32, P, P, ctypes.c_longlong, ctypes.c_longlong, i32, i32,
                                        i32, i32, i32, i32, i32, P, P, P, P, P, P]
    L.spc_rethead_qk.argtypes = [P, P, i32, i32, P, f32, P, P, f32, P, i32, i32, i32, i32, i32,
                                 P, P, P, P, P]
    i64 = ctypes.c_int64
    L.spc_plan_mem_part.argtypes = [ctypes.POINTER(PlanCfg), i64, i32]
    L.spc_plan_mem_part.restype = i64
    L.spc_plan_thresholds.argtypes = [ctypes.POINTER(PlanCfg), P]
    L.spc_plan_max_resident.argtypes = [ctypes.POINTER(PlanCfg), i64, ctypes.POINTER(i32),
                                        ctypes.POINTER(i64)]
    L.spc_plan_step.argtypes = [P, i32, i64, ctypes.POINTER(i32), P, ctypes.POINTER(i32)]
    L.spc_mla_workspace.argtypes = [i32, i32, i32, i32]
    L.spc_mla_workspace.restype = sz
    L.spc_mla_sparse_attn.argtypes = [P, P, P, P, P, P, i32, i32, i32, i32, i32, i32, i32, i32, i32,
                                      f32, P, P, P, sz, P]
    L.spc_decode_step_workspace.argtypes = [i32, i32, i32, i32, i32, i32, i32]
    L.spc_decode_step_workspace.restype = sz
    L.spc_decode_step.argtypes = [ctypes.POINTER(StepArgs), P]
    L.spc_attn_workspace.argtypes = [i32, i32, i32, i32, i32]
    L.spc_attn_workspace.restype = sz
    L.spc_sparse_decode_attn.argtypes = [i32, P, P, P, i32, P, P, i32, i32, i32, i32, i32, i32,
                                         i32, i32, i32, f32, P, P, P, sz, P]
    L.spc_attn_merge.argtypes = [P, P, i32, i32, i32, P, P, P]
    L.spc_debug_build.restype = i32
    L.spc_check_device_errors.argtypes = [P]
    L.spc_score_select_supported.argtypes = [i32, i32, i32, i32, i32, i32]
    L.spc_score_select_workspace.argtypes = [i32, i32, i32, i32]
    L.spc_score_select_workspace.restype = sz
    L.spc_score_select.argtypes = [P, P, P, i32, i32, i32, i32, i32, f32, i32, i32, P, P, P, P, P,
                                   P, P, P, P, P, P, P, P, sz, P]
    L.spc_kv_desc_bytes.argtypes = [i32]
    L.spc_kv_desc_bytes.restype = sz
    L.spc_kv_desc_init.argtypes = [P, P, P, i32, i32, i32, i32, i32]
    L.spc_sparse_decode_attn_kv.argtypes = [P, P, i32, P, P, i32, i32, i32, i32, i32, i32, i32,
                                            i32, i32, f32, P, P, P, sz, P]
    L.spc_select.argtypes = [P, P, P, i32, i32, i32, i32, i32, i32, P, P, P, P, P, P, P, P, P, P,
                             P]
    L.spc_llm_embed.argtypes = [P, P, i32, i32, i32, P, P]
    L.spc_llm_add_rmsnorm.argtypes = [P, P, P, i32, i32, f32, P, P]
    L.spc_llm_rope_append.argtypes = [P, P, P, i32, i32, i32, i32, i32, P, P, P, P, i32, P, P, P]
    L.spc_llm_swiglu.argtypes = [P, i32, i32, P, P]
    L.spc_llm_f32_to_bf16.argtypes = [P, ctypes.c_longlong, P, P]
    L.spc_llm_argmax.argtypes = [P, i32, i32, P, P, P]
    for name in EXPORTS:  # every symbol must resolve (raises AttributeError otherwise)
        getattr(L, name)
    return L


def lib():
    global _lib
    if _lib is None:
        _lib = load_library()
    return _lib


def _check(rc: int, what: str):
    if rc != 0:
        msg = lib().spc_status_string(rc).decode()
        if rc == 8:
            msg += " — " + lib().spc_last_cuda_error().decode()
        raise SpcError(f"{what}: {msg}")


def _p(t):
    if t is None:
        return None
    if isinstance(t, int):
        return ctypes.c_void_p(t)
    assert t.is_contiguous(), "libspc tensors must be contiguous"
    return ctypes.c_void_p(t.data_ptr())


def _s(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return BF16
    if t.dtype == torch.float32:
        return F32
    raise SpcError(f"unsupported dtype {t.dtype}")


def launch_count() -> int:
    return int(lib().spc_launch_count())


def version() -> int:
    return int(lib().spc_version())


def ptr_table(tensors, device) -> torch.Tensor:
    """Device array of data pointers (the per-layer pointer tables of the ABI)."""
    return torch.tensor([int(t.data_ptr()) for t in tensors], dtype=torch.int64, device=device)


# ------------------------------------------------------------------ workspaces
def score_workspace(B: int, Hq: int, Smax: int) -> int:
    return int(lib().spc_score_workspace(B, Hq, Smax))


def topk_workspace(B: int, G: int, n_cols: int, k: int) -> int:
    return int(lib().spc_topk_workspace(B, G, n_cols, k))


def topk_merge_workspace(P: int, R: int, k: int) -> int:
    return int(lib().spc_topk_merge_workspace(P, R, k))


def attn_workspace(L: int, B: int, Hq: int, D: int, k: int) -> int:
    return int(lib().spc_attn_workspace(L, B, Hq, D, k))


def check_device_errors(stream=None) -> int:
    """spc_check_device_errors: synchronise and return (and clear) the first device-side
    contract violation (SPC_DEBUG builds) as a spc_status code; 0 = none."""
    return int(lib().spc_check_device_errors(_s(stream)))


def alloc_workspace(nbytes: int, device) -> torch.Tensor:
    """Workspaces must start zero-filled (the library leaves them zero-filled)."""
    return torch.zeros(max(int(nbytes), 1), dtype=torch.uint8, device=device)


# ------------------------------------------------------------------ calls
def score(q, kr, seq_len, G: int, scale: float, logits, head_max, head_sumfix, group_score, ws,
          phases: int = SCORE_ALL, stream=None):
    B, Hq, D = q.shape
    Smax = kr.shape[2]
    _check(lib().spc_score(_dtype_code(q), _p(q), _p(kr), _p(seq_len), B, Hq, G, D, Smax,
                           float(scale), phases, _p(logits), _p(head_max), _p(head_sumfix),
                           _p(group_score), _p(ws), ws.numel(), _s(stream)), "spc_score")


def topk(val, seq_len, k: int, out_idx, out_count, ws, out_val=None, out_thresh=None,
         force_last: bool = False, id_stride: int = 1, id_offset: int = 0, stream=None):
    B, G, n_cols = val.shape
    _check(lib().spc_topk(_p(val), _p(seq_len), B, G, n_cols, k, int(force_last), id_stride,
                          id_offset, _p(out_idx), _p(out_val), _p(out_count), _p(out_thresh),
                          _p(ws), ws.numel(), _s(stream)), "spc_topk")


def topk_merge(cand_val, cand_pos, cand_count, k: int, out_thresh, ws=None, stream=None):
    P, R = cand_count.shape
    _check(lib().spc_topk_merge(_p(cand_val), _p(cand_pos), _p(cand_count), P, R, k,
                                _p(out_thresh), _p(ws), 0 if ws is None else ws.numel(),
                                _s(stream)), "spc_topk_merge")


def topk_filter(idx, val, count, thresh, k: int, id_stride: int, id_offset: int, stream=None):
    R = count.numel()
    _check(lib().spc_topk_filter(_p(idx), _p(val), _p(count), _p(thresh), R, k, id_stride,
                                 id_offset, _s(stream)), "spc_topk_filter")


def elastic_diff(prev_idx, prev_count, cur_idx, cur_count, load_tok, n_load, slot_tok=None,
                 load_slot=None, evict_tok=None, n_evict=None, stream=None):
    B, G, k = cur_idx.shape
    _check(lib().spc_elastic_diff(_p(prev_idx), _p(prev_count), _p(cur_idx), _p(cur_count), B, G,
                                  k, _p(slot_tok), _p(load_tok), _p(load_slot), _p(n_load),
                                  _p(evict_tok), _p(n_evict), _s(stream)), "spc_elastic_diff")


def gather_kv(k_src_tab, v_src_tab, L: int, B: int, G: int, D: int, Smax: int, k: int,
              load_tok, load_slot, n_load, k_buf_tab, v_buf_tab, layer_begin: int = 0,
              layer_end=None, dtype: int = BF16, stream=None):
    layer_end = L if layer_end is None else layer_end
    _check(lib().spc_gather_kv(dtype, _p(k_src_tab), _p(v_src_tab), L, B, G, D, Smax, k,
                               layer_begin, layer_end, _p(load_tok), _p(load_slot), _p(n_load),
                               _p(k_buf_tab), _p(v_buf_tab), _s(stream)), "spc_gather_kv")


def gather_kv_strided(k_src_tab, v_src_tab, row_stride: int, bg_stride: int, L: int, B: int,
                      G: int, D: int, k: int, load_tok, load_slot, n_load, k_buf_tab, v_buf_tab,
                      layer_begin: int = 0, layer_end=None, dtype: int = BF16, stream=None):
    """spc_gather_kv_strided: the O9 copy from sources with explicit (token, (b,g)) strides,
    e.g. token-major offloaded KV records."""
    layer_end = L if layer_end is None else layer_end
    _check(lib().spc_gather_kv_strided(dtype, _p(k_src_tab), _p(v_src_tab), int(row_stride),
                                       int(bg_stride), L, B, G, D, k, layer_begin, layer_end,
                                       _p(load_tok), _p(load_slot), _p(n_load), _p(k_buf_tab),
                                       _p(v_buf_tab), _s(stream)), "spc_gather_kv_strided")


def rethead_qk(token, emb, norm_w, eps: float, w_qk, inv_freq, mscale: float, pos, Hq: int,
               G: int, q_out, kr, seq_len_out=None, x_out=None, stream=None):
    """spc_rethead_qk: embedding -> RMSNorm -> Q/K projection -> RoPE -> K append."""
    V, H = emb.shape
    B = token.numel()
    D = q_out.shape[-1]
    Smax = kr.shape[2]
    _check(lib().spc_rethead_qk(_p(token), _p(emb), V, H, _p(norm_w), float(eps), _p(w_qk),
                                _p(inv_freq), float(mscale), _p(pos), B, Hq, G, D, Smax,
                                _p(q_out), _p(kr), _p(seq_len_out), _p(x_out), _s(stream)),
           "spc_rethead_qk")


def mla_workspace(L: int, B: int, H: int, k: int) -> int:
    return int(lib().spc_mla_workspace(L, B, H, k))


def mla_sparse_attn(q, cache_tab, w_uk_tab, w_uv_tab, idx, count, Smax: int, DN: int, DV: int,
                    scale: float, out, lse, ws, DC: int = 512, DR: int = 64, stream=None):
    """spc_mla_sparse_attn: MLA attention over each head's selected latent rows, all layers
    (NEXT-3).  q [L][B][H][DN+DR]; *_tab: device pointer tables (ptr_table) per layer."""
    L, B, H, _ = q.shape
    k = idx.shape[2]
    _check(lib().spc_mla_sparse_attn(_p(q), _p(cache_tab), _p(w_uk_tab), _p(w_uv_tab), _p(idx),
                                     _p(count), L, B, H, Smax, k, DC, DR, DN, DV, float(scale),
                                     _p(out), _p(lse), _p(ws), ws.numel(), _s(stream)),
           "spc_mla_sparse_attn")


def decode_step_workspace(L: int, B: int, Hq: int, G: int, D: int, Smax: int, k: int) -> int:
    return int(lib().spc_decode_step_workspace(L, B, Hq, G, D, Smax, k))


def decode_step(args: "StepArgs", stream=None):
    """spc_decode_step: the whole single-device step (score -> select -> attention) in one
    C call; `args` is a StepArgs filled with data pointers (see make_step_args)."""
    _check(lib().spc_decode_step(ctypes.byref(args), _s(stream)), "spc_decode_step")


def make_step_args(q_ret, kr, seq_len, q_llm, k_tab, v_tab, rows: int, k: int, scale: float,
                   logits, head_max, head_sumfix, group_score, prev_idx, prev_count, cur_idx,
                   cur_count, load_tok, n_load, out, lse, ws, force_last: bool = True,
                   kv_desc=None) -> StepArgs:
    L, B, Hq, D = q_llm.shape
    G = kr.shape[1]
    ptr = lambda t: None if t is None else int(t.data_ptr())  # noqa: E731
    return StepArgs(L, B, Hq, G, D, kr.shape[2], rows, k, int(force_last), float(scale),
                    ptr(q_ret), ptr(kr), ptr(seq_len), ptr(q_llm), ptr(k_tab), ptr(v_tab),
                    ptr(logits), ptr(head_max), ptr(head_sumfix), ptr(group_score), ptr(prev_idx),
                    ptr(prev_count), ptr(cur_idx), ptr(cur_count), ptr(load_tok), ptr(n_load),
                    ptr(out), ptr(lse), ptr(ws), ws.numel(), ptr(kv_desc))


def sparse_decode_attn(q, k_tab, v_tab, kv_mode: int, idx, count, rows: int, k: int, scale: float,
                       out, lse, ws, G: int, layer_begin: int = 0, layer_end=None, stream=None):
    L, B, Hq, D = q.shape
    layer_end = L if layer_end is None else layer_end
    _check(lib().spc_sparse_decode_attn(_dtype_code(q), _p(q), _p(k_tab), _p(v_tab), kv_mode,
                                        _p(idx), _p(count), L, layer_begin, layer_end, B, Hq, G, D,
                                        rows, k, float(scale), _p(out), _p(lse), _p(ws),
                                        ws.numel(), _s(stream)), "spc_sparse_decode_attn")


class KvDesc:
    """spc_kv_desc_init: the per-layer TMA descriptors of an LLM KV cache, held in a device
    buffer.  k_layers / v_layers: L bf16 tensors, each holding a [B][G][rows][D] cache from
    its first element (4-D tensors of that shape, or flat views with B, G, rows, D given).
    The tensors must outlive the descriptor (it keeps references)."""

    def __init__(self, k_layers, v_layers, B=None, G=None, rows=None, D=None):
        L = len(k_layers)
        if B is None:
            B, G, rows, D = k_layers[0].shape
        for t in list(k_layers) + list(v_layers):
            assert t.dtype == torch.bfloat16 and t.is_contiguous() and t.is_cuda
            # 4-D caches hold every declared row; flat views (aliased layers at row offsets,
            # bench config C) need only hold the rows the selections address
            assert t.dim() == 1 or t.numel() >= B * G * rows * D
        self.L, self.B, self.G, self.rows, self.D = L, B, G, rows, D
        self._keep = (list(k_layers), list(v_layers))
        nbytes = int(lib().spc_kv_desc_bytes(L))
        self.buf = torch.empty(nbytes, dtype=torch.uint8, device=k_layers[0].device)
        kp = (ctypes.c_void_p * L)(*[t.data_ptr() for t in k_layers])
        vp = (ctypes.c_void_p * L)(*[t.data_ptr() for t in v_layers])
        _check(lib().spc_kv_desc_init(_p(self.buf), kp, vp, L, B, G, D, rows), "spc_kv_desc_init")

    def data_ptr(self) -> int:
        return self.buf.data_ptr()


def sparse_decode_attn_kv(desc: KvDesc, q, kv_mode: int, idx, count, k: int, scale: float, out,
                          lse, ws, layer_begin: int = 0, layer_end=None, stream=None):
    """spc_sparse_decode_attn_kv: the attention with TMA row gathers (bf16)."""
    L, B, Hq, D = q.shape
    layer_end = L if layer_end is None else layer_end
    _check(lib().spc_sparse_decode_attn_kv(_p(desc.buf), _p(q), kv_mode, _p(idx), _p(count), L,
                                           layer_begin, layer_end, B, Hq, desc.G, D, desc.rows, k,
                                           float(scale), _p(out), _p(lse), _p(ws), ws.numel(),
                                           _s(stream)), "spc_sparse_decode_attn_kv")


def score_select_supported(B: int, Hq: int, G: int, D: int, Smax: int, k: int) -> bool:
    return bool(lib().spc_score_select_supported(B, Hq, G, D, Smax, k))


def score_select_workspace(B: int, Hq: int, G: int, Smax: int) -> int:
    return int(lib().spc_score_select_workspace(B, Hq, G, Smax))


def score_select(q, kr, seq_len, scale: float, k: int, head_max, head_sumfix, group_score, out_idx,
                 out_count, prev_idx, prev_count, load_tok, n_load, ws, logits=None, evict_tok=None,
                 n_evict=None, force_last: bool = True, stream=None):
    """spc_score_select: LOGITS + NORM + GROUP + top-k + INDEXED diff in one launch."""
    B, G, Smax, D = kr.shape
    Hq = q.shape[1]
    _check(lib().spc_score_select(_p(q), _p(kr), _p(seq_len), B, Hq, G, D, Smax, float(scale), k,
                                  int(force_last), _p(logits), _p(head_max), _p(head_sumfix),
                                  _p(group_score), _p(out_idx), _p(out_count), _p(prev_idx),
                                  _p(prev_count), _p(load_tok), _p(n_load), _p(evict_tok),
                                  _p(n_evict), _p(ws), ws.numel(), _s(stream)), "spc_score_select")


def select(logits, head_max, seq_len, G: int, k: int, head_sumfix, group_score, out_idx,
           out_count, prev_idx, prev_count, load_tok, n_load, evict_tok=None, n_evict=None,
           force_last: bool = False, stream=None):
    """spc_select: fused NORM + GROUP + top-k + INDEXED elastic diff (one launch)."""
    B, Hq, Smax = logits.shape
    _check(lib().spc_select(_p(logits), _p(head_max), _p(seq_len), B, Hq, G, Smax, k,
                            int(force_last), _p(head_sumfix), _p(group_score), _p(out_idx),
                            _p(out_count), _p(prev_idx), _p(prev_count), _p(load_tok),
                            _p(n_load), _p(evict_tok), _p(n_evict), _s(stream)), "spc_select")


def attn_merge(o_parts, lse_parts, out, lse_out=None, stream=None):
    P, n, D = o_parts.shape
    _check(lib().spc_attn_merge(_p(o_parts), _p(lse_parts), P, n, D, _p(out), _p(lse_out),
                                _s(stream)), "spc_attn_merge")


# ------------------------------------------------------------------ adaptive memory planner
def plan_cfg(mem_gpu, model_bytes, L, H, D, R, B, extra_layers=1, runtime_factor=1.3,
             bytes_per_elem=2) -> PlanCfg:
    return PlanCfg(int(mem_gpu), int(model_bytes), float(runtime_factor), int(L), int(H), int(D),
                   int(extra_layers), int(R), int(B), int(bytes_per_elem))


def plan_mem_part(cfg: PlanCfg, S: int, l_gpu: int) -> int:
    return int(lib().spc_plan_mem_part(ctypes.byref(cfg), int(S), int(l_gpu)))


def plan_thresholds(cfg: PlanCfg):
    import numpy as np
    out = np.zeros(cfg.L + 1, np.int64)
    _check(lib().spc_plan_thresholds(ctypes.byref(cfg), out.ctypes.data_as(ctypes.c_void_p)),
           "spc_plan_thresholds")
    return out


def plan_max_resident(cfg: PlanCfg, S: int):
    """(l_gpu, shortfall); l_gpu = -1 when even l_gpu = 0 does not fit."""
    lg, sf = ctypes.c_int(0), ctypes.c_int64(0)
    rc = lib().spc_plan_max_resident(ctypes.byref(cfg), int(S), ctypes.byref(lg), ctypes.byref(sf))
    if rc not in (0, 3):
        _check(rc, "spc_plan_max_resident")
    return lg.value, sf.value


def plan_step(thresholds, L: int, S: int, l_cpu: int):
    """Algorithm 2 at sequence length S: (new l_cpu, [offloaded layers])."""
    import numpy as np
    th = np.ascontiguousarray(np.asarray(thresholds, np.int64))
    lc, n = ctypes.c_int(int(l_cpu)), ctypes.c_int(0)
    lay = np.zeros(L, np.int32)
    _check(lib().spc_plan_step(th.ctypes.data_as(ctypes.c_void_p), L, int(S), ctypes.byref(lc),
                               lay.ctypes.data_as(ctypes.c_void_p), ctypes.byref(n)), "spc_plan_step")
    return lc.value, lay[:n.value].tolist()


# ---------------------------------------------------------------- LLM layer ops (NEXT-4)
def llm_embed(token, emb, h, stream=None):
    """spc_llm_embed: h [B][H] f32 = emb[token]."""
    V, H = emb.shape
    _check(lib().spc_llm_embed(_p(token), _p(emb), V, H, token.numel(), _p(h), _s(stream)),
           "spc_llm_embed")


def llm_add_rmsnorm(h, delta, w, eps: float, xn, stream=None):
    """spc_llm_add_rmsnorm: h += delta (if given); xn = RMSNorm(h) * w (bf16)."""
    B, H = h.shape
    _check(lib().spc_llm_add_rmsnorm(_p(h), _p(delta), _p(w), B, H, float(eps), _p(xn),
                                     _s(stream)), "spc_llm_add_rmsnorm")


def llm_rope_append(qkv, inv_freq, seq_len, Hq: int, G: int, q_out, k_cache, v_cache,
                    slot_tok=None, k_buf=None, v_buf=None, stream=None):
    """spc_llm_rope_append: RoPE on q / k of the fused projection, append k / v at position
    seq_len - 1 of the layer caches (and into the budget slot holding it, SLOTS mode).
    k_cache / v_cache: [B][G][rows][D] (device or pinned host tensors)."""
    B = qkv.shape[0]
    D = q_out.shape[-1]
    rows = k_cache.shape[2]
    kb = 0 if slot_tok is None else slot_tok.shape[-1]
    _check(lib().spc_llm_rope_append(_p(qkv), _p(inv_freq), _p(seq_len), B, Hq, G, D, rows,
                                     _p(q_out), _p(k_cache), _p(v_cache), _p(slot_tok), kb,
                                     _p(k_buf), _p(v_buf), _s(stream)), "spc_llm_rope_append")


def llm_swiglu(gu, y, stream=None):
    B, F2 = gu.shape
    _check(lib().spc_llm_swiglu(_p(gu), B, F2 // 2, _p(y), _s(stream)), "spc_llm_swiglu")


def llm_f32_to_bf16(x, y, stream=None):
    assert x.numel() == y.numel()
    _check(lib().spc_llm_f32_to_bf16(_p(x), x.numel(), _p(y), _s(stream)), "spc_llm_f32_to_bf16")


def llm_argmax(logits, token_out, seq_len=None, stream=None):
    """spc_llm_argmax: token_out = argmax(logits) per row (lowest index on ties); seq_len += 1."""
    B, V = logits.shape
    _check(lib().spc_llm_argmax(_p(logits), B, V, _p(token_out), _p(seq_len), _s(stream)),
           "spc_llm_argmax")
