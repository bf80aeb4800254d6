"""Context-sharded decode step over P ranks (DESIGN.md §3 O13, §8).

Rank r of P owns the global tokens t ≡ r (mod P) of the retrieval-key cache and
of every layer's KV cache; local position u holds global token t = u*P + r.  One
step (BASELINE config E):

  1. LOGITS on the local keys            -> all-reduce MAX of head_max   (exact)
  2. NORM with the global max            -> all-reduce SUM of int64 sums (exact)
  3. GROUP; local top-k with global ids  -> ONE all-gather of packed (value, pos, count)
  4. global threshold = k-th composite of the union (spc_topk_merge); each rank
     keeps its entries >= threshold (spc_topk_filter): the union equals the
     single-device selection bit for bit (O13)
  5. sparse attention over the local rows for all L layers
                                         -> ONE all-gather of packed (o, lse); LSE merge (O12)

Every compute step is a libspc call (``SpcOps``); collectives are
torch.distributed calls on the current stream (NCCL over NVLink on a GPU box).
The phases are plain functions so that the same orchestration also runs with P
emulated ranks in one process (``run_emulated``) and, in tests, with a CPU
backend on gloo.  There is no CPU fallback in the product path: ``SpcOps`` only
calls libspc.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch

from . import spc


def local_len(S: int, P: int, r: int) -> int:
    """Number of the first S global tokens owned by rank r (t ≡ r mod P)."""
    return max(0, (S - r + P - 1) // P)


def owner(t: int, P: int) -> int:
    return t % P


def shard_rows(x: torch.Tensor, P: int, r: int, axis: int) -> torch.Tensor:
    """Rows t ≡ r (mod P) of a global tensor along `axis` (contiguous copy)."""
    idx = [slice(None)] * x.dim()
    idx[axis] = slice(r, None, P)
    return x[tuple(idx)].contiguous()


@dataclass
class ShardState:
    """Inputs and buffers of one rank for one step.  Global shapes: B requests, G KV
    groups, Hq query heads, D head dim, L layers, budget k."""
    rank: int
    P: int
    S: list                      # global context length per request (host ints)
    kr: torch.Tensor             # [B][G][Smax_loc][D] local retrieval keys
    k_layers: list               # L x [B][G][rows_loc][D] local K cache
    v_layers: list               # L x [B][G][rows_loc][D] local V cache
    q_ret: torch.Tensor          # [B][Hq][D]
    q_llm: torch.Tensor          # [L][B][Hq][D]
    k: int
    scale: float
    bufs: dict = field(default_factory=dict)

    @property
    def B(self):
        return self.kr.shape[0]

    @property
    def G(self):
        return self.kr.shape[1]

    @property
    def Hq(self):
        return self.q_ret.shape[1]

    @property
    def L(self):
        return len(self.k_layers)

    def local_seq(self):
        return [local_len(s, self.P, self.rank) for s in self.S]

    def owns_last(self, b: int) -> bool:
        return owner(self.S[b] - 1, self.P) == self.rank


class SpcOps:
    """libspc-backed phase kernels (GPU).  Buffers are cached in ``st.bufs``."""

    def _buf(self, st, name, shape, dtype):
        t = st.bufs.get(name)
        if t is None or tuple(t.shape) != tuple(shape) or t.dtype != dtype:
            t = torch.zeros(shape, dtype=dtype, device=st.kr.device)
            st.bufs[name] = t
        return t

    def _seq(self, st):
        """The local seq_len buffer: one per state, refreshed in place when S changes (a
        decode loop that advances S reuses it; refresh outside graph capture)."""
        t = st.bufs.get("seq_loc")
        key = tuple(st.S)
        if t is None:
            t = st.bufs["seq_loc"] = torch.tensor(st.local_seq(), dtype=torch.int32,
                                                  device=st.kr.device)
            st.bufs["seq_key"] = key
        elif st.bufs.get("seq_key") != key:
            t.copy_(torch.tensor(st.local_seq(), dtype=torch.int32))
            st.bufs["seq_key"] = key
        return t

    def _score(self, st, phases, head_max=None, sumfix=None):
        B, G, Smax, D = st.kr.shape
        dev = st.kr.device
        lg = self._buf(st, "logits", (B, st.Hq, Smax), torch.float32)
        hm = head_max if head_max is not None else self._buf(st, "hm", (B, st.Hq), torch.float32)
        F = sumfix if sumfix is not None else self._buf(st, "F", (B, st.Hq), torch.int64)
        gs = self._buf(st, "gs", (B, G, Smax), torch.float32)
        ws = st.bufs.get("ws_score")
        if ws is None:
            ws = st.bufs["ws_score"] = spc.alloc_workspace(spc.score_workspace(B, st.Hq, Smax), dev)
        spc.score(st.q_ret, st.kr, self._seq(st), G, st.scale, lg, hm, F, gs, ws, phases=phases)
        return hm, F, gs

    def logits(self, st):
        hm, _, _ = self._score(st, spc.SCORE_LOGITS)
        return hm

    def norm(self, st, head_max):
        _, F, _ = self._score(st, spc.SCORE_NORM, head_max=head_max)
        return F

    def group(self, st, head_max, sumfix):
        _, _, gs = self._score(st, spc.SCORE_GROUP, head_max=head_max, sumfix=sumfix)
        return gs

    def topk_local(self, st, gs):
        B, G, n = gs.shape
        idx = self._buf(st, "cand_pos", (B, G, st.k), torch.int32)
        val = self._buf(st, "cand_val", (B, G, st.k), torch.float32)
        cnt = self._buf(st, "cand_cnt", (B, G), torch.int32)
        ws = st.bufs.get("ws_topk")
        if ws is None:
            ws = st.bufs["ws_topk"] = spc.alloc_workspace(spc.topk_workspace(B, G, n, st.k),
                                                         gs.device)
        # force_last applies per request on the owner of global token S-1; requests are
        # handled together, so a rank forces when it owns the last token of every request
        # (B = 1 in the sharded configs); other cases force via a per-request call
        force = all(st.owns_last(b) for b in range(B))
        if B == 1 or force or not any(st.owns_last(b) for b in range(B)):
            spc.topk(gs, self._seq(st), st.k, idx, cnt, ws, out_val=val, force_last=force,
                     id_stride=st.P, id_offset=st.rank)
        else:
            for b in range(B):
                sl = self._buf(st, f"seq1_{b}", (1,), torch.int32)
                sl.fill_(st.local_seq()[b])
                spc.topk(gs[b:b + 1], sl, st.k, idx[b:b + 1], cnt[b:b + 1], ws,
                         out_val=val[b:b + 1], force_last=st.owns_last(b), id_stride=st.P,
                         id_offset=st.rank)
        return val, idx, cnt

    def merge(self, st, cand_val, cand_pos, cand_cnt):
        P, B, G, k = cand_val.shape
        th = self._buf(st, "thresh", (B * G,), torch.int64)
        spc.topk_merge(cand_val.reshape(P, B * G, k), cand_pos.reshape(P, B * G, k),
                       cand_cnt.reshape(P, B * G), k, th)
        return th

    def filter(self, st, pos, val, cnt, thresh):
        B, G, k = pos.shape
        spc.topk_filter(pos, val, cnt, thresh, k, st.P, st.rank)
        return pos, cnt

    def attn(self, st, pos, cnt):
        L, B, Hq, D = st.q_llm.shape
        dev = st.q_llm.device
        out = self._buf(st, "o", (L, B, Hq, D), torch.float32)
        lse = self._buf(st, "lse", (L, B, Hq), torch.float32)
        ws = st.bufs.get("ws_attn")
        if ws is None:
            ws = st.bufs["ws_attn"] = spc.alloc_workspace(spc.attn_workspace(L, B, Hq, D, st.k),
                                                         dev)
        rows = st.k_layers[0].shape[2]
        if st.k_layers[0].dtype == torch.bfloat16:  # TMA row gathers over the layer descriptors
            if "kvdesc" not in st.bufs:
                st.bufs["kvdesc"] = spc.KvDesc(st.k_layers, st.v_layers)
            spc.sparse_decode_attn_kv(st.bufs["kvdesc"], st.q_llm, spc.KV_INDEXED, pos, cnt, st.k,
                                      st.scale, out, lse, ws)
        else:
            if "ktab" not in st.bufs:
                st.bufs["ktab"] = spc.ptr_table(st.k_layers, dev)
                st.bufs["vtab"] = spc.ptr_table(st.v_layers, dev)
            spc.sparse_decode_attn(st.q_llm, st.bufs["ktab"], st.bufs["vtab"], spc.KV_INDEXED, pos,
                                   cnt, rows, st.k, st.scale, out, lse, ws, st.G)
        return out, lse

    def attn_merge(self, st, o_parts, lse_parts):
        P = o_parts.shape[0]
        D = o_parts.shape[-1]
        n = o_parts[0].numel() // D
        out = self._buf(st, "o_merged", o_parts.shape[1:], torch.float32)
        lse = self._buf(st, "lse_merged", lse_parts.shape[1:], torch.float32)
        spc.attn_merge(o_parts.reshape(P, n, D), lse_parts.reshape(P, n), out.view(n, D),
                       lse.view(n))
        return out, lse


# ---------------------------------------------------------------- the step, by phase
def phase_logits(ops, st):
    return ops.logits(st)


def phase_norm(ops, st, head_max):
    return ops.norm(st, head_max)


def phase_candidates(ops, st, head_max, sumfix):
    gs = ops.group(st, head_max, sumfix)
    return ops.topk_local(st, gs)


def phase_select_attend(ops, st, cand_val_all, cand_pos_all, cand_cnt_all):
    th = ops.merge(st, cand_val_all, cand_pos_all, cand_cnt_all)
    r = st.rank
    pos = cand_pos_all[r].clone()
    cnt = cand_cnt_all[r].clone()
    pos, cnt = ops.filter(st, pos, cand_val_all[r].contiguous(), cnt, th)
    o, lse = ops.attn(st, pos, cnt)
    return pos, cnt, o, lse


def phase_merge(ops, st, o_all, lse_all):
    return ops.attn_merge(st, o_all, lse_all)


def _gather_packed(parts, P, group):
    """ONE all-gather of several tensors of one rank: their bytes are packed into a flat
    buffer, gathered into [P][nbytes], and returned as dense per-part tensors [P][...]."""
    import torch.distributed as dist
    words = [t.contiguous().view(torch.uint8).reshape(-1) for t in parts]
    send = torch.cat(words)
    recv = torch.empty(P * send.numel(), dtype=torch.uint8, device=send.device)
    dist.all_gather_into_tensor(recv, send, group=group)  # flat [P * n]: NCCL and gloo
    recv = recv.view(P, send.numel())
    out, off = [], 0
    for t, w in zip(parts, words):
        # one small contiguous copy per part: the kernels take dense [P][...] operands
        out.append(recv[:, off:off + w.numel()].view(t.dtype).reshape((P,) + tuple(t.shape))
                   .contiguous())
        off += w.numel()
    return out


def run_distributed(ops, st: ShardState, group=None):
    """One sharded step on this rank; collectives through torch.distributed (NCCL for
    CUDA tensors, gloo for CPU tensors).  FOUR collectives per step: the
    all-reduce MAX of head_max, the all-reduce SUM of the int64 normalisers, ONE all-gather
    of the packed (value, position, count) candidates and ONE all-gather of the packed
    (o, lse) partials.  Returns (local pos, count, merged o, merged lse)."""
    import torch.distributed as dist
    P = st.P
    hm = phase_logits(ops, st)
    dist.all_reduce(hm, op=dist.ReduceOp.MAX, group=group)
    F = phase_norm(ops, st, hm)
    dist.all_reduce(F, op=dist.ReduceOp.SUM, group=group)
    val, pos, cnt = phase_candidates(ops, st, hm, F)
    gv, gp, gc = _gather_packed([val, pos, cnt], P, group)
    lpos, lcnt, o, lse = phase_select_attend(ops, st, gv, gp, gc)
    go, gl = _gather_packed([o, lse], P, group)
    out, lse_m = phase_merge(ops, st, go.contiguous(), gl.contiguous())
    return lpos, lcnt, out, lse_m


def run_emulated(ops, states):
    """The same step with P ranks emulated in one process (collectives by stacking)."""
    hms = [phase_logits(ops, st) for st in states]
    hm = torch.stack(hms).amax(0)
    Fs = [phase_norm(ops, st, hm.clone()) for st in states]
    F = torch.stack([f.clone() for f in Fs]).sum(0)
    cands = [phase_candidates(ops, st, hm.clone(), F.clone()) for st in states]
    cv = torch.stack([c[0].clone() for c in cands])
    cp = torch.stack([c[1].clone() for c in cands])
    cc = torch.stack([c[2].clone() for c in cands])
    res = [phase_select_attend(ops, st, cv, cp, cc) for st in states]
    o_all = torch.stack([r[2].clone() for r in res])
    l_all = torch.stack([r[3].clone() for r in res])
    out, lse = phase_merge(ops, states[0], o_all, l_all)
    return [(r[0].clone(), r[1].clone()) for r in res], out, lse


def make_shard(rank: int, P: int, kr, k_layers, v_layers, q_ret, q_llm, S, k, scale=None):
    """Build rank r's ShardState from GLOBAL tensors (tests / small configs)."""
    D = kr.shape[-1]
    scale = float(torch.tensor(1.0 / math.sqrt(D), dtype=torch.float32)) if scale is None else scale
    return ShardState(rank=rank, P=P, S=list(S), kr=shard_rows(kr, P, rank, 2),
                      k_layers=[shard_rows(t, P, rank, 2) for t in k_layers],
                      v_layers=[shard_rows(t, P, rank, 2) for t in v_layers], q_ret=q_ret,
                      q_llm=q_llm, k=k, scale=scale)
