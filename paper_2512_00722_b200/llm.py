"""The LLM decode step around the sparse-attention hot path.

SpeContext's dataflow (Fig. 3; "concurrent execution of computation and KV
cache prefetching"; P:374 elastic loading): per decode step the retrieval head runs ONCE
(front-end -> scores -> top-k budget -> elastic diff, ``DecodeStep.enqueue(attend=False)``),
then every LLM layer runs its dense compute and attends only the selected K/V.  With the LLM
KV in pinned host memory (SLOTS mode) the elastic gather of layer l's newly selected rows
runs on a prefetch stream as soon as the selection exists, all layers in order, while the
main stream computes layers 0..l-1: layer l waits only for its own gather event, so the
PCIe transfer hides behind the weights-bound dense layers instead of serialising with them.

Layer l (Llama-3 architecture, the DeepSeek-R1-Distill-Llama-8B shape; random weights,
reading R30):
    xn = RMSNorm(h; ln1)                          spc_llm_add_rmsnorm (adds the MLP delta)
    qkv = W_qkv xn                                cuBLAS (plain GEMM)
    q, k, v = RoPE(q), RoPE(k), v; append k, v    spc_llm_rope_append
    a = SparseAttn(q, selected K/V)               spc_sparse_decode_attn_kv (layer l)
    h += W_o bf16(a); xn = RMSNorm(h; ln2)        spc_llm_f32_to_bf16, cuBLAS, add_rmsnorm
    h += W_down(silu(W_g xn) * W_u xn)            cuBLAS, spc_llm_swiglu, cuBLAS
then logits = lm_head RMSNorm(h) and the next token = argmax (spc_llm_argmax, which also
advances seq_len on the device), so consecutive steps chain without a host round trip and
one CUDA graph per step parity replays the whole step.  Every non-GEMM operation is a libspc
kernel; the projections are cuBLAS GEMMs (``torch.mm`` into preallocated outputs).
"""
from __future__ import annotations

import torch

from . import rope, spc
from .pipeline import DecodeStep


class LlmDecoder:
    def __init__(self, w: dict, cfg: dict, ret: dict, kr: torch.Tensor, k_cache, v_cache,
                 seq_len: torch.Tensor, k: int, kv: str = "resident", prefetch: bool = True,
                 force_last: bool = True, trace_queries=None, pf_priority: int = -1):
        """w: llm weights (synth.llm_weights).  cfg: L, H, Hq, G, D, F, V, rope_base, eps.
        ret: the retrieval head's front-end (emb, norm_w, w_qk, inv_freq [D/2] f32 device,
        mscale, Hq); kr [B][G][Smax][D] its key cache.  k_cache / v_cache: L tensors
        [B][G][rows][D] bf16 -- HBM (kv="resident": INDEXED attention over the caches) or
        pinned host memory (kv="offload": SLOTS, the elastic gather of the new rows into HBM
        budget buffers, on a prefetch stream when prefetch=True, else on the main stream
        right before each layer).  seq_len [B] int32 device: counts the step's new token
        (its position is seq_len - 1); the step advances it.
        trace_queries [n][B][Hq][D] bf16 (device) or None: score query i % n of this sequence at
        step i instead of the front-end's query (the front-end still runs and appends its key).
        A benchmark mode: with random weights consecutive tokens are unrelated, so the model's
        own queries select nearly disjoint sets step after step; the synthetic trace (AR(1)
        drift) has the adjacent-step similarity of a real trace."""
        assert kv in ("resident", "offload")
        self.cfg, self.w, self.kv, self.prefetch = cfg, w, kv, bool(prefetch)
        L, H, Hq, G, D, F, V = (cfg[x] for x in ("L", "H", "Hq", "G", "D", "F", "V"))
        self.L, self.H, self.Hq, self.G, self.D, self.F, self.V = L, H, Hq, G, D, F, V
        self.eps = float(cfg.get("eps", 1e-5))
        dev = kr.device
        self.dev = dev
        B = kr.shape[0]
        self.B, self.k = B, k
        self.k_cache, self.v_cache = list(k_cache), list(v_cache)
        inv, _ = rope.yarn_inv_freq(D, base=float(cfg.get("rope_base", 500000.0)))
        self.inv_freq = torch.from_numpy(inv).to(dev)
        self.seq_len = seq_len
        bf = torch.bfloat16
        if kv == "resident":
            self.st = DecodeStep(kr, self.k_cache, self.v_cache, seq_len, L, Hq, k,
                                 mode="indexed", force_last=force_last)
            self.kb = self.vb = None
        else:
            self.kb = torch.zeros((L, B, G, k, D), dtype=bf, device=dev)
            self.vb = torch.zeros_like(self.kb)
            self.st = DecodeStep(kr, [self.kb[l] for l in range(L)], [self.vb[l] for l in range(L)],
                                 seq_len, L, Hq, k, mode="slots", kv_rows=k,
                                 k_src_layers=self.k_cache, v_src_layers=self.v_cache,
                                 force_last=force_last)
            # the prefetch stream at high priority: its gathers' CTAs are scheduled ahead of
            # the next dense kernel's whenever SMs free up
            self._pf = torch.cuda.Stream(device=dev, priority=pf_priority)
            self._ev_sel = torch.cuda.Event()
            self._ev = [torch.cuda.Event() for _ in range(L)]
        self.st.set_frontend(ret["emb"], ret["norm_w"], ret["w_qk"], ret["inv_freq"],
                             ret["mscale"], ret.get("eps", 1e-5))
        self.scale = self.st.scale
        f32 = torch.float32
        self.h = torch.zeros((B, H), dtype=f32, device=dev)
        self.xn = torch.zeros((B, H), dtype=bf, device=dev)
        self.qkv = torch.zeros((B, (Hq + 2 * G) * D), dtype=bf, device=dev)
        self.q = torch.zeros((L, B, Hq, D), dtype=bf, device=dev)
        self.a = torch.zeros((B, Hq * D), dtype=bf, device=dev)
        self.o = torch.zeros((B, H), dtype=bf, device=dev)
        self.gu = torch.zeros((B, 2 * F), dtype=bf, device=dev)
        self.y = torch.zeros((B, F), dtype=bf, device=dev)
        self.logits = torch.zeros((B, V), dtype=bf, device=dev)
        self.out = self.st.outs[0]  # [L][B][Hq][D] f32 attention outputs (one buffer)
        self.lse = self.st.lses[0]
        self.parity = 0
        self.graphs = {}
        self.trace = trace_queries
        self.q_trace = None if trace_queries is None else torch.zeros_like(trace_queries[0])
        self.n_steps = 0

    @property
    def tokens(self):
        """tokens[p] [B] int32: the input token of the step with parity p."""
        return self.st.tokens

    def _attend(self, l: int, stream):
        st, p = self.st, self.parity_cur
        if self.kv == "resident":
            spc.sparse_decode_attn_kv(st.desc, self.q, spc.KV_INDEXED, st.idx[p], st.cnt[p],
                                      self.k, self.scale, self.out, self.lse, st.ws_attn,
                                      layer_begin=l, layer_end=l + 1, stream=stream)
        else:
            spc.sparse_decode_attn_kv(st.desc, self.q, spc.KV_SLOTS, None, st.cnt[p], self.k,
                                      self.scale, self.out, self.lse, st.ws_attn,
                                      layer_begin=l, layer_end=l + 1, stream=stream)

    def enqueue(self, parity: int, stream=None):
        """One decode step of parity p: input token tokens[p] at position seq_len - 1; writes
        the next token into tokens[1 - p] and advances seq_len."""
        main = torch.cuda.current_stream(self.dev) if stream is None else stream
        with torch.cuda.stream(main):  # the cuBLAS GEMMs run on torch's current stream
            self._enqueue(parity, main)

    def _enqueue(self, parity: int, main):
        w, st = self.w, self.st
        self.parity_cur = parity
        st.enqueue(parity, stream=main, attend=False, q_score=self.q_trace)  # front-end .. diff
        off = self.kv == "offload"
        if off and self.prefetch:
            # the elastic gathers of all layers, in layer order, on the prefetch stream
            self._ev_sel.record(main)
            self._pf.wait_event(self._ev_sel)
            for l in range(self.L):
                st._gather(l, l + 1, self._pf)
                self._ev[l].record(self._pf)
        spc.llm_embed(self.tokens[parity], w["emb"], self.h, stream=main)
        delta = None
        for l in range(self.L):
            spc.llm_add_rmsnorm(self.h, delta, w["ln1"][l], self.eps, self.xn, stream=main)
            torch.mm(self.xn, w["w_qkv"][l].t(), out=self.qkv)
            if off:
                if self.prefetch:
                    main.wait_event(self._ev[l])
                else:
                    st._gather(l, l + 1, main)
                spc.llm_rope_append(self.qkv, self.inv_freq, self.seq_len, self.Hq, self.G,
                                    self.q[l], self.k_cache[l], self.v_cache[l],
                                    slot_tok=st.slot_tok, k_buf=self.kb[l], v_buf=self.vb[l],
                                    stream=main)
            else:
                spc.llm_rope_append(self.qkv, self.inv_freq, self.seq_len, self.Hq, self.G,
                                    self.q[l], self.k_cache[l], self.v_cache[l], stream=main)
            self._attend(l, main)
            spc.llm_f32_to_bf16(self.out[l], self.a, stream=main)
            torch.mm(self.a, w["w_o"][l].t(), out=self.o)
            spc.llm_add_rmsnorm(self.h, self.o, w["ln2"][l], self.eps, self.xn, stream=main)
            torch.mm(self.xn, w["w_gu"][l].t(), out=self.gu)
            spc.llm_swiglu(self.gu, self.y, stream=main)
            torch.mm(self.y, w["w_down"][l].t(), out=self.o)
            delta = self.o
        spc.llm_add_rmsnorm(self.h, delta, w["norm"], self.eps, self.xn, stream=main)
        torch.mm(self.xn, w["lm_head"].t(), out=self.logits)
        spc.llm_argmax(self.logits, self.tokens[1 - parity], self.seq_len, stream=main)
        if off and self.prefetch:  # join the prefetch stream (graph capture needs it)
            main.wait_event(self._ev[self.L - 1])

    def step(self, use_graph: bool = False):
        """Run one step; returns the tokens tensor holding its output (tokens[1 - p])."""
        p = self.parity
        if self.trace is not None:
            self.q_trace.copy_(self.trace[self.n_steps % self.trace.shape[0]], non_blocking=True)
        self.n_steps += 1
        if use_graph:
            if p not in self.graphs:
                self.capture()
            self.graphs[p].replay()
        else:
            self.enqueue(p)
        self.parity ^= 1
        return self.tokens[1 - p]

    def capture(self):
        """Capture the even and the odd step as CUDA graphs (after an eager warm-up step)."""
        s = torch.cuda.Stream(device=self.dev)
        s.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(s):
            for p in (0, 1):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    self.enqueue(p, stream=s)
                self.graphs[p] = g
        torch.cuda.current_stream(self.dev).wait_stream(s)

    def reset(self, token0: torch.Tensor, seq_len0: torch.Tensor):
        """Start a sequence: the first token and seq_len (counting it); clears the selection
        state."""
        self.st.reset_state()
        self.parity = 0
        self.n_steps = 0
        self.tokens[0].copy_(token0)
        self.seq_len.copy_(seq_len0)

    def weight_bytes(self) -> int:
        w = self.w
        n = sum(t.numel() for key in ("ln1", "ln2", "w_qkv", "w_o", "w_gu", "w_down")
                for t in w[key])
        n += w["norm"].numel() + w["lm_head"].numel()
        return 2 * n
