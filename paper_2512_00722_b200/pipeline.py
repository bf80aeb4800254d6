"""One SpeContext decode step on one GPU, built only from libspc calls.

Step: spc_score (LOGITS, NORM, GROUP) -> spc_topk (force the
newest token, R10) -> spc_elastic_diff against the previous step's selection
 -> [SLOTS mode: spc_gather_kv of the new rows into budget slots] ->
spc_sparse_decode_attn_kv (TMA row gathers; spc_sparse_decode_attn for fp32) over all L
layers (one launch + its LSE merge).  In INDEXED mode with
Smax <= 135168 the NORM..diff calls are the single fused spc_select launch, and where
spc_score_select applies (config B) LOGITS through the diff are ONE persistent launch.

The step state (previous selection, slot map) ping-pongs between two buffers,
so two CUDA graphs (even / odd step) replay the whole step with one launch
each.  Inputs are written into fixed device buffers (``q_ret``, ``q_llm``)
before a replay; ``step_host`` is the end-to-end public call that takes pinned
host inputs and returns host outputs.
"""
from __future__ import annotations

import math

import torch

from . import spc


class DecodeStep:
    def __init__(self, kr: torch.Tensor, k_layers, v_layers, seq_len: torch.Tensor, L: int,
                 Hq: int, k: int, mode: str = "indexed", force_last: bool = True, scale=None,
                 kv_rows=None, k_src_layers=None, v_src_layers=None, fused=None,
                 src_rows=None, src_strides=None, retrieval: str = "head", one_launch=False,
                 prefetch_groups: int = 1):
        """kr: retrieval keys [B][G][Smax][D] bf16.  k_layers/v_layers: L tensors [B][G][rows][D]
        (INDEXED: the full caches; SLOTS: the budget buffers [B][G][k][D], with
        k_src_layers/v_src_layers the full caches, device or mapped host).  src_strides =
        (row_stride, bg_stride) in elements: the sources are strided views (e.g. the layers of
        token-major KV records) and the elastic load uses spc_gather_kv_strided.
        retrieval: "head" (head-level, the paper's choice: group max) or "batch"
        (batch-level: one set per request from the sum over all heads; NEXT-3).
        prefetch_groups (SLOTS): gather / attend the layers in this many groups, the gather of
        group j on a prefetch stream overlapping the attention of group j-1."""
        assert retrieval in ("head", "batch")
        self.retrieval = retrieval
        self.dev = kr.device
        # fused spc_select (one launch for NORM..diff) where it applies: INDEXED mode, Smax <=
        # 135168 and a multiple of 4, and every row's 8-CTA cluster resident in one wave
        # (B*G*8 <= SMs); otherwise the separate ABI calls.  Measured: config B (8 rows)
        # fused is faster; config C (128 rows: 7 waves of clusters) 2.03 ms fused vs 1.84 ms
        # with the grid-wide NORM / GROUP kernels + cluster top-k + diff.
        n_sm = torch.cuda.get_device_properties(kr.device).multi_processor_count
        self.fused = (mode == "indexed" and kr.shape[2] <= 135168 and kr.shape[2] % 4 == 0
                      and kr.shape[0] * kr.shape[1] * 8 <= n_sm and retrieval == "head") \
            if fused is None else fused
        self.B, self.G, self.Smax, self.D = kr.shape
        # one_launch: spc_score_select (LOGITS through the diff in ONE persistent cooperative
        # launch, bit-identical) instead of spc_score(LOGITS) + spc_select.  Off by default:
        # measured slower on config B (47 us in-kernel vs ~41 us for the two launches; its
        # three grid-wide barriers cost ~2 us each)
        self.one_launch = bool(one_launch) and (
            mode == "indexed" and retrieval == "head" and kr.dtype == torch.bfloat16
            and spc.score_select_supported(kr.shape[0], Hq, kr.shape[1], kr.shape[3], kr.shape[2], k))
        self.L, self.Hq, self.k = L, Hq, k
        self.alpha = Hq // self.G
        self.mode = mode
        self.force_last = force_last
        self.scale = float(torch.tensor(1.0 / math.sqrt(self.D), dtype=torch.float32)) \
            if scale is None else float(scale)
        self.kr, self.seq_len = kr, seq_len
        self.k_layers, self.v_layers = list(k_layers), list(v_layers)
        self.kv_dtype = self.k_layers[0].dtype
        self.rows = kv_rows if kv_rows is not None else self.k_layers[0].shape[2]
        self.k_tab = spc.ptr_table(self.k_layers, self.dev)
        self.v_tab = spc.ptr_table(self.v_layers, self.dev)
        # bf16 attention runs spc_sparse_decode_attn_kv (TMA row gathers) over per-layer
        # descriptors of the caches (INDEXED) or of the budget buffers (SLOTS)
        self.desc = self._make_desc(self.k_layers, self.v_layers, kr.shape[0], kr.shape[1],
                                    self.rows if mode != "slots" else k, kr.shape[3])
        if mode == "slots":
            assert k_src_layers is not None
            self.k_src, self.v_src = list(k_src_layers), list(v_src_layers)
            # pinned host tensors are device-addressable under UVA (zero-copy PCIe reads)
            self.k_src_tab = spc.ptr_table(self.k_src, self.dev)
            self.v_src_tab = spc.ptr_table(self.v_src, self.dev)
            self.src_rows = src_rows if src_rows is not None else self.k_src[0].shape[2]
            self.src_strides = src_strides
        # SLOTS: the layers are gathered and attended in `prefetch_groups` groups; with more
        # than one, group j's gather (prefetch stream) overlaps group j-1's attention
        n = max(1, min(int(prefetch_groups), L))
        self.layer_groups = [(L * j // n, L * (j + 1) // n) for j in range(n)]
        if mode == "slots" and n > 1:
            self._pf_stream = torch.cuda.Stream(device=kr.device)
            self._pf_events = [torch.cuda.Event() for _ in range(n + 1)]
        B, G, Hq, D, dev = self.B, self.G, Hq, self.D, self.dev
        f32, i32 = torch.float32, torch.int32
        # step inputs and outputs are double-buffered by step parity, so the host copies of
        # one step (step_host) overlap the neighbouring steps' kernels
        self.q_rets = [torch.zeros((B, Hq, D), dtype=torch.bfloat16, device=dev) for _ in range(2)]
        self.q_llms = [torch.zeros((L, B, Hq, D), dtype=self.kv_dtype, device=dev)
                       for _ in range(2)]
        self.logits = torch.zeros((B, Hq, self.Smax), dtype=f32, device=dev)
        self.head_max = torch.zeros((B, Hq), dtype=f32, device=dev)
        self.head_sumfix = torch.zeros((B, Hq), dtype=torch.int64, device=dev)
        self.gs = torch.zeros((B, G, self.Smax), dtype=f32, device=dev)
        self.idx = [torch.full((B, G, k), -1, dtype=i32, device=dev) for _ in range(2)]
        self.cnt = [torch.zeros((B, G), dtype=i32, device=dev) for _ in range(2)]
        self.load_tok = torch.full((B, G, k), -1, dtype=i32, device=dev)
        self.n_load = torch.zeros((B, G), dtype=i32, device=dev)
        self.slot_tok = torch.full((B, G, k), -1, dtype=i32, device=dev) if mode == "slots" else None
        self.load_slot = torch.full((B, G, k), -1, dtype=i32, device=dev) if mode == "slots" else None
        self.outs = [torch.zeros((L, B, Hq, D), dtype=f32, device=dev) for _ in range(2)]
        self.lses = [torch.zeros((L, B, Hq), dtype=f32, device=dev) for _ in range(2)]
        self.last = 0  # parity of the most recent step (out / lse / q_ret / q_llm views)
        self._h2d = self._d2h = None  # copy streams of step_host, created on first use
        self._ev = {}
        self.ws_score = spc.alloc_workspace(spc.score_workspace(B, Hq, self.Smax), dev)
        self.ws_ss = spc.alloc_workspace(
            spc.score_select_workspace(B, Hq, G, self.Smax) if self.one_launch else 1, dev)
        self.ws_topk = spc.alloc_workspace(spc.topk_workspace(B, G, self.Smax, k), dev)
        self.ws_attn = spc.alloc_workspace(spc.attn_workspace(L, B, Hq, D, k), dev)
        self.parity = 0
        # input sets: address-distinct copies of (kr, K, V) that the step can rotate through
        # (benchmarks use this instead of an L2 flush); set 0 is the one given above
        self.sets = [(self.kr, self.k_tab, self.v_tab, [self.k_layers, self.v_layers], self.desc)]
        self.cur_set = 0
        self.graphs = {}
        self.fe = None  # retrieval-head front-end (set_frontend)

    # the input buffers of the next step and the outputs of the most recent one
    @property
    def q_ret(self):
        return self.q_rets[self.parity]

    @property
    def q_llm(self):
        return self.q_llms[self.parity]

    @property
    def out(self):
        return self.outs[self.last]

    @property
    def lse(self):
        return self.lses[self.last]

    def _make_desc(self, k_layers, v_layers, B, G, rows, D):
        if self.kv_dtype != torch.bfloat16 or not k_layers[0].is_cuda:
            return None
        return spc.KvDesc(k_layers, v_layers, B, G, rows, D)

    def add_input_set(self, kr, k_layers, v_layers):
        """Register another (retrieval keys, K layers, V layers) copy; returns its index."""
        k_layers, v_layers = list(k_layers), list(v_layers)
        self.sets.append((kr, spc.ptr_table(k_layers, self.dev), spc.ptr_table(v_layers, self.dev),
                          [k_layers, v_layers],
                          self._make_desc(k_layers, v_layers, self.B, self.G, self.rows, self.D)))
        return len(self.sets) - 1

    def use_set(self, i: int):
        self.cur_set = i
        self.kr, self.k_tab, self.v_tab, _, self.desc = self.sets[i]

    def set_frontend(self, emb, norm_w, w_qk, inv_freq, mscale: float, eps: float = 1e-5):
        """Start every step with the retrieval head's front-end (spc_rethead_qk, NEXT-1): the
        step then takes token ids (tokens[parity], [B] int32) instead of retrieval queries;
        the front-end writes the query into q_rets[parity] and the token's key into row
        seq_len - 1 of the retrieval key cache (the newest position, Z6), then the step
        scores it -- seq_len is read on the device every step, so a growing context (seq_len
        advanced in place) appends every new key at its own row.  Graphs captured before this
        call are dropped."""
        self.fe = dict(emb=emb, norm_w=norm_w, w_qk=w_qk, inv=inv_freq, mscale=float(mscale),
                       eps=float(eps))
        self.tokens = [torch.zeros(self.B, dtype=torch.int32, device=self.dev) for _ in range(2)]
        self.graphs = {}

    # ------------------------------------------------------------------ eager
    def enqueue(self, parity: int, stream=None, q_ret=None, q_llm=None, attend: bool = True,
                q_score=None):
        """Enqueue one step writing the selection into idx[parity] (prev = idx[1-parity]).
        q_ret / q_llm: read the step's queries in place from these tensors instead of the
        step's own input buffers.  attend=False stops after the selection and the diff (the
        LLM decoder, llm.py, gathers and attends layer by layer between its dense layers).
        q_score: score this query instead of q_ret (the front-end still writes q_ret and
        appends its key; llm.py's trace-query benchmark mode)."""
        cur, prev = parity, 1 - parity
        q_ret = self.q_rets[parity] if q_ret is None else q_ret
        q_llm = self.q_llms[parity] if q_llm is None else q_llm
        out, lse = self.outs[parity], self.lses[parity]
        if self.fe is not None:  # token -> query + appended key (NEXT-1)
            f = self.fe
            # position = seq_len - 1, read on the device every step (pos = NULL): a loop that
            # advances seq_len in place appends each new key at its own row
            spc.rethead_qk(self.tokens[parity], f["emb"], f["norm_w"], f["eps"], f["w_qk"], f["inv"],
                           f["mscale"], None, self.Hq, self.G, q_ret, self.kr,
                           seq_len_out=self.seq_len, stream=stream)
        if q_score is not None:
            q_ret = q_score
        if self.one_launch:
            spc.score_select(q_ret, self.kr, self.seq_len, self.scale, self.k, self.head_max,
                             self.head_sumfix, self.gs, self.idx[cur], self.cnt[cur], self.idx[prev],
                             self.cnt[prev], self.load_tok, self.n_load, self.ws_ss,
                             force_last=self.force_last, stream=stream)
        elif self.fused:
            # LOGITS, then NORM + GROUP + top-k + diff in one cluster launch (spc_select)
            spc.score(q_ret, self.kr, self.seq_len, self.G, self.scale, self.logits,
                      self.head_max, self.head_sumfix, self.gs, self.ws_score,
                      phases=spc.SCORE_LOGITS, stream=stream)
            spc.select(self.logits, self.head_max, self.seq_len, self.G, self.k,
                       self.head_sumfix, self.gs, self.idx[cur], self.cnt[cur], self.idx[prev],
                       self.cnt[prev], self.load_tok, self.n_load, force_last=self.force_last,
                       stream=stream)
        else:
            spc.score(q_ret, self.kr, self.seq_len, self.G, self.scale, self.logits,
                      self.head_max, self.head_sumfix, self.gs, self.ws_score,
                      phases=spc.SCORE_ALL | (spc.SCORE_BATCH if self.retrieval == "batch" else 0),
                      stream=stream)
            spc.topk(self.gs, self.seq_len, self.k, self.idx[cur], self.cnt[cur], self.ws_topk,
                     force_last=self.force_last, stream=stream)
            spc.elastic_diff(self.idx[prev], self.cnt[prev], self.idx[cur], self.cnt[cur],
                             self.load_tok, self.n_load, slot_tok=self.slot_tok,
                             load_slot=self.load_slot, stream=stream)
        if not attend:
            return
        if self.mode == "slots":
            main = torch.cuda.current_stream(self.dev) if stream is None else stream
            groups = self.layer_groups
            if len(groups) == 1:
                self._gather(0, self.L, main)
                self._attn_slots(cur, q_llm, out, lse, 0, self.L, main)
            else:
                # asynchronous prefetch ("concurrent execution of computation and KV
                # cache prefetching"; elastic loading in that dataflow): the elastic
                # gather of layer group j runs on the prefetch stream while the attention of
                # group j - 1 runs on the step's stream; group j's attention waits only for
                # group j's gather event
                ev = self._pf_events
                ev[0].record(main)
                self._pf_stream.wait_event(ev[0])
                for j, (l0, l1) in enumerate(groups):
                    self._gather(l0, l1, self._pf_stream)
                    ev[j + 1].record(self._pf_stream)
                for j, (l0, l1) in enumerate(groups):
                    main.wait_event(ev[j + 1])
                    self._attn_slots(cur, q_llm, out, lse, l0, l1, main)
        elif self.desc is not None:
            spc.sparse_decode_attn_kv(self.desc, q_llm, spc.KV_INDEXED, self.idx[cur],
                                      self.cnt[cur], self.k, self.scale, out, lse, self.ws_attn,
                                      stream=stream)
        else:
            spc.sparse_decode_attn(q_llm, self.k_tab, self.v_tab, spc.KV_INDEXED,
                                   self.idx[cur], self.cnt[cur], self.rows, self.k, self.scale,
                                   out, lse, self.ws_attn, self.G, stream=stream)

    def _gather(self, l0, l1, stream):
        """The elastic load (O9) of layers [l0, l1): the new tokens' rows into their slots."""
        if self.src_strides is not None:
            spc.gather_kv_strided(self.k_src_tab, self.v_src_tab, self.src_strides[0],
                                  self.src_strides[1], self.L, self.B, self.G, self.D, self.k,
                                  self.load_tok, self.load_slot, self.n_load, self.k_tab,
                                  self.v_tab, layer_begin=l0, layer_end=l1, stream=stream)
        else:
            spc.gather_kv(self.k_src_tab, self.v_src_tab, self.L, self.B, self.G, self.D,
                          self.src_rows, self.k, self.load_tok, self.load_slot, self.n_load,
                          self.k_tab, self.v_tab, layer_begin=l0, layer_end=l1,
                          dtype=spc.BF16 if self.kv_dtype == torch.bfloat16 else spc.F32,
                          stream=stream)

    def _attn_slots(self, cur, q_llm, out, lse, l0, l1, stream):
        if self.desc is not None:
            spc.sparse_decode_attn_kv(self.desc, q_llm, spc.KV_SLOTS, None, self.cnt[cur], self.k,
                                      self.scale, out, lse, self.ws_attn, layer_begin=l0,
                                      layer_end=l1, stream=stream)
        else:
            spc.sparse_decode_attn(q_llm, self.k_tab, self.v_tab, spc.KV_SLOTS, None,
                                   self.cnt[cur], self.k, self.k, self.scale, out, lse,
                                   self.ws_attn, self.G, layer_begin=l0, layer_end=l1,
                                   stream=stream)

    def step(self, q_ret=None, q_llm=None, use_graph: bool = False):
        """Run one decode step on device tensors (copied into the step's input buffers)."""
        p = self.parity
        if q_ret is not None:
            self.q_rets[p].copy_(q_ret, non_blocking=True)
        if q_llm is not None:
            self.q_llms[p].copy_(q_llm, non_blocking=True)
        if use_graph:
            key = (self.cur_set, p)
            if key not in self.graphs:
                self.capture()
            self.graphs[key].replay()
        else:
            self.enqueue(p)
        self.last = p
        self.parity ^= 1
        return self.idx[p], self.cnt[p]

    def capture(self):
        """Capture the even and odd step of every input set as CUDA graphs (call after an
        eager warm-up so kernel attributes are set)."""
        keep = self.cur_set
        s = torch.cuda.Stream(device=self.dev)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for si in range(len(self.sets)):
                self.use_set(si)
                for p in (0, 1):
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=s):
                        self.enqueue(p)
                    self.graphs[(si, p)] = g
        torch.cuda.current_stream().wait_stream(s)
        self.use_set(keep)

    def capture_sequence(self, items, bounds=None):
        """CUDA graphs of a fixed input sequence: items[i] = (input set, q_ret, q_llm); step i
        runs with parity i % 2 (call reset_state() before replaying from step 0).  The kernels
        read each step's queries in place: no staging copies.  bounds: [(a, b), ...] index
        ranges, each captured as ONE graph of the consecutive steps a .. b-1 (a decode loop
        with no host work between steps: the steps' kernels then chain without a graph launch
        boundary); default one graph per step."""
        if bounds is None:
            bounds = [(i, i + 1) for i in range(len(items))]
        graphs = []
        keep = self.cur_set
        s = torch.cuda.Stream(device=self.dev)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for a, b in bounds:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    for i in range(a, b):
                        si, qr, ql = items[i]
                        self.use_set(si)
                        self.enqueue(i % 2, q_ret=qr, q_llm=ql)
                graphs.append(g)
        torch.cuda.current_stream().wait_stream(s)
        self.use_set(keep)
        return graphs

    def reset_state(self):
        for c in self.cnt:
            c.zero_()
        for i in self.idx:
            i.fill_(-1)
        if self.slot_tok is not None:
            self.slot_tok.fill_(-1)
        self.parity = 0

    # ------------------------------------------------------------------ end to end
    def step_host(self, q_ret_host: torch.Tensor, q_llm_host: torch.Tensor,
                  out_host: torch.Tensor, use_graph: bool = True):
        """Public end-to-end call: pinned host inputs -> step -> host attention output, all
        asynchronous.  The step's host->device copies run on one copy stream, its
        device->host read on another, ordered with events against the step's kernels, so
        consecutive calls overlap one step's copies with the neighbouring steps' kernels.
        `out_host` is complete after `sync_host()` (or a device synchronisation).
        With a front-end (set_frontend) `q_ret_host` holds the step's token ids [B] int32.
        Returns (bytes host->device, bytes device->host)."""
        main = torch.cuda.current_stream(self.dev)
        if self._h2d is None:
            self._h2d = torch.cuda.Stream(device=self.dev)
            self._d2h = torch.cuda.Stream(device=self.dev)
        p = self.parity
        ev = self._ev
        # inputs of parity p: the step two calls ago (same parity) must have consumed them
        if ("done", p) in ev:
            self._h2d.wait_event(ev[("done", p)])
        with torch.cuda.stream(self._h2d):
            if self.fe is not None:  # token ids instead of the retrieval query
                self.tokens[p].copy_(q_ret_host, non_blocking=True)
            else:
                self.q_rets[p].copy_(q_ret_host, non_blocking=True)
            self.q_llms[p].copy_(q_llm_host, non_blocking=True)
            ev[("in", p)] = torch.cuda.Event()
            ev[("in", p)].record(self._h2d)
        main.wait_event(ev[("in", p)])
        if ("read", p) in ev:  # outs[p] of two calls ago has been read back
            main.wait_event(ev[("read", p)])
        self.step(use_graph=use_graph)
        ev[("done", p)] = torch.cuda.Event()
        ev[("done", p)].record(main)
        self._d2h.wait_event(ev[("done", p)])
        with torch.cuda.stream(self._d2h):
            out_host.copy_(self.outs[p], non_blocking=True)
            ev[("read", p)] = torch.cuda.Event()
            ev[("read", p)].record(self._d2h)
        return (q_ret_host.numel() * q_ret_host.element_size() +
                q_llm_host.numel() * q_llm_host.element_size(),
                out_host.numel() * out_host.element_size())

    def sync_host(self):
        """Make every pending step_host copy part of the current stream's history."""
        if self._d2h is not None:
            torch.cuda.current_stream(self.dev).wait_stream(self._d2h)
            torch.cuda.current_stream(self.dev).wait_stream(self._h2d)
