"""Algorithm 2 at run time: progressive per-layer KV offload during decode (NEXT-2).

Paper §6.3: before each step, while the sequence length S has reached the next
compile-time threshold S^T_{L_CPU} (Algorithm 1, spc_plan_thresholds), the KV cache of layer
L - L_CPU - 1 is offloaded to CPU memory ("progressively offloads the KV cache of each LLM
layer to the CPU as the context length increases") and L_CPU grows by one.  Here
(readings R25-R27):

* resident layers [0, L - L_CPU) keep their full K/V caches in HBM and are attended in
  place through the selection (INDEXED, spc_sparse_decode_attn_kv);
* offloaded layers [L - L_CPU, L) live in pinned host memory as token-major records
  ([B][G][Smax][n_off][K,V][D], record slot i = the i-th offloaded layer) plus k-row HBM
  budget buffers; every step the elastic diff's new rows are gathered into their slots over
  PCIe (spc_gather_kv_strided) and the offloaded layers are attended from the buffers
  (SLOTS) -- the paper's "reuse ... in-place" elastic loading;
* one slot map per (b, g) row serves every offloaded layer (the selection is the same for
  all layers, reading R11); it is maintained from the first step, so a layer offloaded later
  fills its budget buffer from HBM through the current slot map (spc_gather_kv) before its
  HBM cache is released.

Every step of the path is a libspc call; the migration copy (HBM -> pinned host, once per
offloaded layer) is a plain device-to-host copy.
"""
from __future__ import annotations

import math

import torch

from . import spc


class OffloadingDecodeStep:
    def __init__(self, kr: torch.Tensor, k_layers, v_layers, seq_len: torch.Tensor, L: int,
                 Hq: int, k: int, thresholds, max_offload=None, force_last: bool = True,
                 scale=None):
        """kr [B][G][Smax][D] bf16; k_layers / v_layers: L HBM caches [B][G][Smax][D] bf16 (the
        step releases the ones it offloads); thresholds: Algorithm 1's S^T list (L + 1 values,
        spc_plan_thresholds or explicit); seq_len [B] int32 on the device, advanced by the
        caller; the step reads S = max(seq_len) from the host copy kept in `S`."""
        self.dev = kr.device
        self.B, self.G, self.Smax, self.D = kr.shape
        self.L, self.Hq, self.k = L, Hq, k
        self.kr, self.seq_len = kr, seq_len
        self.force_last = force_last
        self.scale = float(torch.tensor(1.0 / math.sqrt(self.D), dtype=torch.float32)) \
            if scale is None else float(scale)
        self.thresholds = [int(x) for x in thresholds]
        self.k_layers, self.v_layers = list(k_layers), list(v_layers)
        self.l_cpu = 0
        self.n_max = L if max_offload is None else int(max_offload)
        n_sm = torch.cuda.get_device_properties(kr.device).multi_processor_count
        self.fused = (self.Smax <= 135168 and self.Smax % 4 == 0 and
                      kr.shape[0] * kr.shape[1] * 8 <= n_sm)
        B, G, D, dev = self.B, self.G, self.D, self.dev
        i32, f32 = torch.int32, torch.float32
        self.q_llm_buf = None
        self.logits = torch.zeros((B, Hq, self.Smax), dtype=f32, device=dev)
        self.head_max = torch.zeros((B, Hq), dtype=f32, device=dev)
        self.head_sumfix = torch.zeros((B, Hq), dtype=torch.int64, device=dev)
        self.gs = torch.zeros((B, G, self.Smax), dtype=f32, device=dev)
        self.idx = [torch.full((B, G, k), -1, dtype=i32, device=dev) for _ in range(2)]
        self.cnt = [torch.zeros((B, G), dtype=i32, device=dev) for _ in range(2)]
        self.slot_tok = torch.full((B, G, k), -1, dtype=i32, device=dev)
        self.load_tok = torch.full((B, G, k), -1, dtype=i32, device=dev)
        self.load_slot = torch.full((B, G, k), -1, dtype=i32, device=dev)
        self.n_load = torch.zeros((B, G), dtype=i32, device=dev)
        self.out = torch.zeros((L, B, Hq, D), dtype=f32, device=dev)
        self.lse = torch.zeros((L, B, Hq), dtype=f32, device=dev)
        self.ws_score = spc.alloc_workspace(spc.score_workspace(B, Hq, self.Smax), dev)
        self.ws_topk = spc.alloc_workspace(spc.topk_workspace(B, G, self.Smax, k), dev)
        self.ws_attn = spc.alloc_workspace(spc.attn_workspace(L, B, Hq, D, k), dev)
        # budget buffers of every layer (k rows per (b, g): small) and their descriptors
        self.kb = torch.zeros((L, B, G, k, D), dtype=torch.bfloat16, device=dev)
        self.vb = torch.zeros_like(self.kb)
        self.kb_tab = spc.ptr_table([self.kb[l] for l in range(L)], dev)
        self.vb_tab = spc.ptr_table([self.vb[l] for l in range(L)], dev)
        self.desc_slots = spc.KvDesc([self.kb[l] for l in range(L)], [self.vb[l] for l in range(L)])
        self.desc_res = spc.KvDesc(self.k_layers, self.v_layers)
        self.host = None  # pinned token-major records of the offloaded layers (lazily)
        self.parity = 0
        self.last = 0
        self.migrations = []  # (S, layer, seconds) of every offload

    # ------------------------------------------------------------------ Algorithm 2
    def offload_due(self, S: int):
        """Layers Algorithm 2 offloads before a step at sequence length S."""
        l_cpu, layers = spc.plan_step(self.thresholds, self.L, S, self.l_cpu)
        return layers[: max(0, self.n_max - self.l_cpu)]

    def _host_records(self):
        if self.host is None:
            B, G, D = self.B, self.G, self.D
            self.host = torch.empty((B, G, self.Smax, self.n_max, 2, D), dtype=torch.bfloat16,
                                    pin_memory=True)
            self.src_k = [self.host[:, :, :, i, 0] for i in range(self.n_max)]
            self.src_v = [self.host[:, :, :, i, 1] for i in range(self.n_max)]
            # the records of offloaded layer l sit at record slot rec_slot[l]
            self.rec_slot = {}
        return self.host

    def migrate(self, layer: int):
        """KV_Cache_Offload(layer) (Algorithm 2 line 5): copy the layer's cache into its host
        record slot, fill its budget buffer through the current slot map (spc_gather_kv from
        HBM), then release the HBM cache."""
        import time
        t0 = time.perf_counter()
        host = self._host_records()
        i = len(self.rec_slot)
        self.rec_slot[layer] = i
        host[:, :, :, i, 0].copy_(self.k_layers[layer])  # device -> pinned host (once)
        host[:, :, :, i, 1].copy_(self.v_layers[layer])
        # budget slots of this layer = the rows of the current slot map (load_tok = slot_tok)
        B, G, k = self.B, self.G, self.k
        ar = torch.arange(k, dtype=torch.int32, device=self.dev).expand(B, G, k).contiguous()
        occupied = (self.slot_tok >= 0)
        lt = torch.where(occupied, self.slot_tok, torch.full_like(self.slot_tok, -1))
        order = torch.argsort((~occupied).to(torch.int8), dim=-1, stable=True)
        lt = torch.gather(lt, -1, order).contiguous()
        ls = torch.gather(ar, -1, order).contiguous()
        nl = occupied.sum(-1).to(torch.int32).contiguous()
        spc.gather_kv(spc.ptr_table(self.k_layers, self.dev), spc.ptr_table(self.v_layers, self.dev),
                      self.L, B, G, self.D, self.Smax, k, lt, ls, nl, self.kb_tab, self.vb_tab,
                      layer_begin=layer, layer_end=layer + 1)
        torch.cuda.synchronize(self.dev)
        # release the HBM cache: the resident descriptor no longer names this layer (offloaded
        # entries alias layer 0, never read: the resident range is [0, L - L_CPU))
        self.l_cpu += 1
        if self.l_cpu < self.L:
            self.k_layers[layer] = self.k_layers[0]
            self.v_layers[layer] = self.v_layers[0]
            self.desc_res = spc.KvDesc(self.k_layers, self.v_layers)
        else:  # everything offloaded
            self.k_layers, self.v_layers, self.desc_res = [], [], None
        self._src_tabs = None
        self.migrations.append((self.S_host, layer, time.perf_counter() - t0))

    # ------------------------------------------------------------------ one step
    def _gather_offloaded(self, stream=None):
        L, n = self.L, self.l_cpu
        if n == 0:
            return
        if self._src_tabs is None:
            # source tables indexed by layer: offloaded layer l reads its record slot
            ks = [self.src_k[self.rec_slot.get(l, 0)] for l in range(L)]
            vs = [self.src_v[self.rec_slot.get(l, 0)] for l in range(L)]
            self._src_tabs = (spc.ptr_table(ks, self.dev), spc.ptr_table(vs, self.dev))
        rec = self.n_max * 2 * self.D  # elements per token record
        spc.gather_kv_strided(self._src_tabs[0], self._src_tabs[1], rec, self.Smax * rec, L,
                              self.B, self.G, self.D, self.k, self.load_tok, self.load_slot,
                              self.n_load, self.kb_tab, self.vb_tab, layer_begin=L - n,
                              layer_end=L, stream=stream)

    def step(self, q_ret, q_llm, S: int, stream=None):
        """One decode step at sequence length S (= max seq_len, host int): Algorithm 2's
        offloads first, then selection (separate calls: the slot-map diff), the elastic
        gather of the offloaded layers, and the attention (resident INDEXED + offloaded
        SLOTS)."""
        self.S_host = int(S)
        if not hasattr(self, "_src_tabs"):
            self._src_tabs = None
        for layer in self.offload_due(self.S_host):
            self.migrate(layer)
        cur, prev = self.parity, 1 - self.parity
        if self.fused:  # LOGITS, then NORM..top-k in one cluster launch (spc_select)
            spc.score(q_ret, self.kr, self.seq_len, self.G, self.scale, self.logits, self.head_max,
                      self.head_sumfix, self.gs, self.ws_score, phases=spc.SCORE_LOGITS,
                      stream=stream)
            spc.select(self.logits, self.head_max, self.seq_len, self.G, self.k, self.head_sumfix,
                       self.gs, self.idx[cur], self.cnt[cur], self.idx[prev], self.cnt[prev],
                       self.load_tok, self.n_load, force_last=self.force_last, stream=stream)
        else:
            spc.score(q_ret, self.kr, self.seq_len, self.G, self.scale, self.logits, self.head_max,
                      self.head_sumfix, self.gs, self.ws_score, stream=stream)
            spc.topk(self.gs, self.seq_len, self.k, self.idx[cur], self.cnt[cur], self.ws_topk,
                     force_last=self.force_last, stream=stream)
        # the slot-map diff (O8 with slots): new rows -> freed slots of the offloaded layers
        spc.elastic_diff(self.idx[prev], self.cnt[prev], self.idx[cur], self.cnt[cur], self.load_tok,
                         self.n_load, slot_tok=self.slot_tok, load_slot=self.load_slot,
                         stream=stream)
        self._gather_offloaded(stream)
        L, n = self.L, self.l_cpu
        if n < L:
            spc.sparse_decode_attn_kv(self.desc_res, q_llm, spc.KV_INDEXED, self.idx[cur],
                                      self.cnt[cur], self.k, self.scale, self.out, self.lse,
                                      self.ws_attn, layer_begin=0, layer_end=L - n, stream=stream)
        if n > 0:
            spc.sparse_decode_attn_kv(self.desc_slots, q_llm, spc.KV_SLOTS, None, self.cnt[cur],
                                      self.k, self.scale, self.out, self.lse, self.ws_attn,
                                      layer_begin=L - n, layer_end=L, stream=stream)
        self.last = cur
        self.parity ^= 1
        return self.idx[cur], self.cnt[cur]

    # ------------------------------------------------------------------ graphs
    def capture(self, items, S: int):
        """One CUDA graph per steady-state step of a fixed input sequence, items[i] = (q_ret,
        q_llm), at sequence length S (no offload may be due: Algorithm 2 runs on the host
        before a step); step i runs with parity (current parity + i) % 2."""
        assert not self.offload_due(int(S)), "an offload is due: step() first"
        self.S_host = int(S)
        graphs = []
        s = torch.cuda.Stream(device=self.dev)
        s.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(s):
            for q_ret, q_llm in items:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    self.step(q_ret, q_llm, S)
                graphs.append(g)
        self.parity ^= len(items) & 1  # capture advanced the parity; replays advance it again
        torch.cuda.current_stream(self.dev).wait_stream(s)
        return graphs
