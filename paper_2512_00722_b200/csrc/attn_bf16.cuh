// attn_bf16.cuh — the bf16 sparse decode-attention kernel (included by attn.cu).
//
// Persistent, per-warp software-pipelined.  The selected rows of all groups
// (layer, b, g) form one virtual row space of n_groups * kpad rows (kpad = k
// rounded up to whole 64-row chunks; rows past a group's count are skipped).
// CTA c owns chunks [c * cpc, (c+1) * cpc); warp w of the CTA owns rows
// [16w, 16w+16) of every chunk.
//
// Each warp runs its own 3-deep cp.async ring (16-byte copies), gathering its
// rows straight from the KV cache (INDEXED: the row list comes from the
// selection; SLOTS: the budget buffers).  The row tokens, the group's valid-row
// count and the layer pointers of chunk j are fetched by the same warp with
// cp.async five chunks ahead inside the same per-iteration commit group, so no
// global-load latency is exposed and no CTA-wide barrier is needed per chunk.
// Measured alternatives: one TMA bulk copy per 256-byte row
// tops out near 1.8 TB/s (per-request cost of the TMA unit); a single producer
// warp issuing the 16-byte copies is issue-bound (~3.3 TB/s).
//
// Math per warp and chunk (mma.sync m16n8k16, fp32 accumulate):
//   S = Q K^T   A = Q (rows 0-7 = heads, alpha real), B = K rows (ldmatrix)
//   O += P V    A = [P_hi ; P_lo] (rows 0-7 = bf16(P), rows 8-15 = bf16(P - P_hi)),
//               so one mma accumulates both halves of a ~16-bit-mantissa P;
//               O = O_hi + O_lo at the end.  B = V rows (ldmatrix.trans).
// Online softmax in registers; the O rescale is skipped when no head's running
// max moved.  At the end of a group segment the 4 warps merge (the only CTA
// barriers) and write one (m, l, o) partial; the last CTA of a group merges the
// group's segments with the LSE rule (O12).
#pragma once

constexpr int CH = 64;      // rows per chunk (4 warps x 16)
constexpr int WR = 16;      // rows per warp per chunk
constexpr int NSTAGE = 3;   // per-warp ring depth (chunks in flight: NSTAGE - 1)
constexpr int NWARP = 4;
constexpr int AT2_THREADS = NWARP * 32;
constexpr int TRING = 8;    // per-warp ring of prefetched chunk metadata
constexpr int MAHEAD = 5;   // metadata fetched this many chunks before its rows are issued

template <int D, int ALPHA>
struct PSmem {
  static constexpr int RS = D + 8;                // padded row (bf16 elements): conflict-free ldmatrix
  static constexpr int KV_BYTES = WR * RS * 2;    // one of K or V, one warp, one stage
  static constexpr int STAGE = 2 * KV_BYTES;
  static constexpr int WARP_BYTES = NSTAGE * STAGE;
  // metadata ring per warp: [TRING] x {int tok[16]; int count; int pad; u64 kptr; u64 vptr}
  static constexpr int META = 96;  // 16-byte multiple: the token block is read as int4
  static constexpr int META_OFF = NWARP * WARP_BYTES;
  static constexpr int NV_OFF = META_OFF + NWARP * TRING * META;  // [NWARP][NSTAGE] int
  static constexpr int BYTES = NV_OFF + NWARP * NSTAGE * 4 + 16;
  static_assert(ALPHA * D * 4 + 64 * 4 <= STAGE, "flush scratch must fit in a warp stage");
};

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// D = A(16x16 bf16, row) * B(16x8 bf16, col) + D with all four A registers.
__device__ __forceinline__ void mma_bf16_4(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                           uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
      "{%8, %9}, {%0, %1, %2, %3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// Debug trace (spc_debug_set_trace; compiled in with -DSPC_TRACE): CTA 0 warp 0
// stamps %globaltimer per chunk: [i][0] rows of chunk i+2 issued, [i][1] chunk i
// landed, [i][2] chunk i computed.
__device__ unsigned long long* g_trace = nullptr;
__device__ __forceinline__ void trace(int i, int slot) {
#ifdef SPC_TRACE
  if (g_trace && blockIdx.x == 0 && threadIdx.x == 0 && i < 256) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    g_trace[i * 4 + slot] = t;
  }
#else
  (void)i;
  (void)slot;
#endif
}

// Position of a chunk, advanced incrementally (no division on the hot path):
// group index, chunk within the group, and the group's (layer, b*G+g).
struct ChunkIt {
  int grp, rc, lr, bg;
  __device__ __forceinline__ void next(int cpg, int BG) {
    if (++rc == cpg) {
      rc = 0;
      ++grp;
      if (++bg == BG) {
        bg = 0;
        ++lr;
      }
    }
  }
};

template <int D, int ALPHA>
__global__ void __launch_bounds__(AT2_THREADS, 2) attn_bf16_kernel(
    const uint16_t* __restrict__ q, const void* const* __restrict__ k_layers,
    const void* const* __restrict__ v_layers, int kv_mode, const int32_t* __restrict__ idx,
    const int32_t* __restrict__ count, int layer_begin, int B, int G, int rows, int kbud, int kpad,
    float scale, int cpc, int n_groups, int segstride, float* __restrict__ part_o,
    float* __restrict__ part_ml, unsigned* __restrict__ cnt, float* __restrict__ out,
    float* __restrict__ lse) {
  using SM = PSmem<D, ALPHA>;
  constexpr int RS = SM::RS;
  constexpr int KS = D / 16;
  constexpr int VPR = D * 2 / 16;  // 16-byte vectors per row = lanes per row
  constexpr int NG = 32 / VPR;     // lane groups (rows per warp-wide copy instruction)
  constexpr int RPL = WR / NG;     // rows per lane group per chunk
  extern __shared__ __align__(128) uint8_t at_smem[];
  __shared__ int flag;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int BG = B * G, Hq = G * ALPHA;
  const int cpg = kpad / CH;              // chunks per group
  const int c_begin = blockIdx.x * cpc;  // first (global) chunk of this CTA
  const int n_chunks = min(cpc, n_groups * cpg - c_begin);
  if (n_chunks <= 0) return;
  ChunkIt it0;
  it0.grp = c_begin / cpg;
  it0.rc = c_begin - it0.grp * cpg;
  it0.lr = it0.grp / BG;
  it0.bg = it0.grp - it0.lr * BG;
  const bool ind = kv_mode == SPC_KV_INDEXED;
  uint8_t* wbase = at_smem + (size_t)warp * SM::WARP_BYTES;
  const uint32_t wsb = smem_u32(wbase);
  uint8_t* meta = at_smem + SM::META_OFF + (size_t)warp * TRING * SM::META;
  int* nv_ring = (int*)(at_smem + SM::NV_OFF) + warp * NSTAGE;
  const int lg = lane / VPR, col = lane % VPR;  // lane group (row block) and 16-byte column

  // zero this warp's K/V ring once: skipped rows then hold finite (zero or stale) data
  for (int i = lane; i < SM::WARP_BYTES / 16; i += 32)
    *(uint4*)(wbase + (size_t)i * 16) = make_uint4(0, 0, 0, 0);
  __syncwarp();

  // ---- metadata of chunk j -> meta slot j % TRING  (j = 0, 1, 2, ... in order)
  ChunkIt it_meta = it0;
  auto fetch_meta = [&](int j) {
    const ChunkIt c = it_meta;
    it_meta.next(cpg, BG);
    if (j >= n_chunks) return;
    const uint32_t m = smem_u32(meta + (j & (TRING - 1)) * SM::META);
    const int r = c.rc * CH + warp * WR + lane;
    if (lane < WR) {
      if (ind && r < kbud) cp_async4(m + lane * 4, idx + (size_t)c.bg * kbud + r);
    } else if (lane == WR) {
      cp_async4(m + 64, count + c.bg);
    } else if (lane == WR + 1) {
      cp_async8(m + 72, k_layers + layer_begin + c.lr);
    } else if (lane == WR + 2) {
      cp_async8(m + 80, v_layers + layer_begin + c.lr);
    }
  };
  // ---- rows of chunk j -> stage s_iss (requires meta of chunk j landed)
  ChunkIt it_rows = it0;
  int s_iss = 0, cached_grp = -1, cnt_g = 0;
  const uint16_t *Kcol = nullptr, *Vcol = nullptr;
  auto issue_rows = [&](int j) {
    const ChunkIt c = it_rows;
    it_rows.next(cpg, BG);
    const int s = s_iss;
    s_iss = s_iss == NSTAGE - 1 ? 0 : s_iss + 1;
    if (j >= n_chunks) return;
    const uint8_t* m = meta + (j & (TRING - 1)) * SM::META;
    if (c.grp != cached_grp) {  // group-invariant values, cached in registers
      cached_grp = c.grp;
      cnt_g = min(*(const int*)(m + 64), kbud);
      Kcol = *(const uint16_t* const*)(m + 72) + (size_t)c.bg * rows * D + col * 8;
      Vcol = *(const uint16_t* const*)(m + 80) + (size_t)c.bg * rows * D + col * 8;
    }
    const int r0 = c.rc * CH;
    const int nvalid = max(0, min(cnt_g - r0, CH));
    if (lane == 0) nv_ring[s] = nvalid;
    const int nrows = min(max(nvalid - warp * WR - lg * RPL, 0), RPL);  // this lane group
    int tok[RPL];
    if (ind) {
#pragma unroll
      for (int t = 0; t < RPL; t += 4) {
        const int4 v = *(const int4*)(m + (lg * RPL + t) * 4);
        tok[t] = v.x;
        tok[t + 1] = v.y;
        tok[t + 2] = v.z;
        tok[t + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int t = 0; t < RPL; ++t) tok[t] = r0 + warp * WR + lg * RPL + t;
    }
    const uint32_t dst = wsb + (uint32_t)s * SM::STAGE + (uint32_t)((lg * RPL * RS + col * 8) * 2);
#pragma unroll
    for (int t = 0; t < RPL; ++t) {
      if (t < nrows) {
        cp_async16(dst + t * RS * 2, Kcol + (size_t)tok[t] * D);
        cp_async16(dst + SM::KV_BYTES + t * RS * 2, Vcol + (size_t)tok[t] * D);
      }
    }
  };
  // query fragments (A operand, row = head gid) of group grp
  uint32_t qa0[KS], qa2[KS], qn0[KS], qn2[KS];
  auto load_q = [&](int lr, int bg, uint32_t (&a0)[KS], uint32_t (&a2)[KS]) {
    const int b = bg / G, g = bg - (bg / G) * G;
    const uint16_t* qh =
        q + (((size_t)(layer_begin + lr) * B + b) * Hq + g * ALPHA + (gid < ALPHA ? gid : 0)) * D;
#pragma unroll
    for (int k = 0; k < KS; ++k) {
      const uint32_t x0 = __ldg((const unsigned int*)(qh + k * 16 + 2 * tig));
      const uint32_t x2 = __ldg((const unsigned int*)(qh + k * 16 + 8 + 2 * tig));
      a0[k] = gid < ALPHA ? x0 : 0u;
      a2[k] = gid < ALPHA ? x2 : 0u;
    }
  };

  // ---- prologue: metadata of chunks 0 .. MAHEAD+1, rows of chunks 0 and 1
  for (int j = 0; j < MAHEAD; ++j) fetch_meta(j);
  cp_async_commit();
  cp_async_wait<0>();
  __syncwarp();
  issue_rows(0);
  fetch_meta(MAHEAD);
  cp_async_commit();
  issue_rows(1);
  fetch_meta(MAHEAD + 1);
  cp_async_commit();
  load_q(it0.lr, it0.bg, qa0, qa2);

  const float sl2 = scale * LOG2E;
  float m_run = -INFINITY, l_run = 0.f;
  float o[D / 8][4];  // [n-tile][c0..c3]: c0,c1 = hi half (heads), c2,c3 = lo half
#pragma unroll
  for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  const int mi = lane >> 3, ri = lane & 7;
  const uint32_t a_off = (uint32_t)(((ri + ((mi & 2) ? 8 : 0)) * RS + ((mi & 1) ? 8 : 0)) * 2);
  const uint32_t b_off = (uint32_t)(((ri + ((mi & 1) ? 8 : 0)) * RS + ((mi & 2) ? 8 : 0)) * 2);
  ChunkIt it_cur = it0;
  int s_cur = 0;

  for (int i = 0; i < n_chunks; ++i) {
    // commit group G_i = {rows of chunk i+2, meta of chunk i+2+MAHEAD};
    // the meta of chunk i+2 is in G_{i-MAHEAD} (or the prologue)
    cp_async_wait<2>();
    __syncwarp();
    issue_rows(i + 2);
    fetch_meta(i + 2 + MAHEAD);
    cp_async_commit();
    trace(i, 0);
    const ChunkIt cc = it_cur;
    const bool grp_end = (i == n_chunks - 1) || (cc.rc == cpg - 1);
    it_cur.next(cpg, BG);
    if (grp_end && i + 1 < n_chunks) load_q(it_cur.lr, it_cur.bg, qn0, qn2);  // next group, early
    cp_async_wait<2>();  // rows of chunk i (G_{i-2}) landed
    __syncwarp();
    trace(i, 1);
    const int nv_w = nv_ring[s_cur] - warp * WR;  // valid rows of this warp in the chunk
    const uint32_t st = wsb + (uint32_t)s_cur * SM::STAGE;
    if (nv_w > 0) {
      // ---- S = Q K^T for this warp's 16 rows: two n8 tiles, two accumulator chains each
      float c0[4] = {0, 0, 0, 0}, c1[4] = {0, 0, 0, 0}, d0[4] = {0, 0, 0, 0},
            d1[4] = {0, 0, 0, 0};
#pragma unroll
      for (int k = 0; k < KS; k += 2) {
        uint32_t b0, b1, b2, b3, e0, e1, e2, e3;
        ldsm_x4(st + a_off + k * 32, b0, b1, b2, b3);
        ldsm_x4(st + a_off + (k + 1) * 32, e0, e1, e2, e3);
        mma_bf16(c0, qa0[k], qa2[k], b0, b1);
        mma_bf16(c1, qa0[k], qa2[k], b2, b3);
        mma_bf16(d0, qa0[k + 1], qa2[k + 1], e0, e1);
        mma_bf16(d1, qa0[k + 1], qa2[k + 1], e2, e3);
      }
      const int rr0 = 2 * tig;
      float sv[4] = {rr0 < nv_w ? (c0[0] + d0[0]) * sl2 : -INFINITY,
                     rr0 + 1 < nv_w ? (c0[1] + d0[1]) * sl2 : -INFINITY,
                     rr0 + 8 < nv_w ? (c1[0] + d1[0]) * sl2 : -INFINITY,
                     rr0 + 9 < nv_w ? (c1[1] + d1[1]) * sl2 : -INFINITY};
      float mx = fmaxf(fmaxf(sv[0], sv[1]), fmaxf(sv[2], sv[3]));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      const float m_new = fmaxf(m_run, mx);  // finite: row 0 of this warp is valid
      if (__any_sync(0xffffffffu, m_new > m_run)) {
        const float corr = exp2f(m_run - m_new);
        l_run *= corr;
#pragma unroll
        for (int d = 0; d < D / 8; ++d) {
          o[d][0] *= corr;
          o[d][1] *= corr;
          o[d][2] *= corr;
          o[d][3] *= corr;
        }
        m_run = m_new;
      }
      float p[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        p[e] = exp2f(sv[e] - m_run);
        l_run += p[e];
      }
      // ---- O += P V with A = [P_hi ; P_lo]
      const uint32_t ah0 = pack_bf16(p[0], p[1]), ah2 = pack_bf16(p[2], p[3]);
      const float2 h0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ah0));
      const float2 h2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ah2));
      const uint32_t al0 = pack_bf16(p[0] - h0.x, p[1] - h0.y);
      const uint32_t al2 = pack_bf16(p[2] - h2.x, p[3] - h2.y);
      const uint32_t vst = st + SM::KV_BYTES + b_off;
#pragma unroll
      for (int dn = 0; dn < D / 16; ++dn) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(vst + dn * 32, b0, b1, b2, b3);
        mma_bf16_4(o[2 * dn], ah0, al0, ah2, al2, b0, b1);
        mma_bf16_4(o[2 * dn + 1], ah0, al0, ah2, al2, b2, b3);
      }
    }
    trace(i, 2);
    // ---- flush at the end of this CTA's segment of the group
    if (grp_end) {
      __syncwarp();  // this warp's ldmatrix reads of stage s_cur are done: reuse it as scratch
      float* sm_m = (float*)(wbase + (size_t)s_cur * SM::STAGE);  // [8]
      float* sm_l = sm_m + 8;                                     // [8]
      float* sm_o = sm_m + 64;                                    // [ALPHA][D]
      float lsum = l_run;
      lsum += __shfl_xor_sync(0xffffffffu, lsum, 1);
      lsum += __shfl_xor_sync(0xffffffffu, lsum, 2);
      if (tig == 0) {
        sm_m[gid] = m_run;
        sm_l[gid] = lsum;
      }
      if (gid < ALPHA) {
#pragma unroll
        for (int d = 0; d < D / 8; ++d) {
          sm_o[gid * D + 8 * d + 2 * tig] = o[d][0] + o[d][2];
          sm_o[gid * D + 8 * d + 2 * tig + 1] = o[d][1] + o[d][3];
        }
      }
      __syncthreads();
      const int b = cc.bg / G, g = cc.bg - (cc.bg / G) * G;
      const int first = (cc.grp * cpg) / cpc;
      const int last = (cc.grp * cpg + cpg - 1) / cpc;
      const int seg = blockIdx.x - first;
      const size_t head_base = ((size_t)cc.lr * B + b) * Hq + g * ALPHA;
      for (int t = tid; t < ALPHA * D; t += AT2_THREADS) {
        const int j = t / D, d = t % D;
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < NWARP; ++w)
          M = fmaxf(M, ((const float*)(at_smem + (size_t)w * SM::WARP_BYTES +
                                       (size_t)s_cur * SM::STAGE))[j]);
        float acc = 0.f, lacc = 0.f;
        if (M != -INFINITY) {
#pragma unroll
          for (int w = 0; w < NWARP; ++w) {
            const float* ws_ =
                (const float*)(at_smem + (size_t)w * SM::WARP_BYTES + (size_t)s_cur * SM::STAGE);
            const float mw = ws_[j];
            if (mw == -INFINITY) continue;
            const float f = exp2f(mw - M);
            acc += f * ws_[64 + j * D + d];
            lacc += f * ws_[8 + j];
          }
        }
        part_o[((head_base + j) * segstride + seg) * D + d] = acc;
        if (d == 0) {
          part_ml[((head_base + j) * segstride + seg) * 2] = M;
          part_ml[((head_base + j) * segstride + seg) * 2 + 1] = lacc;
        }
      }
      if (last_block_ticket(&cnt[cc.grp], last - first + 1, &flag))
        merge_partials<D, ALPHA>(part_o, part_ml, last - first + 1, segstride, head_base, out, lse,
                                 ((size_t)(layer_begin + cc.lr) * B + b) * Hq + g * ALPHA,
                                 AT2_THREADS);
      __syncthreads();  // scratch (stage s_cur) reads done before the ring refills it
      m_run = -INFINITY;
      l_run = 0.f;
#pragma unroll
      for (int d = 0; d < D / 8; ++d) o[d][0] = o[d][1] = o[d][2] = o[d][3] = 0.f;
      if (i + 1 < n_chunks) {
#pragma unroll
        for (int k = 0; k < KS; ++k) {
          qa0[k] = qn0[k];
          qa2[k] = qn2[k];
        }
      }
    }
    s_cur = s_cur == NSTAGE - 1 ? 0 : s_cur + 1;
  }
  cp_async_wait<0>();
}
