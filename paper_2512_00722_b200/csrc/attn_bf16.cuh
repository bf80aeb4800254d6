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
// Math per warp and chunk (mma.sync m16n8k16, fp32 accumulate), both products
// transposed so the 16 K/V rows fill the M dimension:
//   S^T = K Q^T   A = the chunk's 16 K rows (ldmatrix), B = Q^T (n = head; heads
//                 >= alpha are zero).  8 HMMA per chunk for D = 128.
//   O^T += V^T P  A = V^T (ldmatrix.trans of the V rows, one m-tile per 16 dims),
//                 B = P (k = row, n = column): columns n < alpha hold bf16(P) of head
//                 n, columns alpha <= n < 2 alpha hold bf16(P - bf16(P)) (the lo part),
//                 so one MMA accumulates both halves of a ~16-bit-mantissa P; alpha = 8
//                 fills all 8 columns with hi parts and runs the lo parts as a second
//                 MMA.  The S^T accumulator fragment is moved into the B-fragment
//                 layout with two movmatrix.trans.  O = O_hi + O_lo at the flush.
// Online softmax in registers (each lane tracks the two heads of its columns); the
// O rescale is skipped when no head's running max moved.  At the end of a group
// segment every warp writes its own (m, l, o) partial with plain stores -- no CTA
// barrier, fence or ticket inside the kernel, so no warp's load stream ever waits
// for another (a CTA-wide flush measured ~5-8 us of stalled loads per group end) --
// and merge_groups_kernel (next launch, PDL) merges each group's partials with the
// LSE rule (O12).
#pragma once

constexpr int CH = 64;      // rows per chunk (4 warps x 16)
constexpr int WR = 16;      // rows per warp per chunk
#ifndef SPC_ATTN_NSTAGE
#define SPC_ATTN_NSTAGE 3
#endif
#ifndef SPC_ATTN_CTAS
#define SPC_ATTN_CTAS 2
#endif
#ifndef SPC_ATTN_PF
#define SPC_ATTN_PF 1  // chunks of L2 prefetch ahead of the cp.async issue point
#endif
constexpr int NSTAGE = SPC_ATTN_NSTAGE;  // per-warp ring depth (chunks in flight: NSTAGE - 1)
// 8 warps/SM.  (3 CTAs x 2 stages measured slower: 70 vs 62 us for config B.)
constexpr int AT2_CTAS_PER_SM = SPC_ATTN_CTAS;
constexpr int NWARP = 4;
constexpr int AT2_THREADS = NWARP * 32;
#ifndef SPC_ATTN_TRING
#define SPC_ATTN_TRING 8
#endif
#ifndef SPC_ATTN_MAHEAD
#define SPC_ATTN_MAHEAD 5
#endif
constexpr int TRING = SPC_ATTN_TRING;    // per-warp ring of prefetched chunk metadata
constexpr int MAHEAD = SPC_ATTN_MAHEAD;  // metadata fetched this many chunks before its rows are issued
static_assert(TRING >= MAHEAD + NSTAGE, "metadata ring too small");
// the prefetch of chunk i + NSTAGE - 1 + PF at iteration i reads metadata that landed
static_assert(SPC_ATTN_PF <= MAHEAD - NSTAGE, "prefetch needs landed metadata");

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
__device__ __forceinline__ uint32_t movm_t(uint32_t a) {
  uint32_t d;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(d) : "r"(a));
  return d;
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
// Also: lane 0 of every warp stamps its start / end at g_trace[1024 + (cta * 4 + warp) * 2].
__device__ unsigned long long* g_trace = nullptr;
__device__ __forceinline__ void trace(int i, int slot) {
#ifdef SPC_TRACE
  if (g_trace && blockIdx.x == 105 && threadIdx.x == 0 && i < 256) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    g_trace[i * 4 + slot] = t;
  }
#else
  (void)i;
  (void)slot;
#endif
}
__device__ __forceinline__ void trace_warp(int which) {
#ifdef SPC_TRACE
  if (g_trace && (threadIdx.x & 31) == 0 && blockIdx.x < 1024) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    g_trace[1024 + (blockIdx.x * 4 + (threadIdx.x >> 5)) * 2 + which] = t;
  }
#else
  (void)which;
#endif
}

// LSE merge (O12) of the np partials of one group by one CTA of NT threads, latency-
// friendly: the weights w_p = exp2(m_p - M) of every head are computed once into shared
// scratch (sm: >= ALPHA * (np + 1) floats), then each thread issues all the loads of
// its R output elements at once.
template <int D, int ALPHA, int NT>
__device__ void merge_group_fast(const float* __restrict__ part_o,
                                 const float* __restrict__ part_ml, int np, int segstride,
                                 size_t head_base, float* __restrict__ out,
                                 float* __restrict__ lse, size_t out_base, float* sm) {
  constexpr int R = (ALPHA * D + NT - 1) / NT;  // outputs per thread (the last may be idle)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  float* w = sm;                  // [ALPHA][np]
  float* inv = sm + ALPHA * np;   // [ALPHA]
  for (int j = warp; j < ALPHA; j += NT / 32) {
    const float* ml = part_ml + (head_base + j) * segstride * 2;
    float M = -INFINITY;
    for (int p = lane; p < np; p += 32) M = fmaxf(M, __ldcg(ml + 2 * p));
    M = warp_max(M);
    float den = 0.f;
    for (int p = lane; p < np; p += 32) {
      const float m = __ldcg(ml + 2 * p);
      const float wp = m == -INFINITY ? 0.f : exp2f(m - M);
      w[j * np + p] = wp;
      den += wp * __ldcg(ml + 2 * p + 1);
    }
    den = warp_sum(den);
    if (lane == 0) {
      inv[j] = den > 0.f ? 1.f / den : 0.f;
      if (lse) lse[out_base + j] = den > 0.f ? (M + log2f(den)) * 0.6931471805599453f : -INFINITY;
    }
  }
  __syncthreads();
  float num[R];
#pragma unroll
  for (int r = 0; r < R; ++r) num[r] = 0.f;
  for (int p0 = 0; p0 < np; p0 += 4) {
    float v[R][4];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = min(tid + r * NT, ALPHA * D - 1), j = i / D, d = i - (i / D) * D;
      const float* po = part_o + ((head_base + j) * segstride + p0) * D + d;
#pragma unroll
      for (int u = 0; u < 4; ++u) v[r][u] = p0 + u < np ? __ldcg(po + (size_t)u * D) : 0.f;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int j = min(tid + r * NT, ALPHA * D - 1) / D;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (p0 + u < np) num[r] += w[j * np + p0 + u] * v[r][u];
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = tid + r * NT, j = i / D, d = i - (i / D) * D;
    if (i < ALPHA * D) out[(out_base + j) * D + d] = num[r] * inv[j];
  }
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
__global__ void __launch_bounds__(AT2_THREADS, AT2_CTAS_PER_SM) attn_bf16_kernel(
    const uint16_t* __restrict__ q, const void* const* __restrict__ k_layers,
    const void* const* __restrict__ v_layers, int kv_mode, const int32_t* __restrict__ idx,
    const int32_t* __restrict__ count, int layer_begin, int B, int G, int rows, int kbud, int kpad,
    float scale, int cpc, int n_groups, int segstride, float* __restrict__ part_o,
    float* __restrict__ part_ml, unsigned* __restrict__ cnt, float* __restrict__ out,
    float* __restrict__ lse) {
  spc_pdl_entry();
  using SM = PSmem<D, ALPHA>;
  constexpr int RS = SM::RS;
  constexpr int KS = D / 16;
  constexpr int VPR = D * 2 / 16;  // 16-byte vectors per row = lanes per row
  constexpr int NG = 32 / VPR;     // lane groups (rows per warp-wide copy instruction)
  constexpr int RPL = WR / NG;     // rows per lane group per chunk
  extern __shared__ __align__(128) uint8_t at_smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int BG = B * G, Hq = G * ALPHA;
  const int cpg = kpad / CH;              // chunks per group
  const int c_begin = blockIdx.x * cpc;  // first (global) chunk of this CTA
  const int n_chunks = min(cpc, n_groups * cpg - c_begin);
  if (n_chunks <= 0) return;
  trace_warp(0);
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
  // ---- L2 prefetch of the rows of chunk j (SPC_ATTN_PF chunks ahead of their cp.async):
  // the DRAM latency is paid by a prefetch that holds no shared memory or registers, so
  // the cp.async ring waits only on L2 latency.  Lanes 0-15: K rows, 16-31: V rows.
  ChunkIt it_pf = it0;
  auto prefetch_rows = [&](int j) {
    const ChunkIt c = it_pf;
    it_pf.next(cpg, BG);
    if (j >= n_chunks) return;
    const uint8_t* m = meta + (j & (TRING - 1)) * SM::META;
    const int rr = lane & 15;
    const int r = c.rc * CH + warp * WR + rr;
    if (r >= min(*(const int*)(m + 64), kbud)) return;
    const int tok = ind ? *(const int*)(m + rr * 4) : r;
    const uint16_t* base = *(const uint16_t* const*)(m + (lane < 16 ? 72 : 80));
    const uint16_t* row = base + ((size_t)c.bg * rows + tok) * D;
    asm volatile("prefetch.global.L2 [%0];" ::"l"(row) : "memory");
    if (D * 2 > 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(row + 64) : "memory");
  };
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
#ifdef SPC_DEBUG  // selected rows must be cache rows; a bad one is not read
#pragma unroll
    for (int t = 0; t < RPL; ++t)
      if (t < nrows) {
        SPC_DCHECK(tok[t] >= 0 && tok[t] < rows, SPC_E_RANGE);
        if (tok[t] < 0 || tok[t] >= rows) tok[t] = 0;
      }
#endif
    const uint32_t dst = wsb + (uint32_t)s * SM::STAGE + (uint32_t)((lg * RPL * RS + col * 8) * 2);
#pragma unroll
    for (int t = 0; t < RPL; ++t) {
      if (t < nrows) {
        cp_async16(dst + t * RS * 2, Kcol + (size_t)tok[t] * D);
        cp_async16(dst + SM::KV_BYTES + t * RS * 2, Vcol + (size_t)tok[t] * D);
      }
    }
  };
  // query fragments: the B operand of S^T = K Q^T (k = dim, n = head gid; heads >= ALPHA
  // are zero): b0 = Q[gid][16k + 2tig ..], b1 = Q[gid][16k + 8 + 2tig ..]
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

  // ---- prologue: metadata of chunks 0 .. MAHEAD+NSTAGE-2, rows of chunks 0 .. NSTAGE-2
  for (int j = 0; j < MAHEAD; ++j) fetch_meta(j);
  cp_async_commit();
  cp_async_wait<0>();
  __syncwarp();
#if SPC_ATTN_PF > 0
  for (int j = 0; j < NSTAGE - 1; ++j) it_pf.next(cpg, BG);  // rows issued below directly
  for (int j = NSTAGE - 1; j < NSTAGE - 1 + SPC_ATTN_PF; ++j) prefetch_rows(j);
#endif
#pragma unroll
  for (int j = 0; j < NSTAGE - 1; ++j) {
    issue_rows(j);
    fetch_meta(MAHEAD + j);
    cp_async_commit();
  }
  load_q(it0.lr, it0.bg, qa0, qa2);

  // P columns n = 2 tig + slot of this lane: mode 0 = hi part of head hd[slot], 1 = lo
  // part, 2 = zero column.  The S^T values of head h sit in lane (gid, h / 2), slot h % 2.
  constexpr bool LOSEP = ALPHA == 8;
  constexpr int NACC = LOSEP ? 2 : 1;
  const int srcl = LOSEP ? lane : ((lane & ~3) | (ALPHA == 4 ? (tig & 1) : 0));
  int cmode[2], hd[2];
#pragma unroll
  for (int sl = 0; sl < 2; ++sl) {
    const int n = 2 * tig + sl;
    cmode[sl] = LOSEP ? 0 : (n < ALPHA ? 0 : (n < 2 * ALPHA ? 1 : 2));
    hd[sl] = LOSEP ? n : n % ALPHA;
  }
  const float sl2 = scale * LOG2E;
  float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};
  float o[NACC][D / 16][4];  // O^T[16 mt + gid (+8)][column 2 tig (+1)]
#pragma unroll
  for (int a = 0; a < NACC; ++a)
#pragma unroll
    for (int i = 0; i < D / 16; ++i) o[a][i][0] = o[a][i][1] = o[a][i][2] = o[a][i][3] = 0.f;
  const int mi = lane >> 3, ri = lane & 7;
  const uint32_t a_off = (uint32_t)(((ri + ((mi & 2) ? 8 : 0)) * RS + ((mi & 1) ? 8 : 0)) * 2);
  const uint32_t b_off = (uint32_t)(((ri + ((mi & 1) ? 8 : 0)) * RS + ((mi & 2) ? 8 : 0)) * 2);
  ChunkIt it_cur = it0;
  int s_cur = 0;

  for (int i = 0; i < n_chunks; ++i) {
    // commit group G_i = {rows of chunk i+NSTAGE-1, meta of chunk i+NSTAGE-1+MAHEAD};
    // the meta of chunk i+NSTAGE-1 is in G_{i-MAHEAD} (or the prologue)
    cp_async_wait<NSTAGE - 1>();
    __syncwarp();
    issue_rows(i + NSTAGE - 1);
#if SPC_ATTN_PF > 0
    prefetch_rows(i + NSTAGE - 1 + SPC_ATTN_PF);
#endif
    fetch_meta(i + NSTAGE - 1 + MAHEAD);
    cp_async_commit();
    trace(i, 0);
    const ChunkIt cc = it_cur;
    const bool grp_end = (i == n_chunks - 1) || (cc.rc == cpg - 1);
    it_cur.next(cpg, BG);
    if (grp_end && i + 1 < n_chunks) load_q(it_cur.lr, it_cur.bg, qn0, qn2);  // next group, early
    cp_async_wait<NSTAGE - 1>();  // rows of chunk i landed
    __syncwarp();
    trace(i, 1);
#ifdef SPC_ATTN_NOMATH  // debug builds only: time the load pipeline alone
    const int nv_w = 0;
#else
    const int nv_w = nv_ring[s_cur] - warp * WR;  // valid rows of this warp in the chunk
#endif
    const uint32_t st = wsb + (uint32_t)s_cur * SM::STAGE;
    if (nv_w > 0) {
      // ---- S^T = K Q^T for this warp's 16 rows: two accumulator chains
      float ce[4] = {0, 0, 0, 0}, co[4] = {0, 0, 0, 0};
#pragma unroll
      for (int kk = 0; kk < KS; kk += 2) {
        uint32_t a0, a1, a2, a3, e0, e1, e2, e3;
        ldsm_x4(st + b_off + kk * 32, a0, a1, a2, a3);
        ldsm_x4(st + b_off + (kk + 1) * 32, e0, e1, e2, e3);
        mma_bf16_4(ce, a0, a1, a2, a3, qa0[kk], qa2[kk]);
        mma_bf16_4(co, e0, e1, e2, e3, qa0[kk + 1], qa2[kk + 1]);
      }
      // values of this lane's columns: [row gid: slot 0, slot 1; row gid + 8: slot 0, slot 1]
      const float raw[4] = {ce[0] + co[0], ce[1] + co[1], ce[2] + co[2], ce[3] + co[3]};
      float sv[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int from = ALPHA == 1 ? (e & 2) : e;  // alpha = 1: both columns are head 0
        const float x = LOSEP ? raw[e] : __shfl_sync(0xffffffffu, raw[from], srcl);
        sv[e] = (e < 2 ? gid : gid + 8) < nv_w ? x * sl2 : -INFINITY;
      }
      float mx0 = fmaxf(sv[0], sv[2]), mx1 = fmaxf(sv[1], sv[3]);
#pragma unroll
      for (int sh = 4; sh < 32; sh <<= 1) {
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, sh));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, sh));
      }
      const float mn0 = fmaxf(m_run[0], mx0), mn1 = fmaxf(m_run[1], mx1);  // finite: row 0 valid
      if (__any_sync(0xffffffffu, mn0 > m_run[0] || mn1 > m_run[1])) {
        const float c0 = exp2f(m_run[0] - mn0), c1 = exp2f(m_run[1] - mn1);
        l_run[0] *= c0;
        l_run[1] *= c1;
#pragma unroll
        for (int a = 0; a < NACC; ++a)
#pragma unroll
          for (int d = 0; d < D / 16; ++d) {
            o[a][d][0] *= c0;
            o[a][d][1] *= c1;
            o[a][d][2] *= c0;
            o[a][d][3] *= c1;
          }
        m_run[0] = mn0;
        m_run[1] = mn1;
      }
      float ph[4], pl[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float pe = exp2f(sv[e] - m_run[e & 1]);
        l_run[e & 1] += pe;
        const float h = __bfloat162float(__float2bfloat16_rn(pe));
        const float lo = pe - h;
        const int md = cmode[e & 1];
        ph[e] = LOSEP ? h : (md == 0 ? h : (md == 1 ? lo : 0.f));
        pl[e] = lo;
      }
      // ---- O^T += V^T P: P's accumulator fragment -> B fragments by two transposes
      const uint32_t pb0 = movm_t(pack_bf16(ph[0], ph[1])), pb1 = movm_t(pack_bf16(ph[2], ph[3]));
      uint32_t pl0 = 0u, pl1 = 0u;
      if (LOSEP) {
        pl0 = movm_t(pack_bf16(pl[0], pl[1]));
        pl1 = movm_t(pack_bf16(pl[2], pl[3]));
      }
      const uint32_t vst = st + SM::KV_BYTES + a_off;
#pragma unroll
      for (int mt = 0; mt < D / 16; ++mt) {
        uint32_t a0, a1, a2, a3;
        ldsm_x4_t(vst + mt * 32, a0, a1, a2, a3);
        mma_bf16_4(o[0][mt], a0, a1, a2, a3, pb0, pb1);
        if (LOSEP) mma_bf16_4(o[NACC - 1][mt], a0, a1, a2, a3, pl0, pl1);
      }
    }
    trace(i, 2);
    // ---- flush at the end of this CTA's segment of the group: every warp writes its own
    // (m, l, o) partial with plain stores (no barrier, fence or ticket, so the load
    // streams of the other warps never stall); merge_groups_kernel combines them (O12)
    if (grp_end) {
      float lsum[2] = {l_run[0], l_run[1]};
#pragma unroll
      for (int sh = 4; sh < 32; sh <<= 1) {
        lsum[0] += __shfl_xor_sync(0xffffffffu, lsum[0], sh);
        lsum[1] += __shfl_xor_sync(0xffffffffu, lsum[1], sh);
      }
      const int b = cc.bg / G, g = cc.bg - (cc.bg / G) * G;
      const int first = (cc.grp * cpg) / cpc;
      const int part = (blockIdx.x - first) * NWARP + warp;
      const size_t head_base = ((size_t)cc.lr * B + b) * Hq + g * ALPHA;
      // O[head][d] = hi column + lo column (lane tig ^ 2 for alpha 4, tig ^ 1 for alpha 2,
      // the other slot for alpha 1, the second accumulator for alpha 8)
      constexpr int PX = ALPHA == 4 ? 2 : 1;
#pragma unroll
      for (int d = 0; d < D / 16; ++d)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          float v = o[0][d][r];
          if (LOSEP) v += o[NACC - 1][d][r];
          else if (ALPHA == 1) v = o[0][d][r & 2] + o[0][d][(r & 2) + 1];
          else v += __shfl_xor_sync(0xffffffffu, v, PX);
          const int sl = r & 1;
          if (cmode[sl] == 0 && (ALPHA != 1 || sl == 0))
            part_o[((head_base + hd[sl]) * segstride + part) * D + 16 * d + gid + (r >= 2 ? 8 : 0)] = v;
        }
      if (gid == 0) {
#pragma unroll
        for (int sl = 0; sl < 2; ++sl)
          if (cmode[sl] == 0 && (ALPHA != 1 || sl == 0)) {
            float* ml = part_ml + ((head_base + hd[sl]) * segstride + part) * 2;
            ml[0] = m_run[sl];
            ml[1] = lsum[sl];
          }
      }
      m_run[0] = m_run[1] = -INFINITY;
      l_run[0] = l_run[1] = 0.f;
#pragma unroll
      for (int a = 0; a < NACC; ++a)
#pragma unroll
        for (int d = 0; d < D / 16; ++d) o[a][d][0] = o[a][d][1] = o[a][d][2] = o[a][d][3] = 0.f;
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
  trace_warp(1);
  cp_async_wait<0>();
  // ---- after the CTA's last chunk (no loads left to stall): one ticket per group this
  // CTA covered; the CTA completing a group merges its partials with the LSE rule (O12)
  __shared__ int merge_flag;
  const int g_first = c_begin / cpg, g_last = (c_begin + n_chunks - 1) / cpg;
  __syncthreads();  // every warp's partial stores are issued
  if (tid == 0) __threadfence();  // ... and visible before the tickets
  for (int gq = g_first; gq <= g_last; ++gq) {
    const int nseg = (gq * cpg + cpg - 1) / cpc - (gq * cpg) / cpc + 1;
    if (tid == 0) {
      const unsigned t = atomicAdd(&cnt[gq], 1u);
      merge_flag = t == (unsigned)nseg - 1;
      if (t == (unsigned)nseg - 1) {
        cnt[gq] = 0u;  // the workspace stays reusable
        __threadfence();
      }
    }
    __syncthreads();
    if (merge_flag) {
      const int lr = gq / BG, bgq = gq - (gq / BG) * BG, b = bgq / G, g = bgq - (bgq / G) * G;
      merge_group_fast<D, ALPHA, AT2_THREADS>(
          part_o, part_ml, nseg * NWARP, segstride, ((size_t)lr * B + b) * Hq + g * ALPHA, out,
          lse, ((size_t)(layer_begin + lr) * B + b) * Hq + g * ALPHA, (float*)at_smem);
    }
    __syncthreads();  // merge_flag is rewritten for the next group
  }
}
