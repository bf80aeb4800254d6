// select.cu — spc_select: NORM + GROUP + top-k + INDEXED elastic diff in ONE launch.
//
// Definitions: O3 exp, O4 int64 fixed-point normaliser and
// reciprocal, O5 weights, O6 group max (P:321/P:328 head-level retrieval), O7
// top-k by the composite key (bits(v) << 32) | ~uint32(id) (R8, R20), O8 elastic
// diff against the previous selection.  Bit-identical to
// spc_score(NORM | GROUP) + spc_topk + spc_elastic_diff (tests/test_gpu_select.py).
//
// One thread-block cluster of SCL CTAs per (b, g) row; CTA `rank` owns the token
// segment [s0, s1) (a multiple of 4 tokens long).  The design minimises
// distributed-shared-memory bytes (DSMEM moves ~20 B/clk/SM, a cluster barrier
// costs ~400 clk):
//   1. NORM: each thread keeps exp(l - m) of its first 4 tokens x alpha heads in
//      registers; int64 partial sums are pushed to every CTA (alpha x SCL words).
//   2. GROUP: gs = max_j e_j * r_j -> shared memory segment + group_score.  The
//      row maximum of gs is exactly max_j r_j (the arg-max token of head j has
//      e = exp(0) = 1), so pass 0 of the radix select bins the values in a
//      256-bin window of 8 bins per binade below that maximum (clamped at both
//      ends) while gs is produced.
//   3. select: every pass pushes only the NONZERO bins of the local histogram
//      into every CTA (red.add over DSMEM), one cluster barrier, then every CTA
//      finds the threshold bin redundantly.  Later passes resolve 8 more key bits
//      of the threshold bucket.  Stop when the whole bucket is selected
//      (threshold = bucket's lower end) or it has <= CANDMAX elements: those are
//      pushed to every CTA and ranked by counting.
//   4. one pass over the segment classifies each token (selected / new / evicted
//      using a bitmap of the previous selection built in the prologue), one
//      packed block scan, one exchange of three counts per CTA, ordered writes.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace spc {
namespace {

#ifdef SPC_SEL_NREG  // register cap (experiment: room for attention CTAs beside a select CTA)
#define SPC_SEL_BOUNDS __maxnreg__(SPC_SEL_NREG)
#else
#define SPC_SEL_BOUNDS __launch_bounds__(ST, 1)
#endif
#ifndef SPC_SEL_SCL
#define SPC_SEL_SCL 8
#endif
constexpr int ST = 512;         // threads per CTA
constexpr int SEGCAP = 16896;   // tokens per CTA segment: rows up to 8 * SEGCAP = 135168
// SCL (template parameter) = CTAs per row = cluster size; 8.  (16-CTA non-portable
// clusters were measured: every phase here is latency-bound, 15.1 vs 14.9 us per row.)
constexpr int NB = 256;         // bins per histogram pass
constexpr int W0_SHIFT = 20;    // pass-0 bin = value bits >> 20: 8 bins per binade
constexpr int W0_BITS = 12;     // key bits (sign + exponent + 3 mantissa) fixed by a pass-0 bin
constexpr int CANDMAX = 128;    // exchange the threshold bucket at this size

// Debug trace (spc_debug_set_select_trace; compiled in with -DSPC_TRACE): thread 0
// of every CTA of rows 0..63 stamps %globaltimer at phase boundaries: [row][rank][slot].
__device__ unsigned long long* g_sel_trace = nullptr;
__device__ __forceinline__ void sel_mark(int slot) {
#ifdef SPC_TRACE
  if (g_sel_trace && blockIdx.y < 64 && threadIdx.x == 0 && slot < 16) {
    unsigned long long t;  // SM clock cycles (compare marks of one CTA only)
    asm volatile("mov.u64 %0, %clock64;" : "=l"(t));
    g_sel_trace[(blockIdx.y * gridDim.x + blockIdx.x) * 16 + slot] = t;
  }
#else
  (void)slot;
#endif
}

constexpr int MAXPASS = 8;  // radix passes: pass 0 fixes 12 key bits, each later one 8 more
constexpr int BAR_NORM = 0, BAR_X = 1, BAR_H = 2;  // mbarriers: NORM, candidates, pass p = BAR_H + p

template <int SCL>
struct SelSm {
  float seg[SEGCAP];                      // group scores of this CTA's segment
  uint32_t bm_prev[SEGCAP / 32];          // previous selection, segment-relative bitmap
  uint4 cand[SCL][CANDMAX];               // threshold bucket, pushed by every rank: key (lo, hi),
                                          // origin thread | previously selected << 16, 0
  unsigned long long flat[CANDMAX];       // the bucket of the whole row, flattened
  uint32_t flati[CANDMAX];                // ... origin thread | previously selected << 16 | rank << 17
  uint64_t bar[BAR_H + MAXPASS];          // exchange mbarriers
  unsigned hist[NB];                      // this CTA's histogram of the current pass
  unsigned rx[2][SCL][NB];                // pass p: every rank's histogram (ping-pong by p & 1)
  long long part[SCL][8];                 // NORM partial sums pushed by every rank
  long long wred[ST / 32][8];             // NORM warp partials
  long long ntot[8];                      // this CTA's NORM partials
  float rj[8];                            // 1 / l per head of the group
  unsigned long long stats[SCL];          // per rank: above | above&prev | bucket | bucket&prev
  unsigned long long my_stats;
  unsigned long long wsc[ST / 32];        // scan scratch
  unsigned wfind[NB / 32];
  unsigned short xsel[ST], xnew[ST];      // per thread: its bucket tokens selected (and new)
  int candn[SCL];                         // bucket elements pushed by every rank
  int lpre[3];                            // previous tokens < s0, < s1, < len
  int csel[SCL], cselp[SCL];              // selected bucket elements per rank (& previous)
  int find[3];                            // bin, above, count
  int ncand;
  unsigned long long T;
  unsigned long long total;
};

// Block-wide exclusive scan of one uint64 per thread (ST threads).
template <int SCL>
__device__ __forceinline__ unsigned long long scan_u64(SelSm<SCL>& s, unsigned long long v) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) s.wsc[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const unsigned long long x = lane < ST / 32 ? s.wsc[lane] : 0ull;
    unsigned long long xi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long t = __shfl_up_sync(0xffffffffu, xi, o);
      if (lane >= o) xi += t;
    }
    if (lane < ST / 32) s.wsc[lane] = xi - x;
    if (lane == 31) s.total = xi;
  }
  __syncthreads();
  return s.wsc[warp] + incl - v;
}

// Histogram exchange of pass `pass`: this CTA's whole histogram (1 KiB, zeros included)
// goes to slot `rank` of rx[pass & 1] in every CTA as 16-byte st.async (64 per destination:
// DSMEM issue, not bytes, is the limit -- 2048 per-bin remote atomics cost ~1 us), completing
// the destination's pass mbarrier, whose byte count (SCL KiB) every receiver expects itself.
// Ping-pong is safe: a rank sends pass p + 2 only after pass p + 1 completed, which needs
// every rank's pass p + 1 data, sent after that rank's find_bin of pass p.
template <int SCL>
__device__ __forceinline__ void exchange_hist(SelSm<SCL>& s, int rank, int pass) {
  const int t = threadIdx.x;
  const uint32_t bar = smem_u32(&s.bar[BAR_H + pass]);
  if (t == 0) tm_expect(bar, (uint32_t)(SCL * NB * 4));
  if (t < NB / 4) {
    const uint4 v = reinterpret_cast<const uint4*>(s.hist)[t];
    const uint32_t a = smem_u32(&s.rx[pass & 1][rank][4 * t]);
#pragma unroll
    for (int q = 0; q < SCL; ++q) dsm_st128(dsm_map(a, q), v, dsm_map(bar, q));
  }
  dsm_wait_cta(bar);
}

// After exchange_hist: bin of the r-th largest element counted from the top of the pass's
// cluster histogram -> s.find = {bin, count above it, count in it}.
template <int SCL>
__device__ __forceinline__ void find_bin(SelSm<SCL>& s, int pass, int r) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  unsigned c = 0, incl = 0;
  if (t < NB) {
    const int bin = NB - 1 - t;  // ascending t = descending bins
#pragma unroll
    for (int q = 0; q < SCL; ++q) c += s.rx[pass & 1][q][bin];
    incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned x = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += x;
    }
    if (lane == 31) s.wfind[warp] = incl;
  }
  __syncthreads();
  if (t < NB) {
    unsigned before = 0;
    for (int w = 0; w < warp; ++w) before += s.wfind[w];
    incl += before;
    if (incl >= (unsigned)r && incl - c < (unsigned)r) {
      s.find[0] = NB - 1 - t;
      s.find[1] = (int)(incl - c);
      s.find[2] = (int)c;
    }
  }
  __syncthreads();
}

template <int ALPHA, int NC, int SCL>
__global__ void SPC_SEL_BOUNDS select_kernel(
    const float* __restrict__ logits, const float* __restrict__ head_max,
    const int32_t* __restrict__ seq_len, int G, int Smax, int k, int force,
    int64_t* __restrict__ head_sumfix, float* __restrict__ group_score,
    int32_t* __restrict__ out_idx, int32_t* __restrict__ out_count,
    const int32_t* __restrict__ prev_idx, const int32_t* __restrict__ prev_count,
    int32_t* __restrict__ load_tok, int32_t* __restrict__ n_load, int32_t* __restrict__ evict_tok,
    int32_t* __restrict__ n_evict) {
  spc_pdl_entry();
  extern __shared__ __align__(16) uint8_t sel_raw[];
  SelSm<SCL>& s = *reinterpret_cast<SelSm<SCL>*>(sel_raw);
  const int rank = (int)cg::this_cluster().block_rank();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int bg = blockIdx.y, b = bg / G, g = bg - b * G;
  const int Hq = G * ALPHA;
  const int len = min(max(seq_len[b], 0), Smax);
  const int need = min(k, len);
  const int per = ((len + SCL - 1) / SCL + 3) & ~3;
  const int s0 = min(len, rank * per), s1 = min(len, s0 + per);
  const int nseg = s1 - s0;
  const int nch = (nseg + 3) >> 2;  // float4 chunks of the segment
  // this thread's tokens: the contiguous chunks [c0, c1) (ordered output needs only a scan)
  const int cpt = max(1, (nch + ST - 1) / ST);
  const int c0 = min(nch, tid * cpt), c1 = min(nch, c0 + cpt);
  const float* lg = logits + ((size_t)b * Hq + g * ALPHA) * Smax + s0;
  const int np = min(max(prev_count[bg], 0), k);
  const int32_t* pv = prev_idx + (size_t)bg * k;
  // the newest token counts as +inf when forced (R10): its group-score bits are replaced
  const int tforce = force ? len - 1 - s0 : -1;  // segment-relative, or out of range
  sel_mark(0);

  // ---- prologue: logits of the first NC chunks and the previous selection in flight
  float4 x0[NC][ALPHA];
#pragma unroll
  for (int u = 0; u < NC; ++u)
#pragma unroll
    for (int j = 0; j < ALPHA; ++j)
      x0[u][j] = c0 + u < c1 ? __ldg(reinterpret_cast<const float4*>(lg + (size_t)j * Smax) + c0 + u)
                             : make_float4(0.f, 0.f, 0.f, 0.f);
  constexpr int PVR = SPC_MAX_K / ST;
  int pvr[PVR];
#pragma unroll
  for (int i = 0; i < PVR; ++i) pvr[i] = tid + i * ST < np ? pv[tid + i * ST] : -1;
#ifdef SPC_DEBUG  // the previous selection: ascending, no duplicates, ids >= 0
  if (rank == 0)
    for (int i = tid; i < np; i += ST) {
      SPC_DCHECK(pv[i] >= 0, SPC_E_RANGE);
      SPC_DCHECK(i == 0 || pv[i - 1] < pv[i], SPC_E_STATE);
    }
#endif
  float m[ALPHA];
#pragma unroll
  for (int j = 0; j < ALPHA; ++j) m[j] = head_max[(size_t)b * Hq + g * ALPHA + j];
  const int nw = (nseg + 31) >> 5;
  for (int i = tid; i < nw; i += ST) s.bm_prev[i] = 0u;
  if (tid < NB) s.hist[tid] = 0u;
  s.xsel[tid] = 0;
  s.xnew[tid] = 0;
  if (tid < 3) s.lpre[tid] = 0;
  if (tid < SCL) s.csel[tid] = s.cselp[tid] = 0;
  if (tid == 0) {
    s.ncand = 0;
    s.my_stats = 0ull;
    for (int i = 0; i < BAR_H + MAXPASS; ++i)  // histogram passes: one local arrive (expect)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&s.bar[i])),
                   "r"(i < BAR_H ? SCL : 1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // every CTA of the cluster must be initialised (zeroed sums, mbarriers) before any remote
  // write into it: arrive now (release), wait right before the first send
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  sel_mark(10);

  // ---- NORM (O3, O4)
  long long acc[ALPHA];
  float e0[NC][ALPHA][4];
#pragma unroll
  for (int j = 0; j < ALPHA; ++j) acc[j] = 0;
#pragma unroll
  for (int u = 0; u < NC; ++u) {
    const int p0 = 4 * (c0 + u);  // segment-relative token of e0[u][.][0]
#pragma unroll
    for (int j = 0; j < ALPHA; ++j) {
      const float2 ea = spc_exp2_dev(__fsub_rn(x0[u][j].x, m[j]), __fsub_rn(x0[u][j].y, m[j]));
      const float2 eb = spc_exp2_dev(__fsub_rn(x0[u][j].z, m[j]), __fsub_rn(x0[u][j].w, m[j]));
      const float es[4] = {ea.x, ea.y, eb.x, eb.y};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float e = (c0 + u < c1 && p0 + c < nseg) ? es[c] : 0.0f;
        e0[u][j][c] = e;
        acc[j] += fixpoint40(e);
      }
    }
  }
  // segments longer than 4 * NC * ST tokens: stream the rest two chunks at a time (both
  // chunks' loads in flight before the first exp)
  for (int ch = c0 + NC; ch < c1; ch += 2) {
    float4 x[2][ALPHA];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int j = 0; j < ALPHA; ++j)
        x[u][j] = ch + u < c1 ? __ldg(reinterpret_cast<const float4*>(lg + (size_t)j * Smax) + ch + u)
                              : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int j = 0; j < ALPHA; ++j) {
        const float2 ea = spc_exp2_dev(__fsub_rn(x[u][j].x, m[j]), __fsub_rn(x[u][j].y, m[j]));
        const float2 eb = spc_exp2_dev(__fsub_rn(x[u][j].z, m[j]), __fsub_rn(x[u][j].w, m[j]));
        const float es[4] = {ea.x, ea.y, eb.x, eb.y};
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (ch + u < c1 && 4 * (ch + u) + c < nseg) acc[j] += fixpoint40(es[c]);
      }
  }
  sel_mark(11);
#pragma unroll
  for (int j = 0; j < ALPHA; ++j) {
    const long long v = warp_sum_ll(acc[j]);
    if (lane == 0) s.wred[warp][j] = v;
  }
  __syncthreads();
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) {  // this CTA's partial of head j to every rank q
    if (lane < ALPHA) {
      long long t = 0;
#pragma unroll
      for (int w = 0; w < ST / 32; ++w) t += s.wred[w][lane];
      s.ntot[lane] = t;
    }
    const uint32_t bar = smem_u32(&s.bar[BAR_NORM]);
    if (lane < SCL) dsm_expect(dsm_map(bar, lane), 8u * ALPHA);
    __syncwarp();
    const uint32_t a = smem_u32(&s.part[rank][0]);
    for (int i = lane; i < ALPHA * SCL; i += 32) {
      const int j = i % ALPHA, q = i / ALPHA;
      dsm_st64(dsm_map(a + 8u * j, q), (unsigned long long)s.ntot[j], dsm_map(bar, q));
    }
  }
  sel_mark(12);
  {  // meanwhile: bitmap of the previous tokens in this segment; prefix counts of the list
    int c_s0 = 0, c_s1 = 0, c_len = 0;
#pragma unroll
    for (int i = 0; i < PVR; ++i) {
      const int t = pvr[i];
      if (t >= 0) {
        if (t >= s0 && t < s1) atomicOr(&s.bm_prev[(t - s0) >> 5], 1u << ((t - s0) & 31));
        c_s0 += t < s0;
        c_s1 += t < s1;
        c_len += t < len;
      }
    }
    c_s0 = __reduce_add_sync(0xffffffffu, c_s0);
    c_s1 = __reduce_add_sync(0xffffffffu, c_s1);
    c_len = __reduce_add_sync(0xffffffffu, c_len);
    if (lane == 0) {
      if (c_s0) atomicAdd(&s.lpre[0], c_s0);
      if (c_s1) atomicAdd(&s.lpre[1], c_s1);
      if (c_len) atomicAdd(&s.lpre[2], c_len);
    }
  }
  dsm_wait_cta(smem_u32(&s.bar[BAR_NORM]));
  sel_mark(1);

  // ---- GROUP (O4..O6) + pass-0 histogram
  // F and r = 1 / l per head once per CTA (thread j), then broadcast through shared memory
  if (tid < ALPHA) {
    long long F = 0;
#pragma unroll
    for (int q = 0; q < SCL; ++q) F += s.part[q][tid];
    if (rank == 0) head_sumfix[(size_t)b * Hq + g * ALPHA + tid] = F;
    s.rj[tid] = __fdiv_rn(1.0f, __fmul_rn(__ll2float_rn(F), 9.094947017729282379150390625e-13f));
  }
  __syncthreads();
  float r[ALPHA];
  float gmax = 0.0f;
#pragma unroll
  for (int j = 0; j < ALPHA; ++j) {
    r[j] = s.rj[j];
    gmax = fmaxf(gmax, r[j]);
  }
  const int top = (int)(__float_as_uint(gmax) >> W0_SHIFT);
  const int base0 = top - (NB - 1);
  float* gso = group_score + (size_t)bg * Smax + s0;
  const bool cut = need < len;
  auto bin0_of = [&](float v, int p) {  // pass-0 bin of segment token p (force: +inf)
    const uint32_t vb = p == tforce ? 0x7F800000u : __float_as_uint(v);
    return min(max((int)(vb >> W0_SHIFT) - base0, 0), NB - 1);
  };
#pragma unroll
  for (int u = 0; u < NC; ++u) {
    const int ch = c0 + u;
    if (ch < c1) {
      float gs[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float v = __fmul_rn(e0[u][0][c], r[0]);
#pragma unroll
        for (int j = 1; j < ALPHA; ++j) v = fmaxf(v, __fmul_rn(e0[u][j][c], r[j]));
        gs[c] = v;
        const int p = 4 * ch + c;
        if (cut && p < nseg) atomicAdd(&s.hist[bin0_of(v, p)], 1u);
      }
      const float4 o = make_float4(gs[0], gs[1], gs[2], gs[3]);
      reinterpret_cast<float4*>(s.seg)[ch] = o;
      reinterpret_cast<float4*>(gso)[ch] = o;  // tokens past len in the chunk get 0
    }
  }
  for (int ch0 = c0 + NC; ch0 < c1; ch0 += 2) {
    float4 x[2][ALPHA];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int j = 0; j < ALPHA; ++j)
        x[u][j] = ch0 + u < c1
                      ? __ldg(reinterpret_cast<const float4*>(lg + (size_t)j * Smax) + ch0 + u)
                      : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int ch = ch0 + u;
      if (ch >= c1) break;
      float e[ALPHA][4];
#pragma unroll
      for (int j = 0; j < ALPHA; ++j) {
        const float2 ea = spc_exp2_dev(__fsub_rn(x[u][j].x, m[j]), __fsub_rn(x[u][j].y, m[j]));
        const float2 eb = spc_exp2_dev(__fsub_rn(x[u][j].z, m[j]), __fsub_rn(x[u][j].w, m[j]));
        const float es[4] = {ea.x, ea.y, eb.x, eb.y};
#pragma unroll
        for (int c = 0; c < 4; ++c) e[j][c] = 4 * ch + c < nseg ? es[c] : 0.0f;
      }
      float gs[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float v = __fmul_rn(e[0][c], r[0]);
#pragma unroll
        for (int j = 1; j < ALPHA; ++j) v = fmaxf(v, __fmul_rn(e[j][c], r[j]));
        gs[c] = v;
        const int p = 4 * ch + c;
        if (cut && p < nseg) atomicAdd(&s.hist[bin0_of(v, p)], 1u);
      }
      const float4 o = make_float4(gs[0], gs[1], gs[2], gs[3]);
      reinterpret_cast<float4*>(s.seg)[ch] = o;
      reinterpret_cast<float4*>(gso)[ch] = o;
    }
  }
  {  // zero-fill group_score [roundup4(len), Smax)
    float4* gz = reinterpret_cast<float4*>(group_score + (size_t)bg * Smax);
    for (int p4 = ((len + 3) >> 2) + rank * ST + tid; p4 < (Smax >> 2); p4 += SCL * ST)
      gz[p4] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __syncthreads();
  sel_mark(2);

  // ---- top-k (O7): selected = {key >= T}, key = composite(group-score bits, id).  Per thread:
  // nsel / nnew = its selected / newly selected tokens, nwas = its previously selected ones
  unsigned long long T = 0ull;
  int b_sel = 0, b_selp = 0, a_sel = 0, a_selp = 0;
  int nsel = 0, nnew = 0, nwas = 0;
  if (cut) {
    sel_mark(13);
    exchange_hist(s, rank, 0);
    sel_mark(14);
    find_bin(s, 0, need);
    const int bin0 = s.find[0];
    int rr = need - s.find[1], cm = s.find[2];
    // the threshold bucket = keys in [klo, khi]; everything above khi is selected
    unsigned long long P = 0ull, xlo = 0ull, xmax = ~0ull;
    int bits = 1;  // key bit 63 (sign of the value) is always 0
    if (bin0 == 0) {
      xmax = ((unsigned long long)(uint32_t)(base0 + 1) << 52) - 1ull;
    } else if (bin0 == NB - 1) {
      xlo = (unsigned long long)(uint32_t)top << 52;
    } else {
      P = (unsigned long long)(uint32_t)(base0 + bin0) << 52;
      bits = W0_BITS;
    }
    sel_mark(3);
    for (int pass = 1; cm != rr && cm > CANDMAX; ++pass) {  // rare: resolve 8 more key bits
      const int db = min(8, 64 - bits), sh = 64 - bits - db;
      const unsigned mask = (1u << db) - 1u;
      const unsigned long long plo = P > xlo ? P : xlo;
      const unsigned long long phi_ = P | (bits >= 64 ? 0ull : ~0ull >> bits);
      const unsigned long long phi = phi_ < xmax ? phi_ : xmax;
      if (tid < NB) s.hist[tid] = 0u;
      __syncthreads();
      for (int ch = c0; ch < c1; ++ch) {
        const float4 v = reinterpret_cast<const float4*>(s.seg)[ch];
        const float vs[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int p = 4 * ch + c;
          if (p < nseg) {
            const uint32_t vb = p == tforce ? 0x7F800000u : __float_as_uint(vs[c]);
            const unsigned long long x = composite(vb, s0 + p);
            if (x >= plo && x <= phi) atomicAdd(&s.hist[(unsigned)(x >> sh) & mask], 1u);
          }
        }
      }
      __syncthreads();
      exchange_hist(s, rank, pass);
      find_bin(s, pass, rr);
      rr -= s.find[1];
      cm = s.find[2];
      P |= (unsigned long long)s.find[0] << sh;
      bits += db;
    }
    sel_mark(4);
    const unsigned long long phi_ = P | (bits >= 64 ? 0ull : ~0ull >> bits);
    const unsigned long long klo = P > xlo ? P : xlo, khi = phi_ < xmax ? phi_ : xmax;
    // classification: tokens above the bucket and in it (each also & previous); the bucket
    // itself is pushed to every CTA unless it is selected whole (cm == rr)
    const bool xchg = cm != rr;
    int nab = 0, nabp = 0, ninb = 0, ninbp = 0;
    for (int ch = c0; ch < c1; ++ch) {
      const float4 v = reinterpret_cast<const float4*>(s.seg)[ch];
      const float vs[4] = {v.x, v.y, v.z, v.w};
      const uint32_t pw = s.bm_prev[ch >> 3] >> ((ch & 7) * 4);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int p = 4 * ch + c;
        if (p < nseg) {
          const uint32_t vb = p == tforce ? 0x7F800000u : __float_as_uint(vs[c]);
          const unsigned long long x = composite(vb, s0 + p);
          const int was = (pw >> c) & 1u;
          nwas += was;
          if (x > khi) {
            ++nab;
            nabp += was;
          } else if (x >= klo) {
            ++ninb;
            ninbp += was;
            if (xchg) {  // the bucket element to every rank (12 bytes on its BAR_X)
              const int slot = atomicAdd(&s.ncand, 1);
              const uint32_t ci = (uint32_t)tid | ((uint32_t)was << 16);
              const uint32_t ak = smem_u32(&s.cand[rank][slot]), bx = smem_u32(&s.bar[BAR_X]);
              const uint4 rec = make_uint4((uint32_t)x, (uint32_t)(x >> 32), ci, 0u);
#pragma unroll
              for (int q = 0; q < SCL; ++q) dsm_st128(dsm_map(ak, q), rec, dsm_map(bx, q));
            }
          }
        }
      }
    }
    sel_mark(6);
    {
      unsigned long long st4 = (unsigned long long)nab + ((unsigned long long)nabp << 16) +
                               ((unsigned long long)ninb << 32) + ((unsigned long long)ninbp << 48);
#pragma unroll
      for (int o = 16; o; o >>= 1) st4 += __shfl_xor_sync(0xffffffffu, st4, o);
      if (lane == 0 && st4) atomicAdd(&s.my_stats, st4);
    }
    __syncthreads();
    if (tid < SCL) {  // this CTA's counts and bucket size to rank tid (its bucket sent above)
      const int nc = xchg ? s.ncand : 0;
      const uint32_t bx = dsm_map(smem_u32(&s.bar[BAR_X]), tid);
      dsm_expect(bx, 12u + 16u * (uint32_t)nc);
      dsm_st64(dsm_map(smem_u32(&s.stats[rank]), tid), s.my_stats, bx);
      dsm_st32(dsm_map(smem_u32(&s.candn[rank]), tid), (uint32_t)nc, bx);
    }
    sel_mark(8);
    dsm_wait_cta(smem_u32(&s.bar[BAR_X]));
    sel_mark(9);
    if (!xchg) {
      T = klo;  // the whole bucket is selected: T = its lower end
      nsel = nab + ninb;
      nnew = (nab - nabp) + (ninb - ninbp);
#pragma unroll
      for (int q = 0; q < SCL; ++q) {
        const unsigned long long sq = s.stats[q];
        const int sl = (int)(sq & 0xFFFF) + (int)((sq >> 32) & 0xFFFF);
        const int sp = (int)((sq >> 16) & 0xFFFF) + (int)(sq >> 48);
        a_sel += sl;
        a_selp += sp;
        b_sel += q < rank ? sl : 0;
        b_selp += q < rank ? sp : 0;
      }
    } else {
      // flatten the row's bucket, then rank it: warp w takes candidates w, w + 16, ..., its
      // lanes hold the keys lane + 32 i in registers (one compare each + a warp sum)
      int nall = 0;
#pragma unroll
      for (int q = 0; q < SCL; ++q) nall += s.candn[q];
      if (tid < nall) {
        int i = tid, q = 0;
        while (i >= s.candn[q]) i -= s.candn[q++];
        const uint4 rec = s.cand[q][i];
        s.flat[tid] = (unsigned long long)rec.x | ((unsigned long long)rec.y << 32);
        s.flati[tid] = rec.z | ((uint32_t)q << 17);
      }
      __syncthreads();
      {
        unsigned long long kk[CANDMAX / 32];
#pragma unroll
        for (int i = 0; i < CANDMAX / 32; ++i)  // keys are > 0 (~id has bit 31 set): 0 pads
          kk[i] = lane + 32 * i < nall ? s.flat[lane + 32 * i] : 0ull;
        for (int c = warp; c < nall; c += ST / 32) {
          const unsigned long long x = s.flat[c];
          int n = 0;
#pragma unroll
          for (int i = 0; i < CANDMAX / 32; ++i) n += kk[i] > x;
          n = __reduce_add_sync(0xffffffffu, n);
          if (lane == 0 && n == rr - 1) s.T = x;
        }
      }
      __syncthreads();
      T = s.T;
      if (tid < nall && s.flat[tid] >= T) {
        const uint32_t info = s.flati[tid];
        const int was = (int)((info >> 16) & 1u), mine_q = (int)(info >> 17);
        atomicAdd(&s.csel[mine_q], 1);
        if (was) atomicAdd(&s.cselp[mine_q], 1);
        if (mine_q == rank) {  // credit the owning thread of this CTA
          const int ot = (int)(info & 0xFFFFu);
          atomicAdd(reinterpret_cast<unsigned*>(&s.xsel[ot & ~1]), 1u << (16 * (ot & 1)));
          if (!was) atomicAdd(reinterpret_cast<unsigned*>(&s.xnew[ot & ~1]), 1u << (16 * (ot & 1)));
        }
      }
      __syncthreads();
      nsel = nab + s.xsel[tid];
      nnew = (nab - nabp) + s.xnew[tid];
#pragma unroll
      for (int q = 0; q < SCL; ++q) {
        const unsigned long long sq = s.stats[q];
        const int sl = (int)(sq & 0xFFFF) + s.csel[q];
        const int sp = (int)((sq >> 16) & 0xFFFF) + s.cselp[q];
        a_sel += sl;
        a_selp += sp;
        b_sel += q < rank ? sl : 0;
        b_selp += q < rank ? sp : 0;
      }
    }
  } else {
    // no cut: every token is selected
    b_sel = s0;
    a_sel = len;
    b_selp = s.lpre[0];
    a_selp = s.lpre[2];
    for (int ch = c0; ch < c1; ++ch) {
      const uint32_t pw = s.bm_prev[ch >> 3] >> ((ch & 7) * 4);
      const int nv = min(4, nseg - 4 * ch);
      nwas += __popc(pw & ((1u << nv) - 1u));
      nsel += nv;
    }
    nnew = nsel - nwas;
  }
  sel_mark(5);

  // ---- ordered writes: selection (O7), new tokens and evictions (O8).  Evicted = previous
  // tokens not selected; the previous tokens >= len (never selected) are listed last.
  const int bs = b_sel, bn = b_sel - b_selp, be = s.lpre[0] - b_selp;
  const int as = a_sel, an = a_sel - a_selp, ae = np - a_selp;
  const int ntail = np - s.lpre[2];
  const int nev = nwas - (nsel - nnew);  // previously selected, not selected now
  const unsigned long long cnt = (unsigned long long)nsel + ((unsigned long long)nnew << 21) +
                                 ((unsigned long long)nev << 42);
  const unsigned long long pos = scan_u64(s, cnt);
  sel_mark(15);
  int32_t* oi = out_idx + (size_t)bg * k;
  int32_t* lt = load_tok + (size_t)bg * k;
  int32_t* et = evict_tok ? evict_tok + (size_t)bg * k : nullptr;
  int ps = bs + (int)(pos & 0x1FFFFF), pn = bn + (int)((pos >> 21) & 0x1FFFFF),
      pe = be + (int)(pos >> 42);
  const uint32_t Thi = (uint32_t)(T >> 32), Tlo = (uint32_t)T;
  for (int ch = c0; ch < c1; ++ch) {
    const float4 v = reinterpret_cast<const float4*>(s.seg)[ch];
    const float vs[4] = {v.x, v.y, v.z, v.w};
    const uint32_t pw = s.bm_prev[ch >> 3] >> ((ch & 7) * 4);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int p = 4 * ch + c;
      if (p < nseg) {
        const int t = s0 + p;
        const uint32_t vb = p == tforce ? 0x7F800000u : __float_as_uint(vs[c]);
        // key >= T on (value bits, ~id) without forming the 64-bit key
        const bool sel = !cut || vb > Thi || (vb == Thi && ~(uint32_t)t >= Tlo);
        const bool was = (pw >> c) & 1u;
        if (sel) oi[ps++] = t;
        if (sel && !was) lt[pn++] = t;
        if (!sel && was && et) et[pe++] = t;
      }
    }
  }
  if (rank == SCL - 1) {
    if (et)
      for (int i = tid; i < ntail; i += ST) et[ae - ntail + i] = pv[np - ntail + i];
    for (int i = as + tid; i < k; i += ST) oi[i] = -1;
    for (int i = an + tid; i < k; i += ST) lt[i] = -1;
    if (et)
      for (int i = ae + tid; i < k; i += ST) et[i] = -1;
  }
  if (rank == 0 && tid == 0) {
    out_count[bg] = as;
    n_load[bg] = an;
    if (n_evict) n_evict[bg] = ae;
  }
  sel_mark(7);
}
}  // namespace
}  // namespace spc

using namespace spc;

// debug only (not in include/spc.h): point the -DSPC_TRACE stamps at a device buffer of
// 64 rows x 16 CTAs x 16 uint64, or NULL to stop
extern "C" int spc_debug_set_select_trace(unsigned long long* buf) {
  return cudaMemcpyToSymbol(spc::g_sel_trace, &buf, sizeof(buf)) == cudaSuccess ? SPC_OK
                                                                                 : SPC_E_CUDA;
}

namespace spc {
namespace {
template <int AA, int SCL>
int launch_select(const float* logits, const float* head_max, const int32_t* seq_len, int B, int G,
                  int Smax, int k, int force_last, int64_t* head_sumfix, float* group_score,
                  int32_t* out_idx, int32_t* out_count, const int32_t* prev_idx,
                  const int32_t* prev_count, int32_t* load_tok, int32_t* n_load,
                  int32_t* evict_tok, int32_t* n_evict, cudaStream_t st) {
  auto kern = select_kernel<AA, (AA > 4 ? 1 : 2), SCL>;
  SPC_TRY(smem_attr((const void*)kern, (int)sizeof(SelSm<SCL>), SCL > 8));
  return launched(launch_kc(kern, dim3(SCL, B * G), dim3(ST), sizeof(SelSm<SCL>), st, SCL,
                            logits, head_max, seq_len, G, Smax, k, force_last, head_sumfix,
                            group_score, out_idx, out_count, prev_idx, prev_count, load_tok,
                            n_load, evict_tok, n_evict));
}

}  // namespace
}  // namespace spc

extern "C" int spc_select(const float* logits, const float* head_max, const int32_t* seq_len, int B,
                          int Hq, int G, int Smax, int k, int force_last, int64_t* head_sumfix,
                          float* group_score, int32_t* out_idx, int32_t* out_count,
                          const int32_t* prev_idx, const int32_t* prev_count, int32_t* load_tok,
                          int32_t* n_load, int32_t* evict_tok, int32_t* n_evict,
                          spc_stream_t stream) {
  if (!logits || !head_max || !seq_len || !head_sumfix || !group_score || !out_idx ||
      !out_count || !prev_idx || !prev_count || !load_tok || !n_load)
    return SPC_E_NULL;
  if (B <= 0 || G <= 0 || Hq <= 0 || Hq % G || Smax <= 0) return SPC_E_SHAPE;
  if (k < 1 || k > SPC_MAX_K) return SPC_E_BUDGET;
  if (Smax > 8 * SEGCAP || Smax % 4) return SPC_E_UNSUPPORTED;
  const int alpha = Hq / G;
  cudaStream_t st = as_stream(stream);
#define SEL(AA)                                                                                 \
  if (alpha == AA)                                                                              \
    return launch_select<AA, SPC_SEL_SCL>(logits, head_max, seq_len, B, G, Smax, k, force_last,           \
                                head_sumfix, group_score, out_idx, out_count, prev_idx,          \
                                prev_count, load_tok, n_load, evict_tok, n_evict, st);
  SEL(1) SEL(2) SEL(4) SEL(8)
#undef SEL
  return SPC_E_UNSUPPORTED;
}
