// score.cu — spc_score: retrieval-head scoring O1..O6.
//
// Paper: Eq.1 softmax(QK^T/sqrt(d)) of the lightweight retrieval
// head over its full key cache, then the GQA group maximum of
// the weights (MQA P:331).
//
// Three kernels (phases), each HBM- or L2-streaming:
//   LOGITS  streams the bf16 key cache once (the dominant bytes): persistent CTAs,
//           per-warp cp.async rings into padded shared rows; one lane owns 4 key
//           rows and runs alpha sequential fp32 FMA chains per row (bit-exact O1),
//           two rows at a time with the packed sm_100 FFMA2 (fma.rn.f32x2: per-lane
//           IEEE fma, order kept).  The key row feeds all alpha query heads of its
//           group (no repeat_kv).  See logits.cuh.
//   NORM    exp + exact int64 fixed-point sums (O3, O4): grid-wide float4 streaming,
//           per-CTA partials added with 64-bit atomics (exact, order-free).
//   GROUP   weights and group max (O5, O6).
// Partial maxima / sums go to the workspace; the last CTA of each group or head
// (ticket) publishes them (order-free: max and integer add), so results are
// deterministic and the workspace is left zero-filled.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace spc {
namespace {




constexpr int NORM_THREADS = 256;
constexpr int NORM_PER = 8;      // elements per thread
constexpr int NORM_TILE = NORM_THREADS * NORM_PER;
constexpr int GRP_THREADS = 256;
constexpr int GRP_PER = 4;
constexpr int GRP_TILE = GRP_THREADS * GRP_PER;

#include "logits.cuh"

// ---------------------------------------------------------------- NORM (O3, O4)
// Grid (blocks per head, B*Hq).  Each thread streams float4 chunks of its head's row
// (two chunks in flight), exp as f32x2 pairs; the CTA's int64 partial is added to the
// head's workspace accumulator with a 64-bit atomic (integer addition: exact, order-
// free); the last CTA of the head (ticket) publishes head_sumfix and re-zeroes it.
constexpr int NM_T = 256;
template <bool VEC>
__global__ void __launch_bounds__(NM_T) norm_kernel(
    const float* __restrict__ logits, const float* __restrict__ head_max,
    const int32_t* __restrict__ seq_len, int Hq, int Smax, unsigned long long* __restrict__ acc_ws,
    unsigned* __restrict__ tickets, int64_t* __restrict__ head_sumfix) {
  spc_pdl_entry();
  __shared__ long long red[NM_T / 32];
  __shared__ int flag;
  const int bh = blockIdx.y, b = bh / Hq;
  const int S = min(max(seq_len[b], 0), Smax);
  const float m = head_max[bh];
  const float* row = logits + (size_t)bh * Smax;
  long long acc = 0;
  if (VEC) {
    const int nch = S >> 2;  // whole float4 chunks; the tail is done below
    const float4* r4 = reinterpret_cast<const float4*>(row);
    const int stride = gridDim.x * NM_T;
    for (int c = blockIdx.x * NM_T + threadIdx.x; c < nch; c += 4 * stride) {  // 4 in flight
      float4 x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        x[u] = c + u * stride < nch ? __ldcg(r4 + c + u * stride)
                                    : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float2 a0 = spc_exp2_dev(__fsub_rn(x[u].x, m), __fsub_rn(x[u].y, m));
        const float2 a1 = spc_exp2_dev(__fsub_rn(x[u].z, m), __fsub_rn(x[u].w, m));
        acc += fixpoint40(a0.x) + fixpoint40(a0.y) + fixpoint40(a1.x) + fixpoint40(a1.y);
      }
    }
    if (blockIdx.x == 0)
      for (int t = (nch << 2) + threadIdx.x; t < S; t += NM_T)
        acc += fixpoint40(spc_exp_dev(__fsub_rn(__ldcg(row + t), m)));
  } else {
    for (int t = blockIdx.x * NM_T + threadIdx.x; t < S; t += gridDim.x * NM_T)
      acc += fixpoint40(spc_exp_dev(__fsub_rn(__ldcg(row + t), m)));
  }
  acc = warp_sum_ll(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long sum = 0;
    for (int w = 0; w < NM_T / 32; ++w) sum += red[w];
    if (sum) atomicAdd(acc_ws + bh, (unsigned long long)sum);
  }
  if (last_block_ticket(&tickets[bh], gridDim.x, &flag) && threadIdx.x == 0) {
    head_sumfix[bh] = (int64_t)__ldcg(acc_ws + bh);
    acc_ws[bh] = 0ull;
  }
}

// ------------------------------------------------------------- GROUP (O4..O6)
template <int ALPHA>
__global__ void __launch_bounds__(GRP_THREADS) group_kernel(
    const float* __restrict__ logits, const float* __restrict__ head_max,
    const int64_t* __restrict__ head_sumfix, const int32_t* __restrict__ seq_len, int G, int Smax,
    float* __restrict__ group_score) {
  spc_pdl_entry();
  const int bg = blockIdx.y, b = bg / G, g = bg % G;
  const int Hq = G * ALPHA;
  const int S = seq_len[b];
  float m[ALPHA], r[ALPHA];
#pragma unroll
  for (int j = 0; j < ALPHA; ++j) {
    const int h = b * Hq + g * ALPHA + j;
    m[j] = head_max[h];
    const float l = __fmul_rn(__ll2float_rn(head_sumfix[h]), 9.094947017729282379150390625e-13f);
    r[j] = __fdiv_rn(1.0f, l);
  }
  const float* lg = logits + ((size_t)b * Hq + g * ALPHA) * Smax;
  float* out = group_score + (size_t)bg * Smax;
  const int t0 = blockIdx.x * GRP_TILE + threadIdx.x;
#pragma unroll
  for (int i = 0; i < GRP_PER; i += 2) {  // tokens t and t + GRP_THREADS as an f32x2 pair
    const int ta = t0 + i * GRP_THREADS, tb = ta + GRP_THREADS;
    if (ta >= Smax) break;
    float ga = 0.0f, gb = 0.0f;
#pragma unroll
    for (int j = 0; j < ALPHA; ++j) {
      const float xa = ta < S ? __ldcg(lg + (size_t)j * Smax + ta) : m[j];
      const float xb = tb < S ? __ldcg(lg + (size_t)j * Smax + tb) : m[j];
      const float2 e = spc_exp2_dev(__fsub_rn(xa, m[j]), __fsub_rn(xb, m[j]));
      const float pa = __fmul_rn(e.x, r[j]), pb = __fmul_rn(e.y, r[j]);
      ga = j ? fmaxf(ga, pa) : pa;
      gb = j ? fmaxf(gb, pb) : pb;
    }
    out[ta] = ta < S ? ga : 0.0f;
    if (tb < Smax) out[tb] = tb < S ? gb : 0.0f;
  }
}

// ---------------------------------------------------------- BATCH (O6b, NEXT-3)
// Batch-level retrieval (Fig. 5(a); SPEC retrieve_batch_level S:125-132): one
// token set per request from the SUM of every query head's weight, bs[t] = fl(...fl(p_0(t)
// + p_1(t)) ... + p_{Hq-1}(t)) (O5's weights, ascending head order, RN adds), written to
// all G rows of group_score so the per-group top-k / diff / attention select the same set.
constexpr int BT_THREADS = 256;
constexpr int BT_MAXH = 128;
__global__ void __launch_bounds__(BT_THREADS) batch_kernel(
    const float* __restrict__ logits, const float* __restrict__ head_max,
    const int64_t* __restrict__ head_sumfix, const int32_t* __restrict__ seq_len, int Hq, int G,
    int Smax, float* __restrict__ group_score) {
  spc_pdl_entry();
  __shared__ float sm_m[BT_MAXH], sm_r[BT_MAXH];
  const int b = blockIdx.y;
  for (int h = threadIdx.x; h < Hq; h += BT_THREADS) {
    sm_m[h] = head_max[(size_t)b * Hq + h];
    const float l = __fmul_rn(__ll2float_rn(head_sumfix[(size_t)b * Hq + h]),
                              9.094947017729282379150390625e-13f);
    sm_r[h] = __fdiv_rn(1.0f, l);
  }
  __syncthreads();
  const int S = seq_len[b];
  const int ta = blockIdx.x * (2 * BT_THREADS) + threadIdx.x, tb = ta + BT_THREADS;
  if (ta >= Smax) return;
  const float* lg = logits + (size_t)b * Hq * Smax;
  float sa = 0.0f, sb = 0.0f;
  for (int h = 0; h < Hq; ++h) {
    const float m = sm_m[h];
    const float xa = ta < S ? __ldcg(lg + (size_t)h * Smax + ta) : m;
    const float xb = tb < S ? __ldcg(lg + (size_t)h * Smax + tb) : m;
    const float2 e = spc_exp2_dev(__fsub_rn(xa, m), __fsub_rn(xb, m));
    const float pa = __fmul_rn(e.x, sm_r[h]), pb = __fmul_rn(e.y, sm_r[h]);
    sa = h ? __fadd_rn(sa, pa) : pa;
    sb = h ? __fadd_rn(sb, pb) : pb;
  }
  for (int g = 0; g < G; ++g) {
    float* out = group_score + ((size_t)b * G + g) * Smax;
    out[ta] = ta < S ? sa : 0.0f;
    if (tb < Smax) out[tb] = tb < S ? sb : 0.0f;
  }
}

template <int D, int ALPHA>
int launch_logits(const uint16_t* kr, const uint16_t* q, const int32_t* seq_len, int B, int G,
                  int Smax, float scale, float* logits, float* tile_max, unsigned* ctr,
                  float* head_max, cudaStream_t st) {
  const int tpr = (Smax + LG_TR - 1) / LG_TR;
  const int ntiles = B * G * tpr;
  const int nh = B * G * ALPHA;
  int tm_per_head = tpr;  // tile_max entries per head (the TMA kernel: one per consumer split)
  if ((long long)B * G * Smax < (1ll << 31)) {  // TMA-fed kernel (int32 row coordinates)
    tm_per_head = tpr * LT_CPR;
    SPC_TRY(smem_attr((const void*)logits_tma_kernel<D, ALPHA>, LtSmem<D, ALPHA>::BYTES));
    CUtensorMap map;
    SPC_TRY(make_tmap_tile_bf16(&map, kr, (uint64_t)B * G * Smax, D, LG_TR));
    // short streams (config B: 14 tiles per SM) claim 1 tile at a time (0.5 us faster than 2)
    // and load with an L2 evict_first policy (the step's small hot set -- code, logits,
    // selections -- stays in L2: step 83.3 -> 79.8 us together with the attention's); long
    // ones (config E: 443 tiles per SM) claim 2 and stream with the normal policy (326 us
    // vs 359 with 1 tile per claim, 364 with evict_first)
    const bool long_stream = ntiles >= 64 * num_sms();
    const int lt_batch = SPC_LT_BATCH > 0 ? SPC_LT_BATCH : (long_stream ? 2 : 1);
    const int ncta = max(1, min(num_sms(), (ntiles + lt_batch - 1) / lt_batch));
    SPC_TRY(launched(launch_k(logits_tma_kernel<D, ALPHA>, dim3(ncta), dim3(32 * (LT_NC + 1)),
                              LtSmem<D, ALPHA>::BYTES, st, map, q, seq_len, G, Smax, scale, tpr,
                              ntiles, logits, tile_max, ctr, lt_batch, long_stream ? 0 : 1)));
  } else {
    const size_t smem = LgSmem<D, ALPHA>::BYTES;
    SPC_TRY(smem_attr((const void*)logits_kernel<D, ALPHA>, (int)smem));
    const int nw = (ntiles + 1) / 2;  // >= 2 tiles per warp
    const int ncta = max(1, min(num_sms(), (nw + lg_warps<ALPHA>() - 1) / lg_warps<ALPHA>()));
    SPC_TRY(launched(launch_k(logits_kernel<D, ALPHA>, dim3(ncta), dim3(32 * lg_warps<ALPHA>()),
                             smem, st, kr, q, seq_len, G, Smax, scale, tpr, ntiles, logits,
                             tile_max, ctr)));
  }
  return launched(launch_k(lg_finalize_kernel, dim3(nh), dim3(256), 0, st,
                           (const float*)tile_max, tm_per_head, nh, head_max, ctr));
}

// GROUP with float4 accesses (Smax % 4 == 0): a thread takes 4 consecutive tokens, one
// float4 load per head (alpha in flight), the same O4..O6 arithmetic per element, one
// float4 store.
template <int ALPHA>
__global__ void __launch_bounds__(GRP_THREADS) group4_kernel(
    const float* __restrict__ logits, const float* __restrict__ head_max,
    const int64_t* __restrict__ head_sumfix, const int32_t* __restrict__ seq_len, int G, int Smax,
    float* __restrict__ group_score) {
  spc_pdl_entry();
  const int bg = blockIdx.y, b = bg / G, g = bg % G;
  const int Hq = G * ALPHA;
  const int S = seq_len[b];
  float m[ALPHA], r[ALPHA];
#pragma unroll
  for (int j = 0; j < ALPHA; ++j) {
    const int h = b * Hq + g * ALPHA + j;
    m[j] = head_max[h];
    const float l = __fmul_rn(__ll2float_rn(head_sumfix[h]), 9.094947017729282379150390625e-13f);
    r[j] = __fdiv_rn(1.0f, l);
  }
  const float4* lg = reinterpret_cast<const float4*>(logits + ((size_t)b * Hq + g * ALPHA) * Smax);
  float4* out = reinterpret_cast<float4*>(group_score + (size_t)bg * Smax);
  const int c = blockIdx.x * GRP_THREADS + threadIdx.x;  // float4 chunk
  if (c * 4 >= Smax) return;
  float4 x[ALPHA];
#pragma unroll
  for (int j = 0; j < ALPHA; ++j) x[j] = __ldcg(lg + (size_t)j * (Smax / 4) + c);
  float gsv[4];
#pragma unroll
  for (int j = 0; j < ALPHA; ++j) {
    const float2 e0 = spc_exp2_dev(__fsub_rn(x[j].x, m[j]), __fsub_rn(x[j].y, m[j]));
    const float2 e1 = spc_exp2_dev(__fsub_rn(x[j].z, m[j]), __fsub_rn(x[j].w, m[j]));
    const float p[4] = {__fmul_rn(e0.x, r[j]), __fmul_rn(e0.y, r[j]), __fmul_rn(e1.x, r[j]),
                        __fmul_rn(e1.y, r[j])};
#pragma unroll
    for (int u = 0; u < 4; ++u) gsv[u] = j ? fmaxf(gsv[u], p[u]) : p[u];
  }
  const int t = c * 4;
  out[c] = make_float4(t < S ? gsv[0] : 0.f, t + 1 < S ? gsv[1] : 0.f, t + 2 < S ? gsv[2] : 0.f,
                       t + 3 < S ? gsv[3] : 0.f);
}

template <int ALPHA>
int launch_group(const float* logits, const float* head_max, const int64_t* sumfix,
                 const int32_t* seq_len, int B, int G, int Smax, float* gs, cudaStream_t st) {
  if (Smax % 4 == 0) {
    dim3 grid4((Smax / 4 + GRP_THREADS - 1) / GRP_THREADS, B * G);
    return launched(launch_k(group4_kernel<ALPHA>, grid4, dim3(GRP_THREADS), 0, st, logits,
                             head_max, sumfix, seq_len, G, Smax, gs));
  }
  dim3 grid((Smax + GRP_TILE - 1) / GRP_TILE, B * G);
  return launched(launch_k(group_kernel<ALPHA>, grid, dim3(GRP_THREADS), 0, st, logits,
                           head_max, sumfix, seq_len, G, Smax, gs));
}

// Debug (tools / tests only; not in include/spc.h): the device O3 exp on an array, scalar
// (spc_exp_dev) or packed f32x2 (spc_exp2_dev, the form NORM / GROUP / select run).
__global__ void exp_debug_kernel(const float* __restrict__ x, float* __restrict__ y, long long n,
                                 int packed) {
  for (long long i = 2 * ((long long)blockIdx.x * blockDim.x + threadIdx.x); i < n;
       i += 2ll * gridDim.x * blockDim.x) {
    const float a = x[i], b = i + 1 < n ? x[i + 1] : 0.f;
    if (packed) {
      const float2 e = spc_exp2_dev(a, b);
      y[i] = e.x;
      if (i + 1 < n) y[i + 1] = e.y;
    } else {
      y[i] = spc_exp_dev(a);
      if (i + 1 < n) y[i + 1] = spc_exp_dev(b);
    }
  }
}

struct ScoreWs {
  float* tile_max;     // [B][Hq][tiles of LG_TR rows] LOGITS: per-tile head maxima
  unsigned* lg_ctr;    // LOGITS: tile-claim counter
  long long* tile_sum;
  unsigned* cnt2;
  size_t bytes;
};
ScoreWs score_ws_layout(void* ws, int B, int Hq, int Smax) {
  const size_t nt2 = (Smax + NORM_TILE - 1) / NORM_TILE;
  uint8_t* p = (uint8_t*)ws;
  ScoreWs w;
  size_t off = 0;
  w.tile_max = (float*)(p + off);
  off = align_up(off + sizeof(float) * B * Hq * ((Smax + LG_TR - 1) / LG_TR) * LT_CPR, 256);
  w.lg_ctr = (unsigned*)(p + off);
  off = align_up(off + sizeof(unsigned) * 2, 256);
  w.tile_sum = (long long*)(p + off);
  off = align_up(off + sizeof(long long) * B * Hq * nt2, 256);
  w.cnt2 = (unsigned*)(p + off);
  off = align_up(off + sizeof(unsigned) * B * Hq, 256);
  w.bytes = off;
  return w;
}

}  // namespace
}  // namespace spc

using namespace spc;

extern "C" int spc_debug_exp(const float* x, float* y, long long n, int packed, spc_stream_t stream) {
  if (!x || !y || n < 0) return SPC_E_NULL;
  if (n == 0) return SPC_OK;
  exp_debug_kernel<<<4 * num_sms(), 256, 0, as_stream(stream)>>>(x, y, n, packed);
  return launched();
}

extern "C" size_t spc_score_workspace(int B, int Hq, int Smax) {
  if (B <= 0 || Hq <= 0 || Smax <= 0) return 0;
  return score_ws_layout(nullptr, B, Hq, Smax).bytes;
}

extern "C" int spc_score(int dtype, const void* q, const void* kr, const int32_t* seq_len, int B,
                         int Hq, int G, int D, int Smax, float scale, int phases, float* logits,
                         float* head_max, int64_t* head_sumfix, float* group_score, void* ws,
                         size_t ws_bytes, spc_stream_t stream) {
  if (!q || !kr || !seq_len || !logits || !head_max || !head_sumfix) return SPC_E_NULL;
  if ((phases & SPC_SCORE_GROUP) && !group_score) return SPC_E_NULL;
  if (B <= 0 || Hq <= 0 || G <= 0 || Smax <= 0 || Hq % G) return SPC_E_SHAPE;
  if (Smax >= SPC_MAX_SEQ) return SPC_E_RANGE;
  if (phases <= 0 || phases > (SPC_SCORE_ALL | SPC_SCORE_BATCH)) return SPC_E_RANGE;
  if ((phases & SPC_SCORE_BATCH) && (!(phases & SPC_SCORE_GROUP) || Hq > BT_MAXH))
    return (phases & SPC_SCORE_GROUP) ? SPC_E_UNSUPPORTED : SPC_E_RANGE;
  if (dtype != SPC_BF16) return SPC_E_UNSUPPORTED;
  const int alpha = Hq / G;
  if (!(D == 64 || D == 128) || !(alpha == 1 || alpha == 2 || alpha == 4 || alpha == 8))
    return SPC_E_UNSUPPORTED;
  if (!ws || ws_bytes < spc_score_workspace(B, Hq, Smax)) return SPC_E_WORKSPACE;
  if (((uintptr_t)kr & 15) != 0 || ((uintptr_t)q & 15) != 0) return SPC_E_RANGE;
  cudaStream_t st = as_stream(stream);
  ScoreWs w = score_ws_layout(ws, B, Hq, Smax);

  if (phases & SPC_SCORE_LOGITS) {
    const uint16_t* qq = (const uint16_t*)q;
#define LG(DD, AA)                                                                            \
  if (D == DD && alpha == AA)                                                                 \
    SPC_TRY((launch_logits<DD, AA>((const uint16_t*)kr, qq, seq_len, B, G, Smax, scale, logits, \
                                   w.tile_max, w.lg_ctr, head_max, st)));
    LG(64, 1) LG(64, 2) LG(64, 4) LG(64, 8) LG(128, 1) LG(128, 2) LG(128, 4) LG(128, 8)
#undef LG
  }
  if (phases & SPC_SCORE_NORM) {
    // enough CTAs per head for 8 CTAs (full occupancy) per SM, each with >= 8 float4 chunks
    // per thread (4 in flight): long rows are latency-bound otherwise (1M tokens: 64 us at
    // 2 CTAs per SM with 2 chunks in flight)
    const int want = (8 * num_sms() + B * Hq - 1) / (B * Hq);
    const int cap = (Smax + 8 * 4 * NM_T - 1) / (8 * 4 * NM_T);
    const int nb = max(1, min(want, cap));
    if (Smax % 4 == 0)
      (void)launch_k(norm_kernel<true>, dim3(nb, B * Hq), dim3(NM_T), 0, st, logits, head_max,
                     seq_len, Hq, Smax, (unsigned long long*)w.tile_sum, w.cnt2, head_sumfix);
    else
      (void)launch_k(norm_kernel<false>, dim3(nb, B * Hq), dim3(NM_T), 0, st, logits, head_max,
                     seq_len, Hq, Smax, (unsigned long long*)w.tile_sum, w.cnt2, head_sumfix);
    SPC_TRY(launched());
  }
  if ((phases & SPC_SCORE_GROUP) && (phases & SPC_SCORE_BATCH)) {
    dim3 grid((Smax + 2 * BT_THREADS - 1) / (2 * BT_THREADS), B);
    SPC_TRY(launched(launch_k(batch_kernel, grid, dim3(BT_THREADS), 0, st, logits, head_max,
                              head_sumfix, seq_len, Hq, G, Smax, group_score)));
  } else if (phases & SPC_SCORE_GROUP) {
    switch (alpha) {
      case 1:
        SPC_TRY(launch_group<1>(logits, head_max, head_sumfix, seq_len, B, G, Smax,
                                 group_score, st));
        break;
      case 2:
        SPC_TRY(launch_group<2>(logits, head_max, head_sumfix, seq_len, B, G, Smax,
                                 group_score, st));
        break;
      case 4:
        SPC_TRY(launch_group<4>(logits, head_max, head_sumfix, seq_len, B, G, Smax,
                                 group_score, st));
        break;
      case 8:
        SPC_TRY(launch_group<8>(logits, head_max, head_sumfix, seq_len, B, G, Smax,
                                 group_score, st));
        break;
    }
  }
  return SPC_OK;
}
