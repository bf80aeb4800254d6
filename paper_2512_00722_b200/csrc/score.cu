// score.cu — spc_score: retrieval-head scoring O1..O6.
//
// Paper: Eq.1 softmax(QK^T/sqrt(d)) of the lightweight retrieval
// head over its full key cache, then the GQA group maximum of
// the weights (MQA P:331).
//
// Three kernels (phases), each HBM- or L2-streaming:
//   LOGITS  streams the bf16 key cache once (the dominant bytes).  TMA 3-D tile
//           loads (256 rows x 64 d, 128B swizzle, one mbarrier per d-chunk) into
//           shared memory; one thread owns 4 key rows and runs alpha sequential
//           fp32 FMA chains per row (bit-exact O1), two rows at a time with the
//           packed sm_100 FFMA2 (fma.rn.f32x2: per-lane IEEE fma, order kept).
//           The key row feeds all alpha query heads of its group (no repeat_kv).
//   NORM    exp + exact int64 fixed-point sums (O3, O4), L2-resident logits.
//   GROUP   weights and group max (O5, O6).
// Per-tile partial max / sums go to the workspace; the last CTA of each group
// reduces them (order-free: max and integer add), so results are deterministic.
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
// One thread-block cluster of NM_CL CTAs per head: each CTA sums its quarter of
// the (L2-resident) logits row, the partial int64 sums meet in CTA 0 through
// distributed shared memory (integer addition: exact, order-free).
constexpr int NM_CL = 4;
constexpr int NM_T = 512;
__global__ void __cluster_dims__(NM_CL, 1, 1) __launch_bounds__(NM_T) norm_kernel(
    const float* __restrict__ logits, const float* __restrict__ head_max,
    const int32_t* __restrict__ seq_len, int Hq, int Smax, int64_t* __restrict__ head_sumfix) {
  spc_pdl_entry();
  __shared__ long long red[NM_T / 32];
  __shared__ long long part;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int bh = blockIdx.y, b = bh / Hq;
  const int S = seq_len[b];
  const float m = head_max[bh];
  const float* row = logits + (size_t)bh * Smax;
  const int per = (S + NM_CL - 1) / NM_CL;
  const int s0 = min(S, rank * per), s1 = min(S, s0 + per);
  long long acc = 0;
#pragma unroll 4
  for (int t = s0 + threadIdx.x; t < s1; t += NM_T)
    acc += fixpoint40(spc_exp_dev(__fsub_rn(__ldcg(row + t), m)));
  acc = warp_sum_ll(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long s = 0;
    for (int w = 0; w < NM_T / 32; ++w) s += red[w];
    part = s;
  }
  cl.sync();
  if (rank == 0 && threadIdx.x == 0) {
    long long s = 0;
    for (int r = 0; r < NM_CL; ++r) s += *cl.map_shared_rank(&part, r);
    head_sumfix[bh] = s;
  }
  cl.sync();  // remote reads of `part` done before any CTA exits
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
  for (int i = 0; i < GRP_PER; ++i) {
    const int t = t0 + i * GRP_THREADS;
    if (t >= Smax) break;
    float gs = 0.0f;
    if (t < S) {
#pragma unroll
      for (int j = 0; j < ALPHA; ++j) {
        const float p = __fmul_rn(spc_exp_dev(__fsub_rn(__ldcg(lg + (size_t)j * Smax + t), m[j])), r[j]);
        gs = j ? fmaxf(gs, p) : p;
      }
    }
    out[t] = gs;
  }
}

template <int D, int ALPHA>
int launch_logits(const uint16_t* kr, const uint16_t* q, const int32_t* seq_len, int B, int G,
                  int Smax, float scale, float* logits, float* seg_max, int segstride,
                  unsigned* counters, float* head_max, cudaStream_t st) {
  const size_t smem = Lg4Smem<D, ALPHA>::BYTES;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(logits_kernel<D, ALPHA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    attr = true;
  }
  const int tpr = (Smax + LG_TR - 1) / LG_TR;
  const int ntiles = B * G * tpr;
  int tpc = (ntiles + num_sms() - 1) / num_sms();
  if (tpc > tpr) tpc = tpr;  // a CTA spans at most two groups
  const int ncta = (ntiles + tpc - 1) / tpc;
  (void)launch_k(logits_kernel<D, ALPHA>, dim3(ncta), dim3(32 * lg_warps<ALPHA>()), smem, st, kr, q, seq_len, G, Smax,
                                                                      scale, tpc, tpr,
                                                    ntiles, logits, seg_max, segstride, counters,
                                                    head_max);
  return launched();
}

template <int ALPHA>
int launch_group(const float* logits, const float* head_max, const int64_t* sumfix,
                 const int32_t* seq_len, int B, int G, int Smax, float* gs, cudaStream_t st) {
  dim3 grid((Smax + GRP_TILE - 1) / GRP_TILE, B * G);
  (void)launch_k(group_kernel<ALPHA>, dim3(grid), dim3(GRP_THREADS), 0, st, logits, head_max, sumfix, seq_len, G, Smax, gs);
  return launched();
}

struct ScoreWs {
  float* tile_max;
  long long* tile_sum;
  unsigned* cnt1;
  unsigned* cnt2;
  size_t nt1;  // segment stride of tile_max
  size_t bytes;
};
ScoreWs score_ws_layout(void* ws, int B, int Hq, int Smax) {
  // nt1 bounds the CTA segments of one group in LOGITS (every CTA owns >= 1 tile)
  const size_t nt1 = (Smax + LG_TR - 1) / LG_TR + 2, nt2 = (Smax + NORM_TILE - 1) / NORM_TILE;
  uint8_t* p = (uint8_t*)ws;
  ScoreWs w;
  size_t off = 0;
  w.tile_max = (float*)(p + off);
  off = align_up(off + sizeof(float) * B * Hq * nt1, 256);
  w.tile_sum = (long long*)(p + off);
  off = align_up(off + sizeof(long long) * B * Hq * nt2, 256);
  w.cnt1 = (unsigned*)(p + off);
  off = align_up(off + sizeof(unsigned) * B * Hq, 256);
  w.cnt2 = (unsigned*)(p + off);
  off = align_up(off + sizeof(unsigned) * B * Hq, 256);
  w.nt1 = nt1;
  w.bytes = off;
  return w;
}

}  // namespace
}  // namespace spc

using namespace spc;

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
  if (phases <= 0 || phases > SPC_SCORE_ALL) return SPC_E_RANGE;
  if (dtype != SPC_BF16) return SPC_E_UNSUPPORTED;
  const int alpha = Hq / G;
  if (!(D == 64 || D == 128) || !(alpha == 1 || alpha == 2 || alpha == 4 || alpha == 8))
    return SPC_E_UNSUPPORTED;
  if (!ws || ws_bytes < spc_score_workspace(B, Hq, Smax)) return SPC_E_WORKSPACE;
  if (((uintptr_t)kr & 15) != 0) return SPC_E_RANGE;
  cudaStream_t st = as_stream(stream);
  ScoreWs w = score_ws_layout(ws, B, Hq, Smax);

  if (phases & SPC_SCORE_LOGITS) {
    const uint16_t* qq = (const uint16_t*)q;
#define LG(DD, AA)                                                                            \
  if (D == DD && alpha == AA)                                                                 \
    SPC_TRY((launch_logits<DD, AA>((const uint16_t*)kr, qq, seq_len, B, G, Smax, scale, logits, w.tile_max, \
                                   (int)w.nt1, w.cnt1, head_max, st)));
    LG(64, 1) LG(64, 2) LG(64, 4) LG(64, 8) LG(128, 1) LG(128, 2) LG(128, 4) LG(128, 8)
#undef LG
  }
  if (phases & SPC_SCORE_NORM) {
    (void)launch_k(norm_kernel, dim3(dim3(NM_CL, B * Hq)), dim3(NM_T), 0, st, logits, head_max, seq_len, Hq, Smax,
                                                      head_sumfix);
    SPC_TRY(launched());
  }
  if (phases & SPC_SCORE_GROUP) {
    switch (alpha) {
      case 1: SPC_TRY(launch_group<1>(logits, head_max, head_sumfix, seq_len, B, G, Smax, group_score, st)); break;
      case 2: SPC_TRY(launch_group<2>(logits, head_max, head_sumfix, seq_len, B, G, Smax, group_score, st)); break;
      case 4: SPC_TRY(launch_group<4>(logits, head_max, head_sumfix, seq_len, B, G, Smax, group_score, st)); break;
      case 8: SPC_TRY(launch_group<8>(logits, head_max, head_sumfix, seq_len, B, G, Smax, group_score, st)); break;
    }
  }
  return SPC_OK;
}
