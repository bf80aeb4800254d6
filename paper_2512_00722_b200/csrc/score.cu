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
#include "common.cuh"

namespace spc {
namespace {

constexpr int LG_ROWS = 256;     // key rows per CTA tile (one TMA box height)
constexpr int LG_THREADS = 64;   // 4 rows per thread
constexpr int LG_DCHUNK = 64;    // d per TMA box (128 B inner extent, SWIZZLE_128B)
constexpr int NORM_THREADS = 256;
constexpr int NORM_PER = 8;      // elements per thread
constexpr int NORM_TILE = NORM_THREADS * NORM_PER;
constexpr int GRP_THREADS = 256;
constexpr int GRP_PER = 4;
constexpr int GRP_TILE = GRP_THREADS * GRP_PER;

template <int D, int ALPHA>
struct LgSmem {
  static constexpr int NCH = D / LG_DCHUNK;
  static constexpr size_t kbytes = (size_t)NCH * LG_ROWS * 128;  // bf16 rows, 128 B per chunk
  static constexpr size_t qbytes = (size_t)D * ALPHA * sizeof(float2);
  static constexpr size_t total = 1024 /*align slack*/ + kbytes + qbytes + 64;
};

template <int D, int ALPHA>
__global__ void __launch_bounds__(LG_THREADS) logits_kernel(
    const __grid_constant__ CUtensorMap kmap, const uint16_t* __restrict__ q,
    const int32_t* __restrict__ seq_len, int G, int Smax, float scale, float* __restrict__ logits,
    float* __restrict__ tile_max, unsigned int* __restrict__ counters,
    float* __restrict__ head_max) {
  constexpr int NCH = D / LG_DCHUNK;
  constexpr int Hq_per_g = ALPHA;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* kbuf = base;
  float2* qdup = (float2*)(base + LgSmem<D, ALPHA>::kbytes);
  uint64_t* bar = (uint64_t*)(base + LgSmem<D, ALPHA>::kbytes + LgSmem<D, ALPHA>::qbytes);
  __shared__ float red[2][ALPHA];
  __shared__ int flag;

  const int tid = threadIdx.x;
  const int tile = blockIdx.x, ntiles = gridDim.x;
  const int bg = blockIdx.y;
  const int b = bg / G, g = bg % G;
  const int Hq = G * ALPHA;
  const int S = seq_len[b];
  const int t0 = tile * LG_ROWS;
  const bool active = t0 < S;

  if (tid == 0) {
    prefetch_tmap(&kmap);
    for (int c = 0; c < NCH; ++c) mbar_init(&bar[c], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (active && tid == 0) {
    for (int c = 0; c < NCH; ++c) {
      mbar_arrive_expect_tx(&bar[c], LG_ROWS * 128);
      tma_load_3d(kbuf + (size_t)c * LG_ROWS * 128, &kmap, c * LG_DCHUNK, t0, bg, &bar[c]);
    }
  }
  // query of this (b, g): alpha heads, duplicated into float2 for FFMA2 row pairs
  for (int i = tid; i < D * ALPHA; i += LG_THREADS) {
    int d = i / ALPHA, j = i % ALPHA;
    float v = __uint_as_float((uint32_t)q[((size_t)b * Hq + g * ALPHA + j) * D + d] << 16);
    qdup[i] = make_float2(v, v);
  }
  __syncthreads();

  float hmax[ALPHA];
#pragma unroll
  for (int j = 0; j < ALPHA; ++j) hmax[j] = -INFINITY;

  if (active) {
    float2 acc[ALPHA][2];
#pragma unroll
    for (int j = 0; j < ALPHA; ++j) acc[j][0] = acc[j][1] = make_float2(0.f, 0.f);
    int r[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) r[k] = tid + LG_THREADS * k;
    const uint32_t kbase = smem_u32(kbuf), qbase = smem_u32(qdup);

#pragma unroll 1
    for (int c = 0; c < NCH; ++c) {
      mbar_wait(&bar[c], 0);
      const uint32_t kc = kbase + (uint32_t)c * LG_ROWS * 128;
#pragma unroll 2
      for (int u = 0; u < 8; ++u) {  // 16-byte granule = 8 consecutive d
        uint4 w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)  // SWIZZLE_128B: granule u of row r lives at u ^ (r & 7)
          w[k] = lds128(kc + r[k] * 128 + ((u ^ (r[k] & 7)) << 4));
        const uint32_t qd = qbase + (uint32_t)(c * LG_DCHUNK + u * 8) * ALPHA * 8;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          uint32_t w0 = (&w[0].x)[e >> 1], w1 = (&w[1].x)[e >> 1];
          uint32_t w2 = (&w[2].x)[e >> 1], w3 = (&w[3].x)[e >> 1];
          float2 k01, k23;
          if (e & 1) {
            k01 = make_float2(bf16hi(w0), bf16hi(w1));
            k23 = make_float2(bf16hi(w2), bf16hi(w3));
          } else {
            k01 = make_float2(bf16lo(w0), bf16lo(w1));
            k23 = make_float2(bf16lo(w2), bf16lo(w3));
          }
#pragma unroll
          for (int j = 0; j < ALPHA; j += 2) {
            float2 qq0, qq1;
            if (ALPHA >= 2) {
              const float4 q4 = lds128f(qd + (uint32_t)(e * ALPHA + j) * 8);
              qq0 = make_float2(q4.x, q4.y);
              qq1 = make_float2(q4.z, q4.w);
            } else {
              qq0 = lds64f(qd + (uint32_t)(e * ALPHA + j) * 8);
            }
            acc[j][0] = ffma2(k01, qq0, acc[j][0]);
            acc[j][1] = ffma2(k23, qq0, acc[j][1]);
            if (ALPHA >= 2) {
              acc[j + 1][0] = ffma2(k01, qq1, acc[j + 1][0]);
              acc[j + 1][1] = ffma2(k23, qq1, acc[j + 1][1]);
            }
          }
        }
      }
    }
    // O1 final multiply by scale, store, O2 partial max
#pragma unroll
    for (int j = 0; j < ALPHA; ++j) {
      float s[4] = {__fmul_rn(acc[j][0].x, scale), __fmul_rn(acc[j][0].y, scale),
                    __fmul_rn(acc[j][1].x, scale), __fmul_rn(acc[j][1].y, scale)};
      float* out = logits + ((size_t)b * Hq + g * ALPHA + j) * Smax + t0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (t0 + r[k] < S) {
          out[r[k]] = s[k];
          hmax[j] = fmaxf(hmax[j], s[k]);
        }
      }
    }
  }
  const int warp = tid >> 5, lane = tid & 31;
#pragma unroll
  for (int j = 0; j < ALPHA; ++j) {
    float m = warp_max(hmax[j]);
    if (lane == 0) red[warp][j] = m;
  }
  __syncthreads();
  if (tid < ALPHA)
    tile_max[((size_t)b * Hq + g * ALPHA + tid) * ntiles + tile] = fmaxf(red[0][tid], red[1][tid]);
  if (last_block_ticket(&counters[bg], ntiles, &flag)) {
    // reduce partial maxima of the ALPHA heads of this group
    for (int j = warp; j < ALPHA; j += LG_THREADS / 32) {
      const float* tm = tile_max + ((size_t)b * Hq + g * ALPHA + j) * ntiles;
      float m = -INFINITY;
      for (int i = lane; i < ntiles; i += 32) m = fmaxf(m, __ldcg(tm + i));
      m = warp_max(m);
      if (lane == 0) head_max[(size_t)b * Hq + g * ALPHA + j] = m;
    }
  }
  (void)Hq_per_g;
}

// ---------------------------------------------------------------- NORM (O3, O4)
__global__ void __launch_bounds__(NORM_THREADS) norm_kernel(
    const float* __restrict__ logits, const float* __restrict__ head_max,
    const int32_t* __restrict__ seq_len, int Hq, int Smax, long long* __restrict__ tile_sum,
    unsigned int* __restrict__ counters, int64_t* __restrict__ head_sumfix) {
  __shared__ long long red[NORM_THREADS / 32];
  __shared__ int flag;
  const int bh = blockIdx.y, b = bh / Hq;
  const int tile = blockIdx.x, ntiles = gridDim.x;
  const int S = seq_len[b];
  const float m = head_max[bh];
  const float* row = logits + (size_t)bh * Smax;
  long long acc = 0;
  const int t0 = tile * NORM_TILE + threadIdx.x;
#pragma unroll
  for (int i = 0; i < NORM_PER; ++i) {
    int t = t0 + i * NORM_THREADS;
    if (t < S) acc += fixpoint40(spc_exp_dev(__fsub_rn(__ldcg(row + t), m)));
  }
  acc = warp_sum_ll(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long s = 0;
    for (int w = 0; w < NORM_THREADS / 32; ++w) s += red[w];
    tile_sum[(size_t)bh * ntiles + tile] = s;
  }
  if (last_block_ticket(&counters[bh], ntiles, &flag)) {
    if (threadIdx.x < 32) {
      long long s = 0;
      for (int i = threadIdx.x; i < ntiles; i += 32) s += __ldcg(tile_sum + (size_t)bh * ntiles + i);
      s = warp_sum_ll(s);
      if (threadIdx.x == 0) head_sumfix[bh] = s;
    }
  }
}

// ------------------------------------------------------------- GROUP (O4..O6)
template <int ALPHA>
__global__ void __launch_bounds__(GRP_THREADS) group_kernel(
    const float* __restrict__ logits, const float* __restrict__ head_max,
    const int64_t* __restrict__ head_sumfix, const int32_t* __restrict__ seq_len, int G, int Smax,
    float* __restrict__ group_score) {
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
int launch_logits(const CUtensorMap& map, const uint16_t* q, const int32_t* seq_len, int B, int G,
                  int Smax, float scale, float* logits, float* tile_max, unsigned* counters,
                  float* head_max, cudaStream_t st) {
  const size_t smem = LgSmem<D, ALPHA>::total;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(logits_kernel<D, ALPHA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    attr = true;
  }
  dim3 grid((Smax + LG_ROWS - 1) / LG_ROWS, B * G);
  logits_kernel<D, ALPHA><<<grid, LG_THREADS, smem, st>>>(map, q, seq_len, G, Smax, scale, logits,
                                                          tile_max, counters, head_max);
  return launched();
}

template <int ALPHA>
int launch_group(const float* logits, const float* head_max, const int64_t* sumfix,
                 const int32_t* seq_len, int B, int G, int Smax, float* gs, cudaStream_t st) {
  dim3 grid((Smax + GRP_TILE - 1) / GRP_TILE, B * G);
  group_kernel<ALPHA><<<grid, GRP_THREADS, 0, st>>>(logits, head_max, sumfix, seq_len, G, Smax, gs);
  return launched();
}

struct ScoreWs {
  float* tile_max;
  long long* tile_sum;
  unsigned* cnt1;
  unsigned* cnt2;
  size_t bytes;
};
ScoreWs score_ws_layout(void* ws, int B, int Hq, int Smax) {
  const size_t nt1 = (Smax + LG_ROWS - 1) / LG_ROWS, nt2 = (Smax + NORM_TILE - 1) / NORM_TILE;
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
    CUtensorMap map;
    SPC_TRY(make_tmap_3d_bf16(&map, kr, D, Smax, (uint64_t)B * G, LG_DCHUNK, LG_ROWS,
                              CU_TENSOR_MAP_SWIZZLE_128B));
    const uint16_t* qq = (const uint16_t*)q;
#define LG(DD, AA)                                                                            \
  if (D == DD && alpha == AA)                                                                 \
    SPC_TRY((launch_logits<DD, AA>(map, qq, seq_len, B, G, Smax, scale, logits, w.tile_max, \
                                   w.cnt1, head_max, st)));
    LG(64, 1) LG(64, 2) LG(64, 4) LG(64, 8) LG(128, 1) LG(128, 2) LG(128, 4) LG(128, 8)
#undef LG
  }
  if (phases & SPC_SCORE_NORM) {
    dim3 grid((Smax + NORM_TILE - 1) / NORM_TILE, B * Hq);
    norm_kernel<<<grid, NORM_THREADS, 0, st>>>(logits, head_max, seq_len, Hq, Smax, w.tile_sum,
                                               w.cnt2, head_sumfix);
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
