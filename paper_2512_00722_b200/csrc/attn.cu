// attn.cu — spc_sparse_decode_attn (O10) and spc_attn_merge (O12).
//
// Paper: the LLM's attention Eq.1 restricted to the tokens the
// retrieval head selected, mapped per KV head (P:324 torch.gather; GQA group
// sets P:328), renormalised over the subset (reading R15).
//
// Split-K flash-decode, three kernels:
//  * attn_tma_kernel + tma_merge_kernel (spc_sparse_decode_attn_kv, the hot path): the
//    selected K and V rows are gathered straight from the cache by the TMA unit
//    (tile::gather4, 4 rows per request, per-layer descriptors from spc_kv_desc_init);
//    one producer warp and one mma.sync consumer warp per CTA, 4 CTAs per SM; per-CTA
//    (m, l, o) partials merged by a PDL-chained merge kernel (attn_tma.cuh).
//  * attn_bf16_kernel (spc_sparse_decode_attn, pointer tables: any device-addressable
//    layer pointers): per-warp 16-byte cp.async rings + the same mma.sync math, partials
//    merged by the CTA completing a group (attn_bf16.cuh).
//  * attn_f32_kernel: CUDA-core dot products for fp32 inputs (the 1e-5 tolerance tests).
// All alpha query heads of a group share each K/V row (GQA: one read serves alpha heads);
// no compacted copy of the selected rows is materialised in HBM.
#include "common.cuh"

namespace spc {
namespace {

constexpr int AT_ROWS = 128;   // selected rows per CTA
constexpr int AT_THREADS = 128;
constexpr float LOG2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;

struct AttnWs {
  float* part_o;   // [L][B][Hq][segstride][D]  (unnormalised o relative to m)
  float* part_ml;  // [L][B][Hq][segstride][2]  (m in log2 units, l)
  unsigned* cnt;   // [L][B][G]
  int segstride;   // max segments (partials) per group
  size_t bytes;
};
AttnWs attn_ws_layout(void* ws, int L, int B, int Hq, int D, int k) {
  // >= the split count of the fp32 path and (CTA segments of a group) x 4 warps of the
  // persistent bf16 path
  const size_t ns = 4 * ((k + 63) / 64 + 2);
  uint8_t* p = (uint8_t*)ws;
  AttnWs w;
  size_t off = 0;
  w.part_o = (float*)(p + off);
  off = align_up(off + sizeof(float) * (size_t)L * B * Hq * ns * D, 256);
  w.part_ml = (float*)(p + off);
  off = align_up(off + sizeof(float) * 2 * (size_t)L * B * Hq * ns, 256);
  w.cnt = (unsigned*)(p + off);
  off = align_up(off + sizeof(unsigned) * (size_t)L * B * Hq, 256);
  w.segstride = (int)ns;
  w.bytes = off;
  return w;
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                          uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
// Merge the nsplit partials of one (layer, b, g) with the LSE rule (O12); run by
// the last CTA of the group.  m is in log2 units.
template <int D, int ALPHA>
__device__ void merge_partials(const float* part_o, const float* part_ml, int nsplit,
                               int segstride, size_t head_base /* (lr*B + b)*Hq + g*ALPHA */, float* out,
                               float* lse, size_t out_head_base, int nthreads) {
  for (int i = threadIdx.x; i < ALPHA * D; i += nthreads) {
    const int j = i / D, d = i % D;
    const size_t h = head_base + j;
    const float* ml = part_ml + h * segstride * 2;
    float M = -INFINITY;
    for (int s = 0; s < nsplit; ++s) M = fmaxf(M, __ldcg(ml + 2 * s));
    float den = 0.f, num = 0.f;
    if (M != -INFINITY) {
      for (int s = 0; s < nsplit; ++s) {
        const float m = __ldcg(ml + 2 * s);
        if (m == -INFINITY) continue;
        const float w = exp2f(m - M);
        den += w * __ldcg(ml + 2 * s + 1);
        num += w * __ldcg(part_o + (h * segstride + s) * D + d);
      }
    }
    out[(out_head_base + j) * D + d] = den > 0.f ? num / den : 0.f;
    if (lse && d == 0) lse[out_head_base + j] = den > 0.f ? (M + log2f(den)) * LN2 : -INFINITY;
  }
}

#include "attn_bf16.cuh"
#include "attn_tma.cuh"

// ---------------------------------------------------------------- fp32 / CUDA-core path
template <int D, int ALPHA>
__global__ void __launch_bounds__(AT_THREADS) attn_f32_kernel(
    const float* __restrict__ q, const void* const* __restrict__ k_layers,
    const void* const* __restrict__ v_layers, int kv_mode, const int32_t* __restrict__ idx,
    const int32_t* __restrict__ count, int layer_begin, int B, int G, int rows, int kbud,
    float scale, int nsplit, int segstride, float* __restrict__ part_o,
    float* __restrict__ part_ml, unsigned* __restrict__ cnt, float* __restrict__ out,
    float* __restrict__ lse) {
  spc_pdl_entry();
  __shared__ float qs[ALPHA][D];
  __shared__ float ps[ALPHA][AT_ROWS];
  __shared__ int toks[AT_ROWS];
  __shared__ float red[AT_THREADS / 32][ALPHA];
  __shared__ float mh[ALPHA], lh[ALPHA];
  __shared__ int flag;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int split = blockIdx.x, bg = blockIdx.y, lr = blockIdx.z;
  const int l = layer_begin + lr;
  const int b = bg / G, g = bg % G;
  const int Hq = G * ALPHA;
  const int n_sel = min(count[bg], kbud);
  const int r0 = split * AT_ROWS;
  const int nrows = max(0, min(AT_ROWS, n_sel - r0));
  const size_t head_base = ((size_t)lr * B + b) * Hq + g * ALPHA;
  const float* Kl = (const float*)k_layers[l] + (size_t)bg * rows * D;
  const float* Vl = (const float*)v_layers[l] + (size_t)bg * rows * D;
  for (int i = tid; i < ALPHA * D; i += AT_THREADS)
    qs[i / D][i % D] = q[(((size_t)l * B + b) * Hq + g * ALPHA) * D + i];
  if (tid < nrows)
    toks[tid] = kv_mode == SPC_KV_INDEXED ? idx[(size_t)bg * kbud + r0 + tid] : r0 + tid;
  __syncthreads();
  float s[ALPHA];
#pragma unroll
  for (int j = 0; j < ALPHA; ++j) s[j] = -INFINITY;
  if (tid < nrows) {
    const float* kr = Kl + (size_t)toks[tid] * D;
#pragma unroll
    for (int j = 0; j < ALPHA; ++j) s[j] = 0.f;
    for (int d = 0; d < D; ++d) {
      const float kv = kr[d];
#pragma unroll
      for (int j = 0; j < ALPHA; ++j) s[j] = fmaf(qs[j][d], kv, s[j]);
    }
#pragma unroll
    for (int j = 0; j < ALPHA; ++j) s[j] *= scale;
  }
#pragma unroll
  for (int j = 0; j < ALPHA; ++j) {
    float m = warp_max(s[j]);
    if (lane == 0) red[warp][j] = m;
  }
  __syncthreads();
  if (tid < ALPHA) {
    float m = -INFINITY;
    for (int w = 0; w < AT_THREADS / 32; ++w) m = fmaxf(m, red[w][tid]);
    mh[tid] = m;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < ALPHA; ++j) {
    const float pj = (tid < nrows) ? expf(s[j] - mh[j]) : 0.f;
    ps[j][tid] = pj;
    float sum = warp_sum(pj);
    if (lane == 0) red[warp][j] = sum;
  }
  __syncthreads();
  if (tid < ALPHA) {
    float t = 0.f;
    for (int w = 0; w < AT_THREADS / 32; ++w) t += red[w][tid];
    lh[tid] = t;
  }
  for (int i = tid; i < ALPHA * D; i += AT_THREADS) {
    const int j = i / D, d = i % D;
    float acc = 0.f;
    for (int r = 0; r < nrows; ++r) acc = fmaf(ps[j][r], Vl[(size_t)toks[r] * D + d], acc);
    part_o[((head_base + j) * segstride + split) * D + d] = acc;
  }
  __syncthreads();
  if (tid < ALPHA) {
    part_ml[((head_base + tid) * segstride + split) * 2] = nrows > 0 ? mh[tid] * LOG2E : -INFINITY;
    part_ml[((head_base + tid) * segstride + split) * 2 + 1] = nrows > 0 ? lh[tid] : 0.f;
  }
  const size_t grp = (size_t)lr * B * G + bg;
  if (last_block_ticket(&cnt[grp], nsplit, &flag))
    merge_partials<D, ALPHA>(part_o, part_ml, nsplit, segstride, head_base, out, lse,
                             ((size_t)l * B + b) * Hq + g * ALPHA, AT_THREADS);
}

__global__ void merge_kernel(const float* __restrict__ o_parts, const float* __restrict__ lse_parts,
                             int P, int n, int D, float* __restrict__ out,
                             float* __restrict__ lse_out) {
  spc_pdl_entry();
  const int row = blockIdx.x;
  float M = -INFINITY;
  for (int p = 0; p < P; ++p) M = fmaxf(M, lse_parts[(size_t)p * n + row]);
  float den = 0.f;
  for (int p = 0; p < P; ++p) {
    const float x = lse_parts[(size_t)p * n + row];
    if (x != -INFINITY) den += expf(x - M);
  }
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    float num = 0.f;
    if (M != -INFINITY)
      for (int p = 0; p < P; ++p) {
        const float x = lse_parts[(size_t)p * n + row];
        if (x != -INFINITY) num += expf(x - M) * o_parts[((size_t)p * n + row) * D + d];
      }
    out[(size_t)row * D + d] = den > 0.f ? num / den : 0.f;
  }
  if (threadIdx.x == 0 && lse_out) lse_out[row] = den > 0.f ? M + logf(den) : -INFINITY;
}

}  // namespace
}  // namespace spc

using namespace spc;

extern "C" size_t spc_attn_workspace(int L, int B, int Hq, int D, int k) {
  if (L <= 0 || B <= 0 || Hq <= 0 || D <= 0 || k <= 0) return 0;
  return attn_ws_layout(nullptr, L, B, Hq, D, k).bytes;
}

extern "C" int spc_sparse_decode_attn(int dtype, const void* q, const void* const* k_layers,
                                      const void* const* v_layers, int kv_mode, const int32_t* idx,
                                      const int32_t* count, int L, int layer_begin, int layer_end,
                                      int B, int Hq, int G, int D, int rows, int k, float scale,
                                      float* out, float* lse, void* ws, size_t ws_bytes,
                                      spc_stream_t stream) {
  if (!q || !k_layers || !v_layers || !count || !out) return SPC_E_NULL;
  if (kv_mode == SPC_KV_INDEXED && !idx) return SPC_E_NULL;
  if (kv_mode != SPC_KV_INDEXED && kv_mode != SPC_KV_SLOTS) return SPC_E_RANGE;
  if (L <= 0 || B <= 0 || Hq <= 0 || G <= 0 || Hq % G || rows <= 0) return SPC_E_SHAPE;
  if (k < 1 || k > SPC_MAX_K) return SPC_E_BUDGET;
  if (kv_mode == SPC_KV_SLOTS && rows < k) return SPC_E_SHAPE;
  if (layer_begin < 0 || layer_end > L || layer_begin > layer_end) return SPC_E_RANGE;
  if (layer_begin == layer_end) return SPC_OK;
  if (!ws || ws_bytes < spc_attn_workspace(L, B, Hq, D, k)) return SPC_E_WORKSPACE;
  const int alpha = Hq / G;
  if (!(D == 64 || D == 128) || !(alpha == 1 || alpha == 2 || alpha == 4 || alpha == 8))
    return SPC_E_UNSUPPORTED;
  if (dtype != SPC_BF16 && dtype != SPC_F32) return SPC_E_UNSUPPORTED;
  AttnWs w = attn_ws_layout(ws, L, B, Hq, D, k);
  const int nsplit = (k + AT_ROWS - 1) / AT_ROWS;
  const int n_groups = (layer_end - layer_begin) * B * G;
  cudaStream_t st = as_stream(stream);
  // persistent bf16 path: AT2_CTAS_PER_SM CTAs per SM, contiguous chunk-aligned row ranges
  const int kpad = (k + CH - 1) / CH * CH;  // groups padded to whole chunks
  const long long v_total = (long long)n_groups * kpad;
#ifndef SPC_ATTN_OVERSUB
#define SPC_ATTN_OVERSUB 1
#endif
  const int ncta_target = AT2_CTAS_PER_SM * num_sms() * SPC_ATTN_OVERSUB;
  long long rpc = (v_total + ncta_target - 1) / ncta_target;
  rpc = (rpc + CH - 1) / CH * CH;
  const int ncta = (int)((v_total + rpc - 1) / rpc);
#define AT(DD, AA)                                                                              \
  if (D == DD && alpha == AA) {                                                                 \
    if (dtype == SPC_BF16) {                                                                    \
      const int smem = PSmem<DD, AA>::BYTES;                                                    \
      SPC_TRY(smem_attr((const void*)attn_bf16_kernel<DD, AA>, smem));                          \
      (void)launch_k(attn_bf16_kernel<DD, AA>, dim3(ncta), dim3(AT2_THREADS), smem, st,      \
          (const uint16_t*)q, k_layers, v_layers, kv_mode, idx, count, layer_begin, B, G, rows, \
          k, kpad, scale, (int)(rpc / CH), n_groups, w.segstride, w.part_o, w.part_ml, w.cnt,   \
          out, lse);                                                                            \
    } else {                                                                                    \
      dim3 grid(nsplit, B * G, layer_end - layer_begin);                                        \
      (void)launch_k(attn_f32_kernel<DD, AA>, dim3(grid), dim3(AT_THREADS), 0, st,          \
          (const float*)q, k_layers, v_layers, kv_mode, idx, count, layer_begin, B, G, rows, k, \
          scale, nsplit, w.segstride, w.part_o, w.part_ml, w.cnt, out, lse);                    \
    }                                                                                           \
    return launched();                                                                          \
  }
  AT(64, 1) AT(64, 2) AT(64, 4) AT(64, 8) AT(128, 1) AT(128, 2) AT(128, 4) AT(128, 8)
#undef AT
  return SPC_E_UNSUPPORTED;
}

extern "C" size_t spc_kv_desc_bytes(int L) { return L > 0 ? (size_t)2 * L * sizeof(CUtensorMap) : 0; }

namespace spc {
namespace {
struct TmPart {
  int n_groups, kpad, cpc, ncta;
};
TmPart tm_partition(int layer_begin, int layer_end, int B, int G, int k) {
  TmPart p;
  p.n_groups = (layer_end - layer_begin) * B * G;
  p.kpad = (k + TM_RPS - 1) / TM_RPS * TM_RPS;
  const long long v_total = (long long)p.n_groups * p.kpad;
  const int ncta_target = TM_CTAS * num_sms();
  long long rpc = (v_total + ncta_target - 1) / ncta_target;
  rpc = (rpc + TM_RPS - 1) / TM_RPS * TM_RPS;
  p.ncta = (int)((v_total + rpc - 1) / rpc);
  p.cpc = (int)(rpc / TM_RPS);
  return p;
}

}  // namespace
}  // namespace spc

extern "C" int spc_kv_desc_init(void* desc, const void* const* k_layers, const void* const* v_layers,
                                int L, int B, int G, int D, int rows) {
  if (!desc || !k_layers || !v_layers) return SPC_E_NULL;
  if (L <= 0 || B <= 0 || G <= 0 || rows <= 0) return SPC_E_SHAPE;
  if (!(D == 64 || D == 128)) return SPC_E_UNSUPPORTED;
  if ((uintptr_t)desc % 64) return SPC_E_RANGE;
  const uint64_t n_rows = (uint64_t)B * G * rows;
  if (n_rows >= (1ull << 31)) return SPC_E_SHAPE;  // TMA row coordinates are int32
  CUtensorMap* h = (CUtensorMap*)std::calloc(2 * (size_t)L, sizeof(CUtensorMap));
  if (!h) return SPC_E_CUDA;
  int rc = SPC_OK;
  for (int l = 0; l < L && rc == SPC_OK; ++l) {
    if (!k_layers[l] || !v_layers[l] || (uintptr_t)k_layers[l] % 16 || (uintptr_t)v_layers[l] % 16) {
      rc = !k_layers[l] || !v_layers[l] ? SPC_E_NULL : SPC_E_RANGE;
      break;
    }
    rc = make_tmap_rows_bf16(h + l, k_layers[l], n_rows, (uint32_t)D);
    if (rc == SPC_OK) rc = make_tmap_rows_bf16(h + L + l, v_layers[l], n_rows, (uint32_t)D);
  }
  if (rc == SPC_OK) {
    const cudaError_t e = cudaMemcpy(desc, h, 2 * (size_t)L * sizeof(CUtensorMap), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      set_cuda_error(e);
      rc = SPC_E_CUDA;
    }
  }
  std::free(h);
  return rc;
}

extern "C" int spc_sparse_decode_attn_kv(const void* kv_desc, const void* q, int kv_mode,
                                         const int32_t* idx, const int32_t* count, int L,
                                         int layer_begin, int layer_end, int B, int Hq, int G, int D,
                                         int rows, int k, float scale, float* out, float* lse,
                                         void* ws, size_t ws_bytes, spc_stream_t stream) {
  if (!kv_desc || !q || !count || !out) return SPC_E_NULL;
  if (kv_mode == SPC_KV_INDEXED && !idx) return SPC_E_NULL;
  if (kv_mode != SPC_KV_INDEXED && kv_mode != SPC_KV_SLOTS) return SPC_E_RANGE;
  if (L <= 0 || B <= 0 || Hq <= 0 || G <= 0 || Hq % G || rows <= 0) return SPC_E_SHAPE;
  if (k < 1 || k > SPC_MAX_K) return SPC_E_BUDGET;
  if (kv_mode == SPC_KV_SLOTS && rows < k) return SPC_E_SHAPE;
  if ((uint64_t)B * G * rows >= (1ull << 31)) return SPC_E_SHAPE;
  if (layer_begin < 0 || layer_end > L || layer_begin > layer_end) return SPC_E_RANGE;
  if ((uintptr_t)kv_desc % 64) return SPC_E_RANGE;
  if (layer_begin == layer_end) return SPC_OK;
  if (!ws || ws_bytes < spc_attn_workspace(L, B, Hq, D, k)) return SPC_E_WORKSPACE;
  const int alpha = Hq / G;
  if (!(D == 64 || D == 128) || !(alpha == 1 || alpha == 2 || alpha == 4 || alpha == 8))
    return SPC_E_UNSUPPORTED;
  AttnWs w = attn_ws_layout(ws, L, B, Hq, D, k);
  const TmPart part = tm_partition(layer_begin, layer_end, B, G, k);
  const int n_groups = part.n_groups, kpad = part.kpad, ncta = part.ncta;
  const long long rpc = (long long)part.cpc * TM_RPS;
  cudaStream_t st = as_stream(stream);
  const CUtensorMap* maps = (const CUtensorMap*)kv_desc;
#define ATK(DD, AA)                                                                               \
  if (D == DD && alpha == AA) {                                                                   \
    SPC_TRY(smem_attr((const void*)attn_tma_kernel<DD, AA>, TmSmem<DD>::BYTES));                  \
    SPC_TRY(launched(launch_k(attn_tma_kernel<DD, AA>, dim3(ncta), dim3(TM_THREADS),             \
                              TmSmem<DD>::BYTES, st, (const uint16_t*)q, maps, L, kv_mode, idx,   \
                              count, layer_begin, B, G, rows, k, kpad, scale,                     \
                              (int)(rpc / TM_RPS), n_groups, w.segstride, w.part_o, w.part_ml)));  \
    return launched(launch_k(tma_merge_kernel<DD, AA>, dim3((n_groups * AA + 3) / 4), dim3(128), \
                             0, st, w.part_o, w.part_ml, kpad / TM_RPS, (int)(rpc / TM_RPS),      \
                             n_groups, B, G, layer_begin, w.segstride, out, lse));                \
  }
  ATK(64, 1) ATK(64, 2) ATK(64, 4) ATK(64, 8) ATK(128, 1) ATK(128, 2) ATK(128, 4) ATK(128, 8)
#undef ATK
  return SPC_E_UNSUPPORTED;
}

extern "C" int spc_attn_merge(const float* o_parts, const float* lse_parts, int P, int n, int D,
                              float* out, float* lse_out, spc_stream_t stream) {
  if (!o_parts || !lse_parts || !out) return SPC_E_NULL;
  if (P < 1 || n < 1 || D < 1) return SPC_E_SHAPE;
  return launched(launch_k(merge_kernel, dim3(n), dim3(128), 0, as_stream(stream), o_parts,
                           lse_parts, P, n, D, out, lse_out));
}

// Debug only (not part of include/spc.h): route the attention kernel's per-chunk
// %globaltimer trace of CTA 0 into `buf` (device, >= 256*4 uint64), NULL = off.
extern "C" int spc_debug_set_trace(void* buf) {
  unsigned long long* p = (unsigned long long*)buf;
  cudaError_t e = cudaMemcpyToSymbol(spc::g_trace, &p, sizeof(p));
  return e == cudaSuccess ? SPC_OK : SPC_E_CUDA;
}
