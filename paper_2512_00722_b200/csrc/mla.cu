// mla.cu — spc_mla_sparse_attn: MLA sparse decode attention over the selected latent rows
// (SURVEY §8(f) NEXT-3).
//
// Paper §4.3 (Fig. 5(e)): "MLA caches a lower-dimensional latent representation c ...
// Since MLA does not reduce the number of attention heads, our retrieval remains similar to
// that in MHA.  The primary difference lies that only the selected c cache is subjected to the
// increase in dimension."  The paper expands the selected rows, K_j = W_UK c_j and
// V_j = W_UV c_j, then attends.  Here the expansion is ABSORBED into the query and the output
// (the same mathematics, R29): per (request, head)
//   q_abs = [W_UK^T q_nope | q_pe]                            (mla_absorb_kernel, fp32)
//   s_j   = scale * q_abs . [c_j | kpe_j]   for j in the head's selection
//   o_c   = sum_j softmax(s)_j c_j                            (mla_attn_kernel, split-K)
//   o     = W_UV o_c,   lse = logsumexp(s)
// so each selected latent row (576 bf16 = 1152 B) is read once per head and nothing of
// size k x H x (DN + DV) is materialised.  HBM-bound: the selected latent rows dominate.
// All L layers run in one launch of each kernel (grid.z = layer; the selection is
// layer-independent), per-layer caches and weights through pointer tables.
#include <algorithm>

#include "common.cuh"

namespace spc {
namespace {

constexpr int ML_DC = 512, ML_DR = 64, ML_W = ML_DC + ML_DR;
#ifndef SPC_ML_ROWS
#define SPC_ML_ROWS 1024
#endif
constexpr int ML_ROWS = SPC_ML_ROWS;  // selected rows per CTA (split-K)
constexpr int ML_WARPS = 8;
#ifndef SPC_ML_UNR
#define SPC_ML_UNR 4
#endif
constexpr int ML_UNR = SPC_ML_UNR;  // rows in flight per warp

struct MlaWs {
  float* qabs;      // [L][B*H][576]
  float* part_o;    // [L][B*H][nsplit][512]
  float* part_ml;   // [L][B*H][nsplit][2]
  unsigned* cnt;    // [L][B*H]
  int nsplit;
  size_t bytes;
};
MlaWs mla_ws_layout(void* ws, int L, int B, int H, int k) {
  MlaWs w;
  const size_t bh = (size_t)L * B * H;
  w.nsplit = (k + ML_ROWS - 1) / ML_ROWS;
  uint8_t* p = (uint8_t*)ws;
  size_t off = 0;
  auto take = [&](size_t n) {
    uint8_t* r = p + off;
    off = align_up(off + n, 256);
    return r;
  };
  w.qabs = (float*)take(sizeof(float) * bh * ML_W);
  w.part_o = (float*)take(sizeof(float) * bh * w.nsplit * ML_DC);
  w.part_ml = (float*)take(sizeof(float) * bh * w.nsplit * 2);
  w.cnt = (unsigned*)take(sizeof(unsigned) * bh);
  w.bytes = off;
  return w;
}

// q_abs[e] = sum_n q_nope[n] W_UK[h][n][e] (e < 512), q_abs[512 + r] = q_pe[r]
// grid (4 slices of 128 dims, B*H, L), 64 threads: two adjacent outputs per thread
// (bf16x2 loads of W_UK rows), 16 rows of W_UK in flight
__global__ void __launch_bounds__(64) mla_absorb_kernel(const uint16_t* __restrict__ q,
                                                        const void* const* __restrict__ w_uk_l,
                                                        int BH, int H, int DN,
                                                        float* __restrict__ qabs) {
  spc_pdl_entry();
  const int bh = blockIdx.y, h = bh % H, l = blockIdx.z, tid = threadIdx.x;
  const uint16_t* qq = q + ((size_t)l * BH + bh) * (DN + ML_DR);
  const uint32_t* W = (const uint32_t*)((const uint16_t*)w_uk_l[l] + (size_t)h * DN * ML_DC);
  float* qa = qabs + ((size_t)l * BH + bh) * ML_W;
  const int e2 = blockIdx.x * 64 + tid;  // pair of outputs 2 e2, 2 e2 + 1
  float a0 = 0.f, a1 = 0.f;
  for (int n0 = 0; n0 < DN; n0 += 16) {
    uint32_t wv[16];
    uint16_t qv[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int n = min(n0 + u, DN - 1);
      wv[u] = __ldg(W + (size_t)n * (ML_DC / 2) + e2);
      qv[u] = qq[n];
    }
#pragma unroll
    for (int u = 0; u < 16; ++u)
      if (n0 + u < DN) {
        const float qn = __uint_as_float((uint32_t)qv[u] << 16);
        a0 = fmaf(qn, bf16lo(wv[u]), a0);
        a1 = fmaf(qn, bf16hi(wv[u]), a1);
      }
  }
  qa[2 * e2] = a0;
  qa[2 * e2 + 1] = a1;
  if (blockIdx.x == 0) qa[ML_DC + tid] = __uint_as_float((uint32_t)qq[DN + tid] << 16);
}

__global__ void __launch_bounds__(ML_WARPS * 32) mla_attn_kernel(
    const void* const* __restrict__ cache_l, const void* const* __restrict__ w_uv_l,
    const int32_t* __restrict__ idx, const int32_t* __restrict__ count, int BH, int H, int Smax,
    int k, int DV, float scale_log2, MlaWs ws, float* __restrict__ out, float* __restrict__ lse) {
  spc_pdl_entry();
  __shared__ float s_o[ML_WARPS][ML_DC];
  __shared__ float s_ml[ML_WARPS][2];
  __shared__ float s_fin[ML_DC];
  __shared__ int flag;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int bhs = blockIdx.y, b = bhs / H, h = bhs % H, split = blockIdx.x, lyr = blockIdx.z;
  const int bh = lyr * BH + bhs;  // (layer, b, h) slot of the workspace and the outputs
  const int n = min(max(count[bhs], 0), k);
  const int r0 = split * ML_ROWS, r1 = min(n, r0 + ML_ROWS);
  const uint16_t* cb = (const uint16_t*)cache_l[lyr] + (size_t)b * Smax * ML_W;
  const int32_t* rows = idx + (size_t)bhs * k;
  // this lane's slice of q_abs: c dims [16 lane, +16), rope dims [2 lane, +2)
  float qa[16], qp[2];
  const float* qs = ws.qabs + (size_t)bh * ML_W;
#pragma unroll
  for (int i = 0; i < 16; ++i) qa[i] = qs[16 * lane + i];
  qp[0] = qs[ML_DC + 2 * lane];
  qp[1] = qs[ML_DC + 2 * lane + 1];
  float m = -INFINITY, l = 0.f, o[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) o[i] = 0.f;
  for (int rb = r0 + warp * ML_UNR; rb < r1; rb += ML_WARPS * ML_UNR) {
    uint4 c0[ML_UNR], c1[ML_UNR];
    uint32_t pe[ML_UNR];
#pragma unroll
    for (int u = 0; u < ML_UNR; ++u) {
      if (rb + u < r1) {
        const uint16_t* row = cb + (size_t)rows[rb + u] * ML_W;
        c0[u] = __ldcs(reinterpret_cast<const uint4*>(row) + 2 * lane);
        c1[u] = __ldcs(reinterpret_cast<const uint4*>(row) + 2 * lane + 1);
        pe[u] = __ldcs(reinterpret_cast<const uint32_t*>(row + ML_DC) + lane);
      }
    }
#pragma unroll
    for (int u = 0; u < ML_UNR; ++u) {
      if (rb + u >= r1) break;
      float cv[16];
      const uint32_t* p0 = &c0[u].x;
      const uint32_t* p1 = &c1[u].x;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        cv[2 * e] = bf16lo(p0[e]);
        cv[2 * e + 1] = bf16hi(p0[e]);
        cv[8 + 2 * e] = bf16lo(p1[e]);
        cv[8 + 2 * e + 1] = bf16hi(p1[e]);
      }
      float s = fmaf(qp[0], bf16lo(pe[u]), qp[1] * bf16hi(pe[u]));
#pragma unroll
      for (int i = 0; i < 16; ++i) s = fmaf(qa[i], cv[i], s);
      s = warp_sum(s) * scale_log2;  // log2 units
      const float mn = fmaxf(m, s);
      const float corr = exp2f(m - mn), w = exp2f(s - mn);
      l = l * corr + w;
#pragma unroll
      for (int i = 0; i < 16; ++i) o[i] = fmaf(w, cv[i], o[i] * corr);
      m = mn;
    }
  }
  // ---- CTA partial: combine the 8 warps (log2 units)
#pragma unroll
  for (int i = 0; i < 16; ++i) s_o[warp][16 * lane + i] = o[i];
  if (lane == 0) {
    s_ml[warp][0] = m;
    s_ml[warp][1] = l;
  }
  __syncthreads();
  float M = -INFINITY;
#pragma unroll
  for (int w = 0; w < ML_WARPS; ++w) M = fmaxf(M, s_ml[w][0]);
  float L = 0.f;
#pragma unroll
  for (int w = 0; w < ML_WARPS; ++w)
    if (s_ml[w][0] != -INFINITY) L += exp2f(s_ml[w][0] - M) * s_ml[w][1];
  float* po = ws.part_o + ((size_t)bh * ws.nsplit + split) * ML_DC;
  for (int d = tid; d < ML_DC; d += ML_WARPS * 32) {
    float v = 0.f;
#pragma unroll
    for (int w = 0; w < ML_WARPS; ++w)
      if (s_ml[w][0] != -INFINITY) v += exp2f(s_ml[w][0] - M) * s_o[w][d];
    po[d] = v;
  }
  if (tid == 0) {
    ws.part_ml[((size_t)bh * ws.nsplit + split) * 2] = M;
    ws.part_ml[((size_t)bh * ws.nsplit + split) * 2 + 1] = L;
  }
  // ---- the last CTA of (b, h) merges the splits (O12) and projects with W_UV
  if (!last_block_ticket(&ws.cnt[bh], gridDim.x, &flag)) return;
  const float* pml = ws.part_ml + (size_t)bh * ws.nsplit * 2;
  float GM = -INFINITY;
  for (int s = 0; s < (int)gridDim.x; ++s) GM = fmaxf(GM, __ldcg(pml + 2 * s));
  float GL = 0.f;
  for (int s = 0; s < (int)gridDim.x; ++s) {
    const float ms = __ldcg(pml + 2 * s);
    if (ms != -INFINITY) GL += exp2f(ms - GM) * __ldcg(pml + 2 * s + 1);
  }
  const float inv = GL > 0.f ? 1.f / GL : 0.f;
  for (int d = tid; d < ML_DC; d += ML_WARPS * 32) {
    float v = 0.f;
    for (int s = 0; s < (int)gridDim.x; ++s) {
      const float ms = __ldcg(pml + 2 * s);
      if (ms != -INFINITY)
        v += exp2f(ms - GM) * __ldcg(ws.part_o + ((size_t)bh * ws.nsplit + s) * ML_DC + d);
    }
    s_fin[d] = v * inv;
  }
  __syncthreads();
  const uint16_t* Wv = (const uint16_t*)w_uv_l[lyr] + (size_t)h * DV * ML_DC;
  for (int a0 = warp * 4; a0 < DV; a0 += ML_WARPS * 4) {  // o[a] = W_UV[h][a] . o_c
    uint4 wr[4][2];  // 4 output rows in flight: 16 bf16 per lane each
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int a = min(a0 + t, DV - 1);
      const uint4* rowp = reinterpret_cast<const uint4*>(Wv + (size_t)a * ML_DC) + 2 * lane;
      wr[t][0] = __ldg(rowp);
      wr[t][1] = __ldg(rowp + 1);
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const uint32_t* p0 = &wr[t][0].x;
      const uint32_t* p1 = &wr[t][1].x;
      float acc = 0.f;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        acc = fmaf(bf16lo(p0[e]), s_fin[16 * lane + 2 * e], acc);
        acc = fmaf(bf16hi(p0[e]), s_fin[16 * lane + 2 * e + 1], acc);
        acc = fmaf(bf16lo(p1[e]), s_fin[16 * lane + 8 + 2 * e], acc);
        acc = fmaf(bf16hi(p1[e]), s_fin[16 * lane + 8 + 2 * e + 1], acc);
      }
      acc = warp_sum(acc);
      if (lane == 0 && a0 + t < DV) out[(size_t)bh * DV + a0 + t] = acc;
    }
  }
  if (lse && tid == 0) lse[bh] = GL > 0.f ? (GM + log2f(GL)) * 0.6931471805599453f : -INFINITY;
}

}  // namespace
}  // namespace spc

using namespace spc;

extern "C" size_t spc_mla_workspace(int L, int B, int H, int k) {
  if (L <= 0 || B <= 0 || H <= 0 || k <= 0) return 0;
  return mla_ws_layout(nullptr, L, B, H, k).bytes;
}

extern "C" int spc_mla_sparse_attn(const void* q, const void* const* cache, const void* const* w_uk,
                                   const void* const* w_uv, const int32_t* idx,
                                   const int32_t* count, int L, int B, int H, int Smax, int k,
                                   int DC, int DR, int DN, int DV, float scale, float* out,
                                   float* lse, void* ws, size_t ws_bytes, spc_stream_t stream) {
  if (!q || !cache || !w_uk || !w_uv || !idx || !count || !out || !ws) return SPC_E_NULL;
  if (L <= 0 || B <= 0 || H <= 0 || Smax <= 0 || DN <= 0 || DV <= 0) return SPC_E_SHAPE;
  if (k < 1 || k > SPC_MAX_K) return SPC_E_BUDGET;
  if (DC != ML_DC || DR != ML_DR || DN > 512 || DV > 1024) return SPC_E_UNSUPPORTED;
  if (ws_bytes < spc_mla_workspace(L, B, H, k)) return SPC_E_WORKSPACE;
  MlaWs w = mla_ws_layout(ws, L, B, H, k);
  cudaStream_t st = as_stream(stream);
  SPC_TRY(launched(launch_k(mla_absorb_kernel, dim3(ML_DC / 128, B * H, L), dim3(64), 0, st,
                            (const uint16_t*)q, w_uk, B * H, H, DN, w.qabs)));
  return launched(launch_k(mla_attn_kernel, dim3(w.nsplit, B * H, L), dim3(ML_WARPS * 32), 0, st,
                           cache, w_uv, idx, count, B * H, H, Smax, k, DV,
                           scale * 1.4426950408889634f, w, out, lse));
}
