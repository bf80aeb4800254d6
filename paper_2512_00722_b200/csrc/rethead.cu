// rethead.cu — spc_rethead_qk: the retrieval head's per-step front-end (SURVEY §8(f)
// NEXT-1), the calls that precede spc_score on the critical path.
//
// Paper §4.3: "This retrieval head retains the essential components of DLM ...
// the embedding module and the QK projection weights ... we enable it to process long
// context using the training-free method provided by YaRN ... the retrieval head
// maintains a full Key (K) cache and calculates attention weights after the QK
// projection"; "the weight of the retrieval head ... is only about 60MB".
// SPEC run_retrieval_head: the new key is appended at position = cache
// length, then scored.
//
// Per request b (DESIGN.md §3 R22-R24):
//   x   = emb[token[b]]                                   (bf16 row of H)
//   xn  = bf16(w * bf16(x * r)),  r = 1 / sqrt(mean(x^2) + eps)   (HF Llama RMSNorm; the sum
//         of squares an exact fixed-point integer sum, R22, so xn is bit-exact)
//   pre = W_qk xn  (fp32 accumulation; rows [0, Hq*D) = W_q, [Hq*D, (Hq+G)*D) = W_k)
//   RoPE on the pairs (i, i + D/2) of every head (rotate_half convention), angle
//   a = fl32(pos[b] * inv_freq[i]), c = cos(a) * mscale, s = sin(a) * mscale
//   (inv_freq / mscale: the caller's YaRN-scaled table, rope.yarn_inv_freq)
//   q_out[b][h] = bf16(rotated q head h);  kr[b][g][pos[b]] = bf16(rotated k head g).
//
// HBM-bound GEMV over the (Hq+G)*D x H bf16 weights (config-B shape: 5120 x 4096 =
// 40 MiB): every CTA first normalises the B input rows into shared memory (8 KiB per
// request); each warp then owns row PAIRS (i, i + D/2) of one head -- the two rows the
// rotation mixes -- and streams them with 16-byte loads, 8 chunks per row in flight per
// lane, dotting each chunk with all B inputs.  After a warp reduction the lanes b < B
// rotate and store request b's two outputs.
#include <algorithm>

#include "common.cuh"

namespace spc {
namespace {

// R22: the RMSNorm reciprocal r = 1 / sqrt(mean(x^2) + eps), determinised so
// the oracle reproduces it bit for bit: e = ilogb(max |x|); F = sum_h trunc(x_h^2 2^(46-2e))
// as int64 (every term exact in fp64 and < 2^48, so the integer sum is exact and
// order-free); mean = RN64(RN64(F) 2^(2e-46) / H); r = RN32(RN64(1 / RN64(sqrt(mean + eps)))).
__device__ __forceinline__ double rms_term_scale(float mx) {
  return mx > 0.f ? ldexp(1.0, 46 - 2 * ilogbf(mx)) : 1.0;
}
__device__ __forceinline__ long long rms_term(float v, double sc) {
  return __double2ll_rz(__dmul_rn(__dmul_rn((double)v, (double)v), sc));
}
__device__ __forceinline__ float rms_r(long long F, float mx, int H, float eps) {
  const double ss = mx > 0.f ? ldexp(__ll2double_rn(F), 2 * ilogbf(mx) - 46) : 0.0;
  const double mean = __ddiv_rn(ss, (double)H);
  return __double2float_rn(__ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(mean, (double)eps))));
}

constexpr int RH_WARPS = 8;
#ifndef SPC_RH_UNR
#define SPC_RH_UNR 4
#endif
#ifndef SPC_RH_CPS
#define SPC_RH_CPS 3
#endif
constexpr int RH_UNR = SPC_RH_UNR;  // 16-byte weight chunks per row in flight per lane
constexpr int RH_CPS = SPC_RH_CPS;  // CTAs per SM of the B <= 4 kernel

__device__ __forceinline__ uint16_t f32_to_bf16_rn(float f) {
  const __nv_bfloat16 h = __float2bfloat16_rn(f);
  return *reinterpret_cast<const uint16_t*>(&h);
}
__device__ __forceinline__ float bf16_to_f32(uint16_t h) {
  return __uint_as_float((uint32_t)h << 16);
}

template <int BT>
__global__ void __launch_bounds__(RH_WARPS * 32, RH_CPS) rethead_kernel(
    const int32_t* __restrict__ token, const uint16_t* __restrict__ emb, int H,
    const uint16_t* __restrict__ norm_w, float eps, const uint16_t* __restrict__ w_qk,
    const float* __restrict__ inv_freq, float mscale, const int32_t* __restrict__ pos, int B,
    int Hq, int G, int D, int Smax, uint16_t* __restrict__ q_out, uint16_t* __restrict__ kr,
    int32_t* __restrict__ seq_len_out, uint16_t* __restrict__ x_out) {
  // the weights are static: before the PDL wait and the RMSNorm prologue, every warp asks for
  // its row pairs in L2 (a hint: the loads below read them through L2), so the 40 MiB stream
  // runs while the embedding rows are normalised
  {
    const int w = (int)threadIdx.x >> 5;
    const int half_ = D / 2, npairs_ = (Hq + G) * half_;
    if ((threadIdx.x & 31) == 0)
      for (int p = blockIdx.x * RH_WARPS + w; p < npairs_; p += gridDim.x * RH_WARPS) {
        const int hh = p / half_, i = p - hh * half_;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(w_qk + ((size_t)hh * D + i) * H),
                     "r"(H * 2)
                     : "memory");
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                         w_qk + ((size_t)hh * D + i + half_) * H),
                     "r"(H * 2)
                     : "memory");
      }
  }
  spc_pdl_entry();
  extern __shared__ __align__(16) uint8_t rh_smem[];
  uint16_t* xs = reinterpret_cast<uint16_t*>(rh_smem);  // [B][H] normalised inputs
  __shared__ float red[RH_WARPS];
  __shared__ long long redl[RH_WARPS];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // ---- RMSNorm of the B embedding rows (every CTA; the rows are L2-resident)
  for (int b = 0; b < B; ++b) {
    const uint16_t* x = emb + (size_t)token[b] * H;
    float mx = 0.f;  // max |x| (exact, order-free)
    for (int h = tid; h < H; h += RH_WARPS * 32) mx = fmaxf(mx, fabsf(bf16_to_f32(x[h])));
    mx = warp_max(mx);
    if (lane == 0) red[warp] = mx;
    __syncthreads();
#pragma unroll
    for (int w = 0; w < RH_WARPS; ++w) mx = fmaxf(mx, red[w]);
    const double sc = rms_term_scale(mx);
    long long F = 0;
    for (int h = tid; h < H; h += RH_WARPS * 32) F += rms_term(bf16_to_f32(x[h]), sc);
    F = warp_sum_ll(F);
    if (lane == 0) redl[warp] = F;
    __syncthreads();
    F = 0;
#pragma unroll
    for (int w = 0; w < RH_WARPS; ++w) F += redl[w];
    const float r = rms_r(F, mx, H, eps);
    for (int h = tid; h < H; h += RH_WARPS * 32) {
      const float t = bf16_to_f32(f32_to_bf16_rn(bf16_to_f32(x[h]) * r));
      const float wv = norm_w ? bf16_to_f32(norm_w[h]) : 1.0f;
      const uint16_t o = f32_to_bf16_rn(wv * t);
      xs[(size_t)b * H + h] = o;
      if (x_out && blockIdx.x == 0) x_out[(size_t)b * H + h] = o;
    }
    __syncthreads();  // red[] is reused by the next request
  }
  if (pos && seq_len_out && blockIdx.x == 0 && tid < B) seq_len_out[tid] = pos[tid] + 1;

  // ---- row pairs (i, i + D/2) of head hh: warp-strided over the grid
  const int half = D / 2;
  const int npairs = (Hq + G) * half;
  const int nchunk = H / 8;  // 16-byte chunks per row
  const uint32_t xs_s = smem_u32(xs);
  for (int p = blockIdx.x * RH_WARPS + warp; p < npairs; p += gridDim.x * RH_WARPS) {
    const int hh = p / half, i = p - hh * half;
    const uint4* w0 = reinterpret_cast<const uint4*>(w_qk + ((size_t)hh * D + i) * H);
    const uint4* w1 = reinterpret_cast<const uint4*>(w_qk + ((size_t)hh * D + i + half) * H);
    float a0[BT], a1[BT];
#pragma unroll
    for (int b = 0; b < BT; ++b) a0[b] = a1[b] = 0.f;
    for (int c0 = lane; c0 < nchunk; c0 += 32 * RH_UNR) {
      uint4 v0[RH_UNR], v1[RH_UNR];
#pragma unroll
      for (int u = 0; u < RH_UNR; ++u) {
        const int c = c0 + 32 * u;
        if (c < nchunk) {
          v0[u] = __ldcs(w0 + c);
          v1[u] = __ldcs(w1 + c);
        }
      }
#pragma unroll
      for (int u = 0; u < RH_UNR; ++u) {
        const int c = c0 + 32 * u;
        if (c >= nchunk) break;
        const uint32_t* p0 = &v0[u].x;
        const uint32_t* p1 = &v1[u].x;
#pragma unroll
        for (int b = 0; b < BT; ++b) {
          if (b < B) {
            const uint4 xv = lds128(xs_s + (uint32_t)(((size_t)b * H + (size_t)c * 8) * 2));
            const uint32_t* px = &xv.x;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float xl = bf16lo(px[e]), xh = bf16hi(px[e]);
              a0[b] = fmaf(bf16lo(p0[e]), xl, a0[b]);
              a0[b] = fmaf(bf16hi(p0[e]), xh, a0[b]);
              a1[b] = fmaf(bf16lo(p1[e]), xl, a1[b]);
              a1[b] = fmaf(bf16hi(p1[e]), xh, a1[b]);
            }
          }
        }
      }
    }
#pragma unroll
    for (int b = 0; b < BT; ++b) {
      a0[b] = warp_sum(a0[b]);
      a1[b] = warp_sum(a1[b]);
    }
    // ---- RoPE (rotate_half pairs) and the bf16 stores: lane b handles request b
#pragma unroll
    for (int b = 0; b < BT; ++b) {
      if (lane == b && b < B) {
        const int pb = pos ? pos[b] : seq_len_out[b] - 1;  // pos NULL: seq_len counts the new token
        const float ang = (float)pb * inv_freq[i];
        float sn, cs;
        sincosf(ang, &sn, &cs);
        cs *= mscale;
        sn *= mscale;
        const float o0 = a0[b] * cs - a1[b] * sn;
        const float o1 = a1[b] * cs + a0[b] * sn;
        uint16_t* dst;
        if (hh < Hq) {
          dst = q_out + ((size_t)b * Hq + hh) * D;
        } else {
          dst = kr + (((size_t)b * G + (hh - Hq)) * Smax + pb) * D;
        }
        dst[i] = f32_to_bf16_rn(o0);
        dst[i + half] = f32_to_bf16_rn(o1);
      }
    }
  }
}

// ---- Batched variant (5 <= B <= 16): the projection is a skinny GEMM, [(Hq+G)*D x H] x
// [H x B], run on the tensor cores (mma.sync m16n8k16, bf16 in, fp32 accumulate).  An
// m-tile holds 8 RoPE pairs of one head: rows i0 + gid (the pair's first row) and
// i0 + D/2 + gid (its partner), so both rows a rotation mixes land in one lane's C
// fragment.  The A operand comes straight from global memory: lane (gid, tig) loads the
// 16-byte chunks tig + 4j of its two rows, and the k index inside every 16-wide MMA slice
// is permuted consistently for A and B (the dot product is order-free across slices, and
// each slice's 16 products are summed by the MMA), so no shared-memory staging or ldmatrix
// is needed for the weights.  Persistent CTAs of 8 warps: each CTA normalises the B rows
// once into shared memory; per m-tile each warp takes an H/8 slice and the 8 partial C
// fragments meet in shared memory; warp 0 rotates and stores.
constexpr int RM_WARPS = 8;
__device__ __forceinline__ void rh_mma(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                       uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
      "{%8, %9}, {%0, %1, %2, %3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int NT>  // n-tiles of 8 requests
__global__ void __launch_bounds__(RM_WARPS * 32, 1) rethead_mma_kernel(
    const int32_t* __restrict__ token, const uint16_t* __restrict__ emb, int H,
    const uint16_t* __restrict__ norm_w, float eps, const uint16_t* __restrict__ w_qk,
    const float* __restrict__ inv_freq, float mscale, const int32_t* __restrict__ pos, int B,
    int Hq, int G, int D, int Smax, uint16_t* __restrict__ q_out, uint16_t* __restrict__ kr,
    int32_t* __restrict__ seq_len_out, uint16_t* __restrict__ x_out) {
  spc_pdl_entry();
  extern __shared__ __align__(16) uint8_t rm_smem[];
  uint16_t* xs = reinterpret_cast<uint16_t*>(rm_smem);  // [8 NT][H] (rows >= B zero)
  __shared__ float red[RM_WARPS][NT][4][32];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int nchunk = H / 8;
  // ---- RMSNorm of the B rows (warp b, b + 8, ...); rows B..8NT-1 are zero
  for (int b = warp; b < 8 * NT; b += RM_WARPS) {
    uint4* dstrow = reinterpret_cast<uint4*>(xs + (size_t)b * H);
    if (b >= B) {
      for (int c = lane; c < nchunk; c += 32) dstrow[c] = make_uint4(0, 0, 0, 0);
      continue;
    }
    const uint4* x = reinterpret_cast<const uint4*>(emb + (size_t)token[b] * H);
    float mx = 0.f;  // R22: max |x|, then the exact fixed-point sum of squares
    for (int c = lane; c < nchunk; c += 32) {
      const uint4 v = __ldg(x + c);
      const uint32_t* pv = &v.x;
#pragma unroll
      for (int e = 0; e < 4; ++e) mx = fmaxf(mx, fmaxf(fabsf(bf16lo(pv[e])), fabsf(bf16hi(pv[e]))));
    }
    mx = warp_max(mx);
    const double sc = rms_term_scale(mx);
    long long F = 0;
    for (int c = lane; c < nchunk; c += 32) {
      const uint4 v = __ldg(x + c);
      const uint32_t* pv = &v.x;
#pragma unroll
      for (int e = 0; e < 4; ++e) F += rms_term(bf16lo(pv[e]), sc) + rms_term(bf16hi(pv[e]), sc);
    }
    F = warp_sum_ll(F);
    const float r = rms_r(F, mx, H, eps);
    for (int c = lane; c < nchunk; c += 32) {
      const uint4 v = __ldg(x + c);
      const uint4 wv = norm_w ? __ldg(reinterpret_cast<const uint4*>(norm_w) + c)
                              : make_uint4(0x3f803f80u, 0x3f803f80u, 0x3f803f80u, 0x3f803f80u);
      const uint32_t* pv = &v.x;
      const uint32_t* pw = &wv.x;
      uint32_t o[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float tl = bf16_to_f32(f32_to_bf16_rn(bf16lo(pv[e]) * r));
        const float th = bf16_to_f32(f32_to_bf16_rn(bf16hi(pv[e]) * r));
        o[e] = (uint32_t)f32_to_bf16_rn(bf16lo(pw[e]) * tl) |
               ((uint32_t)f32_to_bf16_rn(bf16hi(pw[e]) * th) << 16);
      }
      const uint4 ov = make_uint4(o[0], o[1], o[2], o[3]);
      dstrow[c] = ov;
      if (x_out && blockIdx.x == 0) reinterpret_cast<uint4*>(x_out + (size_t)b * H)[c] = ov;
    }
  }
  if (pos && seq_len_out && blockIdx.x == 0 && tid < B) seq_len_out[tid] = pos[tid] + 1;
  __syncthreads();

  const int half = D / 2;
  const int tiles = (Hq + G) * (half / 8);       // m-tiles: 8 pairs of one head
  const int wch = nchunk / RM_WARPS;              // chunks of this warp's H slice
  const uint32_t xs_s = smem_u32(xs);
  for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int hh = t / (half / 8), i0 = (t - hh * (half / 8)) * 8;
    const uint4* wlo = reinterpret_cast<const uint4*>(w_qk + ((size_t)hh * D + i0 + gid) * H);
    const uint4* whi = reinterpret_cast<const uint4*>(w_qk + ((size_t)hh * D + half + i0 + gid) * H);
    float c[NT][4];
#pragma unroll
    for (int n = 0; n < NT; ++n) c[n][0] = c[n][1] = c[n][2] = c[n][3] = 0.f;
    const int cbeg = warp * wch;
    for (int j0 = 0; j0 < wch; j0 += 32) {      // 8 groups of 4 lanes' chunks in flight
      uint4 alo[8], ahi[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int ch = cbeg + j0 + tig + 4 * u;
        if (j0 + tig + 4 * u < wch) {
          alo[u] = __ldcs(wlo + ch);
          ahi[u] = __ldcs(whi + ch);
        } else {
          alo[u] = ahi[u] = make_uint4(0, 0, 0, 0);
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int ch = cbeg + j0 + tig + 4 * u;
        if (j0 + 4 * u >= wch) break;
        const int chs = min(ch, nchunk - 1);
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          const uint4 xb = lds128(xs_s + (uint32_t)((((size_t)(n * 8 + gid)) * H + (size_t)chs * 8) * 2));
          const bool ok = j0 + tig + 4 * u < wch;
          // two MMA k-slices per 16-byte chunk: elements 0-3 then 4-7 (k permuted alike)
          rh_mma(c[n], alo[u].x, ahi[u].x, alo[u].y, ahi[u].y, ok ? xb.x : 0u, ok ? xb.y : 0u);
          rh_mma(c[n], alo[u].z, ahi[u].z, alo[u].w, ahi[u].w, ok ? xb.z : 0u, ok ? xb.w : 0u);
        }
      }
    }
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) red[warp][n][e][lane] = c[n][e];
    __syncthreads();
    if (warp == 0) {
      const int i = i0 + gid;
      const float inv = inv_freq[i];
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        float s[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float v = 0.f;
#pragma unroll
          for (int w = 0; w < RM_WARPS; ++w) v += red[w][n][e][lane];
          s[e] = v;
        }
#pragma unroll
        for (int col = 0; col < 2; ++col) {  // C columns 2 tig + col = request
          const int b = n * 8 + 2 * tig + col;
          if (b < B) {
            const float u = s[col], vv = s[2 + col];  // row gid: pair first, gid + 8: partner
            const int pb = pos ? pos[b] : seq_len_out[b] - 1;  // pos NULL: seq_len counts the new token
            float sn, cs;
            sincosf((float)pb * inv, &sn, &cs);
            cs *= mscale;
            sn *= mscale;
            uint16_t* dst = hh < Hq ? q_out + ((size_t)b * Hq + hh) * D
                                    : kr + (((size_t)b * G + (hh - Hq)) * Smax + pb) * D;
            dst[i] = f32_to_bf16_rn(u * cs - vv * sn);
            dst[i + half] = f32_to_bf16_rn(vv * cs + u * sn);
          }
        }
      }
    }
    __syncthreads();  // red[] is rewritten by the next tile
  }
}

}  // namespace
}  // namespace spc

using namespace spc;

extern "C" int spc_rethead_qk(const int32_t* token, const void* emb, int V, int H,
                              const void* norm_w, float eps, const void* w_qk,
                              const float* inv_freq, float mscale, const int32_t* pos, int B,
                              int Hq, int G, int D, int Smax, void* q_out, void* kr,
                              int32_t* seq_len_out, void* x_out, spc_stream_t stream) {
  if (!token || !emb || !w_qk || !inv_freq || (!pos && !seq_len_out) || !q_out || !kr)
    return SPC_E_NULL;
  if (V <= 0 || H <= 0 || B <= 0 || Hq <= 0 || G <= 0 || Hq % G || Smax <= 0) return SPC_E_SHAPE;
  if (!(D == 64 || D == 128) || H % 8 || H > 16384 || B > 16) return SPC_E_UNSUPPORTED;
  if (((uintptr_t)emb & 15) || ((uintptr_t)w_qk & 15)) return SPC_E_RANGE;
  const size_t smem = (size_t)B * H * 2;
  if (smem > 200 * 1024) return SPC_E_UNSUPPORTED;
  const int npairs = (Hq + G) * (D / 2);
  const int ncta = std::max(1, std::min(RH_CPS * num_sms(), (npairs + RH_WARPS - 1) / RH_WARPS));
  cudaStream_t st = as_stream(stream);
#define RH(BT)                                                                                    \
  {                                                                                               \
    SPC_TRY(smem_attr((const void*)rethead_kernel<BT>, 200 * 1024));                              \
    return launched(launch_k(rethead_kernel<BT>, dim3(ncta), dim3(RH_WARPS * 32), smem, st,      \
                             token, (const uint16_t*)emb, H, (const uint16_t*)norm_w, eps,        \
                             (const uint16_t*)w_qk, inv_freq, mscale, pos, B, Hq, G, D, Smax,     \
                             (uint16_t*)q_out, (uint16_t*)kr, seq_len_out, (uint16_t*)x_out));    \
  }
  if (B == 1) RH(1)
  if (B <= 4) RH(4)
  if (H % (8 * RM_WARPS) == 0 && (D / 2) % 8 == 0) {  // tensor-core batched path
    const int nt = B <= 8 ? 1 : 2;
    const size_t msm = (size_t)8 * nt * H * 2;
    if (msm <= 200 * 1024) {
      const int tiles = (Hq + G) * (D / 2 / 8);
      const int nct = std::max(1, std::min(num_sms(), tiles));
#define RM(NT)                                                                                    \
  {                                                                                               \
    SPC_TRY(smem_attr((const void*)rethead_mma_kernel<NT>, 200 * 1024));                          \
    return launched(launch_k(rethead_mma_kernel<NT>, dim3(nct), dim3(RM_WARPS * 32), msm, st,    \
                             token, (const uint16_t*)emb, H, (const uint16_t*)norm_w, eps,        \
                             (const uint16_t*)w_qk, inv_freq, mscale, pos, B, Hq, G, D, Smax,     \
                             (uint16_t*)q_out, (uint16_t*)kr, seq_len_out, (uint16_t*)x_out));    \
  }
      if (nt == 1) RM(1)
      RM(2)
#undef RM
    }
  }
  RH(16)
#undef RH
}
