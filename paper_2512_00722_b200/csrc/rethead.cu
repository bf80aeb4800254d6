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
//   xn  = bf16(w * bf16(x * r)),  r = 1 / sqrt(mean(x^2) + eps)   (HF Llama RMSNorm)
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

constexpr int RH_WARPS = 8;
constexpr int RH_UNR = 8;  // 16-byte weight chunks per row in flight per lane

__device__ __forceinline__ uint16_t f32_to_bf16_rn(float f) {
  const __nv_bfloat16 h = __float2bfloat16_rn(f);
  return *reinterpret_cast<const uint16_t*>(&h);
}
__device__ __forceinline__ float bf16_to_f32(uint16_t h) {
  return __uint_as_float((uint32_t)h << 16);
}

template <int BT>
__global__ void __launch_bounds__(RH_WARPS * 32) rethead_kernel(
    const int32_t* __restrict__ token, const uint16_t* __restrict__ emb, int H,
    const uint16_t* __restrict__ norm_w, float eps, const uint16_t* __restrict__ w_qk,
    const float* __restrict__ inv_freq, float mscale, const int32_t* __restrict__ pos, int B,
    int Hq, int G, int D, int Smax, uint16_t* __restrict__ q_out, uint16_t* __restrict__ kr,
    int32_t* __restrict__ seq_len_out, uint16_t* __restrict__ x_out) {
  spc_pdl_entry();
  extern __shared__ __align__(16) uint8_t rh_smem[];
  uint16_t* xs = reinterpret_cast<uint16_t*>(rh_smem);  // [B][H] normalised inputs
  __shared__ float red[RH_WARPS];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // ---- RMSNorm of the B embedding rows (every CTA; the rows are L2-resident)
  for (int b = 0; b < B; ++b) {
    const uint16_t* x = emb + (size_t)token[b] * H;
    float ss = 0.f;
    for (int h = tid; h < H; h += RH_WARPS * 32) {
      const float v = bf16_to_f32(x[h]);
      ss = fmaf(v, v, ss);
    }
    ss = warp_sum(ss);
    if (lane == 0) red[warp] = ss;
    __syncthreads();
    float tot = 0.f;
#pragma unroll
    for (int w = 0; w < RH_WARPS; ++w) tot += red[w];
    const float r = 1.0f / sqrtf(tot / (float)H + eps);
    for (int h = tid; h < H; h += RH_WARPS * 32) {
      const float t = bf16_to_f32(f32_to_bf16_rn(bf16_to_f32(x[h]) * r));
      const float wv = norm_w ? bf16_to_f32(norm_w[h]) : 1.0f;
      const uint16_t o = f32_to_bf16_rn(wv * t);
      xs[(size_t)b * H + h] = o;
      if (x_out && blockIdx.x == 0) x_out[(size_t)b * H + h] = o;
    }
    __syncthreads();  // red[] is reused by the next request
  }
  if (seq_len_out && blockIdx.x == 0 && tid < B) seq_len_out[tid] = pos[tid] + 1;

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
        const int pb = pos[b];
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

}  // namespace
}  // namespace spc

using namespace spc;

extern "C" int spc_rethead_qk(const int32_t* token, const void* emb, int V, int H,
                              const void* norm_w, float eps, const void* w_qk,
                              const float* inv_freq, float mscale, const int32_t* pos, int B,
                              int Hq, int G, int D, int Smax, void* q_out, void* kr,
                              int32_t* seq_len_out, void* x_out, spc_stream_t stream) {
  if (!token || !emb || !w_qk || !inv_freq || !pos || !q_out || !kr) return SPC_E_NULL;
  if (V <= 0 || H <= 0 || B <= 0 || Hq <= 0 || G <= 0 || Hq % G || Smax <= 0) return SPC_E_SHAPE;
  if (!(D == 64 || D == 128) || H % 8 || H > 16384 || B > 16) return SPC_E_UNSUPPORTED;
  if (((uintptr_t)emb & 15) || ((uintptr_t)w_qk & 15)) return SPC_E_RANGE;
  const size_t smem = (size_t)B * H * 2;
  if (smem > 200 * 1024) return SPC_E_UNSUPPORTED;
  const int npairs = (Hq + G) * (D / 2);
  const int ncta = std::max(1, std::min(2 * num_sms(), (npairs + RH_WARPS - 1) / RH_WARPS));
  cudaStream_t st = as_stream(stream);
#define RH(BT)                                                                                    \
  {                                                                                               \
    static int attr_bytes = 0;                                                                    \
    if ((int)smem > attr_bytes) {                                                                 \
      cudaFuncSetAttribute(rethead_kernel<BT>, cudaFuncAttributeMaxDynamicSharedMemorySize,       \
                           (int)std::max<size_t>(smem, 48 * 1024));                               \
      attr_bytes = (int)std::max<size_t>(smem, 48 * 1024);                                        \
    }                                                                                             \
    return launched(launch_k(rethead_kernel<BT>, dim3(ncta), dim3(RH_WARPS * 32), smem, st,      \
                             token, (const uint16_t*)emb, H, (const uint16_t*)norm_w, eps,        \
                             (const uint16_t*)w_qk, inv_freq, mscale, pos, B, Hq, G, D, Smax,     \
                             (uint16_t*)q_out, (uint16_t*)kr, seq_len_out, (uint16_t*)x_out));    \
  }
  if (B == 1) RH(1)
  if (B <= 4) RH(4)
  RH(16)
#undef RH
}
