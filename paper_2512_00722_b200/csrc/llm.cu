// llm.cu — the LLM's per-layer decode operations around the sparse attention (SURVEY §8(f)
// NEXT-4): the elementwise parts of a Llama-style decoder layer (RMSNorm with the residual
// add, RoPE + KV-cache append, SwiGLU, fp32 -> bf16), so that one decode step can run end
// to end -- the retrieval head and selection once, then every layer's dense compute
// (projections on the tensor cores through cuBLAS: plain library GEMMs) with the selected-
// row attention of libspc, the elastic KV prefetch of the next layers overlapping it on a
// side stream (Fig. 3; "concurrent execution of computation and KV cache
// prefetching").  Random-init weights (accuracy is out of scope).
//
// All kernels: one CTA per request row (B rows), fp32 arithmetic, bf16 storage, launched
// with PDL like the rest of libspc.
#include "common.cuh"

namespace spc {
namespace {

constexpr int LL_T = 256;

__device__ __forceinline__ float bf(uint16_t h) { return __uint_as_float((uint32_t)h << 16); }
__device__ __forceinline__ uint16_t tobf(float f) {
  uint32_t u = __float_as_uint(f);
  if ((u & 0x7FFFFFFFu) > 0x7F800000u) return 0x7FC0u;  // NaN (canonical, as torch)
  u += 0x7FFFu + ((u >> 16) & 1u);  // RN-even
  return (uint16_t)(u >> 16);
}

// h[b] += delta[b] (if delta != NULL; delta bf16), then xn[b] = bf16(w * bf16(h * r)),
// r = 1 / sqrt(mean(h^2) + eps) (the HF Llama RMSNorm two-rounding form).  h is the fp32
// residual stream.  One CTA of NR_T threads per row; the row is held in registers (H <=
// NR_T * 4 * NR_V, float4 / 8-byte bf16x4 accesses when H % 4 == 0), so h is read once.
constexpr int NR_T = 1024, NR_V = 4;
__global__ void __launch_bounds__(NR_T) add_rmsnorm_kernel(float* __restrict__ h,
                                                           const uint16_t* __restrict__ delta,
                                                           const uint16_t* __restrict__ w, int H,
                                                           float eps, uint16_t* __restrict__ xn) {
  spc_pdl_entry();
  __shared__ float red[NR_T / 32];
  const int b = blockIdx.x;
  float* hb = h + (size_t)b * H;
  float4 v[NR_V];
  float ss = 0.f;
  const int H4 = H / 4;
#pragma unroll
  for (int j = 0; j < NR_V; ++j) {
    const int i = threadIdx.x + j * NR_T;
    if (i < H4) {
      float4 x = reinterpret_cast<const float4*>(hb)[i];
      if (delta) {
        const uint2 d = reinterpret_cast<const uint2*>(delta + (size_t)b * H)[i];
        x.x += bf(d.x & 0xFFFFu);
        x.y += bf(d.x >> 16);
        x.z += bf(d.y & 0xFFFFu);
        x.w += bf(d.y >> 16);
        reinterpret_cast<float4*>(hb)[i] = x;
      }
      v[j] = x;
      ss = fmaf(x.x, x.x, fmaf(x.y, x.y, fmaf(x.z, x.z, fmaf(x.w, x.w, ss))));
    }
  }
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < NR_T / 32; ++i) t += red[i];
  const float r = rsqrtf(t / (float)H + eps);
#pragma unroll
  for (int j = 0; j < NR_V; ++j) {
    const int i = threadIdx.x + j * NR_T;
    if (i < H4) {
      const uint2 wv = reinterpret_cast<const uint2*>(w)[i];
      const uint32_t o0 = tobf(bf(wv.x & 0xFFFFu) * bf(tobf(v[j].x * r)));
      const uint32_t o1 = tobf(bf(wv.x >> 16) * bf(tobf(v[j].y * r)));
      const uint32_t o2 = tobf(bf(wv.y & 0xFFFFu) * bf(tobf(v[j].z * r)));
      const uint32_t o3 = tobf(bf(wv.y >> 16) * bf(tobf(v[j].w * r)));
      reinterpret_cast<uint2*>(xn + (size_t)b * H)[i] = make_uint2(o0 | (o1 << 16), o2 | (o3 << 16));
    }
  }
}

// qkv [B][(Hq + 2G) D] bf16 (the fused projection) -> q_out [B][Hq][D] bf16 rotated, and
// the rotated key / the value of the new token (position p = seq_len[b] - 1) written at row
// p of the layer's caches k_cache / v_cache [B][G][rows][D] (device or mapped host memory).
// With slot_tok (SLOTS mode) they are also written into the budget slot that holds token p
// (slot_tok [B][G][k], the slot map after spc_elastic_diff), so the attention sees the new
// token without a gather of it.  RoPE: rotate_half pairs (i, i + D/2), angle
// fl32(p * inv_freq[i]).
constexpr int RA_T = 64;  // = D/2 for D = 128; D = 64 uses half the threads
__global__ void __launch_bounds__(RA_T) rope_append_kernel(
    const uint16_t* __restrict__ qkv, const float* __restrict__ inv_freq,
    const int32_t* __restrict__ seq_len, int Hq, int G, int D, int rows,
    uint16_t* __restrict__ q_out, uint16_t* __restrict__ k_cache, uint16_t* __restrict__ v_cache,
    const int32_t* __restrict__ slot_tok, int k, uint16_t* __restrict__ k_buf,
    uint16_t* __restrict__ v_buf) {
  spc_pdl_entry();
  __shared__ int slot;
  const int hh = blockIdx.x, b = blockIdx.y, half = D / 2;  // one CTA per (head, request)
  const int p = seq_len[b] - 1;
  SPC_DCHECK(p >= 0 && p < rows, SPC_E_RANGE);
  if (p < 0 || p >= rows) return;
  const uint16_t* x = qkv + ((size_t)b * (Hq + 2 * G) + hh) * D;
  if (hh < Hq + G) {  // a query or key head: rotate the pair (i, i + D/2)
    uint16_t o0 = 0, o1 = 0;
    const int i = threadIdx.x;
    if (i < half) {
      float sn, cs;
      sincosf((float)p * inv_freq[i], &sn, &cs);
      const float u = bf(x[i]), v = bf(x[i + half]);
      o0 = tobf(u * cs - v * sn);
      o1 = tobf(v * cs + u * sn);
    }
    if (hh < Hq) {
      if (i < half) {
        q_out[((size_t)b * Hq + hh) * D + i] = o0;
        q_out[((size_t)b * Hq + hh) * D + i + half] = o1;
      }
      return;
    }
    const int g = hh - Hq;
    if (i < half) {
      uint16_t* kr = k_cache + (((size_t)b * G + g) * rows + p) * D;
      kr[i] = o0;
      kr[i + half] = o1;
    }
    if (!slot_tok) return;
    if (threadIdx.x == 0) slot = -1;
    __syncthreads();
    const int4* st = reinterpret_cast<const int4*>(slot_tok + ((size_t)b * G + g) * k);
    if ((k & 3) == 0) {
      for (int e = threadIdx.x; e < k / 4; e += RA_T) {
        const int4 t = st[e];
        if (t.x == p) slot = 4 * e;
        if (t.y == p) slot = 4 * e + 1;
        if (t.z == p) slot = 4 * e + 2;
        if (t.w == p) slot = 4 * e + 3;
      }
    } else {
      for (int e = threadIdx.x; e < k; e += RA_T)
        if (slot_tok[((size_t)b * G + g) * k + e] == p) slot = e;
    }
    __syncthreads();
    if (slot >= 0 && i < half) {
      uint16_t* kb = k_buf + (((size_t)b * G + g) * k + slot) * D;
      kb[i] = o0;
      kb[i + half] = o1;
    }
    return;
  }
  // a value head: copied
  const int g = hh - Hq - G;
  for (int d = threadIdx.x; d < D; d += RA_T)
    v_cache[(((size_t)b * G + g) * rows + p) * D + d] = x[d];
  if (!slot_tok) return;
  if (threadIdx.x == 0) slot = -1;
  __syncthreads();
  for (int e = threadIdx.x; e < k; e += RA_T)
    if (slot_tok[((size_t)b * G + g) * k + e] == p) slot = e;
  __syncthreads();
  if (slot >= 0)
    for (int d = threadIdx.x; d < D; d += RA_T)
      v_buf[(((size_t)b * G + g) * k + slot) * D + d] = x[d];
}

// h[b] = f32(emb[token[b]]) (a token outside [0, V) gives zeros; SPC_DEBUG flags it)
__global__ void __launch_bounds__(LL_T) embed_kernel(const int32_t* __restrict__ token,
                                                     const uint16_t* __restrict__ emb, int V, int H,
                                                     float* __restrict__ h) {
  spc_pdl_entry();
  const int b = blockIdx.x, t = token[b];
  SPC_DCHECK(t >= 0 && t < V, SPC_E_RANGE);
  const bool ok = t >= 0 && t < V;
  for (int i = threadIdx.x; i < H; i += LL_T)
    h[(size_t)b * H + i] = ok ? bf(emb[(size_t)t * H + i]) : 0.f;
}

// token_out[b] = argmax_v logits[b][v] (bf16; the lowest index among equal maxima, NaN never
// wins), then seq_len[b] += 1 if seq_len != NULL: closes the autoregressive loop on the
// device (the next step's token is at position seq_len - 1).
constexpr int AM_T = 1024;
__global__ void __launch_bounds__(AM_T) argmax_kernel(const uint16_t* __restrict__ logits, int V,
                                                      int32_t* __restrict__ token_out,
                                                      int32_t* __restrict__ seq_len) {
  spc_pdl_entry();
  __shared__ unsigned long long red[AM_T / 32];
  const int b = blockIdx.x;
  const uint16_t* x = logits + (size_t)b * V;
  // key: order-preserving map of the bf16 value in the high bits, ~index in the low bits
  // (max key = max value, then lowest index)
  unsigned long long best = 0;
  for (int v = threadIdx.x; v < V; v += AM_T) {
    const uint32_t u = x[v];
    if ((u & 0x7FFFu) > 0x7F80u) continue;  // NaN
    const uint32_t ord = (u & 0x8000u) ? (~u & 0xFFFFu) : (u | 0x8000u);
    const unsigned long long key = ((unsigned long long)(ord + 1) << 32) | (uint32_t)~(uint32_t)v;
    best = key > best ? key : best;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const unsigned long long t = __shfl_xor_sync(0xffffffffu, best, o);
    best = t > best ? t : best;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < AM_T / 32; ++w) best = red[w] > best ? red[w] : best;
    token_out[b] = best ? (int32_t)~(uint32_t)(best & 0xFFFFFFFFu) : 0;
    if (seq_len) seq_len[b] += 1;
  }
}

// gu [B][2F] bf16 (gate rows then up rows) -> y [B][F] = bf16(silu(gate) * up)
__global__ void __launch_bounds__(LL_T) swiglu_kernel(const uint16_t* __restrict__ gu, int F,
                                                      uint16_t* __restrict__ y) {
  spc_pdl_entry();
  const int b = blockIdx.y;
  for (int i = blockIdx.x * LL_T + threadIdx.x; i < F; i += gridDim.x * LL_T) {
    const float g = bf(gu[(size_t)b * 2 * F + i]), u = bf(gu[(size_t)b * 2 * F + F + i]);
    y[(size_t)b * F + i] = tobf(g / (1.f + __expf(-g)) * u);
  }
}

__global__ void __launch_bounds__(LL_T) f32_to_bf16_kernel(const float* __restrict__ x, long long n,
                                                           uint16_t* __restrict__ y) {
  spc_pdl_entry();
  for (long long i = blockIdx.x * (long long)LL_T + threadIdx.x; i < n; i += (long long)gridDim.x * LL_T)
    y[i] = tobf(x[i]);
}

}  // namespace
}  // namespace spc

using namespace spc;

extern "C" int spc_llm_add_rmsnorm(float* h, const void* delta, const void* w, int B, int H, float eps,
                                   void* xn, spc_stream_t stream) {
  if (!h || !w || !xn) return SPC_E_NULL;
  if (B <= 0 || H <= 0) return SPC_E_SHAPE;
  if (H > NR_T * 4 * NR_V || H % 4) return SPC_E_UNSUPPORTED;
  if (((uintptr_t)h | (uintptr_t)w | (uintptr_t)xn | (uintptr_t)delta) % 16) return SPC_E_RANGE;
  return launched(launch_k(add_rmsnorm_kernel, dim3(B), dim3(NR_T), 0, as_stream(stream), h,
                           (const uint16_t*)delta, (const uint16_t*)w, H, eps, (uint16_t*)xn));
}

extern "C" int spc_llm_rope_append(const void* qkv, const float* inv_freq, const int32_t* seq_len,
                                   int B, int Hq, int G, int D, int rows, void* q_out, void* k_cache,
                                   void* v_cache, const int32_t* slot_tok, int k, void* k_buf,
                                   void* v_buf, spc_stream_t stream) {
  if (!qkv || !inv_freq || !seq_len || !q_out || !k_cache || !v_cache) return SPC_E_NULL;
  if (slot_tok && (!k_buf || !v_buf)) return SPC_E_NULL;
  if (B <= 0 || Hq <= 0 || G <= 0 || Hq % G || D <= 0 || D % 2 || rows <= 0 || (slot_tok && k <= 0))
    return SPC_E_SHAPE;
  if (D > 2 * RA_T) return SPC_E_UNSUPPORTED;
  if (slot_tok && (uintptr_t)slot_tok % 16) return SPC_E_RANGE;
  return launched(launch_k(rope_append_kernel, dim3(Hq + 2 * G, B), dim3(RA_T), 0, as_stream(stream),
                           (const uint16_t*)qkv, inv_freq, seq_len, Hq, G, D, rows, (uint16_t*)q_out,
                           (uint16_t*)k_cache, (uint16_t*)v_cache, slot_tok, k, (uint16_t*)k_buf,
                           (uint16_t*)v_buf));
}

extern "C" int spc_llm_embed(const int32_t* token, const void* emb, int V, int H, int B, float* h,
                             spc_stream_t stream) {
  if (!token || !emb || !h) return SPC_E_NULL;
  if (B <= 0 || V <= 0 || H <= 0) return SPC_E_SHAPE;
  return launched(launch_k(embed_kernel, dim3(B), dim3(LL_T), 0, as_stream(stream), token,
                           (const uint16_t*)emb, V, H, h));
}

extern "C" int spc_llm_argmax(const void* logits, int B, int V, int32_t* token_out, int32_t* seq_len,
                              spc_stream_t stream) {
  if (!logits || !token_out) return SPC_E_NULL;
  if (B <= 0 || V <= 0) return SPC_E_SHAPE;
  return launched(launch_k(argmax_kernel, dim3(B), dim3(AM_T), 0, as_stream(stream),
                           (const uint16_t*)logits, V, token_out, seq_len));
}

extern "C" int spc_llm_swiglu(const void* gu, int B, int F, void* y, spc_stream_t stream) {
  if (!gu || !y) return SPC_E_NULL;
  if (B <= 0 || F <= 0) return SPC_E_SHAPE;
  const int nx = std::min((F + LL_T - 1) / LL_T, 64);
  return launched(launch_k(swiglu_kernel, dim3(nx, B), dim3(LL_T), 0, as_stream(stream),
                           (const uint16_t*)gu, F, (uint16_t*)y));
}

extern "C" int spc_llm_f32_to_bf16(const float* x, long long n, void* y, spc_stream_t stream) {
  if (!x || !y) return SPC_E_NULL;
  if (n < 0) return SPC_E_SHAPE;
  if (n == 0) return SPC_OK;
  const long long nb = std::min<long long>((n + LL_T - 1) / LL_T, 4 * num_sms());
  return launched(launch_k(f32_to_bf16_kernel, dim3((unsigned)nb), dim3(LL_T), 0, as_stream(stream),
                           x, n, (uint16_t*)y));
}
