// ffma_bench.cu — throughput of the LOGITS inner-loop instruction mix on one SM
// (tools only).  Each warp repeatedly runs the per-16-byte-granule body:
// LDS.128 of its rows' keys (RPT rows), broadcast LDS.128 of {q,q} pairs,
// bf16->fp32 unpack, and ALPHA x RPT/2 FFMA2 (mode 0) or ALPHA x RPT FFMA (mode 1).
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "mov.b64 rc, {%6, %7};\n\tfma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}

template <int RPT, int ALPHA, int MODE>
__global__ void k(int iters, float* out, unsigned long long* cyc) {
  __shared__ __align__(16) uint4 keys[32 * RPT * 8];
  __shared__ __align__(16) float2 qd[8 * ALPHA * 8];
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 32 * RPT * 8; i += blockDim.x)
    keys[i] = make_uint4(0x3f803f80u + i, 0x3f803f81u, 0x3f803f82u, 0x3f803f83u);
  for (int i = threadIdx.x; i < 8 * ALPHA * 8; i += blockDim.x) qd[i] = make_float2(1e-7f * i, 1e-7f * i);
  __syncthreads();
  float2 acc[ALPHA][RPT / 2];
  float accs[ALPHA][RPT];
#pragma unroll
  for (int j = 0; j < ALPHA; ++j) {
#pragma unroll
    for (int p = 0; p < RPT / 2; ++p) acc[j][p] = make_float2(0.f, 0.f);
#pragma unroll
    for (int p = 0; p < RPT; ++p) accs[j][p] = 0.f;
  }
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int u = it & 7;
    uint4 w[RPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i) w[i] = keys[(lane + 32 * i) * 8 + (u ^ (lane & 7))];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      if (MODE == 0) {
        float2 kk[RPT / 2];
#pragma unroll
        for (int p = 0; p < RPT / 2; ++p) {
          const uint32_t x0 = (&w[2 * p].x)[e >> 1], x1 = (&w[2 * p + 1].x)[e >> 1];
          kk[p] = (e & 1) ? make_float2(__uint_as_float(x0 & 0xffff0000u), __uint_as_float(x1 & 0xffff0000u))
                          : make_float2(__uint_as_float(x0 << 16), __uint_as_float(x1 << 16));
        }
#pragma unroll
        for (int j = 0; j < ALPHA; j += 2) {
          const float4 q4 = *(const float4*)&qd[(u * 8 + e) * ALPHA + j];
#pragma unroll
          for (int p = 0; p < RPT / 2; ++p) {
            acc[j][p] = ffma2(kk[p], make_float2(q4.x, q4.y), acc[j][p]);
            acc[j + 1][p] = ffma2(kk[p], make_float2(q4.z, q4.w), acc[j + 1][p]);
          }
        }
      } else {
        float kk[RPT];
#pragma unroll
        for (int p = 0; p < RPT; ++p) {
          const uint32_t x = (&w[p].x)[e >> 1];
          kk[p] = (e & 1) ? __uint_as_float(x & 0xffff0000u) : __uint_as_float(x << 16);
        }
#pragma unroll
        for (int j = 0; j < ALPHA; j += 2) {
          const float4 q4 = *(const float4*)&qd[(u * 8 + e) * ALPHA + j];
#pragma unroll
          for (int p = 0; p < RPT; ++p) {
            accs[j][p] = __fmaf_rn(kk[p], q4.x, accs[j][p]);
            accs[j + 1][p] = __fmaf_rn(kk[p], q4.z, accs[j + 1][p]);
          }
        }
      }
    }
  }
  unsigned long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < ALPHA; ++j) {
#pragma unroll
    for (int p = 0; p < RPT / 2; ++p) s += acc[j][p].x + acc[j][p].y;
#pragma unroll
    for (int p = 0; p < RPT; ++p) s += accs[j][p];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

extern "C" int ffma_bench(int rpt, int mode, int warps, int iters, float* out,
                          unsigned long long* cyc) {
  dim3 grid(148), block(32 * warps);
  if (rpt == 2 && mode == 0) k<2, 4, 0><<<grid, block>>>(iters, out, cyc);
  else if (rpt == 4 && mode == 0) k<4, 4, 0><<<grid, block>>>(iters, out, cyc);
  else if (rpt == 8 && mode == 0) k<8, 4, 0><<<grid, block>>>(iters, out, cyc);
  else if (rpt == 4 && mode == 1) k<4, 4, 1><<<grid, block>>>(iters, out, cyc);
  else return -1;
  return (int)cudaGetLastError();
}
