// exp_probe.cu — intermediates of spc_exp_dev vs spc_exp2_dev on given inputs (tools only).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2512_00722_b200/csrc -o tools/exp_probe tools/exp_probe.cu
#include <cstdio>
#include "common.cuh"
using namespace spc;
__global__ void probe(const float* xs, int n) {
  for (int i = 0; i < n; ++i) {
    const float x = xs[i];
    const float y = __uint_as_float(__float_as_uint(x) + 1u);  // the neighbour in the sweep
    const float2 e2 = spc_exp2_dev(x, y);
    const float2 e3 = spc_exp2_dev(y, x);
    printf("pair (x, next): %a %a   swapped: %a %a   scalar: %a %a\n", e2.x, e2.y, e3.y, e3.x,
           spc_exp_dev(x), spc_exp_dev(y));
    const float t = __fmul_rn(x, __uint_as_float(0x3FB8AA3Bu));
    const float big = __fadd_rn(t, 12582912.0f);
    const float nn = __fsub_rn(big, 12582912.0f);
    float r = __fmaf_rn(-nn, __uint_as_float(0x3F317200u), x);
    const float r1 = r;
    r = __fmaf_rn(-nn, __uint_as_float(0x35BFBE8Eu), r);
    // packed
    const unsigned long long X = f2_pack(x, __uint_as_float(__float_as_uint(x) + 1u));
    const unsigned long long T = f2_mul(X, f2_splat(__uint_as_float(0x3FB8AA3Bu)));
    const unsigned long long BIG = f2_add(T, f2_splat(12582912.0f));
    const unsigned long long N = f2_add(BIG, f2_splat(-12582912.0f));
    const float2 nf = f2_unpack(N);
    const unsigned long long NN = f2_pack(-nf.x, -nf.y);
    unsigned long long R = f2_fma(NN, f2_splat(__uint_as_float(0x3F317200u)), X);
    const float2 R1 = f2_unpack(R);
    R = f2_fma(NN, f2_splat(__uint_as_float(0x35BFBE8Eu)), R);
    const float2 R2 = f2_unpack(R);
    unsigned long long P = f2_splat(__uint_as_float(0x39500D01u));
    P = f2_fma(P, R, f2_splat(__uint_as_float(0x3AB60B61u)));
    P = f2_fma(P, R, f2_splat(__uint_as_float(0x3C088889u)));
    P = f2_fma(P, R, f2_splat(__uint_as_float(0x3D2AAAABu)));
    P = f2_fma(P, R, f2_splat(__uint_as_float(0x3E2AAAABu)));
    P = f2_fma(P, R, f2_splat(__uint_as_float(0x3F000000u)));
    P = f2_fma(P, R, f2_splat(__uint_as_float(0x3F800000u)));
    P = f2_fma(P, R, f2_splat(__uint_as_float(0x3F800000u)));
    float p = __uint_as_float(0x39500D01u);
    p = __fmaf_rn(p, r, __uint_as_float(0x3AB60B61u));
    p = __fmaf_rn(p, r, __uint_as_float(0x3C088889u));
    p = __fmaf_rn(p, r, __uint_as_float(0x3D2AAAABu));
    p = __fmaf_rn(p, r, __uint_as_float(0x3E2AAAABu));
    p = __fmaf_rn(p, r, __uint_as_float(0x3F000000u));
    p = __fmaf_rn(p, r, __uint_as_float(0x3F800000u));
    p = __fmaf_rn(p, r, __uint_as_float(0x3F800000u));
    printf("x %a t %a/%a big %a/%a n %a/%a r1 %a/%a r2 %a/%a p %a/%a (lane1 t %a n %a r2 %a p %a)\n", x, t,
           f2_unpack(T).x, big, f2_unpack(BIG).x, nn, nf.x, r1, R1.x, r, R2.x, p, f2_unpack(P).x,
           f2_unpack(T).y, nf.y, R2.y, f2_unpack(P).y);
  }
}
int main() {
  float h[] = {-6.584897994995117f, -7.971192359924316f, -12.130075454711914f, -50.253173828125f};
  float* d;
  cudaMalloc(&d, sizeof h);
  cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
  probe<<<1, 1>>>(d, 4);
  cudaDeviceSynchronize();
  return 0;
}
