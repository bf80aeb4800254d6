// lg_bench2.cu — the product LOGITS kernel (csrc/logits.cuh) launched back to back over
// 16 address-distinct 64 MiB key copies, fresh claim counters per launch (the finalize
// kernel that resets them in the library is not launched here).  Tools only.
#include <cstdio>
#include <vector>
#include "../paper_2512_00722_b200/csrc/common.cuh"
namespace spc {
int num_sms() { int n; cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, 0); return n; }
namespace {
#include "../paper_2512_00722_b200/csrc/logits.cuh"
}
}
using namespace spc;
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)
int main(int argc, char** argv) {
  const int B = 1, G = 8, A = 4, D = 128, S = 32768, NC = 16;
  const size_t win = (size_t)B * G * S * D;
  uint16_t *keys, *q; float *out, *hm, *tmax; unsigned *ctr; int* seq;
  CK(cudaMalloc(&keys, win * 2 * NC)); CK(cudaMemset(keys, 0x3c, win * 2 * NC));
  CK(cudaMalloc(&q, B * G * A * D * 2)); CK(cudaMemset(q, 0x3c, B * G * A * D * 2));
  CK(cudaMalloc(&out, (size_t)B * G * A * S * 4)); CK(cudaMalloc(&hm, 4096));
  CK(cudaMalloc(&tmax, (size_t)B * G * A * (S / LG_TR) * 4));
  CK(cudaMalloc(&ctr, 4096)); CK(cudaMemset(ctr, 0, 4096));
  CK(cudaMalloc(&seq, 4)); CK(cudaMemcpy(seq, &S, 4, cudaMemcpyHostToDevice));
  auto k = logits_kernel<D, A>;
  const int smem = LgSmem<D, A>::BYTES;  // (the LOGITS kernel of csrc/logits.cuh)
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int tpr = S / LG_TR, ntiles = B * G * tpr;
  const int nsm = num_sms();
  for (int pdl = 0; pdl < 2; ++pdl) {
    cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
    for (int rep = 0; rep < 2; ++rep) {
      CK(cudaMemset(ctr, 0, 4096));
      CK(cudaEventRecord(a));
      for (int it = 0; it < 30; ++it) {
        if (pdl) CK(launch_k(k, dim3(nsm), dim3(32 * lg_warps<A>()), smem, (cudaStream_t)0, keys + (it % NC) * win, q, seq, G, S, 0.0883883476f, tpr, ntiles, out, tmax, ctr + 2 * it));
        else k<<<nsm, 32 * lg_warps<A>(), smem>>>(keys + (it % NC) * win, q, seq, G, S, 0.0883883476f, tpr, ntiles, out, tmax, ctr + 2 * it);
      }
      CK(cudaEventRecord(b)); CK(cudaDeviceSynchronize());
      float ms; CK(cudaEventElapsedTime(&ms, a, b));
      printf("%s pdl=%d  %7.2f us\n", argc > 1 ? argv[1] : "", pdl, ms * 1e3f / 30);
    }
  }
  return 0;
}
