// pciegather.cu — zero-copy gather bandwidth from pinned host memory vs contiguous record
// size and loads in flight (tools only).  Random records (sorted ids) of R bytes are copied
// host -> HBM by warps (LDG.128 from the mapped host pointer, STG to device).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pciegather tools/pciegather.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

// one warp per record; each lane moves UNR 16-byte vectors per iteration
template <int UNR>
__global__ void __launch_bounds__(256) gather(const uint4* __restrict__ src, const int* __restrict__ ids, int n,
                                              int vpr, uint4* __restrict__ dst) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int r = gw; r < n; r += nw) {
    const uint4* s = src + (size_t)ids[r] * vpr;
    uint4* d = dst + (size_t)r * vpr;
    for (int v0 = 0; v0 < vpr; v0 += 32 * UNR) {
      uint4 x[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int v = v0 + u * 32 + lane;
        if (v < vpr) x[u] = __ldcv(s + v);
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int v = v0 + u * 32 + lane;
        if (v < vpr) d[v] = x[u];
      }
    }
  }
}

int main() {
  int nsm; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const size_t hbytes = (size_t)(getenv("PG_GB") ? atoi(getenv("PG_GB")) : 8) << 30;
  const bool sorted = !getenv("PG_UNSORTED");
  uint8_t* h; CK(cudaHostAlloc(&h, hbytes, cudaHostAllocMapped)); memset(h, 1, hbytes);
  uint8_t* hd; CK(cudaHostGetDevicePointer((void**)&hd, h, 0));
  const size_t total = 256ull << 20;
  uint8_t* d; CK(cudaMalloc(&d, total));
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  {  // DMA reference
    CK(cudaMemcpy(d, h, total, cudaMemcpyHostToDevice));
    CK(cudaEventRecord(a)); CK(cudaMemcpyAsync(d, h, total, cudaMemcpyHostToDevice)); CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b)); float ms; CK(cudaEventElapsedTime(&ms, a, b));
    printf("cudaMemcpy H2D 256 MiB: %.1f GB/s\n", total / (ms * 1e-3) / 1e9);
  }
  for (int R : {256, 16384}) {
    const int n = (int)(total / R), vpr = R / 16;
    std::vector<int> ids(n); std::mt19937 g(7);
    for (auto& x : ids) x = (int)(g() % (hbytes / R));
    if (sorted) std::sort(ids.begin(), ids.end());
    int* di; CK(cudaMalloc(&di, n * 4)); CK(cudaMemcpy(di, ids.data(), n * 4, cudaMemcpyHostToDevice));
    for (int cfg = 1; cfg < 3; ++cfg) {
      const int grid = nsm * (cfg == 0 ? 2 : 8);
      auto run = [&]() {
        if (cfg < 2) gather<1><<<grid, 256>>>((const uint4*)hd, di, n, vpr, (uint4*)d);
        else gather<4><<<grid, 256>>>((const uint4*)hd, di, n, vpr, (uint4*)d);
      };
      run(); CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(a)); run(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
      float ms; CK(cudaEventElapsedTime(&ms, a, b));
      printf("record %6d B  grid %4d x 256  unroll %d: %6.1f GB/s\n", R, grid, cfg == 2 ? 4 : 1, total / (ms * 1e-3) / 1e9);
    }
    CK(cudaFree(di));
  }
  return 0;
}
