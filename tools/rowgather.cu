// rowgather.cu — HBM gather bandwidth vs contiguous row size (tools only).
// Reads `total` bytes as random rows of R bytes (sorted random row ids per 8 MiB region,
// like a top-k selection at density 1/16) with LDG.128, many loads in flight per lane.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rowgather tools/rowgather.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

// each warp-iteration reads UNR rows (rows of R bytes = R/16 lanes-worth of 16-B vectors)
template <int R, int UNR>
__global__ void __launch_bounds__(256) gather(const uint4* __restrict__ src, const int* __restrict__ rows,
                                              int n_rows, unsigned* sink) {
  constexpr int VPR = R / 16;                  // 16-B vectors per row
  constexpr int RPW = VPR >= 32 ? 1 : 32 / VPR;  // rows per warp instruction
  constexpr int IPR = VPR >= 32 ? VPR / 32 : 1;  // instructions per row
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  uint32_t acc = 0;
  const int rows_per_it = RPW * UNR;
  for (int r0 = gw * rows_per_it; r0 < n_rows; r0 += nw * rows_per_it) {
    uint4 v[UNR][IPR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int r = r0 + u * RPW + (VPR >= 32 ? 0 : lane / VPR);
      const int row = rows[min(r, n_rows - 1)];
#pragma unroll
      for (int i = 0; i < IPR; ++i)
        v[u][i] = __ldcs(src + (size_t)row * VPR + (VPR >= 32 ? lane + 32 * i : lane % VPR));
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u)
#pragma unroll
      for (int i = 0; i < IPR; ++i) acc ^= v[u][i].x ^ v[u][i].w;
  }
  if (acc == 0x9e3779b9u) *sink = acc;
}

template <int R, int UNR>
void run(uint8_t* buf, size_t bufbytes, unsigned* sink, int nsm) {
  const size_t total = 256ull << 20;       // bytes gathered per launch
  const int n_rows = (int)(total / R);
  const size_t space_rows = bufbytes / R;  // 16x sparser than the gathered bytes
  std::vector<int> h(n_rows);
  std::mt19937 g(1);
  const size_t region = (8u << 20) / R;    // sorted ids within 8 MiB regions
  for (int i = 0; i < n_rows; ++i) h[i] = (int)(g() % space_rows);
  const char* mode = getenv("RG_MODE");
  if (!mode || mode[0] == 's') {  // sorted within 8 MiB-worth chunks of the list
    for (size_t a = 0; a < (size_t)n_rows; a += region / 16) {
      const size_t b = std::min((size_t)n_rows, a + region / 16);
      std::sort(h.begin() + a, h.begin() + b);
    }
  } else if (mode[0] == 'g') {  // fully sorted
    std::sort(h.begin(), h.end());
  }  // 'u': unsorted
  int* rows; CK(cudaMalloc(&rows, n_rows * 4)); CK(cudaMemcpy(rows, h.data(), n_rows * 4, cudaMemcpyHostToDevice));
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  const int grid = nsm * 8;
  for (int rep = 0; rep < 2; ++rep) {
    CK(cudaEventRecord(a));
    for (int it = 0; it < 10; ++it) gather<R, UNR><<<grid, 256>>>((const uint4*)buf, rows, n_rows, sink);
    CK(cudaEventRecord(b)); CK(cudaDeviceSynchronize());
    float ms; CK(cudaEventElapsedTime(&ms, a, b));
    if (rep) printf("row %5d B  unroll %d: %7.2f us per 256 MiB  %7.1f GB/s\n", R, UNR, ms * 100, total / (ms * 1e-4) / 1e9);
  }
  CK(cudaFree(rows));
}

int main() {
  int nsm; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const size_t bufbytes = 4ull << 30;  // 4 GiB (16 x the gathered bytes)
  uint8_t* buf; CK(cudaMalloc(&buf, bufbytes)); CK(cudaMemset(buf, 1, bufbytes));
  unsigned* sink; CK(cudaMalloc(&sink, 4));
  run<256, 8>(buf, bufbytes, sink, nsm); run<512, 8>(buf, bufbytes, sink, nsm);
  return 0;
}
