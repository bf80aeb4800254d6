// tmatile.cu — contiguous streaming of the retrieval-key cache with TMA 2-D tile loads
// (tools only): 64 MiB (config B's [8][32768][128] bf16 keys), boxes of 64 d x R rows
// with the 128-byte swizzle (the LOGITS smem layout), a producer lane per CTA and a
// trivial consumer, 4 address-distinct copies rotated launch to launch.  Compared with a
// plain LDG.128 stream of the same bytes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmatile tools/tmatile.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#define CK(x)                                                               \
  do {                                                                      \
    cudaError_t e_ = (x);                                                   \
    if (e_ != cudaSuccess) {                                                \
      printf("%s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e_));         \
      exit(1);                                                              \
    }                                                                       \
  } while (0)

constexpr int D = 128;
constexpr size_t NROWS = 8ull * 32768;  // 64 MiB
constexpr int NCOPY = 4;

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait_(uint32_t a, unsigned ph) {
  asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(a),
               "r"(ph)
               : "memory");
}

// CTA: warp 0 lane 0 = producer, warps 1..NC = consumers (each consumes every NC-th stage).
// Static tiles: CTA b takes tiles b, b + grid, ...; a tile = R rows x both 64-d halves.
template <int R, int NST, int NC>
__global__ void __launch_bounds__(32 * (NC + 1)) tile_stream(const __grid_constant__ CUtensorMap m, int ntiles,
                                                             unsigned* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  constexpr int STAGE = R * 128;  // one half tile
  __shared__ __align__(8) uint64_t full[NST], empty[NST];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t base = (su(sm) + 1023) & ~1023u;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nsteps = ((ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x) * 2;
  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      unsigned ph = 0;
      for (int i = 0; i < nsteps; ++i) {
        const int tile = blockIdx.x + (i >> 1) * gridDim.x, half = i & 1;
        if (i >= NST) wait_(su(&empty[s]), ph ^ 1);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(STAGE)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
            "[%4];" ::"r"(base + s * STAGE),
            "l"(&m), "r"(64 * half), "r"(tile * R), "r"(su(&full[s]))
            : "memory");
        if (++s == NST) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else {
    uint32_t acc = 0;
    int s = 0;
    unsigned ph = 0;
    for (int i = 0; i < nsteps; ++i) {
      if ((i % NC) == warp - 1) {
        wait_(su(&full[s]), ph);
        acc ^= *(const uint32_t*)(sm + (base - su(sm)) + s * STAGE + lane * 4);
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[s])) : "memory");
      }
      if (++s == NST) {
        s = 0;
        ph ^= 1;
      }
    }
    if (acc == 0x9e3779b9u) *sink = acc;
  }
}

__global__ void __launch_bounds__(256) ldg_stream(const uint4* __restrict__ p, size_t n, unsigned* sink) {
  uint32_t acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    const uint4 a = __ldcs(p + i), b = __ldcs(p + i + stride), c = __ldcs(p + i + 2 * stride),
                d = __ldcs(p + i + 3 * stride);
    acc ^= a.x ^ b.y ^ c.z ^ d.w;
  }
  for (; i < n; i += stride) acc ^= __ldcs(p + i).x;
  if (acc == 0x9e3779b9u) *sink = acc;
}

static CUtensorMap make_map(void* base, int boxrows) {
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fp, 12000, cudaEnableDefault, &q));
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
  CUtensorMap m;
  cuuint64_t dims[2] = {D, NROWS};
  cuuint64_t strides[1] = {D * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)boxrows};
  cuuint32_t es[2] = {1, 1};
  if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
      CUDA_SUCCESS) {
    printf("encode failed\n");
    exit(1);
  }
  return m;
}

template <typename F>
static void timeit(const char* name, F launch) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (int i = 0; i < 8; ++i) launch(i);
  CK(cudaDeviceSynchronize());
  float best = 1e9;
  for (int rep = 0; rep < 5; ++rep) {
    CK(cudaEventRecord(a));
    for (int i = 0; i < 40; ++i) launch(i);
    CK(cudaEventRecord(b));
    CK(cudaDeviceSynchronize());
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    best = std::min(best, ms / 40);
  }
  CK(cudaGetLastError());
  printf("%-40s %7.2f us per launch  %7.1f GB/s\n", name, best * 1e3, NROWS * D * 2 / (best * 1e-3) / 1e9);
}

template <int R, int NST, int NC>
static void run(CUtensorMap* maps, unsigned* sink, int nsm, int ctas) {
  auto k = tile_stream<R, NST, NC>;
  const int smem = R * 128 * NST + 1024;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  char name[96];
  snprintf(name, sizeof name, "tma tile %d rows x%d stages c%d x%d/SM", R, NST, NC, ctas);
  const int ntiles = (int)(NROWS / R);
  timeit(name, [&](int i) { k<<<nsm * ctas, 32 * (NC + 1), smem>>>(maps[i % NCOPY], ntiles, sink); });
}

int main() {
  int nsm;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  uint16_t* buf[NCOPY];
  CUtensorMap m128[NCOPY], m256[NCOPY], m64[NCOPY];
  for (int c = 0; c < NCOPY; ++c) {
    CK(cudaMalloc(&buf[c], NROWS * D * 2));
    CK(cudaMemset(buf[c], c + 1, NROWS * D * 2));
    m128[c] = make_map(buf[c], 128);
    m256[c] = make_map(buf[c], 256);
    m64[c] = make_map(buf[c], 64);
  }
  unsigned* sink;
  CK(cudaMalloc(&sink, 4));
  timeit("ldg.128 x4 unroll, 8x256 thr/SM", [&](int i) {
    ldg_stream<<<nsm * 8, 256>>>((const uint4*)buf[i % NCOPY], NROWS * D * 2 / 16, sink);
  });
  run<128, 12, 1>(m128, sink, nsm, 1);
  run<128, 12, 4>(m128, sink, nsm, 1);
  run<256, 6, 4>(m256, sink, nsm, 1);
  run<128, 6, 2>(m128, sink, nsm, 2);
  run<64, 12, 2>(m64, sink, nsm, 2);
  run<64, 24, 4>(m64, sink, nsm, 1);
  return 0;
}
