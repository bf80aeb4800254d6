// tmagather.cu — selected-row gather throughput: TMA tile::gather4 vs LDG (tools only).
// The attention's access pattern: K and V rows (256 B, D = 128 bf16) of the same random
// sorted row ids, 256 MiB per launch (2^19 rows of each), 4 address-disjoint row lists
// rotated launch to launch (1 GiB of distinct rows > L2).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmagather tools/tmagather.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>
#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      printf("%s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e_));                 \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

constexpr int D = 128;
constexpr size_t TROWS = 1ull << 23;  // rows per tensor (2 GiB)
constexpr int NROWS = 1 << 19;        // rows gathered per tensor per launch (128 MiB)
constexpr int NLIST = 4;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t a, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t a, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, unsigned ph) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(a),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void g4(uint32_t dst, const CUtensorMap* m, uint32_t bar, int col, int4 r) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst),
      "l"(m), "r"(bar), "r"(col), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w)
      : "memory");
}

// One producer warp (lane i issues request i of a stage), NCONS consumer warps that wait
// for a stage, optionally touch it (sum one word per lane), and release it.
// BOXW = 128: one gather4 per 4 rows per tensor (1 KiB); 64: two (SWIZZLE_128B halves).
template <int BOXW, int RPS, int NST, int NCONS, bool TOUCH>
__global__ void __launch_bounds__(32 * (NCONS + 1)) tma_gather(const __grid_constant__ CUtensorMap tk,
                                                               const __grid_constant__ CUtensorMap tv,
                                                               const int* __restrict__ rows, int n_rows,
                                                               unsigned* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  constexpr int STAGE = RPS * D * 2 * 2;
  constexpr int NREQ = RPS / 4;  // gather4 requests per tensor per d-half
  static_assert(NREQ <= 32, "one request per producer lane");
  __shared__ __align__(8) uint64_t full[NST], empty[NST];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), NCONS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nch = n_rows / RPS;
  const int per = (nch + gridDim.x - 1) / gridDim.x;
  const int c0 = min(nch, (int)blockIdx.x * per), c1 = min(nch, c0 + per);
  const uint32_t base = smem_u32(sm);
  if (warp == NCONS) {  // producer: indices of stage c + PF loaded while stage c issues
    constexpr int PF = 4;
    int s = 0;
    unsigned ph = 0;
    int4 rr[PF];
#pragma unroll
    for (int u = 0; u < PF; ++u)
      rr[u] = (lane < NREQ && c0 + u < c1) ? __ldg(reinterpret_cast<const int4*>(rows + (size_t)(c0 + u) * RPS) + lane)
                                           : make_int4(0, 0, 0, 0);
    for (int cb = c0; cb < c1; cb += PF) {
#pragma unroll
      for (int u = 0; u < PF; ++u) {
        const int c = cb + u;
        if (c >= c1) break;
        if (c - c0 >= NST) mbar_wait(smem_u32(&empty[s]), ph ^ 1);
        const int4 r = rr[u];
        rr[u] = (lane < NREQ && c + PF < c1)
                    ? __ldg(reinterpret_cast<const int4*>(rows + (size_t)(c + PF) * RPS) + lane)
                    : make_int4(0, 0, 0, 0);
        const uint32_t fb = smem_u32(&full[s]);
        if (lane == 0) mbar_expect(fb, STAGE);
        __syncwarp();
        if (lane < NREQ) {
          const uint32_t st = base + (uint32_t)s * STAGE;
          if (BOXW == 128) {
            g4(st + lane * 1024, &tk, fb, 0, r);
            g4(st + STAGE / 2 + lane * 1024, &tv, fb, 0, r);
          } else {
            g4(st + lane * 512, &tk, fb, 0, r);
            g4(st + RPS * 128 + lane * 512, &tk, fb, 64, r);
            g4(st + STAGE / 2 + lane * 512, &tv, fb, 0, r);
            g4(st + STAGE / 2 + RPS * 128 + lane * 512, &tv, fb, 64, r);
          }
        }
        if (++s == NST) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else {
    int s = 0;
    unsigned ph = 0;
    uint32_t acc = 0;
    for (int c = c0; c < c1; ++c) {
      mbar_wait(smem_u32(&full[s]), ph);
      if (TOUCH) {
        const uint32_t* w = reinterpret_cast<const uint32_t*>(sm + (size_t)s * STAGE);
        for (int i = warp * 32 + lane; i < STAGE / 4; i += NCONS * 32 * 8) acc ^= w[i];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&empty[s]));
      if (++s == NST) {
        s = 0;
        ph ^= 1;
      }
    }
    if (acc == 0x9e3779b9u) *sink = acc;
  }
}

// LDG reference: a warp gathers K and V rows (lanes 0-15 row r, 16-31 row r+1), UNR pairs
// of rows in flight per lane
template <int UNR>
__global__ void __launch_bounds__(256) ldg_gather(const uint4* __restrict__ k, const uint4* __restrict__ v,
                                                  const int* __restrict__ rows, int n_rows, unsigned* sink) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  uint32_t acc = 0;
  for (int r0 = gw * 2 * UNR; r0 < n_rows; r0 += nw * 2 * UNR) {
    uint4 a[UNR], b[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int row = rows[min(r0 + 2 * u + (lane >> 4), n_rows - 1)];
      a[u] = __ldcs(k + (size_t)row * 16 + (lane & 15));
      b[u] = __ldcs(v + (size_t)row * 16 + (lane & 15));
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) acc ^= a[u].x ^ b[u].w;
  }
  if (acc == 0x9e3779b9u) *sink = acc;
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q));
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}
static CUtensorMap make_map(void* base, int boxw) {
  CUtensorMap m;
  cuuint64_t dims[2] = {D, TROWS};
  cuuint64_t strides[1] = {D * 2};
  cuuint32_t box[2] = {(cuuint32_t)boxw, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE,
                     boxw == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("encode failed %d\n", (int)r);
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
  float best = 1e9, sum = 0;
  for (int rep = 0; rep < 5; ++rep) {
    CK(cudaEventRecord(a));
    for (int i = 0; i < 20; ++i) launch(i);
    CK(cudaEventRecord(b));
    CK(cudaDeviceSynchronize());
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    best = std::min(best, ms / 20);
    sum += ms / 20;
  }
  CK(cudaGetLastError());
  const double bytes = 2.0 * NROWS * D * 2;
  printf("%-44s best %7.2f us  mean %7.2f us  %7.1f GB/s\n", name, best * 1e3, sum / 5 * 1e3,
         bytes / (best * 1e-3) / 1e9);
}

template <int BOXW, int RPS, int NST, int NCONS, bool TOUCH>
static void run_tma(const CUtensorMap& mk, const CUtensorMap& mv, int* const* lists, unsigned* sink,
                    int nsm, int ctas) {
  auto kern = tma_gather<BOXW, RPS, NST, NCONS, TOUCH>;
  const int smem = RPS * D * 2 * 2 * NST;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  char name[128];
  snprintf(name, sizeof name, "tma g4 box%d rps%d nst%d cons%d %s x%d/SM", BOXW, RPS, NST, NCONS,
           TOUCH ? "touch" : "", ctas);
  timeit(name, [&](int i) {
    kern<<<nsm * ctas, 32 * (NCONS + 1), smem>>>(mk, mv, lists[i % NLIST], NROWS, sink);
  });
}

int main() {
  int nsm;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  uint16_t *k, *v;
  CK(cudaMalloc(&k, TROWS * D * 2));
  CK(cudaMalloc(&v, TROWS * D * 2));
  CK(cudaMemset(k, 1, TROWS * D * 2));
  CK(cudaMemset(v, 2, TROWS * D * 2));
  unsigned* sink;
  CK(cudaMalloc(&sink, 4));
  // list i: rows in [i * TROWS/4, (i+1) * TROWS/4), 2048 sorted rows per 32768-row group
  int* lists[NLIST];
  std::mt19937 g(7);
  for (int i = 0; i < NLIST; ++i) {
    std::vector<int> h(NROWS);
    const int groups = NROWS / 2048;
    const size_t span = getenv("TG_DENSE") ? TROWS / NLIST / groups : TROWS / groups;  // 1/4 or 1/16
    for (int gq = 0; gq < groups; ++gq) {
      std::vector<int> pick;
      while ((int)pick.size() < 2048) {
        pick.push_back((int)(g() % span));
        if ((int)pick.size() == 2048) {
          std::sort(pick.begin(), pick.end());
          pick.erase(std::unique(pick.begin(), pick.end()), pick.end());
        }
      }
      const size_t off = getenv("TG_DENSE") ? i * (TROWS / NLIST) : 0;
      for (int j = 0; j < 2048; ++j) h[gq * 2048 + j] = (int)(off + gq * span + pick[j]);
    }
    CK(cudaMalloc(&lists[i], NROWS * 4));
    CK(cudaMemcpy(lists[i], h.data(), NROWS * 4, cudaMemcpyHostToDevice));
  }
  const CUtensorMap k128 = make_map(k, 128), v128 = make_map(v, 128);
  const CUtensorMap k64 = make_map(k, 64), v64 = make_map(v, 64);

  timeit("ldg unr4 x8 CTAs(256)/SM", [&](int i) {
    ldg_gather<4><<<nsm * 8, 256>>>((const uint4*)k, (const uint4*)v, lists[i % NLIST], NROWS, sink);
  });
  timeit("ldg unr8 x8 CTAs(256)/SM", [&](int i) {
    ldg_gather<8><<<nsm * 8, 256>>>((const uint4*)k, (const uint4*)v, lists[i % NLIST], NROWS, sink);
  });
  run_tma<128, 32, 3, 1, false>(k128, v128, lists, sink, nsm, 4);
  run_tma<64, 32, 3, 1, false>(k64, v64, lists, sink, nsm, 4);
  run_tma<64, 64, 3, 1, false>(k64, v64, lists, sink, nsm, 2);
  run_tma<64, 32, 6, 1, false>(k64, v64, lists, sink, nsm, 2);
  return 0;
}
