// membench.cu — standalone microbenchmarks of 256-byte row-gather bandwidth on
// B200 (tools only, not part of libspc).  Each kernel reads n_rows rows of
// 256 bytes at rows[i] from src and folds them into a checksum.
//   mode 0: LDGSTS (cp.async 16 B) into a per-warp shared ring of `depth` stages of 16 rows
//   mode 1: LDG.128 into registers, `depth` rows per lane in flight (unrolled)
//   mode 2: cp.async.bulk (TMA) of whole 256-B rows into a per-warp ring, mbarrier completion
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int DEPTH>
__global__ void k_ldgsts(const uint4* __restrict__ src, const int* __restrict__ rows, int n_rows,
                         unsigned long long* sink) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  uint8_t* ring = sm + (size_t)warp * DEPTH * 16 * 256;
  const int gw = blockIdx.x * nw + warp, tw = gridDim.x * nw;
  const int n_blk = (n_rows + 15) / 16;
  uint32_t acc = 0;
  int s = 0;
  int issued = 0;
  // each warp handles blocks gw, gw+tw, ...
  auto issue = [&](int blk, int stage) {
    const int r = blk * 16 + (lane >> 4) * 8;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int row = rows[min(r + t, n_rows - 1)];
      const uint32_t dst = su32(ring + (size_t)stage * 4096 + ((lane >> 4) * 8 + t) * 256 + (lane & 15) * 16);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src + (size_t)row * 16 + (lane & 15)));
    }
  };
  for (int p = 0; p < DEPTH - 1; ++p) {
    const int blk = gw + (issued++) * tw;
    if (blk < n_blk) issue(blk, p);
    asm volatile("cp.async.commit_group;");
  }
  for (int c = 0;; ++c) {
    const int blk = gw + c * tw;
    if (blk >= n_blk) break;
    const int nb = gw + (issued++) * tw;
    if (nb < n_blk) issue(nb, (s + DEPTH - 1) % DEPTH);
    asm volatile("cp.async.commit_group;");
    asm volatile("cp.async.wait_group %0;" ::"n"(DEPTH - 1));
    __syncwarp();
    acc += *(const uint32_t*)(ring + (size_t)s * 4096 + lane * 128);
    __syncwarp();
    s = (s + 1) % DEPTH;
  }
  asm volatile("cp.async.wait_group 0;");
  if (acc == 0x12345678u) sink[0] = acc;
}

// row of gather slot i without an index load: sorted, one random row in every 32-row
// window (density 1/32), like a top-k selection of a long context
__device__ __forceinline__ int hrow(int i) {
  unsigned h = (unsigned)i * 2654435761u;
  h ^= h >> 15;
  return i * 32 + (int)(h & 31u);
}

template <int DEPTH, bool CONTIG>
__device__ __forceinline__ void k_ldgsts_h_body(const uint4* __restrict__ src,
                                                const int* __restrict__ rows, int n_rows,
                                                unsigned long long* sink) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  uint8_t* ring = sm + (size_t)warp * DEPTH * 16 * 256;
  const int gw = blockIdx.x * nw + warp, tw = gridDim.x * nw;
  const int n_blk = (n_rows + 15) / 16;
  uint32_t acc = 0;
  int s = 0, issued = 0;
  // CONTIG: warp gw owns the contiguous block range [gw * per, (gw + 1) * per)
  const int per = (n_blk + tw - 1) / tw;
  auto map = [&](int blk) { return CONTIG ? (blk - gw) / tw + gw * per : blk; };
  auto issue = [&](int blk, int stage) {
    const int r = map(blk) * 16 + (lane >> 4) * 8;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int row = hrow(min(r + t, n_rows - 1));
      const uint32_t dst = su32(ring + (size_t)stage * 4096 + ((lane >> 4) * 8 + t) * 256 + (lane & 15) * 16);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src + (size_t)row * 16 + (lane & 15)));
    }
  };
  for (int p = 0; p < DEPTH - 1; ++p) {
    const int blk = gw + (issued++) * tw;
    if (blk < n_blk) issue(blk, p);
    asm volatile("cp.async.commit_group;");
  }
  for (int c = 0;; ++c) {
    const int blk = gw + c * tw;
    if (blk >= n_blk) break;
    const int nb = gw + (issued++) * tw;
    if (nb < n_blk) issue(nb, (s + DEPTH - 1) % DEPTH);
    asm volatile("cp.async.commit_group;");
    asm volatile("cp.async.wait_group %0;" ::"n"(DEPTH - 1));
    __syncwarp();
    acc += *(const uint32_t*)(ring + (size_t)s * 4096 + lane * 128);
    __syncwarp();
    s = (s + 1) % DEPTH;
  }
  asm volatile("cp.async.wait_group 0;");
  if (acc == 0x12345678u) sink[0] = acc;
}

template <int DEPTH>
__global__ void k_ldgsts_h(const uint4* __restrict__ src, const int* __restrict__ rows, int n_rows,
                           unsigned long long* sink) {
  k_ldgsts_h_body<DEPTH, false>(src, rows, n_rows, sink);
}
template <int DEPTH>
__global__ void k_ldgsts_c(const uint4* __restrict__ src, const int* __restrict__ rows, int n_rows,
                           unsigned long long* sink) {
  k_ldgsts_h_body<DEPTH, true>(src, rows, n_rows, sink);
}

// attention-shaped stage: 16 rows of array A and the same 16 rows of array B (8 KiB),
// destination rows padded to 272 B like the attention ring
template <int DEPTH, int PAD, bool META = false>
__device__ __forceinline__ void k_kv(const uint4* __restrict__ src, const int* __restrict__ rows, int n_rows,
                     unsigned long long* sink) {
  __shared__ __align__(16) int meta_sm[32][32];
  extern __shared__ __align__(16) uint8_t sm[];
  constexpr int RB = 256 + PAD, STG = 2 * 16 * RB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  uint8_t* ring = sm + (size_t)warp * DEPTH * STG;
  const int gw = blockIdx.x * nw + warp, tw = gridDim.x * nw;
  const int n_blk = (n_rows / 2 + 15) / 16;  // n_rows/2 tokens: each moves 2 rows
  const uint4* srcB = src + (size_t)(n_rows / 2) * 32 * 16;  // second array past the first
  uint32_t acc = 0;
  int s = 0, issued = 0;
  auto issue = [&](int blk, int stage) {
    const int r = blk * 16 + (lane >> 4) * 8;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int row = hrow(min(r + t, n_rows / 2 - 1));
      const uint32_t dst = su32(ring + (size_t)stage * STG + ((lane >> 4) * 8 + t) * RB + (lane & 15) * 16);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src + (size_t)row * 16 + (lane & 15)));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16 * RB), "l"(srcB + (size_t)row * 16 + (lane & 15)));
    }
    if (META && lane < 16)  // attention-like metadata: 16 x 4-byte L1-allocating copies
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(su32(&meta_sm[warp][lane])), "l"(rows + ((blk * 16 + lane) & 1023)));
  };
  for (int p = 0; p < DEPTH - 1; ++p) {
    const int blk = gw + (issued++) * tw;
    if (blk < n_blk) issue(blk, p);
    asm volatile("cp.async.commit_group;");
  }
  for (int c = 0;; ++c) {
    const int blk = gw + c * tw;
    if (blk >= n_blk) break;
    const int nb = gw + (issued++) * tw;
    if (nb < n_blk) issue(nb, (s + DEPTH - 1) % DEPTH);
    asm volatile("cp.async.commit_group;");
    asm volatile("cp.async.wait_group %0;" ::"n"(DEPTH - 1));
    __syncwarp();
    acc += *(const uint32_t*)(ring + (size_t)s * STG + lane * 128);
    __syncwarp();
    s = (s + 1) % DEPTH;
  }
  asm volatile("cp.async.wait_group 0;");
  if (acc == 0x12345678u) sink[0] = acc;
}

template <int DEPTH>
__global__ void k_kv_p(const uint4* a, const int* b, int c, unsigned long long* d) {
  k_kv<DEPTH, 16>(a, b, c, d);
}
template <int DEPTH>
__global__ void k_kv_d(const uint4* a, const int* b, int c, unsigned long long* d) {
  k_kv<DEPTH, 0>(a, b, c, d);
}
template <int DEPTH>
__global__ void k_kv_m(const uint4* a, const int* b, int c, unsigned long long* d) {
  k_kv<DEPTH, 16, true>(a, b, c, d);
}

template <int DEPTH>
__global__ void k_ldg_h(const uint4* __restrict__ src, const int* __restrict__ rows, int n_rows,
                        unsigned long long* sink) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int tw = (gridDim.x * blockDim.x) >> 5;
  uint32_t acc = 0;
  for (int base = gw * 2 * DEPTH; base < n_rows; base += tw * 2 * DEPTH) {
    uint4 v[DEPTH];
#pragma unroll
    for (int d = 0; d < DEPTH; ++d) {
      const int r = min(base + d * 2 + (lane >> 4), n_rows - 1);
      v[d] = __ldcg(src + (size_t)hrow(r) * 16 + (lane & 15));
    }
#pragma unroll
    for (int d = 0; d < DEPTH; ++d) acc += v[d].x ^ v[d].w;
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

template <int DEPTH>
__global__ void k_ldg(const uint4* __restrict__ src, const int* __restrict__ rows, int n_rows,
                      unsigned long long* sink) {
  // each lane reads 16 B of a row; 16 lanes per row, 2 rows per warp-instruction
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int tw = (gridDim.x * blockDim.x) >> 5;
  uint32_t acc = 0;
  for (int base = gw * 2 * DEPTH; base < n_rows; base += tw * 2 * DEPTH) {
    uint4 v[DEPTH];
#pragma unroll
    for (int d = 0; d < DEPTH; ++d) {
      const int r = min(base + d * 2 + (lane >> 4), n_rows - 1);
      v[d] = __ldg(src + (size_t)rows[r] * 16 + (lane & 15));
    }
#pragma unroll
    for (int d = 0; d < DEPTH; ++d) acc += v[d].x ^ v[d].w;
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

template <int DEPTH>
__global__ void k_bulk(const uint4* __restrict__ src, const int* __restrict__ rows, int n_rows,
                       unsigned long long* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[32][DEPTH];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  uint8_t* ring = sm + (size_t)warp * DEPTH * 32 * 256;
  if (lane == 0)
    for (int d = 0; d < DEPTH; ++d)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[warp][d])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  __syncwarp();
  const int gw = blockIdx.x * nw + warp, tw = gridDim.x * nw;
  const int n_blk = (n_rows + 31) / 32;
  uint32_t acc = 0;
  int ph[DEPTH];
  for (int d = 0; d < DEPTH; ++d) ph[d] = 0;
  auto issue = [&](int blk, int st) {
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[warp][st])), "r"(32 * 256));
    __syncwarp();
    const int row = rows[min(blk * 32 + lane, n_rows - 1)];
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];" ::"r"(
                     su32(ring + (size_t)st * 8192 + lane * 256)),
                 "l"(src + (size_t)row * 16), "r"(su32(&bar[warp][st])));
  };
  int issued = 0;
  for (int p = 0; p < DEPTH; ++p) {
    const int blk = gw + (issued++) * tw;
    if (blk < n_blk) issue(blk, p);
  }
  for (int c = 0;; ++c) {
    const int blk = gw + c * tw;
    if (blk >= n_blk) break;
    const int st = c % DEPTH;
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
                     su32(&bar[warp][st])), "r"(ph[st]));
    ph[st] ^= 1;
    acc += *(const uint32_t*)(ring + (size_t)st * 8192 + lane * 256);
    __syncwarp();
    const int nb = gw + (issued++) * tw;
    if (nb < n_blk) issue(nb, st);
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

extern "C" int membench(int mode, int depth, int ctas, int threads, const void* src, const int* rows,
                        int n_rows, void* sink, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const uint4* s = (const uint4*)src;
  unsigned long long* k = (unsigned long long*)sink;
  const int nw = threads / 32;
#define L(KERN, D, SMEM)                                                                       \
  {                                                                                             \
    cudaFuncSetAttribute(KERN<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);           \
    KERN<D><<<ctas, threads, SMEM, st>>>(s, rows, n_rows, k);                                   \
  }
  if (mode == 0) {
    switch (depth) {
      case 2: L(k_ldgsts, 2, nw * 2 * 4096) break;
      case 3: L(k_ldgsts, 3, nw * 3 * 4096) break;
      case 4: L(k_ldgsts, 4, nw * 4 * 4096) break;
      case 6: L(k_ldgsts, 6, nw * 6 * 4096) break;
      case 8: L(k_ldgsts, 8, nw * 8 * 4096) break;
      case 12: L(k_ldgsts, 12, nw * 12 * 4096) break;
      default: return -1;
    }
  } else if (mode == 1) {
    switch (depth) {
      case 4: L(k_ldg, 4, 0) break;
      case 8: L(k_ldg, 8, 0) break;
      case 16: L(k_ldg, 16, 0) break;
      default: return -1;
    }
  } else if (mode == 3) {
    switch (depth) {
      case 2: L(k_ldgsts_h, 2, nw * 2 * 4096) break;
      case 3: L(k_ldgsts_h, 3, nw * 3 * 4096) break;
      case 4: L(k_ldgsts_h, 4, nw * 4 * 4096) break;
      case 6: L(k_ldgsts_h, 6, nw * 6 * 4096) break;
      default: return -1;
    }
  } else if (mode == 5) {
    switch (depth) {
      case 3: L(k_ldgsts_c, 3, nw * 3 * 4096) break;
      case 6: L(k_ldgsts_c, 6, nw * 6 * 4096) break;
      default: return -1;
    }
  } else if (mode == 8) {  // padded rows + attention-like 4-byte .ca metadata copies
    switch (depth) {
      case 2: L(k_kv_m, 2, nw * 2 * 2 * 16 * 272) break;
      case 3: L(k_kv_m, 3, nw * 3 * 2 * 16 * 272) break;
      default: return -1;
    }
  } else if (mode == 6 || mode == 7) {  // 6: padded 272-B rows, 7: dense 256-B rows
    if (mode == 6) {
      switch (depth) {
        case 2: L(k_kv_p, 2, nw * 2 * 2 * 16 * 272) break;
        case 3: L(k_kv_p, 3, nw * 3 * 2 * 16 * 272) break;
        default: return -1;
      }
    } else {
      switch (depth) {
        case 2: L(k_kv_d, 2, nw * 2 * 2 * 16 * 256) break;
        case 3: L(k_kv_d, 3, nw * 3 * 2 * 16 * 256) break;
        default: return -1;
      }
    }
  } else if (mode == 4) {
    switch (depth) {
      case 4: L(k_ldg_h, 4, 0) break;
      case 8: L(k_ldg_h, 8, 0) break;
      case 16: L(k_ldg_h, 16, 0) break;
      default: return -1;
    }
  } else {
    switch (depth) {
      case 2: L(k_bulk, 2, nw * 2 * 8192) break;
      case 4: L(k_bulk, 4, nw * 4 * 8192) break;
      default: return -1;
    }
  }
  return (int)cudaGetLastError();
}
