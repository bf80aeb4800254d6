// common.cuh — device/host helpers shared by the libspc kernels (sm_100a).
// Nothing here is shared with the CPU oracle (oracle/); the contract functions
// below are written from DESIGN.md §3, independently of oracle/spcref.c.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>

#include "../../include/spc.h"

namespace spc {

// ----------------------------------------------------------------- host side
extern std::atomic<uint64_t> g_launches;
void set_cuda_error(cudaError_t e);
inline int launched(cudaError_t pre = cudaSuccess) {
  cudaError_t e = pre != cudaSuccess ? pre : cudaGetLastError();
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (e != cudaSuccess) {
    set_cuda_error(e);
    return SPC_E_CUDA;
  }
  return SPC_OK;
}
#define SPC_TRY(x)               \
  do {                           \
    int _rc = (x);               \
    if (_rc != SPC_OK) return _rc; \
  } while (0)

inline cudaStream_t as_stream(spc_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// Programmatic dependent launch: every libspc kernel starts with spc_pdl_entry()
// (griddepcontrol.wait before ANY global memory access, then launch_dependents), so a
// kernel launched with the PDL attribute behind another kernel only overlaps its launch
// and CTA scheduling with the predecessor's tail; memory semantics stay stream-ordered.
// SPC_PDL=0 in the environment launches without the attribute.
inline bool pdl_enabled() {
  static const int v = [] {
    const char* e = std::getenv("SPC_PDL");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  return v != 0;
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t st, Args... args) {
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
// launch_k with a runtime thread-block cluster size along x (grid.x a multiple of it)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_kc(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                             cudaStream_t st, int cluster_x, Args... args) {
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)cluster_x;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
// SPC_DEBUG builds: each translation unit's device error word is read (and cleared) through
// a reader registered here; spc_check_device_errors() polls them all (runtime.cu).
int register_err_reader(unsigned (*read_and_clear)(), const char* file);
// The max-dynamic-shared-memory attribute of a kernel (and optionally the non-portable
// cluster size), set once per (kernel, device, bytes): thread-safe, failures are returned
// (never remembered as set).
int smem_attr(const void* kern, int bytes, bool nonportable_cluster = false);
int num_sms();
// Encode the row-gather TMA descriptor of a bf16 [n_rows][D] tensor (driver entry point
// fetched through cudart): 64-element x 1-row boxes, 128-byte swizzle.
int make_tmap_rows_bf16(CUtensorMap* map, const void* base, uint64_t n_rows, uint32_t D);
// ... and the tile-streaming one: boxes of 64 elements x box_rows rows, 128-byte swizzle.
int make_tmap_tile_bf16(CUtensorMap* map, const void* base, uint64_t n_rows, uint32_t D,
                        uint32_t box_rows);

// ------------------------------------------- SPC_DEBUG device-side contract checks
// A violated data-dependent contract (include/spc.h: out-of-range index, unsorted set,
// slot map != previous set, NaN input) records its first spc_status and source line in this
// translation unit's error word; spc_check_device_errors() returns and clears it.  Release
// builds compile the checks out.
#ifdef SPC_DEBUG
static __device__ unsigned g_spc_dev_err = 0u;  // status | line << 8; one per translation unit
__device__ __forceinline__ void spc_dev_fail(int code, int line) {
  atomicCAS(&g_spc_dev_err, 0u, (unsigned)code | ((unsigned)line << 8));
}
#define SPC_DCHECK(cond, code)                                  \
  do {                                                          \
    if (!(cond)) ::spc::spc_dev_fail((code), __LINE__);         \
  } while (0)
static unsigned spc_read_and_clear_err() {
  unsigned v = 0u, z = 0u;
  if (cudaMemcpyFromSymbol(&v, g_spc_dev_err, sizeof v) != cudaSuccess) return 0u;
  cudaMemcpyToSymbol(g_spc_dev_err, &z, sizeof z);
  return v;
}
static const int spc_err_reader_registered = register_err_reader(spc_read_and_clear_err, __BASE_FILE__);
#else
#define SPC_DCHECK(cond, code) \
  do {                         \
  } while (0)
#endif

// --------------------------------------------------------------- device side
__device__ __forceinline__ void spc_pdl_entry() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ float bf16lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

// O3, written from DESIGN.md §3: exp for x <= 0 with IEEE RN ops only.
// n = rint(x * log2 e) by the 1.5 * 2^23 magic-number addition (RN-even, exact for
// |t| < 2^22, identical to rintf) and its integer read from the sum's bits, so no
// conversion-pipe instruction (FRND / F2I) is issued.
__device__ __forceinline__ float spc_exp_dev(float x) {
  const float t = __fmul_rn(x, __uint_as_float(0x3FB8AA3Bu));
  const float big = __fadd_rn(t, 12582912.0f);
  const float n = __fsub_rn(big, 12582912.0f);
  const int ni = (int)(__float_as_uint(big) - 0x4B400000u);
  float r = __fmaf_rn(-n, __uint_as_float(0x3F317200u), x);
  r = __fmaf_rn(-n, __uint_as_float(0x35BFBE8Eu), r);
  float p = __uint_as_float(0x39500D01u);                 // 1/7!
  p = __fmaf_rn(p, r, __uint_as_float(0x3AB60B61u));      // 1/6!
  p = __fmaf_rn(p, r, __uint_as_float(0x3C088889u));      // 1/5!
  p = __fmaf_rn(p, r, __uint_as_float(0x3D2AAAABu));      // 1/4!
  p = __fmaf_rn(p, r, __uint_as_float(0x3E2AAAABu));      // 1/3!
  p = __fmaf_rn(p, r, __uint_as_float(0x3F000000u));      // 1/2!
  p = __fmaf_rn(p, r, __uint_as_float(0x3F800000u));      // 1/1!
  p = __fmaf_rn(p, r, __uint_as_float(0x3F800000u));      // 1/0!
  const float two_n = __uint_as_float((uint32_t)(ni + 127) << 23);
  return x < -87.0f ? 0.0f : __fmul_rn(p, two_n);
}

// trunc(e * 2^40) as int64 for 0 <= e <= 1 (e * 2^40 is exact in fp32).
#ifdef SPC_FIXPOINT_INT
// from the bits: (1.mantissa) * 2^(E - 127 - 23 + 40), shifted with truncation (ALU pipe)
__device__ __forceinline__ long long fixpoint40(float e) {
  const uint32_t u = __float_as_uint(e);
  const int sh = (int)(u >> 23) - 110;
  const unsigned long long m = (unsigned long long)((u & 0x7FFFFFu) | 0x800000u);
  const unsigned long long v = sh >= 0 ? m << sh : (sh > -64 ? m >> -sh : 0ull);
  return u == 0u ? 0ll : (long long)v;
}
#else
__device__ __forceinline__ long long fixpoint40(float e) {
  return __float2ll_rz(__fmul_rn(e, 1099511627776.0f));
}
#endif

// Packed (f32x2) IEEE-RN arithmetic, per element identical to the scalar RN ops.
__device__ __forceinline__ unsigned long long f2_pack(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 f2_unpack(unsigned long long v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ unsigned long long f2_fma(unsigned long long a, unsigned long long b,
                                                     unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ unsigned long long f2_mul(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ unsigned long long f2_add(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ unsigned long long f2_splat(float a) { return f2_pack(a, a); }

// spc_exp_dev on two values at once with f32x2 instructions (same ops, same order,
// per element bit-identical to spc_exp_dev).
__device__ __forceinline__ float2 spc_exp2_dev(float x0, float x1) {
  const unsigned long long x = f2_pack(x0, x1);
  // t = RN(x log2 e) and big = RN(t + 1.5 2^23) as SCALAR ops: ptxas contracts a packed
  // mul.rn.f32x2 feeding an add.rn.f32x2 into one FFMA2 (a single rounding), which moves the
  // rint tie points x log2 e = k + 1/2 and flipped 12 of the 1.12e9 exp inputs by one ulp
  // (tests/test_gpu_score.py::test_exp_exhaustive_bit_identity); scalar FMUL / FADD keep
  // both roundings of O3
  const float b0 = __fadd_rn(__fmul_rn(x0, __uint_as_float(0x3FB8AA3Bu)), 12582912.0f);
  const float b1 = __fadd_rn(__fmul_rn(x1, __uint_as_float(0x3FB8AA3Bu)), 12582912.0f);
  const unsigned long long big = f2_pack(b0, b1);
  const unsigned long long n = f2_add(big, f2_splat(-12582912.0f));
  const float2 bigf = make_float2(b0, b1);
  const float2 nf = f2_unpack(n);
  const unsigned long long nn = f2_pack(-nf.x, -nf.y);
  unsigned long long r = f2_fma(nn, f2_splat(__uint_as_float(0x3F317200u)), x);
  r = f2_fma(nn, f2_splat(__uint_as_float(0x35BFBE8Eu)), r);
  unsigned long long p = f2_splat(__uint_as_float(0x39500D01u));
  p = f2_fma(p, r, f2_splat(__uint_as_float(0x3AB60B61u)));
  p = f2_fma(p, r, f2_splat(__uint_as_float(0x3C088889u)));
  p = f2_fma(p, r, f2_splat(__uint_as_float(0x3D2AAAABu)));
  p = f2_fma(p, r, f2_splat(__uint_as_float(0x3E2AAAABu)));
  p = f2_fma(p, r, f2_splat(__uint_as_float(0x3F000000u)));
  p = f2_fma(p, r, f2_splat(__uint_as_float(0x3F800000u)));
  p = f2_fma(p, r, f2_splat(__uint_as_float(0x3F800000u)));
  const int n0 = (int)(__float_as_uint(bigf.x) - 0x4B400000u);
  const int n1 = (int)(__float_as_uint(bigf.y) - 0x4B400000u);
  const float2 e = f2_unpack(f2_mul(p, f2_pack(__uint_as_float((uint32_t)(n0 + 127) << 23),
                                               __uint_as_float((uint32_t)(n1 + 127) << 23))));
  return make_float2(x0 < -87.0f ? 0.0f : e.x, x1 < -87.0f ? 0.0f : e.y);
}

// Composite key of the O7 order: (bits(v) << 32) | ~uint32(id); larger = earlier.
__device__ __forceinline__ unsigned long long composite(uint32_t vbits, int id) {
  return ((unsigned long long)vbits << 32) | (unsigned long long)(uint32_t)(~(uint32_t)id);
}

// -------------------------------------------- packed fp32 FMA (sm_100 FFMA2)
// d = a*b + c per lane, IEEE RN, no FTZ: per-element identical to fmaf().
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\t"
      "mov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}

// ------------------------------------------------------------- TMA descriptors
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
// mbarrier arrive / arrive.expect_tx / parity wait on 32-bit shared addresses
__device__ __forceinline__ void tm_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tm_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tm_wait(uint32_t bar, uint32_t ph) {
#ifdef SPC_SS_DEBUG
  for (long long n = 0;; ++n) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(ph)
        : "memory");
    if (ok) return;
    if (n == (1ll << 24)) {
      printf("mbarrier stuck: cta %d tid %d bar %u phase %u\n", blockIdx.x, threadIdx.x, bar, ph);
      return;
    }
  }
#endif
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "TMW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra TMW_%=;\n\t}" ::"r"(bar),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

// ---- DSMEM exchanges without cluster barriers.  A sender writes with remote st.async /
// red.async whose bytes complete the destination CTA's mbarrier (complete_tx) and arrives
// once on that mbarrier with the byte count it sends (arrive.expect_tx, relaxed: no fence
// that would wait for this CTA's outstanding global stores, as barrier.cluster.arrive's
// release does); the receiver waits for the phase (acquire, cluster scope), i.e. until every
// sender's bytes have landed.  Every mbarrier is used for one phase per launch (parity 0).
__device__ __forceinline__ uint32_t dsm_map(uint32_t a, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void dsm_st64(uint32_t ra, unsigned long long v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(ra),
               "l"(v), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void dsm_st32(uint32_t ra, uint32_t v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(ra),
               "r"(v), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void dsm_st128(uint32_t ra, uint4 v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                   ra),
               "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void dsm_red_add(uint32_t ra, uint32_t v, uint32_t rbar) {
  asm volatile(
      "red.async.relaxed.cluster.shared::cluster.mbarrier::complete_tx::bytes.add.u32 [%0], %1, [%2];" ::"r"(
          ra),
      "r"(v), "r"(rbar)
      : "memory");
}
__device__ __forceinline__ void dsm_expect(uint32_t rbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.relaxed.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(rbar),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void dsm_wait(uint32_t bar) {
  const long long t0 = clock64();
  for (;;) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], 0;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar)
        : "memory");
    if (ok) return;
    if (clock64() - t0 > 8000000000ll) __trap();  // ~4 s: a lost exchange fails loudly
  }
}
// The whole CTA waits for an exchange: ONE thread acquires the phase (cluster scope), the
// CTA barrier then orders everyone else after it (16 warps spinning on cluster-scope
// acquires slowed every exchange's exit).
__device__ __forceinline__ void dsm_wait_cta(uint32_t bar) {
  if (threadIdx.x == 0) dsm_wait(bar);
  __syncthreads();
}


// explicit shared-memory loads by 32-bit shared address (never generic LD)
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(a));
  return v;
}
__device__ __forceinline__ float4 lds128f(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(a));
  return v;
}
__device__ __forceinline__ float2 lds64f(uint32_t a) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
  return v;
}

// -------------------------------------------------------- warp reductions
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide exclusive scan of one int per thread.
// (requires blockDim.x a multiple of 32, <= 1024; contains __syncthreads)
__device__ __forceinline__ int block_excl_scan(int v, int* wsum, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();  // wsum may still be read by a previous call
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x / 32;
    int x = lane < nw ? wsum[lane] : 0;
    int xi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, xi, o);
      if (lane >= o) xi += t;
    }
    if (lane < nw) wsum[lane] = xi - x;
    if (lane == 31) *total = xi;
  }
  __syncthreads();
  return wsum[warp] + incl - v;
}

// "Last block done" ticket: returns true in exactly one CTA of a group after
// all `total` CTAs of that group have published their results; that CTA also
// resets the counter to 0 so the workspace stays reusable.
__device__ __forceinline__ bool last_block_ticket(unsigned int* counter, unsigned int total,
                                                  int* smem_flag) {
#ifndef SPC_DEBUG_NOFENCE  // timing experiments only: unsafe without the fence
  __threadfence();
#endif
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int t = atomicAdd(counter, 1u);
    *smem_flag = (t == total - 1);
    if (t == total - 1) *counter = 0u;
  }
  __syncthreads();
  bool last = *smem_flag != 0;
  if (last) __threadfence();
  return last;
}

}  // namespace spc
