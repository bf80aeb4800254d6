// runtime.cu — status strings, launch counter, device queries, TMA descriptor
// encoding (row-gather maps of spc_kv_desc_init).  Part of libspc.so (see include/spc.h).
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstring>
#include <mutex>

#include "common.cuh"

#include <set>
#include <tuple>
#include <vector>

namespace spc {
std::atomic<uint64_t> g_launches{0};

struct ErrReader {
  unsigned (*fn)();
  const char* file;
};
static std::vector<ErrReader>& err_readers() {
  static std::vector<ErrReader> v;
  return v;
}
static std::mutex g_reader_mu;
int register_err_reader(unsigned (*read_and_clear)(), const char* file) {
  std::lock_guard<std::mutex> lk(g_reader_mu);
  err_readers().push_back({read_and_clear, file});
  return 1;
}
static thread_local char g_err[256] = "";

void set_cuda_error(cudaError_t e) {
  snprintf(g_err, sizeof(g_err), "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
}

int smem_attr(const void* kern, int bytes, bool nonportable_cluster) {
  static std::mutex mu;
  static std::set<std::tuple<const void*, int, int>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) {
    set_cuda_error(e);
    return SPC_E_CUDA;
  }
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(kern, dev, bytes);
  if (done.count(key)) return SPC_OK;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess && nonportable_cluster)
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) {
    set_cuda_error(e);
    return SPC_E_CUDA;
  }
  done.insert(key);
  return SPC_OK;
}

int num_sms() {  // per device (a process may drive several GPUs)
  static std::atomic<int> cache[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  int n = cache[dev].load(std::memory_order_relaxed);
  if (!n) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
    cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault,
                                         &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D descriptors of a bf16 [n_rows][D] tensor with the 128-byte swizzle: row gathers
// (boxes of 64 elements x 1 row, tile::gather4 loads, attn_tma.cuh) and tile streams
// (64 elements x box_rows rows, logits_tma_kernel).
int make_tmap_rows_bf16(CUtensorMap* map, const void* base, uint64_t n_rows, uint32_t D) {
  return make_tmap_tile_bf16(map, base, n_rows, D, 1);
}
int make_tmap_tile_bf16(CUtensorMap* map, const void* base, uint64_t n_rows, uint32_t D,
                        uint32_t box_rows) {
  auto enc = get_encode();
  if (!enc) {
    snprintf(g_err, sizeof(g_err), "cuTensorMapEncodeTiled unavailable");
    return SPC_E_CUDA;
  }
  cuuint64_t dims[2] = {D, n_rows};
  cuuint64_t strides[1] = {(cuuint64_t)D * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    snprintf(g_err, sizeof(g_err), "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return SPC_E_CUDA;
  }
  return SPC_OK;
}
}  // namespace spc

extern "C" {

const char* spc_status_string(int s) {
  switch (s) {
    case SPC_OK: return "SPC_OK";
    case SPC_E_NULL: return "SPC_E_NULL: required pointer is NULL";
    case SPC_E_SHAPE: return "SPC_E_SHAPE: invalid shape";
    case SPC_E_BUDGET: return "SPC_E_BUDGET: budget k out of range";
    case SPC_E_RANGE: return "SPC_E_RANGE: argument out of range";
    case SPC_E_STATE: return "SPC_E_STATE: inconsistent state";
    case SPC_E_WORKSPACE: return "SPC_E_WORKSPACE: workspace too small";
    case SPC_E_UNSUPPORTED: return "SPC_E_UNSUPPORTED: configuration not compiled in";
    case SPC_E_CUDA: return "SPC_E_CUDA: CUDA error";
    default: return "unknown spc_status";
  }
}
const char* spc_last_cuda_error(void) { return spc::g_err; }

int spc_debug_build(void) {
#ifdef SPC_DEBUG
  return 1;
#else
  return 0;
#endif
}

int spc_check_device_errors(spc_stream_t stream) {
  cudaError_t e = cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream));
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    spc::set_cuda_error(e);
    return SPC_E_CUDA;
  }
  int rc = SPC_OK;
  std::lock_guard<std::mutex> lk(spc::g_reader_mu);
  for (const auto& r : spc::err_readers()) {
    const unsigned v = r.fn();
    if (v && rc == SPC_OK) {
      rc = (int)(v & 0xFFu);
      snprintf(spc::g_err, sizeof(spc::g_err), "device contract violation (%s) at %s:%u",
               spc_status_string(rc), r.file, v >> 8);
    }
  }
  return rc;
}
int spc_version(void) { return 100; }
uint64_t spc_launch_count(void) { return spc::g_launches.load(); }
}
