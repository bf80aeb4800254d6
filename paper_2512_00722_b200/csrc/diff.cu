// diff.cu — spc_elastic_diff (O8) and spc_gather_kv (O9).
//
// Paper §5.4: with S_last the previous selection and S_now the
// current one, load S_now − S_last and overwrite S_last − S_now in place with
// Tensor.copy_(); the fixed budget makes both sets equally large.  Prefetch on
// separate CUDA streams; the KV source may live in CPU DRAM.
//
// spc_elastic_diff: one CTA per (b,g) row.  Sorted-set membership by binary
// search in shared memory, order-preserving compaction with a ballot/shuffle
// block scan, slot reuse in ascending slot order (reading R13).
// spc_gather_kv: vectorised 16-byte row copies, one warp per (layer, row);
// sources may be mapped pinned host memory (zero-copy PCIe reads).
#include <algorithm>

#include "common.cuh"

namespace spc {
namespace {

constexpr int DF_THREADS = 256;
constexpr int DF_PER = SPC_MAX_K / DF_THREADS;
constexpr int DF_BM_WORDS = 1 << 14;  // 64 KiB bitmap per list: token ids < 2^19

__device__ __forceinline__ bool contains(const int32_t* a, int n, int x) {
  int lo = 0, hi = n;  // a ascending
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    int v = a[mid];
    if (v == x) return true;
    if (v < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  return false;
}

__global__ void __launch_bounds__(DF_THREADS) diff_kernel(
    const int32_t* __restrict__ prev_idx, const int32_t* __restrict__ prev_count,
    const int32_t* __restrict__ cur_idx, const int32_t* __restrict__ cur_count, int k,
    int32_t* __restrict__ slot_tok, int32_t* __restrict__ load_tok, int32_t* __restrict__ load_slot,
    int32_t* __restrict__ n_load, int32_t* __restrict__ evict_tok, int32_t* __restrict__ n_evict) {
  spc_pdl_entry();
  extern __shared__ int32_t dsm[];
  int32_t* sprev = dsm;       // [k]
  int32_t* scur = dsm + k;    // [k]
  int32_t* snew = dsm + 2 * k;  // [k]
  __shared__ int wsum[DF_THREADS / 32];
  __shared__ int total;
  const int row = blockIdx.x, tid = threadIdx.x;
  const int np = min(max(prev_count[row], 0), k), nc = min(max(cur_count[row], 0), k);
  const int32_t* pv = prev_idx + (size_t)row * k;
  const int32_t* cv = cur_idx + (size_t)row * k;
  // membership bitmaps over token ids (both lists ascending: the last entries bound the ids);
  // binary search in the sorted lists when the ids exceed the bitmap capacity
  uint32_t* bm_prev = (uint32_t*)(dsm + 3 * k);
  uint32_t* bm_cur = bm_prev + DF_BM_WORDS;
  const int maxtok = max(np ? __ldg(pv + np - 1) : -1, nc ? __ldg(cv + nc - 1) : -1);
  const bool use_bm = maxtok < DF_BM_WORDS * 32;
  const int nwords = use_bm ? (maxtok >> 5) + 1 : 0;
  for (int i = tid; i < nwords; i += DF_THREADS) bm_prev[i] = bm_cur[i] = 0u;
  for (int i = tid; i < np; i += DF_THREADS) sprev[i] = pv[i];
  for (int i = tid; i < nc; i += DF_THREADS) scur[i] = cv[i];
  __syncthreads();
#ifdef SPC_DEBUG  // both lists ascending, no duplicates, ids >= 0
  for (int i = tid; i < np; i += DF_THREADS) {
    SPC_DCHECK(sprev[i] >= 0, SPC_E_RANGE);
    SPC_DCHECK(i == 0 || sprev[i - 1] < sprev[i], SPC_E_STATE);
  }
  for (int i = tid; i < nc; i += DF_THREADS) {
    SPC_DCHECK(scur[i] >= 0, SPC_E_RANGE);
    SPC_DCHECK(i == 0 || scur[i - 1] < scur[i], SPC_E_STATE);
  }
#endif
  if (use_bm) {
    for (int i = tid; i < np; i += DF_THREADS) atomicOr(&bm_prev[sprev[i] >> 5], 1u << (sprev[i] & 31));
    for (int i = tid; i < nc; i += DF_THREADS) atomicOr(&bm_cur[scur[i] >> 5], 1u << (scur[i] & 31));
    __syncthreads();
  }
  auto in_prev = [&](int x) {
    if (x < 0 || x > maxtok) return false;
    return use_bm ? ((bm_prev[x >> 5] >> (x & 31)) & 1u) != 0u : contains(sprev, np, x);
  };
  auto in_cur = [&](int x) {
    if (x < 0 || x > maxtok) return false;
    return use_bm ? ((bm_cur[x >> 5] >> (x & 31)) & 1u) != 0u : contains(scur, nc, x);
  };
  const int per = (k + DF_THREADS - 1) / DF_THREADS;
  const int e0 = tid * per;

  // new = cur \ prev (ascending)
  int flag[DF_PER];
  int cnt = 0;
#pragma unroll
  for (int i = 0; i < DF_PER; ++i) {
    const int e = e0 + i;
    flag[i] = (i < per && e < nc) ? !in_prev(scur[e]) : 0;
    cnt += flag[i];
  }
  int pos = block_excl_scan(cnt, wsum, &total);
#pragma unroll
  for (int i = 0; i < DF_PER; ++i)
    if (flag[i]) snew[pos++] = scur[e0 + i];
  __syncthreads();
  const int nl = total;
  int32_t* lt = load_tok + (size_t)row * k;
  for (int i = tid; i < k; i += DF_THREADS) lt[i] = i < nl ? snew[i] : -1;
  if (tid == 0) n_load[row] = nl;

  // evicted = prev \ cur (ascending)
  if (evict_tok || n_evict) {
    cnt = 0;
#pragma unroll
    for (int i = 0; i < DF_PER; ++i) {
      const int e = e0 + i;
      flag[i] = (i < per && e < np) ? !in_cur(sprev[e]) : 0;
      cnt += flag[i];
    }
    pos = block_excl_scan(cnt, wsum, &total);
    if (evict_tok) {
      int32_t* et = evict_tok + (size_t)row * k;
#pragma unroll
      for (int i = 0; i < DF_PER; ++i)
        if (flag[i]) et[pos++] = sprev[e0 + i];
      for (int i = total + tid; i < k; i += DF_THREADS) et[i] = -1;
    }
    if (n_evict && tid == 0) n_evict[row] = total;
  }

  // slot reuse: freed slots (empty or token not in cur) in ascending slot order
  if (slot_tok) {
    int32_t* st = slot_tok + (size_t)row * k;
#ifdef SPC_DEBUG  // the non-empty slots hold exactly the previous set
    {
      int c = 0;
      for (int s2 = tid; s2 < k; s2 += DF_THREADS) {
        const int t2 = st[s2];
        if (t2 >= 0) {
          ++c;
          SPC_DCHECK(contains(sprev, np, t2), SPC_E_STATE);
        }
      }
      c = block_excl_scan(c, wsum, &total);
      (void)c;
      SPC_DCHECK(total == np, SPC_E_STATE);
    }
#endif
    int tok[DF_PER];
    cnt = 0;
#pragma unroll
    for (int i = 0; i < DF_PER; ++i) {
      const int s = e0 + i;
      tok[i] = (i < per && s < k) ? st[s] : -2;
      flag[i] = tok[i] != -2 && (tok[i] < 0 || !in_cur(tok[i]));
      cnt += flag[i];
    }
    pos = block_excl_scan(cnt, wsum, &total);
    SPC_DCHECK(total >= nl, SPC_E_BUDGET);  // #new <= #freed for consistent inputs (O8)
    int32_t* ls = load_slot + (size_t)row * k;
#pragma unroll
    for (int i = 0; i < DF_PER; ++i) {
      if (!flag[i]) continue;
      const int s = e0 + i;
      if (pos < nl) {
        st[s] = snew[pos];
        ls[pos] = s;
      } else {
        st[s] = -1;
      }
      ++pos;
    }
    for (int i = nl + tid; i < k; i += DF_THREADS) ls[i] = -1;
  }
}

// ------------------------------------------------------------------ gather (O9)
template <typename VecT>
__global__ void __launch_bounds__(256) gather_kernel(
    const void* const* __restrict__ k_src, const void* const* __restrict__ v_src, int B, int G,
    int Smax, int kbud, int row_vecs, int layer_begin, const int32_t* __restrict__ load_tok,
    const int32_t* __restrict__ load_slot, const int32_t* __restrict__ n_load,
    void* const* __restrict__ k_buf, void* const* __restrict__ v_buf) {
  spc_pdl_entry();
  // grid: x = chunks of the budget, y strides over the B*G rows, z = layer
  const int l = layer_begin + blockIdx.z;
  const int lanes_per_row = row_vecs;  // 16-byte vectors per row (8 or 16)
  const int rows_per_block = blockDim.x / lanes_per_row;
  const int sub = threadIdx.x / lanes_per_row, lane = threadIdx.x % lanes_per_row;
  const VecT* ks = (const VecT*)k_src[l];
  const VecT* vs = (const VecT*)v_src[l];
  VecT* kd = (VecT*)k_buf[l];
  VecT* vd = (VecT*)v_buf[l];
  for (int bg = blockIdx.y; bg < B * G; bg += gridDim.y) {
    const int n = n_load[bg];
    const size_t src_base = (size_t)bg * Smax * row_vecs, dst_base = (size_t)bg * kbud * row_vecs;
    for (int i = blockIdx.x * rows_per_block + sub; i < n; i += gridDim.x * rows_per_block) {
      const int t = load_tok[(size_t)bg * kbud + i];
      const int s = load_slot[(size_t)bg * kbud + i];
#ifdef SPC_DEBUG  // an index out of range is an error (skipped, not read)
      SPC_DCHECK(t >= 0 && t < Smax && s >= 0 && s < kbud, SPC_E_RANGE);
      if (t < 0 || t >= Smax || s < 0 || s >= kbud) continue;
#endif
      const VecT a = ks[src_base + (size_t)t * row_vecs + lane];
      const VecT b = vs[src_base + (size_t)t * row_vecs + lane];
      kd[dst_base + (size_t)s * row_vecs + lane] = a;
      vd[dst_base + (size_t)s * row_vecs + lane] = b;
    }
  }
}

// Strided / token-major gather (spc_gather_kv_strided): one warp per (b*G+g, i); the
// warp walks the layers of token load_tok[i], SPC_GT_UNR layers in flight per lane.
// A bf16 D = 128 row pair (K + V) is 512 bytes: lanes 0-15 move the K row, 16-31 the V
// row, 16 bytes each.  With a token-major source ([.][tok][L][2][D]) the whole walk reads
// one contiguous record: over PCIe one address translation per record instead of one per
// 256-byte row (random 256-byte rows of 32 GB of pinned memory: 12-30 GB/s; 16 KiB
// records: 51 GB/s of the 55 GB/s DMA copy, tools/pciegather.cu).
constexpr int GT_WARPS = 8;
#ifndef SPC_GT_UNR
#define SPC_GT_UNR 8
#endif
__global__ void __launch_bounds__(GT_WARPS * 32) gather_strided_kernel(
    const void* const* __restrict__ k_src, const void* const* __restrict__ v_src,
    long long row_stride, long long bg_stride, int kbud, int vpr, int layer_begin, int nl,
    const int32_t* __restrict__ load_tok, const int32_t* __restrict__ load_slot,
    const int32_t* __restrict__ n_load, void* const* __restrict__ k_buf,
    void* const* __restrict__ v_buf) {
  spc_pdl_entry();
  const int bg = blockIdx.y, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = n_load[bg];
  const int rpw = 32 / (2 * vpr);             // token rows (K + V pairs) per warp pass: 1 or 2
  const int sub = lane / (2 * vpr), r = lane % (2 * vpr);
  const bool isv = r >= vpr;
  const int vec = isv ? r - vpr : r;
  const int tpb = GT_WARPS * rpw;
  for (int i0 = blockIdx.x * tpb; i0 < n; i0 += gridDim.x * tpb) {
    const int i = i0 + warp * rpw + sub;
    if (i >= n) continue;
    const long long t = load_tok[(size_t)bg * kbud + i];
    const long long s = load_slot[(size_t)bg * kbud + i];
#ifdef SPC_DEBUG
    SPC_DCHECK(t >= 0 && s >= 0 && s < kbud, SPC_E_RANGE);
    if (t < 0 || s < 0 || s >= kbud) continue;
#endif
    const size_t soff = (size_t)(bg * bg_stride + t * row_stride) * 2 / 16 + vec;  // 16-B units
    const size_t doff = ((size_t)bg * kbud + s) * vpr + vec;
    for (int l0 = 0; l0 < nl; l0 += SPC_GT_UNR) {
      uint4 x[SPC_GT_UNR];
#pragma unroll
      for (int u = 0; u < SPC_GT_UNR; ++u)
        if (l0 + u < nl) {
          const uint4* src = (const uint4*)(isv ? v_src[layer_begin + l0 + u] : k_src[layer_begin + l0 + u]);
          x[u] = __ldcs(src + soff);
        }
#pragma unroll
      for (int u = 0; u < SPC_GT_UNR; ++u)
        if (l0 + u < nl) {
          uint4* dst = (uint4*)(isv ? v_buf[layer_begin + l0 + u] : k_buf[layer_begin + l0 + u]);
          dst[doff] = x[u];
        }
    }
  }
}

}  // namespace
}  // namespace spc

using namespace spc;

extern "C" int spc_elastic_diff(const int32_t* prev_idx, const int32_t* prev_count,
                                const int32_t* cur_idx, const int32_t* cur_count, int B, int G,
                                int k, int32_t* slot_tok, int32_t* load_tok, int32_t* load_slot,
                                int32_t* n_load, int32_t* evict_tok, int32_t* n_evict,
                                spc_stream_t stream) {
  if (!prev_idx || !prev_count || !cur_idx || !cur_count || !load_tok || !n_load) return SPC_E_NULL;
  if (slot_tok && !load_slot) return SPC_E_NULL;
  if (B <= 0 || G <= 0) return SPC_E_SHAPE;
  if (k < 1 || k > SPC_MAX_K) return SPC_E_BUDGET;
  const size_t smem = sizeof(int32_t) * 3 * (size_t)k + sizeof(uint32_t) * 2 * DF_BM_WORDS;
  SPC_TRY(smem_attr((const void*)diff_kernel,
                    (int)(sizeof(int32_t) * 3 * SPC_MAX_K + sizeof(uint32_t) * 2 * DF_BM_WORDS)));
  return launched(launch_k(diff_kernel, dim3(B * G), dim3(DF_THREADS), smem, as_stream(stream),
                           prev_idx, prev_count, cur_idx, cur_count, k, slot_tok, load_tok,
                           load_slot, n_load, evict_tok, n_evict));
}

// CTAs of one gather launch (env SPC_GATHER_CTAS overrides, tools): the strided gather
// half the SMs (config D's prefetch groups, measured); the layer-major one 32 CTAs of 256
// threads -- 256 KB of zero-copy loads in flight already reach the PCIe rate, and llm.py's
// per-layer prefetch measured 8.69 ms serial / 5.65 ms overlapped at 32 CTAs vs 6.50 at 64
// and 7.44 at 128 (the gather's CTAs take SMs from the dense layers it overlaps)
static int gather_cap(int dflt) {
  static const int cap_env = [] {
    const char* e = std::getenv("SPC_GATHER_CTAS");
    return e ? std::atoi(e) : 0;
  }();
  return cap_env > 0 ? cap_env : dflt;
}

extern "C" int spc_gather_kv(int dtype, const void* const* k_src, const void* const* v_src, int L,
                             int B, int G, int D, int Smax, int k, int layer_begin, int layer_end,
                             const int32_t* load_tok, const int32_t* load_slot,
                             const int32_t* n_load, void* const* k_buf, void* const* v_buf,
                             spc_stream_t stream) {
  if (!k_src || !v_src || !load_tok || !load_slot || !n_load || !k_buf || !v_buf) return SPC_E_NULL;
  if (L <= 0 || B <= 0 || G <= 0 || Smax <= 0) return SPC_E_SHAPE;
  if (k < 1 || k > SPC_MAX_K) return SPC_E_BUDGET;
  if (layer_begin < 0 || layer_end > L || layer_begin > layer_end) return SPC_E_RANGE;
  if (layer_begin == layer_end) return SPC_OK;
  const int esz = dtype == SPC_BF16 ? 2 : (dtype == SPC_F32 ? 4 : 0);
  if (!esz) return SPC_E_UNSUPPORTED;
  if ((D * esz) % 16 || D * esz / 16 > 32 || 32 % (D * esz / 16)) return SPC_E_UNSUPPORTED;
  const int row_vecs = D * esz / 16;
  // grid capped like the strided gather's (gather_cap): a PCIe-bound copy needs a few hundred
  // KB in flight, not the whole GPU, and the rest of the SMs stay free for the compute it
  // overlaps (DecodeStep's prefetch groups, llm.py's per-layer prefetch)
  const int nl = layer_end - layer_begin;
  const int cap = std::max(nl, gather_cap(32));
  const int ny = std::max(1, std::min(B * G, cap / nl));
  const int nx = std::max(1, std::min((k + 63) / 64, cap / (ny * nl)));
  dim3 grid((unsigned)nx, (unsigned)ny, nl);
  return launched(launch_k(gather_kernel<uint4>, grid, dim3(256), 0, as_stream(stream), k_src,
                           v_src, B, G, Smax, k, row_vecs, layer_begin, load_tok, load_slot,
                           n_load, k_buf, v_buf));
}

extern "C" int spc_gather_kv_strided(int dtype, const void* const* k_src, const void* const* v_src,
                                     long long row_stride, long long bg_stride, int L, int B, int G,
                                     int D, int k, int layer_begin, int layer_end,
                                     const int32_t* load_tok, const int32_t* load_slot,
                                     const int32_t* n_load, void* const* k_buf, void* const* v_buf,
                                     spc_stream_t stream) {
  if (!k_src || !v_src || !load_tok || !load_slot || !n_load || !k_buf || !v_buf) return SPC_E_NULL;
  if (L <= 0 || B <= 0 || G <= 0 || D <= 0 || row_stride < D || bg_stride < 0) return SPC_E_SHAPE;
  if (k < 1 || k > SPC_MAX_K) return SPC_E_BUDGET;
  if (layer_begin < 0 || layer_end > L || layer_begin > layer_end) return SPC_E_RANGE;
  if (layer_begin == layer_end) return SPC_OK;
  if (dtype != SPC_BF16) return SPC_E_UNSUPPORTED;
  const int vpr = D * 2 / 16;  // 16-byte vectors per row
  if (!(vpr == 8 || vpr == 16) || (row_stride * 2) % 16 || (bg_stride * 2) % 16)
    return SPC_E_UNSUPPORTED;
  const int tpb = GT_WARPS * (32 / (2 * vpr));
  // PCIe-bound: a few MB in flight saturate the link, so the grid is capped at half the SMs
  // in total -- the other half stays free for the attention of the previous layer group
  // (the prefetch pipeline of DecodeStep); env SPC_GATHER_CTAS overrides (tools)
  const int cap = gather_cap(std::max(1, num_sms() / 2));
  const int nx = std::max(1, std::min((k + tpb - 1) / tpb, (cap + B * G - 1) / (B * G)));
  dim3 grid((unsigned)nx, B * G);
  return launched(launch_k(gather_strided_kernel, grid, dim3(GT_WARPS * 32), 0,
                           as_stream(stream), k_src, v_src, row_stride, bg_stride, k, vpr,
                           layer_begin, layer_end - layer_begin, load_tok, load_slot, n_load,
                           k_buf, v_buf));
}
