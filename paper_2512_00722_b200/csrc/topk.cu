// topk.cu — spc_topk / spc_topk_merge / spc_topk_filter: O7 and O13.
//
// Paper: "select the Top-K candidates" per KV group (head-level
// retrieval), budget k = 2048.  Order (R8):
// value descending, global id ascending, realised by the 64-bit composite key
// (bits(v) << 32) | ~uint32(id) — values are >= 0 so float bits order like
// unsigned integers (R20).  The k-th largest composite T is found by radix
// select; the selection is then exactly {x : composite(x) >= T}.
//
// spc_topk: ONE kernel, one thread-block cluster of CL = 8 CTAs per row.  Each
// CTA owns a contiguous 1/8 of the row.
//   1. 2048-bin histogram of the top 11 key bits per CTA (shared atomics);
//      every CTA sums the 8 histograms through distributed shared memory and
//      finds the threshold bin and the residual rank redundantly.
//   2. while more than CAND_CAP elements share the prefix: another 8-bit digit
//      (distributed histogram over the elements matching the prefix).
//   3. the matching elements are gathered into CTA 0's shared memory (DSMEM,
//      warp-aggregated slot claims), radix-refined there to T, and T is
//      broadcast to the cluster.
//   4. ordered compaction: each CTA counts its elements >= T, the counts are
//      exchanged through DSMEM, and each CTA writes its positions ascending at
//      its offset.  No workspace, no global atomics, no extra launches.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace spc {
namespace {

constexpr int NBIN0 = 2048;     // top digit: 11 bits of the composite
constexpr int CAND_CAP = 8192;  // candidates refined in shared memory
constexpr int SEL_THREADS = 1024;
constexpr int RANK_MAX = 128;   // rank by counting (O(n^2)) only below this many candidates
constexpr int CL = 8;           // CTAs per row (cluster size)

// composite of position p of a dense row
__device__ __forceinline__ unsigned long long row_key(const float* row, int p, int len, int force,
                                                      int stride, int offset) {
  uint32_t vb = (force && p == len - 1) ? 0x7F800000u : __float_as_uint(__ldg(row + p));
  return composite(vb, p * stride + offset);
}

__device__ __forceinline__ int row_len(const int32_t* seq_len, int row, int G, int n_cols) {
  int s = seq_len[row / G];
  return s < n_cols ? (s < 0 ? 0 : s) : n_cols;
}

// Warp-cooperative search from the top bin down: returns (bin, above) with
// above = sum of counts of bins > bin, above < r <= above + h[bin].
template <int NB>
__device__ __forceinline__ void find_bin_warp(const unsigned* h, int r, int* bin_out,
                                              int* above_out) {
  constexpr int PER = NB / 32;
  const int lane = threadIdx.x & 31;
  const int hi = NB - 1 - lane * PER;  // this lane owns bins hi .. hi-PER+1
  unsigned s = 0;
#pragma unroll 8
  for (int i = 0; i < PER; ++i) s += h[hi - i];
  unsigned incl = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  const unsigned ballot = __ballot_sync(0xffffffffu, incl >= (unsigned)r);
  const int L = __ffs(ballot) - 1;  // first lane whose cumulative count reaches r
  unsigned before = __shfl_sync(0xffffffffu, incl - s, L);
  if (lane == L) {
    unsigned run = before;
    int b = hi;
    for (int i = 0; i < PER; ++i) {
      b = hi - i;
      if (run + h[b] >= (unsigned)r) break;
      run += h[b];
    }
    *bin_out = b;
    *above_out = (int)run;
  }
  __syncwarp();
}

// --------------------------------------------------------------- selection core
// Shared-memory state of one selecting CTA.
struct SelSmem {
  unsigned long long cand[2][CAND_CAP];
  unsigned hist[256];
  int n[2];
  int bin, above;
  unsigned long long T;
  int wsum[SEL_THREADS / 32];
};

// r-th largest among the cm composites in s.cand[cur][0..cm), all sharing the
// top `bits` bits.  Radix passes of 8 bits until cm <= RANK_MAX, then rank by
// counting.  Returns T in s.T (valid after the final __syncthreads).
__device__ void refine_in_smem(SelSmem& s, int cur, int cm, int r, int bits) {
  const int tid = threadIdx.x;
  while (cm > RANK_MAX && bits < 64) {
    const int db = (64 - bits) < 8 ? (64 - bits) : 8;
    const int shift = 64 - bits - db;
    const unsigned mask = (1u << db) - 1;
    for (int i = tid; i < 256; i += SEL_THREADS) s.hist[i] = 0;
    if (tid == 0) s.n[cur ^ 1] = 0;
    __syncthreads();
    for (int i = tid; i < cm; i += SEL_THREADS)
      atomicAdd(&s.hist[(unsigned)(s.cand[cur][i] >> shift) & mask], 1u);
    __syncthreads();
    if (tid < 32) find_bin_warp<256>(s.hist, r, &s.bin, &s.above);
    __syncthreads();
    const unsigned b = (unsigned)s.bin;
    for (int i = tid; i < cm; i += SEL_THREADS) {
      const unsigned long long x = s.cand[cur][i];
      if (((unsigned)(x >> shift) & mask) == b) s.cand[cur ^ 1][atomicAdd(&s.n[cur ^ 1], 1)] = x;
    }
    r -= s.above;
    bits += db;
    __syncthreads();
    cm = s.n[cur ^ 1];
    cur ^= 1;
  }
  // rank by counting: exactly one candidate has r-1 larger ones (composites unique)
  for (int i = tid; i < cm; i += SEL_THREADS) {
    const unsigned long long x = s.cand[cur][i];
    int larger = 0;
    for (int j = 0; j < cm; ++j) larger += s.cand[cur][j] > x;
    if (larger == r - 1) s.T = x;
  }
  __syncthreads();
}

__device__ __forceinline__ bool prefix_match(unsigned long long x, unsigned long long prefix, int bits) {
  return bits == 0 || (x >> (64 - bits)) == (prefix >> (64 - bits));
}

// Row-scan refinement for degenerate rows (threshold bin > CAND_CAP): narrow
// the prefix with 8-bit passes over the row until at most CAND_CAP elements
// match, then collect them into shared memory.  Returns (cm, r, bits) updated.
template <class KeyFn>
__device__ void narrow_by_row_scan(SelSmem& s, const KeyFn& key, int len, unsigned long long& prefix,
                                   int& bits, int& r, int& cm) {
  const int tid = threadIdx.x;
  while (cm > CAND_CAP && bits < 64) {
    const int db = (64 - bits) < 8 ? (64 - bits) : 8;
    const int shift = 64 - bits - db;
    const unsigned mask = (1u << db) - 1;
    for (int i = tid; i < 256; i += SEL_THREADS) s.hist[i] = 0;
    __syncthreads();
    for (int p = tid; p < len; p += SEL_THREADS) {
      const unsigned long long x = key(p);
      if (prefix_match(x, prefix, bits)) atomicAdd(&s.hist[(unsigned)(x >> shift) & mask], 1u);
    }
    __syncthreads();
    if (tid < 32) find_bin_warp<256>(s.hist, r, &s.bin, &s.above);
    __syncthreads();
    r -= s.above;
    cm = (int)s.hist[s.bin];
    prefix |= (unsigned long long)s.bin << shift;
    bits += db;
    __syncthreads();
  }
  if (tid == 0) s.n[0] = 0;
  __syncthreads();
  for (int p = tid; p < len; p += SEL_THREADS) {
    const unsigned long long x = key(p);
    if (prefix_match(x, prefix, bits)) s.cand[0][atomicAdd(&s.n[0], 1)] = x;
  }
  __syncthreads();
}

struct DenseKey {
  const float* row;
  int len, force, stride, offset;
  bool vec;  // row 16-byte aligned: quad() reads one float4 (p is a multiple of 4)
  __device__ unsigned long long operator()(int p) const {
    return row_key(row, p, len, force, stride, offset);
  }
  // the raw quad at p (vec rows) and its keys: scans load several quads before using any
  __device__ __forceinline__ float4 raw(int p) const {
    return __ldg(reinterpret_cast<const float4*>(row + p));
  }
  __device__ __forceinline__ void keys(const float4& v, int p, unsigned long long (&x)[4]) const {
    const float vs[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t vb = (force && p + i == len - 1) ? 0x7F800000u : __float_as_uint(vs[i]);
      x[i] = composite(vb, (p + i) * stride + offset);
    }
  }
  // keys of positions p .. p+3 (p a multiple of 4; positions >= len are never used)
  __device__ __forceinline__ void quad(int p, unsigned long long (&x)[4]) const {
    if (vec) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(row + p));
      const float vs[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t vb = (force && p + i == len - 1) ? 0x7F800000u : __float_as_uint(vs[i]);
        x[i] = composite(vb, (p + i) * stride + offset);
      }
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) x[i] = p + i < len ? row_key(row, p + i, len, force, stride, offset) : 0ull;
    }
  }
};

// f(p, x) for the quads p = a, a + st, a + 2 st, ... < b (x = keys of p .. p+3): SCAN_UNR
// quads' loads are issued before the first is used -- a row pass issued one dependent
// float4 load per quad and waited on each (config E's 1M-token rows: 32 quads per thread,
// ncu: 42% of the top-k's stall samples on those loads)
constexpr int SCAN_UNR = 4;
template <class KeyFn, class F>
__device__ __forceinline__ void scan_quads(const KeyFn& key, int a, int b, int st, F&& f) {
  if (key.vec) {
    for (int p0 = a; p0 < b; p0 += st * SCAN_UNR) {
      float4 v[SCAN_UNR];
#pragma unroll
      for (int u = 0; u < SCAN_UNR; ++u)
        if (p0 + u * st < b) v[u] = key.raw(p0 + u * st);
#pragma unroll
      for (int u = 0; u < SCAN_UNR; ++u) {
        const int p = p0 + u * st;
        if (p < b) {
          unsigned long long x[4];
          key.keys(v[u], p, x);
          f(p, x);
        }
      }
    }
  } else {
    for (int p = a; p < b; p += st) {
      unsigned long long x[4];
      key.quad(p, x);
      f(p, x);
    }
  }
}

struct ClSmem {
  SelSmem sel;               // CTA 0: gathered candidates + refinement scratch
  unsigned hist[NBIN0];      // this CTA's histogram (read remotely by the cluster)
  unsigned rhist[NBIN0];     // cluster-reduced histogram
  unsigned long long T;      // broadcast threshold
  int counts[CL];            // selected elements per cluster rank
  int total;
};

// The selection of one row by a cluster: every CTA passes the key functor for its
// own segment [s0, s1) of the row (key(p) is only called for p in the segment).
// Writes out_idx/out_val/out_count/out_thresh of the row; returns this CTA's
// offset and number of selected positions (its part of the ascending list).
template <class KeyFn>
__device__ void cluster_select(ClSmem& s, cg::cluster_group& cl, const KeyFn& key, int len, int k,
                               int s0, int s1, int32_t* oi, float* ov, int32_t* out_count,
                               unsigned long long* out_thresh, int* my_base, int* my_count) {
  const int rank = (int)cl.block_rank();
  const int tid = threadIdx.x, lane = tid & 31;
  const int need = k < len ? k : len;
  unsigned long long T = 0;
  if (need < len) {
    // ---- 1. top-11-bit histogram, reduced over the cluster
    for (int i = tid; i < NBIN0; i += SEL_THREADS) s.hist[i] = 0;
    __syncthreads();
    scan_quads(key, s0 + 4 * tid, s1, 4 * SEL_THREADS, [&](int p, const unsigned long long(&x)[4]) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (p + i < s1) atomicAdd(&s.hist[x[i] >> 53], 1u);
    });
    cl.sync();
    for (int i = tid; i < NBIN0; i += SEL_THREADS) {
      unsigned t = 0;
#pragma unroll
      for (int r = 0; r < CL; ++r) t += cl.map_shared_rank(s.hist, r)[i];
      s.rhist[i] = t;
    }
    __syncthreads();
    if (tid < 32) find_bin_warp<NBIN0>(s.rhist, need, &s.sel.bin, &s.sel.above);
    __syncthreads();
    int r = need - s.sel.above, cm = (int)s.rhist[s.sel.bin], bits = 11;
    unsigned long long prefix = (unsigned long long)s.sel.bin << 53;
    cl.sync();  // remote reads of s.hist done before it is reused
    // ---- 2. distributed refinement while too many elements share the prefix
    while (cm > CAND_CAP && bits < 64) {
      const int db = (64 - bits) < 8 ? (64 - bits) : 8;
      const int shift = 64 - bits - db;
      const unsigned mask = (1u << db) - 1;
      for (int i = tid; i < 256; i += SEL_THREADS) s.hist[i] = 0;
      __syncthreads();
      scan_quads(key, s0 + 4 * tid, s1, 4 * SEL_THREADS, [&](int p, const unsigned long long(&x)[4]) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (p + i < s1 && prefix_match(x[i], prefix, bits))
            atomicAdd(&s.hist[(unsigned)(x[i] >> shift) & mask], 1u);
      });
      cl.sync();
      for (int i = tid; i < 256; i += SEL_THREADS) {
        unsigned t = 0;
#pragma unroll
        for (int q = 0; q < CL; ++q) t += cl.map_shared_rank(s.hist, q)[i];
        s.rhist[i] = t;
      }
      __syncthreads();
      if (tid < 32) find_bin_warp<256>(s.rhist, r, &s.sel.bin, &s.sel.above);
      __syncthreads();
      r -= s.sel.above;
      cm = (int)s.rhist[s.sel.bin];
      prefix |= (unsigned long long)s.sel.bin << shift;
      bits += db;
      cl.sync();
    }
    // ---- 3. gather the matching elements into CTA 0 and refine there
    if (rank == 0 && tid == 0) s.sel.n[0] = 0;
    cl.sync();
    int* n0 = cl.map_shared_rank(&s.sel.n[0], 0);
    unsigned long long* c0 = cl.map_shared_rank(&s.sel.cand[0][0], 0);
    for (int p00 = s0; p00 < s1; p00 += 4 * SEL_THREADS * SCAN_UNR) {  // warp-uniform trips
      float4 v[SCAN_UNR];
#pragma unroll
      for (int u = 0; u < SCAN_UNR; ++u) {  // every quad's load in flight first
        const int p = p00 + u * 4 * SEL_THREADS + 4 * tid;
        if (key.vec && p < s1) v[u] = key.raw(p);
      }
#pragma unroll
      for (int u = 0; u < SCAN_UNR; ++u) {
        const int p = p00 + u * 4 * SEL_THREADS + 4 * tid;
        unsigned long long x[4] = {0, 0, 0, 0};
        if (p < s1) {
          if (key.vec) key.keys(v[u], p, x);
          else key.quad(p, x);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const bool hit = p + i < s1 && prefix_match(x[i], prefix, bits);
          const unsigned m = __ballot_sync(0xffffffffu, hit);
          if (!m) continue;
          const int leader = __ffs(m) - 1;
          int base = 0;
          if (lane == leader) base = atomicAdd(n0, __popc(m));
          base = __shfl_sync(0xffffffffu, base, leader);
          if (hit) c0[base + __popc(m & ((1u << lane) - 1))] = x[i];
        }
      }
    }
    cl.sync();
    if (rank == 0) {
      refine_in_smem(s.sel, 0, s.sel.n[0], r, bits);
      if (tid < CL) *cl.map_shared_rank(&s.T, tid) = s.sel.T;
    }
    cl.sync();
    T = s.T;
  } else {
    cl.sync();  // no cut: every CTA must have started before the remote writes below
  }
  // ---- 4. ordered compaction over the cluster
  const int seg = s1 - s0;
  const int pt = ((seg + SEL_THREADS - 1) / SEL_THREADS + 3) & ~3;  // multiple of 4
  const int q0 = min(s1, s0 + tid * pt), q1 = min(s1, q0 + pt);
  int cnt = 0;
  scan_quads(key, q0, q1, 4, [&](int p, const unsigned long long(&x)[4]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) cnt += (p + i < q1 && x[i] >= T);
  });
  int pos = block_excl_scan(cnt, s.sel.wsum, &s.total);
  __syncthreads();
  if (tid < CL) cl.map_shared_rank(s.counts, tid)[rank] = s.total;
  cl.sync();
  int base = 0, all = 0;
#pragma unroll
  for (int q = 0; q < CL; ++q) {
    base += q < rank ? s.counts[q] : 0;
    all += s.counts[q];
  }
  *my_base = base;
  *my_count = s.counts[rank];
  pos += base;
  scan_quads(key, q0, q1, 4, [&](int p, const unsigned long long(&x)[4]) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (p + i < q1 && x[i] >= T) {
        oi[pos] = p + i;
        if (ov) ov[pos] = __uint_as_float((uint32_t)(x[i] >> 32));
        ++pos;
      }
  });
  if (rank == CL - 1)
    for (int i = all + tid; i < k; i += SEL_THREADS) {
      oi[i] = -1;
      if (ov) ov[i] = 0.0f;
    }
  if (rank == 0 && tid == 0) {
    *out_count = all;
    if (out_thresh) *out_thresh = need < len ? T : 0ull;
  }
}

__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(SEL_THREADS, 1)
    topk_cluster_kernel(const float* __restrict__ val, const int32_t* __restrict__ seq_len, int G,
                        int n_cols, int k, int force, int stride, int offset,
                        int32_t* __restrict__ out_idx, float* __restrict__ out_val,
                        int32_t* __restrict__ out_count, unsigned long long* __restrict__ out_thresh) {
  spc_pdl_entry();
  extern __shared__ __align__(16) uint8_t cl_raw[];
  ClSmem& s = *reinterpret_cast<ClSmem*>(cl_raw);
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int row = blockIdx.y;
  const int len = row_len(seq_len, row, G, n_cols);
  const float* rowp = val + (size_t)row * n_cols;
  const DenseKey key{rowp, len, force, stride, offset,
                     (n_cols & 3) == 0 && ((uintptr_t)rowp & 15) == 0};
  const int per = ((len + CL - 1) / CL + 3) & ~3;  // multiple of 4: quads never straddle
  const int s0 = min(len, rank * per), s1 = min(len, s0 + per);
  int my_base, my_count;
  cluster_select(s, cl, key, len, k, s0, s1, out_idx + (size_t)row * k,
                 out_val ? out_val + (size_t)row * k : nullptr, out_count + row,
                 out_thresh ? out_thresh + row : nullptr, &my_base, &my_count);
}

// ------------------------------------------------------------------ merge (O13)
struct UnionKey {
  const float* val;
  const int32_t* pos;
  const int* off;  // prefix offsets per shard (shared memory), P+1 entries
  int P, R, k, row;
  __device__ unsigned long long operator()(int i) const {
    int p = 0;
    while (i >= off[p + 1]) ++p;
    const size_t e = ((size_t)p * R + row) * k + (i - off[p]);
    return composite(__float_as_uint(val[e]), pos[e] * P + p);
  }
};

__global__ void __launch_bounds__(SEL_THREADS, 1) merge_kernel(
    const float* __restrict__ cval, const int32_t* __restrict__ cpos,
    const int32_t* __restrict__ ccnt, int P, int R, int k,
    unsigned long long* __restrict__ out_thresh) {
  spc_pdl_entry();
  extern __shared__ __align__(16) uint8_t sel_raw[];
  SelSmem& s = *reinterpret_cast<SelSmem*>(sel_raw);
  __shared__ int off[65];
  const int row = blockIdx.x, tid = threadIdx.x;
  if (tid == 0) {
    off[0] = 0;
    for (int p = 0; p < P; ++p) off[p + 1] = off[p] + min(ccnt[(size_t)p * R + row], k);
  }
  __syncthreads();
  const int n = off[P];
  if (n <= k) {
    if (tid == 0) out_thresh[row] = 0ull;
    return;
  }
  UnionKey key{cval, cpos, off, P, R, k, row};
  unsigned long long prefix = 0;
  int bits = 0, r = k, cm = n;
  narrow_by_row_scan(s, key, n, prefix, bits, r, cm);
  refine_in_smem(s, 0, s.n[0], r, bits);
  if (tid == 0) out_thresh[row] = s.T;
}

// ------------------------------------------------------------------ filter (O13)
__global__ void __launch_bounds__(SEL_THREADS) filter_kernel(
    int32_t* __restrict__ idx, const float* __restrict__ val, int32_t* __restrict__ count,
    const unsigned long long* __restrict__ thresh, int k, int stride, int offset) {
  spc_pdl_entry();
  __shared__ int wsum[SEL_THREADS / 32];
  __shared__ int total;
  const int row = blockIdx.x, tid = threadIdx.x;
  const int n = count[row];
  const unsigned long long T = thresh[row];
  constexpr int MAXPER = SPC_MAX_K / SEL_THREADS;
  int keep[MAXPER];
  int nk = 0;
  const int per = (k + SEL_THREADS - 1) / SEL_THREADS;
  const int p0 = tid * per;
#pragma unroll
  for (int i = 0; i < MAXPER; ++i) {
    const int p = p0 + i;
    keep[i] = -1;
    if (i < per && p < n) {
      const int id = idx[(size_t)row * k + p];
      const unsigned long long x =
          composite(__float_as_uint(val[(size_t)row * k + p]), id * stride + offset);
      if (x >= T) {
        keep[i] = id;
        ++nk;
      }
    }
  }
  int pos = block_excl_scan(nk, wsum, &total);
  __syncthreads();  // every read of idx happened before any write below
#pragma unroll
  for (int i = 0; i < MAXPER; ++i)
    if (keep[i] >= 0) idx[(size_t)row * k + pos++] = keep[i];
  __syncthreads();
  for (int i = total + tid; i < k; i += SEL_THREADS) idx[(size_t)row * k + i] = -1;
  if (tid == 0) count[row] = total;
}


}  // namespace
}  // namespace spc

using namespace spc;

extern "C" size_t spc_topk_workspace(int B, int G, int n_cols, int k) {
  (void)n_cols;
  (void)k;
  if (B <= 0 || G <= 0) return 0;
  return 256;  // the cluster kernel needs no global scratch
}

extern "C" int spc_topk(const float* val, const int32_t* seq_len, int B, int G, int n_cols, int k,
                        int force_last, int id_stride, int id_offset, int32_t* out_idx,
                        float* out_val, int32_t* out_count, uint64_t* out_thresh, void* ws,
                        size_t ws_bytes, spc_stream_t stream) {
  (void)ws;
  (void)ws_bytes;
  if (!val || !seq_len || !out_idx || !out_count) return SPC_E_NULL;
  if (B <= 0 || G <= 0 || n_cols <= 0) return SPC_E_SHAPE;
  if (k < 1 || k > SPC_MAX_K) return SPC_E_BUDGET;
  if (n_cols >= SPC_MAX_SEQ || id_stride < 1 || id_offset < 0) return SPC_E_RANGE;
  if ((long long)n_cols * id_stride + id_offset >= 0x7FFFFFFFLL) return SPC_E_RANGE;
  SPC_TRY(smem_attr((const void*)topk_cluster_kernel, (int)sizeof(ClSmem)));
  return launched(launch_k(topk_cluster_kernel, dim3(CL, B * G), dim3(SEL_THREADS),
                           sizeof(ClSmem), as_stream(stream), val, seq_len, G, n_cols, k,
                           force_last, id_stride, id_offset, out_idx, out_val, out_count,
                           (unsigned long long*)out_thresh));
}

extern "C" size_t spc_topk_merge_workspace(int P, int R, int k) {
  (void)P;
  (void)R;
  (void)k;
  return 256;
}

extern "C" int spc_topk_merge(const float* cand_val, const int32_t* cand_pos,
                              const int32_t* cand_count, int P, int R, int k, uint64_t* out_thresh,
                              void* ws, size_t ws_bytes, spc_stream_t stream) {
  (void)ws;
  (void)ws_bytes;
  if (!cand_val || !cand_pos || !cand_count || !out_thresh) return SPC_E_NULL;
  if (P < 1 || P > 64 || R < 1) return SPC_E_SHAPE;
  if (k < 1 || k > SPC_MAX_K) return SPC_E_BUDGET;
  SPC_TRY(smem_attr((const void*)merge_kernel, (int)sizeof(SelSmem)));
  return launched(launch_k(merge_kernel, dim3(R), dim3(SEL_THREADS), sizeof(SelSmem),
                           as_stream(stream), cand_val, cand_pos, cand_count, P, R, k,
                           (unsigned long long*)out_thresh));
}

extern "C" int spc_topk_filter(int32_t* idx, const float* val, int32_t* count,
                               const uint64_t* thresh, int R, int k, int id_stride, int id_offset,
                               spc_stream_t stream) {
  if (!idx || !val || !count || !thresh) return SPC_E_NULL;
  if (R < 1) return SPC_E_SHAPE;
  if (k < 1 || k > SPC_MAX_K) return SPC_E_BUDGET;
  return launched(launch_k(filter_kernel, dim3(R), dim3(SEL_THREADS), 0, as_stream(stream), idx,
                           val, count, (const unsigned long long*)thresh, k, id_stride,
                           id_offset));
}
