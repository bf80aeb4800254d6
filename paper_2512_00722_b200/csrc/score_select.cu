// score_select.cu — spc_score_select: the whole selection of one decode step in ONE
// persistent launch: LOGITS (O1, O2), NORM (O3, O4), GROUP (O5, O6), top-k (O7) and the
// INDEXED elastic diff (O8).  Definitions: DESIGN.md §3 (Eq.1 P:228-231 softmax of the
// retrieval head over its key cache; GQA group max P:328; "select the Top-K candidates"
// P:267; S_now - S_last P:374).  Bit-identical to spc_score(LOGITS) + spc_select.
//
// Why one kernel: the separate launches spend most of their time in ramps, tails and
// dependent round trips -- LOGITS' last tiles, its finalize launch, and spc_select's
// eight-CTA cluster phases on 64 SMs (~15 us in-kernel).  Here every SM keeps the logits
// of its own key tiles in shared memory and the phases are separated by three grid-wide
// barriers and one per-row hand-off:
//   A  LOGITS: one TMA producer warp + SS_NC consumer warps per CTA (logits_tma_kernel's
//      pipeline, a ring of stages per consumer warp); CTA c owns the contiguous key tiles [c n / N, (c+1) n / N) -- at most
//      SS_TPC tiles of 128 tokens, within at most two (b, g) rows ("slots").  The
//      logits go to shared memory; per-(row, head) maxima -> global atomicMax on an
//      order-preserving integer encoding (exact).                         grid barrier 1
//   B  NORM: e = spc_exp(s - m) over the CTA's tokens (kept in shared memory), int64
//      fixed-point sums -> global 64-bit atomicAdd (exact, order-free).    grid barrier 2
//   C  GROUP: r = 1 / (F 2^-40), gs = max_j e_j r_j into shared memory and group_score;
//      the pass-0 radix histogram (256-bin window, 8 bins per binade, anchored at the
//      exact row maximum max_j r_j) -> global per-row histogram.          grid barrier 3
//   D  every CTA finds the threshold bin of its rows; tokens above it are counted, the
//      bucket's keys pushed to a per-row candidate list; the row's first CTA ("leader")
//      waits for the row's CTAs (arrival counter), resolves the exact threshold key T
//      (counting for small buckets, an 8-bit radix select otherwise: any bucket size,
//      ties included), prefix-sums the per-CTA selected counts and releases a row flag.
//   E  ordered writes: selection (ascending), new tokens = cur \ prev, evictions.
// The global scratch is left zero-filled: each buffer is cleared by the CTA that last
// needs it, and the last CTA to finish clears the barrier and the row flags.
// Requires all CTAs co-resident (<= one per SM, launched cooperatively).
#include "common.cuh"

namespace spc {
namespace {

#include "logits.cuh"

constexpr int SS_NC = 4;                 // LOGITS consumer warps; warp SS_NC = TMA producer
constexpr int SS_NT = 512;               // threads per CTA: warps past the producer build the
                                         // previous-selection bitmap during LOGITS; every
                                         // warp works in phases B..E
constexpr int SS_TPC = 16;               // max key tiles per CTA (2048 tokens)
constexpr int SS_TOK = SS_TPC * LG_TR;   // token capacity per CTA
constexpr int SS_NB = 256;               // bins of the pass-0 histogram
constexpr int SS_W0_SHIFT = 20;          // pass-0 bin = value bits >> 20: 8 bins per binade
constexpr int SS_W0_BITS = 12;
constexpr int SS_COUNT_MAX = 1024;       // rank the bucket by counting up to this size

template <int D, int ALPHA>
struct SsSmem {
  static constexpr int NCH = D / 64;
  static constexpr int QRAW = ALPHA * D * 2;
  static constexpr int QF = D * ALPHA * 4;
  static constexpr int BM = SS_TOK / 8;           // previous-selection bitmap
  static constexpr int FIXED = 1024 + SS_NC * QF + BM;
  static constexpr int NST0 = (232448 - 6144 - FIXED) / (LT_STAGE + QRAW);  // 6 KiB: static smem
  static constexpr int K = (NST0 > 12 ? 12 : NST0) / SS_NC;  // stages per consumer ring
  static constexpr int NST = K * SS_NC;
  static constexpr int QSLOT_OFF = NST * LT_STAGE;
  static constexpr int QF_OFF = QSLOT_OFF + NST * QRAW;
  static constexpr int BM_OFF = QF_OFF + SS_NC * QF;
  static constexpr int BYTES = 1024 + BM_OFF + BM;
  // after LOGITS the ring holds the CTA's exps [ALPHA][SS_TOK] and group scores [SS_TOK]
  // (then the bucket keys ranked by a row leader)
  static constexpr int LGS_OFF = 0;
  static constexpr int LGS = ALPHA * SS_TOK * 4;
  static constexpr int GSM_OFF = LGS;
  static constexpr int CAND_CAP = LGS / 8;
  static_assert(K >= 2, "ring too shallow");
  static_assert(LGS + SS_TOK * 4 <= NST * LT_STAGE, "exps and scores must fit the ring");
};

struct SsWs {  // global scratch, zero-filled between launches
  unsigned* sync;               // [0] grid barrier, [1] exit counter
  unsigned* maxenc;             // [B*Hq] encoded head maxima
  unsigned long long* sumacc;   // [B*Hq] O4 sums
  unsigned* hist;               // [B*G][SS_NB]
  unsigned* arrive;             // [B*G] CTAs of the row done with phase D
  unsigned* flag;               // [B*G] leader released the row
  unsigned* candn;              // [B*G] bucket keys pushed
  unsigned long long* cand;     // [B*G][Smax] bucket keys
  unsigned* cmeta;              // [B*G][Smax] (CTA << 1) | previously selected
  unsigned* stats;              // [ncta][2][2] above, above & previous (plain stores)
  float* lg;                    // [B][Hq][Smax] logits when the caller passes none
  unsigned long long* rowT;     // [B*G] threshold key
  int* rowtot;                  // [B*G][2] selected, selected & previous
  int* offs;                    // [ncta][2][2] selected / selected&prev before the CTA
  size_t bytes;
};
SsWs ss_ws_layout(void* ws, int B, int Hq, int G, int Smax, int ncta) {
  uint8_t* p = (uint8_t*)ws;
  SsWs w;
  size_t off = 0;
  auto take = [&](size_t n) {
    uint8_t* q = p + off;
    off = align_up(off + n, 256);
    return q;
  };
  const size_t BG = (size_t)B * G;
  w.sync = (unsigned*)take(8);
  w.maxenc = (unsigned*)take(4 * (size_t)B * Hq);
  w.sumacc = (unsigned long long*)take(8 * (size_t)B * Hq);
  w.hist = (unsigned*)take(4 * BG * SS_NB);
  w.arrive = (unsigned*)take(4 * BG);
  w.flag = (unsigned*)take(4 * BG);
  w.candn = (unsigned*)take(4 * BG);
  w.cand = (unsigned long long*)take(8 * BG * Smax);
  w.cmeta = (unsigned*)take(4 * BG * Smax);
  w.stats = (unsigned*)take(16 * (size_t)ncta);
  w.lg = (float*)take(4 * (size_t)B * Hq * Smax);
  w.rowT = (unsigned long long*)take(8 * BG);
  w.rowtot = (int*)take(8 * BG);
  w.offs = (int*)take(16 * (size_t)ncta);
  w.bytes = off;
  return w;
}

__device__ __forceinline__ unsigned ord_enc(float f) {
  const unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord_dec(unsigned e) {
  return __uint_as_float((e & 0x80000000u) ? (e & 0x7FFFFFFFu) : ~e);
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void spin_geq(const unsigned* p, unsigned v, int site = 0) {
#ifdef SPC_SS_DEBUG  // debug builds: report a wait that does not end, then give up
  long long n = 0;
  while (ld_acquire(p) < v) {
    if (++n == (1ll << 26)) {
      printf("score_select stuck: cta %d tid %d site %d value %u target %u\n", blockIdx.x, threadIdx.x,
             site, ld_acquire(p), v);
      return;
    }
  }
#else
  (void)site;
  while (ld_acquire(p) < v) __nanosleep(64);  // back off: spinners must not starve the SMs still working
#endif
}
// grid-wide barrier number n (1, 2, ...) of this launch: all CTAs are co-resident
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned n) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    red_release(bar, 1u);
    spin_geq(bar, n * gridDim.x, (int)n);
    __threadfence();
  }
  __syncthreads();
}
// CTA owning key tile x under the split [c n / N, (c+1) n / N)
__device__ __forceinline__ int cta_of(int x, int ntiles, int ncta) {
  return (int)((((long long)x + 1) * ncta - 1) / ntiles);
}

// Debug (spc_debug_set_ss_progress, tools only): per CTA, the last phase mark reached
// (volatile stores to host-mapped memory, readable while a launch hangs).
__device__ volatile int* g_ss_prog = nullptr;
__device__ unsigned long long* g_ss_time = nullptr;  // [cta][16] %globaltimer per mark
__device__ __forceinline__ void ss_mark(int v) {
  if (threadIdx.x == 0) {
    if (g_ss_prog) g_ss_prog[blockIdx.x] = v;
    if (g_ss_time) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      g_ss_time[blockIdx.x * 16 + v] = t;
    }
  }
}

struct SsSlot {
  int bg, b, g, len, need, cut, u0, u1, t0, first, last, np;
  int lpre_t0;   // previous tokens < t0 (in the row)
  int lpre_end;  // previous tokens < min(t0 + (u1 - u0), len)
  int lpre_len;  // previous tokens < len
};

template <int D, int ALPHA>
__global__ void __launch_bounds__(SS_NT, 1) score_select_kernel(
    const __grid_constant__ CUtensorMap kmap, const uint16_t* __restrict__ q,
    const int32_t* __restrict__ seq_len, int B, int G, int Smax, float scale, int tpr, int ntiles,
    int k, int force, float* __restrict__ logits, float* __restrict__ head_max,
    int64_t* __restrict__ head_sumfix, float* __restrict__ group_score, int32_t* __restrict__ out_idx,
    int32_t* __restrict__ out_count, const int32_t* __restrict__ prev_idx,
    const int32_t* __restrict__ prev_count, int32_t* __restrict__ load_tok, int32_t* __restrict__ n_load,
    int32_t* __restrict__ evict_tok, int32_t* __restrict__ n_evict, SsWs w) {
  using SM = SsSmem<D, ALPHA>;
  constexpr int NCH = SM::NCH, NST = SM::NST;
  __shared__ __align__(8) uint64_t full[NST], empty[NST];
  __shared__ SsSlot sl[2];
  __shared__ unsigned mx_s[2][ALPHA];
  __shared__ unsigned long long sum_s[2][ALPHA];
  __shared__ unsigned hist_s[2][SS_NB];
  __shared__ int find_s[2][3];        // bin, above, count in bin
  __shared__ unsigned long long wsc[SS_NT / 32];
  __shared__ int cnt_s[2][2];         // above, above & previous (this CTA)
  __shared__ int rk_s[SS_NB];         // leader: radix histogram / per-CTA counts
  __shared__ int rk2_s[SS_NB];
  __shared__ unsigned long long T_s[2];
  __shared__ int off_s[2][2];         // selected / selected&prev before this CTA (row)
  __shared__ int tot_s[2][2];         // row totals
  __shared__ int misc_s[4];
  __shared__ float m_s[2][ALPHA], r_s[2][ALPHA];
  __shared__ int base0_s[2];
  extern __shared__ __align__(16) uint8_t ss_raw[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int Hq = G * ALPHA;
  const int ncta = gridDim.x;
  const uint32_t base = (smem_u32(ss_raw) + 1023u) & ~1023u;
  uint8_t* basep = ss_raw + (base - smem_u32(ss_raw));
  float* lgs = (float*)(basep + SM::LGS_OFF);   // [ALPHA][SS_TOK] (ring, after LOGITS)
  float* gsm = (float*)(basep + SM::GSM_OFF);   // [SS_TOK]           (ring, after LOGITS)
  float* lgout = logits ? logits : w.lg;        // LOGITS' output, re-read (L2) by NORM
  uint32_t* bm = (uint32_t*)(basep + SM::BM_OFF);
  const uint32_t full0 = smem_u32(&full[0]), empty0 = smem_u32(&empty[0]);
  const int tb = (int)(((long long)blockIdx.x * ntiles) / ncta);
  const int te = (int)(((long long)(blockIdx.x + 1) * ntiles) / ncta);
  const int nloc = (te - tb) * LG_TR;
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(full0 + 8 * s));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(empty0 + 8 * s));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_tmap(&kmap);
  }
  for (int i = tid; i < SS_TOK / 32; i += SS_NT) bm[i] = 0u;
  for (int i = tid; i < 2 * SS_NB; i += SS_NT) (&hist_s[0][0])[i] = 0u;
  if (tid < 2 * ALPHA) {
    (&mx_s[0][0])[tid] = 0u;
    (&sum_s[0][0])[tid] = 0ull;
  }
  if (tid < 4) (&cnt_s[0][0])[tid] = 0;
  spc_pdl_entry();
  ss_mark(1);
  if (tid < 2) {  // the (at most two) rows of this CTA's tiles
    SsSlot& S = sl[tid];
    const int r0 = tb / tpr;
    const int row = r0 + tid;
    const int t_lo = max(tb, row * tpr), t_hi = min(te, (row + 1) * tpr);
    if (t_lo < t_hi) {
      S.bg = row;
      S.b = row / G;
      S.g = row - S.b * G;
      S.len = min(max(seq_len[S.b], 0), Smax);
      S.need = min(k, S.len);
      S.cut = S.need < S.len;
      S.u0 = (t_lo - tb) * LG_TR;
      S.u1 = (t_hi - tb) * LG_TR;
      S.t0 = (t_lo - row * tpr) * LG_TR;
      S.first = cta_of(row * tpr, ntiles, ncta);
      S.last = cta_of(row * tpr + tpr - 1, ntiles, ncta);
      S.np = min(max(prev_count[row], 0), k);
    } else {
      S.bg = -1;
      S.u0 = S.u1 = nloc;
    }
    S.lpre_t0 = S.lpre_end = S.lpre_len = 0;
  }
  __syncthreads();
  const int nslot = sl[1].bg >= 0 ? 2 : 1;

  if (warp == SS_NC) {
    // ============================================================ A: producer (lane 0)
    if (lane == 0) {
      int nt = 0;  // active-tile counter
      for (int tile = tb; tile < te; ++tile) {
        const int bg = tile / tpr, tt = tile - bg * tpr;
        if (tt * LG_TR >= min(max(__ldg(seq_len + bg / G), 0), Smax)) continue;  // empty tile
        const int w = nt % SS_NC, n = nt / SS_NC;  // consumer warp and its tile count
        ++nt;
        for (int c = 0; c < NCH; ++c) {
          const int j = n * NCH + c;  // sequence number in warp w's ring
          const int s = w * SM::K + j % SM::K;
          if (j >= SM::K) tm_wait(empty0 + 8 * s, ((j / SM::K) - 1) & 1);
          if (g_ss_prog) g_ss_prog[256 + blockIdx.x * 8 + 7] = nt;
          const uint32_t fb = full0 + 8 * s;
          tm_expect(fb, LT_STAGE + (c == 0 ? SM::QRAW : 0));
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%2, %3}], [%4];" ::"r"(base + s * LT_STAGE),
              "l"(&kmap), "r"(64 * c), "r"(bg * Smax + tt * LG_TR), "r"(fb)
              : "memory");
          if (c == 0) {
            const int b = bg / G, g = bg - b * G;
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    base + SM::QSLOT_OFF + s * SM::QRAW),
                "l"(q + ((size_t)b * Hq + g * ALPHA) * D), "r"(SM::QRAW), "r"(fb)
                : "memory");
          }
        }
      }
    }
  } else if (warp > SS_NC) {
    // ============================================================ A: helper warps
    // bitmap of the previous selection over the CTA's token range and the prefix counts
    // of the previous list (needed from phase D on)
    const int ht = tid - (SS_NC + 1) * 32, nht = SS_NT - (SS_NC + 1) * 32;
    for (int s = 0; s < nslot; ++s) {
      const SsSlot& S = sl[s];
      const int32_t* pv = prev_idx + (size_t)S.bg * k;
      const int tend = min(S.t0 + (S.u1 - S.u0), S.len);
      int c0 = 0, c1 = 0, c2 = 0;
      for (int i = ht; i < S.np; i += nht) {
        const int t = __ldg(pv + i);
        SPC_DCHECK(t >= 0 && (i == 0 || __ldg(pv + i - 1) < t), t < 0 ? SPC_E_RANGE : SPC_E_STATE);
        if (t >= S.t0 && t < tend) atomicOr(&bm[(S.u0 + t - S.t0) >> 5], 1u << ((S.u0 + t - S.t0) & 31));
        c0 += t < S.t0;
        c1 += t < tend;
        c2 += t < S.len;
      }
      c0 = __reduce_add_sync(0xffffffffu, c0);
      c1 = __reduce_add_sync(0xffffffffu, c1);
      c2 = __reduce_add_sync(0xffffffffu, c2);
      if (lane == 0) {
        atomicAdd(&sl[s].lpre_t0, c0);
        atomicAdd(&sl[s].lpre_end, c1);
        atomicAdd(&sl[s].lpre_len, c2);
      }
    }
  } else {
    // ============================================================ A: consumers
    float* qf = (float*)(basep + SM::QF_OFF + warp * SM::QF);
    const uint32_t qf_s = smem_u32(qf);
    int nt = 0;  // active-tile counter; tile nt goes to warp nt % SS_NC (its own ring)
    for (int tile = tb; tile < te; ++tile) {
      const int bg = tile / tpr, tt = tile - bg * tpr, t0 = tt * LG_TR;
      const int b = bg / G, g = bg - b * G;
      const int len = min(max(__ldg(seq_len + b), 0), Smax);
      if (t0 >= len) continue;
      const int mine = (nt % SS_NC) == warp, n = nt / SS_NC;
      ++nt;
      if (!mine) continue;
      float2 acc[ALPHA][LG_RPT / 2];
#pragma unroll
      for (int j = 0; j < ALPHA; ++j)
#pragma unroll
        for (int p = 0; p < LG_RPT / 2; ++p) acc[j][p] = make_float2(0.f, 0.f);
      for (int c = 0; c < NCH; ++c) {
        const int j = n * NCH + c;
        const int s = warp * SM::K + j % SM::K;
        tm_wait(full0 + 8 * s, (j / SM::K) & 1);
        if (c == 0) {
          const uint16_t* qr = (const uint16_t*)(basep + SM::QSLOT_OFF + s * SM::QRAW);
          for (int e = lane; e < ALPHA * D; e += 32) {
            const int j = e / D, d = e - j * D;
            qf[d * ALPHA + j] = __uint_as_float((uint32_t)qr[e] << 16);
          }
          __syncwarp();
        }
        lt_stage_math<D, ALPHA>(acc, base + s * LT_STAGE, qf_s, qf, c, lane);
        if (g_ss_prog && lane == 0) g_ss_prog[256 + blockIdx.x * 8 + warp] = j + 1;
        __syncwarp();
        if (lane == 0) tm_arrive(empty0 + 8 * s);
      }
      const int slot = bg == sl[0].bg ? 0 : 1;
#pragma unroll
      for (int j = 0; j < ALPHA; ++j) {
        float m = -INFINITY;
#pragma unroll
        for (int r = 0; r < LG_RPT; ++r) {
          const int row = lane + 32 * r;
          const float sv = __fmul_rn((r & 1) ? acc[j][r >> 1].y : acc[j][r >> 1].x, scale);
          if (t0 + row < len) {
            SPC_DCHECK(sv == sv, SPC_E_RANGE);  // NaN key / query (reading R20)
            lgout[((size_t)b * Hq + g * ALPHA + j) * Smax + t0 + row] = sv;
            m = fmaxf(m, sv);
          }
        }
        m = warp_max(m);
        if (lane == 0) atomicMax(&mx_s[slot][j], ord_enc(m));
      }
    }
  }
  __syncthreads();
  if (tid < nslot * ALPHA) {
    const int s = tid / ALPHA, j = tid - s * ALPHA;
    const unsigned e = mx_s[s][j];
    if (e) atomicMax(&w.maxenc[(size_t)sl[s].b * Hq + sl[s].g * ALPHA + j], e);
  }
  ss_mark(2);
  grid_sync(w.sync, 1);
  ss_mark(3);

  // ============================================================ B: NORM (O3, O4)
  // thread chunk: local tokens [u_a, u_a + cpt), inside one slot (cpt divides 128)
  constexpr int cpt = 4;  // a warp's 128 tokens = one key tile (one slot)
  static_assert(cpt * SS_NT >= SS_TOK && 32 * cpt == LG_TR, "token chunking");
  const int u_a = tid * cpt;
  const int my_slot = u_a < sl[0].u1 ? 0 : 1;
  const bool have = u_a < nloc;
  if (tid < nslot * ALPHA) {
    const int s = tid / ALPHA, j = tid - s * ALPHA;
    const size_t h = (size_t)sl[s].b * Hq + sl[s].g * ALPHA + j;
    const float mv = ord_dec(__ldcg(&w.maxenc[h]));
    m_s[s][j] = mv;
    if (sl[s].first == (int)blockIdx.x) head_max[h] = mv;  // the row's leader publishes O2
  }
  __syncthreads();
  float m[ALPHA];
#pragma unroll
  for (int j = 0; j < ALPHA; ++j) m[j] = m_s[my_slot][j];
  if (have) {
    const SsSlot& S = sl[my_slot];
    long long acc[ALPHA];
#pragma unroll
    for (int j = 0; j < ALPHA; ++j) acc[j] = 0;
    for (int u = u_a; u < u_a + cpt; u += 4) {
      const int t = S.t0 + (u - S.u0);
      float4 xs[ALPHA];
#pragma unroll
      for (int j = 0; j < ALPHA; ++j) {  // this CTA's own logits (its stores, L2)
        const float* src = lgout + ((size_t)S.b * Hq + S.g * ALPHA + j) * Smax + t;
        xs[j] = make_float4(t < S.len ? __ldcg(src) : 0.f, t + 1 < S.len ? __ldcg(src + 1) : 0.f,
                            t + 2 < S.len ? __ldcg(src + 2) : 0.f, t + 3 < S.len ? __ldcg(src + 3) : 0.f);
      }
#pragma unroll
      for (int j = 0; j < ALPHA; ++j) {
        const float4 x = xs[j];
        const float2 ea = spc_exp2_dev(__fsub_rn(x.x, m[j]), __fsub_rn(x.y, m[j]));
        const float2 eb = spc_exp2_dev(__fsub_rn(x.z, m[j]), __fsub_rn(x.w, m[j]));
        const float4 e = make_float4(t < S.len ? ea.x : 0.f, t + 1 < S.len ? ea.y : 0.f,
                                     t + 2 < S.len ? eb.x : 0.f, t + 3 < S.len ? eb.y : 0.f);
        acc[j] += fixpoint40(e.x) + fixpoint40(e.y) + fixpoint40(e.z) + fixpoint40(e.w);
        *reinterpret_cast<float4*>(lgs + j * SS_TOK + u) = e;
      }
    }
#pragma unroll
    for (int j = 0; j < ALPHA; ++j) acc[j] = warp_sum_ll(acc[j]);  // the warp's tile: one slot
    if (lane == 0)
#pragma unroll
      for (int j = 0; j < ALPHA; ++j)
        if (acc[j]) atomicAdd(&sum_s[my_slot][j], (unsigned long long)acc[j]);
  }
  __syncthreads();
  if (tid < nslot * ALPHA) {
    const int s = tid / ALPHA, j = tid - s * ALPHA;
    const unsigned long long v = sum_s[s][j];
    if (v) atomicAdd(&w.sumacc[(size_t)sl[s].b * Hq + sl[s].g * ALPHA + j], v);
  }
  ss_mark(4);
  grid_sync(w.sync, 2);
  ss_mark(5);
  if (blockIdx.x == 0)  // every CTA read its maxima before barrier 2
    for (int i = tid; i < B * Hq; i += SS_NT) w.maxenc[i] = 0u;

  // ============================================================ C: GROUP (O4..O6) + pass-0 histogram
  if (tid < nslot * ALPHA) {
    const int s = tid / ALPHA, j = tid - s * ALPHA;
    const size_t h = (size_t)sl[s].b * Hq + sl[s].g * ALPHA + j;
    const long long F = (long long)__ldcg(&w.sumacc[h]);
    r_s[s][j] = __fdiv_rn(1.0f, __fmul_rn(__ll2float_rn(F), 9.094947017729282379150390625e-13f));
    if (sl[s].first == (int)blockIdx.x) head_sumfix[h] = F;
  }
  __syncthreads();
  if (tid < nslot) {  // pass-0 window: 256 bins below the row maximum max_j r_j
    float gm = 0.f;
#pragma unroll
    for (int j = 0; j < ALPHA; ++j) gm = fmaxf(gm, r_s[tid][j]);
    base0_s[tid] = (int)(__float_as_uint(gm) >> SS_W0_SHIFT) - (SS_NB - 1);
  }
  __syncthreads();
  float r[ALPHA];
#pragma unroll
  for (int j = 0; j < ALPHA; ++j) r[j] = r_s[my_slot][j];
  const int base0 = base0_s[my_slot];
  if (have) {
    const SsSlot& S = sl[my_slot];
    float* gso = group_score + (size_t)S.bg * Smax;
    for (int u = u_a; u < u_a + cpt; u += 4) {
      const int t = S.t0 + (u - S.u0);
      float gv[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float v = __fmul_rn(lgs[u + c], r[0]);
#pragma unroll
        for (int j = 1; j < ALPHA; ++j) v = fmaxf(v, __fmul_rn(lgs[j * SS_TOK + u + c], r[j]));
        gv[c] = t + c < S.len ? v : 0.f;
        if (S.cut && t + c < S.len) {
          const unsigned long long key = composite(
              (force && t + c == S.len - 1) ? 0x7F800000u : __float_as_uint(gv[c]), t + c);
          atomicAdd(&hist_s[my_slot][min(max((int)(key >> 52) - base0, 0), SS_NB - 1)], 1u);
        }
      }
      *reinterpret_cast<float4*>(gsm + u) = make_float4(gv[0], gv[1], gv[2], gv[3]);
      if (t < Smax) {
        if (t + 3 < Smax) *reinterpret_cast<float4*>(gso + t) = make_float4(gv[0], gv[1], gv[2], gv[3]);
        else
          for (int c = 0; c < 4 && t + c < Smax; ++c) gso[t + c] = gv[c];
      }
    }
  }
  __syncthreads();
  for (int i = tid; i < nslot * SS_NB; i += SS_NT) {
    const int s = i / SS_NB, bin = i - s * SS_NB;
    const unsigned h = hist_s[s][bin];
    if (h && sl[s].cut) atomicAdd(&w.hist[(size_t)sl[s].bg * SS_NB + bin], h);
  }
  ss_mark(6);
  grid_sync(w.sync, 3);
  ss_mark(7);
  if (blockIdx.x == 0)
    for (int i = tid; i < B * Hq; i += SS_NT) w.sumacc[i] = 0ull;

  // ============================================================ D: threshold
  // find the bin of the need-th largest key from the top of the row's histogram
  if (warp < nslot && sl[warp].cut) {
    const SsSlot& S = sl[warp];
    const unsigned* gh = w.hist + (size_t)S.bg * SS_NB;
    unsigned c8[8], tot = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {  // lane l: bins 255 - 8l - i
      c8[i] = __ldcg(gh + (SS_NB - 1 - 8 * lane - i));
      tot += c8[i];
    }
    unsigned incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned x = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += x;
    }
    const unsigned need = (unsigned)S.need;
    if (incl >= need && incl - tot < need) {
      unsigned run = incl - tot;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (run + c8[i] >= need && run < need) {
          find_s[warp][0] = SS_NB - 1 - 8 * lane - i;
          find_s[warp][1] = (int)run;
          find_s[warp][2] = (int)c8[i];
        }
        run += c8[i];
      }
    }
  }
  __syncthreads();
  // bucket of each slot: keys x with (x >> (64 - bits)) == (P >> (64 - bits)), xlo <= x <= xmax
  unsigned long long Pb[2] = {0ull, 0ull}, xlo[2] = {0ull, 0ull}, xmax[2] = {~0ull, ~0ull};
  int bits[2] = {1, 1};
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    if (s < nslot && sl[s].cut) {
      const int bin0 = find_s[s][0];
      const int b0 = base0_s[s];
      if (bin0 == 0) {
        xmax[s] = ((unsigned long long)(uint32_t)(b0 + 1) << 52) - 1ull;
      } else if (bin0 == SS_NB - 1) {
        xlo[s] = (unsigned long long)(uint32_t)(b0 + SS_NB - 1) << 52;
      } else {
        Pb[s] = (unsigned long long)(uint32_t)(b0 + bin0) << 52;
        bits[s] = SS_W0_BITS;
      }
    }
  }
  // classify this thread's tokens: above the bucket / in it (pushed as candidates)
  if (have && sl[my_slot].cut) {  // warp-uniform: a warp's tokens are one tile of one slot
    const SsSlot& S = sl[my_slot];
    const int s = my_slot, sh = 64 - bits[s];
    int ab = 0, abp = 0;
    for (int u = u_a; u < u_a + cpt; ++u) {
      const int t = S.t0 + (u - S.u0);
      const bool valid = t < S.len;
      const unsigned long long x =
          composite((force && t == S.len - 1) ? 0x7F800000u : __float_as_uint(gsm[u]), t);
      const bool was = (bm[u >> 5] >> (u & 31)) & 1u;
      const bool above = valid && (x > xmax[s] || (x >> sh) > (Pb[s] >> sh));
      const bool inb = valid && (x >> sh) == (Pb[s] >> sh) && x >= xlo[s] && x <= xmax[s];
      ab += above;
      abp += above && was;
      const unsigned m = __ballot_sync(0xffffffffu, inb);
      if (m) {
        unsigned base_slot = 0;
        if (lane == 0) base_slot = atomicAdd(&w.candn[S.bg], (unsigned)__popc(m));
        base_slot = __shfl_sync(0xffffffffu, base_slot, 0);
        if (inb) {
          const unsigned slot = base_slot + __popc(m & ((1u << lane) - 1u));
          w.cand[(size_t)S.bg * Smax + slot] = x;
          w.cmeta[(size_t)S.bg * Smax + slot] = (blockIdx.x << 1) | (unsigned)was;
        }
      }
    }
    ab = __reduce_add_sync(0xffffffffu, ab);
    abp = __reduce_add_sync(0xffffffffu, abp);
    if (lane == 0) {
      if (ab) atomicAdd(&cnt_s[s][0], ab);
      if (abp) atomicAdd(&cnt_s[s][1], abp);
    }
  }
  __syncthreads();
  if (tid < nslot && sl[tid].cut) {
    w.stats[(blockIdx.x * 2 + tid) * 2] = (unsigned)cnt_s[tid][0];
    w.stats[(blockIdx.x * 2 + tid) * 2 + 1] = (unsigned)cnt_s[tid][1];
    __threadfence();
    red_release(&w.arrive[sl[tid].bg], 1u);
  }
  ss_mark(10);
  // leader of a cut row: resolve T exactly, per-CTA offsets, release the row
  for (int s = 0; s < nslot; ++s) {
    const SsSlot& S = sl[s];
    if (!S.cut || S.first != (int)blockIdx.x) continue;
    if (tid == 0) spin_geq(&w.arrive[S.bg], (unsigned)(S.last - S.first + 1), 10 + s);
    __syncthreads();
    const int cm = (int)__ldcg(&w.candn[S.bg]);
    const int rr = S.need - find_s[s][1];  // rank of T inside the bucket (1-based)
    const unsigned long long* cg_ = w.cand + (size_t)S.bg * Smax;
    const unsigned* cmt = w.cmeta + (size_t)S.bg * Smax;
    unsigned long long* ck = reinterpret_cast<unsigned long long*>(lgs);  // shared copy
    const bool in_smem = cm <= SM::CAND_CAP;
    if (in_smem)
      for (int i = tid; i < cm; i += SS_NT) ck[i] = __ldcg(cg_ + i);
    __syncthreads();
    auto K = [&](int i) { return in_smem ? ck[i] : __ldcg(cg_ + i); };
    if (cm <= SS_COUNT_MAX) {
      for (int i = tid; i < cm; i += SS_NT) {
        const unsigned long long x = K(i);
        int larger = 0;
        for (int j = 0; j < cm; ++j) larger += K(j) > x;
        if (larger == rr - 1) T_s[s] = x;
      }
    } else {  // 8-bit radix select over the bucket, most significant byte first
      // the bucket fixes the top `bits` key bits: digits of 8 bits below them
      const int fixed = bits[s];
      unsigned long long pre = fixed > 1 ? (Pb[s] & (~0ull << (64 - fixed))) : 0ull;
      int rem = rr;
      for (int shift = 64 - fixed - 8; shift > -8; shift -= 8) {
        const int sh8 = shift < 0 ? 0 : shift;  // the last digit may be narrower
        const int nb8 = shift < 0 ? 8 + shift : 8;
        for (int i = tid; i < SS_NB; i += SS_NT) rk_s[i] = 0;
        __syncthreads();
        const unsigned long long hm = ~0ull << (sh8 + nb8);
        for (int i = tid; i < cm; i += SS_NT) {
          const unsigned long long x = K(i);
          if ((x & hm) == pre) atomicAdd(&rk_s[(x >> sh8) & ((1u << nb8) - 1u)], 1);
        }
        __syncthreads();
        if (warp == 0) {
          int c8[8], t8 = 0;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            c8[i] = rk_s[255 - 8 * lane - i];
            t8 += c8[i];
          }
          int incl = t8;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int x = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += x;
          }
          if (incl >= rem && incl - t8 < rem) {
            int run = incl - t8;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              if (run + c8[i] >= rem && run < rem) {
                misc_s[0] = 255 - 8 * lane - i;
                misc_s[1] = run;
              }
              run += c8[i];
            }
          }
        }
        __syncthreads();
        pre |= (unsigned long long)misc_s[0] << sh8;
        rem -= misc_s[1];
        __syncthreads();
      }
      if (tid == 0) T_s[s] = pre;
    }
    __syncthreads();
    const unsigned long long T = T_s[s];
    // per-CTA selected bucket keys (and of those, previously selected)
    const int nr = S.last - S.first + 1;
    for (int i = tid; i < nr; i += SS_NT) {
      rk_s[i] = 0;
      rk2_s[i] = 0;
    }
    __syncthreads();
    for (int i = tid; i < cm; i += SS_NT)
      if (K(i) >= T) {
        const unsigned mt = __ldcg(cmt + i);
        atomicAdd(&rk_s[(int)(mt >> 1) - S.first], 1);
        if (mt & 1u) atomicAdd(&rk2_s[(int)(mt >> 1) - S.first], 1);
      }
    __syncthreads();
    if (warp == 0) {  // prefix over the row's CTAs: lane l takes CTAs first + l, + 32, ...
      int carry = 0, carryp = 0;
      for (int c0 = S.first; c0 <= S.last; c0 += 32) {
        const int c = c0 + lane;
        int sel = 0, selp = 0, sc = 0;
        if (c <= S.last) {
          // slot of this row in CTA c: 0 when c's first tile belongs to it
          sc = (int)(((long long)c * ntiles / ncta) / tpr) == S.bg ? 0 : 1;
          sel = (int)__ldcg(&w.stats[(c * 2 + sc) * 2]) + rk_s[c - S.first];
          selp = (int)__ldcg(&w.stats[(c * 2 + sc) * 2 + 1]) + rk2_s[c - S.first];
        }
        int is = sel, isp = selp;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int x = __shfl_up_sync(0xffffffffu, is, o), xp = __shfl_up_sync(0xffffffffu, isp, o);
          if (lane >= o) {
            is += x;
            isp += xp;
          }
        }
        if (c <= S.last) {
          w.offs[(c * 2 + sc) * 2] = carry + is - sel;
          w.offs[(c * 2 + sc) * 2 + 1] = carryp + isp - selp;
        }
        carry += __shfl_sync(0xffffffffu, is, 31);
        carryp += __shfl_sync(0xffffffffu, isp, 31);
      }
      if (lane == 0) {
        w.rowT[S.bg] = T;
        w.rowtot[S.bg * 2] = carry;
        w.rowtot[S.bg * 2 + 1] = carryp;
        w.arrive[S.bg] = 0u;
        w.candn[S.bg] = 0u;
      }
      __syncwarp();
      if (lane == 0) {
        __threadfence();
        red_release(&w.flag[S.bg], 1u);
      }
    }
    for (int i = tid; i < SS_NB; i += SS_NT) w.hist[(size_t)S.bg * SS_NB + i] = 0u;
    __syncthreads();
  }
  ss_mark(8);
  // every CTA: threshold, offsets and row totals of its slots
  if (tid < nslot) {
    const SsSlot& S = sl[tid];
    if (S.cut) {
      spin_geq(&w.flag[S.bg], 1u, 20 + tid);
      T_s[tid] = __ldcg(&w.rowT[S.bg]);
      off_s[tid][0] = __ldcg(&w.offs[(blockIdx.x * 2 + tid) * 2]);
      off_s[tid][1] = __ldcg(&w.offs[(blockIdx.x * 2 + tid) * 2 + 1]);
      tot_s[tid][0] = __ldcg(&w.rowtot[S.bg * 2]);
      tot_s[tid][1] = __ldcg(&w.rowtot[S.bg * 2 + 1]);
    } else {  // every valid token is selected
      T_s[tid] = 0ull;
      off_s[tid][0] = min(S.t0, S.len);
      off_s[tid][1] = S.lpre_t0;
      tot_s[tid][0] = S.len;
      tot_s[tid][1] = S.lpre_len;
    }
  }
  __syncthreads();

  ss_mark(11);
  // ============================================================ E: ordered writes
  for (int s = 0; s < nslot; ++s) {
    const SsSlot& S = sl[s];
    const unsigned long long T = T_s[s];
    unsigned long long cnt = 0ull;  // selected | new << 21 | evicted << 42
    const bool mine = have && my_slot == s;
    if (mine)
      for (int u = u_a; u < u_a + cpt; ++u) {
        const int t = S.t0 + (u - S.u0);
        if (t >= S.len) break;
        const bool sel =
            composite((force && t == S.len - 1) ? 0x7F800000u : __float_as_uint(gsm[u]), t) >= T;
        const bool was = (bm[u >> 5] >> (u & 31)) & 1u;
        cnt += (unsigned long long)sel + ((unsigned long long)(sel && !was) << 21) +
               ((unsigned long long)(!sel && was) << 42);
      }
    // block-wide exclusive scan of cnt
    unsigned long long incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long x = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += x;
    }
    if (lane == 31) wsc[warp] = incl;
    __syncthreads();
    unsigned long long before = 0ull;
    for (int i = 0; i < warp; ++i) before += wsc[i];
    const unsigned long long pos = before + incl - cnt;
    const int sb = off_s[s][0], spb = off_s[s][1];
    int ps = sb + (int)(pos & 0x1FFFFF), pn = sb - spb + (int)((pos >> 21) & 0x1FFFFF),
        pe = S.lpre_t0 - spb + (int)(pos >> 42);
    int32_t* oi = out_idx + (size_t)S.bg * k;
    int32_t* lt = load_tok + (size_t)S.bg * k;
    int32_t* et = evict_tok ? evict_tok + (size_t)S.bg * k : nullptr;
    if (mine)
      for (int u = u_a; u < u_a + cpt; ++u) {
        const int t = S.t0 + (u - S.u0);
        if (t >= S.len) break;
        const bool sel =
            composite((force && t == S.len - 1) ? 0x7F800000u : __float_as_uint(gsm[u]), t) >= T;
        const bool was = (bm[u >> 5] >> (u & 31)) & 1u;
        if (sel) oi[ps++] = t;
        if (sel && !was) lt[pn++] = t;
        if (!sel && was && et) et[pe++] = t;
      }
    // the row's last CTA: padding, the evicted tail (previous tokens >= len), counts
    if (S.last == (int)blockIdx.x) {
      const int as = tot_s[s][0], asp = tot_s[s][1];
      const int an = as - asp, ae = S.np - asp, ntail = S.np - S.lpre_len;
      const int32_t* pv = prev_idx + (size_t)S.bg * k;
      if (et)
        for (int i = tid; i < ntail; i += SS_NT) et[ae - ntail + i] = pv[S.np - ntail + i];
      for (int i = as + tid; i < k; i += SS_NT) oi[i] = -1;
      for (int i = an + tid; i < k; i += SS_NT) lt[i] = -1;
      if (et)
        for (int i = ae + tid; i < k; i += SS_NT) et[i] = -1;
      if (tid == 0) {
        out_count[S.bg] = as;
        n_load[S.bg] = an;
        if (n_evict) n_evict[S.bg] = ae;
      }
    }
    __syncthreads();
  }
  ss_mark(9);
  // exit: the last CTA out clears the barrier and the row flags for the next launch
  if (tid == 0) {
    __threadfence();
    const unsigned t = atomicAdd(&w.sync[1], 1u);
    if (t == (unsigned)ncta - 1) {
      for (int i = 0; i < B * G; ++i) w.flag[i] = 0u;
      w.sync[0] = 0u;
      w.sync[1] = 0u;
      __threadfence();
    }
  }
}

}  // namespace
}  // namespace spc

using namespace spc;

namespace {
constexpr int SS_MAX_CTAS = 256;
// CTAs of the launch and whether the fused kernel applies: every CTA's tile range fits
// its shared memory (<= SS_TPC tiles) and spans at most two rows (<= tiles per row)
int ss_geometry(int B, int Hq, int G, int D, int Smax, int k, int* ncta_out) {
  if (B <= 0 || Hq <= 0 || G <= 0 || Smax <= 0 || Hq % G) return SPC_E_SHAPE;
  if (k < 1 || k > SPC_MAX_K) return SPC_E_BUDGET;
  const int alpha = Hq / G;
  if (!(D == 64 || D == 128) || !(alpha == 1 || alpha == 2 || alpha == 4 || alpha == 8))
    return SPC_E_UNSUPPORTED;
  if ((long long)B * G * Smax >= (1ll << 31) || Smax >= SPC_MAX_SEQ) return SPC_E_UNSUPPORTED;
  const int tpr = (Smax + LG_TR - 1) / LG_TR;
  const long long ntiles = (long long)B * G * tpr;
  const int ncta = (int)std::min<long long>(std::min(num_sms(), SS_MAX_CTAS), ntiles);
  const long long per = (ntiles + ncta - 1) / ncta;
  if (per > SS_TPC || per > tpr) return SPC_E_UNSUPPORTED;
  if (ncta_out) *ncta_out = ncta;
  return SPC_OK;
}

template <int DD, int AA>
int ss_launch(const uint16_t* q, const uint16_t* kr, const int32_t* seq_len, int B, int G, int Smax,
              float scale, int k, int force, float* logits, float* head_max, int64_t* head_sumfix,
              float* group_score, int32_t* out_idx, int32_t* out_count, const int32_t* prev_idx,
              const int32_t* prev_count, int32_t* load_tok, int32_t* n_load, int32_t* evict_tok,
              int32_t* n_evict, SsWs w, int ncta, cudaStream_t st) {
  SPC_TRY(smem_attr((const void*)score_select_kernel<DD, AA>, SsSmem<DD, AA>::BYTES));
  const int tpr = (Smax + LG_TR - 1) / LG_TR;
  CUtensorMap map;
  SPC_TRY(make_tmap_tile_bf16(&map, kr, (uint64_t)B * G * Smax, DD, LG_TR));
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident (grid barriers)
  at[0].val.cooperative = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ncta);
  cfg.blockDim = dim3(SS_NT);
  cfg.dynamicSmemBytes = SsSmem<DD, AA>::BYTES;
  cfg.stream = st;
  static const bool coop = [] {
    const char* e = std::getenv("SPC_SS_COOP");
    return !(e && e[0] == '0');
  }();
  cfg.attrs = coop ? at : at + 1;
  cfg.numAttrs = (coop ? 1 : 0) + (pdl_enabled() ? 1 : 0);
  return launched(cudaLaunchKernelEx(&cfg, score_select_kernel<DD, AA>, map, q, seq_len, B, G, Smax,
                                     scale, tpr, B * G * tpr, k, force, logits, head_max, head_sumfix,
                                     group_score, out_idx, out_count, prev_idx, prev_count, load_tok,
                                     n_load, evict_tok, n_evict, w));
}
}  // namespace

extern "C" int spc_debug_set_ss_progress(void* p) {  // tools only; not in include/spc.h
  volatile int* q = (volatile int*)p;
  return cudaMemcpyToSymbol(spc::g_ss_prog, &q, sizeof(q)) == cudaSuccess ? SPC_OK : SPC_E_CUDA;
}

extern "C" int spc_debug_set_ss_time(void* p) {  // tools only; not in include/spc.h
  unsigned long long* q = (unsigned long long*)p;
  return cudaMemcpyToSymbol(spc::g_ss_time, &q, sizeof(q)) == cudaSuccess ? SPC_OK : SPC_E_CUDA;
}

extern "C" int spc_score_select_supported(int B, int Hq, int G, int D, int Smax, int k) {
  return ss_geometry(B, Hq, G, D, Smax, k, nullptr) == SPC_OK;
}

extern "C" size_t spc_score_select_workspace(int B, int Hq, int G, int Smax) {
  if (B <= 0 || Hq <= 0 || G <= 0 || Smax <= 0) return 0;
  return ss_ws_layout(nullptr, B, Hq, G, Smax, SS_MAX_CTAS).bytes;
}

extern "C" int spc_score_select(const void* q, const void* kr, const int32_t* seq_len, int B, int Hq,
                                int G, int D, int Smax, float scale, int k, int force_last,
                                float* logits, float* head_max, int64_t* head_sumfix,
                                float* group_score, int32_t* out_idx, int32_t* out_count,
                                const int32_t* prev_idx, const int32_t* prev_count,
                                int32_t* load_tok, int32_t* n_load, int32_t* evict_tok,
                                int32_t* n_evict, void* ws, size_t ws_bytes, spc_stream_t stream) {
  if (!q || !kr || !seq_len || !head_max || !head_sumfix || !group_score || !out_idx ||
      !out_count || !prev_idx || !prev_count || !load_tok || !n_load)
    return SPC_E_NULL;
  int ncta = 0;
  SPC_TRY(ss_geometry(B, Hq, G, D, Smax, k, &ncta));
  if (((uintptr_t)kr & 15) != 0 || ((uintptr_t)q & 15) != 0) return SPC_E_RANGE;
  if (!ws || ws_bytes < spc_score_select_workspace(B, Hq, G, Smax)) return SPC_E_WORKSPACE;
  const SsWs w = ss_ws_layout(ws, B, Hq, G, Smax, SS_MAX_CTAS);
  cudaStream_t st = as_stream(stream);
  const int alpha = Hq / G;
#define SS(DD, AA)                                                                               \
  if (D == DD && alpha == AA)                                                                    \
    return ss_launch<DD, AA>((const uint16_t*)q, (const uint16_t*)kr, seq_len, B, G, Smax, scale, k, \
                             force_last, logits, head_max, head_sumfix, group_score, out_idx,      \
                             out_count, prev_idx, prev_count, load_tok, n_load, evict_tok, n_evict, \
                             w, ncta, st);
  SS(64, 1) SS(64, 2) SS(64, 4) SS(64, 8) SS(128, 1) SS(128, 2) SS(128, 4) SS(128, 8)
#undef SS
  return SPC_E_UNSUPPORTED;
}
