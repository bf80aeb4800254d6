// logits.cuh — phase LOGITS of spc_score (O1, O2); included by score.cu.
//
// Persistent, one CTA of LG_W warps per SM, every warp an autonomous cp.async
// pipeline.  The retrieval-key cache [B*G][Smax][D] is cut into tiles of 128 rows;
// warps claim tiles from ONE grid-wide counter (a warp's first tile is its grid-wide
// warp index; later claims are prefetched one tile ahead, so the atomic's latency hides
// behind the math), which balances the grid to within one tile.  A tile is streamed in steps of 64 d (128 rows x 128 B =
// 16 KiB, 16-byte cp.async copies) through a per-warp 2-stage ring; rows are
// stored unpadded with the 16-byte granule index XOR-swizzled by (row & 7), so the
// lane-per-row LDS.128 reads are conflict-free.  A tile's first step also carries
// the raw bf16 query of its group (alpha x D), which the warp converts once into a
// per-warp fp32 [D][alpha] table: any warp can take any group's tile.
//   Measured alternatives: per-CTA tile ranges (a CTA's 14 tiles
//   over 6 warps: 3-vs-2.3 imbalance, 25-27 us on config B); TMA 2-D boxes (per-row
//   rate bound, ~1.9-2.6 TB/s).
//
// Lane l owns rows l, l+32, l+64, l+96 of a tile and runs, per row and per query
// head of the group, the contract's sequential fp32 FMA chain over d (O1), two rows
// at a time with the packed sm_100 FFMA2 (fma.rn.f32x2 = two IEEE fmaf, order
// kept; the query value is a scalar-broadcast operand): 2 x alpha independent
// chains per lane.  One key row serves all alpha query heads (no repeat_kv).
// O2 (head max, exact and order-free): per tile a warp max per head, stored to a
// [B*Hq][tiles] workspace table with plain stores; lg_finalize_kernel (launched
// right behind, PDL) reduces each head's row to head_max and re-zeroes the claim
// counter.  Measured (tools/lg_bench2.cu, config B): an atomicMax per tile on 32
// addresses (+2.5 us: same-address serialisation) and a grid-wide last-warp ticket
// with its fences (+2.7 us) both cost more than the extra launch.
#pragma once

#ifndef SPC_LG_WARPS
#define SPC_LG_WARPS 6
#endif
#ifndef SPC_LG_RPT
#define SPC_LG_RPT 4
#endif
constexpr int LG_RPT = SPC_LG_RPT;        // rows per lane (LG_RPT / 2 FFMA2 row pairs)
constexpr int LG_TR = 32 * LG_RPT;        // rows per tile
constexpr int LG_DCH = 64;                // d per pipeline step (128-byte row pieces)
constexpr int LG_STAGE = LG_TR * LG_DCH * 2;  // 16 KiB at 4 rows per lane, unpadded (swizzled granules)
constexpr int LG_NST = 2;                 // per-warp ring depth: one step loads while one computes
template <int ALPHA>
constexpr int lg_warps() {  // warps per CTA (one CTA per SM), bounded by shared memory
  return ALPHA >= 8 ? SPC_LG_WARPS * 5 / 6 : SPC_LG_WARPS;
}

template <int D, int ALPHA>
struct LgSmem {
  static constexpr int LG_W = lg_warps<ALPHA>();
  static constexpr int NCH = D / LG_DCH;
  static constexpr int QRAW = ALPHA * D * 2;                  // raw bf16 query of a tile's group
  static constexpr int SLOT = LG_STAGE + QRAW;                // one ring stage
  static constexpr int RING = LG_W * LG_NST * SLOT;
  static constexpr int QF_OFF = RING;                         // per warp: fp32 [D][ALPHA]
  static constexpr int QF = D * ALPHA * 4;
  static constexpr int META_OFF = QF_OFF + LG_W * QF;         // per warp: stage codes [NST]
  static constexpr int BYTES = META_OFF + LG_W * LG_NST * 4 + 16;
};

template <int D, int ALPHA>
__global__ void __launch_bounds__(32 * lg_warps<ALPHA>(), 1) logits_kernel(
    const uint16_t* __restrict__ kr, const uint16_t* __restrict__ q,
    const int32_t* __restrict__ seq_len, int G, int Smax, float scale, int tpr, int ntiles,
    float* __restrict__ logits, float* __restrict__ tile_max, unsigned* __restrict__ ctr) {
  spc_pdl_entry();
  using SM = LgSmem<D, ALPHA>;
  constexpr int NCH = SM::NCH, LG_W = SM::LG_W;
  constexpr int GPR = LG_DCH / 8;  // 16-byte granules per row piece (8)
  constexpr int RPI = 32 / GPR;    // rows per warp-wide copy instruction (4)
  constexpr int QG = SM::QRAW / 16;  // 16-byte granules of the raw query
  extern __shared__ __align__(128) uint8_t lg_raw[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int Hq = G * ALPHA;
  int* stage_code = (int*)(lg_raw + SM::META_OFF) + warp * LG_NST;
  const uint32_t ring = smem_u32(lg_raw + (size_t)warp * LG_NST * SM::SLOT);
  float* qf = (float*)(lg_raw + SM::QF_OFF + warp * SM::QF);
  const uint32_t qf_s = smem_u32(qf);

  // ---- per-warp pipeline over steps (tile, chunk); tiles claimed from the grid counter
  int cur = 0, chunk = NCH;  // producer cursor
  // the first tile of every warp is static (its grid-wide warp index: no atomic round trip
  // before the first loads); later claims come from the counter, offset past those
  const int nwarps = gridDim.x * LG_W;
  int nxt = blockIdx.x * LG_W + warp;
  const int r_lane = lane / GPR, gr = lane % GPR;
  // swizzled destination granule for the two row parities of the copy pattern
  const uint32_t sw0 = (uint32_t)((gr ^ (r_lane & 7)) << 4), sw1 = (uint32_t)((gr ^ ((r_lane + 4) & 7)) << 4);
  auto issue = [&](int st) {  // next step -> stage st (or an end marker)
    if (chunk == NCH) {       // next tile: take the prefetched claim, prefetch the one after
      for (;;) {
        cur = nxt;
        if (cur >= ntiles) break;
        int t = 0;
        if (lane == 0) t = (int)atomicAdd(ctr, 1u) + nwarps;
        nxt = __shfl_sync(0xffffffffu, t, 0);
        const int bg = cur / tpr;
        if ((cur - bg * tpr) * LG_TR < __ldg(seq_len + bg / G)) break;
        if (lane < ALPHA) {  // an empty tile (ragged batch): its maxima are -inf
          const int b = bg / G, g = bg - b * G;
          tile_max[((size_t)b * Hq + g * ALPHA + lane) * tpr + (cur - bg * tpr)] = -INFINITY;
        }
      }
      chunk = 0;
    }
    if (lane == 0) stage_code[st] = cur < ntiles ? cur * NCH + chunk : -1;
    if (cur < ntiles) {
      const int bg = cur / tpr, t0 = (cur - bg * tpr) * LG_TR;
      const int S = __ldg(seq_len + bg / G);
      const uint16_t* src = kr + ((size_t)bg * Smax + t0 + r_lane) * D + chunk * LG_DCH + gr * 8;
      const uint32_t dst = ring + (uint32_t)st * SM::SLOT + r_lane * (LG_DCH * 2);
      if (t0 + LG_TR <= S) {  // full tile: no per-row predicates
#pragma unroll
        for (int j = 0; j < LG_TR / RPI; ++j)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                           dst + j * RPI * (LG_DCH * 2) + ((j & 1) ? sw1 : sw0)),
                       "l"(src + (size_t)j * RPI * D)
                       : "memory");
      } else {
#pragma unroll
        for (int j = 0; j < LG_TR / RPI; ++j)
          if (t0 + j * RPI + r_lane < S)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                             dst + j * RPI * (LG_DCH * 2) + ((j & 1) ? sw1 : sw0)),
                         "l"(src + (size_t)j * RPI * D)
                         : "memory");
      }
      if (chunk == 0) {  // the group's raw query rides along with the tile's first step
        const int b = bg / G, g = bg - b * G;
        const uint16_t* qs = q + ((size_t)b * Hq + g * ALPHA) * D;
        for (int i = lane; i < QG; i += 32)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                           ring + (uint32_t)st * SM::SLOT + LG_STAGE + i * 16),
                       "l"(qs + i * 8)
                       : "memory");
      }
    }
    ++chunk;
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  float2 acc[ALPHA][LG_RPT / 2];  // [head][row pair]: pair p = rows lane + 64p, lane + 64p + 32
  const uint32_t swz = (uint32_t)(lane & 7) << 4;

  for (int s = 0; s < LG_NST - 1; ++s) issue(s);
  for (int st = 0;; st = st == LG_NST - 1 ? 0 : st + 1) {
    issue(st == 0 ? LG_NST - 1 : st - 1);  // the stage consumed last iteration
    asm volatile("cp.async.wait_group %0;" ::"n"(LG_NST - 1) : "memory");
    __syncwarp();
    const int code = stage_code[st];
    if (code < 0) break;  // steps are consumed in order: the first end marker ends the warp
    const int tile = code / NCH, c = code - tile * NCH;
    const int bg = tile / tpr, t0 = (tile - bg * tpr) * LG_TR;
    const int b = bg / G;
    const int S = __ldg(seq_len + b);
    const uint32_t kc = ring + (uint32_t)st * SM::SLOT;
    if (c == 0) {
#pragma unroll
      for (int j = 0; j < ALPHA; ++j)
#pragma unroll
        for (int p = 0; p < LG_RPT / 2; ++p) acc[j][p] = make_float2(0.f, 0.f);
      // raw [ALPHA][D] bf16 -> fp32 [D][ALPHA]
      const uint16_t* qr = (const uint16_t*)(lg_raw + (size_t)warp * LG_NST * SM::SLOT +
                                             (size_t)st * SM::SLOT + LG_STAGE);
      for (int i = lane; i < ALPHA * D; i += 32) {
        const int j = i / D, d = i - j * D;
        qf[d * ALPHA + j] = __uint_as_float((uint32_t)qr[i] << 16);
      }
      __syncwarp();
    }
    {
      const uint32_t kl = kc + (uint32_t)lane * (LG_DCH * 2);
#pragma unroll 2
      for (int u = 0; u < LG_DCH / 8; ++u) {  // 16-byte granule = 8 consecutive d
        uint4 w[LG_RPT];
        const uint32_t ka = kl + (((uint32_t)u << 4) ^ swz);
#pragma unroll
        for (int i = 0; i < LG_RPT; ++i) w[i] = lds128(ka + i * 32 * (LG_DCH * 2));
        const uint32_t qd = qf_s + (uint32_t)(c * LG_DCH + u * 8) * ALPHA * 4;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          float2 kk[LG_RPT / 2];
#pragma unroll
          for (int p = 0; p < LG_RPT / 2; ++p) {
            const uint32_t x0 = (&w[2 * p].x)[e >> 1], x1 = (&w[2 * p + 1].x)[e >> 1];
            kk[p] = (e & 1) ? make_float2(bf16hi(x0), bf16hi(x1)) : make_float2(bf16lo(x0), bf16lo(x1));
          }
#pragma unroll
          for (int j = 0; j < ALPHA; j += 4) {
            if (ALPHA >= 4) {
              const float4 q4 = lds128f(qd + (uint32_t)(e * ALPHA + j) * 4);
#pragma unroll
              for (int p = 0; p < LG_RPT / 2; ++p) {
                acc[j][p] = ffma2(kk[p], make_float2(q4.x, q4.x), acc[j][p]);
                acc[j + 1][p] = ffma2(kk[p], make_float2(q4.y, q4.y), acc[j + 1][p]);
                acc[j + 2][p] = ffma2(kk[p], make_float2(q4.z, q4.z), acc[j + 2][p]);
                acc[j + 3][p] = ffma2(kk[p], make_float2(q4.w, q4.w), acc[j + 3][p]);
              }
            } else if (ALPHA == 2) {
              const float2 q2 = lds64f(qd + (uint32_t)(e * ALPHA) * 4);
#pragma unroll
              for (int p = 0; p < LG_RPT / 2; ++p) {
                acc[0][p] = ffma2(kk[p], make_float2(q2.x, q2.x), acc[0][p]);
                acc[ALPHA - 1][p] = ffma2(kk[p], make_float2(q2.y, q2.y), acc[ALPHA - 1][p]);
              }
            } else {
              const float q1 = qf[c * LG_DCH + u * 8 + e];
#pragma unroll
              for (int p = 0; p < LG_RPT / 2; ++p) acc[0][p] = ffma2(kk[p], make_float2(q1, q1), acc[0][p]);
            }
          }
        }
      }
    }
    if (c == NCH - 1) {  // O1 final multiply by scale, store, O2 tile max -> tile_max
      const int g = bg - b * G;
      float tm = 0.0f;
#pragma unroll
      for (int j = 0; j < ALPHA; ++j) {
        float* o = logits + ((size_t)b * Hq + g * ALPHA + j) * Smax + t0;
        float m = -INFINITY;
#pragma unroll
        for (int i = 0; i < LG_RPT; ++i) {  // row lane + 32 i = pair i/2, half i%2
          const int r = lane + 32 * i;
          const float sv = __fmul_rn((i & 1) ? acc[j][i >> 1].y : acc[j][i >> 1].x, scale);
          if (t0 + r < S) {
            SPC_DCHECK(sv == sv, SPC_E_RANGE);  // NaN key / query (reading R20)
            o[r] = sv;
            m = fmaxf(m, sv);
          }
        }
        m = warp_max(m);
        if (lane == j) tm = m;
      }
      if (lane < ALPHA) tile_max[((size_t)b * Hq + g * ALPHA + lane) * tpr + (tile - bg * tpr)] = tm;
    }
    __syncwarp();  // every lane is done with stage st before it is refilled
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");

}

// head_max[h] = max over the head's tile maxima (O2): one CTA of 256 threads per head,
// float4 loads when the row allows (8,192 tiles per head at 1M tokens).  Also re-zeroes the
// tile-claim counter for the next LOGITS launch (stream order: LOGITS is complete).
__global__ void __launch_bounds__(256) lg_finalize_kernel(const float* __restrict__ tile_max, int tpr,
                                                          int nheads, float* __restrict__ head_max,
                                                          unsigned* __restrict__ ctr) {
  spc_pdl_entry();
  __shared__ float red[8];
  const int h = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (h == 0 && tid == 0) ctr[0] = 0u;
  const float* row = tile_max + (size_t)h * tpr;
  float m = -INFINITY;
  if ((tpr & 3) == 0) {
    const float4* r4 = reinterpret_cast<const float4*>(row);
    for (int i = tid; i < tpr / 4; i += 256) {
      const float4 v = __ldcg(r4 + i);
      m = fmaxf(fmaxf(m, v.x), fmaxf(v.y, fmaxf(v.z, v.w)));
    }
  } else {
    for (int i = tid; i < tpr; i += 256) m = fmaxf(m, __ldcg(row + i));
  }
  m = warp_max(m);
  if (lane == 0) red[warp] = m;
  __syncthreads();
  if (tid == 0) {
    float r = red[0];
#pragma unroll
    for (int w = 1; w < 8; ++w) r = fmaxf(r, red[w]);
    head_max[h] = r;
  }
  (void)nheads;
}

// ------------------------------------------------------------------------------------
// logits_tma_kernel — the same phase (O1 chains, O2 per-tile maxima, same outputs) with the
// key tiles streamed by the TMA unit.  One CTA per SM = one producer warp + LT_NC consumer
// warps over a ring of half-tile stages (128 rows x 64 d = 16 KiB, 2-D tensor-map boxes
// with the 128-byte swizzle: granule g of row r at g ^ (r & 7), the layout the consumer's
// conflict-free LDS.128 expects).  The producer lane issues, per stage, one
// cp.async.bulk.tensor.2d box (and on a tile's first stage a 1-D bulk copy of the group's
// raw bf16 query), completion counted on the stage's mbarrier; consumers take whole tiles
// round robin, each from its own ring of K stages, run the unchanged FFMA2 inner loop and
// release each stage.  CTA c owns the
// contiguous tiles [c*n/grid, (c+1)*n/grid).  Measured (tools/tmatile.cu): 64 MiB streamed
// by 16 KiB TMA boxes in 12.65 us per back-to-back launch vs 12.41 us for an LDG.128 stream
// -- the consumers no longer spend issue slots on 16-byte copies.
#ifndef SPC_LT_NC
#define SPC_LT_NC 8  // consumer warps
#endif
#ifndef SPC_LT_CPR
#define SPC_LT_CPR 2  // consumer warps per ring: they split every stage's 128 rows
#endif
#ifndef SPC_LT_BATCH
#define SPC_LT_BATCH 0  // tiles per claim of a producer lane; 0: by the launch (below)
#endif
constexpr int LT_NC = SPC_LT_NC;     // consumer warps
constexpr int LT_CPR = SPC_LT_CPR;   // consumers per ring (= tile_max entries per tile)
constexpr int LT_RINGS = LT_NC / LT_CPR;
constexpr int LT_RPT = LG_RPT / LT_CPR;  // key rows per lane
static_assert(LT_NC % LT_CPR == 0 && LT_RPT >= 2 && LT_RPT % 2 == 0, "LOGITS consumer split");
constexpr int LT_STAGE = LG_TR * 128;  // 128 rows x 128 bytes
template <int D, int ALPHA>
struct LtSmem {
  static constexpr int NCH = D / 64;
  static constexpr int QRAW = ALPHA * D * 2;
  static constexpr int QF = D * ALPHA * 4;
  static constexpr int NST0 = (232448 - 2048 - LT_NC * QF) / (LT_STAGE + QRAW);
  static constexpr int K = (NST0 > 12 ? 12 : NST0) / LT_RINGS;  // stages per ring
  static constexpr int NST = K * LT_RINGS;
  static_assert(K >= 1, "ring too shallow");
  static constexpr int QSLOT_OFF = NST * LT_STAGE;
  static constexpr int QF_OFF = QSLOT_OFF + NST * QRAW;
  static constexpr int BYTES = 1024 + QF_OFF + LT_NC * QF;
};

// O1 on RPT rows per lane of one TMA stage (128 rows x 64 d, 128-byte swizzle): lane l
// accumulates rows row0 + l + 32 r (r < RPT; row0 a multiple of 32), alpha sequential fp32
// chains per row, d ascending (chunk c covers d = 64 c .. 64 c + 63), FFMA2 on row pairs
// with the query value as a scalar-broadcast operand.  qf: the warp's fp32 [D][ALPHA] table.
template <int D, int ALPHA, int RPT>
__device__ __forceinline__ void lt_rows_math(float2 (&acc)[ALPHA][RPT / 2], uint32_t kc, int row0,
                                             uint32_t qf_s, const float* qf, int c, int lane) {
  const uint32_t swz = (uint32_t)(lane & 7) << 4;  // granule g of row r sits at g ^ (r & 7)
  const uint32_t kl = kc + (uint32_t)(row0 + lane) * 128u;
#ifdef SPC_LT_NOMATH  // debug builds only: the load pipeline alone
  if (lane < 0)
#endif
#pragma unroll 2
    for (int u = 0; u < 8; ++u) {  // 16-byte granule = 8 consecutive d
      uint4 w[RPT];
      const uint32_t ka = kl + (((uint32_t)u << 4) ^ swz);
#pragma unroll
      for (int r = 0; r < RPT; ++r) w[r] = lds128(ka + r * 32 * 128);
      const uint32_t qd = qf_s + (uint32_t)(c * 64 + u * 8) * ALPHA * 4;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        float2 kk[RPT / 2];
#pragma unroll
        for (int p = 0; p < RPT / 2; ++p) {
          const uint32_t x0 = (&w[2 * p].x)[e >> 1], x1 = (&w[2 * p + 1].x)[e >> 1];
          kk[p] = (e & 1) ? make_float2(bf16hi(x0), bf16hi(x1)) : make_float2(bf16lo(x0), bf16lo(x1));
        }
#pragma unroll
        for (int j = 0; j < ALPHA; j += 4) {
          if (ALPHA >= 4) {
            const float4 q4 = lds128f(qd + (uint32_t)(e * ALPHA + j) * 4);
#pragma unroll
            for (int p = 0; p < RPT / 2; ++p) {
              acc[j][p] = ffma2(kk[p], make_float2(q4.x, q4.x), acc[j][p]);
              acc[j + 1][p] = ffma2(kk[p], make_float2(q4.y, q4.y), acc[j + 1][p]);
              acc[j + 2][p] = ffma2(kk[p], make_float2(q4.z, q4.z), acc[j + 2][p]);
              acc[j + 3][p] = ffma2(kk[p], make_float2(q4.w, q4.w), acc[j + 3][p]);
            }
          } else if (ALPHA == 2) {
            const float2 q2 = lds64f(qd + (uint32_t)(e * ALPHA) * 4);
#pragma unroll
            for (int p = 0; p < RPT / 2; ++p) {
              acc[0][p] = ffma2(kk[p], make_float2(q2.x, q2.x), acc[0][p]);
              acc[ALPHA - 1][p] = ffma2(kk[p], make_float2(q2.y, q2.y), acc[ALPHA - 1][p]);
            }
          } else {
            const float q1 = qf[c * 64 + u * 8 + e];
#pragma unroll
            for (int p = 0; p < RPT / 2; ++p) acc[0][p] = ffma2(kk[p], make_float2(q1, q1), acc[0][p]);
          }
        }
      }
    }
}
// all LG_RPT rows of a lane (score_select.cu's LOGITS phase)
template <int D, int ALPHA>
__device__ __forceinline__ void lt_stage_math(float2 (&acc)[ALPHA][LG_RPT / 2], uint32_t kc,
                                              uint32_t qf_s, const float* qf, int c, int lane) {
  lt_rows_math<D, ALPHA, LG_RPT>(acc, kc, 0, qf_s, qf, c, lane);
}

template <int D, int ALPHA>
__global__ void __launch_bounds__(32 * (LT_NC + 1), 1) logits_tma_kernel(
    const __grid_constant__ CUtensorMap kmap, const uint16_t* __restrict__ q,
    const int32_t* __restrict__ seq_len, int G, int Smax, float scale, int tpr, int ntiles,
    float* __restrict__ logits, float* __restrict__ tile_max, unsigned* __restrict__ ctr,
    int lt_batch, int evict_first) {
  using SM = LtSmem<D, ALPHA>;
  constexpr int NCH = SM::NCH, NST = SM::NST, K = SM::K;
  constexpr int HROWS = LG_TR / LT_CPR;  // rows of a stage per consumer warp
  __shared__ __align__(8) uint64_t full[NST], empty[NST];
  __shared__ int stage_tile[NST];  // tile id of a tile's first stage (-1: end of the work)
  extern __shared__ __align__(16) uint8_t lt_raw[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int Hq = G * ALPHA;
  const uint32_t base = (smem_u32(lt_raw) + 1023u) & ~1023u;
  uint8_t* basep = lt_raw + (base - smem_u32(lt_raw));
  const uint32_t full0 = smem_u32(&full[0]), empty0 = smem_u32(&empty[0]);
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(full0 + 8 * s));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(empty0 + 8 * s), "r"(LT_CPR));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_tmap(&kmap);
  }
  __syncthreads();
  // before the PDL wait (the previous launch may still be running): pull this CTA's first,
  // static tiles into L2.  Only an L2 hint -- the keys are read by the TMA loads after the
  // wait, and L2 is coherent with any kernel that writes them (the front-end's newest key) --
  // so the HBM stream starts while the previous kernel drains (its last CTAs, its merge)
  if (warp == LT_NC && lane < LT_RINGS) {
    const int t_lo = ((int)blockIdx.x * LT_RINGS + lane) * lt_batch;
    for (int tile = t_lo; tile < min(t_lo + lt_batch, ntiles); ++tile) {
      const int bg = tile / tpr, tt = tile - bg * tpr;
#pragma unroll
      for (int c = 0; c < LtSmem<D, ALPHA>::NCH; ++c)
        asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(&kmap), "r"(64 * c),
                     "r"(bg * Smax + tt * LG_TR)
                     : "memory");
    }
  }
  spc_pdl_entry();
  if (warp == LT_NC) {
    // ------------------------------------------------------------ producers (lanes)
    // lane w < LT_RINGS feeds ring w on its own (divergent lanes progress independently), so
    // a ring whose consumers lag never blocks the issue for the other rings.  Tiles come in
    // batches of LT_BATCH consecutive tiles: a lane's first batch is static, the next ones
    // are claimed from one grid-wide counter, each claim issued a batch ahead (its latency
    // hides behind the current batch); the counter balances the SMs, whose streaming rates
    // differ (config E: 443 tiles per SM).  The LT_CPR consumers of a ring split each of its
    // stages' rows.
    if (lane < LT_RINGS) {
      const int LT_BATCH = lt_batch;
      const int w = lane;
      const int nstatic = (int)gridDim.x * LT_RINGS;
      int n = 0;  // tiles handed to ring w
      int batch = (int)blockIdx.x * LT_RINGS + w;
      int next = nstatic + (int)atomicAdd(ctr, 1u);
      for (;;) {
        const int t_lo = batch * LT_BATCH;
        if (t_lo >= ntiles) break;
        for (int tile = t_lo; tile < min(t_lo + LT_BATCH, ntiles); ++tile) {
          const int bg = tile / tpr, tt = tile - bg * tpr;
          if (tt * LG_TR >= __ldg(seq_len + bg / G)) {  // an empty tile (ragged batch)
            const int b = bg / G, g = bg - b * G;
            for (int j = 0; j < ALPHA; ++j)
              for (int hh = 0; hh < LT_CPR; ++hh)
                tile_max[(((size_t)b * Hq + g * ALPHA + j) * tpr + tt) * LT_CPR + hh] = -INFINITY;
            continue;
          }
          for (int c = 0; c < NCH; ++c) {
            const int j = n * NCH + c;  // sequence number in ring w
            const int s = w * K + j % K;
            if (j >= K) tm_wait(empty0 + 8 * s, ((j / K) - 1) & 1);
            const uint32_t fb = full0 + 8 * s;
            if (c == 0) stage_tile[s] = tile;  // published by the arrive below (release)
            tm_expect(fb, LT_STAGE + (c == 0 ? SM::QRAW : 0));
            if (evict_first) {  // a short stream inside a step: keep the step's hot set in L2
              uint64_t pol;
              asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
              asm volatile(
                  "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
                  " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(base + s * LT_STAGE),
                  "l"(&kmap), "r"(64 * c), "r"(bg * Smax + tt * LG_TR), "r"(fb), "l"(pol)
                  : "memory");
            } else {
              asm volatile(
                  "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                  " [%0], [%1, {%2, %3}], [%4];" ::"r"(base + s * LT_STAGE),
                  "l"(&kmap), "r"(64 * c), "r"(bg * Smax + tt * LG_TR), "r"(fb)
                  : "memory");
            }
            if (c == 0) {
              const int b = bg / G, g = bg - b * G;
              asm volatile(
                  "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                      base + SM::QSLOT_OFF + s * SM::QRAW),
                  "l"(q + ((size_t)b * Hq + g * ALPHA) * D), "r"(SM::QRAW), "r"(fb)
                  : "memory");
            }
          }
          ++n;
        }
        batch = next;
        if (batch * LT_BATCH < ntiles) next = nstatic + (int)atomicAdd(ctr, 1u);
      }
      // end of the work: the ring's next tile slot gets the end code
      const int j = n * NCH, s = w * K + j % K;
      if (j >= K) tm_wait(empty0 + 8 * s, ((j / K) - 1) & 1);
      stage_tile[s] = -1;
      tm_arrive(full0 + 8 * s);
    }
    return;
  }
  // -------------------------------------------------------------- consumers
  // per-ring consumers: each waits for every stage of its ring in order, so a parity wait is
  // never more than one phase ahead of its barrier (consumers skipping each other's stages
  // could alias phases); the LT_CPR consumers of a ring take rows half*HROWS .. +HROWS of
  // every stage, so two warps per scheduler hide each other's dependency stalls
  const int ring = warp / LT_CPR, half = warp - ring * LT_CPR;
  float* qf = (float*)(basep + SM::QF_OFF + warp * SM::QF);
  const uint32_t qf_s = smem_u32(qf);
  int qf_bg = -1;  // group whose query qf holds (consecutive tiles are mostly one group's)
  for (int n = 0;; ++n) {
    int tile = 0, bg = 0, t0 = 0, b = 0, g = 0, S = 0;
    float2 acc[ALPHA][LT_RPT / 2];
#pragma unroll
    for (int j = 0; j < ALPHA; ++j)
#pragma unroll
      for (int p = 0; p < LT_RPT / 2; ++p) acc[j][p] = make_float2(0.f, 0.f);
    bool done = false;
    for (int c = 0; c < NCH; ++c) {
      const int j = n * NCH + c;
      const int s = ring * K + j % K;
      tm_wait(full0 + 8 * s, (j / K) & 1);
      if (c == 0) {
        tile = stage_tile[s];
        if (tile < 0) {
          done = true;
          break;
        }
        bg = tile / tpr;
        t0 = (tile - bg * tpr) * LG_TR;
        b = bg / G;
        g = bg - b * G;
        S = __ldg(seq_len + b);
        if (bg != qf_bg) {  // raw [ALPHA][D] bf16 -> fp32 [D][ALPHA]
          qf_bg = bg;
          const uint16_t* qr = (const uint16_t*)(basep + SM::QSLOT_OFF + s * SM::QRAW);
          if (ALPHA == 4 && D % 128 == 0) {  // lane: 4 consecutive d of every head, 16-byte stores
#pragma unroll
            for (int d0 = 4 * lane; d0 < D; d0 += 128) {
              uint2 h[4];
#pragma unroll
              for (int jj = 0; jj < 4; ++jj) h[jj] = *reinterpret_cast<const uint2*>(qr + jj * D + d0);
#pragma unroll
              for (int dd = 0; dd < 4; ++dd) {
                float4 v;
                const int sh = (dd & 1) ? 0 : 16;
                const uint32_t m = (dd & 1) ? 0xFFFF0000u : 0xFFFFFFFFu;
                v.x = __uint_as_float(((dd < 2 ? h[0].x : h[0].y) << sh) & m);
                v.y = __uint_as_float(((dd < 2 ? h[1].x : h[1].y) << sh) & m);
                v.z = __uint_as_float(((dd < 2 ? h[2].x : h[2].y) << sh) & m);
                v.w = __uint_as_float(((dd < 2 ? h[3].x : h[3].y) << sh) & m);
                reinterpret_cast<float4*>(qf)[d0 + dd] = v;
              }
            }
          } else {
#pragma unroll 4
            for (int e = lane; e < ALPHA * D; e += 32) {
              const int jj = e / D, d = e - jj * D;
              qf[d * ALPHA + jj] = __uint_as_float((uint32_t)qr[e] << 16);
            }
          }
          __syncwarp();
        }
      }
      lt_rows_math<D, ALPHA, LT_RPT>(acc, base + s * LT_STAGE, half * HROWS, qf_s, qf, c, lane);
      __syncwarp();
      if (lane == 0) tm_arrive(empty0 + 8 * s);  // this warp's share of the stage is consumed
    }
    if (done) break;
    // O1 final multiply by scale, store, O2 maximum of this warp's rows -> tile_max
    float tm = 0.0f;
#pragma unroll
    for (int j = 0; j < ALPHA; ++j) {
      float* o = logits + ((size_t)b * Hq + g * ALPHA + j) * Smax + t0 + half * HROWS;
      float m = -INFINITY;
#pragma unroll
      for (int r = 0; r < LT_RPT; ++r) {  // row lane + 32 r = pair r/2, half r%2
        const int row = lane + 32 * r;
        const int tok = t0 + half * HROWS + row;
        const float sv = __fmul_rn((r & 1) ? acc[j][r >> 1].y : acc[j][r >> 1].x, scale);
        if (tok < S && tok < Smax) {
          SPC_DCHECK(sv == sv, SPC_E_RANGE);  // NaN key / query (reading R20)
          o[row] = sv;
          m = fmaxf(m, sv);
        }
      }
      m = warp_max(m);
      if (lane == j) tm = m;
    }
    if (lane < ALPHA)
      tile_max[(((size_t)b * Hq + g * ALPHA + lane) * tpr + (tile - bg * tpr)) * LT_CPR + half] = tm;
  }
}
