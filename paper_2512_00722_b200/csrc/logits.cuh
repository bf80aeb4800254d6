// logits.cuh — phase LOGITS of spc_score (O1, O2); included by score.cu.
//
// Persistent, one CTA of LG_W warps per SM, per-warp cp.async pipelines.
// The retrieval-key cache [B*G][Smax][D] is cut into tiles of 128 rows; CTA c
// owns tiles [c*tpc, (c+1)*tpc) (tpc <= tiles per group, so a CTA spans at most
// two KV groups).  The CTA's warps claim tiles dynamically (shared counter).
// A tile is streamed in steps of 32 d (128 rows x 64 B = 8 KiB, 16-byte
// cp.async copies into 80-byte padded shared rows: conflict-free LDS.128) through
// a per-warp 3-stage ring, two steps in flight while one is consumed.
//   Measured alternative: TMA 2-D boxes of 64/128-byte rows are
//   limited by the TMA unit's per-row rate (~1.9-2.6 TB/s for this kernel).
//
// Lane l owns rows l, l+32, l+64, l+96 of a tile and runs, per row and per
// query head of the group, the contract's sequential fp32 FMA chain over d (O1),
// two rows at a time with the packed sm_100 FFMA2 (fma.rn.f32x2 = two IEEE fmaf,
// order kept): 8 independent chains per lane.  The group's query is staged once
// per CTA in shared memory as {q, q} pairs.  One key row serves all alpha query
// heads (no repeat_kv).  Running maxima are reduced per CTA and group; the last
// CTA of a group (ticket) reduces the segments to head_max (O2: exact).
#pragma once

#ifndef SPC_LG_RPT
#define SPC_LG_RPT 4
#endif
#ifndef SPC_LG_WARPS
#define SPC_LG_WARPS 6
#endif
constexpr int LG_RPT = SPC_LG_RPT;        // rows per lane (LG_RPT / 2 FFMA2 row pairs)
constexpr int LG_TR = 32 * LG_RPT;        // rows per tile
#ifndef SPC_LG_DCH
#define SPC_LG_DCH 64
#endif
constexpr int LG_DCH = SPC_LG_DCH;        // d per pipeline step
constexpr int LG_RS = LG_DCH * 2 + 16;    // padded shared row: 144 B (conflict-free LDS.128)
constexpr int LG_STAGE = LG_TR * LG_RS;   // 18 KiB at 4 rows per lane
constexpr int LG_NST = 2;                 // per-warp ring depth: one step loads while one computes
template <int ALPHA>
constexpr int lg_warps() {  // warps per CTA (one CTA per SM), bounded by the shared ring
  return ALPHA >= 8 ? SPC_LG_WARPS * 5 / 6 : SPC_LG_WARPS;
}

template <int D, int ALPHA>
struct Lg4Smem {
  static constexpr int LG_W = lg_warps<ALPHA>();
  static constexpr int NCH = D < LG_DCH ? 1 : D / LG_DCH;
  static constexpr int DCH = D < LG_DCH ? D : LG_DCH;   // d per step
  static constexpr int RING = LG_W * LG_NST * LG_STAGE;
  static constexpr int Q_OFF = RING;                          // [2 groups][D][ALPHA] float2
  static constexpr int Q_BYTES = D * ALPHA * 8;
  static constexpr int META_OFF = Q_OFF + 2 * Q_BYTES;        // per warp: stage tiles [NST]
  static constexpr int RED_OFF = META_OFF + LG_W * LG_NST * 4;  // [LG_W][2][ALPHA] float
  static constexpr int BYTES = RED_OFF + LG_W * 2 * ALPHA * 4 + 16;
};

template <int D, int ALPHA>
__global__ void __launch_bounds__(32 * lg_warps<ALPHA>(), 1) logits_kernel(
    const uint16_t* __restrict__ kr, const uint16_t* __restrict__ q,
    const int32_t* __restrict__ seq_len, int G, int Smax, float scale, int tpc, int tpr,
    int ntiles, float* __restrict__ logits, float* __restrict__ seg_max, int segstride,
    unsigned int* __restrict__ counters, float* __restrict__ head_max) {
  spc_pdl_entry();
  using SM = Lg4Smem<D, ALPHA>;
  constexpr int NCH = SM::NCH, DCH = SM::DCH, LG_W = SM::LG_W, LG_T = 32 * LG_W;
  constexpr int GPR = DCH / 8;         // 16-byte granules per row and step
  constexpr int RPI = 32 / GPR;        // rows per warp-wide copy instruction
  extern __shared__ __align__(16) uint8_t lg_raw[];
  __shared__ int next_tile, flag;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int Hq = G * ALPHA;
  const int t_begin = blockIdx.x * tpc;
  const int t_end = min(t_begin + tpc, ntiles);
  if (t_begin >= t_end) return;
  const int bg0 = t_begin / tpr;                 // first group of this CTA
  const int ngrp = (t_end - 1) / tpr - bg0 + 1;  // 1 or 2
  float* red = (float*)(lg_raw + SM::RED_OFF);
  int* stage_tile = (int*)(lg_raw + SM::META_OFF) + warp * LG_NST;
  const uint32_t ring = smem_u32(lg_raw + (size_t)warp * LG_NST * LG_STAGE);

  // stage the query of the (at most two) groups as {q, q} pairs
  for (int i = tid; i < ngrp * D * ALPHA; i += LG_T) {
    const int gi = i / (D * ALPHA), r = i - gi * (D * ALPHA);
    const int d = r / ALPHA, j = r - (r / ALPHA) * ALPHA;
    const int bg = bg0 + gi, b = bg / G, g = bg - (bg / G) * G;
    const float v = __uint_as_float((uint32_t)q[((size_t)b * Hq + g * ALPHA + j) * D + d] << 16);
    ((float2*)(lg_raw + SM::Q_OFF))[i] = make_float2(v, v);
  }
  if (tid == 0) next_tile = t_begin;
  __syncthreads();

  // ---- per-warp pipeline over steps (tile, chunk); tiles claimed from the CTA range
  int p_tile = -1, p_chunk = NCH;  // producer cursor
  auto issue = [&](int st) {       // next step -> stage st (or an empty group)
    if (p_chunk == NCH) {
      int t = 0;
      if (lane == 0) t = atomicAdd(&next_tile, 1);
      p_tile = __shfl_sync(0xffffffffu, t, 0);
      p_chunk = 0;
    }
    if (lane == 0) stage_tile[st] = p_tile < t_end ? p_tile * NCH + p_chunk : -1;
    if (p_tile < t_end) {
      const int bg = p_tile / tpr, t0 = (p_tile - bg * tpr) * LG_TR;
      const int S = __ldg(seq_len + bg / G);
      const int r_lane = lane / GPR, gr = lane % GPR;
      const uint16_t* src = kr + ((size_t)bg * Smax + t0 + r_lane) * D + p_chunk * DCH + gr * 8;
      const uint32_t dst = ring + (uint32_t)st * LG_STAGE + r_lane * LG_RS + gr * 16;
      if (t0 + LG_TR <= S) {  // full tile: no per-row predicates
#pragma unroll
        for (int j = 0; j < LG_TR / RPI; ++j)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + j * RPI * LG_RS),
                       "l"(src + (size_t)j * RPI * D)
                       : "memory");
      } else {
#pragma unroll
        for (int j = 0; j < LG_TR / RPI; ++j)
          if (t0 + j * RPI + r_lane < S)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + j * RPI * LG_RS),
                         "l"(src + (size_t)j * RPI * D)
                         : "memory");
      }
    }
    ++p_chunk;
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  float2 acc[ALPHA][LG_RPT / 2];  // [head][row pair]: pair p = rows lane + 64p, lane + 64p + 32
  float hm[2][ALPHA];
#pragma unroll
  for (int j = 0; j < ALPHA; ++j) hm[0][j] = hm[1][j] = -INFINITY;

  for (int s = 0; s < LG_NST - 1; ++s) issue(s);
  for (int st = 0;; st = st == LG_NST - 1 ? 0 : st + 1) {
    issue(st == 0 ? LG_NST - 1 : st - 1);  // the stage consumed last iteration
    asm volatile("cp.async.wait_group %0;" ::"n"(LG_NST - 1) : "memory");
    __syncwarp();
    const int code = stage_tile[st];
    if (code < 0) break;  // steps are consumed in order: the first empty one ends the warp
    const int tile = code / NCH, c = code - tile * NCH;
    const int bg = tile / tpr, t0 = (tile - bg * tpr) * LG_TR;
    const int b = bg / G, gi = bg - bg0;
    const int S = __ldg(seq_len + b);
    if (c == 0) {
#pragma unroll
      for (int j = 0; j < ALPHA; ++j)
#pragma unroll
        for (int p = 0; p < LG_RPT / 2; ++p) acc[j][p] = make_float2(0.f, 0.f);
    }
    if (t0 < S) {
      const uint32_t kc = ring + (uint32_t)st * LG_STAGE;
      const uint32_t qbase = smem_u32(lg_raw + SM::Q_OFF + gi * SM::Q_BYTES);
#pragma unroll 2
      for (int u = 0; u < DCH / 8; ++u) {  // 16-byte granule = 8 consecutive d
        uint4 w[LG_RPT];
#pragma unroll
        for (int i = 0; i < LG_RPT; ++i) w[i] = lds128(kc + (lane + 32 * i) * LG_RS + u * 16);
        const uint32_t qd = qbase + (uint32_t)(c * DCH + u * 8) * ALPHA * 8;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          float2 kk[LG_RPT / 2];
#pragma unroll
          for (int p = 0; p < LG_RPT / 2; ++p) {
            const uint32_t x0 = (&w[2 * p].x)[e >> 1], x1 = (&w[2 * p + 1].x)[e >> 1];
            kk[p] = (e & 1) ? make_float2(bf16hi(x0), bf16hi(x1)) : make_float2(bf16lo(x0), bf16lo(x1));
          }
#pragma unroll
          for (int j = 0; j < ALPHA; j += 2) {
            if (ALPHA >= 2) {
              const float4 q4 = lds128f(qd + (uint32_t)(e * ALPHA + j) * 8);
#pragma unroll
              for (int p = 0; p < LG_RPT / 2; ++p) {
                acc[j][p] = ffma2(kk[p], make_float2(q4.x, q4.y), acc[j][p]);
                acc[j + 1][p] = ffma2(kk[p], make_float2(q4.z, q4.w), acc[j + 1][p]);
              }
            } else {
              const float2 q2 = lds64f(qd + (uint32_t)(e * ALPHA + j) * 8);
#pragma unroll
              for (int p = 0; p < LG_RPT / 2; ++p) acc[j][p] = ffma2(kk[p], q2, acc[j][p]);
            }
          }
        }
      }
      if (c == NCH - 1) {  // O1 final multiply by scale, store, O2 running max
        const int g = bg - b * G;
#pragma unroll
        for (int j = 0; j < ALPHA; ++j) {
          float* o = logits + ((size_t)b * Hq + g * ALPHA + j) * Smax + t0;
#pragma unroll
          for (int i = 0; i < LG_RPT; ++i) {  // row lane + 32 i = pair i/2, half i%2
            const int r = lane + 32 * i;
            const float sv = __fmul_rn((i & 1) ? acc[j][i >> 1].y : acc[j][i >> 1].x, scale);
            if (t0 + r < S) {
              o[r] = sv;
              if (gi == 0)
                hm[0][j] = fmaxf(hm[0][j], sv);
              else
                hm[1][j] = fmaxf(hm[1][j], sv);
            }
          }
        }
      }
    }
    __syncwarp();  // every lane is done with stage st before it is refilled
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");

  // ---- per-CTA maxima of the (one or two) groups -> seg_max; group tickets -> head_max
#pragma unroll
  for (int gi = 0; gi < 2; ++gi)
#pragma unroll
    for (int j = 0; j < ALPHA; ++j) {
      const float m = warp_max(hm[gi][j]);
      if (lane == 0) red[(warp * 2 + gi) * ALPHA + j] = m;
    }
  __syncthreads();
  for (int gi = 0; gi < ngrp; ++gi) {
    const int bg = bg0 + gi, b = bg / G, g = bg - (bg / G) * G;
    const int first = (bg * tpr) / tpc, last = (bg * tpr + tpr - 1) / tpc;
    if (tid < ALPHA) {
      float m = -INFINITY;
      for (int w = 0; w < LG_W; ++w) m = fmaxf(m, red[(w * 2 + gi) * ALPHA + tid]);
      seg_max[((size_t)b * Hq + g * ALPHA + tid) * segstride + (blockIdx.x - first)] = m;
    }
    if (last_block_ticket(&counters[bg], last - first + 1, &flag)) {
      if (tid < ALPHA) {
        const float* sm = seg_max + ((size_t)b * Hq + g * ALPHA + tid) * segstride;
        float m = -INFINITY;
        for (int i = 0; i <= last - first; ++i) m = fmaxf(m, __ldcg(sm + i));
        head_max[(size_t)b * Hq + g * ALPHA + tid] = m;
      }
    }
  }
}
