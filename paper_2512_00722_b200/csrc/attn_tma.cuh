// attn_tma.cuh — the bf16 sparse decode-attention kernel fed by TMA row gathers
// (spc_sparse_decode_attn_kv; included by attn.cu).  O10 per (layer, b, g), split over
// CTAs, partials merged with the LSE rule O12 (Eq.1 over the P:324 selected rows).
//
// Persistent, TM_CTAS CTAs per SM, each CTA = one TMA producer warp + TM_NCONS MMA consumer
// warps over a TM_NST-deep ring of TM_RPS-row stages (K and V of the same 32 selected rows;
// 5 CTAs x 2 stages x 2 consumers per SM, consumer c taking the stages j = c mod 2).
// The selected rows of all groups (layer, b, g) form one virtual row space of
// n_groups x kpad rows (kpad = k rounded up to whole stages); CTA c owns a contiguous
// range of stages.
//
// Producer (warp 0): lane i < TM_RPS/4 issues, per stage, the
//   cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4
// requests for rows 4i..4i+3 of K and of V (one per 128-byte half row: SWIZZLE_128B boxes
// of 64 bf16 x 1 row, 4 rows per request), against the layer's tensor map from the
// caller's spc_kv_desc (tensor = [B*G*rows][D]).  Row coordinate = bg*rows + token; rows
// past the group's count get coordinate -1, which the TMA unit zero-fills (OOB).  The
// tokens and the group count of stage j + TM_PF are loaded while stage j issues.
// Measured (tools/tmagather.cu, 256 MiB of random 256-byte K+V rows): 45.7 us with 4
// producer warps per SM (5.87 TB/s) vs 43.1 us for a 64-warp LDG gather; one producer
// warp per SM is issue-bound at ~2 TB/s.  The consumer's smem reads are conflict-free
// because the 16-byte granule c of row r sits at c ^ (r & 7) (128-byte swizzle).
//
// Consumers (warps 1, 2): the transposed mma.sync products of attn_bf16.cuh on two 16-row
// tiles per stage -- S^T = K Q^T (K rows fill M) and O^T += V^T P with P's columns
// [P_hi | P_lo] of the alpha heads -- one online-softmax update per 32-row stage,
// release of the stage to the producer (mbarrier arrive), and at each group end one
// (m, l, o) partial per consumer with plain stores; tma_merge_kernel (next launch, PDL)
// merges each group's partials (O12).  The KV rows are loaded with an L2 evict_first
// policy (read once per step: the step's small hot data stays in L2).
#pragma once

constexpr int TM_RPS = 32;      // rows per stage
#ifndef SPC_TM_NST
#define SPC_TM_NST 2
#endif
#ifndef SPC_TM_CTAS
#define SPC_TM_CTAS 5
#endif
constexpr int TM_NST = SPC_TM_NST;    // ring depth
constexpr int TM_CTAS = SPC_TM_CTAS;  // CTAs per SM
#ifndef SPC_TM_NCONS
#define SPC_TM_NCONS 2
#endif
// consumer warps: consumer c takes the stages j = c mod TM_NCONS, with its own (m, l, o) state
// and partials.  Measured (config B step, tools/step_parts.py): 5 CTAs x 2 stages x 2
// consumers 77.5 us; 4 x 3 x 1 (round 2's first TMA kernel) 79.5; 4 x 3 x 3 80.5; 3 CTAs
// per SM 96 (the producers' gather rate per CTA is the limit); NOMATH 4 x 3 x 1 saves 3.6 us:
// a second consumer overlaps one stage's MMA / softmax latency with the next stage's
constexpr int TM_NCONS = SPC_TM_NCONS;
constexpr int TM_THREADS = 32 * (1 + TM_NCONS);  // warp 0 producer, warps 1.. consumers
// every ring slot must belong to ONE consumer (slot s = j mod TM_NST, consumer j mod
// TM_NCONS), or a consumer could wait on a slot's parity one phase ahead and alias it
static_assert(SPC_TM_NST % SPC_TM_NCONS == 0, "ring slots must map to one consumer each");
#ifndef SPC_TM_PF
#define SPC_TM_PF 4
#endif
constexpr int TM_PF = SPC_TM_PF;      // stages of token metadata loaded ahead by the producer
constexpr int TM_NREQ = TM_RPS / 4;   // producer lanes (4 rows per gather4)

template <int D>
struct TmSmem {
  static constexpr int NH = D / 64;            // 128-byte halves of a row (one TMA box each)
  static constexpr int HALF = TM_RPS * 128;    // one half of K (or V) of one stage
  static constexpr int STAGE = 2 * NH * HALF;  // K halves, then V halves
  static constexpr int BYTES = TM_NST * STAGE + 1024;  // + alignment slack (SW128 wants 1024)
};

__device__ __forceinline__ void tm_gather4(uint32_t dst, const CUtensorMap* map, uint32_t bar, int col,
                                           int r0, int r1, int r2, int r3) {
#ifndef SPC_TM_EVICT_NORMAL
  // the KV rows are read once per step: evict them first, so the step's small hot data (its
  // kernels' code, logits, selections) is not pushed out of L2 by the 256 MiB stream
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2], %8;" ::"r"(dst),
      "l"(map), "r"(bar), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "l"(pol)
      : "memory");
#else
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst),
      "l"(map), "r"(bar), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
      : "memory");
#endif
}
// Debug trace (-DSPC_TRACE builds, spc_debug_set_trace): per CTA c < 2048,
// g_trace[4096 + 4c + i] = %globaltimer at (0) entry after the PDL wait, (1) the consumer's
// first stage landed, (2) the consumer's last stage done (the CTA's end).
__device__ __forceinline__ void tm_trace(int i) {
#ifdef SPC_TRACE
  if (g_trace && blockIdx.x < 2048 && (threadIdx.x & 31) == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    g_trace[4096 + blockIdx.x * 4 + i] = t;
  }
#else
  (void)i;
#endif
}

template <int D, int ALPHA>
__global__ void __launch_bounds__(TM_THREADS, TM_CTAS) attn_tma_kernel(
    const uint16_t* __restrict__ q, const CUtensorMap* __restrict__ maps /* [2][L] */, int L,
    int kv_mode, const int32_t* __restrict__ idx, const int32_t* __restrict__ count, int layer_begin,
    int B, int G, int rows, int kbud, int kpad, float scale, int cpc, int n_groups, int segstride,
    float* __restrict__ part_o, float* __restrict__ part_ml) {
  using SM = TmSmem<D>;
  constexpr int NH = SM::NH, KS = D / 16;
  __shared__ __align__(8) uint64_t full[TM_NST], empty[TM_NST];
  extern __shared__ __align__(16) uint8_t tm_raw[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int BG = B * G, Hq = G * ALPHA;
  const int cpg = kpad / TM_RPS;  // stages per group
  const int c_begin = blockIdx.x * cpc;
  const int n_chunks = min(cpc, n_groups * cpg - c_begin);
  const uint32_t ring = (smem_u32(tm_raw) + 1023u) & ~1023u;
  const uint32_t full0 = smem_u32(&full[0]), empty0 = smem_u32(&empty[0]);
  if (tid == 0) {
    for (int s = 0; s < TM_NST; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(full0 + 8 * s));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(empty0 + 8 * s));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (n_chunks > 0 && warp == 0 && lane < 2) {  // the descriptors are inputs: warm them early
    const int l0 = layer_begin + (c_begin / cpg) / BG;
    prefetch_tmap(maps + lane * L + l0);
  }
  __syncthreads();
  // PDL: no global input is read before griddepcontrol.wait -- not even the LLM queries,
  // which no libspc launch writes: before the wait an SM may still serve lines cached by
  // earlier kernels (measured: reading the queries early returned a previous step's values
  // under graph replay, tests/test_gpu_pipeline.py config A)
  spc_pdl_entry();
  if (n_chunks <= 0) return;
  if (warp == 0) tm_trace(0);
  const int g0 = c_begin / cpg;
  const bool ind = kv_mode == SPC_KV_INDEXED;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    // metadata of chunk j: the tokens of rows 4*lane .. 4*lane + 3 and the group's count,
    // loaded TM_PF chunks ahead with no use of either until then (no stall at issue)
    int grp_m = g0, rc_m = c_begin - g0 * cpg;  // position of the next chunk to fetch
    struct Meta {
      int t[4];
      int nv, base, r0;
    };
    auto fetch = [&](int j, Meta& m) {
      const int grp = grp_m, rc = rc_m;
      if (++rc_m == cpg) {
        rc_m = 0;
        ++grp_m;
      }
      m.nv = 0;
      m.base = 0;
      m.r0 = rc * TM_RPS + 4 * lane;
      if (j >= n_chunks || lane >= TM_NREQ) return;
      const int bg = grp % BG;
      m.nv = __ldg(count + bg);
      m.base = bg * rows;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        m.t[u] = ind ? __ldg(idx + (size_t)bg * kbud + min(m.r0 + u, kbud - 1)) : m.r0 + u;
    };
    Meta pre[TM_PF];
#pragma unroll
    for (int u = 0; u < TM_PF; ++u) fetch(u, pre[u]);
    int grp = g0, rc = c_begin - g0 * cpg, s = 0;
    uint32_t ph = 0;
    const CUtensorMap* km = nullptr;
    const CUtensorMap* vm = nullptr;
    int cur_layer = -1;
    for (int jb = 0; jb < n_chunks; jb += TM_PF) {
#pragma unroll
      for (int u = 0; u < TM_PF; ++u) {
        const int j = jb + u;
        if (j >= n_chunks) break;
        int4 r;
        {
          Meta& m = pre[u];
          const int nv = min(m.nv, kbud);
#ifdef SPC_DEBUG  // selected rows must be cache rows; a bad one is zero-filled
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (m.r0 + u < nv) {
              SPC_DCHECK(m.t[u] >= 0 && m.t[u] < rows, SPC_E_RANGE);
              if (m.t[u] < 0 || m.t[u] >= rows) m.t[u] = -1 - m.base;
            }
#endif
          r.x = m.r0 + 0 < nv ? m.base + m.t[0] : -1;
          r.y = m.r0 + 1 < nv ? m.base + m.t[1] : -1;
          r.z = m.r0 + 2 < nv ? m.base + m.t[2] : -1;
          r.w = m.r0 + 3 < nv ? m.base + m.t[3] : -1;
        }
        fetch(j + TM_PF, pre[u]);
        const int layer = layer_begin + grp / BG;
        if (layer != cur_layer) {
          cur_layer = layer;
          km = maps + layer;
          vm = maps + L + layer;
        }
        if (j >= TM_NST) tm_wait(empty0 + 8 * s, ph ^ 1u);
        const uint32_t fb = full0 + 8 * s;
        const bool any = __any_sync(0xffffffffu, r.x >= 0);
        if (lane == 0) {
          if (any) tm_expect(fb, SM::STAGE);
          else tm_arrive(fb);  // nothing valid in this stage: complete the phase without bytes
        }
        __syncwarp();
        if (any && lane < TM_NREQ) {
          const uint32_t st = ring + (uint32_t)s * SM::STAGE + (uint32_t)lane * 512u;
#pragma unroll
          for (int h = 0; h < NH; ++h) {
            tm_gather4(st + h * SM::HALF, km, fb, 64 * h, r.x, r.y, r.z, r.w);
            tm_gather4(st + (NH + h) * SM::HALF, vm, fb, 64 * h, r.x, r.y, r.z, r.w);
          }
        }
        if (++rc == cpg) {
          rc = 0;
          ++grp;
        }
        if (++s == TM_NST) {
          s = 0;
          ph ^= 1u;
        }
      }
    }
  } else {
    // ------------------------------------------------------------ consumer
    const int gid = lane >> 2, tig = lane & 3;
    const int mi = lane >> 3, ri = lane & 7;
    // ldmatrix row offsets: K (A operand, rows ri + 8 (mi & 1)), V^T (trans, rows ri + 8 (mi >> 1))
    const uint32_t krow = (uint32_t)((ri + ((mi & 1) ? 8 : 0)) * 128);
    const uint32_t vrow = (uint32_t)((ri + ((mi & 2) ? 8 : 0)) * 128);
    uint32_t koff[KS], voff[KS];
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {
      const int ck = kk * 2 + (mi >> 1), cv = kk * 2 + (mi & 1);  // 16-byte granule of the row
      koff[kk] = (uint32_t)((ck >> 3) * SM::HALF) + krow + (uint32_t)((((ck & 7) ^ ri)) << 4);
      voff[kk] = (uint32_t)((NH + (cv >> 3)) * SM::HALF) + vrow + (uint32_t)((((cv & 7) ^ ri)) << 4);
    }
    uint32_t qa0[KS], qa2[KS];
    auto load_q = [&](int lr, int bg, uint32_t(&a0)[KS], uint32_t(&a2)[KS]) {
      const int b = bg / G, g = bg - (bg / G) * G;
      const uint16_t* qh =
          q + (((size_t)(layer_begin + lr) * B + b) * Hq + g * ALPHA + (gid < ALPHA ? gid : 0)) * D;
#pragma unroll
      for (int k = 0; k < KS; ++k) {
        const uint32_t x0 = __ldg((const unsigned int*)(qh + k * 16 + 2 * tig));
        const uint32_t x2 = __ldg((const unsigned int*)(qh + k * 16 + 8 + 2 * tig));
        a0[k] = gid < ALPHA ? x0 : 0u;
        a2[k] = gid < ALPHA ? x2 : 0u;
      }
    };
    int grp = g0, rc = c_begin - g0 * cpg;
    // q and count of the current group, and of the next one (loaded a group ahead)
    uint32_t qn0[KS], qn2[KS];
    load_q(grp / BG, grp % BG, qa0, qa2);
    const int g_last_c = (c_begin + n_chunks - 1) / cpg;
    if (grp + 1 <= g_last_c) load_q((grp + 1) / BG, (grp + 1) % BG, qn0, qn2);
    int cnt_g = __ldg(count + grp % BG);
    int cnt_n = 0;
    if (grp + 1 <= g_last_c) cnt_n = __ldg(count + (grp + 1) % BG);
    constexpr bool LOSEP = ALPHA == 8;
    constexpr int NACC = LOSEP ? 2 : 1;
    const int srcl = LOSEP ? lane : ((lane & ~3) | (ALPHA == 4 ? (tig & 1) : 0));
    int cmode[2], hd[2];
#pragma unroll
    for (int sl = 0; sl < 2; ++sl) {
      const int n = 2 * tig + sl;
      cmode[sl] = LOSEP ? 0 : (n < ALPHA ? 0 : (n < 2 * ALPHA ? 1 : 2));
      hd[sl] = LOSEP ? n : n % ALPHA;
    }
    const float sl2 = scale * LOG2E;
    float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};
    float o[NACC][D / 16][4];
#pragma unroll
    for (int a = 0; a < NACC; ++a)
#pragma unroll
      for (int i = 0; i < D / 16; ++i) o[a][i][0] = o[a][i][1] = o[a][i][2] = o[a][i][3] = 0.f;
    int s = 0;
    uint32_t ph = 0;
    const int cw = warp - 1;  // this consumer's stages: j = cw mod TM_NCONS (its own partials)
    for (int j = 0; j < n_chunks; ++j) {
      const bool grp_end = (j == n_chunks - 1) || (rc == cpg - 1);
      const bool mine = TM_NCONS == 1 || j % TM_NCONS == cw;
      const int nv = mine ? min(cnt_g, kbud) - rc * TM_RPS : 0;  // valid rows (<= 0 or > 32 too)
      if (mine) tm_wait(full0 + 8 * s, ph);
      if (j == 0) tm_trace(1);
      const uint32_t st = ring + (uint32_t)s * SM::STAGE;
#ifdef SPC_TM_NOMATH  // debug builds only: the load pipeline alone
      if (false) {
#else
      if (nv > 0) {
#endif
        // ---- S^T = K Q^T for the two 16-row tiles
        float c[2][2][4];
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
          for (int e = 0; e < 4; ++e) c[t][0][e] = c[t][1][e] = 0.f;
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            uint32_t a0, a1, a2, a3;
            ldsm_x4(st + t * 16 * 128 + koff[kk], a0, a1, a2, a3);
            mma_bf16_4(c[t][kk & 1], a0, a1, a2, a3, qa0[kk], qa2[kk]);
          }
        }
        float sv[2][4];
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const float raw[4] = {c[t][0][0] + c[t][1][0], c[t][0][1] + c[t][1][1], c[t][0][2] + c[t][1][2],
                                c[t][0][3] + c[t][1][3]};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int from = ALPHA == 1 ? (e & 2) : e;
            const float x = LOSEP ? raw[e] : __shfl_sync(0xffffffffu, raw[from], srcl);
            sv[t][e] = (16 * t + (e < 2 ? gid : gid + 8)) < nv ? x * sl2 : -INFINITY;
          }
        }
        float mx0 = fmaxf(fmaxf(sv[0][0], sv[0][2]), fmaxf(sv[1][0], sv[1][2]));
        float mx1 = fmaxf(fmaxf(sv[0][1], sv[0][3]), fmaxf(sv[1][1], sv[1][3]));
#pragma unroll
        for (int sh = 4; sh < 32; sh <<= 1) {
          mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, sh));
          mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, sh));
        }
        const float mn0 = fmaxf(m_run[0], mx0), mn1 = fmaxf(m_run[1], mx1);  // row 0 valid: finite
        if (__any_sync(0xffffffffu, mn0 > m_run[0] || mn1 > m_run[1])) {
          const float c0 = exp2f(m_run[0] - mn0), c1 = exp2f(m_run[1] - mn1);
          l_run[0] *= c0;
          l_run[1] *= c1;
#pragma unroll
          for (int a = 0; a < NACC; ++a)
#pragma unroll
            for (int d = 0; d < D / 16; ++d) {
              o[a][d][0] *= c0;
              o[a][d][1] *= c1;
              o[a][d][2] *= c0;
              o[a][d][3] *= c1;
            }
          m_run[0] = mn0;
          m_run[1] = mn1;
        }
        uint32_t pb[2][2], pl[2][2];
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          float ph4[4], pl4[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float pe = exp2f(sv[t][e] - m_run[e & 1]);
            l_run[e & 1] += pe;
            const float h = __bfloat162float(__float2bfloat16_rn(pe));
            const float lo = pe - h;
            const int md = cmode[e & 1];
            ph4[e] = LOSEP ? h : (md == 0 ? h : (md == 1 ? lo : 0.f));
            pl4[e] = lo;
          }
          pb[t][0] = movm_t(pack_bf16(ph4[0], ph4[1]));
          pb[t][1] = movm_t(pack_bf16(ph4[2], ph4[3]));
          pl[t][0] = pl[t][1] = 0u;
          if (LOSEP) {
            pl[t][0] = movm_t(pack_bf16(pl4[0], pl4[1]));
            pl[t][1] = movm_t(pack_bf16(pl4[2], pl4[3]));
          }
        }
        // ---- O^T += V^T P
#pragma unroll
        for (int mt = 0; mt < D / 16; ++mt) {
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            uint32_t a0, a1, a2, a3;
            ldsm_x4_t(st + t * 16 * 128 + voff[mt], a0, a1, a2, a3);
            mma_bf16_4(o[0][mt], a0, a1, a2, a3, pb[t][0], pb[t][1]);
            if (LOSEP) mma_bf16_4(o[NACC - 1][mt], a0, a1, a2, a3, pl[t][0], pl[t][1]);
          }
        }
      }
      __syncwarp();
      if (mine && lane == 0) tm_arrive(empty0 + 8 * s);  // the stage's smem is consumed
      if (++s == TM_NST) {
        s = 0;
        ph ^= 1u;
      }
      if (grp_end) {
        // ---- this CTA's (m, l, o) partial of the group, plain stores
        float lsum[2] = {l_run[0], l_run[1]};
#pragma unroll
        for (int sh = 4; sh < 32; sh <<= 1) {
          lsum[0] += __shfl_xor_sync(0xffffffffu, lsum[0], sh);
          lsum[1] += __shfl_xor_sync(0xffffffffu, lsum[1], sh);
        }
        const int lr = grp / BG, bg = grp % BG;
        const int b = bg / G, g = bg - (bg / G) * G;
        const int part = (blockIdx.x - (grp * cpg) / cpc) * TM_NCONS + cw;
        const size_t head_base = ((size_t)lr * B + b) * Hq + g * ALPHA;
        constexpr int PX = ALPHA == 4 ? 2 : 1;
#pragma unroll
        for (int d = 0; d < D / 16; ++d)
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            float v = o[0][d][r];
            if (LOSEP) v += o[NACC - 1][d][r];
            else if (ALPHA == 1) v = o[0][d][r & 2] + o[0][d][(r & 2) + 1];
            else v += __shfl_xor_sync(0xffffffffu, v, PX);
            const int sl = r & 1;
            if (cmode[sl] == 0 && (ALPHA != 1 || sl == 0))
              part_o[((head_base + hd[sl]) * segstride + part) * D + 16 * d + gid + (r >= 2 ? 8 : 0)] = v;
          }
        if (gid == 0) {
#pragma unroll
          for (int sl = 0; sl < 2; ++sl)
            if (cmode[sl] == 0 && (ALPHA != 1 || sl == 0)) {
              float* ml = part_ml + ((head_base + hd[sl]) * segstride + part) * 2;
              ml[0] = m_run[sl];
              ml[1] = lsum[sl];
            }
        }
        m_run[0] = m_run[1] = -INFINITY;
        l_run[0] = l_run[1] = 0.f;
#pragma unroll
        for (int a = 0; a < NACC; ++a)
#pragma unroll
          for (int d = 0; d < D / 16; ++d) o[a][d][0] = o[a][d][1] = o[a][d][2] = o[a][d][3] = 0.f;
        if (j + 1 < n_chunks) {
#pragma unroll
          for (int kq = 0; kq < KS; ++kq) {
            qa0[kq] = qn0[kq];
            qa2[kq] = qn2[kq];
          }
          cnt_g = cnt_n;
          if (grp + 2 <= g_last_c) {
            load_q((grp + 2) / BG, (grp + 2) % BG, qn0, qn2);
            cnt_n = __ldg(count + (grp + 2) % BG);
          }
        }
      }
      if (++rc == cpg) {
        rc = 0;
        ++grp;
      }
    }
  }
  if (warp == 1) tm_trace(2);
}

// LSE merge (O12) of the per-CTA partials of every group, launched right behind
// attn_tma_kernel (PDL: its CTAs wait at griddepcontrol.wait while the attention drains,
// so the merge costs one L2 round trip per 8 partials instead of a ticketed tail in the
// attention kernel -- measured: in-kernel tickets + merges, inline or after each CTA's loop,
// made the attention 3-10 us slower).  One warp per (group, head): every lane reads the
// (m, l) of up to 8 partials and its D/32 dims of each, all loads before any use.  The
// partials of group gq are segments (gq*cpg)/cpc .. (gq*cpg+cpg-1)/cpc.
template <int D, int ALPHA>
__global__ void __launch_bounds__(128) tma_merge_kernel(
    const float* __restrict__ part_o, const float* __restrict__ part_ml, int cpg, int cpc,
    int n_groups, int B, int G, int layer_begin, int segstride, float* __restrict__ out,
    float* __restrict__ lse) {
  spc_pdl_entry();
  constexpr int DPL = D / 32;  // dims per lane
  constexpr int PU = 8;        // partials per round: all loads of a round issued before any use
  const int wg = blockIdx.x * 4 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (wg >= n_groups * ALPHA) return;
  const int gq = wg / ALPHA, j = wg - gq * ALPHA;
  const int BG = B * G, Hq = G * ALPHA;
  const int lr = gq / BG, bg = gq - lr * BG, b = bg / G, g = bg - b * G;
  const int np = ((gq * cpg + cpg - 1) / cpc - (gq * cpg) / cpc + 1) * TM_NCONS;
  const size_t h = ((size_t)lr * B + b) * Hq + g * ALPHA + j;  // partial head index
  const size_t oh = ((size_t)(layer_begin + lr) * B + b) * Hq + g * ALPHA + j;
  const float* ml = part_ml + h * segstride * 2;
  const float* po = part_o + h * segstride * D + lane * DPL;
  // one L2 round trip per PU partials: every lane loads the (m, l) of all of them (broadcast
  // loads) and its own DPL dims of each, then merges (M = running maximum, rescaled sums)
  float M = -INFINITY, den = 0.f;
  float acc[DPL];
#pragma unroll
  for (int i = 0; i < DPL; ++i) acc[i] = 0.f;
  for (int p0 = 0; p0 < np; p0 += PU) {
    float2 m_l[PU];
    float v[PU][DPL];
#pragma unroll
    for (int u = 0; u < PU; ++u) {
      const int p = p0 + u;
      m_l[u] = p < np ? __ldcg(reinterpret_cast<const float2*>(ml) + p) : make_float2(-INFINITY, 0.f);
#pragma unroll
      for (int i = 0; i < DPL; i += (DPL % 4 == 0 ? 4 : 1)) {
        if (DPL % 4 == 0) {
          const float4 x = p < np ? __ldcg(reinterpret_cast<const float4*>(po + (size_t)p * D + i))
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
          v[u][i] = x.x;
          v[u][(i + 1) % DPL] = x.y;
          v[u][(i + 2) % DPL] = x.z;
          v[u][(i + 3) % DPL] = x.w;
        } else {
          v[u][i] = p < np ? __ldcg(po + (size_t)p * D + i) : 0.f;
        }
      }
    }
    float Mn = M;
#pragma unroll
    for (int u = 0; u < PU; ++u) Mn = fmaxf(Mn, m_l[u].x);
    if (Mn != -INFINITY) {
      const float c = M == -INFINITY ? 0.f : exp2f(M - Mn);
      den *= c;
#pragma unroll
      for (int i = 0; i < DPL; ++i) acc[i] *= c;
#pragma unroll
      for (int u = 0; u < PU; ++u) {
        const float w = m_l[u].x == -INFINITY ? 0.f : exp2f(m_l[u].x - Mn);
        den += w * m_l[u].y;
#pragma unroll
        for (int i = 0; i < DPL; ++i) acc[i] += w * v[u][i];
      }
      M = Mn;
    }
  }
  const float inv = den > 0.f ? 1.f / den : 0.f;
#pragma unroll
  for (int i = 0; i < DPL; ++i) out[oh * D + lane * DPL + i] = acc[i] * inv;
  if (lse && lane == 0) lse[oh] = den > 0.f ? (M + log2f(den)) * 0.6931471805599453f : -INFINITY;
}
