/*
 * spcref.c — CPU ORACLE (test infrastructure only; see spcref.h).
 *
 * A plain, slow, obviously-correct C implementation of the hot path of
 * SpeContext (arXiv 2512.00722), written step by step in the paper's order:
 *   Eq.1 attention weights of the retrieval head
 *   -> GQA group max (MQA P:331)  -> top-k
 *   -> elastic-loading set difference
 *   -> attention of the LLM over the selected KV (Eq.1).
 * Where the paper leaves precision or order open, this file follows the
 * determinised contract O1..O13 written in DESIGN.md §3 (readings R1..R21).
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math (no FTZ/DAZ,
 * no contraction: every fmaf() below is an explicit fused multiply-add and
 * every other operation is one IEEE-754 round-to-nearest-even operation).
 *
 * PARITY PINS: see tests/test_oracle_*.py (closed forms, brute force,
 * the paper's worked examples, exhaustive exp sweep, fp64 faithfulness).
 */
#include "spcref.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------- small helpers (bit views) ---------- */
static float f_from_bits(uint32_t u) {
  float f;
  memcpy(&f, &u, 4);
  return f;
}
static uint32_t bits_from_f(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  return u;
}
/* bf16 -> f32 is exact: the bf16 pattern is the top half of the f32 pattern. */
static float bf16_to_f(uint16_t h) { return f_from_bits(((uint32_t)h) << 16); }

/* ---------- O3: exponential of the contract ----------
 * spc_exp(x), x <= 0:
 *   x < -87           -> 0
 *   n = rint(x*L2E)   (one RN multiply, then round-half-even to integer)
 *   r = fma(-n, LN2_HI, x); r = fma(-n, LN2_LO, r)        (Cody-Waite)
 *   p = c7; p = fma(p, r, c_i) for i = 6..0               (Horner, Taylor c_i = 1/i!)
 *   result = p * 2^n  (2^n built from exponent bits; n >= -126 so 2^n is normal)
 */
float spcref_exp(float x) {
  const float L2E = f_from_bits(0x3FB8AA3Bu);    /* log2(e) rounded to float */
  const float LN2_HI = f_from_bits(0x3F317200u); /* ln2 high part (exact n*LN2_HI) */
  const float LN2_LO = f_from_bits(0x35BFBE8Eu); /* ln2 - LN2_HI */
  const float c[8] = {f_from_bits(0x3F800000u), f_from_bits(0x3F800000u),
                      f_from_bits(0x3F000000u), f_from_bits(0x3E2AAAABu),
                      f_from_bits(0x3D2AAAABu), f_from_bits(0x3C088889u),
                      f_from_bits(0x3AB60B61u), f_from_bits(0x39500D01u)};
  if (x < -87.0f) return 0.0f;
  float t = x * L2E;
  float n = rintf(t);
  float r = fmaf(-n, LN2_HI, x);
  r = fmaf(-n, LN2_LO, r);
  float p = c[7];
  for (int i = 6; i >= 0; --i) p = fmaf(p, r, c[i]);
  int ni = (int)n;
  float two_n = f_from_bits((uint32_t)(ni + 127) << 23);
  return p * two_n;
}

/* O3 elementwise over an array (the exhaustive GPU bit-identity sweep). */
void spcref_exp_array(const float* x, float* y, long long n) {
  for (long long i = 0; i < n; ++i) y[i] = spcref_exp(x[i]);
}

double spcref_exp_max_ulp(uint32_t lo_bits, uint32_t hi_bits, uint64_t* n_subnormal) {
  double worst = 0.0;
  uint64_t sub = 0;
  for (uint64_t u = lo_bits; u <= hi_bits; ++u) {
    float x = f_from_bits((uint32_t)u);
    float y = spcref_exp(x);
    double ref = exp((double)x);
    if (!isfinite(y)) return INFINITY;
    if (y != 0.0f && fabsf(y) < FLT_MIN) ++sub;
    int e;
    frexp(ref, &e); /* ref = m * 2^e, m in [0.5, 1) -> ulp = 2^(e-24) for float */
    double ulp = ldexp(1.0, (e - 24) < -149 ? -149 : (e - 24));
    double err = fabs((double)y - ref) / ulp;
    if (err > worst) worst = err;
  }
  if (n_subnormal) *n_subnormal = sub;
  return worst;
}

/* ---------- O1 + O2: logits and per-head max (phase LOGITS) ----------
 * Eq.1 numerator Q K^T / sqrt(d) for the retrieval head:
 *   s[b][h][t] = fl( dot_seq(q[b][h], kr[b][g][t]) * scale ),
 *   dot_seq: acc = 0; for d = 0..D-1 ascending: acc = fma(q_d, k_d, acc).
 * Query head h reads KV group g = h / alpha (reading R4, HF repeat_kv).
 * Entries t >= seq_len[b] are left untouched. */
void spcref_logits(const uint16_t* q, const uint16_t* kr, const int32_t* seq_len, int B, int Hq,
                   int G, int D, int Smax, float scale, float* logits, float* head_max) {
  int alpha = Hq / G;
  for (int b = 0; b < B; ++b) {
    int S = seq_len[b];
    for (int h = 0; h < Hq; ++h) {
      int g = h / alpha;
      const uint16_t* qh = q + ((size_t)b * Hq + h) * D;
      float m = -INFINITY;
      for (int t = 0; t < S; ++t) {
        const uint16_t* kt = kr + (((size_t)b * G + g) * Smax + t) * D;
        float acc = 0.0f;
        for (int d = 0; d < D; ++d) acc = fmaf(bf16_to_f(qh[d]), bf16_to_f(kt[d]), acc);
        float s = acc * scale;
        logits[((size_t)b * Hq + h) * Smax + t] = s;
        if (s > m) m = s; /* O2: max is exact and order-free */
      }
      head_max[(size_t)b * Hq + h] = m;
    }
  }
}

/* ---------- O3 + O4: fixed-point softmax normaliser (phase NORM) ----------
 * Eq.1 denominator sum_t exp(s_t - m):  F = sum_t trunc(e_t * 2^40) as int64,
 * e_t = spc_exp(s_t - m) (one RN subtract, x <= 0).  Exact and order-free. */
void spcref_norm(const float* logits, const float* head_max, const int32_t* seq_len, int B, int Hq,
                 int Smax, int64_t* head_sumfix) {
  for (int b = 0; b < B; ++b) {
    int S = seq_len[b];
    for (int h = 0; h < Hq; ++h) {
      float m = head_max[(size_t)b * Hq + h];
      int64_t F = 0;
      for (int t = 0; t < S; ++t) {
        float e = spcref_exp(logits[((size_t)b * Hq + h) * Smax + t] - m);
        F += (int64_t)(e * 0x1p40f); /* scaling by 2^40 is exact; cast truncates */
      }
      head_sumfix[(size_t)b * Hq + h] = F;
    }
  }
}

/* ---------- O4..O6: weights and GQA group max (phase GROUP) ----------
 * l = fl((float)F) * 2^-40 ; r = 1/l (IEEE division) ; p = fl(e * r)   (Eq.1)
 * gs[b][g][t] = max_{j < alpha} p[b][g*alpha + j][t] */
void spcref_group(const float* logits, const float* head_max, const int64_t* head_sumfix,
                  const int32_t* seq_len, int B, int Hq, int G, int Smax, float* group_score) {
  int alpha = Hq / G;
  for (int b = 0; b < B; ++b) {
    int S = seq_len[b];
    for (int g = 0; g < G; ++g) {
      float* out = group_score + ((size_t)b * G + g) * Smax;
      for (int t = 0; t < Smax; ++t) out[t] = 0.0f;
      for (int j = 0; j < alpha; ++j) {
        int h = g * alpha + j;
        float m = head_max[(size_t)b * Hq + h];
        float l = (float)head_sumfix[(size_t)b * Hq + h] * 0x1p-40f;
        float r = 1.0f / l;
        for (int t = 0; t < S; ++t) {
          float e = spcref_exp(logits[((size_t)b * Hq + h) * Smax + t] - m);
          float p = e * r;
          if (j == 0 || p > out[t]) out[t] = p;
        }
      }
    }
  }
}

/* ---------- fp64 mathematical definition (faithfulness check) ---------- */
void spcref_group_score_f64(const uint16_t* q, const uint16_t* kr, const int32_t* seq_len, int B,
                            int Hq, int G, int D, int Smax, double scale, double* group_score) {
  int alpha = Hq / G;
  for (int b = 0; b < B; ++b) {
    int S = seq_len[b];
    double* s = (double*)malloc(sizeof(double) * (size_t)(S > 0 ? S : 1));
    for (int g = 0; g < G; ++g) {
      double* out = group_score + ((size_t)b * G + g) * Smax;
      for (int t = 0; t < Smax; ++t) out[t] = 0.0;
      for (int j = 0; j < alpha; ++j) {
        int h = g * alpha + j;
        const uint16_t* qh = q + ((size_t)b * Hq + h) * D;
        double m = -INFINITY;
        for (int t = 0; t < S; ++t) {
          const uint16_t* kt = kr + (((size_t)b * G + g) * Smax + t) * D;
          double acc = 0.0;
          for (int d = 0; d < D; ++d) acc += (double)bf16_to_f(qh[d]) * (double)bf16_to_f(kt[d]);
          s[t] = acc * scale;
          if (s[t] > m) m = s[t];
        }
        double l = 0.0;
        for (int t = 0; t < S; ++t) l += exp(s[t] - m);
        double lse = m + log(l);
        for (int t = 0; t < S; ++t) {
          double p = exp(s[t] - lse);
          if (j == 0 || p > out[t]) out[t] = p;
        }
      }
    }
    free(s);
  }
}

/* ---------- O7: top-k by (value desc, id asc), output ascending ---------- */
uint64_t spcref_composite(float value, int32_t id) {
  return ((uint64_t)bits_from_f(value) << 32) | (uint64_t)(uint32_t)(~(uint32_t)id);
}

typedef struct {
  float v;
  int32_t id;
  int32_t pos;
} cand_t;

static int cmp_rank(const void* a, const void* b) {
  const cand_t* x = (const cand_t*)a;
  const cand_t* y = (const cand_t*)b;
  if (x->v > y->v) return -1; /* value descending */
  if (x->v < y->v) return 1;
  if (x->id < y->id) return -1; /* ties: lower id first (reading R8) */
  if (x->id > y->id) return 1;
  return 0;
}
static int cmp_int(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

int spcref_topk_row(const float* val, const int32_t* cand_id, int n, int k, int force_pos,
                    int id_stride, int id_offset, int32_t* out_pos, float* out_val,
                    uint64_t* out_thresh) {
  cand_t* c = (cand_t*)malloc(sizeof(cand_t) * (size_t)(n > 0 ? n : 1));
  for (int p = 0; p < n; ++p) {
    c[p].v = (p == force_pos) ? INFINITY : val[p];
    c[p].id = cand_id ? cand_id[p] : p * id_stride + id_offset;
    c[p].pos = p;
  }
  qsort(c, (size_t)n, sizeof(cand_t), cmp_rank); /* full sort: the plain definition */
  int cnt = k < n ? k : n;
  if (out_thresh) *out_thresh = cnt > 0 ? spcref_composite(c[cnt - 1].v, c[cnt - 1].id) : 0;
  for (int i = 0; i < cnt; ++i) out_pos[i] = c[i].pos;
  qsort(out_pos, (size_t)cnt, sizeof(int32_t), cmp_int); /* emit ascending */
  if (out_val)
    for (int i = 0; i < cnt; ++i)
      out_val[i] = (out_pos[i] == force_pos) ? INFINITY : val[out_pos[i]];
  free(c);
  return cnt;
}

/* ---------- O8: elastic-loading set difference + slot assignment ----------
 * load S_now - S_last, evict S_last - S_now, update in place.
 * Slots (reading R13): kept rows never move; new token i (ascending) takes
 * the i-th freed slot in ascending slot order, freed = empty or not in cur. */
static int member(const int32_t* set, int n, int32_t x) {
  for (int i = 0; i < n; ++i)
    if (set[i] == x) return 1;
  return 0;
}

int spcref_elastic_diff_row(const int32_t* prev, int n_prev, const int32_t* cur, int n_cur, int k,
                            int32_t* slot_tok, int32_t* load_tok, int32_t* load_slot, int* n_load,
                            int32_t* evict_tok, int* n_evict) {
  int nl = 0, ne = 0;
  for (int i = 0; i < n_cur; ++i)
    if (!member(prev, n_prev, cur[i])) load_tok[nl++] = cur[i];
  for (int i = nl; i < k; ++i) load_tok[i] = -1;
  if (evict_tok) {
    for (int i = 0; i < n_prev; ++i)
      if (!member(cur, n_cur, prev[i])) evict_tok[ne++] = prev[i];
    for (int i = ne; i < k; ++i) evict_tok[i] = -1;
  } else {
    for (int i = 0; i < n_prev; ++i)
      if (!member(cur, n_cur, prev[i])) ++ne;
  }
  *n_load = nl;
  if (n_evict) *n_evict = ne;
  if (!slot_tok) return 0;
  /* state check: the non-empty slots hold exactly the previous set */
  int occupied = 0;
  for (int s = 0; s < k; ++s) {
    if (slot_tok[s] < 0) continue;
    ++occupied;
    if (!member(prev, n_prev, slot_tok[s])) return -1;
  }
  if (occupied != n_prev) return -1;
  int i = 0;
  for (int s = 0; s < k && i < nl; ++s) {
    if (slot_tok[s] < 0 || !member(cur, n_cur, slot_tok[s])) {
      slot_tok[s] = load_tok[i];
      load_slot[i] = s;
      ++i;
    }
  }
  if (i < nl) return -1;
  for (int j = nl; j < k; ++j) load_slot[j] = -1;
  /* evicted tokens that were not overwritten leave their slot empty */
  for (int s = 0; s < k; ++s)
    if (slot_tok[s] >= 0 && !member(cur, n_cur, slot_tok[s])) slot_tok[s] = -1;
  return 0;
}

/* ---------- O10: attention over selected rows, fp64 ----------
 * Eq.1: softmax(q K_J^T * scale) V_J, renormalised over J (reading R15). */
static double elem(const void* p, int is_bf16, size_t i) {
  return is_bf16 ? (double)bf16_to_f(((const uint16_t*)p)[i]) : (double)((const float*)p)[i];
}

double spcref_attn_head(const void* q, const void* k, const void* v, int is_bf16, const int32_t* rows,
                        int n, int D, double scale, double* out) {
  for (int d = 0; d < D; ++d) out[d] = 0.0;
  if (n <= 0) return -INFINITY;
  double* z = (double*)malloc(sizeof(double) * (size_t)n);
  double m = -INFINITY;
  for (int j = 0; j < n; ++j) {
    double acc = 0.0;
    for (int d = 0; d < D; ++d) acc += elem(q, is_bf16, (size_t)d) * elem(k, is_bf16, (size_t)rows[j] * D + d);
    z[j] = acc * scale;
    if (z[j] > m) m = z[j];
  }
  double l = 0.0;
  for (int j = 0; j < n; ++j) l += exp(z[j] - m);
  for (int j = 0; j < n; ++j) {
    double w = exp(z[j] - m) / l;
    for (int d = 0; d < D; ++d) out[d] += w * elem(v, is_bf16, (size_t)rows[j] * D + d);
  }
  free(z);
  return m + log(l);
}

/* ---------- O12: log-sum-exp merge of partial attentions ---------- */
double spcref_attn_merge_row(const double* o_parts, const double* lse_parts, int P, int D,
                             double* out) {
  double M = -INFINITY;
  for (int p = 0; p < P; ++p)
    if (lse_parts[p] > M) M = lse_parts[p];
  for (int d = 0; d < D; ++d) out[d] = 0.0;
  if (M == -INFINITY) return -INFINITY; /* every part empty */
  double den = 0.0;
  for (int p = 0; p < P; ++p) {
    if (lse_parts[p] == -INFINITY) continue; /* empty part contributes nothing */
    double w = exp(lse_parts[p] - M);
    den += w;
    for (int d = 0; d < D; ++d) out[d] += w * o_parts[(size_t)p * D + d];
  }
  for (int d = 0; d < D; ++d) out[d] /= den;
  return M + log(den);
}

/* =====================================================================
 * NEXT-1: the retrieval head's front-end.  Paper §4.3: the head keeps the
 * DLM's embedding module and QK projection weights and a full K cache, with YaRN
 * for long context; SPEC run_retrieval_head appends the new key at
 * position = cache length.  The normalisation follows the HF Llama RMSNorm the
 * EAGLE-3 DLM uses (reading R22); the rotation is rotate_half RoPE with the
 * caller's (YaRN-scaled) frequency table and attention scale (R23, R24).
 * ===================================================================== */
static uint16_t f_to_bf16_rn(float f) { /* IEEE RN-even of a finite float to bf16 */
  uint32_t u = bits_from_f(f);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

/* Reading R22: r = 1/sqrt(mean(x^2) + eps) with the sum of squares made
 * exact and order-free: e = ilogb(max|x|), F = sum_h trunc(x_h^2 * 2^(46-2e)) as int64
 * (each term exact in double and < 2^48), mean = fl64(fl64(F) * 2^(2e-46) / H),
 * r = fl32(fl64(1 / fl64(sqrt(mean + eps)))); then t = bf16(fl32(x r)), xn = bf16(fl32(w t)). */
void spcref_rmsnorm_bf16(const uint16_t* x, const uint16_t* w, int H, double eps, uint16_t* out) {
  float mx = 0.0f;
  for (int h = 0; h < H; ++h) {
    const float a = fabsf(bf16_to_f(x[h]));
    if (a > mx) mx = a;
  }
  const int e = mx > 0.0f ? ilogbf(mx) : 0;
  const double sc = mx > 0.0f ? ldexp(1.0, 46 - 2 * e) : 1.0;
  long long F = 0;
  for (int h = 0; h < H; ++h) {
    const double v = (double)bf16_to_f(x[h]);
    F += (long long)((v * v) * sc); /* C conversion truncates toward zero */
  }
  const double ss = mx > 0.0f ? ldexp((double)F, 2 * e - 46) : 0.0;
  const double mean = ss / (double)H;
  const float r = (float)(1.0 / sqrt(mean + (double)(float)eps));
  for (int h = 0; h < H; ++h) {
    const float t = bf16_to_f(f_to_bf16_rn(bf16_to_f(x[h]) * r));
    const float wv = w ? bf16_to_f(w[h]) : 1.0f;
    out[h] = f_to_bf16_rn(wv * t);
  }
}

void spcref_rethead_qk(const uint16_t* W, int N, int H, const uint16_t* xn, const float* inv_freq, int D,
                       int pos, double mscale, double* out, double* bound) {
  double* pre = (double*)malloc(sizeof(double) * (size_t)N);
  for (int n = 0; n < N; ++n) {
    double acc = 0.0, ab = 0.0;
    for (int h = 0; h < H; ++h) {
      const double t = (double)bf16_to_f(W[(size_t)n * H + h]) * (double)bf16_to_f(xn[h]);
      acc += t;
      ab += fabs(t);
    }
    pre[n] = acc;
    bound[n] = ab;
  }
  const int half = D / 2;
  for (int hd = 0; hd < N / D; ++hd)
    for (int i = 0; i < half; ++i) {
      const float a = (float)pos * inv_freq[i]; /* fl32 angle, as the kernel */
      const double c = cos((double)a) * mscale, s = sin((double)a) * mscale;
      const double u = pre[hd * D + i], v = pre[hd * D + i + half];
      out[hd * D + i] = u * c - v * s;
      out[hd * D + i + half] = v * c + u * s;
    }
  free(pre);
}

/* =====================================================================
 * NEXT-2: adaptive memory management, paper §6.  Eq. 6/7: the model
 * with 30% runtime memory plus the KV cache, coefficient 2 bytes x (K, V) = 4
 * at fp16, (L_GPU + 1 + alpha) resident layers (the retrieval head's layer and
 * the repeat_kv buffer; `extra_layers` = 1 + alpha) and a B-row buffer for each
 * offloaded layer.  Algorithm 1 is checked here by SEARCH over S, Eq. 8 by a linear scan.
 * ===================================================================== */
int64_t spcref_plan_mem(int64_t model_bytes, double runtime_factor, int L, int H, int D, int extra_layers,
                        int R, int64_t B, int bytes_per_elem, int64_t S, int l_gpu) {
  const int64_t m_model = (int64_t)(runtime_factor * (double)model_bytes);
  const int64_t per_tok_layer = (int64_t)2 * bytes_per_elem * R * H * D; /* K and V */
  const int64_t resident = (int64_t)(l_gpu + extra_layers) * S * per_tok_layer;
  const int64_t buffers = (int64_t)(L - l_gpu) * B * per_tok_layer;
  return m_model + resident + buffers;
}

void spcref_plan_thresholds_search(int64_t mem_gpu, int64_t model_bytes, double runtime_factor, int L, int H,
                                   int D, int extra_layers, int R, int64_t B, int bytes_per_elem,
                                   int64_t s_cap, int64_t* th) {
  const int64_t per_tok_layer = (int64_t)2 * bytes_per_elem * R * H * D;
  if (s_cap > mem_gpu / per_tok_layer + 1) s_cap = mem_gpu / per_tok_layer + 1; /* no overflow */
  for (int i = 0; i <= L; ++i) { /* i layers offloaded: l_gpu = L - i */
    int64_t lo = -1, hi = s_cap;     /* invariant: fits(lo) or lo = -1; largest fitting S in [lo, hi] */
    if (spcref_plan_mem(model_bytes, runtime_factor, L, H, D, extra_layers, R, B, bytes_per_elem, 0, L - i) >
        mem_gpu) {
      th[i] = -1;
      continue;
    }
    lo = 0;
    while (lo < hi) { /* monotone in S: binary search for the last S that fits */
      const int64_t mid = lo + (hi - lo + 1) / 2;
      if (spcref_plan_mem(model_bytes, runtime_factor, L, H, D, extra_layers, R, B, bytes_per_elem, mid,
                          L - i) <= mem_gpu)
        lo = mid;
      else
        hi = mid - 1;
    }
    th[i] = lo;
  }
}

int spcref_plan_max_resident(int64_t mem_gpu, int64_t model_bytes, double runtime_factor, int L, int H, int D,
                             int extra_layers, int R, int64_t B, int bytes_per_elem, int64_t S) {
  int best = -1;
  for (int l = 0; l <= L; ++l)
    if (spcref_plan_mem(model_bytes, runtime_factor, L, H, D, extra_layers, R, B, bytes_per_elem, S, l) <=
        mem_gpu)
      best = l;
  return best;
}

int spcref_plan_step(const int64_t* th, int L, int64_t S, int l_cpu, int32_t* out, int* n_out) {
  int n = 0;
  while (S >= th[l_cpu] && l_cpu < L) { /* Alg. 2 line 4, in the paper's order */
    out[n++] = L - l_cpu - 1;          /* line 5: offload Layer_{L - L_CPU - 1} */
    l_cpu = l_cpu + 1;                 /* line 6 */
  }
  *n_out = n;
  return l_cpu;
}

/* =====================================================================
 * NEXT-3: batch-level retrieval.  Paper §4.2 (Fig. 5(a)): "the batch-level
 * retrieval adopts a coarse-grained approach, retaining a single set of important tokens
 * that apply to all attention heads"; sum the weights over all heads per
 * position, then top-B.  The weights are O3-O5's; the sum runs over ascending h (O6b).
 * ===================================================================== */
void spcref_batch_score(const float* logits, const float* head_max, const int64_t* head_sumfix,
                        const int32_t* seq_len, int B, int Hq, int Smax, float* out) {
  for (int b = 0; b < B; ++b) {
    const int S = seq_len[b];
    for (int t = 0; t < Smax; ++t) {
      float acc = 0.0f;
      if (t < S)
        for (int h = 0; h < Hq; ++h) {
          const float m = head_max[(size_t)b * Hq + h];
          const float l = (float)head_sumfix[(size_t)b * Hq + h] * 0x1p-40f;
          const float r = 1.0f / l;
          const float p = spcref_exp(logits[((size_t)b * Hq + h) * Smax + t] - m) * r;
          acc = h == 0 ? p : acc + p;
        }
      out[(size_t)b * Smax + t] = acc;
    }
  }
}

/* =====================================================================
 * NEXT-3: MLA select-then-expand.  Paper §4.3: "MLA caches a lower-dimensional
 * latent representation c ... only the selected c cache is subjected to the increase in
 * dimension" (Fig. 5(e)); the retrieval stays head-level as for MHA.  Written in the paper's
 * order: expand the selected rows, then the attention of O10 over them (fp64).
 * ===================================================================== */
double spcref_mla_head(const uint16_t* q, const uint16_t* cache, const uint16_t* w_uk,
                       const uint16_t* w_uv, const int32_t* rows, int n, int DC, int DR, int DN,
                       int DV, double scale, double* out) {
  const int W = DC + DR;
  for (int d = 0; d < DV; ++d) out[d] = 0.0;
  if (n <= 0) return -INFINITY;
  double* z = (double*)malloc(sizeof(double) * (size_t)n);
  double* vexp = (double*)malloc(sizeof(double) * (size_t)n * DV);
  double m = -INFINITY;
  for (int j = 0; j < n; ++j) {
    const uint16_t* c = cache + (size_t)rows[j] * W;
    double acc = 0.0;
    for (int a = 0; a < DN; ++a) { /* K_j[a] = W_UK[a] . c_j (the expansion) */
      double kj = 0.0;
      for (int e = 0; e < DC; ++e) kj += (double)bf16_to_f(w_uk[(size_t)a * DC + e]) * (double)bf16_to_f(c[e]);
      acc += (double)bf16_to_f(q[a]) * kj;
    }
    for (int r = 0; r < DR; ++r) acc += (double)bf16_to_f(q[DN + r]) * (double)bf16_to_f(c[DC + r]);
    z[j] = acc * scale;
    if (z[j] > m) m = z[j];
    for (int a = 0; a < DV; ++a) { /* V_j[a] = W_UV[a] . c_j */
      double vj = 0.0;
      for (int e = 0; e < DC; ++e) vj += (double)bf16_to_f(w_uv[(size_t)a * DC + e]) * (double)bf16_to_f(c[e]);
      vexp[(size_t)j * DV + a] = vj;
    }
  }
  double l = 0.0;
  for (int j = 0; j < n; ++j) l += exp(z[j] - m);
  for (int j = 0; j < n; ++j) {
    const double w = exp(z[j] - m) / l;
    for (int a = 0; a < DV; ++a) out[a] += w * vexp[(size_t)j * DV + a];
  }
  free(z);
  free(vexp);
  return m + log(l);
}
