/*
 * spcref.h — CPU ORACLE for the SpeContext retrieval + sparse-attention hot
 * path.  TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * path (libspc, paper_2512_00722_b200) never links, imports or calls it.
 *
 * It shares no code, header, constant table or helper with the CUDA path:
 * every definition here is written from PAPER.md and the arithmetic contract
 * in DESIGN.md §3 (O1..O13).  Plain, slow, single-threaded C.
 *
 * bf16 values are passed as uint16_t bit patterns.
 */
#ifndef SPCREF_H_
#define SPCREF_H_
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* O3: the contract's exponential for x <= 0. */
float spcref_exp(float x);
void spcref_exp_array(const float* x, float* y, long long n);

/* Max |spcref_exp(x) - exp(x)| in ulps of the float result, over every float
 * x whose bit pattern lies in [lo_bits, hi_bits] (negative floats: sign bit
 * set; pass lo_bits <= hi_bits as unsigned ranges).  Also counts results that
 * are not finite or are subnormal.  Used by the pin tests (exhaustive sweep). */
double spcref_exp_max_ulp(uint32_t lo_bits, uint32_t hi_bits, uint64_t* n_subnormal);

/* O1 + O2 (phase LOGITS).  logits [B][Hq][Smax], head_max [B][Hq]. */
void spcref_logits(const uint16_t* q, const uint16_t* kr, const int32_t* seq_len, int B, int Hq,
                   int G, int D, int Smax, float scale, float* logits, float* head_max);
/* O3 + O4 (phase NORM).  head_sumfix [B][Hq]. */
void spcref_norm(const float* logits, const float* head_max, const int32_t* seq_len, int B, int Hq,
                 int Smax, int64_t* head_sumfix);
/* O3..O6 (phase GROUP).  group_score [B][G][Smax]; t >= seq_len[b] -> 0. */
void spcref_group(const float* logits, const float* head_max, const int64_t* head_sumfix,
                  const int32_t* seq_len, int B, int Hq, int G, int Smax, float* group_score);

/* The fp64 mathematical definition (Eq.1 + P:328) used to check that the
 * determinised contract is faithful: gs[b][g][t] = max_h exp(s_h(t) - LSE_h)
 * with s in fp64 and scale applied in fp64. */
void spcref_group_score_f64(const uint16_t* q, const uint16_t* kr, const int32_t* seq_len, int B,
                            int Hq, int G, int D, int Smax, double scale, double* group_score);

/* O7: top-k of one row by (value desc, id asc), ids = pos*id_stride +
 * id_offset (or cand_id[pos] when cand_id != NULL); force_pos >= 0 makes that
 * position +inf.  Writes min(k, n) selected POSITIONS ascending into out_pos,
 * their values into out_val (may be NULL); returns the count.  *out_thresh
 * (may be NULL) = composite key of the last selected element, 0 if none. */
int spcref_topk_row(const float* val, const int32_t* cand_id, int n, int k, int force_pos,
                    int id_stride, int id_offset, int32_t* out_pos, float* out_val,
                    uint64_t* out_thresh);

/* Composite key of O7's total order: larger = earlier. */
uint64_t spcref_composite(float value, int32_t id);

/* O8: elastic diff of one (b,g) row.  slot_tok may be NULL (INDEXED mode);
 * load_slot required iff slot_tok != NULL.  Returns 0, or -1 if the slot map
 * is inconsistent with prev (state error) or a new token has no free slot. */
int spcref_elastic_diff_row(const int32_t* prev, int n_prev, const int32_t* cur, int n_cur, int k,
                            int32_t* slot_tok, int32_t* load_tok, int32_t* load_slot, int* n_load,
                            int32_t* evict_tok, int* n_evict);

/* O10: attention of ONE query head over the rows listed in rows[0..n) of a
 * [n_rows_total][D] key/value block, everything in fp64.  is_bf16 selects the
 * element type of q/k/v (uint16 bf16 bits or float).  out [D]; returns lse
 * (natural log), -inf and out = 0 for n == 0. */
double spcref_attn_head(const void* q, const void* k, const void* v, int is_bf16, const int32_t* rows,
                        int n, int D, double scale, double* out);

/* O12: merge P partials (o [P][D], lse [P]) -> out [D]; returns lse. */
double spcref_attn_merge_row(const double* o_parts, const double* lse_parts, int P, int D,
                             double* out);

/* ---- NEXT-1: retrieval-head front-end (DESIGN R22-R24) ----
 * RMSNorm of one bf16 row, HF Llama reading: r = 1/sqrt(mean(x^2) + eps) (fp64), t = bf16(fl32(x*r)),
 * out = bf16(fl32(w*t)) (w = 1 when NULL). */
void spcref_rmsnorm_bf16(const uint16_t* x, const uint16_t* w, int H, double eps, uint16_t* out);
/* Projection + RoPE of one request in fp64: pre[n] = sum_h W[n][h]*xn[h], bound[n] = sum_h |W[n][h]*xn[h]|,
 * pairs (i, i+D/2) of each of the N/D heads rotated by a = fl32(pos*inv_freq[i]),
 * c = cos(a)*mscale, s = sin(a)*mscale: out[i] = pre[i]c - pre[i+D/2]s, out[i+D/2] = pre[i+D/2]c + pre[i]s. */
void spcref_rethead_qk(const uint16_t* W, int N, int H, const uint16_t* xn, const float* inv_freq, int D,
                       int pos, double mscale, double* out, double* bound);

/* ---- NEXT-2: adaptive memory management (Eq. 6-8, Alg. 1-2; SPEC memory-planner) ----
 * Eq. 7 term by term (Eq. 6: l_gpu = L); model term trunc(runtime_factor * model_bytes). */
int64_t spcref_plan_mem(int64_t model_bytes, double runtime_factor, int L, int H, int D, int extra_layers,
                        int R, int64_t B, int bytes_per_elem, int64_t S, int l_gpu);
/* Alg. 1 by SEARCH (not the closed form): th[i] = the largest S >= 0 with
 * M_part(S, L - i) <= mem_gpu, or -1 if none (S searched in [0, s_cap]). */
void spcref_plan_thresholds_search(int64_t mem_gpu, int64_t model_bytes, double runtime_factor, int L, int H,
                                   int D, int extra_layers, int R, int64_t B, int bytes_per_elem,
                                   int64_t s_cap, int64_t* th);
/* Eq. 8 by linear scan from l_gpu = 0 upward: the largest feasible l_gpu, -1 if none. */
int spcref_plan_max_resident(int64_t mem_gpu, int64_t model_bytes, double runtime_factor, int L, int H, int D,
                             int extra_layers, int R, int64_t B, int bytes_per_elem, int64_t S);
/* Alg. 2, lines 4-7, at sequence length S: returns the new L_CPU; offloaded layers in out. */
int spcref_plan_step(const int64_t* th, int L, int64_t S, int l_cpu, int32_t* out, int* n_out);

/* ---- NEXT-3: batch-level retrieval (Fig. 5(a); SPEC retrieve_batch_level S:125-132) ----
 * out[b][t] = sum over h = 0..Hq-1 (ascending, fp32 RN adds) of O5's weight p_h(t); 0 for t >= S (O6b). */
void spcref_batch_score(const float* logits, const float* head_max, const int64_t* head_sumfix,
                        const int32_t* seq_len, int B, int Hq, int Smax, float* out);

/* ---- NEXT-3: MLA select-then-expand (Fig. 5(e)) ----
 * One head of one request, fp64, in the paper's order: only the selected latent rows are
 * up-projected -- K_j = [W_UK c_j | kpe_j] (DN + DR), V_j = W_UV c_j (DV) -- then softmax
 * attention of q = [q_nope | q_pe] over them (scale given), o = sum_j w_j V_j.
 * cache [rows][DC + DR] bf16 (latent c then the shared rope key), W_UK [DN][DC], W_UV [DV][DC]
 * bf16, q [DN + DR] bf16.  Returns lse (natural log); -inf and o = 0 when n = 0. */
double spcref_mla_head(const uint16_t* q, const uint16_t* cache, const uint16_t* w_uk,
                       const uint16_t* w_uv, const int32_t* rows, int n, int DC, int DR, int DN,
                       int DV, double scale, double* out);

#ifdef __cplusplus
}
#endif
#endif
