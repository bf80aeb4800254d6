// step.cu — spc_decode_step: one whole single-device decode step of the hot path in ONE
// C-ABI call (the native step executor): spc_score(LOGITS) -> spc_select (NORM, GROUP,
// top-k, INDEXED elastic diff) -> spc_sparse_decode_attn over every layer, enqueued on
// one stream with the library's PDL launches, so a C/C++ caller (or a CUDA-graph capture)
// runs the §8(a) path without per-kernel marshalling.  Falls back to spc_score(ALL) +
// spc_topk + spc_elastic_diff when spc_select does not apply (Smax > 135168, Smax % 4, or
// more (b, g) rows than one wave of 8-CTA clusters).  State (the previous selection) is
// the caller's: prev_idx / prev_count in, cur_idx / cur_count out (swap them per step).
#include "common.cuh"


using namespace spc;

extern "C" size_t spc_decode_step_workspace(int L, int B, int Hq, int G, int D, int Smax, int k) {
  if (L <= 0 || B <= 0 || Hq <= 0 || G <= 0 || Smax <= 0 || k <= 0) return 0;
  return align_up(spc_score_workspace(B, Hq, Smax), 256) +
         align_up(spc_topk_workspace(B, G, Smax, k), 256) +
         align_up(spc_attn_workspace(L, B, Hq, D, k), 256);
}

extern "C" int spc_decode_step(const spc_step_args* a, spc_stream_t stream) {
  if (!a) return SPC_E_NULL;
  const int L = a->L, B = a->B, Hq = a->Hq, G = a->G, D = a->D, Smax = a->Smax, k = a->k;
  // every argument of every call is checked here, before the first launch: an error never
  // leaves the selection state half-written
  if (!a->ws || !a->q_ret || !a->kr || !a->seq_len || !a->q_llm || !a->logits || !a->head_max ||
      !a->head_sumfix || !a->group_score || !a->prev_idx || !a->prev_count || !a->cur_idx ||
      !a->cur_count || !a->load_tok || !a->n_load || !a->out)
    return SPC_E_NULL;
  if (!a->kv_desc && (!a->k_layers || !a->v_layers)) return SPC_E_NULL;
  if (L <= 0 || B <= 0 || Hq <= 0 || G <= 0 || Hq % G || Smax <= 0 || a->rows <= 0)
    return SPC_E_SHAPE;
  if (k < 1 || k > SPC_MAX_K) return SPC_E_BUDGET;
  if (Smax >= SPC_MAX_SEQ) return SPC_E_RANGE;
  {
    const int alpha = Hq / G;
    if (!(D == 64 || D == 128) || !(alpha == 1 || alpha == 2 || alpha == 4 || alpha == 8))
      return SPC_E_UNSUPPORTED;
  }
  if (((uintptr_t)a->kr & 15) || ((uintptr_t)a->q_ret & 15)) return SPC_E_RANGE;
  if (a->kv_desc && ((uintptr_t)a->kv_desc % 64 || (uint64_t)B * G * a->rows >= (1ull << 31)))
    return SPC_E_RANGE;
  if (a->ws_bytes < spc_decode_step_workspace(L, B, Hq, G, D, Smax, k)) return SPC_E_WORKSPACE;
  uint8_t* ws = (uint8_t*)a->ws;
  const size_t s_b = align_up(spc_score_workspace(B, Hq, Smax), 256);
  const size_t t_b = align_up(spc_topk_workspace(B, G, Smax, k), 256);
  const size_t a_b = align_up(spc_attn_workspace(L, B, Hq, D, k), 256);
  const bool fused = Smax <= 135168 && Smax % 4 == 0 && (long long)B * G * 8 <= num_sms();
  if (fused) {
    SPC_TRY(spc_score(SPC_BF16, a->q_ret, a->kr, a->seq_len, B, Hq, G, D, Smax, a->scale,
                      SPC_SCORE_LOGITS, a->logits, a->head_max, a->head_sumfix, a->group_score, ws,
                      s_b, stream));
    SPC_TRY(spc_select(a->logits, a->head_max, a->seq_len, B, Hq, G, Smax, k, a->force_last,
                       a->head_sumfix, a->group_score, a->cur_idx, a->cur_count, a->prev_idx,
                       a->prev_count, a->load_tok, a->n_load, nullptr, nullptr, stream));
  } else {
    SPC_TRY(spc_score(SPC_BF16, a->q_ret, a->kr, a->seq_len, B, Hq, G, D, Smax, a->scale,
                      SPC_SCORE_ALL, a->logits, a->head_max, a->head_sumfix, a->group_score, ws,
                      s_b, stream));
    SPC_TRY(spc_topk(a->group_score, a->seq_len, B, G, Smax, k, a->force_last, 1, 0, a->cur_idx,
                     nullptr, a->cur_count, nullptr, ws + s_b, t_b, stream));
    SPC_TRY(spc_elastic_diff(a->prev_idx, a->prev_count, a->cur_idx, a->cur_count, B, G, k,
                             nullptr, a->load_tok, nullptr, a->n_load, nullptr, nullptr, stream));
  }
  if (a->kv_desc)
    return spc_sparse_decode_attn_kv(a->kv_desc, a->q_llm, SPC_KV_INDEXED, a->cur_idx, a->cur_count, L,
                                     0, L, B, Hq, G, D, a->rows, k, a->scale, a->out, a->lse,
                                     ws + s_b + t_b, a_b, stream);
  return spc_sparse_decode_attn(SPC_BF16, a->q_llm, a->k_layers, a->v_layers, SPC_KV_INDEXED,
                                a->cur_idx, a->cur_count, L, 0, L, B, Hq, G, D, a->rows, k,
                                a->scale, a->out, a->lse, ws + s_b + t_b, a_b, stream);
}
