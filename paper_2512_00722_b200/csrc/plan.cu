// plan.cu — adaptive memory management: the paper's memory model
// (Eq. 6-8) and its compile-time threshold list (Algorithm 1) and per-step offload rule
// (Algorithm 2), as host functions of the C ABI (no GPU work, R25-R27).
//
// Paper §6: "we develop a theoretical memory overhead model based on LLM
// architecture, hardware specifications and inference workload" -- runtime memory is 30%
// of the model, K and V at 2 bytes give the KV coefficient 4, and the
// retrieval head's single layer plus the repeat_kv buffer add 1 + alpha KV layers
// (P:439).  Eq. 7 charges offloaded layers a budget buffer of B rows on the GPU.
// Algorithm 1 precomputes S^T_i, the longest sequence that fits with the last i layers
// offloaded; Algorithm 2 offloads one more layer (from the last one down) whenever the
// sequence length reaches the next threshold.
//
// Readings: the B term of Algorithm 1 takes Eq. 7's coefficient (2 * bytes per element),
// SURVEY Z19 / SPEC "Open Questions"; the model term is trunc(runtime_factor * bytes).
// This framework never materialises repeat_kv (one key row serves all alpha heads), so
// its own deployments pass extra_layers = 1; the paper's setting is 1 + alpha.
#include <cstdint>
#include <limits>

#include "common.cuh"

namespace {

int64_t model_term(const spc_plan_cfg* c) {
  return (int64_t)(c->runtime_factor * (double)c->model_bytes);
}
int64_t coef(const spc_plan_cfg* c) {  // bytes per (token x layer) of KV cache: 2 * bpe * R * H * D
  return 2LL * c->bytes_per_elem * c->R * c->H * c->D;
}
bool valid(const spc_plan_cfg* c) {
  return c && c->L >= 1 && c->H >= 1 && c->D >= 1 && c->R >= 1 && c->B >= 0 &&
         c->extra_layers >= 0 && c->bytes_per_elem >= 1 && c->mem_gpu > 0 && c->model_bytes >= 0 &&
         c->runtime_factor >= 0.0;
}
int64_t floor_div(int64_t a, int64_t b) {  // b > 0
  int64_t q = a / b;
  if ((a % b != 0) && (a < 0)) --q;
  return q;
}

}  // namespace

extern "C" int64_t spc_plan_mem_part(const spc_plan_cfg* cfg, int64_t S, int l_gpu) {
  if (!valid(cfg) || S < 0 || l_gpu < 0 || l_gpu > cfg->L) return -1;
  return model_term(cfg) +
         coef(cfg) * ((int64_t)(l_gpu + cfg->extra_layers) * S + (int64_t)(cfg->L - l_gpu) * cfg->B);
}

extern "C" int spc_plan_thresholds(const spc_plan_cfg* cfg, int64_t* thresholds) {
  if (!cfg || !thresholds) return SPC_E_NULL;
  if (!valid(cfg)) return SPC_E_SHAPE;
  const int64_t C = cfg->mem_gpu - model_term(cfg), c = coef(cfg);
  if (C <= 0) return SPC_E_BUDGET;
  for (int i = 0; i <= cfg->L; ++i) {
    const int64_t layers = (int64_t)cfg->L + cfg->extra_layers - i;  // KV layers left on the GPU
    thresholds[i] = layers > 0 ? floor_div(C - c * i * cfg->B, c * layers)
                               : std::numeric_limits<int64_t>::max();
  }
  return SPC_OK;
}

extern "C" int spc_plan_max_resident(const spc_plan_cfg* cfg, int64_t S, int* l_gpu,
                                     int64_t* shortfall) {
  if (!cfg || !l_gpu) return SPC_E_NULL;
  if (!valid(cfg) || S < 0) return SPC_E_SHAPE;
  // M_part is affine in l_gpu with slope coef * (S - B): scan from the top (L + 1 values)
  for (int l = cfg->L; l >= 0; --l)
    if (spc_plan_mem_part(cfg, S, l) <= cfg->mem_gpu) {
      *l_gpu = l;
      if (shortfall) *shortfall = 0;
      return SPC_OK;
    }
  *l_gpu = -1;
  if (shortfall) *shortfall = spc_plan_mem_part(cfg, S, 0) - cfg->mem_gpu;
  return SPC_E_BUDGET;
}

extern "C" int spc_plan_step(const int64_t* thresholds, int L, int64_t S, int* l_cpu,
                             int32_t* offload_layers, int* n_offload) {
  if (!thresholds || !l_cpu || !n_offload) return SPC_E_NULL;
  if (L < 1 || *l_cpu < 0 || *l_cpu > L || S < 0) return SPC_E_SHAPE;
  int n = 0;
  while (*l_cpu < L && S >= thresholds[*l_cpu]) {  // Algorithm 2, inner while
    if (offload_layers) offload_layers[n] = L - *l_cpu - 1;
    ++n;
    ++*l_cpu;
  }
  *n_offload = n;
  return SPC_OK;
}
