/*
 * spc.h — C ABI of libspc: the per-decode-step retrieval + sparse-attention
 * hot path of SpeContext (arXiv 2512.00722), hand-written for sm_100a (B200).
 *
 * Citation keys: P:n = PAPER.md line n (the paper's LaTeX source);
 * "O<n>" = the arithmetic contract in DESIGN.md §3 (the written, bit-level
 * definition that both this library and the independent CPU oracle follow).
 *
 * Conventions (apply to every call below)
 * ---------------------------------------
 *  - extern "C", stateless, reentrant.  Every compute call only ENQUEUES work on
 *    `stream` (a cudaStream_t passed as void*; NULL = legacy default stream).
 *    No call synchronises the host, allocates memory or keeps state between
 *    calls.  The caller owns the rolling state (previous selection, slot map).
 *  - All tensors are caller-owned, dense, row-major with the innermost
 *    dimension last, and must stay valid until the enqueued work completes.
 *    Pointers are DEVICE pointers unless stated; a KV source for
 *    spc_gather_kv / spc_sparse_decode_attn may also be mapped pinned host
 *    memory (cudaHostAlloc(..., cudaHostAllocMapped) or cudaHostRegister with
 *    the device alias), read zero-copy over PCIe.
 *  - bf16 tensors are passed as raw 16-bit words (IEEE bfloat16 bit pattern).
 *  - Errors: host-checkable argument errors are reported as a spc_status
 *    BEFORE anything is enqueued (nothing aborts, nothing throws across the
 *    ABI).  Data-dependent contract violations (index out of range -> SPC_E_RANGE
 *    (S:178), unsorted / duplicated index list or slot map inconsistent with the
 *    previous set -> SPC_E_STATE, more new rows than free slots ->
 *    SPC_E_BUDGET, NaN keys or scores -> SPC_E_RANGE (reading R20)) are
 *    checked on the device only by a library built with SPC_DEBUG (libspc_debug.so,
 *    spc_debug_build() == 1): the first violation is recorded with its source line
 *    and returned by spc_check_device_errors(); in release builds they are
 *    undefined behaviour.  SPC_E_CUDA means a CUDA error; its text (and a device
 *    violation's location) is available from spc_last_cuda_error().
 *  - Index lists are int32, ascending, padded with -1 after `count` entries.
 */
#ifndef SPC_H_
#define SPC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* spc_stream_t; /* a cudaStream_t */

typedef enum { SPC_BF16 = 0, SPC_F32 = 1 } spc_dtype;

typedef enum {
  SPC_OK = 0,
  SPC_E_NULL = 1,        /* a required pointer is NULL                              */
  SPC_E_SHAPE = 2,       /* Hq % G != 0, D not in {64,128}, k < 1, sizes <= 0 ...  */
  SPC_E_BUDGET = 3,      /* k larger than the supported maximum (SPC_MAX_K)          */
  SPC_E_RANGE = 4,       /* a host-checkable index/range argument is out of range    */
  SPC_E_STATE = 5,       /* reserved: slot map inconsistent with previous set        */
  SPC_E_WORKSPACE = 6,   /* ws NULL or ws_bytes smaller than the *_workspace() value */
  SPC_E_UNSUPPORTED = 7, /* dtype / alpha / head-dim combination not compiled in     */
  SPC_E_CUDA = 8         /* CUDA launch error, see spc_last_cuda_error()             */
} spc_status;

enum { SPC_MAX_K = 4096 };      /* largest supported budget k                       */
enum { SPC_MAX_SEQ = 1 << 23 }; /* O4's fixed-point sum is exact for S < 2^23       */

const char* spc_status_string(int status);
const char* spc_last_cuda_error(void);
int spc_version(void);
/* 1 when this library was built with SPC_DEBUG (device-side contract checks), else 0. */
int spc_debug_build(void);
/* Synchronises `stream`; returns SPC_E_CUDA on a CUDA error, else the first device-side
 * contract violation recorded since the last call (SPC_DEBUG builds; cleared by the call;
 * location via spc_last_cuda_error()), else SPC_OK.  Not capturable in a CUDA graph. */
int spc_check_device_errors(spc_stream_t stream);
/* Number of kernels this library has launched since it was loaded (all
 * threads).  Used by bench.py to report how many of its own kernels ran. */
uint64_t spc_launch_count(void);

/* ------------------------------------------------------------------------
 * spc_score — retrieval-head scoring, O1..O6.
 *
 * Paper: Eq.1 attn_weight = softmax(Q K^T / sqrt(d)) of the
 * retrieval head over every cached retrieval key ("matrix
 * multiplication of Query ... with Keys_candidate to get the importance
 * scores"; "maintains a full Key (K) cache and calculates attention
 * weights"); GQA mapping P:328: "element-wise maximum ... within the same
 * group of heads ... to generate the group-level attention weights"
 * (MQA P:331 = one group; MHA = alpha 1).
 *
 * Query head h belongs to KV group g = h / alpha, alpha = Hq / G (DESIGN.md
 * reading R4).  For request b only tokens t < seq_len[b] exist.
 *
 * Phases (bit flags, so a context-sharded caller can all-reduce between them):
 *   SPC_SCORE_LOGITS: logits[b][h][t] = fl(dot_seq(q[b][h], kr[b][g][t]) * scale)
 *                     (O1: fp32 fma chain over d ascending, then one RN mul);
 *                     head_max[b][h] = max_t logits (O2).          (overwrites)
 *   SPC_SCORE_NORM:   head_sumfix[b][h] = sum_t trunc(spc_exp(s - m) * 2^40)
 *                     as exact int64 (O3, O4); m = head_max (input). (overwrites)
 *   SPC_SCORE_GROUP:  group_score[b][g][t] = max_{j<alpha} fl(spc_exp(s - m) * r)
 *                     with r = 1 / fl((float)F * 2^-40) (O4..O6).  Entries
 *                     t >= seq_len[b] are written as 0.
 *
 * q           [B][Hq][D]     bf16      retrieval-head query of this step
 * kr          [B][G][Smax][D] bf16     retrieval-head key cache
 * seq_len     [B]            int32, DEVICE; 1 <= seq_len[b] <= Smax
 * logits      [B][Hq][Smax]  f32       out (LOGITS) / in (NORM, GROUP)
 * head_max    [B][Hq]        f32       out (LOGITS) / in (NORM, GROUP)
 * head_sumfix [B][Hq]        int64     out (NORM)   / in (GROUP)
 * group_score [B][G][Smax]   f32       out (GROUP); may be NULL otherwise
 * ws          >= spc_score_workspace(B, Hq, Smax) bytes of device scratch, zero-filled
 *             once before first use (LOGITS' tile-claim counter and NORM's tickets
 *             start at 0; every launch leaves them 0); not shared by calls executing at
 *             the same time.  A launch that failed mid-way leaves it undefined: zero it again.
 *   SPC_SCORE_BATCH (with GROUP): batch-level retrieval
 *                     (Fig. 5(a)): one token set per
 *                     request from the sum over ALL query heads of their weights,
 *                     bs[b][t] = fl(...fl(p_0 + p_1) ... + p_{Hq-1}) (O5's p_h,
 *                     ascending h, RN adds; O6b), written to every g of
 *                     group_score[b][g][:] (so per-group top-k / diff / attention
 *                     all select the same set).  Hq <= 128.
 * Supported: dtype SPC_BF16; D in {64, 128}; alpha in {1, 2, 4, 8};
 * Smax < SPC_MAX_SEQ.
 * ---------------------------------------------------------------------- */
enum { SPC_SCORE_LOGITS = 1, SPC_SCORE_NORM = 2, SPC_SCORE_GROUP = 4, SPC_SCORE_ALL = 7,
       SPC_SCORE_BATCH = 16 /* with GROUP: batch-level retrieval, see below */ };
size_t spc_score_workspace(int B, int Hq, int Smax);
int spc_score(int dtype, const void* q, const void* kr, const int32_t* seq_len, int B, int Hq, int G,
              int D, int Smax, float scale, int phases, float* logits, float* head_max,
              int64_t* head_sumfix, float* group_score, void* ws, size_t ws_bytes,
              spc_stream_t stream);

/* ------------------------------------------------------------------------
 * spc_topk — per-(b,g) top-k selection, O7.
 *
 * Paper: "select the Top-K candidates"; head-level (per KV group)
 * retrieval; budget k = 2048.  The selection is the
 * first n = min(k, len) positions under the total order
 *     (value descending, global id ascending)         (reading R8)
 * emitted ASCENDING by position, -1 padded; len = min(seq_len[b], n_cols).
 * The global id of position p is p*id_stride + id_offset (single device:
 * stride 1, offset 0; context shard r of P: stride P, offset r).  Because
 * that map is increasing, ties among one shard's positions break by position.
 * force_last != 0 treats position len-1 as +inf (R10: the newest token is
 * always selected); its out_val is +inf.
 *
 * val        [B][G][n_cols] f32 >= 0 (a group_score)
 * seq_len    [B] int32 DEVICE
 * out_idx    [B][G][k] int32 out: selected positions, ascending, -1 padded
 * out_val    [B][G][k] f32 out or NULL: value at each selected position
 * out_count  [B][G] int32 out: min(k, len)
 * out_thresh [B][G] uint64 out or NULL: composite key of the LAST selected
 *            element in the total order, (bits(value) << 32) | ~uint32(id),
 *            when len > k (a real cut); 0 when every valid element is kept.
 *            The selection is exactly {positions whose composite >= thresh}.
 * ws         >= spc_topk_workspace(B, G, n_cols, k) bytes
 * Supported: 1 <= k <= SPC_MAX_K, n_cols < SPC_MAX_SEQ.
 * ---------------------------------------------------------------------- */
size_t spc_topk_workspace(int B, int G, int n_cols, int k);
int spc_topk(const float* val, const int32_t* seq_len, int B, int G, int n_cols, int k, int force_last,
             int id_stride, int id_offset, int32_t* out_idx, float* out_val, int32_t* out_count,
             uint64_t* out_thresh, void* ws, size_t ws_bytes, spc_stream_t stream);

/* spc_topk_merge — global threshold from P shards' local top-k lists (O13).
 * cand_val/cand_pos [P][R][k], cand_count [P][R] (R = B*G rows) as produced by
 * spc_topk on shard p with id_stride P, id_offset p; global id = pos*P + p.
 * out_thresh [R]: composite key of the k-th element of the union in the O7
 * order (0 if the union has fewer than k elements: everything is kept).
 * ws >= spc_topk_merge_workspace(P, R, k). */
size_t spc_topk_merge_workspace(int P, int R, int k);
int spc_topk_merge(const float* cand_val, const int32_t* cand_pos, const int32_t* cand_count, int P,
                   int R, int k, uint64_t* out_thresh, void* ws, size_t ws_bytes,
                   spc_stream_t stream);

/* spc_topk_filter — keep, in place and in order, the entries of an ascending
 * list whose composite key (bits(val) << 32 | ~uint32(pos*id_stride+id_offset))
 * is >= thresh[r]; pads with -1 and rewrites count.  idx/val [R][k],
 * count [R], thresh [R]. */
int spc_topk_filter(int32_t* idx, const float* val, int32_t* count, const uint64_t* thresh, int R,
                    int k, int id_stride, int id_offset, spc_stream_t stream);

/* ------------------------------------------------------------------------
 * spc_score_select — the whole single-device selection of a decode step in ONE
 * persistent launch: spc_score(LOGITS) + spc_select, bit-identical to them (O1..O8:
 * Eq.1, group max P:328, top-k P:267, S_now - S_last P:374).  Each SM keeps the
 * logits of its own key tiles in shared memory; the phases meet at grid-wide barriers
 * (the launch is cooperative: all CTAs co-resident).
 * q [B][Hq][D] bf16, kr [B][G][Smax][D] bf16 (16-byte aligned); logits [B][Hq][Smax]
 * f32 is written when non-NULL (tokens >= seq_len untouched); head_max [B][Hq],
 * head_sumfix [B][Hq], group_score [B][G][Smax] (0 past seq_len), out_idx / out_count,
 * load_tok / n_load, evict_tok / n_evict (may be NULL) as spc_select; prev_idx rows
 * ascending.  ws >= spc_score_select_workspace(B, Hq, G, Smax) bytes, zero-filled once
 * (the kernel leaves it zero-filled); not shared by calls executing at the same time.
 * Supported when spc_score_select_supported() returns 1: D in {64,128}, alpha in
 * {1,2,4,8}, 1 <= k <= SPC_MAX_K, and B*G*ceil(Smax/128) key tiles spread over the SMs
 * at <= 16 tiles per SM (config B: 2048 tiles, 14 per SM) -- SPC_E_UNSUPPORTED
 * otherwise (use spc_score + spc_select or the separate calls).
 * Errors: SPC_E_NULL, SPC_E_SHAPE, SPC_E_BUDGET, SPC_E_RANGE (alignment),
 * SPC_E_WORKSPACE, SPC_E_UNSUPPORTED, SPC_E_CUDA.
 * ---------------------------------------------------------------------- */
int spc_score_select_supported(int B, int Hq, int G, int D, int Smax, int k);
size_t spc_score_select_workspace(int B, int Hq, int G, int Smax);
int spc_score_select(const void* q, const void* kr, const int32_t* seq_len, int B, int Hq, int G,
                     int D, int Smax, float scale, int k, int force_last, float* logits,
                     float* head_max, int64_t* head_sumfix, float* group_score, int32_t* out_idx,
                     int32_t* out_count, const int32_t* prev_idx, const int32_t* prev_count,
                     int32_t* load_tok, int32_t* n_load, int32_t* evict_tok, int32_t* n_evict,
                     void* ws, size_t ws_bytes, spc_stream_t stream);

/* ------------------------------------------------------------------------
 * spc_select — the single-device step from the logits to the elastic diff in ONE
 * launch: spc_score(NORM | GROUP) + spc_topk(id_stride 1, id_offset 0) +
 * spc_elastic_diff(INDEXED mode, slot_tok = NULL), bit-identical to those
 * calls in sequence (same definitions O3..O8, same outputs, out_val and
 * out_thresh not produced).  One thread-block cluster per (b, g) row.
 * logits/head_max come from spc_score(LOGITS).  prev_idx/prev_count is the
 * previous step's selection (count 0 on the first step).
 * Supported: alpha in {1,2,4,8}, 1 <= k <= SPC_MAX_K, Smax <= 135168 and a
 * multiple of 4 (SPC_E_UNSUPPORTED otherwise: use the separate calls).
 * prev_idx rows must be ascending (as spc_topk / spc_select write them).
 * evict_tok / n_evict may be NULL.  Errors: SPC_E_NULL, SPC_E_SHAPE,
 * SPC_E_BUDGET, SPC_E_UNSUPPORTED, SPC_E_CUDA (launch failure).
 * ---------------------------------------------------------------------- */
int spc_select(const float* logits, const float* head_max, const int32_t* seq_len, int B, int Hq,
               int G, int Smax, int k, int force_last, int64_t* head_sumfix, float* group_score,
               int32_t* out_idx, int32_t* out_count, const int32_t* prev_idx,
               const int32_t* prev_count, int32_t* load_tok, int32_t* n_load, int32_t* evict_tok,
               int32_t* n_evict, spc_stream_t stream);

/* ------------------------------------------------------------------------
 * spc_elastic_diff — elastic loading set difference, O8.
 *
 * Paper §5.4: evict S_last - S_now, load S_now - S_last
 * ("S_pre" read as S_last, reading R12), fixed budget, in-place update of
 * the GPU-resident KV through Tensor.copy_().
 *
 * prev_idx/cur_idx [B][G][k] ascending lists with counts prev_count/cur_count
 * [B][G] (prev_count may be 0: first step).
 *   load_tok  [B][G][k] out: cur \ prev, ascending, -1 padded; n_load [B][G].
 *   evict_tok [B][G][k] out or NULL: prev \ cur, ascending; n_evict or NULL.
 * Slot bookkeeping (SLOTS mode; slot_tok != NULL), reading R13:
 *   slot_tok [B][G][k] in/out: token resident in each slot, -1 = empty.
 *   Freed slots = slots whose token is -1 or not in cur, ascending by slot;
 *   new token i (ascending) goes to freed slot i: load_slot[i] = freed[i],
 *   slot_tok[freed[i]] = load_tok[i].  Kept slots never move.  The caller
 *   guarantees the non-empty slot tokens equal prev (then #new <= #freed).
 *   load_slot [B][G][k] out (required iff slot_tok != NULL).
 * ---------------------------------------------------------------------- */
int spc_elastic_diff(const int32_t* prev_idx, const int32_t* prev_count, const int32_t* cur_idx,
                     const int32_t* cur_count, int B, int G, int k, int32_t* slot_tok,
                     int32_t* load_tok, int32_t* load_slot, int32_t* n_load, int32_t* evict_tok,
                     int32_t* n_evict, spc_stream_t stream);

/* ------------------------------------------------------------------------
 * spc_gather_kv — elastic load of newly selected KV rows into budget slots, O9.
 *
 * Paper: P:374 in-place copy_ of the rows S_now - S_last; P:350 prefetch on
 * separate CUDA streams; source may be CPU DRAM.
 * For every layer l in [layer_begin, layer_end), every (b,g), i < n_load[b][g]:
 *   k_buf[l][b][g][load_slot[i]][:] = k_src[l][b][g][load_tok[i]][:]   (same for v)
 * k_src/v_src: DEVICE arrays of L pointers, one per layer, each to
 *   [B][G][Smax][D] (device memory or mapped pinned host memory).
 * k_buf/v_buf: DEVICE arrays of L pointers, each to [B][G][k][D] (device).
 * ---------------------------------------------------------------------- */
int spc_gather_kv(int dtype, const void* const* k_src, const void* const* v_src, int L, int B, int G,
                  int D, int Smax, int k, int layer_begin, int layer_end, const int32_t* load_tok,
                  const int32_t* load_slot, const int32_t* n_load, void* const* k_buf,
                  void* const* v_buf, spc_stream_t stream);

/* ------------------------------------------------------------------------
 * spc_gather_kv_strided — spc_gather_kv (O9, same copy) for sources laid out
 * with explicit strides, in particular TOKEN-MAJOR offloaded KV where one
 * token's K and V rows of every layer form one contiguous record
 * ([B][G][Smax][L][2][D]: k_src[l] = base + l*2*D, v_src[l] = k_src[l] + D,
 * row_stride = L*2*D, bg_stride = Smax*L*2*D).  Paper: P:374 elastic copy_,
 * P:180/P:197 KV in CPU DRAM, P:363-365 (loading I/O dominates): a selected
 * token is then one contiguous PCIe read (config D).
 * K row of token t of (b,g) in layer l (bf16 elements):
 *   k_src[l] + (b*G+g)*bg_stride + t*row_stride        (same for v_src)
 * For every l in [layer_begin, layer_end), (b,g), i < n_load[b][g]:
 *   k_buf[l][b][g][load_slot[i]][:] = K row of token load_tok[i]  (same for V)
 * k_src/v_src/k_buf/v_buf: DEVICE arrays of L pointers (sources may be mapped
 * pinned host memory); row_stride >= D; strides in elements, 16-byte aligned.
 * Supported: SPC_BF16, D in {64, 128}.  Errors: SPC_E_NULL, SPC_E_SHAPE,
 * SPC_E_BUDGET, SPC_E_RANGE, SPC_E_UNSUPPORTED, SPC_E_CUDA.
 * ---------------------------------------------------------------------- */
int spc_gather_kv_strided(int dtype, const void* const* k_src, const void* const* v_src,
                          long long row_stride, long long bg_stride, int L, int B, int G, int D,
                          int k, int layer_begin, int layer_end, const int32_t* load_tok,
                          const int32_t* load_slot, const int32_t* n_load, void* const* k_buf,
                          void* const* v_buf, spc_stream_t stream);

/* ------------------------------------------------------------------------
 * spc_sparse_decode_attn — GQA decode attention over the selected rows, O10.
 *
 * Paper: Eq.1 softmax(QK^T/sqrt(d)) V restricted to the selected tokens,
 * mapped to the LLM's KV heads (P:324 torch.gather, P:328 GQA group sets);
 * renormalised over the subset (reading R15).
 * For every layer l in [layer_begin, layer_end), request b, query head h
 * (group g = h / alpha):
 *   J = the selected rows of (b, g);  z_j = scale * <q[l][b][h], K_j>
 *   out[l][b][h][:] = sum_j softmax(z)_j V_j ;  lse[l][b][h] = log sum_j e^{z_j}
 * kv_mode SPC_KV_INDEXED: k_layers/v_layers[l] -> [B][G][rows][D] full cache,
 *   J = idx[b][g][0 .. count[b][g]) (positions < rows).
 * kv_mode SPC_KV_SLOTS:   k_layers/v_layers[l] -> [B][G][rows][D] budget
 *   buffers (rows = k), J = slots 0 .. count[b][g]) ; idx ignored (may be NULL).
 * k_layers/v_layers: DEVICE arrays of L pointers (device or mapped host).
 * q [L][B][Hq][D] (dtype), out [L][B][Hq][D] f32, lse [L][B][Hq] f32 or NULL.
 * A (b,g) with count 0 yields out = 0, lse = -inf.
 * ws >= spc_attn_workspace(L, B, Hq, D, k) bytes, zero-filled once before first use (the
 * per-group merge tickets start at 0; every launch leaves them 0); not shared by calls
 * executing at the same time.  A launch that failed mid-way leaves it undefined.
 * Supported: dtype SPC_BF16 or SPC_F32; D in {64, 128}; alpha in {1,2,4,8}.
 * ---------------------------------------------------------------------- */
enum { SPC_KV_INDEXED = 0, SPC_KV_SLOTS = 1 };
size_t spc_attn_workspace(int L, int B, int Hq, int D, int k);
int spc_sparse_decode_attn(int dtype, const void* q, const void* const* k_layers,
                           const void* const* v_layers, int kv_mode, const int32_t* idx,
                           const int32_t* count, int L, int layer_begin, int layer_end, int B, int Hq,
                           int G, int D, int rows, int k, float scale, float* out, float* lse,
                           void* ws, size_t ws_bytes, spc_stream_t stream);

/* ------------------------------------------------------------------------
 * spc_kv_desc_init / spc_sparse_decode_attn_kv — the same attention (O10, reading
 * R15; Eq.1 restricted to the selected rows) with the selected rows
 * gathered by the TMA unit (tile::gather4, 4 rows per request) instead of per-thread
 * copies: the hot path's kernel.
 *
 * spc_kv_desc_init is a SETUP call (synchronous, not capturable, once per KV cache):
 * it encodes one TMA descriptor per layer for K and for V, each over the layer's
 * [B*G*rows][D] bf16 tensor, and copies them to `desc` (DEVICE memory of
 * spc_kv_desc_bytes(L) bytes, 64-byte aligned, caller-owned; valid as long as the
 * cache allocations it describes).  k_layers / v_layers here are HOST arrays of L
 * device pointers (16-byte aligned; HBM, not mapped host memory).
 * Errors: SPC_E_NULL, SPC_E_SHAPE (sizes <= 0, B*G*rows >= 2^31), SPC_E_UNSUPPORTED
 * (D not 64/128), SPC_E_RANGE (misaligned desc or layer pointer), SPC_E_CUDA.
 *
 * spc_sparse_decode_attn_kv: arguments as spc_sparse_decode_attn, with the KV cache
 * given by `kv_desc` (from spc_kv_desc_init with the same L, B, G, D, rows) instead of
 * pointer tables; bf16 only.  kv_mode SPC_KV_INDEXED or SPC_KV_SLOTS (then the desc
 * describes the [B][G][k][D] budget buffers and rows = k).  Same workspace
 * (spc_attn_workspace, zero-filled once; not shared by calls executing at the same
 * time).  Results agree with spc_sparse_decode_attn within the O10 tolerance.
 * ---------------------------------------------------------------------- */
size_t spc_kv_desc_bytes(int L);
int spc_kv_desc_init(void* desc, const void* const* k_layers, const void* const* v_layers, int L,
                     int B, int G, int D, int rows);
int spc_sparse_decode_attn_kv(const void* kv_desc, const void* q, int kv_mode, const int32_t* idx,
                              const int32_t* count, int L, int layer_begin, int layer_end, int B,
                              int Hq, int G, int D, int rows, int k, float scale, float* out,
                              float* lse, void* ws, size_t ws_bytes, spc_stream_t stream);

/* spc_attn_merge — log-sum-exp merge of P partial attentions, O12.
 * o_parts [P][n][D] f32, lse_parts [P][n] f32 (-inf = empty part);
 * out [n][D] = sum_p e^{lse_p - M} o_p / sum_p e^{lse_p - M}, M = max_p lse_p;
 * lse_out [n] (or NULL) = M + log sum_p e^{lse_p - M}. */
int spc_attn_merge(const float* o_parts, const float* lse_parts, int P, int n, int D, float* out,
                   float* lse_out, spc_stream_t stream);

/* ------------------------------------------------------------------------
 * spc_rethead_qk — the retrieval head's per-step front-end (SURVEY §8(f)
 * NEXT-1): embedding lookup -> RMSNorm -> Q/K projection GEMV -> RoPE (YaRN
 * scaled) -> K-cache append.  It precedes spc_score on the critical path.
 *
 * Paper §4.3: the retrieval head keeps the DLM's embedding module and
 * QK projection weights, extends its context with YaRN, and maintains a full
 * K cache; ~60 MB of weights.  SPEC run_retrieval_head: the
 * new key is appended at position = cache length, then scored (reading R6).
 * Per request b (readings R22-R24):
 *   x  = emb[token[b]];  xn = bf16(w * bf16(x / sqrt(mean(x^2) + eps)))
 *   pre = W_qk xn (fp32 accumulation);  RoPE on pairs (i, i + D/2) of every
 *   head with a = fl32(pos[b] * inv_freq[i]), c = cos(a)*mscale,
 *   s = sin(a)*mscale: (u, v) -> (u c - v s, v c + u s);  results rounded to bf16.
 * token    [B] int32 DEVICE, 0 <= token < V (UB otherwise)
 * emb      [V][H] bf16;  norm_w [H] bf16 or NULL (unit weight);  eps > 0
 * w_qk     [(Hq+G)*D][H] bf16: rows h*D + d for query head h < Hq, then
 *          (Hq + g)*D + d for key head g (W_q then W_k, nn.Linear layout)
 * inv_freq [D/2] f32 (the caller's rotary table, e.g. YaRN-scaled); mscale
 *          multiplies cos and sin (YaRN attention scaling; 1 = plain RoPE)
 * pos      [B] int32 DEVICE: the new token's position = keys already cached,
 *          0 <= pos < Smax; or NULL: pos[b] = seq_len_out[b] - 1, read on the device
 *          (a decode loop whose seq_len already counts the new token, e.g. a growing
 *          context that advances seq_len in place every step)
 * q_out    [B][Hq][D] bf16 out (the query spc_score takes)
 * kr       [B][G][Smax][D] bf16 in/out: row pos[b] of every group written
 * seq_len_out [B] int32: with pos, out (pos + 1, the seq_len spc_score takes) or NULL;
 *          with pos NULL, in (unchanged)
 * x_out    [B][H] bf16 out or NULL: xn (the normalised input)
 * Supported: D in {64, 128}, H % 8 == 0, B <= 16, B*H*2 <= 200 KiB.
 * Errors: SPC_E_NULL (also: pos and seq_len_out both NULL), SPC_E_SHAPE, SPC_E_RANGE
 * (16-byte alignment of emb, w_qk), SPC_E_UNSUPPORTED, SPC_E_CUDA.
 * ---------------------------------------------------------------------- */
int spc_rethead_qk(const int32_t* token, const void* emb, int V, int H, const void* norm_w,
                   float eps, const void* w_qk, const float* inv_freq, float mscale,
                   const int32_t* pos, int B, int Hq, int G, int D, int Smax, void* q_out,
                   void* kr, int32_t* seq_len_out, void* x_out, spc_stream_t stream);

/* ------------------------------------------------------------------------
 * spc_llm_* — the LLM decoder layer's elementwise operations around the sparse
 * attention (the per-layer dense compute that the KV prefetch
 * overlaps, Fig. 3 / P:199, "concurrent execution of computation and KV cache
 * prefetching").  A Llama-style layer (DeepSeek-R1-Distill-Llama-8B shape, random
 * weights, reading R30): x = RMSNorm(h); [q k v] = W_qkv x; RoPE(q, k); append k, v;
 * a = SparseAttn(q, selected K/V) (spc_sparse_decode_attn_kv); h += W_o a;
 * x = RMSNorm(h); h += W_down(silu(W_g x) * W_u x).  The projections are plain cuBLAS
 * GEMMs issued by the caller; these calls are the rest.  bf16 storage (raw uint16
 * bits), fp32 arithmetic, all on `stream`, asynchronous, PDL-chained.
 * Errors: SPC_E_NULL (required pointer NULL), SPC_E_SHAPE (sizes <= 0, Hq % G, odd D),
 * SPC_E_UNSUPPORTED (add_rmsnorm: H % 4 or H > 16384; rope_append: D > 128),
 * SPC_E_RANGE (add_rmsnorm: h, delta, w, xn not 16-byte aligned; rope_append: slot_tok
 * not 16-byte aligned), SPC_E_CUDA.  Data-dependent violations (token or position out of
 * range) give zeros / no write; SPC_DEBUG builds flag them (spc_check_device_errors).
 *
 * spc_llm_embed:       h [B][H] f32 out = emb[token[b]] ([V][H] bf16; token DEVICE).
 * spc_llm_add_rmsnorm: h [B][H] f32 in/out (the residual stream); if delta [B][H] bf16
 *   is not NULL, h += delta first.  xn [B][H] bf16 out = bf16(w * bf16(h * r)),
 *   r = 1/sqrt(mean_i h_i^2 + eps) (the HF Llama form: normalise, round, scale, round).
 * spc_llm_rope_append: qkv [B][(Hq + 2G) D] bf16 (W_qkv rows: q heads, k heads, v heads);
 *   p = seq_len[b] - 1 (the new token's position, DEVICE; 0 <= p < rows).
 *   q_out [B][Hq][D] bf16 = RoPE(q); k_cache / v_cache [B][G][rows][D] bf16 (device or
 *   mapped host): row p = RoPE(k) / v.  RoPE on pairs (i, i + D/2) with angle
 *   fl32(p * inv_freq[i]) (inv_freq [D/2] f32): (u, v) -> (u cos - v sin, v cos + u sin).
 *   slot_tok [B][G][k] int32 or NULL (SLOTS mode: the slot map after
 *   spc_elastic_diff): when slot s of (b, g) holds token p, row s of the budget
 *   buffers k_buf / v_buf [B][G][k][D] receives the same key / value.
 * spc_llm_swiglu:      gu [B][2F] bf16 (gate then up) -> y [B][F] bf16 =
 *   bf16(silu(gate) * up), silu(g) = g / (1 + e^-g).
 * spc_llm_f32_to_bf16: y[i] = bf16_rn(x[i]), n elements.
 * spc_llm_argmax:      token_out[b] = argmax_v logits[b][v] ([B][V] bf16; lowest index
 *   among equal maxima; NaN ignored; 0 if all NaN), then seq_len[b] += 1 when seq_len is
 *   not NULL: the next step's token and position, without a host round trip.
 * ---------------------------------------------------------------------- */
int spc_llm_embed(const int32_t* token, const void* emb, int V, int H, int B, float* h,
                  spc_stream_t stream);
int spc_llm_add_rmsnorm(float* h, const void* delta, const void* w, int B, int H, float eps,
                        void* xn, spc_stream_t stream);
int spc_llm_rope_append(const void* qkv, const float* inv_freq, const int32_t* seq_len, int B,
                        int Hq, int G, int D, int rows, void* q_out, void* k_cache, void* v_cache,
                        const int32_t* slot_tok, int k, void* k_buf, void* v_buf,
                        spc_stream_t stream);
int spc_llm_swiglu(const void* gu, int B, int F, void* y, spc_stream_t stream);
int spc_llm_f32_to_bf16(const float* x, long long n, void* y, spc_stream_t stream);
int spc_llm_argmax(const void* logits, int B, int V, int32_t* token_out, int32_t* seq_len,
                   spc_stream_t stream);

/* ------------------------------------------------------------------------
 * Adaptive memory management — HOST functions (no GPU work).
 * Paper §6: Eq. 6-8, Algorithm 1 (thresholds at compile time) and
 * Algorithm 2 (progressive per-layer offload during decode).  Readings R25-R27.
 *   M_part(S, l_gpu) = trunc(runtime_factor * model_bytes)
 *       + 2*bytes_per_elem*R*[(l_gpu + extra_layers)*S + (L - l_gpu)*B]*H*D   (Eq. 7;
 *   Eq. 6 is l_gpu = L).  extra_layers: the paper's 1 + alpha (retrieval-head cache +
 *   repeat_kv buffer); this framework never materialises repeat_kv, so 1.
 * ---------------------------------------------------------------------- */
typedef struct {
  int64_t mem_gpu;        /* Mem_GPU, bytes */
  int64_t model_bytes;    /* M_O + M_D, bytes */
  double runtime_factor;  /* 1.3: runtime memory = 30% of the model */
  int L, H, D;            /* LLM layers, KV heads, head dim */
  int extra_layers;       /* KV layers besides the L of the LLM (paper: 1 + alpha) */
  int R;                  /* concurrent requests */
  int64_t B;              /* retrieval budget, tokens */
  int bytes_per_elem;     /* 2 (fp16 / bf16): the KV coefficient 4 = 2 * 2 */
} spc_plan_cfg;
/* Eq. 7 in bytes (-1 on invalid arguments). */
int64_t spc_plan_mem_part(const spc_plan_cfg* cfg, int64_t S, int l_gpu);
/* Algorithm 1: thresholds[0..L]; S^T_i = floor((C - c*i*B) / (c*(L + extra - i))) with
 * C = mem_gpu - trunc(runtime_factor*model_bytes), c = 2*bytes_per_elem*R*H*D (Eq. 7's
 * coefficient on the B term, reading R25); INT64_MAX where no KV layer stays on the GPU.
 * Errors: SPC_E_NULL, SPC_E_SHAPE, SPC_E_BUDGET (C <= 0). */
int spc_plan_thresholds(const spc_plan_cfg* cfg, int64_t* thresholds);
/* Eq. 8: the largest l_gpu in [0, L] with M_part(S, l_gpu) <= mem_gpu.  SPC_E_BUDGET (and
 * *l_gpu = -1, *shortfall = M_part(S, 0) - mem_gpu) when even l_gpu = 0 does not fit. */
int spc_plan_max_resident(const spc_plan_cfg* cfg, int64_t S, int* l_gpu, int64_t* shortfall);
/* Algorithm 2, one check at sequence length S: while S >= thresholds[*l_cpu] and
 * *l_cpu < L, offload layer L - *l_cpu - 1 (listed in offload_layers, may be NULL) and
 * increment *l_cpu; *n_offload = layers offloaded by this call (0 = no action). */
int spc_plan_step(const int64_t* thresholds, int L, int64_t S, int* l_cpu, int32_t* offload_layers,
                  int* n_offload);

/* ------------------------------------------------------------------------
 * spc_mla_sparse_attn — MLA decode attention over each head's selected latent rows
 * (SURVEY §8(f) NEXT-3).  Paper §4.3 (Fig. 5(e)): MLA caches a latent c per
 * token; retrieval stays head-level as for MHA (alpha = 1: one selection per head,
 * e.g. spc_score with G = H); "only the selected c cache is subjected to the increase
 * in dimension".  Result (reading R29: the expansion absorbed into query and output,
 * mathematically identical to expanding the selected rows):
 *   o[b][h] = sum_j softmax_j(scale * [q_nope.W_UK c_j + q_pe.kpe_j]) W_UV c_j
 * over j in idx[b][h][0 .. count[b][h]); lse[b][h] natural-log log-sum-exp (-inf, o = 0
 * when the count is 0).
 * All L layers in one call (the selection is layer-independent):
 * q      [L][B][H][DN + DR] bf16 (no-rope part, then the rope part)
 * cache  DEVICE array of L pointers, each [B][Smax][DC + DR] bf16: latent c (DC) then
 *        the shared rope key kpe (DR), 16-byte aligned
 * w_uk   DEVICE array of L pointers to [H][DN][DC] bf16; w_uv likewise to [H][DV][DC]
 * idx    [B][H][k] int32 rows (< Smax), count [B][H] int32 DEVICE
 * out    [L][B][H][DV] f32;  lse [L][B][H] f32 or NULL
 * ws     >= spc_mla_workspace(L, B, H, k) bytes, zero-filled on first use (left so)
 * Supported: DC = 512, DR = 64 (DeepSeek-V2/V3 MLA), DN <= 512, DV <= 1024.
 * Errors: SPC_E_NULL, SPC_E_SHAPE, SPC_E_BUDGET, SPC_E_UNSUPPORTED, SPC_E_WORKSPACE,
 * SPC_E_CUDA.
 * ---------------------------------------------------------------------- */
size_t spc_mla_workspace(int L, int B, int H, int k);
int spc_mla_sparse_attn(const void* q, const void* const* cache, const void* const* w_uk,
                        const void* const* w_uv, const int32_t* idx, const int32_t* count, int L,
                        int B, int H, int Smax, int k, int DC, int DR, int DN, int DV, float scale,
                        float* out, float* lse, void* ws, size_t ws_bytes, spc_stream_t stream);

/* ------------------------------------------------------------------------
 * spc_decode_step — the whole single-device §8(a) step in ONE call (native executor):
 * spc_score(LOGITS) -> spc_select (NORM, GROUP, top-k, INDEXED elastic diff) ->
 * spc_sparse_decode_attn over all L layers (INDEXED), enqueued on `stream`; when
 * spc_select does not apply (Smax > 135168, Smax % 4, or B*G*8 > SMs) the separate
 * spc_score(ALL) + spc_topk + spc_elastic_diff calls are used.  Same definitions and
 * results as those calls in sequence.  The caller owns all buffers and the rolling
 * state: prev_idx / prev_count (previous selection, count 0 on the first step) in,
 * cur_idx / cur_count out -- swap them between steps.  scale is both the retrieval
 * head's and the LLM's softmax scale (fl(1/sqrt(D)) in the paper's setting).
 * ws >= spc_decode_step_workspace(L, B, Hq, G, D, Smax, k) bytes, zero-filled once.
 * Errors: those of the calls it makes, and SPC_E_NULL / SPC_E_WORKSPACE.
 * ---------------------------------------------------------------------- */
typedef struct {
  int L, B, Hq, G, D, Smax, rows, k, force_last;
  float scale;
  const void* q_ret;              /* [B][Hq][D] bf16 retrieval query */
  const void* kr;                 /* [B][G][Smax][D] bf16 retrieval keys */
  const int32_t* seq_len;         /* [B] */
  const void* q_llm;              /* [L][B][Hq][D] bf16 */
  const void* const* k_layers;    /* [L] -> [B][G][rows][D] bf16 */
  const void* const* v_layers;
  float* logits;                  /* [B][Hq][Smax] scratch */
  float* head_max;                /* [B][Hq] */
  int64_t* head_sumfix;           /* [B][Hq] */
  float* group_score;             /* [B][G][Smax] */
  const int32_t* prev_idx;        /* [B][G][k] */
  const int32_t* prev_count;      /* [B][G] */
  int32_t* cur_idx;               /* [B][G][k] out */
  int32_t* cur_count;             /* [B][G] out */
  int32_t* load_tok;              /* [B][G][k] out: cur \ prev */
  int32_t* n_load;                /* [B][G] out */
  float* out;                     /* [L][B][Hq][D] f32 */
  float* lse;                     /* [L][B][Hq] or NULL */
  void* ws;
  size_t ws_bytes;
  const void* kv_desc;            /* NULL, or spc_kv_desc_init of k_layers / v_layers:
                                     the attention then runs spc_sparse_decode_attn_kv */
} spc_step_args;
size_t spc_decode_step_workspace(int L, int B, int Hq, int G, int D, int Smax, int k);
int spc_decode_step(const spc_step_args* args, spc_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* SPC_H_ */
