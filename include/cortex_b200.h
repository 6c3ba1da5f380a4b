/*
 * cortex_b200.h — C ABI of the B200 stage-engine kernels (libcortex_b200.so).
 *
 * The reference (arXiv 2510.14126 "Cortex", package `stagesim`) has no native
 * code and no FFI: its engine is the pure-Python `EngineState`
 * (/root/reference/pkg/src/stagesim/engines.py:101-246). These exports are the
 * device-side half of that engine's state transitions; the Python host mirror
 * (paper_2510_14126_b200/engine.py, `GpuEngineState`) keeps the reference's
 * method names and calls these through ctypes. Each entry point below names the
 * EngineState transition it implements.
 *
 * Conventions
 *  - Every export returns int32: 0 = ok, <0 = error (CortexStatus). The host
 *    raises InternalInvariantViolation (stagesim/errors.py:8) on non-zero.
 *  - Pointers are device pointers unless stated; sizes are element counts.
 *  - No allocation happens inside any call; the caller owns all buffers.
 *  - Work is enqueued on `stream` (a cudaStream_t passed as void*); nothing
 *    synchronises the host.
 *  - Block tables are int32 matrices [rows, table_stride]; a sequence's row holds
 *    its stage-prefix blocks (ceil(P/16)) followed by its private blocks.
 *  - KV cache: one bf16 allocation cache[layer][k|v][block][kv_head][16][128];
 *    k_row0 / v_row0 are the 128-wide row offsets of a layer's K and V planes.
 */
#ifndef CORTEX_B200_H_
#define CORTEX_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(CORTEX_BUILDING)
typedef struct CUstream_st* cortex_stream_t; /* == cudaStream_t */
#else
typedef void* cortex_stream_t; /* cudaStream_t */
#endif

enum {
  CORTEX_OK = 0,
  CORTEX_EBADARG = -1,
  CORTEX_ECUDA = -2,
  CORTEX_ENOBLOCKS = -3,
  CORTEX_EUNSUPPORTED = -4,
  CORTEX_ETIMEOUT = -5 /* a cross-GPU wait exceeded its bound (peer rank gone) */
};

/* ABI version (major * 100 + minor). Tuning / test knobs (kernel variants, PDL on/off)
 * are NOT part of this interface: see paper_2510_14126_b200/csrc/cortex_dev.h. */
int32_t cortex_abi_version(void);

/* ---- KV block pool (bitmap, bit = 1 -> free) -------------------------------
 * EngineState.admit (engines.py:142-166): cold prefix blocks + prompt blocks;
 * the lazy per-16-token append during EngineState.advance_decode
 * (engines.py:172-194).
 * Requests are served in order, lowest free block first; request i writes its
 * counts[i] block ids to table[rows[i]][cols[i] ...]. All-or-nothing: if the
 * batch does not fit, nothing changes and *status is set to CORTEX_ENOBLOCKS.
 */
int32_t cortex_kv_alloc(uint32_t* bitmap, int32_t nblocks, int32_t id_base,
                        const int32_t* counts, const int32_t* rows, const int32_t* cols,
                        int32_t n_req, int32_t* table, int32_t table_stride, int32_t* status,
                        cortex_stream_t stream);

/* EngineState.complete_call (engines.py:206-214) frees the call's private
 * blocks; EngineState.evict_idle_prefix (engines.py:219-226) frees a prefix.
 * A double free or an id outside the pool sets *status = CORTEX_EBADARG. */
int32_t cortex_kv_free(uint32_t* bitmap, int32_t nblocks, int32_t id_base, const int32_t* table,
                       int32_t table_stride, const int32_t* rows, const int32_t* cols,
                       const int32_t* counts, int32_t n_req, int32_t* status,
                       cortex_stream_t stream);

/* Warm admit (engines.py:149-150): copy a resident prefix's block ids into the
 * call's row: table[dst_rows[i]][dst_cols[i] + k] = table[src_rows[i]][k]. */
int32_t cortex_table_copy(int32_t* table, int32_t table_stride, const int32_t* src_rows,
                          const int32_t* dst_rows, const int32_t* dst_cols,
                          const int32_t* counts, int32_t n, cortex_stream_t stream);

/* Same three operations with the request arrays in HOST memory (plain int32 arrays,
 * read during the call and passed to the kernel by value, in chunks of 256 requests for
 * alloc / free and 128 for copies; allocation chunks are served in order). No staging
 * copy precedes the kernel, so the allocator adds no copy-engine round trip to a step. */
int32_t cortex_kv_alloc_h(uint32_t* bitmap, int32_t nblocks, int32_t id_base,
                          const int32_t* counts, const int32_t* rows, const int32_t* cols,
                          int32_t n_req, int32_t* table, int32_t table_stride, int32_t* status,
                          cortex_stream_t stream);
int32_t cortex_kv_free_h(uint32_t* bitmap, int32_t nblocks, int32_t id_base, const int32_t* table,
                         int32_t table_stride, const int32_t* rows, const int32_t* cols,
                         const int32_t* counts, int32_t n_req, int32_t* status,
                         cortex_stream_t stream);
int32_t cortex_table_copy_h(int32_t* table, int32_t table_stride, const int32_t* src_rows,
                            const int32_t* dst_rows, const int32_t* dst_cols,
                            const int32_t* counts, int32_t n, cortex_stream_t stream);

/* Free-block count (occupancy metric; adds into *out_free). */
int32_t cortex_kv_count_free(const uint32_t* bitmap, int32_t nblocks, int32_t* out_free,
                             cortex_stream_t stream);

/* ---- TMA descriptors ---------------------------------------------------------
 * Encode a 128-byte CUtensorMap (host memory at tmap_out) over a bf16 row-major
 * matrix [rows, cols] with row pitch in bytes; box = (box_rows, box_cols),
 * box_cols * 2 == 128 (SWIZZLE_128B). */
int32_t cortex_tmap_encode_2d_bf16(void* tmap_out, const void* gptr, uint64_t rows, uint64_t cols,
                                   uint64_t row_pitch_bytes, uint32_t box_rows,
                                   uint32_t box_cols);

/* ---- decoder forward (the GPU work behind admit's prefill and
 * advance_decode's emitted tokens) -------------------------------------------- */

/* tcgen05/TMEM GEMM: out[m, n] = sum_k X[m, k] W[n, k] (+ residual[m, n], fp32 with row
 * pitch ldr; the residual stream is fp32, so residual GEMMs use out_f32 = 1).
 * tmap_w over W [N, K] with box (128, 64); tmap_x over X [>= M, K] with box (16, 64).
 * out_f32: 0 = bf16 out, 1 = fp32 out, 2 = fused SwiGLU: W's rows are interleaved in
 * blocks of 64 gate rows then 64 matching up rows, and out[m, f] (bf16, N/2 features) =
 * silu(g) * u with g, u the fp32 accumulators (no residual); 3 = greedy-token partials
 * (the lm_head of a decode step, EngineState.advance_decode's emitted token): out is
 * float2 [M, ldo = N / 128] of (max, first index of the max as int bits) of each
 * 128-column chunk of the row, the full logits are never written (no residual);
 * cortex_argmax_partials reduces them.
 * workspace / counters: the split-K partials and the per-tile arrival counters (kept
 * zeroed) of the decode-sized kernels; 16 Mi floats and 64 Ki counters cover every
 * shape of the Llama-3-8B step (GemmWorkspace in ops.py). */
int32_t cortex_gemm_bf16(const void* tmap_w, const void* tmap_x, int32_t M, int32_t N, int32_t K,
                         void* out, int32_t ldo, int32_t out_f32, const void* residual,
                         int32_t ldr, float* workspace, uint64_t workspace_bytes,
                         int32_t* counters, int32_t n_counters, cortex_stream_t stream);

/* QKV projection with RoPE and the paged KV append fused into the GEMM epilogue (the
 * per-token KV write of EngineState.admit's prefill and advance_decode's decode steps,
 * engines.py:142-194): W is [N = (hq + 2 hkv) * 128, K] ([q heads | k heads | v heads]);
 * for token m the accumulators are rounded to bf16, q / k heads rotated (rotate-half)
 * and rounded again, q written to q_out [M, hq, 128] and k / v to the token's paged slot
 * of the layer's K / V plane (128-wide rows k_row0 / v_row0 of cache). The qkv
 * activation is never written. tok_dst / tok_cs come from cortex_rope_token_prep (once
 * per step): tok_dst[m] = (table[tok_row[m]][tok_col[m]] * hkv) * 16 + tok_off[m], the
 * token's row within a plane for kv head 0; tok_cs[m] = cos | sin [128] fp32 at
 * tok_pos[m] (tables [max_pos, 64]). */
typedef struct {
  void* q_out;
  void* cache;
  int64_t k_row0, v_row0;
  const int32_t* tok_dst;
  const float* tok_cs;
  int32_t hq, hkv;
} cortex_rope_epilogue_t;
int32_t cortex_rope_token_prep(const int32_t* table, int32_t table_stride, const int32_t* tok_pos,
                               const int32_t* tok_row, const int32_t* tok_col,
                               const int32_t* tok_off, const float* cos_tab, const float* sin_tab,
                               int32_t n_tok, int32_t hkv, int32_t* tok_dst, float* tok_cs,
                               cortex_stream_t stream);
int32_t cortex_gemm_qkv_rope(const void* tmap_w, const void* tmap_x, int32_t M, int32_t N,
                             int32_t K, const cortex_rope_epilogue_t* epi, float* workspace,
                             uint64_t workspace_bytes, int32_t* counters, int32_t n_counters,
                             cortex_stream_t stream);

/* out[t] (fp32, the residual stream) = emb[tokens[index ? index[t] : t]] (bf16 table). */
int32_t cortex_embed(const void* emb, const int32_t* tokens, const int32_t* index, int32_t n_tok,
                     int32_t d, void* out, cortex_stream_t stream);

/* y[r] (bf16) = x[rows ? rows[r] : r] (fp32) * rsqrt(mean(x^2) + eps) * w (bf16). */
int32_t cortex_rmsnorm(const void* x, const int32_t* rows, int32_t n_rows, const void* w,
                       int32_t d, float eps, void* y, cortex_stream_t stream);

/* RoPE on q/k + write k, v of each token into its paged slot
 * (table[tok_row][tok_col], offset tok_off). */
int32_t cortex_rope_kv_append(const void* qkv, void* q_out, void* cache, int64_t k_row0,
                              int64_t v_row0, const int32_t* table, int32_t table_stride,
                              const int32_t* tok_pos, const int32_t* tok_row,
                              const int32_t* tok_col, const int32_t* tok_off,
                              const float* cos_tab, const float* sin_tab, int32_t n_tok,
                              int32_t hq, int32_t hkv, cortex_stream_t stream);

/* Greedy token per row from cortex_gemm_bf16's out mode 3 partials (float2 [n_rows,
 * n_chunks]); the same token as cortex_argmax over the full logits. */
int32_t cortex_argmax_partials(const void* partials, int32_t n_chunks, int32_t n_rows,
                               int32_t* out_tok, const int32_t* slot, int32_t* slot_tok,
                               int32_t* hist, int32_t hist_stride, const int32_t* hist_pos,
                               cortex_stream_t stream);

/* Greedy token per row; optional scatter into per-slot state. */
int32_t cortex_argmax(const float* logits, int64_t ld, int32_t n_rows, int32_t vocab,
                      int32_t* out_tok, const int32_t* slot, int32_t* slot_tok, int32_t* hist,
                      int32_t hist_stride, const int32_t* hist_pos, cortex_stream_t stream);

/* ---- fp32 decoder step (tiny config-1 model; storage and arithmetic fp32) ----
 * Replaces the same EngineState transitions as the bf16 exports (admit -> prefill,
 * advance_decode -> decode steps, stagesim/engines.py:142-194) when the engine is built
 * with precision "f32": the north star's "1e-5 in fp32, greedy tokens identical" bar.
 * cortex_f32_gemm: out[M, N] = X[M, K] W[N, K]^T; mode 0 plain, 1 + residual (out may
 * alias it), 2 SwiGLU: W is [2N, K] (gate rows then up rows), out = silu(g) * u.
 * cortex_f32_attention: per token t, causal attention over keys 0..tok_pos[t] of table
 * row tok_row[t] (stage-prefix blocks for positions < tok_prefix[t], then private
 * blocks); q / out [n_tok, hq, 128], KV cache rows of 128 fp32 (same layout as bf16). */
int32_t cortex_f32_gemm(const float* x, int32_t ldx, const float* w, int32_t M, int32_t N,
                        int32_t K, float* out, int32_t ldo, const float* residual, int32_t ldr,
                        int32_t mode, cortex_stream_t stream);
int32_t cortex_f32_embed(const float* emb, const int32_t* tokens, const int32_t* index,
                         int32_t n_tok, int32_t d, float* out, cortex_stream_t stream);
int32_t cortex_f32_rmsnorm(const float* x, const int32_t* rows, int32_t n_rows, const float* w,
                           int32_t d, float eps, float* y, cortex_stream_t stream);
int32_t cortex_f32_rope_kv_append(const float* qkv, float* q_out, float* cache, int64_t k_row0,
                                  int64_t v_row0, const int32_t* table, int32_t table_stride,
                                  const int32_t* tok_pos, const int32_t* tok_row,
                                  const int32_t* tok_col, const int32_t* tok_off,
                                  const float* cos_tab, const float* sin_tab, int32_t n_tok,
                                  int32_t hq, int32_t hkv, cortex_stream_t stream);
int32_t cortex_f32_attention(const float* q, const float* cache, int64_t k_row0, int64_t v_row0,
                             const int32_t* table, int32_t table_stride, const int32_t* tok_row,
                             const int32_t* tok_prefix, const int32_t* tok_pos, int32_t n_tok,
                             int32_t hq, int32_t hkv, float scale, float* out,
                             cortex_stream_t stream);

/* Paged decode attention (one query token per sequence), the GPU work of every token
 * EngineState.advance_decode emits (engines.py:172-194). Split along the context in
 * fixed 512-token chunks + LSE combine. o_part/lse_part: [n_seqs, max_splits, Hq, 128] /
 * [n_seqs, max_splits, Hq] fp32 workspace.
 * Without groups (n_groups = 0): max_splits >= max cortex_decode_splits(prefix, kv_len).
 * Cascade (n_groups > 0): the decode calls sharing a resident stage prefix are
 * contiguous (group g = calls [grp_first, grp_first + grp_count), prefix in table row
 * grp_row, grp_plen tokens); their prefix attention runs once per group (partials in
 * slots [0, prefix_slots), prefix_slots >= max ceil(ceil(P/16)/16)), the private
 * tokens per call (slots prefix_slots + ...). Every call with prefix_len > 0 must
 * belong to a group. max_group_count = largest grp_count. tmap_q (cortex_tmap_encode_q)
 * selects the tcgen05 cascade pass.
 * parts (bitmask): 1 = shared-prefix cascade pass, 2 = per-call context splits, 4 = LSE
 * combine (7 = all), so the cascade pass can run on a second stream concurrently with
 * the splits (join before the combine).
 * Balanced ("flat") plan (seq_tile_start != NULL): call b's tiles (its private tiles
 * under cascade, all tiles otherwise) are flat tiles [seq_tile_start[b],
 * seq_tile_start[b] + n_b) of one sequence of total_tiles; CTA (c, kv head) streams
 * flat tiles [c W, (c+1) W), W = tiles_per_chunk <= 48, so every CTA does equal work
 * whatever the context lengths; call b's partials go to slots off + [0, (S_b + n_b - 1)
 * / W - S_b / W] (off = prefix_slots under cascade, else 0). NULL: fixed splits. */
int32_t cortex_decode_splits(int32_t prefix_len, int32_t kv_len);
int32_t cortex_paged_decode_attn(
    const void* tmap_kv, const void* q, const int32_t* table, int32_t table_stride,
    const int32_t* seq_row, const int32_t* seq_prefix, const int32_t* seq_kvlen,
    const int32_t* seq_tile_start, int32_t total_tiles, int32_t tiles_per_chunk, int32_t n_seqs,
    int32_t n_kv_heads, int32_t group, int64_t k_row0, int64_t v_row0, float softmax_scale,
    float* o_part, float* lse_part, int32_t max_splits, void* out, const int32_t* grp_row,
    const int32_t* grp_plen, const int32_t* grp_first, const int32_t* grp_count, int32_t n_groups,
    int32_t max_group_count, int32_t prefix_slots, const void* tmap_q, int32_t parts,
    cortex_stream_t stream);

/* TMA descriptor over q [n_tok, hq, 128] (box 64 dims x group heads x 128/group tokens)
 * for the tensor-core attention kernels; tmap_q above selects the tcgen05 cascade pass. */
int32_t cortex_tmap_encode_q(void* tmap_out, const void* q, uint64_t n_tok, int32_t hq,
                             int32_t group);

/* tcgen05 flash attention, 128 query rows (tokens x GQA group) per CTA, paged K/V in
 * 8-block key tiles, TMEM S/O accumulators, P entering PV as bf16 hi + lo. Prefill (the
 * GPU work of EngineState.admit's prompt / cold-prefix prefill, engines.py:142-166):
 * causal over the sequence's row (seq_prefix tokens of stage prefix, then private
 * positions); query token i of sequence s is row seq_qstart[s] + i of q / out
 * [n_tok, hq, 128] at position seq_kvlen[s] - seq_qlen[s] + i. Cascade: the
 * shared-prefix pass of decode (partials into slots [0, prefix_slots) of o_part /
 * lse_part, rows = decode index). */
int32_t cortex_fmha_prefill_tc(const void* tmap_kv, const void* tmap_q, void* out,
                               const int32_t* table, int32_t table_stride, const int32_t* seq_row,
                               const int32_t* seq_prefix, const int32_t* seq_kvlen,
                               const int32_t* seq_qstart, const int32_t* seq_qlen, int32_t n_seqs,
                               int32_t max_qlen, int32_t n_kv_heads, int32_t group,
                               int64_t k_row0, int64_t v_row0, float softmax_scale,
                               cortex_stream_t stream);
int32_t cortex_fmha_cascade_tc(const void* tmap_kv, const void* tmap_q, const int32_t* table,
                               int32_t table_stride, const int32_t* grp_row,
                               const int32_t* grp_plen, const int32_t* grp_first,
                               const int32_t* grp_count, int32_t n_groups, int32_t max_count,
                               int32_t prefix_slots, int32_t n_kv_heads, int32_t group,
                               int64_t k_row0, int64_t v_row0, float softmax_scale,
                               float* o_part, float* lse_part, int32_t max_splits,
                               cortex_stream_t stream);

/* ---- a decoder step's layer loop from native code -----------------------------------
 * The layers [layer_begin, layer_end) of one step (the GPU work behind an engine step's
 * admit prefills and advance_decode tokens, stagesim/engines.py:142-194), launched in the
 * order and with the arguments the per-op exports above take one call at a time: per
 * layer cortex_rmsnorm (attn_norm) -> cortex_gemm_qkv_rope -> decode attention
 * (cortex_paged_decode_attn; with cascade groups and a side stream: parts 1 on
 * side_stream, the prompt prefill on side_stream2 (or after parts 1 on side_stream),
 * parts 2 on stream, join, parts 4) -> prompt prefill
 * (cortex_fmha_prefill_tc, when not on the side stream) -> O projection + residual
 * (mode 1) -> cortex_rmsnorm (mlp_norm) -> gate/up with SwiGLU (mode 2) -> down +
 * residual (mode 1). cortex_decoder_t describes the model (built once); cortex_step_t
 * one step (device metadata uploaded by the caller; embed, rope_token_prep, final norm
 * and lm_head stay with the caller). Weight tensor maps are the 128-byte host
 * CUtensorMaps of cortex_tmap_encode_2d_bf16 (wgu rows interleaved as mode 2 expects);
 * tmap_xn / tmap_attn / tmap_act are the activation maps (box rows cortex's GEMMs
 * use), tmap_q from cortex_tmap_encode_q (required: the tcgen05 attention). K / V of
 * layer l are the 128-wide cache rows starting at 2 l plane_rows / (2 l + 1) plane_rows.
 * Returns the first failing launch's status. */
typedef struct {
  int32_t n_layers, d_model, hq, hkv, ffn;
  float eps, softmax_scale;
  const void* const* tmap_wqkv; /* [n_layers] */
  const void* const* tmap_wo;
  const void* const* tmap_wgu;
  const void* const* tmap_wd;
  const void* const* attn_norm; /* [n_layers] device bf16 [d_model] */
  const void* const* mlp_norm;
  const void* tmap_xn;
  const void* tmap_attn;
  const void* tmap_act;
  const void* tmap_kv;
  const void* tmap_q;
  float* x;    /* fp32 residual stream [>= n_tok, d_model] */
  void* xn;    /* bf16 [>= n_tok, d_model] */
  void* q;     /* bf16 [>= n_tok, hq * 128] */
  void* attn;  /* bf16 [>= n_tok, hq * 128] */
  void* act;   /* bf16 [>= n_tok, ffn] */
  void* cache;
  int64_t plane_rows;
  const int32_t* table;
  int32_t table_stride;
  const int32_t* tok_dst; /* cortex_rope_token_prep outputs of the step */
  const float* tok_cs;
  float* workspace;
  uint64_t workspace_bytes;
  int32_t* counters;
  int32_t n_counters;
} cortex_decoder_t;
typedef struct {
  int32_t n_tok, n_dec, n_pf, max_qlen, max_splits;
  int32_t layer_begin, layer_end;
  const int32_t *dec_row, *dec_prefix, *dec_kvlen;                      /* [n_dec] */
  const int32_t *pf_row, *pf_prefix, *pf_kvlen, *pf_qstart, *pf_qlen;   /* [n_pf] */
  const int32_t *grp_row, *grp_plen, *grp_first, *grp_count;            /* [n_groups] */
  int32_t n_groups, max_group_count, prefix_slots;
  float* o_part;
  float* lse_part;
  cortex_stream_t stream;
  cortex_stream_t side_stream;  /* NULL: every attention pass on stream */
  cortex_stream_t side_stream2; /* non-NULL: the prompt prefill here, beside the cascade */
} cortex_step_t;
int32_t cortex_decoder_layers(const cortex_decoder_t* model, const cortex_step_t* step);

/* ---- Tensor parallelism (TP = 2 inside one engine replica, BASELINE config 5) -------
 * the only collective on the path. The reference engine has no
 * model and hence no TP (engines.py:101-246); these exports implement the
 * all-reduce of the O / down projection partials that a TP = 2 replica of the
 * decoder forward (the GPU half of EngineState.advance_decode / admit) needs.
 *
 * cortex_sym_alloc: zeroed device buffer [flags (cortex_tp_flag_bytes()) | partial
 * parity 0 | partial parity 1], shareable with the peer rank through CUDA IPC
 * (cortex_ipc_get_handle -> 64-byte handle -> cortex_ipc_open_handle in the peer).
 * cortex_tp_signal: after the stream's preceding work (the partial-output GEMM),
 * publish `epoch` into the peer's flag word (system-scope release).
 * cortex_tp_allreduce_rmsnorm: wait until *flag >= epoch (system-scope acquire;
 * CORTEX_ETIMEOUT into *status after 10 s), then for each of n_rows rows
 * x += y0 + y1 (rank 0's partial first: bit-identical residuals on both ranks) and,
 * when w != NULL, out = bf16(x * rsqrt(mean(x^2) + eps) * w). y0 / y1 may be peer
 * (NVLink) pointers. flag == NULL skips the wait.
 */
int32_t cortex_sym_alloc(uint64_t bytes, void** out_ptr);
int32_t cortex_sym_free(void* ptr);
int32_t cortex_ipc_get_handle(void* ptr, void* handle_out /* 64 bytes */);
int32_t cortex_ipc_open_handle(const void* handle, void** out_ptr);
int32_t cortex_ipc_close(void* ptr);
int32_t cortex_tp_flag_bytes(void);
int32_t cortex_tp_signal(uint32_t* peer_flag, uint32_t epoch, cortex_stream_t stream);
int32_t cortex_tp_allreduce_rmsnorm(const float* y0, const float* y1, float* x, int32_t n_rows,
                                    int32_t d, const void* w, float eps, void* out,
                                    const uint32_t* flag, uint32_t epoch, int32_t* status,
                                    cortex_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* CORTEX_B200_H_ */
