/*
 * cortex_dev.h — PRIVATE tuning / test interface of libcortex_b200.so.
 *
 * Not part of the reference-facing boundary (include/cortex_b200.h): nothing on the
 * product path calls these. They let tests pin a kernel variant (to cross-check it
 * against the default) and let the benchmarks in benchmarks/ run A/B comparisons.
 * Every knob has a compiled-in default that is the product behaviour; the library reads
 * no environment variables.
 */
#ifndef CORTEX_DEV_H_
#define CORTEX_DEV_H_

#include <stdint.h>

#include "cortex_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

enum CortexKnob {
  CORTEX_KNOB_PDL = 0,        /* programmatic dependent launch: 1 on (default), 0 off */
  CORTEX_KNOB_GEMM_MODE,      /* 0 auto, 1 force 1-SM, 2 force 2-SM, 3 prefer cluster split-K */
  CORTEX_KNOB_GEMM_STREAM_K,  /* 2-SM scheduling: -1 auto (whole tiles), 0 whole, 1 stream-K */
  CORTEX_KNOB_GEMM_TN,        /* 2-SM token tile width: -1 planner, else 64..256 step 32 */
  CORTEX_KNOB_GEMM_L2PF,      /* weight K blocks prefetched to L2 before the PDL wait (0) */
  CORTEX_KNOB_SK_KS,          /* cluster split-K: splits (-1 planner, 2..4) */
  CORTEX_KNOB_SK_MT,          /* cluster split-K: token tiles (-1 planner, 1..4) */
  CORTEX_KNOB_SK_NW,          /* cluster split-K: weight sub-tiles per pair (-1 auto, 2) */
  CORTEX_KNOB_SK_ISSUE,       /* cluster split-K: TMA issuing threads (1, 2 default, 4) */
  CORTEX_KNOB_FMHA_2Q,        /* tcgen05 attention: 1 two Q tiles (default), 0 one, -1 by waves */
  CORTEX_KNOB_FMHA_PLO,       /* tcgen05 attention: P as bf16 hi + lo (1, default) or hi (0) */
  CORTEX_KNOB_GEMM_TILE_OVH,  /* 2-SM tile planner: per-tile overhead in token columns (32) */
  CORTEX_KNOB_COUNT
};

int32_t cortex_dev_set_knob(int32_t knob, int32_t value);
int32_t cortex_dev_get_knob(int32_t knob);
/* cudaGetLastError() of the library's runtime (diagnosing a CORTEX_ECUDA status). */
int32_t cortex_dev_last_cuda_error(void);

/* Introspection of the GEMM planner (host functions). */
int32_t cortex_gemm_splits(int32_t M, int32_t N, int32_t K);
int32_t cortex_gemm_path(int32_t M, int32_t N, int32_t K); /* 1: 1-SM, 2: 2-SM, 3: split-K */
int32_t cortex_gemm2_tile(int32_t M, int32_t N, int32_t K); /* TN | (stream_k << 16) */
int32_t cortex_gemm_splitk_plan(int32_t M, int32_t N, int32_t K, int32_t* tn_out,
                                int32_t* m_tiles_out, int32_t* weight_subtiles_out);
int32_t cortex_decode_tiles_per_chunk(int32_t total_tiles, int32_t n_kv_heads);
int32_t cortex_act_box_rows(void); /* token rows per TMA box of the GEMMs' activation maps */

/* mma.sync causal paged prefill attention: the cross-check of cortex_fmha_prefill_tc. */
int32_t cortex_paged_prefill_attn(const void* tmap_kv, const void* q, void* out,
                                  const int32_t* table, int32_t table_stride,
                                  const int32_t* seq_row, const int32_t* seq_prefix,
                                  const int32_t* seq_kvlen, const int32_t* seq_qstart,
                                  const int32_t* seq_qlen, int32_t n_seqs, int32_t max_qlen,
                                  int32_t n_kv_heads, int32_t group, int64_t k_row0,
                                  int64_t v_row0, float softmax_scale, cortex_stream_t stream);

#ifdef __cplusplus
}
/* knob values, indexed by CortexKnob (defaults in kvpool.cu) */
extern int g_cortex_knob[CORTEX_KNOB_COUNT];
#endif

#endif /* CORTEX_DEV_H_ */
