// Native launcher of a decoder step's layer loop.
//
// The GPU work of one engine step (the prefills EngineState.admit starts and the tokens
// advance_decode emits, stagesim/engines.py:142-194) is ~10 launches per layer. Issued one
// by one from Python through ctypes they cost 4.0 ms of host time per config-2 step (32
// layers; benchmarks/host_overhead.py, forward timed on a drained GPU), a third of the
// ~12.5 ms of GPU work, host time that grows with every engine a process drives. This
// file issues the same launches, in the same order, with the same arguments, from C++
// (1.4 ms per step): the per-step plan (metadata upload, cascade groups, split counts)
// stays in Python (model.py), the loop over layers runs here. Every launch goes through
// the public entry points, so the GPU sees exactly the kernels the Python loop launches
// (bit-identical results, tests/test_step_gpu.py).
#include <cuda_runtime.h>

#include <mutex>

#include "common.cuh"

namespace {

struct StepEvents {
  int device = -1;
  cudaEvent_t fork = nullptr, join = nullptr, join2 = nullptr;
};

// fork / join events of the side stream, one pair per device of the process
cudaError_t step_events(StepEvents** out) {
  static StepEvents ev[16];
  static std::mutex mu;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 16) return cudaErrorInvalidDevice;
  std::lock_guard<std::mutex> lock(mu);
  StepEvents& s = ev[dev];
  if (s.device < 0) {
    if ((e = cudaEventCreateWithFlags(&s.fork, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&s.join, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&s.join2, cudaEventDisableTiming)) != cudaSuccess)
      return e;
    s.device = dev;
  }
  *out = &s;
  return cudaSuccess;
}

}  // namespace

extern "C" {

int32_t cortex_decoder_layers(const cortex_decoder_t* m, const cortex_step_t* s) {
  if (!m || !s || s->layer_begin < 0 || s->layer_end > m->n_layers ||
      s->layer_begin > s->layer_end || s->n_tok <= 0 || s->n_dec < 0 || s->n_pf < 0 ||
      s->n_dec + s->n_pf <= 0 || !m->tmap_wqkv || !m->tmap_wo || !m->tmap_wgu || !m->tmap_wd ||
      !m->attn_norm || !m->mlp_norm || !m->tmap_q || m->hkv < 1 || m->hq % m->hkv)
    return CORTEX_EBADARG;
  const int32_t T = s->n_tok, d = m->d_model, hq = m->hq, hkv = m->hkv;
  const int32_t group = hq / hkv, dq = hq * 128;
  const int32_t n_qkv = (hq + 2 * hkv) * 128;
  cudaStream_t main = reinterpret_cast<cudaStream_t>(s->stream);
  cudaStream_t side = reinterpret_cast<cudaStream_t>(s->side_stream);
  cudaStream_t side2 = reinterpret_cast<cudaStream_t>(s->side_stream2);
  const bool cascade = s->n_groups > 0;
  const bool overlap = cascade && side != nullptr && m->tmap_q != nullptr;
  StepEvents* ev = nullptr;
  if (overlap && step_events(&ev) != cudaSuccess) return CORTEX_ECUDA;
  int32_t rc = CORTEX_OK;
#define STEP_CALL(expr)              \
  do {                               \
    if ((rc = (expr)) != CORTEX_OK) \
      return rc;                     \
  } while (0)

  for (int32_t l = s->layer_begin; l < s->layer_end; ++l) {
    const int64_t k0 = 2 * static_cast<int64_t>(l) * m->plane_rows;
    const int64_t v0 = k0 + m->plane_rows;
    STEP_CALL(cortex_rmsnorm(m->x, nullptr, T, m->attn_norm[l], d, m->eps, m->xn, s->stream));
    // QKV projection, RoPE + paged KV append in the epilogue
    cortex_rope_epilogue_t epi{m->q, m->cache, k0, v0, m->tok_dst, m->tok_cs, hq, hkv};
    STEP_CALL(cortex_gemm_qkv_rope(m->tmap_wqkv[l], m->tmap_xn, T, n_qkv, d, &epi, m->workspace,
                                   m->workspace_bytes, m->counters, m->n_counters, s->stream));
    auto decode = [&](int32_t parts, cortex_stream_t st) {
      return cortex_paged_decode_attn(
          m->tmap_kv, m->q, m->table, m->table_stride, s->dec_row, s->dec_prefix, s->dec_kvlen,
          nullptr, 0, 0, s->n_dec, hkv, group, k0, v0, m->softmax_scale, s->o_part, s->lse_part,
          s->max_splits, m->attn, s->grp_row, s->grp_plen, s->grp_first, s->grp_count,
          s->n_groups, s->max_group_count, s->prefix_slots, m->tmap_q, parts, st);
    };
    auto prefill = [&](cortex_stream_t st) {
      return cortex_fmha_prefill_tc(m->tmap_kv, m->tmap_q, m->attn, m->table, m->table_stride,
                                    s->pf_row, s->pf_prefix, s->pf_kvlen, s->pf_qstart,
                                    s->pf_qlen, s->n_pf, s->max_qlen, hkv, group, k0, v0,
                                    m->softmax_scale, st);
    };
    bool pf_done = false;
    if (s->n_dec > 0) {
      if (overlap) {
        // tensor-core passes (shared-prefix cascade; the prompt prefill on a second side
        // stream when given) concurrent with the per-call context splits on the main
        // stream; join before the LSE combine (model.py, the same schedule)
        const bool two = side2 != nullptr && s->n_pf > 0;
        if (cudaEventRecord(ev->fork, main) != cudaSuccess ||
            cudaStreamWaitEvent(side, ev->fork, 0) != cudaSuccess ||
            (two && cudaStreamWaitEvent(side2, ev->fork, 0) != cudaSuccess))
          return CORTEX_ECUDA;
        STEP_CALL(decode(1, s->side_stream));
        if (s->n_pf > 0) {
          STEP_CALL(prefill(two ? s->side_stream2 : s->side_stream));
          pf_done = true;
        }
        STEP_CALL(decode(2, s->stream));
        if (cudaEventRecord(ev->join, side) != cudaSuccess ||
            cudaStreamWaitEvent(main, ev->join, 0) != cudaSuccess ||
            (two && (cudaEventRecord(ev->join2, side2) != cudaSuccess ||
                     cudaStreamWaitEvent(main, ev->join2, 0) != cudaSuccess)))
          return CORTEX_ECUDA;
        STEP_CALL(decode(4, s->stream));
      } else {
        STEP_CALL(decode(7, s->stream));
      }
    }
    if (s->n_pf > 0 && !pf_done) STEP_CALL(prefill(s->stream));
    // O projection + residual, MLP norm, gate/up with SwiGLU, down + residual
    STEP_CALL(cortex_gemm_bf16(m->tmap_wo[l], m->tmap_attn, T, d, dq, m->x, d, 1, m->x, d,
                               m->workspace, m->workspace_bytes, m->counters, m->n_counters,
                               s->stream));
    STEP_CALL(cortex_rmsnorm(m->x, nullptr, T, m->mlp_norm[l], d, m->eps, m->xn, s->stream));
    STEP_CALL(cortex_gemm_bf16(m->tmap_wgu[l], m->tmap_xn, T, 2 * m->ffn, d, m->act, m->ffn, 2,
                               nullptr, 0, m->workspace, m->workspace_bytes, m->counters,
                               m->n_counters, s->stream));
    STEP_CALL(cortex_gemm_bf16(m->tmap_wd[l], m->tmap_act, T, d, m->ffn, m->x, d, 1, m->x, d,
                               m->workspace, m->workspace_bytes, m->counters, m->n_counters,
                               s->stream));
  }
#undef STEP_CALL
  return CORTEX_OK;
}

}  // extern "C"
