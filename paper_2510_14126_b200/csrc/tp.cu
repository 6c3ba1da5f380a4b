// Tensor-parallel (TP = 2) exchange of a stage-engine replica over NVLink peer memory.
//
// the only collective on the path is the all-reduce of the fp32
// [T, d] partial outputs of the O and down projections inside one TP = 2 replica
// (BASELINE config 5). Instead of a separate all-reduce followed by the residual
// add and the next RMSNorm, one kernel does all three: every rank reads its own
// partial and the peer's partial straight out of the peer's HBM (one-shot
// all-reduce, d * 4 bytes per token over NVLink), adds both to the residual stream
// in a fixed order (rank 0's partial first, so both ranks hold bit-identical
// residuals), and writes the normalised bf16 input of the next GEMM.
//
// Symmetric buffer (one cudaMalloc per rank, mapped into the peer by CUDA IPC):
//   [0, 256)                  flag words; word 0 is written by the PEER (its epoch)
//   [256, 256 + P)            partial output, parity 0   (P = max_tokens * d * 4)
//   [256 + P, 256 + 2P)       partial output, parity 1
// Protocol per exchange e (1, 2, ...): the GEMM writes parity e & 1 of the local
// buffer; cortex_tp_signal publishes e into the peer's flag word (system-scope
// release after the GEMM completed, stream order); the reduce kernel waits until its
// own flag word reaches e (system-scope acquire) before reading the peer's parity
// e & 1. Two parities are enough: a rank can only start writing parity e & 1 again
// (exchange e + 2) after its reduce of e + 1 saw the peer's signal e + 1, which the
// peer issued after finishing its reduce of e (the last read of that parity).
#include <cstring>

#include "common.cuh"

namespace {

constexpr int kFlagBytes = 256;

CORTEX_DEVICE uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

CORTEX_DEVICE void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

CORTEX_DEVICE uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void tp_signal_kernel(uint32_t* peer_flag, uint32_t epoch) {
  __threadfence_system();
  st_release_sys(peer_flag, epoch);
}

// One CTA per token row. x[r] += y0[r] + y1[r]; if w: out[r] = bf16(norm(x[r]) * w).
__global__ void tp_allreduce_rmsnorm_kernel(const float* y0, const float* y1,
                                            float* __restrict__ x,
                                            const __nv_bfloat16* __restrict__ w, int d, float eps,
                                            __nv_bfloat16* __restrict__ out, const uint32_t* flag,
                                            uint32_t epoch, int32_t* status) {
  __shared__ float red[32];
  __shared__ int timed_out;
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0) {
    timed_out = 0;
    if (flag) {
      const uint64_t t0 = globaltimer_ns();
      while (static_cast<int32_t>(ld_acquire_sys(flag) - epoch) < 0) {
        if (globaltimer_ns() - t0 > 10ull * 1000 * 1000 * 1000) {  // peer gone: 10 s
          timed_out = 1;
          if (status) atomicExch(status, CORTEX_ETIMEOUT);
          break;
        }
        __nanosleep(64);
      }
    }
  }
  __syncthreads();
  if (timed_out) return;
  const int r = blockIdx.x;
  const int64_t off = static_cast<int64_t>(r) * d;
  const float4* a = reinterpret_cast<const float4*>(y0 + off);
  const float4* b = reinterpret_cast<const float4*>(y1 + off);
  float4* xr = reinterpret_cast<float4*>(x + off);
  const int nvec = d / 4;
  // d <= 4 * 8 * blockDim: up to 8 float4 per thread in registers
  float4 v[8];
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int i = threadIdx.x + k * blockDim.x;
    if (i < nvec) {
      // peer memory: volatile loads (no stale L1 lines from an earlier exchange)
      const float4 p = __ldcv(a + i), q = __ldcv(b + i);
      float4 s = xr[i];
      s.x += p.x + q.x;
      s.y += p.y + q.y;
      s.z += p.z + q.z;
      s.w += p.w + q.w;
      xr[i] = s;
      v[k] = s;
      ss += s.x * s.x + s.y * s.y + s.z * s.z + s.w * s.w;
    }
  }
  if (!w) return;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if (lane_id() == 0) red[warp_id()] = ss;
  __syncthreads();
  float tot = 0.f;
  for (int i = 0; i < static_cast<int>(blockDim.x / 32); ++i) tot += red[i];
  const float rstd = rsqrtf(tot / static_cast<float>(d) + eps);
  const __nv_bfloat162* w2 = reinterpret_cast<const __nv_bfloat162*>(w);
  __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(out + off);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int i = threadIdx.x + k * blockDim.x;
    if (i < nvec) {
      const float2 w01 = __bfloat1622float2(w2[2 * i]);
      const float2 w23 = __bfloat1622float2(w2[2 * i + 1]);
      o2[2 * i] = __floats2bfloat162_rn(v[k].x * rstd * w01.x, v[k].y * rstd * w01.y);
      o2[2 * i + 1] = __floats2bfloat162_rn(v[k].z * rstd * w23.x, v[k].w * rstd * w23.y);
    }
  }
}

}  // namespace

extern "C" {

int32_t cortex_sym_alloc(uint64_t bytes, void** out_ptr) {
  if (!out_ptr || bytes == 0) return CORTEX_EBADARG;
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) return CORTEX_ECUDA;
  if (cudaMemset(p, 0, bytes) != cudaSuccess) {
    cudaFree(p);
    return CORTEX_ECUDA;
  }
  *out_ptr = p;
  return CORTEX_OK;
}

int32_t cortex_sym_free(void* ptr) {
  if (!ptr) return CORTEX_EBADARG;
  return cudaFree(ptr) == cudaSuccess ? CORTEX_OK : CORTEX_ECUDA;
}

int32_t cortex_ipc_get_handle(void* ptr, void* handle_out) {
  if (!ptr || !handle_out) return CORTEX_EBADARG;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, ptr) != cudaSuccess) return CORTEX_ECUDA;
  memcpy(handle_out, &h, sizeof(h));
  return CORTEX_OK;
}

int32_t cortex_ipc_open_handle(const void* handle, void** out_ptr) {
  if (!handle || !out_ptr) return CORTEX_EBADARG;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void* p = nullptr;
  if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
    return CORTEX_ECUDA;
  *out_ptr = p;
  return CORTEX_OK;
}

int32_t cortex_ipc_close(void* ptr) {
  if (!ptr) return CORTEX_EBADARG;
  return cudaIpcCloseMemHandle(ptr) == cudaSuccess ? CORTEX_OK : CORTEX_ECUDA;
}

int32_t cortex_tp_signal(uint32_t* peer_flag, uint32_t epoch, cudaStream_t stream) {
  if (!peer_flag) return CORTEX_EBADARG;
  // a plain (non-PDL) launch: the signal must follow the partial GEMM's completion
  tp_signal_kernel<<<1, 1, 0, stream>>>(peer_flag, epoch);
  CORTEX_CHECK_LAUNCH();
  return CORTEX_OK;
}

int32_t cortex_tp_allreduce_rmsnorm(const float* y0, const float* y1, float* x, int32_t n_rows,
                                    int32_t d, const void* w, float eps, void* out,
                                    const uint32_t* flag, uint32_t epoch, int32_t* status,
                                    cudaStream_t stream) {
  if (!y0 || !y1 || !x || n_rows < 0 || d % 4 || d > 4 * 8 * 1024 || (w && !out))
    return CORTEX_EBADARG;
  if (n_rows == 0) return CORTEX_OK;
  int threads = 64;
  while (threads * 4 * 8 < d) threads *= 2;
  if (pdl_launch(tp_allreduce_rmsnorm_kernel, n_rows, threads, 0, stream, 1, y0, y1, x,
                 reinterpret_cast<const __nv_bfloat16*>(w), d, eps,
                 reinterpret_cast<__nv_bfloat16*>(out), flag, epoch, status) != cudaSuccess)
    return CORTEX_ECUDA;
  return CORTEX_OK;
}

int32_t cortex_tp_flag_bytes(void) { return kFlagBytes; }

}  // extern "C"
