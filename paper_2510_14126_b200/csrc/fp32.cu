// fp32 decoder step for the tiny config-1 model (BASELINE configs[0]: "tiny random-init
// decoder (4L, d=256)"), where the north star's parity bar is "1e-5 in fp32, greedy
// tokens identical". Storage AND arithmetic are fp32 end to end (weights, residual
// stream, activations, paged KV cache, logits), so the GPU and the CPU fp32 oracle
// (oracle/decoder_ref.py, exact mode) differ only by summation order.
//
// The shapes are tiny (d 256, FFN 768, vocab 1024), so these are plain SIMT kernels:
//   * f32_gemm_kernel      C = X W^T (+ residual | SwiGLU of the gate / up row pair),
//                          64 x 64 output tile per CTA, K staged through shared memory
//                          in 32-wide chunks, 4 x 4 outputs per thread, k summed in order;
//   * f32_rmsnorm_kernel   (optionally gathering rows), fp32 in and out;
//   * f32_rope_kv_kernel   RoPE of q / k and the paged KV append (same block-table
//                          addressing as the bf16 path, 128-wide fp32 rows);
//   * f32_attn_kernel      one warp per (token, q head): causal attention over the
//                          token's row of the block table (stage-prefix blocks, then the
//                          private blocks at positions P, P + 1, ...), online softmax,
//                          keys in position order, each lane owning 4 of the 128 dims;
//   * f32_embed_kernel.
// The bf16 path's allocator, block tables and greedy argmax are shared.
#include "common.cuh"

namespace {

constexpr int kHD = 128;
constexpr int kBlk = 16;

// ---------------------------------------------------------------- GEMM
// mode 0: out = X W^T; 1: out = X W^T + residual (out may alias residual);
// 2: SwiGLU, N = F outputs, out[m, j] = silu(x . W[j]) * (x . W[F + j]).
constexpr int kTM = 64, kTN = 64, kTK = 32;

template <int NW>
__global__ void __launch_bounds__(256) f32_gemm_kernel(const float* __restrict__ X, int ldx,
                                                       const float* __restrict__ W, int M, int N,
                                                       int K, float* out, int ldo,
                                                       const float* residual, int ldr, int mode) {
  pdl_wait();
  pdl_trigger();
  __shared__ float xs[kTK][kTM + 1];
  __shared__ float ws[NW][kTK][kTN + 1];
  const int m0 = blockIdx.y * kTM, n0 = blockIdx.x * kTN;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  constexpr int nw = NW;
  float acc[NW][4][4] = {};
  for (int k0 = 0; k0 < K; k0 += kTK) {
    for (int i = threadIdx.x; i < kTM * kTK; i += 256) {
      const int r = i / kTK, c = i % kTK;
      const int m = m0 + r, k = k0 + c;
      xs[c][r] = (m < M && k < K) ? X[static_cast<int64_t>(m) * ldx + k] : 0.f;
    }
#pragma unroll
    for (int w = 0; w < nw; ++w)
      for (int i = threadIdx.x; i < kTN * kTK; i += 256) {
        const int r = i / kTK, c = i % kTK;
        const int n = n0 + r, k = k0 + c;
        ws[w][c][r] = (n < N && k < K) ? W[static_cast<int64_t>(n + w * N) * K + k] : 0.f;
      }
    __syncthreads();
    for (int kk = 0; kk < kTK; ++kk) {
      float a[4], b[NW][4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = xs[kk][ty + 16 * i];
#pragma unroll
      for (int w = 0; w < nw; ++w)
#pragma unroll
        for (int j = 0; j < 4; ++j) b[w][j] = ws[w][kk][tx + 16 * j];
#pragma unroll
      for (int w = 0; w < nw; ++w)
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[w][i][j] = fmaf(a[i], b[w][j], acc[w][i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty + 16 * i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx + 16 * j;
      if (n >= N) continue;
      float v = acc[0][i][j];
      if (mode == 1) v += residual[static_cast<int64_t>(m) * ldr + n];
      if constexpr (NW == 2) v = v / (1.f + expf(-v)) * acc[NW - 1][i][j];
      out[static_cast<int64_t>(m) * ldo + n] = v;
    }
  }
}

// ---------------------------------------------------------------- row ops
__global__ void f32_embed_kernel(const float* __restrict__ emb, const int* __restrict__ tokens,
                                 const int* __restrict__ index, int d, float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int t = blockIdx.x;
  const int tok = tokens[index ? index[t] : t];
  for (int i = threadIdx.x; i < d; i += blockDim.x)
    out[static_cast<int64_t>(t) * d + i] = emb[static_cast<int64_t>(tok) * d + i];
}

__global__ void f32_rmsnorm_kernel(const float* __restrict__ x, const int* __restrict__ rows,
                                   const float* __restrict__ w, int d, float eps,
                                   float* __restrict__ y) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[32];
  const int r = blockIdx.x;
  const float* xr = x + static_cast<int64_t>(rows ? rows[r] : r) * d;
  float ss = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) ss = fmaf(xr[i], xr[i], ss);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if (lane_id() == 0) red[warp_id()] = ss;
  __syncthreads();
  float tot = 0.f;
  for (int i = 0; i < static_cast<int>(blockDim.x / 32); ++i) tot += red[i];
  const float rstd = rsqrtf(tot / static_cast<float>(d) + eps);
  for (int i = threadIdx.x; i < d; i += blockDim.x)
    y[static_cast<int64_t>(r) * d + i] = xr[i] * rstd * w[i];
}

struct F32RopeArgs {
  const float* qkv;  // [T, (hq + 2 hkv) * 128]
  float* q_out;      // [T, hq, 128]
  float* cache;      // base of the fp32 KV allocation (128-wide rows)
  int64_t k_row0, v_row0;
  const int* table;
  int table_stride;
  const int *tok_pos, *tok_row, *tok_col, *tok_off;
  const float *cos_tab, *sin_tab;
  int hq, hkv;
};

__global__ void f32_rope_kv_kernel(const F32RopeArgs a) {
  pdl_wait();
  pdl_trigger();
  const int t = blockIdx.x;
  const int pos = a.tok_pos[t];
  const float* src = a.qkv + static_cast<int64_t>(t) * (a.hq + 2 * a.hkv) * kHD;
  const float* ct = a.cos_tab + static_cast<int64_t>(pos) * 64;
  const float* st = a.sin_tab + static_cast<int64_t>(pos) * 64;
  const int block = a.table[static_cast<int64_t>(a.tok_row[t]) * a.table_stride + a.tok_col[t]];
  const int off = a.tok_off[t];
  for (int item = threadIdx.x; item < (a.hq + a.hkv) * 64; item += blockDim.x) {
    const int h = item / 64, i = item % 64;
    const float x0 = src[h * kHD + i], x1 = src[h * kHD + 64 + i];
    const float y0 = x0 * ct[i] - x1 * st[i];
    const float y1 = x1 * ct[i] + x0 * st[i];
    float* dst = h < a.hq
                     ? a.q_out + (static_cast<int64_t>(t) * a.hq + h) * kHD
                     : a.cache + (a.k_row0 + (static_cast<int64_t>(block) * a.hkv + (h - a.hq)) *
                                                 kBlk + off) * kHD;
    dst[i] = y0;
    dst[64 + i] = y1;
  }
  for (int item = threadIdx.x; item < a.hkv * kHD; item += blockDim.x) {
    const int kh = item / kHD, e = item % kHD;
    a.cache[(a.v_row0 + (static_cast<int64_t>(block) * a.hkv + kh) * kBlk + off) * kHD + e] =
        src[(a.hq + a.hkv + kh) * kHD + e];
  }
}

// ---------------------------------------------------------------- attention
struct F32AttnArgs {
  const float* q;    // [T, hq, 128] (rotated)
  const float* cache;
  int64_t k_row0, v_row0;
  const int* table;
  int table_stride;
  const int* tok_row;     // [T] block-table row of the token's sequence
  const int* tok_prefix;  // [T] tokens of the row's stage-prefix segment
  const int* tok_pos;     // [T] logical position; keys 0..pos
  float* out;             // [T, hq, 128]
  int T, hq, hkv;
  float scale;
};

__global__ void f32_attn_kernel(const F32AttnArgs a) {
  pdl_wait();
  pdl_trigger();
  const int item = blockIdx.x * (blockDim.x / 32) + warp_id();
  if (item >= a.T * a.hq) return;
  const int t = item / a.hq, h = item % a.hq;
  const int kh = h / (a.hq / a.hkv);
  const int lane = lane_id();
  const float4 q = reinterpret_cast<const float4*>(a.q + static_cast<int64_t>(item) * kHD)[lane];
  const int* trow = a.table + static_cast<int64_t>(a.tok_row[t]) * a.table_stride;
  const int P = a.tok_prefix[t];
  const int npb = (P + kBlk - 1) / kBlk;
  const int pos = a.tok_pos[t];
  float m = -INFINITY, l = 0.f;
  float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int j = 0; j <= pos; ++j) {
    int col, off;
    if (j < P) {
      col = j / kBlk;
      off = j % kBlk;
    } else {
      col = npb + (j - P) / kBlk;
      off = (j - P) % kBlk;
    }
    const int64_t r = (static_cast<int64_t>(trow[col]) * a.hkv + kh) * kBlk + off;
    const float4 k = reinterpret_cast<const float4*>(a.cache + (a.k_row0 + r) * kHD)[lane];
    float s = q.x * k.x + q.y * k.y + q.z * k.z + q.w * k.w;
#pragma unroll
    for (int sh = 16; sh > 0; sh >>= 1) s += __shfl_xor_sync(0xffffffffu, s, sh);
    s *= a.scale;
    const float m_new = fmaxf(m, s);
    const float corr = expf(m - m_new);  // exp(-inf) = 0 on the first key
    const float p = expf(s - m_new);
    const float4 v = reinterpret_cast<const float4*>(a.cache + (a.v_row0 + r) * kHD)[lane];
    l = l * corr + p;
    o.x = o.x * corr + p * v.x;
    o.y = o.y * corr + p * v.y;
    o.z = o.z * corr + p * v.z;
    o.w = o.w * corr + p * v.w;
    m = m_new;
  }
  const float inv = 1.f / l;
  reinterpret_cast<float4*>(a.out + static_cast<int64_t>(item) * kHD)[lane] =
      make_float4(o.x * inv, o.y * inv, o.z * inv, o.w * inv);
}

}  // namespace

extern "C" {

int32_t cortex_f32_gemm(const float* x, int32_t ldx, const float* w, int32_t M, int32_t N,
                        int32_t K, float* out, int32_t ldo, const float* residual, int32_t ldr,
                        int32_t mode, cudaStream_t stream) {
  if (!x || !w || !out || M < 0 || N < 1 || K < 1 || mode < 0 || mode > 2 ||
      (mode == 1 && !residual))
    return CORTEX_EBADARG;
  if (M == 0) return CORTEX_OK;
  const dim3 grid((N + kTN - 1) / kTN, (M + kTM - 1) / kTM);
  const cudaError_t e =
      mode == 2 ? pdl_launch(f32_gemm_kernel<2>, grid, 256, 0, stream, 1, x, ldx, w, M, N, K,
                             out, ldo, residual, ldr, mode)
                : pdl_launch(f32_gemm_kernel<1>, grid, 256, 0, stream, 1, x, ldx, w, M, N, K,
                             out, ldo, residual, ldr, mode);
  if (e != cudaSuccess) return CORTEX_ECUDA;
  return CORTEX_OK;
}

int32_t cortex_f32_embed(const float* emb, const int32_t* tokens, const int32_t* index,
                         int32_t n_tok, int32_t d, float* out, cudaStream_t stream) {
  if (!emb || !tokens || !out || n_tok < 0 || d < 1) return CORTEX_EBADARG;
  if (n_tok == 0) return CORTEX_OK;
  if (pdl_launch(f32_embed_kernel, n_tok, 128, 0, stream, 1, emb, tokens, index, d, out) !=
      cudaSuccess)
    return CORTEX_ECUDA;
  return CORTEX_OK;
}

int32_t cortex_f32_rmsnorm(const float* x, const int32_t* rows, int32_t n_rows, const float* w,
                           int32_t d, float eps, float* y, cudaStream_t stream) {
  if (!x || !w || !y || n_rows < 0 || d < 1) return CORTEX_EBADARG;
  if (n_rows == 0) return CORTEX_OK;
  if (pdl_launch(f32_rmsnorm_kernel, n_rows, 256, 0, stream, 1, x, rows, w, d, eps, y) !=
      cudaSuccess)
    return CORTEX_ECUDA;
  return CORTEX_OK;
}

int32_t cortex_f32_rope_kv_append(const float* qkv, float* q_out, float* cache, int64_t k_row0,
                                  int64_t v_row0, const int32_t* table, int32_t table_stride,
                                  const int32_t* tok_pos, const int32_t* tok_row,
                                  const int32_t* tok_col, const int32_t* tok_off,
                                  const float* cos_tab, const float* sin_tab, int32_t n_tok,
                                  int32_t hq, int32_t hkv, cudaStream_t stream) {
  if (!qkv || !q_out || !cache || !table || !tok_pos || !tok_row || !tok_col || !tok_off ||
      !cos_tab || !sin_tab || n_tok < 0 || hq < 1 || hkv < 1 || hq % hkv)
    return CORTEX_EBADARG;
  if (n_tok == 0) return CORTEX_OK;
  const F32RopeArgs a{qkv, q_out, cache, k_row0, v_row0, table, table_stride, tok_pos, tok_row,
                      tok_col, tok_off, cos_tab, sin_tab, hq, hkv};
  if (pdl_launch(f32_rope_kv_kernel, n_tok, 256, 0, stream, 1, a) != cudaSuccess)
    return CORTEX_ECUDA;
  return CORTEX_OK;
}

int32_t cortex_f32_attention(const float* q, const float* cache, int64_t k_row0, int64_t v_row0,
                             const int32_t* table, int32_t table_stride, const int32_t* tok_row,
                             const int32_t* tok_prefix, const int32_t* tok_pos, int32_t n_tok,
                             int32_t hq, int32_t hkv, float scale, float* out,
                             cudaStream_t stream) {
  if (!q || !cache || !table || !tok_row || !tok_prefix || !tok_pos || !out || n_tok < 0 ||
      hq < 1 || hkv < 1 || hq % hkv)
    return CORTEX_EBADARG;
  if (n_tok == 0) return CORTEX_OK;
  const F32AttnArgs a{q, cache, k_row0, v_row0, table, table_stride, tok_row, tok_prefix,
                      tok_pos, out, n_tok, hq, hkv, scale};
  const int warps = 8;
  const int grid = (n_tok * hq + warps - 1) / warps;
  if (pdl_launch(f32_attn_kernel, grid, 32 * warps, 0, stream, 1, a) != cudaSuccess)
    return CORTEX_ECUDA;
  return CORTEX_OK;
}

}  // extern "C"
