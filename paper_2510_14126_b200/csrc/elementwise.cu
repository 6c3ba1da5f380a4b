// Row-wise and element-wise pieces of the decoder step: embedding gather,
// RMSNorm (optionally gathering rows), RoPE + paged KV append, and the
// greedy argmax over the vocabulary. All are HBM-bound SIMT kernels with 16-byte
// vector accesses; arithmetic is fp32, storage bf16.
#include "common.cuh"

namespace {

constexpr int kHeadDim = 128;
constexpr int kTile = 16;

struct alignas(16) bf16x8 {
  __nv_bfloat162 v[4];
};

CORTEX_DEVICE void unpack8(const bf16x8& x, float (&f)[8]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __bfloat1622float2(x.v[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

CORTEX_DEVICE bf16x8 pack8(const float (&f)[8]) {
  bf16x8 x;
#pragma unroll
  for (int i = 0; i < 4; ++i) x.v[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return x;
}

// out[t] = float(emb[tok]), tok = tokens[index ? index[t] : t]  (fp32 residual stream)
__global__ void embed_kernel(const __nv_bfloat16* __restrict__ emb, const int* __restrict__ tokens,
                             const int* __restrict__ index, int d, float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int t = blockIdx.x;
  const int tok = tokens[index ? index[t] : t];
  const bf16x8* src = reinterpret_cast<const bf16x8*>(emb + static_cast<int64_t>(tok) * d);
  float4* dst = reinterpret_cast<float4*>(out + static_cast<int64_t>(t) * d);
  for (int i = threadIdx.x; i < d / 8; i += blockDim.x) {
    float f[8];
    unpack8(src[i], f);
    dst[2 * i] = make_float4(f[0], f[1], f[2], f[3]);
    dst[2 * i + 1] = make_float4(f[4], f[5], f[6], f[7]);
  }
}

CORTEX_DEVICE float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int nw = blockDim.x / 32;
  if (lane_id() == 0) red[warp_id()] = v;
  __syncthreads();
  float s = 0.f;
  for (int i = 0; i < nw; ++i) s += red[i];
  __syncthreads();
  return s;
}

// y[r] = bf16(x[src] * rsqrt(mean(x[src]^2) + eps) * w), src = rows ? rows[r] : r
__global__ void rmsnorm_kernel(const float* __restrict__ x, const int* __restrict__ rows,
                               const __nv_bfloat16* __restrict__ w, int d, float eps,
                               __nv_bfloat16* __restrict__ y) {
  // the (immutable) norm weights load before the PDL wait, under the predecessor's tail
  const bf16x8* wr = reinterpret_cast<const bf16x8*>(w);
  const int nvec = d / 8;
  bf16x8 wv[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int i = threadIdx.x + k * blockDim.x;
    if (i < nvec) wv[k] = wr[i];
  }
  pdl_wait();
  pdl_trigger();
  __shared__ float red[32];
  const int r = blockIdx.x;
  const int src = rows ? rows[r] : r;
  const float4* xr = reinterpret_cast<const float4*>(x + static_cast<int64_t>(src) * d);
  bf16x8* yr = reinterpret_cast<bf16x8*>(y + static_cast<int64_t>(r) * d);
  // d <= 8 * 4 * blockDim: keep up to 4 vectors per thread in registers
  float f[4][8];
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int i = threadIdx.x + k * blockDim.x;
    if (i < nvec) {
      const float4 a = xr[2 * i], b = xr[2 * i + 1];
      f[k][0] = a.x; f[k][1] = a.y; f[k][2] = a.z; f[k][3] = a.w;
      f[k][4] = b.x; f[k][5] = b.y; f[k][6] = b.z; f[k][7] = b.w;
#pragma unroll
      for (int e = 0; e < 8; ++e) ss += f[k][e] * f[k][e];
    }
  }
  const float tot = block_sum(ss, red);
  const float rstd = rsqrtf(tot / static_cast<float>(d) + eps);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int i = threadIdx.x + k * blockDim.x;
    if (i < nvec) {
      float wf[8], o[8];
      unpack8(wv[k], wf);
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = f[k][e] * rstd * wf[e];
      yr[i] = pack8(o);
    }
  }
}

// RoPE (rotate-half, pairs (i, i+64)) on q and k of each token, q -> q_out,
// k and v -> paged cache row of (table[row][col], kv_head, off).
struct RopeArgs {
  const __nv_bfloat16* qkv;  // [T, (Hq + 2 Hkv) * 128]
  __nv_bfloat16* q_out;      // [T, Hq, 128]
  __nv_bfloat16* cache;      // base of the whole KV allocation (128-wide rows)
  int64_t k_row0, v_row0;
  const int* table;
  int table_stride;
  const int* tok_pos;  // [T] logical position (rope angle)
  const int* tok_row;  // [T] block-table row
  const int* tok_col;  // [T] block index within the row
  const int* tok_off;  // [T] token offset inside the block
  const float* cos_tab;  // [max_pos, 64]
  const float* sin_tab;
  int hq, hkv;
};

__global__ void rope_kv_append_kernel(const RopeArgs a) {
  pdl_wait();
  pdl_trigger();
  const int t = blockIdx.x;
  const int pos = a.tok_pos[t];
  const int ldq = (a.hq + 2 * a.hkv) * kHeadDim;
  const __nv_bfloat16* src = a.qkv + static_cast<int64_t>(t) * ldq;
  const float* ct = a.cos_tab + static_cast<int64_t>(pos) * 64;
  const float* st = a.sin_tab + static_cast<int64_t>(pos) * 64;
  const int block = a.table[static_cast<int64_t>(a.tok_row[t]) * a.table_stride + a.tok_col[t]];
  const int off = a.tok_off[t];
  // rotate q and k heads: work item = (head, 8 consecutive pairs (i, i + 64)), 16-byte
  // loads and stores of both halves, cos / sin as float4
  const int n_rot = (a.hq + a.hkv) * 8;
  for (int item = threadIdx.x; item < n_rot; item += blockDim.x) {
    const int h = item >> 3;
    const int i0 = (item & 7) * 8;
    const __nv_bfloat16* xh = src + h * kHeadDim;
    float x0[8], x1[8], c[8], sn[8], y0[8], y1[8];
    unpack8(*reinterpret_cast<const bf16x8*>(xh + i0), x0);
    unpack8(*reinterpret_cast<const bf16x8*>(xh + 64 + i0), x1);
    *reinterpret_cast<float4*>(c) = *reinterpret_cast<const float4*>(ct + i0);
    *reinterpret_cast<float4*>(c + 4) = *reinterpret_cast<const float4*>(ct + i0 + 4);
    *reinterpret_cast<float4*>(sn) = *reinterpret_cast<const float4*>(st + i0);
    *reinterpret_cast<float4*>(sn + 4) = *reinterpret_cast<const float4*>(st + i0 + 4);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      y0[e] = x0[e] * c[e] - x1[e] * sn[e];
      y1[e] = x1[e] * c[e] + x0[e] * sn[e];
    }
    __nv_bfloat16* dst;
    if (h < a.hq) {
      dst = a.q_out + (static_cast<int64_t>(t) * a.hq + h) * kHeadDim;
    } else {
      const int kh = h - a.hq;
      dst = a.cache + (a.k_row0 + (static_cast<int64_t>(block) * a.hkv + kh) * kTile + off) * kHeadDim;
    }
    *reinterpret_cast<bf16x8*>(dst + i0) = pack8(y0);
    *reinterpret_cast<bf16x8*>(dst + 64 + i0) = pack8(y1);
  }
  // v: straight copy, 8 elements per item
  const int n_v = a.hkv * kHeadDim / 8;
  for (int item = threadIdx.x; item < n_v; item += blockDim.x) {
    const int kh = item / (kHeadDim / 8);
    const int e = item % (kHeadDim / 8);
    const bf16x8* vs =
        reinterpret_cast<const bf16x8*>(src + (a.hq + a.hkv + kh) * kHeadDim) + e;
    bf16x8* vd = reinterpret_cast<bf16x8*>(
                     a.cache + (a.v_row0 + (static_cast<int64_t>(block) * a.hkv + kh) * kTile + off) *
                                   kHeadDim) +
                 e;
    *vd = *vs;
  }
}

// Greedy token per row (first index of the maximum). Optionally scatters the token
// into slot_tok[slot[r]] and hist[slot[r] * hist_stride + hist_pos[r]].
__global__ void argmax_kernel(const float* __restrict__ logits, int64_t ld, int vocab,
                              int* __restrict__ out_tok, const int* __restrict__ slot,
                              int* __restrict__ slot_tok, int* __restrict__ hist,
                              int hist_stride, const int* __restrict__ hist_pos) {
  pdl_wait();
  pdl_trigger();
  __shared__ float sv[32];
  __shared__ int si[32];
  const int r = blockIdx.x;
  const float* row = logits + r * ld;
  // NaN never compares greater, so a row of NaN logits yields index 0 (a valid token id
  // for the embedding lookup of the next step) rather than an out-of-range sentinel
  float best = -INFINITY;
  int bi = vocab;
  auto take = [&](float v, int i) {
    if (v > best) {  // strictly greater: keeps the first index within a thread
      best = v;
      bi = i;
    }
  };
  // 16-byte loads, 4 in flight per thread (a scalar loop keeps one 4-byte load in flight
  // per thread: ~1.6 TB/s over the 128K-entry rows); indices stay increasing per thread
  const bool vec = (reinterpret_cast<uintptr_t>(row) & 15) == 0;
  const int n4 = vec ? vocab / 4 : 0;
  const float4* row4 = reinterpret_cast<const float4*>(row);
  int i4 = threadIdx.x;
  for (; i4 + 3 * static_cast<int>(blockDim.x) < n4; i4 += 4 * blockDim.x) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldcs(row4 + i4 + u * blockDim.x);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = 4 * (i4 + u * blockDim.x);
      take(v[u].x, i);
      take(v[u].y, i + 1);
      take(v[u].z, i + 2);
      take(v[u].w, i + 3);
    }
  }
  for (; i4 < n4; i4 += blockDim.x) {
    const float4 v = __ldcs(row4 + i4);
    take(v.x, 4 * i4);
    take(v.y, 4 * i4 + 1);
    take(v.z, 4 * i4 + 2);
    take(v.w, 4 * i4 + 3);
  }
  for (int i = 4 * n4 + threadIdx.x; i < vocab; i += blockDim.x) take(row[i], i);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) {
      best = ov;
      bi = oi;
    }
  }
  if (lane_id() == 0) {
    sv[warp_id()] = best;
    si[warp_id()] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < static_cast<int>(blockDim.x / 32); ++w) {
      if (sv[w] > best || (sv[w] == best && si[w] < bi)) {
        best = sv[w];
        bi = si[w];
      }
    }
    if (bi >= vocab) bi = 0;  // no finite logit in the row
    if (out_tok) out_tok[r] = bi;
    if (slot) {
      const int s = slot[r];
      if (slot_tok) slot_tok[s] = bi;
      if (hist) hist[static_cast<int64_t>(s) * hist_stride + hist_pos[r]] = bi;
    }
  }
}

// Per-token operands of the QKV GEMM's RoPE epilogue, once per step (shared by every
// layer): the token's K / V row within a plane and cos | sin at its position.
__global__ void rope_token_prep_kernel(const int* __restrict__ table, int table_stride,
                                       const int* __restrict__ tok_pos,
                                       const int* __restrict__ tok_row,
                                       const int* __restrict__ tok_col,
                                       const int* __restrict__ tok_off,
                                       const float* __restrict__ cos_tab,
                                       const float* __restrict__ sin_tab, int n_tok, int hkv,
                                       int* __restrict__ tok_dst, float* __restrict__ tok_cs) {
  pdl_wait();
  pdl_trigger();
  const int t = blockIdx.x * (blockDim.x / 32) + warp_id();
  if (t >= n_tok) return;
  const int lane = lane_id();
  const int pos = tok_pos[t];
  // 128 floats: lanes 0-15 copy cos, 16-31 sin, float4 each
  const float* src = lane < 16 ? cos_tab + static_cast<int64_t>(pos) * 64 + 4 * lane
                               : sin_tab + static_cast<int64_t>(pos) * 64 + 4 * (lane - 16);
  reinterpret_cast<float4*>(tok_cs + static_cast<int64_t>(t) * 128)[lane] =
      *reinterpret_cast<const float4*>(src);
  if (lane == 0) {
    const int block = table[static_cast<int64_t>(tok_row[t]) * table_stride + tok_col[t]];
    tok_dst[t] = (block * hkv) * 16 + tok_off[t];
  }
}

// Greedy token per row from the lm_head GEMM's per-128-column partials (out mode 3):
// (max, first index) over the row's n_chunks partials, chunk order = column order, so
// the result is the first index of the row maximum, exactly argmax_kernel's.
__global__ void argmax_partials_kernel(const float2* __restrict__ part, int n_chunks,
                                       int* __restrict__ out_tok, const int* __restrict__ slot,
                                       int* __restrict__ slot_tok, int* __restrict__ hist,
                                       int hist_stride, const int* __restrict__ hist_pos) {
  pdl_wait();
  pdl_trigger();
  __shared__ float sv[32];
  __shared__ int si[32];
  const int r = blockIdx.x;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  for (int c = threadIdx.x; c < n_chunks; c += blockDim.x) {
    const float2 p = part[static_cast<size_t>(r) * n_chunks + c];
    const int i = __float_as_int(p.y);
    if (p.x > best || (p.x == best && i < bi)) {
      best = p.x;
      bi = i;
    }
  }
  warp_argmax(best, bi);
  if (lane_id() == 0) {
    sv[warp_id()] = best;
    si[warp_id()] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < static_cast<int>(blockDim.x / 32); ++w) {
      if (sv[w] > best || (sv[w] == best && si[w] < bi)) {
        best = sv[w];
        bi = si[w];
      }
    }
    if (bi == 0x7fffffff) bi = 0;  // no finite logit in the row (argmax_kernel's rule)
    if (out_tok) out_tok[r] = bi;
    if (slot) {
      const int s = slot[r];
      if (slot_tok) slot_tok[s] = bi;
      if (hist) hist[static_cast<int64_t>(s) * hist_stride + hist_pos[r]] = bi;
    }
  }
}

}  // namespace

extern "C" {

int32_t cortex_embed(const void* emb, const int32_t* tokens, const int32_t* index, int32_t n_tok,
                     int32_t d, void* out, cudaStream_t stream) {
  if (!emb || !tokens || !out || n_tok < 0 || d % 8) return CORTEX_EBADARG;
  if (n_tok == 0) return CORTEX_OK;
  if (pdl_launch(embed_kernel, n_tok, 128, 0, stream, 1,
                 reinterpret_cast<const __nv_bfloat16*>(emb), tokens, index, d,
                 reinterpret_cast<float*>(out)) != cudaSuccess)
    return CORTEX_ECUDA;
  return CORTEX_OK;
}

int32_t cortex_rmsnorm(const void* x, const int32_t* rows, int32_t n_rows, const void* w,
                       int32_t d, float eps, void* y, cudaStream_t stream) {
  if (!x || !w || !y || n_rows < 0 || d % 8 || d > 8 * 4 * 512) return CORTEX_EBADARG;
  if (n_rows == 0) return CORTEX_OK;
  int threads = 32;
  while (threads * 8 * 4 < d) threads *= 2;
  if (threads < 64) threads = 64;
  if (pdl_launch(rmsnorm_kernel, n_rows, threads, 0, stream, 1,
                 reinterpret_cast<const float*>(x), rows,
                 reinterpret_cast<const __nv_bfloat16*>(w), d, eps,
                 reinterpret_cast<__nv_bfloat16*>(y)) != cudaSuccess)
    return CORTEX_ECUDA;
  return CORTEX_OK;
}

int32_t cortex_rope_kv_append(const void* qkv, void* q_out, void* cache, int64_t k_row0,
                              int64_t v_row0, const int32_t* table, int32_t table_stride,
                              const int32_t* tok_pos, const int32_t* tok_row,
                              const int32_t* tok_col, const int32_t* tok_off,
                              const float* cos_tab, const float* sin_tab, int32_t n_tok,
                              int32_t hq, int32_t hkv, cudaStream_t stream) {
  if (!qkv || !q_out || !cache || !table || !tok_pos || !tok_row || !tok_col || !tok_off ||
      !cos_tab || !sin_tab || n_tok < 0 || hq < 1 || hkv < 1)
    return CORTEX_EBADARG;
  if (n_tok == 0) return CORTEX_OK;
  RopeArgs a{};
  a.qkv = reinterpret_cast<const __nv_bfloat16*>(qkv);
  a.q_out = reinterpret_cast<__nv_bfloat16*>(q_out);
  a.cache = reinterpret_cast<__nv_bfloat16*>(cache);
  a.k_row0 = k_row0;
  a.v_row0 = v_row0;
  a.table = table;
  a.table_stride = table_stride;
  a.tok_pos = tok_pos;
  a.tok_row = tok_row;
  a.tok_col = tok_col;
  a.tok_off = tok_off;
  a.cos_tab = cos_tab;
  a.sin_tab = sin_tab;
  a.hq = hq;
  a.hkv = hkv;
  if (pdl_launch(rope_kv_append_kernel, n_tok, 256, 0, stream, 1, a) != cudaSuccess)
    return CORTEX_ECUDA;
  return CORTEX_OK;
}

int32_t cortex_rope_token_prep(const int32_t* table, int32_t table_stride, const int32_t* tok_pos,
                               const int32_t* tok_row, const int32_t* tok_col,
                               const int32_t* tok_off, const float* cos_tab, const float* sin_tab,
                               int32_t n_tok, int32_t hkv, int32_t* tok_dst, float* tok_cs,
                               cudaStream_t stream) {
  if (!table || !tok_pos || !tok_row || !tok_col || !tok_off || !cos_tab || !sin_tab ||
      !tok_dst || !tok_cs || n_tok < 0 || hkv < 1)
    return CORTEX_EBADARG;
  if (n_tok == 0) return CORTEX_OK;
  if (pdl_launch(rope_token_prep_kernel, (n_tok + 7) / 8, 256, 0, stream, 1, table, table_stride,
                 tok_pos, tok_row, tok_col, tok_off, cos_tab, sin_tab, n_tok, hkv, tok_dst,
                 tok_cs) != cudaSuccess)
    return CORTEX_ECUDA;
  return CORTEX_OK;
}

int32_t cortex_argmax_partials(const void* partials, int32_t n_chunks, int32_t n_rows,
                               int32_t* out_tok, const int32_t* slot, int32_t* slot_tok,
                               int32_t* hist, int32_t hist_stride, const int32_t* hist_pos,
                               cudaStream_t stream) {
  if (!partials || n_rows < 0 || n_chunks <= 0) return CORTEX_EBADARG;
  if (hist && (!slot || !hist_pos)) return CORTEX_EBADARG;
  if (n_rows == 0) return CORTEX_OK;
  if (pdl_launch(argmax_partials_kernel, n_rows, 256, 0, stream, 1,
                 reinterpret_cast<const float2*>(partials), n_chunks, out_tok, slot, slot_tok,
                 hist, hist_stride, hist_pos) != cudaSuccess)
    return CORTEX_ECUDA;
  return CORTEX_OK;
}

int32_t cortex_argmax(const float* logits, int64_t ld, int32_t n_rows, int32_t vocab,
                      int32_t* out_tok, const int32_t* slot, int32_t* slot_tok, int32_t* hist,
                      int32_t hist_stride, const int32_t* hist_pos, cudaStream_t stream) {
  if (!logits || n_rows < 0 || vocab <= 0) return CORTEX_EBADARG;
  if (hist && (!slot || !hist_pos)) return CORTEX_EBADARG;
  if (n_rows == 0) return CORTEX_OK;
  if (pdl_launch(argmax_kernel, n_rows, 1024, 0, stream, 1, logits, ld, vocab, out_tok, slot,
                 slot_tok, hist, hist_stride, hist_pos) != cudaSuccess)
    return CORTEX_ECUDA;
  return CORTEX_OK;
}

}  // extern "C"
