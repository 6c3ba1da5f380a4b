// KV block pool: a free-list bitmap per engine (bit = 1 means the block is free)
// with warp-cooperative allocation that writes straight into block-table rows.
//
// Allocation policy (the contract the CPU oracle restates): requests are served
// in the order given, and the pool hands out free blocks lowest-index-first, so
// request i receives the free blocks of global free-rank [off_i, off_i + n_i)
// where off_i = n_0 + ... + n_{i-1}. A batch that does not fit changes nothing
// and reports CORTEX_ENOBLOCKS.
//
// One CTA of 1024 threads: each lane owns one 32-bit bitmap word per round,
// free-bit ranks come from a warp shuffle scan of popcounts plus a block scan of
// warp totals, and each lane then walks its word's set bits (__fns) to place them.
#include "common.cuh"

namespace {

constexpr int kAllocThreads = 1024;
constexpr int kMaxReq = 2048;

CORTEX_DEVICE int warp_incl_scan(int v) {
  const int lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

// Block-wide exclusive scan of one int per thread; returns the exclusive prefix,
// writes the block total to *total. Uses smem[32].
CORTEX_DEVICE int block_excl_scan(int v, int* smem, int* total) {
  const int lane = lane_id();
  const int warp = warp_id();
  const int incl = warp_incl_scan(v);
  if (lane == 31) smem[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x / 32;
    int w = lane < nw ? smem[lane] : 0;
    w = warp_incl_scan(w);
    if (lane < nw) smem[lane] = w;
  }
  __syncthreads();
  const int warp_base = warp == 0 ? 0 : smem[warp - 1];
  *total = smem[blockDim.x / 32 - 1];
  __syncthreads();
  return warp_base + incl - v;
}

CORTEX_DEVICE void kv_alloc_impl(uint32_t* bitmap, int nblocks, int id_base, const int* counts,
                                 const int* rows, const int* cols, int n_req, int* table,
                                 int table_stride, int* status) {
  __shared__ int s_off[kMaxReq + 1];
  __shared__ int s_scan[32];
  const int tid = threadIdx.x;

  // exclusive offsets of the requests (n_req <= kMaxReq)
  int carry = 0;
  for (int base = 0; base < n_req; base += kAllocThreads) {
    const int i = base + tid;
    const int c = i < n_req ? counts[i] : 0;
    int tot;
    const int ex = block_excl_scan(c, s_scan, &tot);
    if (i < n_req) s_off[i] = carry + ex;
    carry += tot;
  }
  if (tid == 0) s_off[n_req] = carry;
  __syncthreads();
  const int need = s_off[n_req];
  if (need == 0) return;

  // free-block count
  const int nwords = (nblocks + 31) / 32;
  int local = 0;
  for (int w = tid; w < nwords; w += kAllocThreads) local += __popc(bitmap[w]);
  int tot;
  block_excl_scan(local, s_scan, &tot);
  if (tot < need) {
    if (tid == 0) atomicExch(status, CORTEX_ENOBLOCKS);
    return;
  }

  // place: rounds of 1024 consecutive words, lane <-> word
  int rank_base = 0;
  for (int w0 = 0; w0 < nwords && rank_base < need; w0 += kAllocThreads) {
    const int w = w0 + tid;
    uint32_t word = w < nwords ? bitmap[w] : 0u;
    const int pc = __popc(word);
    int round_total;
    int r = rank_base + block_excl_scan(pc, s_scan, &round_total);
    if (pc && r < need) {
      uint32_t taken = 0;
      uint32_t rest = word;
      while (rest && r < need) {
        const int bit = __ffs(rest) - 1;
        rest &= rest - 1;
        // request owning rank r: largest i with s_off[i] <= r
        int lo = 0, hi = n_req - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (s_off[mid] <= r) lo = mid;
          else hi = mid - 1;
        }
        // skip zero-count requests sharing the same offset
        while (lo + 1 < n_req && s_off[lo + 1] <= r) ++lo;
        const int k = r - s_off[lo];
        table[static_cast<int64_t>(rows[lo]) * table_stride + cols[lo] + k] = id_base + w * 32 + bit;
        taken |= 1u << bit;
        ++r;
      }
      bitmap[w] = word & ~taken;
    }
    rank_base += round_total;
  }
}

__global__ void __launch_bounds__(kAllocThreads)
    kv_alloc_kernel(uint32_t* bitmap, int nblocks, int id_base, const int* counts,
                    const int* rows, const int* cols, int n_req, int* table, int table_stride,
                    int* status) {
  kv_alloc_impl(bitmap, nblocks, id_base, counts, rows, cols, n_req, table, table_stride, status);
}

// Requests passed by value in the kernel parameters (the _h exports: host arrays, no
// staging copy - an H2D copy before a kernel costs a copy-engine round trip of ~10-40 us
// of GPU idle time per allocator call, profiles/r1_step_trace_pdl.txt).
constexpr int kParamReq = 256;
struct PoolReqs {
  int n;
  int a[kParamReq];
  int b[kParamReq];
  int c[kParamReq];
};

__global__ void __launch_bounds__(kAllocThreads)
    kv_alloc_param_kernel(uint32_t* bitmap, int nblocks, int id_base,
                          const __grid_constant__ PoolReqs r, int* table, int table_stride,
                          int* status) {
  pdl_wait();
  pdl_trigger();
  // a = counts, b = rows, c = cols
  kv_alloc_impl(bitmap, nblocks, id_base, r.a, r.b, r.c, r.n, table, table_stride, status);
}

// Return blocks named by table[rows[i]][cols[i] .. cols[i]+counts[i]) to the pool.
CORTEX_DEVICE void kv_free_impl(uint32_t* bitmap, int nblocks, int id_base, const int* table,
                                int table_stride, const int* rows, const int* cols,
                                const int* counts, int n_req, int* status) {
  const int i = blockIdx.x;
  if (i >= n_req) return;
  const int c = counts[i];
  const int* src = table + static_cast<int64_t>(rows[i]) * table_stride + cols[i];
  for (int k = threadIdx.x; k < c; k += blockDim.x) {
    const int id = src[k] - id_base;
    if (id < 0 || id >= nblocks) {
      atomicExch(status, CORTEX_EBADARG);
      continue;
    }
    const uint32_t bit = 1u << (id & 31);
    const uint32_t old = atomicOr(&bitmap[id >> 5], bit);
    if (old & bit) atomicExch(status, CORTEX_EBADARG);  // double free
  }
}

__global__ void kv_free_kernel(uint32_t* bitmap, int nblocks, int id_base, const int* table,
                               int table_stride, const int* rows, const int* cols,
                               const int* counts, int n_req, int* status) {
  kv_free_impl(bitmap, nblocks, id_base, table, table_stride, rows, cols, counts, n_req, status);
}

__global__ void kv_free_param_kernel(uint32_t* bitmap, int nblocks, int id_base, const int* table,
                                     int table_stride, const __grid_constant__ PoolReqs r,
                                     int* status) {
  pdl_wait();
  pdl_trigger();
  // a = rows, b = cols, c = counts
  kv_free_impl(bitmap, nblocks, id_base, table, table_stride, r.a, r.b, r.c, r.n, status);
}

// table[dst_rows[i]][dst_cols[i] + k] = table[src_rows[i]][k], k < counts[i]
__global__ void table_copy_kernel(int* table, int table_stride, const int* src_rows,
                                  const int* dst_rows, const int* dst_cols, const int* counts,
                                  int n) {
  const int i = blockIdx.x;
  if (i >= n) return;
  const int* src = table + static_cast<int64_t>(src_rows[i]) * table_stride;
  int* dst = table + static_cast<int64_t>(dst_rows[i]) * table_stride + dst_cols[i];
  for (int k = threadIdx.x; k < counts[i]; k += blockDim.x) dst[k] = src[k];
}

struct CopyReqs {
  int n;
  int src[kParamReq / 2];
  int dst[kParamReq / 2];
  int col[kParamReq / 2];
  int cnt[kParamReq / 2];
};

__global__ void table_copy_param_kernel(int* table, int table_stride,
                                        const __grid_constant__ CopyReqs r) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x;
  if (i >= r.n) return;
  const int* src = table + static_cast<int64_t>(r.src[i]) * table_stride;
  int* dst = table + static_cast<int64_t>(r.dst[i]) * table_stride + r.col[i];
  for (int k = threadIdx.x; k < r.cnt[i]; k += blockDim.x) dst[k] = src[k];
}

__global__ void popcount_kernel(const uint32_t* bitmap, int nwords, int* out_free) {
  int local = 0;
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < nwords; w += gridDim.x * blockDim.x)
    local += __popc(bitmap[w]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if (lane_id() == 0 && local) atomicAdd(out_free, local);
}

}  // namespace

// Tuning / test knobs (cortex_dev.h) with the product defaults.
int g_cortex_knob[CORTEX_KNOB_COUNT] = {
    /* PDL */ 1, /* GEMM_MODE */ 0, /* GEMM_STREAM_K */ -1, /* GEMM_TN */ -1,
    /* GEMM_L2PF */ 0, /* SK_KS */ -1, /* SK_MT */ -1, /* SK_NW */ -1, /* SK_ISSUE */ 2,
    /* FMHA_2Q */ 1, /* FMHA_PLO */ 1,
    /* GEMM_TILE_OVH */ 32};

namespace {
bool knob_ok(int knob, int v) {
  switch (knob) {
    case CORTEX_KNOB_PDL: return v == 0 || v == 1;
    case CORTEX_KNOB_GEMM_MODE: return v >= 0 && v <= 3;
    case CORTEX_KNOB_GEMM_STREAM_K: return v >= -1 && v <= 1;
    case CORTEX_KNOB_GEMM_TN: return v == -1 || (v >= 64 && v <= 256 && v % 32 == 0);
    case CORTEX_KNOB_GEMM_L2PF: return v >= 0 && v <= 64;
    case CORTEX_KNOB_SK_KS: return v == -1 || (v >= 2 && v <= 4);
    case CORTEX_KNOB_SK_MT: return v == -1 || (v >= 1 && v <= 4);
    case CORTEX_KNOB_SK_NW: return v == -1 || v == 2;
    case CORTEX_KNOB_SK_ISSUE: return v == 1 || v == 2 || v == 4;
    case CORTEX_KNOB_FMHA_2Q: return v >= -1 && v <= 1;
    case CORTEX_KNOB_FMHA_PLO: return v == 0 || v == 1;
    case CORTEX_KNOB_GEMM_TILE_OVH: return v >= 0 && v <= 256;
    default: return false;
  }
}
}  // namespace

extern "C" {

int32_t cortex_abi_version(void) { return 103; }

int32_t cortex_dev_set_knob(int32_t knob, int32_t value) {
  if (!knob_ok(knob, value)) return CORTEX_EBADARG;
  g_cortex_knob[knob] = value;
  return CORTEX_OK;
}

int32_t cortex_dev_last_cuda_error(void) { return static_cast<int32_t>(cudaGetLastError()); }

int32_t cortex_dev_get_knob(int32_t knob) {
  if (knob < 0 || knob >= CORTEX_KNOB_COUNT) return CORTEX_EBADARG;
  return g_cortex_knob[knob];
}

int32_t cortex_kv_alloc(uint32_t* bitmap, int32_t nblocks, int32_t id_base,
                        const int32_t* counts, const int32_t* rows, const int32_t* cols,
                        int32_t n_req, int32_t* table, int32_t table_stride, int32_t* status,
                        cudaStream_t stream) {
  if (!bitmap || nblocks <= 0 || n_req < 0 || n_req > kMaxReq || !table || !status)
    return CORTEX_EBADARG;
  if (n_req == 0) return CORTEX_OK;
  if (!counts || !rows || !cols) return CORTEX_EBADARG;
  kv_alloc_kernel<<<1, kAllocThreads, 0, stream>>>(bitmap, nblocks, id_base, counts, rows, cols,
                                                    n_req, table, table_stride, status);
  CORTEX_CHECK_LAUNCH();
  return CORTEX_OK;
}

int32_t cortex_kv_free(uint32_t* bitmap, int32_t nblocks, int32_t id_base, const int32_t* table,
                       int32_t table_stride, const int32_t* rows, const int32_t* cols,
                       const int32_t* counts, int32_t n_req, int32_t* status,
                       cudaStream_t stream) {
  if (!bitmap || nblocks <= 0 || n_req < 0 || !table || !status) return CORTEX_EBADARG;
  if (n_req == 0) return CORTEX_OK;
  if (!rows || !cols || !counts) return CORTEX_EBADARG;
  kv_free_kernel<<<n_req, 128, 0, stream>>>(bitmap, nblocks, id_base, table, table_stride, rows,
                                            cols, counts, n_req, status);
  CORTEX_CHECK_LAUNCH();
  return CORTEX_OK;
}

int32_t cortex_table_copy(int32_t* table, int32_t table_stride, const int32_t* src_rows,
                          const int32_t* dst_rows, const int32_t* dst_cols, const int32_t* counts,
                          int32_t n, cudaStream_t stream) {
  if (!table || n < 0) return CORTEX_EBADARG;
  if (n == 0) return CORTEX_OK;
  if (!src_rows || !dst_rows || !dst_cols || !counts) return CORTEX_EBADARG;
  table_copy_kernel<<<n, 128, 0, stream>>>(table, table_stride, src_rows, dst_rows, dst_cols,
                                           counts, n);
  CORTEX_CHECK_LAUNCH();
  return CORTEX_OK;
}

// Number of free blocks (adds into *out_free, which the caller zeroes).
int32_t cortex_kv_count_free(const uint32_t* bitmap, int32_t nblocks, int32_t* out_free,
                             cudaStream_t stream) {
  if (!bitmap || nblocks <= 0 || !out_free) return CORTEX_EBADARG;
  const int nwords = (nblocks + 31) / 32;
  const int grid = (nwords + 255) / 256;
  popcount_kernel<<<grid < 148 ? grid : 148, 256, 0, stream>>>(bitmap, nwords, out_free);
  CORTEX_CHECK_LAUNCH();
  return CORTEX_OK;
}

// Host-array variants: the request arrays are host memory, packed into the kernel
// parameters (chunks of kParamReq requests, served in order).
int32_t cortex_kv_alloc_h(uint32_t* bitmap, int32_t nblocks, int32_t id_base,
                          const int32_t* counts, const int32_t* rows, const int32_t* cols,
                          int32_t n_req, int32_t* table, int32_t table_stride, int32_t* status,
                          cudaStream_t stream) {
  if (!bitmap || nblocks <= 0 || n_req < 0 || !table || !status || (n_req && (!counts || !rows || !cols)))
    return CORTEX_EBADARG;
  for (int base = 0; base < n_req; base += kParamReq) {
    PoolReqs r;
    r.n = n_req - base < kParamReq ? n_req - base : kParamReq;
    for (int i = 0; i < r.n; ++i) {
      r.a[i] = counts[base + i];
      r.b[i] = rows[base + i];
      r.c[i] = cols[base + i];
    }
    if (pdl_launch(kv_alloc_param_kernel, 1, kAllocThreads, 0, stream, 1, bitmap, nblocks, id_base,
                   r, table, table_stride, status) != cudaSuccess)
      return CORTEX_ECUDA;
  }
  return CORTEX_OK;
}

int32_t cortex_kv_free_h(uint32_t* bitmap, int32_t nblocks, int32_t id_base, const int32_t* table,
                         int32_t table_stride, const int32_t* rows, const int32_t* cols,
                         const int32_t* counts, int32_t n_req, int32_t* status,
                         cudaStream_t stream) {
  if (!bitmap || nblocks <= 0 || n_req < 0 || !table || !status || (n_req && (!counts || !rows || !cols)))
    return CORTEX_EBADARG;
  for (int base = 0; base < n_req; base += kParamReq) {
    PoolReqs r;
    r.n = n_req - base < kParamReq ? n_req - base : kParamReq;
    for (int i = 0; i < r.n; ++i) {
      r.a[i] = rows[base + i];
      r.b[i] = cols[base + i];
      r.c[i] = counts[base + i];
    }
    if (pdl_launch(kv_free_param_kernel, r.n, 128, 0, stream, 1, bitmap, nblocks, id_base, table,
                   table_stride, r, status) != cudaSuccess)
      return CORTEX_ECUDA;
  }
  return CORTEX_OK;
}

int32_t cortex_table_copy_h(int32_t* table, int32_t table_stride, const int32_t* src_rows,
                            const int32_t* dst_rows, const int32_t* dst_cols,
                            const int32_t* counts, int32_t n, cudaStream_t stream) {
  if (!table || n < 0 || (n && (!src_rows || !dst_rows || !dst_cols || !counts)))
    return CORTEX_EBADARG;
  for (int base = 0; base < n; base += kParamReq / 2) {
    CopyReqs r;
    r.n = n - base < kParamReq / 2 ? n - base : kParamReq / 2;
    for (int i = 0; i < r.n; ++i) {
      r.src[i] = src_rows[base + i];
      r.dst[i] = dst_rows[base + i];
      r.col[i] = dst_cols[base + i];
      r.cnt[i] = counts[base + i];
    }
    if (pdl_launch(table_copy_param_kernel, r.n, 128, 0, stream, 1, table, table_stride, r) !=
        cudaSuccess)
      return CORTEX_ECUDA;
  }
  return CORTEX_OK;
}

}  // extern "C"
