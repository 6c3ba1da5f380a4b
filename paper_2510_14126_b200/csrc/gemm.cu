// Dense projections of the stage-engine decoder on 5th-gen tensor cores.
//
//   C[m, n] = sum_k X[m, k] * W[n, k]        (+ residual[m, n], fp32)
//
// X is the activation matrix [M, K] (tokens x features, bf16, row-major), W the
// weight matrix [N, K] (nn.Linear layout, bf16). The kernel is "swap-AB": the
// weight rows form the 128-wide MMA M dimension and the tokens the MMA N
// dimension (TN = 32..256), so a decode step with a handful of sequences still
// issues full 128-row tcgen05.mma instructions while streaming the weights
// exactly once. Operands are staged by TMA (128-byte swizzle) through a
// STAGES-deep mbarrier ring, the accumulator lives in TMEM, and the epilogue is
// tcgen05.ld -> registers -> global. Decode-sized problems split K across CTAs
// with a deterministic (fixed-order) reduction done by the last CTA of a tile,
// so a token's result does not depend on which other tokens share the batch.
#include <algorithm>

#include <cudaTypedefs.h>

#include "common.cuh"

namespace {

constexpr int kBlockN = 128;  // weight rows per tile (MMA M)
constexpr int kBlockK = 64;   // K per stage (one 128-byte swizzle row)
constexpr int kXBox = CORTEX_XBOX;  // activation rows per TMA box
constexpr int kThreads = 128;

struct GemmArgs {
  int M, N, K;
  void* out;
  int ldo;
  int out_f32;
  const float* residual;  // fp32 (the residual stream)
  int ldr;
  int kb_per_split;
  int splits;
  float* workspace;
  int* counters;
  int evict_first_w;
  RopeEpi rope;  // out mode 4 (QKV: RoPE + paged KV append in the epilogue)
};

template <int TN, int STAGES>
struct GemmSmem {
  static constexpr int kABytes = kBlockN * kBlockK * 2;  // 16 KiB
  static constexpr int kBBytes = TN * kBlockK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kBarOffset = STAGES * kStageBytes;
  static constexpr int kTotal = kBarOffset + 256 + 1024;  // barriers + alignment slack
  static constexpr uint32_t kTmemCols = TN < 32 ? 32 : TN;
};

// Final store of rows r0, r0+4, ... < rows of the smem tile: optional fp32 residual,
// bf16 or fp32 output. Each warp covers one 128-column row with 16-byte accesses;
// four rows' loads are issued before any store (out may alias residual).
CORTEX_DEVICE void epilogue_rows(const GemmArgs& a, const float* stile, int m0, int rows, int r0,
                                 int lane, int col) {
  if (a.out_f32 == 4) {  // QKV: the tile's 128 columns are one head; 8 rows' operands at once
    const int h = (col - 4 * lane) / kBlockN;
    for (int rb = r0; rb < rows; rb += 32) {
      RopeRow rr[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (rb + 4 * u < rows) rr[u] = rope_fetch(a.rope, m0 + rb + 4 * u, h);
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (rb + 4 * u < rows)
          rope_store_row(a.rope, rr[u], m0 + rb + 4 * u, h,
                         reinterpret_cast<const float4*>(stile + (rb + 4 * u) * kBlockN)[lane]);
    }
    return;
  }
  if (a.out_f32 == 3) {  // greedy-token partials: (max, index) of this tile's 128 columns
    for (int r = r0; r < rows; r += 4)
      store_argmax_partial(reinterpret_cast<float2*>(a.out), a.ldo, m0 + r, col - 4 * lane,
                           reinterpret_cast<const float4*>(stile + r * kBlockN)[lane], col);
    return;
  }
  if (a.out_f32 == 2) {  // fused SwiGLU: tile rows = 64 gate + 64 up features
    const int f = (col - 4 * lane) / 2 + 2 * lane;
    for (int r = r0; r < rows; r += 4) {
      const float2 g = reinterpret_cast<const float2*>(stile + r * kBlockN)[lane];
      const float2 u = reinterpret_cast<const float2*>(stile + r * kBlockN + 64)[lane];
      *reinterpret_cast<uint32_t*>(reinterpret_cast<__nv_bfloat16*>(a.out) +
                                   static_cast<size_t>(m0 + r) * a.ldo + f) =
          pack_bf16(g.x / (1.f + __expf(-g.x)) * u.x, g.y / (1.f + __expf(-g.y)) * u.y);
    }
    return;
  }
  for (int rb = r0; rb < rows; rb += 16) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int r = rb + 4 * u;
      if (r < rows) {
        v[u] = reinterpret_cast<const float4*>(stile + r * kBlockN)[lane];
        if (a.residual) {
          const float4 res = *reinterpret_cast<const float4*>(
              a.residual + static_cast<size_t>(m0 + r) * a.ldr + col);
          v[u].x += res.x;
          v[u].y += res.y;
          v[u].z += res.z;
          v[u].w += res.w;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int r = rb + 4 * u;
      if (r < rows) {
        const size_t off = static_cast<size_t>(m0 + r) * a.ldo + col;
        if (a.out_f32) {
          *reinterpret_cast<float4*>(reinterpret_cast<float*>(a.out) + off) = v[u];
        } else {
          uint2 packed;
          packed.x = pack_bf16(v[u].x, v[u].y);
          packed.y = pack_bf16(v[u].z, v[u].w);
          *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(a.out) + off) = packed;
        }
      }
    }
  }
}

template <int TN, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_tcgen05(const __grid_constant__ CUtensorMap tmap_w,
                      const __grid_constant__ CUtensorMap tmap_x, const GemmArgs args) {
  using L = GemmSmem<TN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBarOffset);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(done + 1);
  int* last_flag = reinterpret_cast<int*>(tmem_holder + 1);

  const int warp = warp_id();
  const int lane = lane_id();
  const int n_tile = blockIdx.x;
  const int m_tile = blockIdx.y;
  const int split = blockIdx.z;
  const int n0 = n_tile * kBlockN;
  const int m0 = m_tile * TN;
  const int total_kb = args.K / kBlockK;
  const int kb0 = split * args.kb_per_split;
  const int kb1 = min(kb0 + args.kb_per_split, total_kb);
  const int nkb = kb1 - kb0;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_w);
    tma_prefetch_desc(&tmap_x);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_holder, L::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  pdl_wait();  // the activations (and residual) come from the previous kernel
  pdl_trigger();

  if (warp == 0) {
    if (elect_one()) {
      // ---- TMA producer ----
      const uint64_t pol_w = policy_evict_first();
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (i / STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* sa = smem + s * L::kStageBytes;
        uint8_t* sb = sa + L::kABytes;
        mbar_arrive_expect_tx(&full[s], L::kStageBytes);
        const int kc = (kb0 + i) * kBlockK;
        if (args.evict_first_w)
          tma_load_2d_hint(sa, &tmap_w, &full[s], kc, n0, pol_w);
        else
          tma_load_2d(sa, &tmap_w, &full[s], kc, n0);
#pragma unroll
        for (int j = 0; j < TN / kXBox; ++j)
          tma_load_2d(sb + j * kXBox * 128, &tmap_x, &full[s], kc, m0 + j * kXBox);
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      // ---- MMA issuer (one thread) ----
      constexpr uint32_t idesc = umma_idesc_bf16(kBlockN, TN);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (i / STAGES) & 1;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t a_addr = smem_u32(smem + s * L::kStageBytes);
        const uint32_t b_addr = a_addr + L::kABytes;
#pragma unroll
        for (int k = 0; k < kBlockK / 16; ++k) {
          umma_bf16_ss(tmem_base, umma_desc_sw128(a_addr + k * 32), umma_desc_sw128(b_addr + k * 32),
                       idesc, (i | k) != 0 ? 1u : 0u);
        }
        umma_commit(&empty[s]);
      }
      umma_commit(done);
    }
  }
  __syncwarp();

  // ---- epilogue: TMEM -> smem tile [m][128 n] fp32 -> coalesced 16-byte rows ----
  // (the pipeline stages are free once `done` fired: every MMA, hence every
  // smem operand read, has completed)
  mbar_wait(done, 0);
  tc_fence_after();
  const uint32_t taddr = tmem_base + (static_cast<uint32_t>(warp * 32) << 16);
  const int m_end = min(m0 + TN, args.M);
  const int rows = m_end - m0;
  float* stile = reinterpret_cast<float*>(smem);
  for (int c0 = 0; c0 < TN && c0 < rows; c0 += 16) {
    uint32_t r[16];
    tmem_ld_32x32b_x16(taddr + c0, r);
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 16; ++j) stile[(c0 + j) * kBlockN + warp * 32 + lane] = __uint_as_float(r[j]);
  }
  __syncthreads();
  // thread -> (row r = tid/32 + 4i, columns 4*lane .. 4*lane+3)
  const int col = n0 + 4 * lane;
  const int r0 = threadIdx.x >> 5;
  if (args.splits == 1) {
    epilogue_rows(args, stile, m0, rows, r0, lane, col);
  } else {
    // Split-K: publish this split's fp32 partial; the last CTA of the tile reduces
    // all partials in split order (deterministic) and runs the epilogue.
    float* ws = args.workspace + static_cast<size_t>(split) * args.M * args.N;
    for (int r = r0; r < rows; r += 4) {
      const float4 v = reinterpret_cast<const float4*>(stile + r * kBlockN)[lane];
      __stcg(reinterpret_cast<float4*>(ws + static_cast<size_t>(m0 + r) * args.N + col), v);
    }
    __threadfence();
    __syncthreads();
    const int tile_id = m_tile * gridDim.x + n_tile;
    if (threadIdx.x == 0) {
      const int prev = atomicAdd(&args.counters[tile_id], 1);
      *last_flag = (prev == args.splits - 1) ? 1 : 0;
    }
    __syncthreads();
    if (*last_flag) {
      __threadfence();
      for (int rb = r0; rb < rows; rb += 32) {
        float4 acc[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int z = 0; z < args.splits; ++z) {  // split order: deterministic sum
          const float* wz = args.workspace + static_cast<size_t>(z) * args.M * args.N;
          float4 v[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {  // 8 independent loads in flight
            const int r = rb + 4 * q;
            if (r < rows)
              v[q] = __ldcg(reinterpret_cast<const float4*>(
                  wz + static_cast<size_t>(m0 + r) * args.N + col));
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            if (rb + 4 * q < rows) {
              acc[q].x += v[q].x;
              acc[q].y += v[q].y;
              acc[q].z += v[q].z;
              acc[q].w += v[q].w;
            }
          }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int r = rb + 4 * q;
          if (r < rows) reinterpret_cast<float4*>(stile + r * kBlockN)[lane] = acc[q];
        }
      }
      __syncwarp();
      epilogue_rows(args, stile, m0, rows, r0, lane, col);
      if (threadIdx.x == 0) args.counters[tile_id] = 0;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, L::kTmemCols);
  }
}

template <int TN, int STAGES>
int32_t launch_gemm(const CUtensorMap* tw, const CUtensorMap* tx, const GemmArgs& a, dim3 grid,
                    cudaStream_t stream) {
  using L = GemmSmem<TN, STAGES>;
  auto kern = gemm_bf16_tcgen05<TN, STAGES>;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kTotal) !=
        cudaSuccess)
      return CORTEX_ECUDA;
    configured = true;
  }
  if (pdl_launch(kern, grid, kThreads, L::kTotal, stream, 1, *tw, *tx, a) != cudaSuccess)
    return CORTEX_ECUDA;
  return CORTEX_OK;
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

}  // namespace

int32_t cortex_gemm_2sm_launch(const void* tmap_w, const void* tmap_x, int32_t M, int32_t N,
                               int32_t K, void* out, int32_t ldo, int32_t out_f32,
                               const void* residual, int32_t ldr, float* workspace,
                               uint64_t workspace_bytes, int32_t* counters, int32_t n_counters,
                               const RopeEpi* rope, cudaStream_t stream);

extern "C" int32_t cortex_gemm_splitk_launch(const void* tmap_w, const void* tmap_x, int32_t M,
                                             int32_t N, int32_t K, void* out, int32_t ldo,
                                             int32_t out_f32, const void* residual, int32_t ldr,
                                             float* workspace, uint64_t workspace_bytes,
                                             int32_t* counters, int32_t n_counters,
                                             const RopeEpi* rope, cudaStream_t stream);

extern "C" {

// Kernel choice: 1 = 1-SM swap-AB kernel with split-K (decode-sized, weight-streaming
// bound; N % 256 != 0 or too many tiles for a split plan), 2 = persistent 2-SM kernel
// (M > 128, compute bound; needs N % 256 == 0).
// 3 = cluster split-K 2-SM kernel (gemm_splitk.cu: decode-sized M with few 256-row tiles).
int32_t cortex_gemm_path(int32_t M, int32_t N, int32_t K) {
  // knob GEMM_MODE (tests): 0 auto, 1 force 1-SM, 2 force 2-SM when legal, 3 prefer split-K
  const int mode = g_cortex_knob[CORTEX_KNOB_GEMM_MODE];
  const bool legal2 = (N % 256) == 0;
  if (mode == 1 || !legal2) return 1;
  if (mode == 2) return 2;
  if (cortex_gemm_splitk_plan(M, N, K, nullptr, nullptr, nullptr) >= 1) return 3;
  if (mode == 3) return 2;
  return M > 128 ? 2 : 1;
}

// Rows per TMA box of the activation (token) operand the GEMMs expect.
int32_t cortex_act_box_rows(void) { return CORTEX_XBOX; }

// Encode a 2-D bf16 TMA descriptor (128 bytes, written to tmap_out) over a
// row-major matrix [rows, cols] with the given row pitch. box_cols * 2 must be
// 128 (one swizzle row); the tile lands in shared memory with SWIZZLE_128B.
int32_t cortex_tmap_encode_2d_bf16(void* tmap_out, const void* gptr, uint64_t rows, uint64_t cols,
                                   uint64_t row_pitch_bytes, uint32_t box_rows,
                                   uint32_t box_cols) {
  if (!tmap_out || !gptr || rows == 0 || cols == 0 || box_cols * 2 != 128 || box_rows == 0 ||
      box_rows > 256 || (row_pitch_bytes % 16) != 0 ||
      (reinterpret_cast<uintptr_t>(gptr) % 16) != 0)
    return CORTEX_EBADARG;
  auto fn = get_encode_fn();
  if (!fn) return CORTEX_ECUDA;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {row_pitch_bytes};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(reinterpret_cast<CUtensorMap*>(tmap_out), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                  const_cast<void*>(gptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? CORTEX_OK : CORTEX_ECUDA;
}

// 3-D bf16 TMA descriptor over q [n_tok, hq, 128] with box (64 dims, group heads,
// 128/group tokens): 128 query rows (token-major, head-minor) of one GQA group.
int32_t cortex_tmap_encode_q(void* tmap_out, const void* q, uint64_t n_tok, int32_t hq,
                             int32_t group) {
  if (!tmap_out || !q || n_tok == 0 || hq <= 0 || group <= 0 || (128 % group) != 0 ||
      (reinterpret_cast<uintptr_t>(q) % 16) != 0)
    return CORTEX_EBADARG;
  auto fn = get_encode_fn();
  if (!fn) return CORTEX_ECUDA;
  cuuint64_t dims[3] = {128, static_cast<cuuint64_t>(hq), n_tok};
  cuuint64_t strides[2] = {256, static_cast<cuuint64_t>(hq) * 256};
  cuuint32_t box[3] = {64, static_cast<cuuint32_t>(group), static_cast<cuuint32_t>(128 / group)};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(reinterpret_cast<CUtensorMap*>(tmap_out), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                  const_cast<void*>(q), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? CORTEX_OK : CORTEX_ECUDA;
}

// Split-K factor the GEMM uses for a problem (exported so the host can size the
// workspace and so tests can pin batch invariance).
int32_t cortex_gemm_splits(int32_t M, int32_t N, int32_t K) {
  if (M <= 0 || N % kBlockN || K % kBlockK) return 1;
  const int n_tiles = N / kBlockN;
  const int total_kb = K / kBlockK;
  if (M > 256) return 1;
  const int target = 148;  // one wave of 1-CTA-per-SM deep pipelines
  int splits = (target + n_tiles - 1) / n_tiles;
  splits = std::min(splits, std::max(1, total_kb / 4));
  splits = std::min(splits, 16);
  splits = std::max(splits, 1);
  // re-balance so every split gets a non-empty K range
  const int kb_per = (total_kb + splits - 1) / splits;
  return (total_kb + kb_per - 1) / kb_per;
}

// C = X . W^T (+ residual). tmap_w: descriptor over W [N, K] with box (128 rows, 64 cols);
// tmap_x: descriptor over X [>=M rows, K] with box (32 rows, 64 cols). Output row pitch ldo
// (elements); out_f32 selects fp32 instead of bf16 output. workspace/counters are only used
// when cortex_gemm_splits(M, N, K) > 1 (workspace >= splits*M*N floats, counters zeroed,
// >= n_tiles*m_tiles ints; the kernel leaves them zeroed).
static int32_t gemm_dispatch(const void* tmap_w, const void* tmap_x, int32_t M, int32_t N,
                             int32_t K, void* out, int32_t ldo, int32_t out_f32,
                             const void* residual, int32_t ldr, float* workspace,
                             uint64_t workspace_bytes, int32_t* counters, int32_t n_counters,
                             const RopeEpi* rope, cudaStream_t stream) {
  if (!tmap_w || !tmap_x || (!out && out_f32 != 4) || M <= 0 || N <= 0 || K <= 0 ||
      N % kBlockN || K % kBlockK || out_f32 < 0 || out_f32 > 4 || (out_f32 >= 2 && residual) ||
      (out_f32 == 4 && !rope))
    return CORTEX_EBADARG;
  int path = cortex_gemm_path(M, N, K);
  if (out_f32 == 3 && path == 3) path = M > 128 ? 2 : 1;  // (lm_head never plans split-K)
  if (path == 3)
    return cortex_gemm_splitk_launch(tmap_w, tmap_x, M, N, K, out, ldo, out_f32, residual, ldr,
                                     workspace, workspace_bytes, counters, n_counters, rope,
                                     stream);
  if (path == 2)
    return cortex_gemm_2sm_launch(tmap_w, tmap_x, M, N, K, out, ldo, out_f32, residual, ldr,
                                  workspace, workspace_bytes, counters, n_counters, rope, stream);
  GemmArgs a{};
  a.M = M;
  a.N = N;
  a.K = K;
  a.out = out;
  a.ldo = ldo;
  a.out_f32 = out_f32;
  a.residual = reinterpret_cast<const float*>(residual);
  a.ldr = ldr;
  const int total_kb = K / kBlockK;
  const int splits = cortex_gemm_splits(M, N, K);
  a.kb_per_split = (total_kb + splits - 1) / splits;
  a.splits = splits;
  a.workspace = workspace;
  a.counters = counters;
  if (rope) a.rope = *rope;
  const int n_tiles = N / kBlockN;
  if (splits > 1) {
    if (!workspace || !counters ||
        workspace_bytes < static_cast<uint64_t>(splits) * M * N * sizeof(float) ||
        n_counters < n_tiles)
      return CORTEX_EBADARG;
  }
  const auto* tw = reinterpret_cast<const CUtensorMap*>(tmap_w);
  const auto* tx = reinterpret_cast<const CUtensorMap*>(tmap_x);
  int tn;
  if (M <= 32) tn = 32;
  else if (M <= 64) tn = 64;
  else if (M <= 128) tn = 128;
  else tn = 256;
  const int m_tiles = (M + tn - 1) / tn;
  a.evict_first_w = m_tiles == 1 ? 1 : 0;
  dim3 grid(n_tiles, m_tiles, splits);
  switch (tn) {
    case 32: return launch_gemm<32, 8>(tw, tx, a, grid, stream);
    case 64: return launch_gemm<64, 7>(tw, tx, a, grid, stream);
    case 128: return launch_gemm<128, 5>(tw, tx, a, grid, stream);
    default: return launch_gemm<256, 4>(tw, tx, a, grid, stream);
  }
}

int32_t cortex_gemm_bf16(const void* tmap_w, const void* tmap_x, int32_t M, int32_t N, int32_t K,
                         void* out, int32_t ldo, int32_t out_f32, const void* residual,
                         int32_t ldr, float* workspace, uint64_t workspace_bytes,
                         int32_t* counters, int32_t n_counters, cudaStream_t stream) {
  if (out_f32 == 4) return CORTEX_EBADARG;  // (cortex_gemm_qkv_rope)
  return gemm_dispatch(tmap_w, tmap_x, M, N, K, out, ldo, out_f32, residual, ldr, workspace,
                       workspace_bytes, counters, n_counters, nullptr, stream);
}

// QKV projection with RoPE + paged KV append in the epilogue (see the header).
int32_t cortex_gemm_qkv_rope(const void* tmap_w, const void* tmap_x, int32_t M, int32_t N,
                             int32_t K, const cortex_rope_epilogue_t* epi, float* workspace,
                             uint64_t workspace_bytes, int32_t* counters, int32_t n_counters,
                             cudaStream_t stream) {
  if (!epi || !epi->q_out || !epi->cache || !epi->tok_dst || !epi->tok_cs || epi->hq < 1 ||
      epi->hkv < 1 || N != (epi->hq + 2 * epi->hkv) * 128)
    return CORTEX_EBADARG;
  RopeEpi r{};
  r.q_out = reinterpret_cast<__nv_bfloat16*>(epi->q_out);
  r.cache = reinterpret_cast<__nv_bfloat16*>(epi->cache);
  r.k_row0 = epi->k_row0;
  r.v_row0 = epi->v_row0;
  r.tok_dst = epi->tok_dst;
  r.tok_cs = epi->tok_cs;
  r.hq = epi->hq;
  r.hkv = epi->hkv;
  return gemm_dispatch(tmap_w, tmap_x, M, N, K, nullptr, 0, 4, nullptr, 0, workspace,
                       workspace_bytes, counters, n_counters, &r, stream);
}

}  // extern "C"
