// Compute-bound projections (prefill / mixed steps, M > 128): persistent
// 2-SM tcgen05 GEMM.
//
//   C[m, n] = sum_k X[m, k] * W[n, k]        (+ residual[m, n], fp32)
//
// A CTA pair (cluster of 2) owns a 256 x TN output tile: each CTA stages 128
// weight rows and TN/2 activation rows per 64-wide K block (TMA, 128-byte
// swizzle, both halves signalling the leader's mbarrier), and the leader issues
// tcgen05.mma.cta_group::2 (M = 256), which reads A from each CTA's own smem and
// B from both — half the operand traffic of two independent 128-row CTAs. The
// accumulator is double-buffered in TMEM (2 x TN columns), so the four epilogue
// warps drain tile i (TMEM -> registers -> smem -> coalesced 16-byte stores,
// optional fp32 residual) while the MMA warp already accumulates tile i + 1.
// Pairs are persistent and walk tiles m-fastest, so concurrently running pairs
// share weight tiles in L2.
#include "common.cuh"

namespace {

constexpr int kPairN = 256;  // weight rows per CTA pair (MMA M)
constexpr int kBK = 64;
constexpr int kXBox2 = 16;   // activation rows per TMA box
constexpr int kEpiRows = 32; // output rows (m) per epilogue chunk
constexpr int kThreads2 = 192;
// K splits for the compute-bound GEMM: the deterministic fix-up (partials through L2 + a
// last-unit reduction) cost more than the wave-quantization it removes at the measured
// shapes (M=700, N=4096: 70 us split vs 37 us unsplit), so it is off.
constexpr int kMaxSplits2 = 1;

struct Gemm2Args {
  int M, N, K;
  void* out;
  int ldo;
  int out_f32;
  const float* residual;
  int ldr;
  int m_tiles;
  int num_tiles;
  int splits;        // K splits per tile (work units = num_tiles * splits)
  int kb_per_split;
  float* workspace;  // [splits][M][N] fp32 partials (splits > 1)
  int* counters;     // [num_tiles * 2] arrival counters, left zeroed
};

template <int TN, int STAGES>
struct G2 {
  static constexpr int kA = 128 * kBK * 2;       // 16 KiB per CTA
  static constexpr int kB = (TN / 2) * kBK * 2;  // TN/2 rows per CTA
  static constexpr int kStage = kA + kB;
  static constexpr int kStaging = kEpiRows * 128 * 4;
  static constexpr int kBar = STAGES * kStage + kStaging;
  static constexpr int kTotal = kBar + 512 + 1024;
  static constexpr uint32_t kTmemCols = 2 * TN <= 128 ? 128 : (2 * TN <= 256 ? 256 : 512);
};

CORTEX_DEVICE uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}

CORTEX_DEVICE uint32_t mapa_shared(uint32_t addr, uint32_t cta) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(addr), "r"(cta));
  return r;
}

CORTEX_DEVICE void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];\n" ::"r"(cluster_addr) : "memory");
}

CORTEX_DEVICE void cluster_sync() {
  asm volatile("barrier.cluster.arrive.aligned;\nbarrier.cluster.wait.aligned;\n" ::: "memory");
}

CORTEX_DEVICE void tma_load_2d_2sm(void* smem_dst, const void* desc, uint32_t bar_cluster, int c0,
                                   int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];\n" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(bar_cluster), "r"(c0), "r"(c1)
      : "memory");
}

CORTEX_DEVICE void umma_bf16_ss_2sm(uint32_t tmem_d, uint64_t desc_a, uint64_t desc_b,
                                    uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(desc_a), "l"(desc_b), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Arrive (once the leader's issued MMAs complete) on the barrier at this smem
// offset in both CTAs of the pair.
CORTEX_DEVICE void umma_commit_2sm_both(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], m;\n\t}\n" ::"r"(smem_u32(bar))
      : "memory");
}

CORTEX_DEVICE void tmem_alloc_2sm(uint32_t* holder, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                   smem_u32(holder)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::: "memory");
}

CORTEX_DEVICE void tmem_dealloc_2sm(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "r"(ncols)
               : "memory");
}

CORTEX_DEVICE void epi_bar_sync() { asm volatile("bar.sync 1, 128;\n" ::: "memory"); }

// Rows ew, ew+4, ... < crow of a staged fp32 chunk -> (+ fp32 residual) -> bf16 / fp32 out.
// Each warp covers one 128-column row with 16-byte accesses; all loads before any store
// (out may alias the residual).
CORTEX_DEVICE void store_chunk(const Gemm2Args& args, const float* staging, int mrow0, int crow,
                               int ew, int lane, int col) {
  if (args.out_f32 == 2) {  // fused SwiGLU: each CTA's 128 rows = 64 gate + 64 up features
    const int f = (col - 4 * lane) / 2 + 2 * lane;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int r = ew + 4 * q;
      if (r < crow) {
        const float2 g = reinterpret_cast<const float2*>(staging + r * 128)[lane];
        const float2 u = reinterpret_cast<const float2*>(staging + r * 128 + 64)[lane];
        *reinterpret_cast<uint32_t*>(reinterpret_cast<__nv_bfloat16*>(args.out) +
                                     static_cast<size_t>(mrow0 + r) * args.ldo + f) =
            pack_bf16(g.x / (1.f + __expf(-g.x)) * u.x, g.y / (1.f + __expf(-g.y)) * u.y);
      }
    }
    return;
  }
  float4 v[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int r = ew + 4 * q;
    if (r < crow) {
      v[q] = reinterpret_cast<const float4*>(staging + r * 128)[lane];
      if (args.residual) {
        const float4 res = *reinterpret_cast<const float4*>(
            args.residual + static_cast<size_t>(mrow0 + r) * args.ldr + col);
        v[q].x += res.x;
        v[q].y += res.y;
        v[q].z += res.z;
        v[q].w += res.w;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int r = ew + 4 * q;
    if (r < crow) {
      const size_t off = static_cast<size_t>(mrow0 + r) * args.ldo + col;
      if (args.out_f32) {
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(args.out) + off) = v[q];
      } else {
        uint2 packed;
        packed.x = pack_bf16(v[q].x, v[q].y);
        packed.y = pack_bf16(v[q].z, v[q].w);
        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(args.out) + off) = packed;
      }
    }
  }
}

template <int TN, int STAGES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads2, 1)
    gemm_bf16_2sm(const __grid_constant__ CUtensorMap tmap_w,
                  const __grid_constant__ CUtensorMap tmap_x, const Gemm2Args args) {
  using L = G2<TN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  float* staging = reinterpret_cast<float*>(smem + STAGES * L::kStage);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1;
  const int npairs = gridDim.x >> 1;
  const int warp = warp_id();
  const int lane = lane_id();
  const int total_kb = args.K / kBK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_w);
    tma_prefetch_desc(&tmap_x);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 2);   // leader: own expect_tx arrive + the peer's arrive
      mbar_init(&empty[s], 1);  // multicast MMA commit
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 8);  // 4 epilogue warps x 2 CTAs
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_2sm(tmem_holder, L::kTmemCols);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    if (elect_one()) {
      // ---- TMA producer (both CTAs load their halves) ----
      uint32_t it = 0;
      for (int u = pair; u < args.num_tiles * args.splits; u += npairs) {
        const int t = u / args.splits;
        const int kb0 = (u % args.splits) * args.kb_per_split;
        const int kb1 = min(total_kb, kb0 + args.kb_per_split);
        const int n_tile = t / args.m_tiles;
        const int m_tile = t % args.m_tiles;
        const int n0 = n_tile * kPairN + rank * 128;
        const int x0 = m_tile * TN + rank * (TN / 2);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          const uint32_t full_leader = mapa_shared(smem_u32(&full[s]), 0);
          if (leader)
            mbar_arrive_expect_tx(&full[s], 2 * L::kStage);
          else
            mbar_arrive_cluster(full_leader);
          uint8_t* sa = smem + s * L::kStage;
          uint8_t* sb = sa + L::kA;
          const int kc = kb * kBK;
          tma_load_2d_2sm(sa, &tmap_w, full_leader, kc, n0);
#pragma unroll
          for (int j = 0; j < TN / 2 / kXBox2; ++j)
            tma_load_2d_2sm(sb + j * kXBox2 * 128, &tmap_x, full_leader, kc, x0 + j * kXBox2);
        }
      }
    }
  } else if (warp == 1) {
    if (leader && elect_one()) {
      // ---- MMA issuer (leader CTA, one thread) ----
      constexpr uint32_t idesc = umma_idesc_bf16(kPairN, TN);
      uint32_t it = 0, tl = 0;
      for (int u = pair; u < args.num_tiles * args.splits; u += npairs, ++tl) {
        const int kb0 = (u % args.splits) * args.kb_per_split;
        const int kb1 = min(total_kb, kb0 + args.kb_per_split);
        const uint32_t b = tl & 1;
        const uint32_t tph = (tl >> 1) & 1;
        mbar_wait(&tempty[b], tph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + b * TN;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smem + s * L::kStage);
          const uint32_t b_addr = a_addr + L::kA;
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)
            umma_bf16_ss_2sm(d, umma_desc_sw128(a_addr + k * 32), umma_desc_sw128(b_addr + k * 32),
                             idesc, (kb != kb0 || k != 0) ? 1u : 0u);
          umma_commit_2sm_both(&empty[s]);
        }
        umma_commit_2sm_both(&tfull[b]);
      }
    }
  } else {
    // ---- epilogue warps 2..5: TMEM lane quadrant = warp % 4 ----
    const int quad = warp & 3;
    const int ew = warp - 2;  // 0..3
    const uint32_t tempty_leader_base = mapa_shared(smem_u32(&tempty[0]), 0);
    int* last_flag = reinterpret_cast<int*>(tmem_holder + 1);
    uint32_t tl = 0;
    for (int u = pair; u < args.num_tiles * args.splits; u += npairs, ++tl) {
      const int t = u / args.splits;
      const int z = u % args.splits;
      const uint32_t b = tl & 1;
      const uint32_t tph = (tl >> 1) & 1;
      const int n_tile = t / args.m_tiles;
      const int m_tile = t % args.m_tiles;
      const int n0 = n_tile * kPairN + rank * 128;
      const int m0 = m_tile * TN;
      const int rows = min(TN, args.M - m0);
      const int col = n0 + 4 * lane;
      mbar_wait(&tfull[b], tph);
      tc_fence_after();
      const uint32_t taddr = tmem_base + b * TN + (static_cast<uint32_t>(quad * 32) << 16);
      for (int c0 = 0; c0 < rows; c0 += kEpiRows) {
        uint32_t r0[16], r1[16];
        tmem_ld_32x32b_x16(taddr + c0, r0);
        tmem_ld_32x32b_x16(taddr + c0 + 16, r1);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          staging[j * 128 + quad * 32 + lane] = __uint_as_float(r0[j]);
          staging[(16 + j) * 128 + quad * 32 + lane] = __uint_as_float(r1[j]);
        }
        epi_bar_sync();
        const int crow = min(kEpiRows, rows - c0);
        if (args.splits == 1) {
          store_chunk(args, staging, m0 + c0, crow, ew, lane, col);
        } else {
          float* ws = args.workspace + static_cast<size_t>(z) * args.M * args.N;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int r = ew + 4 * q;
            if (r < crow)
              __stcg(reinterpret_cast<float4*>(ws + static_cast<size_t>(m0 + c0 + r) * args.N + col),
                     reinterpret_cast<const float4*>(staging + r * 128)[lane]);
          }
        }
        epi_bar_sync();
      }
      // the accumulator is drained: release it to the MMA warp before any fix-up work
      tc_fence_before();
      if (lane == 0) mbar_arrive_cluster(tempty_leader_base + b * 8);
      if (args.splits > 1) {
        // last unit of this (tile, CTA half) reduces the partials in split order
        __threadfence();
        epi_bar_sync();
        if (threadIdx.x == 64) {
          const int prev = atomicAdd(&args.counters[t * 2 + rank], 1);
          *last_flag = prev == args.splits - 1 ? 1 : 0;
        }
        epi_bar_sync();
        if (*last_flag) {
          __threadfence();
          for (int c0 = 0; c0 < rows; c0 += kEpiRows) {
            const int crow = min(kEpiRows, rows - c0);
            float4 acc[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int zz = 0; zz < args.splits; ++zz) {  // split order: deterministic sum
              const float* wz = args.workspace + static_cast<size_t>(zz) * args.M * args.N;
              float4 v[8];
#pragma unroll
              for (int q = 0; q < 8; ++q) {  // 8 independent loads in flight
                const int r = ew + 4 * q;
                if (r < crow)
                  v[q] = __ldcg(reinterpret_cast<const float4*>(
                      wz + static_cast<size_t>(m0 + c0 + r) * args.N + col));
              }
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                if (ew + 4 * q < crow) {
                  acc[q].x += v[q].x;
                  acc[q].y += v[q].y;
                  acc[q].z += v[q].z;
                  acc[q].w += v[q].w;
                }
              }
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const int r = ew + 4 * q;
              if (r < crow) reinterpret_cast<float4*>(staging + r * 128)[lane] = acc[q];
            }
            __syncwarp();
            store_chunk(args, staging, m0 + c0, crow, ew, lane, col);
            __syncwarp();
          }
          if (threadIdx.x == 64) args.counters[t * 2 + rank] = 0;
        }
        epi_bar_sync();
      }
    }
  }

  __syncwarp();
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_2sm(tmem_base, L::kTmemCols);
  }
}

template <int TN, int STAGES>
int32_t launch2(const CUtensorMap* tw, const CUtensorMap* tx, const Gemm2Args& a, int n_sms,
                cudaStream_t stream) {
  using L = G2<TN, STAGES>;
  auto kern = gemm_bf16_2sm<TN, STAGES>;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kTotal) !=
        cudaSuccess)
      return CORTEX_ECUDA;
    configured = true;
  }
  const int units = a.num_tiles * a.splits;
  const int pairs = units < n_sms / 2 ? units : n_sms / 2;
  kern<<<2 * pairs, kThreads2, L::kTotal, stream>>>(*tw, *tx, a);
  CORTEX_CHECK_LAUNCH();
  return CORTEX_OK;
}

int g_num_sms = 0;

}  // namespace

// Tile width (m) and K splits the 2-SM GEMM uses for a problem: fewest waves of
// work units x (per-unit MMA time + overhead), a split costing ~10 % for its fix-up.
void cortex_gemm2_plan(int M, int N, int K, int n_sms, int* tn_out, int* splits_out) {
  const int n_tiles = N / kPairN;
  const int pairs = n_sms / 2;
  const int total_kb = K / kBK;
  double best = -1.0;
  for (int tn : {256, 224, 192, 160, 128, 96, 64}) {
    for (int sp = 1; sp <= kMaxSplits2; ++sp) {
      if (sp > 1 && total_kb / sp < 8) break;
      const long units = static_cast<long>(n_tiles) * ((M + tn - 1) / tn) * sp;
      const long waves = (units + pairs - 1) / pairs;
      const double cost = waves * (tn + 32.0) / sp * (sp > 1 ? 1.1 : 1.0);
      if (best < 0 || cost < best - 1e-9) {
        best = cost;
        *tn_out = tn;
        *splits_out = sp;
      }
    }
  }
}

int32_t cortex_gemm_2sm_launch(const void* tmap_w, const void* tmap_x, int32_t M, int32_t N,
                               int32_t K, void* out, int32_t ldo, int32_t out_f32,
                               const void* residual, int32_t ldr, float* workspace,
                               uint64_t workspace_bytes, int32_t* counters, int32_t n_counters,
                               cudaStream_t stream) {
  if (N % kPairN || K % kBK || M <= 0) return CORTEX_EBADARG;
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms < 2) g_num_sms = 148;
  }
  int tn = 256, splits = 1;
  cortex_gemm2_plan(M, N, K, g_num_sms, &tn, &splits);
  const int m_tiles = (M + tn - 1) / tn;
  const int num_tiles = (N / kPairN) * m_tiles;
  if (splits > 1 && (!workspace || !counters ||
                     workspace_bytes < static_cast<uint64_t>(splits) * M * N * sizeof(float) ||
                     n_counters < 2 * num_tiles))
    splits = 1;
  Gemm2Args a{};
  a.M = M;
  a.N = N;
  a.K = K;
  a.out = out;
  a.ldo = ldo;
  a.out_f32 = out_f32;
  a.residual = reinterpret_cast<const float*>(residual);
  a.ldr = ldr;
  a.m_tiles = m_tiles;
  a.num_tiles = num_tiles;
  a.splits = splits;
  a.kb_per_split = (K / kBK + splits - 1) / splits;
  a.workspace = workspace;
  a.counters = counters;
  const auto* tw = reinterpret_cast<const CUtensorMap*>(tmap_w);
  const auto* tx = reinterpret_cast<const CUtensorMap*>(tmap_x);
  switch (tn) {
    case 64: return launch2<64, 8>(tw, tx, a, g_num_sms, stream);
    case 96: return launch2<96, 8>(tw, tx, a, g_num_sms, stream);
    case 128: return launch2<128, 7>(tw, tx, a, g_num_sms, stream);
    case 160: return launch2<160, 7>(tw, tx, a, g_num_sms, stream);
    case 192: return launch2<192, 6>(tw, tx, a, g_num_sms, stream);
    case 224: return launch2<224, 6>(tw, tx, a, g_num_sms, stream);
    default: return launch2<256, 5>(tw, tx, a, g_num_sms, stream);
  }
}
