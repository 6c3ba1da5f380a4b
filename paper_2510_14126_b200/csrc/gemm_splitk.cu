// Decode-sized projections: 2-SM tcgen05 GEMM, split-K over CTA pairs synchronised
// through global flags.
//
//   C[m, n] = sum_k X[m, k] * W[n, k]        (+ residual[m, n], fp32)
//
// At decode batch sizes (M <= 256 tokens) a projection streams its weights once per
// step and the limit is how fast the SMs can ingest them. Two things keep the weight
// stream at full rate here:
//   * all M tokens form ONE MMA N tile (TN >= M), so each weight byte is fetched once
//     (tiling M into several narrow tiles re-reads the weights per tile), and each CTA
//     of a pair stages only TN/2 token rows per 64-wide K block next to its 128 weight
//     rows (cta_group::2, M = 256), which keeps the activation share of every CTA's
//     TMA ingest low;
//   * the N = 4096 / 6144 projections have too few 256-row tiles (16 / 24) to occupy
//     148 SMs, so each tile's K range is split over `ks` pairs, up to 74 pairs (148
//     CTAs) in one wave. Every CTA writes its fp32 partial [TN tokens][128 rows] to a
//     workspace slot and publishes it with a release store of the launch's epoch into
//     its flag; then the pair of split s waits (acquire) for the flags of the tile's
//     other splits and reduces token rows [s * R, (s + 1) * R) of the tile over all
//     splits in split order (deterministic), adds the residual and stores — the
//     reduction is spread over all CTAs instead of serialised on one. (The first
//     version synchronised the splits with a cluster barrier, clusters of 2 ks CTAs:
//     the GPCs hold only 16 clusters of 6 / 37 of 4, so qkv / o / down ran on 96 of
//     148 SMs; with flags every pair is an independent 2-CTA cluster.) All pairs of a
//     launch are co-resident (grid <= 148 CTAs, one per SM), so a waiting CTA never
//     keeps a producer from being scheduled.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "pair.cuh"

#ifndef CORTEX_G2_DEEP  // one more pipeline stage where shared memory allows (0: the round-1 depths;
                        // benchmarks/gemm.py: 1-3.5 % faster at M = 204 ... 2048)
#define CORTEX_G2_DEEP 1
#endif

namespace {

constexpr int kPairN = 256;
constexpr int kBK = 64;
constexpr int kXBox = CORTEX_XBOX;
constexpr int kThreads = 192;

struct SkArgs {
  int M, N, K;
  void* out;
  int ldo;
  int out_f32;  // 0 bf16, 1 fp32, 2 fused SwiGLU (bf16 [M, N/2])
  const float* residual;
  int ldr;
  int ks;       // K splits per tile (= pairs per cluster)
  int kb_per;   // K blocks per split
  int m_tiles;
  float* ws;    // [tiles][ks][2][TN][128] fp32 partials
  int* flags;   // [tiles][ks][2] split-published flags (epoch values)
  uint32_t epoch;  // this launch's flag value (strictly increasing per launch)
  int n_issue;  // TMA issuing threads: 1, 2 (weights | tokens) or 4 (two of each)
  int l2pf;     // weight K blocks prefetched into L2 beyond the stages, before the PDL wait
  RopeEpi rope;  // out mode 4 (QKV: RoPE + paged KV append in the epilogue)
};

// NW weight sub-tiles of 256 rows per pair (one MMA each, sharing the staged token rows):
// NW = 2 halves the token rows' share of a CTA's ingest for the wide projections.
template <int TN, int STAGES, int NW>
struct SkL {
  static constexpr int kA1 = 128 * kBK * 2;  // one sub-tile's 128 rows in this CTA
  static constexpr int kA = NW * kA1;
  static constexpr int kB = (TN / 2) * kBK * 2;
  static constexpr int kStage = kA + kB;
  static constexpr int kBar = STAGES * kStage;
  static constexpr int kTotal = kBar + 256 + 1024;
  static constexpr uint32_t kTmemCols = NW * TN <= 128 ? 128 : (NW * TN <= 256 ? 256 : 512);
};

CORTEX_DEVICE uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;\n" : "=r"(r));
  return r;
}

// Rows [r_lo, r_hi) of this CTA's 128 output columns: sum of the KS split partials in split
// order (+ residual), then the epilogue. All threads of the CTA take part; a warp covers one
// 128-column row (lane -> 4 columns) and every thread keeps 8 rows' loads of all splits in
// flight before it adds (the partials come from L2: latency, not bandwidth, is the limit).
template <int KS>
CORTEX_DEVICE void reduce_rows(const SkArgs& args, const float* base, size_t split_stride,
                               int r_lo, int r_hi, int m0, int n0) {
  constexpr int kB = 8;
  const int lane = lane_id();
  const int nw = blockDim.x / 32;
  const bool swiglu = args.out_f32 == 2;
  const bool res = args.residual != nullptr && !swiglu;
  const int col = n0 + 4 * lane;
  for (int rb = r_lo + warp_id(); rb < r_hi; rb += nw * kB) {
    float4 p[KS][kB];
    float4 acc[kB];
    RopeRow rr[kB];
#pragma unroll
    for (int i = 0; i < kB; ++i) {
      const int r = rb + i * nw;
      acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r < r_hi && args.out_f32 == 4) rr[i] = rope_fetch(args.rope, m0 + r, n0 / 128);
      if (r < r_hi) {
#pragma unroll
        for (int q = 0; q < KS; ++q)
          p[q][i] = __ldcg(reinterpret_cast<const float4*>(base + q * split_stride +
                                                           static_cast<size_t>(r) * 128) + lane);
        if (res)  // (out may alias the residual: no .nc)
          acc[i] = *reinterpret_cast<const float4*>(args.residual +
                                                    static_cast<size_t>(m0 + r) * args.ldr + col);
      }
    }
#pragma unroll
    for (int i = 0; i < kB; ++i) {
      const int r = rb + i * nw;
      if (r >= r_hi) break;  // (warp-uniform)
      float4 sum = p[0][i];
#pragma unroll
      for (int q = 1; q < KS; ++q) {
        sum.x += p[q][i].x;
        sum.y += p[q][i].y;
        sum.z += p[q][i].z;
        sum.w += p[q][i].w;
      }
      if (args.out_f32 == 4) {  // QKV: the 128 columns are one head
        rope_store_row(args.rope, rr[i], m0 + r, n0 / 128, sum);
        continue;
      }
      if (swiglu) {  // lanes 0-15 hold gate features, 16-31 the matching ups
        const float ux = __shfl_down_sync(0xffffffffu, sum.x, 16);
        const float uy = __shfl_down_sync(0xffffffffu, sum.y, 16);
        const float uz = __shfl_down_sync(0xffffffffu, sum.z, 16);
        const float uw = __shfl_down_sync(0xffffffffu, sum.w, 16);
        if (lane < 16) {
          uint2 packed;
          packed.x = pack_bf16(sum.x / (1.f + __expf(-sum.x)) * ux,
                               sum.y / (1.f + __expf(-sum.y)) * uy);
          packed.y = pack_bf16(sum.z / (1.f + __expf(-sum.z)) * uz,
                               sum.w / (1.f + __expf(-sum.w)) * uw);
          *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(args.out) +
                                    static_cast<size_t>(m0 + r) * args.ldo + n0 / 2 + 4 * lane) =
              packed;
        }
        continue;
      }
      const float4 o = make_float4(sum.x + acc[i].x, sum.y + acc[i].y, sum.z + acc[i].z,
                                   sum.w + acc[i].w);
      const size_t off = static_cast<size_t>(m0 + r) * args.ldo + col;
      if (args.out_f32) {
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(args.out) + off) = o;
      } else {
        uint2 packed;
        packed.x = pack_bf16(o.x, o.y);
        packed.y = pack_bf16(o.z, o.w);
        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(args.out) + off) = packed;
      }
    }
  }
}

// Tuning builds (-DCORTEX_SK_TRACE): globaltimer stamps per CTA into the workspace tail
// ([cta][8] u64 at float offset 15 Mi): 0 start, 1 setup done, 2 accumulator ready,
// 3 partial written, 4 after the cluster barrier, 5 reduced.
#ifdef CORTEX_SK_TRACE
#define SK_TRACE(ev)                                                                     \
  do {                                                                                   \
    if (threadIdx.x == 64) {                                                             \
      uint64_t t_;                                                                       \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                             \
      reinterpret_cast<uint64_t*>(args.ws + (15u << 20))[blockIdx.x * 8 + (ev)] = t_;     \
    }                                                                                    \
  } while (0)
#else
#define SK_TRACE(ev) \
  do {               \
  } while (0)
#endif

template <int TN, int STAGES, int NW>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_2sm_splitk(const __grid_constant__ CUtensorMap tmap_w,
                         const __grid_constant__ CUtensorMap tmap_x, const SkArgs args) {
  using L = SkL<TN, STAGES, NW>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tfull + 1);

  const uint32_t rank = cluster_rank();  // CTA within the pair (the cluster)
  const uint32_t lead = 0;               // the pair leader's cluster rank
  const int pair_id = static_cast<int>(blockIdx.x >> 1);
  const int split = pair_id % args.ks;
  const int tile = pair_id / args.ks;
  const int n_tile = tile / args.m_tiles;
  const int m_tile = tile % args.m_tiles;
  const int total_kb = args.K / kBK;
  const int kb0 = split * args.kb_per;
  const int kb1 = min(total_kb, kb0 + args.kb_per);
  const int warp = warp_id();
  const int lane = lane_id();
  SK_TRACE(0);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_w);
    tma_prefetch_desc(&tmap_x);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 2);   // leader's expect_tx arrive + the peer's arrive
      mbar_init(&empty[s], 1);  // multicast MMA commit
    }
    mbar_init(tfull, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_2sm(tmem_holder, L::kTmemCols);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  SK_TRACE(1);
  const uint16_t pair_mask = static_cast<uint16_t>(3u << lead);

  // ---- TMA issuers. The copies one thread issues complete one after another, so the
  // weight boxes and the token-row boxes of a stage come from different warps, and with
  // n_issue = 4 successive stages alternate between two issuers of each kind
  // (benchmarks/micro/tma_tile.cu): warps 0 / 3 weights, warps 2 / 4 token rows (the
  // epilogue warps 2-4 are idle until the accumulator is ready). The weight issuer of a
  // stage arms its barrier; token-row bytes may land first (transiently negative count).
  const int n_w = args.n_issue >= 4 ? 2 : 1;
  const int w_idx = warp == 0 ? 0 : (warp == 3 && n_w == 2 ? 1 : -1);
  const int x_idx = args.n_issue == 1 ? (warp == 0 ? 0 : -1)
                                      : (warp == 2 ? 0 : (warp == 4 && n_w == 2 ? 1 : -1));
  // The weights are immutable: a weights-only issuer fills the pipeline while the
  // previous kernel of the stream is still running, and waits for it afterwards (its
  // warp may drain partials into the workspace the previous kernel reads). Everyone
  // else waits first: the activations (and residual) come from that kernel.
  const bool w_only = w_idx >= 0 && x_idx < 0;
  if (!w_only) pdl_wait();
  pdl_trigger();
  if ((w_idx >= 0 || x_idx >= 0) && elect_one()) {
    const int n0 = n_tile * kPairN * NW + static_cast<int>(rank) * 128;
    if (w_idx == 0 && w_only) {
      // the K blocks after the first STAGES: into L2 while the predecessor runs
      const int pf1 = min(kb1, kb0 + STAGES + args.l2pf);
      for (int kb = kb0 + STAGES; kb < pf1; ++kb)
#pragma unroll
        for (int w = 0; w < NW; ++w) tma_prefetch_l2_2d(&tmap_w, kb * kBK, n0 + w * kPairN);
    }
    const int x0 = m_tile * TN + static_cast<int>(rank) * (TN / 2);
    const uint64_t pol_w = policy_evict_first();  // weights: streamed once per step
    for (int kb = kb0, it = 0; kb < kb1; ++kb, ++it) {
      const bool do_w = w_idx >= 0 && it % n_w == w_idx;
      const bool do_x = x_idx >= 0 && (args.n_issue == 1 || it % n_w == x_idx);
      if (!do_w && !do_x) continue;
      const int s = it % STAGES;
      const uint32_t ph = (it / STAGES) & 1;
      mbar_wait(&empty[s], ph ^ 1);
      const uint32_t full_leader = mapa_shared(smem_u32(&full[s]), lead);
      uint8_t* sa = smem + s * L::kStage;
      uint8_t* sb = sa + L::kA;
      const int kc = kb * kBK;
      if (do_w) {
        if (rank == 0)
          mbar_arrive_expect_tx(&full[s], 2 * L::kStage);
        else
          mbar_arrive_cluster(full_leader);
#pragma unroll
        for (int w = 0; w < NW; ++w)
          asm volatile(
              "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx"
              "::bytes.L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;\n" ::"r"(
                  smem_u32(sa + w * L::kA1)),
              "l"(reinterpret_cast<uint64_t>(&tmap_w)), "r"(full_leader), "r"(kc),
              "r"(n0 + w * kPairN), "l"(pol_w)
              : "memory");
      }
      if (do_x) {
#pragma unroll
        for (int j = 0; j < TN / 2 / kXBox; ++j)
          tma_load_2d_2sm(sb + j * kXBox * 128, &tmap_x, full_leader, kc, x0 + j * kXBox);
      }
    }
  }
  if (warp == 1) {
    if (rank == 0 && elect_one()) {
      // ---- MMA issuer (pair leader, one thread) ----
      constexpr uint32_t idesc = umma_idesc_bf16(kPairN, TN);
      for (int kb = kb0, it = 0; kb < kb1; ++kb, ++it) {
        const int s = it % STAGES;
        const uint32_t ph = (it / STAGES) & 1;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t a_addr = smem_u32(smem + s * L::kStage);
        const uint32_t b_addr = a_addr + L::kA;
#pragma unroll
        for (int w = 0; w < NW; ++w)
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)
            umma_bf16_ss_2sm(tmem_base + w * TN, umma_desc_sw128(a_addr + w * L::kA1 + k * 32),
                             umma_desc_sw128(b_addr + k * 32), idesc,
                             (kb != kb0 || k != 0) ? 1u : 0u);
        umma_commit_2sm_mask(&empty[s], pair_mask);
      }
      umma_commit_2sm_mask(tfull, pair_mask);
    }
  }

  if (w_only) pdl_wait();
  __syncwarp();  // reconverge the issuing lanes before the warp-collective TMEM loads
  const int m0 = m_tile * TN;
  const int rows = min(TN, args.M - m0);
  // this CTA's partials: NW x [TN tokens][128 weight rows] fp32
  const size_t tile_slot = static_cast<size_t>(tile) * args.ks;
  const size_t part = static_cast<size_t>(TN) * 128;
  float* mine = args.ws + ((tile_slot + split) * 2 + rank) * NW * part;
  if (warp >= 2) {
    // ---- drain the partial: TMEM lane quadrant = warp % 4 ----
    const int quad = warp & 3;
    mbar_wait(tfull, 0);
    tc_fence_after();
    SK_TRACE(2);
    for (int w = 0; w < NW; ++w) {
      const uint32_t taddr = tmem_base + w * TN + (static_cast<uint32_t>(quad * 32) << 16);
      float* dst = mine + w * part + quad * 32 + lane;
      for (int c0 = 0; c0 < rows; c0 += 32) {
        uint32_t r0[16], r1[16];
        tmem_ld_32x32b_x16(taddr + c0, r0);
        tmem_ld_32x32b_x16(taddr + c0 + 16, r1);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          __stcg(dst + static_cast<size_t>(c0 + j) * 128, __uint_as_float(r0[j]));
          __stcg(dst + static_cast<size_t>(c0 + 16 + j) * 128, __uint_as_float(r1[j]));
        }
      }
    }
  }
  // every split's partial is in the workspace before any pair reduces: publish this
  // CTA's partial (release, gpu scope, after the CTA barrier), then acquire the other
  // splits' flags for this rank's 128 columns
  SK_TRACE(3);
  tc_fence_before();
  __syncthreads();
  int* tflags = args.flags + static_cast<size_t>(tile) * args.ks * 2;
  if (threadIdx.x == 0) {
    __threadfence();
    st_release_gpu_u32(tflags + split * 2 + rank, args.epoch);
  }
  if (threadIdx.x < args.ks && static_cast<int>(threadIdx.x) != split)
    wait_flag_gpu(tflags + threadIdx.x * 2 + rank, args.epoch);
  __syncthreads();
  SK_TRACE(4);

  {
    // ---- reduce token rows [r_lo, r_hi) over the ks splits (split order), epilogue ----
    const int R = ((rows + args.ks - 1) / args.ks + 3) & ~3;
    const int r_lo = split * R;
    const int r_hi = min(rows, r_lo + R);
    for (int w = 0; w < NW; ++w) {
      const float* base = args.ws + (tile_slot * 2 + rank) * NW * part + w * part;
      const int n0 = (n_tile * NW + w) * kPairN + static_cast<int>(rank) * 128;
      const size_t stride = 2 * NW * part;  // between splits
      switch (args.ks) {
        case 1: reduce_rows<1>(args, base, stride, r_lo, r_hi, m0, n0); break;
        case 2: reduce_rows<2>(args, base, stride, r_lo, r_hi, m0, n0); break;
        case 3: reduce_rows<3>(args, base, stride, r_lo, r_hi, m0, n0); break;
        default: reduce_rows<4>(args, base, stride, r_lo, r_hi, m0, n0); break;
      }
    }
  }

  SK_TRACE(5);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_2sm(tmem_base, L::kTmemCols);
  }
}

template <int TN, int STAGES, int NW>
int32_t launch_sk(const CUtensorMap* tw, const CUtensorMap* tx, const SkArgs& a, int n_clusters,
                  cudaStream_t stream) {
  using L = SkL<TN, STAGES, NW>;
  auto kern = gemm_bf16_2sm_splitk<TN, STAGES, NW>;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kTotal) !=
        cudaSuccess)
      return CORTEX_ECUDA;
    configured = true;
  }
  if (pdl_launch(kern, n_clusters * 2 * a.ks, kThreads, L::kTotal, stream, 2, *tw, *tx, a) !=
      cudaSuccess)
    return CORTEX_ECUDA;
  return CORTEX_OK;
}

}  // namespace

extern "C" {

// Plan of the split-K kernel for (M, N, K): returns ks (>= 2) and writes the token tile
// TN and the number of token tiles, or returns 0 when the problem should use another
// kernel. The split count depends on N and K only, so within the regime a token's result
// does not depend on the batch it is in (the K split points are fixed; the tile width
// does not change a dot product's summation order):
//   * tiles x ks pairs must run as one co-resident wave (<= 74 pairs, 148 CTAs): the
//     largest ks <= 4 that fits (o / down: 16 tiles -> ks 4, 64 pairs; qkv: 24 -> ks 3,
//     72 pairs);
//   * the fp32 partials (ks x M x N x 4 bytes) must stay small next to the weights.
// Measured at M = 16 ... 256 (benchmarks/gemm_sk_sweep.py): 0.7-0.85x the time of the
// whole-tile 2-SM kernel for o / down / qkv, 0.45-0.6x the 1-SM split-K kernel.
int32_t cortex_gemm_splitk_plan(int32_t M, int32_t N, int32_t K, int32_t* tn_out,
                                int32_t* mt_out, int32_t* nw_out) {
  const int g_sk_mt_force = g_cortex_knob[CORTEX_KNOB_SK_MT];
  const int g_sk_ks_force = g_cortex_knob[CORTEX_KNOB_SK_KS];
  const int g_sk_nw_force = g_cortex_knob[CORTEX_KNOB_SK_NW];
  if (M <= 0 || M > 256 || N % kPairN || K % kBK) return 0;
  const int total_kb = K / kBK;
  const int mt = g_sk_mt_force > 0 ? g_sk_mt_force : 1;
  int tn = ((M + mt - 1) / mt + 31) / 32 * 32;
  if (tn < 64) tn = 64;
  if ((mt - 1) * tn >= M) return 0;  // an empty token tile
  int ks = 0, nw = 1;
  const int tiles = N / kPairN;
  if (g_sk_ks_force > 0) {
    ks = g_sk_ks_force;
    if (tiles * mt * ks > 74) return 0;
  } else {
    ks = 4;
    while (ks >= 2 && tiles * mt * ks > 74) --ks;
    while (ks >= 2 && 2 * ks * tn * mt > K) --ks;  // partials <= weights / 2
    if (ks < 2) ks = 0;
    // (wide projections such as gate_up - 112 tiles - stay on the persistent 2-SM kernel:
    // at M ~ 200 they are compute-bound, and a one-wave plan with two weight sub-tiles per
    // pair (nw = 2, 56 pairs) measured 70 us vs 57 us on all 148 SMs)
    if (g_sk_nw_force == 2 && N % (2 * kPairN) == 0 && (N / (2 * kPairN)) * mt <= 74) {
      nw = 2;
      ks = 1;
    }
  }
  if (ks < 1 || (ks - 1) * ((total_kb + ks - 1) / ks) >= total_kb) return 0;  // empty split
  if (tn_out) *tn_out = tn;
  if (mt_out) *mt_out = mt;
  if (nw_out) *nw_out = nw;
  return ks;
}

int32_t cortex_gemm_splitk_launch(const void* tmap_w, const void* tmap_x, int32_t M, int32_t N,
                                  int32_t K, void* out, int32_t ldo, int32_t out_f32,
                                  const void* residual, int32_t ldr, float* workspace,
                                  uint64_t workspace_bytes, int32_t* counters,
                                  int32_t n_counters, const RopeEpi* rope, cudaStream_t stream) {
  int tn = 0, mt = 1, nw = 1;
  const int ks = cortex_gemm_splitk_plan(M, N, K, &tn, &mt, &nw);
  if (ks < 1 || !workspace || !counters || n_counters < 1024 || (out_f32 == 4 && !rope))
    return CORTEX_EBADARG;
  const int total_kb = K / kBK;
  const int tiles = N / (kPairN * nw) * mt;
  if (workspace_bytes < static_cast<uint64_t>(tiles) * ks * 2 * nw * tn * 128 * sizeof(float))
    return CORTEX_EBADARG;
  SkArgs a{};
  a.M = M;
  a.N = N;
  a.K = K;
  a.out = out;
  a.ldo = ldo;
  a.out_f32 = out_f32;
  a.residual = reinterpret_cast<const float*>(residual);
  a.ldr = ldr;
  a.ks = ks;
  a.kb_per = (total_kb + ks - 1) / ks;
  a.m_tiles = mt;
  a.ws = workspace;
  // split flags: the last 512 counters (the 1-SM kernel's tile counters use the first
  // n_tiles); a strictly increasing epoch per launch means they never need resetting
  static uint32_t epoch = 0;
  epoch = epoch == 0x7fffffffu ? 1u : epoch + 1u;
  a.flags = counters + (n_counters - 512);
  a.epoch = epoch;
  if (tiles * ks * 2 > 512) return CORTEX_EBADARG;
  // TMA issuers (knob SK_ISSUE, default 2: 1, 2 and 4 issuers measured within noise of
  // each other at M = 64 ... 256 - the decode GEMMs are bound by L2 throughput, weights
  // plus the token rows every weight tile re-reads, not by TMA issue)
  a.n_issue = g_cortex_knob[CORTEX_KNOB_SK_ISSUE];
  a.l2pf = g_cortex_knob[CORTEX_KNOB_GEMM_L2PF];
  if (rope) a.rope = *rope;
  const auto* tw = reinterpret_cast<const CUtensorMap*>(tmap_w);
  const auto* tx = reinterpret_cast<const CUtensorMap*>(tmap_x);
  if (nw == 2) {
    switch (tn) {
      case 64: return launch_sk<64, 5, 2>(tw, tx, a, tiles, stream);
      case 96: return launch_sk<96, 5, 2>(tw, tx, a, tiles, stream);
      case 128: return launch_sk<128, 4, 2>(tw, tx, a, tiles, stream);
      case 160: return launch_sk<160, 4, 2>(tw, tx, a, tiles, stream);
      case 192: return launch_sk<192, 4, 2>(tw, tx, a, tiles, stream);
      case 224: return launch_sk<224, 4, 2>(tw, tx, a, tiles, stream);
      default: return launch_sk<256, 4, 2>(tw, tx, a, tiles, stream);
    }
  }
  switch (tn) {
    case 64: return launch_sk<64, 8, 1>(tw, tx, a, tiles, stream);
    case 96: return launch_sk<96, 8, 1>(tw, tx, a, tiles, stream);
    case 128: return launch_sk<128, 8, 1>(tw, tx, a, tiles, stream);
    case 160: return launch_sk<160, 6 + CORTEX_G2_DEEP, 1>(tw, tx, a, tiles, stream);
    case 192: return launch_sk<192, 6 + CORTEX_G2_DEEP, 1>(tw, tx, a, tiles, stream);
    case 224: return launch_sk<224, 6 + CORTEX_G2_DEEP, 1>(tw, tx, a, tiles, stream);
    default: return launch_sk<256, 6 + CORTEX_G2_DEEP, 1>(tw, tx, a, tiles, stream);
  }
}

}  // extern "C"
