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
//
// Stream-K mode (when tiles do not fill whole waves of pairs, e.g. the N = 4096
// projections at M ~ 700: 64 tiles for 74 pairs): the tiles' K blocks are laid
// end to end and pair p takes the contiguous range [p U / P, (p+1) U / P) of the
// U = tiles x K-blocks units, so every pair does the same MMA work. A pair whose
// range starts inside a tile writes that partial accumulator to a per-pair
// workspace slot and raises a flag; the pair holding the tile's first K blocks
// (it reaches them last) waits for the flags and adds the partials in pair order
// (deterministic) before its epilogue. Pairs only ever wait on later pairs'
// first segments, which those pairs compute first, so the grid (all pairs
// resident) cannot deadlock.
#include <cstdlib>

#include "common.cuh"
#include "pair.cuh"

#ifndef CORTEX_G2_DEEP  // one more pipeline stage where shared memory allows (0: the round-1 depths;
                        // benchmarks/gemm.py: 1-3.5 % faster at M = 204 ... 2048)
#define CORTEX_G2_DEEP 1
#endif

namespace {

constexpr int kPairN = 256;  // weight rows per CTA pair (MMA M)
constexpr int kBK = 64;
constexpr int kXBox2 = CORTEX_XBOX;  // activation rows per TMA box
constexpr int kEpiRows = 32; // output rows (m) per epilogue chunk
constexpr int kThreads2 = 224;  // warps: 0 TMA (weights), 1 MMA, 2-5 epilogue, 6 TMA (tokens)
struct Gemm2Args {
  int M, N, K;
  void* out;
  int ldo;
  int out_f32;
  const float* residual;
  int ldr;
  int m_tiles;
  int num_tiles;
  int npairs;        // persistent CTA pairs (grid / 2)
  int sk;            // 1: stream-K ranges, 0: whole tiles round-robin
  int total_units;   // num_tiles * K blocks
  float* workspace;  // stream-K: [npairs * 2][TN][128] fp32 partials
  int* flags;        // stream-K: [npairs * 2] partial-ready flags, left zeroed
  int l2pf;          // weight K blocks prefetched into L2 beyond the stages (first segment)
  RopeEpi rope;      // out mode 4 (QKV: RoPE + paged KV append in the epilogue)
};

struct Seg {
  int t, kb0, kb1;  // tile, K-block range
};

CORTEX_DEVICE int sk_begin(const Gemm2Args& a, int p) {
  return static_cast<int>(static_cast<long long>(p) * a.total_units / a.npairs);
}

// Next segment of a pair's work; `pos` starts at seg_start() and is advanced.
CORTEX_DEVICE int seg_start(const Gemm2Args& a, int pair) { return a.sk ? sk_begin(a, pair) : pair; }

CORTEX_DEVICE bool seg_next(const Gemm2Args& a, int pair, int& pos, Seg& g) {
  const int tkb = a.K / kBK;
  if (!a.sk) {
    if (pos >= a.num_tiles) return false;
    g.t = pos;
    g.kb0 = 0;
    g.kb1 = tkb;
    pos += a.npairs;
    return true;
  }
  const int end = sk_begin(a, pair + 1);
  if (pos >= end) return false;
  g.t = pos / tkb;
  g.kb0 = pos % tkb;
  g.kb1 = min(tkb, g.kb0 + (end - pos));
  pos += g.kb1 - g.kb0;
  return true;
}

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

CORTEX_DEVICE int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

CORTEX_DEVICE void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

CORTEX_DEVICE float4 ws_load(const float4* p) { return __ldcg(p); }

// Tuning builds (-DCORTEX_GEMM_TRACE): globaltimer stamps of the epilogue's segment
// events into the tail of the workspace: [pair][rank][16] u64 at float offset 15 Mi.
#ifdef CORTEX_GEMM_TRACE
#define GEMM_TRACE(ev)                                                                       \
  do {                                                                                      \
    if (threadIdx.x == 64 && (ev) < 16) {                                                   \
      uint64_t t_;                                                                          \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                \
      reinterpret_cast<uint64_t*>(args.workspace + (15u << 20))[(2 * pair + rank) * 16 + (ev)] = \
          t_;                                                                               \
    }                                                                                       \
  } while (0)
#else
#define GEMM_TRACE(ev) \
  do {                 \
  } while (0)
#endif

CORTEX_DEVICE void epi_bar_sync() { asm volatile("bar.sync 1, 128;\n" ::: "memory"); }

// Rows ew, ew+4, ... < crow of a staged fp32 chunk -> (+ fp32 residual) -> bf16 / fp32 out.
// Each warp covers one 128-column row with 16-byte accesses; all loads before any store
// (out may alias the residual).
CORTEX_DEVICE void store_chunk(const Gemm2Args& args, const float* staging, int mrow0, int crow,
                               int ew, int lane, int col, const RopeRow* rr) {
  if (args.out_f32 == 4) {  // QKV: this CTA's 128 columns are one head
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int r = ew + 4 * q;
      if (r < crow)  // (warp-uniform)
        rope_store_row(args.rope, rr[q], mrow0 + r, (col - 4 * lane) / 128,
                       reinterpret_cast<const float4*>(staging + r * 128)[lane]);
    }
    return;
  }
  if (args.out_f32 == 3) {  // greedy-token partials: (max, index) of this CTA's 128 columns
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int r = ew + 4 * q;
      if (r < crow)  // (warp-uniform)
        store_argmax_partial(reinterpret_cast<float2*>(args.out), args.ldo, mrow0 + r,
                             col - 4 * lane, reinterpret_cast<const float4*>(staging + r * 128)[lane],
                             col);
    }
    return;
  }
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
  const int warp = warp_id();
  const int lane = lane_id();
  const int total_kb = args.K / kBK;
  GEMM_TRACE(15);

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
  // The weights are immutable: their producer (warp 0) fills the pipeline while the
  // previous kernel of the stream is still running; everyone else waits for it first
  // (the activations and residual come from it, and the outputs may alias its inputs).
  if (warp != 0) pdl_wait();
  pdl_trigger();

  if (warp == 0) {
    if (elect_one()) {
      // ---- TMA producer, weights (both CTAs load their halves; warp 6 the tokens) ----
      uint32_t it = 0;
      int pos = seg_start(args, pair);
      Seg g;
      bool first = true;
      while (seg_next(args, pair, pos, g)) {
        const int n_tile = g.t / args.m_tiles;
        const int m_tile = g.t % args.m_tiles;
        (void)m_tile;
        const int n0 = n_tile * kPairN + rank * 128;
        if (first) {  // the K blocks after the first STAGES: into L2 before the wait
          const int pf1 = min(g.kb1, g.kb0 + STAGES + args.l2pf);
          for (int kb = g.kb0 + STAGES; kb < pf1; ++kb) tma_prefetch_l2_2d(&tmap_w, kb * kBK, n0);
          first = false;
        }
        for (int kb = g.kb0; kb < g.kb1; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          const uint32_t full_leader = mapa_shared(smem_u32(&full[s]), 0);
#if defined(CORTEX_G2_NOFEED)  // tuning builds only: MMA issue rate without operand traffic
          if (it >= STAGES) {
            if (leader)
              mbar_arrive(&full[s]);
            else
              mbar_arrive_cluster(full_leader);
            continue;
          }
#endif
#if defined(CORTEX_G2_NOFEED) || defined(CORTEX_G2_NOFEED_X)
          constexpr uint32_t kExpect = 2 * L::kA;  // the weights only
#else
          constexpr uint32_t kExpect = 2 * L::kStage;
#endif
          if (leader)
            mbar_arrive_expect_tx(&full[s], kExpect);
          else
            mbar_arrive_cluster(full_leader);
          tma_load_2d_2sm(smem + s * L::kStage, &tmap_w, full_leader, kb * kBK, n0);
        }
      }
    }
    pdl_wait();  // nothing below touches memory, but keep every thread ordered
  } else if (warp == 6) {
    if (elect_one()) {
      // ---- second TMA issuer: the token rows. A TMA-issuing thread's copies complete
      // one after another, so two issuers keep more bytes in flight per SM
      // (benchmarks/micro/tma_tile.cu: 235 MB of weights in 47 us with one issuer,
      // 40 us with two). The stage's expected bytes were armed by warp 0 (or are
      // counted before the arm: the transaction count may go transiently negative).
#if defined(CORTEX_G2_NOFEED) || defined(CORTEX_G2_NOFEED_X)
      constexpr bool kFeedX = false;
#else
      constexpr bool kFeedX = true;
#endif
      uint32_t it = 0;
      int pos = seg_start(args, pair);
      Seg g;
      while (kFeedX && seg_next(args, pair, pos, g)) {
        const int m_tile = g.t % args.m_tiles;
        const int x0 = m_tile * TN + rank * (TN / 2);
        for (int kb = g.kb0; kb < g.kb1; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          const uint32_t full_leader = mapa_shared(smem_u32(&full[s]), 0);
          uint8_t* sb = smem + s * L::kStage + L::kA;
          const int kc = kb * kBK;
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
      int pos = seg_start(args, pair);
      Seg g;
      for (; seg_next(args, pair, pos, g); ++tl) {
        const int kb0 = g.kb0, kb1 = g.kb1;
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
  } else if (warp < 6) {
    // ---- epilogue warps 2..5: TMEM lane quadrant = warp % 4 ----
    const int quad = warp & 3;
    const int ew = warp - 2;  // 0..3
    const uint32_t tempty_leader_base = mapa_shared(smem_u32(&tempty[0]), 0);
    uint32_t tl = 0;
    int pos = seg_start(args, pair);
    Seg g;
    for (; seg_next(args, pair, pos, g); ++tl) {
      const int t = g.t;
      const uint32_t b = tl & 1;
      const uint32_t tph = (tl >> 1) & 1;
      const int n_tile = t / args.m_tiles;
      const int m_tile = t % args.m_tiles;
      const int n0 = n_tile * kPairN + rank * 128;
      const int m0 = m_tile * TN;
      const int rows = min(TN, args.M - m0);
      const int col = n0 + 4 * lane;
      // stream-K roles: a segment starting inside its tile contributes a partial; the
      // segment with the tile's first K blocks (and not its last) collects them
      const bool contrib = g.kb0 > 0;
      const bool head = g.kb0 == 0 && g.kb1 < total_kb;
      int q_end = pair + 1;
      if (head) {
        while (q_end < args.npairs && sk_begin(args, q_end) < (t + 1) * total_kb) ++q_end;
        if (threadIdx.x == 64) {
          for (int q = pair + 1; q < q_end; ++q) {
            const int* f = args.flags + 2 * q + rank;
            while (ld_acquire_gpu(f) == 0) __nanosleep(64);
          }
        }
        epi_bar_sync();
      }
      if (tl < 2) GEMM_TRACE(4 * static_cast<int>(tl) + 0);
      mbar_wait(&tfull[b], tph);
      if (tl < 2) GEMM_TRACE(4 * static_cast<int>(tl) + 1);
      tc_fence_after();
      const uint32_t taddr = tmem_base + b * TN + (static_cast<uint32_t>(quad * 32) << 16);
      for (int c0 = 0; c0 < rows; c0 += kEpiRows) {
        const int crow = min(kEpiRows, rows - c0);
        // global operands of this chunk first (residual, stream-K partials): their round
        // trip overlaps the TMEM read and the staging transpose
        float4 acc[8];
        RopeRow rr[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (!contrib && args.out_f32 == 4) {
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (ew + 4 * q < crow) rr[q] = rope_fetch(args.rope, m0 + c0 + ew + 4 * q, n0 / 128);
        }
        if (!contrib) {
          if (args.residual && args.out_f32 != 2) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const int r = ew + 4 * q;
              if (r < crow)
                acc[q] = *reinterpret_cast<const float4*>(  // (out may alias: no .nc)
                    args.residual + static_cast<size_t>(m0 + c0 + r) * args.ldr + col);
            }
          }
          if (head) {  // + the later pairs' partials of this tile, in pair order
            for (int qp = pair + 1; qp < q_end; ++qp) {
              const float* ws = args.workspace + static_cast<size_t>(2 * qp + rank) * TN * 128;
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                const int r = ew + 4 * q;
                if (r < crow) {
                  const float4 v = ws_load(reinterpret_cast<const float4*>(
                      ws + static_cast<size_t>(c0 + r) * 128 + 4 * lane));
                  acc[q].x += v.x;
                  acc[q].y += v.y;
                  acc[q].z += v.z;
                  acc[q].w += v.w;
                }
              }
            }
          }
        }
        if (c0 == 0) GEMM_TRACE(8);
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
        if (c0 == 0) GEMM_TRACE(9);
        if (c0 == 32) GEMM_TRACE(10);
        if (contrib) {
          float* ws = args.workspace + static_cast<size_t>(2 * pair + rank) * TN * 128;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int r = ew + 4 * q;
            if (r < crow)
              __stcg(reinterpret_cast<float4*>(ws + static_cast<size_t>(c0 + r) * 128 + 4 * lane),
                     reinterpret_cast<const float4*>(staging + r * 128)[lane]);
          }
        } else if (args.out_f32 >= 2) {  // SwiGLU / argmax read other lanes' columns
          if (head) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const int r = ew + 4 * q;
              if (r < crow) {
                float4& d = reinterpret_cast<float4*>(staging + r * 128)[lane];
                d.x += acc[q].x;
                d.y += acc[q].y;
                d.z += acc[q].z;
                d.w += acc[q].w;
              }
            }
            __syncwarp();
          }
          store_chunk(args, staging, m0 + c0, crow, ew, lane, col, rr);
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int r = ew + 4 * q;
            if (r < crow) {
              const float4 v = reinterpret_cast<const float4*>(staging + r * 128)[lane];
              const float4 o = make_float4(v.x + acc[q].x, v.y + acc[q].y, v.z + acc[q].z,
                                           v.w + acc[q].w);
              const size_t off = static_cast<size_t>(m0 + c0 + r) * args.ldo + col;
              if (args.out_f32) {
                *reinterpret_cast<float4*>(reinterpret_cast<float*>(args.out) + off) = o;
              } else {
                uint2 packed;
                packed.x = pack_bf16(o.x, o.y);
                packed.y = pack_bf16(o.z, o.w);
                *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(args.out) + off) =
                    packed;
              }
            }
          }
        }
        epi_bar_sync();
      }
      // the accumulator is drained: release it to the MMA warp
      tc_fence_before();
      if (lane == 0) mbar_arrive_cluster(tempty_leader_base + b * 8);
      if (contrib) {  // publish the partial
        if (tl < 2) GEMM_TRACE(4 * static_cast<int>(tl) + 2);
        __threadfence();
        epi_bar_sync();
        if (threadIdx.x == 64) st_release_gpu(args.flags + 2 * pair + rank, 1);
        if (tl < 2) GEMM_TRACE(4 * static_cast<int>(tl) + 3);
      } else if (head && threadIdx.x == 64) {
        for (int q = pair + 1; q < q_end; ++q) args.flags[2 * q + rank] = 0;  // consumed
      }
    }
  }

  GEMM_TRACE(13);
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  GEMM_TRACE(14);
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
  Gemm2Args b = a;
  b.npairs = b.sk ? n_sms / 2 : (a.num_tiles < n_sms / 2 ? a.num_tiles : n_sms / 2);
#ifdef CORTEX_GEMM_MAXPAIRS  // (tuning experiment: fewer concurrent pairs)
  if (b.npairs > CORTEX_GEMM_MAXPAIRS) b.npairs = CORTEX_GEMM_MAXPAIRS;
#endif
  if (b.sk && b.total_units < b.npairs) b.npairs = b.total_units;
  if (pdl_launch(kern, 2 * b.npairs, kThreads2, L::kTotal, stream, 1, *tw, *tx, b) !=
      cudaSuccess)
    return CORTEX_ECUDA;
  return CORTEX_OK;
}

int g_num_sms = 0;

}  // namespace

// Tile width (m) and mode the 2-SM GEMM uses for a problem: the lowest modelled
// time over TN of whole tiles (waves x (TN + 32)). Stream-K is only used when forced
// (knob GEMM_STREAM_K = 1): it balances the MMA work, but the head pair's fix-up
// epilogue (reading the partials) measured ~5 us per 32-row chunk at the end of the
// kernel, so e.g. the down projection at M = 700 takes 107 us vs 73 us in whole tiles
// (benchmarks/gemm_trace.py with a -DCORTEX_GEMM_TRACE build). A hybrid (whole tiles for
// the full waves, stream-K for the remainder) measured 17.4 vs 13.2 ms per config-2 step
// (benchmarks/replay_ab.py) and was removed.
void cortex_gemm2_plan(int M, int N, int K, int n_sms, int* tn_out, int* sk_out) {
  const int force = g_cortex_knob[CORTEX_KNOB_GEMM_STREAM_K] == 1 ? 1 : 0;
  const int tn_force = g_cortex_knob[CORTEX_KNOB_GEMM_TN];  // tuning: pin the token tile
  if (tn_force > 0) {
    *tn_out = tn_force;
    *sk_out = force;
    return;
  }
  const int n_tiles = N / kPairN;
  const int pairs = n_sms / 2;
  double best = -1.0;
  for (int tn : {256, 224, 192, 160, 128, 96, 64}) {
    const long units = static_cast<long>(n_tiles) * ((M + tn - 1) / tn);
    for (int sk = 0; sk <= 1; ++sk) {
      if (force >= 0 && sk != force) continue;
      const long waves = (units + pairs - 1) / pairs;
      const double ovh = g_cortex_knob[CORTEX_KNOB_GEMM_TILE_OVH];
      const double cost = sk ? static_cast<double>(units) / pairs * (tn + ovh) * 1.06 + 16.0
                             : waves * (tn + ovh);
      if (best < 0 || cost < best - 1e-9) {
        best = cost;
        *tn_out = tn;
        *sk_out = sk;
      }
    }
  }
}

int32_t cortex_gemm2_tile(int32_t M, int32_t N, int32_t K) {
  if (g_num_sms == 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
        g_num_sms < 2)
      g_num_sms = 148;
  }
  int tn = 256, sk = 0;
  cortex_gemm2_plan(M, N, K, g_num_sms, &tn, &sk);
  return tn | (sk << 16);
}

int32_t cortex_gemm_2sm_launch(const void* tmap_w, const void* tmap_x, int32_t M, int32_t N,
                               int32_t K, void* out, int32_t ldo, int32_t out_f32,
                               const void* residual, int32_t ldr, float* workspace,
                               uint64_t workspace_bytes, int32_t* counters, int32_t n_counters,
                               const RopeEpi* rope, cudaStream_t stream) {
  if (N % kPairN || K % kBK || M <= 0 || (out_f32 == 4 && !rope)) return CORTEX_EBADARG;
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms < 2) g_num_sms = 148;
  }
  int tn = 256, sk = 0;
  cortex_gemm2_plan(M, N, K, g_num_sms, &tn, &sk);
  const int m_tiles = (M + tn - 1) / tn;
  const int num_tiles = (N / kPairN) * m_tiles;
  if (sk && (!workspace || !counters ||
             workspace_bytes < static_cast<uint64_t>(g_num_sms) * tn * 128 * sizeof(float) ||
             n_counters < g_num_sms))
    sk = 0;
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
  a.sk = sk;
  a.total_units = num_tiles * (K / kBK);
  a.workspace = workspace;
  a.flags = counters;
  a.l2pf = g_cortex_knob[CORTEX_KNOB_GEMM_L2PF];
  if (rope) a.rope = *rope;
  const auto* tw = reinterpret_cast<const CUtensorMap*>(tmap_w);
  const auto* tx = reinterpret_cast<const CUtensorMap*>(tmap_x);
  switch (tn) {
    case 64: return launch2<64, 8 + 2 * CORTEX_G2_DEEP>(tw, tx, a, g_num_sms, stream);
    case 96: return launch2<96, 8 + CORTEX_G2_DEEP>(tw, tx, a, g_num_sms, stream);
    case 128: return launch2<128, 7 + CORTEX_G2_DEEP>(tw, tx, a, g_num_sms, stream);
    case 160: return launch2<160, 7 + CORTEX_G2_DEEP>(tw, tx, a, g_num_sms, stream);
    case 192: return launch2<192, 6 + CORTEX_G2_DEEP>(tw, tx, a, g_num_sms, stream);
    case 224: return launch2<224, 6>(tw, tx, a, g_num_sms, stream);
    default: return launch2<256, 5 + CORTEX_G2_DEEP>(tw, tx, a, g_num_sms, stream);
  }
}
