// Tensor-core (tcgen05) paged flash attention for the many-query cases:
//   * prompt / stage-prefix prefill (causal over prefix + own tokens), and
//   * the shared-prefix ("cascade") pass of decode: all decode queries of the
//     calls on one resident stage prefix against that prefix.
//
// One CTA = 128 query rows (128/group query tokens x the GQA group of q heads
// that share one kv head) against a range of KV blocks of one block-table row.
// Key tiles are 8 paged blocks (<= 128 keys); a block may be partial (the last
// prefix block when P % 16 != 0, the last private block), so every key column
// carries (position, valid) from its block descriptor.
//
//   warp 0      TMA producer: Q once (3-D map: tokens x heads x dims), then per
//               key tile 8 blocks x {K lo, K hi, V lo, V hi} 64-column boxes into a
//               2-stage ring (128-byte swizzle)
//   warp 1      MMA issuer (one thread): S_t = Q K_t^T  (M=128, N=128, K=128) into
//               one of two TMEM S buffers; O += P_{t-1} V_{t-1}  (A = P from smem,
//               K-major; B = V from smem, MN-major) into the TMEM O accumulator
//   warps 2..9  softmax, two warps per TMEM lane quarter: thread = (query row, half
//               of the tile's keys); S -> mask -> running max agreed between the two
//               halves (rescale O in TMEM only when the max grows by > 2^8) -> P as
//               bf16 hi + lo back into TMEM -> final O / l (bf16 output, or fp32
//               partial + LSE), each half emitting 64 of the 128 dims
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace {

constexpr int kHD = 128;
constexpr int kBlk = 16;
constexpr int kBlocksPerTile = 8;  // 128 keys
constexpr int kRows = 128;
constexpr int kThreadsTC = 320;  // TMA, MMA, 8 softmax warps
constexpr float kLog2eTC = 1.4426950408889634f;
constexpr float kRescaleThresh = 8.0f;  // log2 units

constexpr int kQBytes = kRows * kHD * 2;                 // 32 KiB
constexpr int kKVHalf = kBlocksPerTile * kBlk * 64 * 2;  // 16 KiB  [128 keys x 64 dims]
constexpr int kKVStage = 4 * kKVHalf;                    // K lo, K hi, V lo, V hi
#ifndef CORTEX_FMHA_STAGES  // (overridable for tuning builds)
#define CORTEX_FMHA_STAGES 2
#endif
constexpr int kStagesTC = CORTEX_FMHA_STAGES;
constexpr int kOffQ = 0;
constexpr int kOffKV = kQBytes;
constexpr int kOffBar = kOffKV + kStagesTC * kKVStage;
constexpr int kOffX = kOffBar + 256;  // row-max / row-sum exchange of the softmax halves
constexpr int kSmemTC = kOffX + 6 * 128 * 4 + 1024;
constexpr uint32_t kTmemColsTC = 512;  // S0 [0,128) S1 [128,256) O [256,384)

struct FmhaArgs {
  const int* table;
  int table_stride;
  int n_kv_heads;
  int group;
  int64_t k_row0, v_row0;
  float scale_log2;
  int mode;  // 0: prefill (final bf16 output), 1: cascade prefix (fp32 partial + LSE)
  // prefill
  const int* seq_row;
  const int* seq_prefix;
  const int* seq_kvlen;
  const int* seq_qstart;
  const int* seq_qlen;
  __nv_bfloat16* out;
  // cascade
  const int* grp_row;
  const int* grp_plen;
  const int* grp_first;
  const int* grp_count;
  int max_psplits;
  float* o_part;
  float* lse_part;
  int max_splits;
  int p_lo;  // 1: P enters PV as bf16 hi + lo (~2^-17), 0: bf16 P only
};

struct BlockRef {
  int block, pos0, nvalid;
};

CORTEX_DEVICE BlockRef block_ref(const int* table_row, int prefix_len, int kv_len, int j,
                                 int blk_end) {
  BlockRef r;
  const int npb = (prefix_len + kBlk - 1) / kBlk;
  if (j >= blk_end) {
    r.block = __ldg(&table_row[0]);  // finite data, fully masked
    r.pos0 = 0;
    r.nvalid = 0;
    return r;
  }
  r.block = __ldg(&table_row[j]);
  if (j < npb) {
    r.pos0 = j * kBlk;
    r.nvalid = min(kBlk, prefix_len - j * kBlk);
  } else {
    const int jj = j - npb;
    r.pos0 = prefix_len + jj * kBlk;
    r.nvalid = min(kBlk, kv_len - prefix_len - jj * kBlk);
  }
  return r;
}

struct BlockSpan {
  int pos0, nvalid;
};

// Positions of block j of a row (no table access): prefix blocks first, then private.
CORTEX_DEVICE BlockSpan block_span(int prefix_len, int kv_len, int j, int blk_end) {
  BlockSpan r;
  const int npb = (prefix_len + kBlk - 1) / kBlk;
  if (j >= blk_end) {
    r.pos0 = 0;
    r.nvalid = 0;
  } else if (j < npb) {
    r.pos0 = j * kBlk;
    r.nvalid = min(kBlk, prefix_len - j * kBlk);
  } else {
    const int jj = j - npb;
    r.pos0 = prefix_len + jj * kBlk;
    r.nvalid = min(kBlk, kv_len - prefix_len - jj * kBlk);
  }
  return r;
}

CORTEX_DEVICE void tma_load_3d(void* smem_dst, const void* desc, uint64_t* bar, int c0, int c1,
                               int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];\n" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// MN-major, 128-byte-swizzled operand: rows of 128 B along K, 64-element atoms along MN
// `lbo` bytes apart, 8-row groups along K 1024 bytes apart.
CORTEX_DEVICE uint64_t umma_desc_sw128_mn(uint32_t smem_addr, uint32_t lbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

CORTEX_DEVICE void tmem_ld_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32"
      " {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15,"
      " %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

CORTEX_DEVICE void tmem_st_x32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0],"
      " {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16,"
      " %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};\n" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
      "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

// D[tmem] (+)= A[tmem] . B[smem]  (A = 128 rows x 16 K, bf16 packed 2 per column)
CORTEX_DEVICE void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t desc_b, uint32_t idesc,
                                uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(desc_b), "r"(idesc), "r"(accumulate)
      : "memory");
}

CORTEX_DEVICE void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

// mbarrier wait that traps (with a diagnostic) instead of hanging forever when a
// phase never completes (~4 s): a logic error must not wedge the GPU.
CORTEX_DEVICE void mbar_wait_guard(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  const long long t0 = clock64();
  while (true) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
    if (done) return;
    if (clock64() - t0 > (8ll << 30)) {
      printf("fmha_tc hang: block (%d,%d,%d) thread %d barrier smem+%u parity %u\n", blockIdx.x,
             blockIdx.y, blockIdx.z, threadIdx.x, addr & 0xffff, parity);
      __trap();
    }
  }
}

CORTEX_DEVICE void named_bar_sync(int id, int n_threads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n_threads) : "memory");
}

CORTEX_DEVICE float ex2_approx(float x) {  // 2^x, one MUFU op (-inf -> 0)
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(y) : "f"(x));
  return y;
}

// Max / sum of 64 values through 8 independent accumulators: a single running
// accumulator is a 64-deep dependent chain (~4 cycles per link) that one softmax warp per
// SM sub-partition cannot hide.
CORTEX_DEVICE float max64(const float (&v)[64], float init) {
  float m[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) m[k] = v[k];
#pragma unroll
  for (int i = 8; i < 64; i += 8)
#pragma unroll
    for (int k = 0; k < 8; ++k) m[k] = fmaxf(m[k], v[i + k]);
#pragma unroll
  for (int w = 4; w > 0; w >>= 1)
#pragma unroll
    for (int k = 0; k < w; ++k) m[k] = fmaxf(m[k], m[k + w]);
  return fmaxf(init, m[0]);
}

CORTEX_DEVICE float sum64(const float (&v)[64]) {
  float t[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) t[k] = v[k];
#pragma unroll
  for (int i = 8; i < 64; i += 8)
#pragma unroll
    for (int k = 0; k < 8; ++k) t[k] += v[i + k];
#pragma unroll
  for (int w = 4; w > 0; w >>= 1)
#pragma unroll
    for (int k = 0; k < w; ++k) t[k] += t[k + w];
  return t[0];
}

__global__ void __launch_bounds__(kThreadsTC, 1)
    fmha_tc_kernel(const __grid_constant__ CUtensorMap tmap_q,
                   const __grid_constant__ CUtensorMap tmap_kv, const FmhaArgs a) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;    // [2]  K and V rings are separate: K of tile t+2 can
  uint64_t* k_empty = bars + 3;   // [2]  stream in as soon as S_t is done, V as soon as
  uint64_t* v_full = bars + 5;    // [2]  PV_t is done
  uint64_t* v_empty = bars + 7;   // [2]
  uint64_t* s_full = bars + 9;    // [2]
  uint64_t* p_full = bars + 11;
  uint64_t* o_ready = bars + 12;  // committed after every PV (O stable for a rescale)
  uint64_t* o_done = bars + 13;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 14);

  const int warp = warp_id();
  const int lane = lane_id();
  const int qb = blockIdx.x;
  const int kvh = blockIdx.y;
  const int item = blockIdx.z;
  const int group = a.group;
  const int tpb = kRows / group;  // query tokens per CTA

  // ---- work item ----
  int row, prefix_len, kv_len, tok0, ntok, qpos_base, blk_begin, blk_end;
  if (a.mode == 0) {
    const int qlen = __ldg(&a.seq_qlen[item]);
    if (qb * tpb >= qlen) return;
    row = __ldg(&a.seq_row[item]);
    prefix_len = __ldg(&a.seq_prefix[item]);
    kv_len = __ldg(&a.seq_kvlen[item]);
    tok0 = __ldg(&a.seq_qstart[item]) + qb * tpb;
    ntok = min(tpb, qlen - qb * tpb);
    qpos_base = kv_len - qlen + qb * tpb;
    const int last = qpos_base + ntok - 1;  // keys needed: positions <= last
    const int npb = (prefix_len + kBlk - 1) / kBlk;
    blk_begin = 0;
    blk_end = last < prefix_len ? last / kBlk + 1 : npb + (last - prefix_len) / kBlk + 1;
  } else {
    const int g = item / a.max_psplits;
    const int ps = item % a.max_psplits;
    const int count = __ldg(&a.grp_count[g]);
    if (qb * tpb >= count) return;
    row = __ldg(&a.grp_row[g]);
    prefix_len = __ldg(&a.grp_plen[g]);
    kv_len = prefix_len;
    const int npb = (prefix_len + kBlk - 1) / kBlk;
    const int psb = prefix_split_blocks(npb, a.max_psplits);  // same split as the combine
    blk_begin = ps * psb;
    if (blk_begin >= npb) return;
    blk_end = min(npb, blk_begin + psb);
    tok0 = __ldg(&a.grp_first[g]) + qb * tpb;
    ntok = min(tpb, count - qb * tpb);
    qpos_base = 0x3fffffff;  // decode queries follow the whole prefix
  }
  const int n_kt = (blk_end - blk_begin + kBlocksPerTile - 1) / kBlocksPerTile;
  const int* table_row = a.table + static_cast<int64_t>(row) * a.table_stride;
  const int hq = a.n_kv_heads * group;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_q);
    tma_prefetch_desc(&tmap_kv);
    mbar_init(q_full, 1);
    for (int s = 0; s < kStagesTC; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
      mbar_init(&s_full[s], 1);
    }
    mbar_init(p_full, 8);
    mbar_init(o_ready, 1);
    mbar_init(o_done, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_holder, kTmemColsTC);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  const uint32_t tmem_s = tmem;         // S buffer b at +128*b
  const uint32_t tmem_o = tmem + 256;

  if (warp == 0) {
    if (elect_one()) {
      // ---- producer ----
      mbar_arrive_expect_tx(q_full, kQBytes);
      tma_load_3d(smem + kOffQ, &tmap_q, q_full, 0, kvh * group, tok0);
      tma_load_3d(smem + kOffQ + kQBytes / 2, &tmap_q, q_full, 64, kvh * group, tok0);
      for (int kt = 0; kt < n_kt; ++kt) {
        const int s = kt % kStagesTC;
        const uint32_t ph = (kt / kStagesTC) & 1;
        uint8_t* st = smem + kOffKV + s * kKVStage;
        int rows[kBlocksPerTile];
#pragma unroll
        for (int j = 0; j < kBlocksPerTile; ++j) {
          const BlockRef b = block_ref(table_row, prefix_len, kv_len,
                                       blk_begin + kt * kBlocksPerTile + j, blk_end);
          rows[j] = static_cast<int>((static_cast<int64_t>(b.block) * a.n_kv_heads + kvh) * kBlk);
        }
        mbar_wait_guard(&k_empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&k_full[s], 2 * kKVHalf);
#pragma unroll
        for (int j = 0; j < kBlocksPerTile; ++j) {
          const int off = j * kBlk * 128;
          tma_load_2d(st + 0 * kKVHalf + off, &tmap_kv, &k_full[s], 0, static_cast<int>(a.k_row0) + rows[j]);
          tma_load_2d(st + 1 * kKVHalf + off, &tmap_kv, &k_full[s], 64, static_cast<int>(a.k_row0) + rows[j]);
        }
        mbar_wait_guard(&v_empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&v_full[s], 2 * kKVHalf);
#pragma unroll
        for (int j = 0; j < kBlocksPerTile; ++j) {
          const int off = j * kBlk * 128;
          tma_load_2d(st + 2 * kKVHalf + off, &tmap_kv, &v_full[s], 0, static_cast<int>(a.v_row0) + rows[j]);
          tma_load_2d(st + 3 * kKVHalf + off, &tmap_kv, &v_full[s], 64, static_cast<int>(a.v_row0) + rows[j]);
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      // ---- MMA issuer ----
      constexpr uint32_t idesc_s = umma_idesc_bf16(128, 128);
      constexpr uint32_t idesc_pv = umma_idesc_bf16(128, 128) | (1u << 16);  // B (V) MN-major
      const uint32_t q_addr = smem_u32(smem + kOffQ);
      mbar_wait_guard(q_full, 0);
      for (int kt = 0; kt <= n_kt; ++kt) {
        if (kt < n_kt) {
          const int s = kt % kStagesTC;
          const uint32_t ph = (kt / kStagesTC) & 1;
          mbar_wait_guard(&k_full[s], ph);
          tc_fence_after();
          const uint32_t k_addr = smem_u32(smem + kOffKV + s * kKVStage);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t off = (kk >> 2) * kKVHalf + (kk & 3) * 32;
#ifndef CORTEX_FMHA_NOMMA
            umma_bf16_ss(tmem_s + 128 * s, umma_desc_sw128(q_addr + off),
                         umma_desc_sw128(k_addr + off), idesc_s, kk != 0 ? 1u : 0u);
#endif
          }
          umma_commit(&k_empty[s]);
          umma_commit(&s_full[s]);
        }
        if (kt > 0) {
          const int t = kt - 1;
          const int s = t % kStagesTC;
          mbar_wait_guard(&v_full[s], (t / kStagesTC) & 1);
          mbar_wait_guard(p_full, t & 1);
          tc_fence_after();
          const uint32_t v_addr = smem_u32(smem + kOffKV + s * kKVStage + 2 * kKVHalf);
          // O += P_hi V + P_lo V  (P = P_hi + P_lo to ~2^-17); P lives in TMEM over the
          // S buffer it was computed from (A operand from TMEM, 8 columns per 16 keys)
          const uint32_t p_tmem = tmem_s + 128 * s;
#pragma unroll
          for (int part = 0; part < 1 + a.p_lo; ++part) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
#ifndef CORTEX_FMHA_NOMMA
              umma_bf16_ts(tmem_o, p_tmem + 64 * part + 8 * kk,
                           umma_desc_sw128_mn(v_addr + kk * 2048, kKVHalf), idesc_pv,
                           (t | kk | part) != 0 ? 1u : 0u);
#endif
            }
          }
          umma_commit(&v_empty[s]);
          umma_commit(o_ready);
          if (t == n_kt - 1) umma_commit(o_done);
        }
      }
    }
  } else {
    // ---- softmax warps 2..9: thread <-> (query row, half of the key columns) ----
    // Warps w and w+4 share TMEM lane quarter w % 4 (the same 32 rows) and split every
    // S row: half 0 owns keys [0, 64) of the tile, half 1 keys [64, 128). They agree on
    // the row max through shared memory (one named barrier per quarter), keep partial
    // row sums, and each rescales / emits its own 64 of the 128 O dims.
    const int quad = warp & 3;
    const int half = (warp - 2) >> 2;
    const int r = quad * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const bool row_ok = r < ntok * group;
    const int qpos = qpos_base + r / group;
    float* xmax = reinterpret_cast<float*>(smem + kOffX);  // [2 slots][2 halves][128 rows]
    float* xsum = xmax + 4 * kRows;                         // [2 halves][128 rows]
    const int bar_id = 1 + quad;
    float m_run = -INFINITY, l_run = 0.f;
    for (int kt = 0; kt < n_kt; ++kt) {
      const int s = kt % kStagesTC;
      mbar_wait_guard(&s_full[s], (kt / kStagesTC) & 1);
      tc_fence_after();
#ifdef CORTEX_FMHA_NOSOFTMAX
      if (true) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full);
        continue;
      }
#endif
      float sv[64];
      {
        uint32_t u0[32], u1[32];  // both loads in flight, one wait
        tmem_ld_x32(tmem_s + 128 * s + lane_off + 64 * half, u0);
        tmem_ld_x32(tmem_s + 128 * s + lane_off + 64 * half + 32, u1);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          sv[i] = __uint_as_float(u0[i]);
          sv[32 + i] = __uint_as_float(u1[i]);
        }
      }
      // tile max (raw scores; scale > 0 commutes with max). Fast path when every key
      // of the tile is valid and visible to every row of the CTA (CTA-uniform test);
      // otherwise mask: invalid slots of partial blocks, causal, rows past the end.
      const int j0 = blk_begin + kt * kBlocksPerTile;
      bool full = j0 + kBlocksPerTile <= blk_end;
#pragma unroll
      for (int j = 0; j < kBlocksPerTile; ++j) {
        const BlockSpan b = block_span(prefix_len, kv_len, j0 + j, blk_end);
        full = full && b.nvalid == kBlk && b.pos0 + kBlk - 1 <= qpos_base;
      }
      if (!full) {
#pragma unroll
        for (int j = 0; j < kBlocksPerTile / 2; ++j) {
          const BlockSpan b = block_span(prefix_len, kv_len, j0 + 4 * half + j, blk_end);
#pragma unroll
          for (int i = 0; i < kBlk; ++i) {
            const bool ok = row_ok && i < b.nvalid && b.pos0 + i <= qpos;
            sv[kBlk * j + i] = ok ? sv[kBlk * j + i] : -INFINITY;
          }
        }
      }
      float mraw = max64(sv, -INFINITY);
      xmax[((kt & 1) * 2 + half) * kRows + r] = mraw;
      named_bar_sync(bar_id, 64);
      mraw = fmaxf(mraw, xmax[((kt & 1) * 2 + (half ^ 1)) * kRows + r]);
      const float mt = mraw * a.scale_log2;  // -inf stays -inf
      // running max: adopt the tile max when the row had none yet (its O row is 0), or
      // when it grew by more than 2^8 (then O and l are rescaled); otherwise keep the
      // stale max (p <= 2^8, exact after the final 1/l).
      const bool adopt = mt > -INFINITY && (m_run == -INFINITY || mt > m_run + kRescaleThresh);
      const float alpha = !adopt ? 1.f : (m_run == -INFINITY ? 0.f : exp2f(m_run - mt));
      const float m_new = adopt ? mt : m_run;
      const float m_use = m_new == -INFINITY ? 0.f : m_new;
      // p = exp2(s * scale - m), computed before waiting for the previous PV
#pragma unroll
      for (int i = 0; i < 64; ++i) sv[i] = ex2_approx(fmaf(sv[i], a.scale_log2, -m_use));
      const float lsum = sum64(sv);
      // O rescale of this half's 64 dims (rare; tcgen05.ld/st are warp-collective:
      // decided per warp - the partner warp sees the same rows - alpha per row) needs
      // PV of the previous tile finished
      if (kt > 0 && __any_sync(0xffffffffu, adopt && m_run != -INFINITY)) {
        mbar_wait_guard(o_ready, (kt - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t u[32];
          tmem_ld_x32(tmem_o + lane_off + 64 * half + 32 * c, u);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) u[i] = __float_as_uint(__uint_as_float(u[i]) * alpha);
          tmem_st_x32(tmem_o + lane_off + 64 * half + 32 * c, u);
        }
        tmem_st_wait();
      }
      l_run = l_run * alpha + lsum;
      m_run = m_new;
      // P (bf16 hi + lo, keys 2c / 2c+1 packed in column c) -> TMEM over this S buffer:
      // hi of keys [64 half, +64) in columns [32 half, +32), lo 64 columns further
      {
        uint32_t hi[32], lo[32];
        if (a.p_lo) {
#pragma unroll
          for (int c = 0; c < 32; ++c) split_bf16(sv[2 * c], sv[2 * c + 1], hi[c], lo[c]);
          tmem_st_x32(tmem_s + 128 * s + lane_off + 32 * half, hi);
          tmem_st_x32(tmem_s + 128 * s + lane_off + 64 + 32 * half, lo);
        } else {
#pragma unroll
          for (int c = 0; c < 32; ++c) hi[c] = pack_bf16(sv[2 * c], sv[2 * c + 1]);
          tmem_st_x32(tmem_s + 128 * s + lane_off + 32 * half, hi);
        }
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
    }
    // ---- epilogue: row sum of both halves, then this half's 64 O dims ----
    xsum[half * kRows + r] = l_run;
    named_bar_sync(bar_id, 64);
    const float l_tot = l_run + xsum[(half ^ 1) * kRows + r];
    mbar_wait_guard(o_done, 0);
    tc_fence_after();
    const int tok = tok0 + r / group;
    const int h = kvh * group + r % group;
    const float inv = l_tot > 0.f ? 1.f / l_tot : 0.f;
    if (a.mode == 0) {
      __nv_bfloat16* orow = a.out + (static_cast<int64_t>(tok) * hq + h) * kHD + 64 * half;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t u[32];
        tmem_ld_x32(tmem_o + lane_off + 64 * half + 32 * c, u);
        tmem_ld_wait();
        if (row_ok) {
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            uint4 v;
            v.x = pack_bf16(__uint_as_float(u[i]) * inv, __uint_as_float(u[i + 1]) * inv);
            v.y = pack_bf16(__uint_as_float(u[i + 2]) * inv, __uint_as_float(u[i + 3]) * inv);
            v.z = pack_bf16(__uint_as_float(u[i + 4]) * inv, __uint_as_float(u[i + 5]) * inv);
            v.w = pack_bf16(__uint_as_float(u[i + 6]) * inv, __uint_as_float(u[i + 7]) * inv);
            *reinterpret_cast<uint4*>(orow + 32 * c + i) = v;
          }
        }
      }
    } else {
      const int ps = item % a.max_psplits;
      const int64_t pidx = (static_cast<int64_t>(tok) * a.max_splits + ps) * hq + h;
      float* o = a.o_part + pidx * kHD + 64 * half;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t u[32];
        tmem_ld_x32(tmem_o + lane_off + 64 * half + 32 * c, u);
        tmem_ld_wait();
        if (row_ok) {
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            *reinterpret_cast<float4*>(o + 32 * c + i) =
                make_float4(__uint_as_float(u[i]) * inv, __uint_as_float(u[i + 1]) * inv,
                            __uint_as_float(u[i + 2]) * inv, __uint_as_float(u[i + 3]) * inv);
        }
      }
      if (row_ok && half == 0) a.lse_part[pidx] = m_run + log2f(l_tot);
    }
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, kTmemColsTC);
  }
}

// ---------------------------------------------------------------------------
// Two-Q-tile variant (ping-pong): one CTA owns 2 x 128 query rows (Q tiles A and B,
// 2 x tpb tokens) and streams every K/V tile once for both, so the L2 -> SM traffic per
// flop halves, and the tensor pipe computes one tile's S / PV while the other tile's
// softmax runs. The work unit is half a key tile (64 keys): S of one half is computed
// while the same warpgroup's softmax works on the other half (S_X(t+1, h) is issued
// right behind PV_X(t, h), which frees those TMEM columns):
//   MMA warp: S(0,0) S(0,1) | per tile X, half h in order: PV_X(t,h) S_X(t+1,h), the two
//   tiles' units interleaved in the order their P becomes ready | ...
//   softmax warpgroup A (warps 2-5) and B (warps 6-9): one thread per query row, 64 keys
//   per unit (no cross-warp max exchange), lazy O rescale, P -> TMEM.
// TMEM: S_A [0,128)  S_B [128,256)  O_A [256,384)  O_B [384,512) (S single-buffered per
// tile: S_X(t+1) is issued after PV_X(t), which consumed P_X(t) in place, in MMA order).
// Smem: Q_A 32 KiB, Q_B 32 KiB, a K ring and a V ring of 32 KiB stages, barriers.
// K and V have their own rings (K lo | K hi, V lo | V hi per stage, 32 KiB each).
#ifndef CORTEX_FMHA2_VSTAGES  // (tuning builds: 1 V stage = 160 KiB, a split CTA fits beside)
#define CORTEX_FMHA2_VSTAGES 2
#endif
constexpr int kKStages2 = kStagesTC;
constexpr int kVStages2 = CORTEX_FMHA2_VSTAGES;
constexpr int kOffQ2 = 0;
constexpr int kOffK2 = 2 * kQBytes;
constexpr int kOffV2 = kOffK2 + kKStages2 * 2 * kKVHalf;
constexpr int kOffBar2 = kOffV2 + kVStages2 * 2 * kKVHalf;
constexpr int kSmemTC2 = kOffBar2 + 256 + 1024;

__global__ void __launch_bounds__(kThreadsTC, 1)
    fmha2_tc_kernel(const __grid_constant__ CUtensorMap tmap_q,
                    const __grid_constant__ CUtensorMap tmap_kv, const FmhaArgs a) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar2);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;   // [2]
  uint64_t* k_empty = bars + 3;  // [2]
  uint64_t* v_full = bars + 5;   // [2]
  uint64_t* v_empty = bars + 7;  // [2]
  uint64_t* s_full = bars + 9;   // [2 tiles][2 key halves]
  uint64_t* p_full = bars + 13;  // [2 tiles][2 key halves]
  uint64_t* o_ready = bars + 17; // [2 tiles] committed after every PV of the tile
  uint64_t* o_done = bars + 19;  // [2 tiles]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 21);

  const int warp = warp_id();
  const int lane = lane_id();
  const int qb = blockIdx.x;  // pair of Q tiles
  const int kvh = blockIdx.y;
  const int item = blockIdx.z;
  const int group = a.group;
  const int tpb = kRows / group;  // query tokens per tile

  // ---- work item (as fmha_tc_kernel, over 2 tpb tokens) ----
  int row, prefix_len, kv_len, tok0, ntok, qpos_base, blk_begin, blk_end;
  if (a.mode == 0) {
    const int qlen = __ldg(&a.seq_qlen[item]);
    if (qb * 2 * tpb >= qlen) return;
    row = __ldg(&a.seq_row[item]);
    prefix_len = __ldg(&a.seq_prefix[item]);
    kv_len = __ldg(&a.seq_kvlen[item]);
    tok0 = __ldg(&a.seq_qstart[item]) + qb * 2 * tpb;
    ntok = min(2 * tpb, qlen - qb * 2 * tpb);
    qpos_base = kv_len - qlen + qb * 2 * tpb;
    const int last = qpos_base + ntok - 1;
    const int npb = (prefix_len + kBlk - 1) / kBlk;
    blk_begin = 0;
    blk_end = last < prefix_len ? last / kBlk + 1 : npb + (last - prefix_len) / kBlk + 1;
  } else {
    const int g = item / a.max_psplits;
    const int ps = item % a.max_psplits;
    const int count = __ldg(&a.grp_count[g]);
    if (qb * 2 * tpb >= count) return;
    row = __ldg(&a.grp_row[g]);
    prefix_len = __ldg(&a.grp_plen[g]);
    kv_len = prefix_len;
    const int npb = (prefix_len + kBlk - 1) / kBlk;
    const int psb = prefix_split_blocks(npb, a.max_psplits);
    blk_begin = ps * psb;
    if (blk_begin >= npb) return;
    blk_end = min(npb, blk_begin + psb);
    tok0 = __ldg(&a.grp_first[g]) + qb * 2 * tpb;
    ntok = min(2 * tpb, count - qb * 2 * tpb);
    qpos_base = 0x3fffffff;
  }
  const bool has_b = ntok > tpb;  // CTA-uniform: tile B holds at least one token
  const int n_kt = (blk_end - blk_begin + kBlocksPerTile - 1) / kBlocksPerTile;
  const int* table_row = a.table + static_cast<int64_t>(row) * a.table_stride;
  const int hq = a.n_kv_heads * group;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_q);
    tma_prefetch_desc(&tmap_kv);
    mbar_init(q_full, 1);
    for (int s = 0; s < kKStages2; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < kVStages2; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int x = 0; x < 4; ++x) {
      mbar_init(&s_full[x], 1);
      mbar_init(&p_full[x], 4);
    }
    for (int x = 0; x < 2; ++x) {
      mbar_init(&o_ready[x], 1);
      mbar_init(&o_done[x], 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_holder, kTmemColsTC);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    if (elect_one()) {
      // ---- producer ----
      mbar_arrive_expect_tx(q_full, (has_b ? 2 : 1) * kQBytes);
      for (int x = 0; x < (has_b ? 2 : 1); ++x) {
        uint8_t* qd = smem + kOffQ2 + x * kQBytes;
        tma_load_3d(qd, &tmap_q, q_full, 0, kvh * group, tok0 + x * tpb);
        tma_load_3d(qd + kQBytes / 2, &tmap_q, q_full, 64, kvh * group, tok0 + x * tpb);
      }
      for (int kt = 0; kt < n_kt; ++kt) {
        const int sk = kt % kKStages2, sv = kt % kVStages2;
        const uint32_t phk = (kt / kKStages2) & 1, phv = (kt / kVStages2) & 1;
        uint8_t* stk = smem + kOffK2 + sk * 2 * kKVHalf;
        uint8_t* stv = smem + kOffV2 + sv * 2 * kKVHalf;
        int rows[kBlocksPerTile];
#pragma unroll
        for (int j = 0; j < kBlocksPerTile; ++j) {
          const BlockRef b = block_ref(table_row, prefix_len, kv_len,
                                       blk_begin + kt * kBlocksPerTile + j, blk_end);
          rows[j] = static_cast<int>((static_cast<int64_t>(b.block) * a.n_kv_heads + kvh) * kBlk);
        }
        mbar_wait_guard(&k_empty[sk], phk ^ 1);
        mbar_arrive_expect_tx(&k_full[sk], 2 * kKVHalf);
#pragma unroll
        for (int j = 0; j < kBlocksPerTile; ++j) {
          const int off = j * kBlk * 128;
          tma_load_2d(stk + 0 * kKVHalf + off, &tmap_kv, &k_full[sk], 0, static_cast<int>(a.k_row0) + rows[j]);
          tma_load_2d(stk + 1 * kKVHalf + off, &tmap_kv, &k_full[sk], 64, static_cast<int>(a.k_row0) + rows[j]);
        }
        mbar_wait_guard(&v_empty[sv], phv ^ 1);
        mbar_arrive_expect_tx(&v_full[sv], 2 * kKVHalf);
#pragma unroll
        for (int j = 0; j < kBlocksPerTile; ++j) {
          const int off = j * kBlk * 128;
          tma_load_2d(stv + 0 * kKVHalf + off, &tmap_kv, &v_full[sv], 0, static_cast<int>(a.v_row0) + rows[j]);
          tma_load_2d(stv + 1 * kKVHalf + off, &tmap_kv, &v_full[sv], 64, static_cast<int>(a.v_row0) + rows[j]);
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      // ---- MMA issuer: work unit = (key tile, 64-key half), so S of one half computes
      // while the same warpgroup's softmax runs on the other half ----
      constexpr uint32_t idesc_s = umma_idesc_bf16(128, 64);                 // N = 64 keys
      constexpr uint32_t idesc_pv = umma_idesc_bf16(128, 128) | (1u << 16);  // V MN-major
      const int nx = has_b ? 2 : 1;
      mbar_wait_guard(q_full, 0);
      auto issue_s = [&](int kt, int x, int h) {  // S_x(kt, h) -> TMEM S_x cols [64h, +64)
        const int s = kt % kKStages2;
        const uint32_t q_addr = smem_u32(smem + kOffQ2 + x * kQBytes);
        const uint32_t k_addr = smem_u32(smem + kOffK2 + s * 2 * kKVHalf) + h * 64 * 128;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk >> 2) * kKVHalf + (kk & 3) * 32;
#ifndef CORTEX_FMHA_NOMMA  // (tuning builds only: pipeline bound without the MMAs)
          umma_bf16_ss(tmem + 128 * x + 64 * h, umma_desc_sw128(q_addr + off),
                       umma_desc_sw128(k_addr + off), idesc_s, kk != 0 ? 1u : 0u);
#endif
        }
        umma_commit(&s_full[2 * x + h]);
      };
      auto issue_pv = [&](int kt, int x, int h) {  // O_x += P_x(kt, h) V(kt, keys of h)
        const int s = kt % kVStages2;
        const uint32_t v_addr = smem_u32(smem + kOffV2 + s * 2 * kKVHalf);
        const uint32_t p_tmem = tmem + 128 * x + 64 * h;
        const uint32_t o_tmem = tmem + 256 + 128 * x;
        // P = hi + lo (p_lo): hi in this half's first 32 columns, lo in the next 32
        for (int part = 0; part < 1 + a.p_lo; ++part) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
#ifndef CORTEX_FMHA_NOMMA
            umma_bf16_ts(o_tmem, p_tmem + 32 * part + 8 * kk,
                         umma_desc_sw128_mn(v_addr + (4 * h + kk) * 2048, kKVHalf), idesc_pv,
                         (kt | h | kk | part) != 0 ? 1u : 0u);
#endif
          }
        }
        umma_commit(&o_ready[x]);
        if (kt == n_kt - 1 && h == 1) umma_commit(&o_done[x]);
      };
      if (n_kt > 0) {
        mbar_wait_guard(&k_full[0], 0);
        tc_fence_after();
        for (int h = 0; h < 2; ++h)
          for (int x = 0; x < nx; ++x) issue_s(0, x, h);
        umma_commit(&k_empty[0]);
      }
      for (int kt = 0; kt < n_kt; ++kt) {
        const int s = kt % kVStages2;
        const bool more = kt + 1 < n_kt;
        const int s1 = (kt + 1) % kKStages2;
        mbar_wait_guard(&v_full[s], (kt / kVStages2) & 1);
        // PV + next S of whichever tile's P is ready first (the order within a tile is
        // fixed: h = 0 then 1), so a slower softmax warpgroup does not hold the other
        // tile's MMAs (prefill 41.6 vs 42.5 us, benchmarks/attn_step.py --fmha-only)
        {
          int next_h[2] = {0, nx > 1 ? 0 : 2};
          bool k_ready = !more;
          const long long t0 = clock64();
          while (next_h[0] < 2 || next_h[1] < 2) {
            for (int x = 0; x < 2; ++x) {
              const int h = next_h[x];
              if (h >= 2 || !mbar_test_wait(&p_full[2 * x + h], kt & 1)) continue;
              tc_fence_after();
              issue_pv(kt, x, h);
              if (more) {
                if (!k_ready) {
                  mbar_wait_guard(&k_full[s1], ((kt + 1) / kKStages2) & 1);
                  tc_fence_after();
                  k_ready = true;
                }
                issue_s(kt + 1, x, h);
              }
              next_h[x] = h + 1;
            }
            if (clock64() - t0 > (8ll << 30)) __trap();
          }
        }

        umma_commit(&v_empty[s]);
        if (more) umma_commit(&k_empty[s1]);
      }
    }
  } else {
    // ---- softmax: warpgroup x = tile (warps 2-5 tile A, 6-9 tile B); thread <-> row ----
    const int x = (warp - 2) >> 2;
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    if (x == 1 && !has_b) goto done;
    {
      const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
      const uint32_t tmem_s = tmem + 128 * x;
      const uint32_t tmem_o = tmem + 256 + 128 * x;
      const int ntok_x = min(tpb, ntok - x * tpb);
      const bool row_ok = r < ntok_x * group;
      const int qpos0 = qpos_base == 0x3fffffff ? qpos_base : qpos_base + x * tpb;
      const int qpos = qpos0 == 0x3fffffff ? qpos0 : qpos0 + r / group;
      float m_run = -INFINITY, l_run = 0.f;
      for (int u = 0; u < 2 * n_kt; ++u) {
        const int kt = u >> 1, h = u & 1;
        mbar_wait_guard(&s_full[2 * x + h], kt & 1);
        tc_fence_after();
#ifdef CORTEX_FMHA_NOSOFTMAX  // (tuning builds only: pipeline bound without the softmax)
        if (true) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&p_full[2 * x + h]);
          continue;
        }
#endif
        float sv[64];
        {
          uint32_t u0[32], u1[32];  // both loads in flight, one wait
          tmem_ld_x32(tmem_s + lane_off + 64 * h, u0);
          tmem_ld_x32(tmem_s + lane_off + 64 * h + 32, u1);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            sv[i] = __uint_as_float(u0[i]);
            sv[32 + i] = __uint_as_float(u1[i]);
          }
        }
        // fast path (unit-uniform): every key valid and visible to every row of the tile;
        // otherwise mask (invalid slots of partial blocks, causal, rows past the end)
        const int jb = blk_begin + kt * kBlocksPerTile + 4 * h;
        bool full = jb + 4 <= blk_end;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const BlockSpan b = block_span(prefix_len, kv_len, jb + j, blk_end);
          full = full && b.nvalid == kBlk && b.pos0 + kBlk - 1 <= qpos0;
        }
        if (!full) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const BlockSpan b = block_span(prefix_len, kv_len, jb + j, blk_end);
#pragma unroll
            for (int i = 0; i < kBlk; ++i) {
              const bool ok = row_ok && i < b.nvalid && b.pos0 + i <= qpos;
              sv[kBlk * j + i] = ok ? sv[kBlk * j + i] : -INFINITY;
            }
          }
        }
        const float mt = max64(sv, -INFINITY) * a.scale_log2;
        const bool adopt = mt > -INFINITY && (m_run == -INFINITY || mt > m_run + kRescaleThresh);
        const float alpha = !adopt ? 1.f : (m_run == -INFINITY ? 0.f : exp2f(m_run - mt));
        const float m_new = adopt ? mt : m_run;
        const float m_use = m_new == -INFINITY ? 0.f : m_new;
        // O rescale (rare) needs the previous unit's PV done; PV of unit u-2 completed
        // before S of this unit (same half, MMA order), so the parity wait is exact
        if (u > 0 && __any_sync(0xffffffffu, adopt && m_run != -INFINITY)) {
          mbar_wait_guard(&o_ready[x], (u - 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t uo[32];
            tmem_ld_x32(tmem_o + lane_off + 32 * c, uo);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) uo[i] = __float_as_uint(__uint_as_float(uo[i]) * alpha);
            tmem_st_x32(tmem_o + lane_off + 32 * c, uo);
          }
          tmem_st_wait();
        }
        // p = exp2(s * scale - m); P as bf16 (keys 2c / 2c+1 packed in column c) over the
        // first 32 columns of this half's S, and with p_lo the residual lo = p - hi over
        // the next 32 (the PV pass then adds P_hi V + P_lo V)
#pragma unroll
        for (int i = 0; i < 64; ++i) sv[i] = ex2_approx(fmaf(sv[i], a.scale_log2, -m_use));
        const float lsum = sum64(sv);
        if (a.p_lo) {
          uint32_t hi[32], lo[32];
#pragma unroll
          for (int c = 0; c < 32; ++c) split_bf16(sv[2 * c], sv[2 * c + 1], hi[c], lo[c]);
          tmem_st_x32(tmem_s + lane_off + 64 * h, hi);
          tmem_st_x32(tmem_s + lane_off + 64 * h + 32, lo);
        } else {
          uint32_t hi[32];
#pragma unroll
          for (int c = 0; c < 32; ++c) hi[c] = pack_bf16(sv[2 * c], sv[2 * c + 1]);
          tmem_st_x32(tmem_s + lane_off + 64 * h, hi);
        }
        l_run = l_run * alpha + lsum;
        m_run = m_new;
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[2 * x + h]);
      }
      // ---- epilogue: this tile's O rows ----
      mbar_wait_guard(&o_done[x], 0);
      tc_fence_after();
      const int tok = tok0 + x * tpb + r / group;
      const int h = kvh * group + r % group;
      const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
      if (a.mode == 0) {
        __nv_bfloat16* orow = a.out + (static_cast<int64_t>(tok) * hq + h) * kHD;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t u[32];
          tmem_ld_x32(tmem_o + lane_off + 32 * c, u);
          tmem_ld_wait();
          if (row_ok) {
#pragma unroll
            for (int i = 0; i < 32; i += 8) {
              uint4 v;
              v.x = pack_bf16(__uint_as_float(u[i]) * inv, __uint_as_float(u[i + 1]) * inv);
              v.y = pack_bf16(__uint_as_float(u[i + 2]) * inv, __uint_as_float(u[i + 3]) * inv);
              v.z = pack_bf16(__uint_as_float(u[i + 4]) * inv, __uint_as_float(u[i + 5]) * inv);
              v.w = pack_bf16(__uint_as_float(u[i + 6]) * inv, __uint_as_float(u[i + 7]) * inv);
              *reinterpret_cast<uint4*>(orow + 32 * c + i) = v;
            }
          }
        }
      } else {
        const int ps = item % a.max_psplits;
        const int64_t pidx = (static_cast<int64_t>(tok) * a.max_splits + ps) * hq + h;
        float* o = a.o_part + pidx * kHD;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t u[32];
          tmem_ld_x32(tmem_o + lane_off + 32 * c, u);
          tmem_ld_wait();
          if (row_ok) {
#pragma unroll
            for (int i = 0; i < 32; i += 4)
              *reinterpret_cast<float4*>(o + 32 * c + i) =
                  make_float4(__uint_as_float(u[i]) * inv, __uint_as_float(u[i + 1]) * inv,
                              __uint_as_float(u[i + 2]) * inv, __uint_as_float(u[i + 3]) * inv);
          }
        }
        if (row_ok) a.lse_part[pidx] = m_run + log2f(l_run);
      }
    }
  done:;
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, kTmemColsTC);
  }
}

// P enters the PV MMA as bf16 hi + lo (P = hi + lo to ~2^-17, a second PV pass; knob
// FMHA_PLO, default on). bf16 P alone (FMHA_PLO = 0, the FlashAttention convention) puts
// a 2^-9 relative error on every probability: at the Llama-3-8B shape the attention
// output then differs from exact softmax by 2.2e-3 (tools/diag_8b.py) and 2-layer logits
// by 4.7e-3, over the north star's 2e-3 bar; with hi + lo the attention error is the bf16
// rounding of the output alone (<= 1.4e-4 beyond it).
int fmha_p_lo() { return g_cortex_knob[CORTEX_KNOB_FMHA_PLO]; }

// Kernel choice per launch (knob FMHA_2Q: -1 automatic, 0 one Q tile, 1 two). A two-tile CTA costs ~1.55x a one-tile
// CTA (benchmarks/fmha.py: 8K causal prefill 614 -> 807 TFLOP/s, 8 x 200-token prompts
// 325 -> 406) but the grid halves, so small grids (decode's cascade pass over a
// 1000-token prefix: 128 one-tile CTAs, 15 us vs 21 us) stay on one tile per CTA:
// pick the lower of waves(n1) and 1.55 waves(n1 / 2) on the SM count.
int g_fmha_sms = 0;

bool fmha_use_2q(const dim3& grid) {
  const int force = g_cortex_knob[CORTEX_KNOB_FMHA_2Q];
  if (force >= 0) return force == 1;
  if (g_fmha_sms == 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&g_fmha_sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      g_fmha_sms = 148;
  }
  const long yz = static_cast<long>(grid.y) * grid.z;
  const long n1 = grid.x * yz, n2 = ((grid.x + 1) / 2) * yz;
  const double w1 = static_cast<double>((n1 + g_fmha_sms - 1) / g_fmha_sms);
  const double w2 = 1.55 * static_cast<double>((n2 + g_fmha_sms - 1) / g_fmha_sms);
  return w2 < w1;
}

// grid.x counts query tiles of tpb tokens; the two-tile kernel takes them in pairs
int32_t launch_fmha(const CUtensorMap* tq, const CUtensorMap* tkv, const FmhaArgs& a, dim3 grid,
                    cudaStream_t stream) {
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(fmha_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kSmemTC) != cudaSuccess ||
        cudaFuncSetAttribute(fmha2_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kSmemTC2) != cudaSuccess)
      return CORTEX_ECUDA;
    configured = true;
  }
  if (fmha_use_2q(grid)) {
    dim3 g2((grid.x + 1) / 2, grid.y, grid.z);
    if (pdl_launch(fmha2_tc_kernel, g2, kThreadsTC, kSmemTC2, stream, 1, *tq, *tkv, a) !=
        cudaSuccess)
      return CORTEX_ECUDA;
    return CORTEX_OK;
  }
  if (pdl_launch(fmha_tc_kernel, grid, kThreadsTC, kSmemTC, stream, 1, *tq, *tkv, a) != cudaSuccess)
    return CORTEX_ECUDA;
  return CORTEX_OK;
}

}  // namespace

extern "C" {

int32_t cortex_fmha_prefill_tc(const void* tmap_kv, const void* tmap_q, void* out,
                               const int32_t* table, int32_t table_stride, const int32_t* seq_row,
                               const int32_t* seq_prefix, const int32_t* seq_kvlen,
                               const int32_t* seq_qstart, const int32_t* seq_qlen, int32_t n_seqs,
                               int32_t max_qlen, int32_t n_kv_heads, int32_t group,
                               int64_t k_row0, int64_t v_row0, float softmax_scale,
                               cudaStream_t stream) {
  if (!tmap_kv || !tmap_q || !out || !table || n_seqs < 0 || group < 1 || (128 % group) != 0)
    return CORTEX_EBADARG;
  if (n_seqs == 0 || max_qlen <= 0) return CORTEX_OK;
  FmhaArgs a{};
  a.table = table;
  a.table_stride = table_stride;
  a.n_kv_heads = n_kv_heads;
  a.group = group;
  a.k_row0 = k_row0;
  a.v_row0 = v_row0;
  a.scale_log2 = softmax_scale * kLog2eTC;
  a.mode = 0;
  a.p_lo = fmha_p_lo();
  a.seq_row = seq_row;
  a.seq_prefix = seq_prefix;
  a.seq_kvlen = seq_kvlen;
  a.seq_qstart = seq_qstart;
  a.seq_qlen = seq_qlen;
  a.out = reinterpret_cast<__nv_bfloat16*>(out);
  const int tpb = kRows / group;
  dim3 grid((max_qlen + tpb - 1) / tpb, n_kv_heads, n_seqs);
  return launch_fmha(reinterpret_cast<const CUtensorMap*>(tmap_q),
                     reinterpret_cast<const CUtensorMap*>(tmap_kv), a, grid, stream);
}

int32_t cortex_fmha_cascade_tc(const void* tmap_kv, const void* tmap_q, const int32_t* table,
                               int32_t table_stride, const int32_t* grp_row,
                               const int32_t* grp_plen, const int32_t* grp_first,
                               const int32_t* grp_count, int32_t n_groups, int32_t max_count,
                               int32_t prefix_slots, int32_t n_kv_heads, int32_t group,
                               int64_t k_row0, int64_t v_row0, float softmax_scale,
                               float* o_part, float* lse_part, int32_t max_splits,
                               cudaStream_t stream) {
  if (!tmap_kv || !tmap_q || !table || !o_part || !lse_part || n_groups < 0 || group < 1 ||
      (128 % group) != 0 || prefix_slots < 1)
    return CORTEX_EBADARG;
  if (n_groups == 0) return CORTEX_OK;
  FmhaArgs a{};
  a.table = table;
  a.table_stride = table_stride;
  a.n_kv_heads = n_kv_heads;
  a.group = group;
  a.k_row0 = k_row0;
  a.v_row0 = v_row0;
  a.scale_log2 = softmax_scale * kLog2eTC;
  a.mode = 1;
  a.p_lo = fmha_p_lo();
  a.grp_row = grp_row;
  a.grp_plen = grp_plen;
  a.grp_first = grp_first;
  a.grp_count = grp_count;
  a.max_psplits = prefix_slots;
  a.o_part = o_part;
  a.lse_part = lse_part;
  a.max_splits = max_splits;
  const int tpb = kRows / group;
  dim3 grid((max_count + tpb - 1) / tpb, n_kv_heads, n_groups * prefix_slots);
  return launch_fmha(reinterpret_cast<const CUtensorMap*>(tmap_q),
                     reinterpret_cast<const CUtensorMap*>(tmap_kv), a, grid, stream);
}

}  // extern "C"
