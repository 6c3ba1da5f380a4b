// Paged attention over a stage engine's block table.
//
// KV layout (one allocation for all layers):
//   cache[layer][k|v][block][kv_head][16 tokens][128 dims]  (bf16)
// seen by TMA as a 2-D matrix of 128-wide rows; one (block, kv_head) tile is 16
// consecutive rows = 4 KiB, loaded as two 64-column boxes with the 128-byte
// swizzle so ldmatrix reads are bank-conflict free.
//
// A sequence's KV is the concatenation of two block lists held in one row of the
// block table: the stage prefix (shared, refcounted, ceil(P/16) blocks whose last
// block holds P%16 tokens) followed by the call's private blocks (positions
// P, P+1, ...). A "tile" is one block of either segment.
//
// Inner products use warp MMA (m16n8k16, bf16 -> f32); one warp owns 16 query
// rows = (query tokens x the GQA group of q heads sharing one kv head). Decode is
// HBM-bound: every KV byte is read once per step, split along the context into
// chunks merged by a log-sum-exp combine - either fixed 16-tile chunks per call
// (chunking depends only on the sequence length, so results are batch-composition
// invariant) or the balanced "flat" plan (equal tile ranges over all calls).
#include "common.cuh"

namespace {

constexpr int kHeadDim = 128;
constexpr int kTile = 16;                  // tokens per KV block
constexpr int kTileBytes = kTile * kHeadDim * 2;  // 4 KiB (K or V)
constexpr int kStageBytes = 2 * kTileBytes;       // K + V
#ifndef CORTEX_DECODE_SPLIT_TILES  // (overridable for tuning builds)
#define CORTEX_DECODE_SPLIT_TILES 32
#endif
#ifndef CORTEX_DECODE_STAGES
#define CORTEX_DECODE_STAGES 2
#endif
constexpr int kTilesPerSplit = CORTEX_DECODE_SPLIT_TILES;
#ifndef CORTEX_DECODE_WARPS  // (overridable for tuning builds)
#define CORTEX_DECODE_WARPS 4
#endif
constexpr int kWarps = CORTEX_DECODE_WARPS;
constexpr float kLog2e = 1.4426950408889634f;

struct TileRef {
  int block;
  int pos0;
  int nvalid;
};

CORTEX_DEVICE int num_tiles(int prefix_len, int kv_len) {
  const int npb = (prefix_len + kTile - 1) / kTile;
  return npb + (kv_len - prefix_len + kTile - 1) / kTile;
}

CORTEX_DEVICE TileRef tile_ref(const int* __restrict__ table_row, int prefix_len, int kv_len,
                               int j) {
  const int npb = (prefix_len + kTile - 1) / kTile;
  TileRef t;
  t.block = __ldg(&table_row[j]);
  if (j < npb) {
    t.pos0 = j * kTile;
    t.nvalid = min(kTile, prefix_len - j * kTile);
  } else {
    const int jj = j - npb;
    t.pos0 = prefix_len + jj * kTile;
    t.nvalid = min(kTile, kv_len - prefix_len - jj * kTile);
  }
  return t;
}

// Issue the four TMA boxes (K lo/hi, V lo/hi) of one tile into a stage buffer.
CORTEX_DEVICE void load_tile(uint8_t* stage, const CUtensorMap* tmap, uint64_t* bar, int64_t k_row0,
                             int64_t v_row0, int block, int kv_head, int n_kv_heads) {
  const int64_t r = (static_cast<int64_t>(block) * n_kv_heads + kv_head) * kTile;
  mbar_arrive_expect_tx(bar, kStageBytes);
  tma_load_2d(stage, tmap, bar, 0, static_cast<int>(k_row0 + r));
  tma_load_2d(stage + 2048, tmap, bar, 64, static_cast<int>(k_row0 + r));
  tma_load_2d(stage + 4096, tmap, bar, 0, static_cast<int>(v_row0 + r));
  tma_load_2d(stage + 6144, tmap, bar, 64, static_cast<int>(v_row0 + r));
}

CORTEX_DEVICE uint32_t kv_elem_addr(uint32_t base, int row, int dim) {
  // base points at a [16 x 128] tile stored as two swizzled [16 x 64] halves.
  return base + (dim >> 6) * 2048 + sw128_offset(row, (dim & 63) >> 3) + (dim & 7) * 2;
}

// Online-softmax state of one warp: rows g and g+8 (g = lane/4).
struct WarpState {
  float m[2];
  float l[2];
  float o[16][4];
};

CORTEX_DEVICE void state_init(WarpState& st) {
  st.m[0] = st.m[1] = -INFINITY;
  st.l[0] = st.l[1] = 0.f;
#pragma unroll
  for (int j = 0; j < 16; ++j)
#pragma unroll
    for (int e = 0; e < 4; ++e) st.o[j][e] = 0.f;
}

// One 16-token KV tile against the warp's 16 query rows.
// qpos[2]: logical position of rows g and g+8 (keys with pos > qpos are masked).
CORTEX_DEVICE void attend_tile(WarpState& st, const uint32_t (&qa)[8][4], uint32_t stage_addr,
                               const TileRef& t, const int (&qpos)[2], float scale_log2) {
  const int lane = lane_id();
  const int tq = lane & 3;
  const uint32_t k_base = stage_addr;
  const uint32_t v_base = stage_addr + kTileBytes;

  float s[2][4];
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) s[nt][e] = 0.f;

  // S = Q K^T : B operand = K rows (token-major, dims contiguous) via ldmatrix.
  const int mi = lane >> 3;
  const int rr = lane & 7;
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) {
    const int token = 8 * (mi >> 1) + rr;
    const int dim0 = 16 * ks + 8 * (mi & 1);
    uint32_t b00, b01, b10, b11;
    ldmatrix_x4(kv_elem_addr(k_base, token, dim0), b00, b01, b10, b11);
    mma_bf16_16816(s[0], qa[ks], b00, b01);
    mma_bf16_16816(s[1], qa[ks], b10, b11);
  }

  float mx[2] = {-INFINITY, -INFINITY};
  if (t.nvalid == kTile && t.pos0 + kTile - 1 <= min(qpos[0], qpos[1])) {
    // every key of the tile is visible to both rows: no masking
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        s[nt][e] *= scale_log2;
        mx[e >> 1] = fmaxf(mx[e >> 1], s[nt][e]);
      }
  } else {
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int i = 8 * nt + 2 * tq + (e & 1);
        const int row = e >> 1;
        const bool ok = i < t.nvalid && t.pos0 + i <= qpos[row];
        const float v = ok ? s[nt][e] * scale_log2 : -INFINITY;
        s[nt][e] = v;
        mx[row] = fmaxf(mx[row], v);
      }
    }
  }
#pragma unroll
  for (int row = 0; row < 2; ++row) {
    mx[row] = fmaxf(mx[row], __shfl_xor_sync(0xffffffffu, mx[row], 1));
    mx[row] = fmaxf(mx[row], __shfl_xor_sync(0xffffffffu, mx[row], 2));
  }
  // lazy rescale: the running max only moves when a score exceeds it by more than
  // 2^8 (p <= 256 otherwise), so O is rescaled on few tiles; m stays the exponent
  // reference of both l and O, so the result and the LSE are unchanged.
  bool bump[2];
  float alpha[2], m_use[2];
#pragma unroll
  for (int row = 0; row < 2; ++row) {
    bump[row] = mx[row] > st.m[row] + 8.f;
    alpha[row] = bump[row] ? exp2f(st.m[row] - mx[row]) : 1.f;
    if (bump[row]) st.m[row] = mx[row];
    m_use[row] = st.m[row] == -INFINITY ? 0.f : st.m[row];
  }
  float p[2][4];
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) p[nt][e] = exp2f(s[nt][e] - m_use[e >> 1]);
#pragma unroll
  for (int row = 0; row < 2; ++row) {
    st.l[row] = st.l[row] * alpha[row] + p[0][2 * row] + p[0][2 * row + 1] + p[1][2 * row] +
                p[1][2 * row + 1];
  }
  if (bump[0]) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      st.o[j][0] *= alpha[0];
      st.o[j][1] *= alpha[0];
    }
  }
  if (bump[1]) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      st.o[j][2] *= alpha[1];
      st.o[j][3] *= alpha[1];
    }
  }
  // P enters the MMA as bf16 hi + lo parts (p = hi + lo to ~2^-17): a single bf16
  // rounding of P would put ~2^-10 relative noise on the output, because the
  // weighted sum of V rows largely cancels.
  uint32_t pa[4], pl[4];
  split_bf16(p[0][0], p[0][1], pa[0], pl[0]);
  split_bf16(p[0][2], p[0][3], pa[1], pl[1]);
  split_bf16(p[1][0], p[1][1], pa[2], pl[2]);
  split_bf16(p[1][2], p[1][3], pa[3], pl[3]);

  // O += P V : B operand = V rows (token-major) via transposed ldmatrix.
#pragma unroll
  for (int j = 0; j < 16; j += 2) {
    const int token = rr + 8 * (mi & 1);
    const int dim0 = 8 * (j + (mi >> 1));
    uint32_t b00, b01, b10, b11;
    ldmatrix_x4_trans(kv_elem_addr(v_base, token, dim0), b00, b01, b10, b11);
    mma_bf16_16816(st.o[j], pa, b00, b01);
    mma_bf16_16816(st.o[j + 1], pa, b10, b11);
    mma_bf16_16816(st.o[j], pl, b00, b01);
    mma_bf16_16816(st.o[j + 1], pl, b10, b11);
  }
}

// Load the A fragments of the warp's 16 query rows; rows >= nrows are zero.
// row r <-> q[(tok0 + r / group) * q_tok_stride + (head0 + r % group) * 128 + d]
CORTEX_DEVICE void load_q_frags(uint32_t (&qa)[8][4], const __nv_bfloat16* __restrict__ q,
                                int64_t tok0, int64_t q_tok_stride, int head0, int group,
                                int nrows) {
  const int lane = lane_id();
  const int g = lane >> 2;
  const int tq = lane & 3;
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int r = g + 8 * half;
    const bool ok = r < nrows;
    const __nv_bfloat16* qrow =
        q + (tok0 + r / group) * q_tok_stride + static_cast<int64_t>(head0 + r % group) * kHeadDim;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const int d = 16 * ks + 2 * tq;
      qa[ks][half] = ok ? *reinterpret_cast<const uint32_t*>(qrow + d) : 0u;
      qa[ks][2 + half] = ok ? *reinterpret_cast<const uint32_t*>(qrow + d + 8) : 0u;
    }
  }
}

CORTEX_DEVICE void quad_reduce_l(WarpState& st) {
#pragma unroll
  for (int row = 0; row < 2; ++row) {
    st.l[row] += __shfl_xor_sync(0xffffffffu, st.l[row], 1);
    st.l[row] += __shfl_xor_sync(0xffffffffu, st.l[row], 2);
  }
}

CORTEX_DEVICE void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// ---------------------------------------------------------------------------
// decode: one query token per sequence, grid (split, kv_head, seq)

struct DecodeArgs {
  const __nv_bfloat16* q;  // [B, Hq, 128]
  const int* table;        // [rows, table_stride]
  int table_stride;
  const int* seq_row;      // [B]
  const int* seq_prefix;   // [B]
  const int* seq_kvlen;    // [B]
  int n_kv_heads;
  int group;
  int64_t k_row0, v_row0;
  float scale_log2;
  float* o_part;    // [B, max_splits, Hq, 128]
  float* lse_part;  // [B, max_splits, Hq]
  int max_splits;   // slots per sequence
  int cascade;      // 1: prefix tiles are handled by the shared-prefix kernel
  int slot_off;     // first slot of the private splits (cascade only)
};

constexpr int kDecodeStages = CORTEX_DECODE_STAGES;
constexpr int kPrefillStages = 3;

// Decode warps run the m16n8k16 MMA key-major: a decode warp has only `group` (<= 8)
// query rows per kv head, so S^T = K Q^T (16 keys x 8 query columns per MMA) and
// O^T += V^T P^T (16 dims x 8 columns) need half the MMAs and accumulator registers
// of the query-major layout (which would pad 4 rows to 16). P^T moves from the
// accumulator layout to the B-operand layout with movmatrix.

CORTEX_DEVICE uint32_t movmatrix_trans(uint32_t a) {
  uint32_t d;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;\n" : "=r"(d) : "r"(a));
  return d;
}

// Online-softmax state of one decode warp for query columns 2tq, 2tq+1 (tq = lane % 4).
// l holds this lane's keys only (reduced over the 8 lanes of a column at the end);
// o[db]: (dim 16db+g, col 2tq), (16db+g, 2tq+1), (16db+g+8, 2tq), (16db+g+8, 2tq+1).
struct DecState {
  float m[2];
  float l[2];
  float o[8][4];
};

CORTEX_DEVICE void dec_state_init(DecState& st) {
  st.m[0] = st.m[1] = -INFINITY;
  st.l[0] = st.l[1] = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int e = 0; e < 4; ++e) st.o[j][e] = 0.f;
}

// Q^T as B fragments: column g = query head g of the kv head (zero when g >= group).
CORTEX_DEVICE void load_q_cols(uint32_t (&qb)[8][2], const __nv_bfloat16* __restrict__ q,
                               int64_t base, int group) {
  const int lane = lane_id();
  const int g = lane >> 2;
  const int tq = lane & 3;
  const bool ok = g < group;
  const __nv_bfloat16* qrow = q + base + static_cast<int64_t>(g) * kHeadDim;
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) {
    qb[ks][0] = ok ? *reinterpret_cast<const uint32_t*>(qrow + 16 * ks + 2 * tq) : 0u;
    qb[ks][1] = ok ? *reinterpret_cast<const uint32_t*>(qrow + 16 * ks + 8 + 2 * tq) : 0u;
  }
}

// One 16-key tile; keys [0, nvalid) of the tile are visible to every query column.
CORTEX_DEVICE void attend_tile_dec(DecState& st, const uint32_t (&qb)[8][2], uint32_t stage_addr,
                                   int nvalid, float scale_log2) {
  const int lane = lane_id();
  const int g = lane >> 2;
  const uint32_t k_base = stage_addr;
  const uint32_t v_base = stage_addr + kTileBytes;
  // (key g, col 2tq), (g, 2tq+1), (g+8, 2tq), (g+8, 2tq+1); two accumulation chains
  float s[4] = {0.f, 0.f, 0.f, 0.f}, s2[4] = {0.f, 0.f, 0.f, 0.f};
  const int ktok = (lane & 7) + 8 * ((lane >> 3) & 1);
  const int kdim = 8 * (lane >> 4);
#pragma unroll
  for (int ks = 0; ks < 8; ks += 2) {
    uint32_t a[4], a2[4];
    ldmatrix_x4(kv_elem_addr(k_base, ktok, 16 * ks + kdim), a[0], a[1], a[2], a[3]);
    ldmatrix_x4(kv_elem_addr(k_base, ktok, 16 * ks + 16 + kdim), a2[0], a2[1], a2[2], a2[3]);
    mma_bf16_16816(s, a, qb[ks][0], qb[ks][1]);
    mma_bf16_16816(s2, a2, qb[ks + 1][0], qb[ks + 1][1]);
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) s[e] += s2[e];
  float mx[2];
  if (nvalid == kTile) {
#pragma unroll
    for (int e = 0; e < 4; ++e) s[e] *= scale_log2;
  } else {
    s[0] = g < nvalid ? s[0] * scale_log2 : -INFINITY;
    s[1] = g < nvalid ? s[1] * scale_log2 : -INFINITY;
    s[2] = g + 8 < nvalid ? s[2] * scale_log2 : -INFINITY;
    s[3] = g + 8 < nvalid ? s[3] * scale_log2 : -INFINITY;
  }
  mx[0] = fmaxf(s[0], s[2]);
  mx[1] = fmaxf(s[1], s[3]);
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    mx[c] = fmaxf(mx[c], __shfl_xor_sync(0xffffffffu, mx[c], 4));
    mx[c] = fmaxf(mx[c], __shfl_xor_sync(0xffffffffu, mx[c], 8));
    mx[c] = fmaxf(mx[c], __shfl_xor_sync(0xffffffffu, mx[c], 16));
  }
  // lazy rescale (see attend_tile): the reference max moves only by > 2^8
  bool bump[2];
  float alpha[2], m_use[2];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    bump[c] = mx[c] > st.m[c] + 8.f;
    alpha[c] = bump[c] ? exp2f(st.m[c] - mx[c]) : 1.f;
    if (bump[c]) st.m[c] = mx[c];
    m_use[c] = st.m[c] == -INFINITY ? 0.f : st.m[c];
  }
  float p[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) p[e] = exp2f(s[e] - m_use[e & 1]);
  st.l[0] = st.l[0] * alpha[0] + p[0] + p[2];
  st.l[1] = st.l[1] * alpha[1] + p[1] + p[3];
  if (bump[0] || bump[1]) {
#pragma unroll
    for (int db = 0; db < 8; ++db) {
      st.o[db][0] *= alpha[0];
      st.o[db][1] *= alpha[1];
      st.o[db][2] *= alpha[0];
      st.o[db][3] *= alpha[1];
    }
  }
  // P^T in bf16 hi + lo (see attend_tile), moved to the B layout: keys 0-7 / 8-15
  uint32_t h0, l0, h1, l1;
  split_bf16(p[0], p[1], h0, l0);
  split_bf16(p[2], p[3], h1, l1);
  const uint32_t bh0 = movmatrix_trans(h0), bh1 = movmatrix_trans(h1);
  const uint32_t bl0 = movmatrix_trans(l0), bl1 = movmatrix_trans(l1);
  const int vtok = (lane & 7) + 8 * (lane >> 4);
  const int vdim = 8 * ((lane >> 3) & 1);
  uint32_t a[8][4];  // all V^T fragments first, then the hi pass, then the lo pass
#pragma unroll
  for (int db = 0; db < 8; ++db)
    ldmatrix_x4_trans(kv_elem_addr(v_base, vtok, 16 * db + vdim), a[db][0], a[db][1], a[db][2],
                      a[db][3]);
#pragma unroll
  for (int db = 0; db < 8; ++db) mma_bf16_16816(st.o[db], a[db], bh0, bh1);
#pragma unroll
  for (int db = 0; db < 8; ++db) mma_bf16_16816(st.o[db], a[db], bl0, bl1);
}

// Write a warp's state for the cross-warp merge: cm/cl [warp][8], co [warp][co_rows][128].
CORTEX_DEVICE void dec_state_store(DecState& st, int warp, int group, float* cm, float* cl,
                                   float* co, int co_rows) {
  const int lane = lane_id();
  const int g = lane >> 2;
  const int tq = lane & 3;
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    st.l[c] += __shfl_xor_sync(0xffffffffu, st.l[c], 4);
    st.l[c] += __shfl_xor_sync(0xffffffffu, st.l[c], 8);
    st.l[c] += __shfl_xor_sync(0xffffffffu, st.l[c], 16);
  }
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const int col = 2 * tq + c;
    if (col < group) {
      if (g == 0) {
        cm[warp * 8 + col] = st.m[c];
        cl[warp * 8 + col] = st.l[c];
      }
      float* dst = co + (warp * co_rows + col) * kHeadDim;
#pragma unroll
      for (int db = 0; db < 8; ++db) {
        dst[16 * db + g] = st.o[db][c];
        dst[16 * db + g + 8] = st.o[db][2 + c];
      }
    }
  }
}

// After a barrier: merge the 4 warps' states of query heads [0, group) and write the
// partial (normalised O, LSE) of slot `slot` of call b.
CORTEX_DEVICE void dec_merge_emit(const float* cm, const float* cl, const float* co, int co_rows,
                                  const DecodeArgs& a, int b, int kvh, int slot) {
  const int hq = a.n_kv_heads * a.group;
  for (int idx = threadIdx.x; idx < a.group * kHeadDim; idx += blockDim.x) {
    const int r = idx / kHeadDim;
    const int d = idx % kHeadDim;
    float M = -INFINITY;
    for (int w = 0; w < kWarps; ++w) M = fmaxf(M, cm[w * 8 + r]);
    float L = 0.f, O = 0.f;
    for (int w = 0; w < kWarps; ++w) {
      // a warp without keys (a split shorter than 4 tiles) left its O rows unwritten
      // (stale stage bytes, possibly NaN patterns): skip it rather than scale it by 0
      if (cm[w * 8 + r] == -INFINITY) continue;
      const float f = exp2f(cm[w * 8 + r] - M);
      L += cl[w * 8 + r] * f;
      O += co[(w * co_rows + r) * kHeadDim + d] * f;
    }
    const int h = kvh * a.group + r;
    const int64_t pidx = (static_cast<int64_t>(b) * a.max_splits + slot) * hq + h;
    a.o_part[pidx * kHeadDim + d] = O / L;
    if (d == 0) a.lse_part[pidx] = M + log2f(L);
  }
}

// Visible keys of tile j of a call (prefix segment, then private segment).
CORTEX_DEVICE int tile_nvalid(int prefix, int kvlen, int j) {
  const int npb = (prefix + kTile - 1) / kTile;
  return j < npb ? min(kTile, prefix - j * kTile) : min(kTile, kvlen - prefix - (j - npb) * kTile);
}

__global__ void __launch_bounds__(kWarps * 32)
    paged_decode_kernel(const __grid_constant__ CUtensorMap tmap_kv, const DecodeArgs a) {
  // Before the PDL wait this kernel reads only what earlier steps or earlier kernels of
  // this step wrote (call metadata, block table, the KV of past tokens): every kernel of
  // the stream waits for its own predecessor before it triggers, so only the immediate
  // predecessor (RoPE / KV append: q and the new token's K/V in the call's last tile)
  // can still be running. The last tile's load and q wait for it.
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const int split = blockIdx.x;
  const int kvh = blockIdx.y;
  const int b = blockIdx.z;
  const int row = __ldg(&a.seq_row[b]);
  const int prefix = __ldg(&a.seq_prefix[b]);
  const int kvlen = __ldg(&a.seq_kvlen[b]);
  const int ntiles = num_tiles(prefix, kvlen);
  const int first_tile = a.cascade ? (prefix + kTile - 1) / kTile : 0;
  const int t_begin = first_tile + split * kTilesPerSplit;
  if (t_begin >= ntiles) {
    pdl_wait();
    pdl_trigger();
    return;
  }
  const int t_end = min(ntiles, t_begin + kTilesPerSplit);
  const int warp = warp_id();
  const int lane = lane_id();
  const int hq = a.n_kv_heads * a.group;

  uint8_t* my_stages = smem + warp * kDecodeStages * kStageBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kWarps * kDecodeStages * kStageBytes) +
                   warp * kDecodeStages;
  if (lane == 0) {
    for (int s = 0; s < kDecodeStages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  // this warp's tiles: t_begin + warp + 4 i; their block ids in one round trip (lane i)
  const int n_mine = (t_end - t_begin - warp + kWarps - 1) / kWarps;
  const int* table_row = a.table + static_cast<int64_t>(row) * a.table_stride;
  static_assert(kTilesPerSplit / kWarps <= 32, "block ids are held one per lane");
  const int my_blk = lane < n_mine ? __ldg(&table_row[t_begin + warp + kWarps * lane]) : 0;
  __syncwarp();
  int deferred = -1;  // stage of the last tile (the new token's K/V), loaded after the wait
#pragma unroll
  for (int i = 0; i < kDecodeStages; ++i) {
    const int blk = __shfl_sync(0xffffffffu, my_blk, i);
    if (i < n_mine && t_begin + warp + kWarps * i == ntiles - 1)
      deferred = i;
    else if (lane == 0 && i < n_mine)
      load_tile(my_stages + i * kStageBytes, &tmap_kv, &bars[i], a.k_row0, a.v_row0, blk, kvh,
                a.n_kv_heads);
  }
  pdl_wait();
  pdl_trigger();
  const int dblk = __shfl_sync(0xffffffffu, my_blk, deferred >= 0 ? deferred : 0);
  if (deferred >= 0 && lane == 0)
    load_tile(my_stages + deferred * kStageBytes, &tmap_kv, &bars[deferred], a.k_row0, a.v_row0,
              dblk, kvh, a.n_kv_heads);

  uint32_t qb[8][2];
  load_q_cols(qb, a.q, (static_cast<int64_t>(b) * hq + kvh * a.group) * kHeadDim, a.group);
  DecState st;
  dec_state_init(st);

  for (int i = 0; i < n_mine; ++i) {
    const int s = i % kDecodeStages;
    const int nvalid = tile_nvalid(prefix, kvlen, t_begin + warp + kWarps * i);
    mbar_wait(&bars[s], (i / kDecodeStages) & 1);
    attend_tile_dec(st, qb, smem_u32(my_stages + s * kStageBytes), nvalid, a.scale_log2);
    __syncwarp();
    const int nxt = i + kDecodeStages;
    const int blk = __shfl_sync(0xffffffffu, my_blk, nxt & 31);
    if (nxt < n_mine && lane == 0) {
      fence_proxy_async();
      load_tile(my_stages + s * kStageBytes, &tmap_kv, &bars[s], a.k_row0, a.v_row0, blk, kvh,
                a.n_kv_heads);
    }
    __syncwarp();
  }

  // merge the 4 warps through shared memory (the stage buffers are idle now)
  __syncthreads();
  float* cm = reinterpret_cast<float*>(smem);  // [4][8]
  float* cl = cm + kWarps * 8;                 // [4][8]
  float* co = cl + kWarps * 8;                 // [4][8][128]
  if (n_mine > 0) {
    dec_state_store(st, warp, a.group, cm, cl, co, 8);
  } else if (lane < 8) {
    cm[warp * 8 + lane] = -INFINITY;
    cl[warp * 8 + lane] = 0.f;
  }
  __syncthreads();
  dec_merge_emit(cm, cl, co, 8, a, b, kvh, (a.cascade ? a.slot_off : 0) + split);
}

// ---------------------------------------------------------------------------
// balanced decode ("flat"): the calls' tiles (private tiles under cascade) are laid
// end to end - call b owns flat tiles [tile_start[b], tile_start[b] + n_b) - and CTA
// (c, kv_head) streams the fixed-size range [c W, (c+1) W) of that sequence,
// whatever calls it crosses. Every CTA does the same work and lives for W tiles, so
// the 2-deep per-warp TMA rings stay full across call boundaries. The range's calls,
// their metadata and block ids are staged in shared memory up front; at each call
// boundary the 4 warps merge their online-softmax states and write the call's
// partial into slot (slot_off + c - tile_start[b] / W), merged by the combine kernel.

struct FlatArgs {
  DecodeArgs d;
  const int* tile_start;  // [B] exclusive prefix sum of per-call tile counts
  int n_seqs;
  int W;      // tiles per chunk
  int total;  // tiles of all calls
};

constexpr int kFlatMaxW = 48;
constexpr int kFlatStatic = 2048;  // bytes of the static shared block
static_assert((5 * (kFlatMaxW + 1) + kFlatMaxW + 2 + 2 * kWarps * 8) * 4 +
                      kWarps * kDecodeStages * 8 <= kFlatStatic,
              "flat decode metadata exceeds its static shared block");

CORTEX_DEVICE int call_tiles(int prefix, int kvlen, int cascade) {
  const int npb = (prefix + kTile - 1) / kTile;
  const int npriv = (kvlen - prefix + kTile - 1) / kTile;
  return cascade ? npriv : npb + npriv;
}

// dynamic part: stages + the cross-warp merge area (the rest is the static block)
inline size_t flat_smem_bytes(int group) {
  return kWarps * kDecodeStages * kStageBytes + static_cast<size_t>(kWarps) * group * kHeadDim * 4;
}

__global__ void __launch_bounds__(kWarps * 32)
    paged_decode_flat_kernel(const __grid_constant__ CUtensorMap tmap_kv, const FlatArgs f) {
  pdl_wait();
  pdl_trigger();
  const DecodeArgs& a = f.d;
  // Shared memory: a 2 KiB static block (metadata, barriers, merge scalars), then the
  // dynamic stages + merge area starting 1 KiB-aligned (the SW128 TMA boxes need it).
  __shared__ __align__(1024) int meta[kFlatStatic / 4];
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if ((smem_u32(smem_raw) & 1023) != 0) __trap();
  const int c = blockIdx.x;
  const int kvh = blockIdx.y;
  const int t0 = c * f.W;
  if (t0 >= f.total) return;
  const int t1 = min(f.total, t0 + f.W);
  const int warp = warp_id();
  const int lane = lane_id();
  const int tid = threadIdx.x;
  const int hq = a.n_kv_heads * a.group;

  uint8_t* stages = smem_raw;
  float* co = reinterpret_cast<float*>(smem_raw + kWarps * kDecodeStages * kStageBytes);
  int* m_S = meta;  // [kFlatMaxW + 1] each
  int* m_first = m_S + (kFlatMaxW + 1);
  int* m_n = m_first + (kFlatMaxW + 1);
  int* m_row = m_n + (kFlatMaxW + 1);
  int* m_kvlen = m_row + (kFlatMaxW + 1);
  int* blk = m_kvlen + (kFlatMaxW + 1);  // [kFlatMaxW]
  int* cnt = blk + kFlatMaxW;            // [2]
  float* cm = reinterpret_cast<float*>(cnt + 2);  // [4][8]
  float* cl = cm + kWarps * 8;                    // [4][8]
  uint64_t* bars = reinterpret_cast<uint64_t*>(meta + kFlatStatic / 4 - 2 * kWarps * kDecodeStages);

  if (tid < 2) cnt[tid] = 0;
  if (lane == 0) {
    for (int s = 0; s < kDecodeStages; ++s) mbar_init(&bars[warp * kDecodeStages + s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  // calls crossing [t0, t1): b0 = #{S_b <= t0} - 1 ... #{S_b < t1} - 1
  int n0 = 0, n1 = 0;
  for (int b = tid; b < f.n_seqs; b += blockDim.x) {
    const int s = __ldg(&f.tile_start[b]);
    n0 += s <= t0;
    n1 += s < t1;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    n0 += __shfl_xor_sync(0xffffffffu, n0, o);
    n1 += __shfl_xor_sync(0xffffffffu, n1, o);
  }
  if (lane == 0) {
    atomicAdd(&cnt[0], n0);
    atomicAdd(&cnt[1], n1);
  }
  __syncthreads();
  const int b0 = cnt[0] - 1;
  const int nc = cnt[1] - b0;
  for (int k = tid; k < nc; k += blockDim.x) {
    const int b = b0 + k;
    const int prefix = __ldg(&a.seq_prefix[b]);
    const int kvlen = __ldg(&a.seq_kvlen[b]);
    m_S[k] = __ldg(&f.tile_start[b]);
    m_first[k] = a.cascade ? (prefix + kTile - 1) / kTile : 0;
    m_n[k] = call_tiles(prefix, kvlen, a.cascade);
    m_row[k] = __ldg(&a.seq_row[b]);
    m_kvlen[k] = kvlen;
  }
  __syncthreads();
  for (int t = t0 + tid; t < t1; t += blockDim.x) {
    int lo = 0, hi = nc - 1;  // last k with m_S[k] <= t
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (m_S[mid] <= t) lo = mid; else hi = mid - 1;
    }
    blk[t - t0] = __ldg(&a.table[static_cast<int64_t>(m_row[lo]) * a.table_stride + m_first[lo] +
                                 (t - m_S[lo])]);
  }
  __syncthreads();

  auto lo_of = [&](int k) { return max(t0, m_S[k]); };
  auto hi_of = [&](int k) { return min(t1, m_S[k] + m_n[k]); };
  // this warp's tiles: lo_of(k) + warp + 4 i < hi_of(k), portion after portion
  int lk = 0, lt = lo_of(0) + warp;
  auto advance = [&]() {
    while (lk < nc && lt >= hi_of(lk)) {
      ++lk;
      if (lk < nc) lt = lo_of(lk) + warp;
    }
  };
  advance();
  uint8_t* my_stages = stages + warp * kDecodeStages * kStageBytes;
  uint64_t* my_bars = bars + warp * kDecodeStages;
  for (int s = 0; s < kDecodeStages && lk < nc; ++s) {
    if (lane == 0)
      load_tile(my_stages + s * kStageBytes, &tmap_kv, &my_bars[s], a.k_row0, a.v_row0,
                blk[lt - t0], kvh, a.n_kv_heads);
    lt += kWarps;
    advance();
  }

  int consumed = 0;
  for (int k = 0; k < nc; ++k) {
    const int b = b0 + k;
    const int lo = lo_of(k), hi = hi_of(k);
    const int kvlen = m_kvlen[k];
    const int prefix = __ldg(&a.seq_prefix[b]);
    uint32_t qb[8][2];
    load_q_cols(qb, a.q, (static_cast<int64_t>(b) * hq + kvh * a.group) * kHeadDim, a.group);
    DecState st;
    dec_state_init(st);
    for (int t = lo + warp; t < hi; t += kWarps) {
      const int s = consumed % kDecodeStages;
      const int nvalid = tile_nvalid(prefix, kvlen, m_first[k] + (t - m_S[k]));
      mbar_wait(&my_bars[s], (consumed / kDecodeStages) & 1);
      attend_tile_dec(st, qb, smem_u32(my_stages + s * kStageBytes), nvalid, a.scale_log2);
      __syncwarp();
      ++consumed;
      if (lk < nc) {
        if (lane == 0) {
          fence_proxy_async();
          load_tile(my_stages + s * kStageBytes, &tmap_kv, &my_bars[s], a.k_row0, a.v_row0,
                    blk[lt - t0], kvh, a.n_kv_heads);
        }
        lt += kWarps;
        advance();
      }
      __syncwarp();
    }
    dec_state_store(st, warp, a.group, cm, cl, co, a.group);  // (idle warp: m = -inf)
    __syncthreads();
    dec_merge_emit(cm, cl, co, a.group, a, b, kvh,
                   (a.cascade ? a.slot_off : 0) + c - m_S[k] / f.W);
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// shared-prefix ("cascade") decode attention: every decode query of the calls that
// share one resident stage prefix attends to that prefix in one pass, so the
// prefix's KV is read once per step instead of once per call. Grid
// (query chunk, kv_head, group * max_psplits); each warp owns 16/group calls x
// group heads; prefix tiles are split in 16-tile chunks (partials -> slots 0..).

struct CascadeArgs {
  const __nv_bfloat16* q;  // [B, Hq, 128] decode queries, groups contiguous
  const int* table;
  int table_stride;
  const int* grp_row;    // prefix's table row
  const int* grp_plen;   // prefix tokens
  const int* grp_first;  // first decode index of the group
  const int* grp_count;  // decode calls in the group
  int max_psplits;
  int n_kv_heads;
  int group;
  int64_t k_row0, v_row0;
  float scale_log2;
  float* o_part;
  float* lse_part;
  int max_splits;  // slots per sequence
};

__global__ void __launch_bounds__(kWarps * 32)
    cascade_prefix_kernel(const __grid_constant__ CUtensorMap tmap_kv, const CascadeArgs a) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const int chunk = blockIdx.x;
  const int kvh = blockIdx.y;
  const int gi = blockIdx.z / a.max_psplits;
  const int ps = blockIdx.z % a.max_psplits;
  const int seqs_per_warp = 16 / a.group;
  const int seqs_per_cta = seqs_per_warp * kWarps;
  const int count = __ldg(&a.grp_count[gi]);
  const int s0 = chunk * seqs_per_cta;
  if (s0 >= count) return;
  const int plen = __ldg(&a.grp_plen[gi]);
  const int npb = (plen + kTile - 1) / kTile;
  const int psb = prefix_split_blocks(npb, a.max_psplits);
  const int t_begin = ps * psb;
  if (t_begin >= npb) return;
  const int t_end = min(npb, t_begin + psb);
  const int ntl = t_end - t_begin;
  const int first = __ldg(&a.grp_first[gi]);
  const int row = __ldg(&a.grp_row[gi]);
  const int warp = warp_id();
  const int lane = lane_id();
  const int hq = a.n_kv_heads * a.group;

  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kPrefillStages * kStageBytes);
  uint64_t* empty = full + kPrefillStages;
  if (threadIdx.x == 0) {
    for (int st = 0; st < kPrefillStages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int* table_row = a.table + static_cast<int64_t>(row) * a.table_stride;
  if (threadIdx.x == 0) {
    for (int i = 0; i < min(ntl, kPrefillStages); ++i) {
      const TileRef t = tile_ref(table_row, plen, plen, t_begin + i);
      load_tile(smem + i * kStageBytes, &tmap_kv, &full[i], a.k_row0, a.v_row0, t.block, kvh,
                a.n_kv_heads);
    }
  }
  const int ws0 = s0 + warp * seqs_per_warp;  // first call (within group) of this warp
  const int wn = max(0, min(seqs_per_warp, count - ws0));
  uint32_t qa[8][4];
  load_q_frags(qa, a.q, static_cast<int64_t>(first) + ws0, static_cast<int64_t>(hq) * kHeadDim,
               kvh * a.group, a.group, wn * a.group);
  WarpState st;
  state_init(st);
  const int qpos[2] = {0x7fffffff, 0x7fffffff};  // decode queries follow the whole prefix
  for (int i = 0; i < ntl; ++i) {
    const int sidx = i % kPrefillStages;
    const TileRef t = tile_ref(table_row, plen, plen, t_begin + i);
    mbar_wait(&full[sidx], (i / kPrefillStages) & 1);
    if (wn > 0) attend_tile(st, qa, smem_u32(smem + sidx * kStageBytes), t, qpos, a.scale_log2);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[sidx]);
    const int nxt = i + kPrefillStages;
    if (threadIdx.x == 0 && nxt < ntl) {
      mbar_wait(&empty[sidx], (i / kPrefillStages) & 1);
      fence_proxy_async();
      const TileRef tn = tile_ref(table_row, plen, plen, t_begin + nxt);
      load_tile(smem + sidx * kStageBytes, &tmap_kv, &full[sidx], a.k_row0, a.v_row0, tn.block,
                kvh, a.n_kv_heads);
    }
    __syncwarp();
  }
  quad_reduce_l(st);
  const int g = lane >> 2;
  const int tq = lane & 3;
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int r = g + 8 * half;
    if (r < wn * a.group) {
      const int b = first + ws0 + r / a.group;
      const int h = kvh * a.group + r % a.group;
      const int64_t pidx = (static_cast<int64_t>(b) * a.max_splits + ps) * hq + h;
      const float inv = 1.f / st.l[half];
      float* o = a.o_part + pidx * kHeadDim;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int d = 8 * j + 2 * tq;
        *reinterpret_cast<float2*>(o + d) =
            make_float2(st.o[j][2 * half] * inv, st.o[j][2 * half + 1] * inv);
      }
      if (tq == 0) a.lse_part[pidx] = st.m[half] + log2f(st.l[half]);
    }
  }
}

struct CombineArgs {
  const float* o_part;
  const float* lse_part;
  const int* seq_prefix;
  const int* seq_kvlen;
  __nv_bfloat16* out;  // [B, Hq, 128]
  int hq;
  int max_splits;
  int cascade;
  int slot_off;
  const int* tile_start;  // flat plan (null: per-call splits of kTilesPerSplit tiles)
  int W;
};

// LSE merge of a call's partials: grid (call, head / 8), warp <-> head, lane <-> 4 dims.
// Up to 8 slots: the LSEs (lane <-> slot) and all partial rows are loaded at once, so a
// head costs one memory round trip; more slots take the general loop.
constexpr int kCombineThreads = 256;

__global__ void __launch_bounds__(kCombineThreads) decode_combine_kernel(const CombineArgs a) {
  pdl_wait();
  pdl_trigger();
  const int b = blockIdx.x;
  const int warp = warp_id();
  const int lane = lane_id();
  const int prefix = __ldg(&a.seq_prefix[b]);
  const int ntiles = num_tiles(prefix, __ldg(&a.seq_kvlen[b]));
  // slot ranges: [0, np) prefix partials (cascade), [off, off + ns) context splits
  int np = 0, off = 0, ns;
  if (a.cascade) {
    const int npb = (prefix + kTile - 1) / kTile;
    const int psb = npb ? prefix_split_blocks(npb, a.slot_off) : 1;
    np = (npb + psb - 1) / psb;
    off = a.slot_off;
    ns = (ntiles - npb + kTilesPerSplit - 1) / kTilesPerSplit;
  } else {
    ns = (ntiles + kTilesPerSplit - 1) / kTilesPerSplit;
  }
  if (a.tile_start) {  // pieces = chunks of W flat tiles that the call's range crosses
    const int S = __ldg(&a.tile_start[b]);
    const int n = call_tiles(prefix, __ldg(&a.seq_kvlen[b]), a.cascade);
    ns = (S + n - 1) / a.W - S / a.W + 1;
  }
  const int nsl = np + ns;
  const int64_t base = static_cast<int64_t>(b) * a.max_splits;
  auto slot = [&](int i) { return i < np ? i : off + (i - np); };
  constexpr int kWarpsC = kCombineThreads / 32;
  for (int h = blockIdx.y * kWarpsC + warp; h < a.hq; h += gridDim.y * kWarpsC) {
    if (nsl <= 8) {
      // common case: every load of the head issued at once (one memory round trip)
      const float lse_i = lane < nsl ? a.lse_part[(base + slot(lane)) * a.hq + h] : -INFINITY;
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (u < nsl)
          v[u] = *reinterpret_cast<const float4*>(
              a.o_part + ((base + slot(u)) * a.hq + h) * kHeadDim + 4 * lane);
      float M = lse_i;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
      const float w = lane < nsl ? exp2f(lse_i - M) : 0.f;
      float L = w;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const float wu = __shfl_sync(0xffffffffu, w, u);
        if (u < nsl) {
          acc.x += wu * v[u].x;
          acc.y += wu * v[u].y;
          acc.z += wu * v[u].z;
          acc.w += wu * v[u].w;
        }
      }
      const float inv = 1.f / L;
      uint2 packed;
      packed.x = pack_bf16(acc.x * inv, acc.y * inv);
      packed.y = pack_bf16(acc.z * inv, acc.w * inv);
      *reinterpret_cast<uint2*>(a.out + (static_cast<int64_t>(b) * a.hq + h) * kHeadDim +
                                4 * lane) = packed;
      continue;
    }
    float M = -INFINITY;
    for (int i = lane; i < nsl; i += 32) M = fmaxf(M, a.lse_part[(base + slot(i)) * a.hq + h]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    float L = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int i0 = 0; i0 < nsl; i0 += 32) {
      const int i = i0 + lane;
      const float w = i < nsl ? exp2f(a.lse_part[(base + slot(i)) * a.hq + h] - M) : 0.f;
      L += w;
      const int cnt = min(32, nsl - i0);
      for (int j = 0; j < cnt; j += 4) {
        float4 v[4];
        float wj[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          wj[u] = __shfl_sync(0xffffffffu, w, (j + u) & 31);
          if (j + u < cnt)
            v[u] = *reinterpret_cast<const float4*>(
                a.o_part + ((base + slot(i0 + j + u)) * a.hq + h) * kHeadDim + 4 * lane);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (j + u < cnt) {
            acc.x += wj[u] * v[u].x;
            acc.y += wj[u] * v[u].y;
            acc.z += wj[u] * v[u].z;
            acc.w += wj[u] * v[u].w;
          }
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
    const float inv = 1.f / L;
    uint2 packed;
    packed.x = pack_bf16(acc.x * inv, acc.y * inv);
    packed.y = pack_bf16(acc.z * inv, acc.w * inv);
    *reinterpret_cast<uint2*>(a.out + (static_cast<int64_t>(b) * a.hq + h) * kHeadDim + 4 * lane) =
        packed;
  }
}

// ---------------------------------------------------------------------------
// prefill: many query tokens per sequence, causal over prefix + own tokens.
// grid (q_chunk, kv_head, seq); each warp owns 16/group query tokens x group heads.

struct PrefillArgs {
  const __nv_bfloat16* q;  // [T, Hq, 128]
  __nv_bfloat16* out;      // [T, Hq, 128]
  const int* table;
  int table_stride;
  const int* seq_row;
  const int* seq_prefix;
  const int* seq_kvlen;
  const int* seq_qstart;  // first query row in q/out
  const int* seq_qlen;    // query tokens (the last q_len positions of the sequence)
  int n_kv_heads;
  int group;
  int64_t k_row0, v_row0;
  float scale_log2;
};


__global__ void __launch_bounds__(kWarps * 32)
    paged_prefill_kernel(const __grid_constant__ CUtensorMap tmap_kv, const PrefillArgs a) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const int chunk = blockIdx.x;
  const int kvh = blockIdx.y;
  const int sidx = blockIdx.z;
  const int toks_per_warp = 16 / a.group;
  const int toks_per_cta = toks_per_warp * kWarps;
  const int qlen = __ldg(&a.seq_qlen[sidx]);
  const int q0 = chunk * toks_per_cta;
  if (q0 >= qlen) return;
  const int row = __ldg(&a.seq_row[sidx]);
  const int prefix = __ldg(&a.seq_prefix[sidx]);
  const int kvlen = __ldg(&a.seq_kvlen[sidx]);
  const int qstart = __ldg(&a.seq_qstart[sidx]);
  const int pos_first = kvlen - qlen;  // logical position of query 0
  const int warp = warp_id();
  const int lane = lane_id();
  const int hq = a.n_kv_heads * a.group;

  // keys needed: positions <= pos of the last query in this CTA
  const int q_last = min(qlen, q0 + toks_per_cta) - 1;
  const int pos_last = pos_first + q_last;
  // tiles covering positions [0, pos_last]
  const int npb = (prefix + kTile - 1) / kTile;
  int ntiles;
  if (pos_last < prefix) ntiles = pos_last / kTile + 1;
  else ntiles = npb + (pos_last - prefix) / kTile + 1;

  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kPrefillStages * kStageBytes);
  uint64_t* empty = full + kPrefillStages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kPrefillStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int* table_row = a.table + static_cast<int64_t>(row) * a.table_stride;
  if (threadIdx.x == 0) {
    for (int i = 0; i < min(ntiles, kPrefillStages); ++i) {
      const TileRef t = tile_ref(table_row, prefix, kvlen, i);
      load_tile(smem + i * kStageBytes, &tmap_kv, &full[i], a.k_row0, a.v_row0, t.block, kvh,
                a.n_kv_heads);
    }
  }

  const int wq0 = q0 + warp * toks_per_warp;  // first query token of this warp
  const int wq_n = max(0, min(toks_per_warp, qlen - wq0));
  uint32_t qa[8][4];
  load_q_frags(qa, a.q, static_cast<int64_t>(qstart) + wq0, static_cast<int64_t>(hq) * kHeadDim,
               kvh * a.group, a.group, wq_n * a.group);
  WarpState st;
  state_init(st);
  const int g = lane >> 2;
  int qpos[2];
  qpos[0] = pos_first + wq0 + g / a.group;
  qpos[1] = pos_first + wq0 + (g + 8) / a.group;

  for (int i = 0; i < ntiles; ++i) {
    const int s = i % kPrefillStages;
    const TileRef t = tile_ref(table_row, prefix, kvlen, i);
    mbar_wait(&full[s], (i / kPrefillStages) & 1);
    if (wq_n > 0) attend_tile(st, qa, smem_u32(smem + s * kStageBytes), t, qpos, a.scale_log2);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    const int nxt = i + kPrefillStages;
    if (threadIdx.x == 0 && nxt < ntiles) {
      mbar_wait(&empty[s], (i / kPrefillStages) & 1);
      fence_proxy_async();
      const TileRef tn = tile_ref(table_row, prefix, kvlen, nxt);
      load_tile(smem + s * kStageBytes, &tmap_kv, &full[s], a.k_row0, a.v_row0, tn.block, kvh,
                a.n_kv_heads);
    }
    __syncwarp();
  }
  quad_reduce_l(st);

  const int tq = lane & 3;
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int r = g + 8 * half;
    const int tok = wq0 + r / a.group;
    if (r < wq_n * a.group && tok < qlen) {
      const float inv = 1.f / st.l[half];
      __nv_bfloat16* orow = a.out + (static_cast<int64_t>(qstart) + tok) * hq * kHeadDim +
                            static_cast<int64_t>(kvh * a.group + r % a.group) * kHeadDim;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int d = 8 * j + 2 * tq;
        *reinterpret_cast<uint32_t*>(orow + d) =
            pack_bf16(st.o[j][2 * half] * inv, st.o[j][2 * half + 1] * inv);
      }
    }
  }
}

}  // namespace

extern "C" {

// Split count the decode kernel uses for a sequence (host sizing helper).
int32_t cortex_decode_splits(int32_t prefix_len, int32_t kv_len) {
  const int npb = (prefix_len + kTile - 1) / kTile;
  const int nt = npb + (kv_len - prefix_len + kTile - 1) / kTile;
  return (nt + kTilesPerSplit - 1) / kTilesPerSplit;
}

int32_t cortex_paged_decode_attn(
    const void* tmap_kv, const void* q, const int32_t* table, int32_t table_stride,
    const int32_t* seq_row, const int32_t* seq_prefix, const int32_t* seq_kvlen,
    const int32_t* seq_tile_start, int32_t total_tiles, int32_t tiles_per_chunk, int32_t n_seqs,
    int32_t n_kv_heads, int32_t group, int64_t k_row0, int64_t v_row0, float softmax_scale,
    float* o_part, float* lse_part, int32_t max_splits, void* out, const int32_t* grp_row,
    const int32_t* grp_plen, const int32_t* grp_first, const int32_t* grp_count, int32_t n_groups,
    int32_t max_group_count, int32_t prefix_slots, const void* tmap_q, int32_t parts,
    cudaStream_t stream) {
  if (!tmap_kv || !q || !table || !seq_row || !seq_prefix || !seq_kvlen || !o_part ||
      !lse_part || !out || n_seqs < 0 || group < 1 || group > 8 || (16 % group) != 0 ||
      max_splits < 1 || n_groups < 0)
    return CORTEX_EBADARG;
  if (seq_tile_start && (tiles_per_chunk < 1 || tiles_per_chunk > kFlatMaxW || total_tiles < 0))
    return CORTEX_EBADARG;
  if (n_seqs == 0) return CORTEX_OK;
  const int cascade = n_groups > 0 ? 1 : 0;
  if (cascade && (!grp_row || !grp_plen || !grp_first || !grp_count || prefix_slots < 1 ||
                  prefix_slots >= max_splits))
    return CORTEX_EBADARG;
  const float scale_log2 = softmax_scale * kLog2e;
  if (!(parts & 1)) {
    // cascade pass launched separately (e.g. on a side stream)
  } else if (cascade && tmap_q) {
    const int32_t rc = cortex_fmha_cascade_tc(
        tmap_kv, tmap_q, table, table_stride, grp_row, grp_plen, grp_first, grp_count, n_groups,
        max_group_count, prefix_slots, n_kv_heads, group, k_row0, v_row0, softmax_scale, o_part,
        lse_part, max_splits, stream);
    if (rc != CORTEX_OK) return rc;
  } else if (cascade) {
    CascadeArgs c{};
    c.q = reinterpret_cast<const __nv_bfloat16*>(q);
    c.table = table;
    c.table_stride = table_stride;
    c.grp_row = grp_row;
    c.grp_plen = grp_plen;
    c.grp_first = grp_first;
    c.grp_count = grp_count;
    c.max_psplits = prefix_slots;
    c.n_kv_heads = n_kv_heads;
    c.group = group;
    c.k_row0 = k_row0;
    c.v_row0 = v_row0;
    c.scale_log2 = scale_log2;
    c.o_part = o_part;
    c.lse_part = lse_part;
    c.max_splits = max_splits;
    const int csmem = kPrefillStages * kStageBytes + 1024 + 256;
    static bool cconf = false;
    if (!cconf) {
      if (cudaFuncSetAttribute(cascade_prefix_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               csmem) != cudaSuccess)
        return CORTEX_ECUDA;
      cconf = true;
    }
    const int spc = (16 / group) * kWarps;
    dim3 cgrid((max_group_count + spc - 1) / spc, n_kv_heads, n_groups * prefix_slots);
    if (pdl_launch(cascade_prefix_kernel, cgrid, kWarps * 32, csmem, stream, 1,
                   *reinterpret_cast<const CUtensorMap*>(tmap_kv), c) != cudaSuccess)
      return CORTEX_ECUDA;
  }
  DecodeArgs a{};
  a.q = reinterpret_cast<const __nv_bfloat16*>(q);
  a.table = table;
  a.table_stride = table_stride;
  a.seq_row = seq_row;
  a.seq_prefix = seq_prefix;
  a.seq_kvlen = seq_kvlen;
  a.n_kv_heads = n_kv_heads;
  a.group = group;
  a.k_row0 = k_row0;
  a.v_row0 = v_row0;
  a.scale_log2 = scale_log2;
  a.o_part = o_part;
  a.lse_part = lse_part;
  a.max_splits = max_splits;
  a.cascade = cascade;
  a.slot_off = cascade ? prefix_slots : 0;
  // stage buffers + their barriers + the 1 KiB alignment slack: 64.06 KiB, so a split CTA
  // fits beside a 160 KiB tcgen05 attention CTA on one SM
  const int smem = kWarps * kDecodeStages * (kStageBytes + 8) + 1024;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(paged_decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             smem) != cudaSuccess)
      return CORTEX_ECUDA;
    configured = true;
  }
  if ((parts & 2) && seq_tile_start && total_tiles > 0) {
    FlatArgs fa{};
    fa.d = a;
    fa.tile_start = seq_tile_start;
    fa.n_seqs = n_seqs;
    fa.W = tiles_per_chunk;
    fa.total = total_tiles;
    const size_t fsmem = flat_smem_bytes(group);
    static int fconf = 0;
    if (static_cast<int>(fsmem) > fconf) {
      if (cudaFuncSetAttribute(paged_decode_flat_kernel,
                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(fsmem)) != cudaSuccess)
        return CORTEX_ECUDA;
      fconf = static_cast<int>(fsmem);
    }
    dim3 grid((total_tiles + tiles_per_chunk - 1) / tiles_per_chunk, n_kv_heads);
    if (pdl_launch(paged_decode_flat_kernel, grid, kWarps * 32, fsmem, stream, 1,
                   *reinterpret_cast<const CUtensorMap*>(tmap_kv), fa) != cudaSuccess)
      return CORTEX_ECUDA;
  } else if ((parts & 2) && !seq_tile_start) {
    dim3 grid(max_splits - a.slot_off, n_kv_heads, n_seqs);
    if (pdl_launch(paged_decode_kernel, grid, kWarps * 32, smem, stream, 1,
                   *reinterpret_cast<const CUtensorMap*>(tmap_kv), a) != cudaSuccess)
      return CORTEX_ECUDA;
  }
  if (!(parts & 4)) return CORTEX_OK;
  CombineArgs cb{};
  cb.o_part = o_part;
  cb.lse_part = lse_part;
  cb.seq_prefix = seq_prefix;
  cb.seq_kvlen = seq_kvlen;
  cb.out = reinterpret_cast<__nv_bfloat16*>(out);
  cb.hq = n_kv_heads * group;
  cb.max_splits = max_splits;
  cb.cascade = cascade;
  cb.slot_off = a.slot_off;
  cb.tile_start = seq_tile_start;
  cb.W = tiles_per_chunk;
  const dim3 cgrid(n_seqs, (cb.hq + kCombineThreads / 32 - 1) / (kCombineThreads / 32));
  if (pdl_launch(decode_combine_kernel, cgrid, kCombineThreads, 0, stream, 1, cb) != cudaSuccess)
    return CORTEX_ECUDA;
  return CORTEX_OK;
}

// Tiles per chunk of the balanced decode plan for `total_tiles` flat tiles: the chunk
// count is a whole number of CTA waves (3 CTAs per SM x n_kv_heads CTAs per chunk)
// with the smallest W <= kFlatMaxW; at least 4 tiles (one per warp) per chunk.
int32_t cortex_decode_tiles_per_chunk(int32_t total_tiles, int32_t n_kv_heads) {
  if (total_tiles <= 0 || n_kv_heads < 1) return 1;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      sms = 148;
  }
  const int per_wave = max(1, 3 * sms / n_kv_heads);  // chunks per full wave of CTAs
  for (int waves = 1;; ++waves) {
    const int chunks = waves * per_wave;
    const int W = (total_tiles + chunks - 1) / chunks;
    if (W <= kFlatMaxW) return W < 4 ? min(4, kFlatMaxW) : W;
  }
}

int32_t cortex_paged_prefill_attn(const void* tmap_kv, const void* q, void* out,
                                  const int32_t* table, int32_t table_stride,
                                  const int32_t* seq_row, const int32_t* seq_prefix,
                                  const int32_t* seq_kvlen, const int32_t* seq_qstart,
                                  const int32_t* seq_qlen, int32_t n_seqs, int32_t max_qlen,
                                  int32_t n_kv_heads, int32_t group, int64_t k_row0,
                                  int64_t v_row0, float softmax_scale, cudaStream_t stream) {
  if (!tmap_kv || !q || !out || !table || !seq_row || !seq_prefix || !seq_kvlen ||
      !seq_qstart || !seq_qlen || n_seqs < 0 || group < 1 || (16 % group) != 0)
    return CORTEX_EBADARG;
  if (n_seqs == 0 || max_qlen <= 0) return CORTEX_OK;
  PrefillArgs a{};
  a.q = reinterpret_cast<const __nv_bfloat16*>(q);
  a.out = reinterpret_cast<__nv_bfloat16*>(out);
  a.table = table;
  a.table_stride = table_stride;
  a.seq_row = seq_row;
  a.seq_prefix = seq_prefix;
  a.seq_kvlen = seq_kvlen;
  a.seq_qstart = seq_qstart;
  a.seq_qlen = seq_qlen;
  a.n_kv_heads = n_kv_heads;
  a.group = group;
  a.k_row0 = k_row0;
  a.v_row0 = v_row0;
  a.scale_log2 = softmax_scale * kLog2e;
  const int smem = kPrefillStages * kStageBytes + 1024 + 256;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(paged_prefill_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             smem) != cudaSuccess)
      return CORTEX_ECUDA;
    configured = true;
  }
  const int toks_per_cta = (16 / group) * kWarps;
  dim3 grid((max_qlen + toks_per_cta - 1) / toks_per_cta, n_kv_heads, n_seqs);
  if (pdl_launch(paged_prefill_kernel, grid, kWarps * 32, smem, stream, 1,
                 *reinterpret_cast<const CUtensorMap*>(tmap_kv), a) != cudaSuccess)
    return CORTEX_ECUDA;
  return CORTEX_OK;
}

}  // extern "C"
