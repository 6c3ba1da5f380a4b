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
// fixed 16-tile chunks (chunking depends only on the sequence length, so results
// are batch-composition invariant) and merged by a log-sum-exp combine.
#include "common.cuh"

namespace {

constexpr int kHeadDim = 128;
constexpr int kTile = 16;                  // tokens per KV block
constexpr int kTileBytes = kTile * kHeadDim * 2;  // 4 KiB (K or V)
constexpr int kStageBytes = 2 * kTileBytes;       // K + V
constexpr int kTilesPerSplit = 16;
constexpr int kWarps = 4;
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
#pragma unroll
  for (int row = 0; row < 2; ++row) {
    mx[row] = fmaxf(mx[row], __shfl_xor_sync(0xffffffffu, mx[row], 1));
    mx[row] = fmaxf(mx[row], __shfl_xor_sync(0xffffffffu, mx[row], 2));
  }
  float alpha[2], m_use[2];
#pragma unroll
  for (int row = 0; row < 2; ++row) {
    const float m_new = fmaxf(st.m[row], mx[row]);
    m_use[row] = m_new == -INFINITY ? 0.f : m_new;
    alpha[row] = exp2f(st.m[row] - m_use[row]);
    st.m[row] = m_new;
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
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    st.o[j][0] *= alpha[0];
    st.o[j][1] *= alpha[0];
    st.o[j][2] *= alpha[1];
    st.o[j][3] *= alpha[1];
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

constexpr int kDecodeStages = 2;
constexpr int kPrefillStages = 3;

__global__ void __launch_bounds__(kWarps * 32)
    paged_decode_kernel(const __grid_constant__ CUtensorMap tmap_kv, const DecodeArgs a) {
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
  if (t_begin >= ntiles) return;
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
  __syncwarp();

  const int* table_row = a.table + static_cast<int64_t>(row) * a.table_stride;
  // tiles owned by this warp: t_begin + warp + 4 i
  const int n_mine = (t_end - t_begin - warp + kWarps - 1) / kWarps;
  if (lane == 0) {
    for (int i = 0; i < min(n_mine, kDecodeStages); ++i) {
      const TileRef t = tile_ref(table_row, prefix, kvlen, t_begin + warp + kWarps * i);
      load_tile(my_stages + i * kStageBytes, &tmap_kv, &bars[i], a.k_row0, a.v_row0, t.block, kvh,
                a.n_kv_heads);
    }
  }

  uint32_t qa[8][4];
  load_q_frags(qa, a.q, b, hq * kHeadDim, kvh * a.group, a.group, a.group);
  WarpState st;
  state_init(st);
  const int qpos[2] = {kvlen - 1, kvlen - 1};

  for (int i = 0; i < n_mine; ++i) {
    const int s = i % kDecodeStages;
    const TileRef t = tile_ref(table_row, prefix, kvlen, t_begin + warp + kWarps * i);
    mbar_wait(&bars[s], (i / kDecodeStages) & 1);
    attend_tile(st, qa, smem_u32(my_stages + s * kStageBytes), t, qpos, a.scale_log2);
    __syncwarp();
    const int nxt = i + kDecodeStages;
    if (nxt < n_mine && lane == 0) {
      fence_proxy_async();
      const TileRef tn = tile_ref(table_row, prefix, kvlen, t_begin + warp + kWarps * nxt);
      load_tile(my_stages + s * kStageBytes, &tmap_kv, &bars[s], a.k_row0, a.v_row0, tn.block,
                kvh, a.n_kv_heads);
    }
    __syncwarp();
  }
  quad_reduce_l(st);

  // combine the 4 warps (rows < group only) through shared memory
  __syncthreads();
  float* cm = reinterpret_cast<float*>(smem);            // [4][8]
  float* cl = cm + kWarps * 8;                           // [4][8]
  float* co = cl + kWarps * 8;                           // [4][8][128]
  const int g = lane >> 2;
  const int tq = lane & 3;
  if (g < a.group) {
    if (tq == 0) {
      cm[warp * 8 + g] = st.m[0];
      cl[warp * 8 + g] = st.l[0];
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      co[(warp * 8 + g) * kHeadDim + 8 * j + 2 * tq] = st.o[j][0];
      co[(warp * 8 + g) * kHeadDim + 8 * j + 2 * tq + 1] = st.o[j][1];
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < a.group * kHeadDim; idx += blockDim.x) {
    const int r = idx / kHeadDim;
    const int d = idx % kHeadDim;
    float M = -INFINITY;
    for (int w = 0; w < kWarps; ++w) M = fmaxf(M, cm[w * 8 + r]);
    float L = 0.f, O = 0.f;
    for (int w = 0; w < kWarps; ++w) {
      const float f = cm[w * 8 + r] == -INFINITY ? 0.f : exp2f(cm[w * 8 + r] - M);
      L += cl[w * 8 + r] * f;
      O += co[(w * 8 + r) * kHeadDim + d] * f;
    }
    const int h = kvh * a.group + r;
    const int64_t pidx =
        (static_cast<int64_t>(b) * a.max_splits + (a.cascade ? a.slot_off : 0) + split) * hq + h;
    a.o_part[pidx * kHeadDim + d] = O / L;
    if (d == 0) a.lse_part[pidx] = M + log2f(L);
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
};

// LSE merge of a call's partials: one CTA per call, warp <-> head, lane <-> 4 dims;
// slot weights computed once per head by the lanes, partial rows loaded 4 at a time.
constexpr int kCombineThreads = 256;

__global__ void __launch_bounds__(kCombineThreads) decode_combine_kernel(const CombineArgs a) {
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
  const int nsl = np + ns;
  const int64_t base = static_cast<int64_t>(b) * a.max_splits;
  auto slot = [&](int i) { return i < np ? i : off + (i - np); };
  for (int h = warp; h < a.hq; h += kCombineThreads / 32) {
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

int32_t cortex_paged_decode_attn(const void* tmap_kv, const void* q, const int32_t* table,
                                 int32_t table_stride, const int32_t* seq_row,
                                 const int32_t* seq_prefix, const int32_t* seq_kvlen,
                                 int32_t n_seqs, int32_t n_kv_heads, int32_t group,
                                 int64_t k_row0, int64_t v_row0, float softmax_scale,
                                 float* o_part, float* lse_part, int32_t max_splits, void* out,
                                 const int32_t* grp_row, const int32_t* grp_plen,
                                 const int32_t* grp_first, const int32_t* grp_count,
                                 int32_t n_groups, int32_t max_group_count,
                                 int32_t prefix_slots, const void* tmap_q, cudaStream_t stream) {
  return cortex_paged_decode_attn_parts(tmap_kv, q, table, table_stride, seq_row, seq_prefix,
                                        seq_kvlen, n_seqs, n_kv_heads, group, k_row0, v_row0,
                                        softmax_scale, o_part, lse_part, max_splits, out, grp_row,
                                        grp_plen, grp_first, grp_count, n_groups, max_group_count,
                                        prefix_slots, tmap_q, 7, stream);
}

int32_t cortex_paged_decode_attn_parts(const void* tmap_kv, const void* q, const int32_t* table,
                                       int32_t table_stride, const int32_t* seq_row,
                                       const int32_t* seq_prefix, const int32_t* seq_kvlen,
                                       int32_t n_seqs, int32_t n_kv_heads, int32_t group,
                                       int64_t k_row0, int64_t v_row0, float softmax_scale,
                                       float* o_part, float* lse_part, int32_t max_splits,
                                       void* out, const int32_t* grp_row, const int32_t* grp_plen,
                                       const int32_t* grp_first, const int32_t* grp_count,
                                       int32_t n_groups, int32_t max_group_count,
                                       int32_t prefix_slots, const void* tmap_q, int32_t parts,
                                       cudaStream_t stream) {
  if (!tmap_kv || !q || !table || !seq_row || !seq_prefix || !seq_kvlen || !o_part ||
      !lse_part || !out || n_seqs < 0 || group < 1 || group > 8 || (16 % group) != 0 ||
      max_splits < 1 || n_groups < 0)
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
    cascade_prefix_kernel<<<cgrid, kWarps * 32, csmem, stream>>>(
        *reinterpret_cast<const CUtensorMap*>(tmap_kv), c);
    CORTEX_CHECK_LAUNCH();
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
  const int smem = kWarps * kDecodeStages * kStageBytes + 1024 + 256;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(paged_decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             smem) != cudaSuccess)
      return CORTEX_ECUDA;
    configured = true;
  }
  if (parts & 2) {
    dim3 grid(max_splits - a.slot_off, n_kv_heads, n_seqs);
    paged_decode_kernel<<<grid, kWarps * 32, smem, stream>>>(
        *reinterpret_cast<const CUtensorMap*>(tmap_kv), a);
    CORTEX_CHECK_LAUNCH();
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
  decode_combine_kernel<<<n_seqs, kCombineThreads, 0, stream>>>(cb);
  CORTEX_CHECK_LAUNCH();
  return CORTEX_OK;
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
  paged_prefill_kernel<<<grid, kWarps * 32, smem, stream>>>(
      *reinterpret_cast<const CUtensorMap*>(tmap_kv), a);
  CORTEX_CHECK_LAUNCH();
  return CORTEX_OK;
}

}  // extern "C"
