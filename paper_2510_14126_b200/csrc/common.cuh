// Shared device helpers for the Cortex stage-engine kernels (sm_100a only).
//
// mbarrier / TMA / tcgen05 wrappers are written as inline PTX: this file is the
// single place that knows the Blackwell encodings (UMMA smem descriptor, the
// kind::f16 instruction descriptor, TMEM addressing).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#ifndef __CUDACC__
#error "common.cuh is CUDA-only"
#endif

#define CORTEX_DEVICE __device__ __forceinline__

// Activation rows per TMA box of the GEMMs' token operand (the host builds the
// activation tensor maps with cortex_act_box_rows() rows per box).
#ifndef CORTEX_XBOX
#define CORTEX_XBOX 16
#endif

#define CORTEX_BUILDING 1
#include <cstdio>

#include "cortex_b200.h"
#include "cortex_dev.h"

#define CORTEX_CHECK_LAUNCH()                      \
  do {                                             \
    cudaError_t _e = cudaGetLastError();           \
    if (_e != cudaSuccess) return CORTEX_ECUDA;    \
  } while (0)

// --------------------------------------------------------------------------
// Programmatic dependent launch (PDL). The decoder step is a chain of ~10 kernels per
// layer on one stream; with PDL a kernel is launched while its predecessor still runs,
// does its prologue (barrier init, TMEM allocation, descriptor prefetch), and blocks in
// pdl_wait() until the predecessor has completed and its memory is visible. Every kernel
// launched through pdl_launch() must call pdl_wait() before it touches memory an earlier
// kernel of the stream writes. pdl_trigger() lets the next kernel launch once every CTA
// of this grid has triggered (or exited). The PDL knob (cortex_dev.h, tests / A-B only)
// turns the attribute off.

CORTEX_DEVICE void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
CORTEX_DEVICE void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" :::); }

// L2 prefetch of one 2-D tensor-map box (no shared memory, no barrier).
CORTEX_DEVICE void tma_prefetch_l2_2d(const void* desc, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];\n" ::"l"(
                   reinterpret_cast<uint64_t>(desc)),
               "r"(c0), "r"(c1)
               : "memory");
}

template <typename... KArgs, typename... Args>
inline cudaError_t pdl_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t stream, int cluster_x, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int n = 0;
  attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[n].val.programmaticStreamSerializationAllowed = g_cortex_knob[CORTEX_KNOB_PDL] ? 1 : 0;
  ++n;
  if (cluster_x > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster_x;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// --------------------------------------------------------------------------
// generic

// ---- greedy-token partials (the lm_head GEMM's argmax epilogue, out mode 3) ----
// (max, first index of the max) of four consecutive columns col .. col + 3; NaN never
// wins a comparison, so a chunk without a finite value keeps index INT_MAX.
CORTEX_DEVICE void best_of4(const float4 v, int col, float& best, int& bi) {
  best = -INFINITY;
  bi = 0x7fffffff;
  if (v.x > best) { best = v.x; bi = col; }
  if (v.y > best) { best = v.y; bi = col + 1; }
  if (v.z > best) { best = v.z; bi = col + 2; }
  if (v.w > best) { best = v.w; bi = col + 3; }
}

// Warp-wide (max, first index) reduction; every lane ends with the result.
CORTEX_DEVICE void warp_argmax(float& best, int& bi) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) {
      best = ov;
      bi = oi;
    }
  }
}

// One warp covers a 128-column output row (lane -> columns col .. col + 3): write its
// (max, first index) as the row's partial for column chunk col0 / 128.
CORTEX_DEVICE void store_argmax_partial(float2* part, int ld, int row, int col0, const float4 v,
                                        int col) {
  float best;
  int bi;
  best_of4(v, col, best, bi);
  warp_argmax(best, bi);
  if ((threadIdx.x & 31) == 0)
    part[static_cast<size_t>(row) * ld + col0 / 128] = make_float2(best, __int_as_float(bi));
}

CORTEX_DEVICE uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

CORTEX_DEVICE int lane_id() { return threadIdx.x & 31; }
CORTEX_DEVICE int warp_id() { return threadIdx.x >> 5; }

CORTEX_DEVICE bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(pred));
  return pred != 0;
}

// Shared-prefix (cascade) decode attention splits a prefix of npb blocks into `slots`
// partial slots of this many blocks each (a multiple of the 8-block key tile).
__host__ __device__ __forceinline__ int prefix_split_blocks(int npb, int slots) {
  const int per = (npb + slots - 1) / slots;
  return (per + 7) / 8 * 8;
}

// --------------------------------------------------------------------------
// mbarrier

CORTEX_DEVICE void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

CORTEX_DEVICE void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

CORTEX_DEVICE void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

CORTEX_DEVICE void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

// Non-blocking probe of a phase (mbarrier.test_wait): true once it has completed.
CORTEX_DEVICE bool mbar_test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(done)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return done != 0;
}

CORTEX_DEVICE bool mbar_try_wait(uint32_t addr, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}\n"
      : "=r"(done)
      : "r"(addr), "r"(parity)
      : "memory");
  return done != 0;
}

// mbarrier wait; a phase that never completes (~9 s of SM clock) traps with a diagnostic
// (grid, block, thread, barrier, parity) instead of hanging the GPU.
CORTEX_DEVICE void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  if (mbar_try_wait(addr, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try_wait(addr, parity)) {
    if (clock64() - t0 > (16ll << 30)) {
      printf("cortex mbar hang: grid (%d,%d,%d) block (%d,%d,%d) thread %d smem+%u parity %u\n",
             gridDim.x, gridDim.y, gridDim.z, blockIdx.x, blockIdx.y, blockIdx.z, threadIdx.x,
             addr & 0x3ffff, parity);
      __trap();
    }
  }
}

// Cross-CTA flags in global memory (split-K publication): release store / acquire spin.
CORTEX_DEVICE void st_release_gpu_u32(int* p, uint32_t v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

// Spin until *p == v (acquire, gpu scope); a flag that never arrives (~9 s of SM clock)
// traps with a diagnostic instead of hanging the GPU.
CORTEX_DEVICE void wait_flag_gpu(const int* p, uint32_t v) {
  const long long t0 = clock64();
  while (true) {
    uint32_t x;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(x) : "l"(p) : "memory");
    if (x == v) return;
    __nanosleep(32);
    if (clock64() - t0 > (16ll << 30)) {
      printf("cortex flag hang: grid %d block %d thread %d want %u have %u\n", gridDim.x,
             blockIdx.x, threadIdx.x, v, x);
      __trap();
    }
  }
}

// --------------------------------------------------------------------------
// TMA (cp.async.bulk.tensor) and 1D bulk copies

CORTEX_DEVICE void tma_prefetch_desc(const void* desc) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(desc)) : "memory");
}

CORTEX_DEVICE void tma_load_2d(void* smem_dst, const void* desc, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];\n" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

CORTEX_DEVICE void tma_load_2d_hint(void* smem_dst, const void* desc, uint64_t* bar, int c0, int c1,
                                    uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;\n" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}

CORTEX_DEVICE uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}

CORTEX_DEVICE uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}

// --------------------------------------------------------------------------
// tcgen05: TMEM allocation, MMA issue, commit, TMEM loads

CORTEX_DEVICE void tmem_alloc(uint32_t* holder_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                   smem_u32(holder_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}

CORTEX_DEVICE void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "r"(ncols)
               : "memory");
}

CORTEX_DEVICE void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
CORTEX_DEVICE void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}

// UMMA shared-memory descriptor for a K-major operand tile stored with the
// 128-byte swizzle (rows of 64 bf16, 8-row / 1024-byte swizzle atoms), exactly
// the layout TMA writes with CU_TENSOR_MAP_SWIZZLE_128B.
CORTEX_DEVICE uint64_t umma_desc_sw128(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr & 0x3FFFFu) >> 4);  // start address  [0,14)
  d |= static_cast<uint64_t>(1) << 16;                        // LBO (unused for SW128 K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;                // SBO = 8 rows * 128 B
  d |= static_cast<uint64_t>(1) << 46;                        // descriptor version (sm100)
  d |= static_cast<uint64_t>(2) << 61;                        // SWIZZLE_128B
  return d;
}

// kind::f16 instruction descriptor: bf16 x bf16 -> f32, both operands K-major.
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int M, int N) {
  return (1u << 4)                              // D format f32
         | (1u << 7)                            // A format bf16
         | (1u << 10)                           // B format bf16
         | (static_cast<uint32_t>(N >> 3) << 17)  // N / 8
         | (static_cast<uint32_t>(M >> 4) << 24);  // M / 16
}

CORTEX_DEVICE void umma_bf16_ss(uint32_t tmem_d, uint64_t desc_a, uint64_t desc_b, uint32_t idesc,
                                uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(desc_a), "l"(desc_b), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Arrive on an mbarrier once every previously issued tcgen05.mma of this thread completes.
CORTEX_DEVICE void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
          smem_u32(bar))
      : "memory");
}

// 32 lanes x 32 bit, 16 consecutive columns per thread (thread i <-> TMEM lane base+i).
CORTEX_DEVICE void tmem_ld_32x32b_x16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32"
      " {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

CORTEX_DEVICE void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

// --------------------------------------------------------------------------
// legacy warp MMA (attention inner products) and ldmatrix

CORTEX_DEVICE void mma_bf16_16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32"
      " {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, {%0, %1, %2, %3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

CORTEX_DEVICE void ldmatrix_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                               uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

CORTEX_DEVICE void ldmatrix_x4_trans(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                     uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

CORTEX_DEVICE uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

CORTEX_DEVICE float round_bf16(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

// ---- RoPE + paged KV append in the QKV GEMM's epilogue (out mode 4) ----
// The QKV projection's 128-column chunks are whole heads ([q heads | k heads | v heads]
// x 128). For one token row m and head h, lane l holds the fp32 accumulators of dims
// 4l .. 4l + 3; the epilogue rounds them to bf16 (the unfused path's qkv activation),
// rotates q / k heads (rotate-half: dim i pairs with i + 64, i.e. lane l with l ^ 16),
// rounds again and stores q into q_out [T, hq, 128] and k / v straight into the token's
// paged slot of the layer's K / V plane. The per-token operands come from
// cortex_rope_token_prep (once per step, shared by every layer): tok_dst[m] = the
// token's 128-wide row within a plane for kv head 0, (block * hkv) * 16 + offset, and
// tok_cs[m] = cos | sin (64 + 64 fp32) at its position. They are independent loads, so
// an epilogue issues a chunk's worth of them together with its other global operands.
struct RopeEpi {
  __nv_bfloat16* q_out;
  __nv_bfloat16* cache;
  int64_t k_row0, v_row0;
  const int* tok_dst;
  const float* tok_cs;
  int hq, hkv;
};

struct RopeRow {
  int dst;
  float4 c, s;
};

CORTEX_DEVICE RopeRow rope_fetch(const RopeEpi& e, int m, int h) {
  RopeRow r;
  const int i0 = 4 * ((threadIdx.x & 31) & 15);
  r.dst = 0;
  r.c = r.s = make_float4(1.f, 1.f, 1.f, 1.f);
  if (h < e.hq + e.hkv) {
    r.c = __ldg(reinterpret_cast<const float4*>(e.tok_cs + static_cast<int64_t>(m) * 128 + i0));
    r.s = __ldg(reinterpret_cast<const float4*>(e.tok_cs + static_cast<int64_t>(m) * 128 + 64 + i0));
  }
  if (h >= e.hq) r.dst = __ldg(e.tok_dst + m);
  return r;
}

CORTEX_DEVICE void rope_store_row(const RopeEpi& e, const RopeRow& rr, int m, int h, float4 v) {
  const int lane = threadIdx.x & 31;
  float x[4] = {round_bf16(v.x), round_bf16(v.y), round_bf16(v.z), round_bf16(v.w)};
  float y[4];
  if (h < e.hq + e.hkv) {  // (warp-uniform)
    const float cc[4] = {rr.c.x, rr.c.y, rr.c.z, rr.c.w}, ss[4] = {rr.s.x, rr.s.y, rr.s.z, rr.s.w};
    const bool upper = lane >= 16;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float p = __shfl_xor_sync(0xffffffffu, x[j], 16);
      y[j] = upper ? x[j] * cc[j] + p * ss[j] : x[j] * cc[j] - p * ss[j];
    }
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) y[j] = x[j];
  }
  __nv_bfloat16* dst;
  if (h < e.hq) {
    dst = e.q_out + (static_cast<int64_t>(m) * e.hq + h) * 128;
  } else {
    const bool is_k = h < e.hq + e.hkv;
    const int kh = is_k ? h - e.hq : h - e.hq - e.hkv;
    dst = e.cache + ((is_k ? e.k_row0 : e.v_row0) + rr.dst + kh * 16) * 128;
  }
  uint2 packed;
  packed.x = pack_bf16(y[0], y[1]);
  packed.y = pack_bf16(y[2], y[3]);
  *reinterpret_cast<uint2*>(dst + 4 * lane) = packed;
}


// (a, b) -> bf16x2 hi = round(a, b) and lo = round((a, b) - hi)
CORTEX_DEVICE void split_bf16(float a, float b, uint32_t& hi, uint32_t& lo) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  const float2 hf = __bfloat1622float2(h);
  hi = *reinterpret_cast<uint32_t*>(&h);
  lo = pack_bf16(a - hf.x, b - hf.y);
}

CORTEX_DEVICE float bf16_lo(uint32_t v) { return __uint_as_float(v << 16); }
CORTEX_DEVICE float bf16_hi(uint32_t v) { return __uint_as_float(v & 0xFFFF0000u); }

// Byte offset of (row, 16-byte chunk) inside a tile written by TMA with SWIZZLE_128B
// (rows of 128 bytes; chunk index XOR row%8).
CORTEX_DEVICE uint32_t sw128_offset(uint32_t row, uint32_t chunk) {
  return row * 128u + ((chunk ^ (row & 7u)) << 4);
}
