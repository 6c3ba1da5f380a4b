// Weight-streaming bandwidth of 2-D tensor TMA boxes (128 rows x 64 bf16 = 16 KiB, 128-byte
// swizzle) over a row-major [N, K] matrix versus the same bytes stored tile-contiguous
// ([N/128][K/64][128][64], a 3-D map whose box is one contiguous 16 KiB tile). Each CTA
// streams its own row block across all of K with `issuers` warps issuing in parallel.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_tile tma_tile.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// grid = (row blocks, k splits): CTA streams rows [128 by, +128) x K-blocks [kb0, kb1)
__global__ void stream2d(const __grid_constant__ CUtensorMap tm, int tiled, int kbs_per, int stages,
                         int issuers, int kb_total, float* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[64];
  const int w = threadIdx.x / 32;
  if (w >= issuers || (threadIdx.x & 31) != 0) return;
  const int rb = blockIdx.x;
  const int kb0 = blockIdx.y * kbs_per;
  uint64_t* mb = bar + w * stages;
  uint8_t* buf = sm + w * stages * 16384;
  for (int s = 0; s < stages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mb[s])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  const int n = kbs_per / issuers;
  float acc = 0.f;
  for (int i = 0; i < n + stages; ++i) {
    if (i >= stages) {
      const int s = (i - stages) % stages;
      const uint32_t ph = ((i - stages) / stages) & 1;
      asm volatile(
          "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
          " @!p bra W;\n}" ::"r"(su32(&mb[s])), "r"(ph));
      acc += static_cast<float>(buf[s * 16384]);
    }
    if (i < n) {
      const int s = i % stages;
      const int kb = kb0 + i * issuers + w;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&mb[s])),
                   "r"(16384));
      if (tiled)
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(su32(buf + s * 16384)),
            "l"(reinterpret_cast<uint64_t>(&tm)), "r"(su32(&mb[s])), "r"(0), "r"(0),
            "r"(rb * kb_total + kb)
            : "memory");
      else
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4}], [%2];" ::"r"(su32(buf + s * 16384)),
            "l"(reinterpret_cast<uint64_t>(&tm)), "r"(su32(&mb[s])), "r"(kb * 64), "r"(rb * 128)
            : "memory");
    }
  }
  if (acc == 12345.f) sink[0] = acc;
}

int main() {
  const int N = 28672, K = 4096;
  const size_t bytes = size_t(N) * K * 2;
  uint8_t* w;
  float* sink;
  cudaMalloc(&w, bytes * 4);  // 4 copies rotate (> L2)
  cudaMemset(w, 1, bytes * 4);
  cudaMalloc(&sink, 4);
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fnp);
  CUtensorMap maps2d[4], maps3d[4];
  for (int c = 0; c < 4; ++c) {
    cuuint64_t d2[2] = {cuuint64_t(K), cuuint64_t(N)};
    cuuint64_t s2[1] = {cuuint64_t(K) * 2};
    cuuint32_t b2[2] = {64, 128}, e2[2] = {1, 1};
    enc(&maps2d[c], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w + c * bytes, d2, s2, b2, e2,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    // tiled: [N/128 * K/64 tiles][128][64] -> dims (64, 128, tiles)
    cuuint64_t d3[3] = {64, 128, cuuint64_t(N / 128) * (K / 64)};
    cuuint64_t s3[2] = {128, 128 * 128};
    cuuint32_t b3[3] = {64, 128, 1}, e3[3] = {1, 1, 1};
    enc(&maps3d[c], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, w + c * bytes, d3, s3, b3, e3,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  cudaFuncSetAttribute(stream2d, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("{\"rows\": [\n");
  bool first = true;
  for (int tiled = 0; tiled < 2; ++tiled) {
    for (int ksplit : {1, 2}) {
      for (int issuers : {1, 2, 4}) {
        const int stages = 12 / issuers;
        const int rblocks = N / 128;  // 224 row blocks
        const int kbs = (K / 64) / ksplit;
        dim3 grid(rblocks, ksplit);
        for (int r = 0; r < 2; ++r)
          stream2d<<<grid, 128, issuers * stages * 16384 + 1024>>>(tiled ? maps3d[r % 4] : maps2d[r % 4],
                                                                  tiled, kbs, stages, issuers,
                                                                  K / 64, sink);
        cudaEventRecord(e0);
        const int it = 8;
        for (int r = 0; r < it; ++r)
          stream2d<<<grid, 128, issuers * stages * 16384 + 1024>>>(tiled ? maps3d[r % 4] : maps2d[r % 4],
                                                                  tiled, kbs, stages, issuers,
                                                                  K / 64, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double gbs = double(bytes) * it / (ms * 1e-3) / 1e9;
        printf("%s{\"layout\": \"%s\", \"ksplit\": %d, \"ctas\": %d, \"issuers\": %d, \"stages\": %d, "
               "\"us\": %.1f, \"GBps\": %.0f}",
               first ? "" : ",\n", tiled ? "tiled" : "rowmajor", ksplit, rblocks * ksplit, issuers,
               stages, ms * 1e3 / it, gbs);
        first = false;
      }
    }
  }
  printf("\n], \"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
