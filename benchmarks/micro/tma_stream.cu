// HBM streaming bandwidth of bulk TMA (cp.async.bulk global->shared) versus the number
// of CTAs and the bytes each CTA keeps in flight: can a few SMs saturate HBM, or does a
// weight-streaming GEMM need every SM pulling? (decode-GEMM design question)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_stream tma_stream.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Each CTA streams its contiguous slice [cta*slice, (cta+1)*slice) through `stages` smem
// buffers of `chunk` bytes; one thread issues, the mbarrier tracks completion.
__global__ void stream(const uint8_t* src, size_t slice, int chunk, int stages, float* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[16];
  const uint8_t* base = src + blockIdx.x * slice;
  const int n = static_cast<int>(slice / chunk);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  float acc = 0.f;
  for (int i = 0; i < n + stages; ++i) {
    if (i >= stages) {  // consume chunk i - stages
      const int s = (i - stages) % stages;
      const uint32_t ph = ((i - stages) / stages) & 1;
      asm volatile(
          "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
          " @!p bra W;\n}" ::"r"(su32(&bar[s])), "r"(ph));
      acc += static_cast<float>(sm[s * chunk]);
    }
    if (i < n) {
      const int s = i % stages;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])),
                   "r"(chunk));
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
          ::"r"(su32(sm + s * chunk)), "l"(base + static_cast<size_t>(i) * chunk), "r"(chunk),
          "r"(su32(&bar[s]))
          : "memory");
    }
  }
  if (acc == 12345.f) sink[0] = acc;
}


// Plain vectorised loads (LSU path): every thread keeps 8 x 16 B in flight.
__global__ void ldg(const float4* src, size_t slice_f4, float* sink) {
  const float4* base = src + blockIdx.x * slice_f4;
  float acc = 0.f;
  for (size_t i = threadIdx.x; i + 7 * blockDim.x < slice_f4; i += 8 * blockDim.x) {
    float4 v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = __ldcs(base + i + q * blockDim.x);
#pragma unroll
    for (int q = 0; q < 8; ++q) acc += v[q].x;
  }
  if (acc == 12345.f) sink[0] = acc;
}

// TMA (thread 0, half the slice) and LDG (warps 1.., other half) at the same time.
__global__ void mixed(const uint8_t* src, size_t slice, int chunk, int stages, float* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[16];
  const uint8_t* base = src + blockIdx.x * slice;
  const size_t half = slice / 2 / chunk * chunk;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  float acc = 0.f;
  if (threadIdx.x == 0) {
    const int n = static_cast<int>(half / chunk);
    for (int i = 0; i < n + stages; ++i) {
      if (i >= stages) {
        const int s = (i - stages) % stages;
        const uint32_t ph = ((i - stages) / stages) & 1;
        asm volatile(
            "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
            " @!p bra W;\n}" ::"r"(su32(&bar[s])), "r"(ph));
        acc += static_cast<float>(sm[s * chunk]);
      }
      if (i < n) {
        const int s = i % stages;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])),
                     "r"(chunk));
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(su32(sm + s * chunk)), "l"(base + static_cast<size_t>(i) * chunk), "r"(chunk),
            "r"(su32(&bar[s]))
            : "memory");
      }
    }
  } else if (threadIdx.x >= 32) {
    const float4* b4 = reinterpret_cast<const float4*>(base + half);
    const size_t n4 = (slice - half) / 16;
    const int t = threadIdx.x - 32, nt = blockDim.x - 32;
    for (size_t i = t; i + 7 * nt < n4; i += 8 * nt) {
      float4 v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = __ldcs(b4 + i + q * nt);
#pragma unroll
      for (int q = 0; q < 8; ++q) acc += v[q].x;
    }
  }
  if (acc == 12345.f) sink[0] = acc;
}


// `nstreams` warps each run an independent bulk-TMA stream (own barriers and buffers) over
// their own part of the CTA's slice: does the per-SM rate grow with issuing threads?
__global__ void multi(const uint8_t* src, size_t slice, int chunk, int stages, int nstreams,
                      float* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[64];
  const int w = threadIdx.x / 32;
  if (w >= nstreams || (threadIdx.x & 31) != 0) return;
  const size_t part = slice / nstreams / chunk * chunk;
  const uint8_t* base = src + blockIdx.x * slice + w * part;
  uint64_t* mb = bar + w * stages;
  uint8_t* buf = sm + w * stages * chunk;
  for (int s = 0; s < stages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mb[s])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  const int n = static_cast<int>(part / chunk);
  float acc = 0.f;
  for (int i = 0; i < n + stages; ++i) {
    if (i >= stages) {
      const int s = (i - stages) % stages;
      const uint32_t ph = ((i - stages) / stages) & 1;
      asm volatile(
          "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
          " @!p bra W;\n}" ::"r"(su32(&mb[s])), "r"(ph));
      acc += static_cast<float>(buf[s * chunk]);
    }
    if (i < n) {
      const int s = i % stages;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&mb[s])),
                   "r"(chunk));
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
          ::"r"(su32(buf + s * chunk)), "l"(base + static_cast<size_t>(i) * chunk), "r"(chunk),
          "r"(su32(&mb[s]))
          : "memory");
    }
  }
  if (acc == 12345.f) sink[0] = acc;
}

int main() {
  const size_t total = size_t(1) << 30;  // 1 GiB read per launch (>> L2)
  uint8_t* src;
  float* sink;
  cudaMalloc(&src, total);
  cudaMemset(src, 1, total);
  cudaMalloc(&sink, 4);
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(mixed, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int grids[] = {16, 32, 48, 64, 74, 96, 128, 148};
  const int inflight_kb[] = {32, 64, 96, 128, 192};
  printf("{\"rows\": [\n");
  bool first = true;
  for (int g : grids) {
    for (int kb : inflight_kb) {
      const int chunk = 16384;
      const int stages = kb * 1024 / chunk;
      const size_t slice = (total / g) / chunk * chunk;
      for (int w = 0; w < 2; ++w) stream<<<g, 32, stages * chunk>>>(src, slice, chunk, stages, sink);
      cudaEventRecord(e0);
      const int it = 5;
      for (int r = 0; r < it; ++r)
        stream<<<g, 32, stages * chunk>>>(src, slice, chunk, stages, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double gbs = double(slice) * g * it / (ms * 1e-3) / 1e9;
      printf("%s{\"ctas\": %d, \"inflight_kb\": %d, \"GBps\": %.0f, \"per_sm_GBps\": %.1f}",
             first ? "" : ",\n", g, kb, gbs, gbs / g);
      first = false;
    }
  }
  printf("\n], \"ldg\": [\n");
  first = true;
  for (int g : grids) {
    const size_t slice_f4 = (total / g) / 16;
    for (int w = 0; w < 2; ++w) ldg<<<g, 512>>>(reinterpret_cast<const float4*>(src), slice_f4, sink);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) ldg<<<g, 512>>>(reinterpret_cast<const float4*>(src), slice_f4, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double gbs = double(slice_f4) * 16 * g * 5 / (ms * 1e-3) / 1e9;
    printf("%s{\"ctas\": %d, \"GBps\": %.0f, \"per_sm_GBps\": %.1f}", first ? "" : ",\n", g, gbs, gbs / g);
    first = false;
  }
  printf("\n], \"mixed\": [\n");
  first = true;
  for (int g : grids) {
    const int chunk = 16384, stages = 6;
    const size_t slice = (total / g) / chunk * chunk;
    for (int w = 0; w < 2; ++w) mixed<<<g, 512, stages * chunk>>>(src, slice, chunk, stages, sink);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) mixed<<<g, 512, stages * chunk>>>(src, slice, chunk, stages, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double gbs = double(slice) * g * 5 / (ms * 1e-3) / 1e9;
    printf("%s{\"ctas\": %d, \"GBps\": %.0f, \"per_sm_GBps\": %.1f}", first ? "" : ",\n", g, gbs, gbs / g);
    first = false;
  }
  printf("\n], \"multi\": [\n");
  first = true;
  cudaFuncSetAttribute(multi, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int g : {16, 64, 148}) {
    for (int ns : {1, 2, 4, 8}) {
      for (int chunk : {4096, 16384}) {
        const int stages = (192 * 1024) / (ns * chunk) > 12 ? 12 : (192 * 1024) / (ns * chunk);
        const size_t slice = (total / g) / (ns * chunk) * (ns * chunk);
        for (int w = 0; w < 2; ++w) multi<<<g, 256, ns * stages * chunk>>>(src, slice, chunk, stages, ns, sink);
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) multi<<<g, 256, ns * stages * chunk>>>(src, slice, chunk, stages, ns, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double gbs = double(slice) * g * 5 / (ms * 1e-3) / 1e9;
        printf("%s{\"ctas\": %d, \"streams\": %d, \"chunk\": %d, \"stages\": %d, \"GBps\": %.0f, \"per_sm_GBps\": %.1f}",
               first ? "" : ",\n", g, ns, chunk, stages, gbs, gbs / g);
        first = false;
      }
    }
  }
  printf("\n], \"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
