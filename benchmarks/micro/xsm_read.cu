// Latency of reading data another SM wrote moments ago (st.cg + fence + flag) vs data
// written by an earlier kernel. nvcc -gencode arch=compute_100a,code=sm_100a -O3 xsm_read.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

// CTA c writes slot c (32 KB per chunk x 8 chunks), publishes; CTA c reads slot (c+1)%n.
__global__ void k(float4* ws, int* flags, uint64_t* out, int fresh) {
  const int c = blockIdx.x, n = gridDim.x, tid = threadIdx.x;
  const int chunk_f4 = 2048;  // 32 KB
  float4* mine = ws + (size_t)c * 8 * chunk_f4;
  if (fresh) {
    for (int i = tid; i < 8 * chunk_f4; i += blockDim.x) __stcg(mine + i, make_float4(c, i, 1, 2));
    __threadfence();
    __syncthreads();
    if (tid == 0) atomicExch(flags + c, 1);
    if (tid == 0) while (atomicAdd(flags + (c + 1) % n, 0) == 0) {}
    __syncthreads();
  }
  const float4* other = ws + (size_t)((c + 1) % n) * 8 * chunk_f4;
  float s = 0.f;
  for (int ch = 0; ch < 8; ++ch) {
    uint64_t t0 = gt();
    float4 v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = __ldcg(other + ch * chunk_f4 + q * 128 + tid);
#pragma unroll
    for (int q = 0; q < 16; ++q) s += v[q].x + v[q].w;
    __syncthreads();
    uint64_t t1 = gt();
    if (tid == 0) out[c * 8 + ch] = t1 - t0;
  }
  if (s == -1.f) out[0] = 0;
  __syncthreads();
  if (tid == 0 && fresh) flags[c] = 0;
}

int main() {
  const int n = 148;
  float4* ws; int* flags; uint64_t* out;
  cudaMalloc(&ws, (size_t)n * 8 * 2048 * 16);
  cudaMalloc(&flags, n * 4);
  cudaMemset(flags, 0, n * 4);
  cudaMalloc(&out, n * 8 * 8);
  uint64_t h[n * 8];
  for (int fresh = 1; fresh >= 0; --fresh) {
    for (int it = 0; it < 3; ++it) k<<<n, 128>>>(ws, flags, out, fresh);
    cudaDeviceSynchronize();
    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    double avg[8] = {0};
    for (int c = 0; c < n; ++c) for (int ch = 0; ch < 8; ++ch) avg[ch] += h[c * 8 + ch] / (double)n;
    printf("fresh=%d per-chunk ns:", fresh);
    for (int ch = 0; ch < 8; ++ch) printf(" %.0f", avg[ch]);
    printf("   (%s)\n", cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
