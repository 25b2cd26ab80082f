// MUFU.EX2 throughput per SM (ex2.approx.ftz.f32) and the FFMA rate for
// comparison: every thread runs 8 independent dependency chains.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 mufu_rate.cu -o mufu_rate
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int MODE>
__global__ void rate(float* out, int iters, unsigned long long* clk) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int k = 0; k < iters; ++k) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = MODE == 0 ? ex2(a[i]) - 1.0f : fmaf(a[i], 0.999f, -0.001f);
  }
  __syncthreads();
  if (threadIdx.x == 0) clk[blockIdx.x] = clock64() - t0;
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.f) out[0] = s;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  unsigned long long* clk;
  cudaMalloc(&out, 4);
  cudaMalloc(&clk, 8 * 1024);
  const int iters = 4096;
  for (int mode = 0; mode < 2; ++mode)
    for (int threads : {256, 512, 1024}) {
      if (mode == 0)
        rate<0><<<sms, threads>>>(out, iters, clk);
      else
        rate<1><<<sms, threads>>>(out, iters, clk);
      cudaDeviceSynchronize();
      unsigned long long c;
      cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
      const double ops = (double)threads * iters * 8;  // per SM (one block per SM)
      printf("%s threads/SM %4d: %.2f ops/clk/SM (%s)\n", mode == 0 ? "MUFU.EX2 (+FADD)" : "FFMA", threads,
             ops / (double)c, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
