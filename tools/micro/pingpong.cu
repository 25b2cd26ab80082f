// Flag ping-pong latency between two CTAs (different SMs): per-hop cost of
// the release/acquire patterns used by the recurrent kernels.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory"); }
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory"); }

template <int MODE>
__global__ void pingpong(uint32_t* flags, int iters, uint4* scratch, int nstores, unsigned long long* out) {
  const int me = blockIdx.x;  // 0 or 1
  uint32_t* mine = flags + me * 64;
  uint32_t* other = flags + (1 - me) * 64;
  long long t0 = clock64();
  for (int i = 1; i <= iters; ++i) {
    if (me == 1 || i > 1) {
      // wait for the other side's i-th (or (i-1)-th) token
      const uint32_t want = me == 1 ? i : i - 1;
      if (threadIdx.x == 0) {
        if (MODE == 2) { while (ld_relaxed(other) < want) {} (void)ld_acquire(other); }
        else { while (ld_acquire(other) < want) {} }
      }
      __syncthreads();
    }
    // optional outstanding stores before publishing (all threads)
    for (int k = 0; k < nstores; ++k) scratch[(size_t)(me * 1024 + k) * blockDim.x + threadIdx.x] = make_uint4(i, k, 0, 0);
    __syncthreads();
    if (threadIdx.x == 0) {
      if (MODE == 1) { __threadfence(); st_relaxed(mine, i); }
      else st_release(mine, i);
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[me] = (unsigned long long)(t1 - t0);
}

int main() {
  uint32_t* flags; uint4* scratch; unsigned long long* out;
  cudaMalloc(&flags, 4096); cudaMalloc(&scratch, 64 << 20); cudaMalloc(&out, 64);
  int iters = 2000;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int mode = 0; mode < 3; ++mode)
    for (int ns : {0, 4, 16}) {
      cudaMemset(flags, 0, 4096);
      cudaEventRecord(e0);
      if (mode == 0) pingpong<0><<<2, 256>>>(flags, iters, scratch, ns, out);
      if (mode == 1) pingpong<1><<<2, 256>>>(flags, iters, scratch, ns, out);
      if (mode == 2) pingpong<2><<<2, 256>>>(flags, iters, scratch, ns, out);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("mode %d (%s) stores/thread %2d: %.3f us per hop\n", mode,
             mode == 0 ? "st.release/ld.acquire poll" : mode == 1 ? "threadfence+relaxed/ld.acquire" : "st.release/relaxed poll+acquire",
             ns, ms * 1e3 / (2 * iters));
    }
  return 0;
}
