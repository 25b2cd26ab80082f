// tcgen05.mma issue rate per SM for the shapes the output-layer kernels use:
// one CTA per SM, operands resident in shared memory (zeros), one thread
// issues R MMAs back to back into a TMEM accumulator, commit, wait.
//   shape: M128 x N{64,128,256} x K16, A from smem (SS) or from TMEM (TS)
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_1904_04956_b200/csrc \
//        mma_rate.cu -o mma_rate -lcuda
#include <cstdio>
#include <vector>

#include "ds_ptx.cuh"

using namespace ds;

__global__ void __launch_bounds__(128, 1) mma_rate(int n, int ts, int reps, int kchain, int nacc, unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  unsigned long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_bf16_f32(128, n, 0, 0);
    const uint32_t a = smem_u32(smem), b = a + 16384;
    t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      for (int k = 0; k < kchain; ++k) {
        const uint64_t bd = smem_desc_sw128(b + (k & 3) * 32, 16, 1024);
        // nacc independent accumulators interleaved (columns 256 + j * n / nacc... each n wide)
        const uint32_t d = nacc == 1 ? tmem + 256 : tmem + (uint32_t)((k % nacc) * (512 / nacc));
        if (ts)
          mma_bf16_ts(d, tmem + 256 + (k & 15) * 8, bd, idesc, k >= nacc ? 1u : 0u);
        else
          mma_bf16_ss(d, smem_desc_sw128(a + (k & 3) * 32, 16, 1024), bd, idesc, k >= nacc ? 1u : 0u);
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

// CTA-pair (cta_group::2) variant: M=256 across the pair, N split into halves staged by each CTA
__global__ void __launch_bounds__(128, 1) mma_rate_pair(int n, int reps, int kchain, unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc_pair(&slot, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0 && rank == 0) {
    const uint32_t idesc = idesc_bf16_f32(256, n, 0, 0);
    const uint32_t a = smem_u32(smem), b = a + 16384;
    const unsigned long long t0 = clock64();
    for (int r = 0; r < reps; ++r)
      for (int k = 0; k < kchain; ++k)
        mma_bf16_ss_pair(tmem, smem_desc_sw128(a + (k & 3) * 32, 16, 1024), smem_desc_sw128(b + (k & 3) * 32, 16, 1024),
                         idesc, k ? 1u : 0u);
    mma_commit_pair_mc(&bar, 0x3);
    mbar_wait(&bar, 0);
    out[blockIdx.x / 2] = clock64() - t0;
  } else if (threadIdx.x == 0) {
    mbar_wait(&bar, 0);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc_pair(tmem, 512);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d;
  cudaMalloc(&d, sizeof(unsigned long long) * sms);
  cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  const int reps = 2000, kchain = 16;
  for (int ts = 0; ts < 2; ++ts)
    for (int n : {64, 128, 256})
      for (int nacc : {1, 2, 4}) {
        if (nacc * n > 512 || (ts && nacc > 1)) continue;
        const int grid = sms;
        mma_rate<<<grid, 128, 65536 + 1024>>>(n, ts, reps, kchain, nacc, d);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<unsigned long long> h(grid);
        cudaMemcpy(h.data(), d, sizeof(unsigned long long) * grid, cudaMemcpyDeviceToHost);
        double mean = 0;
        for (auto c : h) mean += (double)c / grid;
        const double flop = 2.0 * 128 * n * 16 * reps * kchain;
        printf("%s N=%3d accumulators %d: %s  %.1f clk per MMA(M128,K16)  %.0f flop/clk/SM\n", ts ? "TS" : "SS", n,
               nacc, cudaGetErrorString(e), mean / (reps * kchain), flop / mean);
      }
  cudaFuncSetAttribute(mma_rate_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  for (int n : {64, 128, 256}) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(sms / 2 * 2);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = 65536 + 1024;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, mma_rate_pair, n, reps, kchain, d);
    cudaError_t e = cudaDeviceSynchronize();
    const int pairs = sms / 2;
    std::vector<unsigned long long> h(pairs);
    cudaMemcpy(h.data(), d, sizeof(unsigned long long) * pairs, cudaMemcpyDeviceToHost);
    double mean = 0;
    for (auto c : h) mean += (double)c / pairs;
    const double flop_per_sm = 2.0 * 128 * n * 16 * reps * kchain;  // each SM holds M=128 of the pair's 256
    printf("PAIR SS M256 N=%3d: %s  %.1f clk per MMA(M256,K16)  %.0f flop/clk/SM\n", n, cudaGetErrorString(e),
           mean / (reps * kchain), flop_per_sm / mean);
  }
  return 0;
}
