// Numerics check of the CTA-pair MMA with A read from tensor memory
// (tcgen05.mma.cta_group::2.kind::f16 [d], [a_tmem], b_desc): A [256 x K]
// split by CTA (rank r holds rows r*128.. in its TMEM, lane = row, column c
// = K elements 2c, 2c+1), B [N x K] K-major SWIZZLE_128B split by CTA along N
// (rank r stages rows r*N/2..), D [128 x N] fp32 in each CTA's TMEM.
// Small integers: every product and sum is exact, so the check is bit-exact.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_1904_04956_b200/csrc \
//        ts_pair_check.cu -o ts_pair_check -lcuda
#include <cstdio>
#include <vector>

#include "ds_ptx.cuh"

using namespace ds;

constexpr int K = 128, N = 128;

__global__ void __launch_bounds__(128, 1) tsk(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const uint32_t rank = cluster_ctarank();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // B half: rows rank*N/2 .. +N/2, K-major, 128-byte swizzle, K in 64-element atoms of (N/2) x 128 B
  for (int i = threadIdx.x; i < (N / 2) * (K / 8); i += blockDim.x) {
    const int n = i / (K / 8), c = i % (K / 8);  // 16-byte chunk c of row n
    const uint4 v = *reinterpret_cast<const uint4*>(B + (size_t)(rank * (N / 2) + n) * K + c * 8);
    const int atom = c / 8, cc = c % 8;
    *reinterpret_cast<uint4*>(smem + atom * (N / 2) * 128 + n * 128 + ((cc ^ (n & 7)) * 16)) = v;
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (w == 0) tmem_alloc_pair(&slot, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  // A rows rank*128 + w*32 + lane -> TMEM lane w*32+lane, columns 256 + k/2
  {
    const int row = rank * 128 + w * 32 + lane;
    uint32_t r[16];
    for (int c0 = 0; c0 < K / 2; c0 += 16) {
      for (int j = 0; j < 16; ++j) {
        const __nv_bfloat16 lo = A[(size_t)row * K + 2 * (c0 + j)], hi = A[(size_t)row * K + 2 * (c0 + j) + 1];
        r[j] = (uint32_t)__bfloat16_as_ushort(lo) | ((uint32_t)__bfloat16_as_ushort(hi) << 16);
      }
      tmem_st16(tmem + ((uint32_t)(w * 32) << 16) + 256 + c0, r);
    }
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  if (threadIdx.x == 0 && rank == 0) {
    const uint32_t idesc = idesc_bf16_f32(256, N, 0, 0);
    for (int k = 0; k < K / 16; ++k) {
      const uint64_t bd = smem_desc_sw128(smem_u32(smem) + (k / 4) * (N / 2) * 128 + (k % 4) * 32, 16, 1024);
      mma_bf16_ts_pair(tmem, tmem + 256 + k * 8, bd, idesc, k ? 1u : 0u);
    }
    mma_commit_pair_mc(&bar, 0x3);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  {
    float v[32];
    for (int c0 = 0; c0 < N; c0 += 32) {
      tmem_ld32(tmem + ((uint32_t)(w * 32) << 16) + c0, v);
      tmem_ld_wait();
      for (int j = 0; j < 32; ++j) D[(size_t)(rank * 128 + w * 32 + lane) * N + c0 + j] = v[j];
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  if (w == 0) tmem_dealloc_pair(tmem, 512);
}

int main() {
  std::vector<__nv_bfloat16> a(256 * K), b(N * K);
  std::vector<float> af(256 * K), bf(N * K);
  for (int i = 0; i < 256 * K; ++i) {
    af[i] = (float)((i * 7 + i / K * 3) % 9 - 4);
    a[i] = __float2bfloat16(af[i]);
  }
  for (int i = 0; i < N * K; ++i) {
    bf[i] = (float)((i * 5 + i / K) % 7 - 3);
    b[i] = __float2bfloat16(bf[i]);
  }
  __nv_bfloat16 *da, *db;
  float* dd;
  cudaMalloc(&da, a.size() * 2);
  cudaMalloc(&db, b.size() * 2);
  cudaMalloc(&dd, 256 * N * 4);
  cudaMemcpy(da, a.data(), a.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), b.size() * 2, cudaMemcpyHostToDevice);
  cudaMemset(dd, 0, 256 * N * 4);
  const int smem = (N / 2) * K * 2 + 1024;
  cudaFuncSetAttribute(tsk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, tsk, (const __nv_bfloat16*)da, (const __nv_bfloat16*)db, dd);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  std::vector<float> d(256 * N);
  cudaMemcpy(d.data(), dd, d.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  double maxerr = 0;
  for (int m = 0; m < 256; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int k = 0; k < K; ++k) ref += (double)af[m * K + k] * bf[n * K + k];
      const double err = fabs(ref - d[m * N + n]);
      if (err > maxerr) maxerr = err;
      if (err > 0 && bad++ < 5) printf("mismatch m=%d n=%d got %f want %f\n", m, n, d[m * N + n], ref);
    }
  printf("ts pair check (%s): %d mismatches of %d, max err %g\n", cudaGetErrorString(e), bad, 256 * N, maxerr);
  return 0;
}
