// TMA load throughput from L2 into shared memory, no compute: the ceiling a
// tcgen05 GEMM mainloop runs into when its tile's bytes/flop are too high.
// 6 stages x 32 KB per CTA, persistent grid over all SMs, 16 MB operand
// (L2-resident after the first pass).
//   mode 0: unicast, every CTA reads its own tiles
//   mode 1: unicast, the two CTAs of a cluster pair read the same tiles
//   mode 2: cluster 2, each CTA loads one 16 KB box multicast to both
//   mode 3: cluster 4, each CTA loads one 8 KB box multicast to all four
//   mode 4: cluster 4 = 2 GEMM pairs sharing the A operand: each CTA loads an
//           8 KB A piece multicast to itself and its counterpart in the other
//           pair (ranks r, r^2) plus its own 16 KB B half unicast
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_1904_04956_b200/csrc \
//        tma_bw.cu ../../paper_1904_04956_b200/csrc/common.cu -o tma_bw -lcuda
#include <cstdio>
#include <vector>

#include "ds_internal.h"
#include "ds_ptx.cuh"

using namespace ds;

constexpr int kStages = 6;
constexpr int kStage = 32768;

struct Args {
  CUtensorMap m128, m64;
  int mode, iters;
  unsigned long long* clk;
};

__device__ __forceinline__ uint32_t cluster_nctas() {
  uint32_t n;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(n));
  return n;
}

__global__ void __launch_bounds__(64, 1) tma_bw(const __grid_constant__ Args a) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStage);
  uint64_t* empty = full + kStages;
  const uint32_t rank = a.mode >= 2 ? cluster_ctarank() : 0;
  const uint32_t ncl = a.mode >= 2 ? cluster_nctas() : 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], a.mode == 4 ? 2 : ncl);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (a.mode >= 2) cluster_sync_all();
  const int cta = blockIdx.x;
  const int group = a.mode == 1 ? cta / 2 : (a.mode >= 2 ? cta / (int)ncl : cta);
  unsigned long long t0 = clock64();
  if (threadIdx.x == 0) {  // producer
    int stage = 0;
    uint32_t phase = 0;
    for (int kb = 0; kb < a.iters; ++kb) {
      mbar_wait(&empty[stage], phase ^ 1);
      const int col = (kb % 16) * 64;
      const int rb = (group * 7 + kb / 16) % 64;  // 128-row block of the 8192-row operand
      uint8_t* dst = smem + stage * kStage;
      mbar_arrive_expect_tx(&full[stage], kStage);
      if (a.mode <= 1) {
        tma_load_2d(dst, &a.m128, &full[stage], col, rb * 128);
        tma_load_2d(dst + 16384, &a.m128, &full[stage], col, (rb ^ 1) * 128);
      } else if (a.mode == 2) {
        tma_load_2d_mc(dst + rank * 16384, &a.m128, &full[stage], col, ((rb ^ rank) & 63) * 128, 0x3);
      } else if (a.mode == 4) {
        const uint16_t mask = (uint16_t)((1u << (rank & 1)) | (1u << ((rank & 1) + 2)));
        tma_load_2d_mc(dst + (rank >> 1) * 8192, &a.m64, &full[stage], col, rb * 128 + (rank >> 1) * 64, mask);
        tma_load_2d(dst + 16384, &a.m128, &full[stage], col, ((rb + 1 + rank) & 63) * 128);
      } else {
        tma_load_2d_mc(dst + rank * 8192, &a.m64, &full[stage], col, (rank >= 2 ? rb ^ 1 : rb) * 128 + (rank & 1) * 64,
                       0xF);
      }
      if (++stage == kStages) {
        stage = 0;
        phase ^= 1;
      }
    }
  } else if (threadIdx.x == 32) {  // consumer: release each stage as soon as it lands
    int stage = 0;
    uint32_t phase = 0;
    const uint32_t e0 = smem_u32(empty);
    for (int kb = 0; kb < a.iters; ++kb) {
      mbar_wait(&full[stage], phase);
      if (a.mode == 4) {
        mbar_arrive(&empty[stage]);
        mbar_arrive_remote(mapa_shared(e0 + stage * 8, rank ^ 2));
      } else {
        for (uint32_t r = 0; r < ncl; ++r) {
          if (ncl == 1)
            mbar_arrive(&empty[stage]);
          else
            mbar_arrive_remote(mapa_shared(e0 + stage * 8, r));
        }
      }
      if (++stage == kStages) {
        stage = 0;
        phase ^= 1;
      }
    }
  }
  __syncthreads();
  if (a.mode >= 2) cluster_sync_all();
  if (threadIdx.x == 0) a.clk[cta] = clock64() - t0;
}

int main() {
  const int rows = 8192, cols = 1024;
  void* buf;
  cudaMalloc(&buf, (size_t)rows * cols * 2);
  cudaMemset(buf, 0, (size_t)rows * cols * 2);
  Args a{};
  if (make_tmap_2d(&a.m128, buf, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, cols, rows, cols * 2, 64, 128) ||
      make_tmap_2d(&a.m64, buf, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, cols, rows, cols * 2, 64, 64)) {
    printf("tmap failed\n");
    return 1;
  }
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaMalloc(&a.clk, sizeof(unsigned long long) * 1024);
  const size_t smem = 1024 + kStages * kStage + 256;
  cudaFuncSetAttribute(tma_bw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(tma_bw, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cl : {2, 4, 8}) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(cl * 64);
    cfg.blockDim = dim3(640);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, tma_bw, &cfg);
    printf("cluster %d, %zu B smem: max active clusters %d (%d CTAs) %s\n", cl, smem, n, n * cl, cudaGetErrorString(e));
  }
  for (int mode = 0; mode < 5; ++mode) {
    for (int nct : {sms / 4 * 4, 136, 128, 74}) {
      a.mode = mode;
      a.iters = 4000;
      const int cl = mode == 2 ? 2 : (mode >= 3 ? 4 : 1);
      const int grid = nct / cl * cl;
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(64);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cl;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaLaunchKernelEx(&cfg, tma_bw, a);  // warm
      cudaEventRecord(e0);
      cudaLaunchKernelEx(&cfg, tma_bw, a);
      cudaEventRecord(e1);
      cudaError_t err = cudaDeviceSynchronize();
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      std::vector<unsigned long long> clk(grid);
      cudaMemcpy(clk.data(), a.clk, sizeof(unsigned long long) * grid, cudaMemcpyDeviceToHost);
      double mean = 0;
      for (auto c : clk) mean += (double)c / grid;
      const double bytes = (double)grid * a.iters * kStage;
      printf("mode %d ctas %3d: %s  %.3f ms  %.2f TB/s delivered to smem, %.1f B/clk/SM (SM clk %.0f MHz)\n", mode,
             grid, cudaGetErrorString(err), ms, bytes / (ms * 1e-3) / 1e12, (double)a.iters * kStage / mean,
             mean / (ms * 1e3));
    }
  }
  return 0;
}
