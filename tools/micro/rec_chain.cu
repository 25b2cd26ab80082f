// Recurrent-step building blocks, measured one at a time on one B200:
//   part 1: latency of ONE recurrent step's MMA chain (K = 512 as 32 x K16
//           MMAs into one accumulator, then commit + mbarrier wait), for
//           single-CTA / CTA-pair issue, A from smem (SS) or TMEM (TS),
//           N = 64 / 128 / 256; also the steady issue rate (throughput).
//   part 2: h all-gather inside a 16-CTA cluster (the forward recurrence's
//           exchange without the math): every CTA writes its 128 x 32 bf16
//           tile, then either
//             mode 0: st.global + fence.proxy.async + TMA multicast load of
//                     its own tile halves into the 8 CTAs of each rank parity
//             mode 1: st.global + release flag; consumers poll 16 flags and
//                     TMA-load every chunk themselves (the current scheme)
//           step period over 200 steps, 4 clusters (B = 256, two directions).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_1904_04956_b200/csrc \
//        rec_chain.cu -o rec_chain -lcuda
#include <cstdio>
#include <vector>

#include "ds_ptx.cuh"

using namespace ds;

// ---------------------------------------------------------------- part 1
__global__ void __launch_bounds__(128, 1) chain1(int n, int ts, int reps, unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
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
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_bf16_f32(128, n, 0, 0);
    const uint32_t a = smem_u32(smem), b = a + 65536;
    unsigned long long tot = 0;
    for (int r = 0; r < reps; ++r) {
      const unsigned long long t0 = clock64();
      for (int k = 0; k < 32; ++k) {
        const uint64_t bd = smem_desc_sw128(b + (k & 3) * 32, 16, 1024);
        if (ts)
          mma_bf16_ts(tmem, tmem + 256 + k * 8, bd, idesc, k ? 1u : 0u);
        else
          mma_bf16_ss(tmem, smem_desc_sw128(a + (k & 3) * 32 + (k >> 2) * 16384 / 2, 16, 1024), bd, idesc, k ? 1u : 0u);
      }
      mma_commit(&bar);
      mbar_wait(&bar, r & 1);
      tot += clock64() - t0;
    }
    out[blockIdx.x] = tot / reps;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

__global__ void __launch_bounds__(128, 1) chain2(int n, int ts, int reps, unsigned long long* out, int gap, int rnd) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = rnd ? (0x3c003c00u ^ (i * 2654435761u & 0x03ff03ffu)) : 0u;
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
  if (rnd) {  // random-ish bf16 A in TMEM columns 256..511
    uint32_t rr[16];
    for (int c0 = 0; c0 < 256; c0 += 16) {
      for (int j = 0; j < 16; ++j) rr[j] = 0x3c003c00u ^ ((threadIdx.x * 977 + (c0 + j) * 131) * 2654435761u & 0x03ff03ffu);
      tmem_st16(tmem + (((threadIdx.x >> 5) * 32) << 16) + 256 + c0, rr);
    }
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  unsigned long long tot = 0;
  for (int r = 0; r < reps; ++r) {
    if (threadIdx.x == 0) {
      if (gap) {
        const unsigned long long g0 = clock64();
        while (clock64() - g0 < (unsigned long long)gap) {
        }
      }
      const unsigned long long t0 = clock64();
      if (rank == 0) {
        const uint32_t idesc = idesc_bf16_f32(256, n, 0, 0);
        const uint32_t a = smem_u32(smem), b = a + 65536;
        for (int k = 0; k < 32; ++k) {
          const uint64_t bd = smem_desc_sw128(b + (k & 3) * 32, 16, 1024);
          if (ts)
            mma_bf16_ts_pair(tmem, tmem + 256 + k * 8, bd, idesc, k ? 1u : 0u);
          else
            mma_bf16_ss_pair(tmem, smem_desc_sw128(a + (k & 3) * 32, 16, 1024), bd, idesc, k ? 1u : 0u);
        }
        mma_commit_pair_mc(&bar, 0x3);
      }
      mbar_wait(&bar, r & 1);
      tot += clock64() - t0;
    }
    // keep the pair in lock-step: the next chain starts after both saw the commit
    __syncthreads();
    cluster_sync_all();
  }
  if (threadIdx.x == 0 && rank == 0) out[blockIdx.x / 2] = tot / reps;
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc_pair(tmem, 512);
}

// ---------------------------------------------------------------- part 2
constexpr int kSteps = 200;
constexpr int kTileBytes = 128 * 32 * 2;      // one CTA's h tile
constexpr int kHalf = 64 * 32 * 2;            // 4 KB: half the tile's rows
constexpr int kRecv = 16 * kHalf;             // one step's B operand per CTA (64 KB)

struct XArgs {
  CUtensorMap tm;  // h [steps*128 rows per cluster...] bf16 [rows, 512], box {32 units, 64 rows}
  __nv_bfloat16* h;
  uint32_t* flags;  // [clusters][16]
  unsigned long long* out;
  int mode;
};

__global__ void __launch_bounds__(288, 1) xchg(const __grid_constant__ XArgs A) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* recv = smem;  // [2][16][4 KB]
  uint64_t* full = reinterpret_cast<uint64_t*>(recv + 2 * kRecv);  // [2]
  const uint32_t me = cluster_ctarank();
  const int cl = blockIdx.x / 16;
  const uint32_t parity_mask = (me & 1) ? 0xAAAAu : 0x5555u;
  (void)parity_mask;
  if (threadIdx.x == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
  cluster_sync_all();
  uint32_t* flags = A.flags + cl * 16;
  const unsigned long long t0 = globaltimer();
  for (int s = 0; s < kSteps; ++s) {
    const int buf = s & 1;
    if (threadIdx.x == 256) mbar_arrive_expect_tx(&full[buf], kRecv);
    // every CTA writes its tile: rows [cl*steps*128 + s*128, +128), units [me*32, +32)
    if (threadIdx.x < 256) {
      const int row = threadIdx.x >> 1, half = threadIdx.x & 1;
      uint4* dst = reinterpret_cast<uint4*>(A.h + ((size_t)(cl * kSteps + s) * 128 + row) * 512 + me * 32 + half * 16);
      dst[0] = make_uint4(s, row, me, 0);
      dst[1] = make_uint4(s, row, me, 1);
      if (A.mode == 0) fence_proxy_async_global();
    }
    named_bar_sync(1, 256 + 32);
    if (threadIdx.x == 256) {
      const int grow = (cl * kSteps + s) * 128;
      if (A.mode == 0) {
        // rows 0-63 -> even ranks' slot `me`, rows 64-127 -> odd ranks'
        tma_load_2d_mc(recv + buf * kRecv + me * kHalf, &A.tm, &full[buf], me * 32, grow, 0x5555);
        tma_load_2d_mc(recv + buf * kRecv + me * kHalf, &A.tm, &full[buf], me * 32, grow + 64, 0xAAAA);
      } else {
        st_release_gpu(flags + me, (uint32_t)(s + 1));
        for (int p = 0; p < 16; ++p) {
          while (ld_acquire_gpu(flags + p) < (uint32_t)(s + 1)) {
          }
          fence_proxy_async_global();
          tma_load_2d(recv + buf * kRecv + p * kHalf, &A.tm, &full[buf], p * 32, grow + (me & 1) * 64);
        }
      }
    }
    mbar_wait(&full[buf], (s >> 1) & 1);
  }
  const unsigned long long t1 = globaltimer();
  if (threadIdx.x == 0) A.out[blockIdx.x] = t1 - t0;
  cluster_sync_all();
}

static int make_tmap_2d(CUtensorMap* out, const void* base, CUtensorMapDataType dtype, uint64_t inner, uint64_t outer,
                       uint64_t pitch, uint32_t bi, uint32_t bo, CUtensorMapSwizzle sw) {
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {pitch};
  cuuint32_t box[2] = {bi, bo};
  cuuint32_t estr[2] = {1, 1};
  return (int)cuTensorMapEncodeTiled(out, dtype, 2, const_cast<void*>(base), dims, strides, box, estr,
                                     CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d;
  cudaMalloc(&d, sizeof(unsigned long long) * 1024);
  std::vector<unsigned long long> h(1024);
  const size_t sm1 = 98304 + 1024;
  cudaFuncSetAttribute(chain1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
  cudaFuncSetAttribute(chain2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
  for (int ts = 0; ts < 2; ++ts)
    for (int n : {64, 128, 256}) {
      if (ts && n > 256) continue;
      chain1<<<sms, 128, sm1>>>(n, ts, 200, d);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h.data(), d, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
      double mean = 0;
      for (int i = 0; i < sms; ++i) mean += (double)h[i] / sms;
      printf("single %s M128 N%3d K512 chain+commit: %s %.0f cycles (%.3f us @1965)\n", ts ? "TS" : "SS", n,
             cudaGetErrorString(e), mean, mean / 1965.0);
    }
  for (int ts = 0; ts < 2; ++ts)
    for (int n : {64, 128, 256})
    for (int gap : {0, 4000, 12000})
    for (int rnd : {0, 1}) {
      if (n != 128 && (gap || rnd)) continue;
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(sms / 2 * 2);
      cfg.blockDim = dim3(128);
      cfg.dynamicSmemBytes = sm1;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, chain2, n, ts, 200, d, gap, rnd);
      cudaError_t e = cudaDeviceSynchronize();
      const int pairs = sms / 2;
      cudaMemcpy(h.data(), d, sizeof(unsigned long long) * pairs, cudaMemcpyDeviceToHost);
      double mean = 0;
      for (int i = 0; i < pairs; ++i) mean += (double)h[i] / pairs;
      printf("pair   %s M256 N%3d K512 chain+commit (idle gap %5d, %s data): %s %.0f cycles (%.3f us @1965)\n",
             ts ? "TS" : "SS", n, gap, rnd ? "random" : "zero", cudaGetErrorString(e), mean, mean / 1965.0);
    }

  // part 2
  const int clusters = 4;
  const size_t rows = (size_t)clusters * kSteps * 128;
  __nv_bfloat16* hb;
  uint32_t* flags;
  cudaMalloc(&hb, rows * 512 * 2);
  cudaMalloc(&flags, 4096);
  XArgs A{};
  if (make_tmap_2d(&A.tm, hb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 512, rows, 1024, 32, 64, CU_TENSOR_MAP_SWIZZLE_64B)) {
    printf("tmap failed\n");
    return 1;
  }
  A.h = hb;
  A.flags = flags;
  A.out = d;
  const size_t sm2 = 2 * kRecv + 1024 + 64;
  cudaFuncSetAttribute(xchg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
  cudaFuncSetAttribute(xchg, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int mode = 0; mode < 2; ++mode)
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(flags, 0, 4096);
      A.mode = mode;
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(16 * clusters);
      cfg.blockDim = dim3(288);
      cfg.dynamicSmemBytes = sm2;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 16;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaError_t e = cudaLaunchKernelEx(&cfg, xchg, A);
      if (e == cudaSuccess) e = cudaDeviceSynchronize();
      cudaMemcpy(h.data(), d, sizeof(unsigned long long) * 16 * clusters, cudaMemcpyDeviceToHost);
      double mx = 0;
      for (int i = 0; i < 16 * clusters; ++i) mx = h[i] > mx ? h[i] : mx;
      printf("xchg mode %d (%s): %s  %.3f us per step (max over CTAs)\n", mode,
             mode == 0 ? "st.global + TMA multicast" : "release flags + per-CTA TMA", cudaGetErrorString(e),
             mx / kSteps / 1000.0);
    }
  return 0;
}
