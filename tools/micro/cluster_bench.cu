// Cluster-primitive microbenchmarks for the recurrent-kernel design:
//   1. hop latency of a remote mbarrier arrive (release.cluster) between two
//      CTAs of a cluster, no data
//   2. hop latency of "st.global 4 KB -> fence -> remote arrive -> TMA-style
//      bulk load of the 4 KB"
//   3. hop latency of a DSMEM bulk push (cp.async.bulk smem -> peer smem,
//      complete_tx on the peer's mbarrier) of `bytes`
//   4. all-to-all DSMEM push bandwidth: every CTA of a 16-CTA cluster pushes
//      `bytes` to 4 peers per round
//   5. max active clusters of 8 / 16 CTAs at ~200 KB smem
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 cluster_bench.cu -o cluster_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t ctarank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) { uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o; }
__device__ __forceinline__ void cl_sync() { asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void arrive_remote(uint32_t ca) { asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ca) : "memory"); }
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t bytes) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory"); }
__device__ __forceinline__ void wait_cl(uint64_t* b, uint32_t ph) {
  asm volatile("{\n\t.reg .pred P1;\n\tW_%=:\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}\n" ::"r"(smem_u32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk_s2c(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst), "r"(smem_u32(src)), "r"(bytes), "r"(mbar) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(mbar)) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }

// MODE 1: arrive only; MODE 2: global data + fence + arrive, bulk load; MODE 3: DSMEM push
template <int MODE>
__global__ void __cluster_dims__(16, 1, 1) hop(int iters, int bytes, uint8_t* gbuf, unsigned long long* out, int fence_gpu) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
  uint8_t* buf = sm + 1024;
  const uint32_t me = ctarank();
  const uint32_t peer = me == 0 ? 8 : 0;  // ranks 0 and 8 play; the rest idle
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    if (MODE == 3) asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
    fence_init();
  }
  __syncthreads();
  cl_sync();
  const bool player = me == 0 || me == 8;
  long long t0 = clock64();
  if (player) {
    for (int i = 0; i < iters; ++i) {
      const bool my_turn_first = me == 0;
      // receive (except the very first send of rank 0)
      if (!(my_turn_first && i == 0)) {
        if (threadIdx.x == 0) {
          if (MODE == 2) {
            wait_cl(bar, (uint32_t)((i - (my_turn_first ? 1 : 0)) & 1) ^ 0);
          } else {
            wait_cl(bar, (uint32_t)((i - (my_turn_first ? 1 : 0)) & 1));
          }
        }
        if (MODE == 3 && threadIdx.x == 0)  // arm for the next incoming copy before replying
          asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
        __syncthreads();
        if (MODE == 2) {  // pull the peer's global data through the bulk engine
          __shared__ __align__(8) uint64_t lbar;
          if (threadIdx.x == 0) {
            mbar_init(&lbar, 1);
            asm volatile("fence.proxy.async.global;" ::: "memory");
            expect_tx(&lbar, bytes);
            bulk_g2s(buf, gbuf + (size_t)peer * 65536, bytes, &lbar);
            wait_cl(&lbar, 0);
          }
          __syncthreads();
        }
      }
      if (my_turn_first || i < iters) {
        // send
        if (MODE == 1) {
          if (threadIdx.x == 0) arrive_remote(mapa(smem_u32(bar), peer));
        } else if (MODE == 2) {
          uint4* g = reinterpret_cast<uint4*>(gbuf + (size_t)me * 65536);
          for (int k = threadIdx.x; k < bytes / 16; k += blockDim.x) g[k] = make_uint4(i, k, me, 1);
          if (fence_gpu) asm volatile("fence.acq_rel.gpu;" ::: "memory");
          __syncthreads();
          if (threadIdx.x == 0) {
            if (!fence_gpu) asm volatile("fence.acq_rel.cluster;" ::: "memory");
            arrive_remote(mapa(smem_u32(bar), peer));
          }
        } else {
          if (threadIdx.x == 0) {
            // peer expects tx on its own barrier: encode as remote expect via arrive.expect_tx isn't
            // available remotely, so the receiver pre-arms; here the sender copies and the copy's
            // complete_tx + one remote arrive complete the phase
            bulk_s2c(mapa(smem_u32(buf), peer), buf, bytes, mapa(smem_u32(bar), peer));
            bulk_commit();
            arrive_remote(mapa(smem_u32(bar), peer));
            bulk_wait_read0();
          }
        }
      }
      __syncthreads();
    }
  }
  long long t1 = clock64();
  if (player && threadIdx.x == 0) out[me == 0 ? 0 : 1] = t1 - t0;
  cl_sync();
}

// all-to-all push bandwidth: each CTA pushes `bytes` to 4 peers (rank+1..+4) per round
__global__ void __cluster_dims__(16, 1, 1) a2a(int rounds, int bytes, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
  uint8_t* src = sm + 1024;
  uint8_t* dst = src + 4 * bytes;  // 4 receive slots
  const uint32_t me = ctarank();
  if (threadIdx.x == 0) { mbar_init(bar, 4); fence_init(); }
  __syncthreads();
  cl_sync();
  long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(4 * bytes) : "memory");
    }
    cl_sync();  // everyone armed (and done reading last round's slots)
    if (threadIdx.x < 4) {
      const uint32_t p = (me + 1 + threadIdx.x) % 16;
      const uint32_t slot = (threadIdx.x + 0) * bytes;  // receiver slot by sender offset
      bulk_s2c(mapa(smem_u32(dst + slot), p), src, bytes, mapa(smem_u32(bar), p));
      bulk_commit();
      arrive_remote(mapa(smem_u32(bar), p));
      bulk_wait_read0();
    }
    if (threadIdx.x == 0) wait_cl(bar, r & 1);
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
  int dev = 0;
  cudaSetDevice(dev);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  uint8_t* g;
  cudaMalloc(&g, 16 * 65536);
  unsigned long long* d_out;
  cudaMalloc(&d_out, 1024 * sizeof(unsigned long long));
  unsigned long long h[1024];
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(hop<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(hop<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(hop<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(a2a, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (auto f : {(const void*)hop<1>, (const void*)hop<2>, (const void*)hop<3>, (const void*)a2a})
    cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  // 5. residency
  for (int cs : {8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 8);
    cfg.blockDim = dim3(384);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (const void*)a2a, &cfg);
    printf("cluster %2d x 200KB smem: max active clusters %d (%s)\n", cs, n, cudaGetErrorString(e));
  }
  const int iters = 2000;
  for (int mode = 1; mode <= 3; ++mode) {
    for (int bytes : {4096, 8192, 16384, 32768}) {
      for (int fg = 0; fg <= (mode == 2 ? 1 : 0); ++fg) {
        if (mode == 1 && bytes != 4096) continue;
        cudaMemset(d_out, 0, 16);
        if (mode == 1) hop<1><<<16, 128, smem>>>(iters, bytes, g, d_out, fg);
        if (mode == 2) hop<2><<<16, 128, smem>>>(iters, bytes, g, d_out, fg);
        if (mode == 3) hop<3><<<16, 128, smem>>>(iters, bytes, g, d_out, fg);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d_out, 16, cudaMemcpyDeviceToHost);
        printf("mode %d bytes %6d fence_gpu %d: %s  %.1f cycles/hop (%.3f us @ %d MHz)\n", mode, bytes, fg,
               cudaGetErrorString(e), (double)h[0] / (2.0 * iters), (double)h[0] / (2.0 * iters) / (clk / 1e3),
               clk / 1000);
      }
    }
  }
  for (int bytes : {2048, 4096, 8192, 16384}) {
    const int rounds = 500;
    a2a<<<16 * 8, 128, smem>>>(rounds, bytes, d_out);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d_out, 128 * 8, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < 128; ++i) mx = h[i] > mx ? h[i] : mx;
    const double cyc = mx / rounds;
    printf("a2a push 4 x %5d B per CTA per round (8 clusters x 16): %s %.0f cycles/round -> %.1f B/cycle/SM out\n",
           bytes, cudaGetErrorString(e), cyc, 4.0 * bytes / cyc);
  }
  return 0;
}
