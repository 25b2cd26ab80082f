// p2p.cu — the multi-process (one process per GPU) synchronisation path:
// CUDA IPC export/import of learner buffers, a device-side barrier over
// peer-mapped flag words, the sharded SSGD step (reduce-scatter in the
// reference's canonical ring order + /divisor + momentum SGD on the owned
// chunk + all-gather of theta and its bf16 snapshot) and the ADPSGD pairwise
// mix, all as kernels that load and store the neighbours' memory directly
// over NVLink P2P.  NCCL is only the comparison transport (bench.py
// --transport nccl).
//
// Reference semantics:
//   SSGD step       engines/ssgd.py:80-90 + RingAllreduceGroup.allreduce
//                   (collective.py:122-163): chunk j (make_chunk_plan,
//                   collective.py:41-57) is owned by rank j % world and summed
//                   in the order owner, owner+1, ..., owner-1 (:133-145);
//                   g/world then sgd_step (optim.py:109-121).  Every learner
//                   applies the same update to bit-identical replicas
//                   (tests/test_ssgd.py:64-72), so the owner updates its own
//                   velocity for its chunks and broadcasts theta.
//   Hybrid average  engines/hybrid.py:97-99 (mode 1: theta <- sum / world).
//   ADPSGD mix      adpsgd_mix (engines/adpsgd.py:36-43): m = (a + b) / 2
//                   stored to both sides; each side of the pair mixes half
//                   of the vector so both NVLink directions carry traffic.
#include <cstring>

#include "../../include/ds_blstm.h"
#include "ds_internal.h"
#include "ds_ptx.cuh"

namespace ds {
namespace {

constexpr int kMaxPeers = 16;
constexpr int kEW = 256;

DS_DEV uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
DS_DEV void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

struct BarrierArgs {
  uint32_t* flags[kMaxPeers];  // member m's flag array (peer-mapped), indexed by world rank
  int ranks[kMaxPeers];        // world rank of member m
};

// one warp: lane m signals member m, then waits for member m's signal
__global__ void peer_barrier_kernel(BarrierArgs a, int n, int my_rank, uint32_t* own, uint32_t epoch, int* err,
                                    unsigned long long timeout_ns) {
  const int m = threadIdx.x;
  if (m < n) st_release_sys(a.flags[m] + my_rank, epoch);
  if (m < n) {
    const uint32_t* f = own + a.ranks[m];
    const uint64_t t0 = globaltimer();
    while (ld_acquire_sys(f) < epoch) {
      if (globaltimer() - t0 > timeout_ns) {  // a peer died or diverged: fail loudly, never hang
        atomicOr(err, 1);
        break;
      }
    }
  }
  __syncwarp();
}

struct ShardArgs {
  const float* g[kMaxPeers];
  float* theta[kMaxPeers];
  __nv_bfloat16* snap[kMaxPeers];
};

// one element of the owner's chunk (reference order: owner, owner+1, ...)
__device__ __forceinline__ float shard_elem(const ShardArgs& a, int world, int rank, int owner, float gsum_or_theta,
                                            float* v_own, int64_t i, float lr, float mu, int mode, float divisor) {
  if (mode == 0) {
    const float gm = __fdiv_rn(gsum_or_theta, divisor);
    const float vv = __fadd_rn(__fmul_rn(v_own[i], mu), gm);
    v_own[i] = vv;
    return __fsub_rn(a.theta[rank][i], __fmul_rn(lr, vv));
  }
  return __fdiv_rn(gsum_or_theta, divisor);
}

// chunks j = rank, rank + world, ... of ceil(n / nchunks) elements; float4
// vectors inside a chunk (scalar at its ragged edges), same arithmetic order
// as the reference's canonical ring sum.
__global__ void shard_step_kernel(ShardArgs a, int world, int rank, int64_t n, int64_t chunk, int nchunks,
                                  float* __restrict__ v_own, float lr, float mu, int mode, float divisor) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
  for (int j = rank; j < nchunks; j += world) {
    const int64_t lo = min(n, (int64_t)j * chunk), hi = min(n, (int64_t)(j + 1) * chunk);
    const int owner = j % world;  // == rank
    const float* const* src = mode == 0 ? a.g : a.theta;
    const int64_t lo4 = (lo + 3) / 4, hi4 = hi / 4;
    for (int64_t i4 = lo4 + tid; i4 < hi4; i4 += nth) {
      float4 sum = reinterpret_cast<const float4*>(src[owner])[i4];
      for (int k = 1; k < world; ++k) {
        const float4 x = reinterpret_cast<const float4*>(src[(owner + k) % world])[i4];
        sum.x = __fadd_rn(sum.x, x.x);
        sum.y = __fadd_rn(sum.y, x.y);
        sum.z = __fadd_rn(sum.z, x.z);
        sum.w = __fadd_rn(sum.w, x.w);
      }
      float4 w;
      if (mode == 0) {
        const float4 tv = reinterpret_cast<const float4*>(a.theta[rank])[i4];
        float4 vv = reinterpret_cast<const float4*>(v_own)[i4];
        vv.x = __fadd_rn(__fmul_rn(vv.x, mu), __fdiv_rn(sum.x, divisor));
        vv.y = __fadd_rn(__fmul_rn(vv.y, mu), __fdiv_rn(sum.y, divisor));
        vv.z = __fadd_rn(__fmul_rn(vv.z, mu), __fdiv_rn(sum.z, divisor));
        vv.w = __fadd_rn(__fmul_rn(vv.w, mu), __fdiv_rn(sum.w, divisor));
        reinterpret_cast<float4*>(v_own)[i4] = vv;
        w = make_float4(__fsub_rn(tv.x, __fmul_rn(lr, vv.x)), __fsub_rn(tv.y, __fmul_rn(lr, vv.y)),
                        __fsub_rn(tv.z, __fmul_rn(lr, vv.z)), __fsub_rn(tv.w, __fmul_rn(lr, vv.w)));
      } else {
        w = make_float4(__fdiv_rn(sum.x, divisor), __fdiv_rn(sum.y, divisor), __fdiv_rn(sum.z, divisor),
                        __fdiv_rn(sum.w, divisor));
      }
      __nv_bfloat162 b0 = __floats2bfloat162_rn(w.x, w.y), b1 = __floats2bfloat162_rn(w.z, w.w);
      uint2 pk;
      pk.x = *reinterpret_cast<uint32_t*>(&b0);
      pk.y = *reinterpret_cast<uint32_t*>(&b1);
      for (int r = 0; r < world; ++r) {  // all-gather: owner's result into every replica
        reinterpret_cast<float4*>(a.theta[r])[i4] = w;
        if (a.snap[r]) reinterpret_cast<uint2*>(a.snap[r])[i4] = pk;
      }
    }
    // ragged chunk edges
    // a chunk with no aligned float4 (lo4 > hi4) is all edge: one scalar range
    const int64_t e0 = lo, e1 = lo4 > hi4 ? hi : min(hi, lo4 * 4), f0 = lo4 > hi4 ? hi : max(lo, hi4 * 4), f1 = hi;
    for (int64_t t = tid; t < (e1 - e0) + (f1 - f0); t += nth) {
      const int64_t i = t < (e1 - e0) ? e0 + t : f0 + (t - (e1 - e0));
      float sum = src[owner][i];
      for (int k = 1; k < world; ++k) sum = __fadd_rn(sum, src[(owner + k) % world][i]);
      const float w = shard_elem(a, world, rank, owner, sum, v_own, i, lr, mu, mode, divisor);
      const __nv_bfloat16 wb = __float2bfloat16_rn(w);
      for (int r = 0; r < world; ++r) {
        a.theta[r][i] = w;
        if (a.snap[r]) a.snap[r][i] = wb;
      }
    }
  }
}

// m = (self + peer) / 2 on [lo, hi), stored to both sides (+ bf16 snapshots)
__global__ void pair_mix_kernel(float* __restrict__ self, float* __restrict__ peer, __nv_bfloat16* snap_self,
                                __nv_bfloat16* snap_peer, int64_t lo, int64_t hi) {
  const int64_t lo4 = (lo + 3) / 4, hi4 = hi / 4;
  for (int64_t i = lo4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hi4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 x = reinterpret_cast<const float4*>(self)[i];
    const float4 y = reinterpret_cast<const float4*>(peer)[i];
    x.x = __fmul_rn(__fadd_rn(x.x, y.x), 0.5f);
    x.y = __fmul_rn(__fadd_rn(x.y, y.y), 0.5f);
    x.z = __fmul_rn(__fadd_rn(x.z, y.z), 0.5f);
    x.w = __fmul_rn(__fadd_rn(x.w, y.w), 0.5f);
    reinterpret_cast<float4*>(self)[i] = x;
    reinterpret_cast<float4*>(peer)[i] = x;
    if (snap_self || snap_peer) {
      __nv_bfloat162 p0 = __floats2bfloat162_rn(x.x, x.y), p1 = __floats2bfloat162_rn(x.z, x.w);
      uint2 pk;
      pk.x = *reinterpret_cast<uint32_t*>(&p0);
      pk.y = *reinterpret_cast<uint32_t*>(&p1);
      if (snap_self) reinterpret_cast<uint2*>(snap_self)[i] = pk;
      if (snap_peer) reinterpret_cast<uint2*>(snap_peer)[i] = pk;
    }
  }
  // ragged edges (lo not 4-aligned / tail)
  const int64_t a0 = lo, a1 = lo4 > hi4 ? hi : min(hi, lo4 * 4), b0 = lo4 > hi4 ? hi : max(lo, hi4 * 4), b1 = hi;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (a1 - a0) + (b1 - b0);
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i < (a1 - a0) ? a0 + i : b0 + (i - (a1 - a0));
    const float m = __fmul_rn(__fadd_rn(self[k], peer[k]), 0.5f);
    self[k] = m;
    peer[k] = m;
    if (snap_self) snap_self[k] = __float2bfloat16_rn(m);
    if (snap_peer) snap_peer[k] = __float2bfloat16_rn(m);
  }
}

using AddrRangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
AddrRangeFn addr_range() {
  static AddrRangeFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<AddrRangeFn>(p);
    tried = true;
  }
  return fn;
}

int ew_grid(int64_t n) {
  int64_t b = (n + kEW - 1) / kEW;
  int64_t cap = (int64_t)num_sms() * 8;
  return (int)(b < cap ? (b > 0 ? b : 1) : cap);
}

}  // namespace
}  // namespace ds

using namespace ds;

extern "C" {

int ds_ipc_export(const void* ptr, void* handle_out, int64_t* offset_out) {
  if (!ptr || !handle_out || !offset_out) return fail_arg("null argument");
  AddrRangeFn range = addr_range();
  if (!range) return fail_arg("cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  CUresult r = range(&base, &size, reinterpret_cast<CUdeviceptr>(ptr));
  if (r != CUDA_SUCCESS) return fail_arg("ds_ipc_export: pointer is not a device allocation");
  cudaIpcMemHandle_t h;
  DS_CUDA_TRY(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  static_assert(sizeof(cudaIpcMemHandle_t) == DS_IPC_HANDLE_BYTES, "IPC handle size");
  memcpy(handle_out, &h, sizeof(h));
  *offset_out = (int64_t)(reinterpret_cast<CUdeviceptr>(ptr) - base);
  return DS_OK;
}

int ds_ipc_open(const void* handle, int64_t offset, void** base_out, void** ptr_out) {
  if (!handle || !base_out || !ptr_out || offset < 0) return fail_arg("null argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void* base = nullptr;
  DS_CUDA_TRY(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  *base_out = base;
  *ptr_out = static_cast<char*>(base) + offset;
  return DS_OK;
}

int ds_ipc_close(void* base) {
  if (!base) return DS_OK;
  DS_CUDA_TRY(cudaIpcCloseMemHandle(base));
  return DS_OK;
}

int ds_device_copy(void* dst, const void* src, int64_t bytes, ds_stream_t stream) {
  if (!dst || !src || bytes < 0) return fail_arg("null argument");
  DS_CUDA_TRY(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault, reinterpret_cast<cudaStream_t>(stream)));
  return DS_OK;
}

int ds_enable_peer_access(int32_t device, int32_t peer) {
  if (device == peer) return DS_OK;
  int can = 0;
  DS_CUDA_TRY(cudaDeviceCanAccessPeer(&can, device, peer));
  if (!can) return fail_arg("devices cannot access each other (no P2P path)");
  DS_CUDA_TRY(cudaSetDevice(device));
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return DS_OK;
  }
  if (e != cudaSuccess) return fail_cuda(e, "cudaDeviceEnablePeerAccess");
  return DS_OK;
}

int ds_peer_barrier(int32_t n, uint32_t* const* member_flags, const int32_t* member_ranks, int32_t my_rank,
                    uint32_t* own_flags, uint32_t epoch, int32_t* err, double timeout_s, ds_stream_t stream) {
  if (n < 1 || n > kMaxPeers) return fail_arg("barrier: member count out of range 1..16");
  if (!member_flags || !member_ranks || !own_flags || !err) return fail_arg("null argument");
  BarrierArgs a;
  memset(&a, 0, sizeof(a));
  for (int m = 0; m < n; ++m) {
    a.flags[m] = member_flags[m];
    a.ranks[m] = member_ranks[m];
    if (!a.flags[m] || a.ranks[m] < 0) return fail_arg("barrier: bad member");
  }
  const unsigned long long to = (unsigned long long)((timeout_s > 0 ? timeout_s : 30.0) * 1e9);
  peer_barrier_kernel<<<1, 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(a, n, my_rank, own_flags, epoch, err, to);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int ds_shard_step(int32_t world, int32_t rank, const float* const* grads, float* const* thetas,
                  void* const* snaps, float* v_own, int64_t n, int32_t nchunks, float lr, float mu, int32_t mode,
                  float divisor, ds_stream_t stream) {
  if (world < 1 || world > kMaxPeers) return fail_arg("group size out of range 1..16");
  if (rank < 0 || rank >= world) return fail_arg("rank out of range");
  if (nchunks < world) return fail_arg("chunk_count must be >= world");
  if (!thetas || n < 1) return fail_arg("null argument");
  if (mode != 0 && mode != 1) return fail_arg("mode must be 0 (sgd) or 1 (average)");
  for (int r = 0; r < world; ++r) {
    const uintptr_t al = reinterpret_cast<uintptr_t>(thetas[r]) | (grads ? reinterpret_cast<uintptr_t>(grads[r]) : 0) |
                         (snaps ? reinterpret_cast<uintptr_t>(snaps[r]) & 7 : 0);
    if (al & 15) return fail_arg("shard step: buffers must be 16-byte aligned");
  }
  if (v_own && (reinterpret_cast<uintptr_t>(v_own) & 15)) return fail_arg("shard step: velocity must be 16-byte aligned");
  if (mode == 0 && (!grads || !v_own)) return fail_arg("SGD step needs gradients and the velocity");
  if (mode == 0 && !(lr > 0.f)) return fail_arg("learning rate must be > 0");
  ShardArgs a;
  memset(&a, 0, sizeof(a));
  for (int r = 0; r < world; ++r) {
    a.g[r] = grads ? grads[r] : nullptr;
    a.theta[r] = thetas[r];
    a.snap[r] = snaps ? reinterpret_cast<__nv_bfloat16*>(snaps[r]) : nullptr;
    if (!a.theta[r] || (mode == 0 && !a.g[r])) return fail_arg("null member buffer");
  }
  const int64_t chunk = (n + nchunks - 1) / nchunks;
  shard_step_kernel<<<ew_grid(chunk / 4 + 1), kEW, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      a, world, rank, n, chunk, nchunks, v_own, lr, mu, mode, divisor > 0.f ? divisor : (float)world);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int ds_pair_mix(float* self, float* peer, void* snap_self, void* snap_peer, int64_t n, int32_t half,
                ds_stream_t stream) {
  if (!self || !peer || n < 1) return fail_arg("null argument");
  if (half < -1 || half > 1) return fail_arg("half must be -1 (all), 0 or 1");
  if (((reinterpret_cast<uintptr_t>(self) | reinterpret_cast<uintptr_t>(peer)) & 15) ||
      ((reinterpret_cast<uintptr_t>(snap_self) | reinterpret_cast<uintptr_t>(snap_peer)) & 7))
    return fail_arg("mix: buffers must be 16-byte aligned");
  const int64_t mid = (n / 2) & ~int64_t(3);
  const int64_t lo = half == 1 ? mid : 0, hi = half == 0 ? mid : n;
  pair_mix_kernel<<<ew_grid((hi - lo) / 4 + 1), kEW, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      self, peer, reinterpret_cast<__nv_bfloat16*>(snap_self), reinterpret_cast<__nv_bfloat16*>(snap_peer), lo, hi);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

}  // extern "C"
