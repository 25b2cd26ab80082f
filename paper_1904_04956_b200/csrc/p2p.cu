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
#include "p2p.h"

namespace ds {
namespace {

constexpr int kMaxPeers = kMaxGroupPeers;
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

// one warp: lane m signals member m, then waits for member m's signal.  The
// epoch is counted per (self, member) pair in device memory (pair_epochs,
// indexed by world rank; the kernel increments it), so ranks may take part in
// different subsets of barriers (pairs, groups) without a stale flag of one
// subset satisfying another's wait, and the barrier can live inside a
// replayed CUDA graph; comparisons are wrap-safe.
__global__ void peer_barrier_kernel(BarrierArgs a, int n, int my_rank, uint32_t* own, uint32_t* pair_epochs,
                                    int* err, unsigned long long timeout_ns) {
  const int m = threadIdx.x;
  uint32_t epoch = 0;
  if (m < n) {
    epoch = pair_epochs[a.ranks[m]] + 1;
    pair_epochs[a.ranks[m]] = epoch;
    st_release_sys(a.flags[m] + my_rank, epoch);
  }
  if (m < n) {
    const uint32_t* f = own + a.ranks[m];
    const uint64_t t0 = globaltimer();
    while ((int32_t)(ld_acquire_sys(f) - epoch) < 0) {
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
                                  float* __restrict__ v_own, float lr, float mu, int mode, float divisor,
                                  int64_t r_lo, int64_t r_hi, const float* lr_dev) {
  if (lr_dev) lr = *lr_dev;  // fused training step: the rate lives in device memory (graph replays)
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
  for (int j = rank; j < nchunks; j += world) {
    // the owned chunk, clipped to the requested element range [r_lo, r_hi)
    const int64_t lo = max(r_lo, min(n, (int64_t)j * chunk)), hi = min(r_hi, min(n, (int64_t)(j + 1) * chunk));
    if (lo >= hi) continue;
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
  __threadfence_system();  // peer stores performed before a following ds_peer_unlock releases the pair
}

// N1 (throughput mode): the sender's momentum step fused with its pairwise
// average in one pass over the vector (one NVLink read + write of the peer):
//   v <- mu v + g;  t' = theta - lr v;  snap <- bf16(t')  (the next gradient
//   is computed on the pre-mix t', engines/adpsgd.py:145 then :196);
//   m = (t' + peer) / 2 stored to theta and peer (adpsgd_mix, :36-43).
__global__ void update_mix_kernel(float* __restrict__ self, float* __restrict__ v, const float* __restrict__ g,
                                  float* __restrict__ peer, __nv_bfloat16* __restrict__ snap, float lr, float mu,
                                  int64_t n, int* flag) {
  const int64_t n4 = n / 4;
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 t = reinterpret_cast<const float4*>(self)[i];
    float4 vv = reinterpret_cast<const float4*>(v)[i];
    const float4 gg = reinterpret_cast<const float4*>(g)[i];
    const float4 p = reinterpret_cast<const float4*>(peer)[i];
    bad |= !isfinite(gg.x) || !isfinite(gg.y) || !isfinite(gg.z) || !isfinite(gg.w);
    vv.x = __fadd_rn(__fmul_rn(vv.x, mu), gg.x);
    vv.y = __fadd_rn(__fmul_rn(vv.y, mu), gg.y);
    vv.z = __fadd_rn(__fmul_rn(vv.z, mu), gg.z);
    vv.w = __fadd_rn(__fmul_rn(vv.w, mu), gg.w);
    t.x = __fsub_rn(t.x, __fmul_rn(lr, vv.x));
    t.y = __fsub_rn(t.y, __fmul_rn(lr, vv.y));
    t.z = __fsub_rn(t.z, __fmul_rn(lr, vv.z));
    t.w = __fsub_rn(t.w, __fmul_rn(lr, vv.w));
    reinterpret_cast<float4*>(v)[i] = vv;
    if (snap) {
      __nv_bfloat162 b0 = __floats2bfloat162_rn(t.x, t.y), b1 = __floats2bfloat162_rn(t.z, t.w);
      uint2 pk;
      pk.x = *reinterpret_cast<uint32_t*>(&b0);
      pk.y = *reinterpret_cast<uint32_t*>(&b1);
      reinterpret_cast<uint2*>(snap)[i] = pk;
    }
    const float4 m = make_float4(__fmul_rn(__fadd_rn(t.x, p.x), 0.5f), __fmul_rn(__fadd_rn(t.y, p.y), 0.5f),
                                 __fmul_rn(__fadd_rn(t.z, p.z), 0.5f), __fmul_rn(__fadd_rn(t.w, p.w), 0.5f));
    reinterpret_cast<float4*>(self)[i] = m;
    reinterpret_cast<float4*>(peer)[i] = m;
  }
  for (int64_t i = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    bad |= !isfinite(g[i]);
    const float vv = __fadd_rn(__fmul_rn(v[i], mu), g[i]);
    const float t = __fsub_rn(self[i], __fmul_rn(lr, vv));
    v[i] = vv;
    if (snap) snap[i] = __float2bfloat16_rn(t);
    const float m = __fmul_rn(__fadd_rn(t, peer[i]), 0.5f);
    self[i] = m;
    peer[i] = m;
  }
  if (bad && flag) atomicOr(flag, 1);
  __threadfence_system();
}

// Exclusive access of a learner's weights across devices: a lock word in the
// owner's memory taken with a system-scope CAS by one thread.  The learner's
// own update and every incoming pairwise mix take it, so a mix and an update
// never interleave (the receiver's atomic region, engines/adpsgd.py:280-285).
__global__ void lock_kernel(uint32_t* word, uint32_t owner, int* err, unsigned long long timeout_ns) {
  const uint64_t t0 = globaltimer();
  while (atomicCAS_system(word, 0u, owner) != 0u) {
    if (globaltimer() - t0 > timeout_ns) {
      atomicOr(err, 2);
      return;
    }
    __nanosleep(256);
  }
  __threadfence_system();
}
__global__ void unlock_kernel(uint32_t* word) {
  __threadfence_system();
  atomicExch_system(word, 0u);
}

// Debug payload digest (WeightMessage.snapshot / validate, engines/common.py:
// 78-104): 128 bits = two wrapping sums of independent 64-bit mixes of
// (index, word) over the buffer's 32-bit words.  Order-independent, so the
// parallel reduction is deterministic; any change of a word changes it with
// overwhelming probability (a torn or mutated payload), not a cryptographic hash.
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__global__ void digest_kernel(const uint32_t* __restrict__ words, int64_t n, unsigned long long* out) {
  uint64_t a = 0, b = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = ((uint64_t)i << 32) | words[i];
    a += mix64(key);
    b += mix64(key ^ 0xD6E8FEB86659FD93ull);
  }
  for (int o = 16; o; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  __shared__ unsigned long long red[2][32];  // per-warp partials, one atomic pair per block
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[0][w] = a;
    red[1][w] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
      a += red[0][i];
      b += red[1][i];
    }
    atomicAdd(out, (unsigned long long)a);
    atomicAdd(out + 1, (unsigned long long)b);
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

int group_barrier(const GroupSync& g, cudaStream_t s) {
  BarrierArgs a;
  memset(&a, 0, sizeof(a));
  for (int m = 0; m < g.n; ++m) {
    a.flags[m] = g.flags[m];
    a.ranks[m] = g.ranks[m];
  }
  const unsigned long long to = (unsigned long long)((g.timeout_s > 0 ? g.timeout_s : 30.0) * 1e9);
  peer_barrier_kernel<<<1, 32, 0, s>>>(a, g.n, g.my_rank, g.own_flags, g.pair_epochs, g.err, to);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int group_shard_range(const GroupSync& g, int64_t n, int64_t lo, int64_t hi, float* v_own, const float* lr_dev,
                      float mu, cudaStream_t s) {
  ShardArgs a;
  memset(&a, 0, sizeof(a));
  for (int m = 0; m < g.n; ++m) {
    a.g[m] = g.grads[m];
    a.theta[m] = g.thetas[m];
    a.snap[m] = reinterpret_cast<__nv_bfloat16*>(g.snaps[m]);
  }
  const int64_t chunk = (n + g.nchunks - 1) / g.nchunks;
  int grid = ew_grid((hi - lo) / g.n / 4 + 1);
  if (g.max_blocks > 0 && grid > g.max_blocks) grid = g.max_blocks;
  shard_step_kernel<<<grid, kEW, 0, s>>>(a, g.n, g.me, n, chunk, g.nchunks, v_own, 1.f, mu, 0,
                                         g.divisor > 0.f ? g.divisor : (float)g.n, lo, hi, lr_dev);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

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
                    uint32_t* own_flags, uint32_t* pair_epochs, int32_t* err, double timeout_s,
                    ds_stream_t stream) {
  if (n < 1 || n > kMaxPeers) return fail_arg("barrier: member count out of range 1..16");
  if (!member_flags || !member_ranks || !own_flags || !err) return fail_arg("null argument");
  BarrierArgs a;
  memset(&a, 0, sizeof(a));
  for (int m = 0; m < n; ++m) {
    a.flags[m] = member_flags[m];
    a.ranks[m] = member_ranks[m];
    if (!a.flags[m] || a.ranks[m] < 0 || a.ranks[m] >= 64) return fail_arg("barrier: bad member");
  }
  if (!pair_epochs) return fail_arg("barrier: null pair epoch array");
  const unsigned long long to = (unsigned long long)((timeout_s > 0 ? timeout_s : 30.0) * 1e9);
  peer_barrier_kernel<<<1, 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(a, n, my_rank, own_flags, pair_epochs,
                                                                            err, to);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int ds_shard_step_range(int32_t world, int32_t rank, const float* const* grads, float* const* thetas,
                        void* const* snaps, float* v_own, int64_t n, int32_t nchunks, float lr, float mu,
                        int32_t mode, float divisor, int64_t range_lo, int64_t range_hi, int32_t max_blocks,
                        ds_stream_t stream) {
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
  if (range_lo < 0 || range_hi > n || range_lo >= range_hi) return fail_arg("shard step: bad element range");
  if (range_lo % 4) return fail_arg("shard step: range start must be a multiple of 4");
  int grid = ew_grid((range_hi - range_lo) / world / 4 + 1);
  if (max_blocks > 0 && grid > max_blocks) grid = max_blocks;
  shard_step_kernel<<<grid, kEW, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      a, world, rank, n, chunk, nchunks, v_own, lr, mu, mode, divisor > 0.f ? divisor : (float)world, range_lo,
      range_hi, nullptr);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int ds_shard_step(int32_t world, int32_t rank, const float* const* grads, float* const* thetas,
                  void* const* snaps, float* v_own, int64_t n, int32_t nchunks, float lr, float mu, int32_t mode,
                  float divisor, ds_stream_t stream) {
  return ds_shard_step_range(world, rank, grads, thetas, snaps, v_own, n, nchunks, lr, mu, mode, divisor, 0, n, 0,
                             stream);
}

int ds_update_mix(float* theta, float* vel, const float* grad, float* theta_peer, void* snap, float lr, float mu,
                  int64_t n, int32_t* nonfinite, ds_stream_t stream) {
  if (!theta || !vel || !grad || !theta_peer || n < 1) return fail_arg("null argument");
  if (!(lr > 0.f)) return fail_arg("learning rate must be > 0");
  if ((reinterpret_cast<uintptr_t>(theta) | reinterpret_cast<uintptr_t>(vel) | reinterpret_cast<uintptr_t>(grad) |
       reinterpret_cast<uintptr_t>(theta_peer)) & 15 || (reinterpret_cast<uintptr_t>(snap) & 7))
    return fail_arg("update_mix: buffers must be 16-byte aligned");
  update_mix_kernel<<<ew_grid(n / 4 + 1), kEW, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      theta, vel, grad, theta_peer, reinterpret_cast<__nv_bfloat16*>(snap), lr, mu, n, nonfinite);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int ds_peer_lock(uint32_t* word, uint32_t owner, int32_t* err, double timeout_s, ds_stream_t stream) {
  if (!word || !err || owner == 0) return fail_arg("lock: null word / error flag or owner id 0");
  const unsigned long long to = (unsigned long long)((timeout_s > 0 ? timeout_s : 30.0) * 1e9);
  lock_kernel<<<1, 1, 0, reinterpret_cast<cudaStream_t>(stream)>>>(word, owner, err, to);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int ds_peer_unlock(uint32_t* word, ds_stream_t stream) {
  if (!word) return fail_arg("unlock: null word");
  unlock_kernel<<<1, 1, 0, reinterpret_cast<cudaStream_t>(stream)>>>(word);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int ds_digest(const void* data, int64_t nbytes, unsigned long long* out2, ds_stream_t stream) {
  if (!data || !out2 || nbytes < 0 || (nbytes & 3)) return fail_arg("digest: null buffer or size not a multiple of 4");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  DS_CUDA_TRY(cudaMemsetAsync(out2, 0, 16, s));
  const int64_t n = nbytes / 4;
  digest_kernel<<<ew_grid(n), kEW, 0, s>>>(reinterpret_cast<const uint32_t*>(data), n, out2);
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
