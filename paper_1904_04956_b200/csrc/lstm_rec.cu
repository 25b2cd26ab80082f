// lstm_rec.cu — persistent recurrent kernels of one bidirectional LSTM layer
// (SURVEY §2.3 K4 forward + cell, K5 BPTT + cell backward).
//
// Layout (per learner, time-major frames n = t*B + b):
//   gates  [N, 4096] bf16  : input projection X W_ih^T + b on entry (forward),
//                            overwritten in place by the post-activation gates
//                            (i, f, g, o) that BPTT consumes.
//   cstate [N, 1024] f32   : cell state c_t, columns dir*512 + unit.
//   Y_full [(T+2)B, 1024]  : layer output h_t at rows (t+1)*B + b; rows
//                            [0, B) and [(T+1)B, (T+2)B) are zero so h_{-1}
//                            and h_T read as zeros for either direction.
// Gate rows are unit-interleaved: row r = unit*4 + gate (gate 0..3 = i,f,g,o),
// so a CTA that owns 32 hidden units owns 128 contiguous gate rows and the
// cell update is thread-local.
//
// Forward CTA (dir, batch tile, unit block of 32):
//   W_hh[dir][unit block] (128 x 512 bf16, 128 KB) stays resident in smem.
//   step s: acc[128 batch, 128 gate rows] = h_prev[128, 512] . W^T (tcgen05,
//   M=128 N=128 K=512, A streamed by TMA from L2), epilogue adds the input
//   projection, applies sigmoid/tanh, updates c and h in registers/HBM, then
//   releases a per-(dir, batch tile) counter; the producer of every CTA in
//   that group acquires it before loading h_t for the next step.
// Backward CTA (dir, batch tile, unit block of 32):
//   W_hh^T[dir][unit block] (32 x 2048 bf16, 128 KB) resident.
//   step s: acc[128 batch, 32 units] = dG_prev[128, 2048] . W^T  (dh from the
//   recurrence), epilogue adds dY, runs the cell backward, writes dG_t.
// The grid (<= #SMs, one CTA per SM) is launched cooperatively so every CTA
// of a group is co-resident.
#include "ds_internal.h"
#include "ds_ptx.cuh"
#include "lstm_rec.h"

namespace ds {

namespace {

constexpr int kThreads = 256;
constexpr int kEpiWarp0 = 4;
constexpr int kUnits = 32;            // hidden units per CTA
constexpr int kRows = 4 * kUnits;     // gate rows per CTA
constexpr int kH = 512;               // hidden units per direction
constexpr int kStages = 4;
constexpr int kTileA = 128 * 64 * 2;  // one 128x64 bf16 A box (16 KB)

// forward: W slice 8 boxes of [128 rows x 64] = 128 KB
constexpr int kFwdWBytes = (kH / 64) * kRows * 64 * 2;
// backward: W^T slice 32 boxes of [32 rows x 64] = 128 KB
constexpr int kBwdWBytes = (4 * kH / 64) * kUnits * 64 * 2;
constexpr size_t kSmemBytes = 1024 + 128 * 1024 + kStages * kTileA + 256;

__device__ __forceinline__ void load_bf16x8(const __nv_bfloat16* p, float* out) {
  uint4 w = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 f = __bfloat1622float2(h[i]);
    out[2 * i] = f.x;
    out[2 * i + 1] = f.y;
  }
}
__device__ __forceinline__ void store_bf16x8(__nv_bfloat16* p, const float* v) {
  uint4 w;
  uint32_t* u = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    u[i] = *reinterpret_cast<uint32_t*>(&h);
  }
  *reinterpret_cast<uint4*>(p) = w;
}

struct Smem {
  uint8_t* w;
  uint8_t* a;
  uint64_t* full;
  uint64_t* empty;
  uint64_t* wbar;
  uint64_t* tfull;
  uint64_t* tempty;
  uint32_t* tmem_slot;
};

__device__ __forceinline__ Smem carve(uint8_t* raw) {
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  Smem m;
  m.w = s;
  m.a = s + 128 * 1024;
  uint64_t* bars = reinterpret_cast<uint64_t*>(m.a + kStages * kTileA);
  m.full = bars;
  m.empty = bars + kStages;
  m.wbar = bars + 2 * kStages;
  m.tfull = m.wbar + 1;
  m.tempty = m.tfull + 1;
  m.tmem_slot = reinterpret_cast<uint32_t*>(m.tempty + 1);
  return m;
}

__device__ __forceinline__ void setup(const Smem& m, uint32_t ncols) {
  const uint32_t warp = warp_id(), lane = lane_id();
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&m.full[s], 1);
      mbar_init(&m.empty[s], 1);
    }
    mbar_init(m.wbar, 1);
    mbar_init(m.tfull, 1);
    mbar_init(m.tempty, 128);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(m.tmem_slot, ncols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
}

__device__ __forceinline__ void wait_group(const uint32_t* ctr, uint32_t target) {
  while (ld_acquire_gpu(ctr) < target) {
  }
  fence_proxy_async_global();
}

// signal: all 128 epilogue threads finished their global writes for this step
__device__ __forceinline__ void epi_signal(uint32_t* ctr) {
  fence_proxy_async_global();
  named_bar_sync(1, 128);
  if (threadIdx.x == kEpiWarp0 * 32) {
    __threadfence();
    red_release_gpu_add(ctr, 1u);
  }
}

// ============================================================================
__global__ void __launch_bounds__(kThreads, 1) lstm_fwd_kernel(const __grid_constant__ LstmParams P) {
  extern __shared__ uint8_t smem_raw[];
  Smem m = carve(smem_raw);
  const uint32_t warp = warp_id(), lane = lane_id();
  const int n_ublk = kH / kUnits;  // 16
  const int ublk = blockIdx.x % n_ublk;
  const int btile = (blockIdx.x / n_ublk) % P.n_btile;
  const int dir = blockIdx.x / (n_ublk * P.n_btile);
  uint32_t* ctr = P.counters + dir * P.n_btile + btile;
  const int T = P.T, B = P.B;
  const int brow0 = P.b0 + btile * 128;  // first batch row of this tile

  setup(m, 128);
  const uint32_t tmem = *m.tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      tma_prefetch_desc(&P.tmA);
      tma_prefetch_desc(&P.tmW);
      // resident W_hh slice: rows dir*2048 + ublk*128 .. +128, K = 512
      mbar_arrive_expect_tx(m.wbar, kFwdWBytes);
      for (int kb = 0; kb < kH / 64; ++kb)
        tma_load_2d(m.w + kb * kRows * 128, &P.tmW, m.wbar, kb * 64, dir * 4 * kH + ublk * kRows);
      int stage = 0;
      uint32_t phase = 0;
      for (int s = 0; s < T; ++s) {
        const int t = dir == 0 ? s : T - 1 - s;
        const int tprev = dir == 0 ? t - 1 : t + 1;  // -1 / T hit the zero pads
        if (s > 0) wait_group(ctr, (uint32_t)(n_ublk * s));
        const int arow = (tprev + 1) * B + brow0;
        for (int kb = 0; kb < kH / 64; ++kb) {
          mbar_wait(&m.empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&m.full[stage], kTileA);
          tma_load_2d(m.a + stage * kTileA, &P.tmA, &m.full[stage], dir * kH + kb * 64, arow);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    mbar_wait(m.wbar, 0);
    const uint32_t idesc = idesc_bf16_f32(128, kRows, 0, 0);
    const uint32_t wbase = smem_u32(m.w);
    int stage = 0;
    uint32_t phase = 0;
    for (int s = 0; s < T; ++s) {
      mbar_wait(m.tempty, (s & 1) ^ 1);
      tc_fence_after();
      for (int kb = 0; kb < kH / 64; ++kb) {
        mbar_wait(&m.full[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t abase = smem_u32(m.a + stage * kTileA);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            uint64_t ad = smem_desc_sw128(abase + k * 32, 16, 1024);
            uint64_t bd = smem_desc_sw128(wbase + kb * kRows * 128 + k * 32, 16, 1024);
            mma_bf16_ss(tmem, ad, bd, idesc, (kb | k) != 0);
          }
          mma_commit(&m.empty[stage]);
          if (kb == kH / 64 - 1) mma_commit(m.tfull);
        }
        __syncwarp();
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp >= kEpiWarp0) {
    const uint32_t q = warp - kEpiWarp0;
    const int r = q * 32 + lane;
    const int b = brow0 + r;
    const bool ok = (r + btile * 128 < P.nb) && b < B;
    const uint32_t trow = tmem + ((q * 32) << 16);
    float creg[kUnits];
#pragma unroll
    for (int u = 0; u < kUnits; ++u) creg[u] = 0.f;
    for (int s = 0; s < T; ++s) {
      const int t = dir == 0 ? s : T - 1 - s;
      const size_t n = (size_t)t * B + b;
      mbar_wait(m.tfull, s & 1);
      tc_fence_after();
      __nv_bfloat16* grow = P.gates + n * (8 * kH) + dir * 4 * kH + ublk * kRows;
      float* crow = P.cstate + n * (2 * kH) + dir * kH + ublk * kUnits;
      __nv_bfloat16* hrow = P.y + ((size_t)(t + 1) * B + b) * (2 * kH) + dir * kH + ublk * kUnits;
#pragma unroll
      for (int c = 0; c < kRows; c += 32) {
        float v[32];
        tmem_ld16(trow + c, v);
        tmem_ld16(trow + c + 16, v + 16);
        tmem_ld_wait();
        if (ok) {
          float gi[32];
#pragma unroll
          for (int j = 0; j < 32; j += 8) load_bf16x8(grow + c + j, gi + j);
          float act[32], hv[8], cv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            float ai = v[4 * u + 0] + gi[4 * u + 0];
            float af = v[4 * u + 1] + gi[4 * u + 1];
            float ag = v[4 * u + 2] + gi[4 * u + 2];
            float ao = v[4 * u + 3] + gi[4 * u + 3];
            float ig = sigmoidf_(ai), fg = sigmoidf_(af), gg = tanhf_(ag), og = sigmoidf_(ao);
            const int uu = c / 4 + u;
            float cn = fg * creg[uu] + ig * gg;
            creg[uu] = cn;
            cv[u] = cn;
            hv[u] = og * tanhf_(cn);
            act[4 * u + 0] = ig;
            act[4 * u + 1] = fg;
            act[4 * u + 2] = gg;
            act[4 * u + 3] = og;
          }
#pragma unroll
          for (int j = 0; j < 32; j += 8) store_bf16x8(grow + c + j, act + j);
          float4* c4 = reinterpret_cast<float4*>(crow + c / 4);
          c4[0] = make_float4(cv[0], cv[1], cv[2], cv[3]);
          c4[1] = make_float4(cv[4], cv[5], cv[6], cv[7]);
          store_bf16x8(hrow + c / 4, hv);
        }
      }
      tc_fence_before();
      mbar_arrive(m.tempty);
      epi_signal(ctr);
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 128);
}

// ============================================================================
__global__ void __launch_bounds__(kThreads, 1) lstm_bwd_kernel(const __grid_constant__ LstmParams P) {
  extern __shared__ uint8_t smem_raw[];
  Smem m = carve(smem_raw);
  const uint32_t warp = warp_id(), lane = lane_id();
  const int n_ublk = kH / kUnits;
  const int ublk = blockIdx.x % n_ublk;
  const int btile = (blockIdx.x / n_ublk) % P.n_btile;
  const int dir = blockIdx.x / (n_ublk * P.n_btile);
  uint32_t* ctr = P.counters + dir * P.n_btile + btile;
  const int T = P.T, B = P.B;
  const int brow0 = P.b0 + btile * 128;
  constexpr int kKB = 4 * kH / 64;  // 32 k-blocks over the direction's 2048 gate rows

  setup(m, 32);
  const uint32_t tmem = *m.tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      tma_prefetch_desc(&P.tmA);
      tma_prefetch_desc(&P.tmW);
      // resident W_hh^T slice: rows dir*512 + ublk*32 .. +32, K = 2048
      mbar_arrive_expect_tx(m.wbar, kBwdWBytes);
      for (int kb = 0; kb < kKB; ++kb)
        tma_load_2d(m.w + kb * kUnits * 128, &P.tmW, m.wbar, kb * 64, dir * kH + ublk * kUnits);
      int stage = 0;
      uint32_t phase = 0;
      for (int s = 1; s < T; ++s) {
        const int t = dir == 0 ? T - 1 - s : s;
        const int tprev = dir == 0 ? t + 1 : t - 1;  // previously processed step
        wait_group(ctr, (uint32_t)(n_ublk * s));
        const int arow = tprev * B + brow0;
        for (int kb = 0; kb < kKB; ++kb) {
          mbar_wait(&m.empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&m.full[stage], kTileA);
          tma_load_2d(m.a + stage * kTileA, &P.tmA, &m.full[stage], dir * 4 * kH + kb * 64, arow);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    mbar_wait(m.wbar, 0);
    const uint32_t idesc = idesc_bf16_f32(128, kUnits, 0, 0);
    const uint32_t wbase = smem_u32(m.w);
    int stage = 0;
    uint32_t phase = 0;
    for (int s = 1; s < T; ++s) {
      mbar_wait(m.tempty, ((s - 1) & 1) ^ 1);
      tc_fence_after();
      for (int kb = 0; kb < kKB; ++kb) {
        mbar_wait(&m.full[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t abase = smem_u32(m.a + stage * kTileA);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            uint64_t ad = smem_desc_sw128(abase + k * 32, 16, 1024);
            uint64_t bd = smem_desc_sw128(wbase + kb * kUnits * 128 + k * 32, 16, 1024);
            mma_bf16_ss(tmem, ad, bd, idesc, (kb | k) != 0);
          }
          mma_commit(&m.empty[stage]);
          if (kb == kKB - 1) mma_commit(m.tfull);
        }
        __syncwarp();
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp >= kEpiWarp0) {
    const uint32_t q = warp - kEpiWarp0;
    const int r = q * 32 + lane;
    const int b = brow0 + r;
    const bool ok = (r + btile * 128 < P.nb) && b < B;
    const uint32_t trow = tmem + ((q * 32) << 16);
    float dcc[kUnits];
#pragma unroll
    for (int u = 0; u < kUnits; ++u) dcc[u] = 0.f;
    for (int s = 0; s < T; ++s) {
      const int t = dir == 0 ? T - 1 - s : s;
      const int tc = dir == 0 ? t - 1 : t + 1;  // forward-order predecessor (c_prev)
      const bool has_cprev = tc >= 0 && tc < T;
      const size_t n = (size_t)t * B + b;
      if (s > 0) {
        mbar_wait(m.tfull, (s - 1) & 1);
        tc_fence_after();
      }
      const __nv_bfloat16* arow = P.gates + n * (8 * kH) + dir * 4 * kH + ublk * kRows;
      const float* crow = P.cstate + n * (2 * kH) + dir * kH + ublk * kUnits;
      const float* cprow = P.cstate + ((size_t)tc * B + b) * (2 * kH) + dir * kH + ublk * kUnits;
      const __nv_bfloat16* dyrow = P.dy + n * (2 * kH) + dir * kH + ublk * kUnits;
      __nv_bfloat16* dgrow = P.dg + n * (8 * kH) + dir * 4 * kH + ublk * kRows;
#pragma unroll
      for (int c = 0; c < kUnits; c += 16) {
        float dh[16];
        if (s > 0) {
          tmem_ld16(trow + c, dh);
          tmem_ld_wait();
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) dh[i] = 0.f;
        }
        if (ok) {
          float dyv[16];
          load_bf16x8(dyrow + c, dyv);
          load_bf16x8(dyrow + c + 8, dyv + 8);
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            float act[32];
#pragma unroll
            for (int j = 0; j < 32; j += 8) load_bf16x8(arow + 4 * (c + 8 * half) + j, act + j);
            float cc[8], cp[8];
            const float4* c4 = reinterpret_cast<const float4*>(crow + c + 8 * half);
            float4 x0 = c4[0], x1 = c4[1];
            cc[0] = x0.x; cc[1] = x0.y; cc[2] = x0.z; cc[3] = x0.w;
            cc[4] = x1.x; cc[5] = x1.y; cc[6] = x1.z; cc[7] = x1.w;
            if (has_cprev) {
              const float4* p4 = reinterpret_cast<const float4*>(cprow + c + 8 * half);
              float4 y0 = p4[0], y1 = p4[1];
              cp[0] = y0.x; cp[1] = y0.y; cp[2] = y0.z; cp[3] = y0.w;
              cp[4] = y1.x; cp[5] = y1.y; cp[6] = y1.z; cp[7] = y1.w;
            } else {
#pragma unroll
              for (int u = 0; u < 8; ++u) cp[u] = 0.f;
            }
            float dgv[32];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int uu = c + 8 * half + u;
              const float ig = act[4 * u + 0], fg = act[4 * u + 1], gg = act[4 * u + 2], og = act[4 * u + 3];
              const float dht = dh[8 * half + u] + dyv[8 * half + u];
              const float tcn = tanhf_(cc[u]);
              const float dct = dht * og * (1.f - tcn * tcn) + dcc[uu];
              dgv[4 * u + 0] = dct * gg * ig * (1.f - ig);
              dgv[4 * u + 1] = dct * cp[u] * fg * (1.f - fg);
              dgv[4 * u + 2] = dct * ig * (1.f - gg * gg);
              dgv[4 * u + 3] = dht * tcn * og * (1.f - og);
              dcc[uu] = dct * fg;
            }
#pragma unroll
            for (int j = 0; j < 32; j += 8) store_bf16x8(dgrow + 4 * (c + 8 * half) + j, dgv + j);
          }
        }
      }
      if (s > 0) {
        tc_fence_before();
        mbar_arrive(m.tempty);
      }
      epi_signal(ctr);
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 32);
}

}  // namespace

static int launch_coop(const void* fn, int grid, const LstmParams& P, cudaStream_t stream) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* args[] = {const_cast<LstmParams*>(&P)};
  DS_CUDA_TRY(cudaLaunchKernelExC(&cfg, fn, args));
  return DS_OK;
}

static int lstm_run(bool fwd, const LstmLayerArgs& a, cudaStream_t stream) {
  static bool attr_set = false;
  if (!attr_set) {
    DS_CUDA_TRY(cudaFuncSetAttribute(lstm_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes));
    DS_CUDA_TRY(cudaFuncSetAttribute(lstm_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes));
    attr_set = true;
  }
  const int B = a.B, T = a.T;
  const int max_tiles = num_sms() / (2 * (kH / kUnits));  // co-resident tiles per launch
  if (max_tiles < 1) return fail_arg("device too small for the recurrent kernel");
  LstmParams P;
  memset(&P, 0, sizeof(P));
  int rc;
  if (fwd) {
    rc = make_tmap_2d(&P.tmA, a.y_full, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2 * kH, (uint64_t)(T + 2) * B,
                      2 * kH * 2, 64, 128);
    if (rc) return rc;
    rc = make_tmap_2d(&P.tmW, a.w, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, kH, 8 * kH, kH * 2, 64, kRows);
    if (rc) return rc;
  } else {
    rc = make_tmap_2d(&P.tmA, a.dg, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 8 * kH, (uint64_t)T * B, 8 * kH * 2, 64, 128);
    if (rc) return rc;
    rc = make_tmap_2d(&P.tmW, a.w, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4 * kH, 2 * kH, 4 * kH * 2, 64, kUnits);
    if (rc) return rc;
  }
  P.gates = a.gates;
  P.cstate = a.cstate;
  P.y = a.y_full;
  P.dy = a.dy;
  P.dg = a.dg;
  P.B = B;
  P.T = T;
  const int chunk_rows = max_tiles * 128;
  for (int b0 = 0; b0 < B; b0 += chunk_rows) {
    const int nb = (B - b0) < chunk_rows ? (B - b0) : chunk_rows;
    P.b0 = b0;
    P.nb = nb;
    P.n_btile = (nb + 127) / 128;
    P.counters = a.counters + (b0 / 128) * 2;
    DS_CUDA_TRY(cudaMemsetAsync(P.counters, 0, sizeof(uint32_t) * 2 * P.n_btile, stream));
    const int grid = 2 * (kH / kUnits) * P.n_btile;
    rc = launch_coop(fwd ? (const void*)lstm_fwd_kernel : (const void*)lstm_bwd_kernel, grid, P, stream);
    if (rc) return rc;
  }
  return DS_OK;
}

int lstm_forward(const LstmLayerArgs& a, cudaStream_t stream) { return lstm_run(true, a, stream); }
int lstm_backward(const LstmLayerArgs& a, cudaStream_t stream) { return lstm_run(false, a, stream); }

}  // namespace ds
