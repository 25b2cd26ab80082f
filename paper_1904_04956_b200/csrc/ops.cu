// ops.cu — the HBM-bound kernels of the step: minibatch gather (K1), the
// weight snapshot / operand cast (K2), momentum SGD fused with the snapshot
// (K9, /root/reference/pkg/src/distsgd/optim.py:109-121), the ADPSGD pairwise
// mix (K10, engines/adpsgd.py:36-43), the canonical-order ring-allreduce
// reduce fused with /lambda and SGD (K11, collective.py:122-163 +
// engines/ssgd.py:85-87), column sums for bias gradients and the
// soft-max/cross-entropy combine.
#include <cmath>
#include <cstring>

#include "ds_internal.h"
#include "ds_ptx.cuh"
#include "layout.h"
#include "ops.h"

namespace ds {

namespace {

constexpr int kEW = 256;  // elementwise block size

// --------------------------------------------------------------------------
// K1: X0[t*B+b, :] = feats[idx[b], t, :]   (rows of kInPad bf16 = 34 x 16 B)
__global__ void gather_kernel(const int64_t* __restrict__ idx, int B, int T, const uint4* __restrict__ feats,
                              const int32_t* __restrict__ labels, uint4* __restrict__ x0, int32_t* __restrict__ lab,
                              int64_t n_seq, int* __restrict__ flag, uint32_t* __restrict__ epoch) {
  constexpr int kVec = kInPad * 2 / 16;  // 34
  if (epoch && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(epoch, 1u);  // new step (lstm_wait_started)
  const int64_t total = (int64_t)T * B * kVec;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / kVec;
    const int v = (int)(i % kVec);
    const int t = (int)(row / B), b = (int)(row % B);
    int64_t s = idx[b];
    if (s < 0 || s >= n_seq) {
      if (flag) atomicOr(flag, 2);
      s = 0;
    }
    x0[i] = feats[(s * T + t) * kVec + v];
    if (v == 0) lab[row] = labels[s * T + t];
  }
}

// --------------------------------------------------------------------------
// column sums of a bf16 [rows, ld] matrix, deterministic two-stage: block =
// 128 rows x 256 columns, thread = 8 columns (one 16-byte load per row) x
// every 8th row; the 8 row lanes are combined in smem in a fixed order.
constexpr int kColRows = 128;
__global__ void colsum_partial_kernel(const __nv_bfloat16* __restrict__ x, int64_t rows, int ncols, int64_t ld,
                                      float* __restrict__ part) {
  __shared__ float red[8][256 + 8];
  const int cg = threadIdx.x & 31, rl = threadIdx.x >> 5;  // 32 column groups of 8, 8 row lanes
  const int c0 = blockIdx.x * 256 + cg * 8;
  const int64_t r0 = (int64_t)blockIdx.y * kColRows;
  float acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.f;
  if (c0 < ncols) {
#pragma unroll 4
    for (int k = 0; k < kColRows / 8; ++k) {
      const int64_t r = r0 + rl + 8 * k;
      if (r < rows) {
        float f[8];
        const uint4 w = *reinterpret_cast<const uint4*>(x + r * ld + c0);
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 t = __bfloat1622float2(h[i]);
          f[2 * i] = t.x;
          f[2 * i + 1] = t.y;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] += f[i];
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) red[rl][cg * 8 + i] = acc[i];
  __syncthreads();
  const int c = threadIdx.x;  // 256 threads = 256 columns
  if (blockIdx.x * 256 + c < ncols) {
    float sum = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) sum += red[k][c];
    part[(int64_t)blockIdx.y * ncols + blockIdx.x * 256 + c] = sum;
  }
}

// out[c] = sum_r part[r][c], rows in order (deterministic)
__global__ void rowsum_kernel(const float* __restrict__ part, int nrows, int ncols, float* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncols) return;
  float s = 0.f;
  int r = 0;
  for (; r + 8 <= nrows; r += 8) {
    float v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = part[(int64_t)(r + k) * ncols + c];
#pragma unroll
    for (int k = 0; k < 8; ++k) s += v[k];
  }
  for (; r < nrows; ++r) s += part[(int64_t)r * ncols + c];
  out[c] = s;
}

// split-K finish: out(bf16)[m][n] = sum_s part[s][m][n] in split order
__global__ void splitk_bf16_kernel(const float* __restrict__ part, int S, int64_t n, __nv_bfloat16* __restrict__ out,
                                   const float* __restrict__ bias, int ncols) {
  if ((n & 3) == 0) {  // 16-byte loads, all S partials of a vector in flight at once
    const int64_t n4 = n >> 2;
    const float4* p4 = reinterpret_cast<const float4*>(part);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
      float4 v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (k < S) v[k] = __ldg(p4 + (int64_t)k * n4 + i);
      float4 a = v[0];
#pragma unroll
      for (int k = 1; k < 8; ++k)
        if (k < S) {
          a.x += v[k].x;
          a.y += v[k].y;
          a.z += v[k].z;
          a.w += v[k].w;
        }
      for (int k = 8; k < S; ++k) {  // beyond 8 splits (not used by the step)
        const float4 b = __ldg(p4 + (int64_t)k * n4 + i);
        a.x += b.x;
        a.y += b.y;
        a.z += b.z;
        a.w += b.w;
      }
      if (bias) {  // + bias[column] after the split sum (ncols % 4 == 0)
        const float4 b = __ldg(reinterpret_cast<const float4*>(bias + (i * 4) % ncols));
        a.x += b.x;
        a.y += b.y;
        a.z += b.z;
        a.w += b.w;
      }
      __nv_bfloat162 lo = __floats2bfloat162_rn(a.x, a.y), hi = __floats2bfloat162_rn(a.z, a.w);
      uint2 w;
      w.x = *reinterpret_cast<uint32_t*>(&lo);
      w.y = *reinterpret_cast<uint32_t*>(&hi);
      reinterpret_cast<uint2*>(out)[i] = w;
    }
    return;
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float s = part[i];
    for (int k = 1; k < S; ++k) s += part[(int64_t)k * n + i];
    if (bias) s += bias[i % ncols];
    out[i] = __float2bfloat16_rn(s);
  }
}

// split-K finish: out(f32)[i] = sum_s part[s][i] in split order
__global__ void splitk_f32_kernel(const float* __restrict__ part, int S, int64_t n, float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float s = part[i];
    for (int k = 1; k < S; ++k) s += part[(int64_t)k * n + i];
    out[i] = s;
  }
}

// --------------------------------------------------------------------------
// soft-max / CE combine: lse[m] = logsumexp over column-tile (max, sumexp)
// partials; per-block loss partials, then one ordered sum (deterministic).
constexpr int kCeRows = 32;   // rows per block (lane = row: coalesced stats reads)
constexpr int kCeGroups = 16;  // tile groups per block (warps)
__global__ void ce_rows_kernel(const float2* __restrict__ stats, int ntiles, int64_t ld, const float* __restrict__ tgt,
                               int M, float* __restrict__ lse, float* __restrict__ part, unsigned* __restrict__ ticket,
                               float* __restrict__ loss_sum, int* __restrict__ flag) {
  __shared__ float smx[kCeGroups][kCeRows], ssum[kCeGroups][kCeRows];
  const int g = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = blockIdx.x * kCeRows + lane;
  float mx = -INFINITY, s = 0.f;
  if (m < M) {
    for (int j0 = g; j0 < ntiles; j0 += 8 * kCeGroups) {  // online combine, eight loads in flight
      float2 st[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = j0 + u * kCeGroups;
        st[u] = j < ntiles ? stats[j * ld + m] : make_float2(-INFINITY, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (!(st[u].y > 0.f)) continue;  // fully masked column block / past the end
        if (st[u].x > mx) {
          s = s * __expf(mx - st[u].x) + st[u].y;
          mx = st[u].x;
        } else {
          s += st[u].y * __expf(st[u].x - mx);
        }
      }
    }
  }
  smx[g][lane] = mx;
  ssum[g][lane] = s;
  __syncthreads();
  if (g == 0) {
    float loss = 0.f;
    if (m < M) {
      float M2 = -INFINITY;
      for (int k = 0; k < kCeGroups; ++k) M2 = fmaxf(M2, smx[k][lane]);
      float S = 0.f;
      for (int k = 0; k < kCeGroups; ++k)
        if (ssum[k][lane] > 0.f) S += ssum[k][lane] * __expf(smx[k][lane] - M2);
      const float l = M2 + __logf(S);
      lse[m] = l;
      loss = l - tgt[m];
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) loss += __shfl_xor_sync(0xffffffffu, loss, off);
    if (lane == 0) part[blockIdx.x] = loss;
  }
  // the last block to finish sums the block partials in index order (deterministic) and
  // re-arms the ticket: no separate reduction launch
  __shared__ bool last;
  __shared__ float red[kCeGroups * 32];
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  float acc = 0.f;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) acc += __ldcg(part + i);
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *loss_sum = red[0];
    if (flag && !isfinite(red[0])) atomicOr(flag, 1);
    *ticket = 0u;
  }
}

// --------------------------------------------------------------------------
// K9 (+K2): v <- mu*v + g ; theta <- theta - lr*v ; snap <- bf16(theta).
// Rounding mirrors the reference order (optim.py:119-121): v*mu, +g, lr*v, -.
__global__ void sgd_kernel(float* __restrict__ theta, float* __restrict__ v, const float* __restrict__ g, float lr,
                           float mu, int64_t n, __nv_bfloat16* __restrict__ snap, int* __restrict__ flag) {
  const int64_t n4 = n / 4;
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 w = reinterpret_cast<float4*>(theta)[i];
    float4 vv = reinterpret_cast<float4*>(v)[i];
    const float4 gg = reinterpret_cast<const float4*>(g)[i];
    bad |= !(isfinite(gg.x) && isfinite(gg.y) && isfinite(gg.z) && isfinite(gg.w));
    vv.x = __fadd_rn(__fmul_rn(vv.x, mu), gg.x);
    vv.y = __fadd_rn(__fmul_rn(vv.y, mu), gg.y);
    vv.z = __fadd_rn(__fmul_rn(vv.z, mu), gg.z);
    vv.w = __fadd_rn(__fmul_rn(vv.w, mu), gg.w);
    w.x = __fsub_rn(w.x, __fmul_rn(lr, vv.x));
    w.y = __fsub_rn(w.y, __fmul_rn(lr, vv.y));
    w.z = __fsub_rn(w.z, __fmul_rn(lr, vv.z));
    w.w = __fsub_rn(w.w, __fmul_rn(lr, vv.w));
    reinterpret_cast<float4*>(theta)[i] = w;
    reinterpret_cast<float4*>(v)[i] = vv;
    if (snap) {
      __nv_bfloat162 a = __floats2bfloat162_rn(w.x, w.y), b = __floats2bfloat162_rn(w.z, w.w);
      uint2 pk;
      pk.x = *reinterpret_cast<uint32_t*>(&a);
      pk.y = *reinterpret_cast<uint32_t*>(&b);
      reinterpret_cast<uint2*>(snap)[i] = pk;
    }
  }
  for (int64_t i = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float gg = g[i];
    bad |= !isfinite(gg);
    float vv = __fadd_rn(__fmul_rn(v[i], mu), gg);
    float w = __fsub_rn(theta[i], __fmul_rn(lr, vv));
    v[i] = vv;
    theta[i] = w;
    if (snap) snap[i] = __float2bfloat16_rn(w);
  }
  if (bad && flag) atomicOr(flag, 1);
}

// K9 for the fused training step: lr read from device memory (the captured
// step graph is reused while the schedule changes lr), two float4 per thread
// per iteration so a small grid (the SMs a recurrence leaves free) still
// keeps enough bytes in flight.  Same rounding order as sgd_kernel.
__device__ __forceinline__ void sgd_mirror4(const SgdMirror& m, int64_t i, float4 w) {
  if (m.wpad && i >= m.wbeg && i < m.wbeg + m.wcnt) {  // 4 consecutive columns of one W_ih0 row
    const int64_t r = (i - m.wbeg) / m.din, c = (i - m.wbeg) % m.din;
    __nv_bfloat162 a = __floats2bfloat162_rn(w.x, w.y), b = __floats2bfloat162_rn(w.z, w.w);
    uint2 pk;
    pk.x = *reinterpret_cast<uint32_t*>(&a);
    pk.y = *reinterpret_cast<uint32_t*>(&b);
    *reinterpret_cast<uint2*>(m.wpad + r * kInPad + c) = pk;
  }
#pragma unroll
  for (int k = 0; k < 3; ++k)
    if (m.fdst[k] && i >= m.fbeg[k] && i < m.fbeg[k] + m.fcnt[k])
      *reinterpret_cast<float4*>(m.fdst[k] + (i - m.fbeg[k])) =
          make_float4(w.x * m.fscale[k], w.y * m.fscale[k], w.z * m.fscale[k], w.w * m.fscale[k]);
}
__global__ void __launch_bounds__(1024) sgd_lr_kernel(float* __restrict__ theta, float* __restrict__ v, const float* __restrict__ g,
                              const float* __restrict__ lr_dev, float mu, int64_t n, __nv_bfloat16* __restrict__ snap,
                              int* __restrict__ flag, const SgdMirror mir, int use_mir) {
  const float lr = *lr_dev;
  const int64_t n4 = n / 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  bool bad = false;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < n4; i0 += 2 * stride) {
    float4 w[2], vv[2], gg[2];
    const int64_t idx[2] = {i0, i0 + stride};
#pragma unroll
    for (int u = 0; u < 2; ++u)
      if (idx[u] < n4) {
        w[u] = reinterpret_cast<float4*>(theta)[idx[u]];
        vv[u] = reinterpret_cast<float4*>(v)[idx[u]];
        gg[u] = reinterpret_cast<const float4*>(g)[idx[u]];
        if (use_mir && mir.add && idx[u] * 4 < mir.add_n) {  // second gradient part, sum stored back
          const float4 a = reinterpret_cast<const float4*>(mir.add)[idx[u]];
          gg[u].x += a.x;
          gg[u].y += a.y;
          gg[u].z += a.z;
          gg[u].w += a.w;
          reinterpret_cast<float4*>(const_cast<float*>(g))[idx[u]] = gg[u];
        }
      }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      if (idx[u] >= n4) continue;
      bad |= !(isfinite(gg[u].x) && isfinite(gg[u].y) && isfinite(gg[u].z) && isfinite(gg[u].w));
      vv[u].x = __fadd_rn(__fmul_rn(vv[u].x, mu), gg[u].x);
      vv[u].y = __fadd_rn(__fmul_rn(vv[u].y, mu), gg[u].y);
      vv[u].z = __fadd_rn(__fmul_rn(vv[u].z, mu), gg[u].z);
      vv[u].w = __fadd_rn(__fmul_rn(vv[u].w, mu), gg[u].w);
      w[u].x = __fsub_rn(w[u].x, __fmul_rn(lr, vv[u].x));
      w[u].y = __fsub_rn(w[u].y, __fmul_rn(lr, vv[u].y));
      w[u].z = __fsub_rn(w[u].z, __fmul_rn(lr, vv[u].z));
      w[u].w = __fsub_rn(w[u].w, __fmul_rn(lr, vv[u].w));
      reinterpret_cast<float4*>(theta)[idx[u]] = w[u];
      reinterpret_cast<float4*>(v)[idx[u]] = vv[u];
      if (snap) {
        __nv_bfloat162 a = __floats2bfloat162_rn(w[u].x, w[u].y), b = __floats2bfloat162_rn(w[u].z, w[u].w);
        uint2 pk;
        pk.x = *reinterpret_cast<uint32_t*>(&a);
        pk.y = *reinterpret_cast<uint32_t*>(&b);
        reinterpret_cast<uint2*>(snap)[idx[u]] = pk;
      }
      if (use_mir) sgd_mirror4(mir, idx[u] * 4, w[u]);
    }
  }
  for (int64_t i = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    float gv = g[i];
    bad |= !isfinite(gv);
    float vn = __fadd_rn(__fmul_rn(v[i], mu), gv);
    float w = __fsub_rn(theta[i], __fmul_rn(lr, vn));
    v[i] = vn;
    theta[i] = w;
    if (snap) snap[i] = __float2bfloat16_rn(w);
  }
  if (bad && flag) atomicOr(flag, 1);
}

__global__ void cast_kernel(const float* __restrict__ theta, int64_t n, __nv_bfloat16* __restrict__ snap) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    snap[i] = __float2bfloat16_rn(theta[i]);
}

// Operand-snapshot extras in one launch: layer-0 W_ih padded to kInPad
// columns (TMA needs a 16-byte row pitch) followed by the fp32 bias copies
// [layers][4096], b_b, b_o.  (W_hh is read straight from the bf16 snapshot by
// both recurrent kernels: no transposed copy.)
struct AuxOffs {
  int64_t off_b[kMaxLayers];
  int64_t off_wih0, off_bb, off_bo;
  int layers, din, bott, classes;
};
__global__ void snapshot_aux_kernel(const float* __restrict__ theta, AuxOffs o, __nv_bfloat16* __restrict__ wpad,
                                    float* __restrict__ bias) {
  const int64_t npad = (int64_t)kGates2 * kInPad;
  const int64_t nb = (int64_t)o.layers * kGates2;
  const int64_t total = npad + nb + o.bott + 2 * (int64_t)o.classes;  // + b_o * log2(e) for the CE-stats pass
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < npad) {
      const int64_t r = i / kInPad;
      const int c = (int)(i % kInPad);
      wpad[i] = __float2bfloat16_rn(c < o.din ? theta[o.off_wih0 + r * o.din + c] : 0.f);
      continue;
    }
    const int64_t j = i - npad;
    int64_t src;
    if (j < nb)
      src = o.off_b[j / kGates2] + j % kGates2;
    else if (j < nb + o.bott)
      src = o.off_bb + (j - nb);
    else if (j < nb + o.bott + o.classes)
      src = o.off_bo + (j - nb - o.bott);
    else {
      bias[j] = theta[o.off_bo + (j - nb - o.bott - o.classes)] * 1.4426950408889634f;
      continue;
    }
    bias[j] = theta[src];
  }
}

// --------------------------------------------------------------------------
// K10: mean = (a + b) / 2 stored to both sides (identical value, exact pair sum)
__global__ void mix_kernel(float* __restrict__ a, float* __restrict__ b, int64_t n) {
  const int64_t n4 = n / 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 x = reinterpret_cast<float4*>(a)[i];
    const float4 y = reinterpret_cast<float4*>(b)[i];
    x.x = __fmul_rn(__fadd_rn(x.x, y.x), 0.5f);
    x.y = __fmul_rn(__fadd_rn(x.y, y.y), 0.5f);
    x.z = __fmul_rn(__fadd_rn(x.z, y.z), 0.5f);
    x.w = __fmul_rn(__fadd_rn(x.w, y.w), 0.5f);
    reinterpret_cast<float4*>(a)[i] = x;
    reinterpret_cast<float4*>(b)[i] = x;
  }
  for (int64_t i = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float m = __fmul_rn(__fadd_rn(a[i], b[i]), 0.5f);
    a[i] = m;
    b[i] = m;
  }
}

// --------------------------------------------------------------------------
// K11/K12 on the chunks owned by `rank`: sum over the group in the canonical
// ring order of collective.py:133-145 (owner, owner+1, ..., owner-1), then
//   mode 0 (SSGD)  : g_mean = sum / world; per-member momentum SGD; snapshot
//   mode 1 (AVG)   : every member's theta <- sum / world (consensus / hybrid)
// and store the result into every member's buffers (peer stores).
struct GroupPtrs {
  float* g[kMaxGroup];
  float* theta[kMaxGroup];
  float* v[kMaxGroup];
  __nv_bfloat16* snap[kMaxGroup];
};

__device__ __forceinline__ float4 f4_step(float4 v, float4 gm, float4& w, float lr, float mu) {
  v.x = __fadd_rn(__fmul_rn(v.x, mu), gm.x);
  v.y = __fadd_rn(__fmul_rn(v.y, mu), gm.y);
  v.z = __fadd_rn(__fmul_rn(v.z, mu), gm.z);
  v.w = __fadd_rn(__fmul_rn(v.w, mu), gm.w);
  w.x = __fsub_rn(w.x, __fmul_rn(lr, v.x));
  w.y = __fsub_rn(w.y, __fmul_rn(lr, v.y));
  w.z = __fsub_rn(w.z, __fmul_rn(lr, v.z));
  w.w = __fsub_rn(w.w, __fmul_rn(lr, v.w));
  return v;
}
__device__ __forceinline__ uint2 f4_bf16(float4 w) {
  __nv_bfloat162 a = __floats2bfloat162_rn(w.x, w.y), b = __floats2bfloat162_rn(w.z, w.w);
  uint2 pk;
  pk.x = *reinterpret_cast<uint32_t*>(&a);
  pk.y = *reinterpret_cast<uint32_t*>(&b);
  return pk;
}

// float4 vectors inside each owned chunk, scalar at its ragged edges
__global__ void group_reduce_kernel(GroupPtrs p, int world, int rank, int64_t dim, int64_t chunk, int nchunks,
                                    float lr, float mu, int mode, float divisor) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
  const float* const* src = mode == 0 ? p.g : p.theta;
  for (int j = rank; j < nchunks; j += world) {
    const int64_t lo = min(dim, (int64_t)j * chunk), hi = min(dim, (int64_t)(j + 1) * chunk);
    const int owner = j % world;
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
      const float4 mean = make_float4(__fdiv_rn(sum.x, divisor), __fdiv_rn(sum.y, divisor), __fdiv_rn(sum.z, divisor),
                                      __fdiv_rn(sum.w, divisor));
      for (int r = 0; r < world; ++r) {
        float4 w = mean;
        if (mode == 0) {
          w = reinterpret_cast<const float4*>(p.theta[r])[i4];
          reinterpret_cast<float4*>(p.v[r])[i4] = f4_step(reinterpret_cast<const float4*>(p.v[r])[i4], mean, w, lr, mu);
        }
        reinterpret_cast<float4*>(p.theta[r])[i4] = w;
        if (p.snap[r]) reinterpret_cast<uint2*>(p.snap[r])[i4] = f4_bf16(w);
      }
    }
    // a chunk with no aligned float4 (lo4 > hi4) is all edge: one scalar range
    const int64_t e0 = lo, e1 = lo4 > hi4 ? hi : min(hi, lo4 * 4), f0 = lo4 > hi4 ? hi : max(lo, hi4 * 4), f1 = hi;
    for (int64_t t = tid; t < (e1 - e0) + (f1 - f0); t += nth) {
      const int64_t i = t < (e1 - e0) ? e0 + t : f0 + (t - (e1 - e0));
      float s = src[owner][i];
      for (int k = 1; k < world; ++k) s = __fadd_rn(s, src[(owner + k) % world][i]);
      const float mean = __fdiv_rn(s, divisor);
      for (int r = 0; r < world; ++r) {
        float w = mean;
        if (mode == 0) {
          const float vv = __fadd_rn(__fmul_rn(p.v[r][i], mu), mean);
          w = __fsub_rn(p.theta[r][i], __fmul_rn(lr, vv));
          p.v[r][i] = vv;
        }
        p.theta[r][i] = w;
        if (p.snap[r]) p.snap[r][i] = __float2bfloat16_rn(w);
      }
    }
  }
}

// consensus: out = (((x0 + x1) + x2) + ...) / n, members in id order
// (np.mean(np.stack(...), axis=0) of engines/adpsgd.py:293-295, in fp32)
__global__ void average_kernel(GroupPtrs p, int n, int64_t dim, float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < dim; i += (int64_t)gridDim.x * blockDim.x) {
    float s = p.theta[0][i];
    for (int k = 1; k < n; ++k) s = __fadd_rn(s, p.theta[k][i]);
    out[i] = __fdiv_rn(s, (float)n);
  }
}

inline int ew_grid(int64_t n) {
  int64_t b = (n + kEW - 1) / kEW;
  int64_t cap = (int64_t)num_sms() * 8;
  return (int)(b < cap ? (b > 0 ? b : 1) : cap);
}

}  // namespace

int op_gather(const int64_t* idx, int B, int T, const __nv_bfloat16* feats, const int32_t* labels, int64_t n_seq,
              __nv_bfloat16* x0, int32_t* lab, int* flag, cudaStream_t s, uint32_t* epoch) {
  gather_kernel<<<ew_grid((int64_t)T * B * 34), kEW, 0, s>>>(idx, B, T, reinterpret_cast<const uint4*>(feats), labels,
                                                            reinterpret_cast<uint4*>(x0), lab, n_seq, flag, epoch);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int op_colsum(const __nv_bfloat16* x, int64_t rows, int ncols, int64_t ld, float* part, float* out, cudaStream_t s) {
  if ((ncols & 7) || (ld & 7)) return fail_arg("colsum: columns and pitch must be multiples of 8");
  const int sp = (int)((rows + kColRows - 1) / kColRows);
  dim3 g1((ncols + 255) / 256, sp);
  colsum_partial_kernel<<<g1, 256, 0, s>>>(x, rows, ncols, ld, part);
  DS_CUDA_TRY(cudaGetLastError());
  return op_rowsum(part, sp, ncols, out, s);
}
int64_t op_colsum_scratch(int64_t rows, int ncols) { return (rows + kColRows - 1) / kColRows * ncols; }

int op_splitk_f32(const float* part, int S, int64_t n, float* out, cudaStream_t s) {
  splitk_f32_kernel<<<ew_grid(n), kEW, 0, s>>>(part, S, n, out);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int op_splitk_bf16(const float* part, int S, int64_t n, __nv_bfloat16* out, cudaStream_t s, const float* bias,
                   int ncols) {
  if (bias && (ncols < 4 || ncols % 4 || n % ncols)) return fail_arg("splitk_bf16: bias needs whole rows of 4k columns");
  splitk_bf16_kernel<<<ew_grid(n), kEW, 0, s>>>(part, S, n, out, bias, ncols);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int op_rowsum(const float* part, int nrows, int ncols, float* out, cudaStream_t s) {
  rowsum_kernel<<<(ncols + 255) / 256, 256, 0, s>>>(part, nrows, ncols, out);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int op_ce_combine(const float2* stats, int ntiles, int64_t ld, const float* tgt, int M, float* lse, float* scratch,
                  unsigned* ticket, float* loss_sum, int* flag, cudaStream_t s) {
  const int nblk = (M + kCeRows - 1) / kCeRows;
  ce_rows_kernel<<<nblk, kCeGroups * 32, 0, s>>>(stats, ntiles, ld, tgt, M, lse, scratch, ticket, loss_sum, flag);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int op_sgd(float* theta, float* v, const float* g, float lr, float mu, int64_t n, __nv_bfloat16* snap, int* flag,
           cudaStream_t s) {
  if (((reinterpret_cast<uintptr_t>(theta) | reinterpret_cast<uintptr_t>(v) | reinterpret_cast<uintptr_t>(g)) & 15))
    return fail_arg("sgd: buffers must be 16-byte aligned");
  sgd_kernel<<<ew_grid(n / 4 + 1), kEW, 0, s>>>(theta, v, g, lr, mu, n, snap, flag);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int op_sgd_lr(float* theta, float* v, const float* g, const float* lr_dev, float mu, int64_t n, __nv_bfloat16* snap,
              int* flag, int max_blocks, cudaStream_t s, const SgdMirror* mir) {
  if (((reinterpret_cast<uintptr_t>(theta) | reinterpret_cast<uintptr_t>(v) | reinterpret_cast<uintptr_t>(g)) & 15))
    return fail_arg("sgd: buffers must be 16-byte aligned");
  if (mir) {  // the float4 path covers the mirrored ranges only when they are 4-aligned inside n / 4 * 4
    bool ok = !mir->wpad || (mir->din % 4 == 0 && mir->wbeg % 4 == 0 && mir->wbeg + mir->wcnt <= n / 4 * 4);
    ok = ok && (!mir->add || (mir->add_n % 4 == 0 && mir->add_n <= n / 4 * 4 &&
                              (reinterpret_cast<uintptr_t>(mir->add) & 15) == 0));
    for (int k = 0; k < 3; ++k)
      ok = ok && (!mir->fdst[k] || (mir->fbeg[k] % 4 == 0 && mir->fcnt[k] % 4 == 0 && mir->fbeg[k] + mir->fcnt[k] <= n / 4 * 4));
    if (!ok) return fail_arg("sgd mirror: ranges must be 4-aligned");
  }
  const int threads = max_blocks > 0 ? 1024 : kEW;
  int64_t blocks = (n / 8 + threads - 1) / threads;
  const int64_t cap = max_blocks > 0 ? max_blocks : (int64_t)num_sms() * 8;
  blocks = blocks < 1 ? 1 : (blocks > cap ? cap : blocks);
  sgd_lr_kernel<<<(int)blocks, threads, 0, s>>>(theta, v, g, lr_dev, mu, n, snap, flag, mir ? *mir : SgdMirror(),
                                                 mir ? 1 : 0);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int op_cast(const float* theta, int64_t n, __nv_bfloat16* snap, cudaStream_t s) {
  cast_kernel<<<ew_grid(n), kEW, 0, s>>>(theta, n, snap);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int op_snapshot_aux(const float* theta, const ModelLayout& L, __nv_bfloat16* wih0pad, float* bias_snap,
                    cudaStream_t s) {
  AuxOffs o;
  memset(&o, 0, sizeof(o));
  for (int l = 0; l < L.layers; ++l) o.off_b[l] = L.off_b[l];
  o.off_wih0 = L.off_wih[0];
  o.off_bb = L.off_bb;
  o.off_bo = L.off_bo;
  o.layers = L.layers;
  o.din = L.input_dim;
  o.bott = L.bottleneck;
  o.classes = L.classes;
  const int64_t total = (int64_t)kGates2 * kInPad + (int64_t)L.layers * kGates2 + L.bottleneck + 2 * (int64_t)L.classes;
  snapshot_aux_kernel<<<ew_grid(total), kEW, 0, s>>>(theta, o, wih0pad, bias_snap);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int op_mix(float* a, float* b, int64_t n, cudaStream_t s) {
  if (((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15))
    return fail_arg("mix: buffers must be 16-byte aligned");
  mix_kernel<<<ew_grid(n / 4 + 1), kEW, 0, s>>>(a, b, n);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int op_group_reduce(int world, int rank, float* const* g, float* const* theta, float* const* v, __nv_bfloat16* const* snap,
                    int64_t dim, int nchunks, float lr, float mu, int mode, float divisor, cudaStream_t s) {
  if (world < 1 || world > kMaxGroup) return fail_arg("group size out of range");
  if (nchunks < world) return fail_arg("chunk_count must be >= world");
  GroupPtrs p;
  memset(&p, 0, sizeof(p));
  for (int r = 0; r < world; ++r) {
    p.g[r] = g ? g[r] : nullptr;
    p.theta[r] = theta[r];
    p.v[r] = v ? v[r] : nullptr;
    p.snap[r] = snap ? snap[r] : nullptr;
  }
  if (mode == 0 && (!g || !v)) return fail_arg("SGD allreduce needs gradient and velocity buffers");
  for (int r = 0; r < world; ++r) {
    uintptr_t al = reinterpret_cast<uintptr_t>(p.theta[r]) | reinterpret_cast<uintptr_t>(p.g[r]) |
                   reinterpret_cast<uintptr_t>(p.v[r]) | (reinterpret_cast<uintptr_t>(p.snap[r]) & 7);
    if (al & 15) return fail_arg("group reduce: buffers must be 16-byte aligned");
  }
  const int64_t chunk = (dim + nchunks - 1) / nchunks;
  group_reduce_kernel<<<ew_grid(chunk / 4 + 1), kEW, 0, s>>>(p, world, rank, dim, chunk, nchunks, lr, mu, mode,
                                                     divisor > 0.f ? divisor : (float)world);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int op_average(int n, float* const* srcs, float* out, int64_t dim, cudaStream_t s) {
  if (n < 1 || n > kMaxGroup) return fail_arg("average: member count out of range");
  GroupPtrs p;
  memset(&p, 0, sizeof(p));
  for (int k = 0; k < n; ++k) p.theta[k] = srcs[k];
  average_kernel<<<ew_grid(dim), kEW, 0, s>>>(p, n, dim, out);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

}  // namespace ds
