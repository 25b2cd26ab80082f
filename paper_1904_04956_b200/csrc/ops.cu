// ops.cu — the HBM-bound kernels of the step: minibatch gather (K1), the
// weight snapshot / operand cast (K2), momentum SGD fused with the snapshot
// (K9, /root/reference/pkg/src/distsgd/optim.py:109-121), the ADPSGD pairwise
// mix (K10, engines/adpsgd.py:36-43), the canonical-order ring-allreduce
// reduce fused with /lambda and SGD (K11, collective.py:122-163 +
// engines/ssgd.py:85-87), column sums for bias gradients and the
// soft-max/cross-entropy combine.
#include <cmath>

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
                              int64_t n_seq, int* __restrict__ flag) {
  constexpr int kVec = kInPad * 2 / 16;  // 34
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
// column sums of a bf16 [rows, ld] matrix, deterministic two-stage.
constexpr int kColSplit = 32;  // minimum split count (scratch is sized for 32 x the widest matrix)
inline int colsum_splits(int ncols) {
  const int cb = (ncols + 255) / 256;
  int sp = 1024 / cb;
  sp = sp < kColSplit ? kColSplit : sp;
  const long long cap = (long long)kColSplit * (ncols > kGates2 ? ncols : kGates2) / ncols;
  return (int)(sp > cap ? cap : sp);
}
__global__ void colsum_partial_kernel(const __nv_bfloat16* __restrict__ x, int64_t rows, int ncols, int64_t ld,
                                      float* __restrict__ part) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  const int split = blockIdx.y;
  if (col >= ncols) return;
  const int64_t per = (rows + gridDim.y - 1) / gridDim.y;
  const int64_t r0 = split * per, r1 = min(rows, r0 + per);
  float s = 0.f;
  for (int64_t r = r0; r < r1; ++r) s += __bfloat162float(x[r * ld + col]);
  part[(int64_t)split * ncols + col] = s;
}
__global__ void colsum_final_kernel(const float* __restrict__ part, int ncols, int splits, float* __restrict__ out) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= ncols) return;
  float s = 0.f;
  for (int k = 0; k < splits; ++k) s += part[(int64_t)k * ncols + col];
  out[col] = s;
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
__global__ void splitk_bf16_kernel(const float* __restrict__ part, int S, int64_t n, __nv_bfloat16* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float s = part[i];
    for (int k = 1; k < S; ++k) s += part[(int64_t)k * n + i];
    out[i] = __float2bfloat16_rn(s);
  }
}

// --------------------------------------------------------------------------
// soft-max / CE combine: lse[m] = logsumexp over column-tile (max, sumexp)
// partials; per-block loss partials, then one ordered sum (deterministic).
constexpr int kCeRows = 32;  // rows per block (lane = row: coalesced stats reads)
constexpr int kCeGroups = 8;  // tile groups per block (warps)
__global__ void ce_rows_kernel(const float2* __restrict__ stats, int ntiles, int64_t ld, const float* __restrict__ tgt,
                               int M, float* __restrict__ lse, float* __restrict__ part) {
  __shared__ float smx[kCeGroups][kCeRows], ssum[kCeGroups][kCeRows];
  const int g = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = blockIdx.x * kCeRows + lane;
  float mx = -INFINITY, s = 0.f;
  if (m < M) {
    for (int j = g; j < ntiles; j += kCeGroups) {  // online combine of this group's tiles
      const float2 st = stats[j * ld + m];
      if (!(st.y > 0.f)) continue;  // fully masked column block
      if (st.x > mx) {
        s = s * __expf(mx - st.x) + st.y;
        mx = st.x;
      } else {
        s += st.y * __expf(st.x - mx);
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
}
__global__ void ce_sum_kernel(const float* __restrict__ part, int n, float* __restrict__ loss_sum, int* __restrict__ flag) {
  __shared__ float red[1024];
  float acc = 0.f;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += part[i];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *loss_sum = red[0];
    if (flag && !isfinite(red[0])) atomicOr(flag, 1);
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

__global__ void cast_kernel(const float* __restrict__ theta, int64_t n, __nv_bfloat16* __restrict__ snap) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    snap[i] = __float2bfloat16_rn(theta[i]);
}

// W_hh^T snapshot: out[l][d][u][r] = W_hh[l][d*2048 + r][u]  (32x32 smem tiles)
__global__ void whh_transpose_kernel(const float* __restrict__ theta, const int64_t* __restrict__ offs, int layers,
                                     __nv_bfloat16* __restrict__ out) {
  __shared__ float tile[32][33];
  const int l = blockIdx.z;
  const float* src = theta + offs[l];  // [4096][512]
  __nv_bfloat16* dst = out + (int64_t)l * kGates2 * kHidden;  // [2][512][2048]
  const int r0 = blockIdx.y * 32;  // gate row (both dirs, 0..4095)
  const int u0 = blockIdx.x * 32;  // unit
  for (int i = threadIdx.y; i < 32; i += blockDim.y) tile[i][threadIdx.x] = src[(int64_t)(r0 + i) * kHidden + u0 + threadIdx.x];
  __syncthreads();
  const int d = r0 / kGates, rr0 = r0 % kGates;
  for (int i = threadIdx.y; i < 32; i += blockDim.y)
    dst[((int64_t)d * kHidden + u0 + i) * kGates + rr0 + threadIdx.x] = __float2bfloat16_rn(tile[threadIdx.x][i]);
}

// layer-0 W_ih padded to kInPad columns (TMA needs a 16-byte row pitch)
__global__ void wih0_pad_kernel(const float* __restrict__ w, int din, __nv_bfloat16* __restrict__ out) {
  const int64_t total = (int64_t)kGates2 * kInPad;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / kInPad;
    const int c = (int)(i % kInPad);
    out[i] = __float2bfloat16_rn(c < din ? w[r * din + c] : 0.f);
  }
}

__global__ void copy_f32_kernel(const float* __restrict__ src, float* __restrict__ dst, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
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

__global__ void group_reduce_kernel(GroupPtrs p, int world, int rank, int64_t dim, int64_t chunk, int nchunks,
                                    float lr, float mu, int mode, float divisor) {
  for (int j = rank; j < nchunks; j += world) {
    const int64_t lo = min(dim, (int64_t)j * chunk), hi = min(dim, (int64_t)(j + 1) * chunk);
    const int owner = j % world;
    for (int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hi; i += (int64_t)gridDim.x * blockDim.x) {
      const float* const* src = mode == 0 ? p.g : p.theta;
      float s = src[owner][i];
      for (int k = 1; k < world; ++k) s = __fadd_rn(s, src[(owner + k) % world][i]);
      const float mean = __fdiv_rn(s, divisor);
      if (mode == 0) {
        for (int r = 0; r < world; ++r) {
          float vv = __fadd_rn(__fmul_rn(p.v[r][i], mu), mean);
          float w = __fsub_rn(p.theta[r][i], __fmul_rn(lr, vv));
          p.v[r][i] = vv;
          p.theta[r][i] = w;
          if (p.snap[r]) p.snap[r][i] = __float2bfloat16_rn(w);
        }
      } else {
        for (int r = 0; r < world; ++r) {
          p.theta[r][i] = mean;
          if (p.snap[r]) p.snap[r][i] = __float2bfloat16_rn(mean);
        }
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
              __nv_bfloat16* x0, int32_t* lab, int* flag, cudaStream_t s) {
  gather_kernel<<<ew_grid((int64_t)T * B * 34), kEW, 0, s>>>(idx, B, T, reinterpret_cast<const uint4*>(feats), labels,
                                                            reinterpret_cast<uint4*>(x0), lab, n_seq, flag);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int op_colsum(const __nv_bfloat16* x, int64_t rows, int ncols, int64_t ld, float* part, float* out, cudaStream_t s) {
  const int sp = colsum_splits(ncols);
  dim3 g1((ncols + 255) / 256, sp);
  colsum_partial_kernel<<<g1, 256, 0, s>>>(x, rows, ncols, ld, part);
  colsum_final_kernel<<<(ncols + 255) / 256, 256, 0, s>>>(part, ncols, sp, out);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}
int64_t op_colsum_scratch(int ncols) { return (int64_t)kColSplit * ncols; }

int op_splitk_bf16(const float* part, int S, int64_t n, __nv_bfloat16* out, cudaStream_t s) {
  splitk_bf16_kernel<<<ew_grid(n), kEW, 0, s>>>(part, S, n, out);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int op_rowsum(const float* part, int nrows, int ncols, float* out, cudaStream_t s) {
  rowsum_kernel<<<(ncols + 255) / 256, 256, 0, s>>>(part, nrows, ncols, out);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int op_ce_combine(const float2* stats, int ntiles, int64_t ld, const float* tgt, int M, float* lse, float* scratch,
                  float* loss_sum, int* flag, cudaStream_t s) {
  const int nblk = (M + kCeRows - 1) / kCeRows;
  ce_rows_kernel<<<nblk, kCeGroups * 32, 0, s>>>(stats, ntiles, ld, tgt, M, lse, scratch);
  ce_sum_kernel<<<1, 1024, 0, s>>>(scratch, nblk, loss_sum, flag);
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

int op_cast(const float* theta, int64_t n, __nv_bfloat16* snap, cudaStream_t s) {
  cast_kernel<<<ew_grid(n), kEW, 0, s>>>(theta, n, snap);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int op_snapshot_aux(const float* theta, const ModelLayout& L, const int64_t* d_whh_offs, __nv_bfloat16* whhT,
                    __nv_bfloat16* wih0pad, float* bias_snap, cudaStream_t s) {
  dim3 grid(kHidden / 32, kGates2 / 32, L.layers);
  whh_transpose_kernel<<<grid, dim3(32, 8), 0, s>>>(theta, d_whh_offs, L.layers, whhT);
  wih0_pad_kernel<<<ew_grid((int64_t)kGates2 * kInPad), kEW, 0, s>>>(theta + L.off_wih[0], L.input_dim, wih0pad);
  // bias snapshot: [layers][4096] then b_b, b_o
  for (int l = 0; l < L.layers; ++l)
    copy_f32_kernel<<<ew_grid(kGates2), kEW, 0, s>>>(theta + L.off_b[l], bias_snap + (int64_t)l * kGates2, kGates2);
  copy_f32_kernel<<<ew_grid(L.bottleneck), kEW, 0, s>>>(theta + L.off_bb, bias_snap + (int64_t)L.layers * kGates2,
                                                        L.bottleneck);
  copy_f32_kernel<<<ew_grid(L.classes), kEW, 0, s>>>(
      theta + L.off_bo, bias_snap + (int64_t)L.layers * kGates2 + L.bottleneck, L.classes);
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
  const int64_t chunk = (dim + nchunks - 1) / nchunks;
  group_reduce_kernel<<<ew_grid(chunk), kEW, 0, s>>>(p, world, rank, dim, chunk, nchunks, lr, mu, mode,
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
