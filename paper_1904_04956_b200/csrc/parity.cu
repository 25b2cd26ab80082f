// parity.cu — FP32-parity mode of the BLSTM training step: every dense
// product on the tcgen05 tensor cores in kind::tf32 with the 3xTF32 split
// (a*b ~= a_hi*b_hi + a_hi*b_lo + a_lo*b_hi, fp32 TMEM accumulation), all
// activations, cell state and soft-max in fp32 with accurate exp/tanh.
//
// Why 3xTF32 and not plain TF32: at BASELINE config 2 the gradient of the
// paper BLSTM is ill-conditioned — a 1e-3 relative weight
// perturbation moves it by ~3 % (tools/precision_study.py) — so single TF32
// operands (2^-11 rounding) already cost ~9e-3 relative gradient error
// against the float64 reference arithmetic (objectives.py:236-263), and BF16
// ~7e-2.  The split keeps ~21 mantissa bits per product, which holds the
// whole step within ~1e-5 of float64.
//
// This path exists for parity (the reference computes in
// float64: objectives.py:3-5, optim.py:109-121); the BF16 path in blstm.cu is
// the performance mode.  It is a straight sequence of launches (no graph):
// per layer an input-projection GEMM, then per time step one 2-problem
// recurrent GEMM (both directions) accumulating h_{t-1} W_hh^T into the gate
// pre-activations plus an fp32 cell kernel; the output layer materialises the
// fp32 logits (688 MB at N = 5376) and the backward mirrors it.  Operands of
// every GEMM are K-major fp32 hi/lo pairs written by their producer kernels
// (split / transpose-split), so one GEMM kernel serves every product.
#include <cmath>
#include <cstring>

#include "ds_internal.h"
#include "ds_ptx.cuh"
#include "layout.h"
#include "parity.h"

namespace ds {

namespace {

// ---------------------------------------------------------------------------
// 3xTF32 GEMM: out[m, n] (=|+=) scale * sum_k A[m, k] B[n, k] (+ bias[n]),
// A and B K-major fp32 given as (hi, lo) pairs.  One 128 x 128 tile per CTA.
constexpr int TBM = 128, TBN = 128, TBK = 32;  // TBK fp32 = 128-byte swizzled rows
constexpr int kT3Stages = 3;
constexpr int kT3Tile = 128 * TBK * 4;       // 16 KB
constexpr int kT3Stage = 4 * kT3Tile;        // A_hi, A_lo, B_hi, B_lo
constexpr int kT3Threads = 256;              // warp 0 TMA, 1 MMA, 2 TMEM, 4..7 epilogue
constexpr size_t kT3Smem = 1024 + (size_t)kT3Stages * kT3Stage + 256;

struct T3Problem {
  CUtensorMap a_hi, a_lo, b_hi, b_lo;
  int M, N, K, tiles_n, tiles;
  float* out;
  long long ldo;
  const float* bias;
  float scale;
  int accumulate;
};
struct T3Batch {
  T3Problem p[2];
  int nprob;
};

__host__ __device__ constexpr uint32_t idesc_tf32_f32(uint32_t M, uint32_t N) {
  return (1u << 4)            // D = f32
         | (2u << 7)          // A = tf32
         | (2u << 10)         // B = tf32
         | ((N >> 3) << 17)   // N
         | ((M >> 4) << 24);  // M (both operands K-major)
}

DS_DEV void mma_tf32_ss(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__global__ void __launch_bounds__(kT3Threads, 1) gemm3_kernel(const __grid_constant__ T3Batch batch) {
  const T3Problem& P = batch.p[blockIdx.y];
  if ((int)blockIdx.x >= P.tiles) return;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kT3Stages * kT3Stage);
  uint64_t* empty = full + kT3Stages;
  uint64_t* tfull = empty + kT3Stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
  const uint32_t warp = warp_id(), lane = lane_id();
  const int m0 = (blockIdx.x / P.tiles_n) * TBM, n0 = (blockIdx.x % P.tiles_n) * TBN;
  const int nkb = (P.K + TBK - 1) / TBK;

  if (warp == 1 && lane == 0) {
    for (int s = 0; s < kT3Stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, TBN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      for (int kb = 0; kb < nkb; ++kb) {
        const int stage = kb % kT3Stages;
        if (kb >= kT3Stages) mbar_wait(&empty[stage], ((kb / kT3Stages) - 1) & 1);
        uint8_t* st = smem + stage * kT3Stage;
        mbar_arrive_expect_tx(&full[stage], kT3Stage);
        const int k0 = kb * TBK;
        tma_load_2d(st, &P.a_hi, &full[stage], k0, m0);
        tma_load_2d(st + kT3Tile, &P.a_lo, &full[stage], k0, m0);
        tma_load_2d(st + 2 * kT3Tile, &P.b_hi, &full[stage], k0, n0);
        tma_load_2d(st + 3 * kT3Tile, &P.b_lo, &full[stage], k0, n0);
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = idesc_tf32_f32(TBM, TBN);
    for (int kb = 0; kb < nkb; ++kb) {
      const int stage = kb % kT3Stages;
      mbar_wait(&full[stage], (kb / kT3Stages) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t base = smem_u32(smem + stage * kT3Stage);
#pragma unroll
        for (int k = 0; k < TBK / 8; ++k) {  // K = 8 tf32 (32 bytes) per instruction
          const uint64_t ah = smem_desc_sw128(base + k * 32, 16, 1024);
          const uint64_t al = smem_desc_sw128(base + kT3Tile + k * 32, 16, 1024);
          const uint64_t bh = smem_desc_sw128(base + 2 * kT3Tile + k * 32, 16, 1024);
          const uint64_t bl = smem_desc_sw128(base + 3 * kT3Tile + k * 32, 16, 1024);
          mma_tf32_ss(tmem_base, al, bh, idesc, (kb | k) != 0);  // small terms first
          mma_tf32_ss(tmem_base, ah, bl, idesc, 1);
          mma_tf32_ss(tmem_base, ah, bh, idesc, 1);
        }
        mma_commit(&empty[stage]);
        if (kb == nkb - 1) mma_commit(tfull);
      }
      __syncwarp();
    }
  } else if (warp >= 4) {
    const uint32_t q = warp & 3;  // TMEM lane quadrant
    mbar_wait(tfull, 0);
    tc_fence_after();
    const int row = m0 + (int)(q * 32 + lane);
    float* orow = P.out + (size_t)row * P.ldo;
#pragma unroll 1
    for (int c = 0; c < TBN; c += 32) {
      float v[32];
      tmem_ld32(tmem_base + ((q * 32) << 16) + c, v);
      tmem_ld_wait();
      if (row >= P.M) continue;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int n = n0 + c + i;
        if (n < P.N) {
          float x = v[i] * P.scale;
          if (P.bias) x += P.bias[n];
          if (P.accumulate) x += orow[n];
          orow[n] = x;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem_base, TBN);
}

int t3_problem(T3Problem* p, const Split& A, long long lda, const Split& B, long long ldb, int M, int N, int K,
               float* out, long long ldo, const float* bias, int accumulate) {
  if (M <= 0 || N <= 0 || K <= 0) return fail_arg("gemm3: empty problem");
  memset(p, 0, sizeof(*p));
  int rc = make_tmap_2d(&p->a_hi, A.hi, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, K, M, (uint64_t)lda * 4, TBK, TBM);
  if (!rc) rc = make_tmap_2d(&p->a_lo, A.lo, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, K, M, (uint64_t)lda * 4, TBK, TBM);
  if (!rc) rc = make_tmap_2d(&p->b_hi, B.hi, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, K, N, (uint64_t)ldb * 4, TBK, TBN);
  if (!rc) rc = make_tmap_2d(&p->b_lo, B.lo, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, K, N, (uint64_t)ldb * 4, TBK, TBN);
  if (rc) return rc;
  p->M = M;
  p->N = N;
  p->K = K;
  p->tiles_n = (N + TBN - 1) / TBN;
  p->tiles = ((M + TBM - 1) / TBM) * p->tiles_n;
  p->out = out;
  p->ldo = ldo;
  p->bias = bias;
  p->scale = 1.f;
  p->accumulate = accumulate;
  return DS_OK;
}

int t3_launch(T3Batch* b, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    DS_CUDA_TRY(cudaFuncSetAttribute(gemm3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kT3Smem));
    attr = true;
  }
  int tiles = 0;
  for (int i = 0; i < b->nprob; ++i) tiles = b->p[i].tiles > tiles ? b->p[i].tiles : tiles;
  gemm3_kernel<<<dim3(tiles, b->nprob), kT3Threads, kT3Smem, s>>>(*b);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

// ---------------------------------------------------------------------------
// elementwise / layout kernels (fp32)
DS_DEV void split1(float x, float& hi, float& lo) {
  uint32_t t;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(t) : "f"(x));
  hi = __uint_as_float(t);
  lo = x - hi;  // exact
}

__global__ void split_kernel(const float* __restrict__ x, int64_t n, float* __restrict__ hi, float* __restrict__ lo) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    split1(x[i], hi[i], lo[i]);
}

// dst[c, r] = src[r + shift, c] (0 when r + shift is outside [0, rows)), as a
// hi/lo pair; src given as one fp32 array or a (hi, lo) pair summed exactly.
__global__ void tsplit_kernel(const float* __restrict__ s0, const float* __restrict__ s1, long long lds, int rows,
                              int cols, int shift, float* __restrict__ hi, float* __restrict__ lo, long long ldd) {
  __shared__ float tile[32][33];
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int r = r0 + j, c = c0 + threadIdx.x, sr = r + shift;
    float v = 0.f;
    if (r < rows && c < cols && sr >= 0 && sr < rows) {
      v = s0[(size_t)sr * lds + c];
      if (s1) v += s1[(size_t)sr * lds + c];
    }
    tile[j][threadIdx.x] = v;
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int c = c0 + j, r = r0 + threadIdx.x;
    if (c < cols && r < rows) split1(tile[threadIdx.x][j], hi[(size_t)c * ldd + r], lo[(size_t)c * ldd + r]);
  }
}

// x0[t*B + b, d] = feats[idx[b], t, d] (bf16 -> fp32, exact), labels alike
__global__ void gather_f32_kernel(const int64_t* __restrict__ idx, int B, int T, int D,
                                  const __nv_bfloat16* __restrict__ feats, const int32_t* __restrict__ labels,
                                  int64_t n_seq, float* __restrict__ x0, int32_t* __restrict__ lab, int* flag) {
  const int64_t total = (int64_t)T * B * kInPad;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int d = (int)(i % kInPad);
    const int64_t f = i / kInPad;
    const int b = (int)(f % B), t = (int)(f / B);
    int64_t q = idx[b];
    if (q < 0 || q >= n_seq) {
      if (d == 0 && t == 0) atomicOr(flag, 2);
      q = 0;
    }
    x0[i] = d < D ? __bfloat162float(feats[(q * T + t) * kInPad + d]) : 0.f;
    if (d == 0) lab[f] = labels[q * T + t];
  }
}

DS_DEV float sigm(float x) { return 1.f / (1.f + expf(-x)); }

// forward cell of both directions at their step s: dir 0 at t = s, dir 1 at
// t = T-1-s.  gates [N, 4096] (in: pre-activations, out: i,f,g,o), c [N, 1024],
// y [N, 1024] (+ hi/lo split for the next recurrent / layer GEMM)
__global__ void cell_fwd_kernel(int B, int T, int s, float* __restrict__ gates, float* __restrict__ cst,
                                float* __restrict__ y, float* __restrict__ yhi, float* __restrict__ ylo) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 2 * B * kHidden) return;
  const int u = i % kHidden, b = (i / kHidden) % B, dir = i / (kHidden * B);
  const int t = dir == 0 ? s : T - 1 - s, tp = dir == 0 ? t - 1 : t + 1;
  const size_t row = (size_t)t * B + b;
  float4 a = *reinterpret_cast<float4*>(gates + row * kGates2 + dir * kGates + u * 4);
  const float ig = sigm(a.x), fg = sigm(a.y), gg = tanhf(a.z), og = sigm(a.w);
  const float cp = (tp >= 0 && tp < T) ? cst[((size_t)tp * B + b) * kLayerOut + dir * kHidden + u] : 0.f;
  const float c = fg * cp + ig * gg;
  const float h = og * tanhf(c);
  *reinterpret_cast<float4*>(gates + row * kGates2 + dir * kGates + u * 4) = make_float4(ig, fg, gg, og);
  const size_t o = row * kLayerOut + dir * kHidden + u;
  cst[o] = c;
  y[o] = h;
  split1(h, yhi[o], ylo[o]);
}

// backward cell of both directions at their step s (dir 0 at t = T-1-s, dir 1
// at t = s): dh = dy[t] (already holding the recurrent dA_{t+-1} W_hh term),
// dc carry [2][B][512] in place; dA [N, 4096] fp32 + hi/lo
__global__ void cell_bwd_kernel(int B, int T, int s, const float* __restrict__ acts, const float* __restrict__ cst,
                                const float* __restrict__ dy, float* __restrict__ dcc, float* __restrict__ da,
                                float* __restrict__ dahi, float* __restrict__ dalo) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 2 * B * kHidden) return;
  const int u = i % kHidden, b = (i / kHidden) % B, dir = i / (kHidden * B);
  const int t = dir == 0 ? T - 1 - s : s, tp = dir == 0 ? t - 1 : t + 1;
  const size_t row = (size_t)t * B + b;
  const float4 a = *reinterpret_cast<const float4*>(acts + row * kGates2 + dir * kGates + u * 4);
  const size_t o = row * kLayerOut + dir * kHidden + u;
  const float c = cst[o];
  const float cp = (tp >= 0 && tp < T) ? cst[((size_t)tp * B + b) * kLayerOut + dir * kHidden + u] : 0.f;
  const float dh = dy[o];
  const float tc = tanhf(c);
  const float dc = dh * a.w * (1.f - tc * tc) + dcc[i];
  float4 d;
  d.x = dc * a.z * a.x * (1.f - a.x);
  d.y = dc * cp * a.y * (1.f - a.y);
  d.z = dc * a.x * (1.f - a.z * a.z);
  d.w = dh * tc * a.w * (1.f - a.w);
  dcc[i] = dc * a.y;
  const size_t g = row * kGates2 + dir * kGates + u * 4;
  *reinterpret_cast<float4*>(da + g) = d;
  split1(d.x, dahi[g], dalo[g]);
  split1(d.y, dahi[g + 1], dalo[g + 1]);
  split1(d.z, dahi[g + 2], dalo[g + 2]);
  split1(d.w, dahi[g + 3], dalo[g + 3]);
}

// one block per row: row loss = lse - logit[label]; with grad: the row becomes
// dlogits = (softmax - onehot) * scale as a hi (in place) / lo pair
__global__ void softmax_ce_kernel(float* __restrict__ logits, int C, const int32_t* __restrict__ lab, float scale,
                                  int grad, float* __restrict__ dlo, float* __restrict__ rowloss, int* flag) {
  const int r = blockIdx.x;
  float* x = logits + (size_t)r * C;
  __shared__ float red[32];
  __shared__ float bc;
  float m = -INFINITY;
  for (int c = threadIdx.x; c < C; c += blockDim.x) m = fmaxf(m, x[c]);
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : -INFINITY;
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (threadIdx.x == 0) bc = v;
  }
  __syncthreads();
  m = bc;
  float sacc = 0.f;
  for (int c = threadIdx.x; c < C; c += blockDim.x) sacc += expf(x[c] - m);
  for (int o = 16; o; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sacc;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) bc = v;
  }
  __syncthreads();
  const float lse = m + logf(bc);
  const int y = lab[r];
  if (threadIdx.x == 0) {
    if (y < 0 || y >= C) atomicOr(flag, 4);
    rowloss[r] = (y >= 0 && y < C) ? lse - x[y] : 0.f;
  }
  __syncthreads();
  if (!grad) return;
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    const float p = expf(x[c] - lse);
    const float d = (p - (c == y ? 1.f : 0.f)) * scale;
    float hi, lo;
    split1(d, hi, lo);
    x[c] = hi;
    dlo[(size_t)r * C + c] = lo;
  }
}

// loss_sum = sum of row losses in row order (one block, fixed tree): deterministic
__global__ void loss_sum_kernel(const float* __restrict__ rowloss, int n, float* loss, int* flag) {
  __shared__ double red[256];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += rowloss[i];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x / 2; o; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const float v = (float)red[0];
    *loss = v;
    if (!isfinite(v)) atomicOr(flag, 1);
  }
}

// out[c] = sum over rows of (a[r, c] (+ b[r, c])), rows in order (deterministic)
__global__ void colsum_f32_kernel(const float* __restrict__ a, const float* __restrict__ b, int rows, int cols,
                                  long long ld, float* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  double acc = 0.0;
  for (int r = 0; r < rows; ++r) {
    float v = a[(size_t)r * ld + c];
    if (b) v += b[(size_t)r * ld + c];
    acc += v;
  }
  out[c] = (float)acc;
}

inline int grid_for(int64_t n, int per = 256) {
  int64_t g = (n + per - 1) / per;
  return (int)(g < 148 * 16 ? (g > 0 ? g : 1) : 148 * 16);
}

}  // namespace

// ---------------------------------------------------------------------------
int split_launch(const float* x, int64_t n, const Split& out, cudaStream_t s) {
  split_kernel<<<grid_for(n), 256, 0, s>>>(x, n, out.hi, out.lo);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int tsplit_launch(const float* s0, const float* s1, long long lds, int rows, int cols, int shift, const Split& out,
                  long long ldd, cudaStream_t s) {
  dim3 grid((cols + 31) / 32, (rows + 31) / 32);
  tsplit_kernel<<<grid, dim3(32, 8), 0, s>>>(s0, s1, lds, rows, cols, shift, out.hi, out.lo, ldd);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int gemm3(const Split& A, long long lda, const Split& B, long long ldb, int M, int N, int K, float* out,
          long long ldo, const float* bias, int accumulate, cudaStream_t s) {
  T3Batch b;
  memset(&b, 0, sizeof(b));
  b.nprob = 1;
  int rc = t3_problem(&b.p[0], A, lda, B, ldb, M, N, K, out, ldo, bias, accumulate);
  if (rc) return rc;
  return t3_launch(&b, s);
}

// ---------------------------------------------------------------------------
// workspace
struct Arena3 {
  size_t off = 0;
  float* take(char* base, size_t n) {
    off = (off + 255) & ~size_t(255);
    float* p = reinterpret_cast<float*>(base + off);
    off += n * sizeof(float);
    return p;
  }
  Split pair(char* base, size_t n) {
    Split sp;
    sp.hi = take(base, n);
    sp.lo = take(base, n);
    return sp;
  }
};

static void carve3(ParityWs* w, const ModelLayout& L, int T, int Bmax, char* base, size_t* total) {
  Arena3 a;
  const size_t N = ((size_t)T * Bmax + 3) & ~size_t(3), C = L.classes, Bn = L.bottleneck;
  w->snap = a.take(base, L.total);
  w->W = a.pair(base, L.total);
  for (int l = 0; l < L.layers; ++l) {
    w->WihT[l] = a.pair(base, (size_t)kGates2 * L.in_dim(l));
    w->WhhT[l] = a.pair(base, (size_t)kGates2 * kHidden);
  }
  w->WoT = a.pair(base, C * Bn);
  w->WbT = a.pair(base, Bn * kLayerOut);
  w->x0 = a.take(base, N * kInPad);
  w->x0s = a.pair(base, N * kInPad);
  w->lab = reinterpret_cast<int32_t*>(a.take(base, N));
  for (int l = 0; l < L.layers; ++l) {
    w->gates[l] = a.take(base, N * kGates2);
    w->cst[l] = a.take(base, N * kLayerOut);
    w->y[l] = a.take(base, N * kLayerOut);
    w->ys[l] = a.pair(base, N * kLayerOut);
  }
  w->z = a.take(base, N * Bn);
  w->zs = a.pair(base, N * Bn);
  w->logits = a.take(base, N * C);
  w->dlo = a.take(base, N * C);
  w->dlT = a.pair(base, N * C);
  w->rowloss = a.take(base, N);
  w->dz = a.take(base, N * Bn);
  w->dzs = a.pair(base, N * Bn);
  w->dzT = a.pair(base, N * Bn);
  w->zT = a.pair(base, N * Bn);
  w->yT = a.pair(base, N * kLayerOut);
  w->dy = a.take(base, N * kLayerOut);
  w->da = a.take(base, N * kGates2);
  w->das = a.pair(base, N * kGates2);
  w->daT = a.pair(base, N * kGates2);
  w->hpT = a.pair(base, N * kLayerOut);
  w->dcc = a.take(base, (size_t)2 * Bmax * kHidden);
  *total = a.off + 256;
}

int parity_create(ParityWs** out, const ModelLayout& L, int T, int Bmax) {
  if (L.input_dim % 4) return fail_arg("fp32 parity mode needs input_dim % 4 == 0 (16-byte weight rows)");
  ParityWs* w = new ParityWs();
  size_t total = 0;
  carve3(w, L, T, Bmax, nullptr, &total);
  cudaError_t e = cudaMalloc(&w->arena, total);
  if (e != cudaSuccess) {
    delete w;
    return fail_cuda(e, "cudaMalloc(parity workspace)");
  }
  carve3(w, L, T, Bmax, reinterpret_cast<char*>(w->arena), &total);
  w->bytes = total;
  *out = w;
  return DS_OK;
}

void parity_destroy(ParityWs* w) {
  if (!w) return;
  if (w->arena) cudaFree(w->arena);
  delete w;
}

// Operand snapshot of theta (engines/adpsgd.py:132-134): an fp32 copy for the
// biases plus hi/lo splits of every weight, K-major as stored and transposed
// where the backward needs W^T as the K-major B operand.
int parity_snapshot(ParityWs* w, const ModelLayout& L, const float* theta, cudaStream_t s) {
  DS_CUDA_TRY(cudaMemcpyAsync(w->snap, theta, sizeof(float) * L.total, cudaMemcpyDeviceToDevice, s));
  int rc = split_launch(theta, L.total, w->W, s);
  for (int l = 0; l < L.layers && !rc; ++l) {
    const int D = L.in_dim(l);
    rc = tsplit_launch(theta + L.off_wih[l], nullptr, D, kGates2, D, 0, w->WihT[l], kGates2, s);  // [D][4096]
    for (int d = 0; d < 2 && !rc; ++d)  // per direction [512][2048]
      rc = tsplit_launch(theta + L.off_whh[l] + (size_t)d * kGates * kHidden, nullptr, kHidden, kGates, kHidden, 0,
                         w->WhhT[l].off((size_t)d * kGates * kHidden), kGates, s);
  }
  if (!rc) rc = tsplit_launch(theta + L.off_wo, nullptr, L.bottleneck, L.classes, L.bottleneck, 0, w->WoT, L.classes, s);
  if (!rc) rc = tsplit_launch(theta + L.off_wb, nullptr, kLayerOut, L.bottleneck, kLayerOut, 0, w->WbT, L.bottleneck, s);
  return rc;
}

// One gradient (grad != nullptr) or loss-only pass.
int parity_step(ParityWs* w, const ModelLayout& L, int T, const int64_t* idx, int B, const __nv_bfloat16* feats,
                const int32_t* labels, int64_t n_seq, float grad_frames, float* grad, float* loss, int* flag,
                cudaStream_t s, int* launches) {
  const int N = T * B, C = L.classes, Bn = L.bottleneck, Lh = L.layers;
  const long long Np = (N + 3) & ~3;  // row pitch of the transposed [*, N] operands (16-byte TMA rows)
  int rc;
  int nl = 0;
#define TRY(x)                 \
  do {                         \
    if ((rc = (x))) return rc; \
    ++nl;                      \
  } while (0)
  const float* th = w->snap;
  const int64_t nx = (int64_t)N * kInPad;
  gather_f32_kernel<<<grid_for(nx), 256, 0, s>>>(idx, B, T, L.input_dim, feats, labels, n_seq, w->x0, w->lab, flag);
  DS_CUDA_TRY(cudaGetLastError());
  TRY(split_launch(w->x0, nx, w->x0s, s));
  const int cell_blocks = (2 * B * kHidden + 255) / 256;

  // ---- forward ----
  for (int l = 0; l < Lh; ++l) {
    const int D = L.in_dim(l);
    const Split X = l == 0 ? w->x0s : w->ys[l - 1];
    TRY(gemm3(X, l == 0 ? kInPad : kLayerOut, w->W.off(L.off_wih[l]), D, N, kGates2, D, w->gates[l], kGates2, th + L.off_b[l], 0, s));
    for (int st = 0; st < T; ++st) {
      if (st > 0) {  // gates_t += h_{t-1} W_hh^T, both directions in one launch
        T3Batch b;
        memset(&b, 0, sizeof(b));
        b.nprob = 2;
        const int t0 = st, t1 = T - 1 - st;
        const Split h0 = w->ys[l].off((size_t)(t0 - 1) * B * kLayerOut);
        const Split h1 = w->ys[l].off((size_t)(t1 + 1) * B * kLayerOut + kHidden);
        rc = t3_problem(&b.p[0], h0, kLayerOut, w->W.off(L.off_whh[l]), kHidden, B, kGates, kHidden,
                        w->gates[l] + (size_t)t0 * B * kGates2, kGates2, nullptr, 1);
        if (!rc)
          rc = t3_problem(&b.p[1], h1, kLayerOut, w->W.off(L.off_whh[l] + (size_t)kGates * kHidden), kHidden, B,
                          kGates, kHidden, w->gates[l] + (size_t)t1 * B * kGates2 + kGates, kGates2, nullptr, 1);
        if (rc) return rc;
        TRY(t3_launch(&b, s));
      }
      cell_fwd_kernel<<<cell_blocks, 256, 0, s>>>(B, T, st, w->gates[l], w->cst[l], w->y[l], w->ys[l].hi,
                                                    w->ys[l].lo);
      DS_CUDA_TRY(cudaGetLastError());
      ++nl;
    }
  }
  TRY(gemm3(w->ys[Lh - 1], kLayerOut, w->W.off(L.off_wb), kLayerOut, N, Bn, kLayerOut, w->z, Bn, th + L.off_bb, 0,
            s));
  TRY(split_launch(w->z, (int64_t)N * Bn, w->zs, s));
  TRY(gemm3(w->zs, Bn, w->W.off(L.off_wo), Bn, N, C, Bn, w->logits, C, th + L.off_bo, 0, s));
  const float scale = 1.f / (grad_frames > 0.f ? grad_frames : (float)N);
  softmax_ce_kernel<<<N, 256, 0, s>>>(w->logits, C, w->lab, scale, grad != nullptr, w->dlo, w->rowloss, flag);
  DS_CUDA_TRY(cudaGetLastError());
  loss_sum_kernel<<<1, 256, 0, s>>>(w->rowloss, N, loss, flag);
  DS_CUDA_TRY(cudaGetLastError());
  nl += 2;
  if (!grad) {
    *launches = nl;
    return DS_OK;
  }

  // ---- backward: output layer and bottleneck ----
  const Split dl{w->logits, w->dlo};
  TRY(gemm3(dl, C, w->WoT, C, N, Bn, C, w->dz, Bn, nullptr, 0, s));  // dZ = dlogits W_o
  TRY(tsplit_launch(w->logits, w->dlo, C, N, C, 0, w->dlT, Np, s));    // dlogits^T [C][N]
  TRY(tsplit_launch(w->z, nullptr, Bn, N, Bn, 0, w->zT, Np, s));       // Z^T [Bn][N]
  TRY(gemm3(w->dlT, Np, w->zT, Np, C, Bn, N, grad + L.off_wo, Bn, nullptr, 0, s));
  colsum_f32_kernel<<<(C + 127) / 128, 128, 0, s>>>(w->logits, w->dlo, N, C, C, grad + L.off_bo);
  DS_CUDA_TRY(cudaGetLastError());
  ++nl;
  TRY(split_launch(w->dz, (int64_t)N * Bn, w->dzs, s));
  TRY(tsplit_launch(w->dz, nullptr, Bn, N, Bn, 0, w->dzT, Np, s));
  TRY(tsplit_launch(w->y[Lh - 1], nullptr, kLayerOut, N, kLayerOut, 0, w->yT, Np, s));
  TRY(gemm3(w->dzT, Np, w->yT, Np, Bn, kLayerOut, N, grad + L.off_wb, kLayerOut, nullptr, 0, s));
  colsum_f32_kernel<<<(Bn + 127) / 128, 128, 0, s>>>(w->dz, nullptr, N, Bn, Bn, grad + L.off_bb);
  DS_CUDA_TRY(cudaGetLastError());
  ++nl;
  TRY(gemm3(w->dzs, Bn, w->WbT, Bn, N, kLayerOut, Bn, w->dy, kLayerOut, nullptr, 0, s));  // dY = dZ W_b

  // ---- backward through the layers ----
  for (int l = Lh - 1; l >= 0; --l) {
    const int D = L.in_dim(l);
    DS_CUDA_TRY(cudaMemsetAsync(w->dcc, 0, sizeof(float) * 2 * B * kHidden, s));
    for (int st = 0; st < T; ++st) {
      const int t0 = T - 1 - st, t1 = st;
      if (st > 0) {  // dh_t += dA_{t+-1} W_hh, accumulated into dY in place
        T3Batch b;
        memset(&b, 0, sizeof(b));
        b.nprob = 2;
        rc = t3_problem(&b.p[0], w->das.off((size_t)(t0 + 1) * B * kGates2), kGates2, w->WhhT[l], kGates, B, kHidden,
                        kGates, w->dy + (size_t)t0 * B * kLayerOut, kLayerOut, nullptr, 1);
        if (!rc)
          rc = t3_problem(&b.p[1], w->das.off((size_t)(t1 - 1) * B * kGates2 + kGates), kGates2,
                          w->WhhT[l].off((size_t)kGates * kHidden), kGates, B, kHidden, kGates,
                          w->dy + (size_t)t1 * B * kLayerOut + kHidden, kLayerOut, nullptr, 1);
        if (rc) return rc;
        TRY(t3_launch(&b, s));
      }
      cell_bwd_kernel<<<cell_blocks, 256, 0, s>>>(B, T, st, w->gates[l], w->cst[l], w->dy, w->dcc, w->da, w->das.hi,
                                                    w->das.lo);
      DS_CUDA_TRY(cudaGetLastError());
      ++nl;
    }
    TRY(tsplit_launch(w->da, nullptr, kGates2, N, kGates2, 0, w->daT, Np, s));  // dA^T [4096][N]
    for (int d = 0; d < 2; ++d) {  // h_{t-1} (dir 0) / h_{t+1} (dir 1) as [512][N]
      TRY(tsplit_launch(w->y[l] + d * kHidden, nullptr, kLayerOut, N, kHidden, d == 0 ? -B : B,
                        w->hpT.off((size_t)d * kHidden * Np), Np, s));
      TRY(gemm3(w->daT.off((size_t)d * kGates * Np), Np, w->hpT.off((size_t)d * kHidden * Np), Np, kGates, kHidden,
                N, grad + L.off_whh[l] + (size_t)d * kGates * kHidden, kHidden, nullptr, 0, s));
    }
    const float* X = l == 0 ? w->x0 : w->y[l - 1];
    TRY(tsplit_launch(X, nullptr, l == 0 ? kInPad : kLayerOut, N, D, 0, w->yT, Np, s));  // X^T [D][N]
    TRY(gemm3(w->daT, Np, w->yT, Np, kGates2, D, N, grad + L.off_wih[l], D, nullptr, 0, s));
    colsum_f32_kernel<<<kGates2 / 128, 128, 0, s>>>(w->da, nullptr, N, kGates2, kGates2, grad + L.off_b[l]);
    DS_CUDA_TRY(cudaGetLastError());
    ++nl;
    if (l > 0) TRY(gemm3(w->das, kGates2, w->WihT[l], kGates2, N, D, kGates2, w->dy, kLayerOut, nullptr, 0, s));
  }
#undef TRY
  *launches = nl;
  return DS_OK;
}

}  // namespace ds

// ---------------------------------------------------------------------------
// test hook: C = A B^T (M x N, fp32) through the 3xTF32 tensor-core GEMM
extern "C" int ds_debug_gemm_tf32x3(const float* A, int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc,
                                    int32_t M, int32_t N, int32_t K, int32_t accumulate, void* stream) {
  using namespace ds;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (!A || !B || !C || M < 1 || N < 1 || K < 1 || lda < K || ldb < K || ldc < N) return fail_arg("bad gemm3 args");
  float* buf = nullptr;
  const size_t na = (size_t)M * lda, nb = (size_t)N * ldb;
  DS_CUDA_TRY(cudaMallocAsync(&buf, sizeof(float) * 2 * (na + nb), s));
  Split sa{buf, buf + na}, sb{buf + 2 * na, buf + 2 * na + nb};
  int rc = split_launch(A, na, sa, s);
  if (!rc) rc = split_launch(B, nb, sb, s);
  if (!rc) rc = gemm3(sa, lda, sb, ldb, M, N, K, C, ldc, nullptr, accumulate, s);
  cudaFreeAsync(buf, s);
  return rc;
}
