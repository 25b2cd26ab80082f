// gemm.cu — persistent tcgen05 GEMM (bf16 x bf16 -> fp32 TMEM) with the
// BLSTM-specific epilogues.
//
// Used for every dense product of the BLSTM training step (SURVEY §2.3 K3,
// K6, K7, K8): input projections G = X W_ih^T + b, weight gradients
// dW = dG^T X (both operands MN-major, K = frames), input gradients
// dX = dG W_ih (B MN-major), the bottleneck, and the 32000-way output layer
// whose epilogue computes soft-max statistics (forward) or
// (softmax - onehot)/N (backward) without ever materialising fp32 logits.
//
// Structure (one CTA per SM, 256 threads):
//   warp 0      : TMA producer (one elected lane), 4-stage smem ring
//   warp 1      : tcgen05.mma issuer (one elected lane)
//   warp 2      : TMEM allocator (512 columns = 2 x 128x256 fp32 accumulators)
//   warps 4..7  : epilogue, thread = accumulator row (TMEM lane)
// Tiles are walked round-robin over the persistent grid; the two TMEM
// accumulators let the epilogue of tile i overlap the main loop of tile i+1.
#include "ds_internal.h"
#include "ds_ptx.cuh"

namespace ds {

namespace {

constexpr int BM = kGemmBM, BN = kGemmBN, BK = kGemmBK;
constexpr int kStages = 4;
constexpr int kABytes = BM * BK * 2;  // 16 KB
constexpr int kBBytes = BN * BK * 2;  // 32 KB
constexpr int kStageBytes = kABytes + kBBytes;
constexpr int kThreads = 256;
constexpr int kEpiWarp0 = 4;
constexpr uint32_t kTmemCols = 512;
constexpr size_t kSmemBytes = 1024 /*align slack*/ + (size_t)kStages * kStageBytes + 256;

struct TileCoord {
  int prob, tm, tn;
};

__device__ __forceinline__ TileCoord locate(const GemmBatch& b, int tile) {
  int p = 0;
#pragma unroll
  for (int i = 1; i < kMaxProblems; ++i)
    if (i < b.nprob && tile >= b.p[i].tile_begin) p = i;
  int local = tile - b.p[p].tile_begin;
  TileCoord c;
  c.prob = p;
  c.tm = local % b.p[p].tiles_m;
  c.tn = local / b.p[p].tiles_m;
  return c;
}

__device__ __forceinline__ void store_bf16x16(__nv_bfloat16* dst, const float* v) {
  uint4 w[2];
  uint32_t* u = reinterpret_cast<uint32_t*>(w);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    u[i] = *reinterpret_cast<uint32_t*>(&h);
  }
  reinterpret_cast<uint4*>(dst)[0] = w[0];
  reinterpret_cast<uint4*>(dst)[1] = w[1];
}

__global__ void __launch_bounds__(kThreads, 1) gemm_kernel(const __grid_constant__ GemmBatch batch) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < batch.nprob; ++i) {
      tma_prefetch_desc(&batch.p[i].tmA);
      tma_prefetch_desc(&batch.p[i].tmB);
    }
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int total = batch.total_tiles;

  if (warp == 0) {
    if (elect_one()) {
      // ---------------- TMA producer ----------------
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
        TileCoord tc = locate(batch, tile);
        const GemmProblem& P = batch.p[tc.prob];
        const int m0 = tc.tm * BM, n0 = tc.tn * BN;
        const int nkb = (P.K + BK - 1) / BK;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sA = smem + stage * kStageBytes;
          uint8_t* sB = sA + kABytes;
          mbar_arrive_expect_tx(&full[stage], kStageBytes);
          const int k0 = kb * BK;
          if (!P.a_mn) {
            tma_load_2d(sA, &P.tmA, &full[stage], k0, m0);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j) tma_load_2d(sA + j * 8192, &P.tmA, &full[stage], m0 + 64 * j, k0);
          }
          if (!P.b_mn) {
            tma_load_2d(sB, &P.tmB, &full[stage], k0, n0);
          } else {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j) tma_load_2d(sB + j * 8192, &P.tmB, &full[stage], n0 + 64 * j, k0);
          }
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++it) {
      TileCoord tc = locate(batch, tile);
      const GemmProblem& P = batch.p[tc.prob];
      const int nkb = (P.K + BK - 1) / BK;
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const uint32_t idesc = idesc_bf16_f32(BM, BN, P.a_mn, P.b_mn);
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t aBase = smem_u32(smem + stage * kStageBytes);
          const uint32_t bBase = aBase + kABytes;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            uint64_t ad = P.a_mn ? smem_desc_sw128(aBase + k * 2048, 8192, 1024)
                                 : smem_desc_sw128(aBase + k * 32, 16, 1024);
            uint64_t bd = P.b_mn ? smem_desc_sw128(bBase + k * 2048, 8192, 1024)
                                 : smem_desc_sw128(bBase + k * 32, 16, 1024);
            mma_bf16_ss(d_tmem, ad, bd, idesc, (kb | k) != 0);
          }
          mma_commit(&empty[stage]);
          if (kb == nkb - 1) mma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp >= kEpiWarp0) {
    // ---------------- epilogue ----------------
    const uint32_t q = warp - kEpiWarp0;  // TMEM lane quadrant (warp % 4)
    int it = 0;
    for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++it) {
      TileCoord tc = locate(batch, tile);
      const GemmProblem& P = batch.p[tc.prob];
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const int row = tc.tm * BM + q * 32 + lane;
      const int n0 = tc.tn * BN;
      const bool row_ok = row < P.m_valid;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t t_row = tmem_base + acc * BN + ((q * 32) << 16);

      if (P.epi == EPI_CE_STATS) {
        float mx = -INFINITY, se = 0.f, tg = 0.f;
        int lbl = row_ok ? P.labels[row] : -1;
        bool have_t = false;
        for (int c = 0; c < BN; c += 16) {
          float v[16];
          tmem_ld16(t_row + c, v);
          tmem_ld_wait();
          float cm = -INFINITY;
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            int n = n0 + c + i;
            float x = (n < P.n_valid) ? v[i] + (P.bias ? __ldg(P.bias + n) : 0.f) : -INFINITY;
            v[i] = x;
            cm = fmaxf(cm, x);
            if (n == lbl) {
              tg = x;
              have_t = true;
            }
          }
          if (cm > -INFINITY) {
            float nm = fmaxf(mx, cm);
            float s = 0.f;
#pragma unroll
            for (int i = 0; i < 16; ++i) s += __expf(v[i] - nm);
            se = se * __expf(mx - nm) + s;
            mx = nm;
          }
        }
        if (row_ok) {
          P.stats[(size_t)tc.tn * P.stats_ld + row] = make_float2(mx, se);
          if (have_t) P.tgt[row] = tg;
        }
      } else if (P.epi == EPI_CE_GRAD) {
        const float l = row_ok ? P.lse[row] : 0.f;
        const int lbl = row_ok ? P.labels[row] : -1;
        __nv_bfloat16* orow = reinterpret_cast<__nv_bfloat16*>(P.out) + (size_t)row * P.ldo;
        for (int c = 0; c < BN; c += 16) {
          float v[16];
          tmem_ld16(t_row + c, v);
          tmem_ld_wait();
          const int nb = n0 + c;
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            int n = nb + i;
            float x = v[i] + ((P.bias && n < P.n_valid) ? __ldg(P.bias + n) : 0.f);
            float p = __expf(x - l) - (n == lbl ? 1.f : 0.f);
            v[i] = p * P.scale;
          }
          if (row_ok && nb < P.n_valid) store_bf16x16(orow + nb, v);
        }
      } else if (P.epi == EPI_BF16) {
        __nv_bfloat16* orow = reinterpret_cast<__nv_bfloat16*>(P.out) + (size_t)row * P.ldo;
        for (int c = 0; c < BN; c += 16) {
          float v[16];
          tmem_ld16(t_row + c, v);
          tmem_ld_wait();
          const int nb = n0 + c;
          if (P.bias) {
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] += (nb + i < P.n_valid) ? __ldg(P.bias + nb + i) : 0.f;
          }
          if (row_ok && nb < P.n_valid) store_bf16x16(orow + nb, v);
        }
      } else {  // EPI_F32
        float* orow = reinterpret_cast<float*>(P.out) + (size_t)row * P.ldo;
        for (int c = 0; c < BN; c += 16) {
          float v[16];
          tmem_ld16(t_row + c, v);
          tmem_ld_wait();
          const int nb = n0 + c;
          if (row_ok) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              int n = nb + i;
              if (n < P.n_valid) {
                float x = v[i] * P.scale;
                if (P.accumulate) x += orow[n];
                orow[n] = x;
              }
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem_base, kTmemCols);
}

}  // namespace

int gemm_problem(GemmProblem* p, const void* A, long long lda, int a_mn, const void* B, long long ldb, int b_mn,
                 int M, int N, int K) {
  if (M <= 0 || N <= 0 || K <= 0) return fail_arg("gemm: empty problem");
  memset(p, 0, sizeof(*p));
  int rc;
  if (!a_mn)
    rc = make_tmap_2d(&p->tmA, A, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, K, M, (uint64_t)lda * 2, 64, BM);
  else
    rc = make_tmap_2d(&p->tmA, A, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, M, K, (uint64_t)lda * 2, 64, 64);
  if (rc) return rc;
  if (!b_mn)
    rc = make_tmap_2d(&p->tmB, B, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, K, N, (uint64_t)ldb * 2, 64, BN);
  else
    rc = make_tmap_2d(&p->tmB, B, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, N, K, (uint64_t)ldb * 2, 64, 64);
  if (rc) return rc;
  p->M = M;
  p->N = N;
  p->K = K;
  p->a_mn = a_mn;
  p->b_mn = b_mn;
  p->tiles_m = (M + BM - 1) / BM;
  p->tiles_n = (N + BN - 1) / BN;
  p->n_valid = N;
  p->m_valid = M;
  p->scale = 1.f;
  return DS_OK;
}

int gemm_launch(GemmBatch* b, cudaStream_t stream) {
  static bool attr_set = false;
  if (!attr_set) {
    DS_CUDA_TRY(cudaFuncSetAttribute(gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes));
    attr_set = true;
  }
  int total = 0;
  for (int i = 0; i < b->nprob; ++i) {
    b->p[i].tile_begin = total;
    total += b->p[i].tiles_m * b->p[i].tiles_n;
  }
  b->total_tiles = total;
  if (total == 0) return DS_OK;
  int grid = total < num_sms() ? total : num_sms();
  gemm_kernel<<<grid, kThreads, kSmemBytes, stream>>>(*b);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

}  // namespace ds
