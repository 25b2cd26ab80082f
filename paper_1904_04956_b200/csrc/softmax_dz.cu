// softmax_dz.cu — fused soft-max gradient and bottleneck input gradient of the
// 32000-way output layer (SURVEY §2.3 K8-bwd + the dZ half of K7-bwd):
//
//   dlogits = (softmax(Z W_o^T + b_o) - onehot(y)) / frames      (bf16, stored)
//   dZ      = dlogits W_o                                        (fp32 partials)
//   db_o    = column sums of dlogits                             (partials)
//
// One CTA owns a 128-row block of Z (resident in smem) and a contiguous range
// of 128-class tiles of W_o.  Per class tile: MMA1 (tcgen05, M128 N128 K=bott)
// puts the logits in TMEM; the epilogue turns them into the dlogits tile,
// writes it as bf16 into smem in the SW128 K-major layout of an MMA operand,
// TMA-stores it to the 64x64-blocked global dlogits (read by the dW_o GEMM)
// and hands it to MMA2 (M128 N=bott K128), which accumulates dZ for the row
// block in TMEM across the whole class range.  The soft-max epilogue is the
// bottleneck of this pass, so MMA2 runs in its shadow and dZ never re-reads
// dlogits from HBM; the class ranges of a row block are reduced afterwards
// (op_splitk_bf16, fixed order).
//
// W_o tile smem layout (bott/64 blocks of [128 classes x 64 bott], SW128) is
// MMA1's K-major B operand and, unchanged, MMA2's MN-major B operand
// (K = classes, N = bott, one N chunk per block).
#include "ds_internal.h"
#include "ds_ptx.cuh"
#include "softmax_dz.h"

#include <cstring>

namespace ds {
namespace {

constexpr int kThreads = 640;   // warps 0-3 roles, 4-19 epilogue
constexpr int kEpiWarp0 = 4;
constexpr int kEpiT = 512;
constexpr int kRows = 128;      // Z rows per CTA (MMA M)
constexpr int kCT = 128;        // classes per tile (MMA1 N, MMA2 K)
constexpr int kMaxBott = 256;
constexpr int kZB = kRows * kMaxBott * 2;  // 64 KB resident Z block
constexpr int kWB = kCT * kMaxBott * 2;    // 64 KB per W_o tile stage
constexpr int kPB = kRows * kCT * 2;       // 32 KB dlogits tile (MMA2 A operand)
constexpr size_t kSmem = 1024 + kZB + 2 * kWB + kPB + 512;
constexpr float kLog2e = 1.4426950408889634f;

__global__ void __launch_bounds__(kThreads, 1) ce_grad_dz_kernel(const __grid_constant__ CeGradDzParams P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sZ = sm;
  uint8_t* sW = sZ + kZB;        // [2 stages]
  uint8_t* sP = sW + 2 * kWB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + kPB);
  uint64_t* zfull = bars;        // Z block landed
  uint64_t* zempty = zfull + 1;  // MMA1s of the item done with sZ
  uint64_t* wfull = zempty + 1;  // [2]
  uint64_t* wempty = wfull + 2;  // [2]
  uint64_t* tfull1 = wempty + 2;  // [2] logits accumulators
  uint64_t* tempty1 = tfull1 + 2;  // [2]
  uint64_t* pfull = tempty1 + 2;   // dlogits tile in sP
  uint64_t* pempty = pfull + 1;    // MMA2 done with sP
  uint64_t* dzfull = pempty + 1;   // dZ accumulator complete
  uint64_t* dzempty = dzfull + 1;  // epilogue drained the dZ accumulator
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dzempty + 1);

  const uint32_t warp = warp_id(), lane = lane_id();
  const int bott = P.bott, nkb = bott / 64;
  const int items = P.n_rb * P.n_cs;

  if (warp == 1 && lane == 0) {
    mbar_init(zfull, 1);
    mbar_init(zempty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&wfull[i], 1);
      mbar_init(&wempty[i], 1);
      mbar_init(&tfull1[i], 1);
      mbar_init(&tempty1[i], kEpiT);
    }
    mbar_init(pfull, 1);
    mbar_init(pempty, 1);
    mbar_init(dzfull, 1);
    mbar_init(dzempty, kEpiT);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t acc2 = tmem + 256;

  if (warp == 0) {
    if (elect_one()) {
      tma_prefetch_desc(&P.tmZ);
      tma_prefetch_desc(&P.tmW);
      int g = 0, it = 0;  // global class-tile counter, item counter
      for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
        const int rb = item % P.n_rb, cs = item / P.n_rb;
        const int ct0 = cs * P.ct_per, ct1 = min(P.n_ct, ct0 + P.ct_per);
        mbar_wait(zempty, (it & 1) ^ 1);
        mbar_arrive_expect_tx(zfull, kRows * bott * 2);
        for (int kb = 0; kb < nkb; ++kb) tma_load_2d(sZ + kb * 16384, &P.tmZ, zfull, kb * 64, rb * kRows);
        for (int ct = ct0; ct < ct1; ++ct, ++g) {
          const int st = g & 1;
          mbar_wait(&wempty[st], ((g >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx(&wfull[st], kCT * bott * 2);
          for (int kb = 0; kb < nkb; ++kb)
            tma_load_2d(sW + st * kWB + kb * 16384, &P.tmW, &wfull[st], kb * 64, ct * kCT);
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      const uint32_t id1 = idesc_bf16_f32(kRows, kCT, 0, 0);
      const uint32_t id2 = idesc_bf16_f32(kRows, bott, 0, 1);
      const uint32_t zb = smem_u32(sZ), wb = smem_u32(sW), pb = smem_u32(sP);
      int g = 0, it = 0;
      auto mma2 = [&](int gp, bool first) {  // dZ += dlogits(gp) W_o(gp)
        const int st = gp & 1;
        mbar_wait(pfull, gp & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < kCT / 16; ++kk) {
          const uint64_t ad = smem_desc_sw128(pb + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
          const uint64_t bd = smem_desc_sw128(wb + st * kWB + kk * 2048, 16384, 1024);
          mma_bf16_ss(acc2, ad, bd, id2, (!first || kk) ? 1u : 0u);
        }
        mma_commit(pempty);
        mma_commit(&wempty[st]);
      };
      for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
        const int cs = item / P.n_rb;
        const int ct0 = cs * P.ct_per, ct1 = min(P.n_ct, ct0 + P.ct_per);
        mbar_wait(zfull, it & 1);
        mbar_wait(dzempty, (it & 1) ^ 1);  // previous item's dZ drained
        tc_fence_after();
        const int g0 = g;
        for (int ct = ct0; ct < ct1; ++ct, ++g) {
          const int st = g & 1, a = g & 1;
          mbar_wait(&wfull[st], (g >> 1) & 1);
          mbar_wait(&tempty1[a], ((g >> 1) & 1) ^ 1);
          tc_fence_after();
#pragma unroll 1
          for (int kk = 0; kk < bott / 16; ++kk) {
            const uint64_t ad = smem_desc_sw128(zb + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
            const uint64_t bd = smem_desc_sw128(wb + st * kWB + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
            mma_bf16_ss(tmem + a * kCT, ad, bd, id1, kk ? 1u : 0u);
          }
          mma_commit(&tfull1[a]);
          if (ct == ct1 - 1) mma_commit(zempty);
          if (g > g0) mma2(g - 1, g - 1 == g0);
        }
        mma2(g - 1, g - 1 == g0);
        mma_commit(dzfull);
      }
    }
  } else if (warp >= kEpiWarp0) {
    const uint32_t e = warp - kEpiWarp0;
    const uint32_t q = e & 3, part = e >> 2;  // TMEM lane quadrant, 32-column quarter
    const int tid = (int)(e * 32 + lane);
    const uint32_t tq = tmem + ((q * 32) << 16);
    const float* __restrict__ bias = P.bias;
    int g = 0, it = 0;
    for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
      const int rb = item % P.n_rb, cs = item / P.n_rb;
      const int ct0 = cs * P.ct_per, ct1 = min(P.n_ct, ct0 + P.ct_per);
      const int rloc = (int)(q * 32 + lane);
      const int row = rb * kRows + rloc;
      const bool row_ok = row < P.m_valid;
      const int lbl = row_ok ? P.labels[row] : -1;
      const float l2 = row_ok ? P.lse[row] * kLog2e : 0.f;
      const float sc = (row_ok && lbl >= 0) ? P.scale : 0.f;
      for (int ct = ct0; ct < ct1; ++ct, ++g) {
        const int a = g & 1;
        const int nb = ct * kCT + (int)part * 32;
        mbar_wait(&tfull1[a], (g >> 1) & 1);
        tc_fence_after();
        float v[32];
        tmem_ld32(tq + a * kCT + part * 32, v);
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&tempty1[a]);
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const float4 bb = __ldg(reinterpret_cast<const float4*>(bias + nb + i));
          v[i] = ex2_fast(fmaf(v[i] + bb.x, kLog2e, -l2));
          v[i + 1] = ex2_fast(fmaf(v[i + 1] + bb.y, kLog2e, -l2));
          v[i + 2] = ex2_fast(fmaf(v[i + 2] + bb.z, kLog2e, -l2));
          v[i + 3] = ex2_fast(fmaf(v[i + 3] + bb.w, kLog2e, -l2));
        }
        if (lbl >= nb && lbl < nb + 32) {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (lbl == nb + i) v[i] -= 1.f;
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] *= sc;
        // sP free: MMA2 of the previous tile is done and its TMA stores read it
        if (tid == 0) bulk_wait_read0();
        if (g > 0) mbar_wait(pempty, (g - 1) & 1);
        named_bar_sync(1, kEpiT);
        {
          uint8_t* blk = sP + (part >> 1) * 16384 + rloc * 128;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint4 w;
            uint32_t* u = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              __nv_bfloat162 h = __floats2bfloat162_rn(v[8 * j + 2 * i], v[8 * j + 2 * i + 1]);
              u[i] = *reinterpret_cast<uint32_t*>(&h);
            }
            const int c = (int)(part & 1) * 4 + j;
            *reinterpret_cast<uint4*>(blk + ((c ^ (rloc & 7)) << 4)) = w;
          }
        }
        fence_proxy_async_smem();
        named_bar_sync(1, kEpiT);
        if (tid == 0) {
          mbar_arrive(pfull);
          for (int b = 0; b < 2; ++b)        // class blocks of the tile
            for (int h = 0; h < 2; ++h)      // 64-row halves
              tma_store_4d(&P.tmP, sP + b * 16384 + h * 8192, 0, 0, ct * 2 + b, rb * 2 + h);
          bulk_commit();
        }
        if (P.colpart) {  // bias gradient: column sums of this warp's 32 rows (fp32, pre-rounding)
          const float csum = warp_colsum32(v);
          if (rb * kRows < P.m_valid) P.colpart[(size_t)(rb * 4 + q) * P.classes + nb + lane] = csum;
        }
      }
      // dZ partial of this (row block, class range): fp32 [cs][row][bott]
      mbar_wait(dzfull, it & 1);
      tc_fence_after();
      const int cols = bott / 4;
      float* dst = P.dzpart + ((size_t)cs * P.dz_rows + row) * bott + part * cols;
      for (int c0 = 0; c0 < cols; c0 += 16) {
        float w[16];
        tmem_ld16(acc2 + ((q * 32) << 16) + part * cols + c0, w);
        tmem_ld_wait();
        if (row_ok) {
#pragma unroll
          for (int i = 0; i < 16; i += 4)
            *reinterpret_cast<float4*>(dst + c0 + i) = make_float4(w[i], w[i + 1], w[i + 2], w[i + 3]);
        }
      }
      tc_fence_before();
      mbar_arrive(dzempty);
    }
    if (tid == 0) bulk_wait0();
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

}  // namespace

bool ce_grad_dz_supported(int classes, int bott) {
  return classes % kCT == 0 && bott % 64 == 0 && bott >= 64 && bott <= kMaxBott;
}

// class ranges per row block: about two work items per SM, so the persistent
// CTAs finish together (one item per row block and split leaves SMs idle when
// the row-block count does not divide the SM count)
int ce_grad_dz_splits(int rows, int classes, int max_splits) {
  const int n_rb = (rows + kRows - 1) / kRows, n_ct = classes / kCT;
  int s = (2 * num_sms()) / n_rb;
  s = s < 1 ? 1 : (s > max_splits ? max_splits : s);
  s = s > n_ct ? n_ct : s;
  const int per = (n_ct + s - 1) / s;
  return (n_ct + per - 1) / per;  // no empty class range
}

int ce_grad_dz_launch(const CeGradDzArgs& a, cudaStream_t stream) {
  static bool attr_set = false;
  if (!attr_set) {
    DS_CUDA_TRY(cudaFuncSetAttribute(ce_grad_dz_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem));
    attr_set = true;
  }
  if (!ce_grad_dz_supported(a.classes, a.bott)) return fail_arg("fused soft-max/dZ: unsupported shape");
  CeGradDzParams P;
  memset(&P, 0, sizeof(P));
  int rc = make_tmap_2d(&P.tmZ, a.z, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, a.bott, a.rows, (uint64_t)a.bott * 2, 64, kRows);
  if (rc) return rc;
  rc = make_tmap_2d(&P.tmW, a.w, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, a.bott, a.classes, (uint64_t)a.bott * 2, 64, kCT);
  if (rc) return rc;
  {  // dlogits, 64x64-blocked [row/64][class/64][64][64]
    const uint64_t nrb = (a.rows + 63) / 64, ncb = a.classes / 64;
    const uint64_t dims[4] = {64, 64, ncb, nrb};
    const uint64_t strides[3] = {128, 8192, ncb * 8192};
    const uint32_t box[4] = {64, 64, 1, 1};
    rc = make_tmap_4d(&P.tmP, a.dlogits, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, dims, strides, box);
    if (rc) return rc;
  }
  P.bias = a.bias;
  P.labels = a.labels;
  P.lse = a.lse;
  P.colpart = a.colpart;
  P.dzpart = a.dzpart;
  P.scale = a.scale;
  P.bott = a.bott;
  P.classes = a.classes;
  P.m_valid = a.rows;
  P.dz_rows = a.rows;
  P.n_rb = (a.rows + kRows - 1) / kRows;
  P.n_ct = a.classes / kCT;
  P.n_cs = a.splits;
  P.ct_per = (P.n_ct + a.splits - 1) / a.splits;
  if ((a.splits - 1) * P.ct_per >= P.n_ct) return fail_arg("fused soft-max/dZ: empty class range");
  const int items = P.n_rb * P.n_cs;
  const int grid = items < num_sms() ? items : num_sms();
  ce_grad_dz_kernel<<<grid, kThreads, kSmem, stream>>>(P);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

}  // namespace ds
