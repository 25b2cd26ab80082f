// softmax_dz.cu — fused soft-max gradient and bottleneck input gradient of the
// 32000-way output layer (SURVEY §2.3 K8-bwd + the dZ half of K7-bwd):
//
//   dlogits = (softmax(Z W_o^T + b_o) - onehot(y)) / frames      (bf16, stored)
//   dZ      = dlogits W_o                                        (fp32 partials)
//   db_o    = column sums of dlogits                             (partials)
//
// One CTA owns a 128-row block of Z (resident in smem) and a contiguous range
// of 64-class tiles of W_o (streamed through a 4-stage ring).  Per class
// tile: MMA1 (tcgen05, M128 N64 K=bott) puts the logits in one of four TMEM
// buffers.  Two groups of 8 epilogue warps take alternate tiles; each warp
// turns its 32 rows x 32 classes into dlogits, TMA-stores them from its own
// 2 KB shared-memory box to the 64x64-blocked global dlogits (read by the
// dW_o GEMM), and writes them back as bf16 into the first 16 columns of its
// TMEM slice, where MMA2 (M128 N=bott K64, A from tensor memory) reads them to
// accumulate dZ for the row block across the class range.  No CTA-wide
// barrier per tile: each warp hands its slice to MMA2 with one mbarrier
// arrive.  MMA1 runs two tiles ahead of MMA2, so the tensor pipe computes
// the next logits while the epilogue finishes a tile; a W_o tile is held from
// its MMA1 until its MMA2, and the 4-deep ring / 4 logits buffers cover that.  The class ranges of a row block are
// reduced afterwards (op_splitk_bf16, fixed order).
//
// W_o tile smem layout (bott/64 blocks of [64 classes x 64 bott], SW128) is
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
constexpr int kEpiWarps = 16;
constexpr int kRows = 128;      // Z rows per CTA (MMA M)
constexpr int kCT = 64;         // classes per tile (MMA1 N, MMA2 K)
constexpr int kWarpCls = kCT / 2;  // classes per epilogue warp and tile (2 halves x 4 lane quadrants)
constexpr int kWStages = 4;
constexpr int kAcc = 4;         // logits buffers (kAcc * kCT + bott <= 512 TMEM columns)
constexpr int kLead = 2;        // MMA1 runs this many tiles ahead of MMA2 (< kAcc, < kWStages)
constexpr int kMaxBott = 256;
constexpr int kZB = kRows * kMaxBott * 2;  // 64 KB resident Z block
constexpr int kWB = kCT * kMaxBott * 2;    // 32 KB per W_o tile stage
constexpr int kCB = 32 * kWarpCls * 2;     // 2 KB dlogits box per epilogue warp
constexpr size_t kSmem = 1024 + kZB + kWStages * kWB + kEpiWarps * kCB + 512;
constexpr float kLog2e = 1.4426950408889634f;

__global__ void __launch_bounds__(kThreads, 1) ce_grad_dz_kernel(const __grid_constant__ CeGradDzParams P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sZ = sm;
  uint8_t* sW = sZ + kZB;  // [kWStages]
  uint8_t* sC = sW + kWStages * kWB;  // [kEpiWarps] dlogits store boxes
  uint64_t* bars = reinterpret_cast<uint64_t*>(sC + kEpiWarps * kCB);
  uint64_t* zfull = bars;               // Z block landed
  uint64_t* zempty = zfull + 1;         // MMA1s of the item done with sZ
  uint64_t* wfull = zempty + 1;         // [kWStages]
  uint64_t* wempty = wfull + kWStages;  // [kWStages] MMA2 of the tile done with the stage
  uint64_t* tfull1 = wempty + kWStages; // [kAcc] logits ready
  uint64_t* tempty1 = tfull1 + kAcc;    // [kAcc] MMA2 done reading the dlogits written back into it
  uint64_t* pfull = tempty1 + kAcc;     // [kAcc] every epilogue warp wrote its dlogits slice
  uint64_t* dzfull = pfull + kAcc;      // dZ accumulator complete
  uint64_t* dzempty = dzfull + 1;       // epilogue drained the dZ accumulator
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dzempty + 1);

  const uint32_t warp = warp_id(), lane = lane_id();
  const int bott = P.bott, nkb = bott / 64;
  // trace: [cta][tile < 80][4]: MMA1 issued, MMA2 issued, epilogue (warp 4) logits seen, epilogue done
  unsigned long long* const tr = P.trace ? P.trace + (size_t)blockIdx.x * 80 * 4 : nullptr;
  const int items = P.n_rb * P.n_cs;

  if (warp == 1 && lane == 0) {
    mbar_init(zfull, 1);
    mbar_init(zempty, 1);
    for (int i = 0; i < kWStages; ++i) {
      mbar_init(&wfull[i], 1);
      mbar_init(&wempty[i], 1);
    }
    for (int i = 0; i < kAcc; ++i) {
      mbar_init(&tfull1[i], 1);
      mbar_init(&tempty1[i], 1);
      mbar_init(&pfull[i], kEpiWarps / 2);
    }
    mbar_init(dzfull, 1);
    mbar_init(dzempty, kEpiWarps * 32);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t acc2 = tmem + kAcc * kCT;
  griddep_wait();  // lse / labels come from the immediately preceding kernels
  griddep_launch();

  if (warp == 0) {
    if (elect_one()) {
      tma_prefetch_desc(&P.tmZ);
      tma_prefetch_desc(&P.tmW);
      tma_prefetch_desc(&P.tmP);
      int g = 0, it = 0;  // global class-tile counter, item counter
      for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
        const int rb = item % P.n_rb, cs = item / P.n_rb;
        const int ct0 = cs * P.ct_per, ct1 = min(P.n_ct, ct0 + P.ct_per);
        mbar_wait(zempty, (it & 1) ^ 1);
        mbar_arrive_expect_tx(zfull, kRows * bott * 2);
        for (int kb = 0; kb < nkb; ++kb) tma_load_2d(sZ + kb * 16384, &P.tmZ, zfull, kb * 64, rb * kRows);
        for (int ct = ct0; ct < ct1; ++ct, ++g) {
          const int st = g % kWStages;
          mbar_wait(&wempty[st], ((g / kWStages) & 1) ^ 1);
          mbar_arrive_expect_tx(&wfull[st], kCT * bott * 2);
          for (int kb = 0; kb < nkb; ++kb)
            tma_load_2d(sW + st * kWB + kb * (kCT * 128), &P.tmW, &wfull[st], kb * 64, ct * kCT);
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      const uint32_t id1 = idesc_bf16_f32(kRows, kCT, 0, 0);
      const uint32_t id2 = idesc_bf16_f32(kRows, bott, 0, 1);
      const uint32_t zb = smem_u32(sZ), wb = smem_u32(sW);
      int g = 0, it = 0;
      auto mma2 = [&](int gp, bool first) {  // dZ += dlogits(gp) W_o(gp), dlogits from TMEM
        const int st = gp % kWStages, a = gp % kAcc;
        mbar_wait(&pfull[a], (gp / kAcc) & 1);
        tc_fence_after();
        if (tr && gp < 80) tr[gp * 4 + 1] = globaltimer();
#pragma unroll
        for (int kk = 0; kk < kCT / 16; ++kk) {
          // classes kk*16.. : written by tile half kk/2 into its columns (kk&1)*8..
          const uint32_t at = tmem + a * kCT + (kk >> 1) * kWarpCls + (kk & 1) * 8;
          const uint64_t bd = smem_desc_sw128(wb + st * kWB + kk * 2048, kCT * 128, 1024);
          mma_bf16_ts(acc2, at, bd, id2, (!first || kk) ? 1u : 0u);
        }
        mma_commit(&tempty1[a]);
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
          const int st = g % kWStages, a = g % kAcc;
          mbar_wait(&wfull[st], (g / kWStages) & 1);
          mbar_wait(&tempty1[a], ((g / kAcc) & 1) ^ 1);  // MMA2 of tile g-kAcc read its dlogits
          tc_fence_after();
          if (tr && g < 80) tr[g * 4 + 0] = globaltimer();
#pragma unroll 1
          for (int kk = 0; kk < bott / 16; ++kk) {
            const uint64_t ad = smem_desc_sw128(zb + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
            const uint64_t bd = smem_desc_sw128(wb + st * kWB + (kk >> 2) * (kCT * 128) + (kk & 3) * 32, 16, 1024);
            mma_bf16_ss(tmem + a * kCT, ad, bd, id1, kk ? 1u : 0u);
          }
          mma_commit(&tfull1[a]);
          if (ct == ct1 - 1) mma_commit(zempty);
          // MMA2 trails MMA1 by kLead tiles: the logits of the next tiles are computed while
          // the epilogue of tile g-kLead finishes (MMA1(g) only needs buffers MMA2(g-kAcc) freed)
          if (g - kLead >= g0) mma2(g - kLead, g - kLead == g0);
        }
        for (int gp = max(g0, g - kLead); gp < g; ++gp) mma2(gp, gp == g0);
        mma_commit(dzfull);
      }
    }
  } else if (warp >= kEpiWarp0) {
    // two groups of 8 warps take alternate tiles, so each warp has two tiles' time for its
    // 32 rows x 32 classes (the per-tile chain of waits, shuffles and stores overlaps)
    const uint32_t e = warp - kEpiWarp0;
    const uint32_t q = e & 3;              // TMEM lane quadrant (== warp % 4)
    const uint32_t part = (e >> 2) & 1;    // 32-class half of the tile
    const int grp = (int)(e >> 3);         // tiles with g % 2 == grp
    const uint32_t tq = tmem + ((q * 32) << 16);
    const float* __restrict__ bias = P.bias;
    uint8_t* const myC = sC + e * kCB;
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
      const int r0 = rb * kRows + (int)q * 32;  // first row of this warp's dlogits box
      // own tiles: g with g % 2 == grp; lane i holds the bias of class nb+i, one own tile ahead
      int c = ct0 + (((grp - g) % 2 + 2) % 2);
      float bnext = c < ct1 ? __ldg(bias + c * kCT + (int)part * kWarpCls + lane) : 0.f;
      g += c - ct0;
      for (; c < ct1; c += 2, g += 2) {
        const int a = g % kAcc;
        const int nb = c * kCT + (int)part * kWarpCls;
        const float bsrc = bnext;
        mbar_wait(&tfull1[a], (g / kAcc) & 1);
        tc_fence_after();
        if (tr && g < 80 && (e & 7) == 0 && lane == 0) tr[g * 4 + 2] = globaltimer();
        float v[kWarpCls];
        const uint32_t tcol = tq + a * kCT + part * kWarpCls;
        tmem_ld32(tcol, v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < kWarpCls; ++i)
          v[i] = ex2_fast(fmaf(v[i] + __shfl_sync(0xffffffffu, bsrc, i), kLog2e, -l2));
        if (lbl >= nb && lbl < nb + kWarpCls) {
#pragma unroll
          for (int i = 0; i < kWarpCls; ++i)
            if (lbl == nb + i) v[i] -= 1.f;
        }
        uint32_t u[kWarpCls / 2];
#pragma unroll
        for (int i = 0; i < kWarpCls / 2; ++i) {
          v[2 * i] *= sc;
          v[2 * i + 1] *= sc;
          __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
          u[i] = *reinterpret_cast<uint32_t*>(&h);
        }
        // dlogits back into the first 16 columns of this warp's logits slice, for MMA2
        tmem_st16(tcol, u);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&pfull[a]);
        {  // dlogits box (32 rows x 32 classes) -> blocked global via TMA
          if (lane == 0) bulk_wait_read0();  // this warp's previous store (two tiles ago) has read the box
          __syncwarp();
          const uint32_t d = smem_u32(myC) + lane * 64;
#pragma unroll
          for (int j = 0; j < 4; ++j) st_shared_v4(d + j * 16, u[4 * j], u[4 * j + 1], u[4 * j + 2], u[4 * j + 3]);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_4d(&P.tmP, myC, (int)part * kWarpCls, r0 & 63, c, r0 >> 6);
            bulk_commit();
          }
        }
        // next own tile's bias: issued after the proxy fence above (which waits for this
        // thread's outstanding loads), so its latency hides behind the rest of this tile
        if (c + 2 < ct1) bnext = __ldg(bias + nb + 2 * kCT + lane);
        if (P.colpart) {  // bias gradient: column sums of this warp's 32 rows (fp32, pre-rounding)
          const float csum = warp_colsum32(v);
          if (rb * kRows < P.m_valid) P.colpart[(size_t)(rb * 4 + q) * P.classes + nb + lane] = csum;
        }
        if (tr && g < 80 && (e & 7) == 0 && lane == 0) tr[g * 4 + 3] = globaltimer();
      }
      g -= c - ct1;  // back to the item's tile count (the loop stepped past ct1)
      // dZ partial of this (row block, class range): fp32 [cs][row][bott]
      mbar_wait(dzfull, it & 1);
      tc_fence_after();
      const int cols = bott / 4;
      const int dpart = (int)(e >> 2);
      float* dst = P.dzpart + ((size_t)cs * P.dz_rows + row) * bott + dpart * cols;
      for (int c0 = 0; c0 < cols; c0 += 16) {
        float w[16];
        tmem_ld16(acc2 + ((q * 32) << 16) + dpart * cols + c0, w);
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
    if (lane == 0) bulk_wait0();
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

static unsigned long long* g_trace = nullptr;
void ce_grad_dz_set_trace(unsigned long long* buf) { g_trace = buf; }

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
  {  // dlogits, 64x64-blocked [row/64][class/64][64][64]; store box = one warp's 32 rows x 16 classes
    const uint64_t nrb = (a.rows + 63) / 64, ncb = a.classes / 64;
    const uint64_t dims[4] = {64, 64, ncb, nrb};
    const uint64_t strides[3] = {128, 8192, ncb * 8192};
    const uint32_t box[4] = {(uint32_t)kWarpCls, 32, 1, 1};
    rc = make_tmap_4d(&P.tmP, a.dlogits, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, dims, strides, box,
                      CU_TENSOR_MAP_SWIZZLE_NONE);
    if (rc) return rc;
  }
  P.trace = g_trace;
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
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = use_pdl() ? 1 : 0;
  DS_CUDA_TRY(cudaLaunchKernelEx(&cfg, ce_grad_dz_kernel, P));
  return DS_OK;
}

}  // namespace ds
