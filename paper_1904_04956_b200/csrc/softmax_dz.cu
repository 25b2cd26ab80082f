// softmax_dz.cu — fused soft-max gradient and bottleneck input gradient of the
// 32000-way output layer (SURVEY §2.3 K8-bwd + the dZ half of K7-bwd):
//
//   dlogits = (softmax(Z W_o^T + b_o) - onehot(y)) / frames      (bf16, stored)
//   dZ      = dlogits W_o                                        (fp32 partials)
//   db_o    = column sums of dlogits                             (partials)
//
// A CTA pair (tcgen05 cta_group::2) owns two 128-row blocks of Z (one per
// CTA, resident in smem) and a contiguous range of 128-class tiles of W_o.
// Per class tile:
//   MMA1 (pair, M=256 N=128 K=bott): logits of both row blocks into one of two
//     TMEM buffers; B split by classes (CTA r stages classes r*64.. of the tile,
//     K-major [64 classes x bott]).
//   epilogue: two groups of 8 warps per CTA take alternate tiles (group =
//     TMEM buffer); a warp owns 32 rows x 64 classes: dlogits = (softmax -
//     onehot) * scale in fp32 -> bf16 into its 4 KB SW128 smem box, bias-gradient
//     column sums of its rows.  The buffer is released to MMA1 as soon as the
//     logits are read; the box is TMA-stored to the 64x64-blocked global
//     dlogits (read by the dW_o GEMM) and read in place by MMA2.
//   MMA2 (pair, M=256 N=bott K=128): dZ of both row blocks accumulated in TMEM
//     over the class range; A = the group's boxes (4 quadrant boxes stacked =
//     a [128 rows x 64 classes] K-major SW128 block per half), B split by bott
//     (CTA r stages [128 classes x bott/2] MN-major, one stage, own producer warp).
// MMA2 trails MMA1 by two tiles.  Pair MMAs run at full tensor rate (measured:
// M256 N128 K16 in 64 cycles, vs 110 cycles for a single-CTA M128 N<=128
// instruction: tools/micro/mma_rate.cu).  The class ranges of a row block are
// reduced afterwards (op_splitk_bf16, fixed order).
#include "ds_internal.h"
#include "ds_ptx.cuh"
#include "softmax_dz.h"

#include <cstring>

namespace ds {
namespace {

constexpr int kThreads = 640;   // warps 0-3 roles, 4-19 epilogue
constexpr int kEpiWarp0 = 4;
constexpr int kEpiWarps = 16;
constexpr int kRows = 128;      // Z rows per CTA (MMA M per CTA)
constexpr int kCT = 128;        // classes per tile (MMA1 N, MMA2 K)
constexpr int kPartCls = 32;       // classes per epilogue chunk / TMEM hand-off slice
constexpr int kWarpCls = 64;       // classes per epilogue warp and tile (2 halves x 4 lane quadrants per group)
constexpr int kMaxBott = 256;
constexpr int kZB = kRows * kMaxBott * 2;        // 64 KB resident Z block
constexpr int kW1B = (kCT / 2) * kMaxBott * 2;   // 32 KB MMA1 view: 64 classes x bott
constexpr int kW2B = kCT * (kMaxBott / 2) * 2;   // 32 KB MMA2 view: 128 classes x bott/2
constexpr int kCB = 32 * kWarpCls * 2;           // 4 KB dlogits box per epilogue warp (32 rows x 64 classes)
constexpr size_t kSmem = 1024 + kZB + 2 * kW1B + kW2B + kEpiWarps * kCB + 512;
constexpr float kLog2e = 1.4426950408889634f;

__global__ void __launch_bounds__(kThreads, 1) ce_grad_dz_kernel(const __grid_constant__ CeGradDzParams P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sZ = sm;
  uint8_t* sW1 = sZ + kZB;        // [2]
  uint8_t* sW2 = sW1 + 2 * kW1B;  // single stage: loaded while the epilogue runs
  uint8_t* sC = sW2 + kW2B;       // [kEpiWarps] dlogits store boxes (SW128)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sC + kEpiWarps * kCB);
  uint64_t* zfull = bars;          // leader: both CTAs' Z blocks landed
  uint64_t* zempty = zfull + 1;    // every CTA: the item's MMA1s are done with its Z
  uint64_t* w1full = zempty + 1;   // [2] leader
  uint64_t* w1empty = w1full + 2;  // [2] every CTA
  uint64_t* w2full = w1empty + 2;  // leader
  uint64_t* w2empty = w2full + 1;  // every CTA
  uint64_t* tfull = w2empty + 1;   // [2] every CTA: logits ready
  uint64_t* tempty = tfull + 2;    // [2] leader: the 2 x 8 epilogue warps of the buffer read their logits
  uint64_t* pfull = tempty + 2;    // [2] leader: ... and wrote their dlogits boxes (MMA2's A operand)
  uint64_t* bfree = pfull + 2;     // [2] every CTA: MMA2 done reading the group's boxes
  uint64_t* dzfull = bfree + 2;    // every CTA: dZ accumulator complete
  uint64_t* dzempty = dzfull + 1;  // leader: both CTAs drained their dZ accumulators
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dzempty + 1);

  const uint32_t warp = warp_id(), lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int bott = P.bott, nkb = bott / 64;
  const int items = P.n_rbp * P.n_cs;
  // trace: [cta][tile < 80][4]: MMA1 issued, MMA2 issued, epilogue (warp 4) logits seen, epilogue done
  unsigned long long* const tr = P.trace ? P.trace + (size_t)blockIdx.x * 80 * 4 : nullptr;

  if (warp == 1 && lane == 0) {
    mbar_init(zfull, 1);
    mbar_init(zempty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&w1full[i], 1);
      mbar_init(&w1empty[i], 1);
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], kEpiWarps);  // 8 warps per CTA x 2 CTAs
      mbar_init(&pfull[i], kEpiWarps);
      mbar_init(&bfree[i], 1);
    }
    mbar_init(w2full, 1);
    mbar_init(w2empty, 1);
    mbar_init(dzfull, 1);
    mbar_init(dzempty, 2 * kEpiWarps);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_pair(tmem_slot, 512);
  tc_fence_before();
  cluster_sync_all();  // barriers of both CTAs initialised before any remote arrive / complete_tx
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t acc2 = tmem + 2 * kCT;
  griddep_wait();  // lse / labels come from the immediately preceding kernels
  griddep_launch();

  if (warp == 0) {
    if (elect_one()) {
      tma_prefetch_desc(&P.tmZ);
      tma_prefetch_desc(&P.tmW1);
      tma_prefetch_desc(&P.tmW2);
      tma_prefetch_desc(&P.tmP);
      const uint32_t zfull_c = mapa_shared(smem_u32(zfull), 0);
      const uint32_t w1full_c = mapa_shared(smem_u32(w1full), 0);
      int g = 0, it = 0;  // global class-tile counter, item counter
      for (int item = pair; item < items; item += npairs, ++it) {
        const int rbp = item % P.n_rbp, cs = item / P.n_rbp;
        const int ct0 = cs * P.ct_per, ct1 = min(P.n_ct, ct0 + P.ct_per);
        mbar_wait(zempty, (it & 1) ^ 1);
        if (leader) mbar_arrive_expect_tx(zfull, 2 * kRows * bott * 2);
        for (int kb = 0; kb < nkb; ++kb)
          tma_load_2d_pair(sZ + kb * 16384, &P.tmZ, zfull_c, kb * 64, (2 * rbp + (int)rank) * kRows);
        for (int ct = ct0; ct < ct1; ++ct, ++g) {
          const int s = g & 1;
          const uint32_t ph = ((g >> 1) & 1) ^ 1;
          // MMA1 view: classes ct*128 + rank*64 .., all bott (K-major 64 x 64 blocks)
          mbar_wait(&w1empty[s], ph);
          if (leader) mbar_arrive_expect_tx(&w1full[s], 2 * (kCT / 2) * bott * 2);
          for (int kb = 0; kb < nkb; ++kb)
            tma_load_2d_pair(sW1 + s * kW1B + kb * 8192, &P.tmW1, w1full_c + s * 8, kb * 64, ct * kCT + (int)rank * 64);
        }
      }
    }
  } else if (warp == 3) {
    if (elect_one()) {  // MMA2 view producer: all 128 classes of the tile, bott rank*bott/2 .. (MN-major 128 x 64)
      const uint32_t w2full_c = mapa_shared(smem_u32(w2full), 0);
      int g = 0;
      for (int item = pair; item < items; item += npairs) {
        const int cs = item / P.n_rbp;
        const int ct0 = cs * P.ct_per, ct1 = min(P.n_ct, ct0 + P.ct_per);
        for (int ct = ct0; ct < ct1; ++ct, ++g) {
          mbar_wait(w2empty, (g & 1) ^ 1);  // MMA2 of the previous tile is done with the stage
          if (leader) mbar_arrive_expect_tx(w2full, 2 * kCT * (bott / 2) * 2);
          for (int j = 0; j < nkb / 2; ++j)
            tma_load_2d_pair(sW2 + j * 16384, &P.tmW2, w2full_c, (int)rank * (bott / 2) + j * 64, ct * kCT);
        }
      }
    }
  } else if (warp == 1) {
    if (leader && elect_one()) {
      const uint32_t id1 = idesc_bf16_f32(2 * kRows, kCT, 0, 0);
      const uint32_t id2 = idesc_bf16_f32(2 * kRows, bott, 0, 1);
      const uint32_t zb = smem_u32(sZ), w1b = smem_u32(sW1), w2b = smem_u32(sW2), cb = smem_u32(sC);
      int g = 0, it = 0;
      auto mma2 = [&](int gp, bool first) {  // dZ += dlogits(gp) W_o(gp), dlogits from TMEM
        const int s = gp & 1;
        mbar_wait_acq_cluster(&pfull[s], (gp >> 1) & 1);
        mbar_wait(w2full, gp & 1);
        tc_fence_after();
        if (tr && gp < 80) tr[gp * 4 + 1] = globaltimer();
#pragma unroll
        for (int kk = 0; kk < kCT / 16; ++kk) {
          // A = the group's dlogits boxes: per 64-class half, 4 quadrant boxes of [32 rows x 128 B]
          // stacked = a [128 rows x 64 classes] K-major SW128 block
          const uint64_t ad = smem_desc_sw128(cb + s * 8 * kCB + (kk >> 2) * 4 * kCB + (kk & 3) * 32, 16, 1024);
          const uint64_t bd = smem_desc_sw128(w2b + kk * 2048, 16384, 1024);
          mma_bf16_ss_pair(acc2, ad, bd, id2, (!first || kk) ? 1u : 0u);
        }
        mma_commit_pair_mc(&bfree[s], 0x3);
        mma_commit_pair_mc(w2empty, 0x3);
      };
      for (int item = pair; item < items; item += npairs, ++it) {
        const int cs = item / P.n_rbp;
        const int ct0 = cs * P.ct_per, ct1 = min(P.n_ct, ct0 + P.ct_per);
        mbar_wait(zfull, it & 1);
        mbar_wait_acq_cluster(dzempty, (it & 1) ^ 1);  // previous item's dZ drained by both CTAs
        tc_fence_after();
        const int g0 = g;
        for (int ct = ct0; ct < ct1; ++ct, ++g) {
          const int s = g & 1;
          mbar_wait(&w1full[s], (g >> 1) & 1);
          mbar_wait_acq_cluster(&tempty[s], ((g >> 1) & 1) ^ 1);  // the epilogue of tile g-2 read its logits
          tc_fence_after();
          if (tr && g < 80) tr[g * 4 + 0] = globaltimer();
#pragma unroll 1
          for (int kk = 0; kk < bott / 16; ++kk) {
            const uint64_t ad = smem_desc_sw128(zb + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
            const uint64_t bd = smem_desc_sw128(w1b + s * kW1B + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024);
            mma_bf16_ss_pair(tmem + s * kCT, ad, bd, id1, kk ? 1u : 0u);
          }
          mma_commit_pair_mc(&tfull[s], 0x3);
          mma_commit_pair_mc(&w1empty[s], 0x3);
          if (ct == ct1 - 1) mma_commit_pair_mc(zempty, 0x3);
          // MMA2 trails MMA1 by two tiles: the issuer never blocks on a tile's epilogue
          // before the next tile's logits are queued
          if (g - 2 >= g0) mma2(g - 2, g - 2 == g0);
        }
        for (int gp = max(g0, g - 2); gp < g; ++gp) mma2(gp, gp == g0);
        mma_commit_pair_mc(dzfull, 0x3);
      }
    }
  } else if (warp >= kEpiWarp0) {
    // two groups of 8 warps take alternate tiles (group = TMEM buffer), so one group's TMEM
    // reads and exponentials overlap the other's stores and column sums
    const uint32_t e = warp - kEpiWarp0;
    const uint32_t q = e & 3;            // TMEM lane quadrant (== warp % 4)
    const uint32_t half = (e >> 2) & 1;  // 64-class half of the tile
    const int grp = (int)(e >> 3);       // tiles with g % 2 == grp
    const uint32_t tq = tmem + ((q * 32) << 16);
    const float* __restrict__ bias = P.bias;
    uint8_t* const myC = sC + e * kCB;
    const uint32_t pfull_c = mapa_shared(smem_u32(pfull), 0);
    const uint32_t tempty_c = mapa_shared(smem_u32(tempty), 0);
    int own = 0;  // own tiles processed (box reuse parity)
    const uint32_t dzempty_c = mapa_shared(smem_u32(dzempty), 0);
    int g = 0, it = 0;
    for (int item = pair; item < items; item += npairs, ++it) {
      const int rbp = item % P.n_rbp, cs = item / P.n_rbp;
      const int rb = 2 * rbp + (int)rank;
      const int ct0 = cs * P.ct_per, ct1 = min(P.n_ct, ct0 + P.ct_per);
      const int row = rb * kRows + (int)(q * 32 + lane);
      const bool row_ok = row < P.m_valid;
      const int lbl = row_ok ? P.labels[row] : -1;
      const float l2 = row_ok ? P.lse[row] * kLog2e : 0.f;
      const float sc = (row_ok && lbl >= 0) ? P.scale : 0.f;
      // (p - onehot) * sc with p * sc = 2^(x log2e - lse log2e + log2 sc) * 2^(b log2e): one FFMA2
      // per class pair before the exponentials, one FMUL2 by the classes' exp(bias) after
      const float nl2 = sc > 0.f ? log2f(sc) - l2 : -INFINITY;
      const int r0 = rb * kRows + (int)q * 32;  // first row of this warp's dlogits box
      // own tiles: g % 2 == grp; lane i holds the bias of classes nb+i and nb+32+i, one own tile ahead
      int c = ct0 + (((grp - g) % 2 + 2) % 2);
      g += c - ct0;
      float bn0 = 0.f, bn1 = 0.f;
      if (c < ct1) {
        bn0 = __ldg(bias + c * kCT + (int)half * kWarpCls + lane);
        bn1 = __ldg(bias + c * kCT + (int)half * kWarpCls + kPartCls + lane);
      }
      for (; c < ct1; c += 2, g += 2) {
        const int s = g & 1;
        const int nb = c * kCT + (int)half * kWarpCls;
        const float eb0 = ex2_fast(bn0 * kLog2e), eb1 = ex2_fast(bn1 * kLog2e);
        mbar_wait(&tfull[s], (g >> 1) & 1);
        tc_fence_after();
        if (tr && g < 80 && (e & 7) == 0 && lane == 0) tr[g * 4 + 2] = globaltimer();
        const bool reuse = own > 0;
        const uint32_t reuse_phase = (uint32_t)(own - 1) & 1;
        ++own;
        const uint32_t tcol0 = tq + s * kCT + half * kWarpCls;
        float v[kPartCls];
        tmem_ld32(tcol0, v);
        tmem_ld_wait();
#pragma unroll 1
        for (int k = 0; k < 2; ++k) {  // two 32-class chunks
          const int nk = nb + k * kPartCls;
          const float ebsrc = k ? eb1 : eb0;
#pragma unroll
          for (int i = 0; i < kPartCls; i += 2) {
            float a0, a1;
            ffma2(a0, a1, v[i], v[i + 1], kLog2e, kLog2e, nl2, nl2);
            fmul2(v[i], v[i + 1], ex2_fast(a0), ex2_fast(a1), __shfl_sync(0xffffffffu, ebsrc, i),
                  __shfl_sync(0xffffffffu, ebsrc, i + 1));
          }
          if (lbl >= nk && lbl < nk + kPartCls) {
#pragma unroll
            for (int i = 0; i < kPartCls; ++i)
              if (lbl == nk + i) v[i] -= sc;
          }
          uint32_t u[kPartCls / 2];
#pragma unroll
          for (int i = 0; i < kPartCls / 2; ++i) {
            __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
            u[i] = *reinterpret_cast<uint32_t*>(&h);
          }
          if (k == 0) {  // second chunk's logits into v (dead now): the TMEM buffer is then free
                         // for MMA1 of tile g + 2 before this chunk's box wait and stores
            tmem_ld32(tcol0 + kPartCls, v);
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
              if (leader)
                mbar_arrive(&tempty[s]);
              else
                mbar_arrive_remote(tempty_c + s * 8);
            }
          }
          // dlogits into the box (row = lane, 128-byte rows, 128-byte swizzle): TMA-stored to the
          // blocked global dlogits and read in place by MMA2 as its A operand
          if (k == 0) {  // box free: this warp's previous store has read it and MMA2 of the
                         // previous own tile is done (waited here, after the first chunk's math)
            if (lane == 0) bulk_wait_read0();
            if (reuse) mbar_wait(&bfree[s], reuse_phase);
            __syncwarp();
          }
          const uint32_t d = smem_u32(myC) + lane * 128;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t chunk = (uint32_t)(k * 4 + j);
            st_shared_v4(d + ((chunk ^ (lane & 7)) << 4), u[4 * j], u[4 * j + 1], u[4 * j + 2], u[4 * j + 3]);
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_4d(&P.tmP, myC, 0, r0 & 63, nb >> 6, r0 >> 6);
          bulk_commit();
          if (leader)
            mbar_arrive(&pfull[s]);
          else
            mbar_arrive_remote(pfull_c + s * 8);
        }
        if (P.colpart && rb * kRows < P.m_valid) {
          // bias gradient: column sums of the box as stored (bf16 dlogits, the values dW_o and
          // dZ use), read back while the TMA store and MMA2 read it too: lane = 16-byte column
          // chunk (8 classes) x row quarter, eight conflict-free 128-byte row reads per quarter
          // warp, then two shuffle steps over the quarters
          const uint32_t c8 = lane & 7, rq = lane >> 3, bx = smem_u32(myC);
          float cs[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) cs[j] = 0.f;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const uint32_t r = rq + 4 * i;
            const uint4 w = ld_shared_v4(bx + r * 128 + ((c8 ^ (r & 7)) << 4));
            const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              cs[2 * j] += __uint_as_float(ww[j] << 16);
              cs[2 * j + 1] += __uint_as_float(ww[j] & 0xffff0000u);
            }
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            cs[j] += __shfl_xor_sync(0xffffffffu, cs[j], 8);
            cs[j] += __shfl_xor_sync(0xffffffffu, cs[j], 16);
          }
          if (lane < 8) {
            float4* cp = reinterpret_cast<float4*>(P.colpart + (size_t)(rb * 4 + q) * P.classes + nb + 8 * c8);
            cp[0] = make_float4(cs[0], cs[1], cs[2], cs[3]);
            cp[1] = make_float4(cs[4], cs[5], cs[6], cs[7]);
          }
        }
        if (c + 2 < ct1) {  // next own tile's bias (after the proxy fence, which waits for loads in flight)
          bn0 = __ldg(bias + nb + 2 * kCT + lane);
          bn1 = __ldg(bias + nb + 2 * kCT + kPartCls + lane);
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
      __syncwarp();
      if (lane == 0) {
        if (leader)
          mbar_arrive(dzempty);
        else
          mbar_arrive_remote(dzempty_c);
      }
    }
    if (lane == 0) bulk_wait0();
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // neither CTA leaves (or frees TMEM) while the pair is still working
  tc_fence_after();
  if (warp == 2) tmem_dealloc_pair(tmem, 512);
}

// ---------------------------------------------------------------------------
// Soft-max statistics (loss pass) on the same CTA-pair skeleton: MMA1 only
// (pair M256 N128 K=bott into four TMEM buffers, W_o MMA1 view through a
// 4-stage ring).  Four epilogue groups of 4 warps (one per TMEM lane quadrant)
// take every fourth tile, offset by one MMA each; a warp keeps a running
// (max, sum 2^(x - max)) for its 32 rows over 128 classes per own tile and
// releases the buffer as soon as its logits are read.  The four partials of a
// row are merged through shared memory once per item.  (Half the exponentials
// as an FMA-pipe polynomial measured slower: the epilogue is issue-bound.)
namespace stp {
constexpr int kWStages = 4;
constexpr int kAcc = 4;  // TMEM logits buffers = epilogue groups
constexpr size_t kSmem = 1024 + kZB + kWStages * kW1B + 4 * kRows * 8 + 256;
}  // namespace stp

__global__ void __launch_bounds__(kThreads, 1) ce_stats_kernel(const __grid_constant__ CeStatsParams P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sZ = sm;
  uint8_t* sW1 = sZ + kZB;  // [kWStages]
  float2* sPart = reinterpret_cast<float2*>(sW1 + stp::kWStages * kW1B);  // [4 partials][128 rows]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sPart + 4 * kRows);
  uint64_t* zfull = bars;
  uint64_t* zempty = zfull + 1;
  uint64_t* w1full = zempty + 1;              // [kWStages] leader
  uint64_t* w1empty = w1full + stp::kWStages;  // [kWStages] every CTA
  uint64_t* tfull = w1empty + stp::kWStages;   // [kAcc] every CTA
  uint64_t* tempty = tfull + stp::kAcc;        // [kAcc] leader: the buffer's 2 x 4 epilogue warps read it
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + stp::kAcc);

  const uint32_t warp = warp_id(), lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int bott = P.bott, nkb = bott / 64;
  const int items = P.n_rbp * P.n_cs;
  if (warp == 1 && lane == 0) {
    mbar_init(zfull, 1);
    mbar_init(zempty, 1);
    for (int i = 0; i < stp::kWStages; ++i) {
      mbar_init(&w1full[i], 1);
      mbar_init(&w1empty[i], 1);
    }
    for (int i = 0; i < stp::kAcc; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 2 * 4);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_pair(tmem_slot, stp::kAcc * kCT);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  griddep_wait();  // Z comes from the preceding bottleneck GEMM
  griddep_launch();

  if (warp == 0) {
    if (elect_one()) {
      tma_prefetch_desc(&P.tmZ);
      tma_prefetch_desc(&P.tmW1);
      const uint32_t zfull_c = mapa_shared(smem_u32(zfull), 0);
      const uint32_t w1full_c = mapa_shared(smem_u32(w1full), 0);
      int g = 0, it = 0;
      for (int item = pair; item < items; item += npairs, ++it) {
        const int rbp = item % P.n_rbp, cs = item / P.n_rbp;
        const int ct0 = cs * P.ct_per, ct1 = min(P.n_ct, ct0 + P.ct_per);
        mbar_wait(zempty, (it & 1) ^ 1);
        if (leader) mbar_arrive_expect_tx(zfull, 2 * kRows * bott * 2);
        for (int kb = 0; kb < nkb; ++kb)
          tma_load_2d_pair(sZ + kb * 16384, &P.tmZ, zfull_c, kb * 64, (2 * rbp + (int)rank) * kRows);
        for (int ct = ct0; ct < ct1; ++ct, ++g) {
          const int st = g % stp::kWStages;
          mbar_wait(&w1empty[st], ((g / stp::kWStages) & 1) ^ 1);
          if (leader) mbar_arrive_expect_tx(&w1full[st], 2 * (kCT / 2) * bott * 2);
          for (int kb = 0; kb < nkb; ++kb)
            tma_load_2d_pair(sW1 + st * kW1B + kb * 8192, &P.tmW1, w1full_c + st * 8, kb * 64,
                             ct * kCT + (int)rank * 64);
        }
      }
    }
  } else if (warp == 1) {
    if (leader && elect_one()) {
      const uint32_t id1 = idesc_bf16_f32(2 * kRows, kCT, 0, 0);
      const uint32_t zb = smem_u32(sZ), w1b = smem_u32(sW1);
      int g = 0, it = 0;
      for (int item = pair; item < items; item += npairs, ++it) {
        const int cs = item / P.n_rbp;
        const int ct0 = cs * P.ct_per, ct1 = min(P.n_ct, ct0 + P.ct_per);
        mbar_wait(zfull, it & 1);
        tc_fence_after();
        for (int ct = ct0; ct < ct1; ++ct, ++g) {
          const int st = g % stp::kWStages, s = g % stp::kAcc;
          mbar_wait(&w1full[st], (g / stp::kWStages) & 1);
          mbar_wait_acq_cluster(&tempty[s], ((g / stp::kAcc) & 1) ^ 1);  // epilogue read tile g-kAcc's logits
          tc_fence_after();
#pragma unroll 1
          for (int kk = 0; kk < bott / 16; ++kk) {
            const uint64_t ad = smem_desc_sw128(zb + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
            const uint64_t bd = smem_desc_sw128(w1b + st * kW1B + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024);
            mma_bf16_ss_pair(tmem + s * kCT, ad, bd, id1, kk ? 1u : 0u);
          }
          mma_commit_pair_mc(&tfull[s], 0x3);
          mma_commit_pair_mc(&w1empty[st], 0x3);
          if (ct == ct1 - 1) mma_commit_pair_mc(zempty, 0x3);
        }
      }
    }
  } else if (warp >= kEpiWarp0) {
    // four groups of 4 warps (one per TMEM lane quadrant) take every fourth tile, one TMEM
    // buffer each: the groups run offset by one MMA, so TMEM reads and exponentials overlap
    const uint32_t e = warp - kEpiWarp0;
    const uint32_t q = e & 3;
    const int grp = (int)(e >> 2);
    const uint32_t tq = tmem + ((q * 32) << 16);
    const uint32_t tempty_c = mapa_shared(smem_u32(tempty), 0);
    const int rloc = (int)(q * 32 + lane);
    int g = 0;
    for (int item = pair; item < items; item += npairs) {
      const int rbp = item % P.n_rbp, cs = item / P.n_rbp;
      const int rb = 2 * rbp + (int)rank;
      const int ct0 = cs * P.ct_per, ct1 = min(P.n_ct, ct0 + P.ct_per);
      const int row = rb * kRows + rloc;
      const bool row_ok = row < P.m_valid;
      const int lbl = row_ok ? P.labels[row] : -1;
      float mx = -INFINITY, se = 0.f, tg = 0.f;
      bool have_t = false;
      int c = ct0 + (((grp - g) % stp::kAcc + stp::kAcc) % stp::kAcc);
      g += c - ct0;
      for (; c < ct1; c += stp::kAcc, g += stp::kAcc) {
        const int s = g % stp::kAcc;
        const int nb = c * kCT;
        float b4[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) b4[j] = __ldg(P.bias_log2 + nb + j * kPartCls + lane);
        mbar_wait(&tfull[s], (g / stp::kAcc) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int k = 0; k < 4; ++k) {
          const int nk = nb + k * kPartCls;
          float bsrc = b4[0];
#pragma unroll
          for (int j = 1; j < 4; ++j)
            if (k == j) bsrc = b4[j];
          float v[kPartCls];
          tmem_ld32(tq + s * kCT + k * kPartCls, v);
          tmem_ld_wait();
          if (k == 3) {  // logits of the tile read: buffer free for MMA1 of tile g + kAcc
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
              if (leader)
                mbar_arrive(&tempty[s]);
              else
                mbar_arrive_remote(tempty_c + s * 8);
            }
          }
          // logits in the log2 domain: one FFMA2 per class pair with the log2(e)-scaled bias
#pragma unroll
          for (int i = 0; i < kPartCls; i += 2)
            ffma2(v[i], v[i + 1], v[i], v[i + 1], kLog2e, kLog2e, __shfl_sync(0xffffffffu, bsrc, i),
                  __shfl_sync(0xffffffffu, bsrc, i + 1));
          float m3[11];
#pragma unroll
          for (int i = 0; i < 10; ++i) m3[i] = fmax3(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
          m3[10] = fmax3(v[30], v[31], mx);
          const float nm = fmax3(fmax3(m3[0], m3[1], m3[2]), fmax3(m3[3], m3[4], m3[5]),
                                 fmax3(fmax3(m3[6], m3[7], m3[8]), m3[9], m3[10]));
          if (lbl >= nk && lbl < nk + kPartCls) {
#pragma unroll
            for (int i = 0; i < kPartCls; ++i)
              if (lbl == nk + i) tg = v[i];
            have_t = true;
          }
          float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
          for (int i = 0; i < kPartCls; i += 4) {
            float a0, a1, a2, a3;
            fadd2(a0, a1, v[i], v[i + 1], -nm, -nm);
            fadd2(a2, a3, v[i + 2], v[i + 3], -nm, -nm);
            fadd2(s0, s1, s0, s1, ex2_fast(a0), ex2_fast(a1));
            fadd2(s2, s3, s2, s3, ex2_fast(a2), ex2_fast(a3));
          }
          se = se * ex2_fast(mx - nm) + ((s0 + s1) + (s2 + s3));
          mx = nm;
        }
      }
      g -= c - ct1;
      if (have_t && row_ok) P.tgt[row] = tg / kLog2e;
      // merge the row's four partials (one per group); natural-log units on output
      sPart[grp * kRows + rloc] = make_float2(mx, se);
      named_bar_sync(1, kEpiWarps * 32);
      if (grp == 0 && row_ok) {
        float M = sPart[rloc].x;
#pragma unroll
        for (int k = 1; k < 4; ++k) M = fmaxf(M, sPart[k * kRows + rloc].x);
        float S = 0.f;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 pk = sPart[k * kRows + rloc];
          if (pk.y > 0.f) S += pk.y * ex2_fast(pk.x - M);
        }
        P.stats[(size_t)cs * P.stats_ld + row] = make_float2(M / kLog2e, S);
      }
      named_bar_sync(1, kEpiWarps * 32);  // sPart reused by the next item
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  if (warp == 2) tmem_dealloc_pair(tmem, stp::kAcc * kCT);
}

}  // namespace

bool ce_grad_dz_supported(int classes, int bott) {
  return classes % kCT == 0 && bott % 128 == 0 && bott <= kMaxBott;
}

// class ranges per row-block pair: about two work items per CTA pair, so the
// persistent pairs finish together
int ce_grad_dz_splits(int rows, int classes, int max_splits) {
  const int n_rbp = (rows + 2 * kRows - 1) / (2 * kRows), n_ct = classes / kCT;
  int s = (2 * (num_sms() / 2)) / n_rbp;
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
  rc = make_tmap_2d(&P.tmW1, a.w, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, a.bott, a.classes, (uint64_t)a.bott * 2, 64,
                    kCT / 2);
  if (rc) return rc;
  rc = make_tmap_2d(&P.tmW2, a.w, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, a.bott, a.classes, (uint64_t)a.bott * 2, 64, kCT);
  if (rc) return rc;
  {  // dlogits, 64x64-blocked [row/64][class/64][64][64]; store box = one warp's 32 rows x 64 classes
    const uint64_t nrb = (a.rows + 63) / 64, ncb = a.classes / 64;
    const uint64_t dims[4] = {64, 64, ncb, nrb};
    const uint64_t strides[3] = {128, 8192, ncb * 8192};
    const uint32_t box[4] = {(uint32_t)kWarpCls, 32, 1, 1};
    rc = make_tmap_4d(&P.tmP, a.dlogits, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, dims, strides, box,
                      CU_TENSOR_MAP_SWIZZLE_128B);
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
  P.n_rbp = (a.rows + 2 * kRows - 1) / (2 * kRows);
  P.n_ct = a.classes / kCT;
  P.n_cs = a.splits;
  P.ct_per = (P.n_ct + a.splits - 1) / a.splits;
  if ((a.splits - 1) * P.ct_per >= P.n_ct) return fail_arg("fused soft-max/dZ: empty class range");
  const int items = P.n_rbp * P.n_cs;
  const int max_pairs = num_sms() / 2;
  const int pairs = items < max_pairs ? items : max_pairs;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = use_pdl(4) ? 2 : 1;
  DS_CUDA_TRY(cudaLaunchKernelEx(&cfg, ce_grad_dz_kernel, P));
  return DS_OK;
}

int ce_stats_launch(const CeStatsArgs& a, cudaStream_t stream) {
  static bool attr_set = false;
  if (!attr_set) {
    DS_CUDA_TRY(cudaFuncSetAttribute(ce_stats_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)stp::kSmem));
    attr_set = true;
  }
  if (!ce_grad_dz_supported(a.classes, a.bott)) return fail_arg("soft-max statistics: unsupported shape");
  CeStatsParams P;
  memset(&P, 0, sizeof(P));
  int rc = make_tmap_2d(&P.tmZ, a.z, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, a.bott, a.rows, (uint64_t)a.bott * 2, 64, kRows);
  if (rc) return rc;
  rc = make_tmap_2d(&P.tmW1, a.w, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, a.bott, a.classes, (uint64_t)a.bott * 2, 64,
                    kCT / 2);
  if (rc) return rc;
  P.bias_log2 = a.bias_log2;
  P.labels = a.labels;
  P.stats = a.stats;
  P.stats_ld = a.stats_ld;
  P.tgt = a.tgt;
  P.bott = a.bott;
  P.classes = a.classes;
  P.m_valid = a.rows;
  P.n_rbp = (a.rows + 2 * kRows - 1) / (2 * kRows);
  P.n_ct = a.classes / kCT;
  P.n_cs = a.splits;
  P.ct_per = (P.n_ct + a.splits - 1) / a.splits;
  if ((a.splits - 1) * P.ct_per >= P.n_ct) return fail_arg("soft-max statistics: empty class range");
  const int items = P.n_rbp * P.n_cs;
  const int max_pairs = num_sms() / 2;
  const int pairs = items < max_pairs ? items : max_pairs;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = stp::kSmem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = use_pdl(4) ? 2 : 1;
  DS_CUDA_TRY(cudaLaunchKernelEx(&cfg, ce_stats_kernel, P));
  return DS_OK;
}

}  // namespace ds
