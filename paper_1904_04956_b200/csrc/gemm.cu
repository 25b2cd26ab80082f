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
// Structure: CTA pairs (2-CTA clusters, tcgen05 cta_group::2), one CTA per
// SM, 640 threads.  A pair owns a 256 x 256 output tile: CTA rank r stages
// rows r*128.. of the A tile and rows r*128.. of the B tile (K-block 64), so
// each SM streams 32 KB per k-block instead of 48 KB and the tensor cores of
// both SMs read the B halves of both (M=256 N=256 K=16 pair MMA).
//   warp 0      : TMA producer (one elected lane, both CTAs), 6-stage ring;
//                 byte counts complete on the leader's (rank 0) barrier
//   warp 1      : tcgen05.mma issuer (leader CTA only, one elected lane)
//   warp 2      : TMEM allocator (512 columns = 2 x 128x256 fp32 accumulators
//                 per CTA, mirrored in the pair)
//   warps 4..19 : epilogue of the CTA's 128 rows, thread = accumulator row
//                 (TMEM lane); warp 4+e takes lane quadrant e%4 and columns
//                 64*(e/4) .. +64
// Pair tiles are walked round-robin over the persistent grid; the two TMEM
// accumulators let the epilogue of tile i overlap the main loop of tile i+1.
#include <algorithm>
#include <cstdlib>
#include <utility>
#include <vector>

#include "ds_internal.h"
#include "ds_ptx.cuh"

namespace ds {

namespace {

constexpr int BM = kGemmBM, BN = kGemmBN, BK = kGemmBK;
constexpr int kStages = 6;
constexpr int kPairM = 2 * BM;             // rows of a pair tile
constexpr int kBHalf = BN / 2;             // B rows staged per CTA
constexpr int kABytes = BM * BK * 2;       // 16 KB
constexpr int kBBytes = kBHalf * BK * 2;   // 16 KB
constexpr int kStageBytes = kABytes + kBBytes;
constexpr int kThreads = 640;  // warps 0-3 roles, 4-19 epilogue (4 lane quadrants x 4 column quarters)
constexpr int kEpiWarp0 = 4;
constexpr uint32_t kTmemCols = 512;
constexpr int kStageC = 32 * 32 * 2;  // per-epilogue-warp bf16 staging box (32 rows x 32 cols, SW64)
constexpr int kEpiWarps = 16;
constexpr int kEpiGroups = 1;  // epilogue warp groups taking alternate tiles (1 or 2; 2 measured slower)
constexpr size_t kSmemBytes = 1024 /*align slack*/ + (size_t)kStages * kStageBytes + kEpiWarps * kStageC + 256;

// trace record: [cta][tile < kTrTiles][kTrFields] (globaltimer ns / clock64 cycles)
constexpr int kTrTiles = 32, kTrFields = 11;
enum { TR_MMA_START, TR_MMA_FULLSTALL, TR_MMA_END, TR_EPI_START, TR_EPI_END, TR_EPI_LAST, TR_PROD_STALL, TR_CTA_START,
       TR_GATE0, TR_GATE1, TR_READY };

struct TileCoord {
  int prob, tm, tn, ks;
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
  const int rest = local / b.p[p].tiles_m;
  c.tn = rest % b.p[p].tiles_n;
  c.ks = rest / b.p[p].tiles_n;
  return c;
}

// the i-th tile of pair `pair` (i < pair_tile_count)
__device__ __forceinline__ int pair_tile_count(const GemmBatch& b, int pair, int npairs) {
  if (b.sched) return b.pstart[pair + 1] - b.pstart[pair];
  return pair < b.total_tiles ? (b.total_tiles - 1 - pair) / npairs + 1 : 0;
}
__device__ __forceinline__ int pair_tile(const GemmBatch& b, int pair, int npairs, int i) {
  return b.sched ? (int)b.order[b.pstart[pair] + i] : pair + i * npairs;
}

// k-block range of split `ks`
__device__ __forceinline__ void kb_range(const GemmProblem& P, int ks, int& kb0, int& kb1) {
  const int nkb = (P.K + BK - 1) / BK;
  const int per = (nkb + P.ksplit - 1) / P.ksplit;
  kb0 = ks * per;
  kb1 = min(nkb, kb0 + per);
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

// Stage this warp's 32 rows x 32 bf16 columns (lane = row) in smem with the
// 64-byte swizzle and TMA-store the box at (col, row0): full 64 B row
// segments reach L2 instead of 16 B pieces of 32 different rows.
__device__ __forceinline__ void store_box_tma(const CUtensorMap* map, uint8_t* stg, const float* v, int col, int row0,
                                              int blk = 0) {
  const uint32_t lane = lane_id();
  if (lane == 0) bulk_wait_read0();  // the previous box has left this buffer
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint4 w;
    uint32_t* u = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __nv_bfloat162 h = __floats2bfloat162_rn(v[8 * j + 2 * i], v[8 * j + 2 * i + 1]);
      u[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    *reinterpret_cast<uint4*>(stg + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4)) = w;
  }
  fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0) {
    if (blk)
      tma_store_4d(map, stg, col & 63, row0 & 63, col >> 6, row0 >> 6);
    else
      tma_store_2d(map, stg, col, row0);
    bulk_commit();
  }
}

__global__ void __launch_bounds__(kThreads, 1) gemm_kernel(const __grid_constant__ GemmBatch batch) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* cstage = smem + kStages * kStageBytes;  // [kEpiWarps][32x32 bf16]
  uint64_t* full = reinterpret_cast<uint64_t*>(cstage + kEpiWarps * kStageC);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t crank = cluster_ctarank();  // 0 = leader (issues the pair MMAs)
  const bool leader = crank == 0;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  unsigned long long* const trace = batch.trace ? batch.trace + (size_t)blockIdx.x * kTrTiles * kTrFields : nullptr;
  if (trace && threadIdx.x == 0) trace[TR_CTA_START] = globaltimer();

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
      mbar_init(&tempty[a], 2 * kEpiWarps / kEpiGroups);  // the accumulator's epilogue warps of both CTAs
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_pair(tmem_slot, kTmemCols);
  tc_fence_before();
  cluster_sync_all();  // barriers of both CTAs initialised before any remote arrive / complete_tx
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // prologue done: wait for the predecessor's outputs, then let the next kernel start its own
  // (b_early: the producer first prefetches the B operand of its first tile —
  // never written by the predecessor kernel — and waits afterwards)
  if (!(batch.b_early && warp == 0)) griddep_wait();
  griddep_launch();


  if (warp == 0) {
    if (elect_one()) {
      // ---------------- TMA producer (both CTAs) ----------------
      const uint32_t full_c = mapa_shared(smem_u32(full), 0);  // leader's full[0]
      int stage = 0;
      uint32_t phase = 0;
      const int ntl = pair_tile_count(batch, pair, npairs);
      int pre = 0;  // stages of tile 0 whose B load (and expect_tx) was issued before griddep_wait
      if (batch.b_early) {
        if (ntl > 0) {
          TileCoord tc = locate(batch, pair_tile(batch, pair, npairs, 0));
          const GemmProblem& P = batch.p[tc.prob];
          const int n0 = tc.tn * BN + (int)crank * kBHalf;
          int kb0, kb1;
          kb_range(P, tc.ks, kb0, kb1);
          pre = min(kStages, kb1 - kb0);
          for (int s = 0; s < pre; ++s) {
            uint8_t* sB = smem + s * kStageBytes + kABytes;
            if (leader) mbar_arrive_expect_tx(&full[s], 2 * kStageBytes);
            const uint32_t bar = full_c + s * 8;
            const int k0 = (kb0 + s) * BK;
            if (!P.b_mn) {
              tma_load_2d_pair(sB, &P.tmB, bar, k0, n0);
            } else {
#pragma unroll
              for (int j = 0; j < kBHalf / 64; ++j) tma_load_2d_pair(sB + j * 8192, &P.tmB, bar, n0 + 64 * j, k0);
            }
          }
        }
        griddep_wait();
      }
      for (int ti = 0; ti < ntl; ++ti) {
        TileCoord tc = locate(batch, pair_tile(batch, pair, npairs, ti));
        const GemmProblem& P = batch.p[tc.prob];
        const int m0 = tc.tm * kPairM + (int)crank * BM, n0 = tc.tn * BN + (int)crank * kBHalf;
        int kb0, kb1;
        kb_range(P, tc.ks, kb0, kb1);
        if (P.gate) {  // this CTA's A rows: every time step they cover has completed upstream
          if (trace && ti < kTrTiles) trace[ti * kTrFields + TR_GATE0] = globaltimer();
          const int t0 = m0 / P.gate_rows;
          int t1 = (m0 + BM - 1) / P.gate_rows;
          if (t1 > P.gate_T - 1) t1 = P.gate_T - 1;
          for (int t = t0; t <= t1; ++t) {
            uint32_t n = 0;
            uint64_t g0 = 0;
            while ((int32_t)(ld_acquire_gpu(P.gate + t) - P.gate_target) < 0) {
              if ((++n & 1023u) == 0) {  // 2 s guard: a recurrence that never completes the step
                if (P.gate_err && (*reinterpret_cast<volatile int*>(P.gate_err) & 8)) break;  // step failed
                const uint64_t now = globaltimer();
                if (!g0) g0 = now;
                else if (now - g0 > 2000000000ull) {
                  if (P.gate_err) atomicOr(P.gate_err, 8);
                  break;
                }
              }
            }
          }
          fence_proxy_async_global();
          if (trace && ti < kTrTiles) trace[ti * kTrFields + TR_GATE1] = globaltimer();
        }
        long long pst = 0;
        for (int kb = kb0; kb < kb1; ++kb) {
          const bool early = ti == 0 && kb - kb0 < pre;
          const long long c0 = trace ? clock64() : 0;
          mbar_wait(&empty[stage], phase ^ 1);  // the pair MMA that read this stage (both CTAs) is done
          if (trace) pst += clock64() - c0;
          uint8_t* sA = smem + stage * kStageBytes;
          uint8_t* sB = sA + kABytes;
          if (leader && !early) mbar_arrive_expect_tx(&full[stage], 2 * kStageBytes);
          const uint32_t bar = full_c + stage * 8;
          const int k0 = kb * BK;
          if (P.a_blk) {  // 64x64-blocked A: whole 8 KB blocks (box spans 2 row blocks when K-major)
            if (!P.a_mn) {
              tma_load_4d_pair(sA, &P.tmA, bar, 0, 0, k0 >> 6, m0 >> 6);
            } else {
#pragma unroll
              for (int j = 0; j < BM / 64; ++j)
                tma_load_4d_pair(sA + j * 8192, &P.tmA, bar, 0, 0, (m0 >> 6) + j, k0 >> 6);
            }
          } else if (!P.a_mn) {
            tma_load_2d_pair(sA, &P.tmA, bar, k0, m0);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j) tma_load_2d_pair(sA + j * 8192, &P.tmA, bar, m0 + 64 * j, k0);
          }
          if (early) {
          } else if (!P.b_mn) {
            tma_load_2d_pair(sB, &P.tmB, bar, k0, n0);
          } else {
#pragma unroll
            for (int j = 0; j < kBHalf / 64; ++j) tma_load_2d_pair(sB + j * 8192, &P.tmB, bar, n0 + 64 * j, k0);
          }
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (trace && ti < kTrTiles) trace[ti * kTrFields + TR_PROD_STALL] = pst;
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader CTA) ----------------
    if (leader) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      const int ntl = pair_tile_count(batch, pair, npairs);
      for (int ti = 0; ti < ntl; ++ti, ++it) {
        TileCoord tc = locate(batch, pair_tile(batch, pair, npairs, ti));
        const GemmProblem& P = batch.p[tc.prob];
        int kb0, kb1;
        kb_range(P, tc.ks, kb0, kb1);
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        const uint32_t idesc = idesc_bf16_f32(kPairM, BN, P.a_mn, P.b_mn);
        mbar_wait_acq_cluster(&tempty[acc], acc_phase ^ 1);  // both CTAs' epilogues drained it
        tc_fence_after();
        const bool tr = trace && ti < kTrTiles;
        if (tr && lane == 0) trace[ti * kTrFields + TR_MMA_START] = globaltimer();
        long long fst = 0;
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          const long long c0 = tr ? clock64() : 0;
          mbar_wait(&full[stage], phase);
          if (tr) fst += clock64() - c0;
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
              mma_bf16_ss_pair(d_tmem, ad, bd, idesc, (kb != kb0) || (k != 0));
            }
            mma_commit_pair_mc(&empty[stage], 0x3);
            if (kb == kb1 - 1) mma_commit_pair_mc(&tfull[acc], 0x3);
          }
          __syncwarp();
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (tr && lane == 0) {
          trace[ti * kTrFields + TR_MMA_END] = globaltimer();
          trace[ti * kTrFields + TR_MMA_FULLSTALL] = fst;
        }
      }
    }
  } else if (warp >= kEpiWarp0) {
    // ---------------- epilogue ----------------
    const uint32_t e = warp - kEpiWarp0;
    const uint32_t q = e & 3;     // TMEM lane quadrant (== warp % 4)
    // kEpiGroups groups of warps take alternate tiles (group = accumulator), so one group's TMEM
    // reads and exponentials overlap the other's stores instead of every warp hitting the same
    // phase at once
    constexpr int kParts = 4 / kEpiGroups;         // column parts of the 256-wide tile
    constexpr int kCols = BN / kParts;             // columns per thread
    const uint32_t part = (e >> 2) % kParts;
    const int grp = (int)(e >> 2) / kParts;
    constexpr float kLog2e = 1.4426950408889634f;
    const uint32_t tempty_c = mapa_shared(smem_u32(tempty), 0);
    int it = 0;
    const int ntl = pair_tile_count(batch, pair, npairs);
    for (int ti = 0; ti < ntl; ++ti, ++it) {
      if ((it & 1) % kEpiGroups != grp) continue;  // kEpiGroups == 2: accumulator it & 1 is group grp's
      TileCoord tc = locate(batch, pair_tile(batch, pair, npairs, ti));
      const GemmProblem& P = batch.p[tc.prob];
      const int rt = tc.tm * 2 + (int)crank;  // 128-row tile of this CTA
      // problem fields into registers once per tile (P is indexed dynamically)
      const int epi = P.epi, n_valid = P.n_valid;
      const float* __restrict__ bias = P.bias;
      const float scale = P.scale;
      const long long ldo = P.ldo;
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const int row = rt * BM + q * 32 + lane;
      const int n0 = tc.tn * BN + part * kCols;
      const bool row_ok = row < P.m_valid;
      const bool full_cols = n0 + kCols <= n_valid;
      // per-row epilogue inputs, fetched before the accumulator wait
      int lbl = -1;
      float l = 0.f;
      if (epi >= EPI_CE_STATS && row_ok) {
        lbl = P.labels[row];
        if (epi == EPI_CE_GRAD) l = P.lse[row];
      }
      // the warp's 64 bias values, lane i holding columns n0+i and n0+32+i (broadcast by
      // shuffles below): the loads' latency hides behind the accumulator wait
      float bias_r[kCols / 32];
#pragma unroll
      for (int j = 0; j < kCols / 32; ++j) {
        bias_r[j] = 0.f;
        if (bias && epi != EPI_CE_GRAD && n0 + 32 * j + (int)lane < n_valid) bias_r[j] = __ldg(bias + n0 + 32 * j + lane);
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      if (trace && ti < kTrTiles && e == 0 && lane == 0) trace[ti * kTrFields + TR_EPI_START] = globaltimer();
      const uint32_t t_row = tmem_base + acc * BN + ((q * 32) << 16) + part * kCols;

      if (epi == EPI_CE_STATS) {
        // online (max, sum exp) over this thread's 64 columns, log2 domain
        float mx = -INFINITY, se = 0.f, tg = 0.f;
        bool have_t = false;
        float vbuf[2][32];
        tmem_ld32(t_row, vbuf[0]);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < kCols; c += 32) {
          float* v = vbuf[(c >> 5) & 1];
          if (c + 32 < kCols) tmem_ld32(t_row + c + 32, vbuf[((c >> 5) + 1) & 1]);  // in flight meanwhile
          const int nb = n0 + c;
          // logits in the log2 domain: one FFMA with the log2(e)-scaled bias
          float cm = -INFINITY;
          const float bsrc = bias_r[c >> 5];
          if (full_cols) {
            float m8[8];
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              v[i] = fmaf(v[i], kLog2e, __shfl_sync(0xffffffffu, bsrc, i));
              v[i + 1] = fmaf(v[i + 1], kLog2e, __shfl_sync(0xffffffffu, bsrc, i + 1));
              v[i + 2] = fmaf(v[i + 2], kLog2e, __shfl_sync(0xffffffffu, bsrc, i + 2));
              v[i + 3] = fmaf(v[i + 3], kLog2e, __shfl_sync(0xffffffffu, bsrc, i + 3));
              m8[i >> 2] = fmaxf(fmaxf(v[i], v[i + 1]), fmaxf(v[i + 2], v[i + 3]));
            }
            // max as a tree (independent FMNMX) instead of a 32-long chain
            cm = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])), fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const bool in = nb + i < n_valid;
              const float bv = __shfl_sync(0xffffffffu, bsrc, i);
              v[i] = in ? fmaf(v[i], kLog2e, bv) : -INFINITY;
              cm = fmaxf(cm, v[i]);
            }
          }
          if (lbl >= nb && lbl < nb + 32) {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (lbl == nb + i) tg = v[i];
            have_t = true;
          }
          if (cm > -INFINITY) {
            const float nm = fmaxf(mx, cm);
            float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;  // independent chains
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              s0 += ex2_fast(v[i] - nm);
              s1 += ex2_fast(v[i + 1] - nm);
              s2 += ex2_fast(v[i + 2] - nm);
              s3 += ex2_fast(v[i + 3] - nm);
            }
            se = se * ex2_fast(mx - nm) + ((s0 + s1) + (s2 + s3));
            mx = nm;
          }
          if (c + 32 < kCols) tmem_ld_wait();
        }
        if (row_ok) {
          // stats in natural-log units: max, sum exp(x - max)
          P.stats[(size_t)(tc.tn * kParts + part) * P.stats_ld + row] = make_float2(mx / kLog2e, se);
          if (have_t) P.tgt[row] = tg / kLog2e;
        }
      } else if (epi == EPI_CE_GRAD) {
        __nv_bfloat16* orow = reinterpret_cast<__nv_bfloat16*>(P.out) + (size_t)row * ldo;
        float* colpart = P.colpart;
        const float l2 = l * kLog2e;
#pragma unroll 1
        for (int c = 0; c < kCols; c += 32) {
          float v[32];
          tmem_ld32(t_row + c, v);
          tmem_ld_wait();
          const int nb = n0 + c;
          if (nb >= n_valid) continue;
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 bb = bias ? __ldg(reinterpret_cast<const float4*>(bias + nb + i))
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
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
          const float sc = row_ok ? scale : 0.f;
          if (nb + 32 <= n_valid) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] *= sc;
          } else {  // last column tile: classes >= n_valid carry no probability (and no store)
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = nb + i < n_valid ? v[i] * sc : 0.f;
          }
          if (P.c_tma) {
            store_box_tma(&P.tmC, cstage + e * kStageC, v, nb, rt * BM + q * 32, P.c_blk);
          } else if (row_ok) {
            store_bf16x16(orow + nb, v);
            if (nb + 16 < n_valid) store_bf16x16(orow + nb + 16, v + 16);  // n_valid is a multiple of 16
          }
          if (colpart && rt * BM < P.m_valid) {  // bias gradient: column sums of this warp's 32 rows (fp32, pre-rounding)
            const float cs = warp_colsum32(v, lane);
            if (nb + (int)lane < n_valid) colpart[(size_t)(rt * 4 + q) * n_valid + nb + lane] = cs;
          }
        }
      } else if (epi == EPI_BF16) {
        __nv_bfloat16* orow = reinterpret_cast<__nv_bfloat16*>(P.out) + (size_t)row * ldo;
#pragma unroll 1
        for (int c = 0; c < kCols; c += 32) {
          float v[32];
          tmem_ld32(t_row + c, v);
          tmem_ld_wait();
          const int nb = n0 + c;
          if (nb >= n_valid) continue;
          if (bias) {
            float bsrc = bias_r[0];
#pragma unroll
            for (int j = 1; j < kCols / 32; ++j)
              if (c == 32 * j) bsrc = bias_r[j];  // selects: no dynamic register indexing
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] += __shfl_sync(0xffffffffu, bsrc, i);
          }
          if (P.c_tma) {
            store_box_tma(&P.tmC, cstage + e * kStageC, v, nb, rt * BM + q * 32);
          } else if (row_ok) {
            store_bf16x16(orow + nb, v);
            if (nb + 16 < n_valid) store_bf16x16(orow + nb + 16, v + 16);
          }
        }
        if (P.ready && rt * BM + (int)q * 32 < P.m_valid) {  // output block stored: count it
          __syncwarp();
          if (lane == 0) {
            if (P.c_tma) bulk_wait0();
            fence_proxy_async_global();  // async-proxy (TMA) stores before the generic release
            const int r0 = rt * BM + (int)q * 32;
            red_release_gpu_add(P.ready + ((r0 / P.ready_rows) * (P.N / P.ready_cols) + n0 / P.ready_cols) * P.ready_stride,
                                1u);
            if (trace && ti < kTrTiles && e == 0) trace[ti * kTrFields + TR_READY] = globaltimer();
          }
        }
      } else {  // EPI_F32
        float* orow = reinterpret_cast<float*>(P.out) + (size_t)tc.ks * P.split_stride + (size_t)row * ldo;
        const int accumulate = P.accumulate;
#pragma unroll 1
        for (int c = 0; c < kCols; c += 32) {
          float v[32];
          tmem_ld32(t_row + c, v);
          tmem_ld_wait();
          const int nb = n0 + c;
          if (!row_ok || nb >= n_valid) continue;
          const bool vec = (nb + 32 <= n_valid) && ((ldo & 3) == 0);
          if (vec && accumulate) {  // this tile's rows were written earlier (a preceding K range): add onto them
            float4 o[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) o[i] = *reinterpret_cast<const float4*>(orow + nb + 4 * i);
#pragma unroll
            for (int i = 0; i < 8; ++i)
              *reinterpret_cast<float4*>(orow + nb + 4 * i) =
                  make_float4(fmaf(v[4 * i], scale, o[i].x), fmaf(v[4 * i + 1], scale, o[i].y),
                              fmaf(v[4 * i + 2], scale, o[i].z), fmaf(v[4 * i + 3], scale, o[i].w));
          } else if (vec) {
#pragma unroll
            for (int i = 0; i < 32; i += 4)
              *reinterpret_cast<float4*>(orow + nb + i) =
                  make_float4(v[i] * scale, v[i + 1] * scale, v[i + 2] * scale, v[i + 3] * scale);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const int n = nb + i;
              if (n < n_valid) {
                float x = v[i] * scale;
                if (accumulate) x = fmaf(v[i], scale, orow[n]);
                orow[n] = x;
              }
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (trace && ti < kTrTiles && lane == 0) {
        if (e == 0) trace[ti * kTrFields + TR_EPI_END] = globaltimer();
        atomicMax(&trace[ti * kTrFields + TR_EPI_LAST], (unsigned long long)globaltimer());
      }
      if (lane == 0) {
        if (leader)
          mbar_arrive(&tempty[acc]);
        else  // TMEM reads are complete (wait::ld + fence): no memory release needed
          mbar_arrive_remote(tempty_c + acc * 8);
      }
    }
    if (lane == 0) bulk_wait0();  // staged output stores complete before exit
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // neither CTA leaves (or frees TMEM) while the pair is still working
  tc_fence_after();
  if (warp == 2) tmem_dealloc_pair(tmem_base, kTmemCols);
}

}  // namespace

int gemm_stats_parts() { return 4 / kEpiGroups; }

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
    rc = make_tmap_2d(&p->tmB, B, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, K, N, (uint64_t)ldb * 2, 64, kBHalf);
  else
    rc = make_tmap_2d(&p->tmB, B, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, N, K, (uint64_t)ldb * 2, 64, 64);
  if (rc) return rc;
  p->M = M;
  p->N = N;
  p->K = K;
  p->a_mn = a_mn;
  p->b_mn = b_mn;
  p->tiles_m = (M + kPairM - 1) / kPairM;  // pair tiles
  p->tiles_n = (N + BN - 1) / BN;
  p->n_valid = N;
  p->m_valid = M;
  p->scale = 1.f;
  p->ksplit = 1;
  return DS_OK;
}

// 64x64-blocked bf16 matrix [ceil(rows/64)][ceil(cols/64)][64][64] (dlogits)
static void blk_dims(int64_t rows, int64_t cols, uint64_t dims[4], uint64_t strides[3]) {
  const uint64_t nrb = (rows + 63) / 64, ncb = (cols + 63) / 64;
  dims[0] = 64;
  dims[1] = 64;
  dims[2] = ncb;
  dims[3] = nrb;
  strides[0] = 128;
  strides[1] = 8192;
  strides[2] = ncb * 8192;
}
int64_t gemm_blocked_elems(int64_t rows, int64_t cols) { return ((rows + 63) / 64) * ((cols + 63) / 64) * 4096; }

int gemm_blocked_a(GemmProblem* p, const void* A, int64_t rows, int64_t cols) {
  uint64_t dims[4], strides[3];
  blk_dims(rows, cols, dims, strides);
  // K-major (rows = M): one box = 2 row blocks x 1 column block = 128 x 64;
  // MN-major (rows = K): one box = 1 x 1 block (64 x 64), two per k-block
  const uint32_t box[4] = {64, 64, 1, p->a_mn ? 1u : 2u};
  int rc = make_tmap_4d(&p->tmA, A, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, dims, strides, box);
  if (rc) return rc;
  p->a_blk = 1;
  return DS_OK;
}

int gemm_blocked_output(GemmProblem* p, int64_t rows, int64_t cols) {
  if (p->epi != EPI_BF16 && p->epi != EPI_CE_GRAD) return fail_arg("TMA store only for bf16 epilogues");
  uint64_t dims[4], strides[3];
  blk_dims(rows, cols, dims, strides);
  const uint32_t box[4] = {32, 32, 1, 1};
  int rc = make_tmap_4d(&p->tmC, p->out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, dims, strides, box,
                        CU_TENSOR_MAP_SWIZZLE_64B);
  if (rc) return rc;
  p->c_tma = 1;
  p->c_blk = 1;
  return DS_OK;
}

int gemm_bf16_output(GemmProblem* p) {
  if (p->epi != EPI_BF16 && p->epi != EPI_CE_GRAD) return fail_arg("TMA store only for bf16 epilogues");
  int rc = make_tmap_2d(&p->tmC, p->out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, (uint64_t)p->n_valid, (uint64_t)p->m_valid,
                        (uint64_t)p->ldo * 2, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B);
  if (rc) return rc;
  p->c_tma = 1;
  return DS_OK;
}

// Tile cost in k-block units (mainloop) plus the epilogue's weight, for the
// host-side LPT assignment.  Uniform batches keep the round-robin walk.
static void schedule_tiles(GemmBatch* b, int pairs) {
  b->sched = 0;
  const int total = b->total_tiles;
  if (total > kMaxSched || total <= pairs) return;
  std::vector<std::pair<int, int>> cost(total);  // (cost, tile)
  bool uniform = true;
  for (int i = 0; i < b->nprob; ++i) {
    const GemmProblem& P = b->p[i];
    const int nkb = (P.K + BK - 1) / BK;
    const int per = (nkb + P.ksplit - 1) / P.ksplit;
    const int epi = P.epi == EPI_CE_STATS || P.epi == EPI_CE_GRAD ? 8 : (P.epi == EPI_F32 ? 3 : 2);
    const int n = P.tiles_m * P.tiles_n * P.ksplit;
    for (int t = 0; t < n; ++t) {
      const int ks = t / (P.tiles_m * P.tiles_n);
      const int len = (ks == P.ksplit - 1) ? nkb - per * (P.ksplit - 1) : per;
      cost[P.tile_begin + t] = {len + epi, P.tile_begin + t};
    }
  }
  for (int t = 1; t < total; ++t) uniform &= cost[t].first == cost[0].first;
  if (uniform) return;
  std::stable_sort(cost.begin(), cost.end(), [](const std::pair<int, int>& x, const std::pair<int, int>& y) {
    return x.first > y.first;
  });
  std::vector<long long> load(pairs, 0);
  std::vector<std::vector<int>> lists(pairs);
  for (const auto& c : cost) {  // longest remaining tile onto the least loaded pair
    int best = 0;
    for (int p = 1; p < pairs; ++p)
      if (load[p] < load[best]) best = p;
    load[best] += c.first;
    lists[best].push_back(c.second);
  }
  int pos = 0;
  for (int p = 0; p < pairs; ++p) {
    b->pstart[p] = (uint16_t)pos;
    for (int t : lists[p]) b->order[pos++] = (uint16_t)t;
  }
  b->pstart[pairs] = (uint16_t)pos;
  b->sched = 1;
}

static unsigned long long* g_trace = nullptr;
static int g_trace_countdown = -1;
static int g_trace_layer = -1;
unsigned long long* gemm_layer_trace(int layer) { return layer == g_trace_layer ? g_trace : nullptr; }
void gemm_set_trace(unsigned long long* buf, int launch) {
  g_trace = buf;
  g_trace_layer = buf && launch <= -2 ? -launch - 2 : -1;
  g_trace_countdown = buf && launch >= 0 ? launch : -1;
}

int gemm_launch(GemmBatch* b, cudaStream_t stream) {
  if (!b->trace_keep) b->trace = nullptr;
  static const bool no_bearly = getenv("DS_NO_BEARLY") != nullptr;  // A/B switch
  if (no_bearly || !use_pdl(1)) b->b_early = 0;
  if (g_trace_countdown >= 0 && g_trace_countdown-- == 0) b->trace = g_trace;
  static bool attr_set = false;
  if (!attr_set) {
    DS_CUDA_TRY(cudaFuncSetAttribute(gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes));
    attr_set = true;
  }
  int total = 0;
  for (int i = 0; i < b->nprob; ++i) {
    GemmProblem& P = b->p[i];
    if (P.ksplit < 1) P.ksplit = 1;
    const int nkb = (P.K + BK - 1) / BK;
    if (P.ksplit > 1 && (P.epi != EPI_F32 || P.accumulate || (P.ksplit - 1) * ((nkb + P.ksplit - 1) / P.ksplit) >= nkb))
      return fail_arg("split-K needs EPI_F32, no accumulate and no empty split");
    if (P.gate && !b->presched) return fail_arg("gated GEMM: needs a host schedule (presched)");
    if (P.ready && P.ready_stride < 1) P.ready_stride = 1;
    if (P.ready && (P.epi != EPI_BF16 || P.ready_rows % 32 || P.ready_cols % 64 || P.ready_rows < 32 || P.N % P.ready_cols))
      return fail_arg("output counters: 32-row / 64-column granularity");
    P.tile_begin = total;
    total += P.tiles_m * P.tiles_n * P.ksplit;
  }
  b->total_tiles = total;
  if (total == 0) return DS_OK;
  int max_pairs = num_sms() / 2 < kMaxPairs ? num_sms() / 2 : kMaxPairs;
  if (b->max_pairs > 0 && b->max_pairs < max_pairs) max_pairs = b->max_pairs;
  int pairs = total < max_pairs ? total : max_pairs;
  if (b->presched > 0) {
    if (!b->sched || b->presched > kMaxPairs || b->pstart[b->presched] != total)
      return fail_arg("gemm: bad host schedule");
    pairs = b->presched;
  } else {
    schedule_tiles(b, pairs);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[3];
  int na = 0;
  attr[na].id = cudaLaunchAttributeClusterDimension;
  attr[na].val.clusterDim.x = 2;
  attr[na].val.clusterDim.y = 1;
  attr[na].val.clusterDim.z = 1;
  ++na;
  if (use_pdl(1)) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (b->prio) {
    attr[na].id = cudaLaunchAttributePriority;
    attr[na].val.priority = b->prio;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  DS_CUDA_TRY(cudaLaunchKernelEx(&cfg, gemm_kernel, *b));
  return DS_OK;
}

}  // namespace ds
