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
// cell update is thread-local (one thread = one batch row).
//
// Forward (lstm_fwd2_kernel): CTA pairs with the batch as the MMA's N
//   operand and W_hh rows stationary as M (see the kernel's comment).
// Backward (lstm_bwd_kernel): CTA = (dir, 128-row batch tile, 64 units, K
//   slice of 512 gate rows) in 4-CTA clusters; W_hh[dir][K slice][units]
//   resident as an MN-major operand; partial dh exchanged through DSMEM.
// Dataflow instead of a group barrier: the producer of every CTA waits only
// for the CTAs that produced the chunk it is about to load, so chunk k's MMA
// overlaps the epilogues still running elsewhere.  Every CTA of a (direction,
// batch tile) group must be co-resident: grids stay <= 128 CTAs, one per SM.
#include <cuda_fp16.h>

#include "ds_internal.h"
#include "ds_ptx.cuh"
#include "layout.h"
#include "lstm_rec.h"

#include <cstdlib>

namespace ds {

namespace {

constexpr int kThreads = 384;
constexpr int kEpiWarp0 = 4;
constexpr int kEpiThreads = 256;
constexpr int kH = 512;               // hidden units per direction
constexpr int kTileA = 128 * 64 * 2;  // one 128x64 bf16 A box (16 KB)

__device__ __forceinline__ void bf16x8_to_f32(uint4 w, float* out) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 f = __bfloat1622float2(h[i]);
    out[2 * i] = f.x;
    out[2 * i + 1] = f.y;
  }
}
__device__ __forceinline__ uint4 f32_to_bf16x8(const float* v) {
  uint4 w;
  uint32_t* u = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    u[i] = *reinterpret_cast<uint32_t*>(&h);
  }
  return w;
}

// Flag words count up forever (never reset, see below), so comparisons are
// wrap-safe: v has reached target when (int32)(v - target) >= 0.
__device__ __forceinline__ bool reached(uint32_t v, uint32_t target) { return (int32_t)(v - target) >= 0; }

// Spin guard: a peer CTA that never publishes (a co-residency failure, a
// killed launch) must not hang the GPU.  After ~2 s of polling the waiter
// sets bit 8 of the step's error flag (raised by the host as RuntimeError)
// and gives up; the step's results are then garbage but the stream drains.
constexpr uint64_t kSpinTimeoutNs = 2000000000ull;
struct SpinGuard {
  uint32_t n = 0;
  uint64_t t0 = 0;
};
__device__ __forceinline__ bool spin_expired(SpinGuard& g, int* err) {
  if ((++g.n & 1023u) != 0) return false;
  if (err && (*reinterpret_cast<volatile int*>(err) & 8)) return true;  // the step already failed: drain
  const uint64_t now = globaltimer();
  if (g.t0 == 0) {
    g.t0 = now;
    return false;
  }
  if (now - g.t0 < kSpinTimeoutNs) return false;
  if (err) atomicOr(err, 8);
  return true;
}

// spin (relaxed, L1-bypassing) until *flag >= target, then acquire and make
// the released generic-proxy writes visible to our async-proxy (TMA) reads.
__device__ __forceinline__ void wait_flag(const uint32_t* flag, uint32_t target, int* err) {
  if (!reached(ld_relaxed_gpu(flag), target)) {
    SpinGuard g;
    while (!reached(ld_relaxed_gpu(flag), target)) {
      if (spin_expired(g, err)) return;
    }
  }
}
// Step flags: 32 per (dir, batch tile) group in four 32-byte segments, one
// per 128-byte line (a single hot line serialised ~128 pollers).  Every
// issuer finds all the flags it needs for a step in ONE segment and polls it
// with a single 32-byte acquire load per round trip:
//   forward: flag f = unit block; chunk kb (produced by blocks 4kb..4kb+3
//     at U=16) has a line of its own, polled with one 16-byte acquire load
//     (packing chunks r and r+4 into one segment measured slower: 8 writers
//     per line);
//   backward: flag c = dG chunk (64 gate rows); K-slice ks streams chunks
//     8ks..8ks+7 = segment ks.
constexpr int kFlagLine = 32;                   // words per line
constexpr int kGroupFlagWords = 8 * kFlagLine;  // 8 lines per group (4 used)
// Flag words per 128 batch rows: backward groups (2 directions) then forward
// lines (2 directions x 2 blocks of 64 rows), so the two kernels never share
// a word.  Flags are never reset: every CTA of a group publishes exactly T
// times per launch, so all flags of a group are equal when a launch starts;
// each CTA reads its own flag as the launch's base and waits / publishes
// relative to it (no memset node ahead of every recurrent launch).
constexpr int kFlagWords128 = 2 * kGroupFlagWords + 4 * kFlagLine;
__device__ __forceinline__ uint32_t* fwd_flag(uint32_t* base, int f) { return base + (f >> 2) * kFlagLine + (f & 3); }
__device__ __forceinline__ uint32_t* bwd_flag(uint32_t* base, int c) { return base + (c >> 3) * kFlagLine + (c & 7); }

// wait until all four consecutive flags (16-byte aligned) reach `target`,
// polling them with one acquire vector load per round trip
__device__ __forceinline__ void wait_flags4(const uint32_t* flags4, uint32_t target, int* err) {
  SpinGuard g;
  while (true) {
    const uint4 v = ld_acquire_gpu_v4(flags4);
    if (reached(v.x, target) && reached(v.y, target) && reached(v.z, target) && reached(v.w, target)) break;
    if (spin_expired(g, err)) return;
  }
}
// segment cache for an issuer walking the flags of one 32-byte segment
struct FlagSeg {
  uint32_t v[8];
};
// wait until flags [pos, pos + n) of the segment reach `target` (n = 1 or 4)
template <int n>
__device__ __forceinline__ void wait_seg(FlagSeg& c, const uint32_t* seg, int pos, uint32_t target, int* err) {
  SpinGuard g;
  while (true) {
    bool ok = reached(c.v[pos], target);
#pragma unroll
    for (int i = 1; i < n; ++i) ok = ok && reached(c.v[pos + i], target);
    if (ok || spin_expired(g, err)) return;
    ld_acquire_gpu_v8(seg, c.v);
  }
}

__device__ __forceinline__ void acquire_for_tma(const uint32_t* flag, int variant) {
  if (variant & 4)
    (void)ld_acquire_gpu(flag);
  else
    fence_acq_rel_gpu();
  if (!(variant & 128)) fence_proxy_async_global();
}

// all epilogue threads finished step s's global writes -> flag = s + 1
__device__ __forceinline__ void publish(uint32_t* flag, uint32_t value, int variant) {
  if (!(variant & 1)) fence_proxy_async_global();
  if (variant & 64) fence_acq_rel_gpu();  // every thread drains its own stores
  named_bar_sync(1, kEpiThreads);
  if (threadIdx.x == kEpiWarp0 * 32) {
    if (!(variant & 2)) fence_acq_rel_gpu();
    if (variant & 64)
      asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"(value) : "memory");
    else
      st_release_gpu(flag, value);
  }
}

constexpr int kTraceSlots = 6;
__device__ __forceinline__ void trace_mark(uint64_t* trace, int T, int s, int k) {
  if (trace) trace[((size_t)blockIdx.x * T + s) * kTraceSlots + k] = globaltimer();
}

// ============================================================================
// Forward, batch-as-N CTA pairs (default): weights stationary as the MMA's M operand.
//   CTA pair (tcgen05 cta_group::2) = (dir, batch block of 64, 64 units =
//   256 gate rows).  Rank r keeps W_hh rows [r*128, +128) of the pair's 256
//   (32 units, 128 KB smem, A operand) and stages batch rows [r*32, +32) of
//   every h_{t-1} chunk (B operand, N split across the pair), so one SM pulls
//   8 x 4 KB = 32 KB of h per step instead of the whole 128 KB tile.
//   acc[128 gate rows (TMEM lanes), 64 batch] per CTA; the epilogue
//   transposes gate quads with two shuffle stages so a thread owns one unit
//   x 8 batch columns (i,f,g,o together), keeps c in registers, stages h_t in
//   smem for coalesced 16-byte stores and publishes one flag per CTA.
//   16 CTAs per (dir, batch block): chunk k of h (64 units) = pair k.
namespace fwd2 {
constexpr int kNB = 64;                 // batch columns per pair (MMA N)
constexpr int kNH = kNB / 2;            // batch rows staged per CTA
constexpr int kPairs = kH / 64;         // 8 pairs per (dir, batch block)
constexpr int kCtas = 2 * kPairs;       // 16
constexpr int kWB = 128 * kH * 2;       // 128 KB resident W slice
constexpr int kChunkB = kNH * 128;      // 4 KB: 32 batch rows x 64 units bf16
constexpr int kBufB = 8 * kChunkB;      // one step's B operand (32 KB)
constexpr int kHst = kNB * 64;          // h staging: 64 batch rows x 32 units bf16 (4 KB)
constexpr int kXKb = 5;                   // fused input projection: K = 272 padded to 5 blocks of 64
constexpr int kXB = kXKb * kChunkB;        // one step's x tile per CTA (32 rows x 320 K, 20 KB)
constexpr uint32_t kXCol = 128;           // W_ih slice in TMEM columns 128 .. 287 (two bf16 per column)
constexpr size_t kSmem = 1024 + kWB + 2 * kBufB + kHst + 1024;  // + kXB for the fused input projection
constexpr size_t kSmemX = kSmem + kXB;
constexpr int kEpiWarps = 16;             // lane quadrant x 16-column group (4 per SM sub-partition)
constexpr int kEpiT = kEpiWarps * 32;
constexpr int kThreadsF2 = 32 * (kEpiWarp0 + kEpiWarps);
constexpr int kGC = 16;                    // batch columns per epilogue warp (TMEM load width)
constexpr int kPub = 2;                 // named barriers 2/3: epilogue <-> publisher
}  // namespace fwd2

// kX: layer 0's input projection fused in (a separate instantiation: the hot loops of the plain one
// carry none of its code)
template <bool kX>
__global__ void __launch_bounds__(fwd2::kThreadsF2, 1) lstm_fwd2_kernel(const __grid_constant__ LstmParams P) {
  using namespace fwd2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sW = sm;
  uint8_t* sB = sW + kWB;                 // [2 steps][8 chunks][32 rows x 128 B]
  uint8_t* sH = sB + 2 * kBufB;           // [64 rows][32 units] bf16
  uint64_t* full = reinterpret_cast<uint64_t*>(sH + kHst);  // [2][8], leader only
  uint64_t* wbar = full + 16;
  uint64_t* tfull = wbar + 1;   // [2]
  uint64_t* tempty = tfull + 2;  // [2], leader: every epilogue warp of both CTAs
  uint64_t* xfull = tempty + 2;  // leader: both CTAs' x tile of the step
  uint64_t* xempty = xfull + 1;  // every CTA: the pair's x MMAs read the tile
  uint64_t* wibar = xempty + 1;  // launch: W_ih boxes staged
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(wibar + 1);
  uint8_t* sX = sH + kHst + 1024;         // fused input projection only: [5 K blocks][32 rows x 128 B]
  constexpr bool xin = kX;

  const uint32_t warp = warp_id(), lane = lane_id();
  const uint32_t rank = cluster_ctarank();  // 0 = leader
  const bool leader = rank == 0;
  const int pg = blockIdx.x >> 1;
  const int pr = pg % kPairs;
  const int bb = (pg / kPairs) % P.n_btile;  // batch block of 64 (n_btile counts blocks here)
  const int dir = pg / (kPairs * P.n_btile);
  const int gblk = P.b0 / kNB + bb;  // global 64-row block
  uint32_t* flags = P.counters + (size_t)(gblk >> 1) * kFlagWords128 + 2 * kGroupFlagWords +
                    ((gblk & 1) * 2 + dir) * kFlagLine;  // 16 flags: CTA = 2*pair + rank
  __shared__ uint32_t s_base;
  const int T = P.T, B = P.B;
  const int b0 = P.b0 + bb * kNB;

  if (warp == 1 && lane == 0) {
    for (int i = 0; i < 16; ++i) mbar_init(&full[i], 1);
    mbar_init(wbar, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 2 * kEpiWarps);
    }
    mbar_init(xfull, 1);
    mbar_init(xempty, 1);
    mbar_init(wibar, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_pair(tmem_slot, xin ? 512 : 128);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // programmatic launch: the W_hh slice (operand snapshot, not written by the predecessor) is
  // fetched before waiting for the predecessor grid; everything else after.  The launch's flag
  // base is read after the wait: a previous launch on the same flags may still be publishing.
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&P.tmA);
    tma_prefetch_desc(&P.tmW);
    mbar_arrive_expect_tx(wbar, kWB);
    const int wrow = dir * 4 * kH + pr * 256 + (int)rank * 128;
    for (int kb = 0; kb < kH / 64; ++kb) tma_load_2d(sW + kb * 16384, &P.tmW, wbar, kb * 64, wrow);
  }
  if (xin) {
    // W_ih rows of this CTA (128 gate rows x 320 K) into TMEM, staged through the B buffers (64 KB) in
    // two rounds: K blocks 0-3, then 4; lane = gate row, column c = K (2c, 2c+1), SW128 chunks
    const int wrow = dir * 4 * kH + pr * 256 + (int)rank * 128;
    for (int round = 0; round < 2; ++round) {
      const int kb0 = round * 4, nkb = round ? kXKb - 4 : 4;
      if (threadIdx.x == 0) {
        if (round == 0) tma_prefetch_desc(&P.tmWi);
        mbar_arrive_expect_tx(wibar, nkb * 16384);
        for (int j = 0; j < nkb; ++j) tma_load_2d(sB + j * 16384, &P.tmWi, wibar, (kb0 + j) * 64, wrow);
      }
      if (warp >= kEpiWarp0) {
        const uint32_t e = warp - kEpiWarp0, q = e & 3, grp = e >> 2;  // 4 groups split the staged blocks
        const uint32_t m = q * 32 + lane;
        mbar_wait(wibar, (uint32_t)round);
        for (int j = (int)grp; j < nkb; j += 4) {
          const uint8_t* row = sB + j * 16384 + m * 128;
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            uint32_t rr[16];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const uint4 w = *reinterpret_cast<const uint4*>(row + (((half * 4 + c) ^ (m & 7)) << 4));
              rr[4 * c] = w.x;
              rr[4 * c + 1] = w.y;
              rr[4 * c + 2] = w.z;
              rr[4 * c + 3] = w.w;
            }
            tmem_st16(tmem + ((q * 32) << 16) + kXCol + (uint32_t)(kb0 + j) * 32 + half * 16, rr);
          }
        }
        tmem_st_wait();
      }
      tc_fence_before();
      __syncthreads();  // the staging area is read (round 0) / free for the B operand (round 1)
      tc_fence_after();
    }
    cluster_sync_all();  // the partner's W_ih in its TMEM before the first pair MMA
    tc_fence_after();
  }
  griddep_wait();
  if (threadIdx.x == 0) s_base = ld_relaxed_gpu(flags + (pr >> 2) * 8 + (pr & 3) * 2 + (int)rank);
  __syncthreads();
  const uint32_t base = s_base;  // flag value at launch start (same for every CTA of the group)

  if (warp == 0) {
    if (elect_one()) {
      const uint32_t full_c = mapa_shared(smem_u32(full), 0);
      FlagSeg seg[2];
#pragma unroll
      for (int i = 0; i < 8; ++i) seg[0].v[i] = seg[1].v[i] = 0;
      for (int s = 0; s < T; ++s) {
        const int t = dir == 0 ? s : T - 1 - s;
        const int tprev = dir == 0 ? t - 1 : t + 1;
        const int arow = (tprev + 1) * B + b0 + (int)rank * kNH;
        const int buf = s & 1;
        if (xin) {  // x_t of my 32 batch rows, once the pair's x MMAs of the previous step read the tile
          if (s > 0) mbar_wait(xempty, (uint32_t)(s - 1) & 1);
          if (leader) mbar_arrive_expect_tx(xfull, 2 * kXB);
          const uint32_t xfull_c = mapa_shared(smem_u32(xfull), 0);
          for (int j = 0; j < kXKb; ++j)
            tma_load_2d_pair(sX + j * kChunkB, &P.tmX, xfull_c, j * 64, t * B + b0 + (int)rank * kNH);
        }
        for (int k = 0; k < kPairs; ++k) {
          uint64_t* fb = &full[buf * 8 + k];
          if (leader) mbar_arrive_expect_tx(fb, 2 * kChunkB);
          if (s > 0) {  // chunk k of h_{t-1} = both CTAs of pair k (flags 2k, 2k+1)
            wait_seg<2>(seg[k >> 2], flags + (k >> 2) * 8, (k & 3) * 2, base + (uint32_t)s, P.err);
            fence_proxy_async_global();
          }
          tma_load_2d_pair(sB + buf * kBufB + k * kChunkB, &P.tmA, full_c + (uint32_t)(buf * 8 + k) * 8,
                           dir * kH + k * 64, arow);
          if (k == 0) trace_mark(P.trace, T, s, 0);
          if (P.trace && blockIdx.x == 0)
            P.trace[(size_t)gridDim.x * T * kTraceSlots + ((size_t)s * 8 + k) * 2] = globaltimer();
        }
        trace_mark(P.trace, T, s, 1);
      }
    }
  } else if (warp == 1) {
    if (leader) {
      mbar_wait(wbar, 0);
      const uint32_t idesc = idesc_bf16_f32(256, kNB, 0, 0);
      const uint32_t wbase = smem_u32(sW), bbase = smem_u32(sB);
      for (int s = 0; s < T; ++s) {
        const int acc = s & 1, buf = s & 1;
        mbar_wait_acq_cluster(&tempty[acc], ((s >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t dacc = tmem + acc * kNB;
        if (xin) {  // x_t W_ih^T first: its operands do not wait for the previous step
          mbar_wait(xfull, (uint32_t)s & 1);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t xb = smem_u32(sX);
#pragma unroll 1
            for (int j = 0; j < kXKb; ++j)
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)
                mma_bf16_ts_pair(dacc, tmem + kXCol + (uint32_t)(j * 4 + kk) * 8,
                                 smem_desc_sw128(xb + j * kChunkB + kk * 32, 16, 1024), idesc, (j | kk) != 0);
            mma_commit_pair_mc(xempty, 0x3);
          }
          __syncwarp();
        }
        for (int k = 0; k < kPairs; ++k) {
          mbar_wait(&full[buf * 8 + k], (s >> 1) & 1);
          tc_fence_after();
          if (P.trace && blockIdx.x == 0 && lane == 0)
            P.trace[(size_t)gridDim.x * T * kTraceSlots + ((size_t)s * 8 + k) * 2 + 1] = globaltimer();
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              uint64_t ad = smem_desc_sw128(wbase + k * 16384 + kk * 32, 16, 1024);
              uint64_t bd = smem_desc_sw128(bbase + buf * kBufB + k * kChunkB + kk * 32, 16, 1024);
              mma_bf16_ss_pair(dacc, ad, bd, idesc, xin || (k | kk) != 0);
            }
            if (k == kPairs - 1) mma_commit_pair_mc(&tfull[acc], 0x3);
          }
          __syncwarp();
        }
      }
    } else {
      mbar_wait(wbar, 0);  // keep the W load's barrier alive until it lands
    }
  } else if (warp == 3) {
    // publisher: h_t of this CTA stored -> release the step flag
    uint32_t* myflag = flags + (pr >> 2) * 8 + (pr & 3) * 2 + (int)rank;  // flag 2*pr + rank: segment /8, pos %8
    for (int s = 0; s < T; ++s) {
      named_bar_sync(kPub, kEpiT + 32);
      if (lane == 0) {
        st_release_gpu(myflag, base + (uint32_t)(s + 1));
        trace_mark(P.trace, T, s, 4);
      }
      __syncwarp();
      asm volatile("bar.arrive %0, %1;" ::"n"(kPub + 1), "n"(kEpiT + 32) : "memory");
    }
  } else if (warp >= kEpiWarp0 && warp < kEpiWarp0 + kEpiWarps) {
    const uint32_t e = warp - kEpiWarp0;
    const uint32_t q = e & 3, hc = e >> 2;      // TMEM lane quadrant, 16-column batch group
    const uint32_t g = lane & 3;                 // gate of this thread's TMEM row (unit-interleaved rows)
    const uint32_t b0b = g & 1, b1b = g >> 1;
    const int uq = (int)(q * 8 + (lane >> 2));   // unit within the CTA's 32
    const int unit = pr * 64 + (int)rank * 32 + uq;  // unit within the direction
    const int col0 = (int)(hc * kGC + g * 4);    // after the transpose: batch columns col0 .. +4
    const uint32_t tcol = tmem + ((q * 32) << 16) + hc * kGC;
    const uint32_t tempty_c = mapa_shared(smem_u32(tempty), 0);
    const size_t gcol = (size_t)dir * 4 * kH + (size_t)unit * 4;
    float c[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) c[i] = 0.f;
    const float4 xb4 = xin ? *reinterpret_cast<const float4*>(P.xbias + gcol) : make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < T; ++s) {
      if (s == T - 1) griddep_launch();  // the next kernel may start its prologue
      const int t = dir == 0 ? s : T - 1 - s;
      // prefetch the input projection (i,f,g,o of this unit) for my 4 batch rows
      uint2 gp[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int b = b0 + col0 + i;
        gp[i] = b < B && !xin ? *reinterpret_cast<const uint2*>(P.gates + ((size_t)t * B + b) * (8 * kH) + gcol)
                              : make_uint2(0u, 0u);
      }
      mbar_wait(&tfull[s & 1], (s >> 1) & 1);
      tc_fence_after();
      if (e == 0 && lane == 0) trace_mark(P.trace, T, s, 2);
      float v[kGC];
      tmem_ld16(tcol + (s & 1) * kNB, v);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader)
          mbar_arrive(&tempty[s & 1]);
        else
          mbar_arrive_remote(tempty_c + (s & 1) * 8);
      }
      // quad transpose: stage 1 (lane ^ 2) splits the 16 columns in halves,
      // stage 2 (lane ^ 1) in quarters -> 4 gates x 4 columns per lane
      float a1[8], a2[8];  // a1: gate g, a2: gate g^2 (columns of my half)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float send = b1b ? v[i] : v[8 + i];
        a1[i] = b1b ? v[8 + i] : v[i];
        a2[i] = __shfl_xor_sync(0xffffffffu, send, 2);
      }
      float k1[4], k2[4], r1[4], r2[4];  // gates g, g^2 (kept), g^1, g^3 (received)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float s1 = b0b ? a1[i] : a1[4 + i];
        const float s2 = b0b ? a2[i] : a2[4 + i];
        k1[i] = b0b ? a1[4 + i] : a1[i];
        k2[i] = b0b ? a2[4 + i] : a2[i];
        r1[i] = __shfl_xor_sync(0xffffffffu, s1, 1);
        r2[i] = __shfl_xor_sync(0xffffffffu, s2, 1);
      }
      float hv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        // gate x lives in: d = g ^ x -> d0 ? (d1 ? r2 : r1) : (d1 ? k2 : k1)
        const float x0 = b0b ? (b1b ? r2[i] : r1[i]) : (b1b ? k2[i] : k1[i]);   // i gate (x = 0)
        const float x1 = b0b ? (b1b ? k2[i] : k1[i]) : (b1b ? r2[i] : r1[i]);   // f gate (x = 1)
        const float x2 = b0b ? (b1b ? r1[i] : r2[i]) : (b1b ? k1[i] : k2[i]);   // g gate (x = 2)
        const float x3 = b0b ? (b1b ? k1[i] : k2[i]) : (b1b ? r1[i] : r2[i]);   // o gate (x = 3)
        const __nv_bfloat162* gg = reinterpret_cast<const __nv_bfloat162*>(&gp[i]);
        float2 g01 = __bfloat1622float2(gg[0]), g23 = __bfloat1622float2(gg[1]);
        if (xin) {  // the accumulator holds x_t W_ih^T + h W_hh^T: add the bias
          g01 = make_float2(xb4.x, xb4.y);
          g23 = make_float2(xb4.z, xb4.w);
        }
        const float ig = sigmoid_fast(x0 + g01.x);
        const float fg = sigmoid_fast(x1 + g01.y);
        const float gt = tanh_fast(x2 + g23.x);
        const float og = sigmoid_fast(x3 + g23.y);
        c[i] = fmaf(fg, c[i], ig * gt);
        hv[i] = og * tanh_fast(c[i]);
        // keep the activations for the BPTT state (written after the release)
        __nv_bfloat162 p0 = __floats2bfloat162_rn(ig, fg), p1 = __floats2bfloat162_rn(gt, og);
        gp[i].x = *reinterpret_cast<uint32_t*>(&p0);
        gp[i].y = *reinterpret_cast<uint32_t*>(&p1);
      }
      if (e == 0 && lane == 0) trace_mark(P.trace, T, s, 5);
      // h_t -> smem [64 rows][32 units] -> coalesced 16-byte stores
#pragma unroll
      for (int i = 0; i < 4; ++i)
        reinterpret_cast<__nv_bfloat16*>(sH)[(col0 + i) * 32 + uq] = __float2bfloat16_rn(hv[i]);
      named_bar_sync(1, kEpiT);
      {
        const int tid = (int)(e * 32 + lane);  // threads 0..255 = 64 rows x 4 segments of 8 units
        const int row = tid >> 2, sg = tid & 3;
        const int b = b0 + row;
        const uint4 w = tid < kNB * 4 ? reinterpret_cast<const uint4*>(sH)[tid] : make_uint4(0u, 0u, 0u, 0u);
        if (tid < kNB * 4 && b < B && row < P.nb - bb * kNB)
          *reinterpret_cast<uint4*>(P.y + ((size_t)(t + 1) * B + b) * (2 * kH) + dir * kH + pr * 64 + rank * 32 +
                                    sg * 8) = w;
      }
      if (e == 0 && lane == 0) trace_mark(P.trace, T, s, 3);
      asm volatile("bar.arrive %0, %1;" ::"n"(kPub), "n"(kEpiT + 32) : "memory");
      named_bar_sync(kPub + 1, kEpiT + 32);  // the release is out: BPTT state, then reuse sH
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int b = b0 + col0 + i;
        if (b < B && col0 + i < P.nb - bb * kNB) {
          const size_t n = (size_t)t * B + b;
          *reinterpret_cast<uint2*>(P.gates + n * (8 * kH) + gcol) = gp[i];
          P.cstate[n * (2 * kH) + dir * kH + unit] = c[i];
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  if (warp == 2) tmem_dealloc_pair(tmem, xin ? 512 : 128);
}

// ============================================================================
// Forward, narrow (DS_FWD=3): 64 CTAs at B = 256 instead of 128, so that the next layer's input
// projection could stream beside the recurrence on the SMs it leaves free.  Measured 5.4 us per
// step (cell 1.4 us: twice fwd2's cell work per SM, MUFU / issue bound) against fwd2's 4.5.
//   CTA pair (cta_group::2) = (dir, batch block of 128, 64 units = 256 gate rows).  Rank r
//   holds W_hh rows [r*128, +128) of the pair's 256 as the MMA's A operand in tensor memory
//   (128 lanes x 512 K = 256 columns, filled once per launch) and stages batch rows [r*64, +64)
//   of every h_{t-1} chunk (B operand, N = 128 split across the pair): per step 32 pair MMAs
//   M256 N128 K16 with A from TMEM into a double-buffered accumulator [128 gate rows, 128 batch]
//   (256 columns).  16 epilogue warps (lane quadrant x 32-column group) transpose gate quads as in
//   fwd2 (a thread owns one unit x 8 batch columns, c in registers), stage h_t in smem for
//   coalesced stores; a publisher warp releases the CTA's step flag and counts the step on
//   P.gate[dir * T + t] (the streamed projection of the next layer waits on those).
//   16 CTAs per (dir, batch block): chunk k of h (64 units) = pair k.
namespace fwd3 {
constexpr int kNB = 128;                 // batch columns per pair (MMA N)
constexpr int kNH = kNB / 2;             // batch rows staged per CTA
constexpr int kPairs = kH / 64;          // 8 pairs per (dir, batch block)
constexpr int kCtas = 2 * kPairs;        // 16
constexpr int kChunkB = kNH * 128;       // 8 KB: 64 batch rows x 64 units bf16 (SWIZZLE_128B)
constexpr int kBufB = 8 * kChunkB;       // one step's B operand (64 KB)
constexpr int kWB = 128 * kH * 2;        // 128 KB W slice, staged once for the TMEM fill (aliases the B buffers)
constexpr int kHst = kNB * 64;           // h staging: 128 batch rows x 32 units bf16 (8 KB)
constexpr size_t kSmem = 1024 + 2 * kBufB + kHst + 512;
constexpr int kEpiWarps = 16;
constexpr int kEpiT = kEpiWarps * 32;
constexpr int kThreadsF = 32 * (4 + kEpiWarps);
constexpr uint32_t kACol = 256;          // A = W slice at TMEM columns 256..511 (two bf16 per column)
constexpr int kPub = 2;                  // named barriers 2/3: epilogue <-> publisher
static_assert(kWB <= 2 * kBufB, "W staging must fit in the B buffers");
}  // namespace fwd3

__global__ void __launch_bounds__(fwd3::kThreadsF, 1) lstm_fwd3_kernel(const __grid_constant__ LstmParams P) {
  using namespace fwd3;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sB = sm;                       // [2 steps][8 chunks][64 rows x 128 B]; launch: W staging
  uint8_t* sH = sB + 2 * kBufB;           // [128 rows][32 units] bf16
  uint64_t* full = reinterpret_cast<uint64_t*>(sH + kHst);  // [2][8], leader only
  uint64_t* wbar = full + 16;
  uint64_t* tfull = wbar + 1;    // [2]
  uint64_t* tempty = tfull + 2;  // [2], leader: every epilogue warp of both CTAs
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  __shared__ uint32_t s_base;

  const uint32_t warp = warp_id(), lane = lane_id();
  const uint32_t rank = cluster_ctarank();  // 0 = leader
  const bool leader = rank == 0;
  const int pg = blockIdx.x >> 1;
  const int pr = pg % kPairs;
  const int bb = (pg / kPairs) % P.n_btile;  // batch block of 128
  const int dir = pg / (kPairs * P.n_btile);
  const int gblk = P.b0 / kNB + bb;  // global 128-row block (its even 64-row flag line, shared with fwd2)
  uint32_t* flags = P.counters + (size_t)gblk * kFlagWords128 + 2 * kGroupFlagWords + dir * kFlagLine;
  const int T = P.T, B = P.B;
  const int b0 = P.b0 + bb * kNB;

  if (warp == 1 && lane == 0) {
    for (int i = 0; i < 16; ++i) mbar_init(&full[i], 1);
    mbar_init(wbar, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 2 * kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_pair(tmem_slot, 512);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // programmatic launch: the W_hh slice (operand snapshot, not written by the predecessor) goes
  // into tensor memory before waiting for the predecessor grid
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&P.tmA);
    tma_prefetch_desc(&P.tmW);
    mbar_arrive_expect_tx(wbar, kWB);
    const int wrow = dir * 4 * kH + pr * 256 + (int)rank * 128;
    for (int kb = 0; kb < kH / 64; ++kb) tma_load_2d(sB + kb * 16384, &P.tmW, wbar, kb * 64, wrow);
  }
  if (warp >= 4) {  // TMEM lane m = gate row, column c = K (2c, 2c+1); 16-byte chunks unswizzled
    const uint32_t e = warp - 4, q = e & 3, cq = e >> 2;  // lane quadrant, K quarter (128 K = 2 boxes)
    const uint32_t m = q * 32 + lane;
    mbar_wait(wbar, 0);
#pragma unroll
    for (int hb = 0; hb < 2; ++hb) {
      const uint8_t* row = sB + (2 * cq + hb) * 16384 + m * 128;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        uint32_t rr[16];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint4 w = *reinterpret_cast<const uint4*>(row + (((half * 4 + j) ^ (m & 7)) << 4));
          rr[4 * j] = w.x;
          rr[4 * j + 1] = w.y;
          rr[4 * j + 2] = w.z;
          rr[4 * j + 3] = w.w;
        }
        tmem_st16(tmem + ((q * 32) << 16) + kACol + (2 * cq + hb) * 32 + half * 16, rr);
      }
    }
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // A in the TMEM of both CTAs; the staging area is free for the B operand
  tc_fence_after();
  griddep_wait();
  if (threadIdx.x == 0) s_base = ld_relaxed_gpu(flags + (pr >> 2) * 8 + (pr & 3) * 2 + (int)rank);
  if (threadIdx.x == 0 && blockIdx.x == 0 && P.seq)  // started: release GEMMs gated on this launch
    st_release_gpu(P.seq + 2, ld_relaxed_gpu(P.seq) * 16u + (uint32_t)P.tag);
  __syncthreads();
  const uint32_t base = s_base;  // flag value at launch start (same for every CTA of the group)

  if (warp == 0) {
    if (elect_one()) {
      const uint32_t full_c = mapa_shared(smem_u32(full), 0);
      FlagSeg seg[2];
#pragma unroll
      for (int i = 0; i < 8; ++i) seg[0].v[i] = seg[1].v[i] = 0;
      for (int s = 0; s < T; ++s) {
        const int t = dir == 0 ? s : T - 1 - s;
        const int tprev = dir == 0 ? t - 1 : t + 1;
        const int arow = (tprev + 1) * B + b0 + (int)rank * kNH;
        const int buf = s & 1;
        for (int k = 0; k < kPairs; ++k) {
          uint64_t* fb = &full[buf * 8 + k];
          if (leader) mbar_arrive_expect_tx(fb, 2 * kChunkB);
          if (s > 0) {  // chunk k of h_{t-1} = both CTAs of pair k (flags 2k, 2k+1)
            wait_seg<2>(seg[k >> 2], flags + (k >> 2) * 8, (k & 3) * 2, base + (uint32_t)s, P.err);
            fence_proxy_async_global();
          }
          tma_load_2d_pair(sB + buf * kBufB + k * kChunkB, &P.tmA, full_c + (uint32_t)(buf * 8 + k) * 8,
                           dir * kH + k * 64, arow);
          if (k == 0) trace_mark(P.trace, T, s, 0);
        }
        trace_mark(P.trace, T, s, 1);
      }
    }
  } else if (warp == 1) {
    if (leader) {
      const uint32_t idesc = idesc_bf16_f32(256, kNB, 0, 0);
      const uint32_t bbase = smem_u32(sB);
      for (int s = 0; s < T; ++s) {
        const int acc = s & 1, buf = s & 1;
        mbar_wait_acq_cluster(&tempty[acc], ((s >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t dacc = tmem + acc * kNB;
        for (int k = 0; k < kPairs; ++k) {
          mbar_wait(&full[buf * 8 + k], (s >> 1) & 1);
          tc_fence_after();
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_bf16_ts_pair(dacc, tmem + kACol + (uint32_t)(k * 4 + kk) * 8,
                               smem_desc_sw128(bbase + buf * kBufB + k * kChunkB + kk * 32, 16, 1024), idesc,
                               (k | kk) != 0);
            if (k == kPairs - 1) mma_commit_pair_mc(&tfull[acc], 0x3);
          }
          __syncwarp();
        }
      }
    }
  } else if (warp == 3) {
    // publisher: h_t of this CTA stored -> release the step flag, count the step for the next layer
    uint32_t* myflag = flags + (pr >> 2) * 8 + (pr & 3) * 2 + (int)rank;
    for (int s = 0; s < T; ++s) {
      named_bar_sync(kPub, kEpiT + 32);
      if (lane == 0) {
        st_release_gpu(myflag, base + (uint32_t)(s + 1));
        if (P.gate) red_release_gpu_add(P.gate + dir * T + (dir == 0 ? s : T - 1 - s), 1u);
        trace_mark(P.trace, T, s, 4);
      }
      __syncwarp();
      asm volatile("bar.arrive %0, %1;" ::"n"(kPub + 1), "n"(kEpiT + 32) : "memory");
    }
  } else if (warp >= 4) {
    const uint32_t e = warp - 4;
    const uint32_t q = e & 3, hc = e >> 2;      // TMEM lane quadrant, 32-column batch group
    const uint32_t g = lane & 3;                 // gate of this thread's TMEM row (unit-interleaved rows)
    const uint32_t b0b = g & 1, b1b = g >> 1;
    const int uq = (int)(q * 8 + (lane >> 2));   // unit within the CTA's 32
    const int unit = pr * 64 + (int)rank * 32 + uq;  // unit within the direction
    const int col0 = (int)(hc * 32 + g * 8);     // after the transpose: batch columns col0 .. +8
    const uint32_t tcol = tmem + ((q * 32) << 16) + hc * 32;
    const uint32_t tempty_c = mapa_shared(smem_u32(tempty), 0);
    const size_t gcol = (size_t)dir * 4 * kH + (size_t)unit * 4;
    const int nrow = P.nb - bb * kNB;            // valid rows of this block in this launch
    float c[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = 0.f;
    for (int s = 0; s < T; ++s) {
      if (s == T - 1) griddep_launch();  // the next kernel may start its prologue
      const int t = dir == 0 ? s : T - 1 - s;
      uint2 gp[8];  // input projection (i,f,g,o of this unit) of my 8 batch rows, fetched before the wait
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int b = b0 + col0 + i;
        gp[i] = b < B ? *reinterpret_cast<const uint2*>(P.gates + ((size_t)t * B + b) * (8 * kH) + gcol)
                      : make_uint2(0u, 0u);
      }
      mbar_wait(&tfull[s & 1], (s >> 1) & 1);
      tc_fence_after();
      if (e == 0 && lane == 0) trace_mark(P.trace, T, s, 2);
      float v[32];
      tmem_ld32(tcol + (s & 1) * kNB, v);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader)
          mbar_arrive(&tempty[s & 1]);
        else
          mbar_arrive_remote(tempty_c + (s & 1) * 8);
      }
      // quad transpose: stage 1 (lane ^ 2) splits the 32 columns in halves,
      // stage 2 (lane ^ 1) in quarters -> 4 gates x 8 columns per lane
      float a1[16], a2[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float send = b1b ? v[i] : v[16 + i];
        a1[i] = b1b ? v[16 + i] : v[i];
        a2[i] = __shfl_xor_sync(0xffffffffu, send, 2);
      }
      float k1[8], k2[8], r1[8], r2[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float s1 = b0b ? a1[i] : a1[8 + i];
        const float s2 = b0b ? a2[i] : a2[8 + i];
        k1[i] = b0b ? a1[8 + i] : a1[i];
        k2[i] = b0b ? a2[8 + i] : a2[i];
        r1[i] = __shfl_xor_sync(0xffffffffu, s1, 1);
        r2[i] = __shfl_xor_sync(0xffffffffu, s2, 1);
      }
      float hv[8];
#pragma unroll
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float x0 = b0b ? (b1b ? r2[i] : r1[i]) : (b1b ? k2[i] : k1[i]);   // i gate
        const float x1 = b0b ? (b1b ? k2[i] : k1[i]) : (b1b ? r2[i] : r1[i]);   // f gate
        const float x2 = b0b ? (b1b ? r1[i] : r2[i]) : (b1b ? k1[i] : k2[i]);   // g gate
        const float x3 = b0b ? (b1b ? k1[i] : k2[i]) : (b1b ? r1[i] : r2[i]);   // o gate
        const __nv_bfloat162* gg = reinterpret_cast<const __nv_bfloat162*>(&gp[i]);
        const float2 g01 = __bfloat1622float2(gg[0]), g23 = __bfloat1622float2(gg[1]);
        const float ig = sigmoid_fast(x0 + g01.x);
        const float fg = sigmoid_fast(x1 + g01.y);
        const float gt = tanh_fast(x2 + g23.x);
        const float og = sigmoid_fast(x3 + g23.y);
        c[i] = fmaf(fg, c[i], ig * gt);
        hv[i] = og * tanh_fast(c[i]);
        __nv_bfloat162 p0 = __floats2bfloat162_rn(ig, fg), p1 = __floats2bfloat162_rn(gt, og);
        gp[i].x = *reinterpret_cast<uint32_t*>(&p0);
        gp[i].y = *reinterpret_cast<uint32_t*>(&p1);
      }
      if (e == 0 && lane == 0) trace_mark(P.trace, T, s, 5);
#pragma unroll
      for (int i = 0; i < 8; ++i)
        reinterpret_cast<__nv_bfloat16*>(sH)[(col0 + i) * 32 + uq] = __float2bfloat16_rn(hv[i]);
      named_bar_sync(1, kEpiT);
      {
        const int tid = (int)(e * 32 + lane);  // 512 threads = 128 rows x 4 segments of 8 units
        const int row = tid >> 2, sg = tid & 3;
        const int b = b0 + row;
        const uint4 w = reinterpret_cast<const uint4*>(sH)[tid];
        if (b < B && row < nrow)
          *reinterpret_cast<uint4*>(P.y + ((size_t)(t + 1) * B + b) * (2 * kH) + dir * kH + pr * 64 + rank * 32 +
                                    sg * 8) = w;
      }
      if (e == 0 && lane == 0) trace_mark(P.trace, T, s, 3);
      asm volatile("bar.arrive %0, %1;" ::"n"(kPub), "n"(kEpiT + 32) : "memory");
      named_bar_sync(kPub + 1, kEpiT + 32);  // the release is out: BPTT state, then reuse sH
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int b = b0 + col0 + i;
        if (b < B && col0 + i < nrow) {
          const size_t n = (size_t)t * B + b;
          *reinterpret_cast<uint2*>(P.gates + n * (8 * kH) + gcol) = gp[i];
          P.cstate[n * (2 * kH) + dir * kH + unit] = c[i];
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  if (warp == 2) tmem_dealloc_pair(tmem, 512);
}

// ============================================================================
// Backward: split-K over a 4-CTA cluster.
//   cluster = (dir, batch tile, unit group ug of 64 units); CTA rank ks holds
//   W_hh[gate rows ks*512 .. +512][64 units of ug] (64 KB, read as an
//   MN-major operand straight from the bf16 snapshot) and streams the
//   matching 512-row K slice of dG_prev (128 KB, all 8 chunks in flight).
//   Partial dh[128 batch, 64 units] (TMEM) is exchanged through DSMEM: CTA ks
//   finalises units ug*64 + ks*16 .. +16, runs their cell backward and writes
//   exactly one 64-gate-row chunk (chunk id ug*4 + ks) of dG_t.
namespace bwd {
constexpr int kKS = 4;                       // K splits (DSMEM exchange group)
// Multicasting each A slice to the two unit groups of an 8-CTA cluster halves
// the L2 reads but measured slower (one batch-tile group ran ~3x behind), so
// the kernel runs with 4-CTA clusters and per-CTA loads.
constexpr bool kMulticastB = false;
constexpr int kClB = kMulticastB ? 8 : 4;
constexpr int kGU = 64;                      // units per cluster
constexpr int kFU = kGU / kKS;               // 16 units finalised per CTA
constexpr int kKSlice = 4 * kH / kKS;        // 512 gate rows per CTA
constexpr int kChunks = kKSlice / 64;        // 8 A chunks per step
constexpr int kStagesB = 8;                 // the whole step's dG slice in flight
constexpr int kWBytesB = kGU * kKSlice * 2;  // 64 KB
// partial dh travels as fp16 scaled by P.xscale (a power of two ~ frames/2,
// so the mean-loss gradients sit in fp16's normal range; 11-bit mantissa)
constexpr int kRecvSlot = 128 * kFU * 2;     // 4 KB: one source's [128 rows x 16 units] fp16
constexpr int kRecvBytes = kKS * kRecvSlot;  // 4 sources
constexpr int kSendBytes = (kKS - 1) * kRecvSlot;  // staged partials for the 3 peers
constexpr size_t kSmem = 1024 + kWBytesB + kStagesB * kTileA + kRecvBytes + kSendBytes + 512;
// [128 rows][16 fp16] slots, 16-byte chunk c of row r stored at chunk c ^ ((r >> 2) & 1)
__device__ __forceinline__ uint32_t slot_off(int r, int c) { return (uint32_t)(r * 32 + 16 * (c ^ ((r >> 2) & 1))); }
__device__ __forceinline__ uint4 pack_h8(const float* v, float sc) {
  uint4 w;
  uint32_t* u = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __half2 h = __floats2half2_rn(v[2 * i] * sc, v[2 * i + 1] * sc);
    u[i] = *reinterpret_cast<uint32_t*>(&h);
  }
  return w;
}
}  // namespace bwd

__global__ void __launch_bounds__(kThreads, 1) lstm_bwd_kernel(const __grid_constant__ LstmParams P) {
  using namespace bwd;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sW = sm;
  uint8_t* sA = sW + kWBytesB;
  uint8_t* recv = sA + kStagesB * kTileA;  // [kKS][128][16] fp16 (swizzled rows)
  uint8_t* send = recv + kRecvBytes;      // [kKS-1][128][16] fp16
  uint64_t* bars = reinterpret_cast<uint64_t*>(send + kSendBytes);
  uint64_t* full = bars;
  uint64_t* empty = full + kStagesB;
  uint64_t* wbar = empty + kStagesB;
  uint64_t* tfull = wbar + 1;    // [2] double-buffered accumulators: MMA iteration i = s-1 uses i & 1
  uint64_t* tempty = tfull + 2;
  uint64_t* rfull = tempty + 2;  // recv buffer complete (all 4 sources)
  uint64_t* rfree = rfull + 1;   // my last partials were consumed by the 3 peer finalisers
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rfree + 1);

  const uint32_t warp = warp_id(), lane = lane_id();
  const int crank = (int)cluster_ctarank();
  const int ks = crank % kKS;
  const int upair = crank / kKS;              // which unit group of the cluster
  const uint32_t rbase = (uint32_t)(upair * kKS);  // cluster rank of (this ug, ks = 0)
  const uint16_t pair_mask = (uint16_t)((1u << ks) | (1u << (kKS + ks)));
  const int ug = (blockIdx.x / kKS) % (kH / kGU);
  const int btile = (blockIdx.x / (kKS * (kH / kGU))) % P.n_btile;
  const int dir = blockIdx.x / (kKS * (kH / kGU) * P.n_btile);
  uint32_t* flags = P.counters + (size_t)(P.b0 / 128 + btile) * kFlagWords128 + dir * kGroupFlagWords;
  const int T = P.T, B = P.B;
  const int brow0 = P.b0 + btile * 128;
  const int my_chunk = ug * kKS + ks;
  __shared__ uint32_t s_base;

  if (warp == 1 && lane == 0) {
    for (int i = 0; i < kStagesB; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kMulticastB ? 2 : 1);  // both CTAs of a multicast pair free the stage
    }
    mbar_init(wbar, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], kEpiThreads);
    }
    mbar_init(rfull, 1);  // local expect_tx arrive; peers complete 3 x 8 KB of tx
    mbar_init(rfree, kKS - 1);  // remote arrives of the 3 finalisers fed by this CTA
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 128);
  tc_fence_before();
  cluster_sync_all();  // peers' barriers initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) {  // programmatic launch: W_hh slice first, flag base after the wait (see forward)
    tma_prefetch_desc(&P.tmA);
    tma_prefetch_desc(&P.tmW);
    mbar_arrive_expect_tx(wbar, kWBytesB);
    for (int j = 0; j < kChunks; ++j)  // W_hh rows (K) ks*512 + 64j.., units (N) ug*64..: MN-major boxes
      tma_load_2d(sW + j * 8192, &P.tmW, wbar, ug * kGU, dir * 4 * kH + ks * kKSlice + j * 64);
  }
  griddep_wait();
  if (threadIdx.x == 0) s_base = ld_relaxed_gpu(bwd_flag(flags, my_chunk));
  __syncthreads();
  const uint32_t base = s_base;  // flag value at launch start (same for every chunk of the group)

  if (warp == 0) {
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      FlagSeg seg;
#pragma unroll
      for (int i = 0; i < 8; ++i) seg.v[i] = 0;
      const uint32_t* myseg = flags + ks * kFlagLine;  // chunks 8ks .. 8ks+7
      for (int s = 1; s < T; ++s) {
        const int t = dir == 0 ? T - 1 - s : s;
        const int tprev = dir == 0 ? t + 1 : t - 1;
        const int arow = tprev * B + brow0;
        for (int j = 0; j < kChunks; ++j) {
          const int chunk = ks * kChunks + j;
          mbar_wait(&empty[stage], phase ^ 1);  // both CTAs of the pair freed it
          mbar_arrive_expect_tx(&full[stage], kTileA);
          if (kMulticastB) {  // the pair alternates chunks; multicast to both
            if ((j & 1) == upair) {
              wait_flag(bwd_flag(flags, chunk), base + (uint32_t)s, P.err);
              acquire_for_tma(bwd_flag(flags, chunk), P.variant);
              tma_load_2d_mc(sA + stage * kTileA, &P.tmA, &full[stage], dir * 4 * kH + chunk * 64, arow,
                             pair_mask);
            }
          } else {
            if (P.variant & 256) {  // experiment: relaxed polls, one acquire load once satisfied
              if (!reached(seg.v[j], base + (uint32_t)s)) {
                do ld_relaxed_gpu_v8(myseg, seg.v);
                while (!reached(seg.v[j], base + (uint32_t)s));
                ld_acquire_gpu_v8(myseg, seg.v);
              }
            } else {
              wait_seg<1>(seg, myseg, j, base + (uint32_t)s, P.err);  // one 32-byte acquire poll covers the step's 8 chunks
            }
            if (!(P.variant & 128)) fence_proxy_async_global();
            tma_load_2d(sA + stage * kTileA, &P.tmA, &full[stage], dir * 4 * kH + chunk * 64, arow);
            if (P.trace && blockIdx.x == 0)
              P.trace[(size_t)gridDim.x * T * kTraceSlots + ((size_t)s * 8 + j) * 2] = globaltimer();
          }
          if (j == 0) trace_mark(P.trace, T, s, 0);
          if (++stage == kStagesB) {
            stage = 0;
            phase ^= 1;
          }
        }
        trace_mark(P.trace, T, s, 1);
      }
    }
  } else if (warp == 1) {
    mbar_wait(wbar, 0);
    const uint32_t idesc = idesc_bf16_f32(128, kGU, 0, 1);  // B = W_hh slice, MN-major (units contiguous)
    const uint32_t wbase = smem_u32(sW);
    int stage = 0;
    uint32_t phase = 0;
    for (int s = 1; s < T; ++s) {
      const int it = s - 1, acc = it & 1;
      mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t dacc = tmem + acc * kGU;
      for (int j = 0; j < kChunks; ++j) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (P.trace && blockIdx.x == 0 && lane == 0)
          P.trace[(size_t)gridDim.x * T * kTraceSlots + ((size_t)s * 8 + j) * 2 + 1] = globaltimer();
        if (elect_one()) {
          const uint32_t abase = smem_u32(sA + stage * kTileA);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            uint64_t ad = smem_desc_sw128(abase + k * 32, 16, 1024);
            uint64_t bd = smem_desc_sw128(wbase + j * 8192 + k * 2048, 8192, 1024);
            mma_bf16_ss(dacc, ad, bd, idesc, (j | k) != 0);
          }
          if (kMulticastB)
            mma_commit_mc(&empty[stage], pair_mask);
          else
            mma_commit(&empty[stage]);
          if (j == kChunks - 1) mma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++stage == kStagesB) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp >= kEpiWarp0) {
    const uint32_t e = warp - kEpiWarp0;
    const uint32_t q = e & 3;
    const uint32_t hf = e >> 2;
    const int r = q * 32 + lane;
    const int b = brow0 + r;
    const bool ok = (r + btile * 128 < P.nb) && b < B;
    // exchange: this thread's partial columns hf*32 .. +32 = finalisers 2hf, 2hf+1
    const uint32_t tcol = tmem + ((q * 32) << 16) + hf * 32;
    // cell backward: row r, units ug*64 + ks*16 + hf*8 .. +8
    const int unit0 = ug * kGU + ks * kFU + hf * 8;
    const int col_g = dir * 4 * kH + unit0 * 4;
    const int col_u = dir * kH + unit0;
    const uint32_t recv_base = smem_u32(recv);
    float dcc[8], dbacc[32];
#pragma unroll
    for (int u = 0; u < 8; ++u) dcc[u] = 0.f;
#pragma unroll
    for (int i = 0; i < 32; ++i) dbacc[i] = 0.f;
    for (int s = 0; s < T; ++s) {
      if (s == T - 1) griddep_launch();  // the next kernel may start its prologue
      const int t = dir == 0 ? T - 1 - s : s;
      const int tc = dir == 0 ? t - 1 : t + 1;
      const bool has_cprev = tc >= 0 && tc < T;
      const size_t n = (size_t)t * B + b;
      uint4 apre[4], dypre;
      float4 cpre[2], cppre[2];
      if (ok) {
        const uint4* ap = reinterpret_cast<const uint4*>(P.gates + n * (8 * kH) + col_g);
#pragma unroll
        for (int j = 0; j < 4; ++j) apre[j] = ap[j];
        dypre = *reinterpret_cast<const uint4*>(P.dy + n * (2 * kH) + col_u);
        const float4* cp = reinterpret_cast<const float4*>(P.cstate + n * (2 * kH) + col_u);
        cpre[0] = cp[0];
        cpre[1] = cp[1];
        if (has_cprev) {
          const float4* pp = reinterpret_cast<const float4*>(P.cstate + ((size_t)tc * B + b) * (2 * kH) + col_u);
          cppre[0] = pp[0];
          cppre[1] = pp[1];
        } else {
          cppre[0] = cppre[1] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      float dh[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) dh[u] = 0.f;
      if (s > 0) {
        const int it = s - 1;
        mbar_wait(&tfull[it & 1], (it >> 1) & 1);
        tc_fence_after();
        if (e == 0 && lane == 0) trace_mark(P.trace, T, s, 2);
        float v[32];
        tmem_ld32(tcol + (it & 1) * kGU, v);
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&tempty[it & 1]);
        const bool issuer = (threadIdx.x == kEpiWarp0 * 32);
        if (issuer && s >= 2) bulk_wait_read0();  // last step's copies have read `send`
        named_bar_sync(3, kEpiThreads);
        // my partial for finalisers 2hf, 2hf+1: own slot in recv, peers' in send
#pragma unroll
        for (int f2 = 0; f2 < 2; ++f2) {
          const int f = 2 * hf + f2;
          uint8_t* slot = f == ks ? reinterpret_cast<uint8_t*>(recv) + ks * kRecvSlot
                                  : send + (f < ks ? f : f - 1) * kRecvSlot;
#pragma unroll
          for (int c = 0; c < 2; ++c)
            *reinterpret_cast<uint4*>(slot + slot_off(r, c)) = pack_h8(v + f2 * kFU + 8 * c, P.xscale);
        }
        fence_proxy_async_smem();
        named_bar_sync(3, kEpiThreads);
        if (issuer) {
          // the finalisers we feed consumed our previous partials (cluster
          // mbarrier: no global-memory polling next to the chunk flags)
          if (s >= 2) mbar_wait_acq_cluster(rfree, (uint32_t)(s - 2) & 1);
          for (int f = 0; f < kKS; ++f) {
            if (f == ks) continue;
            const uint32_t peer = rbase + (uint32_t)f;
            const uint32_t dst = mapa_shared(smem_u32(reinterpret_cast<uint8_t*>(recv) + ks * kRecvSlot), peer);
            bulk_copy_s2cluster(dst, send + (f < ks ? f : f - 1) * kRecvSlot, kRecvSlot,
                                mapa_shared(smem_u32(rfull), peer));
          }
          bulk_commit();
          mbar_arrive_expect_tx(rfull, (kKS - 1) * kRecvSlot);
        }
        mbar_wait(rfull, (s - 1) & 1);
        if (e == 0 && lane == 0) trace_mark(P.trace, T, s, 5);
        const uint8_t* rb = reinterpret_cast<const uint8_t*>(recv);
#pragma unroll
        for (int src = 0; src < kKS; ++src) {
          const uint4 w = *reinterpret_cast<const uint4*>(rb + src * kRecvSlot + slot_off(r, hf));
          const __half2* hx = reinterpret_cast<const __half2*>(&w);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float2 f = __half22float2(hx[i]);
            dh[2 * i] += f.x;
            dh[2 * i + 1] += f.y;
          }
        }
        const float inv = 1.f / P.xscale;
#pragma unroll
        for (int i = 0; i < 8; ++i) dh[i] *= inv;
        named_bar_sync(3, kEpiThreads);  // every thread has read this exchange
        if (issuer) {
          for (int f = 0; f < kKS; ++f)
            if (f != ks) mbar_arrive_remote(mapa_shared(smem_u32(rfree), rbase + (uint32_t)f));  // CTA-scope release: no GPU membar
        }
      }
      if (ok) {
        float dyv[8], cc[8], cp[8];
        bf16x8_to_f32(dypre, dyv);
        cc[0] = cpre[0].x; cc[1] = cpre[0].y; cc[2] = cpre[0].z; cc[3] = cpre[0].w;
        cc[4] = cpre[1].x; cc[5] = cpre[1].y; cc[6] = cpre[1].z; cc[7] = cpre[1].w;
        cp[0] = cppre[0].x; cp[1] = cppre[0].y; cp[2] = cppre[0].z; cp[3] = cppre[0].w;
        cp[4] = cppre[1].x; cp[5] = cppre[1].y; cp[6] = cppre[1].z; cp[7] = cppre[1].w;
        uint4* dgrow = reinterpret_cast<uint4*>(P.dg + n * (8 * kH) + col_g);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float act[8], dgv[8];
          bf16x8_to_f32(apre[j], act);
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const int u = 2 * j + h2;
            const float ig = act[4 * h2 + 0], fg = act[4 * h2 + 1], gg = act[4 * h2 + 2], og = act[4 * h2 + 3];
            const float dht = dh[u] + dyv[u];
            const float tcn = tanh_fast(cc[u]);
            const float dct = fmaf(dht * og, 1.f - tcn * tcn, dcc[u]);
            dgv[4 * h2 + 0] = dct * gg * ig * (1.f - ig);
            dgv[4 * h2 + 1] = dct * cp[u] * fg * (1.f - fg);
            dgv[4 * h2 + 2] = dct * ig * (1.f - gg * gg);
            dgv[4 * h2 + 3] = dht * tcn * og * (1.f - og);
            dcc[u] = dct * fg;
          }
          dgrow[j] = f32_to_bf16x8(dgv);
#pragma unroll
          for (int i = 0; i < 8; ++i) dbacc[8 * j + i] += dgv[i];
        }
      }
      if (e == 0 && lane == 0) trace_mark(P.trace, T, s, 3);
      publish(bwd_flag(flags, my_chunk), base + (uint32_t)(s + 1), P.variant);
      if (e == 0 && lane == 0) trace_mark(P.trace, T, s, 4);
    }
    if (threadIdx.x == kEpiWarp0 * 32) bulk_wait0();  // outgoing exchange copies complete
    if (P.dbpart) {  // fused bias gradient: sum over this warp's 32 batch rows and all steps
      const float cs = warp_colsum32(dbacc, lane);
      P.dbpart[((size_t)(P.b0 / 128 + btile) * 4 + q) * (8 * kH) + col_g + lane] = cs;
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // no CTA leaves while a peer may still touch its smem
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 128);
}

// ============================================================================
// Backward, transposed (default): dh^T[units, batch] = W_hh^T[units, gates] .
// dG^T[gates, batch], so the weights are the stationary M operand read from
// tensor memory and the freshly produced dG is the streamed B operand in its
// natural [frame, gate] layout.
//   cluster of 8 = (dir, 128-row batch tile, unit half uh of 256 units);
//   cluster rank = 2*ks + r: CTA pair ks (tcgen05 cta_group::2) owns gate
//   slice ks (gate rows ks*512 .. +512 of the direction = units ks*128 ..
//   +128, all four gates) and rank r holds units uh*256 + r*128 .. +128 as
//   TMEM lanes with W_hh^T[its units][slice] (128 KB, columns 256..511).
//   Per step the pair issues 32 M256 N128 K16 MMAs (A from TMEM, B = the
//   slice's 8 dG chunks of 64 gate columns, each CTA staging its 64 batch
//   rows) into a double-buffered fp32 accumulator [128 units, 128 batch].
//   The four K-slices' partials are reduce-scattered through DSMEM (fp16,
//   power-of-two scaled): lane quadrant q of CTA (ks, r) goes to CTA (q, r),
//   which then owns 32 units x 128 rows: it sums the four partials in slice
//   order, runs the cell backward, writes two 64-column dG chunks and
//   publishes one flag.  The next step's consumers of those chunks are the
//   four CTAs of slice uh*2 + r (both unit halves, both batch halves).
//   64 CTAs at B = 256 instead of 128, 4x less dG traffic through L2, and a
//   per-step MMA chain measured at 1.6 us instead of 2.06 us
//   (tools/micro/rec_chain.cu).
namespace bwd3 {
constexpr int kKS = 4;                     // gate slices (split-K) = finalisers per unit block
constexpr int kSlice = 4 * kH / kKS;       // 512 gate rows per slice
constexpr int kUnits = 128;                // units per CTA (TMEM lanes)
constexpr int kFin = kUnits / kKS;         // 32 units finalised per CTA
constexpr int kRows = 128;                 // batch rows per tile (MMA N)
constexpr int kHalfRows = kRows / 2;       // staged per CTA (N split across the pair)
constexpr int kChunk = kHalfRows * 128;    // 8 KB: 64 rows x 64 gate columns bf16, SWIZZLE_128B
constexpr int kChunks = kSlice / 64;       // 8 B chunks per step
constexpr int kStages = 7;                 // (8 measured no faster; the 8 KB pay for the second dY input)
constexpr int kPitch = 144;                // bytes per unit row of an exchange block (64 fp16 + pad)
constexpr int kBlock = kFin * kPitch;      // 4608: one (source slice, batch half) block
constexpr int kRecvBuf = kKS * 2 * kBlock; // one step's incoming partials (own + 3 peers)
constexpr int kSendBytes = (kKS - 1) * 2 * kBlock;
constexpr int kWBytes = kSlice * kUnits * 2;  // 128 KB W slice, staged once (aliases ring + recv)
constexpr int kRingBytes = kStages * kChunk;
constexpr int kInG = kRows * kFin * 4 * 2;  // 32 KB
constexpr int kInC = kRows * kFin * 4;      // 16 KB
constexpr int kInDY = kRows * kFin * 2;     // 8 KB per dY input (dY, or the two per-direction halves of a streamed dX)
constexpr size_t kSmem = 1024 + kRingBytes + 2 * kRecvBuf + kSendBytes + kInG + kInC + 2 * kInDY + 256;
static_assert(kWBytes <= kRingBytes + 2 * kRecvBuf + kSendBytes, "W staging must fit in the ring + recv + send region");
static_assert(kSmem <= 232448, "shared memory");
static_assert(kChunks == kStages + 1, "producer lanes: chunk 7 reuses the stage of the same step's chunk 0");
constexpr uint32_t kACol = 256;            // A = W^T slice at TMEM columns 256..511 (two bf16 per column)
constexpr int kEpi = 16;                   // epilogue warps 0..15 (warp % 4 = TMEM lane quadrant)
constexpr int kProdWarp = 16, kMmaWarp = 17;  // TMA producer, MMA issuer (+ TMEM allocation)
constexpr int kThreads3 = 32 * (kEpi + 2);
constexpr int kCellRows = kRows / kEpi;    // 8 batch rows per finaliser thread
// flags: lines 4..7 of the backward group area (the split-K kernel uses lines 0..3);
// producer (slice sigma = 2*uh + r, ks) publishes word sigma*32 + ks
constexpr int kFlagLine0 = 4;
}  // namespace bwd3

// stage one step's cell-backward inputs of a finaliser (32 units x 128 batch rows) in smem
__device__ __forceinline__ void issue_inputs(const LstmParams& P, uint64_t* bar, uint8_t* g, uint8_t* c, uint8_t* dy,
                                             int t, int tc, int brow0, int dir, int unit0) {
  const bool cprev = tc >= 0 && tc < P.T;
  mbar_arrive_expect_tx(bar, bwd3::kInG + (P.dy2 ? 2 : 1) * bwd3::kInDY + (cprev ? bwd3::kInC : 0));
  const int row = t * P.B + brow0;
  tma_load_2d(g, &P.tmG, bar, dir * 4 * kH + unit0 * 4, row);
  if (P.dyready) {  // dY of (t, dir) written by the GEMM streaming behind the previous BPTT (both halves)
    for (int src = 0; src < (P.dy2 ? 2 : 1); ++src) {
      const uint32_t* w = P.dyready + (2 * t + dir) * 2 + src;
      if (ld_acquire_gpu(w) < P.dyready_target) {
        SpinGuard sg;
        while (ld_acquire_gpu(w) < P.dyready_target)
          if (spin_expired(sg, P.err)) break;
      }
    }
    fence_proxy_async_global();
  }
  tma_load_2d(dy, &P.tmDY, bar, dir * kH + unit0, row);
  if (P.dy2) tma_load_2d(dy + bwd3::kInDY, &P.tmDY2, bar, dir * kH + unit0, row);
  if (cprev) tma_load_2d(c, &P.tmC, bar, dir * kH + unit0, tc * P.B + brow0);
}

__global__ void __launch_bounds__(bwd3::kThreads3, 1) lstm_bwd3_kernel(const __grid_constant__ LstmParams P) {
  using namespace bwd3;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = sm;                       // [kStages][64 rows x 128 B]
  uint8_t* recv = ring + kRingBytes;        // [2][src slice 4][batch half 2][32 units][kPitch]
  uint8_t* send = recv + 2 * kRecvBuf;      // [dst 3][batch half 2][32 units][kPitch]
  uint8_t* in_g = send + kSendBytes;        // next step's cell inputs: gates [128 rows][32 units x 4] bf16
  uint8_t* in_c = in_g + kInG;              //   c_{t-1} [128 rows][32] f32
  uint8_t* in_dy = in_c + kInC;             //   dY [128 rows][32] bf16 (+ the second half at in_dy + kInDY)
  uint8_t* wstage = ring;                   // launch only: [unit half 2][512 gate rows][64 units] bf16
  uint64_t* bars = reinterpret_cast<uint64_t*>(in_dy + 2 * kInDY);
  uint64_t* full = bars;                    // [kStages] leader only: both CTAs' chunk bytes
  uint64_t* empty = full + kStages;         // [kStages] per CTA: the pair's MMAs read the stage
  uint64_t* wbar = empty + kStages;
  uint64_t* tfull = wbar + 1;               // [2] per CTA (commit multicast)
  uint64_t* tempty = tfull + 2;             // [2] leader: every epilogue warp of both CTAs
  uint64_t* rfull = tempty + 2;             // [2] my recv buffer complete
  uint64_t* rfree = rfull + 2;              // [2] my 3 destinations read their recv buffer
  uint64_t* inbar = rfree + 2;              // cell inputs landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(inbar + 1);
  __shared__ uint32_t s_base;

  const uint32_t warp = warp_id(), lane = lane_id();
  const uint32_t crank = cluster_ctarank();
  const int ks = (int)(crank >> 1), r = (int)(crank & 1);
  const bool leader = r == 0;
  const uint32_t pair0 = crank & ~1u;
  const int cl = blockIdx.x >> 3;
  const int uh = cl & 1;
  const int btile = (cl >> 1) % P.n_btile;
  const int dir = (cl >> 1) / P.n_btile;
  const int T = P.T, B = P.B;
  const int brow0 = P.b0 + btile * kRows;
  const int ubase = uh * 256 + r * 128;     // my 128 units (TMEM lanes)
  uint32_t* flags =
      P.counters + (size_t)(P.b0 / 128 + btile) * kFlagWords128 + dir * kGroupFlagWords + kFlagLine0 * kFlagLine;
  uint32_t* myflag = flags + (uh * 2 + r) * kFlagLine + ks;

  if (threadIdx.x == 0) trace_mark(P.trace, T, 0, 0);  // (slot 0 of step 0 is unused below: launch start)
  if (warp == kProdWarp && lane == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(wbar, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 2 * kEpi);
      mbar_init(&rfull[i], 1);
      mbar_init(&rfree[i], kKS - 1);
    }
    mbar_init(inbar, 1);
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc_pair(tmem_slot, 512);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // programmatic launch: the W_hh slice (operand snapshot, not written by the predecessor) first
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&P.tmA);
    tma_prefetch_desc(&P.tmW);
    tma_prefetch_desc(&P.tmG);
    tma_prefetch_desc(&P.tmC);
    tma_prefetch_desc(&P.tmDY);
    if (P.dy2) tma_prefetch_desc(&P.tmDY2);
    mbar_arrive_expect_tx(wbar, kWBytes);
    for (int uq = 0; uq < 2; ++uq)
      for (int kh = 0; kh < 2; ++kh)
        tma_load_2d(wstage + uq * 65536 + kh * 32768, &P.tmW, wbar, ubase + uq * 64,
                    dir * 4 * kH + ks * kSlice + kh * 256);
  }
  if (warp < kEpi) {
    // W^T into tensor memory: lane = unit, column c = gate rows (2c, 2c+1) of the slice
    const uint32_t e = warp, q = e & 3, cq = e >> 2;
    const int m = (int)(q * 32 + lane);
    const uint16_t* wsrc = reinterpret_cast<const uint16_t*>(wstage + (m >> 6) * 65536) + (m & 63);
    mbar_wait(wbar, 0);
    uint32_t rr[16];
    for (int c0 = (int)cq * 64; c0 < (int)cq * 64 + 64; c0 += 16) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int k = 2 * (c0 + j);
        rr[j] = (uint32_t)wsrc[k * 64] | ((uint32_t)wsrc[(k + 1) * 64] << 16);
      }
      tmem_st16(tmem + ((q * 32) << 16) + kACol + (uint32_t)c0, rr);
    }
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // both halves of A in TMEM; every CTA done with its staging area
  tc_fence_after();
  griddep_wait();
  if (threadIdx.x == 0) s_base = ld_relaxed_gpu(myflag);
  if (threadIdx.x == 0 && blockIdx.x == 0 && P.seq) {  // started: release GEMMs gated on this launch
    st_release_gpu(P.seq + 1, ld_relaxed_gpu(P.seq) * 16u + (uint32_t)P.tag);  // epoch: bumped by the step's gather
  }
  __syncthreads();
  if (threadIdx.x == 0) trace_mark(P.trace, T, 0, 1);  // prologue done (W^T in TMEM, predecessor waited)
  const uint32_t base = s_base;  // flag value at launch start (same for every flag of the group)

  if (warp == kProdWarp) {
    // lane j stages chunk j of every step: the chunks' stage waits, byte counts, flag polls and TMA
    // issues run side by side (one issuing thread spent ~260 cycles per chunk on them in sequence,
    // ~1.1 us per step before the last chunk was in flight).  Parity waits on the 7-stage ring stay
    // sound as long as a stage's previous use was issued before its next wait: chunks 0..6 of a step
    // reuse stages of the previous step's chunks 1..7 (issued before the step's first __syncwarp), and
    // chunk 7 reuses the stage of the same step's chunk 0, so it waits after the lanes 0..6 issued.
    const int j = (int)lane;
    if (j < kChunks) {
      const uint32_t full_c = mapa_shared(smem_u32(full), pair0);
      const uint32_t* word = flags + ks * kFlagLine + (j >> 1);  // producer of my chunk (2 chunks each)
      for (int s = 1; s < T; ++s) {
        const int t = dir == 0 ? T - 1 - s : s;
        const int tprev = dir == 0 ? t + 1 : t - 1;
        const int arow = tprev * B + brow0 + r * kHalfRows;
        const int g = (s - 1) * kChunks + j;  // running chunk count: ring stage and phase
        const int stage = g % kStages;
#pragma unroll 1
        for (int round = 0; round < 2; ++round) {
          if ((j == kChunks - 1) == (round == 1)) {
            mbar_wait(&empty[stage], ((uint32_t)(g / kStages) & 1u) ^ 1u);
            if (leader) mbar_arrive_expect_tx(&full[stage], 2 * kChunk);
            const uint32_t target = base + (uint32_t)s;
            if (!reached(ld_acquire_gpu(word), target)) {
              SpinGuard sg;
              while (!reached(ld_acquire_gpu(word), target))
                if (spin_expired(sg, P.err)) break;
            }
            fence_proxy_async_global();
            if (j == 0) trace_mark(P.trace, T, s, 0);
            tma_load_2d_pair(ring + stage * kChunk, &P.tmA, full_c + (uint32_t)stage * 8,
                             dir * 4 * kH + ks * kSlice + j * 64, arow);
            if (P.trace && blockIdx.x == 0)
              P.trace[(size_t)gridDim.x * T * kTraceSlots + ((size_t)s * 8 + j) * 2] = globaltimer();
            if (j == kChunks - 1) trace_mark(P.trace, T, s, 1);
          }
          __syncwarp(0xffu);
        }
      }
    }
  } else if (warp == kMmaWarp) {
    if (leader) {
      const uint32_t idesc = idesc_bf16_f32(256, kRows, 0, 0);
      const uint16_t mask = (uint16_t)(3u << pair0);
      int stage = 0;
      uint32_t phase = 0;
      for (int s = 1; s < T; ++s) {
        const int it = s - 1, acc = it & 1;
        mbar_wait_acq_cluster(&tempty[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t dacc = tmem + (uint32_t)acc * kRows;
        if (P.variant & 2) {  // experiment: all chunks landed before the first MMA (kStages == kChunks)
          for (int j = 0; j < kChunks; ++j) mbar_wait(&full[j], phase);
          if (P.trace && blockIdx.x == 0 && lane == 0)
            P.trace[(size_t)gridDim.x * T * kTraceSlots + ((size_t)s * 8 + 0) * 2 + 1] = globaltimer();
        }
        for (int j = 0; j < kChunks; ++j) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (P.trace && blockIdx.x == 0 && lane == 0)
            P.trace[(size_t)gridDim.x * T * kTraceSlots + ((size_t)s * 8 + j) * 2 + 1] = globaltimer();
          if (elect_one()) {
            const uint32_t bb = smem_u32(ring + stage * kChunk);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_bf16_ts_pair(dacc, tmem + kACol + (uint32_t)(j * 4 + kk) * 8, smem_desc_sw128(bb + kk * 32, 16, 1024),
                               idesc, (j | kk) != 0);
            if (!(P.variant & 1)) mma_commit_pair_mc(&empty[stage], mask);
            if (j == kChunks - 1) {
              mma_commit_pair_mc(&tfull[acc], mask);
              if (P.variant & 1)
                for (int st = 0; st < kStages; ++st) mma_commit_pair_mc(&empty[st], mask);
            }
          }
          __syncwarp();
          if ((P.variant & 4) && j == kChunks - 1 && P.trace && blockIdx.x == 0) {
            if (lane == 0) {
              P.trace[(size_t)gridDim.x * T * kTraceSlots + (size_t)T * 16 + 2 * s] = globaltimer();
              mbar_wait(&tfull[acc], (it >> 1) & 1);
              P.trace[(size_t)gridDim.x * T * kTraceSlots + (size_t)T * 16 + 2 * s + 1] = globaltimer();
            }
            __syncwarp();
          }
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else {
    const uint32_t e = warp;
    const uint32_t q = e & 3, cg = e >> 2;    // partial: lane quadrant q, batch columns cg*32 .. +32
    const uint32_t half = cg >> 1;            // exchange block (batch half) of those columns
    const int fh = (int)(e >> 3), fr = (int)(e & 7) * kCellRows;  // finaliser: batch half fh, rows fr .. +8
    const int unit = ubase + ks * kFin + (int)lane;               // finalised unit (lane)
    const int col_g = dir * 4 * kH + unit * 4;
    const int col_u = dir * kH + unit;
    const int row0 = fh * kHalfRows + fr;                         // first of my 8 rows within the tile
    const uint32_t tcol = tmem + ((q * 32) << 16) + cg * 32;
    const uint32_t tempty_c = mapa_shared(smem_u32(tempty), pair0);
    const int sidx = (int)q < ks ? (int)q : (int)q - 1;           // send slot for destination q
    const bool issuer = (cg & 1) == 0;                            // copies the (q, half) block
    const uint32_t pbar = 4 + q * 2 + half;                       // named barrier of the two warps of a block
    const bool kEpiLead = threadIdx.x == 0;
    uint32_t okmask = 0;  // my rows inside the batch and this launch
#pragma unroll
    for (int i = 0; i < kCellRows; ++i)
      okmask |= (row0 + i + btile * kRows < P.nb && brow0 + row0 + i < B ? 1u : 0u) << i;
    const uint32_t cg_in = smem_u32(in_g) + row0 * 256 + lane * 8;  // staged inputs of my (unit, first row)
    const uint32_t cc_in = smem_u32(in_c) + row0 * 128 + lane * 4;
    const uint32_t cdy_in = smem_u32(in_dy) + row0 * 64 + lane * 2;
    float dcc[kCellRows], cc[kCellRows], db[4];  // cc: c_t of my rows (c_{t-1} becomes the next step's c_t)
#pragma unroll
    for (int i = 0; i < kCellRows; ++i) dcc[i] = 0.f;
#pragma unroll
    for (int g = 0; g < 4; ++g) db[g] = 0.f;
    for (int s = 0; s < T; ++s) {
      if (s == T - 1) griddep_launch();
      const int t = dir == 0 ? T - 1 - s : s;
      const int tc = dir == 0 ? t - 1 : t + 1;
      const bool has_cprev = tc >= 0 && tc < T;
      if (s == 0) {  // first step: c_t from global; every step's gates / c_{t-1} / dY are staged by TMA
        if (kEpiLead) issue_inputs(P, inbar, in_g, in_c, in_dy, t, tc, brow0, dir, ubase + ks * kFin);
#pragma unroll
        for (int i = 0; i < kCellRows; ++i) {
          const int b = brow0 + row0 + i;
          cc[i] = b < B ? P.cstate[((size_t)t * B + b) * (2 * kH) + col_u] : 0.f;
        }
      }
      float dh[kCellRows];
#pragma unroll
      for (int i = 0; i < kCellRows; ++i) dh[i] = 0.f;
      if (s > 0) {
        const int it = s - 1, acc = it & 1, buf = it & 1;
        uint8_t* rb = recv + buf * kRecvBuf;
        const bool remote = q != (uint32_t)ks;
        if (remote) {
          if (issuer && lane == 0 && it >= 1) bulk_wait_read0();  // the block's last copy has read `send`
          named_bar_sync(pbar, 64);
        }
        mbar_wait(&tfull[acc], (it >> 1) & 1);
        tc_fence_after();
        if (e == 0 && lane == 0) trace_mark(P.trace, T, s, 2);
        float v[32];
        tmem_ld32(tcol + (uint32_t)acc * kRows, v);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (leader)
            mbar_arrive(&tempty[acc]);
          else
            mbar_arrive_remote(tempty_c + (uint32_t)acc * 8);
        }
        // my partial for finaliser q: [32 units (lanes)][32 batch] fp16 into the (q, half) block
        uint8_t* blk = remote ? send + (sidx * 2 + half) * kBlock : rb + (ks * 2 + half) * kBlock;
        uint8_t* dst = blk + lane * kPitch + (cg & 1) * 64;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint4 w;
          uint32_t* u = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            __half2 h2 = __floats2half2_rn(v[c * 8 + 2 * i] * P.xscale, v[c * 8 + 2 * i + 1] * P.xscale);
            u[i] = *reinterpret_cast<uint32_t*>(&h2);
          }
          *reinterpret_cast<uint4*>(dst + c * 16) = w;
        }
        if (remote) {
          fence_proxy_async_smem();
          named_bar_sync(pbar, 64);
          if (issuer && lane == 0) {
            if (it >= 2) mbar_wait_acq_cluster(&rfree[buf], ((it >> 1) & 1) ^ 1);
            const uint32_t peer = q * 2 + (uint32_t)r;
            bulk_copy_s2cluster(mapa_shared(smem_u32(rb + (ks * 2 + half) * kBlock), peer), blk, kBlock,
                                mapa_shared(smem_u32(&rfull[buf]), peer));
            bulk_commit();
          }
        }
        named_bar_sync(3, kEpi * 32);  // own-slice partials in recv; local expect below
        if (kEpiLead) mbar_arrive_expect_tx(&rfull[buf], (kKS - 1) * 2 * kBlock);
        // the peers' partials arrive by bulk copies completing on rfull (async proxy, complete_tx): the
        // phase flip makes them visible like a TMA load's, no cluster-scope acquire (an L1 invalidation
        // per waiting warp) needed
        mbar_wait(&rfull[buf], (it >> 1) & 1);
        if (e == 0 && lane == 0) trace_mark(P.trace, T, s, 5);
#pragma unroll
        for (int src = 0; src < kKS; ++src) {
          const uint4 w0 = *reinterpret_cast<const uint4*>(rb + (src * 2 + fh) * kBlock + lane * kPitch + fr * 2);
          const __half2* h0 = reinterpret_cast<const __half2*>(&w0);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float2 a = __half22float2(h0[i]);
            fadd2(dh[2 * i], dh[2 * i + 1], dh[2 * i], dh[2 * i + 1], a.x, a.y);
          }
        }
        const float inv = 1.f / P.xscale;
#pragma unroll
        for (int i = 0; i < kCellRows; i += 2) fmul2(dh[i], dh[i + 1], dh[i], dh[i + 1], inv, inv);
        named_bar_sync(3, kEpi * 32);  // every finaliser thread has read recv[buf]
        if (kEpiLead) {
          for (int f = 0; f < kKS; ++f)
            if (f != ks) mbar_arrive_remote(mapa_shared(smem_u32(&rfree[buf]), (uint32_t)(f * 2 + r)));
        }
      }
      // cell backward of my 8 rows (inputs staged in smem by the previous step)
      if (P.trace && blockIdx.x == 0 && threadIdx.x == 0)
        P.trace[(size_t)gridDim.x * T * kTraceSlots + (size_t)T * 18 + 2 * s] = globaltimer();
      mbar_wait(inbar, (uint32_t)s & 1);
      if (P.trace && blockIdx.x == 0 && threadIdx.x == 0)
        P.trace[(size_t)gridDim.x * T * kTraceSlots + (size_t)T * 18 + 2 * s + 1] = globaltimer();
      uint2* dgp = reinterpret_cast<uint2*>(P.dg + ((size_t)t * B + brow0 + row0) * (8 * kH) + col_g);
      // two rows per iteration on the packed fp32 pipe (FFMA2 / FMUL2 / FADD2): the same per-element
      // operations in the same order as the scalar form (fma where it contracted), about half the
      // float instructions of this issue-bound loop
#pragma unroll
      for (int i = 0; i < kCellRows; i += 2) {
        const uint2 aw0 = ld_shared_v2(cg_in + i * 256), aw1 = ld_shared_v2(cg_in + (i + 1) * 256);
        const float ig0 = __uint_as_float(aw0.x << 16), fg0 = __uint_as_float(aw0.x & 0xffff0000u);
        const float gg0 = __uint_as_float(aw0.y << 16), og0 = __uint_as_float(aw0.y & 0xffff0000u);
        const float ig1 = __uint_as_float(aw1.x << 16), fg1 = __uint_as_float(aw1.x & 0xffff0000u);
        const float gg1 = __uint_as_float(aw1.y << 16), og1 = __uint_as_float(aw1.y & 0xffff0000u);
        float dy0 = __uint_as_float(ld_shared_u16(cdy_in + i * 64) << 16);
        float dy1 = __uint_as_float(ld_shared_u16(cdy_in + (i + 1) * 64) << 16);
        if (P.dy2)
          fadd2(dy0, dy1, dy0, dy1, __uint_as_float(ld_shared_u16(cdy_in + kInDY + i * 64) << 16),
                __uint_as_float(ld_shared_u16(cdy_in + kInDY + (i + 1) * 64) << 16));
        const float cp0 = has_cprev ? ld_shared_f32(cc_in + i * 128) : 0.f;
        const float cp1 = has_cprev ? ld_shared_f32(cc_in + (i + 1) * 128) : 0.f;
        float dht0, dht1, om0, om1, a0, a1, dct0, dct1;
        fadd2(dht0, dht1, dh[i], dh[i + 1], dy0, dy1);
        const float tc0 = tanh_fast(cc[i]), tc1 = tanh_fast(cc[i + 1]);
        ffma2(om0, om1, -tc0, -tc1, tc0, tc1, 1.f, 1.f);  // 1 - tanh^2
        fmul2(a0, a1, dht0, dht1, og0, og1);
        ffma2(dct0, dct1, a0, a1, om0, om1, dcc[i], dcc[i + 1]);
        float x0, x1, y0, y1, d0[4], d1[4];
        // dg_i = dct gg ig (1 - ig)
        fmul2(x0, x1, dct0, dct1, gg0, gg1);
        fmul2(x0, x1, x0, x1, ig0, ig1);
        fadd2(y0, y1, 1.f, 1.f, -ig0, -ig1);
        fmul2(d0[0], d1[0], x0, x1, y0, y1);
        // dg_f = dct c_{t-1} fg (1 - fg)
        fmul2(x0, x1, dct0, dct1, cp0, cp1);
        fmul2(x0, x1, x0, x1, fg0, fg1);
        fadd2(y0, y1, 1.f, 1.f, -fg0, -fg1);
        fmul2(d0[1], d1[1], x0, x1, y0, y1);
        // dg_g = dct ig (1 - gg^2)
        fmul2(x0, x1, dct0, dct1, ig0, ig1);
        ffma2(y0, y1, -gg0, -gg1, gg0, gg1, 1.f, 1.f);
        fmul2(d0[2], d1[2], x0, x1, y0, y1);
        // dg_o = dh tanh(c) og (1 - og)
        fmul2(x0, x1, dht0, dht1, tc0, tc1);
        fmul2(x0, x1, x0, x1, og0, og1);
        fadd2(y0, y1, 1.f, 1.f, -og0, -og1);
        fmul2(d0[3], d1[3], x0, x1, y0, y1);
        fmul2(dcc[i], dcc[i + 1], dct0, dct1, fg0, fg1);
        cc[i] = cp0;
        cc[i + 1] = cp1;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float* dg = h ? d1 : d0;
          if ((okmask >> (i + h)) & 1u) {
            __nv_bfloat162 p0 = __floats2bfloat162_rn(dg[0], dg[1]), p1 = __floats2bfloat162_rn(dg[2], dg[3]);
            uint2 w;
            w.x = *reinterpret_cast<uint32_t*>(&p0);
            w.y = *reinterpret_cast<uint32_t*>(&p1);
            dgp[(size_t)(i + h) * (8 * kH / 4)] = w;
            fadd2(db[0], db[1], db[0], db[1], dg[0], dg[1]);
            fadd2(db[2], db[3], db[2], db[3], dg[2], dg[3]);
          }
        }
      }
      if (e == 0 && lane == 0) trace_mark(P.trace, T, s, 3);
      named_bar_sync(3, kEpi * 32);  // dG of this step stored; staged inputs consumed
      if (kEpiLead) {
        st_release_gpu(myflag, base + (uint32_t)(s + 1));
        if (P.gate) red_release_gpu_add(P.gate + dir * T + t, 1u);  // dG of (dir, t): this CTA's part stored
        trace_mark(P.trace, T, s, 4);
        if (s + 1 < T) {
          const int t1 = dir == 0 ? T - 2 - s : s + 1;
          issue_inputs(P, inbar, in_g, in_c, in_dy, t1, dir == 0 ? t1 - 1 : t1 + 1, brow0, dir, ubase + ks * kFin);
        }
      }
    }
    if (q != (uint32_t)ks && issuer && lane == 0) bulk_wait0();  // outgoing exchange copies complete
    if (P.dbpart) {  // fused bias gradient: warps e, e+4, e+8, e+12 summed in that order
      float* scratch = reinterpret_cast<float*>(send);  // free now (my copies completed; peers only write recv)
      named_bar_sync(3, kEpi * 32);
      if (e >= 4) *reinterpret_cast<float4*>(scratch + ((e - 4) * 32 + lane) * 4) = make_float4(db[0], db[1], db[2], db[3]);
      named_bar_sync(3, kEpi * 32);
      if (e < 4) {
        float4 o = make_float4(db[0], db[1], db[2], db[3]);
#pragma unroll
        for (int k2 = 0; k2 < 3; ++k2) {
          const float4 x = *reinterpret_cast<const float4*>(scratch + ((e + 4 * k2) * 32 + lane) * 4);
          o.x += x.x;
          o.y += x.y;
          o.z += x.z;
          o.w += x.w;
        }
        *reinterpret_cast<float4*>(P.dbpart + ((size_t)(P.b0 / 128 + btile) * 4 + e) * (8 * kH) + col_g) = o;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // no CTA leaves while a peer may still touch its smem / TMEM
  tc_fence_after();
  if (warp == kMmaWarp) tmem_dealloc_pair(tmem, 512);
}

__global__ void wait_started_kernel(const uint32_t* seq, int tag, int slot, int* err) {
  const uint32_t target = ld_relaxed_gpu(seq) * 16u + (uint32_t)tag;  // this step's epoch (bumped by its gather)
  SpinGuard g;
  while (!reached(ld_acquire_gpu(seq + slot), target))
    if (spin_expired(g, err)) return;
}

__global__ void wait_counters_kernel(const uint32_t* a, const uint32_t* b, uint32_t target, int* err) {
  SpinGuard g;
  while (ld_acquire_gpu(a) < target || ld_acquire_gpu(b) < target)
    if (spin_expired(g, err)) return;
}

}  // namespace

int lstm_wait_counters(const uint32_t* a, const uint32_t* b, uint32_t target, int* err, cudaStream_t stream) {
  wait_counters_kernel<<<1, 32, 0, stream>>>(a, b, target, err);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int lstm_wait_started(uint32_t* seq, int tag, int* err, cudaStream_t stream, bool forward) {
  wait_started_kernel<<<1, 32, 0, stream>>>(seq, tag, forward ? 2 : 1, err);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

static int launch_coop(const void* fn, int grid, const LstmParams& P, cudaStream_t stream, size_t smem,
                       int cluster, int threads = kThreads, int prio = 0, int pdl_kind = 2) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[4];
  int na = 0;
  if (prio) {
    attr[na].id = cudaLaunchAttributePriority;
    attr[na].val.priority = prio;
    ++na;
  }
  if (cluster > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = cluster;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  } else {
    attr[na].id = cudaLaunchAttributeCooperative;
    attr[na].val.cooperative = 1;
    ++na;
  }
  if (pdl_kind >= 0 && use_pdl(pdl_kind)) {  // the transposed BPTT measured faster without (kind -1)
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  void* args[] = {const_cast<LstmParams*>(&P)};
  DS_CUDA_TRY(cudaLaunchKernelExC(&cfg, fn, args));
  return DS_OK;
}

// batch tiles per launch: forward 32 CTAs / tile; backward 64 CTAs / tile in
// clusters of 4 (cluster placement leaves some SMs unusable: keep <= 128)
// <= 128 CTAs per launch: forward 32 CTAs per 64-row batch block, backward
// 64 CTAs per 128-row batch tile in clusters of 4
//
// The recurrent grids synchronise through flags, so every CTA of a launch
// must be co-resident.  The per-launch batch is capped by what the device
// can actually co-schedule in clusters of 2 (forward) / 4 (backward) at the
// kernels' shared-memory size (cudaOccupancyMaxActiveClusters on an idle
// device), not just by the SM count: cluster placement inside GPCs leaves
// SMs unusable.  A larger batch runs as several launches.
struct RecCaps {
  int fwd_ctas = 0, fwd3_ctas = 0, bwd_ctas = 0, bwd3_ctas = 0;  // co-resident CTAs in recurrent-kernel clusters
  int err = 0;
};
// DS_BWD=1 selects the round-1 split-K BPTT (single-CTA MMAs, 4-CTA clusters); default: transposed CTA-pair BPTT
static bool use_bwd3() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DS_BWD");
    v = (e && e[0] == '1') ? 0 : 1;
  }
  return v == 1;
}
// DS_FWD=3 selects the 64-CTA forward (W_hh in tensor memory, 128-row batch blocks: 5.4 us per step
// against 4.5 for the default 128-CTA forward, whose cell work per SM is half; it would leave 84 SMs
// to a projection streaming beside it)
static bool use_fwd3() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DS_FWD");
    v = (e && e[0] == '3') ? 1 : 0;
  }
  return v == 1;
}
static int cluster_cap(const void* fn, size_t smem, int cluster, int threads = kThreads) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cluster * 64);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = cluster;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return n * cluster;
}
static const RecCaps& rec_caps() {
  static RecCaps caps;
  static bool done = false;
  if (!done) {
    done = true;
    if (cudaFuncSetAttribute(lstm_fwd2_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fwd2::kSmem) !=
            cudaSuccess ||
        cudaFuncSetAttribute(lstm_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bwd::kSmem) !=
            cudaSuccess ||
        cudaFuncSetAttribute(lstm_bwd3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bwd3::kSmem) !=
            cudaSuccess ||
        cudaFuncSetAttribute(lstm_fwd3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fwd3::kSmem) !=
            cudaSuccess ||
        cudaFuncSetAttribute(lstm_fwd2_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fwd2::kSmemX) !=
            cudaSuccess) {
      cudaGetLastError();
      caps.err = 1;
      return caps;
    }
    const int sm = num_sms() >= 132 ? 128 : num_sms();
    const int f = cluster_cap((const void*)lstm_fwd2_kernel<false>, fwd2::kSmem, 2, fwd2::kThreadsF2);
    const int f3 = cluster_cap((const void*)lstm_fwd3_kernel, fwd3::kSmem, 2, fwd3::kThreadsF);
    const int b = cluster_cap((const void*)lstm_bwd_kernel, bwd::kSmem, 4);
    const int b3 = cluster_cap((const void*)lstm_bwd3_kernel, bwd3::kSmem, 8, bwd3::kThreads3);
    caps.fwd_ctas = f < 0 ? sm : (f < sm ? f : sm);
    caps.fwd3_ctas = f3 < 0 ? sm : (f3 < sm ? f3 : sm);
    caps.bwd_ctas = b < 0 ? sm : (b < sm ? b : sm);
    caps.bwd3_ctas = b3 < 0 ? sm : (b3 < sm ? b3 : sm);
  }
  return caps;
}
// 128-row batch tiles per launch: forward 64 CTAs per tile, backward 64 (split-K) or 32 (transposed)
static int lstm_bwd_max_tiles() { return use_bwd3() ? rec_caps().bwd3_ctas / 32 : rec_caps().bwd_ctas / 64; }
int lstm_bwd_gate_target(int B) { return 16 * ((B + 127) / 128); }
int lstm_bwd_narrow_ctas(int B) {
  if (!use_bwd3()) return 0;
  const int tiles = (B + 127) / 128, cap = lstm_bwd_max_tiles();
  return 32 * (tiles < cap ? tiles : cap);
}
int lstm_max_tiles() {
  const int f = use_fwd3() ? rec_caps().fwd3_ctas / 32 : rec_caps().fwd_ctas / 64, b = lstm_bwd_max_tiles();
  const int t = b < f ? b : f;
  return t > 0 ? t : 0;
}
int lstm_counter_words(int B) { return kFlagWords128 * ((B + 127) / 128); }

static int lstm_run(bool fwd, const LstmLayerArgs& a, cudaStream_t stream) {
  if (rec_caps().err) return fail_arg("recurrent kernels: cannot set the shared-memory attribute");
  const int B = a.B, T = a.T;
  if (fwd && use_fwd3() && a.xin) return fail_arg("the fused input projection runs in the 128-CTA forward");
  if (fwd && use_fwd3()) {
    // 32 CTAs (2 directions x 8 pairs x 2) per 128-row batch block
    const int max_blocks = rec_caps().fwd3_ctas / (2 * fwd3::kCtas);
    if (max_blocks < 1) return fail_arg("device too small for the recurrent kernel");
    LstmParams P;
    memset(&P, 0, sizeof(P));
    int rc = make_tmap_2d(&P.tmA, a.y_full, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2 * kH, (uint64_t)(T + 2) * B,
                          2 * kH * 2, 64, fwd3::kNH);
    if (rc) return rc;
    rc = make_tmap_2d(&P.tmW, a.w, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, kH, 8 * kH, kH * 2, 64, 128);
    if (rc) return rc;
    P.gates = a.gates;
    P.cstate = a.cstate;
    P.y = a.y_full;
    P.trace = a.trace;
    P.err = a.err;
    P.seq = a.seq;
    P.tag = a.tag;
    P.gate = a.gate;
    P.B = B;
    P.T = T;
    const int chunk_rows = max_blocks * fwd3::kNB;
    for (int b0 = 0; b0 < B; b0 += chunk_rows) {
      const int nb = (B - b0) < chunk_rows ? (B - b0) : chunk_rows;
      P.b0 = b0;
      P.nb = nb;
      P.n_btile = (nb + fwd3::kNB - 1) / fwd3::kNB;  // 128-row blocks
      P.counters = a.counters;
      rc = launch_coop((const void*)lstm_fwd3_kernel, 2 * fwd3::kCtas * P.n_btile, P, stream, fwd3::kSmem, 2,
                       fwd3::kThreadsF, a.prio);
      if (rc) return rc;
      P.trace = nullptr;  // trace only the first chunk
      P.seq = nullptr;    // the start signal is the first launch's
    }
    return DS_OK;
  }
  if (fwd) {
    // 32 CTAs (2 directions x 8 pairs x 2) per 64-row batch block
    const int max_blocks = rec_caps().fwd_ctas / (2 * fwd2::kCtas);
    if (max_blocks < 1) return fail_arg("device too small for the recurrent kernel");
    LstmParams P;
    memset(&P, 0, sizeof(P));
    int rc = make_tmap_2d(&P.tmA, a.y_full, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2 * kH, (uint64_t)(T + 2) * B,
                          2 * kH * 2, 64, fwd2::kNH);
    if (rc) return rc;
    rc = make_tmap_2d(&P.tmW, a.w, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, kH, 8 * kH, kH * 2, 64, 128);
    if (rc) return rc;
    P.gates = a.gates;
    P.cstate = a.cstate;
    P.y = a.y_full;
    P.trace = a.trace;
    P.err = a.err;
    P.B = B;
    P.T = T;
    if (a.xin) {  // fused input projection: x rows (box 64 K x 32 rows) and W_ih rows (64 K x 128 rows)
      if (!a.wih || !a.xbias) return fail_arg("fused input projection needs W_ih and the bias");
      rc = make_tmap_2d(&P.tmX, a.xin, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, kInPad, (uint64_t)T * B, kInPad * 2, 64,
                        fwd2::kNH);
      if (!rc)
        rc = make_tmap_2d(&P.tmWi, a.wih, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, kInPad, 8 * kH, kInPad * 2, 64, 128);
      if (rc) return rc;
      P.xbias = a.xbias;
    }
    const int chunk_rows = max_blocks * fwd2::kNB;
    for (int b0 = 0; b0 < B; b0 += chunk_rows) {
      const int nb = (B - b0) < chunk_rows ? (B - b0) : chunk_rows;
      P.b0 = b0;
      P.nb = nb;
      P.n_btile = (nb + fwd2::kNB - 1) / fwd2::kNB;  // 64-row blocks
      P.counters = a.counters;
      rc = launch_coop(P.xbias ? (const void*)lstm_fwd2_kernel<true> : (const void*)lstm_fwd2_kernel<false>,
                       2 * fwd2::kCtas * P.n_btile, P, stream, P.xbias ? fwd2::kSmemX : fwd2::kSmem, 2,
                       fwd2::kThreadsF2);
      if (rc) return rc;
      P.trace = nullptr;  // trace only the first chunk
    }
    return DS_OK;
  }
  const int max_tiles = lstm_bwd_max_tiles();
  if (max_tiles < 1) return fail_arg("device too small for the recurrent kernel");
  const bool v3 = use_bwd3();
  LstmParams P;
  memset(&P, 0, sizeof(P));
  int rc = make_tmap_2d(&P.tmA, a.dg, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 8 * kH, (uint64_t)T * B, 8 * kH * 2, 64,
                        v3 ? bwd3::kHalfRows : 128);
  if (rc) return rc;
  if (v3)  // W_hh [gate rows][units] staged as [64 units x 256 gate rows] boxes, transposed into TMEM
    rc = make_tmap_2d(&P.tmW, a.w, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, kH, 8 * kH, kH * 2, 64, 256,
                      CU_TENSOR_MAP_SWIZZLE_NONE);
  else
    rc = make_tmap_2d(&P.tmW, a.w, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, kH, 8 * kH, kH * 2, bwd::kGU, 64);
  if (rc) return rc;
  if (v3) {  // cell inputs of a finaliser: 128 rows x (32 units x 4 gates | 32 cells | 32 dY)
    rc = make_tmap_2d(&P.tmG, a.gates, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 8 * kH, (uint64_t)T * B, 8 * kH * 2,
                      bwd3::kFin * 4, bwd3::kRows, CU_TENSOR_MAP_SWIZZLE_NONE);
    if (!rc)
      rc = make_tmap_2d(&P.tmC, a.cstate, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2 * kH, (uint64_t)T * B, 2 * kH * 4,
                        bwd3::kFin, bwd3::kRows, CU_TENSOR_MAP_SWIZZLE_NONE);
    if (!rc)
      rc = make_tmap_2d(&P.tmDY, a.dy, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2 * kH, (uint64_t)T * B, 2 * kH * 2,
                        bwd3::kFin, bwd3::kRows, CU_TENSOR_MAP_SWIZZLE_NONE);
    if (!rc && a.dy2)
      rc = make_tmap_2d(&P.tmDY2, a.dy2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2 * kH, (uint64_t)T * B, 2 * kH * 2,
                        bwd3::kFin, bwd3::kRows, CU_TENSOR_MAP_SWIZZLE_NONE);
    if (rc) return rc;
  }
  P.gates = a.gates;
  P.cstate = a.cstate;
  P.y = a.y_full;
  P.dy = a.dy;
  P.dg = a.dg;
  P.trace = a.trace;
  P.dbpart = a.dbpart;
  P.err = a.err;
  P.seq = a.seq;
  P.tag = a.tag;
  P.gate = v3 ? a.gate : nullptr;
  P.dyready = v3 ? a.dyready : nullptr;
  P.dy2 = v3 ? a.dy2 : nullptr;
  if (a.dy2 && !v3) return fail_arg("a second dY input needs the transposed BPTT");
  P.dyready_target = a.dyready_target;
  if (a.dyready && !v3) return fail_arg("streamed dY needs the transposed BPTT");
  P.variant = 7;  // acquire by ld.acquire, no writer-side fences
  if (v3) {
    const char* ev = getenv("DS_VARIANT");
    P.variant = ev ? atoi(ev) : 0;
  }
  {  // fp16 exchange scale: power of two ~ frames / 2 (dh ~ 1/frames for a mean loss)
    float sc = 1.f;
    while (sc * 4.f <= (float)T * B && sc < 16384.f) sc *= 2.f;
    P.xscale = sc;
  }
  P.B = B;
  P.T = T;
  const int chunk_rows = max_tiles * 128;
  for (int b0 = 0; b0 < B; b0 += chunk_rows) {
    const int nb = (B - b0) < chunk_rows ? (B - b0) : chunk_rows;
    P.b0 = b0;
    P.nb = nb;
    P.n_btile = (nb + 127) / 128;
    P.counters = a.counters;
    rc = v3 ? launch_coop((const void*)lstm_bwd3_kernel, 32 * P.n_btile, P, stream, bwd3::kSmem, 8, bwd3::kThreads3,
                          a.prio, -1)
            : launch_coop((const void*)lstm_bwd_kernel, 64 * P.n_btile, P, stream, bwd::kSmem, bwd::kClB, kThreads, 0, 3);
    if (rc) return rc;
    P.trace = nullptr;  // trace only the first chunk
  }
  return DS_OK;
}

int lstm_forward(const LstmLayerArgs& a, cudaStream_t stream) { return lstm_run(true, a, stream); }
int lstm_backward(const LstmLayerArgs& a, cudaStream_t stream) { return lstm_run(false, a, stream); }

}  // namespace ds
