// lstm_rec.h — launch interface of the persistent recurrent kernels.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "ds_internal.h"

namespace ds {

struct LstmParams {
  CUtensorMap tmA;  // forward: Y_full; backward: dG
  CUtensorMap tmW;  // W_hh [4096, 512] bf16 (forward: K-major B; backward: MN-major B)
  CUtensorMap tmG, tmC, tmDY;  // transposed BPTT: per-step cell inputs (gates, c_{t-1}, dY) staged by TMA
  CUtensorMap tmDY2;           //   second dY input (dY = dy + dy2), when dy2 != null
  CUtensorMap tmX, tmWi;       // forward, fused input projection: X [N, 272] rows, W_ih [4096, 272]
  __nv_bfloat16* gates;
  float* cstate;
  __nv_bfloat16* y;
  const __nv_bfloat16* dy;
  __nv_bfloat16* dg;
  uint32_t* counters;
  const float* xbias;  // forward, fused input projection (x_t W_ih^T + b in the recurrent MMA): b [4096]
  uint64_t* trace;  // optional per-(CTA, step) globaltimer marks (debug)
  float* dbpart;    // backward: optional [(B/128)*4][4096] bias-gradient partials
  int B, T, b0, nb, n_btile;
  int variant;  // debug: bit0 skip writer proxy fence, bit1 skip release fence
  float xscale; // BPTT: fp16 scale of the exchanged partial dh (power of two)
  int* err;     // optional: |= 8 when a flag wait times out (a peer CTA never published)
  uint32_t* seq;  // [0] step epoch, [1] last started BPTT launch, [2] last started forward launch (epoch*16 + tag)
  int tag;        // position of this backward launch in the step (0 = first: bumps the epoch)
  uint32_t* gate; // narrow forward / transposed BPTT: per-(direction, time step) counters, +1 per CTA once its h / dG
                  // of that step is stored
  const __nv_bfloat16* dy2;  // transposed BPTT: optional second dY input
  const uint32_t* dyready;  // transposed BPTT: per-(time step, direction, input) dY counters of the GEMM producing dY
  uint32_t dyready_target;  //   (0 / null: dY is complete when the launch starts)
};

struct LstmLayerArgs {
  int B, T;
  __nv_bfloat16* gates;     // [T*B, 4096]
  float* cstate;            // [T*B, 1024]
  __nv_bfloat16* y_full;    // [(T+2)*B, 1024]
  const __nv_bfloat16* w;   // W_hh bf16 [4096, 512] (rows dir*2048 + unit*4 + gate)
  const __nv_bfloat16* dy;  // backward: [T*B, 1024]
  __nv_bfloat16* dg;        // backward: [T*B, 4096]
  uint32_t* counters;       // >= lstm_counter_words(B)
  uint64_t* trace = nullptr;
  float* dbpart = nullptr;  // backward: per-(batch tile, lane quadrant) column sums of dG
  int* err = nullptr;       // step error flag: |= 8 on a flag-wait timeout
  int prio = 0;             // != 0: launch priority (ahead of GEMMs issued beside the recurrence)
  uint32_t* seq = nullptr;  // start signal for GEMMs gated on this launch (lstm_wait_started)
  int tag = 0;
  uint32_t* gate = nullptr;  // [2][T] per-(direction, time step) completion counters (lstm_bwd_gate_target)
  // backward: dY = dy + dy2 (the two per-direction halves of dX_{l+1}) when dy2 != null
  const __nv_bfloat16* dy2 = nullptr;
  // forward: the input projection inside the recurrence (layer 0, K = 272): pre-activation =
  // x_t W_ih^T (W_ih slice in tensor memory, x tiles staged a step ahead) + bias + h W_hh^T; `gates`
  // then only receives the activations
  const __nv_bfloat16* xin = nullptr;  // [T*B, 272] time-major
  const __nv_bfloat16* wih = nullptr;  // [4096, 272] (zero-padded columns)
  const float* xbias = nullptr;        // [4096]
  // dY streamed in by a GEMM still running: frame t of direction d's units of input i is complete once
  // dyready[(2t + d) * 2 + i] >= dyready_target (GemmProblem::ready with ready_rows = B, ready_cols = 512,
  // ready_stride = 2)
  const uint32_t* dyready = nullptr;
  uint32_t dyready_target = 0;
};
// value of a backward launch's per-(direction, time step) counter once every CTA of that direction
// stored its dG of that step
int lstm_bwd_gate_target(int B);
// Block `stream` until the backward launch with `tag` of the current step has started (its grid is
// placed), so a GEMM issued next on `stream` only takes the SMs the recurrence left free.
int lstm_wait_started(uint32_t* seq, int tag, int* err, cudaStream_t stream, bool forward = false);
// Block `stream` until the (per-step zeroed) counters *a and *b both reach `target`.
int lstm_wait_counters(const uint32_t* a, const uint32_t* b, uint32_t target, int* err, cudaStream_t stream);

int lstm_max_tiles();
// CTAs of the first backward launch for a batch of B (the SMs a concurrent GEMM must leave free),
// 0 when the backward kernel is the 128-CTA split-K variant (nothing to overlap)
int lstm_bwd_narrow_ctas(int B);
int lstm_counter_words(int B);
int lstm_forward(const LstmLayerArgs& a, cudaStream_t stream);
int lstm_backward(const LstmLayerArgs& a, cudaStream_t stream);

}  // namespace ds
