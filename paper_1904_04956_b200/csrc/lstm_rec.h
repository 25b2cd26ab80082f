// lstm_rec.h — launch interface of the persistent recurrent kernels.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "ds_internal.h"

namespace ds {

struct LstmParams {
  CUtensorMap tmA;  // forward: Y_full; backward: dG
  CUtensorMap tmW;  // W_hh [4096, 512] bf16 (forward: K-major B; backward: MN-major B)
  __nv_bfloat16* gates;
  float* cstate;
  __nv_bfloat16* y;
  const __nv_bfloat16* dy;
  __nv_bfloat16* dg;
  uint32_t* counters;
  uint64_t* trace;  // optional per-(CTA, step) globaltimer marks (debug)
  float* dbpart;    // backward: optional [(B/128)*4][4096] bias-gradient partials
  int B, T, b0, nb, n_btile;
  int variant;  // debug: bit0 skip writer proxy fence, bit1 skip release fence
  float xscale; // BPTT: fp16 scale of the exchanged partial dh (power of two)
  int* err;     // optional: |= 8 when a flag wait times out (a peer CTA never published)
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
};

int lstm_max_tiles();
int lstm_counter_words(int B);
int lstm_forward(const LstmLayerArgs& a, cudaStream_t stream);
int lstm_backward(const LstmLayerArgs& a, cudaStream_t stream);

}  // namespace ds
