// softmax_dz.h — fused soft-max gradient + dZ of the output layer (softmax_dz.cu).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "ds_internal.h"

namespace ds {

struct CeGradDzParams {
  CUtensorMap tmZ;   // Z [rows][bott] bf16, box 64 x 128
  CUtensorMap tmW1;  // W_o [classes][bott] bf16 (operand snapshot), box 64 x 64 (MMA1 view)
  CUtensorMap tmW2;  // same tensor, box 64 x 128 (MMA2 view)
  CUtensorMap tmP;   // dlogits, 64x64-blocked 4D [ceil(rows/64)][classes/64][64][64], box 32 x 32 (TMA store)
  const float* bias;    // b_o [classes]
  const int* labels;    // [rows], -1 = no target
  const float* lse;     // [rows]
  float* colpart;       // [ceil(rows/128)*4][classes] bias-gradient partials (nullable)
  float* dzpart;        // [n_cs][rows][bott] fp32 dZ partials
  float scale;          // 1 / frames
  int bott, classes, m_valid, dz_rows;
  int n_rbp, n_ct, n_cs, ct_per;  // row-block pairs, 128-class tiles, class ranges, tiles per range
  unsigned long long* trace;  // debug timeline (tools/cedz_trace.py), null in production
};
void ce_grad_dz_set_trace(unsigned long long* buf);

struct CeGradDzArgs {
  const __nv_bfloat16* z;
  const __nv_bfloat16* w;
  const float* bias;
  const int* labels;
  const float* lse;
  __nv_bfloat16* dlogits;  // blocked, gemm_blocked_elems(rows, classes)
  float* colpart;
  float* dzpart;           // [splits][rows][bott]
  float scale;
  int rows, classes, bott, splits;
};

// Soft-max statistics of the logits Z W_o^T + b_o on CTA pairs (the loss pass):
// per row and class range (max, sum exp(x - max)) in natural-log units, and the
// target logit of every labelled row; same work split as the gradient kernel,
// combined across class ranges by op_ce_combine.
struct CeStatsArgs {
  const __nv_bfloat16* z;
  const __nv_bfloat16* w;
  const float* bias_log2;  // b_o * log2(e)
  const int* labels;
  float2* stats;           // [splits][stats_ld]
  int64_t stats_ld;
  float* tgt;              // [rows]
  int rows, classes, bott, splits;
};
struct CeStatsParams {
  CUtensorMap tmZ, tmW1;
  const float* bias_log2;
  const int* labels;
  float2* stats;
  int64_t stats_ld;
  float* tgt;
  int bott, classes, m_valid;
  int n_rbp, n_ct, n_cs, ct_per;
};
int ce_stats_launch(const CeStatsArgs& a, cudaStream_t stream);

bool ce_grad_dz_supported(int classes, int bott);
int ce_grad_dz_splits(int rows, int classes, int max_splits);  // class ranges per row block (none empty)
int ce_grad_dz_launch(const CeGradDzArgs& a, cudaStream_t stream);

}  // namespace ds
