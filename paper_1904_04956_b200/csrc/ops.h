// ops.h — host launchers for the HBM-bound kernels in ops.cu.
#pragma once
#include <cuda_bf16.h>

#include "ds_internal.h"
#include "layout.h"

namespace ds {

constexpr int kMaxGroup = 16;

int op_gather(const int64_t* idx, int B, int T, const __nv_bfloat16* feats, const int32_t* labels, int64_t n_seq,
              __nv_bfloat16* x0, int32_t* lab, int* flag, cudaStream_t s, uint32_t* epoch = nullptr);
int op_colsum(const __nv_bfloat16* x, int64_t rows, int ncols, int64_t ld, float* part, float* out, cudaStream_t s);
int64_t op_colsum_scratch(int64_t rows, int ncols);
// out = bf16(sum of the S partials [S][n] (+ bias[i % ncols]))
int op_splitk_bf16(const float* part, int S, int64_t n, __nv_bfloat16* out, cudaStream_t s, const float* bias = nullptr,
                   int ncols = 0);
int op_splitk_f32(const float* part, int S, int64_t n, float* out, cudaStream_t s);
int op_rowsum(const float* part, int nrows, int ncols, float* out, cudaStream_t s);
int op_ce_combine(const float2* stats, int ntiles, int64_t ld, const float* tgt, int M, float* lse, float* scratch,
                  unsigned* ticket, float* loss_sum, int* flag, cudaStream_t s);  // ticket: zeroed word, re-armed
int op_sgd(float* theta, float* v, const float* g, float lr, float mu, int64_t n, __nv_bfloat16* snap, int* flag,
           cudaStream_t s);
// Operand-snapshot extras written by the update of a parameter block as it goes (instead of a pass
// after the step): the layer-0 W_ih rows padded to kInPad bf16 columns, and fp32 copies (times a
// scale) of bias ranges.  Offsets are relative to the block; all multiples of 4 (din too).
struct SgdMirror {
  __nv_bfloat16* wpad = nullptr;
  int64_t wbeg = 0, wcnt = 0;
  int din = 0;
  float* fdst[3] = {};
  int64_t fbeg[3] = {}, fcnt[3] = {};
  float fscale[3] = {1.f, 1.f, 1.f};
  // a second gradient part summed in first (g[i] += add[i] for i < add_n, the sum stored back into g):
  // the layer-0 weight gradients computed after BPTT_0, added to the part computed beside it
  const float* add = nullptr;
  int64_t add_n = 0;
};
// lr from device memory; max_blocks > 0: at most that many 1024-thread blocks
int op_sgd_lr(float* theta, float* v, const float* g, const float* lr_dev, float mu, int64_t n, __nv_bfloat16* snap,
              int* flag, int max_blocks, cudaStream_t s, const SgdMirror* mir = nullptr);
int op_cast(const float* theta, int64_t n, __nv_bfloat16* snap, cudaStream_t s);
int op_snapshot_aux(const float* theta, const ModelLayout& L, __nv_bfloat16* wih0pad, float* bias_snap,
                    cudaStream_t s);
int op_mix(float* a, float* b, int64_t n, cudaStream_t s);
int op_group_reduce(int world, int rank, float* const* g, float* const* theta, float* const* v,
                    __nv_bfloat16* const* snap, int64_t dim, int nchunks, float lr, float mu, int mode, float divisor,
                    cudaStream_t s);
int op_average(int n, float* const* srcs, float* out, int64_t dim, cudaStream_t s);

}  // namespace ds
