// parity.h — FP32-parity mode (3xTF32 tcgen05 GEMMs, fp32 activations): see parity.cu.
#pragma once
#include <cuda_bf16.h>

#include "ds_internal.h"
#include "layout.h"

namespace ds {

// an fp32 operand as (hi, lo): hi = tf32(x) (round to nearest), lo = x - hi exactly
struct Split {
  float* hi = nullptr;
  float* lo = nullptr;
  Split off(size_t n) const { return Split{hi + n, lo + n}; }
};

struct ParityWs {
  void* arena = nullptr;
  size_t bytes = 0;
  float* snap = nullptr;  // fp32 copy of the snapshot theta (biases)
  Split W;                // hi/lo of every parameter, flat packing
  Split WihT[kMaxLayers], WhhT[kMaxLayers], WoT, WbT;  // transposed weights (K-major B operands)
  float* x0 = nullptr;
  Split x0s;
  int32_t* lab = nullptr;
  float* gates[kMaxLayers] = {};  // pre-activations -> i,f,g,o  [N][4096]
  float* cst[kMaxLayers] = {};    // cell state [N][1024]
  float* y[kMaxLayers] = {};      // layer outputs [N][1024]
  Split ys[kMaxLayers];
  float *z = nullptr, *logits = nullptr, *dlo = nullptr, *rowloss = nullptr, *dz = nullptr, *dy = nullptr,
        *da = nullptr, *dcc = nullptr;
  Split zs, dlT, dzs, dzT, zT, yT, das, daT, hpT;
};

int parity_create(ParityWs** out, const ModelLayout& L, int T, int Bmax);
void parity_destroy(ParityWs* w);
int parity_snapshot(ParityWs* w, const ModelLayout& L, const float* theta, cudaStream_t s);
int parity_step(ParityWs* w, const ModelLayout& L, int T, const int64_t* idx, int B, const __nv_bfloat16* feats,
                const int32_t* labels, int64_t n_seq, float grad_frames, float* grad, float* loss, int* flag,
                cudaStream_t s, int* launches);
int split_launch(const float* x, int64_t n, const Split& out, cudaStream_t s);
int tsplit_launch(const float* s0, const float* s1, long long lds, int rows, int cols, int shift, const Split& out,
                  long long ldd, cudaStream_t s);
int gemm3(const Split& A, long long lda, const Split& B, long long ldb, int M, int N, int K, float* out,
          long long ldo, const float* bias, int accumulate, cudaStream_t s);

}  // namespace ds
