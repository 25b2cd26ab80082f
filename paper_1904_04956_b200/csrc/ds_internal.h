// ds_internal.h — host-side interfaces shared by the .cu translation units of
// libds (not part of the public C ABI in include/ds_blstm.h).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include <string>

namespace ds {

// ---------------------------------------------------------------------------
// error plumbing: every C-ABI entry returns 0 or a negative code and records a
// thread-local message (ds_last_error()).
#ifndef DS_OK
#define DS_OK 0
#define DS_ERR_ARG (-1)       /* bad shape / config (maps to ValueError) */
#define DS_ERR_CUDA (-2)      /* CUDA runtime/driver failure (RuntimeError) */
#define DS_ERR_NONFINITE (-3) /* non-finite loss/gradient (ValueError) */
#endif
void set_error(const std::string& msg);
int fail_arg(const std::string& msg);
int fail_cuda(cudaError_t e, const char* where);

#define DS_CUDA_TRY(expr)                                  \
  do {                                                     \
    cudaError_t _e = (expr);                               \
    if (_e != cudaSuccess) return ::ds::fail_cuda(_e, #expr); \
  } while (0)

int num_sms();

// ---------------------------------------------------------------------------
// TMA descriptors
// 2D row-major tensor [outer][inner] of `elem_bytes` elements, row pitch in
// bytes; box = box_inner x box_outer elements; SWIZZLE_128B (box_inner *
// elem_bytes must be 128).
bool use_pdl(int kind = 0);  // programmatic dependent launch on (DS_NO_PDL=1: off; see common.cu)
int make_tmap_2d(CUtensorMap* out, const void* base, CUtensorMapDataType dtype, uint64_t inner, uint64_t outer,
                 uint64_t row_pitch_bytes, uint32_t box_inner, uint32_t box_outer,
                 CUtensorMapSwizzle swizzle = CU_TENSOR_MAP_SWIZZLE_128B);

// 4D tensor [d3][d2][d1][d0] (d0 contiguous); strides of d1..d3 in bytes.
int make_tmap_4d(CUtensorMap* out, const void* base, CUtensorMapDataType dtype, const uint64_t dims[4],
                 const uint64_t strides_bytes[3], const uint32_t box[4],
                 CUtensorMapSwizzle swizzle = CU_TENSOR_MAP_SWIZZLE_128B);

// ---------------------------------------------------------------------------
// GEMM: C[m, n] = sum_k A[m, k] * B[n, k], bf16 operands, fp32 accumulate in
// TMEM (tcgen05), persistent tile loop, up to kMaxProblems per launch.
//
// Operand storage:
//   a_mn = 0: A stored [M][K] (K contiguous)   a_mn = 1: A stored [K][M]
//   b_mn = 0: B stored [N][K] (K contiguous)   b_mn = 1: B stored [K][N]
enum Epilogue : int {
  EPI_BF16 = 0,      // out bf16 [M, ldo] = acc (+ bias[n])
  EPI_F32 = 1,       // out f32  [M, ldo] = acc*scale (+ out if accumulate)
  EPI_CE_STATS = 2,  // per-row partial (max, sumexp) of acc + b[n] over n < n_valid, target logit;
                     // bias holds b * log2(e)
  EPI_CE_GRAD = 3,   // out bf16 = (exp(acc+bias-lse[m]) - [n==label[m]]) * scale
};

constexpr int kGemmBM = 128;
constexpr int kGemmBN = 256;
constexpr int kGemmBK = 64;
constexpr int kMaxProblems = 4;

struct GemmProblem {
  CUtensorMap tmA;  // 64-byte aligned (first member)
  CUtensorMap tmB;
  CUtensorMap tmC;  // bf16 outputs (EPI_BF16 / EPI_CE_GRAD): [m_valid][n_valid], 32x32 boxes, SW64
  int M, N, K;
  int a_mn, b_mn;
  int epi;
  int tiles_m, tiles_n, tile_begin;
  int n_valid;      // columns >= n_valid are not stored (and masked in CE)
  int m_valid;      // rows >= m_valid are not stored
  long long ldo;    // output row pitch in elements
  void* out;
  const float* bias;
  float scale;
  int accumulate;
  // CE
  const int* labels;      // [m_valid]
  const float* lse;       // [m_valid]
  float2* stats;          // [tiles_n][stats_ld]
  float* tgt;             // [m_valid]
  int stats_ld;
  float* colpart;         // EPI_CE_GRAD: optional [tiles_m*4][n_valid] column-sum partials
  int c_tma;              // bf16 output stored through smem staging + TMA (tmC valid)
  // 64x64-blocked [row/64][col/64][64][64] bf16 operand / output (dlogits):
  // tmA / tmC are then 4D maps over (col%64, row%64, col/64, row/64)
  int a_blk;
  int c_blk;
  int ksplit;             // split-K factor (EPI_F32 only): split s writes out + s*split_stride
  long long split_stride;
  // Row gate (a GEMM streaming behind a recurrence): rows are time-major, gate_rows per time step;
  // a tile's A rows are loaded once gate[t] >= gate_target for every time step t < gate_T they
  // cover.  A gated launch needs a host schedule (GemmBatch::presched: its units in the order the
  // recurrence completes them).
  const uint32_t* gate;
  uint32_t gate_target;
  int gate_rows, gate_T;
  int* gate_err;          // |= 8 when a gate wait times out
  // Completion counters of the bf16 output: +1 (release) per stored 32-row x 64-column warp block on
  // ready[((row / ready_rows) * (N / ready_cols) + col / ready_cols) * ready_stride] (a recurrence
  // consuming the rows of one time step and one column group waits for (ready_rows / 32) *
  // (ready_cols / 64))
  uint32_t* ready;
  int ready_rows, ready_cols, ready_stride;
};


// Pair-tile schedule: when the tiles of a launch differ in length the host
// assigns them to the persistent CTA pairs longest-first onto the least
// loaded pair (LPT) and passes the per-pair lists here; otherwise pairs walk
// the tiles round-robin.
constexpr int kMaxSched = 2048;
constexpr int kMaxPairs = 80;

struct GemmBatch {
  GemmProblem p[kMaxProblems];
  int nprob;
  int total_tiles;
  int sched;                            // 1: use order/pstart
  int presched;                         // order/pstart/sched filled by the caller for `presched` pairs
  int b_early;                          // B of every problem is not written by the predecessor kernel:
                                        // prefetch it before griddep_wait (PDL)
  int max_pairs;                        // > 0: at most this many CTA pairs (a GEMM running beside a
                                        // recurrent kernel on the SMs it leaves free)
  int prio;                             // != 0: launch priority (cudaLaunchAttributePriority)
  uint16_t pstart[kMaxPairs + 1];       // pair p runs order[pstart[p] .. pstart[p+1])
  uint16_t order[kMaxSched];
  // debug: per-CTA per-tile timeline (tools/gemm_trace.py, tools/dx_trace.py), null in production
  unsigned long long* trace;
  int trace_keep;                       // the caller set `trace` (gemm_layer_trace)
};
// debug: trace the `launch`-th gemm_launch from now on into `buf` (null: off); launch <= -2: the
// streamed dX of layer -launch-2 inside the step graph (gemm_layer_trace)
void gemm_set_trace(unsigned long long* buf, int launch);
unsigned long long* gemm_layer_trace(int layer);

// Host helpers -------------------------------------------------------------
// Describe one problem. A/B are device pointers with the given row pitches
// (elements).  Returns DS_OK or an error.
int gemm_problem(GemmProblem* p, const void* A, long long lda, int a_mn, const void* B, long long ldb, int b_mn,
                 int M, int N, int K);
int gemm_launch(GemmBatch* batch, cudaStream_t stream);
int gemm_stats_parts();  // EPI_CE_STATS partial statistics per column tile
// Attach the TMA store map for a bf16 output (call after setting out/ldo/n_valid/m_valid).
int gemm_bf16_output(GemmProblem* p);
// 64x64-blocked bf16 matrices (rows x cols, see GemmProblem::a_blk): element
// count of the buffer, A operand view (call after gemm_problem, sets tmA), and
// TMA-stored bf16 output view (call after setting out/epi).
int64_t gemm_blocked_elems(int64_t rows, int64_t cols);
int gemm_blocked_a(GemmProblem* p, const void* A, int64_t rows, int64_t cols);
int gemm_blocked_output(GemmProblem* p, int64_t rows, int64_t cols);

}  // namespace ds
