/* ds_blstm.h — C ABI of libds: the B200 (sm_100a) hot path of arXiv
 * 1904.04956 behind the reference `distsgd` plug-in points.
 *
 * Conventions
 *   - every function returns 0 on success or a negative DS_ERR_* code and never
 *     throws; ds_last_error() returns a thread-local message for the last
 *     failure of the calling thread;
 *   - all tensor pointers are DEVICE pointers owned by the caller (PyTorch);
 *     all work is asynchronous on the given cudaStream_t; nothing allocates
 *     after ds_blstm_create;
 *   - weights/gradients are flat float32 vectors in the canonical BLSTM
 *     packing documented in paper_1904_04956_b200/csrc/layout.h (the
 *     reference's flat-float64 convention, objectives.py:3-5, at 4 B/param).
 *
 * Each entry point names the reference interface it replaces
 * (/root/reference/pkg/src/distsgd/...).
 */
#ifndef DS_BLSTM_H
#define DS_BLSTM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DS_OK 0
#define DS_ERR_ARG (-1)       /* shape / config error  -> ValueError   */
#define DS_ERR_CUDA (-2)      /* CUDA failure          -> RuntimeError */
#define DS_ERR_NONFINITE (-3) /* non-finite loss/grad  -> ValueError   */

typedef struct ds_blstm ds_blstm;
typedef void* ds_stream_t; /* cudaStream_t */

typedef struct {
  int32_t layers;     /* bidirectional LSTM layers (paper: 6)             */
  int32_t input_dim;  /* feature dim (paper: 260), <= 272                 */
  int32_t bottleneck; /* linear bottleneck units (paper: 256), %64 == 0   */
  int32_t classes;    /* soft-max outputs (paper: 32000), %16 == 0        */
  int32_t frames;     /* unrolled frames T (paper: 21)                    */
  int32_t max_batch;  /* workspace is sized for this many sequences       */
} ds_blstm_cfg;       /* hidden size is fixed at 512 cells per direction  */

/* Number of parameters of the packed model (objective.param_dim,
 * objectives.py:93-95 for the reference's tiny-mlp analogue). */
int64_t ds_blstm_param_dim(const ds_blstm_cfg* cfg);

/* Objective construction (objectives.py:111-131 make_objective). */
int ds_blstm_create(const ds_blstm_cfg* cfg, int device, ds_blstm** out);
int ds_blstm_destroy(ds_blstm* h);

/* Bind the device-resident dataset (objectives.py:23-43 Dataset):
 * feats bf16 [n_seq, frames, 272] (columns >= input_dim zero), labels int32
 * [n_seq, frames].  Pointers are borrowed. */
int ds_blstm_set_dataset(ds_blstm* h, const void* feats_bf16, const int32_t* labels, int64_t n_seq);

/* K2: operand snapshot of theta (the copy `snap = st.weights.copy()` of
 * engines/adpsgd.py:132-134 that the gradient is computed on). */
int ds_blstm_cast_snapshot(ds_blstm* h, const float* theta, ds_stream_t stream);

/* K1,K3-K8: gradient(objective, snapshot, batch, dataset)
 * (objectives.py:236-263): grad <- d/dtheta mean-over-frames CE of the
 * minibatch `idx` (int64 [B], device).  *loss_sum <- sum of per-frame CE
 * (device float); *nonfinite |= 1 when the loss is not finite.  Uses the
 * snapshot set by the last ds_blstm_cast_snapshot / ds_sgd_momentum. */
int ds_blstm_fwd_bwd(ds_blstm* h, const int64_t* idx, int32_t B, float* grad, float* loss_sum, int32_t* nonfinite,
                     ds_stream_t stream);

/* K13: evaluate/heldout_loss forward only (objectives.py:223-233, 286-291). */
/* One run_single / ADPSGD-local training step in a single call (the
 * reference's gradient(...) followed by sgd_step(...), engines/single.py:
 * 49-55, optim.py:109-121): forward, backward into `grad`, and the momentum
 * update v <- mu v + g, theta <- theta - lr v with the bf16 operand snapshot
 * refreshed.  Each layer's update starts as soon as its gradient is final and
 * runs beside the next layer's BPTT; arithmetic is identical to
 * ds_blstm_fwd_bwd + ds_sgd_momentum. */
int ds_blstm_train_step(ds_blstm* h, const int64_t* idx, int32_t B, float* theta, float* vel, float* grad, float lr,
                        float mu, float* loss_sum, int32_t* nonfinite, ds_stream_t stream);

int ds_blstm_loss(ds_blstm* h, const int64_t* idx, int32_t B, float* loss_sum, int32_t* nonfinite,
                  ds_stream_t stream);

/* K9 (+K2 fused): sgd_step (optim.py:109-121): v <- mu*v + g;
 * theta <- theta - lr*v; if snap_owner != NULL also refresh its operand
 * snapshot from the new theta.  *nonfinite |= 1 on a non-finite gradient. */
int ds_sgd_momentum(float* theta, float* v, const float* g, float lr, float mu, int64_t n, ds_blstm* snap_owner,
                    int32_t* nonfinite, ds_stream_t stream);

/* K10: adpsgd_mix (engines/adpsgd.py:36-43) + the receiver's atomic
 * reply-and-mix (:280-286): a <- b <- (a + b) / 2, the identical fp32 value
 * stored to both sides (peer pointer allowed: NVLink P2P). */
int ds_adpsgd_mix(float* theta_a, float* theta_b, int64_t n, ds_stream_t stream);

/* K11/K12: RingAllreduceGroup.allreduce (collective.py:122-163) fused with
 * the SSGD update of engines/ssgd.py:85-87, executed for the chunks owned by
 * `rank` of make_chunk_plan(n, world, nchunks) (collective.py:79-95):
 *   mode 0: g_mean = (sum in canonical owner-first ring order) / world, then
 *           per-member sgd_step; results stored into every member's buffers;
 *   mode 1: theta <- (canonical sum of theta) / world for every member
 *           (epoch consensus, engines/adpsgd.py:293-295; Hybrid pull).
 * Arrays hold one device pointer per member (peer pointers allowed).
 * snap_owners may be NULL or hold per-member handles to refresh. */
int ds_group_reduce(int32_t world, int32_t rank, float* const* grads, float* const* thetas, float* const* vels,
                    ds_blstm* const* snap_owners, int64_t n, int32_t nchunks, float lr, float mu, int32_t mode,
                    float divisor, ds_stream_t stream);
/* `divisor` (mode 0): g_mean = canonical_sum / divisor; <= 0 selects `world`
 * (the SSGD `/ learners` of engines/ssgd.py:85).  H-ADPSGD passes 1 with
 * member gradients already scaled by 1/(group frames). */

/* K12: consensus out = (((x_0 + x_1) + ...) + x_{n-1}) / n in member order
 * (np.mean(np.stack(..)) of engines/adpsgd.py:293-295 / :339-342). */
int ds_average(int32_t n, float* const* srcs, float* out, int64_t dim, ds_stream_t stream);

/* CE gradient divisor override for the following ds_blstm_fwd_bwd calls:
 * frames_total > 0 scales dlogits by 1/frames_total instead of 1/(B*T) so a
 * group's member gradients sum to the gradient of the union batch (H-ADPSGD,
 * SURVEY §8 a19).  0 restores the per-batch mean. */
int ds_blstm_set_grad_scale(ds_blstm* h, float frames_total);

/* Read one device float (the step's loss sum) back to the host: 4-byte copy
 * through the handle's pinned slot on `stream`, then waits for the stream
 * (everything queued before it included). */
int ds_blstm_read_loss(ds_blstm* h, const float* loss_sum_dev, ds_stream_t stream, float* out);

/* Precision mode of the handle's gradient / loss / train-step calls:
 *   DS_PREC_BF16 (default) — the performance path: bf16 tensor-core operands
 *     and stored activations, fp32 accumulation, cell state and master weights;
 *   DS_PREC_FP32 — the parity path for the reference's float64 arithmetic
 *     (objectives.py:3-5, 236-263): every GEMM on tcgen05 kind::tf32 with the
 *     3xTF32 split (hi*hi + hi*lo + lo*hi, ~fp32 products), fp32 activations,
 *     accurate exp/tanh, materialised fp32 logits.  Allocates its own
 *     workspace (~6 GB at B = 256 paper size) on first selection; the operand
 *     snapshot becomes the fp32 hi/lo splits (call ds_blstm_cast_snapshot
 *     after switching). */
#define DS_PREC_BF16 0
#define DS_PREC_FP32 1
int ds_blstm_set_precision(ds_blstm* h, int32_t mode);
int32_t ds_blstm_get_precision(ds_blstm* h);

/* Phase profiling (bench/tests): when enabled the step is issued without the
 * CUDA graph and CUDA events bracket every phase; ds_blstm_profile_read sums
 * the per-kind milliseconds since the last read into ms_by_kind[0..nkinds):
 * 0 = tcgen05 GEMMs, 1 = recurrent forward, 2 = recurrent backward,
 * 3 = gather / soft-max combine / bias column sums. */
int ds_blstm_set_profile(ds_blstm* h, int32_t enable);
int ds_blstm_profile_read(ds_blstm* h, float* ms_by_kind, int32_t nkinds);
/* Individual phase intervals (in issue order) since the last read, without
 * clearing them (call before ds_blstm_profile_read). */
int ds_blstm_profile_list(ds_blstm* h, float* ms, int32_t* kinds, int32_t max_n, int32_t* n_out);
/* Kernel launches issued by the last ds_blstm_fwd_bwd / ds_blstm_loss. */
int32_t ds_blstm_kernel_count(ds_blstm* h);

/* GEMM self-test hook (tests only): C[M,N] f32 = A . B^T with bf16 operands,
 * a_mn/b_mn select MN-major storage ([K][M] / [K][N]). */
int ds_debug_gemm_bf16(const void* A, int64_t lda, int32_t a_mn, const void* B, int64_t ldb, int32_t b_mn, float* C,
                       int64_t ldc, int32_t M, int32_t N, int32_t K, ds_stream_t stream);
/* Record a per-CTA, per-tile timeline of the `launch`-th GEMM launch issued
 * from now on into `buf` (device, zeroed, >= 2*80*8*8 uint64); buf = NULL turns
 * it off; launch = -1 traces the fused soft-max/dZ kernel instead.  Profiling
 * aid for tools/gemm_trace.py and tools/cedz_trace.py; never used on the
 * product path. */
int ds_debug_gemm_trace(void* buf, int32_t launch);
/* debug: marks (globaltimer ns) of the BPTT of `layer` inside the step graph, layout of
 * tools/bwd_step_trace.py ([CTA][step][6] + per-chunk slots; null: off); takes effect at the next
 * graph capture */
int ds_debug_bptt_trace(void* buf, int32_t layer);

/* ---------------------------------------------------------------------------
 * Multi-process data parallelism (one process per GPU, NVLink P2P).
 * These replace the reference's in-process transports for a learner group
 * (RingAllreduceGroup, collective.py:81-163; the ADPSGD channels and
 * adpsgd_mix, engines/adpsgd.py:36-43,184-207,280-286) when every learner is
 * its own process: buffers are shared through CUDA IPC and the sync kernels
 * read and write the peers' memory directly.  NCCL is only the comparison.
 */
#define DS_IPC_HANDLE_BYTES 64

/* Export the allocation holding `ptr`: 64-byte IPC handle + byte offset. */
int ds_ipc_export(const void* ptr, void* handle_out, int64_t* offset_out);
/* Map a peer's exported allocation into this process (current device);
 * *base_out is what ds_ipc_close takes, *ptr_out = base + offset. */
int ds_ipc_open(const void* handle, int64_t offset, void** base_out, void** ptr_out);
int ds_ipc_close(void* base);
/* Stream-ordered copy between any two device (or peer-mapped) pointers. */
int ds_device_copy(void* dst, const void* src, int64_t bytes, ds_stream_t stream);
/* Single-process multi-device groups: enable device -> peer access. */
int ds_enable_peer_access(int32_t device, int32_t peer);

/* bf16 operand snapshot buffer of a handle (param_dim elements) so a peer
 * can refresh it together with theta, and the snapshot extras (padded layer-0
 * W_ih, fp32 biases) a learner re-derives from its own theta afterwards. */
void* ds_blstm_snapshot_ptr(ds_blstm* h);
int ds_blstm_snapshot_aux(ds_blstm* h, const float* theta, ds_stream_t stream);

/* Device-side barrier of n members: flag word member_flags[m][my_rank] is set
 * to e_m = ++pair_epochs[member_ranks[m]] for every member m, then the call
 * waits on the stream until own_flags[member_ranks[m]] >= e_m (wrap-safe).
 * pair_epochs is a device array [64] of this rank's per-pair barrier counts
 * (incremented by the kernel, so ranks may take part in different subsets of
 * barriers and the barrier can be replayed inside a CUDA graph).  After
 * timeout_s the wait gives up and sets *err |= 1 (checked by the host): a
 * lost peer never hangs. */
int ds_peer_barrier(int32_t n, uint32_t* const* member_flags, const int32_t* member_ranks, int32_t my_rank,
                    uint32_t* own_flags, uint32_t* pair_epochs, int32_t* err, double timeout_s, ds_stream_t stream);

/* SSGD group of the fused training step (engines/ssgd.py:80-90 with the
 * allreduce of collective.py:122-163 overlapped with the backward): when set,
 * ds_blstm_train_step replaces each layer's local momentum update by
 *   barrier -> reduce the owned chunks of that layer's gradient block in the
 *   canonical owner-first order, / divisor, momentum SGD, store theta and its
 *   bf16 snapshot into every member -> barrier
 * on the side stream as soon as the layer's gradient is final (while the
 * BPTT of the layer below runs).  Results are bit-identical to the
 * whole-vector ds_shard_step.  Member buffers are peer-mapped pointers. */
#define DS_MAX_GROUP 16
typedef struct {
  int32_t n;          /* members (learners of the group)                       */
  int32_t me;         /* this learner's member index = chunk owner id           */
  int32_t my_rank;    /* this process's world rank (barrier flag slot)          */
  int32_t nchunks;    /* make_chunk_plan(param_dim, n, nchunks), >= n           */
  float divisor;      /* g_mean = sum / divisor; <= 0 selects n                 */
  int32_t max_blocks; /* grid cap of the per-layer sync kernels (0: default 64) */
  int32_t ranks[DS_MAX_GROUP];
  float* thetas[DS_MAX_GROUP];
  const float* grads[DS_MAX_GROUP];
  void* snaps[DS_MAX_GROUP];
  uint32_t* flags[DS_MAX_GROUP];
  uint32_t* own_flags;
  uint32_t* pair_epochs;
  int32_t* err;
  double timeout_s;
} ds_group_desc;
/* NULL clears (back to the local momentum update). */
int ds_blstm_set_group(ds_blstm* h, const ds_group_desc* g);

/* Exclusive access to one learner's weights across devices (the receiver's
 * atomic region of engines/adpsgd.py:280-285 without a receiver thread): a
 * system-scope CAS on a lock word in the owner's memory (peer pointer
 * allowed) by one thread on `stream`; owner != 0 identifies the holder.
 * Timeout sets *err |= 2.  Every work item ordered between ds_peer_lock and
 * ds_peer_unlock on the stream runs while the lock is held. */
int ds_peer_lock(uint32_t* word, uint32_t owner, int32_t* err, double timeout_s, ds_stream_t stream);
int ds_peer_unlock(uint32_t* word, ds_stream_t stream);

/* N1, ADPSGD throughput mode: the sender's sgd_step (optim.py:109-121) and
 * its pairwise average (adpsgd_mix, engines/adpsgd.py:36-43) in one pass:
 * v <- mu v + g; t' = theta - lr v; snap <- bf16(t') (nullable: the next
 * gradient's operands, pre-mix as in the reference); m = (t' + peer) / 2
 * stored to theta and peer (peer pointer: one NVLink read + write). */
int ds_update_mix(float* theta, float* vel, const float* grad, float* theta_peer, void* snap, float lr, float mu,
                  int64_t n, int32_t* nonfinite, ds_stream_t stream);

/* Debug payload digest replacing the reference's blake2b WeightMessage
 * checksum (engines/common.py:78-104): 128 bits over the buffer's 32-bit
 * words written to out2[0..1] (device) on `stream`. */
int ds_digest(const void* data, int64_t nbytes, unsigned long long* out2, ds_stream_t stream);

/* Sharded group step of rank `rank` (RingAllreduceGroup.allreduce + /world +
 * sgd_step, engines/ssgd.py:84-87): for the chunks this rank owns
 * (j % world == rank, make_chunk_plan) sum the members' gradients in the
 * canonical ring order, divide, update this rank's velocity and theta, and
 * store theta (+ bf16 snapshot) into every member.  mode 1 averages theta
 * instead (Hybrid, engines/hybrid.py:97-99).  Call between two barriers. */
int ds_shard_step(int32_t world, int32_t rank, const float* const* grads, float* const* thetas,
                  void* const* snaps, float* v_own, int64_t n, int32_t nchunks, float lr, float mu, int32_t mode,
                  float divisor, ds_stream_t stream);
/* The same restricted to elements [range_lo, range_hi) (range_lo % 4 == 0):
 * one parameter block (a layer) synchronised as soon as its gradient is
 * final, with the chunk ownership and summation order of the whole-vector
 * plan (bit-identical results); max_blocks > 0 caps the grid (side stream). */
int ds_shard_step_range(int32_t world, int32_t rank, const float* const* grads, float* const* thetas,
                        void* const* snaps, float* v_own, int64_t n, int32_t nchunks, float lr, float mu,
                        int32_t mode, float divisor, int64_t range_lo, int64_t range_hi, int32_t max_blocks,
                        ds_stream_t stream);

/* ADPSGD pairwise average (adpsgd_mix) over P2P: m = (self + peer) / 2 on
 * half 0 ([0, n/2)), half 1 ([n/2, n)) or -1 (all), stored to both sides and
 * to their bf16 snapshots (nullable). */
int ds_pair_mix(float* self, float* peer, void* snap_self, void* snap_peer, int64_t n, int32_t half,
                ds_stream_t stream);

/* Recurrent-kernel self-test hooks (tests only): run one bidirectional layer's
 * forward / backward recurrence on caller buffers (layouts of lstm_rec.cu;
 * whh = W_hh bf16 [4096, 512] for both directions of recurrence).
 * counters: >= 640*ceil(B/128) words, zeroed once (the flags count up across
 * launches, so the buffer is reused without resetting); trace (nullable): [grid][T][4] u64
 * globaltimer marks (producer ready, loads issued, MMA done, step published). */
int ds_debug_lstm_fwd(int32_t B, int32_t T, void* gates, float* cstate, void* y_full, const void* whh,
                      uint32_t* counters, uint64_t* trace, ds_stream_t stream);
int ds_debug_lstm_bwd(int32_t B, int32_t T, const void* gates, const float* cstate, const void* whh, const void* dy,
                      void* dg, uint32_t* counters, uint64_t* trace, ds_stream_t stream);

/* GEMM self-test hook (tests only): C[M,N] (+)= A . B^T, fp32 row-major
 * operands through the FP32-parity 3xTF32 tcgen05 GEMM. */
int ds_debug_gemm_tf32x3(const float* A, int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc, int32_t M,
                         int32_t N, int32_t K, int32_t accumulate, ds_stream_t stream);

const char* ds_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* DS_BLSTM_H */
