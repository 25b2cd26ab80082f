// blstm.cu — the ds_blstm handle: workspace, operand snapshot and the full
// training-step schedule of the paper BLSTM issued as one CUDA
// graph per (batch, buffer) binding.  Implements the C ABI of
// include/ds_blstm.h.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/ds_blstm.h"
#include "ds_internal.h"
#include "layout.h"
#include "lstm_rec.h"
#include "ops.h"
#include "p2p.h"
#include "parity.h"
#include "softmax_dz.h"

using namespace ds;

struct ds_blstm {
  ds_blstm_cfg cfg;
  ModelLayout L;
  int device = 0;
  int T = 0, Bmax = 0;
  int64_t Nmax = 0;
  int ntiles_c = 0;
  // dataset (borrowed)
  const __nv_bfloat16* feats = nullptr;
  const int32_t* labels = nullptr;
  int64_t n_seq = 0;
  // one device allocation holding everything below
  void* arena = nullptr;
  // operand snapshot
  __nv_bfloat16* snap = nullptr;
  __nv_bfloat16* wih0pad = nullptr;
  float* bias_snap = nullptr;
  // activations
  __nv_bfloat16* x0 = nullptr;
  int32_t* lab = nullptr;
  std::vector<__nv_bfloat16*> gates, yfull;
  std::vector<float*> cstate;
  __nv_bfloat16* z = nullptr;
  float2* stats = nullptr;
  float* tgt = nullptr;
  float* lse = nullptr;
  __nv_bfloat16* dlogits = nullptr;
  __nv_bfloat16* dz = nullptr;
  __nv_bfloat16* dy = nullptr;
  __nv_bfloat16* dg = nullptr;
  __nv_bfloat16* dg2 = nullptr;  // overlapped backward: dG of layer l in buffer l % 3 (dg, dg2, dg3), so
  __nv_bfloat16* dg3 = nullptr;  //   BPTT_{l-1} waits only for the readers of layer l+2's
  float* colpart = nullptr;
  float* biaspart = nullptr;  // fused bias-gradient partials (CE grad epilogue / BPTT kernel)
  float* biaspart2 = nullptr;  // BPTT bias partials of layer l in buffer l % 3 (biaspart, biaspart2, biaspart3)
  float* biaspart3 = nullptr;
  float* splitk = nullptr;    // split-K fp32 partials of dZ
  uint32_t* counters = nullptr;
  float* d_lr = nullptr;  // fused training step: learning rate read by the SGD kernels
  float lr_host = -1.f;   // value last written to d_lr (written again only when it changes)
  float* loss_pinned = nullptr;  // pinned host slot for ds_blstm_read_loss
  // fused training step: per-layer SGD on a side stream while the next BPTT runs
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork[kMaxLayers + 2] = {}, ev_join[kMaxLayers + 2] = {};
  cudaEvent_t ev_aux[4] = {};  // output-layer bias reductions on the side stream
  // per-layer bias-gradient row sums beside the layer's weight-gradient GEMMs
  cudaStream_t side2 = nullptr;
  cudaEvent_t ev_rs[kMaxLayers][2] = {};
  // weight-gradient GEMMs of layer l beside BPTT_{l-1} (narrow BPTT only): low-priority stream
  cudaStream_t side3 = nullptr;
  cudaEvent_t ev_dw[kMaxLayers][2] = {};  // [0] BPTT_l done, [1] dW_l done
  cudaEvent_t ev_x[kMaxLayers] = {};      // dX_l (streamed behind BPTT_l on side4) done
  // dX_l = dG_l W_ih_l streamed behind BPTT_l in direction-split units (high-priority stream)
  cudaStream_t side4 = nullptr;
  // its outputs: dY_{l-1} = dyx[l & 1][0] (direction-0 dG) + dyx[l & 1][1] (direction-1 dG); by layer
  // parity, since a half gated on one BPTT direction must not overwrite rows the other still reads
  __nv_bfloat16* dyx[2][2] = {};
  cudaEvent_t ev_gz[2] = {};              // gate counters zeroed (fork / join)
  int prio_hi = 0, prio_lo = 0;
  // graph cache
  struct Key {
    int B;
    const int64_t* idx;
    float* grad;
    float* loss;
    int* flag;
    int bwd;
    float gscale;
    float* theta;
    float* vel;
    float mu;
    const void* grp;
    bool operator==(const Key& o) const {
      return B == o.B && idx == o.idx && grad == o.grad && loss == o.loss && flag == o.flag && bwd == o.bwd &&
             gscale == o.gscale && theta == o.theta && vel == o.vel && mu == o.mu && grp == o.grp;
    }
  };
  struct Entry {
    Key key;
    cudaGraphExec_t exec;
  };
  std::vector<Entry> graphs;
  // phase profiling (tests / bench only; bypasses the graph)
  int profile = 0;
  // debug timeline (DS_TIMELINE=1): timing events recorded inside the step graph on every stream
  unsigned long long* tl_buf = nullptr;  // device globaltimer stamps (graph-safe, unlike event timing)
  std::vector<std::string> tl_name;
  int tl_n = 0;
  std::vector<cudaEvent_t> ev;
  std::vector<int> ev_kind;
  int launches = 0;  // kernel launches issued by the last step
  float grad_frames = 0.f;  // CE gradient divisor override (0: B*T)
  int pad_B = -1;           // batch size the Y_full zero pads were laid out for
  // precision mode: 0 = BF16 perf path, 1 = FP32 parity (3xTF32 tcgen05, parity.cu)
  int prec = 0;
  ParityWs* par = nullptr;
  // SSGD peer group of the fused training step (ds_blstm_set_group)
  GroupSync grp;
  bool grp_on = false;
};

namespace {

// dZ = dlogits . W_o has K = classes (500 k-blocks at 32000): split it so its
// tiles match the length of the concurrent dW_o tiles (K = frames).
constexpr int kDzSplit = 5;
constexpr int kDzPartMax = 8;  // dZ partial slices of the fused soft-max kernel
int dz_split(int classes) {
  const int nkb = (classes + kGemmBK - 1) / kGemmBK;
  return (nkb % kDzSplit == 0 && nkb >= 4 * kDzSplit) ? kDzSplit : 1;
}

// dW_b = dZ^T Y is 256 x 1024 with K = frames: 4 pair tiles of 84 k-blocks at
// B=256, so split K to spread it over the pairs that run the dY tiles.
constexpr int kWbSplit = 12;
// largest S <= target whose ceil-split leaves no split empty
int ksplit_for(int K, int target) {
  const int nkb = (K + kGemmBK - 1) / kGemmBK;
  for (int S = target < nkb ? target : nkb; S > 1; --S) {
    const int per = (nkb + S - 1) / S;
    if ((S - 1) * per < nkb) return S;
  }
  return 1;
}

// dlogits in 64x64 blocks: the dW_o (MN-major) and dZ (K-major) operand
// boxes become contiguous 8 KB reads instead of 128-byte pieces of rows 64 KB
// apart (DS_DLOGITS_ROWMAJOR=1 keeps the row-major layout)
bool blocked_dlogits(const ds_blstm* h) {
  static int off = -1;
  if (off < 0) {
    const char* e = getenv("DS_DLOGITS_ROWMAJOR");
    off = (e && e[0] == '1') ? 1 : 0;
  }
  return !off && h->L.classes % 64 == 0;
}

// fused soft-max gradient + dZ (softmax_dz.cu) when dlogits is blocked and
// the shape fits (DS_NO_FUSED_CE=1 keeps the separate GEMMs)
bool fused_ce_dz(const ds_blstm* h) {
  static int off = -1;
  if (off < 0) {
    const char* e = getenv("DS_NO_FUSED_CE");
    off = (e && e[0] == '1') ? 1 : 0;
  }
  return !off && blocked_dlogits(h) && ce_grad_dz_supported(h->L.classes, h->L.bottleneck);
}
// the soft-max combine's last-block ticket: a word of the zeroed slack after the recurrent flags
unsigned* ce_ticket(const ds_blstm* h) { return h->counters + lstm_counter_words(h->Bmax); }
uint32_t* seq_words(const ds_blstm* h) { return h->counters + lstm_counter_words(h->Bmax) + 32; }
int dw0_early() {  // frames per direction of layer 0's weight gradients computed beside BPTT_0 (DS_DW0_EARLY)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DS_DW0_EARLY");
    v = e ? atoi(e) : 8;
    if (v < 0) v = 0;
  }
  return v;
}
int dx_pairs() {  // CTA pairs the streamed dX holds beside the BPTT (DS_DX_PAIRS)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DS_DX_PAIRS");
    v = e ? atoi(e) : 16;
    if (v < 1) v = 1;
  }
  return v;
}
// Per-step counters after the recurrent flags (zeroed per step, one memset), per layer: [2][T] BPTT
// completion counters (per direction and time step, gating dX_l) and [T][2][2] dY completion counters
// (dX_{l+1}'s two per-direction outputs, per frame and unit direction, gating BPTT_l)
uint32_t* gate_words(const ds_blstm* h, int l) { return h->counters + lstm_counter_words(h->Bmax) + 64 + (size_t)l * 6 * h->T; }
uint32_t* ready_words(const ds_blstm* h, int l) { return gate_words(h, l) + 2 * h->T; }
size_t counter_words_total(const ds_blstm* h) { return lstm_counter_words(h->Bmax) + 64 + (size_t)kMaxLayers * 6 * h->T; }
// Host list schedule of the streamed dX: a unit (direction d's problem, row tile, column tile) becomes
// available when direction d of the BPTT has finished all its frames (direction 0 finishes frame t at
// step T-1-t, direction 1 at step t); units go, in order of availability, to the CTA pair that frees
// up first under a simple cost model (a BPTT step ~ 14 k-blocks of a pair tile).
int dx_schedule(GemmBatch& g, int pairs, int B, int T) {
  struct Unit {
    int avail, need, tile;
    double dur;
  };
  std::vector<Unit> us;
  int begin = 0;
  for (int d = 0; d < g.nprob; ++d) {
    const GemmProblem& P = g.p[d];
    const int n = P.tiles_m * P.tiles_n;
    for (int local = 0; local < n; ++local) {  // the kernel's mapping: row tile fastest, then column tile
      const int tm = local % P.tiles_m, tn = local / P.tiles_m;
      const int r0 = tm * 2 * kGemmBM, r1 = std::min(r0 + 2 * kGemmBM, P.M) - 1;
      // the dY columns of the tile belong to the next BPTT's direction u (units u*512 ..), which reads
      // frame t at its step T-1-t (u = 0) or t (u = 1): among units released at the same step, the
      // ones that BPTT needs first go first
      const int u = (tn * kGemmBN) / kHidden;
      int avail = 0, need = T;
      for (int t = r0 / B; t <= r1 / B; ++t) {
        avail = std::max(avail, d == 0 ? T - 1 - t : t);
        need = std::min(need, u == 0 ? T - 1 - t : t);
      }
      us.push_back({avail, need, begin + local, (P.K + kGemmBK - 1) / kGemmBK + 3.0});
    }
    begin += n;
  }
  if ((int)us.size() > kMaxSched || pairs > kMaxPairs) return fail_arg("streamed dX: too many units");
  std::stable_sort(us.begin(), us.end(), [](const Unit& a, const Unit& b) {
    return a.avail != b.avail ? a.avail < b.avail : a.need < b.need;
  });
  std::vector<double> fr(pairs, 0.0);
  std::vector<std::vector<int>> lists(pairs);
  for (const Unit& u : us) {
    int best = 0;
    for (int q = 1; q < pairs; ++q)
      if (fr[q] < fr[best]) best = q;
    fr[best] = std::max(fr[best], 14.0 * u.avail) + u.dur;
    lists[best].push_back(u.tile);
  }
  int pos = 0;
  for (int q = 0; q < pairs; ++q) {
    g.pstart[q] = (uint16_t)pos;
    for (int t : lists[q]) g.order[pos++] = (uint16_t)t;
  }
  g.pstart[pairs] = (uint16_t)pos;
  g.sched = 1;
  g.presched = pairs;
  return DS_OK;
}
// debug (tools/bptt_insitu.py): per-(CTA, step) marks of one layer's BPTT inside the step graph
uint64_t* g_bptt_trace = nullptr;
int g_bptt_layer = -1;
int fused_dz_splits(const ds_blstm* h, int N) {
  // h->splitk holds kDzPartMax x N x bottleneck floats
  return ce_grad_dz_splits(N, h->L.classes, kDzPartMax);
}

struct Arena {
  size_t off = 0;
  template <class T>
  T* take(char* base, size_t count) {
    off = (off + 255) & ~size_t(255);
    T* p = reinterpret_cast<T*>(base + off);
    off += count * sizeof(T);
    return p;
  }
};

int carve(ds_blstm* h, char* base, size_t* total) {
  Arena a;
  const ModelLayout& L = h->L;
  const int64_t N = h->Nmax;
  h->snap = a.take<__nv_bfloat16>(base, L.total);
  h->wih0pad = a.take<__nv_bfloat16>(base, (size_t)kGates2 * kInPad);
  // [layers][4096] b, b_b, b_o, b_o * log2(e) (CE-stats epilogue: one FFMA per logit)
  h->bias_snap = a.take<float>(base, (size_t)L.layers * kGates2 + L.bottleneck + 2 * (size_t)L.classes);
  h->x0 = a.take<__nv_bfloat16>(base, (size_t)N * kInPad);
  h->lab = a.take<int32_t>(base, N);
  h->gates.resize(L.layers);
  h->cstate.resize(L.layers);
  h->yfull.resize(L.layers);
  for (int l = 0; l < L.layers; ++l) {
    h->gates[l] = a.take<__nv_bfloat16>(base, (size_t)N * kGates2);
    h->cstate[l] = a.take<float>(base, (size_t)N * kLayerOut);
    h->yfull[l] = a.take<__nv_bfloat16>(base, (size_t)(h->T + 2) * h->Bmax * kLayerOut);
  }
  h->z = a.take<__nv_bfloat16>(base, (size_t)N * L.bottleneck);
  h->stats = a.take<float2>(base, (size_t)4 * h->ntiles_c * N);  // four column quarters per tile
  h->tgt = a.take<float>(base, N);
  h->lse = a.take<float>(base, N);
  {  // row-major [N][C], or 64x64-blocked when C % 64 == 0
    const int64_t e1 = (int64_t)N * L.classes, e2 = gemm_blocked_elems(N, L.classes);
    h->dlogits = a.take<__nv_bfloat16>(base, e1 > e2 ? e1 : e2);
  }
  h->dz = a.take<__nv_bfloat16>(base, (size_t)N * L.bottleneck);
  h->dy = a.take<__nv_bfloat16>(base, (size_t)N * kLayerOut);
  for (int i = 0; i < 4; ++i) h->dyx[i / 2][i % 2] = a.take<__nv_bfloat16>(base, (size_t)N * kLayerOut);
  h->dg = a.take<__nv_bfloat16>(base, (size_t)N * kGates2);
  h->dg2 = a.take<__nv_bfloat16>(base, (size_t)N * kGates2);
  h->dg3 = a.take<__nv_bfloat16>(base, (size_t)N * kGates2);
  {  // bottleneck bias colsum partials / CE loss partials
    const int64_t c1 = op_colsum_scratch(N, L.bottleneck), c2 = (N + 31) / 32 + 64;
    h->colpart = a.take<float>(base, c1 > c2 ? c1 : c2);
  }
  {
    const int64_t tiles_m = (N + kGemmBM - 1) / kGemmBM;
    const int64_t a1 = tiles_m * 4 * L.classes;
    const int64_t a2 = (int64_t)((h->Bmax + 127) / 128) * 4 * kGates2;
    h->biaspart = a.take<float>(base, a1 > a2 ? a1 : a2);
    h->biaspart2 = a.take<float>(base, a2);
    h->biaspart3 = a.take<float>(base, a2);
  }
  {  // split-K fp32 partials: dZ (K = classes) and dW_b (K = frames)
    const int64_t s1 = (int64_t)kDzPartMax * N * L.bottleneck, s2 = (int64_t)kWbSplit * L.bottleneck * kLayerOut;
    const int64_t s3 = L.off_b[0] - L.off_wih[0];  // the late layer-0 weight gradients of the fused step
    h->splitk = a.take<float>(base, std::max(std::max(s1, s2), s3));
  }
  h->counters = a.take<uint32_t>(base, counter_words_total(h));
  h->d_lr = a.take<float>(base, 4);
  *total = a.off + 256;
  return DS_OK;
}

int validate_cfg(const ds_blstm_cfg* c) {
  if (!c) return fail_arg("null config");
  if (c->layers < 1 || c->layers > kMaxLayers) return fail_arg("layers must be in 1..16");
  if (c->input_dim < 1 || c->input_dim > kInPad) return fail_arg("input_dim must be in 1..272");
  if (c->bottleneck < 64 || c->bottleneck % 64) return fail_arg("bottleneck must be a positive multiple of 64");
  if (c->classes < 16 || c->classes % 16) return fail_arg("classes must be a positive multiple of 16");
  if (c->frames < 1 || c->frames > 1024) return fail_arg("frames must be in 1..1024");
  if (c->max_batch < 1 || c->max_batch > 65536) return fail_arg("max_batch must be in 1..65536");
  return DS_OK;
}

// phase kinds for profiling
enum { PH_GEMM = 0, PH_LSTM_FWD = 1, PH_LSTM_BWD = 2, PH_OTHER = 3, PH_END = 4 };

bool use_timeline() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DS_TIMELINE");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}
__global__ void tl_stamp_kernel(unsigned long long* slot) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *slot = t;
}
int tl_mark(ds_blstm* h, const std::string& name, cudaStream_t s) {
  if (!use_timeline()) return DS_OK;
  if (!h->tl_buf || h->tl_n >= 256) return DS_OK;
  if (h->tl_n >= (int)h->tl_name.size()) h->tl_name.push_back(name);
  h->tl_name[h->tl_n] = name;
  tl_stamp_kernel<<<1, 1, 0, s>>>(h->tl_buf + h->tl_n++);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int mark(ds_blstm* h, int kind, cudaStream_t s) {
  if (!h->profile) return DS_OK;
  cudaEvent_t e;
  DS_CUDA_TRY(cudaEventCreate(&e));
  DS_CUDA_TRY(cudaEventRecord(e, s));
  h->ev.push_back(e);
  h->ev_kind.push_back(kind);
  return DS_OK;
}

// ---------------------------------------------------------------------------
// The step schedule.  Forward always runs; backward when `grad` != nullptr.
// Fused momentum SGD (K9+K2) of the parameter block [off, off + n) once its
// gradient is final.  side: on the handle's side stream (<= 16 SMs, the ones
// a recurrence leaves free), forked from / joined back into `s`.
struct SgdCtx {
  const float* add0 = nullptr;     // layer 0: late weight-gradient part to sum into the gradient in its update
  int64_t add0_n = 0;
  float* theta = nullptr;
  float* vel = nullptr;
  float mu = 0.f;
  int nfork = 0;
  const GroupSync* grp = nullptr;  // SSGD: per-layer group sync instead of the local update
  bool mirror = false;             // the local updates also write the padded W_ih0 / bias snapshot copies
};
// the operand-snapshot extras (op_snapshot_aux) inside the update of the block [off, off + n)
SgdMirror segment_mirror(const ds_blstm* h, int64_t off, int64_t n) {
  const ModelLayout& L = h->L;
  SgdMirror m;
  auto in = [&](int64_t b, int64_t c) { return b >= off && b + c <= off + n; };
  if (in(L.off_wih[0], (int64_t)kGates2 * L.input_dim)) {
    m.wpad = h->wih0pad;
    m.wbeg = L.off_wih[0] - off;
    m.wcnt = (int64_t)kGates2 * L.input_dim;
    m.din = L.input_dim;
  }
  int k = 0;
  auto add = [&](int64_t b, int64_t c, float* dst, float scale) {
    if (k < 3 && in(b, c)) {
      m.fdst[k] = dst;
      m.fbeg[k] = b - off;
      m.fcnt[k] = c;
      m.fscale[k] = scale;
      ++k;
    }
  };
  float* bs = h->bias_snap;
  for (int l = 0; l < L.layers; ++l) add(L.off_b[l], kGates2, bs + (size_t)l * kGates2, 1.f);
  float* bo = bs + (size_t)L.layers * kGates2;
  add(L.off_bb, L.bottleneck, bo, 1.f);
  add(L.off_bo, L.classes, bo + L.bottleneck, 1.f);
  add(L.off_bo, L.classes, bo + L.bottleneck + L.classes, 1.4426950408889634f);  // b_o * log2(e) (CE statistics)
  return m;
}
bool mirror_ok(const ds_blstm* h) {  // every mirrored range 4-aligned (float4 update path)
  const ModelLayout& L = h->L;
  bool ok = L.input_dim % 4 == 0 && L.off_wih[0] % 4 == 0 && L.off_bb % 4 == 0 && L.off_bo % 4 == 0 &&
            L.bottleneck % 4 == 0 && L.classes % 4 == 0;
  for (int l = 0; l < L.layers; ++l) ok = ok && L.off_b[l] % 4 == 0;
  return ok;
}
// SSGD group update of [off, off + n): barrier, sharded reduce + SGD + all-gather, barrier
int group_segment(ds_blstm* h, SgdCtx& c, int64_t off, int64_t n, cudaStream_t s) {
  int rc = group_barrier(*c.grp, s);
  if (!rc) rc = group_shard_range(*c.grp, h->L.total, off, off + n, c.vel, h->d_lr, c.mu, s);
  if (!rc) rc = group_barrier(*c.grp, s);
  return rc;
}
bool use_dw_overlap() {  // DS_DW_OVERLAP=0: weight gradients after each BPTT on the main stream
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DS_DW_OVERLAP");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}
bool use_dx_stream() {  // DS_DX_STREAM=0: dX after each BPTT instead of streaming behind it
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DS_DX_STREAM");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}
int dw_pair_margin() {  // CTA pairs kept free beside the BPTT for the side-stream SGD (DS_DW_MARGIN)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DS_DW_MARGIN");
    v = e ? atoi(e) : 0;
  }
  return v;
}

int sgd_segment(ds_blstm* h, SgdCtx& c, float* grad, int* flag, int64_t off, int64_t n, bool side, cudaStream_t s) {
  if (!c.theta) return DS_OK;
  if (c.grp) {
    if (!side) return group_segment(h, c, off, n, s);
    const int k = c.nfork++;
    DS_CUDA_TRY(cudaEventRecord(h->ev_fork[k], s));
    DS_CUDA_TRY(cudaStreamWaitEvent(h->side, h->ev_fork[k], 0));
    int rc = group_segment(h, c, off, n, h->side);
    if (rc) return rc;
    DS_CUDA_TRY(cudaEventRecord(h->ev_join[k], h->side));
    return DS_OK;
  }
  SgdMirror mir = segment_mirror(h, off, n);
  if (c.add0 && off == h->L.off_wih[0]) {
    mir.add = c.add0;
    mir.add_n = c.add0_n;
  }
  if (!side)
    return op_sgd_lr(c.theta + off, c.vel + off, grad + off, h->d_lr, c.mu, n, h->snap + off, flag, 0, s,
                     c.mirror ? &mir : nullptr);
  const int k = c.nfork++;
  DS_CUDA_TRY(cudaEventRecord(h->ev_fork[k], s));
  DS_CUDA_TRY(cudaStreamWaitEvent(h->side, h->ev_fork[k], 0));
  static const int side_blocks = getenv("DS_SGD_BLOCKS") ? atoi(getenv("DS_SGD_BLOCKS")) : 48;  // 16 left the last layer's update on the critical path
  int rc = op_sgd_lr(c.theta + off, c.vel + off, grad + off, h->d_lr, c.mu, n, h->snap + off, flag, side_blocks,
                     h->side, c.mirror ? &mir : nullptr);
  if (rc) return rc;
  if ((rc = tl_mark(h, "sgd" + std::to_string(k), h->side))) return rc;
  DS_CUDA_TRY(cudaEventRecord(h->ev_join[k], h->side));
  return DS_OK;
}

int issue_step(ds_blstm* h, const int64_t* idx, int B, float* grad, float* loss, int* flag, cudaStream_t s,
               SgdCtx sg = SgdCtx()) {
  const ModelLayout& L = h->L;
  const int T = h->T;
  const int N = T * B;
  const int Lh = L.layers;
  const int bott = L.bottleneck, C = L.classes;
  const float* bias_l = h->bias_snap;
  const float* bias_b = h->bias_snap + (size_t)Lh * kGates2;
  const float* bias_o = bias_b + bott;
  int rc;
#define TRY(x)            \
  do {                    \
    if ((rc = (x))) return rc; \
  } while (0)
#define MARK(k) TRY(mark(h, k, s))
#define TL(name, st) TRY(tl_mark(h, name, st))
  int& nl = h->launches;
  nl = 0;
  h->tl_n = 0;
  TL("start", s);
  bool aux_join = false;
  bool out_side_done = false;  // ev_dw[0][1] recorded: the output-layer weight gradients ran beside BPTT_{L-1}

  MARK(PH_OTHER);
  TRY(op_gather(idx, B, T, h->feats, h->labels, h->n_seq, h->x0, h->lab, flag, s, seq_words(h)));
  auto Y = [&](int l) { return h->yfull[l] + (size_t)B * kLayerOut; };

  // ---- forward ----
  // layer 0's input projection (K = 272) inside its recurrence (DS_FWD_XFUSE=0: a GEMM before it)
  static const bool xfuse = (!getenv("DS_FWD_XFUSE") || getenv("DS_FWD_XFUSE")[0] != '0') &&
                            !(getenv("DS_FWD") && getenv("DS_FWD")[0] == '3');
  for (int l = 0; l < Lh; ++l) {
    if (l == 0 && xfuse) {
      LstmLayerArgs la{B, T, h->gates[0], h->cstate[0], h->yfull[0], h->snap + L.off_whh[0], nullptr, nullptr,
                       h->counters};
      la.err = flag;
      la.xin = h->x0;
      la.wih = h->wih0pad;
      la.xbias = bias_l;
      MARK(PH_LSTM_FWD);
      TRY(lstm_forward(la, s));
      TL("proj0", s);
      TL("fwd0", s);
      nl += 1 + (B - 1) / (128 * lstm_max_tiles());
      continue;
    }
    GemmBatch gb;
    memset(&gb, 0, sizeof(gb));
    gb.nprob = 1;
    gb.b_early = l > 0;  // B = W_ih snapshot; the predecessor (LSTM l-1) writes only A
    GemmProblem& p = gb.p[0];
    if (l == 0)
      TRY(gemm_problem(&p, h->x0, kInPad, 0, h->wih0pad, kInPad, 0, N, kGates2, kInPad));
    else
      TRY(gemm_problem(&p, Y(l - 1), kLayerOut, 0, h->snap + L.off_wih[l], kLayerOut, 0, N, kGates2, kLayerOut));
    p.epi = EPI_BF16;
    p.out = h->gates[l];
    p.ldo = kGates2;
    p.bias = bias_l + (size_t)l * kGates2;
    TRY(gemm_bf16_output(&p));
    MARK(PH_GEMM);
    TRY(gemm_launch(&gb, s));
    TL("proj" + std::to_string(l), s);
    LstmLayerArgs la{B, T, h->gates[l], h->cstate[l], h->yfull[l], h->snap + L.off_whh[l], nullptr, nullptr,
                     h->counters};
    la.err = flag;
    MARK(PH_LSTM_FWD);
    TRY(lstm_forward(la, s));
    TL("fwd" + std::to_string(l), s);
    nl += 2 + (B - 1) / (128 * lstm_max_tiles());
  }
  {
    GemmBatch gb;
    memset(&gb, 0, sizeof(gb));
    gb.nprob = 1;
    gb.b_early = 1;  // B = W_b snapshot
    GemmProblem& p = gb.p[0];
    TRY(gemm_problem(&p, Y(Lh - 1), kLayerOut, 0, h->snap + L.off_wb, kLayerOut, 0, N, bott, kLayerOut));
    p.epi = EPI_BF16;
    p.out = h->z;
    p.ldo = bott;
    p.bias = bias_b;
    TRY(gemm_bf16_output(&p));
    MARK(PH_GEMM);
    TRY(gemm_launch(&gb, s));
    MARK(PH_GEMM);
    nl += 1;
  }
  if (fused_ce_dz(h)) {  // soft-max statistics on CTA pairs (softmax_dz.cu): (max, sum) per row and class range
    const int S = fused_dz_splits(h, N);
    CeStatsArgs ca;
    ca.z = h->z;
    ca.w = h->snap + L.off_wo;
    ca.bias_log2 = bias_o + C;  // pre-scaled by log2(e)
    ca.labels = h->lab;
    ca.stats = h->stats;
    ca.stats_ld = h->Nmax;
    ca.tgt = h->tgt;
    ca.rows = N;
    ca.classes = C;
    ca.bott = bott;
    ca.splits = S;
    MARK(PH_GEMM);
    TRY(ce_stats_launch(ca, s));
    MARK(PH_OTHER);
    TRY(op_ce_combine(h->stats, S, h->Nmax, h->tgt, N, h->lse, h->colpart, ce_ticket(h), loss, flag, s));
    nl += 3;  // gather, statistics kernel, combine
  } else {
    GemmBatch gb;
    memset(&gb, 0, sizeof(gb));
    gb.nprob = 1;
    GemmProblem& p = gb.p[0];
    TRY(gemm_problem(&p, h->z, bott, 0, h->snap + L.off_wo, bott, 0, N, C, bott));
    p.epi = EPI_CE_STATS;
    p.bias = bias_o + C;  // pre-scaled by log2(e)
    p.labels = h->lab;
    p.stats = h->stats;
    p.stats_ld = (int)h->Nmax;
    p.tgt = h->tgt;
    TRY(gemm_launch(&gb, s));
    MARK(PH_OTHER);
    TRY(op_ce_combine(h->stats, gemm_stats_parts() * p.tiles_n, h->Nmax, h->tgt, N, h->lse, h->colpart,
                      ce_ticket(h), loss, flag, s));
    nl += 3;  // gather, ce stats gemm, combine
  }
  TL("ce", s);
  if (!grad) {
    MARK(PH_END);
    return DS_OK;
  }
  // Weight gradients beside the recurrence (narrow 64-CTA BPTT only): dW_o / dW_b beside BPTT_{L-1},
  // layer l's dW_ih / dW_hh beside BPTT_{l-1}, on a low-priority stream, each gated on the BPTT's
  // start and capped to the SMs it leaves free; only dY / dX stay between two BPTTs.
  const int narrow = lstm_bwd_narrow_ctas(B);
  const bool ovl = narrow > 0 && !h->profile && use_dw_overlap();
  int dw_pairs = (num_sms() - narrow) / 2 - dw_pair_margin();
  if (dw_pairs < 1) dw_pairs = 1;
  // dX_l streamed behind BPTT_l (side4, direction-split units finished in the kernel) and consumed by
  // BPTT_{l-1} frame by frame: its per-step counters are zeroed on side2 beside the output layer
  // (not with an SSGD group attached: with two learners time-sliced on one device, --same-device, the
  // group barriers timed out against the spin-gated streams; the group step keeps stream-ordered dX)
  const bool xstream = ovl && use_dx_stream() && B % 32 == 0 && !sg.grp;
  const int dxp = xstream ? std::min(dx_pairs(), dw_pairs - 1) : 0;
  if (xstream) {
    DS_CUDA_TRY(cudaEventRecord(h->ev_gz[0], s));
    DS_CUDA_TRY(cudaStreamWaitEvent(h->side2, h->ev_gz[0], 0));
    DS_CUDA_TRY(cudaMemsetAsync(gate_words(h, 0), 0, sizeof(uint32_t) * (size_t)Lh * 6 * T, h->side2));
    DS_CUDA_TRY(cudaEventRecord(h->ev_gz[1], h->side2));
    DS_CUDA_TRY(cudaStreamWaitEvent(h->side4, h->ev_gz[1], 0));
  }

  // ---- backward ----
  GemmProblem pwo;  // fused path: dW_o joins the dW_b / dY launch below
  bool have_wo = false;
  if (fused_ce_dz(h)) {
    // soft-max gradient + dZ in one pass (softmax_dz.cu); dW_o then shares one GEMM launch
    // with dW_b and dY (their tiles fill the wave-quantisation gap of dW_o's 125 tiles)
    const int S = fused_dz_splits(h, N);
    CeGradDzArgs ca;
    ca.z = h->z;
    ca.w = h->snap + L.off_wo;
    ca.bias = bias_o;
    ca.labels = h->lab;
    ca.lse = h->lse;
    ca.dlogits = h->dlogits;
    ca.colpart = h->biaspart;
    ca.dzpart = h->splitk;
    ca.scale = 1.0f / (h->grad_frames > 0.f ? h->grad_frames : (float)N);
    ca.rows = N;
    ca.classes = C;
    ca.bott = bott;
    ca.splits = S;
    MARK(PH_GEMM);
    TRY(ce_grad_dz_launch(ca, s));
    MARK(PH_OTHER);
    // db_o only feeds the output-layer update: reduce it on the side stream
    // (joined before the first BPTT, which reuses the partials buffer)
    cudaStream_t rs = s;
    if (sg.theta && !h->profile) {
      DS_CUDA_TRY(cudaEventRecord(h->ev_aux[0], s));
      DS_CUDA_TRY(cudaStreamWaitEvent(h->side, h->ev_aux[0], 0));
      rs = h->side;
    }
    TRY(op_rowsum(h->biaspart, ((N + kGemmBM - 1) / kGemmBM) * 4, C, grad + L.off_bo, rs));
    if (rs != s) DS_CUDA_TRY(cudaEventRecord(h->ev_aux[1], rs));
    aux_join = rs != s;
    TRY(op_splitk_bf16(h->splitk, S, (int64_t)N * bott, h->dz, s));
    TRY(gemm_problem(&pwo, h->dlogits, C, 1, h->z, bott, 1, C, bott, N));  // dW_o = dlogits^T Z
    TRY(gemm_blocked_a(&pwo, h->dlogits, N, C));
    pwo.epi = EPI_F32;
    pwo.out = grad + L.off_wo;
    pwo.ldo = bott;
    have_wo = true;
    nl += 3;
  } else {
  {
    GemmBatch gb;
    memset(&gb, 0, sizeof(gb));
    gb.nprob = 1;
    GemmProblem& p = gb.p[0];
    TRY(gemm_problem(&p, h->z, bott, 0, h->snap + L.off_wo, bott, 0, N, C, bott));
    p.epi = EPI_CE_GRAD;
    p.bias = bias_o;
    p.labels = h->lab;
    p.lse = h->lse;
    p.out = h->dlogits;
    p.ldo = C;
    p.scale = 1.0f / (h->grad_frames > 0.f ? h->grad_frames : (float)N);
    p.colpart = h->biaspart;
    if (blocked_dlogits(h))  // 64x64 blocks: the two readers below fetch contiguous 8 KB boxes
      TRY(gemm_blocked_output(&p, N, C));
    else
      TRY(gemm_bf16_output(&p));
    MARK(PH_GEMM);
    TRY(gemm_launch(&gb, s));
    MARK(PH_OTHER);
    TRY(op_rowsum(h->biaspart, ((N + kGemmBM - 1) / kGemmBM) * 4, C, grad + L.off_bo, s));
    nl += 2;
    MARK(PH_GEMM);
  }
  {
    GemmBatch gb;
    memset(&gb, 0, sizeof(gb));
    gb.nprob = 2;
    GemmProblem& p0 = gb.p[0];  // dW_o = dlogits^T Z
    TRY(gemm_problem(&p0, h->dlogits, C, 1, h->z, bott, 1, C, bott, N));
    if (blocked_dlogits(h)) TRY(gemm_blocked_a(&p0, h->dlogits, N, C));
    p0.epi = EPI_F32;
    p0.out = grad + L.off_wo;
    p0.ldo = bott;
    GemmProblem& p1 = gb.p[1];  // dZ = dlogits W_o (split-K, fp32 partials)
    TRY(gemm_problem(&p1, h->dlogits, C, 0, h->snap + L.off_wo, bott, 1, N, bott, C));
    if (blocked_dlogits(h)) TRY(gemm_blocked_a(&p1, h->dlogits, N, C));
    const int S = dz_split(C);
    if (S > 1) {
      p1.epi = EPI_F32;
      p1.out = h->splitk;
      p1.ldo = bott;
      p1.ksplit = S;
      p1.split_stride = (long long)N * bott;
      // longest tiles first: dZ split tiles lead the persistent schedule
      GemmProblem tmp = gb.p[0];
      gb.p[0] = gb.p[1];
      gb.p[1] = tmp;
    } else {
      p1.epi = EPI_BF16;
      p1.out = h->dz;
      p1.ldo = bott;
    }
    TRY(gemm_launch(&gb, s));
    if (S > 1) TRY(op_splitk_bf16(h->splitk, S, (int64_t)N * bott, h->dz, s));
    nl += S > 1 ? 2 : 1;
  }
  }
  {
    GemmBatch gb;
    memset(&gb, 0, sizeof(gb));
    const int q0 = have_wo ? 1 : 0;
    if (have_wo) gb.p[0] = pwo;
    gb.nprob = q0 + 2;
    const bool out_side = ovl && have_wo;  // dW_o + dW_b beside BPTT_{L-1}, dY alone here
    GemmProblem& p0 = gb.p[q0];  // dW_b = dZ^T Y (alone: split-K fp32 partials, reduced below in split order)
    TRY(gemm_problem(&p0, h->dz, bott, 1, Y(Lh - 1), kLayerOut, 1, bott, kLayerOut, N));
    p0.epi = EPI_F32;
    const int Sb = have_wo ? 1 : ksplit_for(N, kWbSplit);
    p0.out = Sb > 1 ? h->splitk : grad + L.off_wb;
    p0.ldo = kLayerOut;
    p0.ksplit = Sb;
    p0.split_stride = (long long)bott * kLayerOut;
    GemmProblem& p1 = gb.p[q0 + 1];  // dY = dZ W_b
    TRY(gemm_problem(&p1, h->dz, bott, 0, h->snap + L.off_wb, kLayerOut, 1, N, kLayerOut, bott));
    p1.epi = EPI_BF16;
    p1.out = h->dy;
    p1.ldo = kLayerOut;
    TRY(gemm_bf16_output(&p1));
    MARK(PH_GEMM);
    if (out_side) {
      GemmBatch gy;
      memset(&gy, 0, sizeof(gy));
      gy.nprob = 1;
      gy.p[0] = p1;
      gy.prio = h->prio_hi;
      gb.nprob = q0 + 1;
      // dW_o streams the 344 MB dlogits: beyond ~24 pairs its HBM traffic slows the BPTT it hides behind
      static const int wo_pairs = getenv("DS_WO_PAIRS") ? atoi(getenv("DS_WO_PAIRS")) : 24;
      gb.max_pairs = wo_pairs > 0 && wo_pairs < dw_pairs - dxp ? wo_pairs : dw_pairs - dxp;
      gb.prio = h->prio_lo;
      DS_CUDA_TRY(cudaEventRecord(h->ev_aux[3], s));
      TRY(gemm_launch(&gy, s));
      TL("dY", s);
      DS_CUDA_TRY(cudaStreamWaitEvent(h->side3, h->ev_aux[3], 0));
      TRY(lstm_wait_started(seq_words(h), 0, flag, h->side3));
      TRY(gemm_launch(&gb, h->side3));
      TL("dWo", h->side3);
      nl += 2;
    } else {
      TRY(gemm_launch(&gb, s));
    }
    MARK(PH_OTHER);
    if (Sb > 1) TRY(op_splitk_f32(h->splitk, Sb, (int64_t)bott * kLayerOut, grad + L.off_wb, s));
    if (aux_join) {  // db_b (column sums of dZ) on the side stream too; the output SGD follows it there
      DS_CUDA_TRY(cudaEventRecord(h->ev_aux[2], s));
      DS_CUDA_TRY(cudaStreamWaitEvent(h->side, h->ev_aux[2], 0));
      TRY(op_colsum(h->dz, N, bott, bott, h->colpart, grad + L.off_bb, h->side));
      // (biaspart is read there: the first BPTT writing it waits below)
    } else {
      TRY(op_colsum(h->dz, N, bott, bott, h->colpart, grad + L.off_bb, s));
    }
    nl += Sb > 1 ? 4 : 3;
    // bottleneck + output layer gradients are final: update them beside BPTT_{L-1}
    TRY(sgd_segment(h, sg, grad, flag, L.off_wb, L.total - L.off_wb, true, out_side ? h->side3 : s));
    if (out_side) {
      DS_CUDA_TRY(cudaEventRecord(h->ev_dw[0][1], h->side3));
      out_side_done = true;
    }
  }
  // Weight gradients beside the recurrence: with the narrow (64-CTA) BPTT, layer l's dW_ih / dW_hh
  // GEMMs run on the SMs BPTT_{l-1} leaves free (low-priority stream, grid capped to those SMs) and
  // only dX = dG W_ih stays between two BPTTs.  dG alternates between two buffers by layer parity.
  for (int l = Lh - 1; l >= 0; --l) {
    // overlap: dG and the bias partials alternate between two buffers by layer parity; the waits for
    // their readers (dW_{l+2}, row sums of l+2) sit before dX_{l+1}, so BPTT_l follows dX_{l+1}
    // directly (programmatic launch: its W_hh^T setup overlaps dX on the SMs dX leaves free)
    const int buf = ovl ? l % 3 : 0;
    __nv_bfloat16* dgl = buf == 0 ? h->dg : buf == 1 ? h->dg2 : h->dg3;
    float* bpl = buf == 0 ? h->biaspart : buf == 1 ? h->biaspart2 : h->biaspart3;
    if (aux_join && buf == 0) {  // the output layer's bias row sums (side stream) have read biaspart
      DS_CUDA_TRY(cudaStreamWaitEvent(s, h->ev_aux[1], 0));
      aux_join = false;
    }
    if (xstream && l == Lh - 1) DS_CUDA_TRY(cudaStreamWaitEvent(s, h->ev_gz[1], 0));  // counters zeroed
    const bool dy_streamed = xstream && l + 1 < Lh;  // dY = the two halves of dX_{l+1}
    LstmLayerArgs la{B, T, h->gates[l], h->cstate[l], h->yfull[l], h->snap + L.off_whh[l],
                     dy_streamed ? h->dyx[(l + 1) & 1][0] : h->dy, dgl, h->counters,
                     l == g_bptt_layer ? g_bptt_trace : nullptr, bpl};
    la.err = flag;
    if (ovl) {
      la.prio = h->prio_hi;
      la.seq = seq_words(h);
      la.tag = Lh - 1 - l;
      if (xstream) {
        la.gate = gate_words(h, l);
        if (dy_streamed) {  // still streaming: frame by frame
          la.dy2 = h->dyx[(l + 1) & 1][1];
          la.dyready = ready_words(h, l);
          la.dyready_target = (uint32_t)((B / 32) * (kHidden / 64));
        }
      }
    }
    TL("pre-bptt" + std::to_string(l), s);
    MARK(PH_LSTM_BWD);
    TRY(lstm_backward(la, s));
    TL("bptt" + std::to_string(l), s);
    nl += 1 + (B - 1) / (128 * lstm_max_tiles());
    GemmBatch gb;
    memset(&gb, 0, sizeof(gb));
    gb.b_early = 1;  // B = X / Y / W_ih (forward pass, snapshot); the predecessor (BPTT l) writes only A = dG
    GemmProblem& p0 = gb.p[0];  // dW_ih = dG^T X
    if (l == 0) {
      TRY(gemm_problem(&p0, dgl, kGates2, 1, h->x0, kInPad, 1, kGates2, kInPad, N));
      p0.n_valid = L.input_dim;
      p0.ldo = L.input_dim;
    } else {
      TRY(gemm_problem(&p0, dgl, kGates2, 1, Y(l - 1), kLayerOut, 1, kGates2, kLayerOut, N));
      p0.ldo = kLayerOut;
    }
    p0.epi = EPI_F32;
    p0.out = grad + L.off_wih[l];
    for (int d = 0; d < 2; ++d) {  // dW_hh[dir] = dG_dir^T H_prev_dir
      GemmProblem& p = gb.p[1 + d];
      const __nv_bfloat16* hp = d == 0 ? h->yfull[l] : h->yfull[l] + (size_t)2 * B * kLayerOut + kHidden;
      TRY(gemm_problem(&p, dgl + d * kGates, kGates2, 1, hp, kLayerOut, 1, kGates, kHidden, N));
      p.epi = EPI_F32;
      p.out = grad + L.off_whh[l] + (size_t)d * kGates * kHidden;
      p.ldo = kHidden;
    }
    gb.nprob = 3;
    GemmBatch gx;  // dY_{l-1} = dG W_ih (the critical path)
    memset(&gx, 0, sizeof(gx));
    if (l > 0) {
      GemmBatch& gt = ovl ? gx : gb;
      GemmProblem& p3 = gt.p[gt.nprob];
      TRY(gemm_problem(&p3, dgl, kGates2, 0, h->snap + L.off_wih[l], kLayerOut, 1, N, kLayerOut, kGates2));
      p3.epi = EPI_BF16;
      p3.out = h->dy;
      p3.ldo = kLayerOut;
      TRY(gemm_bf16_output(&p3));
      ++gt.nprob;
      gx.b_early = 1;
    }
    // db = row sums of the BPTT's bias partials: off the critical path, beside the GEMMs; joined
    // before the layer's update and before BPTT_{l-1} reuses biaspart
    const bool rs_side = !h->profile;
    MARK(PH_OTHER);
    if (rs_side) {
      DS_CUDA_TRY(cudaEventRecord(h->ev_rs[l][0], s));
      DS_CUDA_TRY(cudaStreamWaitEvent(h->side2, h->ev_rs[l][0], 0));
    }
    TRY(op_rowsum(bpl, ((B + 127) / 128) * 4, kGates2, grad + L.off_b[l], rs_side ? h->side2 : s));
    if (rs_side) DS_CUDA_TRY(cudaEventRecord(h->ev_rs[l][1], h->side2));
    MARK(PH_GEMM);
    if (ovl && l > 0) {
      DS_CUDA_TRY(cudaEventRecord(h->ev_dw[l][0], s));
      if (xstream) {
        // dX_l = dG_l W_ih_l behind BPTT_l on side4 as two problems, one per BPTT direction (K = its
        // 2048 gate columns, rows gated on that direction's per-step counters, units list-scheduled in
        // completion order), into dy / dy2; every stored block is counted per (frame, unit direction,
        // half) and BPTT_{l-1} sums the halves frame by frame as they land
        GemmBatch gd;
        memset(&gd, 0, sizeof(gd));
        gd.nprob = 2;
        for (int d = 0; d < 2; ++d) {  // dY_d = dG[:, dir d] W_ih[dir d rows]: K = one direction's 2048 gates
          GemmProblem& px = gd.p[d];
          TRY(gemm_problem(&px, dgl + (size_t)d * kGates, kGates2, 0, h->snap + L.off_wih[l] + (size_t)d * kGates * kLayerOut,
                           kLayerOut, 1, N, kLayerOut, kGates));
          px.epi = EPI_BF16;
          px.out = h->dyx[l & 1][d];
          px.ldo = kLayerOut;
          TRY(gemm_bf16_output(&px));
          px.gate = gate_words(h, l) + (size_t)d * T;
          px.gate_target = (uint32_t)lstm_bwd_gate_target(B);
          px.gate_rows = B;
          px.gate_T = T;
          px.gate_err = flag;
          px.ready = ready_words(h, l - 1) + d;
          px.ready_rows = B;
          px.ready_cols = kHidden;
          px.ready_stride = 2;
        }
        TRY(dx_schedule(gd, dxp, B, T));
        gd.prio = h->prio_hi;
        gd.trace = gemm_layer_trace(l);
        gd.trace_keep = gd.trace != nullptr;
        TRY(lstm_wait_started(seq_words(h), Lh - 1 - l, flag, h->side4));  // BPTT_l holds its SMs
        TRY(gemm_launch(&gd, h->side4));
        TL("dX" + std::to_string(l), h->side4);
        DS_CUDA_TRY(cudaEventRecord(h->ev_x[l], h->side4));
        nl += 2;
      }
      DS_CUDA_TRY(cudaStreamWaitEvent(h->side3, h->ev_dw[l][0], 0));
      // beside BPTT_0 no dX runs: layer 1's weight gradients take its pairs too (its update then runs
      // beside BPTT_0 instead of competing with the layer-0 gradients after it); the early layer-0
      // gradients follow on the pairs it frees
      static const bool dw1_all = !getenv("DS_DW1_ALL") || getenv("DS_DW1_ALL")[0] != '0';
      gb.max_pairs = (l == 1 && dw1_all) ? dw_pairs : dw_pairs - dxp;
      gb.prio = h->prio_lo;
      gb.b_early = 0;  // its stream predecessor is the previous layer's dW, not BPTT_l
      // dW_l only once BPTT_{l-1} holds its SMs (dX_l runs alone on the machine first)
      TRY(lstm_wait_started(seq_words(h), Lh - l, flag, h->side3));
      TRY(gemm_launch(&gb, h->side3));
      TL("dW" + std::to_string(l), h->side3);
      if (l + 2 < Lh) {  // BPTT_{l-1} overwrites the dG / bias-partial buffers of layer l+2
        DS_CUDA_TRY(cudaStreamWaitEvent(s, h->ev_dw[l + 2][1], 0));
        DS_CUDA_TRY(cudaStreamWaitEvent(s, h->ev_rs[l + 2][1], 0));
        if (xstream) DS_CUDA_TRY(cudaStreamWaitEvent(s, h->ev_x[l + 2], 0));
      }
      if (!xstream) {
        gx.max_pairs = dw_pairs;  // same two tile waves; the next BPTT's CTAs set up beside it
        TRY(gemm_launch(&gx, s));
        TL("dX" + std::to_string(l), s);
      }
      DS_CUDA_TRY(cudaStreamWaitEvent(h->side3, h->ev_rs[l][1], 0));
      // layer l's update rewrites the W_ih snapshot dX_l reads: after it (dX_l ends long before dW_l)
      if (xstream) DS_CUDA_TRY(cudaStreamWaitEvent(h->side3, h->ev_x[l], 0));
      DS_CUDA_TRY(cudaEventRecord(h->ev_dw[l][1], h->side3));
      nl += 3;
      // layer l's gradients are final once dW_l is: update them beside BPTT_{l-1}
      TRY(sgd_segment(h, sg, grad, flag, L.off_wih[l], L.off_b[l] + kGates2 - L.off_wih[l], true, h->side3));
      continue;
    }
    const int E = dw0_early();
    if (xstream && l == 0 && E > 0 && E < T) {
      // layer 0 (no dX): the frames BPTT_0 completes first (direction 0 from t = T-1 down, direction 1
      // from t = 0 up) go into its weight gradients beside it, on the pairs dX left, once E frames of
      // each direction are final; the rest after it, accumulated onto them (early + late, fixed order)
      GemmBatch ge, gl;
      memset(&ge, 0, sizeof(ge));
      memset(&gl, 0, sizeof(gl));
      // fused step: the late part goes to scratch (plain stores) and the layer-0 update sums it in
      // (a streaming pass), instead of an accumulate epilogue re-reading the early part row by row
      const bool late_scratch = sg.theta && !sg.grp && sg.mirror;
      const int64_t w0 = L.off_b[0] - L.off_wih[0];  // W_ih0 + W_hh0
      for (int part = 0; part < 2; ++part) {
        GemmBatch& g = part ? gl : ge;
        for (int d = 0; d < 2; ++d) {
          // frames: early dir 0 [T-E, T), dir 1 [0, E); late dir 0 [0, T-E), dir 1 [E, T)
          const int nf = part == 0 ? E : T - E;
          const int r0 = (d == 0 ? (part == 0 ? T - E : 0) : (part == 0 ? 0 : E)) * B;
          GemmProblem& pi = g.p[g.nprob++];  // dW_ih0 rows of direction d = dG[:, dir d]^T X0
          TRY(gemm_problem(&pi, dgl + (size_t)r0 * kGates2 + (size_t)d * kGates, kGates2, 1, h->x0 + (size_t)r0 * kInPad,
                           kInPad, 1, kGates, kInPad, nf * B));
          pi.n_valid = L.input_dim;
          pi.ldo = L.input_dim;
          pi.epi = EPI_F32;
          pi.out = grad + L.off_wih[0] + (size_t)d * kGates * L.input_dim;
          pi.accumulate = part;
          if (part && late_scratch) {
            pi.out = h->splitk + (size_t)d * kGates * L.input_dim;
            pi.accumulate = 0;
          }
          GemmProblem& ph = g.p[g.nprob++];  // dW_hh0[d] = dG[:, dir d]^T H_prev[d]
          const __nv_bfloat16* hp = d == 0 ? h->yfull[0] : h->yfull[0] + (size_t)2 * B * kLayerOut + kHidden;
          TRY(gemm_problem(&ph, dgl + (size_t)r0 * kGates2 + (size_t)d * kGates, kGates2, 1, hp + (size_t)r0 * kLayerOut,
                           kLayerOut, 1, kGates, kHidden, nf * B));
          ph.epi = EPI_F32;
          ph.out = grad + L.off_whh[0] + (size_t)d * kGates * kHidden;
          ph.ldo = kHidden;
          ph.accumulate = part;
          if (part && late_scratch) {
            ph.out = h->splitk + (L.off_whh[0] - L.off_wih[0]) + (size_t)d * kGates * kHidden;
            ph.accumulate = 0;
          }
        }
      }
      const uint32_t* g0 = gate_words(h, 0);
      TRY(lstm_wait_counters(g0 + (T - E), g0 + T + (E - 1), (uint32_t)lstm_bwd_gate_target(B), flag, h->side4));
      ge.max_pairs = dxp;
      ge.prio = h->prio_hi;
      TRY(gemm_launch(&ge, h->side4));
      TL("dW0-early", h->side4);
      DS_CUDA_TRY(cudaEventRecord(h->ev_x[0], h->side4));
      // into scratch the late part does not depend on the early one: only the update joins them
      if (!late_scratch) DS_CUDA_TRY(cudaStreamWaitEvent(s, h->ev_x[0], 0));
      gl.trace = gemm_layer_trace(0);  // tools/dx_trace.py 0 traces this late part
      gl.trace_keep = gl.trace != nullptr;
      TRY(gemm_launch(&gl, s));
      if (late_scratch) {
        DS_CUDA_TRY(cudaStreamWaitEvent(s, h->ev_x[0], 0));
        sg.add0 = h->splitk;
        sg.add0_n = w0;
      }
      nl += 3;
    } else {
      TRY(gemm_launch(&gb, s));
    }
    TL("grp" + std::to_string(l), s);
    if (rs_side) DS_CUDA_TRY(cudaStreamWaitEvent(s, h->ev_rs[l][1], 0));
    nl += 2;
    // layer l's gradients are final: update them beside BPTT_{l-1} (layer 0 on the critical path)
    TRY(sgd_segment(h, sg, grad, flag, L.off_wih[l], L.off_b[l] + kGates2 - L.off_wih[l], l > 0, s));
    if (l == 0) TL("sgd-main", s);
  }
  if (ovl)  // every weight gradient is complete when the step ends (also without an update)
    for (int l = out_side_done ? 0 : 1; l < Lh; ++l) DS_CUDA_TRY(cudaStreamWaitEvent(s, h->ev_dw[l][1], 0));
  if (xstream && Lh > 1) DS_CUDA_TRY(cudaStreamWaitEvent(s, h->ev_x[1], 0));  // side4 joined (its last dX)
  TL("dW-joined", s);
  if (sg.theta) {
    MARK(PH_OTHER);
    for (int k = 0; k < sg.nfork; ++k) DS_CUDA_TRY(cudaStreamWaitEvent(s, h->ev_join[k], 0));
    TL("sgd-joined", s);
    if (!sg.mirror) TRY(op_snapshot_aux(sg.theta, L, h->wih0pad, h->bias_snap, s));  // else written by the updates
    nl += L.layers + (sg.mirror ? 1 : 2);
  }
  TL("end", s);
  MARK(PH_END);
#undef TL
#undef MARK
#undef TRY
  return DS_OK;
}

bool use_graphs() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DS_NO_GRAPH");
    v = (e && e[0] == '1') ? 0 : 1;
  }
  return v == 1;
}

int run_step(ds_blstm* h, const int64_t* idx, int B, float* grad, float* loss, int* flag, cudaStream_t s,
             SgdCtx sg = SgdCtx()) {
  if (B < 1 || B > h->Bmax) return fail_arg("batch size out of range 1..max_batch");
  if (!h->feats) return fail_arg("dataset not bound (ds_blstm_set_dataset)");
  if (!loss) return fail_arg("loss_sum pointer is required");
  DS_CUDA_TRY(cudaSetDevice(h->device));
  if (h->prec == 1) {  // FP32 parity: plain launch sequence, then the unfused update
    int rc = parity_step(h->par, h->L, h->T, idx, B, h->feats, h->labels, h->n_seq, h->grad_frames, grad, loss, flag,
                         s, &h->launches);
    if (rc || !sg.theta) return rc;
    rc = op_sgd_lr(sg.theta, sg.vel, grad, h->d_lr, sg.mu, h->L.total, nullptr, flag, 0, s);
    if (!rc) rc = parity_snapshot(h->par, h->L, sg.theta, s);
    h->launches += 1 + 4 * h->L.layers + 3;
    return rc;
  }
  if (h->pad_B != B) {  // zero rows of Y_full (h_{-1}, h_T): no kernel ever writes them
    for (int l = 0; l < h->L.layers; ++l) {
      DS_CUDA_TRY(cudaMemsetAsync(h->yfull[l], 0, (size_t)B * kLayerOut * 2, s));
      DS_CUDA_TRY(
          cudaMemsetAsync(h->yfull[l] + (size_t)(h->T + 1) * B * kLayerOut, 0, (size_t)B * kLayerOut * 2, s));
    }
    h->pad_B = B;
  }
  cudaStreamCaptureStatus cs;
  DS_CUDA_TRY(cudaStreamIsCapturing(s, &cs));
  if (!use_graphs() || h->profile || cs != cudaStreamCaptureStatusNone)
    return issue_step(h, idx, B, grad, loss, flag, s, sg);
  ds_blstm::Key key{B, idx, grad, loss, flag, grad != nullptr, h->grad_frames, sg.theta, sg.vel, sg.mu, sg.grp};
  for (auto& e : h->graphs)
    if (e.key == key) {
      DS_CUDA_TRY(cudaGraphLaunch(e.exec, s));
      return DS_OK;
    }
  cudaStream_t cap;
  DS_CUDA_TRY(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
  DS_CUDA_TRY(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
  int rc = issue_step(h, idx, B, grad, loss, flag, cap, sg);
  cudaGraph_t g = nullptr;
  cudaError_t ce = cudaStreamEndCapture(cap, &g);
  cudaStreamDestroy(cap);
  if (rc) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  if (ce != cudaSuccess) return fail_cuda(ce, "cudaStreamEndCapture");
  cudaGraphExec_t ex;
  ce = cudaGraphInstantiate(&ex, g, cudaGraphInstantiateFlagUseNodePriority);
  cudaGraphDestroy(g);
  if (ce != cudaSuccess) return fail_cuda(ce, "cudaGraphInstantiate");
  if (h->graphs.size() >= 16) {
    cudaGraphExecDestroy(h->graphs.front().exec);
    h->graphs.erase(h->graphs.begin());
  }
  h->graphs.push_back({key, ex});
  DS_CUDA_TRY(cudaGraphLaunch(ex, s));
  return DS_OK;
}

}  // namespace

// ===========================================================================
extern "C" {

int64_t ds_blstm_param_dim(const ds_blstm_cfg* c) {
  if (validate_cfg(c)) return -1;
  return make_layout(c->layers, c->input_dim, c->bottleneck, c->classes).total;
}

int ds_blstm_create(const ds_blstm_cfg* c, int device, ds_blstm** out) {
  int rc = validate_cfg(c);
  if (rc) return rc;
  if (!out) return fail_arg("null output handle");
  DS_CUDA_TRY(cudaSetDevice(device));
  ds_blstm* h = new ds_blstm();
  h->cfg = *c;
  h->L = make_layout(c->layers, c->input_dim, c->bottleneck, c->classes);
  h->device = device;
  h->T = c->frames;
  h->Bmax = c->max_batch;
  h->Nmax = (int64_t)c->frames * c->max_batch;
  h->ntiles_c = (c->classes + kGemmBN - 1) / kGemmBN;
  size_t total = 0;
  carve(h, nullptr, &total);
  cudaError_t e = cudaMalloc(&h->arena, total);
  if (e != cudaSuccess) {
    delete h;
    return fail_cuda(e, "cudaMalloc(workspace)");
  }
  carve(h, reinterpret_cast<char*>(h->arena), &total);
  // recurrent-kernel flags count up across launches: zero once
  e = cudaMemset(h->counters, 0, sizeof(uint32_t) * counter_words_total(h));
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking);
  for (int k = 0; k < kMaxLayers + 2 && e == cudaSuccess; ++k) {
    e = cudaEventCreateWithFlags(&h->ev_fork[k], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_join[k], cudaEventDisableTiming);
  }
  for (int k = 0; k < 4 && e == cudaSuccess; ++k) e = cudaEventCreateWithFlags(&h->ev_aux[k], cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->side2, cudaStreamNonBlocking);
  for (int k = 0; k < kMaxLayers * 2 && e == cudaSuccess; ++k)
    e = cudaEventCreateWithFlags(&h->ev_rs[k / 2][k % 2], cudaEventDisableTiming);
  if (e == cudaSuccess && use_timeline()) e = cudaMalloc(&h->tl_buf, 256 * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaDeviceGetStreamPriorityRange(&h->prio_lo, &h->prio_hi);
  if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&h->side3, cudaStreamNonBlocking, h->prio_lo);
  if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&h->side4, cudaStreamNonBlocking, h->prio_hi);
  for (int k = 0; k < kMaxLayers * 2 && e == cudaSuccess; ++k)
    e = cudaEventCreateWithFlags(&h->ev_dw[k / 2][k % 2], cudaEventDisableTiming);
  for (int k = 0; k < kMaxLayers && e == cudaSuccess; ++k) e = cudaEventCreateWithFlags(&h->ev_x[k], cudaEventDisableTiming);
  for (int k = 0; k < 2 && e == cudaSuccess; ++k) e = cudaEventCreateWithFlags(&h->ev_gz[k], cudaEventDisableTiming);
  if (e != cudaSuccess) {
    cudaFree(h->arena);
    delete h;
    return fail_cuda(e, "workspace init");
  }
  *out = h;
  return DS_OK;
}

int ds_blstm_destroy(ds_blstm* h) {
  if (!h) return DS_OK;
  cudaSetDevice(h->device);
  for (auto& e : h->graphs) cudaGraphExecDestroy(e.exec);
  for (int k = 0; k < kMaxLayers + 2; ++k) {
    if (h->ev_fork[k]) cudaEventDestroy(h->ev_fork[k]);
    if (h->ev_join[k]) cudaEventDestroy(h->ev_join[k]);
  }
  for (int k = 0; k < 4; ++k)
    if (h->ev_aux[k]) cudaEventDestroy(h->ev_aux[k]);
  for (int k = 0; k < kMaxLayers * 2; ++k) {
    if (h->ev_rs[k / 2][k % 2]) cudaEventDestroy(h->ev_rs[k / 2][k % 2]);
    if (h->ev_dw[k / 2][k % 2]) cudaEventDestroy(h->ev_dw[k / 2][k % 2]);
  }
  for (int k = 0; k < kMaxLayers; ++k)
    if (h->ev_x[k]) cudaEventDestroy(h->ev_x[k]);
  for (int k = 0; k < 2; ++k)
    if (h->ev_gz[k]) cudaEventDestroy(h->ev_gz[k]);
  if (h->side2) cudaStreamDestroy(h->side2);
  if (h->side3) cudaStreamDestroy(h->side3);
  if (h->side4) cudaStreamDestroy(h->side4);
  if (h->tl_buf) cudaFree(h->tl_buf);
  if (h->side) cudaStreamDestroy(h->side);
  if (h->loss_pinned) cudaFreeHost(h->loss_pinned);
  parity_destroy(h->par);
  if (h->arena) cudaFree(h->arena);
  delete h;
  return DS_OK;
}

int ds_blstm_set_dataset(ds_blstm* h, const void* feats, const int32_t* labels, int64_t n_seq) {
  if (!h || !feats || !labels || n_seq < 1) return fail_arg("bad dataset binding");
  h->feats = reinterpret_cast<const __nv_bfloat16*>(feats);
  h->labels = labels;
  h->n_seq = n_seq;
  for (auto& e : h->graphs) cudaGraphExecDestroy(e.exec);
  h->graphs.clear();
  return DS_OK;
}

int ds_blstm_cast_snapshot(ds_blstm* h, const float* theta, ds_stream_t stream) {
  if (!h || !theta) return fail_arg("null argument");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  DS_CUDA_TRY(cudaSetDevice(h->device));
  if (h->prec == 1) return parity_snapshot(h->par, h->L, theta, s);
  int rc = op_cast(theta, h->L.total, h->snap, s);
  if (rc) return rc;
  return op_snapshot_aux(theta, h->L, h->wih0pad, h->bias_snap, s);
}

int ds_blstm_set_precision(ds_blstm* h, int32_t mode) {
  if (!h) return fail_arg("null handle");
  if (mode != DS_PREC_BF16 && mode != DS_PREC_FP32) return fail_arg("precision mode must be 0 (bf16) or 1 (fp32)");
  DS_CUDA_TRY(cudaSetDevice(h->device));
  if (mode == DS_PREC_FP32 && !h->par) {
    int rc = parity_create(&h->par, h->L, h->T, h->Bmax);
    if (rc) return rc;
  }
  h->prec = mode;
  return DS_OK;
}

int32_t ds_blstm_get_precision(ds_blstm* h) { return h ? h->prec : -1; }

int ds_blstm_set_group(ds_blstm* h, const ds_group_desc* g) {
  if (!h) return fail_arg("null handle");
  for (auto& e : h->graphs) cudaGraphExecDestroy(e.exec);  // graphs bake the update path
  h->graphs.clear();
  if (!g) {
    h->grp_on = false;
    return DS_OK;
  }
  if (g->n < 1 || g->n > kMaxGroupPeers || g->me < 0 || g->me >= g->n) return fail_arg("group: bad member count / index");
  if (g->nchunks < g->n) return fail_arg("group: chunk_count must be >= members");
  if (!g->own_flags || !g->pair_epochs || !g->err) return fail_arg("group: null flag / epoch / error buffer");
  GroupSync gs;
  gs.n = g->n;
  gs.me = g->me;
  gs.my_rank = g->my_rank;
  gs.nchunks = g->nchunks;
  gs.divisor = g->divisor;
  gs.max_blocks = g->max_blocks > 0 ? g->max_blocks : 64;
  for (int m = 0; m < g->n; ++m) {
    if (!g->thetas[m] || !g->grads[m] || !g->snaps[m] || !g->flags[m] || g->ranks[m] < 0 || g->ranks[m] >= 64)
      return fail_arg("group: null member buffer");
    if ((reinterpret_cast<uintptr_t>(g->thetas[m]) | reinterpret_cast<uintptr_t>(g->grads[m])) & 15)
      return fail_arg("group: buffers must be 16-byte aligned");
    gs.ranks[m] = g->ranks[m];
    gs.thetas[m] = g->thetas[m];
    gs.grads[m] = g->grads[m];
    gs.snaps[m] = g->snaps[m];
    gs.flags[m] = g->flags[m];
  }
  gs.own_flags = g->own_flags;
  gs.pair_epochs = g->pair_epochs;
  gs.err = g->err;
  gs.timeout_s = g->timeout_s;
  h->grp = gs;
  h->grp_on = true;
  return DS_OK;
}

int ds_blstm_snapshot_aux(ds_blstm* h, const float* theta, ds_stream_t stream) {
  if (!h || !theta) return fail_arg("null argument");
  DS_CUDA_TRY(cudaSetDevice(h->device));
  return op_snapshot_aux(theta, h->L, h->wih0pad, h->bias_snap, reinterpret_cast<cudaStream_t>(stream));
}

void* ds_blstm_snapshot_ptr(ds_blstm* h) { return h ? h->snap : nullptr; }

int ds_blstm_fwd_bwd(ds_blstm* h, const int64_t* idx, int32_t B, float* grad, float* loss_sum, int32_t* nonfinite,
                     ds_stream_t stream) {
  if (!h || !idx || !grad) return fail_arg("null argument");
  return run_step(h, idx, B, grad, loss_sum, nonfinite, reinterpret_cast<cudaStream_t>(stream));
}

int ds_blstm_train_step(ds_blstm* h, const int64_t* idx, int32_t B, float* theta, float* vel, float* grad, float lr,
                        float mu, float* loss_sum, int32_t* nonfinite, ds_stream_t stream) {
  if (!h || !idx || !grad || !theta || !vel) return fail_arg("null argument");
  if (!(lr > 0.f)) return fail_arg("learning rate must be > 0");
  if (((reinterpret_cast<uintptr_t>(theta) | reinterpret_cast<uintptr_t>(vel) | reinterpret_cast<uintptr_t>(grad)) &
       15))
    return fail_arg("sgd: buffers must be 16-byte aligned");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  DS_CUDA_TRY(cudaSetDevice(h->device));
  // pageable source: staged by the driver before the call returns.  Only when the rate
  // changes (schedules change it per epoch): a copy-engine node ahead of every step's graph
  // costs several microseconds of device time
  if (lr != h->lr_host) {
    DS_CUDA_TRY(cudaMemcpyAsync(h->d_lr, &lr, sizeof(float), cudaMemcpyHostToDevice, s));
    h->lr_host = lr;
  }
  SgdCtx sg;
  sg.theta = theta;
  sg.vel = vel;
  sg.mu = mu;
  if (h->grp_on) {
    if (h->prec != 0) return fail_arg("the fused SSGD group step runs in BF16 mode only");
    if (h->grp.thetas[h->grp.me] != theta || h->grp.grads[h->grp.me] != grad)
      return fail_arg("group step: theta / grad differ from this member's buffers in the group");
    sg.grp = &h->grp;
  }
  sg.mirror = !sg.grp && mirror_ok(h) && !getenv("DS_NO_SGD_MIRROR");
  return run_step(h, idx, B, grad, loss_sum, nonfinite, s, sg);
}

int ds_blstm_loss(ds_blstm* h, const int64_t* idx, int32_t B, float* loss_sum, int32_t* nonfinite,
                  ds_stream_t stream) {
  if (!h || !idx) return fail_arg("null argument");
  return run_step(h, idx, B, nullptr, loss_sum, nonfinite, reinterpret_cast<cudaStream_t>(stream));
}

int ds_sgd_momentum(float* theta, float* v, const float* g, float lr, float mu, int64_t n, ds_blstm* snap_owner,
                    int32_t* nonfinite, ds_stream_t stream) {
  if (!theta || !v || !g || n < 0) return fail_arg("null argument");
  if (!(lr > 0.f)) return fail_arg("learning rate must be > 0");
  if (snap_owner && snap_owner->L.total != n) return fail_arg("snapshot owner has a different param_dim");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (snap_owner && snap_owner->prec == 1) {  // FP32 parity snapshot: hi/lo splits of the new theta
    int rc = op_sgd(theta, v, g, lr, mu, n, nullptr, nonfinite, s);
    return rc ? rc : parity_snapshot(snap_owner->par, snap_owner->L, theta, s);
  }
  int rc = op_sgd(theta, v, g, lr, mu, n, snap_owner ? snap_owner->snap : nullptr, nonfinite, s);
  if (rc || !snap_owner) return rc;
  return op_snapshot_aux(theta, snap_owner->L, snap_owner->wih0pad, snap_owner->bias_snap, s);
}

int ds_adpsgd_mix(float* a, float* b, int64_t n, ds_stream_t stream) {
  if (!a || !b || n < 0) return fail_arg("null argument");
  return op_mix(a, b, n, reinterpret_cast<cudaStream_t>(stream));
}

int ds_group_reduce(int32_t world, int32_t rank, float* const* grads, float* const* thetas, float* const* vels,
                    ds_blstm* const* snap_owners, int64_t n, int32_t nchunks, float lr, float mu, int32_t mode,
                    float divisor, ds_stream_t stream) {
  if (!thetas || n < 1) return fail_arg("null argument");
  if (rank < 0 || rank >= world) return fail_arg("rank out of range");
  if (mode != 0 && mode != 1) return fail_arg("mode must be 0 (sgd) or 1 (average)");
  if (mode == 0 && !(lr > 0.f)) return fail_arg("learning rate must be > 0");
  __nv_bfloat16* snaps[kMaxGroup] = {};
  bool any = false;
  if (snap_owners)
    for (int r = 0; r < world && r < kMaxGroup; ++r)
      if (snap_owners[r]) {
        snaps[r] = snap_owners[r]->snap;
        any = true;
      }
  return op_group_reduce(world, rank, grads, thetas, vels, any ? snaps : nullptr, n, nchunks, lr, mu, mode, divisor,
                         reinterpret_cast<cudaStream_t>(stream));
}

int ds_average(int32_t n, float* const* srcs, float* out, int64_t dim, ds_stream_t stream) {
  if (!srcs || !out || dim < 1) return fail_arg("null argument");
  return op_average(n, srcs, out, dim, reinterpret_cast<cudaStream_t>(stream));
}

int ds_blstm_set_grad_scale(ds_blstm* h, float frames_total) {
  if (!h) return fail_arg("null handle");
  if (frames_total < 0.f) return fail_arg("frames_total must be >= 0");
  h->grad_frames = frames_total;
  return DS_OK;
}

int ds_blstm_read_loss(ds_blstm* h, const float* loss_sum_dev, ds_stream_t stream, float* out) {
  if (!h || !loss_sum_dev || !out) return fail_arg("null argument");
  DS_CUDA_TRY(cudaSetDevice(h->device));
  if (!h->loss_pinned) DS_CUDA_TRY(cudaMallocHost(&h->loss_pinned, sizeof(float)));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  DS_CUDA_TRY(cudaMemcpyAsync(h->loss_pinned, loss_sum_dev, sizeof(float), cudaMemcpyDeviceToHost, s));
  DS_CUDA_TRY(cudaStreamSynchronize(s));
  *out = *h->loss_pinned;
  return DS_OK;
}

int ds_blstm_set_profile(ds_blstm* h, int32_t enable) {
  if (!h) return fail_arg("null handle");
  h->profile = enable ? 1 : 0;
  return DS_OK;
}

int ds_blstm_profile_read(ds_blstm* h, float* ms_by_kind, int32_t nkinds) {
  if (!h || !ms_by_kind) return fail_arg("null argument");
  for (int k = 0; k < nkinds; ++k) ms_by_kind[k] = 0.f;
  DS_CUDA_TRY(cudaSetDevice(h->device));
  if (!h->ev.empty()) DS_CUDA_TRY(cudaEventSynchronize(h->ev.back()));
  for (size_t i = 0; i + 1 < h->ev.size(); ++i) {
    float ms = 0.f;
    DS_CUDA_TRY(cudaEventElapsedTime(&ms, h->ev[i], h->ev[i + 1]));
    int k = h->ev_kind[i];
    if (k >= 0 && k < nkinds) ms_by_kind[k] += ms;
  }
  for (auto e : h->ev) cudaEventDestroy(e);
  h->ev.clear();
  h->ev_kind.clear();
  return DS_OK;
}

int32_t ds_blstm_kernel_count(ds_blstm* h) { return h ? h->launches : -1; }

int ds_blstm_profile_list(ds_blstm* h, float* ms, int32_t* kinds, int32_t max_n, int32_t* n_out) {
  if (!h || !ms || !kinds || !n_out) return fail_arg("null argument");
  DS_CUDA_TRY(cudaSetDevice(h->device));
  if (!h->ev.empty()) DS_CUDA_TRY(cudaEventSynchronize(h->ev.back()));
  int n = 0;
  for (size_t i = 0; i + 1 < h->ev.size() && n < max_n; ++i, ++n) {
    DS_CUDA_TRY(cudaEventElapsedTime(&ms[n], h->ev[i], h->ev[i + 1]));
    kinds[n] = h->ev_kind[i];
  }
  *n_out = n;
  return DS_OK;
}

// debug: "name ms" lines of the last step's timeline (DS_TIMELINE=1), relative to its start
int ds_debug_timeline(ds_blstm* h, char* buf, int32_t len) {
  if (!h || !buf || len < 1) return fail_arg("ds_debug_timeline: bad arguments");
  DS_CUDA_TRY(cudaDeviceSynchronize());
  std::string out;
  std::vector<unsigned long long> t(h->tl_n > 0 ? h->tl_n : 1);
  if (h->tl_n > 0)
    DS_CUDA_TRY(cudaMemcpy(t.data(), h->tl_buf, sizeof(unsigned long long) * h->tl_n, cudaMemcpyDeviceToHost));
  for (int i = 0; i < h->tl_n; ++i) out += h->tl_name[i] + " " + std::to_string((double)(t[i] - t[0]) * 1e-6) + "\n";
  if (h->tl_n > 0) out += "base_ns " + std::to_string(t[0]) + "\n";  // absolute globaltimer of "start"
  snprintf(buf, (size_t)len, "%s", out.c_str());
  return DS_OK;
}

int ds_debug_bptt_trace(void* buf, int32_t layer) {
  g_bptt_trace = static_cast<uint64_t*>(buf);
  g_bptt_layer = buf ? layer : -1;
  return DS_OK;
}

int ds_debug_gemm_trace(void* buf, int32_t launch) {
  if (launch == -1) {  // the fused soft-max/dZ kernel instead (every launch while set)
    ce_grad_dz_set_trace(static_cast<unsigned long long*>(buf));
    return DS_OK;
  }
  if (buf && launch < 0 && launch > -2 - kMaxLayers)  // -2 - l: the streamed dX of layer l (graph capture)
    return gemm_set_trace(static_cast<unsigned long long*>(buf), launch), DS_OK;
  if (buf && launch < 0) return fail_arg("launch index must be >= 0 (or -1: soft-max/dZ kernel, -2-l: dX of layer l)");
  gemm_set_trace(static_cast<unsigned long long*>(buf), launch);
  return DS_OK;
}

int ds_debug_gemm_bf16(const void* A, int64_t lda, int32_t a_mn, const void* B, int64_t ldb, int32_t b_mn, float* C,
                       int64_t ldc, int32_t M, int32_t N, int32_t K, ds_stream_t stream) {
  GemmBatch gb;
  memset(&gb, 0, sizeof(gb));
  gb.nprob = 1;
  int rc = gemm_problem(&gb.p[0], A, lda, a_mn, B, ldb, b_mn, M, N, K);
  if (rc) return rc;
  gb.p[0].epi = EPI_F32;
  gb.p[0].out = C;
  gb.p[0].ldo = ldc;
  return gemm_launch(&gb, reinterpret_cast<cudaStream_t>(stream));
}

int ds_debug_lstm_fwd(int32_t B, int32_t T, void* gates, float* cstate, void* y_full, const void* whh,
                      uint32_t* counters, uint64_t* trace, ds_stream_t stream) {
  LstmLayerArgs a{B, T, reinterpret_cast<__nv_bfloat16*>(gates), cstate, reinterpret_cast<__nv_bfloat16*>(y_full),
                  reinterpret_cast<const __nv_bfloat16*>(whh), nullptr, nullptr, counters, trace};
  return lstm_forward(a, reinterpret_cast<cudaStream_t>(stream));
}

int ds_debug_lstm_bwd(int32_t B, int32_t T, const void* gates, const float* cstate, const void* whh, const void* dy,
                      void* dg, uint32_t* counters, uint64_t* trace, ds_stream_t stream) {
  LstmLayerArgs a{B,
                  T,
                  const_cast<__nv_bfloat16*>(reinterpret_cast<const __nv_bfloat16*>(gates)),
                  const_cast<float*>(cstate),
                  nullptr,
                  reinterpret_cast<const __nv_bfloat16*>(whh),
                  reinterpret_cast<const __nv_bfloat16*>(dy),
                  reinterpret_cast<__nv_bfloat16*>(dg),
                  counters,
                  trace};
  return lstm_backward(a, reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
