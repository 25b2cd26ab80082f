// p2p.h — the peer group of the fused SSGD training step (blstm.cu):
// per-layer device barrier + sharded canonical-order reduce / SGD /
// all-gather over peer-mapped buffers (kernels in p2p.cu).
#pragma once
#include <cstdint>

#include "ds_internal.h"

namespace ds {

constexpr int kMaxGroupPeers = 16;

struct GroupSync {
  int n = 0;           // members
  int me = 0;          // this learner's member index (chunk owner id)
  int my_rank = 0;     // this process's world rank (flag slot)
  int nchunks = 0;     // make_chunk_plan(param_dim, n, nchunks)
  float divisor = 0.f; // <= 0: n
  int max_blocks = 0;  // SM cap of the per-layer sync kernels
  int ranks[kMaxGroupPeers] = {};
  float* thetas[kMaxGroupPeers] = {};
  const float* grads[kMaxGroupPeers] = {};
  void* snaps[kMaxGroupPeers] = {};
  uint32_t* flags[kMaxGroupPeers] = {};
  uint32_t* own_flags = nullptr;
  uint32_t* pair_epochs = nullptr;
  int* err = nullptr;
  double timeout_s = 60.0;
};

int group_barrier(const GroupSync& g, cudaStream_t s);
// canonical-order reduce / divisor / momentum SGD of the chunks this member
// owns, clipped to [lo, hi); theta + snapshot stored into every member;
// learning rate read from lr_dev (graph replays)
int group_shard_range(const GroupSync& g, int64_t n, int64_t lo, int64_t hi, float* v_own, const float* lr_dev,
                      float mu, cudaStream_t s);

}  // namespace ds
