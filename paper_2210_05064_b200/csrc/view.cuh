// view.cuh — device-resident RolloutView (rollout.hpp:33-78): the gathered learner
// fields as one record per slot, everything else SoA.
//
// HBM layout (fp32 values, int32 indices, u8 flags; S = size, K = num_seqs):
//   rec[S*RS]: the learner record of a slot, RS = D + AW + 1 floats:
//              obs[D] | action (AW = 1: the int32 bits; continuous AW = A) | log_prob
//   ar[S*2]:   advantage, returns (written by compute_gae)
//   value reward latency [S]   done stale replayed [S] (u8)
//   env_index seq_of_slot step_in_episode [S] (i32)  episode_index version [S] (64-bit)
//   seqs[K] (ver_seq_desc, 32 B)   h0[K*H]
//   per_env_counts[N] env_bootstrap[N] env_bootstrap_valid[N]
//   env_offsets[N+1]  — exclusive scan of the per-env fresh counts, valid when
//                       `env_contiguous` (every close_rollout/backfill output)
// Capacities are sized for T*N so backfill_stale appends in place.
// The time-major minibatch gather reads exactly rec and ar: two contiguous runs
// per sequence piece instead of five scattered 4-byte fields, so short pieces
// waste far fewer partial DRAM sectors (SURVEY §7 hard part 5).
#pragma once

#include "common.cuh"

namespace verg {

struct DView {
  Ctx* ctx = nullptr;
  int T = 0, N = 0, action_kind = 0, obs_dim = 0, act_dim = 0, hidden_dim = 0;
  int size = 0, num_seqs = 0, h0_rows = 0;
  int cap = 0, seq_cap = 0, h0_cap = 0;
  int deficit = 0, stale_steps = 0, replayed_steps = 0;
  uint64_t snapshot_version = 0;
  double collect_wall_time = 0;
  // fresh slots are [0, fresh) and env-major contiguous with env_offsets
  bool env_contiguous = false;
  int fresh_prefix = 0;

  DBuf<float> rec, ar, value, reward, latency;
  DBuf<int32_t> env_index, seq_of_slot, step_in_episode;
  DBuf<uint8_t> done, stale, replayed;
  DBuf<int64_t> episode_index;
  DBuf<uint64_t> version;
  DBuf<ver_seq_desc> seqs;
  DBuf<float> h0;
  DBuf<int32_t> per_env_counts, env_offsets;
  DBuf<float> env_bootstrap;
  DBuf<uint8_t> env_bootstrap_valid;

  int act_width() const { return action_kind ? act_dim : 1; }
  int rs() const { return obs_dim + act_width() + 1; }  // record stride (floats)
  // allocate slot arrays for `cap_` slots (contents not preserved)
  void alloc_slots(int cap_);
  // grow slot arrays to cap_ keeping the first `size` slots
  void grow_slots(int cap_);
  void alloc_seqs(int seq_cap_, int h0_cap_);
  void grow_seqs(int seq_cap_, int h0_cap_);
  void alloc_env();
};

}  // namespace verg

struct ver_view_s {
  verg::DView v;
};
