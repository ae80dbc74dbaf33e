// ver_oracle.cpp — CPU double-precision restatement of the VER learner hot
// path of /root/reference/proj (C++20 + Eigen3, not buildable here: Eigen3,
// doctest and CLI11 are absent).
//
// TEST INFRASTRUCTURE ONLY: this is the checker and the timed CPU baseline.
// The product (paper_2210_05064_b200/) never links or calls it.
//
// Every function follows the cited reference lines.  Eigen is replaced by the
// small row-major `Mat` below; the reverse-mode tape is restated op by op
// (tape.cpp) so the sub-gradient conventions (inclusive clip mask, cmin tie ->
// first argument, full-size `rows` scatter) and the algorithmic structure the
// CPU baseline is timed on (O(N*S) GAE, per-timestep packed GRU, tape
// backward) are the reference's own.
#include "ver_oracle.h"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <numeric>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace vo {

// ---------------------------------------------------------------- errors
// types.hpp:41-49
struct ProtocolError : std::runtime_error {
  explicit ProtocolError(const std::string& w) : std::runtime_error(w) {}
};
struct ConfigError : std::runtime_error {
  explicit ConfigError(const std::string& w) : std::runtime_error(w) {}
};

// ---------------------------------------------------------------- matrix
// Row-major dense double matrix standing in for Eigen::MatrixXd (types.hpp:12-15).
struct Mat {
  int r = 0, c = 0;
  std::vector<double> d;
  Mat() = default;
  Mat(int rows, int cols, double fill = 0.0) : r(rows), c(cols), d((size_t)rows * cols, fill) {}
  double& operator()(int i, int j) { return d[(size_t)i * c + j]; }
  double operator()(int i, int j) const { return d[(size_t)i * c + j]; }
  size_t size() const { return d.size(); }
  bool all_finite() const {
    for (double x : d)
      if (!std::isfinite(x)) return false;
    return true;
  }
  double sum() const {
    double s = 0;
    for (double x : d) s += x;
    return s;
  }
  Mat row(int i) const {
    Mat o(1, c);
    std::memcpy(o.d.data(), &d[(size_t)i * c], sizeof(double) * c);
    return o;
  }
  Mat middle_rows(int start, int count) const {
    Mat o(count, c);
    if (count > 0) std::memcpy(o.d.data(), &d[(size_t)start * c], sizeof(double) * count * c);
    return o;
  }
  Mat transpose() const {
    Mat o(c, r);
    for (int i = 0; i < r; ++i)
      for (int j = 0; j < c; ++j) o.d[(size_t)j * r + i] = d[(size_t)i * c + j];
    return o;
  }
};

// Threading (OpenMP, vo_set_num_threads): every parallel loop below splits
// OUTPUT elements across threads and keeps each element's accumulation order
// exactly as in the serial loop, so results are bit-identical for any thread
// count (the parity tests rely on this).  Default 1 thread: the reference's
// learner thread (bench.cpp:95-205, one thread per replica).
static bool par_ok(size_t work) { return work >= (size_t)1 << 16; }
// Test-speed switch (vo_set_sparse_rows): the `rows` backward adds its slice into
// the parent's gradient directly instead of through a full-size zero matrix
// (tape.cpp:166-173).  Identical sums; the timed CPU baseline keeps it off so
// it runs the reference's O(L * S * E) scatter.
static bool g_sparse_rows = false;

// C += A * B   (A: m x k, B: k x n), blocked i-k-j; stands in for Eigen's GEMM.
static void gemm_acc(const Mat& A, const Mat& B, Mat& C) {
  const int m = A.r, k = A.c, n = B.c;
  const int KB = 128, NB = 128, RB = 16;
  const int rb = (m + RB - 1) / RB, nb = (n + NB - 1) / NB;
  // tasks = (row block, column block); each output element still sums kk ascending
#pragma omp parallel for schedule(dynamic, 1) if (par_ok((size_t)m * k * n / 64))
  for (int task = 0; task < rb * nb; ++task) {
    const int i0 = (task / nb) * RB, i1 = std::min(m, i0 + RB);
    const int n0 = (task % nb) * NB, n1 = std::min(n, n0 + NB);
    for (int k0 = 0; k0 < k; k0 += KB) {
      const int k1 = std::min(k, k0 + KB);
      for (int i = i0; i < i1; ++i) {
        double* crow = &C.d[(size_t)i * n];
        const double* arow = &A.d[(size_t)i * k];
        for (int kk = k0; kk < k1; ++kk) {
          const double a = arow[kk];
          if (a == 0.0) continue;
          const double* brow = &B.d[(size_t)kk * n];
          for (int j = n0; j < n1; ++j) crow[j] += a * brow[j];
        }
      }
    }
  }
}
static Mat matmul(const Mat& A, const Mat& B) {
  if (A.c != B.r) throw ProtocolError("oracle: matmul shape mismatch");
  Mat C(A.r, B.c);
  gemm_acc(A, B, C);
  return C;
}
// A^T * B  (A: m x k, B: m x n) -> k x n; rows i of A/B are consumed in
// ascending order for every output element (threads own output rows kk)
static Mat matmul_tn(const Mat& A, const Mat& B) {
  const int m = A.r, k = A.c, n = B.c;
  Mat C(k, n);
  const int IB = 256;
#pragma omp parallel if (par_ok((size_t)m * k * n / 64))
  for (int i0 = 0; i0 < m; i0 += IB) {
    const int i1 = std::min(m, i0 + IB);
#pragma omp for schedule(static)
    for (int kk = 0; kk < k; ++kk) {
      double* crow = &C.d[(size_t)kk * n];
      for (int i = i0; i < i1; ++i) {
        const double a = A.d[(size_t)i * k + kk];
        if (a == 0.0) continue;
        const double* brow = &B.d[(size_t)i * n];
        for (int j = 0; j < n; ++j) crow[j] += a * brow[j];
      }
    }
  }
  return C;
}
// A * B^T  (A: m x n, B: k x n) -> m x k
static Mat matmul_nt(const Mat& A, const Mat& B) { return matmul(A, B.transpose()); }

// ---------------------------------------------------------------- rng
// rng.hpp:16-75
namespace rng {
inline uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
inline uint64_t mix(uint64_t a, uint64_t b) {
  return splitmix64(a ^ (0x9e3779b97f4a7c15ull + (b << 6) + (b >> 2) + splitmix64(b)));
}
}  // namespace rng

class CounterRng {
 public:
  CounterRng() : key_(0) {}
  explicit CounterRng(uint64_t seed) : key_(rng::splitmix64(seed)) {}
  CounterRng stream(uint64_t id) const {
    CounterRng r;
    r.key_ = rng::mix(key_, id);
    return r;
  }
  uint64_t next_u64() { return rng::mix(key_, counter_++); }
  double uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double normal() {
    double u1 = uniform();
    double u2 = uniform();
    if (u1 <= 0) u1 = 0x1.0p-53;
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
  }

 private:
  uint64_t key_;
  uint64_t counter_ = 0;
};

// ---------------------------------------------------------------- types
enum class ActionKind { Discrete = 0, Continuous = 1 };

// rollout.hpp:19-28
struct SequenceDescriptor {
  int seq_id = 0;
  int env_index = 0;
  int length = 0;
  int start_offset = 0;
  int h0_index = -1;
  bool stale = false;
  int parent_start_offset = 0;
  int skip = 0;
};

// types.hpp:54-67 (Action folded in)
struct EnvStepRecord {
  int env_index = 0;
  int64_t episode_index = 0;
  int step_in_episode = 0;
  std::vector<double> obs;
  int act_index = 0;
  std::vector<double> act_values;
  double log_prob = 0, value = 0, reward = 0;
  bool done = false;
  double latency = 0;
  std::vector<double> h_before;  // empty == absent
  uint64_t snapshot_version = 0;
};

// rollout.hpp:33-78
struct RolloutView {
  int T = 0, N = 0;
  ActionKind action_kind = ActionKind::Discrete;
  int obs_dim = 0, act_dim = 0, hidden_dim = 0;
  Mat obs, act_cont;
  std::vector<int> act_disc;
  std::vector<double> log_prob, value, reward, latency, advantage, returns;
  std::vector<uint8_t> done, stale, replayed;
  std::vector<int> env_index, seq_of_slot;
  std::vector<int64_t> episode_index;
  std::vector<int> step_in_episode;
  std::vector<uint64_t> version;
  std::vector<SequenceDescriptor> seqs;
  Mat h0;
  std::vector<int> per_env_counts;
  std::vector<double> env_bootstrap;
  std::vector<uint8_t> env_bootstrap_valid;
  int deficit = 0, stale_steps = 0, replayed_steps = 0;
  uint64_t snapshot_version = 0;
  double collect_wall_time = 0;

  int size() const { return static_cast<int>(done.size()); }
  int fresh_steps() const { return size() - replayed_steps; }

  // rollout.cpp:15-22
  void restale(uint64_t learner_version) {
    for (int i = 0; i < size(); ++i) {
      if (version[i] != learner_version && !stale[i]) {
        stale[i] = 1;
        ++stale_steps;
      }
    }
  }
};

enum class RolloutMode { Fixed = 0, Variable = 1 };
enum class AppendOutcome { Accepted = 0, RolloutFull = 1 };

// ---------------------------------------------------------------- rollout
// rollout.hpp:87-142, rollout.cpp:24-190
class RolloutBuffer {
 public:
  struct Config {
    int T = 0, N = 0;
    RolloutMode mode = RolloutMode::Variable;
    ActionKind action_kind = ActionKind::Discrete;
    int obs_dim = 0, act_dim = 0, hidden_dim = 0;
  };
  explicit RolloutBuffer(Config cfg) : cfg_(cfg) {  // rollout.cpp:24-31
    per_env_counts_.assign(cfg_.N, 0);
    env_prev_done_.assign(cfg_.N, 0);
    carryover_.resize(cfg_.N);
    bootstrap_.assign(cfg_.N, 0.0);
    bootstrap_valid_.assign(cfg_.N, 0);
    steps_.reserve(capacity());
  }
  int committed() const { return static_cast<int>(steps_.size()); }
  int capacity() const { return cfg_.T * cfg_.N; }
  bool open() const { return open_; }
  bool env_at_cap(int env) const {
    return cfg_.mode == RolloutMode::Fixed && per_env_counts_[env] >= cfg_.T;
  }
  int carryover_count() const {  // rollout.cpp:33-37
    int n = 0;
    for (const auto& c : carryover_) n += c.has_value() ? 1 : 0;
    return n;
  }
  void begin_rollout(uint64_t snapshot_version) {  // rollout.cpp:39-57
    open_ = true;
    snapshot_version_ = snapshot_version;
    steps_.clear();
    env_slots_.assign(cfg_.N, {});
    std::fill(per_env_counts_.begin(), per_env_counts_.end(), 0);
    std::fill(env_prev_done_.begin(), env_prev_done_.end(), 0);
    std::fill(bootstrap_.begin(), bootstrap_.end(), 0.0);
    std::fill(bootstrap_valid_.begin(), bootstrap_valid_.end(), 0);
    collect_time_ = 0;
    for (int e = 0; e < cfg_.N && open_; ++e) {
      if (carryover_[e]) {
        EnvStepRecord rec = std::move(*carryover_[e]);
        carryover_[e].reset();
        commit(rec);
      }
    }
  }
  AppendOutcome append_step(const EnvStepRecord& rec) {  // rollout.cpp:59-77
    if (rec.env_index < 0 || rec.env_index >= cfg_.N)
      throw ProtocolError("append_step: env_index out of range");
    if (!open_) {
      if (cfg_.mode == RolloutMode::Variable) {
        if (carryover_[rec.env_index])
          throw ProtocolError("append_step: two pending carryovers for env " +
                              std::to_string(rec.env_index));
        carryover_[rec.env_index] = rec;
      }
      return AppendOutcome::RolloutFull;
    }
    if (env_at_cap(rec.env_index)) return AppendOutcome::RolloutFull;
    return commit(rec);
  }
  void force_close() { open_ = false; }
  void set_bootstrap(int env, double value) {
    if (env < 0 || env >= cfg_.N) throw ProtocolError("set_bootstrap: env out of range");
    bootstrap_[env] = value;
    bootstrap_valid_[env] = 1;
  }
  RolloutView close_rollout();  // rollout.cpp:102-190

 private:
  AppendOutcome commit(const EnvStepRecord& rec) {  // rollout.cpp:79-93
    const int slot = static_cast<int>(steps_.size());
    steps_.push_back(rec);
    env_slots_[rec.env_index].push_back(slot);
    ++per_env_counts_[rec.env_index];
    if (cfg_.mode == RolloutMode::Variable) {
      if (committed() >= capacity()) open_ = false;
    } else {
      bool all_full = true;
      for (int e = 0; e < cfg_.N; ++e) all_full &= per_env_counts_[e] >= cfg_.T;
      if (all_full) open_ = false;
    }
    return AppendOutcome::Accepted;
  }

  Config cfg_;
  bool open_ = false;
  uint64_t snapshot_version_ = 0;
  std::vector<EnvStepRecord> steps_;
  std::vector<std::vector<int>> env_slots_;
  std::vector<int> per_env_counts_;
  std::vector<uint8_t> env_prev_done_;
  std::vector<std::optional<EnvStepRecord>> carryover_;
  std::vector<double> bootstrap_;
  std::vector<uint8_t> bootstrap_valid_;
  double collect_time_ = 0;
  int next_seq_id_ = 0;
};

RolloutView RolloutBuffer::close_rollout() {
  if (steps_.empty()) throw ProtocolError("close_rollout: buffer is empty");
  if (open_) throw ProtocolError("close_rollout: buffer still open (force_close for preemption)");
  const int s = committed();
  RolloutView v;
  v.T = cfg_.T;
  v.N = cfg_.N;
  v.action_kind = cfg_.action_kind;
  v.obs_dim = cfg_.obs_dim;
  v.act_dim = cfg_.act_dim;
  v.hidden_dim = cfg_.hidden_dim;
  v.obs = Mat(s, cfg_.obs_dim);
  if (cfg_.action_kind == ActionKind::Continuous) v.act_cont = Mat(s, cfg_.act_dim);
  else v.act_disc.resize(s);
  v.log_prob.resize(s);
  v.value.resize(s);
  v.reward.resize(s);
  v.latency.resize(s);
  v.advantage.assign(s, 0.0);
  v.returns.assign(s, 0.0);
  v.done.resize(s);
  v.stale.assign(s, 0);
  v.replayed.assign(s, 0);
  v.env_index.resize(s);
  v.seq_of_slot.resize(s);
  v.episode_index.resize(s);
  v.step_in_episode.resize(s);
  v.version.resize(s);
  v.per_env_counts = per_env_counts_;
  v.env_bootstrap = bootstrap_;
  v.env_bootstrap_valid = bootstrap_valid_;
  v.deficit = capacity() - s;
  v.snapshot_version = snapshot_version_;
  v.collect_wall_time = collect_time_;

  std::vector<std::vector<double>> h0_rows;
  int offset = 0;
  for (int e = 0; e < cfg_.N; ++e) {  // rollout.cpp:143-184
    bool start_seq = true;
    for (int k = 0; k < static_cast<int>(env_slots_[e].size()); ++k) {
      const EnvStepRecord& rec = steps_[env_slots_[e][k]];
      if (start_seq) {
        SequenceDescriptor d;
        d.seq_id = next_seq_id_++;
        d.env_index = e;
        d.length = 0;
        d.start_offset = offset;
        d.parent_start_offset = offset;
        d.h0_index = static_cast<int>(h0_rows.size());
        std::vector<double> h = rec.h_before;
        if (static_cast<int>(h.size()) != cfg_.hidden_dim) h.assign(cfg_.hidden_dim, 0.0);
        h0_rows.push_back(std::move(h));
        v.seqs.push_back(d);
        start_seq = false;
      }
      SequenceDescriptor& d = v.seqs.back();
      ++d.length;
      for (int j = 0; j < cfg_.obs_dim; ++j) v.obs(offset, j) = rec.obs[j];
      if (cfg_.action_kind == ActionKind::Continuous) {
        for (int j = 0; j < cfg_.act_dim; ++j) v.act_cont(offset, j) = rec.act_values[j];
      } else {
        v.act_disc[offset] = rec.act_index;
      }
      v.log_prob[offset] = rec.log_prob;
      v.value[offset] = rec.value;
      v.reward[offset] = rec.reward;
      v.latency[offset] = rec.latency;
      v.done[offset] = rec.done ? 1 : 0;
      v.env_index[offset] = e;
      v.seq_of_slot[offset] = static_cast<int>(v.seqs.size()) - 1;
      v.episode_index[offset] = rec.episode_index;
      v.step_in_episode[offset] = rec.step_in_episode;
      v.version[offset] = rec.snapshot_version;
      ++offset;
      if (rec.done) start_seq = true;
    }
  }
  v.h0 = Mat(static_cast<int>(h0_rows.size()), cfg_.hidden_dim);
  for (int i = 0; i < v.h0.r; ++i)
    for (int j = 0; j < cfg_.hidden_dim; ++j) v.h0(i, j) = h0_rows[i][j];
  return v;
}

// rollout.cpp:208-276
void backfill_stale(RolloutView& view, const RolloutView& prev, int deficit) {
  if (deficit == 0) return;
  if (deficit > prev.size())
    throw ProtocolError("backfill_stale: deficit exceeds previous rollout size");
  int max_id = 0;
  for (const auto& d : view.seqs) max_id = std::max(max_id, d.seq_id);
  std::vector<int> order;
  for (int i = 0; i < static_cast<int>(prev.seqs.size()); ++i)
    if (!prev.seqs[i].stale) order.push_back(i);
  for (int i = 0; i < static_cast<int>(prev.seqs.size()); ++i)
    if (prev.seqs[i].stale) order.push_back(i);

  auto append_rows = [](Mat& dst, const Mat& src, int begin, int count) {
    const int old = dst.r;
    Mat n(old + count, src.c);
    if (old) std::memcpy(n.d.data(), dst.d.data(), sizeof(double) * dst.d.size());
    std::memcpy(&n.d[(size_t)old * src.c], &src.d[(size_t)begin * src.c],
                sizeof(double) * (size_t)count * src.c);
    dst = std::move(n);
  };
  auto append_vals = [](std::vector<double>& dst, const std::vector<double>& src, int begin,
                        int count) {
    dst.insert(dst.end(), src.begin() + begin, src.begin() + begin + count);
  };

  int remaining = deficit;
  for (int idx : order) {
    if (remaining == 0) break;
    const SequenceDescriptor& src = prev.seqs[idx];
    const int take = std::min(src.length, remaining);
    const int dst_offset = view.size();
    SequenceDescriptor d;
    d.seq_id = ++max_id;
    d.env_index = src.env_index;
    d.length = take;
    d.start_offset = dst_offset;
    d.parent_start_offset = dst_offset;
    d.h0_index = view.h0.r;
    d.stale = true;
    append_rows(view.h0, prev.h0, src.h0_index, 1);
    append_rows(view.obs, prev.obs, src.start_offset, take);
    if (view.action_kind == ActionKind::Continuous) {
      append_rows(view.act_cont, prev.act_cont, src.start_offset, take);
    } else {
      view.act_disc.insert(view.act_disc.end(), prev.act_disc.begin() + src.start_offset,
                           prev.act_disc.begin() + src.start_offset + take);
    }
    append_vals(view.log_prob, prev.log_prob, src.start_offset, take);
    append_vals(view.value, prev.value, src.start_offset, take);
    append_vals(view.reward, prev.reward, src.start_offset, take);
    append_vals(view.latency, prev.latency, src.start_offset, take);
    append_vals(view.advantage, prev.advantage, src.start_offset, take);
    append_vals(view.returns, prev.returns, src.start_offset, take);
    const int seq_index = static_cast<int>(view.seqs.size());
    for (int k = 0; k < take; ++k) {
      const int sp = src.start_offset + k;
      view.done.push_back(prev.done[sp]);
      view.stale.push_back(1);
      view.replayed.push_back(1);
      view.env_index.push_back(prev.env_index[sp]);
      view.seq_of_slot.push_back(seq_index);
      view.episode_index.push_back(prev.episode_index[sp]);
      view.step_in_episode.push_back(prev.step_in_episode[sp]);
      view.version.push_back(prev.version[sp]);
    }
    view.seqs.push_back(d);
    view.stale_steps += take;
    view.replayed_steps += take;
    remaining -= take;
  }
}

// ---------------------------------------------------------------- packseq
// packseq.hpp:11-29
struct SequenceGroup {
  std::vector<SequenceDescriptor> seqs;
  int total_steps = 0;
};
struct PackedBatch {
  std::vector<SequenceDescriptor> seqs;
  std::vector<int> sorted_to_group, batch_sizes, offsets, slots;
  int total_steps = 0;
  int max_len() const { return static_cast<int>(batch_sizes.size()); }
};

// packseq.cpp:18-54
std::vector<SequenceGroup> split_in_order(const RolloutView& view, int B,
                                          const std::vector<int>& perm) {
  if (B < 1) throw ProtocolError("split_minibatches: B must be >= 1");
  const int total = view.size();
  if (total == 0) throw ProtocolError("split_minibatches: empty view");
  if (total == view.T * view.N && total % B != 0)
    throw ProtocolError("split_minibatches: B=" + std::to_string(B) +
                        " does not divide T*N=" + std::to_string(total));
  const int base = total / B;
  const int rem = total % B;
  std::vector<SequenceGroup> groups(B);
  int b = 0;
  int room = base + (rem > 0 ? 1 : 0);
  for (int pi : perm) {
    SequenceDescriptor cur = view.seqs[pi];
    while (cur.length > 0) {
      if (room == 0) {
        ++b;
        room = base + (b < rem ? 1 : 0);
      }
      const int take = std::min(cur.length, room);
      SequenceDescriptor part = cur;
      part.length = take;
      groups[b].seqs.push_back(part);
      groups[b].total_steps += take;
      room -= take;
      cur.start_offset += take;
      cur.skip += take;
      cur.length -= take;
    }
  }
  return groups;
}

// packseq.cpp:10-16
std::vector<int> shuffle_perm(int n, uint64_t seed) {
  std::vector<int> perm(n);
  std::iota(perm.begin(), perm.end(), 0);
  std::mt19937_64 gen(seed);
  std::shuffle(perm.begin(), perm.end(), gen);
  return perm;
}
std::vector<SequenceGroup> split_minibatches(const RolloutView& view, int B, uint64_t seed) {
  return split_in_order(view, B, shuffle_perm(static_cast<int>(view.seqs.size()), seed));
}

// packseq.cpp:56-88
PackedBatch pack(const SequenceGroup& group) {
  if (group.seqs.empty()) throw ProtocolError("pack: empty sequence group");
  PackedBatch out;
  const int k = static_cast<int>(group.seqs.size());
  out.sorted_to_group.resize(k);
  std::iota(out.sorted_to_group.begin(), out.sorted_to_group.end(), 0);
  std::stable_sort(out.sorted_to_group.begin(), out.sorted_to_group.end(),
                   [&](int a, int b) { return group.seqs[a].length > group.seqs[b].length; });
  out.seqs.reserve(k);
  for (int i : out.sorted_to_group) out.seqs.push_back(group.seqs[i]);
  const int max_len = out.seqs.front().length;
  out.batch_sizes.resize(max_len);
  out.offsets.resize(max_len);
  int pos = 0;
  for (int t = 0; t < max_len; ++t) {
    int alive = 0;
    while (alive < k && out.seqs[alive].length > t) ++alive;
    out.batch_sizes[t] = alive;
    out.offsets[t] = pos;
    pos += alive;
  }
  out.total_steps = pos;
  out.slots.resize(pos);
  for (int t = 0; t < max_len; ++t)
    for (int j = 0; j < out.batch_sizes[t]; ++j)
      out.slots[out.offsets[t] + j] = out.seqs[j].start_offset + t;
  return out;
}

// ---------------------------------------------------------------- tape
// tape.hpp:13-68, tape.cpp:9-268
class Tape {
 public:
  using NodeId = int;
  NodeId constant(Mat v) { return push(std::move(v), false, nullptr); }
  NodeId leaf(Mat v) {
    if (!v.all_finite()) throw ProtocolError("tape: non-finite leaf value");
    return push(std::move(v), true, nullptr);
  }
  NodeId matmul_op(NodeId a, NodeId b) {  // tape.cpp:35-42
    Mat v = matmul(val(a), val(b));
    const bool rg = rgf(a) || rgf(b);
    return push(std::move(v), rg, [a, b](Tape& t, const Mat& g) {
      // both adjoints are evaluated before accum() filters, as tape.cpp:38-41 does
      t.accum(a, matmul_nt(g, t.val(b)));
      t.accum(b, matmul_tn(t.val(a), g));
    });
  }
  NodeId add(NodeId a, NodeId b) {
    const Mat& x = val(a);
    const Mat& y = val(b);
    Mat v(x.r, x.c);
    for (size_t i = 0; i < v.size(); ++i) v.d[i] = x.d[i] + y.d[i];
    return push(std::move(v), rgf(a) || rgf(b), [a, b](Tape& t, const Mat& g) {
      t.accum(a, g);
      t.accum(b, g);
    });
  }
  NodeId sub(NodeId a, NodeId b) {
    const Mat& x = val(a);
    const Mat& y = val(b);
    Mat v(x.r, x.c);
    for (size_t i = 0; i < v.size(); ++i) v.d[i] = x.d[i] - y.d[i];
    return push(std::move(v), rgf(a) || rgf(b), [a, b](Tape& t, const Mat& g) {
      t.accum(a, g);
      Mat ng = g;
      for (double& z : ng.d) z = -z;
      t.accum(b, ng);
    });
  }
  NodeId cmul(NodeId a, NodeId b) {
    const Mat& x = val(a);
    const Mat& y = val(b);
    Mat v(x.r, x.c);
    for (size_t i = 0; i < v.size(); ++i) v.d[i] = x.d[i] * y.d[i];
    return push(std::move(v), rgf(a) || rgf(b), [a, b](Tape& t, const Mat& g) {
      Mat ga(g.r, g.c), gb(g.r, g.c);
      const Mat& xa = t.val(a);
      const Mat& yb = t.val(b);
      for (size_t i = 0; i < g.size(); ++i) {
        ga.d[i] = g.d[i] * yb.d[i];
        gb.d[i] = g.d[i] * xa.d[i];
      }
      t.accum(a, ga);
      t.accum(b, gb);
    });
  }
  NodeId add_rowvec(NodeId a, NodeId bias) {  // tape.cpp:74-77
    const Mat& x = val(a);
    const Mat& bb = val(bias);
    Mat v(x.r, x.c);
    for (int i = 0; i < x.r; ++i)
      for (int j = 0; j < x.c; ++j) v(i, j) = x(i, j) + bb(0, j);
    return push(std::move(v), rgf(a) || rgf(bias), [a, bias](Tape& t, const Mat& g) {
      t.accum(a, g);
      t.accum(bias, colsum(g));
    });
  }
  NodeId broadcast_rows(NodeId a, int rows) {
    const Mat& x = val(a);
    Mat v(rows, x.c);
    for (int i = 0; i < rows; ++i)
      for (int j = 0; j < x.c; ++j) v(i, j) = x(0, j);
    return push(std::move(v), rgf(a), [a](Tape& t, const Mat& g) { t.accum(a, colsum(g)); });
  }
  NodeId replicate_cols(NodeId a, int cols) {
    const Mat& x = val(a);
    Mat v(x.r, cols);
    for (int i = 0; i < x.r; ++i)
      for (int j = 0; j < cols; ++j) v(i, j) = x(i, 0);
    return push(std::move(v), rgf(a), [a](Tape& t, const Mat& g) { t.accum(a, rowsum(g)); });
  }
  NodeId scale(NodeId a, double s) {
    Mat v = val(a);
    for (double& z : v.d) z *= s;
    return push(std::move(v), rgf(a), [a, s](Tape& t, const Mat& g) {
      Mat gs = g;
      for (double& z : gs.d) z *= s;
      t.accum(a, gs);
    });
  }
  NodeId add_scalar(NodeId a, double c) {
    Mat v = val(a);
    for (double& z : v.d) z += c;
    return push(std::move(v), rgf(a), [a](Tape& t, const Mat& g) { t.accum(a, g); });
  }
  NodeId tanh_op(NodeId a) {  // tape.cpp:107-115
    Mat v = val(a);
    for (double& z : v.d) z = std::tanh(z);
    NodeId out = push(std::move(v), rgf(a), nullptr);
    nodes_[out].back = [a, out](Tape& t, const Mat& g) {
      const Mat& y = t.val(out);
      Mat ga(g.r, g.c);
      for (size_t i = 0; i < g.size(); ++i) ga.d[i] = g.d[i] * (1.0 - y.d[i] * y.d[i]);
      t.accum(a, ga);
    };
    return out;
  }
  NodeId sigmoid_op(NodeId a) {  // tape.cpp:117-125
    Mat v = val(a);
    for (double& z : v.d) z = 1.0 / (1.0 + std::exp(-z));
    NodeId out = push(std::move(v), rgf(a), nullptr);
    nodes_[out].back = [a, out](Tape& t, const Mat& g) {
      const Mat& y = t.val(out);
      Mat ga(g.r, g.c);
      for (size_t i = 0; i < g.size(); ++i) ga.d[i] = g.d[i] * y.d[i] * (1.0 - y.d[i]);
      t.accum(a, ga);
    };
    return out;
  }
  NodeId exp_op(NodeId a) {
    Mat v = val(a);
    for (double& z : v.d) z = std::exp(z);
    NodeId out = push(std::move(v), rgf(a), nullptr);
    nodes_[out].back = [a, out](Tape& t, const Mat& g) {
      const Mat& y = t.val(out);
      Mat ga(g.r, g.c);
      for (size_t i = 0; i < g.size(); ++i) ga.d[i] = g.d[i] * y.d[i];
      t.accum(a, ga);
    };
    return out;
  }
  NodeId log_op(NodeId a) {
    Mat v = val(a);
    for (double& z : v.d) z = std::log(z);
    return push(std::move(v), rgf(a), [a](Tape& t, const Mat& g) {
      const Mat& x = t.val(a);
      Mat ga(g.r, g.c);
      for (size_t i = 0; i < g.size(); ++i) ga.d[i] = g.d[i] / x.d[i];
      t.accum(a, ga);
    });
  }
  NodeId clip(NodeId a, double lo, double hi) {  // tape.cpp:143-150: inclusive mask
    Mat v = val(a);
    for (double& z : v.d) z = std::min(std::max(z, lo), hi);
    return push(std::move(v), rgf(a), [a, lo, hi](Tape& t, const Mat& g) {
      const Mat& x = t.val(a);
      Mat ga(g.r, g.c);
      for (size_t i = 0; i < g.size(); ++i)
        ga.d[i] = g.d[i] * ((x.d[i] >= lo ? 1.0 : 0.0) * (x.d[i] <= hi ? 1.0 : 0.0));
      t.accum(a, ga);
    });
  }
  NodeId cmin(NodeId a, NodeId b) {  // tape.cpp:152-162: tie -> first argument
    const Mat& x = val(a);
    const Mat& y = val(b);
    Mat v(x.r, x.c);
    for (size_t i = 0; i < v.size(); ++i) v.d[i] = std::min(x.d[i], y.d[i]);
    return push(std::move(v), rgf(a) || rgf(b), [a, b](Tape& t, const Mat& g) {
      const Mat& xa = t.val(a);
      const Mat& xb = t.val(b);
      Mat ga(g.r, g.c), gb(g.r, g.c);
      for (size_t i = 0; i < g.size(); ++i) {
        const double m = xa.d[i] <= xb.d[i] ? 1.0 : 0.0;
        ga.d[i] = g.d[i] * m;
        gb.d[i] = g.d[i] * (1.0 - m);
      }
      t.accum(a, ga);
      t.accum(b, gb);
    });
  }
  NodeId rows(NodeId a, int start, int count) {  // tape.cpp:166-173: full-size scatter
    Mat v = val(a).middle_rows(start, count);
    return push(std::move(v), rgf(a), [a, start, count](Tape& t, const Mat& g) {
      if (g_sparse_rows) {  // same sums (x + 0 == x), without the full-size temporary
        t.accum_rows(a, g, start);
        return;
      }
      Mat full(t.val(a).r, t.val(a).c);
      std::memcpy(&full.d[(size_t)start * full.c], g.d.data(),
                  sizeof(double) * (size_t)count * full.c);
      t.accum(a, full);
    });
  }
  NodeId concat_rows(const std::vector<NodeId>& parts) {  // tape.cpp:175-200
    if (parts.empty()) throw ProtocolError("tape: concat_rows on empty list");
    int nrows = 0;
    bool rg = false;
    const int cols = val(parts[0]).c;
    for (NodeId p : parts) {
      nrows += val(p).r;
      rg = rg || rgf(p);
    }
    Mat v(nrows, cols);
    int at = 0;
    for (NodeId p : parts) {
      const Mat& x = val(p);
      std::memcpy(&v.d[(size_t)at * cols], x.d.data(), sizeof(double) * x.d.size());
      at += x.r;
    }
    std::vector<NodeId> ids = parts;
    return push(std::move(v), rg, [ids](Tape& t, const Mat& g) {
      int at2 = 0;
      for (NodeId p : ids) {
        const int r = t.val(p).r;
        t.accum(p, g.middle_rows(at2, r));
        at2 += r;
      }
    });
  }
  NodeId row_sum(NodeId a) {
    Mat v = rowsum(val(a));
    return push(std::move(v), rgf(a), [a](Tape& t, const Mat& g) {
      const int cols = t.val(a).c;
      Mat ga(g.r, cols);
      for (int i = 0; i < g.r; ++i)
        for (int j = 0; j < cols; ++j) ga(i, j) = g(i, 0);
      t.accum(a, ga);
    });
  }
  NodeId sum_all(NodeId a) {
    Mat v(1, 1);
    v(0, 0) = val(a).sum();
    return push(std::move(v), rgf(a), [a](Tape& t, const Mat& g) {
      t.accum(a, Mat(t.val(a).r, t.val(a).c, g(0, 0)));
    });
  }
  NodeId mean_all(NodeId a) {  // tape.cpp:218-226
    const double inv = 1.0 / static_cast<double>(val(a).size());
    Mat v(1, 1);
    v(0, 0) = val(a).sum() * inv;
    return push(std::move(v), rgf(a), [a, inv](Tape& t, const Mat& g) {
      t.accum(a, Mat(t.val(a).r, t.val(a).c, g(0, 0) * inv));
    });
  }
  NodeId gather_cols(NodeId a, std::vector<int> idx) {  // tape.cpp:228-240
    const Mat& x = val(a);
    if (static_cast<int>(idx.size()) != x.r)
      throw ProtocolError("tape: gather_cols index count mismatch");
    Mat v(x.r, 1);
    for (int i = 0; i < x.r; ++i) v(i, 0) = x(i, idx[i]);
    return push(std::move(v), rgf(a), [a, idx = std::move(idx)](Tape& t, const Mat& g) {
      Mat full(t.val(a).r, t.val(a).c);
      for (int i = 0; i < full.r; ++i) full(i, idx[i]) += g(i, 0);
      t.accum(a, full);
    });
  }

  const Mat& value(NodeId id) const { return nodes_[id].value; }

  void backward(NodeId root) {  // tape.cpp:242-257
    const Node& r = nodes_[root];
    if (r.value.r != 1 || r.value.c != 1) throw ProtocolError("tape: backward root must be 1x1");
    if (!std::isfinite(r.value(0, 0))) throw ProtocolError("tape: non-finite loss value");
    accum(root, Mat(1, 1, 1.0));
    for (NodeId id = root; id >= 0; --id) {
      Node& n = nodes_[id];
      if (n.grad.size() != 0 && n.back) n.back(*this, n.grad);
    }
  }
  Mat grad(NodeId id) const {  // tape.cpp:259-264
    const Node& n = nodes_[id];
    if (n.grad.size() == 0) return Mat(n.value.r, n.value.c);
    if (!n.grad.all_finite()) throw ProtocolError("tape: non-finite gradient");
    return n.grad;
  }

 private:
  struct Node {
    Mat value, grad;
    bool requires_grad = false;
    std::function<void(Tape&, const Mat&)> back;
  };
  const Mat& val(NodeId id) const { return nodes_[id].value; }
  bool rgf(NodeId id) const { return nodes_[id].requires_grad; }
  static Mat colsum(const Mat& g) {  // rows in ascending order per column
    Mat o(1, g.c);
    const int nb = (g.c + 15) / 16;
#pragma omp parallel for schedule(static) if (par_ok(g.size()))
    for (int b = 0; b < nb; ++b) {
      const int j0 = b * 16, j1 = std::min(g.c, j0 + 16);
      for (int i = 0; i < g.r; ++i)
        for (int j = j0; j < j1; ++j) o.d[j] += g.d[(size_t)i * g.c + j];
    }
    return o;
  }
  static Mat rowsum(const Mat& g) {
    Mat o(g.r, 1);
    for (int i = 0; i < g.r; ++i) {
      double s = 0;
      for (int j = 0; j < g.c; ++j) s += g(i, j);
      o(i, 0) = s;
    }
    return o;
  }
  NodeId push(Mat v, bool rg, std::function<void(Tape&, const Mat&)> back) {
    Node n;
    n.value = std::move(v);
    n.requires_grad = rg;
    n.back = std::move(back);
    nodes_.push_back(std::move(n));
    return static_cast<NodeId>(nodes_.size()) - 1;
  }
  void accum_rows(NodeId id, const Mat& g, int start) {  // accum of rows(start, g.r) only
    Node& n = nodes_[id];
    if (!n.requires_grad) return;
    if (n.grad.size() == 0) n.grad = Mat(n.value.r, n.value.c);
    double* dst = n.grad.d.data() + (size_t)start * n.grad.c;
    const double* src = g.d.data();
    const int64_t sz = (int64_t)g.size();
#pragma omp parallel for schedule(static) if (par_ok((size_t)sz))
    for (int64_t i = 0; i < sz; ++i) dst[i] += src[i];
  }
  void accum(NodeId id, const Mat& g) {  // tape.cpp:20-27
    Node& n = nodes_[id];
    if (!n.requires_grad) return;
    if (n.grad.size() == 0) n.grad = Mat(n.value.r, n.value.c);
    double* dst = n.grad.d.data();
    const double* src = g.d.data();
    const int64_t sz = (int64_t)g.size();
#pragma omp parallel for schedule(static) if (par_ok((size_t)sz))
    for (int64_t i = 0; i < sz; ++i) dst[i] += src[i];
  }
  std::vector<Node> nodes_;
};

// ---------------------------------------------------------------- nn
struct ModelConfig {  // nn.hpp:17-24
  int obs_dim = 0, encoder_dim = 64, hidden_dim = 64;
  ActionKind action_kind = ActionKind::Discrete;
  int num_actions = 0, act_dim = 0;
};
constexpr double kLogStdMin = -5.0;
constexpr double kLogStdMax = 2.0;
constexpr double kLog2Pi = 1.8378770664093453;

// nn.hpp:33-52; tensors() order nn.cpp:83-95
struct PolicyParams {
  ModelConfig cfg;
  Mat enc_w1, enc_b1, enc_w2, enc_b2;
  Mat gru_wr, gru_ur, gru_br, gru_wz, gru_uz, gru_bz, gru_wn, gru_un, gru_bn;
  Mat head_w, head_b, log_std, value_w, value_b;

  std::vector<Mat*> tensors() {
    std::vector<Mat*> out = {&enc_w1, &enc_b1, &enc_w2, &enc_b2, &gru_wr, &gru_ur,
                             &gru_br, &gru_wz, &gru_uz, &gru_bz, &gru_wn, &gru_un,
                             &gru_bn, &head_w, &head_b, &value_w, &value_b};
    if (cfg.action_kind == ActionKind::Continuous) out.push_back(&log_std);
    return out;
  }
  std::vector<const Mat*> tensors() const {
    std::vector<const Mat*> o;
    for (Mat* m : const_cast<PolicyParams*>(this)->tensors()) o.push_back(m);
    return o;
  }
  void clamp_log_std() {  // nn.cpp:105-109
    for (double& z : log_std.d) z = std::min(std::max(z, kLogStdMin), kLogStdMax);
  }
  bool all_finite() const {
    for (const Mat* t : tensors())
      if (!t->all_finite()) return false;
    return true;
  }
  int64_t count() const {
    int64_t n = 0;
    for (const Mat* t : tensors()) n += (int64_t)t->size();
    return n;
  }
  void to_flat(double* out) const {
    for (const Mat* t : tensors()) {
      std::memcpy(out, t->d.data(), sizeof(double) * t->size());
      out += t->size();
    }
  }
  void from_flat(const double* in) {
    for (Mat* t : tensors()) {
      std::memcpy(t->d.data(), in, sizeof(double) * t->size());
      in += t->size();
    }
  }
};

static void shape_params(PolicyParams& p, const ModelConfig& cfg) {
  const int E = cfg.encoder_dim, H = cfg.hidden_dim;
  const int A = cfg.action_kind == ActionKind::Discrete ? cfg.num_actions : cfg.act_dim;
  p.cfg = cfg;
  p.enc_w1 = Mat(cfg.obs_dim, E);
  p.enc_b1 = Mat(1, E);
  p.enc_w2 = Mat(E, E);
  p.enc_b2 = Mat(1, E);
  p.gru_wr = Mat(E, H);
  p.gru_ur = Mat(H, H);
  p.gru_br = Mat(1, H);
  p.gru_wz = Mat(E, H);
  p.gru_uz = Mat(H, H);
  p.gru_bz = Mat(1, H);
  p.gru_wn = Mat(E, H);
  p.gru_un = Mat(H, H);
  p.gru_bn = Mat(1, H);
  p.head_w = Mat(H, A);
  p.head_b = Mat(1, A);
  p.log_std = cfg.action_kind == ActionKind::Continuous ? Mat(1, cfg.act_dim) : Mat(0, 0);
  p.value_w = Mat(H, 1);
  p.value_b = Mat(1, 1);
}

// nn.cpp:16-30.  Eigen::HouseholderQR replaced by an explicit Householder QR;
// after the sign fix (diag(R) > 0) the thin Q factor is unique, so the result
// equals the reference's up to rounding.
static Mat orthogonal(int rows, int cols, double gain, CounterRng rng) {
  const int big = std::max(rows, cols);
  const int small = std::min(rows, cols);
  Mat g(big, small);
  for (int i = 0; i < big; ++i)
    for (int j = 0; j < small; ++j) g(i, j) = rng.normal();
  // Householder QR of g (big x small): R in-place, reflectors stored separately
  Mat a = g;
  std::vector<std::vector<double>> vs(small);
  std::vector<double> rdiag(small);
  for (int k = 0; k < small; ++k) {
    double norm = 0;
    for (int i = k; i < big; ++i) norm += a(i, k) * a(i, k);
    norm = std::sqrt(norm);
    const double alpha = a(k, k) > 0 ? -norm : norm;
    std::vector<double> v(big - k);
    for (int i = k; i < big; ++i) v[i - k] = a(i, k);
    v[0] -= alpha;
    double vn = 0;
    for (double z : v) vn += z * z;
    if (vn > 0) {
      for (int j = k; j < small; ++j) {
        double s = 0;
        for (int i = k; i < big; ++i) s += v[i - k] * a(i, j);
        s = 2.0 * s / vn;
        for (int i = k; i < big; ++i) a(i, j) -= s * v[i - k];
      }
    }
    rdiag[k] = a(k, k);
    vs[k] = std::move(v);
  }
  // thin Q = H_0 ... H_{small-1} * I(big, small)
  Mat q(big, small);
  for (int j = 0; j < small; ++j) q(j, j) = 1.0;
  for (int k = small - 1; k >= 0; --k) {
    const std::vector<double>& v = vs[k];
    double vn = 0;
    for (double z : v) vn += z * z;
    if (vn == 0) continue;
    for (int j = 0; j < small; ++j) {
      double s = 0;
      for (int i = k; i < big; ++i) s += v[i - k] * q(i, j);
      s = 2.0 * s / vn;
      for (int i = k; i < big; ++i) q(i, j) -= s * v[i - k];
    }
  }
  for (int j = 0; j < small; ++j)
    if (rdiag[j] < 0)
      for (int i = 0; i < big; ++i) q(i, j) = -q(i, j);
  if (rows < cols) q = q.transpose();
  for (double& z : q.d) z *= gain;
  return q;
}

// nn.cpp:44-81
PolicyParams init_params(const ModelConfig& cfg, uint64_t seed) {
  PolicyParams p;
  shape_params(p, cfg);
  CounterRng rng(seed);
  const int E = cfg.encoder_dim, H = cfg.hidden_dim;
  const int A = cfg.action_kind == ActionKind::Discrete ? cfg.num_actions : cfg.act_dim;
  p.enc_w1 = orthogonal(cfg.obs_dim, E, std::sqrt(2.0), rng.stream(1));
  p.enc_w2 = orthogonal(E, E, std::sqrt(2.0), rng.stream(2));
  p.gru_wr = orthogonal(E, H, 1.0, rng.stream(3));
  p.gru_ur = orthogonal(H, H, 1.0, rng.stream(4));
  p.gru_wz = orthogonal(E, H, 1.0, rng.stream(5));
  p.gru_uz = orthogonal(H, H, 1.0, rng.stream(6));
  p.gru_wn = orthogonal(E, H, 1.0, rng.stream(7));
  p.gru_un = orthogonal(H, H, 1.0, rng.stream(8));
  p.head_w = orthogonal(H, A, 0.01, rng.stream(9));
  p.value_w = orthogonal(H, 1, 1.0, rng.stream(10));
  return p;
}

static Mat add_row(Mat m, const Mat& b) {
  for (int i = 0; i < m.r; ++i)
    for (int j = 0; j < m.c; ++j) m(i, j) += b(0, j);
  return m;
}

// nn.cpp:32-46
static Mat gru_cell(const PolicyParams& p, const Mat& x, const Mat& h) {
  Mat rr = add_row(matmul(x, p.gru_wr), p.gru_br);
  gemm_acc(h, p.gru_ur, rr);
  Mat rz = add_row(matmul(x, p.gru_wz), p.gru_bz);
  gemm_acc(h, p.gru_uz, rz);
  Mat hun = matmul(h, p.gru_un);
  Mat xn = matmul(x, p.gru_wn);
  Mat out(x.r, p.cfg.hidden_dim);
  for (int i = 0; i < x.r; ++i) {
    for (int j = 0; j < out.c; ++j) {
      const double sr = 1.0 / (1.0 + std::exp(-rr(i, j)));
      const double sz = 1.0 / (1.0 + std::exp(-rz(i, j)));
      const double n = std::tanh(xn(i, j) + sr * hun(i, j) + p.gru_bn(0, j));
      out(i, j) = (1.0 - sz) * n + sz * h(i, j);
    }
  }
  return out;
}
static Mat encode(const PolicyParams& p, const Mat& obs) {
  Mat e1 = add_row(matmul(obs, p.enc_w1), p.enc_b1);
  for (double& z : e1.d) z = std::tanh(z);
  Mat e2 = add_row(matmul(e1, p.enc_w2), p.enc_b2);
  for (double& z : e2.d) z = std::tanh(z);
  return e2;
}

struct ActResult {
  Mat dist, h_new;
  std::vector<double> value;
};
// nn.cpp:118-126
ActResult act(const PolicyParams& p, const Mat& obs, const Mat& h) {
  if (!obs.all_finite()) throw ProtocolError("act: non-finite observation");
  ActResult out;
  Mat e = encode(p, obs);
  out.h_new = gru_cell(p, e, h);
  out.dist = add_row(matmul(out.h_new, p.head_w), p.head_b);
  Mat v = add_row(matmul(out.h_new, p.value_w), p.value_b);
  out.value.resize(v.r);
  for (int i = 0; i < v.r; ++i) out.value[i] = v(i, 0);
  return out;
}

// nn.cpp:147-163
double categorical_log_prob(const double* logits, int A, int action) {
  double m = logits[0];
  for (int i = 1; i < A; ++i) m = std::max(m, logits[i]);
  double s = 0;
  for (int i = 0; i < A; ++i) s += std::exp(logits[i] - m);
  return logits[action] - (m + std::log(s));
}
double categorical_entropy(const double* logits, int A) {
  double m = logits[0];
  for (int i = 1; i < A; ++i) m = std::max(m, logits[i]);
  std::vector<double> z(A);
  double s = 0;
  for (int i = 0; i < A; ++i) {
    z[i] = std::exp(logits[i] - m);
    s += z[i];
  }
  double h = 0;
  for (int i = 0; i < A; ++i) {
    const double p = z[i] / s;
    if (p > 0) h -= p * (logits[i] - m - std::log(s));
  }
  return h;
}

struct TapeParams {  // nn.hpp:82-89
  Tape::NodeId enc_w1, enc_b1, enc_w2, enc_b2;
  Tape::NodeId gru_wr, gru_ur, gru_br, gru_wz, gru_uz, gru_bz, gru_wn, gru_un, gru_bn;
  Tape::NodeId head_w, head_b, log_std = -1, value_w, value_b;
  std::vector<Tape::NodeId> ids;
};
// nn.cpp:187-217
TapeParams register_params(Tape& tape, const PolicyParams& p) {
  TapeParams tp;
  tp.enc_w1 = tape.leaf(p.enc_w1);
  tp.enc_b1 = tape.leaf(p.enc_b1);
  tp.enc_w2 = tape.leaf(p.enc_w2);
  tp.enc_b2 = tape.leaf(p.enc_b2);
  tp.gru_wr = tape.leaf(p.gru_wr);
  tp.gru_ur = tape.leaf(p.gru_ur);
  tp.gru_br = tape.leaf(p.gru_br);
  tp.gru_wz = tape.leaf(p.gru_wz);
  tp.gru_uz = tape.leaf(p.gru_uz);
  tp.gru_bz = tape.leaf(p.gru_bz);
  tp.gru_wn = tape.leaf(p.gru_wn);
  tp.gru_un = tape.leaf(p.gru_un);
  tp.gru_bn = tape.leaf(p.gru_bn);
  tp.head_w = tape.leaf(p.head_w);
  tp.head_b = tape.leaf(p.head_b);
  tp.value_w = tape.leaf(p.value_w);
  tp.value_b = tape.leaf(p.value_b);
  tp.ids = {tp.enc_w1, tp.enc_b1, tp.enc_w2, tp.enc_b2, tp.gru_wr, tp.gru_ur,
            tp.gru_br, tp.gru_wz, tp.gru_uz, tp.gru_bz, tp.gru_wn, tp.gru_un,
            tp.gru_bn, tp.head_w, tp.head_b, tp.value_w, tp.value_b};
  if (p.cfg.action_kind == ActionKind::Continuous) {
    tp.log_std = tape.leaf(p.log_std);
    tp.ids.push_back(tp.log_std);
  }
  return tp;
}

struct PackedForward {
  Tape::NodeId log_prob = -1, entropy = -1, value = -1;
};
// nn.cpp:219-280
PackedForward forward_packed(Tape& tape, const TapeParams& tp, const ModelConfig& cfg,
                             const Mat& obs_packed, const std::vector<int>& act_disc,
                             const Mat& act_cont, const std::vector<int>& batch_sizes,
                             const std::vector<int>& offsets, const Mat& h0_sorted) {
  if (!obs_packed.all_finite()) throw ProtocolError("forward_packed: non-finite observations");
  const int S = obs_packed.r;
  auto obs = tape.constant(obs_packed);
  auto e1 = tape.tanh_op(tape.add_rowvec(tape.matmul_op(obs, tp.enc_w1), tp.enc_b1));
  auto enc = tape.tanh_op(tape.add_rowvec(tape.matmul_op(e1, tp.enc_w2), tp.enc_b2));
  auto h = tape.constant(h0_sorted);
  int h_rows = h0_sorted.r;
  std::vector<Tape::NodeId> parts;
  parts.reserve(batch_sizes.size());
  for (size_t t = 0; t < batch_sizes.size(); ++t) {
    const int bs = batch_sizes[t];
    auto x = tape.rows(enc, offsets[t], bs);
    auto hp = bs < h_rows ? tape.rows(h, 0, bs) : h;
    auto r = tape.sigmoid_op(tape.add_rowvec(
        tape.add(tape.matmul_op(x, tp.gru_wr), tape.matmul_op(hp, tp.gru_ur)), tp.gru_br));
    auto z = tape.sigmoid_op(tape.add_rowvec(
        tape.add(tape.matmul_op(x, tp.gru_wz), tape.matmul_op(hp, tp.gru_uz)), tp.gru_bz));
    auto n = tape.tanh_op(tape.add_rowvec(
        tape.add(tape.matmul_op(x, tp.gru_wn), tape.cmul(r, tape.matmul_op(hp, tp.gru_un))),
        tp.gru_bn));
    auto omz = tape.add_scalar(tape.scale(z, -1.0), 1.0);
    h = tape.add(tape.cmul(omz, n), tape.cmul(z, hp));
    h_rows = bs;
    parts.push_back(h);
  }
  auto hidden = parts.size() == 1 ? parts[0] : tape.concat_rows(parts);
  PackedForward out;
  out.value = tape.add_rowvec(tape.matmul_op(hidden, tp.value_w), tp.value_b);
  auto dist = tape.add_rowvec(tape.matmul_op(hidden, tp.head_w), tp.head_b);
  if (cfg.action_kind == ActionKind::Discrete) {
    const int A = cfg.num_actions;
    const Mat& dv = tape.value(dist);
    Mat shift(dv.r, A);
    for (int i = 0; i < dv.r; ++i) {
      double m = dv(i, 0);
      for (int j = 1; j < A; ++j) m = std::max(m, dv(i, j));
      for (int j = 0; j < A; ++j) shift(i, j) = m;
    }
    auto shifted = tape.sub(dist, tape.constant(shift));
    auto lse = tape.log_op(tape.row_sum(tape.exp_op(shifted)));
    auto logp_all = tape.sub(shifted, tape.replicate_cols(lse, A));
    out.log_prob = tape.gather_cols(logp_all, act_disc);
    auto probs = tape.exp_op(logp_all);
    out.entropy = tape.scale(tape.row_sum(tape.cmul(probs, logp_all)), -1.0);
  } else {
    const int D = cfg.act_dim;
    auto logstd = tape.broadcast_rows(tp.log_std, S);
    auto inv_std = tape.exp_op(tape.scale(logstd, -1.0));
    auto diff = tape.sub(tape.constant(act_cont), dist);
    auto zsc = tape.cmul(diff, inv_std);
    auto quad = tape.scale(tape.row_sum(tape.cmul(zsc, zsc)), -0.5);
    out.log_prob = tape.add_scalar(tape.sub(quad, tape.row_sum(logstd)),
                                   -0.5 * kLog2Pi * static_cast<double>(D));
    out.entropy = tape.add_scalar(tape.row_sum(logstd),
                                  0.5 * (1.0 + kLog2Pi) * static_cast<double>(D));
  }
  return out;
}

// nn.hpp:105-118, nn.cpp:284-312
struct AdamState {
  std::vector<Mat> m, v;
  long step = 0;
  double beta1 = 0.9, beta2 = 0.999, eps = 1e-8;
};
AdamState make_adam(const PolicyParams& p) {
  AdamState st;
  for (const Mat* t : p.tensors()) {
    st.m.emplace_back(t->r, t->c);
    st.v.emplace_back(t->r, t->c);
  }
  return st;
}
void adam_step(AdamState& st, PolicyParams& p, const std::vector<Mat>& grads, double lr) {
  auto ts = p.tensors();
  if (grads.size() != ts.size()) throw ProtocolError("adam_step: gradient count mismatch");
  ++st.step;
  const double bc1 = 1.0 - std::pow(st.beta1, static_cast<double>(st.step));
  const double bc2 = 1.0 - std::pow(st.beta2, static_cast<double>(st.step));
  for (size_t i = 0; i < ts.size(); ++i) {
    Mat& w = *ts[i];
    const Mat& g = grads[i];
    for (size_t k = 0; k < w.size(); ++k) {
      st.m[i].d[k] = st.beta1 * st.m[i].d[k] + (1.0 - st.beta1) * g.d[k];
      st.v[i].d[k] = st.beta2 * st.v[i].d[k] + (1.0 - st.beta2) * (g.d[k] * g.d[k]);
      const double mhat = st.m[i].d[k] / bc1;
      const double vhat = st.v[i].d[k] / bc2;
      w.d[k] -= lr * mhat / (std::sqrt(vhat) + st.eps);
    }
  }
}
struct CosineSchedule {
  double base_lr = 2.5e-4;
  long total_steps = 1;
  double lr_at(long consumed) const {
    double progress = static_cast<double>(consumed) / static_cast<double>(std::max(1L, total_steps));
    progress = std::min(std::max(progress, 0.0), 1.0);
    return base_lr * 0.5 * (1.0 + std::cos(M_PI * progress));
  }
};

// ---------------------------------------------------------------- learner
struct PPOConfig {  // learner.hpp:14-22
  double gamma = 0.99, gae_lambda = 0.95, clip = 0.2;
  int epochs = 3, minibatches = 2;
  double value_loss_coef = 0.5, is_cap = 1.0;
};
struct EntropyController {  // learner.hpp:29-40
  double alpha = 1e-3, target = 0.0, lower = 1e-4, upper = 1.0, lr = 2.5e-4;
  void update(double mean_entropy) {
    alpha += lr * (target - mean_entropy);
    alpha = std::min(std::max(alpha, lower), upper);
  }
};
inline double entropy_loss_value(double mean_entropy, const EntropyController& c) {
  return c.alpha * (c.target - mean_entropy) - c.alpha * mean_entropy;
}

// learner.cpp:11-41
void compute_gae(RolloutView& view, double gamma, double lambda) {
  for (int e = 0; e < view.N; ++e) {
    std::vector<int> slots;
    for (int i = 0; i < view.size(); ++i)
      if (view.env_index[i] == e && !view.replayed[i]) slots.push_back(i);
    if (slots.empty()) continue;
    double next_adv = 0;
    double next_value = 0;
    {
      const int last = slots.back();
      if (!view.done[last]) {
        if (!view.env_bootstrap_valid[e])
          throw ProtocolError("compute_gae: missing bootstrap value for env " + std::to_string(e));
        next_value = view.env_bootstrap[e];
      }
    }
    for (int k = static_cast<int>(slots.size()) - 1; k >= 0; --k) {
      const int i = slots[k];
      const double mask = view.done[i] ? 0.0 : 1.0;
      const double delta = view.reward[i] + gamma * next_value * mask - view.value[i];
      next_adv = delta + gamma * lambda * mask * next_adv;
      view.advantage[i] = next_adv;
      view.returns[i] = next_adv + view.value[i];
      next_value = view.value[i];
    }
  }
}

struct TrainStats {  // learner.hpp:55-71
  long update_index = 0;
  int steps = 0, fresh_steps = 0, stale_steps = 0;
  double loss = 0, policy_loss = 0, value_loss = 0, entropy = 0, entropy_loss = 0,
         mean_ratio = 0, clip_fraction = 0, mean_is_weight = 0, max_is_weight = 0, alpha = 0,
         lr = 0;
};
struct PPOLossResult {  // learner.hpp:80-92
  double loss = 0, policy_loss = 0, value_loss = 0, mean_entropy = 0, ratio_sum = 0,
         clip_count = 0, w_sum = 0, w_max = 0;
  int steps = 0;
  Mat is_weights;
  std::vector<Mat> grads;
};

// learner.cpp:52-117
PPOLossResult ppo_loss(const PolicyParams& params, const RolloutView& view,
                       const PackedBatch& batch, const PPOConfig& cfg, double alpha,
                       const Mat& h0_sorted, bool want_grads, const Mat* frozen_is_weights) {
  const int S = batch.total_steps;
  Mat obs(S, view.obs_dim);
  std::vector<int> act_disc(view.action_kind == ActionKind::Discrete ? S : 0);
  Mat act_cont(view.action_kind == ActionKind::Continuous ? S : 0, view.act_dim);
  Mat old_logp(S, 1), adv(S, 1), ret(S, 1);
  for (int i = 0; i < S; ++i) {  // learner.cpp:56-70
    const int slot = batch.slots[i];
    for (int j = 0; j < view.obs_dim; ++j) obs(i, j) = view.obs(slot, j);
    if (view.action_kind == ActionKind::Discrete) act_disc[i] = view.act_disc[slot];
    else
      for (int j = 0; j < view.act_dim; ++j) act_cont(i, j) = view.act_cont(slot, j);
    old_logp(i, 0) = view.log_prob[slot];
    adv(i, 0) = view.advantage[slot];
    ret(i, 0) = view.returns[slot];
  }
  Tape tape;
  TapeParams tp = register_params(tape, params);
  PackedForward f = forward_packed(tape, tp, params.cfg, obs, act_disc, act_cont,
                                   batch.batch_sizes, batch.offsets, h0_sorted);
  auto ratio = tape.exp_op(tape.sub(f.log_prob, tape.constant(old_logp)));
  auto adv_c = tape.constant(adv);
  auto s1 = tape.cmul(ratio, adv_c);
  auto s2 = tape.cmul(tape.clip(ratio, 1.0 - cfg.clip, 1.0 + cfg.clip), adv_c);
  auto surrogate = tape.cmin(s1, s2);
  Mat w;
  if (frozen_is_weights) {
    w = *frozen_is_weights;
  } else {
    w = tape.value(ratio);
    for (double& z : w.d) z = std::min(z, cfg.is_cap);
  }
  auto policy_loss = tape.scale(tape.mean_all(tape.cmul(tape.constant(w), surrogate)), -1.0);
  auto verr = tape.sub(f.value, tape.constant(ret));
  auto value_loss = tape.scale(tape.mean_all(tape.cmul(verr, verr)), 0.5);
  auto mean_entropy = tape.mean_all(f.entropy);
  auto total = tape.add(tape.add(policy_loss, tape.scale(value_loss, cfg.value_loss_coef)),
                        tape.scale(mean_entropy, -alpha));
  PPOLossResult out;
  out.steps = S;
  out.loss = tape.value(total)(0, 0);
  out.policy_loss = tape.value(policy_loss)(0, 0);
  out.value_loss = tape.value(value_loss)(0, 0);
  out.mean_entropy = tape.value(mean_entropy)(0, 0);
  const Mat& rv = tape.value(ratio);
  out.ratio_sum = rv.sum();
  for (int i = 0; i < S; ++i)
    if (rv(i, 0) < 1.0 - cfg.clip || rv(i, 0) > 1.0 + cfg.clip) out.clip_count += 1;
  out.w_sum = w.sum();
  if (S > 0) {
    double mx = w.d[0];
    for (double z : w.d) mx = std::max(mx, z);
    out.w_max = mx;
  }
  out.is_weights = std::move(w);
  if (want_grads) {
    if (!std::isfinite(out.loss)) throw ProtocolError("ppo_loss: non-finite loss");
    tape.backward(total);
    out.grads.reserve(tp.ids.size());
    for (auto id : tp.ids) out.grads.push_back(tape.grad(id));
  }
  return out;
}

class Learner {  // learner.hpp:102-138, learner.cpp:43-193
 public:
  Learner(PolicyParams params, PPOConfig cfg, EntropyController entropy, CosineSchedule schedule,
          uint64_t run_seed)
      : params_(std::move(params)),
        cfg_(cfg),
        entropy_(entropy),
        schedule_(schedule),
        adam_(make_adam(params_)),
        run_seed_(run_seed) {}

  // learner.cpp:119-130
  Mat batch_h0(const RolloutView& view, const PackedBatch& batch) const {
    Mat h0(static_cast<int>(batch.seqs.size()), view.hidden_dim);
    for (size_t s = 0; s < batch.seqs.size(); ++s) {
      const SequenceDescriptor& d = batch.seqs[s];
      Mat h = view.h0.row(d.h0_index);
      for (int t = 0; t < d.skip; ++t) h = act(params_, view.obs.row(d.parent_start_offset + t), h).h_new;
      for (int j = 0; j < view.hidden_dim; ++j) h0((int)s, j) = h(0, j);
    }
    return h0;
  }

  // learner.cpp:146-193 (max_minibatches < 0: the whole update)
  TrainStats update(RolloutView& view, int max_minibatches = -1) {
    compute_gae(view, cfg_.gamma, cfg_.gae_lambda);
    const double lr = schedule_.lr_at(consumed_steps_);
    TrainStats out;
    out.update_index = update_index_;
    out.steps = view.size();
    out.fresh_steps = view.fresh_steps();
    out.stale_steps = view.stale_steps;
    out.lr = lr;
    double ratio_sum = 0, clip_count = 0, w_sum = 0;
    long total_steps = 0;
    int batches = 0;
    for (int epoch = 0; epoch < cfg_.epochs; ++epoch) {
      const uint64_t seed = rng::mix(rng::mix(run_seed_, update_index_), epoch);
      auto groups = split_minibatches(view, cfg_.minibatches, seed);
      for (const auto& g : groups) {
        if (max_minibatches >= 0 && batches >= max_minibatches) break;
        PackedBatch batch = pack(g);
        PPOLossResult st = run_minibatch(view, batch, lr);
        out.loss += st.loss;
        out.policy_loss += st.policy_loss;
        out.value_loss += st.value_loss;
        out.entropy += st.mean_entropy;
        ratio_sum += st.ratio_sum;
        clip_count += st.clip_count;
        w_sum += st.w_sum;
        out.max_is_weight = std::max(out.max_is_weight, st.w_max);
        total_steps += st.steps;
        ++batches;
      }
    }
    out.loss /= batches;
    out.policy_loss /= batches;
    out.value_loss /= batches;
    out.entropy /= batches;
    out.entropy_loss = entropy_loss_value(out.entropy, entropy_);
    out.mean_ratio = ratio_sum / static_cast<double>(total_steps);
    out.clip_fraction = clip_count / static_cast<double>(total_steps);
    out.mean_is_weight = w_sum / static_cast<double>(total_steps);
    out.alpha = entropy_.alpha;
    if (max_minibatches < 0) {
      consumed_steps_ += view.fresh_steps();
      ++update_index_;
    }
    return out;
  }

  PolicyParams params_;
  PPOConfig cfg_;
  EntropyController entropy_;
  CosineSchedule schedule_;
  AdamState adam_;
  uint64_t run_seed_;
  long consumed_steps_ = 0;
  long update_index_ = 0;
  vo_grad_hook_fn grad_hook = nullptr;
  vo_entropy_hook_fn entropy_hook = nullptr;
  void* hook_user = nullptr;

 private:
  // learner.cpp:132-144
  PPOLossResult run_minibatch(const RolloutView& view, const PackedBatch& batch, double lr) {
    Mat h0 = batch_h0(view, batch);
    PPOLossResult res = ppo_loss(params_, view, batch, cfg_, entropy_.alpha, h0, true, nullptr);
    if (grad_hook) {
      std::vector<double> flat;
      for (const Mat& g : res.grads) flat.insert(flat.end(), g.d.begin(), g.d.end());
      grad_hook(flat.data(), (int64_t)flat.size(), hook_user);
      size_t at = 0;
      for (Mat& g : res.grads) {
        std::memcpy(g.d.data(), &flat[at], sizeof(double) * g.size());
        at += g.size();
      }
    }
    adam_step(adam_, params_, res.grads, lr);
    params_.clamp_log_std();
    if (!params_.all_finite()) throw ProtocolError("update: non-finite parameters");
    entropy_.update(entropy_hook ? entropy_hook(res.mean_entropy, hook_user) : res.mean_entropy);
    return res;
  }
};

// ---------------------------------------------------------------- distributed
// distributed.cpp:16-65
struct PreemptionEstimator {
  double learn_time = 0;
  std::vector<double> step_times;
  long max_steps = 0;
};
static long count_yields(const PreemptionEstimator& m, double t) {
  long c = 0;
  for (double tau : m.step_times) c += static_cast<long>(std::floor(t / tau));
  return c;
}
double estimate_time(const PreemptionEstimator& m, long steps) {
  if (steps < 0 || steps > m.max_steps) throw ProtocolError("estimate_time: S out of range [0, S_max]");
  if (steps == 0) return 0.0;
  if (m.step_times.empty()) throw ProtocolError("estimate_time: no step-time estimates");
  for (double tau : m.step_times)
    if (!(tau > 0)) throw ProtocolError("estimate_time: non-positive step time");
  double tau_min = *std::min_element(m.step_times.begin(), m.step_times.end());
  double lo = 0.0;
  double hi = tau_min * static_cast<double>(steps);
  while (count_yields(m, hi) < steps) hi *= 2;
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (mid <= lo || mid >= hi) break;
    if (count_yields(m, mid) >= steps) hi = mid;
    else lo = mid;
  }
  double best = hi;
  for (double tau : m.step_times) {
    const double c = std::floor(hi / tau) * tau;
    if (c > lo && c < best) best = c;
  }
  return best;
}
long optimal_preempt_steps(const PreemptionEstimator& m) {
  if (!(m.learn_time > 0)) throw ProtocolError("optimal_preempt_steps: LT must be positive");
  long best_s = 1;
  double best_rate = -1;
  for (long s = 1; s <= m.max_steps; ++s) {
    const double rate = static_cast<double>(s) / (estimate_time(m, s) + m.learn_time);
    if (rate > best_rate) {
      best_rate = rate;
      best_s = s;
    }
  }
  return best_s;
}
// test_distributed.cpp:16-37: the merge/sort formulation (k * tau as double(k)*tau)
std::vector<double> merged_times(const PreemptionEstimator& m, long steps) {
  std::vector<double> yields;
  for (double tau : m.step_times)
    for (long k = 1; k <= steps; ++k) yields.push_back(static_cast<double>(k) * tau);
  std::sort(yields.begin(), yields.end());
  yields.resize(steps);
  return yields;
}
long optimal_preempt_steps_sorted(const PreemptionEstimator& m) {
  if (!(m.learn_time > 0)) throw ProtocolError("optimal_preempt_steps: LT must be positive");
  // bound the enumeration by Time(S_max) so it stays O(S_max log S_max)
  const double tmax = estimate_time(m, m.max_steps);
  std::vector<double> yields;
  yields.reserve(m.max_steps + m.step_times.size());
  for (double tau : m.step_times) {
    for (long k = 1;; ++k) {
      const double y = static_cast<double>(k) * tau;
      if (y > tmax * (1 + 1e-9) || k > m.max_steps) break;
      yields.push_back(y);
    }
  }
  std::sort(yields.begin(), yields.end());
  long best_s = 1;
  double best = -1;
  for (long s = 1; s <= m.max_steps; ++s) {
    const double rate = static_cast<double>(s) / (yields[s - 1] + m.learn_time);
    if (rate > best) {
      best = rate;
      best_s = s;
    }
  }
  return best_s;
}

}  // namespace vo

// ======================================================================= C shim
using namespace vo;

static thread_local std::string g_err;

#define VO_TRY(...)                           \
  try {                                       \
    __VA_ARGS__;                                  \
    return 0;                                 \
  } catch (const vo::ProtocolError& e) {      \
    g_err = e.what();                         \
    return 1;                                 \
  } catch (const std::exception& e) {         \
    g_err = e.what();                         \
    return 2;                                 \
  }

struct vo_view_s {
  RolloutView v;
};
struct vo_rollout_s {
  RolloutBuffer b;
  RolloutBuffer::Config cfg;
};
struct vo_groups_s {
  std::vector<SequenceGroup> g;
};
struct vo_packed_s {
  PackedBatch p;
};
struct vo_learner_s {
  Learner l;
};

static SequenceDescriptor desc_from(const int32_t* s) {
  SequenceDescriptor d;
  d.seq_id = s[0];
  d.env_index = s[1];
  d.length = s[2];
  d.start_offset = s[3];
  d.h0_index = s[4];
  d.stale = s[5] != 0;
  d.parent_start_offset = s[6];
  d.skip = s[7];
  return d;
}
static void desc_to(const SequenceDescriptor& d, int32_t* s) {
  s[0] = d.seq_id;
  s[1] = d.env_index;
  s[2] = d.length;
  s[3] = d.start_offset;
  s[4] = d.h0_index;
  s[5] = d.stale ? 1 : 0;
  s[6] = d.parent_start_offset;
  s[7] = d.skip;
}

static ModelConfig model_from(const vo_model_config* c) {
  ModelConfig m;
  m.obs_dim = c->obs_dim;
  m.encoder_dim = c->encoder_dim;
  m.hidden_dim = c->hidden_dim;
  m.action_kind = c->action_kind ? ActionKind::Continuous : ActionKind::Discrete;
  m.num_actions = c->num_actions;
  m.act_dim = c->act_dim;
  return m;
}
static PolicyParams params_from(const vo_model_config* c, const double* flat) {
  PolicyParams p;
  shape_params(p, model_from(c));
  p.from_flat(flat);
  return p;
}
static PPOConfig ppo_from(const vo_ppo_config* c) {
  PPOConfig p;
  p.gamma = c->gamma;
  p.gae_lambda = c->gae_lambda;
  p.clip = c->clip;
  p.epochs = c->epochs;
  p.minibatches = c->minibatches;
  p.value_loss_coef = c->value_loss_coef;
  p.is_cap = c->is_cap;
  return p;
}

template <class T, class U>
static void cp(U* dst, const std::vector<T>& src) {
  if (dst) for (size_t i = 0; i < src.size(); ++i) dst[i] = static_cast<U>(src[i]);
}

extern "C" {

const char* vo_last_error(void) { return g_err.c_str(); }
uint64_t vo_splitmix64(uint64_t x) { return rng::splitmix64(x); }
uint64_t vo_mix(uint64_t a, uint64_t b) { return rng::mix(a, b); }

int vo_view_create(const vo_view_data* d, vo_view* out) {
  VO_TRY({
    auto* h = new vo_view_s();
    RolloutView& v = h->v;
    const int s = d->size;
    v.T = d->T;
    v.N = d->N;
    v.action_kind = d->action_kind ? ActionKind::Continuous : ActionKind::Discrete;
    v.obs_dim = d->obs_dim;
    v.act_dim = d->act_dim;
    v.hidden_dim = d->hidden_dim;
    v.obs = Mat(s, d->obs_dim);
    if (s) std::memcpy(v.obs.d.data(), d->obs, sizeof(double) * s * d->obs_dim);
    if (v.action_kind == ActionKind::Continuous) {
      v.act_cont = Mat(s, d->act_dim);
      if (s) std::memcpy(v.act_cont.d.data(), d->act_cont, sizeof(double) * s * d->act_dim);
    } else {
      v.act_disc.assign(d->act_disc, d->act_disc + s);
    }
    v.log_prob.assign(d->log_prob, d->log_prob + s);
    v.value.assign(d->value, d->value + s);
    v.reward.assign(d->reward, d->reward + s);
    v.latency.assign(d->latency, d->latency + s);
    v.advantage.assign(d->advantage, d->advantage + s);
    v.returns.assign(d->returns, d->returns + s);
    v.done.assign(d->done, d->done + s);
    v.stale.assign(d->stale, d->stale + s);
    v.replayed.assign(d->replayed, d->replayed + s);
    v.env_index.assign(d->env_index, d->env_index + s);
    v.seq_of_slot.assign(d->seq_of_slot, d->seq_of_slot + s);
    v.step_in_episode.assign(d->step_in_episode, d->step_in_episode + s);
    v.episode_index.assign(d->episode_index, d->episode_index + s);
    v.version.assign(d->version, d->version + s);
    for (int i = 0; i < d->num_seqs; ++i) v.seqs.push_back(desc_from(d->seqs + 8 * i));
    v.h0 = Mat(d->h0_rows, d->hidden_dim);
    if (d->h0_rows) std::memcpy(v.h0.d.data(), d->h0, sizeof(double) * d->h0_rows * d->hidden_dim);
    v.per_env_counts.assign(d->per_env_counts, d->per_env_counts + d->N);
    v.env_bootstrap.assign(d->env_bootstrap, d->env_bootstrap + d->N);
    v.env_bootstrap_valid.assign(d->env_bootstrap_valid, d->env_bootstrap_valid + d->N);
    v.deficit = d->deficit;
    v.stale_steps = d->stale_steps;
    v.replayed_steps = d->replayed_steps;
    v.snapshot_version = d->snapshot_version;
    v.collect_wall_time = d->collect_wall_time;
    *out = h;
  })
}

int vo_view_info(vo_view h, vo_view_data* d) {
  VO_TRY({
    const RolloutView& v = h->v;
    d->T = v.T;
    d->N = v.N;
    d->action_kind = v.action_kind == ActionKind::Continuous;
    d->obs_dim = v.obs_dim;
    d->act_dim = v.act_dim;
    d->hidden_dim = v.hidden_dim;
    d->size = v.size();
    d->num_seqs = static_cast<int>(v.seqs.size());
    d->h0_rows = v.h0.r;
    d->deficit = v.deficit;
    d->stale_steps = v.stale_steps;
    d->replayed_steps = v.replayed_steps;
    d->snapshot_version = v.snapshot_version;
    d->collect_wall_time = v.collect_wall_time;
  })
}

int vo_view_read(vo_view h, vo_view_data* d) {
  VO_TRY({
    const RolloutView& v = h->v;
    if (d->obs) std::memcpy(d->obs, v.obs.d.data(), sizeof(double) * v.obs.size());
    if (d->act_cont && v.act_cont.size())
      std::memcpy(d->act_cont, v.act_cont.d.data(), sizeof(double) * v.act_cont.size());
    cp(d->act_disc, v.act_disc);
    cp(d->log_prob, v.log_prob);
    cp(d->value, v.value);
    cp(d->reward, v.reward);
    cp(d->latency, v.latency);
    cp(d->advantage, v.advantage);
    cp(d->returns, v.returns);
    cp(d->done, v.done);
    cp(d->stale, v.stale);
    cp(d->replayed, v.replayed);
    cp(d->env_index, v.env_index);
    cp(d->seq_of_slot, v.seq_of_slot);
    cp(d->step_in_episode, v.step_in_episode);
    cp(d->episode_index, v.episode_index);
    cp(d->version, v.version);
    if (d->seqs)
      for (size_t i = 0; i < v.seqs.size(); ++i) desc_to(v.seqs[i], d->seqs + 8 * i);
    if (d->h0 && v.h0.size()) std::memcpy(d->h0, v.h0.d.data(), sizeof(double) * v.h0.size());
    cp(d->per_env_counts, v.per_env_counts);
    cp(d->env_bootstrap, v.env_bootstrap);
    cp(d->env_bootstrap_valid, v.env_bootstrap_valid);
  })
}

int vo_view_clone(vo_view v, vo_view* out) {
  VO_TRY({
    auto* h = new vo_view_s();
    h->v = v->v;
    *out = h;
  })
}
void vo_view_destroy(vo_view v) { delete v; }

int vo_rollout_create(int T, int N, int mode, int action_kind, int obs_dim, int act_dim,
                      int hidden_dim, vo_rollout* out) {
  VO_TRY({
    if (T < 1 || N < 1) throw ConfigError("rollout: T and N must be >= 1");
    RolloutBuffer::Config c;
    c.T = T;
    c.N = N;
    c.mode = mode ? RolloutMode::Variable : RolloutMode::Fixed;
    c.action_kind = action_kind ? ActionKind::Continuous : ActionKind::Discrete;
    c.obs_dim = obs_dim;
    c.act_dim = act_dim;
    c.hidden_dim = hidden_dim;
    *out = new vo_rollout_s{RolloutBuffer(c), c};
  })
}
void vo_rollout_destroy(vo_rollout r) { delete r; }
int vo_rollout_begin(vo_rollout r, uint64_t sv) { VO_TRY(r->b.begin_rollout(sv)) }

static EnvStepRecord make_rec(const RolloutBuffer::Config& c, int env, int64_t episode, int t,
                              const double* obs, int act_index, const double* act_values,
                              double log_prob, double value, double reward, int done,
                              double latency, const double* h_before, uint64_t sv) {
  EnvStepRecord rec;
  rec.env_index = env;
  rec.episode_index = episode;
  rec.step_in_episode = t;
  rec.obs.assign(obs, obs + c.obs_dim);
  rec.act_index = act_index;
  if (act_values) rec.act_values.assign(act_values, act_values + c.act_dim);
  rec.log_prob = log_prob;
  rec.value = value;
  rec.reward = reward;
  rec.done = done != 0;
  rec.latency = latency;
  if (h_before) rec.h_before.assign(h_before, h_before + c.hidden_dim);
  rec.snapshot_version = sv;
  return rec;
}

int vo_rollout_append(vo_rollout r, int env, int64_t episode, int t, const double* obs,
                      int act_index, const double* act_values, double log_prob, double value,
                      double reward, int done, double latency, const double* h_before,
                      uint64_t sv, int* outcome) {
  VO_TRY({
    auto o = r->b.append_step(make_rec(r->cfg, env, episode, t, obs, act_index, act_values,
                                       log_prob, value, reward, done, latency, h_before, sv));
    if (outcome) *outcome = static_cast<int>(o);
  })
}

int vo_rollout_append_batch(vo_rollout r, int n, const int32_t* env, const int64_t* episode,
                            const int32_t* t, const double* obs, const int32_t* act_index,
                            const double* act_values, const double* log_prob,
                            const double* value, const double* reward, const uint8_t* done,
                            const double* latency, const double* h_before,
                            const uint8_t* h_before_valid, const uint64_t* sv,
                            int32_t* outcomes) {
  VO_TRY({
    const auto& c = r->cfg;
    for (int i = 0; i < n; ++i) {
      const double* hb = nullptr;
      if (h_before && (!h_before_valid || h_before_valid[i])) hb = h_before + (size_t)i * c.hidden_dim;
      auto o = r->b.append_step(make_rec(
          c, env[i], episode ? episode[i] : 0, t ? t[i] : 0, obs + (size_t)i * c.obs_dim,
          act_index ? act_index[i] : 0, act_values ? act_values + (size_t)i * c.act_dim : nullptr,
          log_prob[i], value[i], reward[i], done[i], latency ? latency[i] : 0.0, hb,
          sv ? sv[i] : 0));
      if (outcomes) outcomes[i] = static_cast<int32_t>(o);
    }
  })
}
int vo_rollout_force_close(vo_rollout r) { VO_TRY(r->b.force_close()) }
int vo_rollout_set_bootstrap(vo_rollout r, int env, double value) {
  VO_TRY(r->b.set_bootstrap(env, value))
}
int vo_rollout_state(vo_rollout r, int* open, int* committed, int* carryover) {
  VO_TRY({
    if (open) *open = r->b.open();
    if (committed) *committed = r->b.committed();
    if (carryover) *carryover = r->b.carryover_count();
  })
}
int vo_rollout_close(vo_rollout r, vo_view* out) {
  VO_TRY({
    auto* h = new vo_view_s();
    try {
      h->v = r->b.close_rollout();
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  })
}
int vo_backfill_stale(vo_view view, vo_view prev, int deficit) {
  VO_TRY(backfill_stale(view->v, prev->v, deficit))
}
int vo_view_restale(vo_view view, uint64_t lv) { VO_TRY(view->v.restale(lv)) }

int vo_split_minibatches(vo_view v, int B, uint64_t seed, vo_groups* out) {
  VO_TRY({
    auto g = split_minibatches(v->v, B, seed);
    *out = new vo_groups_s{std::move(g)};
  })
}
int vo_split_in_order(vo_view v, int B, const int32_t* perm, int n, vo_groups* out) {
  VO_TRY({
    std::vector<int> p(perm, perm + n);
    for (int x : p)
      if (x < 0 || x >= static_cast<int>(v->v.seqs.size())) throw ProtocolError("split_in_order: bad index");
    auto g = split_in_order(v->v, B, p);
    *out = new vo_groups_s{std::move(g)};
  })
}
int vo_shuffle_perm(int n, uint64_t seed, int32_t* perm_out) {
  VO_TRY({
    auto p = shuffle_perm(n, seed);
    for (int i = 0; i < n; ++i) perm_out[i] = p[i];
  })
}
int vo_groups_count(vo_groups g, int* B) { VO_TRY(*B = static_cast<int>(g->g.size())) }
int vo_groups_get(vo_groups g, int b, int* num_seqs, int* total_steps, int32_t* seqs_out) {
  VO_TRY({
    const SequenceGroup& sg = g->g.at(b);
    if (num_seqs) *num_seqs = static_cast<int>(sg.seqs.size());
    if (total_steps) *total_steps = sg.total_steps;
    if (seqs_out)
      for (size_t i = 0; i < sg.seqs.size(); ++i) desc_to(sg.seqs[i], seqs_out + 8 * i);
  })
}
void vo_groups_destroy(vo_groups g) { delete g; }

int vo_pack(const int32_t* seqs, int k, vo_packed* out) {
  VO_TRY({
    SequenceGroup g;
    for (int i = 0; i < k; ++i) {
      g.seqs.push_back(desc_from(seqs + 8 * i));
      g.total_steps += g.seqs.back().length;
    }
    auto p = pack(g);
    *out = new vo_packed_s{std::move(p)};
  })
}
int vo_packed_info(vo_packed p, int* num_seqs, int* max_len, int* total_steps) {
  VO_TRY({
    if (num_seqs) *num_seqs = static_cast<int>(p->p.seqs.size());
    if (max_len) *max_len = p->p.max_len();
    if (total_steps) *total_steps = p->p.total_steps;
  })
}
int vo_packed_get(vo_packed p, int32_t* seqs_out, int32_t* s2g, int32_t* bs, int32_t* offs,
                  int32_t* slots) {
  VO_TRY({
    const PackedBatch& b = p->p;
    if (seqs_out)
      for (size_t i = 0; i < b.seqs.size(); ++i) desc_to(b.seqs[i], seqs_out + 8 * i);
    cp(s2g, b.sorted_to_group);
    cp(bs, b.batch_sizes);
    cp(offs, b.offsets);
    cp(slots, b.slots);
  })
}
void vo_packed_destroy(vo_packed p) { delete p; }

int vo_param_count(const vo_model_config* c, int64_t* count, int* num_tensors) {
  VO_TRY({
    PolicyParams p;
    shape_params(p, model_from(c));
    if (count) *count = p.count();
    if (num_tensors) *num_tensors = static_cast<int>(p.tensors().size());
  })
}
int vo_param_tensor(const vo_model_config* c, int idx, char* name, int* rows, int* cols,
                    int64_t* offset) {
  static const char* names[] = {"enc_w1", "enc_b1", "enc_w2", "enc_b2", "gru_wr", "gru_ur",
                                "gru_br", "gru_wz", "gru_uz", "gru_bz", "gru_wn", "gru_un",
                                "gru_bn", "head_w", "head_b", "value_w", "value_b", "log_std"};
  VO_TRY({
    PolicyParams p;
    shape_params(p, model_from(c));
    auto ts = p.tensors();
    if (idx < 0 || idx >= static_cast<int>(ts.size())) throw ConfigError("param_tensor: bad index");
    int64_t off = 0;
    for (int i = 0; i < idx; ++i) off += (int64_t)ts[i]->size();
    if (name) std::strcpy(name, names[idx]);
    if (rows) *rows = ts[idx]->r;
    if (cols) *cols = ts[idx]->c;
    if (offset) *offset = off;
  })
}
int vo_set_num_threads(int n) {
#ifdef _OPENMP
  omp_set_num_threads(n < 1 ? 1 : n);
#endif
  return 0;
}
int vo_set_sparse_rows(int on) {
  g_sparse_rows = on != 0;
  return 0;
}
int vo_get_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

int vo_params_init(const vo_model_config* c, uint64_t seed, double* out) {
  VO_TRY(init_params(model_from(c), seed).to_flat(out))
}
int vo_act(const vo_model_config* c, const double* params, int n, const double* obs,
           const double* h, double* dist_out, double* value_out, double* h_new_out) {
  VO_TRY({
    PolicyParams p = params_from(c, params);
    Mat o(n, c->obs_dim), hh(n, c->hidden_dim);
    std::memcpy(o.d.data(), obs, sizeof(double) * o.size());
    std::memcpy(hh.d.data(), h, sizeof(double) * hh.size());
    ActResult r = act(p, o, hh);
    if (dist_out) std::memcpy(dist_out, r.dist.d.data(), sizeof(double) * r.dist.size());
    if (value_out) std::memcpy(value_out, r.value.data(), sizeof(double) * r.value.size());
    if (h_new_out) std::memcpy(h_new_out, r.h_new.d.data(), sizeof(double) * r.h_new.size());
  })
}
int vo_forward_packed(const vo_model_config* c, const double* params, int S, const double* obs,
                      const int32_t* act_disc, const double* act_cont, int L, const int32_t* bs,
                      const int32_t* offs, const double* h0, int h0_rows, double* logp_out,
                      double* ent_out, double* value_out) {
  VO_TRY({
    PolicyParams p = params_from(c, params);
    Mat o(S, c->obs_dim), ac(c->action_kind ? S : 0, c->act_dim), hh(h0_rows, c->hidden_dim);
    std::memcpy(o.d.data(), obs, sizeof(double) * o.size());
    if (c->action_kind) std::memcpy(ac.d.data(), act_cont, sizeof(double) * ac.size());
    std::memcpy(hh.d.data(), h0, sizeof(double) * hh.size());
    std::vector<int> ad;
    if (!c->action_kind) ad.assign(act_disc, act_disc + S);
    std::vector<int> b(bs, bs + L), f(offs, offs + L);
    Tape tape;
    TapeParams tp = register_params(tape, p);
    PackedForward fw = forward_packed(tape, tp, p.cfg, o, ad, ac, b, f, hh);
    for (int i = 0; i < S; ++i) {
      if (logp_out) logp_out[i] = tape.value(fw.log_prob)(i, 0);
      if (ent_out) ent_out[i] = tape.value(fw.entropy)(i, 0);
      if (value_out) value_out[i] = tape.value(fw.value)(i, 0);
    }
  })
}
double vo_categorical_log_prob(const double* logits, int A, int action) {
  return categorical_log_prob(logits, A, action);
}
double vo_categorical_entropy(const double* logits, int A) { return categorical_entropy(logits, A); }

int vo_compute_gae(vo_view v, double gamma, double lambda) {
  VO_TRY(compute_gae(v->v, gamma, lambda))
}

// compute_gae (learner.cpp:11-41) over bare SoA arrays, for the C5 CPU
// baseline.  reference_loop = 1: the reference's own O(N*S)
// structure (every env scans the whole view for its slots); 0: the same
// per-env reverse recursion with the slots bucketed by env in one O(S) pass.
int vo_gae_arrays(const float* reward, const float* value, const uint8_t* done, const int32_t* env,
                  const uint8_t* replayed, int S, int N, const float* boot, const uint8_t* boot_valid,
                  double gamma, double lambda, int reference_loop, float* adv, float* ret) {
  VO_TRY({
    auto env_pass = [&](int e, const std::vector<int>& slots) {
      if (slots.empty()) return;
      double next_adv = 0, next_value = 0;
      const int last = slots.back();
      if (!(done[last] & 1)) {
        if (!boot_valid[e]) throw ProtocolError("compute_gae: missing bootstrap value for env " + std::to_string(e));
        next_value = boot[e];
      }
      for (int k = (int)slots.size() - 1; k >= 0; --k) {
        const int i = slots[k];
        const double mask = (done[i] & 1) ? 0.0 : 1.0;
        const double delta = reward[i] + gamma * next_value * mask - value[i];
        next_adv = delta + gamma * lambda * mask * next_adv;
        adv[i] = (float)next_adv;
        ret[i] = (float)(next_adv + value[i]);
        next_value = value[i];
      }
    };
    if (reference_loop) {
      std::vector<int> slots;
      for (int e = 0; e < N; ++e) {
        slots.clear();
        for (int i = 0; i < S; ++i)
          if (env[i] == e && !replayed[i]) slots.push_back(i);
        env_pass(e, slots);
      }
    } else {
      std::vector<int> cnt(N + 1, 0), order(S);
      for (int i = 0; i < S; ++i)
        if (!replayed[i]) ++cnt[env[i] + 1];
      for (int e = 0; e < N; ++e) cnt[e + 1] += cnt[e];
      std::vector<int> pos(cnt.begin(), cnt.end() - 1);
      for (int i = 0; i < S; ++i)
        if (!replayed[i]) order[pos[env[i]]++] = i;
      std::vector<int> slots;
      for (int e = 0; e < N; ++e) {
        slots.assign(order.begin() + cnt[e], order.begin() + cnt[e + 1]);
        env_pass(e, slots);
      }
    }
  })
}

int vo_ppo_loss(const vo_model_config* c, const double* params, vo_view v, vo_packed p,
                const vo_ppo_config* cfg, double alpha, const double* h0_sorted, int want_grads,
                const double* frozen_w, vo_loss_result* out, double* grads_out, double* is_w_out) {
  VO_TRY({
    PolicyParams pp = params_from(c, params);
    const int k = static_cast<int>(p->p.seqs.size());
    Mat h0(k, c->hidden_dim);
    std::memcpy(h0.d.data(), h0_sorted, sizeof(double) * h0.size());
    Mat fw;
    if (frozen_w) {
      fw = Mat(p->p.total_steps, 1);
      std::memcpy(fw.d.data(), frozen_w, sizeof(double) * fw.size());
    }
    PPOLossResult r = ppo_loss(pp, v->v, p->p, ppo_from(cfg), alpha, h0, want_grads != 0,
                               frozen_w ? &fw : nullptr);
    out->loss = r.loss;
    out->policy_loss = r.policy_loss;
    out->value_loss = r.value_loss;
    out->mean_entropy = r.mean_entropy;
    out->ratio_sum = r.ratio_sum;
    out->clip_count = r.clip_count;
    out->w_sum = r.w_sum;
    out->w_max = r.w_max;
    out->steps = r.steps;
    if (grads_out && want_grads)
      for (const Mat& g : r.grads) {
        std::memcpy(grads_out, g.d.data(), sizeof(double) * g.size());
        grads_out += g.size();
      }
    if (is_w_out) std::memcpy(is_w_out, r.is_weights.d.data(), sizeof(double) * r.is_weights.size());
  })
}

int vo_learner_create(const vo_model_config* c, const double* params, const vo_ppo_config* cfg,
                      const vo_entropy_controller* ec, double base_lr, int64_t total_steps,
                      uint64_t run_seed, vo_learner* out) {
  VO_TRY({
    EntropyController e;
    e.alpha = ec->alpha;
    e.target = ec->target;
    e.lower = ec->lower;
    e.upper = ec->upper;
    e.lr = ec->lr;
    CosineSchedule s;
    s.base_lr = base_lr;
    s.total_steps = total_steps;
    *out = new vo_learner_s{Learner(params_from(c, params), ppo_from(cfg), e, s, run_seed)};
  })
}
void vo_learner_destroy(vo_learner l) { delete l; }
int vo_learner_set_hooks(vo_learner l, vo_grad_hook_fn g, vo_entropy_hook_fn e, void* user) {
  VO_TRY({
    l->l.grad_hook = g;
    l->l.entropy_hook = e;
    l->l.hook_user = user;
  })
}
static void stats_to(const TrainStats& s, vo_train_stats* o) {
  o->update_index = s.update_index;
  o->steps = s.steps;
  o->fresh_steps = s.fresh_steps;
  o->stale_steps = s.stale_steps;
  o->loss = s.loss;
  o->policy_loss = s.policy_loss;
  o->value_loss = s.value_loss;
  o->entropy = s.entropy;
  o->entropy_loss = s.entropy_loss;
  o->mean_ratio = s.mean_ratio;
  o->clip_fraction = s.clip_fraction;
  o->mean_is_weight = s.mean_is_weight;
  o->max_is_weight = s.max_is_weight;
  o->alpha = s.alpha;
  o->lr = s.lr;
}
int vo_learner_update(vo_learner l, vo_view v, vo_train_stats* out) {
  VO_TRY(stats_to(l->l.update(v->v), out))
}
int vo_learner_update_partial(vo_learner l, vo_view v, int max_mb, vo_train_stats* out) {
  VO_TRY(stats_to(l->l.update(v->v, max_mb), out))
}
int vo_learner_batch_h0(vo_learner l, vo_view v, vo_packed p, double* h0_out) {
  VO_TRY({
    Mat h = l->l.batch_h0(v->v, p->p);
    std::memcpy(h0_out, h.d.data(), sizeof(double) * h.size());
  })
}
int vo_learner_get_params(vo_learner l, double* out) { VO_TRY(l->l.params_.to_flat(out)) }
int vo_learner_set_params(vo_learner l, const double* in) { VO_TRY(l->l.params_.from_flat(in)) }
int vo_learner_get_adam(vo_learner l, double* m, double* v, int64_t* step) {
  VO_TRY({
    for (size_t i = 0; i < l->l.adam_.m.size(); ++i) {
      const Mat& a = l->l.adam_.m[i];
      const Mat& b = l->l.adam_.v[i];
      if (m) {
        std::memcpy(m, a.d.data(), sizeof(double) * a.size());
        m += a.size();
      }
      if (v) {
        std::memcpy(v, b.d.data(), sizeof(double) * b.size());
        v += b.size();
      }
    }
    if (step) *step = l->l.adam_.step;
  })
}
int vo_learner_get_state(vo_learner l, double* alpha, int64_t* consumed, int64_t* ui) {
  VO_TRY({
    if (alpha) *alpha = l->l.entropy_.alpha;
    if (consumed) *consumed = l->l.consumed_steps_;
    if (ui) *ui = l->l.update_index_;
  })
}
int vo_learner_set_state(vo_learner l, double alpha, int64_t consumed, int64_t ui) {
  VO_TRY({
    l->l.entropy_.alpha = alpha;
    l->l.consumed_steps_ = consumed;
    l->l.update_index_ = ui;
  })
}

int vo_adam_step(int64_t count, double* params, const double* grads, double* m, double* v,
                 int64_t* step, double lr) {
  VO_TRY({
    // one tensor holding everything: identical per-element arithmetic
    PolicyParams p;
    AdamState st;
    st.step = *step;
    Mat w(1, (int)count), g(1, (int)count), mm(1, (int)count), vv(1, (int)count);
    std::memcpy(w.d.data(), params, sizeof(double) * count);
    std::memcpy(g.d.data(), grads, sizeof(double) * count);
    std::memcpy(mm.d.data(), m, sizeof(double) * count);
    std::memcpy(vv.d.data(), v, sizeof(double) * count);
    ++st.step;
    const double bc1 = 1.0 - std::pow(st.beta1, static_cast<double>(st.step));
    const double bc2 = 1.0 - std::pow(st.beta2, static_cast<double>(st.step));
    for (int64_t k = 0; k < count; ++k) {
      mm.d[k] = st.beta1 * mm.d[k] + (1.0 - st.beta1) * g.d[k];
      vv.d[k] = st.beta2 * vv.d[k] + (1.0 - st.beta2) * (g.d[k] * g.d[k]);
      w.d[k] -= lr * (mm.d[k] / bc1) / (std::sqrt(vv.d[k] / bc2) + st.eps);
    }
    std::memcpy(params, w.d.data(), sizeof(double) * count);
    std::memcpy(m, mm.d.data(), sizeof(double) * count);
    std::memcpy(v, vv.d.data(), sizeof(double) * count);
    *step = st.step;
  })
}
double vo_cosine_lr(double base_lr, int64_t total_steps, int64_t consumed) {
  CosineSchedule s;
  s.base_lr = base_lr;
  s.total_steps = total_steps;
  return s.lr_at(consumed);
}
double vo_entropy_update(vo_entropy_controller* ec, double h) {
  EntropyController e;
  e.alpha = ec->alpha;
  e.target = ec->target;
  e.lower = ec->lower;
  e.upper = ec->upper;
  e.lr = ec->lr;
  e.update(h);
  ec->alpha = e.alpha;
  return e.alpha;
}

static PreemptionEstimator est_from(const double* tau, int n, double lt, int64_t max_steps) {
  PreemptionEstimator m;
  m.step_times.assign(tau, tau + n);
  m.learn_time = lt;
  m.max_steps = max_steps;
  return m;
}
int vo_estimate_time(const double* tau, int n, int64_t max_steps, int64_t steps, double* out) {
  VO_TRY(*out = estimate_time(est_from(tau, n, 0, max_steps), steps))
}
int vo_optimal_preempt_steps(const double* tau, int n, double lt, int64_t max_steps, int64_t* out) {
  VO_TRY(*out = optimal_preempt_steps(est_from(tau, n, lt, max_steps)))
}
double vo_merged_time(const double* tau, int n, int64_t steps) {
  if (steps == 0) return 0.0;
  return merged_times(est_from(tau, n, 0, steps), steps)[steps - 1];
}
int vo_optimal_preempt_steps_sorted(const double* tau, int n, double lt, int64_t max_steps,
                                    int64_t* out) {
  VO_TRY(*out = optimal_preempt_steps_sorted(est_from(tau, n, lt, max_steps)))
}

}  // extern "C"
