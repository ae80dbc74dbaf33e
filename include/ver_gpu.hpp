// ver_gpu.hpp — header-only C++17 wrapper over the C-ABI in ver_gpu.h.
//
// Gives C++ callers written against the reference's API (namespace ver,
// /root/reference/proj/src/*.hpp) the same shapes: RAII objects instead of
// handles, and exceptions instead of status codes:
//   VER_ERR_PROTOCOL  -> ProtocolError (types.hpp:41-44)
//   VER_ERR_CONFIG    -> ConfigError   (types.hpp:46-49)
//   VER_ERR_NONFINITE -> ProtocolError (the reference throws ProtocolError on a
//                        non-finite loss / parameters, learner.cpp:111,140)
//   VER_ERR_CUDA / VER_ERR_NCCL -> DeviceError
// Define VER_GPU_REFERENCE_ERRORS before including this header (after the
// reference's types.hpp) to throw the reference's own ver::ProtocolError /
// ver::ConfigError, so its doctest CHECK_THROWS_AS assertions hold unchanged.
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "ver_gpu.h"

namespace ver {
namespace gpu {

#ifdef VER_GPU_REFERENCE_ERRORS
using ProtocolError = ::ver::ProtocolError;
using ConfigError = ::ver::ConfigError;
#else
struct ProtocolError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
#endif
struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(ver_status s) {
  if (s == VER_OK) return;
  const std::string msg = ver_last_error();
  switch (s) {
    case VER_ERR_PROTOCOL:
    case VER_ERR_NONFINITE: throw ProtocolError(msg);
    case VER_ERR_CONFIG: throw ConfigError(msg);
    default: throw DeviceError(msg);
  }
}

// Move-only owner of one opaque handle.
template <class H, ver_status (*Destroy)(H)>
class Handle {
 public:
  Handle() = default;
  explicit Handle(H h) : h_(h) {}
  Handle(const Handle&) = delete;
  Handle& operator=(const Handle&) = delete;
  Handle(Handle&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
  Handle& operator=(Handle&& o) noexcept {
    if (this != &o) {
      reset();
      h_ = std::exchange(o.h_, nullptr);
    }
    return *this;
  }
  ~Handle() { reset(); }
  void reset() {
    if (h_) Destroy(h_);
    h_ = nullptr;
  }
  H get() const { return h_; }
  explicit operator bool() const { return h_ != nullptr; }

 private:
  H h_ = nullptr;
};

// Device + stream (+ NCCL communicator for DD-PPO replicas).
class Context : public Handle<ver_ctx, ver_ctx_destroy> {
 public:
  explicit Context(int device = 0) : Handle(make(device)) {}
  void synchronize() const { check(ver_ctx_synchronize(get())); }
  void init_nccl(const uint8_t id[128], int nranks, int rank) const {
    check(ver_ctx_init_nccl(get(), id, nranks, rank));
  }

 private:
  static ver_ctx make(int device) {
    ver_ctx c = nullptr;
    check(ver_ctx_create(device, &c));
    return c;
  }
};

// RolloutView (rollout.hpp:33-78), device resident.
class RolloutView : public Handle<ver_view, ver_view_destroy> {
 public:
  RolloutView() = default;
  explicit RolloutView(ver_view v) : Handle(v) {}
  ver_view_host info() const {
    ver_view_host h{};
    check(ver_view_info(get(), &h));
    return h;
  }
  int size() const { return info().size; }
  // RolloutView::fresh_steps (rollout.hpp:72-73)
  int fresh_steps() const {
    const auto h = info();
    return h.size - h.replayed_steps;
  }
  RolloutView clone() const {
    ver_view out = nullptr;
    check(ver_view_clone(get(), &out));
    return RolloutView(out);
  }
  void restale(uint64_t learner_version) { check(ver_view_restale(get(), learner_version)); }
};

// RolloutBuffer (rollout.hpp:99-123).
class RolloutBuffer : public Handle<ver_rollout, ver_rollout_destroy> {
 public:
  RolloutBuffer(const Context& ctx, const ver_rollout_config& cfg) : Handle(make(ctx, cfg)) {}
  void begin_rollout(uint64_t snapshot_version) { check(ver_rollout_begin(get(), snapshot_version)); }
  // append_step for a batch of records in arrival order; returns per-record
  // outcomes (0 Accepted, 1 RolloutFull)
  std::vector<int32_t> append(const ver_step_batch& b) {
    std::vector<int32_t> out(b.n > 0 ? b.n : 0);
    check(ver_rollout_append(get(), &b, out.data()));
    return out;
  }
  void force_close() { check(ver_rollout_force_close(get())); }
  void set_bootstrap(int env, float v) { check(ver_rollout_set_bootstrap(get(), env, v)); }
  // set_bootstrap for many envs in one call
  void set_bootstraps(const std::vector<int32_t>& envs, const std::vector<float>& values) {
    if (envs.size() != values.size()) throw ConfigError("set_bootstraps: size mismatch");
    check(ver_rollout_set_bootstraps(get(), (int)envs.size(), envs.data(), values.data()));
  }
  RolloutView close_rollout() {
    ver_view v = nullptr;
    check(ver_rollout_close(get(), &v));
    return RolloutView(v);
  }

 private:
  static ver_rollout make(const Context& ctx, const ver_rollout_config& cfg) {
    ver_rollout r = nullptr;
    check(ver_rollout_create(ctx.get(), &cfg, &r));
    return r;
  }
};

// backfill_stale (rollout.hpp:147)
inline void backfill_stale(RolloutView& view, const RolloutView& prev, int deficit) {
  check(ver_backfill_stale(view.get(), prev.get(), deficit));
}
// compute_gae (learner.hpp:53)
inline void compute_gae(RolloutView& view, double gamma, double lambda) {
  check(ver_compute_gae(view.get(), gamma, lambda));
}

// vector<SequenceGroup> (packseq.hpp:35-39)
class SequenceGroups : public Handle<ver_groups, ver_groups_destroy> {
 public:
  explicit SequenceGroups(ver_groups g) : Handle(g) {}
  int size() const {
    int b = 0;
    check(ver_groups_count(get(), &b));
    return b;
  }
  std::vector<ver_seq_desc> seqs(int b) const {
    int k = 0, steps = 0;
    check(ver_groups_get(get(), b, &k, &steps, nullptr));
    std::vector<ver_seq_desc> out(k);
    check(ver_groups_get(get(), b, &k, &steps, out.data()));
    return out;
  }
};
inline SequenceGroups split_minibatches(const RolloutView& v, int B, uint64_t seed) {
  ver_groups g = nullptr;
  check(ver_split_minibatches(v.get(), B, seed, &g));
  return SequenceGroups(g);
}
inline SequenceGroups split_in_order(const RolloutView& v, int B, const std::vector<int32_t>& order) {
  ver_groups g = nullptr;
  check(ver_split_in_order(v.get(), B, order.data(), (int)order.size(), &g));
  return SequenceGroups(g);
}

// PackedBatch (packseq.hpp:20-29)
class PackedBatch : public Handle<ver_packed, ver_packed_destroy> {
 public:
  explicit PackedBatch(ver_packed p) : Handle(p) {}
  struct Host {
    std::vector<ver_seq_desc> seqs;
    std::vector<int32_t> sorted_to_group, batch_sizes, offsets, slots;
  };
  Host host() const {
    int k = 0, L = 0, S = 0;
    check(ver_packed_info(get(), &k, &L, &S));
    Host h;
    h.seqs.resize(k);
    h.sorted_to_group.resize(k);
    h.batch_sizes.resize(L);
    h.offsets.resize(L);
    h.slots.resize(S);
    check(ver_packed_get(get(), h.seqs.data(), h.sorted_to_group.data(), h.batch_sizes.data(),
                         h.offsets.data(), h.slots.data()));
    return h;
  }
};
inline PackedBatch pack(const RolloutView& v, const SequenceGroups& g, int b) {
  ver_packed p = nullptr;
  check(ver_pack(v.get(), g.get(), b, &p));
  return PackedBatch(p);
}

// Learner (learner.hpp:102-138); params / Adam state in tensors() order.
class Learner : public Handle<ver_learner, ver_learner_destroy> {
 public:
  Learner(const Context& ctx, const ver_model_config& mc, const std::vector<float>& params,
          const ver_ppo_config& cfg, const ver_entropy_controller& ec, double base_lr, int64_t total_steps,
          uint64_t run_seed)
      : Handle(make(ctx, mc, params, cfg, ec, base_lr, total_steps, run_seed)), P_(params.size()) {}
  ver_train_stats update(RolloutView& v) {
    ver_train_stats s{};
    check(ver_learner_update(get(), v.get(), &s));
    return s;
  }
  // DD-PPO: average gradients over the ctx's NCCL communicator before Adam
  // (the grad_hook / entropy_hook of distributed.cpp:152-157)
  void enable_allreduce(bool on) { check(ver_learner_enable_allreduce(get(), on ? 1 : 0)); }
  std::vector<float> params() const {
    std::vector<float> out(P_);
    check(ver_learner_get_params(get(), out.data()));
    return out;
  }
  void set_params(const std::vector<float>& p) { check(ver_learner_set_params(get(), p.data())); }

 private:
  size_t P_;
  static ver_learner make(const Context& ctx, const ver_model_config& mc, const std::vector<float>& params,
                          const ver_ppo_config& cfg, const ver_entropy_controller& ec, double base_lr,
                          int64_t total_steps, uint64_t run_seed) {
    int64_t P = 0;
    int nt = 0;
    check(ver_param_count(&mc, &P, &nt));
    if ((int64_t)params.size() != P) throw ConfigError("Learner: parameter count mismatch");
    ver_learner l = nullptr;
    check(ver_learner_create(ctx.get(), &mc, params.data(), &cfg, &ec, base_lr, total_steps, run_seed, &l));
    return l;
  }
};

// InferenceEngine (runtime.hpp:96-160) on the device; requests as SoA arrays
// (ver_request_batch), dispatches returned as (env, action) arrays.
class InferenceEngine : public Handle<ver_engine, ver_engine_destroy> {
 public:
  struct Dispatches {
    std::vector<int32_t> env, action;  // discrete
    std::vector<float> action_cont;    // continuous: act_dim per dispatch
    int new_commits = 0;
    bool closed_now = false;
  };
  InferenceEngine(const Context& ctx, const ver_engine_config& cfg, const std::vector<float>& params,
                  uint64_t version)
      : Handle(make(ctx, cfg, params, version)), cfg_(cfg) {}
  void set_snapshot(const std::vector<float>& params, uint64_t version) {
    check(ver_engine_set_snapshot(get(), params.data(), version));
  }
  void set_snapshot(const Learner& l, uint64_t version) {
    check(ver_engine_set_snapshot_learner(get(), l.get(), version));
  }
  Dispatches begin_rollout() {
    Dispatches d = sized(cfg_.rollout.N);
    ver_batch_result r{};
    check(ver_engine_begin_rollout(get(), &r, d.env.data(), d.action.data(), d.action_cont.data()));
    return finish(d, r);
  }
  Dispatches process_batch(const ver_request_batch& reqs) {
    Dispatches d = sized(reqs.n);
    ver_batch_result r{};
    check(ver_engine_process_batch(get(), &reqs, &r, d.env.data(), d.action.data(), d.action_cont.data()));
    return finish(d, r);
  }
  void force_close() { check(ver_engine_force_close(get())); }
  // joint preemption: commits added from the sampling kernel, force-close when the group fires
  void attach_preempt(ver_preempt counter) { check(ver_engine_attach_preempt(get(), counter)); }
  void finalize_bootstraps() { check(ver_engine_finalize_bootstraps(get())); }
  RolloutView close() {
    ver_view v = nullptr;
    check(ver_engine_close(get(), &v));
    return RolloutView(v);
  }
  bool rollout_done() const {
    int open = 0;
    check(ver_engine_state(get(), &open, nullptr, nullptr, nullptr, nullptr));
    return !open;
  }

 private:
  ver_engine_config cfg_;
  Dispatches sized(int n) const {
    Dispatches d;
    const int A = cfg_.model.action_kind ? cfg_.model.act_dim : 1;
    d.env.resize(std::max(n, 1));
    d.action.resize(std::max(n, 1));
    d.action_cont.resize((size_t)std::max(n, 1) * A);
    return d;
  }
  Dispatches finish(Dispatches& d, const ver_batch_result& r) const {
    const int A = cfg_.model.action_kind ? cfg_.model.act_dim : 1;
    d.env.resize(r.n_dispatch);
    d.action.resize(r.n_dispatch);
    d.action_cont.resize((size_t)r.n_dispatch * A);
    d.new_commits = r.new_commits;
    d.closed_now = r.closed_now != 0;
    return std::move(d);
  }
  static ver_engine make(const Context& ctx, const ver_engine_config& cfg, const std::vector<float>& params,
                         uint64_t version) {
    int64_t P = 0;
    int nt = 0;
    check(ver_param_count(&cfg.model, &P, &nt));
    if ((int64_t)params.size() != P) throw ConfigError("InferenceEngine: parameter count mismatch");
    ver_engine e = nullptr;
    check(ver_engine_create(ctx.get(), &cfg, params.data(), version, &e));
    return e;
  }
};

// PreemptCoordinator (distributed.hpp:95-128) across processes: the owning
// replica creates the counter and ships ipc_handle() to the others, which open
// it; or (Nccl{}) one counter per rank, summed by the collective tick().
class PreemptCounter : public Handle<ver_preempt, ver_preempt_destroy> {
 public:
  struct Nccl {};
  explicit PreemptCounter(const Context& ctx) : Handle(make(ctx)) {}
  PreemptCounter(const Context& ctx, Nccl) : Handle(make_nccl(ctx)) {}
  PreemptCounter(const Context& ctx, const std::vector<uint8_t>& handle) : Handle(open(ctx, handle)) {}
  std::vector<uint8_t> ipc_handle() const {
    std::vector<uint8_t> h(64);
    check(ver_preempt_ipc_handle(get(), h.data()));
    return h;
  }
  void start_iteration(int64_t threshold) { check(ver_preempt_start(get(), threshold)); }
  // returns true on exactly one add per iteration (then every replica force-closes)
  bool add_steps(int64_t n, int64_t* total = nullptr) {
    int64_t t = 0;
    int f = 0;
    check(ver_preempt_add(get(), n, &t, &f));
    if (total) *total = t;
    return f != 0;
  }
  bool fired(int64_t* total = nullptr) const {
    int64_t t = 0;
    int f = 0;
    check(ver_preempt_state(get(), &t, &f));
    if (total) *total = t;
    return f != 0;
  }
  // NCCL mode: collective over the ranks; true on the tick that reaches the threshold
  bool tick(int64_t* total = nullptr) {
    int64_t t = 0;
    int f = 0;
    check(ver_preempt_tick(get(), &t, &f));
    if (total) *total = t;
    return f != 0;
  }

 private:
  static ver_preempt make(const Context& ctx) {
    ver_preempt p = nullptr;
    check(ver_preempt_create(ctx.get(), &p));
    return p;
  }
  static ver_preempt make_nccl(const Context& ctx) {
    ver_preempt p = nullptr;
    check(ver_preempt_create_nccl(ctx.get(), &p));
    return p;
  }
  static ver_preempt open(const Context& ctx, const std::vector<uint8_t>& h) {
    if (h.size() != 64) throw ConfigError("PreemptCounter: the IPC handle has 64 bytes");
    ver_preempt p = nullptr;
    check(ver_preempt_open(ctx.get(), h.data(), &p));
    return p;
  }
};

// PolicyParams::init (nn.cpp:16-81) as flat fp32 in tensors() order
inline std::vector<float> params_init(const ver_model_config& mc, uint64_t seed) {
  int64_t P = 0;
  int nt = 0;
  check(ver_param_count(&mc, &P, &nt));
  std::vector<double> d(P);
  check(ver_params_init(&mc, seed, d.data()));
  return std::vector<float>(d.begin(), d.end());
}

// estimate_time / optimal_preempt_steps (distributed.hpp:29-32)
inline double estimate_time(const Context& ctx, const std::vector<double>& tau, int64_t max_steps,
                            int64_t steps) {
  double out = 0;
  check(ver_estimate_time(ctx.get(), tau.data(), (int)tau.size(), max_steps, steps, &out));
  return out;
}
inline int64_t optimal_preempt_steps(const Context& ctx, const std::vector<double>& tau, double learn_time,
                                     int64_t max_steps) {
  int64_t out = 0;
  check(ver_optimal_preempt_steps(ctx.get(), tau.data(), (int)tau.size(), learn_time, max_steps, &out));
  return out;
}

}  // namespace gpu
}  // namespace ver
