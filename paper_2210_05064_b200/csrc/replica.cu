// replica.cu — the learner section of ReplicaGroup::replica_main
// (distributed.cpp:208-264) for one process per GPU.
//
// The reference runs R replicas as threads that meet in SyncBarriers and in the
// shared AllReduce / PreemptCoordinator objects.  Here each GPU's process owns
// one ver_replica; the exchanges the reference does through shared memory are
// collectives (NCCL on the ctx communicator by default, or caller-supplied
// reducers -- e.g. gloo in the tests), and every rank computes the pooled
// preemption threshold S* itself from identical all-gathered inputs instead of
// rank 0 publishing it.  Per iteration, after the caller has collected and
// closed its rollout:
//
//   tau_e = wall / max(1, count_e)                       distributed.cpp:213-216
//   fresh = view.size(); global totals += sum(fresh)      :217, :221-226
//   learner.set_consumed_steps(global total before)       :228
//   backfill_stale(view, prev, deficit) if deficit > 0    :229-231
//   learner.update(view), learn_time (steady clock)       :232-235
//   prev = view                                           :240
//   LT = mean(learn_time); tau pooled over replicas;      :244-253
//   S* = optimal_preempt_steps(tau, LT, T*N*R) unless the last iteration
//   per-replica budget S*/R (ablation)                    :257-259
//   counter.start_iteration(threshold) (rank 0) + barrier :260-262, :200
//
// This file is a client of the C-ABI (ver_gpu.h) only, exactly as replica_main
// is a client of Learner / backfill_stale / optimal_preempt_steps.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <vector>

#include "common.cuh"

struct ver_replica_s {
  ver_ctx ctx = nullptr;
  ver_learner learner = nullptr;
  ver_replica_config cfg{};
  ver_replica_comm comm{};
  bool user_comm = false;
  int nranks = 1, rank = 0;
  ver_view prev = nullptr;
  ver_preempt counter = nullptr;
  int64_t global_consumed = 0;
  int64_t iteration = 0;
};

namespace {

void chk(ver_status s) {
  if (s != VER_OK) throw verg::Error(s, ver_last_error());
}

void sum_i64(ver_replica_s* r, int64_t* v, int n) {
  if (r->user_comm) {
    if (!r->comm.sum_i64 || r->comm.sum_i64(r->comm.user, v, n) != 0)
      verg::config_error("replica: sum_i64 collective failed");
    return;
  }
  chk(ver_allreduce_sum_i64(r->ctx, v, n));
}
void mean_f64(ver_replica_s* r, double* v, int n) {
  if (r->user_comm) {
    if (!r->comm.mean_f64 || r->comm.mean_f64(r->comm.user, v, n) != 0)
      verg::config_error("replica: mean_f64 collective failed");
    return;
  }
  chk(ver_allreduce_mean_f64(r->ctx, v, n));
}
void allgather_f64(ver_replica_s* r, const double* in, int n, double* out) {
  if (r->user_comm) {
    if (!r->comm.allgather_f64 || r->comm.allgather_f64(r->comm.user, in, n, out) != 0)
      verg::config_error("replica: allgather_f64 collective failed");
    return;
  }
  chk(ver_allgather_f64(r->ctx, in, n, out));
}

}  // namespace

extern "C" {

ver_status ver_replica_create(ver_ctx ctx, ver_learner learner, const ver_replica_config* cfg,
                              const ver_replica_comm* comm, ver_replica* out) {
  VER_API_BEGIN
  if (!ctx || !learner || !cfg || !out) verg::config_error("ver_replica_create: null argument");
  if (cfg->T < 1 || cfg->N < 1) verg::config_error("ver_replica_create: T and N must be >= 1");
  if (cfg->preempt != 0 && cfg->preempt != 1) verg::config_error("ver_replica_create: preempt must be 0 or 1");
  auto* r = new ver_replica_s();
  r->ctx = ctx;
  r->learner = learner;
  r->cfg = *cfg;
  if (comm) {
    if (comm->nranks < 1 || comm->rank < 0 || comm->rank >= comm->nranks) {
      delete r;
      verg::config_error("ver_replica_create: bad rank");
    }
    r->comm = *comm;
    r->user_comm = true;
    r->nranks = comm->nranks;
    r->rank = comm->rank;
  } else {
    r->nranks = ctx->c.comm ? ctx->c.nranks : 1;
    r->rank = ctx->c.comm ? ctx->c.rank : 0;
  }
  *out = r;
  VER_API_END
}

ver_status ver_replica_destroy(ver_replica r) {
  VER_API_BEGIN
  if (r) {
    if (r->prev) ver_view_destroy(r->prev);
    delete r;
  }
  VER_API_END
}

ver_status ver_replica_attach_preempt(ver_replica r, ver_preempt counter) {
  VER_API_BEGIN
  r->counter = counter;
  VER_API_END
}

ver_status ver_replica_learn(ver_replica r, ver_view view, double collect_wall_time, int last_iteration,
                             ver_iteration_result* out) {
  VER_API_BEGIN
  if (!r || !view) verg::config_error("ver_replica_learn: null argument");
  ver_view_host info{};
  chk(ver_view_info(view, &info));
  const int N = info.N;
  if (N != r->cfg.N) verg::config_error("ver_replica_learn: view N does not match the replica config");
  ver_iteration_result res{};
  res.iteration = r->iteration;
  res.rank = r->rank;
  res.deficit = info.deficit;

  // per-env step-time estimates from this rollout (distributed.cpp:213-216)
  std::vector<int32_t> counts(N);
  {
    ver_view_host h{};
    h.per_env_counts = counts.data();
    chk(ver_view_download(view, &h));
  }
  const double wall = collect_wall_time >= 0.0 ? collect_wall_time : info.collect_wall_time;
  std::vector<double> tau(N);
  for (int e = 0; e < N; ++e) tau[e] = wall / (double)std::max(1, counts[e]);

  // fresh counts -> global consumed steps for the LR schedule (:217, :221-228)
  int64_t fresh = info.size;
  sum_i64(r, &fresh, 1);
  const int64_t pre = r->global_consumed;
  r->global_consumed += fresh;
  res.global_consumed_before = pre;
  res.global_fresh = fresh;
  {
    double alpha = 0;
    int64_t consumed = 0, ui = 0;
    chk(ver_learner_get_state(r->learner, &alpha, &consumed, &ui));
    chk(ver_learner_set_state(r->learner, alpha, pre, ui));
  }

  // backfill with the previous rollout's stale steps (:229-231)
  if (info.deficit > 0 && r->prev) {
    ver_view_host ph{};
    chk(ver_view_info(r->prev, &ph));
    if (ph.size > 0) chk(ver_backfill_stale(view, r->prev, info.deficit));
  }

  // the update, timed as the reference does (steady clock around update, :232-235)
  const auto t0 = std::chrono::steady_clock::now();
  chk(ver_learner_update(r->learner, view, &res.train));
  const double learn_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  res.learn_time = learn_time;
  {
    ver_view_host a{};
    chk(ver_view_info(view, &a));
    res.stale_steps = a.stale_steps;
  }

  // prev_views_[rank] = view (:240); the caller keeps its handle
  ver_view keep = nullptr;
  chk(ver_view_clone(view, &keep));
  if (r->prev) ver_view_destroy(r->prev);
  r->prev = keep;

  // pooled statistics for the next threshold (:244-259); identical on every rank
  double lt = learn_time;
  mean_f64(r, &lt, 1);
  std::vector<double> pooled((size_t)N * r->nranks);
  allgather_f64(r, tau.data(), N, pooled.data());
  int64_t threshold = 0;
  if (r->cfg.preempt == 1 && !last_iteration && lt > 0.0) {
    const int64_t max_steps = (int64_t)r->cfg.T * N * r->nranks;
    chk(ver_optimal_preempt_steps(r->ctx, pooled.data(), (int)pooled.size(), lt, max_steps, &threshold));
  }
  res.mean_learn_time = lt;
  res.next_threshold = threshold;
  res.per_replica_threshold = r->cfg.per_replica_budget && threshold > 0 ? threshold / r->nranks : 0;

  // coordinator_.start_iteration(...) on rank 0, then every rank waits for it
  // before collecting again (the phase barrier at the top of the iteration, :200)
  if (r->counter && r->rank == 0) chk(ver_preempt_start(r->counter, r->cfg.per_replica_budget ? 0 : threshold));
  int64_t bar = 1;
  sum_i64(r, &bar, 1);
  if (bar != r->nranks) verg::protocol_error("replica: barrier count mismatch");
  ++r->iteration;
  if (out) *out = res;
  VER_API_END
}

ver_status ver_replica_state(ver_replica r, int64_t* global_consumed, int64_t* iteration, int* has_prev) {
  VER_API_BEGIN
  if (global_consumed) *global_consumed = r->global_consumed;
  if (iteration) *iteration = r->iteration;
  if (has_prev) *has_prev = r->prev != nullptr;
  VER_API_END
}

}  // extern "C"
