/*
 * ver_gpu.h — C-ABI of the B200-native VER learner hot path.
 *
 * Every entry point replaces one function of the reference's C++ API
 * (/root/reference/proj, namespace ver); the reference file:line is cited on
 * each.  Plain pointers and sizes only: no torch / CUDA / C++ types cross this
 * boundary.  The C++ wrapper include/ver_gpu.hpp rethrows the status codes as
 * ver::ProtocolError / ver::ConfigError so callers written against the
 * reference (train_single bench.cpp:155, ReplicaGroup::replica_main
 * distributed.cpp:230-234, run_replay bench.cpp:386-409) keep their shape.
 *
 * Conventions
 *  - Every function returns ver_status; ver_last_error() holds the message of
 *    the last failure on the calling thread.
 *  - Handles are device-resident and stream-ordered on their ver_ctx's stream.
 *    They are not thread-safe: one learner per host thread per GPU (the
 *    reference's replica-per-thread model, distributed.cpp:271-276).
 *  - Only functions returning host values synchronize the stream.
 *  - Floating-point payloads are fp32 at the boundary (the reference is
 *    double; parity tolerances are stated in DESIGN.md).
 *  - There is no CPU fallback: every compute entry point launches sm_100a
 *    kernels and fails with VER_ERR_CUDA if no device is present.
 */
#ifndef VER_GPU_H
#define VER_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  VER_OK = 0,
  VER_ERR_PROTOCOL = 1,  /* ver::ProtocolError (types.hpp:41-44) */
  VER_ERR_CONFIG = 2,    /* ver::ConfigError   (types.hpp:46-49) / bad argument */
  VER_ERR_NONFINITE = 3, /* non-finite loss / parameters (learner.cpp:111,140) */
  VER_ERR_CUDA = 4,
  VER_ERR_NCCL = 5
} ver_status;

const char* ver_last_error(void);
/* library build string (arch, precision modes) */
const char* ver_version(void);

/* ------------------------------------------------------------------ context */
typedef struct ver_ctx_s* ver_ctx;
/* device ordinal; creates a non-blocking stream and the stream-ordered pool */
ver_status ver_ctx_create(int device, ver_ctx* out);
ver_status ver_ctx_destroy(ver_ctx ctx);
ver_status ver_ctx_synchronize(ver_ctx ctx);
/* the ctx stream as an opaque integer (cudaStream_t) for event timing */
ver_status ver_ctx_stream(ver_ctx ctx, uint64_t* stream_out);
/* number of kernels this library launched on ctx since creation / last reset */
ver_status ver_ctx_launch_count(ver_ctx ctx, int64_t* count, int reset);
/* precision of the tensor-core policy GEMMs: 0 = fp32-grade (the parity
   default: 3xTF32, or fp16x2 -- scaled fp16 hi + lo pairs, 22 significant bits,
   three kind::f16 MMAs per product -- for the forward GEMMs, the forward
   recurrence steps on CTA pairs and the backward data gradients; environment
   VER_TC_F16=0 keeps 3xTF32 everywhere), 1 = 1xTF32 (fast mode, looser bound
   stated in DESIGN.md) */
ver_status ver_ctx_set_precision(ver_ctx ctx, int mode);
/* 1 (default): batched policy GEMMs on tcgen05 tensor cores; 0: fp32 SIMT */
ver_status ver_ctx_set_tensor_cores(ver_ctx ctx, int enable);

/* NCCL (DD-PPO gradient AllReduce, distributed.cpp:86-116 / C1-C4 of SURVEY §2.2) */
ver_status ver_nccl_unique_id(uint8_t id_out[128]);
ver_status ver_ctx_init_nccl(ver_ctx ctx, const uint8_t id[128], int nranks, int rank);
/* in-place sum of n int64 across ranks (PreemptCoordinator step counts,
   fresh-step totals; distributed.hpp:111-119, distributed.cpp:222-226) */
ver_status ver_allreduce_sum_i64(ver_ctx ctx, int64_t* host_inout, int n);
/* in-place element-wise mean of n doubles across ranks (learn time, C4) */
ver_status ver_allreduce_mean_f64(ver_ctx ctx, double* host_inout, int n);
/* all-gather of n doubles per rank into out (nranks * n): pooled tau, C4 */
ver_status ver_allgather_f64(ver_ctx ctx, const double* host_in, int n, double* host_out);

/* ------------------------------------------------------------- view (L2) */
/* SequenceDescriptor (rollout.hpp:19-28): 8 x int32 */
typedef struct {
  int32_t seq_id, env_index, length, start_offset, h0_index, stale, parent_start_offset, skip;
} ver_seq_desc;

/* Host image of a RolloutView (rollout.hpp:33-78).  Used to upload an
   arbitrary view (test fixtures, load_view replay) and to read one back.
   Array pointers may be NULL on read to skip a field. */
typedef struct {
  int T, N, action_kind /*0 discrete, 1 continuous*/, obs_dim, act_dim, hidden_dim;
  int size, num_seqs, h0_rows;
  int deficit, stale_steps, replayed_steps;
  uint64_t snapshot_version;
  double collect_wall_time;
  float* obs;        /* size x obs_dim */
  float* act_cont;   /* size x act_dim  (continuous) */
  int32_t* act_disc; /* size            (discrete)   */
  float *log_prob, *value, *reward, *latency, *advantage, *returns;
  uint8_t *done, *stale, *replayed;
  int32_t *env_index, *seq_of_slot, *step_in_episode;
  int64_t* episode_index;
  uint64_t* version;
  ver_seq_desc* seqs; /* num_seqs */
  float* h0;          /* h0_rows x hidden_dim */
  int32_t* per_env_counts;
  float* env_bootstrap;
  uint8_t* env_bootstrap_valid;
} ver_view_host;

typedef struct ver_view_s* ver_view;
ver_status ver_view_upload(ver_ctx ctx, const ver_view_host* h, ver_view* out);
/* fills scalars and sizes of h; pointers untouched */
ver_status ver_view_info(ver_view v, ver_view_host* h);
/* copies every field whose pointer is non-NULL (synchronizes) */
ver_status ver_view_download(ver_view v, ver_view_host* h);
ver_status ver_view_clone(ver_view v, ver_view* out);
ver_status ver_view_destroy(ver_view v);
/* RolloutView::restale (rollout.cpp:15-22) */
ver_status ver_view_restale(ver_view v, uint64_t learner_version);

/* ------------------------------------------------------ rollout store (L2) */
typedef struct {
  int T, N;
  int mode;        /* 0 Fixed, 1 Variable (rollout.hpp:12) */
  int action_kind; /* 0 discrete, 1 continuous */
  int obs_dim, act_dim, hidden_dim;
} ver_rollout_config;

/* A batch of EnvStepRecords (types.hpp:54-67) in arrival order, SoA.
   h_before rows are only read for records that start a sequence (the
   reference copies h_before on every commit but reads it only there,
   rollout.cpp:81 vs :155); h_before == NULL or h_before_valid[i] == 0 means
   "absent" (zeros, rollout.cpp:156). */
typedef struct {
  int n;
  const int32_t* env_index;
  const int64_t* episode_index;   /* may be NULL (0) */
  const int32_t* step_in_episode; /* may be NULL (0) */
  const float* obs;               /* n x obs_dim */
  const int32_t* act_disc;        /* n (discrete) */
  const float* act_cont;          /* n x act_dim (continuous) */
  const float *log_prob, *value, *reward;
  const float* latency;           /* may be NULL (0) */
  const uint8_t* done;
  const float* h_before;          /* n x hidden_dim or NULL */
  const uint8_t* h_before_valid;  /* n or NULL */
  const uint64_t* snapshot_version; /* may be NULL (0) */
} ver_step_batch;

typedef struct ver_rollout_s* ver_rollout;
/* RolloutBuffer(Config) (rollout.cpp:24-31) */
ver_status ver_rollout_create(ver_ctx ctx, const ver_rollout_config* cfg, ver_rollout* out);
ver_status ver_rollout_destroy(ver_rollout r);
/* begin_rollout (rollout.cpp:39-57): commits pending carryovers first, env order */
ver_status ver_rollout_begin(ver_rollout r, uint64_t snapshot_version);
/* append_step (rollout.cpp:59-93) for each record in order; outcomes[i] =
   0 Accepted / 1 RolloutFull (may be NULL).  A ProtocolError stops the batch
   at that record (earlier records stay applied, as in the reference). */
ver_status ver_rollout_append(ver_rollout r, const ver_step_batch* batch, int32_t* outcomes);
ver_status ver_rollout_force_close(ver_rollout r);          /* rollout.cpp:95 */
ver_status ver_rollout_set_bootstrap(ver_rollout r, int env, float value); /* :97-100 */
/* set_bootstrap for n envs at once (same semantics, one call) */
ver_status ver_rollout_set_bootstraps(ver_rollout r, int n, const int32_t* env, const float* value);
ver_status ver_rollout_state(ver_rollout r, int* open, int* committed, int* carryover);
/* close_rollout (rollout.cpp:102-190): device compaction of the arrival log
   into the env-major, sequence-contiguous view */
ver_status ver_rollout_close(ver_rollout r, ver_view* out);

/* Synthetic ragged closed view generated on the device (benchmark workload,
   SURVEY §8d C5): env e holds lengths[e] (>= 1) steps, counter-hash payload,
   done ~ Bernoulli(p_done); discrete actions, T = 0 (no T*N divisibility). */
ver_status ver_view_synth(ver_ctx ctx, const int32_t* lengths, int n_envs, int obs_dim, int hidden_dim,
                          uint64_t seed, float p_done, ver_view* out);

/* backfill_stale (rollout.cpp:208-276) */
ver_status ver_backfill_stale(ver_view view, ver_view prev, int deficit);

/* ---------------------------------------------------------------- GAE (L5) */
/* compute_gae (learner.cpp:11-41): segmented reverse scan on device */
ver_status ver_compute_gae(ver_view v, double gamma, double lambda);

/* ------------------------------------------------------------ sampler (L3) */
typedef struct ver_groups_s* ver_groups;
/* split_minibatches (packseq.cpp:10-16): libstdc++ std::shuffle with
   mt19937_64(seed) of the K sequence ids on the host (O(K)), the greedy deal
   with split tails on the device */
ver_status ver_split_minibatches(ver_view v, int B, uint64_t seed, ver_groups* out);
/* split_in_order (packseq.cpp:18-54) */
ver_status ver_split_in_order(ver_view v, int B, const int32_t* order, int n, ver_groups* out);
ver_status ver_groups_count(ver_groups g, int* B);
/* group b: number of pieces, steps, and (if seqs != NULL) the pieces in deal order */
ver_status ver_groups_get(ver_groups g, int b, int* num_seqs, int* total_steps, ver_seq_desc* seqs);
ver_status ver_groups_destroy(ver_groups g);

typedef struct ver_packed_s* ver_packed;
/* pack (packseq.cpp:56-88) of group b, plus the time-major gather of the
   view's learner fields (learner.cpp:56-70) into the packed order */
ver_status ver_pack(ver_view v, ver_groups g, int b, ver_packed* out);
/* pack of an explicit group (tests / replay) */
ver_status ver_pack_seqs(ver_view v, const ver_seq_desc* seqs, int k, ver_packed* out);
ver_status ver_packed_info(ver_packed p, int* num_seqs, int* max_len, int* total_steps);
ver_status ver_packed_get(ver_packed p, ver_seq_desc* seqs, int32_t* sorted_to_group,
                          int32_t* batch_sizes, int32_t* offsets, int32_t* slots);
/* the gathered, time-major learner fields (obs S x D, act, old log-prob, A, R) */
ver_status ver_packed_get_gathered(ver_packed p, float* obs, int32_t* act_disc, float* act_cont,
                                   float* old_logp, float* adv, float* ret);
ver_status ver_packed_destroy(ver_packed p);

/* ------------------------------------------------------------ policy (L4) */
typedef struct {
  int obs_dim, encoder_dim, hidden_dim;
  int action_kind; /* 0 discrete, 1 continuous */
  int num_actions, act_dim;
} ver_model_config;

/* parameter registry in PolicyParams::tensors() order (nn.cpp:83-95) */
ver_status ver_param_count(const ver_model_config* c, int64_t* count, int* num_tensors);
ver_status ver_param_tensor(const ver_model_config* c, int idx, char name[16], int* rows,
                            int* cols, int64_t* offset);
/* PolicyParams::init (nn.cpp:16-81), host double, one-off setup */
ver_status ver_params_init(const ver_model_config* c, uint64_t seed, double* out);

typedef struct {
  double gamma, gae_lambda, clip;
  int epochs, minibatches;
  double value_loss_coef, is_cap;
} ver_ppo_config; /* PPOConfig (learner.hpp:14-22) */

typedef struct {
  double loss, policy_loss, value_loss, mean_entropy, ratio_sum, clip_count, w_sum, w_max;
  int steps;
} ver_loss_result; /* PPOLossResult (learner.hpp:80-92) */

/* ppo_loss (learner.cpp:52-117): forward_packed + fused loss (+ backward).
   params: host fp32 (P); h0_sorted: host fp32 (k x H); frozen_w: host (S) or
   NULL; grads_out: host (P) or NULL; is_w_out: host (S) or NULL. */
ver_status ver_ppo_loss(ver_ctx ctx, const ver_model_config* c, const float* params, ver_view v,
                        ver_packed p, const ver_ppo_config* cfg, double alpha,
                        const float* h0_sorted, int want_grads, const float* frozen_w,
                        ver_loss_result* out, float* grads_out, float* is_w_out);

/* forward_packed (nn.cpp:219-280) over S packed rows with explicit
   batch_sizes/offsets (L timesteps) and h0 (batch_sizes[0] x H); per-row
   log-prob, entropy and value; all host arrays */
ver_status ver_forward_packed(ver_ctx ctx, const ver_model_config* c, const float* params, int S,
                              const float* obs, const int32_t* act_disc, const float* act_cont,
                              int L, const int32_t* batch_sizes, const int32_t* offsets,
                              const float* h0, float* logp_out, float* ent_out, float* value_out);

/* act (nn.cpp:118-126) on n rows: dist (n x A), value (n), h_new (n x H); host */
ver_status ver_act(ver_ctx ctx, const ver_model_config* c, const float* params, int n,
                   const float* obs, const float* h, float* dist_out, float* value_out,
                   float* h_new_out);

/* adam_step (nn.cpp:291-306) on flat host arrays; step is incremented */
ver_status ver_adam_step(ver_ctx ctx, int64_t count, float* params, const float* grads, float* m,
                         float* v, int64_t* step, double lr);
/* CosineSchedule::lr_at (nn.cpp:308-312) */
double ver_cosine_lr(double base_lr, int64_t total_steps, int64_t consumed);

/* ----------------------------------------------------------- learner (L5) */
typedef struct {
  double alpha, target, lower, upper, lr;
} ver_entropy_controller; /* learner.hpp:29-40 */

typedef struct {
  int64_t update_index;
  int steps, fresh_steps, stale_steps;
  double loss, policy_loss, value_loss, entropy, entropy_loss, mean_ratio, clip_fraction,
      mean_is_weight, max_is_weight, alpha, lr;
} ver_train_stats; /* TrainStats (learner.hpp:55-71) */

typedef struct ver_learner_s* ver_learner;

/* ------------------------------- joint preemption counter */
/* PreemptCoordinator (distributed.hpp:95-128) across one process per GPU: a device
   counter owned by one replica, mapped into the others with CUDA IPC (peer memory
   over NVLink); add is one system-scope atomic, exactly one add per iteration
   reports fired_now, no collective (replicas commit asynchronously). */
typedef struct ver_preempt_s* ver_preempt;
ver_status ver_preempt_create(ver_ctx ctx, ver_preempt* out);          /* owning replica */
ver_status ver_preempt_ipc_handle(ver_preempt p, uint8_t handle_out[64]);
ver_status ver_preempt_open(ver_ctx ctx, const uint8_t handle[64], ver_preempt* out); /* other replicas */
ver_status ver_preempt_destroy(ver_preempt p);
ver_status ver_preempt_start(ver_preempt p, int64_t threshold);        /* start_iteration; <= 0 disables */
ver_status ver_preempt_add(ver_preempt p, int64_t n, int64_t* total, int* fired_now); /* add_steps */
ver_status ver_preempt_state(ver_preempt p, int64_t* total, int* fired);
/* NCCL mode ("global committed-step ncclAllReduce(int64) per
   tick"): every rank creates its own counter on a ctx with NCCL initialised;
   adds (ver_preempt_add, or an attached engine) accumulate locally, and
   ver_preempt_tick -- a collective every rank calls once per collection tick,
   in the same order -- sums the deltas over the ranks, so every rank holds the
   same global count and fires on the same tick.  start runs on every rank. */
ver_status ver_preempt_create_nccl(ver_ctx ctx, ver_preempt* out);
ver_status ver_preempt_tick(ver_preempt p, int64_t* total, int* fired_now);

/* ------------------------------------------ on-disk formats */
/* dump_view / load_view (rollout.cpp:293-432): the reference's JSONL rollout trace
   (one "meta", one "seq" per sequence with its h0 row, one "step" per slot) */
ver_status ver_view_dump_jsonl(ver_view v, const char* path);
ver_status ver_view_load_jsonl(ver_ctx ctx, const char* path, ver_view* out);
/* save_checkpoint / load_checkpoint (bench.cpp:411-441, nn.cpp:314-387): the
   "ver-checkpoint" v1 JSON (params by tensor name, Adam m / v / step, alpha,
   consumed_steps, update_index) */
ver_status ver_learner_save_checkpoint(ver_learner l, const char* path);
ver_status ver_checkpoint_model_config(const char* path, ver_model_config* out);
ver_status ver_learner_load_checkpoint(ver_learner l, const char* path);

/* ------------------------------------- inference engine */
/* InferenceEngine (runtime.hpp:96-160, runtime.cpp:60-229) on the device: the
   policy snapshot, every env's GRU state and the pending records' h_before stay
   in device memory; act (nn.cpp:118-126) runs batched on the GPU and actions are
   sampled there with the reference's counter RNG stream
   CounterRng(seed).stream(0xAC7101, env).stream(obs_episode, obs_step)
   (runtime.cpp:166-169); completed steps are appended to the engine's own
   rollout store (h_before copied device to device, only for records that
   start a sequence). */
typedef struct {
  ver_rollout_config rollout; /* RolloutBuffer config (runtime.cpp:64-74) */
  ver_model_config model;
  uint64_t seed;              /* RuntimeConfig::seed */
} ver_engine_config;

/* InferenceRequest (runtime.hpp:30-42), SoA; NULL optional fields read as 0 */
typedef struct {
  int n;
  const int32_t* env_index;
  const float* obs;           /* n x obs_dim */
  const float* reward;
  const uint8_t* done;
  const uint8_t* first;       /* initial request after reset: completes nothing */
  const float* latency;
  const int64_t* obs_episode;
  const int32_t* obs_step;
} ver_request_batch;

/* InferenceEngine::BatchResult (runtime.hpp:102-106); the dispatches go to the
   caller's arrays (env, discrete action or act_dim floats), n_dispatch of them */
typedef struct {
  int n_dispatch;
  int new_commits;
  int closed_now;
  int preempt_fired; /* attached counter: the group has fired (this rollout was force-closed) */
} ver_batch_result;

typedef struct ver_engine_s* ver_engine;
/* InferenceEngine(cfg, snapshot) (runtime.cpp:76-80): params in tensors() order */
ver_status ver_engine_create(ver_ctx ctx, const ver_engine_config* cfg, const float* params, uint64_t version,
                             ver_engine* out);
ver_status ver_engine_destroy(ver_engine e);
/* set_snapshot (runtime.cpp:82): from host params, or device to device from a learner */
ver_status ver_engine_set_snapshot(ver_engine e, const float* params, uint64_t version);
ver_status ver_engine_set_snapshot_learner(ver_engine e, ver_learner l, uint64_t version);
/* begin_rollout (runtime.cpp:84-113): dispatch arrays hold >= N entries */
ver_status ver_engine_begin_rollout(ver_engine e, ver_batch_result* res, int32_t* disp_env, int32_t* disp_act,
                                    float* disp_act_cont);
/* process_batch (runtime.cpp:192-215): dispatch arrays hold >= reqs->n entries */
ver_status ver_engine_process_batch(ver_engine e, const ver_request_batch* reqs, ver_batch_result* res,
                                    int32_t* disp_env, int32_t* disp_act, float* disp_act_cont);
ver_status ver_engine_force_close(ver_engine e);        /* runtime.hpp:120 */
/* Joint preemption (distributed.hpp:95-128, runtime.cpp:592-599): each batch's
   commits are added to `counter` by the batch's sampling kernel (one
   system-scope atomic on the owner's device word through peer memory, or the
   local delta of an NCCL-mode counter), and the group's fired flag comes back
   with the actions in mapped host memory; the first batch that sees it fired
   force-closes this engine's rollout (closed_now = 1).  NULL detaches. */
ver_status ver_engine_attach_preempt(ver_engine e, ver_preempt counter);
ver_status ver_engine_finalize_bootstraps(ver_engine e); /* runtime.cpp:217-229 */
ver_status ver_engine_close(ver_engine e, ver_view* out); /* runtime.cpp:231-234 */
ver_status ver_engine_state(ver_engine e, int* open, int* committed, int* capacity, int* carryover,
                            int* active_envs);
/* every env's current GRU state, N x hidden_dim (tests) */
ver_status ver_engine_hidden(ver_engine e, float* h_out);
/* Learner(params, cfg, entropy, schedule, run_seed) (learner.cpp:43-50) */
ver_status ver_learner_create(ver_ctx ctx, const ver_model_config* c, const float* params,
                              const ver_ppo_config* cfg, const ver_entropy_controller* ec,
                              double base_lr, int64_t total_steps, uint64_t run_seed,
                              ver_learner* out);
ver_status ver_learner_destroy(ver_learner l);
/* gradient AllReduce over the ctx's NCCL communicator before every Adam step
   (grad_hook / entropy_hook -> AllReduce::average, distributed.cpp:152-157):
   one ncclAllReduce(ncclAvg) of the P gradients + the minibatch mean entropy.
   Runs whenever the ctx has a communicator, a 1-rank one included. */
ver_status ver_learner_enable_allreduce(ver_learner l, int enable);
/* Learner::grad_hook (learner.hpp:119-120, called at learner.cpp:137): once per
   minibatch, between backward and Adam, on the calling host thread.  dev_grads
   holds `count` = P fp32 gradients in the library's device layout (element-wise
   reducers are layout-agnostic; ver_param_device_index maps tensors() order to
   it) on the ctx's device; `stream` is the ctx stream (cudaStream_t).  The hook
   averages in place, ordered on `stream` (enqueue on it, or finish before
   returning).  Non-zero return fails the update (VER_ERR_CONFIG).  NULL clears.
   The built-in NCCL reducer (ver_learner_enable_allreduce) takes precedence. */
typedef int (*ver_grad_hook)(void* user, float* dev_grads, int64_t count, uint64_t stream);
ver_status ver_learner_set_grad_hook(ver_learner l, ver_grad_hook fn, void* user);
/* Learner::entropy_hook (learner.hpp:121-122, called at learner.cpp:142): the
   minibatch mean entropy (one fp32 on the device) that drives the alpha update;
   the hook replaces it with the cross-replica mean, same rules as above. */
typedef int (*ver_entropy_hook)(void* user, float* dev_entropy, uint64_t stream);
ver_status ver_learner_set_entropy_hook(ver_learner l, ver_entropy_hook fn, void* user);
/* index_out[k] = device-layout position of tensors()-order parameter k (P entries) */
ver_status ver_param_device_index(const ver_model_config* c, int64_t* index_out);
/* Learner::update (learner.cpp:146-193).  stats may be NULL: then the stats are
   not returned.  The call synchronizes once at the end (the reference's
   per-minibatch non-finite errors, learner.cpp:111 and :139-140, are latched on
   the device and raised here with the reference's message and state). */
ver_status ver_learner_update(ver_learner l, ver_view v, ver_train_stats* stats);
/* Learner::batch_h0 (learner.cpp:119-130): h0 rows for packed batch (k x H) */
ver_status ver_learner_batch_h0(ver_learner l, ver_view v, ver_packed p, float* h0_out);
ver_status ver_learner_get_params(ver_learner l, float* out);
ver_status ver_learner_set_params(ver_learner l, const float* in);
ver_status ver_learner_get_adam(ver_learner l, float* m, float* v, int64_t* step);
ver_status ver_learner_set_adam(ver_learner l, const float* m, const float* v, int64_t step);
ver_status ver_learner_get_state(ver_learner l, double* alpha, int64_t* consumed_steps,
                                 int64_t* update_index);
ver_status ver_learner_set_state(ver_learner l, double alpha, int64_t consumed_steps,
                                 int64_t update_index);
/* per-phase device time of the last update, ms, from CUDA events on the ctx
   stream: gae, sampler (split + pack + gather), replay (batch_h0), forward,
   loss, backward, allreduce, adam, then the recurrence kernels alone
   (rec_fwd nested in forward, rec_bwd nested in backward) and the tcgen05
   GEMM launches alone (gemm_fwd / gemm_bwd, nested likewise); n in/out */
ver_status ver_learner_last_timing(ver_learner l, float* ms, int* n);
/* number of timed intervals (kernel launches for rec_fwd / rec_bwd) behind each
   phase of ver_learner_last_timing; n in/out */
ver_status ver_learner_last_timing_counts(ver_learner l, int* counts, int* n);
/* Algorithmic FLOPs (2 M N K per launch) of the tcgen05 GEMM launches of the last
   update, per phase of ver_learner_last_timing (nonzero for gemm_fwd / gemm_bwd
   only); n in/out.  Bench-only instrumentation, like the timing above. */
ver_status ver_learner_last_flop(ver_learner l, double* flop, int* n);

/* Measurement: device time (CUDA events, averaged over reps) of compute_gae on
   v and of the time-major gather of all B minibatches of one
   split_minibatches(v, B, seed) deal.  ms_out[0] = GAE call (scan kernel, its
   counter resets and the missing-bootstrap check), ms_out[1] = gather launches;
   ms_out[2] / ms_out[3] = the GAE scan kernel / the gather kernels alone
   (events around the launches).  ms_out holds 4 floats. */
ver_status ver_bench_gae_gather(ver_view v, double gamma, double lambda, int B, uint64_t seed, int reps,
                                float* ms_out);

/* Diagnostic: C (M x N, row-major) = op(A) op(B) through the library's GEMM
   path (op(A) = A^T if transA: A stored K x M; op(B) = B^T if transB: B stored
   N x K).  engine: 0 fp32 SIMT, 1 tcgen05 3xTF32, 2 tcgen05 1xTF32;
   splitk > 1 uses the deterministic split-K partial + reduce path. */
ver_status ver_debug_gemm(ver_ctx ctx, int engine, int transA, int transB, int M, int N, int K,
                          const float* A, int lda, const float* B, int ldb, float* C, int splitk);
/* Measurement: average device time (CUDA events on the ctx stream, after one
   warm-up) of `reps` GEMMs of the shape above on library-allocated operands
   (contents arbitrary; no host copies).  ms_out[0] = ms per GEMM. */
ver_status ver_debug_gemm_time(ver_ctx ctx, int engine, int transA, int transB, int M, int N, int K, int splitk,
                               int reps, float* ms_out);
/* debug: tcgen05 GEMM wait-cycle counters of the launches in between (on = 1
   zeroes + enables, on = 0 disables; out[16] = current sums, may be NULL) */
ver_status ver_debug_gemm_prof(ver_ctx ctx, int on, unsigned long long* out);

/* ------------------------------------------------ replica driver (L7, DD-PPO) */
/* The learner section of ReplicaGroup::replica_main (distributed.cpp:208-264),
   one process per GPU.  Collectives default to NCCL on the ctx communicator
   (ver_ctx_init_nccl; identity without one); a caller may supply its own
   host-side reducers instead (all three, blocking, 0 = success). */
typedef struct {
  void* user;
  int (*sum_i64)(void* user, int64_t* host_inout, int n);
  int (*mean_f64)(void* user, double* host_inout, int n);
  int (*allgather_f64)(void* user, const double* host_in, int n, double* host_out); /* nranks*n */
  int nranks, rank;
} ver_replica_comm;

typedef struct {
  int T, N;               /* per-replica rollout shape; S_max = T*N*nranks (:249) */
  int preempt;            /* 0 None, 1 Optimal (PreemptMode, distributed.hpp:34); FixedFraction is collection-side */
  int per_replica_budget; /* ablation: threshold / R per replica (:257-259) */
} ver_replica_config;

typedef struct {
  int64_t iteration;
  int rank;
  int deficit, stale_steps;
  int64_t global_consumed_before; /* consumed_steps handed to the learner (:228) */
  int64_t global_fresh;           /* fresh steps summed over replicas (:221-226) */
  double learn_time, mean_learn_time; /* this replica's / the pooled LT (:233-235, :247) */
  int64_t next_threshold;         /* S* for the next iteration, 0 = no preemption */
  int64_t per_replica_threshold;  /* S* / R under per_replica_budget, else 0 */
  ver_train_stats train;
} ver_iteration_result; /* IterationResult (distributed.hpp:138-147) */

typedef struct ver_replica_s* ver_replica;
/* comm == NULL: NCCL on ctx */
ver_status ver_replica_create(ver_ctx ctx, ver_learner learner, const ver_replica_config* cfg,
                              const ver_replica_comm* comm, ver_replica* out);
ver_status ver_replica_destroy(ver_replica r);
/* the joint counter whose start_iteration this replica group drives (rank 0 starts it) */
ver_status ver_replica_attach_preempt(ver_replica r, ver_preempt counter);
/* one iteration after collection closed `view` (collect_wall_time < 0: the
   view's own collect_wall_time): global step count, backfill from the previous
   rollout, Learner::update, pooled tau / LT -> S*, counter start, barrier */
ver_status ver_replica_learn(ver_replica r, ver_view view, double collect_wall_time, int last_iteration,
                             ver_iteration_result* out);
ver_status ver_replica_state(ver_replica r, int64_t* global_consumed, int64_t* iteration, int* has_prev);

/* ------------------------------------------------------- distributed (L7) */
/* estimate_time (distributed.cpp:24-51), bisection with device counting */
ver_status ver_estimate_time(ver_ctx ctx, const double* tau, int n, int64_t max_steps,
                             int64_t steps, double* out);
/* optimal_preempt_steps (distributed.cpp:53-65), sort formulation on device
   (the equivalence test_distributed.cpp:16-37,122-132 pins) */
ver_status ver_optimal_preempt_steps(ver_ctx ctx, const double* tau, int n, double learn_time,
                                     int64_t max_steps, int64_t* out);

#ifdef __cplusplus
}
#endif
#endif
