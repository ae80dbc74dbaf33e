/*
 * ver_oracle.h — C shim over the CPU double-precision restatement of the
 * VER learner hot path (oracle/ver_oracle.cpp).
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in paper_2210_05064_b200/ links, loads or
 * calls this library.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may use it, and only as the checker or
 * the timed CPU baseline.
 *
 * Parity status: the reference (/root/reference/proj, C++20 + Eigen3) cannot be
 * built in this image (Eigen3, doctest and CLI11 are absent, no network; see
 * DESIGN.md "Oracle").  The oracle is therefore a line-by-line restatement,
 * pinned against every known-answer / property test the reference holds for
 * this path (tests/test_oracle_*.py port tests/test_{rollout,packseq,learner,
 * nn,tape,distributed}.cpp).
 *
 * Conventions: all functions return 0 on success, 1 on a reference
 * ProtocolError (message via vo_last_error()), 2 on ConfigError / bad args.
 */
#ifndef VER_ORACLE_H
#define VER_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* vo_last_error(void);

/* ---- rng.hpp:16-75 ---------------------------------------------------- */
uint64_t vo_splitmix64(uint64_t x);
uint64_t vo_mix(uint64_t a, uint64_t b);

/* ---- RolloutView field block (rollout.hpp:33-78), double precision ------ */
typedef struct {
  int T, N, action_kind, obs_dim, act_dim, hidden_dim;
  int size, num_seqs;
  int deficit, stale_steps, replayed_steps;
  uint64_t snapshot_version;
  double collect_wall_time;
  /* per slot (size) */
  double* obs;          /* size x obs_dim */
  double* act_cont;     /* size x act_dim (continuous) */
  int32_t* act_disc;    /* size (discrete) */
  double *log_prob, *value, *reward, *latency, *advantage, *returns;
  uint8_t *done, *stale, *replayed;
  int32_t *env_index, *seq_of_slot, *step_in_episode;
  int64_t* episode_index;
  uint64_t* version;
  /* per sequence (num_seqs) */
  int32_t* seqs;        /* num_seqs x 8: seq_id, env, length, start_offset, h0_index,
                           stale, parent_start_offset, skip */
  double* h0;           /* (rows of h0) x hidden_dim; rows == num_seqs for close_rollout */
  int h0_rows;
  /* per env (N) */
  int32_t* per_env_counts;
  double* env_bootstrap;
  uint8_t* env_bootstrap_valid;
} vo_view_data;

typedef struct vo_view_s* vo_view;
int vo_view_create(const vo_view_data* d, vo_view* out);
/* fills scalar members and sizes; pointer members untouched */
int vo_view_info(vo_view v, vo_view_data* d);
/* copies every field whose pointer is non-NULL */
int vo_view_read(vo_view v, vo_view_data* d);
int vo_view_clone(vo_view v, vo_view* out);
void vo_view_destroy(vo_view v);

/* ---- RolloutBuffer (rollout.hpp:87-142) --------------------------------- */
typedef struct vo_rollout_s* vo_rollout;
int vo_rollout_create(int T, int N, int mode /*0 fixed,1 variable*/, int action_kind,
                      int obs_dim, int act_dim, int hidden_dim, vo_rollout* out);
void vo_rollout_destroy(vo_rollout r);
int vo_rollout_begin(vo_rollout r, uint64_t snapshot_version);
/* one EnvStepRecord (types.hpp:54-67); h_before may be NULL (absent);
   outcome: 0 Accepted, 1 RolloutFull */
int vo_rollout_append(vo_rollout r, int env, int64_t episode, int step_in_episode,
                      const double* obs, int act_index, const double* act_values,
                      double log_prob, double value, double reward, int done,
                      double latency, const double* h_before, uint64_t snapshot_version,
                      int* outcome);
/* n records in SoA arrays (same fields), applied in order */
int vo_rollout_append_batch(vo_rollout r, int n, const int32_t* env, const int64_t* episode,
                            const int32_t* step_in_episode, const double* obs,
                            const int32_t* act_index, const double* act_values,
                            const double* log_prob, const double* value, const double* reward,
                            const uint8_t* done, const double* latency,
                            const double* h_before, const uint8_t* h_before_valid,
                            const uint64_t* snapshot_version, int32_t* outcomes);
int vo_rollout_force_close(vo_rollout r);
int vo_rollout_set_bootstrap(vo_rollout r, int env, double value);
int vo_rollout_state(vo_rollout r, int* open, int* committed, int* carryover);
int vo_rollout_close(vo_rollout r, vo_view* out);

/* rollout.cpp:208-276 */
int vo_backfill_stale(vo_view view, vo_view prev, int deficit);
/* rollout.cpp:15-22 */
int vo_view_restale(vo_view view, uint64_t learner_version);

/* ---- packseq (packseq.hpp:35-44) ---------------------------------------- */
typedef struct vo_groups_s* vo_groups;
int vo_split_minibatches(vo_view v, int B, uint64_t seed, vo_groups* out);
int vo_split_in_order(vo_view v, int B, const int32_t* perm, int n, vo_groups* out);
/* libstdc++ std::shuffle of iota(n) with mt19937_64(seed) (packseq.cpp:11-14) */
int vo_shuffle_perm(int n, uint64_t seed, int32_t* perm_out);
int vo_groups_count(vo_groups g, int* B);
int vo_groups_get(vo_groups g, int b, int* num_seqs, int* total_steps, int32_t* seqs_out /*k x 8*/);
void vo_groups_destroy(vo_groups g);

typedef struct vo_packed_s* vo_packed;
int vo_pack(const int32_t* seqs /*k x 8*/, int k, vo_packed* out);
int vo_packed_info(vo_packed p, int* num_seqs, int* max_len, int* total_steps);
int vo_packed_get(vo_packed p, int32_t* seqs_out, int32_t* sorted_to_group,
                  int32_t* batch_sizes, int32_t* offsets, int32_t* slots);
void vo_packed_destroy(vo_packed p);

/* ---- nn (nn.hpp) --------------------------------------------------------- */
typedef struct {
  int obs_dim, encoder_dim, hidden_dim, action_kind /*0 discrete,1 continuous*/;
  int num_actions, act_dim;
} vo_model_config;

int vo_param_count(const vo_model_config* c, int64_t* count, int* num_tensors);
int vo_param_tensor(const vo_model_config* c, int idx, char* name /*>=16*/, int* rows,
                    int* cols, int64_t* offset);
/* PolicyParams::init (nn.cpp:16-81), flat tensors() order */
int vo_params_init(const vo_model_config* c, uint64_t seed, double* out);
/* act (nn.cpp:118-126): n rows */
int vo_act(const vo_model_config* c, const double* params, int n, const double* obs,
           const double* h, double* dist_out, double* value_out, double* h_new_out);
/* forward_packed (nn.cpp:219-280): per packed row log-prob, entropy, value */
int vo_forward_packed(const vo_model_config* c, const double* params, int S, const double* obs,
                      const int32_t* act_disc, const double* act_cont, int L,
                      const int32_t* batch_sizes, const int32_t* offsets, const double* h0,
                      int h0_rows, double* logp_out, double* ent_out, double* value_out);
double vo_categorical_log_prob(const double* logits, int A, int action);
double vo_categorical_entropy(const double* logits, int A);

/* ---- learner (learner.hpp) ---------------------------------------------- */
typedef struct {
  double gamma, gae_lambda, clip;
  int epochs, minibatches;
  double value_loss_coef, is_cap;
} vo_ppo_config;

typedef struct {
  double loss, policy_loss, value_loss, mean_entropy, ratio_sum, clip_count, w_sum, w_max;
  int steps;
} vo_loss_result;

int vo_compute_gae(vo_view v, double gamma, double lambda);
int vo_gae_arrays(const float* reward, const float* value, const uint8_t* done, const int32_t* env,
                  const uint8_t* replayed, int S, int N, const float* boot, const uint8_t* boot_valid,
                  double gamma, double lambda, int reference_loop, float* adv, float* ret);
/* OpenMP threads of the oracle's GEMMs / reductions (bit-identical for any count; default 1) */
int vo_set_num_threads(int n);
int vo_get_num_threads(void);
/* 1: `rows` backward accumulates its slice only (same sums; test speed); 0 (default): reference's full-size scatter */
int vo_set_sparse_rows(int on);

/* ppo_loss (learner.cpp:52-117) over packed batch p; h0_sorted k x H;
   grads_out (P) and is_w_out (S) may be NULL; frozen_w may be NULL */
int vo_ppo_loss(const vo_model_config* c, const double* params, vo_view v, vo_packed p,
                const vo_ppo_config* cfg, double alpha, const double* h0_sorted,
                int want_grads, const double* frozen_w, vo_loss_result* out,
                double* grads_out, double* is_w_out);

typedef struct {
  double alpha, target, lower, upper, lr;
} vo_entropy_controller;

typedef struct {
  int64_t update_index;
  int steps, fresh_steps, stale_steps;
  double loss, policy_loss, value_loss, entropy, entropy_loss, mean_ratio, clip_fraction,
      mean_is_weight, max_is_weight, alpha, lr;
} vo_train_stats;

typedef void (*vo_grad_hook_fn)(double* grads, int64_t count, void* user);
typedef double (*vo_entropy_hook_fn)(double h, void* user);

typedef struct vo_learner_s* vo_learner;
int vo_learner_create(const vo_model_config* c, const double* params, const vo_ppo_config* cfg,
                      const vo_entropy_controller* ec, double base_lr, int64_t total_steps,
                      uint64_t run_seed, vo_learner* out);
void vo_learner_destroy(vo_learner l);
int vo_learner_set_hooks(vo_learner l, vo_grad_hook_fn g, vo_entropy_hook_fn e, void* user);
int vo_learner_update(vo_learner l, vo_view v, vo_train_stats* out);
/* timing helper for the CPU baseline: GAE + the first `max_minibatches`
   minibatches of the update loop exactly as Learner::update runs them */
int vo_learner_update_partial(vo_learner l, vo_view v, int max_minibatches, vo_train_stats* out);
int vo_learner_batch_h0(vo_learner l, vo_view v, vo_packed p, double* h0_out);
int vo_learner_get_params(vo_learner l, double* out);
int vo_learner_set_params(vo_learner l, const double* in);
int vo_learner_get_adam(vo_learner l, double* m, double* v, int64_t* step);
int vo_learner_get_state(vo_learner l, double* alpha, int64_t* consumed, int64_t* update_index);
int vo_learner_set_state(vo_learner l, double alpha, int64_t consumed, int64_t update_index);

/* nn.cpp:291-312, learner.hpp:36-39 */
int vo_adam_step(int64_t count, double* params, const double* grads, double* m, double* v,
                 int64_t* step, double lr);
double vo_cosine_lr(double base_lr, int64_t total_steps, int64_t consumed);
double vo_entropy_update(vo_entropy_controller* ec, double mean_entropy);

/* ---- distributed (distributed.cpp:16-65) -------------------------------- */
int vo_estimate_time(const double* tau, int n, int64_t max_steps, int64_t steps, double* out);
/* the reference's exact O(S_max * I * N) scan */
int vo_optimal_preempt_steps(const double* tau, int n, double learn_time, int64_t max_steps,
                             int64_t* out);
/* the merge/sort formulation the reference's own test pins as equivalent
   (test_distributed.cpp:16-37) */
double vo_merged_time(const double* tau, int n, int64_t steps);
int vo_optimal_preempt_steps_sorted(const double* tau, int n, double learn_time,
                                    int64_t max_steps, int64_t* out);

#ifdef __cplusplus
}
#endif
#endif
