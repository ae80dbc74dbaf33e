// policy.cuh — encoder + GRU + heads (nn.cpp:219-280) on the device.
//
// Device parameter layout (one flat fp32 buffer; gradients, Adam moments and
// the NCCL AllReduce use the same layout):
//   w1[D*E] b1[E] w2[E*E] b2[E]
//   wx[E*3H] ux[H*3H] bx[3H]      GRU gates interleaved per unit: column 3u+g,
//                                 g = 0 r, 1 z, 2 n  (so one output tile holds
//                                 all three gates of its units)
//   wh[H*(A+1)] bh[A+1]           policy head columns 0..A-1, value column A
//   log_std[A]                    (continuous only)
// The reference's tensors() order (nn.cpp:83-95) is a fixed permutation of
// this layout, applied only at the C-ABI (params/grads/Adam get/set).
#pragma once

#include <cuda_fp16.h>

#include "packed.cuh"

struct ver_learner_s;

namespace verg {

struct Model {
  int D = 0, E = 0, H = 0, A = 0, AH = 0;
  int continuous = 0;
  int64_t P = 0;
  int64_t o_w1, o_b1, o_w2, o_b2, o_wx, o_ux, o_bx, o_wh, o_bh, o_ls;
  std::vector<int64_t> dev_index;  // tensors()-order flat index -> device index
  static Model make(const ver_model_config& c);
};

// max |x| over n floats into *out (float bits; atomicMax, *out zeroed by the caller)
__global__ void maxabs_kernel(int64_t n, const float* __restrict__ x, unsigned* __restrict__ out);

struct LossStats {  // device-side per-minibatch loss statistics (double)
  double loss, policy_loss, value_loss, mean_entropy, ratio_sum, clip_count, w_sum, w_max;
  double steps;
};

struct Workspace {
  Ctx* ctx = nullptr;
  size_t rows = 0;
  DBuf<float> e1, enc, xp, hu, gates, hidden, hprev;  // forward
  DBuf<float> dhidden, dhead, g, dpre, dhu, carry, dpre2, dpre1;  // backward
  DBuf<float> splitk;                                   // split-K partials
  DBuf<double> part;                                    // loss partials
  DBuf<float> wpart;                                    // head-weight partials
  DBuf<float> is_w;
  DBuf<unsigned> bar;                                   // grid barrier of the recurrence
  DBuf<long long> trace;                                // VER_REC_TRACE experiments only
  DBuf<float> step;                                     // per-step GEMM output of the big recurrence steps
  DBuf<float> sgsteps, sgmaps;                          // stepgemm.cu: step table, per-step A tensor maps
  DBuf<unsigned long long> hx;                          // K-split kernels: tagged h / dhU rows of short steps
  DBuf<float> wlo;                                      // lo = x - trunc_tf32(x) of the parameters (3xTF32 B operands)
  // fp16x2 operands (tc_gemm.cuh F16): the forward weights transposed to K-major
  // (wx: 3H x E, w2: E x E) as scaled hi / lo halves, refreshed with wlo; per
  // weight the max |w| (float bits) and the GEMM's 1 / (s_A s_B); the activation
  // operand's halves (enc / e1, fixed scale 2^14: tanh outputs)
  DBuf<__half> w16hi, w16lo, a16hi, a16lo;
  DBuf<__half> h16hi, h16lo;                            // fp16x2 halves of h (forward pair steps; h0's at the end)
  DBuf<unsigned> hmax;                                  // max |h0| bits of the current forward pair launch
  DBuf<float> hsc;                                      // [s_h, 1 / (s_h s_U)] of that launch
  bool f16_fwd = false;  // this forward's weight halves are fresh (policy_forward): fp16x2 pair steps
  DBuf<unsigned> w16max;
  DBuf<unsigned> gmax;  // max |dpre|, max |dpre2| (float bits) of this backward: the fp16x2 data-gradient scales
  DBuf<float> w16inv;
  // wlo holds the lo of wlo_src's current values unless wlo_stale; owners whose
  // parameters change in place (the learner's Adam) leave it stale (the default)
  const float* wlo_src = nullptr;
  bool wlo_stale = true;
  bool wlo_keep = false;  // the caller promises the parameters stay unchanged until it clears this
  unsigned hx_epoch = 0;                                // tag epoch, one per K-split launch
  void ensure(const Model& m, size_t S, bool train);
};

// Forward of the encoder + GRU over a packed batch of S rows.
//   obs: S x D (packed), h0: bs[0] x H, d_bs/d_offs: device batch sizes /
//   offsets of the L timesteps.  store: keep e1/enc/xp/hUn/gates/hprev for
//   the backward pass.
//   h_bs: optional host copy of the batch sizes; with it the tail of short
//   timesteps runs on the single-cluster kernels (recurrence.cu).
void policy_forward(Ctx* c, const Model& m, const float* params, int S, const float* obs,
                    const float* h0, int L, const int32_t* d_bs, const int32_t* d_offs, Workspace& ws,
                    bool store, const int32_t* h_bs = nullptr, const int32_t* h_offs = nullptr);

// Persistent recurrence kernels (recurrence.cu)
void gru_forward_recurrence(Ctx* c, const Model& m, const float* params, int L, const int32_t* d_bs,
                            const int32_t* d_offs, Workspace& ws, const float* h0, bool store,
                            const int32_t* h_bs = nullptr, const int32_t* h_offs = nullptr);
void gru_backward_recurrence(Ctx* c, const Model& m, const float* params, int L, const int32_t* d_bs,
                             const int32_t* d_offs, Workspace& ws, const int32_t* h_bs = nullptr,
                             const int32_t* h_offs = nullptr);
// Big recurrence steps on the tensor cores: the timesteps with many rows
// (forward: steps [0, t_end); backward: steps t_top .. 1) in one persistent
// cooperative launch per minibatch and direction, a split-K 3xTF32 tcgen05
// GEMM phase and a gate phase per step (stepgemm.cu).  Host batch sizes /
// offsets required.
int gru_big_steps(Ctx* c, const Model& m, const int32_t* h_bs, int L, bool backward);
void gru_forward_big_persist(Ctx* c, const Model& m, const float* params, int t_end, const int32_t* h_bs,
                             const int32_t* h_offs, Workspace& ws, const float* h0, bool store);
void gru_backward_big_persist(Ctx* c, const Model& m, const float* params, int t_top, const int32_t* h_bs,
                              const int32_t* h_offs, Workspace& ws);

// Fused heads + PPO loss (learner.cpp:77-115) + head backward.  Writes
// dhidden, the head/log_std gradient slots of `grad`, the per-row IS weights
// and the LossStats at *stats (device).  alpha: device double.
struct LossArgs {
  const float* act_cont;
  const int32_t* act_disc;
  const float* old_logp;
  const float* adv;
  const float* ret;
  const float* frozen_w;  // may be null
  double clip, is_cap, vcoef;
  const double* alpha;
};
void policy_loss(Ctx* c, const Model& m, const float* params, int S, const LossArgs& a, Workspace& ws,
                 float* grad, LossStats* stats, bool want_grads);

// Backward through the recurrence and the encoder; fills the remaining
// gradient slots of `grad` (device layout).  Requires policy_forward(store).
void policy_backward(Ctx* c, const Model& m, const float* params, int S, const float* obs, int L,
                     const int32_t* d_bs, const int32_t* d_offs, Workspace& ws, float* grad,
                     const int32_t* h_bs = nullptr, const int32_t* h_offs = nullptr);

// Per-row log-prob / entropy / value of the heads (nn.cpp:251-278)
void policy_rows(Ctx* c, const Model& m, const float* params, int S, const float* hidden,
                 const int32_t* act_disc, const float* act_cont, float* logp, float* ent, float* value);

// Heads on n rows of hidden: out n x (A+1) = hidden * wh + bh
void policy_heads(Ctx* c, const Model& m, const float* params, int n, const float* hidden, float* out);

// Adam (nn.cpp:291-306) + log_std clamp (nn.cpp:105-109) + finiteness flag.
// guard (learner): skip the step when guard->loss is non-finite or
// nonfinite_flag[1] (an earlier minibatch failed) is set; NULL = always step.
void adam_update(Ctx* c, const Model& m, float* params, const float* grad, float* mom, float* vel,
                 int64_t step, double lr, int* nonfinite_flag, const LossStats* guard = nullptr);

// Host-double parameter init in tensors() order (nn.cpp:16-81).
void init_params_host(const ver_model_config& c, uint64_t seed, double* out);

// tensors()-order host parameters -> device layout (learner.cu)
void to_device_layout(const Model& m, const float* tensors_order, std::vector<float>& dev);
// the learner's device parameters (learner.cu), for the inference engine's snapshot
const float* learner_device_params(ver_learner_s* l, Ctx** ctx, int64_t* count);

}  // namespace verg
