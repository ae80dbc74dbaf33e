// learner.cu — Learner::update (learner.cpp:146-193) and its pieces on the
// device: GAE -> per epoch split -> per minibatch pack/gather -> split-tail
// h0 replay (learner.cpp:119-130) -> forward -> fused loss -> backward ->
// NCCL gradient AllReduce (DD-PPO, distributed.cpp:86-116, with the mean
// entropy riding in the same buffer, :103-116) -> Adam + log_std clamp ->
// entropy-controller update (learner.hpp:36-39).  Parameters, Adam moments,
// alpha and all statistics stay on the device for the whole update; the
// host reads back once at the end.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>

#include "policy.cuh"

namespace verg {

void compute_gae(DView& V, double gamma, double lambda);
DGroups* split_minibatches(DView& V, int B, uint64_t seed);
std::vector<int32_t> shuffle_perm(int n, uint64_t seed);

namespace {
inline uint64_t splitmix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
inline uint64_t mix64(uint64_t a, uint64_t b) {
  return splitmix(a ^ (0x9e3779b97f4a7c15ull + (b << 6) + (b >> 2) + splitmix(b)));
}
}  // namespace

enum Phase {
  PH_GAE, PH_SAMPLER, PH_REPLAY, PH_FORWARD, PH_LOSS, PH_BACKWARD, PH_ALLREDUCE, PH_ADAM,
  PH_REC_FWD, PH_REC_BWD,  // recurrence kernels alone (nested in forward / backward)
  PH_GEMM_FWD, PH_GEMM_BWD,  // tcgen05 GEMM launches alone (nested in forward / backward)
  PH_N
};

struct Learner {
  Ctx* ctx = nullptr;
  ver_model_config mc{};
  Model m;
  ver_ppo_config cfg{};
  ver_entropy_controller ec{};
  double base_lr = 2.5e-4;
  int64_t total_steps = 1;
  uint64_t run_seed = 0;
  int64_t consumed = 0, update_index = 0, adam_step = 0;
  bool allreduce = false;
  // grad_hook / entropy_hook (learner.hpp:119-122): user reducers on the device
  // buffers, called between backward and Adam (learner.cpp:137, :142)
  ver_grad_hook grad_hook = nullptr;
  void* grad_user = nullptr;
  ver_entropy_hook ent_hook = nullptr;
  void* ent_user = nullptr;
  DBuf<float> params, grad, mom, vel;
  DBuf<double> alpha;        // entropy coefficient (device)
  DBuf<double> acc;          // per-update statistics accumulator
  DBuf<LossStats> lstats;
  // [0] non-finite parameters after this minibatch's Adam step (atomicOr in Adam),
  // [1] stopped (set once by the guard; later Adam / alpha updates are skipped),
  // [2] minibatch index of the failure, [3] 1 = non-finite loss, 2 = non-finite params
  DBuf<int> flags;
  Workspace ws, wr;          // minibatch / h0-replay workspaces
  DBuf<float> h0s;           // sorted h0 of the current minibatch
  DBuf<float> robs, rh0;     // split-tail replay inputs
  // sampler context: splits / packs run on their own stream, so pack b+1 (with
  // its host round trips) overlaps minibatch b on ctx->stream
  Ctx side{};
  ~Learner() {
    if (side.stream) {
      cudaStreamSynchronize(side.stream);
      cudaStreamDestroy(side.stream);
    }
    if (side.pinned) cudaFreeHost(side.pinned);
  }
  // per-phase device timing of the last update (events on ctx->stream)
  std::vector<std::tuple<int, cudaEvent_t, cudaEvent_t>> evlog;
  std::vector<std::pair<int, cudaEvent_t>> open;
  float phase_ms[PH_N] = {};
  int phase_n[PH_N] = {};
  double flop_acc[PH_N] = {}, phase_flop[PH_N] = {};  // 2MNK of the tagged tcgen05 GEMMs
  bool timing = true;

  void mark_begin(int phase) {
    if (!timing) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, ctx->stream);
    open.push_back({phase, e});
  }
  void mark_end() {
    if (!timing || open.empty()) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, ctx->stream);
    evlog.emplace_back(open.back().first, open.back().second, e);
    open.pop_back();
  }
  void collect_timing() {
    for (int k = 0; k < PH_N; ++k) phase_ms[k] = 0.f, phase_n[k] = 0, phase_flop[k] = flop_acc[k], flop_acc[k] = 0.0;
    for (auto& [tag, a, b] : evlog) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, a, b);
      phase_ms[tag] += ms;
      phase_n[tag] += 1;
      cudaEventDestroy(a);
      cudaEventDestroy(b);
    }
    evlog.clear();
  }
};

// -------------------------------------------------------------- kernels
__global__ void h0_gather_kernel(const ver_seq_desc* __restrict__ seqs, int k, const float* __restrict__ h0,
                                 int H, float* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)k * H) return;
  const int j = (int)(i / H), u = (int)(i % H);
  out[i] = h0[(size_t)seqs[j].h0_index * H + u];
}

// replay batch rows: row offr[t] + i = the obs of view slot parent_i + t (the
// first D floats of its learner record, stride rs)
__global__ void replay_obs_kernel(const int32_t* __restrict__ offr, int L, const int32_t* __restrict__ parent,
                                  int R, const float* __restrict__ vrec, int rs, int D, float* __restrict__ out) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= R) return;
  int lo = 0, hi = L;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (offr[mid] <= p) lo = mid;
    else hi = mid;
  }
  const int t = lo, i = p - offr[t];
  const int s = parent[i] + t;
  for (int d = 0; d < D; ++d) out[(size_t)p * D + d] = vrec[(size_t)s * rs + d];
}
__global__ void replay_h0_kernel(const int32_t* __restrict__ h0_index, int n, const float* __restrict__ vh0, int H,
                                 float* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)n * H) return;
  const int j = (int)(i / H), u = (int)(i % H);
  out[i] = vh0[(size_t)h0_index[j] * H + u];
}
__global__ void replay_final_kernel(const int32_t* __restrict__ last_row, const int32_t* __restrict__ dst, int n,
                                    const float* __restrict__ hidden, int H, float* __restrict__ h0s) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)n * H) return;
  const int j = (int)(i / H), u = (int)(i % H);
  h0s[(size_t)dst[j] * H + u] = hidden[(size_t)last_row[j] * H + u];
}

__global__ void alpha_update_kernel(double* __restrict__ alpha, const LossStats* __restrict__ st,
                                    const float* __restrict__ ent_avg, double target, double lr, double lo,
                                    double hi, int* __restrict__ flags, int mb) {
  // The reference throws per minibatch: ProtocolError on a non-finite loss before
  // backward / hook / Adam (learner.cpp:111), and on non-finite parameters after
  // Adam, before the entropy update (learner.cpp:139-140).  The device loop does
  // not stop, so the first failure latches flags[1]: Adam (adam_kernel) and this
  // update skip from then on, and the host raises the reference's error at the end.
  if (flags[1]) return;
  const bool loss_bad = !isfinite(st->loss), par_bad = flags[0] != 0;
  if (loss_bad || par_bad) {
    flags[1] = 1;
    flags[2] = mb;
    flags[3] = loss_bad ? 1 : 2;
    return;
  }
  // EntropyController::update (learner.hpp:36-39)
  const double h = ent_avg ? (double)*ent_avg : st->mean_entropy;
  double a = *alpha + lr * (target - h);
  *alpha = fmin(fmax(a, lo), hi);
}

// acc: loss, policy, value, entropy, ratio_sum, clip, w_sum, w_max, steps, batches
__global__ void stats_accum_kernel(double* __restrict__ acc, const LossStats* __restrict__ st) {
  acc[0] += st->loss;
  acc[1] += st->policy_loss;
  acc[2] += st->value_loss;
  acc[3] += st->mean_entropy;
  acc[4] += st->ratio_sum;
  acc[5] += st->clip_count;
  acc[6] += st->w_sum;
  acc[7] = fmax(acc[7], st->w_max);
  acc[8] += st->steps;
  acc[9] += 1.0;
}

// ------------------------------------------------------------ batch_h0
// learner.cpp:119-130.  Pieces with skip > 0 (split tails) replay `skip`
// steps of act() from parent_start_offset with the current parameters; all
// tails of a minibatch replay together as one packed GRU forward sorted by
// skip (descending), so the replay costs max(skip) recurrent steps.
// host plan of the replay (depends on the pack only, not on the parameters):
// built once per pack, before the minibatch loop, so the loop has no host sync
static void prepare_replay(Ctx* c, DPacked& P) {
  if (P.rp_ready) return;
  P.rp_ready = true;
  struct Tail {
    int j, skip, parent, h0i;
  };
  std::vector<Tail> tails;
  for (int j = 0; j < P.k; ++j)
    if (P.h_seqs[j].skip > 0)
      tails.push_back({j, P.h_seqs[j].skip, P.h_seqs[j].parent_start_offset, P.h_seqs[j].h0_index});
  P.rp_n = (int)tails.size();
  if (tails.empty()) return;
  std::stable_sort(tails.begin(), tails.end(), [](const Tail& a, const Tail& b) { return a.skip > b.skip; });
  const int n = (int)tails.size();
  const int L = tails[0].skip;
  std::vector<int32_t> bs(L), offs(L);
  int R = 0;
  for (int t = 0, alive = n; t < L; ++t) {
    while (alive > 0 && tails[alive - 1].skip <= t) --alive;
    bs[t] = alive;
    offs[t] = R;
    R += alive;
  }
  std::vector<int32_t> meta(4 * (size_t)n + 2 * (size_t)L);
  for (int i = 0; i < n; ++i) {
    meta[i] = tails[i].parent;
    meta[n + i] = tails[i].h0i;
    meta[2 * n + i] = offs[tails[i].skip - 1] + i;  // row of the last replayed step
    meta[3 * n + i] = tails[i].j;
  }
  std::copy(offs.begin(), offs.end(), meta.begin() + 4 * n);
  std::copy(bs.begin(), bs.end(), meta.begin() + 4 * n + L);
  P.rp_L = L;
  P.rp_R = R;
  P.rp_bs = bs;
  P.rp_offs = offs;
  P.rp_meta.reserve(c, meta.size());
  P.rp_meta.upload(meta.data(), meta.size());  // pageable source: consumed before the call returns
}

static void batch_h0(Learner& Ln, DView& V, DPacked& P, const float* params, float* h0s) {
  Ctx* c = Ln.ctx;
  const int H = V.hidden_dim;
  h0_gather_kernel<<<cdiv((size_t)P.k * H, 256), 256, 0, c->stream>>>(P.seqs.p, P.k, V.h0.p, H, h0s);
  after_launch(c);
  prepare_replay(c, P);
  if (P.rp_n == 0) return;
  const int n = P.rp_n, L = P.rp_L, R = P.rp_R;
  const int32_t* dm = P.rp_meta.p;
  Ln.wr.ensure(Ln.m, R, false);
  Ln.robs.reserve(c, (size_t)R * V.obs_dim);
  Ln.rh0.reserve(c, (size_t)n * H);
  replay_obs_kernel<<<cdiv(R, 256), 256, 0, c->stream>>>(dm + 4 * n, L, dm, R, V.rec.p, V.rs(), V.obs_dim,
                                                         Ln.robs.p);
  after_launch(c);
  replay_h0_kernel<<<cdiv((size_t)n * H, 256), 256, 0, c->stream>>>(dm + n, n, V.h0.p, H, Ln.rh0.p);
  after_launch(c);
  policy_forward(c, Ln.m, params, R, Ln.robs.p, Ln.rh0.p, L, dm + 4 * n + L, dm + 4 * n, Ln.wr, false,
                 P.rp_bs.data(), P.rp_offs.data());
  replay_final_kernel<<<cdiv((size_t)n * H, 256), 256, 0, c->stream>>>(dm + 2 * n, dm + 3 * n, n,
                                                                      Ln.wr.hidden.p, H, h0s);
  after_launch(c);
}

// ---------------------------------------------------------- minibatch
// learner.cpp:132-144
static void run_minibatch(Learner& Ln, DView& V, DPacked& P, double lr, int mb) {
  Ctx* c = Ln.ctx;
  const Model& m = Ln.m;
  const int S = P.total;
  Ln.h0s.reserve(c, (size_t)P.k * m.H);
  Ln.mark_begin(PH_REPLAY);
  batch_h0(Ln, V, P, Ln.params.p, Ln.h0s.p);
  Ln.mark_end();
  Ln.ws.ensure(m, S, true);
  Ln.mark_begin(PH_FORWARD);
  c->rec_tag = PH_REC_FWD;
  c->gemm_tag = PH_GEMM_FWD;
  policy_forward(c, m, Ln.params.p, S, P.obs.p, Ln.h0s.p, P.max_len, P.bs.p, P.offs.p, Ln.ws, true,
                 P.h_bs.data(), P.h_offs.data());
  c->rec_tag = -1;
  c->gemm_tag = -1;
  Ln.mark_end();
  LossArgs la{P.act_cont.p, P.act_disc.p, P.old_logp.p, P.adv.p, P.ret.p, nullptr,
              Ln.cfg.clip, Ln.cfg.is_cap, Ln.cfg.value_loss_coef, Ln.alpha.p};
  Ln.mark_begin(PH_LOSS);
  policy_loss(c, m, Ln.params.p, S, la, Ln.ws, Ln.grad.p, Ln.lstats.p, true);
  Ln.mark_end();
  Ln.mark_begin(PH_BACKWARD);
  c->rec_tag = PH_REC_BWD;
  c->gemm_tag = PH_GEMM_BWD;
  policy_backward(c, m, Ln.params.p, S, P.obs.p, P.max_len, P.bs.p, P.offs.p, Ln.ws, Ln.grad.p,
                  P.h_bs.data(), P.h_offs.data());
  c->rec_tag = -1;
  c->gemm_tag = -1;
  Ln.mark_end();
  // grad_hook -> AllReduce::average, entropy_hook -> average_scalar (distributed.cpp:152-157):
  // the built-in reducer is one ncclAllReduce(avg) of grads + mean entropy (P + 1
  // floats, the entropy at [P]); user hooks see the same device buffers instead
  const bool nccl = Ln.allreduce && c->comm;
  const bool hook_g = nccl || Ln.grad_hook, hook_h = nccl || Ln.ent_hook;
  if (hook_g || hook_h) {
    Ln.mark_begin(PH_ALLREDUCE);
    if (nccl) {
      VER_NCCL(ncclAllReduce(Ln.grad.p, Ln.grad.p, (size_t)m.P + 1, ncclFloat32, ncclAvg, c->comm, c->stream));
    } else {
      const uint64_t st = reinterpret_cast<uint64_t>(c->stream);
      if (Ln.grad_hook && Ln.grad_hook(Ln.grad_user, Ln.grad.p, m.P, st) != 0)
        config_error("grad_hook failed");
      if (Ln.ent_hook && Ln.ent_hook(Ln.ent_user, Ln.grad.p + m.P, st) != 0)
        config_error("entropy_hook failed");
    }
    Ln.mark_end();
  }
  Ln.mark_begin(PH_ADAM);
  ++Ln.adam_step;
  adam_update(c, m, Ln.params.p, Ln.grad.p, Ln.mom.p, Ln.vel.p, Ln.adam_step, lr, Ln.flags.p, Ln.lstats.p);
  alpha_update_kernel<<<1, 1, 0, c->stream>>>(Ln.alpha.p, Ln.lstats.p, hook_h ? Ln.grad.p + m.P : nullptr,
                                              Ln.ec.target, Ln.ec.lr, Ln.ec.lower, Ln.ec.upper, Ln.flags.p, mb);
  after_launch(c);
  stats_accum_kernel<<<1, 1, 0, c->stream>>>(Ln.acc.p, Ln.lstats.p);
  after_launch(c);
  Ln.mark_end();
}


double cosine_lr(double base, int64_t total, int64_t consumed) {  // nn.cpp:308-312
  double progress = (double)consumed / (double)std::max<int64_t>(1, total);
  progress = std::min(std::max(progress, 0.0), 1.0);
  return base * 0.5 * (1.0 + std::cos(M_PI * progress));
}

// stream `to` waits for the work queued on `from` so far
static void record_wait(cudaStream_t from, cudaStream_t to) {
  if (from == to) return;
  cudaEvent_t e;
  VER_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  VER_CUDA(cudaEventRecord(e, from));
  VER_CUDA(cudaStreamWaitEvent(to, e, 0));
  VER_CUDA(cudaEventDestroy(e));
}

// learner.cpp:146-193
static void learner_update(Learner& Ln, DView& V, ver_train_stats* out) {
  Ctx* c = Ln.ctx;
  if (V.obs_dim != Ln.m.D || V.hidden_dim != Ln.m.H || (V.action_kind == 1) != (Ln.m.continuous == 1))
    config_error("learner_update: view shape does not match the model");
  struct EvGuard {  // the ctx logs recurrence launches into this learner's timing
    Ctx* c;
    ~EvGuard() { c->evlog = nullptr, c->flop_log = nullptr, c->rec_tag = -1, c->gemm_tag = -1; }
  } evg{c};
  c->evlog = Ln.timing ? &Ln.evlog : nullptr;
  for (double& f : Ln.flop_acc) f = 0.0;
  c->flop_log = Ln.flop_acc;
  // The view may belong to another context (an engine's close() on the collector
  // thread).  Everything of this update -- GAE included -- allocates, launches and
  // synchronizes on the learner's own context: the learner stream first waits for
  // the view's producer, and the view's stream waits for the update at the end.
  Ctx* const vc = V.ctx;
  struct CtxSwap {  // compute_gae / split / pack allocate and launch through V.ctx
    DView& V;
    Ctx* keep;
    Ctx* learner;
    ~CtxSwap() {
      if (keep != learner) record_wait(learner->stream, keep->stream);
      V.ctx = keep;
    }
  } swap{V, vc, c};
  record_wait(vc->stream, c->stream);
  V.ctx = c;
  Ln.mark_begin(PH_GAE);
  compute_gae(V, Ln.cfg.gamma, Ln.cfg.gae_lambda);
  Ln.mark_end();
  const double lr = cosine_lr(Ln.base_lr, Ln.total_steps, Ln.consumed);
  Ln.acc.zero(10);
  // Splits, packs and replay plans depend on the view and the seeds only.  They
  // run on the sampler stream (Ln.side): while the host waits on pack b+1's
  // round trips, minibatch b runs on ctx->stream, which waits only on the
  // event of its own pack.  The minibatch loop has no host sync.
  if (!Ln.side.stream) {
    Ln.side.device = c->device;
    Ln.side.num_sms = c->num_sms;
    Ln.side.precision = c->precision;
    Ln.side.tensor_cores = c->tensor_cores;
    VER_CUDA(cudaStreamCreateWithFlags(&Ln.side.stream, cudaStreamNonBlocking));
  }
  Ctx* sc = &Ln.side;
  record_wait(c->stream, sc->stream);  // GAE (advantages / returns) before the gathers
  const int64_t adam0 = Ln.adam_step;
  std::vector<std::unique_ptr<DPacked>> packs;
  int mb = 0;
  for (int epoch = 0; epoch < Ln.cfg.epochs; ++epoch) {
    const uint64_t seed = mix64(mix64(Ln.run_seed, (uint64_t)Ln.update_index), (uint64_t)epoch);
    V.ctx = sc;
    std::unique_ptr<DGroups> G(split_minibatches(V, Ln.cfg.minibatches, seed));
    for (int b = 0; b < G->B; ++b) {
      V.ctx = sc;
      packs.emplace_back(pack_pieces(V, G->pieces.p + G->gstart[b], G->gstart[b + 1] - G->gstart[b]));
      prepare_replay(sc, *packs.back());
      V.ctx = c;
      record_wait(sc->stream, c->stream);
      run_minibatch(Ln, V, *packs.back(), lr, mb++);
    }
  }
  c->launches += sc->launches;
  sc->launches = 0;
  // one read-back per update
  double* h = static_cast<double*>(c->pinned_buf(sizeof(double) * 13));
  VER_CUDA(cudaMemcpyAsync(h, Ln.acc.p, sizeof(double) * 10, cudaMemcpyDeviceToHost, c->stream));
  VER_CUDA(cudaMemcpyAsync(h + 10, Ln.alpha.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  VER_CUDA(cudaMemcpyAsync(h + 11, Ln.flags.p, 4 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  if (Ln.timing) Ln.collect_timing();
  const int* fl = reinterpret_cast<const int*>(h + 11);
  if (fl[1]) {
    // the reference's state at its throw: Adam steps of the minibatches before the
    // failing one (+ the failing one's when its parameters went non-finite);
    // consumed_steps / update_index unchanged
    const int fmb = fl[2], kind = fl[3];
    Ln.adam_step = adam0 + fmb + (kind == 2 ? 1 : 0);
    Ln.flags.zero(4);
    if (kind == 1) throw Error(VER_ERR_NONFINITE, "ppo_loss: non-finite loss");
    throw Error(VER_ERR_NONFINITE, "update: non-finite parameters");
  }
  if (out) {
    const double batches = h[9], steps = h[8];
    ver_train_stats s{};
    s.update_index = Ln.update_index;
    s.steps = V.size;
    s.fresh_steps = V.size - V.replayed_steps;
    s.stale_steps = V.stale_steps;
    s.lr = lr;
    s.loss = h[0] / batches;
    s.policy_loss = h[1] / batches;
    s.value_loss = h[2] / batches;
    s.entropy = h[3] / batches;
    s.mean_ratio = h[4] / steps;
    s.clip_fraction = h[5] / steps;
    s.mean_is_weight = h[6] / steps;
    s.max_is_weight = h[7];
    s.alpha = h[10];
    // entropy_loss_value (learner.hpp:44-46) with the final alpha
    s.entropy_loss = s.alpha * (Ln.ec.target - s.entropy) - s.alpha * s.entropy;
    *out = s;
  }
  Ln.consumed += V.size - V.replayed_steps;
  ++Ln.update_index;
}

void to_device_layout(const Model& m, const float* tensors_order, std::vector<float>& dev) {
  dev.assign(m.P, 0.f);
  for (int64_t k = 0; k < m.P; ++k) dev[m.dev_index[k]] = tensors_order[k];
}
static void to_tensor_order(const Model& m, const float* dev, float* out) {
  for (int64_t k = 0; k < m.P; ++k) out[k] = dev[m.dev_index[k]];
}

}  // namespace verg

using namespace verg;

struct ver_learner_s {
  Learner l;
};

namespace verg {
// the learner's current parameters (device layout) for the inference engine's snapshot
const ver_model_config* learner_model_config(ver_learner_s* l) { return &l->l.mc; }
const float* learner_device_params(ver_learner_s* l, Ctx** ctx, int64_t* count) {
  *ctx = l->l.ctx;
  *count = l->l.m.P;
  return l->l.params.p;
}
}  // namespace verg

extern "C" {

ver_status ver_param_count(const ver_model_config* c, int64_t* count, int* num_tensors) {
  VER_API_BEGIN
  const Model m = Model::make(*c);
  if (count) *count = m.P;
  if (num_tensors) *num_tensors = m.continuous ? 18 : 17;
  VER_API_END
}

ver_status ver_param_tensor(const ver_model_config* c, int idx, char name[16], int* rows, int* cols,
                            int64_t* offset) {
  VER_API_BEGIN
  static const char* names[] = {"enc_w1", "enc_b1", "enc_w2", "enc_b2", "gru_wr", "gru_ur",
                                "gru_br", "gru_wz", "gru_uz", "gru_bz", "gru_wn", "gru_un",
                                "gru_bn", "head_w", "head_b", "value_w", "value_b", "log_std"};
  const Model m = Model::make(*c);
  const int nt = m.continuous ? 18 : 17;
  if (idx < 0 || idx >= nt) config_error("ver_param_tensor: index out of range");
  const int D = m.D, E = m.E, H = m.H, A = m.A;
  const int shp[18][2] = {{D, E}, {1, E}, {E, E}, {1, E}, {E, H}, {H, H}, {1, H}, {E, H}, {H, H},
                          {1, H}, {E, H}, {H, H}, {1, H}, {H, A}, {1, A}, {H, 1}, {1, 1}, {1, A}};
  int64_t off = 0;
  for (int i = 0; i < idx; ++i) off += (int64_t)shp[i][0] * shp[i][1];
  if (name) std::strncpy(name, names[idx], 16);
  if (rows) *rows = shp[idx][0];
  if (cols) *cols = shp[idx][1];
  if (offset) *offset = off;
  VER_API_END
}

ver_status ver_params_init(const ver_model_config* c, uint64_t seed, double* out) {
  VER_API_BEGIN
  init_params_host(*c, seed, out);
  VER_API_END
}

double ver_cosine_lr(double base_lr, int64_t total_steps, int64_t consumed) {
  return cosine_lr(base_lr, total_steps, consumed);
}

ver_status ver_ppo_loss(ver_ctx ctx, const ver_model_config* mc, const float* params, ver_view v, ver_packed p,
                        const ver_ppo_config* cfg, double alpha, const float* h0_sorted, int want_grads,
                        const float* frozen_w, ver_loss_result* out, float* grads_out, float* is_w_out) {
  VER_API_BEGIN
  Ctx* c = &ctx->c;
  activate(c);
  const Model m = Model::make(*mc);
  DView& V = v->v;
  DPacked& P = p->p;
  if (V.obs_dim != m.D || V.hidden_dim != m.H) config_error("ppo_loss: view shape does not match the model");
  const int S = P.total;
  std::vector<float> dev;
  to_device_layout(m, params, dev);
  DBuf<float> dparams, grad, h0, fw;
  DBuf<double> dalpha;
  DBuf<LossStats> st;
  dparams.reserve(c, m.P);
  dparams.upload(dev.data(), m.P);
  grad.reserve(c, m.P + 1);
  grad.zero(m.P + 1);
  h0.reserve(c, (size_t)P.k * m.H);
  h0.upload(h0_sorted, (size_t)P.k * m.H);
  dalpha.reserve(c, 1);
  dalpha.upload(&alpha, 1);
  st.reserve(c, 1);
  if (frozen_w) {
    fw.reserve(c, S);
    fw.upload(frozen_w, S);
  }
  Workspace ws;
  ws.ctx = c;
  ws.ensure(m, S, true);
  policy_forward(c, m, dparams.p, S, P.obs.p, h0.p, P.max_len, P.bs.p, P.offs.p, ws, true, P.h_bs.data(),
                 P.h_offs.data());
  LossArgs la{P.act_cont.p, P.act_disc.p, P.old_logp.p, P.adv.p, P.ret.p, frozen_w ? fw.p : nullptr,
              cfg->clip, cfg->is_cap, cfg->value_loss_coef, dalpha.p};
  policy_loss(c, m, dparams.p, S, la, ws, grad.p, st.p, want_grads != 0);
  if (want_grads)
    policy_backward(c, m, dparams.p, S, P.obs.p, P.max_len, P.bs.p, P.offs.p, ws, grad.p, P.h_bs.data(),
                    P.h_offs.data());
  LossStats hs;
  st.download(&hs, 1);
  std::vector<float> g(m.P);
  if (want_grads && grads_out) grad.download(g.data(), m.P);
  if (is_w_out) ws.is_w.download(is_w_out, S);
  sync(c);
  out->loss = hs.loss;
  out->policy_loss = hs.policy_loss;
  out->value_loss = hs.value_loss;
  out->mean_entropy = hs.mean_entropy;
  out->ratio_sum = hs.ratio_sum;
  out->clip_count = hs.clip_count;
  out->w_sum = hs.w_sum;
  out->w_max = hs.w_max;
  out->steps = S;
  if (want_grads && !std::isfinite(hs.loss)) throw Error(VER_ERR_PROTOCOL, "ppo_loss: non-finite loss");
  if (want_grads && grads_out) to_tensor_order(m, g.data(), grads_out);
  VER_API_END
}

ver_status ver_forward_packed(ver_ctx ctx, const ver_model_config* mc, const float* params, int S,
                              const float* obs, const int32_t* act_disc, const float* act_cont, int L,
                              const int32_t* batch_sizes, const int32_t* offsets, const float* h0,
                              float* logp_out, float* ent_out, float* value_out) {
  VER_API_BEGIN
  Ctx* c = &ctx->c;
  activate(c);
  const Model m = Model::make(*mc);
  if (S <= 0 || L <= 0) config_error("forward_packed: empty batch");
  for (int64_t i = 0; i < (int64_t)S * m.D; ++i)
    if (!std::isfinite(obs[i])) protocol_error("forward_packed: non-finite observations");
  std::vector<float> dev;
  to_device_layout(m, params, dev);
  DBuf<float> dparams, dobs, dh0, dac, out;
  DBuf<int32_t> dad, dbo;
  dbo.reserve(c, 2 * (size_t)L);
  dbo.upload(batch_sizes, L);
  VER_CUDA(cudaMemcpyAsync(dbo.p + L, offsets, sizeof(int32_t) * L, cudaMemcpyHostToDevice, c->stream));
  dparams.reserve(c, m.P);
  dparams.upload(dev.data(), m.P);
  dobs.reserve(c, (size_t)S * m.D);
  dobs.upload(obs, (size_t)S * m.D);
  dh0.reserve(c, (size_t)batch_sizes[0] * m.H);
  dh0.upload(h0, (size_t)batch_sizes[0] * m.H);
  if (m.continuous) {
    dac.reserve(c, (size_t)S * m.A);
    dac.upload(act_cont, (size_t)S * m.A);
  } else {
    dad.reserve(c, S);
    dad.upload(act_disc, S);
  }
  out.reserve(c, (size_t)3 * S);
  Workspace ws;
  ws.ctx = c;
  ws.ensure(m, S, false);
  policy_forward(c, m, dparams.p, S, dobs.p, dh0.p, L, dbo.p, dbo.p + L, ws, false);
  policy_rows(c, m, dparams.p, S, ws.hidden.p, dad.p, dac.p, out.p, out.p + S, out.p + 2 * (size_t)S);
  if (logp_out) out.download(logp_out, S);
  if (ent_out) VER_CUDA(cudaMemcpyAsync(ent_out, out.p + S, sizeof(float) * S, cudaMemcpyDeviceToHost, c->stream));
  if (value_out)
    VER_CUDA(cudaMemcpyAsync(value_out, out.p + 2 * (size_t)S, sizeof(float) * S, cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  VER_API_END
}

ver_status ver_act(ver_ctx ctx, const ver_model_config* mc, const float* params, int n, const float* obs,
                   const float* h, float* dist_out, float* value_out, float* h_new_out) {
  VER_API_BEGIN
  Ctx* c = &ctx->c;
  activate(c);
  const Model m = Model::make(*mc);
  if (n <= 0) return VER_OK;
  for (int64_t i = 0; i < (int64_t)n * m.D; ++i)
    if (!std::isfinite(obs[i])) protocol_error("act: non-finite observation");
  std::vector<float> dev;
  to_device_layout(m, params, dev);
  DBuf<float> dparams, dobs, dh, out;
  dparams.reserve(c, m.P);
  dparams.upload(dev.data(), m.P);
  dobs.reserve(c, (size_t)n * m.D);
  dobs.upload(obs, (size_t)n * m.D);
  dh.reserve(c, (size_t)n * m.H);
  dh.upload(h, (size_t)n * m.H);
  out.reserve(c, (size_t)n * m.AH);
  Workspace ws;
  ws.ctx = c;
  ws.ensure(m, n, false);
  DBuf<int32_t> bo;
  bo.reserve(c, 2);
  const int32_t hbo[2] = {n, 0};
  bo.upload(hbo, 2);
  policy_forward(c, m, dparams.p, n, dobs.p, dh.p, 1, bo.p, bo.p + 1, ws, false);
  policy_heads(c, m, dparams.p, n, ws.hidden.p, out.p);
  std::vector<float> ho((size_t)n * m.AH);
  out.download(ho.data(), ho.size());
  if (h_new_out) ws.hidden.download(h_new_out, (size_t)n * m.H);
  sync(c);
  for (int i = 0; i < n; ++i) {
    if (dist_out)
      for (int a = 0; a < m.A; ++a) dist_out[(size_t)i * m.A + a] = ho[(size_t)i * m.AH + a];
    if (value_out) value_out[i] = ho[(size_t)i * m.AH + m.A];
  }
  VER_API_END
}

ver_status ver_adam_step(ver_ctx ctx, int64_t count, float* params, const float* grads, float* mo, float* ve,
                         int64_t* step, double lr) {
  VER_API_BEGIN
  Ctx* c = &ctx->c;
  activate(c);
  if (count <= 0) return VER_OK;
  DBuf<float> w, g, m, v;
  DBuf<int> flag;
  w.reserve(c, count);
  g.reserve(c, count);
  m.reserve(c, count);
  v.reserve(c, count);
  flag.reserve(c, 1);
  flag.zero(1);
  w.upload(params, count);
  g.upload(grads, count);
  m.upload(mo, count);
  v.upload(ve, count);
  Model flat;
  flat.P = count;
  flat.continuous = 0;
  ++*step;
  adam_update(c, flat, w.p, g.p, m.p, v.p, *step, lr, flag.p);
  w.download(params, count);
  m.download(mo, count);
  v.download(ve, count);
  sync(c);
  VER_API_END
}

ver_status ver_learner_create(ver_ctx ctx, const ver_model_config* mc, const float* params,
                              const ver_ppo_config* cfg, const ver_entropy_controller* ec, double base_lr,
                              int64_t total_steps, uint64_t run_seed, ver_learner* out) {
  VER_API_BEGIN
  Ctx* c = &ctx->c;
  activate(c);
  if (cfg->epochs < 0 || cfg->minibatches < 1) config_error("learner: epochs >= 0 and minibatches >= 1");
  auto* h = new ver_learner_s();
  Learner& L = h->l;
  L.ctx = c;
  L.mc = *mc;
  L.m = Model::make(*mc);
  L.cfg = *cfg;
  L.ec = *ec;
  L.base_lr = base_lr;
  L.total_steps = total_steps;
  L.run_seed = run_seed;
  L.ws.ctx = c;
  L.wr.ctx = c;
  const int64_t P = L.m.P;
  L.params.reserve(c, P);
  L.grad.reserve(c, P + 1);
  L.mom.reserve(c, P);
  L.vel.reserve(c, P);
  L.mom.zero(P);
  L.vel.zero(P);
  L.grad.zero(P + 1);
  std::vector<float> dev;
  to_device_layout(L.m, params, dev);
  L.params.upload(dev.data(), P);
  L.alpha.reserve(c, 1);
  L.alpha.upload(&ec->alpha, 1);
  L.acc.reserve(c, 10);
  L.lstats.reserve(c, 1);
  L.flags.reserve(c, 4);
  L.flags.zero(4);
  sync(c);
  *out = h;
  VER_API_END
}

ver_status ver_learner_destroy(ver_learner l) {
  VER_API_BEGIN
  if (l) {
    activate(l->l.ctx);
    sync(l->l.ctx);
    delete l;
  }
  VER_API_END
}

ver_status ver_learner_enable_allreduce(ver_learner l, int enable) {
  VER_API_BEGIN
  l->l.allreduce = enable != 0;
  VER_API_END
}

ver_status ver_learner_set_grad_hook(ver_learner l, ver_grad_hook fn, void* user) {
  VER_API_BEGIN
  l->l.grad_hook = fn;
  l->l.grad_user = user;
  VER_API_END
}

ver_status ver_learner_set_entropy_hook(ver_learner l, ver_entropy_hook fn, void* user) {
  VER_API_BEGIN
  l->l.ent_hook = fn;
  l->l.ent_user = user;
  VER_API_END
}

ver_status ver_param_device_index(const ver_model_config* c, int64_t* index_out) {
  VER_API_BEGIN
  const Model m = Model::make(*c);
  for (int64_t k = 0; k < m.P; ++k) index_out[k] = m.dev_index[k];
  VER_API_END
}

ver_status ver_learner_update(ver_learner l, ver_view v, ver_train_stats* stats) {
  VER_API_BEGIN
  activate(l->l.ctx);
  learner_update(l->l, v->v, stats);
  VER_API_END
}

ver_status ver_learner_batch_h0(ver_learner l, ver_view v, ver_packed p, float* h0_out) {
  VER_API_BEGIN
  Learner& L = l->l;
  Ctx* c = L.ctx;
  activate(c);
  DPacked& P = p->p;
  DBuf<float> h0;
  h0.reserve(c, (size_t)P.k * L.m.H);
  batch_h0(L, v->v, P, L.params.p, h0.p);
  h0.download(h0_out, (size_t)P.k * L.m.H);
  sync(c);
  VER_API_END
}

ver_status ver_learner_get_params(ver_learner l, float* out) {
  VER_API_BEGIN
  Learner& L = l->l;
  activate(L.ctx);
  std::vector<float> dev(L.m.P);
  L.params.download(dev.data(), L.m.P);
  sync(L.ctx);
  to_tensor_order(L.m, dev.data(), out);
  VER_API_END
}

ver_status ver_learner_set_params(ver_learner l, const float* in) {
  VER_API_BEGIN
  Learner& L = l->l;
  activate(L.ctx);
  std::vector<float> dev;
  to_device_layout(L.m, in, dev);
  L.params.upload(dev.data(), L.m.P);
  sync(L.ctx);
  VER_API_END
}

ver_status ver_learner_get_adam(ver_learner l, float* mo, float* ve, int64_t* step) {
  VER_API_BEGIN
  Learner& L = l->l;
  activate(L.ctx);
  std::vector<float> a(L.m.P), b(L.m.P);
  L.mom.download(a.data(), L.m.P);
  L.vel.download(b.data(), L.m.P);
  sync(L.ctx);
  if (mo) to_tensor_order(L.m, a.data(), mo);
  if (ve) to_tensor_order(L.m, b.data(), ve);
  if (step) *step = L.adam_step;
  VER_API_END
}

ver_status ver_learner_set_adam(ver_learner l, const float* mo, const float* ve, int64_t step) {
  VER_API_BEGIN
  Learner& L = l->l;
  activate(L.ctx);
  std::vector<float> a, b;
  to_device_layout(L.m, mo, a);
  to_device_layout(L.m, ve, b);
  L.mom.upload(a.data(), L.m.P);
  L.vel.upload(b.data(), L.m.P);
  sync(L.ctx);
  L.adam_step = step;
  VER_API_END
}

ver_status ver_learner_get_state(ver_learner l, double* alpha, int64_t* consumed, int64_t* ui) {
  VER_API_BEGIN
  Learner& L = l->l;
  activate(L.ctx);
  if (alpha) {
    L.alpha.download(alpha, 1);
    sync(L.ctx);
  }
  if (consumed) *consumed = L.consumed;
  if (ui) *ui = L.update_index;
  VER_API_END
}

ver_status ver_learner_set_state(ver_learner l, double alpha, int64_t consumed, int64_t ui) {
  VER_API_BEGIN
  Learner& L = l->l;
  activate(L.ctx);
  L.alpha.upload(&alpha, 1);
  sync(L.ctx);
  L.consumed = consumed;
  L.update_index = ui;
  VER_API_END
}

ver_status ver_bench_gae_gather(ver_view v, double gamma, double lambda, int B, uint64_t seed, int reps,
                                float* ms_out) {
  VER_API_BEGIN
  DView& V = v->v;
  Ctx* c = V.ctx;
  activate(c);
  reps = std::max(1, reps);
  cudaEvent_t e0, e1;
  VER_CUDA(cudaEventCreate(&e0));
  VER_CUDA(cudaEventCreate(&e1));
  std::vector<std::tuple<int, cudaEvent_t, cudaEvent_t>> log;
  struct Restore {
    Ctx* c;
    ~Restore() { c->evlog = nullptr, c->hbm_tag = -1; }
  } restore{c};
  auto elapsed = [](cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    VER_CUDA(cudaEventElapsedTime(&ms, a, b));
    return ms;
  };
  compute_gae(V, gamma, lambda);  // warm
  c->evlog = &log;
  c->hbm_tag = 0;
  float gae = 0.f;
  for (int r = 0; r < reps; ++r) {
    VER_CUDA(cudaEventRecord(e0, c->stream));
    compute_gae(V, gamma, lambda);
    VER_CUDA(cudaEventRecord(e1, c->stream));
    VER_CUDA(cudaEventSynchronize(e1));
    gae += elapsed(e0, e1);
  }
  c->evlog = nullptr;
  std::unique_ptr<DGroups> G(split_minibatches(V, B, seed));
  std::vector<std::unique_ptr<DPacked>> packs;
  for (int b = 0; b < G->B; ++b)
    if (G->gstart[b + 1] > G->gstart[b])
      packs.emplace_back(pack_pieces(V, G->pieces.p + G->gstart[b], G->gstart[b + 1] - G->gstart[b]));
  for (auto& P : packs) gather_packed(V, *P);  // warm (tile tables built)
  sync(c);
  c->evlog = &log;
  float gat = 0.f;
  for (int r = 0; r < reps; ++r) {
    VER_CUDA(cudaEventRecord(e0, c->stream));
    for (auto& P : packs) gather_packed(V, *P);
    VER_CUDA(cudaEventRecord(e1, c->stream));
    VER_CUDA(cudaEventSynchronize(e1));
    gat += elapsed(e0, e1);
  }
  float kern[2] = {0.f, 0.f};
  for (auto& [tag, a, b] : log) {
    if (tag == 0 || tag == 1) kern[tag] += elapsed(a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  ms_out[0] = gae / reps;
  ms_out[1] = gat / reps;
  ms_out[2] = kern[0] / reps;
  ms_out[3] = kern[1] / reps;
  VER_API_END
}

ver_status ver_learner_last_timing(ver_learner l, float* ms, int* n) {
  VER_API_BEGIN
  const int k = std::min(*n, (int)PH_N);
  for (int i = 0; i < k; ++i) ms[i] = l->l.phase_ms[i];
  *n = PH_N;
  VER_API_END
}

ver_status ver_learner_last_flop(ver_learner l, double* flop, int* n) {
  VER_API_BEGIN
  const int k = std::min(*n, (int)PH_N);
  for (int i = 0; i < k; ++i) flop[i] = l->l.phase_flop[i];
  *n = PH_N;
  VER_API_END
}

ver_status ver_learner_last_timing_counts(ver_learner l, int* counts, int* n) {
  VER_API_BEGIN
  const int k = std::min(*n, (int)PH_N);
  for (int i = 0; i < k; ++i) counts[i] = l->l.phase_n[i];
  *n = PH_N;
  VER_API_END
}

}  // extern "C"
