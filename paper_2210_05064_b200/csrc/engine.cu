// engine.cu — the collection-side inference engine on the device (SURVEY
// §8(f) row 1): InferenceEngine (runtime.hpp:96-160, runtime.cpp:60-215) with
// batched act (nn.cpp:118-126) and on-device action sampling (nn.cpp:134-185)
// writing its records into the rollout store.
//
// Device-resident: the policy snapshot, every env's GRU state h (N x H) and
// the pending record's h_before (N x H).  Per compute_actions call one H2D of
// the requests (obs, env, episode, step) and one D2H of the sampled actions,
// log-probs and values (the env simulators need the actions on the host);
// h_before never crosses PCIe: the store copies a sequence-starting record's
// row device to device (rollout.cuh append_rec), where the reference copies H
// doubles on every commit (rollout.cpp:81).
//
// Sampling restates the reference bit for bit on the integer side: the
// counter RNG (rng.hpp: splitmix64 / mix, uniform = (u >> 11) * 2^-53,
// Box-Muller normal) keyed CounterRng(seed).stream(0xAC7101, env)
// .stream(obs_episode, obs_step) (runtime.cpp:166-169), and the categorical /
// Gaussian draws and log-probs in double from the fp32 logits.
//
// The protocol (complete_pending, done -> h = 0, parking when the store is
// closed or the env is at its Fixed-mode cap, begin_rollout unparking,
// finalize_bootstraps) is host integer bookkeeping mirroring runtime.cpp line
// by line.
#include <optional>

#include "coordinator.cuh"
#include "policy.cuh"
#include "rollout.cuh"

namespace verg {
namespace eng {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
// rng.hpp:23-25
__device__ __forceinline__ uint64_t mix(uint64_t a, uint64_t b) {
  return splitmix64(a ^ (0x9e3779b97f4a7c15ull + (b << 6) + (b >> 2) + splitmix64(b)));
}
struct Rng {  // CounterRng (rng.hpp:30-73)
  uint64_t key, counter;
  __device__ double uniform() { return (double)(mix(key, counter++) >> 11) * 0x1.0p-53; }
  __device__ double normal() {
    double u1 = uniform();
    const double u2 = uniform();
    if (u1 <= 0) u1 = 0x1.0p-53;
    return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
  }
};

// h rows of the requesting envs -> batch matrix (and the pending h_before)
__global__ void gather_h_kernel(int m, int H, const int32_t* __restrict__ env, const float* __restrict__ h,
                                float* __restrict__ hb, float* __restrict__ batch, int write_hb) {
  const int i = blockIdx.x;
  if (i >= m) return;
  const int e = env[i];
  for (int j = threadIdx.x; j < H; j += blockDim.x) {
    const float v = h[(size_t)e * H + j];
    batch[(size_t)i * H + j] = v;
    if (write_hb) hb[(size_t)e * H + j] = v;
  }
}

__global__ void zero_rows_kernel(int m, int H, const int32_t* __restrict__ env, float* __restrict__ h) {
  const int i = blockIdx.x;
  if (i >= m) return;
  for (int j = threadIdx.x; j < H; j += blockDim.x) h[(size_t)env[i] * H + j] = 0.f;
}

__global__ void scatter_h_kernel(int m, int H, const int32_t* __restrict__ env, const float* __restrict__ hnew,
                                 float* __restrict__ h) {
  const int i = blockIdx.x;
  if (i >= m) return;
  for (int j = threadIdx.x; j < H; j += blockDim.x) h[(size_t)env[i] * H + j] = hnew[(size_t)i * H + j];
}

// The attached joint preemption counter (coordinator.cuh): add this batch's
// commits (add_steps, distributed.hpp:110-119; the reference's driver calls it
// from on_commits after process_batch, runtime.cpp:592) and mirror the group's
// fired flag into mapped host memory: flag[0] = fired, flag[1] = this add fired.
__device__ __forceinline__ void preempt_commit(PreemptWords* pw, long long nadd, int* flag) {
  const int now = preempt_add_dev(pw, nadd);
  flag[0] = preempt_fired_dev(pw);
  flag[1] = now;
}
__global__ void preempt_commit_kernel(PreemptWords* pw, long long nadd, int* flag) { preempt_commit(pw, nadd, flag); }

// compute_actions' sampling (runtime.cpp:163-188): one thread per request.
// out: [m] action index | [m x A] continuous action | [m] log-prob | [m] value.
// Thread 0 also commits the batch's steps to the attached preemption counter.
__global__ void sample_kernel(int m, int A, int AH, int continuous, uint64_t key0, const int32_t* __restrict__ env,
                              const int64_t* __restrict__ obs_ep, const int32_t* __restrict__ obs_step,
                              const float* __restrict__ heads, const float* __restrict__ log_std,
                              int32_t* __restrict__ act_d, float* __restrict__ act_c, float* __restrict__ logp,
                              float* __restrict__ value, PreemptWords* pw, long long nadd, int* pflag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0 && pw) preempt_commit(pw, nadd, pflag);
  if (i >= m) return;
  Rng rng{mix(mix(mix(mix(key0, 0xAC7101ull), (uint64_t)env[i]), (uint64_t)obs_ep[i]), (uint64_t)obs_step[i]), 0};
  const float* row = heads + (size_t)i * AH;
  value[i] = row[A];
  if (!continuous) {
    // sample_categorical (nn.cpp:134-146) and categorical_log_prob (:148-152)
    double mx = row[0];
    for (int a = 1; a < A; ++a) mx = fmax(mx, (double)row[a]);
    double sum = 0.0;
    for (int a = 0; a < A; ++a) sum += exp((double)row[a] - mx);
    const double u = rng.uniform();
    double acc = 0.0;
    int pick = A - 1;
    for (int a = 0; a < A; ++a) {
      acc += exp((double)row[a] - mx) / sum;
      if (u < acc) {
        pick = a;
        break;
      }
    }
    act_d[i] = pick;
    logp[i] = (float)((double)row[pick] - (mx + log(sum)));
  } else {
    // sample_gaussian (nn.cpp:167-173) and gaussian_log_prob (:175-183)
    double lp = -0.5 * 1.8378770664093454836 * (double)A;  // log(2 pi)
    for (int a = 0; a < A; ++a) {
      const double ls = log_std[a], s = exp(ls), mean = row[a];
      const double x = mean + s * rng.normal();
      act_c[(size_t)i * A + a] = (float)x;
      const double z = (x - mean) / s;
      lp += -0.5 * z * z - ls;
    }
    logp[i] = (float)lp;
  }
}

__host__ inline uint64_t h_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

struct Request {  // InferenceRequest (runtime.hpp:30-42); obs points into the caller's batch
  int env = 0;
  const float* obs = nullptr;
  float reward = 0.f, latency = 0.f;
  uint8_t done = 0, first = 0;
  int64_t obs_episode = 0;
  int32_t obs_step = 0;
};
struct Parked {  // a parked request owns its observation
  Request r;
  std::vector<float> obs;
};
struct Slot {  // EnvSlot (runtime.hpp:145-150); h lives on the device, the
               // PendingStep in the engine's per-env arrays (pend_*)
  std::optional<Parked> parked;
  bool paused = false;
};
struct Result {
  int32_t* env = nullptr;
  int32_t* act_d = nullptr;
  float* act_c = nullptr;
  int nd = 0, new_commits = 0;
  bool closed_now = false;
  bool preempt_fired = false;
};

struct Engine {
  Ctx* c = nullptr;
  ver_engine_config cfg{};
  Model m;
  ver_rollout_s store;
  DBuf<float> params;
  uint64_t version = 0;
  uint64_t key0 = 0;
  DBuf<float> h, hb;
  std::vector<Slot> envs;
  // PendingStep (runtime.hpp:135-144) per env, flat; h_before is row `env` of hb
  std::vector<uint8_t> has_pend;
  std::vector<float> pend_obs, pend_ac, pend_lp, pend_v;
  std::vector<int32_t> pend_ad, pend_t;
  std::vector<int64_t> pend_ep;
  std::vector<uint64_t> pend_ver;

  void init_envs(int N) {
    envs.resize(N);
    has_pend.assign(N, 0);
    pend_obs.assign((size_t)N * m.D, 0.f);
    pend_ac.assign((size_t)N * std::max(1, m.A), 0.f);
    pend_lp.assign(N, 0.f);
    pend_v.assign(N, 0.f);
    pend_ad.assign(N, 0);
    pend_t.assign(N, 0);
    pend_ep.assign(N, 0);
    pend_ver.assign(N, 0);
  }
  void park(const Request& r) {
    Parked p;
    p.obs.assign(r.obs, r.obs + m.D);
    p.r = r;
    envs[r.env].parked = std::move(p);
    envs[r.env].parked->r.obs = envs[r.env].parked->obs.data();
  }
  Workspace ws;
  DBuf<float> heads, dobs, hbatch, dres;
  DBuf<int32_t> didx, bo;
  DBuf<int64_t> dep;
  Pinned<float> pobs, pres;
  Pinned<int32_t> pidx;
  Pinned<int64_t> pep;

  Rollout& buf() { return store.r; }

  // attached joint preemption counter: commits are added by the sampling kernel,
  // the group's fired flag comes back in mapped host memory with the actions
  ver_preempt_s* pre = nullptr;
  int* pflag_h = nullptr;  // [fired, fired_now], cudaHostAllocMapped
  int* pflag_d = nullptr;
  long long commit_add = 0;  // this batch's commits, added by the next sampling launch
  bool committed_this_batch = false;
  ~Engine() {
    if (pflag_h) cudaFreeHost(pflag_h);
  }

  // forward of the listed envs (act: encode + gru_cell + heads) -> heads (m x AH);
  // with `sample`: pending h_before, sampled actions, h <- h_new
  void run(const std::vector<const Request*>& rq, bool sample) {
    const int n = (int)rq.size(), D = m.D, H = m.H, A = m.A;
    for (const Request* r : rq)
      for (int k = 0; k < D; ++k)
        if (!std::isfinite(r->obs[k])) protocol_error("act: non-finite observation");  // nn.cpp:119
    pobs.ensure((size_t)n * D);
    pidx.ensure((size_t)2 * n);
    pep.ensure(n);
    for (int i = 0; i < n; ++i) {
      const Request& r = *rq[i];
      std::memcpy(pobs.p + (size_t)i * D, r.obs, sizeof(float) * D);
      pidx.p[i] = r.env;
      pidx.p[n + i] = r.obs_step;
      pep.p[i] = r.obs_episode;
    }
    dobs.reserve(c, (size_t)n * D);
    didx.reserve(c, (size_t)2 * n);
    dep.reserve(c, n);
    hbatch.reserve(c, (size_t)n * H);
    heads.reserve(c, (size_t)n * m.AH);
    VER_CUDA(cudaMemcpyAsync(dobs.p, pobs.p, sizeof(float) * n * D, cudaMemcpyHostToDevice, c->stream));
    VER_CUDA(cudaMemcpyAsync(didx.p, pidx.p, sizeof(int32_t) * 2 * n, cudaMemcpyHostToDevice, c->stream));
    VER_CUDA(cudaMemcpyAsync(dep.p, pep.p, sizeof(int64_t) * n, cudaMemcpyHostToDevice, c->stream));
    gather_h_kernel<<<n, 128, 0, c->stream>>>(n, H, didx.p, h.p, hb.p, hbatch.p, sample ? 1 : 0);
    after_launch(c);
    ws.ensure(m, n, false);
    const int32_t hbo[2] = {n, 0};
    bo.reserve(c, 2);
    bo.upload(hbo, 2);
    // one timestep of n rows: with the host batch sizes the GRU step runs on the
    // tensor cores (stepgemm.cu) once n reaches the big-step threshold
    policy_forward(c, m, params.p, n, dobs.p, hbatch.p, 1, bo.p, bo.p + 1, ws, false, hbo, hbo + 1);
    policy_heads(c, m, params.p, n, ws.hidden.p, heads.p);
    if (sample) {
      scatter_h_kernel<<<n, 128, 0, c->stream>>>(n, H, didx.p, ws.hidden.p, h.p);
      after_launch(c);
    }
    // results: act_d [n] | logp [n] | value [n] | act_c [n x A]
    const size_t nres = (size_t)n * (3 + A);
    dres.reserve(c, nres);
    pres.ensure(nres);
    if (sample) {
      sample_kernel<<<cdiv(n, 128), 128, 0, c->stream>>>(
          n, A, m.AH, m.continuous, key0, didx.p, dep.p, didx.p + n, heads.p,
          m.continuous ? params.p + m.o_ls : nullptr, reinterpret_cast<int32_t*>(dres.p), dres.p + 3 * n,
          dres.p + n, dres.p + 2 * n, pre ? pre->w : nullptr, commit_add, pflag_d);
      after_launch(c);
      if (pre) committed_this_batch = true;
      VER_CUDA(cudaMemcpyAsync(pres.p, dres.p, sizeof(float) * nres, cudaMemcpyDeviceToHost, c->stream));
    } else {
      VER_CUDA(cudaMemcpy2DAsync(pres.p + 2 * n, sizeof(float), heads.p + A, sizeof(float) * m.AH, sizeof(float), n,
                                 cudaMemcpyDeviceToHost, c->stream));
    }
    sync(c);
  }

  // compute_actions (runtime.cpp:149-190)
  void compute_actions(const std::vector<const Request*>& needs, Result& out) {
    if (needs.empty()) return;
    run(needs, true);
    const int n = (int)needs.size(), A = m.A;
    const int32_t* ad = reinterpret_cast<const int32_t*>(pres.p);
    for (int i = 0; i < n; ++i) {
      const Request& r = *needs[i];
      const int e = r.env;
      has_pend[e] = 1;
      std::memcpy(pend_obs.data() + (size_t)e * m.D, r.obs, sizeof(float) * m.D);
      if (m.continuous) std::memcpy(pend_ac.data() + (size_t)e * A, pres.p + 3 * n + (size_t)i * A, sizeof(float) * A);
      else pend_ad[e] = ad[i];
      pend_lp[e] = pres.p[n + i];
      pend_v[e] = pres.p[2 * n + i];
      pend_ep[e] = r.obs_episode;
      pend_t[e] = r.obs_step;
      pend_ver[e] = version;
      const int k = out.nd++;
      if (out.env) out.env[k] = e;
      if (!m.continuous && out.act_d) out.act_d[k] = pend_ad[e];
      if (m.continuous && out.act_c) std::memcpy(out.act_c + (size_t)k * A, pend_ac.data() + (size_t)e * A, sizeof(float) * A);
    }
  }

  // complete_pending (runtime.cpp:116-147)
  void complete_pending(const Request& req, Result& out) {
    const int e = req.env;
    if (!has_pend[e])
      protocol_error("inference: completion for env " + std::to_string(e) + " without an outstanding action");
    has_pend[e] = 0;
    const int oc = buf().append_rec(e, pend_ep[e], pend_t[e], pend_obs.data() + (size_t)e * m.D, pend_ad[e],
                                    m.continuous ? pend_ac.data() + (size_t)e * m.A : nullptr, pend_lp[e], pend_v[e],
                                    req.reward, req.latency, req.done ? 1 : 0, nullptr, hb.p + (size_t)e * m.H,
                                    pend_ver[e]);
    if (oc == 0) {
      ++out.new_commits;
      if (!buf().open) out.closed_now = true;
    } else if (pend_t[e] > 0) {
      buf().bootstrap[e] = pend_v[e];
      buf().bootstrap_valid[e] = 1;
    }
  }

  // process_batch (runtime.cpp:192-215)
  void process_batch(std::vector<Request>& reqs, Result& out) {
    std::vector<const Request*> needs;
    std::vector<int32_t> zero;
    for (auto& req : reqs) {
      if (req.env < 0 || req.env >= cfg.rollout.N) protocol_error("inference: env index out of range");
      Slot& es = envs[req.env];
      if (es.parked)
        protocol_error("inference: request for env " + std::to_string(req.env) + " which is already parked");
      if (!req.first) complete_pending(req, out);
      if (req.done) zero.push_back(req.env);
      const bool capped = cfg.rollout.mode == 0 && buf().env_at_cap(req.env);
      if (buf().open && !capped) {
        needs.push_back(&req);
      } else {
        park(req);
        if (capped) es.paused = true;
      }
    }
    commit_add = out.new_commits;
    committed_this_batch = false;
    if (!zero.empty()) {  // es.h.setZero() for done envs (parked ones too)
      pidx.ensure(std::max<size_t>(zero.size(), 2 * needs.size()));
      DBuf<int32_t> dz;
      dz.reserve(c, zero.size());
      dz.upload(zero.data(), zero.size());
      zero_rows_kernel<<<(int)zero.size(), 128, 0, c->stream>>>((int)zero.size(), m.H, dz.p, h.p);
      after_launch(c);
      sync(c);
    }
    compute_actions(needs, out);
    if (pre) preempt_after_batch(out);
  }

  // the group's preemption after a batch: commit if no sampling launch carried the
  // add, then force-close this replica's rollout once the group has fired
  // (ThreadedDriver::request_force_close -> engine_.force_close() after the
  // batch, runtime.cpp:596-599)
  void preempt_after_batch(Result& out) {
    if (!committed_this_batch) {
      if (commit_add <= 0) return;
      preempt_commit_kernel<<<1, 1, 0, c->stream>>>(pre->w, commit_add, pflag_d);
      after_launch(c);
      sync(c);
    }
    commit_add = 0;
    const int fired = *(volatile int*)pflag_h;
    out.preempt_fired = fired != 0;
    if (fired && buf().open && buf().committed > 0) {
      buf().open = false;
      out.closed_now = true;
    }
  }

  // begin_rollout (runtime.cpp:84-113)
  void begin_rollout(Result& out) {
    sync(c);  // the store's pinned log may still be read by the last close's H2D
    buf().begin(version);
    out.new_commits = buf().committed;
    for (auto& es : envs) es.paused = false;
    std::vector<Parked> parked;
    for (auto& es : envs) {
      if (es.parked) {
        parked.push_back(std::move(*es.parked));
        es.parked.reset();
      }
    }
    std::vector<const Request*> needs;
    for (auto& pk : parked) {
      pk.r.obs = pk.obs.data();
      if (buf().open && !buf().env_at_cap(pk.r.env)) needs.push_back(&pk.r);
      else park(pk.r);
    }
    commit_add = 0;  // carryover commits are not counted toward the group (runtime.cpp:521-531)
    compute_actions(needs, out);
    if (!buf().open) out.closed_now = true;
  }

  // finalize_bootstraps (runtime.cpp:217-229)
  void finalize_bootstraps() {
    std::vector<const Request*> vo;
    for (int e = 0; e < cfg.rollout.N; ++e) {
      Slot& es = envs[e];
      if (buf().bootstrap_valid[e]) continue;
      if (has_pend[e]) {
        if (pend_t[e] > 0) {
          buf().bootstrap[e] = pend_v[e];
          buf().bootstrap_valid[e] = 1;
        }
      } else if (es.parked && es.parked->r.obs_step > 0) {
        vo.push_back(&es.parked->r);
      }
    }
    if (vo.empty()) return;
    run(vo, false);  // value_only (nn.cpp:128-132) with the env's current h
    const int n = (int)vo.size();
    for (int i = 0; i < n; ++i) {
      buf().bootstrap[vo[i]->env] = pres.p[2 * n + i];
      buf().bootstrap_valid[vo[i]->env] = 1;
    }
  }

  void set_params_host(const float* p) {
    std::vector<float> dev;
    to_device_layout(m, p, dev);
    params.reserve(c, m.P);
    params.upload(dev.data(), m.P);
    ws.wlo_stale = true;  // the snapshot is constant until the next set_snapshot
    ws.wlo_keep = true;
  }
};

}  // namespace eng
}  // namespace verg

using namespace verg;

struct ver_engine_s {
  eng::Engine e;
};

static void to_result(const eng::Result& r, ver_batch_result* out) {
  if (!out) return;
  out->n_dispatch = r.nd;
  out->new_commits = r.new_commits;
  out->closed_now = r.closed_now ? 1 : 0;
  out->preempt_fired = r.preempt_fired ? 1 : 0;
}

extern "C" {

ver_status ver_engine_create(ver_ctx ctx, const ver_engine_config* cfg, const float* params, uint64_t version,
                             ver_engine* out) {
  VER_API_BEGIN
  Ctx* c = &ctx->c;
  activate(c);
  const ver_rollout_config& rc = cfg->rollout;
  if (rc.T < 1 || rc.N < 1) config_error("engine: T and N must be >= 1");
  if (cfg->model.obs_dim != rc.obs_dim || cfg->model.hidden_dim != rc.hidden_dim ||
      cfg->model.action_kind != rc.action_kind)
    config_error("engine: model and rollout dimensions differ");
  auto* w = new ver_engine_s();
  eng::Engine& E = w->e;
  E.c = c;
  E.cfg = *cfg;
  E.m = Model::make(cfg->model);
  E.store.r.ctx = c;
  E.store.r.cfg = rc;
  E.store.r.init();
  E.key0 = eng::h_splitmix64(cfg->seed);  // CounterRng(seed) (rng.hpp:33)
  E.version = version;
  E.set_params_host(params);
  E.h.reserve(c, (size_t)rc.N * E.m.H);
  E.h.zero((size_t)rc.N * E.m.H);
  E.hb.reserve(c, (size_t)rc.N * E.m.H);
  E.hb.zero((size_t)rc.N * E.m.H);
  E.init_envs(rc.N);
  E.ws.ctx = c;
  *out = w;
  VER_API_END
}

ver_status ver_engine_destroy(ver_engine e) {
  VER_API_BEGIN
  if (e) {
    sync(e->e.c);
    delete e;
  }
  VER_API_END
}

ver_status ver_engine_set_snapshot(ver_engine e, const float* params, uint64_t version) {
  VER_API_BEGIN
  activate(e->e.c);
  e->e.set_params_host(params);
  e->e.version = version;
  VER_API_END
}

ver_status ver_engine_set_snapshot_learner(ver_engine e, ver_learner l, uint64_t version) {
  VER_API_BEGIN
  eng::Engine& E = e->e;
  activate(E.c);
  Ctx* lc = nullptr;
  int64_t count = 0;
  const float* src = learner_device_params(l, &lc, &count);
  if (count != E.m.P) config_error("engine: learner model differs from the engine's");
  sync(lc);
  E.params.reserve(E.c, E.m.P);
  VER_CUDA(cudaMemcpyAsync(E.params.p, src, sizeof(float) * E.m.P, cudaMemcpyDeviceToDevice, E.c->stream));
  E.ws.wlo_stale = true;
  E.ws.wlo_keep = true;
  E.version = version;
  VER_API_END
}

ver_status ver_engine_begin_rollout(ver_engine e, ver_batch_result* res, int32_t* disp_env, int32_t* disp_act,
                                    float* disp_act_cont) {
  VER_API_BEGIN
  activate(e->e.c);
  eng::Result r{disp_env, disp_act, disp_act_cont};
  e->e.begin_rollout(r);
  to_result(r, res);
  VER_API_END
}

ver_status ver_engine_process_batch(ver_engine e, const ver_request_batch* b, ver_batch_result* res,
                                    int32_t* disp_env, int32_t* disp_act, float* disp_act_cont) {
  VER_API_BEGIN
  eng::Engine& E = e->e;
  activate(E.c);
  const int D = E.m.D;
  std::vector<eng::Request> reqs(b->n);
  for (int i = 0; i < b->n; ++i) {
    eng::Request& q = reqs[i];
    q.env = b->env_index[i];
    q.obs = b->obs + (size_t)i * D;
    q.reward = b->reward ? b->reward[i] : 0.f;
    q.done = b->done ? b->done[i] : 0;
    q.first = b->first ? b->first[i] : 0;
    q.latency = b->latency ? b->latency[i] : 0.f;
    q.obs_episode = b->obs_episode ? b->obs_episode[i] : 0;
    q.obs_step = b->obs_step ? b->obs_step[i] : 0;
  }
  eng::Result r{disp_env, disp_act, disp_act_cont};
  E.process_batch(reqs, r);
  to_result(r, res);
  VER_API_END
}

ver_status ver_engine_attach_preempt(ver_engine e, ver_preempt p) {
  VER_API_BEGIN
  eng::Engine& E = e->e;
  activate(E.c);
  if (p && p->c->device != E.c->device) config_error("engine: the preemption counter lives on another device");
  if (p && !E.pflag_h) {
    VER_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&E.pflag_h), 2 * sizeof(int), cudaHostAllocMapped));
    VER_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&E.pflag_d), E.pflag_h, 0));
  }
  if (E.pflag_h) E.pflag_h[0] = E.pflag_h[1] = 0;
  E.pre = p;
  VER_API_END
}

ver_status ver_engine_force_close(ver_engine e) {
  VER_API_BEGIN
  e->e.buf().open = false;
  VER_API_END
}

ver_status ver_engine_finalize_bootstraps(ver_engine e) {
  VER_API_BEGIN
  activate(e->e.c);
  e->e.finalize_bootstraps();
  VER_API_END
}

ver_status ver_engine_close(ver_engine e, ver_view* out) {
  VER_API_BEGIN
  activate(e->e.c);
  return ver_rollout_close(&e->e.store, out);
  VER_API_END
}

ver_status ver_engine_state(ver_engine e, int* open, int* committed, int* capacity, int* carryover, int* active) {
  VER_API_BEGIN
  eng::Engine& E = e->e;
  if (open) *open = E.buf().open;
  if (committed) *committed = E.buf().committed;
  if (capacity) *capacity = E.buf().capacity();
  if (carryover) {
    int k = 0;
    for (uint8_t v : E.buf().has_carry) k += v;
    *carryover = k;
  }
  if (active) {
    int k = 0;
    for (const auto& s : E.envs) k += s.parked ? 0 : 1;
    *active = k;
  }
  VER_API_END
}

ver_status ver_engine_hidden(ver_engine e, float* h_out) {
  VER_API_BEGIN
  eng::Engine& E = e->e;
  activate(E.c);
  E.h.download(h_out, (size_t)E.cfg.rollout.N * E.m.H);
  sync(E.c);
  VER_API_END
}

}  // extern "C"
