// rollout.cuh — the host side of the rollout store (rollout.hpp:87-142,
// rollout.cpp:24-100), shared by the C-ABI in rollout.cu and the device
// inference engine (engine.cu), which appends its records through append_rec.
#pragma once
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "view.cuh"

namespace verg {

// ------------------------------------------------------------ RolloutBuffer
template <class T>
struct Pinned {
  T* p = nullptr;
  size_t n = 0;
  ~Pinned() {
    if (p) cudaFreeHost(p);
  }
  void ensure(size_t count, size_t keep = 0) {
    if (count <= n) return;
    size_t want = std::max(count, n * 2);
    T* q = nullptr;
    VER_CUDA(cudaMallocHost(reinterpret_cast<void**>(&q), std::max<size_t>(want, 1) * sizeof(T)));
    if (p && keep) std::memcpy(q, p, keep * sizeof(T));
    if (p) cudaFreeHost(p);
    p = q;
    n = want;
  }
};

struct CarryRec {
  int32_t env, step;
  int64_t episode;
  std::vector<float> obs, act_cont, h;
  int32_t act_disc;
  float log_prob, value, reward, latency;
  uint8_t done, has_h;
  uint8_t h_dev;  // h_before is row `env` of the device carry buffer (engine records)
  uint64_t version;
};

struct Rollout {
  Ctx* ctx = nullptr;
  ver_rollout_config cfg{};
  bool open = false;
  uint64_t snapshot_version = 0;
  int committed = 0;
  std::vector<int32_t> counts;
  std::vector<uint8_t> last_done;
  int envs_at_cap = 0;
  std::vector<CarryRec> carry;
  std::vector<uint8_t> has_carry;
  std::vector<float> bootstrap;
  std::vector<uint8_t> bootstrap_valid;
  int next_seq_id = 0;
  // pinned arrival log (capacity T*N)
  Pinned<int32_t> env, rank, hslot, act_disc, step;
  Pinned<float> obs, act_cont, log_prob, value, reward, latency, hlog;
  Pinned<uint8_t> done;
  Pinned<int64_t> episode;
  Pinned<uint64_t> version;
  int h_used = 0;
  // device mirror
  DBuf<int32_t> d_env, d_rank, d_hslot, d_act_disc, d_step;
  DBuf<float> d_obs, d_act_cont, d_log_prob, d_value, d_reward, d_latency, d_hlog;
  DBuf<uint8_t> d_done;
  DBuf<int64_t> d_episode;
  DBuf<uint64_t> d_version;
  // h_before rows of sequence-starting records that come from the device
  // inference engine (engine.cu): copied device to device at commit (hslot
  // -3 - row), never through the host; d_carry_h holds a parked record's row
  DBuf<float> d_hdev, d_carry_h;
  int h_dev_used = 0;

  int capacity() const { return cfg.T * cfg.N; }

  void init() {
    const int C = capacity();
    counts.assign(cfg.N, 0);
    last_done.assign(cfg.N, 0);
    carry.resize(cfg.N);
    has_carry.assign(cfg.N, 0);
    bootstrap.assign(cfg.N, 0.f);
    bootstrap_valid.assign(cfg.N, 0);
    env.ensure(C);
    rank.ensure(C);
    hslot.ensure(C);
    step.ensure(C);
    obs.ensure((size_t)C * cfg.obs_dim);
    if (cfg.action_kind) act_cont.ensure((size_t)C * cfg.act_dim);
    else act_disc.ensure(C);
    log_prob.ensure(C);
    value.ensure(C);
    reward.ensure(C);
    latency.ensure(C);
    done.ensure(C);
    episode.ensure(C);
    version.ensure(C);
    hlog.ensure((size_t)std::max(1, cfg.N) * cfg.hidden_dim);
  }

  bool env_at_cap(int e) const { return cfg.mode == 0 && counts[e] >= cfg.T; }

  // rollout.cpp:79-93 (rank / sequence-start bookkeeping added)
  void commit(int32_t e, int64_t episode_, int32_t step_, const float* obs_, int32_t act_d,
              const float* act_c, float lp, float v, float rw, float lat, uint8_t dn,
              const float* h, uint64_t ver, const float* h_dev = nullptr) {
    const int r = committed;
    const int rk = counts[e];
    const bool start = rk == 0 || last_done[e];
    int hs = -2;
    if (start) {
      if (h) {
        hlog.ensure((size_t)(h_used + 1) * cfg.hidden_dim, (size_t)h_used * cfg.hidden_dim);
        std::memcpy(hlog.p + (size_t)h_used * cfg.hidden_dim, h, sizeof(float) * cfg.hidden_dim);
        hs = h_used++;
      } else if (h_dev && cfg.hidden_dim > 0) {
        const size_t H = cfg.hidden_dim;
        if ((size_t)(h_dev_used + 1) * H > d_hdev.n)
          d_hdev.grow_keep(ctx, std::max<size_t>((size_t)(h_dev_used + 1) * H, 2 * d_hdev.n), (size_t)h_dev_used * H);
        VER_CUDA(cudaMemcpyAsync(d_hdev.p + (size_t)h_dev_used * H, h_dev, H * sizeof(float),
                                 cudaMemcpyDeviceToDevice, ctx->stream));
        hs = -3 - h_dev_used++;
      } else {
        hs = -1;
      }
    }
    env.p[r] = e;
    rank.p[r] = rk;
    hslot.p[r] = hs;
    episode.p[r] = episode_;
    step.p[r] = step_;
    std::memcpy(obs.p + (size_t)r * cfg.obs_dim, obs_, sizeof(float) * cfg.obs_dim);
    if (cfg.action_kind) std::memcpy(act_cont.p + (size_t)r * cfg.act_dim, act_c, sizeof(float) * cfg.act_dim);
    else act_disc.p[r] = act_d;
    log_prob.p[r] = lp;
    value.p[r] = v;
    reward.p[r] = rw;
    latency.p[r] = lat;
    done.p[r] = dn;
    version.p[r] = ver;
    ++committed;
    ++counts[e];
    last_done[e] = dn;
    if (cfg.mode == 1) {
      if (committed >= capacity()) open = false;
    } else {
      if (counts[e] == cfg.T) ++envs_at_cap;
      if (envs_at_cap >= cfg.N) open = false;
    }
  }

  // rollout.cpp:39-57
  void begin(uint64_t sv) {
    open = true;
    snapshot_version = sv;
    committed = 0;
    h_used = 0;
    h_dev_used = 0;
    envs_at_cap = 0;
    std::fill(counts.begin(), counts.end(), 0);
    std::fill(last_done.begin(), last_done.end(), 0);
    std::fill(bootstrap.begin(), bootstrap.end(), 0.f);
    std::fill(bootstrap_valid.begin(), bootstrap_valid.end(), 0);
    for (int e = 0; e < cfg.N && open; ++e) {
      if (has_carry[e]) {
        has_carry[e] = 0;
        const CarryRec& c = carry[e];
        commit(c.env, c.episode, c.step, c.obs.data(), c.act_disc, c.act_cont.data(), c.log_prob,
               c.value, c.reward, c.latency, c.done, c.has_h ? c.h.data() : nullptr, c.version,
               c.h_dev ? d_carry_h.p + (size_t)e * cfg.hidden_dim : nullptr);
      }
    }
  }

  // rollout.cpp:59-77 for record i of the batch
  int append_one(const ver_step_batch* b, int i) {
    const int e = b->env_index[i];
    if (e < 0 || e >= cfg.N) protocol_error("append_step: env_index out of range");
    const float* h = nullptr;
    if (b->h_before && (!b->h_before_valid || b->h_before_valid[i]))
      h = b->h_before + (size_t)i * cfg.hidden_dim;
    const float* o = b->obs + (size_t)i * cfg.obs_dim;
    const float* ac = cfg.action_kind ? b->act_cont + (size_t)i * cfg.act_dim : nullptr;
    const int32_t ad = cfg.action_kind ? 0 : b->act_disc[i];
    const int64_t ep = b->episode_index ? b->episode_index[i] : 0;
    const int32_t st = b->step_in_episode ? b->step_in_episode[i] : 0;
    const float lat = b->latency ? b->latency[i] : 0.f;
    const uint64_t ver = b->snapshot_version ? b->snapshot_version[i] : 0;
    return append_rec(e, ep, st, o, ad, ac, b->log_prob[i], b->value[i], b->reward[i], lat, b->done[i] ? 1 : 0, h,
                      nullptr, ver);
  }

  // Variable-mode fast path of a batch (same outcome as append_one per record):
  // while the store stays open every record commits, so the payload columns are
  // block-copied into the arrival log and only rank / sequence-start / h_before
  // bookkeeping runs per record.  Returns how many records [i0, i0 + k) it took.
  int append_bulk(const ver_step_batch* b, int i0) {
    if (cfg.mode != 1 || !open) return 0;
    int n = std::min(b->n - i0, capacity() - committed);
    for (int i = 0; i < n; ++i)  // a bad env index stops the fast path there (append_one throws)
      if (b->env_index[i0 + i] < 0 || b->env_index[i0 + i] >= cfg.N) {
        n = i;
        break;
      }
    if (n <= 0) return 0;
    const int r0 = committed, D = cfg.obs_dim;
    auto col = [&](auto* dst, const auto* src, size_t width, auto fill) {
      if (src) std::memcpy(dst + (size_t)r0 * width, src + (size_t)i0 * width, sizeof(*dst) * width * n);
      else std::fill(dst + (size_t)r0 * width, dst + (size_t)(r0 + n) * width, fill);
    };
    col(env.p, b->env_index, 1, 0);
    col(episode.p, b->episode_index, 1, (int64_t)0);
    col(step.p, b->step_in_episode, 1, 0);
    col(obs.p, b->obs, D, 0.f);
    if (cfg.action_kind) col(act_cont.p, b->act_cont, cfg.act_dim, 0.f);
    else col(act_disc.p, b->act_disc, 1, 0);
    col(log_prob.p, b->log_prob, 1, 0.f);
    col(value.p, b->value, 1, 0.f);
    col(reward.p, b->reward, 1, 0.f);
    col(latency.p, b->latency, 1, 0.f);
    col(version.p, b->snapshot_version, 1, (uint64_t)0);
    for (int i = 0; i < n; ++i) {
      const int e = b->env_index[i0 + i];
      const int rk = counts[e];
      const uint8_t dn = b->done[i0 + i] ? 1 : 0;
      int hs = -2;
      if (rk == 0 || last_done[e]) {
        const bool has = b->h_before && (!b->h_before_valid || b->h_before_valid[i0 + i]);
        if (has) {
          hlog.ensure((size_t)(h_used + 1) * cfg.hidden_dim, (size_t)h_used * cfg.hidden_dim);
          std::memcpy(hlog.p + (size_t)h_used * cfg.hidden_dim, b->h_before + (size_t)(i0 + i) * cfg.hidden_dim,
                      sizeof(float) * cfg.hidden_dim);
          hs = h_used++;
        } else {
          hs = -1;
        }
      }
      rank.p[r0 + i] = rk;
      hslot.p[r0 + i] = hs;
      done.p[r0 + i] = dn;
      counts[e] = rk + 1;
      last_done[e] = dn;
    }
    committed += n;
    if (committed >= capacity()) open = false;
    return n;
  }

  // one record; h_before from the host (h) or from device memory (h_dev: the
  // inference engine's pending row, copied device to device)
  int append_rec(int e, int64_t ep, int32_t st, const float* o, int32_t ad, const float* ac, float lp, float v,
                 float rw, float lat, uint8_t dn, const float* h, const float* h_dev, uint64_t ver) {
    if (e < 0 || e >= cfg.N) protocol_error("append_step: env_index out of range");
    if (!open) {
      if (cfg.mode == 1) {
        if (has_carry[e])
          protocol_error("append_step: two pending carryovers for env " + std::to_string(e));
        CarryRec& c = carry[e];
        c.env = e;
        c.step = st;
        c.episode = ep;
        c.obs.assign(o, o + cfg.obs_dim);
        if (ac) c.act_cont.assign(ac, ac + cfg.act_dim);
        c.act_disc = ad;
        c.log_prob = lp;
        c.value = v;
        c.reward = rw;
        c.latency = lat;
        c.done = dn;
        c.has_h = h != nullptr;
        if (h) c.h.assign(h, h + cfg.hidden_dim);
        c.h_dev = (!h && h_dev && cfg.hidden_dim > 0) ? 1 : 0;
        if (c.h_dev) {
          d_carry_h.reserve(ctx, (size_t)cfg.N * cfg.hidden_dim);
          VER_CUDA(cudaMemcpyAsync(d_carry_h.p + (size_t)e * cfg.hidden_dim, h_dev, sizeof(float) * cfg.hidden_dim,
                                   cudaMemcpyDeviceToDevice, ctx->stream));
        }
        c.version = ver;
        has_carry[e] = 1;
      }
      return 1;
    }
    if (env_at_cap(e)) return 1;
    commit(e, ep, st, o, ad, ac, lp, v, rw, lat, dn, h, ver, h_dev);
    return 0;
  }
};


// close_rollout (rollout.cpp:102-190): the device compaction of the arrival log
DView* close_rollout(Rollout* R);

}  // namespace verg

struct ver_rollout_s {
  verg::Rollout r;
};
