// rollout.cuh — the host side of the rollout store (rollout.hpp:87-142,
// rollout.cpp:24-100), shared by the C-ABI in rollout.cu and the device
// inference engine (engine.cu), which appends its records through append_rec.
#pragma once
#include <algorithm>
#include <cstring>
#include <string>
#include <thread>
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

// f(lo, hi) over [0, n) in chunks of >= grain, on up to 16 host threads (the
// calling thread takes the first chunk); below 2 grains it runs inline
template <class F>
inline void host_par_for(size_t n, size_t grain, F f) {
  const size_t hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  const size_t T = std::min(hw, std::max<size_t>(1, n / std::max<size_t>(grain, 1)));
  if (T <= 1) {
    f(size_t(0), n);
    return;
  }
  std::vector<std::thread> th;
  th.reserve(T - 1);
  const size_t per = (n + T - 1) / T;
  for (size_t t = 1; t < T; ++t) {
    const size_t lo = std::min(n, t * per), hi = std::min(n, lo + per);
    if (lo < hi) th.emplace_back(f, lo, hi);
  }
  f(size_t(0), std::min(n, per));
  for (auto& x : th) x.join();
}

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
  // rows of the log (and h_before rows) already copied to the device mirror: the
  // bulk append uploads what it wrote right away, close_rollout the rest
  int uploaded = 0, h_uploaded = 0;
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

  // copy log rows [a, z) of every column to the device mirror (sized to capacity)
  void upload_rows(int a, int z) {  // (z == a: only sizes the mirror)
    const size_t C = (size_t)std::max(capacity(), 1), n = (size_t)std::max(z - a, 0);
    auto up = [&](auto& d, auto& h, size_t w) {
      d.reserve(ctx, C * std::max<size_t>(w, 1));
      if (n * w)
        VER_CUDA(cudaMemcpyAsync(d.p + (size_t)a * w, h.p + (size_t)a * w, n * w * sizeof(*h.p), cudaMemcpyHostToDevice,
                               ctx->stream));
    };
    up(d_env, env, 1);
    up(d_rank, rank, 1);
    up(d_hslot, hslot, 1);
    up(d_step, step, 1);
    up(d_obs, obs, (size_t)cfg.obs_dim);
    if (cfg.action_kind) up(d_act_cont, act_cont, (size_t)cfg.act_dim);
    else up(d_act_disc, act_disc, 1);
    up(d_log_prob, log_prob, 1);
    up(d_value, value, 1);
    up(d_reward, reward, 1);
    up(d_latency, latency, 1);
    up(d_done, done, 1);
    up(d_episode, episode, 1);
    up(d_version, version, 1);
  }
  // copy h_before rows [a, z) (the device copy keeps rows [0, a))
  void upload_hrows(int a, int z) {
    const size_t Hd = (size_t)cfg.hidden_dim;
    if (z <= a || !Hd) return;
    d_hlog.grow_keep(ctx, std::max(hlog.n, (size_t)z * Hd), (size_t)a * Hd);
    VER_CUDA(cudaMemcpyAsync(d_hlog.p + (size_t)a * Hd, hlog.p + (size_t)a * Hd, (size_t)(z - a) * Hd * sizeof(float),
                             cudaMemcpyHostToDevice, ctx->stream));
  }

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
    // the pinned log is about to be rewritten: no copy of it may still be in flight
    if (uploaded || h_uploaded) VER_CUDA(cudaStreamSynchronize(ctx->stream));
    uploaded = 0;
    h_uploaded = 0;
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
    const int r0 = committed, D = cfg.obs_dim, Hd = cfg.hidden_dim, NE = cfg.N;
    // Bookkeeping (rollout.cpp:79-93 + the rank / sequence-start log of this
    // store) in parallel over record chunks: (1) per chunk and env the record count
    // and the last record's done flag; (2) a serial prefix over chunks x envs gives
    // each chunk the env's rank and "previous record done" on entry; (3) per chunk
    // the ranks / starts and the chunk's count of h_before rows, whose prefix (4)
    // numbers the rows in record order; (5) columns and rows copied on all threads.
    const size_t hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    const int nch = (int)std::max<size_t>(1, std::min(hw, (size_t)n / 16384));
    const int per = (n + nch - 1) / nch;
    std::vector<int32_t> lc((size_t)nch * NE, 0);    // records of env e in chunk c, then rank base
    std::vector<int8_t> ld((size_t)nch * NE, -1);    // last record's done in chunk c (-1: none), then done on entry
    std::vector<int32_t> hcount(nch + 1, 0);
    auto chunks = [&](auto f) {
      host_par_for((size_t)nch, 1, [&](size_t lo, size_t hi) {
        for (size_t c = lo; c < hi; ++c) f((int)c, i0 + (int)c * per, i0 + std::min(n, ((int)c + 1) * per));
      });
    };
    chunks([&](int c, int a, int z) {
      int32_t* l = lc.data() + (size_t)c * NE;
      int8_t* d = ld.data() + (size_t)c * NE;
      for (int i = a; i < z; ++i) {
        const int e = b->env_index[i];
        ++l[e];
        d[e] = b->done[i] ? 1 : 0;
      }
    });
    for (int e = 0; e < NE; ++e) {
      int32_t base = counts[e];
      int8_t prev = (int8_t)last_done[e];
      for (int c = 0; c < nch; ++c) {
        const size_t q = (size_t)c * NE + e;
        const int32_t cnt = lc[q];
        const int8_t dl = ld[q];
        lc[q] = base;
        ld[q] = prev;
        base += cnt;
        if (cnt) prev = dl;
      }
      counts[e] = base;
      last_done[e] = (uint8_t)prev;
    }
    const bool hb = b->h_before != nullptr;
    chunks([&](int c, int a, int z) {
      int32_t* base = lc.data() + (size_t)c * NE;
      int8_t* prev = ld.data() + (size_t)c * NE;
      int32_t nh = 0;
      for (int i = a; i < z; ++i) {
        const int e = b->env_index[i];
        const int rk = base[e]++;
        const uint8_t dn = b->done[i] ? 1 : 0;
        int hs = -2;
        if (rk == 0 || prev[e] == 1) hs = (hb && (!b->h_before_valid || b->h_before_valid[i])) ? nh++ : -1;
        prev[e] = (int8_t)dn;
        const int r = r0 + (i - i0);
        rank.p[r] = rk;
        hslot.p[r] = hs;  // chunk-local row number for now
        done.p[r] = dn;
      }
      hcount[c + 1] = nh;
    });
    for (int c = 0; c < nch; ++c) hcount[c + 1] += hcount[c];
    const int h0 = h_used, nh_tot = hcount[nch];
    if (nh_tot) hlog.ensure((size_t)(h_used + nh_tot) * Hd, (size_t)h_used * Hd);
    h_used += nh_tot;
    auto col = [&](auto* dst, const auto* src, size_t width, auto fill, size_t lo, size_t hi) {
      if (src) std::memcpy(dst + (r0 + lo) * width, src + (i0 + lo) * width, sizeof(*dst) * width * (hi - lo));
      else std::fill(dst + (r0 + lo) * width, dst + (r0 + hi) * width, fill);
    };
    // rows committed one by one since the last upload (carryovers, append_one), then
    // each chunk's rows as soon as they are in the pinned log: the H2D copies overlap
    // the other chunks' host copies instead of waiting for close_rollout
    const bool early = ctx != nullptr;
    if (early) {
      upload_rows(uploaded, r0);
      upload_hrows(h_uploaded, h0);
      if (nh_tot) d_hlog.grow_keep(ctx, std::max(hlog.n, (size_t)(h0 + nh_tot) * Hd), (size_t)h0 * Hd);
      upload_rows(r0, r0);  // sizes every device column to capacity before the threads use them
    }
    chunks([&](int c, int a, int z) {
      const size_t lo = (size_t)(a - i0), hi = (size_t)(z - i0);
      col(env.p, b->env_index, 1, 0, lo, hi);
      col(episode.p, b->episode_index, 1, (int64_t)0, lo, hi);
      col(step.p, b->step_in_episode, 1, 0, lo, hi);
      col(obs.p, b->obs, D, 0.f, lo, hi);
      if (cfg.action_kind) col(act_cont.p, b->act_cont, cfg.act_dim, 0.f, lo, hi);
      else col(act_disc.p, b->act_disc, 1, 0, lo, hi);
      col(log_prob.p, b->log_prob, 1, 0.f, lo, hi);
      col(value.p, b->value, 1, 0.f, lo, hi);
      col(reward.p, b->reward, 1, 0.f, lo, hi);
      col(latency.p, b->latency, 1, 0.f, lo, hi);
      col(version.p, b->snapshot_version, 1, (uint64_t)0, lo, hi);
      // this chunk's h_before rows, numbered after the earlier chunks' in record order
      const int hb0 = h0 + hcount[c];
      for (size_t q = lo; q < hi; ++q) {
        int32_t& hs = hslot.p[r0 + q];
        if (hs >= 0) {
          hs += hb0;
          std::memcpy(hlog.p + (size_t)hs * Hd, b->h_before + (i0 + q) * Hd, sizeof(float) * Hd);
        }
      }
      if (early) {
        VER_CUDA(cudaSetDevice(ctx->device));  // a worker thread
        upload_rows(r0 + (int)lo, r0 + (int)hi);
        if (Hd && hcount[c + 1] > hcount[c])
          VER_CUDA(cudaMemcpyAsync(d_hlog.p + (size_t)hb0 * Hd, hlog.p + (size_t)hb0 * Hd,
                                   (size_t)(hcount[c + 1] - hcount[c]) * Hd * sizeof(float), cudaMemcpyHostToDevice,
                                   ctx->stream));
      }
    });
    if (early) {
      uploaded = r0 + n;
      h_uploaded = h_used;
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
