// rollout.cu — the ragged rollout store (rollout.hpp:87-142, rollout.cpp).
//
// Host side: the per-record append protocol (open/closed, Fixed-mode caps,
// per-env carryover, rollout.cpp:39-100) is O(1) integer bookkeeping per
// record and stays on the host thread, writing the payload into a pinned
// arrival log.  For every record it fixes the record's rank within its env
// and whether it starts a sequence, so `h_before` is stored only for
// sequence-starting records (the reference copies it on every commit,
// rollout.cpp:81, but reads it only at :155).
//
// Device side (close_rollout, rollout.cpp:102-190): one H2D of the log, then
//   offsets   = exclusive_scan(per_env_counts)                    [N]
//   scatter   : slot = offsets[env] + rank, all payload fields     [S]
//   seq ids   = exclusive_scan(start flags)                        [S]
//   descriptors + h0 gather                                        [K]
// and backfill_stale (rollout.cpp:208-276) as a stable partition + length
// prefix sum + gather-append.
#include <algorithm>
#include <cstring>

#include "rollout.cuh"

namespace verg {

// ------------------------------------------------------------ DView alloc
void DView::alloc_slots(int c) {
  cap = c;
  rec.reserve(ctx, (size_t)c * rs());
  ar.reserve(ctx, (size_t)c * 2);
  value.reserve(ctx, c);
  reward.reserve(ctx, c);
  latency.reserve(ctx, c);
  done.reserve(ctx, c);
  stale.reserve(ctx, c);
  replayed.reserve(ctx, c);
  env_index.reserve(ctx, c);
  seq_of_slot.reserve(ctx, c);
  step_in_episode.reserve(ctx, c);
  episode_index.reserve(ctx, c);
  version.reserve(ctx, c);
}
void DView::grow_slots(int c) {
  if (c <= cap) return;
  const size_t s = size;
  rec.grow_keep(ctx, (size_t)c * rs(), s * rs());
  ar.grow_keep(ctx, (size_t)c * 2, s * 2);
  value.grow_keep(ctx, c, s);
  reward.grow_keep(ctx, c, s);
  latency.grow_keep(ctx, c, s);
  done.grow_keep(ctx, c, s);
  stale.grow_keep(ctx, c, s);
  replayed.grow_keep(ctx, c, s);
  env_index.grow_keep(ctx, c, s);
  seq_of_slot.grow_keep(ctx, c, s);
  step_in_episode.grow_keep(ctx, c, s);
  episode_index.grow_keep(ctx, c, s);
  version.grow_keep(ctx, c, s);
  cap = c;
}
void DView::alloc_seqs(int sc, int hc) {
  seq_cap = sc;
  h0_cap = hc;
  seqs.reserve(ctx, sc);
  h0.reserve(ctx, (size_t)hc * hidden_dim);
}
void DView::grow_seqs(int sc, int hc) {
  if (sc > seq_cap) {
    seqs.grow_keep(ctx, sc, num_seqs);
    seq_cap = sc;
  }
  if (hc > h0_cap) {
    h0.grow_keep(ctx, (size_t)hc * hidden_dim, (size_t)h0_rows * hidden_dim);
    h0_cap = hc;
  }
}
void DView::alloc_env() {
  per_env_counts.reserve(ctx, N);
  env_offsets.reserve(ctx, N + 1);
  env_bootstrap.reserve(ctx, N);
  env_bootstrap_valid.reserve(ctx, N);
}

// --------------------------------------------------------------- kernels
struct LogDev {  // device mirror of the arrival log (SoA)
  const int32_t *env, *rank, *hslot;
  const float* obs;
  const int32_t* act_disc;
  const float* act_cont;
  const float *log_prob, *value, *reward, *latency;
  const uint8_t* done;
  const int64_t* episode;
  const int32_t* step;
  const uint64_t* version;
};

struct ViewDev {  // raw pointers of a DView for kernels
  float* rec;  // rs floats per slot: obs[D] | action | log_prob
  float* ar;   // advantage, returns per slot
  int rs;
  float *value, *reward, *latency;
  uint8_t *done, *stale, *replayed;
  int32_t *env_index, *seq_of_slot, *step_in_episode;
  int64_t* episode_index;
  uint64_t* version;
  ver_seq_desc* seqs;
  float* h0;
};
static ViewDev vdev(DView& v) {
  return ViewDev{v.rec.p,      v.ar.p,        v.rs(),          v.value.p,           v.reward.p,
                 v.latency.p,  v.done.p,      v.stale.p,       v.replayed.p,        v.env_index.p,
                 v.seq_of_slot.p, v.step_in_episode.p, v.episode_index.p, v.version.p, v.seqs.p,
                 v.h0.p};
}

// Scatter of the arrival log into env-major view order (rollout.cpp:143-181).
// One thread per record; every field write is to slot offsets[env]+rank.
__global__ void compact_scatter_kernel(LogDev L, ViewDev V, const int32_t* __restrict__ offsets,
                                       const int32_t* __restrict__ counts, int S, int D, int A, int continuous,
                                       uint8_t* __restrict__ start_flag,
                                       int32_t* __restrict__ hslot_by_slot) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= S) return;
  const int e = L.env[r];
  const int dst = offsets[e] + L.rank[r];
  float* rc = V.rec + (size_t)dst * V.rs;
  for (int j = 0; j < D; ++j) rc[j] = L.obs[(size_t)r * D + j];
  if (continuous) {
    for (int j = 0; j < A; ++j) rc[D + j] = L.act_cont[(size_t)r * A + j];
  } else {
    rc[D] = __int_as_float(L.act_disc[r]);
  }
  rc[V.rs - 1] = L.log_prob[r];
  V.value[dst] = L.value[r];
  V.reward[dst] = L.reward[r];
  V.latency[dst] = L.latency[r];
  reinterpret_cast<float2*>(V.ar)[dst] = make_float2(0.f, 0.f);
  // bit 0: done; bit 1: last fresh slot of its env (the GAE scan's segment tail)
  V.done[dst] = (L.done[r] ? 1 : 0) | (L.rank[r] == counts[e] - 1 ? 2 : 0);
  V.stale[dst] = 0;
  V.replayed[dst] = 0;
  V.env_index[dst] = e;
  V.episode_index[dst] = L.episode[r];
  V.step_in_episode[dst] = L.step[r];
  V.version[dst] = L.version[r];
  const int hs = L.hslot[r];
  start_flag[dst] = hs != -2 ? 1 : 0;
  hslot_by_slot[dst] = hs;
}

// seq_of_slot and sequence starts from the exclusive scan of start flags.
__global__ void seq_ids_kernel(const uint8_t* __restrict__ flag, const int32_t* __restrict__ excl,
                               int S, int32_t* __restrict__ seq_of_slot, int32_t* __restrict__ starts) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= S) return;
  const int f = flag[i];
  const int k = excl[i] + f - 1;
  seq_of_slot[i] = k;
  if (f) starts[k] = i;
}

// Descriptor + h0 row per sequence (rollout.cpp:147-160, 185-188): one block each.
__global__ void seq_desc_kernel(const int32_t* __restrict__ starts, int K, int S, int seq_id_base,
                                const int32_t* __restrict__ env_index,
                                const int32_t* __restrict__ hslot_by_slot,
                                const float* __restrict__ hlog, const float* __restrict__ hdev, int H,
                                ver_seq_desc* __restrict__ seqs, float* __restrict__ h0) {
  const int k = blockIdx.x;
  if (k >= K) return;
  const int st = starts[k];
  if (threadIdx.x == 0) {
    const int nx = (k + 1 < K) ? starts[k + 1] : S;
    ver_seq_desc d;
    d.seq_id = seq_id_base + k;
    d.env_index = env_index[st];
    d.length = nx - st;
    d.start_offset = st;
    d.h0_index = k;
    d.stale = 0;
    d.parent_start_offset = st;
    d.skip = 0;
    seqs[k] = d;
  }
  const int hs = hslot_by_slot ? hslot_by_slot[st] : -1;
  float* dst = h0 + (size_t)k * H;
  if (hs >= 0 || hs <= -3) {  // host-logged row, or a device row of the inference engine
    const float* src = hs >= 0 ? hlog + (size_t)hs * H : hdev + (size_t)(-3 - hs) * H;
    for (int j = threadIdx.x; j < H; j += blockDim.x) dst[j] = src[j];
  } else {
    for (int j = threadIdx.x; j < H; j += blockDim.x) dst[j] = 0.f;
  }
}

static void upload_log(Rollout* R, int S) {
  // what the bulk appends have not already copied
  R->upload_rows(R->uploaded, S);
  R->upload_hrows(R->h_uploaded, R->h_used);
  if (!R->d_hlog.p) R->d_hlog.reserve(R->ctx, 1);  // seq_desc_kernel takes a valid pointer
  R->uploaded = S;
  R->h_uploaded = R->h_used;
}

// rollout.cpp:102-190
DView* close_rollout(Rollout* R) {
  if (R->committed == 0) protocol_error("close_rollout: buffer is empty");
  if (R->open) protocol_error("close_rollout: buffer still open (force_close for preemption)");
  Ctx* c = R->ctx;
  const auto& cfg = R->cfg;
  const int S = R->committed;
  upload_log(R, S);

  auto* V = new DView();
  V->ctx = c;
  V->T = cfg.T;
  V->N = cfg.N;
  V->action_kind = cfg.action_kind;
  V->obs_dim = cfg.obs_dim;
  V->act_dim = cfg.act_dim;
  V->hidden_dim = cfg.hidden_dim;
  V->size = S;
  V->deficit = R->capacity() - S;
  V->snapshot_version = R->snapshot_version;
  V->env_contiguous = true;
  V->fresh_prefix = S;
  V->alloc_slots(std::max(S, R->capacity()));
  V->alloc_env();
  V->per_env_counts.upload(R->counts.data(), cfg.N);
  V->env_bootstrap.upload(R->bootstrap.data(), cfg.N);
  V->env_bootstrap_valid.upload(R->bootstrap_valid.data(), cfg.N);
  // env offsets: exclusive scan of the per-env counts; offsets[N] = S
  exclusive_scan_i32(c, V->per_env_counts.p, V->env_offsets.p, cfg.N, V->env_offsets.p + cfg.N);

  DBuf<uint8_t> flag;
  DBuf<int32_t> hsl, excl, starts, K;
  flag.reserve(c, S);
  hsl.reserve(c, S);
  excl.reserve(c, S);
  starts.reserve(c, S);
  K.reserve(c, 1);
  LogDev L{R->d_env.p,      R->d_rank.p,    R->d_hslot.p,  R->d_obs.p,     R->d_act_disc.p,
           R->d_act_cont.p, R->d_log_prob.p, R->d_value.p, R->d_reward.p,  R->d_latency.p,
           R->d_done.p,     R->d_episode.p, R->d_step.p,   R->d_version.p};
  ViewDev VD = vdev(*V);
  compact_scatter_kernel<<<cdiv(S, 256), 256, 0, c->stream>>>(
      L, VD, V->env_offsets.p, V->per_env_counts.p, S, cfg.obs_dim, cfg.act_dim, cfg.action_kind, flag.p, hsl.p);
  after_launch(c);
  exclusive_scan_u8(c, flag.p, excl.p, S, K.p);
  seq_ids_kernel<<<cdiv(S, 256), 256, 0, c->stream>>>(flag.p, excl.p, S, V->seq_of_slot.p, starts.p);
  after_launch(c);
  int32_t* hK = static_cast<int32_t*>(c->pinned_buf(sizeof(int32_t)));
  K.download(hK, 1);
  sync(c);
  const int nK = *hK;
  V->num_seqs = nK;
  V->h0_rows = nK;
  V->alloc_seqs(nK + V->deficit, nK + V->deficit);
  seq_desc_kernel<<<std::max(nK, 1), 128, 0, c->stream>>>(starts.p, nK, S, R->next_seq_id,
                                                           V->env_index.p, hsl.p, R->d_hlog.p, R->d_hdev.p,
                                                           cfg.hidden_dim, V->seqs.p, V->h0.p);
  after_launch(c);
  R->next_seq_id += nK;
  return V;
}

// ---------------------------------------------------- synthetic ragged view
// Device generator of a closed, env-contiguous view for the ragged-length
// stress sweep: env e holds lengths[e] steps; counter-hash
// payload; done ~ Bernoulli(p_done) inside each env; sequence structure built
// with the same scan + descriptor kernels as close_rollout.
__device__ __forceinline__ uint64_t hmix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ float hunif(uint64_t seed, uint64_t i, uint64_t f) {
  return (float)((hmix(seed ^ hmix(i * 64 + f)) >> 40) * (1.0 / 16777216.0));
}
__device__ __forceinline__ float hnorm(uint64_t seed, uint64_t i, uint64_t f) {
  const float u1 = fmaxf(hunif(seed, i, f), 1e-7f), u2 = hunif(seed, i, f + 32);
  return sqrtf(-2.f * logf(u1)) * cospif(2.f * u2);
}
__global__ void synth_view_kernel(const int32_t* __restrict__ off, uint64_t seed, float p_done, ViewDev V, int D,
                                  uint8_t* __restrict__ flag, float* __restrict__ boot, uint8_t* __restrict__ valid) {
  const int e = blockIdx.x;
  const int s0 = off[e], len = off[e + 1] - s0;
  for (int t = threadIdx.x; t < len; t += blockDim.x) {
    const int i = s0 + t;
    float* rc = V.rec + (size_t)i * V.rs;
    for (int q = 0; q < D; ++q) rc[q] = hnorm(seed, i, 1 + q);
    rc[D] = __int_as_float((int)(hmix(seed ^ hmix((uint64_t)i * 64 + 20)) & 1));
    rc[D + 1] = -0.6931472f + 0.1f * hnorm(seed, i, 21);
    V.value[i] = hnorm(seed, i, 22);
    V.reward[i] = hnorm(seed, i, 23);
    V.latency[i] = 0.f;
    reinterpret_cast<float2*>(V.ar)[i] = make_float2(0.f, 0.f);
    const bool d = hunif(seed, i, 24) < p_done;
    V.done[i] = (d ? 1 : 0) | (t == len - 1 ? 2 : 0);
    V.stale[i] = 0;
    V.replayed[i] = 0;
    V.env_index[i] = e;
    V.episode_index[i] = (int64_t)e * 1000;
    V.step_in_episode[i] = t;
    V.version[i] = 1;
    flag[i] = (t == 0 || hunif(seed, i - 1, 24) < p_done) ? 1 : 0;
    if (t == len - 1) {
      valid[e] = d ? 0 : 1;
      boot[e] = d ? 0.f : hnorm(seed, i, 25);
    }
  }
}

static DView* synth_view(Ctx* c, const int32_t* lengths, int N, int obs_dim, int hidden_dim, uint64_t seed,
                         float p_done) {
  long long S = 0;
  for (int e = 0; e < N; ++e) {
    if (lengths[e] < 1) config_error("view_synth: lengths must be >= 1");
    S += lengths[e];
  }
  if (S > 0x7fffffffLL) config_error("view_synth: more than 2^31-1 steps");
  auto* V = new DView();
  V->ctx = c;
  V->T = 0;
  V->N = N;
  V->obs_dim = obs_dim;
  V->hidden_dim = hidden_dim;
  V->size = (int)S;
  V->env_contiguous = true;
  V->fresh_prefix = (int)S;
  V->alloc_slots((int)S);
  V->alloc_env();
  V->per_env_counts.upload(lengths, N);
  exclusive_scan_i32(c, V->per_env_counts.p, V->env_offsets.p, N, V->env_offsets.p + N);
  DBuf<uint8_t> flag;
  DBuf<int32_t> excl, starts, K;
  flag.reserve(c, S);
  excl.reserve(c, S);
  starts.reserve(c, S);
  K.reserve(c, 1);
  ViewDev VD = vdev(*V);
  synth_view_kernel<<<N, 256, 0, c->stream>>>(V->env_offsets.p, seed, p_done, VD, obs_dim, flag.p,
                                              V->env_bootstrap.p, V->env_bootstrap_valid.p);
  after_launch(c);
  exclusive_scan_u8(c, flag.p, excl.p, S, K.p);
  seq_ids_kernel<<<cdiv(S, 256), 256, 0, c->stream>>>(flag.p, excl.p, (int)S, V->seq_of_slot.p, starts.p);
  after_launch(c);
  int32_t* hK = static_cast<int32_t*>(c->pinned_buf(sizeof(int32_t)));
  K.download(hK, 1);
  sync(c);
  const int nK = *hK;
  V->num_seqs = nK;
  V->h0_rows = nK;
  V->alloc_seqs(nK, nK);
  seq_desc_kernel<<<std::max(nK, 1), 128, 0, c->stream>>>(starts.p, nK, (int)S, 0, V->env_index.p, nullptr, nullptr,
                                                           nullptr, hidden_dim, V->seqs.p, V->h0.p);
  after_launch(c);
  sync(c);
  return V;
}

// ------------------------------------------------------------ backfill
__global__ void max_seq_id_kernel(const ver_seq_desc* __restrict__ seqs, int K, int32_t* __restrict__ out) {
  __shared__ int32_t red[32];
  int m = 0;  // rollout.cpp:214: max over seq ids, starting at 0
  for (int i = threadIdx.x; i < K; i += blockDim.x) m = max(m, seqs[i].seq_id);
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0;
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) *out = m;
  }
}

__global__ void nonstale_flags_kernel(const ver_seq_desc* __restrict__ seqs, int K, uint8_t* __restrict__ f) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < K) f[i] = seqs[i].stale ? 0 : 1;
}

// stable partition: non-stale first (rollout.cpp:217-224); lengths in that order
__global__ void backfill_order_kernel(const ver_seq_desc* __restrict__ seqs, int K,
                                      const uint8_t* __restrict__ f, const int32_t* __restrict__ excl,
                                      const int32_t* __restrict__ n_ns, int32_t* __restrict__ ord,
                                      int32_t* __restrict__ lens) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= K) return;
  const int pos = f[i] ? excl[i] : (*n_ns + (i - excl[i]));
  ord[pos] = i;
  lens[pos] = seqs[i].length;
}

__global__ void backfill_count_kernel(const int32_t* __restrict__ cum, int K, int deficit,
                                      int32_t* __restrict__ n_taken) {
  // cum is non-decreasing: count j with cum[j] < deficit by binary search
  if (threadIdx.x != 0) return;
  int lo = 0, hi = K;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (cum[mid] < deficit) lo = mid + 1;
    else hi = mid;
  }
  *n_taken = lo;
}

// rollout.cpp:229-243: descriptor + h0 row of every taken sequence (block each)
__global__ void backfill_desc_kernel(const ver_seq_desc* __restrict__ pseqs, const float* __restrict__ ph0,
                                     const int32_t* __restrict__ ord, const int32_t* __restrict__ cum,
                                     const int32_t* __restrict__ n_taken, const int32_t* __restrict__ max_id,
                                     int deficit, int S, int K, int h0_rows, int H,
                                     ver_seq_desc* __restrict__ seqs, float* __restrict__ h0) {
  const int j = blockIdx.x;
  if (j >= *n_taken) return;
  const ver_seq_desc src = pseqs[ord[j]];
  if (threadIdx.x == 0) {
    ver_seq_desc d;
    d.seq_id = *max_id + 1 + j;
    d.env_index = src.env_index;
    d.length = min(src.length, deficit - cum[j]);
    d.start_offset = S + cum[j];
    d.parent_start_offset = S + cum[j];
    d.h0_index = h0_rows + j;
    d.stale = 1;
    d.skip = 0;
    seqs[K + j] = d;
  }
  const float* s = ph0 + (size_t)src.h0_index * H;
  float* t = h0 + (size_t)(h0_rows + j) * H;
  for (int u = threadIdx.x; u < H; u += blockDim.x) t[u] = s[u];
}

// rollout.cpp:244-269: gather-append of the taken steps (thread per new slot)
__global__ void backfill_slots_kernel(ViewDev P, ViewDev V, const ver_seq_desc* __restrict__ pseqs,
                                      const int32_t* __restrict__ ord, const int32_t* __restrict__ cum,
                                      const int32_t* __restrict__ n_taken, int deficit, int S, int K,
                                      int D, int A, int continuous) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= deficit) return;
  int lo = 0, hi = *n_taken - 1;  // largest j with cum[j] <= q
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (cum[mid] <= q) lo = mid;
    else hi = mid - 1;
  }
  const int j = lo;
  const int sp = pseqs[ord[j]].start_offset + (q - cum[j]);
  const int dst = S + q;
  for (int k = 0; k < V.rs; ++k) V.rec[(size_t)dst * V.rs + k] = P.rec[(size_t)sp * P.rs + k];
  V.value[dst] = P.value[sp];
  V.reward[dst] = P.reward[sp];
  V.latency[dst] = P.latency[sp];
  reinterpret_cast<float2*>(V.ar)[dst] = reinterpret_cast<const float2*>(P.ar)[sp];
  V.done[dst] = P.done[sp] & 1;  // replayed slots carry no segment-tail bit
  V.stale[dst] = 1;
  V.replayed[dst] = 1;
  V.env_index[dst] = P.env_index[sp];
  V.seq_of_slot[dst] = K + j;
  V.episode_index[dst] = P.episode_index[sp];
  V.step_in_episode[dst] = P.step_in_episode[sp];
  V.version[dst] = P.version[sp];
}

static void backfill_stale(DView& V, DView& P, int deficit) {
  if (deficit == 0) return;
  if (deficit < 0) protocol_error("backfill_stale: negative deficit");
  if (deficit > P.size) protocol_error("backfill_stale: deficit exceeds previous rollout size");
  if (V.obs_dim != P.obs_dim || V.action_kind != P.action_kind || V.hidden_dim != P.hidden_dim ||
      V.act_dim != P.act_dim)
    config_error("backfill_stale: views have different shapes");
  Ctx* c = V.ctx;
  const int K = V.num_seqs, Kp = P.num_seqs, S = V.size;
  V.grow_slots(S + deficit);
  V.grow_seqs(K + std::min(deficit, Kp), V.h0_rows + std::min(deficit, Kp));
  DBuf<int32_t> scratch;
  scratch.reserve(c, 4 + 3 * (size_t)std::max(Kp, 1));
  int32_t* max_id = scratch.p;
  int32_t* n_ns = scratch.p + 1;
  int32_t* n_taken = scratch.p + 2;
  int32_t* excl = scratch.p + 4;
  int32_t* ord = excl + Kp;
  int32_t* lens = ord + Kp;
  DBuf<uint8_t> f;
  f.reserve(c, std::max(Kp, 1));
  max_seq_id_kernel<<<1, 1024, 0, c->stream>>>(V.seqs.p, K, max_id);
  after_launch(c);
  nonstale_flags_kernel<<<cdiv(Kp, 256), 256, 0, c->stream>>>(P.seqs.p, Kp, f.p);
  after_launch(c);
  exclusive_scan_u8(c, f.p, excl, Kp, n_ns);
  backfill_order_kernel<<<cdiv(Kp, 256), 256, 0, c->stream>>>(P.seqs.p, Kp, f.p, excl, n_ns, ord, lens);
  after_launch(c);
  exclusive_scan_i32(c, lens, lens, Kp, nullptr);  // lens -> cum
  backfill_count_kernel<<<1, 32, 0, c->stream>>>(lens, Kp, deficit, n_taken);
  after_launch(c);
  int32_t* hn = static_cast<int32_t*>(c->pinned_buf(sizeof(int32_t)));
  VER_CUDA(cudaMemcpyAsync(hn, n_taken, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  const int taken = *hn;
  backfill_desc_kernel<<<std::max(taken, 1), 128, 0, c->stream>>>(
      P.seqs.p, P.h0.p, ord, lens, n_taken, max_id, deficit, S, K, V.h0_rows, V.hidden_dim,
      V.seqs.p, V.h0.p);
  after_launch(c);
  ViewDev PD = vdev(P), VD = vdev(V);
  backfill_slots_kernel<<<cdiv(deficit, 256), 256, 0, c->stream>>>(
      PD, VD, P.seqs.p, ord, lens, n_taken, deficit, S, K, V.obs_dim, V.act_dim, V.action_kind);
  after_launch(c);
  V.size += deficit;
  V.num_seqs += taken;
  V.h0_rows += taken;
  V.stale_steps += deficit;
  V.replayed_steps += deficit;
}

// ------------------------------------------------------------- restale
__global__ void restale_kernel(const uint64_t* __restrict__ version, uint8_t* __restrict__ stale, int S,
                               uint64_t lv, int32_t* __restrict__ count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  int add = 0;
  if (i < S && version[i] != lv && !stale[i]) {
    stale[i] = 1;
    add = 1;
  }
  add = __reduce_add_sync(0xffffffffu, add);
  if ((threadIdx.x & 31) == 0 && add) atomicAdd(count, add);
}

// ------------------------------------------------------- upload/download
// record / pair columns <-> the reference's separate arrays (4-byte words, so
// the int32 action bits travel as they are)
__global__ void unpack_cols_kernel(const uint32_t* __restrict__ src, int stride, int off, int width, int n,
                                   uint32_t* __restrict__ dst) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= (size_t)n * width) return;
  const size_t i = k / width, j = k % width;
  dst[k] = src[i * stride + off + j];
}
__global__ void pack_cols_kernel(const uint32_t* __restrict__ src, int width, int n, uint32_t* __restrict__ dst,
                                 int stride, int off) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= (size_t)n * width) return;
  const size_t i = k / width, j = k % width;
  dst[i * stride + off + j] = src[k];
}
// host array (n x width 4-byte words) -> columns [off, off + width) of the strided device buffer
static void up_cols(Ctx* c, float* dst, int stride, int off, const void* h, int width, int n) {
  if (!n || !width) return;
  if (!h) config_error("ver_view_upload: missing array");
  DBuf<uint32_t> tmp;
  tmp.reserve(c, (size_t)n * width);
  tmp.upload(static_cast<const uint32_t*>(h), (size_t)n * width);
  pack_cols_kernel<<<cdiv((size_t)n * width, 256), 256, 0, c->stream>>>(tmp.p, width, n,
                                                                          reinterpret_cast<uint32_t*>(dst), stride, off);
  after_launch(c);
  sync(c);  // tmp and the (possibly pageable) host array
}
static void down_cols(Ctx* c, const float* src, int stride, int off, void* h, int width, int n) {
  if (!h || !n || !width) return;
  DBuf<uint32_t> tmp;
  tmp.reserve(c, (size_t)n * width);
  unpack_cols_kernel<<<cdiv((size_t)n * width, 256), 256, 0, c->stream>>>(reinterpret_cast<const uint32_t*>(src),
                                                                            stride, off, width, n, tmp.p);
  after_launch(c);
  tmp.download(static_cast<uint32_t*>(h), (size_t)n * width);
  sync(c);
}

template <class T>
static void up_arr(Ctx* c, DBuf<T>& d, const T* h, size_t n) {
  if (n && !h) config_error("ver_view_upload: missing array");
  d.upload(h, n);
}

static DView* upload_view(Ctx* c, const ver_view_host* h) {
  if (h->size < 0 || h->num_seqs < 0 || h->N < 0 || h->hidden_dim < 0 || h->obs_dim < 0)
    config_error("ver_view_upload: negative size");
  auto* V = new DView();
  V->ctx = c;
  V->T = h->T;
  V->N = h->N;
  V->action_kind = h->action_kind;
  V->obs_dim = h->obs_dim;
  V->act_dim = h->act_dim;
  V->hidden_dim = h->hidden_dim;
  V->size = h->size;
  V->num_seqs = h->num_seqs;
  V->h0_rows = h->h0_rows;
  V->deficit = h->deficit;
  V->stale_steps = h->stale_steps;
  V->replayed_steps = h->replayed_steps;
  V->snapshot_version = h->snapshot_version;
  V->collect_wall_time = h->collect_wall_time;
  const int S = h->size;
  V->alloc_slots(std::max(S, 1));
  V->alloc_seqs(std::max(h->num_seqs, 1), std::max(h->h0_rows, 1));
  V->alloc_env();
  const int rs = V->rs(), D = h->obs_dim, AW = V->act_width();
  up_cols(c, V->rec.p, rs, 0, h->obs, D, S);
  if (h->action_kind) up_cols(c, V->rec.p, rs, D, h->act_cont, AW, S);
  else up_cols(c, V->rec.p, rs, D, h->act_disc, 1, S);
  up_cols(c, V->rec.p, rs, rs - 1, h->log_prob, 1, S);
  up_arr(c, V->value, h->value, S);
  up_arr(c, V->reward, h->reward, S);
  up_arr(c, V->latency, h->latency, S);
  up_cols(c, V->ar.p, 2, 0, h->advantage, 1, S);
  up_cols(c, V->ar.p, 2, 1, h->returns, 1, S);
  std::vector<uint8_t> done_bits;  // filled below once contiguity is known
  up_arr(c, V->stale, h->stale, S);
  up_arr(c, V->replayed, h->replayed, S);
  up_arr(c, V->env_index, h->env_index, S);
  up_arr(c, V->seq_of_slot, h->seq_of_slot, S);
  up_arr(c, V->step_in_episode, h->step_in_episode, S);
  up_arr(c, V->episode_index, h->episode_index, S);
  up_arr(c, V->version, h->version, S);
  up_arr(c, V->seqs, h->seqs, h->num_seqs);
  up_arr(c, V->h0, h->h0, (size_t)h->h0_rows * h->hidden_dim);
  up_arr(c, V->per_env_counts, h->per_env_counts, h->N);
  up_arr(c, V->env_bootstrap, h->env_bootstrap, h->N);
  up_arr(c, V->env_bootstrap_valid, h->env_bootstrap_valid, h->N);
  // Fresh slots env-major contiguous?  (then GAE runs the flat scan directly;
  // otherwise it first stable-sorts the fresh slots by env on the device)
  int fresh = 0;
  while (fresh < S && !h->replayed[fresh]) ++fresh;
  bool contiguous = true;
  for (int i = fresh; i < S && contiguous; ++i)
    if (!h->replayed[i]) contiguous = false;
  for (int i = 1; i < fresh && contiguous; ++i)
    if (h->env_index[i] < h->env_index[i - 1]) contiguous = false;
  for (int i = 0; i < fresh && contiguous; ++i)
    if (h->env_index[i] < 0 || h->env_index[i] >= h->N) contiguous = false;
  V->env_contiguous = contiguous;
  V->fresh_prefix = fresh;
  // done bit 0 as given; bit 1 marks the last fresh slot of each env (GAE segment tail)
  if (S && !h->done) config_error("ver_view_upload: missing array");
  done_bits.assign(h->done, h->done + S);
  for (int i = 0; i < S; ++i) done_bits[i] = done_bits[i] ? 1 : 0;
  if (contiguous)
    for (int i = 0; i < fresh; ++i)
      if (i + 1 == fresh || h->env_index[i + 1] != h->env_index[i]) done_bits[i] |= 2;
  if (S) {
    V->done.upload(done_bits.data(), S);
    sync(c);
  }
  if (contiguous) {
    std::vector<int32_t> off(h->N + 1, 0);
    for (int i = 0; i < fresh; ++i) off[h->env_index[i] + 1]++;
    for (int e = 0; e < h->N; ++e) off[e + 1] += off[e];
    V->env_offsets.upload(off.data(), h->N + 1);
    sync(c);  // `off` is pageable host memory
  }
  return V;
}

template <class T>
static void down_arr(const DBuf<T>& d, T* h, size_t n) {
  if (h) d.download(h, n);
}

static void download_view(DView& V, ver_view_host* h) {
  const int S = V.size, rs = V.rs(), D = V.obs_dim;
  Ctx* c = V.ctx;
  down_cols(c, V.rec.p, rs, 0, h->obs, D, S);
  if (V.action_kind) down_cols(c, V.rec.p, rs, D, h->act_cont, V.act_dim, S);
  else down_cols(c, V.rec.p, rs, D, h->act_disc, 1, S);
  down_cols(c, V.rec.p, rs, rs - 1, h->log_prob, 1, S);
  down_arr(V.value, h->value, S);
  down_arr(V.reward, h->reward, S);
  down_arr(V.latency, h->latency, S);
  down_cols(c, V.ar.p, 2, 0, h->advantage, 1, S);
  down_cols(c, V.ar.p, 2, 1, h->returns, 1, S);
  down_arr(V.done, h->done, S);
  down_arr(V.stale, h->stale, S);
  down_arr(V.replayed, h->replayed, S);
  down_arr(V.env_index, h->env_index, S);
  down_arr(V.seq_of_slot, h->seq_of_slot, S);
  down_arr(V.step_in_episode, h->step_in_episode, S);
  down_arr(V.episode_index, h->episode_index, S);
  down_arr(V.version, h->version, S);
  down_arr(V.seqs, h->seqs, V.num_seqs);
  down_arr(V.h0, h->h0, (size_t)V.h0_rows * V.hidden_dim);
  down_arr(V.per_env_counts, h->per_env_counts, V.N);
  down_arr(V.env_bootstrap, h->env_bootstrap, V.N);
  down_arr(V.env_bootstrap_valid, h->env_bootstrap_valid, V.N);
  sync(V.ctx);
  if (h->done)
    for (int i = 0; i < S; ++i) h->done[i] &= 1;  // drop the internal segment-tail bit
}

template <class T>
static void clone_arr(Ctx* c, DBuf<T>& dst, const DBuf<T>& src, size_t n) {
  if (n)
    VER_CUDA(cudaMemcpyAsync(dst.p, src.p, n * sizeof(T), cudaMemcpyDeviceToDevice, c->stream));
}

static DView* clone_view(DView& V) {
  Ctx* c = V.ctx;
  auto* W = new DView();
  W->ctx = c;
  W->T = V.T;
  W->N = V.N;
  W->action_kind = V.action_kind;
  W->obs_dim = V.obs_dim;
  W->act_dim = V.act_dim;
  W->hidden_dim = V.hidden_dim;
  W->size = V.size;
  W->num_seqs = V.num_seqs;
  W->h0_rows = V.h0_rows;
  W->deficit = V.deficit;
  W->stale_steps = V.stale_steps;
  W->replayed_steps = V.replayed_steps;
  W->snapshot_version = V.snapshot_version;
  W->collect_wall_time = V.collect_wall_time;
  W->env_contiguous = V.env_contiguous;
  W->fresh_prefix = V.fresh_prefix;
  W->alloc_slots(V.cap);
  W->alloc_seqs(V.seq_cap, V.h0_cap);
  W->alloc_env();
  const size_t S = V.size;
  clone_arr(c, W->rec, V.rec, S * V.rs());
  clone_arr(c, W->ar, V.ar, S * 2);
  clone_arr(c, W->value, V.value, S);
  clone_arr(c, W->reward, V.reward, S);
  clone_arr(c, W->latency, V.latency, S);
  clone_arr(c, W->done, V.done, S);
  clone_arr(c, W->stale, V.stale, S);
  clone_arr(c, W->replayed, V.replayed, S);
  clone_arr(c, W->env_index, V.env_index, S);
  clone_arr(c, W->seq_of_slot, V.seq_of_slot, S);
  clone_arr(c, W->step_in_episode, V.step_in_episode, S);
  clone_arr(c, W->episode_index, V.episode_index, S);
  clone_arr(c, W->version, V.version, S);
  clone_arr(c, W->seqs, V.seqs, V.num_seqs);
  clone_arr(c, W->h0, V.h0, (size_t)V.h0_rows * V.hidden_dim);
  clone_arr(c, W->per_env_counts, V.per_env_counts, V.N);
  clone_arr(c, W->env_offsets, V.env_offsets, V.N + 1);
  clone_arr(c, W->env_bootstrap, V.env_bootstrap, V.N);
  clone_arr(c, W->env_bootstrap_valid, V.env_bootstrap_valid, V.N);
  return W;
}

}  // namespace verg

using namespace verg;

extern "C" {

ver_status ver_view_upload(ver_ctx ctx, const ver_view_host* h, ver_view* out) {
  VER_API_BEGIN
  activate(&ctx->c);
  DView* V = upload_view(&ctx->c, h);
  auto* w = new ver_view_s();
  w->v = std::move(*V);
  delete V;
  *out = w;
  VER_API_END
}

ver_status ver_view_info(ver_view v, ver_view_host* h) {
  VER_API_BEGIN
  const DView& V = v->v;
  h->T = V.T;
  h->N = V.N;
  h->action_kind = V.action_kind;
  h->obs_dim = V.obs_dim;
  h->act_dim = V.act_dim;
  h->hidden_dim = V.hidden_dim;
  h->size = V.size;
  h->num_seqs = V.num_seqs;
  h->h0_rows = V.h0_rows;
  h->deficit = V.deficit;
  h->stale_steps = V.stale_steps;
  h->replayed_steps = V.replayed_steps;
  h->snapshot_version = V.snapshot_version;
  h->collect_wall_time = V.collect_wall_time;
  VER_API_END
}

ver_status ver_view_download(ver_view v, ver_view_host* h) {
  VER_API_BEGIN
  activate(v->v.ctx);
  download_view(v->v, h);
  VER_API_END
}

ver_status ver_view_clone(ver_view v, ver_view* out) {
  VER_API_BEGIN
  activate(v->v.ctx);
  DView* W = clone_view(v->v);
  auto* w = new ver_view_s();
  w->v = std::move(*W);
  delete W;
  *out = w;
  VER_API_END
}

ver_status ver_view_destroy(ver_view v) {
  VER_API_BEGIN
  if (v) {
    activate(v->v.ctx);
    delete v;
  }
  VER_API_END
}

ver_status ver_view_restale(ver_view v, uint64_t lv) {
  VER_API_BEGIN
  DView& V = v->v;
  Ctx* c = V.ctx;
  activate(c);
  DBuf<int32_t> cnt;
  cnt.reserve(c, 1);
  cnt.zero(1);
  if (V.size) {
    restale_kernel<<<cdiv(V.size, 256), 256, 0, c->stream>>>(V.version.p, V.stale.p, V.size, lv, cnt.p);
    after_launch(c);
  }
  int32_t* h = static_cast<int32_t*>(c->pinned_buf(4));
  cnt.download(h, 1);
  sync(c);
  V.stale_steps += *h;
  VER_API_END
}

ver_status ver_rollout_create(ver_ctx ctx, const ver_rollout_config* cfg, ver_rollout* out) {
  VER_API_BEGIN
  activate(&ctx->c);
  if (cfg->T < 1 || cfg->N < 1) config_error("rollout: T and N must be >= 1");
  if (cfg->obs_dim < 1 || cfg->hidden_dim < 0) config_error("rollout: bad dims");
  if (cfg->action_kind == 1 && cfg->act_dim < 1) config_error("rollout: continuous needs act_dim");
  auto* h = new ver_rollout_s();
  h->r.ctx = &ctx->c;
  h->r.cfg = *cfg;
  h->r.init();
  *out = h;
  VER_API_END
}

ver_status ver_rollout_destroy(ver_rollout r) {
  VER_API_BEGIN
  if (r) {
    activate(r->r.ctx);
    sync(r->r.ctx);
    delete r;
  }
  VER_API_END
}

ver_status ver_rollout_begin(ver_rollout r, uint64_t sv) {
  VER_API_BEGIN
  // the pinned log may still be read by an in-flight H2D of the last close
  sync(r->r.ctx);
  r->r.begin(sv);
  VER_API_END
}

ver_status ver_rollout_append(ver_rollout r, const ver_step_batch* b, int32_t* outcomes) {
  VER_API_BEGIN
  int i = 0;
  while (i < b->n) {
    const int k = r->r.append_bulk(b, i);
    if (k > 0) {
      if (outcomes) std::fill(outcomes + i, outcomes + i + k, 0);
      i += k;
      continue;
    }
    const int o = r->r.append_one(b, i);
    if (outcomes) outcomes[i] = o;
    ++i;
  }
  VER_API_END
}

ver_status ver_rollout_set_bootstraps(ver_rollout r, int n, const int32_t* env, const float* value) {
  VER_API_BEGIN
  for (int i = 0; i < n; ++i)
    if (env[i] < 0 || env[i] >= r->r.cfg.N) protocol_error("set_bootstrap: env out of range");
  for (int i = 0; i < n; ++i) {
    r->r.bootstrap[env[i]] = value[i];
    r->r.bootstrap_valid[env[i]] = 1;
  }
  VER_API_END
}

ver_status ver_rollout_force_close(ver_rollout r) {
  VER_API_BEGIN
  r->r.open = false;
  VER_API_END
}

ver_status ver_rollout_set_bootstrap(ver_rollout r, int env, float value) {
  VER_API_BEGIN
  if (env < 0 || env >= r->r.cfg.N) protocol_error("set_bootstrap: env out of range");
  r->r.bootstrap[env] = value;
  r->r.bootstrap_valid[env] = 1;
  VER_API_END
}

ver_status ver_rollout_state(ver_rollout r, int* open, int* committed, int* carryover) {
  VER_API_BEGIN
  if (open) *open = r->r.open;
  if (committed) *committed = r->r.committed;
  if (carryover) {
    int n = 0;
    for (auto f : r->r.has_carry) n += f;
    *carryover = n;
  }
  VER_API_END
}

ver_status ver_rollout_close(ver_rollout r, ver_view* out) {
  VER_API_BEGIN
  activate(r->r.ctx);
  DView* V = close_rollout(&r->r);
  auto* w = new ver_view_s();
  w->v = std::move(*V);
  delete V;
  *out = w;
  VER_API_END
}

ver_status ver_view_synth(ver_ctx ctx, const int32_t* lengths, int n_envs, int obs_dim, int hidden_dim,
                          uint64_t seed, float p_done, ver_view* out) {
  VER_API_BEGIN
  activate(&ctx->c);
  DView* V = synth_view(&ctx->c, lengths, n_envs, obs_dim, hidden_dim, seed, p_done);
  auto* w = new ver_view_s();
  w->v = std::move(*V);
  delete V;
  *out = w;
  VER_API_END
}

ver_status ver_backfill_stale(ver_view view, ver_view prev, int deficit) {
  VER_API_BEGIN
  activate(view->v.ctx);
  backfill_stale(view->v, prev->v, deficit);
  VER_API_END
}

}  // extern "C"
