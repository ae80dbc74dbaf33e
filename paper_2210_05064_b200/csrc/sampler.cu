// sampler.cu — minibatch construction (packseq.cpp, learner.cpp:56-70).
//
// split_minibatches (packseq.cpp:10-54):
//   host : perm = std::shuffle(iota(K), std::mt19937_64(seed)) — libstdc++'s
//          shuffle is implementation-defined, so it runs on the host with the
//          same libstdc++ the reference links (O(K) ints, bit-exact).
//   device: dealt lengths -> exclusive scan -> every group boundary inside a
//          sequence splits it; piece p of sequence i lands in group
//          grp(cum_i) + p with skip += (piece start - cum_i).
// pack (packseq.cpp:56-88):
//   stable sort by length desc as a sort of unique keys
//   ((INT_MAX - len) << 32 | index), batch_sizes[t] = #{len > t} by binary
//   search on the sorted lengths, offsets = exclusive scan, slots by
//   binary search of offsets.  All integer, bit-exact.
// gather: time-major copy of obs / action / old log-prob / A / R by slot.
#include <algorithm>
#include <numeric>
#include <random>

#include "packed.cuh"

namespace verg {

__device__ __forceinline__ int group_of(long long x, int base, int rem) {
  const long long big = (long long)rem * (base + 1);
  if (x < big) return (int)(x / (base + 1));
  return rem + (int)((x - big) / base);
}
__device__ __forceinline__ long long group_start(int b, int base, int rem) {
  return (long long)b * base + min(b, rem);
}

__global__ void dealt_lengths_kernel(const ver_seq_desc* __restrict__ seqs, const int32_t* __restrict__ order,
                                     int n, int32_t* __restrict__ lens) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) lens[i] = seqs[order[i]].length;
}

__global__ void piece_count_kernel(const int32_t* __restrict__ lens, const int32_t* __restrict__ cum, int n,
                                   int base, int rem, int32_t* __restrict__ np) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int len = lens[i];
  if (len <= 0) {
    np[i] = 0;
    return;
  }
  const long long c0 = cum[i];
  np[i] = group_of(c0 + len - 1, base, rem) - group_of(c0, base, rem) + 1;
}

// packseq.cpp:35-52
__global__ void piece_write_kernel(const ver_seq_desc* __restrict__ seqs, const int32_t* __restrict__ order,
                                   const int32_t* __restrict__ lens, const int32_t* __restrict__ cum,
                                   const int32_t* __restrict__ poff, int n, int base, int rem,
                                   ver_seq_desc* __restrict__ pieces, int32_t* __restrict__ pgroup) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int len = lens[i];
  if (len <= 0) return;
  const ver_seq_desc src = seqs[order[i]];
  const long long c0 = cum[i], c1 = c0 + len;
  int b = group_of(c0, base, rem);
  int q = poff[i];
  for (long long lo = c0; lo < c1; ++b) {
    const long long hi = min(c1, group_start(b + 1, base, rem));
    if (hi <= lo) continue;  // zero-capacity group (base == 0 tail)
    ver_seq_desc part = src;
    part.length = (int)(hi - lo);
    part.start_offset = src.start_offset + (int)(lo - c0);
    part.skip = src.skip + (int)(lo - c0);
    pieces[q] = part;
    pgroup[q] = b;
    ++q;
    lo = hi;
  }
}

__global__ void group_start_kernel(const int32_t* __restrict__ pgroup, int P, int32_t* __restrict__ gstart) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  if (p == 0 || pgroup[p] != pgroup[p - 1]) gstart[pgroup[p]] = p;
}

static DGroups* split_in_order(DView& V, int B, const int32_t* order, int n) {
  if (B < 1) protocol_error("split_minibatches: B must be >= 1");
  const int total = V.size;
  if (total == 0) protocol_error("split_minibatches: empty view");
  if (total == V.T * V.N && total % B != 0)
    protocol_error("split_minibatches: B=" + std::to_string(B) + " does not divide T*N=" +
                   std::to_string(total));
  for (int i = 0; i < n; ++i)
    if (order[i] < 0 || order[i] >= V.num_seqs) protocol_error("split_in_order: sequence index out of range");
  Ctx* c = V.ctx;
  const int base = total / B, rem = total % B;
  auto* G = new DGroups();
  G->ctx = c;
  G->B = B;
  G->total = total;
  const int nn = std::max(n, 1);
  DBuf<int32_t> buf;
  buf.reserve(c, 4 * (size_t)nn + 2 + B + 1);
  int32_t* d_order = buf.p;
  int32_t* lens = d_order + nn;
  int32_t* cum = lens + nn;
  int32_t* np = cum + nn;
  int32_t* sums = np + nn;  // [0] dealt, [1] pieces
  int32_t* gstart = sums + 2;
  int32_t* hbuf = static_cast<int32_t*>(c->pinned_buf(sizeof(int32_t) * (size_t)std::max(nn, B + 3)));
  std::copy(order, order + n, hbuf);
  VER_CUDA(cudaMemcpyAsync(d_order, hbuf, sizeof(int32_t) * n, cudaMemcpyHostToDevice, c->stream));
  if (n > 0) {
    dealt_lengths_kernel<<<cdiv(n, 256), 256, 0, c->stream>>>(V.seqs.p, d_order, n, lens);
    after_launch(c);
  }
  exclusive_scan_i32(c, lens, cum, n, sums);
  if (n > 0) {
    piece_count_kernel<<<cdiv(n, 256), 256, 0, c->stream>>>(lens, cum, n, base, rem, np);
    after_launch(c);
  }
  exclusive_scan_i32(c, np, np, n, sums + 1);  // np -> piece offsets
  VER_CUDA(cudaMemcpyAsync(hbuf, sums, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  const int dealt = hbuf[0], P = hbuf[1];
  if (dealt > total) protocol_error("split_in_order: dealt more steps than the view holds");
  G->dealt = dealt;
  G->pieces.reserve(c, std::max(P, 1));
  DBuf<int32_t> pgroup;
  pgroup.reserve(c, std::max(P, 1));
  if (n > 0) {
    piece_write_kernel<<<cdiv(n, 256), 256, 0, c->stream>>>(V.seqs.p, d_order, lens, cum, np, n, base, rem,
                                                            G->pieces.p, pgroup.p);
    after_launch(c);
  }
  VER_CUDA(cudaMemsetAsync(gstart, 0xff, sizeof(int32_t) * (B + 1), c->stream));
  if (P > 0) {
    group_start_kernel<<<cdiv(P, 256), 256, 0, c->stream>>>(pgroup.p, P, gstart);
    after_launch(c);
  }
  VER_CUDA(cudaMemcpyAsync(hbuf, gstart, sizeof(int32_t) * (B + 1), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  G->gstart.assign(hbuf, hbuf + B + 1);
  G->gstart[B] = P;
  for (int b = B - 1; b >= 0; --b)
    if (G->gstart[b] < 0) G->gstart[b] = G->gstart[b + 1];
  G->gsteps.resize(B);
  for (int b = 0; b < B; ++b) {
    const long long g0 = (long long)b * base + std::min(b, rem);
    const long long cap = base + (b < rem ? 1 : 0);
    G->gsteps[b] = (int)std::max(0LL, std::min(cap, (long long)dealt - g0));
  }
  return G;
}

// packseq.cpp:10-16: the epoch permutation (host libstdc++)
std::vector<int32_t> shuffle_perm(int n, uint64_t seed) {
  std::vector<int32_t> perm(n);
  std::iota(perm.begin(), perm.end(), 0);
  std::mt19937_64 gen(seed);
  std::shuffle(perm.begin(), perm.end(), gen);
  return perm;
}

DGroups* split_minibatches(DView& V, int B, uint64_t seed) {
  auto perm = shuffle_perm(V.num_seqs, seed);
  return split_in_order(V, B, perm.data(), (int)perm.size());
}

// ------------------------------------------------------------------- pack
__global__ void pack_keys_kernel(const ver_seq_desc* __restrict__ pieces, int k, uint64_t* __restrict__ keys) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < k) keys[j] = ((uint64_t)(0x7fffffff - pieces[j].length) << 32) | (uint32_t)j;
}
__global__ void pack_sorted_kernel(const ver_seq_desc* __restrict__ pieces, const uint64_t* __restrict__ keys,
                                   int k, ver_seq_desc* __restrict__ sorted, int32_t* __restrict__ s2g,
                                   int32_t* __restrict__ lens) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= k) return;
  const int g = (int)(keys[j] & 0xffffffffu);
  const ver_seq_desc d = pieces[g];
  sorted[j] = d;
  s2g[j] = g;
  lens[j] = d.length;
}
// batch_sizes[t] = #{j : len_j > t}; lens sorted descending
__global__ void batch_sizes_kernel(const int32_t* __restrict__ lens, int k, int T, int32_t* __restrict__ bs) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  int lo = 0, hi = k;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (lens[mid] > t) lo = mid + 1;
    else hi = mid;
  }
  bs[t] = lo;
}
// Time-major gather (learner.cpp:56-70) + slots (packseq.cpp:78-85) as a
// shared-memory transpose.  Tile = 32 consecutive sorted pieces x 32
// timesteps.  Read phase: each warp reads one piece's consecutive view slots,
// i.e. two contiguous runs (the slots' learner records, 16 B each at D = 2,
// and their (A, R) pairs; view.cuh), so a short piece wastes at most the
// partial DRAM sectors at the ends of two runs, not of five fields.  Write
// phase: each warp writes one timestep's 32 consecutive packed rows per field
// (coalesced: rows offsets[t] + j, j = 0..bs_t-1).  Algorithmic bytes:
// SURVEY §8d's 8D+36 B/step including the 4-byte slot.
constexpr int kGT = 32;  // pieces per tile
// Tile table entry: {piece block jb, (t0 << 3) | log2(TT)}.  TT (timesteps
// per tile, power of two <= 32) follows the block's longest piece, so blocks
// of short pieces (the sorted tail of a heavy-tailed length distribution)
// still fill the CTA: the read phase maps lanes to (piece, t) pairs.
// view loads of the gather: ld.global.cg (L2 only; measured 11% faster than
// ld.global.cs at C5 2^26, r02g)
template <class T>
__device__ __forceinline__ T gld(const T* p) {
  return __ldcg(p);
}
__global__ void __launch_bounds__(256) gather_tiled_kernel(
    const int2* __restrict__ tiles, const ver_seq_desc* __restrict__ sorted, int k,
    const int32_t* __restrict__ offs, const int32_t* __restrict__ bs, int32_t* __restrict__ slots,
    const float* __restrict__ v_rec, int rs, const float* __restrict__ v_ar,
    float* __restrict__ obs, int32_t* __restrict__ act, float* __restrict__ actc, float* __restrict__ lp,
    float* __restrict__ adv, float* __restrict__ ret, int D, int A, int continuous, int ntiles, int S) {
  extern __shared__ float tl[];  // F fields x 32 pieces x 33 (padded)
  __shared__ int s_start[kGT], s_len[kGT];
  const int2 te = tiles[blockIdx.x];
  const int jb = te.x, t0 = te.y >> 3, lg = te.y & 7, TT = 1 << lg;
  const int j0 = jb * kGT;
  const int AC = continuous ? A : 0;
  if (threadIdx.x < kGT) {
    const int j = j0 + threadIdx.x;
    s_start[threadIdx.x] = j < k ? sorted[j].start_offset : 0;
    s_len[threadIdx.x] = j < k ? sorted[j].length : 0;
  }
  __syncthreads();
  auto cell = [&](int f, int jl, int tt) -> float& { return tl[(f * kGT + jl) * (kGT + 1) + tt]; };
  // read: lanes -> (piece jl, timestep tt), tt fastest: a piece's slots are contiguous
  for (int r = threadIdx.x; r < kGT * TT; r += blockDim.x) {
    const int jl = r >> lg, tt = r & (TT - 1);
    const int t = t0 + tt;
    if (t < s_len[jl]) {
      const int sl = s_start[jl] + t;
      int f = 0;
      const float2 arv = gld(reinterpret_cast<const float2*>(v_ar) + sl);  // (A, R)
      if (rs == 4 && !continuous) {  // D = 2 discrete: the whole record in one 16-byte load
        const float4 r4 = gld(reinterpret_cast<const float4*>(v_rec) + sl);
        cell(f++, jl, tt) = r4.x;
        cell(f++, jl, tt) = r4.y;
        cell(f++, jl, tt) = r4.w;
        cell(f++, jl, tt) = arv.x;
        cell(f++, jl, tt) = arv.y;
        cell(f++, jl, tt) = r4.z;  // action bits
      } else {
        const float* rc = v_rec + (size_t)sl * rs;
        for (int q = 0; q < D; ++q) cell(f++, jl, tt) = gld(rc + q);
        for (int q = 0; q < AC; ++q) cell(f++, jl, tt) = gld(rc + D + q);
        cell(f++, jl, tt) = gld(rc + rs - 1);
        cell(f++, jl, tt) = arv.x;
        cell(f++, jl, tt) = arv.y;
        if (!continuous) cell(f++, jl, tt) = gld(rc + D);
      }
    }
  }
  __syncthreads();
  // write: lanes -> (timestep tt, piece jl), jl fastest: rows offsets[t] + j are contiguous
  for (int r = threadIdx.x; r < kGT * TT; r += blockDim.x) {
    const int tt = r >> 5, jl = r & 31;
    const int t = t0 + tt;
    if (t >= s_len[0]) continue;  // the block's first piece is its longest
    if (j0 + jl < bs[t]) {
      const size_t p = (size_t)offs[t] + j0 + jl;
      slots[p] = s_start[jl] + t;
      int f = 0;
      if (D == 2) {
        const float a0 = cell(f++, jl, tt), a1 = cell(f++, jl, tt);
        reinterpret_cast<float2*>(obs)[p] = make_float2(a0, a1);
      } else {
        for (int q = 0; q < D; ++q) obs[p * D + q] = cell(f++, jl, tt);
      }
      for (int q = 0; q < AC; ++q) actc[p * A + q] = cell(f++, jl, tt);
      lp[p] = cell(f++, jl, tt);
      adv[p] = cell(f++, jl, tt);
      ret[p] = cell(f++, jl, tt);
      if (!continuous) act[p] = __float_as_int(cell(f++, jl, tt));
    }
  }
}

// launch of the tiled gather over an existing pack (P.seqs / lens / offs / bs set)
void gather_packed(DView& V, DPacked& P) {
  Ctx* c = V.ctx;
  if (P.tile_table.empty()) {
    const int nblk = (P.k + kGT - 1) / kGT;
    for (int b = 0; b < nblk; ++b) {
      const int Lb = P.h_seqs[b * kGT].length;
      int lg = 0;
      while ((1 << lg) < Lb && lg < 5) ++lg;
      const int TT = 1 << lg;
      for (int t0 = 0; t0 < Lb; t0 += TT) P.tile_table.push_back(int2{b, (t0 << 3) | lg});
    }
    P.tiles.reserve(c, P.tile_table.size());
    P.tiles.upload(P.tile_table.data(), P.tile_table.size());
    sync(c);
  }
  const int F = V.obs_dim + (V.action_kind ? V.act_dim : 0) + 3 + (V.action_kind ? 0 : 1);
  const size_t smem = sizeof(float) * (size_t)F * kGT * (kGT + 1);
  auto kern = gather_tiled_kernel;
  if (smem > 48 * 1024)
    VER_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  ScopedEv ev(c, c->hbm_tag >= 0 ? c->hbm_tag + 1 : -1);
  kern<<<(unsigned)P.tile_table.size(), 256, smem, c->stream>>>(
      P.tiles.p, P.seqs.p, P.k, P.offs.p, P.bs.p, P.slots.p, V.rec.p, V.rs(), V.ar.p, P.obs.p, P.act_disc.p,
      P.act_cont.p, P.old_logp.p, P.adv.p, P.ret.p, V.obs_dim,
      V.act_dim, V.action_kind, (int)P.tile_table.size(), V.size);
  after_launch(c);
}

DPacked* pack_pieces(DView& V, const ver_seq_desc* d_pieces, int k) {
  if (k <= 0) protocol_error("pack: empty sequence group");
  Ctx* c = V.ctx;
  auto* P = new DPacked();
  P->ctx = c;
  P->k = k;
  P->obs_dim = V.obs_dim;
  P->act_dim = V.act_dim;
  P->action_kind = V.action_kind;
  P->hidden_dim = V.hidden_dim;
  P->seqs.reserve(c, k);
  P->s2g.reserve(c, k);
  P->lens.reserve(c, k);
  DBuf<uint64_t> keys;
  keys.reserve(c, k);
  pack_keys_kernel<<<cdiv(k, 256), 256, 0, c->stream>>>(d_pieces, k, keys.p);
  after_launch(c);
  sort_u64(c, keys.p, k);
  pack_sorted_kernel<<<cdiv(k, 256), 256, 0, c->stream>>>(d_pieces, keys.p, k, P->seqs.p, P->s2g.p, P->lens.p);
  after_launch(c);
  // L and S_mb to the host: they size the per-timestep launches
  P->h_seqs.resize(k);
  P->seqs.download(P->h_seqs.data(), k);
  sync(c);
  const int L = P->h_seqs[0].length;
  long long tot = 0;
  for (const auto& d : P->h_seqs) tot += d.length;
  if (L <= 0) protocol_error("pack: empty sequence group");
  P->max_len = L;
  P->total = (int)tot;
  P->bs.reserve(c, L + 1);
  P->offs.reserve(c, L + 1);
  batch_sizes_kernel<<<cdiv(L, 256), 256, 0, c->stream>>>(P->lens.p, k, L, P->bs.p);
  after_launch(c);
  exclusive_scan_i32(c, P->bs.p, P->offs.p, L, P->offs.p + L);
  const int S = P->total;
  P->slots.reserve(c, S);
  P->obs.reserve(c, (size_t)S * V.obs_dim);
  if (V.action_kind) P->act_cont.reserve(c, (size_t)S * V.act_dim);
  else P->act_disc.reserve(c, S);
  P->old_logp.reserve(c, S);
  P->adv.reserve(c, S);
  P->ret.reserve(c, S);
  gather_packed(V, *P);
  P->h_bs.resize(L);
  P->h_offs.resize(L);
  P->bs.download(P->h_bs.data(), L);
  P->offs.download(P->h_offs.data(), L);
  sync(c);
  return P;
}

}  // namespace verg

using namespace verg;

extern "C" {

ver_status ver_split_minibatches(ver_view v, int B, uint64_t seed, ver_groups* out) {
  VER_API_BEGIN
  activate(v->v.ctx);
  DGroups* G = split_minibatches(v->v, B, seed);
  auto* h = new ver_groups_s();
  h->g = std::move(*G);
  delete G;
  *out = h;
  VER_API_END
}

ver_status ver_split_in_order(ver_view v, int B, const int32_t* order, int n, ver_groups* out) {
  VER_API_BEGIN
  activate(v->v.ctx);
  DGroups* G = split_in_order(v->v, B, order, n);
  auto* h = new ver_groups_s();
  h->g = std::move(*G);
  delete G;
  *out = h;
  VER_API_END
}

ver_status ver_groups_count(ver_groups g, int* B) {
  VER_API_BEGIN
  *B = g->g.B;
  VER_API_END
}

ver_status ver_groups_get(ver_groups g, int b, int* num_seqs, int* total_steps, ver_seq_desc* seqs) {
  VER_API_BEGIN
  DGroups& G = g->g;
  if (b < 0 || b >= G.B) config_error("ver_groups_get: group index out of range");
  const int k = G.gstart[b + 1] - G.gstart[b];
  if (num_seqs) *num_seqs = k;
  if (total_steps) *total_steps = G.gsteps[b];
  if (seqs && k) {
    activate(G.ctx);
    VER_CUDA(cudaMemcpyAsync(seqs, G.pieces.p + G.gstart[b], sizeof(ver_seq_desc) * k,
                             cudaMemcpyDeviceToHost, G.ctx->stream));
    sync(G.ctx);
  }
  VER_API_END
}

ver_status ver_groups_destroy(ver_groups g) {
  VER_API_BEGIN
  if (g) {
    activate(g->g.ctx);
    delete g;
  }
  VER_API_END
}

ver_status ver_pack(ver_view v, ver_groups g, int b, ver_packed* out) {
  VER_API_BEGIN
  DGroups& G = g->g;
  if (b < 0 || b >= G.B) config_error("ver_pack: group index out of range");
  activate(v->v.ctx);
  DPacked* P = pack_pieces(v->v, G.pieces.p + G.gstart[b], G.gstart[b + 1] - G.gstart[b]);
  auto* h = new ver_packed_s();
  h->p = std::move(*P);
  delete P;
  *out = h;
  VER_API_END
}

ver_status ver_pack_seqs(ver_view v, const ver_seq_desc* seqs, int k, ver_packed* out) {
  VER_API_BEGIN
  if (k <= 0) protocol_error("pack: empty sequence group");
  Ctx* c = v->v.ctx;
  activate(c);
  DBuf<ver_seq_desc> d;
  d.reserve(c, k);
  d.upload(seqs, k);
  DPacked* P = pack_pieces(v->v, d.p, k);
  auto* h = new ver_packed_s();
  h->p = std::move(*P);
  delete P;
  *out = h;
  VER_API_END
}

ver_status ver_packed_info(ver_packed p, int* num_seqs, int* max_len, int* total_steps) {
  VER_API_BEGIN
  if (num_seqs) *num_seqs = p->p.k;
  if (max_len) *max_len = p->p.max_len;
  if (total_steps) *total_steps = p->p.total;
  VER_API_END
}

ver_status ver_packed_get(ver_packed p, ver_seq_desc* seqs, int32_t* s2g, int32_t* bs, int32_t* offs,
                          int32_t* slots) {
  VER_API_BEGIN
  DPacked& P = p->p;
  activate(P.ctx);
  if (seqs) P.seqs.download(seqs, P.k);
  if (s2g) P.s2g.download(s2g, P.k);
  if (bs) P.bs.download(bs, P.max_len);
  if (offs) P.offs.download(offs, P.max_len);
  if (slots) P.slots.download(slots, P.total);
  sync(P.ctx);
  VER_API_END
}

ver_status ver_packed_get_gathered(ver_packed p, float* obs, int32_t* act_disc, float* act_cont,
                                   float* old_logp, float* adv, float* ret) {
  VER_API_BEGIN
  DPacked& P = p->p;
  activate(P.ctx);
  const size_t S = P.total;
  if (obs) P.obs.download(obs, S * P.obs_dim);
  if (act_disc && !P.action_kind) P.act_disc.download(act_disc, S);
  if (act_cont && P.action_kind) P.act_cont.download(act_cont, S * P.act_dim);
  if (old_logp) P.old_logp.download(old_logp, S);
  if (adv) P.adv.download(adv, S);
  if (ret) P.ret.download(ret, S);
  sync(P.ctx);
  VER_API_END
}

ver_status ver_packed_destroy(ver_packed p) {
  VER_API_BEGIN
  if (p) {
    activate(p->p.ctx);
    delete p;
  }
  VER_API_END
}

}  // extern "C"
