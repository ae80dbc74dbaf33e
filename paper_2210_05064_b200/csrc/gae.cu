// gae.cu — compute_gae (learner.cpp:11-41) as one flat segmented reverse scan.
//
// For fresh slot i of env e (fresh slots env-major contiguous, env e owning
// [off[e], off[e+1]); true for every close_rollout / backfill_stale output):
//   tail_i  = (i + 1 == off[e+1])
//   Vnext_i = tail_i ? (done_i ? 0 : bootstrap[e] (ProtocolError if invalid))
//                    : value[i+1]
//   delta_i = r_i + gamma * Vnext_i * (1 - d_i) - V_i
//   a_i     = tail_i ? 0 : gamma * lambda * (1 - d_i)
//   A_i     = delta_i + a_i * A_{i+1},   R_i = A_i + V_i
// i.e. a reverse scan of the affine maps x -> delta_i + a_i x; env boundaries
// and dones are just a_i = 0, so no segment bookkeeping is needed.  Carries
// and compositions are fp64 (the kernel is HBM-bound; fp64 is free here) so
// 1024-step segments stay inside fp32 rounding of the fp64 reference.
//
// Two launches.  (1) gae_boot_kernel, one thread per env: the bootstrap of
// every env tail that is not done is parked in the advantage word of the
// tail's (A, R) pair (output only, so free scratch until the scan overwrites
// it), missing ones are reported.  (2) gae_scan_kernel: one pass over 512-slot WARP tiles, no block
// barrier and (in practice) no inter-tile waiting.  A warp claims tiles from
// the END of the array (dynamic tile ids) and keeps the next tile in flight in
// a per-warp ring of bulk copies.  Each tile also reads a 128-slot HALO above
// it (r, V, done of the next tile's bottom, which that tile's warp has just
// fetched, so the halo is mostly an L2 hit).  A reset (env tail or done,
// a_i = 0) inside the halo makes the carry A_hi local: the halo's composed
// map is a constant.  Only when the halo has no reset does the tile wait for
// the value A_lo(t-1) = A_hi(t) the tile above publishes; a tile publishes
// exactly when its own bottom 128 slots have no reset, i.e. exactly when the
// tile below will ask.  With heavy-tailed segments (C5: a reset every ~30
// slots) that practically never happens, so the scan streams.
// Per tile: lane l owns 8 consecutive slots of each of the two 256-slot rows
// (+ 4 halo slots): per-item maps and the lane composite sequentially in
// fp32, then one fp64 warp suffix scan per row (the lane composite's discount
// is the exact fp64 (gamma lambda)^8), rows / halo / carry composed in fp64,
// then every slot is written once (float4 stores).
// HBM traffic: r, V (4+4 B), done (1 B) read once, the (A, R) pair (8 B) written once
// = 17 B/step (the halo re-read is an L2 hit), plus 17 B per env tail for
// the bootstrap pass.
//
// Views whose fresh slots are not env-major contiguous (arbitrary uploads,
// e.g. make_view fixtures with env = seq % N) first stable-sort the fresh
// slots by (env, slot) on the device, run the same scan on the gathered
// arrays and scatter back.
#include <algorithm>
#include <cstdlib>

#include "view.cuh"

namespace verg {

constexpr int kGItems = 8;                 // consecutive slots per lane and row
constexpr int kGRow = 32 * kGItems;        // 256 slots
constexpr int kGTile = 2 * kGRow;          // 512 slots
constexpr int kGHalo = 128;                // 4 slots per lane
constexpr int kGSpan = kGTile + kGHalo;
constexpr int kGWarps = 8;                 // warps per CTA
constexpr int kGStages = 2;                // tiles in flight per warp
constexpr int kGClaim = 4;                 // tiles per tile-counter atomic (consecutive, processed in order)
// stage layout (bytes): V [span + 4] | r [span] | done [span]
constexpr int kGOffR = 4 * kGSpan + 16;
constexpr int kGOffD = kGOffR + 4 * kGSpan;
constexpr int kGStageBytes = (kGOffD + kGSpan + 127) & ~127;
constexpr int kGSmem = kGWarps * kGStages * kGStageBytes;

struct GaeTileState {
  double inc;  // A at the tile's first slot (published only when its bottom 128 slots have no reset)
  int flag;    // 0 not yet, 2 published
  int pad;
};

__device__ __forceinline__ uint32_t gsm(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void gae_bulk(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(mbar)
               : "memory");
}
__device__ __forceinline__ void gae_wait(uint32_t a, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "GW_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra GW_WAIT;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}
// tile-state flag protocol: payload store, then a release store of the flag;
// the reader acquire-loads the flag before reading the payload
__device__ __forceinline__ void flag_release(volatile int* f, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
}
__device__ __forceinline__ int flag_acquire(volatile int* f) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
  return v;
}

// learner.cpp:23-27 at env tails: V_next = bootstrap[e] unless done (ProtocolError
// when it was never set).  One thread per env, the value parked in ar[2 tail].
__global__ void gae_boot_kernel(const int32_t* __restrict__ off, const uint8_t* __restrict__ done,
                                const float* __restrict__ boot, const uint8_t* __restrict__ valid, int N,
                                float* __restrict__ ar, int* __restrict__ err_env) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= N) return;
  const int o0 = off[e], o1 = off[e + 1];
  if (o1 <= o0 || (done[o1 - 1] & 1)) return;
  if (!valid[e]) atomicMin(err_env, e);
  ar[2 * (size_t)(o1 - 1)] = boot[e];
}

// Lane composite of n items: x -> b + a x, a = (gamma lambda)^n in fp64 or 0 (a
// reset among the items).  Scan operator: x earlier (lower index), y later.
// fp64 across lanes: a 256-slot row's partial sums reach O(30) at gamma lambda
// near 1, and fp32 roundings of those would cost ~1e-5 of a small A_i.
struct Aff {
  double a, b;
};
__device__ __forceinline__ Aff compose(Aff x, Aff y) { return Aff{x.a * y.a, fma(x.a, y.b, x.b)}; }
__device__ __forceinline__ Aff shfl_down_aff(Aff x, int o) {
  return Aff{__shfl_down_sync(0xffffffffu, x.a, o), __shfl_down_sync(0xffffffffu, x.b, o)};
}
__device__ __forceinline__ Aff shfl_aff(Aff x, int src) {
  return Aff{__shfl_sync(0xffffffffu, x.a, src), __shfl_sync(0xffffffffu, x.b, src)};
}
__device__ __forceinline__ Aff warp_suffix(Aff v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const Aff y = shfl_down_aff(v, o);
    if (lane + o < 32) v = compose(v, y);
  }
  return v;
}

// Persistent CTAs of 8 independent warps.  Progress: a tile only ever waits
// for a lower-numbered (earlier-claimed) tile, and a warp processes its claims
// in order, so the lowest unfinished tile is always at the head of some
// warp's ring and never waits.
__global__ void __launch_bounds__(32 * kGWarps) gae_scan_kernel(
    const float* __restrict__ reward, const float* __restrict__ value, const uint8_t* __restrict__ done,
    const int32_t* __restrict__ env_of, const int32_t* __restrict__ off, const float* __restrict__ boot, int F,
    double gamma, double lambda, float* __restrict__ ar, volatile GaeTileState* tiles, int* tile_counter) {
  extern __shared__ __align__(128) uint8_t gsmem[];
  __shared__ uint64_t s_full[kGWarps][kGStages];
  const int ntiles = (F + kGTile - 1) / kGTile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float gf = (float)gamma, glf = (float)(gamma * lambda);
  const double gld = gamma * lambda, gl2 = gld * gld, gl4 = gl2 * gl2, gl8 = gl4 * gl4;  // lane discounts
  uint8_t* wsm = gsmem + warp * kGStages * kGStageBytes;
  if (lane == 0) {
    for (int s = 0; s < kGStages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(gsm(&s_full[warp][s])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  // claim the next tile and (lane 0) start its bulk copies into stage s when the
  // whole span (+ 4 V) lies below F; otherwise the lanes fill the stage from
  // global memory at processing time (the top tile or two)
  int c_next = 0, c_left = 0;  // lane 0: tiles left of the last counter claim
  auto claim = [&](int s, int& eh) -> int {
    int t = 0;
    if (lane == 0) {
      if (c_left == 0) {
        c_next = atomicAdd(tile_counter, kGClaim);
        c_left = kGClaim;
      }
      t = c_next++;
      --c_left;
      const uint32_t mb = gsm(&s_full[warp][s]);
      const int lo = (ntiles - 1 - t) * kGTile;
      if (t < ntiles && lo + kGTile < F) eh = env_of[lo + kGTile];  // env of the halo's first slot
      if (t < ntiles && lo + kGSpan + 4 <= F) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(9 * kGSpan + 16)
                     : "memory");
        uint8_t* st = wsm + s * kGStageBytes;
        gae_bulk(gsm(st), value + lo, 4 * kGSpan + 16, mb);
        gae_bulk(gsm(st + kGOffR), reward + lo, 4 * kGSpan, mb);
        gae_bulk(gsm(st + kGOffD), done + lo, kGSpan, mb);
      } else {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(mb) : "memory");
      }
    }
    return __shfl_sync(0xffffffffu, t, 0);
  };
  int tq[kGStages], eq[kGStages];
#pragma unroll
  for (int s = 0; s < kGStages; ++s) {
    eq[s] = 0;
    tq[s] = claim(s, eq[s]);
  }

  for (int it = 0;; ++it) {
    const int s = it % kGStages;
    int tid = tq[0], eh = eq[0];
#pragma unroll
    for (int q = 1; q < kGStages; ++q)
      if (s == q) tid = tq[q], eh = eq[q];
    if (tid >= ntiles) break;
    eh = __shfl_sync(0xffffffffu, eh, 0);
    gae_wait(gsm(&s_full[warp][s]), (it / kGStages) & 1);
    const int lo = (ntiles - 1 - tid) * kGTile;
    const int hi = min(F, lo + kGTile);
    uint8_t* st = wsm + s * kGStageBytes;
    float* sv = reinterpret_cast<float*>(st);
    float* sr = reinterpret_cast<float*>(st + kGOffR);
    uint8_t* sd = st + kGOffD;
    if (lo + kGSpan + 4 > F) {  // not bulk-copied: fill from global, inert (tail + done) beyond F
      for (int j = lane; j < kGSpan + 4; j += 32) {
        const int i = lo + j;
        sv[j] = i < F ? value[i] : 0.f;
        if (j < kGSpan) {
          sr[j] = i < F ? reward[i] : 0.f;
          sd[j] = i < F ? done[i] : 3;
        }
      }
      __syncwarp();
    }
    // ---- the two 256-slot rows: lane l owns slots 8l .. 8l+7 of each
    float v[2][kGItems], dl[2][kGItems];
    uint32_t dd[2][2];
    Aff lc[2];
    bool reset0 = false;  // a reset among this lane's row-0 slots (bytes, not the float map)
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int j0 = kGRow * k + kGItems * lane;
      const float4 r0 = *reinterpret_cast<const float4*>(sr + j0), r1 = *reinterpret_cast<const float4*>(sr + j0 + 4);
      const float4 v0 = *reinterpret_cast<const float4*>(sv + j0), v1 = *reinterpret_cast<const float4*>(sv + j0 + 4);
      const uint2 d2 = *reinterpret_cast<const uint2*>(sd + j0);
      const float rr[kGItems] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
      v[k][0] = v0.x; v[k][1] = v0.y; v[k][2] = v0.z; v[k][3] = v0.w;
      v[k][4] = v1.x; v[k][5] = v1.y; v[k][6] = v1.z; v[k][7] = v1.w;
      dd[k][0] = d2.x;
      dd[k][1] = d2.y;
      float vnext = sv[j0 + kGItems];  // the next lane's first slot (row 1 lane 31: the halo's)
      float mb = 0.f;
      bool reset = false;
#pragma unroll
      for (int q = kGItems - 1; q >= 0; --q) {
        const uint32_t b = (dd[k][q >> 2] >> (8 * (q & 3))) & 3u;
        float vn = vnext;
        if (b == 2u) vn = __ldcg(ar + 2 * (size_t)(lo + j0 + q));  // env tail, not done: its bootstrap
        const float mask = (b & 1u) ? 0.f : 1.f;
        const float ac = b ? 0.f : glf;
        dl[k][q] = fmaf(gf * vn, mask, rr[q]) - v[k][q];
        mb = fmaf(ac, mb, dl[k][q]);
        reset |= b != 0u;
        vnext = v[k][q];
      }
      lc[k] = Aff{reset ? 0.0 : gl8, (double)mb};
      if (k == 0) reset0 = reset;
    }
    // ---- the halo: 4 slots per lane, only its composed map is needed.  Its env
    // tails belong to the tile above, which may already have overwritten their
    // parked bootstraps in ar: read boot[env] instead, the r-th tail of the
    // halo being env eh + r (or env_of when an env without fresh slots intervenes)
    Aff hc;
    {
      const int j0 = kGTile + 4 * lane;
      const float4 r0 = *reinterpret_cast<const float4*>(sr + j0);
      const float4 v0 = *reinterpret_cast<const float4*>(sv + j0);
      const uint32_t d4 = *reinterpret_cast<const uint32_t*>(sd + j0);
      const float rr[4] = {r0.x, r0.y, r0.z, r0.w}, vv[4] = {v0.x, v0.y, v0.z, v0.w};
      uint32_t tm = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if ((d4 >> (8 * q)) & 2u) tm |= 1u << q;
      int rk = __popc(tm);
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, rk, o);
        if (lane >= o) rk += y;
      }
      rk -= __popc(tm);
      float hb[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        hb[q] = 0.f;
        const int i = lo + j0 + q;
        if (((d4 >> (8 * q)) & 3u) == 2u && i < F) {
          int e = eh + rk + __popc(tm & ((1u << q) - 1u));
          const int o1 = __ldg(off + e + 1);
          float b = __ldg(boot + e);
          if (o1 != i + 1) b = __ldg(boot + __ldg(env_of + i));
          hb[q] = b;
        }
      }
      float vnext = sv[j0 + 4];
      float mb = 0.f;
      bool reset = false;
#pragma unroll
      for (int q = 3; q >= 0; --q) {
        const uint32_t b = (d4 >> (8 * q)) & 3u;
        const float vn = b == 2u ? hb[q] : vnext;
        const float mask = (b & 1u) ? 0.f : 1.f;
        mb = fmaf(b ? 0.f : glf, mb, fmaf(gf * vn, mask, rr[q]) - vv[q]);
        reset |= b != 0u;
        vnext = vv[q];
      }
      hc = Aff{reset ? 0.0 : gl4, (double)mb};
    }
    __syncwarp();
    if (lane == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    // the stage is consumed: refill it with the tile after next
    {
      int e2 = 0;
      const int t2 = claim(s, e2);
#pragma unroll
      for (int q = 0; q < kGStages; ++q)
        if (s == q) tq[q] = t2, eq[q] = e2;
    }
    // ---- suffix scans over the lanes, the rows and the carry (fp64)
    const Aff in0 = warp_suffix(lc[0], lane), in1 = warp_suffix(lc[1], lane);
    const Aff hagg = shfl_aff(warp_suffix(hc, lane), 0);
    double carry = hagg.b;  // A_hi when the halo holds a reset (a == 0)
    if (hagg.a != 0.0) {  // no reset in the halo: the tile above published A_hi
      if (lane == 0) {
        while (flag_acquire(&tiles[tid - 1].flag) == 0) {
        }
        carry = tiles[tid - 1].inc;
      }
      carry = __shfl_sync(0xffffffffu, carry, 0);
    }
    const Aff row1 = shfl_aff(in1, 0), row0 = shfl_aff(in0, 0);
    const double c1 = carry;                      // A at the top of row 1
    const double c0 = fma(row1.a, c1, row1.b);    // A at the top of row 0
    // ---- final values: the lane's top value, then its 8 items (fp32)
#pragma unroll
    for (int k = 1; k >= 0; --k) {
      Aff ex = shfl_down_aff(k ? in1 : in0, 1);
      if (lane == 31) ex = Aff{1.0, 0.0};
      float x = (float)fma(ex.a, k ? c1 : c0, ex.b);
      float av[kGItems], rv[kGItems];
#pragma unroll
      for (int q = kGItems - 1; q >= 0; --q) {
        const uint32_t b = (dd[k][q >> 2] >> (8 * (q & 3))) & 3u;
        x = fmaf(b ? 0.f : glf, x, dl[k][q]);
        av[q] = x;
        rv[q] = x + v[k][q];
      }
      const int i0 = lo + kGRow * k + kGItems * lane;
      if (i0 + kGItems <= hi) {  // (A, R) pairs: 64 contiguous bytes per lane
        float4* o4 = reinterpret_cast<float4*>(ar + 2 * (size_t)i0);
#pragma unroll
        for (int q = 0; q < kGItems; q += 2) __stcs(o4 + q / 2, make_float4(av[q], rv[q], av[q + 1], rv[q + 1]));
      } else {
#pragma unroll
        for (int q = 0; q < kGItems; ++q)
          if (i0 + q < hi) reinterpret_cast<float2*>(ar)[i0 + q] = make_float2(av[q], rv[q]);
      }
    }
    // the tile below reads A_lo from here iff this tile's bottom 128 slots (its
    // halo) have no reset: lanes 0..15 of row 0
    if (tid + 1 < ntiles) {
      if (!__any_sync(0xffffffffu, lane < 16 && reset0) && lane == 0) {
        tiles[tid].inc = fma(row0.a, c0, row0.b);
        flag_release(&tiles[tid].flag, 2);
      }
    }
  }
}

// ----------------------------------------------------- general (any order)
__global__ void gae_keys_kernel(const int32_t* __restrict__ env, const uint8_t* __restrict__ replayed,
                                int S, int N, uint64_t* __restrict__ keys, int32_t* __restrict__ counts) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= S) return;
  const int e = env[i];
  const bool fresh = !replayed[i] && e >= 0 && e < N;
  keys[i] = ((uint64_t)(fresh ? e : N) << 32) | (uint32_t)i;
  if (fresh) atomicAdd(&counts[e], 1);
}
__global__ void gae_gather_kernel(const uint64_t* __restrict__ keys, int F, const float* __restrict__ r,
                                  const float* __restrict__ v, const uint8_t* __restrict__ d,
                                  float* __restrict__ r2, float* __restrict__ v2, uint8_t* __restrict__ d2,
                                  int32_t* __restrict__ e2) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= F) return;
  const int i = (int)(keys[j] & 0xffffffffu);
  const int e = (int)(keys[j] >> 32);
  const bool tail = j + 1 == F || (int)(keys[j + 1] >> 32) != e;
  r2[j] = r[i];
  v2[j] = v[i];
  d2[j] = (d[i] & 1) | (tail ? 2 : 0);
  e2[j] = e;
}
__global__ void gae_scatter_kernel(const uint64_t* __restrict__ keys, int F, const float2* __restrict__ ar2,
                                   float2* __restrict__ ar) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= F) return;
  const int i = (int)(keys[j] & 0xffffffffu);
  ar[i] = ar2[j];
}

static void run_scan(Ctx* c, const float* r, const float* v, const uint8_t* d, const int32_t* env, int F,
                     const float* boot, const uint8_t* valid, const int32_t* off, int N, double gamma,
                     double lambda, float* ar) {
  if (F <= 0) return;
  const int ntiles = (F + kGTile - 1) / kGTile;
  DBuf<GaeTileState> tiles;
  DBuf<int> misc;  // [0] tile counter, [1] lowest env with a missing bootstrap
  tiles.reserve(c, ntiles);
  misc.reserve(c, 2);
  tiles.zero(ntiles);
  VER_CUDA(cudaMemsetAsync(misc.p, 0, sizeof(int), c->stream));
  VER_CUDA(cudaMemsetAsync(misc.p + 1, 0x7f, sizeof(int), c->stream));  // 0x7f7f7f7f: none
  gae_boot_kernel<<<cdiv(N, 256), 256, 0, c->stream>>>(off, d, boot, valid, N, ar, misc.p + 1);
  after_launch(c);
  static std::atomic<int> per_sm_cache[kMaxDevices];  // per device (0 = not probed yet)
  int per_sm = per_sm_cache[dev_slot(c)].load();
  if (!per_sm) {
    VER_CUDA(cudaFuncSetAttribute(gae_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kGSmem));
    VER_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gae_scan_kernel, 32 * kGWarps, kGSmem));
    per_sm = std::max(1, per_sm);
    per_sm_cache[dev_slot(c)].store(per_sm);
  }
  // warps claim tiles dynamically: CTAs that are not resident yet simply start later
  const int grid = std::min((ntiles + kGWarps - 1) / kGWarps, per_sm * c->num_sms);
  {
    ScopedEv ev(c, c->hbm_tag);
    gae_scan_kernel<<<grid, 32 * kGWarps, kGSmem, c->stream>>>(r, v, d, env, off, boot, F, gamma, lambda, ar,
                                                               tiles.p, misc.p);
    after_launch(c);
  }
  int* h = static_cast<int*>(c->pinned_buf(2 * sizeof(int)));
  misc.download(h, 2);
  sync(c);
  if (h[1] != 0x7f7f7f7f)
    protocol_error("compute_gae: missing bootstrap value for env " + std::to_string(h[1]));
}

void compute_gae(DView& V, double gamma, double lambda) {
  Ctx* c = V.ctx;
  if (V.size == 0) return;
  if (V.env_contiguous) {
    run_scan(c, V.reward.p, V.value.p, V.done.p, V.env_index.p, V.fresh_prefix, V.env_bootstrap.p,
             V.env_bootstrap_valid.p, V.env_offsets.p, V.N, gamma, lambda, V.ar.p);
    return;
  }
  const int S = V.size, N = V.N;
  DBuf<uint64_t> keys;
  DBuf<int32_t> off;
  keys.reserve(c, S);
  off.reserve(c, N + 1);
  off.zero(N + 1);
  gae_keys_kernel<<<cdiv(S, 256), 256, 0, c->stream>>>(V.env_index.p, V.replayed.p, S, N, keys.p, off.p);
  after_launch(c);
  sort_u64(c, keys.p, S);
  exclusive_scan_i32(c, off.p, off.p, N, off.p + N);
  int32_t* hF = static_cast<int32_t*>(c->pinned_buf(4));
  VER_CUDA(cudaMemcpyAsync(hF, off.p + N, 4, cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  const int F = *hF;
  if (F == 0) return;
  DBuf<float> r2, v2, ar2;
  DBuf<uint8_t> d2;
  DBuf<int32_t> e2;
  e2.reserve(c, F);
  r2.reserve(c, F);
  v2.reserve(c, F);
  ar2.reserve(c, 2 * (size_t)F);
  d2.reserve(c, F);
  gae_gather_kernel<<<cdiv(F, 256), 256, 0, c->stream>>>(keys.p, F, V.reward.p, V.value.p, V.done.p, r2.p,
                                                         v2.p, d2.p, e2.p);
  after_launch(c);
  run_scan(c, r2.p, v2.p, d2.p, e2.p, F, V.env_bootstrap.p, V.env_bootstrap_valid.p, off.p, N, gamma, lambda, ar2.p);
  gae_scatter_kernel<<<cdiv(F, 256), 256, 0, c->stream>>>(keys.p, F, reinterpret_cast<const float2*>(ar2.p),
                                                          reinterpret_cast<float2*>(V.ar.p));
  after_launch(c);
}

}  // namespace verg

using namespace verg;

extern "C" ver_status ver_compute_gae(ver_view v, double gamma, double lambda) {
  VER_API_BEGIN
  activate(v->v.ctx);
  compute_gae(v->v, gamma, lambda);
  VER_API_END
}
