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
// One pass, decoupled look-back: each CTA claims tiles from the END of the
// array (dynamic tile id), composes its 2048 maps, publishes the aggregate,
// looks back only until it meets a tile whose map has a = 0 (any done/env
// tail inside) or an inclusive value.  HBM traffic: r, V (4+4 B), done (1 B)
// read once, A, R (4+4 B) written once = 17 B/step, plus offsets per env.
//
// Views whose fresh slots are not env-major contiguous (arbitrary uploads,
// e.g. make_view fixtures with env = seq % N) first stable-sort the fresh
// slots by (env, slot) on the device, run the same scan on the gathered
// arrays and scatter back.
#include <algorithm>
#include <cstdlib>

#include "view.cuh"

namespace verg {

constexpr int kGaeThreads = 256;                     // compute threads (8 warps)
constexpr int kGaeItems = 8;
constexpr int kGaeTile = kGaeThreads * kGaeItems;  // 2048 slots per tile
constexpr int kGaeWarps = kGaeThreads / 32;
constexpr int kGaeBlock = kGaeThreads + 64;          // + producer warp + look-back / fix-up warp
constexpr int kGaeStages = 3;                        // tiles in flight per CTA
constexpr int kGaeWin = 128;                         // env window staged per tile
// stage layout (bytes): V [tile + 4] | r [tile] | done [tile] | boot [win] | valid [win] | off [win + 4]
constexpr int kGaeOffR = 4 * kGaeTile + 16;
constexpr int kGaeOffD = kGaeOffR + 4 * kGaeTile;
constexpr int kGaeOffB = kGaeOffD + kGaeTile;
constexpr int kGaeOffBV = kGaeOffB + 4 * kGaeWin;
constexpr int kGaeOffO = kGaeOffBV + kGaeWin;
constexpr int kGaeStageBytes = kGaeOffO + 4 * (kGaeWin + 4);

struct Affine {
  double a, b;  // x -> b + a x
};
// x earlier (lower index), y later: A_x = b_x + a_x (b_y + a_y X)
__device__ __forceinline__ Affine compose(Affine x, Affine y) {
  return Affine{x.a * y.a, fma(x.a, y.b, x.b)};
}

struct GaeTileState {
  double a, b, inc;
  int flag;  // 0 none, 1 aggregate (a,b), 2 inclusive (inc = A at tile start)
  int pad;
};

struct GaeStageHdr {
  int tid;         // claimed tile id (-1: no more tiles)
  int e0;          // env of the tile's first slot = env of its first tail
  int wbase;       // first env of the staged window (16-aligned)
  int nb, nv, no;  // boot / valid / off entries staged from wbase
  int seg;         // first slot of the carry-dependent top segment (compute warps: atomicMin)
  int pad;
  double sa, sb;   // tile aggregate
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
__device__ __forceinline__ void gae_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
// tile-state flag protocol: payload stores, then a release store of the flag;
// readers acquire-load the flag before reading the payload
__device__ __forceinline__ void flag_release(volatile int* f, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
}
__device__ __forceinline__ int flag_acquire(volatile int* f) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
  return v;
}
__device__ __forceinline__ void gae_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kGaeThreads) : "memory"); }

// Persistent CTAs, decoupled look-back, warp-specialised, 3-deep ring.
//  * Producer warp: claims tiles (dynamic ids from the END of the array:
//    carries flow downwards), reads env_of at the tile's first slot and
//    bulk-copies r, V (+ the next tile's first 4 V), done and a window of the
//    envs' bootstrap values / flags / offsets into the ring.
//  * 8 compute warps (thread t: 8 consecutive slots): env tails (done bit 1)
//    are numbered by a block-wide count (tail -> env from the staged offsets,
//    no dependent DRAM loads); per-item affine maps, block suffix scan, the
//    tile aggregate is published at once (flag 1), and every slot whose value
//    does not depend on the carry (all slots below the tile's last reset) is
//    stored.  The carry-dependent top segment's partial values (carry = 0) go
//    to shared memory.  The compute warps never wait for a look-back, so an
//    aggregate is never held back behind another tile's look-back.
//  * Fix-up warp: looks back (terminates at the first predecessor with a
//    reset, or an inclusive value), publishes this tile's inclusive value and
//    patches the top segment: A_i = A_i(0) + (gamma lambda)^(hi - i) carry.
// A CTA processes its tiles in claim order and all CTAs are resident, so every
// aggregate a look-back waits on is published without further waiting.
// Per-thread recursions are fp32 over <= 8 items; compositions and carries
// are fp64.  The single partial tile at the end is read from global memory.
__global__ void __launch_bounds__(kGaeBlock) gae_scan_kernel(
    const float* __restrict__ reward, const float* __restrict__ value, const uint8_t* __restrict__ done,
    const int32_t* __restrict__ env_of, int F, const float* __restrict__ boot,
    const uint8_t* __restrict__ boot_valid, const int32_t* __restrict__ off, int N, double gamma, double lambda,
    float* __restrict__ adv, float* __restrict__ ret, volatile GaeTileState* tiles, int* tile_counter,
    int* err_env) {
  extern __shared__ __align__(128) uint8_t gsmem[];
  __shared__ uint64_t s_full[kGaeStages], s_ready[kGaeStages], s_empty[kGaeStages];
  __shared__ GaeStageHdr s_hdr[kGaeStages];
  __shared__ Affine s_warp[kGaeWarps];
  __shared__ int s_cnt[kGaeWarps];
  const int ntiles = (F + kGaeTile - 1) / kGaeTile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float glf = (float)(gamma * lambda);
  auto stage = [&](int s) { return gsmem + s * kGaeStageBytes; };
  if (threadIdx.x == 0) {
    for (int s = 0; s < kGaeStages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(gsm(&s_full[s])) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(gsm(&s_ready[s])), "r"(kGaeWarps) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(gsm(&s_empty[s])) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kGaeWarps) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      for (int k = 0;; ++k) {
        const int s = k % kGaeStages;
        gae_wait(gsm(&s_empty[s]), ((k / kGaeStages) & 1) ^ 1);
        const uint32_t mb = gsm(&s_full[s]);
        const int tid = atomicAdd(tile_counter, 1);
        GaeStageHdr h{};
        h.tid = -1;
        if (tid >= ntiles) {
          s_hdr[s] = h;
          gae_arrive(mb);
          break;
        }
        const int lo = (ntiles - 1 - tid) * kGaeTile;
        h.tid = tid;
        h.e0 = env_of[lo];
        h.seg = 0x7fffffff;
        if (lo + kGaeTile > F) {  // partial tile: the compute threads read global memory
          s_hdr[s] = h;
          gae_arrive(mb);
          continue;
        }
        h.wbase = h.e0 & ~15;
        h.nb = max(0, min(kGaeWin, N - h.wbase)) & ~3;
        h.nv = max(0, min(kGaeWin, N - h.wbase)) & ~15;
        h.no = max(0, min(kGaeWin + 4, N + 1 - h.wbase)) & ~3;
        s_hdr[s] = h;
        const uint32_t vb = 4 * kGaeTile + (lo + kGaeTile + 4 <= F ? 16 : 0);  // + V of the slots above
        const uint32_t bytes = vb + 5 * kGaeTile + 4 * h.nb + h.nv + 4 * h.no;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
        uint8_t* st = stage(s);
        gae_bulk(gsm(st), value + lo, vb, mb);
        gae_bulk(gsm(st + kGaeOffR), reward + lo, 4 * kGaeTile, mb);
        gae_bulk(gsm(st + kGaeOffD), done + lo, kGaeTile, mb);
        if (h.nb) gae_bulk(gsm(st + kGaeOffB), boot + h.wbase, 4 * h.nb, mb);
        if (h.nv) gae_bulk(gsm(st + kGaeOffBV), boot_valid + h.wbase, h.nv, mb);
        if (h.no) gae_bulk(gsm(st + kGaeOffO), off + h.wbase, 4 * h.no, mb);
      }
    }
    return;
  }

  if (warp == kGaeWarps + 1) {
    // ------------------------------------------------- look-back + fix-up
    for (int it = 0;; ++it) {
      const int s = it % kGaeStages;
      gae_wait(gsm(&s_full[s]), (it / kGaeStages) & 1);
      if (s_hdr[s].tid < 0) break;
      gae_wait(gsm(&s_ready[s]), (it / kGaeStages) & 1);
      const GaeStageHdr hd = s_hdr[s];
      const int tid = hd.tid;
      const int lo = (ntiles - 1 - tid) * kGaeTile, hi = min(F, lo + kGaeTile);
      double carry = 0.0;  // A at hi
      if (lane == 0 && tid != 0) {
        Affine acc{1.0, 0.0};
        int p = tid - 1;
        for (;;) {
          int f;
          do {
            f = flag_acquire(&tiles[p].flag);
          } while (f == 0);
          if (f == 2) {
            carry = fma(acc.a, tiles[p].inc, acc.b);
            break;
          }
          acc = compose(acc, Affine{tiles[p].a, tiles[p].b});
          if (acc.a == 0.0 || p == 0) {
            carry = acc.b;
            break;
          }
          --p;
        }
        tiles[tid].inc = fma(hd.sa, carry, hd.sb);
        flag_release(&tiles[tid].flag, 2);
      }
      carry = __shfl_sync(0xffffffffu, carry, 0);
      // top segment [seg, hi): partial values (carry 0) staged by the compute warps
      const float* pa = reinterpret_cast<const float*>(stage(s) + kGaeOffR);
      const float* pr = reinterpret_cast<const float*>(stage(s));
      const int seg = max(lo, min(hd.seg, hi));
      const double lg2 = log2((double)glf);
      for (int i = seg + lane; i < hi; i += 32) {
        // (gamma lambda)^(hi - i): the top segment has no reset, every a_i = gamma lambda
        const double cf = exp2(lg2 * (double)(hi - i)) * carry;
        const float av = (float)((double)pa[i - lo] + cf);
        adv[i] = av;
        ret[i] = (float)((double)pr[i - lo] + cf);
      }
      __syncwarp();
      if (lane == 0) gae_arrive(gsm(&s_empty[s]));
    }
    return;
  }

  // -------------------------------------------------------------- compute
  const float gf = (float)gamma;
  for (int it = 0;; ++it) {
    const int s = it % kGaeStages;
    gae_wait(gsm(&s_full[s]), (it / kGaeStages) & 1);
    const GaeStageHdr hd = s_hdr[s];
    if (hd.tid < 0) break;
    const int tid = hd.tid;
    const int tile = ntiles - 1 - tid;
    const int lo = tile * kGaeTile;
    const int hi = min(F, lo + kGaeTile);
    const int l0 = threadIdx.x * kGaeItems;  // tile-local first item
    const int i0 = lo + l0;
    uint8_t* st = stage(s);
    float* sv = reinterpret_cast<float*>(st);
    float* sr = reinterpret_cast<float*>(st + kGaeOffR);
    float r[kGaeItems], v[kGaeItems + 1];
    uint32_t dw[2];
    const bool full = hi - lo == kGaeTile;
    if (full) {
      const float4* r4 = reinterpret_cast<const float4*>(sr + l0);
      const float4* v4 = reinterpret_cast<const float4*>(sv + l0);
      const float4 x0 = r4[0], x1 = r4[1], y0 = v4[0], y1 = v4[1];
      const uint2 dd = *reinterpret_cast<const uint2*>(st + kGaeOffD + l0);
      r[0] = x0.x; r[1] = x0.y; r[2] = x0.z; r[3] = x0.w;
      r[4] = x1.x; r[5] = x1.y; r[6] = x1.z; r[7] = x1.w;
      v[0] = y0.x; v[1] = y0.y; v[2] = y0.z; v[3] = y0.w;
      v[4] = y1.x; v[5] = y1.y; v[6] = y1.z; v[7] = y1.w;
      dw[0] = dd.x;
      dw[1] = dd.y;
      v[kGaeItems] = (l0 + kGaeItems < kGaeTile || hi + 4 <= F) ? sv[l0 + kGaeItems] : (hi < F ? value[hi] : 0.f);
    } else {
      dw[0] = dw[1] = 0x03030303u;  // beyond the end: tail + done (inert)
#pragma unroll
      for (int q = 0; q < kGaeItems; ++q) {
        const int i = i0 + q;
        r[q] = i < hi ? reward[i] : 0.f;
        v[q] = i < hi ? value[i] : 0.f;
        if (i < hi) {
          const uint32_t sh = 8 * (q & 3);
          dw[q >> 2] = (dw[q >> 2] & ~(0xffu << sh)) | ((uint32_t)done[i] << sh);
        }
      }
      v[kGaeItems] = (i0 + kGaeItems < F) ? value[i0 + kGaeItems] : 0.f;
    }
    // env tails (done bit 1) in slot order: rank -> env
    uint32_t tmask = 0;
#pragma unroll
    for (int q = 0; q < kGaeItems; ++q)
      if (i0 + q < hi && ((dw[q >> 2] >> (8 * (q & 3))) & 2u)) tmask |= 1u << q;
    int incl_cnt = __popc(tmask);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl_cnt, o);
      if (lane >= o) incl_cnt += y;
    }
    if (lane == 31) s_cnt[warp] = incl_cnt;
    gae_sync();
    int rank = incl_cnt - __popc(tmask);
    for (int w = 0; w < warp; ++w) rank += s_cnt[w];
    // per-item maps A_i = delta_i + a_i A_{i+1} (fp32); bootstrap at env tails
    float dl[kGaeItems], ac[kGaeItems];
#pragma unroll
    for (int q = 0; q < kGaeItems; ++q) {
      const uint32_t b = (dw[q >> 2] >> (8 * (q & 3))) & 0xffu;
      const bool dn = b & 1, tail = b & 2;
      float vnext = v[q + 1];
      if (tail) {
        vnext = 0.f;
        if (!dn && i0 + q < hi) {
          // the rank-th non-empty env from e0; env e's tail slot is off[e+1]-1
          // (empty envs, off[e+1] == off[e], are skipped)
          int e = hd.e0 + rank;
          const int32_t* so = reinterpret_cast<const int32_t*>(st + kGaeOffO);
          for (;;) {
            const int j1 = e + 1 - hd.wbase;
            const int o1 = (full && j1 >= 0 && j1 < hd.no) ? so[j1] : off[e + 1];
            if (o1 - 1 >= i0 + q) break;
            ++e;
          }
          const int j = e - hd.wbase;
          float bv;
          bool ok;
          if (full && j >= 0 && j < hd.nb && j < hd.nv) {
            bv = reinterpret_cast<const float*>(st + kGaeOffB)[j];
            ok = st[kGaeOffBV + j] != 0;
          } else {
            bv = boot[e];
            ok = boot_valid[e] != 0;
          }
          if (!ok) atomicMin(err_env, e);
          vnext = bv;
        }
      }
      if (tail) ++rank;
      const float mask = dn ? 0.f : 1.f;
      dl[q] = fmaf(gf * vnext, mask, r[q]) - v[q];
      ac[q] = tail ? 0.f : glf * mask;
    }
    float ma = 1.f, mb = 0.f;  // thread composite, fp32 over <= 8 steps
#pragma unroll
    for (int q = kGaeItems - 1; q >= 0; --q) {
      mb = fmaf(ac[q], mb, dl[q]);
      ma = ac[q] * ma;
    }
    // block-level suffix scan of thread maps (fp64)
    Affine incl{(double)ma, (double)mb};
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      Affine y{__shfl_down_sync(0xffffffffu, incl.a, o), __shfl_down_sync(0xffffffffu, incl.b, o)};
      if (lane + o < 32) incl = compose(incl, y);
    }
    if (lane == 0) s_warp[warp] = incl;
    gae_sync();
    if (threadIdx.x == 0) {
      Affine suf{1.0, 0.0};
      for (int w = kGaeWarps - 1; w >= 0; --w) {
        const Affine cur = s_warp[w];
        s_warp[w] = suf;
        suf = compose(cur, suf);
      }
      s_hdr[s].sa = suf.a;
      s_hdr[s].sb = suf.b;
    }
    Affine lane_ex{__shfl_down_sync(0xffffffffu, incl.a, 1), __shfl_down_sync(0xffffffffu, incl.b, 1)};
    if (lane == 31) lane_ex = Affine{1.0, 0.0};
    gae_sync();
    if (threadIdx.x == 0) {
      // publish the tile aggregate (the top tile's is already its inclusive
      // value); after the barrier, so the fence holds up warp 0 only
      const double sa = s_hdr[s].sa, sb = s_hdr[s].sb;
      if (tid == 0) {
        tiles[tid].inc = sb;
        flag_release(&tiles[tid].flag, 2);
      } else {
        tiles[tid].a = sa;
        tiles[tid].b = sb;
        flag_release(&tiles[tid].flag, 1);
      }
    }
    const Affine after = compose(lane_ex, s_warp[warp]);  // A at hi -> A after this thread's items
    // values with carry 0; c: does the item still depend on the carry
    float xf = (float)after.b;
    double cf = after.a;
    float av[kGaeItems], rv[kGaeItems];
    uint32_t dep = 0;
#pragma unroll
    for (int q = kGaeItems - 1; q >= 0; --q) {
      xf = fmaf(ac[q], xf, dl[q]);
      cf *= (double)ac[q];
      av[q] = xf;
      rv[q] = xf + v[q];
      if (cf != 0.0) dep |= 1u << q;
    }
    if (dep) {
      // carry-dependent slots (the tile's top segment) -> staged for the fix-up warp
      atomicMin(&s_hdr[s].seg, i0 + (__ffs(dep) - 1));
#pragma unroll
      for (int q = 0; q < kGaeItems; ++q)
        if ((dep >> q) & 1) {
          sr[l0 + q] = av[q];
          sv[l0 + q] = rv[q];
        }
    }
    if (dep == 0 && i0 + kGaeItems <= hi) {
      float4* a4 = reinterpret_cast<float4*>(adv + i0);
      float4* q4 = reinterpret_cast<float4*>(ret + i0);
      __stcs(a4, make_float4(av[0], av[1], av[2], av[3]));
      __stcs(a4 + 1, make_float4(av[4], av[5], av[6], av[7]));
      __stcs(q4, make_float4(rv[0], rv[1], rv[2], rv[3]));
      __stcs(q4 + 1, make_float4(rv[4], rv[5], rv[6], rv[7]));
    } else {
      for (int q = 0; q < kGaeItems; ++q)
        if (i0 + q < hi && !((dep >> q) & 1)) {
          adv[i0 + q] = av[q];
          ret[i0 + q] = rv[q];
        }
    }
    __syncwarp();
    if (lane == 0) gae_arrive(gsm(&s_ready[s]));
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
__global__ void gae_scatter_kernel(const uint64_t* __restrict__ keys, int F, const float* __restrict__ a2,
                                   const float* __restrict__ ret2, float* __restrict__ adv,
                                   float* __restrict__ ret) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= F) return;
  const int i = (int)(keys[j] & 0xffffffffu);
  adv[i] = a2[j];
  ret[i] = ret2[j];
}

static void run_scan(Ctx* c, const float* r, const float* v, const uint8_t* d, const int32_t* env, int F,
                     const float* boot, const uint8_t* valid, const int32_t* off, int N, double gamma,
                     double lambda, float* adv, float* ret) {
  if (F <= 0) return;
  const int ntiles = (F + kGaeTile - 1) / kGaeTile;
  DBuf<GaeTileState> tiles;
  DBuf<int> misc;  // [0] tile counter, [1] lowest env with a missing bootstrap
  tiles.reserve(c, ntiles);
  misc.reserve(c, 2);
  tiles.zero(ntiles);
  VER_CUDA(cudaMemsetAsync(misc.p, 0, sizeof(int), c->stream));
  VER_CUDA(cudaMemsetAsync(misc.p + 1, 0x7f, sizeof(int), c->stream));  // 0x7f7f7f7f: none
  const int smem = kGaeStages * kGaeStageBytes;
  static std::atomic<int> per_sm_cache[kMaxDevices];  // per device (0 = not probed yet)
  int per_sm = per_sm_cache[dev_slot(c)].load();
  if (!per_sm) {
    VER_CUDA(cudaFuncSetAttribute(gae_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    VER_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gae_scan_kernel, kGaeBlock, smem));
    per_sm = std::max(1, per_sm);
    per_sm_cache[dev_slot(c)].store(per_sm);
  }
  const int grid = std::min(ntiles, per_sm * c->num_sms);
  gae_scan_kernel<<<grid, kGaeBlock, smem, c->stream>>>(r, v, d, env, F, boot, valid, off, N, gamma, lambda, adv, ret,
                                                       tiles.p, misc.p, misc.p + 1);
  after_launch(c);
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
             V.env_bootstrap_valid.p, V.env_offsets.p, V.N, gamma, lambda, V.advantage.p, V.returns.p);
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
  DBuf<float> r2, v2, a2, ret2;
  DBuf<uint8_t> d2;
  DBuf<int32_t> e2;
  e2.reserve(c, F);
  r2.reserve(c, F);
  v2.reserve(c, F);
  a2.reserve(c, F);
  ret2.reserve(c, F);
  d2.reserve(c, F);
  gae_gather_kernel<<<cdiv(F, 256), 256, 0, c->stream>>>(keys.p, F, V.reward.p, V.value.p, V.done.p, r2.p,
                                                         v2.p, d2.p, e2.p);
  after_launch(c);
  run_scan(c, r2.p, v2.p, d2.p, e2.p, F, V.env_bootstrap.p, V.env_bootstrap_valid.p, off.p, N, gamma, lambda,
           a2.p, ret2.p);
  gae_scatter_kernel<<<cdiv(F, 256), 256, 0, c->stream>>>(keys.p, F, a2.p, ret2.p, V.advantage.p,
                                                          V.returns.p);
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
