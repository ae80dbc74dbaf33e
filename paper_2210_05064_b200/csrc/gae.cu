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
#include <cstdlib>

#include "view.cuh"

namespace verg {

constexpr int kGaeThreads = 256;
constexpr int kGaeItems = 8;
constexpr int kGaeTile = kGaeThreads * kGaeItems;  // 2048 slots per tile
constexpr int kGaeStages = 4;                       // TMA prefetch depth (tiles)

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

// one tile's inputs staged by TMA: r[lo, hi), V[lo, hi + 4) (V[hi] = next tile's
// first value), done bits[lo, hi)
struct alignas(128) GaeStage {
  float r[kGaeTile];
  float v[kGaeTile + 4];
  uint8_t d[kGaeTile];
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}

// Persistent decoupled-look-back reverse scan.  Each CTA keeps kGaeStages
// tiles in flight: thread 0 claims tiles (dynamic tickets, last tile first)
// and TMA-bulk-copies their r / V / done into a shared-memory ring, so HBM
// reads for the next tiles overlap this tile's scan, look-back and stores.
// done bit 1 marks an env's last fresh slot (set by close_rollout / upload /
// the device generators), so no per-env offsets are read at all; only env
// tails without `done` look up their env's bootstrap.
__global__ void __launch_bounds__(kGaeThreads) gae_scan_kernel(
    const float* __restrict__ reward, const float* __restrict__ value, const uint8_t* __restrict__ done,
    const int32_t* __restrict__ env_of, int F, const float* __restrict__ boot,
    const uint8_t* __restrict__ boot_valid, double gamma, double lambda, float* __restrict__ adv,
    float* __restrict__ ret, volatile GaeTileState* tiles, int* tile_counter, int* err_env, int dbg) {
  extern __shared__ __align__(128) uint8_t gsm[];
  GaeStage* st = reinterpret_cast<GaeStage*>(gsm);
  __shared__ __align__(8) uint64_t s_bar[kGaeStages];
  __shared__ int s_ticket[kGaeStages];
  __shared__ int s_direct[kGaeStages];
  __shared__ Affine s_warp[kGaeThreads / 32];
  __shared__ double s_carry;
  const int ntiles = (F + kGaeTile - 1) / kGaeTile;
  const double gl = gamma * lambda;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  auto issue = [&](int s, int t) {  // thread 0 only
    s_ticket[s] = t;
    if (t >= ntiles) return;
    const int lo = (ntiles - 1 - t) * kGaeTile;
    if (lo + kGaeTile + 4 <= F) {
      s_direct[s] = 0;
      constexpr uint32_t kBytes = kGaeTile * 4 + (kGaeTile + 4) * 4 + kGaeTile;  // r + V (+4) + done
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&s_bar[s])),
                   "r"(kBytes)
                   : "memory");
      bulk_g2s(st[s].r, reward + lo, kGaeTile * 4, &s_bar[s]);
      bulk_g2s(st[s].v, value + lo, (kGaeTile + 4) * 4, &s_bar[s]);
      bulk_g2s(st[s].d, done + lo, kGaeTile, &s_bar[s]);
    } else {  // the array's tail tile: read straight from global, complete the phase
      s_direct[s] = 1;
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&s_bar[s])) : "memory");
    }
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kGaeStages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&s_bar[s])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < kGaeStages; ++s) issue(s, atomicAdd(tile_counter, 1));
  }
  __syncthreads();

  for (int k = 0;; ++k) {
    const int s = k % kGaeStages;
    const int tid = s_ticket[s];
    if (tid >= ntiles) break;
    const int tile = ntiles - 1 - tid;
    const int lo = tile * kGaeTile;
    const int hi = min(F, lo + kGaeTile);
    const uint32_t ph = (k / kGaeStages) & 1;
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_addr(&s_bar[s])),
        "r"(ph)
        : "memory");
    const bool direct = s_direct[s];
    const int j0 = threadIdx.x * kGaeItems;  // tile-relative
    const int i0 = lo + j0;
    float r[kGaeItems], v[kGaeItems + 1];
    uint8_t d[kGaeItems];
    if (!direct) {
      const float4* r4 = reinterpret_cast<const float4*>(st[s].r + j0);
      const float4* v4 = reinterpret_cast<const float4*>(st[s].v + j0);
      const float4 x0 = r4[0], x1 = r4[1], y0 = v4[0], y1 = v4[1];
      r[0] = x0.x; r[1] = x0.y; r[2] = x0.z; r[3] = x0.w;
      r[4] = x1.x; r[5] = x1.y; r[6] = x1.z; r[7] = x1.w;
      v[0] = y0.x; v[1] = y0.y; v[2] = y0.z; v[3] = y0.w;
      v[4] = y1.x; v[5] = y1.y; v[6] = y1.z; v[7] = y1.w;
      v[8] = st[s].v[j0 + 8];
      const uint2 dd = *reinterpret_cast<const uint2*>(st[s].d + j0);
      const uint8_t* db = reinterpret_cast<const uint8_t*>(&dd);
#pragma unroll
      for (int q = 0; q < kGaeItems; ++q) d[q] = db[q];
    } else {
#pragma unroll
      for (int q = 0; q < kGaeItems; ++q) {
        const int i = i0 + q;
        r[q] = i < hi ? reward[i] : 0.f;
        v[q] = i < hi ? value[i] : 0.f;
        d[q] = i < hi ? done[i] : 3;
      }
      v[kGaeItems] = (i0 + kGaeItems < F) ? value[i0 + kGaeItems] : 0.f;
    }
    // per-item maps x -> delta + a x (tail: a = 0; V_next = bootstrap unless done)
    auto item = [&](int q, double& delta, double& acoef) {
      const int i = i0 + q;
      if (i >= hi) {
        delta = 0.0;
        acoef = 1.0;
        return;
      }
      const bool dn = d[q] & 1, tail = d[q] & 2;
      double vnext = 0.0;
      if (tail) {
        if (!dn) {
          const int e = env_of[i];
          if (!boot_valid[e]) atomicMin(err_env, e);
          vnext = (double)boot[e];
        }
      } else {
        vnext = (double)v[q + 1];
      }
      const double mask = dn ? 0.0 : 1.0;
      delta = (double)r[q] + gamma * vnext * mask - (double)v[q];
      acoef = tail ? 0.0 : gl * mask;
    };
    Affine mine{1.0, 0.0};
#pragma unroll
    for (int q = kGaeItems - 1; q >= 0; --q) {
      double dl, ac;
      item(q, dl, ac);
      mine = compose(Affine{ac, dl}, mine);
    }
    // block-level suffix scan of thread maps
    Affine incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      Affine y{__shfl_down_sync(0xffffffffu, incl.a, o), __shfl_down_sync(0xffffffffu, incl.b, o)};
      if (lane + o < 32) incl = compose(incl, y);
    }
    if (lane == 0) s_warp[warp] = incl;
    __syncthreads();  // also: every thread has read stage s
    if (threadIdx.x == 0) {
      Affine suf{1.0, 0.0};
      for (int w = kGaeThreads / 32 - 1; w >= 0; --w) {
        const Affine cur = s_warp[w];
        s_warp[w] = suf;
        suf = compose(cur, suf);
      }
      double carry = 0.0;
      if (tid == 0) {
        tiles[tid].inc = suf.b;
        __threadfence();
        tiles[tid].flag = 2;
      } else {
        tiles[tid].a = suf.a;
        tiles[tid].b = suf.b;
        __threadfence();
        tiles[tid].flag = 1;
        Affine acc{1.0, 0.0};
        int p = tid - 1;
        while (!(dbg & 1)) {
          int f;
          do {
            f = tiles[p].flag;
          } while (f == 0);
          __threadfence();
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
        tiles[tid].inc = fma(suf.a, carry, suf.b);
        __threadfence();
        tiles[tid].flag = 2;
      }
      s_carry = carry;
      issue(s, atomicAdd(tile_counter, 1));  // refill this stage (all threads are past reading it)
    }
    __syncthreads();
    Affine lane_ex{__shfl_down_sync(0xffffffffu, incl.a, 1), __shfl_down_sync(0xffffffffu, incl.b, 1)};
    if (lane == 31) lane_ex = Affine{1.0, 0.0};
    const Affine after = compose(lane_ex, s_warp[warp]);
    double x = fma(after.a, s_carry, after.b);
    float av[kGaeItems], rv[kGaeItems];
#pragma unroll
    for (int q = kGaeItems - 1; q >= 0; --q) {
      double dl, ac;
      item(q, dl, ac);
      x = fma(ac, x, dl);
      av[q] = (float)x;
      rv[q] = (float)(x + (double)v[q]);
    }
    if (i0 + kGaeItems <= hi) {
      float4* a4 = reinterpret_cast<float4*>(adv + i0);
      float4* r4 = reinterpret_cast<float4*>(ret + i0);
      __stcs(a4, make_float4(av[0], av[1], av[2], av[3]));
      __stcs(a4 + 1, make_float4(av[4], av[5], av[6], av[7]));
      __stcs(r4, make_float4(rv[0], rv[1], rv[2], rv[3]));
      __stcs(r4 + 1, make_float4(rv[4], rv[5], rv[6], rv[7]));
    } else {
      for (int q = 0; q < kGaeItems; ++q)
        if (i0 + q < hi) {
          adv[i0 + q] = av[q];
          ret[i0 + q] = rv[q];
        }
    }
    __syncthreads();  // s_warp / s_carry reuse by the next tile
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

static int gae_debug_mode() {
  const char* e = getenv("VER_GAE_DEBUG");  // experiments only: 1 = skip the look-back wait
  return e ? atoi(e) : 0;
}

static void run_scan(Ctx* c, const float* r, const float* v, const uint8_t* d, const int32_t* env, int F,
                     const float* boot, const uint8_t* valid, double gamma, double lambda, float* adv,
                     float* ret) {
  if (F <= 0) return;
  const int ntiles = (F + kGaeTile - 1) / kGaeTile;
  DBuf<GaeTileState> tiles;
  DBuf<int> misc;
  tiles.reserve(c, ntiles);
  misc.reserve(c, 2);
  tiles.zero(ntiles);
  int* h = static_cast<int*>(c->pinned_buf(2 * sizeof(int)));
  h[0] = 0;
  h[1] = 0x7fffffff;
  misc.upload(h, 2);
  const size_t smem = sizeof(GaeStage) * kGaeStages;
  VER_CUDA(cudaFuncSetAttribute(gae_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  VER_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gae_scan_kernel, kGaeThreads, smem));
  const int grid = std::max(1, std::min(ntiles, per_sm * c->num_sms));
  gae_scan_kernel<<<grid, kGaeThreads, smem, c->stream>>>(r, v, d, env, F, boot, valid, gamma, lambda, adv, ret,
                                                          tiles.p, misc.p, misc.p + 1, gae_debug_mode());
  after_launch(c);
  misc.download(h, 2);
  sync(c);
  if (h[1] != 0x7fffffff)
    protocol_error("compute_gae: missing bootstrap value for env " + std::to_string(h[1]));
}

void compute_gae(DView& V, double gamma, double lambda) {
  Ctx* c = V.ctx;
  if (V.size == 0) return;
  if (V.env_contiguous) {
    run_scan(c, V.reward.p, V.value.p, V.done.p, V.env_index.p, V.fresh_prefix, V.env_bootstrap.p,
             V.env_bootstrap_valid.p, gamma, lambda, V.advantage.p, V.returns.p);
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
  run_scan(c, r2.p, v2.p, d2.p, e2.p, F, V.env_bootstrap.p, V.env_bootstrap_valid.p, gamma, lambda, a2.p,
           ret2.p);
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
