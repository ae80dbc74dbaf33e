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
constexpr int kGaeOffSmem = 2048;                   // env offsets staged per tile

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

__device__ __forceinline__ int upper_bound_i32(const int32_t* p, int n, int x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (p[mid] <= x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(kGaeThreads) gae_scan_kernel(
    const float* __restrict__ reward, const float* __restrict__ value,
    const uint8_t* __restrict__ done, int F, const int32_t* __restrict__ off, int N,
    const float* __restrict__ boot, const uint8_t* __restrict__ boot_valid, double gamma,
    double lambda, float* __restrict__ adv, float* __restrict__ ret,
    volatile GaeTileState* tiles, int* tile_counter, int* err_env, const int32_t* __restrict__ tile_env,
    int dbg) {
  __shared__ int s_tile;
  __shared__ int s_e0, s_ne;
  __shared__ int32_t s_off[kGaeOffSmem + 1];
  __shared__ Affine s_warp[kGaeThreads / 32];
  __shared__ double s_carry;
  const int ntiles = (F + kGaeTile - 1) / kGaeTile;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1);
  __syncthreads();
  const int tid = s_tile;                // 0 = last tile of the array
  const int tile = ntiles - 1 - tid;
  const int lo = tile * kGaeTile;
  const int hi = min(F, lo + kGaeTile);
  const int i0 = lo + threadIdx.x * kGaeItems;

  // 1) the tile's r, V, done: issued first so their latency overlaps the env setup
  float r[kGaeItems], v[kGaeItems + 1];
  uint8_t d[kGaeItems];
  if (i0 + kGaeItems <= hi && (((uintptr_t)(reward + i0)) & 15) == 0) {
    const float4* r4 = reinterpret_cast<const float4*>(reward + i0);
    const float4* v4 = reinterpret_cast<const float4*>(value + i0);
    float4 x0 = __ldcs(r4), x1 = __ldcs(r4 + 1), y0 = __ldcs(v4), y1 = __ldcs(v4 + 1);
    r[0] = x0.x; r[1] = x0.y; r[2] = x0.z; r[3] = x0.w;
    r[4] = x1.x; r[5] = x1.y; r[6] = x1.z; r[7] = x1.w;
    v[0] = y0.x; v[1] = y0.y; v[2] = y0.z; v[3] = y0.w;
    v[4] = y1.x; v[5] = y1.y; v[6] = y1.z; v[7] = y1.w;
    const uint2 dd = __ldcs(reinterpret_cast<const uint2*>(done + i0));
    const uint8_t* db = reinterpret_cast<const uint8_t*>(&dd);
#pragma unroll
    for (int k = 0; k < kGaeItems; ++k) d[k] = db[k];
  } else {
#pragma unroll
    for (int k = 0; k < kGaeItems; ++k) {
      const int i = i0 + k;
      r[k] = i < hi ? reward[i] : 0.f;
      v[k] = i < hi ? value[i] : 0.f;
      d[k] = i < hi ? done[i] : 1;
    }
  }
  v[kGaeItems] = (i0 + kGaeItems < F) ? value[i0 + kGaeItems] : 0.f;

  // 2) env range of this tile (precomputed per tile); stage its offsets in smem
  if (threadIdx.x == 0) {
    const int e0 = tile_env[tile];
    const int e1 = tile_env[tile + 1];  // env of slot hi (or N)
    s_e0 = e0;
    s_ne = min(e1, N - 1) - e0 + 2;  // offsets e0 .. e1+1
  }
  __syncthreads();
  const int e0 = s_e0, ne = s_ne;
  const bool smem_off = ne <= kGaeOffSmem + 1;
  if (smem_off)
    for (int k = threadIdx.x; k < ne; k += kGaeThreads) s_off[k] = off[e0 + k];
  __syncthreads();

  // 3) thread-local maps
  double delta[kGaeItems], acoef[kGaeItems];
  Affine mine{1.0, 0.0};
  const double gl = gamma * lambda;
  if (i0 < hi) {
    int e = smem_off ? e0 + upper_bound_i32(s_off, ne, i0) - 1 : upper_bound_i32(off, N + 1, i0) - 1;
    int next_bound = smem_off ? s_off[e - e0 + 1] : off[e + 1];
#pragma unroll
    for (int k = 0; k < kGaeItems; ++k) {
      const int i = i0 + k;
      if (i >= hi) {
        delta[k] = 0.0;
        acoef[k] = 1.0;  // identity map beyond the end
        continue;
      }
      while (i >= next_bound) {  // advance env (skips empty envs)
        ++e;
        next_bound = smem_off ? s_off[e - e0 + 1] : off[e + 1];
      }
      const bool tail = (i + 1 == next_bound);
      const double mask = d[k] ? 0.0 : 1.0;
      double vnext = 0.0;
      if (tail) {
        if (!d[k]) {
          if (!boot_valid[e]) atomicMin(err_env, e);
          vnext = (double)boot[e];
        }
      } else {
        vnext = (double)v[k + 1];
      }
      delta[k] = (double)r[k] + gamma * vnext * mask - (double)v[k];
      acoef[k] = tail ? 0.0 : gl * mask;
    }
#pragma unroll
    for (int k = kGaeItems - 1; k >= 0; --k) mine = compose(Affine{acoef[k], delta[k]}, mine);
  }

  // block-level suffix scan of thread maps (thread t needs threads > t)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Affine incl = mine;  // inclusive suffix within warp
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    Affine y{__shfl_down_sync(0xffffffffu, incl.a, o), __shfl_down_sync(0xffffffffu, incl.b, o)};
    if (lane + o < 32) incl = compose(incl, y);
  }
  if (lane == 0) s_warp[warp] = incl;
  __syncthreads();
  if (threadIdx.x == 0) {
    // tile aggregate and warp suffixes (warps > w)
    Affine suf{1.0, 0.0};
    for (int w = kGaeThreads / 32 - 1; w >= 0; --w) {
      const Affine cur = s_warp[w];
      s_warp[w] = suf;  // exclusive suffix of warp w
      suf = compose(cur, suf);
    }
    // publish aggregate, then look back toward the end of the array
    double carry = 0.0;  // A at `hi` (0 past the last fresh slot)
    if (tid == 0) {
      tiles[tid].inc = suf.b;  // a applies to A_F which is never used (tail)
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
  }
  __syncthreads();
  if (i0 >= hi) return;
  // A after this thread's last item: apply (lane-exclusive warp suffix) then warp suffix
  Affine lane_ex{__shfl_down_sync(0xffffffffu, incl.a, 1), __shfl_down_sync(0xffffffffu, incl.b, 1)};
  if (lane == 31) lane_ex = Affine{1.0, 0.0};
  const Affine wsuf = s_warp[warp];
  const Affine after = compose(lane_ex, wsuf);
  double x = fma(after.a, s_carry, after.b);
  float av[kGaeItems], rv[kGaeItems];
#pragma unroll
  for (int k = kGaeItems - 1; k >= 0; --k) {
    x = fma(acoef[k], x, delta[k]);
    av[k] = (float)x;
    const int i = i0 + k;
    rv[k] = i < hi ? (float)(x + (double)v[k]) : 0.f;
  }
  if (i0 + kGaeItems <= hi && (((uintptr_t)(adv + i0)) & 15) == 0) {
    float4* a4 = reinterpret_cast<float4*>(adv + i0);
    float4* r4 = reinterpret_cast<float4*>(ret + i0);
    __stcs(a4, make_float4(av[0], av[1], av[2], av[3]));
    __stcs(a4 + 1, make_float4(av[4], av[5], av[6], av[7]));
    __stcs(r4, make_float4(rv[0], rv[1], rv[2], rv[3]));
    __stcs(r4 + 1, make_float4(rv[4], rv[5], rv[6], rv[7]));
  } else {
    for (int k = 0; k < kGaeItems; ++k)
      if (i0 + k < hi) {
        adv[i0 + k] = av[k];
        ret[i0 + k] = rv[k];
      }
  }
}

// env containing the first slot of every tile (+ the env of slot F at [ntiles])
__global__ void gae_tile_env_kernel(const int32_t* __restrict__ off, int N, int F, int ntiles,
                                    int32_t* __restrict__ tile_env) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > ntiles) return;
  const int slot = min(t * kGaeTile, F - 1);
  tile_env[t] = (t == ntiles ? upper_bound_i32(off, N + 1, F - 1) : upper_bound_i32(off, N + 1, slot)) - 1;
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
                                  float* __restrict__ r2, float* __restrict__ v2, uint8_t* __restrict__ d2) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= F) return;
  const int i = (int)(keys[j] & 0xffffffffu);
  r2[j] = r[i];
  v2[j] = v[i];
  d2[j] = d[i];
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

static void run_scan(Ctx* c, const float* r, const float* v, const uint8_t* d, int F,
                     const int32_t* off, int N, const float* boot, const uint8_t* valid, double gamma,
                     double lambda, float* adv, float* ret) {
  if (F <= 0) return;
  const int ntiles = (F + kGaeTile - 1) / kGaeTile;
  DBuf<GaeTileState> tiles;
  DBuf<int> misc;
  DBuf<int32_t> tile_env;
  tiles.reserve(c, ntiles);
  misc.reserve(c, 2);
  tile_env.reserve(c, ntiles + 1);
  tiles.zero(ntiles);
  gae_tile_env_kernel<<<cdiv(ntiles + 1, 256), 256, 0, c->stream>>>(off, N, F, ntiles, tile_env.p);
  after_launch(c);
  const int init[2] = {0, 0x7fffffff};
  int* h = static_cast<int*>(c->pinned_buf(2 * sizeof(int)));
  h[0] = init[0];
  h[1] = init[1];
  misc.upload(h, 2);
  gae_scan_kernel<<<ntiles, kGaeThreads, 0, c->stream>>>(r, v, d, F, off, N, boot, valid, gamma, lambda,
                                                         adv, ret, tiles.p, misc.p, misc.p + 1, tile_env.p,
                                                         gae_debug_mode());
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
    run_scan(c, V.reward.p, V.value.p, V.done.p, V.fresh_prefix, V.env_offsets.p, V.N,
             V.env_bootstrap.p, V.env_bootstrap_valid.p, gamma, lambda, V.advantage.p, V.returns.p);
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
  r2.reserve(c, F);
  v2.reserve(c, F);
  a2.reserve(c, F);
  ret2.reserve(c, F);
  d2.reserve(c, F);
  gae_gather_kernel<<<cdiv(F, 256), 256, 0, c->stream>>>(keys.p, F, V.reward.p, V.value.p, V.done.p, r2.p,
                                                         v2.p, d2.p);
  after_launch(c);
  run_scan(c, r2.p, v2.p, d2.p, F, off.p, N, V.env_bootstrap.p, V.env_bootstrap_valid.p, gamma, lambda,
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
