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

// One tile (2048 slots) per CTA, decoupled look-back.  Per thread the 8-item
// recursion runs in fp32 (<= 8 chained steps); warp / tile compositions and
// the cross-tile carry are fp64, which keeps long segments (gamma*lambda -> 1,
// 1024 steps) inside the fp32 rounding of the fp64 reference.  done bit 1
// marks an env's last fresh slot, so no per-env offsets are read; only env
// tails without `done` look up their env's bootstrap.  After the tile's
// compositions are known, only threads whose suffix reaches the tile end
// without a reset (a != 0) wait for the look-back; all others store at once.
__global__ void __launch_bounds__(kGaeThreads) gae_scan_kernel(
    const float* __restrict__ reward, const float* __restrict__ value, const uint8_t* __restrict__ done,
    const int32_t* __restrict__ env_of, int F, const float* __restrict__ boot,
    const uint8_t* __restrict__ boot_valid, double gamma, double lambda, float* __restrict__ adv,
    float* __restrict__ ret, volatile GaeTileState* tiles, int* tile_counter, int* err_env, int dbg) {
  __shared__ int s_tile;
  __shared__ Affine s_warp[kGaeThreads / 32];
  __shared__ double s_carry;
  __shared__ volatile int s_ready;
  const int ntiles = (F + kGaeTile - 1) / kGaeTile;
  if (threadIdx.x == 0) {
    s_tile = atomicAdd(tile_counter, 1);
    s_ready = 0;
  }
  __syncthreads();
  const int tid = s_tile;  // 0 = last tile of the array
  const int tile = ntiles - 1 - tid;
  const int lo = tile * kGaeTile;
  const int hi = min(F, lo + kGaeTile);
  const int i0 = lo + threadIdx.x * kGaeItems;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float gf = (float)gamma, glf = (float)(gamma * lambda);

  float r[kGaeItems], v[kGaeItems + 1];
  uint32_t dw[2];
  if (i0 + kGaeItems <= hi) {
    const float4* r4 = reinterpret_cast<const float4*>(reward + i0);
    const float4* v4 = reinterpret_cast<const float4*>(value + i0);
    const float4 x0 = __ldcs(r4), x1 = __ldcs(r4 + 1), y0 = __ldcs(v4), y1 = __ldcs(v4 + 1);
    const uint2 dd = __ldcs(reinterpret_cast<const uint2*>(done + i0));
    r[0] = x0.x; r[1] = x0.y; r[2] = x0.z; r[3] = x0.w;
    r[4] = x1.x; r[5] = x1.y; r[6] = x1.z; r[7] = x1.w;
    v[0] = y0.x; v[1] = y0.y; v[2] = y0.z; v[3] = y0.w;
    v[4] = y1.x; v[5] = y1.y; v[6] = y1.z; v[7] = y1.w;
    dw[0] = dd.x;
    dw[1] = dd.y;
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
  }
  v[kGaeItems] = (i0 + kGaeItems < F) ? value[i0 + kGaeItems] : 0.f;

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
        const int e = env_of[i0 + q];
        if (!boot_valid[e]) atomicMin(err_env, e);
        vnext = boot[e];
      }
    }
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
  __syncthreads();
  Affine lane_ex{__shfl_down_sync(0xffffffffu, incl.a, 1), __shfl_down_sync(0xffffffffu, incl.b, 1)};
  if (lane == 31) lane_ex = Affine{1.0, 0.0};
  if (warp == 0) {
    if (lane == 0) {
      Affine suf{1.0, 0.0};
      for (int w = kGaeThreads / 32 - 1; w >= 0; --w) {
        const Affine cur = s_warp[w];
        s_warp[w] = suf;
        suf = compose(cur, suf);
      }
      // publish the tile aggregate first, then release the other warps
      if (tid == 0) {
        tiles[tid].inc = suf.b;
        __threadfence();
        tiles[tid].flag = 2;
      } else {
        tiles[tid].a = suf.a;
        tiles[tid].b = suf.b;
        __threadfence();
        tiles[tid].flag = 1;
      }
      __threadfence_block();
      s_ready = 1;
      double carry = 0.0;  // A at hi
      if (tid != 0) {
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
      __threadfence_block();
      s_ready = 2;
    }
    __syncwarp();
  } else {
    while (s_ready == 0) {
    }
  }
  const Affine after = compose(lane_ex, s_warp[warp]);  // maps A at hi to A after this thread's items
  double x = after.b;
  if (after.a != 0.0) {  // this thread's values depend on the carry
    while (s_ready != 2) {
    }
    x = fma(after.a, s_carry, after.b);
  }
  float xf = (float)x;
  float av[kGaeItems], rv[kGaeItems];
#pragma unroll
  for (int q = kGaeItems - 1; q >= 0; --q) {
    xf = fmaf(ac[q], xf, dl[q]);
    av[q] = xf;
    rv[q] = xf + v[q];
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
  gae_scan_kernel<<<ntiles, kGaeThreads, 0, c->stream>>>(r, v, d, env, F, boot, valid, gamma, lambda, adv, ret,
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
