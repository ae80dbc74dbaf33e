// stepgemm.cu — the big recurrence timesteps as one persistent cooperative
// kernel: per step a 3xTF32 tcgen05 GEMM phase (split-K work items, at most one
// per CTA) and an elementwise gate phase, separated by grid barriers.
//
//   forward  step t: hU = h_{t-1}[0:B] U   (M = B, N = 3H, K = H), then the GRU
//                    gates of rows j < B (nn.cpp:235-250);
//   backward step t: dh = dhU_t[0:B] U^T   (M = B, N = H, K = 3H), then the gate
//                    gradient of the rows j < B_{t-1} of step t-1.
//
// Against one GEMM launch + one gate launch per step (policy.cu
// gru_forward_big / gru_backward_big) this removes two launches, the TMEM
// allocation and the tensor-map prefetch per step: the A operand's tensor map
// of every step is built on the host up front (the batch offsets are known
// after the pack) and read from global memory.  Warp roles as in the tcgen05
// GEMM (tc_gemm.cuh): TMA producer, MMA issuer, 4 split warps, 4 epilogue
// warps; the smem ring, the TMEM accumulator buffers and their mbarrier phases
// run on across steps.  All 320 threads join the gate phase.
#include <cstdlib>

#include "policy.cuh"
#include "tc_gemm.cuh"

namespace verg {
namespace sg {

using namespace tc;

struct Step {
  int B;        // GEMM rows (forward: bs_t; backward: bs_t, rows with a successor)
  int Bg;       // gate rows (forward: bs_t; backward: bs_{t-1})
  int o, op;    // packed offsets of the GEMM / gate rows (forward: o = offs_t, op = offs_{t-1} or -1 for h0)
  int Z, per;   // split-K count, K-blocks per split
  int tilesM;
  int pad;      // pair forward: 1 = the gates run in the GEMM epilogue (Z == 1, H % 32 == 0)
};

__device__ __forceinline__ void grid_sync(unsigned* count, unsigned& target) {
  __syncthreads();
  target += gridDim.x;
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(count, 1u);
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(count) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

// wait until *p >= need (acquire at gpu scope: the counted-in stores are visible)
__device__ __forceinline__ void spin_acquire(const unsigned* p, unsigned need) {
  unsigned v;
  do {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  } while (v < need);
}

// VER_REC_TRACE slots per step (CTA 0): start, first stage landed, last
// accumulator ready, partial stored, GEMM-phase barrier passed, gate done
constexpr int TR = 6;
// K-blocks per TMEM accumulation group (tc::PROMOTE in the general GEMM): the
// split-K items here hold <= 4 K-blocks at C2, so one drain per item
constexpr int SGP = 4;
// fp16x2 operand of the forward step GEMM: h_{t-1} s_h = hi + lo.  GRU states are
// convex combinations of tanh outputs and the initial state, so |h_t| <= M =
// max(1, max |h0|) for the whole launch; s_h = 2^(14 - floor(log2 M)) keeps
// M s_h < 2^15 < 65504 (hscale_kernel, from the max over h0).
__device__ __forceinline__ void split_h(float y, __half& hi, __half& lo) {
  hi = __float2half_rn(y);
  lo = __float2half_rn(y - __half2float(hi));
}
// hsc[0] = s_h, hsc[1] = (1 / s_U) / s_h for the GEMM epilogue
__global__ void hscale_kernel(const unsigned* __restrict__ hmax, const float* __restrict__ inv_u,
                              float* __restrict__ hsc) {
  float mx = __uint_as_float(*hmax);
  if (!(mx >= 1.f) || !isfinite(mx)) mx = 1.f;  // (a NaN / inf h0 makes the result non-finite anyway)
  const float sh = exp2f((float)(14 - ilogbf(mx)));
  hsc[0] = sh;
  hsc[1] = *inv_u / sh;
}
__global__ void h16_kernel(int64_t n, const float* __restrict__ x, const float* __restrict__ hsc,
                           __half* __restrict__ hi, __half* __restrict__ lo) {
  const float sh = hsc[0];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    split_h(x[i] * sh, hi[i], lo[i]);
}

// element i of a register-resident float4 array (i a compile-time constant after
// unrolling, so no local-memory copy)
template <int N>
__device__ __forceinline__ float f4at(const float4 (&a)[N], int i) {
  const float4 v = a[i >> 2];
  const int k = i & 3;
  return k == 0 ? v.x : k == 1 ? v.y : k == 2 ? v.z : v.w;
}
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}


// gate phase of one step over the grid: thread `tid` of `nthreads` walks
// (row j, units 4x .. 4x+3).  Forward: sum the Z partials of hU, GRU gates,
// h_t (nn.cpp:235-250); backward: sum the partials of dh_{t-1}, gate gradient
// of the rows of step t-1.
template <int DIR>
__device__ __forceinline__ void gate_phase(const Step& S, int H, const float* __restrict__ part,
                                           const float* __restrict__ xp, const float* __restrict__ h0,
                                           float* __restrict__ hidden, float* __restrict__ gates_out,
                                           float* __restrict__ hun_out, float* __restrict__ hprev_out,
                                           const float* __restrict__ dhidden, const float* __restrict__ gates,
                                           const float* __restrict__ hun, const float* __restrict__ hprev,
                                           float* __restrict__ dpre, float* __restrict__ dhu,
                                           float* __restrict__ gz, int tid, int nthreads,
                                           __half* __restrict__ h16hi = nullptr, __half* __restrict__ h16lo = nullptr,
                                           float hs = 1.f) {
  const int H3 = 3 * H, N = DIR == 0 ? H3 : H;
  const int H4 = H / 4;
  const size_t zs = (size_t)S.B * N;
  for (int idx = tid; idx < S.Bg * H4; idx += nthreads) {
    const int j = idx / H4, u4 = idx % H4;
    if (DIR == 0) {
      const size_t row3 = ((size_t)S.o + j) * H3 + 12 * (size_t)u4, row = ((size_t)S.o + j) * H + 4 * (size_t)u4;
      const size_t prow = (size_t)j * H3 + 12 * (size_t)u4;
      float s12[12];
#pragma unroll
      for (int e = 0; e < 12; ++e) s12[e] = 0.f;
#pragma unroll
      for (int z = 0; z < 8; ++z) {
        if (z < S.Z) {  // predicated, so all Z partial loads are in flight together
          const float4* p4 = reinterpret_cast<const float4*>(part + z * zs + prow);
          const float4 a = p4[0], b = p4[1], c = p4[2];
          s12[0] += a.x; s12[1] += a.y; s12[2] += a.z; s12[3] += a.w; s12[4] += b.x; s12[5] += b.y;
          s12[6] += b.z; s12[7] += b.w; s12[8] += c.x; s12[9] += c.y; s12[10] += c.z; s12[11] += c.w;
        }
      }
      const float4* x4 = reinterpret_cast<const float4*>(xp + row3);
      const float4 xa = x4[0], xb = x4[1], xc = x4[2];
      const float x[12] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w, xc.x, xc.y, xc.z, xc.w};
      const float* hp = S.op < 0 ? h0 + (size_t)j * H : hidden + ((size_t)S.op + j) * H;
      const float4 hp4 = *reinterpret_cast<const float4*>(hp + 4 * u4);
      const float hpv[4] = {hp4.x, hp4.y, hp4.z, hp4.w};
      float hn[4], g[12];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float rg = gate_sigm(x[3 * e] + s12[3 * e]);
        const float zg = gate_sigm(x[3 * e + 1] + s12[3 * e + 1]);
        const float ng = gate_tanh(x[3 * e + 2] + rg * s12[3 * e + 2]);
        hn[e] = (1.f - zg) * ng + zg * hpv[e];
        g[3 * e] = rg;
        g[3 * e + 1] = zg;
        g[3 * e + 2] = ng;
      }
      *reinterpret_cast<float4*>(hidden + row) = make_float4(hn[0], hn[1], hn[2], hn[3]);
      if (h16hi) {  // fp16x2 halves of h_t for the next fp16x2 step GEMM
        __half hh[4], hl[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) split_h(hn[e] * hs, hh[e], hl[e]);
        reinterpret_cast<__half2*>(h16hi + row)[0] = __halves2half2(hh[0], hh[1]);
        reinterpret_cast<__half2*>(h16hi + row)[1] = __halves2half2(hh[2], hh[3]);
        reinterpret_cast<__half2*>(h16lo + row)[0] = __halves2half2(hl[0], hl[1]);
        reinterpret_cast<__half2*>(h16lo + row)[1] = __halves2half2(hl[2], hl[3]);
      }
      if (gates_out) {
        float4* g4 = reinterpret_cast<float4*>(gates_out + row3);
        g4[0] = make_float4(g[0], g[1], g[2], g[3]);
        g4[1] = make_float4(g[4], g[5], g[6], g[7]);
        g4[2] = make_float4(g[8], g[9], g[10], g[11]);
        *reinterpret_cast<float4*>(hun_out + row) = make_float4(s12[2], s12[5], s12[8], s12[11]);
        *reinterpret_cast<float4*>(hprev_out + row) = hp4;
      }
    } else {
      const size_t row = ((size_t)S.op + j) * H + 4 * (size_t)u4, row3 = ((size_t)S.op + j) * H3 + 12 * (size_t)u4;
      float dh[4] = {0.f, 0.f, 0.f, 0.f};
      if (j < S.B) {
#pragma unroll
        for (int z = 0; z < 8; ++z) {
          if (z < S.Z) {
            const float4 p = *reinterpret_cast<const float4*>(part + z * zs + (size_t)j * H + 4 * u4);
            dh[0] += p.x; dh[1] += p.y; dh[2] += p.z; dh[3] += p.w;
          }
        }
        const float4 q = *reinterpret_cast<const float4*>(gz + ((size_t)S.o + j) * H + 4 * u4);
        dh[0] += q.x; dh[1] += q.y; dh[2] += q.z; dh[3] += q.w;
      }
      const float4 d4 = *reinterpret_cast<const float4*>(dhidden + row);
      const float4 hn4 = *reinterpret_cast<const float4*>(hun + row);
      const float4 hp4 = *reinterpret_cast<const float4*>(hprev + row);
      const float dv[4] = {d4.x, d4.y, d4.z, d4.w}, hnv[4] = {hn4.x, hn4.y, hn4.z, hn4.w},
                  hpv[4] = {hp4.x, hp4.y, hp4.z, hp4.w};
      const float4* g4 = reinterpret_cast<const float4*>(gates + row3);
      const float4 ga = g4[0], gb = g4[1], gc = g4[2];
      const float gt[12] = {ga.x, ga.y, ga.z, ga.w, gb.x, gb.y, gb.z, gb.w, gc.x, gc.y, gc.z, gc.w};
      float o1[12], o2[12], gzv[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float gg = dv[e] + dh[e];
        const float r = gt[3 * e], zg = gt[3 * e + 1], n = gt[3 * e + 2];
        const float dn = gg * (1.f - zg);
        const float dz = gg * (hpv[e] - n);
        const float dpn = dn * (1.f - n * n);
        const float dr = dpn * hnv[e];
        const float dpr = dr * r * (1.f - r);
        const float dpz = dz * zg * (1.f - zg);
        o1[3 * e] = dpr;
        o1[3 * e + 1] = dpz;
        o1[3 * e + 2] = dpn;
        o2[3 * e] = dpr;
        o2[3 * e + 1] = dpz;
        o2[3 * e + 2] = dpn * r;
        gzv[e] = gg * zg;
      }
      float4* p1 = reinterpret_cast<float4*>(dpre + row3);
      float4* p2 = reinterpret_cast<float4*>(dhu + row3);
      p1[0] = make_float4(o1[0], o1[1], o1[2], o1[3]);
      p1[1] = make_float4(o1[4], o1[5], o1[6], o1[7]);
      p1[2] = make_float4(o1[8], o1[9], o1[10], o1[11]);
      p2[0] = make_float4(o2[0], o2[1], o2[2], o2[3]);
      p2[1] = make_float4(o2[4], o2[5], o2[6], o2[7]);
      p2[2] = make_float4(o2[8], o2[9], o2[10], o2[11]);
      *reinterpret_cast<float4*>(gz + row) = make_float4(gzv[0], gzv[1], gzv[2], gzv[3]);
    }
  }
}

// F16 (forward only): the fp16x2 GEMM phase of the pair kernel on single CTAs --
// A = h_{t-1} halves (amaps[2 si], [2 si + 1]), B = U's transposed K-major halves,
// accumulator x fscale[1]; the gate phase writes h_t's halves (scale fscale[0])
template <int DIR, int F16 = 0>  // 0 forward (B MN-major: U stored K x N), 1 backward (B K-major: U stored N x K)
__global__ void __launch_bounds__(THREADS, 1) gru_step_gemm_kernel(
    int nsteps, const Step* __restrict__ steps, const CUtensorMap* __restrict__ amaps,
    const __grid_constant__ CUtensorMap bmap, int H, float* __restrict__ part, unsigned* bar,
    // forward
    const float* __restrict__ xp, const float* __restrict__ h0, float* __restrict__ hidden,
    float* __restrict__ gates_out, float* __restrict__ hun_out, float* __restrict__ hprev_out,
    // backward
    const float* __restrict__ dhidden, const float* __restrict__ gates, const float* __restrict__ hun,
    const float* __restrict__ hprev, float* __restrict__ dpre, float* __restrict__ dhu, float* __restrict__ gz,
    long long* trace, const __grid_constant__ CUtensorMap bmap_lo, int blo, __half* __restrict__ h16hi,
    __half* __restrict__ h16lo, const float* __restrict__ fscale) {
  // blo: U's lo part (x - trunc_tf32(x)) comes pre-split from the parameters' lo
  // copy (policy.cu split_lo_kernel) by TMA; the split warps then only split A
  static_assert(!F16 || DIR == 0, "fp16x2 single-CTA steps: forward only");
  constexpr int AMAJ = 0, BMAJ = (DIR == 0 && !F16) ? 1 : 0;
  constexpr int BKE = F16 ? 64 : BK;  // K elements per stage
  extern __shared__ uint8_t smem_raw[];
  // 1024-aligned by pointer arithmetic on the __shared__ array, so that the compiler
  // keeps the shared address space (LDS/STS, not generic LD/ST) for derived pointers
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* stg_all = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES + EPI_BYTES);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * STAGES + 2 * NACC);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int H3 = 3 * H, N = DIR == 0 ? H3 : H, K = DIR == 0 ? H : H3;
  const int tilesN = (N + BN - 1) / BN;
  const int nkb_total = (K + BKE - 1) / BKE;
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar0 = smem_u32(bars);
  auto full_bar = [&](int s) { return bar0 + 8 * s; };
  auto split_bar = [&](int s) { return bar0 + 8 * (STAGES + s); };
  auto empty_bar = [&](int s) { return bar0 + 8 * (2 * STAGES + s); };
  auto acc_full = [&](int b) { return bar0 + 8 * (3 * STAGES + b); };
  auto acc_empty = [&](int b) { return bar0 + 8 * (3 * STAGES + NACC + b); };
  auto tile = [&](int s, int which) { return sbase + s * STAGE_BYTES + which * TILE_BYTES; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(split_bar(s), SPLIT_WARPS);
      mbar_init(empty_bar(s), 1);
    }
    for (int b = 0; b < NACC; ++b) {
      mbar_init(acc_full(b), 1);
      mbar_init(acc_empty(b), EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&bmap)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(NACC * BN)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  unsigned target = 0;
  // pipeline counters, continued across steps (each role advances its own)
  int it_tma = 0, it_mma = 0, it_split = 0, g_mma = 0, g_epi = 0;
  int b_pre = 0;  // producer: B tiles of this step's first stages already issued
  auto load_b = [&](int s, int k0, int n0) {
    if (BMAJ == 0) {
      tma_load_2d(tile(s, 2), &bmap, full_bar(s), k0, n0);
      if (blo) tma_load_2d(tile(s, 3), &bmap_lo, full_bar(s), k0, n0);
    } else {
#pragma unroll
      for (int c = 0; c < BN / 32; ++c) tma_load_2d(tile(s, 2) + c * 4096, &bmap, full_bar(s), n0 + 32 * c, k0);
      if (blo) {
#pragma unroll
        for (int c = 0; c < BN / 32; ++c)
          tma_load_2d(tile(s, 3) + c * 4096, &bmap_lo, full_bar(s), n0 + 32 * c, k0);
      }
    }
  };
  const uint32_t stage_tx = (F16 ? 4u : (blo ? 3u : 2u)) * TILE_BYTES;
  const float fsc = F16 ? fscale[1] : 1.f, hs = F16 ? fscale[0] : 1.f;

  for (int si = 0; si < nsteps; ++si) {
    if (trace && blockIdx.x == 0 && threadIdx.x == 0) trace[TR * si] = gtimer();
    const Step S = steps[si];
    // work items (tilesM x tilesN output tiles x Z K-splits) walked grid-stride:
    // a step with more tiles than CTAs (B > 1536 rows forward, > 4736 backward at
    // H = 512, i.e. C3's first steps) gives a CTA several items in a row; every
    // role walks the same item sequence
    const int W = S.B > 0 ? S.tilesM * tilesN * S.Z : 0;
    const CUtensorMap* amap = amaps + (F16 ? 2 * si : si);
    for (int item = blockIdx.x; item < W; item += gridDim.x) {
      const bool first_item = item == (int)blockIdx.x, last_item = item + (int)gridDim.x >= W;
      const int nt = item % tilesN, q = item / tilesN;
      const int m0 = (q % S.tilesM) * BM, n0 = nt * BN, z = q / S.tilesM;
      const int kb0 = z * S.per;
      const int nkb = max(0, min(nkb_total, kb0 + S.per) - kb0);
      if (warp == 0) {
        if (lane == 0) {
          if (first_item) asm volatile("fence.proxy.async.global;" ::: "memory");  // rows of the gate phase
          for (int i = 0; i < nkb; ++i, ++it_tma) {
            const int s = it_tma % STAGES;
            const uint32_t ph = (it_tma / STAGES) & 1;
            const int k0 = (kb0 + i) * BKE;
            if (!first_item || i >= b_pre) {
              mbar_wait(empty_bar(s), ph ^ 1);
              mbar_expect_tx(full_bar(s), stage_tx);
              load_b(s, k0, n0);
            }
            tma_load_2d(tile(s, 0), amap, full_bar(s), k0, m0);
            if (F16) tma_load_2d(tile(s, 1), amap + 1, full_bar(s), k0, m0);
          }
          // after this CTA's last item: the next step's first B tiles (U does not
          // change across steps) and its A tensor map, issued before the grid barriers
          if (last_item) b_pre = 0;
          if (last_item && si + 1 < nsteps) {
            const Step S2 = steps[si + 1];
            if (S2.B > 0 && (int)blockIdx.x < S2.tilesM * tilesN * S2.Z) {
              const int item2 = blockIdx.x;
              asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(amaps + (F16 ? 2 : 1) * (si + 1)))
                           : "memory");
              const int z2 = item2 / tilesN / S2.tilesM;
              const int kb2 = z2 * S2.per;
              const int nkb2 = max(0, min(nkb_total, kb2 + S2.per) - kb2);
              b_pre = min(nkb2, STAGES);
              for (int i = 0; i < b_pre; ++i) {
                const int s = (it_tma + i) % STAGES;
                mbar_wait(empty_bar(s), ((it_tma + i) / STAGES & 1) ^ 1);
                mbar_expect_tx(full_bar(s), stage_tx);
                load_b(s, (kb2 + i) * BKE, (item2 % tilesN) * BN);
              }
            }
          }
        }
      } else if (warp == 1) {
        const uint32_t fmt = F16 ? 0u : 2u;  // A / B f16 or tf32
        const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)AMAJ << 15) | ((uint32_t)BMAJ << 16) |
                               ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
        if (lane == 0) {
          int buf = 0;
          for (int i = 0; i < nkb; ++i, ++it_mma) {
            const int s = it_mma % STAGES;
            const uint32_t ph = (it_mma / STAGES) & 1;
            const bool first = (i % SGP) == 0;
            if (first) {
              buf = g_mma % NACC;
              const int u = g_mma / NACC;
              if (u >= 1) mbar_wait(acc_empty(buf), (u - 1) & 1);
            }
            mbar_wait(split_bar(s), ph);
            tc_fence_after();
            const uint32_t d = tmem + (uint32_t)(buf * BN);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {  // 32 bytes of K per MMA
              const uint64_t ah = operand_desc<AMAJ>(tile(s, 0), kk);
              const uint64_t bh = operand_desc<BMAJ>(tile(s, 2), kk);
              if (F16) {
                mma_f16(d, ah, bh, idesc, (!first || kk > 0) ? 1u : 0u);
                mma_f16(d, operand_desc<AMAJ>(tile(s, 1), kk), bh, idesc, 1u);
                mma_f16(d, ah, operand_desc<BMAJ>(tile(s, 3), kk), idesc, 1u);
              } else {
                mma_tf32(d, ah, bh, idesc, (!first || kk > 0) ? 1u : 0u);
                mma_tf32(d, operand_desc<AMAJ>(tile(s, 1), kk), bh, idesc, 1u);
                mma_tf32(d, ah, operand_desc<BMAJ>(tile(s, 3), kk), idesc, 1u);
              }
            }
            umma_commit(empty_bar(s));
            if ((i % SGP) == SGP - 1 || i == nkb - 1) {
              umma_commit(acc_full(buf));
              ++g_mma;
            }
          }
        }
        __syncwarp();
      } else if (warp < 2 + SPLIT_WARPS) {
        const int et = threadIdx.x - 64;
        for (int i = 0; i < nkb; ++i, ++it_split) {
          const int s = it_split % STAGES;
          const uint32_t ph = (it_split / STAGES) & 1;
          mbar_wait(full_bar(s), ph);
          if (trace && i == 0 && threadIdx.x == 64 && blockIdx.x == 0) trace[TR * si + 1] = gtimer();
          if (F16) {  // pre-split operands: relay
            __syncwarp();
            if (lane == 0) mbar_arrive(split_bar(s));
            continue;
          }
          uint8_t* st = smem + s * STAGE_BYTES;
          float4* ahi = reinterpret_cast<float4*>(st);
          float4* alo = reinterpret_cast<float4*>(st + TILE_BYTES);
          float4* bhi = reinterpret_cast<float4*>(st + 2 * TILE_BYTES);
          float4* blo_t = reinterpret_cast<float4*>(st + 3 * TILE_BYTES);
          if (blo) {
#pragma unroll 4
            for (int qq = et; qq < TILE_BYTES / 16; qq += 32 * SPLIT_WARPS) alo[qq] = lo_tf32(ahi[qq]);
          } else {
#pragma unroll 4
            for (int qq = et; qq < TILE_BYTES / 16; qq += 32 * SPLIT_WARPS) {
              alo[qq] = lo_tf32(ahi[qq]);
              blo_t[qq] = lo_tf32(bhi[qq]);
            }
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(split_bar(s));
        }
      } else {
        // accumulator promotion + partial-tile epilogue: part[z][m][n]
        const int lane_base = 32 * (warp & 3);
        float* stg = stg_all + (warp & 3) * 32 * EPI_LD;
        const int ngroups = (nkb + SGP - 1) / SGP;
        float sums[BN];
#pragma unroll
        for (int j = 0; j < BN; ++j) sums[j] = 0.f;
        for (int gq = 0; gq < ngroups; ++gq, ++g_epi) {
          const int buf = g_epi % NACC;
          mbar_wait(acc_full(buf), (g_epi / NACC) & 1);
          tc_fence_after();
          if (trace && gq == ngroups - 1 && threadIdx.x == 192 && blockIdx.x == 0) trace[TR * si + 2] = gtimer();
#pragma unroll
          for (int cc = 0; cc < BN / 32; ++cc) {
            uint32_t r[32];
            const uint32_t taddr = tmem + ((uint32_t)lane_base << 16) + (uint32_t)(buf * BN + cc * 32);
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                  "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                  "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                  "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                  "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int j = 0; j < 32; ++j) sums[cc * 32 + j] += __uint_as_float(r[j]);
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(acc_empty(buf));
        }
        if (F16) {  // undo the operand scales (powers of two)
#pragma unroll
          for (int j = 0; j < BN; ++j) sums[j] *= fsc;
        }
        const int rr = lane >> 3, c4 = (lane & 7) * 4;
#pragma unroll
        for (int cc = 0; cc < BN / 32; ++cc) {
#pragma unroll
          for (int qq = 0; qq < 8; ++qq)
            *reinterpret_cast<float4*>(stg + lane * EPI_LD + 4 * qq) =
                make_float4(sums[cc * 32 + 4 * qq], sums[cc * 32 + 4 * qq + 1], sums[cc * 32 + 4 * qq + 2],
                            sums[cc * 32 + 4 * qq + 3]);
          __syncwarp();
          const int n = n0 + cc * 32 + c4;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int r = 4 * k + rr;
            const int m = m0 + lane_base + r;
            const float4 v = *reinterpret_cast<const float4*>(stg + r * EPI_LD + c4);
            if (m < S.B && n < N) *reinterpret_cast<float4*>(part + ((size_t)z * S.B + m) * N + n) = v;
          }
          __syncwarp();
        }
        if (trace && threadIdx.x == 192 && blockIdx.x == 0) trace[TR * si + 3] = gtimer();
      }
    }
    grid_sync(bar, target);  // all partials of step si written
    if (trace && blockIdx.x == 0 && threadIdx.x == 0) trace[TR * si + 4] = gtimer();

    gate_phase<DIR>(S, H, part, xp, h0, hidden, gates_out, hun_out, hprev_out, dhidden, gates, hun, hprev, dpre, dhu,
                    gz, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x, F16 ? h16hi : nullptr,
                    F16 ? h16lo : nullptr, hs);
    if (trace && blockIdx.x == 0 && threadIdx.x == 0) trace[TR * si + 5] = gtimer();
    if (si + 1 < nsteps) grid_sync(bar, target);  // step si's rows before step si+1's GEMM reads them
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(NACC * BN) : "memory");
  }
}

// ---------------------------------------------- CTA-pair step kernel (big C3 steps)
// The same per-step schedule (split-K GEMM phase, grid barrier, gate phase,
// grid barrier) with the GEMM phase on CTA pairs and 256 x 256 tiles
// (tc_gemm.cuh p2::tc_gemm2_kernel): per SM and MMA cycle half the TMA bytes
// of the 128 x 128 single-CTA phase.  Used for the steps with >= 1024 rows
// (the first ~50 steps of a C3 minibatch; VER_REC_PAIR_ROWS), launched as
// clusters of 2 with all CTAs resident (one per SM).
// Pair tile width per direction: the forward's N = 3H columns interleave the three
// gates of each unit (column 3u + g), so its tiles are 192 columns = 64 whole
// units (a 256-column tile would cut a unit at every boundary); that lets a
// split-K-free forward step apply the GRU gates in the GEMM epilogue.
template <int DIR>
struct PairTile {
  static constexpr int BN = DIR == 0 ? 192 : p2::BN2;
  static constexpr int BNH = BN / 2;           // B columns per CTA
  static constexpr int BBYTES = BNH * BK * 4;  // one CTA's B half of a stage
};
constexpr int kPairAccStride = p2::BN2;         // TMEM columns per accumulator buffer (2 x 256 allocated)
// Shared memory of the pair step kernel: NST operand stages, then the epilogue
// staging per warp -- the partial-tile path 32 x SLD floats, the fused gate path
// CH accumulator rows [CH][kFRow] + a RING-slot cp.async ring of xp rows [2][kFRow] and
// h_{t-1} rows [2][32] (row stride 100: conflict-free float4 rows).  The fp16x2
// variant trades one operand stage for a deep ring: its MMAs are twice as fast,
// and the gate epilogue needs ~9 groups of loads in flight to run at HBM speed.
constexpr int kFRow = 100;
template <int F16>
struct PairCfg {
  static constexpr int NST = F16 ? 2 : p2::STAGES2;
  static constexpr int RING = F16 ? 4 : 2;
  static constexpr int CH = F16 ? 8 : 4;  // accumulator rows staged at a time
  static constexpr int GR = F16 ? 4 : 2;  // rows per epilogue group (cp.async ring slot)
  static constexpr int FUSED = CH * kFRow + RING * GR * (kFRow + 32);
  static constexpr int WF = FUSED > 32 * p2::SLD ? FUSED : 32 * p2::SLD;  // floats per epilogue warp
  static constexpr int EPI = p2::EPIW * WF * 4;
  static constexpr int SMEM = NST * p2::STAGE2 + EPI + 1024 + 256;
  static_assert(SMEM <= 232448, "smem budget");
};

// F16 (forward only): fp16x2 GEMM phase (tc_gemm.cuh F16): A = h_{t-1} halves
// (amaps[2 si], amaps[2 si + 1]; written next to h_t by the previous step's
// epilogue / gate phase), B = U's transposed K-major halves (bmap / bmap_lo),
// accumulator x *fscale; 64 K per stage, the split warps only relay.
template <int DIR, int F16 = 0>
__global__ void __launch_bounds__(p2::THREADS2, 1) gru_step_gemm2_kernel(
    int nsteps, const Step* __restrict__ steps, const CUtensorMap* __restrict__ amaps,
    const __grid_constant__ CUtensorMap bmap, int H, float* __restrict__ part, unsigned* bar,
    const float* __restrict__ xp, const float* __restrict__ h0, float* __restrict__ hidden,
    float* __restrict__ gates_out, float* __restrict__ hun_out, float* __restrict__ hprev_out,
    const float* __restrict__ dhidden, const float* __restrict__ gates, const float* __restrict__ hun,
    const float* __restrict__ hprev, float* __restrict__ dpre, float* __restrict__ dhu, float* __restrict__ gz,
    const __grid_constant__ CUtensorMap bmap_lo, int blo, long long* __restrict__ trace, int rbs,
    __half* __restrict__ h16hi, __half* __restrict__ h16lo, const float* __restrict__ fscale) {
  using namespace p2;
  static_assert(!F16 || DIR == 0, "fp16x2 step GEMMs: forward only");
  constexpr int AMAJ = 0, BMAJ = (DIR == 0 && !F16) ? 1 : 0;
  constexpr int BKE = F16 ? 64 : BK;  // K elements per stage
  constexpr int NST = PairCfg<F16>::NST, RING = PairCfg<F16>::RING;
  constexpr int PBN = PairTile<DIR>::BN, PBNH = PairTile<DIR>::BNH;
  extern __shared__ uint8_t smem_raw[];
  // 1024-aligned by pointer arithmetic on the __shared__ array, so that the compiler
  // keeps the shared address space (LDS/STS, not generic LD/ST) for derived pointers
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* stg_all = reinterpret_cast<float*>(smem + NST * STAGE2);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NST * STAGE2 + PairCfg<F16>::EPI);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * NST + 2 * NACC2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cta_rank();
  const bool leader = rank == 0;
  const int pair_id = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int H3 = 3 * H, N = DIR == 0 ? H3 : H, K = DIR == 0 ? H : H3;
  const int tilesN = (N + PBN - 1) / PBN;
  const int nkb_total = (K + BKE - 1) / BKE;
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar0 = smem_u32(bars);
  auto full_bar = [&](int s) { return bar0 + 8 * s; };
  auto split_bar = [&](int s) { return bar0 + 8 * (NST + s); };
  auto empty_bar = [&](int s) { return bar0 + 8 * (2 * NST + s); };
  auto acc_full = [&](int b) { return bar0 + 8 * (3 * NST + b); };
  auto acc_empty = [&](int b) { return bar0 + 8 * (3 * NST + NACC2 + b); };
  auto tileA = [&](int s, int lo) { return sbase + s * STAGE2 + lo * TILE; };
  auto tileB = [&](int s, int lo) { return sbase + s * STAGE2 + (2 + lo) * TILE; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(split_bar(s), 2 * SPLITW);
      mbar_init(empty_bar(s), 1);
    }
    for (int b = 0; b < NACC2; ++b) {
      mbar_init(acc_full(b), 1);
      mbar_init(acc_empty(b), 2 * EPIW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&bmap)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(NACC2 * BN2)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  unsigned target = 0;
  unsigned* const rbf = bar + 32;  // row-tile counters of the fused steps, [nsteps][rbs]
  const float fsc = F16 ? fscale[1] : 1.f;  // 1 / (s_h s_U) of the fp16x2 GEMM (hscale_kernel)
  const float hs = F16 ? fscale[0] : 1.f;   // s_h: h_t's halves for the next step
  int it_tma = 0, it_mma = 0, it_split = 0, g_mma = 0, g_epi = 0;
  const uint32_t stage_tx = (F16 ? 2u : 1u) * TILE + (blo ? 2u : 1u) * (uint32_t)PairTile<DIR>::BBYTES;

  for (int si = 0; si < nsteps; ++si) {
    const Step S = steps[si];
    const int W = S.B > 0 ? S.tilesM * tilesN * S.Z : 0;  // tilesM in 256-row pair tiles
    if (trace && blockIdx.x == 0 && threadIdx.x == 0) trace[TR * si] = gtimer();
    const CUtensorMap* amap = amaps + (F16 ? 2 * si : si);
    for (int item = pair_id; item < W; item += npairs) {
      const bool first_item = item == pair_id;
      const int nt = item % tilesN, q = item / tilesN;
      const int m0 = (q % S.tilesM) * BM2, n0 = nt * PBN, z = q / S.tilesM;
      const int kb0 = z * S.per;
      const int nkb = max(0, min(nkb_total, kb0 + S.per) - kb0);
      // K-blocks per accumulation group: a fused item accumulates all of K in TMEM,
      // so the accumulator buffers alternate per item and the gate epilogue of one
      // item overlaps the MMAs of the next
      const int sgp = DIR == 0 && S.pad != 0 ? max(nkb, 1) : SGP;
      // Row-block dataflow after a fused step (no grid barrier): this item's A rows
      // (h_{t-1}, pair row tile m0 / BM2) are complete once all 2 x EPIW epilogue
      // warps of the previous step's tilesN items on that row tile have counted in
      unsigned* dep = DIR == 0 && si > 0 && steps[si - 1].pad != 0 ? rbf + (size_t)(si - 1) * rbs + m0 / BM2 : nullptr;
      const unsigned dep_need = 2u * EPIW * (unsigned)tilesN;
      if (warp == 0) {
        if (lane == 0) {
          if (dep) {
            spin_acquire(dep, dep_need);
            asm volatile("fence.proxy.async.global;" ::: "memory");  // generic stores -> TMA reads
          } else if (first_item) {
            asm volatile("fence.proxy.async.global;" ::: "memory");  // rows of the gate phase
          }
          const int am = m0 + (int)rank * BM, bn = n0 + (int)rank * PBNH;
          for (int i = 0; i < nkb; ++i, ++it_tma) {
            const int s = it_tma % NST;
            const uint32_t ph = (it_tma / NST) & 1;
            const int k0 = (kb0 + i) * BKE;
            mbar_wait(empty_bar(s), ph ^ 1);
            mbar_expect_tx(full_bar(s), stage_tx);
            if (F16) {
              tma_load_2d(tileB(s, 0), &bmap, full_bar(s), k0, bn);
              tma_load_2d(tileB(s, 1), &bmap_lo, full_bar(s), k0, bn);
              tma_load_2d(tileA(s, 0), amap, full_bar(s), k0, am);
              tma_load_2d(tileA(s, 1), amap + 1, full_bar(s), k0, am);
              continue;
            }
            if (BMAJ == 0) {
              tma_load_2d(tileB(s, 0), &bmap, full_bar(s), k0, bn);
              if (blo) tma_load_2d(tileB(s, 1), &bmap_lo, full_bar(s), k0, bn);
            } else {
#pragma unroll
              for (int c = 0; c < PBNH / 32; ++c)
                tma_load_2d(tileB(s, 0) + c * 4096, &bmap, full_bar(s), bn + 32 * c, k0);
              if (blo) {
#pragma unroll
                for (int c = 0; c < PBNH / 32; ++c)
                  tma_load_2d(tileB(s, 1) + c * 4096, &bmap_lo, full_bar(s), bn + 32 * c, k0);
              }
            }
            tma_load_2d(tileA(s, 0), amap, full_bar(s), k0, am);
          }
        }
      } else if (warp == 1) {
        const uint32_t fmt = F16 ? 0u : 2u;  // A / B f16 or tf32
        const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)AMAJ << 15) |
                               ((uint32_t)BMAJ << 16) | ((uint32_t)(PBN >> 3) << 17) | ((uint32_t)(BM2 >> 4) << 24);
        if (leader && lane == 0) {
          int buf = 0;
          for (int i = 0; i < nkb; ++i, ++it_mma) {
            const int s = it_mma % NST;
            const uint32_t ph = (it_mma / NST) & 1;
            const bool first = (i % sgp) == 0;
            if (first) {
              buf = g_mma % NACC2;
              const int u = g_mma / NACC2;
              if (u >= 1) mbar_wait(acc_empty(buf), (u - 1) & 1);
            }
            mbar_wait(split_bar(s), ph);
            tc_fence_after();
            const uint32_t d = tmem + (uint32_t)(buf * kPairAccStride);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {  // 32 bytes of K per MMA
              const uint64_t ah = operand_desc<AMAJ>(tileA(s, 0), kk);
              const uint64_t bh = operand_desc<BMAJ>(tileB(s, 0), kk);
              if (F16) {
                mma2_f16(d, ah, bh, idesc, (!first || kk > 0) ? 1u : 0u);
                mma2_f16(d, operand_desc<AMAJ>(tileA(s, 1), kk), bh, idesc, 1u);
                mma2_f16(d, ah, operand_desc<BMAJ>(tileB(s, 1), kk), idesc, 1u);
              } else {
                mma2_tf32(d, ah, bh, idesc, (!first || kk > 0) ? 1u : 0u);
                mma2_tf32(d, operand_desc<AMAJ>(tileA(s, 1), kk), bh, idesc, 1u);
                mma2_tf32(d, ah, operand_desc<BMAJ>(tileB(s, 1), kk), idesc, 1u);
              }
            }
            commit2(empty_bar(s));
            if ((i % sgp) == sgp - 1 || i == nkb - 1) {
              if (trace && blockIdx.x == 0) trace[TR * si + 1] = gtimer();  // last group issued
              commit2(acc_full(buf));
              ++g_mma;
            }
          }
        }
        __syncwarp();
      } else if (warp < 2 + SPLITW) {
        const int et = threadIdx.x - 64;
        for (int i = 0; i < nkb; ++i, ++it_split) {
          const int s = it_split % NST;
          const uint32_t ph = (it_split / NST) & 1;
          mbar_wait(full_bar(s), ph);
          if (F16) {  // pre-split operands: relay the landed stage to the leader
            __syncwarp();
            if (lane == 0) arrive_remote(to_rank(split_bar(s), 0));
            continue;
          }
          uint8_t* st = smem + s * STAGE2;
          const float4* ahi = reinterpret_cast<const float4*>(st);
          float4* alo = reinterpret_cast<float4*>(st + TILE);
          const float4* bhi = reinterpret_cast<const float4*>(st + 2 * TILE);
          float4* blo_t = reinterpret_cast<float4*>(st + 3 * TILE);
          if (blo) {
#pragma unroll 4
            for (int qq = et; qq < TILE / 16; qq += 32 * SPLITW) alo[qq] = lo_tf32(ahi[qq]);
          } else {
#pragma unroll 4
            for (int qq = et; qq < TILE / 16; qq += 32 * SPLITW) {
              alo[qq] = lo_tf32(ahi[qq]);
              if (qq < PairTile<DIR>::BBYTES / 16) blo_t[qq] = lo_tf32(bhi[qq]);
            }
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) arrive_remote(to_rank(split_bar(s), 0));
        }
      } else {
        // accumulator promotion + partial-tile epilogue: part[z][m][n] (own 128 rows,
        // column half (warp - 4) / 4)
        const int lq = warp & 3, half = (warp - 4) >> 2;
        const int lane_base = 32 * lq;
        float* stg = stg_all + (warp - 4) * PairCfg<F16>::WF;
        const int mrow0 = m0 + (int)rank * BM + lane_base, ncol0 = n0 + half * PBNH;
        if (DIR == 0 && S.pad != 0) {
          // GRU gates (nn.cpp:235-250) in the epilogue of a split-K-free item: this
          // warp's 32 rows x the 32 whole units [ncol0 / 3, ncol0 / 3 + 32).  The
          // accumulator arrives lane = row (TMEM lanes); the gate math runs lane = unit
          // so that every global access is a contiguous row segment (h / hUn / h_prev:
          // 128 B, xp / gates: 384 B).  Rows go in 16 groups of 2 through the warp's
          // staging area: hU rows from their owner lanes (CH at a time); the xp and h_{t-1} rows by
          // cp.async into a 3-buffer ring, two groups ahead (the first two during the
          // item's MMAs), so the loads cost no registers and their latency hides
          // behind two groups of gate math.
          float* fh = stg_all + (warp - 4) * PairCfg<F16>::WF;  // [CH][kFRow] hU rows
          float* fx0 = fh + PairCfg<F16>::CH * kFRow;            // [RING][2][kFRow] xp rows, then gates
          constexpr int GR = PairCfg<F16>::GR, NG = 32 / GR;    // rows per group, groups per item
          float* fp0 = fx0 + RING * GR * kFRow;                  // [RING][GR][32] h_{t-1} rows
          const int u0 = ncol0 / 3;
          const bool colok = ncol0 < N;
          const int blast = max(S.B - 1, 0);
          const float* hsrc = S.op < 0 ? h0 : hidden + (size_t)S.op * H;
          {
            const int m = min(mrow0 + lane, blast);
            const float* xr = xp + ((size_t)S.o + m) * N + (colok ? ncol0 : 0);
            asm volatile("prefetch.global.L2 [%0];" ::"l"(xr));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(xr + 32));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(xr + 64));
          }
          if (dep) spin_acquire(dep, dep_need);  // h_{t-1} rows of this row tile (read below)
          const int xl = lane < 24 ? 4 * lane : 0;  // this lane's float4 of a 96-column xp row
          auto issue = [&](int k) {  // rows GR k .. GR k + GR - 1 -> ring slot k % RING
            float* fx = fx0 + (k % RING) * GR * kFRow;
            float* fp = fp0 + (k % RING) * GR * 32;
#pragma unroll
            for (int r = 0; r < GR; ++r) {
              const int m = min(mrow0 + GR * k + r, blast);
              if (lane < 24)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(fx + r * kFRow + xl)),
                             "l"(xp + ((size_t)S.o + m) * N + (colok ? ncol0 + xl : 0))
                             : "memory");
              asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(fp + r * 32 + lane)),
                           "l"(hsrc + (size_t)m * H + (colok ? u0 + lane : 0))
                           : "memory");
            }
          };
#pragma unroll
          for (int k = 0; k < RING - 1; ++k) {  // the first RING - 1 groups during the item's MMAs
            issue(k);
            asm volatile("cp.async.commit_group;" ::: "memory");
          }
          const int buf = g_epi % NACC2;
          mbar_wait(acc_full(buf), (g_epi / NACC2) & 1);
          if (trace && blockIdx.x == 0 && threadIdx.x == 128) trace[TR * si + 2] = gtimer();  // last acc ready
          tc_fence_after();
          float acc[PBNH];
#pragma unroll
          for (int cc = 0; cc < PBNH / 32; ++cc) {
            uint32_t r[32];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                  "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                  "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                  "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                  "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                : "r"(tmem + ((uint32_t)lane_base << 16) + (uint32_t)(buf * kPairAccStride + half * PBNH + cc * 32)));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int j = 0; j < 32; ++j) acc[cc * 32 + j] = __uint_as_float(r[j]) * fsc;
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) arrive_remote(to_rank(acc_empty(buf), 0));  // TMEM free for the item after next
          ++g_epi;
#pragma unroll 1
          for (int k = 0; k < NG; ++k) {
            if (k + RING - 1 < NG) issue(k + RING - 1);
            asm volatile("cp.async.commit_group;" ::: "memory");  // (empty near the end: keeps the count)
            asm volatile("cp.async.wait_group %0;" ::"n"(RING - 1) : "memory");  // group k has landed
            constexpr int CH = PairCfg<F16>::CH, GPC = CH / GR;  // groups per staged chunk
            if (k % GPC == 0) {  // rows CH c .. CH c + CH - 1 from their owner lanes (fh is free: last group synced)
              if (lane / CH == k / GPC) {
                float4* d = reinterpret_cast<float4*>(fh + (lane % CH) * kFRow);
#pragma unroll
                for (int q = 0; q < PBNH / 4; ++q)
                  d[q] = make_float4(acc[4 * q], acc[4 * q + 1], acc[4 * q + 2], acc[4 * q + 3]);
              }
            }
            __syncwarp();
            float* fx = fx0 + (k % RING) * GR * kFRow;
            const float* fp = fp0 + (k % RING) * GR * 32;
#pragma unroll
            for (int r = 0; r < GR; ++r) {
              const int m = mrow0 + GR * k + r;
              const float* sh = fh + (GR * (k % GPC) + r) * kFRow + 3 * lane;
              float* sx = fx + r * kFRow + 3 * lane;
              const float hpv = fp[r * 32 + lane];
              const float rg = gate_sigm(sx[0] + sh[0]);
              const float zg = gate_sigm(sx[1] + sh[1]);
              const float ng = gate_tanh(sx[2] + rg * sh[2]);
              if (m < S.B && colok) {
                const size_t row = ((size_t)S.o + m) * H + u0 + lane;
                const float hnv = (1.f - zg) * ng + zg * hpv;
                hidden[row] = hnv;
                if (F16) split_h(hnv * hs, h16hi[row], h16lo[row]);
                if (gates_out) {
                  hun_out[row] = sh[2];
                  hprev_out[row] = hpv;
                }
              }
              sx[0] = rg;
              sx[1] = zg;
              sx[2] = ng;
            }
            __syncwarp();
            if (gates_out && lane < 24 && colok) {
#pragma unroll
              for (int r = 0; r < GR; ++r) {
                const int m = mrow0 + GR * k + r;
                if (m < S.B)
                  *reinterpret_cast<float4*>(gates_out + ((size_t)S.o + m) * N + ncol0 + xl) =
                      *reinterpret_cast<const float4*>(fx + r * kFRow + xl);
              }
            }
            __syncwarp();  // this ring slot and fh are rewritten by later groups
          }
          asm volatile("cp.async.wait_group 0;" ::: "memory");
          // this warp's h_t rows of row tile m0 / BM2 are written: count in
          __threadfence();
          __syncwarp();
          if (lane == 0) atomicAdd(rbf + (size_t)si * rbs + m0 / BM2, 1u);
          continue;
        }
        const int ngroups = (nkb + sgp - 1) / sgp;
        float sums[PBNH];
#pragma unroll
        for (int j = 0; j < PBNH; ++j) sums[j] = 0.f;
        for (int gq = 0; gq < ngroups; ++gq, ++g_epi) {
          const int buf = g_epi % NACC2;
          mbar_wait(acc_full(buf), (g_epi / NACC2) & 1);
          if (trace && blockIdx.x == 0 && threadIdx.x == 128) trace[TR * si + 2] = gtimer();  // last acc ready
          tc_fence_after();
#pragma unroll
          for (int cc = 0; cc < PBNH / 32; ++cc) {
            uint32_t r[32];
            const uint32_t taddr =
                tmem + ((uint32_t)lane_base << 16) + (uint32_t)(buf * kPairAccStride + half * PBNH + cc * 32);
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                  "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                  "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                  "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                  "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int j = 0; j < 32; ++j) sums[cc * 32 + j] += __uint_as_float(r[j]);
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) arrive_remote(to_rank(acc_empty(buf), 0));
        }
        if (F16) {
#pragma unroll
          for (int j = 0; j < PBNH; ++j) sums[j] *= fsc;
        }
        const int rr = lane >> 2, c4 = (lane & 3) * 4;
        // partial tile part[z][m][n] through the staging buffer (each warp store
        // covers 4 rows x 64 contiguous bytes)
#pragma unroll
        for (int cb = 0; cb < PBNH / 16; ++cb) {
#pragma unroll
          for (int qq = 0; qq < 4; ++qq)
            *reinterpret_cast<float4*>(stg + lane * SLD + 4 * qq) =
                make_float4(sums[cb * 16 + 4 * qq], sums[cb * 16 + 4 * qq + 1], sums[cb * 16 + 4 * qq + 2],
                            sums[cb * 16 + 4 * qq + 3]);
          __syncwarp();
          const int n = ncol0 + cb * 16 + c4;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int r = 8 * k + rr;
            const int m = mrow0 + r;
            const float4 v = *reinterpret_cast<const float4*>(stg + r * SLD + c4);
            if (m < S.B && n < N) *reinterpret_cast<float4*>(part + ((size_t)z * S.B + m) * N + n) = v;
          }
          __syncwarp();
        }
      }
    }
    if (trace && blockIdx.x == 0 && threadIdx.x == 128) trace[TR * si + 3] = gtimer();  // CTA 0's items stored
    if (DIR == 0 && S.pad != 0) continue;  // gates applied in the epilogues; the next step's items wait per row tile
    grid_sync(bar, target);  // all partials of step si written
    if (trace && blockIdx.x == 0 && threadIdx.x == 0) trace[TR * si + 4] = gtimer();
    gate_phase<DIR>(S, H, part, xp, h0, hidden, gates_out, hun_out, hprev_out, dhidden, gates, hun, hprev, dpre, dhu,
                    gz, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x, F16 ? h16hi : nullptr,
                    F16 ? h16lo : nullptr, hs);
    if (trace && blockIdx.x == 0 && threadIdx.x == 0) trace[TR * si + 5] = gtimer();
    if (si + 1 < nsteps) grid_sync(bar, target);  // step si's rows before step si+1's GEMM reads them
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(NACC2 * BN2) : "memory");
  }
}

// host: per-step split-K so that tilesM x tilesN x Z <= grid
static Step make_step(int B, int Bg, int o, int op, int N, int K, int grid, int bk = BK) {
  Step s{};
  s.B = B;
  s.Bg = Bg;
  s.o = o;
  s.op = op;
  s.tilesM = (int)cdiv(std::max(B, 1), BM);
  const int tilesN = (int)cdiv(N, BN);
  const int nkb = (K + bk - 1) / bk;
  int Z = std::max(1, std::min(grid / std::max(1, s.tilesM * tilesN), std::max(1, nkb / 2)));
  Z = std::min(Z, 8);
  const int per = (nkb + Z - 1) / Z;
  s.Z = (nkb + per - 1) / per;
  s.per = per;
  return s;
}

// pair mode: 256-row x BN-column tiles over the resident CTA pairs.  fuse (the
// forward with H % 32 == 0): a step whose split-K count comes out 1 runs with the
// gates in the GEMM epilogue (forcing Z = 1 on the smaller steps measured slower;
// force_fuse is for the sanitizer / small tests, which never reach Z = 1 naturally)
// (bk: K elements per stage -- 32 for tf32, 64 for the fp16x2 forward.)  Unfused
// steps take the split-K count with the least modelled time: rounds of items over
// the pairs x K-blocks per item (+2 of pipeline fill), plus the extra partial tiles
// the gate phase reads back (~0.00065 K-block times per row and extra split at
// H = 512; B200 step traces): e.g. 5,000 backward rows run Z = 3 (2 rounds of 16
// K-blocks) instead of Z = 1 (one round of 48 on 40 of the 74 pairs).
static Step make_step2(int B, int Bg, int o, int op, int N, int K, int pairs, int BN, bool fuse,
                       bool force_fuse = false, int bk = BK) {
  Step s{};
  s.B = B;
  s.Bg = Bg;
  s.o = o;
  s.op = op;
  s.tilesM = (int)cdiv(std::max(B, 1), p2::BM2);
  const int tilesN = (int)cdiv(N, BN);
  const int nkb = (K + bk - 1) / bk;
  const int items = s.tilesM * tilesN;
  int Z = std::max(1, std::min(pairs / std::max(1, items), std::max(1, nkb / 2)));
  Z = std::min(Z, 8);
  if (!fuse) {
    double best = 1e300;
    for (int z = 1; z <= std::min(8, std::max(1, nkb / 2)); ++z) {
      const double rounds = (double)cdiv((long long)items * z, std::max(1, pairs));
      const double cost = rounds * (double)(cdiv(nkb, z) + 2) + (z - 1) * (double)B * 0.00065;
      if (cost < best * 0.999) {
        best = cost;
        Z = z;
      }
    }
  }
  if (fuse && force_fuse) Z = 1;
  const int per = (nkb + Z - 1) / Z;
  s.Z = (nkb + per - 1) / per;
  s.per = per;
  s.pad = fuse && s.Z == 1 ? 1 : 0;
  return s;
}

// CTA pairs resident at once for the pair step kernel (all its CTAs must be, for
// the grid barriers), per device
template <int DIR, int F16 = 0>
static int step_pairs(Ctx* c) {
  static std::atomic<int> cache[kMaxDevices];
  int pairs = cache[dev_slot(c)].load();
  if (!pairs) {
    const void* fn = reinterpret_cast<const void*>(gru_step_gemm2_kernel<DIR, F16>);
    VER_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, PairCfg<F16>::SMEM));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(c->num_sms);
    cfg.blockDim = dim3(p2::THREADS2);
    cfg.dynamicSmemBytes = PairCfg<F16>::SMEM;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nc = 0;
    VER_CUDA(cudaOccupancyMaxActiveClusters(&nc, gru_step_gemm2_kernel<DIR, F16>, &cfg));
    pairs = std::max(1, std::min(nc, c->num_sms / 2));
    cache[dev_slot(c)].store(pairs);
  }
  return pairs;
}

template <int DIR>
static void launch(Ctx* c, const Model& m, const float* params, const std::vector<Step>& hs,
                   const std::vector<CUtensorMap>& maps, Workspace& ws, const float* h0, bool store,
                   bool pair = false, bool f16 = false) {
  const int nsteps = (int)hs.size();
  if (nsteps == 0) return;
  const int H = m.H, H3 = 3 * H;
  const int N = DIR == 0 ? H3 : H;
  size_t part_n = 0;
  for (const Step& s : hs) part_n = std::max(part_n, (size_t)s.Z * s.B * N);
  ws.step.reserve(c, std::max<size_t>(part_n, 4));
  ws.sgsteps.reserve(c, (size_t)nsteps * sizeof(Step) / 4 + 1);
  const size_t nmaps = maps.size();  // one per step (two with f16: hi, lo)
  ws.sgmaps.reserve(c, nmaps * sizeof(CUtensorMap) / 4 + 16);
  // 64-byte aligned tensor-map array inside the buffer
  uint8_t* mbase = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(ws.sgmaps.p) + 63) & ~uintptr_t(63));
  VER_CUDA(cudaMemcpyAsync(ws.sgsteps.p, hs.data(), sizeof(Step) * nsteps, cudaMemcpyHostToDevice, c->stream));
  VER_CUDA(cudaMemcpyAsync(mbase, maps.data(), sizeof(CUtensorMap) * nmaps, cudaMemcpyHostToDevice, c->stream));
  int rbs = 1;  // row tiles per step in the pair launch (step 0 has the most rows)
  for (const Step& st : hs) rbs = std::max(rbs, st.tilesM);
  const size_t nbar = pair ? 32 + (size_t)nsteps * rbs : 32;
  ws.bar.reserve(c, nbar);
  ws.bar.zero(nbar);
  const float* ux = params + m.o_ux;
  CUtensorMap bmap = DIR == 0 ? make_map(ux, H, H3, H3, 32, true) : make_map(ux, H, H3, H3, BN, false);
  // U's lo copy (made by the forward that precedes this launch, policy.cu)
  const float* ulo = (ws.wlo.n >= (size_t)m.P && env_int("VER_TC_BLO", 1)) ? ws.wlo.p + m.o_ux : nullptr;
  int blo = ulo != nullptr ? 1 : 0;
  CUtensorMap bmap_lo =
      !blo ? bmap : (DIR == 0 ? make_map(ulo, H, H3, H3, 32, true) : make_map(ulo, H, H3, H3, BN, false));
  const float* fscale = nullptr;
  if (f16) {  // U's transposed fp16x2 halves (policy.cu refresh_weights_f16 slot 2): 3H x H, K-major
    const size_t off = (size_t)H3 * m.E + (size_t)m.E * m.E;
    const int brows = pair ? PairTile<0>::BNH : BN;  // a CTA's B rows: its half of a pair tile, or a 128-column tile
    bmap = make_map16(ws.w16hi.p + off, H3, H, H, brows);
    bmap_lo = make_map16(ws.w16lo.p + off, H3, H, H, brows);
    blo = 1;
    fscale = ws.hsc.p;  // [s_h, 1 / (s_h s_U)] (gru_forward_big_persist)
  }
  const int grid = c->num_sms;
  const bool f16s = f16 && DIR == 0 && !pair;  // the single-CTA kernel's fp16x2 variant
  const void* fn = f16s ? reinterpret_cast<const void*>(gru_step_gemm_kernel<0, 1>)
                        : reinterpret_cast<const void*>(gru_step_gemm_kernel<DIR>);
  static std::atomic<bool> attr[kMaxDevices][3];  // per device: a function attribute is per device
  const int av = f16s ? 2 : DIR;
  if (!attr[dev_slot(c)][av].load()) {
    VER_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
    attr[dev_slot(c)][av].store(true);
  }
  int ns = nsteps;
  const Step* dsteps = reinterpret_cast<const Step*>(ws.sgsteps.p);
  const CUtensorMap* dmaps = reinterpret_cast<const CUtensorMap*>(mbase);
  float* part = ws.step.p;
  unsigned* bar = ws.bar.p;
  const float* xp = ws.xp.p;
  float* hidden = ws.hidden.p;
  float* gts = store ? ws.gates.p : nullptr;
  float* hun_o = ws.hu.p;
  float* hpv_o = ws.hprev.p;
  const float* dh = ws.dhidden.p;
  const float* gates = ws.gates.p;
  const float* hun = ws.hu.p;
  const float* hprev = ws.hprev.p;
  float* dpre = ws.dpre.p;
  float* dhu = ws.dhu.p;
  float* gz = ws.g.p;
  // VER_REC_TRACE (experiments): GEMM-phase start / gate-phase start of every step
  long long* tr = nullptr;
  const char* tpath = getenv("VER_REC_TRACE");
  if (tpath) {
    ws.trace.reserve(c, TR * (size_t)nsteps + 1);
    ws.trace.zero(TR * (size_t)nsteps + 1);
    tr = ws.trace.p;
  }
  if (pair) {
    const int pairs = (DIR == 0 && f16) ? step_pairs<0, 1>(c) : step_pairs<DIR>(c);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * pairs);
    cfg.blockDim = dim3(p2::THREADS2);
    cfg.dynamicSmemBytes = (DIR == 0 && f16) ? PairCfg<1>::SMEM : PairCfg<0>::SMEM;
    cfg.stream = c->stream;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative;  // every CTA resident: the grid barriers spin on each other
    at[1].val.cooperative = 1;
    cfg.attrs = at;
    // ncu cannot replay a cooperative cluster launch (LaunchFailed); it serializes
    // kernels, so a plain cluster launch of <= one CTA per SM is co-resident there
    cfg.numAttrs = profiling() ? 1 : 2;
    ScopedEv ev(c, c->rec_tag);
    __half* h16hi = ws.h16hi.p;
    __half* h16lo = ws.h16lo.p;
    if (f16 && DIR == 0)
      VER_CUDA(cudaLaunchKernelEx(&cfg, gru_step_gemm2_kernel<0, 1>, ns, dsteps, dmaps, bmap, H, part, bar, xp, h0,
                                  hidden, gts, hun_o, hpv_o, dh, gates, hun, hprev, dpre, dhu, gz, bmap_lo, blo, tr,
                                  rbs, h16hi, h16lo, fscale));
    else
      VER_CUDA(cudaLaunchKernelEx(&cfg, gru_step_gemm2_kernel<DIR>, ns, dsteps, dmaps, bmap, H, part, bar, xp, h0,
                                  hidden, gts, hun_o, hpv_o, dh, gates, hun, hprev, dpre, dhu, gz, bmap_lo, blo, tr,
                                  rbs, h16hi, h16lo, fscale));
    after_launch(c);
  } else {
    __half* sh16hi = ws.h16hi.p;
    __half* sh16lo = ws.h16lo.p;
    void* args[] = {&ns,    &dsteps, &dmaps,  const_cast<CUtensorMap*>(&bmap), const_cast<int*>(&H),
                    &part,  &bar,    &xp,     &h0,  &hidden, &gts, &hun_o, &hpv_o, &dh, &gates, &hun, &hprev, &dpre,
                    &dhu,   &gz,     &tr,     const_cast<CUtensorMap*>(&bmap_lo), &blo, &sh16hi, &sh16lo,
                    const_cast<const float**>(&fscale)};
    ScopedEv ev(c, c->rec_tag);
    VER_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(THREADS), args, SMEM_BYTES, c->stream));
    after_launch(c);
  }
  if (tr) {
    std::vector<long long> h(TR * (size_t)nsteps);
    VER_CUDA(cudaMemcpyAsync(h.data(), tr, sizeof(long long) * h.size(), cudaMemcpyDeviceToHost, c->stream));
    VER_CUDA(cudaStreamSynchronize(c->stream));
    // per step: rows, Z, then each slot and the next step's start relative to this step's start (ns)
    if (FILE* f = fopen(tpath, "a")) {
      fprintf(f, "%s%d %d", pair ? "pair" : "persist", DIR, nsteps);
      for (int i = 0; i < nsteps; ++i) {
        const long long t0 = h[TR * i];
        fprintf(f, " %d:%d", hs[i].Bg, hs[i].Z);
        for (int k = 1; k < TR; ++k) fprintf(f, ":%lld", h[TR * i + k] ? h[TR * i + k] - t0 : -1);
        fprintf(f, ":%lld", i + 1 < nsteps ? h[TR * (i + 1)] - t0 : -1);
      }
      fprintf(f, "\n");
      fclose(f);
    }
  }
}

}  // namespace sg


// rows from which a big step runs in the CTA-pair kernel (0: never)
static int pair_rows(const Ctx* c) { return c->precision == 0 ? env_int("VER_REC_PAIR_ROWS", 1024) : 0; }

// forward big steps t = 0 .. t_end-1: the steps with >= pair_rows rows in the
// CTA-pair launch, the rest in the single-CTA launch
void gru_forward_big_persist(Ctx* c, const Model& m, const float* params, int t_end, const int32_t* h_bs,
                             const int32_t* h_offs, Workspace& ws, const float* h0, bool store) {
  const int H = m.H, H3 = 3 * H;
  const int pr = pair_rows(c);
  int t1 = 0;
  if (pr > 0)
    while (t1 < t_end && h_bs[t1] >= pr) ++t1;
  if (t_end <= 0) return;
  // fp16x2 GEMM phase (pair and single-CTA steps) when this forward's weight halves
  // are fresh (policy_forward) and H fits 64-element K blocks: h halves for the rows
  // of every big step (packed offsets), h0's after them, h's scale from max |h0|
  const bool f16 = ws.f16_fwd && H % 64 == 0;
  const size_t rows = (size_t)h_offs[t_end - 1] + h_bs[t_end - 1];
  if (f16) {
    // (sized by the workspace rows: no regrowth from one minibatch to the next)
    const size_t need = std::max(rows + (size_t)h_bs[0], 2 * ws.rows) * H;
    ws.h16hi.reserve(c, need);
    ws.h16lo.reserve(c, need);
    const size_t n0 = (size_t)h_bs[0] * H;
    ws.hmax.reserve(c, 1);
    ws.hsc.reserve(c, 2);
    ws.hmax.zero(1);
    maxabs_kernel<<<(unsigned)std::min<size_t>(cdiv(n0, 256), 2 * c->num_sms), 256, 0, c->stream>>>(
        (int64_t)n0, h0, ws.hmax.p);
    after_launch(c);
    sg::hscale_kernel<<<1, 1, 0, c->stream>>>(ws.hmax.p, ws.w16inv.p + 2, ws.hsc.p);
    after_launch(c);
    sg::h16_kernel<<<(unsigned)std::min<size_t>(cdiv(n0, 256), 4 * c->num_sms), 256, 0, c->stream>>>(
        (int64_t)n0, h0, ws.hsc.p, ws.h16hi.p + rows * H, ws.h16lo.p + rows * H);
    after_launch(c);
  }
  for (int part = 0; part < 2; ++part) {
    const int ta = part == 0 ? 0 : t1, tz = part == 0 ? t1 : t_end;
    if (ta >= tz) continue;
    std::vector<sg::Step> hs;
    std::vector<CUtensorMap> maps;
    const int pairs = part == 0 ? (f16 ? sg::step_pairs<0, 1>(c) : sg::step_pairs<0>(c)) : 0;
    const bool fuse = H % 32 == 0;
    const bool force_fuse = env_int("VER_REC_FUSE_ALL", 0) != 0;  // tests / sanitizer
    for (int t = ta; t < tz; ++t) {
      const int B = h_bs[t];
      const int op = t == 0 ? -1 : h_offs[t - 1];
      hs.push_back(part == 0 ? sg::make_step2(B, B, h_offs[t], op, H3, H, pairs, sg::PairTile<0>::BN, fuse,
                                              force_fuse, f16 ? 64 : tc::BK)
                             : sg::make_step(B, B, h_offs[t], op, H3, H, c->num_sms, f16 ? 64 : tc::BK));
      if (f16) {
        const size_t r0 = t == 0 ? rows : (size_t)h_offs[t - 1];
        maps.push_back(tc::make_map16(ws.h16hi.p + r0 * H, B, H, H, tc::BM));
        maps.push_back(tc::make_map16(ws.h16lo.p + r0 * H, B, H, H, tc::BM));
      } else {
        const float* hp = t == 0 ? h0 : ws.hidden.p + (size_t)h_offs[t - 1] * H;
        maps.push_back(tc::make_map(hp, B, H, H, tc::BM, false));
      }
    }
    sg::launch<0>(c, m, params, hs, maps, ws, h0, store, part == 0, f16);
  }
}

// backward big steps t = t_top .. 1: the single-CTA launch for the steps with
// fewer than pair_rows rows first, then the CTA-pair launch
void gru_backward_big_persist(Ctx* c, const Model& m, const float* params, int t_top, const int32_t* h_bs,
                              const int32_t* h_offs, Workspace& ws) {
  const int H = m.H, H3 = 3 * H;
  const int pr = pair_rows(c);
  int t1 = 0;  // steps 1 .. t1 have >= pr rows
  if (pr > 0)
    while (t1 + 1 <= t_top && h_bs[t1 + 1] >= pr) ++t1;
  for (int part = 0; part < 2; ++part) {
    const int hi = part == 0 ? t_top : t1, lo = part == 0 ? t1 + 1 : 1;
    if (hi < lo) continue;
    std::vector<sg::Step> hs;
    std::vector<CUtensorMap> maps;
    const int pairs = part == 1 ? sg::step_pairs<1>(c) : 0;
    for (int t = hi; t >= lo; --t) {
      const int B = h_bs[t], Bp = h_bs[t - 1];
      hs.push_back(part == 1 ? sg::make_step2(B, Bp, h_offs[t], h_offs[t - 1], H, H3, pairs, sg::PairTile<1>::BN, false)
                             : sg::make_step(B, Bp, h_offs[t], h_offs[t - 1], H, H3, c->num_sms));
      maps.push_back(tc::make_map(ws.dhu.p + (size_t)h_offs[t] * H3, std::max(B, 1), H3, H3, tc::BM, false));
    }
    sg::launch<1>(c, m, params, hs, maps, ws, nullptr, false, part == 1);
  }
}

}  // namespace verg
