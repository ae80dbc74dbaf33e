// stepfused.cu — the big recurrence timesteps as one persistent kernel of
// 4-CTA clusters, with the split-K reduction and the gate math fused into the
// GEMM epilogue: ONE grid barrier per step.
//
//   forward  step t: hU = h_{t-1}[0:B] U   (M = B, N = 3H, K = H), then the GRU
//                    gates of rows j < B (nn.cpp:235-250);
//   backward step t: dh = dhU_t[0:B] U^T   (M = B, N = H, K = 3H), then the gate
//                    gradient of the rows j < B_{t-1} of step t-1.
//
// Against stepgemm.cu (split-K partials through L2, a grid-wide gate phase and
// two grid barriers per step):
// * output tile = 128 rows x BN columns, owned by one cluster of CZ = 4 CTAs;
//   CTA rank z multiplies K-slice z (3xTF32 tcgen05, accumulator in TMEM);
// * reduction over distributed shared memory: epilogue warp q of every CTA
//   holds TMEM lanes 32q..32q+31 (rows) and pushes them into CTA q's reduce
//   buffer (st.shared::cluster, slot = sender rank), then arrives on CTA q's
//   mbarrier; CTA q sums its 4 slots in rank order (deterministic) for its
//   32 rows;
// * the gate math runs right there on the reduced 32 x BN block.  The forward
//   tile is BN = 96 columns = 32 units x (r, z, n) (U's columns are unit-major
//   interleaved, 3u + g), the backward tile BN = 64 units;
// * the gate operands that do not depend on the GEMM (xp, h_{t-1}; the saved
//   gates, hUn, h_prev, dhidden, the carried dh) are loaded before waiting for
//   the reduction.
// Warp roles as in the tcgen05 GEMM (tc_gemm.cuh): TMA producer, MMA issuer,
// 4 split warps (lo = x - trunc_tf32(x)), 4 epilogue warps.  All counters and
// mbarrier phases run on across tiles and steps.
#include <cstdlib>

#include "policy.cuh"
#include "tc_gemm.cuh"

namespace verg {
namespace sf {

using namespace tc;

constexpr int CZ = 4;        // CTAs per cluster = K slices per output tile
constexpr int RS = BM / CZ;  // rows per CTA in the reduction = one epilogue warp's TMEM lanes
constexpr int FST = 4;       // smem ring stages (A hi | B hi | B lo; A hi / lo go on to TMEM)
static_assert(RS == 32, "one epilogue warp per reduction slice");

template <int DIR>
struct Cfg {
  static constexpr int BN = DIR == 0 ? 96 : 64;  // forward: 32 units x (r, z, n); backward: 64 units
  static constexpr int BT = BN * BK * 4;          // B tile bytes
  static constexpr int STAGE = TILE_BYTES + 2 * BT;
  static constexpr int RLD = BN + 4;  // reduce-buffer row stride (floats): float4 pushes conflict-free
  static constexpr int RB = CZ * RS * RLD * 4;
  static constexpr int NACC = DIR == 0 ? 2 : 4;
  static constexpr int ACOL = DIR == 0 ? 128 : 64;  // TMEM column stride of the accumulator buffers
  static constexpr int TCOLS = 512;
  static constexpr int A_COL0 = NACC * ACOL;  // stage s: A hi at A_COL0 + 64 s, A lo at + 32
  static constexpr int PUSH = CZ * RS * BN * 4;  // bytes received per pass
  static constexpr int NBAR = 3 * FST + 2 * NACC + 1 + CZ;
  static constexpr int SMEM = FST * STAGE + RB + 1024 /*align*/ + 8 * NBAR + 16;
  static_assert(A_COL0 + FST * 64 <= TCOLS, "TMEM budget");
  static_assert(STAGE % 1024 == 0 && BT % 1024 == 0, "1024-byte aligned operand tiles");
};
static_assert(Cfg<0>::SMEM <= 232448 && Cfg<1>::SMEM <= 232448, "shared memory budget");

struct Step {
  int B;       // GEMM rows (forward: bs_t; backward: bs_t, rows with a successor)
  int Bg;      // gate rows (forward: bs_t; backward: bs_{t-1})
  int o, op;   // packed offsets of the GEMM / gate rows (forward: op = offs_{t-1} or -1 for h0)
  int tilesM;  // 128-row tiles covering max(B, Bg)
  int pad[3];
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t cta) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(cta));
  return r;
}
// async store into a peer CTA's shared memory; completes `bytes` on the peer's mbarrier
__device__ __forceinline__ void st_async4(uint32_t a, float4 v, uint32_t mbar_cluster) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(a),
               "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(mbar_cluster)
               : "memory");
}
__device__ __forceinline__ void arrive_remote(uint32_t a_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(a_cluster) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t a, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "LAB_WAITC:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra LAB_WAITC;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void grid_sync(unsigned* count, unsigned& target) {
  __syncthreads();
  target += gridDim.x;
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(count) : "memory");
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(count) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

// VER_REC_TRACE slots per step (CTA 0, first tile): start, stage 0 landed,
// accumulator ready, pushed, reduction received, gate done
constexpr int TRF = 6;
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void st4(float* p, float a, float b, float c, float d) {
  *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d);
}

template <int DIR>  // 0 forward (B MN-major: U stored K x N), 1 backward (B K-major: U stored N x K)
__global__ void __launch_bounds__(THREADS, 1) gru_step_fused_kernel(
    int nsteps, const Step* __restrict__ steps, const CUtensorMap* __restrict__ amaps,
    const __grid_constant__ CUtensorMap bmap, int H, unsigned* bar,
    // forward
    const float* __restrict__ xp, const float* __restrict__ h0, float* __restrict__ hidden,
    float* __restrict__ gates_out, float* __restrict__ hun_out, float* __restrict__ hprev_out,
    // backward
    const float* __restrict__ dhidden, const float* __restrict__ gates, const float* __restrict__ hun,
    const float* __restrict__ hprev, float* __restrict__ dpre, float* __restrict__ dhu, float* __restrict__ gz,
    long long* trace) {
  using C = Cfg<DIR>;
  constexpr int BN = C::BN, AMAJ = 0, BMAJ = DIR == 0 ? 1 : 0;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* rbuf = reinterpret_cast<float*>(smem + FST * C::STAGE);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + FST * C::STAGE + C::RB);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NBAR);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int cl = blockIdx.x / CZ, ncl = gridDim.x / CZ;
  const int H3 = 3 * H, N = DIR == 0 ? H3 : H, K = DIR == 0 ? H : H3;
  const int tilesN = N / BN;
  const int per = K / BK / CZ;  // K-blocks per CTA (the host checks divisibility)
  const int kb0 = (int)rank * per;
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar0 = smem_u32(bars);
  auto full_bar = [&](int s) { return bar0 + 8 * s; };
  auto split_bar = [&](int s) { return bar0 + 8 * (FST + s); };
  auto empty_bar = [&](int s) { return bar0 + 8 * (2 * FST + s); };
  auto acc_full = [&](int b) { return bar0 + 8 * (3 * FST + b); };
  auto acc_empty = [&](int b) { return bar0 + 8 * (3 * FST + C::NACC + b); };
  const uint32_t recv_full = bar0 + 8 * (3 * FST + 2 * C::NACC);
  auto free_bar = [&](int q) { return bar0 + 8 * (3 * FST + 2 * C::NACC + 1 + q); };
  auto a_tile = [&](int s) { return sbase + s * C::STAGE; };
  auto b_tile = [&](int s, int lo) { return sbase + s * C::STAGE + TILE_BYTES + lo * C::BT; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < FST; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(split_bar(s), SPLIT_WARPS);
      mbar_init(empty_bar(s), 1);
    }
    for (int b = 0; b < C::NACC; ++b) {
      mbar_init(acc_full(b), 1);
      mbar_init(acc_empty(b), EPI_WARPS);
    }
    mbar_init(recv_full, 1);  // the owner's expect_tx; the peers' st.async complete the bytes
    for (int q = 0; q < CZ; ++q) mbar_init(free_bar(q), EPI_WARPS);  // CTA q's gate warps done reading
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(recv_full, C::PUSH);  // pass 0
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&bmap)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(C::TCOLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // every CTA's barriers initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  unsigned target = 0;
  int it_tma = 0, it_mma = 0, it_split = 0, g_mma = 0, g_epi = 0, np = 0;

  for (int si = 0; si < nsteps; ++si) {
    if (trace && blockIdx.x == 0 && threadIdx.x == 0) trace[TRF * si] = gtimer();
    const Step S = steps[si];
    const int ntiles = S.tilesM * tilesN;
    const CUtensorMap* amap = amaps + si;
    if (warp == 0) {
      if (lane == 0) {
        asm volatile("fence.proxy.async.global;" ::: "memory");  // h / dhU rows written by last step's gates
        for (int tile = cl; tile < ntiles; tile += ncl) {
          const int m0 = (tile / tilesN) * BM, n0 = (tile % tilesN) * BN;
          for (int i = 0; i < per; ++i, ++it_tma) {
            const int s = it_tma % FST;
            mbar_wait(empty_bar(s), ((it_tma / FST) & 1) ^ 1);
            mbar_expect_tx(full_bar(s), TILE_BYTES + C::BT);
            const int k0 = (kb0 + i) * BK;
            tma_load_2d(a_tile(s), amap, full_bar(s), k0, m0);
            if (BMAJ == 0) {
              tma_load_2d(b_tile(s, 0), &bmap, full_bar(s), k0, n0);
            } else {
#pragma unroll
              for (int c = 0; c < BN / 32; ++c) tma_load_2d(b_tile(s, 0) + c * 4096, &bmap, full_bar(s), n0 + 32 * c, k0);
            }
          }
        }
      }
    } else if (warp == 1) {
      constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)AMAJ << 15) |
                                 ((uint32_t)BMAJ << 16) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
      if (lane == 0) {
        for (int tile = cl; tile < ntiles; tile += ncl, ++g_mma) {
          const int buf = g_mma % C::NACC;
          if (g_mma >= C::NACC) mbar_wait(acc_empty(buf), ((g_mma / C::NACC) - 1) & 1);
          tc_fence_after();
          const uint32_t d = tmem + (uint32_t)(buf * C::ACOL);
          for (int i = 0; i < per; ++i, ++it_mma) {
            const int s = it_mma % FST;
            mbar_wait(split_bar(s), (it_mma / FST) & 1);
            tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk) {
              const uint32_t ah = tmem + (uint32_t)(C::A_COL0 + 64 * s + 8 * kk);
              const uint64_t bh = operand_desc<BMAJ>(b_tile(s, 0), kk);
              mma_tf32_ts(d, ah, bh, idesc, (i > 0 || kk > 0) ? 1u : 0u);
              mma_tf32_ts(d, ah + 32, bh, idesc, 1u);
              mma_tf32_ts(d, ah, operand_desc<BMAJ>(b_tile(s, 1), kk), idesc, 1u);
            }
            umma_commit(empty_bar(s));
          }
          umma_commit(acc_full(buf));
        }
      }
      __syncwarp();
    } else if (warp < 2 + SPLIT_WARPS) {
      const int et = threadIdx.x - 64;
      for (int tile = cl; tile < ntiles; tile += ncl) {
        for (int i = 0; i < per; ++i, ++it_split) {
          const int s = it_split % FST;
          mbar_wait(full_bar(s), (it_split / FST) & 1);
          if (trace && i == 0 && tile == cl && threadIdx.x == 64 && blockIdx.x == 0) trace[TRF * si + 1] = gtimer();
          uint8_t* st = smem + s * C::STAGE;
          // A row r = this thread's TMEM lane: 32 K values from the SW128 K-major tile
          // (16-byte chunk c of row r sits at chunk c ^ (r % 8)) -> hi / lo columns
          const int ar = 32 * (warp & 3) + lane;
          const uint8_t* rowp = st + (ar >> 3) * 1024 + (ar & 7) * 128;
          uint32_t hv[32], lv[32];
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float4 x = *reinterpret_cast<const float4*>(rowp + ((c ^ (ar & 7)) << 4));
            const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const uint32_t hb = __float_as_uint(xs[j]) & 0xffffe000u;
              hv[4 * c + j] = hb;
              lv[4 * c + j] = __float_as_uint(xs[j] - __uint_as_float(hb));
            }
          }
          const uint32_t ta = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(C::A_COL0 + 64 * s);
          tmem_st32(ta, hv);
          tmem_st32(ta + 32, lv);
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          const float4* bhi = reinterpret_cast<const float4*>(st + TILE_BYTES);
          float4* blo = reinterpret_cast<float4*>(st + TILE_BYTES + C::BT);
#pragma unroll 3
          for (int qq = et; qq < C::BT / 16; qq += 32 * SPLIT_WARPS) blo[qq] = lo_tf32(bhi[qq]);
          tc_fence_before();
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(split_bar(s));
        }
      }
    } else {
      // epilogue: drain + push to the slice owner, then the gate of this CTA's slice
      const int q = warp & 3;           // TMEM lanes 32q.. = tile rows 32q.. -> owned by cluster CTA q
      const int e = threadIdx.x - 192;  // gate thread 0..127
      const int r = e >> 2;             // row of this CTA's 32-row slice
      const uint32_t push_base = mapa(smem_u32(rbuf + ((int)rank * RS + lane) * C::RLD), (uint32_t)q);
      const uint32_t push_bar = mapa(recv_full, (uint32_t)q);
      for (int tile = cl; tile < ntiles; tile += ncl, ++g_epi, ++np) {
        const int mt = tile / tilesN, nt = tile % tilesN;
        const int buf = g_epi % C::NACC;
        mbar_wait(acc_full(buf), (g_epi / C::NACC) & 1);
        tc_fence_after();
        const bool tr0 = trace && tile == cl && threadIdx.x == 192 && blockIdx.x == 0;
        if (tr0) trace[TRF * si + 2] = gtimer();
        mbar_wait_cluster(free_bar(q), (np & 1) ^ 1);  // CTA q has read the previous pass
#pragma unroll
        for (int cc = 0; cc < BN / 32; ++cc) {
          uint32_t v[32];
          const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(buf * C::ACOL + cc * 32);
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
              "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
              : "r"(taddr));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int k = 0; k < 8; ++k)
            st_async4(push_base + (uint32_t)((cc * 32 + 4 * k) * 4),
                      make_float4(__uint_as_float(v[4 * k]), __uint_as_float(v[4 * k + 1]),
                                  __uint_as_float(v[4 * k + 2]), __uint_as_float(v[4 * k + 3])),
                      push_bar);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(acc_empty(buf));
        if (tr0) trace[TRF * si + 3] = gtimer();

        // ---- gate of rows m0 + 32 rank + r of this tile
        const int m = mt * BM + (int)rank * RS + r;
        const float* rrow = rbuf + r * C::RLD;
        if (DIR == 0) {
          // units 32 nt + 8 (e & 3) .. + 8; columns 24 (e & 3) .. + 24 of the tile
          const int cu = 24 * (e & 3), u0 = 32 * nt + 8 * (e & 3);
          const bool ok = m < S.B;
          float x[24], hp[8];
          if (ok) {
            const float* xr = xp + ((size_t)S.o + m) * H3 + 3 * u0;
#pragma unroll
            for (int k = 0; k < 6; ++k) {
              const float4 t = ld4(xr + 4 * k);
              x[4 * k] = t.x; x[4 * k + 1] = t.y; x[4 * k + 2] = t.z; x[4 * k + 3] = t.w;
            }
            const float* hr = (S.op < 0 ? h0 + (size_t)m * H : hidden + ((size_t)S.op + m) * H) + u0;
            const float4 a = ld4(hr), b = ld4(hr + 4);
            hp[0] = a.x; hp[1] = a.y; hp[2] = a.z; hp[3] = a.w; hp[4] = b.x; hp[5] = b.y; hp[6] = b.z; hp[7] = b.w;
          }
          mbar_wait_cluster(recv_full, np & 1);
          if (e == 0) mbar_expect_tx(recv_full, C::PUSH);  // next pass (its senders wait for our free arrivals)
          if (tr0) trace[TRF * si + 4] = gtimer();
          float s24[24];
#pragma unroll
          for (int k = 0; k < 24; ++k) s24[k] = 0.f;
#pragma unroll
          for (int z = 0; z < CZ; ++z) {
            const float* p = rrow + z * RS * C::RLD + cu;
#pragma unroll
            for (int k = 0; k < 6; ++k) {
              const float4 t = ld4(p + 4 * k);
              s24[4 * k] += t.x; s24[4 * k + 1] += t.y; s24[4 * k + 2] += t.z; s24[4 * k + 3] += t.w;
            }
          }
          if (ok) {
            float hn[8], g[24];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const float rg = gate_sigm(x[3 * u] + s24[3 * u]);
              const float zg = gate_sigm(x[3 * u + 1] + s24[3 * u + 1]);
              const float ng = gate_tanh(x[3 * u + 2] + rg * s24[3 * u + 2]);
              hn[u] = (1.f - zg) * ng + zg * hp[u];
              g[3 * u] = rg;
              g[3 * u + 1] = zg;
              g[3 * u + 2] = ng;
            }
            const size_t row = ((size_t)S.o + m) * H + u0, row3 = ((size_t)S.o + m) * H3 + 3 * u0;
            st4(hidden + row, hn[0], hn[1], hn[2], hn[3]);
            st4(hidden + row + 4, hn[4], hn[5], hn[6], hn[7]);
            if (gates_out) {
#pragma unroll
              for (int k = 0; k < 6; ++k) st4(gates_out + row3 + 4 * k, g[4 * k], g[4 * k + 1], g[4 * k + 2], g[4 * k + 3]);
              st4(hun_out + row, s24[2], s24[5], s24[8], s24[11]);
              st4(hun_out + row + 4, s24[14], s24[17], s24[20], s24[23]);
              st4(hprev_out + row, hp[0], hp[1], hp[2], hp[3]);
              st4(hprev_out + row + 4, hp[4], hp[5], hp[6], hp[7]);
            }
          }
        } else {
          // units 64 nt + 32 h + 8 (e & 3) .. + 8 for h = 0, 1
          const bool ok = m < S.Bg, carry = m < S.B;
          bool waited = false;
#pragma unroll 1
          for (int h = 0; h < 2; ++h) {
            const int cu = 32 * h + 8 * (e & 3), u0 = 64 * nt + cu;
            float d[8], hn[8], hp[8], gt[24], gc[8];
            if (ok) {
              const size_t row = ((size_t)S.op + m) * H + u0, row3 = ((size_t)S.op + m) * H3 + 3 * u0;
#pragma unroll
              for (int k = 0; k < 2; ++k) {
                const float4 a = ld4(dhidden + row + 4 * k), b = ld4(hun + row + 4 * k), c = ld4(hprev + row + 4 * k);
                d[4 * k] = a.x; d[4 * k + 1] = a.y; d[4 * k + 2] = a.z; d[4 * k + 3] = a.w;
                hn[4 * k] = b.x; hn[4 * k + 1] = b.y; hn[4 * k + 2] = b.z; hn[4 * k + 3] = b.w;
                hp[4 * k] = c.x; hp[4 * k + 1] = c.y; hp[4 * k + 2] = c.z; hp[4 * k + 3] = c.w;
              }
#pragma unroll
              for (int k = 0; k < 6; ++k) {
                const float4 t = ld4(gates + row3 + 4 * k);
                gt[4 * k] = t.x; gt[4 * k + 1] = t.y; gt[4 * k + 2] = t.z; gt[4 * k + 3] = t.w;
              }
#pragma unroll
              for (int k = 0; k < 8; ++k) gc[k] = 0.f;
              if (carry) {
                const float* gr = gz + ((size_t)S.o + m) * H + u0;
                const float4 a = ld4(gr), b = ld4(gr + 4);
                gc[0] = a.x; gc[1] = a.y; gc[2] = a.z; gc[3] = a.w; gc[4] = b.x; gc[5] = b.y; gc[6] = b.z; gc[7] = b.w;
              }
            }
            if (!waited) {
              mbar_wait_cluster(recv_full, np & 1);
              if (e == 0) mbar_expect_tx(recv_full, C::PUSH);
              if (tr0) trace[TRF * si + 4] = gtimer();
              waited = true;
            }
            float dh[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) dh[k] = 0.f;
#pragma unroll
            for (int z = 0; z < CZ; ++z) {
              const float* p = rrow + z * RS * C::RLD + cu;
              const float4 a = ld4(p), b = ld4(p + 4);
              dh[0] += a.x; dh[1] += a.y; dh[2] += a.z; dh[3] += a.w;
              dh[4] += b.x; dh[5] += b.y; dh[6] += b.z; dh[7] += b.w;
            }
            if (ok) {
              float o1[24], o2[24], gzv[8];
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const float gg = d[u] + (dh[u] + gc[u]);
                const float rr = gt[3 * u], zg = gt[3 * u + 1], n = gt[3 * u + 2];
                const float dn = gg * (1.f - zg);
                const float dz = gg * (hp[u] - n);
                const float dpn = dn * (1.f - n * n);
                const float dr = dpn * hn[u];
                const float dpr = dr * rr * (1.f - rr);
                const float dpz = dz * zg * (1.f - zg);
                o1[3 * u] = dpr;
                o1[3 * u + 1] = dpz;
                o1[3 * u + 2] = dpn;
                o2[3 * u] = dpr;
                o2[3 * u + 1] = dpz;
                o2[3 * u + 2] = dpn * rr;
                gzv[u] = gg * zg;
              }
              const size_t row = ((size_t)S.op + m) * H + u0, row3 = ((size_t)S.op + m) * H3 + 3 * u0;
#pragma unroll
              for (int k = 0; k < 6; ++k) {
                st4(dpre + row3 + 4 * k, o1[4 * k], o1[4 * k + 1], o1[4 * k + 2], o1[4 * k + 3]);
                st4(dhu + row3 + 4 * k, o2[4 * k], o2[4 * k + 1], o2[4 * k + 2], o2[4 * k + 3]);
              }
              st4(gz + row, gzv[0], gzv[1], gzv[2], gzv[3]);
              st4(gz + row + 4, gzv[4], gzv[5], gzv[6], gzv[7]);
            }
          }
        }
        __syncwarp();
        if (tr0) trace[TRF * si + 5] = gtimer();
        if (trace && threadIdx.x == 192) trace[TRF * nsteps + (size_t)si * gridDim.x + blockIdx.x] = gtimer();
        if (lane == 0) {
#pragma unroll
          for (int z = 0; z < CZ; ++z) arrive_remote(mapa(free_bar((int)rank), (uint32_t)z));
        }
      }
    }
    if (si + 1 < nsteps) grid_sync(bar, target);  // step si's rows before step si+1's GEMM reads them
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // no CTA leaves while a peer may still push to it or arrive on its barriers
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TCOLS) : "memory");
  }
}

template <int DIR>
static int max_clusters(Ctx* c) {
  static int ncl[2] = {-1, -1};
  if (ncl[DIR] < 0) {
    const void* fn = reinterpret_cast<const void*>(gru_step_fused_kernel<DIR>);
    VER_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<DIR>::SMEM));
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CZ;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(CZ * (c->num_sms / CZ));
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = Cfg<DIR>::SMEM;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    VER_CUDA(cudaOccupancyMaxActiveClusters(&n, fn, &cfg));
    ncl[DIR] = std::min(n, c->num_sms / CZ);
  }
  return ncl[DIR];
}

template <int DIR>
static void launch(Ctx* c, const Model& m, const float* params, const std::vector<Step>& hs,
                   const std::vector<CUtensorMap>& maps, Workspace& ws, const float* h0, bool store) {
  const int nsteps = (int)hs.size();
  if (nsteps == 0) return;
  const int H = m.H, H3 = 3 * H;
  ws.sgsteps.reserve(c, (size_t)nsteps * sizeof(Step) / 4 + 1);
  ws.sgmaps.reserve(c, (size_t)nsteps * sizeof(CUtensorMap) / 4 + 16);
  uint8_t* mbase = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(ws.sgmaps.p) + 63) & ~uintptr_t(63));
  VER_CUDA(cudaMemcpyAsync(ws.sgsteps.p, hs.data(), sizeof(Step) * nsteps, cudaMemcpyHostToDevice, c->stream));
  VER_CUDA(cudaMemcpyAsync(mbase, maps.data(), sizeof(CUtensorMap) * nsteps, cudaMemcpyHostToDevice, c->stream));
  ws.bar.reserve(c, 32);
  ws.bar.zero(32);
  const float* ux = params + m.o_ux;
  const CUtensorMap bmap = DIR == 0 ? make_map(ux, H, H3, H3, 32, true) : make_map(ux, H, H3, H3, Cfg<1>::BN, false);
  const int ncl = max_clusters<DIR>(c);
  if (ncl < 1) throw Error(VER_ERR_CUDA, "step kernel: no co-resident 4-CTA cluster");
  int ns = nsteps;
  const Step* dsteps = reinterpret_cast<const Step*>(ws.sgsteps.p);
  const CUtensorMap* dmaps = reinterpret_cast<const CUtensorMap*>(mbase);
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
  long long* tr = nullptr;
  const char* tpath = getenv("VER_REC_TRACE");
  if (tpath) {
    ws.trace.reserve(c, (TRF + CZ * (size_t)ncl) * nsteps + 1);
    ws.trace.zero((TRF + CZ * (size_t)ncl) * nsteps + 1);
    tr = ws.trace.p;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CZ;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(CZ * ncl);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = Cfg<DIR>::SMEM;
  cfg.stream = c->stream;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  // the grid barrier needs all CTAs resident: one CTA per SM (shared memory), at most
  // cudaOccupancyMaxActiveClusters clusters; CTAs of other streams' kernels only delay it
  {
    ScopedEv ev(c, c->rec_tag);
    VER_CUDA(cudaLaunchKernelEx(&cfg, gru_step_fused_kernel<DIR>, ns, dsteps, dmaps, bmap, H, bar, xp, h0, hidden,
                                gts, hun_o, hpv_o, dh, gates, hun, hprev, dpre, dhu, gz, tr));
    after_launch(c);
  }
  if (tr) {
    std::vector<long long> h((TRF + CZ * (size_t)ncl) * nsteps);
    VER_CUDA(cudaMemcpyAsync(h.data(), tr, sizeof(long long) * h.size(), cudaMemcpyDeviceToHost, c->stream));
    VER_CUDA(cudaStreamSynchronize(c->stream));
    // same format as stepgemm.cu's trace (scripts/step_trace.py), Z = clusters
    if (FILE* f = fopen(tpath, "a")) {
      fprintf(f, "fused%d %d", DIR, nsteps);
      for (int i = 0; i < nsteps; ++i) {
        const long long t0 = h[TRF * i];
        fprintf(f, " %d:%d", hs[i].Bg, ncl);
        for (int k = 1; k < TRF; ++k) fprintf(f, ":%lld", h[TRF * i + k] ? h[TRF * i + k] - t0 : -1);
        fprintf(f, ":%lld", i + 1 < nsteps ? h[TRF * (i + 1)] - t0 : -1);
      }
      fprintf(f, "\n");
      // per step: rows, then every CTA's last gate-done time after the step start (ns)
      for (int i = 0; i < nsteps; ++i) {
        fprintf(f, "ctas%d %d", DIR, hs[i].Bg);
        for (int b = 0; b < CZ * ncl; ++b) {
          const long long v = h[TRF * nsteps + (size_t)i * CZ * ncl + b];
          fprintf(f, " %lld", v ? v - h[TRF * i] : -1);
        }
        fprintf(f, "\n");
      }
      fclose(f);
    }
  }
}

}  // namespace sf

// Opt-in (VER_REC_PERSIST=2; backward also VER_REC_FUSED_BWD=1).  Correct, but
// measured slower than stepgemm.cu at C2: forward recurrence 9.9 against 8.9 ms
// per update.  Its 4-CTA clusters finish a step 2-3 us apart (per-CTA trace), a
// 4-way K split leaves each CTA 4 (forward) / 12 (backward) K-blocks of 3xTF32
// MMAs at ~0.7 us each, and only 33 clusters are co-resident (132 of 148 SMs).
// H = 256 / 512: the tile shapes need 3H % 96 == 0, H % 64 == 0 and K-blocks divisible by 4.
bool step_fused_ok(int H, bool backward) {
  return env_int("VER_REC_PERSIST", 1) == 2 && (H == 256 || H == 512) && (!backward || env_int("VER_REC_FUSED_BWD", 0));
}

void gru_forward_big_fused(Ctx* c, const Model& m, const float* params, int t_end, const int32_t* h_bs,
                           const int32_t* h_offs, Workspace& ws, const float* h0, bool store) {
  const int H = m.H;
  std::vector<sf::Step> hs;
  std::vector<CUtensorMap> maps;
  for (int t = 0; t < t_end; ++t) {
    const int B = h_bs[t];
    sf::Step s{};
    s.B = s.Bg = B;
    s.o = h_offs[t];
    s.op = t == 0 ? -1 : h_offs[t - 1];
    s.tilesM = (int)cdiv(std::max(B, 1), tc::BM);
    hs.push_back(s);
    const float* hp = t == 0 ? h0 : ws.hidden.p + (size_t)h_offs[t - 1] * H;
    maps.push_back(tc::make_map(hp, std::max(B, 1), H, H, tc::BM, false));
  }
  sf::launch<0>(c, m, params, hs, maps, ws, h0, store);
}

void gru_backward_big_fused(Ctx* c, const Model& m, const float* params, int t_top, const int32_t* h_bs,
                            const int32_t* h_offs, Workspace& ws) {
  const int H = m.H, H3 = 3 * H;
  std::vector<sf::Step> hs;
  std::vector<CUtensorMap> maps;
  for (int t = t_top; t >= 1; --t) {
    const int B = h_bs[t], Bp = h_bs[t - 1];
    sf::Step s{};
    s.B = B;
    s.Bg = Bp;
    s.o = h_offs[t];
    s.op = h_offs[t - 1];
    s.tilesM = (int)cdiv(std::max(std::max(B, Bp), 1), tc::BM);
    hs.push_back(s);
    maps.push_back(tc::make_map(ws.dhu.p + (size_t)h_offs[t] * H3, std::max(B, 1), H3, H3, tc::BM, false));
  }
  sf::launch<1>(c, m, params, hs, maps, ws, nullptr, false);
}

}  // namespace verg
