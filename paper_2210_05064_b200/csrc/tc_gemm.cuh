// tc_gemm.cu — the policy's batched GEMMs on the 5th-generation tensor cores.
//
// C (M x N) = op(A) op(B) with fused epilogue, fp32 in / fp32 out, on
// tcgen05.mma kind::tf32 with accumulators in TMEM:
//   * operands are staged by TMA (cp.async.bulk.tensor.2d, 128-byte swizzle)
//     into a 3-stage shared-memory ring; K-major and MN-major operands are
//     both native (no transposes in HBM);
//   * parity mode (3xTF32): four split warps write lo = x - trunc_tf32(x) of
//     every landed stage next to it; the landed fp32 tile itself is the hi
//     operand (the tensor core reads fp32 as tf32 by truncation).  Each K-step
//     issues hi*hi + lo*hi + hi*lo; dropping lo*lo leaves ~2^-21 relative
//     error per product: fp32-grade results, which is what the 1e-5 parity
//     bound needs;  fast mode issues hi*hi only;
//   * one elected thread issues the MMAs (M = 128, N = 128, K = 8 per
//     instruction) and commits each stage back to the TMA producer through an
//     mbarrier; the epilogue warps read the accumulator with tcgen05.ld
//     (32x32b.x32), transpose 32x32 blocks through shared memory and store
//     rows as float4 with the fused bias / tanh / tanh-gradient / split-K
//     functor (coalesced: 4 rows x 128 B per warp store);
//   * persistent CTAs (one per SM) with the accumulator in four TMEM buffers,
//     so the next tile's MMAs overlap this tile's epilogue.
// Warp roles (320 threads): 0 TMA producer, 1 TMEM allocator + MMA issuer,
// 2..5 3xTF32 operand split, 6..9 accumulator promotion + epilogue.
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "epilogue.cuh"

namespace verg {
namespace tc {

constexpr int BM = 128, BN = 128, BK = 32;  // BK in fp32 elements: one 128-byte swizzle row
constexpr int STAGES = 3;
constexpr int SPLIT_WARPS = 4, EPI_WARPS = 4;
constexpr int THREADS = 32 * (2 + SPLIT_WARPS + EPI_WARPS);  // TMA, MMA, split x4, epilogue x4
constexpr int TILE_BYTES = BM * BK * 4;  // 16 KB (A and B tiles alike: BM == BN)
constexpr int STAGE_BYTES = 4 * TILE_BYTES;  // A hi, A lo, B hi, B lo
constexpr int NACC = 4;                      // TMEM accumulator buffers: 4 x 128 columns = all 512
constexpr int EPI_LD = 36;                   // epilogue staging row stride (floats): float4 writes conflict-free
constexpr int EPI_BYTES = EPI_WARPS * 32 * EPI_LD * 4;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + EPI_BYTES + 1024 /*align*/ + 256 /*barriers*/;
// The tensor core's fp32 accumulation truncates; so that 3xTF32 stays
// fp32-grade for long K, each group of PROMOTE K-blocks (128 K) accumulates
// into one TMEM buffer which the epilogue warps drain into fp32 registers
// (round-to-nearest adds) while the MMA fills the next one.  The drains read
// 64 KB of TMEM each (tcgen05.ld: ~64 B/cycle/SM), so 4 rather than 2 K-blocks
// per group: C3 update -3 ms at unchanged parity.
constexpr int PROMOTE = 4;

// Debug instrumentation (ver_debug_gemm_prof): per-role clock64 cycles spent
// waiting, summed over CTAs; off unless g_tc_prof_on is set.  Slots: 0 MMA
// waits acc_empty, 1 MMA waits split, 2 MMA loop total, 3 split waits full,
// 4 split waits A slot, 5 epilogue waits acc_full, 6 epilogue final stores,
// 7 producer waits empty, 8 stages issued, 9 epilogue drains
static __device__ unsigned long long g_tc_prof[16];
static __device__ int g_tc_prof_on;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra LAB_WAIT;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t mbar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(mbar), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void umma_commit(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar)
               : "memory");
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// D (tmem) += A (tmem, K-major, lane = row, one 32-bit column per k) x B (smem)
__device__ __forceinline__ void mma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// 32 consecutive TMEM columns of this warp's 32 lanes <- v[0..31] (one per lane per column)
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
      "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
      "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}

// shared-memory matrix descriptors (sm_100 UMMA, 128-byte swizzle, version 1)
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;       // version (sm_100)
  d |= (uint64_t)layout << 61;  // 2 = SWIZZLE_128B, 1 = SWIZZLE_128B_BASE32B
  return d;
}
// K-major (SWIZZLE_128B): rows of 128 B (32 tf32 along K), 8-row atoms
// 1024 B apart (SBO); one MMA (K = 8) advances 32 B inside the swizzled row.
// MN-major: 32-bit elements need the 32-byte-atom 128B swizzle
// (SWIZZLE_128B_BASE32B, TMA CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B): 128 B
// along M/N per K-row, 4-row atoms 512 B apart along K (SBO), 32-element
// M/N chunks 4096 B apart (LBO); one MMA (K = 8) advances 8 K-rows = 1024 B.
template <int MAJ>
__device__ __forceinline__ uint64_t operand_desc(uint32_t tile, int kk) {
  if (MAJ == 0) return desc_sw128(tile + kk * 32, 16, 1024, 2);
  return desc_sw128(tile + kk * 1024, 4096, 512, 1);
}

__device__ __forceinline__ float rna_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
// lo = x - trunc_tf32(x) (tf32 keeps sign, exponent and the top 10 mantissa
// bits; the difference is exact in fp32 and the tensor core reads its top 11
// significant bits).  Rounding lo with cvt.rna would cost ~10% of the split
// throughput for a term below the dropped lo*lo.
__device__ __forceinline__ float lo1(float x) { return x - __uint_as_float(__float_as_uint(x) & 0xffffe000u); }
__device__ __forceinline__ float4 lo_tf32(float4 x) { return make_float4(lo1(x.x), lo1(x.y), lo1(x.z), lo1(x.w)); }

// A: MAJ 0 = K-major (M x K row-major), 1 = MN-major (K x M row-major)
// B: MAJ 0 = K-major (N x K row-major), 1 = MN-major (K x N row-major)
//
// Persistent: CTA b walks tiles b, b + grid, ... (n-tile fastest, so the CTAs
// running at the same time share an A row block in L2).  Every role keeps
// running counters across tiles, so the smem ring and the four TMEM
// accumulator buffers flow from one tile into the next: the MMA issuer starts
// tile i+1 while the epilogue warps are still storing tile i.
// ATM (K-major A, 3xTF32 only): the split warps move A's hi / lo into tensor
// memory with tcgen05.st and the MMAs read A from TMEM (the .kind::tf32 [a_tmem]
// form), so shared memory carries only the B operand reads: a third less
// shared-memory traffic per stage.  Two accumulator buffers then (TMEM:
// 2 x 128 accumulator columns + 3 stages x 64 A columns).
// BLO (3xTF32): B's lo part comes pre-split from global memory through a second
// tensor map (tmBl, e.g. the weights' lo copy made once per minibatch), so the
// split warps only split A; bit-identical to splitting B in shared memory.
template <int AMAJ, int BMAJ, int SPLIT3, class Epi, int ATM = 0, int BLO = 0>
__global__ void __launch_bounds__(THREADS, 1) tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                                                             const __grid_constant__ CUtensorMap tmB, int M,
                                                             int N, int K, int kb_per_split, int nsplit, Epi epi,
                                                             const __grid_constant__ CUtensorMap tmBl, int promote) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-aligned by pointer arithmetic on the __shared__ array, so that the compiler
  // keeps the shared address space (LDS/STS, not generic LD/ST) for derived pointers
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* stg_all = reinterpret_cast<float*>(smem + tc::STAGES * tc::STAGE_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + tc::STAGES * tc::STAGE_BYTES + EPI_BYTES);
  // bars: full[S] split[S] empty[S] acc_full[NACC] acc_empty[NACC]; then the TMEM address slot
  // ATM 1: 2 accumulator buffers + a 4-deep TMEM ring of A stages; ATM 2: 3
  // accumulator buffers + a 2-deep TMEM A ring (the split warps then also wait
  // for the MMAs of stage it - 2 before overwriting its A slot)
  constexpr int NACC = ATM == 2 ? 3 : (ATM ? 2 : tc::NACC);
  // ATM stages hold A hi, B hi, B lo only (A lo lives in TMEM): 4 x 48 KB
  constexpr int STAGES = ATM ? 4 : tc::STAGES;
  constexpr int STAGE_BYTES = ATM ? 3 * TILE_BYTES : tc::STAGE_BYTES;
  static_assert(STAGES * STAGE_BYTES <= tc::STAGES * tc::STAGE_BYTES, "smem budget");
  constexpr int ARING = ATM == 2 ? 2 : STAGES;
  static_assert(!ATM || NACC * BN + ARING * 64 <= 512, "TMEM budget");
  constexpr int A_COL0 = NACC * BN;  // ATM: A slot q hi at A_COL0 + 64 q, lo at + 32
  static_assert(!ATM || SPLIT3, "A via TMEM: 3xTF32");
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * 4 + 2 * tc::NACC);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tilesN = (N + BN - 1) / BN, tilesM = (M + BM - 1) / BM;
  const int ntiles = tilesN * tilesM * nsplit;
  const int nkb_total = (K + BK - 1) / BK;
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar0 = smem_u32(bars);
  auto full_bar = [&](int s) { return bar0 + 8 * s; };
  auto split_bar = [&](int s) { return bar0 + 8 * (STAGES + s); };
  auto empty_bar = [&](int s) { return bar0 + 8 * (2 * STAGES + s); };
  auto acc_full = [&](int b) { return bar0 + 8 * (3 * STAGES + b); };
  auto acc_empty = [&](int b) { return bar0 + 8 * (3 * STAGES + NACC + b); };
  // 0 A hi, 1 A lo, 2 B hi, 3 B lo (ATM: A hi, B hi, B lo)
  auto tile = [&](int s, int which) {
    return sbase + s * STAGE_BYTES + (ATM ? (which == 0 ? 0 : which - 1) : which) * TILE_BYTES;
  };
  struct Tile {
    int m0, n0, z, kb0, nkb;
  };
  auto decode = [&](int t) {
    Tile r;
    const int nt = t % tilesN, q = t / tilesN;
    r.n0 = nt * BN;
    r.m0 = (q % tilesM) * BM;
    r.z = q / tilesM;
    r.kb0 = r.z * kb_per_split;
    r.nkb = max(0, min(nkb_total, r.kb0 + kb_per_split) - r.kb0);
    return r;
  };

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
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    if (BLO) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmBl)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const bool prof = g_tc_prof_on != 0;
  // programmatic dependent launch: the prologue above overlapped the previous
  // kernel's tail; its results are visible after this wait.  The next kernel may
  // be scheduled as soon as SMs free up (it waits the same way).
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      int it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const Tile T = decode(t);
        for (int i = 0; i < T.nkb; ++i, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          const long long w0 = prof ? clock64() : 0;
          mbar_wait(empty_bar(s), ph ^ 1);
          if (prof) atomicAdd(&g_tc_prof[7], (unsigned long long)(clock64() - w0));
          mbar_expect_tx(full_bar(s), (BLO ? 3 : 2) * TILE_BYTES);
          const int k0 = (T.kb0 + i) * BK;
          if (AMAJ == 0) {
            tma_load_2d(tile(s, 0), &tmA, full_bar(s), k0, T.m0);
          } else {
#pragma unroll
            for (int c = 0; c < BM / 32; ++c) tma_load_2d(tile(s, 0) + c * 4096, &tmA, full_bar(s), T.m0 + 32 * c, k0);
          }
          if (BMAJ == 0) {
            tma_load_2d(tile(s, 2), &tmB, full_bar(s), k0, T.n0);
            if (BLO) tma_load_2d(tile(s, 3), &tmBl, full_bar(s), k0, T.n0);
          } else {
#pragma unroll
            for (int c = 0; c < BN / 32; ++c) tma_load_2d(tile(s, 2) + c * 4096, &tmB, full_bar(s), T.n0 + 32 * c, k0);
            if (BLO) {
#pragma unroll
              for (int c = 0; c < BN / 32; ++c)
                tma_load_2d(tile(s, 3) + c * 4096, &tmBl, full_bar(s), T.n0 + 32 * c, k0);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one thread)
    const uint32_t idesc = (1u << 4)                         // D format F32
                           | (2u << 7) | (2u << 10)          // A, B format TF32
                           | ((uint32_t)(ATM ? 0 : AMAJ) << 15) | ((uint32_t)BMAJ << 16)
                           | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
    if (lane == 0) {
      int it = 0, g = 0, buf = 0;
      unsigned long long wa = 0, ws_ = 0;
      const long long t_start = prof ? clock64() : 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const Tile T = decode(t);
        for (int i = 0; i < T.nkb; ++i, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          const bool first = (i % promote) == 0;
          if (first) {
            buf = g % NACC;
            const int u = g / NACC;
            const long long w0 = prof ? clock64() : 0;
            if (u >= 1) mbar_wait(acc_empty(buf), (u - 1) & 1);
            if (prof) wa += clock64() - w0;
          }
          const long long w1 = prof ? clock64() : 0;
          if (SPLIT3) mbar_wait(split_bar(s), ph);
          else mbar_wait(full_bar(s), ph);
          if (prof) ws_ += clock64() - w1;
          tc_fence_after();
          const uint32_t d = tmem + (uint32_t)(buf * BN);
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            const uint64_t bh = operand_desc<BMAJ>(tile(s, 2), kk);
            const uint32_t acc = (!first || kk > 0) ? 1u : 0u;
            if (ATM) {
              const uint32_t ah = tmem + (uint32_t)(A_COL0 + 64 * (it % ARING) + 8 * kk);
              const uint64_t bl = operand_desc<BMAJ>(tile(s, 3), kk);
              mma_tf32_ts(d, ah, bh, idesc, acc);
              mma_tf32_ts(d, ah + 32, bh, idesc, 1u);
              mma_tf32_ts(d, ah, bl, idesc, 1u);
            } else {
              const uint64_t ah = operand_desc<AMAJ>(tile(s, 0), kk);
              mma_tf32(d, ah, bh, idesc, acc);
              if (SPLIT3) {
                const uint64_t al = operand_desc<AMAJ>(tile(s, 1), kk);
                const uint64_t bl = operand_desc<BMAJ>(tile(s, 3), kk);
                mma_tf32(d, al, bh, idesc, 1u);
                mma_tf32(d, ah, bl, idesc, 1u);
              }
            }
          }
          umma_commit(empty_bar(s));
          if ((i % promote) == promote - 1 || i == T.nkb - 1) {
            umma_commit(acc_full(buf));
            ++g;
          }
        }
      }
      if (prof) {
        atomicAdd(&g_tc_prof[0], wa);
        atomicAdd(&g_tc_prof[1], ws_);
        atomicAdd(&g_tc_prof[2], (unsigned long long)(clock64() - t_start));
        atomicAdd(&g_tc_prof[8], (unsigned long long)it);
      }
    }
    __syncwarp();
  } else if (warp < 2 + SPLIT_WARPS) {
    // ---------------- 3xTF32 operand split, warps 2..5
    if (SPLIT3) {
      const int et = threadIdx.x - 64;  // 0..127
      int it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const Tile T = decode(t);
        for (int i = 0; i < T.nkb; ++i, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          const long long w0 = prof ? clock64() : 0;
          mbar_wait(full_bar(s), ph);
          if (prof && lane == 0) atomicAdd(&g_tc_prof[3], (unsigned long long)(clock64() - w0));
          uint8_t* st = smem + s * STAGE_BYTES;
          float4* ahi = reinterpret_cast<float4*>(st);
          float4* alo = reinterpret_cast<float4*>(st + TILE_BYTES);
          float4* bhi = reinterpret_cast<float4*>(st + (ATM ? 1 : 2) * TILE_BYTES);
          float4* blo = reinterpret_cast<float4*>(st + (ATM ? 2 : 3) * TILE_BYTES);
          if (ATM) {
            // row r = this thread's TMEM lane: its 32 K values
            const int r = 32 * (warp & 3) + lane;
            uint32_t hv[32], lv[32];
            if (AMAJ == 0) {
              // SW128 K-major tile: 16-byte chunk c of row r sits at chunk c ^ (r % 8)
              const uint8_t* rowp = st + (r >> 3) * 1024 + (r & 7) * 128;
#pragma unroll
              for (int c = 0; c < 8; ++c) {
                const float4 x = *reinterpret_cast<const float4*>(rowp + ((c ^ (r & 7)) << 4));
                const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const uint32_t hb = __float_as_uint(xs[j]) & 0xffffe000u;
                  hv[4 * c + j] = hb;
                  lv[4 * c + j] = __float_as_uint(xs[j] - __uint_as_float(hb));
                }
              }
            } else {
              // unswizzled MN-major tile (A never feeds the MMA from shared memory
              // here): 32-row chunk r / 32 at 4096 B, K-row k at 128 B, row r % 32 at
              // 4 B -- a warp reads one 128-byte K-row per load (conflict-free)
              const float* colp = reinterpret_cast<const float*>(st + (r >> 5) * 4096) + (r & 31);
#pragma unroll
              for (int k = 0; k < 32; ++k) {
                const float x = colp[32 * k];
                const uint32_t hb = __float_as_uint(x) & 0xffffe000u;
                hv[k] = hb;
                lv[k] = __float_as_uint(x - __uint_as_float(hb));
              }
            }
            if (ATM == 2 && it >= ARING) {  // the MMAs of stage it - ARING have read this A slot
              const int q = it - ARING;
              const long long w1 = prof ? clock64() : 0;
              mbar_wait(empty_bar(q % STAGES), (q / STAGES) & 1);
              if (prof && lane == 0) atomicAdd(&g_tc_prof[4], (unsigned long long)(clock64() - w1));
              tc_fence_after();
            }
            const uint32_t ta = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(A_COL0 + 64 * (it % ARING));
            tmem_st32(ta, hv);
            tmem_st32(ta + 32, lv);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            if (!BLO) {
#pragma unroll 4
              for (int q = et; q < TILE_BYTES / 16; q += 32 * SPLIT_WARPS) blo[q] = lo_tf32(bhi[q]);
            }
            (void)alo;
            tc_fence_before();
          } else {
#pragma unroll 4
            for (int q = et; q < TILE_BYTES / 16; q += 32 * SPLIT_WARPS) {
              // the tensor core reads an fp32 operand as tf32 by truncation, so the
              // landed tile already is hi = trunc_tf32(x); only lo = x - hi is written
              alo[q] = lo_tf32(ahi[q]);
              if (!BLO) blo[q] = lo_tf32(bhi[q]);
            }
          }
          // generic-proxy smem writes -> visible to the tensor core (async proxy)
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(split_bar(s));
        }
      }
    }
  } else {
    // ---------------- accumulator promotion + epilogue, warps 6..9
    // TMEM lane quarter of warp w is w % 4; rows lane_base .. lane_base + 31
    const int lane_base = 32 * (warp & 3);
    float* stg = stg_all + (warp & 3) * 32 * EPI_LD;
    int g = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const Tile T = decode(t);
      const int ngroups = (T.nkb + promote - 1) / promote;
      {  // second epilogue operand (tanh-gradient Y, added term T) of this thread's row -> L2
        const int m = T.m0 + lane_base + lane;
        if (m < M) epi.prefetch_row(m, T.n0, min(BN, N - T.n0));
      }
      float sums[BN];
#pragma unroll
      for (int j = 0; j < BN; ++j) sums[j] = 0.f;
      for (int q = 0; q < ngroups; ++q, ++g) {
        const int buf = g % NACC;
        const long long w0 = prof ? clock64() : 0;
        mbar_wait(acc_full(buf), (g / NACC) & 1);
        if (prof && lane == 0) {
          atomicAdd(&g_tc_prof[5], (unsigned long long)(clock64() - w0));
          atomicAdd(&g_tc_prof[9], 1ull);
        }
        tc_fence_after();
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
      // epilogue: transpose 32 x 32 blocks through shared memory so each warp
      // store covers 4 rows x 128 contiguous bytes (float4 per lane)
      const long long e0 = prof ? clock64() : 0;
      const int rr = lane >> 3, c4 = (lane & 7) * 4;
#pragma unroll
      for (int cc = 0; cc < BN / 32; ++cc) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
          *reinterpret_cast<float4*>(stg + lane * EPI_LD + 4 * q) =
              make_float4(sums[cc * 32 + 4 * q], sums[cc * 32 + 4 * q + 1], sums[cc * 32 + 4 * q + 2],
                          sums[cc * 32 + 4 * q + 3]);
        __syncwarp();
        const int n = T.n0 + cc * 32 + c4;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int r = 4 * k + rr;
          const int m = T.m0 + lane_base + r;
          const float4 v = *reinterpret_cast<const float4*>(stg + r * EPI_LD + c4);
          if (m < M && n < N) epi.vec4(m, n, v, T.z);
        }
        __syncwarp();
      }
      if (prof && lane == 0) atomicAdd(&g_tc_prof[6], (unsigned long long)(clock64() - e0));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

// ------------------------------------------------- CTA-pair 256 x 256 tiles
// cta_group::2: a cluster of 2 CTAs (one TPC) computes a 256 x 256 output tile
// with one tcgen05.mma.cta_group::2 (M = 256, N = 256, K = 8) per K-step and
// 3xTF32 term, issued by the leader CTA (rank 0).  Each CTA holds its 128 rows
// of A and its 128-column half of B in its own shared memory; the MMA reads
// both CTAs' tiles, and each CTA's TMEM receives its 128 rows x 256 columns.
// Per SM and per MMA cycle this moves half the TMA bytes of the single-CTA
// 128 x 128 kernel (whose weight GEMMs sit at the chip's TMA/L2 throughput):
// per K-block stage each CTA loads 16 KB of A + 16 KB of B (+ 16 KB of B lo)
// for 1536 MMA cycles instead of 48 KB for 768.
//  * each CTA's TMA signals its own full barrier; its 2 split warps then
//    arrive on the LEADER's split barrier (2 x 2 arrivals) before the MMA reads;
//  * MMA completion is multicast to both CTAs' empty / acc_full barriers;
//  * each CTA runs 8 epilogue warps (TMEM lane quarter = warp % 4, column half
//    = (warp - 4) / 4) that arrive on the leader's acc_empty (2 x 8).
// A always comes from shared memory here (two 256-column accumulators fill the
// 512 TMEM columns).
namespace p2 {
constexpr int BM2 = 256, BN2 = 256, BNH = 128;  // pair tile; B columns per CTA
constexpr int SPLITW = 2, EPIW = 8;
constexpr int THREADS2 = 32 * (2 + SPLITW + EPIW);  // 384
constexpr int STAGES2 = 3;
constexpr int TILE = BM * BK * 4;                 // 16 KB: A rows of one CTA, or its B half
constexpr int STAGE2 = 4 * TILE;                  // A hi, A lo, B hi, B lo
constexpr int NACC2 = 2;                          // 2 x 256 TMEM columns
constexpr int SLD = 20;                           // epilogue staging row stride (16 columns + 4)
constexpr int EPI2 = EPIW * 32 * SLD * 4;
constexpr int SMEM2 = STAGES2 * STAGE2 + EPI2 + 1024 + 256;
static_assert(SMEM2 <= 232448, "smem budget");

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t to_rank(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ void arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void commit2(uint32_t mbar) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
          mbar)
      : "memory");
}
__device__ __forceinline__ void mma2_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void mma2_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// F16 = 1 ("fp16x2", fp32-grade like 3xTF32 at twice the MMA rate): both operands
// come pre-split from global memory as scaled fp16 pairs, x s = hi + lo (hi =
// fp16(x s), lo = fp16(x s - hi): 22 significant bits), K-major, 64 elements
// (128 bytes) per swizzle row, so a stage has the byte layout of the tf32 one
// with twice the K.  Each K-step issues hi*hi + lo*hi + hi*lo (kind::f16, fp32
// accumulate; fp16 x fp16 products are exact in fp32); the epilogue multiplies
// by *fscale = 1 / (s_A s_B), a power of two.  The split warps only relay the
// stage-landed signal to the leader CTA.
template <int AMAJ, int BMAJ, class Epi, int BLO, int F16 = 0>
__global__ void __launch_bounds__(THREADS2, 1) tc_gemm2_kernel(const __grid_constant__ CUtensorMap tmA,
                                                               const __grid_constant__ CUtensorMap tmB, int M,
                                                               int N, int K, int kb_per_split, int nsplit, Epi epi,
                                                               const __grid_constant__ CUtensorMap tmBl,
                                                               int promote,
                                                               const __grid_constant__ CUtensorMap tmAl,
                                                               const float* __restrict__ fscale,
                                                               const unsigned* __restrict__ amax) {
  static_assert(!F16 || (AMAJ == 0 && BMAJ == 0), "fp16x2 operands are K-major");
  constexpr int BKE = F16 ? 64 : BK;  // K elements per stage
  // F16 == 2: A lands as fp32 (two 32-K boxes) and the split warps write its scaled
  // halves; stage = A fp32 32 KB | A hi | A lo | B hi | B lo, two stages
  constexpr int NS = F16 == 2 ? 2 : STAGES2;
  constexpr int SB = F16 == 2 ? 6 * TILE : STAGE2;
  constexpr int A0 = F16 == 2 ? 2 * TILE : 0;  // A hi offset in the stage
  extern __shared__ uint8_t smem_raw[];
  // 1024-aligned by pointer arithmetic on the __shared__ array, so that the compiler
  // keeps the shared address space (LDS/STS, not generic LD/ST) for derived pointers
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* stg_all = reinterpret_cast<float*>(smem + NS * SB);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NS * SB + EPI2);
  // bars: full[S] split[S] empty[S] acc_full[NACC2] acc_empty[NACC2]; then the TMEM address slot
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * NS + 2 * NACC2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cta_rank();
  const bool leader = rank == 0;
  const int pair_id = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int tilesN = (N + BN2 - 1) / BN2, tilesM = (M + BM2 - 1) / BM2;
  const int ntiles = tilesN * tilesM * nsplit;
  const int nkb_total = (K + BKE - 1) / BKE;
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar0 = smem_u32(bars);
  auto full_bar = [&](int s) { return bar0 + 8 * s; };
  auto split_bar = [&](int s) { return bar0 + 8 * (NS + s); };
  auto empty_bar = [&](int s) { return bar0 + 8 * (2 * NS + s); };
  auto acc_full = [&](int b) { return bar0 + 8 * (3 * NS + b); };
  auto acc_empty = [&](int b) { return bar0 + 8 * (3 * NS + NACC2 + b); };
  auto tileA = [&](int s, int lo) { return sbase + s * SB + A0 + lo * TILE; };
  auto tileB = [&](int s, int lo) { return sbase + s * SB + A0 + (2 + lo) * TILE; };
  struct Tile {
    int m0, n0, z, kb0, nkb;
  };
  auto decode = [&](int t) {
    Tile r;
    const int nt = t % tilesN, q = t / tilesN;
    r.n0 = nt * BN2;
    r.m0 = (q % tilesM) * BM2;
    r.z = q / tilesM;
    r.kb0 = r.z * kb_per_split;
    r.nkb = max(0, min(nkb_total, r.kb0 + kb_per_split) - r.kb0);
    return r;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(split_bar(s), 2 * SPLITW);
      mbar_init(empty_bar(s), 1);
    }
    for (int b = 0; b < NACC2; ++b) {
      mbar_init(acc_full(b), 1);
      mbar_init(acc_empty(b), 2 * EPIW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    if (BLO || F16) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmBl)) : "memory");
    if (F16 == 1) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmAl)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(NACC2 * BN2)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();  // barriers of both CTAs initialised, TMEM allocated
  __syncthreads();     // (the same, as a CTA barrier: the TMEM address slot in shared memory)
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs: own 128 rows of A, own half of B)
    if (lane == 0) {
      int it = 0;
      for (int t = pair_id; t < ntiles; t += npairs) {
        const Tile T = decode(t);
        const int am = T.m0 + (int)rank * BM, bn = T.n0 + (int)rank * BNH;
        for (int i = 0; i < T.nkb; ++i, ++it) {
          const int s = it % NS;
          const uint32_t ph = (it / NS) & 1;
          mbar_wait(empty_bar(s), ph ^ 1);
          if (F16 == 2) {
            mbar_expect_tx(full_bar(s), 4 * TILE);
            const int k0 = (T.kb0 + i) * BKE;
            const uint32_t a32 = sbase + s * SB;
            tma_load_2d(a32, &tmA, full_bar(s), k0, am);
            tma_load_2d(a32 + TILE, &tmA, full_bar(s), k0 + 32, am);
            tma_load_2d(tileB(s, 0), &tmB, full_bar(s), k0, bn);
            tma_load_2d(tileB(s, 1), &tmBl, full_bar(s), k0, bn);
            continue;
          }
          if (F16) {
            mbar_expect_tx(full_bar(s), 4 * TILE);
            const int k0 = (T.kb0 + i) * BKE;
            tma_load_2d(tileA(s, 0), &tmA, full_bar(s), k0, am);
            tma_load_2d(tileA(s, 1), &tmAl, full_bar(s), k0, am);
            tma_load_2d(tileB(s, 0), &tmB, full_bar(s), k0, bn);
            tma_load_2d(tileB(s, 1), &tmBl, full_bar(s), k0, bn);
            continue;
          }
          mbar_expect_tx(full_bar(s), (BLO ? 3 : 2) * TILE);
          const int k0 = (T.kb0 + i) * BK;
          if (AMAJ == 0) {
            tma_load_2d(tileA(s, 0), &tmA, full_bar(s), k0, am);
          } else {
#pragma unroll
            for (int c = 0; c < BM / 32; ++c) tma_load_2d(tileA(s, 0) + c * 4096, &tmA, full_bar(s), am + 32 * c, k0);
          }
          if (BMAJ == 0) {
            tma_load_2d(tileB(s, 0), &tmB, full_bar(s), k0, bn);
            if (BLO) tma_load_2d(tileB(s, 1), &tmBl, full_bar(s), k0, bn);
          } else {
#pragma unroll
            for (int c = 0; c < BNH / 32; ++c) tma_load_2d(tileB(s, 0) + c * 4096, &tmB, full_bar(s), bn + 32 * c, k0);
            if (BLO) {
#pragma unroll
              for (int c = 0; c < BNH / 32; ++c)
                tma_load_2d(tileB(s, 1) + c * 4096, &tmBl, full_bar(s), bn + 32 * c, k0);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader CTA, one thread)
    // D f32; A / B tf32 (2) or f16 (0)
    const uint32_t fmt = F16 ? 0u : 2u;
    const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)AMAJ << 15) | ((uint32_t)BMAJ << 16) |
                           ((uint32_t)(BN2 >> 3) << 17) | ((uint32_t)(BM2 >> 4) << 24);
    if (leader && lane == 0) {
      int it = 0, g = 0, buf = 0;
      for (int t = pair_id; t < ntiles; t += npairs) {
        const Tile T = decode(t);
        for (int i = 0; i < T.nkb; ++i, ++it) {
          const int s = it % NS;
          const uint32_t ph = (it / NS) & 1;
          const bool first = (i % promote) == 0;
          if (first) {
            buf = g % NACC2;
            const int u = g / NACC2;
            if (u >= 1) mbar_wait(acc_empty(buf), (u - 1) & 1);
          }
          mbar_wait(split_bar(s), ph);
          tc_fence_after();
          const uint32_t d = tmem + (uint32_t)(buf * BN2);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {  // 32 bytes of K per MMA: 8 tf32 or 16 f16
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
          if ((i % promote) == promote - 1 || i == T.nkb - 1) {
            commit2(acc_full(buf));
            ++g;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp < 2 + SPLITW) {
    // ---------------- 3xTF32 operand split (both CTAs), then arrive on the leader
    const int et = threadIdx.x - 64;  // 0..63
    // A's scale (F16 == 2): 2^(14 - floor(log2 max|A|)) from the max its producer pass took
    float a_s = 1.f;
    if (F16 == 2) {
      const float mx = __uint_as_float(*amax);
      a_s = (mx > 0.f && isfinite(mx)) ? exp2f((float)(14 - ilogbf(mx))) : 1.f;
    }
    int it = 0;
    for (int t = pair_id; t < ntiles; t += npairs) {
      const Tile T = decode(t);
      for (int i = 0; i < T.nkb; ++i, ++it) {
        const int s = it % NS;
        const uint32_t ph = (it / NS) & 1;
        mbar_wait(full_bar(s), ph);
        if (F16 == 2) {
          // fp32 A (two 32-K swizzled boxes: row r's 16-byte chunk j at j ^ (r & 7))
          // -> scaled halves, 64 K per 128-byte row (chunk c' = 8 halves at c' ^ (r & 7))
          const uint8_t* a32 = smem + s * SB;
          uint8_t* ahi = smem + s * SB + A0;
          uint8_t* alo = ahi + TILE;
#pragma unroll 4
          for (int q = et; q < BM * 8; q += 32 * SPLITW) {
            const int r = q >> 3, c = q & 7, sw = r & 7;
            const uint8_t* src = a32 + (c >> 2) * TILE + r * 128;
            const int j0 = (2 * c) & 7;
            const float4 x0 = *reinterpret_cast<const float4*>(src + ((j0 ^ sw) << 4));
            const float4 x1 = *reinterpret_cast<const float4*>(src + (((j0 + 1) ^ sw) << 4));
            const float2 v[4] = {make_float2(x0.x * a_s, x0.y * a_s), make_float2(x0.z * a_s, x0.w * a_s),
                                 make_float2(x1.x * a_s, x1.y * a_s), make_float2(x1.z * a_s, x1.w * a_s)};
            uint32_t hw[4], lw[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {  // packed conversions: one cvt per pair of values
              const __half2 hh = __float22half2_rn(v[e]);
              const float2 hb = __half22float2(hh);
              const __half2 ll = __float22half2_rn(make_float2(v[e].x - hb.x, v[e].y - hb.y));
              hw[e] = *reinterpret_cast<const uint32_t*>(&hh);
              lw[e] = *reinterpret_cast<const uint32_t*>(&ll);
            }
            const int o = r * 128 + ((c ^ sw) << 4);
            *reinterpret_cast<uint4*>(ahi + o) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
            *reinterpret_cast<uint4*>(alo + o) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        } else if (!F16) {
          uint8_t* st = smem + s * STAGE2;
          const float4* ahi = reinterpret_cast<const float4*>(st);
          float4* alo = reinterpret_cast<float4*>(st + TILE);
          const float4* bhi = reinterpret_cast<const float4*>(st + 2 * TILE);
          float4* blo = reinterpret_cast<float4*>(st + 3 * TILE);
#pragma unroll 4
          for (int q = et; q < TILE / 16; q += 32 * SPLITW) {
            alo[q] = lo_tf32(ahi[q]);
            if (!BLO) blo[q] = lo_tf32(bhi[q]);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        __syncwarp();
        if (lane == 0) arrive_remote(to_rank(split_bar(s), 0));
      }
    }
  } else {
    // ---------------- accumulator promotion + epilogue (both CTAs: own 128 rows;
    // warp w: TMEM lanes 32 (w % 4) .., columns 128 ((w - 4) / 4) ..)
    const int lq = warp & 3, half = (warp - 4) >> 2;
    const int lane_base = 32 * lq;
    float* stg = stg_all + (warp - 4) * 32 * SLD;
    int g = 0;
    for (int t = pair_id; t < ntiles; t += npairs) {
      const Tile T = decode(t);
      const int ngroups = (T.nkb + promote - 1) / promote;
      const int mrow0 = T.m0 + (int)rank * BM + lane_base;
      const int ncol0 = T.n0 + half * BNH;
      {  // second epilogue operand of this thread's row -> L2
        const int m = mrow0 + lane;
        if (m < M && ncol0 < N) epi.prefetch_row(m, ncol0, min(BNH, N - ncol0));
      }
      float sums[BNH];
#pragma unroll
      for (int j = 0; j < BNH; ++j) sums[j] = 0.f;
      for (int q = 0; q < ngroups; ++q, ++g) {
        const int buf = g % NACC2;
        mbar_wait(acc_full(buf), (g / NACC2) & 1);
        tc_fence_after();
#pragma unroll
        for (int cc = 0; cc < BNH / 32; ++cc) {
          uint32_t r[32];
          const uint32_t taddr =
              tmem + ((uint32_t)lane_base << 16) + (uint32_t)(buf * BN2 + half * BNH + cc * 32);
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
      if (F16) {  // undo the operand scales (a power of two: exact)
        float sc = *fscale;
        if (F16 == 2) {
          const float mx = __uint_as_float(*amax);
          sc /= (mx > 0.f && isfinite(mx)) ? exp2f((float)(14 - ilogbf(mx))) : 1.f;
        }
#pragma unroll
        for (int j = 0; j < BNH; ++j) sums[j] *= sc;
      }
      // epilogue: transpose 32 x 16 blocks through shared memory so each warp
      // store covers 8 rows x 64 contiguous bytes (float4 per lane)
      const int rr = lane >> 2, c4 = (lane & 3) * 4;
#pragma unroll
      for (int cb = 0; cb < BNH / 16; ++cb) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          *reinterpret_cast<float4*>(stg + lane * SLD + 4 * q) =
              make_float4(sums[cb * 16 + 4 * q], sums[cb * 16 + 4 * q + 1], sums[cb * 16 + 4 * q + 2],
                          sums[cb * 16 + 4 * q + 3]);
        __syncwarp();
        const int n = ncol0 + cb * 16 + c4;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int r = 8 * k + rr;
          const int m = mrow0 + r;
          const float4 v = *reinterpret_cast<const float4*>(stg + r * SLD + c4);
          if (m < M && n < N) epi.vec4(m, n, v, T.z);
        }
        __syncwarp();
      }
    }
  }
  tc_fence_before();
  cluster_sync_all();  // both CTAs done with TMEM and with remote arrivals
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(NACC2 * BN2) : "memory");
  }
}
}  // namespace p2

// ------------------------------------------------------------- host side
inline PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
inline std::once_flag g_encode_once;

inline PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (!g_encode) throw Error(VER_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  return g_encode;
}

// 2D fp32 row-major tensor (rows x cols, row stride ld elements), box {32, box_rows};
// `plain`: no swizzle (an MN-major A tile that only the split warps read)
inline CUtensorMap make_map(const float* base, int rows, int cols, int ld, int box_rows, bool mn_major,
                            bool plain = false) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  const cuuint32_t box[2] = {32, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box,
                         estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         plain ? CU_TENSOR_MAP_SWIZZLE_NONE
                               : (mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B),
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(VER_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
}

inline bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
// the coalesced epilogue stores float4: N, every leading dimension and every
// epilogue pointer must be 4-float aligned (Epi::vec_ok)
template <class Epi>
inline bool usable(int M, int N, int K, const float* A, int lda, const float* B, int ldb, const Epi& epi) {
  // TMA boxes (128 or 32 rows) may overhang the tensor: out-of-bounds rows / columns load as zero
  return M >= 1 && N >= 16 && K >= 8 && (N % 4) == 0 && (lda % 4) == 0 && (ldb % 4) == 0 && al16(A) &&
         al16(B) && epi.vec_ok();
}

// Blo (optional, 3xTF32): B's lo part (x - trunc_tf32(x)) in global memory with
// B's layout, e.g. a weight's copy made once per minibatch (BLO kernel variant).
// Tile geometry of a launch: 3xTF32 GEMMs with M >= 256 and N > 128 run on
// CTA pairs with 256 x 256 tiles (p2::tc_gemm2_kernel, one work unit per TPC),
// the rest on single CTAs with 128 x 128 tiles.
struct Geo {
  int bm, bn, units;
  bool pair;
};
inline Geo geo(const Ctx* c, int M, int N) {
  if (c->precision == 0 && M >= p2::BM2 && N > BN)
    return Geo{p2::BM2, p2::BN2, c->num_sms / 2, true};
  return Geo{BM, BN, c->num_sms, false};
}

template <int AMAJ, int BMAJ, class Epi>
void launch_pair(Ctx* c, int M, int N, int K, const float* A, int lda, const float* B, int ldb, Epi epi,
                 int splits, const float* Blo) {
  // A: K-major M x K (box 32 x 128) or MN-major K x M (box 32 x 32, swizzled: the
  // MMA reads A from shared memory here); B: its 128-column halves
  const CUtensorMap ta = AMAJ == 0 ? make_map(A, M, K, lda, BM, false) : make_map(A, K, M, lda, 32, true);
  const CUtensorMap tb = BMAJ == 0 ? make_map(B, N, K, ldb, p2::BNH, false) : make_map(B, K, N, ldb, 32, true);
  const bool blo = Blo && env_int("VER_TC_BLO", 1) && al16(Blo);
  const CUtensorMap tbl =
      !blo ? tb : (BMAJ == 0 ? make_map(Blo, N, K, ldb, p2::BNH, false) : make_map(Blo, K, N, ldb, 32, true));
  const int nkb = (K + BK - 1) / BK;
  splits = std::max(1, std::min(splits, nkb));
  const int per = (nkb + splits - 1) / splits;
  splits = (nkb + per - 1) / per;
  const long long ntiles = cdiv(N, p2::BN2) * cdiv(M, p2::BM2) * (long long)splits;
  const int promote = PROMOTE;
  auto run = [&](auto kern) {
    VER_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, p2::SMEM2));
    cudaLaunchConfig_t cfg{};
    cfg.blockDim = dim3(p2::THREADS2);
    cfg.dynamicSmemBytes = p2::SMEM2;
    cfg.stream = c->stream;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    // persistent: as many pairs as can be resident at once (one per TPC)
    static std::atomic<int> pairs_cache[kMaxDevices];
    int pairs = pairs_cache[dev_slot(c)].load();
    if (!pairs) {
      cfg.gridDim = dim3(c->num_sms);
      int nc = 0;
      VER_CUDA(cudaOccupancyMaxActiveClusters(&nc, kern, &cfg));
      pairs = std::max(1, std::min(nc, c->num_sms / 2));
      pairs_cache[dev_slot(c)].store(pairs);
    }
    cfg.gridDim = dim3(2 * (int)std::min<long long>(ntiles, pairs));
    VER_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb, M, N, K, per, splits, epi, tbl, promote, ta,
                                static_cast<const float*>(nullptr), static_cast<const unsigned*>(nullptr)));
    after_launch(c);
  };
  if (blo) run(p2::tc_gemm2_kernel<AMAJ, BMAJ, Epi, 1>);
  else run(p2::tc_gemm2_kernel<AMAJ, BMAJ, Epi, 0>);
}

// 2D fp16 row-major tensor (rows x cols, row stride ld elements), K-major box
// {64, box_rows} with the 128-byte swizzle (one swizzle row = 64 halves)
inline CUtensorMap make_map16(const __half* base, int rows, int cols, int ld, int box_rows) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  const cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(base), dims, strides, box,
                         estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(VER_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
}

// C = (A_hi + A_lo)(B_hi + B_lo)^T * fscale, fp16x2 on CTA pairs (p2::tc_gemm2_kernel
// F16): A M x K and B N x K, both K-major fp16 (row stride lda / ldb halves,
// 16-byte aligned rows); *fscale (device) = 1 / (s_A s_B).  M >= 256, N % 4 == 0.
inline bool usable_f16(int M, int N, int K, int lda, int ldb) {
  return M >= p2::BM2 && N >= 16 && (N % 4) == 0 && K >= 16 && (lda % 8) == 0 && (ldb % 8) == 0;
}
template <class Epi>
void launch_f16(Ctx* c, int M, int N, int K, const __half* Ahi, const __half* Alo, int lda, const __half* Bhi,
                const __half* Blo, int ldb, const float* fscale, Epi epi, int splits) {
  ScopedEv ev(c, c->gemm_tag);
  if (c->evlog && c->flop_log && c->gemm_tag >= 0) c->flop_log[c->gemm_tag] += 2.0 * M * (double)N * K;
  const CUtensorMap ta = make_map16(Ahi, M, K, lda, BM), tal = make_map16(Alo, M, K, lda, BM);
  const CUtensorMap tb = make_map16(Bhi, N, K, ldb, p2::BNH), tbl = make_map16(Blo, N, K, ldb, p2::BNH);
  const int nkb = (K + 63) / 64;
  splits = std::max(1, std::min(splits, nkb));
  const int per = (nkb + splits - 1) / splits;
  splits = (nkb + per - 1) / per;
  const long long ntiles = cdiv(N, p2::BN2) * cdiv(M, p2::BM2) * (long long)splits;
  const int promote = PROMOTE;
  auto kern = p2::tc_gemm2_kernel<0, 0, Epi, 0, 1>;
  VER_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, p2::SMEM2));
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(p2::THREADS2);
  cfg.dynamicSmemBytes = p2::SMEM2;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  static std::atomic<int> pairs_cache[kMaxDevices];
  int pairs = pairs_cache[dev_slot(c)].load();
  if (!pairs) {
    cfg.gridDim = dim3(c->num_sms);
    int nc = 0;
    VER_CUDA(cudaOccupancyMaxActiveClusters(&nc, kern, &cfg));
    pairs = std::max(1, std::min(nc, c->num_sms / 2));
    pairs_cache[dev_slot(c)].store(pairs);
  }
  cfg.gridDim = dim3(2 * (int)std::min<long long>(ntiles, pairs));
  VER_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb, M, N, K, per, splits, epi, tbl, promote, tal, fscale,
                              static_cast<const unsigned*>(nullptr)));
  after_launch(c);
}

// C = A (B_hi + B_lo)^T / s_B with A fp32 (M x K, K-major, row stride lda floats)
// converted to scaled fp16 halves inside the kernel (F16 == 2): *amax (device) =
// max |A| bits taken by a pass before, *binv = 1 / s_B; B N x K K-major halves.
constexpr int SMEM2_F16A = 2 * 6 * p2::TILE + p2::EPI2 + 1024 + 256;
static_assert(SMEM2_F16A <= 232448, "smem budget");
template <class Epi>
void launch_f16a(Ctx* c, int M, int N, int K, const float* A, int lda, const __half* Bhi, const __half* Blo,
                 int ldb, const unsigned* amax, const float* binv, Epi epi, int splits) {
  ScopedEv ev(c, c->gemm_tag);
  if (c->evlog && c->flop_log && c->gemm_tag >= 0) c->flop_log[c->gemm_tag] += 2.0 * M * (double)N * K;
  const CUtensorMap ta = make_map(A, M, K, lda, BM, false);
  const CUtensorMap tb = make_map16(Bhi, N, K, ldb, p2::BNH), tbl = make_map16(Blo, N, K, ldb, p2::BNH);
  const int nkb = (K + 63) / 64;
  splits = std::max(1, std::min(splits, nkb));
  const int per = (nkb + splits - 1) / splits;
  splits = (nkb + per - 1) / per;
  const long long ntiles = cdiv(N, p2::BN2) * cdiv(M, p2::BM2) * (long long)splits;
  const int promote = PROMOTE;
  auto kern = p2::tc_gemm2_kernel<0, 0, Epi, 0, 2>;
  VER_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM2_F16A));
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(p2::THREADS2);
  cfg.dynamicSmemBytes = SMEM2_F16A;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  static std::atomic<int> pairs_cache[kMaxDevices];
  int pairs = pairs_cache[dev_slot(c)].load();
  if (!pairs) {
    cfg.gridDim = dim3(c->num_sms);
    int nc = 0;
    VER_CUDA(cudaOccupancyMaxActiveClusters(&nc, kern, &cfg));
    pairs = std::max(1, std::min(nc, c->num_sms / 2));
    pairs_cache[dev_slot(c)].store(pairs);
  }
  cfg.gridDim = dim3(2 * (int)std::min<long long>(ntiles, pairs));
  VER_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb, M, N, K, per, splits, epi, tbl, promote, ta, binv, amax));
  after_launch(c);
}

template <int AMAJ, int BMAJ, class Epi>
void launch(Ctx* c, int M, int N, int K, const float* A, int lda, const float* B, int ldb, Epi epi, int splits,
            const float* Blo = nullptr) {
  ScopedEv ev(c, c->gemm_tag);  // learner timing of the GEMM family (bench roofline)
  if (c->evlog && c->flop_log && c->gemm_tag >= 0) c->flop_log[c->gemm_tag] += 2.0 * M * (double)N * K;
  if (geo(c, M, N).pair) {
    launch_pair<AMAJ, BMAJ>(c, M, N, K, A, lda, B, ldb, epi, splits, Blo);
    return;
  }
  // A: K-major M x K (box 32 x 128) or MN-major K x M (box 32 x 32; unswizzled when
  // the split warps move it into tensor memory)
  const bool atm = c->precision == 0 && env_int("VER_TC_ATM", 1) && (AMAJ == 0 || env_int("VER_TC_ATM_MN", 1));
  const CUtensorMap ta =
      AMAJ == 0 ? make_map(A, M, K, lda, BM, false) : make_map(A, K, M, lda, 32, true, atm);
  const CUtensorMap tb = BMAJ == 0 ? make_map(B, N, K, ldb, BN, false) : make_map(B, K, N, ldb, 32, true);
  const bool blo = Blo && c->precision == 0 && env_int("VER_TC_BLO", 1) && al16(Blo);
  const CUtensorMap tbl =
      !blo ? tb : (BMAJ == 0 ? make_map(Blo, N, K, ldb, BN, false) : make_map(Blo, K, N, ldb, 32, true));
  const int nkb = (K + BK - 1) / BK;
  splits = std::max(1, std::min(splits, nkb));
  const int per = (nkb + splits - 1) / splits;
  splits = (nkb + per - 1) / per;
  const long long ntiles = cdiv(N, BN) * cdiv(M, BM) * (long long)splits;
  const int grid = (int)std::min<long long>(ntiles, c->num_sms);
  const int promote = PROMOTE;
  auto run = [&](auto kern) {
    VER_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = SMEM_BYTES;
    cfg.stream = c->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    VER_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb, M, N, K, per, splits, epi, tbl, promote));
    after_launch(c);
  };
  if (c->precision == 0) {
    if (atm) {  // TMEM-A with 3 accumulator buffers
      if (blo) run(tc_gemm_kernel<AMAJ, BMAJ, 1, Epi, 2, 1>);
      else run(tc_gemm_kernel<AMAJ, BMAJ, 1, Epi, 2>);
      return;
    }
    if (blo) run(tc_gemm_kernel<AMAJ, BMAJ, 1, Epi, 0, 1>);
    else run(tc_gemm_kernel<AMAJ, BMAJ, 1, Epi>);
  } else {
    run(tc_gemm_kernel<AMAJ, BMAJ, 0, Epi>);
  }
}

// split-K count: the persistent kernel walks tiles x Z work items over the SMs,
// so the time goes as ceil(tiles Z / SMs) waves of K / Z (+ a per-item overhead)
// each; pick the cheapest Z (ties: fewer partials), >= 4 K-blocks per split.
// (Z = ceil(2 SMs / tiles) gave 2.3 waves for the 48-tile weight gradients.)
inline int splits_for(const Ctx* c, int M, int N, int K) {
  const Geo g = geo(c, M, N);
  const long long tiles = cdiv(N, g.bn) * cdiv(M, g.bm);
  const int nkb = (K + BK - 1) / BK;
  const int zmax = std::max(1, std::min(64, nkb / 4));
  int best = 1;
  double best_cost = 1e300;
  for (int z = 1; z <= zmax; ++z) {
    const long long waves = (tiles * z + g.units - 1) / g.units;
    // + ~6 K-blocks' worth of per-item overhead (pipeline fill, accumulator
    // drain, 64 KB partial-tile store)
    const double cost = (double)waves * (double)((nkb + z - 1) / z + 6);
    if (cost < best_cost * 0.999) {
      best_cost = cost;
      best = z;
    }
  }
  return best;
}

}  // namespace tc
}  // namespace verg
