// scratch: persistent 3-stage bulk-copy ring (r, V 8 KB + done 2 KB per 2048-slot tile) -> smem -> A, R stores
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int T = 256, I = 8, TILE = T * I, NS = 3, SB = TILE * 9;
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void __launch_bounds__(T + 32) ring(const float* r, const float* v, const uint8_t* d, float* a, float* o,
                                               int ntiles, int* ctr, int dyn) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t full[NS], empty[NS];
  __shared__ int stile[NS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(sa(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  auto wait = [&](uint64_t* b, uint32_t ph) {
    asm volatile("{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(sa(b)), "r"(ph));
  };
  if (warp == T / 32) {
    if (lane == 0) {
      for (int k = 0;; ++k) {
        const int s = k % NS;
        wait(&empty[s], ((k / NS) & 1) ^ 1);
        const int t = dyn ? atomicAdd(ctr, 1) : blockIdx.x + k * gridDim.x;
        if (t >= ntiles) { stile[s] = -1; asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&full[s]))); break; }
        stile[s] = t;
        const uint32_t mb = sa(&full[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(SB));
        uint8_t* st = sm + s * SB;
        const size_t lo = (size_t)t * TILE;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(st)), "l"(r + lo), "r"(4 * TILE), "r"(mb));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(st + 4 * TILE)), "l"(v + lo), "r"(4 * TILE), "r"(mb));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(st + 8 * TILE)), "l"(d + lo), "r"(TILE), "r"(mb));
      }
    }
    return;
  }
  for (int k = 0;; ++k) {
    const int s = k % NS;
    wait(&full[s], (k / NS) & 1);
    const int t = stile[s];
    if (t < 0) break;
    const uint8_t* st = sm + s * SB;
    const int l0 = threadIdx.x * I;
    const float4* r4 = (const float4*)(st) + l0 / 4;
    const float4* v4 = (const float4*)(st + 4 * TILE) + l0 / 4;
    float4 x0 = r4[0], x1 = r4[1], y0 = v4[0], y1 = v4[1];
    uint2 dd = *(const uint2*)(st + 8 * TILE + l0);
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[s])));
    float m = (dd.x & 1) ? 0.f : 1.f;
    const size_t g = (size_t)t * TILE + l0;
    __stcs((float4*)(a + g), make_float4(x0.x * m, x0.y, x0.z, x0.w));
    __stcs((float4*)(a + g) + 1, x1);
    __stcs((float4*)(o + g), make_float4(y0.x, y0.y * m, y0.z, y0.w));
    __stcs((float4*)(o + g) + 1, y1);
  }
}
int main() {
  const int F = 1 << 26, ntiles = F / TILE;
  float *r, *v, *a, *o; uint8_t* d; int* ctr;
  cudaMalloc(&r, 4ull*F); cudaMalloc(&v, 4ull*F); cudaMalloc(&a, 4ull*F); cudaMalloc(&o, 4ull*F); cudaMalloc(&d, F); cudaMalloc(&ctr, 4);
  cudaMemset(r, 0, 4ull*F); cudaMemset(v, 0, 4ull*F); cudaMemset(d, 0, F);
  cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, NS * SB);
  int per = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, ring, T + 32, NS * SB);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int dyn = 0; dyn < 2; ++dyn) for (int mult = 1; mult <= per; ++mult) {
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaMemset(ctr, 0, 4);
      cudaEventRecord(e0);
      ring<<<148 * mult, T + 32, NS * SB>>>(r, v, d, a, o, ntiles, ctr, dyn);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("ring dyn=%d ctas/SM=%d (max %d): %.3f ms %.0f GB/s  err=%s\n", dyn, mult, per, best, 17.0 * F / best / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
