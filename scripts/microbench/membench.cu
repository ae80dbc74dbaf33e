// scratch: streaming r, V, done -> A, R with the GAE tile shapes, no scan
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int T, int I>
__global__ void __launch_bounds__(T) stream8(const float* __restrict__ r, const float* __restrict__ v,
                                             const uint8_t* __restrict__ d, float* a, float* o, int F, int* ctr, int dyn) {
  __shared__ int s_tile;
  if (dyn) { if (threadIdx.x == 0) s_tile = atomicAdd(ctr, 1); __syncthreads(); }
  const int tile = dyn ? s_tile : blockIdx.x;
  const int i0 = tile * T * I + threadIdx.x * I;
  if (i0 + I > F) return;
  float x[I], y[I];
#pragma unroll
  for (int q = 0; q < I; q += 4) {
    float4 p = __ldcs((const float4*)(r + i0 + q)), s = __ldcs((const float4*)(v + i0 + q));
    x[q] = p.x; x[q+1] = p.y; x[q+2] = p.z; x[q+3] = p.w; y[q] = s.x; y[q+1] = s.y; y[q+2] = s.z; y[q+3] = s.w;
  }
  uint32_t dd = *(const uint32_t*)(d + i0);
#pragma unroll
  for (int q = 0; q < I; q += 4) {
    float m = (dd & 1) ? 0.f : 1.f;
    __stcs((float4*)(a + i0 + q), make_float4(x[q]*m, x[q+1], x[q+2], x[q+3]));
    __stcs((float4*)(o + i0 + q), make_float4(y[q], y[q+1]*m, y[q+2], y[q+3]));
  }
}
int main() {
  const int F = 1 << 26;
  float *r, *v, *a, *o; uint8_t* d; int* ctr;
  cudaMalloc(&r, 4ull*F); cudaMalloc(&v, 4ull*F); cudaMalloc(&a, 4ull*F); cudaMalloc(&o, 4ull*F); cudaMalloc(&d, F); cudaMalloc(&ctr, 4);
  cudaMemset(r, 0, 4ull*F); cudaMemset(v, 0, 4ull*F); cudaMemset(d, 0, F);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](auto k, int T, int I, int dyn, const char* name) {
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaMemset(ctr, 0, 4);
      cudaEventRecord(e0);
      k<<<F / (T * I), T>>>(r, v, d, a, o, F, ctr, dyn);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("%-28s dyn=%d  %.3f ms  %.0f GB/s (17 B/item)\n", name, dyn, best, 17.0 * F / best / 1e6);
  };
  for (int dyn = 0; dyn < 2; ++dyn) {
    run(stream8<256, 4>, 256, 4, dyn, "256 thr x 4 items");
    run(stream8<256, 8>, 256, 8, dyn, "256 thr x 8 items");
    run(stream8<512, 4>, 512, 4, dyn, "512 thr x 4 items");
    run(stream8<256, 16>, 256, 16, dyn, "256 thr x 16 items");
    run(stream8<128, 16>, 128, 16, dyn, "128 thr x 16 items");
  }
  return 0;
}
