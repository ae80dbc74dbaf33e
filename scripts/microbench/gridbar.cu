// Grid-barrier cost for the persistent step kernel's shape: 148 CTAs x 320
// threads, one CTA per SM (cooperative launch), N back-to-back barriers.
//   v0: __syncthreads; thread 0: __threadfence + atomicAdd + ld.acquire spin
//   v1: __syncthreads; thread 0: red.release.gpu + ld.acquire spin
//   v2: as v1, with a small per-barrier store from every thread before it
//       (the step kernel's partial / gate writes)
#include <cooperative_groups.h>
#include <cstdio>

__device__ __forceinline__ void bar_v0(unsigned* count, unsigned& target) {
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

__device__ __forceinline__ void bar_v1(unsigned* count, unsigned& target) {
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

// v3: per-CTA epoch flags; thread t < gridDim polls CTA t's flag
__device__ __forceinline__ void bar_v3(unsigned* flags, unsigned& epoch) {
  __syncthreads();
  ++epoch;
  if (threadIdx.x == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + blockIdx.x), "r"(epoch) : "memory");
  if (threadIdx.x < gridDim.x) {
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + threadIdx.x) : "memory");
    } while ((int)(v - epoch) < 0);
  }
  __syncthreads();
}

// v4: 8 spread counters (CTA i adds to counter i % 8, 128 B apart); 8 threads poll
__device__ __forceinline__ void bar_v4(unsigned* count, unsigned& epoch) {
  __syncthreads();
  ++epoch;
  if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(count + 32 * (blockIdx.x & 7)) : "memory");
  if (threadIdx.x < 8) {
    const unsigned need = epoch * ((gridDim.x - threadIdx.x + 7) / 8);
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(count + 32 * threadIdx.x) : "memory");
    } while (v < need);
  }
  __syncthreads();
}

template <int V>
__global__ void __launch_bounds__(320, 1) kbar(int n, unsigned* count, float* sink, long long* t) {
  unsigned target = 0;
  long long t0;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  for (int i = 0; i < n; ++i) {
    if (V == 2) sink[(size_t)(blockIdx.x * blockDim.x + threadIdx.x) * 4 + (i & 3)] = (float)i;
    if (V == 0) bar_v0(count, target);
    else if (V == 3) bar_v3(count, target);
    else if (V == 4) bar_v4(count, target);
    else bar_v1(count, target);
  }
  long long t1;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
  if (blockIdx.x == 0 && threadIdx.x == 0) *t = t1 - t0;
}

template <int V>
void run(int sms, unsigned* count, float* sink, long long* t) {
  int n = 2000;
  void* args[] = {&n, &count, &sink, &t};
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(count, 0, 4096);
    cudaLaunchCooperativeKernel((const void*)kbar<V>, dim3(sms), dim3(320), args, 0, 0);
    cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
    printf("v%d rep%d: %.3f us per barrier\n", V, rep, h / 1000.0 / n);
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* count;
  float* sink;
  long long* t;
  cudaMalloc(&count, 4096);
  cudaMalloc(&sink, (size_t)sms * 320 * 16);
  cudaMalloc(&t, 8);
  run<0>(sms, count, sink, t);
  run<1>(sms, count, sink, t);
  run<2>(sms, count, sink, t);
  run<3>(sms, count, sink, t);
  run<4>(sms, count, sink, t);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
