// epilogue.cuh — fused GEMM epilogues shared by the SIMT and tcgen05 GEMMs:
// each is called once per output element (m, n) with the accumulated value
// and the split-K index z.
#pragma once

#include "common.cuh"

namespace verg {

struct EpiStore {
  float* C;
  int ldc;
  __device__ void operator()(int m, int n, float v, int) const { C[(size_t)m * ldc + n] = v; }
};
struct EpiBias {
  float* C;
  int ldc;
  const float* bias;
  __device__ void operator()(int m, int n, float v, int) const { C[(size_t)m * ldc + n] = v + bias[n]; }
};
struct EpiBiasTanh {
  float* C;
  int ldc;
  const float* bias;
  __device__ void operator()(int m, int n, float v, int) const {
    C[(size_t)m * ldc + n] = tanhf(v + bias[n]);
  }
};
struct EpiAddTerm {  // C = acc + T
  float* C;
  int ldc;
  const float* T;
  int ldt;
  __device__ void operator()(int m, int n, float v, int) const {
    C[(size_t)m * ldc + n] = v + T[(size_t)m * ldt + n];
  }
};
struct EpiTanhGrad {  // C = acc * (1 - Y^2)
  float* C;
  int ldc;
  const float* Y;
  int ldy;
  __device__ void operator()(int m, int n, float v, int) const {
    const float y = Y[(size_t)m * ldy + n];
    C[(size_t)m * ldc + n] = v * (1.f - y * y);
  }
};
struct EpiPartial {  // split-K partial z
  float* W;
  int M, N;
  __device__ void operator()(int m, int n, float v, int z) const {
    W[((size_t)z * M + m) * N + n] = v;
  }
};

}  // namespace verg
