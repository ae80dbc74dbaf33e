// epilogue.cuh — fused GEMM epilogues shared by the SIMT and tcgen05 GEMMs.
// operator()(m, n, v, z): one output element (SIMT GEMM).
// vec4(m, n, v4, z): four consecutive columns n..n+3 of row m (tcgen05 GEMM's
// coalesced epilogue; n % 4 == 0, every leading dimension % 4 == 0).
#pragma once
#include <cuda_fp16.h>

#include "common.cuh"

namespace verg {

inline bool ptr16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// L2 prefetch of `ncols` floats of a row (the tcgen05 GEMM's epilogue warps issue
// it when a tile starts, for the epilogues that read a second operand: the
// loads at the tile's end then hit L2 instead of stalling the accumulator drain)
__device__ __forceinline__ void prefetch_row_l2(const float* row, int ncols) {
  for (int c = 0; c < ncols; c += 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(row + c));
}

__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}

struct EpiStore {
  float* C;
  int ldc;
  __device__ void prefetch_row(int, int, int) const {}
  bool vec_ok() const { return ptr16(C) && ldc % 4 == 0; }
  EpiStore shifted(int m0) const { return EpiStore{C + (size_t)m0 * ldc, ldc}; }  // rows m0.. (tail split)
  __device__ void operator()(int m, int n, float v, int) const { C[(size_t)m * ldc + n] = v; }
  __device__ void vec4(int m, int n, float4 v, int) const {
    *reinterpret_cast<float4*>(C + (size_t)m * ldc + n) = v;
  }
};
struct EpiBias {
  float* C;
  int ldc;
  const float* bias;
  __device__ void prefetch_row(int, int, int) const {}
  bool vec_ok() const { return ptr16(C) && ldc % 4 == 0 && ptr16(bias); }
  EpiBias shifted(int m0) const { return EpiBias{C + (size_t)m0 * ldc, ldc, bias}; }
  __device__ void operator()(int m, int n, float v, int) const { C[(size_t)m * ldc + n] = v + bias[n]; }
  __device__ void vec4(int m, int n, float4 v, int) const {
    *reinterpret_cast<float4*>(C + (size_t)m * ldc + n) = add4(v, __ldg(reinterpret_cast<const float4*>(bias + n)));
  }
};
struct EpiBiasTanh {
  float* C;
  int ldc;
  const float* bias;
  __device__ void prefetch_row(int, int, int) const {}
  bool vec_ok() const { return ptr16(C) && ldc % 4 == 0 && ptr16(bias); }
  EpiBiasTanh shifted(int m0) const { return EpiBiasTanh{C + (size_t)m0 * ldc, ldc, bias}; }
  __device__ void operator()(int m, int n, float v, int) const {
    C[(size_t)m * ldc + n] = tanhf(v + bias[n]);
  }
  __device__ void vec4(int m, int n, float4 v, int) const {
    const float4 b = __ldg(reinterpret_cast<const float4*>(bias + n));
    *reinterpret_cast<float4*>(C + (size_t)m * ldc + n) =
        make_float4(tanhf(v.x + b.x), tanhf(v.y + b.y), tanhf(v.z + b.z), tanhf(v.w + b.w));
  }
};
// EpiBiasTanh that also writes the result as fp16x2 halves (scale 2^14, tanh
// outputs) for the next fp16x2 GEMM (tc_gemm.cuh F16), same row stride
struct EpiBiasTanhH {
  float* C;
  int ldc;
  const float* bias;
  __half* hi;
  __half* lo;
  __device__ void prefetch_row(int, int, int) const {}
  bool vec_ok() const { return ptr16(C) && ldc % 4 == 0 && ptr16(bias) && ptr16(hi) && ptr16(lo) && ldc % 8 == 0; }
  EpiBiasTanhH shifted(int m0) const {
    return EpiBiasTanhH{C + (size_t)m0 * ldc, ldc, bias, hi + (size_t)m0 * ldc, lo + (size_t)m0 * ldc};
  }
  __device__ void operator()(int m, int n, float v, int) const {
    const float y = tanhf(v + bias[n]);
    const size_t i = (size_t)m * ldc + n;
    C[i] = y;
    const __half h = __float2half_rn(y * 16384.f);
    hi[i] = h;
    lo[i] = __float2half_rn(y * 16384.f - __half2float(h));
  }
  __device__ void vec4(int m, int n, float4 v, int) const {
    const float4 b = __ldg(reinterpret_cast<const float4*>(bias + n));
    const float4 y = make_float4(tanhf(v.x + b.x), tanhf(v.y + b.y), tanhf(v.z + b.z), tanhf(v.w + b.w));
    const size_t i = (size_t)m * ldc + n;
    *reinterpret_cast<float4*>(C + i) = y;
    const float ys[4] = {y.x * 16384.f, y.y * 16384.f, y.z * 16384.f, y.w * 16384.f};
    __half h[4], l[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      h[q] = __float2half_rn(ys[q]);
      l[q] = __float2half_rn(ys[q] - __half2float(h[q]));
    }
    reinterpret_cast<__half2*>(hi + i)[0] = __halves2half2(h[0], h[1]);
    reinterpret_cast<__half2*>(hi + i)[1] = __halves2half2(h[2], h[3]);
    reinterpret_cast<__half2*>(lo + i)[0] = __halves2half2(l[0], l[1]);
    reinterpret_cast<__half2*>(lo + i)[1] = __halves2half2(l[2], l[3]);
  }
};
struct EpiAddTerm {  // C = acc + T
  float* C;
  int ldc;
  const float* T;
  int ldt;
  __device__ void prefetch_row(int m, int n0, int ncols) const { prefetch_row_l2(T + (size_t)m * ldt + n0, ncols); }
  bool vec_ok() const { return ptr16(C) && ldc % 4 == 0 && ptr16(T) && ldt % 4 == 0; }
  EpiAddTerm shifted(int m0) const { return EpiAddTerm{C + (size_t)m0 * ldc, ldc, T + (size_t)m0 * ldt, ldt}; }
  __device__ void operator()(int m, int n, float v, int) const {
    C[(size_t)m * ldc + n] = v + T[(size_t)m * ldt + n];
  }
  __device__ void vec4(int m, int n, float4 v, int) const {
    *reinterpret_cast<float4*>(C + (size_t)m * ldc + n) =
        add4(v, *reinterpret_cast<const float4*>(T + (size_t)m * ldt + n));
  }
};
struct EpiTanhGrad {  // C = acc * (1 - Y^2)
  float* C;
  int ldc;
  const float* Y;
  int ldy;
  __device__ void prefetch_row(int m, int n0, int ncols) const { prefetch_row_l2(Y + (size_t)m * ldy + n0, ncols); }
  bool vec_ok() const { return ptr16(C) && ldc % 4 == 0 && ptr16(Y) && ldy % 4 == 0; }
  EpiTanhGrad shifted(int m0) const { return EpiTanhGrad{C + (size_t)m0 * ldc, ldc, Y + (size_t)m0 * ldy, ldy}; }
  __device__ void operator()(int m, int n, float v, int) const {
    const float y = Y[(size_t)m * ldy + n];
    C[(size_t)m * ldc + n] = v * (1.f - y * y);
  }
  __device__ void vec4(int m, int n, float4 v, int) const {
    const float4 y = *reinterpret_cast<const float4*>(Y + (size_t)m * ldy + n);
    *reinterpret_cast<float4*>(C + (size_t)m * ldc + n) =
        make_float4(v.x * (1.f - y.x * y.x), v.y * (1.f - y.y * y.y), v.z * (1.f - y.z * y.z),
                    v.w * (1.f - y.w * y.w));
  }
};
struct EpiPartial {  // split-K partial z
  float* W;
  int M, N;
  __device__ void prefetch_row(int, int, int) const {}
  bool vec_ok() const { return ptr16(W) && N % 4 == 0; }
  __device__ void operator()(int m, int n, float v, int z) const {
    W[((size_t)z * M + m) * N + n] = v;
  }
  __device__ void vec4(int m, int n, float4 v, int z) const {
    *reinterpret_cast<float4*>(W + ((size_t)z * M + m) * N + n) = v;
  }
};

}  // namespace verg
