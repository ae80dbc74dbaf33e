// preempt.cu — VER's optimal preemption threshold (distributed.cpp:16-65).
//
// estimate_time: the reference's counting bisection (Time(S) = S-th smallest
// of the merged progressions {k tau_i}), run by one CTA whose threads split
// the per-iteration count sum_i floor(t / tau_i).  The integer count is
// order-independent, so every bisection step and the final snap take the
// exact branches of the reference: bit-identical result.
//
// optimal_preempt_steps: the reference scans S = 1..S_max calling
// estimate_time for each (O(S_max * I * N), infeasible at S_max = 4.19M).
// Here: T* = Time(S_max); enumerate every yield double(k)*tau_i <= T*;
// sort them (bitonic, as uint64 bit patterns of positive doubles); then
// Time(S) = sorted[S-1] for all S at once and a parallel argmax of
// S / (Time(S) + LT) with ties -> smallest S.  This is the merge-sort
// formulation the reference's own tests pin as equivalent
// (test_distributed.cpp:16-37, :88-132).
#include <cfloat>
#include <cmath>

#include "common.cuh"

namespace verg {

constexpr int kPT = 1024;

__device__ long long block_sum_ll(long long v, long long* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  long long s = 0;
  for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s += red[k];
  return s;
}

__device__ long long count_yields(const double* tau, int n, double t, long long* red) {
  long long c = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) c += (long long)floor(t / tau[i]);
  return block_sum_ll(c, red);
}

// distributed.cpp:24-51 (argument checks done on the host)
__global__ void __launch_bounds__(kPT) estimate_time_kernel(const double* __restrict__ tau, int n,
                                                             long long steps, double* __restrict__ out) {
  __shared__ long long red[kPT / 32];
  __shared__ double s_min[kPT / 32];
  double m = DBL_MAX;
  for (int i = threadIdx.x; i < n; i += blockDim.x) m = fmin(m, tau[i]);
  for (int o = 16; o > 0; o >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) s_min[threadIdx.x >> 5] = m;
  __syncthreads();
  double tau_min = DBL_MAX;
  for (int k = 0; k < (int)(blockDim.x >> 5); ++k) tau_min = fmin(tau_min, s_min[k]);
  double lo = 0.0;
  double hi = tau_min * (double)steps;
  while (count_yields(tau, n, hi, red) < steps) hi *= 2;
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (mid <= lo || mid >= hi) break;
    if (count_yields(tau, n, mid, red) >= steps) hi = mid;
    else lo = mid;
  }
  // snap to the exact member (the smallest floor(hi/tau)*tau in (lo, hi])
  double best = hi;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double c = floor(hi / tau[i]) * tau[i];
    if (c > lo && c < best) best = c;
  }
  for (int o = 16; o > 0; o >>= 1) best = fmin(best, __shfl_xor_sync(0xffffffffu, best, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) s_min[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = hi;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) b = fmin(b, s_min[k]);
    *out = b;
  }
}

// yields per env: #{k >= 1 : double(k) * tau <= bound}, capped at S_max
__global__ void yield_count_kernel(const double* __restrict__ tau, int n, const double* __restrict__ tstar,
                                   long long smax, int32_t* __restrict__ cnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // the bisection's snapped T* can sit an ulp below the S_max-th product
  // k*tau (floor(t/tau) vs k*tau rounding): enumerate with a relative slack;
  // surplus yields beyond S_max are harmless (only sorted[0, S_max) is read)
  const double bound = *tstar * (1.0 + 1e-9);
  long long k = (long long)floor(bound / tau[i]);
  while (k > 0 && (double)k * tau[i] > bound) --k;
  while ((double)(k + 1) * tau[i] <= bound) ++k;
  cnt[i] = (int32_t)min(k, smax);
}
__global__ void yield_write_kernel(const double* __restrict__ tau, int n, const int32_t* __restrict__ cnt,
                                   const int32_t* __restrict__ off, double* __restrict__ y) {
  const int i = blockIdx.x;
  if (i >= n) return;
  const double t = tau[i];
  const int base = off[i];
  for (int k = threadIdx.x; k < cnt[i]; k += blockDim.x) y[base + k] = (double)(k + 1) * t;
}

struct BestRate {
  double rate;
  long long s;
};
__device__ __forceinline__ BestRate better(BestRate a, BestRate b) {
  if (b.rate > a.rate || (b.rate == a.rate && b.s < a.s)) return b;
  return a;
}
__global__ void argmax_rate_kernel(const double* __restrict__ y, long long smax, double lt,
                                   BestRate* __restrict__ part) {
  __shared__ BestRate red[32];
  BestRate b{-1.0, 1};
  for (long long s = 1 + (long long)blockIdx.x * blockDim.x + threadIdx.x; s <= smax;
       s += (long long)gridDim.x * blockDim.x) {
    const double r = (double)s / (y[s - 1] + lt);
    b = better(b, BestRate{r, s});
  }
  for (int o = 16; o > 0; o >>= 1) {
    BestRate q{__shfl_xor_sync(0xffffffffu, b.rate, o), __shfl_xor_sync(0xffffffffu, b.s, o)};
    b = better(b, q);
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    BestRate r = red[0];
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) r = better(r, red[k]);
    part[blockIdx.x] = r;
  }
}
__global__ void argmax_final_kernel(const BestRate* __restrict__ part, int n, long long* __restrict__ out) {
  BestRate r = part[0];
  for (int k = 1; k < n; ++k) r = better(r, part[k]);
  *out = r.s;
}

static void check_tau(const double* tau, int n) {
  if (n <= 0) protocol_error("estimate_time: no step-time estimates");
  for (int i = 0; i < n; ++i)
    if (!(tau[i] > 0)) protocol_error("estimate_time: non-positive step time");
}

static double estimate_time(Ctx* c, const double* tau, int n, long long smax, long long steps) {
  if (steps < 0 || steps > smax) protocol_error("estimate_time: S out of range [0, S_max]");
  if (steps == 0) return 0.0;
  check_tau(tau, n);
  DBuf<double> d;
  d.reserve(c, (size_t)n + 1);
  double* pin = static_cast<double*>(c->pinned_buf(sizeof(double) * ((size_t)n + 1)));
  std::copy(tau, tau + n, pin);
  d.upload(pin, n);
  estimate_time_kernel<<<1, kPT, 0, c->stream>>>(d.p, n, steps, d.p + n);
  after_launch(c);
  VER_CUDA(cudaMemcpyAsync(pin + n, d.p + n, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  return pin[n];
}

static long long optimal_preempt_steps(Ctx* c, const double* tau, int n, double lt, long long smax) {
  if (!(lt > 0)) protocol_error("optimal_preempt_steps: LT must be positive");
  if (smax < 1) return 1;
  check_tau(tau, n);
  DBuf<double> d;
  d.reserve(c, (size_t)n + 1);
  double* pin = static_cast<double*>(c->pinned_buf(sizeof(double) * ((size_t)n + 2)));
  std::copy(tau, tau + n, pin);
  d.upload(pin, n);
  estimate_time_kernel<<<1, kPT, 0, c->stream>>>(d.p, n, smax, d.p + n);
  after_launch(c);
  DBuf<int32_t> cnt, off;
  cnt.reserve(c, (size_t)n);
  off.reserve(c, (size_t)n + 1);
  yield_count_kernel<<<cdiv(n, 256), 256, 0, c->stream>>>(d.p, n, d.p + n, smax, cnt.p);
  after_launch(c);
  exclusive_scan_i32(c, cnt.p, off.p, n, off.p + n);
  int32_t* htot = static_cast<int32_t*>(static_cast<void*>(pin + n + 1));
  VER_CUDA(cudaMemcpyAsync(htot, off.p + n, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  const long long Y = *htot;
  if (Y < smax) protocol_error("optimal_preempt_steps: yield enumeration short of S_max");
  DBuf<double> y;
  y.reserve(c, Y);
  yield_write_kernel<<<n, 128, 0, c->stream>>>(d.p, n, cnt.p, off.p, y.p);
  after_launch(c);
  sort_pos_f64(c, y.p, Y);
  const int nb = std::min<long long>(4 * c->num_sms, (smax + 255) / 256);
  DBuf<BestRate> part;
  part.reserve(c, nb);
  DBuf<long long> res;
  res.reserve(c, 1);
  argmax_rate_kernel<<<nb, 256, 0, c->stream>>>(y.p, smax, lt, part.p);
  after_launch(c);
  argmax_final_kernel<<<1, 1, 0, c->stream>>>(part.p, nb, res.p);
  after_launch(c);
  long long* hres = reinterpret_cast<long long*>(pin);
  res.download(hres, 1);
  sync(c);
  return *hres;
}

}  // namespace verg

using namespace verg;

extern "C" {

ver_status ver_estimate_time(ver_ctx ctx, const double* tau, int n, int64_t max_steps, int64_t steps,
                             double* out) {
  VER_API_BEGIN
  activate(&ctx->c);
  *out = estimate_time(&ctx->c, tau, n, max_steps, steps);
  VER_API_END
}

ver_status ver_optimal_preempt_steps(ver_ctx ctx, const double* tau, int n, double learn_time, int64_t max_steps,
                                     int64_t* out) {
  VER_API_BEGIN
  activate(&ctx->c);
  *out = optimal_preempt_steps(&ctx->c, tau, n, learn_time, max_steps);
  VER_API_END
}

}  // extern "C"
