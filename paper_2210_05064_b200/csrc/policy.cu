// policy.cu — policy/value network forward + backward, fused PPO loss, Adam.
//
// GEMMs (parity mode): a tiled fp32 SIMT GEMM (128x128x8 tiles, 8x8 per
// thread, double-buffered shared memory) with fused epilogues (bias, tanh,
// tanh-gradient, additive term) and deterministic split-K for the weight
// gradients whose K is the packed row count.  fp32 keeps the gradients
// inside the 1e-5 parity bound the north star sets for fp32.
//
// Recurrence (nn.cpp:235-250): per timestep t the rows of t are a prefix of
// the rows of t-1, so h_{t-1}[0:bs_t] is contiguous and one GEMM
// hU = h_{t-1} U (bs_t x 3H) plus a gate kernel advances the whole batch.
// Backward runs the same structure in reverse: a gate-gradient kernel then
// dh_{t-1} = dhU U^T + g*z; the weight gradients dU = Hprev^T dhU,
// dWx = enc^T dpre are then single large GEMMs over all rows.
#include <cmath>
#include <cstring>

#include "policy.cuh"
#include "tc_gemm.cuh"

namespace verg {

// ------------------------------------------------------------- model
Model Model::make(const ver_model_config& c) {
  Model m;
  m.D = c.obs_dim;
  m.E = c.encoder_dim;
  m.H = c.hidden_dim;
  m.continuous = c.action_kind == 1;
  m.A = m.continuous ? c.act_dim : c.num_actions;
  m.AH = m.A + 1;
  if (m.D < 1 || m.E < 1 || m.H < 1 || m.A < 1) config_error("model: dims must be >= 1");
  if (m.AH > 32) config_error("model: at most 31 actions supported by the fused loss");
  if (m.D > 8) config_error("model: obs_dim <= 8 supported by the encoder-gradient kernel");
  const int64_t D = m.D, E = m.E, H = m.H, A = m.A, AH = m.AH;
  int64_t o = 0;
  m.o_w1 = o; o += D * E;
  m.o_b1 = o; o += E;
  m.o_w2 = o; o += E * E;
  m.o_b2 = o; o += E;
  m.o_wx = o; o += E * 3 * H;
  m.o_ux = o; o += H * 3 * H;
  m.o_bx = o; o += 3 * H;
  m.o_wh = o; o += H * AH;
  m.o_bh = o; o += AH;
  m.o_ls = o; o += m.continuous ? A : 0;
  m.P = o;
  // tensors() order (nn.cpp:83-95) -> device index
  m.dev_index.resize(m.P);
  int64_t k = 0;
  auto put = [&](int64_t dev) { m.dev_index[k++] = dev; };
  for (int64_t i = 0; i < D * E; ++i) put(m.o_w1 + i);
  for (int64_t i = 0; i < E; ++i) put(m.o_b1 + i);
  for (int64_t i = 0; i < E * E; ++i) put(m.o_w2 + i);
  for (int64_t i = 0; i < E; ++i) put(m.o_b2 + i);
  for (int g = 0; g < 3; ++g) {  // gru_w{r,z,n} (E x H), gru_u{r,z,n} (H x H), gru_b{r,z,n}
    for (int64_t r = 0; r < E; ++r)
      for (int64_t u = 0; u < H; ++u) put(m.o_wx + r * 3 * H + 3 * u + g);
    for (int64_t r = 0; r < H; ++r)
      for (int64_t u = 0; u < H; ++u) put(m.o_ux + r * 3 * H + 3 * u + g);
    for (int64_t u = 0; u < H; ++u) put(m.o_bx + 3 * u + g);
  }
  for (int64_t r = 0; r < H; ++r)
    for (int64_t a = 0; a < A; ++a) put(m.o_wh + r * AH + a);  // head_w
  for (int64_t a = 0; a < A; ++a) put(m.o_bh + a);            // head_b
  for (int64_t r = 0; r < H; ++r) put(m.o_wh + r * AH + A);   // value_w
  put(m.o_bh + A);                                           // value_b
  if (m.continuous)
    for (int64_t a = 0; a < A; ++a) put(m.o_ls + a);  // log_std
  if (k != m.P) config_error("model: layout size mismatch");
  return m;
}

void Workspace::ensure(const Model& m, size_t S, bool train) {
  if (S <= rows && e1.p) return;
  // 1/8 headroom: minibatch row counts vary from split to split, and every growth
  // reallocates gigabytes (the stream-ordered pool maps new memory inside a step)
  const size_t R = std::max<size_t>(S + S / 8, 1);
  const size_t E = m.E, H = m.H;
  e1.reserve(ctx, R * E);
  enc.reserve(ctx, R * E);
  xp.reserve(ctx, R * 3 * H);
  hu.reserve(ctx, R * H);  // hUn (the n-gate recurrent term) for the backward
  gates.reserve(ctx, R * 3 * H);
  hidden.reserve(ctx, R * H);
  hprev.reserve(ctx, R * H);
  if (train) {
    dhidden.reserve(ctx, R * H);
    dhead.reserve(ctx, R * m.AH);
    g.reserve(ctx, R * H);
    dpre.reserve(ctx, R * 3 * H);
    dhu.reserve(ctx, R * 3 * H);
    carry.reserve(ctx, R * H);
    dpre2.reserve(ctx, R * E);
    dpre1.reserve(ctx, R * E);
    is_w.reserve(ctx, R);
  }
  rows = R;
}

// -------------------------------------------------------------- GEMM
constexpr int BM = 128, BN = 128, BK = 8, GT = 256;

template <bool TA, bool TB, class Epi>
__global__ void __launch_bounds__(GT) sgemm_kernel(int M, int N, int K, const float* __restrict__ A,
                                                   int lda, const float* __restrict__ B, int ldb, Epi epi,
                                                   int kchunk) {
  __shared__ __align__(16) float As[2][BK][BM];
  __shared__ __align__(16) float Bs[2][BK][BN];
  const int tid = threadIdx.x;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int kb = blockIdx.z * kchunk;
  const int ke = min(K, kb + kchunk);
  const int tx = tid & 15, ty = tid >> 4;
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
  float ra[4], rb[4];
  auto load = [&](int k0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int idx = tid * 4 + q;
      int m, k;
      if (!TA) {
        m = idx / BK;
        k = idx % BK;
      } else {
        k = idx / BM;
        m = idx % BM;
      }
      const int gm = m0 + m, gk = k0 + k;
      ra[q] = (gm < M && gk < ke) ? (TA ? A[(size_t)gk * lda + gm] : A[(size_t)gm * lda + gk]) : 0.f;
      int n;
      if (!TB) {
        k = idx / BN;
        n = idx % BN;
      } else {
        n = idx / BK;
        k = idx % BK;
      }
      const int gn = n0 + n, gk2 = k0 + k;
      rb[q] = (gn < N && gk2 < ke) ? (TB ? B[(size_t)gn * ldb + gk2] : B[(size_t)gk2 * ldb + gn]) : 0.f;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int idx = tid * 4 + q;
      if (!TA) As[buf][idx % BK][idx / BK] = ra[q];
      else As[buf][idx / BM][idx % BM] = ra[q];
      if (!TB) Bs[buf][idx / BN][idx % BN] = rb[q];
      else Bs[buf][idx % BK][idx / BK] = rb[q];
    }
  };
  const int nk = ke > kb ? (ke - kb + BK - 1) / BK : 0;
  if (nk > 0) {
    load(kb);
    store(0);
  }
  __syncthreads();
  for (int it = 0; it < nk; ++it) {
    const int buf = it & 1;
    if (it + 1 < nk) load(kb + (it + 1) * BK);
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][k][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][k][64 + ty * 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][k][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][k][64 + tx * 4]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    if (it + 1 < nk) store(buf ^ 1);
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int n = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
      if (n < N) epi(m, n, acc[i][j], blockIdx.z);
    }
  }
}

// split-K partials of the tail rows summed in a fixed order, then the GEMM's epilogue
template <class Epi>
__global__ void tail_reduce_kernel(const float* __restrict__ W, int Z, int M, int N, Epi epi) {
  pdl_wait();
  pdl_trigger();
  const int64_t i4 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (4 * i4 >= (int64_t)M * N) return;
  const int64_t i = 4 * i4;
  const size_t MN = (size_t)M * N;
  float4 s = __ldcg(reinterpret_cast<const float4*>(W + i));
  for (int z = 1; z < Z; ++z) {
    const float4 v = __ldcg(reinterpret_cast<const float4*>(W + (size_t)z * MN + i));
    s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
  }
  epi.vec4((int)(i / N), (int)(i % N), s, 0);
}

// lo = x - trunc_tf32(x) of every parameter, once per forward: the weights'
// 3xTF32 lo operand then comes in by TMA instead of being split per stage
__global__ void split_lo_kernel(int64_t n, const float* __restrict__ x, float* __restrict__ lo) {
  pdl_wait();
  pdl_trigger();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) lo[i] = tc::lo1(x[i]);
}

// ---------------------------------------------------------------- fp16x2 operands
// x s = hi + lo with hi = fp16_rn(x s), lo = fp16_rn(x s - hi) (22 significant
// bits; tc_gemm.cuh F16).  Activations that are tanh outputs (|x| < 1) use the
// fixed scale 2^14; a weight's scale is 2^(14 - floor(log2 max|w|)), so that
// max |w| s < 2^15 < 65504 and its small entries stay normal for ~28 binades.
constexpr float kActScale = 16384.f;  // 2^14
__device__ __forceinline__ void split_h2(float y, __half& hi, __half& lo) {
  hi = __float2half_rn(y);
  lo = __float2half_rn(y - __half2float(hi));
}
__global__ void maxabs_kernel(int64_t n, const float* __restrict__ x, unsigned* __restrict__ out) {
  pdl_wait();
  float m = 0.f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = fmaxf(m, fabsf(x[i]));
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(m));  // non-negative floats order as uints
}
__device__ __forceinline__ float weight_scale(unsigned maxbits) {
  const float mx = __uint_as_float(maxbits);
  if (!(mx > 0.f) || !isfinite(mx)) return 1.f;
  return exp2f((float)(14 - ilogbf(mx)));
}
// W: K x N row-major (the MN-major B of x W) -> Wt hi / lo: N x K row-major; 32 x 32
// tiles through shared memory.  inv = 1 / (2^14 s_W) for the GEMM epilogue.
__global__ void __launch_bounds__(256) weight_f16x2_kernel(const float* __restrict__ W, int K, int N,
                                                           const unsigned* __restrict__ maxbits, __half* __restrict__ hi,
                                                           __half* __restrict__ lo, float* __restrict__ inv,
                                                           float act_scale) {
  __shared__ float t[32][33];
  const float s = weight_scale(*maxbits);
  const int k0 = blockIdx.y * 32, n0 = blockIdx.x * 32;
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int k = k0 + r, n = n0 + threadIdx.x;
    t[r][threadIdx.x] = (k < K && n < N) ? W[(size_t)k * N + n] : 0.f;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int n = n0 + r, k = k0 + threadIdx.x;
    if (n < N && k < K) split_h2(t[threadIdx.x][r] * s, hi[(size_t)n * K + k], lo[(size_t)n * K + k]);
  }
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0 && threadIdx.y == 0) *inv = 1.f / (act_scale * s);
}
// fp16x2 forward GEMMs (VER_TC_F16=0 restores 3xTF32 for them)
static bool f16x2_on(const Ctx* c) { return c->precision == 0 && c->tensor_cores && env_int("VER_TC_F16", 1) != 0; }
// the weight copies of the fp16x2 forward GEMMs (transposed to K-major): slot 0
// wx (3H x E), slot 1 w2 (E x E), slot 2 ux (3H x H, the recurrent forward step
// GEMMs, activation scale 2^13); w16hi / w16lo hold them back to back
// slots 3 / 4: wx (E x 3H) and w2 (E x E) as they lie (K-major B of the backward
// data-gradient GEMMs, fp16x2 with the gradient converted in-kernel), inv = 1 / s_W
__global__ void weight_f16x2_plain_kernel(int64_t n, const float* __restrict__ W,
                                          const unsigned* __restrict__ maxbits, __half* __restrict__ hi,
                                          __half* __restrict__ lo, float* __restrict__ inv) {
  const float s = weight_scale(*maxbits);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    split_h2(W[i] * s, hi[i], lo[i]);
  if (blockIdx.x == 0 && threadIdx.x == 0) *inv = 1.f / s;
}
void refresh_weights_f16(Ctx* c, const Model& m, const float* params, Workspace& ws) {
  const int E = m.E, H = m.H, H3 = 3 * H;
  const size_t n0 = (size_t)H3 * E, n1 = (size_t)E * E, n2 = (size_t)H3 * H;
  ws.w16hi.reserve(c, 2 * (n0 + n1) + n2);
  ws.w16lo.reserve(c, 2 * (n0 + n1) + n2);
  ws.w16max.reserve(c, 3);
  ws.w16inv.reserve(c, 5);
  ws.w16max.zero(3);
  maxabs_kernel<<<64, 256, 0, c->stream>>>((int64_t)E * H3, params + m.o_wx, ws.w16max.p);
  after_launch(c);
  maxabs_kernel<<<64, 256, 0, c->stream>>>((int64_t)E * E, params + m.o_w2, ws.w16max.p + 1);
  after_launch(c);
  maxabs_kernel<<<64, 256, 0, c->stream>>>((int64_t)H * H3, params + m.o_ux, ws.w16max.p + 2);
  after_launch(c);
  weight_f16x2_kernel<<<dim3(cdiv(H3, 32), cdiv(E, 32)), dim3(32, 8), 0, c->stream>>>(
      params + m.o_wx, E, H3, ws.w16max.p, ws.w16hi.p, ws.w16lo.p, ws.w16inv.p, kActScale);
  after_launch(c);
  weight_f16x2_kernel<<<dim3(cdiv(E, 32), cdiv(E, 32)), dim3(32, 8), 0, c->stream>>>(
      params + m.o_w2, E, E, ws.w16max.p + 1, ws.w16hi.p + n0, ws.w16lo.p + n0, ws.w16inv.p + 1, kActScale);
  after_launch(c);
  weight_f16x2_kernel<<<dim3(cdiv(H3, 32), cdiv(H, 32)), dim3(32, 8), 0, c->stream>>>(
      params + m.o_ux, H, H3, ws.w16max.p + 2, ws.w16hi.p + n0 + n1, ws.w16lo.p + n0 + n1, ws.w16inv.p + 2,
      1.f);  // 1 / s_U: the step kernel divides by h's scale, set per launch from max |h0|
  after_launch(c);
  const size_t o3 = n0 + n1 + n2, o4 = o3 + n0;
  weight_f16x2_plain_kernel<<<(unsigned)cdiv(n0, 256), 256, 0, c->stream>>>((int64_t)n0, params + m.o_wx, ws.w16max.p,
                                                                           ws.w16hi.p + o3, ws.w16lo.p + o3,
                                                                           ws.w16inv.p + 3);
  after_launch(c);
  weight_f16x2_plain_kernel<<<(unsigned)cdiv(n1, 256), 256, 0, c->stream>>>((int64_t)n1, params + m.o_w2,
                                                                           ws.w16max.p + 1, ws.w16hi.p + o4,
                                                                           ws.w16lo.p + o4, ws.w16inv.p + 4);
  after_launch(c);
}
template <bool TA, bool TB, class Epi>
static void gemm(Ctx* c, int M, int N, int K, const float* A, int lda, const float* B, int ldb, Epi epi,
                 const float* Blo = nullptr) {
  if (M <= 0 || N <= 0) return;
  if (c->tensor_cores && tc::usable(M, N, K, A, lda, B, ldb, epi)) {
    // op(A): TA ? MN-major : K-major;  op(B): TB ? K-major : MN-major
    // Tail split: when the last wave of output tiles would leave most SMs idle,
    // the last m-tiles run as a second launch split two ways along K (twice as
    // many half-size items fill that wave), reduced with the same epilogue.
    const tc::Geo g = tc::geo(c, M, N);
    const int tilesN = (int)cdiv(N, g.bn), tilesM = (int)cdiv(M, g.bm);
    const long long tiles = (long long)tilesN * tilesM, sms = g.units;
    const long long rem = tiles % sms;
    const int tail_mt = (int)cdiv(rem, tilesN);
    const int nkb = (K + tc::BK - 1) / tc::BK;
    if (c->precision == 0 && tiles > sms && rem > 0 && 10 * rem < 6 * sms &&
        tail_mt < tilesM && nkb >= 32 && N % 4 == 0) {  // K < 1024: half a wave saves less than the extra launches
      const int M1 = (tilesM - tail_mt) * g.bm, M2 = M - M1;
      tc::launch<TA ? 1 : 0, TB ? 0 : 1>(c, M1, N, K, A, lda, B, ldb, epi, 1, Blo);
      const float* A2 = TA ? A + M1 : A + (size_t)M1 * lda;
      float* W = nullptr;
      VER_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&W), sizeof(float) * 2 * (size_t)M2 * N, c->stream));
      tc::launch<TA ? 1 : 0, TB ? 0 : 1>(c, M2, N, K, A2, lda, B, ldb, EpiPartial{W, M2, N}, 2, Blo);
      launch_pdl(c, tail_reduce_kernel<Epi>, dim3(cdiv((size_t)M2 * N / 4, 256)), dim3(256), 0, (const float*)W, 2,
                 M2, N, epi.shifted(M1));
      VER_CUDA(cudaFreeAsync(W, c->stream));
      return;
    }
    tc::launch<TA ? 1 : 0, TB ? 0 : 1>(c, M, N, K, A, lda, B, ldb, epi, 1, Blo);
    return;
  }
  dim3 grid(cdiv(N, BN), cdiv(M, BM), 1);
  sgemm_kernel<TA, TB, Epi><<<grid, GT, 0, c->stream>>>(M, N, K, A, lda, B, ldb, epi, std::max(K, 1));
  after_launch(c);
}

__global__ void splitk_reduce_kernel(const float* __restrict__ W, int Z, int M, int N, float* __restrict__ C,
                                     int ldc) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)M * N) return;
  const int m = (int)(i / N), n = (int)(i % N);
  float s = 0.f;
  for (int z = 0; z < Z; ++z) s += W[(size_t)z * M * N + i];
  C[(size_t)m * ldc + n] = s;
}

// float4 variant (N % 4 == 0): 4 outputs per thread, the Z partial loads of a
// group of 4 splits issued together (the partials are L2-resident)
__global__ void splitk_reduce4_kernel(const float* __restrict__ W, int Z, int M, int N, float* __restrict__ C,
                                      int ldc, int vec_store) {
  pdl_wait();
  pdl_trigger();
  const int64_t i4 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (4 * i4 >= (int64_t)M * N) return;
  const int64_t i = 4 * i4;
  const int m = (int)(i / N), n = (int)(i % N);
  const size_t MN = (size_t)M * N;
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  int z = 0;
  for (; z + 4 <= Z; z += 4) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldcg(reinterpret_cast<const float4*>(W + (size_t)(z + u) * MN + i));
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      s.x += v[u].x; s.y += v[u].y; s.z += v[u].z; s.w += v[u].w;
    }
  }
  for (; z < Z; ++z) {
    const float4 v = __ldcg(reinterpret_cast<const float4*>(W + (size_t)z * MN + i));
    s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
  }
  float* out = C + (size_t)m * ldc + n;
  if (vec_store) {
    *reinterpret_cast<float4*>(out) = s;
  } else {
    out[0] = s.x; out[1] = s.y; out[2] = s.z; out[3] = s.w;
  }
}

// C (M x N, ldc) = op(A) op(B) with deterministic split-K over K.
template <bool TA, bool TB>
static void gemm_splitk(Ctx* c, Workspace& ws, int M, int N, int K, const float* A, int lda, const float* B,
                        int ldb, float* C, int ldc) {
  if (M <= 0 || N <= 0) return;
  if (c->tensor_cores && tc::usable(M, N, K, A, lda, B, ldb, EpiStore{C, ldc})) {
    int Z = tc::splits_for(c, M, N, K);
    if (Z == 1) {
      tc::launch<TA ? 1 : 0, TB ? 0 : 1>(c, M, N, K, A, lda, B, ldb, EpiStore{C, ldc}, 1);
      return;
    }
    const int nkb = (K + tc::BK - 1) / tc::BK;
    const int per = (nkb + Z - 1) / Z;
    Z = (nkb + per - 1) / per;
    ws.splitk.reserve(c, (size_t)Z * M * N);
    tc::launch<TA ? 1 : 0, TB ? 0 : 1>(c, M, N, K, A, lda, B, ldb, EpiPartial{ws.splitk.p, M, N}, Z);
    if (N % 4 == 0) {
      const int vs = (ldc % 4 == 0 && (reinterpret_cast<uintptr_t>(C) & 15) == 0) ? 1 : 0;
      launch_pdl(c, splitk_reduce4_kernel, dim3(cdiv((size_t)M * N / 4, 256)), dim3(256), 0,
                 (const float*)ws.splitk.p, Z, M, N, C, ldc, vs);
      return;
    } else {
      splitk_reduce_kernel<<<cdiv((size_t)M * N, 256), 256, 0, c->stream>>>(ws.splitk.p, Z, M, N, C, ldc);
    }
    after_launch(c);
    return;
  }
  const int tiles = (int)(cdiv(N, BN) * cdiv(M, BM));
  int Z = std::max(1, std::min((2 * c->num_sms + tiles - 1) / tiles, (int)cdiv(K, 256)));
  Z = std::min(Z, 64);
  if (Z == 1) {
    gemm<TA, TB>(c, M, N, K, A, lda, B, ldb, EpiStore{C, ldc});
    return;
  }
  const int kchunk = (int)((cdiv(K, Z) + BK - 1) / BK) * BK;
  Z = (int)cdiv(K, kchunk);
  ws.splitk.reserve(c, (size_t)Z * M * N);
  dim3 grid(cdiv(N, BN), cdiv(M, BM), Z);
  sgemm_kernel<TA, TB, EpiPartial><<<grid, GT, 0, c->stream>>>(M, N, K, A, lda, B, ldb,
                                                                EpiPartial{ws.splitk.p, M, N}, kchunk);
  after_launch(c);
  splitk_reduce_kernel<<<cdiv((size_t)M * N, 256), 256, 0, c->stream>>>(ws.splitk.p, Z, M, N, C, ldc);
  after_launch(c);
}

// column sums out[n] = sum_m X[m, n] (deterministic two-stage)
__global__ void colsum_partial_kernel(const float* __restrict__ X, int M, int N, int ld, int rows_per,
                                      float* __restrict__ part) {
  __shared__ float red[8][33];
  const int n = blockIdx.x * 32 + (threadIdx.x & 31);
  const int r = threadIdx.x >> 5;
  const int m0 = blockIdx.y * rows_per, m1 = min(M, m0 + rows_per);
  float s = 0.f;
  if (n < N)
    for (int m = m0 + r; m < m1; m += 8) s += X[(size_t)m * ld + n];
  red[r][threadIdx.x & 31] = s;
  __syncthreads();
  if (r == 0 && n < N) {
    float t = 0.f;
    for (int k = 0; k < 8; ++k) t += red[k][threadIdx.x & 31];
    part[(size_t)blockIdx.y * N + n] = t;
  }
}
__global__ void colsum_final_kernel(const float* __restrict__ part, int chunks, int N, float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  float s = 0.f;
  for (int k = 0; k < chunks; ++k) s += part[(size_t)k * N + n];
  out[n] = s;
}
// float4 variant (N, ld multiples of 4, X 16-byte aligned): a block covers 128
// columns (lane: 4 columns) and a row chunk; each warp walks every 8th row with
// 4 independent accumulators, so ~2 KB per warp are in flight (HBM-bound)
// (maxout: also max |X| into *maxout as float bits -- the fp16x2 scale of X as the
// next GEMM's operand, taken on the same pass)
__global__ void __launch_bounds__(256) colsum4_partial_kernel(const float* __restrict__ X, int M, int N, int ld,
                                                              int rows_per, float* __restrict__ part,
                                                              unsigned* __restrict__ maxout) {
  pdl_wait();
  pdl_trigger();
  __shared__ float4 red[8][32];
  const int lane = threadIdx.x & 31, r = threadIdx.x >> 5;
  const int n = blockIdx.x * 128 + 4 * lane;
  const int m0 = blockIdx.y * rows_per, m1 = min(M, m0 + rows_per);
  float4 a[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) a[u] = make_float4(0.f, 0.f, 0.f, 0.f);
  float mxu[4] = {0.f, 0.f, 0.f, 0.f};  // one running max per unrolled row (no serial chain)
  if (n < N) {
    int m = m0 + r;
    for (; m + 24 < m1; m += 32) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float4 x = __ldg(reinterpret_cast<const float4*>(X + (size_t)(m + 8 * u) * ld + n));
        a[u].x += x.x; a[u].y += x.y; a[u].z += x.z; a[u].w += x.w;
        if (maxout) mxu[u] = fmaxf(mxu[u], fmaxf(fmaxf(fabsf(x.x), fabsf(x.y)), fmaxf(fabsf(x.z), fabsf(x.w))));
      }
    }
    for (; m < m1; m += 8) {
      const float4 x = __ldg(reinterpret_cast<const float4*>(X + (size_t)m * ld + n));
      a[0].x += x.x; a[0].y += x.y; a[0].z += x.z; a[0].w += x.w;
      if (maxout) mxu[0] = fmaxf(mxu[0], fmaxf(fmaxf(fabsf(x.x), fabsf(x.y)), fmaxf(fabsf(x.z), fabsf(x.w))));
    }
  }
  if (maxout) {  // (fmaxf drops NaN: a NaN gradient is caught by the finite checks, not by the scale)
    float mx = fmaxf(fmaxf(mxu[0], mxu[1]), fmaxf(mxu[2], mxu[3]));
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) atomicMax(maxout, __float_as_uint(mx));
  }
  red[r][lane] = make_float4((a[0].x + a[1].x) + (a[2].x + a[3].x), (a[0].y + a[1].y) + (a[2].y + a[3].y),
                             (a[0].z + a[1].z) + (a[2].z + a[3].z), (a[0].w + a[1].w) + (a[2].w + a[3].w));
  __syncthreads();
  if (r == 0 && n < N) {
    float4 t = red[0][lane];
#pragma unroll
    for (int k = 1; k < 8; ++k) {
      const float4 q = red[k][lane];
      t.x += q.x; t.y += q.y; t.z += q.z; t.w += q.w;
    }
    *reinterpret_cast<float4*>(part + (size_t)blockIdx.y * N + n) = t;
  }
}

static void colsum(Ctx* c, Workspace& ws, const float* X, int M, int N, int ld, float* out,
                   unsigned* maxout = nullptr) {
  if (N % 4 == 0 && ld % 4 == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0) {
    const int col_blocks = (int)cdiv(N, 128);
    int rows_per = 256;
    while ((int64_t)col_blocks * cdiv(M, rows_per) > 4 * c->num_sms && rows_per < 8192) rows_per *= 2;
    const int chunks = std::max(1, (int)cdiv(M, rows_per));
    ws.splitk.reserve(c, (size_t)chunks * N);
    launch_pdl(c, colsum4_partial_kernel, dim3(col_blocks, chunks), dim3(256), 0, X, M, N, ld, rows_per, ws.splitk.p,
               maxout);
    launch_pdl(c, colsum_final_kernel, dim3(cdiv(N, 256)), dim3(256), 0, (const float*)ws.splitk.p, chunks, N, out);
    return;
  }
  // enough row chunks for ~4 blocks per SM: each thread walks rows_per / 8 rows
  const int col_blocks = (int)cdiv(N, 32);
  int rows_per = 64;
  while ((int64_t)col_blocks * cdiv(M, rows_per) > 4 * c->num_sms && rows_per < 4096) rows_per *= 2;
  const int chunks = std::max(1, (int)cdiv(M, rows_per));
  ws.splitk.reserve(c, (size_t)chunks * N);
  dim3 grid(cdiv(N, 32), chunks);
  colsum_partial_kernel<<<grid, 256, 0, c->stream>>>(X, M, N, ld, rows_per, ws.splitk.p);
  after_launch(c);
  colsum_final_kernel<<<cdiv(N, 256), 256, 0, c->stream>>>(ws.splitk.p, chunks, N, out);
  after_launch(c);
}

constexpr int kMaxD = 8;  // obs_dim bound of the encoder-input kernels (Model::make checks it)

// ----------------------------------------------------------- forward
// e1 = tanh(obs w1 + b1)  (K = D is tiny: direct).  Write-bound (4E bytes per row):
// block (32 x 8), each thread 4 consecutive features (w1 / b1 columns in registers,
// one float4 store per row) and 4 rows in flight per iteration
__global__ void __launch_bounds__(256) enc1_kernel(const float* __restrict__ obs, int S, int D, int E,
                                                   const float* __restrict__ w1, const float* __restrict__ b1,
                                                   float* __restrict__ e1, __half* __restrict__ e1hi,
                                                   __half* __restrict__ e1lo) {
  pdl_wait();
  pdl_trigger();
  const int k = 4 * (blockIdx.x * 32 + threadIdx.x);
  if (k >= E) return;
  float4 w[kMaxD];
#pragma unroll
  for (int d = 0; d < kMaxD; ++d)
    w[d] = d < D ? *reinterpret_cast<const float4*>(w1 + (size_t)d * E + k) : make_float4(0.f, 0.f, 0.f, 0.f);
  const float4 b = *reinterpret_cast<const float4*>(b1 + k);
  const int stride = gridDim.y * blockDim.y;
  for (int p0 = blockIdx.y * blockDim.y + threadIdx.y; p0 < S; p0 += 4 * stride) {
    float4 s[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int p = min(p0 + u * stride, S - 1);
      s[u] = make_float4(0.f, 0.f, 0.f, 0.f);  // same order as the scalar kernel: bias last
#pragma unroll
      for (int d = 0; d < kMaxD; ++d)
        if (d < D) {
          const float o = __ldg(obs + (size_t)p * D + d);
          s[u].x = fmaf(o, w[d].x, s[u].x);
          s[u].y = fmaf(o, w[d].y, s[u].y);
          s[u].z = fmaf(o, w[d].z, s[u].z);
          s[u].w = fmaf(o, w[d].w, s[u].w);
        }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int p = p0 + u * stride;
      if (p < S) {
        const float4 y = make_float4(gate_tanh(s[u].x + b.x), gate_tanh(s[u].y + b.y), gate_tanh(s[u].z + b.z),
                                     gate_tanh(s[u].w + b.w));
        *reinterpret_cast<float4*>(e1 + (size_t)p * E + k) = y;
        if (e1hi) {  // fp16x2 halves for the next GEMM (scale 2^14)
          const float ys[4] = {y.x * 16384.f, y.y * 16384.f, y.z * 16384.f, y.w * 16384.f};
          __half h[4], l[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            h[q] = __float2half_rn(ys[q]);
            l[q] = __float2half_rn(ys[q] - __half2float(h[q]));
          }
          __half2* hp = reinterpret_cast<__half2*>(e1hi + (size_t)p * E + k);
          __half2* lp = reinterpret_cast<__half2*>(e1lo + (size_t)p * E + k);
          hp[0] = __halves2half2(h[0], h[1]);
          hp[1] = __halves2half2(h[2], h[3]);
          lp[0] = __halves2half2(l[0], l[1]);
          lp[1] = __halves2half2(l[2], l[3]);
        }
      }
    }
  }
}

// the scalar kernel above for E % 4 != 0 (float4 columns need E % 4 == 0)
__global__ void __launch_bounds__(256) enc1_scalar_kernel(const float* __restrict__ obs, int S, int D, int E,
                                                          const float* __restrict__ w1, const float* __restrict__ b1,
                                                          float* __restrict__ e1) {
  pdl_wait();
  pdl_trigger();
  const int k = blockIdx.x * 32 + threadIdx.x;
  if (k >= E) return;
  float w[kMaxD];
#pragma unroll
  for (int d = 0; d < kMaxD; ++d) w[d] = d < D ? w1[(size_t)d * E + k] : 0.f;
  const float b = b1[k];
  for (int p = blockIdx.y * blockDim.y + threadIdx.y; p < S; p += gridDim.y * blockDim.y) {
    float s = 0.f;
#pragma unroll
    for (int d = 0; d < kMaxD; ++d)
      if (d < D) s = fmaf(__ldg(obs + (size_t)p * D + d), w[d], s);
    e1[(size_t)p * E + k] = gate_tanh(s + b);
  }
}


void policy_forward(Ctx* c, const Model& m, const float* params, int S, const float* obs, const float* h0,
                    int L, const int32_t* d_bs, const int32_t* d_offs, Workspace& ws, bool store,
                    const int32_t* h_bs, const int32_t* h_offs) {
  const int E = m.E, H3 = 3 * m.H;
  const bool f16 = f16x2_on(c) && tc::usable_f16(S, H3, E, E, E) && tc::usable_f16(S, E, E, E, E) &&
                   EpiBias{ws.xp.p, H3, params + m.o_bx}.vec_ok() && E % 8 == 0;
  const size_t nSE = (size_t)S * E;
  if (f16) {  // e1's halves at [0, nSE), enc's at [nSE, 2 nSE) (sized by the workspace rows)
    const size_t cap = 2 * std::max(ws.rows, (size_t)S) * E;
    ws.a16hi.reserve(c, cap);
    ws.a16lo.reserve(c, cap);
  }
  if (E % 4 == 0) {
    const unsigned gx = cdiv(E, 128);
    dim3 g(gx, std::max(1u, std::min(cdiv(S, 32), (unsigned)(8 * c->num_sms / gx))));
    launch_pdl(c, enc1_kernel, g, dim3(32, 8), 0, obs, S, m.D, E, params + m.o_w1, params + m.o_b1, ws.e1.p,
               f16 ? ws.a16hi.p : nullptr, f16 ? ws.a16lo.p : nullptr);
  } else {
    dim3 g(cdiv(E, 32), std::max(1u, std::min(cdiv(S, 8), (unsigned)(8 * c->num_sms / std::max(1u, cdiv(E, 32))))));
    launch_pdl(c, enc1_scalar_kernel, g, dim3(32, 8), 0, obs, S, m.D, E, params + m.o_w1, params + m.o_b1, ws.e1.p);
  }
  if (ws.wlo_stale || ws.wlo_src != params || ws.wlo.n < (size_t)m.P) {
    ws.wlo.reserve(c, m.P);
    launch_pdl(c, split_lo_kernel, dim3(cdiv(m.P, 256)), dim3(256), 0, (int64_t)m.P, params, ws.wlo.p);
    if (f16) refresh_weights_f16(c, m, params, ws);
    ws.wlo_src = params;
  } else if (f16 && ws.w16inv.n < 5) {
    refresh_weights_f16(c, m, params, ws);
  }
  ws.wlo_stale = !ws.wlo_keep;
  ws.f16_fwd = f16;
  if (f16) {
    // fp16x2: e1 and enc are tanh outputs (fixed scale), the weights' copies are
    // transposed to K-major
    // (the enc1 kernel and the enc2 epilogue write the halves next to the fp32 rows)
    const size_t nW = (size_t)H3 * E;
    tc::launch_f16(c, S, E, E, ws.a16hi.p, ws.a16lo.p, E, ws.w16hi.p + nW, ws.w16lo.p + nW, E, ws.w16inv.p + 1,
                   EpiBiasTanhH{ws.enc.p, E, params + m.o_b2, ws.a16hi.p + nSE, ws.a16lo.p + nSE}, 1);
    tc::launch_f16(c, S, H3, E, ws.a16hi.p + nSE, ws.a16lo.p + nSE, E, ws.w16hi.p, ws.w16lo.p, E, ws.w16inv.p,
                   EpiBias{ws.xp.p, H3, params + m.o_bx}, 1);
  } else {
    gemm<false, false>(c, S, E, E, ws.e1.p, E, params + m.o_w2, E, EpiBiasTanh{ws.enc.p, E, params + m.o_b2},
                       ws.wlo.p + m.o_w2);
    gemm<false, false>(c, S, H3, E, ws.enc.p, E, params + m.o_wx, H3, EpiBias{ws.xp.p, H3, params + m.o_bx},
                       ws.wlo.p + m.o_wx);
  }
  gru_forward_recurrence(c, m, params, L, d_bs, d_offs, ws, h0, store, h_bs, h_offs);
}

// ------------------------------------------------ big recurrence steps
// Steps whose batch has >= 150 rows (a prefix of the timesteps: bs is
// non-increasing) run in the persistent tcgen05 step kernel (stepgemm.cu)
// instead of the persistent FMA kernel (recurrence.cu), whose step time grows
// with the rows (~36 us at 623 rows, H = 512).  The threshold was measured on
// B200 at C2 (scripts/ab_bench.py sweeps); VER_REC_BIG_FWD / _BWD override it.
int gru_big_steps(Ctx* c, const Model& m, const int32_t* h_bs, int L, bool backward) {
  if (m.H % 4 != 0) return 0;  // the gate phase moves 4 units per thread
  const int min_rows = backward ? env_int("VER_REC_BIG_BWD", 150) : env_int("VER_REC_BIG_FWD", 150);
  if (!h_bs || !c->tensor_cores || m.H % 32 != 0 || min_rows <= 0) return 0;
  int t = 0;
  while (t < L && h_bs[t] >= min_rows) ++t;
  return t;
}

void policy_heads(Ctx* c, const Model& m, const float* params, int n, const float* hidden, float* out) {
  gemm<false, false>(c, n, m.AH, m.H, hidden, m.H, params + m.o_wh, m.AH,
                     EpiBias{out, m.AH, params + m.o_bh});
}

// per-row heads: warp per row (nn.cpp:251-278)
__global__ void policy_rows_kernel(int S, int H, int A, int continuous, const float* __restrict__ hidden,
                                   const float* __restrict__ wh, const float* __restrict__ bh,
                                   const float* __restrict__ log_std, const int32_t* __restrict__ act_disc,
                                   const float* __restrict__ act_cont, float* __restrict__ logp_out,
                                   float* __restrict__ ent_out, float* __restrict__ value_out) {
  const int lane = threadIdx.x & 31;
  const int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (p >= S) return;
  const int AH = A + 1;
  double lg[32];
  for (int c = 0; c < AH; ++c) {
    float acc = 0.f;
    for (int u = lane; u < H; u += 32) acc = fmaf(hidden[(size_t)p * H + u], wh[(size_t)u * AH + c], acc);
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    lg[c] = (double)acc + (double)bh[c];
  }
  if (lane != 0) return;
  double logp, ent;
  if (!continuous) {
    double mx = lg[0];
    for (int c = 1; c < A; ++c) mx = fmax(mx, lg[c]);
    double se = 0.0;
    for (int c = 0; c < A; ++c) se += exp(lg[c] - mx);
    const double lse = log(se);
    logp = lg[act_disc[p]] - mx - lse;
    ent = 0.0;
    for (int c = 0; c < A; ++c) {
      const double lp = lg[c] - mx - lse;
      ent -= exp(lp) * lp;
    }
  } else {
    double q = 0.0, sls = 0.0;
    for (int c = 0; c < A; ++c) {
      const double ls = log_std[c];
      const double z = ((double)act_cont[(size_t)p * A + c] - lg[c]) * exp(-ls);
      q += z * z;
      sls += ls;
    }
    logp = -0.5 * q - sls - 0.5 * 1.8378770664093453 * A;
    ent = sls + 0.5 * (1.0 + 1.8378770664093453) * A;
  }
  if (logp_out) logp_out[p] = (float)logp;
  if (ent_out) ent_out[p] = (float)ent;
  if (value_out) value_out[p] = (float)lg[A];
}

void policy_rows(Ctx* c, const Model& m, const float* params, int S, const float* hidden,
                 const int32_t* act_disc, const float* act_cont, float* logp, float* ent, float* value) {
  policy_rows_kernel<<<cdiv(S, 8), 256, 0, c->stream>>>(S, m.H, m.A, m.continuous, hidden, params + m.o_wh,
                                                        params + m.o_bh, m.continuous ? params + m.o_ls : nullptr,
                                                        act_disc, act_cont, logp, ent, value);
  after_launch(c);
}

// ---------------------------------------------------------------- loss
constexpr int kLossWarps = 8;
constexpr int kHL = 16;  // fused head gradient: H / 32 <= kHL
constexpr int kLossStats = 8;  // ws, verr2, H, ratio, clip, w, wmax, (pad)
constexpr int kLossRows = 8;   // rows per warp-iteration of ppo_loss_rows_kernel
constexpr double kLog2Pi = 1.8378770664093453;

// One warp per packed row: heads (H -> A+1 dot products), log-softmax /
// Gaussian log-prob, ratio / clip / IS weight / surrogate / value / entropy,
// and the row's head gradient dhead (A+1) and dhidden = dhead wh^T.
// Per-block double partials of the loss statistics (deterministic order).
// NA = A+1 at compile time (common head sizes; every per-head array stays in
// registers), or 32 with a runtime bound (generic instantiation).
template <int NA>
__global__ void __launch_bounds__(kLossWarps * 32, 2) ppo_loss_kernel(
    int S, int H, int A, int continuous, const float* __restrict__ hidden, const float* __restrict__ wh,
    const float* __restrict__ bh, const float* __restrict__ log_std, const float* __restrict__ act_cont,
    const int32_t* __restrict__ act_disc, const float* __restrict__ old_logp, const float* __restrict__ adv,
    const float* __restrict__ ret, const float* __restrict__ frozen_w, double clip, double is_cap,
    double vcoef, const double* __restrict__ alpha_p, double inv_S, float* __restrict__ dhead,
    float* __restrict__ dhidden, float* __restrict__ is_w, double* __restrict__ part, int want_grads,
    float* __restrict__ hpart) {
  extern __shared__ float s_wh[];  // H x AH, then (fused head gradient) H x AH + AH block sums
  __shared__ double s_red[kLossWarps][kLossStats + 32];
  const int AH = A + 1;
  // fused head gradient (H % 32 == 0, H <= 32 kHL): dwh = hidden^T dhead and
  // dbh = colsum(dhead) accumulated per lane from the rows' registers
  const int hl = H / 32;
  const bool fuse = hpart != nullptr;
  float* s_hg = s_wh + H * AH;
  float wacc[kHL][NA], bacc[NA];
#pragma unroll
  for (int i = 0; i < kHL; ++i)
#pragma unroll
    for (int c = 0; c < NA; ++c) wacc[i][c] = 0.f;
#pragma unroll
  for (int c = 0; c < NA; ++c) bacc[c] = 0.f;
  for (int i = threadIdx.x; i < H * AH; i += blockDim.x) s_wh[i] = wh[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double alpha = *alpha_p;
  const double gH = -alpha * inv_S;
  double st[kLossStats] = {0, 0, 0, 0, 0, 0, 0, 0};
  double dls = 0.0;  // lane c < A: log_std gradient (continuous)
  // fused path: the next row's hidden values are loaded while this row is
  // processed (the kernel is bound by that load's latency otherwise)
  const int pstride = gridDim.x * kLossWarps;
  float hn[kHL];
  if (fuse) {
    const int p0 = blockIdx.x * kLossWarps + warp;
#pragma unroll
    for (int i = 0; i < kHL; ++i) hn[i] = (p0 < S && i < hl) ? __ldcs(hidden + (size_t)p0 * H + lane + 32 * i) : 0.f;
  }
  for (int p = blockIdx.x * kLossWarps + warp; p < S; p += pstride) {
    const float* hrow = hidden + (size_t)p * H;
    float acc[NA];
#pragma unroll
    for (int c = 0; c < NA; ++c) acc[c] = 0.f;
    float hv[kHL];
    if (fuse) {
#pragma unroll
      for (int i = 0; i < kHL; ++i) hv[i] = hn[i];
      const int pn = p + pstride;
#pragma unroll
      for (int i = 0; i < kHL; ++i) hn[i] = (pn < S && i < hl) ? __ldcs(hidden + (size_t)pn * H + lane + 32 * i) : 0.f;
      // NA independent partial sums per lane, 2 chains each
      float acc2[NA];
#pragma unroll
      for (int c = 0; c < NA; ++c) acc2[c] = 0.f;
#pragma unroll
      for (int i = 0; i < kHL; i += 2) {
#pragma unroll
        for (int c = 0; c < NA; ++c)
          if (c < AH) {
            if (i < hl) acc[c] = fmaf(hv[i], s_wh[(lane + 32 * i) * AH + c], acc[c]);
            if (i + 1 < hl) acc2[c] = fmaf(hv[i + 1], s_wh[(lane + 32 * (i + 1)) * AH + c], acc2[c]);
          }
      }
#pragma unroll
      for (int c = 0; c < NA; ++c) acc[c] += acc2[c];
    } else {
      for (int u = lane; u < H; u += 32) {
        const float h = hrow[u];
#pragma unroll
        for (int c = 0; c < NA; ++c)
          if (c < AH) acc[c] = fmaf(h, s_wh[u * AH + c], acc[c]);
      }
    }
    double lg[NA];
#pragma unroll
    for (int c = 0; c < NA; ++c) {
      if (c < AH) {
        float v = acc[c];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        lg[c] = (double)v + (double)bh[c];
      } else {
        lg[c] = 0.0;
      }
    }
    double value = 0.0;
#pragma unroll
    for (int c = 0; c < NA; ++c)
      if (c == A) value = lg[c];
    double logp, ent, mx = 0.0, lse = 0.0;
    const int a = continuous ? 0 : act_disc[p];
    if (!continuous) {
      mx = lg[0];
#pragma unroll
      for (int c = 1; c < NA; ++c)
        if (c < A) mx = fmax(mx, lg[c]);
      double se = 0.0;
#pragma unroll
      for (int c = 0; c < NA; ++c)
        if (c < A) se += exp(lg[c] - mx);
      lse = log(se);
      double lga = 0.0;
#pragma unroll
      for (int c = 0; c < NA; ++c)
        if (c == a) lga = lg[c];
      logp = lga - mx - lse;
      ent = 0.0;
#pragma unroll
      for (int c = 0; c < NA; ++c)
        if (c < A) {
          const double lp = lg[c] - mx - lse;
          ent -= exp(lp) * lp;
        }
    } else {
      double q = 0.0, sls = 0.0;
#pragma unroll
      for (int c = 0; c < NA; ++c)
        if (c < A) {
          const double ls = log_std[c];
          const double z = ((double)act_cont[(size_t)p * A + c] - lg[c]) * exp(-ls);
          q += z * z;
          sls += ls;
        }
      logp = -0.5 * q - sls - 0.5 * kLog2Pi * A;
      ent = sls + 0.5 * (1.0 + kLog2Pi) * A;
    }
    const double ratio = exp(logp - (double)old_logp[p]);
    const double A_ = adv[p];
    const double w = frozen_w ? (double)frozen_w[p] : fmin(ratio, is_cap);
    const double s1 = ratio * A_;
    const double cr = fmin(fmax(ratio, 1.0 - clip), 1.0 + clip);
    const double s2 = cr * A_;
    const double sur = fmin(s1, s2);
    const double verr = value - (double)ret[p];
    st[0] += w * sur;
    st[1] += verr * verr;
    st[2] += ent;
    st[3] += ratio;
    st[4] += (ratio < 1.0 - clip || ratio > 1.0 + clip) ? 1.0 : 0.0;  // strict (learner.cpp:104)
    st[5] += w;
    st[6] = fmax(st[6], w);
    if (lane == 0 && is_w) is_w[p] = (float)w;
    if (want_grads) {
      // cmin tie -> first argument (tape.cpp:157); clip mask inclusive (tape.cpp:146)
      const double m1 = s1 <= s2 ? 1.0 : 0.0;
      const double cm = (ratio >= 1.0 - clip && ratio <= 1.0 + clip) ? 1.0 : 0.0;
      const double dratio = -w * inv_S * (m1 * A_ + (1.0 - m1) * A_ * cm);
      const double dlogp = dratio * ratio;
      double dh[NA];
#pragma unroll
      for (int c = 0; c < NA; ++c) dh[c] = 0.0;
      if (!continuous) {
        double G[NA], sumG = 0.0;
#pragma unroll
        for (int c = 0; c < NA; ++c) {
          G[c] = 0.0;
          if (c < A) {
            const double lp = lg[c] - mx - lse;
            const double pc = exp(lp);
            G[c] = (c == a ? dlogp : 0.0) + gH * (-pc - pc * lp);
            sumG += G[c];
          }
        }
#pragma unroll
        for (int c = 0; c < NA; ++c)
          if (c < A) dh[c] = G[c] - exp(lg[c] - mx - lse) * sumG;
      } else {
#pragma unroll
        for (int c = 0; c < NA; ++c)
          if (c < A) {
            const double ls = log_std[c];
            const double inv = exp(-ls);
            const double z = ((double)act_cont[(size_t)p * A + c] - lg[c]) * inv;
            dh[c] = dlogp * z * inv;
            if (lane == c) dls += dlogp * (z * z - 1.0) + gH;
          }
      }
#pragma unroll
      for (int c = 0; c < NA; ++c)
        if (c == A) dh[c] = vcoef * verr * inv_S;
      float mine = 0.f;
#pragma unroll
      for (int c = 0; c < NA; ++c)
        if (c == lane) mine = (float)dh[c];
      if (lane < AH) dhead[(size_t)p * AH + lane] = mine;
      float dhf[NA];
#pragma unroll
      for (int c = 0; c < NA; ++c) dhf[c] = (float)dh[c];
      if (fuse) {
#pragma unroll
        for (int c = 0; c < NA; ++c) {
          bacc[c] += dhf[c];
#pragma unroll
          for (int i = 0; i < kHL; ++i) wacc[i][c] = fmaf(hv[i], dhf[c], wacc[i][c]);
        }
      }
      for (int u = lane; u < H; u += 32) {
        float sacc = 0.f;
#pragma unroll
        for (int c = 0; c < NA; ++c)
          if (c < AH) sacc = fmaf(dhf[c], s_wh[u * AH + c], sacc);
        dhidden[(size_t)p * H + u] = sacc;
      }
    }
  }
  if (fuse && want_grads) {
    // block sums of the head gradient, warps added in a fixed order (deterministic)
    for (int i = threadIdx.x; i < H * AH + AH; i += blockDim.x) s_hg[i] = 0.f;
    for (int w = 0; w < kLossWarps; ++w) {
      __syncthreads();
      if (warp == w) {
#pragma unroll
        for (int i = 0; i < kHL; ++i)
#pragma unroll
          for (int c = 0; c < NA; ++c)
            if (i < hl && c < AH) s_hg[(lane + 32 * i) * AH + c] += wacc[i][c];
        if (lane == 0)
#pragma unroll
          for (int c = 0; c < NA; ++c)
            if (c < AH) s_hg[H * AH + c] += bacc[c];
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < H * AH + AH; i += blockDim.x)
      hpart[(size_t)blockIdx.x * (H * AH + AH) + i] = s_hg[i];
  }
  // block reduction of the statistics (lane 0 of each warp holds identical st)
  if (lane == 0)
    for (int k = 0; k < kLossStats; ++k) s_red[warp][k] = st[k];
  if (lane < 32) s_red[warp][kLossStats + lane] = dls;
  __syncthreads();
  if (threadIdx.x < kLossStats + 32) {
    const int k = threadIdx.x;
    double s = 0.0;
    for (int w = 0; w < kLossWarps; ++w) s = (k == 6) ? fmax(s, s_red[w][k]) : s + s_red[w][k];
    part[(size_t)blockIdx.x * (kLossStats + 32) + k] = s;
  }
}

// Fused-path variant (H % 32 == 0, H <= 32 kHL, gradients wanted): a warp takes
// RBT rows at a time.  The heads (H -> A+1 dot products), the head gradient and
// dhidden stay warp-cooperative per row, but the per-row double-precision loss
// math (log-softmax / Gaussian log-prob, ratio, clip, IS weight, surrogate,
// value error, entropy and dhead) runs once per row in lane r instead of
// redundantly in all 32 lanes; statistics then reduce over the lanes in a fixed
// shuffle tree (deterministic).
template <int NA, int RBT>
__global__ void __launch_bounds__(kLossWarps * 32, 2) ppo_loss_rows_kernel(
    int S, int H, int A, int continuous, const float* __restrict__ hidden, const float* __restrict__ wh,
    const float* __restrict__ bh, const float* __restrict__ log_std, const float* __restrict__ act_cont,
    const int32_t* __restrict__ act_disc, const float* __restrict__ old_logp, const float* __restrict__ adv,
    const float* __restrict__ ret, const float* __restrict__ frozen_w, double clip, double is_cap,
    double vcoef, const double* __restrict__ alpha_p, double inv_S, float* __restrict__ dhead,
    float* __restrict__ dhidden, float* __restrict__ is_w, double* __restrict__ part, int want_grads,
    float* __restrict__ hpart) {
  extern __shared__ float s_wh[];  // H x AH, then H x AH + AH block sums of the head gradient
  __shared__ double s_red[kLossWarps][kLossStats + 32];
  const int AH = A + 1;
  const int hl = H / 32;
  float* s_hg = s_wh + H * AH;
  float wacc[kHL][NA], bacc[NA];
#pragma unroll
  for (int i = 0; i < kHL; ++i)
#pragma unroll
    for (int c = 0; c < NA; ++c) wacc[i][c] = 0.f;
#pragma unroll
  for (int c = 0; c < NA; ++c) bacc[c] = 0.f;
  for (int i = threadIdx.x; i < H * AH; i += blockDim.x) s_wh[i] = wh[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double alpha = *alpha_p;
  const double gH = -alpha * inv_S;
  double st[kLossStats] = {0, 0, 0, 0, 0, 0, 0, 0};
  double dlsv[NA];
#pragma unroll
  for (int c = 0; c < NA; ++c) dlsv[c] = 0.0;
  const int gw = blockIdx.x * kLossWarps + warp, nwarps = gridDim.x * kLossWarps;
  for (int pb = gw * RBT; pb < S; pb += nwarps * RBT) {
    const int nr = min(RBT, S - pb);
    // ---- heads of rows pb .. pb + nr - 1 (lane r keeps row r's logits)
    float lgm[NA];
#pragma unroll
    for (int c = 0; c < NA; ++c) lgm[c] = 0.f;
    float hn[kHL];
#pragma unroll
    for (int i = 0; i < kHL; ++i) hn[i] = i < hl ? __ldg(hidden + (size_t)pb * H + lane + 32 * i) : 0.f;
    for (int r = 0; r < nr; ++r) {
      float hv[kHL];
#pragma unroll
      for (int i = 0; i < kHL; ++i) hv[i] = hn[i];
      if (r + 1 < nr) {
#pragma unroll
        for (int i = 0; i < kHL; ++i) hn[i] = i < hl ? __ldg(hidden + (size_t)(pb + r + 1) * H + lane + 32 * i) : 0.f;
      }
      float acc[NA], acc2[NA];
#pragma unroll
      for (int c = 0; c < NA; ++c) acc[c] = acc2[c] = 0.f;
#pragma unroll
      for (int i = 0; i < kHL; i += 2) {
#pragma unroll
        for (int c = 0; c < NA; ++c)
          if (c < AH) {
            if (i < hl) acc[c] = fmaf(hv[i], s_wh[(lane + 32 * i) * AH + c], acc[c]);
            if (i + 1 < hl) acc2[c] = fmaf(hv[i + 1], s_wh[(lane + 32 * (i + 1)) * AH + c], acc2[c]);
          }
      }
#pragma unroll
      for (int c = 0; c < NA; ++c) {
        if (c < AH) {
          float v = acc[c] + acc2[c];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          if (lane == r) lgm[c] = v;
        }
      }
    }
    // ---- the loss math of row pb + lane (lanes < nr)
    float dhm[NA];
#pragma unroll
    for (int c = 0; c < NA; ++c) dhm[c] = 0.f;
    if (lane < nr) {
      const int p = pb + lane;
      double lg[NA];
#pragma unroll
      for (int c = 0; c < NA; ++c) lg[c] = c < AH ? (double)lgm[c] + (double)bh[c] : 0.0;
      double value = 0.0;
#pragma unroll
      for (int c = 0; c < NA; ++c)
        if (c == A) value = lg[c];
      double logp, ent, mx = 0.0, lse = 0.0;
      const int a = continuous ? 0 : act_disc[p];
      if (!continuous) {
        mx = lg[0];
#pragma unroll
        for (int c = 1; c < NA; ++c)
          if (c < A) mx = fmax(mx, lg[c]);
        double se = 0.0;
#pragma unroll
        for (int c = 0; c < NA; ++c)
          if (c < A) se += exp(lg[c] - mx);
        lse = log(se);
        double lga = 0.0;
#pragma unroll
        for (int c = 0; c < NA; ++c)
          if (c == a) lga = lg[c];
        logp = lga - mx - lse;
        ent = 0.0;
#pragma unroll
        for (int c = 0; c < NA; ++c)
          if (c < A) {
            const double lp = lg[c] - mx - lse;
            ent -= exp(lp) * lp;
          }
      } else {
        double q = 0.0, sls = 0.0;
#pragma unroll
        for (int c = 0; c < NA; ++c)
          if (c < A) {
            const double ls = log_std[c];
            const double z = ((double)act_cont[(size_t)p * A + c] - lg[c]) * exp(-ls);
            q += z * z;
            sls += ls;
          }
        logp = -0.5 * q - sls - 0.5 * kLog2Pi * A;
        ent = sls + 0.5 * (1.0 + kLog2Pi) * A;
      }
      const double ratio = exp(logp - (double)old_logp[p]);
      const double A_ = adv[p];
      const double w = frozen_w ? (double)frozen_w[p] : fmin(ratio, is_cap);
      const double s1 = ratio * A_;
      const double cr = fmin(fmax(ratio, 1.0 - clip), 1.0 + clip);
      const double s2 = cr * A_;
      const double sur = fmin(s1, s2);
      const double verr = value - (double)ret[p];
      st[0] += w * sur;
      st[1] += verr * verr;
      st[2] += ent;
      st[3] += ratio;
      st[4] += (ratio < 1.0 - clip || ratio > 1.0 + clip) ? 1.0 : 0.0;  // strict (learner.cpp:104)
      st[5] += w;
      st[6] = fmax(st[6], w);
      if (is_w) is_w[p] = (float)w;
      if (want_grads) {
        // cmin tie -> first argument (tape.cpp:157); clip mask inclusive (tape.cpp:146)
        const double m1 = s1 <= s2 ? 1.0 : 0.0;
        const double cm = (ratio >= 1.0 - clip && ratio <= 1.0 + clip) ? 1.0 : 0.0;
        const double dratio = -w * inv_S * (m1 * A_ + (1.0 - m1) * A_ * cm);
        const double dlogp = dratio * ratio;
        double dh[NA];
#pragma unroll
        for (int c = 0; c < NA; ++c) dh[c] = 0.0;
        if (!continuous) {
          double G[NA], sumG = 0.0;
#pragma unroll
          for (int c = 0; c < NA; ++c) {
            G[c] = 0.0;
            if (c < A) {
              const double lp = lg[c] - mx - lse;
              const double pc = exp(lp);
              G[c] = (c == a ? dlogp : 0.0) + gH * (-pc - pc * lp);
              sumG += G[c];
            }
          }
#pragma unroll
          for (int c = 0; c < NA; ++c)
            if (c < A) dh[c] = G[c] - exp(lg[c] - mx - lse) * sumG;
        } else {
#pragma unroll
          for (int c = 0; c < NA; ++c)
            if (c < A) {
              const double ls = log_std[c];
              const double inv = exp(-ls);
              const double z = ((double)act_cont[(size_t)p * A + c] - lg[c]) * inv;
              dh[c] = dlogp * z * inv;
              dlsv[c] += dlogp * (z * z - 1.0) + gH;
            }
        }
#pragma unroll
        for (int c = 0; c < NA; ++c)
          if (c == A) dh[c] = vcoef * verr * inv_S;
#pragma unroll
        for (int c = 0; c < NA; ++c)
          if (c < AH) {
            dhm[c] = (float)dh[c];
            dhead[(size_t)p * AH + c] = dhm[c];
          }
      }
    }
    if (!want_grads) continue;
    // ---- head gradient and dhidden = dhead wh^T, warp-cooperative per row
    for (int r = 0; r < nr; ++r) {
      const int p = pb + r;
      float dhf[NA];
#pragma unroll
      for (int c = 0; c < NA; ++c) dhf[c] = __shfl_sync(0xffffffffu, dhm[c], r);
      float hv[kHL];
#pragma unroll
      for (int i = 0; i < kHL; ++i) hv[i] = i < hl ? __ldg(hidden + (size_t)p * H + lane + 32 * i) : 0.f;
#pragma unroll
      for (int c = 0; c < NA; ++c) {
        bacc[c] += dhf[c];
#pragma unroll
        for (int i = 0; i < kHL; ++i) wacc[i][c] = fmaf(hv[i], dhf[c], wacc[i][c]);
      }
#pragma unroll
      for (int i = 0; i < kHL; ++i) {
        if (i < hl) {
          const int u = lane + 32 * i;
          float sacc = 0.f;
#pragma unroll
          for (int c = 0; c < NA; ++c)
            if (c < AH) sacc = fmaf(dhf[c], s_wh[u * AH + c], sacc);
          dhidden[(size_t)p * H + u] = sacc;
        }
      }
    }
  }
  if (want_grads) {
    // block sums of the head gradient, warps added in a fixed order (deterministic)
    for (int i = threadIdx.x; i < H * AH + AH; i += blockDim.x) s_hg[i] = 0.f;
    for (int w = 0; w < kLossWarps; ++w) {
      __syncthreads();
      if (warp == w) {
#pragma unroll
        for (int i = 0; i < kHL; ++i)
#pragma unroll
          for (int c = 0; c < NA; ++c)
            if (i < hl && c < AH) s_hg[(lane + 32 * i) * AH + c] += wacc[i][c];
        if (lane == 0)
#pragma unroll
          for (int c = 0; c < NA; ++c)
            if (c < AH) s_hg[H * AH + c] += bacc[c];
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < H * AH + AH; i += blockDim.x)
      hpart[(size_t)blockIdx.x * (H * AH + AH) + i] = s_hg[i];
  }
  // statistics and the log_std gradient over the lanes (fixed xor tree), then the block
#pragma unroll
  for (int k = 0; k < kLossStats; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double y = __shfl_xor_sync(0xffffffffu, st[k], o);
      st[k] = (k == 6) ? fmax(st[k], y) : st[k] + y;
    }
  }
  double dls = 0.0;
#pragma unroll
  for (int c = 0; c < NA; ++c) {
    double v = dlsv[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == c) dls = v;
  }
  if (lane == 0)
    for (int k = 0; k < kLossStats; ++k) s_red[warp][k] = st[k];
  s_red[warp][kLossStats + lane] = dls;
  __syncthreads();
  if (threadIdx.x < kLossStats + 32) {
    const int k = threadIdx.x;
    double s = 0.0;
    for (int w = 0; w < kLossWarps; ++w) s = (k == 6) ? fmax(s, s_red[w][k]) : s + s_red[w][k];
    part[(size_t)blockIdx.x * (kLossStats + 32) + k] = s;
  }
}

// Staged variant of the fused loss (H % 128 == 0, H <= 512, A + 1 == NA <= 3,
// gradients wanted): each warp stages its group of kStageRows consecutive
// packed rows of `hidden` (contiguous, kStageRows x H x 4 B) into shared
// memory with one bulk copy, so the rows are read from HBM once and both the
// head pass and the gradient pass read them as float4 from shared memory.
// The head weights live in registers (lane l owns columns 4l + 128i .. +3),
// the per-row double loss math runs in lane r for row r (as in
// ppo_loss_rows_kernel), dhead is not materialised.  Per row: 2H + 16 B read,
// 2H B... i.e. the head-fused 8H + 16 B of SURVEY §8(d).
constexpr int kStageRows = 8;
constexpr int kStageWarps = 4;
template <int NA>
__global__ void __launch_bounds__(kStageWarps * 32, 3) ppo_loss_stage_kernel(
    int S, int H, int A, int continuous, const float* __restrict__ hidden, const float* __restrict__ wh,
    const float* __restrict__ bh, const float* __restrict__ log_std, const float* __restrict__ act_cont,
    const int32_t* __restrict__ act_disc, const float* __restrict__ old_logp, const float* __restrict__ adv,
    const float* __restrict__ ret, const float* __restrict__ frozen_w, double clip, double is_cap,
    double vcoef, const double* __restrict__ alpha_p, double inv_S, float* __restrict__ dhidden,
    float* __restrict__ is_w, double* __restrict__ part, float* __restrict__ hpart) {
  constexpr int HV = 4;  // float4 columns per lane at H = 512 (fewer at smaller H: masked)
  extern __shared__ __align__(128) float s_rows[];  // kStageWarps x kStageRows x H
  __shared__ uint64_t s_bar[kStageWarps];
  __shared__ double s_red[kStageWarps][kLossStats + 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int hv = H / 128;
  float* rows = s_rows + (size_t)warp * kStageRows * H;
  const uint32_t bar = static_cast<uint32_t>(__cvta_generic_to_shared(&s_bar[warp]));
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  // head weights of this lane's columns: w[i][e][c] = wh[(4 lane + 128 i + e) * NA + c]
  float w[HV][4][NA], wacc[HV][4][NA], bacc[NA];
#pragma unroll
  for (int i = 0; i < HV; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e)
#pragma unroll
      for (int c = 0; c < NA; ++c) {
        w[i][e][c] = i < hv ? __ldg(wh + (size_t)(4 * lane + 128 * i + e) * NA + c) : 0.f;
        wacc[i][e][c] = 0.f;
      }
#pragma unroll
  for (int c = 0; c < NA; ++c) bacc[c] = 0.f;
  float bhv[NA];
#pragma unroll
  for (int c = 0; c < NA; ++c) bhv[c] = bh[c];
  const double alpha = *alpha_p;
  const double gH = -alpha * inv_S;
  double st[kLossStats] = {0, 0, 0, 0, 0, 0, 0, 0};
  double dlsv[NA];
#pragma unroll
  for (int c = 0; c < NA; ++c) dlsv[c] = 0.0;
  const int gw = blockIdx.x * kStageWarps + warp, nwarps = gridDim.x * kStageWarps;
  uint32_t phase = 0;
  for (int pb = gw * kStageRows; pb < S; pb += nwarps * kStageRows, phase ^= 1) {
    const int nr = min(kStageRows, S - pb);
    if (lane == 0) {
      const uint32_t bytes = (uint32_t)nr * H * 4;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the last group's generic reads first
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       static_cast<uint32_t>(__cvta_generic_to_shared(rows))),
                   "l"(hidden + (size_t)pb * H), "r"(bytes), "r"(bar)
                   : "memory");
    }
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "LS_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra LS_WAIT;\n\t}" ::"r"(bar),
        "r"(phase)
        : "memory");
    // ---- heads of the staged rows: lane r keeps row r's logits
    float lgm[NA];
#pragma unroll
    for (int c = 0; c < NA; ++c) lgm[c] = 0.f;
    for (int r = 0; r < nr; ++r) {
      const float* row = rows + (size_t)r * H;
      float acc[NA];
#pragma unroll
      for (int c = 0; c < NA; ++c) acc[c] = 0.f;
#pragma unroll
      for (int i = 0; i < HV; ++i)
        if (i < hv) {
          const float4 x = *reinterpret_cast<const float4*>(row + 4 * lane + 128 * i);
#pragma unroll
          for (int c = 0; c < NA; ++c)
            acc[c] = fmaf(x.x, w[i][0][c], fmaf(x.y, w[i][1][c], fmaf(x.z, w[i][2][c], fmaf(x.w, w[i][3][c], acc[c]))));
        }
#pragma unroll
      for (int c = 0; c < NA; ++c) {
        float v = acc[c];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == r) lgm[c] = v;
      }
    }
    // ---- the loss math of row pb + lane (lanes < nr), learner.cpp:77-115
    float dhm[NA];
#pragma unroll
    for (int c = 0; c < NA; ++c) dhm[c] = 0.f;
    if (lane < nr) {
      const int p = pb + lane;
      double lg[NA];
#pragma unroll
      for (int c = 0; c < NA; ++c) lg[c] = (double)lgm[c] + (double)bhv[c];
      const double value = lg[NA - 1];
      double logp, ent, mx = 0.0, lse = 0.0;
      const int a = continuous ? 0 : act_disc[p];
      if (!continuous) {
        mx = lg[0];
#pragma unroll
        for (int c = 1; c < NA - 1; ++c) mx = fmax(mx, lg[c]);
        double se = 0.0;
#pragma unroll
        for (int c = 0; c < NA - 1; ++c) se += exp(lg[c] - mx);
        lse = log(se);
        double lga = 0.0;
#pragma unroll
        for (int c = 0; c < NA - 1; ++c)
          if (c == a) lga = lg[c];
        logp = lga - mx - lse;
        ent = 0.0;
#pragma unroll
        for (int c = 0; c < NA - 1; ++c) {
          const double lp = lg[c] - mx - lse;
          ent -= exp(lp) * lp;
        }
      } else {
        double q = 0.0, sls = 0.0;
#pragma unroll
        for (int c = 0; c < NA - 1; ++c) {
          const double ls = log_std[c];
          const double z = ((double)act_cont[(size_t)p * A + c] - lg[c]) * exp(-ls);
          q += z * z;
          sls += ls;
        }
        logp = -0.5 * q - sls - 0.5 * kLog2Pi * A;
        ent = sls + 0.5 * (1.0 + kLog2Pi) * A;
      }
      const double ratio = exp(logp - (double)old_logp[p]);
      const double A_ = adv[p];
      const double wv = frozen_w ? (double)frozen_w[p] : fmin(ratio, is_cap);
      const double s1 = ratio * A_;
      const double cr = fmin(fmax(ratio, 1.0 - clip), 1.0 + clip);
      const double s2 = cr * A_;
      const double sur = fmin(s1, s2);
      const double verr = value - (double)ret[p];
      st[0] += wv * sur;
      st[1] += verr * verr;
      st[2] += ent;
      st[3] += ratio;
      st[4] += (ratio < 1.0 - clip || ratio > 1.0 + clip) ? 1.0 : 0.0;  // strict (learner.cpp:104)
      st[5] += wv;
      st[6] = fmax(st[6], wv);
      if (is_w) is_w[p] = (float)wv;
      // cmin tie -> first argument (tape.cpp:157); clip mask inclusive (tape.cpp:146)
      const double m1 = s1 <= s2 ? 1.0 : 0.0;
      const double cm = (ratio >= 1.0 - clip && ratio <= 1.0 + clip) ? 1.0 : 0.0;
      const double dratio = -wv * inv_S * (m1 * A_ + (1.0 - m1) * A_ * cm);
      const double dlogp = dratio * ratio;
      double dh[NA];
#pragma unroll
      for (int c = 0; c < NA; ++c) dh[c] = 0.0;
      if (!continuous) {
        double G[NA], sumG = 0.0;
#pragma unroll
        for (int c = 0; c < NA - 1; ++c) {
          const double lp = lg[c] - mx - lse;
          const double pc = exp(lp);
          G[c] = (c == a ? dlogp : 0.0) + gH * (-pc - pc * lp);
          sumG += G[c];
        }
#pragma unroll
        for (int c = 0; c < NA - 1; ++c) dh[c] = G[c] - exp(lg[c] - mx - lse) * sumG;
      } else {
#pragma unroll
        for (int c = 0; c < NA - 1; ++c) {
          const double ls = log_std[c];
          const double inv = exp(-ls);
          const double z = ((double)act_cont[(size_t)p * A + c] - lg[c]) * inv;
          dh[c] = dlogp * z * inv;
          dlsv[c] += dlogp * (z * z - 1.0) + gH;
        }
      }
      dh[NA - 1] = vcoef * verr * inv_S;
#pragma unroll
      for (int c = 0; c < NA; ++c) dhm[c] = (float)dh[c];
    }
    // ---- head gradient and dhidden = dhead wh^T from the staged rows
    for (int r = 0; r < nr; ++r) {
      const int p = pb + r;
      const float* row = rows + (size_t)r * H;
      float dhf[NA];
#pragma unroll
      for (int c = 0; c < NA; ++c) {
        dhf[c] = __shfl_sync(0xffffffffu, dhm[c], r);
        bacc[c] += dhf[c];
      }
#pragma unroll
      for (int i = 0; i < HV; ++i)
        if (i < hv) {
          const float4 x = *reinterpret_cast<const float4*>(row + 4 * lane + 128 * i);
          const float xe[4] = {x.x, x.y, x.z, x.w};
          float o[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float sacc = 0.f;
#pragma unroll
            for (int c = 0; c < NA; ++c) {
              wacc[i][e][c] = fmaf(xe[e], dhf[c], wacc[i][e][c]);
              sacc = fmaf(dhf[c], w[i][e][c], sacc);
            }
            o[e] = sacc;
          }
          __stcs(reinterpret_cast<float4*>(dhidden + (size_t)p * H + 4 * lane + 128 * i),
                 make_float4(o[0], o[1], o[2], o[3]));
        }
    }
    __syncwarp();  // every lane is done with the staged rows before the next bulk copy lands there
  }
  // block sums of the head gradient, warps added in a fixed order (deterministic);
  // the staged-row buffer of warp 0 is reused as the accumulator
  __syncthreads();
  float* s_hg = s_rows;
  for (int i = threadIdx.x; i < H * NA + NA; i += blockDim.x) s_hg[i] = 0.f;
  for (int ww = 0; ww < kStageWarps; ++ww) {
    __syncthreads();
    if (warp == ww) {
#pragma unroll
      for (int i = 0; i < HV; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e)
#pragma unroll
          for (int c = 0; c < NA; ++c)
            if (i < hv) s_hg[(4 * lane + 128 * i + e) * NA + c] += wacc[i][e][c];
      if (lane == 0)
#pragma unroll
        for (int c = 0; c < NA; ++c) s_hg[H * NA + c] += bacc[c];
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < H * NA + NA; i += blockDim.x) hpart[(size_t)blockIdx.x * (H * NA + NA) + i] = s_hg[i];
  // statistics and the log_std gradient over the lanes (fixed xor tree), then the block
#pragma unroll
  for (int k = 0; k < kLossStats; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double y = __shfl_xor_sync(0xffffffffu, st[k], o);
      st[k] = (k == 6) ? fmax(st[k], y) : st[k] + y;
    }
  }
  double dls = 0.0;
#pragma unroll
  for (int c = 0; c < NA; ++c) {
    double v = dlsv[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == c) dls = v;
  }
  if (lane == 0)
    for (int k = 0; k < kLossStats; ++k) s_red[warp][k] = st[k];
  s_red[warp][kLossStats + lane] = dls;
  __syncthreads();
  if (threadIdx.x < kLossStats + 32) {
    const int k = threadIdx.x;
    double sum = 0.0;
    for (int ww = 0; ww < kStageWarps; ++ww) sum = (k == 6) ? fmax(sum, s_red[ww][k]) : sum + s_red[ww][k];
    part[(size_t)blockIdx.x * (kLossStats + 32) + k] = sum;
  }
}

__global__ void ppo_loss_final_kernel(const double* __restrict__ part, int nblk, int A, int continuous,
                                      double inv_S, int S, double vcoef, const double* __restrict__ alpha_p,
                                      LossStats* __restrict__ out, float* __restrict__ grad_ls,
                                      float* __restrict__ ent_slot) {
  pdl_wait();
  pdl_trigger();
  __shared__ double tot[kLossStats + 32];
  // warp w reduces statistics w, w + 32 over the block partials (lane-strided,
  // then a fixed shuffle tree: deterministic)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = warp; k < kLossStats + 32; k += blockDim.x >> 5) {
    double s = 0.0;
    for (int b = lane; b < nblk; b += 32) {
      const double v = part[(size_t)b * (kLossStats + 32) + k];
      s = (k == 6) ? fmax(s, v) : s + v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double y = __shfl_xor_sync(0xffffffffu, s, o);
      s = (k == 6) ? fmax(s, y) : s + y;
    }
    if (lane == 0) tot[k] = s;
  }
  __syncthreads();
  const int k = threadIdx.x;
  if (k == 0) {
    LossStats r;
    r.policy_loss = -tot[0] * inv_S;
    r.value_loss = 0.5 * tot[1] * inv_S;
    r.mean_entropy = tot[2] * inv_S;
    r.loss = r.policy_loss + vcoef * r.value_loss - (*alpha_p) * r.mean_entropy;
    r.ratio_sum = tot[3];
    r.clip_count = tot[4];
    r.w_sum = tot[5];
    r.w_max = S > 0 ? tot[6] : 0.0;
    r.steps = S;
    *out = r;
    if (ent_slot) *ent_slot = (float)r.mean_entropy;
  }
  if (continuous && grad_ls && k < A) grad_ls[k] = (float)tot[kLossStats + k];
}

// head gradient: sum of the per-block partials -> grad wh, bh.  Block = 32
// outputs (lanes) x 32 warps; warp w sums partials b = w, w + 32, ...; the 32
// warp sums are added in a fixed order (deterministic).
__global__ void __launch_bounds__(1024) head_grad_final_kernel(const float* __restrict__ hpart, int nblk, int n,
                                                               int nw, float* __restrict__ gwh,
                                                               float* __restrict__ gbh) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[32][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i = blockIdx.x * 32 + lane;
  float s = 0.f;
  if (i < n)
    for (int b = warp; b < nblk; b += 32) s += hpart[(size_t)b * n + i];
  red[warp][lane] = s;
  __syncthreads();
  if (warp == 0 && i < n) {
    float t = 0.f;
    for (int w = 0; w < 32; ++w) t += red[w][lane];
    if (i < nw) gwh[i] = t;
    else gbh[i - nw] = t;
  }
}

void policy_loss(Ctx* c, const Model& m, const float* params, int S, const LossArgs& a, Workspace& ws,
                 float* grad, LossStats* stats, bool want_grads) {
  // staged path (ppo_loss_stage_kernel): the bench shapes (H = 512, A + 1 = 3)
  if (want_grads && m.H % 128 == 0 && m.H <= 512 && (m.AH == 2 || m.AH == 3) && S > 0) {
    const int blk_rows = kStageWarps * kStageRows;
    const size_t ssmem = sizeof(float) * std::max((size_t)kStageWarps * kStageRows * m.H, (size_t)m.H * m.AH + m.AH);
    static std::atomic<int> per_sm_cache[kMaxDevices][2];
    std::atomic<int>& ps = per_sm_cache[dev_slot(c)][m.AH - 2];
    auto kern = m.AH == 3 ? ppo_loss_stage_kernel<3> : ppo_loss_stage_kernel<2>;
    int per_sm = ps.load();
    if (!per_sm) {  // attribute and occupancy for the largest staging buffer (H = 512), whatever H comes first
      const size_t smax = sizeof(float) * (size_t)kStageWarps * kStageRows * 512;
      VER_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax));
      VER_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kStageWarps * 32, smax));
      per_sm = std::max(1, per_sm);
      ps.store(per_sm);
    }
    const int nblk = std::max(1, std::min((int)cdiv(S, blk_rows), per_sm * c->num_sms));
    const size_t nhg = (size_t)m.H * m.AH + m.AH;
    ws.part.reserve(c, (size_t)nblk * (kLossStats + 32));
    ws.splitk.reserve(c, (size_t)nblk * nhg);
    kern<<<nblk, kStageWarps * 32, ssmem, c->stream>>>(
        S, m.H, m.A, m.continuous, ws.hidden.p, params + m.o_wh, params + m.o_bh,
        m.continuous ? params + m.o_ls : nullptr, a.act_cont, a.act_disc, a.old_logp, a.adv, a.ret, a.frozen_w,
        a.clip, a.is_cap, a.vcoef, a.alpha, 1.0 / (double)S, ws.dhidden.p, ws.is_w.p, ws.part.p, ws.splitk.p);
    after_launch(c);
    launch_pdl(c, ppo_loss_final_kernel, dim3(1), dim3(1024), 0, (const double*)ws.part.p, nblk, m.A, m.continuous,
               1.0 / (double)S, S, a.vcoef, a.alpha, stats, m.continuous ? grad + m.o_ls : nullptr, grad + m.P);
    launch_pdl(c, head_grad_final_kernel, dim3(cdiv(nhg, 32)), dim3(1024), 0, (const float*)ws.splitk.p, nblk,
               (int)nhg, m.H * m.AH, grad + m.o_wh, grad + m.o_bh);
    return;
  }
  const bool fuse = want_grads && m.H % 32 == 0 && m.H / 32 <= kHL;
  // fused path: kLossRows rows per warp-iteration with the loss math once per row
  // (ppo_loss_rows_kernel)
  const int rows = fuse ? kLossRows : 0;
  const int per_blk = kLossWarps * std::max(1, rows);
  const int nblk = std::max(1, std::min((int)cdiv(S, per_blk), 4 * c->num_sms));
  ws.part.reserve(c, (size_t)nblk * (kLossStats + 32));
  const size_t nhg = (size_t)m.H * m.AH + m.AH;
  const size_t smem = sizeof(float) * ((size_t)m.H * m.AH + (fuse ? nhg : 0));
  if (fuse) ws.splitk.reserve(c, (size_t)nblk * nhg);
  float* hpart = fuse ? ws.splitk.p : nullptr;
  float* dhead = ws.dhead.p;  // S x (A+1)
  auto run = [&](auto kern) {
    if (smem > 48 * 1024)
      VER_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<nblk, kLossWarps * 32, smem, c->stream>>>(
        S, m.H, m.A, m.continuous, ws.hidden.p, params + m.o_wh, params + m.o_bh,
        m.continuous ? params + m.o_ls : nullptr, a.act_cont, a.act_disc, a.old_logp, a.adv, a.ret, a.frozen_w,
        a.clip, a.is_cap, a.vcoef, a.alpha, 1.0 / (double)S, dhead, ws.dhidden.p, ws.is_w.p, ws.part.p,
        want_grads ? 1 : 0, hpart);
    after_launch(c);
  };
  if (rows == kLossRows && m.AH == 3) {
    run(ppo_loss_rows_kernel<3, kLossRows>);
  } else if (rows == kLossRows && m.AH == 2) {
    run(ppo_loss_rows_kernel<2, kLossRows>);
  } else if (rows == kLossRows && m.AH <= 9) {
    run(ppo_loss_rows_kernel<9, kLossRows>);
  } else switch (m.AH) {
    case 2: run(ppo_loss_kernel<2>); break;
    case 3: run(ppo_loss_kernel<3>); break;
    case 4: run(ppo_loss_kernel<4>); break;
    case 5: run(ppo_loss_kernel<5>); break;
    case 7: run(ppo_loss_kernel<7>); break;
    case 9: run(ppo_loss_kernel<9>); break;
    default: run(ppo_loss_kernel<32>); break;
  }
  launch_pdl(c, ppo_loss_final_kernel, dim3(1), dim3(1024), 0, (const double*)ws.part.p, nblk, m.A, m.continuous,
             1.0 / (double)S, S, a.vcoef, a.alpha, stats, want_grads && m.continuous ? grad + m.o_ls : nullptr,
             want_grads ? grad + m.P : nullptr);
  if (fuse) {
    launch_pdl(c, head_grad_final_kernel, dim3(cdiv(nhg, 32)), dim3(1024), 0, (const float*)hpart, nblk, (int)nhg,
               m.H * m.AH, grad + m.o_wh, grad + m.o_bh);
  } else if (want_grads) {
    // head weights / biases: dwh = hidden^T dhead, dbh = colsum(dhead)
    gemm_splitk<true, false>(c, ws, m.H, m.AH, S, ws.hidden.p, m.H, dhead, m.AH, grad + m.o_wh, m.AH);
    colsum(c, ws, dhead, S, m.AH, m.AH, grad + m.o_bh);
  }
}

// ------------------------------------------------------------ backward
// db1 and dw1 in one pass over dpre1 (K = S rows, D = obs_dim small):
// out[0][k] = sum_p dpre1[p,k];  out[1+d][k] = sum_p obs[p,d] dpre1[p,k]
__global__ void enc1_grad_partial_kernel(const float* __restrict__ obs, const float* __restrict__ dpre1, int S,
                                         int D, int E, int rows_per, float* __restrict__ part) {
  __shared__ float red[8][33 * (kMaxD + 1)];
  const int k = blockIdx.x * 32 + (threadIdx.x & 31);
  const int r = threadIdx.x >> 5;
  const int m0 = blockIdx.y * rows_per, m1 = min(S, m0 + rows_per);
  float acc[kMaxD + 1];
#pragma unroll
  for (int d = 0; d <= kMaxD; ++d) acc[d] = 0.f;
  if (k < E)
    for (int m = m0 + r; m < m1; m += 8) {
      const float g = dpre1[(size_t)m * E + k];
      acc[0] += g;
#pragma unroll
      for (int d = 0; d < kMaxD; ++d)
        if (d < D) acc[1 + d] = fmaf(obs[(size_t)m * D + d], g, acc[1 + d]);
    }
  for (int d = 0; d <= D; ++d) red[r][(threadIdx.x & 31) * (kMaxD + 1) + d] = acc[d];
  __syncthreads();
  if (r == 0 && k < E)
    for (int d = 0; d <= D; ++d) {
      float t = 0.f;
      for (int q = 0; q < 8; ++q) t += red[q][(threadIdx.x & 31) * (kMaxD + 1) + d];
      part[((size_t)blockIdx.y * (D + 1) + d) * E + k] = t;
    }
}
// float4 variant (E % 4 == 0): lane = 4 features, a block = 128 features x a row
// chunk, each warp walks every 8th row two rows at a time
__global__ void __launch_bounds__(256) enc1_grad4_partial_kernel(const float* __restrict__ obs,
                                                                 const float* __restrict__ dpre1, int S, int D,
                                                                 int E, int rows_per, float* __restrict__ part) {
  pdl_wait();
  pdl_trigger();
  __shared__ float4 red[8][32][kMaxD + 1];
  const int lane = threadIdx.x & 31, r = threadIdx.x >> 5;
  const int k = blockIdx.x * 128 + 4 * lane;
  const int m0 = blockIdx.y * rows_per, m1 = min(S, m0 + rows_per);
  float4 acc[kMaxD + 1];
#pragma unroll
  for (int d = 0; d <= kMaxD; ++d) acc[d] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (k < E) {
    int m = m0 + r;
    for (; m + 8 < m1; m += 16) {
      const float4 g0 = __ldg(reinterpret_cast<const float4*>(dpre1 + (size_t)m * E + k));
      const float4 g1 = __ldg(reinterpret_cast<const float4*>(dpre1 + (size_t)(m + 8) * E + k));
      acc[0].x += g0.x + g1.x; acc[0].y += g0.y + g1.y; acc[0].z += g0.z + g1.z; acc[0].w += g0.w + g1.w;
#pragma unroll
      for (int d = 0; d < kMaxD; ++d)
        if (d < D) {
          const float o0 = __ldg(obs + (size_t)m * D + d), o1 = __ldg(obs + (size_t)(m + 8) * D + d);
          acc[1 + d].x = fmaf(o1, g1.x, fmaf(o0, g0.x, acc[1 + d].x));
          acc[1 + d].y = fmaf(o1, g1.y, fmaf(o0, g0.y, acc[1 + d].y));
          acc[1 + d].z = fmaf(o1, g1.z, fmaf(o0, g0.z, acc[1 + d].z));
          acc[1 + d].w = fmaf(o1, g1.w, fmaf(o0, g0.w, acc[1 + d].w));
        }
    }
    for (; m < m1; m += 8) {
      const float4 g = __ldg(reinterpret_cast<const float4*>(dpre1 + (size_t)m * E + k));
      acc[0].x += g.x; acc[0].y += g.y; acc[0].z += g.z; acc[0].w += g.w;
#pragma unroll
      for (int d = 0; d < kMaxD; ++d)
        if (d < D) {
          const float o = __ldg(obs + (size_t)m * D + d);
          acc[1 + d].x = fmaf(o, g.x, acc[1 + d].x);
          acc[1 + d].y = fmaf(o, g.y, acc[1 + d].y);
          acc[1 + d].z = fmaf(o, g.z, acc[1 + d].z);
          acc[1 + d].w = fmaf(o, g.w, acc[1 + d].w);
        }
    }
  }
#pragma unroll
  for (int d = 0; d <= kMaxD; ++d)
    if (d <= D) red[r][lane][d] = acc[d];
  __syncthreads();
  if (r == 0 && k < E)
    for (int d = 0; d <= D; ++d) {
      float4 t = red[0][lane][d];
      for (int q = 1; q < 8; ++q) {
        const float4 u = red[q][lane][d];
        t.x += u.x; t.y += u.y; t.z += u.z; t.w += u.w;
      }
      *reinterpret_cast<float4*>(part + ((size_t)blockIdx.y * (D + 1) + d) * E + k) = t;
    }
}
// block (32 outputs x 8 chunk groups): thread (i, q) sums chunks q, q + 8, ...;
// the 8 group sums reduce in a fixed order (deterministic)
__global__ void enc1_grad_final_kernel(const float* __restrict__ part, int chunks, int D, int E,
                                       float* __restrict__ db1, float* __restrict__ dw1) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[8][33];
  const int i = blockIdx.x * 32 + threadIdx.x, q = threadIdx.y;
  float s = 0.f;
  if (i < (D + 1) * E)
    for (int c = q; c < chunks; c += 8) s += part[(size_t)c * (D + 1) * E + i];
  red[q][threadIdx.x] = s;
  __syncthreads();
  if (q != 0 || i >= (D + 1) * E) return;
  float t = 0.f;
  for (int k = 0; k < 8; ++k) t += red[k][threadIdx.x];
  const int d = i / E, k = i % E;
  if (d == 0) db1[k] = t;
  else dw1[(size_t)(d - 1) * E + k] = t;
}

void policy_backward(Ctx* c, const Model& m, const float* params, int S, const float* obs, int L,
                     const int32_t* d_bs, const int32_t* d_offs, Workspace& ws, float* grad,
                     const int32_t* h_bs, const int32_t* h_offs) {
  const int E = m.E, H = m.H, H3 = 3 * m.H;
  gru_backward_recurrence(c, m, params, L, d_bs, d_offs, ws, h_bs, h_offs);
  // weight gradients over all rows
  gemm_splitk<true, false>(c, ws, H, H3, S, ws.hprev.p, H, ws.dhu.p, H3, grad + m.o_ux, H3);
  gemm_splitk<true, false>(c, ws, E, H3, S, ws.enc.p, E, ws.dpre.p, H3, grad + m.o_wx, H3);
  // data gradients: fp16x2 when this minibatch's forward made the weight halves
  // (the gradient operand's max taken by its bias column-sum pass, its halves
  // written in the GEMM)
  const bool f16 = ws.f16_fwd && ws.w16inv.n >= 5 && tc::usable_f16(S, E, H3, H3, H3) &&
                   tc::usable_f16(S, E, E, E, E) && H3 % 4 == 0 && E % 4 == 0 &&
                   tc::usable(S, E, H3, ws.dpre.p, H3, ws.dpre.p, H3, EpiTanhGrad{ws.dpre2.p, E, ws.enc.p, E});
  if (f16) {
    ws.gmax.reserve(c, 2);
    ws.gmax.zero(2);
  }
  colsum(c, ws, ws.dpre.p, S, H3, H3, grad + m.o_bx, f16 ? ws.gmax.p : nullptr);
  // slots 3 / 4 of refresh_weights_f16: after wx^T (3H x E), w2^T (E x E), ux^T (3H x H)
  const size_t o3 = (size_t)H3 * E + (size_t)E * E + (size_t)H3 * H, o4 = o3 + (size_t)H3 * E;
  if (f16) {
    tc::launch_f16a(c, S, E, H3, ws.dpre.p, H3, ws.w16hi.p + o3, ws.w16lo.p + o3, H3, ws.gmax.p, ws.w16inv.p + 3,
                    EpiTanhGrad{ws.dpre2.p, E, ws.enc.p, E}, 1);
  } else {
    gemm<false, true>(c, S, E, H3, ws.dpre.p, H3, params + m.o_wx, H3, EpiTanhGrad{ws.dpre2.p, E, ws.enc.p, E},
                      ws.wlo.n >= (size_t)m.P ? ws.wlo.p + m.o_wx : nullptr);
  }
  gemm_splitk<true, false>(c, ws, E, E, S, ws.e1.p, E, ws.dpre2.p, E, grad + m.o_w2, E);
  colsum(c, ws, ws.dpre2.p, S, E, E, grad + m.o_b2, f16 ? ws.gmax.p + 1 : nullptr);
  if (f16) {
    tc::launch_f16a(c, S, E, E, ws.dpre2.p, E, ws.w16hi.p + o4, ws.w16lo.p + o4, E, ws.gmax.p + 1, ws.w16inv.p + 4,
                    EpiTanhGrad{ws.dpre1.p, E, ws.e1.p, E}, 1);
  } else {
    gemm<false, true>(c, S, E, E, ws.dpre2.p, E, params + m.o_w2, E, EpiTanhGrad{ws.dpre1.p, E, ws.e1.p, E},
                      ws.wlo.n >= (size_t)m.P ? ws.wlo.p + m.o_w2 : nullptr);
  }
  {
    // ~4 blocks per SM: 128-feature blocks (float4 path) or 32-feature blocks
    const int col_blocks = (int)cdiv(E, E % 4 == 0 ? 128 : 32);
    int rows_per = 64;
    while ((int64_t)col_blocks * cdiv(S, rows_per) > 4 * c->num_sms && rows_per < 8192) rows_per *= 2;
    const int chunks = std::max(1, (int)cdiv(S, rows_per));
    ws.splitk.reserve(c, (size_t)chunks * (m.D + 1) * E);
    if (E % 4 == 0) {
      launch_pdl(c, enc1_grad4_partial_kernel, dim3(cdiv(E, 128), chunks), dim3(256), 0, obs,
                 (const float*)ws.dpre1.p, S, m.D, E, rows_per, ws.splitk.p);
    } else {
      enc1_grad_partial_kernel<<<dim3(cdiv(E, 32), chunks), 256, 0, c->stream>>>(obs, ws.dpre1.p, S, m.D, E,
                                                                                 rows_per, ws.splitk.p);
    }
    after_launch(c);
    enc1_grad_final_kernel<<<cdiv((size_t)(m.D + 1) * E, 32), dim3(32, 8), 0, c->stream>>>(
        ws.splitk.p, chunks, m.D, E, grad + m.o_b1, grad + m.o_w1);
    after_launch(c);
  }
}

// ---------------------------------------------------------------- Adam
__global__ void adam_kernel(int64_t P, float* __restrict__ w, const float* __restrict__ g, float* __restrict__ m,
                            float* __restrict__ v, float lr, float bc1, float bc2, int64_t ls0, int64_t ls1,
                            int* __restrict__ nonfinite, const LossStats* __restrict__ st) {
  pdl_wait();
  pdl_trigger();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P) return;
  // learner guard (alpha_update_kernel): no step after a failed minibatch
  // (flag [1]) or on a non-finite loss (the reference throws before Adam,
  // learner.cpp:111)
  if (st && (nonfinite[1] || !isfinite(st->loss))) return;
  const float gi = g[i];
  const float mi = 0.9f * m[i] + (1.f - 0.9f) * gi;
  const float vi = 0.999f * v[i] + (1.f - 0.999f) * (gi * gi);
  m[i] = mi;
  v[i] = vi;
  float wi = w[i] - lr * (mi / bc1) / (sqrtf(vi / bc2) + 1e-8f);
  if (i >= ls0 && i < ls1) wi = fminf(fmaxf(wi, -5.f), 2.f);  // kLogStdMin/Max (nn.hpp:26-27)
  w[i] = wi;
  if (!isfinite(wi)) atomicOr(nonfinite, 1);
}

void adam_update(Ctx* c, const Model& m, float* params, const float* grad, float* mom, float* vel, int64_t step,
                 double lr, int* nonfinite_flag, const LossStats* guard) {
  const double bc1 = 1.0 - std::pow(0.9, (double)step);
  const double bc2 = 1.0 - std::pow(0.999, (double)step);
  const int64_t ls0 = m.continuous ? m.o_ls : -1, ls1 = m.continuous ? m.o_ls + m.A : -1;
  launch_pdl(c, adam_kernel, dim3(cdiv(m.P, 256)), dim3(256), 0, (int64_t)m.P, params, (const float*)grad, mom, vel,
             (float)lr, (float)bc1, (float)bc2, ls0, ls1, nonfinite_flag, guard);
}

// --------------------------------------------------------- host init
// rng.hpp:16-75 (CounterRng) and nn.cpp:16-30 (orthogonal): the thin Q
// factor of a Gaussian matrix with diag(R) > 0 is unique, computed here by
// twice-iterated modified Gram-Schmidt.
namespace {
inline uint64_t splitmix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
inline uint64_t mix64(uint64_t a, uint64_t b) {
  return splitmix(a ^ (0x9e3779b97f4a7c15ull + (b << 6) + (b >> 2) + splitmix(b)));
}
struct Stream {
  uint64_t key, ctr = 0;
  double normal() {
    double u1 = (double)(mix64(key, ctr++) >> 11) * 0x1.0p-53;
    double u2 = (double)(mix64(key, ctr++) >> 11) * 0x1.0p-53;
    if (u1 <= 0) u1 = 0x1.0p-53;
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
  }
};
// rows x cols, row-major
std::vector<double> orthogonal(int rows, int cols, double gain, Stream s) {
  const int big = std::max(rows, cols), small = std::min(rows, cols);
  std::vector<double> g((size_t)big * small);  // column j at g[i*small + j]
  for (int i = 0; i < big; ++i)
    for (int j = 0; j < small; ++j) g[(size_t)i * small + j] = s.normal();
  std::vector<double> q = g;
  for (int j = 0; j < small; ++j) {
    for (int pass = 0; pass < 2; ++pass) {
      for (int k = 0; k < j; ++k) {
        double d = 0;
        for (int i = 0; i < big; ++i) d += q[(size_t)i * small + k] * q[(size_t)i * small + j];
        for (int i = 0; i < big; ++i) q[(size_t)i * small + j] -= d * q[(size_t)i * small + k];
      }
    }
    double nrm = 0;
    for (int i = 0; i < big; ++i) nrm += q[(size_t)i * small + j] * q[(size_t)i * small + j];
    nrm = std::sqrt(nrm);
    for (int i = 0; i < big; ++i) q[(size_t)i * small + j] /= nrm;
  }
  std::vector<double> out((size_t)rows * cols);
  for (int i = 0; i < big; ++i)
    for (int j = 0; j < small; ++j) {
      const double v = gain * q[(size_t)i * small + j];
      if (rows >= cols) out[(size_t)i * cols + j] = v;
      else out[(size_t)j * cols + i] = v;  // transpose
    }
  return out;
}
}  // namespace

void init_params_host(const ver_model_config& c, uint64_t seed, double* out) {
  const Model m = Model::make(c);
  std::memset(out, 0, sizeof(double) * m.P);
  Stream root{splitmix(seed)};
  auto sub = [&](uint64_t id) { return Stream{mix64(root.key, id)}; };
  const int D = m.D, E = m.E, H = m.H, A = m.A;
  int64_t off = 0;
  auto put = [&](const std::vector<double>& v) {
    std::memcpy(out + off, v.data(), sizeof(double) * v.size());
    off += (int64_t)v.size();
  };
  auto zeros = [&](int64_t n) { off += n; };
  put(orthogonal(D, E, std::sqrt(2.0), sub(1)));
  zeros(E);
  put(orthogonal(E, E, std::sqrt(2.0), sub(2)));
  zeros(E);
  put(orthogonal(E, H, 1.0, sub(3)));
  put(orthogonal(H, H, 1.0, sub(4)));
  zeros(H);
  put(orthogonal(E, H, 1.0, sub(5)));
  put(orthogonal(H, H, 1.0, sub(6)));
  zeros(H);
  put(orthogonal(E, H, 1.0, sub(7)));
  put(orthogonal(H, H, 1.0, sub(8)));
  zeros(H);
  put(orthogonal(H, A, 0.01, sub(9)));
  zeros(A);
  put(orthogonal(H, 1, 1.0, sub(10)));
  zeros(1);
  if (m.continuous) zeros(A);
}

}  // namespace verg

using namespace verg;

extern "C" ver_status ver_debug_gemm(ver_ctx ctx, int engine, int transA, int transB, int M, int N, int K,
                                     const float* A, int lda, const float* B, int ldb, float* C, int splitk) {
  VER_API_BEGIN
  Ctx* c = &ctx->c;
  activate(c);
  const size_t na = transA ? (size_t)K * lda : (size_t)M * lda;
  const size_t nb = transB ? (size_t)N * ldb : (size_t)K * ldb;
  DBuf<float> dA, dB, dC;
  dA.reserve(c, na);
  dB.reserve(c, nb);
  dC.reserve(c, (size_t)M * N);
  dA.upload(A, na);
  dB.upload(B, nb);
  const bool tc0 = c->tensor_cores;
  const int p0 = c->precision;
  c->tensor_cores = engine != 0;
  c->precision = engine == 2 ? 1 : 0;
  Workspace ws;
  ws.ctx = c;
  try {
    auto go = [&](auto ta, auto tb) {
      constexpr bool TA = decltype(ta)::value, TB = decltype(tb)::value;
      if (splitk > 1) gemm_splitk<TA, TB>(c, ws, M, N, K, dA.p, lda, dB.p, ldb, dC.p, N);
      else gemm<TA, TB>(c, M, N, K, dA.p, lda, dB.p, ldb, EpiStore{dC.p, N});
    };
    if (!transA && !transB) go(std::false_type{}, std::false_type{});
    else if (!transA && transB) go(std::false_type{}, std::true_type{});
    else if (transA && !transB) go(std::true_type{}, std::false_type{});
    else go(std::true_type{}, std::true_type{});
  } catch (...) {
    c->tensor_cores = tc0;
    c->precision = p0;
    throw;
  }
  c->tensor_cores = tc0;
  c->precision = p0;
  dC.download(C, (size_t)M * N);
  sync(c);
  VER_API_END
}

extern "C" ver_status ver_debug_gemm_time(ver_ctx ctx, int engine, int transA, int transB, int M, int N, int K,
                                          int splitk, int reps, float* ms_out) {
  VER_API_BEGIN
  Ctx* c = &ctx->c;
  activate(c);
  if (M <= 0 || N <= 0 || K <= 0 || reps <= 0) config_error("debug_gemm_time: bad shape");
  DBuf<float> dA, dB, dC;
  dA.reserve(c, (size_t)M * K);
  dB.reserve(c, (size_t)K * N);
  dC.reserve(c, (size_t)M * N);
  VER_CUDA(cudaMemsetAsync(dA.p, 0x3f, sizeof(float) * (size_t)M * K, c->stream));
  VER_CUDA(cudaMemsetAsync(dB.p, 0x3e, sizeof(float) * (size_t)K * N, c->stream));
  const int lda = transA ? M : K, ldb = transB ? K : N;
  const bool tc0 = c->tensor_cores;
  const int p0 = c->precision;
  c->tensor_cores = engine != 0;
  c->precision = engine == 2 ? 1 : 0;
  Workspace ws;
  ws.ctx = c;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  try {
    VER_CUDA(cudaEventCreate(&e0));
    VER_CUDA(cudaEventCreate(&e1));
    auto go = [&](auto ta, auto tb) {
      constexpr bool TA = decltype(ta)::value, TB = decltype(tb)::value;
      for (int r = 0; r <= reps; ++r) {
        if (r == 1) VER_CUDA(cudaEventRecord(e0, c->stream));
        if (splitk > 1) gemm_splitk<TA, TB>(c, ws, M, N, K, dA.p, lda, dB.p, ldb, dC.p, N);
        else gemm<TA, TB>(c, M, N, K, dA.p, lda, dB.p, ldb, EpiStore{dC.p, N});
      }
      VER_CUDA(cudaEventRecord(e1, c->stream));
    };
    if (!transA && !transB) go(std::false_type{}, std::false_type{});
    else if (!transA && transB) go(std::false_type{}, std::true_type{});
    else if (transA && !transB) go(std::true_type{}, std::false_type{});
    else go(std::true_type{}, std::true_type{});
    VER_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    VER_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    ms_out[0] = ms / reps;
  } catch (...) {
    c->tensor_cores = tc0;
    c->precision = p0;
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    throw;
  }
  c->tensor_cores = tc0;
  c->precision = p0;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  VER_API_END
}

// tcgen05 GEMM wait-cycle counters (tc_gemm.cuh g_tc_prof): on = 1 zeroes and
// enables them, on = 0 disables; `out` (16 values) receives the current sums
extern "C" ver_status ver_debug_gemm_prof(ver_ctx ctx, int on, unsigned long long* out) {
  VER_API_BEGIN
  Ctx* c = &ctx->c;
  activate(c);
  VER_CUDA(cudaStreamSynchronize(c->stream));
  if (out) VER_CUDA(cudaMemcpyFromSymbol(out, tc::g_tc_prof, sizeof(unsigned long long) * 16));
  if (on) {
    unsigned long long z[16] = {};
    VER_CUDA(cudaMemcpyToSymbol(tc::g_tc_prof, z, sizeof(z)));
  }
  const int f = on ? 1 : 0;
  VER_CUDA(cudaMemcpyToSymbol(tc::g_tc_prof_on, &f, sizeof(int)));
  VER_API_END
}
