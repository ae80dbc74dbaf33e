// recurrence.cu — the GRU recurrence over a packed minibatch (nn.cpp:235-250)
// forward and backward as persistent cooperative kernels.
//
// Work split: the H hidden units are cut into UB unit blocks of UPB = 16
// units; the grid is UB x RB CTAs (H = 512: 32 x 4 = 128 CTAs, one per SM).
// A CTA keeps the recurrent weights of its units resident in shared memory
// for the whole minibatch:
//   forward : U[:, gates of its units]   (H x 48 fp32  = 96 KB at H = 512)
//   backward: U[its units, :]            (16 x 3H fp32 = 96 KB)
// Every timestep t the bs_t live rows (a prefix of the rows of t-1, packed
// sorted by length) are re-split across the RB CTAs of each unit block, the
// rows' h_{t-1} (forward) / dhU_t (backward) are staged through shared memory
// from L2, each (row, unit) dot product is split over K by up to 16 threads,
// and one grid-wide barrier separates timesteps.  No launches per timestep.
//
// Forward per (row j, unit u):  r = s(xr + h Ur), z = s(xz + h Uz),
//   n = tanh(xn + r * (h Un)), h' = (1-z) n + z h      (xp holds x W + b)
// Backward per (row j, unit u) at step t-1, fused with step t's
//   dh_{t-1}[j,u] = dhU_t[j,:] . U[u,:] + g_t z_t    (j < bs_t)
//   g = dhidden + dh_{t-1};  dn = g(1-z), dz = g(h-n), dpre_n = dn(1-n^2),
//   dr = dpre_n hUn, dpre_r = dr r(1-r), dpre_z = dz z(1-z)
// so the backward also needs one barrier per timestep.
#include "policy.cuh"

namespace verg {

constexpr int RT = 256;   // threads per CTA
constexpr int UPB = 16;   // units per unit block
constexpr int RCHF = 16;  // forward rows staged per chunk
constexpr int RCHB = 8;   // backward rows staged per chunk

__device__ __forceinline__ void grid_barrier(unsigned* count, unsigned target) {
  __syncthreads();
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

__device__ __forceinline__ float sigm(float x) { return 1.f / (1.f + expf(-x)); }

struct RecGeom {
  int UB, RB;
};
static RecGeom geom(const Ctx* c, int H) {
  RecGeom g;
  g.UB = (H + UPB - 1) / UPB;
  g.RB = std::max(1, c->num_sms / g.UB);
  return g;
}

// ------------------------------------------------------------ forward
__global__ void __launch_bounds__(RT, 1) gru_fwd_persistent(
    int L, const int32_t* __restrict__ bs, const int32_t* __restrict__ offs, int H, int UB, int RB,
    const float* __restrict__ ux, const float* __restrict__ xp, const float* h0, float* hidden,
    float* __restrict__ gates, float* __restrict__ hun, float* __restrict__ hprev_store, unsigned* bar) {
  extern __shared__ float sm[];
  constexpr int US = 3 * UPB + 1;
  float* Us = sm;               // H x US
  float* hs = Us + H * US;      // RCHF x H
  float* red = hs + RCHF * H;   // 16 x UPB x 3
  const int ub = blockIdx.x % UB, rb = blockIdx.x / UB;
  const int u0 = ub * UPB, nu = min(UPB, H - u0);
  const int H3 = 3 * H;
  for (int i = threadIdx.x; i < H * 3 * UPB; i += RT) {
    const int k = i / (3 * UPB), c = i % (3 * UPB);
    Us[k * US + c] = (c / 3 < nu) ? ux[(size_t)k * H3 + 3 * u0 + c] : 0.f;
  }
  __syncthreads();
  const int ul = threadIdx.x % UPB, q = threadIdx.x / UPB;
  unsigned target = 0;
  for (int t = 0; t < L; ++t) {
    const int B = bs[t], o = offs[t];
    const float* hp = (t == 0) ? h0 : hidden + (size_t)offs[t - 1] * H;
    const int rpc = (B + RB - 1) / RB;
    const int r0 = rb * rpc, r1 = min(B, r0 + rpc);
    for (int c0 = r0; c0 < r1; c0 += RCHF) {
      const int nr = min(RCHF, r1 - c0);
      const float* src = hp + (size_t)c0 * H;
      for (int i = threadIdx.x; i < nr * H; i += RT) hs[i] = __ldcg(src + i);
      __syncthreads();
      int nrp = 1;
      while (nrp < nr) nrp <<= 1;
      const int KS = 16 / nrp;
      const int row = q / KS, ks = q % KS;
      float ar = 0.f, az = 0.f, an = 0.f;
      if (row < nr) {
        const int k0 = (ks * H) / KS, k1 = ((ks + 1) * H) / KS;
        const float* hrow = hs + row * H;
        const float* uc = Us + 3 * ul;
#pragma unroll 4
        for (int k = k0; k < k1; ++k) {
          const float h = hrow[k];
          const float* uk = uc + k * US;
          ar = fmaf(h, uk[0], ar);
          az = fmaf(h, uk[1], az);
          an = fmaf(h, uk[2], an);
        }
      }
      float* rq = red + (q * UPB + ul) * 3;
      rq[0] = ar;
      rq[1] = az;
      rq[2] = an;
      __syncthreads();
      if (ks == 0 && row < nr && ul < nu) {
        float sr = 0.f, sz = 0.f, sn = 0.f;
        for (int s = 0; s < KS; ++s) {
          const float* rr = red + ((row * KS + s) * UPB + ul) * 3;
          sr += rr[0];
          sz += rr[1];
          sn += rr[2];
        }
        const int u = u0 + ul;
        const size_t p = (size_t)o + c0 + row;
        const float* x = xp + p * H3 + 3 * u;
        const float r = sigm(x[0] + sr);
        const float z = sigm(x[1] + sz);
        const float n = tanhf(x[2] + r * sn);
        const float hprev = hs[row * H + u];
        hidden[p * H + u] = (1.f - z) * n + z * hprev;
        if (gates) {
          float* gp = gates + p * H3 + 3 * u;
          gp[0] = r;
          gp[1] = z;
          gp[2] = n;
          hun[p * H + u] = sn;
          hprev_store[p * H + u] = hprev;
        }
      }
      __syncthreads();
    }
    target += gridDim.x;
    if (t + 1 < L) grid_barrier(bar, target);
  }
}

// ----------------------------------------------------------- backward
struct GateIn {
  float r, z, n, hn, hp, dh;  // gates, hUn, h_{t-1}, dhidden
};
__device__ __forceinline__ GateIn gate_load(size_t p, int u, int H, const float* __restrict__ gates,
                                           const float* __restrict__ hun, const float* __restrict__ hprev,
                                           const float* __restrict__ dhidden) {
  const float* gp = gates + p * 3 * H + 3 * u;
  return GateIn{__ldg(gp), __ldg(gp + 1), __ldg(gp + 2), __ldg(hun + p * H + u), __ldg(hprev + p * H + u),
                __ldg(dhidden + p * H + u)};
}
__device__ __forceinline__ void gate_grad_v(size_t p, int u, int H, float g, const GateIn& in,
                                            float* __restrict__ dpre, float* __restrict__ dhu,
                                            float* __restrict__ gz) {
  const float dn = g * (1.f - in.z);
  const float dz = g * (in.hp - in.n);
  const float dpn = dn * (1.f - in.n * in.n);
  const float dr = dpn * in.hn;
  const float dpr = dr * in.r * (1.f - in.r);
  const float dpz = dz * in.z * (1.f - in.z);
  float* d = dpre + p * 3 * H + 3 * u;
  d[0] = dpr;
  d[1] = dpz;
  d[2] = dpn;
  float* e = dhu + p * 3 * H + 3 * u;
  e[0] = dpr;
  e[1] = dpz;
  e[2] = dpn * in.r;
  gz[p * H + u] = g * in.z;
}

__device__ __forceinline__ void gate_grad(size_t p, int u, int H, float g, const float* __restrict__ gates,
                                          const float* __restrict__ hun, const float* __restrict__ hprev,
                                          float* __restrict__ dpre, float* __restrict__ dhu,
                                          float* __restrict__ gz) {
  const float* gp = gates + p * 3 * H + 3 * u;
  const float r = gp[0], z = gp[1], n = gp[2];
  const float hn = hun[p * H + u];
  const float hp = hprev[p * H + u];
  const float dn = g * (1.f - z);
  const float dz = g * (hp - n);
  const float dpn = dn * (1.f - n * n);
  const float dr = dpn * hn;
  const float dpr = dr * r * (1.f - r);
  const float dpz = dz * z * (1.f - z);
  float* d = dpre + p * 3 * H + 3 * u;
  d[0] = dpr;
  d[1] = dpz;
  d[2] = dpn;
  float* e = dhu + p * 3 * H + 3 * u;
  e[0] = dpr;
  e[1] = dpz;
  e[2] = dpn * r;
  gz[p * H + u] = g * z;
}

__global__ void __launch_bounds__(RT, 1) gru_bwd_persistent(
    int L, const int32_t* __restrict__ bs, const int32_t* __restrict__ offs, int H, int UB, int RB,
    const float* __restrict__ ux, const float* __restrict__ dhidden, const float* __restrict__ gates,
    const float* __restrict__ hun, const float* __restrict__ hprev, float* dpre, float* dhu, float* gz,
    unsigned* bar) {
  extern __shared__ float sm[];
  const int H3 = 3 * H;
  const int WS = H3 + 1;
  float* Ws = sm;                 // UPB x WS : U rows of this block's units
  float* ds = Ws + UPB * WS;      // RCHB x H3 : staged dhU rows
  float* red = ds + RCHB * H3;    // 16 x UPB
  const int ub = blockIdx.x % UB, rb = blockIdx.x / UB;
  const int u0 = ub * UPB, nu = min(UPB, H - u0);
  for (int i = threadIdx.x; i < UPB * H3; i += RT) {
    const int r = i / H3, c = i % H3;
    Ws[r * WS + c] = r < nu ? ux[(size_t)(u0 + r) * H3 + c] : 0.f;
  }
  __syncthreads();
  const int ul = threadIdx.x % UPB, q = threadIdx.x / UPB;
  unsigned target = 0;
  // step L-1: no carry
  {
    const int B = bs[L - 1], o = offs[L - 1];
    const int rpc = (B + RB - 1) / RB;
    const int r0 = rb * rpc, r1 = min(B, r0 + rpc);
    for (int idx = threadIdx.x; idx < (r1 - r0) * UPB; idx += RT) {
      const int j = r0 + idx / UPB, l = idx % UPB;
      if (l < nu) {
        const size_t p = (size_t)o + j;
        gate_grad(p, u0 + l, H, dhidden[p * H + u0 + l], gates, hun, hprev, dpre, dhu, gz);
      }
    }
  }
  target += gridDim.x;
  if (L > 1) grid_barrier(bar, target);
  for (int t = L - 1; t >= 1; --t) {
    const int B = bs[t], Bp = bs[t - 1], o = offs[t], op = offs[t - 1];
    const int rpc = (Bp + RB - 1) / RB;
    const int r0 = rb * rpc, r1 = min(Bp, r0 + rpc);
    // rows with a successor at step t: dh_{t-1} = dhU_t U^T + g_t z_t
    const int rc1 = min(r1, B);
    for (int c0 = r0; c0 < rc1; c0 += RCHB) {
      const int nr = min(RCHB, rc1 - c0);
      const float* src = dhu + ((size_t)o + c0) * H3;
      for (int i = threadIdx.x; i < nr * H3; i += RT) ds[i] = __ldcg(src + i);
      __syncthreads();
      int nrp = 1;
      while (nrp < nr) nrp <<= 1;
      const int KS = 16 / nrp;
      const int row = q / KS, ks = q % KS;
      float acc = 0.f;
      if (row < nr) {
        const int k0 = (ks * H3) / KS, k1 = ((ks + 1) * H3) / KS;
        const float* drow = ds + row * H3;
        const float* wr = Ws + ul * WS;
#pragma unroll 4
        for (int k = k0; k < k1; ++k) acc = fmaf(drow[k], wr[k], acc);
      }
      red[q * UPB + ul] = acc;
      __syncthreads();
      if (ks == 0 && row < nr && ul < nu) {
        float s = 0.f;
        for (int k = 0; k < KS; ++k) s += red[(row * KS + k) * UPB + ul];
        const int u = u0 + ul;
        const int j = c0 + row;
        const float dh = s + __ldcg(gz + ((size_t)o + j) * H + u);
        const size_t pp = (size_t)op + j;
        gate_grad(pp, u, H, dhidden[pp * H + u] + dh, gates, hun, hprev, dpre, dhu, gz);
      }
      __syncthreads();
    }
    // rows that end at step t-1 (j >= bs_t): gradient from the heads only
    const int re0 = max(r0, B);
    for (int idx = threadIdx.x; idx < max(0, r1 - re0) * UPB; idx += RT) {
      const int j = re0 + idx / UPB, l = idx % UPB;
      if (l < nu) {
        const size_t pp = (size_t)op + j;
        gate_grad(pp, u0 + l, H, dhidden[pp * H + u0 + l], gates, hun, hprev, dpre, dhu, gz);
      }
    }
    target += gridDim.x;
    if (t > 1) grid_barrier(bar, target);
  }
}

// ----------------------------------------- register-resident fast path
// H multiple of 32.  Warp w of a CTA owns units u0+2w, u0+2w+1; lane l owns
// the K indices VEC*l + 32*VEC*i + j (vector shared-memory loads, bank
// conflict free).  The lane keeps its weights in registers for the whole
// minibatch (forward: (H/32) x 2 units x 3 gates = 96 fp32 at H = 512;
// backward: (3H/32) x 2 units = 96), so each staged row costs FMAs against
// vector LDS only.  Rows are processed 4 at a time; the 4 x 2 x 4 (3 gates +
// pad) forward partial sums are reduce-scattered across the 32 lanes in 31
// shuffles (lane l ends with value l), the backward's 4 x 2 in 9.
constexpr int RCF = 32;  // forward rows per staged chunk (32 x H fp32)

template <int NV>
__device__ __forceinline__ void load_vec(const float* p, float* out) {
  if constexpr (NV == 4) {
    const float4 v = *reinterpret_cast<const float4*>(p);
    out[0] = v.x; out[1] = v.y; out[2] = v.z; out[3] = v.w;
  } else if constexpr (NV == 2) {
    const float2 v = *reinterpret_cast<const float2*>(p);
    out[0] = v.x; out[1] = v.y;
  } else {
    out[0] = p[0];
  }
}

// 32 partial sums per lane -> lane l holds the warp total of value l
__device__ __forceinline__ float reduce_scatter32(float* a, int lane) {
#pragma unroll
  for (int s = 16, n = 16; s > 0; s >>= 1, n >>= 1) {
    const bool up = lane & s;
#pragma unroll
    for (int v = 0; v < n; ++v) {
      const float send = up ? a[v] : a[v + n];
      const float keep = up ? a[v + n] : a[v];
      a[v] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  return a[0];
}

template <int H>
__global__ void __launch_bounds__(RT, 1) gru_fwd_reg(
    int L, const int32_t* __restrict__ bs, const int32_t* __restrict__ offs, int UB, int RB,
    const float* __restrict__ ux, const float* __restrict__ xp, const float* h0, float* hidden,
    float* __restrict__ gates, float* __restrict__ hun, float* __restrict__ hprev_store, unsigned* bar) {
  constexpr int H3 = 3 * H;
  constexpr int KPL = H / 32;
  constexpr int VEC = KPL % 4 == 0 ? 4 : (KPL % 2 == 0 ? 2 : 1);
  constexpr int NI = KPL / VEC;
  extern __shared__ float4 sm4[];
  float* hs = reinterpret_cast<float*>(sm4);  // RCF x H
  const int ub = blockIdx.x % UB, rb = blockIdx.x / UB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ua = ub * UPB + 2 * warp;  // units ua, ua + 1
  float w[NI][VEC][2][3];
#pragma unroll
  for (int i = 0; i < NI; ++i)
#pragma unroll
    for (int j = 0; j < VEC; ++j)
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int g = 0; g < 3; ++g)
          w[i][j][q][g] = ux[(size_t)(VEC * lane + 32 * VEC * i + j) * H3 + 3 * (ua + q) + g];
  unsigned target = 0;
  for (int t = 0; t < L; ++t) {
    const int B = bs[t], o = offs[t];
    const float* hp = (t == 0) ? h0 : hidden + (size_t)offs[t - 1] * H;
    const int rpc = (B + RB - 1) / RB;
    const int r0 = rb * rpc, r1 = min(B, r0 + rpc);
    for (int c0 = r0; c0 < r1; c0 += RCF) {
      const int nr = min(RCF, r1 - c0);
      const float4* src = reinterpret_cast<const float4*>(hp + (size_t)c0 * H);
      for (int i = threadIdx.x; i < nr * H / 4; i += RT) sm4[i] = __ldcg(src + i);
      __syncthreads();
      for (int g0 = 0; g0 < nr; g0 += 4) {
        // gate pre-activations of this lane's (row, unit), loaded ahead of the FMAs
        const int pr = lane >> 3, pq = (lane >> 2) & 1;
        const bool owner = (lane & 3) == 0 && g0 + pr < nr;
        float x0 = 0.f, x1 = 0.f, x2 = 0.f;
        if (owner) {
          const float* x = xp + ((size_t)o + c0 + g0 + pr) * H3 + 3 * (ua + pq);
          x0 = __ldg(x);
          x1 = __ldg(x + 1);
          x2 = __ldg(x + 2);
        }
        float acc[32];
#pragma unroll
        for (int v = 0; v < 32; ++v) acc[v] = 0.f;
#pragma unroll
        for (int i = 0; i < NI; ++i) {
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            float h[VEC];
            load_vec<VEC>(hs + (g0 + r) * H + VEC * lane + 32 * VEC * i, h);
#pragma unroll
            for (int j = 0; j < VEC; ++j)
#pragma unroll
              for (int q = 0; q < 2; ++q)
#pragma unroll
                for (int g = 0; g < 3; ++g) acc[r * 8 + q * 4 + g] = fmaf(h[j], w[i][j][q][g], acc[r * 8 + q * 4 + g]);
          }
        }
        const float mine = reduce_scatter32(acc, lane);  // value index = lane = r*8 + q*4 + g
        const float sz = __shfl_down_sync(0xffffffffu, mine, 1);
        const float sn = __shfl_down_sync(0xffffffffu, mine, 2);
        if (owner) {
          const int u = ua + pq;
          const int row = g0 + pr;
          const size_t p = (size_t)o + c0 + row;
          const float rg = sigm(x0 + mine);
          const float zg = sigm(x1 + sz);
          const float ng = tanhf(x2 + rg * sn);
          const float hprev = hs[row * H + u];
          hidden[p * H + u] = (1.f - zg) * ng + zg * hprev;
          if (gates) {
            float* gp = gates + p * H3 + 3 * u;
            gp[0] = rg;
            gp[1] = zg;
            gp[2] = ng;
            hun[p * H + u] = sn;
            hprev_store[p * H + u] = hprev;
          }
        }
      }
      __syncthreads();
    }
    target += gridDim.x;
    if (t + 1 < L) grid_barrier(bar, target);
  }
}

template <int H, int RCB>
__global__ void __launch_bounds__(RT, 1) gru_bwd_reg(
    int L, const int32_t* __restrict__ bs, const int32_t* __restrict__ offs, int UB, int RB,
    const float* __restrict__ ux, const float* __restrict__ dhidden, const float* __restrict__ gates,
    const float* __restrict__ hun, const float* __restrict__ hprev, float* dpre, float* dhu, float* gz,
    unsigned* bar) {
  constexpr int H3 = 3 * H;
  constexpr int CPL = H3 / 32;  // columns per lane
  constexpr int VEC = CPL % 4 == 0 ? 4 : (CPL % 2 == 0 ? 2 : 1);
  constexpr int NI = CPL / VEC;
  extern __shared__ float4 sm4[];
  float* ds = reinterpret_cast<float*>(sm4);  // RCB x H3
  const int ub = blockIdx.x % UB, rb = blockIdx.x / UB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ua = ub * UPB + 2 * warp;
  float w[NI][VEC][2];
#pragma unroll
  for (int i = 0; i < NI; ++i)
#pragma unroll
    for (int j = 0; j < VEC; ++j)
#pragma unroll
      for (int q = 0; q < 2; ++q) w[i][j][q] = ux[(size_t)(ua + q) * H3 + VEC * lane + 32 * VEC * i + j];
  unsigned target = 0;
  {
    const int B = bs[L - 1], o = offs[L - 1];
    const int rpc = (B + RB - 1) / RB;
    const int r0 = rb * rpc, r1 = min(B, r0 + rpc);
    for (int idx = threadIdx.x; idx < (r1 - r0) * UPB; idx += RT) {
      const int j = r0 + idx / UPB, l = idx % UPB;
      const size_t p = (size_t)o + j;
      gate_grad(p, ub * UPB + l, H, dhidden[p * H + ub * UPB + l], gates, hun, hprev, dpre, dhu, gz);
    }
  }
  target += gridDim.x;
  if (L > 1) grid_barrier(bar, target);
  for (int t = L - 1; t >= 1; --t) {
    const int B = bs[t], Bp = bs[t - 1], o = offs[t], op = offs[t - 1];
    const int rpc = (Bp + RB - 1) / RB;
    const int r0 = rb * rpc, r1 = min(Bp, r0 + rpc);
    const int rc1 = min(r1, B);
    for (int c0 = r0; c0 < rc1; c0 += RCB) {
      const int nr = min(RCB, rc1 - c0);
      const float4* src = reinterpret_cast<const float4*>(dhu + ((size_t)o + c0) * H3);
      for (int i = threadIdx.x; i < nr * H3 / 4; i += RT) sm4[i] = __ldcg(src + i);
      __syncthreads();
      for (int g0 = 0; g0 < nr; g0 += 4) {
        // this lane's (row, unit) operands for the gate gradient, loaded ahead of the FMAs
        const int pv = lane >> 2, pr = pv >> 1, pq = pv & 1;
        const bool owner = (lane & 3) == 0 && g0 + pr < nr;
        GateIn gin{};
        float gzv = 0.f;
        if (owner) {
          const size_t pp = (size_t)op + c0 + g0 + pr;
          gin = gate_load(pp, ua + pq, H, gates, hun, hprev, dhidden);
          gzv = __ldcg(gz + ((size_t)o + c0 + g0 + pr) * H + ua + pq);
        }
        float acc[8];
#pragma unroll
        for (int v = 0; v < 8; ++v) acc[v] = 0.f;
#pragma unroll
        for (int i = 0; i < NI; ++i) {
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            float d[VEC];
            load_vec<VEC>(ds + (g0 + r) * H3 + VEC * lane + 32 * VEC * i, d);
#pragma unroll
            for (int j = 0; j < VEC; ++j)
#pragma unroll
              for (int q = 0; q < 2; ++q) acc[r * 2 + q] = fmaf(d[j], w[i][j][q], acc[r * 2 + q]);
          }
        }
        // reduce-scatter 8 values over lane bits 16, 8, 4; then xor over bits 2, 1
#pragma unroll
        for (int s = 16, n = 4; s >= 4; s >>= 1, n >>= 1) {
          const bool up = lane & s;
#pragma unroll
          for (int v = 0; v < n; ++v) {
            const float send = up ? acc[v] : acc[v + n];
            const float keep = up ? acc[v + n] : acc[v];
            acc[v] = keep + __shfl_xor_sync(0xffffffffu, send, s);
          }
        }
        float tot = acc[0];
        tot += __shfl_xor_sync(0xffffffffu, tot, 2);
        tot += __shfl_xor_sync(0xffffffffu, tot, 1);
        if (owner) {  // lane holds value pv = r * 2 + q
          const size_t pp = (size_t)op + c0 + g0 + pr;
          gate_grad_v(pp, ua + pq, H, gin.dh + tot + gzv, gin, dpre, dhu, gz);
        }
      }
      __syncthreads();
    }
    const int re0 = max(r0, B);
    for (int idx = threadIdx.x; idx < max(0, r1 - re0) * UPB; idx += RT) {
      const int j = re0 + idx / UPB, l = idx % UPB;
      const size_t pp = (size_t)op + j;
      gate_grad(pp, ub * UPB + l, H, dhidden[pp * H + ub * UPB + l], gates, hun, hprev, dpre, dhu, gz);
    }
    target += gridDim.x;
    if (t > 1) grid_barrier(bar, target);
  }
}

template <int H>
static const void* fwd_reg_fn() {
  return reinterpret_cast<const void*>(gru_fwd_reg<H>);
}
constexpr int RCB = 32;  // backward rows per staged chunk (32 x 3H fp32 = 192 KB at H = 512)
template <int H>
static const void* bwd_reg_fn() {
  return reinterpret_cast<const void*>(gru_bwd_reg<H, RCB>);
}
static const void* pick_fwd(int H) {
  switch (H) {
    case 32: return fwd_reg_fn<32>();
    case 64: return fwd_reg_fn<64>();
    case 96: return fwd_reg_fn<96>();
    case 128: return fwd_reg_fn<128>();
    case 256: return fwd_reg_fn<256>();
    case 512: return fwd_reg_fn<512>();
    default: return nullptr;
  }
}
static const void* pick_bwd(int H) {
  switch (H) {
    case 32: return bwd_reg_fn<32>();
    case 64: return bwd_reg_fn<64>();
    case 96: return bwd_reg_fn<96>();
    case 128: return bwd_reg_fn<128>();
    case 256: return bwd_reg_fn<256>();
    case 512: return bwd_reg_fn<512>();
    default: return nullptr;
  }
}

// ------------------------------------------------------------ launch
static void coop_launch(Ctx* c, const void* fn, int grid, size_t smem, void** args) {
  ScopedEv ev(c, c->rec_tag);
  VER_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  VER_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, RT, smem));
  if (per_sm * c->num_sms < grid)
    config_error("recurrence: grid does not fit co-resident (hidden dim too large for this build)");
  VER_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(RT), args, smem, c->stream));
  after_launch(c);
}

void gru_forward_recurrence(Ctx* c, const Model& m, const float* params, int L, const int32_t* d_bs,
                            const int32_t* d_offs, Workspace& ws, const float* h0, bool store) {
  const RecGeom g = geom(c, m.H);
  const int grid = g.UB * g.RB;
  ws.bar.reserve(c, 1);
  ws.bar.zero(1);
  int H = m.H, UB = g.UB, RB = g.RB;
  const float* ux = params + m.o_ux;
  const float* xp = ws.xp.p;
  float* hidden = ws.hidden.p;
  float* gates = store ? ws.gates.p : nullptr;
  float* hun = ws.hu.p;
  float* hps = ws.hprev.p;
  unsigned* bar = ws.bar.p;
  if (const void* fn = pick_fwd(m.H)) {
    const size_t smem = sizeof(float) * (size_t)RCF * m.H;
    void* args[] = {&L, &d_bs, &d_offs, &UB, &RB, &ux, &xp, &h0, &hidden, &gates, &hun, &hps, &bar};
    coop_launch(c, fn, grid, smem, args);
    return;
  }
  const size_t smem = sizeof(float) * ((size_t)m.H * (3 * UPB + 1) + (size_t)RCHF * m.H + 16 * UPB * 3);
  void* args[] = {&L, &d_bs, &d_offs, &H, &UB, &RB, &ux, &xp, &h0, &hidden, &gates, &hun, &hps, &bar};
  coop_launch(c, reinterpret_cast<const void*>(gru_fwd_persistent), grid, smem, args);
}

void gru_backward_recurrence(Ctx* c, const Model& m, const float* params, int L, const int32_t* d_bs,
                             const int32_t* d_offs, Workspace& ws) {
  const RecGeom g = geom(c, m.H);
  const int grid = g.UB * g.RB;
  ws.bar.reserve(c, 1);
  ws.bar.zero(1);
  int H = m.H, UB = g.UB, RB = g.RB;
  const float* ux = params + m.o_ux;
  const float* dh = ws.dhidden.p;
  const float* gates = ws.gates.p;
  const float* hun = ws.hu.p;
  const float* hps = ws.hprev.p;
  float* dpre = ws.dpre.p;
  float* dhu = ws.dhu.p;
  float* gz = ws.g.p;
  unsigned* bar = ws.bar.p;
  if (const void* fn = pick_bwd(m.H)) {
    const size_t smem = sizeof(float) * (size_t)RCB * 3 * m.H;
    void* args[] = {&L, &d_bs, &d_offs, &UB, &RB, &ux, &dh, &gates, &hun, &hps, &dpre, &dhu, &gz, &bar};
    coop_launch(c, fn, grid, smem, args);
    return;
  }
  const size_t smem = sizeof(float) * ((size_t)UPB * (3 * m.H + 1) + (size_t)RCHB * 3 * m.H + 16 * UPB);
  void* args[] = {&L, &d_bs, &d_offs, &H, &UB, &RB, &ux, &dh, &gates, &hun, &hps, &dpre, &dhu, &gz, &bar};
  coop_launch(c, reinterpret_cast<const void*>(gru_bwd_persistent), grid, smem, args);
}

}  // namespace verg
