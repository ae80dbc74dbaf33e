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
#include <cstdlib>

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
        const float r = gate_sigm(x[0] + sr);
        const float z = gate_sigm(x[1] + sz);
        const float n = gate_tanh(x[2] + r * sn);
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

// Row groups: packed row j of any timestep belongs to row block j % RB for
// the whole minibatch (rows of step t are a prefix of the rows of t-1, so the
// interleave stays balanced as bs_t shrinks).  Row j's recurrence only reads
// row j, so row block rb depends only on its own UB unit-block CTAs: each row
// block synchronises on its own counter (UB arrivals per step) and the row
// blocks run independently.  A row block whose rows have all ended leaves.
__device__ __forceinline__ void group_barrier(unsigned* count, unsigned target) {
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
constexpr int kBarStride = 32;  // one 128-byte line per row-block counter

__device__ __forceinline__ int rows_of(int B, int rb, int RB) { return B > rb ? (B - rb + RB - 1) / RB : 0; }
// rows [lo, hi) of step-t rows 0..B-1 owned by row block rb: interleaved
// (j = rb + RB i, independent row-block groups) or contiguous ranges (all
// CTAs synchronise every step, VER_REC_MODE=1: A/B measurements)
struct RowMap {
  int base, stride, n;
  __device__ __forceinline__ int row(int i) const { return base + stride * i; }
};
__device__ __forceinline__ RowMap rows_in(int inter, int B, int rb, int RB, int lo, int hi) {
  // the rows j in [lo, hi) with j < B of row block rb
  if (inter) {
    const int a = rows_of(lo, rb, RB), b = rows_of(min(hi, B), rb, RB);
    return RowMap{rb + RB * a, RB, max(0, b - a)};
  }
  const int rpc = (B + RB - 1) / RB;
  const int r0 = max(lo, rb * rpc), r1 = min(min(hi, B), rb * rpc + rpc);
  return RowMap{r0, 1, max(0, r1 - r0)};
}

template <int H>
__global__ void __launch_bounds__(RT, 1) gru_fwd_reg(
    int L, const int32_t* __restrict__ bs, const int32_t* __restrict__ offs, int UB, int RB,
    const float* __restrict__ ux, const float* __restrict__ xp, const float* h0, float* hidden,
    float* __restrict__ gates, float* __restrict__ hun, float* __restrict__ hprev_store, unsigned* bar,
    int inter) {
  constexpr int H3 = 3 * H;
  constexpr int KPL = H / 32;
  constexpr int VEC = KPL % 4 == 0 ? 4 : (KPL % 2 == 0 ? 2 : 1);
  constexpr int NI = KPL / VEC;
  extern __shared__ float4 sm4[];
  float* hs = reinterpret_cast<float*>(sm4);  // RCF x H
  const int ub = blockIdx.x % UB, rb = blockIdx.x / UB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ua = ub * UPB + 2 * warp;  // units ua, ua + 1
  unsigned* cnt = inter ? bar + rb * kBarStride : bar;
  const unsigned arrivals = inter ? UB : gridDim.x;
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
    const RowMap rm = rows_in(inter, bs[t], rb, RB, 0, 1 << 30);
    const int nrows = rm.n;
    if (inter && nrows == 0) break;  // bs is non-increasing: this row block is done
    if (t > 0) {
      target += arrivals;
      group_barrier(cnt, target);
    }
    const int o = offs[t];
    const float* hp = (t == 0) ? h0 : hidden + (size_t)offs[t - 1] * H;
    for (int c0 = 0; c0 < nrows; c0 += RCF) {
      const int nr = min(RCF, nrows - c0);
      const float4* src = reinterpret_cast<const float4*>(hp);
      for (int i = threadIdx.x; i < nr * H / 4; i += RT) {
        const int r = i / (H / 4), k = i % (H / 4);
        sm4[i] = __ldcg(src + (size_t)rm.row(c0 + r) * (H / 4) + k);
      }
      __syncthreads();
      for (int g0 = 0; g0 < nr; g0 += 4) {
        // gate pre-activations of this lane's (row, unit), loaded ahead of the FMAs
        const int pr = lane >> 3, pq = (lane >> 2) & 1;
        const bool owner = (lane & 3) == 0 && g0 + pr < nr;
        const size_t p = (size_t)o + rm.row(c0 + g0 + pr);
        float x0 = 0.f, x1 = 0.f, x2 = 0.f;
        if (owner) {
          const float* x = xp + p * H3 + 3 * (ua + pq);
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
          const float rg = gate_sigm(x0 + mine);
          const float zg = gate_sigm(x1 + sz);
          const float ng = gate_tanh(x2 + rg * sn);
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
  }
}

template <int H, int RCB>
__global__ void __launch_bounds__(RT, 1) gru_bwd_reg(
    int L, const int32_t* __restrict__ bs, const int32_t* __restrict__ offs, int UB, int RB,
    const float* __restrict__ ux, const float* __restrict__ dhidden, const float* __restrict__ gates,
    const float* __restrict__ hun, const float* __restrict__ hprev, float* dpre, float* dhu, float* gz,
    unsigned* bar, int inter) {
  constexpr int H3 = 3 * H;
  constexpr int CPL = H3 / 32;  // columns per lane
  constexpr int VEC = CPL % 4 == 0 ? 4 : (CPL % 2 == 0 ? 2 : 1);
  constexpr int NI = CPL / VEC;
  extern __shared__ float4 sm4[];
  float* ds = reinterpret_cast<float*>(sm4);  // RCB x H3
  const int ub = blockIdx.x % UB, rb = blockIdx.x / UB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ua = ub * UPB + 2 * warp;
  unsigned* cnt = inter ? bar + rb * kBarStride : bar;
  const unsigned arrivals = inter ? UB : gridDim.x;
  float w[NI][VEC][2];
#pragma unroll
  for (int i = 0; i < NI; ++i)
#pragma unroll
    for (int j = 0; j < VEC; ++j)
#pragma unroll
      for (int q = 0; q < 2; ++q) w[i][j][q] = ux[(size_t)(ua + q) * H3 + VEC * lane + 32 * VEC * i + j];
  unsigned target = 0;
  bool any = false;  // has this row block produced rows yet (then later steps need a barrier)
  {
    const RowMap rm = rows_in(inter, bs[L - 1], rb, RB, 0, 1 << 30);
    const int n = rm.n, o = offs[L - 1];
    for (int idx = threadIdx.x; idx < n * UPB; idx += RT) {
      const int j = rm.row(idx / UPB), l = idx % UPB;
      const size_t p = (size_t)o + j;
      gate_grad(p, ub * UPB + l, H, dhidden[p * H + ub * UPB + l], gates, hun, hprev, dpre, dhu, gz);
    }
    any = n > 0 || !inter;
  }
  for (int t = L - 1; t >= 1; --t) {
    const int B = bs[t], Bp = bs[t - 1], o = offs[t], op = offs[t - 1];
    const RowMap rc = rows_in(inter, Bp, rb, RB, 0, B);   // rows with a successor at step t
    const RowMap re = rows_in(inter, Bp, rb, RB, B, Bp);  // rows that end at step t-1
    const int nc = rc.n;
    if (inter && nc + re.n == 0) continue;  // nothing yet for this row block (bs grows as t falls)
    if (any) {
      target += arrivals;
      group_barrier(cnt, target);
    }
    any = true;
    // rows with a successor at step t: dh_{t-1} = dhU_t U^T + g_t z_t
    for (int c0 = 0; c0 < nc; c0 += RCB) {
      const int nr = min(RCB, nc - c0);
      const float4* src = reinterpret_cast<const float4*>(dhu + (size_t)o * H3);
      for (int i = threadIdx.x; i < nr * H3 / 4; i += RT) {
        const int r = i / (H3 / 4), k = i % (H3 / 4);
        sm4[i] = __ldcg(src + (size_t)rc.row(c0 + r) * (H3 / 4) + k);
      }
      __syncthreads();
      for (int g0 = 0; g0 < nr; g0 += 4) {
        // this lane's (row, unit) operands for the gate gradient, loaded ahead of the FMAs
        const int pv = lane >> 2, pr = pv >> 1, pq = pv & 1;
        const bool owner = (lane & 3) == 0 && g0 + pr < nr;
        const int j = rc.row(c0 + g0 + pr);
        GateIn gin{};
        float gzv = 0.f;
        if (owner) {
          gin = gate_load((size_t)op + j, ua + pq, H, gates, hun, hprev, dhidden);
          gzv = __ldcg(gz + ((size_t)o + j) * H + ua + pq);
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
            for (int jj = 0; jj < VEC; ++jj)
#pragma unroll
              for (int q = 0; q < 2; ++q) acc[r * 2 + q] = fmaf(d[jj], w[i][jj][q], acc[r * 2 + q]);
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
        if (owner)  // lane holds value pv = r * 2 + q
          gate_grad_v((size_t)op + j, ua + pq, H, gin.dh + tot + gzv, gin, dpre, dhu, gz);
      }
      __syncthreads();
    }
    // rows that end at step t-1 (j >= bs_t): gradient from the heads only
    for (int idx = threadIdx.x; idx < re.n * UPB; idx += RT) {
      const int j = re.row(idx / UPB), l = idx % UPB;
      const size_t pp = (size_t)op + j;
      gate_grad(pp, ub * UPB + l, H, dhidden[pp * H + ub * UPB + l], gates, hun, hprev, dpre, dhu, gz);
    }
  }
}

// ------------------------------------------ K-split fast path (H % 256 == 0)
// The register kernels above give every warp 2 units and the whole K range,
// so each staged row is read from shared memory by all 8 warps and each
// value feeds 2 (backward) or 6 (forward) FMAs: the backward is bound by
// shared-memory bandwidth.  Here warp w owns the K slice [w KW, (w+1) KW)
// for ALL 16 units of the CTA, lane (cq = lane / 8, kq = lane % 8) owns
// KL = KW / 8 K indices (k = w KW + 4 kq + 32 i + v) of 4 units (cq): each
// staged value is read once per CTA (broadcast to the 4 cq lanes) and feeds
// 12 (forward: 4 units x 3 gates) or 4 (backward) FMAs per lane, i.e. the
// CTA does 48 / 16 FMAs per shared-memory word instead of 6 / 2.  Partial sums
// are reduce-scattered over the 8 kq lanes by shuffles, then over the 8 warps
// through shared memory by the threads that apply the gate math.  Rows are
// staged with TMA bulk copies (one per row) into a 2-deep ring, so the next
// chunk of a step lands while this one is computed.
__device__ __forceinline__ void bulk_row(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(mbar)
               : "memory");
}
__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mb_init(uint32_t a, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(n) : "memory");
}
__device__ __forceinline__ void mb_expect(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_wait(uint32_t a, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "RW_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra RW_WAIT;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}
// stage rows map.row(c0 .. c0+nr-1) of src (row stride `row_floats`) into dst
__device__ __forceinline__ void stage_rows(float* dst, const float* src, int row_floats, const RowMap& rm, int c0,
                                           int nr, uint32_t mbar) {
  const uint32_t bytes = (uint32_t)row_floats * 4u;
  mb_expect(mbar, bytes * (uint32_t)nr);
  for (int r = 0; r < nr; ++r)
    bulk_row(su32(dst + (size_t)r * row_floats), src + (size_t)rm.row(c0 + r) * row_floats, bytes, mbar);
}

// the same by the 32 lanes of one warp: lane 0 posts the byte count, then the
// lanes issue the row copies in parallel (one issuing thread serialises them)
__device__ __forceinline__ void stage_rows_warp(float* dst, const float* src, int row_floats, const RowMap& rm,
                                                int c0, int nr, uint32_t mbar) {
  const int lane = threadIdx.x & 31;
  const uint32_t bytes = (uint32_t)row_floats * 4u;
  if (lane == 0) mb_expect(mbar, bytes * (uint32_t)nr);
  __syncwarp();
  for (int r = lane; r < nr; r += 32)
    bulk_row(su32(dst + (size_t)r * row_floats), src + (size_t)rm.row(c0 + r) * row_floats, bytes, mbar);
}

__device__ __forceinline__ long long globaltimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

constexpr int ks_fr(int nw) { return nw == 16 ? 24 : 32; }  // forward rows per chunk (smem)
constexpr int KS_BR = 16;  // backward rows per chunk

// values a[0..2n) over the lanes differing in bit s: keep half, add the partner's other half
template <int N>
__device__ __forceinline__ void rs_level(float* a, int lane, int s) {
  const bool up = lane & s;
#pragma unroll
  for (int v = 0; v < N; ++v) {
    const float send = up ? a[v] : a[v + N];
    const float keep = up ? a[v + N] : a[v];
    a[v] = keep + __shfl_xor_sync(0xffffffffu, send, s);
  }
}

// Forward lane layout: kq = lane % 2, cq = lane / 2 = unit u0 + cq (3 gate
// columns); lane K indices k = w KW + 8 i + 4 kq + v, so one LDS.128 per lane
// feeds 12 FMAs and the reduction over kq is one shuffle level.
template <int H, int NW>
__global__ void __launch_bounds__(NW * 32, 1) gru_fwd_ks(
    int L, const int32_t* __restrict__ bs, const int32_t* __restrict__ offs, int UB, int RB,
    const float* __restrict__ ux, const float* __restrict__ xp, const float* h0, float* hidden,
    float* __restrict__ gates, float* __restrict__ hun, float* __restrict__ hprev_store, unsigned* bar,
    long long* trace, int t_begin, unsigned long long* hx, int tag_th, unsigned epoch) {
  constexpr int H3 = 3 * H, NT = NW * 32;
  constexpr int KS_FR = ks_fr(NW);
  constexpr int KW = H / NW, NI = KW / 8;
  static_assert(KW % 8 == 0, "forward K slice");
  constexpr int NC = 3 * UPB;  // 48 gate columns of the CTA
  constexpr int PPT = (KS_FR * UPB + NT - 1) / NT;  // (row, unit) pairs per thread per chunk
  extern __shared__ float4 sm4[];
  float* hs = reinterpret_cast<float*>(sm4);   // [2][KS_FR][H]
  float* red = hs + 2 * KS_FR * H;             // [NW][KS_FR][NC]
  uint64_t* mbar = reinterpret_cast<uint64_t*>(red + NW * KS_FR * NC);
  const int ub = blockIdx.x % UB, rb = blockIdx.x / UB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kq = lane & 1, cq = lane >> 1;
  const int u0 = ub * UPB;
  unsigned* cnt = bar + rb * kBarStride;
  if (threadIdx.x == 0) {
    mb_init(su32(&mbar[0]), 1);
    mb_init(su32(&mbar[1]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  float w[NI][4][3];
#pragma unroll
  for (int i = 0; i < NI; ++i)
#pragma unroll
    for (int v = 0; v < 4; ++v)
#pragma unroll
      for (int g = 0; g < 3; ++g)
        w[i][v][g] = ux[(size_t)(warp * KW + 8 * i + 4 * kq + v) * H3 + 3 * (u0 + cq) + g];
  __syncthreads();
  unsigned target = 0;
  uint32_t phase = 0;  // bit b: parity of the next completion of mbar[b]
  int buf = 0;
  float xr[PPT][3];
  // x W + b of this thread's (row, unit) pairs of chunk [c0, c0 + nr): loaded a chunk ahead
  auto load_x = [&](const RowMap& rm, int o, int c0, int nr) {
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      const int pidx = threadIdx.x + k * NT;
      if (pidx < nr * UPB) {
        const float* x = xp + ((size_t)o + rm.row(c0 + pidx / UPB)) * H3 + 3 * (u0 + pidx % UPB);
        xr[k][0] = __ldg(x);
        xr[k][1] = __ldg(x + 1);
        xr[k][2] = __ldg(x + 2);
      }
    }
  };
  // Short steps (bs_t <= tag_th) skip the group barrier and the bulk staging:
  // the producers of h_{t-1} also write each value with its step tag into hx
  // (64-bit words: tag << 32 | bits), and the consumers poll those words
  // straight into shared memory, so data and synchronisation take one L2
  // round trip instead of two.  hx is double-buffered by step parity (a CTA
  // reaches step t+1 only after every CTA of its group wrote h_t, i.e. after
  // they all finished reading h_{t-1}); the host zeroes it per launch and the
  // tag (epoch * 4096 + t) is unique within and across launches.
  auto tagged = [&](int s) { return s > t_begin && s < L && bs[s] <= tag_th; };
  for (int t = t_begin; t < L; ++t) {
    const RowMap rm = rows_in(1, bs[t], rb, RB, 0, 1 << 30);
    if (rm.n == 0) break;  // bs is non-increasing: this row block is done
    const int o = offs[t];
    const bool tag_in = tagged(t), tag_out = tagged(t + 1);
    load_x(rm, o, 0, min(KS_FR, rm.n));
    if (t > t_begin && !tag_in) {
      target += UB;
      group_barrier(cnt, target);
    }
    if (trace && blockIdx.x == 0 && threadIdx.x == 0) trace[t] = globaltimer();
    const float* hp = (t == 0) ? h0 : hidden + (size_t)offs[t - 1] * H;
    const int nch = (rm.n + KS_FR - 1) / KS_FR;
    if (threadIdx.x < 32 && !tag_in) {
      asm volatile("fence.proxy.async.global;" ::: "memory");  // generic stores of other CTAs -> bulk-copy reads
      stage_rows_warp(hs + buf * KS_FR * H, hp, H, rm, 0, min(KS_FR, rm.n), su32(&mbar[buf]));
    }
    for (int ch = 0; ch < nch; ++ch) {
      const int c0 = ch * KS_FR, nr = min(KS_FR, rm.n - c0);
      if (tag_in) {  // one chunk: rm.n <= tag_th / RB <= KS_FR
        const unsigned want = epoch * 4096u + (unsigned)(t - 1);
        const unsigned long long* src = hx + (size_t)((t - 1) & 1) * tag_th * H;
        float* dst = hs + buf * KS_FR * H;
        for (int i = threadIdx.x; i < nr * (H / 2); i += NT) {
          const int r = i / (H / 2), k2 = 2 * (i % (H / 2));
          const unsigned long long* a = src + (size_t)rm.row(c0 + r) * H + k2;
          unsigned long long v0, v1;
          do {
            asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(v0), "=l"(v1) : "l"(a) : "memory");
          } while ((unsigned)(v0 >> 32) != want || (unsigned)(v1 >> 32) != want);
          *reinterpret_cast<float2*>(dst + r * H + k2) =
              make_float2(__uint_as_float((unsigned)v0), __uint_as_float((unsigned)v1));
        }
        __syncthreads();
      } else {
        if (threadIdx.x < 32 && ch + 1 < nch)
          stage_rows_warp(hs + (buf ^ 1) * KS_FR * H, hp, H, rm, c0 + KS_FR, min(KS_FR, rm.n - c0 - KS_FR),
                          su32(&mbar[buf ^ 1]));
        mb_wait(su32(&mbar[buf]), (phase >> buf) & 1);
        phase ^= 1u << buf;
      }
      const float* hc = hs + buf * KS_FR * H;
      for (int g0 = 0; g0 < nr; g0 += 4) {
        float acc[12];
#pragma unroll
        for (int v = 0; v < 12; ++v) acc[v] = 0.f;
#pragma unroll
        for (int i = 0; i < NI; ++i) {
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const float4 h4 = *reinterpret_cast<const float4*>(hc + (g0 + r) * H + warp * KW + 8 * i + 4 * kq);
            const float hv[4] = {h4.x, h4.y, h4.z, h4.w};
#pragma unroll
            for (int v = 0; v < 4; ++v)
#pragma unroll
              for (int g = 0; g < 3; ++g) acc[r * 3 + g] = fmaf(hv[v], w[i][v][g], acc[r * 3 + g]);
          }
        }
        // reduce over kq: lane keeps values 6 kq .. 6 kq + 5 = rows 2 kq, 2 kq + 1, gates 0..2
        rs_level<6>(acc, lane, 1);
        float* dst = red + ((size_t)warp * KS_FR + g0 + 2 * kq) * NC + 3 * cq;
        dst[0] = acc[0];
        dst[1] = acc[1];
        dst[2] = acc[2];
        dst[NC] = acc[3];
        dst[NC + 1] = acc[4];
        dst[NC + 2] = acc[5];
      }
      __syncthreads();
      // gate math: (row, unit) pairs, partials summed over the 8 warps
#pragma unroll
      for (int k = 0; k < PPT; ++k) {
        const int pidx = threadIdx.x + k * NT;
        if (pidx >= nr * UPB) continue;
        const int row = pidx / UPB, ul = pidx % UPB;
        float sr = 0.f, sz = 0.f, sn = 0.f;
#pragma unroll
        for (int q = 0; q < NW; ++q) {
          const float* rq = red + ((size_t)q * KS_FR + row) * NC + 3 * ul;
          sr += rq[0];
          sz += rq[1];
          sn += rq[2];
        }
        const int u = u0 + ul;
        const size_t p = (size_t)o + rm.row(c0 + row);
        const float rg = gate_sigm(xr[k][0] + sr);
        const float zg = gate_sigm(xr[k][1] + sz);
        const float ng = gate_tanh(xr[k][2] + rg * sn);
        const float hprev = hc[row * H + u];
        const float hnew = (1.f - zg) * ng + zg * hprev;
        hidden[p * H + u] = hnew;
        const int jrow = rm.row(c0 + row);
        if (tag_out && jrow < bs[t + 1])
          hx[((size_t)(t & 1) * tag_th + jrow) * H + u] =
              ((unsigned long long)(epoch * 4096u + (unsigned)t) << 32) | __float_as_uint(hnew);
        if (gates) {
          float* gp = gates + p * H3 + 3 * u;
          gp[0] = rg;
          gp[1] = zg;
          gp[2] = ng;
          hun[p * H + u] = sn;
          hprev_store[p * H + u] = hprev;
        }
      }
      if (ch + 1 < nch) load_x(rm, o, c0 + KS_FR, min(KS_FR, rm.n - c0 - KS_FR));
      __syncthreads();
      buf ^= 1;
    }
  }
}

template <int H, int NW>
__global__ void __launch_bounds__(NW * 32, 1) gru_bwd_ks(
    int L, const int32_t* __restrict__ bs, const int32_t* __restrict__ offs, int UB, int RB,
    const float* __restrict__ ux, const float* __restrict__ dhidden, const float* __restrict__ gates,
    const float* __restrict__ hun, const float* __restrict__ hprev, float* dpre, float* dhu, float* gz,
    unsigned* bar, long long* trace, int t_start, int do_init, int t_stop) {
  constexpr int H3 = 3 * H, NT = NW * 32;
  constexpr int KW = H3 / NW, KL = KW / 8, NV = KL / 4;
  static_assert(KL % 4 == 0, "backward K slice");
  extern __shared__ float4 sm4[];
  float* ds = reinterpret_cast<float*>(sm4);   // [2][KS_BR][H3]
  float* red = ds + 2 * KS_BR * H3;            // [NW][KS_BR][UPB]
  uint64_t* mbar = reinterpret_cast<uint64_t*>(red + NW * KS_BR * UPB);
  const int ub = blockIdx.x % UB, rb = blockIdx.x / UB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kq = lane & 7, cq = lane >> 3;
  const int u0 = ub * UPB;
  unsigned* cnt = bar + rb * kBarStride;
  if (threadIdx.x == 0) {
    mb_init(su32(&mbar[0]), 1);
    mb_init(su32(&mbar[1]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // w[i][v][c] = U[u0 + 4 cq + c, k], k = warp KW + 4 kq + 32 i + v
  float w[NV][4][4];
#pragma unroll
  for (int i = 0; i < NV; ++i)
#pragma unroll
    for (int v = 0; v < 4; ++v)
#pragma unroll
      for (int c = 0; c < 4; ++c)
        w[i][v][c] = ux[(size_t)(u0 + 4 * cq + c) * H3 + warp * KW + 4 * kq + 32 * i + v];
  __syncthreads();
  unsigned target = 0;
  uint32_t phase = 0;
  int buf = 0;
  bool any = false;
  if (do_init) {  // step L-1: no carry (else the cluster tail kernel ran steps > t_start)
    const RowMap rm = rows_in(1, bs[L - 1], rb, RB, 0, 1 << 30);
    const int o = offs[L - 1];
    for (int idx = threadIdx.x; idx < rm.n * UPB; idx += NT) {
      const int j = rm.row(idx / UPB), l = idx % UPB;
      const size_t p = (size_t)o + j;
      gate_grad(p, u0 + l, H, dhidden[p * H + u0 + l], gates, hun, hprev, dpre, dhu, gz);
    }
    any = rm.n > 0;
  }
  for (int t = t_start; t > t_stop; --t) {
    const int B = bs[t], Bp = bs[t - 1], o = offs[t], op = offs[t - 1];
    const RowMap rc = rows_in(1, Bp, rb, RB, 0, B);   // rows with a successor at step t
    const RowMap re = rows_in(1, Bp, rb, RB, B, Bp);  // rows that end at step t-1
    if (rc.n + re.n == 0) continue;
    if (any) {
      target += UB;
      group_barrier(cnt, target);
    }
    any = true;
    if (trace && blockIdx.x == 0 && threadIdx.x == 0) trace[t] = globaltimer();
    const float* src = dhu + (size_t)o * H3;
    const int nch = (rc.n + KS_BR - 1) / KS_BR;
    if (threadIdx.x < 32 && nch > 0) {
      asm volatile("fence.proxy.async.global;" ::: "memory");
      stage_rows_warp(ds + buf * KS_BR * H3, src, H3, rc, 0, min(KS_BR, rc.n), su32(&mbar[buf]));
    }
    // rows that end at step t-1 (j >= bs_t): gradient from the heads only (overlaps the staging)
    for (int idx = threadIdx.x; idx < re.n * UPB; idx += NT) {
      const int j = re.row(idx / UPB), l = idx % UPB;
      const size_t pp = (size_t)op + j;
      gate_grad(pp, u0 + l, H, dhidden[pp * H + u0 + l], gates, hun, hprev, dpre, dhu, gz);
    }
    // this thread's (row, unit) pair of the chunk: forward-pass operands, loaded a chunk ahead
    GateIn gin{};
    auto load_g = [&](int c0, int nr) {
      if (threadIdx.x < nr * UPB)
        gin = gate_load((size_t)op + rc.row(c0 + threadIdx.x / UPB), u0 + threadIdx.x % UPB, H, gates, hun, hprev,
                        dhidden);
    };
    if (nch > 0) load_g(0, min(KS_BR, rc.n));
    for (int ch = 0; ch < nch; ++ch) {
      const int c0 = ch * KS_BR, nr = min(KS_BR, rc.n - c0);
      if (threadIdx.x < 32 && ch + 1 < nch)
        stage_rows_warp(ds + (buf ^ 1) * KS_BR * H3, src, H3, rc, c0 + KS_BR, min(KS_BR, rc.n - c0 - KS_BR),
                        su32(&mbar[buf ^ 1]));
      float gzv = 0.f;
      if (threadIdx.x < nr * UPB)
        gzv = __ldcg(gz + ((size_t)o + rc.row(c0 + threadIdx.x / UPB)) * H + u0 + threadIdx.x % UPB);
      mb_wait(su32(&mbar[buf]), (phase >> buf) & 1);
      phase ^= 1u << buf;
      const float* dc = ds + buf * KS_BR * H3;
      for (int g0 = 0; g0 < nr; g0 += 4) {
        float acc[16];
#pragma unroll
        for (int v = 0; v < 16; ++v) acc[v] = 0.f;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
#pragma unroll
          for (int i = 0; i < NV; ++i) {
            const float4 d4 = *reinterpret_cast<const float4*>(dc + (g0 + r) * H3 + warp * KW + 4 * kq + 32 * i);
            const float dv[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
            for (int v = 0; v < 4; ++v)
#pragma unroll
              for (int c = 0; c < 4; ++c) acc[r * 4 + c] = fmaf(dv[v], w[i][v][c], acc[r * 4 + c]);
          }
        }
        // reduce-scatter over kq: lane keeps values 2 kq, 2 kq + 1 = row kq / 2, units 2 (kq & 1) + {0, 1}
        rs_level<8>(acc, lane, 4);
        rs_level<4>(acc, lane, 2);
        rs_level<2>(acc, lane, 1);
        const int row = g0 + (kq >> 1), col = 4 * cq + 2 * (kq & 1);
        *reinterpret_cast<float2*>(red + ((size_t)warp * KS_BR + row) * UPB + col) = make_float2(acc[0], acc[1]);
      }
      __syncthreads();
      static_assert(KS_BR * UPB <= NT, "one (row, unit) pair per thread");
      if (threadIdx.x < nr * UPB) {
        const int row = threadIdx.x / UPB, ul = threadIdx.x % UPB;
        float tot = 0.f;
#pragma unroll
        for (int q = 0; q < NW; ++q) tot += red[((size_t)q * KS_BR + row) * UPB + ul];
        gate_grad_v((size_t)op + rc.row(c0 + row), u0 + ul, H, gin.dh + tot + gzv, gin, dpre, dhu, gz);
      }
      if (ch + 1 < nch) load_g(c0 + KS_BR, min(KS_BR, rc.n - c0 - KS_BR));
      __syncthreads();
      buf ^= 1;
    }
  }
}

// warps per K-split CTA (a 16-warp variant sharing the weights measured equal
// on B200: the steps are not bound by latency hiding)
static int ks_warps(int) { return 8; }
static size_t ks_fwd_smem(int H) {
  const int nw = ks_warps(H);
  return sizeof(float) * ((size_t)2 * ks_fr(nw) * H + (size_t)nw * ks_fr(nw) * 3 * UPB) + 16;
}
static size_t ks_bwd_smem(int H) {
  const int nw = ks_warps(H);
  return sizeof(float) * ((size_t)2 * KS_BR * 3 * H + (size_t)nw * KS_BR * UPB) + 16;
}
static const void* pick_fwd_ks(int H) {
  switch (H) {
    case 256: return reinterpret_cast<const void*>(gru_fwd_ks<256, 8>);
    case 512: return reinterpret_cast<const void*>(gru_fwd_ks<512, 8>);
    default: return nullptr;
  }
}
static const void* pick_bwd_ks(int H) {
  switch (H) {
    case 256: return reinterpret_cast<const void*>(gru_bwd_ks<256, 8>);
    case 512: return reinterpret_cast<const void*>(gru_bwd_ks<512, 8>);
    default: return nullptr;
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
// experiments only: VER_REC_TRACE=<file> appends, per K-split launch, the
// globaltimer (ns) at which CTA 0 starts each timestep, with bs_t
static void trace_dump(Ctx* c, const char* tag, int L, const int32_t* d_bs, long long* d_tr) {
  const char* path = getenv("VER_REC_TRACE");
  if (!path || !d_tr) return;
  std::vector<long long> tr(L);
  std::vector<int32_t> b(L);
  VER_CUDA(cudaMemcpyAsync(tr.data(), d_tr, sizeof(long long) * L, cudaMemcpyDeviceToHost, c->stream));
  VER_CUDA(cudaMemcpyAsync(b.data(), d_bs, sizeof(int32_t) * L, cudaMemcpyDeviceToHost, c->stream));
  VER_CUDA(cudaStreamSynchronize(c->stream));
  FILE* f = fopen(path, "a");
  if (!f) return;
  fprintf(f, "%s %d", tag, L);
  for (int t = 0; t < L; ++t) fprintf(f, " %d:%lld", b[t], tr[t]);
  fprintf(f, "\n");
  fclose(f);
}
static long long* trace_buf(Ctx* c, Workspace& ws, int L) {
  if (!getenv("VER_REC_TRACE")) return nullptr;
  ws.trace.reserve(c, (size_t)L);
  ws.trace.zero((size_t)L);
  return ws.trace.p;
}

static int rec_mode() {
  // experiments only: 0 = K-split kernels (H = 256, 512), 1 = register kernels with contiguous
  // rows and a grid-wide barrier, 2 = register kernels with interleaved row-block groups
  const char* e = getenv("VER_REC_MODE");
  return e ? atoi(e) : 0;
}
static void coop_launch(Ctx* c, const void* fn, int grid, size_t smem, void** args, int threads = RT) {
  ScopedEv ev(c, c->rec_tag);
  VER_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  VER_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem));
  if (per_sm * c->num_sms < grid)
    config_error("recurrence: grid does not fit co-resident (hidden dim too large for this build)");
  VER_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(threads), args, smem, c->stream));
  after_launch(c);
}


// -------------------------------------- single-cluster tail (H = 512)
// The last timesteps of a packed minibatch carry few rows (sequences sorted
// by length: bs_t falls to 1).  There the K-split kernels are bound by the
// per-step cross-SM handshake (group barrier through L2 + bulk re-staging).
// For steps with bs_t <= TC_TH one cluster of 16 CTAs holds all of U in
// registers (CTA r: units 32r .. 32r+31, 96 floats per thread), keeps h_{t-1}
// (forward) / dhU_t (backward) of all rows in every CTA's shared memory, and
// pushes each new value to the 16 CTAs with st.shared::cluster; steps are
// separated by the hardware cluster barrier.  Thread (warp w, lane u): K
// slice w of unit u; partials reduce over the 16 warps through shared memory.
constexpr int TC_CL = 16;   // CTAs per cluster (non-portable size)
constexpr int TC_T = 512;   // threads per CTA
constexpr int TC_TH = 8;    // steps with at most this many rows run on the cluster

__device__ __forceinline__ uint32_t cl_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// store v at the same shared-memory offset as `local` in every CTA of the cluster
__device__ __forceinline__ void cl_bcast(const float* local, float v) {
  const uint32_t a = su32(local);
#pragma unroll
  for (int r = 0; r < TC_CL; ++r) {
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(r));
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(ra), "f"(v) : "memory");
  }
}

// copy `n4` float4 of local shared memory at src to offset dst (same layout
// in every CTA) of all cluster CTAs; item i = (destination, float4)
__device__ __forceinline__ void cl_push4(const float* src_base, const float* dst_base, int rows, int row_f4,
                                         int src_ld, int dst_ld) {
  const int per_dst = rows * row_f4;
  for (int i = threadIdx.x; i < TC_CL * per_dst; i += blockDim.x) {
    const int r = i / per_dst, q = i % per_dst, row = q / row_f4, c = q % row_f4;
    const float4 v = *reinterpret_cast<const float4*>(src_base + row * src_ld + 4 * c);
    const uint32_t a = su32(dst_base + row * dst_ld + 4 * c);
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(r));
    asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(ra), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w)
                 : "memory");
  }
}

// as cl_push4, with st.async: every store completes its bytes on the same-offset
// mbarrier `bar` of the destination CTA (the owner waits for data, not for a
// cluster-wide barrier)
__device__ __forceinline__ void cl_push4_async(const float* src_base, const float* dst_base, int rows, int row_f4,
                                               int src_ld, int dst_ld, uint32_t bar) {
  const int per_dst = rows * row_f4;
  for (int i = threadIdx.x; i < TC_CL * per_dst; i += blockDim.x) {
    const int r = i / per_dst, q = i % per_dst, row = q / row_f4, c = q % row_f4;
    const float4 v = *reinterpret_cast<const float4*>(src_base + row * src_ld + 4 * c);
    const uint32_t a = su32(dst_base + row * dst_ld + 4 * c);
    uint32_t ra, rb;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(r));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(bar), "r"(r));
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(ra),
                 "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(rb)
                 : "memory");
  }
}
__device__ __forceinline__ void tl_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tl_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "TL_WAIT:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra TL_WAIT;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

template <int H>
__global__ void __launch_bounds__(TC_T, 1) gru_fwd_tail(
    int t0, int L, const int32_t* __restrict__ bs, const int32_t* __restrict__ offs, const float* __restrict__ ux,
    const float* __restrict__ xp, const float* h0, float* hidden, float* __restrict__ gates, float* __restrict__ hun,
    float* __restrict__ hprev_store, long long* trace, int tail_async) {
  constexpr int H3 = 3 * H, UT = H / TC_CL, KW = H / (TC_T / 32);
  static_assert(UT == 32 && KW % 4 == 0, "tail kernel: H = 512");
  extern __shared__ float4 sm4[];
  float* hs = reinterpret_cast<float*>(sm4);    // [2][TC_TH][H]
  float* red = hs + 2 * TC_TH * H;              // [16][TC_TH][3 UT]
  float* stg = red + (TC_T / 32) * TC_TH * 3 * UT;  // [TC_TH][UT] this CTA's new h slice
  // one mbarrier per h buffer: the 16 CTAs' slices of step s land in buffer s & 1
  // with st.async; the owner expects bs[s] x H x 4 bytes (posted two steps ahead)
  uint64_t* bars = reinterpret_cast<uint64_t*>(stg + TC_TH * UT);
  const uint32_t bar_a[2] = {su32(bars), su32(bars + 1)};
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int u0 = (int)cl_rank() * UT, u = u0 + lane;
  const bool async_push = tail_async != 0;
  float w[KW][3];
#pragma unroll
  for (int k = 0; k < KW; ++k)
#pragma unroll
    for (int g = 0; g < 3; ++g) w[k][g] = ux[(size_t)(warp * KW + k) * H3 + 3 * u + g];
  {
    const int B = bs[t0];
    const float* hp = t0 == 0 ? h0 : hidden + (size_t)offs[t0 - 1] * H;
    for (int i = threadIdx.x; i < B * H; i += TC_T) hs[(t0 & 1) * TC_TH * H + i] = __ldcg(hp + i);
  }
  if (async_push && threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_a[0]) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_a[1]) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s2 = t0 + 1; s2 <= t0 + 2 && s2 < L; ++s2) tl_expect(bar_a[s2 & 1], (uint32_t)bs[s2] * H * 4);
  }
  cl_sync();
  const int j = warp;  // gate pair (row warp, unit lane)
  // x W + b of (row j, unit u) at step t, loaded one step ahead
  auto load_x = [&](int t, float* x3) {
    if (t < L && j < bs[t]) {
      const float* x = xp + ((size_t)offs[t] + j) * H3 + 3 * u;
      x3[0] = __ldg(x);
      x3[1] = __ldg(x + 1);
      x3[2] = __ldg(x + 2);
    }
  };
  float xc[3] = {0.f, 0.f, 0.f}, xn[3] = {0.f, 0.f, 0.f};
  load_x(t0, xc);
  for (int t = t0; t < L; ++t) {
    if (async_push && t > t0) {
      tl_wait(bar_a[t & 1], (uint32_t)(((t - t0 - 1) >> 1) & 1));
      if (threadIdx.x == 0 && t + 2 < L) tl_expect(bar_a[t & 1], (uint32_t)bs[t + 2] * H * 4);
    }
    if (trace && blockIdx.x == 0 && threadIdx.x == 0) trace[t] = globaltimer();
    const int B = bs[t], o = offs[t];
    const float* hc = hs + (t & 1) * TC_TH * H;
    float* hn = hs + ((t + 1) & 1) * TC_TH * H;
    load_x(t + 1, xn);
    const float x0 = xc[0], x1 = xc[1], x2 = xc[2];
    for (int r0 = 0; r0 < B; r0 += 2) {
      float a[2][3] = {{0.f, 0.f, 0.f}, {0.f, 0.f, 0.f}};
#pragma unroll
      for (int k = 0; k < KW; k += 4) {
        const float4 p = *reinterpret_cast<const float4*>(hc + r0 * H + warp * KW + k);
        const float4 q = *reinterpret_cast<const float4*>(hc + (r0 + 1) * H + warp * KW + k);
        const float pv[4] = {p.x, p.y, p.z, p.w}, qv[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int v = 0; v < 4; ++v)
#pragma unroll
          for (int g = 0; g < 3; ++g) {
            a[0][g] = fmaf(pv[v], w[k + v][g], a[0][g]);
            a[1][g] = fmaf(qv[v], w[k + v][g], a[1][g]);
          }
      }
#pragma unroll
      for (int g = 0; g < 3; ++g) {
        red[(warp * TC_TH + r0) * 3 * UT + 3 * lane + g] = a[0][g];
        red[(warp * TC_TH + r0 + 1) * 3 * UT + 3 * lane + g] = a[1][g];
      }
    }
    __syncthreads();
    if (j < B) {
      float sr = 0.f, sz = 0.f, sn = 0.f;
#pragma unroll
      for (int q = 0; q < TC_T / 32; ++q) {
        const float* rq = red + (q * TC_TH + j) * 3 * UT + 3 * lane;
        sr += rq[0];
        sz += rq[1];
        sn += rq[2];
      }
      const float rg = gate_sigm(x0 + sr);
      const float zg = gate_sigm(x1 + sz);
      const float ng = gate_tanh(x2 + rg * sn);
      const float hprev = hc[j * H + u];
      const float hnew = (1.f - zg) * ng + zg * hprev;
      const size_t p = (size_t)o + j;
      hidden[p * H + u] = hnew;
      if (gates) {
        float* gp = gates + p * H3 + 3 * u;
        gp[0] = rg;
        gp[1] = zg;
        gp[2] = ng;
        hun[p * H + u] = sn;
        hprev_store[p * H + u] = hprev;
      }
      stg[j * UT + lane] = hnew;
    }
    if (t + 1 < L) {
      __syncthreads();
      if (async_push) {
        cl_push4_async(stg, hn + u0, bs[t + 1], UT / 4, UT, H, bar_a[(t + 1) & 1]);
      } else {
        cl_push4(stg, hn + u0, B, UT / 4, UT, H);
      }
    }
    xc[0] = xn[0];
    xc[1] = xn[1];
    xc[2] = xn[2];
    if (!async_push) cl_sync();
  }
  if (async_push) cl_sync();  // no CTA exits while a peer may still push into it
}

// backward: steps t = L-1 .. t_stop+1 (rows of step t-1 <= TC_TH), plus the
// no-carry step L-1; dhU rows of all 3H columns are pushed to every CTA
template <int H>
__global__ void __launch_bounds__(TC_T, 1) gru_bwd_tail(
    int L, int t_stop, const int32_t* __restrict__ bs, const int32_t* __restrict__ offs,
    const float* __restrict__ ux, const float* __restrict__ dhidden, const float* __restrict__ gates,
    const float* __restrict__ hun, const float* __restrict__ hprev, float* __restrict__ dpre, float* __restrict__ dhu,
    float* __restrict__ gz, long long* trace, int tail_async) {
  constexpr int H3 = 3 * H, UT = H / TC_CL, KW = H3 / (TC_T / 32);
  static_assert(UT == 32 && KW % 4 == 0, "tail kernel: H = 512");
  extern __shared__ float4 sm4[];
  float* ds = reinterpret_cast<float*>(sm4);    // [2][TC_TH][3H]
  float* red = ds + 2 * TC_TH * H3;             // [16][TC_TH][UT]
  float* gzs = red + (TC_T / 32) * TC_TH * UT;  // [2][TC_TH][UT]
  float* stg = gzs + 2 * TC_TH * UT;            // [TC_TH][3 UT] this CTA's new dhU slice
  // async handoff (as gru_fwd_tail): fill f of the dhU buffers (f = 0: the
  // no-carry step L-1, f >= 1: pushed by iteration f-1) lands in buffer f & 1
  // and completes bs[L-1-f] x 3H x 4 bytes on that buffer's mbarrier
  uint64_t* bars = reinterpret_cast<uint64_t*>(stg + TC_TH * 3 * UT);
  const uint32_t bar_a[2] = {su32(bars), su32(bars + 1)};
  const bool async_push = tail_async != 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int u0 = (int)cl_rank() * UT, u = u0 + lane;
  float w[KW];
#pragma unroll
  for (int k = 0; k < KW; ++k) w[k] = ux[(size_t)u * H3 + warp * KW + k];
  const int j = warp;  // gate pair (row warp, unit lane)
  // gate gradient of (row j, unit u) at packed row p (operands `in`, loaded
  // ahead); pushes dhU to every CTA and keeps g z
  auto gate = [&](size_t p, const GateIn& in, float gsum, float* dnext, float* gznext) {
    const float g = in.dh + gsum;
    const float dn = g * (1.f - in.z);
    const float dz = g * (in.hp - in.n);
    const float dpn = dn * (1.f - in.n * in.n);
    const float dr = dpn * in.hn;
    const float dpr = dr * in.r * (1.f - in.r);
    const float dpz = dz * in.z * (1.f - in.z);
    float* d = dpre + p * H3 + 3 * u;
    d[0] = dpr;
    d[1] = dpz;
    d[2] = dpn;
    float* e = dhu + p * H3 + 3 * u;
    e[0] = dpr;
    e[1] = dpz;
    e[2] = dpn * in.r;
    gz[p * H + u] = g * in.z;
    gznext[j * UT + lane] = g * in.z;
    stg[j * 3 * UT + 3 * lane] = dpr;
    stg[j * 3 * UT + 3 * lane + 1] = dpz;
    stg[j * 3 * UT + 3 * lane + 2] = dpn * in.r;
  };
  // this step's dhU slices of rows 0..n-1 -> every CTA's buffer dnext
  auto push = [&](int n, float* dnext, int fill) {
    __syncthreads();
    if (async_push) cl_push4_async(stg, dnext + 3 * u0, n, 3 * UT / 4, 3 * UT, H3, bar_a[fill & 1]);
    else cl_push4(stg, dnext + 3 * u0, n, 3 * UT / 4, 3 * UT, H3);
  };
  // fill f exists iff f == 0 or iteration f-1 (t = L-f) pushes, i.e. L-1-f > t_stop
  auto fill_rows = [&](int f) { return (f == 0 || L - 1 - f > t_stop) ? bs[L - 1 - f] : -1; };
  if (async_push) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_a[0]) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_a[1]) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      for (int f = 0; f < 2; ++f)
        if (L - 1 - f >= 0 && fill_rows(f) >= 0) tl_expect(bar_a[f & 1], (uint32_t)fill_rows(f) * H3 * 4);
    }
    cl_sync();  // every CTA's barriers are live before the first push
  }
  int cur = 0;
  if (j < bs[L - 1]) {
    const size_t p = (size_t)offs[L - 1] + j;
    gate(p, gate_load(p, u, H, gates, hun, hprev, dhidden), 0.f, ds, gzs);
  }
  push(bs[L - 1], ds, 0);
  if (trace && blockIdx.x == 0 && threadIdx.x == 0) trace[L - 1] = globaltimer();
  if (!async_push) cl_sync();
  // forward-pass operands of (row j, unit u) at step t-1, loaded one step ahead
  GateIn gin{}, gnext{};
  if (L - 1 > t_stop && j < bs[L - 2]) gin = gate_load((size_t)offs[L - 2] + j, u, H, gates, hun, hprev, dhidden);
  for (int t = L - 1; t > t_stop; --t) {
    const int B = bs[t], Bp = bs[t - 1], op = offs[t - 1];
    const int fi = L - 1 - t;  // this iteration reads fill fi
    if (async_push) {
      tl_wait(bar_a[fi & 1], (uint32_t)((fi >> 1) & 1));
      if (threadIdx.x == 0 && L - 1 - (fi + 2) >= 0 && fill_rows(fi + 2) >= 0)
        tl_expect(bar_a[fi & 1], (uint32_t)fill_rows(fi + 2) * H3 * 4);
    }
    const float* dc = ds + cur * TC_TH * H3;
    if (t - 1 > t_stop && j < bs[t - 2])
      gnext = gate_load((size_t)offs[t - 2] + j, u, H, gates, hun, hprev, dhidden);
    for (int r0 = 0; r0 < B; r0 += 2) {
      float a0 = 0.f, a1 = 0.f, b0 = 0.f, b1 = 0.f;
#pragma unroll
      for (int k = 0; k < KW; k += 4) {
        const float4 p = *reinterpret_cast<const float4*>(dc + r0 * H3 + warp * KW + k);
        const float4 q = *reinterpret_cast<const float4*>(dc + (r0 + 1) * H3 + warp * KW + k);
        a0 = fmaf(p.x, w[k], a0);
        a1 = fmaf(p.y, w[k + 1], a1);
        a0 = fmaf(p.z, w[k + 2], a0);
        a1 = fmaf(p.w, w[k + 3], a1);
        b0 = fmaf(q.x, w[k], b0);
        b1 = fmaf(q.y, w[k + 1], b1);
        b0 = fmaf(q.z, w[k + 2], b0);
        b1 = fmaf(q.w, w[k + 3], b1);
      }
      red[(warp * TC_TH + r0) * UT + lane] = a0 + a1;
      red[(warp * TC_TH + r0 + 1) * UT + lane] = b0 + b1;
    }
    __syncthreads();
    if (j < Bp) {
      float tot = 0.f;
      if (j < B) {
#pragma unroll
        for (int q = 0; q < TC_T / 32; ++q) tot += red[(q * TC_TH + j) * UT + lane];
        tot += gzs[cur * TC_TH * UT + j * UT + lane];
      }
      gate((size_t)op + j, gin, tot, ds + (cur ^ 1) * TC_TH * H3, gzs + (cur ^ 1) * TC_TH * UT);
    }
    if (t - 1 > t_stop) push(Bp, ds + (cur ^ 1) * TC_TH * H3, fi + 1);
    gin = gnext;
    cur ^= 1;
    if (!async_push) cl_sync();
    if (trace && blockIdx.x == 0 && threadIdx.x == 0) trace[t - 1] = globaltimer();
  }
  if (async_push) {
    if (L - 1 <= t_stop) tl_wait(bar_a[0], 0);  // fill 0 had no consumer: let it land first
    cl_sync();  // no CTA exits while a peer may still push into it
  }
}

static size_t tail_fwd_smem(int H) {
  return sizeof(float) *
             ((size_t)2 * TC_TH * H + (size_t)(TC_T / 32) * TC_TH * 3 * (H / TC_CL) + (size_t)TC_TH * (H / TC_CL)) +
         16 /* two mbarriers */;
}
static size_t tail_bwd_smem(int H) {
  return sizeof(float) * ((size_t)2 * TC_TH * 3 * H + (size_t)(TC_T / 32) * TC_TH * (H / TC_CL) +
                          (size_t)2 * TC_TH * (H / TC_CL) + (size_t)TC_TH * 3 * (H / TC_CL)) +
         16 /* two mbarriers */;
}

// 1 if this device can run one 16-CTA cluster of the tail kernels
static bool tail_ok(Ctx* c, int H) {
  static std::atomic<int> ok_cache[kMaxDevices];  // per device: 0 unknown, 1 no, 2 yes
  if (H != 512 || rec_mode() != 0 || env_int("VER_REC_TAIL", 1) == 0) return false;
  std::atomic<int>& okc = ok_cache[dev_slot(c)];
  if (okc.load() != 0) return okc.load() == 2;
  okc.store(1);
  const void* fns[2] = {reinterpret_cast<const void*>(gru_fwd_tail<512>),
                        reinterpret_cast<const void*>(gru_bwd_tail<512>)};
  const size_t sm[2] = {tail_fwd_smem(512), tail_bwd_smem(512)};
  for (int i = 0; i < 2; ++i) {
    if (cudaFuncSetAttribute(fns[i], cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess ||
        cudaFuncSetAttribute(fns[i], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm[i]) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(TC_CL);
    cfg.blockDim = dim3(TC_T);
    cfg.dynamicSmemBytes = sm[i];
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = TC_CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, fns[i], &cfg) != cudaSuccess || n < 1) {
      cudaGetLastError();
      return false;
    }
  }
  okc.store(2);
  return true;
}
static void tail_launch(Ctx* c, const void* fn, size_t smem, void** args) {
  ScopedEv ev(c, c->rec_tag);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(TC_CL);
  cfg.blockDim = dim3(TC_T);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = TC_CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  VER_CUDA(cudaLaunchKernelExC(&cfg, fn, args));
  after_launch(c);
}
// first timestep whose batch is small enough for the cluster tail (L: none).
// The cluster does the whole matvec on 16 SMs, so its step time grows with the
// rows (measured on B200 at H = 512: forward 2.0 us at 1 row, 3.7 us at 6;
// backward 2.2 / 5.3 us) while the K-split kernels take ~3.2 us per short step:
// the tail takes steps of <= 2 (forward, whose short K-split steps use the
// tagged handoff) / <= 3 (backward) rows.
static int tail_start(const int32_t* h_bs, int L, int th) {
  if (!h_bs) return L;
  th = std::min(th, TC_TH);
  int t0 = L;
  while (t0 > 0 && h_bs[t0 - 1] <= th) --t0;
  return t0;
}

static void fwd_ks_launch(Ctx* c, const Model& m, const float* params, int t_begin, int L, const int32_t* d_bs,
                          const int32_t* d_offs, Workspace& ws, const float* h0, bool store);

void gru_forward_recurrence(Ctx* c, const Model& m, const float* params, int L, const int32_t* d_bs,
                            const int32_t* d_offs, Workspace& ws, const float* h0, bool store,
                            const int32_t* h_bs, const int32_t* h_offs) {
  // big steps (many rows) as per-step tensor-core GEMMs, then the persistent
  // FMA kernel, then the cluster tail
  const int tb = (h_bs && h_offs && pick_fwd_ks(m.H) && rec_mode() == 0) ? gru_big_steps(c, m, h_bs, L, false) : 0;
  if (tb > 0) {
    gru_forward_big_persist(c, m, params, tb, h_bs, h_offs, ws, h0, store);
    const int t0 = tail_ok(c, m.H) ? std::max(tb, tail_start(h_bs, L, env_int("VER_REC_TAIL_FWD", 2))) : L;
    if (t0 > tb) fwd_ks_launch(c, m, params, tb, t0, d_bs, d_offs, ws, h0, store);
    if (t0 < L) {
      int t0_ = t0, L_ = L;
      const float* ux = params + m.o_ux;
      const float* xp = ws.xp.p;
      float* hidden = ws.hidden.p;
      float* gates = store ? ws.gates.p : nullptr;
      float* hun = ws.hu.p;
      float* hps = ws.hprev.p;
      long long* tr = trace_buf(c, ws, L);
      int ta = 1;  // st.async + mbarrier handoff (0: cluster barrier)
      void* args[] = {&t0_, &L_, &d_bs, &d_offs, &ux, &xp, &h0, &hidden, &gates, &hun, &hps, &tr, &ta};
      tail_launch(c, reinterpret_cast<const void*>(gru_fwd_tail<512>), tail_fwd_smem(512), args);
      trace_dump(c, "fwdtail", L, d_bs, tr);
    }
    return;
  }
  if (L > 0 && tail_ok(c, m.H)) {
    const int t0 = tail_start(h_bs, L, env_int("VER_REC_TAIL_FWD", 2));
    if (t0 < L) {
      if (t0 > 0) gru_forward_recurrence(c, m, params, t0, d_bs, d_offs, ws, h0, store, nullptr);
      int t0_ = t0, L_ = L;
      const float* ux = params + m.o_ux;
      const float* xp = ws.xp.p;
      float* hidden = ws.hidden.p;
      float* gates = store ? ws.gates.p : nullptr;
      float* hun = ws.hu.p;
      float* hps = ws.hprev.p;
      long long* tr = trace_buf(c, ws, L);
      int ta = 1;  // st.async + mbarrier handoff (0: cluster barrier)
      void* args[] = {&t0_, &L_, &d_bs, &d_offs, &ux, &xp, &h0, &hidden, &gates, &hun, &hps, &tr, &ta};
      tail_launch(c, reinterpret_cast<const void*>(gru_fwd_tail<512>), tail_fwd_smem(512), args);
      trace_dump(c, "fwdtail", L, d_bs, tr);
      return;
    }
  }
  const RecGeom g = geom(c, m.H);
  const int grid = g.UB * g.RB;
  ws.bar.reserve(c, (size_t)kBarStride * g.RB);
  ws.bar.zero((size_t)kBarStride * g.RB);
  int H = m.H, UB = g.UB, RB = g.RB;
  const float* ux = params + m.o_ux;
  const float* xp = ws.xp.p;
  float* hidden = ws.hidden.p;
  float* gates = store ? ws.gates.p : nullptr;
  float* hun = ws.hu.p;
  float* hps = ws.hprev.p;
  unsigned* bar = ws.bar.p;
  if (rec_mode() == 0 && pick_fwd_ks(m.H)) {
    fwd_ks_launch(c, m, params, 0, L, d_bs, d_offs, ws, h0, store);
    return;
  }
  if (const void* fn = pick_fwd(m.H)) {
    const size_t smem = sizeof(float) * (size_t)RCF * m.H;
    int inter = rec_mode() == 2 ? 1 : 0;
    void* args[] = {&L, &d_bs, &d_offs, &UB, &RB, &ux, &xp, &h0, &hidden, &gates, &hun, &hps, &bar, &inter};
    coop_launch(c, fn, grid, smem, args);
    return;
  }
  const size_t smem = sizeof(float) * ((size_t)m.H * (3 * UPB + 1) + (size_t)RCHF * m.H + 16 * UPB * 3);
  void* args[] = {&L, &d_bs, &d_offs, &H, &UB, &RB, &ux, &xp, &h0, &hidden, &gates, &hun, &hps, &bar};
  coop_launch(c, reinterpret_cast<const void*>(gru_fwd_persistent), grid, smem, args);
}

static void fwd_ks_launch(Ctx* c, const Model& m, const float* params, int t_begin, int L, const int32_t* d_bs,
                          const int32_t* d_offs, Workspace& ws, const float* h0, bool store) {
  const RecGeom g = geom(c, m.H);
  const int grid = g.UB * g.RB;
  ws.bar.reserve(c, (size_t)kBarStride * g.RB);
  ws.bar.zero((size_t)kBarStride * g.RB);
  int UB = g.UB, RB = g.RB, tbeg = t_begin;
  const float* ux = params + m.o_ux;
  const float* xp = ws.xp.p;
  float* hidden = ws.hidden.p;
  float* gates = store ? ws.gates.p : nullptr;
  float* hun = ws.hu.p;
  float* hps = ws.hprev.p;
  unsigned* bar = ws.bar.p;
  long long* tr = trace_buf(c, ws, L);
  const void* fn = pick_fwd_ks(m.H);
  // short steps hand h over through tagged words (up to 24 rows; beyond: group barrier + bulk staging).
  // Measured on B200 at C2: forward recurrence 9.11 -> 8.73 ms per update at 16 rows, 8.61 ms at 24
  // rows with the cluster tail limited to <= 2 rows (VER_REC_TAIL_FWD), worse at 64.  The backward (dhU rows are 3H wide) measured slower with the same scheme.
  int tag_th = std::min(24, ks_fr(ks_warps(m.H)) * RB);
  if (L > 4096) tag_th = 0;  // tags: epoch * 4096 + t
  ws.hx.reserve(c, (size_t)2 * std::max(tag_th, 1) * m.H);
  ws.hx.zero((size_t)2 * std::max(tag_th, 1) * m.H);  // no stale tag can match (epochs start at 1)
  unsigned long long* hx = ws.hx.p;
  unsigned epoch = ++ws.hx_epoch;
  void* args[] = {&L,   &d_bs, &d_offs, &UB, &RB,   &ux, &xp,     &h0,    &hidden, &gates,
                  &hun, &hps,  &bar,    &tr, &tbeg, &hx, &tag_th, &epoch};
  coop_launch(c, fn, grid, ks_fwd_smem(m.H), args, 32 * ks_warps(m.H));
  trace_dump(c, "fwd", L, d_bs, tr);
}

void gru_backward_recurrence(Ctx* c, const Model& m, const float* params, int L, const int32_t* d_bs,
                             const int32_t* d_offs, Workspace& ws, const int32_t* h_bs, const int32_t* h_offs) {
  // steps t > t_stop (rows of t-1 <= TC_TH) on the cluster tail, then t_stop .. 1
  int t_stop = L, do_init = 1;
  if (L > 0 && tail_ok(c, m.H)) {
    const int t0 = tail_start(h_bs, L, env_int("VER_REC_TAIL_BWD", 3));
    if (t0 < L) {
      t_stop = t0;
      int L_ = L, ts = t0;
      const float* ux = params + m.o_ux;
      const float* dh = ws.dhidden.p;
      const float* gates = ws.gates.p;
      const float* hun = ws.hu.p;
      const float* hps = ws.hprev.p;
      float* dpre = ws.dpre.p;
      float* dhu = ws.dhu.p;
      float* gz = ws.g.p;
      long long* tr = trace_buf(c, ws, L);
      int ta = 1;  // st.async + mbarrier handoff (0: cluster barrier)
      void* args[] = {&L_, &ts, &d_bs, &d_offs, &ux, &dh, &gates, &hun, &hps, &dpre, &dhu, &gz, &tr, &ta};
      tail_launch(c, reinterpret_cast<const void*>(gru_bwd_tail<512>), tail_bwd_smem(512), args);
      trace_dump(c, "bwdtail", L, d_bs, tr);
      if (t0 == 0) return;
      do_init = 0;
    }
  }
  int t_start = std::min(L - 1, t_stop);
  // big steps t = t_big .. 1 (rows of t-1 >= VER_REC_BIG) run after the
  // persistent kernel as per-step tensor-core GEMMs
  const int tb = (h_bs && h_offs && pick_bwd_ks(m.H) && rec_mode() == 0) ? gru_big_steps(c, m, h_bs, L, true) : 0;
  int t_big = std::min(tb, L - 1);
  if (t_big > t_start) t_big = t_start;  // (cannot happen: big and tail steps are disjoint)
  const RecGeom g = geom(c, m.H);
  const int grid = g.UB * g.RB;
  ws.bar.reserve(c, (size_t)kBarStride * g.RB);
  ws.bar.zero((size_t)kBarStride * g.RB);
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
  if (const void* fn = rec_mode() == 0 ? pick_bwd_ks(m.H) : nullptr) {
    long long* tr = trace_buf(c, ws, L);
    if (t_start > t_big || do_init) {
      void* args[] = {&L,    &d_bs, &d_offs, &UB, &RB, &ux,      &dh,      &gates,  &hun,
                      &hps,  &dpre, &dhu,    &gz, &bar, &tr, &t_start, &do_init, &t_big};
      coop_launch(c, fn, grid, ks_bwd_smem(m.H), args, 32 * ks_warps(m.H));
      trace_dump(c, "bwd", L, d_bs, tr);
    }
    if (t_big > 0) gru_backward_big_persist(c, m, params, t_big, h_bs, h_offs, ws);
    return;
  }
  if (const void* fn = pick_bwd(m.H)) {
    const size_t smem = sizeof(float) * (size_t)RCB * 3 * m.H;
    int inter = rec_mode() == 2 ? 1 : 0;
    void* args[] = {&L, &d_bs, &d_offs, &UB, &RB, &ux, &dh, &gates, &hun, &hps, &dpre, &dhu, &gz, &bar, &inter};
    coop_launch(c, fn, grid, smem, args);
    return;
  }
  const size_t smem = sizeof(float) * ((size_t)UPB * (3 * m.H + 1) + (size_t)RCHB * 3 * m.H + 16 * UPB);
  void* args[] = {&L, &d_bs, &d_offs, &H, &UB, &RB, &ux, &dh, &gates, &hun, &hps, &dpre, &dhu, &gz, &bar};
  coop_launch(c, reinterpret_cast<const void*>(gru_bwd_persistent), grid, smem, args);
}

}  // namespace verg
