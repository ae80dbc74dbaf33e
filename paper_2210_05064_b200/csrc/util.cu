// util.cu — context lifecycle, error state, NCCL plumbing and the device
// primitives shared by the hot-path kernels: int32 exclusive scan (3-phase,
// 1024-thread blocks) and a bitonic sort of unique uint64 keys.
#include "common.cuh"

#include <cstdlib>
#include <cstring>
#include <mutex>

namespace verg {

bool profiling() {
  static const bool on = env_int("VER_PROFILING", 0) != 0;
  return on;
}

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

static thread_local std::string g_last_error;
void set_last_error(const std::string& w) { g_last_error = w; }

void activate(Ctx* c) { VER_CUDA(cudaSetDevice(c->device)); }

void* Ctx::pinned_buf(size_t bytes) {
  if (bytes > pinned_bytes) {
    if (pinned) cudaFreeHost(pinned);
    pinned = nullptr;
    VER_CUDA(cudaMallocHost(&pinned, bytes));
    pinned_bytes = bytes;
  }
  return pinned;
}

// ------------------------------------------------------------------- scan
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;                       // per thread
constexpr int kScanTile = kScanThreads * kScanItems;  // 4096 per block

template <class T>
__device__ __forceinline__ int32_t block_exclusive_scan(int32_t v, int32_t* smem_warp,
                                                        int32_t* block_total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int32_t w = lane < (blockDim.x >> 5) ? smem_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    smem_warp[lane] = w;  // inclusive warp totals
  }
  __syncthreads();
  const int32_t warp_prefix = warp ? smem_warp[warp - 1] : 0;
  if (block_total) *block_total = smem_warp[(blockDim.x >> 5) - 1];
  return warp_prefix + x - v;
}

template <class T>
__global__ void __launch_bounds__(kScanThreads) scan_tile_kernel(const T* in,  // may alias out
                                                                 int32_t* out,
                                                                 int32_t* __restrict__ block_sums,
                                                                 int64_t n) {
  __shared__ int32_t sw[32];
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int32_t v[kScanItems];
  int32_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = (base + i < n) ? static_cast<int32_t>(in[base + i]) : 0;
    s += v[i];
  }
  int32_t total;
  int32_t pre = block_exclusive_scan<T>(s, sw, &total);
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < n) out[base + i] = pre;
    pre += v[i];
  }
  if (threadIdx.x == 0 && block_sums) block_sums[blockIdx.x] = total;
}

__global__ void scan_add_kernel(int32_t* __restrict__ out, const int32_t* __restrict__ block_pre,
                                int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * kScanTile;
  const int32_t add = block_pre[blockIdx.x];
  for (int64_t j = i + threadIdx.x; j < i + kScanTile && j < n; j += blockDim.x) out[j] += add;
}

template <class T>
__global__ void copy_last_kernel(const T* __restrict__ in, int64_t n, int32_t* __restrict__ last) {
  *last = static_cast<int32_t>(in[n - 1]);
}

__global__ void scan_total_kernel(const int32_t* __restrict__ excl, const int32_t* __restrict__ last,
                                  int64_t n, int32_t* __restrict__ total) {
  *total = excl[n - 1] + *last;
}

template <class T>
static void exclusive_scan_impl(Ctx* c, const T* in, int32_t* out, int64_t n, int32_t* total) {
  if (n <= 0) {
    if (total) VER_CUDA(cudaMemsetAsync(total, 0, sizeof(int32_t), c->stream));
    return;
  }
  DBuf<int32_t> last;  // `in` may alias `out`: keep the last input for the total
  if (total) {
    last.reserve(c, 1);
    copy_last_kernel<T><<<1, 1, 0, c->stream>>>(in, n, last.p);
    after_launch(c);
  }
  const int64_t nb = (n + kScanTile - 1) / kScanTile;
  if (nb == 1) {
    scan_tile_kernel<T><<<1, kScanThreads, 0, c->stream>>>(in, out, nullptr, n);
    after_launch(c);
  } else {
    DBuf<int32_t> sums;
    sums.reserve(c, nb);
    scan_tile_kernel<T><<<(unsigned)nb, kScanThreads, 0, c->stream>>>(in, out, sums.p, n);
    after_launch(c);
    exclusive_scan_impl<int32_t>(c, sums.p, sums.p, nb, nullptr);
    scan_add_kernel<<<(unsigned)nb, 256, 0, c->stream>>>(out, sums.p, n);
    after_launch(c);
  }
  if (total) {
    scan_total_kernel<<<1, 1, 0, c->stream>>>(out, last.p, n, total);
    after_launch(c);
  }
}

void exclusive_scan_i32(Ctx* c, const int32_t* in, int32_t* out, int64_t n, int32_t* total) {
  exclusive_scan_impl<int32_t>(c, in, out, n, total);
}
void exclusive_scan_u8(Ctx* c, const uint8_t* in, int32_t* out, int64_t n, int32_t* total) {
  exclusive_scan_impl<uint8_t>(c, in, out, n, total);
}

// ---------------------------------------------------------------- bitonic
// Sorts n unique uint64 keys ascending.  Pads to a power of two with
// UINT64_MAX (never a real key: callers build keys below 2^63).
constexpr int kSortSmem = 4096;  // keys sorted entirely in shared memory per block

__global__ void bitonic_local_kernel(uint64_t* __restrict__ k, int64_t n2, int start_size) {
  // start_size == 2: full local sort of each kSortSmem chunk;
  // otherwise: finish merge stages j < kSortSmem for size `start_size`.
  __shared__ uint64_t s[kSortSmem];
  const int64_t base = (int64_t)blockIdx.x * kSortSmem;
  for (int i = threadIdx.x; i < kSortSmem; i += blockDim.x) s[i] = k[base + i];
  __syncthreads();
  if (start_size == 2) {
    for (int size = 2; size <= kSortSmem; size <<= 1) {
      for (int j = size >> 1; j > 0; j >>= 1) {
        for (int t = threadIdx.x; t < kSortSmem / 2; t += blockDim.x) {
          const int i = 2 * t - (t & (j - 1));
          const int l = i + j;
          const int64_t gi = base + i;
          const bool up = ((gi & size) == 0);
          uint64_t a = s[i], b = s[l];
          if ((a > b) == up) {
            s[i] = b;
            s[l] = a;
          }
        }
        __syncthreads();
      }
    }
  } else {
    const int64_t size = start_size;
    for (int j = kSortSmem >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < kSortSmem / 2; t += blockDim.x) {
        const int i = 2 * t - (t & (j - 1));
        const int l = i + j;
        const int64_t gi = base + i;
        const bool up = ((gi & size) == 0);
        uint64_t a = s[i], b = s[l];
        if ((a > b) == up) {
          s[i] = b;
          s[l] = a;
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < kSortSmem; i += blockDim.x) k[base + i] = s[i];
}

__global__ void bitonic_global_kernel(uint64_t* __restrict__ k, int64_t n2, int64_t size, int64_t j) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n2 / 2) return;
  const int64_t i = 2 * t - (t & (j - 1));
  const int64_t l = i + j;
  const bool up = ((i & size) == 0);
  uint64_t a = k[i], b = k[l];
  if ((a > b) == up) {
    k[i] = b;
    k[l] = a;
  }
}

__global__ void fill_u64_kernel(uint64_t* p, int64_t from, int64_t to, uint64_t v) {
  const int64_t i = from + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < to) p[i] = v;
}

void sort_u64(Ctx* c, uint64_t* keys, int64_t n) {
  if (n <= 1) return;
  int64_t n2 = kSortSmem;
  while (n2 < n) n2 <<= 1;
  DBuf<uint64_t> buf;
  buf.reserve(c, n2);
  VER_CUDA(cudaMemcpyAsync(buf.p, keys, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, c->stream));
  if (n2 > n) {
    fill_u64_kernel<<<cdiv(n2 - n, 256), 256, 0, c->stream>>>(buf.p, n, n2, ~0ull);
    after_launch(c);
  }
  const unsigned nblk = (unsigned)(n2 / kSortSmem);
  bitonic_local_kernel<<<nblk, 1024, 0, c->stream>>>(buf.p, n2, 2);
  after_launch(c);
  for (int64_t size = 2 * kSortSmem; size <= n2; size <<= 1) {
    for (int64_t j = size >> 1; j >= kSortSmem; j >>= 1) {
      bitonic_global_kernel<<<cdiv(n2 / 2, 256), 256, 0, c->stream>>>(buf.p, n2, size, j);
      after_launch(c);
    }
    bitonic_local_kernel<<<nblk, 1024, 0, c->stream>>>(buf.p, n2, (int)size);
    after_launch(c);
  }
  VER_CUDA(cudaMemcpyAsync(keys, buf.p, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, c->stream));
}

}  // namespace verg

using namespace verg;

extern "C" {

const char* ver_last_error(void) { return g_last_error.c_str(); }

const char* ver_version(void) {
  return "ver_b200 0.1 (sm_100a; fp32 parity GEMMs + fp64 scan carries; NCCL DD-PPO)";
}

ver_status ver_ctx_create(int device, ver_ctx* out) {
  VER_API_BEGIN
  int n = 0;
  VER_CUDA(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) config_error("ver_ctx_create: no such CUDA device");
  auto* h = new ver_ctx_s();
  h->c.device = device;
  VER_CUDA(cudaSetDevice(device));
  VER_CUDA(cudaDeviceGetAttribute(&h->c.num_sms, cudaDevAttrMultiProcessorCount, device));
  VER_CUDA(cudaStreamCreateWithFlags(&h->c.stream, cudaStreamNonBlocking));
  // keep freed pool memory cached across updates
  cudaMemPool_t pool;
  VER_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t thr = UINT64_MAX;
  VER_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  *out = h;
  VER_API_END
}

ver_status ver_ctx_destroy(ver_ctx ctx) {
  VER_API_BEGIN
  if (!ctx) return VER_OK;
  activate(&ctx->c);
  cudaStreamSynchronize(ctx->c.stream);
  if (ctx->c.comm) ncclCommDestroy(ctx->c.comm);
  if (ctx->c.pinned) cudaFreeHost(ctx->c.pinned);
  cudaStreamDestroy(ctx->c.stream);
  delete ctx;
  VER_API_END
}

ver_status ver_ctx_synchronize(ver_ctx ctx) {
  VER_API_BEGIN
  activate(&ctx->c);
  sync(&ctx->c);
  VER_API_END
}

ver_status ver_ctx_stream(ver_ctx ctx, uint64_t* s) {
  VER_API_BEGIN
  *s = reinterpret_cast<uint64_t>(ctx->c.stream);
  VER_API_END
}

ver_status ver_ctx_launch_count(ver_ctx ctx, int64_t* count, int reset) {
  VER_API_BEGIN
  if (count) *count = ctx->c.launches;
  if (reset) ctx->c.launches = 0;
  VER_API_END
}

ver_status ver_ctx_set_precision(ver_ctx ctx, int mode) {
  VER_API_BEGIN
  if (mode != 0 && mode != 1) config_error("ver_ctx_set_precision: mode must be 0 or 1");
  ctx->c.precision = mode;
  VER_API_END
}

ver_status ver_ctx_set_tensor_cores(ver_ctx ctx, int enable) {
  VER_API_BEGIN
  ctx->c.tensor_cores = enable != 0;
  VER_API_END
}

ver_status ver_nccl_unique_id(uint8_t id_out[128]) {
  VER_API_BEGIN
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  VER_NCCL(ncclGetUniqueId(&id));
  std::memcpy(id_out, &id, 128);
  VER_API_END
}

ver_status ver_ctx_init_nccl(ver_ctx ctx, const uint8_t id[128], int nranks, int rank) {
  VER_API_BEGIN
  activate(&ctx->c);
  if (nranks < 1 || rank < 0 || rank >= nranks) config_error("ver_ctx_init_nccl: bad rank");
  if (ctx->c.comm) {
    ncclCommDestroy(ctx->c.comm);
    ctx->c.comm = nullptr;
  }
  ncclUniqueId uid;
  std::memcpy(&uid, id, 128);
  VER_NCCL(ncclCommInitRank(&ctx->c.comm, nranks, uid, rank));
  ctx->c.nranks = nranks;
  ctx->c.rank = rank;
  VER_API_END
}

ver_status ver_allreduce_sum_i64(ver_ctx ctx, int64_t* h, int n) {
  VER_API_BEGIN
  Ctx* c = &ctx->c;
  activate(c);
  if (!c->comm || n == 0) return VER_OK;  // no communicator: one replica, identity
  DBuf<int64_t> d;
  d.reserve(c, n);
  d.upload(h, n);
  VER_NCCL(ncclAllReduce(d.p, d.p, n, ncclInt64, ncclSum, c->comm, c->stream));
  d.download(h, n);
  sync(c);
  VER_API_END
}

ver_status ver_allreduce_mean_f64(ver_ctx ctx, double* h, int n) {
  VER_API_BEGIN
  Ctx* c = &ctx->c;
  activate(c);
  if (!c->comm || n == 0) return VER_OK;  // no communicator: one replica, identity
  DBuf<double> d;
  d.reserve(c, n);
  d.upload(h, n);
  VER_NCCL(ncclAllReduce(d.p, d.p, n, ncclFloat64, ncclAvg, c->comm, c->stream));
  d.download(h, n);
  sync(c);
  VER_API_END
}

ver_status ver_allgather_f64(ver_ctx ctx, const double* in, int n, double* out) {
  VER_API_BEGIN
  Ctx* c = &ctx->c;
  activate(c);
  if (!c->comm) {  // no communicator: one replica, identity
    std::memcpy(out, in, sizeof(double) * n);
    return VER_OK;
  }
  DBuf<double> d, o;
  d.reserve(c, n);
  o.reserve(c, (size_t)n * c->nranks);
  d.upload(in, n);
  VER_NCCL(ncclAllGather(d.p, o.p, n, ncclFloat64, c->comm, c->stream));
  o.download(out, (size_t)n * c->nranks);
  sync(c);
  VER_API_END
}

}  // extern "C"
