// common.cuh — shared plumbing of the VER learner library: status/error
// handling, the per-device context (stream, pool, launch accounting, NCCL),
// stream-ordered device buffers and small launch helpers.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "ver_gpu.h"

namespace verg {

// ------------------------------------------------------------------ errors
// Exceptions never cross the C-ABI: every entry point catches and maps them.
struct Error : std::runtime_error {
  ver_status code;
  Error(ver_status c, const std::string& w) : std::runtime_error(w), code(c) {}
};
[[noreturn]] inline void protocol_error(const std::string& w) { throw Error(VER_ERR_PROTOCOL, w); }
[[noreturn]] inline void config_error(const std::string& w) { throw Error(VER_ERR_CONFIG, w); }

void set_last_error(const std::string& w);

#define VER_CUDA(expr)                                                                  \
  do {                                                                                  \
    cudaError_t e__ = (expr);                                                           \
    if (e__ != cudaSuccess)                                                             \
      throw ::verg::Error(VER_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e__)); \
  } while (0)

#define VER_NCCL(expr)                                                                  \
  do {                                                                                  \
    ncclResult_t r__ = (expr);                                                          \
    if (r__ != ncclSuccess)                                                             \
      throw ::verg::Error(VER_ERR_NCCL, std::string(#expr) + ": " + ncclGetErrorString(r__)); \
  } while (0)

// Wraps the body of a C-ABI entry point.
#define VER_API_BEGIN try {
#define VER_API_END                                       \
  return VER_OK;                                          \
  }                                                       \
  catch (const ::verg::Error& e) {                        \
    ::verg::set_last_error(e.what());                     \
    return e.code;                                        \
  }                                                       \
  catch (const std::exception& e) {                       \
    ::verg::set_last_error(e.what());                     \
    return VER_ERR_CONFIG;                                \
  }

// --------------------------------------------------------------- context
struct Ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  int64_t launches = 0;  // kernels launched by this library on `stream`
  int precision = 0;     // tensor-core GEMMs: 0 = 3xTF32 (fp32 parity), 1 = 1xTF32 (fast)
  bool tensor_cores = true;  // tcgen05 GEMMs on (off: fp32 SIMT GEMMs)
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  // optional device-time log: (tag, start, end) event pairs recorded on `stream`
  std::vector<std::tuple<int, cudaEvent_t, cudaEvent_t>>* evlog = nullptr;
  int rec_tag = -1;  // tag for recurrence launches (>= 0 while a learner minibatch is timed)
  int gemm_tag = -1;  // tag for tcgen05 GEMM launches (same)
  double* flop_log = nullptr;  // per-tag algorithmic FLOPs (2 M N K) of the tagged GEMM launches
  int hbm_tag = -1;  // tag for the GAE scan (tag) and gather (tag + 1) launches (ver_bench_gae_gather)
  // pinned scratch for small synchronous reads
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
  void* pinned_buf(size_t bytes);
};

// Records a (tag, start, end) event pair into ctx->evlog around a scope
// (no-op when the log is off or tag < 0).
struct ScopedEv {
  Ctx* c;
  int tag;
  cudaEvent_t a = nullptr;
  ScopedEv(Ctx* c_, int tag_) : c(c_), tag(tag_) {
    if (c->evlog && tag >= 0) {
      cudaEventCreate(&a);
      cudaEventRecord(a, c->stream);
    }
  }
  ~ScopedEv() {
    if (a) {
      cudaEvent_t b;
      cudaEventCreate(&b);
      cudaEventRecord(b, c->stream);
      c->evlog->emplace_back(tag, a, b);
    }
  }
};

// Make the ctx's device current for this thread (entry points call this).
void activate(Ctx* c);

// ---------------------------------------------------------------- buffers
// Device buffer allocated from the stream-ordered pool of ctx's device.
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;  // capacity in elements
  Ctx* ctx = nullptr;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept { *this = std::move(o); }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      n = o.n;
      ctx = o.ctx;
      o.p = nullptr;
      o.n = 0;
    }
    return *this;
  }
  ~DBuf() { release(); }
  void release() {
    if (p && ctx) cudaFreeAsync(p, ctx->stream);
    p = nullptr;
    n = 0;
  }
  // grow to at least `count` elements (contents not preserved)
  void reserve(Ctx* c, size_t count) {
    if (count <= n && ctx == c) return;
    release();
    ctx = c;
    size_t want = count ? count : 1;
    VER_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), want * sizeof(T), c->stream));
    n = want;
  }
  // grow preserving the first `keep` elements
  void grow_keep(Ctx* c, size_t count, size_t keep) {
    if (count <= n && ctx == c) return;
    T* q = nullptr;
    size_t want = count ? count : 1;
    VER_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&q), want * sizeof(T), c->stream));
    if (p && keep)
      VER_CUDA(cudaMemcpyAsync(q, p, keep * sizeof(T), cudaMemcpyDeviceToDevice, c->stream));
    release();
    ctx = c;
    p = q;
    n = want;
  }
  void zero(size_t count) {
    if (count) VER_CUDA(cudaMemsetAsync(p, 0, count * sizeof(T), ctx->stream));
  }
  void upload(const T* h, size_t count) {
    if (count) VER_CUDA(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
  }
  void download(T* h, size_t count) const {
    if (count && h)
      VER_CUDA(cudaMemcpyAsync(h, p, count * sizeof(T), cudaMemcpyDeviceToHost, ctx->stream));
  }
};

inline void sync(Ctx* c) { VER_CUDA(cudaStreamSynchronize(c->stream)); }

// L2 prefetch of [p, p + bytes) (bulk-copy engine, no registers held): the
// range is widened to 16-byte alignment and clipped to [lo, hi).
__device__ __forceinline__ void prefetch_l2(const void* p, size_t bytes, const void* lo, const void* hi) {
  uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
  uintptr_t b = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~uintptr_t(15);
  const uintptr_t l = (reinterpret_cast<uintptr_t>(lo) + 15) & ~uintptr_t(15);
  const uintptr_t h = reinterpret_cast<uintptr_t>(hi) & ~uintptr_t(15);
  if (a < l) a = l;
  if (b > h) b = h;
  if (b > a)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((uint32_t)(b - a)) : "memory");
}
// Per-device once-caches (function attributes, occupancy probes): a process may
// drive several GPUs from several host threads (one learner thread per GPU), so
// anything derived from a device is cached per device ordinal, never globally.
constexpr int kMaxDevices = 64;
inline int dev_slot(const Ctx* c) { return c->device >= 0 && c->device < kMaxDevices ? c->device : 0; }
// experiments only: integer tuning knob from the environment
int env_int(const char* name, int dflt);
// VER_PROFILING=1: launches that a kernel profiler cannot replay take a
// profiler-compatible form (the CTA-pair step kernel drops the cooperative
// attribute; ncu serializes kernels, so its CTAs are co-resident anyway)
bool profiling();

inline unsigned cdiv(size_t a, size_t b) { return static_cast<unsigned>((a + b - 1) / b); }

// Launch accounting + error check after every kernel launch.
// GRU gate nonlinearities (nn.cpp:235-250) of every recurrence kernel, on the
// SFU (ex2 + rcp): absolute error ~1e-7, far inside the 1e-5 parity bar, and
// both tails saturate exactly (exp -> 0 / inf).  They sit on the per-step
// critical path of the recurrence, where expf / tanhf cost ~3x the latency.
__device__ __forceinline__ float gate_sigm(float x) { return __fdividef(1.f, 1.f + __expf(-x)); }
__device__ __forceinline__ float gate_tanh(float x) { return 1.f - __fdividef(2.f, 1.f + __expf(2.f * x)); }

inline void after_launch(Ctx* c) {
  c->launches++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw Error(VER_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
}

// Programmatic dependent launch of the small kernels between the GEMMs: the
// kernel must start with pdl_wait() (its inputs are visible after it) and may
// let its own successor be scheduled early with pdl_trigger().
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
int env_int(const char* name, int dflt);
template <class... KArgs, class... Args>
inline void launch_pdl(Ctx* c, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
  if (e != cudaSuccess) throw Error(VER_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
  after_launch(c);
}

// ------------------------------------------------------------- scans etc.
// Exclusive scan of n int32 on ctx's stream (out may alias in).  If total is
// non-null it receives the sum (device).  Implemented in util.cu.
void exclusive_scan_i32(Ctx* c, const int32_t* in, int32_t* out, int64_t n, int32_t* total);
// Exclusive scan of n uint8 flags into int32.
void exclusive_scan_u8(Ctx* c, const uint8_t* in, int32_t* out, int64_t n, int32_t* total);
// Ascending sort of n unique uint64 keys in place (bitonic; n arbitrary).
void sort_u64(Ctx* c, uint64_t* keys, int64_t n);
// Ascending sort of n non-negative doubles (as uint64 bit patterns) in place.
inline void sort_pos_f64(Ctx* c, double* keys, int64_t n) {
  sort_u64(c, reinterpret_cast<uint64_t*>(keys), n);
}

}  // namespace verg

// The opaque handle types of the C-ABI.
struct ver_ctx_s {
  verg::Ctx c;
};
