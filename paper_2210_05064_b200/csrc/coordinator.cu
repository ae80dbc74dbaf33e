// coordinator.cu — VER's joint preemption counter across replicas (SURVEY
// §8(f) row 2; PreemptCoordinator, distributed.hpp:95-128, driven from
// ReplicaGroup::replica_main, distributed.cpp:208-264).
//
// The reference keeps one std::atomic<long> shared by the replica threads:
// every commit adds to it, and the first add that reaches the threshold
// force-closes every replica's rollout.  With one process per GPU the counter
// is a device word owned by one rank and mapped into the others through CUDA
// IPC (NVLink / NVSwitch peer memory on a multi-GPU node, the same device
// otherwise): add_steps is one system-scope atomicAdd from a tiny kernel, and
// the "fired" word is set with atomicExch so exactly one add fires.  No
// collective is involved, so replicas commit asynchronously as in the
// reference.
#include <cstring>

#include "common.cuh"

namespace verg {

struct PreemptWords {  // device layout shared by all replicas
  unsigned long long count;
  long long threshold;  // <= 0: preemption disabled this iteration
  int fired;
  int pad;
};

__global__ void preempt_start_kernel(PreemptWords* w, long long threshold) {
  w->count = 0;
  w->fired = 0;
  __threadfence_system();
  w->threshold = threshold;
}

// out[0] = total after the add, out[1] = 1 iff this add fired the preemption
__global__ void preempt_add_kernel(PreemptWords* w, long long n, long long* out) {
  const long long th = *(volatile long long*)&w->threshold;
  if (th <= 0) {
    out[0] = (long long)atomicAdd_system(&w->count, 0ull);
    out[1] = 0;
    return;
  }
  const unsigned long long c = atomicAdd_system(&w->count, (unsigned long long)n) + (unsigned long long)n;
  int fired = 0;
  if ((long long)c >= th) fired = atomicExch_system(&w->fired, 1) == 0 ? 1 : 0;
  out[0] = (long long)c;
  out[1] = fired;
}

__global__ void preempt_read_kernel(PreemptWords* w, long long* out) {
  out[0] = (long long)atomicAdd_system(&w->count, 0ull);
  out[1] = atomicAdd_system(&w->fired, 0);
}

}  // namespace verg

using namespace verg;

struct ver_preempt_s {
  Ctx* c = nullptr;
  PreemptWords* w = nullptr;
  bool owner = false;
  long long* dout = nullptr;
};

static void preempt_call(ver_preempt_s* p, long long* out2) {
  VER_CUDA(cudaMemcpyAsync(out2, p->dout, 2 * sizeof(long long), cudaMemcpyDeviceToHost, p->c->stream));
  VER_CUDA(cudaStreamSynchronize(p->c->stream));
}

extern "C" {

ver_status ver_preempt_create(ver_ctx ctx, ver_preempt* out) {
  VER_API_BEGIN
  Ctx* c = &ctx->c;
  activate(c);
  auto* p = new ver_preempt_s();
  p->c = c;
  p->owner = true;
  VER_CUDA(cudaMalloc(reinterpret_cast<void**>(&p->w), sizeof(PreemptWords)));
  VER_CUDA(cudaMemset(p->w, 0, sizeof(PreemptWords)));
  VER_CUDA(cudaMalloc(reinterpret_cast<void**>(&p->dout), 2 * sizeof(long long)));
  *out = p;
  VER_API_END
}

ver_status ver_preempt_ipc_handle(ver_preempt p, uint8_t handle_out[64]) {
  VER_API_BEGIN
  if (!p->owner) config_error("preempt: only the owning replica exports the counter");
  activate(p->c);
  cudaIpcMemHandle_t h;
  VER_CUDA(cudaIpcGetMemHandle(&h, p->w));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t");
  std::memcpy(handle_out, &h, 64);
  VER_API_END
}

ver_status ver_preempt_open(ver_ctx ctx, const uint8_t handle[64], ver_preempt* out) {
  VER_API_BEGIN
  Ctx* c = &ctx->c;
  activate(c);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  auto* p = new ver_preempt_s();
  p->c = c;
  VER_CUDA(cudaIpcOpenMemHandle(reinterpret_cast<void**>(&p->w), h, cudaIpcMemLazyEnablePeerAccess));
  VER_CUDA(cudaMalloc(reinterpret_cast<void**>(&p->dout), 2 * sizeof(long long)));
  *out = p;
  VER_API_END
}

ver_status ver_preempt_destroy(ver_preempt p) {
  VER_API_BEGIN
  if (!p) return VER_OK;
  activate(p->c);
  cudaStreamSynchronize(p->c->stream);
  if (p->owner) cudaFree(p->w);
  else cudaIpcCloseMemHandle(p->w);
  cudaFree(p->dout);
  delete p;
  VER_API_END
}

// start_iteration (distributed.hpp:104-108): the owner resets the count
ver_status ver_preempt_start(ver_preempt p, int64_t threshold) {
  VER_API_BEGIN
  if (!p->owner) config_error("preempt: start_iteration runs on the owning replica");
  activate(p->c);
  preempt_start_kernel<<<1, 1, 0, p->c->stream>>>(p->w, threshold);
  after_launch(p->c);
  VER_CUDA(cudaStreamSynchronize(p->c->stream));
  VER_API_END
}

// add_steps (distributed.hpp:110-119): fired_now = 1 on exactly one add per iteration
ver_status ver_preempt_add(ver_preempt p, int64_t n, int64_t* total, int* fired_now) {
  VER_API_BEGIN
  activate(p->c);
  preempt_add_kernel<<<1, 1, 0, p->c->stream>>>(p->w, n, p->dout);
  after_launch(p->c);
  long long r[2];
  preempt_call(p, r);
  if (total) *total = r[0];
  if (fired_now) *fired_now = (int)r[1];
  VER_API_END
}

// count() (distributed.hpp:121) and whether this iteration has fired
ver_status ver_preempt_state(ver_preempt p, int64_t* total, int* fired) {
  VER_API_BEGIN
  activate(p->c);
  preempt_read_kernel<<<1, 1, 0, p->c->stream>>>(p->w, p->dout);
  after_launch(p->c);
  long long r[2];
  preempt_call(p, r);
  if (total) *total = r[0];
  if (fired) *fired = (int)r[1];
  VER_API_END
}

}  // extern "C"
