// coordinator.cu — VER's joint preemption counter across replicas (SURVEY
// §8(f) row 2; PreemptCoordinator, distributed.hpp:95-128, driven from
// ReplicaGroup::replica_main, distributed.cpp:208-264).
//
// The reference keeps one std::atomic<long> shared by the replica threads:
// every commit adds to it, and the first add that reaches the threshold
// force-closes every replica's rollout.  With one process per GPU the counter
// is a device word owned by one rank and mapped into the others through CUDA
// IPC (NVLink / NVSwitch peer memory on a multi-GPU node, the same device
// otherwise): add_steps is one system-scope atomicAdd (from a tiny kernel, or
// fused into the inference engine's sampling kernel: ver_engine_attach_preempt),
// and the "fired" word is set with atomicExch so exactly one add fires.  No
// collective is involved, so replicas commit asynchronously as in the
// reference.
//
// NCCL mode (ver_preempt_create_nccl, SURVEY §8(e) "global committed-step
// ncclAllReduce(int64) per tick"): every rank owns a local counter; adds
// accumulate locally and ver_preempt_tick -- a collective all ranks call once
// per collection tick -- sums the deltas with ncclAllReduce, so every rank
// sees the same global count and fires on the same tick.
#include <cstring>

#include "coordinator.cuh"

namespace verg {

__global__ void preempt_start_kernel(PreemptWords* w, long long threshold) {
  w->count = 0;
  w->fired = 0;
  w->local = 0;
  __threadfence_system();
  w->threshold = threshold;
}

// out[0] = total after the add, out[1] = 1 iff this add fired the preemption
__global__ void preempt_add_kernel(PreemptWords* w, long long n, long long* out) {
  const int f = preempt_add_dev(w, n);
  out[0] = (long long)atomicAdd_system(&w->count, 0ull) + (w->nccl ? (long long)atomicAdd(&w->local, 0ull) : 0);
  out[1] = f;
}

__global__ void preempt_read_kernel(PreemptWords* w, long long* out) {
  out[0] = (long long)atomicAdd_system(&w->count, 0ull);
  out[1] = atomicAdd_system(&w->fired, 0);
}

// NCCL tick, before the collective: this rank's delta since the last tick -> send
__global__ void preempt_tick_take_kernel(PreemptWords* w, unsigned long long* send) {
  send[0] = atomicExch(&w->local, 0ull);
}
// after it: every rank adds the same global delta and fires on the same tick
__global__ void preempt_tick_apply_kernel(PreemptWords* w, const unsigned long long* recv, long long* out) {
  w->count += recv[0];
  const long long th = w->threshold;
  int fired_now = 0;
  if (th > 0 && (long long)w->count >= th && !w->fired) {
    w->fired = 1;
    fired_now = 1;
  }
  out[0] = (long long)w->count;
  out[1] = fired_now;
}

}  // namespace verg

using namespace verg;

static void preempt_call(ver_preempt_s* p, long long* out2) {
  VER_CUDA(cudaMemcpyAsync(out2, p->dout, 2 * sizeof(long long), cudaMemcpyDeviceToHost, p->s));
  VER_CUDA(cudaStreamSynchronize(p->s));
}

extern "C" {

ver_status ver_preempt_create(ver_ctx ctx, ver_preempt* out) {
  VER_API_BEGIN
  Ctx* c = &ctx->c;
  activate(c);
  auto* p = new ver_preempt_s();
  p->c = c;
  p->owner = true;
  VER_CUDA(cudaStreamCreateWithFlags(&p->s, cudaStreamNonBlocking));
  VER_CUDA(cudaMalloc(reinterpret_cast<void**>(&p->w), sizeof(PreemptWords)));
  VER_CUDA(cudaMemsetAsync(p->w, 0, sizeof(PreemptWords), p->s));
  VER_CUDA(cudaMalloc(reinterpret_cast<void**>(&p->dout), 4 * sizeof(long long)));
  VER_CUDA(cudaStreamSynchronize(p->s));
  *out = p;
  VER_API_END
}

ver_status ver_preempt_create_nccl(ver_ctx ctx, ver_preempt* out) {
  VER_API_BEGIN
  Ctx* c = &ctx->c;
  activate(c);
  if (!c->comm) config_error("preempt: ver_preempt_create_nccl needs ver_ctx_init_nccl first");
  auto* p = new ver_preempt_s();
  p->c = c;
  p->owner = true;
  p->nccl = true;
  VER_CUDA(cudaStreamCreateWithFlags(&p->s, cudaStreamNonBlocking));
  VER_CUDA(cudaMalloc(reinterpret_cast<void**>(&p->w), sizeof(PreemptWords)));
  VER_CUDA(cudaMemsetAsync(p->w, 0, sizeof(PreemptWords), p->s));
  VER_CUDA(cudaMemsetAsync(&p->w->nccl, 1, 1, p->s));  // nccl = 1 (little-endian low byte)
  VER_CUDA(cudaMalloc(reinterpret_cast<void**>(&p->dout), 4 * sizeof(long long)));
  VER_CUDA(cudaStreamSynchronize(p->s));
  *out = p;
  VER_API_END
}

// one collective tick (every rank, same order): global count += sum of the
// ranks' deltas; fired_now = 1 on the tick that reaches the threshold
ver_status ver_preempt_tick(ver_preempt p, int64_t* total, int* fired_now) {
  VER_API_BEGIN
  if (!p->nccl) config_error("preempt: ver_preempt_tick is the NCCL-mode collective");
  Ctx* c = p->c;
  activate(c);
  auto* buf = reinterpret_cast<unsigned long long*>(p->dout + 2);  // send, recv
  preempt_tick_take_kernel<<<1, 1, 0, p->s>>>(p->w, buf);
  after_launch(c);
  VER_NCCL(ncclAllReduce(buf, buf + 1, 1, ncclUint64, ncclSum, c->comm, p->s));
  preempt_tick_apply_kernel<<<1, 1, 0, p->s>>>(p->w, buf + 1, p->dout);
  after_launch(c);
  long long r[2];
  VER_CUDA(cudaMemcpyAsync(r, p->dout, 2 * sizeof(long long), cudaMemcpyDeviceToHost, p->s));
  VER_CUDA(cudaStreamSynchronize(p->s));
  if (total) *total = r[0];
  if (fired_now) *fired_now = (int)r[1];
  VER_API_END
}

ver_status ver_preempt_ipc_handle(ver_preempt p, uint8_t handle_out[64]) {
  VER_API_BEGIN
  if (!p->owner || p->nccl) config_error("preempt: only the owning replica of an IPC counter exports it");
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
  VER_CUDA(cudaStreamCreateWithFlags(&p->s, cudaStreamNonBlocking));
  VER_CUDA(cudaMalloc(reinterpret_cast<void**>(&p->dout), 4 * sizeof(long long)));
  *out = p;
  VER_API_END
}

ver_status ver_preempt_destroy(ver_preempt p) {
  VER_API_BEGIN
  if (!p) return VER_OK;
  activate(p->c);
  cudaStreamSynchronize(p->s);
  if (p->owner) cudaFree(p->w);
  else cudaIpcCloseMemHandle(p->w);
  cudaFree(p->dout);
  cudaStreamDestroy(p->s);
  delete p;
  VER_API_END
}

// start_iteration (distributed.hpp:104-108): the owner resets the count
ver_status ver_preempt_start(ver_preempt p, int64_t threshold) {
  VER_API_BEGIN
  if (!p->owner) config_error("preempt: start_iteration runs on the owning replica (every rank in NCCL mode)");
  activate(p->c);
  preempt_start_kernel<<<1, 1, 0, p->s>>>(p->w, threshold);
  after_launch(p->c);
  VER_CUDA(cudaStreamSynchronize(p->s));
  VER_API_END
}

// add_steps (distributed.hpp:110-119): fired_now = 1 on exactly one add per iteration
ver_status ver_preempt_add(ver_preempt p, int64_t n, int64_t* total, int* fired_now) {
  VER_API_BEGIN
  activate(p->c);
  preempt_add_kernel<<<1, 1, 0, p->s>>>(p->w, n, p->dout);
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
  preempt_read_kernel<<<1, 1, 0, p->s>>>(p->w, p->dout);
  after_launch(p->c);
  long long r[2];
  preempt_call(p, r);
  if (total) *total = r[0];
  if (fired) *fired = (int)r[1];
  VER_API_END
}

}  // extern "C"
