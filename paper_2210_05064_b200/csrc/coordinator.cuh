// coordinator.cuh — device words of VER's joint preemption counter
// (PreemptCoordinator, distributed.hpp:95-128) shared by coordinator.cu (the
// ver_preempt handle) and engine.cu (the commit add fused into the sampling
// kernel).
#pragma once

#include "common.cuh"

namespace verg {

struct PreemptWords {  // device layout shared by all replicas
  unsigned long long count;  // committed steps of this iteration (IPC: all replicas; NCCL: ticks summed)
  long long threshold;       // <= 0: preemption disabled this iteration
  int fired;
  int nccl;                   // 1: adds go to `local`, ver_preempt_tick sums them over the ranks
  unsigned long long local;  // NCCL mode: this rank's commits since the last tick
};

// add_steps (distributed.hpp:110-119) from device code: IPC mode adds to the
// shared count and sets `fired` on exactly one add per iteration; NCCL mode
// accumulates locally until the next collective tick.  Returns 1 iff this add fired.
__device__ __forceinline__ int preempt_add_dev(PreemptWords* w, long long n) {
  if (n <= 0) return 0;
  if (*(volatile int*)&w->nccl) {
    atomicAdd(&w->local, (unsigned long long)n);
    return 0;
  }
  const long long th = *(volatile long long*)&w->threshold;
  if (th <= 0) return 0;
  const unsigned long long c = atomicAdd_system(&w->count, (unsigned long long)n) + (unsigned long long)n;
  if ((long long)c >= th) return atomicExch_system(&w->fired, 1) == 0 ? 1 : 0;
  return 0;
}
__device__ __forceinline__ int preempt_fired_dev(PreemptWords* w) { return atomicAdd_system(&w->fired, 0); }

}  // namespace verg

// handle of a counter (owned, or mapped from the owner through CUDA IPC, or NCCL-ticked)
struct ver_preempt_s {
  verg::Ctx* c = nullptr;
  verg::PreemptWords* w = nullptr;
  bool owner = false;
  bool nccl = false;
  long long* dout = nullptr;
  // its own non-blocking stream: add / state / start / tick never queue behind
  // the learner's or the engine's work on the ctx stream
  cudaStream_t s = nullptr;
};
