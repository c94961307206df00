// Kernel launch helper: every kernel of the path is launched with
// programmatic dependent launch (PDL) enabled, so a kernel's CTAs can start
// (TMEM allocation, barrier init, tensor-map prefetch) while its predecessor
// drains. Kernels call pdl_wait() before touching predecessor outputs and
// pdl_trigger() right after, which keeps the usual stream ordering for data.
// MTG_NO_PDL=1 in the environment launches plainly (debugging). Measured
// alternatives: triggering before the wait (-6 % int8: waiting CTAs of the
// next grid take SM slots early) and at block exit (-4 %).
#pragma once

#include <cstdlib>
#include <utility>

#include <cuda_runtime.h>

#include "errors.hpp"

namespace mtg {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// In-graph kernel timeline (MTG_TRACE=1, diagnostics only): a traced kernel
// records the first post-wait time of its CTAs and the last CTA exit time
// (%globaltimer, ns) into buf[2 * (step * per_step + slot) + {0, 1}].
struct KTrace {
  unsigned long long* buf = nullptr;
  int slot = 0;
  int per_step = 0;
  const int* d_step = nullptr;
  // MTG_TRACE=2 (MTG_TRACE_PHASES builds): per-phase times (latest CTA to
  // reach phase i), kTracePhases per (step, slot)
  unsigned long long* ph = nullptr;
};
constexpr int kTracePhases = 8;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void trace_begin(const KTrace& k) {
  if (k.buf && threadIdx.x == 0)
    atomicMin(&k.buf[2 * (static_cast<long long>(*k.d_step) * k.per_step + k.slot)], gtimer());
}
__device__ __forceinline__ void trace_end(const KTrace& k) {
  if (k.buf && threadIdx.x == 0)
    atomicMax(&k.buf[2 * (static_cast<long long>(*k.d_step) * k.per_step + k.slot) + 1], gtimer());
}
// Compiled in only for diagnostics builds (make EXTRA=-DMTG_TRACE_PHASES=1,
// tools/build_phases.sh): even untaken, the checks cost ~0.1-0.4 us per GEMM.
#ifndef MTG_TRACE_PHASES
#define MTG_TRACE_PHASES 0
#endif
__device__ __forceinline__ void trace_phase(const KTrace& k, int i) {
  if constexpr (MTG_TRACE_PHASES != 0) {
    if (k.ph)
      atomicMax(&k.ph[(static_cast<long long>(*k.d_step) * k.per_step + k.slot) * kTracePhases + i],
                gtimer());
  }
}
__device__ __forceinline__ void trace_phase_at(const KTrace& k, int t, int i) {
  if constexpr (MTG_TRACE_PHASES != 0) {
    if (k.ph)
      atomicMax(&k.ph[(static_cast<long long>(t) * k.per_step + k.slot) * kTracePhases + i], gtimer());
  }
}
// Variants with the step passed in (kernels that advance the step counter).
__device__ __forceinline__ void trace_begin_at(const KTrace& k, int t) {
  if (k.buf && threadIdx.x == 0)
    atomicMin(&k.buf[2 * (static_cast<long long>(t) * k.per_step + k.slot)], gtimer());
}
__device__ __forceinline__ void trace_end_at(const KTrace& k, int t) {
  if (k.buf && threadIdx.x == 0)
    atomicMax(&k.buf[2 * (static_cast<long long>(t) * k.per_step + k.slot) + 1], gtimer());
}

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("MTG_NO_PDL");
    return !(e && e[0] == '1');
  }();
  return on;
}

// Raises `fn`'s dynamic shared-memory limit to at least `bytes` on the
// calling thread's current device. Function attributes are per device, so
// the cache is keyed by (device, function); thread-safe (kernels.cu).
void ensure_smem_attr(const void* fn, size_t bytes);
template <typename... KArgs>
inline void ensure_smem_attr(void (*fn)(KArgs...), size_t bytes) {
  ensure_smem_attr(reinterpret_cast<const void*>(fn), bytes);
}

// RAII: makes `device` current for the scope, restoring the previous device.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int device) {
    MTG_CUDA(cudaGetDevice(&prev));
    if (prev != device) MTG_CUDA(cudaSetDevice(device));
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

template <typename... KArgs, typename... Args>
inline void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                     cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  MTG_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

}  // namespace mtg
