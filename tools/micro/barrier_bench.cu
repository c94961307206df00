// Micro-benchmark: grid-wide barrier variants inside one persistent kernel
// (148 CTAs, one per SM) against a dependent PDL kernel boundary. Each phase
// reads a value the previous phase wrote (a true dependency).
//   naive     : counter reset by the last arriver + generation flag (chain_bench.cu)
//   monotonic : red.release.gpu add on a monotonically increasing counter,
//               ld.acquire.gpu spin until counter >= (phase + 1) * nblocks
//   mono+sleep: same with __nanosleep(20) between polls
//   flags     : per-CTA arrival flag words (no atomics), CTA 0 gathers them and
//               publishes a release flag
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void step_kernel(float* buf, int i) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const float v = buf[(i & 1) * 1024 + threadIdx.x];
  buf[((i + 1) & 1) * 1024 + threadIdx.x] = v + 1.0f;
}

template <int MODE>
__global__ void persistent_kernel(float* buf, int phases, unsigned* count, unsigned* flags) {
  const unsigned nb = gridDim.x;
  for (int i = 0; i < phases; ++i) {
    const float v = __ldcg(buf + (i & 1) * 1024 + (blockIdx.x * 7 + threadIdx.x) % 1024);
    __stcg(buf + ((i + 1) & 1) * 1024 + (blockIdx.x * 7 + threadIdx.x) % 1024, v + 1.0f);
    __syncthreads();
    if (threadIdx.x == 0) {
      if (MODE == 0 || MODE == 1) {
        red_release_add(count, 1);
        const unsigned target = (i + 1) * nb;
        while (ld_acquire(count) < target) {
          if (MODE == 1) __nanosleep(20);
        }
      } else {
        // flags: CTA b writes flags[b] = i + 1; CTA 0 waits for all, then
        // publishes flags[nb] = i + 1 which everyone polls.
        st_release(flags + blockIdx.x * 32, i + 1);
        if (blockIdx.x == 0) {
          for (unsigned b = 0; b < nb; ++b)
            while (ld_acquire(flags + b * 32) < unsigned(i + 1)) {
            }
          st_release(flags + nb * 32, i + 1);
        } else {
          while (ld_acquire(flags + nb * 32) < unsigned(i + 1)) {
          }
        }
      }
    }
    __syncthreads();
  }
}

// Same, but the first warp polls with all lanes over the flags (warp-parallel gather).
__global__ void persistent_warpgather(float* buf, int phases, unsigned* flags) {
  const unsigned nb = gridDim.x;
  for (int i = 0; i < phases; ++i) {
    const float v = __ldcg(buf + (i & 1) * 1024 + (blockIdx.x * 7 + threadIdx.x) % 1024);
    __stcg(buf + ((i + 1) & 1) * 1024 + (blockIdx.x * 7 + threadIdx.x) % 1024, v + 1.0f);
    __syncthreads();
    if (threadIdx.x < 32) {
      if (threadIdx.x == 0) st_release(flags + blockIdx.x * 32, i + 1);
      if (blockIdx.x == 0) {
        for (unsigned b = threadIdx.x; b < nb; b += 32)
          while (ld_acquire(flags + b * 32) < unsigned(i + 1)) {
          }
        __syncwarp();
        if (threadIdx.x == 0) st_release(flags + nb * 32, i + 1);
      } else if (threadIdx.x == 0) {
        while (ld_acquire(flags + nb * 32) < unsigned(i + 1)) {
        }
      }
      __syncwarp();
    }
    __syncthreads();
  }
}

int main() {
  const int phases = 2000;
  float* buf;
  unsigned *count, *flags;
  cudaMalloc(&buf, 2048 * sizeof(float));
  cudaMalloc(&count, 4);
  cudaMalloc(&flags, 160 * 32 * 4);
  cudaMemset(buf, 0, 2048 * 4);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  {
    cudaGraph_t g;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < phases; ++i) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = 148;
      cfg.blockDim = 256;
      cfg.stream = st;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, step_kernel, buf, i);
    }
    cudaStreamEndCapture(st, &g);
    cudaGraphExec_t ge;
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, st);
    cudaStreamSynchronize(st);
    cudaEventRecord(a, st);
    cudaGraphLaunch(ge, st);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("graph of %d dependent PDL kernels (148 CTAs): %.3f us per kernel\n", phases,
           1000.0f * ms / phases);
  }
  const char* names[] = {"monotonic", "mono+sleep", "flags"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(count, 0, 4);
      cudaMemset(flags, 0, 160 * 32 * 4);
      cudaEventRecord(a, st);
      if (mode == 0) persistent_kernel<0><<<148, 256, 0, st>>>(buf, phases, count, flags);
      if (mode == 1) persistent_kernel<1><<<148, 256, 0, st>>>(buf, phases, count, flags);
      if (mode == 2) persistent_kernel<2><<<148, 256, 0, st>>>(buf, phases, count, flags);
      if (mode == 3) persistent_warpgather<<<148, 256, 0, st>>>(buf, phases, flags);
      cudaEventRecord(b, st);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep == 1)
        printf("persistent kernel, %-12s barrier: %.3f us per phase (%s)\n",
               mode < 3 ? names[mode] : "warp-gather", 1000.0f * ms / phases,
               cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
