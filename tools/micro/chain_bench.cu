// Micro-benchmark: cost of a dependent kernel boundary (PDL launches captured
// in a CUDA graph, 148 CTAs each) vs a grid-wide barrier inside one persistent
// kernel (148 CTAs, atomic counter + generation flag). Each phase reads a
// value written by the previous phase (a true dependency).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void step_kernel(float* buf, int i) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const float v = buf[(i & 1) * 1024 + threadIdx.x];
  buf[((i + 1) & 1) * 1024 + threadIdx.x] = v + 1.0f;
}

__device__ void grid_barrier(unsigned* count, volatile unsigned* gen, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(count, 1) == nblocks - 1) {
      *count = 0;
      __threadfence();
      *gen = g + 1;
    } else {
      while (*gen == g) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void persistent_kernel(float* buf, int phases, unsigned* count, unsigned* gen) {
  for (int i = 0; i < phases; ++i) {
    const float v = __ldcg(buf + (i & 1) * 1024 + threadIdx.x);
    __stcg(buf + ((i + 1) & 1) * 1024 + threadIdx.x, v + 1.0f);
    grid_barrier(count, gen, gridDim.x);
  }
}

int main() {
  const int phases = 1000;
  float* buf;
  unsigned *count, *gen;
  cudaMalloc(&buf, 2048 * sizeof(float));
  cudaMalloc(&count, 4);
  cudaMalloc(&gen, 4);
  cudaMemset(buf, 0, 2048 * 4);
  cudaMemset(count, 0, 4);
  cudaMemset(gen, 0, 4);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  for (int pdl = 0; pdl < 2; ++pdl) {
    cudaGraph_t g;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < phases; ++i) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = 148;
      cfg.blockDim = 256;
      cfg.stream = st;
      cfg.attrs = attr;
      cfg.numAttrs = pdl;
      cudaLaunchKernelEx(&cfg, step_kernel, buf, i);
    }
    cudaStreamEndCapture(st, &g);
    cudaGraphExec_t ge;
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, st);
    cudaStreamSynchronize(st);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, st);
    cudaGraphLaunch(ge, st);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("graph of %d dependent kernels (148 CTAs), pdl=%d: %.3f us per kernel\n", phases, pdl,
           1000.0f * ms / phases);
  }
  for (int rep = 0; rep < 2; ++rep) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, st);
    persistent_kernel<<<148, 256, 0, st>>>(buf, phases, count, gen);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("persistent kernel, %d grid barriers: %.3f us per phase (%s)\n", phases,
           1000.0f * ms / phases, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
