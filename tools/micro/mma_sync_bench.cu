// mma.sync latency / throughput on sm_100a (legacy warp-level MMA, the
// small-batch GEMV's instruction): cycles per instruction for one dependent
// chain and for C independent chains per warp, W warps per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_sync_bench mma_sync_bench.cu
#include <cstdio>
#include <cstdint>

template <int KIND>
__device__ __forceinline__ void mma(uint32_t (&d)[4], uint32_t a0, uint32_t b0) {
  if constexpr (KIND == 0)
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%4,%4,%4}, {%5,%5}, {%0,%1,%2,%3};"
                 : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3]) : "r"(a0), "r"(b0));
  else if constexpr (KIND == 1)
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%4,%4,%4}, {%5,%5}, {%0,%1,%2,%3};"
                 : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3]) : "r"(a0), "r"(b0));
  else
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%4,%4,%4}, {%5,%5}, {%0,%1,%2,%3};"
                 : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3]) : "r"(a0), "r"(b0));
}

template <int KIND, int C>
__global__ void bench(int iters, uint32_t seed, unsigned long long* cyc, uint32_t* sink) {
  uint32_t d[C][4];
#pragma unroll
  for (int c = 0; c < C; ++c)
    for (int e = 0; e < 4; ++e) d[c][e] = 0;
  const uint32_t a = seed ^ threadIdx.x, b = seed * 3u + threadIdx.x;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < C; ++c) mma<KIND>(d[c], a + c, b);
  }
  const unsigned long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s ^= d[c][0] ^ d[c][1] ^ d[c][2] ^ d[c][3];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int KIND, int C>
void run(const char* name, int warps) {
  unsigned long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, 8);
  cudaMalloc(&sink, 148 * 1024 * 4);
  const int iters = 2048;
  bench<KIND, C><<<148, 32 * warps>>>(iters, 1, cyc, sink);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  bench<KIND, C><<<148, 32 * warps>>>(iters, 1, cyc, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double per = static_cast<double>(c) / (iters * C);
  const int k = KIND == 0 ? 8 : KIND == 1 ? 16 : 32;
  const double ops = 2.0 * 16 * 8 * k * iters * C * warps * 148;
  printf("%-5s chains=%d warps/SM=%2d: %6.2f cycles/mma per warp, %7.1f T(FL)OP/s\n", name, C, warps, per,
         ops / (ms * 1e-3) / 1e12);
  cudaFree(cyc);
  cudaFree(sink);
}

int main() {
  for (int w : {1, 4, 8, 16, 32}) {
    run<0, 1>("tf32", w);
    run<0, 4>("tf32", w);
    run<1, 1>("bf16", w);
    run<1, 4>("bf16", w);
    run<2, 1>("s8", w);
    run<2, 4>("s8", w);
  }
  return 0;
}
