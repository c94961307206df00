// Dependent-latency cost of the row routines used inside the small-batch
// GEMV (rowops.cuh): one warp, clock64 around each piece, averaged over reps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -I../../paper_2008_04885_b200/csrc -o /tmp/ln_chain_bench ln_chain_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "rowops.cuh"

using namespace mtg;

__global__ void k(const float* x, const float* g, const float* b, float* out, long long* cyc, int reps) {
  const int lane = threadIdx.x;
  float xv[16], gv[16], bv[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    xv[i] = x[lane + 32 * i];
    gv[i] = g[lane + 32 * i];
    bv[i] = b[lane + 32 * i];
  }
  long long t_sum = 0, t_ln = 0, t_q = 0, t_div = 0;
  float acc = 0.0f;
  for (int r = 0; r < reps; ++r) {
    long long c0 = clock64();
    float s = warp_allsum(xv[r & 15] + acc);
    long long c1 = clock64();
    float v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = xv[i] + s * 1e-30f;
    int bad = 0;
    const float mx = ln_normalize_regs<16>(v, gv, bv, 512, lane, &bad);
    long long c2 = clock64();
    const float scale = qscale_of(mx);
    int qs = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) qs += quant1(v[i], scale);
    long long c3 = clock64();
    const float dv = __fdiv_rn(127.0f, mx + acc);
    long long c4 = clock64();
    acc += (qs + dv) * 1e-30f;
    if (r == 0 && lane == 0) {
      cyc[4] = c1 - c0;
      cyc[5] = c2 - c1;
      cyc[6] = c3 - c2;
    }
    t_sum += c1 - c0;
    t_ln += c2 - c1;
    t_q += c3 - c2;
    t_div += c4 - c3;
  }
  out[lane] = acc;
  if (lane == 0) {
    cyc[0] = t_sum / reps;
    cyc[1] = t_ln / reps;
    cyc[2] = t_q / reps;
    cyc[3] = t_div / reps;
  }
}

int main() {
  float *x, *g, *b, *o;
  long long* cyc;
  cudaMalloc(&x, 2048); cudaMalloc(&g, 2048); cudaMalloc(&b, 2048); cudaMalloc(&o, 128); cudaMalloc(&cyc, 64);
  float h[512];
  for (int i = 0; i < 512; ++i) h[i] = (i * 37 % 101) * 0.01f - 0.5f;
  cudaMemcpy(x, h, 2048, cudaMemcpyHostToDevice);
  for (int i = 0; i < 512; ++i) h[i] = 1.0f;
  cudaMemcpy(g, h, 2048, cudaMemcpyHostToDevice);
  for (int i = 0; i < 512; ++i) h[i] = 0.0f;
  cudaMemcpy(b, h, 2048, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(x, g, b, o, cyc, 100);
  long long c[7];
  cudaMemcpy(c, cyc, 56, cudaMemcpyDeviceToHost);
  printf("warp_allsum %lld cycles, ln_normalize_regs<16> %lld, qscale + 16 quant1 %lld, one __fdiv_rn %lld\n",
         c[0], c[1], c[2], c[3]);
  printf("first (cold) iteration: warp_allsum %lld, ln %lld, quant %lld\n", c[4], c[5], c[6]);
  return 0;
}
