// One warp's bitonic sort of (score, parent, token) triples (the beam
// selection's), timed with clock64 and %globaltimer; plus the globaltimer
// update granularity.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 [-DBRANCHY] -o /tmp/warp_sort_bench warp_sort_bench.cu
#include <climits>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#ifdef BRANCHY
__device__ __forceinline__ bool better3(float a, int pa, int ta, float b, int pb, int tb) {
  if (a != b) return a > b;
  if (pa != pb) return pa < pb;
  return ta < tb;
}
#else
__device__ __forceinline__ bool better3(float a, int pa, int ta, float b, int pb, int tb) {
  return (a > b) | ((a == b) & ((pa < pb) | ((pa == pb) & (ta < tb))));
}
#endif

__global__ void k(const float* in, float* out, long long* cyc, unsigned long long* ns, int reps) {
  const int lane = threadIdx.x;
  float ss = in[lane];
  int sp = lane / 5, st = (lane * 7919) % 32000;
  if (lane >= 25) { ss = -__int_as_float(0x7f800000); sp = INT_MAX; st = INT_MAX; }
  __syncwarp();
  const long long c0 = clock64();
  const unsigned long long t0 = gt();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
      for (int jj = k >> 1; jj > 0; jj >>= 1) {
        const float os = __shfl_xor_sync(0xffffffffu, ss, jj);
        const int op = __shfl_xor_sync(0xffffffffu, sp, jj);
        const int ot = __shfl_xor_sync(0xffffffffu, st, jj);
        const bool o_better = ot != INT_MAX && (st == INT_MAX || better3(os, op, ot, ss, sp, st));
        const bool keep_better = ((lane & k) == 0) == ((lane & jj) == 0);
        if (keep_better ? o_better : (!o_better && (ot != st || op != sp))) {
          ss = os; sp = op; st = ot;
        }
      }
    }
    ss = ss * 1.0000001f;  // keep the reps dependent
  }
  const long long c1 = clock64();
  const unsigned long long t1 = gt();
  // rank variant: every lane counts the candidates above it (shared copy)
  __shared__ float xs[32];
  __shared__ int xp[32], xt[32];
  xs[lane] = ss; xp[lane] = sp; xt[lane] = st;
  __syncwarp();
  const int nc = 25;
  int rank = 0;
  const long long c2 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll 5
    for (int j = 0; j < nc; ++j) {
      const float sj = xs[j];
      const int pj = xp[j], tj = xt[j];
      rank += tj != INT_MAX && better3(sj, pj, tj, ss, sp, st);
    }
    ss = ss * 1.0000001f;
  }
  const long long c3 = clock64();
  out[lane] = ss + sp + st + rank;
  if (lane == 0) { cyc[0] = c1 - c0; ns[0] = t1 - t0; cyc[1] = c3 - c2; }
  // globaltimer granularity: smallest nonzero delta over 2000 reads
  unsigned long long prev = gt(), mind = ~0ull;
  for (int i = 0; i < 2000; ++i) {
    const unsigned long long x = gt();
    if (x != prev && x - prev < mind) mind = x - prev;
    prev = x;
  }
  if (lane == 0) ns[1] = mind;
}

int main() {
  float *in, *out; long long* cyc; unsigned long long* ns;
  cudaMalloc(&in, 128); cudaMalloc(&out, 128); cudaMalloc(&cyc, 16); cudaMalloc(&ns, 16);
  float h[32];
  for (int i = 0; i < 32; ++i) h[i] = (i * 37 % 29) * 0.5f - 3.0f;
  cudaMemcpy(in, h, 128, cudaMemcpyHostToDevice);
  for (int reps : {1, 10, 100}) {
    k<<<1, 32>>>(in, out, cyc, ns, reps);
    long long c, cc[2]; unsigned long long n[2];
    cudaMemcpy(cc, cyc, 16, cudaMemcpyDeviceToHost);
    c = cc[0];
    cudaMemcpy(n, ns, 16, cudaMemcpyDeviceToHost);
    printf("reps %3d: %lld cycles (%.0f per sort), %llu ns; globaltimer step %llu ns; rank loop %.0f cycles\n", reps, c,
           double(c) / reps, n[0], n[1], double(cc[1]) / reps);
  }
  return 0;
}
