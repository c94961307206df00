// Micro-benchmark: per-SM weight streaming, 148 CTAs x 256 threads, each CTA
// reading its own contiguous slice of a 64 MB buffer (L2-resident after the
// first pass, and from HBM with a 512 MB buffer):
//   bulk  : cp.async.bulk chunks of `chunk` bytes into a ring of `nst` smem stages
//   ldg   : LDG.128 by all threads, `unroll` loads in flight per thread
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void bulk_kernel(const uint8_t* src, long long per_cta, int chunk, int nst, float* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + nst * chunk);
  const uint8_t* s = src + blockIdx.x * per_cta;
  const int n = (int)(per_cta / chunk);
  if (threadIdx.x == 0) {
    for (int i = 0; i < nst; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int i) {
    uint64_t* b = &bar[i % nst];
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(chunk) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(sm + (i % nst) * chunk)), "l"(s + (long long)i * chunk), "r"(chunk), "r"(su32(b)) : "memory");
  };
  if (threadIdx.x == 0) for (int i = 0; i < nst && i < n; ++i) issue(i);
  float acc = 0.f;
  for (int i = 0; i < n; ++i) {
    const uint32_t ph = (i / nst) & 1;
    asm volatile("{\n\t.reg .pred P1;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}" ::"r"(
                     su32(&bar[i % nst])), "r"(ph) : "memory");
    acc += reinterpret_cast<const float*>(sm + (i % nst) * chunk)[threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0 && i + nst < n) issue(i + nst);
  }
  if (acc == 12345.f) sink[0] = acc;
}

template <int U>
__global__ void ldg_kernel(const uint8_t* src, long long per_cta, float* sink) {
  const uint4* s = reinterpret_cast<const uint4*>(src + blockIdx.x * per_cta);
  const long long n = per_cta / 16;
  uint32_t acc = 0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long j = i + (long long)u * blockDim.x;
      v[u] = j < n ? __ldg(s + j) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].w;
  }
  if (acc == 12345u) sink[0] = (float)acc;
}

int main() {
  float* sink; cudaMalloc(&sink, 4);
  for (long long total : {64LL << 20, 512LL << 20}) {
    uint8_t* buf; cudaMalloc(&buf, total); cudaMemset(buf, 1, total);
    const long long per = total / 148 / 65536 * 65536;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
    for (int chunk : {16384, 65536}) for (int nst : {2, 3, 6}) {
      if (chunk * nst > 200 * 1024) continue;
      const int smem = chunk * nst + 64;
      cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      bulk_kernel<<<148, 256, smem>>>(buf, per, chunk, nst, sink);
      cudaEventRecord(a); for (int r = 0; r < 5; ++r) bulk_kernel<<<148, 256, smem>>>(buf, per, chunk, nst, sink);
      cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
      printf("total %4lld MB bulk chunk %6d nst %d: %7.1f GB/s (%s)\n", total >> 20, chunk, nst,
             5.0 * per * 148 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    ldg_kernel<8><<<148, 256>>>(buf, per, sink);
    cudaEventRecord(a); for (int r = 0; r < 5; ++r) ldg_kernel<8><<<148, 256>>>(buf, per, sink);
    cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    printf("total %4lld MB ldg x8 : %7.1f GB/s\n", total >> 20, 5.0 * per * 148 / (ms * 1e-3) / 1e9);
    ldg_kernel<16><<<148, 512>>>(buf, per, sink);
    cudaEventRecord(a); for (int r = 0; r < 5; ++r) ldg_kernel<16><<<148, 512>>>(buf, per, sink);
    cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    printf("total %4lld MB ldg x16 (512 thr): %7.1f GB/s\n", total >> 20, 5.0 * per * 148 / (ms * 1e-3) / 1e9);
    cudaFree(buf);
  }
  return 0;
}
