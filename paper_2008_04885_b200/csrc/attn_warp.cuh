// Shared pieces of the head-dim-64 decoder attention kernels (attn_small.cu,
// gemv.cu's fused cross-attention): the swizzled key / value staging and the
// warp-per-query attention of kernels.cu attend_warp_staged64 (P3 dots, P1
// softmax over lane-strided keys, contexts summed in key order).
#pragma once

#include <cuda_runtime.h>

#include "detmath.cuh"
#include "kernels.cuh"

namespace mtg {

constexpr int kAttnDh = 64;

__device__ __forceinline__ void cp_async16s(float* smem_dst, const float* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   static_cast<unsigned>(__cvta_generic_to_shared(smem_dst))),
               "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// Row j of a [keys][64] block, 16-byte chunk c stored at chunk c ^ (j & 15):
// lane-per-key reads and column-per-thread reads are both conflict-free.
__device__ __forceinline__ int swz(int j, int c4) { return j * kAttnDh + ((c4 ^ (j & 15)) << 2); }

// Copies key / value rows [j0, j1) (row pointers from kp / vp) into K / V.
template <class KP, class VP>
__device__ __forceinline__ void stage_kv(float* K, float* V, int j0, int j1, KP kp, VP vp) {
  for (int i = threadIdx.x; i < (j1 - j0) * 16; i += blockDim.x) {
    const int j = j0 + (i >> 4), c4 = i & 15;
    cp_async16s(K + swz(j, c4), kp(j) + 4 * c4);
    cp_async16s(V + swz(j, c4), vp(j) + 4 * c4);
  }
}

// Shared-memory float4 load the compiler keeps in place: the query is
// re-read per key instead of being hoisted into 64 registers (which cut the
// batched cross-attention's occupancy below one wave: 40 -> 106 registers).
__device__ __forceinline__ float4 lds4(const float* p) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(static_cast<unsigned>(__cvta_generic_to_shared(p)))
               : "memory");
  return v;
}

// One warp attends one query (wq, 64 values in shared memory) over n staged
// keys; ws holds n scores. Lane l returns the context columns l and l + 32.
__device__ __forceinline__ void attend_warp64(const float* K, const float* V, const float* wq,
                                              float* ws, int n, float scale, int lane, float& ca,
                                              float& cb) {
  // scores (P3): lane per key, dot over the head dimension in order, x scale
  float mx = -__int_as_float(0x7f800000);
  for (int j = lane; j < n; j += 32) {
    float acc = 0.0f;
#pragma unroll
    for (int c4 = 0; c4 < 16; ++c4) {
      const float4 kv = *reinterpret_cast<const float4*>(K + swz(j, c4));
      const float4 qv = lds4(wq + 4 * c4);
      acc = __fadd_rn(acc, __fmul_rn(qv.x, kv.x));
      acc = __fadd_rn(acc, __fmul_rn(qv.y, kv.y));
      acc = __fadd_rn(acc, __fmul_rn(qv.z, kv.z));
      acc = __fadd_rn(acc, __fmul_rn(qv.w, kv.w));
    }
    const float v = __fmul_rn(acc, scale);
    ws[j] = v;
    mx = fmaxf(mx, v);
  }
  mx = warp_allmax(mx);
  float part = 0.0f;  // P1: lane-strided keys in order, then the butterfly
  for (int j = lane; j < n; j += 32) {
    const float e = det_expf_nonpos(__fsub_rn(ws[j], mx));
    ws[j] = e;
    part = __fadd_rn(part, e);
  }
  const float sum = warp_allsum(part);
  for (int j = lane; j < n; j += 32) ws[j] = __fdiv_rn(ws[j], sum);
  __syncwarp();
  // context: lane owns columns lane and lane + 32, keys in order
  float acc_a = 0.0f, acc_b = 0.0f;
  for (int j = 0; j < n; ++j) {
    const float p = ws[j];
    acc_a = __fadd_rn(acc_a, __fmul_rn(p, V[swz(j, lane >> 2) + (lane & 3)]));
    acc_b = __fadd_rn(acc_b, __fmul_rn(p, V[swz(j, 8 + (lane >> 2)) + (lane & 3)]));
  }
  ca = acc_a;
  cb = acc_b;
}

}  // namespace mtg
