// Host-side planning/launch of the tcgen05 GEMM (gemm_tc.cuh).
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "gemm_tc.cuh"

namespace mtg {

// Pads K so every operand row is a whole number of 128-byte TMA/UMMA slabs.
inline int pad_k(int k, int prec) {
  const int per = 128 / prec_elem_bytes(prec);
  return k <= 0 ? per : (k + per - 1) / per * per;
}

// A K-major device matrix [rows x k_pad] in the precision's operand format
// (int8, bf16, or fp32 hi with a separate fp32 lo part for TF32x3).
struct Operand {
  const void* ptr = nullptr;
  const void* ptr_lo = nullptr;  // TF32x3 only
  int rows = 0;                  // allocated rows (TMA bound)
  int k_pad = 0;
  int prec = kPrecI8;
};

struct GemmPlan {
  CUtensorMap a, b, a2, b2;
  CUtensorMap at, at2;  // CTA-pair projection: 64-row A boxes (M = 128 pair tiles)
  int prec = 0;
  int bn = 0;
  int num_kb = 0;
  int m_tiles = 0;
  int n_tiles = 0;
  int nst = 0;     // pipeline stages
  int smem = 0;    // dynamic shared memory bytes
  int splits = 1;  // split-K factor (grid.z)
  bool persistent = false;  // output projection: logits_tc_kernel
  bool pair = false;        // ... as CTA pairs (logits_tc2_kernel, TF32x3)
  // Rows of the A tile fetched by TMA: m_max rounded up to 8 when one m tile
  // covers all rows (decoding at small batch), else 128. The MMA still reads
  // 128 rows; the rows beyond the box hold stale shared memory whose
  // accumulator rows the epilogue masks and never stores.
  int a_box = 128;
};


// Plans C[M x N] = A[M x K] . B[N x K]^T for at most m_max rows of A.
// min_bn: smallest tile width the planner may pick (the softmax-partials
// epilogue needs >= 128).
// allow_split: pick a split-K factor when the tile grid cannot fill the GPU.
GemmPlan plan_gemm(const Operand& a, const Operand& b, int m_max, int n,
                   int force_bn = 0, int min_bn = 32, bool allow_split = false);
// Output projection with softmax partials (logits_tc.cuh): persistent CTAs,
// double-buffered TMEM accumulators. Launch with launch_gemm.
GemmPlan plan_logits(const Operand& a, const Operand& b, int m_max, int n);
// TF32x3 projection on CTA pairs (cta_group::2, 256 x 256 tiles; logits_tc2.cuh).
GemmPlan plan_logits_pair(const Operand& a, const Operand& b, int m_max, int n);
void launch_gemm(const GemmPlan& plan, const GemmEpilogue& ep, cudaStream_t stream);

}  // namespace mtg
