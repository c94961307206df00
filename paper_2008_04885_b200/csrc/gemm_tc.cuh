// tcgen05 GEMM for sm_100a: C[M x N] = epilogue(A[M x K] . B[N x K]^T).
//
// Both operands are K-major (row-major with K contiguous), staged by TMA with
// 128-byte swizzle, one 128-byte K slab per pipeline stage. A single thread
// issues tcgen05.mma into a TMEM accumulator (M = 128 lanes x BN columns); four
// epilogue warps drain TMEM with tcgen05.ld and apply the fused epilogue of the
// reference's linear layers:
//
//   int8  (quant.cpp:155-193, model.cpp:461-466):
//         v = float(acc_s32) * (1.0f / (sa[row] * sw[col]))
//   bf16 / fp32 (model.cpp:422-429): v = acc_f32
//   then  v += bias[col] (add_rowvec, tensor.cpp:240-263)
//         v = max(v, 0)  (relu, tensor.cpp:314-329)
//         v = res + v    (residual add, tensor.cpp:220-238; model.cpp:592-593)
//
// The fp32 path ("TF32x3") splits each fp32 operand into hi + lo tf32 parts
// and accumulates A_lo.B_hi + A_hi.B_lo + A_hi.B_hi in fp32 TMEM, giving ~fp32
// accuracy on the tensor pipe.
//
// Warp roles (192 threads): warp 0 = TMEM allocator + TMA producer, warp 1 =
// MMA issuer, warps 2..5 = epilogue (warp w drains TMEM lanes 32*(w%4)..+31).
#pragma once

#include <cstdint>
#include <cuda.h>

#include "ptx.cuh"

namespace mtg {

struct GemmEpilogue {
  float* C;                  // output base
  long long ldc;             // row pitch of C (elements)
  long long c_step_stride;   // C += (*d_step) * c_step_stride when d_step != null
  const int* d_step;
  const float* bias;         // [N] or null
  const float* residual;     // [M x ldr] or null (may alias C)
  long long ldr;
  const float* a_scale;      // int8: per-row activation scale
  const float* w_scale;      // int8: per-column weight scale
  int relu;
  int M;                     // rows, unless d_M != null
  const int* d_M;
  int N;
  int vec;                   // 1: C/residual rows are 16-byte aligned (float4 path)
};

enum GemmPrec : int { kPrecI8 = 0, kPrecBF16 = 1, kPrecTF32x3 = 2 };

__host__ __device__ constexpr int prec_elem_bytes(int prec) {
  return prec == kPrecI8 ? 1 : prec == kPrecBF16 ? 2 : 4;
}
__host__ __device__ constexpr int prec_mma_kind(int prec) {
  return prec == kPrecI8 ? kKindI8 : prec == kPrecBF16 ? kKindF16 : kKindTF32;
}
__host__ __device__ constexpr int gemm_stage_bytes(int prec, int bn) {
  return (128 * 128 + bn * 128) * (prec == kPrecTF32x3 ? 2 : 1);
}
__host__ __device__ constexpr int gemm_stages(int prec, int bn) {
  return (200 * 1024 / gemm_stage_bytes(prec, bn)) > 8
             ? 8
             : (200 * 1024 / gemm_stage_bytes(prec, bn));
}
__host__ __device__ constexpr int gemm_tmem_cols(int bn) {
  return bn <= 32 ? 32 : bn <= 64 ? 64 : bn <= 128 ? 128 : 256;
}
__host__ __device__ constexpr int gemm_smem_bytes(int prec, int bn) {
  return gemm_stages(prec, bn) * gemm_stage_bytes(prec, bn) + 1024 /*align*/ +
         256 /*barriers*/;
}

constexpr int kGemmThreads = 192;

template <int PREC, int BN>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap mapA,
                   const __grid_constant__ CUtensorMap mapB,
                   const __grid_constant__ CUtensorMap mapA2,
                   const __grid_constant__ CUtensorMap mapB2, int num_kb,
                   GemmEpilogue ep) {
  constexpr bool kSplit = (PREC == kPrecTF32x3);
  constexpr int kKind = prec_mma_kind(PREC);
  constexpr int kElem = prec_elem_bytes(PREC);
  constexpr int kKbElems = 128 / kElem;      // K elements per 128-byte slab
  constexpr int kStages = gemm_stages(PREC, BN);
  constexpr int kATile = 128 * 128;
  constexpr int kBTile = BN * 128;
  constexpr int kStageBytes = gemm_stage_bytes(PREC, BN);
  constexpr int kTmemCols = gemm_tmem_cols(BN);

  const int M = ep.d_M ? *ep.d_M : ep.M;
  const int m0 = blockIdx.y * 128;
  if (m0 >= M) return;  // uniform across the CTA
  const int n0 = blockIdx.x * BN;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty_bar = full_bar + kStages;
  uint64_t* accum_bar = empty_bar + kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum_bar + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&mapA);
      tma_prefetch_desc(&mapB);
      if constexpr (kSplit) {
        tma_prefetch_desc(&mapA2);
        tma_prefetch_desc(&mapB2);
      }
    }
    tmem_alloc<kTmemCols>(tmem_slot);
  } else if (warp == 1 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(accum_bar, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer ----
      for (int kb = 0; kb < num_kb; ++kb) {
        const int s = kb % kStages;
        const uint32_t ph = (kb / kStages) & 1;
        if (kb >= kStages) mbar_wait(&empty_bar[s], ph ^ 1);
        uint8_t* st = smem + s * kStageBytes;
        mbar_arrive_expect_tx(&full_bar[s], kStageBytes);
        tma_load_2d(st, &mapA, &full_bar[s], kb * kKbElems, m0);
        tma_load_2d(st + kATile, &mapB, &full_bar[s], kb * kKbElems, n0);
        if constexpr (kSplit) {
          tma_load_2d(st + kATile + kBTile, &mapA2, &full_bar[s], kb * kKbElems, m0);
          tma_load_2d(st + 2 * kATile + kBTile, &mapB2, &full_bar[s], kb * kKbElems,
                      n0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---- MMA issuer ----
      constexpr uint32_t idesc = make_idesc(kKind, 128, BN);
      for (int kb = 0; kb < num_kb; ++kb) {
        const int s = kb % kStages;
        const uint32_t ph = (kb / kStages) & 1;
        mbar_wait(&full_bar[s], ph);
        tc_fence_after();
        const uint32_t a_base = smem_u32(smem + s * kStageBytes);
        const uint32_t b_base = a_base + kATile;
#pragma unroll
        for (int k = 0; k < 4; ++k) {  // 4 x 32-byte MMA K steps per slab
          const uint64_t ad = umma_desc_sw128(a_base + k * 32);
          const uint64_t bd = umma_desc_sw128(b_base + k * 32);
          if constexpr (kSplit) {
            const uint64_t ad_lo = umma_desc_sw128(a_base + kATile + kBTile + k * 32);
            const uint64_t bd_lo =
                umma_desc_sw128(a_base + 2 * kATile + kBTile + k * 32);
            tc_mma<kKind>(tmem, ad_lo, bd, idesc, (kb | k) != 0);
            tc_mma<kKind>(tmem, ad, bd_lo, idesc, 1u);
            tc_mma<kKind>(tmem, ad, bd, idesc, 1u);
          } else {
            tc_mma<kKind>(tmem, ad, bd, idesc, (kb | k) != 0);
          }
        }
        tc_commit(&empty_bar[s]);  // slot reusable once these MMAs retire
      }
      tc_commit(accum_bar);        // accumulator complete
    }
  } else {
    // ---- epilogue: TMEM -> registers -> fused ops -> global ----
    const int q = warp & 3;
    const int row = m0 + q * 32 + lane;
    const bool row_ok = row < M;
    mbar_wait(accum_bar, 0);
    tc_fence_after();

    float* crow = ep.C + (ep.d_step ? static_cast<long long>(*ep.d_step) * ep.c_step_stride
                                    : 0LL) +
                  static_cast<long long>(row) * ep.ldc;
    const float* rrow =
        ep.residual ? ep.residual + static_cast<long long>(row) * ep.ldr : nullptr;
    float sa = 1.0f;
    if constexpr (PREC == kPrecI8) sa = row_ok ? ep.a_scale[row] : 1.0f;

#pragma unroll 1
    for (int c = 0; c < BN; c += 16) {
      uint32_t r[16];
      tmem_ld16(tmem + (static_cast<uint32_t>(q * 32) << 16) + c, r);
      tmem_ld_wait();
      const int col0 = n0 + c;
      if (!row_ok || col0 >= ep.N) continue;
      float v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if constexpr (PREC == kPrecI8) {
          const int col = min(col0 + j, ep.N - 1);
          const float inv = 1.0f / (sa * ep.w_scale[col]);
          v[j] = __int2float_rn(static_cast<int>(r[j])) * inv;
        } else {
          v[j] = __uint_as_float(r[j]);
        }
      }
      const bool full = ep.vec && (col0 + 16 <= ep.N);
      if (ep.bias) {
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (full || col0 + j < ep.N) v[j] = v[j] + ep.bias[col0 + j];
      }
      if (ep.relu) {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = v[j] > 0.0f ? v[j] : 0.0f;
      }
      if (rrow) {
        if (full) {
#pragma unroll
          for (int j = 0; j < 16; j += 4) {
            const float4 t = *reinterpret_cast<const float4*>(rrow + col0 + j);
            v[j] = t.x + v[j];
            v[j + 1] = t.y + v[j + 1];
            v[j + 2] = t.z + v[j + 2];
            v[j + 3] = t.w + v[j + 3];
          }
        } else {
          for (int j = 0; j < 16; ++j)
            if (col0 + j < ep.N) v[j] = rrow[col0 + j] + v[j];
        }
      }
      if (full) {
#pragma unroll
        for (int j = 0; j < 16; j += 4)
          *reinterpret_cast<float4*>(crow + col0 + j) =
              make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      } else {
        for (int j = 0; j < 16; ++j)
          if (col0 + j < ep.N) crow[col0 + j] = v[j];
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
}

}  // namespace mtg
