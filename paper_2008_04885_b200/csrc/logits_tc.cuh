// Persistent tcgen05 output projection (model.cpp:431-472 project_logits) with
// the log-softmax / top-k partial epilogue of gemm_tc.cuh (kEpiSoftmaxParts).
//
// One CTA per SM walks the output tiles t = blockIdx.x, +gridDim.x, ...
// (m fastest, so concurrent CTAs share weight tiles in L2). The TMA producer
// streams K slabs through an nst-deep ring across tile boundaries; the MMA
// issuer accumulates tile i into TMEM buffer i & 1 (two BN-column
// accumulators), so the epilogue of tile i (TMEM drain, int8 scale, slice
// max / argmax / sum exp, coalesced logits store) overlaps the MMAs of tile
// i + 1. Arithmetic per element is identical to gemm_tc_kernel's.
#pragma once

#include <cstdint>
#include <cuda.h>

#include "detmath.cuh"
#include "gemm_tc.cuh"
#include "launch.cuh"
#include "ptx.cuh"

namespace mtg {

// EG epilogue groups of 8 warps: with EG = 2, group g drains the tiles that
// use accumulator g, doubling the epilogue issue rate (the int8 bottleneck).
template <int PREC, int BN, int EG>
__global__ void __launch_bounds__(64 + EG * 256, 1)
    logits_tc_kernel(const __grid_constant__ CUtensorMap mapA,
                     const __grid_constant__ CUtensorMap mapB,
                     const __grid_constant__ CUtensorMap mapA2,
                     const __grid_constant__ CUtensorMap mapB2, int num_kb, int nst, int n_tiles,
                     GemmEpilogue ep) {
  constexpr bool kSplit = (PREC == kPrecTF32x3);
  constexpr int kKind = prec_mma_kind(PREC);
  constexpr int kElem = prec_elem_bytes(PREC);
  constexpr int kKbElems = 128 / kElem;
  constexpr int kATile = 128 * 128;
  constexpr int kBTile = BN * 128;
  constexpr int kStageBytes = gemm_stage_bytes(PREC, BN);
  constexpr int kTmemCols = gemm_tmem_cols(BN);
  constexpr int kHalf = BN / 2;
  constexpr int kChunk = 32;
  constexpr int kSubs = kHalf / 32;
  static_assert(kHalf % 32 == 0, "logits tiles need >= 64 columns");
  static_assert(2 * kTmemCols <= 512, "two accumulators must fit in TMEM");

  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned, as an offset from the shared array (an integer round
  // trip of the pointer would turn every shared access generic: LD.E / ST.E).
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* staging = reinterpret_cast<float*>(smem + nst * kStageBytes);
  uint64_t* full_bar =
      reinterpret_cast<uint64_t*>(smem + nst * kStageBytes + EG * kEpiStageBytes);
  uint64_t* empty_bar = full_bar + kMaxStages;
  uint64_t* tfull_bar = empty_bar + kMaxStages;  // [2] accumulator ready
  uint64_t* tempty_bar = tfull_bar + 2;          // [2] accumulator drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

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
    tmem_alloc<2 * kTmemCols>(tmem_slot);
  } else if (warp == 1 && lane == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], kEpiWarps);
    }
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  pdl_wait();
  pdl_trigger();
  trace_begin(ep.tr);
  const int M = ep.d_M ? *ep.d_M : ep.M;
  const int m_live = (M + 127) / 128;
  const int total = m_live * n_tiles;

  const int load_bytes = (ep.a_box * 128 + kBTile) * (kSplit ? 2 : 1);
  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer: one ring across all tiles ----
      int g = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const int m0 = (t % m_live) * 128, n0 = (t / m_live) * BN;
        for (int kb = 0; kb < num_kb; ++kb, ++g) {
          const int s = g % nst;
          const uint32_t ph = (g / nst) & 1;
          if (g >= nst) mbar_wait(&empty_bar[s], ph ^ 1);
          uint8_t* st = smem + s * kStageBytes;
          mbar_arrive_expect_tx(&full_bar[s], load_bytes);
          tma_load_2d(st, &mapA, &full_bar[s], kb * kKbElems, m0);
          tma_load_2d(st + kATile, &mapB, &full_bar[s], kb * kKbElems, n0);
          if constexpr (kSplit) {
            tma_load_2d(st + kATile + kBTile, &mapA2, &full_bar[s], kb * kKbElems, m0);
            tma_load_2d(st + 2 * kATile + kBTile, &mapB2, &full_bar[s], kb * kKbElems, n0);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer: tile i -> accumulator i & 1 ----
      constexpr uint32_t idesc = make_idesc(kKind, 128, BN);
      int g = 0, i = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++i) {
        const int buf = i & 1;
        if (i >= 2) mbar_wait(&tempty_bar[buf], ((i >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + buf * kTmemCols;
        for (int kb = 0; kb < num_kb; ++kb, ++g) {
          const int s = g % nst;
          const uint32_t ph = (g / nst) & 1;
          mbar_wait(&full_bar[s], ph);
          tc_fence_after();
          const uint32_t a_base = smem_u32(smem + s * kStageBytes);
          const uint32_t b_base = a_base + kATile;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t ad = umma_desc_sw128(a_base + k * 32);
            const uint64_t bd = umma_desc_sw128(b_base + k * 32);
            if constexpr (kSplit) {
              const uint64_t ad_lo = umma_desc_sw128(a_base + kATile + kBTile + k * 32);
              const uint64_t bd_lo = umma_desc_sw128(a_base + 2 * kATile + kBTile + k * 32);
              tc_mma<kKind>(d, ad_lo, bd, idesc, (kb | k) != 0);
              tc_mma<kKind>(d, ad, bd_lo, idesc, 1u);
              tc_mma<kKind>(d, ad, bd, idesc, 1u);
            } else {
              tc_mma<kKind>(d, ad, bd, idesc, (kb | k) != 0);
            }
          }
          tc_commit(&empty_bar[s]);
        }
        tc_commit(&tfull_bar[buf]);
      }
    }
  } else {
    // ---- epilogue (8 warps): warp w drains TMEM lanes 32*(w%4).., column
    // half (w-2)/4, of accumulator i & 1, then releases it ----
    const int q = warp & 3;
    const int grp = (warp - 2) >> 3;  // epilogue group
    const int half = ((warp - 2) & 7) >> 2;
    float* stage = staging + (warp - 2) * (32 * 33);
    const int N = ep.N;
    const long long ldc = ep.ldc;
    int i = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++i) {
      const int buf = i & 1;
      if (EG == 2 && buf != grp) continue;  // the other group drains this tile
      const int m0 = (t % m_live) * 128, n0 = (t / m_live) * BN;
      const int rbase = m0 + q * 32;
      const int nrows = min(32, M - rbase);  // warp-uniform, may be <= 0
      float iv = 1.0f;
      if constexpr (PREC == kPrecI8) {
        const float sa = lane < nrows ? ep.a_scale[rbase + lane] : 1.0f;
        iv = __frcp_rn(__fmul_rn(sa, ep.w_seg_scale[0]));
      }
      float* const Cbase = ep.C + static_cast<long long>(rbase) * ldc;
      float sub_m[kSubs], sub_s[kSubs];
      int sub_a[kSubs];
      mbar_wait(&tfull_bar[buf], (i >> 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int c = half * kHalf; c < (half + 1) * kHalf; c += kChunk) {
        uint32_t r[32];
        tmem_ld32(tmem + buf * kTmemCols + (static_cast<uint32_t>(q * 32) << 16) + c, r);
        tmem_ld_wait();
        if (nrows <= 0 || n0 + c >= N) continue;  // warp-uniform
        if (nrows < 32 && lane >= nrows) {  // rows past M: stale A rows (GemmPlan::a_box)
#pragma unroll
          for (int j = 0; j < kChunk; ++j) r[j] = 0u;
        }
        float v[kChunk];
#pragma unroll
        for (int j = 0; j < kChunk; ++j)
          v[j] = PREC == kPrecI8 ? __fmul_rn(__int2float_rn(static_cast<int>(r[j])), iv)
                                 : __uint_as_float(r[j]);
#pragma unroll
        for (int j = 0; j < kChunk; ++j) stage[lane * 33 + j] = v[j];
        // Slice max / first argmax (strict >), sequential sum of exp(x - max).
        const int col0 = n0 + c;
        const int nv = min(kChunk, N - col0);
        float best = -__int_as_float(0x7f800000);
        float mn = __int_as_float(0x7f800000);
        int bi = -1;
#pragma unroll
        for (int j = 0; j < kChunk; ++j) {
          const bool take = j < nv && v[j] > best;
          best = take ? v[j] : best;
          bi = take ? col0 + j : bi;
          mn = j < nv ? fminf(mn, v[j]) : mn;
        }
        // all-NaN / all -inf slices: (best, sum, argmax) = (-inf, 0, -1)
        const float sum =
            det_sum_exp(stage + lane * 33, bi >= 0 ? nv : 0, best, bi >= 0 ? mn : 0.0f);
        const int k = (c - half * kHalf) / 32;
#pragma unroll
        for (int kk = 0; kk < kSubs; ++kk)
          if (kk == k) {
            sub_m[kk] = best;
            sub_s[kk] = sum;
            sub_a[kk] = bi;
          }
        __syncwarp();
        const int col = n0 + c + lane;
        if (col < N) {
          float* cp = Cbase + col;
#pragma unroll 8
          for (int rr = 0; rr < 32; ++rr)
            if (rr < nrows) cp[rr * ldc] = stage[rr * 33 + lane];
        }
        __syncwarp();
      }
      // Accumulator fully read: hand it back to the MMA issuer.
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar[buf]);
      // Partials of row rbase+lane, slices sub0 .. sub0+kSubs-1.
      const int sub0 = (n0 + half * kHalf) / 32;
      const int nsub = (N + 31) / 32;
      if (lane < nrows && sub0 < nsub) {
        const long long o = static_cast<long long>(rbase + lane) * ep.part_ld + sub0;
        if (sub0 + kSubs <= nsub && kSubs == 4) {
          *reinterpret_cast<float4*>(ep.part_m + o) =
              make_float4(sub_m[0], sub_m[1 % kSubs], sub_m[2 % kSubs], sub_m[3 % kSubs]);
          *reinterpret_cast<float4*>(ep.part_s + o) =
              make_float4(sub_s[0], sub_s[1 % kSubs], sub_s[2 % kSubs], sub_s[3 % kSubs]);
          *reinterpret_cast<int4*>(ep.part_arg + o) =
              make_int4(sub_a[0], sub_a[1 % kSubs], sub_a[2 % kSubs], sub_a[3 % kSubs]);
        } else {
#pragma unroll
          for (int kk = 0; kk < kSubs; ++kk)
            if (sub0 + kk < nsub) {
              ep.part_m[o + kk] = sub_m[kk];
              ep.part_s[o + kk] = sub_s[kk];
              ep.part_arg[o + kk] = sub_a[kk];
            }
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<2 * kTmemCols>(tmem);
  }
  trace_end(ep.tr);
}

}  // namespace mtg
