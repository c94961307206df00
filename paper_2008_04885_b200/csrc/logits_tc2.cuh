// Persistent CTA-pair (tcgen05 cta_group::2) output projection for the fp32
// (3xTF32) executor: model.cpp:431-450 project_logits with the log-softmax /
// top-k partial epilogue of logits_tc.cuh.
//
// Why a pair: the fp32 projection streams hi+lo operands (8 B per element)
// and is bound by L2 -> SM traffic, not by the MMAs. A 128 x 128 tile on one
// SM reads 512 KB of A and 512 KB of B per tile. Two SMs of a TPC computing
// one 256 x 256 tile with cta_group::2 each load 128 rows of A and 128 rows
// of B (each SM's MMA operands are read by the pair), so every SM moves
// 1 MB per 128 x 256 outputs: a third less traffic per logit.
//
// Roles per CTA (cluster of 2, rank 0 = leader):
//   warp 0 lane 0: TMA producer for this CTA's halves (A rows m0 + 128 rank,
//     B rows n0 + 128 rank); completion bytes land on the LEADER's full
//     barrier (the leader expects both CTAs' bytes). A rows wholly past M are
//     not loaded, and a batch of <= 128 rows loads a box of that many rows
//     (GemmPlan::a_box); the stale rows' accumulators are masked, never stored.
//   warp 1 lane 0 of the leader: cta_group::2 MMAs (M = 256, N = 256) into
//     TMEM buffer i & 1; commits multicast to both CTAs' empty / tfull
//     barriers.
//   warps 2..9: epilogue of this CTA's 128 accumulator rows (identical
//     per-element arithmetic to logits_tc_kernel), then arrive on the
//     leader's tempty barrier.
#pragma once

#include <cstdint>
#include <cuda.h>

#include "detmath.cuh"
#include "gemm_tc.cuh"
#include "launch.cuh"
#include "ptx.cuh"

namespace mtg {

namespace pair2 {

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// Spin on an mbarrier phase; traps instead of hanging if it never completes.
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  for (uint32_t it = 0; !done; ++it) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (it > (1u << 26)) __trap();
  }
}

// TMA 2-D load whose completion bytes are counted on the leader CTA's
// barrier (`leader_bar`: shared::cluster address).
__device__ __forceinline__ void tma_load_2d_pair(void* smem_dst, const CUtensorMap* map,
                                                 uint32_t leader_bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// Arrive on the barrier at this smem offset in both CTAs of the pair once the
// issued MMAs complete.
__device__ __forceinline__ void commit_both(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}

__device__ __forceinline__ void arrive_remote(uint32_t cluster_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar)
               : "memory");
}

template <int kCols>
__device__ __forceinline__ void tmem_alloc2(uint32_t* smem_result) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(smem_result)),
               "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}

template <int kCols>
__device__ __forceinline__ void tmem_dealloc2(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols)
               : "memory");
}

}  // namespace pair2

// Launch: grid = 2 * pairs CTAs, cluster (2,1,1), 320 threads.
__global__ void __launch_bounds__(320, 1)
    logits_tc2_kernel(const __grid_constant__ CUtensorMap mapA,
                      const __grid_constant__ CUtensorMap mapB,
                      const __grid_constant__ CUtensorMap mapA2,
                      const __grid_constant__ CUtensorMap mapB2,
                      const __grid_constant__ CUtensorMap mapA64,
                      const __grid_constant__ CUtensorMap mapA2_64, int num_kb, int nst,
                      int n_tiles, GemmEpilogue ep) {
  constexpr int BN = 256;             // pair tile width (each CTA loads 128 B rows)
  constexpr int kKind = prec_mma_kind(kPrecTF32x3);
  constexpr int kKbElems = 32;        // fp32 elements per 128-byte slab
  constexpr int kHalfTile = 128 * 128;  // 128 rows x 128 B
  constexpr int kStageBytes = 4 * kHalfTile;  // A hi | B hi | A lo | B lo
  constexpr int kTmemCols = BN;
  constexpr int kHalf = BN / 2;       // columns per epilogue warp
  constexpr int kChunk = 32;
  constexpr int kSubs = kHalf / 32;

  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned, as an offset from the shared array (an integer round
  // trip of the pointer would turn every shared access generic: LD.E / ST.E).
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* staging = reinterpret_cast<float*>(smem + nst * kStageBytes);
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + nst * kStageBytes + kEpiStageBytes);
  uint64_t* empty_bar = full_bar + kMaxStages;
  uint64_t* tfull_bar = empty_bar + kMaxStages;  // [2]
  uint64_t* tempty_bar = tfull_bar + 2;          // [2] (leader's are used)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = pair2::cta_rank();
  const bool leader = rank == 0;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&mapA);
      tma_prefetch_desc(&mapB);
      tma_prefetch_desc(&mapA2);
      tma_prefetch_desc(&mapB2);
      tma_prefetch_desc(&mapA64);
      tma_prefetch_desc(&mapA2_64);
    }
    pair2::tmem_alloc2<2 * kTmemCols>(tmem_slot);
  } else if (warp == 1 && lane == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 2 * kEpiWarps);
    }
    fence_barrier_init();
  }
  tc_fence_before();
  cluster_sync_all();  // both CTAs' barriers initialised, TMEM allocated
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  pdl_wait();
  pdl_trigger();
  trace_begin(ep.tr);
  const int M = ep.d_M ? *ep.d_M : ep.M;
  const int m_pairs = (M + 255) / 256;
  const int total = m_pairs * n_tiles;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer (both CTAs) ----
      const uint32_t full0 = dsmem_map(smem_u32(full_bar), 0);
      const int a_bytes = ep.a_box * 128;  // one A box (GemmPlan::a_box rows)
      int g = 0;
      for (int t = pair; t < total; t += npairs) {
        const int mp = (t % m_pairs) * 256, n0 = (t / m_pairs) * BN;
        // A last pair tile of <= 128 live rows runs as an M = 128 pair MMA
        // (64 rows per CTA): half the MMA time of M = 256.
        const bool light = M - mp <= 128;
        const int arows = light ? 64 : 128;
        const int my_m0 = mp + arows * static_cast<int>(rank);
        const bool a_mine = my_m0 < M;
        const bool a_peer = mp + arows < M;  // the leader's A rows are always live
        const int a_bytes_t = light ? 64 * 128 : a_bytes;
        for (int kb = 0; kb < num_kb; ++kb, ++g) {
          const int s = g % nst;
          const uint32_t ph = (g / nst) & 1;
          if (g >= nst) pair2::wait(&empty_bar[s], ph ^ 1);
          uint8_t* st = smem + s * kStageBytes;
          if (leader)  // A hi+lo of each live half, B hi+lo of both halves
            mbar_arrive_expect_tx(&full_bar[s], 2 * (a_bytes_t * (a_peer ? 2 : 1) + 2 * kHalfTile));
          const uint32_t fb = full0 + s * 8;
          const int kx = kb * kKbElems;
          if (a_mine) {
            pair2::tma_load_2d_pair(st, light ? &mapA64 : &mapA, fb, kx, my_m0);
            pair2::tma_load_2d_pair(st + 2 * kHalfTile, light ? &mapA2_64 : &mapA2, fb, kx,
                                    my_m0);
          }
          pair2::tma_load_2d_pair(st + kHalfTile, &mapB, fb, kx, n0 + 128 * static_cast<int>(rank));
          pair2::tma_load_2d_pair(st + 3 * kHalfTile, &mapB2, fb, kx,
                                  n0 + 128 * static_cast<int>(rank));
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {  // ---- MMA issuer (leader only) ----
      constexpr uint32_t idesc256 = make_idesc(kKind, 256, BN);
      constexpr uint32_t idesc128 = make_idesc(kKind, 128, BN);
      int g = 0, i = 0;
      for (int t = pair; t < total; t += npairs, ++i) {
        const int buf = i & 1;
        const uint32_t idesc = (M - (t % m_pairs) * 256 <= 128) ? idesc128 : idesc256;
        if (i >= 2) pair2::wait(&tempty_bar[buf], ((i >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + buf * kTmemCols;
        for (int kb = 0; kb < num_kb; ++kb, ++g) {
          const int s = g % nst;
          const uint32_t ph = (g / nst) & 1;
          pair2::wait(&full_bar[s], ph);
          tc_fence_after();
          const uint32_t a_base = smem_u32(smem + s * kStageBytes);
          const uint32_t b_base = a_base + kHalfTile;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t ad = umma_desc_sw128(a_base + k * 32);
            const uint64_t bd = umma_desc_sw128(b_base + k * 32);
            const uint64_t ad_lo = umma_desc_sw128(a_base + 2 * kHalfTile + k * 32);
            const uint64_t bd_lo = umma_desc_sw128(a_base + 3 * kHalfTile + k * 32);
            pair2::mma_tf32(d, ad_lo, bd, idesc, (kb | k) != 0);
            pair2::mma_tf32(d, ad, bd_lo, idesc, 1u);
            pair2::mma_tf32(d, ad, bd, idesc, 1u);
          }
          pair2::commit_both(&empty_bar[s]);
        }
        pair2::commit_both(&tfull_bar[buf]);
      }
    }
  } else {
    // ---- epilogue (8 warps): warp w drains TMEM lanes 32*(w%4).., column
    // half (w-2)/4 of accumulator i & 1 (this CTA's 128 rows), then
    // releases it on the leader's tempty barrier ----
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    float* stage = staging + (warp - 2) * (32 * 33);
    const int N = ep.N;
    const long long ldc = ep.ldc;
    const uint32_t tempty0 = dsmem_map(smem_u32(tempty_bar), 0);
    int i = 0;
    for (int t = pair; t < total; t += npairs, ++i) {
      const int buf = i & 1;
      const int mp = (t % m_pairs) * 256;
      const int n0 = (t / m_pairs) * BN;
      // M = 256 tiles: lanes = this CTA's 128 rows, TMEM columns = the 256
      // output columns. M = 128 tiles (64 rows per CTA): lanes 0-63 hold
      // columns 0-127 and lanes 64-127 columns 128-255 of the same 64 rows.
      const bool light = M - mp <= 128;
      const int rbase = light ? mp + 64 * static_cast<int>(rank) + (q & 1) * 32
                              : mp + 128 * static_cast<int>(rank) + q * 32;
      const int cb = light ? (q >> 1) * 128 : 0;        // output column of TMEM column 0
      const int c_lo = light ? half * 64 : half * kHalf;  // this warp's TMEM columns
      const int c_hi = c_lo + (light ? 64 : kHalf);
      const int nrows = min(32, M - rbase);  // warp-uniform, may be <= 0
      float* const Cbase = ep.C + static_cast<long long>(rbase) * ldc;
      float sub_m[kSubs], sub_s[kSubs];
      int sub_a[kSubs];
      pair2::wait(&tfull_bar[buf], (i >> 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int c = c_lo; c < c_hi; c += kChunk) {
        uint32_t r[32];
        tmem_ld32(tmem + buf * kTmemCols + (static_cast<uint32_t>(q * 32) << 16) + c, r);
        tmem_ld_wait();
        if (nrows <= 0 || n0 + cb + c >= N) continue;  // warp-uniform
        if (nrows < 32 && lane >= nrows) {  // rows past M: stale or zero A rows
#pragma unroll
          for (int j = 0; j < kChunk; ++j) r[j] = 0u;
        }
        float v[kChunk];
#pragma unroll
        for (int j = 0; j < kChunk; ++j) v[j] = __uint_as_float(r[j]);
#pragma unroll
        for (int j = 0; j < kChunk; ++j) stage[lane * 33 + j] = v[j];
        // Slice max / first argmax (strict >), sequential sum of exp(x - max).
        const int col0 = n0 + cb + c;
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
        const float sum =
            det_sum_exp(stage + lane * 33, bi >= 0 ? nv : 0, best, bi >= 0 ? mn : 0.0f);
        const int k = (c - c_lo) / 32;
#pragma unroll
        for (int kk = 0; kk < kSubs; ++kk)
          if (kk == k) {
            sub_m[kk] = best;
            sub_s[kk] = sum;
            sub_a[kk] = bi;
          }
        __syncwarp();
        const int col = col0 + lane;
        if (col < N) {
          float* cp = Cbase + col;
#pragma unroll 8
          for (int rr = 0; rr < 32; ++rr)
            if (rr < nrows) cp[rr * ldc] = stage[rr * 33 + lane];
        }
        __syncwarp();
      }
      // Accumulator fully read: hand it back to the leader's MMA issuer.
      tc_fence_before();
      __syncwarp();
      if (lane == 0) pair2::arrive_remote(tempty0 + buf * 8);
      const int sub0 = (n0 + cb + c_lo) / 32;
      const int nsub = (N + 31) / 32;
      const int my_subs = (c_hi - c_lo) / 32;  // 4 (M = 256) or 2 (M = 128)
      if (lane < nrows && sub0 < nsub) {
        const long long o = static_cast<long long>(rbase + lane) * ep.part_ld + sub0;
        if (my_subs == 2) {
#pragma unroll
          for (int kk = 0; kk < 2; ++kk)
            if (sub0 + kk < nsub) {
              ep.part_m[o + kk] = sub_m[kk];
              ep.part_s[o + kk] = sub_s[kk];
              ep.part_arg[o + kk] = sub_a[kk];
            }
        } else if (sub0 + kSubs <= nsub) {
          *reinterpret_cast<float4*>(ep.part_m + o) =
              make_float4(sub_m[0], sub_m[1], sub_m[2], sub_m[3]);
          *reinterpret_cast<float4*>(ep.part_s + o) =
              make_float4(sub_s[0], sub_s[1], sub_s[2], sub_s[3]);
          *reinterpret_cast<int4*>(ep.part_arg + o) =
              make_int4(sub_a[0], sub_a[1], sub_a[2], sub_a[3]);
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

  // Both CTAs: every MMA has completed (the epilogues waited on the last
  // tfull) and no TMA is in flight (each stage filled was consumed).
  tc_fence_before();
  cluster_sync_all();
  if (warp == 0) {
    tc_fence_after();
    pair2::tmem_dealloc2<2 * kTmemCols>(tmem);
  }
  trace_end(ep.tr);
}

}  // namespace mtg
