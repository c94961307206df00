// tcgen05 GEMM for sm_100a: C[M x N] = epilogue(A[M x K] . B[N x K]^T).
//
// Both operands are K-major (row-major with K contiguous), staged by TMA with
// 128-byte swizzle, one 128-byte K slab per pipeline stage. A single thread
// issues tcgen05.mma into a TMEM accumulator (M = 128 lanes x BN columns);
// eight epilogue warps drain TMEM with tcgen05.ld and apply the fused
// epilogue of the reference's linear layers:
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
// Warp roles (320 threads): warp 0 = TMEM allocator + TMA producer, warp 1 =
// MMA issuer, warps 2..9 = epilogue (warp w drains TMEM lanes 32*(w%4)..+31,
// column half (w-2)/4). The pipeline depth is a launch parameter so small-K
// GEMMs run two CTAs per SM (one CTA's epilogue overlaps the other's MMAs).
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>

#include "detmath.cuh"
#include "launch.cuh"
#include "ptx.cuh"

namespace mtg {

struct GemmEpilogue {
  int a_box;                 // A rows per TMA box (GemmPlan::a_box; set by launch_gemm)
  float* C;                  // output base
  long long ldc;             // row pitch of C (elements)
  long long c_step_stride;   // C += (*d_step) * c_step_stride when d_step != null
  const int* d_step;
  const float* bias;         // [N] or null
  const float* residual;     // [M x ldr] or null (may alias C)
  long long ldr;
  const float* a_scale;      // int8: per-row activation scale
  const float* w_seg_scale;  // int8: weight scale per column segment
  int seg_width;             // columns per weight segment (fused q|k|v)
  int relu;
  int M;                     // rows, unless d_M != null
  const int* d_M;
  int N;
  // Output-projection mode (EPI = 1, see kEpiSoftmaxParts): per 32-column
  // slice of each row, its max, first argmax column and sum of exp(x - max).
  float* part_m;             // [M x part_ld]
  float* part_s;
  int* part_arg;
  long long part_ld;
  // Per-segment max |output| (float bits, atomicMax) for a following int8
  // quantize with one scale per sentence; bias and ReLU then apply in the
  // row-per-thread phase. Segment of row r: row_seg[r].
  unsigned* seg_absmax;
  const int* row_seg;
  int* nonfinite;
  // Optional: write the output as a TF32x3 operand, C = tf32(y), C_lo = y - C
  // (the next GEMM's A), instead of plain y.
  float* C_lo;
  // Optional: write the output as a bf16 operand (C then points at the bf16
  // buffer, reinterpreted; element offsets as for fp32).
  int bf16_out;
  KTrace tr;  // MTG_TRACE timeline slot
  int split_dist;  // split-K sums by all epilogue threads (1) or per owner warp (0)
};

// Stores y at C[off] (or its tf32 hi / lo split for the kEpiTf32Out
// epilogue, or its bf16 rounding for kEpiBf16Out: C0 is the buffer base, the
// element index is (C - C0) + off).
template <int EPIK>
__device__ __forceinline__ void gemm_store(float* C, float* C_lo, long long off, float y,
                                           float* C0) {
  if constexpr (EPIK == 3) {  // kEpiTf32Out
    uint32_t hb;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(y));
    C[off] = __uint_as_float(hb);
    C_lo[off] = __fsub_rn(y, __uint_as_float(hb));
  } else if constexpr (EPIK == 4) {  // kEpiBf16Out
    reinterpret_cast<__nv_bfloat16*>(C0)[(C - C0) + off] = __float2bfloat16_rn(y);
  } else {
    C[off] = y;
  }
}

// EPI = 0: linear-layer epilogue. EPI = 1: output projection; also emits the
// log-softmax / top-k partials (no bias, relu or residual).
constexpr int kEpiLinear = 0;
constexpr int kEpiSoftmaxParts = 1;
constexpr int kEpiSegMax = 2;  // linear + per-segment max |y| (bias/ReLU in phase 1)
constexpr int kEpiTf32Out = 3;  // linear, output written as a TF32x3 operand (hi + lo)
constexpr int kEpiBf16Out = 4;  // linear, output written as a bf16 operand

// kPrecTF32x3A: TF32x3 whose A operand arrives as plain fp32 and is split
// into hi + lo inside the kernel (half the activation bytes); B as kPrecTF32x3.
enum GemmPrec : int { kPrecI8 = 0, kPrecBF16 = 1, kPrecTF32x3 = 2, kPrecTF32x3A = 3 };
__host__ __device__ constexpr bool prec_is_tf32x3(int prec) {
  return prec == kPrecTF32x3 || prec == kPrecTF32x3A;
}

constexpr int kMaxSegments = 4;
constexpr int kMaxStages = 8;
constexpr int kMaxSplits = 8;  // split-K cluster size (portable cluster limit)
constexpr int kGemmThreads = 320;
constexpr int kEpiWarps = 8;

__host__ __device__ constexpr int prec_elem_bytes(int prec) {
  return prec == kPrecI8 ? 1 : prec == kPrecBF16 ? 2 : 4;
}
__host__ __device__ constexpr int prec_mma_kind(int prec) {
  return prec == kPrecI8 ? kKindI8 : prec == kPrecBF16 ? kKindF16 : kKindTF32;
}
__host__ __device__ constexpr int gemm_stage_bytes(int prec, int bn) {
  return (128 * 128 + bn * 128) * (prec_is_tf32x3(prec) ? 2 : 1);
}
__host__ __device__ constexpr int gemm_tmem_cols(int bn) {
  return bn <= 32 ? 32 : bn <= 64 ? 64 : bn <= 128 ? 128 : 256;
}
constexpr int kGemmSmemExtra = 1024 /*align*/ + 256 /*barriers*/;
constexpr int kEpiStageBytes = kEpiWarps * 32 * 33 * 4;  // aliases the drained pipeline

// FL >= 0 fixes the epilogue options at compile time (bit 0 bias, 1 ReLU,
// 2 residual, 3 step offset) -- the hot small GEMMs measure faster with no
// runtime option checks; FL = -1 reads them from the GemmEpilogue.
template <int PREC, int BN, int EPI, int FL = -1>
__global__ void __launch_bounds__(kGemmThreads, 2)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap mapA,
                   const __grid_constant__ CUtensorMap mapB,
                   const __grid_constant__ CUtensorMap mapA2,
                   const __grid_constant__ CUtensorMap mapB2, int num_kb, int nst,
                   GemmEpilogue ep) {
  constexpr bool kSplit = prec_is_tf32x3(PREC);
  constexpr bool kSplitA = (PREC == kPrecTF32x3A);  // A split by the epilogue warps
  constexpr int kKind = prec_mma_kind(PREC);
  constexpr int kElem = prec_elem_bytes(PREC);
  constexpr int kKbElems = 128 / kElem;      // K elements per 128-byte slab
  constexpr int kATile = 128 * 128;
  constexpr int kBTile = BN * 128;
  constexpr int kStageBytes = gemm_stage_bytes(PREC, BN);
  constexpr int kTmemCols = gemm_tmem_cols(BN);
  constexpr int kHalf = BN / 2;                   // columns per epilogue warp
  constexpr int kChunk = kHalf >= 32 ? 32 : 16;  // columns per TMEM load

  const int m0 = blockIdx.y * 128;
  const int n0 = blockIdx.x * BN;
  // Split-K: this CTA's contiguous range of 128-byte K slabs.
  const int splits = gridDim.z, z = blockIdx.z;
  const int kb_begin = z * (num_kb / splits) + min(z, num_kb % splits);
  const int kb_count = num_kb / splits + (z < num_kb % splits ? 1 : 0);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + nst * kStageBytes);
  uint64_t* empty_bar = full_bar + kMaxStages;
  uint64_t* accum_bar = empty_bar + kMaxStages;
  uint64_t* conv_bar = accum_bar + 1;  // [kMaxStages] A split done (kSplitA)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(conv_bar + kMaxStages);

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
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
      mbar_init(&conv_bar[s], kEpiWarps);
    }
    mbar_init(accum_bar, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // Weights (B) do not depend on the previous kernel: the producer starts
  // their first stages before the programmatic-dependency wait, so the weight
  // fetch overlaps the predecessor's tail. Everything that reads predecessor
  // outputs (A operand, row count, scales, residual) comes after pdl_wait.
  const int kABytes = ep.a_box * 128 * (kSplit && !kSplitA ? 2 : 1);  // A bytes loaded by TMA
  constexpr int kBBytes = kBTile * (kSplit ? 2 : 1);
  const int kLoadBytes = kABytes + kBBytes;
  const int npre = min(nst, kb_count);
  if (warp == 0 && lane == 0) {
    for (int kb = 0; kb < npre; ++kb) {
      uint8_t* st = smem + kb * kStageBytes;
      const int kx = (kb_begin + kb) * kKbElems;
      mbar_expect_tx(&full_bar[kb], kBBytes);
      tma_load_2d(st + kATile, &mapB, &full_bar[kb], kx, n0);
      if constexpr (kSplit) tma_load_2d(st + 2 * kATile + kBTile, &mapB2, &full_bar[kb], kx, n0);
    }
  }
  pdl_wait();
  pdl_trigger();
  trace_begin(ep.tr);
  if (threadIdx.x == 0) trace_phase(ep.tr, 0);
  const int M = ep.d_M ? *ep.d_M : ep.M;
  if (m0 >= M) {  // uniform across the CTA
    if (warp == 0 && lane == 0) {  // let the prefetched weight stages land first
      for (int kb = 0; kb < npre; ++kb) {
        mbar_arrive(&full_bar[kb]);
        mbar_wait(&full_bar[kb], 0);
      }
    }
    __syncwarp();
    if (warp == 0) tmem_dealloc<kTmemCols>(tmem);
    return;
  }

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer ----
      for (int kb = 0; kb < kb_count; ++kb) {
        const int s = kb % nst;
        const uint32_t ph = (kb / nst) & 1;
        const int kx = (kb_begin + kb) * kKbElems;
        uint8_t* st = smem + s * kStageBytes;
        if (kb < npre) {  // B already in flight
          mbar_arrive_expect_tx(&full_bar[s], kABytes);
          tma_load_2d(st, &mapA, &full_bar[s], kx, m0);
          if constexpr (kSplit && !kSplitA)
            tma_load_2d(st + kATile + kBTile, &mapA2, &full_bar[s], kx, m0);
          continue;
        }
        mbar_wait(&empty_bar[s], ph ^ 1);
        mbar_arrive_expect_tx(&full_bar[s], kLoadBytes);
        tma_load_2d(st, &mapA, &full_bar[s], kx, m0);
        tma_load_2d(st + kATile, &mapB, &full_bar[s], kx, n0);
        if constexpr (kSplit) {
          if constexpr (!kSplitA) tma_load_2d(st + kATile + kBTile, &mapA2, &full_bar[s], kx, m0);
          tma_load_2d(st + 2 * kATile + kBTile, &mapB2, &full_bar[s], kx, n0);
        }
      }
    }
    __syncwarp();
    if (splits > 1) {  // split-K cluster barriers (1) and (2), see the epilogue
      cluster_sync_all();
      cluster_sync_all();
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---- MMA issuer ----
      constexpr uint32_t idesc = make_idesc(kKind, 128, BN);
      for (int kb = 0; kb < kb_count; ++kb) {
        const int s = kb % nst;
        const uint32_t ph = (kb / nst) & 1;
        mbar_wait(kSplitA ? &conv_bar[s] : &full_bar[s], ph);
        tc_fence_after();
        if (kb == 0) trace_phase(ep.tr, 1);
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
      trace_phase(ep.tr, 2);
    }
    __syncwarp();
    if (splits > 1) {
      cluster_sync_all();
      cluster_sync_all();
    }
  } else {
    if constexpr (kSplitA) {
      // ---- A split: the epilogue warps turn each landed fp32 A slab into
      // tf32 hi (in place) + lo (the A-lo slot) while the MMAs run ----
      const int t = threadIdx.x - 64;  // 0..255
      for (int kb = 0; kb < kb_count; ++kb) {
        const int s = kb % nst;
        mbar_wait(&full_bar[s], (kb / nst) & 1);
        float* a = reinterpret_cast<float*>(smem + s * kStageBytes);
        float* alo = reinterpret_cast<float*>(smem + s * kStageBytes + kATile + kBTile);
#pragma unroll
        for (int i = 4 * t; i < kATile / 4; i += 4 * 256) {
          float4 v = *reinterpret_cast<const float4*>(a + i);
          float4 h;
          asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(*reinterpret_cast<uint32_t*>(&h.x)) : "f"(v.x));
          asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(*reinterpret_cast<uint32_t*>(&h.y)) : "f"(v.y));
          asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(*reinterpret_cast<uint32_t*>(&h.z)) : "f"(v.z));
          asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(*reinterpret_cast<uint32_t*>(&h.w)) : "f"(v.w));
          *reinterpret_cast<float4*>(a + i) = h;
          *reinterpret_cast<float4*>(alo + i) =
              make_float4(__fsub_rn(v.x, h.x), __fsub_rn(v.y, h.y), __fsub_rn(v.z, h.z),
                          __fsub_rn(v.w, h.w));
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv_bar[s]);
      }
    }
    // ---- epilogue: TMEM -> registers -> smem transpose -> coalesced global ----
    // Phase 1 (thread = row): convert a 32 x kChunk accumulator sub-tile
    // (int8: x 1/(sa*sw), reciprocal hoisted per weight segment) into padded
    // smem. Phase 2 (lane = column): bias / relu / residual and 128-byte
    // coalesced row stores. The staging area aliases pipeline stage memory,
    // which is drained once the accumulator barrier fires.
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    float* stage = reinterpret_cast<float*>(smem) + (warp - 2) * (32 * 33);
    const int rbase = m0 + q * 32;
    // Split-K: the 8 (row quarter, column half) regions of the tile are
    // reduced and stored by different splits of the cluster (region r by
    // split r % splits), spreading the DSMEM reads over the SMs.
    const bool owner = splits <= 1 || ((q * 2 + half) % splits) == z;
    int nrows = owner ? min(32, M - rbase) : 0;  // warp-uniform, may be <= 0
    float inv[kMaxSegments];
    if constexpr (PREC == kPrecI8) {
      const float sa = lane < nrows ? ep.a_scale[rbase + lane] : 1.0f;
#pragma unroll
      for (int s = 0; s < kMaxSegments; ++s) {
        const int c0 = s * ep.seg_width;
        inv[s] = c0 < ep.N ? __frcp_rn(__fmul_rn(sa, ep.w_seg_scale[s])) : 1.0f;
      }
    }
    const bool has_step = FL >= 0 ? (FL & 8) != 0 : ep.d_step != nullptr;
    const long long step_off =
        has_step ? static_cast<long long>(*ep.d_step) * ep.c_step_stride : 0LL;
    const bool has_bias = FL >= 0 ? (FL & 1) != 0 : ep.bias != nullptr;
    const bool has_res = FL >= 0 ? (FL & 4) != 0 : ep.residual != nullptr;
    const bool relu = FL >= 0 ? (FL & 2) != 0 : ep.relu != 0;
    constexpr bool seg_mode = EPI == kEpiSegMax;  // host: no residual
    float seg_max = 0.0f;
    int seg_bad = 0;
    const int N = ep.N;
    const long long ldc = ep.ldc, ldr = ep.ldr;
    float* const Cbase = ep.C + step_off + static_cast<long long>(rbase) * ldc;
    // BN = 32 (the N = d_model residual GEMMs) and the BN = 64 FFN-down
    // (compile-time bias + residual): each epilogue warp owns one 32-row x
    // BN/2-column chunk, so its residual and bias are fetched while the MMAs
    // are still running (after the accumulator wait they cost a dependent L2
    // round trip per 8 rows; without a residual, BN = 64 measured slower).
    constexpr bool kPrefetch =
        EPI != kEpiSoftmaxParts && (BN == 32 || (BN == 64 && FL >= 0 && (FL & 4) != 0));
    float res_pre[kPrefetch ? 32 : 1];
    float bias_pre = 0.0f;
    if constexpr (kPrefetch) {
      const int col = n0 + half * kHalf + (lane % kChunk);
      const bool col_ok = col < N && lane < kChunk;
#pragma unroll
      for (int i = 0; i < 32; ++i)
        res_pre[i] = (has_res && col_ok && i < nrows)
                         ? ep.residual[static_cast<long long>(rbase + i) * ldr + col]
                         : 0.0f;
      if (has_bias && col_ok) bias_pre = ep.bias[col];
    }
    // Softmax partials of this thread's row over its kHalf columns.
    constexpr int kSubs = EPI == kEpiSoftmaxParts ? kHalf / 32 : 1;
    float sub_m[kSubs], sub_s[kSubs];
    int sub_a[kSubs];
    mbar_wait(accum_bar, 0);
    tc_fence_after();
    if (warp == 2 && lane == 0) trace_phase(ep.tr, 3);
    // Split-K over a thread-block cluster along z: every split parks its raw
    // accumulator tile in its own (drained) shared memory; each region of the
    // tile has an owner split, whose 256 epilogue threads read the region's
    // partials from all splits through DSMEM (one float4 per thread and
    // split, all loads in flight together), sum them in z order (int32 exact,
    // float ordered) into the owner's own parked copy, and then run the
    // epilogue for it. Two cluster barriers bracket the remote reads.
    constexpr int kPartPitch = BN + 4;  // words; conflict-free row-per-thread float4
    uint32_t* part = reinterpret_cast<uint32_t*>(smem + kEpiStageBytes);
    const uint32_t* my_part_row = part + (q * 32 + lane) * kPartPitch;
    if (splits > 1) {
#pragma unroll 1
      for (int c = half * kHalf; c < (half + 1) * kHalf; c += kChunk) {
        uint32_t r[32];
        if constexpr (kChunk == 32) {
          tmem_ld32(tmem + (static_cast<uint32_t>(q * 32) << 16) + c, r);
        } else {
          tmem_ld16(tmem + (static_cast<uint32_t>(q * 32) << 16) + c,
                    *reinterpret_cast<uint32_t(*)[16]>(r));
        }
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < kChunk; j += 4)
          *reinterpret_cast<uint4*>(part + (q * 32 + lane) * kPartPitch + c + j) =
              make_uint4(r[j], r[j + 1], r[j + 2], r[j + 3]);
      }
      cluster_sync_all();  // (1) all partials parked
      if (warp == 2 && lane == 0) trace_phase(ep.tr, 4);
      // Owned regions g = z, z + splits, ... (region g = row quarter g / 2,
      // column half g % 2). Other splits read only their own regions of this
      // CTA's copy, so the sums can overwrite the owned ones in place.
      constexpr int kQ4 = kHalf / 4;  // float4 per region row
      constexpr int kPerRegion = 32 * kQ4;
      const int nreg = ep.split_dist ? (2 * 4 - 1 - z) / splits + 1 : 0;
      for (int e = threadIdx.x - 64; e < nreg * kPerRegion; e += kEpiWarps * 32) {
        const int ri = e / kPerRegion, w = e - ri * kPerRegion;
        const int g = z + ri * splits;
        const int row = (g >> 1) * 32 + w / kQ4;
        if (m0 + row >= M) continue;
        uint32_t* loc = part + row * kPartPitch + (g & 1) * kHalf + (w % kQ4) * 4;
        const uint32_t addr = smem_u32(loc);
        uint4 pz[kMaxSplits];
#pragma unroll
        for (int zz = 0; zz < kMaxSplits; ++zz)
          if (zz < splits)
            pz[zz] = zz == z ? *reinterpret_cast<const uint4*>(loc) : dsmem_ld4(dsmem_map(addr, zz));
        uint4 a = pz[0];
#pragma unroll
        for (int zz = 1; zz < kMaxSplits; ++zz) {
          if (zz >= splits) break;
          const uint4 b = pz[zz];
          if constexpr (PREC == kPrecI8) {
            a.x += b.x;
            a.y += b.y;
            a.z += b.z;
            a.w += b.w;
          } else {
            a.x = __float_as_uint(__fadd_rn(__uint_as_float(a.x), __uint_as_float(b.x)));
            a.y = __float_as_uint(__fadd_rn(__uint_as_float(a.y), __uint_as_float(b.y)));
            a.z = __float_as_uint(__fadd_rn(__uint_as_float(a.z), __uint_as_float(b.z)));
            a.w = __float_as_uint(__fadd_rn(__uint_as_float(a.w), __uint_as_float(b.w)));
          }
        }
        *reinterpret_cast<uint4*>(loc) = a;
      }
      if (ep.split_dist) asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
    }
#pragma unroll 1
    for (int c = half * kHalf; c < (half + 1) * kHalf; c += kChunk) {
      if (nrows <= 0) break;  // warp-uniform
      uint32_t r[32];
      if (splits > 1 && ep.split_dist) {  // this region's split sum (above)
#pragma unroll
        for (int j = 0; j < kChunk; j += 4) {
          const uint4 a = *reinterpret_cast<const uint4*>(my_part_row + c + j);
          r[j] = a.x;
          r[j + 1] = a.y;
          r[j + 2] = a.z;
          r[j + 3] = a.w;
        }
      } else if (splits > 1) {  // the owner warp reads every split's partials
        const uint32_t my_addr = smem_u32(my_part_row + c);
#pragma unroll
        for (int j = 0; j < kChunk; j += 4) {
          uint4 a = z == 0 ? *reinterpret_cast<const uint4*>(my_part_row + c + j)
                           : dsmem_ld4(dsmem_map(my_addr + 4 * j, 0));
          for (int zz = 1; zz < splits; ++zz) {
            const uint4 b = dsmem_ld4(dsmem_map(my_addr + 4 * j, zz));
            if constexpr (PREC == kPrecI8) {
              a.x += b.x;
              a.y += b.y;
              a.z += b.z;
              a.w += b.w;
            } else {
              a.x = __float_as_uint(__fadd_rn(__uint_as_float(a.x), __uint_as_float(b.x)));
              a.y = __float_as_uint(__fadd_rn(__uint_as_float(a.y), __uint_as_float(b.y)));
              a.z = __float_as_uint(__fadd_rn(__uint_as_float(a.z), __uint_as_float(b.z)));
              a.w = __float_as_uint(__fadd_rn(__uint_as_float(a.w), __uint_as_float(b.w)));
            }
          }
          r[j] = a.x;
          r[j + 1] = a.y;
          r[j + 2] = a.z;
          r[j + 3] = a.w;
        }
      } else if constexpr (kChunk == 32) {
        tmem_ld32(tmem + (static_cast<uint32_t>(q * 32) << 16) + c, r);
        tmem_ld_wait();
      } else {
        tmem_ld16(tmem + (static_cast<uint32_t>(q * 32) << 16) + c,
                  *reinterpret_cast<uint32_t(*)[16]>(r));
        tmem_ld_wait();
      }
      if (lane == 0 && c == half * kHalf) trace_phase(ep.tr, 6);
      if (n0 + c >= N) continue;  // warp-uniform
      if (nrows < 32 && lane >= nrows) {  // rows past M: stale A rows (GemmPlan::a_box)
#pragma unroll
        for (int j = 0; j < kChunk; ++j) r[j] = 0u;
      }
      float v[kChunk];
      if constexpr (PREC == kPrecI8) {
        if (ep.seg_width == 0 || ep.seg_width % kChunk == 0) {
          // The weight segment is uniform over the chunk.
          const int seg = ep.seg_width > 0 ? min((n0 + c) / ep.seg_width, kMaxSegments - 1) : 0;
          float iv = inv[0];
#pragma unroll
          for (int s = 1; s < kMaxSegments; ++s) iv = seg == s ? inv[s] : iv;
#pragma unroll
          for (int j = 0; j < kChunk; ++j)
            v[j] = __fmul_rn(__int2float_rn(static_cast<int>(r[j])), iv);
        } else {  // narrow fused segments (tiny models): per column
#pragma unroll
          for (int j = 0; j < kChunk; ++j) {
            const int seg = min((n0 + c + j) / ep.seg_width, kMaxSegments - 1);
            float iv = inv[0];
#pragma unroll
            for (int s = 1; s < kMaxSegments; ++s) iv = seg == s ? inv[s] : iv;
            v[j] = __fmul_rn(__int2float_rn(static_cast<int>(r[j])), iv);
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < kChunk; ++j) v[j] = __uint_as_float(r[j]);
      }
      if constexpr (seg_mode) {  // bias + ReLU here, row max for the sentence scale
#pragma unroll
        for (int j = 0; j < kChunk; ++j) {
          const int col = n0 + c + j;
          if (col < N) {
            float x = v[j];
            if (has_bias) x = __fadd_rn(x, ep.bias[col]);
            if (relu) x = x > 0.0f ? x : 0.0f;
            v[j] = x;
            seg_max = fmaxf(seg_max, fabsf(x));
            seg_bad |= !isfinite(x);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < kChunk; ++j) stage[lane * 33 + j] = v[j];
      if constexpr (EPI == kEpiSoftmaxParts) {
        // Slice max / first argmax (strict >, so NaN never wins), then the
        // sequential sum of exp(x - max) in column order (P6),
        // re-reading the values from the staging tile (keeps the code small).
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
      }
      __syncwarp();
      const int col = n0 + c + (lane % kChunk);
      const bool col_ok = col < N && lane < kChunk;
      float* cp = Cbase + col;
      float* cp_lo = EPI == kEpiTf32Out ? ep.C_lo + (cp - ep.C) : nullptr;
      if constexpr (kPrefetch) {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          float x = stage[i * 33 + (lane % kChunk)];
          if (has_bias && !seg_mode) x = __fadd_rn(x, bias_pre);
          if (relu && !seg_mode) x = x > 0.0f ? x : 0.0f;
          if (has_res) x = __fadd_rn(res_pre[i], x);
          if (col_ok && i < nrows) gemm_store<EPI>(cp, cp_lo, i * ldc, x, ep.C);
        }
        __syncwarp();
        continue;
      }
      if (EPI == kEpiSoftmaxParts || (!has_bias && !relu && !has_res) || seg_mode) {
        if (col_ok) {
#pragma unroll 8
          for (int i = 0; i < 32; ++i)
            if (i < nrows) gemm_store<EPI>(cp, cp_lo, i * ldc, stage[i * 33 + lane], ep.C);
        }
        __syncwarp();
        continue;
      }
      const float bias = (col_ok && has_bias) ? ep.bias[col] : 0.0f;
      const float* rp = has_res ? ep.residual + static_cast<long long>(rbase) * ldr + col : nullptr;
      // Residual loads of a row group are issued before its stores: C may
      // alias the residual, so loads placed after stores would serialise.
#pragma unroll 1
      for (int i0 = 0; i0 < 32; i0 += 8) {
        float res[8];
        if (has_res) {
#pragma unroll
          for (int i = 0; i < 8; ++i)
            res[i] = (col_ok && i0 + i < nrows) ? rp[(i0 + i) * ldr] : 0.0f;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float x = stage[(i0 + i) * 33 + (lane % kChunk)];
          if (has_bias) x = __fadd_rn(x, bias);
          if (relu) x = x > 0.0f ? x : 0.0f;
          if (has_res) x = __fadd_rn(res[i], x);
          if (col_ok && i0 + i < nrows) gemm_store<EPI>(cp, cp_lo, (i0 + i) * ldc, x, ep.C);
        }
      }
      __syncwarp();
    }
    if (lane == 0) trace_phase(ep.tr, 5);
    if (seg_mode && nrows > 0) {  // constexpr-false for the other epilogues
      // Segmented max over the warp's rows (segments are contiguous row
      // ranges), then one atomic per segment present in the warp.
      const int sg = lane < nrows ? ep.row_seg[rbase + lane] : -1;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const float ov = __shfl_down_sync(0xffffffffu, seg_max, o);
        const int os = __shfl_down_sync(0xffffffffu, sg, o);
        if (lane + o < 32 && os == sg) seg_max = fmaxf(seg_max, ov);
      }
      const int prev = __shfl_up_sync(0xffffffffu, sg, 1);
      if (__any_sync(0xffffffffu, seg_bad && lane < nrows) && lane == 0)
        atomicExch(ep.nonfinite, 1);
      if (sg >= 0 && (lane == 0 || prev != sg))
        atomicMax(ep.seg_absmax + sg, __float_as_uint(seg_max));
    }
    if constexpr (EPI == kEpiSoftmaxParts) {
      // Row rbase+lane, slices sub0 .. sub0+kSubs-1 (sub0 % kSubs == 0).
      const int sub0 = (n0 + half * kHalf) / 32;
      const int nsub = (N + 31) / 32;
      if (lane < nrows && sub0 < nsub) {
        const long long o = static_cast<long long>(rbase + lane) * ep.part_ld + sub0;
        if (sub0 + kSubs <= nsub) {
          if constexpr (kSubs == 4) {
            *reinterpret_cast<float4*>(ep.part_m + o) =
                make_float4(sub_m[0], sub_m[1], sub_m[2], sub_m[3]);
            *reinterpret_cast<float4*>(ep.part_s + o) =
                make_float4(sub_s[0], sub_s[1], sub_s[2], sub_s[3]);
            *reinterpret_cast<int4*>(ep.part_arg + o) =
                make_int4(sub_a[0], sub_a[1], sub_a[2], sub_a[3]);
          } else {
#pragma unroll
            for (int k = 0; k < kSubs; ++k) {
              ep.part_m[o + k] = sub_m[k];
              ep.part_s[o + k] = sub_s[k];
              ep.part_arg[o + k] = sub_a[k];
            }
          }
        } else {
#pragma unroll
          for (int k = 0; k < kSubs; ++k)
            if (sub0 + k < nsub) {
              ep.part_m[o + k] = sub_m[k];
              ep.part_s[o + k] = sub_s[k];
              ep.part_arg[o + k] = sub_a[k];
            }
        }
      }
    }
    if (splits > 1) cluster_sync_all();  // (2) every owner is done reading the partials
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
  trace_end(ep.tr);
}

}  // namespace mtg
