// Small-batch linears (gemv.cuh): weights prefetched by bulk copies before
// the PDL wait, the activation operand (LayerNorm / embedding / int8
// quantization) built in every CTA, mma.sync fragments with the weights as
// the 16-row A operand and the <= 8 activation rows as B, reference
// epilogues; optional deterministic split-K across CTAs (fp32 / bf16).
#include "gemv.cuh"

#include <algorithm>
#include <cstdlib>
#include <string>

#include <cuda_bf16.h>

#include "detmath.cuh"
#include "errors.hpp"
#include "launch.cuh"
#include "ptx.cuh"
#include "rowops.cuh"

namespace mtg {

namespace {

constexpr int kGemvThreads = 256;
constexpr int kGemvWarps = kGemvThreads / 32;
// The output projection adds kEpiWarps epilogue warps: chunk i's logits /
// softmax partials overlap chunk i + 1's MMAs (named barriers, partials
// double-buffered).
constexpr int kEpiWarps = 8;
constexpr int kLogitsThreads = kGemvThreads + 32 * kEpiWarps;
__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
constexpr int kMaxGemvStages = 4;
constexpr int kLnKpl = 16;       // LayerNorm rows of d <= 512 in registers
constexpr int kKStepBytes = 32;  // one mma K step: 32 int8 / 16 bf16 / 8 tf32 elements
constexpr int kRowV4Max = 16;    // plain operand rows up to 2048 values in registers
#define kNegInfF (-__int_as_float(0x7f800000))

template <int PREC>
struct GemvElem {
  static constexpr int bytes = PREC == 0 ? 1 : PREC == 1 ? 2 : 4;
};

// Shared-memory carve-up (bytes), identical on host and device. Weight
// chunks arrive in fragment order (launch_gemv_pack); the operand rows of
// this CTA's K range are stored row-major with a pitch of range + 16 bytes,
// so the B-fragment loads of the 8 rows of a tile fall on distinct banks.
struct GemvSmem {
  int stage_bytes, nst, a_off, part_off, scale_off, ex_off, bar_off, total;
};
__host__ __device__ inline GemvSmem gemv_smem(int chunk, int ks, int kz_bytes, int nst, bool logits) {
  GemvSmem s;
  s.stage_bytes = (chunk * kz_bytes + 127) / 128 * 128;
  s.nst = nst;
  s.a_off = nst * s.stage_bytes;
  s.part_off = s.a_off + kGemvRows * (kz_bytes + 16);
  // the projection double-buffers the partials: a chunk's epilogue overlaps
  // the next chunk's MMAs (no CTA barrier between them)
  s.scale_off = s.part_off + (logits ? 2 : 1) * ks * kGemvRows * chunk * 4;
  s.ex_off = s.scale_off + kGemvRows * 4 * 4;  // [rows][4 segments] int8 epilogue factors
  s.bar_off = (s.ex_off + (logits ? kEpiWarps * kGemvRows * 33 * 4 : 0) + 7) / 8 * 8;
  s.total = s.bar_off + kMaxGemvStages * 8 + 8;
  return s;
}

// TF32x3 split by truncation: hi = the top 19 bits (what the tensor core
// reads of an fp32 register), lo = x - hi (exact). One LOP instead of the
// four-instruction cvt.rna emulation per element -- the split is most of
// the small-batch fp32 GEMV's instruction count. The dropped lo.lo term is
// below 2^-20 relative (2^-22 with rounding), far inside the fp32 bar.
__device__ __forceinline__ uint32_t tf32_hi(uint32_t x) { return x & 0xffffe000u; }

// D += A (16 weight rows x 1 K step) . B (1 K step x 8 operand rows).
template <int PREC>
__device__ __forceinline__ void mma_frag(uint32_t (&d)[4], const uint32_t (&a)[4],
                                         const uint32_t (&b)[2]) {
  if constexpr (PREC == 0) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  } else if constexpr (PREC == 1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  } else {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
}

// One K step: the weight fragment (16 bytes per lane, fragment order) and
// the operand fragment (row g of the padded row-major block: b0 at 4q,
// b1 at 16 + 4q). fp32 is TF32x3 as on the tcgen05 path: x = hi + lo,
// acc += lo.hi + hi.lo + hi.hi.
template <int PREC>
__device__ __forceinline__ void mma_step(uint32_t (&d)[4], const uint8_t* wf, const uint8_t* xf) {
  const uint4 av = *reinterpret_cast<const uint4*>(wf);
  uint32_t a[4] = {av.x, av.y, av.z, av.w};
  uint32_t b[2] = {*reinterpret_cast<const uint32_t*>(xf), *reinterpret_cast<const uint32_t*>(xf + 16)};
  if constexpr (PREC == 2) {
    uint32_t ah[4], al[4], bh[2], bl[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      ah[i] = tf32_hi(a[i]);
      al[i] = __float_as_uint(__fsub_rn(__uint_as_float(a[i]), __uint_as_float(ah[i])));
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      bh[i] = tf32_hi(b[i]);
      bl[i] = __float_as_uint(__fsub_rn(__uint_as_float(b[i]), __uint_as_float(bh[i])));
    }
    mma_frag<2>(d, al, bh);
    mma_frag<2>(d, ah, bl);
    mma_frag<2>(d, ah, bh);
  } else {
    mma_frag<PREC>(d, a, b);
  }
}

// fp32 (TF32x3) with the three products in separate accumulators: three
// independent MMA chains instead of one chain three times as long (the MMA
// phase of the batch-1 projection GEMV is latency-bound on that chain).
// Final value (lo.hi + hi.lo) + hi.hi.
__device__ __forceinline__ void mma_step_tf32x3(uint32_t (&d_lh)[4], uint32_t (&d_hl)[4],
                                                uint32_t (&d_hh)[4], const uint8_t* wf,
                                                const uint8_t* xf) {
  const uint4 av = *reinterpret_cast<const uint4*>(wf);
  const uint32_t a[4] = {av.x, av.y, av.z, av.w};
  const uint32_t b[2] = {*reinterpret_cast<const uint32_t*>(xf), *reinterpret_cast<const uint32_t*>(xf + 16)};
  uint32_t ah[4], al[4], bh[2], bl[2];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    ah[i] = tf32_hi(a[i]);
    al[i] = __float_as_uint(__fsub_rn(__uint_as_float(a[i]), __uint_as_float(ah[i])));
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    bh[i] = tf32_hi(b[i]);
    bl[i] = __float_as_uint(__fsub_rn(__uint_as_float(b[i]), __uint_as_float(bh[i])));
  }
  mma_frag<2>(d_lh, al, bh);
  mma_frag<2>(d_hl, ah, bl);
  mma_frag<2>(d_hh, ah, bh);
}

// Stores one operand element (row n, column c of the CTA's K range; pitch P).
template <int PREC>
__device__ __forceinline__ void store_elem(uint8_t* A, int P, int n, int c, float x, int8_t q) {
  constexpr int E = GemvElem<PREC>::bytes;
  uint8_t* p = A + n * P + c * E;
  if constexpr (PREC == 0)
    *reinterpret_cast<int8_t*>(p) = q;
  else if constexpr (PREC == 1)
    *reinterpret_cast<__nv_bfloat16*>(p) = __float2bfloat16_rn(x);
  else
    *reinterpret_cast<float*>(p) = x;
}

// Four consecutive operand values (c % 4 == 0) of row n.
template <int PREC>
__device__ __forceinline__ void store_vec4(uint8_t* A, int P, int n, int c, float4 v, float scale) {
  constexpr int E = GemvElem<PREC>::bytes;
  uint8_t* p = A + n * P + c * E;
  if constexpr (PREC == 0) {  // scale from the row's own max: in range
    const uint32_t lo = __byte_perm(quant1_in_range(v.x, scale), quant1_in_range(v.y, scale), 0x0040);
    const uint32_t hi = __byte_perm(quant1_in_range(v.z, scale), quant1_in_range(v.w, scale), 0x0040);
    *reinterpret_cast<uint32_t*>(p) = __byte_perm(lo, hi, 0x5410);
  } else if constexpr (PREC == 1) {
    const __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
    *reinterpret_cast<uint2*>(p) =
        make_uint2(*reinterpret_cast<const uint32_t*>(&lo), *reinterpret_cast<const uint32_t*>(&hi));
  } else {
    *reinterpret_cast<float4*>(p) = v;
  }
}

// One CTA processes chunks of `chunk` output columns (weight rows) over its
// K range (split-K: blockIdx.y of gridDim.y); the 8 warps split a chunk into
// chunk/16 column groups x ks K ranges, whose partial sums meet in shared
// memory and are added in K-range order (int8 exact). Split-K partials go
// through `ws`; the last CTA of a chunk (ticket `sem`) adds them in split
// order and runs the epilogue.
template <int PREC, bool LOGITS, int kRowV4>
__global__ void __launch_bounds__(LOGITS ? kLogitsThreads : kGemvThreads, 1)
    gemv_kernel(const GemvArgs a, int chunk, int ks, int nst, uint32_t piece) {
  constexpr int E = GemvElem<PREC>::bytes;
  extern __shared__ __align__(128) uint8_t sm[];
  const int row_bytes = a.k_pad * E;
  const int nz = gridDim.y, z = blockIdx.y;
  const int kz_bytes = row_bytes / nz;                             // this CTA's K range (bytes)
  const int kz0 = z * kz_bytes / E, kz1 = (z + 1) * kz_bytes / E;  // element range
  const GemvSmem L = gemv_smem(chunk, ks, kz_bytes, nst, LOGITS);
  uint8_t* stages = sm;
  uint8_t* A = sm + L.a_off;
  const int AP = kz_bytes + 16;  // operand row pitch (bytes)
  uint32_t* const part_base = reinterpret_cast<uint32_t*>(sm + L.part_off);
  float* inv = reinterpret_cast<float*>(sm + L.scale_off);  // [r][seg] (int8)
  float* ex = reinterpret_cast<float*>(sm + L.ex_off);      // [warp][row][33] (projection)
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + L.bar_off);
  int* flag = reinterpret_cast<int*>(sm + L.bar_off + kMaxGemvStages * 8);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_chunks = (a.N + chunk - 1) / chunk;
  const int G = gridDim.x;
  const int my_count = static_cast<int>(blockIdx.x) < n_chunks
                           ? (n_chunks - 1 - static_cast<int>(blockIdx.x)) / G + 1
                           : 0;
  const int ksteps = row_bytes / kKStepBytes, kz_steps = kz_bytes / kKStepBytes;
  const uint8_t* W = static_cast<const uint8_t*>(a.w);
  // Chunk i of this CTA -> stage i % nst. A 16-row group's K steps are
  // contiguous in the fragment-order copy: one bulk copy per group (of the
  // CTA's K range), issued by warp 0.
  auto issue = [&](int i) {
    const int n0 = (blockIdx.x + i * G) * chunk;
    const int groups = (min(chunk, (a.N + 15) / 16 * 16 - n0) + 15) / 16;
    const uint32_t gbytes = static_cast<uint32_t>(kz_steps) * 512;
    uint64_t* bar = &full[i % nst];
    if (lane == 0) mbar_arrive_expect_tx(bar, gbytes * groups);
    __syncwarp();
    uint8_t* dst = stages + (i % nst) * L.stage_bytes;
    for (int gq = 0; gq < groups; ++gq) {
      const uint8_t* src =
          W + (static_cast<long long>(n0 / 16 + gq) * ksteps + static_cast<long long>(z) * kz_steps) * 512;
      for (uint32_t o = lane * piece; o < gbytes; o += 32u * piece)
        bulk_load(dst + gq * gbytes + o, src + o, min(piece, gbytes - o), bar);
    }
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  // Everything that does not depend on the previous kernel is fetched before
  // the programmatic-dependency wait: the weight chunks, LayerNorm gain /
  // bias, the output bias of this CTA's first chunk, the int8 weight scales.
  if (warp == 0)
    for (int i = 0; i < min(nst, my_count); ++i) issue(i);
  const bool ln = a.a_mode != 0;
  float gv[kLnKpl], bv[kLnKpl];
  if (ln) {
#pragma unroll
    for (int i = 0; i < kLnKpl; ++i) {
      const int c = lane + 32 * i;
      gv[i] = c < a.K ? a.ln_g[c] : 0.0f;
      bv[i] = c < a.K ? a.ln_b[c] : 0.0f;
    }
  }
  const int n_first = blockIdx.x * chunk;
  const int ep_r = threadIdx.x / chunk, ep_c = threadIdx.x % chunk;  // first-chunk epilogue slot
  const bool ep_ok = !LOGITS && nz == 1 && my_count > 0 && ep_r < a.rows_alloc && n_first + ep_c < a.N;
  const float bias0 = ep_ok && a.bias ? a.bias[n_first + ep_c] : 0.0f;
  const float sw = PREC == 0 && lane < 4 ? a.w_seg_scale[a.seg_width > 0 ? lane : 0] : 1.0f;
  pdl_wait();
  pdl_trigger();
  trace_begin(a.trace);
  if (threadIdx.x == 0) trace_phase(a.trace, 0);
  // Dependent loads, all issued together: live-row count, step, the operand
  // row of this warp (every allocated row; rows >= R are computed and
  // discarded), the first chunk's residual.
  const int R_dev = *a.d_rows;
  const int t = a.d_step ? *a.d_step : 0;
  const float res0 = ep_ok && a.residual ? a.residual[ep_r * a.ldr + n_first + ep_c] : 0.0f;
  const int r = warp;
  const bool have_row = r < a.rows_alloc;
  const int kzn = kz1 - kz0;
  // Plain rows (attention contexts, FFN hidden rows): this CTA's K range in
  // registers, float4 per lane (element kz0 + 4 lane + 128 i). LayerNorm
  // rows: value c = lane + 32 i (the P1 order).
  const bool vec = !ln && a.K % 4 == 0 && a.ldx % 4 == 0 && kz0 % 4 == 0 && kzn <= 128 * kRowV4;
  constexpr int kRegs = 4 * kRowV4 > kLnKpl ? 4 * kRowV4 : kLnKpl;
  float xv[kRegs];
  if (have_row) {
    if (vec) {
      const float* xr = a.x + r * a.ldx + kz0;
#pragma unroll
      for (int i = 0; i < kRowV4; ++i) {
        const int c = 4 * lane + 128 * i;
        const float4 v = c < kzn && kz0 + c < a.K ? *reinterpret_cast<const float4*>(xr + c)
                                                  : make_float4(0.f, 0.f, 0.f, 0.f);
        xv[4 * i] = v.x;
        xv[4 * i + 1] = v.y;
        xv[4 * i + 2] = v.z;
        xv[4 * i + 3] = v.w;
      }
    } else if (ln) {
      const int n = a.K;
      if (a.a_mode == 2) {
        const long long id = min(max(a.prev[r], 0), a.table_rows - 1);
        const float* pe = a.pe + static_cast<long long>(t) * n;
#pragma unroll
        for (int i = 0; i < kLnKpl; ++i) {
          const int c = lane + 32 * i;
          xv[i] = c < n ? __fadd_rn(__fmul_rn(a.table[id * n + c], a.sqrt_d), pe[c]) : 0.0f;
        }
      } else {
#pragma unroll
        for (int i = 0; i < kLnKpl; ++i) {
          const int c = lane + 32 * i;
          xv[i] = c < n ? a.x[r * a.ldx + c] : 0.0f;
        }
      }
    }
  }
  const int R = min(R_dev, kGemvRows);
  if (threadIdx.x == 0) trace_phase(a.trace, 1);  // operand row loaded (warp 0)

  // ---- step start: beam history reorder (beam.cu beam_reorder_kernel) ----
  if (a.a_mode == 2 && a.reorder && t >= 1 && blockIdx.x == G - 1) {
    const int cur = (t - 1) & 1, nxt = t & 1;
    for (int rr = 0; rr < R; ++rr) {
      const int pr = a.row_parent[rr];
      const int* ac = a.anc[cur] + static_cast<long long>(pr) * a.T;
      int* an = a.anc[nxt] + static_cast<long long>(rr) * a.T;
      const int* tc = a.tok[cur] + static_cast<long long>(pr) * a.T;
      int* tn = a.tok[nxt] + static_cast<long long>(rr) * a.T;
      for (int j = threadIdx.x; j < t && j < a.T; j += blockDim.x) an[j] = ac[j];
      for (int j = threadIdx.x; j < t - 1; j += blockDim.x) tn[j] = tc[j];
      if (threadIdx.x == 0) {
        if (t < a.T) an[t] = rr;
        if (t - 1 < a.T) tn[t - 1] = a.prev[rr];
      }
    }
  }

  // ---- operand row r = warp (rows past the allocation are zero) ----
  // int8: one scale per row (each hypothesis row is one quantize call,
  // quant.cpp:108-122).
  if (r < kGemvRows) {
    int bad = 0;
    float scale = 1.0f;
    uint8_t* arow = A + r * AP;
    if (!have_row) {
      for (int c = 4 * lane; c < kz_bytes; c += 128) *reinterpret_cast<uint32_t*>(arow + c) = 0u;
    } else if (ln) {  // LayerNorm (d <= 512) of x or of the target embedding
      float(&v)[kLnKpl] = *reinterpret_cast<float(*)[kLnKpl]>(xv);
      if (a.a_mode == 2 && blockIdx.x == 0 && r < R) {
#pragma unroll
        for (int i = 0; i < kLnKpl; ++i)
          if (lane + 32 * i < a.K) a.x_out[r * a.ldx_out + lane + 32 * i] = v[i];
      }
      const float mx = ln_normalize_regs<kLnKpl>(v, gv, bv, a.K, lane, &bad);
      if (MTG_TRACE_PHASES == 2 && threadIdx.x == 0) trace_phase(a.trace, 6);
      scale = qscale_of(mx);
      if (kzn >= 32 * kLnKpl) {
        // whole register row inside the operand row: unconditional stores
        // (values past K are 0 and quantize to 0). The per-element guards
        // compiled to a branch per value and cost ~1 us per int8 GEMV.
#pragma unroll
        for (int i = 0; i < kLnKpl; ++i)
          store_elem<PREC>(A, AP, r, lane + 32 * i, v[i],
                           PREC == 0 ? static_cast<int8_t>(quant1_in_range(v[i], scale)) : int8_t(0));
      } else {
#pragma unroll
        for (int i = 0; i < kLnKpl; ++i) {
          const int c = lane + 32 * i;
          if (c < kzn) store_elem<PREC>(A, AP, r, c, v[i], c < a.K && PREC == 0 ? quant1(v[i], scale) : int8_t(0));
        }
      }
      for (int c = 32 * kLnKpl + lane; c < kzn; c += 32) store_elem<PREC>(A, AP, r, c, 0.0f, 0);
      if (MTG_TRACE_PHASES == 2 && threadIdx.x == 0) trace_phase(a.trace, 7);
    } else if (vec) {
      if constexpr (PREC == 0) {
        // max |x| and the non-finite test (x * 0 is NaN only for inf / NaN)
        // as four independent chains
        float m4[4] = {0.0f, 0.0f, 0.0f, 0.0f}, z4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
        for (int i = 0; i < 4 * kRowV4; ++i) {
          m4[i & 3] = fmaxf(m4[i & 3], fabsf(xv[i]));
          z4[i & 3] = __fmaf_rn(xv[i], 0.0f, z4[i & 3]);
        }
        const float z = __fadd_rn(__fadd_rn(z4[0], z4[1]), __fadd_rn(z4[2], z4[3]));
        bad = z != z;
        scale = qscale_of(warp_allmax(fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]))));
      }
      if (kzn >= 128 * kRowV4) {  // unconditional stores, as above
#pragma unroll
        for (int i = 0; i < kRowV4; ++i)
          store_vec4<PREC>(A, AP, r, 4 * lane + 128 * i,
                           make_float4(xv[4 * i], xv[4 * i + 1], xv[4 * i + 2], xv[4 * i + 3]), scale);
      } else {
#pragma unroll
        for (int i = 0; i < kRowV4; ++i) {
          const int c = 4 * lane + 128 * i;
          if (c >= kzn) break;
          store_vec4<PREC>(A, AP, r, c, make_float4(xv[4 * i], xv[4 * i + 1], xv[4 * i + 2], xv[4 * i + 3]),
                           scale);
        }
      }
    } else {  // plain fp32 rows, generic shapes
      const float* xr = a.x + r * a.ldx;
      if constexpr (PREC == 0) {
        float m = 0.0f;
        for (int c = lane; c < a.K; c += 32) {
          const float x = xr[c];
          m = fmaxf(m, fabsf(x));
          bad |= !isfinite(x);
        }
        scale = qscale_of(warp_allmax(m));
      }
      for (int c = lane; c < kzn; c += 32) {
        const float x = kz0 + c < a.K ? xr[kz0 + c] : 0.0f;
        store_elem<PREC>(A, AP, r, c, x, PREC == 0 && kz0 + c < a.K ? quant1(x, scale) : int8_t(0));
      }
    }
    if constexpr (PREC == 0) {
      // quantize() throws on non-finite input (quant.cpp:110-112)
      if (r < R && blockIdx.x == 0 && z == 0 && __any_sync(0xffffffffu, bad) && lane == 0)
        atomicExch(a.nonfinite, 1);
      // epilogue factor 1 / (sa * sw) per weight segment (quant.cpp:160, 189)
      if (lane < 4) inv[r * 4 + lane] = __frcp_rn(__fmul_rn(scale, sw));
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) trace_phase(a.trace, 2);  // operand rows built

  const int gi = warp / ks, kr = warp % ks;  // column group, K range within the CTA's K range
  const int s_begin = kr * kz_steps / ks, s_end = (kr + 1) * kz_steps / ks;
  const int g = lane >> 2, q = lane & 3;
  const long long step_off = a.c_step_stride ? static_cast<long long>(t) * a.c_step_stride : 0LL;
  const bool mma_warp = warp < kGemvWarps;  // projection: warps >= 8 run the epilogues
  for (int i = 0; i < my_count; ++i) {
    const int s = i % nst;
    // Projection: partial buffer b = i & 1, barriers ready[b] (id 1 + b: MMA
    // warps arrive, epilogue warps wait) and free[b] (id 3 + b: epilogue
    // warps arrive after chunk i, MMA warps wait before chunk i + 2).
    const int b = i & 1;
    uint32_t* const part = part_base + (LOGITS ? b * ks * kGemvRows * chunk : 0);
    const int cidx = blockIdx.x + i * G;
    const int n0 = cidx * chunk;
    const int ncols = min(chunk, a.N - n0);
    if (mma_warp) {
      if constexpr (LOGITS) {
        if (i >= 2) named_sync(3 + b, kLogitsThreads);
      }
      mbar_wait(&full[s], (i / nst) & 1);
      if (threadIdx.x == 0 && i == 0) trace_phase(a.trace, 3);  // weights landed
      if (MTG_TRACE_PHASES != 2 && threadIdx.x == 0 && i == my_count - 1)
        trace_phase(a.trace, 6);  // last chunk landed
      if (gi * 16 < chunk) {
        // group gi of the chunk: [K step][lane][16 bytes]
        const uint8_t* wf = stages + s * L.stage_bytes + gi * kz_steps * 512 + lane * 16;
        const uint8_t* xf = A + g * AP + 4 * q;  // operand row g, the lane's K bytes
        uint32_t d[4] = {0u, 0u, 0u, 0u};
        if constexpr (PREC == 2) {
          uint32_t d1[4] = {0u, 0u, 0u, 0u}, d2[4] = {0u, 0u, 0u, 0u};
#pragma unroll 4
          for (int st = s_begin; st < s_end; ++st)
            mma_step_tf32x3(d1, d2, d, wf + st * 512, xf + st * kKStepBytes);
#pragma unroll
          for (int e = 0; e < 4; ++e)
            d[e] = __float_as_uint(__fadd_rn(
                __fadd_rn(__uint_as_float(d1[e]), __uint_as_float(d2[e])), __uint_as_float(d[e])));
        } else {
#pragma unroll 4
          for (int st = s_begin; st < s_end; ++st) mma_step<PREC>(d, wf + st * 512, xf + st * kKStepBytes);
        }
        uint32_t* pp = part + kr * kGemvRows * chunk;
        const int c0 = gi * 16 + g;
        pp[(2 * q) * chunk + c0] = d[0];
        pp[(2 * q + 1) * chunk + c0] = d[1];
        pp[(2 * q) * chunk + c0 + 8] = d[2];
        pp[(2 * q + 1) * chunk + c0 + 8] = d[3];
      }
      if constexpr (LOGITS) {
        named_arrive(1 + b, kLogitsThreads);  // partials complete
        named_sync(5, kGemvThreads);          // stage s consumed
      } else {
        __syncthreads();  // stage s consumed, partials complete
      }
      if (threadIdx.x == 0 && i == 0) trace_phase(a.trace, 4);  // first chunk's MMAs done
      if (MTG_TRACE_PHASES != 2 && threadIdx.x == 0 && i == my_count - 1)
        trace_phase(a.trace, 7);  // last chunk's MMAs done
      if (warp == 0 && i + nst < my_count) issue(i + nst);
    }

    // Split-K: publish this CTA's sums; the chunk's last CTA adds all splits
    // in split order (deterministic) and runs the epilogue.
    bool last = true;
    if (!LOGITS && nz > 1) {
      float* wsc = a.ws + static_cast<long long>(cidx) * nz * kGemvRows * chunk;
      for (int idx = threadIdx.x; idx < R * chunk; idx += blockDim.x) {
        const int rr = idx / chunk, c = idx - rr * chunk;
        uint32_t v;
        if constexpr (PREC == 0) {
          int acc = 0;
          for (int k = 0; k < ks; ++k) acc += static_cast<int>(part[(k * kGemvRows + rr) * chunk + c]);
          v = static_cast<uint32_t>(acc);
        } else {
          float acc = __uint_as_float(part[rr * chunk + c]);
          for (int k = 1; k < ks; ++k)
            acc = __fadd_rn(acc, __uint_as_float(part[(k * kGemvRows + rr) * chunk + c]));
          v = __float_as_uint(acc);
        }
        reinterpret_cast<uint32_t*>(wsc)[(z * kGemvRows + rr) * chunk + c] = v;
      }
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) {
        const int tk = atomicAdd(a.sem + cidx, 1);
        *flag = tk == nz - 1;
        if (tk == nz - 1) a.sem[cidx] = 0;  // ready for the next launch
      }
      __syncthreads();
      last = *flag != 0;
      if (last) {
        __threadfence();
        for (int idx = threadIdx.x; idx < R * chunk; idx += blockDim.x) {
          const int rr = idx / chunk, c = idx - rr * chunk;
          uint32_t v;
          if constexpr (PREC == 0) {
            int acc = 0;
            for (int k = 0; k < nz; ++k)
              acc += static_cast<int>(__ldcg(reinterpret_cast<const unsigned*>(wsc) + (k * kGemvRows + rr) * chunk + c));
            v = static_cast<uint32_t>(acc);
          } else {
            float acc = __ldcg(wsc + rr * chunk + c);
            for (int k = 1; k < nz; ++k) acc = __fadd_rn(acc, __ldcg(wsc + (k * kGemvRows + rr) * chunk + c));
            v = __float_as_uint(acc);
          }
          part[rr * chunk + c] = v;  // split total, read back as range 0 below
        }
        __syncthreads();
      }
    }
    const int ksum = nz > 1 ? 1 : ks;

    // Sum of the K-range partials (in order) and the reference epilogue
    // conversion: int8 float(acc) * (1 / (sa * sw)).
    auto value = [&](int rr, int c) -> float {
      if constexpr (PREC == 0) {
        int acc = 0;
        for (int k = 0; k < ksum; ++k) acc += static_cast<int>(part[(k * kGemvRows + rr) * chunk + c]);
        const int n = n0 + c;
        const int seg = a.seg_width > 0 ? min(n / a.seg_width, 3) : 0;
        return __fmul_rn(__int2float_rn(acc), inv[rr * 4 + seg]);
      } else {
        float acc = __uint_as_float(part[rr * chunk + c]);
        for (int k = 1; k < ksum; ++k)
          acc = __fadd_rn(acc, __uint_as_float(part[(k * kGemvRows + rr) * chunk + c]));
        return acc;
      }
    };
    if constexpr (!LOGITS) {
      if (last) {
        for (int idx = threadIdx.x; idx < R * ncols; idx += blockDim.x) {
          const int rr = idx / ncols, c = idx - rr * ncols, n = n0 + c;
          // first chunk: bias / residual already in registers (slot == idx)
          const bool pre = ep_ok && i == 0 && rr == ep_r && c == ep_c;
          float y = value(rr, c);
          if (a.bias) y = __fadd_rn(y, pre ? bias0 : a.bias[n]);
          if (a.relu) y = y > 0.0f ? y : 0.0f;
          if (a.residual) y = __fadd_rn(pre ? res0 : a.residual[rr * a.ldr + n], y);
          a.C[step_off + rr * a.ldc + n] = y;
        }
      }
    } else if (!mma_warp) {
      named_sync(1 + b, kLogitsThreads);  // chunk i's partials
      // Output projection: warps take (32-column slice, block of RB rows)
      // items and store the logits of those rows and the slice partials --
      // max, first argmax (strict >, so NaN never wins) and the sum of
      // exp(x - max) in column order (P6). The exps are lane-parallel; the
      // ordered sums run one row per lane.
      const int n_sl = (ncols + 31) / 32;
      const int ew = warp - kGemvWarps;
      const int RB = max(1, (R * n_sl + kEpiWarps - 1) / kEpiWarps);
      const int nrb = (R + RB - 1) / RB;
      float* e = ex + ew * (kGemvRows * 33);
      for (int it = ew; it < n_sl * nrb; it += kEpiWarps) {
        const int sl = it / nrb, r0 = (it - sl * nrb) * RB, r1 = min(R, r0 + RB);
        const int c = sl * 32 + lane;
        const int nv = min(32, ncols - sl * 32);
        const bool ok = lane < nv;
        float my_best = 0.0f;
        int my_bi = -1;
#pragma unroll
        for (int k = 0; k < kGemvRows; ++k) {
          const int rr = r0 + k;
          if (rr >= r1) break;
          const float v = ok ? value(rr, c) : 0.0f;
          if (ok) a.C[rr * a.ldc + n0 + c] = v;
          const float best = warp_allmax(ok && v == v ? v : kNegInfF);
          const unsigned hit = __ballot_sync(0xffffffffu, ok && v == best && best > kNegInfF);
          const int bi = hit ? n0 + sl * 32 + __ffs(hit) - 1 : -1;
          if (bi >= 0 && ok) {
            // the fast exp has the same bits on [-86.5, 0] (and NaN); other
            // lanes take the full one (lane-local choice, no warp minimum)
            const float zz = __fsub_rn(v, best);
            float ez = det_expf_nonpos_fast(zz);
            if (!(zz >= -86.5f)) ez = det_expf_nonpos(zz);
            e[k * 33 + lane] = ez;
          }
          if (lane == k) {
            my_best = best;
            my_bi = bi;
          }
        }
        __syncwarp();
        if (lane < r1 - r0) {
          float sum = 0.0f;
          if (my_bi >= 0) {
            const float* er = e + lane * 33;
            if (nv == 32) {
              float t32[32];
#pragma unroll
              for (int j = 0; j < 32; ++j) t32[j] = er[j];
#pragma unroll
              for (int j = 0; j < 32; ++j) sum = __fadd_rn(sum, t32[j]);
            } else {
              for (int j = 0; j < nv; ++j) sum = __fadd_rn(sum, er[j]);
            }
          }
          const long long o = static_cast<long long>(r0 + lane) * a.part_ld + (n0 + sl * 32) / 32;
          a.part_m[o] = my_best;
          a.part_s[o] = sum;
          a.part_arg[o] = my_bi;
        }
        __syncwarp();
      }
      if (i + 2 < my_count) named_arrive(3 + b, kLogitsThreads);  // buffer b free
    }
    if constexpr (!LOGITS) __syncthreads();  // partials reused by the next chunk
  }
  if (LOGITS && a.trace.buf) __syncthreads();  // the exit time includes the epilogue warps
  if (threadIdx.x == 0) trace_phase(a.trace, 5);
  trace_end(a.trace);
}

template <int PREC, bool LOGITS>
void launch_gemv_t(const GemvArgs& a, cudaStream_t st) {
  constexpr int E = GemvElem<PREC>::bytes;
  const int row_bytes = a.k_pad * E;
  if (row_bytes % 128 != 0) fail(kStateError, "gemv: k_pad must be a whole 128-byte slab");
  if (a.a_mode != 0 && a.K > 32 * kLnKpl) fail(kUsageError, "gemv: LayerNorm rows above 512");
  if (a.rows_alloc > kGemvRows) fail(kStateError, "gemv: more than 8 operand rows");
  const int nz = std::max(1, a.ksplit);
  // int8 rows are quantized with their own max: every CTA needs whole rows
  if (nz > 1 && (LOGITS || PREC == 0 || a.a_mode != 0 || !a.ws || !a.sem || row_bytes % (nz * 128) != 0))
    fail(kStateError, "gemv: split-K needs fp32 / bf16 plain operand rows, a workspace and "
                      "128-byte ranges");
  const int kz_bytes = row_bytes / nz;
  const int ksteps = kz_bytes / kKStepBytes;
  // Column groups per chunk (16 columns each) and K ranges: groups x ranges
  // = 8 warps. Linear layers: one group, K split 8 ways (spreads small
  // layers over more SMs); projection: whole 32-column slices per chunk.
  int groups = 1;
  if (LOGITS) {
    // MTG_GEMV_LOGITS_GROUPS caps the 16-column groups per chunk (A/B)
    static const int cap = [] {
      const char* e = std::getenv("MTG_GEMV_LOGITS_GROUPS");
      return e ? std::max(2, std::atoi(e)) : 8;
    }();
    groups = 2;
    while (groups < std::min(8, cap) && 16 * (2 * groups) * kz_bytes <= 64 * 1024) groups *= 2;
  }
  const int ks = std::min(kGemvWarps / groups, ksteps);
  const int chunk = 16 * groups;
  const int n_chunks = (a.N + chunk - 1) / chunk;
  const int grid = std::min(148, n_chunks);
  const int per_cta = (n_chunks + grid - 1) / grid;
  if (nz > 1 && per_cta > 1) fail(kStateError, "gemv: split-K with more than one chunk per CTA");
  int nst = std::min(kMaxGemvStages, per_cta);
  constexpr int kBudget = 227 * 1024;
  while (nst > 1 && gemv_smem(chunk, ks, kz_bytes, nst, LOGITS).total > kBudget) --nst;
  const GemvSmem L = gemv_smem(chunk, ks, kz_bytes, nst, LOGITS);
  if (L.total > kBudget) fail(kUsageError, "gemv: operand rows too large for shared memory");
  // Plain operand rows are held in registers (float4 per lane): the wide
  // variant (up to 2048 values per row) only where needed, it costs occupancy.
  const bool wide = a.a_mode == 0 && kz_bytes / E > 512;
  auto k = wide ? gemv_kernel<PREC, LOGITS, kRowV4Max> : gemv_kernel<PREC, LOGITS, 4>;
  ensure_smem_attr(k, L.total);
  // Bulk-copy piece size (MTG_GEMV_PIECE bytes, A/B; multiple of 16).
  static const uint32_t piece = [] {
    const char* e = std::getenv("MTG_GEMV_PIECE");
    const long v = e ? std::atol(e) : 1L << 20;  // measured: one copy per group is fastest
    return static_cast<uint32_t>(std::max<long>(16, v / 16 * 16));
  }();
  launch_k(k, dim3(grid, nz), LOGITS ? kLogitsThreads : kGemvThreads, L.total, st, a, chunk, ks, nst,
           piece);
  MTG_CUDA(cudaGetLastError());
}

// One thread per 16-byte lane slot of the fragment-order copy.
__global__ void gemv_pack_kernel(const uint8_t* __restrict__ w, int n, int row_bytes,
                                 uint8_t* __restrict__ out, long long slots) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= slots) return;
  const int lane = static_cast<int>(i & 31);
  const long long blk = i >> 5;  // (group, K step)
  const int ksteps = row_bytes / kKStepBytes;
  const int grp = static_cast<int>(blk / ksteps), st = static_cast<int>(blk % ksteps);
  const int g = lane >> 2, q = lane & 3;
  uint32_t v[4];
#pragma unroll
  for (int reg = 0; reg < 4; ++reg) {
    const int row = grp * 16 + g + 8 * (reg & 1);
    const int off = st * kKStepBytes + 16 * (reg >> 1) + 4 * q;
    v[reg] = row < n ? *reinterpret_cast<const uint32_t*>(w + static_cast<long long>(row) * row_bytes + off)
                     : 0u;
  }
  *reinterpret_cast<uint4*>(out + i * 16) = make_uint4(v[0], v[1], v[2], v[3]);
}

}  // namespace

void launch_gemv_pack(const void* w, int n, int k_pad, int elem, void* out, cudaStream_t st) {
  const int row_bytes = k_pad * elem;
  if (row_bytes % 128 != 0) fail(kStateError, "gemv pack: rows must be whole 128-byte slabs");
  const long long slots = gemv_pack_bytes(n, k_pad, elem) / 16;
  if (slots == 0) return;
  gemv_pack_kernel<<<static_cast<unsigned>((slots + 255) / 256), 256, 0, st>>>(
      static_cast<const uint8_t*>(w), n, row_bytes, static_cast<uint8_t*>(out), slots);
  MTG_CUDA(cudaGetLastError());
}

void launch_gemv(int prec, bool logits, const GemvArgs& a, cudaStream_t st) {
  if (prec == 0)
    logits ? launch_gemv_t<0, true>(a, st) : launch_gemv_t<0, false>(a, st);
  else if (prec == 1)
    logits ? launch_gemv_t<1, true>(a, st) : launch_gemv_t<1, false>(a, st);
  else
    logits ? launch_gemv_t<2, true>(a, st) : launch_gemv_t<2, false>(a, st);
}

}  // namespace mtg
