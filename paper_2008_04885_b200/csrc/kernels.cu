// Embedding, LayerNorm, segment quantization, attention and log-softmax/top-k
// kernels. Pinned float orders: P1 lane-strided warp sums with
// xor butterfly, P2 512-thread block sums, P3 sequential dot products,
// context sums in key order, Cephes exp/log (detmath.cuh).
#include <climits>
#include <map>
#include <mutex>
#include <string>

#include "detmath.cuh"
#include "errors.hpp"
#include "launch.cuh"
#include "kernels.cuh"
#include "rowops.cuh"

namespace mtg {

namespace {

#define kNegInf (-__int_as_float(0x7f800000))

// Writes row r of an operand from x[0..n) with `stride`-spaced workers
// (a warp: lane/32, a CTA: tid/blockDim). scale is used for int8 only.
__device__ __forceinline__ void write_operand(const OperandOut& o, long long r, const float* x,
                                              int n, float scale, int tid, int stride) {
  if (o.prec < 0) return;  // no operand (the consumer converts the fp32 row itself)
  if (o.prec == 0) {
    int8_t* q = o.q + r * o.k_pad;
    for (int c = tid; c < o.k_pad; c += stride) q[c] = c < n ? quant1(x[c], scale) : 0;
    if (tid == 0) o.row_scale[r] = scale;
  } else if (o.prec == 1) {
    __nv_bfloat16* h = o.h + r * o.k_pad;
    for (int c = tid; c < o.k_pad; c += stride) h[c] = __float2bfloat16_rn(c < n ? x[c] : 0.0f);
  } else if (o.prec == 3) {  // plain fp32 (split into tf32 hi + lo by the GEMM)
    float* h = o.hi + r * o.k_pad;
    for (int c = tid; c < o.k_pad; c += stride) h[c] = c < n ? x[c] : 0.0f;
  } else {
    float* hi = o.hi + r * o.k_pad;
    float* lo = o.lo + r * o.k_pad;
    for (int c = tid; c < o.k_pad; c += stride) {
      const float v = c < n ? x[c] : 0.0f;
      uint32_t hb;
      asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(v));
      const float hf = __uint_as_float(hb);
      hi[c] = hf;
      lo[c] = __fsub_rn(v, hf);
    }
  }
}

// ---- embeddings -------------------------------------------------------------------

__global__ void embed_src_kernel(const int* __restrict__ ids, const int* __restrict__ pos,
                                 SrcEmbed se, int d, float sqrt_d, const float* __restrict__ pe,
                                 float* __restrict__ out, long long ldo) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x;
  const float* w = se.word + static_cast<long long>(ids[r]) * se.wdim;
  const float* p = pe + static_cast<long long>(pos[r]) * d;
  float* o = out + r * ldo;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float e;
    if (se.n_factors == 0) {
      e = w[c];
    } else if (se.mode == 0) {  // concat_cols(word, f0, f1, ...)
      if (c < se.wdim) {
        e = w[c];
      } else {
        int cc = c - se.wdim, f = 0;
        while (f + 1 < se.n_factors && cc >= se.fdim[f]) cc -= se.fdim[f++];
        e = se.table[f][static_cast<long long>(se.fids[f * se.fstride + r]) * se.fdim[f] + cc];
      }
    } else {  // add(word, f0), add(., f1), ...; average scales by 1/(1+F)
      e = w[c];
      for (int f = 0; f < se.n_factors; ++f)
        e = __fadd_rn(e, se.table[f][static_cast<long long>(se.fids[f * se.fstride + r]) *
                                         se.fdim[f] + c]);
      if (se.mode == 2) e = __fmul_rn(e, se.avg_scale);
    }
    o[c] = __fadd_rn(__fmul_rn(e, sqrt_d), p[c]);
  }
}

__global__ void embed_tgt_kernel(const int* __restrict__ prev, const int* d_rows,
                                 const int* d_step, const float* __restrict__ table,
                                 const int8_t* __restrict__ table_q, float q_scale, int d,
                                 float sqrt_d, const float* __restrict__ pe,
                                 float* __restrict__ out, long long ldo) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x;
  if (r >= *d_rows) return;
  const int t = *d_step;
  const long long id = prev[r];
  const float* p = pe + static_cast<long long>(t) * d;
  float* o = out + r * ldo;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    const float e = table_q ? __fdiv_rn(static_cast<float>(table_q[id * d + c]), q_scale)
                            : table[id * d + c];
    o[c] = __fadd_rn(__fmul_rn(e, sqrt_d), p[c]);
  }
}

// ---- layer norm (P1 sums) ---------------------------------------------------------------

// Row value c = lane + 32 i kept in registers (n <= 32*KPL): one pass over
// HBM, no reload-after-store. Same P1 order as the generic kernel.
// LayerNorm of one row held in registers (value c = lane + 32 i, n <= 32*KPL)
// by one warp; writes y (optional), rowmax (optional) and the next GEMM's
// operand (optional). P1 sums.
template <int KPL>
__device__ __forceinline__ void ln_row_regs(float (&xv)[KPL], const float (&gv)[KPL],
                                            const float (&bv)[KPL], int n, int lane, long long r,
                                            float* __restrict__ y, long long ldy,
                                            float* __restrict__ rowmax, const OperandOut& op,
                                            int has_op) {
  int bad = 0;
  const float mx = ln_normalize_regs<KPL>(xv, gv, bv, n, lane, &bad);
  if (y) {
    float* yr = y + r * ldy;
#pragma unroll
    for (int i = 0; i < KPL; ++i)
      if (lane + 32 * i < n) yr[lane + 32 * i] = xv[i];
  }
  if (rowmax && lane == 0) rowmax[r] = mx;
  if (!has_op) return;
  if (op.prec == 0) {
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicExch(op.nonfinite, 1);
    const float scale = qscale_of(mx);
    int8_t* q = op.q + r * op.k_pad;
#pragma unroll
    for (int i = 0; i < KPL; ++i) {
      const int c = lane + 32 * i;
      if (c < op.k_pad) q[c] = c < n ? quant1(xv[i], scale) : 0;
    }
    for (int c = 32 * KPL + lane; c < op.k_pad; c += 32) q[c] = 0;
    if (lane == 0) op.row_scale[r] = scale;
  } else if (op.prec == 1) {
    __nv_bfloat16* h = op.h + r * op.k_pad;
#pragma unroll
    for (int i = 0; i < KPL; ++i) {
      const int c = lane + 32 * i;
      if (c < op.k_pad) h[c] = __float2bfloat16_rn(c < n ? xv[i] : 0.0f);
    }
    for (int c = 32 * KPL + lane; c < op.k_pad; c += 32) h[c] = __float2bfloat16_rn(0.0f);
  } else if (op.prec == 3) {  // plain fp32
    float* h = op.hi + r * op.k_pad;
#pragma unroll
    for (int i = 0; i < KPL; ++i) {
      const int c = lane + 32 * i;
      if (c < op.k_pad) h[c] = c < n ? xv[i] : 0.0f;
    }
    for (int c = 32 * KPL + lane; c < op.k_pad; c += 32) h[c] = 0.0f;
  } else {
    float* hi = op.hi + r * op.k_pad;
    float* lo = op.lo + r * op.k_pad;
#pragma unroll
    for (int i = 0; i < KPL; ++i) {
      const int c = lane + 32 * i;
      if (c < op.k_pad) {
        const float v = c < n ? xv[i] : 0.0f;
        uint32_t hb;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(v));
        hi[c] = __uint_as_float(hb);
        lo[c] = __fsub_rn(v, __uint_as_float(hb));
      }
    }
    for (int c = 32 * KPL + lane; c < op.k_pad; c += 32) {
      hi[c] = 0.0f;
      lo[c] = 0.0f;
    }
  }
}

// Row value c = lane + 32 i kept in registers (n <= 32*KPL): one pass over
// HBM, no reload-after-store. Same P1 order as the generic kernel.
template <int KPL>
__global__ void layernorm_reg_kernel(const float* __restrict__ x, long long ldx, int max_rows,
                                     const int* d_rows, int n, const float* __restrict__ g,
                                     const float* __restrict__ b, float* __restrict__ y,
                                     long long ldy, float* __restrict__ rowmax, OperandOut op,
                                     int has_op) {
  pdl_wait();
  pdl_trigger();
  trace_begin(op.tr);
  const int rows = d_rows ? *d_rows : max_rows;
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float* xr = x + r * ldx;
  float xv[KPL], gv[KPL], bv[KPL];  // gain/bias loaded up front with x
#pragma unroll
  for (int i = 0; i < KPL; ++i) {
    const int c = lane + 32 * i;
    xv[i] = c < n ? xr[c] : 0.0f;
    gv[i] = c < n ? g[c] : 0.0f;
    bv[i] = c < n ? b[c] : 0.0f;
  }
  ln_row_regs<KPL>(xv, gv, bv, n, lane, r, y, ldy, rowmax, op, has_op);
  trace_end(op.tr);
}

// First kernel of a decode step, one warp per live row r:
//  * (reorder) copy the parent's ancestor / token history into row r
//    (decode.cpp:82-86 hypothesis copy) when step >= 1 and reorder != 0;
//  * target embedding of the previous token + positional encoding
//    (model.cpp:600-612), written to the residual stream x;
//  * the first decoder LayerNorm, written as the next GEMM's operand.
template <int KPL>
__global__ void step_begin_kernel(StepBegin sb, const float* __restrict__ g,
                                  const float* __restrict__ bln, OperandOut op) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= *sb.d_rows) return;
  const int t = *sb.d_step;
  const int n = sb.d;
  const long long id = sb.prev[r];
  const bool reo = sb.reorder && t >= 1;
  const int pr = reo ? sb.row_parent[r] : 0;
  float xv[KPL], gv[KPL], bv[KPL];
  const float* pe = sb.pe + static_cast<long long>(t) * n;
#pragma unroll
  for (int i = 0; i < KPL; ++i) {
    const int c = lane + 32 * i;
    float e = 0.0f;
    if (c < n)
      e = sb.table_q ? __fdiv_rn(static_cast<float>(sb.table_q[id * n + c]), sb.q_scale)
                     : sb.table[id * n + c];
    xv[i] = c < n ? __fadd_rn(__fmul_rn(e, sb.sqrt_d), pe[c]) : 0.0f;
    gv[i] = c < n ? g[c] : 0.0f;
    bv[i] = c < n ? bln[c] : 0.0f;
  }
  if (reo) {  // all history loads first, then the stores
    const int T = sb.T;
    const int cur = (t - 1) & 1, nxt = t & 1;
    const int* ac = sb.anc[cur] + static_cast<long long>(pr) * T;
    int* an = sb.anc[nxt] + static_cast<long long>(r) * T;
    const int* tc = sb.tok[cur] + static_cast<long long>(pr) * T;
    int* tn = sb.tok[nxt] + static_cast<long long>(r) * T;
    const int na = min(t, T), nt = t - 1;
    constexpr int kH = 4;
    int av[kH], tv[kH];
#pragma unroll
    for (int k = 0; k < kH; ++k) {
      const int j = lane + 32 * k;
      av[k] = j < na ? ac[j] : 0;
      tv[k] = j < nt ? tc[j] : 0;
    }
#pragma unroll
    for (int k = 0; k < kH; ++k) {
      const int j = lane + 32 * k;
      if (j < na) an[j] = av[k];
      if (j < nt) tn[j] = tv[k];
    }
    for (int j = 32 * kH + lane; j < na; j += 32) an[j] = ac[j];
    for (int j = 32 * kH + lane; j < nt; j += 32) tn[j] = tc[j];
    if (lane == 0) {
      if (t < T) an[t] = r;
      if (t - 1 < T) tn[t - 1] = static_cast<int>(id);
    }
  }
  float* xr = sb.x + r * sb.ldx;
#pragma unroll
  for (int i = 0; i < KPL; ++i)
    if (lane + 32 * i < n) xr[lane + 32 * i] = xv[i];
  ln_row_regs<KPL>(xv, gv, bv, n, lane, r, nullptr, 0, nullptr, op, 1);
}

__global__ void layernorm_kernel(const float* __restrict__ x, long long ldx, int max_rows,
                                 const int* d_rows, int n, const float* __restrict__ g,
                                 const float* __restrict__ b, float* __restrict__ y,
                                 long long ldy, float* __restrict__ rowmax, OperandOut op,
                                 int has_op) {
  pdl_wait();
  pdl_trigger();
  const int rows = d_rows ? *d_rows : max_rows;
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float* xr = x + r * ldx;
  float part = 0.0f;
  for (int c = lane; c < n; c += 32) part = __fadd_rn(part, xr[c]);
  const float nf = static_cast<float>(n);
  const float mu = __fdiv_rn(warp_allsum(part), nf);
  float part2 = 0.0f;
  for (int c = lane; c < n; c += 32) {
    const float dv = __fsub_rn(xr[c], mu);
    part2 = __fadd_rn(part2, __fmul_rn(dv, dv));
  }
  const float var = __fdiv_rn(warp_allsum(part2), nf);
  const float inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var, 1e-5f)));
  // y is optional (decoder LayerNorms only feed the next GEMM): the operand
  // pass recomputes the normalized values instead of re-reading y.
  auto norm = [&](int c) {
    return __fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(xr[c], mu), inv), g[c]), b[c]);
  };
  float mx = 0.0f;
  int bad = 0;
  for (int c = lane; c < n; c += 32) {
    const float v = norm(c);
    if (y) y[r * ldy + c] = v;
    mx = fmaxf(mx, fabsf(v));
    bad |= !isfinite(v);
  }
  mx = warp_allmax(mx);
  if (rowmax && lane == 0) rowmax[r] = mx;
  if (has_op && op.prec >= 0) {
    if (op.prec == 0 && __any_sync(0xffffffffu, bad) && lane == 0) atomicExch(op.nonfinite, 1);
    const float scale = qscale_of(mx);
    for (int c = lane; c < op.k_pad; c += 32) {
      const float v = c < n ? norm(c) : 0.0f;
      if (op.prec == 0) {
        op.q[r * op.k_pad + c] = c < n ? quant1(v, scale) : 0;
      } else if (op.prec == 1) {
        op.h[r * op.k_pad + c] = __float2bfloat16_rn(v);
      } else if (op.prec == 3) {
        op.hi[r * op.k_pad + c] = v;
      } else {
        uint32_t hb;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(v));
        op.hi[r * op.k_pad + c] = __uint_as_float(hb);
        op.lo[r * op.k_pad + c] = __fsub_rn(v, __uint_as_float(hb));
      }
    }
    if (op.prec == 0 && lane == 0) op.row_scale[r] = scale;
  }
}

// ---- segment quantization ---------------------------------------------------------------

__global__ void rowmax_kernel(const float* __restrict__ x, long long ldx, int rows, int n,
                              float* __restrict__ rowmax, int* nonfinite) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float* xr = x + r * ldx;
  float m = 0.0f;
  int bad = 0;
  for (int c = lane; c < n; c += 32) {
    const float v = xr[c];
    bad |= !isfinite(v);
    m = fmaxf(m, fabsf(v));
  }
  m = warp_allmax(m);
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicExch(nonfinite, 1);
  if (lane == 0) rowmax[r] = m;
}

__global__ void quantize_seg_kernel(const float* __restrict__ x, long long ldx, int rows, int n,
                                    const int* __restrict__ row_seg,
                                    const int* __restrict__ seg_off,
                                    const float* __restrict__ rowmax, OperandOut op) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const int s = row_seg[r];
  float m = 0.0f;
  for (int i = seg_off[s] + lane; i < seg_off[s + 1]; i += 32) m = fmaxf(m, rowmax[i]);
  m = warp_allmax(m);
  write_operand(op, r, x + r * ldx, n, qscale_of(m), lane, 32);
}

// Encoder LayerNorm + int8 operand with one scale per sentence (the quantize
// call tensor is the sentence's [S x d] block, model.cpp:461-466): CTA per
// sentence. Pass 1 normalises each row (warp per row, P1 sums) into y and
// tracks max |y|; pass 2 quantizes with 127 / max. Also clears this
// sentence's abs-max slot for the kernels that accumulate into it later.
template <int KPL>
__global__ void __launch_bounds__(1024)
    ln_quant_sent_kernel(const float* __restrict__ x, long long ldx, const int* __restrict__ off,
                         int n, const float* __restrict__ g, const float* __restrict__ b,
                         float* __restrict__ y, long long ldy, OperandOut op,
                         unsigned* __restrict__ sent_absmax, int stage_rows) {
  pdl_wait();
  pdl_trigger();
  trace_begin(op.tr);
  if (threadIdx.x == 0) trace_phase(op.tr, 0);
  __shared__ float red[32];
  // Dynamic smem (stage_rows > 0): the sentence's normalized rows, so the
  // quantization pass after the sentence max reads them back from shared
  // memory instead of global (which measured ~4 us of the kernel's 8).
  extern __shared__ __align__(16) float ysm[];
  const int s = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int r0 = off[s], r1 = off[s + 1];
  const bool staged = stage_rows >= r1 - r0;
  // gain / bias in shared memory (in registers they push the 16-value rows
  // past the 64-register cap of 1024 threads: spills)
  __shared__ float gs[32 * KPL], bs[32 * KPL];
  for (int c = threadIdx.x; c < 32 * KPL; c += blockDim.x) {
    gs[c] = c < n ? g[c] : 0.0f;
    bs[c] = c < n ? b[c] : 0.0f;
  }
  __syncthreads();
  float mx = 0.0f;
  int bad = 0;
  for (int r = r0 + warp; r < r1; r += nw) {
    const float* xr = x + r * ldx;
    float xv[KPL];
#pragma unroll
    for (int i = 0; i < KPL; ++i) {
      const int c = lane + 32 * i;
      xv[i] = c < n ? xr[c] : 0.0f;
    }
    float part = 0.0f;
#pragma unroll
    for (int i = 0; i < KPL; ++i)
      if (lane + 32 * i < n) part = __fadd_rn(part, xv[i]);
    const float nf = static_cast<float>(n);
    const float mu = __fdiv_rn(warp_allsum(part), nf);
    float part2 = 0.0f;
#pragma unroll
    for (int i = 0; i < KPL; ++i)
      if (lane + 32 * i < n) {
        const float dv = __fsub_rn(xv[i], mu);
        part2 = __fadd_rn(part2, __fmul_rn(dv, dv));
      }
    const float var = __fdiv_rn(warp_allsum(part2), nf);
    const float inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var, 1e-5f)));
    float* yr = y + r * ldy;
#pragma unroll
    for (int i = 0; i < KPL; ++i) {
      const int c = lane + 32 * i;
      if (c < n) {
        const float v = __fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(xv[i], mu), inv), gs[c]), bs[c]);
        yr[c] = v;
        if (staged) ysm[(r - r0) * n + c] = v;
        mx = fmaxf(mx, fabsf(v));
        bad |= !isfinite(v);
      }
    }
  }
  mx = warp_allmax(mx);
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicExch(op.nonfinite, 1);
  if (lane == 0) red[warp] = mx;
  if (threadIdx.x == 0 && sent_absmax) sent_absmax[s] = 0u;
  if (lane == 0) trace_phase(op.tr, 1);
  __syncthreads();
  if (threadIdx.x == 0) trace_phase(op.tr, 2);
  float m = lane < nw ? red[lane] : 0.0f;
  m = warp_allmax(m);
  const float scale = qscale_of(m);
  for (int r = r0 + warp; r < r1; r += nw) {  // same warp re-reads its own rows
    const float* yr = staged ? ysm + (r - r0) * n : y + r * ldy;
    int8_t* q = op.q + static_cast<long long>(r) * op.k_pad;
#pragma unroll
    for (int i = 0; i < KPL; ++i) {
      const int c = lane + 32 * i;
      if (c < op.k_pad) q[c] = c < n ? quant1(yr[c], scale) : 0;
    }
    for (int c = 32 * KPL + lane; c < op.k_pad; c += 32) q[c] = 0;
    if (lane == 0) op.row_scale[r] = scale;
  }
  if (lane == 0) trace_phase(op.tr, 3);
  trace_end(op.tr);
}

// int8 operand of rows with one scale per sentence, from a per-sentence max
// |x| accumulated by the producing kernel (float bits, atomicMax).
__global__ void quantize_sent_kernel(const float* __restrict__ x, long long ldx, int rows, int n,
                                     const int* __restrict__ row_seg,
                                     const unsigned* __restrict__ sent_absmax, OperandOut op) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float m = __uint_as_float(sent_absmax[row_seg[r]]);
  write_operand(op, r, x + r * ldx, n, qscale_of(m), lane, 32);
}

// Register-resident variant (n % 4 == 0, n <= 128 * V4, 16-byte aligned
// rows, int8 operand): lane owns elements 4 lane + 128 i, loaded as float4
// all at once (one round trip; the scalar loop above waits on one load per
// element group), quantized into 32-bit stores.
template <int V4>
__global__ void quantize_sent_vec_kernel(const float* __restrict__ x, long long ldx, int rows,
                                         int n, const int* __restrict__ row_seg,
                                         const unsigned* __restrict__ sent_absmax,
                                         OperandOut op) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float* xr = x + r * ldx;
  float4 v[V4];
#pragma unroll
  for (int i = 0; i < V4; ++i) {
    const int c = 4 * lane + 128 * i;
    v[i] = c < n ? *reinterpret_cast<const float4*>(xr + c) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const float scale = qscale_of(__uint_as_float(sent_absmax[row_seg[r]]));
  int8_t* qr = op.q + static_cast<long long>(r) * op.k_pad;
#pragma unroll
  for (int i = 0; i < V4; ++i) {
    const int c = 4 * lane + 128 * i;
    if (c < op.k_pad) {
      const uint32_t w = static_cast<uint32_t>(static_cast<uint8_t>(quant1(v[i].x, scale))) |
                         (static_cast<uint32_t>(static_cast<uint8_t>(quant1(v[i].y, scale))) << 8) |
                         (static_cast<uint32_t>(static_cast<uint8_t>(quant1(v[i].z, scale))) << 16) |
                         (static_cast<uint32_t>(static_cast<uint8_t>(quant1(v[i].w, scale))) << 24);
      *reinterpret_cast<uint32_t*>(qr + c) = w;  // columns >= n hold quantized zeros
    }
  }
  for (int c = 128 * V4 + 4 * lane; c < op.k_pad; c += 128) *reinterpret_cast<uint32_t*>(qr + c) = 0u;
  if (lane == 0) op.row_scale[r] = scale;
}

// ---- attention ---------------------------------------------------------------------------

// Shared-memory float4 load the compiler cannot hoist out of the key loop
// (keeping q in registers would spill at the 80-register occupancy target).
__device__ __forceinline__ float4 lds_f4(const float* p) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(static_cast<unsigned>(__cvta_generic_to_shared(p))));
  return v;
}

// One query against n keys, one warp. q: dh floats in smem (16-byte aligned);
// s: n floats of per-warp smem scratch. P3 dots, P1 softmax denominator,
// context summed over keys in ascending order per column. DH > 0 fixes the head dim at compile time (float4 paths, all
// of a key row's loads issued before its dot product); DH == 0 is generic.
// Key/value rows must be 16-byte aligned when DH % 4 == 0.
template <int DH, class KP, class VP>
__device__ __forceinline__ void attend_warp(const float* q, int n, int dh_rt, float scale, KP kp,
                                            VP vp, float* s, float* out,
                                            float* last = nullptr) {
  const int lane = threadIdx.x & 31;
  const int dh = DH > 0 ? DH : dh_rt;
  constexpr bool kVec = DH > 0 && DH % 4 == 0;
  float mx = kNegInf;
  for (int j = lane; j < n; j += 32) {
    const float* k = kp(j);
    float acc = 0.0f;
    if constexpr (kVec) {
      constexpr int G = DH / 4 < 16 ? DH / 4 : 16;  // float4 loads in flight per group
#pragma unroll
      for (int g = 0; g < DH / 4; g += G) {
        float4 kv[G];
#pragma unroll
        for (int i = 0; i < G; ++i) kv[i] = *reinterpret_cast<const float4*>(k + 4 * (g + i));
#pragma unroll
        for (int i = 0; i < G; ++i) {
          const float4 qv = lds_f4(q + 4 * (g + i));
          acc = __fadd_rn(acc, __fmul_rn(qv.x, kv[i].x));
          acc = __fadd_rn(acc, __fmul_rn(qv.y, kv[i].y));
          acc = __fadd_rn(acc, __fmul_rn(qv.z, kv[i].z));
          acc = __fadd_rn(acc, __fmul_rn(qv.w, kv[i].w));
        }
      }
    } else {
      for (int c = 0; c < dh; ++c) acc = __fadd_rn(acc, __fmul_rn(q[c], k[c]));
    }
    const float v = __fmul_rn(acc, scale);
    s[j] = v;
    mx = fmaxf(mx, v);
  }
  mx = warp_allmax(mx);
  float part = 0.0f;
  for (int j = lane; j < n; j += 32) {
    const float e = det_expf_nonpos(__fsub_rn(s[j], mx));
    s[j] = e;
    part = __fadd_rn(part, e);
  }
  const float sum = warp_allsum(part);
  for (int j = lane; j < n; j += 32) s[j] = __fdiv_rn(s[j], sum);
  __syncwarp();
  // Context: lane owns columns lane, lane + 32, ... and walks the keys in
  // ascending order (ctx[c] = sum_j p_j * v_j[c], oracle attend_row).
#pragma unroll 1
  for (int c0 = 0; c0 < dh; c0 += 64) {
    const int ca = c0 + lane, cb = c0 + 32 + lane;
    float acc_a = 0.0f, acc_b = 0.0f;
    for (int j = 0; j < n; ++j) {
      const float p = s[j];
      const float* v = vp(j);
      if (ca < dh) acc_a = __fadd_rn(acc_a, __fmul_rn(p, v[ca]));
      if (cb < dh) acc_b = __fadd_rn(acc_b, __fmul_rn(p, v[cb]));
    }
    if (ca < dh) out[ca] = acc_a;
    if (cb < dh) out[cb] = acc_b;
    if (last) {  // the lane's values of the last column block (all of them for dh <= 64)
      last[0] = acc_a;
      last[1] = acc_b;
    }
  }
  __syncwarp();
}

__host__ __device__ constexpr int enc_kv_pitch(int dh) { return dh % 4 == 0 ? dh + 4 : dh + 1; }
constexpr int kEncNQ = 4;  // queries per warp attended together (sentences <= 32 tokens)

// Encoder self-attention (model.cpp:418-470 / attention): CTA per (sentence,
// head). K and V are staged once in smem (row pitch dh+4: conflict-free
// float4 reads with lane = key); warps take queries round-robin.
template <int DH>
__global__ void enc_attention_kernel(const float* __restrict__ qkv, long long ldq,
                                     const int* __restrict__ off, int d, int dh_rt, int max_len,
                                     float scale, float* __restrict__ ctx, long long ldc,
                                     float* __restrict__ ctx_lo,
                                     unsigned* __restrict__ sent_absmax, int* nonfinite,
                                     KTrace tr, int out_bf16) {
  pdl_wait();
  pdl_trigger();
  trace_begin(tr);
  if (threadIdx.x == 0) trace_phase(tr, 0);
  extern __shared__ __align__(16) float sm[];
  const int dh = DH > 0 ? DH : dh_rt;
  const int P = enc_kv_pitch(dh);
  const int s = blockIdx.x, h = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int r0 = off[s], n = off[s + 1] - r0;
  // Queries, keys and values of the (sentence, head) staged together (one
  // round trip; a per-query load of q cost a dependent L2 trip per query).
  float* Ks = sm;
  float* Vs = Ks + max_len * P;
  float* Qs = Vs + max_len * P;
  float* ss = Qs + max_len * P + warp * kEncNQ * ((max_len + 3) & ~3);
  float* gscratch = Qs + max_len * P + nw * kEncNQ * ((max_len + 3) & ~3) + warp * 64;
  const float* base = qkv + static_cast<long long>(r0) * ldq + h * dh;
  if constexpr (DH > 0 && DH % 4 == 0) {
    constexpr int Q4 = DH / 4;
    for (int idx = threadIdx.x; idx < n * Q4; idx += blockDim.x) {
      const int j = idx / Q4, c = 4 * (idx - j * Q4);
      const float4 kq = *reinterpret_cast<const float4*>(base + j * ldq + d + c);
      const float4 vq = *reinterpret_cast<const float4*>(base + j * ldq + 2 * d + c);
      const float4 qq = *reinterpret_cast<const float4*>(base + j * ldq + c);
      *reinterpret_cast<float4*>(Ks + j * P + c) = kq;
      *reinterpret_cast<float4*>(Vs + j * P + c) = vq;
      *reinterpret_cast<float4*>(Qs + j * P + c) = qq;
    }
  } else {
    for (int idx = threadIdx.x; idx < n * dh; idx += blockDim.x) {
      const int j = idx / dh, c = idx - j * dh;
      Ks[j * P + c] = base[j * ldq + d + c];
      Vs[j * P + c] = base[j * ldq + 2 * d + c];
      Qs[j * P + c] = base[j * ldq + c];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) trace_phase(tr, 1);
  float mx = 0.0f;
  int bad = 0;
  // Handles the epilogue of one context value pair of query row i (fp32
  // context, sentence max / non-finite for int8, TF32 hi + lo for fp32).
  auto finish = [&](int i, float va, float vb) {
    float* out = ctx + static_cast<long long>(r0 + i) * ldc + h * dh;
    if (out_bf16) {  // ctx is the bf16 operand of the Wo GEMM (reinterpreted)
      __nv_bfloat16* o =
          reinterpret_cast<__nv_bfloat16*>(ctx) + static_cast<long long>(r0 + i) * ldc + h * dh;
      o[lane] = __float2bfloat16_rn(va);
      o[lane + 32] = __float2bfloat16_rn(vb);
      return;
    }
    if (sent_absmax) {
      mx = fmaxf(mx, fmaxf(fabsf(va), fabsf(vb)));
      bad |= !isfinite(va) | !isfinite(vb);
    }
    if (ctx_lo) {
      float* lo = ctx_lo + (out - ctx);
      const float vv[2] = {va, vb};
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        uint32_t hb;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(vv[u]));
        out[lane + 32 * u] = __uint_as_float(hb);
        lo[lane + 32 * u] = __fsub_rn(vv[u], __uint_as_float(hb));
      }
    } else {
      out[lane] = va;
      out[lane + 32] = vb;
    }
  };
  // Queries of this CTA: blockIdx.z of gridDim.z query groups (more CTAs
  // for batches of few sentences); warp-global index gw of TW warps.
  const int TW = nw * static_cast<int>(gridDim.z);
  const int gw = static_cast<int>(blockIdx.z) * nw + warp;
  bool multi = false;
  if constexpr (DH == 64) {
    if (n <= 32 && n <= TW * kEncNQ) {
      multi = true;
      // Short sentences (n <= 32 keys): each warp attends its up to kEncNQ
      // queries together -- lane = key for the scores, lane = column pair for
      // the contexts -- so every key / value load serves all of them and the
      // queries' dependent chains interleave. Per (query, key) the arithmetic
      // is attend_warp's: P3 dot over the head dimension, P1 softmax (one key
      // per lane, then the butterfly), context summed over keys in order.
      // this warp's queries: gw + k TW (query groups over gridDim.z CTAs)
      const int nq = gw < n ? (n - gw + TW - 1) / TW : 0;
      const float* kr = Ks + lane * P;          // rows past n: ignored
      float acc[kEncNQ];
#pragma unroll
      for (int k = 0; k < kEncNQ; ++k) acc[k] = 0.0f;
#pragma unroll
      for (int c4 = 0; c4 < DH / 4; ++c4) {
        const float4 kv = lds_f4(kr + 4 * c4);
#pragma unroll
        for (int k = 0; k < kEncNQ; ++k) {
          if (k < nq) {
            const float4 qv = lds_f4(Qs + (gw + k * TW) * P + 4 * c4);
            acc[k] = __fadd_rn(acc[k], __fmul_rn(qv.x, kv.x));
            acc[k] = __fadd_rn(acc[k], __fmul_rn(qv.y, kv.y));
            acc[k] = __fadd_rn(acc[k], __fmul_rn(qv.z, kv.z));
            acc[k] = __fadd_rn(acc[k], __fmul_rn(qv.w, kv.w));
          }
        }
      }
      const int W4 = (max_len + 3) & ~3;
#pragma unroll
      for (int k = 0; k < kEncNQ; ++k) {
        if (k < nq) {
          const float v = __fmul_rn(acc[k], scale);
          const float m = warp_allmax(lane < n ? v : kNegInf);
          const float e = lane < n ? det_expf_nonpos(__fsub_rn(v, m)) : 0.0f;
          const float sum = warp_allsum(lane < n ? __fadd_rn(0.0f, e) : 0.0f);
          if (lane < n) ss[k * W4 + lane] = __fdiv_rn(e, sum);
        }
      }
      __syncwarp();
      float ca[kEncNQ], cb[kEncNQ];
#pragma unroll
      for (int k = 0; k < kEncNQ; ++k) ca[k] = cb[k] = 0.0f;
      for (int j = 0; j < n; ++j) {
        const float* vr = Vs + j * P;
        const float va = vr[lane], vb = vr[32 + lane];
#pragma unroll
        for (int k = 0; k < kEncNQ; ++k) {
          if (k < nq) {
            const float pj = ss[k * W4 + j];
            ca[k] = __fadd_rn(ca[k], __fmul_rn(pj, va));
            cb[k] = __fadd_rn(cb[k], __fmul_rn(pj, vb));
          }
        }
      }
#pragma unroll
      for (int k = 0; k < kEncNQ; ++k)
        if (k < nq) finish(gw + k * TW, ca[k], cb[k]);
      __syncwarp();
    }
  }
  for (int i = multi ? n : gw; i < n; i += TW) {
    const float* qs = Qs + i * P;
    float* out = out_bf16 ? gscratch : ctx + static_cast<long long>(r0 + i) * ldc + h * dh;
    float vals[2];
    attend_warp<DH>(
        qs, n, dh, scale, [&](int j) { return Ks + j * P; }, [&](int j) { return Vs + j * P; },
        ss, out, vals);
    if (out_bf16) {  // dh == 64 (host): the values are in registers
      finish(i, vals[0], vals[1]);
      continue;
    }
    // dh <= 64: the lane's two context values are still in registers (a
    // read-back of the just-written global row costs a round trip per query)
    if (dh <= 64) {
      const float va = lane < dh ? vals[0] : 0.0f, vb = 32 + lane < dh ? vals[1] : 0.0f;
      if (sent_absmax) {
        mx = fmaxf(mx, fmaxf(fabsf(va), fabsf(vb)));
        bad |= (lane < dh && !isfinite(va)) | (32 + lane < dh && !isfinite(vb));
      }
      if (ctx_lo) {
        float* lo = ctx_lo + (out - ctx);
        const float vv[2] = {va, vb};
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int c = lane + 32 * u;
          if (c < dh) {
            uint32_t hb;
            asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(vv[u]));
            out[c] = __uint_as_float(hb);
            lo[c] = __fsub_rn(vv[u], __uint_as_float(hb));
          }
        }
      }
      continue;
    }
    if (sent_absmax) {
      for (int c = lane; c < dh; c += 32) {  // lane wrote these itself
        mx = fmaxf(mx, fabsf(out[c]));
        bad |= !isfinite(out[c]);
      }
    }
    if (ctx_lo) {  // fp32 path: the context row is the next GEMM's hi + lo operand
      float* lo = ctx_lo + (out - ctx);
      for (int c = lane; c < dh; c += 32) {
        const float v = out[c];
        uint32_t hb;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(v));
        out[c] = __uint_as_float(hb);
        lo[c] = __fsub_rn(v, __uint_as_float(hb));
      }
    }
  }
  if (lane == 0) trace_phase(tr, 2);
  if (sent_absmax) {  // the quantize call tensor is the sentence's context block
    mx = warp_allmax(mx);
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicExch(nonfinite, 1);
    if (lane == 0) atomicMax(sent_absmax + s, __float_as_uint(mx));
  }
  trace_end(tr);
}

// CTA epilogue shared by the decoder attention kernels: the context row sits
// in smem (d floats, one slice per head-warp); write fp32 and the operand.
__device__ __forceinline__ void finish_ctx_row(const float* row, int d, long long r, float* ctx,
                                               long long ldc, const OperandOut& op, float* red) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  float m = 0.0f;
  int bad = 0;
  for (int c = tid; c < d; c += blockDim.x) {
    const float v = row[c];
    ctx[r * ldc + c] = v;
    m = fmaxf(m, fabsf(v));
    bad |= !isfinite(v);
  }
  m = warp_allmax(m);
  bad = __any_sync(0xffffffffu, bad);
  if (lane == 0) red[warp] = m;
  if (bad && lane == 0 && op.prec == 0) atomicExch(op.nonfinite, 1);
  __syncthreads();
  if (warp == 0) {
    float v = lane < nw ? red[lane] : 0.0f;
    v = warp_allmax(v);
    if (lane == 0) red[32] = v;
  }
  __syncthreads();
  write_operand(op, r, row, d, qscale_of(red[32]), tid, blockDim.x);
}

__host__ __device__ constexpr int round4(int x) { return (x + 3) & ~3; }

// ---- staged decoder attention (head dim 64) ----------------------------------
// Key and value rows are copied global -> shared with cp.async, a whole row
// per half-warp (coalesced), into a per-warp stage with an XOR swizzle of the
// 16-byte columns, so the lane-per-key reads that follow are conflict-free.
// Same arithmetic (P3 dots, P1 softmax, key-ordered context) as attend_warp<64>.
constexpr int kStageFloats = 32 * 64;  // one 32-key chunk of 64-float rows

__device__ __forceinline__ void cp_async16(float* smem_dst, const float* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   static_cast<unsigned>(__cvta_generic_to_shared(smem_dst))),
               "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_warp() {
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncwarp();
}

// Rows c0 .. c0+31 (< n) as [32][64]; float4 column c of row jr at c ^ (jr & 15).
template <class KP>
__device__ __forceinline__ void stage_rows64(float* stage, int c0, int n, KP kp, int lane) {
  const int c = lane & 15, half = lane >> 4;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int jr = 2 * i + half, j = c0 + jr;
    if (j < n) cp_async16(stage + jr * 64 + ((c ^ (jr & 15)) << 2), kp(j) + 4 * c);
  }
  cp_async_commit();
}

// Row j (stage row jr) alone, by lanes 0-15, as its own cp.async group.
__device__ __forceinline__ void stage_row64(float* stage, int jr, const float* src, int lane) {
  if (lane < 16) cp_async16(stage + jr * 64 + ((lane ^ (jr & 15)) << 2), src + 4 * lane);
  cp_async_commit();
}

// L2 prefetch of rows c0 .. c0+31 (< n), 256 B each (lane = row).
template <class VP>
__device__ __forceinline__ void prefetch_rows64(int c0, int n, VP vp, int lane) {
  if (c0 + lane < n)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], 256;" ::"l"(vp(c0 + lane)) : "memory");
}

// k0_staged: the caller already issued (committed) the copies of key chunk 0.
template <class KP, class VP>
__device__ __forceinline__ void attend_warp_staged64(const float* q, int n, float scale, KP kp,
                                                     VP vp, float* stage, float* s, float* out,
                                                     const KTrace* tr = nullptr,
                                                     bool k0_staged = false) {
  const int lane = threadIdx.x & 31;
  const bool ph = tr && lane == 0;
  float mx = kNegInf;
  for (int c0 = 0; c0 < n; c0 += 32) {
    if (!(k0_staged && c0 == 0)) stage_rows64(stage, c0, n, kp, lane);
    cp_async_wait_warp();
    if (ph && c0 == 0) trace_phase(*tr, 1);
    const int j = c0 + lane;
    if (j < n) {
      const float* kr = stage + lane * 64;
      float acc = 0.0f;
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const float4 kv = lds_f4(kr + ((c ^ (lane & 15)) << 2));
        const float4 qv = lds_f4(q + 4 * c);
        acc = __fadd_rn(acc, __fmul_rn(qv.x, kv.x));
        acc = __fadd_rn(acc, __fmul_rn(qv.y, kv.y));
        acc = __fadd_rn(acc, __fmul_rn(qv.z, kv.z));
        acc = __fadd_rn(acc, __fmul_rn(qv.w, kv.w));
      }
      const float v = __fmul_rn(acc, scale);
      s[j] = v;
      mx = fmaxf(mx, v);
    }
    __syncwarp();
  }
  if (ph) trace_phase(*tr, 2);
  stage_rows64(stage, 0, n, vp, lane);  // first value chunk overlaps the softmax
  mx = warp_allmax(mx);
  float part = 0.0f;
  for (int j = lane; j < n; j += 32) {
    const float e = det_expf_nonpos(__fsub_rn(s[j], mx));
    s[j] = e;
    part = __fadd_rn(part, e);
  }
  const float sum = warp_allsum(part);
  for (int j = lane; j < n; j += 32) s[j] = __fdiv_rn(s[j], sum);
  __syncwarp();
  // Context: lane owns columns lane and lane + 32 and walks the keys in
  // ascending order through the staged 32-key chunks (swizzled rows).
  const int ga = lane >> 2, gb = 8 + (lane >> 2), e4 = lane & 3;
  float acc_a = 0.0f, acc_b = 0.0f;
  for (int c0 = 0; c0 < n; c0 += 32) {
    if (c0 != 0) stage_rows64(stage, c0, n, vp, lane);
    cp_async_wait_warp();
    if (ph && c0 == 0) trace_phase(*tr, 3);
    const int nk = min(32, n - c0);
    for (int jr = 0; jr < nk; ++jr) {
      const float p = s[c0 + jr];
      const float* vr = stage + jr * 64;
      acc_a = __fadd_rn(acc_a, __fmul_rn(p, vr[((ga ^ (jr & 15)) << 2) + e4]));
      acc_b = __fadd_rn(acc_b, __fmul_rn(p, vr[((gb ^ (jr & 15)) << 2) + e4]));
    }
    __syncwarp();
  }
  out[lane] = acc_a;
  out[32 + lane] = acc_b;
  if (ph) trace_phase(*tr, 4);
  __syncwarp();
}

// Warps per decoder-attention CTA (matches __launch_bounds__(256, 3)); with
// more heads each warp attends several.
constexpr int kDecAttnWarps = 8;

// Per-warp smem floats of the decoder attention kernels.
__host__ __device__ constexpr int dec_attn_warp_floats(int dh, int nkeys) {
  return (dh == 64 ? kStageFloats : 0) + round4(dh) + round4(nkeys);
}

// Decoder self-attention over the cached prefix (model.cpp:620-660): CTA per
// hypothesis row, warp per head; key j of row r lives at cache row
// anc[r][j] of step j. Smem: per-head [q | scores] blocks (16-byte aligned),
// then the context row, the reduction scratch and the ancestor row.
template <int DH>
__global__ void __launch_bounds__(256, 3)
    dec_self_attention_kernel(const float* __restrict__ cache, int r_max, int T,
                              const int* __restrict__ anc0, const int* __restrict__ anc1,
                              const int* d_rows, const int* d_step, int d, int dh_rt, float scale,
                              float* __restrict__ ctx, long long ldc, OperandOut op, int early,
                              HistReorder hist) {
  extern __shared__ __align__(16) float sm[];
  const int r = blockIdx.x;
  // early bit 0: before the dependency wait, the row count, step and ancestry
  // (written by the previous step's tail and the step-start reorder, two or
  // more kernels back) and an L2 prefetch of the cached keys / values of
  // positions < t (bit 1; 4 KB per position: k | v of all heads), which the QKV GEMM
  // running in front of this kernel does not touch. early = 0 (the reorder
  // ran in the kernel just before): all of it after the wait.
  if (!early) pdl_wait();
  const int R = *d_rows;
  const int t = *d_step;
  if (r >= R) {
    if (early) pdl_wait();
    pdl_trigger();
    return;
  }
  const int dh = DH > 0 ? DH : dh_rt;
  // Warp w attends heads w, w + nw, ... (at most 8 warps per CTA).
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int heads = d / dh;
  const int W = dec_attn_warp_floats(DH > 0 ? DH : dh, T);
  float* stage = sm + warp * W;                              // [kStageFloats] (DH = 64)
  float* qs = stage + (DH == 64 ? kStageFloats : 0);
  float* ss = qs + round4(dh);
  float* row = sm + nw * W;                      // [d] context row
  float* red = row + d;                          // [33]
  int* arow = reinterpret_cast<int*>(red + 33);  // [T] ancestor rows
  const long long ld3 = 3LL * d;
  // With the folded reorder (hist.on, early only): positions < t from the
  // parent's table of step t-1, itself at t; the step's tables are written
  // here (nothing reads them before this kernel).
  const bool fold = hist.on && early && t >= 1;
  const int* ar = fold ? ((t - 1) & 1 ? anc1 : anc0) + static_cast<long long>(hist.row_parent[r]) * T
                       : ((t & 1) ? anc1 : anc0) + static_cast<long long>(r) * T;
  int* an = fold ? hist.anc[t & 1] + static_cast<long long>(r) * T : nullptr;
  if (fold) {
    const int* tc = hist.tok[(t - 1) & 1] + static_cast<long long>(hist.row_parent[r]) * T;
    int* tn = hist.tok[t & 1] + static_cast<long long>(r) * T;
    for (int j = threadIdx.x; j < t - 1; j += blockDim.x) tn[j] = tc[j];
    if (threadIdx.x == 0 && t - 1 < T) tn[t - 1] = hist.row_prev[r];
  }
  for (int j = threadIdx.x; j <= t; j += blockDim.x) {
    const int a = fold && j == t ? r : ar[j];
    arow[j] = a;
    if (fold && j < T) an[j] = a;
    if (j < t && (early & 2))
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                       cache + (static_cast<long long>(j) * r_max + a) * ld3 + d),
                   "r"(static_cast<unsigned>(2 * d * sizeof(float)))
                   : "memory");
  }
  __syncthreads();  // ancestry rows visible to every warp
  // Early (DH = 64): the first head's cached keys of chunk 0 (positions < t,
  // written in earlier steps) are copied now and its values prefetched into
  // L2; after the wait only the query and position t's key follow.
  const bool pre = DH == 64 && early && warp < heads;
  auto kp_of = [&](int h) {
    const float* kb = cache + d + h * dh;
    return [=](int j) { return kb + (static_cast<long long>(j) * r_max + arow[j]) * ld3; };
  };
  if (pre) {
    stage_rows64(stage, 0, min(t, 32), kp_of(warp), lane);
    const float* vb = cache + 2 * d + warp * dh;
    prefetch_rows64(
        0, min(t, 32),
        [=](int j) { return vb + (static_cast<long long>(j) * r_max + arow[j]) * ld3; }, lane);
  }
  if (early) pdl_wait();
  pdl_trigger();
  trace_begin(op.tr);
  if (threadIdx.x == 0) trace_phase(op.tr, 0);
  for (int h = warp; h < heads; h += nw) {
    const float* q = cache + (static_cast<long long>(t) * r_max + r) * ld3 + h * dh;
    const float* kb = cache + d + h * dh;
    auto kp = [&](int j) { return kb + (static_cast<long long>(j) * r_max + arow[j]) * ld3; };
    auto vp = [&](int j) { return kb + (static_cast<long long>(j) * r_max + arow[j]) * ld3 + d; };
    const bool k0 = pre && h == warp;
    if (k0 && t < 32) stage_row64(stage, t, kp(t), lane);  // this step's key (the QKV GEMM's)
    for (int c = lane; c < dh; c += 32) qs[c] = q[c];
    __syncwarp();
    if constexpr (DH == 64)
      attend_warp_staged64(qs, t + 1, scale, kp, vp, stage, ss, row + h * dh,
                           h == 0 ? &op.tr : nullptr, k0);
    else
      attend_warp<DH>(qs, t + 1, dh, scale, kp, vp, ss, row + h * dh);
    __syncwarp();
  }
  __syncthreads();
  if (threadIdx.x == 0) trace_phase(op.tr, 5);
  finish_ctx_row(row, d, r, ctx, ldc, op, red);
  trace_end(op.tr);
}

// Decoder cross-attention over the sentence's encoder keys/values.
template <int DH>
__global__ void __launch_bounds__(256, 3)
    dec_cross_attention_kernel(const float* __restrict__ cq, long long ldq,
                               const float* __restrict__ ckv, const int* __restrict__ row_sent,
                               const int* __restrict__ enc_off, const int* __restrict__ enc_len,
                               const int* d_rows, int max_src, int d, int dh_rt, float scale,
                               float* __restrict__ ctx, long long ldc, OperandOut op) {
  extern __shared__ __align__(16) float sm[];
  const int r = blockIdx.x;
  // Before the dependency wait: the row's sentence (beam state of the
  // previous step's tail) and, for the first head, the copies of the
  // encoder keys of chunk 0 plus an L2 prefetch of its values; after the
  // wait only the query (the cross-Wq GEMM's output).
  const int R = *d_rows;
  if (r >= R) {
    pdl_wait();
    pdl_trigger();
    return;
  }
  const int dh = DH > 0 ? DH : dh_rt;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int heads = d / dh;
  const int s = row_sent[r];
  const int n = enc_len[s];
  const long long off = static_cast<long long>(enc_off[s]) * 2 * d;
  const int W = dec_attn_warp_floats(DH > 0 ? DH : dh, max_src);
  float* stage = sm + warp * W;
  float* qs = stage + (DH == 64 ? kStageFloats : 0);
  float* ss = qs + round4(dh);
  float* row = sm + nw * W;
  float* red = row + d;
  const bool pre = DH == 64 && warp < heads;
  if (pre) {
    const float* kv = ckv + off + warp * dh;
    stage_rows64(stage, 0, n, [=](int j) { return kv + static_cast<long long>(j) * 2 * d; }, lane);
    prefetch_rows64(0, n, [=](int j) { return kv + static_cast<long long>(j) * 2 * d + d; }, lane);
  }
  pdl_wait();
  pdl_trigger();
  trace_begin(op.tr);
  for (int h = warp; h < heads; h += nw) {
    const float* kv = ckv + off + h * dh;
    for (int c = lane; c < dh; c += 32) qs[c] = cq[r * ldq + h * dh + c];
    __syncwarp();
    auto kp = [&](int j) { return kv + static_cast<long long>(j) * 2 * d; };
    auto vp = [&](int j) { return kv + static_cast<long long>(j) * 2 * d + d; };
    if constexpr (DH == 64)
      attend_warp_staged64(qs, n, scale, kp, vp, stage, ss, row + h * dh, nullptr,
                           pre && h == warp);
    else
      attend_warp<DH>(qs, n, dh, scale, kp, vp, ss, row + h * dh);
    __syncwarp();
  }
  __syncthreads();
  finish_ctx_row(row, d, r, ctx, ldc, op, red);
  trace_end(op.tr);
}

}  // namespace

// ---- launchers ------------------------------------------------------------------------------

void ensure_smem_attr(const void* fn, size_t bytes) {
  if (bytes > 227 * 1024) fail(kUsageError, "kernel shared memory above 227 KB");
  if (bytes <= 48 * 1024) return;
  int dev = 0;
  MTG_CUDA(cudaGetDevice(&dev));
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> cur;
  std::lock_guard<std::mutex> lock(mu);
  size_t& c = cur[{dev, fn}];
  if (bytes <= c) return;
  MTG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(bytes)));
  c = bytes;
}

namespace {
void set_smem_limit(const void* fn, size_t bytes, const char* what) {
  if (bytes > 227 * 1024) fail(kUsageError, std::string(what) + ": shared memory too large");
  ensure_smem_attr(fn, bytes);
}
}  // namespace

namespace {
__global__ void noop_kernel() {
  pdl_wait();
  pdl_trigger();
}
}  // namespace

void launch_noop(cudaStream_t st) {
  launch_k(noop_kernel, 148, 256, 0, st);
  MTG_CUDA(cudaGetLastError());
}

void launch_embed_src(const int* ids, const int* pos, int rows, const SrcEmbed& se, int d,
                      float sqrt_d, const float* pe, float* out, long long ldo, cudaStream_t st) {
  if (rows <= 0) return;
  if (se.n_factors > kMaxFactors) fail(kUsageError, "at most 4 source factors are supported");
  launch_k(embed_src_kernel, rows, 128, 0, st, ids, pos, se, d, sqrt_d, pe, out, ldo);
  MTG_CUDA(cudaGetLastError());
}

void launch_embed_tgt(const int* prev, const int* d_rows, int max_rows, const int* d_step,
                      const float* table, const int8_t* table_q, float q_scale, int d,
                      float sqrt_d, const float* pe, float* out, long long ldo, cudaStream_t st) {
  if (max_rows <= 0) return;
  launch_k(embed_tgt_kernel, max_rows, 128, 0, st, prev, d_rows, d_step, table, table_q, q_scale, d,
                                             sqrt_d, pe, out, ldo);
  MTG_CUDA(cudaGetLastError());
}

void launch_step_begin(const StepBegin& sb, int max_rows, const float* g, const float* b,
                       const OperandOut& op, cudaStream_t st) {
  if (max_rows <= 0) return;
  const int wpb = 4;
  const dim3 grid((max_rows + wpb - 1) / wpb), block(wpb * 32);
  const int kpl = (sb.d + 31) / 32;
  if (kpl <= 1)
    launch_k(step_begin_kernel<1>, grid, block, 0, st, sb, g, b, op);
  else if (kpl <= 4)
    launch_k(step_begin_kernel<4>, grid, block, 0, st, sb, g, b, op);
  else if (kpl <= 16)
    launch_k(step_begin_kernel<16>, grid, block, 0, st, sb, g, b, op);
  else
    fail(kUsageError, "step_begin: d_model above 512");
  MTG_CUDA(cudaGetLastError());
}

void launch_layernorm(const float* x, long long ldx, int max_rows, const int* d_rows, int n,
                      const float* g, const float* b, float* y, long long ldy, float* rowmax,
                      const OperandOut* op, cudaStream_t st) {
  if (max_rows <= 0) return;
  const int wpb = 4;
  const dim3 grid((max_rows + wpb - 1) / wpb), block(wpb * 32);
  const OperandOut o = op ? *op : OperandOut{};
  const int has = op ? 1 : 0;
  const int kpl = (n + 31) / 32;
  if (kpl <= 1)
    launch_k(layernorm_reg_kernel<1>, grid, block, 0, st, x, ldx, max_rows, d_rows, n, g, b, y, ldy,
                                                     rowmax, o, has);
  else if (kpl <= 4)
    launch_k(layernorm_reg_kernel<4>, grid, block, 0, st, x, ldx, max_rows, d_rows, n, g, b, y, ldy,
                                                     rowmax, o, has);
  else if (kpl <= 16)
    launch_k(layernorm_reg_kernel<16>, grid, block, 0, st, x, ldx, max_rows, d_rows, n, g, b, y, ldy,
                                                      rowmax, o, has);
  else
    launch_k(layernorm_kernel, grid, block, 0, st, x, ldx, max_rows, d_rows, n, g, b, y, ldy, rowmax, o,
                                             has);
  MTG_CUDA(cudaGetLastError());
}

void launch_rowmax(const float* x, long long ldx, int rows, int n, float* rowmax, int* nonfinite,
                   cudaStream_t st) {
  if (rows <= 0) return;
  const int wpb = 8;
  launch_k(rowmax_kernel, (rows + wpb - 1) / wpb, wpb * 32, 0, st, x, ldx, rows, n, rowmax, nonfinite);
  MTG_CUDA(cudaGetLastError());
}

template <class K, class... A>
static void launch_ln_quant_sent_k(K k, int n_sent, size_t smem, cudaStream_t st, A... args) {
  if (smem > 48 * 1024) ensure_smem_attr(k, smem);
  launch_k(k, n_sent, 1024, smem, st, args...);
}

void launch_ln_quant_sent(const float* x, long long ldx, const int* off, int n_sent, int n,
                          const float* g, const float* b, float* y, long long ldy,
                          const OperandOut& op, unsigned* sent_absmax, cudaStream_t st,
                          int max_rows) {
  if (n_sent <= 0) return;
  if (op.prec != 0) fail(kStateError, "ln_quant_sent: int8 operands only");
  const int kpl = (n + 31) / 32;
  // rows of a sentence staged in shared memory when the longest fits
  const int stage_rows = max_rows > 0 && size_t(max_rows) * n * sizeof(float) <= 96 * 1024 ? max_rows : 0;
  const size_t smem = size_t(stage_rows) * n * sizeof(float);
  if (kpl <= 1)
    launch_ln_quant_sent_k(ln_quant_sent_kernel<1>, n_sent, smem, st, x, ldx, off, n, g, b, y, ldy,
                           op, sent_absmax, stage_rows);
  else if (kpl <= 4)
    launch_ln_quant_sent_k(ln_quant_sent_kernel<4>, n_sent, smem, st, x, ldx, off, n, g, b, y, ldy,
                           op, sent_absmax, stage_rows);
  else if (kpl <= 16)
    launch_ln_quant_sent_k(ln_quant_sent_kernel<16>, n_sent, smem, st, x, ldx, off, n, g, b, y, ldy,
                           op, sent_absmax, stage_rows);
  else
    fail(kUsageError, "ln_quant_sent: d_model above 512");
  MTG_CUDA(cudaGetLastError());
}

void launch_quantize_sent(const float* x, long long ldx, int rows, int n, const int* row_seg,
                          const unsigned* sent_absmax, const OperandOut& op, cudaStream_t st) {
  if (rows <= 0) return;
  const int wpb = 8;
  const bool vec = op.prec == 0 && n % 4 == 0 && ldx % 4 == 0 && op.k_pad % 4 == 0 &&
                   reinterpret_cast<uintptr_t>(x) % 16 == 0;
  if (vec && n <= 512) {
    launch_k(quantize_sent_vec_kernel<4>, (rows + 3) / 4, 4 * 32, 0, st, x, ldx, rows, n, row_seg,
             sent_absmax, op);
  } else if (vec && n <= 2048) {
    launch_k(quantize_sent_vec_kernel<16>, (rows + 3) / 4, 4 * 32, 0, st, x, ldx, rows, n, row_seg,
             sent_absmax, op);
  } else {
    launch_k(quantize_sent_kernel, (rows + wpb - 1) / wpb, wpb * 32, 0, st, x, ldx, rows, n,
             row_seg, sent_absmax, op);
  }
  MTG_CUDA(cudaGetLastError());
}

void launch_quantize_seg(const float* x, long long ldx, int rows, int n, const int* row_seg,
                         const int* seg_off, const float* rowmax, const OperandOut& op,
                         cudaStream_t st) {
  if (rows <= 0) return;
  const int wpb = 8;
  launch_k(quantize_seg_kernel, (rows + wpb - 1) / wpb, wpb * 32, 0, st, x, ldx, rows, n, row_seg,
                                                                   seg_off, rowmax, op);
  MTG_CUDA(cudaGetLastError());
}

void launch_enc_attention(const float* qkv, long long ldq, const int* off, int n_sent,
                          int max_len, int d, int heads, float scale, float* ctx, long long ldc,
                          float* ctx_lo, unsigned* sent_absmax, int* nonfinite, cudaStream_t st,
                          const KTrace& tr, bool out_bf16) {
  if (n_sent <= 0) return;
  const int dh = d / heads;
  const int nw = 8;
  const int P = enc_kv_pitch(dh);
  const size_t smem =
      sizeof(float) * (size_t(max_len) * 3 * P + size_t(nw) * (kEncNQ * round4(max_len) + 64));
  if (smem > 227 * 1024)
    fail(kUsageError, "encoder attention: sentence x head dimension too large for smem");
  auto k = dh == 64 ? enc_attention_kernel<64> : enc_attention_kernel<0>;
  ensure_smem_attr(k, smem);
  // Few (sentence, head) CTAs (small batches): split each sentence's
  // queries over up to 4 CTAs, so more SMs attend (each stages the keys).
  int qg = 1;
  while (qg < 4 && n_sent * heads * qg * 2 <= 148 && max_len > nw * qg) qg *= 2;
  if (out_bf16 && dh != 64) fail(kStateError, "encoder attention: bf16 output needs head dim 64");
  launch_k(k, dim3(n_sent, heads, qg), nw * 32, smem, st, qkv, ldq, off, d, dh, max_len, scale,
           ctx, ldc, ctx_lo, sent_absmax, nonfinite, tr, out_bf16 ? 1 : 0);
  MTG_CUDA(cudaGetLastError());
}

void launch_dec_self_attention(const float* qkv_cache, int r_max, int T, const int* anc0,
                               const int* anc1, const int* d_rows, const int* d_step, int d,
                               int heads, float scale, float* ctx, long long ldc,
                               const OperandOut& op, cudaStream_t st, int early,
                               const HistReorder& hist) {
  if (r_max <= 0) return;
  const int dh = d / heads;
  if (heads < 1 || heads * dh != d) fail(kUsageError, "attention: heads must divide d_model");
  const int nw = std::min(heads, kDecAttnWarps);  // warps loop over the heads
  const size_t smem = sizeof(float) * (size_t(nw) * dec_attn_warp_floats(dh, T) + d + 33 + T);
  auto k = dh == 64 ? dec_self_attention_kernel<64> : dec_self_attention_kernel<0>;
  set_smem_limit(reinterpret_cast<const void*>(k), smem, "decoder self-attention");
  // MTG_KV_PREFETCH=1: L2 prefetch of the cached keys / values before the
  // wait (A/B; measured -0.8 % fp32 at batch 64: the prefetch competes with
  // the QKV GEMM's L2 traffic).
  static const bool prefetch = [] {
    const char* e = std::getenv("MTG_KV_PREFETCH");
    return e && e[0] == '1';
  }();
  const int mode = early ? (prefetch ? 3 : 1) : 0;
  launch_k(k, r_max, nw * 32, smem, st, qkv_cache, r_max, T, anc0, anc1, d_rows, d_step, d, dh,
           scale, ctx, ldc, op, mode, hist);
  MTG_CUDA(cudaGetLastError());
}

void launch_dec_cross_attention(const float* cq, long long ldq, const float* ckv,
                                const int* row_sent, const int* enc_off, const int* enc_len,
                                const int* d_rows, int max_rows, int max_src, int d, int heads,
                                float scale, float* ctx, long long ldc, const OperandOut& op,
                                cudaStream_t st) {
  if (max_rows <= 0) return;
  const int dh = d / heads;
  if (heads < 1 || heads * dh != d) fail(kUsageError, "attention: heads must divide d_model");
  const int nw = std::min(heads, kDecAttnWarps);
  const size_t smem = sizeof(float) * (size_t(nw) * dec_attn_warp_floats(dh, max_src) + d + 33);
  auto k = dh == 64 ? dec_cross_attention_kernel<64> : dec_cross_attention_kernel<0>;
  set_smem_limit(reinterpret_cast<const void*>(k), smem, "decoder cross-attention");
  launch_k(k, max_rows, nw * 32, smem, st, cq, ldq, ckv, row_sent, enc_off, enc_len, d_rows,
           max_src, d, dh, scale, ctx, ldc, op);
  MTG_CUDA(cudaGetLastError());
}

}  // namespace mtg
