// Small-batch decoder attention (<= kGemvRows live rows, head dim 64): one
// CTA per (row, head), model.cpp:642-665.
//
// Latency, not bandwidth, bounds batch-1 decoding, so the kernel moves every
// load it can in front of the programmatic-dependency wait. Anything written
// two or more kernels earlier is complete once this kernel's CTAs run (the
// predecessor has passed its own wait), which covers
//   * self-attention: the step and row count, the row's ancestry -- derived
//     from its parent's table exactly as the history reorder does
//     (beam.cu beam_reorder_kernel) -- and the cached keys / values of
//     positions 0..t-1;
//   * cross-attention: the row's sentence and the encoder keys / values.
// After the wait only the current query (and, for self-attention, the current
// key / value row written by the QKV GEMV) is loaded. The arithmetic is the
// staged decoder attention's (kernels.cu attend_warp_staged64): P3 dots,
// P1 softmax over lane-strided keys, contexts summed in key order.
#include <algorithm>

#include "attn_warp.cuh"
#include "detmath.cuh"
#include "errors.hpp"
#include "gemv.cuh"
#include "kernels.cuh"
#include "launch.cuh"

namespace mtg {

namespace {

constexpr int kAttnThreads = 128;
constexpr int kDh = kAttnDh;

struct AttnSmallArgs {
  int self_mode;  // 1: self-attention over the KV cache, 0: cross-attention
  const int* d_rows;
  const int* d_step;
  int rows_alloc;
  int d;
  float scale;
  float* ctx;
  long long ldc;
  // self
  const float* cache;  // [T][r_max][3d]
  int r_max, T;
  const int* anc0;
  const int* anc1;
  const int* row_parent;
  int reorder;
  // history reorder (beam.cu beam_reorder_kernel), done by the layer-0
  // attention: row r's ancestry / token tables of step t
  int hist;
  int* anc_out[2];
  int* tok_out[2];
  const int* row_prev;
  // cross
  const float* cq;
  long long ldq;
  const float* ckv;  // [M_enc][2d]
  const int* row_sent;
  const int* enc_off;
  const int* enc_len;
  KTrace trace;
};

__global__ void __launch_bounds__(kAttnThreads)
    attn_small_kernel(const AttnSmallArgs a) {
  extern __shared__ __align__(16) float sm[];
  const int r = blockIdx.x, h = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int d = a.d;
  // ---- before the wait: data written two or more kernels ago ----
  const int R = *a.d_rows;
  const int t = a.self_mode ? *a.d_step : 0;
  int n = 0;  // keys
  float* K = sm;
  int Tk = a.self_mode ? a.T : 0;
  if (r < R) {
    if (a.self_mode) {
      n = t + 1;
      Tk = a.T;
      float* V = K + Tk * kDh;
      int* arow = reinterpret_cast<int*>(V + Tk * kDh + 2 * kDh + Tk);
      // ancestry of row r at step t: its parent's table for positions < t
      // (the reorder's copy), itself at t
      const int* src = (a.reorder && t >= 1)
                           ? ((t - 1) & 1 ? a.anc1 : a.anc0) + static_cast<long long>(a.row_parent[r]) * a.T
                           : ((t & 1) ? a.anc1 : a.anc0) + static_cast<long long>(r) * a.T;
      for (int j = tid; j < t; j += blockDim.x) arow[j] = src[j];
      if (tid == 0) arow[t] = r;
      __syncthreads();
      if (a.hist && a.reorder && t >= 1 && h == 0) {
        // Nothing reads step t's tables before this kernel (the attention
        // derives the ancestry from the parent): the next step's attention
        // and this step's beam selection come later.
        int* an = a.anc_out[t & 1] + static_cast<long long>(r) * a.T;
        const int* tc = a.tok_out[(t - 1) & 1] + static_cast<long long>(a.row_parent[r]) * a.T;
        int* tn = a.tok_out[t & 1] + static_cast<long long>(r) * a.T;
        for (int j = tid; j <= t && j < a.T; j += blockDim.x) an[j] = arow[j];
        for (int j = tid; j < t - 1; j += blockDim.x) tn[j] = tc[j];
        if (tid == 0 && t - 1 < a.T) tn[t - 1] = a.row_prev[r];
      }
      const long long ld3 = 3LL * d;
      const float* kb = a.cache + d + h * kDh;
      stage_kv(
          K, V, 0, t,
          [&](int j) { return kb + (static_cast<long long>(j) * a.r_max + arow[j]) * ld3; },
          [&](int j) { return kb + (static_cast<long long>(j) * a.r_max + arow[j]) * ld3 + d; });
    } else {
      const int s = a.row_sent[r];
      n = a.enc_len[s];
      Tk = n;
      float* V = K + Tk * kDh;
      const float* kv = a.ckv + static_cast<long long>(a.enc_off[s]) * 2 * d + h * kDh;
      stage_kv(
          K, V, 0, n, [&](int j) { return kv + static_cast<long long>(j) * 2 * d; },
          [&](int j) { return kv + static_cast<long long>(j) * 2 * d + d; });
    }
  }
  pdl_wait();
  pdl_trigger();
  trace_begin(a.trace);
  if (r >= R) {
    trace_end(a.trace);
    return;
  }
  float* V = K + Tk * kDh;
  float* q = V + Tk * kDh;  // [64]
  float* s = q + 2 * kDh;   // [n] scores -> probabilities
  // ---- after the wait: the current query (and key / value at step t) ----
  if (a.self_mode) {
    const long long ld3 = 3LL * d;
    const float* row = a.cache + (static_cast<long long>(t) * a.r_max + r) * ld3 + h * kDh;
    if (tid < 16) {
      cp_async16s(q + 4 * tid, row + 4 * tid);
    } else if (tid < 32) {
      cp_async16s(K + swz(t, tid - 16), row + d + 4 * (tid - 16));
    } else if (tid < 48) {
      cp_async16s(V + swz(t, tid - 32), row + 2 * d + 4 * (tid - 32));
    }
  } else if (tid < 16) {
    cp_async16s(q + 4 * tid, a.cq + r * a.ldq + h * kDh + 4 * tid);
  }
  cp_async_wait_all();
  __syncthreads();
  // scores (P3): dot over the head dimension in order, then x scale
  for (int j = tid; j < n; j += blockDim.x) {
    float acc = 0.0f;
#pragma unroll
    for (int c4 = 0; c4 < 16; ++c4) {
      const float4 kv = *reinterpret_cast<const float4*>(K + swz(j, c4));
      const float4 qv = *reinterpret_cast<const float4*>(q + 4 * c4);
      acc = __fadd_rn(acc, __fmul_rn(qv.x, kv.x));
      acc = __fadd_rn(acc, __fmul_rn(qv.y, kv.y));
      acc = __fadd_rn(acc, __fmul_rn(qv.z, kv.z));
      acc = __fadd_rn(acc, __fmul_rn(qv.w, kv.w));
    }
    s[j] = __fmul_rn(acc, a.scale);
  }
  __syncthreads();
  // softmax (P1 over lane-strided keys), warp 0
  if (warp == 0) {
    float mx = -__int_as_float(0x7f800000);
    for (int j = lane; j < n; j += 32) mx = fmaxf(mx, s[j]);
    mx = warp_allmax(mx);
    float part = 0.0f;
    for (int j = lane; j < n; j += 32) {
      const float e = det_expf_nonpos(__fsub_rn(s[j], mx));
      s[j] = e;
      part = __fadd_rn(part, e);
    }
    const float sum = warp_allsum(part);
    for (int j = lane; j < n; j += 32) s[j] = __fdiv_rn(s[j], sum);
  }
  __syncthreads();
  // context: column c sums p_j * v_j[c] over keys in order
  if (tid < kDh) {
    const int c = tid, c4 = c >> 2, e = c & 3;
    float acc = 0.0f;
    for (int j = 0; j < n; ++j) acc = __fadd_rn(acc, __fmul_rn(s[j], V[swz(j, c4) + e]));
    a.ctx[r * a.ldc + h * kDh + c] = acc;
  }
  trace_end(a.trace);
}

// Batched cross-attention, one CTA per (sentence, head), one warp per live
// beam row of the sentence. The sentence's encoder keys / values of the head
// are staged once for all its rows, before the programmatic-dependency wait
// (the beam state that locates them is written two or more kernels back);
// after the wait each warp loads its query and attends. Same arithmetic as
// kernels.cu attend_warp_staged64. Writes the fp32 context and, element by
// element, the next GEMM's bf16 / TF32x3 operand (int8 needs whole-row scales
// and keeps the per-row kernel).
struct AttnCrossArgs {
  const float* cq;
  long long ldq;
  const float* ckv;
  const int* enc_off;
  const int* enc_len;
  const int* sent_row0;
  const int* sent_live;
  const int* sent_done;
  int d;
  float scale;
  float* ctx;
  long long ldc;
  OperandOut op;
};

__global__ void __launch_bounds__(512)
    attn_cross_sent_kernel(const AttnCrossArgs a, int max_src) {
  extern __shared__ __align__(16) float sm[];
  const int s = blockIdx.x, h = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int d = a.d;
  float* K = sm;
  float* V = K + max_src * kDh;
  const int wstride = kDh + (max_src + 3) / 4 * 4;          // 16-byte aligned per-warp blocks
  float* wq = V + max_src * kDh + warp * wstride;  // [64] query, then [max_src] scores
  float* ws = wq + kDh;
  // ---- before the wait: beam state (previous step's selection) and keys ----
  const int live = a.sent_done[s] ? 0 : a.sent_live[s];
  const int r0 = a.sent_row0[s];
  const int n = a.enc_len[s];
  if (live > 0) {
    const float* kv = a.ckv + static_cast<long long>(a.enc_off[s]) * 2 * d + h * kDh;
    stage_kv(
        K, V, 0, n, [&](int j) { return kv + static_cast<long long>(j) * 2 * d; },
        [&](int j) { return kv + static_cast<long long>(j) * 2 * d + d; });
  }
  pdl_wait();
  pdl_trigger();
  trace_begin(a.op.tr);
  if (threadIdx.x == 0) trace_phase(a.op.tr, 0);
  cp_async_wait_all();
  __syncthreads();  // keys / values staged by every thread's copies
  if (threadIdx.x == 0) trace_phase(a.op.tr, 1);
  for (int w = warp; w < live; w += nw) {
    const long long r = r0 + w;
    for (int c = lane; c < kDh; c += 32) wq[c] = a.cq[r * a.ldq + h * kDh + c];
    __syncwarp();
    float acc_a, acc_b;
    attend_warp64(K, V, wq, ws, n, a.scale, lane, acc_a, acc_b);
    const float vals[2] = {acc_a, acc_b};
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const long long c = h * kDh + lane + 32 * u;
      const float v = vals[u];
      a.ctx[r * a.ldc + c] = v;
      const OperandOut& o = a.op;
      if (o.prec == 1) {
        o.h[r * o.k_pad + c] = __float2bfloat16_rn(v);
      } else if (o.prec == 3) {
        o.hi[r * o.k_pad + c] = v;
      } else if (o.prec == 2) {
        uint32_t hb;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(v));
        o.hi[r * o.k_pad + c] = __uint_as_float(hb);
        o.lo[r * o.k_pad + c] = __fsub_rn(v, __uint_as_float(hb));
      }
    }
    __syncwarp();
  }
  trace_end(a.op.tr);
}

size_t attn_small_smem(int keys) {
  return sizeof(float) * (2 * size_t(keys) * kDh + 2 * kDh + size_t(keys)) +
         sizeof(int) * size_t(keys);
}

}  // namespace

size_t attn_cross_sent_smem(int max_src, int warps) {
  return sizeof(float) * (2 * size_t(max_src) * kDh + size_t(warps) * (kDh + (max_src + 3) / 4 * 4));
}

bool attn_cross_sent_supported(int d, int heads, int max_src, int beam) {
  return heads > 0 && d == heads * kDh && beam <= 16 &&
         attn_cross_sent_smem(max_src, beam) <= 100 * 1024;
}

void launch_attn_cross_sent(const float* cq, long long ldq, const float* ckv, const int* enc_off,
                            const int* enc_len, const int* sent_row0, const int* sent_live,
                            const int* sent_done, int n_sent, int beam, int max_src, int d,
                            int heads, float scale, float* ctx, long long ldc,
                            const OperandOut& op, cudaStream_t st) {
  if (n_sent <= 0) return;
  if (op.prec == 0) fail(kStateError, "cross attention per sentence: no int8 operand rows");
  AttnCrossArgs a{cq, ldq, ckv, enc_off, enc_len, sent_row0, sent_live, sent_done, d, scale, ctx,
                  ldc, op};
  const int warps = std::max(1, std::min(beam, 16));
  const size_t smem = attn_cross_sent_smem(max_src, warps);
  ensure_smem_attr(attn_cross_sent_kernel, smem);
  launch_k(attn_cross_sent_kernel, dim3(n_sent, heads), warps * 32, smem, st, a, max_src);
  MTG_CUDA(cudaGetLastError());
}

bool attn_small_supported(int d, int heads, int T, int max_src) {
  return heads > 0 && d == heads * kDh && attn_small_smem(std::max(T, max_src)) <= 200 * 1024;
}

void launch_attn_small_self(const float* cache, int r_max, int T, int* anc0, int* anc1,
                            const int* row_parent, int reorder, int* tok0, int* tok1,
                            const int* row_prev, int hist, const int* d_rows, const int* d_step,
                            int rows_alloc, int d, int heads, float scale, float* ctx,
                            long long ldc, cudaStream_t st, const KTrace& tr) {
  AttnSmallArgs a{};
  a.hist = hist;
  a.anc_out[0] = anc0;
  a.anc_out[1] = anc1;
  a.tok_out[0] = tok0;
  a.tok_out[1] = tok1;
  a.row_prev = row_prev;
  a.trace = tr;
  a.self_mode = 1;
  a.d_rows = d_rows;
  a.d_step = d_step;
  a.rows_alloc = rows_alloc;
  a.d = d;
  a.scale = scale;
  a.ctx = ctx;
  a.ldc = ldc;
  a.cache = cache;
  a.r_max = r_max;
  a.T = T;
  a.anc0 = anc0;
  a.anc1 = anc1;
  a.row_parent = row_parent;
  a.reorder = reorder;
  const size_t smem = attn_small_smem(T);
  ensure_smem_attr(attn_small_kernel, smem);
  launch_k(attn_small_kernel, dim3(rows_alloc, heads), kAttnThreads, smem, st, a);
  MTG_CUDA(cudaGetLastError());
}

void launch_attn_small_cross(const float* cq, long long ldq, const float* ckv,
                             const int* row_sent, const int* enc_off, const int* enc_len,
                             const int* d_rows, int rows_alloc, int max_src, int d, int heads,
                             float scale, float* ctx, long long ldc, cudaStream_t st,
                             const KTrace& tr) {
  AttnSmallArgs a{};
  a.trace = tr;
  a.self_mode = 0;
  a.d_rows = d_rows;
  a.rows_alloc = rows_alloc;
  a.d = d;
  a.scale = scale;
  a.ctx = ctx;
  a.ldc = ldc;
  a.cq = cq;
  a.ldq = ldq;
  a.ckv = ckv;
  a.row_sent = row_sent;
  a.enc_off = enc_off;
  a.enc_len = enc_len;
  const size_t smem = attn_small_smem(max_src);
  ensure_smem_attr(attn_small_kernel, smem);
  launch_k(attn_small_kernel, dim3(rows_alloc, heads), kAttnThreads, smem, st, a);
  MTG_CUDA(cudaGetLastError());
}

}  // namespace mtg
