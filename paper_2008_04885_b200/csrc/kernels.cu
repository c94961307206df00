#include "kernels.cuh"

#include <climits>

#include "detmath.cuh"
#include "errors.hpp"

namespace mtg {

namespace {

#define kNegInf (-__int_as_float(0x7f800000))
constexpr int kBosIdDev = 2;  // model.hpp:18
constexpr int kEosIdDev = 3;  // model.hpp:19

// ---- embeddings -------------------------------------------------------------------

__global__ void embed_src_kernel(const int* __restrict__ ids, const int* __restrict__ pos,
                                 const float* __restrict__ table, int d, float sqrt_d,
                                 const float* __restrict__ pe, float* __restrict__ out,
                                 long long ldo) {
  const int r = blockIdx.x;
  const float* e = table + static_cast<long long>(ids[r]) * d;
  const float* p = pe + static_cast<long long>(pos[r]) * d;
  float* o = out + r * ldo;
  for (int c = threadIdx.x; c < d; c += blockDim.x) o[c] = __fadd_rn(__fmul_rn(e[c], sqrt_d), p[c]);
}

__global__ void embed_tgt_kernel(const int* __restrict__ prev, const int* d_rows,
                                 const int* d_step, const float* __restrict__ table,
                                 const int8_t* __restrict__ table_q, float q_scale, int d,
                                 float sqrt_d, const float* __restrict__ pe,
                                 float* __restrict__ out, long long ldo) {
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

// ---- layer norm: one warp per row, P1 sums ------------------------------------------

__global__ void layernorm_kernel(const float* __restrict__ x, long long ldx, int max_rows,
                                 const int* d_rows, int n, const float* __restrict__ g,
                                 const float* __restrict__ b, float* __restrict__ y,
                                 long long ldy) {
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
  float* yr = y + r * ldy;
  for (int c = lane; c < n; c += 32)
    yr[c] = __fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(xr[c], mu), inv), g[c]), b[c]);
}

// ---- attention -------------------------------------------------------------------------

// One query against n keys, one warp. q: dh floats in smem; s: n floats of
// per-warp smem scratch. Orders: P3 dot, P1 sum, j-ascending context.
template <class KP, class VP>
__device__ __forceinline__ void attend_warp(const float* q, int n, int dh, float scale, KP kp,
                                            VP vp, float* s, float* out) {
  const int lane = threadIdx.x & 31;
  float mx = kNegInf;
  for (int j = lane; j < n; j += 32) {
    const float* k = kp(j);
    float acc = 0.0f;
    if ((dh & 3) == 0) {
      for (int c = 0; c < dh; c += 4) {
        const float4 kv = *reinterpret_cast<const float4*>(k + c);
        acc = __fadd_rn(acc, __fmul_rn(q[c], kv.x));
        acc = __fadd_rn(acc, __fmul_rn(q[c + 1], kv.y));
        acc = __fadd_rn(acc, __fmul_rn(q[c + 2], kv.z));
        acc = __fadd_rn(acc, __fmul_rn(q[c + 3], kv.w));
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
    const float e = det_expf(__fsub_rn(s[j], mx));
    s[j] = e;
    part = __fadd_rn(part, e);
  }
  const float sum = warp_allsum(part);
  for (int j = lane; j < n; j += 32) s[j] = __fdiv_rn(s[j], sum);
  __syncwarp();
  for (int c = lane; c < dh; c += 32) {
    float acc = 0.0f;
    for (int j = 0; j < n; ++j) acc = __fadd_rn(acc, __fmul_rn(s[j], vp(j)[c]));
    out[c] = acc;
  }
  __syncwarp();
}

__global__ void enc_attention_kernel(const float* __restrict__ qkv, long long ldq,
                                     const int* __restrict__ off, int d, int dh, int max_len,
                                     float scale, float* __restrict__ ctx, long long ldc) {
  extern __shared__ float sm[];
  const int s = blockIdx.x, h = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int r0 = off[s], n = off[s + 1] - r0;
  float* qs = sm + warp * (dh + max_len);
  float* ss = qs + dh;
  const float* base = qkv + static_cast<long long>(r0) * ldq + h * dh;
  for (int i = warp; i < n; i += nw) {
    for (int c = lane; c < dh; c += 32) qs[c] = base[i * ldq + c];
    __syncwarp();
    attend_warp(
        qs, n, dh, scale, [&](int j) { return base + j * ldq + d; },
        [&](int j) { return base + j * ldq + 2 * d; }, ss,
        ctx + static_cast<long long>(r0 + i) * ldc + h * dh);
  }
}

__global__ void dec_self_attention_kernel(const float* __restrict__ cache, int r_max, int T,
                                          const int* __restrict__ anc0,
                                          const int* __restrict__ anc1, const int* d_rows,
                                          const int* d_step, int d, int dh, float scale,
                                          float* __restrict__ ctx, long long ldc) {
  extern __shared__ float sm[];
  const int r = blockIdx.x;
  if (r >= *d_rows) return;
  const int t = *d_step;
  const int h = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int* ar = ((t & 1) ? anc1 : anc0) + static_cast<long long>(r) * T;
  const long long ld3 = 3LL * d;
  float* qs = sm + h * (dh + T);
  float* ss = qs + dh;
  const float* q = cache + (static_cast<long long>(t) * r_max + r) * ld3 + h * dh;
  for (int c = lane; c < dh; c += 32) qs[c] = q[c];
  __syncwarp();
  attend_warp(
      qs, t + 1, dh, scale,
      [&](int j) { return cache + (static_cast<long long>(j) * r_max + ar[j]) * ld3 + d + h * dh; },
      [&](int j) {
        return cache + (static_cast<long long>(j) * r_max + ar[j]) * ld3 + 2 * d + h * dh;
      },
      ss, ctx + r * ldc + h * dh);
}

__global__ void dec_cross_attention_kernel(const float* __restrict__ cq, long long ldq,
                                           const float* __restrict__ ckv,
                                           const int* __restrict__ row_sent,
                                           const int* __restrict__ enc_off,
                                           const int* __restrict__ enc_len, const int* d_rows,
                                           int max_src, int d, int dh, float scale,
                                           float* __restrict__ ctx, long long ldc) {
  extern __shared__ float sm[];
  const int r = blockIdx.x;
  if (r >= *d_rows) return;
  const int h = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = row_sent[r];
  const float* kv = ckv + static_cast<long long>(enc_off[s]) * 2 * d + h * dh;
  const int n = enc_len[s];
  float* qs = sm + h * (dh + max_src);
  float* ss = qs + dh;
  for (int c = lane; c < dh; c += 32) qs[c] = cq[r * ldq + h * dh + c];
  __syncwarp();
  attend_warp(
      qs, n, dh, scale, [&](int j) { return kv + static_cast<long long>(j) * 2 * d; },
      [&](int j) { return kv + static_cast<long long>(j) * 2 * d + d; }, ss,
      ctx + r * ldc + h * dh);
}

// ---- beam search ------------------------------------------------------------------------

__device__ __forceinline__ bool better2(float a, int ta, float b, int tb) {
  return a > b || (a == b && ta < tb);
}

// decode.cpp:64-69 total order: score desc, parent asc, token asc.
__device__ __forceinline__ bool better3(float a, int pa, int ta, float b, int pb, int tb) {
  if (a != b) return a > b;
  if (pa != pb) return pa < pb;
  return ta < tb;
}

__global__ void beam_init_kernel(BeamDev b) {
  if (threadIdx.x != 0) return;
  int base = 0;
  for (int s = 0; s < b.N; ++s) {
    b.best_has[s] = 0;
    if (b.sent_done[s]) {
      b.sent_live[s] = 0;
      b.sent_row0[s] = base;
      continue;
    }
    b.sent_row0[s] = base;
    b.sent_live[s] = 1;
    b.row_sent[base] = s;
    b.row_lp[base] = 0.0f;
    b.row_prev[base] = kBosIdDev;
    b.anc[0][static_cast<long long>(base) * b.T] = base;
    ++base;
  }
  *b.n_rows = base;
  *b.step = 0;
}

// One CTA (1024 threads) per live row. P2 sum order.
__global__ void __launch_bounds__(1024) topk_kernel(const float* __restrict__ logits,
                                                    long long ldl, BeamDev b) {
  const int r = blockIdx.x;
  if (r >= *b.n_rows) return;
  __shared__ float red_f[32];
  __shared__ int red_i[32];
  __shared__ int red_o[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int V = b.V;
  const float* x = logits + r * ldl;

  float mx = kNegInf;
  for (int base = 4 * tid; base < V; base += 4096)
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (base + c < V) mx = fmaxf(mx, x[base + c]);
  mx = warp_allmax(mx);
  if (lane == 0) red_f[warp] = mx;
  __syncthreads();
  mx = warp_allmax(red_f[lane]);
  __syncthreads();

  float part = 0.0f;
  for (int base = 4 * tid; base < V; base += 4096)
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (base + c < V) part = __fadd_rn(part, det_expf(__fsub_rn(x[base + c], mx)));
  part = warp_allsum(part);
  if (lane == 0) red_f[warp] = part;
  __syncthreads();
  const float total = warp_allsum(red_f[lane]);
  const float lse = __fadd_rn(det_logf(total), mx);
  const float plp = b.row_lp[r];
  __syncthreads();

  const int kB = min(b.B, V);
  float sc[kMaxBeam];
  int tk[kMaxBeam];
  int cnt = 0;
  for (int base = 4 * tid; base < V; base += 4096)
    for (int c = 0; c < 4; ++c) {
      const int j = base + c;
      if (j >= V) break;
      const float v = __fadd_rn(plp, __fsub_rn(x[j], lse));
      if (cnt == kB && !better2(v, j, sc[kB - 1], tk[kB - 1])) continue;
      int pos = cnt < kB ? cnt++ : kB - 1;
      while (pos > 0 && better2(v, j, sc[pos - 1], tk[pos - 1])) {
        sc[pos] = sc[pos - 1];
        tk[pos] = tk[pos - 1];
        --pos;
      }
      sc[pos] = v;
      tk[pos] = j;
    }

  int head = 0;
  for (int k = 0; k < kB; ++k) {
    float bs = head < cnt ? sc[head] : kNegInf;
    int bt = head < cnt ? tk[head] : INT_MAX;
    int bo = head < cnt ? tid : -1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float os = __shfl_xor_sync(0xffffffffu, bs, o);
      const int ot = __shfl_xor_sync(0xffffffffu, bt, o);
      const int oo = __shfl_xor_sync(0xffffffffu, bo, o);
      if (oo >= 0 && (bo < 0 || better2(os, ot, bs, bt))) {
        bs = os;
        bt = ot;
        bo = oo;
      }
    }
    if (lane == 0) {
      red_f[warp] = bs;
      red_i[warp] = bt;
      red_o[warp] = bo;
    }
    __syncthreads();
    if (warp == 0) {
      bs = red_f[lane];
      bt = red_i[lane];
      bo = red_o[lane];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float os = __shfl_xor_sync(0xffffffffu, bs, o);
        const int ot = __shfl_xor_sync(0xffffffffu, bt, o);
        const int oo = __shfl_xor_sync(0xffffffffu, bo, o);
        if (oo >= 0 && (bo < 0 || better2(os, ot, bs, bt))) {
          bs = os;
          bt = ot;
          bo = oo;
        }
      }
      if (lane == 0) {
        b.cand_score[static_cast<long long>(r) * b.B + k] = bs;
        b.cand_tok[static_cast<long long>(r) * b.B + k] = bt;
        red_o[0] = bo;
      }
    }
    __syncthreads();
    if (red_o[0] == tid) ++head;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(1024) beam_select_kernel(BeamDev b) {
  const int t = *b.step;
  const int cur = t & 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kB = min(b.B, b.V);
  const int T = b.T;
  __shared__ uint32_t taken_all[32][kMaxBeam * kMaxBeam / 32];
  uint32_t* taken = taken_all[warp];
  const int* tok_cur = b.tok[cur];

  for (int s = warp; s < b.N; s += 32) {
    if (b.sent_done[s]) continue;
    const int L = b.sent_live[s], r0 = b.sent_row0[s];
    const int nc = L * kB;
    for (int w = lane; w < kMaxBeam * kMaxBeam / 32; w += 32) taken[w] = 0;
    __syncwarp();
    const int n_sel = min(b.B, nc);
    int q = 0;
    for (int k = 0; k < n_sel; ++k) {
      float bs = kNegInf;
      int bp = INT_MAX, bt = INT_MAX, bc = -1;
      for (int c = lane; c < nc; c += 32) {
        if (taken[c >> 5] & (1u << (c & 31))) continue;
        const int p = c / kB, e = c % kB;
        const long long idx = static_cast<long long>(r0 + p) * b.B + e;
        const float sc = b.cand_score[idx];
        const int tk = b.cand_tok[idx];
        if (bc < 0 || better3(sc, p, tk, bs, bp, bt)) {
          bs = sc;
          bp = p;
          bt = tk;
          bc = c;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float os = __shfl_xor_sync(0xffffffffu, bs, o);
        const int op = __shfl_xor_sync(0xffffffffu, bp, o);
        const int ot = __shfl_xor_sync(0xffffffffu, bt, o);
        const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
        if (oc >= 0 && (bc < 0 || better3(os, op, ot, bs, bp, bt))) {
          bs = os;
          bp = op;
          bt = ot;
          bc = oc;
        }
      }
      if (lane == 0) taken[bc >> 5] |= 1u << (bc & 31);
      const int pr = r0 + bp;
      if (bt == kEosIdDev) {
        // decode.cpp:77-80 + first max of normalized_score over finished.
        const float len = static_cast<float>(t) + 1.0f;
        const float norm = __fdiv_rn(bs, det_powf(__fdiv_rn(__fadd_rn(5.0f, len), 6.0f), b.alpha));
        const bool repl = !b.best_has[s] || norm > b.best_norm[s];
        __syncwarp();
        if (repl) {
          for (int j = lane; j < t; j += 32)
            b.best_tok[static_cast<long long>(s) * T + j] = tok_cur[static_cast<long long>(pr) * T + j];
          if (lane == 0) {
            b.best_has[s] = 1;
            b.best_norm[s] = norm;
            b.best_lp[s] = bs;
            b.best_len[s] = t;
          }
        }
      } else {
        if (lane == 0) {
          b.sel_parent[s * b.B + q] = pr;
          b.sel_tok[s * b.B + q] = bt;
          b.sel_lp[s * b.B + q] = bs;
        }
        ++q;
      }
      __syncwarp();
    }

    int new_live = q;
    if (new_live > 0 && t + 1 >= b.max_seq_len && b.sent_maxlen[s] > b.max_seq_len) {
      // decode_step would be called past max_seq_len (model.cpp:618-619).
      if (lane == 0) {
        b.res_status[s] = 2;  // ValueError
        b.res_flags[s] = 4u;
        b.res_len[s] = 0;
        b.sent_done[s] = 1;
      }
      new_live = 0;
    } else if (new_live == 0 || t + 1 >= b.sent_maxlen[s]) {
      if (b.best_has[s]) {  // decode.cpp:89-98
        const int n = b.best_len[s];
        for (int j = lane; j < n; j += 32)
          b.res_tok[static_cast<long long>(s) * T + j] = b.best_tok[static_cast<long long>(s) * T + j];
        if (lane == 0) {
          b.res_len[s] = n;
          b.res_lp[s] = b.best_lp[s];
          b.res_norm[s] = b.best_norm[s];
          b.res_flags[s] = 1u;
        }
      } else {  // decode.cpp:99-108: first max over live, truncated
        const float len = static_cast<float>(t + 1) + 1.0f;
        const float den = det_powf(__fdiv_rn(__fadd_rn(5.0f, len), 6.0f), b.alpha);
        int bq = 0;
        float bn = __fdiv_rn(b.sel_lp[s * b.B], den);
        for (int qq = 1; qq < new_live; ++qq) {
          const float nq = __fdiv_rn(b.sel_lp[s * b.B + qq], den);
          if (nq > bn) {
            bn = nq;
            bq = qq;
          }
        }
        const int pr = b.sel_parent[s * b.B + bq];
        for (int j = lane; j < t; j += 32)
          b.res_tok[static_cast<long long>(s) * T + j] = tok_cur[static_cast<long long>(pr) * T + j];
        if (lane == 0) {
          b.res_tok[static_cast<long long>(s) * T + t] = b.sel_tok[s * b.B + bq];
          b.res_len[s] = t + 1;
          b.res_lp[s] = b.sel_lp[s * b.B + bq];
          b.res_norm[s] = bn;
          b.res_flags[s] = 2u;
        }
      }
      if (lane == 0) {
        b.res_status[s] = 0;
        b.sent_done[s] = 1;
      }
      new_live = 0;
    }
    if (lane == 0) b.sent_live[s] = new_live;
    __syncwarp();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int base = 0;
    for (int s = 0; s < b.N; ++s) {
      b.sent_row0[s] = base;
      base += b.sent_live[s];
    }
    *b.n_rows = base;
  }
  __syncthreads();
  for (int s = warp; s < b.N; s += 32) {
    const int L = b.sent_live[s];
    for (int q = lane; q < L; q += 32) {
      const int row = b.sent_row0[s] + q;
      b.row_sent[row] = s;
      b.row_parent[row] = b.sel_parent[s * b.B + q];
      b.row_prev[row] = b.sel_tok[s * b.B + q];
      b.row_lp[row] = b.sel_lp[s * b.B + q];
    }
  }
  if (threadIdx.x == 0) *b.step = t + 1;
}

__global__ void beam_reorder_kernel(BeamDev b) {
  const int r = blockIdx.x;
  if (r >= *b.n_rows) return;
  const int tn = *b.step;
  const int cur = (tn - 1) & 1, nxt = tn & 1;
  const int T = b.T;
  const int pr = b.row_parent[r];
  const int* ac = b.anc[cur] + static_cast<long long>(pr) * T;
  int* an = b.anc[nxt] + static_cast<long long>(r) * T;
  const int* tc = b.tok[cur] + static_cast<long long>(pr) * T;
  int* tnw = b.tok[nxt] + static_cast<long long>(r) * T;
  for (int j = threadIdx.x; j < tn && j < T; j += blockDim.x) an[j] = ac[j];
  for (int j = threadIdx.x; j < tn - 1; j += blockDim.x) tnw[j] = tc[j];
  if (threadIdx.x == 0) {
    if (tn < T) an[tn] = r;
    if (tn - 1 < T) tnw[tn - 1] = b.row_prev[r];
  }
}

}  // namespace

// ---- launchers ------------------------------------------------------------------------------

void launch_embed_src(const int* ids, const int* pos, int rows, const float* table, int d,
                      float sqrt_d, const float* pe, float* out, long long ldo, cudaStream_t st) {
  if (rows <= 0) return;
  embed_src_kernel<<<rows, 128, 0, st>>>(ids, pos, table, d, sqrt_d, pe, out, ldo);
  MTG_CUDA(cudaGetLastError());
}

void launch_embed_tgt(const int* prev, const int* d_rows, int max_rows, const int* d_step,
                      const float* table, const int8_t* table_q, float q_scale, int d,
                      float sqrt_d, const float* pe, float* out, long long ldo, cudaStream_t st) {
  if (max_rows <= 0) return;
  embed_tgt_kernel<<<max_rows, 128, 0, st>>>(prev, d_rows, d_step, table, table_q, q_scale, d,
                                             sqrt_d, pe, out, ldo);
  MTG_CUDA(cudaGetLastError());
}

void launch_layernorm(const float* x, long long ldx, int max_rows, const int* d_rows, int n,
                      const float* g, const float* b, float* y, long long ldy, cudaStream_t st) {
  if (max_rows <= 0) return;
  const int wpb = 8;
  layernorm_kernel<<<(max_rows + wpb - 1) / wpb, wpb * 32, 0, st>>>(x, ldx, max_rows, d_rows, n,
                                                                    g, b, y, ldy);
  MTG_CUDA(cudaGetLastError());
}

void launch_enc_attention(const float* qkv, long long ldq, const int* off, int n_sent,
                          int max_len, int d, int heads, float scale, float* ctx, long long ldc,
                          cudaStream_t st) {
  if (n_sent <= 0) return;
  const int dh = d / heads;
  const int nw = 4;
  const size_t smem = sizeof(float) * nw * (dh + max_len);
  enc_attention_kernel<<<dim3(n_sent, heads), nw * 32, smem, st>>>(qkv, ldq, off, d, dh, max_len,
                                                                   scale, ctx, ldc);
  MTG_CUDA(cudaGetLastError());
}

void launch_dec_self_attention(const float* qkv_cache, int r_max, int T, const int* anc0,
                               const int* anc1, const int* d_rows, const int* d_step, int d,
                               int heads, float scale, float* ctx, long long ldc,
                               cudaStream_t st) {
  if (r_max <= 0) return;
  const int dh = d / heads;
  const size_t smem = sizeof(float) * heads * (dh + T);
  dec_self_attention_kernel<<<r_max, heads * 32, smem, st>>>(qkv_cache, r_max, T, anc0, anc1,
                                                             d_rows, d_step, d, dh, scale, ctx,
                                                             ldc);
  MTG_CUDA(cudaGetLastError());
}

void launch_dec_cross_attention(const float* cq, long long ldq, const float* ckv,
                                const int* row_sent, const int* enc_off, const int* enc_len,
                                const int* d_rows, int max_rows, int max_src, int d, int heads,
                                float scale, float* ctx, long long ldc, cudaStream_t st) {
  if (max_rows <= 0) return;
  const int dh = d / heads;
  const size_t smem = sizeof(float) * heads * (dh + max_src);
  dec_cross_attention_kernel<<<max_rows, heads * 32, smem, st>>>(
      cq, ldq, ckv, row_sent, enc_off, enc_len, d_rows, max_src, d, dh, scale, ctx, ldc);
  MTG_CUDA(cudaGetLastError());
}

void launch_beam_init(const BeamDev& b, cudaStream_t st) {
  beam_init_kernel<<<1, 32, 0, st>>>(b);
  MTG_CUDA(cudaGetLastError());
}

void launch_topk(const float* logits, long long ldl, const BeamDev& b, cudaStream_t st) {
  topk_kernel<<<b.R_max, 1024, 0, st>>>(logits, ldl, b);
  MTG_CUDA(cudaGetLastError());
}

void launch_beam_select(const BeamDev& b, cudaStream_t st) {
  beam_select_kernel<<<1, 1024, 0, st>>>(b);
  MTG_CUDA(cudaGetLastError());
}

void launch_beam_reorder(const BeamDev& b, cudaStream_t st) {
  beam_reorder_kernel<<<b.R_max, 128, 0, st>>>(b);
  MTG_CUDA(cudaGetLastError());
}

}  // namespace mtg
