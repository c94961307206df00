// Beam bookkeeping kernels (decode.cpp:34-109): root rows, per-sentence
// selection / finished list / termination, and history gathers.
#include <climits>

#include "detmath.cuh"
#include "errors.hpp"
#include "launch.cuh"
#include "kernels.cuh"

namespace mtg {

namespace {

#define kNegInf (-__int_as_float(0x7f800000))
constexpr int kBosIdDev = 2;  // model.hpp:18
constexpr int kEosIdDev = 3;  // model.hpp:19

// ---- beam search ------------------------------------------------------------------------

// decode.cpp:64-69 total order: score desc, parent asc, token asc.
__device__ __forceinline__ bool better3(float a, int pa, int ta, float b, int pb, int tb) {
  if (a != b) return a > b;
  if (pa != pb) return pa < pb;
  return ta < tb;
}

__global__ void beam_init_kernel(BeamDev b) {
  pdl_wait();
  pdl_trigger();
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

__global__ void __launch_bounds__(1024) beam_select_kernel(BeamDev b) {
  pdl_wait();
  pdl_trigger();
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
        if (tk < 0 || tk >= b.V || sc != sc) continue;  // no candidate (NaN logits)
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
      if (bc < 0) {  // invalid logits for this sentence: fail it (ValueError)
        if (lane == 0) {
          b.res_status[s] = 2;
          b.res_flags[s] = 4u;
          b.res_len[s] = 0;
          b.sent_done[s] = 1;
        }
        q = -1;
        break;
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

    if (q < 0) {
      if (lane == 0) b.sent_live[s] = 0;
      __syncwarp();
      continue;
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
  pdl_wait();
  pdl_trigger();
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

void launch_beam_init(const BeamDev& b, cudaStream_t st) {
  launch_k(beam_init_kernel, 1, 32, 0, st, b);
  MTG_CUDA(cudaGetLastError());
}

void launch_beam_select(const BeamDev& b, cudaStream_t st) {
  launch_k(beam_select_kernel, 1, 1024, 0, st, b);
  MTG_CUDA(cudaGetLastError());
}

void launch_beam_reorder(const BeamDev& b, cudaStream_t st) {
  launch_k(beam_reorder_kernel, b.R_max, 128, 0, st, b);
  MTG_CUDA(cudaGetLastError());
}

}  // namespace mtg
