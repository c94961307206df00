// Per-sentence beam selection and the grid-level row compaction of one
// decode step (decode.cpp:34-109), shared by beam_select_kernel (beam.cu)
// and the fused top-k + select kernel (topk.cu).
#pragma once

#include <climits>

#include "detmath.cuh"
#include "kernels.cuh"

#ifndef kNegInf
#define kNegInf (-__int_as_float(0x7f800000))
#endif

namespace mtg {

constexpr int kEosIdDev = 3;  // model.hpp:19
constexpr int kCandPerLane = kMaxBeam * kMaxBeam / 32;  // <= 8

// decode.cpp:64-69 total order: score desc, parent asc, token asc.
// Branch-free (bitwise on the comparisons): the short-circuit form compiles to
// divergent branches, ~125 cycles per comparison in a warp-wide rank loop
// (tools/micro/warp_sort_bench.cu). NaN scores compare false either way.
__device__ __forceinline__ bool better3(float a, int pa, int ta, float b, int pb, int tb) {
  return (a > b) | ((a == b) & ((pa < pb) | ((pa == pb) & (ta < tb))));
}

// Per-sentence beam state, loaded together (one round trip). It is written
// only by the step tail, so a tail kernel may load it before its dependency
// wait.
struct SentState {
  int done, L, r0, maxlen, has, blen;
  float bnorm, blp;
};
__device__ __forceinline__ SentState load_sent_state(const BeamDev& b, int s) {
  SentState st;
  st.done = b.sent_done[s];
  st.L = b.sent_live[s];
  st.r0 = b.sent_row0[s];
  st.maxlen = b.sent_maxlen[s];
  st.has = b.best_has[s];
  st.blen = b.best_len[s];
  st.bnorm = b.best_norm[s];
  st.blp = b.best_lp[s];
  return st;
}

// Sequential form (kB selection rounds of warp argmax), for sentences with
// more than 32 candidates (beam * beam > 32).
__device__ __forceinline__ void select_sentence_seq(const BeamDev& b, int s, int t, int lane,
                                                    const SentState& st) {
  const int kB = min(b.B, b.V);
  const int T = b.T;
  const int* tok_cur = b.tok[t & 1];
  const int done = st.done, L = st.L, r0 = st.r0;
  const int maxlen = st.maxlen;
  int has = st.has, blen = st.blen;
  float bnorm = st.bnorm, blp = st.blp;
  if (done) return;
  const int nc = L * kB;
  // Candidates of this sentence, loaded once: lane owns c = lane + 32 i.
  float cs[kCandPerLane];
  int cp[kCandPerLane], ct[kCandPerLane];
  unsigned ok = 0u;
#pragma unroll
  for (int i = 0; i < kCandPerLane; ++i) {
    const int c = lane + 32 * i;
    cs[i] = kNegInf;
    cp[i] = INT_MAX;
    ct[i] = INT_MAX;
    if (c < nc) {
      const int p = c / kB, e = c - p * kB;
      const long long idx = static_cast<long long>(r0 + p) * b.B + e;
      cs[i] = b.cand_score[idx];
      ct[i] = b.cand_tok[idx];
      cp[i] = p;
    }
  }
#pragma unroll
  for (int i = 0; i < kCandPerLane; ++i)  // no candidate (NaN logits) never competes
    if (lane + 32 * i < nc && ct[i] >= 0 && ct[i] < b.V && cs[i] == cs[i]) ok |= 1u << i;
  // decode.cpp:71: take min(|cands|, beam) -- a shortlist can leave fewer
  // valid candidates than beam slots; none at all means invalid logits.
  int n_valid = __popc(ok);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) n_valid += __shfl_xor_sync(0xffffffffu, n_valid, o);
  const int n_sel = n_valid > 0 ? min(b.B, n_valid) : 1;
  int q = 0;
  // Lane q keeps the q-th surviving (non-EOS) selection.
  float my_lp = 0.0f;
  int my_parent = 0, my_tok = 0;
  for (int k = 0; k < n_sel; ++k) {
    float bs = kNegInf;
    int bp = INT_MAX, bt = INT_MAX, bi = -1;
#pragma unroll
    for (int i = 0; i < kCandPerLane; ++i)
      if (((ok >> i) & 1u) && (bi < 0 || better3(cs[i], cp[i], ct[i], bs, bp, bt))) {
        bs = cs[i];
        bp = cp[i];
        bt = ct[i];
        bi = i;
      }
    int bl = bi >= 0 ? lane : -1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float os = __shfl_xor_sync(0xffffffffu, bs, o);
      const int op = __shfl_xor_sync(0xffffffffu, bp, o);
      const int ot = __shfl_xor_sync(0xffffffffu, bt, o);
      const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
      if (ol >= 0 && (bl < 0 || better3(os, op, ot, bs, bp, bt))) {
        bs = os;
        bp = op;
        bt = ot;
        bl = ol;
      }
    }
    if (bl < 0) {  // invalid logits for this sentence: fail it (ValueError)
      if (lane == 0) {
        b.res_status[s] = 2;
        b.res_flags[s] = 4u;
        b.res_len[s] = 0;
        b.sent_done[s] = 1;
      }
      q = -1;
      break;
    }
    if (lane == bl) ok &= ~(1u << bi);
    const int pr = r0 + bp;
    if (bt == kEosIdDev) {
      // decode.cpp:77-80 + first max of normalized_score over finished.
      const float len = static_cast<float>(t) + 1.0f;
      const float norm = __fdiv_rn(bs, det_powf(__fdiv_rn(__fadd_rn(5.0f, len), 6.0f), b.alpha));
      if (!has || norm > bnorm) {
        for (int j = lane; j < t; j += 32)
          b.best_tok[static_cast<long long>(s) * T + j] = tok_cur[static_cast<long long>(pr) * T + j];
        has = 1;
        bnorm = norm;
        blp = bs;
        blen = t;
        if (lane == 0) {
          b.best_has[s] = 1;
          b.best_norm[s] = norm;
          b.best_lp[s] = bs;
          b.best_len[s] = t;
        }
      }
    } else {
      if (lane == q) {
        my_lp = bs;
        my_parent = pr;
        my_tok = bt;
      }
      if (lane == 0) {
        b.sel_parent[s * b.B + q] = pr;
        b.sel_tok[s * b.B + q] = bt;
        b.sel_lp[s * b.B + q] = bs;
      }
      ++q;
    }
  }
  __syncwarp();

  if (q < 0) {
    if (lane == 0) b.sent_live[s] = 0;
    __syncwarp();
    return;
  }
  int new_live = q;
  if (new_live > 0 && t + 1 >= b.max_seq_len && maxlen > b.max_seq_len) {
    // decode_step would be called past max_seq_len (model.cpp:618-619).
    if (lane == 0) {
      b.res_status[s] = 2;  // ValueError
      b.res_flags[s] = 4u;
      b.res_len[s] = 0;
      b.sent_done[s] = 1;
    }
    new_live = 0;
  } else if (new_live == 0 || t + 1 >= maxlen) {
    if (has) {  // decode.cpp:89-98
      for (int j = lane; j < blen; j += 32)
        b.res_tok[static_cast<long long>(s) * T + j] = b.best_tok[static_cast<long long>(s) * T + j];
      if (lane == 0) {
        b.res_len[s] = blen;
        b.res_lp[s] = blp;
        b.res_norm[s] = bnorm;
        b.res_flags[s] = 1u;
      }
    } else {  // decode.cpp:99-108: first max over live, truncated
      const float len = static_cast<float>(t + 1) + 1.0f;
      const float den = det_powf(__fdiv_rn(__fadd_rn(5.0f, len), 6.0f), b.alpha);
      // First max of my_lp / den over lanes < new_live (lowest lane on ties).
      float bn = lane < new_live ? __fdiv_rn(my_lp, den) : kNegInf;
      int bq = lane < new_live ? lane : INT_MAX;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float on = __shfl_xor_sync(0xffffffffu, bn, o);
        const int oq = __shfl_xor_sync(0xffffffffu, bq, o);
        if (oq != INT_MAX && (bq == INT_MAX || on > bn || (on == bn && oq < bq))) {
          bn = on;
          bq = oq;
        }
      }
      const int pr = __shfl_sync(0xffffffffu, my_parent, bq);
      const int tk = __shfl_sync(0xffffffffu, my_tok, bq);
      const float lpq = __shfl_sync(0xffffffffu, my_lp, bq);
      for (int j = lane; j < t; j += 32)
        b.res_tok[static_cast<long long>(s) * T + j] = tok_cur[static_cast<long long>(pr) * T + j];
      if (lane == 0) {
        b.res_tok[static_cast<long long>(s) * T + t] = tk;
        b.res_len[s] = t + 1;
        b.res_lp[s] = lpq;
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

// One warp: candidates of sentence s (cand_score / cand_tok of its live rows,
// or cs_sm / ct_sm in shared memory at [row of the sentence * B + slot];
// scratch: 96 words of the warp's shared memory)
// -> sel_* (surviving hypotheses), finished-list update, termination and the
// sentence result; writes sent_live[s]. decode.cpp:55-109 with the stable
// sort of the candidates replaced by ranks in the same total order
// (score desc, parent asc, token asc): lane c holds candidate c and counts
// the candidates ranked above it, so the kB-way selection needs no
// sequential argmax rounds. Of the selected EOS candidates only the best
// ranked can update the finished best (its normalised score is the largest
// of this step's, and later ones only replace it on a strictly larger one).
__device__ __forceinline__ void select_sentence(const BeamDev& b, int s, int t, int lane,
                                                const SentState& st,
                                                float* scratch, const float* cs_sm = nullptr,
                                                const int* ct_sm = nullptr) {
  const int kB = min(b.B, b.V);
  if (st.done) return;
  const int nc = st.L * kB;
  if (nc > 32) {
    select_sentence_seq(b, s, t, lane, st);
    return;
  }
  const int T = b.T;
  const int* tok_cur = b.tok[t & 1];
  const int r0 = st.r0;
  float cs = kNegInf;
  int cp = INT_MAX, ct = INT_MAX;
  if (lane < nc) {
    const int p = lane / kB, e = lane - p * kB;
    cs = cs_sm ? cs_sm[p * b.B + e] : b.cand_score[static_cast<long long>(r0 + p) * b.B + e];
    ct = ct_sm ? ct_sm[p * b.B + e] : b.cand_tok[static_cast<long long>(r0 + p) * b.B + e];
    cp = p;
  }
  // no candidate (NaN logits) never competes
  const bool valid = lane < nc && ct >= 0 && ct < b.V && cs == cs;
  const unsigned vmask = __ballot_sync(0xffffffffu, valid);
  const int n_valid = __popc(vmask);
  if (n_valid == 0) {  // invalid logits for this sentence: fail it (ValueError)
    if (lane == 0) {
      b.res_status[s] = 2;
      b.res_flags[s] = 4u;
      b.res_len[s] = 0;
      b.sent_done[s] = 1;
      b.sent_live[s] = 0;
    }
    __syncwarp();
    return;
  }
  // decode.cpp:71: take min(|cands|, beam)
  const int n_sel = min(b.B, n_valid);
  // Ranks: every lane compares its candidate with all others through a
  // per-warp shared copy (independent broadcast loads; a shuffle-based sort
  // costs ~200 cycles per dependent stage, tools/micro/warp_sort_bench.cu).
  float* x_s = scratch;
  int* x_p = reinterpret_cast<int*>(scratch + 32);
  int* x_t = reinterpret_cast<int*>(scratch + 64);
  x_s[lane] = cs;
  x_p[lane] = cp;
  x_t[lane] = valid ? ct : INT_MAX;
  __syncwarp();
  int rank = 0, eos_above = 0;
#pragma unroll 5
  for (int j = 0; j < nc; ++j) {
    const float sj = x_s[j];
    const int pj = x_p[j], tj = x_t[j];
    const bool above = tj != INT_MAX && better3(sj, pj, tj, cs, cp, ct);
    rank += above;
    eos_above += above && tj == kEosIdDev;
  }
  __syncwarp();
  const bool valid_sorted = valid;
  const bool sel = valid_sorted && rank < n_sel;
  const bool eos = sel && ct == kEosIdDev;
  // decode.cpp:77-80 + first max of normalized_score over finished
  const unsigned first_eos = __ballot_sync(0xffffffffu, eos && eos_above == 0);
  int has = st.has, blen = st.blen;
  float bnorm = st.bnorm, blp = st.blp;
  if (first_eos) {
    const int src = __ffs(first_eos) - 1;
    const float bs = __shfl_sync(0xffffffffu, cs, src);
    const int pr = r0 + __shfl_sync(0xffffffffu, cp, src);
    const float len = static_cast<float>(t) + 1.0f;
    const float norm = __fdiv_rn(bs, det_powf(__fdiv_rn(__fadd_rn(5.0f, len), 6.0f), b.alpha));
    if (!has || norm > bnorm) {
      for (int j = lane; j < t; j += 32)
        b.best_tok[static_cast<long long>(s) * T + j] = tok_cur[static_cast<long long>(pr) * T + j];
      has = 1;
      bnorm = norm;
      blp = bs;
      blen = t;
      if (lane == 0) {
        b.best_has[s] = 1;
        b.best_norm[s] = norm;
        b.best_lp[s] = bs;
        b.best_len[s] = t;
      }
    }
  }
  // Surviving selections in rank order: slot q = rank - EOS ranked above.
  const bool keep = sel && !eos;
  const int q = keep ? rank - eos_above : INT_MAX;
  if (keep) {
    b.sel_parent[s * b.B + q] = r0 + cp;
    b.sel_tok[s * b.B + q] = ct;
    b.sel_lp[s * b.B + q] = cs;
  }
  int new_live = __popc(__ballot_sync(0xffffffffu, keep));
  const int maxlen = st.maxlen;
  if (new_live > 0 && t + 1 >= b.max_seq_len && maxlen > b.max_seq_len) {
    // decode_step would be called past max_seq_len (model.cpp:618-619).
    if (lane == 0) {
      b.res_status[s] = 2;  // ValueError
      b.res_flags[s] = 4u;
      b.res_len[s] = 0;
      b.sent_done[s] = 1;
    }
    new_live = 0;
  } else if (new_live == 0 || t + 1 >= maxlen) {
    if (has) {  // decode.cpp:89-98
      for (int j = lane; j < blen; j += 32)
        b.res_tok[static_cast<long long>(s) * T + j] = b.best_tok[static_cast<long long>(s) * T + j];
      if (lane == 0) {
        b.res_len[s] = blen;
        b.res_lp[s] = blp;
        b.res_norm[s] = bnorm;
        b.res_flags[s] = 1u;
      }
    } else {  // decode.cpp:99-108: first max over live, truncated
      const float len = static_cast<float>(t + 1) + 1.0f;
      const float den = det_powf(__fdiv_rn(__fadd_rn(5.0f, len), 6.0f), b.alpha);
      // First max of lp / den over the survivors (lowest slot q on ties).
      float bn = keep ? __fdiv_rn(cs, den) : kNegInf;
      int bq = q, bl = lane;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float on = __shfl_xor_sync(0xffffffffu, bn, o);
        const int oq = __shfl_xor_sync(0xffffffffu, bq, o);
        const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
        if (oq != INT_MAX && (bq == INT_MAX || on > bn || (on == bn && oq < bq))) {
          bn = on;
          bq = oq;
          bl = ol;
        }
      }
      const int pr = r0 + __shfl_sync(0xffffffffu, cp, bl);
      const int tk = __shfl_sync(0xffffffffu, ct, bl);
      const float lpq = __shfl_sync(0xffffffffu, cs, bl);
      for (int j = lane; j < t; j += 32)
        b.res_tok[static_cast<long long>(s) * T + j] = tok_cur[static_cast<long long>(pr) * T + j];
      if (lane == 0) {
        b.res_tok[static_cast<long long>(s) * T + t] = tk;
        b.res_len[s] = t + 1;
        b.res_lp[s] = lpq;
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

// All threads of the CTA: ticket on sel_count; the last CTA of the grid
// (shared live_s [N], row0_s [N + N / 32 + 1])
// scans the live counts, writes the compacted rows and advances the step.
// live_s / row0_s: [N] shared ints; is_last: one shared int.
__device__ __forceinline__ void finish_select(const BeamDev& b, int t, int* live_s, int* row0_s,
                                              int* is_last, const KTrace* tr = nullptr) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // Last-CTA election: every CTA's writes are made visible before its ticket.
  // A single-CTA grid (batch-1) is its own last CTA: the block barrier makes
  // its global writes visible to its threads without the fence round trips.
  __syncthreads();
  if (gridDim.x > 1) {
    if (threadIdx.x == 0) {
      __threadfence();
      *is_last = atomicAdd(b.sel_count, 1) == static_cast<int>(gridDim.x) - 1;
    }
    __syncthreads();
    if (!*is_last) return;
    __threadfence();
  }
  if (tr && threadIdx.x == 0) trace_phase_at(*tr, t, 3);
  // One round trip: the live counts and the first batch of selections (all
  // slots; the dead ones are filtered after the scan).
  constexpr int kBatch = 4;
  const int total = b.N * b.B;
  int par[kBatch], tok[kBatch];
  float lp[kBatch];
#pragma unroll
  for (int u = 0; u < kBatch; ++u) {
    const int idx = threadIdx.x + u * blockDim.x;
    const bool on = idx < total;
    par[u] = on ? __ldcg(b.sel_parent + idx) : 0;
    tok[u] = on ? __ldcg(b.sel_tok + idx) : 0;
    lp[u] = on ? __ldcg(b.sel_lp + idx) : 0.0f;
  }
  for (int s = threadIdx.x; s < b.N; s += blockDim.x) live_s[s] = __ldcg(b.sent_live + s);
  __syncthreads();
  // Exclusive scan of the live counts: warps scan 32-sentence chunks in
  // parallel (inclusive, into row0_s), thread 0 chains the chunk totals.
  const int nwarps = blockDim.x >> 5, nchunks = (b.N + 31) / 32;
  for (int c = warp; c < nchunks; c += nwarps) {
    const int s = c * 32 + lane;
    const int v = s < b.N ? live_s[s] : 0;
    int inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += u;
    }
    if (s < b.N) row0_s[s] = inc;
  }
  __syncthreads();
  int* chunk_base = row0_s + b.N;  // [N / 32 + 1]
  if (threadIdx.x == 0) {
    int base = 0;
    for (int c = 0; c < nchunks; ++c) {
      chunk_base[c] = base;
      base += row0_s[min(b.N, c * 32 + 32) - 1];
    }
    *b.n_rows = base;
  }
  __syncthreads();
  for (int s = threadIdx.x; s < b.N; s += blockDim.x) {  // exclusive offsets
    const int ex = chunk_base[s >> 5] + row0_s[s] - live_s[s];
    row0_s[s] = ex;
    b.sent_row0[s] = ex;
  }
  __syncthreads();
  // Compacted rows: thread per (sentence, slot), the first batch already in
  // registers.
  for (int base = threadIdx.x; base < total; base += kBatch * blockDim.x) {
    if (base != threadIdx.x) {
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        const int idx = base + u * blockDim.x;
        const bool on = idx < total;
        par[u] = on ? __ldcg(b.sel_parent + idx) : 0;
        tok[u] = on ? __ldcg(b.sel_tok + idx) : 0;
        lp[u] = on ? __ldcg(b.sel_lp + idx) : 0.0f;
      }
    }
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const int idx = base + u * blockDim.x;
      if (idx < total) {
        const int s = idx / b.B, q = idx % b.B;
        if (q < live_s[s]) {
          const int row = row0_s[s] + q;
          b.row_sent[row] = s;
          b.row_parent[row] = par[u];
          b.row_prev[row] = tok[u];
          b.row_lp[row] = lp[u];
        }
      }
    }
  }
  if (threadIdx.x == 0) {
    *b.step = t + 1;
    *b.sel_count = 0;
    if (tr) trace_phase_at(*tr, t, 4);
  }
}

}  // namespace mtg
