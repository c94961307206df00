// log_softmax_row + candidate scores + per-row top-kB (decode.cpp:25-30,
// 55-69), from the partials the output-projection GEMM epilogue leaves behind
// (gemm_tc.cuh, kEpiSoftmaxParts): for every 32-column slice k of a row, its
// max m_k, first argmax column a_k and s_k = sum_j exp(x_j - m_k) in column
// order. One 128-thread CTA per live hypothesis row:
//
//   M   = max_k m_k
//   S   = sum over k of u_k,  u_k = s_k * exp(m_k - M)  (0 if m_k = -inf), in
//         the P6 order: thread t of 128 sums k = t + 128 i in i order, P1
//         butterfly per warp, then (W0 + W1) + (W2 + W3)
//   lse = log(S) + M                                      (P6)
//   score(x) = fl(parent_logprob + fl(x - lse))
//
// Top-kB by (score desc, token asc), exact: score is monotone in x, so an
// element of slice k scores at most score(m_k). Let S_kB be the kB-th best
// slice-max score (by the same order). Every element outside the slices with
// score(m_k) >= S_kB scores < S_kB and ranks below kB slice maxima, so the
// exact top-kB lies in those slices -- normally exactly kB of them -- which
// are rescanned from the logits the GEMM wrote.
#include <algorithm>
#include <climits>
#include <map>
#include <mutex>
#include <type_traits>

#include "beam_dev.cuh"
#include "detmath.cuh"
#include "errors.hpp"
#include "kernels.cuh"
#include "launch.cuh"

namespace mtg {

namespace {

#define kNegInf (-__int_as_float(0x7f800000))
#define kPosInf (__int_as_float(0x7f800000))
constexpr int kMT = 128;                                 // threads per row (4 warps)
constexpr int kSubPerThread = kMaxSoftmaxSlices / kMT;  // slices per thread (registers)
constexpr int kCache = 4;                                // rescanned slices per warp in registers

// Branch-free, as better3 (beam_dev.cuh).
__device__ __forceinline__ bool better2(float a, int ta, float b, int tb) {
  return (a > b) | ((a == b) & (ta < tb));
}

// Warp-wide argmax of (score desc, token asc); every lane gets the winner.
__device__ __forceinline__ void warp_best(float& bs, int& bt) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float os = __shfl_xor_sync(0xffffffffu, bs, o);
    const int ot = __shfl_xor_sync(0xffffffffu, bt, o);
    if (ot != INT_MAX && (bt == INT_MAX || better2(os, ot, bs, bt))) {
      bs = os;
      bt = ot;
    }
  }
}

// Barrier of one 128-thread group (id 0 with a 128-thread CTA == __syncthreads).
__device__ __forceinline__ void grp_sync(int id) {
  asm volatile("bar.sync %0, 128;" ::"r"(id) : "memory");
}

// Group-wide (4 warps) argmax; every thread gets the winner. tid: 0..127.
__device__ __forceinline__ void block_best(float& bs, int& bt, float* rf, int* ri, int tid,
                                           int bar) {
  const int lane = tid & 31, warp = tid >> 5;
  warp_best(bs, bt);
  if (lane == 0) {
    rf[warp] = bs;
    ri[warp] = bt;
  }
  grp_sync(bar);
  bs = rf[0];
  bt = ri[0];
#pragma unroll
  for (int w = 1; w < kMT / 32; ++w)
    if (ri[w] != INT_MAX && (bt == INT_MAX || better2(rf[w], ri[w], bs, bt))) {
      bs = rf[w];
      bt = ri[w];
    }
  grp_sync(bar);
}

// Bitonic sort of one (score, token) pair per lane across the warp, best
// first in the (score desc, token asc) order; empty entries (token INT_MAX)
// sort last. Lane k ends with the k-th best.
__device__ __forceinline__ void warp_sort_best_first(float& s, int& t, int lane) {
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const float os = __shfl_xor_sync(0xffffffffu, s, j);
      const int ot = __shfl_xor_sync(0xffffffffu, t, j);
      const bool o_better =
          ot != INT_MAX && (t == INT_MAX || better2(os, ot, s, t));
      const bool keep_better = ((lane & k) == 0) == ((lane & j) == 0);
      if (keep_better ? o_better : (!o_better && ot != t)) {
        s = os;
        t = ot;
      }
    }
  }
}

// Per-group shared scratch of the row routines: CAP ints of rescan list
// (merge, kMaxSoftmaxSlices) or shortlist logits (kMaxShortlist).
constexpr int kSurvCap = 128;  // rescanned elements at or above the threshold

template <int CAP>
struct RowScratchT {
  float red_f[kMT / 32];
  int red_i[kMT / 32];
  int n_list;
  int n_surv;
  float surv_s[kSurvCap];
  int surv_t[kSurvCap];
  int list[CAP];
};
using MergeScratch = RowScratchT<kMaxSoftmaxSlices>;
using ShortlistScratch = RowScratchT<kMaxShortlist>;

// One CTA (128 threads) per live hypothesis row; thread t owns slices
// t + 128 i. Sum order P6: thread partials in i order, P1 butterfly per warp,
// then (W0 + W1) + (W2 + W3).
__device__ __forceinline__ void merge_row(int r, const float* __restrict__ logits, long long ldl,
                                      const float* __restrict__ part_m,
                                      const float* __restrict__ part_s,
                                      const int* __restrict__ part_arg, long long part_ld,
                                      int nsub, const BeamDev& b, int tid, int bar,
                                      MergeScratch& sc_, const KTrace* tr = nullptr, int t = 0,
                                      float* cs_sm = nullptr, int* ct_sm = nullptr) {
  // Candidate slot k of this row: shared memory (fused tail) or global.
  auto put = [&](int k, float score, int tok) {
    if (cs_sm) {
      cs_sm[k] = score;
      ct_sm[k] = tok;
    } else {
      b.cand_score[static_cast<long long>(r) * b.B + k] = score;
      b.cand_tok[static_cast<long long>(r) * b.B + k] = tok;
    }
  };
  float* red_f = sc_.red_f;
  int* red_i = sc_.red_i;
  int* list_s = sc_.list;
  int& n_list_s = sc_.n_list;
  const int lane = tid & 31, warp = tid >> 5;
  const int V = b.V;
  const int kB = min(b.B, V);
  const float* pm = part_m + r * part_ld;
  const float* ps = part_s + r * part_ld;
  const int* pa = part_arg + r * part_ld;
  const float* x = logits + r * ldl;
  const float plp = b.row_lp[r];
  if (tid == 0) {
    n_list_s = 0;
    sc_.n_surv = 0;
  }

  // All partial loads first (one L2 round trip), then the math.
  float mv[kSubPerThread], sv[kSubPerThread];
  int at[kSubPerThread];
#pragma unroll
  for (int i = 0; i < kSubPerThread; ++i) {
    const int k = tid + kMT * i;
    const bool ok = k < nsub;
    mv[i] = ok ? pm[k] : kNegInf;
    sv[i] = ok ? ps[k] : 0.0f;
    at[i] = ok ? pa[k] : -1;
  }
  float mloc = kNegInf;
#pragma unroll
  for (int i = 0; i < kSubPerThread; ++i) mloc = fmaxf(mloc, mv[i]);
  mloc = warp_allmax(mloc);
  if (lane == 0) red_f[warp] = mloc;
  grp_sync(bar);
  const float M = fmaxf(fmaxf(red_f[0], red_f[1]), fmaxf(red_f[2], red_f[3]));
  grp_sync(bar);
  float part = 0.0f;
#pragma unroll
  for (int i = 0; i < kSubPerThread; ++i) {
    if (tid + kMT * i < nsub) {
      const float u =
          mv[i] == kNegInf ? 0.0f : __fmul_rn(sv[i], det_expf_nonpos(__fsub_rn(mv[i], M)));
      part = __fadd_rn(part, u);
    }
  }
  part = warp_allsum(part);
  if (lane == 0) red_f[warp] = part;
  grp_sync(bar);
  const float total = __fadd_rn(__fadd_rn(red_f[0], red_f[1]), __fadd_rn(red_f[2], red_f[3]));
  grp_sync(bar);
  const float lse = __fadd_rn(det_logf(total), M);
  if (tr && tid == 0) trace_phase_at(*tr, t, 5);

  // Slice-max scores; a slice with no max (all NaN / empty) never competes.
  float sc[kSubPerThread];
#pragma unroll
  for (int i = 0; i < kSubPerThread; ++i) {
    sc[i] = __fadd_rn(plp, __fsub_rn(mv[i], lse));
    if (sc[i] != sc[i]) at[i] = -1;
  }
  // Rescan threshold T <= the kB-th best slice maximum (exactness needs no
  // more): every warp sorts its 32 threads' best slice maxima and offers its
  // kB-th; T = the best offer. That warp has kB slice maxima at or above T,
  // so the kB-th best slice maximum is too, and the rescan set (slices whose
  // maximum scores >= T) holds every top-kB element. No offer (fewer than kB
  // valid slices in every warp): every valid slice is rescanned.
  float thr = kNegInf;
  {
    float ts = kNegInf;
    int tt = INT_MAX;
#pragma unroll
    for (int i = 0; i < kSubPerThread; ++i)
      if (at[i] >= 0 && (tt == INT_MAX || better2(sc[i], at[i], ts, tt))) {
        ts = sc[i];
        tt = at[i];
      }
    warp_sort_best_first(ts, tt, lane);
    const float ws = __shfl_sync(0xffffffffu, ts, kB - 1);
    const int wt = __shfl_sync(0xffffffffu, tt, kB - 1);
    if (lane == 0) {
      red_f[warp] = ws;
      red_i[warp] = wt;
    }
    grp_sync(bar);
    float bs = kNegInf;
    int bt = INT_MAX;
#pragma unroll
    for (int w = 0; w < kMT / 32; ++w)
      if (red_i[w] != INT_MAX && (bt == INT_MAX || better2(red_f[w], red_i[w], bs, bt))) {
        bs = red_f[w];
        bt = red_i[w];
      }
    grp_sync(bar);
    if (bt != INT_MAX) thr = bs;
  }
  if (tr && tid == 0) trace_phase_at(*tr, t, 6);
  // Slices to rescan: score(m_k) >= thr (normally exactly kB of them).
#pragma unroll
  for (int i = 0; i < kSubPerThread; ++i)
    if (at[i] >= 0 && sc[i] >= thr) list_s[atomicAdd(&n_list_s, 1)] = tid + kMT * i;
  grp_sync(bar);
  const int n_list = n_list_s;
  // Exact top-kB over the rescanned slices: warp w takes list entries
  // w, w + 4, ...; lane = column within the slice.
  constexpr int kW = kMT / 32;
  float cs[kCache];
  int cc[kCache];
#pragma unroll
  for (int e = 0; e < kCache; ++e) {  // loads issued back to back (clamped address)
    const int idx = warp + kW * e;
    cc[e] = idx < n_list ? list_s[idx] * 32 + lane : V;
    cs[e] = x[min(cc[e], V - 1)];
  }
#pragma unroll
  for (int e = 0; e < kCache; ++e)
    cs[e] = cc[e] < V ? __fadd_rn(plp, __fsub_rn(cs[e], lse)) : kNegInf;
  // Survivors: rescanned elements scoring >= T (at least kB of them: the
  // kB slice maxima at or above T). Their rank in (score desc, token asc)
  // order is their candidate slot.
  int* n_surv_s = &sc_.n_surv;
#pragma unroll
  for (int e = 0; e < kCache; ++e) {
    const int col = cc[e];
    if (col < V && cs[e] == cs[e] && cs[e] >= thr) {
      const int at_ = atomicAdd(n_surv_s, 1);
      if (at_ < kSurvCap) {
        sc_.surv_s[at_] = cs[e];
        sc_.surv_t[at_] = col;
      }
    }
  }
  for (int idx = warp + kW * kCache; idx < n_list; idx += kW) {  // long lists (ties)
    const int col = list_s[idx] * 32 + lane;
    if (col < V) {
      const float sv = __fadd_rn(plp, __fsub_rn(x[col], lse));
      if (sv == sv && sv >= thr) {
        const int at_ = atomicAdd(n_surv_s, 1);
        if (at_ < kSurvCap) {
          sc_.surv_s[at_] = sv;
          sc_.surv_t[at_] = col;
        }
      }
    }
  }
  grp_sync(bar);
  const int n_surv = *n_surv_s;
  if (n_surv <= kSurvCap) {
    for (int i = tid; i < n_surv; i += kMT) {
      const float si = sc_.surv_s[i];
      const int ti = sc_.surv_t[i];
      int rank = 0;
      for (int j = 0; j < n_surv; ++j) rank += better2(sc_.surv_s[j], sc_.surv_t[j], si, ti);
      if (rank < kB) put(rank, si, ti);
    }
    for (int k = n_surv + tid; k < kB; k += kMT) put(k, kNegInf, INT_MAX);  // fewer valid elements than kB
  } else {
    // Many ties at T (degenerate logits): kB group-wide argmax rounds.
    float last_s = kPosInf;
    int last_t = -1;
    for (int k = 0; k < kB; ++k) {
      float bs = kNegInf;
      int bt = INT_MAX;
#pragma unroll
      for (int e = 0; e < kCache; ++e) {
        const int col = cc[e];
        if (col < V && cs[e] == cs[e] && better2(last_s, last_t, cs[e], col) &&
            (bt == INT_MAX || better2(cs[e], col, bs, bt))) {
          bs = cs[e];
          bt = col;
        }
      }
      for (int idx = warp + kW * kCache; idx < n_list; idx += kW) {  // long lists (ties)
        const int col = list_s[idx] * 32 + lane;
        if (col < V) {
          const float s = __fadd_rn(plp, __fsub_rn(x[col], lse));
          if (s == s && better2(last_s, last_t, s, col) && (bt == INT_MAX || better2(s, col, bs, bt))) {
            bs = s;
            bt = col;
          }
        }
      }
      block_best(bs, bt, red_f, red_i, tid, bar);
      if (tid == 0) {
        for (int kk = k; kk < (bt == INT_MAX ? kB : k + 1); ++kk)  // the rest invalid too
          put(kk, bt == INT_MAX ? kNegInf : bs, bt);
      }
      if (bt == INT_MAX) break;
      last_s = bs;
      last_t = bt;
    }
  }
  if (tr && tid == 0) trace_phase_at(*tr, t, 7);
  // Slots past kB (a vocabulary smaller than the beam) are invalid.
  for (int k = kB + tid; k < b.B; k += kMT) put(k, kNegInf, INT_MAX);
}

__global__ void __launch_bounds__(kMT)
    softmax_topk_kernel(const float* __restrict__ logits, long long ldl,
                        const float* __restrict__ part_m, const float* __restrict__ part_s,
                        const int* __restrict__ part_arg, long long part_ld, int nsub,
                        BeamDev b) {
  pdl_wait();
  pdl_trigger();
  const int t0 = b.tr_a.buf ? *b.step : 0;
  trace_begin_at(b.tr_a, t0);
  __shared__ MergeScratch sc;
  const int r = blockIdx.x;
  if (r < *b.n_rows)  // uniform over the CTA
    merge_row(r, logits, ldl, part_m, part_s, part_arg, part_ld, nsub, b, threadIdx.x, 0, sc);
  trace_end_at(b.tr_a, t0);
}

// ---- vocabulary shortlist (decode.cpp:55-61 with rows; model.cpp:440-449) ----
// One 128-thread CTA per live row r of sentence s with shortlist L_s (sorted
// full-vocabulary ids, n = |L_s| <= kMaxShortlist): logits of the shortlist
// rows only, then log_softmax over those n values (P6 over subset
// positions, exactly as over a full row) and the top-kB by (score desc,
// token asc) with token = L_s[j].
//   int8 : acc = sum a_q * w_q (exact int32), x = float(acc) * (1/(sa*sw))
//          -- the same value the full projection produces (qmatmul_nt rows).
//   fp32 : 8 interleaved partial sums, ((a0+a1)+(a2+a3))+((a4+a5)+(a6+a7))
//          (the oracle's dot8 stand-in for Eigen's dot, tensor.cpp:125-133).
//   bf16 : bf16 operands, products summed in fp32 in k order.
template <int PREC>
__device__ __forceinline__ void shortlist_row(int r, const ShortlistArgs& a, const BeamDev& b,
                                          int tid, int bar, ShortlistScratch& sc_) {
  float* lg = reinterpret_cast<float*>(sc_.list);  // kMaxShortlist floats
  float* red_f = sc_.red_f;
  int* red_i = sc_.red_i;
  const int lane = tid & 31, warp = tid >> 5;
  const int s = b.row_sent[r];
  const int* ids = a.sl_ids + a.sl_off[s];
  const int n = a.sl_off[s + 1] - a.sl_off[s];
  const int K = a.K;
  const float plp = b.row_lp[r];
  float inv = 1.0f;
  if constexpr (PREC == 0) inv = __frcp_rn(__fmul_rn(a.a_scale[r], a.w_scale));
  for (int j = tid; j < n; j += kMT) {
    const long long col = ids[j];
    float x;
    if constexpr (PREC == 0) {  // int8, K padded to 16 bytes
      const int4* av = reinterpret_cast<const int4*>(a.aq + static_cast<long long>(r) * a.lda);
      const int4* wv = reinterpret_cast<const int4*>(a.wq + col * a.ldw);
      int acc = 0;
      for (int k = 0; k < a.lda / 16; ++k) {
        const int4 p = av[k], q = wv[k];
        acc = __dp4a(p.x, q.x, acc);
        acc = __dp4a(p.y, q.y, acc);
        acc = __dp4a(p.z, q.z, acc);
        acc = __dp4a(p.w, q.w, acc);
      }
      x = __fmul_rn(__int2float_rn(acc), inv);
    } else if constexpr (PREC == 1) {
      const __nv_bfloat16* ar = a.ah + static_cast<long long>(r) * a.lda;
      const __nv_bfloat16* wr = a.wh + col * a.ldw;
      float acc = 0.0f;
      for (int k = 0; k < K; ++k)
        acc = __fadd_rn(acc, __fmul_rn(__bfloat162float(ar[k]), __bfloat162float(wr[k])));
      x = acc;
    } else {
      const float* ar = a.af + static_cast<long long>(r) * a.lda;
      const float* wr = a.wf + col * a.ldw;
      float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      int k = 0;
      for (; k + 8 <= K; k += 8)
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] = __fadd_rn(acc[u], __fmul_rn(ar[k + u], wr[k + u]));
      for (; k < K; ++k) acc[k & 7] = __fadd_rn(acc[k & 7], __fmul_rn(ar[k], wr[k]));
      x = __fadd_rn(__fadd_rn(__fadd_rn(acc[0], acc[1]), __fadd_rn(acc[2], acc[3])),
                    __fadd_rn(__fadd_rn(acc[4], acc[5]), __fadd_rn(acc[6], acc[7])));
    }
    lg[j] = x;
  }
  grp_sync(bar);
  // log-sum-exp in the P6 order over the n subset positions.
  const int nsub = (n + 31) / 32;
  float mloc = kNegInf;
  float mv[kMaxShortlist / 32 / kMT + 1];
  float sv[kMaxShortlist / 32 / kMT + 1];
#pragma unroll
  for (int i = 0; i < kMaxShortlist / 32 / kMT + 1; ++i) {
    const int k = tid + kMT * i;
    mv[i] = kNegInf;
    sv[i] = 0.0f;
    if (k < nsub) {
      const int j0 = 32 * k, j1 = min(n, j0 + 32);
      float best = kNegInf;
      bool any = false;
      for (int j = j0; j < j1; ++j)
        if (lg[j] > best) {
          best = lg[j];
          any = true;
        }
      float sum = 0.0f;
      if (any)
        for (int j = j0; j < j1; ++j) sum = __fadd_rn(sum, det_expf_nonpos(__fsub_rn(lg[j], best)));
      mv[i] = best;
      sv[i] = sum;
      mloc = fmaxf(mloc, best);
    }
  }
  mloc = warp_allmax(mloc);
  if (lane == 0) red_f[warp] = mloc;
  grp_sync(bar);
  const float M = fmaxf(fmaxf(red_f[0], red_f[1]), fmaxf(red_f[2], red_f[3]));
  grp_sync(bar);
  float part = 0.0f;
#pragma unroll
  for (int i = 0; i < kMaxShortlist / 32 / kMT + 1; ++i)
    if (tid + kMT * i < nsub) {
      const float u =
          mv[i] == kNegInf ? 0.0f : __fmul_rn(sv[i], det_expf_nonpos(__fsub_rn(mv[i], M)));
      part = __fadd_rn(part, u);
    }
  part = warp_allsum(part);
  if (lane == 0) red_f[warp] = part;
  grp_sync(bar);
  const float total = __fadd_rn(__fadd_rn(red_f[0], red_f[1]), __fadd_rn(red_f[2], red_f[3]));
  grp_sync(bar);
  const float lse = __fadd_rn(det_logf(total), M);
  // Top-kB by (score desc, token asc), token = ids[j].
  const int kB = min(b.B, n);
  float last_s = kPosInf;
  int last_t = -1;
  for (int k = 0; k < kB; ++k) {
    float bs = kNegInf;
    int bt = INT_MAX;
    for (int j = tid; j < n; j += kMT) {
      const float sc = __fadd_rn(plp, __fsub_rn(lg[j], lse));
      const int tk = ids[j];
      if (sc == sc && better2(last_s, last_t, sc, tk) && (bt == INT_MAX || better2(sc, tk, bs, bt))) {
        bs = sc;
        bt = tk;
      }
    }
    block_best(bs, bt, red_f, red_i, tid, bar);
    if (tid == 0) {
      b.cand_score[static_cast<long long>(r) * b.B + k] = bt == INT_MAX ? kNegInf : bs;
      b.cand_tok[static_cast<long long>(r) * b.B + k] = bt;
    }
    if (bt == INT_MAX) break;
    last_s = bs;
    last_t = bt;
  }
  for (int k = kB + tid; k < b.B; k += kMT) {
    b.cand_score[static_cast<long long>(r) * b.B + k] = kNegInf;
    b.cand_tok[static_cast<long long>(r) * b.B + k] = INT_MAX;
  }
}

template <int PREC>
__global__ void __launch_bounds__(kMT) shortlist_topk_kernel(ShortlistArgs a, BeamDev b) {
  pdl_wait();
  pdl_trigger();
  __shared__ ShortlistScratch sc;
  const int r = blockIdx.x;
  if (r >= *b.n_rows) return;
  shortlist_row<PREC>(r, a, b, threadIdx.x, 0, sc);
}

// ---- fused step tail --------------------------------------------------------
// One CTA per sentence: G = blockDim / 128 groups each run merge_row (or
// shortlist_row) for the sentence's live rows, then warp 0 runs the
// sentence's beam selection from those candidates and the last CTA compacts
// the rows (beam_dev.cuh) -- the work of softmax_topk_kernel +
// beam_select_kernel without the kernel boundary between them.
struct TailArgs {
  const float* logits;
  long long ldl;
  const float* part_m;
  const float* part_s;
  const int* part_arg;
  long long part_ld;
  int nsub;
};

template <int MODE>  // 0 full vocabulary; 1..3 shortlist with PREC = MODE - 1
__global__ void __launch_bounds__(1024) topk_select_kernel(TailArgs ta, ShortlistArgs sa,
                                                           BeamDev b) {
  extern __shared__ __align__(16) unsigned char tail_smem[];
  const int G = blockDim.x / kMT, g = threadIdx.x / kMT, tid = threadIdx.x % kMT;
  using Scratch = std::conditional_t<MODE == 0, MergeScratch, ShortlistScratch>;
  Scratch* scr = reinterpret_cast<Scratch*>(tail_smem);
  int* live_s = reinterpret_cast<int*>(scr + G);
  int* row0_s = live_s + b.N;
  float* cs_sm = reinterpret_cast<float*>(row0_s + b.N + b.N / 32 + 1);  // [B rows][B slots]
  int* ct_sm = reinterpret_cast<int*>(cs_sm + kMaxBeam * kMaxBeam);
  float* sel_scratch = reinterpret_cast<float*>(ct_sm + kMaxBeam * kMaxBeam);  // [96]
  __shared__ int is_last;
  __shared__ SentState st_s;
  const int s = blockIdx.x;
  // The sentence's beam state is the previous step tail's: loaded before the
  // dependency wait.
  if (threadIdx.x == 0) st_s = load_sent_state(b, s);
  pdl_wait();
  pdl_trigger();
  const int t = *b.step;
  trace_begin_at(b.tr_a, t);
  if (threadIdx.x == 0) trace_phase_at(b.tr_a, t, 0);
  __syncthreads();
  const SentState st = st_s;
  if (!st.done) {
    for (int i = g; i < st.L; i += G) {
      if constexpr (MODE == 0)
        merge_row(st.r0 + i, ta.logits, ta.ldl, ta.part_m, ta.part_s, ta.part_arg, ta.part_ld,
                  ta.nsub, b, tid, 1 + g, scr[g], g == 0 ? &b.tr_a : nullptr, t,
                  cs_sm + i * b.B, ct_sm + i * b.B);
      else
        shortlist_row<MODE - 1>(st.r0 + i, sa, b, tid, 1 + g, scr[g]);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) trace_phase_at(b.tr_a, t, 1);
  if (threadIdx.x < 32) {
    if constexpr (MODE == 0)
      select_sentence(b, s, t, threadIdx.x, st, sel_scratch, cs_sm, ct_sm);
    else
      select_sentence(b, s, t, threadIdx.x, st, sel_scratch);
  }
  if (threadIdx.x == 0) trace_phase_at(b.tr_a, t, 2);
  finish_select(b, t, live_s, row0_s, &is_last, &b.tr_a);
  trace_end_at(b.tr_a, t);
}

}  // namespace

long long topk_pitch(int V) {
  const long long per = 128;
  return (static_cast<long long>(V) + per - 1) / per * per;
}

long long softmax_part_pitch(int V) { return ((V + 31) / 32 + 3) / 4 * 4; }

void launch_topk_select(const float* logits, long long ldl, const float* part_m,
                        const float* part_s, const int* part_arg, long long part_ld,
                        const ShortlistArgs* sa, int prec, const BeamDev& b, cudaStream_t st) {
  if (b.B > kMaxBeam) fail(kUsageError, "beam size above 16 is not supported");
  const int nsub = (b.V + 31) / 32;
  if (!sa && nsub > kMaxSoftmaxSlices)
    fail(kUsageError, "target vocabularies above 32768 are not supported by top-k yet");
  const int G = std::min(b.B, 8);
  const size_t smem = (sa ? sizeof(ShortlistScratch) : sizeof(MergeScratch)) * G +
                      sizeof(int) * (2 * static_cast<size_t>(b.N) + b.N / 32 + 1) +
                      (sizeof(float) + sizeof(int)) * kMaxBeam * kMaxBeam + sizeof(float) * 96;
  if (smem > 227 * 1024) fail(kUsageError, "beam search: too many sentences in one batch");
  TailArgs ta{logits, ldl, part_m, part_s, part_arg, part_ld, nsub};
  const ShortlistArgs none{};
  auto launch = [&](auto kern) {
    ensure_smem_attr(kern, smem);
    launch_k(kern, b.N, kMT * G, smem, st, ta, sa ? *sa : none, b);
  };
  if (!sa) launch(topk_select_kernel<0>);
  else if (prec == 0) launch(topk_select_kernel<1>);
  else if (prec == 1) launch(topk_select_kernel<2>);
  else launch(topk_select_kernel<3>);
  MTG_CUDA(cudaGetLastError());
}

void launch_shortlist_topk(int prec, const ShortlistArgs& a, const BeamDev& b, cudaStream_t st) {
  if (b.B > kMaxBeam) fail(kUsageError, "beam size above 16 is not supported");
  if (prec == 0 && a.lda % 16 != 0) fail(kStateError, "shortlist: int8 operand pitch");
  const dim3 grid(b.R_max), block(kMT);
  if (prec == 0)
    launch_k(shortlist_topk_kernel<0>, grid, block, 0, st, a, b);
  else if (prec == 1)
    launch_k(shortlist_topk_kernel<1>, grid, block, 0, st, a, b);
  else
    launch_k(shortlist_topk_kernel<2>, grid, block, 0, st, a, b);
  MTG_CUDA(cudaGetLastError());
}

void launch_softmax_topk(const float* logits, long long ldl, const float* part_m,
                         const float* part_s, const int* part_arg, long long part_ld,
                         const BeamDev& b, cudaStream_t st) {
  if (b.B > kMaxBeam) fail(kUsageError, "beam size above 16 is not supported");
  const int nsub = (b.V + 31) / 32;
  if (nsub > kMaxSoftmaxSlices)
    fail(kUsageError, "target vocabularies above 32768 are not supported by top-k yet");
  if (part_ld < nsub || ldl < b.V) fail(kStateError, "softmax_topk: pitches");
  const dim3 grid(b.R_max), block(kMT);
  launch_k(softmax_topk_kernel, grid, block, 0, st, logits, ldl, part_m, part_s, part_arg, part_ld,
           nsub, b);
  MTG_CUDA(cudaGetLastError());
}

}  // namespace mtg
