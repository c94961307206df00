// log_softmax_row + candidate scores + per-row top-kB (decode.cpp:25-30,
// 55-69), one 1024-thread CTA per live hypothesis row.
//
// Thread t owns logits 4(t + 1024 i) + c, i < NV4, held in registers (one
// HBM pass). The logits pitch is a multiple of 4096 and the pad columns hold
// -inf (written once at allocation), so there are no bounds checks: a pad
// element adds exp(-inf) = +0 to the sum and never scores. Sum order P2.
//
// Top-kB by (score desc, token asc), score = fl(parent + fl(x - lse)), exact:
// tau = kB-th largest per-warp max is <= the kB-th largest logit and score
// is monotone in x, so every true top-kB element has score >= score(tau).
// Those go to a shared list (normally ~kB entries) and warp 0 selects them
// exactly; larger lists take block-wide rounds, and rows whose list
// overflows (e.g. all-equal logits) take the exact slow path.
#include <climits>

#include "detmath.cuh"
#include "errors.hpp"
#include "kernels.cuh"
#include "launch.cuh"

namespace mtg {

namespace {

#define kNegInf (-__int_as_float(0x7f800000))
constexpr int kListCap = 2048;

__device__ __forceinline__ bool better2(float a, int ta, float b, int tb) {
  return a > b || (a == b && ta < tb);
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

// Block-wide argmax over one candidate per thread; every thread gets it.
__device__ __forceinline__ void block_best(float& bs, int& bt, float* red_f, int* red_i) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  warp_best(bs, bt);
  __syncthreads();
  if (lane == 0) {
    red_f[warp] = bs;
    red_i[warp] = bt;
  }
  __syncthreads();
  bs = red_f[lane];
  bt = red_i[lane];
  warp_best(bs, bt);
}

template <int NV4>
__global__ void __launch_bounds__(kTopkThreads) topk_kernel(const float* __restrict__ logits,
                                                            long long ldl, BeamDev b) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x;
  if (r >= *b.n_rows) return;
  __shared__ float red_f[32];
  __shared__ int red_i[32];
  __shared__ float list_s[kListCap];
  __shared__ int list_t[kListCap];
  __shared__ int list_n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int V = b.V;
  const float* x = logits + r * ldl;
  if (tid == 0) list_n = 0;

  float v[NV4 * 4];
#pragma unroll
  for (int i = 0; i < NV4; ++i) {
    const float4 f = *reinterpret_cast<const float4*>(x + 4 * (tid + kTopkThreads * i));
    v[4 * i] = f.x;
    v[4 * i + 1] = f.y;
    v[4 * i + 2] = f.z;
    v[4 * i + 3] = f.w;
  }
  float tmax = kNegInf;
#pragma unroll
  for (int i = 0; i < NV4 * 4; ++i) tmax = fmaxf(tmax, v[i]);
  const float wmax = warp_allmax(tmax);
  if (lane == 0) red_f[warp] = wmax;
  __syncthreads();
  const float wm = red_f[lane];  // lane l holds warp l's max
  const float mx = warp_allmax(wm);
  const int kB = min(b.B, V);
  // tau = kB-th largest warp max: kB warps each hold an element >= tau, so
  // tau <= the kB-th largest logit. Every warp computes it (shuffles only).
  float tau = kNegInf;
  {
    float c = wm;
    int ct = wm == kNegInf ? INT_MAX : lane;
    for (int k = 0; k < kB; ++k) {
      float bs = c;
      int bt = ct;
      warp_best(bs, bt);
      if (bt == INT_MAX) {
        tau = kNegInf;
        break;
      }
      tau = bs;
      if (bt == lane) {
        c = kNegInf;
        ct = INT_MAX;
      }
    }
  }
  __syncthreads();

  float part = 0.0f;
#pragma unroll
  for (int i = 0; i < NV4 * 4; ++i) part = __fadd_rn(part, det_expf_nonpos(__fsub_rn(v[i], mx)));
  part = warp_allsum(part);
  if (lane == 0) red_f[warp] = part;
  __syncthreads();
  const float total = warp_allsum(red_f[lane]);
  const float lse = __fadd_rn(det_logf(total), mx);
  const float plp = b.row_lp[r];

  // Candidates: score >= score(tau). Branch-free mask first; the few threads
  // holding candidates append them (one shared atomic per thread).
  const float s_lb = tau == kNegInf ? kNegInf : __fadd_rn(plp, __fsub_rn(tau, lse));
  unsigned mask = 0u;
#pragma unroll
  for (int i = 0; i < NV4 * 4; ++i) {
    const float sc = __fadd_rn(plp, __fsub_rn(v[i], lse));
    mask |= (sc >= s_lb && v[i] != kNegInf) ? (1u << i) : 0u;  // -inf: pad column
  }
  if (mask) {
    int slot = atomicAdd(&list_n, __popc(mask));
#pragma unroll
    for (int i = 0; i < NV4 * 4; ++i)
      if ((mask >> i) & 1u) {
        if (slot < kListCap) {
          list_s[slot] = __fadd_rn(plp, __fsub_rn(v[i], lse));
          list_t[slot] = 4 * (tid + kTopkThreads * (i >> 2)) + (i & 3);
        }
        ++slot;
      }
  }
  __syncthreads();
  const int n_list = list_n;

  if (n_list <= 64) {  // common case: warp 0 alone, shuffles only
    if (warp != 0) return;
    unsigned taken = 0u;
    for (int k = 0; k < kB; ++k) {
      float bs = kNegInf;
      int bt = INT_MAX, be = -1;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int idx = lane + 32 * e;
        if (idx < n_list && !((taken >> e) & 1u) &&
            (bt == INT_MAX || better2(list_s[idx], list_t[idx], bs, bt))) {
          bs = list_s[idx];
          bt = list_t[idx];
          be = e;
        }
      }
      float ws = bs;
      int wt = bt;
      warp_best(ws, wt);
      if (lane == 0) {
        b.cand_score[static_cast<long long>(r) * b.B + k] = ws;
        b.cand_tok[static_cast<long long>(r) * b.B + k] = wt;
      }
      if (bt == wt && be >= 0) taken |= 1u << be;
    }
    return;
  }

  if (n_list <= kListCap) {  // block-wide rounds over the list
    unsigned taken = 0u;
    for (int k = 0; k < kB; ++k) {
      float bs = kNegInf;
      int bt = INT_MAX;
#pragma unroll
      for (int e = 0; e < kListCap / kTopkThreads; ++e) {
        const int idx = tid + kTopkThreads * e;
        if (idx < n_list && !((taken >> e) & 1u) &&
            (bt == INT_MAX || better2(list_s[idx], list_t[idx], bs, bt))) {
          bs = list_s[idx];
          bt = list_t[idx];
        }
      }
      block_best(bs, bt, red_f, red_i);
      if (tid == 0) {
        b.cand_score[static_cast<long long>(r) * b.B + k] = bs;
        b.cand_tok[static_cast<long long>(r) * b.B + k] = bt;
      }
#pragma unroll
      for (int e = 0; e < kListCap / kTopkThreads; ++e) {
        const int idx = tid + kTopkThreads * e;
        if (idx < n_list && list_t[idx] == bt) taken |= 1u << e;
      }
    }
    return;
  }

  // Slow exact path: kB block rounds over every element with a taken mask.
  unsigned long long taken = 0ull;
  for (int k = 0; k < kB; ++k) {
    float bs = kNegInf;
    int bt = INT_MAX;
#pragma unroll
    for (int i = 0; i < NV4 * 4; ++i) {
      const int j = 4 * (tid + kTopkThreads * (i >> 2)) + (i & 3);
      if (j < V && !((taken >> i) & 1ull)) {
        const float sc = __fadd_rn(plp, __fsub_rn(v[i], lse));
        if (bt == INT_MAX || better2(sc, j, bs, bt)) {
          bs = sc;
          bt = j;
        }
      }
    }
    block_best(bs, bt, red_f, red_i);
    if (tid == 0) {
      b.cand_score[static_cast<long long>(r) * b.B + k] = bs;
      b.cand_tok[static_cast<long long>(r) * b.B + k] = bt;
    }
    if (((bt >> 2) % kTopkThreads) == tid)
      taken |= 1ull << (4 * ((bt >> 2) / kTopkThreads) + (bt & 3));
  }
}

}  // namespace

long long topk_pitch(int V) {
  const long long per = 4LL * kTopkThreads;
  return (static_cast<long long>(V) + per - 1) / per * per;
}

void launch_topk(const float* logits, long long ldl, const BeamDev& b, cudaStream_t st) {
  const int nv4 = static_cast<int>(topk_pitch(b.V) / (4 * kTopkThreads));
  if (ldl < topk_pitch(b.V)) fail(kStateError, "topk: logits pitch must be topk_pitch(V)");
  if (b.B > kMaxBeam) fail(kUsageError, "beam size above 16 is not supported");
  const dim3 grid(b.R_max), block(kTopkThreads);
  if (nv4 <= 1)
    launch_k(topk_kernel<1>, grid, block, 0, st, logits, ldl, b);
  else if (nv4 <= 2)
    launch_k(topk_kernel<2>, grid, block, 0, st, logits, ldl, b);
  else if (nv4 <= 4)
    launch_k(topk_kernel<4>, grid, block, 0, st, logits, ldl, b);
  else if (nv4 <= 8)
    launch_k(topk_kernel<8>, grid, block, 0, st, logits, ldl, b);
  else
    fail(kUsageError, "target vocabularies above 32768 are not supported by top-k yet");
  MTG_CUDA(cudaGetLastError());
}

}  // namespace mtg
