// Beam bookkeeping kernels (decode.cpp:34-109): root rows, per-sentence
// selection / finished list / termination, and history gathers.
#include <climits>

#include "detmath.cuh"
#include "errors.hpp"
#include "launch.cuh"
#include "beam_dev.cuh"
#include "kernels.cuh"

namespace mtg {

namespace {

#define kNegInf (-__int_as_float(0x7f800000))
constexpr int kBosIdDev = 2;  // model.hpp:18

// ---- beam search ------------------------------------------------------------------------

__global__ void beam_init_kernel(BeamDev b) {
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x != 0) return;
  *b.sel_count = 0;
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


constexpr int kSelWarps = 4;

// Warp per sentence across the grid; the last CTA to finish (atomic ticket)
// computes the row offsets and writes the compacted rows.
__global__ void __launch_bounds__(kSelWarps * 32) beam_select_kernel(BeamDev b) {
  extern __shared__ int sel_smem[];  // [N] live counts, [N + N/32 + 1] first rows, [warps][96] scratch
  int* live_s = sel_smem;
  int* row0_s = sel_smem + b.N;
  __shared__ int is_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  // The first sentence's beam state (the previous step tail's) is loaded
  // before the dependency wait.
  const int s0 = blockIdx.x * nwarps + warp;
  SentState st0{};
  if (s0 < b.N) st0 = load_sent_state(b, s0);
  pdl_wait();
  pdl_trigger();
  const int t = *b.step;
  trace_begin_at(b.tr_b, t);
  for (int s = s0; s < b.N; s += gridDim.x * nwarps)
    select_sentence(b, s, t, lane, s == s0 ? st0 : load_sent_state(b, s),
                    reinterpret_cast<float*>(row0_s + b.N + b.N / 32 + 1) + warp * 96);
  finish_select(b, t, live_s, row0_s, &is_last);
  trace_end_at(b.tr_b, t);
}

__global__ void beam_reorder_kernel(BeamDev b) {
  pdl_wait();
  pdl_trigger();
  trace_begin(b.tr_b);  // (the fused step tail leaves tr_b to the reorder)
  const int r = blockIdx.x;
  if (r >= *b.n_rows) return;
  const int tn = *b.step;
  if (tn < 1) return;
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
  trace_end(b.tr_b);
}

}  // namespace

// While-node condition of the device-side decode loop: another chunk of k
// steps while hypotheses are alive and the chunk fits below loop_end.
__global__ void decode_loop_cond_kernel(cudaGraphConditionalHandle h, const int* n_rows,
                                        const int* step, const int* loop_end, int k) {
  cudaGraphSetConditional(h, (*n_rows > 0 && *step + k <= *loop_end) ? 1u : 0u);
}

void launch_decode_loop_cond(cudaGraphConditionalHandle h, const int* n_rows, const int* step,
                             const int* loop_end, int k, cudaStream_t st) {
  decode_loop_cond_kernel<<<1, 1, 0, st>>>(h, n_rows, step, loop_end, k);
  MTG_CUDA(cudaGetLastError());
}

void launch_beam_init(const BeamDev& b, cudaStream_t st) {
  launch_k(beam_init_kernel, 1, 32, 0, st, b);
  MTG_CUDA(cudaGetLastError());
}

void launch_beam_select(const BeamDev& b, cudaStream_t st) {
  const size_t smem = sizeof(int) * (2 * static_cast<size_t>(b.N) + b.N / 32 + 1) +
                      sizeof(float) * 96 * kSelWarps;
  if (smem > 227 * 1024) fail(kUsageError, "beam search: too many sentences in one batch");
  ensure_smem_attr(beam_select_kernel, smem);
  launch_k(beam_select_kernel, (b.N + kSelWarps - 1) / kSelWarps, kSelWarps * 32, smem, st, b);
  MTG_CUDA(cudaGetLastError());
}

void launch_beam_reorder(const BeamDev& b, cudaStream_t st) {
  launch_k(beam_reorder_kernel, b.R_max, 128, 0, st, b);
  MTG_CUDA(cudaGetLastError());
}

}  // namespace mtg
