// Small-batch decode linears (at most kGemvRows live hypothesis rows, i.e.
// batch-1 serving at beam <= 8). With m <= 8 the decoder's linear layers are
// GEMVs: every weight byte is used m times, so the roofline is the weight
// stream from L2/HBM plus the dependent-latency chain between layers, not the
// tensor pipe. These kernels therefore
//   * prefetch the CTA's weight slice into shared memory with 1-D bulk copies
//     BEFORE the programmatic-dependency wait (the weights do not depend on
//     the previous kernel), so the stream overlaps the predecessor;
//   * build the activation operand of all live rows inside every CTA after
//     the wait -- including the LayerNorm that precedes the layer and the
//     per-row int8 quantization (quant.cpp:108-122) -- so no separate
//     LayerNorm / quantize kernels run between layers;
//   * run warp-per-output dot products (int8 dp4a with exact int32
//     accumulation, bf16 / fp32 FMA) and the reference linear epilogue.
// The output-projection variant also emits the per-32-column log-softmax
// partials of the tcgen05 projection epilogue (gemm_tc.cuh kEpiSoftmaxParts,
// DESIGN.md §3 P6), so the same top-k tail follows. int8 results are bit-
// identical to the tcgen05 path (integer accumulation, same epilogue).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "launch.cuh"

namespace mtg {

constexpr int kGemvRows = 8;

struct GemvArgs {
  // ---- activation rows (fp32 source, converted in the CTA) ----
  int a_mode = 0;  // 0: rows of x; 1: LayerNorm(x); 2: LayerNorm(target embedding)
  const float* x = nullptr;
  long long ldx = 0;
  const float* ln_g = nullptr;
  const float* ln_b = nullptr;
  const int* d_rows = nullptr;  // live rows (<= kGemvRows)
  int rows_alloc = 0;           // allocated rows of x / residual / C (operand rows built)
  int K = 0;
  // a_mode 2 (decode-step start, model.cpp:624-626): x = table[prev] * sqrt_d
  // + pe[step]; block 0 stores it to x_out (the residual stream).
  const int* prev = nullptr;
  const float* table = nullptr;
  int table_rows = 0;
  const float* pe = nullptr;
  float sqrt_d = 1.0f;
  const int* d_step = nullptr;
  float* x_out = nullptr;
  long long ldx_out = 0;
  // a_mode 2, optional: beam history reorder (beam_reorder_kernel) by the
  // last block.
  int reorder = 0;
  const int* row_parent = nullptr;
  int* anc[2] = {nullptr, nullptr};
  int* tok[2] = {nullptr, nullptr};
  int T = 0;
  // ---- weights: [N x k_pad] K-major in the path's precision ----
  const void* w = nullptr;
  int k_pad = 0;
  int N = 0;
  const float* w_seg_scale = nullptr;  // int8: scale per fused segment
  int seg_width = 0;
  // ---- epilogue ----
  float* C = nullptr;
  long long ldc = 0;
  long long c_step_stride = 0;  // C += (*d_step) * c_step_stride (KV-cache slab)
  const float* bias = nullptr;
  const float* residual = nullptr;
  long long ldr = 0;
  int relu = 0;
  // output projection: softmax partials per 32-column slice
  float* part_m = nullptr;
  float* part_s = nullptr;
  int* part_arg = nullptr;
  long long part_ld = 0;
  int* nonfinite = nullptr;
  // ---- split-K across CTAs (fp32 / bf16 plain operand rows): partials in
  // ws, the last CTA of a chunk (ticket in sem, one int per chunk,
  // zero-initialised) adds them in split order ----
  int ksplit = 1;
  float* ws = nullptr;
  int* sem = nullptr;
  KTrace trace;
};

// prec: 0 int8, 1 bf16, 2 fp32. logits: output-projection epilogue.
// a.w is the fragment-order copy made by launch_gemv_pack.
void launch_gemv(int prec, bool logits, const GemvArgs& a, cudaStream_t st);

// Bytes of the fragment-order copy of an [n x k_pad] weight (elem bytes per
// value): rows padded to a multiple of 16.
inline long long gemv_pack_bytes(int n, int k_pad, int elem) {
  return static_cast<long long>((n + 15) / 16) * 16 * k_pad * elem;
}
// Repacks a K-major [n x k_pad] weight into mma.sync A-fragment order: for
// each 16-row group and each 32-byte K step, 32 lanes x 16 bytes holding the
// lane's {a0, a1, a2, a3} registers, so a warp loads a whole fragment with
// one conflict-free 16-byte shared load per lane (pure byte permutation).
void launch_gemv_pack(const void* w, int n, int k_pad, int elem, void* out, cudaStream_t st);

// Small-batch decoder attention (attn_small.cu): CTA per (row, head), head
// dim 64, keys / values prefetched before the programmatic-dependency wait;
// fp32 contexts only (the consuming GEMV builds the operand).
bool attn_small_supported(int d, int heads, int T, int max_src);
// Batched cross-attention (fp32 / bf16 operands), CTA per (sentence, head),
// warp per live beam row; the sentence's keys / values staged once, before
// the programmatic-dependency wait (attn_small.cu).
bool attn_cross_sent_supported(int d, int heads, int max_src, int beam);
void launch_attn_cross_sent(const float* cq, long long ldq, const float* ckv, const int* enc_off,
                            const int* enc_len, const int* sent_row0, const int* sent_live,
                            const int* sent_done, int n_sent, int beam, int max_src, int d,
                            int heads, float scale, float* ctx, long long ldc,
                            const OperandOut& op, cudaStream_t st);
// hist != 0 (layer 0 of a beam step): also writes the step's ancestry /
// token-history rows (the beam reorder), off the step's critical path.
void launch_attn_small_self(const float* cache, int r_max, int T, int* anc0, int* anc1,
                            const int* row_parent, int reorder, int* tok0, int* tok1,
                            const int* row_prev, int hist, const int* d_rows, const int* d_step,
                            int rows_alloc, int d, int heads, float scale, float* ctx,
                            long long ldc, cudaStream_t st, const KTrace& tr = {});
void launch_attn_small_cross(const float* cq, long long ldq, const float* ckv,
                             const int* row_sent, const int* enc_off, const int* enc_len,
                             const int* d_rows, int rows_alloc, int max_src, int d, int heads,
                             float scale, float* ctx, long long ldc, cudaStream_t st,
                             const KTrace& tr = {});

}  // namespace mtg
