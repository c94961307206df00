// Non-GEMM kernels of the translation hot path. Float reduction orders are
// pinned so the CPU oracle reproduces them bit for bit.
#pragma once

#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "launch.cuh"

namespace mtg {

constexpr int kMaxBeam = 16;
constexpr int kTopkThreads = 1024;

// Destination of a row's GEMM operand (the next linear layer's A matrix):
// int8 + per-row scale (quant.cpp:108-122), bf16, or fp32 hi/lo (3xTF32).
// prec uses the GemmPrec numbering (0 = int8, 1 = bf16, 2 = tf32x3).
struct OperandOut {
  int prec = 0;
  int k_pad = 0;
  int8_t* q = nullptr;
  float* row_scale = nullptr;
  __nv_bfloat16* h = nullptr;
  float* hi = nullptr;
  float* lo = nullptr;
  int* nonfinite = nullptr;
  KTrace tr;  // MTG_TRACE timeline slot of the kernel writing this operand
};

// Beam history reorder folded into the layer-0 decoder self-attention
// (beam.cu beam_reorder_kernel): row r's ancestry / token tables of step t
// from its parent's, written by the attention before its dependency wait.
struct HistReorder {
  int on = 0;
  int* anc[2] = {nullptr, nullptr};
  int* tok[2] = {nullptr, nullptr};
  const int* row_parent = nullptr;
  const int* row_prev = nullptr;
};

// Empty dependent kernel (148 CTAs): the PDL launch floor, for timing.
void launch_noop(cudaStream_t st);

// ---- embeddings (model.cpp:539-581, 624-626) -----------------------------------

// out[r] = table[ids[r]] * sqrt_d + pe[pos[r]]
// Source embedding (model.cpp:539-581): word row (width wdim) combined with up
// to kMaxFactors factor rows -- concat (columns appended), sum, or average
// (sum x 1/(1+F)) -- then x sqrt(d) + PE[pos].
constexpr int kMaxFactors = 4;
struct SrcEmbed {
  const float* word = nullptr;
  int wdim = 0;
  int n_factors = 0;
  int mode = 0;  // 0 concat, 1 sum, 2 average
  const float* table[kMaxFactors] = {};
  int fdim[kMaxFactors] = {};
  const int* fids = nullptr;  // [n_factors][rows]
  long long fstride = 0;
  float avg_scale = 1.0f;
};
void launch_embed_src(const int* ids, const int* pos, int rows, const SrcEmbed& se, int d,
                      float sqrt_d, const float* pe, float* out, long long ldo, cudaStream_t st);

// Decoder input rows (d_rows on device), position = *d_step. table_q != null:
// int8 table dequantised as q / scale (model.cpp:485).
// Fused first kernel of a decode step (kernels.cu step_begin_kernel):
// history reorder + target embedding + the first decoder LayerNorm.
struct StepBegin {
  const int* d_rows;
  const int* d_step;
  const int* prev;        // [R] previous token per row
  const float* table;     // fp32 target embedding (or null with table_q)
  const int8_t* table_q;  // int8 target embedding
  float q_scale;
  float sqrt_d;
  const float* pe;
  int d;
  float* x;  // residual stream [R x ldx]
  long long ldx;
  int reorder;  // copy histories from row_parent (beam search) when step >= 1
  const int* row_parent;
  int* anc[2];
  int* tok[2];
  int T;
};
void launch_step_begin(const StepBegin& sb, int max_rows, const float* g, const float* b,
                       const OperandOut& op, cudaStream_t st);
void launch_embed_tgt(const int* prev, const int* d_rows, int max_rows, const int* d_step,
                      const float* table, const int8_t* table_q, float q_scale, int d,
                      float sqrt_d, const float* pe, float* out, long long ldo, cudaStream_t st);

// ---- layer norm (tensor.cpp:368-387) -------------------------------------------
// One warp per row. Optional outputs: y (fp32), rowmax (max |y| per row, for
// segment quantization), op (the row's GEMM operand; only valid when the
// quantization segment is the row itself or the precision is not int8).
void launch_layernorm(const float* x, long long ldx, int max_rows, const int* d_rows, int n,
                      const float* g, const float* b, float* y, long long ldy, float* rowmax,
                      const OperandOut* op, cudaStream_t st);

// ---- int8 segment quantization (quant.cpp:108-122) ----------------
void launch_rowmax(const float* x, long long ldx, int rows, int n, float* rowmax, int* nonfinite,
                   cudaStream_t st);
// Row r belongs to segment row_seg[r] = rows [seg_off[s], seg_off[s+1]); its
// scale is 127 / max(rowmax over the segment).
void launch_quantize_seg(const float* x, long long ldx, int rows, int n, const int* row_seg,
                         const int* seg_off, const float* rowmax, const OperandOut& op,
                         cudaStream_t st);

// ---- attention (model.cpp:509-528, 642-665) ------------------------------------

// Encoder self-attention over each sentence (rows off[s]..off[s+1]).
// qkv rows: [q | k | v] each d wide, pitch ldq. ctx pitch ldc.
// sent_absmax (optional): max |ctx| per sentence accumulated as float bits
// (atomicMax) for the per-sentence int8 scale; non-finite values set *nonfinite.
// ctx_lo (optional, fp32 path): write the rows as a TF32x3 operand (ctx =
// tf32 hi, ctx_lo = residual) for the next GEMM.
void launch_enc_attention(const float* qkv, long long ldq, const int* off, int n_sent,
                          int max_len, int d, int heads, float scale, float* ctx, long long ldc,
                          float* ctx_lo, unsigned* sent_absmax, int* nonfinite, cudaStream_t st,
                          const KTrace& tr = {},
                          bool out_bf16 = false);
// Encoder LayerNorm -> int8 operand with one scale per sentence (CTA per
// sentence); zeroes sent_absmax[s] for later accumulation.
void launch_ln_quant_sent(const float* x, long long ldx, const int* off, int n_sent, int n,
                          const float* g, const float* b, float* y, long long ldy,
                          const OperandOut& op, unsigned* sent_absmax, cudaStream_t st,
                          int max_rows = 0);
// int8 operand rows scaled by their sentence's accumulated max |x|.
void launch_quantize_sent(const float* x, long long ldx, int rows, int n, const int* row_seg,
                          const unsigned* sent_absmax, const OperandOut& op, cudaStream_t st);

// Decoder self-attention for live row r at step t over positions 0..t; the key
// of position j lives in row anc[r*T + j] of the step-j slab of qkv_cache
// ([T][R_max][3d]). anc0/anc1: the double-buffered ancestor tables (t & 1).
// The context row is written as fp32 (ctx) and as the next GEMM's operand.
void launch_dec_self_attention(const float* qkv_cache, int r_max, int T, const int* anc0,
                               const int* anc1, const int* d_rows, const int* d_step, int d,
                               int heads, float scale, float* ctx, long long ldc,
                               const OperandOut& op, cudaStream_t st,
                               int early = 1, const HistReorder& hist = {});

// Decoder cross-attention: row r attends to its sentence's encoder rows
// (enc_off[s]..+enc_len[s]) in ckv ([M_enc][2d] = [k | v]).
void launch_dec_cross_attention(const float* cq, long long ldq, const float* ckv,
                                const int* row_sent, const int* enc_off, const int* enc_len,
                                const int* d_rows, int max_rows, int max_src, int d, int heads,
                                float scale, float* ctx, long long ldc, const OperandOut& op,
                                cudaStream_t st);

// ---- beam search (decode.cpp:25-109) -------------------------------------------

struct BeamDev {
  int* step;        // [1]
  int* n_rows;      // [1]
  int* row_sent;    // [R_max]
  float* row_lp;    // [R_max]
  int* row_prev;    // [R_max]
  int* row_parent;  // [R_max]
  int* anc[2];      // [R_max * T]
  int* tok[2];      // [R_max * T]
  float* cand_score;  // [R_max * B]
  int* cand_tok;      // [R_max * B]
  int* sent_row0;     // [N]
  int* sent_live;     // [N]
  int* sent_maxlen;   // [N]
  int* sent_done;     // [N]
  int* best_has;      // [N]
  float* best_norm;
  float* best_lp;
  int* best_len;
  int* best_tok;      // [N * T]
  int* res_len;       // [N]
  float* res_lp;
  float* res_norm;
  unsigned* res_flags;
  int* res_status;
  int* res_tok;       // [N * T]
  int* sel_parent;    // [N * B]
  int* sel_tok;
  float* sel_lp;
  int* sel_count;     // [1] CTAs of beam_select done this step (last one compacts)
  int N, B, T, R_max, V;
  float alpha;
  int max_seq_len;
  KTrace tr_a, tr_b;  // MTG_TRACE: top-k (or fused tail) and beam select
};

// Step 0: one root row (BOS, logprob 0) per active sentence.
void launch_beam_init(const BeamDev& b, cudaStream_t st);
void launch_decode_loop_cond(cudaGraphConditionalHandle h, const int* n_rows, const int* step,
                             const int* loop_end, int k, cudaStream_t st);

// log_softmax_row + candidate scores + per-row top-min(B,V) by (score desc,
// token asc), one warp per live row, from the per-32-column softmax partials
// of the output-projection GEMM (gemm_tc.cuh kEpiSoftmaxParts) plus a
// rescan of the few slices that can hold the winners (topk.cu). V <= 32768.
constexpr int kMaxSoftmaxSlices = 1024;
long long topk_pitch(int V);          // logits row pitch (elements)
long long softmax_part_pitch(int V);  // partials row pitch (slices, multiple of 4)
// Vocabulary shortlist path (topk.cu shortlist_topk_kernel): per-sentence
// sorted id lists in CSR; operand row r of the final LayerNorm output and the
// tied output embedding in the path's precision (0 int8, 1 bf16, 2 fp32).
constexpr int kMaxShortlist = 4096;
struct ShortlistArgs {
  const int* sl_ids = nullptr;
  const int* sl_off = nullptr;  // [N + 1]
  int K = 0;
  long long lda = 0, ldw = 0;   // row pitches (elements)
  const int8_t* aq = nullptr;
  const float* a_scale = nullptr;
  const int8_t* wq = nullptr;
  float w_scale = 1.0f;
  const __nv_bfloat16* ah = nullptr;
  const __nv_bfloat16* wh = nullptr;
  const float* af = nullptr;
  const float* wf = nullptr;
};
void launch_shortlist_topk(int prec, const ShortlistArgs& a, const BeamDev& b, cudaStream_t st);
// Fused step tail (topk.cu): per-sentence CTA running the top-k of its rows
// (full vocabulary from the projection partials, or the shortlist when sa is
// set) and then the beam selection + compaction of launch_beam_select.
void launch_topk_select(const float* logits, long long ldl, const float* part_m,
                        const float* part_s, const int* part_arg, long long part_ld,
                        const ShortlistArgs* sa, int prec, const BeamDev& b, cudaStream_t st);
void launch_softmax_topk(const float* logits, long long ldl, const float* part_m,
                         const float* part_s, const int* part_arg, long long part_ld,
                         const BeamDev& b, cudaStream_t st);

// Per-sentence selection of beam_size candidates by (score desc, parent asc,
// token asc), EOS -> finished (running first-max of the GNMT score), live
// rows compacted in rank order, termination + result extraction; step += 1.
void launch_beam_select(const BeamDev& b, cudaStream_t st);

// Gathers ancestor-row and token histories of the new rows from their parents.
void launch_beam_reorder(const BeamDev& b, cudaStream_t st);

}  // namespace mtg
