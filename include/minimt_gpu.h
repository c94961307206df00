/*
 * minimt_gpu.h -- C ABI of the B200-native (sm_100a) translation hot path:
 * batched transformer encoder + incremental beam-search decoding.
 *
 * Each entry point replaces one interface of the CPU reference ("minimt",
 * /root/reference/proj); the reference location is cited beside it. Plain
 * pointers and sizes only; host buffers in and out. All functions return an
 * MTG_STATUS code; on failure mtg_last_error() (thread-local) holds the
 * message. Status codes map 1:1 onto the reference exception taxonomy
 * (proj/include/minimt/errors.hpp:8-34).
 *
 * Threading: a model handle owns one CUDA stream; calls on one handle are
 * serialised internally. Distinct handles may be used from distinct threads
 * (the reference's "Executor is immutable and shareable", model.hpp:113-129,
 * becomes "one stream per handle").
 */
#ifndef MINIMT_GPU_H_
#define MINIMT_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MTG_ABI_VERSION 1

/* ---- status codes (errors.hpp:8-34) ------------------------------------ */
#define MTG_OK 0
#define MTG_SHAPE_ERROR 1  /* minimt::ShapeError  */
#define MTG_VALUE_ERROR 2  /* minimt::ValueError  */
#define MTG_INDEX_ERROR 3  /* minimt::IndexError  */
#define MTG_STATE_ERROR 4  /* minimt::StateError  */
#define MTG_FORMAT_ERROR 5 /* minimt::FormatError */
#define MTG_USAGE_ERROR 6  /* minimt::UsageError  */
#define MTG_IO_ERROR 7     /* minimt::IoError     */
#define MTG_CUDA_ERROR 8   /* device failure (no reference counterpart) */

/* ---- precisions ----------------------------------------------------------
 * F32  : F32Executor (model.hpp:131-145); GEMMs on tcgen05 kind::tf32 as
 *        3xTF32 split products (fp32-class accuracy).
 * BF16 : bf16 operands, fp32 accumulate (extension; stated logit tolerance).
 * INT8 : Int8Executor (model.hpp:157-171); tcgen05 kind::i8, bit-exact
 *        int32 accumulation and the reference epilogue.                      */
#define MTG_PREC_F32 0
#define MTG_PREC_BF16 1
#define MTG_PREC_INT8 2

/* Hypothesis flags (decode.hpp:15-25). */
#define MTG_HYP_FINISHED 1u  /* ended with EOS                     */
#define MTG_HYP_TRUNCATED 2u /* no finished hypothesis within max_len */
#define MTG_HYP_FAILED 4u    /* the sentence raised; see status[i]   */

const char* mtg_last_error(void);
int mtg_abi_version(void);

/* ---- raw operators (quant.hpp:45-68; tensor.hpp:150-154) ----------------- */

/* quantize(): scale = 127/max|x| (1 if all zero), q = clamp(round(x*scale)).
 * quant.cpp:108-122. ValueError on non-finite input. */
int mtg_quantize(const float* x, int64_t n, int8_t* q_out, float* scale_out);

/* qmatmul(): C[m x n] = (int32 sum_k a*b) * (1/(sa*sb)); a [m x k], b [k x n]
 * row-major int8. quant.cpp:155-193. ValueError if k > 65536. */
int mtg_qmatmul(const int8_t* a, float a_scale, const int8_t* b, float b_scale,
                int m, int k, int n, float* c);

/* qmatmul_nt(): C = A . B^T over rows of b [b_rows x k]; row_subset (may be
 * NULL) selects/reorders output features. quant.cpp:195-239. IndexError on a
 * bad row. */
int mtg_qmatmul_nt(const int8_t* a, float a_scale, const int8_t* b, float b_scale,
                   int m, int k, int b_rows, const int32_t* row_subset,
                   int n_subset, float* c);

/* gemm_f32(): c[m x n] = a[m x k] . b[k x n] at precision F32 (3xTF32) or
 * BF16. tensor.cpp:156-161. */
int mtg_gemm(int precision, const float* a, const float* b, int m, int k, int n,
             float* c);

/* ---- model handle (model.hpp:33-207) -------------------------------------- */

typedef struct mtg_model mtg_model;

/* Loads an SQNT file (io.hpp:10-18). An f32 file loads as F32/BF16, or as
 * INT8 with on-load quantization (load_model_quantized_on_load,
 * model.cpp:805-807); an int8 file always decodes INT8 (load_quantized,
 * model.cpp:775-803; tools/minimt.cpp:311-329). */
int mtg_model_load(const char* path, int precision, int device, mtg_model** out);

/* Builds a model from a ModelConfig JSON (model.cpp:102-148) with
 * init_params(Rng(seed)) weights (model.cpp:229-238). */
int mtg_model_create(const char* config_json, uint64_t seed, int precision,
                     int device, mtg_model** out);

/* Writes the model's weights as an SQNT file (save_params /
 * save_quantized, model.cpp:699-773). */
int mtg_model_save(const mtg_model* m, const char* path);

void mtg_model_free(mtg_model* m);

/* ModelConfig::to_json() of the loaded model into buf (NUL-terminated). */
int mtg_model_config_json(const mtg_model* m, char* buf, size_t cap);
int mtg_model_precision(const mtg_model* m);

/* ---- beam search (decode.hpp:27-38; decode.cpp:34-109, 320-359) ---------- */

typedef struct mtg_beam_config {
  int beam_size;              /* BeamConfig::beam_size            */
  int max_len;                /* <= 0: min(max_seq_len, 2|src|+5)  */
  float length_penalty_alpha; /* GNMT alpha                        */
  int max_batch;              /* sentences per device batch; 0 = all */
} mtg_beam_config;

/* Batched beam_search over n sentences given as CSR source ids (each already
 * carrying its trailing EOS, as translate_one builds it). Outputs, per
 * sentence i: tokens (EOS excluded) at out_tokens[i*out_stride ...],
 * out_len[i], out_logprob[i], out_norm_score[i], out_flags[i] (MTG_HYP_*),
 * out_status[i] (MTG_* of that sentence). Any output pointer may be NULL.
 * Sentence-level errors (empty source, too long, bad ids) are reported per
 * sentence like translate_corpus (decode.cpp:403-410); a bad BeamConfig
 * fails the call (decode.cpp:38). */
int mtg_translate(mtg_model* m, const int32_t* src_ids, const int64_t* src_offsets,
                  int n_sentences, const mtg_beam_config* cfg, int32_t* out_tokens,
                  int out_stride, int32_t* out_len, float* out_logprob,
                  float* out_norm_score, uint32_t* out_flags, int32_t* out_status);

/* Parity entry for decode_step (model.cpp:614-672): for each sentence, feed
 * BOS + forced[0..n_forced-1) and return the logits of every step,
 * out_logits[(i*n_forced + t)*V + v]. All sentences share n_forced. */
/* Source factors (model.cpp:539-581, decode.cpp:334-342): factor_ids holds
 * n_factors streams, each aligned with src_ids (stream f at
 * factor_ids + f * src_offsets[n_sentences]; same CSR offsets, EOS position
 * included). n_factors must equal the model's factor count, otherwise the
 * sentence fails with MTG_SHAPE_ERROR, like embed_source_infer. */
int mtg_translate_factors(mtg_model* m, const int32_t* src_ids, const int64_t* src_offsets,
                          int n_sentences, const int32_t* factor_ids, int n_factors,
                          const mtg_beam_config* cfg, int32_t* out_tokens, int out_stride,
                          int32_t* out_len, float* out_logprob, float* out_norm_score,
                          uint32_t* out_flags, int32_t* out_status);
int mtg_encode_factors(mtg_model* m, const int32_t* src_ids, const int64_t* src_offsets,
                       int n_sentences, const int32_t* factor_ids, int n_factors, float* out);

/* Full form: optional source factors (as above, or NULL / 0) and optional
 * vocabulary shortlists (decode.cpp:113-165, 344-349; model.cpp:440-449):
 * sentence s uses target ids shortlist_ids[shortlist_offsets[s] ..
 * shortlist_offsets[s+1]) -- strictly increasing, < tgt_vocab_size, at most
 * 4096 -- or the full vocabulary when that range is empty (or the arrays are
 * NULL). Logits, log-softmax and candidates cover the shortlist only; the
 * candidate token is the full-vocabulary id. */
int mtg_translate_ex(mtg_model* m, const int32_t* src_ids, const int64_t* src_offsets,
                     int n_sentences, const int32_t* factor_ids, int n_factors,
                     const int32_t* shortlist_ids, const int64_t* shortlist_offsets,
                     const mtg_beam_config* cfg, int32_t* out_tokens, int out_stride,
                     int32_t* out_len, float* out_logprob, float* out_norm_score,
                     uint32_t* out_flags, int32_t* out_status);

int mtg_forced_logits(mtg_model* m, const int32_t* src_ids, const int64_t* src_offsets,
                      int n_sentences, const int32_t* forced, int n_forced,
                      float* out_logits);

/* Parity entry for encode_infer(embed_source_infer(...)) (model.cpp:539-596):
 * encoder output rows [sum |src_i| x d_model]. */
int mtg_encode(mtg_model* m, const int32_t* src_ids, const int64_t* src_offsets,
               int n_sentences, float* out);

/* Device-resident timing helpers for the benchmark: stage sources once,
 * then run the batched search with no host copies in the timed region. */
int mtg_stage_sources(mtg_model* m, const int32_t* src_ids, const int64_t* src_offsets,
                      int n_sentences);
int mtg_translate_staged(mtg_model* m, const mtg_beam_config* cfg);
/* Kernel launches issued by the last translate call (for gpu_launches). */
int64_t mtg_last_launch_count(const mtg_model* m);
/* The handle's CUDA stream (cudaStream_t as void*), for event timing. */
void* mtg_model_stream(const mtg_model* m);
/* Times `iters` back-to-back launches of one hot kernel on the staged batch
 * (kernel: 0 = decoder output-projection GEMM, 1 = log-softmax/top-k,
 * 2 = decoder self-attention, 3 = encoder FFN w1 GEMM) with CUDA events on
 * the handle's stream. Writes the mean milliseconds per launch and the
 * algorithmic bytes and FLOPs of one launch. Small-batch (<= 8 live rows)
 * step kernels, chained `iters` times in one CUDA graph with programmatic
 * dependent launch: 10 = empty kernel (launch floor), 11 = Wo GEMV + residual,
 * 12 = LayerNorm + W1 GEMV, 13 = LayerNorm + output projection + softmax
 * partials, 14 = batched self-attention, 15 = log-softmax/top-k merge,
 * 16 = small-batch self-attention, 17 = small-batch cross-attention. */
int mtg_time_kernel(mtg_model* m, int kernel, int iters, float* ms_per_launch,
                    double* bytes_per_launch, double* flops_per_launch);

/* Diagnostics: with MTG_DIAG_EVENTS=1 in the environment, the decode-step graph
 * records an event after every kernel (serialising them) and this returns the
 * per-kernel average step times of the last translate call as text. */
int mtg_diag_report(mtg_model* m, char* buf, size_t buf_size);

#ifdef __cplusplus
}
#endif

#endif /* MINIMT_GPU_H_ */
