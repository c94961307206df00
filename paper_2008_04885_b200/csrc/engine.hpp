// The device engine: weights laid out K-major for the tcgen05 GEMM, a
// workspace sized per batch, the batched encoder, and the device-resident
// beam-search step loop. One engine = one model on one device + one stream.
#pragma once

#include <cstdint>
#include <memory>
#include <mutex>
#include <map>
#include <set>
#include <tuple>
#include <string>
#include <vector>

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "device_buffer.hpp"
#include "gemm.hpp"
#include "gemv.cuh"
#include "kernels.cuh"
#include "model_host.hpp"

namespace mtg {

enum Precision : int { kF32 = 0, kBF16 = 1, kINT8 = 2 };  // == MTG_PREC_*

// One GEMM weight [N x K] (K-major), possibly the concatenation of several
// reference tensors along N (q|k|v, k|v).
struct DevLinear {
  int n = 0, k = 0, k_pad = 0, prec = 0;
  DeviceBuffer<int8_t> q;
  DeviceBuffer<__nv_bfloat16> h;
  DeviceBuffer<float> hi, lo;
  DeviceBuffer<uint8_t> frag;     // small-batch GEMV copy in mma fragment order (gemv.cuh)
  DeviceBuffer<float> seg_scale;  // int8: weight scale per fused segment
  int seg_width = 0;              // columns per segment (0: one segment)
  Operand op() const;
};

// GEMM activation operand buffer for a given K.
struct ActOperand {
  int rows = 0, k = 0, k_pad = 0, prec = 0;
  DeviceBuffer<int8_t> q;
  DeviceBuffer<__nv_bfloat16> h;
  DeviceBuffer<float> hi, lo;
  DeviceBuffer<float> row_scale;
  Operand op() const;
  void allocate(int rows, int k, int prec);
};

struct BeamConfigC {
  int beam_size = 4;
  int max_len = 0;  // <= 0: derive per sentence
  float alpha = 1.0f;
};

struct SentenceResult {
  std::vector<int> tokens;
  float logprob = 0.0f;
  float norm = 0.0f;
  unsigned flags = 0;
  int status = 0;
};

class Engine {
 public:
  Engine(HostModel model, int precision, int device);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  const ModelConfig& config() const { return host_.config; }
  int precision() const { return prec_; }
  const HostModel& host_model() const { return host_; }
  std::mutex& mutex() { return mu_; }

  // Per sentence: the model's source-factor streams, each aligned with the
  // source ids (model.cpp:539-546).
  using FactorStreams = std::vector<std::vector<std::vector<int>>>;

  // Batched beam search over one device batch (sources carry their EOS).
  // shortlists: per sentence a strictly increasing target-id list (all
  // sentences of the batch, or null for full-vocabulary decoding).
  std::vector<SentenceResult> translate_batch(
      const std::vector<std::vector<int>>& srcs, const BeamConfigC& cfg,
      const FactorStreams* factors = nullptr,
      const std::vector<std::vector<int>>* shortlists = nullptr);
  // decode_step logits along forced prefixes; out[(i*nf + t)*V + v].
  void forced_logits(const std::vector<std::vector<int>>& srcs, const int* forced, int nf,
                     float* out, const FactorStreams* factors = nullptr);
  // encode_infer(embed_source_infer(.)) rows.
  void encode(const std::vector<std::vector<int>>& srcs, float* out,
              const FactorStreams* factors = nullptr);

  // Benchmark support: keep a staged batch resident and re-run it.
  void stage(const std::vector<std::vector<int>>& srcs, const FactorStreams* factors = nullptr,
             const std::vector<std::vector<int>>* shortlists = nullptr);
  void run_staged(const BeamConfigC& cfg);
  int64_t last_launches() const { return last_launches_; }
  std::string diag_report();  // per-kernel step times (MTG_DIAG_EVENTS=1)
  cudaStream_t stream() const { return stream_; }
  // Times one hot kernel in isolation on the staged batch (see minimt_gpu.h).
  void time_kernel(int kernel, int iters, float* ms, double* bytes, double* flops);

 private:
  struct Layer;  // device weights of one layer
  void upload_weights();
  void ensure_workspace(int n_sent, int m_enc, int beam);
  void prep(const float* x, long long ldx, int k, int max_rows, const int* d_rows,
            const int* seg_off, int n_seg, ActOperand& out);
  OperandOut opout(ActOperand& a);
  void prep_enc(const float* x, long long ldx, int k, int m, ActOperand& out, bool have_rowmax);
  struct LN;
  void ln_enc(const float* x, int m, const LN& ln, float* y, ActOperand& out);
  void gemm(const ActOperand& a, const DevLinear& w, int m, const int* d_m, float* c,
            long long ldc, const float* bias, const float* residual, int relu,
            long long c_step_stride = 0, const int* d_step = nullptr,
            unsigned* seg_absmax = nullptr, float* c_lo = nullptr, bool bf16_out = false);
  // Output projection into logits_ plus the per-slice softmax partials.
  void gemm_logits(int m, const int* d_m);
  int stage_sources(const std::vector<std::vector<int>>& srcs, std::vector<int>& status);
  void run_encoder(int n_sent, int m_enc, int max_src);
  void run_encoder_body(int n_sent, int m_enc, int max_src);
  // reorder: beam search (copy histories from row_parent at step >= 1).
  void decoder_body(bool reorder);  // decoder layers + dec_final + logits for the live rows
  // Small batches (<= kGemvRows live rows): the step as GEMV kernels with the
  // LayerNorms / quantization folded into the consumers (gemv.cuh).
  bool small_path() const;
  void decoder_body_small(bool reorder);
  GemvArgs gemv_args(const DevLinear& w) const;
  DeviceBuffer<float> gemv_ws_;       // split-K partials
  DeviceBuffer<int> gemv_sem_;        // split-K tickets (zero between launches)
  // MTG_TRACE=1: in-graph timeline of the small-batch step kernels.
  bool trace_ = false;
  static constexpr int kTraceSlots = 48;  // timeline slots per decode step
  DeviceBuffer<unsigned long long> trace_buf_;
  DeviceBuffer<unsigned long long> phase_buf_;  // MTG_TRACE=2
  // Encoder GEMM timeline (MTG_TRACE): slot k of layer l, layer = "step"
  static constexpr int kEncTraceSlots = 8;
  DeviceBuffer<unsigned long long> enc_trace_buf_;
  DeviceBuffer<unsigned long long> enc_phase_buf_;
  DeviceBuffer<int> enc_layer_ids_;
  std::vector<std::string> enc_trace_names_;
  int enc_trace_layers_ = 0;
  KTrace enc_trace(int layer, int slot, const char* name);
  KTrace enc_ln_tr_;  // timeline slot of the next encoder LayerNorm (int8 fused)
  bool trace_phases_ = false;
  int trace_slot_ = 0, trace_per_step_ = 0;
  std::vector<std::string> trace_names_;
  KTrace next_trace(const char* name);
  KTrace cur_tr_;  // consumed by the next gemm() / gemm_logits() launch
  void trace_reset();
  std::string trace_report();
  void decode_loop(int t_run);
  // Launch accounting; with MTG_DIAG_EVENTS=1 the step graph also records an
  // event after every kernel (breaks PDL overlap -- diagnostics only) and
  // decode_loop accumulates per-kernel times for diag_report().
  void count(const char* tag = "kernel");

  struct PlanKey {
    const void* a;
    const void* b;
    int m;
    bool operator<(const PlanKey& o) const { return std::tie(a, b, m) < std::tie(o.a, o.b, o.m); }
  };
  std::map<PlanKey, GemmPlan> plans_;
  std::map<PlanKey, GemmPlan>& plan_cache();

  HostModel host_;
  int prec_;
  int device_;
  cudaStream_t stream_ = nullptr;
  std::mutex mu_;
  int64_t launches_ = 0, last_launches_ = 0;
  bool diag_ = false, capturing_ = false;
  struct DiagMark {
    std::string name;
    cudaEvent_t ev;
  };
  std::vector<DiagMark> diag_marks_;
  std::vector<double> diag_ms_;
  int diag_steps_ = 0;
  bool enc_diag_active_ = false;          // encoder kernels are recorded eagerly
  std::vector<DiagMark> enc_marks_;
  std::map<std::string, std::pair<double, int>> enc_agg_;  // tag -> (ms, launches)
  double enc_total_ms_ = 0.0;
  int enc_runs_ = 0;
  void diag_clear();

  // ---- weights ----
  DeviceBuffer<float> src_embed_, tgt_embed_f32_, pe_;
  DeviceBuffer<int8_t> tgt_embed_q_;
  float tgt_scale_ = 1.0f;
  DevLinear logits_w_;
  struct LN {
    DeviceBuffer<float> g, b;
  };
  struct EncLayer {
    LN n1, n2;
    DevLinear qkv, wo, w1, w2;
    DeviceBuffer<float> b1, b2;
  };
  struct DecLayer {
    LN n1, n2, n3;
    DevLinear self_qkv, self_wo, cross_q, cross_kv, cross_wo, w1, w2;
    DeviceBuffer<float> b1, b2;
  };
  std::vector<EncLayer> enc_;
  std::vector<DecLayer> dec_;
  LN enc_final_, dec_final_;

  // ---- workspace ----
  int cap_sent_ = 0, cap_enc_ = 0, cap_beam_ = 0, r_max_ = 0, act_rows_ = 0;
  int d_ = 0, dff_ = 0, V_ = 0, Vp_ = 0, T_ = 0, heads_ = 0;
  ActOperand act_d_, act_ff_;
  ActOperand act_logits_;  // fp32: hi + lo operand of the output projection
  ActOperand& logits_act() { return prec_ == kF32 ? act_logits_ : act_d_; }
  DeviceBuffer<float> enc_x_, enc_a_, enc_qkv_, enc_ctx_, ffh_;
  std::vector<DeviceBuffer<float>> ckv_;
  DeviceBuffer<float> dec_y_, dec_a_, dec_ctx_, dec_cq_, logits_;
  DeviceBuffer<float> part_m_, part_s_;  // [r_max x part_ld_] softmax partials
  DeviceBuffer<int> part_arg_;
  DeviceBuffer<unsigned> sent_absmax_;
  std::vector<DeviceBuffer<float>> factor_embed_;  // non-shared factor tables
  DeviceBuffer<int> src_fids_;                     // [F][M] staged factor ids
  FactorStreams staged_factors_;
  DeviceBuffer<int> sl_ids_, sl_off_;  // shortlist CSR of the staged batch
  bool use_shortlist_ = false;
  std::vector<int> sl_status_;  // per staged sentence: shortlist validation status
  ShortlistArgs shortlist_args() const;  // per-sentence max |x| (float bits), encoder int8
  int enc_n_sent_ = 0;
  int enc_max_src_ = 0;  // longest source of the running encoder batch
  bool enc_fused_ = false;
  bool split_k_ = true;
  long long part_ld_ = 0;
  std::vector<DeviceBuffer<float>> qkv_cache_;
  DeviceBuffer<int> src_ids_, src_pos_, src_off_, enc_off_, enc_len_, src_rowseg_;
  DeviceBuffer<float> rowmax_;  // per-row max |x| for int8 segment scales
  DeviceBuffer<int> nonfinite_;
  // beam state
  DeviceBuffer<int> step_, n_rows_, row_sent_, row_prev_, row_parent_, anc0_, anc1_, tok0_, tok1_,
      cand_tok_, sent_row0_, sent_live_, sent_maxlen_, sent_done_, best_has_, best_len_, best_tok_,
      res_len_, res_status_, res_tok_, sel_parent_, sel_tok_, sel_count_;
  DeviceBuffer<float> row_lp_, cand_score_, best_norm_, best_lp_, res_lp_, res_norm_, sel_lp_;
  DeviceBuffer<unsigned> res_flags_;
  BeamDev beam_{};
  int* h_pinned_ = nullptr;  // pinned host mailbox (n_rows polling)
  int* res_host_ = nullptr;  // pinned staging of a batch's results
  size_t res_host_words_ = 0;

  // staged batch (benchmark)
  std::vector<std::vector<int>> staged_;
  int staged_m_ = 0, staged_max_src_ = 0, staged_n_ = 0;
  std::vector<int> staged_status_;
  int last_beam_ = 0, last_t_run_ = 0;
  DeviceBuffer<int> scratch_rows_;  // fixed row count for kernel timing

  // One decode step (decoder layers, logits, top-k, beam bookkeeping) as a
  // CUDA graph, re-captured when the batch shape / beam / alpha changes.
  void ensure_step_graph();
  struct EncKey {
    int gen, n, m, max_src;
    const void* fids;
    bool operator<(const EncKey& o) const {
      return std::tie(gen, n, m, max_src, fids) < std::tie(o.gen, o.n, o.m, o.max_src, o.fids);
    }
  };
  std::map<EncKey, std::pair<cudaGraphExec_t, int64_t>> enc_graphs_;
  std::set<EncKey> enc_seen_;
  void clear_enc_graphs();
  cudaGraph_t step_graph_ = nullptr;
  cudaGraphExec_t step_exec_ = nullptr;
  cudaGraphExec_t multi_exec_ = nullptr;  // steps_per_graph() steps per launch
  cudaGraphExec_t loop_exec_ = nullptr;   // while node over multi-step bodies
  DeviceBuffer<int> loop_end_;
  void capture_device_loop(int k);
  int steps_per_graph() const;
  int64_t capture_steps(int k, cudaGraphExec_t* exec, cudaGraph_t* graph);
  void capture_one_step();
  int64_t step_kernels_ = 0;
  int ws_gen_ = 0;
  struct StepKey {
    int n = -1, b = -1, r_max = -1, gen = -1, max_src = -1;
    float alpha = 0.0f;
    bool shortlist = false;
    const void* sl_ids = nullptr;  // graph kernels capture these pointers
    const void* sl_off = nullptr;
    bool operator==(const StepKey& o) const {
      return n == o.n && b == o.b && r_max == o.r_max && gen == o.gen && max_src == o.max_src &&
             alpha == o.alpha &&
             shortlist == o.shortlist && sl_ids == o.sl_ids && sl_off == o.sl_off;
    }
  } step_key_;
};

}  // namespace mtg
