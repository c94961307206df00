// Device engine: weight layout, workspace, batched encoder (model.cpp:539-612)
// and the device-resident beam-search loop (decode.cpp:34-109).
#include "engine.hpp"

#include <cstdio>
#include <cstdlib>

#include <algorithm>
#include <cmath>
#include <functional>
#include <map>
#include <tuple>

#include "errors.hpp"
#include "prep.cuh"

namespace mtg {

namespace {

int gemm_prec_of(int prec) {
  return prec == kINT8 ? kPrecI8 : prec == kBF16 ? kPrecBF16 : kPrecTF32x3;
}
// Activation operands: fp32 activations stay plain fp32 (the GEMM splits
// them into tf32 hi + lo in shared memory, gemm_tc.cuh kPrecTF32x3A).
// MTG_F32_SPLIT_A=1 selects that in-kernel split (A/B: measured slower with
// the two-stage fp32 pipelines); by default producers write hi + lo.
int act_prec_of(int prec) {
  static const bool split_a = [] {
    const char* e = std::getenv("MTG_F32_SPLIT_A");
    return e && e[0] == '1';
  }();
  return prec == kF32 && split_a ? kPrecTF32x3A : gemm_prec_of(prec);
}


// Converts fp32 K-major rows (host, [n x k]) into the operand format.
void upload_f32_operand(const std::vector<float>& kmaj, int n, int k, int prec, DevLinear& L,
                        cudaStream_t st) {
  DeviceBuffer<float> tmp(std::max<size_t>(1, size_t(n) * k));
  tmp.upload(kmaj.data(), kmaj.size());
  if (prec == kBF16) {
    L.h.resize(size_t(n) * L.k_pad);
    launch_cast_bf16(tmp.get(), k, k, n, nullptr, L.h.get(), L.k_pad, st);
  } else {
    L.hi.resize(size_t(n) * L.k_pad);
    L.lo.resize(size_t(n) * L.k_pad);
    launch_split_tf32(tmp.get(), k, k, n, nullptr, L.hi.get(), L.lo.get(), L.k_pad, st);
  }
  MTG_CUDA(cudaStreamSynchronize(st));
}

// Builds a [N x K] K-major weight from reference tensors. `nt`: tensors are
// already [rows = N x cols = K] (tgt_embed); otherwise [K x N] (y = x.W).
// Fragment-order copy of a weight for the small-batch GEMV path (gemv.cuh).
void build_gemv_copy(DevLinear& L, const void* src, int elem, cudaStream_t st) {
  L.frag.resize(static_cast<size_t>(gemv_pack_bytes(L.n, L.k_pad, elem)));
  launch_gemv_pack(src, L.n, L.k_pad, elem, L.frag.get(), st);
  MTG_CUDA(cudaStreamSynchronize(st));
}

void build_linear(DevLinear& L, const std::vector<const HostTensor*>& parts, bool nt, int prec,
                  cudaStream_t st, bool gemv_copy = false) {
  const int k = static_cast<int>(nt ? parts[0]->cols() : parts[0]->rows());
  int n = 0;
  for (auto* p : parts) n += static_cast<int>(nt ? p->rows() : p->cols());
  L.n = n;
  L.k = k;
  L.prec = gemm_prec_of(prec);
  L.k_pad = pad_k(k, L.prec);
  if (prec == kINT8) {
    std::vector<int8_t> buf(size_t(n) * L.k_pad, 0);
    // One max-abs scale per reference tensor; fused tensors are equal-width
    // column segments (q|k|v, k|v).
    std::vector<float> seg(kMaxSegments, 1.0f);
    if (parts.size() > static_cast<size_t>(kMaxSegments))
      fail(kStateError, "too many fused weight segments");
    L.seg_width = parts.size() > 1 ? static_cast<int>(nt ? parts[0]->rows() : parts[0]->cols()) : 0;
    for (size_t i = 0; i < parts.size(); ++i) {
      seg[i] = parts[i]->scale;
      const int pn = static_cast<int>(nt ? parts[i]->rows() : parts[i]->cols());
      if (parts.size() > 1 && pn != L.seg_width) fail(kStateError, "unequal fused segments");
    }
    L.seg_scale.resize(kMaxSegments);
    L.seg_scale.upload(seg.data(), kMaxSegments);
    int n0 = 0;
    for (auto* p : parts) {
      if (!p->is_int8) fail(kStateError, "no quantized copy of a weight");
      const int pn = static_cast<int>(nt ? p->rows() : p->cols());
      for (int j = 0; j < pn; ++j) {
        int8_t* dst = buf.data() + size_t(n0 + j) * L.k_pad;
        if (nt)
          std::copy(p->q.begin() + size_t(j) * k, p->q.begin() + size_t(j + 1) * k, dst);
        else
          for (int kk = 0; kk < k; ++kk) dst[kk] = p->q[size_t(kk) * pn + j];
      }
      n0 += pn;
    }
    L.q.resize(buf.size());
    L.q.upload(buf.data(), buf.size());
    if (gemv_copy) build_gemv_copy(L, L.q.get(), 1, st);
  } else {
    std::vector<float> kmaj(size_t(n) * k);
    int n0 = 0;
    for (auto* p : parts) {
      if (p->f32.empty()) fail(kStateError, "no f32 copy of a weight");
      const int pn = static_cast<int>(nt ? p->rows() : p->cols());
      for (int j = 0; j < pn; ++j) {
        float* dst = kmaj.data() + size_t(n0 + j) * k;
        if (nt)
          std::copy(p->f32.begin() + size_t(j) * k, p->f32.begin() + size_t(j + 1) * k, dst);
        else
          for (int kk = 0; kk < k; ++kk) dst[kk] = p->f32[size_t(kk) * pn + j];
      }
      n0 += pn;
    }
    upload_f32_operand(kmaj, n, k, prec, L, st);
    if (gemv_copy && prec == kBF16) {
      build_gemv_copy(L, L.h.get(), 2, st);
    } else if (gemv_copy) {  // plain fp32 rows (the GEMV splits them into tf32 hi + lo)
      std::vector<float> padded(size_t(n) * L.k_pad, 0.0f);
      for (int j = 0; j < n; ++j)
        std::copy(kmaj.begin() + size_t(j) * k, kmaj.begin() + size_t(j + 1) * k,
                  padded.begin() + size_t(j) * L.k_pad);
      DeviceBuffer<float> f(padded.size());
      f.upload(padded.data(), padded.size());
      build_gemv_copy(L, f.get(), 4, st);
    }
  }
}

void upload_vec(DeviceBuffer<float>& dst, const HostTensor& t) {
  dst.resize(t.f32.size());
  dst.upload(t.f32.data(), t.f32.size());
}

}  // namespace

Operand DevLinear::op() const {
  if (prec == kPrecI8) return Operand{q.get(), nullptr, n, k_pad, prec};
  if (prec == kPrecBF16) return Operand{h.get(), nullptr, n, k_pad, prec};
  return Operand{hi.get(), lo.get(), n, k_pad, prec};
}

void ActOperand::allocate(int rows_, int k_, int prec_) {
  rows = rows_;
  k = k_;
  prec = prec_;
  k_pad = pad_k(k, prec);
  const size_t n = size_t(rows) * k_pad;
  if (prec == kPrecI8) {
    q.resize(n);
    row_scale.resize(rows);
  } else if (prec == kPrecBF16) {
    h.resize(n);
  } else if (prec == kPrecTF32x3A) {
    hi.resize(n);  // plain fp32
  } else {
    hi.resize(n);
    lo.resize(n);
  }
}

Operand ActOperand::op() const {
  if (prec == kPrecI8) return Operand{q.get(), nullptr, rows, k_pad, prec};
  if (prec == kPrecBF16) return Operand{h.get(), nullptr, rows, k_pad, prec};
  return Operand{hi.get(), lo.get(), rows, k_pad, prec};
}

// ============================================================================
// construction / weights
// ============================================================================

// Narrowest GEMM tile the planner may pick (MTG_MIN_BN A/B switch; default 32).
static int gemm_min_bn() {
  static const int v = [] {
    const char* e = std::getenv("MTG_MIN_BN");
    const int b = e ? std::atoi(e) : 32;
    return (b == 64 || b == 128) ? b : 32;
  }();
  return v;
}

// Tile width forced for large-M (encoder) GEMMs (MTG_ENC_BN A/B switch; 0 = planner).
// MTG_ENC_BN_MAP="NxK:bn,..." overrides per shape (tuning).
static int enc_force_bn(int n, int k) {
  static const std::string map = [] {
    const char* e = std::getenv("MTG_ENC_BN_MAP");
    return std::string(e ? e : "");
  }();
  const std::string key = std::to_string(n) + "x" + std::to_string(k) + ":";
  const auto pos = map.find(key);
  if (pos != std::string::npos) return std::atoi(map.c_str() + pos + key.size());
  static const int v = [] {
    const char* e = std::getenv("MTG_ENC_BN");
    const int b = e ? std::atoi(e) : 0;
    return (b == 32 || b == 64 || b == 128 || b == 256) ? b : 0;
  }();
  return v;
}

// MTG_DEC_BN_MAP="NxK:bn,..." forces tile widths of the small-M (decoder) GEMMs (tuning).
static int dec_force_bn(int n, int k) {
  static const std::string map = [] {
    const char* e = std::getenv("MTG_DEC_BN_MAP");
    return std::string(e ? e : "");
  }();
  const std::string key = std::to_string(n) + "x" + std::to_string(k) + ":";
  const auto pos = map.find(key);
  return pos == std::string::npos ? 0 : std::atoi(map.c_str() + pos + key.size());
}

// Per-engine GEMM plans (tensor maps + tiling), used under the engine mutex.
std::map<Engine::PlanKey, GemmPlan>& Engine::plan_cache() {
  // Plans are keyed by row count; a ragged corpus brings a new one nearly
  // every batch. Graphs copy the tensor maps at capture, so dropping is safe.
  if (plans_.size() >= 8192) plans_.clear();
  return plans_;
}

Engine::Engine(HostModel model, int precision, int device)
    : host_(std::move(model)), prec_(precision), device_(device) {
  if (prec_ != kF32 && prec_ != kBF16 && prec_ != kINT8)
    fail(kUsageError, "unknown precision " + std::to_string(prec_));
  if (host_.quantized && prec_ != kINT8) prec_ = kINT8;  // tools/minimt.cpp:317-320
  if (const char* e = std::getenv("MTG_DIAG_EVENTS")) diag_ = e[0] == '1';
  if (const char* e = std::getenv("MTG_TRACE")) {
    trace_ = e[0] == '1' || e[0] == '2';
    trace_phases_ = e[0] == '2';
  }
  if (const char* e = std::getenv("MTG_NO_SPLIT_K")) split_k_ = e[0] != '1';
  if (prec_ == kINT8 && !host_.quantized) quantize_weights(host_);
  const ModelConfig& c = host_.config;
  c.validate();
  if (static_cast<int>(c.factor_configs.size()) > kMaxFactors)
    fail(kUsageError, "at most 4 source factors are supported by the GPU path");
  int ndev = 0;
  MTG_CUDA(cudaGetDeviceCount(&ndev));
  if (device_ < 0 || device_ >= ndev) fail(kUsageError, "bad device id " + std::to_string(device_));
  DeviceGuard guard(device_);
  MTG_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  MTG_CUDA(cudaMallocHost(&h_pinned_, 16 * sizeof(int)));
  d_ = c.d_model;
  dff_ = c.d_ff;
  V_ = c.tgt_vocab_size;
  Vp_ = static_cast<int>(topk_pitch(V_));
  part_ld_ = softmax_part_pitch(V_);
  T_ = c.max_seq_len;
  heads_ = c.num_heads;
  upload_weights();
}

Engine::~Engine() {
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(device_);
  diag_clear();
  clear_enc_graphs();
  plan_cache().clear();
  if (step_exec_) cudaGraphExecDestroy(step_exec_);
  if (multi_exec_) cudaGraphExecDestroy(multi_exec_);
  if (loop_exec_) cudaGraphExecDestroy(loop_exec_);
  if (step_graph_) cudaGraphDestroy(step_graph_);
  if (h_pinned_) cudaFreeHost(h_pinned_);
  if (res_host_) cudaFreeHost(res_host_);
  if (stream_) cudaStreamDestroy(stream_);
  if (prev >= 0 && prev != device_) cudaSetDevice(prev);
}

void Engine::upload_weights() {
  const ModelConfig& c = host_.config;
  auto P = [&](const std::string& n) -> const HostTensor& { return host_.at(n); };
  upload_vec(src_embed_, P("src_embed"));
  factor_embed_.clear();
  factor_embed_.resize(c.factor_configs.size());
  for (size_t i = 0; i < c.factor_configs.size(); ++i)
    if (!c.factor_configs[i].share_with_word_embedding)
      upload_vec(factor_embed_[i], P("factor" + std::to_string(i) + "_embed"));
  std::vector<float> pe = make_pos_enc(c.max_seq_len, c.d_model);
  pe_.resize(pe.size());
  pe_.upload(pe.data(), pe.size(), stream_);
  const HostTensor& te = P("tgt_embed");
  if (prec_ == kINT8) {
    tgt_embed_q_.resize(te.q.size());
    tgt_embed_q_.upload(te.q.data(), te.q.size(), stream_);
    tgt_scale_ = te.scale;
    // The int8 embedding lookup is q / scale (quant.cpp dequantize); the
    // table is dequantized once here (IEEE division, same bits as on device)
    // so the per-step lookup is a plain fp32 row read.
    std::vector<float> deq(te.q.size());
    for (size_t i = 0; i < deq.size(); ++i) deq[i] = static_cast<float>(te.q[i]) / te.scale;
    tgt_embed_f32_.resize(deq.size());
    tgt_embed_f32_.upload(deq.data(), deq.size(), stream_);
    MTG_CUDA(cudaStreamSynchronize(stream_));
  } else {
    upload_vec(tgt_embed_f32_, te);
  }
  build_linear(logits_w_, {&te}, true, prec_, stream_, true);
  auto ln = [&](LN& l, const std::string& p) {
    upload_vec(l.g, P(p + ".gain"));
    upload_vec(l.b, P(p + ".bias"));
  };
  enc_.clear();
  enc_.resize(c.num_encoder_layers);
  for (int l = 0; l < c.num_encoder_layers; ++l) {
    const std::string p = "enc" + std::to_string(l);
    EncLayer& L = enc_[l];
    ln(L.n1, p + ".norm1");
    ln(L.n2, p + ".norm2");
    build_linear(L.qkv, {&P(p + ".attn.wq"), &P(p + ".attn.wk"), &P(p + ".attn.wv")}, false, prec_,
                 stream_);
    build_linear(L.wo, {&P(p + ".attn.wo")}, false, prec_, stream_);
    build_linear(L.w1, {&P(p + ".ffn.w1")}, false, prec_, stream_);
    build_linear(L.w2, {&P(p + ".ffn.w2")}, false, prec_, stream_);
    upload_vec(L.b1, P(p + ".ffn.b1"));
    upload_vec(L.b2, P(p + ".ffn.b2"));
  }
  if (c.num_encoder_layers > 0) ln(enc_final_, "enc_final");
  dec_.clear();
  dec_.resize(c.num_decoder_layers);
  for (int l = 0; l < c.num_decoder_layers; ++l) {
    const std::string p = "dec" + std::to_string(l);
    DecLayer& L = dec_[l];
    ln(L.n1, p + ".norm1");
    ln(L.n2, p + ".norm2");
    ln(L.n3, p + ".norm3");
    build_linear(L.self_qkv, {&P(p + ".self.wq"), &P(p + ".self.wk"), &P(p + ".self.wv")}, false,
                 prec_, stream_, true);
    build_linear(L.self_wo, {&P(p + ".self.wo")}, false, prec_, stream_, true);
    build_linear(L.cross_q, {&P(p + ".cross.wq")}, false, prec_, stream_, true);
    build_linear(L.cross_kv, {&P(p + ".cross.wk"), &P(p + ".cross.wv")}, false, prec_, stream_);
    build_linear(L.cross_wo, {&P(p + ".cross.wo")}, false, prec_, stream_, true);
    build_linear(L.w1, {&P(p + ".ffn.w1")}, false, prec_, stream_, true);
    build_linear(L.w2, {&P(p + ".ffn.w2")}, false, prec_, stream_, true);
    upload_vec(L.b1, P(p + ".ffn.b1"));
    upload_vec(L.b2, P(p + ".ffn.b2"));
  }
  ln(dec_final_, "dec_final");
  MTG_CUDA(cudaStreamSynchronize(stream_));
}

// ============================================================================
// workspace
// ============================================================================

void Engine::ensure_workspace(int n_sent, int m_enc, int beam) {
  n_sent = std::max(n_sent, 1);
  m_enc = std::max(m_enc, 1);
  beam = std::max(beam, 1);
  // Grids, GEMM plans (split-K, tile widths) and the step graph are sized by
  // the capacity, so a much smaller batch after a big one (batch-1 serving)
  // shrinks the workspace instead of running mostly-idle grids.
  const bool shrink = cap_sent_ > 0 && 8 * n_sent <= cap_sent_ && 8 * m_enc <= cap_enc_;
  if (!shrink && n_sent <= cap_sent_ && m_enc <= cap_enc_ && beam <= cap_beam_) return;
  if (shrink) {
    cap_sent_ = n_sent;
    cap_enc_ = m_enc;
  } else {
    cap_sent_ = std::max(n_sent, cap_sent_);
    // Encoder rows grow geometrically (up to every sentence at max_seq_len):
    // a length-sorted corpus otherwise reallocates, re-plans and re-captures
    // on almost every batch. Only buffer sizes depend on cap_enc_.
    if (m_enc > cap_enc_)
      cap_enc_ = std::max(
          m_enc, std::min(2 * cap_enc_, cap_sent_ * std::max(host_.config.max_seq_len, 1)));
  }
  cap_beam_ = std::max(beam, cap_beam_);
  plan_cache().clear();
  clear_enc_graphs();
  ++ws_gen_;
  const ModelConfig& c = host_.config;
  const int N = cap_sent_, M = cap_enc_, B = cap_beam_;
  r_max_ = N * B;
  act_rows_ = std::max(M, r_max_);
  const int gp = act_prec_of(prec_);
  act_d_.allocate(act_rows_, d_, gp);
  act_ff_.allocate(act_rows_, dff_, gp);
  if (prec_ == kF32) act_logits_.allocate(act_rows_, d_, kPrecTF32x3);  // hi + lo for the projection
  const size_t d = d_, dff = dff_;
  enc_x_.resize(M * d);
  enc_a_.resize(M * d);
  enc_qkv_.resize(M * 3 * d);
  enc_ctx_.resize(M * d);
  ffh_.resize(size_t(act_rows_) * dff);
  ckv_.resize(c.num_decoder_layers);
  for (auto& b : ckv_) b.resize(M * 2 * d);
  dec_y_.resize(r_max_ * d);
  dec_a_.resize(r_max_ * d);
  dec_ctx_.resize(r_max_ * d);
  dec_cq_.resize(r_max_ * d);
  logits_.resize(size_t(r_max_) * Vp_);
  part_m_.resize(size_t(r_max_) * part_ld_);
  part_s_.resize(size_t(r_max_) * part_ld_);
  part_arg_.resize(size_t(r_max_) * part_ld_);
  qkv_cache_.resize(c.num_decoder_layers);
  for (auto& b : qkv_cache_) b.resize(size_t(T_) * r_max_ * 3 * d);
  src_ids_.resize(M);
  src_rowseg_.resize(M);
  rowmax_.resize(act_rows_);
  src_pos_.resize(M);
  src_off_.resize(N + 1);
  sent_absmax_.resize(N);
  if (gemv_ws_.size() == 0) {  // split-K partials and tickets of the GEMV kernels
    gemv_ws_.resize(size_t(1) << 18);
    gemv_sem_.resize(4096);
    MTG_CUDA(cudaMemsetAsync(gemv_sem_.get(), 0, gemv_sem_.size() * sizeof(int), stream_));
  }
  enc_off_.resize(N);
  enc_len_.resize(N);
  nonfinite_.resize(1);
  const size_t RT = size_t(r_max_) * T_;
  step_.resize(1);
  n_rows_.resize(1);
  row_sent_.resize(r_max_);
  row_prev_.resize(r_max_);
  row_parent_.resize(r_max_);
  row_lp_.resize(r_max_);
  anc0_.resize(RT);
  anc1_.resize(RT);
  tok0_.resize(RT);
  tok1_.resize(RT);
  cand_tok_.resize(size_t(r_max_) * B);
  cand_score_.resize(size_t(r_max_) * B);
  sent_row0_.resize(N);
  sent_live_.resize(N);
  sent_maxlen_.resize(N);
  sent_done_.resize(N);
  best_has_.resize(N);
  best_len_.resize(N);
  best_norm_.resize(N);
  best_lp_.resize(N);
  best_tok_.resize(size_t(N) * T_);
  res_len_.resize(N);
  res_status_.resize(N);
  res_lp_.resize(N);
  res_norm_.resize(N);
  res_flags_.resize(N);
  res_tok_.resize(size_t(N) * T_);
  sel_parent_.resize(size_t(N) * B);
  sel_tok_.resize(size_t(N) * B);
  sel_lp_.resize(size_t(N) * B);
  sel_count_.resize(1);

  BeamDev& b = beam_;
  b.step = step_.get();
  b.n_rows = n_rows_.get();
  b.row_sent = row_sent_.get();
  b.row_lp = row_lp_.get();
  b.row_prev = row_prev_.get();
  b.row_parent = row_parent_.get();
  b.anc[0] = anc0_.get();
  b.anc[1] = anc1_.get();
  b.tok[0] = tok0_.get();
  b.tok[1] = tok1_.get();
  b.cand_score = cand_score_.get();
  b.cand_tok = cand_tok_.get();
  b.sent_row0 = sent_row0_.get();
  b.sent_live = sent_live_.get();
  b.sent_maxlen = sent_maxlen_.get();
  b.sent_done = sent_done_.get();
  b.best_has = best_has_.get();
  b.best_norm = best_norm_.get();
  b.best_lp = best_lp_.get();
  b.best_len = best_len_.get();
  b.best_tok = best_tok_.get();
  b.res_len = res_len_.get();
  b.res_lp = res_lp_.get();
  b.res_norm = res_norm_.get();
  b.res_flags = res_flags_.get();
  b.res_status = res_status_.get();
  b.res_tok = res_tok_.get();
  b.sel_parent = sel_parent_.get();
  b.sel_tok = sel_tok_.get();
  b.sel_lp = sel_lp_.get();
  b.sel_count = sel_count_.get();
  b.N = N;
  b.B = B;
  b.T = T_;
  b.R_max = r_max_;
  b.V = V_;
  b.alpha = 1.0f;
  b.max_seq_len = c.max_seq_len;
}

// ============================================================================
// building blocks
// ============================================================================

void Engine::prep(const float* x, long long ldx, int k, int max_rows, const int* d_rows,
                  const int* seg_off, int n_seg, ActOperand& out) {
  if (prec_ == kINT8) {
    if (seg_off)
      launch_quantize_segments(x, ldx, k, seg_off, n_seg, nullptr, out.q.get(), out.k_pad,
                               out.row_scale.get(), nonfinite_.get(), stream_);
    else
      launch_quantize_rows(x, ldx, k, max_rows, d_rows, out.q.get(), out.k_pad,
                           out.row_scale.get(), nonfinite_.get(), stream_);
  } else if (prec_ == kBF16) {
    launch_cast_bf16(x, ldx, k, max_rows, d_rows, out.h.get(), out.k_pad, stream_);
  } else {  // kPrecTF32x3A: plain copy (lo == null); kPrecTF32x3: hi + lo
    launch_split_tf32(x, ldx, k, max_rows, d_rows, out.hi.get(),
                      out.prec == kPrecTF32x3 ? out.lo.get() : nullptr, out.k_pad, stream_);
  }
  count("operand prep");
}

void Engine::gemm(const ActOperand& a, const DevLinear& w, int m, const int* d_m, float* c,
                  long long ldc, const float* bias, const float* residual, int relu,
                  long long c_step_stride, const int* d_step, unsigned* seg_absmax,
                  float* c_lo, bool bf16_out) {
  auto& cache = plan_cache();
  PlanKey key{a.op().ptr, w.op().ptr, m};
  auto it = cache.find(key);
  if (it == cache.end())
    it = cache
             .emplace(key, plan_gemm(a.op(), w.op(), m, w.n,
                                     m > 512 ? enc_force_bn(w.n, a.op().k_pad)
                                             : dec_force_bn(w.n, a.op().k_pad),
                                     gemm_min_bn(), split_k_))
             .first;
  GemmEpilogue ep{};
  ep.C = c;
  ep.ldc = ldc;
  ep.c_step_stride = c_step_stride;
  ep.d_step = d_step;
  ep.bias = bias;
  ep.residual = residual;
  ep.ldr = ldc;
  ep.a_scale = a.row_scale.get();
  ep.w_seg_scale = w.seg_scale.get();
  ep.seg_width = w.seg_width;
  ep.relu = relu;
  ep.M = m;
  ep.d_M = d_m;
  ep.N = w.n;
  ep.C_lo = c_lo;
  ep.bf16_out = bf16_out ? 1 : 0;
  ep.tr = cur_tr_;
  cur_tr_ = KTrace{};
  if (seg_absmax) {
    if (residual) fail(kStateError, "gemm: sentence-max epilogue takes no residual");
    ep.seg_absmax = seg_absmax;
    ep.row_seg = src_rowseg_.get();
    ep.nonfinite = nonfinite_.get();
  }
  launch_gemm(it->second, ep, stream_);
  if (enc_diag_active_)
    count(w.n == 3 * d_ ? "enc gemm qkv" : w.n == 2 * d_ ? "enc gemm cross kv"
          : w.n == dff_ ? "enc gemm w1" : w.k == dff_ ? "enc gemm w2" : "enc gemm d x d");
  else
    count(w.n == 3 * d_ ? "gemm qkv" : w.n == 2 * d_ ? "gemm kv" : w.n == dff_ ? "gemm w1"
          : w.k == dff_ ? "gemm w2" : "gemm d x d");
}

void Engine::count(const char* tag) {
  ++launches_;
  if (diag_ && enc_diag_active_) {
    enc_marks_.push_back({tag, nullptr});
    MTG_CUDA(cudaEventCreate(&enc_marks_.back().ev));
    MTG_CUDA(cudaEventRecord(enc_marks_.back().ev, stream_));
  }
  if (diag_ && capturing_) {
    diag_marks_.push_back({tag, nullptr});
    MTG_CUDA(cudaEventCreate(&diag_marks_.back().ev));
    MTG_CUDA(cudaEventRecordWithFlags(diag_marks_.back().ev, stream_, cudaEventRecordExternal));
  }
}

void Engine::diag_clear() {
  for (auto& m : diag_marks_)
    if (m.ev) cudaEventDestroy(m.ev);
  diag_marks_.clear();
  diag_ms_.clear();
  diag_steps_ = 0;
  enc_agg_.clear();
  enc_total_ms_ = 0.0;
  enc_runs_ = 0;
}

std::string Engine::diag_report() {
  if (trace_) return trace_report();
  std::string out = "steps " + std::to_string(diag_steps_) + "\n";
  if (diag_steps_ == 0) return out;
  double total = 0.0;
  for (size_t i = 1; i < diag_ms_.size(); ++i) total += diag_ms_[i];
  for (size_t i = 1; i < diag_ms_.size(); ++i) {
    char line[160];
    std::snprintf(line, sizeof line, "%3zu %-32s %8.2f us\n", i, diag_marks_[i].name.c_str(),
                  1000.0 * diag_ms_[i] / diag_steps_);
    out += line;
  }
  char tl[96];
  std::snprintf(tl, sizeof tl, "total per step %.2f us\n", 1000.0 * total / diag_steps_);
  out += tl;
  if (enc_runs_ > 0) {
    out += "encoder (per run, " + std::to_string(enc_runs_) + " runs)\n";
    for (const auto& [tag, v] : enc_agg_) {
      char line[160];
      std::snprintf(line, sizeof line, "    %-32s %9.2f us  %4d launches  %7.2f us each\n",
                    tag.c_str(), 1000.0 * v.first / enc_runs_, v.second / enc_runs_,
                    1000.0 * v.first / v.second);
      out += line;
    }
    std::snprintf(tl, sizeof tl, "encoder total %.2f us\n", 1000.0 * enc_total_ms_ / enc_runs_);
    out += tl;
  }
  return out;
}

ShortlistArgs Engine::shortlist_args() const {
  ShortlistArgs a;
  a.sl_ids = sl_ids_.get();
  a.sl_off = sl_off_.get();
  a.K = d_;
  if (prec_ == kINT8) {
    a.aq = act_d_.q.get();
    a.a_scale = act_d_.row_scale.get();
    a.lda = act_d_.k_pad;
    a.wq = logits_w_.q.get();
    a.ldw = logits_w_.k_pad;
    a.w_scale = tgt_scale_;
  } else if (prec_ == kBF16) {
    a.ah = act_d_.h.get();
    a.lda = act_d_.k_pad;
    a.wh = logits_w_.h.get();
    a.ldw = logits_w_.k_pad;
  } else {
    a.af = dec_a_.get();
    a.lda = d_;
    a.wf = tgt_embed_f32_.get();
    a.ldw = d_;
  }
  return a;
}

// Tile width of the one-tile-per-CTA projection (MTG_LOGITS_BN A/B; 0 = planner).
static int logits_force_bn() {
  static const int v = [] {
    const char* e = std::getenv("MTG_LOGITS_BN");
    const int b = e ? std::atoi(e) : 0;
    return (b == 128 || b == 256) ? b : 0;
  }();
  return v;
}

void Engine::gemm_logits(int m, const int* d_m) {
  auto& cache = plan_cache();
  ActOperand& la = logits_act();
  PlanKey key{la.op().ptr, logits_w_.op().ptr, m};
  auto it = cache.find(key);
  // Persistent double-buffered kernel for TF32x3 (MMA-bound); the int8 / bf16
  // projection is epilogue-bound and measured faster as one tile per CTA at
  // two CTAs per SM. MTG_LOGITS_PERSISTENT=0/1 overrides (A/B).
  static const int persistent_env = [] {
    const char* e = std::getenv("MTG_LOGITS_PERSISTENT");
    return e ? std::atoi(e) : -1;
  }();
  const bool persistent = persistent_env >= 0 ? persistent_env != 0 : prec_ == kF32;
  // fp32: CTA-pair tiles (cta_group::2) cut the L2 -> SM operand traffic the
  // TF32x3 projection is bound by (MTG_LOGITS_PAIR=0: one CTA per tile, A/B).
  static const bool pair_env = [] {
    const char* e = std::getenv("MTG_LOGITS_PAIR");
    return !(e && e[0] == '0');
  }();
  // One 128-row tile (small batches) gains nothing from a pair: single CTA.
  const bool pair = persistent && pair_env && la.op().prec == kPrecTF32x3 && m > 128;
  if (it == cache.end())
    it = cache
             .emplace(key, pair         ? plan_logits_pair(la.op(), logits_w_.op(), m, logits_w_.n)
                           : persistent ? plan_logits(la.op(), logits_w_.op(), m, logits_w_.n)
                                        : plan_gemm(la.op(), logits_w_.op(), m, logits_w_.n,
                                                    logits_force_bn(), 128))
             .first;
  GemmEpilogue ep{};
  ep.C = logits_.get();
  ep.ldc = Vp_;
  ep.a_scale = la.row_scale.get();
  ep.w_seg_scale = logits_w_.seg_scale.get();
  ep.seg_width = logits_w_.seg_width;
  ep.M = m;
  ep.d_M = d_m;
  ep.N = logits_w_.n;
  ep.part_m = part_m_.get();
  ep.part_s = part_s_.get();
  ep.part_arg = part_arg_.get();
  ep.part_ld = part_ld_;
  ep.tr = cur_tr_;
  cur_tr_ = KTrace{};
  launch_gemm(it->second, ep, stream_);
  count("logits gemm + softmax partials");
}

// Validates and uploads sources (translate_one / beam_search / embed_source
// preconditions: decode.cpp:38-39, model.cpp:548, tensor.cpp:456-458).
int Engine::stage_sources(const std::vector<std::vector<int>>& srcs, std::vector<int>& status) {
  const int n = static_cast<int>(srcs.size());
  const ModelConfig& c = host_.config;
  const int nf = static_cast<int>(c.factor_configs.size());
  const auto* fac = staged_factors_.empty() ? nullptr : &staged_factors_;
  status.assign(n, 0);
  std::vector<int> ids, pos, seg, off(n + 1, 0), eoff(n, 0), elen(n, 0);
  std::vector<std::vector<int>> fids(nf);
  for (int s = 0; s < n; ++s) {
    const auto& src = srcs[s];
    // beam_search (decode.cpp:38-39), then embed_source_infer's checks in
    // order (model.cpp:541-548, tensor.cpp:456-458).
    const int have = fac ? static_cast<int>((*fac)[s].size()) : 0;
    if (src.empty()) {
      status[s] = kUsageError;
    } else if (have != nf) {
      status[s] = kShapeError;
    } else {
      for (int f = 0; f < nf; ++f)
        if ((*fac)[s][f].size() != src.size()) status[s] = kShapeError;
      if (status[s] == 0 && static_cast<int>(src.size()) > c.max_seq_len) status[s] = kValueError;
      if (status[s] == 0)
        for (int id : src)
          if (id < 0 || id >= c.src_vocab_size) status[s] = kIndexError;
      for (int f = 0; f < nf && status[s] == 0; ++f) {
        const int rows = c.factor_configs[f].share_with_word_embedding
                             ? c.src_vocab_size
                             : c.factor_configs[f].factor_vocab_size;
        for (int id : (*fac)[s][f])
          if (id < 0 || id >= rows) status[s] = kIndexError;
      }
    }
    if (status[s] == 0 && s < static_cast<int>(sl_status_.size())) status[s] = sl_status_[s];
    off[s] = static_cast<int>(ids.size());
    eoff[s] = off[s];
    if (status[s] == 0) {
      for (size_t i = 0; i < src.size(); ++i) {
        ids.push_back(src[i]);
        pos.push_back(static_cast<int>(i));
        seg.push_back(s);
        for (int f = 0; f < nf; ++f) fids[f].push_back((*fac)[s][f][i]);
      }
      elen[s] = static_cast<int>(src.size());
    }
  }
  off[n] = static_cast<int>(ids.size());
  const int m = off[n];
  if (m) {
    src_ids_.upload(ids.data(), m, stream_);
    src_pos_.upload(pos.data(), m, stream_);
    src_rowseg_.upload(seg.data(), m, stream_);
    if (nf > 0) {
      src_fids_.resize(static_cast<size_t>(nf) * m);
      for (int f = 0; f < nf; ++f) src_fids_.upload(fids[f].data(), m, stream_, size_t(f) * m);
      MTG_CUDA(cudaStreamSynchronize(stream_));  // host vectors are freed on return
    }
  }
  src_off_.upload(off.data(), n + 1, stream_);
  enc_off_.upload(eoff.data(), n, stream_);
  enc_len_.upload(elen.data(), n, stream_);
  return m;
}

OperandOut Engine::opout(ActOperand& a) {
  OperandOut o;
  o.prec = a.prec;
  o.k_pad = a.k_pad;
  o.q = a.q.get();
  o.row_scale = a.row_scale.get();
  o.h = a.h.get();
  o.hi = a.hi.get();
  o.lo = a.lo.get();
  o.nonfinite = nonfinite_.get();
  return o;
}

// Encoder operand for the next GEMM. int8: one scale per sentence (the
// reference quantizes the [S x k] tensor its Executor::linear receives).
void Engine::prep_enc(const float* x, long long ldx, int k, int m, ActOperand& out,
                      bool have_rowmax) {
  if (prec_ == kINT8) {
    if (!have_rowmax) {
      launch_rowmax(x, ldx, m, k, rowmax_.get(), nonfinite_.get(), stream_);
      count("enc rowmax");
    }
    launch_quantize_seg(x, ldx, m, k, src_rowseg_.get(), src_off_.get(), rowmax_.get(),
                        opout(out), stream_);
    count("enc quantize_seg");
  } else {
    prep(x, ldx, k, m, nullptr, nullptr, 0, out);
  }
}

// Encoder LayerNorm; int8 also records per-row max |y| for the segment scale.
void Engine::ln_enc(const float* x, int m, const LN& ln, float* y, ActOperand& out) {
  if (prec_ == kINT8 && enc_fused_) {  // fused LN + per-sentence quantization
    OperandOut o = opout(out);
    o.tr = enc_ln_tr_;
    enc_ln_tr_ = KTrace{};
    launch_ln_quant_sent(x, d_, src_off_.get(), enc_n_sent_, d_, ln.g.get(), ln.b.get(), y, d_,
                         o, sent_absmax_.get(), stream_, std::max(enc_max_src_, 1));
    count("enc layernorm+quantize");
    return;
  }
  if (prec_ == kINT8) {
    launch_layernorm(x, d_, m, nullptr, d_, ln.g.get(), ln.b.get(), y, d_, rowmax_.get(),
                     nullptr, stream_);
    count("enc layernorm");
    prep_enc(y, d_, d_, m, out, true);
  } else {
    const OperandOut o = opout(out);
    launch_layernorm(x, d_, m, nullptr, d_, ln.g.get(), ln.b.get(), y, d_, nullptr, &o, stream_);
    count("enc layernorm");
  }
}

void Engine::run_encoder(int n_sent, int m, int max_src) {
  if (m <= 0) return;
  if (diag_ && !capturing_) {
    enc_diag_active_ = true;
    enc_marks_.push_back({"start", nullptr});
    MTG_CUDA(cudaEventCreate(&enc_marks_.back().ev));
    MTG_CUDA(cudaEventRecord(enc_marks_.back().ev, stream_));
  }
  static const bool graphs = [] {
    const char* e = std::getenv("MTG_ENC_GRAPH");
    return !(e && e[0] == '0');
  }();
  if (graphs && !diag_ && !capturing_) {
    // The encoder's ~9 kernels per layer replay as one CUDA graph per batch
    // shape (exact key: workspace generation, sizes, factor-id buffer).
    const EncKey key{ws_gen_, n_sent, m, max_src, src_fids_.get()};
    auto it = enc_graphs_.find(key);
    // Capture a shape on its second use: a corpus of ragged batches (a new
    // row count nearly every call) runs eagerly instead of paying a capture
    // and instantiation per call.
    if (it == enc_graphs_.end() && enc_seen_.insert(key).second) {
      if (enc_seen_.size() >= 4096) enc_seen_.clear();
      run_encoder_body(n_sent, m, max_src);
      return;
    }
    if (it == enc_graphs_.end()) {
      if (enc_graphs_.size() >= 256) clear_enc_graphs();
      const int64_t before = launches_;
      cudaGraph_t g = nullptr;
      MTG_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
      capturing_ = true;
      try {
        run_encoder_body(n_sent, m, max_src);
      } catch (...) {
        capturing_ = false;
        cudaStreamEndCapture(stream_, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      capturing_ = false;
      MTG_CUDA(cudaStreamEndCapture(stream_, &g));
      cudaGraphExec_t exec = nullptr;
      const cudaError_t err = cudaGraphInstantiate(&exec, g, 0);
      cudaGraphDestroy(g);
      MTG_CUDA(err);
      it = enc_graphs_.emplace(key, std::make_pair(exec, launches_ - before)).first;
      launches_ = before;
    }
    MTG_CUDA(cudaGraphLaunch(it->second.first, stream_));
    launches_ += it->second.second;
    return;
  }
  run_encoder_body(n_sent, m, max_src);
  if (enc_diag_active_) {
    enc_diag_active_ = false;
    MTG_CUDA(cudaStreamSynchronize(stream_));
    for (size_t i = 1; i < enc_marks_.size(); ++i) {
      float ms = 0.0f;
      MTG_CUDA(cudaEventElapsedTime(&ms, enc_marks_[i - 1].ev, enc_marks_[i].ev));
      auto& a = enc_agg_[enc_marks_[i].name];
      a.first += ms;
      a.second += 1;
      enc_total_ms_ += ms;
    }
    for (auto& mk : enc_marks_) cudaEventDestroy(mk.ev);
    enc_marks_.clear();
    ++enc_runs_;
  }
}

void Engine::clear_enc_graphs() {
  for (auto& kv : enc_graphs_) cudaGraphExecDestroy(kv.second.first);
  enc_graphs_.clear();
}

void Engine::run_encoder_body(int n_sent, int m, int max_src) {
  const ModelConfig& c = host_.config;
  const long long d = d_;
  const float sqrt_d = std::sqrt(static_cast<float>(c.d_model));
  const float scale = 1.0f / std::sqrt(static_cast<float>(d_ / heads_));
  SrcEmbed se;
  se.word = src_embed_.get();
  se.wdim = c.word_embed_dim();
  se.n_factors = static_cast<int>(c.factor_configs.size());
  if (se.n_factors > 0) {
    const FactorCombine mode = c.factor_configs.front().combine;
    se.mode = mode == FactorCombine::kConcat ? 0 : mode == FactorCombine::kSum ? 1 : 2;
    for (int f = 0; f < se.n_factors; ++f) {
      se.table[f] = c.factor_configs[f].share_with_word_embedding ? src_embed_.get()
                                                                  : factor_embed_[f].get();
      se.fdim[f] = c.factor_configs[f].embed_dim;
    }
    se.fids = src_fids_.get();
    se.fstride = m;
    se.avg_scale = 1.0f / (1.0f + static_cast<float>(se.n_factors));  // model.cpp:573
  }
  launch_embed_src(src_ids_.get(), src_pos_.get(), m, se, d_, sqrt_d, pe_.get(), enc_x_.get(), d,
                   stream_);
  count("enc embed");
  enc_n_sent_ = n_sent;
  enc_max_src_ = max_src;
  // int8 with d <= 512: the LayerNorms quantize per sentence themselves and
  // zero the sentence max that attention / the FFN-up epilogue accumulate,
  // so each remaining quantize is a single pass (9 kernels per layer).
  static const bool no_enc_fusion = [] {
    const char* e = std::getenv("MTG_NO_ENC_FUSION");
    return e && e[0] == '1';
  }();
  const bool fused = prec_ == kINT8 && d_ <= 512 && !no_enc_fusion;
  enc_fused_ = fused;
  // MTG_BF16_DIRECT=0: bf16 contexts / hidden rows through cast kernels (A/B)
  static const bool bf16_direct_ok = [] {
    const char* e = std::getenv("MTG_BF16_DIRECT");
    return !(e && e[0] == '0');
  }();
  const OperandOut od = opout(act_d_), off_ = opout(act_ff_);
  for (int l = 0; l < c.num_encoder_layers; ++l) {
    EncLayer& L = enc_[l];
    enc_ln_tr_ = enc_trace(l, 0, "enc layernorm 1");
    ln_enc(enc_x_.get(), m, L.n1, enc_a_.get(), act_d_);
    cur_tr_ = enc_trace(l, 1, "enc gemm qkv");
    gemm(act_d_, L.qkv, m, nullptr, enc_qkv_.get(), 3 * d, nullptr, nullptr, 0);
    const bool plain = prec_is_tf32x3(act_d_.prec);  // fp32: contexts are the operand
    // bf16 (head dim 64, unpadded rows): the attention writes the bf16
    // operand and the FFN-up GEMM its bf16 hidden operand (no cast kernels)
    const bool bf16_direct = bf16_direct_ok && prec_ == kBF16 && d_ / heads_ == 64 &&
                             act_d_.k_pad == d_ && act_ff_.k_pad == dff_;
    float* const ctx_out = plain ? act_d_.hi.get()
                           : bf16_direct ? reinterpret_cast<float*>(act_d_.h.get())
                                         : enc_ctx_.get();
    launch_enc_attention(enc_qkv_.get(), 3 * d, src_off_.get(), n_sent, std::max(max_src, 1), d_,
                         heads_, scale, ctx_out, plain || bf16_direct ? act_d_.k_pad : d,
                         act_d_.prec == kPrecTF32x3 ? act_d_.lo.get() : nullptr,
                         fused ? sent_absmax_.get() : nullptr, nonfinite_.get(), stream_,
                         enc_trace(l, 2, "enc attention"), bf16_direct);
    count("enc attention");
    if (plain || bf16_direct) {
    } else if (fused) {
      launch_quantize_sent(enc_ctx_.get(), d, m, d_, src_rowseg_.get(), sent_absmax_.get(), od,
                           stream_);
      count("enc quantize (sentence max)");
    } else {
      prep_enc(enc_ctx_.get(), d, d_, m, act_d_, false);
    }
    cur_tr_ = enc_trace(l, 3, "enc gemm wo (+res)");
    gemm(act_d_, L.wo, m, nullptr, enc_x_.get(), d, nullptr, enc_x_.get(), 0);
    enc_ln_tr_ = enc_trace(l, 4, "enc layernorm 2");
    ln_enc(enc_x_.get(), m, L.n2, enc_a_.get(), act_d_);
    cur_tr_ = enc_trace(l, 5, "enc gemm w1 (+b1, relu)");
    if (plain) {
      gemm(act_d_, L.w1, m, nullptr, act_ff_.hi.get(), act_ff_.k_pad, L.b1.get(), nullptr, 1, 0,
           nullptr, nullptr, act_ff_.prec == kPrecTF32x3 ? act_ff_.lo.get() : nullptr);
    } else if (bf16_direct) {
      gemm(act_d_, L.w1, m, nullptr, reinterpret_cast<float*>(act_ff_.h.get()), act_ff_.k_pad,
           L.b1.get(), nullptr, 1, 0, nullptr, nullptr, nullptr, true);
    } else {
      gemm(act_d_, L.w1, m, nullptr, ffh_.get(), dff_, L.b1.get(), nullptr, 1, 0, nullptr,
           fused ? sent_absmax_.get() : nullptr);
    }
    if (plain || bf16_direct) {
    } else if (fused) {
      launch_quantize_sent(ffh_.get(), dff_, m, dff_, src_rowseg_.get(), sent_absmax_.get(), off_,
                           stream_);
      count("enc quantize (sentence max)");
    } else {
      prep_enc(ffh_.get(), dff_, dff_, m, act_ff_, false);
    }
    cur_tr_ = enc_trace(l, 6, "enc gemm w2 (+b2, res)");
    gemm(act_ff_, L.w2, m, nullptr, enc_x_.get(), d, L.b2.get(), enc_x_.get(), 0);
  }
  if (c.num_decoder_layers == 0) {
    if (c.num_encoder_layers > 0) {
      launch_layernorm(enc_x_.get(), d, m, nullptr, d_, enc_final_.g.get(), enc_final_.b.get(),
                       enc_a_.get(), d, nullptr, nullptr, stream_);
      count();
    }
    return;
  }
  // init_decoder (model.cpp:598-612): one quantization of enc_out per
  // sentence feeds every layer's cross K and V.
  if (c.num_encoder_layers > 0)
    ln_enc(enc_x_.get(), m, enc_final_, enc_a_.get(), act_d_);
  else
    prep_enc(enc_x_.get(), d, d_, m, act_d_, false);
  for (int l = 0; l < c.num_decoder_layers; ++l)
    gemm(act_d_, dec_[l].cross_kv, m, nullptr, ckv_[l].get(), 2 * d, nullptr, nullptr, 0);
}

bool Engine::small_path() const {
  static const bool enabled = [] {
    const char* e = std::getenv("MTG_SMALL_BATCH");
    return !(e && e[0] == '0');
  }();
  return enabled && r_max_ <= kGemvRows && d_ <= 512 && !use_shortlist_;
}

GemvArgs Engine::gemv_args(const DevLinear& w) const {
  GemvArgs g;
  g.d_rows = n_rows_.get();
  g.rows_alloc = std::min(r_max_, kGemvRows);
  g.d_step = step_.get();
  g.K = w.k;
  g.k_pad = w.k_pad;
  g.N = w.n;
  g.w = w.frag.get();
  if (!g.w) fail(kStateError, "gemv: fragment-order weight copy missing");
  g.w_seg_scale = w.seg_scale.get();
  g.seg_width = w.seg_width;
  g.nonfinite = nonfinite_.get();
  return g;
}

KTrace Engine::next_trace(const char* name) {
  KTrace k;
  if (!trace_) return k;
  const int per = kTraceSlots;
  if (trace_buf_.size() < size_t(2) * T_ * per) return k;  // sized by trace_reset
  if (trace_slot_ >= per) return k;
  if (static_cast<int>(trace_names_.size()) <= trace_slot_) trace_names_.push_back(name);
  k.buf = trace_buf_.get();
  if (trace_phases_) k.ph = phase_buf_.get();
  k.slot = trace_slot_++;
  k.per_step = per;
  k.d_step = step_.get();
  trace_per_step_ = per;
  return k;
}

KTrace Engine::enc_trace(int layer, int slot, const char* name) {
  KTrace k;
  if (!trace_ || slot >= kEncTraceSlots || layer >= enc_trace_layers_) return k;
  if (static_cast<int>(enc_trace_names_.size()) <= slot) enc_trace_names_.resize(slot + 1);
  enc_trace_names_[slot] = name;
  k.buf = enc_trace_buf_.get();
  k.slot = slot;
  k.per_step = kEncTraceSlots;
  k.d_step = enc_layer_ids_.get() + layer;
  if (trace_phases_) {
    k.ph = enc_phase_buf_.get();
    k.d_step = enc_layer_ids_.get() + layer;
  }
  return k;
}

void Engine::trace_reset() {
  if (!trace_) return;
  const int L = host_.config.num_encoder_layers;
  if (L > 0) {
    if (enc_trace_layers_ < L) {
      enc_layer_ids_.resize(L);
      std::vector<int> ids(L);
      for (int i = 0; i < L; ++i) ids[i] = i;
      enc_layer_ids_.upload(ids.data(), ids.size(), stream_);
      enc_trace_buf_.resize(size_t(2) * L * kEncTraceSlots);
      enc_phase_buf_.resize(size_t(kTracePhases) * L * kEncTraceSlots);
      enc_trace_layers_ = L;
    }
    std::vector<unsigned long long> z(enc_phase_buf_.size(), 0ull);
    enc_phase_buf_.upload(z.data(), z.size(), stream_);
    std::vector<unsigned long long> e(enc_trace_buf_.size());
    for (size_t i = 0; i < e.size(); ++i) e[i] = (i & 1) ? 0ull : ~0ull;
    enc_trace_buf_.upload(e.data(), e.size(), stream_);
  }
  const size_t need = size_t(2) * T_ * kTraceSlots;
  if (trace_buf_.size() < need) trace_buf_.resize(need);
  std::vector<unsigned long long> init(trace_buf_.size());
  for (size_t i = 0; i < init.size(); ++i) init[i] = (i & 1) ? 0ull : ~0ull;
  trace_buf_.upload(init.data(), init.size(), stream_);
  if (trace_phases_) {
    const size_t np = size_t(kTracePhases) * T_ * kTraceSlots;
    if (phase_buf_.size() < np) phase_buf_.resize(np);
    std::vector<unsigned long long> z(phase_buf_.size(), 0ull);
    phase_buf_.upload(z.data(), z.size(), stream_);
  }
}

// Per kernel of the step: mean gap from the previous traced kernel's last CTA
// exit to this kernel's first post-wait CTA, and mean duration (post-wait to
// last exit); "tail" = from the last traced kernel of a step to the first of
// the next (top-k + beam select + launch gaps).
std::string Engine::trace_report() {
  if (!trace_ || trace_per_step_ == 0) return "";
  std::vector<unsigned long long> b(trace_buf_.size());
  MTG_CUDA(cudaStreamSynchronize(stream_));
  trace_buf_.download(b.data(), b.size());
  const int per = trace_per_step_;
  auto valid = [&](const unsigned long long* s, int k) { return s[2 * k] != ~0ull && s[2 * k + 1] != 0ull; };
  std::vector<double> gap(per, 0.0), dur(per, 0.0);
  std::vector<int> ngap(per, 0), ndur(per, 0);
  std::vector<unsigned long long> pb;
  if (trace_phases_) {
    pb.resize(phase_buf_.size());
    phase_buf_.download(pb.data(), pb.size());
  }
  std::vector<double> ph(size_t(per) * kTracePhases, 0.0);
  std::vector<int> nph(size_t(per) * kTracePhases, 0);
  double total = 0.0;
  int steps = 0;
  for (int t = 0; t + 1 < T_; ++t) {
    const unsigned long long* s = b.data() + size_t(2) * t * per;
    const unsigned long long* nx = s + 2 * per;
    int first = -1, prev = -1, last = -1, nfirst = -1;
    for (int k = 0; k < per; ++k) {
      if (!valid(s, k)) continue;
      if (first < 0) first = k;
      dur[k] += double(s[2 * k + 1]) - double(s[2 * k]);
      ++ndur[k];
      if (!pb.empty()) {
        const unsigned long long* p = pb.data() + (size_t(t) * per + k) * kTracePhases;
        for (int i = 0; i < kTracePhases; ++i)
          if (p[i] != 0ull) {
            ph[size_t(k) * kTracePhases + i] += double(p[i]) - double(s[2 * k]);
            ++nph[size_t(k) * kTracePhases + i];
          }
      }
      if (prev >= 0) {
        gap[k] += double(s[2 * k]) - double(s[2 * prev + 1]);
        ++ngap[k];
      }
      prev = last = k;
    }
    for (int k = 0; k < per && nfirst < 0; ++k)
      if (valid(nx, k)) nfirst = k;
    if (first < 0 || nfirst < 0) break;
    gap[nfirst] += double(nx[2 * nfirst]) - double(s[2 * last + 1]);
    ++ngap[nfirst];
    total += double(nx[2 * nfirst]) - double(s[2 * first]);
    ++steps;
  }
  if (steps == 0) return "trace: no complete step\n";
  std::string out = "trace (" + std::to_string(steps) + " steps, us): gap before / duration\n";
  for (int k = 0; k < per; ++k) {
    if (ndur[k] == 0) continue;
    char line[200];
    std::snprintf(line, sizeof line, "  %2d %-34s %6.2f  %6.2f\n", k,
                  k < static_cast<int>(trace_names_.size()) ? trace_names_[k].c_str() : "?",
                  ngap[k] ? gap[k] / ngap[k] / 1000.0 : 0.0, dur[k] / ndur[k] / 1000.0);
    out += line;
    std::string pl;
    for (int i = 0; i < kTracePhases; ++i) {
      const int n = nph[size_t(k) * kTracePhases + i];
      if (n == 0) continue;
      char b2[48];
      std::snprintf(b2, sizeof b2, " p%d %.2f", i, ph[size_t(k) * kTracePhases + i] / n / 1000.0);
      pl += b2;
    }
    if (!pl.empty()) out += "      phases (us after first start):" + pl + "\n";
  }
  char tl[200];
  std::snprintf(tl, sizeof tl, "  step %.2f us (first kernel's gap: from the previous step's last)\n",
                total / steps / 1000.0);
  out += tl;
  // Encoder GEMMs: gap from the previous traced GEMM (the untraced LayerNorm /
  // attention / quantize kernels in between fall into it), duration; over
  // layers 1.. (the first follows the embedding).
  if (enc_trace_layers_ > 0 && !enc_trace_names_.empty()) {
    std::vector<unsigned long long> e(enc_trace_buf_.size());
    enc_trace_buf_.download(e.data(), e.size());
    const int K = kEncTraceSlots, L = enc_trace_layers_;
    std::vector<double> g(K, 0.0), du(K, 0.0);
    std::vector<int> ng(K, 0), nd(K, 0);
    double lay = 0.0;
    int nl = 0;
    long long prev_end = -1;
    long long layer_first = -1, prev_layer_first = -1;
    int first_slot = 0;  // first traced slot of a layer (the LayerNorm only for int8)
    while (first_slot < K && (e[2 * first_slot] == ~0ull || e[2 * first_slot + 1] == 0ull)) ++first_slot;
    for (int l = 0; l < L; ++l) {
      for (int k = 0; k < K; ++k) {
        const unsigned long long b0 = e[2 * (size_t(l) * K + k)], b1 = e[2 * (size_t(l) * K + k) + 1];
        if (b0 == ~0ull || b1 == 0ull) continue;
        du[k] += double(b1) - double(b0);
        ++nd[k];
        if (prev_end >= 0 && l > 0) {
          g[k] += double(b0) - double(prev_end);
          ++ng[k];
        }
        if (k == first_slot) {
          prev_layer_first = layer_first;
          layer_first = static_cast<long long>(b0);
          if (prev_layer_first >= 0) {
            lay += double(layer_first) - double(prev_layer_first);
            ++nl;
          }
        }
        prev_end = static_cast<long long>(b1);
      }
    }
    std::vector<unsigned long long> pe;
    if (trace_phases_) {
      pe.resize(enc_phase_buf_.size());
      enc_phase_buf_.download(pe.data(), pe.size());
    }
    out += "encoder (" + std::to_string(L) + " layers, us): gap before / duration\n";
    for (int k = 0; k < K && k < static_cast<int>(enc_trace_names_.size()); ++k) {
      if (nd[k] == 0) continue;
      char line[200];
      std::snprintf(line, sizeof line, "  %2d %-34s %6.2f  %6.2f\n", k, enc_trace_names_[k].c_str(),
                    ng[k] ? g[k] / ng[k] / 1000.0 : 0.0, du[k] / nd[k] / 1000.0);
      out += line;
      if (!pe.empty()) {
        std::string pl;
        for (int i = 0; i < kTracePhases; ++i) {
          double acc = 0.0;
          int cnt = 0;
          for (int l = 0; l < L; ++l) {
            const unsigned long long v = pe[(size_t(l) * K + k) * kTracePhases + i];
            const unsigned long long b0 = e[2 * (size_t(l) * K + k)];
            if (v != 0ull && b0 != ~0ull) {
              acc += double(v) - double(b0);
              ++cnt;
            }
          }
          if (cnt == 0) continue;
          char b2[48];
          std::snprintf(b2, sizeof b2, " p%d %.2f", i, acc / cnt / 1000.0);
          pl += b2;
        }
        if (!pl.empty()) out += "      phases (us after first start):" + pl + "\n";
      }
    }
    if (nl > 0) {
      std::snprintf(tl, sizeof tl, "  layer %.2f us\n", lay / nl / 1000.0);
      out += tl;
    }
  }
  return out;
}

// decode_step (model.cpp:614-672) for <= kGemvRows live rows: per decoder
// layer QKV, self-attention, Wo(+res), cross-Wq, cross-attention,
// cross-Wo(+res), W1(+b1, ReLU), W2(+b2, res); the LayerNorms, the target
// embedding (+ history reorder) and every int8 row quantization run inside
// the consuming GEMV, so a step is 8 kernels per layer + projection + tail.
void Engine::decoder_body_small(bool reorder) {
  const ModelConfig& c = host_.config;
  const long long d = d_;
  const int R = r_max_;
  const int* dr = n_rows_.get();
  const float sqrt_d = std::sqrt(static_cast<float>(c.d_model));
  const float scale = 1.0f / std::sqrt(static_cast<float>(d_ / heads_));
  const int gp = prec_ == kINT8 ? 0 : prec_ == kBF16 ? 1 : 2;
  trace_slot_ = 0;
  OperandOut none;
  none.prec = -1;  // attention writes the fp32 context only
  static const bool small_attn_env = [] {
    const char* e = std::getenv("MTG_SMALL_ATTN");
    return !(e && e[0] == '0');
  }();
  const bool small_attn = small_attn_env && attn_small_supported(d_, heads_, T_, T_);
  auto set_start = [&](GemvArgs& g) {  // first consumer of the step: embedding + reorder
    g.a_mode = 2;
    g.prev = row_prev_.get();
    g.table = tgt_embed_f32_.get();  // int8: q / scale, dequantized at load
    g.table_rows = V_;
    g.pe = pe_.get();
    g.sqrt_d = sqrt_d;
    g.x_out = dec_y_.get();
    g.ldx_out = d;
    // with the small attention, the layer-0 attention kernel does the reorder
    g.reorder = reorder && !(small_attn && c.num_decoder_layers > 0) ? 1 : 0;
    g.row_parent = row_parent_.get();
    g.anc[0] = anc0_.get();
    g.anc[1] = anc1_.get();
    g.tok[0] = tok0_.get();
    g.tok[1] = tok1_.get();
    g.T = T_;
  };
  auto ln_from = [&](GemvArgs& g, const LN& ln) {
    g.a_mode = 1;
    g.x = dec_y_.get();
    g.ldx = d;
    g.ln_g = ln.g.get();
    g.ln_b = ln.b.get();
  };
  auto rows_from = [&](GemvArgs& g, const float* x, long long ldx) {
    g.a_mode = 0;
    g.x = x;
    g.ldx = ldx;
  };
  auto out_to = [&](GemvArgs& g, float* C, long long ldc, const float* bias, bool res, int relu) {
    g.C = C;
    g.ldc = ldc;
    g.bias = bias;
    g.residual = res ? C : nullptr;
    g.ldr = ldc;
    g.relu = relu;
  };
  for (int l = 0; l < c.num_decoder_layers; ++l) {
    DecLayer& L = dec_[l];
    GemvArgs q = gemv_args(L.self_qkv);
    if (l == 0) set_start(q);
    q.x = dec_y_.get();  // a_mode 2 ignores x; LayerNorm params below
    q.ldx = d;
    if (l > 0) ln_from(q, L.n1);
    q.ln_g = L.n1.g.get();
    q.ln_b = L.n1.b.get();
    out_to(q, qkv_cache_[l].get(), 3 * d, nullptr, false, 0);
    q.c_step_stride = static_cast<long long>(R) * 3 * d;
    q.trace = next_trace(l == 0 ? "gemv qkv (+embed, LN)" : "gemv qkv (+LN)");
    launch_gemv(gp, false, q, stream_);
    count(l == 0 ? "gemv qkv (+embed, LN)" : "gemv qkv (+LN)");
    if (small_attn) {
      launch_attn_small_self(qkv_cache_[l].get(), R, T_, anc0_.get(), anc1_.get(),
                             row_parent_.get(), reorder ? 1 : 0, tok0_.get(), tok1_.get(),
                             row_prev_.get(), l == 0 ? 1 : 0, dr, step_.get(),
                             std::min(R, kGemvRows), d_, heads_, scale, dec_ctx_.get(), d, stream_,
                             next_trace("self attention"));
    } else {
      // the QKV GEMV of layer 0 did the history reorder: no early reads
      launch_dec_self_attention(qkv_cache_[l].get(), R, T_, anc0_.get(), anc1_.get(), dr,
                                step_.get(), d_, heads_, scale, dec_ctx_.get(), d, none, stream_,
                                l == 0 && reorder ? 0 : 1);
    }
    count("self attention");
    GemvArgs o = gemv_args(L.self_wo);
    rows_from(o, dec_ctx_.get(), d);
    out_to(o, dec_y_.get(), d, nullptr, true, 0);
    o.trace = next_trace("gemv wo (+res)");
    launch_gemv(gp, false, o, stream_);
    count("gemv wo (+res)");
    GemvArgs cq = gemv_args(L.cross_q);
    ln_from(cq, L.n2);
    out_to(cq, dec_cq_.get(), d, nullptr, false, 0);
    cq.trace = next_trace("gemv cross wq (+LN)");
    launch_gemv(gp, false, cq, stream_);
    count("gemv cross wq (+LN)");
    if (small_attn) {
      launch_attn_small_cross(dec_cq_.get(), d, ckv_[l].get(), row_sent_.get(), enc_off_.get(),
                              enc_len_.get(), dr, std::min(R, kGemvRows), T_, d_, heads_, scale,
                              dec_ctx_.get(), d, stream_, next_trace("cross attention"));
    } else {
      launch_dec_cross_attention(dec_cq_.get(), d, ckv_[l].get(), row_sent_.get(), enc_off_.get(),
                                 enc_len_.get(), dr, R, T_, d_, heads_, scale, dec_ctx_.get(), d,
                                 none, stream_);
    }
    count("cross attention");
    GemvArgs co = gemv_args(L.cross_wo);
    rows_from(co, dec_ctx_.get(), d);
    out_to(co, dec_y_.get(), d, nullptr, true, 0);
    co.trace = next_trace("gemv cross wo (+res)");
    launch_gemv(gp, false, co, stream_);
    count("gemv cross wo (+res)");
    GemvArgs f1 = gemv_args(L.w1);
    ln_from(f1, L.n3);
    out_to(f1, ffh_.get(), dff_, L.b1.get(), false, 1);
    f1.trace = next_trace("gemv w1 (+LN, b1, relu)");
    launch_gemv(gp, false, f1, stream_);
    count("gemv w1 (+LN, b1, relu)");
    GemvArgs f2 = gemv_args(L.w2);
    rows_from(f2, ffh_.get(), dff_);
    out_to(f2, dec_y_.get(), d, L.b2.get(), true, 0);
    // MTG_GEMV_W2_SPLIT=k: fp32 / bf16 FFN-down split over k CTAs per column
    // chunk (partials added in split order; int8 rows need their whole-row
    // max and stay unsplit). Default unsplit: the split's ticket and partial
    // round trip measured slower at batch 1 (bf16 step 86.5 -> 81.5 us
    // unsplit, fp32 107.4 -> 105.2 us).
    static const int w2_split = [] {
      const char* e = std::getenv("MTG_GEMV_W2_SPLIT");
      return e ? std::atoi(e) : 1;
    }();
    if (prec_ != kINT8 && w2_split > 1 && L.w2.k_pad * (prec_ == kF32 ? 4 : 2) % (w2_split * 128) == 0 &&
        L.w2.k_pad >= 1024) {
      f2.ksplit = w2_split;
      f2.ws = gemv_ws_.get();
      f2.sem = gemv_sem_.get();
    }
    f2.trace = next_trace("gemv w2 (+b2, res)");
    launch_gemv(gp, false, f2, stream_);
    count("gemv w2 (+b2, res)");
  }
  GemvArgs lg = gemv_args(logits_w_);
  if (c.num_decoder_layers == 0) set_start(lg);
  else ln_from(lg, dec_final_);
  lg.x = dec_y_.get();
  lg.ldx = d;
  lg.ln_g = dec_final_.g.get();
  lg.ln_b = dec_final_.b.get();
  lg.C = logits_.get();
  lg.ldc = Vp_;
  lg.part_m = part_m_.get();
  lg.part_s = part_s_.get();
  lg.part_arg = part_arg_.get();
  lg.part_ld = part_ld_;
  lg.trace = next_trace("gemv logits + partials (+LN)");
  launch_gemv(gp, true, lg, stream_);
  count("gemv logits + softmax partials (+LN)");
}

void Engine::decoder_body(bool reorder) {
  if (small_path()) {
    decoder_body_small(reorder);
    return;
  }
  const ModelConfig& c = host_.config;
  const long long d = d_;
  const int R = r_max_;
  const int* dr = n_rows_.get();
  const float sqrt_d = std::sqrt(static_cast<float>(c.d_model));
  const float scale = 1.0f / std::sqrt(static_cast<float>(d_ / heads_));
  // Decoder rows are their own quantization segments (one hypothesis row per
  // Executor::linear call in decode_step), so LayerNorm and attention write
  // the next GEMM's operand directly.
  const OperandOut od = opout(act_d_);
  trace_slot_ = 0;
  auto tr_od = [&](const char* name) {  // operand writer with a timeline slot (MTG_TRACE)
    OperandOut o = od;
    o.tr = next_trace(name);
    return o;
  };
  auto ln_dec = [&](const LN& ln, float* y = nullptr) {
    const OperandOut o = tr_od("layernorm");
    launch_layernorm(dec_y_.get(), d, R, dr, d_, ln.g.get(), ln.b.get(), y, d, nullptr, &o,
                     stream_);
    count("layernorm");
  };
  // Shortlist decoding reads the final LayerNorm rows themselves (fp32 path).
  float* final_y = use_shortlist_ ? dec_a_.get() : nullptr;
  // Step start: history reorder + target embedding + first LayerNorm fused
  // into one kernel (d_model <= 512), else three kernels.
  // MTG_STEP_FUSION: 0 = three kernels, 1 = reorder + fused embed/LN,
  // 2 = one kernel (A/B switch; default 0: measured fastest with PDL).
  static const int fusion = [] {
    const char* e = std::getenv("MTG_STEP_FUSION");
    return e ? std::atoi(e) : 0;
  }();
  const bool fused = d_ <= 512 && fusion > 0 && !(use_shortlist_ && c.num_decoder_layers == 0);
  static const bool fold_env = [] {
    const char* e = std::getenv("MTG_FOLD_REORDER");
    return !(e && e[0] == '0');
  }();
  const bool fold_reorder = fold_env && !(fused && fusion == 2) && c.num_decoder_layers > 0;
  HistReorder hist;
  if (fold_reorder && reorder) {
    hist.on = 1;
    hist.anc[0] = anc0_.get();
    hist.anc[1] = anc1_.get();
    hist.tok[0] = tok0_.get();
    hist.tok[1] = tok1_.get();
    hist.row_parent = row_parent_.get();
    hist.row_prev = row_prev_.get();
  }
  const LN& ln0 = c.num_decoder_layers > 0 ? dec_[0].n1 : dec_final_;
  if (fused) {
    StepBegin sb{};
    sb.d_rows = dr;
    sb.d_step = step_.get();
    sb.prev = row_prev_.get();
    sb.table = tgt_embed_f32_.get();
    sb.table_q = nullptr;  // int8: tgt_embed_f32_ holds q / scale
    sb.q_scale = tgt_scale_;
    sb.sqrt_d = sqrt_d;
    sb.pe = pe_.get();
    sb.d = d_;
    sb.x = dec_y_.get();
    sb.ldx = d;
    sb.reorder = reorder && fusion == 2 ? 1 : 0;
    if (reorder && fusion != 2 && !fold_reorder) {
      launch_beam_reorder(beam_, stream_);
      count("beam reorder");
    }
    sb.row_parent = row_parent_.get();
    sb.anc[0] = anc0_.get();
    sb.anc[1] = anc1_.get();
    sb.tok[0] = tok0_.get();
    sb.tok[1] = tok1_.get();
    sb.T = T_;
    launch_step_begin(sb, R, ln0.g.get(), ln0.b.get(), od, stream_);
    count(sb.reorder ? "step begin (reorder+embed+LN)" : "step begin (embed+LN)");
  } else {
    // The history reorder runs inside the layer-0 self-attention (before its
    // dependency wait, off the critical path); MTG_FOLD_REORDER=0: own kernel.
    if (reorder && !fold_reorder) {
      BeamDev bd = beam_;
      bd.tr_b = next_trace("beam reorder");
      launch_beam_reorder(bd, stream_);
      count("beam reorder");
    }
    launch_embed_tgt(row_prev_.get(), dr, R, step_.get(), tgt_embed_f32_.get(), nullptr,
                     tgt_scale_, d_, sqrt_d,
                     pe_.get(), dec_y_.get(), d, stream_);
    count("embed_tgt");
    ln_dec(ln0, c.num_decoder_layers == 0 ? final_y : nullptr);
  }
  // Cross-attention per (sentence, head) with the keys staged before the
  // dependency wait (fp32 / bf16; MTG_CROSS_SENT=0: per row, A/B).
  static const bool cross_sent_env = [] {
    const char* e = std::getenv("MTG_CROSS_SENT");
    return !(e && e[0] == '0');
  }();
  const bool cross_sent = cross_sent_env && prec_ != kINT8 &&
                          attn_cross_sent_supported(d_, heads_, std::max(staged_max_src_, 1), beam_.B);
  for (int l = 0; l < c.num_decoder_layers; ++l) {
    DecLayer& L = dec_[l];
    if (l > 0) ln_dec(L.n1);
    cur_tr_ = next_trace("gemm qkv");
    gemm(act_d_, L.self_qkv, R, dr, qkv_cache_[l].get(), 3 * d, nullptr, nullptr, 0,
         static_cast<long long>(R) * 3 * d, step_.get());
    launch_dec_self_attention(qkv_cache_[l].get(), R, T_, anc0_.get(), anc1_.get(), dr,
                              step_.get(), d_, heads_, scale, dec_ctx_.get(), d,
                              tr_od("self attention"), stream_, 1, l == 0 ? hist : HistReorder{});
    count("self attention");
    cur_tr_ = next_trace("gemm wo (+res)");
    gemm(act_d_, L.self_wo, R, dr, dec_y_.get(), d, nullptr, dec_y_.get(), 0);
    ln_dec(L.n2);
    cur_tr_ = next_trace("gemm cross wq");
    gemm(act_d_, L.cross_q, R, dr, dec_cq_.get(), d, nullptr, nullptr, 0);
    if (cross_sent) {
      launch_attn_cross_sent(dec_cq_.get(), d, ckv_[l].get(), enc_off_.get(), enc_len_.get(),
                             sent_row0_.get(), sent_live_.get(), sent_done_.get(), beam_.N,
                             beam_.B, std::max(staged_max_src_, 1), d_, heads_, scale,
                             dec_ctx_.get(), d, tr_od("cross attention (per sentence)"), stream_);
    } else {
      launch_dec_cross_attention(dec_cq_.get(), d, ckv_[l].get(), row_sent_.get(),
                                 enc_off_.get(), enc_len_.get(), dr, R, T_, d_, heads_, scale,
                                 dec_ctx_.get(), d, tr_od("cross attention"), stream_);
    }
    count("cross attention");
    cur_tr_ = next_trace("gemm cross wo (+res)");
    gemm(act_d_, L.cross_wo, R, dr, dec_y_.get(), d, nullptr, dec_y_.get(), 0);
    ln_dec(L.n3);
    cur_tr_ = next_trace("gemm w1 (+b1, relu)");
    static const bool bf16_direct = [] {  // MTG_BF16_DIRECT=0: cast kernel (A/B)
      const char* e = std::getenv("MTG_BF16_DIRECT");
      return !(e && e[0] == '0');
    }();
    if (prec_is_tf32x3(act_ff_.prec)) {  // FFN-up writes the FFN-down operand itself
      gemm(act_d_, L.w1, R, dr, act_ff_.hi.get(), act_ff_.k_pad, L.b1.get(), nullptr, 1, 0,
           nullptr, nullptr, act_ff_.prec == kPrecTF32x3 ? act_ff_.lo.get() : nullptr);
    } else if (bf16_direct && prec_ == kBF16 && act_ff_.k_pad == dff_) {  // ... as bf16
      gemm(act_d_, L.w1, R, dr, reinterpret_cast<float*>(act_ff_.h.get()), act_ff_.k_pad,
           L.b1.get(), nullptr, 1, 0, nullptr, nullptr, nullptr, true);
    } else {
      gemm(act_d_, L.w1, R, dr, ffh_.get(), dff_, L.b1.get(), nullptr, 1);
      prep(ffh_.get(), dff_, dff_, R, dr, nullptr, 0, act_ff_);
    }
    cur_tr_ = next_trace("gemm w2 (+b2, res)");
    gemm(act_ff_, L.w2, R, dr, dec_y_.get(), d, L.b2.get(), dec_y_.get(), 0);
  }
  if (c.num_decoder_layers > 0) {
    OperandOut ol = opout(logits_act());
    ol.tr = next_trace("layernorm (final)");
    launch_layernorm(dec_y_.get(), d, R, dr, d_, dec_final_.g.get(), dec_final_.b.get(), final_y,
                     d, nullptr, &ol, stream_);
    count("layernorm");
  }
  cur_tr_ = next_trace("logits gemm + partials");
  if (!use_shortlist_) gemm_logits(R, dr);  // shortlists project inside their top-k kernel
  cur_tr_ = KTrace{};
}

void Engine::ensure_step_graph() {
  StepKey key;
  key.n = beam_.N;
  key.b = beam_.B;
  key.r_max = r_max_;
  key.gen = ws_gen_;
  key.alpha = beam_.alpha;
  key.shortlist = use_shortlist_;
  key.sl_ids = sl_ids_.get();
  key.sl_off = sl_off_.get();
  key.max_src = staged_max_src_;
  if (step_exec_ && key == step_key_) return;
  if (step_exec_) cudaGraphExecDestroy(step_exec_);
  if (step_graph_) cudaGraphDestroy(step_graph_);
  if (multi_exec_) cudaGraphExecDestroy(multi_exec_);
  if (loop_exec_) cudaGraphExecDestroy(loop_exec_);
  step_exec_ = nullptr;
  step_graph_ = nullptr;
  multi_exec_ = nullptr;
  loop_exec_ = nullptr;
  diag_clear();
  step_kernels_ = capture_steps(1, &step_exec_, &step_graph_);
  if (steps_per_graph() > 1 && !diag_) {
    cudaGraph_t g = nullptr;
    capture_steps(steps_per_graph(), &multi_exec_, &g);
    cudaGraphDestroy(g);
    static const bool device_loop = [] {
      const char* e = std::getenv("MTG_DEVICE_LOOP");
      return !(e && e[0] == '0');
    }();
    if (device_loop) capture_device_loop(steps_per_graph());
  }
  step_key_ = key;
}

// The decode loop as one graph: a while node whose body is k steps plus a
// condition kernel (hypotheses alive and another k steps below loop_end),
// so the host neither polls nor relaunches between chunks.
void Engine::capture_device_loop(int k) {
  loop_end_.resize(1);
  cudaGraph_t g = nullptr;
  MTG_CUDA(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  MTG_CUDA(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp{};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  MTG_CUDA(cudaGraphAddNode(&node, g, nullptr, 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  const int64_t before = launches_;
  MTG_CUDA(cudaStreamBeginCaptureToGraph(stream_, body, nullptr, nullptr, 0,
                                         cudaStreamCaptureModeThreadLocal));
  capturing_ = true;
  try {
    for (int rep = 0; rep < k; ++rep) capture_one_step();
    launch_decode_loop_cond(h, n_rows_.get(), step_.get(), loop_end_.get(), k, stream_);
  } catch (...) {
    capturing_ = false;
    cudaGraph_t tmp = nullptr;
    cudaStreamEndCapture(stream_, &tmp);
    cudaGraphDestroy(g);
    throw;
  }
  capturing_ = false;
  cudaGraph_t captured = nullptr;
  MTG_CUDA(cudaStreamEndCapture(stream_, &captured));
  const cudaError_t err = cudaGraphInstantiate(&loop_exec_, g, 0);
  cudaGraphDestroy(g);
  launches_ = before;
  if (err != cudaSuccess) {  // fall back to host-driven chunks
    cudaGetLastError();
    loop_exec_ = nullptr;
  }
}

int Engine::steps_per_graph() const {
  // Decode steps per graph launch (1, 2, 4 or 8: the host polls for
  // termination every 8 steps).
  static const int k = [] {
    const char* e = std::getenv("MTG_STEPS_PER_GRAPH");
    const int v = e ? std::atoi(e) : 8;  // measured: 8 > 1 by ~1% (PDL across steps)
    return (v == 2 || v == 4 || v == 8) ? v : 1;
  }();
  return k;
}

int64_t Engine::capture_steps(int k, cudaGraphExec_t* exec, cudaGraph_t* graph) {
  const int64_t before = launches_;
  MTG_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
  capturing_ = true;
  try {
    for (int rep = 0; rep < k; ++rep) capture_one_step();
  } catch (...) {
    capturing_ = false;
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(stream_, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  capturing_ = false;
  MTG_CUDA(cudaStreamEndCapture(stream_, graph));
  MTG_CUDA(cudaGraphInstantiate(exec, *graph, 0));
  const int64_t n = launches_ - before;
  launches_ = before;
  return n / k;
}

void Engine::capture_one_step() {
  {
    if (diag_) {
      diag_marks_.push_back({"start", nullptr});
      MTG_CUDA(cudaEventCreate(&diag_marks_.back().ev));
      MTG_CUDA(cudaEventRecordWithFlags(diag_marks_.back().ev, stream_, cudaEventRecordExternal));
    }
    decoder_body(true);
    // Step tail: top-k of every live row + per-sentence selection, fused into
    // one kernel by default (MTG_FUSED_TAIL=0: two kernels, A/B).
    static const bool fused_tail = [] {
      const char* e = std::getenv("MTG_FUSED_TAIL");
      return !(e && e[0] == '0');
    }();
    const int sl_prec = prec_ == kINT8 ? 0 : prec_ == kBF16 ? 1 : 2;
    const ShortlistArgs sla = shortlist_args();
    BeamDev bd = beam_;  // + trace slots of the step tail (MTG_TRACE)
    static const int fused_min_n = [] {  // measured: neutral-to-worse for batch-1
      const char* e = std::getenv("MTG_FUSED_TAIL_MIN_N");
      return e ? std::atoi(e) : 8;
    }();
    if (fused_tail && beam_.N >= fused_min_n) {
      bd.tr_a = next_trace("fused top-k + select");
      launch_topk_select(logits_.get(), Vp_, part_m_.get(), part_s_.get(), part_arg_.get(),
                         part_ld_, use_shortlist_ ? &sla : nullptr, sl_prec, bd, stream_);
      count("top-k + beam select");
    } else {
      bd.tr_a = next_trace("softmax + top-k");
      bd.tr_b = next_trace("beam select");
      if (use_shortlist_) {
        launch_shortlist_topk(sl_prec, sla, bd, stream_);
        count("shortlist logits + softmax + top-k");
      } else {
        launch_softmax_topk(logits_.get(), Vp_, part_m_.get(), part_s_.get(), part_arg_.get(),
                            part_ld_, bd, stream_);
        count("softmax + top-k merge");
      }
      launch_beam_select(bd, stream_);
      count("beam select");
    }
  }
}

void Engine::decode_loop(int t_run) {
  launch_beam_init(beam_, stream_);
  count();
  ensure_step_graph();
  const int k = multi_exec_ ? steps_per_graph() : 1;
  int t0 = 0;
  if (loop_exec_ && t_run >= k) {
    // Device loop over the whole k-step chunks (stops early once every
    // hypothesis is done), then the remaining steps; steps after completion
    // are no-ops (no live rows).
    const int t_loop = t_run / k * k;
    loop_end_.upload(&t_loop, 1, stream_);
    MTG_CUDA(cudaGraphLaunch(loop_exec_, stream_));
    launches_ += static_cast<int64_t>(t_loop) * step_kernels_ + t_loop / k;  // + conditions
    for (int t = t_loop; t < t_run; ++t) {
      MTG_CUDA(cudaGraphLaunch(step_exec_, stream_));
      launches_ += step_kernels_;
    }
    return;
  }
  for (int t = t0; t < t_run; ++t) {
    if (k > 1 && t % k == 0 && t + k <= t_run) {
      MTG_CUDA(cudaGraphLaunch(multi_exec_, stream_));
      launches_ += k * step_kernels_;
      t += k - 1;
    } else {
      MTG_CUDA(cudaGraphLaunch(step_exec_, stream_));
      launches_ += step_kernels_;
    }
    if (diag_) {
      MTG_CUDA(cudaStreamSynchronize(stream_));
      diag_ms_.resize(diag_marks_.size(), 0.0);
      for (size_t i = 1; i < diag_marks_.size(); ++i) {
        float ms = 0.0f;
        MTG_CUDA(cudaEventElapsedTime(&ms, diag_marks_[i - 1].ev, diag_marks_[i].ev));
        diag_ms_[i] += ms;
      }
      ++diag_steps_;
    }
    if ((t + 1) % 8 == 0 && t + 1 < t_run) {
      MTG_CUDA(cudaMemcpyAsync(h_pinned_, n_rows_.get(), sizeof(int), cudaMemcpyDeviceToHost,
                               stream_));
      MTG_CUDA(cudaStreamSynchronize(stream_));
      if (*h_pinned_ == 0) break;
    }
  }
}

// ============================================================================
// public entry points
// ============================================================================

std::vector<SentenceResult> Engine::translate_batch(const std::vector<std::vector<int>>& srcs,
                                                    const BeamConfigC& cfg,
                                                    const FactorStreams* factors,
                                                    const std::vector<std::vector<int>>* shortlists) {
  DeviceGuard guard(device_);
  stage(srcs, factors, shortlists);
  run_staged(cfg);
  const int n = staged_n_;
  std::vector<SentenceResult> out(n);
  if (n == 0) return out;
  // All results in one pinned staging area: the copies queue behind the
  // decode loop and the host waits once.
  const size_t nt = size_t(n) * T_;
  const size_t words = 5 * size_t(n) + nt + 1;
  if (words > res_host_words_) {
    if (res_host_) cudaFreeHost(res_host_);
    res_host_ = nullptr;
    MTG_CUDA(cudaMallocHost(&res_host_, words * sizeof(int)));
    res_host_words_ = words;
  }
  int* const len = res_host_;
  int* const status = len + n;
  float* const lp = reinterpret_cast<float*>(status + n);
  float* const norm = lp + n;
  unsigned* const flags = reinterpret_cast<unsigned*>(norm + n);
  int* const tok = reinterpret_cast<int*>(flags + n);
  int* const badp = tok + nt;
  auto d2h = [&](void* dst, const void* src, size_t bytes) {
    MTG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, stream_));
  };
  d2h(len, res_len_.get(), n * sizeof(int));
  d2h(status, res_status_.get(), n * sizeof(int));
  d2h(lp, res_lp_.get(), n * sizeof(float));
  d2h(norm, res_norm_.get(), n * sizeof(float));
  d2h(flags, res_flags_.get(), n * sizeof(unsigned));
  d2h(tok, res_tok_.get(), nt * sizeof(int));
  d2h(badp, nonfinite_.get(), sizeof(int));
  MTG_CUDA(cudaStreamSynchronize(stream_));
  const int bad = *badp;
  for (int s = 0; s < n; ++s) {
    SentenceResult& r = out[s];
    if (staged_status_[s]) {
      r.status = staged_status_[s];
      r.flags = 4u;
      continue;
    }
    r.status = bad ? kValueError : status[s];
    r.flags = bad ? 4u : flags[s];
    if (r.status) continue;
    r.tokens.assign(tok + size_t(s) * T_, tok + size_t(s) * T_ + len[s]);
    r.logprob = lp[s];
    r.norm = norm[s];
  }
  if (bad && n > 1) {
    // A non-finite quantize input (quant.cpp:110-112) fails only the sentence
    // it came from (translate_corpus, decode.cpp:403-410). The device flag is
    // per batch, so the batch's sentences are re-decoded one by one: their
    // results do not depend on the batch composition (every quantization
    // segment is a sentence or one of its rows).
    const std::vector<int> status0 = staged_status_;
    for (int s = 0; s < n; ++s) {
      if (status0[s]) continue;
      FactorStreams fs1;
      if (factors) fs1.push_back((*factors)[s]);
      std::vector<std::vector<int>> sl1;
      if (shortlists) sl1.push_back((*shortlists)[s]);
      out[s] = translate_batch({srcs[s]}, cfg, factors ? &fs1 : nullptr,
                               shortlists ? &sl1 : nullptr)[0];
    }
  }
  return out;
}

void Engine::stage(const std::vector<std::vector<int>>& srcs, const FactorStreams* factors,
                   const std::vector<std::vector<int>>* shortlists) {
  DeviceGuard guard(device_);
  const int n = static_cast<int>(srcs.size());
  if (factors && static_cast<int>(factors->size()) != n)
    fail(kShapeError, "factor streams: one entry per sentence");
  staged_factors_ = factors ? *factors : FactorStreams{};
  // Shortlists (decode.cpp:344-349): all or none of a device batch; ids must
  // be valid target rows (IndexError, model.cpp:446) in increasing order.
  use_shortlist_ = false;
  sl_status_.clear();
  if (shortlists) {
    if (static_cast<int>(shortlists->size()) != n) fail(kShapeError, "one shortlist per sentence");
    std::vector<int> ids, off(n + 1, 0);
    sl_status_.assign(n, 0);
    for (int s = 0; s < n; ++s) {
      const auto& l = (*shortlists)[s];
      if (l.empty()) fail(kStateError, "shortlist batch mixes sentences without a shortlist");
      // Per-sentence failures (the reference throws from the first
      // decode_step, after source validation).
      if (static_cast<int>(l.size()) > kMaxShortlist) sl_status_[s] = kUsageError;
      for (size_t j = 0; j < l.size() && !sl_status_[s]; ++j) {
        if (l[j] < 0 || l[j] >= V_) sl_status_[s] = kIndexError;  // model.cpp:446
        else if (j > 0 && l[j] <= l[j - 1]) sl_status_[s] = kUsageError;  // must be sorted
      }
      if (!sl_status_[s]) ids.insert(ids.end(), l.begin(), l.end());
      off[s + 1] = static_cast<int>(ids.size());
    }
    sl_ids_.resize(std::max<size_t>(ids.size(), 1));
    sl_off_.resize(n + 1);
    sl_ids_.upload(ids.data(), ids.size(), stream_);
    sl_off_.upload(off.data(), n + 1, stream_);
    MTG_CUDA(cudaStreamSynchronize(stream_));
    use_shortlist_ = true;
  }
  int m = 0, max_src = 0;
  for (const auto& s : srcs) {
    if (static_cast<int>(s.size()) <= host_.config.max_seq_len) m += static_cast<int>(s.size());
    max_src = std::max(max_src, static_cast<int>(s.size()));
  }
  ensure_workspace(n, m, std::max(cap_beam_, 1));
  staged_ = srcs;
  staged_n_ = n;
  staged_m_ = stage_sources(srcs, staged_status_);
  staged_max_src_ = std::min(max_src, host_.config.max_seq_len);
}

void Engine::run_staged(const BeamConfigC& cfg) {
  DeviceGuard guard(device_);
  if (cfg.beam_size < 1) fail(kUsageError, "beam_search: beam size >= 1");
  if (cfg.beam_size > kMaxBeam)
    fail(kUsageError, "beam size above " + std::to_string(kMaxBeam) + " is not supported");
  const int n = staged_n_;
  if (n == 0) return;
  if (cfg.beam_size > cap_beam_) {
    ensure_workspace(n, staged_m_, cfg.beam_size);
    stage_sources(staged_, staged_status_);
  }
  launches_ = 0;
  const ModelConfig& c = host_.config;
  std::vector<int> maxlen(n, 0), done(n, 0), zero(n, 0);
  int t_run = 0;
  for (int s = 0; s < n; ++s) {
    done[s] = staged_status_[s] != 0;
    if (done[s]) continue;
    const int sl = static_cast<int>(staged_[s].size());
    maxlen[s] = cfg.max_len > 0 ? cfg.max_len : std::min(c.max_seq_len, sl * 2 + 5);
    t_run = std::max(t_run, std::min(maxlen[s], c.max_seq_len));
  }
  sent_maxlen_.upload(maxlen.data(), n, stream_);
  sent_done_.upload(done.data(), n, stream_);
  res_status_.upload(zero.data(), n, stream_);
  MTG_CUDA(cudaMemsetAsync(nonfinite_.get(), 0, sizeof(int), stream_));
  beam_.N = n;
  beam_.B = cfg.beam_size;
  beam_.alpha = cfg.alpha;
  trace_reset();
  run_encoder(n, staged_m_, staged_max_src_);
  if (t_run > 0) decode_loop(t_run);
  last_launches_ = launches_;
  last_beam_ = cfg.beam_size;
  last_t_run_ = t_run;
}

void Engine::time_kernel(int kernel, int iters, float* ms, double* bytes, double* flops) {
  DeviceGuard guard(device_);
  if (staged_n_ == 0 || last_beam_ == 0)
    fail(kStateError, "time_kernel: stage a batch and run it once first");
  if (iters < 1) fail(kUsageError, "time_kernel: iters >= 1");
  const ModelConfig& c = host_.config;
  const int R = staged_n_ * last_beam_;
  const int eb = prec_elem_bytes(gemm_prec_of(prec_));
  const int split = prec_ == kF32 ? 2 : 1;  // hi + lo operands
  scratch_rows_.resize(1);
  scratch_rows_.upload(&R, 1, stream_);
  cudaEvent_t e0, e1;
  MTG_CUDA(cudaEventCreate(&e0));
  MTG_CUDA(cudaEventCreate(&e1));
  std::function<void()> launch;
  if (kernel == 0) {  // decoder output projection (tied tgt_embed)
    launch = [&] {
      gemm_logits(r_max_, scratch_rows_.get());
    };
    *bytes = double(split) * eb * (double(V_) * logits_w_.k_pad + double(R) * act_d_.k_pad) +
             4.0 * R * V_;
    *flops = 2.0 * R * V_ * d_ * (prec_ == kF32 ? 3 : 1);
  } else if (kernel == 1) {  // log-softmax + top-k over R x V logits
    n_rows_.upload(&R, 1, stream_);
    launch = [&] {
      launch_softmax_topk(logits_.get(), Vp_, part_m_.get(), part_s_.get(), part_arg_.get(),
                          part_ld_, beam_, stream_);
    };
    *bytes = 12.0 * R * ((V_ + 31) / 32) + 4.0 * R * 32 * last_beam_;
    *flops = 0.0;
  } else if (kernel == 2) {  // decoder self-attention at the last step
    if (c.num_decoder_layers == 0) fail(kStateError, "no decoder layers");
    const int t = std::max(0, last_t_run_ - 1);
    n_rows_.upload(&R, 1, stream_);
    step_.upload(&t, 1, stream_);
    const float scale = 1.0f / std::sqrt(static_cast<float>(d_ / heads_));
    launch = [&, scale] {
      launch_dec_self_attention(qkv_cache_[0].get(), r_max_, T_, anc0_.get(), anc1_.get(),
                                n_rows_.get(), step_.get(), d_, heads_, scale, dec_ctx_.get(), d_,
                                opout(act_d_), stream_);
    };
    *bytes = 4.0 * R * (double(t + 1) * 2 * d_ + 2.0 * d_);
    *flops = 4.0 * R * (t + 1) * d_;
  } else if (kernel == 3) {  // encoder FFN w1 GEMM
    if (c.num_encoder_layers == 0) fail(kStateError, "no encoder layers");
    const int M = staged_m_;
    launch = [&, M] {
      gemm(act_d_, enc_[0].w1, M, nullptr, ffh_.get(), dff_, enc_[0].b1.get(), nullptr, 1);
    };
    *bytes = double(split) * eb * (double(dff_) * enc_[0].w1.k_pad + double(M) * act_d_.k_pad) +
             4.0 * M * dff_;
    *flops = 2.0 * M * dff_ * d_ * (prec_ == kF32 ? 3 : 1);
  } else if (kernel >= 10 && kernel <= 17) {
    // Small-batch step pieces, each chained `iters` times inside one CUDA
    // graph with PDL (the in-graph cost of one dependent launch).
    if (!small_path()) fail(kStateError, "time_kernel: the staged batch does not use the GEMV step");
    const int t = std::max(0, last_t_run_ - 1);
    n_rows_.upload(&R, 1, stream_);
    step_.upload(&t, 1, stream_);
    const int gp = prec_ == kINT8 ? 0 : prec_ == kBF16 ? 1 : 2;
    const long long d = d_;
    const float scale = 1.0f / std::sqrt(static_cast<float>(d_ / heads_));
    OperandOut none;
    none.prec = -1;
    DecLayer& L = dec_.at(0);
    std::function<void()> one;
    if (kernel == 10) {  // empty dependent kernel: the launch / PDL floor
      one = [&] { launch_noop(stream_); };
      *bytes = 0.0;
    } else if (kernel == 11) {  // Wo GEMV + residual
      one = [&] {
        GemvArgs o = gemv_args(L.self_wo);
        o.x = dec_ctx_.get();
        o.ldx = d;
        o.C = dec_y_.get();
        o.ldc = d;
        o.residual = dec_y_.get();
        o.ldr = d;
        launch_gemv(gp, false, o, stream_);
      };
      *bytes = double(L.self_wo.n) * L.self_wo.k_pad * prec_elem_bytes(gemm_prec_of(prec_));
    } else if (kernel == 12) {  // LayerNorm + W1 GEMV + bias + ReLU
      one = [&] {
        GemvArgs f1 = gemv_args(L.w1);
        f1.a_mode = 1;
        f1.x = dec_y_.get();
        f1.ldx = d;
        f1.ln_g = L.n3.g.get();
        f1.ln_b = L.n3.b.get();
        f1.C = ffh_.get();
        f1.ldc = dff_;
        f1.bias = L.b1.get();
        f1.relu = 1;
        launch_gemv(gp, false, f1, stream_);
      };
      *bytes = double(L.w1.n) * L.w1.k_pad * prec_elem_bytes(gemm_prec_of(prec_));
    } else if (kernel == 13) {  // final LayerNorm + output projection + partials
      one = [&] {
        GemvArgs lg = gemv_args(logits_w_);
        lg.a_mode = 1;
        lg.x = dec_y_.get();
        lg.ldx = d;
        lg.ln_g = dec_final_.g.get();
        lg.ln_b = dec_final_.b.get();
        lg.C = logits_.get();
        lg.ldc = Vp_;
        lg.part_m = part_m_.get();
        lg.part_s = part_s_.get();
        lg.part_arg = part_arg_.get();
        lg.part_ld = part_ld_;
        launch_gemv(gp, true, lg, stream_);
      };
      *bytes = double(logits_w_.n) * logits_w_.k_pad * prec_elem_bytes(gemm_prec_of(prec_));
    } else if (kernel == 14) {  // decoder self-attention at the last step
      one = [&, scale] {
        launch_dec_self_attention(qkv_cache_[0].get(), r_max_, T_, anc0_.get(), anc1_.get(),
                                  n_rows_.get(), step_.get(), d_, heads_, scale, dec_ctx_.get(),
                                  d_, none, stream_);
      };
      *bytes = 4.0 * R * (double(t + 1) * 2 * d_);
    } else if (kernel == 16) {  // small-batch self-attention (attn_small.cu)
      one = [&, scale] {
        launch_attn_small_self(qkv_cache_[0].get(), r_max_, T_, anc0_.get(), anc1_.get(),
                               row_parent_.get(), 1, tok0_.get(), tok1_.get(), row_prev_.get(), 0,
                               n_rows_.get(), step_.get(),
                               std::min(r_max_, kGemvRows), d_, heads_, scale, dec_ctx_.get(), d_,
                               stream_);
      };
      *bytes = 4.0 * R * (double(t + 1) * 2 * d_);
    } else if (kernel == 17) {  // small-batch cross-attention
      one = [&, scale] {
        launch_attn_small_cross(dec_cq_.get(), d_, ckv_[0].get(), row_sent_.get(), enc_off_.get(),
                                enc_len_.get(), n_rows_.get(), std::min(r_max_, kGemvRows), T_, d_,
                                heads_, scale, dec_ctx_.get(), d_, stream_);
      };
      *bytes = 4.0 * R * (double(staged_max_src_) * 2 * d_);
    } else {  // log-softmax / top-k merge over the live rows
      one = [&] {
        launch_softmax_topk(logits_.get(), Vp_, part_m_.get(), part_s_.get(), part_arg_.get(),
                            part_ld_, beam_, stream_);
      };
      *bytes = 12.0 * R * ((V_ + 31) / 32);
    }
    *flops = 0.0;
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    MTG_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < iters; ++i) one();
    MTG_CUDA(cudaStreamEndCapture(stream_, &g));
    MTG_CUDA(cudaGraphInstantiate(&ge, g, 0));
    cudaGraphDestroy(g);
    launch = [&] { MTG_CUDA(cudaGraphLaunch(ge, stream_)); };
    launch();  // warm
    MTG_CUDA(cudaEventRecord(e0, stream_));
    launch();
    MTG_CUDA(cudaEventRecord(e1, stream_));
    MTG_CUDA(cudaEventSynchronize(e1));
    float total = 0.0f;
    MTG_CUDA(cudaEventElapsedTime(&total, e0, e1));
    *ms = total / iters;
    cudaGraphExecDestroy(ge);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return;
  } else {
    fail(kUsageError, "time_kernel: unknown kernel id");
  }
  launch();  // warm
  MTG_CUDA(cudaEventRecord(e0, stream_));
  for (int i = 0; i < iters; ++i) launch();
  MTG_CUDA(cudaEventRecord(e1, stream_));
  MTG_CUDA(cudaEventSynchronize(e1));
  float total = 0.0f;
  MTG_CUDA(cudaEventElapsedTime(&total, e0, e1));
  *ms = total / iters;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
}

void Engine::forced_logits(const std::vector<std::vector<int>>& srcs, const int* forced, int nf,
                           float* out, const FactorStreams* factors) {
  DeviceGuard guard(device_);
  const int n = static_cast<int>(srcs.size());
  if (n == 0 || nf <= 0) return;
  stage(srcs, factors);
  for (int s = 0; s < n; ++s)
    if (staged_status_[s]) fail(static_cast<Status>(staged_status_[s]), "bad source sentence");
  if (nf > host_.config.max_seq_len) fail(kValueError, "decode_step: past max_seq_len");
  launches_ = 0;
  MTG_CUDA(cudaMemsetAsync(nonfinite_.get(), 0, sizeof(int), stream_));
  std::vector<int> done(n, 0);
  sent_done_.upload(done.data(), n, stream_);
  beam_.N = n;
  beam_.B = 1;
  run_encoder(n, staged_m_, staged_max_src_);
  launch_beam_init(beam_, stream_);
  // One hypothesis per sentence: row r = sentence r, ancestors all r.
  std::vector<int> anc(size_t(r_max_) * T_);
  for (int r = 0; r < r_max_; ++r)
    for (int j = 0; j < T_; ++j) anc[size_t(r) * T_ + j] = r;
  anc0_.upload(anc.data(), anc.size(), stream_);
  anc1_.upload(anc.data(), anc.size(), stream_);
  std::vector<float> rows(size_t(n) * Vp_);
  std::vector<int> prev(n);
  for (int t = 0; t < nf; ++t) {
    decoder_body(false);
    MTG_CUDA(cudaStreamSynchronize(stream_));
    logits_.download(rows.data(), rows.size(), stream_);
    for (int s = 0; s < n; ++s)
      std::copy(rows.begin() + size_t(s) * Vp_, rows.begin() + size_t(s) * Vp_ + V_,
                out + (size_t(s) * nf + t) * V_);
    for (int s = 0; s < n; ++s) prev[s] = forced[t];
    row_prev_.upload(prev.data(), n, stream_);
    const int next = t + 1;
    step_.upload(&next, 1, stream_);
  }
  int bad = 0;
  nonfinite_.download(&bad, 1, stream_);
  if (bad) fail(kValueError, "quantize: non-finite values in tensor");
  last_launches_ = launches_;
}

void Engine::encode(const std::vector<std::vector<int>>& srcs, float* out,
                    const FactorStreams* factors) {
  DeviceGuard guard(device_);
  const int n = static_cast<int>(srcs.size());
  if (n == 0) return;
  stage(srcs, factors);
  for (int s = 0; s < n; ++s)
    if (staged_status_[s]) fail(static_cast<Status>(staged_status_[s]), "bad source sentence");
  MTG_CUDA(cudaMemsetAsync(nonfinite_.get(), 0, sizeof(int), stream_));
  run_encoder(n, staged_m_, staged_max_src_);
  MTG_CUDA(cudaStreamSynchronize(stream_));
  const float* src = host_.config.num_encoder_layers > 0 ? enc_a_.get() : enc_x_.get();
  MTG_CUDA(cudaMemcpy(out, src, sizeof(float) * size_t(staged_m_) * d_, cudaMemcpyDeviceToHost));
}

}  // namespace mtg
