// TEST INFRASTRUCTURE (oracle) -- not product code.
//
// CPU restatement of the reference ("minimt", /root/reference/proj) inference
// hot path: model config + parameter layout + seeded init, SQNT container,
// int8 quantization, f32/int8 executors, encoder, incremental decoder and
// beam search. Each function cites the reference file:line it restates.
//
// The reference cannot be built in this image (Eigen3 at /usr/include/eigen3
// and vendor/ are absent; proj/CMakeLists.txt:5,23-25), so it cannot be run
// as an oracle. Its fp32 reduction orders live in Eigen expression templates
// and are unpinned. This restatement pins every float reduction to the order
// the GPU kernels use (documented per function below), which
// makes the int8 path bit-exact end to end and the fp32 path exact apart from
// the GEMM accumulation (tensor cores). Parity of this oracle with the
// reference is pinned by the reference's own known-answer tests and
// properties (tests/test_oracle_kats.py cites each one).
#pragma once

#include <cstdint>
#include <functional>
#include <map>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace orc {

using Index = long long;

constexpr float kLayerNormEps = 1e-5f;  // model.hpp:14
constexpr int kPadId = 0, kUnkId = 1, kBosId = 2, kEosId = 3;  // model.hpp:16-19

// errors.hpp:8-34, numbered like include/minimt_gpu.h.
enum ErrCode { kShape = 1, kValue = 2, kIndex = 3, kState = 4, kFormat = 5, kUsage = 6, kIo = 7 };
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void fail(int code, const std::string& msg);

// ---- config (model.hpp:21-60, model.cpp:37-172) -----------------------------

enum class FactorCombine { kConcat, kSum, kAverage };

struct SourceFactorConfig {
  int factor_vocab_size = 0;
  int embed_dim = 0;
  FactorCombine combine = FactorCombine::kSum;
  bool share_with_word_embedding = false;
};

struct ModelConfig {
  int num_encoder_layers = 6;
  int num_decoder_layers = 6;
  int d_model = 32;
  int d_ff = 128;
  int num_heads = 4;
  int src_vocab_size = 0;
  int tgt_vocab_size = 0;
  std::vector<SourceFactorConfig> factor_configs;
  float dropout = 0.1f;
  int max_seq_len = 128;

  int word_embed_dim() const;
  void validate() const;
  std::string to_json() const;
  static ModelConfig from_json(const std::string& json);
};

// ---- tensors -----------------------------------------------------------------

struct Tensor {
  std::vector<Index> shape;
  std::vector<float> data;
  Tensor() = default;
  explicit Tensor(std::vector<Index> s);
  Index rank() const { return static_cast<Index>(shape.size()); }
  Index rows() const { return rank() == 2 ? shape[0] : 1; }
  Index cols() const { return rank() == 2 ? shape[1] : (rank() == 1 ? shape[0] : 0); }
  Index numel() const { return static_cast<Index>(data.size()); }
  float* row(Index r) { return data.data() + r * cols(); }
  const float* row(Index r) const { return data.data() + r * cols(); }
};

// quant.hpp:13-40
struct QTensor {
  std::vector<Index> shape;
  std::vector<int8_t> q;
  float scale = 1.0f;
  std::vector<int32_t> row_sums;
  Index rows() const { return shape.size() == 2 ? shape[0] : 1; }
  Index cols() const { return shape.size() == 2 ? shape[1] : (shape.size() == 1 ? shape[0] : 0); }
  Index numel() const { return static_cast<Index>(q.size()); }
  void finish();
};

// ---- model (model.hpp:62-90, model.cpp:174-260) --------------------------------

struct Model {
  ModelConfig config;
  std::map<std::string, Tensor> params;
  std::vector<float> pe;  // [max_seq_len x d_model], make_pos_enc model.cpp:13-22
  const Tensor& param(const std::string& name) const;
  Tensor& param(const std::string& name);
  size_t param_count() const;
};

std::vector<std::pair<std::string, std::vector<Index>>> param_shapes(const ModelConfig& c);
std::vector<float> make_pos_enc(int max_len, int d);
Model make_model(const ModelConfig& c);  // zero params + PE
void init_params(Model& m, uint64_t seed);  // model.cpp:229-238 with Rng(seed)

struct QModel {  // model.hpp:150-155
  ModelConfig config;
  std::map<std::string, Tensor> f32;
  std::map<std::string, QTensor> q;
  std::vector<float> pe;
};
bool is_quantized_param(const std::string& name);  // model.cpp:676-681
QModel quantize_model(const Model& m);             // model.cpp:733-748

// ---- SQNT container (io.hpp, io.cpp) -------------------------------------------

struct ParamRecord {
  std::string name;
  uint8_t dtype = 0;
  std::vector<uint32_t> dims;
  float scale = 0.0f;
  std::vector<uint8_t> payload;
  size_t numel() const;
};
struct ParamFile {
  std::string config_json;
  std::vector<ParamRecord> params;
  const ParamRecord* find(const std::string& name) const;
};
void write_param_file(const std::string& path, const ParamFile& f);
ParamFile read_param_file(const std::string& path);
void save_params(const Model& m, const std::string& path);         // model.cpp:699-712
Model load_params(const std::string& path);                        // model.cpp:714-731
void save_quantized(const QModel& m, const std::string& path);     // model.cpp:750-773
QModel load_quantized(const std::string& path);                    // model.cpp:775-803

// ---- quantization (quant.cpp:108-239) -------------------------------------------

QTensor quantize(const float* x, std::vector<Index> shape);
QTensor quantize(const Tensor& x);
// c[m x n] = int32 sum a*b * (1/(sa*sb)); b is [k x n] (qmatmul) or [n x k] (nt).
void qmatmul(const QTensor& a, const QTensor& b, float* c);
void qmatmul_nt(const QTensor& a, const QTensor& b, const std::vector<int>* rows, float* c);

// ---- executors (model.hpp:113-171, model.cpp:422-497) ---------------------------

class Executor {
 public:
  virtual ~Executor() = default;
  virtual const ModelConfig& config() const = 0;
  virtual Tensor linear(const Tensor& x, const std::string& name) const = 0;
  virtual Tensor project_logits(const Tensor& x, const std::vector<int>* rows) const = 0;
  virtual Tensor embed_rows(const std::string& table, const std::vector<int>& ids) const = 0;
  virtual const Tensor& f32_param(const std::string& name) const = 0;
  virtual const std::vector<float>& pos_enc() const = 0;
};

class F32Executor final : public Executor {
 public:
  explicit F32Executor(const Model& m) : m_(&m) {}
  const ModelConfig& config() const override { return m_->config; }
  Tensor linear(const Tensor& x, const std::string& name) const override;
  Tensor project_logits(const Tensor& x, const std::vector<int>* rows) const override;
  Tensor embed_rows(const std::string& table, const std::vector<int>& ids) const override;
  const Tensor& f32_param(const std::string& name) const override { return m_->param(name); }
  const std::vector<float>& pos_enc() const override { return m_->pe; }

 private:
  const Model* m_;
};

class Int8Executor final : public Executor {
 public:
  explicit Int8Executor(const QModel& m);
  const ModelConfig& config() const override { return m_->config; }
  Tensor linear(const Tensor& x, const std::string& name) const override;
  Tensor project_logits(const Tensor& x, const std::vector<int>* rows) const override;
  Tensor embed_rows(const std::string& table, const std::vector<int>& ids) const override;
  const Tensor& f32_param(const std::string& name) const override;
  const std::vector<float>& pos_enc() const override { return m_->pe; }

 private:
  const QModel* m_;
  // Weights pre-transposed to [n x k] so the m = 1 GEMV streams rows.
  std::map<std::string, QTensor> wt_;
};

// ---- inference forward (model.cpp:499-672) ---------------------------------------

Tensor layer_norm(const Tensor& x, const Tensor& g, const Tensor& b, float eps);
Tensor embed_source_infer(const Executor& ex, const std::vector<int>& ids,
                          const std::vector<std::vector<int>>& factor_ids);
Tensor encode_infer(const Executor& ex, const Tensor& src_embedded);

struct DecoderState {  // model.hpp:180-185
  const Executor* exec = nullptr;
  std::vector<std::vector<float>> self_k, self_v;  // per layer, rows of d
  std::vector<Tensor> cross_k, cross_v;
  int pos = 0;
};
DecoderState init_decoder(const Executor& ex, const Tensor& enc_out);
Tensor decode_step(DecoderState& st, int prev_token, const std::vector<int>* shortlist);

// Teacher-forced logits through the full causal decoder (model.cpp:382-418),
// computed with the same pinned ops (f32 model only).
Tensor forward_teacher_forced(const Model& m, const std::vector<int>& src,
                              const std::vector<std::vector<int>>& factors,
                              const std::vector<int>& tgt);

// ---- search (decode.hpp:15-38, decode.cpp:18-109) ---------------------------------

struct Hypothesis {
  std::vector<int> tokens;
  float logprob = 0.0f;
  bool finished = false;
  bool truncated = false;
  DecoderState state;
  float normalized_score(float alpha) const;
};

struct BeamConfig {
  int beam_size = 4;
  int max_len = 64;
  float length_penalty_alpha = 1.0f;
};

// log-softmax of one logits row in the GPU's 1024-thread reduction order.
std::vector<float> log_softmax_row(const float* x, int n);

Hypothesis beam_search(const Executor& ex, const std::vector<int>& src_ids,
                       const std::vector<std::vector<int>>& factor_ids,
                       const BeamConfig& cfg, const std::vector<int>* shortlist);

// translate_one length rules on ids (decode.cpp:326-356): append EOS, truncate
// to max_seq_len keeping EOS, derive max_len when <= 0.
std::vector<int> prepare_source(const std::vector<int>& word_ids, int max_seq_len);
int derive_max_len(const BeamConfig& cfg, int src_len, int max_seq_len);

// eval.cpp:120-128 nearest-rank percentile.
double percentile(std::vector<double> v, double p);

}  // namespace orc
