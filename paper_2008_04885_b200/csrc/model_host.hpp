// Host-side model description: ModelConfig (model.hpp:21-60), the parameter
// layout (model.cpp:174-219), seeded init (model.cpp:229-238), the SQNT
// container (io.hpp/io.cpp) and int8 quantization of weights
// (model.cpp:676-681, 733-748). Weights live here only until they are laid
// out on the device (engine.cu).
#pragma once

#include <cstdint>
#include <map>
#include <string>
#include <vector>

namespace mtg {

constexpr float kLayerNormEps = 1e-5f;  // model.hpp:14
constexpr int kPadId = 0, kUnkId = 1, kBosId = 2, kEosId = 3;  // model.hpp:16-19

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

struct HostTensor {
  std::vector<int64_t> shape;
  std::vector<float> f32;   // dtype 0
  std::vector<int8_t> q;    // dtype 1
  float scale = 1.0f;       // int8 only
  bool is_int8 = false;
  int64_t rows() const { return shape.size() == 2 ? shape[0] : 1; }
  int64_t cols() const { return shape.size() == 2 ? shape[1] : (shape.size() == 1 ? shape[0] : 0); }
  int64_t numel() const;
};

struct HostModel {
  ModelConfig config;
  std::map<std::string, HostTensor> params;
  bool quantized = false;  // weights hold int8 copies (file or on-load quantization)
  const HostTensor& at(const std::string& name) const;
};

std::vector<std::pair<std::string, std::vector<int64_t>>> param_shapes(const ModelConfig& c);
std::vector<float> make_pos_enc(int max_len, int d);
bool is_quantized_param(const std::string& name);

HostModel make_random_model(const ModelConfig& c, uint64_t seed);
HostModel load_sqnt(const std::string& path);
void save_sqnt(const HostModel& m, const std::string& path);
// quantize_model (model.cpp:733-748): every is_quantized_param tensor gets an
// int8 copy with one max-abs scale; f32 copies are kept for lookups.
void quantize_weights(HostModel& m);

}  // namespace mtg
