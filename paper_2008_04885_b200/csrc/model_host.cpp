#include "model_host.hpp"

#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstring>
#include <fstream>
#include <iterator>
#include <random>

#include "errors.hpp"

namespace mtg {

// ---- tiny JSON reader for ModelConfig (the reference uses nlohmann/json) ----
namespace {

struct JVal {
  enum T { Null, Bool, Num, Str, Arr, Obj } t = Null;
  double num = 0;
  bool b = false;
  std::string s;
  std::vector<JVal> arr;
  std::vector<std::pair<std::string, JVal>> obj;
  const JVal* get(const char* k) const {
    for (auto& kv : obj)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
};

class JsonReader {
 public:
  explicit JsonReader(const std::string& s) : s_(s) {}
  JVal value() {
    skip();
    if (i_ >= s_.size()) bad();
    const char c = s_[i_];
    if (c == '{') return object();
    if (c == '[') return array();
    if (c == '"') {
      JVal v;
      v.t = JVal::Str;
      v.s = string();
      return v;
    }
    if (lit("true")) return boolean(true);
    if (lit("false")) return boolean(false);
    if (lit("null")) return JVal{};
    return number();
  }

 private:
  [[noreturn]] void bad() { fail(kFormatError, "bad model config JSON"); }
  void skip() {
    while (i_ < s_.size() && std::isspace(static_cast<unsigned char>(s_[i_]))) ++i_;
  }
  bool lit(const char* w) {
    const size_t n = std::strlen(w);
    if (s_.compare(i_, n, w) == 0) {
      i_ += n;
      return true;
    }
    return false;
  }
  static JVal boolean(bool b) {
    JVal v;
    v.t = JVal::Bool;
    v.b = b;
    return v;
  }
  std::string string() {
    ++i_;  // opening quote
    std::string out;
    while (i_ < s_.size() && s_[i_] != '"') {
      if (s_[i_] == '\\' && i_ + 1 < s_.size()) ++i_;
      out += s_[i_++];
    }
    if (i_ >= s_.size()) bad();
    ++i_;
    return out;
  }
  JVal number() {
    size_t j = i_;
    while (j < s_.size() && (std::isdigit(static_cast<unsigned char>(s_[j])) || s_[j] == '-' ||
                             s_[j] == '+' || s_[j] == '.' || s_[j] == 'e' || s_[j] == 'E'))
      ++j;
    if (j == i_) bad();
    JVal v;
    v.t = JVal::Num;
    v.num = std::strtod(s_.substr(i_, j - i_).c_str(), nullptr);
    i_ = j;
    return v;
  }
  JVal array() {
    JVal v;
    v.t = JVal::Arr;
    ++i_;
    skip();
    if (i_ < s_.size() && s_[i_] == ']') {
      ++i_;
      return v;
    }
    for (;;) {
      v.arr.push_back(value());
      skip();
      if (i_ < s_.size() && s_[i_] == ',') {
        ++i_;
        continue;
      }
      if (i_ < s_.size() && s_[i_] == ']') {
        ++i_;
        return v;
      }
      bad();
    }
  }
  JVal object() {
    JVal v;
    v.t = JVal::Obj;
    ++i_;
    skip();
    if (i_ < s_.size() && s_[i_] == '}') {
      ++i_;
      return v;
    }
    for (;;) {
      skip();
      if (i_ >= s_.size() || s_[i_] != '"') bad();
      std::string k = string();
      skip();
      if (i_ >= s_.size() || s_[i_] != ':') bad();
      ++i_;
      v.obj.emplace_back(std::move(k), value());
      skip();
      if (i_ < s_.size() && s_[i_] == ',') {
        ++i_;
        continue;
      }
      if (i_ < s_.size() && s_[i_] == '}') {
        ++i_;
        return v;
      }
      bad();
    }
  }
  const std::string& s_;
  size_t i_ = 0;
};

int jint(const JVal& o, const char* k, int dflt) {
  const JVal* v = o.get(k);
  if (!v || v->t == JVal::Null) return dflt;
  if (v->t != JVal::Num) fail(kFormatError, std::string("bad model config JSON: ") + k);
  return static_cast<int>(v->num);
}

std::string json_double(double d) {  // shortest round-trip, nlohmann style
  char buf[64];
  for (int prec = 1; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof buf, "%.*g", prec, d);
    if (std::strtod(buf, nullptr) == d) break;
  }
  std::string s = buf;
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}

const char* combine_name(FactorCombine c) {
  return c == FactorCombine::kConcat ? "concat" : c == FactorCombine::kAverage ? "average" : "sum";
}

}  // namespace

// ---- ModelConfig (model.cpp:53-148) ------------------------------------------

int ModelConfig::word_embed_dim() const {
  if (!factor_configs.empty() && factor_configs.front().combine == FactorCombine::kConcat) {
    int total = 0;
    for (const auto& f : factor_configs) total += f.embed_dim;
    return d_model - total;
  }
  return d_model;
}

void ModelConfig::validate() const {
  if (d_model <= 0 || d_ff <= 0 || num_heads <= 0)
    fail(kUsageError, "d_model, d_ff, num_heads must be positive");
  if (d_model % num_heads != 0) fail(kUsageError, "d_model must be divisible by num_heads");
  if (num_encoder_layers < 0 || num_decoder_layers < 0)
    fail(kUsageError, "layer counts must be non-negative");
  if (src_vocab_size < 4 || tgt_vocab_size < 4)
    fail(kUsageError, "vocabulary sizes must cover the reserved tokens");
  if (max_seq_len < 1) fail(kUsageError, "max_seq_len must be positive");
  if (!factor_configs.empty()) {
    const FactorCombine mode = factor_configs.front().combine;
    for (const auto& f : factor_configs) {
      if (f.combine != mode) fail(kUsageError, "all source factors must use one combine mode");
      if (f.factor_vocab_size < 4 || f.embed_dim <= 0)
        fail(kUsageError, "bad factor vocab size or embed dim");
    }
    const int wdim = word_embed_dim();
    if (mode == FactorCombine::kConcat) {
      if (wdim <= 0) fail(kUsageError, "concat factors: word dim + factor dims must equal d_model");
    } else {
      for (const auto& f : factor_configs)
        if (f.embed_dim != wdim) fail(kUsageError, "sum/average factors need embed_dim == word dim");
    }
    for (const auto& f : factor_configs)
      if (f.share_with_word_embedding) {
        if (f.embed_dim != wdim) fail(kUsageError, "shared factor embedding needs word embed dim");
        if (f.factor_vocab_size > src_vocab_size)
          fail(kUsageError, "shared factor vocabulary must fit inside the word vocabulary");
      }
  }
}

std::string ModelConfig::to_json() const {
  std::string f = "[";
  for (size_t i = 0; i < factor_configs.size(); ++i) {
    const auto& c = factor_configs[i];
    if (i) f += ",";
    f += std::string("{\"combine\":\"") + combine_name(c.combine) +
         "\",\"embed_dim\":" + std::to_string(c.embed_dim) +
         ",\"share\":" + (c.share_with_word_embedding ? "true" : "false") +
         ",\"vocab_size\":" + std::to_string(c.factor_vocab_size) + "}";
  }
  f += "]";
  return "{\"d_ff\":" + std::to_string(d_ff) + ",\"d_model\":" + std::to_string(d_model) +
         ",\"dropout\":" + json_double(static_cast<double>(dropout)) + ",\"factors\":" + f +
         ",\"max_seq_len\":" + std::to_string(max_seq_len) +
         ",\"num_decoder_layers\":" + std::to_string(num_decoder_layers) +
         ",\"num_encoder_layers\":" + std::to_string(num_encoder_layers) +
         ",\"num_heads\":" + std::to_string(num_heads) +
         ",\"src_vocab_size\":" + std::to_string(src_vocab_size) +
         ",\"tgt_vocab_size\":" + std::to_string(tgt_vocab_size) + "}";
}

ModelConfig ModelConfig::from_json(const std::string& json) {
  JsonReader r(json);
  JVal j = r.value();
  if (j.t != JVal::Obj) fail(kFormatError, "bad model config JSON: not an object");
  ModelConfig c;
  c.num_encoder_layers = jint(j, "num_encoder_layers", 6);
  c.num_decoder_layers = jint(j, "num_decoder_layers", 6);
  c.d_model = jint(j, "d_model", 32);
  c.d_ff = jint(j, "d_ff", 128);
  c.num_heads = jint(j, "num_heads", 4);
  c.src_vocab_size = jint(j, "src_vocab_size", 0);
  c.tgt_vocab_size = jint(j, "tgt_vocab_size", 0);
  if (const JVal* d = j.get("dropout"); d && d->t == JVal::Num) c.dropout = static_cast<float>(d->num);
  c.max_seq_len = jint(j, "max_seq_len", 128);
  if (const JVal* fs = j.get("factors"); fs && fs->t == JVal::Arr) {
    for (const JVal& f : fs->arr) {
      SourceFactorConfig fc;
      fc.factor_vocab_size = jint(f, "vocab_size", 0);
      fc.embed_dim = jint(f, "embed_dim", 0);
      std::string comb = "sum";
      if (const JVal* cv = f.get("combine"); cv && cv->t == JVal::Str) comb = cv->s;
      if (comb == "concat") fc.combine = FactorCombine::kConcat;
      else if (comb == "sum") fc.combine = FactorCombine::kSum;
      else if (comb == "average") fc.combine = FactorCombine::kAverage;
      else fail(kUsageError, "unknown factor combine mode: " + comb);
      if (const JVal* sh = f.get("share"); sh && sh->t == JVal::Bool) fc.share_with_word_embedding = sh->b;
      c.factor_configs.push_back(fc);
    }
  }
  return c;
}

// ---- layout / init ---------------------------------------------------------------

int64_t HostTensor::numel() const {
  int64_t n = 1;
  for (int64_t d : shape) n *= d;
  return n;
}

const HostTensor& HostModel::at(const std::string& name) const {
  auto it = params.find(name);
  if (it == params.end()) fail(kStateError, "unknown parameter: " + name);
  return it->second;
}

std::vector<std::pair<std::string, std::vector<int64_t>>> param_shapes(const ModelConfig& c) {
  std::vector<std::pair<std::string, std::vector<int64_t>>> out;
  const int64_t d = c.d_model, dff = c.d_ff;
  out.emplace_back("src_embed", std::vector<int64_t>{c.src_vocab_size, c.word_embed_dim()});
  for (size_t i = 0; i < c.factor_configs.size(); ++i)
    if (!c.factor_configs[i].share_with_word_embedding)
      out.emplace_back("factor" + std::to_string(i) + "_embed",
                       std::vector<int64_t>{c.factor_configs[i].factor_vocab_size,
                                            c.factor_configs[i].embed_dim});
  out.emplace_back("tgt_embed", std::vector<int64_t>{c.tgt_vocab_size, d});
  auto norm = [&](const std::string& p) {
    out.emplace_back(p + ".gain", std::vector<int64_t>{d});
    out.emplace_back(p + ".bias", std::vector<int64_t>{d});
  };
  auto attn = [&](const std::string& p) {
    for (const char* w : {".wq", ".wk", ".wv", ".wo"}) out.emplace_back(p + w, std::vector<int64_t>{d, d});
  };
  auto ffn = [&](const std::string& p) {
    out.emplace_back(p + ".w1", std::vector<int64_t>{d, dff});
    out.emplace_back(p + ".b1", std::vector<int64_t>{dff});
    out.emplace_back(p + ".w2", std::vector<int64_t>{dff, d});
    out.emplace_back(p + ".b2", std::vector<int64_t>{d});
  };
  for (int l = 0; l < c.num_encoder_layers; ++l) {
    const std::string p = "enc" + std::to_string(l);
    norm(p + ".norm1");
    attn(p + ".attn");
    norm(p + ".norm2");
    ffn(p + ".ffn");
  }
  if (c.num_encoder_layers > 0) norm("enc_final");
  for (int l = 0; l < c.num_decoder_layers; ++l) {
    const std::string p = "dec" + std::to_string(l);
    norm(p + ".norm1");
    attn(p + ".self");
    norm(p + ".norm2");
    attn(p + ".cross");
    norm(p + ".norm3");
    ffn(p + ".ffn");
  }
  norm("dec_final");
  return out;
}

std::vector<float> make_pos_enc(int max_len, int d) {  // model.cpp:13-22
  std::vector<float> pe(static_cast<size_t>(max_len) * d, 0.0f);
  for (int pos = 0; pos < max_len; ++pos)
    for (int i = 0; i < d; i += 2) {
      const double angle = pos / std::pow(10000.0, static_cast<double>(i) / d);
      pe[size_t(pos) * d + i] = static_cast<float>(std::sin(angle));
      if (i + 1 < d) pe[size_t(pos) * d + i + 1] = static_cast<float>(std::cos(angle));
    }
  return pe;
}

bool is_quantized_param(const std::string& name) {  // model.cpp:676-681
  if (name == "tgt_embed") return true;
  for (const char* s : {".wq", ".wk", ".wv", ".wo", ".w1", ".w2"}) {
    const size_t n = std::strlen(s);
    if (name.size() >= n && name.compare(name.size() - n, n, s) == 0) return true;
  }
  return false;
}

// model.cpp:229-238: std::map (name-sorted) order, one mt19937_64 stream,
// Xavier-uniform per rank-2 tensor, gains 1 / biases 0.
HostModel make_random_model(const ModelConfig& c, uint64_t seed) {
  c.validate();
  HostModel m;
  m.config = c;
  for (auto& [name, shape] : param_shapes(c)) {
    HostTensor t;
    t.shape = shape;
    t.f32.assign(static_cast<size_t>(t.numel()), 0.0f);
    m.params.emplace(name, std::move(t));
  }
  std::mt19937_64 engine(seed);
  for (auto& [name, t] : m.params) {
    if (t.shape.size() == 2) {
      const float limit = std::sqrt(6.0f / static_cast<float>(t.rows() + t.cols()));
      for (auto& v : t.f32) {
        std::uniform_real_distribution<float> dist(-limit, limit);
        v = dist(engine);
      }
    } else {
      const bool gain = name.size() >= 5 && name.compare(name.size() - 5, 5, ".gain") == 0;
      std::fill(t.f32.begin(), t.f32.end(), gain ? 1.0f : 0.0f);
    }
  }
  return m;
}

// quantize_model (model.cpp:733-748) + quantize (quant.cpp:108-122): every
// parameter is checked for non-finite values in name order (check_finite runs
// before the quantizable test), then the quantizable ones get one scale each.
void quantize_weights(HostModel& m) {
  for (auto& [name, t] : m.params) {
    if (t.is_int8) continue;
    for (float v : t.f32)
      if (!std::isfinite(v)) fail(kValueError, "quantize_model(" + name + "): non-finite values");
    if (!is_quantized_param(name)) continue;
    float max_abs = 0.0f;
    for (float v : t.f32) max_abs = std::max(max_abs, std::fabs(v));
    t.scale = max_abs == 0.0f ? 1.0f : 127.0f / max_abs;
    t.q.resize(t.f32.size());
    for (size_t i = 0; i < t.f32.size(); ++i) {
      float v = std::round(t.f32[i] * t.scale);
      v = std::min(127.0f, std::max(-127.0f, v));
      t.q[i] = static_cast<int8_t>(v);
    }
    t.is_int8 = true;
  }
  m.quantized = true;
}

// ---- SQNT (io.cpp:12-129; model.cpp:699-807) ----------------------------------

namespace {
template <typename T>
void put(std::string& out, T v) {
  char b[sizeof(T)];
  std::memcpy(b, &v, sizeof(T));
  out.append(b, sizeof(T));
}
struct Reader {
  const uint8_t* d;
  size_t n, pos = 0;
  void need(size_t k) {
    if (pos + k > n) fail(kFormatError, "truncated parameter file");
  }
  template <typename T>
  T get() {
    need(sizeof(T));
    T v;
    std::memcpy(&v, d + pos, sizeof(T));
    pos += sizeof(T);
    return v;
  }
  std::string str(size_t k) {
    need(k);
    std::string s(reinterpret_cast<const char*>(d + pos), k);
    pos += k;
    return s;
  }
};
}  // namespace

HostModel load_sqnt(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) fail(kIoError, "cannot open: " + path);
  std::vector<uint8_t> bytes((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  Reader r{bytes.data(), bytes.size()};
  if (r.str(4) != "SQNT") fail(kFormatError, "bad magic in " + path);
  const uint32_t ver = r.get<uint32_t>();
  if (ver != 1) fail(kFormatError, "unsupported file version " + std::to_string(ver));
  HostModel m;
  m.config = ModelConfig::from_json(r.str(r.get<uint32_t>()));
  m.config.validate();
  std::map<std::string, HostTensor> recs;
  const uint32_t count = r.get<uint32_t>();
  bool any_int8 = false;
  for (uint32_t i = 0; i < count; ++i) {
    std::string name = r.str(r.get<uint16_t>());
    HostTensor t;
    const uint8_t dtype = r.get<uint8_t>();
    if (dtype > 1) fail(kFormatError, "unknown dtype tag for " + name);
    const uint8_t rank = r.get<uint8_t>();
    for (uint8_t k = 0; k < rank; ++k) t.shape.push_back(r.get<uint32_t>());
    if (dtype == 1) {
      t.scale = r.get<float>();
      t.is_int8 = true;
      any_int8 = true;
    }
    const size_t n = static_cast<size_t>(t.numel());
    const size_t nbytes = n * (dtype == 0 ? 4 : 1);
    r.need(nbytes);
    if (dtype == 0) {
      t.f32.resize(n);
      std::memcpy(t.f32.data(), bytes.data() + r.pos, nbytes);
    } else {
      t.q.resize(n);
      std::memcpy(t.q.data(), bytes.data() + r.pos, nbytes);
    }
    r.pos += nbytes;
    recs.emplace(std::move(name), std::move(t));
  }
  if (r.pos != r.n) fail(kFormatError, "trailing bytes in " + path);
  for (auto& [name, shape] : param_shapes(m.config)) {
    auto it = recs.find(name);
    if (it == recs.end()) fail(kFormatError, "missing parameter: " + name);
    if (it->second.shape != shape) fail(kFormatError, "shape mismatch for parameter: " + name);
    if (it->second.is_int8 && (!(it->second.scale > 0.0f) || !std::isfinite(it->second.scale)))
      fail(kFormatError, "bad scale for parameter: " + name);
    m.params.emplace(name, std::move(it->second));
  }
  m.quantized = any_int8;
  return m;
}

void save_sqnt(const HostModel& m, const std::string& path) {
  std::string out("SQNT", 4);
  put<uint32_t>(out, 1);
  const std::string cfg = m.config.to_json();
  put<uint32_t>(out, static_cast<uint32_t>(cfg.size()));
  out += cfg;
  const auto shapes = param_shapes(m.config);
  put<uint32_t>(out, static_cast<uint32_t>(shapes.size()));
  for (auto& [name, shape] : shapes) {
    const HostTensor& t = m.at(name);
    const bool q = m.quantized && t.is_int8;
    put<uint16_t>(out, static_cast<uint16_t>(name.size()));
    out += name;
    put<uint8_t>(out, q ? 1 : 0);
    put<uint8_t>(out, static_cast<uint8_t>(t.shape.size()));
    for (int64_t d : t.shape) put<uint32_t>(out, static_cast<uint32_t>(d));
    if (q) {
      put<float>(out, t.scale);
      out.append(reinterpret_cast<const char*>(t.q.data()), t.q.size());
    } else {
      if (t.f32.size() != static_cast<size_t>(t.numel()))
        fail(kStateError, "no f32 payload for " + name);
      out.append(reinterpret_cast<const char*>(t.f32.data()), t.f32.size() * 4);
    }
  }
  std::ofstream f(path, std::ios::binary | std::ios::trunc);
  if (!f) fail(kIoError, "cannot open for writing: " + path);
  f.write(out.data(), static_cast<std::streamsize>(out.size()));
  if (!f) fail(kIoError, "write failed: " + path);
}

}  // namespace mtg
