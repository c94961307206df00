// TEST INFRASTRUCTURE (oracle) -- not product code. See oracle.hpp.
//
// Pinned float orders (the reference leaves them to Eigen; the GPU kernels and
// this file agree on the ones below):
//   P1 lane sum     : 32 partials, partial l = sum of v[l], v[l+32], ... in
//                     order, then xor-butterfly (16,8,4,2,1). (warp_sum)
//   P6 log-sum-exp  : per 32-column slice k: m_k = max, s_k = sum in column
//                     order of exp(x - m_k) (0 if m_k = -inf); M = max m_k;
//                     S = sum over k of s_k * exp(m_k - M) (0 if m_k = -inf):
//                     128 partials (t sums k = t + 128 i), P1 butterfly per
//                     32, then (W0 + W1) + (W2 + W3);
//                     lse = log(S) + M. (log_softmax_row; the GPU computes the
//                     slices in the output-projection GEMM epilogue)
//   P3 dot          : acc = 0; acc = acc + a[c]*b[c] for c ascending (no FMA).
//   attention ctx   : ctx[c] = sum over keys j ascending of p_j * v_j[c].
//   P4 exp/log/pow  : detmath.h.
//   P5 f32 GEMM     : per output element, k-ascending mul+add (gemm_rows order,
//                     tensor.cpp:113-123); the GPU uses 3xTF32 tensor cores,
//                     compared within tolerance.
#include "oracle.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <iterator>
#include <memory>
#include <sstream>

#include "detmath.h"

namespace orc {

void fail(int code, const std::string& msg) { throw Error(code, msg); }

// =============================================================================
// minimal JSON (the reference uses nlohmann/json; model.cpp:102-148)
// =============================================================================
namespace {

struct JVal {
  enum T { Null, Bool, Num, Str, Arr, Obj } t = Null;
  double num = 0;
  bool b = false;
  std::string s;
  std::vector<JVal> arr;
  std::vector<std::pair<std::string, JVal>> obj;
  const JVal* get(const std::string& k) const {
    for (auto& kv : obj)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
};

struct JParser {
  const std::string& s;
  size_t i = 0;
  [[noreturn]] void bad() { fail(kFormat, "bad model config JSON"); }
  void ws() {
    while (i < s.size() && std::isspace(static_cast<unsigned char>(s[i]))) ++i;
  }
  JVal parse() {
    ws();
    if (i >= s.size()) bad();
    JVal v;
    char c = s[i];
    if (c == '{') {
      v.t = JVal::Obj;
      ++i;
      ws();
      if (i < s.size() && s[i] == '}') { ++i; return v; }
      for (;;) {
        ws();
        JVal k = parse();
        if (k.t != JVal::Str) bad();
        ws();
        if (i >= s.size() || s[i] != ':') bad();
        ++i;
        JVal val = parse();
        v.obj.emplace_back(k.s, std::move(val));
        ws();
        if (i < s.size() && s[i] == ',') { ++i; continue; }
        if (i < s.size() && s[i] == '}') { ++i; break; }
        bad();
      }
    } else if (c == '[') {
      v.t = JVal::Arr;
      ++i;
      ws();
      if (i < s.size() && s[i] == ']') { ++i; return v; }
      for (;;) {
        v.arr.push_back(parse());
        ws();
        if (i < s.size() && s[i] == ',') { ++i; continue; }
        if (i < s.size() && s[i] == ']') { ++i; break; }
        bad();
      }
    } else if (c == '"') {
      v.t = JVal::Str;
      ++i;
      while (i < s.size() && s[i] != '"') {
        if (s[i] == '\\') {
          ++i;
          if (i >= s.size()) bad();
          char e = s[i];
          v.s += e == 'n' ? '\n' : e == 't' ? '\t' : e;
        } else {
          v.s += s[i];
        }
        ++i;
      }
      if (i >= s.size()) bad();
      ++i;
    } else if (s.compare(i, 4, "true") == 0) {
      v.t = JVal::Bool; v.b = true; i += 4;
    } else if (s.compare(i, 5, "false") == 0) {
      v.t = JVal::Bool; v.b = false; i += 5;
    } else if (s.compare(i, 4, "null") == 0) {
      v.t = JVal::Null; i += 4;
    } else {
      size_t end = i;
      while (end < s.size() && (std::isdigit(static_cast<unsigned char>(s[end])) ||
                                s[end] == '-' || s[end] == '+' || s[end] == '.' ||
                                s[end] == 'e' || s[end] == 'E'))
        ++end;
      if (end == i) bad();
      v.t = JVal::Num;
      v.num = std::strtod(s.substr(i, end - i).c_str(), nullptr);
      i = end;
    }
    return v;
  }
};

int jint(const JVal& o, const char* k, int dflt) {
  const JVal* v = o.get(k);
  if (!v || v->t == JVal::Null) return dflt;
  if (v->t != JVal::Num) fail(kFormat, std::string("bad model config JSON: ") + k);
  return static_cast<int>(v->num);
}

std::string json_double(double d) {  // nlohmann-style shortest round trip
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
  switch (c) {
    case FactorCombine::kConcat: return "concat";
    case FactorCombine::kSum: return "sum";
    case FactorCombine::kAverage: return "average";
  }
  return "sum";
}

}  // namespace

// model.cpp:53-61
int ModelConfig::word_embed_dim() const {
  if (!factor_configs.empty() && factor_configs.front().combine == FactorCombine::kConcat) {
    int total = 0;
    for (const auto& f : factor_configs) total += f.embed_dim;
    return d_model - total;
  }
  return d_model;
}

// model.cpp:63-100
void ModelConfig::validate() const {
  if (d_model <= 0 || d_ff <= 0 || num_heads <= 0)
    fail(kUsage, "d_model, d_ff, num_heads must be positive");
  if (d_model % num_heads != 0) fail(kUsage, "d_model must be divisible by num_heads");
  if (num_encoder_layers < 0 || num_decoder_layers < 0)
    fail(kUsage, "layer counts must be non-negative");
  if (src_vocab_size < 4 || tgt_vocab_size < 4)
    fail(kUsage, "vocabulary sizes must cover the reserved tokens");
  if (max_seq_len < 1) fail(kUsage, "max_seq_len must be positive");
  if (!factor_configs.empty()) {
    FactorCombine mode = factor_configs.front().combine;
    for (const auto& f : factor_configs) {
      if (f.combine != mode) fail(kUsage, "all source factors must use one combine mode");
      if (f.factor_vocab_size < 4 || f.embed_dim <= 0)
        fail(kUsage, "bad factor vocab size or embed dim");
    }
    int wdim = word_embed_dim();
    if (mode == FactorCombine::kConcat) {
      if (wdim <= 0) fail(kUsage, "concat factors: word dim + factor dims must equal d_model");
    } else {
      for (const auto& f : factor_configs)
        if (f.embed_dim != wdim) fail(kUsage, "sum/average factors need embed_dim == word dim");
    }
    for (const auto& f : factor_configs)
      if (f.share_with_word_embedding) {
        if (f.embed_dim != wdim) fail(kUsage, "shared factor embedding needs word embed dim");
        if (f.factor_vocab_size > src_vocab_size)
          fail(kUsage, "shared factor vocabulary must fit inside the word vocabulary");
      }
  }
}

// model.cpp:102-120 (nlohmann dump: keys sorted, compact)
std::string ModelConfig::to_json() const {
  std::string f = "[";
  for (size_t i = 0; i < factor_configs.size(); ++i) {
    const auto& c = factor_configs[i];
    if (i) f += ",";
    f += std::string("{\"combine\":\"") + combine_name(c.combine) + "\",\"embed_dim\":" +
         std::to_string(c.embed_dim) + ",\"share\":" +
         (c.share_with_word_embedding ? "true" : "false") +
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

// model.cpp:122-148
ModelConfig ModelConfig::from_json(const std::string& json) {
  JParser p{json};
  JVal j = p.parse();
  if (j.t != JVal::Obj) fail(kFormat, "bad model config JSON: not an object");
  ModelConfig c;
  c.num_encoder_layers = jint(j, "num_encoder_layers", 6);
  c.num_decoder_layers = jint(j, "num_decoder_layers", 6);
  c.d_model = jint(j, "d_model", 32);
  c.d_ff = jint(j, "d_ff", 128);
  c.num_heads = jint(j, "num_heads", 4);
  c.src_vocab_size = jint(j, "src_vocab_size", 0);
  c.tgt_vocab_size = jint(j, "tgt_vocab_size", 0);
  if (const JVal* d = j.get("dropout"); d && d->t == JVal::Num)
    c.dropout = static_cast<float>(d->num);
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
      else fail(kUsage, "unknown factor combine mode: " + comb);
      if (const JVal* sh = f.get("share"); sh && sh->t == JVal::Bool)
        fc.share_with_word_embedding = sh->b;
      c.factor_configs.push_back(fc);
    }
  }
  return c;
}

// =============================================================================
// tensors, model layout, init
// =============================================================================

Tensor::Tensor(std::vector<Index> s) : shape(std::move(s)) {
  Index n = 1;
  for (Index d : shape) n *= d;
  data.assign(static_cast<size_t>(n), 0.0f);
}

// quant.cpp:124-131
void QTensor::finish() {
  row_sums.assign(static_cast<size_t>(rows()), 0);
  for (Index i = 0; i < rows(); ++i) {
    int32_t s = 0;
    for (Index j = 0; j < cols(); ++j) s += q[i * cols() + j];
    row_sums[i] = s;
  }
}

const Tensor& Model::param(const std::string& name) const {
  auto it = params.find(name);
  if (it == params.end()) fail(kState, "unknown parameter: " + name);
  return it->second;
}
Tensor& Model::param(const std::string& name) {
  auto it = params.find(name);
  if (it == params.end()) fail(kState, "unknown parameter: " + name);
  return it->second;
}
size_t Model::param_count() const {
  size_t n = 0;
  for (const auto& kv : params) n += kv.second.data.size();
  return n;
}

// model.cpp:174-219
std::vector<std::pair<std::string, std::vector<Index>>> param_shapes(const ModelConfig& c) {
  std::vector<std::pair<std::string, std::vector<Index>>> out;
  Index d = c.d_model, dff = c.d_ff;
  out.emplace_back("src_embed", std::vector<Index>{c.src_vocab_size, c.word_embed_dim()});
  for (size_t i = 0; i < c.factor_configs.size(); ++i)
    if (!c.factor_configs[i].share_with_word_embedding)
      out.emplace_back("factor" + std::to_string(i) + "_embed",
                       std::vector<Index>{c.factor_configs[i].factor_vocab_size,
                                          c.factor_configs[i].embed_dim});
  out.emplace_back("tgt_embed", std::vector<Index>{c.tgt_vocab_size, d});
  auto norm = [&](const std::string& p) {
    out.emplace_back(p + ".gain", std::vector<Index>{d});
    out.emplace_back(p + ".bias", std::vector<Index>{d});
  };
  auto attn = [&](const std::string& p) {
    for (const char* w : {".wq", ".wk", ".wv", ".wo"})
      out.emplace_back(p + w, std::vector<Index>{d, d});
  };
  auto ffn = [&](const std::string& p) {
    out.emplace_back(p + ".w1", std::vector<Index>{d, dff});
    out.emplace_back(p + ".b1", std::vector<Index>{dff});
    out.emplace_back(p + ".w2", std::vector<Index>{dff, d});
    out.emplace_back(p + ".b2", std::vector<Index>{d});
  };
  for (int l = 0; l < c.num_encoder_layers; ++l) {
    std::string p = "enc" + std::to_string(l);
    norm(p + ".norm1");
    attn(p + ".attn");
    norm(p + ".norm2");
    ffn(p + ".ffn");
  }
  if (c.num_encoder_layers > 0) norm("enc_final");
  for (int l = 0; l < c.num_decoder_layers; ++l) {
    std::string p = "dec" + std::to_string(l);
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

// model.cpp:13-22 (double-precision angles cast to float)
std::vector<float> make_pos_enc(int max_len, int d) {
  std::vector<float> pe(static_cast<size_t>(max_len) * d, 0.0f);
  for (int pos = 0; pos < max_len; ++pos)
    for (int i = 0; i < d; i += 2) {
      double angle = pos / std::pow(10000.0, static_cast<double>(i) / d);
      pe[size_t(pos) * d + i] = static_cast<float>(std::sin(angle));
      if (i + 1 < d) pe[size_t(pos) * d + i + 1] = static_cast<float>(std::cos(angle));
    }
  return pe;
}

// model.cpp:221-227
Model make_model(const ModelConfig& c) {
  c.validate();
  Model m;
  m.config = c;
  for (auto& [name, shape] : param_shapes(c)) m.params.emplace(name, Tensor(shape));
  m.pe = make_pos_enc(c.max_seq_len, c.d_model);
  return m;
}

// model.cpp:229-238 with tensor.hpp:62-78 Rng (mt19937_64, a fresh
// uniform_real_distribution<float> per draw), std::map name order.
void init_params(Model& m, uint64_t seed) {
  std::mt19937_64 engine(seed);
  for (auto& [name, t] : m.params) {
    if (t.rank() == 2) {
      float limit = std::sqrt(6.0f / static_cast<float>(t.rows() + t.cols()));
      for (auto& v : t.data) {
        std::uniform_real_distribution<float> dist(-limit, limit);
        v = dist(engine);
      }
    } else {
      bool gain = name.size() >= 5 && name.compare(name.size() - 5, 5, ".gain") == 0;
      std::fill(t.data.begin(), t.data.end(), gain ? 1.0f : 0.0f);
    }
  }
}

// model.cpp:676-681
bool is_quantized_param(const std::string& name) {
  if (name == "tgt_embed") return true;
  for (const char* s : {".wq", ".wk", ".wv", ".wo", ".w1", ".w2"}) {
    size_t n = std::strlen(s);
    if (name.size() >= n && name.compare(name.size() - n, n, s) == 0) return true;
  }
  return false;
}

// =============================================================================
// quantization (quant.cpp:108-239)
// =============================================================================

QTensor quantize(const float* x, std::vector<Index> shape) {
  QTensor q;
  q.shape = std::move(shape);
  Index n = 1;
  for (Index d : q.shape) n *= d;
  q.q.resize(static_cast<size_t>(n));
  float max_abs = 0.0f;
  for (Index i = 0; i < n; ++i) {
    if (!std::isfinite(x[i])) fail(kValue, "quantize: non-finite values in tensor");
    max_abs = std::max(max_abs, std::fabs(x[i]));
  }
  q.scale = max_abs == 0.0f ? 1.0f : 127.0f / max_abs;
  for (Index i = 0; i < n; ++i) {
    float v = std::round(x[i] * q.scale);
    v = std::min(127.0f, std::max(-127.0f, v));
    q.q[i] = static_cast<int8_t>(v);
  }
  q.finish();
  return q;
}
QTensor quantize(const Tensor& x) { return quantize(x.data.data(), x.shape); }

// Scalar int32 ground truth (quant.cpp:182-192 and 226-238).
void qmatmul(const QTensor& a, const QTensor& b, float* c) {
  Index m = a.rows(), k = a.cols(), n = b.cols();
  if (k != b.rows()) fail(kShape, "qmatmul: inner dimensions disagree");
  if (k > 65536) fail(kValue, "qmatmul: inner dimension above 65536");
  float inv = 1.0f / (a.scale * b.scale);
  std::vector<int32_t> acc(static_cast<size_t>(n));
  for (Index i = 0; i < m; ++i) {
    std::fill(acc.begin(), acc.end(), 0);
    for (Index kk = 0; kk < k; ++kk) {
      int32_t av = a.q[i * k + kk];
      const int8_t* br = b.q.data() + kk * n;
      for (Index j = 0; j < n; ++j) acc[j] += av * static_cast<int32_t>(br[j]);
    }
    for (Index j = 0; j < n; ++j) c[i * n + j] = static_cast<float>(acc[j]) * inv;
  }
}

static int32_t dot_i8(const int8_t* a, const int8_t* b, Index k) {
  int32_t acc = 0;
  for (Index i = 0; i < k; ++i) acc += static_cast<int32_t>(a[i]) * static_cast<int32_t>(b[i]);
  return acc;
}

void qmatmul_nt(const QTensor& a, const QTensor& b, const std::vector<int>* rows, float* c) {
  Index m = a.rows(), k = a.cols();
  if (k != b.cols()) fail(kShape, "qmatmul_nt: inner dimensions disagree");
  if (k > 65536) fail(kValue, "qmatmul_nt: inner dimension above 65536");
  Index n = rows ? static_cast<Index>(rows->size()) : b.rows();
  float inv = 1.0f / (a.scale * b.scale);
  for (Index j = 0; j < n; ++j) {
    Index r = rows ? (*rows)[j] : j;
    if (r < 0 || r >= b.rows()) fail(kIndex, "qmatmul_nt: row out of range");
    for (Index i = 0; i < m; ++i)
      c[i * n + j] = static_cast<float>(dot_i8(a.q.data() + i * k, b.q.data() + r * k, k)) * inv;
  }
}

// model.cpp:733-748
QModel quantize_model(const Model& m) {
  QModel qm;
  qm.config = m.config;
  qm.pe = m.pe;
  for (const auto& [name, t] : m.params) {
    for (float v : t.data)
      if (!std::isfinite(v)) fail(kValue, "quantize_model(" + name + "): non-finite values");
    if (is_quantized_param(name))
      qm.q.emplace(name, quantize(t));
    else
      qm.f32.emplace(name, t);
  }
  return qm;
}

// =============================================================================
// SQNT container (io.cpp:12-129)
// =============================================================================

size_t ParamRecord::numel() const {
  size_t n = 1;
  for (auto d : dims) n *= d;
  return n;
}
const ParamRecord* ParamFile::find(const std::string& name) const {
  for (const auto& p : params)
    if (p.name == name) return &p;
  return nullptr;
}

namespace {
template <typename T>
void put(std::string& out, T v) {
  char buf[sizeof(T)];
  std::memcpy(buf, &v, sizeof(T));
  out.append(buf, sizeof(T));
}
struct Reader {
  const uint8_t* d;
  size_t n, pos = 0;
  void need(size_t k) {
    if (pos + k > n) fail(kFormat, "truncated parameter file");
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

void write_param_file(const std::string& path, const ParamFile& file) {
  std::string out("SQNT", 4);
  put<uint32_t>(out, 1);
  put<uint32_t>(out, static_cast<uint32_t>(file.config_json.size()));
  out += file.config_json;
  put<uint32_t>(out, static_cast<uint32_t>(file.params.size()));
  for (const auto& p : file.params) {
    if (p.name.size() > 0xffff) fail(kFormat, "parameter name too long");
    put<uint16_t>(out, static_cast<uint16_t>(p.name.size()));
    out += p.name;
    put<uint8_t>(out, p.dtype);
    put<uint8_t>(out, static_cast<uint8_t>(p.dims.size()));
    for (auto d : p.dims) put<uint32_t>(out, d);
    if (p.dtype == 1) put<float>(out, p.scale);
    size_t elem = p.dtype == 0 ? 4 : 1;
    if (p.payload.size() != p.numel() * elem) fail(kFormat, "payload size mismatch for " + p.name);
    out.append(reinterpret_cast<const char*>(p.payload.data()), p.payload.size());
  }
  std::ofstream f(path, std::ios::binary | std::ios::trunc);
  if (!f) fail(kIo, "cannot open for writing: " + path);
  f.write(out.data(), static_cast<std::streamsize>(out.size()));
  if (!f) fail(kIo, "write failed: " + path);
}

ParamFile read_param_file(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) fail(kIo, "cannot open: " + path);
  std::vector<uint8_t> bytes((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  Reader r{bytes.data(), bytes.size()};
  if (r.str(4) != "SQNT") fail(kFormat, "bad magic in " + path);
  uint32_t ver = r.get<uint32_t>();
  if (ver != 1) fail(kFormat, "unsupported file version " + std::to_string(ver));
  ParamFile out;
  out.config_json = r.str(r.get<uint32_t>());
  uint32_t count = r.get<uint32_t>();
  for (uint32_t i = 0; i < count; ++i) {
    ParamRecord p;
    p.name = r.str(r.get<uint16_t>());
    p.dtype = r.get<uint8_t>();
    if (p.dtype > 1) fail(kFormat, "unknown dtype tag for " + p.name);
    uint8_t rank = r.get<uint8_t>();
    for (uint8_t d = 0; d < rank; ++d) p.dims.push_back(r.get<uint32_t>());
    if (p.dtype == 1) p.scale = r.get<float>();
    size_t nbytes = p.numel() * (p.dtype == 0 ? 4 : 1);
    r.need(nbytes);
    p.payload.assign(bytes.data() + r.pos, bytes.data() + r.pos + nbytes);
    r.pos += nbytes;
    out.params.push_back(std::move(p));
  }
  if (r.pos != r.n) fail(kFormat, "trailing bytes in " + path);
  return out;
}

static std::vector<uint32_t> dims_of(const std::vector<Index>& s) {
  std::vector<uint32_t> d;
  for (Index v : s) d.push_back(static_cast<uint32_t>(v));
  return d;
}

void save_params(const Model& m, const std::string& path) {
  ParamFile file;
  file.config_json = m.config.to_json();
  for (auto& [name, shape] : param_shapes(m.config)) {
    const Tensor& t = m.param(name);
    ParamRecord rec;
    rec.name = name;
    rec.dims = dims_of(t.shape);
    rec.payload.resize(t.data.size() * 4);
    std::memcpy(rec.payload.data(), t.data.data(), rec.payload.size());
    file.params.push_back(std::move(rec));
  }
  write_param_file(path, file);
}

Model load_params(const std::string& path) {
  ParamFile file = read_param_file(path);
  Model m = make_model(ModelConfig::from_json(file.config_json));
  for (auto& [name, shape] : param_shapes(m.config)) {
    const ParamRecord* rec = file.find(name);
    if (!rec) fail(kFormat, "missing parameter: " + name);
    if (rec->dtype != 0) fail(kFormat, "expected f32 parameter: " + name);
    Tensor& t = m.param(name);
    if (dims_of(t.shape) != rec->dims) fail(kFormat, "shape mismatch for parameter: " + name);
    std::memcpy(t.data.data(), rec->payload.data(), rec->payload.size());
  }
  return m;
}

void save_quantized(const QModel& m, const std::string& path) {
  ParamFile file;
  file.config_json = m.config.to_json();
  for (auto& [name, shape] : param_shapes(m.config)) {
    ParamRecord rec;
    rec.name = name;
    auto qit = m.q.find(name);
    if (qit != m.q.end()) {
      rec.dtype = 1;
      rec.dims = dims_of(qit->second.shape);
      rec.scale = qit->second.scale;
      rec.payload.assign(reinterpret_cast<const uint8_t*>(qit->second.q.data()),
                         reinterpret_cast<const uint8_t*>(qit->second.q.data()) + qit->second.q.size());
    } else {
      const Tensor& t = m.f32.at(name);
      rec.dims = dims_of(t.shape);
      rec.payload.resize(t.data.size() * 4);
      std::memcpy(rec.payload.data(), t.data.data(), rec.payload.size());
    }
    file.params.push_back(std::move(rec));
  }
  write_param_file(path, file);
}

QModel load_quantized(const std::string& path) {
  ParamFile file = read_param_file(path);
  QModel m;
  m.config = ModelConfig::from_json(file.config_json);
  m.config.validate();
  m.pe = make_pos_enc(m.config.max_seq_len, m.config.d_model);
  for (auto& [name, shape] : param_shapes(m.config)) {
    const ParamRecord* rec = file.find(name);
    if (!rec) fail(kFormat, "missing parameter: " + name);
    std::vector<Index> sh(rec->dims.begin(), rec->dims.end());
    if (rec->dtype == 1) {
      QTensor q;
      q.shape = sh;
      q.scale = rec->scale;
      if (!(q.scale > 0.0f) || !std::isfinite(q.scale))
        fail(kFormat, "bad scale for parameter: " + name);
      q.q.assign(reinterpret_cast<const int8_t*>(rec->payload.data()),
                 reinterpret_cast<const int8_t*>(rec->payload.data()) + rec->payload.size());
      q.finish();
      m.q.emplace(name, std::move(q));
    } else {
      Tensor t(sh);
      std::memcpy(t.data.data(), rec->payload.data(), rec->payload.size());
      m.f32.emplace(name, std::move(t));
    }
  }
  return m;
}

// =============================================================================
// pinned reductions
// =============================================================================
namespace {

// P1
float warp_sum(const float* v, Index n) {
  float p[32];
  for (int l = 0; l < 32; ++l) {
    float s = 0.0f;
    for (Index j = l; j < n; j += 32) s = s + v[j];
    p[l] = s;
  }
  for (int off = 16; off > 0; off >>= 1) {
    float t[32];
    for (int l = 0; l < 32; ++l) t[l] = p[l] + p[l ^ off];
    std::memcpy(p, t, sizeof p);
  }
  return p[0];
}

// P3
inline float dot_seq(const float* a, const float* b, Index n) {
  float acc = 0.0f;
  for (Index c = 0; c < n; ++c) acc = acc + a[c] * b[c];
  return acc;
}

// One attention row (model.cpp:517-525, 642-651): s_j = dot(q, k_j) * scale
// (+ mask), softmax with max subtraction, ctx = sum_j p_j v_j (j ascending).
void attend_row(const float* q, const float* K, Index ldk, const float* V, Index ldv, Index n,
                Index dh, float scale, const float* mask_row, float* ctx) {
  static thread_local std::vector<float> s;
  s.resize(static_cast<size_t>(n));
  float mx = -INFINITY;
  for (Index j = 0; j < n; ++j) {
    float v = dot_seq(q, K + j * ldk, dh) * scale;
    if (mask_row) v = v + mask_row[j];
    s[j] = v;
    mx = std::max(mx, v);
  }
  for (Index j = 0; j < n; ++j) s[j] = orc_expf(s[j] - mx);
  const float sum = warp_sum(s.data(), n);
  for (Index j = 0; j < n; ++j) s[j] = s[j] / sum;
  // ctx[c] = sum over keys in ascending order of p_j * v_j[c] (the GPU's
  // lanes own columns and walk the keys; model.cpp:649-650 P.V).
  for (Index c = 0; c < dh; ++c) {
    float acc = 0.0f;
    for (Index j = 0; j < n; ++j) acc = acc + s[j] * V[j * ldv + c];
    ctx[c] = acc;
  }
}

// P5: c = a . w with w [k x n] row-major, k-ascending per element.
void gemm_f32(const float* a, const float* w, float* c, Index m, Index k, Index n) {
  for (Index i = 0; i < m; ++i) {
    float* cr = c + i * n;
    std::fill(cr, cr + n, 0.0f);
    const float* ar = a + i * k;
    for (Index kk = 0; kk < k; ++kk) {
      const float av = ar[kk];
      const float* wr = w + kk * n;
      for (Index j = 0; j < n; ++j) cr[j] = cr[j] + av * wr[j];
    }
  }
}

// Eigen-dot stand-in for gemm_nt (tensor.cpp:125-133): 8 interleaved partial
// sums (unpinned in the reference; fp32 is compared within tolerance).
inline float dot8(const float* a, const float* b, Index n) {
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  Index i = 0;
  for (; i + 8 <= n; i += 8)
    for (int u = 0; u < 8; ++u) acc[u] = acc[u] + a[i + u] * b[i + u];
  for (; i < n; ++i) acc[i & 7] = acc[i & 7] + a[i] * b[i];
  return ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
}

Tensor add(const Tensor& a, const Tensor& b) {  // tensor.cpp:220-238
  if (a.shape != b.shape) fail(kShape, "add: shape mismatch");
  Tensor o = a;
  for (size_t i = 0; i < o.data.size(); ++i) o.data[i] = o.data[i] + b.data[i];
  return o;
}

Tensor add_rowvec(const Tensor& a, const Tensor& r) {  // tensor.cpp:240-247
  if (r.numel() != a.cols()) fail(kShape, "add_rowvec: row length");
  Tensor o = a;
  for (Index i = 0; i < o.rows(); ++i)
    for (Index j = 0; j < o.cols(); ++j) o.row(i)[j] = o.row(i)[j] + r.data[j];
  return o;
}

Tensor relu(Tensor a) {  // tensor.cpp:314-318
  for (auto& v : a.data) v = v > 0.0f ? v : 0.0f;
  return a;
}

Tensor lookup(const Tensor& table, const std::vector<int>& ids) {  // tensor.cpp:448-460
  Index rows = table.rows(), dim = table.cols();
  Tensor out({static_cast<Index>(ids.size()), dim});
  for (size_t t = 0; t < ids.size(); ++t) {
    if (ids[t] < 0 || ids[t] >= rows)
      fail(kIndex, "embedding_lookup: id " + std::to_string(ids[t]) + " out of range [0," +
                       std::to_string(rows) + ")");
    std::memcpy(out.row(static_cast<Index>(t)), table.row(ids[t]), sizeof(float) * dim);
  }
  return out;
}

}  // namespace

// P1 per row (tensor.cpp:368-387): mu = sum/n; var = sum((x-mu)^2)/n;
// inv = 1/sqrt(var+eps); y = ((x-mu)*inv)*g + b.
Tensor layer_norm(const Tensor& x, const Tensor& g, const Tensor& b, float eps) {
  Index n = x.cols();
  if (g.numel() != n || b.numel() != n) fail(kShape, "layer_norm: gain/bias length vs normalized dim");
  Tensor out({x.rows(), n});
  std::vector<float> sq(static_cast<size_t>(n));
  for (Index i = 0; i < x.rows(); ++i) {
    const float* xr = x.row(i);
    const float mu = warp_sum(xr, n) / static_cast<float>(n);
    for (Index j = 0; j < n; ++j) {
      const float d = xr[j] - mu;
      sq[j] = d * d;
    }
    const float var = warp_sum(sq.data(), n) / static_cast<float>(n);
    const float inv = 1.0f / std::sqrt(var + eps);
    float* o = out.row(i);
    for (Index j = 0; j < n; ++j) o[j] = ((xr[j] - mu) * inv) * g.data[j] + b.data[j];
  }
  return out;
}

// =============================================================================
// executors (model.cpp:422-497)
// =============================================================================

Tensor F32Executor::linear(const Tensor& x, const std::string& name) const {
  const Tensor& w = m_->param(name);
  if (x.cols() != w.rows()) fail(kShape, "linear: shape mismatch " + name);
  Tensor out({x.rows(), w.cols()});
  gemm_f32(x.data.data(), w.data.data(), out.data.data(), x.rows(), x.cols(), w.cols());
  return out;
}

Tensor F32Executor::project_logits(const Tensor& x, const std::vector<int>* rows) const {
  const Tensor& e = m_->param("tgt_embed");
  Index n = rows ? static_cast<Index>(rows->size()) : e.rows();
  Tensor out({x.rows(), n});
  for (Index j = 0; j < n; ++j) {
    Index r = rows ? (*rows)[j] : j;
    if (r < 0 || r >= e.rows()) fail(kIndex, "project_logits: bad row");
    for (Index i = 0; i < x.rows(); ++i) out.row(i)[j] = dot8(x.row(i), e.row(r), x.cols());
  }
  return out;
}

Tensor F32Executor::embed_rows(const std::string& table, const std::vector<int>& ids) const {
  return lookup(m_->param(table), ids);
}

Int8Executor::Int8Executor(const QModel& m) : m_(&m) {
  for (const auto& [name, q] : m.q) {
    if (name == "tgt_embed") continue;
    QTensor t;
    t.shape = {q.cols(), q.rows()};
    t.scale = q.scale;
    t.q.resize(q.q.size());
    for (Index i = 0; i < q.rows(); ++i)
      for (Index j = 0; j < q.cols(); ++j) t.q[j * q.rows() + i] = q.q[i * q.cols() + j];
    wt_.emplace(name, std::move(t));
  }
}

// model.cpp:461-466: qmatmul(quantize(x), W) with one scale over all of x.
Tensor Int8Executor::linear(const Tensor& x, const std::string& name) const {
  auto it = wt_.find(name);
  if (it == wt_.end()) fail(kState, "no quantized parameter: " + name);
  const QTensor& wt = it->second;  // [n x k]
  if (x.cols() != wt.cols()) fail(kShape, "qmatmul: inner dimensions disagree");
  QTensor a = quantize(x);
  Tensor out({x.rows(), wt.rows()});
  qmatmul_nt(a, wt, nullptr, out.data.data());  // same int32 sums as qmatmul
  return out;
}

Tensor Int8Executor::project_logits(const Tensor& x, const std::vector<int>* rows) const {
  const QTensor& e = m_->q.at("tgt_embed");
  QTensor a = quantize(x);
  Index n = rows ? static_cast<Index>(rows->size()) : e.rows();
  Tensor out({x.rows(), n});
  qmatmul_nt(a, e, rows, out.data.data());
  return out;
}

// model.cpp:474-490: int8 tables dequantise as q / scale (a division).
Tensor Int8Executor::embed_rows(const std::string& table, const std::vector<int>& ids) const {
  auto qit = m_->q.find(table);
  if (qit != m_->q.end()) {
    const QTensor& q = qit->second;
    Tensor out({static_cast<Index>(ids.size()), q.cols()});
    for (size_t i = 0; i < ids.size(); ++i) {
      if (ids[i] < 0 || ids[i] >= q.rows()) fail(kIndex, "embed_rows: id out of range");
      for (Index j = 0; j < q.cols(); ++j)
        out.row(static_cast<Index>(i))[j] = static_cast<float>(q.q[ids[i] * q.cols() + j]) / q.scale;
    }
    return out;
  }
  return lookup(m_->f32.at(table), ids);
}

const Tensor& Int8Executor::f32_param(const std::string& name) const {
  auto it = m_->f32.find(name);
  if (it == m_->f32.end()) fail(kState, "no f32 parameter: " + name);
  return it->second;
}

// =============================================================================
// inference forward (model.cpp:499-672)
// =============================================================================
namespace {

Tensor norm_infer(const Executor& ex, const std::string& p, const Tensor& x) {
  return layer_norm(x, ex.f32_param(p + ".gain"), ex.f32_param(p + ".bias"), kLayerNormEps);
}

// model.cpp:509-528 (mask: the teacher-forced causal mask, model.cpp:24-29)
Tensor mha_infer(const Executor& ex, const std::string& p, const Tensor& q_in,
                 const Tensor& kv_in, bool causal) {
  const ModelConfig& c = ex.config();
  Index dh = c.d_model / c.num_heads, d = c.d_model;
  Tensor q = ex.linear(q_in, p + ".wq");
  Tensor k = ex.linear(kv_in, p + ".wk");
  Tensor v = ex.linear(kv_in, p + ".wv");
  const float scale = 1.0f / std::sqrt(static_cast<float>(dh));
  Tensor ctx({q.rows(), d});
  std::vector<float> mask;
  for (int h = 0; h < c.num_heads; ++h)
    for (Index i = 0; i < q.rows(); ++i) {
      const float* mrow = nullptr;
      if (causal) {
        mask.assign(static_cast<size_t>(k.rows()), 0.0f);
        for (Index j = i + 1; j < k.rows(); ++j) mask[j] = -1e9f;
        mrow = mask.data();
      }
      attend_row(q.row(i) + h * dh, k.data.data() + h * dh, d, v.data.data() + h * dh, d,
                 k.rows(), dh, scale, mrow, ctx.row(i) + h * dh);
    }
  return ex.linear(ctx, p + ".wo");
}

Tensor ffn_infer(const Executor& ex, const std::string& p, const Tensor& x) {
  Tensor h = relu(add_rowvec(ex.linear(x, p + ".w1"), ex.f32_param(p + ".b1")));
  return add_rowvec(ex.linear(h, p + ".w2"), ex.f32_param(p + ".b2"));
}

Tensor scale_t(Tensor a, float s) {
  for (auto& v : a.data) v = v * s;
  return a;
}

}  // namespace

// model.cpp:539-581
Tensor embed_source_infer(const Executor& ex, const std::vector<int>& ids,
                          const std::vector<std::vector<int>>& factor_ids) {
  const ModelConfig& c = ex.config();
  if (factor_ids.size() != c.factor_configs.size())
    fail(kShape, "embed_source: factor stream count vs config");
  for (const auto& f : factor_ids)
    if (f.size() != ids.size()) fail(kShape, "embed_source: factor stream not aligned with words");
  Index t = static_cast<Index>(ids.size());
  if (t > c.max_seq_len) fail(kValue, "embed_source: sequence too long");
  Tensor word = ex.embed_rows("src_embed", ids);
  std::vector<Tensor> factors;
  for (size_t i = 0; i < factor_ids.size(); ++i) {
    std::string table = c.factor_configs[i].share_with_word_embedding
                            ? "src_embed"
                            : "factor" + std::to_string(i) + "_embed";
    factors.push_back(ex.embed_rows(table, factor_ids[i]));
  }
  Tensor combined;
  if (factors.empty()) {
    combined = word;
  } else if (c.factor_configs.front().combine == FactorCombine::kConcat) {
    Index total = word.cols();
    for (auto& f : factors) total += f.cols();
    combined = Tensor({t, total});
    for (Index r = 0; r < t; ++r) {
      Index off = 0;
      std::memcpy(combined.row(r), word.row(r), sizeof(float) * word.cols());
      off += word.cols();
      for (auto& f : factors) {
        std::memcpy(combined.row(r) + off, f.row(r), sizeof(float) * f.cols());
        off += f.cols();
      }
    }
  } else {
    combined = word;
    for (auto& f : factors) combined = add(combined, f);
    if (c.factor_configs.front().combine == FactorCombine::kAverage)
      combined = scale_t(combined, 1.0f / (1.0f + factors.size()));
  }
  combined = scale_t(combined, std::sqrt(static_cast<float>(c.d_model)));
  for (Index r = 0; r < t; ++r)
    for (Index j = 0; j < c.d_model; ++j)
      combined.row(r)[j] = combined.row(r)[j] + ex.pos_enc()[r * c.d_model + j];
  return combined;
}

// model.cpp:583-596
Tensor encode_infer(const Executor& ex, const Tensor& src_embedded) {
  const ModelConfig& c = ex.config();
  if (src_embedded.rows() > c.max_seq_len) fail(kValue, "encode: sequence longer than max_seq_len");
  if (c.num_encoder_layers == 0) return src_embedded;
  Tensor x = src_embedded;
  for (int l = 0; l < c.num_encoder_layers; ++l) {
    std::string p = "enc" + std::to_string(l);
    Tensor a = norm_infer(ex, p + ".norm1", x);
    x = add(x, mha_infer(ex, p + ".attn", a, a, false));
    x = add(x, ffn_infer(ex, p + ".ffn", norm_infer(ex, p + ".norm2", x)));
  }
  return norm_infer(ex, "enc_final", x);
}

// model.cpp:598-612
DecoderState init_decoder(const Executor& ex, const Tensor& enc_out) {
  const ModelConfig& c = ex.config();
  DecoderState st;
  st.exec = &ex;
  st.self_k.resize(c.num_decoder_layers);
  st.self_v.resize(c.num_decoder_layers);
  for (int l = 0; l < c.num_decoder_layers; ++l) {
    std::string p = "dec" + std::to_string(l) + ".cross";
    st.cross_k.push_back(ex.linear(enc_out, p + ".wk"));
    st.cross_v.push_back(ex.linear(enc_out, p + ".wv"));
  }
  return st;
}

// model.cpp:614-672
Tensor decode_step(DecoderState& st, int prev, const std::vector<int>* shortlist) {
  const Executor& ex = *st.exec;
  const ModelConfig& c = ex.config();
  if (st.pos >= c.max_seq_len) fail(kValue, "decode_step: past max_seq_len");
  const Index d = c.d_model, dh = d / c.num_heads;
  const float scale = 1.0f / std::sqrt(static_cast<float>(dh));
  Tensor y = ex.embed_rows("tgt_embed", {prev});
  y = scale_t(y, std::sqrt(static_cast<float>(d)));
  for (Index j = 0; j < d; ++j) y.data[j] = y.data[j] + ex.pos_enc()[st.pos * d + j];
  for (int l = 0; l < c.num_decoder_layers; ++l) {
    std::string p = "dec" + std::to_string(l);
    Tensor a = norm_infer(ex, p + ".norm1", y);
    Tensor q = ex.linear(a, p + ".self.wq");
    Tensor k = ex.linear(a, p + ".self.wk");
    Tensor v = ex.linear(a, p + ".self.wv");
    auto& ks = st.self_k[l];
    auto& vs = st.self_v[l];
    ks.insert(ks.end(), k.data.begin(), k.data.end());
    vs.insert(vs.end(), v.data.begin(), v.data.end());
    const Index n = static_cast<Index>(ks.size()) / d;
    Tensor ctx({1, d});
    for (int h = 0; h < c.num_heads; ++h)
      attend_row(q.data.data() + h * dh, ks.data() + h * dh, d, vs.data() + h * dh, d, n, dh,
                 scale, nullptr, ctx.data.data() + h * dh);
    y = add(y, ex.linear(ctx, p + ".self.wo"));
    Tensor cq = ex.linear(norm_infer(ex, p + ".norm2", y), p + ".cross.wq");
    Tensor cctx({1, d});
    const Tensor& ck = st.cross_k[l];
    const Tensor& cv = st.cross_v[l];
    for (int h = 0; h < c.num_heads; ++h)
      attend_row(cq.data.data() + h * dh, ck.data.data() + h * dh, d, cv.data.data() + h * dh, d,
                 ck.rows(), dh, scale, nullptr, cctx.data.data() + h * dh);
    y = add(y, ex.linear(cctx, p + ".cross.wo"));
    y = add(y, ffn_infer(ex, p + ".ffn", norm_infer(ex, p + ".norm3", y)));
  }
  st.pos += 1;
  Tensor h = norm_infer(ex, "dec_final", y);
  return ex.project_logits(h, shortlist);
}

// model.cpp:382-418 (inference ops, dropout off)
Tensor forward_teacher_forced(const Model& m, const std::vector<int>& src,
                              const std::vector<std::vector<int>>& factors,
                              const std::vector<int>& tgt) {
  const ModelConfig& c = m.config;
  if (tgt.empty()) fail(kValue, "teacher forcing needs a target");
  Index tt = static_cast<Index>(tgt.size());
  if (tt > c.max_seq_len) fail(kValue, "target longer than max_seq_len");
  F32Executor ex(m);
  Tensor enc = encode_infer(ex, embed_source_infer(ex, src, factors));
  std::vector<int> tin(tgt.size());
  tin[0] = kBosId;
  for (size_t i = 1; i < tgt.size(); ++i) tin[i] = tgt[i - 1];
  Tensor y = scale_t(lookup(m.param("tgt_embed"), tin), std::sqrt(static_cast<float>(c.d_model)));
  for (Index r = 0; r < tt; ++r)
    for (Index j = 0; j < c.d_model; ++j) y.row(r)[j] = y.row(r)[j] + m.pe[r * c.d_model + j];
  for (int l = 0; l < c.num_decoder_layers; ++l) {
    std::string p = "dec" + std::to_string(l);
    Tensor n1 = norm_infer(ex, p + ".norm1", y);
    y = add(y, mha_infer(ex, p + ".self", n1, n1, true));
    y = add(y, mha_infer(ex, p + ".cross", norm_infer(ex, p + ".norm2", y), enc, false));
    y = add(y, ffn_infer(ex, p + ".ffn", norm_infer(ex, p + ".norm3", y)));
  }
  Tensor h = norm_infer(ex, "dec_final", y);
  return ex.project_logits(h, nullptr);
}

// =============================================================================
// beam search (decode.cpp:18-109)
// =============================================================================

float Hypothesis::normalized_score(float alpha) const {
  float len = static_cast<float>(tokens.size()) + 1.0f;
  return logprob / orc_powf((5.0f + len) / 6.0f, alpha);
}

// decode.cpp:25-30 in the P6 order: lse = log(sum exp(x - max)) + max, the sum
// taken per 32-column slice against the slice max and then rescaled.
std::vector<float> log_softmax_row(const float* x, int n) {
  const int nsub = (n + 31) / 32;
  std::vector<float> u(static_cast<size_t>(nsub));
  std::vector<float> m(static_cast<size_t>(nsub));
  float M = -INFINITY;
  for (int k = 0; k < nsub; ++k) {
    const int j0 = 32 * k, j1 = std::min(n, j0 + 32);
    float best = -INFINITY;
    bool any = false;
    for (int j = j0; j < j1; ++j)
      if (x[j] > best) {
        best = x[j];
        any = true;
      }
    float s = 0.0f;
    if (any)
      for (int j = j0; j < j1; ++j) s = s + orc_expf(x[j] - best);
    m[k] = best;
    u[k] = s;
    M = std::max(M, best);
  }
  for (int k = 0; k < nsub; ++k) u[k] = m[k] == -INFINITY ? 0.0f : u[k] * orc_expf(m[k] - M);
  // 128 thread partials (t sums k = t + 128 i), P1 butterfly per 32-thread
  // warp, then (W0 + W1) + (W2 + W3).
  float tp[128];
  for (int t = 0; t < 128; ++t) {
    float a = 0.0f;
    for (int k = t; k < nsub; k += 128) a = a + u[k];
    tp[t] = a;
  }
  float w[4];
  for (int j = 0; j < 4; ++j) {
    float* p = tp + 32 * j;
    for (int off = 16; off > 0; off >>= 1) {
      float tt[32];
      for (int l = 0; l < 32; ++l) tt[l] = p[l] + p[l ^ off];
      std::memcpy(p, tt, sizeof tt);
    }
    w[j] = p[0];
  }
  const float lse = orc_logf((w[0] + w[1]) + (w[2] + w[3])) + M;
  std::vector<float> e(static_cast<size_t>(n));
  for (int j = 0; j < n; ++j) e[j] = x[j] - lse;
  return e;
}

Hypothesis beam_search(const Executor& ex, const std::vector<int>& src_ids,
                       const std::vector<std::vector<int>>& factor_ids, const BeamConfig& cfg,
                       const std::vector<int>* shortlist) {
  if (cfg.beam_size < 1) fail(kUsage, "beam_search: beam size >= 1");
  if (src_ids.empty()) fail(kUsage, "beam_search: empty source");
  Tensor enc = encode_infer(ex, embed_source_infer(ex, src_ids, factor_ids));
  Hypothesis root;
  root.state = init_decoder(ex, enc);
  std::vector<Hypothesis> live{root};
  std::vector<Hypothesis> finished;
  const float alpha = cfg.length_penalty_alpha;
  struct Cand {
    size_t parent;
    int token;
    float logprob;
  };
  std::vector<Cand> cands;
  for (int step = 0; step < cfg.max_len && !live.empty(); ++step) {
    cands.clear();
    for (size_t h = 0; h < live.size(); ++h) {
      int prev = live[h].tokens.empty() ? kBosId : live[h].tokens.back();
      Tensor logits = decode_step(live[h].state, prev, shortlist);
      std::vector<float> logp = log_softmax_row(logits.data.data(), static_cast<int>(logits.cols()));
      for (size_t j = 0; j < logp.size(); ++j) {
        int tok = shortlist ? (*shortlist)[j] : static_cast<int>(j);
        cands.push_back({h, tok, live[h].logprob + logp[j]});
      }
    }
    // decode.cpp:64-69 total order; only the first beam_size are consumed, so
    // a partial sort yields the same prefix as the reference's full sort.
    auto cmp = [](const Cand& a, const Cand& b) {
      if (a.logprob != b.logprob) return a.logprob > b.logprob;
      if (a.parent != b.parent) return a.parent < b.parent;
      return a.token < b.token;
    };
    size_t take = std::min(cands.size(), static_cast<size_t>(cfg.beam_size));
    std::partial_sort(cands.begin(), cands.begin() + take, cands.end(), cmp);
    std::vector<Hypothesis> next;
    for (size_t i = 0; i < take; ++i) {
      const Cand& c = cands[i];
      Hypothesis h = live[c.parent];
      h.logprob = c.logprob;
      if (c.token == kEosId) {
        h.finished = true;
        h.state = DecoderState{};
        finished.push_back(std::move(h));
      } else {
        h.tokens.push_back(c.token);
        next.push_back(std::move(h));
      }
    }
    live = std::move(next);
  }
  auto by_norm = [alpha](const Hypothesis& a, const Hypothesis& b) {
    return a.normalized_score(alpha) < b.normalized_score(alpha);
  };
  if (!finished.empty()) {
    Hypothesis out = *std::max_element(finished.begin(), finished.end(), by_norm);
    out.state = DecoderState{};
    return out;
  }
  Hypothesis out = *std::max_element(live.begin(), live.end(), by_norm);
  out.truncated = true;
  out.state = DecoderState{};
  return out;
}

std::vector<int> prepare_source(const std::vector<int>& word_ids, int max_seq_len) {
  std::vector<int> src = word_ids;
  src.push_back(kEosId);
  if (static_cast<int>(src.size()) > max_seq_len) {
    src.resize(max_seq_len - 1);
    src.push_back(kEosId);
  }
  return src;
}

int derive_max_len(const BeamConfig& cfg, int src_len, int max_seq_len) {
  if (cfg.max_len > 0) return cfg.max_len;
  return std::min(max_seq_len, src_len * 2 + 5);
}

double percentile(std::vector<double> v, double p) {
  if (v.empty()) fail(kUsage, "percentile: empty list");
  if (p <= 0.0 || p > 100.0) fail(kUsage, "percentile: need 0 < p <= 100");
  std::sort(v.begin(), v.end());
  size_t rank = static_cast<size_t>(std::ceil(p / 100.0 * static_cast<double>(v.size())));
  if (rank == 0) rank = 1;
  return v[rank - 1];
}

}  // namespace orc
