// TEST INFRASTRUCTURE (oracle) -- not product code.
// extern "C" surface of the oracle for the Python tests (ctypes) and for the
// CPU baseline leg of bench.py. Mirrors the reference entry points cited in
// oracle.hpp.
#include <atomic>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>

#include "detmath.h"
#include "oracle.hpp"

using namespace orc;

namespace {

thread_local std::string g_err;
thread_local int g_code = 0;

struct Handle {
  std::unique_ptr<Model> f32;
  std::unique_ptr<QModel> q;
  std::unique_ptr<F32Executor> fx;
  std::unique_ptr<Int8Executor> ix;
  ModelConfig config() const { return f32 ? f32->config : q->config; }
  const Executor& exec(int int8) {
    if (int8) {
      if (!ix) {
        if (!q) q = std::make_unique<QModel>(quantize_model(*f32));
        ix = std::make_unique<Int8Executor>(*q);
      }
      return *ix;
    }
    if (!f32) fail(kState, "oracle: model has no f32 weights (int8 file)");
    if (!fx) fx = std::make_unique<F32Executor>(*f32);
    return *fx;
  }
};

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    g_code = e.code;
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    g_code = kState;
    return kState;
  }
}

std::vector<int> vec(const int* p, int n) { return std::vector<int>(p, p + n); }

void write_hyp(const Hypothesis& h, float alpha, int* out_tokens, int cap, int* out_len,
               float* out_lp, float* out_norm, int* out_flags) {
  int n = static_cast<int>(h.tokens.size());
  if (out_len) *out_len = n;
  if (out_tokens)
    for (int i = 0; i < std::min(n, cap); ++i) out_tokens[i] = h.tokens[i];
  if (out_lp) *out_lp = h.logprob;
  if (out_norm) *out_norm = h.normalized_score(alpha);
  if (out_flags) *out_flags = (h.finished ? 1 : 0) | (h.truncated ? 2 : 0);
}

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
int orc_last_error_code(void) { return g_code; }

void* orc_model_create(const char* cfg_json, uint64_t seed, int do_init) {
  Handle* h = nullptr;
  int rc = guard([&] {
    auto m = std::make_unique<Model>(make_model(ModelConfig::from_json(cfg_json)));
    if (do_init) init_params(*m, seed);
    h = new Handle();
    h->f32 = std::move(m);
  });
  return rc ? nullptr : h;
}

void* orc_model_load(const char* path) {
  Handle* h = nullptr;
  int rc = guard([&] {
    ParamFile pf = read_param_file(path);
    bool quant = false;
    for (const auto& p : pf.params) quant |= p.dtype == 1;
    h = new Handle();
    if (quant)
      h->q = std::make_unique<QModel>(load_quantized(path));
    else
      h->f32 = std::make_unique<Model>(load_params(path));
  });
  return rc ? nullptr : h;
}

void orc_model_free(void* h) { delete static_cast<Handle*>(h); }

int orc_model_save(void* hv, const char* path, int quantized) {
  return guard([&] {
    Handle* h = static_cast<Handle*>(hv);
    if (quantized) {
      h->exec(1);
      save_quantized(*h->q, path);
    } else {
      if (!h->f32) fail(kState, "no f32 weights");
      save_params(*h->f32, path);
    }
  });
}

int orc_model_config_json(void* hv, char* buf, size_t cap) {
  return guard([&] {
    std::string s = static_cast<Handle*>(hv)->config().to_json();
    if (s.size() + 1 > cap) fail(kShape, "buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

long long orc_param_count(void* hv) {
  Handle* h = static_cast<Handle*>(hv);
  return h->f32 ? static_cast<long long>(h->f32->param_count()) : -1;
}

// Copies a named f32 parameter (or the dequantised-free int8 payload as
// floats when only an int8 copy exists is not supported).
int orc_get_param(void* hv, const char* name, float* out, long long n) {
  return guard([&] {
    Handle* h = static_cast<Handle*>(hv);
    const Tensor& t = h->f32 ? h->f32->param(name) : h->q->f32.at(name);
    if (static_cast<long long>(t.data.size()) != n) fail(kShape, "size mismatch");
    std::memcpy(out, t.data.data(), sizeof(float) * n);
  });
}

int orc_set_param(void* hv, const char* name, const float* in, long long n) {
  return guard([&] {
    Handle* h = static_cast<Handle*>(hv);
    if (!h->f32) fail(kState, "no f32 weights");
    Tensor& t = h->f32->param(name);
    if (static_cast<long long>(t.data.size()) != n) fail(kShape, "size mismatch");
    std::memcpy(t.data.data(), in, sizeof(float) * n);
    h->q.reset();
    h->ix.reset();
    h->fx.reset();
  });
}

int orc_get_qparam(void* hv, const char* name, int8_t* out, long long n, float* scale) {
  return guard([&] {
    Handle* h = static_cast<Handle*>(hv);
    h->exec(1);
    const QTensor& q = h->q->q.at(name);
    if (static_cast<long long>(q.q.size()) != n) fail(kShape, "size mismatch");
    std::memcpy(out, q.q.data(), n);
    *scale = q.scale;
  });
}

int orc_pos_enc(void* hv, float* out) {
  return guard([&] {
    Handle* h = static_cast<Handle*>(hv);
    const auto& pe = h->f32 ? h->f32->pe : h->q->pe;
    std::memcpy(out, pe.data(), sizeof(float) * pe.size());
  });
}

int orc_beam_search(void* hv, int int8, const int* src, int n_src, int beam, int max_len,
                    float alpha, const int* shortlist, int n_short, int* out_tokens, int cap,
                    int* out_len, float* out_lp, float* out_norm, int* out_flags) {
  return guard([&] {
    Handle* h = static_cast<Handle*>(hv);
    BeamConfig cfg{beam, max_len, alpha};
    std::vector<int> sl;
    if (shortlist) sl = vec(shortlist, n_short);
    Hypothesis hyp = beam_search(h->exec(int8), vec(src, n_src), {}, cfg, shortlist ? &sl : nullptr);
    write_hyp(hyp, alpha, out_tokens, cap, out_len, out_lp, out_norm, out_flags);
  });
}

// Sentence-parallel batch (decode.cpp:370-398 parallel_sentences mode). Each
// sentence is already prepared (EOS appended); max_len <= 0 derives
// min(max_seq_len, 2|src|+5) per sentence (decode.cpp:352-355).
int orc_translate_batch(void* hv, int int8, const int* ids, const long long* off, int n,
                        int beam, int max_len, float alpha, int threads, int* out_tokens,
                        int stride, int* out_len, float* out_lp, float* out_norm,
                        int* out_flags, int* out_status) {
  return guard([&] {
    Handle* h = static_cast<Handle*>(hv);
    const Executor& ex = h->exec(int8);
    const int msl = h->config().max_seq_len;
    std::atomic<int> next{0};
    auto worker = [&] {
      for (int i = next++; i < n; i = next++) {
        std::vector<int> src = vec(ids + off[i], static_cast<int>(off[i + 1] - off[i]));
        BeamConfig cfg{beam, max_len, alpha};
        cfg.max_len = derive_max_len(cfg, static_cast<int>(src.size()), msl);
        try {
          Hypothesis hyp = beam_search(ex, src, {}, cfg, nullptr);
          write_hyp(hyp, alpha, out_tokens ? out_tokens + static_cast<long long>(i) * stride : nullptr,
                    stride, out_len ? out_len + i : nullptr, out_lp ? out_lp + i : nullptr,
                    out_norm ? out_norm + i : nullptr, out_flags ? out_flags + i : nullptr);
          if (out_status) out_status[i] = 0;
        } catch (const Error& e) {
          if (out_status) out_status[i] = e.code;
          if (out_len) out_len[i] = 0;
          if (out_flags) out_flags[i] = 4;
        }
      }
    };
    int nt = std::max(1, threads);
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(worker);
    worker();
    for (auto& t : pool) t.join();
  });
}

// decode_step logits along a forced prefix (BOS, forced[0], ...).
int orc_forced_logits(void* hv, int int8, const int* src, int n_src, const int* forced, int nf,
                      float* out) {
  return guard([&] {
    Handle* h = static_cast<Handle*>(hv);
    const Executor& ex = h->exec(int8);
    Tensor enc = encode_infer(ex, embed_source_infer(ex, vec(src, n_src), {}));
    DecoderState st = init_decoder(ex, enc);
    int prev = kBosId;
    const int V = ex.config().tgt_vocab_size;
    for (int t = 0; t < nf; ++t) {
      Tensor lg = decode_step(st, prev, nullptr);
      std::memcpy(out + static_cast<long long>(t) * V, lg.data.data(), sizeof(float) * V);
      prev = forced[t];
    }
  });
}

int orc_teacher_forced(void* hv, const int* src, int n_src, const int* tgt, int nt, float* out) {
  return guard([&] {
    Handle* h = static_cast<Handle*>(hv);
    if (!h->f32) fail(kState, "no f32 weights");
    Tensor lg = forward_teacher_forced(*h->f32, vec(src, n_src), {}, vec(tgt, nt));
    std::memcpy(out, lg.data.data(), sizeof(float) * lg.data.size());
  });
}

int orc_encode(void* hv, int int8, const int* src, int n_src, float* out) {
  return guard([&] {
    Handle* h = static_cast<Handle*>(hv);
    const Executor& ex = h->exec(int8);
    Tensor enc = encode_infer(ex, embed_source_infer(ex, vec(src, n_src), {}));
    std::memcpy(out, enc.data.data(), sizeof(float) * enc.data.size());
  });
}

// Source-factor variants: fids holds n_factors streams of n_src ids each
// (stream f at fids + f * n_src), aligned with src (model.cpp:539-581).
static std::vector<std::vector<int>> factor_streams(const int* fids, int n_factors, int n_src) {
  std::vector<std::vector<int>> f;
  for (int i = 0; i < n_factors; ++i)
    f.push_back(vec(fids + static_cast<long long>(i) * n_src, n_src));
  return f;
}

int orc_encode_factors(void* hv, int int8, const int* src, int n_src, const int* fids,
                       int n_factors, float* out) {
  return guard([&] {
    Handle* h = static_cast<Handle*>(hv);
    const Executor& ex = h->exec(int8);
    Tensor enc = encode_infer(
        ex, embed_source_infer(ex, vec(src, n_src), factor_streams(fids, n_factors, n_src)));
    std::memcpy(out, enc.data.data(), sizeof(float) * enc.data.size());
  });
}

int orc_beam_search_factors(void* hv, int int8, const int* src, int n_src, const int* fids,
                            int n_factors, int beam, int max_len, float alpha, int* out_tokens,
                            int cap, int* out_len, float* out_lp, float* out_norm,
                            int* out_flags) {
  return guard([&] {
    Handle* h = static_cast<Handle*>(hv);
    BeamConfig cfg{beam, max_len, alpha};
    Hypothesis hyp = beam_search(h->exec(int8), vec(src, n_src),
                                 factor_streams(fids, n_factors, n_src), cfg, nullptr);
    write_hyp(hyp, alpha, out_tokens, cap, out_len, out_lp, out_norm, out_flags);
  });
}

int orc_quantize(const float* x, long long n, int8_t* q, float* scale) {
  return guard([&] {
    QTensor t = quantize(x, {n});
    std::memcpy(q, t.q.data(), n);
    *scale = t.scale;
  });
}

int orc_qmatmul(const int8_t* a, float sa, const int8_t* b, float sb, int m, int k, int n,
                float* c) {
  return guard([&] {
    QTensor qa, qb;
    qa.shape = {m, k};
    qa.q.assign(a, a + static_cast<long long>(m) * k);
    qa.scale = sa;
    qb.shape = {k, n};
    qb.q.assign(b, b + static_cast<long long>(k) * n);
    qb.scale = sb;
    qmatmul(qa, qb, c);
  });
}

int orc_layer_norm(const float* x, int rows, int n, const float* g, const float* b, float* out) {
  return guard([&] {
    Tensor tx({rows, n}), tg({n}), tb({n});
    std::memcpy(tx.data.data(), x, sizeof(float) * rows * n);
    std::memcpy(tg.data.data(), g, sizeof(float) * n);
    std::memcpy(tb.data.data(), b, sizeof(float) * n);
    Tensor y = layer_norm(tx, tg, tb, kLayerNormEps);
    std::memcpy(out, y.data.data(), sizeof(float) * rows * n);
  });
}

int orc_log_softmax(const float* x, int n, float* out) {
  return guard([&] {
    auto v = log_softmax_row(x, n);
    std::memcpy(out, v.data(), sizeof(float) * n);
  });
}

float orc_det_expf(float x) { return orc_expf(x); }
float orc_det_logf(float x) { return orc_logf(x); }
float orc_det_powf(float b, float a) { return orc_powf(b, a); }

float orc_normalized_score(const int n_tokens, float logprob, float alpha) {
  Hypothesis h;
  h.tokens.resize(n_tokens);
  h.logprob = logprob;
  return h.normalized_score(alpha);
}

int orc_percentile(const double* v, int n, double p, double* out) {
  return guard([&] { *out = percentile(std::vector<double>(v, v + n), p); });
}

int orc_prepare_source(const int* words, int n, int max_seq_len, int* out, int* out_n) {
  return guard([&] {
    auto s = prepare_source(vec(words, n), max_seq_len);
    std::memcpy(out, s.data(), sizeof(int) * s.size());
    *out_n = static_cast<int>(s.size());
  });
}

}  // extern "C"
