// Model / search entry points of the C ABI (include/minimt_gpu.h).
#include <algorithm>
#include <cstring>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/minimt_gpu.h"
#include "capi_util.hpp"
#include "engine.hpp"

using namespace mtg;

struct mtg_model {
  std::unique_ptr<Engine> eng;
};

namespace {

std::vector<std::vector<int>> csr(const int32_t* ids, const int64_t* off, int n) {
  if (n < 0) fail(kShapeError, "negative sentence count");
  std::vector<std::vector<int>> out(n);
  for (int i = 0; i < n; ++i) {
    if (off[i + 1] < off[i]) fail(kShapeError, "source offsets must be non-decreasing");
    out[i].assign(ids + off[i], ids + off[i + 1]);
  }
  return out;
}

Engine& engine(mtg_model* m) {
  if (!m || !m->eng) fail(kStateError, "null model handle");
  return *m->eng;
}

}  // namespace

extern "C" {

int mtg_model_load(const char* path, int precision, int device, mtg_model** out) {
  return guarded([&] {
    *out = nullptr;
    auto m = std::make_unique<mtg_model>();
    m->eng = std::make_unique<Engine>(load_sqnt(path), precision, device);
    *out = m.release();
  });
}

int mtg_model_create(const char* config_json, uint64_t seed, int precision, int device,
                     mtg_model** out) {
  return guarded([&] {
    *out = nullptr;
    ModelConfig c = ModelConfig::from_json(config_json);
    auto m = std::make_unique<mtg_model>();
    m->eng = std::make_unique<Engine>(make_random_model(c, seed), precision, device);
    *out = m.release();
  });
}

int mtg_model_save(const mtg_model* m, const char* path) {
  return guarded([&] {
    if (!m || !m->eng) fail(kStateError, "null model handle");
    save_sqnt(m->eng->host_model(), path);
  });
}

void mtg_model_free(mtg_model* m) { delete m; }

int mtg_model_config_json(const mtg_model* m, char* buf, size_t cap) {
  return guarded([&] {
    if (!m || !m->eng) fail(kStateError, "null model handle");
    const std::string s = m->eng->config().to_json();
    if (s.size() + 1 > cap) fail(kShapeError, "config buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

int mtg_model_precision(const mtg_model* m) { return m && m->eng ? m->eng->precision() : -1; }

}  // extern "C"

namespace {

// Factor streams of sentence s: stream f is factor_ids[f * total + off[s] ..).
Engine::FactorStreams factor_streams(const int32_t* factor_ids, int n_factors,
                                     const int64_t* off, int n) {
  Engine::FactorStreams fs(n);
  if (!factor_ids || n_factors <= 0) return fs;
  const int64_t total = off[n];
  for (int s = 0; s < n; ++s)
    for (int f = 0; f < n_factors; ++f)
      fs[s].emplace_back(factor_ids + f * total + off[s], factor_ids + f * total + off[s + 1]);
  return fs;
}

int translate_impl(mtg_model* m, const int32_t* src_ids, const int64_t* src_offsets,
                   int n_sentences, const int32_t* factor_ids, int n_factors,
                   const int32_t* sl_ids, const int64_t* sl_offsets,
                   const mtg_beam_config* cfg, int32_t* out_tokens, int out_stride,
                   int32_t* out_len, float* out_logprob, float* out_norm_score,
                   uint32_t* out_flags, int32_t* out_status) {
  return guarded([&] {
    Engine& e = engine(m);
    std::lock_guard<std::mutex> lock(e.mutex());
    if (!cfg) fail(kUsageError, "null beam config");
    if (cfg->beam_size < 1) fail(kUsageError, "beam_search: beam size >= 1");
    if (out_tokens && out_stride < e.config().max_seq_len)
      fail(kShapeError, "out_stride must be >= max_seq_len");
    auto srcs = csr(src_ids, src_offsets, n_sentences);
    const bool has_f = factor_ids && n_factors > 0;
    const Engine::FactorStreams all_f =
        factor_streams(factor_ids, n_factors, src_offsets, n_sentences);
    BeamConfigC bc{cfg->beam_size, cfg->max_len, cfg->length_penalty_alpha};
    // Length-bucketed batching: stable sort by source length so a
    // device batch runs for about as many steps as each of its sentences.
    std::vector<int> order(n_sentences);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(),
                     [&](int a, int b) { return srcs[a].size() < srcs[b].size(); });
    const int per = cfg->max_batch > 0 ? cfg->max_batch : std::max(n_sentences, 1);
    // Sentences with a shortlist (non-empty CSR entry) and without one run
    // as separate device batches (the projection differs).
    auto has_sl = [&](int s) { return sl_ids && sl_offsets && sl_offsets[s + 1] > sl_offsets[s]; };
    std::stable_partition(order.begin(), order.end(), [&](int s) { return !has_sl(s); });
    const int n_plain = static_cast<int>(
        std::count_if(order.begin(), order.end(), [&](int s) { return !has_sl(s); }));
    std::vector<std::pair<int, int>> chunks;
    for (int b0 = 0; b0 < n_plain; b0 += per) chunks.push_back({b0, std::min(n_plain, b0 + per)});
    for (int b0 = n_plain; b0 < n_sentences; b0 += per)
      chunks.push_back({b0, std::min(n_sentences, b0 + per)});
    for (const auto& [b0, b1] : chunks) {
      std::vector<std::vector<int>> chunk, chunk_sl;
      Engine::FactorStreams chunk_f;
      for (int i = b0; i < b1; ++i) {
        chunk.push_back(srcs[order[i]]);
        if (has_f) chunk_f.push_back(all_f[order[i]]);
        if (b0 >= n_plain)
          chunk_sl.emplace_back(sl_ids + sl_offsets[order[i]], sl_ids + sl_offsets[order[i] + 1]);
      }
      std::vector<SentenceResult> res = e.translate_batch(
          chunk, bc, has_f ? &chunk_f : nullptr, b0 >= n_plain ? &chunk_sl : nullptr);
      for (int i = b0; i < b1; ++i) {
        const int s = order[i];
        const SentenceResult& r = res[i - b0];
        const int n = static_cast<int>(r.tokens.size());
        if (out_tokens)
          std::copy(r.tokens.begin(), r.tokens.end(), out_tokens + int64_t(s) * out_stride);
        if (out_len) out_len[s] = n;
        if (out_logprob) out_logprob[s] = r.logprob;
        if (out_norm_score) out_norm_score[s] = r.norm;
        if (out_flags) out_flags[s] = r.flags;
        if (out_status) out_status[s] = r.status;
      }
    }
  });
}

}  // namespace

extern "C" {

int mtg_translate(mtg_model* m, const int32_t* src_ids, const int64_t* src_offsets,
                  int n_sentences, const mtg_beam_config* cfg, int32_t* out_tokens,
                  int out_stride, int32_t* out_len, float* out_logprob, float* out_norm_score,
                  uint32_t* out_flags, int32_t* out_status) {
  return translate_impl(m, src_ids, src_offsets, n_sentences, nullptr, 0, nullptr, nullptr, cfg,
                        out_tokens, out_stride, out_len, out_logprob, out_norm_score, out_flags,
                        out_status);
}

int mtg_translate_factors(mtg_model* m, const int32_t* src_ids, const int64_t* src_offsets,
                          int n_sentences, const int32_t* factor_ids, int n_factors,
                          const mtg_beam_config* cfg, int32_t* out_tokens, int out_stride,
                          int32_t* out_len, float* out_logprob, float* out_norm_score,
                          uint32_t* out_flags, int32_t* out_status) {
  return translate_impl(m, src_ids, src_offsets, n_sentences, factor_ids, n_factors, nullptr,
                        nullptr, cfg, out_tokens, out_stride, out_len, out_logprob,
                        out_norm_score, out_flags, out_status);
}

int mtg_translate_ex(mtg_model* m, const int32_t* src_ids, const int64_t* src_offsets,
                     int n_sentences, const int32_t* factor_ids, int n_factors,
                     const int32_t* shortlist_ids, const int64_t* shortlist_offsets,
                     const mtg_beam_config* cfg, int32_t* out_tokens, int out_stride,
                     int32_t* out_len, float* out_logprob, float* out_norm_score,
                     uint32_t* out_flags, int32_t* out_status) {
  return translate_impl(m, src_ids, src_offsets, n_sentences, factor_ids, n_factors,
                        shortlist_ids, shortlist_offsets, cfg, out_tokens, out_stride, out_len,
                        out_logprob, out_norm_score, out_flags, out_status);
}

int mtg_encode_factors(mtg_model* m, const int32_t* src_ids, const int64_t* src_offsets,
                       int n_sentences, const int32_t* factor_ids, int n_factors, float* out) {
  return guarded([&] {
    Engine& e = engine(m);
    std::lock_guard<std::mutex> lock(e.mutex());
    const Engine::FactorStreams fs =
        factor_streams(factor_ids, n_factors, src_offsets, n_sentences);
    e.encode(csr(src_ids, src_offsets, n_sentences), out,
             factor_ids && n_factors > 0 ? &fs : nullptr);
  });
}

int mtg_forced_logits(mtg_model* m, const int32_t* src_ids, const int64_t* src_offsets,
                      int n_sentences, const int32_t* forced, int n_forced, float* out_logits) {
  return guarded([&] {
    Engine& e = engine(m);
    std::lock_guard<std::mutex> lock(e.mutex());
    e.forced_logits(csr(src_ids, src_offsets, n_sentences), forced, n_forced, out_logits);
  });
}

int mtg_encode(mtg_model* m, const int32_t* src_ids, const int64_t* src_offsets,
               int n_sentences, float* out) {
  return guarded([&] {
    Engine& e = engine(m);
    std::lock_guard<std::mutex> lock(e.mutex());
    e.encode(csr(src_ids, src_offsets, n_sentences), out);
  });
}

int mtg_stage_sources(mtg_model* m, const int32_t* src_ids, const int64_t* src_offsets,
                      int n_sentences) {
  return guarded([&] {
    Engine& e = engine(m);
    std::lock_guard<std::mutex> lock(e.mutex());
    e.stage(csr(src_ids, src_offsets, n_sentences));
  });
}

int mtg_translate_staged(mtg_model* m, const mtg_beam_config* cfg) {
  return guarded([&] {
    Engine& e = engine(m);
    std::lock_guard<std::mutex> lock(e.mutex());
    if (!cfg) fail(kUsageError, "null beam config");
    e.run_staged(BeamConfigC{cfg->beam_size, cfg->max_len, cfg->length_penalty_alpha});
  });
}

int64_t mtg_last_launch_count(const mtg_model* m) {
  return m && m->eng ? m->eng->last_launches() : -1;
}

void* mtg_model_stream(const mtg_model* m) {
  return m && m->eng ? static_cast<void*>(m->eng->stream()) : nullptr;
}

int mtg_time_kernel(mtg_model* m, int kernel, int iters, float* ms_per_launch,
                    double* bytes_per_launch, double* flops_per_launch) {
  return guarded([&] {
    Engine& e = engine(m);
    std::lock_guard<std::mutex> lock(e.mutex());
    e.time_kernel(kernel, iters, ms_per_launch, bytes_per_launch, flops_per_launch);
  });
}

int mtg_diag_report(mtg_model* m, char* buf, size_t buf_size) {
  return guarded([&] {
    Engine& e = engine(m);
    std::lock_guard<std::mutex> lock(e.mutex());
    const std::string r = e.diag_report();
    if (!buf || buf_size == 0) fail(kUsageError, "diag_report: empty buffer");
    const size_t n = std::min(buf_size - 1, r.size());
    std::memcpy(buf, r.data(), n);
    buf[n] = '\0';
  });
}

}  // extern "C"
