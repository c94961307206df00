// minimt_gpu.hpp -- header-only C++ shim over the C ABI (minimt_gpu.h) that
// re-exposes the reference's decode API (proj/include/minimt/decode.hpp,
// model.hpp, errors.hpp) so callers of minimt::beam_search /
// translate_corpus switch by changing the namespace and the executor type:
//
//   minimt::F32Executor ex(model);                 // reference
//   minimt::gpu::GpuExecutor ex(path, MTG_PREC_F32);  // this library
//   Hypothesis h = beam_search(ex, src_ids, {}, cfg);
//
// Error behaviour mirrors errors.hpp: status codes are rethrown as the same
// exception types. The text layer (Vocabulary, tokenize) stays host-side; the
// id-level batched entry point is translate_ids().
#ifndef MINIMT_GPU_HPP_
#define MINIMT_GPU_HPP_

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <fstream>
#include <functional>
#include <map>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "minimt_gpu.h"

namespace minimt {
namespace gpu {

// ---- errors.hpp:8-34 --------------------------------------------------------
struct ShapeError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ValueError : std::runtime_error { using std::runtime_error::runtime_error; };
struct IndexError : std::out_of_range { using std::out_of_range::out_of_range; };
struct StateError : std::logic_error { using std::logic_error::logic_error; };
struct FormatError : std::runtime_error { using std::runtime_error::runtime_error; };
struct UsageError : std::runtime_error { using std::runtime_error::runtime_error; };
struct IoError : std::runtime_error { using std::runtime_error::runtime_error; };
struct CudaError : std::runtime_error { using std::runtime_error::runtime_error; };

[[noreturn]] inline void throw_status(int rc, const std::string& msg) {
  switch (rc) {
    case MTG_SHAPE_ERROR: throw ShapeError(msg);
    case MTG_VALUE_ERROR: throw ValueError(msg);
    case MTG_INDEX_ERROR: throw IndexError(msg);
    case MTG_STATE_ERROR: throw StateError(msg);
    case MTG_FORMAT_ERROR: throw FormatError(msg);
    case MTG_USAGE_ERROR: throw UsageError(msg);
    case MTG_IO_ERROR: throw IoError(msg);
    default: throw CudaError(msg);
  }
}
inline void check(int rc) {
  if (rc != MTG_OK) throw_status(rc, mtg_last_error());
}

constexpr int kPadId = 0, kUnkId = 1, kBosId = 2, kEosId = 3;  // model.hpp:16-19

// ---- decode.hpp:15-31 ----------------------------------------------------------
struct Hypothesis {
  std::vector<int> tokens;
  float logprob = 0.0f;
  bool finished = false;
  bool truncated = false;
  float normalized = 0.0f;  // normalized_score(alpha) as computed on device
  float normalized_score(float alpha) const {
    const float len = static_cast<float>(tokens.size()) + 1.0f;
    return logprob / std::pow((5.0f + len) / 6.0f, alpha);
  }
};

struct BeamConfig {
  int beam_size = 4;
  int max_len = 64;
  float length_penalty_alpha = 1.0f;
};

// ---- the Executor plugin point (model.hpp:113-171) -----------------------------
// Owns a device-resident model. MTG_PREC_F32 ~ F32Executor, MTG_PREC_INT8 ~
// Int8Executor (int8 files always decode int8), MTG_PREC_BF16 extension.
class GpuExecutor {
 public:
  GpuExecutor(const std::string& sqnt_path, int precision, int device = 0) {
    check(mtg_model_load(sqnt_path.c_str(), precision, device, &m_));
  }
  GpuExecutor(const std::string& config_json, uint64_t seed, int precision, int device = 0) {
    check(mtg_model_create(config_json.c_str(), seed, precision, device, &m_));
  }
  ~GpuExecutor() { mtg_model_free(m_); }
  GpuExecutor(const GpuExecutor&) = delete;
  GpuExecutor& operator=(const GpuExecutor&) = delete;

  mtg_model* handle() const { return m_; }
  int precision() const { return mtg_model_precision(m_); }
  std::string config_json() const {
    std::string buf(4096, '\0');
    check(mtg_model_config_json(m_, buf.data(), buf.size()));
    return std::string(buf.c_str());
  }
  int max_seq_len() const {
    const std::string j = config_json();
    const auto p = j.find("\"max_seq_len\":");
    return p == std::string::npos ? 128 : std::stoi(j.substr(p + 14));
  }
  void save(const std::string& path) const { check(mtg_model_save(m_, path.c_str())); }

  // encode_infer(embed_source_infer(src, factors)) (model.cpp:539-596): the
  // encoder output rows [|src| x d_model], row-major.
  std::vector<float> encode(const std::vector<int>& src,
                            const std::vector<std::vector<int>>& factor_ids = {}) const {
    const int64_t off[2] = {0, static_cast<int64_t>(src.size())};
    const std::string cfg = config_json();
    const auto p = cfg.find("\"d_model\":");
    const int d = std::stoi(cfg.substr(p + 10));
    std::vector<int32_t> block;
    for (const auto& f : factor_ids) {
      if (f.size() != src.size()) throw ShapeError("embed_source: factor stream not aligned with words");
      block.insert(block.end(), f.begin(), f.end());
    }
    std::vector<float> out(src.size() * static_cast<size_t>(d));
    check(mtg_encode_factors(m_, src.data(), off, 1, block.empty() ? nullptr : block.data(),
                             static_cast<int>(factor_ids.size()), out.data()));
    return out;
  }

  // decode_step along a forced prefix (model.cpp:614-672): logits per step.
  std::vector<float> forced_logits(const std::vector<int>& src,
                                   const std::vector<int>& forced) const {
    const int64_t off[2] = {0, static_cast<int64_t>(src.size())};
    std::string cfg = config_json();
    const auto p = cfg.find("\"tgt_vocab_size\":");
    const int V = std::stoi(cfg.substr(p + 17));
    std::vector<float> out(forced.size() * static_cast<size_t>(V));
    check(mtg_forced_logits(m_, src.data(), off, 1, forced.data(),
                            static_cast<int>(forced.size()), out.data()));
    return out;
  }

 private:
  mtg_model* m_ = nullptr;
};

// Batched id-level search: one call, many sentences (each ending with EOS).
// Per-sentence failures come back as empty hypotheses with status != 0.
struct BatchResult {
  std::vector<Hypothesis> hyps;
  std::vector<int> status;
};

// Per sentence: the model's source-factor id streams, each aligned with the
// sentence's ids (EOS position included).
using FactorStreams = std::vector<std::vector<std::vector<int>>>;

inline BatchResult translate_ids(const GpuExecutor& ex,
                                 const std::vector<std::vector<int>>& sources,
                                 const BeamConfig& config, int max_batch = 0,
                                 const FactorStreams* factors = nullptr,
                                 const std::vector<std::vector<int>>* shortlists = nullptr) {
  std::vector<int32_t> ids;
  std::vector<int64_t> off{0};
  for (const auto& s : sources) {
    ids.insert(ids.end(), s.begin(), s.end());
    off.push_back(static_cast<int64_t>(ids.size()));
  }
  const int n = static_cast<int>(sources.size());
  const int T = ex.max_seq_len();
  std::vector<int32_t> toks(static_cast<size_t>(std::max(n, 1)) * T), len(std::max(n, 1)),
      status(std::max(n, 1));
  std::vector<float> lp(std::max(n, 1)), norm(std::max(n, 1));
  std::vector<uint32_t> flags(std::max(n, 1));
  mtg_beam_config c{config.beam_size, config.max_len, config.length_penalty_alpha, max_batch};
  std::vector<int32_t> block;
  int nf = 0;
  if (factors) {  // [F][total] block aligned with ids (minimt_gpu.h)
    if (static_cast<int>(factors->size()) != n)
      throw ShapeError("factor streams: one entry per sentence");
    nf = n ? static_cast<int>((*factors)[0].size()) : 0;
    block.assign(static_cast<size_t>(std::max(nf, 1)) * std::max<size_t>(ids.size(), 1), 0);
    for (int i = 0; i < n; ++i) {
      if (static_cast<int>((*factors)[i].size()) != nf)
        throw ShapeError("factor streams: every sentence needs the same stream count");
      for (int f = 0; f < nf; ++f) {
        const auto& st = (*factors)[i][f];
        if (static_cast<int64_t>(st.size()) != off[i + 1] - off[i])
          throw ShapeError("embed_source: factor stream not aligned with words");
        std::copy(st.begin(), st.end(), block.begin() + f * ids.size() + off[i]);
      }
    }
  }
  std::vector<int32_t> sl_ids;
  std::vector<int64_t> sl_off{0};
  if (shortlists) {  // CSR; an empty list decodes over the full vocabulary
    if (static_cast<int>(shortlists->size()) != n) throw ShapeError("one shortlist per sentence");
    for (const auto& l : *shortlists) {
      sl_ids.insert(sl_ids.end(), l.begin(), l.end());
      sl_off.push_back(static_cast<int64_t>(sl_ids.size()));
    }
    if (sl_ids.empty()) sl_ids.push_back(0);
  }
  check(mtg_translate_ex(ex.handle(), ids.data(), off.data(), n, factors ? block.data() : nullptr,
                         nf, shortlists ? sl_ids.data() : nullptr,
                         shortlists ? sl_off.data() : nullptr, &c, toks.data(), T, len.data(),
                         lp.data(), norm.data(), flags.data(), status.data()));
  BatchResult r;
  for (int i = 0; i < n; ++i) {
    Hypothesis h;
    h.tokens.assign(toks.begin() + static_cast<size_t>(i) * T,
                    toks.begin() + static_cast<size_t>(i) * T + len[i]);
    h.logprob = lp[i];
    h.normalized = norm[i];
    h.finished = flags[i] & MTG_HYP_FINISHED;
    h.truncated = flags[i] & MTG_HYP_TRUNCATED;
    r.hyps.push_back(std::move(h));
    r.status.push_back(status[i]);
  }
  return r;
}

// decode.hpp:35-38.
inline Hypothesis beam_search(const GpuExecutor& ex, const std::vector<int>& src_ids,
                              const std::vector<std::vector<int>>& factor_ids,
                              const BeamConfig& config,
                              const std::vector<int>* shortlist = nullptr) {
  if (config.beam_size < 1) throw UsageError("beam_search: beam size >= 1");
  if (src_ids.empty()) throw UsageError("beam_search: empty source");
  if (config.max_len <= 0) {
    // decode.cpp:48-108 with max_len <= 0: the source is still encoded (its
    // checks throw as in the reference), no search step runs, and the
    // unfinished root hypothesis comes back truncated. (The C ABI's
    // max_len <= 0 means "derive 2|src|+5", which is translate_one's rule,
    // decode.cpp:352-355, not beam_search's.)
    ex.encode(src_ids, factor_ids);
    Hypothesis root;
    root.truncated = true;
    root.normalized = root.normalized_score(config.length_penalty_alpha);
    return root;
  }
  const FactorStreams fs{factor_ids};
  const std::vector<std::vector<int>> sl{shortlist ? *shortlist : std::vector<int>{}};
  BatchResult r = translate_ids(ex, {src_ids}, config, 0, &fs, shortlist ? &sl : nullptr);
  if (r.status[0] != MTG_OK) throw_status(r.status[0], "beam_search failed");
  return r.hyps[0];
}

// ---- lexical shortlist (decode.cpp:113-199) --------------------------------------
// Source id -> target candidates ranked by co-occurrence count (desc, id asc).
struct ShortlistTable {
  std::map<int, std::vector<std::pair<int, long>>> candidates;

  void save(const std::string& path) const {  // "s t:c t:c ..." per line
    std::ofstream f(path, std::ios::trunc);
    if (!f) throw IoError("cannot write shortlist table: " + path);
    for (const auto& [s, ranked] : candidates) {
      f << s;
      for (const auto& [t, c] : ranked) f << ' ' << t << ':' << c;
      f << '\n';
    }
  }
  static ShortlistTable load(const std::string& path) {
    std::ifstream f(path);
    if (!f) throw IoError("cannot read shortlist table: " + path);
    ShortlistTable table;
    std::string line;
    while (std::getline(f, line)) {
      if (line.empty()) continue;
      std::istringstream ss(line);
      int s;
      ss >> s;
      std::string entry;
      auto& ranked = table.candidates[s];
      while (ss >> entry) {
        const auto colon = entry.find(':');
        if (colon == std::string::npos) throw FormatError("bad shortlist entry: " + entry);
        ranked.emplace_back(std::stoi(entry.substr(0, colon)), std::stol(entry.substr(colon + 1)));
      }
    }
    return table;
  }
};

// Merged candidates of the source ids (best count per target), ranked, plus
// the four reserved ids, cut at k; sorted ascending. k <= 0 or k >= V: all ids.
inline std::vector<int> build_shortlist(const ShortlistTable& table, const std::vector<int>& src_ids,
                                        int k, int tgt_vocab_size) {
  std::vector<int> out;
  if (k <= 0 || k >= tgt_vocab_size) {
    out.resize(tgt_vocab_size);
    for (int i = 0; i < tgt_vocab_size; ++i) out[i] = i;
    return out;
  }
  std::map<int, long> merged;
  for (int s : src_ids) {
    const auto it = table.candidates.find(s);
    if (it == table.candidates.end()) continue;
    for (const auto& [t, c] : it->second) merged[t] = std::max(merged[t], c);
  }
  std::vector<std::pair<int, long>> ranked(merged.begin(), merged.end());
  std::sort(ranked.begin(), ranked.end(), [](const auto& a, const auto& b) {
    return a.second != b.second ? a.second > b.second : a.first < b.first;
  });
  std::set<int> result{kPadId, kUnkId, kBosId, kEosId};
  for (const auto& [t, c] : ranked) {
    if (static_cast<int>(result.size()) >= k) break;
    if (t < tgt_vocab_size) result.insert(t);
  }
  return std::vector<int>(result.begin(), result.end());
}

// ---- decode.hpp:81-113 ------------------------------------------------------------
struct LatencyReport {
  std::vector<double> durations_s;
  long output_tokens = 0;
  double total_time_s = 0.0;
  int count() const { return static_cast<int>(durations_s.size()); }
  double percentile_ms(double p) const {  // eval.cpp:120-128 nearest rank
    if (durations_s.empty()) return 0.0;
    std::vector<double> v = durations_s;
    std::sort(v.begin(), v.end());
    size_t rank = static_cast<size_t>(std::ceil(p / 100.0 * static_cast<double>(v.size())));
    if (rank == 0) rank = 1;
    return v[rank - 1] * 1000.0;
  }
  double p50_ms() const { return percentile_ms(50.0); }
  double p90_ms() const { return percentile_ms(90.0); }
  double mean_ms() const {
    if (durations_s.empty()) return 0.0;
    double s = 0.0;
    for (double d : durations_s) s += d;
    return s / static_cast<double>(durations_s.size()) * 1000.0;
  }
  double tokens_per_sec() const { return total_time_s > 0.0 ? output_tokens / total_time_s : 0.0; }
};

using Clock = std::function<double()>;
inline Clock steady_clock_seconds() {
  return [] {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
        .count();
  };
}

// translate_corpus on ids (decode.cpp:363-419 after tokenisation): sequential
// batch-1 mode records per-sentence latency; batch_sentences > 1 runs
// length-bucketed device batches and records only the total time. Failed
// sentences yield empty hypotheses, like the reference's empty lines.
inline std::vector<Hypothesis> translate_corpus_ids(const GpuExecutor& ex,
                                                    const std::vector<std::vector<int>>& words,
                                                    const BeamConfig& beam,
                                                    LatencyReport* report = nullptr,
                                                    int batch_sentences = 1, Clock clock = {}) {
  if (!clock) clock = steady_clock_seconds();
  const int msl = ex.max_seq_len();
  std::vector<std::vector<int>> srcs;
  for (const auto& w : words) {  // translate_one: append EOS, truncate keeping EOS
    std::vector<int> s = w;
    s.push_back(kEosId);
    if (static_cast<int>(s.size()) > msl) {
      s.resize(msl - 1);
      s.push_back(kEosId);
    }
    srcs.push_back(std::move(s));
  }
  BeamConfig cfg = beam;  // max_len <= 0: derived per sentence on device
  std::vector<Hypothesis> out(srcs.size());
  if (batch_sentences > 1) {
    const double t0 = clock();
    BatchResult r = translate_ids(ex, srcs, cfg, batch_sentences);
    for (size_t i = 0; i < srcs.size(); ++i)
      if (r.status[i] == MTG_OK) out[i] = r.hyps[i];
    if (report) {
      report->total_time_s += clock() - t0;
      for (const auto& h : out) report->output_tokens += static_cast<long>(h.tokens.size());
    }
    return out;
  }
  for (size_t i = 0; i < srcs.size(); ++i) {
    const double t0 = clock();
    BatchResult r = translate_ids(ex, {srcs[i]}, cfg);
    if (r.status[0] == MTG_OK) out[i] = r.hyps[0];
    const double dt = clock() - t0;
    if (report) {
      report->durations_s.push_back(dt);
      report->total_time_s += dt;
      report->output_tokens += static_cast<long>(out[i].tokens.size());
    }
  }
  return out;
}

}  // namespace gpu
}  // namespace minimt

#endif  // MINIMT_GPU_HPP_
