// minimt_gpu_text.hpp -- the text-level caller side of the decode path over
// the GPU library (header-only, host C++): vocabularies, whitespace
// tokenisation, case factors, translate_corpus and the latency report, with
// the reference's semantics (proj/src/data.cpp:40-125, 332-345;
// proj/src/decode.cpp:200-419; proj/include/minimt/decode.hpp:60-113).
//
// The one deliberate difference is batching: TranslateOptions::batch_sentences
// > 1 sends length-bucketed device batches through one translate_ids call
// (the GPU analogue of the reference's parallel_sentences mode, which also
// drops per-sentence latency); batch_sentences == 1 is the reference's
// sequential batch-1 mode with per-sentence wall times.
#ifndef MINIMT_GPU_TEXT_HPP_
#define MINIMT_GPU_TEXT_HPP_

#include <cctype>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <unordered_map>
#include <vector>

#include "minimt_gpu.hpp"

namespace minimt {
namespace gpu {

using TokenSeq = std::vector<std::string>;

// ---- data.cpp:40-56 ----------------------------------------------------------
inline TokenSeq tokenize(const std::string& line) {
  TokenSeq out;
  std::istringstream ss(line);
  std::string tok;
  while (ss >> tok) out.push_back(tok);
  return out;
}

inline std::string detokenize(const TokenSeq& tokens) {
  std::string out;
  for (size_t i = 0; i < tokens.size(); ++i) {
    if (i) out += ' ';
    out += tokens[i];
  }
  return out;
}

// ---- Vocabulary (data.hpp:18-38, data.cpp:58-115) -------------------------------
class Vocabulary {
 public:
  Vocabulary() {
    for (const char* r : {"<pad>", "<unk>", "<s>", "</s>"}) add(r);
  }
  int add(const std::string& token) {  // idempotent
    const auto it = to_id_.find(token);
    if (it != to_id_.end()) return it->second;
    const int id = size();
    to_id_.emplace(token, id);
    to_tok_.push_back(token);
    return id;
  }
  int id(const std::string& token) const {  // UNK when missing
    const auto it = to_id_.find(token);
    return it == to_id_.end() ? kUnkId : it->second;
  }
  bool contains(const std::string& token) const { return to_id_.count(token) > 0; }
  const std::string& token(int id) const {
    if (id < 0 || id >= size()) throw IndexError("vocabulary id out of range");
    return to_tok_[id];
  }
  int size() const { return static_cast<int>(to_tok_.size()); }
  std::vector<int> encode(const TokenSeq& tokens) const {
    std::vector<int> out;
    out.reserve(tokens.size());
    for (const auto& t : tokens) out.push_back(id(t));
    return out;
  }
  TokenSeq decode(const std::vector<int>& ids) const {
    TokenSeq out;
    out.reserve(ids.size());
    for (int i : ids) out.push_back(token(i));
    return out;
  }
  // One non-reserved token per line; id = line number - 1 + 4.
  void save(const std::string& path) const {
    std::ofstream f(path, std::ios::trunc);
    if (!f) throw IoError("cannot write vocabulary: " + path);
    for (int i = 4; i < size(); ++i) f << to_tok_[i] << '\n';
  }
  static Vocabulary load(const std::string& path) {
    std::ifstream f(path);
    if (!f) throw IoError("cannot read vocabulary: " + path);
    Vocabulary v;
    std::string line;
    while (std::getline(f, line))
      if (!line.empty()) v.add(line);
    return v;
  }

 private:
  std::vector<std::string> to_tok_;
  std::unordered_map<std::string, int> to_id_;
};

// ---- case factors (decode.cpp:200-277) -----------------------------------------
enum class FactorScheme { kNone, kSfCase, kSfWord, kSfWordShare };

inline FactorScheme factor_scheme_from_string(const std::string& s) {
  if (s == "none") return FactorScheme::kNone;
  if (s == "sf-case" || s == "sf_case") return FactorScheme::kSfCase;
  if (s == "sf-word" || s == "sf_word") return FactorScheme::kSfWord;
  if (s == "sf-word-share" || s == "sf_word_share") return FactorScheme::kSfWordShare;
  throw UsageError("unknown factor scheme: " + s);
}

inline const char* const* case_category_names() {
  static const char* names[4] = {"lowercase", "capitalized", "all_uppercase", "mixed"};
  return names;
}

inline std::string case_category(const std::string& token) {
  bool has_upper = false, has_lower = false, first_upper = false, upper_after = false;
  for (size_t i = 0; i < token.size(); ++i) {
    const unsigned char c = static_cast<unsigned char>(token[i]);
    if (std::isupper(c)) {
      has_upper = true;
      (i == 0 ? first_upper : upper_after) = true;
    } else if (std::islower(c)) {
      has_lower = true;
    }
  }
  const char* const* n = case_category_names();
  if (!has_upper) return n[0];
  if (first_upper && !upper_after) return n[1];
  if (!has_lower) return n[2];
  return n[3];
}

inline Vocabulary case_factor_vocabulary() {
  Vocabulary v;
  for (int i = 0; i < 4; ++i) v.add(case_category_names()[i]);
  return v;
}

struct FactoredInput {
  TokenSeq words;
  std::vector<TokenSeq> factors;  // one stream per factor, token-aligned
};

inline FactoredInput apply_case_factors(const std::string& line, FactorScheme scheme) {
  FactoredInput out;
  out.words = tokenize(line);
  if (scheme == FactorScheme::kNone) return out;
  TokenSeq factor;
  factor.reserve(out.words.size());
  for (auto& w : out.words) {
    factor.push_back(scheme == FactorScheme::kSfCase ? case_category(w) : w);
    for (char& c : w) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
  }
  out.factors.push_back(std::move(factor));
  return out;
}

// ---- LatencyReport::to_json (decode.cpp:281-308): nlohmann dump, sorted keys --
inline std::string json_number(double d) {  // shortest round-trip, like nlohmann
  char buf[64];
  for (int prec = 1; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof buf, "%.*g", prec, d);
    if (std::strtod(buf, nullptr) == d) break;
  }
  std::string s = buf;
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}

inline std::string latency_json(const LatencyReport& r) {
  return "{\"count\":" + std::to_string(r.count()) + ",\"mean_ms\":" + json_number(r.mean_ms()) +
         ",\"p50_ms\":" + json_number(r.p50_ms()) + ",\"p90_ms\":" + json_number(r.p90_ms()) +
         ",\"tokens_per_sec\":" + json_number(r.tokens_per_sec()) + "}";
}

// ---- translate_corpus (decode.hpp:94-113, decode.cpp:320-419) --------------------
struct TranslateOptions {
  FactorScheme scheme = FactorScheme::kNone;
  BeamConfig beam;
  int shortlist_k = 0;  // 0 disables shortlisting
  const ShortlistTable* shortlist_table = nullptr;
  int batch_sentences = 1;  // > 1: device batches, no per-sentence latency
};

namespace detail {

// translate_one's preprocessing (decode.cpp:325-349): ids + EOS truncated to
// max_seq_len keeping EOS; factor streams + EOS padded/cut to the same
// length; shortlist only when it is smaller than the vocabulary.
struct Prepared {
  std::vector<int> src;
  std::vector<std::vector<int>> factors;
  std::vector<int> shortlist;  // empty: full vocabulary
};

inline Prepared prepare(const GpuExecutor& ex, const Vocabulary& src_vocab,
                        const std::vector<Vocabulary>& factor_vocabs, const std::string& line,
                        const TranslateOptions& o, int max_seq_len, int tgt_vocab) {
  Prepared p;
  FactoredInput input = apply_case_factors(line, o.scheme);
  p.src = src_vocab.encode(input.words);
  p.src.push_back(kEosId);
  if (static_cast<int>(p.src.size()) > max_seq_len) {
    p.src.resize(max_seq_len - 1);
    p.src.push_back(kEosId);
  }
  for (size_t f = 0; f < input.factors.size(); ++f) {
    if (f >= factor_vocabs.size()) throw UsageError("translate: factor vocabulary missing");
    std::vector<int> ids = factor_vocabs[f].encode(input.factors[f]);
    ids.push_back(kEosId);
    ids.resize(p.src.size(), kEosId);
    p.factors.push_back(std::move(ids));
  }
  if (o.shortlist_k > 0 && o.shortlist_table) {
    std::vector<int> sl = build_shortlist(*o.shortlist_table, p.src, o.shortlist_k, tgt_vocab);
    if (static_cast<int>(sl.size()) < tgt_vocab) p.shortlist = std::move(sl);
  }
  (void)ex;
  return p;
}

inline int config_int(const std::string& json, const std::string& key, int dflt) {
  const auto p = json.find("\"" + key + "\":");
  return p == std::string::npos ? dflt : std::stoi(json.substr(p + key.size() + 3));
}

}  // namespace detail

inline std::vector<std::string> translate_corpus(const GpuExecutor& ex, const Vocabulary& src_vocab,
                                                 const Vocabulary& tgt_vocab,
                                                 const std::vector<Vocabulary>& factor_vocabs,
                                                 const std::vector<std::string>& lines,
                                                 const TranslateOptions& options,
                                                 LatencyReport* report = nullptr,
                                                 Clock clock = {}) {
  if (!clock) clock = steady_clock_seconds();
  const std::string cfg = ex.config_json();
  const int msl = detail::config_int(cfg, "max_seq_len", 128);
  const int V = detail::config_int(cfg, "tgt_vocab_size", 0);
  std::vector<std::string> out(lines.size());
  auto run = [&](const std::vector<size_t>& idx) -> long {
    std::vector<std::vector<int>> srcs;
    FactorStreams facs;
    std::vector<std::vector<int>> sls;
    std::vector<int> bad(idx.size(), 0);
    bool any_f = false, any_sl = false;
    for (size_t k = 0; k < idx.size(); ++k) {
      detail::Prepared p;
      try {
        p = detail::prepare(ex, src_vocab, factor_vocabs, lines[idx[k]], options, msl, V);
      } catch (const std::exception& e) {
        bad[k] = 1;
        std::cerr << "translate: sentence " << idx[k] + 1 << " failed: " << e.what() << "\n";
        p.src = {kEosId};
      }
      any_f |= !p.factors.empty();
      any_sl |= !p.shortlist.empty();
      srcs.push_back(std::move(p.src));
      facs.push_back(std::move(p.factors));
      sls.push_back(std::move(p.shortlist));
    }
    BatchResult r = translate_ids(ex, srcs, options.beam,
                                  options.batch_sentences > 1 ? options.batch_sentences : 0,
                                  any_f ? &facs : nullptr, any_sl ? &sls : nullptr);
    long tokens = 0;
    for (size_t k = 0; k < idx.size(); ++k) {
      if (bad[k] || r.status[k] != MTG_OK) {  // decode.cpp:403-410: empty line
        if (!bad[k])
          std::cerr << "translate: sentence " << idx[k] + 1 << " failed (status " << r.status[k]
                    << ")\n";
        out[idx[k]].clear();
        continue;
      }
      out[idx[k]] = detokenize(tgt_vocab.decode(r.hyps[k].tokens));
      tokens += static_cast<long>(r.hyps[k].tokens.size());
    }
    return tokens;
  };
  if (options.batch_sentences > 1) {
    std::vector<size_t> all(lines.size());
    for (size_t i = 0; i < lines.size(); ++i) all[i] = i;
    const double t0 = clock();
    const long tokens = lines.empty() ? 0 : run(all);
    if (report) {
      report->total_time_s = clock() - t0;
      report->output_tokens += tokens;
    }
    return out;
  }
  for (size_t i = 0; i < lines.size(); ++i) {
    const double t0 = clock();
    const long n = run({i});
    const double dt = clock() - t0;
    if (report) {
      report->durations_s.push_back(dt);
      report->total_time_s += dt;
      report->output_tokens += n;
    }
  }
  return out;
}

inline std::vector<std::string> read_lines(const std::string& path) {
  std::ifstream f(path);
  if (!f) throw IoError("cannot read: " + path);
  std::vector<std::string> lines;
  std::string line;
  while (std::getline(f, line)) lines.push_back(line);
  return lines;
}

inline void write_lines(const std::string& path, const std::vector<std::string>& lines) {
  std::ofstream f(path, std::ios::trunc);
  if (!f) throw IoError("cannot write: " + path);
  for (const auto& l : lines) f << l << '\n';
}

}  // namespace gpu
}  // namespace minimt

#endif  // MINIMT_GPU_TEXT_HPP_
