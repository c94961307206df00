// minimt_gpu -- `translate` and `benchmark` commands of the reference CLI
// (proj/tools/minimt.cpp:290-462, 546-566) over the GPU library.
//
//   minimt_gpu translate --model m.bin --input in.txt [--output out.txt]
//   minimt_gpu benchmark --model m.bin --input in.txt [--repeat N]
//
// Same flags and defaults (vocabularies / shortlist table / meta.json next to
// the model), the same LatencyReport JSON; --workers is accepted and ignored,
// --precision f32|bf16|int8 picks the executor (--int8 == --precision int8),
// --batch N > 1 decodes length-bucketed device batches (no per-sentence
// latency, like --parallel-sentences). Exit codes: 2 UsageError, 1 others.
//
// Build: g++ -std=c++17 -O2 -Iinclude tools/minimt_gpu_cli.cpp
//        -Lpaper_2008_04885_b200 -lminimt_gpu -Wl,-rpath,<that dir>
#include <filesystem>
#include <iostream>
#include <map>
#include <string>
#include <vector>

#include "minimt_gpu_text.hpp"

namespace fs = std::filesystem;
using namespace minimt::gpu;

namespace {

struct Args {
  std::string model, input, output = "-";
  std::string src_vocab, tgt_vocab, factor_vocab, shortlist_table, case_scheme, latency_out;
  std::string precision;
  bool int8 = false;
  int beam = 4, max_len = 0, shortlist_k = 0, repeat = 1, batch = 1;
  float alpha = 1.0f;
};

std::string sibling(const std::string& model, const std::string& name) {
  return (fs::path(model).parent_path() / name).string();
}

FactorScheme resolve_scheme(const Args& a) {  // minimt.cpp:334-345
  if (!a.case_scheme.empty()) return factor_scheme_from_string(a.case_scheme);
  const std::string meta = sibling(a.model, "meta.json");
  if (fs::exists(meta)) {
    std::ifstream f(meta);
    std::stringstream ss;
    ss << f.rdbuf();
    const std::string j = ss.str();
    const auto k = j.find("\"factors_scheme\"");
    if (k != std::string::npos) {
      const auto q1 = j.find('"', j.find(':', k) + 1);
      const auto q2 = j.find('"', q1 + 1);
      if (q1 != std::string::npos && q2 != std::string::npos)
        return factor_scheme_from_string(j.substr(q1 + 1, q2 - q1 - 1));
    }
  }
  return FactorScheme::kNone;
}

std::string indent_obj(const std::string& flat, const std::string& pad) {
  // {"a":1,"b":2} -> nlohmann dump(2) layout at the given indentation
  std::string out = "{\n";
  const std::string body = flat.substr(1, flat.size() - 2);
  size_t start = 0;
  while (start < body.size()) {
    size_t end = body.find(',', start);
    if (end == std::string::npos) end = body.size();
    std::string item = body.substr(start, end - start);
    const auto colon = item.find(':');
    out += pad + "  " + item.substr(0, colon) + ": " + item.substr(colon + 1);
    out += end < body.size() ? ",\n" : "\n";
    start = end + 1;
  }
  return out + pad + "}";
}

int run(const Args& a, bool benchmark) {  // minimt.cpp:347-433
  int prec = MTG_PREC_F32;
  if (a.int8 || a.precision == "int8") prec = MTG_PREC_INT8;
  else if (a.precision == "bf16") prec = MTG_PREC_BF16;
  else if (!a.precision.empty() && a.precision != "f32")
    throw UsageError("unknown precision: " + a.precision);
  GpuExecutor ex(a.model, prec);
  auto vpath = [&](const std::string& o, const std::string& name) {
    return o.empty() ? sibling(a.model, name) : o;
  };
  const Vocabulary src_vocab = Vocabulary::load(vpath(a.src_vocab, "src.vocab"));
  const Vocabulary tgt_vocab = Vocabulary::load(vpath(a.tgt_vocab, "tgt.vocab"));
  FactorScheme scheme = resolve_scheme(a);
  std::vector<Vocabulary> factor_vocabs;
  if (ex.config_json().find("\"factors\":[]") == std::string::npos) {
    if (scheme == FactorScheme::kNone)
      throw UsageError("translate: model has factors; pass --case-scheme");
    if (scheme == FactorScheme::kSfCase) factor_vocabs.push_back(case_factor_vocabulary());
    else if (scheme == FactorScheme::kSfWordShare) factor_vocabs.push_back(src_vocab);
    else factor_vocabs.push_back(Vocabulary::load(vpath(a.factor_vocab, "factor0.vocab")));
  } else {
    scheme = FactorScheme::kNone;
  }
  TranslateOptions o;
  o.scheme = scheme;
  o.beam = BeamConfig{a.beam, a.max_len, a.alpha};
  o.shortlist_k = a.shortlist_k;
  o.batch_sentences = a.batch;
  ShortlistTable table;
  if (a.shortlist_k > 0) {
    table = ShortlistTable::load(a.shortlist_table.empty() ? sibling(a.model, "shortlist.txt")
                                                           : a.shortlist_table);
    o.shortlist_table = &table;
  }
  const std::vector<std::string> lines = read_lines(a.input);
  const int repeats = benchmark ? std::max(1, a.repeat) : 1;
  std::vector<std::string> out;
  LatencyReport aggregate;
  std::vector<std::string> per_repeat;
  for (int r = 0; r < repeats; ++r) {
    LatencyReport report;
    out = translate_corpus(ex, src_vocab, tgt_vocab, factor_vocabs, lines, o, &report);
    per_repeat.push_back(latency_json(report));
    aggregate.durations_s.insert(aggregate.durations_s.end(), report.durations_s.begin(),
                                 report.durations_s.end());
    aggregate.output_tokens += report.output_tokens;
    aggregate.total_time_s += report.total_time_s;
  }
  if (benchmark) {
    std::cout << "{\n  \"aggregate\": " << indent_obj(latency_json(aggregate), "  ")
              << ",\n  \"repeats\": [\n";
    for (size_t i = 0; i < per_repeat.size(); ++i)
      std::cout << "    " << indent_obj(per_repeat[i], "    ")
                << (i + 1 < per_repeat.size() ? ",\n" : "\n");
    std::cout << "  ]\n}\n";
  } else if (a.output == "-") {
    for (const auto& l : out) std::cout << l << "\n";
  } else {
    write_lines(a.output, out);
  }
  if (!a.latency_out.empty()) {
    std::ofstream f(a.latency_out, std::ios::trunc);
    if (!f) throw IoError("cannot write latency report: " + a.latency_out);
    f << latency_json(aggregate) << "\n";
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2 || (std::string(argv[1]) != "translate" && std::string(argv[1]) != "benchmark")) {
    std::cerr << "usage: minimt_gpu translate|benchmark --model FILE --input FILE [options]\n";
    return 2;
  }
  const bool benchmark = std::string(argv[1]) == "benchmark";
  Args a;
  try {
    std::map<std::string, std::string*> s{
        {"--model", &a.model},         {"--input", &a.input},
        {"--output", &a.output},       {"--src-vocab", &a.src_vocab},
        {"--tgt-vocab", &a.tgt_vocab}, {"--factor-vocab", &a.factor_vocab},
        {"--shortlist-table", &a.shortlist_table},
        {"--case-scheme", &a.case_scheme},
        {"--latency", &a.latency_out}, {"--precision", &a.precision}};
    std::map<std::string, int*> n{{"--beam", &a.beam},           {"--max-len", &a.max_len},
                                  {"--shortlist", &a.shortlist_k}, {"--repeat", &a.repeat},
                                  {"--batch", &a.batch},         {"--parallel-sentences", &a.batch}};
    int workers = 1;
    n["--workers"] = &workers;
    for (int i = 2; i < argc; ++i) {
      const std::string k = argv[i];
      if (k == "--int8") {
        a.int8 = true;
      } else if (i + 1 < argc && s.count(k)) {
        *s[k] = argv[++i];
      } else if (i + 1 < argc && n.count(k)) {
        *n[k] = std::stoi(argv[++i]);
      } else if (i + 1 < argc && k == "--alpha") {
        a.alpha = std::stof(argv[++i]);
      } else {
        throw UsageError("unknown or incomplete option: " + k);
      }
    }
    if (a.model.empty() || a.input.empty()) throw UsageError("--model and --input are required");
    return run(a, benchmark);
  } catch (const UsageError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
