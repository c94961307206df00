// Reference-style tests (proj/tests/test_decode.cpp) written against the C++
// shim include/minimt_gpu.hpp; run by tests/test_cpp_shim.py on a B200.
// argv[1] = all-zero-parameter model (SQNT), argv[2] = random micro model.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "minimt_gpu.hpp"

using namespace minimt::gpu;

static int failures = 0;
#define CHECK(c)                                                        \
  do {                                                                  \
    if (!(c)) {                                                         \
      std::printf("CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); \
      ++failures;                                                       \
    }                                                                   \
  } while (0)
template <typename E, typename F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

int main(int argc, char** argv) {
  if (argc < 3) return 2;
  // test_decode.cpp:41-50 GNMT penalty
  Hypothesis h;
  h.tokens = {5, 6, 7, 8};
  h.logprob = -1.0f;
  CHECK(h.normalized_score(0.0f) == -1.0f);
  CHECK(std::fabs(h.normalized_score(1.0f) - (-1.0f / (10.0f / 6.0f))) < 1e-6f);

  GpuExecutor micro(argv[2], MTG_PREC_F32);
  // test_decode.cpp:93-101 input validation
  BeamConfig bad;
  bad.beam_size = 0;
  CHECK(throws<UsageError>([&] { beam_search(micro, {4, kEosId}, {}, bad); }));
  BeamConfig one;
  one.beam_size = 1;
  CHECK(throws<UsageError>([&] { beam_search(micro, {}, {}, one); }));
  CHECK(throws<FormatError>([&] { GpuExecutor x(argv[0], MTG_PREC_F32); }));  // not SQNT

  // test_decode.cpp:52-76 beam 1 == stepwise greedy argmax
  std::vector<int> src{4, 7, 5, kEosId};
  BeamConfig g;
  g.beam_size = 1;
  g.max_len = 10;
  g.length_penalty_alpha = 0.0f;
  Hypothesis beam = beam_search(micro, src, {}, g);
  std::vector<int> greedy;
  for (int t = 0; t < g.max_len; ++t) {
    std::vector<int> forced = greedy;
    forced.push_back(0);
    std::vector<float> lg = micro.forced_logits(src, forced);
    const size_t V = lg.size() / forced.size();
    const float* row = lg.data() + static_cast<size_t>(t) * V;
    int best = 0;
    for (size_t j = 1; j < V; ++j)
      if (row[j] > row[best]) best = static_cast<int>(j);
    if (best == kEosId) break;
    greedy.push_back(best);
  }
  CHECK(beam.tokens == greedy);

  // decode.cpp:48 with max_len <= 0: no search step, the source is still
  // encoded (bad ids throw), the unfinished root comes back truncated.
  BeamConfig none;
  none.max_len = 0;
  Hypothesis root = beam_search(micro, src, {}, none);
  CHECK(root.tokens.empty() && root.logprob == 0.0f && root.truncated && !root.finished);
  CHECK(root.normalized == 0.0f);
  CHECK(throws<IndexError>([&] { beam_search(micro, {4, 99, kEosId}, {}, none); }));

  // test_decode.cpp:171-206 latency percentiles from an injected clock on the
  // all-zero model: 10 sentences, sentence i takes (i+1) ms.
  GpuExecutor zero(argv[1], MTG_PREC_F32);
  std::vector<double> times;
  double now = 0.0;
  for (int i = 0; i < 10; ++i) {
    times.push_back(now);
    now += (i + 1) * 1e-3;
    times.push_back(now);
  }
  size_t tick = 0;
  Clock clock = [&] { return times.at(tick++); };
  BeamConfig z;
  z.beam_size = 1;
  z.max_len = 3;
  LatencyReport report;
  std::vector<std::vector<int>> words(10, std::vector<int>{4, 5});
  auto out = translate_corpus_ids(zero, words, z, &report, 1, clock);
  CHECK(out.size() == 10);
  CHECK(report.count() == 10);
  CHECK(std::fabs(report.p50_ms() - 5.0) < 1e-9);
  CHECK(std::fabs(report.p90_ms() - 9.0) < 1e-9);
  CHECK(std::fabs(report.mean_ms() - 5.5) < 1e-9);
  CHECK(report.output_tokens == 30);
  CHECK(std::fabs(report.tokens_per_sec() - 30.0 / 0.055) < 1e-6);
  std::printf(failures ? "SHIM_FAIL %d\n" : "SHIM_OK\n", failures);
  return failures ? 1 : 0;
}
