// C++ drop-in surface test: the reference's own known-answer tests, written
// against include/polycert_b200.hpp exactly as proj/tests/test_analyzer.cpp
// writes them against polycert's analyze / verify_robustness.
//   identity margins ~0.4 / ~-0.2 (widened)        test_analyzer.cpp:61-76
//   margins 1/8 and 3/16 (labels, class order)     test_analyzer.cpp:104-122
//   relu-free net: exact affine image, output 0    test_analyzer.cpp:79-102
//   exception classes and messages                 backsub.hpp:318, model_io.cpp:27-29,
//                                                  network.hpp:164-171
// Exit status 0 iff every check passed. Needs a CUDA device (no CPU fallback).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "polycert_b200.hpp"

using namespace polycert_b200;

static int g_fail = 0;
#define CHECK(c)                                                    \
  do {                                                              \
    if (!(c)) {                                                     \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
      ++g_fail;                                                     \
    }                                                               \
  } while (0)

static Network dense_net(Shape in, const std::vector<std::pair<std::vector<std::vector<double>>, std::vector<double>>>& specs,
                         bool relu_between = false) {
  Network net;
  net.input_shape = in;
  Layer l0;
  l0.kind = LayerKind::Input;
  net.layers.push_back(l0);
  for (size_t s = 0; s < specs.size(); ++s) {
    Layer d;
    d.id = (int)net.layers.size();
    d.kind = LayerKind::Dense;
    d.preds = {d.id - 1};
    for (const auto& row : specs[s].first) d.weights.insert(d.weights.end(), row.begin(), row.end());
    d.bias = specs[s].second;
    d.n_out = (int)d.bias.size();
    net.layers.push_back(d);
    if (relu_between && s + 1 < specs.size()) {
      Layer r;
      r.id = (int)net.layers.size();
      r.kind = LayerKind::Relu;
      r.preds = {r.id - 1};
      net.layers.push_back(r);
    }
  }
  return net;
}

int main() {
  AnalysisOptions opt;
  {  // identity network (test_util.hpp identity_doc)
    Network net = instantiate(dense_net(Shape{1, 1, 2}, {{{{1, 0}, {0, 1}}, {0, 0}}}), opt);
    const Verdict v1 = verify_robustness(net, input_box({0.7, 0.1}, 0.1, true), 0, opt);
    CHECK(v1.verified);
    CHECK(v1.margins.size() == 1 && v1.margins[0].first == 1);
    CHECK(std::fabs(v1.margins[0].second - 0.4) <= 1e-12 * 0.4);
    const Verdict v2 = verify_robustness(net, input_box({0.7, 0.1}, 0.4, true), 0, opt);
    CHECK(!v2.verified);
    CHECK(std::fabs(v2.margins[0].second + 0.2) <= 1e-12 * 0.2);
    bool threw = false;
    try {
      verify_robustness(net, input_box({0.7, 0.1}, 0.1, true), 2, opt);
    } catch (const std::invalid_argument& e) {
      threw = std::string(e.what()) == "margin: label out of range";
    }
    CHECK(threw);
    threw = false;
    try {
      input_box({1.5, 0.1}, 0.1, true);
    } catch (const std::invalid_argument& e) {
      threw = std::string(e.what()) == "input_box: clamped center outside [0,1]";
    }
    CHECK(threw);
    threw = false;
    try {
      input_box({0.5, 0.1}, -0.1, true);
    } catch (const std::invalid_argument& e) {
      threw = std::string(e.what()) == "input_box: negative epsilon";
    }
    CHECK(threw);
  }
  {  // margins match explicit output differences: exact 1/8 and 3/16 (rational mode);
     // widened mode certifies slightly less (inference-deviation allowances)
    Network net = instantiate(dense_net(Shape{1, 1, 2}, {{{{1, 0}, {0, 1}, {0.5, 0.5}}, {0, 0.25, 0}}}), opt);
    const Verdict v = verify_robustness(net, input_box({0.5, 0.5}, 1.0 / 16, true), 1, opt);
    CHECK(v.margins.size() == 2);
    CHECK(v.margins[0].first == 0 && v.margins[1].first == 2);
    CHECK(v.margins[0].second <= 1.0 / 8 && 1.0 / 8 - v.margins[0].second < 1e-12);
    CHECK(v.margins[1].second <= 3.0 / 16 && 3.0 / 16 - v.margins[1].second < 1e-12);
    CHECK(v.verified);
  }
  {  // relu-free networks get the exact affine image
    Network net = instantiate(
        dense_net(Shape{1, 1, 3}, {{{{1, -1, 0.5}, {0, 2, -1}}, {0.25, 0}}, {{{1, 1}, {1, -1}}, {0, 0.5}}}), opt);
    const AnalysisResult r = analyze(net, input_box({0.5, 0.25, 0.75}, 1.0 / 8, true), opt);
    CHECK(r.state.bounds.size() == 3);
    const double want = 0.5 - 0.125 + 0.25 - 0.125 - (0.875 * 0.5) + 0.25;
    // widened: the certified lower end is <= the exact one and within a few ulps
    CHECK(r.state.bounds.back()[0].lo <= want && want - r.state.bounds.back()[0].lo < 1e-12);
    CHECK(r.state.raw.size() == 3);
  }
  {  // validation errors keep the reference's messages (model_io.cpp:27-29)
    Network bad = dense_net(Shape{1, 1, 2}, {{{{1, 0}, {0, 1}}, {0, 0}}}, false);
    Layer r1;
    r1.id = 2; r1.kind = LayerKind::Relu; r1.preds = {1};
    Layer r2;
    r2.id = 3; r2.kind = LayerKind::Relu; r2.preds = {2};
    bad.layers.push_back(r1);
    bad.layers.push_back(r2);
    bool threw = false;
    try {
      bad.validate();
    } catch (const std::runtime_error& e) {
      threw = std::string(e.what()) == "model: layer 3: relu fed by relu";
    }
    CHECK(threw);
  }
  {  // a relu net: analyze bounds contain the forward interval refinement
    Network net = instantiate(dense_net(Shape{1, 1, 2},
                                        {{{{1, -1}, {0.5, 0.5}, {-1, 2}}, {0.1, -0.2, 0}},
                                         {{{1, 1, -1}, {0.5, -1, 1}}, {0, 0}}},
                                        true),
                              opt);
    const AnalysisResult r = analyze(net, input_box({0.4, 0.6}, 0.05, true), opt);
    for (const auto& layer : r.state.bounds)
      for (const Interval& iv : layer) CHECK(iv.lo <= iv.hi);
    const Verdict v = verify_robustness(net, input_box({0.4, 0.6}, 0.05, true), 0, opt);
    CHECK(v.margins.size() == 1 && v.stats.rows_total > 0);
  }
  {  // one Network, concurrent calls with different options (the handle is
     // bound once; options travel per call), then an edited copy re-uploads
    Network net = instantiate(dense_net(Shape{1, 1, 2},
                                        {{{{1, -1}, {0.5, 0.5}, {-1, 2}}, {0.1, -0.2, 0}},
                                         {{{1, 1, -1}, {0.5, -1, 1}}, {0, 0}}},
                                        true),
                              opt);
    const InputBox box = input_box({0.4, 0.6}, 0.05, true);
    const Verdict want = verify_robustness(net, box, 0, opt);
    std::vector<std::thread> th;
    std::vector<int> ok(8, 0);
    for (int t = 0; t < 8; ++t)
      th.emplace_back([&, t] {
        AnalysisOptions o;
        o.early_term = (t & 1) != 0;
        o.chunk_rows = (t & 2) ? 1 : 0;
        for (int k = 0; k < 4; ++k) {
          const Verdict v = verify_robustness(net, box, 0, o);
          ok[t] += v.margins.size() == want.margins.size() &&
                   std::memcmp(&v.margins[0].second, &want.margins[0].second, 8) == 0;
        }
      });
    for (auto& x : th) x.join();
    for (int t = 0; t < 8; ++t) CHECK(ok[t] == 4);
    Network edited = net;
    edited.layers[3].bias[0] += 1.0;  // out_0 - out_1 grows by exactly 1
    const Verdict v2 = verify_robustness(edited, box, 0, opt);
    CHECK(v2.margins[0].second > want.margins[0].second + 0.5);
    const Verdict v3 = verify_robustness(net, box, 0, opt);  // the original is untouched
    CHECK(std::memcmp(&v3.margins[0].second, &want.margins[0].second, 8) == 0);
  }
  std::printf("%s (%d failures)\n", g_fail ? "FAILED" : "facade ok", g_fail);
  return g_fail ? 1 : 0;
}
