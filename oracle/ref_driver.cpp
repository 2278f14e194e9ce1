// ref_driver.cpp — C-ABI driver over the UNMODIFIED reference verifier.
//
// ORACLE / TEST INFRASTRUCTURE ONLY (never linked into the product). Compiled
// by oracle/build_ref.sh against the reference's own headers and sources where
// they lie under /root/reference/proj (nothing is copied), together with the
// GMP shim in oracle/shim. The output library oracle/_ref/libpolycert_ref.so
// is git-ignored and travels to the GPU box with the snapshot.
//
// Every entry point calls the reference's public functions:
//   gen::generate / gen::random_inputs      (proj/src/gen.cpp:367-392)
//   model_from_json_text / model_to_json    (proj/src/model_io.cpp:223-311)
//   instantiate<P>, input_box<P>            (proj/include/polycert/network.hpp:110-177)
//   forward_eval + unique argmax            (eval.hpp:39-102, tools/main.cpp:86-100)
//   analyze + run_margin_pass               (analyzer.hpp:198-276, backsub.hpp:1070-1096)
// i.e. exactly what verify_robustness() does (analyzer.hpp:256-276), with the
// analysis state kept so per-neuron bounds can be compared too.

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <optional>
#include <string>
#include <thread>
#include <vector>

#include "polycert/analyzer.hpp"
#include "polycert/gen.hpp"
#include "polycert/network.hpp"
#include "polycert/oracle.hpp"

using namespace polycert;

namespace {

thread_local std::string g_err;

struct RefModel {
  ModelDoc doc;
  Network<WidenedFloat64> net;
};

int fail(const std::exception& e) {
  g_err = e.what();
  return -1;
}

template <class S>
std::optional<int> unique_argmax(const std::vector<S>& v) {  // tools/main.cpp:86-100
  int best = 0;
  bool tie = false;
  for (size_t j = 1; j < v.size(); ++j) {
    if (v[j] > v[best]) {
      best = static_cast<int>(j);
      tie = false;
    } else if (v[j] == v[best]) {
      tie = true;
    }
  }
  if (tie) return std::nullopt;
  return best;
}

AnalysisOptions make_opts(int early_term, long long chunk_rows, long long memory_budget,
                          int workers) {
  AnalysisOptions o;
  o.early_term = early_term != 0;
  o.chunk_rows = chunk_rows;
  o.memory_budget = memory_budget > 0 ? memory_budget : (1ll << 30);
  o.workers = workers > 0 ? workers : 1;
  return o;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void* ref_generate(uint64_t seed, const char* arch) {
  try {
    auto* m = new RefModel;
    m->doc = gen::generate(seed, arch);
    m->net = instantiate<WidenedFloat64>(m->doc);
    return m;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void* ref_from_json(const char* text) {
  try {
    auto* m = new RefModel;
    m->doc = model_from_json_text(text);
    m->net = instantiate<WidenedFloat64>(m->doc);
    return m;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_free(void* h) { delete static_cast<RefModel*>(h); }

// Caller frees with ref_free_str.
char* ref_to_json(void* h) {
  const std::string s = model_to_json_text(static_cast<RefModel*>(h)->doc);
  char* out = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(out, s.c_str(), s.size() + 1);
  return out;
}
void ref_free_str(char* s) { std::free(s); }

int ref_num_layers(void* h) { return static_cast<int>(static_cast<RefModel*>(h)->net.layers.size()); }

// info[16]: kind, n_preds, pred0, pred1, out_w, out_h, out_c, fw, fh, sw, sh, pw, ph,
//           cin, cout, join_head
int ref_layer_info(void* h, int k, int* info, long long* n_weights, long long* n_bias) {
  const auto& L = static_cast<RefModel*>(h)->net.layers.at(k);
  info[0] = static_cast<int>(L.kind);
  info[1] = static_cast<int>(L.preds.size());
  info[2] = L.preds.size() > 0 ? L.preds[0] : -1;
  info[3] = L.preds.size() > 1 ? L.preds[1] : -1;
  info[4] = L.out_shape.w; info[5] = L.out_shape.h; info[6] = L.out_shape.c;
  info[7] = L.fw; info[8] = L.fh; info[9] = L.sw; info[10] = L.sh;
  info[11] = L.pw; info[12] = L.ph; info[13] = L.cin; info[14] = L.cout;
  info[15] = L.join_head;
  *n_weights = static_cast<long long>(L.kind == LayerKind::Conv ? L.filter.size() : L.weights.size());
  *n_bias = static_cast<long long>(L.bias.size());
  return 0;
}

int ref_layer_params(void* h, int k, double* weights, double* bias) {
  const auto& L = static_cast<RefModel*>(h)->net.layers.at(k);
  const auto& w = L.kind == LayerKind::Conv ? L.filter : L.weights;
  if (weights && !w.empty()) std::memcpy(weights, w.data(), w.size() * sizeof(double));
  if (bias && !L.bias.empty()) std::memcpy(bias, L.bias.data(), L.bias.size() * sizeof(double));
  return 0;
}

// gen::random_inputs(seed, count, dim) parsed to doubles (exact: k/256).
int ref_random_inputs(uint64_t seed, int count, int dim, double* out) {
  try {
    const auto rows = gen::random_inputs(seed, count, dim);
    for (int r = 0; r < count; ++r)
      for (int i = 0; i < dim; ++i) out[static_cast<size_t>(r) * dim + i] = double_from_decimal(rows[r][i]);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

double ref_double_from_decimal(const char* s) { return double_from_decimal(s); }

// Candidate label (unique argmax of the concrete forward pass), -1 on a tie.
int ref_candidate(void* h, const double* center) {
  const auto& net = static_cast<RefModel*>(h)->net;
  std::vector<double> c(center, center + net.input_shape.numel());
  const auto acts = forward_eval(net, c);
  const auto l = unique_argmax(acts.back());
  return l ? *l : -1;
}

long long ref_total_neurons(void* h) {
  long long t = 0;
  for (const auto& L : static_cast<RefModel*>(h)->net.layers) t += L.out_shape.numel();
  return t;
}

// One widened-mode analysis + margin pass = verify_robustness (analyzer.hpp:256-276).
// label < 0: analysis only (no margin pass). stats[6] = PassStats fields in
// declaration order (backsub.hpp:119-125). bounds arrays (optional) are
// concatenated over layers 0..L-1 in layer order.
int ref_verify(void* h, const double* center, double eps, int clamp, int label, int early_term,
               long long chunk_rows, long long memory_budget, int workers, int* verified,
               double* margins, long long* stats, double* b_lo, double* b_hi, double* r_lo,
               double* r_hi, double* seconds) {
  try {
    const auto& net = static_cast<RefModel*>(h)->net;
    std::vector<double> c(center, center + net.input_shape.numel());
    const InputBox<WidenedFloat64> box = input_box<WidenedFloat64>(c, eps, clamp != 0);
    const AnalysisOptions opt = make_opts(early_term, chunk_rows, memory_budget, workers);
    const auto t0 = std::chrono::steady_clock::now();
    AnalysisResult<WidenedFloat64> ar = analyze(net, box, opt);
    std::vector<double> lows;
    if (label >= 0) lows = run_margin_pass(net, ar.state, label, pass_options(opt), ar.stats);
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    if (verified) {
      bool v = label >= 0;
      for (double x : lows)
        if (!(x > 0.0)) v = false;
      *verified = v ? 1 : 0;
    }
    if (margins)
      for (size_t i = 0; i < lows.size(); ++i) margins[i] = lows[i];
    if (stats) {
      stats[0] = ar.stats.rows_total;
      stats[1] = ar.stats.rows_terminated_early;
      stats[2] = ar.stats.gbc_madds;
      stats[3] = ar.stats.gbc_dense_equiv;
      stats[4] = ar.stats.dense_madds;
      stats[5] = ar.stats.checkpoints;
    }
    size_t off = 0;
    for (size_t k = 0; k < ar.state.bounds.size(); ++k) {
      for (size_t j = 0; j < ar.state.bounds[k].size(); ++j) {
        if (b_lo) b_lo[off + j] = ar.state.bounds[k][j].lo;
        if (b_hi) b_hi[off + j] = ar.state.bounds[k][j].hi;
        if (r_lo) r_lo[off + j] = ar.state.raw[k][j].lo;
        if (r_hi) r_hi[off + j] = ar.state.raw[k][j].hi;
      }
      off += ar.state.bounds[k].size();
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Forward interval bounds only (eval.hpp:230-237), padded and raw twins.
int ref_forward(void* h, const double* center, double eps, int clamp, double* b_lo, double* b_hi,
                double* r_lo, double* r_hi) {
  try {
    const auto& net = static_cast<RefModel*>(h)->net;
    std::vector<double> c(center, center + net.input_shape.numel());
    const auto box = input_box<WidenedFloat64>(c, eps, clamp != 0);
    const auto pb = forward_interval(net, box);
    const auto rb = forward_interval<WidenedFloat64, false>(net, box);
    size_t off = 0;
    for (size_t k = 0; k < pb.size(); ++k) {
      for (size_t j = 0; j < pb[k].size(); ++j) {
        b_lo[off + j] = pb[k][j].lo;
        b_hi[off + j] = pb[k][j].hi;
        r_lo[off + j] = rb[k][j].lo;
        r_hi[off + j] = rb[k][j].hi;
      }
      off += pb[k].size();
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Exact-rational soundness check: runs the rational engine (ExactRational
// analyze + margin pass) and counts widened values that fail to contain the
// exact ones. eps_num/eps_den gives the exact radius. Returns #violations or -1.
int ref_rational_contains(void* h, const double* center, long eps_num, long eps_den, int clamp,
                          int label, const double* b_lo, const double* b_hi,
                          const double* margins, int* verified_exact) {
  try {
    const ModelDoc& doc = static_cast<RefModel*>(h)->doc;
    const auto qnet = instantiate<ExactRational>(doc);
    std::vector<mpq_class> c;
    for (int i = 0; i < qnet.input_shape.numel(); ++i) c.emplace_back(center[i]);
    const auto box = input_box<ExactRational>(c, mpq_class(eps_num, eps_den), clamp != 0);
    AnalysisOptions opt;
    auto ar = analyze(qnet, box, opt);
    int bad = 0;
    size_t off = 0;
    for (size_t k = 0; k < ar.state.bounds.size(); ++k) {
      for (size_t j = 0; j < ar.state.bounds[k].size(); ++j) {
        if (!(mpq_class(b_lo[off + j]) <= ar.state.bounds[k][j].lo)) ++bad;
        if (!(ar.state.bounds[k][j].hi <= mpq_class(b_hi[off + j]))) ++bad;
      }
      off += ar.state.bounds[k].size();
    }
    if (label >= 0) {
      const auto lows = run_margin_pass(qnet, ar.state, label, pass_options(opt), ar.stats);
      bool v = true;
      for (size_t i = 0; i < lows.size(); ++i) {
        if (!(mpq_class(margins[i]) <= lows[i])) ++bad;
        if (!(lows[i] > mpq_class(0))) v = false;
      }
      if (verified_exact) *verified_exact = v ? 1 : 0;
    }
    return bad;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// CPU baseline: verify n images with `threads` host threads, one image per
// thread at a time (the CLI's worker pool, tools/main.cpp:117; each analysis
// single-threaded, main.cpp:57). label[i] < 0 → candidate from forward_eval;
// images without a unique argmax are skipped (verdict -1).
int ref_verify_batch(void* h, const double* centers, int n, double eps, int clamp, int threads,
                     int early_term, int* verdicts, double* wall_seconds,
                     double* per_image_seconds) {
  try {
    const auto& net = static_cast<RefModel*>(h)->net;
    const int dim = net.input_shape.numel();
    std::atomic<int> next{0};
    std::atomic<int> errors{0};
    const AnalysisOptions opt = make_opts(early_term, 0, 0, 1);
    auto work = [&]() {
      for (;;) {
        const int i = next.fetch_add(1);
        if (i >= n) return;
        try {
          std::vector<double> c(centers + static_cast<size_t>(i) * dim,
                                centers + static_cast<size_t>(i + 1) * dim);
          const auto acts = forward_eval(net, c);
          const auto lab = unique_argmax(acts.back());
          if (!lab) {
            verdicts[i] = -1;
            if (per_image_seconds) per_image_seconds[i] = 0.0;
            continue;
          }
          const auto box = input_box<WidenedFloat64>(c, eps, clamp != 0);
          const auto t0 = std::chrono::steady_clock::now();
          const Verdict<WidenedFloat64> v = verify_robustness(net, box, *lab, opt);
          const auto t1 = std::chrono::steady_clock::now();
          verdicts[i] = v.verified ? 1 : 0;
          if (per_image_seconds) per_image_seconds[i] = std::chrono::duration<double>(t1 - t0).count();
        } catch (...) {
          verdicts[i] = -2;
          errors.fetch_add(1);
        }
      }
    };
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 1; t < std::max(1, threads); ++t) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    const auto t1 = std::chrono::steady_clock::now();
    if (wall_seconds) *wall_seconds = std::chrono::duration<double>(t1 - t0).count();
    return errors.load();
  } catch (const std::exception& e) {
    return fail(e);
  }
}

}  // extern "C"
