// polycert_b200.hpp — header-only C++ façade over the C-ABI (polycert_b200.h)
// that keeps the reference's C++ verifier API as the drop-in surface:
//
//   reference (WidenedFloat64 mode)                  here
//   ---------------------------------------------   ---------------------------------------
//   polycert::Shape / LayerKind / Layer<P>           polycert_b200::Shape / LayerKind / Layer
//     (proj/include/polycert/network.hpp:16-99)
//   polycert::Network<P>, instantiate<P>(doc)        polycert_b200::Network, instantiate(net)
//     (network.hpp:101-141, model_io.cpp:49-135)       -> validate + upload (pc_net_create)
//   polycert::InputBox<P>, input_box(c, eps, clamp)  polycert_b200::InputBox, input_box(...)
//     (network.hpp:150-177)                            (pc_input_box)
//   polycert::AnalysisOptions (analyzer.hpp:164-169) polycert_b200::AnalysisOptions (+ device)
//   polycert::PassStats (backsub.hpp:119-136)        polycert_b200::PassStats
//   analyze(net, box, opt) (analyzer.hpp:198-242)    polycert_b200::analyze(net, box, opt)
//   verify_robustness(net, box, label, opt)          polycert_b200::verify_robustness(...)
//     (analyzer.hpp:256-276)                           (pc_net_test)
//
// Exceptions keep the reference's classes: std::invalid_argument for bad
// labels / eps / centers (backsub.hpp:318, network.hpp:164-171), std::runtime_error
// "model: layer N: ..." for validation (model_io.cpp:27-29), std::logic_error
// for internal invariants; CUDA failures (no device: there is no CPU
// fallback) raise std::runtime_error("cuda: ...").
//
// Link with -lpolycert_b200 (paper_2007_10868_b200/libpolycert_b200.so).
#ifndef POLYCERT_B200_HPP
#define POLYCERT_B200_HPP

#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "polycert_b200.h"

namespace polycert_b200 {

struct Shape {  // network.hpp:16-21; flat index (h*W + w)*C + c
  int w = 1, h = 1, c = 1;
  int numel() const { return w * h * c; }
  bool operator==(const Shape& o) const { return w == o.w && h == o.h && c == o.c; }
};

enum class LayerKind { Input = PC_INPUT, Dense = PC_DENSE, Conv = PC_CONV, Relu = PC_RELU, Join = PC_JOIN };

struct Layer {  // network.hpp:84-99 with P = WidenedFloat64 (scalars are doubles)
  int id = 0;
  LayerKind kind = LayerKind::Input;
  std::vector<int> preds;
  Shape out_shape;               // filled by instantiate()
  std::vector<double> weights;   // dense, [out * in] row-major
  std::vector<double> bias;      // dense or conv
  std::vector<double> filter;    // conv, ((fy*fw + fx)*cin + ci)*cout + co
  int n_out = 0;                 // dense rows
  int fw = 0, fh = 0, cin = 0, cout = 0, sw = 1, sh = 1, pw = 0, ph = 0;
};

struct Interval {  // interval.hpp:127-158
  double lo = 0, hi = 0;
};

struct InputBox {  // network.hpp:155-158
  std::vector<Interval> pixels;
};

struct AnalysisOptions {  // analyzer.hpp:164-169
  bool early_term = true;
  long long chunk_rows = 0;     // 0: derive from memory_budget
  long long memory_budget = 0;  // device workspace bytes per pass; 0: engine default
  int workers = 1;              // accepted for source compatibility; the GPU grid is the parallelism
  int device = -1;              // CUDA ordinal; -1: current
  int exec_mode = 0;            // 0 auto, 1 host-driven schedule, 2 device-driven (CUDA graph)
  int numeric_mode = 0;         // 0 WidenedFloat64 bit for bit; 1 fast native directed rounding (sound)
  bool operator==(const AnalysisOptions& o) const {
    return early_term == o.early_term && chunk_rows == o.chunk_rows &&
           memory_budget == o.memory_budget && device == o.device && exec_mode == o.exec_mode &&
           numeric_mode == o.numeric_mode;
  }
};

struct PassStats {  // backsub.hpp:119-136
  long long rows_total = 0, rows_terminated_early = 0, gbc_madds = 0, gbc_dense_equiv = 0,
            dense_madds = 0, checkpoints = 0;
};

using LayerBounds = std::vector<std::vector<Interval>>;

struct AnalysisState {  // backsub.hpp:71-80 (the parts analyze() exposes)
  LayerBounds bounds;   // padded per-layer per-neuron bounds
  LayerBounds raw;      // unpadded freeze-test twin
};

struct AnalysisResult {  // analyzer.hpp:171-175
  AnalysisState state;
  PassStats stats;
};

struct Verdict {  // analyzer.hpp:247-254
  bool verified = false;
  int label = 0;
  std::vector<std::pair<int, double>> margins;  // (class j, lower bound of out_label - out_j), ascending j
  PassStats stats;
};

namespace detail {

[[noreturn]] inline void raise(pc_status st) {
  const std::string msg = pc_last_error();
  switch (st) {
    case PC_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case PC_ERR_LOGIC: throw std::logic_error(msg);
    case PC_ERR_OOM: throw std::runtime_error("out of memory: " + msg);
    default: throw std::runtime_error(msg);
  }
}

inline void check(pc_status st) {
  if (st != PC_OK) raise(st);
}

inline PassStats stats_of(const pc_stats& s) {
  return PassStats{s.rows_total, s.rows_terminated_early, s.gbc_madds,
                   s.gbc_dense_equiv, s.dense_madds, s.checkpoints};
}

struct Handle {
  pc_net* h = nullptr;
  int device = -1;
  uint64_t fingerprint = 0;  // layers + parameters the device copy was built from
  ~Handle() { if (h) pc_net_destroy(h); }
};

// Per-call options for pc_net_test_ex (the device is the handle's).
inline pc_options call_options(const AnalysisOptions& opt) {
  pc_options o;
  pc_default_options(&o);
  o.early_term = opt.early_term ? 1 : 0;
  o.chunk_rows = opt.chunk_rows;
  o.memory_budget = opt.memory_budget;
  o.device = opt.device;
  o.exec_mode = opt.exec_mode;
  o.numeric_mode = opt.numeric_mode;
  return o;
}

inline uint64_t mix(uint64_t h, uint64_t v) {
  h ^= v + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
  return h * 0xFF51AFD7ED558CCDull;
}

}  // namespace detail

// Network<WidenedFloat64> analogue. The device copy (pc_net: validated layers
// and uploaded weights) is created once by instantiate() (or on first use) and
// shared by copies; every call passes its own AnalysisOptions through
// pc_net_test_ex, so concurrent calls with different options are safe, as on
// the reference's immutable Network (analyzer.hpp:198-276). Each call holds a
// reference to the handle for its whole duration. Editing layers or weights
// after instantiate() is detected (content fingerprint) and re-uploads.
class Network {
 public:
  Shape input_shape;
  std::vector<Layer> layers;  // layers[0] is the input layer

  int output_layer() const { return static_cast<int>(layers.size()) - 1; }
  int output_size() const { return layers.back().out_shape.numel(); }

  // validate_model (model_io.cpp:49-135): fills out_shape, throws runtime_error.
  void validate() {
    std::vector<pc_layer_desc> d = descs();
    std::vector<int> shapes(3 * layers.size());
    detail::check(pc_validate(d.data(), (int)d.size(), input_shape.w, input_shape.h,
                              input_shape.c, shapes.data()));
    for (size_t k = 0; k < layers.size(); ++k)
      layers[k].out_shape = Shape{shapes[3 * k], shapes[3 * k + 1], shapes[3 * k + 2]};
  }

  // The device handle (created on first use, or again after the layers or
  // the device changed). The returned reference keeps it alive for the call.
  std::shared_ptr<detail::Handle> handle(const AnalysisOptions& opt) const {
    const uint64_t fp = fingerprint();
    std::lock_guard<std::mutex> lk(*mu_);
    if (!dev_ || dev_->fingerprint != fp || dev_->device != opt.device) {
      std::vector<pc_layer_desc> d = descs();
      const pc_options copt = detail::call_options(opt);
      auto h = std::make_shared<detail::Handle>();
      h->device = opt.device;
      h->fingerprint = fp;
      detail::check(pc_net_create(d.data(), (int)d.size(), input_shape.w, input_shape.h,
                                  input_shape.c, &copt, &h->h));
      dev_ = std::move(h);
    }
    return dev_;
  }

 private:
  mutable std::shared_ptr<detail::Handle> dev_;
  std::shared_ptr<std::mutex> mu_ = std::make_shared<std::mutex>();

  uint64_t fingerprint() const {
    uint64_t h = detail::mix(0, (uint64_t)input_shape.numel());
    auto words = [&h](const std::vector<double>& v) {  // 4 independent lanes: ~1 word/cycle
      uint64_t a[4] = {v.size(), 1, 2, 3};
      size_t i = 0;
      for (; i + 4 <= v.size(); i += 4)
        for (int l = 0; l < 4; ++l) {
          uint64_t b;
          std::memcpy(&b, &v[i + l], 8);
          a[l] = (a[l] ^ b) * 0x9E3779B97F4A7C15ull;
        }
      for (; i < v.size(); ++i) {
        uint64_t b;
        std::memcpy(&b, &v[i], 8);
        a[0] = (a[0] ^ b) * 0x9E3779B97F4A7C15ull;
      }
      for (uint64_t x : a) h = detail::mix(h, x);
    };
    for (const Layer& l : layers) {
      h = detail::mix(h, (uint64_t)l.kind);
      for (int p : l.preds) h = detail::mix(h, (uint64_t)p);
      for (int v : {l.n_out, l.fw, l.fh, l.cin, l.cout, l.sw, l.sh, l.pw, l.ph})
        h = detail::mix(h, (uint64_t)(uint32_t)v);
      words(l.weights);
      words(l.bias);
      words(l.filter);
    }
    return h;
  }

  std::vector<pc_layer_desc> descs() const {
    std::vector<pc_layer_desc> d(layers.size());
    for (size_t k = 0; k < layers.size(); ++k) {
      const Layer& l = layers[k];
      pc_layer_desc& x = d[k];
      x = pc_layer_desc{};
      x.kind = static_cast<int>(l.kind);
      x.n_preds = (int)l.preds.size();
      for (size_t p = 0; p < l.preds.size() && p < 2; ++p) x.preds[p] = l.preds[p];
      x.n_out = l.kind == LayerKind::Dense ? (l.n_out ? l.n_out : (int)l.bias.size()) : 0;
      x.fw = l.fw; x.fh = l.fh; x.sw = l.sw; x.sh = l.sh; x.pw = l.pw; x.ph = l.ph;
      x.cin = l.cin; x.cout = l.cout;
      x.weights = l.kind == LayerKind::Conv ? l.filter.data() : l.weights.data();
      x.bias = l.bias.data();
    }
    return d;
  }
};

// instantiate<WidenedFloat64> (network.hpp:110-141): validate, then upload.
inline Network instantiate(Network net, const AnalysisOptions& opt = {}) {
  net.validate();
  net.handle(opt);
  return net;
}

// input_box<WidenedFloat64> (network.hpp:160-177).
inline InputBox input_box(const std::vector<double>& center, double eps, bool clamp01) {
  std::vector<double> lo(center.size()), hi(center.size());
  detail::check(pc_input_box(center.data(), (int)center.size(), eps, clamp01 ? 1 : 0, lo.data(),
                             hi.data()));
  InputBox b;
  b.pixels.resize(center.size());
  for (size_t i = 0; i < center.size(); ++i) b.pixels[i] = Interval{lo[i], hi[i]};
  return b;
}

namespace detail {

inline void split(const InputBox& box, std::vector<double>& lo, std::vector<double>& hi) {
  lo.resize(box.pixels.size());
  hi.resize(box.pixels.size());
  for (size_t i = 0; i < box.pixels.size(); ++i) {
    lo[i] = box.pixels[i].lo;
    hi[i] = box.pixels[i].hi;
  }
}

}  // namespace detail

// analyze (analyzer.hpp:198-242): refined per-layer per-neuron bounds.
inline AnalysisResult analyze(const Network& net, const InputBox& box, const AnalysisOptions& opt) {
  const auto hold = net.handle(opt);
  pc_net* h = hold->h;
  const pc_options copt = detail::call_options(opt);
  std::vector<double> lo, hi;
  detail::split(box, lo, hi);
  const long long T = pc_net_total_neurons(h);
  std::vector<double> bl(T), bh(T), rl(T), rh(T);
  pc_stats st{};
  int verified = 0;
  detail::check(pc_net_test_ex(h, &copt, lo.data(), hi.data(), -1, &verified, nullptr, bl.data(),
                               bh.data(), rl.data(), rh.data(), &st));
  AnalysisResult r;
  r.stats = detail::stats_of(st);
  long long o = 0;
  for (int k = 0; k < pc_net_num_layers(h); ++k) {
    const long long n = pc_net_layer_numel(h, k);
    std::vector<Interval> b(n), w(n);
    for (long long j = 0; j < n; ++j) {
      b[j] = Interval{bl[o + j], bh[o + j]};
      w[j] = Interval{rl[o + j], rh[o + j]};
    }
    r.state.bounds.push_back(std::move(b));
    r.state.raw.push_back(std::move(w));
    o += n;
  }
  return r;
}

// verify_robustness (analyzer.hpp:256-276): analyze + margin pass; verified
// iff every margin lower bound is > 0.
inline Verdict verify_robustness(const Network& net, const InputBox& box, int label,
                                 const AnalysisOptions& opt) {
  const auto hold = net.handle(opt);
  pc_net* h = hold->h;
  const pc_options copt = detail::call_options(opt);
  const int n_out = pc_net_output_size(h);
  if (label < 0 || label >= n_out) throw std::invalid_argument("margin: label out of range");
  std::vector<double> lo, hi;
  detail::split(box, lo, hi);
  std::vector<double> m(n_out > 1 ? n_out - 1 : 1);
  pc_stats st{};
  int verified = 0;
  detail::check(pc_net_test_ex(h, &copt, lo.data(), hi.data(), label, &verified, m.data(), nullptr,
                               nullptr, nullptr, nullptr, &st));
  Verdict v;
  v.label = label;
  v.verified = verified != 0;
  v.stats = detail::stats_of(st);
  int r = 0;
  for (int j = 0; j < n_out; ++j)
    if (j != label) v.margins.emplace_back(j, m[r++]);
  return v;
}

}  // namespace polycert_b200

#endif  // POLYCERT_B200_HPP
