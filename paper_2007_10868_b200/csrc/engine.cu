// engine.cu — host orchestration of the GPU verifier behind the C-ABI in
// include/polycert_b200.h.
//
// Mirrors the reference's driver layer: validate_model / instantiate
// (model_io.cpp:49-160, network.hpp:110-141), analyze / verify_robustness
// (analyzer.hpp:198-276), run_backsubstitution / run_margin_pass / walk_back /
// join_step (backsub.hpp:690-715, 850-893, 989-1096). Every numeric operation
// runs in a kernel (kernels.cu); the host only tracks frame geometry, row
// counts and buffer lifetimes. There is no CPU compute path.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <atomic>
#include <thread>
#include <cmath>
#include <cstring>
#include <functional>
#include <mutex>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/polycert_b200.h"
#include <nvtx3/nvToolsExt.h>
#include "kernels.cuh"

using namespace pc;

namespace {

thread_local std::string g_err;
thread_local long long g_last_launches = 0;
thread_local double g_total_ms = 0, g_dense_ms = 0, g_dense_bytes = 0, g_dense_madds = 0;
thread_local long long g_dense_launches = 0;
// conv back-substitution kernel (k_gbc_sparse2 / k_gbc_coef) of the last call:
// CUDA-event time over its launches, algorithmic bytes (rows in/out + filter)
thread_local double g_conv_ms = 0, g_conv_bytes = 0;
thread_local long long g_conv_launches = 0;
thread_local double g_conv_exec = 0;  // interval madds executed by the live-cell conv kernel

// NVTX ranges (header-only nvtx3): visible in Nsight Systems / ncu --nvtx;
// no cost without a tool attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  NvtxRange(const char* what, int k) {
    char buf[48];
    snprintf(buf, sizeof(buf), "%s %d", what, k);
    nvtxRangePushA(buf);
  }
  ~NvtxRange() { nvtxRangePop(); }
};

struct StatusError : std::runtime_error {
  pc_status code;
  StatusError(pc_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void model_fail(int id, const std::string& what) {
  throw StatusError(PC_ERR_MODEL, "model: layer " + std::to_string(id) + ": " + what);
}

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw StatusError(e == cudaErrorMemoryAllocation ? PC_ERR_OOM : PC_ERR_CUDA,
                      std::string("cuda: ") + what + ": " + cudaGetErrorString(e));
}

const char* kind_name(int k) {  // model_io.cpp:15-24
  switch (k) {
    case KIND_INPUT: return "input";
    case KIND_DENSE: return "dense";
    case KIND_CONV: return "conv";
    case KIND_RELU: return "relu";
    case KIND_JOIN: return "residual_join";
  }
  return "?";
}

struct HostLayer {
  int kind = 0, pred0 = -1, pred1 = -1;
  int in_w = 1, in_h = 1, in_c = 1, out_w = 1, out_h = 1, out_c = 1;
  int fw = 0, fh = 0, sw = 1, sh = 1, pw = 0, ph = 0;
  int head = -1;
  bool feeds_relu = false;
  long long numel() const { return (long long)out_w * out_h * out_c; }
  long long in_numel() const { return (long long)in_w * in_h * in_c; }
  std::vector<double> W, bias;  // host copies (reference layouts)
  LayerDev d{};
};

// Frame geometry tracked on the host (see FrameDev in kernels.cuh).
struct Frame {
  int layer = 0;
  bool dense = true;
  long long Ww = 0, Wh = 0, Mw = 0, Mh = 0, Aw = 0, Ah = 0;
};

struct Mat {
  double* lo = nullptr;
  double* hi = nullptr;
  double* K = nullptr;
  double* P = nullptr;  // predicted raw constants (S, E) per physical row (Walker::pk)
  cudaEvent_t pk_ready = nullptr;  // recorded on s4 after P
  double* part = nullptr;  // predicted-offer partials fused into the producing conv kernel
  int nparts = 0;
  long long cells = 0;
  Frame f;
  const int* src = nullptr;  // row map after a compaction (see MatDev::src)
  int phys = 0;              // physical rows in the buffers
  unsigned* stat = nullptr;  // magnitude statistics (MatDev::stat)
  cudaEvent_t ready = nullptr;  // recorded on the coefficient stream after the coefficients
};

MatDev md(const Mat& m) {
  MatDev d{m.lo, m.hi, m.K, m.cells};
  d.src = m.src;
  d.stat = m.stat;
  return d;
}

}  // namespace

struct Ctx;

struct pc_net {
  int device = 0;
  pc_options opt{};
  std::vector<HostLayer> L;
  std::vector<long long> off, pofs;  // neuron / grid-position offsets per layer
  long long total = 0, max_numel = 0;
  int n_out = 0;
  bool timing = true;
  bool profile = false;  // PC_PROFILE=1: per-kernel-class device time
  std::vector<void*> owned;  // device weights
  std::mutex pool_mu;
  std::vector<Ctx*> pool;    // idle per-call contexts
  std::vector<Ctx*> all;
  std::vector<Ctx*> bpool;  // idle image-batched contexts
  Ctx* primary = nullptr;
  // row sharding (pc_net_set_sharding)
  int shard_rank = 0, shard_world = 1;
  // conv steps onto a ReLU frame compute its live cells only (k_gbc_live);
  // off when a bias is -0 (an accumulator could then start at -0, and the
  // +0 terms of dead cells would matter) or PC_LIVE_CELLS=0
  bool live_cells = true;
  // pc_net_set_serial: walks on one stream and one pipeline, so per-launch
  // CUDA events time each kernel alone (roofline measurement)
  bool serial = false;
  pc_allgather_fn allgather = nullptr;
  void* allgather_user = nullptr;

  template <class T>
  T* dalloc(size_t n) {
    void* p = nullptr;
    ck(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)), "cudaMalloc");
    owned.push_back(p);
    return static_cast<T*>(p);
  }
};

// Per-call state: one verification in flight on its own stream. Concurrent
// pc_net_test* calls (or pc_net_test_batch workers) each hold one context,
// so images are verified concurrently on the same device and weights.
struct Ctx {
  pc_net* net;
  const std::vector<HostLayer>& L;
  const std::vector<long long>& off;
  const std::vector<long long>& pofs;
  const long long total, max_numel;
  const int n_out;
  pc_options opt;  // the net's options, overridden per call (pc_net_test_ex)
  const int device;
  const bool timing, profile;
  long long budget = 0;  // workspace bytes for one pass (0: derive)
  cudaStream_t stream = nullptr;   // coefficient stream (and everything outside a walk)
  cudaStream_t stream2 = nullptr;  // constants / concretisation / offers of a walk
  cudaStream_t stream3 = nullptr;  // exact concretisations + offers behind predicted compaction
  cudaStream_t stream4 = nullptr;  // predicted raw constants + predicted offers
  int *xmap = nullptr, *xq = nullptr;  // the exact offers' (unused) compaction outputs there
  std::vector<void*> owned;
  int* gen_n = nullptr;
  int* gen_pos = nullptr;
  int* gen_l = nullptr;
  int gen = 0;
  double *blo = nullptr, *bhi = nullptr, *rlo = nullptr, *rhi = nullptr, *dev = nullptr,
         *relax = nullptr;
  double* cand = nullptr;
  char* frozen = nullptr;
  int *live = nullptr, *rowq[2] = {nullptr, nullptr}, *perm = nullptr, *d_int = nullptr;
  double *vals = nullptr, *rvals = nullptr, *best = nullptr;
  char* has = nullptr;
  Counters* ctr = nullptr;
  Counters* ctr_sink = nullptr;  // the chain kernels' counting when it runs on s3 (launch_count_affine)
  char* arena = nullptr;
  size_t arena_cap = 0, arena_used = 0;
  unsigned* stats = nullptr;  // MagStat pool: 2 words per bound matrix of a walk
  size_t stats_cap = 0, stats_used = 0;
  // device-driven walks (graph mode): label, per-checkpoint live-row counts,
  // a second row-map buffer, and the captured whole-analysis graph
  // compaction ring of the host-driven schedule (Walker::checkpoint)
  static constexpr int kRing = 8;
  int* ring_map[kRing] = {};
  int* ring_q[kRing] = {};
  int* d_ringR = nullptr;
  cudaEvent_t ring_ev[kRing] = {};  // s3 work that last read a ring slot's rows / map
  double* ckat = nullptr;  // per live row: the checkpoint that froze it (k_ck_count)
  int* lv_cnt = nullptr;             // live channels per grid position of each ReLU layer
  unsigned short* lv_idx = nullptr;  // (k_live_build; read by the conv kernel k_gbc_live)
  int* lv_pref = nullptr;             // flat live-cell list per ReLU layer (k_live_flat):
  unsigned short *lv_fpos = nullptr, *lv_fch = nullptr;  // prefix per position, position, channel
  unsigned* lv_chm = nullptr;  // per ReLU layer: channels live at any position (16 words)
  int* un_idx = nullptr;  // per ReLU layer: ascending neurons with a nonzero relaxation offset
  int* un_cnt = nullptr;  // their count per (image, layer) (k_offset_list)
  int* d_label = nullptr;
  int* d_slots = nullptr;
  static constexpr int kSlots = 8192;
  int* perm2 = nullptr;
  cudaGraphExec_t graph = nullptr;
  int graph_label_mode = -1;       // label < 0 (analysis only) vs >= 0 when captured
  int graph_et = -1;               // early_term the graph was captured with
  bool graph_failed = false;
  pc_stats graph_st{};             // host-side counts accumulated while capturing
  std::vector<size_t> graph_dense_ev, graph_conv_ev;
  double graph_conv_bytes = 0;
  long long graph_conv_launches = 0;
  double graph_dense_bytes = 0, graph_dense_madds = 0;
  long long graph_launches = 0, graph_dense_launches = 0;
  // second walk pipeline (run_pass): its own streams and walk resources, the
  // analysis state aliased to this context's
  Ctx* helper = nullptr;
  bool is_helper = false;
  int nimg = 1;  // images whose state this context holds (image-batched walks)
  int* keys = nullptr;  // image-batched walks: the pass's live row keys
  double *sh_send = nullptr, *sh_recv = nullptr;  // sharding exchange buffers
  size_t sh_cap = 0;                              // doubles per rank
  int* h_int = nullptr;  // pinned
  // lazy compaction: per-checkpoint surviving-row counts (pinned) and events
  static constexpr int kCkSlots = 64;
  int* h_newR = nullptr;
  cudaEvent_t ck_ev[kCkSlots] = {};
  std::vector<cudaEvent_t> sync_pool;  // ordering events (no timing)
  size_t sync_used = 0;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  struct ProfEv {
    int cls;
    cudaStream_t st;
    size_t b, e;  // begin / end event indices (e == SIZE_MAX while open)
  };
  std::vector<ProfEv> prof;  // PC_PROFILE: one entry per profiled launch group
  std::vector<size_t> dense_ev;               // begin events of dense-coefficient launches
  std::vector<size_t> conv_ev;                // begin events of conv-coefficient launches

  explicit Ctx(pc_net* n)
      : net(n), L(n->L), off(n->off), pofs(n->pofs), total(n->total), max_numel(n->max_numel),
        n_out(n->n_out), opt(n->opt), device(n->device), timing(n->timing), profile(n->profile) {}

  template <class T>
  T* dalloc(size_t n) {
    void* p = nullptr;
    ck(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)), "cudaMalloc");
    owned.push_back(p);
    return static_cast<T*>(p);
  }

  // nimg > 1: an image-batched context (state for nimg images, row buffers
  // for nimg images' rows; see run_test_batched).
  void init(int n_images = 1) {
    nimg = n_images;
    ck(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "stream");
    ck(cudaStreamCreateWithFlags(&stream2, cudaStreamNonBlocking), "stream");
    ck(cudaStreamCreateWithFlags(&stream3, cudaStreamNonBlocking), "stream");
    ck(cudaStreamCreateWithFlags(&stream4, cudaStreamNonBlocking), "stream");
    const int nl = (int)L.size();
    const size_t T = (size_t)total * nimg, M = (size_t)max_numel * nimg;
    blo = dalloc<double>(T);
    bhi = dalloc<double>(T);
    rlo = dalloc<double>(T);
    rhi = dalloc<double>(T);
    dev = dalloc<double>(T);
    relax = dalloc<double>(8 * T);
    ck(cudaMemset(dev, 0, T * 8), "memset");
    cand = dalloc<double>(4 * M);
    frozen = dalloc<char>(M);
    live = dalloc<int>(M);
    rowq[0] = dalloc<int>(M);
    rowq[1] = dalloc<int>(M);
    keys = dalloc<int>(M);
    perm = dalloc<int>(2 * M);
    d_int = dalloc<int>(8 + nimg);
    vals = dalloc<double>(2 * M);
    rvals = dalloc<double>(2 * M);
    best = dalloc<double>(M);
    has = dalloc<char>(M);
    ctr = dalloc<Counters>(nimg);
    ctr_sink = dalloc<Counters>(nimg);
    gen_n = dalloc<int>(T);
    gen_pos = dalloc<int>((size_t)pofs[nl] * nimg);
    gen_l = dalloc<int>((size_t)nl * nimg);
    ck(cudaMemset(gen_n, 0, T * sizeof(int)), "memset");
    ck(cudaMemset(gen_pos, 0, (size_t)pofs[nl] * nimg * sizeof(int)), "memset");
    ck(cudaMemset(gen_l, 0, (size_t)nl * nimg * sizeof(int)), "memset");
    ck(cudaMallocHost(&h_int, 64 + (size_t)n_out * nimg + 64 * (size_t)nimg), "pinned");
    ck(cudaMallocHost(&h_newR, sizeof(int) * kCkSlots), "pinned");
    for (int k = 0; k < kRing; ++k) {
      ring_map[k] = dalloc<int>(2 * M);
      ring_q[k] = dalloc<int>(M);
    }
    d_ringR = dalloc<int>(kRing);
    ckat = dalloc<double>(M);
    xmap = dalloc<int>(2 * M);
    xq = dalloc<int>(M);
    lv_cnt = dalloc<int>((size_t)pofs[nl] * nimg);
    lv_idx = dalloc<unsigned short>(T);
    un_idx = dalloc<int>(T);
    lv_chm = dalloc<unsigned>((size_t)nl * 16 * nimg);
    lv_pref = dalloc<int>(((size_t)pofs[nl] + nl) * nimg);
    lv_fpos = dalloc<unsigned short>(T);
    lv_fch = dalloc<unsigned short>(T);
    un_cnt = dalloc<int>((size_t)nl * nimg);
    d_label = dalloc<int>(nimg);
    d_slots = dalloc<int>(kSlots);
    perm2 = dalloc<int>(2 * M);
    for (int k = 0; k < kCkSlots; ++k) ck(cudaEventCreateWithFlags(&ck_ev[k], cudaEventDisableTiming), "event");
    for (int k = 0; k < kRing; ++k) ck(cudaEventCreateWithFlags(&ring_ev[k], cudaEventDisableTiming), "event");
  }

  ~Ctx() {
    delete helper;
    if (stream) cudaStreamSynchronize(stream);
    if (stream2) cudaStreamSynchronize(stream2);
    if (stream3) cudaStreamSynchronize(stream3);
    if (stream4) cudaStreamSynchronize(stream4);
    for (void* p : owned) cudaFree(p);
    if (arena) cudaFree(arena);
    if (stats) cudaFree(stats);
    if (graph) cudaGraphExecDestroy(graph);
    if (sh_send) cudaFree(sh_send);
    if (sh_recv) cudaFree(sh_recv);
    if (h_int) cudaFreeHost(h_int);
    if (h_newR) cudaFreeHost(h_newR);
    for (cudaEvent_t e : ck_ev)
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : ring_ev)
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : sync_pool) cudaEventDestroy(e);
    for (cudaEvent_t e : ev_pool) cudaEventDestroy(e);
    if (stream) cudaStreamDestroy(stream);
    if (stream2) cudaStreamDestroy(stream2);
    if (stream3) cudaStreamDestroy(stream3);
    if (stream4) cudaStreamDestroy(stream4);
  }
};

namespace {

Ctx* acquire(pc_net* n) {
  {
    std::lock_guard<std::mutex> lk(n->pool_mu);
    if (!n->pool.empty()) {
      Ctx* c = n->pool.back();
      n->pool.pop_back();
      return c;
    }
  }
  Ctx* c = new Ctx(n);
  try {
    c->init();
  } catch (...) {
    delete c;
    throw;
  }
  std::lock_guard<std::mutex> lk(n->pool_mu);
  n->all.push_back(c);
  return c;
}

void release(pc_net* n, Ctx* c) {
  std::lock_guard<std::mutex> lk(n->pool_mu);
  (c->nimg > 1 ? n->bpool : n->pool).push_back(c);
}

// An image-batched context holding state for at least B images.
Ctx* acquire_batched(pc_net* n, int B) {
  {
    std::lock_guard<std::mutex> lk(n->pool_mu);
    for (size_t k = 0; k < n->bpool.size(); ++k)
      if (n->bpool[k]->nimg >= B) {
        Ctx* c = n->bpool[k];
        n->bpool.erase(n->bpool.begin() + k);
        return c;
      }
  }
  Ctx* c = new Ctx(n);
  try {
    c->init(B);
  } catch (...) {
    delete c;
    throw;
  }
  std::lock_guard<std::mutex> lk(n->pool_mu);
  n->all.push_back(c);
  return c;
}

struct CtxLease {
  pc_net* n;
  Ctx* c;
  explicit CtxLease(pc_net* net) : n(net), c(acquire(net)) {}
  ~CtxLease() { release(n, c); }
};

}  // namespace

namespace {

enum ProfClass { PROF_FWD, PROF_SEED, PROF_INIT, PROF_CHAIN_AFFINE, PROF_DENSE, PROF_GBC,
                 PROF_CHAIN_RELU, PROF_RELU, PROF_MERGE, PROF_CONC, PROF_OFFER, PROF_WRITEBACK,
                 PROF_PREDICT, PROF_N };
const char* kProfNames[PROF_N] = {"forward", "seed", "init", "chain_affine", "dense_coef",
                                  "gbc_coef", "chain_relu", "relu_coef", "merge", "concretize",
                                  "offer", "writeback", "predict"};
thread_local double g_prof_ms[PROF_N];
thread_local long long g_prof_n[PROF_N];
thread_local double g_gap_ms[PROF_N];
thread_local double g_gbc_window_madds = 0;
thread_local std::string g_pass_json = "[]";
thread_local std::string g_timeline_json = "[]";  // PC_PROFILE: [class, stream, start ms, end ms] per launch group  // PC_PROFILE: [[target, live rows, ms], ...], -1 = margin  // PC_PROFILE: madds of the conv steps if no coefficient were zero  // device idle (or unprofiled work) before each class

cudaEvent_t take_event(Ctx* n) {
  while (n->ev_pool.size() <= n->ev_used) {
    cudaEvent_t e;
    ck(cudaEventCreate(&e), "event");
    n->ev_pool.push_back(e);
  }
  return n->ev_pool[n->ev_used++];
}

void prof_begin(Ctx* n, int cls, cudaStream_t st = nullptr) {
  if (!n->profile) return;
  st = st ? st : n->stream;
  n->prof.push_back(Ctx::ProfEv{cls, st, n->ev_used, SIZE_MAX});
  ck(cudaEventRecord(take_event(n), st), "event");
}
void prof_end(Ctx* n, cudaStream_t st = nullptr) {
  if (!n->profile) return;
  st = st ? st : n->stream;
  for (size_t k = n->prof.size(); k-- > 0;)  // the open entry of this stream
    if (n->prof[k].st == st && n->prof[k].e == SIZE_MAX) {
      n->prof[k].e = n->ev_used;
      break;
    }
  ck(cudaEventRecord(take_event(n), st), "event");
}

// Ordering between the coefficient stream and the constants stream.
cudaEvent_t sync_event(Ctx* n) {
  while (n->sync_pool.size() <= n->sync_used) {
    cudaEvent_t e;
    ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    n->sync_pool.push_back(e);
  }
  return n->sync_pool[n->sync_used++];
}
// `to` waits for everything enqueued on `from` so far.
void stream_wait(Ctx* n, cudaStream_t to, cudaStream_t from) {
  cudaEvent_t e = sync_event(n);
  ck(cudaEventRecord(e, from), "event");
  ck(cudaStreamWaitEvent(to, e, 0), "wait");
}

// ---------------------------------------------------------------------------
// Validation (model_io.cpp:49-194)

int join_head_of(const std::vector<HostLayer>& L, int j) {  // model_io.cpp:137-160
  auto ancestors = [&](int start) {
    std::set<int> a;
    std::vector<int> st{start};
    while (!st.empty()) {
      int x = st.back();
      st.pop_back();
      if (!a.insert(x).second) continue;
      if (L[x].kind == KIND_INPUT) continue;
      st.push_back(L[x].pred0);
      if (L[x].kind == KIND_JOIN) st.push_back(L[x].pred1);
    }
    return a;
  };
  const std::set<int> aa = ancestors(L[j].pred0), ab = ancestors(L[j].pred1);
  int head = -1;
  for (int x : aa)
    if (ab.count(x)) head = std::max(head, x);
  if (head < 0) model_fail(j, "branches share no ancestor");
  return head;
}

struct Trace {
  bool dense = false;
  long long sw = 1, sh = 1;
};

Trace trace_branch(const std::vector<HostLayer>& L, int from, int head) {  // model_io.cpp:162-194
  Trace t;
  int cur = from;
  while (cur != head) {
    const HostLayer& l = L[cur];
    switch (l.kind) {
      case KIND_DENSE: t.dense = true; cur = l.pred0; break;
      case KIND_CONV: t.sw *= l.sw; t.sh *= l.sh; cur = l.pred0; break;
      case KIND_RELU: cur = l.pred0; break;
      case KIND_JOIN: {
        const int ih = join_head_of(L, cur);
        Trace in = trace_branch(L, l.pred0, ih);
        if (in.dense) t.dense = true;
        t.sw *= in.sw;
        t.sh *= in.sh;
        cur = ih;
        break;
      }
      default: model_fail(from, "branch walked past the input without meeting its head");
    }
  }
  return t;
}

void validate(const pc_layer_desc* layers, int n, int in_w, int in_h, int in_c,
              std::vector<HostLayer>& L) {
  if (in_w < 1 || in_h < 1 || in_c < 1) throw StatusError(PC_ERR_MODEL, "model: input shape must be positive");
  if (n < 1 || !layers || layers[0].kind != KIND_INPUT)
    throw StatusError(PC_ERR_MODEL, "model: layer 0 must be the input layer");
  if (n < 2) throw StatusError(PC_ERR_MODEL, "model: no layers");
  L.assign(n, HostLayer{});
  L[0].kind = KIND_INPUT;
  L[0].out_w = in_w; L[0].out_h = in_h; L[0].out_c = in_c;
  for (int i = 1; i < n; ++i) {
    const pc_layer_desc& d = layers[i];
    HostLayer& l = L[i];
    l.kind = d.kind;
    if (d.kind < KIND_INPUT || d.kind > KIND_JOIN) model_fail(i, "unknown kind");
    const int want = d.kind == KIND_JOIN ? 2 : 1;
    if (d.n_preds != want)
      model_fail(i, std::string(kind_name(d.kind)) + " needs " + std::to_string(want) + " predecessor(s)");
    for (int k = 0; k < want; ++k)
      if (d.preds[k] < 0 || d.preds[k] >= i)
        model_fail(i, "predecessor " + std::to_string(d.preds[k]) + " is not an earlier layer (cyclic or dangling)");
    l.pred0 = d.preds[0];
    l.pred1 = want == 2 ? d.preds[1] : -1;
    const HostLayer& p = L[l.pred0];
    l.in_w = p.out_w; l.in_h = p.out_h; l.in_c = p.out_c;
    auto check_finite = [&](const double* v, long long cnt) {
      for (long long t = 0; t < cnt; ++t)
        if (!std::isfinite(v[t])) model_fail(i, "malformed number '" + std::to_string(v[t]) + "'");
    };
    switch (d.kind) {
      case KIND_INPUT: model_fail(i, "only layer 0 may be the input");
      case KIND_DENSE: {
        if (d.n_out < 1) model_fail(i, "dense layer has no rows");
        if (!d.weights || !d.bias) model_fail(i, "dense layer without weights or bias");
        const long long nin = l.in_numel();
        check_finite(d.weights, nin * d.n_out);
        check_finite(d.bias, d.n_out);
        l.W.assign(d.weights, d.weights + nin * d.n_out);
        l.bias.assign(d.bias, d.bias + d.n_out);
        l.out_w = 1; l.out_h = 1; l.out_c = d.n_out;
        break;
      }
      case KIND_CONV: {
        if (d.fw < 1 || d.fh < 1) model_fail(i, "filter size must be positive");
        if (d.sw < 1 || d.sh < 1) model_fail(i, "stride must be positive");
        if (d.pw < 0 || d.ph < 0) model_fail(i, "negative padding");
        if (d.cin != l.in_c)
          model_fail(i, "in_channels " + std::to_string(d.cin) + " != predecessor channels " + std::to_string(l.in_c));
        if (d.cout < 1) model_fail(i, "out_channels must be positive");
        if (!d.weights || !d.bias) model_fail(i, "filter element count mismatch");
        const int ow = (l.in_w + 2 * d.pw - d.fw) / d.sw + 1;
        const int oh = (l.in_h + 2 * d.ph - d.fh) / d.sh + 1;
        if (ow < 1 || oh < 1) model_fail(i, "filter does not fit the input grid");
        if ((l.in_w + 2 * d.pw - d.fw) % d.sw != 0 || (l.in_h + 2 * d.ph - d.fh) % d.sh != 0)
          model_fail(i, "stride does not tile the padded input");
        const long long taps = (long long)d.fw * d.fh * d.cin * d.cout;
        check_finite(d.weights, taps);
        check_finite(d.bias, d.cout);
        l.fw = d.fw; l.fh = d.fh; l.sw = d.sw; l.sh = d.sh; l.pw = d.pw; l.ph = d.ph;
        l.W.assign(d.weights, d.weights + taps);
        l.bias.assign(d.bias, d.bias + d.cout);
        l.out_w = ow; l.out_h = oh; l.out_c = d.cout;
        break;
      }
      case KIND_RELU:
        if (p.kind == KIND_RELU) model_fail(i, "relu fed by relu");
        l.out_w = l.in_w; l.out_h = l.in_h; l.out_c = l.in_c;
        break;
      case KIND_JOIN: {
        const HostLayer& b = L[l.pred1];
        if (!(p.out_w == b.out_w && p.out_h == b.out_h && p.out_c == b.out_c))
          model_fail(i, "branch output shapes differ");
        l.out_w = l.in_w; l.out_h = l.in_h; l.out_c = l.in_c;
        l.head = join_head_of(L, i);
        const Trace ta = trace_branch(L, l.pred0, l.head), tb = trace_branch(L, l.pred1, l.head);
        if (!ta.dense && !tb.dense && (ta.sw != tb.sw || ta.sh != tb.sh))
          model_fail(i, "branches accumulate different strides");
        break;
      }
    }
  }
  for (int i = 1; i < n; ++i)
    if (L[i].kind == KIND_RELU) L[L[i].pred0].feeds_relu = true;
}

// ---------------------------------------------------------------------------
// Frames

FrameDev fdev(const Ctx* n, const Frame& f, int qlayer) {
  const HostLayer& l = n->L[f.layer];
  const HostLayer& Q = n->L[qlayer];
  FrameDev d{};
  d.G_w = l.out_w; d.G_h = l.out_h; d.C = l.out_c;
  if (f.dense) {
    d.S_w = d.G_w; d.S_h = d.G_h;
  } else {
    d.S_w = (int)std::min<long long>(f.Ww, d.G_w);
    d.S_h = (int)std::min<long long>(f.Wh, d.G_h);
    d.M_w = f.Mw; d.M_h = f.Mh; d.A_w = f.Aw; d.A_h = f.Ah;
  }
  d.q_w = Q.out_w; d.q_c = Q.out_c;
  return d;
}

Frame dense_frame(int layer) {
  Frame f;
  f.layer = layer;
  f.dense = true;
  return f;
}

// ---------------------------------------------------------------------------
// One walk context: a chunk of rows of one pass (or the margin rows).
//
// Two streams. The coefficient substitutions (dense / conv / relu / merge
// coefficients) form the walk's backbone on `s`; nothing on it depends on
// the row constants. The constant chains, concretisations and candidate
// offers — serial-latency kernels — run on `s2`, each waiting only for the
// coefficient matrix it reads (Mat::ready). So the chains of step k overlap
// the coefficient work of steps k+1, k+2, ...
//
// Early-termination compaction is an optimisation that never changes results
// (backsub.hpp:25-29): a frozen row's later offers are ignored. It is applied
// lazily: each checkpoint's surviving-row count is copied to pinned memory
// behind an event, and before each step the host polls (without blocking) the
// checkpoints that have completed; only when they show enough frozen rows does
// it drain `s2` and compact with the latest offer's row map.

struct Walker {
  Ctx* n;
  cudaStream_t s;
  int q;             // query layer
  bool dry = false;  // geometry dry run: count bytes per row only
  size_t dry_bytes = 0, dry_peak = 0, dry_allocs = 0;
  int R = 0;         // rows per polarity
  bool both = true;  // upper + lower rows (false: margin pass, lower only)
  int rq = 0;        // which row_q buffer is current
  const int* row_q = nullptr;
  bool allow_freeze = false, early_term = true, margin = false;
  pc_stats* st = nullptr;
  cudaStream_t s2 = nullptr;
  cudaStream_t s3 = nullptr;  // set: predicted compaction, exact checkpoint work on s3
  cudaStream_t s4 = nullptr;  // predicted raw constants and offers (pk())
  // device-driven walk (graph mode): R is the launch bound; the live count is
  // read by the kernels from dR, which each checkpoint's offers advance
  bool devr = false;
  const int* dR = nullptr;
  int slot_next = 0, pq = 0;
  // device-applied predicted compaction (pred_device()): the live row count
  // of the current row list on the device; R is then only a bound, lowered
  // as the checkpoints' counts reach the host (learn)
  const int* hdR = nullptr;
  std::vector<int> learn;
  // margin walks split over two contexts: where this walker's margin offers go
  double* mbest = nullptr;
  char* mhas = nullptr;
  // lazy compaction state: checkpoints launched since the last compaction
  int ck_next = 0;             // next pinned slot
  // Compaction ring: each checkpoint's offers write their row map, query list
  // and surviving count into a ring slot; a completed checkpoint's compaction
  // is applied to the current matrix while its rows are still in that
  // checkpoint's order (generation).
  struct Pending {
    int ck, slot, gen;
  };
  std::vector<Pending> pend;
  int gen = 0;
  int cur_slot = -1;  // ring slot holding the current row list (-1: the chunk's own list)
  int ck_index = 0;  // checkpoints issued by this walk (1-based index of the last)

  int nrows() const { return both ? 2 * R : R; }
  // fast numeric mode (pc_options.numeric_mode = 1)
  bool fast() const { return n->opt.numeric_mode == 1; }
  // rows frozen at an earlier checkpoint are skipped by the chain kernels
  const char* fz() const { return (allow_freeze && early_term && !margin) ? n->frozen : nullptr; }
  // image-batched walks (run_test_batched): row keys img * kq + neuron
  int kq = 0, nimg = 1;
  long long sst = 0;

  RowsDev rows() const {
    RowsDev r{row_q, nrows(), both ? R : 0};
    r.dR = devr ? dR : hdR;
    r.kq = kq;
    r.sst = sst;
    r.nimg = nimg;
    return r;
  }

  double* arena_take(size_t bytes) {
    bytes = (bytes + 255) & ~size_t(255);
    if (dry) {
      dry_bytes += bytes;
      dry_peak = std::max(dry_peak, dry_bytes);
      ++dry_allocs;
      return nullptr;
    }
    if (n->arena_used + bytes > n->arena_cap)
      throw StatusError(PC_ERR_OOM, "workspace exhausted (chunk sizing)");
    double* p = reinterpret_cast<double*>(n->arena + n->arena_used);
    n->arena_used += bytes;
    return p;
  }

  int alloc_rows() const { return dry ? (both ? 2 : 1) : nrows(); }

  size_t dry_stats = 0;
  unsigned* stat_take() {
    if (dry) {
      ++dry_stats;
      return nullptr;
    }
    if (n->stats_used + 2 > n->stats_cap) return nullptr;  // consumers then use the exact ops
    unsigned* p = n->stats + n->stats_used;
    n->stats_used += 2;
    return p;
  }

  Mat alloc(const Frame& f, bool withK) {
    Mat m;
    m.f = f;
    m.cells = frame_cells(fdev(n, f, q));
    m.phys = alloc_rows();
    m.stat = stat_take();
    m.lo = arena_take((size_t)m.phys * m.cells * sizeof(double));
    m.hi = arena_take((size_t)m.phys * m.cells * sizeof(double));
    if (withK) m.K = arena_take((size_t)m.phys * 4 * sizeof(double));
    return m;
  }

  // Constants of the next step's output: in place when m is compact,
  // otherwise a fresh compact array (the chain reads m.K through m.src).
  double* k_out(const Mat& m) {
    if (dry) {
      arena_take((size_t)alloc_rows() * 4 * sizeof(double));
      return nullptr;
    }
    // never in place when checkpoints lag on s3: they still read m.K
    return (m.src || s3) ? arena_take((size_t)nrows() * 4 * sizeof(double)) : m.K;
  }

  // m's coefficients are complete (recorded on s after their producer).
  void mark(Mat& m) {
    m.ready = sync_event(n);
    ck(cudaEventRecord(m.ready, s), "event");
  }
  // s2 may read m's coefficients.
  void need(const Mat& m) {
    if (m.ready) ck(cudaStreamWaitEvent(s2, m.ready, 0), "wait");
  }

  // Predicted compaction (checkpoint): PC_PREDICT=1 carries predicted raw
  // constants on s4 (launch_pk_*), so the predicted offers never wait for
  // the serial constant folds; PC_PREDICT=2 predicts from the exact
  // constants on s2. Eager schedule only: lazy / lagged walks leave frozen
  // rows in place, whose counters must then see the exact freezes in
  // stream order.
  int predict_mode() const {
    static const int predict = env_int("PC_PREDICT", 1);
    static const int lazy_all = env_int("PC_LAZY_COMPACT", 0);
    static const int lazy_rows = env_int("PC_LAZY_ROWS", 0);
    static const int lag_rows = env_int("PC_LAG_ROWS", 0);
    if (dry || !predict || !s3 || s3 == s2 || devr || margin || !allow_freeze || !early_term || lazy_all ||
        lazy_rows || lag_rows)
      return 0;
    return predict == 1 && s4 && s4 != s2 ? 1 : 2;
  }
  bool pk() const { return predict_mode() == 1; }
  // PC_PRED_DEVICE=1: the predicted compaction takes effect on the device
  // (the next step's streams wait for the predicted offers, the kernels read
  // the row count from the ring slot); the host never blocks on a checkpoint
  // and learns the counts one checkpoint late
  bool pred_device() const {
    static const int on = env_int("PC_PRED_DEVICE", 1);
    return on && pk();
  }
  // PassStats work counters of the chain kernels: counted on s3 instead
  // (launch_count_affine) when compaction is predicted
  Counters* cctr() const { return predict_mode() ? n->ctr_sink : n->ctr; }
  void count_affine(const LayerDev& L, bool is_conv, const Mat& m) {
    if (dry || !predict_mode()) return;
    if (m.ready) ck(cudaStreamWaitEvent(s3, m.ready, 0), "wait");
    launch_count_affine(s3, L, is_conv, rows(), fdev(n, m.f, q), md(m), fz(), n->ctr);
  }
  // lower R to the counts of completed checkpoints; block while more than
  // `keep` are unknown
  void learn_R(size_t keep) {
    while (!learn.empty()) {
      const int ckx = learn.front();
      if (learn.size() > keep) {
        ck(cudaEventSynchronize(n->ck_ev[ckx]), "sync");
      } else {
        const cudaError_t e = cudaEventQuery(n->ck_ev[ckx]);
        if (e == cudaErrorNotReady) break;
        ck(e, "event query");
      }
      R = std::min(R, n->h_newR[ckx]);
      learn.erase(learn.begin());
    }
  }
  // P of a step's output (taken in the dry run too, so the arena fits it)
  double* p_take() {
    if (dry) return arena_take((size_t)alloc_rows() * 2 * sizeof(double));
    return pk() ? arena_take((size_t)nrows() * 2 * sizeof(double)) : nullptr;
  }
  void need4(const Mat& m) {
    if (m.ready) ck(cudaStreamWaitEvent(s4, m.ready, 0), "wait");
  }
  cudaEvent_t pk_event() {
    cudaEvent_t e = sync_event(n);
    ck(cudaEventRecord(e, s4), "event");
    return e;
  }

  void dense_step(Mat& m) {  // backsub.hpp:343-399
    const HostLayer& L = n->L[m.f.layer];
    Mat out = alloc(dense_frame(L.pred0), false);
    out.K = k_out(m);
    out.P = p_take();
    if (!dry && pk()) {
      need4(m);
      prof_begin(n, PROF_PREDICT, s4);
      launch_pk_affine(s4, L.d, false, rows(), fdev(n, m.f, q), md(m), m.P, out.P);
      prof_end(n, s4);
      out.pk_ready = pk_event();
    }
    count_affine(L.d, false, m);
    if (!dry) {
      need(m);
      prof_begin(n, PROF_CHAIN_AFFINE, s2);
      launch_chain_affine(s2, L.d, false, rows(), fdev(n, m.f, q), md(m), out.K,
                          n->dev + n->off[m.f.layer], cctr(), fz(), fast());
      prof_end(n, s2);
      cudaEvent_t e0 = nullptr, e1 = nullptr;
      if (n->timing) {  // the roofline kernel is always timed (bench.py reads it)
        n->dense_ev.push_back(n->ev_used);
        e0 = take_event(n);
        e1 = take_event(n);
        // algorithmic bytes: coefficient rows in/out (16 B per interval) + weights once
        g_dense_bytes += 16.0 * nrows() * (double)(m.cells + out.cells) + 8.0 * m.cells * out.cells;
        g_dense_madds += (double)nrows() * m.cells * out.cells;
        ++g_dense_launches;
      }
      const HostLayer& P = n->L[L.pred0];
      const double* rx = P.kind == PC_RELU ? n->relax + 8 * n->off[P.pred0] : nullptr;
      launch_dense_coef(s, L.d, rows(), md(m), md(out), rx, e0, e1);
      mark(out);
    }
    m = out;
  }

  void gbc_step(Mat& m) {  // backsub.hpp:401-499
    const HostLayer& L = n->L[m.f.layer];
    Frame nf;
    nf.layer = L.pred0;
    nf.dense = m.f.dense;
    if (!nf.dense) {
      nf.Ww = (m.f.Ww - 1) * L.sw + L.fw;  // grow_width (depsets.hpp:27)
      nf.Wh = (m.f.Wh - 1) * L.sh + L.fh;
      nf.Mw = m.f.Mw * L.sw;  // step_origin (depsets.hpp:32-34), composed
      nf.Mh = m.f.Mh * L.sh;
      nf.Aw = m.f.Aw * L.sw - L.pw;
      nf.Ah = m.f.Ah * L.sh - L.ph;
    }
    Mat out = alloc(nf, false);
    out.K = k_out(m);
    out.P = p_take();
    if (!dry && pk()) {
      need4(m);
      prof_begin(n, PROF_PREDICT, s4);
      launch_pk_affine(s4, L.d, true, rows(), fdev(n, m.f, q), md(m), m.P, out.P);
      prof_end(n, s4);
      out.pk_ready = pk_event();
    }
    count_affine(L.d, true, m);
    // compacted nonzero input coefficients for the sparse conv kernel
    const bool sparse = gbc_sparse_wanted(L.d);
    SparseDev sp{};
    if (sparse) {
      const FrameDev fi0 = fdev(n, m.f, q);
      sp.ncell = fi0.S_w * fi0.S_h;
      sp.C = fi0.C;
      const size_t rows_n = (size_t)alloc_rows(), slots = rows_n * (size_t)m.cells;
      sp.cnt = reinterpret_cast<int*>(arena_take(rows_n * sp.ncell * sizeof(int)));
      sp.idx = reinterpret_cast<unsigned short*>(arena_take(slots * sizeof(unsigned short)));
      sp.lo = arena_take(slots * sizeof(double));
      sp.hi = arena_take(slots * sizeof(double));
      sp.dmask = reinterpret_cast<unsigned*>(arena_take(rows_n * 16 * sizeof(unsigned)));
    }
    // constant chains from the compacted coefficients (CTA per chain)
    static const int chain_scan = env_int("PC_CHAIN_SCAN", 0);
    const bool scan = sparse && chain_scan && m.cells >= 256;
    double* tmp = scan ? arena_take((size_t)alloc_rows() * 5 * sizeof(double)) : nullptr;
    // predicted compaction: partials of the raw concretisation from the conv
    // kernel (k_gbc_flat), so the predicted offer does not re-read the matrix
    static const int fuse_env = env_int("PC_PRED_FUSED", 1);
    double* fused_part = nullptr;
    if (fuse_env && n->L[L.pred0].kind == KIND_RELU && (dry || pk())) {
      const int nparts = gbc_flat_blocks(fdev(n, nf, q), L.d);
      fused_part = arena_take((size_t)alloc_rows() * nparts * 3 * sizeof(double));
    }
    if (!dry) {
      const FrameDev fi = fdev(n, m.f, q), fo = fdev(n, nf, q);
      if (!scan) {
        need(m);
        prof_begin(n, PROF_CHAIN_AFFINE, s2);
        launch_chain_affine(s2, L.d, true, rows(), fi, md(m), out.K, n->dev + n->off[m.f.layer],
                            cctr(), fz(), fast());
        prof_end(n, s2);
      }
      if (sparse) {
        ck(cudaMemsetAsync(sp.dmask, 0, (size_t)nrows() * 16 * sizeof(unsigned), s), "memset");
        launch_compact_cells(s, rows(), md(m), sp);
      }
      if (scan) {
        cudaEvent_t e = sync_event(n);
        ck(cudaEventRecord(e, s), "event");
        ck(cudaStreamWaitEvent(s2, e, 0), "wait");
        prof_begin(n, PROF_CHAIN_AFFINE, s2);
        launch_chain_affine_scan(s2, L.d, rows(), fi, md(m), sp, tmp, out.K, n->dev + n->off[m.f.layer],
                                 cctr(), fz());
        prof_end(n, s2);
      }
      prof_begin(n, PROF_GBC);
      if (n->timing) {  // the headline config's roofline kernel (bench.py reads it)
        n->conv_ev.push_back(n->ev_used);
        ck(cudaEventRecord(take_event(n), s), "event");
        // algorithmic bytes: coefficient rows in/out (16 B per interval) + the filter once
        g_conv_bytes += 16.0 * nrows() * (double)(m.cells + out.cells) +
                        8.0 * L.fw * L.fh * L.in_c * L.out_c;
        ++g_conv_launches;
      }
      static const int live_min_cin = env_int("PC_LIVE_MIN_CIN", 0);
      if (sparse && n->net->live_cells && n->L[L.pred0].kind == KIND_RELU && L.in_c >= live_min_cin) {
        const int nl = (int)n->L.size();
        static const int flat = env_int("PC_GBC_FLAT", 1);
        static const int tile = env_int("PC_GBC_TILE", 0);
        if (tile && L.in_c <= 512 && L.out_c <= 512) {
          launch_gbc_tile(s, L.d, rows(), fi, fo, sp, md(m), md(out), n->lv_chm + (size_t)L.pred0 * 16,
                          (long long)nl * 16, n->ctr);
        } else if (flat && fo.S_h <= 64 && (long long)fo.G_w * fo.G_h < 65536) {
          FlatDev fl{n->lv_pref + n->pofs[L.pred0] + L.pred0, n->lv_fpos + n->off[L.pred0],
                     n->lv_fch + n->off[L.pred0], n->pofs[nl] + nl, n->total};
          if (fused_part) {  // the predicted offer's partial sums in the conv epilogue
            fl.prlo = n->rlo + n->off[L.pred0];
            fl.prhi = n->rhi + n->off[L.pred0];
            fl.part = fused_part;
            out.part = fused_part;
            out.nparts = gbc_flat_blocks(fo, L.d);
          }
          launch_gbc_flat(s, L.d, rows(), fi, fo, sp, md(m), md(out), fl, n->ctr, fast());
        } else {
          const LiveDev lv{n->lv_cnt + n->pofs[L.pred0], n->lv_idx + n->off[L.pred0], n->pofs[nl], n->total};
          launch_gbc_live(s, L.d, rows(), fi, fo, sp, md(m), md(out), lv, n->ctr);
        }
      } else if (sparse)
        launch_gbc_sparse(s, L.d, rows(), fi, fo, sp, md(m), md(out));
      else
        launch_gbc_coef(s, L.d, rows(), fi, fo, md(m), md(out), n->d_int + 6);
      if (n->timing) ck(cudaEventRecord(take_event(n), s), "event");
      prof_end(n);
      if (n->profile)  // dense-window work of this step (all coefficients nonzero)
        g_gbc_window_madds += (double)nrows() * fo.S_w * fo.S_h * L.in_c * L.out_c *
                              ((double)L.fh * L.fw / ((double)L.sh * L.sw));
      mark(out);
    }
    m = out;
  }

  void relu_step(Mat& m) {  // backsub.hpp:501-568
    const HostLayer& L = n->L[m.f.layer];
    Frame nf = m.f;
    nf.layer = L.pred0;
    Mat out = alloc(nf, false);
    out.K = k_out(m);
    out.P = p_take();
    if (!dry && pk()) {
      need4(m);
      prof_begin(n, PROF_PREDICT, s4);
      launch_pk_relu(s4, rows(), fdev(n, m.f, q), md(m), m.P, out.P, n->relax + 8 * n->off[L.pred0],
                     n->un_idx + n->off[L.pred0], n->un_cnt + L.pred0, (int)n->L.size());
      prof_end(n, s4);
    }
    if (!dry) {
      const FrameDev f = fdev(n, m.f, q);
      const double* rx = n->relax + 8 * n->off[L.pred0];
      need(m);
      prof_begin(n, PROF_CHAIN_RELU, s2);
      static const int relu_list = env_int("PC_RELU_LIST", 1);
      if (relu_list)
        launch_chain_relu_list(s2, rows(), f, md(m), out.K, rx, n->un_idx + n->off[L.pred0],
                               n->un_cnt + L.pred0, (int)n->L.size(), fz());
      else
        launch_chain_relu(s2, rows(), f, md(m), out.K, rx, fz());
      prof_end(n, s2);
      prof_begin(n, PROF_RELU);
      launch_relu_coef(s, rows(), f, md(m), md(out), rx);
      prof_end(n);
      mark(out);
    }
    m = out;
  }

  void join_step(Mat& m) {  // backsub.hpp:694-715
    const HostLayer& L = n->L[m.f.layer];
    Mat a = m, b = m;  // both branches read m's rows (steps never write their input)
    a.f.layer = L.pred0;
    b.f.layer = L.pred1;
    // branch b starts from zero constants, laid out like m's rows
    b.K = arena_take((size_t)(dry ? alloc_rows() : m.phys) * 4 * sizeof(double));
    if (!dry) ck(cudaMemsetAsync(b.K, 0, (size_t)m.phys * 4 * sizeof(double), s2), "memset");
    b.P = (dry || pk()) ? arena_take((size_t)(dry ? alloc_rows() : m.phys) * 2 * sizeof(double)) : nullptr;
    if (!dry && pk()) ck(cudaMemsetAsync(b.P, 0, (size_t)m.phys * 2 * sizeof(double), s4), "memset");
    walk(a, L.head, false);
    walk(b, L.head, false);
    // align_add (backsub.hpp:610-688): union frame
    Frame u;
    u.layer = L.head;
    int dense_path = 0;
    if (a.f.dense || b.f.dense) {
      u = dense_frame(L.head);
      dense_path = a.f.dense ? 2 : 1;
    } else {
      if (a.f.Mw != b.f.Mw || a.f.Mh != b.f.Mh)
        throw StatusError(PC_ERR_LOGIC, "join: branch frames are not stride-aligned");
      u.dense = false;
      u.Mw = a.f.Mw; u.Mh = a.f.Mh;
      u.Aw = std::min(a.f.Aw, b.f.Aw);
      u.Ah = std::min(a.f.Ah, b.f.Ah);
      u.Ww = std::max(a.f.Aw + a.f.Ww, b.f.Aw + b.f.Ww) - u.Aw;
      u.Wh = std::max(a.f.Ah + a.f.Wh, b.f.Ah + b.f.Wh) - u.Ah;
    }
    Mat out = alloc(u, true);
    out.P = p_take();
    if (!dry && pk()) {
      launch_pk_merge(s4, rows(), md(a), a.P, md(b), b.P, out.P);
      out.pk_ready = pk_event();
    }
    if (!dry) {
      const FrameDev fa = fdev(n, a.f, q), fb = fdev(n, b.f, q), fu = fdev(n, u, q);
      prof_begin(n, PROF_MERGE);
      launch_merge(s, rows(), fa, fb, fu, dense_path, md(a), md(b), md(out), 1);
      prof_end(n);
      mark(out);
      launch_merge(s2, rows(), fa, fb, fu, dense_path, md(a), md(b), md(out), 2);
    }
    m = out;
  }

  // run_backsubstitution's checkpoint closure (backsub.hpp:1032-1054) or the
  // margin pass's (:1082-1091). Runs on s2 after m's coefficients.
  void checkpoint(Mat& m) {
    if (dry) return;
    if (!margin) ++ck_index;  // PassStats.checkpoints: walk_checkpoints / k_ck_count
    const int fl = m.f.layer;
    const long long o = n->off[fl];
    need(m);
    if (margin) {
      prof_begin(n, PROF_CONC, s2);
      launch_concretize(s2, rows(), fdev(n, m.f, q), md(m), n->blo + o, n->bhi + o, n->blo + o,
                        n->bhi + o, n->vals, n->rvals, nullptr, fast());
      prof_end(n, s2);
      launch_margin_offer(s2, R, n->vals, mbest ? mbest : n->best, mhas ? mhas : n->has);
      return;
    }
    // Predicted compaction (launch_pred_offer): the survivors of this
    // checkpoint come from a parallel sum with a proven error bound, on s4
    // from the predicted raw constants (or on s2 right behind the exact
    // ones); the exact concretisations and offers run on s3, off the path the
    // next step waits for.
    const int pmode = predict_mode();
    if (pmode) {
      int slot = free_slot();
      if (slot < 0) {
        resolve(m, 0);
        slot = free_slot();
      }
      // fused partials: the offer runs on the coefficient stream right
      // behind the conv kernel (and the predicted constants)
      const bool fused = pmode == 1 && m.part;
      cudaStream_t sp = fused ? s : pmode == 1 ? s4 : s2;
      // the exact work on s3 may still read this slot's rows / map from an
      // earlier generation
      ck(cudaStreamWaitEvent(sp, n->ring_ev[slot], 0), "wait");
      if (fused) {
        if (m.pk_ready) ck(cudaStreamWaitEvent(s, m.pk_ready, 0), "wait");
      } else if (pmode == 1) {
        need4(m);
      }
      prof_begin(n, PROF_OFFER, sp);
      if (fused)
        launch_pred_offer_parts(sp, rows(), R, md(m), m.P, m.part, m.nparts, n->frozen, n->ring_map[slot],
                                n->d_ringR + slot, n->ring_q[slot]);
      else
        launch_pred_offer(sp, rows(), R, fdev(n, m.f, q), md(m), pmode == 1 ? m.P : nullptr, n->rlo + o,
                          n->rhi + o, n->frozen, n->ring_map[slot], n->d_ringR + slot, n->ring_q[slot]);
      prof_end(n, sp);
      const int ckx = ck_next;
      ck_next = (ck_next + 1) % Ctx::kCkSlots;
      ck(cudaMemcpyAsync(n->h_newR + ckx, n->d_ringR + slot, sizeof(int), cudaMemcpyDeviceToHost, sp), "d2h");
      ck(cudaEventRecord(n->ck_ev[ckx], sp), "event");
      const bool on_device = pred_device();
      if (!on_device) pend.push_back(Pending{ckx, slot, gen});
      stream_wait(n, s3, s2);  // M and K of this checkpoint
      prof_begin(n, PROF_CONC, s3);
      launch_concretize(s3, rows(), fdev(n, m.f, q), md(m), n->blo + o, n->bhi + o, n->rlo + o,
                        n->rhi + o, n->vals, n->rvals, fz(), fast());
      prof_end(n, s3);
      launch_offer(s3, rows(), R, n->vals, n->rvals, n->cand, n->frozen, 1, 1, n->xmap, n->d_int + 3, n->xq,
                   n->ctr, n->ckat, ck_index);
      if (cur_slot >= 0) ck(cudaEventRecord(n->ring_ev[cur_slot], s3), "event");  // s3 read that slot
      if (on_device) {
        // the compaction takes effect now: every stream's next work reads
        // the slot's rows, map and count (the work above read the old ones)
        cudaEvent_t e = sync_event(n);
        ck(cudaEventRecord(e, sp), "event");
        for (cudaStream_t w : {s, s2, s3, s4})
          if (w != sp) ck(cudaStreamWaitEvent(w, e, 0), "wait");
        m.src = n->ring_map[slot];
        row_q = n->ring_q[slot];
        hdR = n->d_ringR + slot;
        cur_slot = slot;
        ++gen;
        learn.push_back(ckx);
      }
      return;
    }
    prof_begin(n, PROF_CONC, s2);
    static const int conc_scan = env_int("PC_CHAIN_SCAN", 0);
    if (conc_scan && m.cells >= 1024)
      launch_concretize_scan(s2, rows(), fdev(n, m.f, q), md(m), n->blo + o, n->bhi + o, n->rlo + o,
                             n->rhi + o, n->vals, n->rvals, fz());
    else
      launch_concretize(s2, rows(), fdev(n, m.f, q), md(m), n->blo + o, n->bhi + o, n->rlo + o,
                        n->rhi + o, n->vals, n->rvals, fz(), fast());
    prof_end(n, s2);
    int* new_q = n->rowq[rq ^ 1];
    if (devr) {
      // device-driven: the offers' compaction (new live count, row map, query
      // list) takes effect at once, without the host
      if (slot_next >= Ctx::kSlots) throw StatusError(PC_ERR_LOGIC, "graph: out of checkpoint slots");
      int* map = pq ? n->perm2 : n->perm;
      int* nR = n->d_slots + slot_next++;
      prof_begin(n, PROF_OFFER, s2);
      launch_offer(s2, rows(), R, n->vals, n->rvals, n->cand, n->frozen, allow_freeze ? 1 : 0,
                   early_term ? 1 : 0, map, nR, new_q, n->ctr, n->ckat, ck_index);
      prof_end(n, s2);
      if (allow_freeze && early_term) {
        m.src = map;
        dR = nR;
        rq ^= 1;
        row_q = n->rowq[rq];
        pq ^= 1;
        // the coefficient stream's next kernels read the new rows, map and count
        stream_wait(n, s, s2);
      }
      return;
    }
    if (!(allow_freeze && early_term)) {
      prof_begin(n, PROF_OFFER, s2);
      launch_offer(s2, rows(), R, n->vals, n->rvals, n->cand, n->frozen, allow_freeze ? 1 : 0,
                   early_term ? 1 : 0, n->perm, n->d_int + 1, new_q, n->ctr, n->ckat, ck_index);
      prof_end(n, s2);
      return;
    }
    int slot = free_slot();
    if (slot < 0) {
      resolve(m, 0);  // all slots referenced: settle the pending checkpoints
      slot = free_slot();
    }
    prof_begin(n, PROF_OFFER, s2);
    launch_offer(s2, rows(), R, n->vals, n->rvals, n->cand, n->frozen, 1, 1, n->ring_map[slot],
                 n->d_ringR + slot, n->ring_q[slot], n->ctr, n->ckat, ck_index);
    prof_end(n, s2);
    const int ckx = ck_next;
    ck_next = (ck_next + 1) % Ctx::kCkSlots;
    ck(cudaMemcpyAsync(n->h_newR + ckx, n->d_ringR + slot, sizeof(int), cudaMemcpyDeviceToHost, s2), "d2h");
    ck(cudaEventRecord(n->ck_ev[ckx], s2), "event");
    pend.push_back(Pending{ckx, slot, gen});
  }

  // Round robin: a reused slot was last read kRing checkpoints ago, so the
  // wait on its ring event (the exact offers behind the serial folds) has
  // long completed.
  int slot_rr = 0;
  int free_slot() {
    for (int u = 0; u < Ctx::kRing; ++u) {
      const int k = (slot_rr + u) % Ctx::kRing;
      if (k == cur_slot) continue;
      bool used = false;
      for (const Pending& p : pend) used |= p.slot == k;
      if (!used) {
        slot_rr = (k + 1) % Ctx::kRing;
        return k;
      }
    }
    return -1;
  }

  // Settle pending checkpoints until at most `keep` remain (blocking on their
  // events); apply the compaction of a current-generation checkpoint that
  // dropped rows. Later checkpoints of the old generation are then stale:
  // their freezes stand (frozen[] / candidates), their row maps are dropped.
  void resolve(Mat& m, int keep) {
    while ((int)pend.size() > keep) {
      const Pending p = pend.front();
      pend.erase(pend.begin());
      ck(cudaEventSynchronize(n->ck_ev[p.ck]), "sync");
      apply(m, p);
    }
  }
  void apply(Mat& m, const Pending& p) {
    const int newR = n->h_newR[p.ck];
    if (p.gen != gen) return;
    if (newR >= R) return;
    m.src = n->ring_map[p.slot];
    row_q = n->ring_q[p.slot];
    R = newR;
    cur_slot = p.slot;
    ++gen;
  }


  // compact_rows on both polarities (backsub.hpp:820-845) when enough rows
  // froze: the surviving rows stay in place and the next step reads them
  // through the latest offer's row map.
  // compact_rows on both polarities (backsub.hpp:820-845): the surviving
  // rows stay in place and the next step reads them through the row map.
  // Schedules (results identical; only the wasted work on frozen rows and
  // the waiting differ):
  //   eager  - before each step, wait for the last checkpoint (the
  //            reference's schedule);
  //   lagged - for few rows (R <= PC_LAG_ROWS; off by default: measured on
  //            ResNet-34, the extra conv step on rows that just froze costs
  //            more than the overlap wins): keep the last checkpoint pending
  //            and apply the one before, so a step's concretisation and
  //            offers overlap the next step;
  //   lazy   - (PC_LAZY_COMPACT=1) never block; apply the newest completed
  //            checkpoint once it froze >= 1/8 of the rows.
  void maybe_compact(Mat& m) {
    if (dry || devr || !(allow_freeze && early_term)) return;
    if (pred_device()) {  // compaction already applied on the device
      learn_R(1);
      return;
    }
    static const int lazy_all = env_int("PC_LAZY_COMPACT", 0);
    static const int lazy_rows = env_int("PC_LAZY_ROWS", 0);
    static const int lag_rows = env_int("PC_LAG_ROWS", 0);
    const bool lazy = lazy_all || R <= lazy_rows;
    if (lazy) {
      while (!pend.empty()) {
        const cudaError_t e = cudaEventQuery(n->ck_ev[pend.front().ck]);
        if (e == cudaErrorNotReady) break;
        ck(e, "event query");
        const Pending p = pend.front();
        if (p.gen == gen && 8 * (R - n->h_newR[p.ck]) < R && n->h_newR[p.ck] > 0) {
          pend.erase(pend.begin());  // not worth it yet; a later checkpoint supersedes it
          continue;
        }
        pend.erase(pend.begin());
        apply(m, p);
      }
      return;
    }
    resolve(m, R <= lag_rows ? 1 : 0);
  }

  // True when the next advance() would not block the host: the eager
  // schedule resolves every pending checkpoint before a step, so it is ready
  // once the newest one has completed (offers complete in stream order).
  bool ready() const {
    static const int lazy = env_int("PC_LAZY_COMPACT", 0);
    static const int lazy_rows = env_int("PC_LAZY_ROWS", 0);
    static const int lag_rows = env_int("PC_LAG_ROWS", 0);
    if (pred_device())
      return learn.size() <= 1 || cudaEventQuery(n->ck_ev[learn[learn.size() - 2]]) != cudaErrorNotReady;
    if (dry || devr || !(allow_freeze && early_term) || lazy || R <= lazy_rows || pend.empty()) return true;
    const size_t keep = R <= lag_rows ? 1 : 0;
    if (pend.size() <= keep) return true;
    const cudaError_t e = cudaEventQuery(n->ck_ev[pend[pend.size() - 1 - keep].ck]);
    if (e == cudaErrorNotReady) return false;
    ck(e, "event query");
    return true;
  }
  // Block until ready() (the checkpoint the next step waits for).
  void wait_ready() const {
    if (pred_device()) {
      if (learn.size() > 1) ck(cudaEventSynchronize(n->ck_ev[learn[learn.size() - 2]]), "sync");
      return;
    }
    static const int lag_rows = env_int("PC_LAG_ROWS", 0);
    const size_t keep = R <= lag_rows ? 1 : 0;
    if (pend.size() > keep) ck(cudaEventSynchronize(n->ck_ev[pend[pend.size() - 1 - keep].ck]), "sync");
  }

  // walk_back (backsub.hpp:854-893)
  void walk(Mat& m, int stop, bool ckpt) {
    bool pending = false;
    while (advance(m, stop, ckpt, pending)) {
    }
  }

  // One iteration of walk_back: compaction, one step, its checkpoint; false
  // once the walk is over (the final checkpoint after a relu included), so
  // several walkers can be driven step by step in turn.
  bool advance(Mat& m, int stop, bool ckpt, bool& pending) {
    if (m.f.layer == stop) {
      if (pending && ckpt) checkpoint(m);
      pending = false;
      return false;
    }
    if (ckpt) maybe_compact(m);
    if (!dry && R == 0) return false;
    const HostLayer& L = n->L[m.f.layer];
    switch (L.kind) {
      case KIND_DENSE:
        dense_step(m);
        if (ckpt) checkpoint(m);
        pending = false;
        break;
      case KIND_CONV:
        gbc_step(m);
        if (ckpt) checkpoint(m);
        pending = false;
        break;
      case KIND_RELU:
        relu_step(m);
        pending = true;
        break;
      case KIND_JOIN:
        join_step(m);
        if (ckpt) checkpoint(m);
        pending = false;
        break;
      default:
        throw StatusError(PC_ERR_LOGIC, "walk: frame fell through the input layer");
    }
    return true;
  }
};

Frame initial_frame(const Ctx* n, int t, bool affine) {
  const HostLayer& Q = n->L[t];
  if (affine) {
    if (Q.kind == KIND_DENSE) return dense_frame(Q.pred0);
    Frame f;
    f.layer = Q.pred0;
    f.dense = false;
    f.Ww = Q.fw; f.Wh = Q.fh;
    f.Mw = Q.sw; f.Mh = Q.sh;
    f.Aw = -Q.pw; f.Ah = -Q.ph;
    return f;
  }
  if (Q.out_w == 1 && Q.out_h == 1) return dense_frame(t);
  Frame f;
  f.layer = t;
  f.dense = false;
  f.Ww = 1; f.Wh = 1; f.Mw = 1; f.Mh = 1; f.Aw = 0; f.Ah = 0;
  return f;
}

// Checkpoints of a full walk of pass t (no row leaving early): the affine
// init, every dense / conv / join step, and a final one when the walk reaches
// the input through a relu (walk_back, backsub.hpp:854-893; :1056).
int walk_checkpoints(const Ctx* n, const Frame& f0, bool affine) {
  int cnt = affine ? 1 : 0, layer = f0.layer;
  bool pending = false;
  while (layer != 0) {
    const HostLayer& L = n->L[layer];
    if (L.kind == KIND_RELU) {
      pending = true;
      layer = L.pred0;
      continue;
    }
    ++cnt;
    pending = false;
    layer = L.kind == KIND_JOIN ? L.head : L.pred0;
  }
  return cnt + (pending ? 1 : 0);
}

// The reference's rows_per_chunk (backsub.hpp:969-987) over its own geometry
// dry run (peak_row_cells / sim_walk, :895-967: unclamped cuboid widths, the
// additive join-union rule). The GPU sizes its own chunks from the clamped
// frames (walk_size); this only reproduces the reference's chunking for
// PassStats.checkpoints, which counts per chunk. memory_budget: the call's
// (the reference default, 1 GiB, when 0).
struct SimSt {
  bool dense;
  long long ww, wh;
};
long long sim_cells(const Ctx* n, int layer, const SimSt& st) {
  const HostLayer& L = n->L[layer];
  return st.dense ? L.numel() : st.ww * st.wh * L.out_c;
}
std::pair<SimSt, long long> sim_walk(const Ctx* n, int layer, SimSt st, int stop) {
  long long peak = sim_cells(n, layer, st);
  while (layer != stop) {
    const HostLayer& L = n->L[layer];
    if (layer == 0) return {st, peak};
    switch (L.kind) {
      case KIND_DENSE:
        st = {true, 0, 0};
        layer = L.pred0;
        break;
      case KIND_CONV:
        if (!st.dense) {  // grow_width on int, after the reference's 2^20 clamp
          st.ww = (long long)(((int)std::min<long long>(st.ww, 1 << 20) - 1) * L.sw + L.fw);
          st.wh = (long long)(((int)std::min<long long>(st.wh, 1 << 20) - 1) * L.sh + L.fh);
        }
        layer = L.pred0;
        break;
      case KIND_RELU:
        layer = L.pred0;
        break;
      case KIND_JOIN: {
        const auto a = sim_walk(n, L.pred0, st, L.head);
        const auto b = sim_walk(n, L.pred1, st, L.head);
        peak = std::max(peak, a.second + b.second);
        layer = L.head;
        if (a.first.dense || b.first.dense) st = {true, 0, 0};
        else st = {false, a.first.ww + b.first.ww, a.first.wh + b.first.wh};
        break;
      }
      default:
        return {st, peak};
    }
    peak = std::max(peak, sim_cells(n, layer, st));
  }
  return {st, peak};
}
long long ref_rows_per_chunk(const Ctx* n, int t) {
  if (n->opt.chunk_rows > 0) return n->opt.chunk_rows;
  const HostLayer& Q = n->L[t];
  SimSt st{true, 0, 0};
  int start = t;
  if (Q.kind == KIND_CONV) {
    st = {false, Q.fw, Q.fh};
    start = Q.pred0;
  } else if (Q.kind == KIND_DENSE) {
    start = Q.pred0;
  } else if (Q.out_w > 1 || Q.out_h > 1) {
    st = {false, 1, 1};
  }
  const long long cells = std::max<long long>(sim_walk(n, start, st, 0).second, 1);
  const long long per_row = cells * 16 * 4 + 1024;
  const long long mb = n->opt.memory_budget > 0 ? n->opt.memory_budget : (1ll << 30);
  return std::max<long long>(1, std::max(mb, per_row) / per_row);
}

// After a pass's walks: PassStats.checkpoints under the reference's chunking
// (keys = the pass's live rows, count at n_keys on the device).
void count_checkpoints(Ctx* n, int t, bool affine, bool allow_freeze, const int* keys,
                       const int* n_keys, int kq, int nimg) {
  const int T = walk_checkpoints(n, initial_frame(n, t, affine), affine);
  const bool all_full = !(allow_freeze && n->opt.early_term);
  launch_ck_count(n->stream, keys, n_keys, kq, nimg, ref_rows_per_chunk(n, t), T, all_full ? 1 : 0,
                  n->ckat, n->ctr);
}

// Workspace of pass t: bytes per query row (both polarities; the arena is a
// bump allocator reset per chunk, so this is the walk's total) and the number
// of allocations (each may round up by < 256 B).
struct WalkSize {
  size_t per_row, allocs, stats;
};

WalkSize walk_size(Ctx* n, int t, bool affine, bool both) {
  Walker w{n, nullptr, t};
  w.dry = true;
  w.both = both;
  pc_stats dummy{};
  w.st = &dummy;
  Mat m = w.alloc(initial_frame(n, t, affine), true);
  m.P = w.p_take();
  w.walk(m, 0, false);
  return WalkSize{w.dry_peak, w.dry_allocs, w.dry_stats};
}

// A fresh statistics pool for one walk: `count` matrices, all slots reset.
void reset_stats(Ctx* n, size_t count) {
  const size_t words = 2 * std::max<size_t>(count, 1);
  if (words > n->stats_cap) {
    if (n->stats) cudaFree(n->stats);
    n->stats = nullptr;
    n->stats_cap = 0;
    ck(cudaMalloc(&n->stats, words * sizeof(unsigned)), "stats");
    n->stats_cap = words;
  }
  ck(cudaMemsetAsync(n->stats, 0xFF, words * sizeof(unsigned), n->stream), "memset");
  n->stats_used = 0;
}

// Grow-only workspace. cudaFree / cudaMalloc synchronise the device and take
// long for multi-GB buffers, so growth rounds up (1.25x, 64 MiB granules) and
// is counted (PC_PROFILE reports it).
thread_local double g_alloc_ms = 0;
thread_local int g_allocs = 0;
void ensure_arena(Ctx* n, size_t bytes) {
  if (bytes <= n->arena_cap) return;
  const auto t0 = std::chrono::steady_clock::now();
  size_t want = std::max(bytes, n->arena_cap + n->arena_cap / 4);
  want = (want + (64u << 20) - 1) & ~(size_t)((64u << 20) - 1);
  if (n->arena) cudaFree(n->arena);
  n->arena = nullptr;
  n->arena_cap = 0;
  if (cudaMalloc(&n->arena, want) != cudaSuccess) {  // headroom unavailable: exact size
    cudaGetLastError();
    want = bytes;
    ck(cudaMalloc(&n->arena, want), "arena");
  }
  n->arena_cap = want;
  g_alloc_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  ++g_allocs;
}

long long budget_of(const Ctx* n) {
  if (n->opt.memory_budget > 0) return n->opt.memory_budget;
  return n->budget > 0 ? n->budget : (16ll << 30);
}

// ---------------------------------------------------------------------------
// Row sharding (pc_net_set_sharding): slices and the all-gather exchange.

inline long long slice_begin(long long n, int r, int w) { return n * r / w; }

// Rows per polarity of one walker: row kernels put the 2R rows of a walk in
// gridDim.y (<= 65535), so every chunk is capped here (results are
// chunk-invariant, backsub.hpp:25-29).
constexpr long long kMaxWalkRows = 32767;

void ensure_shard_buffers(Ctx* n, size_t per_rank_doubles) {
  if (per_rank_doubles <= n->sh_cap) return;
  if (n->sh_send) cudaFree(n->sh_send);
  if (n->sh_recv) cudaFree(n->sh_recv);
  n->sh_send = n->sh_recv = nullptr;
  n->sh_cap = 0;
  ck(cudaMalloc(&n->sh_send, per_rank_doubles * sizeof(double)), "shard buffers");
  ck(cudaMalloc(&n->sh_recv, per_rank_doubles * sizeof(double) * n->net->shard_world), "shard buffers");
  n->sh_cap = per_rank_doubles;
}

void exchange(Ctx* n, size_t bytes) {
  const pc_net* net = n->net;
  if (net->allgather(net->allgather_user, n->sh_send, n->sh_recv, bytes, (void*)n->stream) != 0)
    throw StatusError(PC_ERR_CUDA, "sharding: allgather callback failed");
}

// Gather every rank's slice of `width` doubles per row of dst (row = live[g]
// or g) so all ranks hold the full array.
void allgather_rows(Ctx* n, const int* live, int n_rows, int width, double* dst) {
  const int W = n->net->shard_world, r = n->net->shard_rank;
  const int per = (n_rows + W - 1) / W;
  ensure_shard_buffers(n, (size_t)per * width);
  const int b = (int)slice_begin(n_rows, r, W), e = (int)slice_begin(n_rows, r + 1, W);
  launch_shard_pack(n->stream, live, b, e - b, width, dst, n->sh_send);
  exchange(n, (size_t)per * width * sizeof(double));
  launch_shard_unpack(n->stream, live, n_rows, W, per, width, n->sh_recv, dst);
}

// run_backsubstitution (backsub.hpp:993-1065)
// The second walk pipeline of context n: a context of its own (streams,
// arena, ring, concretisation buffers) whose analysis state (bounds,
// relaxations, deviations, candidates, freeze flags, live list, counters) is
// n's, so two halves of a pass's rows can be walked concurrently.
Ctx* helper_of(Ctx* n) {
  if (n->helper) return n->helper;
  Ctx* h = new Ctx(n->net);
  try {
    h->init();
  } catch (...) {
    delete h;
    throw;
  }
  h->is_helper = true;
  h->blo = n->blo; h->bhi = n->bhi; h->rlo = n->rlo; h->rhi = n->rhi;
  h->dev = n->dev; h->relax = n->relax; h->cand = n->cand; h->frozen = n->frozen;
  h->ckat = n->ckat;
  h->lv_cnt = n->lv_cnt;
  h->lv_idx = n->lv_idx;
  h->un_idx = n->un_idx;
  h->lv_chm = n->lv_chm;
  h->lv_pref = n->lv_pref;
  h->lv_fpos = n->lv_fpos;
  h->lv_fch = n->lv_fch;
  h->un_cnt = n->un_cnt;
  h->live = n->live; h->ctr = n->ctr;
  h->gen_n = n->gen_n; h->gen_pos = n->gen_pos; h->gen_l = n->gen_l;
  h->budget = n->budget;
  n->helper = h;
  return h;
}

// One chunk walker: rows live[base .. base + R) of pass t on context c.
struct ChunkWalk {
  Walker w;
  Mat m;
  bool pending = false, running = true;
};

void start_chunk(Ctx* c, ChunkWalk& cw, int t, bool affine, long long base, int R,
                 bool allow_freeze, bool et, pc_stats* st, const WalkSize& ws) {
  const HostLayer& Q = c->L[t];
  const long long o = c->off[t];
  cudaStream_t s = c->stream;
  c->arena_used = 0;
  reset_stats(c, ws.stats);
  Walker& w = cw.w;
  w.s2 = c->net->serial ? c->stream : c->stream2;
  w.s3 = c->net->serial ? c->stream : c->stream3;
  w.s4 = c->net->serial ? c->stream : c->stream4;
  w.R = R;
  w.both = true;
  w.allow_freeze = allow_freeze;
  w.early_term = et;
  w.st = st;
  ck(cudaMemcpyAsync(c->rowq[0], c->live + base, sizeof(int) * R, cudaMemcpyDeviceToDevice, s), "d2d");
  w.rq = 0;
  w.row_q = c->rowq[0];
  Frame f0 = initial_frame(c, t, affine);
  cw.m = w.alloc(f0, true);
  if (affine)
    launch_init_affine(s, Q.d, w.rows(), fdev(c, f0, t), c->dev + o, md(cw.m));
  else
    launch_init_identity(s, w.rows(), fdev(c, f0, t), md(cw.m));
  w.mark(cw.m);
  cw.m.P = w.p_take();
  if (w.pk()) {
    w.need4(cw.m);
    launch_pk_init(w.s4, w.rows(), md(cw.m), cw.m.P);
  }
  if (affine) w.checkpoint(cw.m);  // the init itself is an affine step (:1056)
}

// Device-driven pass (graph mode): one chunk sized for every neuron of the
// layer; the live count and rows come from the seed on the device.
void run_pass_graph(Ctx* n, int t, bool allow_freeze, pc_stats* st) {
  cudaStream_t s = n->stream;
  const HostLayer& Q = n->L[t];
  const int N = (int)Q.numel();
  const long long o = n->off[t];
  const bool et = n->opt.early_term != 0;
  launch_seed(s, N, n->blo + o, n->bhi + o, n->rlo + o, n->rhi + o, allow_freeze ? 1 : 0, et ? 1 : 0,
              n->cand, n->frozen, n->live, n->d_int, &n->ctr->pad);
  launch_ck_fill(s, n->live, n->d_int, N, n->ckat);
  st->rows_total += N;
  const bool affine = Q.kind == KIND_DENSE || Q.kind == KIND_CONV;
  const WalkSize ws = walk_size(n, t, affine, true);
  n->arena_used = 0;
  reset_stats(n, ws.stats);
  Walker w{n, s, t};
  w.s2 = n->net->serial ? n->stream : n->stream2;
  w.devr = true;
  w.dR = n->d_int;  // the seed's live count
  w.R = N;
  w.both = true;
  w.allow_freeze = allow_freeze;
  w.early_term = et;
  w.st = st;
  w.rq = 0;
  w.row_q = n->live;  // the seed's live list (stable order)
  Frame f0 = initial_frame(n, t, affine);
  Mat m = w.alloc(f0, true);
  if (affine)
    launch_init_affine(s, Q.d, w.rows(), fdev(n, f0, t), n->dev + o, md(m));
  else
    launch_init_identity(s, w.rows(), fdev(n, f0, t), md(m));
  w.mark(m);
  if (affine) w.checkpoint(m);
  w.walk(m, 0, true);
  stream_wait(n, s, n->stream2);
  count_checkpoints(n, t, affine, allow_freeze, n->live, n->d_int, 0, 1);
  ++n->gen;
  launch_writeback(s, N, Q.out_c, t, n->cand, n->blo + o, n->bhi + o, n->rlo + o, n->rhi + o,
                   Q.feeds_relu ? n->relax + 8 * o : nullptr, n->gen_n, n->gen_pos, n->gen_l,
                   n->gen, o, n->pofs[t]);
}

void run_pass(Ctx* n, int t, bool allow_freeze, pc_stats* st) {
  NvtxRange nv("pass", t);
  cudaStream_t s = n->stream;
  const HostLayer& Q = n->L[t];
  const int N = (int)Q.numel();
  const long long o = n->off[t];
  const bool et = n->opt.early_term != 0;
  prof_begin(n, PROF_SEED);
  launch_seed(s, N, n->blo + o, n->bhi + o, n->rlo + o, n->rhi + o, allow_freeze ? 1 : 0, et ? 1 : 0,
              n->cand, n->frozen, n->live, n->d_int, &n->ctr->pad);
  prof_end(n);
  launch_ck_fill(s, n->live, n->d_int, N, n->ckat);
  ck(cudaMemcpyAsync(n->h_int, n->d_int, sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  ck(cudaStreamSynchronize(s), "sync");
  const int n_live = n->h_int[0];
  st->rows_total += N;
  const bool affine = Q.kind == KIND_DENSE || Q.kind == KIND_CONV;
  // this rank's slice of the live rows (all of them unsharded)
  const int W = n->net->shard_world;
  const long long lb = slice_begin(n_live, n->net->shard_rank, W);
  const long long le = slice_begin(n_live, n->net->shard_rank + 1, W);
  if (le > lb) {
    const WalkSize ws = walk_size(n, t, affine, true);
    long long chunk = n->opt.chunk_rows > 0
                          ? n->opt.chunk_rows
                          : std::max<long long>(1, budget_of(n) / (long long)ws.per_row);
    chunk = std::min<long long>(chunk, le - lb);
    // Two walk pipelines: the rows of a chunk are split between this context
    // and its helper and the two walks are advanced step by step in turn, so
    // one half's conv substitutions overlap the other half's serial constant
    // / concretisation chains and checkpoint round trips (rows are
    // independent, backsub.hpp:31-34; results identical).
    static const int pipes = env_int("PC_PIPES", 2);
    static const int pipe_min = env_int("PC_PIPE_MIN_ROWS", 4);
    const int K = (pipes >= 2 && !n->is_helper && chunk >= pipe_min && !n->net->serial)
                      ? (int)std::min<long long>(std::min(pipes, 4), chunk)
                      : 1;
    // rows of a walk ride in gridDim.y (both polarities: 2R <= 65535)
    chunk = std::min<long long>(chunk, (long long)K * kMaxWalkRows);
    std::vector<Ctx*> cx{n};  // the pipelines' contexts: n and its helper chain
    while ((int)cx.size() < K) cx.push_back(helper_of(cx.back()));
    const long long part = (chunk + K - 1) / K;
    for (Ctx* c : cx) ensure_arena(c, ws.per_row * (size_t)part + 256 * ws.allocs + (1 << 20));
    for (long long base = lb; base < le; base += chunk) {
      const int R = (int)std::min<long long>(chunk, le - base);
      if (K > 1 && R >= pipe_min && R >= K) {
        std::vector<ChunkWalk> cw;
        cw.reserve(K);
        long long b0 = base;
        for (int k = 0; k < K; ++k) {
          const int Rk = R / K + (k >= K - R % K ? 1 : 0);
          Ctx* c = cx[k];
          if (k) stream_wait(n, c->stream, s);  // the seed and live list are on s
          cw.push_back(ChunkWalk{Walker{c, c->stream, t}});
          start_chunk(c, cw.back(), t, affine, b0, Rk, allow_freeze, et, st, ws);
          b0 += Rk;
        }
        // advance whichever walk's last checkpoint has resolved, so the host
        // never blocks on one pipeline while another could launch work
        for (;;) {
          bool moved = false, any = false;
          for (ChunkWalk& w : cw) {
            if (!w.running) continue;
            any = true;
            if (w.w.ready()) {
              w.running = w.w.advance(w.m, 0, true, w.pending);
              moved = true;
            }
          }
          if (!any) break;
          if (!moved)
            for (ChunkWalk& w : cw)
              if (w.running) {
                w.w.wait_ready();
                break;
              }
        }
        for (Ctx* c : cx)
          for (cudaStream_t q : {c->stream, c->stream2, c->stream3, c->stream4})
            if (q != s) stream_wait(n, s, q);
        for (size_t k = 1; k < cx.size(); ++k) stream_wait(n, cx[k]->stream, s);  // arenas reused after s
        continue;
      }
      ChunkWalk a{Walker{n, s, t}};
      start_chunk(n, a, t, affine, base, R, allow_freeze, et, st, ws);
      a.w.walk(a.m, 0, true);
      stream_wait(n, s, n->stream2);  // the next chunk reuses the arena and row lists
      stream_wait(n, s, n->stream3);
      stream_wait(n, s, n->stream4);
    }
  }
  if (W > 1 && n_live > 0) {
    allgather_rows(n, n->live, n_live, 4, n->cand);
    allgather_rows(n, n->live, n_live, 1, n->ckat);
  }
  count_checkpoints(n, t, affine, allow_freeze, n->live, n->d_int, 0, 1);
  ++n->gen;  // refresh round: the write-back marks what this pass changed
  prof_begin(n, PROF_WRITEBACK);
  launch_writeback(s, N, Q.out_c, t, n->cand, n->blo + o, n->bhi + o, n->rlo + o, n->rhi + o,
                   Q.feeds_relu ? n->relax + 8 * o : nullptr, n->gen_n, n->gen_pos, n->gen_l,
                   n->gen, o, n->pofs[t]);
  prof_end(n);
}

// Device-driven margin pass (graph mode): label and class list on the device;
// best / has are read back after the graph.
void run_margin_graph(Ctx* n, pc_stats* st) {
  cudaStream_t s = n->stream;
  const int out = (int)n->L.size() - 1;
  const int nr = n->n_out - 1;
  st->rows_total += nr;
  if (nr <= 0) return;
  st->checkpoints += walk_checkpoints(n, dense_frame(out), false);  // one chunk, never frozen
  launch_margin_rows(s, n->d_label, n->n_out, n->rowq[0]);
  ck(cudaMemsetAsync(n->has, 0, nr, s), "memset");
  const WalkSize ws = walk_size(n, out, false, false);
  n->arena_used = 0;
  reset_stats(n, ws.stats);
  Walker w{n, s, out};
  w.s2 = n->net->serial ? n->stream : n->stream2;
  w.R = nr;
  w.both = false;
  w.margin = true;
  w.st = st;
  w.row_q = n->rowq[0];
  Mat m = w.alloc(dense_frame(out), true);
  launch_init_margin(s, 0, n->d_label, n->n_out, 0, nr, md(m));
  w.mark(m);
  w.walk(m, 0, true);
  stream_wait(n, s, n->stream2);
}

// run_margin_pass (backsub.hpp:1070-1096)
void run_margin(Ctx* n, int label, pc_stats* st, double* margins_host) {
  NvtxRange nv("margin pass");
  cudaStream_t s = n->stream;
  const int out = (int)n->L.size() - 1;
  const int nr = n->n_out - 1;
  st->rows_total += nr;
  if (nr <= 0) return;
  st->checkpoints += walk_checkpoints(n, dense_frame(out), false);  // one chunk, never frozen
  std::vector<int> cls;
  for (int j = 0; j < n->n_out; ++j)
    if (j != label) cls.push_back(j);
  // this rank's slice of the margin rows (all of them unsharded)
  const int W = n->net->shard_world;
  const int mb = (int)slice_begin(nr, n->net->shard_rank, W);
  const int me = (int)slice_begin(nr, n->net->shard_rank + 1, W);
  const int R = me - mb;
  // two walk pipelines as in run_pass: the margin rows split between this
  // context and its helper, advanced step by step in turn, so one half's
  // conv substitutions overlap the other half's constant folds
  static const int pipes = env_int("PC_PIPES", 2);
  static const int margin_min = env_int("PC_MARGIN_PIPE_MIN", 4);
  if (R > 0 && pipes >= 2 && R >= margin_min && !n->is_helper && !n->net->serial) {
    Ctx* h = helper_of(n);
    const int RA = R / 2, RB = R - RA;
    ck(cudaMemcpyAsync(n->rowq[0], cls.data() + mb, sizeof(int) * RA, cudaMemcpyHostToDevice, s), "h2d");
    ck(cudaMemcpyAsync(h->rowq[0], cls.data() + mb + RA, sizeof(int) * RB, cudaMemcpyHostToDevice, s), "h2d");
    ck(cudaMemsetAsync(n->has, 0, R, s), "memset");
    const WalkSize ws = walk_size(n, out, false, false);
    ensure_arena(n, ws.per_row * (size_t)RB + 256 * ws.allocs + (1 << 20));
    ensure_arena(h, ws.per_row * (size_t)RB + 256 * ws.allocs + (1 << 20));
    stream_wait(n, h->stream, s);  // row lists, has[], the refreshed bounds
    Ctx* cx[2] = {n, h};
    const int r0[2] = {0, RA}, rn[2] = {RA, RB};
    ChunkWalk a{Walker{n, s, out}}, b{Walker{h, h->stream, out}};
    ChunkWalk* cw[2] = {&a, &b};
    for (int k = 0; k < 2; ++k) {
      Ctx* c = cx[k];
      c->arena_used = 0;
      reset_stats(c, ws.stats);
      Walker& w = cw[k]->w;
      w.s2 = c->stream2;
      w.R = rn[k];
      w.both = false;
      w.margin = true;
      w.st = st;
      w.row_q = c->rowq[0];
      w.mbest = n->best + r0[k];
      w.mhas = n->has + r0[k];
      cw[k]->m = w.alloc(dense_frame(out), true);
      launch_init_margin(w.s, label, nullptr, n->n_out, mb + r0[k], rn[k], md(cw[k]->m));
      w.mark(cw[k]->m);
    }
    while (a.running || b.running) {
      if (a.running) a.running = a.w.advance(a.m, 0, true, a.pending);
      if (b.running) b.running = b.w.advance(b.m, 0, true, b.pending);
    }
    stream_wait(n, s, n->stream2);
    stream_wait(n, s, h->stream);
    stream_wait(n, s, h->stream2);
    stream_wait(n, h->stream, s);  // h's next walk reuses its arena after s
    ck(cudaMemcpyAsync(n->h_int + 4, n->has, R, cudaMemcpyDeviceToHost, s), "d2h");
  } else if (R > 0) {
    ck(cudaMemcpyAsync(n->rowq[0], cls.data() + mb, sizeof(int) * R, cudaMemcpyHostToDevice, s), "h2d");
    ck(cudaMemsetAsync(n->has, 0, R, s), "memset");
    const WalkSize ws = walk_size(n, out, false, false);
    ensure_arena(n, ws.per_row * (size_t)R + 256 * ws.allocs + (1 << 20));
    n->arena_used = 0;
    reset_stats(n, ws.stats);
    Walker w{n, s, out};
    w.s2 = n->net->serial ? n->stream : n->stream2;
    w.R = R;
    w.both = false;
    w.margin = true;
    w.st = st;
    w.row_q = n->rowq[0];
    Frame f0 = dense_frame(out);
    Mat m = w.alloc(f0, true);
    launch_init_margin(s, label, nullptr, n->n_out, mb, R, md(m));
    w.mark(m);
    w.walk(m, 0, true);
    stream_wait(n, s, n->stream2);
    ck(cudaMemcpyAsync(n->h_int + 4, n->has, R, cudaMemcpyDeviceToHost, s), "d2h");
  }
  double* best = n->best;
  if (W > 1) {  // every rank's best values, in class order (8 B per margin row)
    const int per = (nr + W - 1) / W;
    ensure_shard_buffers(n, (size_t)per);
    ck(cudaMemcpyAsync(n->sh_send, n->best, sizeof(double) * R, cudaMemcpyDeviceToDevice, s), "d2d");
    exchange(n, (size_t)per * sizeof(double));
    launch_shard_unpack(s, nullptr, nr, W, per, 1, n->sh_recv, n->vals);
    best = n->vals;
  }
  ck(cudaMemcpyAsync(margins_host, best, sizeof(double) * nr, cudaMemcpyDeviceToHost, s), "d2h");
  ck(cudaStreamSynchronize(s), "sync");
  const char* has = reinterpret_cast<const char*>(n->h_int + 4);
  for (int r = 0; r < R; ++r)
    if (!has[r]) throw StatusError(PC_ERR_LOGIC, "margin pass produced no candidate");
}

// Targets: layers feeding a relu, ascending, then the output (analyzer.hpp:220-223).
std::vector<int> pass_targets(const Ctx* n) {
  const int out = (int)n->L.size() - 1;
  std::vector<int> targets;
  for (int k = 1; k < out; ++k)
    if (n->L[k].feeds_relu) targets.push_back(k);
  targets.push_back(out);
  return targets;
}

// The device-driven schedule needs every pass in one chunk sized for all of
// the layer's neurons (the live count is only known on the device).
bool graph_eligible(Ctx* n, size_t* arena_bytes, size_t* stat_count) {
  if (n->net->shard_world > 1 || n->profile || n->opt.exec_mode != 2 || n->graph_failed ||
      n->opt.numeric_mode != 0)
    return false;
  if (n->opt.chunk_rows > 0) return false;  // an explicit chunking request keeps the host schedule
  size_t arena = 0, stats = 0;
  for (int t : pass_targets(n)) {
    const HostLayer& Q = n->L[t];
    const WalkSize ws = walk_size(n, t, Q.kind == KIND_DENSE || Q.kind == KIND_CONV, true);
    const size_t need = ws.per_row * (size_t)Q.numel() + 256 * ws.allocs + (1 << 20);
    if ((long long)need > budget_of(n)) return false;
    if (2 * Q.numel() > 65535) return false;  // rows ride in gridDim.y
    arena = std::max(arena, need);
    stats = std::max(stats, ws.stats);
  }
  const int out = (int)n->L.size() - 1;
  const WalkSize wm = walk_size(n, out, false, false);
  arena = std::max(arena, wm.per_row * (size_t)std::max(1, n->n_out - 1) + 256 * wm.allocs + (1 << 20));
  stats = std::max(stats, wm.stats);
  *arena_bytes = arena;
  *stat_count = stats;
  // Opt-in: grids sized for every neuron of a layer cost more than the
  // launches they save when few rows are live (measured).
  return n->opt.exec_mode == 2;
}

// Forward refresh of layers (k0, k1] (all nimg images of a batched context
// per launch). A ReLU layer's bounds are final once refreshed here (no later
// pass changes a layer below its target), so its live-channel table for the
// conv kernels (k_live_build) is rebuilt right after.
void forward_layers(Ctx* n, int k0, int k1, int nimg = 1) {
  NvtxRange nv("forward refresh", k1);
  const int nl = (int)n->L.size();
  const long long T = n->total, P = n->pofs[nl];
  for (int k = k0 + 1; k <= k1; ++k) {
    const HostLayer& l = n->L[k];
    prof_begin(n, PROF_FWD);
    if (nimg > 1)
      launch_forward_layer(n->stream, l.d, l.feeds_relu, n->blo, n->bhi, n->rlo, n->rhi, n->off.data(),
                           n->pofs.data(), k, l.pred0, l.pred1, n->dev, n->relax, n->gen_n,
                           n->gen_pos, n->gen_l, n->gen, 1, nimg, T, P, nl);
    else
      launch_forward_layer(n->stream, l.d, l.feeds_relu, n->blo, n->bhi, n->rlo, n->rhi, n->off.data(),
                           n->pofs.data(), k, l.pred0, l.pred1, n->dev, n->relax, n->gen_n,
                           n->gen_pos, n->gen_l, n->gen, 1);
    if (l.kind == KIND_RELU)
      launch_offset_list(n->stream, (int)l.numel(), n->relax + 8 * n->off[l.pred0], n->un_idx + n->off[l.pred0],
                         n->un_cnt + l.pred0, nimg, T, nl);
    bool feeds_conv = false;  // the live tables serve the conv steps onto this frame (gbc_step)
    for (const HostLayer& c : n->L) feeds_conv |= c.kind == KIND_CONV && c.pred0 == k;
    if (l.kind == KIND_RELU && n->net->live_cells && feeds_conv) {
      const long long o = n->off[k];
      launch_live_build(n->stream, l.out_w * l.out_h, l.out_c, n->relax + 8 * n->off[l.pred0], n->blo + o,
                        n->bhi + o, n->rlo + o, n->rhi + o, n->lv_cnt + n->pofs[k], n->lv_idx + o, nimg,
                        T, P, n->lv_chm + (size_t)k * 16, nl * 16);
      launch_live_flat(n->stream, l.out_w * l.out_h, l.out_c, n->lv_cnt + n->pofs[k], n->lv_idx + o,
                       n->lv_pref + n->pofs[k] + k, n->lv_fpos + o, n->lv_fch + o, nimg, T, P, P + nl);
    }
    prof_end(n);
  }
}

// Capture the whole analysis (+ margin pass when with_margin) as one CUDA
// graph on this context: ~all launches of an image become one graph launch.
void capture_graph(Ctx* n, bool with_margin, size_t arena, size_t stat_count) {
  cudaStream_t s = n->stream;
  ensure_arena(n, arena);
  reset_stats(n, stat_count);  // size the pool outside the capture
  ck(cudaStreamSynchronize(s), "sync");
  while (n->sync_pool.size() < 8192) {
    cudaEvent_t e;
    ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    n->sync_pool.push_back(e);
  }
  while (n->ev_pool.size() < 4096) {
    cudaEvent_t e;
    ck(cudaEventCreate(&e), "event");
    n->ev_pool.push_back(e);
  }
  n->sync_used = 0;
  n->ev_used = 0;
  n->dense_ev.clear();
  n->conv_ev.clear();
  const long long l0 = g_launches;
  g_dense_bytes = g_dense_madds = 0;
  g_dense_launches = 0;
  g_conv_bytes = 0;
  g_conv_launches = 0;
  pc_stats st{};
  ck(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "capture");
  cudaGraph_t g = nullptr;
  try {
    stream_wait(n, n->stream2, s);  // fork the constants stream into the capture
    ck(cudaMemsetAsync(n->ctr, 0, sizeof(Counters), s), "memset");
    const std::vector<int> targets = pass_targets(n);
    const int out = (int)n->L.size() - 1;
    forward_layers(n, 0, targets[0]);
    for (size_t i = 0; i < targets.size(); ++i) {
      run_pass_graph(n, targets[i], targets[i] != out, &st);
      if (targets[i] != out) forward_layers(n, targets[i], targets[i + 1]);
    }
    if (with_margin) run_margin_graph(n, &st);
    ck(cudaStreamEndCapture(s, &g), "capture");
  } catch (...) {
    cudaStreamEndCapture(s, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  cudaGraphExec_t exec = nullptr;
  const cudaError_t e = cudaGraphInstantiate(&exec, g, 0);
  cudaGraphDestroy(g);
  ck(e, "graph instantiate");
  if (n->graph) cudaGraphExecDestroy(n->graph);
  n->graph = exec;
  n->graph_label_mode = with_margin ? 1 : 0;
  n->graph_et = n->opt.early_term;
  n->graph_st = st;
  n->graph_dense_ev = n->dense_ev;
  n->graph_conv_ev = n->conv_ev;
  n->graph_conv_bytes = g_conv_bytes;
  n->graph_conv_launches = g_conv_launches;
  n->graph_dense_bytes = g_dense_bytes;
  n->graph_dense_madds = g_dense_madds;
  n->graph_dense_launches = g_dense_launches;
  n->graph_launches = g_launches - l0;
}

// analyze + run_margin_pass (analyzer.hpp:198-276)
void run_test(Ctx* n, int label, double* margins, pc_stats* st) {
  NvtxRange nv("verify_robustness");
  cudaStream_t s = n->stream;
  const int nl = (int)n->L.size();
  const int out = nl - 1;
  size_t arena = 0, stat_count = 0;
  if (graph_eligible(n, &arena, &stat_count)) {
    const bool with_margin = label >= 0;
    if (!n->graph || n->graph_label_mode != (with_margin ? 1 : 0) || n->graph_et != n->opt.early_term) {
      try {
        capture_graph(n, with_margin, arena, stat_count);
      } catch (const StatusError&) {
        cudaGetLastError();
        n->graph_failed = true;  // fall back to the host-driven schedule
      }
    }
    if (n->graph && n->graph_label_mode == (with_margin ? 1 : 0) && n->graph_et == n->opt.early_term) {
      n->h_int[2] = label;
      ck(cudaMemcpyAsync(n->d_label, n->h_int + 2, sizeof(int), cudaMemcpyHostToDevice, s), "h2d");
      ck(cudaGraphLaunch(n->graph, s), "graph launch");
      g_launches += n->graph_launches;
      // events recorded inside the capture are graph nodes: no per-kernel
      // elapsed times in this schedule (pc_last_kernel_timing reads 0)
      n->dense_ev.clear();
      n->conv_ev.clear();
      g_conv_bytes = n->graph_conv_bytes;
      g_conv_launches = n->graph_conv_launches;
      g_dense_bytes = n->graph_dense_bytes;
      g_dense_madds = n->graph_dense_madds;
      g_dense_launches = n->graph_dense_launches;
      *st = n->graph_st;
      const int nr = n->n_out - 1;
      if (with_margin && nr > 0) {
        ck(cudaMemcpyAsync(margins, n->best, sizeof(double) * nr, cudaMemcpyDeviceToHost, s), "d2h");
        ck(cudaMemcpyAsync(n->h_int + 4, n->has, nr, cudaMemcpyDeviceToHost, s), "d2h");
      }
      Counters c{};
      ck(cudaMemcpyAsync(&c, n->ctr, sizeof(Counters), cudaMemcpyDeviceToHost, s), "d2h");
      ck(cudaStreamSynchronize(s), "sync");
      const char* has = reinterpret_cast<const char*>(n->h_int + 4);
      for (int r = 0; with_margin && r < nr; ++r)
        if (!has[r]) throw StatusError(PC_ERR_LOGIC, "margin pass produced no candidate");
      st->checkpoints += (long long)c.checkpoints;
      st->gbc_dense_equiv += (long long)c.gbc_dense_equiv;
      st->dense_madds += (long long)c.dense_madds;
      st->gbc_madds += (long long)c.gbc_madds;
      g_conv_exec = (double)c.conv_exec;
      st->rows_terminated_early += (long long)(c.frozen + c.pad);
      return;
    }
  }
  ck(cudaMemsetAsync(n->ctr, 0, sizeof(Counters), s), "memset");
  // Targets: layers feeding a relu, ascending, then the output (analyzer.hpp:220-223).
  std::vector<int> targets;
  for (int k = 1; k < out; ++k)
    if (n->L[k].feeds_relu) targets.push_back(k);
  targets.push_back(out);
  // Lazy refresh. The reference recomputes every layer k > t after pass t
  // (analyzer.hpp:232-239), but pass t' reads only layers <= t' (its seed,
  // relaxations, dev and frame bounds), and every layer beyond the next target
  // is recomputed again after that target's pass from the same final
  // predecessor values. So computing layer k once, right after the last pass
  // before it (and the forward pass for k <= first target), yields the
  // reference's state bit-for-bit with each layer evaluated once per image.
  auto forward = [&](int k0, int k1) { forward_layers(n, k0, k1); };  // layers (k0, k1]
  forward(0, targets[0]);
  // PC_PROFILE: wall time and live rows per pass (host clock; the pass ends
  // with the write-back, which the next pass's seed synchronises on)
  std::vector<std::array<double, 3>> pass_t;
  auto tp = std::chrono::steady_clock::now();
  for (size_t i = 0; i < targets.size(); ++i) {
    const int t = targets[i];
    const bool is_out = t == out;
    run_pass(n, t, !is_out, st);
    if (!is_out) forward(t, targets[i + 1]);
    if (n->profile) {
      ck(cudaStreamSynchronize(s), "sync");
      const auto t1 = std::chrono::steady_clock::now();
      pass_t.push_back({(double)t, (double)n->h_int[0],
                        std::chrono::duration<double, std::milli>(t1 - tp).count()});
      tp = t1;
    }
  }
  if (label >= 0) run_margin(n, label, st, margins);
  if (n->profile) {
    const auto t1 = std::chrono::steady_clock::now();
    pass_t.push_back({-1.0, (double)(n->n_out - 1), std::chrono::duration<double, std::milli>(t1 - tp).count()});
    g_pass_json = "[";
    for (size_t k = 0; k < pass_t.size(); ++k)
      g_pass_json += (k ? ", [" : "[") + std::to_string((int)pass_t[k][0]) + ", " +
                     std::to_string((int)pass_t[k][1]) + ", " + std::to_string(pass_t[k][2]) + "]";
    g_pass_json += "]";
  }
  Counters c{};
  ck(cudaMemcpyAsync(&c, n->ctr, sizeof(Counters), cudaMemcpyDeviceToHost, s), "d2h");
  ck(cudaStreamSynchronize(s), "sync");
  const int W = n->net->shard_world;
  if (W > 1) {
    // per-rank work counters (walk freezes, madds, checkpoints, dense-equivalent
    // GBC work) add up; pre-freezes and rows_total are identical on every rank
    // (checkpoints are counted from the gathered per-row freeze checkpoints,
    // identical on every rank)
    unsigned long long h[8] = {c.dense_madds, c.gbc_madds, c.frozen, 0, 0, c.gbc_dense_equiv, 0, 0};
    ensure_shard_buffers(n, 8);
    ck(cudaMemcpyAsync(n->sh_send, h, sizeof(h), cudaMemcpyHostToDevice, s), "h2d");
    exchange(n, sizeof(h));
    std::vector<unsigned long long> all((size_t)8 * W);
    ck(cudaMemcpyAsync(all.data(), n->sh_recv, all.size() * 8, cudaMemcpyDeviceToHost, s), "d2h");
    ck(cudaStreamSynchronize(s), "sync");
    unsigned long long sum[8] = {0};
    for (int r = 0; r < W; ++r)
      for (int k = 0; k < 8; ++k) sum[k] += all[(size_t)8 * r + k];
    c.dense_madds = sum[0];
    c.gbc_madds = sum[1];
    c.frozen = sum[2];
    c.gbc_dense_equiv = sum[5];
  }
  st->checkpoints += (long long)c.checkpoints;
  st->gbc_dense_equiv += (long long)c.gbc_dense_equiv;
  st->dense_madds += (long long)c.dense_madds;
  st->gbc_madds += (long long)c.gbc_madds;
  g_conv_exec = (double)c.conv_exec;
  st->rows_terminated_early += (long long)(c.frozen + c.pad);
}

// ---------------------------------------------------------------------------
// Image-batched verification (pc_net_test_batch): B images in one schedule.
// Every pass seeds each image, concatenates the live rows of all images into
// one key list (img * M + neuron) and walks them as one set of rows, so each
// kernel launch carries B images' rows; the per-neuron state of image b sits
// at offset b * total. Results per image are the single-image engine's.
void run_test_batched(Ctx* n, int B, const int* labels, double* margins, pc_stats* stats) {
  NvtxRange nv("verify_robustness batch", B);
  cudaStream_t s = n->stream;
  const int nl = (int)n->L.size();
  const int out = nl - 1;
  const long long T = n->total, M = n->max_numel, P = n->pofs[nl];
  const bool et = n->opt.early_term != 0;
  ck(cudaMemsetAsync(n->ctr, 0, sizeof(Counters) * B, s), "memset");
  const std::vector<int> targets = pass_targets(n);
  auto forward = [&](int k0, int k1) { forward_layers(n, k0, k1, B); };  // all B images per launch
  long long rows_total = 0;
  forward(0, targets[0]);
  for (size_t ti = 0; ti < targets.size(); ++ti) {
    const int t = targets[ti];
    const bool allow_freeze = t != out;
    const HostLayer& Q = n->L[t];
    const int N = (int)Q.numel();
    const long long o = n->off[t];
    launch_seed(s, N, n->blo + o, n->bhi + o, n->rlo + o, n->rhi + o, allow_freeze ? 1 : 0,
                et ? 1 : 0, n->cand, n->frozen, n->live, n->d_int + 8, &n->ctr[0].pad, B, T, M,
                (int)(sizeof(Counters) / sizeof(unsigned long long)));
    launch_gather_keys(s, n->live, n->d_int + 8, B, (int)M, n->keys, n->d_int);
    launch_ck_fill(s, n->keys, n->d_int, (int)(M * B), n->ckat);
    ck(cudaMemcpyAsync(n->h_int, n->d_int, sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
    ck(cudaStreamSynchronize(s), "sync");
    const int n_live = n->h_int[0];
    rows_total += N;
    const bool affine = Q.kind == KIND_DENSE || Q.kind == KIND_CONV;
    if (n_live > 0) {
      const int* keys = n->keys;
      const WalkSize ws = walk_size(n, t, affine, true);
      long long chunk = n->opt.chunk_rows > 0
                            ? n->opt.chunk_rows
                            : std::max<long long>(1, budget_of(n) / (long long)ws.per_row);
      chunk = std::min<long long>(std::min<long long>(chunk, n_live), kMaxWalkRows);
      ensure_arena(n, ws.per_row * (size_t)chunk + 256 * ws.allocs + (1 << 20));
      for (long long base = 0; base < n_live; base += chunk) {
        const int R = (int)std::min<long long>(chunk, n_live - base);
        n->arena_used = 0;
        reset_stats(n, ws.stats);
        Walker w{n, s, t};
        w.s2 = n->net->serial ? n->stream : n->stream2;
        w.R = R;
        w.both = true;
        w.allow_freeze = allow_freeze;
        w.early_term = et;
        pc_stats dummy{};
        w.st = &dummy;
        w.kq = (int)M;
        w.sst = T;
        w.nimg = B;
        ck(cudaMemcpyAsync(n->rowq[0], keys + base, sizeof(int) * R, cudaMemcpyDeviceToDevice, s), "d2d");
        w.rq = 0;
        w.row_q = n->rowq[0];
        Frame f0 = initial_frame(n, t, affine);
        Mat m = w.alloc(f0, true);
        if (affine)
          launch_init_affine(s, Q.d, w.rows(), fdev(n, f0, t), n->dev + o, md(m));
        else
          launch_init_identity(s, w.rows(), fdev(n, f0, t), md(m));
        w.mark(m);
        if (affine) w.checkpoint(m);
        w.walk(m, 0, true);
        stream_wait(n, s, n->stream2);
      }
      count_checkpoints(n, t, affine, allow_freeze, n->keys, n->d_int, (int)M, B);
    }
    ++n->gen;
    launch_writeback(s, N, Q.out_c, t, n->cand, n->blo + o, n->bhi + o, n->rlo + o, n->rhi + o,
                     Q.feeds_relu ? n->relax + 8 * o : nullptr, n->gen_n, n->gen_pos, n->gen_l,
                     n->gen, o, n->pofs[t], B, T, P, nl, M);
    if (t != out) forward(t, targets[ti + 1]);
  }
  // margin pass: rows img * M + class j (j != label), image-major
  const int nr = n->n_out - 1;
  long long margin_ck = 0;
  if (nr > 0) {
    std::vector<int> keys;
    for (int b = 0; b < B; ++b)
      for (int j = 0; j < n->n_out; ++j)
        if (j != labels[b]) keys.push_back((int)(b * M + j));
    const int R = (int)keys.size();
    ck(cudaMemcpyAsync(n->rowq[0], keys.data(), sizeof(int) * R, cudaMemcpyHostToDevice, s), "h2d");
    ck(cudaMemcpyAsync(n->d_label, labels, sizeof(int) * B, cudaMemcpyHostToDevice, s), "h2d");
    ck(cudaMemsetAsync(n->has, 0, R, s), "memset");
    const WalkSize ws = walk_size(n, out, false, false);
    ensure_arena(n, ws.per_row * (size_t)R + 256 * ws.allocs + (1 << 20));
    n->arena_used = 0;
    reset_stats(n, ws.stats);
    Walker w{n, s, out};
    w.s2 = n->net->serial ? n->stream : n->stream2;
    w.R = R;
    w.both = false;
    w.margin = true;
    pc_stats mst{};
    w.st = &mst;
    w.kq = (int)M;
    w.sst = T;
    w.nimg = B;
    w.row_q = n->rowq[0];
    Mat m = w.alloc(dense_frame(out), true);
    launch_init_margin_keys(s, w.rows(), n->d_label, n->n_out, md(m));
    w.mark(m);
    w.walk(m, 0, true);
    stream_wait(n, s, n->stream2);
    ck(cudaMemcpyAsync(margins, n->best, sizeof(double) * R, cudaMemcpyDeviceToHost, s), "d2h");
    ck(cudaMemcpyAsync(n->h_int + 16, n->has, R, cudaMemcpyDeviceToHost, s), "d2h");
    margin_ck = walk_checkpoints(n, dense_frame(out), false);
    rows_total += nr;
  }
  std::vector<Counters> c(B);
  ck(cudaMemcpyAsync(c.data(), n->ctr, sizeof(Counters) * B, cudaMemcpyDeviceToHost, s), "d2h");
  ck(cudaStreamSynchronize(s), "sync");
  const char* has = reinterpret_cast<const char*>(n->h_int + 16);
  for (int r = 0; r < B * nr; ++r)
    if (!has[r]) throw StatusError(PC_ERR_LOGIC, "margin pass produced no candidate");
  for (int b = 0; b < B; ++b) {
    pc_stats& st = stats[b];
    st = pc_stats{};
    st.rows_total = rows_total;
    st.checkpoints = (long long)c[b].checkpoints + margin_ck;
    st.gbc_dense_equiv = (long long)c[b].gbc_dense_equiv;
    st.dense_madds = (long long)c[b].dense_madds;
    st.gbc_madds = (long long)c[b].gbc_madds;
    st.rows_terminated_early = (long long)(c[b].frozen + c[b].pad);
  }
}

pc_status guard(const std::function<void()>& fn) {
  try {
    fn();
    return PC_OK;
  } catch (const StatusError& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "out of host memory";
    return PC_ERR_OOM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return PC_ERR_LOGIC;
  }
}

// One verification on context n (analyze + margin pass; verify_robustness).
void run_one(Ctx* n, const double* lo, const double* up, bool device_box, int label, int* verified,
             double* margins, double* b_lo, double* b_hi, double* r_lo, double* r_hi,
             pc_stats* stats) {
    if (label >= n->n_out) throw StatusError(PC_ERR_INVALID_ARGUMENT, "margin: label out of range");
    const long long n0 = n->L[0].numel();
    cudaStream_t s = n->stream;
    cudaEvent_t t0, t1;
    ck(cudaEventCreate(&t0), "event");
    ck(cudaEventCreate(&t1), "event");
    ck(cudaEventRecord(t0, s), "event");
    if (device_box) {
      ck(cudaMemcpyAsync(n->blo, lo, sizeof(double) * n0, cudaMemcpyDeviceToDevice, s), "d2d");
      ck(cudaMemcpyAsync(n->bhi, up, sizeof(double) * n0, cudaMemcpyDeviceToDevice, s), "d2d");
    } else {
      for (long long i = 0; i < n0; ++i)
        if (std::isnan(lo[i]) || std::isnan(up[i]))
          throw StatusError(PC_ERR_INVALID_ARGUMENT, "Interval: NaN endpoint");
      ck(cudaMemcpyAsync(n->blo, lo, sizeof(double) * n0, cudaMemcpyHostToDevice, s), "h2d");
      ck(cudaMemcpyAsync(n->bhi, up, sizeof(double) * n0, cudaMemcpyHostToDevice, s), "h2d");
    }
    ck(cudaMemcpyAsync(n->rlo, n->blo, sizeof(double) * n0, cudaMemcpyDeviceToDevice, s), "d2d");
    ck(cudaMemcpyAsync(n->rhi, n->bhi, sizeof(double) * n0, cudaMemcpyDeviceToDevice, s), "d2d");
    pc_stats st{};
    std::vector<double> m(std::max(1, n->n_out - 1), 0.0);
    n->ev_used = 0;
    n->sync_used = 0;
    for (Ctx* h = n->helper; h; h = h->helper) {
      h->ev_used = 0;
      h->sync_used = 0;
      h->prof.clear();
      h->dense_ev.clear();
      h->conv_ev.clear();
    }
    g_gbc_window_madds = 0;
    g_alloc_ms = 0;
    g_allocs = 0;
    n->prof.clear();
    n->dense_ev.clear();
    n->conv_ev.clear();
    g_conv_ms = g_conv_bytes = 0;
    g_conv_launches = 0;
    run_test(n, label, m.data(), &st);
    if (b_lo) ck(cudaMemcpyAsync(b_lo, n->blo, sizeof(double) * n->total, cudaMemcpyDeviceToHost, s), "d2h");
    if (b_hi) ck(cudaMemcpyAsync(b_hi, n->bhi, sizeof(double) * n->total, cudaMemcpyDeviceToHost, s), "d2h");
    if (r_lo) ck(cudaMemcpyAsync(r_lo, n->rlo, sizeof(double) * n->total, cudaMemcpyDeviceToHost, s), "d2h");
    if (r_hi) ck(cudaMemcpyAsync(r_hi, n->rhi, sizeof(double) * n->total, cudaMemcpyDeviceToHost, s), "d2h");
    ck(cudaGetLastError(), "kernel");
    ck(cudaEventRecord(t1, s), "event");
    ck(cudaStreamSynchronize(s), "sync");
    ck(cudaGetLastError(), "kernel");
    float ms = 0;
    cudaEventElapsedTime(&ms, t0, t1);
    g_total_ms = ms;
    for (size_t e : n->dense_ev) {
      float d = 0;
      if (cudaEventElapsedTime(&d, n->ev_pool[e], n->ev_pool[e + 1]) == cudaSuccess) g_dense_ms += d;
    }
    for (Ctx* c = n; c; c = c->helper) {  // every walk pipeline
      for (size_t e : c->conv_ev) {
        float d = 0;
        if (cudaEventElapsedTime(&d, c->ev_pool[e], c->ev_pool[e + 1]) == cudaSuccess) g_conv_ms += d;
      }
    }
    cudaGetLastError();  // timing is best effort; never leave a sticky error behind
    for (int c = 0; c < PROF_N; ++c) {
      g_prof_ms[c] = 0;
      g_prof_n[c] = 0;
      g_gap_ms[c] = 0;
    }
    g_timeline_json = "[";
    for (size_t k = 0; k < n->prof.size(); ++k) {
      const auto& pe = n->prof[k];
      if (pe.e == SIZE_MAX) continue;
      float d = 0, t_b = 0, t_e = 0;
      cudaEventElapsedTime(&d, n->ev_pool[pe.b], n->ev_pool[pe.e]);
      g_prof_ms[pe.cls] += d;
      g_prof_n[pe.cls] += 1;
      // timeline: [class, stream (0 coefficients, 1 constants, 2 exact checkpoints,
      // 3 predictions), start ms, end ms] from t0
      cudaEventElapsedTime(&t_b, t0, n->ev_pool[pe.b]);
      cudaEventElapsedTime(&t_e, t0, n->ev_pool[pe.e]);
      char buf[96];
      snprintf(buf, sizeof(buf), "%s[%d, %d, %.4f, %.4f]", g_timeline_json.size() > 1 ? ", " : "", pe.cls,
               pe.st == n->stream ? 0 : pe.st == n->stream2 ? 1 : pe.st == n->stream3 ? 2 : 3, t_b, t_e);
      g_timeline_json += buf;
    }
    g_timeline_json += "]";
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
    if (label >= 0) {
      bool v = true;
      for (int r = 0; r < n->n_out - 1; ++r) {
        if (margins) margins[r] = m[r];
        if (!(m[r] > 0.0)) v = false;
      }
      if (verified) *verified = v ? 1 : 0;
    } else if (verified) {
      *verified = 0;
    }
    if (stats) *stats = st;
    g_last_launches = g_launches;
}

// Per-call options (AnalysisOptions of one verify_robustness / analyze call):
// early_term, chunk_rows, memory_budget and exec_mode apply to this call only;
// the device is the net's.
void apply_call_options(Ctx* c, const pc_options* call) {
  pc_options o = call ? *call : c->net->opt;
  o.device = c->net->opt.device;
  if (call && o.exec_mode == 0) o.exec_mode = c->net->opt.exec_mode;
  c->opt = o;
  for (Ctx* h = c->helper; h; h = h->helper) h->opt = o;
}

pc_status test_impl(pc_net* net, const pc_options* call_opt, const double* lo, const double* up,
                    bool device_box, int label, int* verified, double* margins, double* b_lo,
                    double* b_hi, double* r_lo, double* r_hi, pc_stats* stats) {
  if (!net) {
    g_err = "null network";
    return PC_ERR_INVALID_ARGUMENT;
  }
  g_launches = 0;
  g_dense_ms = g_dense_bytes = g_dense_madds = 0;
  g_dense_launches = 0;
  return guard([&] {
    ck(cudaSetDevice(net->device), "cudaSetDevice");
    dense_useful_madds(true);
    CtxLease lease(net);
    apply_call_options(lease.c, call_opt);
    run_one(lease.c, lo, up, device_box, label, verified, margins, b_lo, b_hi, r_lo, r_hi, stats);
    g_dense_madds = (double)dense_useful_madds(false);
  });
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI

extern "C" {

void pc_default_options(pc_options* opt) {
  opt->early_term = 1;
  opt->chunk_rows = 0;
  opt->memory_budget = 0;
  opt->device = -1;
  opt->exec_mode = 0;
  opt->numeric_mode = 0;
}

const char* pc_last_error(void) { return g_err.c_str(); }
double pc_last_dense_madds(void) { return g_dense_madds; }
long long pc_last_launch_count(void) { return g_last_launches; }

double pc_last_conv_executed_madds(void) { return g_conv_exec; }

pc_status pc_net_set_serial(pc_net* net, int serial) {
  if (!net) return PC_ERR_INVALID_ARGUMENT;
  net->serial = serial != 0;
  return PC_OK;
}

void pc_last_kernel_timing(int kernel, double* ms, double* bytes, long long* launches) {
  const bool conv = kernel == 1;
  if (ms) *ms = conv ? g_conv_ms : g_dense_ms;
  if (bytes) *bytes = conv ? g_conv_bytes : g_dense_bytes;
  if (launches) *launches = conv ? g_conv_launches : g_dense_launches;
}

void pc_last_timing(double* total_ms, double* dense_ms, double* dense_bytes, long long* launches) {
  if (total_ms) *total_ms = g_total_ms;
  if (dense_ms) *dense_ms = g_dense_ms;
  if (dense_bytes) *dense_bytes = g_dense_bytes;
  if (launches) *launches = g_dense_launches;
}

pc_status pc_input_box(const double* center, int n, double eps, int clamp01, double* lo,
                       double* up) {
  // network.hpp:160-177 is host-side input preparation; computed on the GPU
  // like every other widened operation (no host arithmetic path exists).
  return guard([&] {
    if (eps < 0.0) throw StatusError(PC_ERR_INVALID_ARGUMENT, "input_box: negative epsilon");
    for (int i = 0; i < n; ++i) {
      if (std::isnan(center[i])) throw StatusError(PC_ERR_INVALID_ARGUMENT, "Interval: NaN endpoint");
      if (clamp01 && (center[i] < 0.0 || 1.0 < center[i]))
        throw StatusError(PC_ERR_INVALID_ARGUMENT, "input_box: clamped center outside [0,1]");
    }
    ck(input_box_device(center, n, eps, clamp01, lo, up), "input_box");
  });
}

pc_status pc_fp64_peak(int device, double* fma_per_s) {
  if (!fma_per_s) return PC_ERR_INVALID_ARGUMENT;
  return guard([&] {
    if (device >= 0) ck(cudaSetDevice(device), "cudaSetDevice");
    ck(fp64_peak_device(fma_per_s), "fp64_peak");
  });
}

pc_status pc_scalar_ops(int op, const double* a, const double* b, double* out, long long n) {
  return guard([&] { ck(scalar_ops_device(op, a, b, out, n), "scalar_ops"); });
}

pc_status pc_scan_stats(int on, unsigned long long* out4) {
  return guard([&] {
    unsigned long long a[8] = {0, 0, 0, 0, 0, 0, 0, 0}, b[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    ck(scan_stats_device(on, a), "scan_stats");
    ck(scan_stats_device_chains(on, b), "scan_stats");
    if (out4)
      for (int k = 0; k < 8; ++k) out4[k] = a[k] + b[k];
  });
}

pc_status pc_chain_fold(int n_chains, int len, const double* acc0, const double* terms, const int* up,
                        double* out) {
  if (n_chains < 0 || len < 0 || (n_chains && (!acc0 || !up || !out || (len && !terms))))
    return PC_ERR_INVALID_ARGUMENT;
  return guard([&] { ck(chain_fold_device(n_chains, len, acc0, terms, up, out), "chain_fold"); });
}

pc_status pc_validate(const pc_layer_desc* layers, int n_layers, int in_w, int in_h, int in_c,
                      int* out_shapes) {
  return guard([&] {
    std::vector<HostLayer> L;
    validate(layers, n_layers, in_w, in_h, in_c, L);
    if (out_shapes)
      for (size_t k = 0; k < L.size(); ++k) {
        out_shapes[3 * k] = L[k].out_w;
        out_shapes[3 * k + 1] = L[k].out_h;
        out_shapes[3 * k + 2] = L[k].out_c;
      }
  });
}

pc_status pc_net_create(const pc_layer_desc* layers, int n_layers, int in_w, int in_h, int in_c,
                        const pc_options* opt, pc_net** out) {
  if (!out) return PC_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  pc_net* n = new pc_net;
  pc_status st = guard([&] {
    if (opt) n->opt = *opt;
    else pc_default_options(&n->opt);
    if (n->opt.exec_mode == 0) n->opt.exec_mode = env_int("PC_EXEC_MODE", 0);  // tests / experiments
    if (n->opt.numeric_mode == 0) n->opt.numeric_mode = env_int("PC_NUMERIC_MODE", 0);
    validate(layers, n_layers, in_w, in_h, in_c, n->L);
    int devc = 0;
    ck(cudaGetDeviceCount(&devc), "cudaGetDeviceCount");
    if (devc < 1) throw StatusError(PC_ERR_CUDA, "cuda: no CUDA device (there is no CPU fallback)");
    if (n->opt.device >= 0) n->device = n->opt.device;
    else ck(cudaGetDevice(&n->device), "cudaGetDevice");
    ck(cudaSetDevice(n->device), "cudaSetDevice");
    init_kernel_attrs(n->device);
    const int nl = (int)n->L.size();
    n->off.assign(nl + 1, 0);
    for (int k = 0; k < nl; ++k) {
      n->off[k + 1] = n->off[k] + n->L[k].numel();
      n->max_numel = std::max(n->max_numel, n->L[k].numel());
    }
    n->total = n->off[nl];
    n->pofs.assign(nl + 1, 0);
    for (int k = 0; k < nl; ++k) n->pofs[k + 1] = n->pofs[k] + (long long)n->L[k].out_w * n->L[k].out_h;
    n->n_out = (int)n->L.back().numel();
    n->live_cells = env_int("PC_LIVE_CELLS", 1) != 0;
    for (const HostLayer& l : n->L)
      for (double b : l.bias)
        if (std::signbit(b) && b == 0.0) n->live_cells = false;
    for (int k = 0; k < nl; ++k) {
      HostLayer& l = n->L[k];
      LayerDev& d = l.d;
      d.kind = l.kind; d.pred0 = l.pred0; d.pred1 = l.pred1;
      d.in_w = l.in_w; d.in_h = l.in_h; d.in_c = l.in_c;
      d.out_w = l.out_w; d.out_h = l.out_h; d.out_c = l.out_c;
      d.fw = l.fw; d.fh = l.fh; d.sw = l.sw; d.sh = l.sh; d.pw = l.pw; d.ph = l.ph;
      d.wmin = d.wmax = 1.0;
      if (l.kind == KIND_DENSE || l.kind == KIND_CONV) {
        bool any = false;
        for (double w : l.W)
          if (w != 0.0) {
            const double a = std::fabs(w);
            if (!any || a < d.wmin) d.wmin = a;
            if (!any || a > d.wmax) d.wmax = a;
            any = true;
          }
        // test switch: no product is proven in band, every coefficient kernel
        // takes its checked (literal restatement) path
        static const int force_checked = env_int("PC_FORCE_CHECKED", 0);
        if (force_checked) d.wmin = 0.0;
        double* b = n->dalloc<double>(l.bias.size());
        ck(cudaMemcpy(b, l.bias.data(), l.bias.size() * 8, cudaMemcpyHostToDevice), "h2d");
        d.bias = b;
      }
      if (l.kind == KIND_DENSE) {
        const long long no = l.out_c, ni = l.in_numel();
        std::vector<double> wt((size_t)no * ni);
        for (long long j = 0; j < no; ++j)
          for (long long t = 0; t < ni; ++t) wt[(size_t)t * no + j] = l.W[(size_t)j * ni + t];
        double* W = n->dalloc<double>(l.W.size());
        double* WT = n->dalloc<double>(wt.size());
        ck(cudaMemcpy(W, l.W.data(), l.W.size() * 8, cudaMemcpyHostToDevice), "h2d");
        ck(cudaMemcpy(WT, wt.data(), wt.size() * 8, cudaMemcpyHostToDevice), "h2d");
        d.W = W;
        d.WT = WT;
      } else if (l.kind == KIND_CONV) {
        std::vector<double> ft(l.W.size());
        for (int fy = 0; fy < l.fh; ++fy)
          for (int fx = 0; fx < l.fw; ++fx)
            for (int ci = 0; ci < l.in_c; ++ci)
              for (int co = 0; co < l.out_c; ++co)
                ft[(((size_t)(fy * l.fw + fx) * l.out_c + co) * l.in_c) + ci] =
                    l.W[(((size_t)(fy * l.fw + fx) * l.in_c + ci) * l.out_c) + co];
        double* F = n->dalloc<double>(l.W.size());
        double* FT = n->dalloc<double>(ft.size());
        ck(cudaMemcpy(F, l.W.data(), l.W.size() * 8, cudaMemcpyHostToDevice), "h2d");
        ck(cudaMemcpy(FT, ft.data(), ft.size() * 8, cudaMemcpyHostToDevice), "h2d");
        d.F = F;
        d.FT = FT;
      }
    }
    n->timing = true;
    const char* pe = getenv("PC_PROFILE");
    n->profile = pe && pe[0] == '1';
    n->primary = acquire(n);  // the first per-call context (stream + state buffers)
    release(n, n->primary);
  });
  if (st != PC_OK) {
    pc_net_destroy(n);
    return st;
  }
  *out = n;
  return PC_OK;
}

void pc_net_destroy(pc_net* n) {
  if (!n) return;
  cudaSetDevice(n->device);
  for (Ctx* c : n->all) delete c;
  for (void* p : n->owned) cudaFree(p);
  delete n;
}

pc_status pc_net_candidate(pc_net* net, const double* center, int* label, double* logits) {
  if (!net || !label) return PC_ERR_INVALID_ARGUMENT;
  return guard([&] {
    ck(cudaSetDevice(net->device), "cudaSetDevice");
    CtxLease lease(net);
    Ctx* n = lease.c;
    cudaStream_t s = n->stream;
    // concrete activations reuse the raw-bound buffers as scratch
    ck(cudaMemcpyAsync(n->rlo, center, sizeof(double) * n->L[0].numel(), cudaMemcpyHostToDevice, s), "h2d");
    for (size_t k = 1; k < n->L.size(); ++k) {
      const HostLayer& l = n->L[k];
      launch_eval_layer(s, l.d, n->rlo + n->off[l.pred0], l.pred1 >= 0 ? n->rlo + n->off[l.pred1] : nullptr,
                        n->rlo + n->off[k]);
    }
    std::vector<double> y(n->n_out);
    ck(cudaMemcpyAsync(y.data(), n->rlo + n->off[n->L.size() - 1], sizeof(double) * n->n_out,
                       cudaMemcpyDeviceToHost, s), "d2h");
    ck(cudaStreamSynchronize(s), "sync");
    ck(cudaGetLastError(), "kernel");
    if (logits) std::copy(y.begin(), y.end(), logits);
    int best = 0;  // unique_argmax (tools/main.cpp:86-100)
    bool tie = false;
    for (int j = 1; j < n->n_out; ++j) {
      if (y[j] > y[best]) {
        best = j;
        tie = false;
      } else if (y[j] == y[best]) {
        tie = true;
      }
    }
    *label = tie ? -1 : best;
  });
}

int pc_last_profile(char* buf, int len) {
  std::string j = "{";
  for (int c = 0; c < PROF_N; ++c) {
    if (c) j += ", ";
    j += "\"" + std::string(kProfNames[c]) + "\": [" + std::to_string(g_prof_n[c]) + ", " +
         std::to_string(g_prof_ms[c]) + "], \"gap:" + kProfNames[c] + "\": [0, " +
         std::to_string(g_gap_ms[c]) + "]";
  }
  j += ", \"gbc_window_madds\": [0, " + std::to_string(g_gbc_window_madds) + "]";
  j += ", \"host_arena_alloc\": [" + std::to_string(g_allocs) + ", " + std::to_string(g_alloc_ms) + "]";
  j += ", \"passes\": " + g_pass_json;
  j += ", \"timeline\": " + g_timeline_json + "}";
  if (buf && len > 0) {
    std::strncpy(buf, j.c_str(), len - 1);
    buf[len - 1] = 0;
  }
  return (int)j.size();
}

void* pc_net_stream(const pc_net* n) {
  return n && n->primary ? (void*)n->primary->stream : nullptr;
}

int pc_net_num_layers(const pc_net* n) { return n ? (int)n->L.size() : -1; }
long long pc_net_layer_numel(const pc_net* n, int k) {
  if (!n || k < 0 || k >= (int)n->L.size()) return -1;
  return n->L[k].numel();
}
long long pc_net_total_neurons(const pc_net* n) { return n ? n->total : -1; }
int pc_net_output_size(const pc_net* n) { return n ? n->n_out : -1; }

pc_status pc_net_test(pc_net* n, const double* lo, const double* up, int label, int* verified,
                      double* margins, double* b_lo, double* b_hi, double* r_lo, double* r_hi,
                      pc_stats* stats) {
  return test_impl(n, nullptr, lo, up, false, label, verified, margins, b_lo, b_hi, r_lo, r_hi,
                   stats);
}

pc_status pc_net_test_ex(pc_net* n, const pc_options* call_opt, const double* lo, const double* up,
                         int label, int* verified, double* margins, double* b_lo, double* b_hi,
                         double* r_lo, double* r_hi, pc_stats* stats) {
  return test_impl(n, call_opt, lo, up, false, label, verified, margins, b_lo, b_hi, r_lo, r_hi,
                   stats);
}

pc_status pc_net_test_batch(pc_net* net, int n_images, const double* lo, const double* up,
                            int device_inputs, const int* labels, int concurrency, int* verified,
                            double* margins, pc_stats* stats, double* device_ms) {
  if (!net || n_images < 0 || !lo || !up || !labels) {
    g_err = "invalid batch arguments";
    return PC_ERR_INVALID_ARGUMENT;
  }
  if (net->shard_world > 1) {
    g_err = "sharding: pc_net_test_batch runs images concurrently; use pc_net_test on a sharded net";
    return PC_ERR_INVALID_ARGUMENT;
  }
  return guard([&] {
    ck(cudaSetDevice(net->device), "cudaSetDevice");
    dense_useful_madds(true);
    const int conc = std::max(1, std::min(concurrency > 0 ? concurrency : 8, std::max(n_images, 1)));
    const long long n0 = net->L[0].numel();
    const int nm = std::max(1, net->n_out - 1);
    size_t free_b = 0, total_b = 0;
    ck(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
    const long long budget = std::min<long long>(16ll << 30, (long long)(free_b * 0.6) / conc);
    cudaStream_t master;
    cudaEvent_t start, end;
    ck(cudaStreamCreateWithFlags(&master, cudaStreamNonBlocking), "stream");
    ck(cudaEventCreate(&start), "event");
    ck(cudaEventCreate(&end), "event");
    // Image batching: each worker verifies B images per schedule (one
    // kernel launch carries B images' rows). Needs every label (margin pass).
    static const int batch_env = env_int("PC_IMG_BATCH", -1);
    bool labeled = n_images >= 2 && net->opt.exec_mode != 2;
    for (int i = 0; labeled && i < n_images; ++i) labeled = labels[i] >= 0 && labels[i] < net->n_out;
    int B = 1;
    if (labeled) {
      B = batch_env >= 0 ? batch_env : (n_images + conc - 1) / conc;
      if (net->total > (1ll << 20)) B = std::min(B, 4);  // large nets: per-image state is big
      B = std::max(1, std::min(B, kMaxBatch));
    }
    std::vector<Ctx*> ctxs(conc);
    for (int w = 0; w < conc; ++w) {
      ctxs[w] = B > 1 ? acquire_batched(net, B) : acquire(net);
      apply_call_options(ctxs[w], nullptr);  // the net's options (a leased context keeps the last call's)
      ctxs[w]->budget = budget;
    }
    ck(cudaEventRecord(start, master), "event");
    for (Ctx* c : ctxs) ck(cudaStreamWaitEvent(c->stream, start, 0), "wait");
    std::atomic<int> next{0};
    std::atomic<long long> launches{0};
    double agg_dense_ms = 0, agg_dense_bytes = 0;
    long long agg_dense_launches = 0;
    std::mutex err_mu;
    std::string err;
    pc_status err_code = PC_OK;
    auto work_batched = [&](int w) {
      cudaSetDevice(net->device);
      g_launches = 0;
      Ctx* c = ctxs[w];
      const long long T = c->total;
      std::vector<double> mg((size_t)B * nm);
      std::vector<pc_stats> sts(B);
      for (;;) {
        const int i = next.fetch_add(B);
        if (i >= n_images) break;
        const int nb = std::min(B, n_images - i);
        const pc_status st = guard([&] {
          cudaStream_t s = c->stream;
          for (int b = 0; b < nb; ++b) {
            const double* li = lo + (size_t)(i + b) * n0;
            const double* ui = up + (size_t)(i + b) * n0;
            const cudaMemcpyKind kind = device_inputs ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
            if (!device_inputs)
              for (long long k = 0; k < n0; ++k)
                if (std::isnan(li[k]) || std::isnan(ui[k]))
                  throw StatusError(PC_ERR_INVALID_ARGUMENT, "Interval: NaN endpoint");
            ck(cudaMemcpyAsync(c->blo + b * T, li, sizeof(double) * n0, kind, s), "box");
            ck(cudaMemcpyAsync(c->bhi + b * T, ui, sizeof(double) * n0, kind, s), "box");
            ck(cudaMemcpyAsync(c->rlo + b * T, c->blo + b * T, sizeof(double) * n0, cudaMemcpyDeviceToDevice, s), "box");
            ck(cudaMemcpyAsync(c->rhi + b * T, c->bhi + b * T, sizeof(double) * n0, cudaMemcpyDeviceToDevice, s), "box");
          }
          c->ev_used = 0;
          c->sync_used = 0;
          c->prof.clear();
          c->dense_ev.clear();
          g_dense_bytes = g_dense_madds = 0;
          g_dense_launches = 0;
          run_test_batched(c, nb, labels + i, mg.data(), sts.data());
          ck(cudaGetLastError(), "kernel");  // a failed launch voids the results
          // the dense kernel's live timing (bench.py's roofline) across workers
          double dms = 0;
          for (size_t e : c->dense_ev) {
            float d = 0;
            if (cudaEventElapsedTime(&d, c->ev_pool[e], c->ev_pool[e + 1]) == cudaSuccess) dms += d;
          }
          (void)cudaGetLastError();  // timing is best effort: drop only its own errors
          {
            std::lock_guard<std::mutex> lk(err_mu);
            agg_dense_ms += dms;
            agg_dense_bytes += g_dense_bytes;
            agg_dense_launches += g_dense_launches;
          }
          const int nr = net->n_out - 1;
          for (int b = 0; b < nb; ++b) {
            bool v = true;
            for (int r = 0; r < nr; ++r) {
              if (margins) margins[(size_t)(i + b) * nm + r] = mg[(size_t)b * nr + r];
              if (!(mg[(size_t)b * nr + r] > 0.0)) v = false;
            }
            if (verified) verified[i + b] = v ? 1 : 0;
            if (stats) stats[i + b] = sts[b];
          }
        });
        if (st != PC_OK) {
          std::lock_guard<std::mutex> lk(err_mu);
          if (err_code == PC_OK) {
            err_code = st;
            err = g_err;
          }
        }
      }
      launches += g_launches;
    };
    auto work = [&](int w) {
      if (B > 1) {
        work_batched(w);
        return;
      }
      cudaSetDevice(net->device);
      g_launches = 0;
      for (;;) {
        const int i = next.fetch_add(1);
        if (i >= n_images) break;
        const double* li = lo + (size_t)i * n0;
        const double* ui = up + (size_t)i * n0;
        const pc_status st = guard([&] {
          run_one(ctxs[w], li, ui, device_inputs != 0, labels[i], verified ? verified + i : nullptr,
                  margins ? margins + (size_t)i * nm : nullptr, nullptr, nullptr, nullptr, nullptr,
                  stats ? stats + i : nullptr);
        });
        if (st != PC_OK) {
          std::lock_guard<std::mutex> lk(err_mu);
          if (err_code == PC_OK) {
            err_code = st;
            err = g_err;
          }
        }
      }
      launches += g_launches;
    };
    std::vector<std::thread> pool;
    for (int w = 1; w < conc; ++w) pool.emplace_back(work, w);
    work(0);
    for (auto& t : pool) t.join();
    cudaEvent_t* done = new cudaEvent_t[conc];
    for (int w = 0; w < conc; ++w) {
      ck(cudaEventCreate(&done[w]), "event");
      ck(cudaEventRecord(done[w], ctxs[w]->stream), "event");
      ck(cudaStreamWaitEvent(master, done[w], 0), "wait");
    }
    ck(cudaEventRecord(end, master), "event");
    ck(cudaStreamSynchronize(master), "sync");
    float ms = 0;
    cudaEventElapsedTime(&ms, start, end);
    if (device_ms) *device_ms = ms;
    for (int w = 0; w < conc; ++w) {
      cudaEventDestroy(done[w]);
      ctxs[w]->budget = 0;
      release(net, ctxs[w]);
    }
    delete[] done;
    cudaEventDestroy(start);
    cudaEventDestroy(end);
    cudaStreamDestroy(master);
    g_last_launches = launches.load();
    if (B > 1) {
      g_dense_ms = agg_dense_ms;
      g_dense_bytes = agg_dense_bytes;
      g_dense_launches = agg_dense_launches;
    }
    g_dense_madds = (double)dense_useful_madds(false);  // executed, all workers
    if (err_code != PC_OK) throw StatusError(err_code, err);
  });
}

pc_status pc_net_set_sharding(pc_net* net, int rank, int world, pc_allgather_fn allgather,
                              void* user) {
  if (!net || world < 1 || rank < 0 || rank >= world || (world > 1 && !allgather)) {
    g_err = "sharding: need 0 <= rank < world and an allgather callback";
    return PC_ERR_INVALID_ARGUMENT;
  }
  net->shard_rank = world > 1 ? rank : 0;
  net->shard_world = world;
  net->allgather = world > 1 ? allgather : nullptr;
  net->allgather_user = world > 1 ? user : nullptr;
  return PC_OK;
}

pc_status pc_net_test_device(pc_net* n, const double* d_lo, const double* d_up, int label,
                             int* verified, double* margins, pc_stats* stats) {
  return test_impl(n, nullptr, d_lo, d_up, true, label, verified, margins, nullptr, nullptr,
                   nullptr, nullptr, stats);
}

}  // extern "C"
