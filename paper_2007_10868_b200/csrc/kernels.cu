// kernels.cu — sm_100a kernels of the DeepPoly back-substitution hot path.
//
// All arithmetic goes through numeric.cuh (bit-exact WidenedFloat64). Every
// accumulation runs in the reference's order; sums are never split or
// reassociated (backsub.hpp:31-34). Parallelism comes from independent rows,
// independent output coefficients and independent neurons; each serial
// constant/concretisation chain is one lane.
#include <cub/block/block_scan.cuh>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <string>

#include "kernels.cuh"
#include "numeric.cuh"
#include "scanfold.cuh"

namespace pc {

thread_local long long g_launches = 0;

void init_kernel_attrs(int device) {
  static std::mutex mu;
  static unsigned long long done = 0;  // one bit per device ordinal (< 64)
  std::lock_guard<std::mutex> lk(mu);
  const unsigned long long bit = 1ull << (device & 63);
  if (done & bit) return;
  init_kernel_attrs_kernels();
  init_kernel_attrs_chains();
  init_kernel_attrs_gbc();
  done |= bit;
}

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e && *e ? atoi(e) : dflt;
}

long long big_chain_cells() {
  static const long long v = [] {
    const char* e = getenv("PC_BIG_CHAIN_CELLS");
    return e && *e ? atoll(e) : 2048ll;
  }();
  return v;
}

// CTA-per-row chain kernels (chains.cu) for long rows. They shorten a lone
// walk's critical path, but hold 512 threads per row while the serial fold
// runs; image-batched walks share the GPU with other worker contexts, where
// the warp-per-row kernels' smaller footprint lets more of the coefficient
// kernels stay resident (PC_BIG_CHAIN_CELLS_BATCHED: the cell count from
// which batched walks still use them).
static bool use_big_chains(long long cells, const RowsDev& rows) {
  static const long long batched = env_int("PC_BIG_CHAIN_CELLS_BATCHED", 4096);
  return cells >= big_chain_cells() && (rows.nimg <= 1 || cells >= batched);
}

#define PC_NAN __longlong_as_double(0x7ff8000000000000ULL)

static inline unsigned cdiv(long long a, long long b) { return (unsigned)((a + b - 1) / b); }

bool debug_skip(const char* what) {
  static const std::string v = [] {
    const char* e = getenv("PC_DEBUG_SKIP");
    return std::string(e ? e : "");
  }();
  return !v.empty() && v.find(what) != std::string::npos;
}

// ===========================================================================
// Forward interval propagation: affine_bound / compute_layer_bounds
// (eval.hpp:109-228), recompute_dev (analyzer.hpp:82-159) and
// relu_relaxation (analyzer.hpp:38-70), fused per layer. Thread = (neuron,
// track): track 0 computes the padded bound from padded predecessor bounds
// plus dev and (if the layer feeds a relu) the relaxation; track 1 computes
// the raw twin from raw predecessor bounds. Each is a serial chain over the
// fan-in in the reference's order.
// ===========================================================================

__device__ __forceinline__ void store_relax(double* relax, long long j, const Iv& b) {
  const Relax r = relu_relaxation(b);
  double* p = relax + 8 * j;
  p[0] = r.alpha.lo; p[1] = r.alpha.hi; p[2] = r.beta.lo; p[3] = r.beta.hi;
  p[4] = r.gamma.lo; p[5] = r.gamma.hi; p[6] = r.delta.lo; p[7] = r.delta.hi;
}

// One affine term of affine_bound (eval.hpp:133-148) for both tracks:
// padded (lo, hi, abs_hi) from padded inputs and raw (rlo, rhi) from raw
// inputs. Zero weights are skipped (selects, no branch, in the fast path).
template <bool FAST>
__device__ __forceinline__ void affine_term(double w, double a, double b, double ra, double rb,
                                            double& lo, double& hi, double& ab, double& rlo,
                                            double& rhi, long long& terms, bool& bad) {
  const bool nz = w != 0.0, pos = w > 0.0;
  const double x1 = pos ? a : b, x2 = pos ? b : a;
  const double r1 = pos ? ra : rb, r2 = pos ? rb : ra;
  if (FAST) {
    const double pl = f_mul_dn(w, x1, bad), ph = f_mul_up(w, x2, bad);
    const double pa = f_mul_up(fabs(w), smax(fabs(a), fabs(b)), bad);
    const double ql = f_mul_dn(w, r1, bad), qh = f_mul_up(w, r2, bad);
    const double n_lo = f_add_dn(lo, pl), n_hi = f_add_up(hi, ph), n_ab = f_add_up(ab, pa);
    const double n_rlo = f_add_dn(rlo, ql), n_rhi = f_add_up(rhi, qh);
    lo = nz ? n_lo : lo;
    hi = nz ? n_hi : hi;
    ab = nz ? n_ab : ab;
    rlo = nz ? n_rlo : rlo;
    rhi = nz ? n_rhi : rhi;
    terms += nz;
  } else {
    if (!nz) return;
    ++terms;
    ab = add_up(ab, mul_up(fabs(w), smax(fabs(a), fabs(b))));
    lo = add_down(lo, mul_down(w, x1));
    hi = add_up(hi, mul_up(w, x2));
    rlo = add_down(rlo, mul_down(w, r1));
    rhi = add_up(rhi, mul_up(w, r2));
  }
}

// Padded result, dev and relaxation of one affine neuron (eval.hpp:149-151,
// analyzer.hpp:109/140, analyzer.hpp:38-70).
__device__ __forceinline__ void affine_finish(long long j, double lo, double hi, double ab,
                                              long long terms, long long dterms, double rlo,
                                              double rhi, double* ylo, double* yhi,
                                              double* yrlo, double* yrhi, double* dev,
                                              double* relax) {
  const double slack = __dmul_rn(__dmul_rn(2.0, (double)(terms + 1)), ulp_above(ab));
  const Iv y{add_down(lo, -slack), add_up(hi, slack)};
  ylo[j] = y.lo;
  yhi[j] = y.hi;
  yrlo[j] = rlo;
  yrhi[j] = rhi;
  // recompute_dev: the |w|*mag chain over all inputs equals abs_hi (zero
  // weights add an exact 0); only the term count differs.
  dev[j] = __dmul_rn(__dmul_rn(2.0, (double)(dterms + 1)), ulp_above(ab));
  if (relax) store_relax(relax, j, y);
}

// Dirty tracking for the refresh after each pass (analyzer.hpp:232-239). A
// refresh is a pure function of predecessor bounds, so a neuron whose inputs
// did not change in this round keeps bit-identical bounds, dev and
// relaxation; it is skipped. gen_n / gen_pos / gen_l record the round in
// which a neuron / grid position / layer last changed (changed = any of the
// four bound bit patterns differs). force: recompute everything (initial
// forward pass).
struct Dirty {
  int* gen_n;    // per neuron (all layers, layer offsets)
  int* gen_pos;  // per grid position (all layers, position offsets)
  int* gen_l;    // per layer
  int g;
  int force;
  // image-batched launches: blockIdx.z = image; per-image strides of the
  // neuron-indexed state (and gen_n), of gen_pos and of gen_l
  long long zs = 0, zp = 0;
  int zl = 0;
};

// Rebase one image's pointers (blockIdx.z) of a forward kernel.
#define PC_FWD_IMAGE(...)                                      \
  const long long pc_zo = (long long)blockIdx.z * dt.zs;       \
  dt.gen_n += pc_zo;                                           \
  dt.gen_pos += (long long)blockIdx.z * dt.zp;                 \
  dt.gen_l += (long long)blockIdx.z * dt.zl;                   \
  __VA_ARGS__

__device__ __forceinline__ bool bits_differ(double a, double b) {
  return __double_as_longlong(a) != __double_as_longlong(b);
}

__device__ __forceinline__ void mark_changed(const Dirty& dt, long long neuron, long long pos,
                                             int layer) {
  dt.gen_n[neuron] = dt.g;
  if (pos >= 0) dt.gen_pos[pos] = dt.g;
  dt.gen_l[layer] = dt.g;
}

// Store one refreshed neuron; mark it if any track changed.
__device__ __forceinline__ void store_bounds(double* ylo, double* yhi, double* yrlo, double* yrhi,
                                             long long j, const Iv& y, double rl, double rh,
                                             const Dirty& dt, long long gofs, long long pos,
                                             int layer) {
  const bool ch = dt.force || bits_differ(ylo[j], y.lo) || bits_differ(yhi[j], y.hi) ||
                  bits_differ(yrlo[j], rl) || bits_differ(yrhi[j], rh);
  ylo[j] = y.lo;
  yhi[j] = y.hi;
  yrlo[j] = rl;
  yrhi[j] = rh;
  if (ch) mark_changed(dt, gofs + j, pos, layer);
}

// Dense layer. Block = 32 neurons x 2 tracks (warp 0: padded lo/hi/abs,
// warp 1: raw lo/hi); weights and inputs staged through shared memory in
// ascending input tiles.
constexpr int kFDN = 32, kFDT = 64;  // kFDT == 2 * kFDN: one input per thread per tile

template <bool FAST>
__device__ __forceinline__ void pad_term(double w, double a, double b, double m, double& lo,
                                         double& hi, double& ab, long long& terms, bool& bad) {
  const bool nz = w != 0.0, pos = w > 0.0;
  const double x1 = pos ? a : b, x2 = pos ? b : a;
  if (FAST) {
    const double pl = f_mul_dn(w, x1, bad), ph = f_mul_up(w, x2, bad);
    const double pa = f_mul_up(fabs(w), m, bad);
    const double n_lo = f_add_dn(lo, pl), n_hi = f_add_up(hi, ph), n_ab = f_add_up(ab, pa);
    lo = nz ? n_lo : lo;
    hi = nz ? n_hi : hi;
    ab = nz ? n_ab : ab;
    terms += nz;
  } else {
    if (!nz) return;
    ++terms;
    ab = add_up(ab, mul_up(fabs(w), m));
    lo = add_down(lo, mul_down(w, x1));
    hi = add_up(hi, mul_up(w, x2));
  }
}

template <bool FAST>
__device__ __forceinline__ void raw_term(double w, double a, double b, double& lo, double& hi,
                                         bool& bad) {
  const bool nz = w != 0.0, pos = w > 0.0;
  const double x1 = pos ? a : b, x2 = pos ? b : a;
  if (FAST) {
    const double pl = f_mul_dn(w, x1, bad), ph = f_mul_up(w, x2, bad);
    const double n_lo = f_add_dn(lo, pl), n_hi = f_add_up(hi, ph);
    lo = nz ? n_lo : lo;
    hi = nz ? n_hi : hi;
  } else {
    if (!nz) return;
    lo = add_down(lo, mul_down(w, x1));
    hi = add_up(hi, mul_up(w, x2));
  }
}

// In-band forms of pad_term / raw_term (see madd_band): valid when every
// nonzero product is in [2^-499, 2^999] (checked per block from the input
// bounds' magnitudes and the layer's weight range) and no accumulator starts
// at -0. A zero weight or bound gives exact +-0 products, which leave the
// accumulators unchanged up to a -0 lower bound (canonicalised at the end),
// so only the term count needs the w != 0 test.
__device__ __forceinline__ void band_pad_term(double w, double a, double b, double m, double& lo,
                                              double& hi, double& ab, long long& terms) {
  const bool neg = __double2hiint(w) < 0;
  double pl, ph;
  band_products_ab(w, neg ? b : a, neg ? a : b, pl, ph);
  const double aw = fabs(w);
  const double p0 = __dmul_rn(aw, m);
  const double pa = __dadd_ru(p0, fabs(__fma_rn(aw, m, -p0)));
  band_sums(pl, ph, lo, hi);
  const double sa = __dadd_rn(ab, pa), da = __dadd_rd(ab, pa), ua = __dadd_ru(ab, pa);
  ab = __fma_ru(__dsub_rn(ua, da), 0.5, sa);
  terms += w != 0.0;
}
__device__ __forceinline__ void band_raw_term(double w, double a, double b, double& lo,
                                              double& hi) {
  const bool neg = __double2hiint(w) < 0;
  double pl, ph;
  band_products_ab(w, neg ? b : a, neg ? a : b, pl, ph);
  band_sums(pl, ph, lo, hi);
}

__global__ void __launch_bounds__(2 * kFDN)
    k_fwd_dense(LayerDev L, int layer, const double* xlo, const double* xhi, const double* xrlo,
                const double* xrhi, double* ylo, double* yhi, double* yrlo, double* yrhi,
                double* dev, double* relax, Dirty dt, long long gofs) {
  PC_FWD_IMAGE(xlo += pc_zo; xhi += pc_zo; xrlo += pc_zo; xrhi += pc_zo; ylo += pc_zo; yhi += pc_zo;
               yrlo += pc_zo; yrhi += pc_zo; dev += pc_zo; if (relax) relax += 8 * pc_zo;)
  if (!dt.force && dt.gen_l[L.pred0] != dt.g) return;  // no input changed this round
  __shared__ double s_w[kFDT][kFDN];
  __shared__ double s_x[5][kFDT];  // padded lo, hi, mag; raw lo, hi
  __shared__ int s_live[kFDT], s_dead[kFDT], s_cnt[2][2];
  const int n_out = L.out_c;
  const int n_in = L.in_w * L.in_h * L.in_c;
  const int lane = threadIdx.x & 31, track = threadIdx.x >> 5;
  const int j0 = blockIdx.x * kFDN, j = j0 + lane;
  const bool act = j < n_out;
  const double bias = act ? L.bias[j] : 0.0;
  double lo = bias, hi = bias, ab = fabs(bias);
  long long terms = 1;
  bool bad = false;
  // Inputs whose padded and raw bounds are both [0, 0] (stably-negative
  // ReLU outputs) add exact zeros: a no-op on the accumulators unless one is
  // still -0, which only a -0 bias can start (RN sums of nonzero terms never
  // return to -0). They only count as terms (w != 0); blocks with a -0 bias
  // run every input.
  const bool neg0_bias = __syncthreads_or(act && __double_as_longlong(bias) == (long long)0x8000000000000000ULL);
  const bool skip_dead = !neg0_bias;
  // Band check for the lean forms: magnitudes of the nonzero input bounds
  // (padded and raw) against the layer's weight range, and the biases.
  bool band;
  {
    MagAcc mag;
    for (int t = threadIdx.x; t < n_in; t += 2 * kFDN) {
      mag.add(xlo[t]);
      mag.add(xhi[t]);
      mag.add(xrlo[t]);
      mag.add(xrhi[t]);
    }
    __shared__ unsigned s_stat[2];
    if (threadIdx.x == 0) s_stat[0] = s_stat[1] = 0xFFFFFFFFu;
    __syncthreads();
    mag.flush_shared(s_stat);
    __syncthreads();
    band = !neg0_bias && n_in < (1 << 20) && products_in_band(s_stat, L.wmin, L.wmax) &&
           !__syncthreads_or(act && !(fabs(bias) <= 0x1p999));
  }
  for (int t0 = 0; t0 < n_in; t0 += kFDT) {
    const int tn = min(kFDT, n_in - t0);
    __syncthreads();
    for (int e = threadIdx.x; e < kFDT * kFDN; e += 2 * kFDN) {
      const int tt = e / kFDN, jj = e % kFDN;
      s_w[tt][jj] = (tt < tn && j0 + jj < n_out) ? L.WT[(size_t)(t0 + tt) * n_out + j0 + jj] : 0.0;
    }
    {  // one input per thread (kFDT == 2 * kFDN)
      const int e = threadIdx.x;
      bool live = false;
      if (e < tn) {
        const double a = xlo[t0 + e], b = xhi[t0 + e], ra = xrlo[t0 + e], rb = xrhi[t0 + e];
        s_x[0][e] = a;
        s_x[1][e] = b;
        s_x[2][e] = smax(fabs(a), fabs(b));
        s_x[3][e] = ra;
        s_x[4][e] = rb;
        live = !skip_dead || !(a == 0.0 && b == 0.0 && ra == 0.0 && rb == 0.0);
      }
      const unsigned bl = __ballot_sync(0xFFFFFFFFu, live);
      const unsigned bd = __ballot_sync(0xFFFFFFFFu, e < tn && !live);
      if (lane == 0) {
        s_cnt[0][track] = __popc(bl);
        s_cnt[1][track] = __popc(bd);
      }
      __syncthreads();
      const unsigned below = (1u << lane) - 1u;
      if (e < tn) {
        if (live) s_live[(track ? s_cnt[0][0] : 0) + __popc(bl & below)] = e;
        else s_dead[(track ? s_cnt[1][0] : 0) + __popc(bd & below)] = e;
      }
    }
    __syncthreads();
    const int n_live = s_cnt[0][0] + s_cnt[0][1], n_dead = s_cnt[1][0] + s_cnt[1][1];
    if (track == 0) {
      for (int i = 0; i < n_dead; ++i) terms += s_w[s_dead[i]][lane] != 0.0;
      if (band) {
#pragma unroll 4
        for (int i = 0; i < n_live; ++i) {
          const int t = s_live[i];
          band_pad_term(s_w[t][lane], s_x[0][t], s_x[1][t], s_x[2][t], lo, hi, ab, terms);
        }
      } else {
#pragma unroll 4
        for (int i = 0; i < n_live; ++i) {
          const int t = s_live[i];
          pad_term<true>(s_w[t][lane], s_x[0][t], s_x[1][t], s_x[2][t], lo, hi, ab, terms, bad);
        }
      }
    } else {
      if (band) {
#pragma unroll 4
        for (int i = 0; i < n_live; ++i) {
          const int t = s_live[i];
          band_raw_term(s_w[t][lane], s_x[3][t], s_x[4][t], lo, hi);
        }
      } else {
#pragma unroll 4
        for (int i = 0; i < n_live; ++i) {
          const int t = s_live[i];
          raw_term<true>(s_w[t][lane], s_x[3][t], s_x[4][t], lo, hi, bad);
        }
      }
    }
  }
  if (band) lo = canon0(lo);  // the reference's accumulators are never -0 here
  if (act && bad) {  // out-of-band operand: redo this chain with the exact ops
    lo = hi = bias;
    ab = fabs(bias);
    terms = 1;
    for (int t = 0; t < n_in; ++t) {
      const double w = L.WT[(size_t)t * n_out + j];
      if (track == 0)
        pad_term<false>(w, xlo[t], xhi[t], smax(fabs(xlo[t]), fabs(xhi[t])), lo, hi, ab, terms, bad);
      else
        raw_term<false>(w, xrlo[t], xrhi[t], lo, hi, bad);
    }
  }
  // exchange: padded warp needs the raw result of its neuron and vice versa
  __shared__ double s_raw[2][kFDN];
  if (track == 1) {
    s_raw[0][lane] = lo;
    s_raw[1][lane] = hi;
  }
  __syncthreads();
  if (track != 0 || !act) return;
  const double slack = __dmul_rn(__dmul_rn(2.0, (double)(terms + 1)), ulp_above(ab));
  const Iv y{add_down(lo, -slack), add_up(hi, slack)};
  const bool ch = dt.force || bits_differ(ylo[j], y.lo) || bits_differ(yhi[j], y.hi) ||
                  bits_differ(yrlo[j], s_raw[0][lane]) || bits_differ(yrhi[j], s_raw[1][lane]);
  ylo[j] = y.lo;
  yhi[j] = y.hi;
  yrlo[j] = s_raw[0][lane];
  yrhi[j] = s_raw[1][lane];
  dev[j] = __dmul_rn(__dmul_rn(2.0, (double)(n_in + 2)), ulp_above(ab));  // analyzer.hpp:109
  if (relax) store_relax(relax, j, y);
  if (ch) mark_changed(dt, gofs + j, -1, layer);
}

// Conv layer: one thread per output neuron (h, w, d), both tracks; taps in
// the reference order (fy, fx, ci), out-of-grid taps skipped.
template <bool FAST>
__device__ __forceinline__ bool fwd_conv_chain(const LayerDev& L, int h, int w, int d,
                                               const double* xl, const double* xh,
                                               const double* xrl, const double* xrh, double& lo,
                                               double& hi, double& ab, double& rlo, double& rhi,
                                               long long& terms, long long& dterms) {
  const double bias = L.bias[d];
  lo = hi = rlo = rhi = bias;
  ab = fabs(bias);
  terms = 1;
  dterms = 1;
  bool bad = false;
  const int cin = L.in_c, cout = L.out_c;
  for (int fy = 0; fy < L.fh; ++fy) {
    const int iy = h * L.sh - L.ph + fy;
    if (iy < 0 || iy >= L.in_h) continue;
    for (int fx = 0; fx < L.fw; ++fx) {
      const int ix = w * L.sw - L.pw + fx;
      if (ix < 0 || ix >= L.in_w) continue;
      const double* fp = L.F + ((size_t)(fy * L.fw + fx) * cin) * cout + d;
      const size_t xb = ((size_t)iy * L.in_w + ix) * cin;
      dterms += cin;
#pragma unroll 4
      for (int ci = 0; ci < cin; ++ci)
        affine_term<FAST>(fp[(size_t)ci * cout], xl[xb + ci], xh[xb + ci], xrl[xb + ci],
                          xrh[xb + ci], lo, hi, ab, rlo, rhi, terms, bad);
    }
  }
  return bad;
}

__global__ void __launch_bounds__(128)
    k_fwd_conv(LayerDev L, int layer, const double* xlo, const double* xhi, const double* xrlo,
               const double* xrhi, double* ylo, double* yhi, double* yrlo, double* yrhi,
               double* dev, double* relax, Dirty dt, long long gofs, long long pofs_in,
               long long pofs_out) {
  PC_FWD_IMAGE(xlo += pc_zo; xhi += pc_zo; xrlo += pc_zo; xrhi += pc_zo; ylo += pc_zo; yhi += pc_zo;
               yrlo += pc_zo; yrhi += pc_zo; dev += pc_zo; if (relax) relax += 8 * pc_zo;)
  if (!dt.force && dt.gen_l[L.pred0] != dt.g) return;
  const long long numel = (long long)L.out_w * L.out_h * L.out_c;
  const long long jj = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (jj >= numel) return;
  const int d = (int)(jj % L.out_c);
  const int w = (int)((jj / L.out_c) % L.out_w);
  const int h = (int)(jj / ((long long)L.out_c * L.out_w));
  if (!dt.force) {  // any input position of the receptive field changed this round?
    bool any = false;
    for (int fy = 0; fy < L.fh && !any; ++fy) {
      const int iy = h * L.sh - L.ph + fy;
      if (iy < 0 || iy >= L.in_h) continue;
      for (int fx = 0; fx < L.fw; ++fx) {
        const int ix = w * L.sw - L.pw + fx;
        if (ix < 0 || ix >= L.in_w) continue;
        if (dt.gen_pos[pofs_in + (long long)iy * L.in_w + ix] == dt.g) {
          any = true;
          break;
        }
      }
    }
    if (!any) return;
  }
  double lo, hi, ab, rlo, rhi;
  long long terms, dterms;
  if (fwd_conv_chain<true>(L, h, w, d, xlo, xhi, xrlo, xrhi, lo, hi, ab, rlo, rhi, terms, dterms))
    fwd_conv_chain<false>(L, h, w, d, xlo, xhi, xrlo, xrhi, lo, hi, ab, rlo, rhi, terms, dterms);
  const double slack = __dmul_rn(__dmul_rn(2.0, (double)(terms + 1)), ulp_above(ab));
  const Iv y{add_down(lo, -slack), add_up(hi, slack)};
  store_bounds(ylo, yhi, yrlo, yrhi, jj, y, rlo, rhi, dt, gofs, pofs_out + (long long)h * L.out_w + w,
               layer);
  dev[jj] = __dmul_rn(__dmul_rn(2.0, (double)(dterms + 1)), ulp_above(ab));  // analyzer.hpp:140
  if (relax) store_relax(relax, jj, y);
}

// Conv layer forward with the taps staged through shared memory. A block is
// 64 output channels of one position (out_c % 64 == 0), so its threads walk
// the same receptive field in the same order (fy, fx, ci; out-of-grid taps
// skipped, eval.hpp:150-200): chunks of kFC taps, their inputs (4 tracks) and
// weight rows (64 channels) are copied by cp.async into a double buffer while
// the previous chunk is folded. The chain per output is the reference's, so
// results equal k_fwd_conv's; the few-warps-per-SM launches of the deep
// layers then wait on shared memory instead of an L2 round trip per tap.
constexpr int kFC = 32;
template <bool FAST>
__device__ __forceinline__ bool fwd_conv_staged(const LayerDev& L, int h, int w, int d0, const double* xl,
                                                const double* xh, const double* xrl, const double* xrh,
                                                double (*sw)[kFC][64], double (*sx)[4][kFC], double& lo,
                                                double& hi, double& ab, double& rlo, double& rhi,
                                                long long& terms, long long& dterms) {
  const int tid = threadIdx.x, d = d0 + tid;
  const int cin = L.in_c, cout = L.out_c;
  const int y0 = h * L.sh - L.ph, x0 = w * L.sw - L.pw;
  const int fy0 = max(0, -y0), fy1 = min(L.fh, L.in_h - y0);  // valid taps [fy0, fy1)
  const int fx0 = max(0, -x0), fx1 = min(L.fw, L.in_w - x0);
  const int ny = max(0, fy1 - fy0), nx = max(0, fx1 - fx0);
  const long long T = (long long)ny * nx * cin;
  const double bias = L.bias[d];
  lo = hi = rlo = rhi = bias;
  ab = fabs(bias);
  terms = 1;
  dterms = 1 + T;
  bool bad = false;
  const int nch = (int)((T + kFC - 1) / kFC);
  // incremental tap cursor of the copies (fy, fx, ci), advanced in issue order
  int cfy = fy0, cfx = fx0, cci = 0;
  auto issue = [&](int c, int buf) {
    const long long g0 = (long long)c * kFC;
    int fy = cfy, fx = cfx, ci = cci;
    for (int t = 0; t < kFC; ++t) {
      const bool v = g0 + t < T;
      const double* src = L.F + ((size_t)(fy * L.fw + fx) * cin + ci) * cout + d;
      cp_async8(&sw[buf][t][tid], v ? src : L.F, v);
      if (tid == t) {
        const size_t xb = ((size_t)(y0 + fy) * L.in_w + (x0 + fx)) * cin + ci;
        cp_async8(&sx[buf][0][t], v ? xl + xb : xl, v);
        cp_async8(&sx[buf][1][t], v ? xh + xb : xh, v);
        cp_async8(&sx[buf][2][t], v ? xrl + xb : xrl, v);
        cp_async8(&sx[buf][3][t], v ? xrh + xb : xrh, v);
      }
      if (v && ++ci == cin) {
        ci = 0;
        if (++fx == fx1) {
          fx = fx0;
          ++fy;
        }
      }
    }
    cfy = fy;
    cfx = fx;
    cci = ci;
    cp_async_commit();
  };
  if (nch > 0) issue(0, 0);
  for (int c = 0; c < nch; ++c) {
    if (c + 1 < nch) {
      issue(c + 1, (c + 1) & 1);
      cp_async_wait_one();
    } else {
      cp_async_wait_all();
    }
    __syncthreads();
    const int b = c & 1;
    const long long rem = T - (long long)c * kFC;
    const int n = rem < kFC ? (int)rem : kFC;
    for (int t = 0; t < n; ++t)
      affine_term<FAST>(sw[b][t][tid], sx[b][0][t], sx[b][1][t], sx[b][2][t], sx[b][3][t], lo, hi, ab, rlo, rhi,
                        terms, bad);
    __syncthreads();
  }
  return bad;
}

__global__ void __launch_bounds__(64)
    k_fwd_conv_staged(LayerDev L, int layer, const double* xlo, const double* xhi, const double* xrlo,
                      const double* xrhi, double* ylo, double* yhi, double* yrlo, double* yrhi, double* dev,
                      double* relax, Dirty dt, long long gofs, long long pofs_in, long long pofs_out) {
  __shared__ __align__(16) double sw[2][kFC][64];
  __shared__ __align__(16) double sx[2][4][kFC];
  PC_FWD_IMAGE(xlo += pc_zo; xhi += pc_zo; xrlo += pc_zo; xrhi += pc_zo; ylo += pc_zo; yhi += pc_zo;
               yrlo += pc_zo; yrhi += pc_zo; dev += pc_zo; if (relax) relax += 8 * pc_zo;)
  if (!dt.force && dt.gen_l[L.pred0] != dt.g) return;
  const int pos = blockIdx.x;
  const int h = pos / L.out_w, w = pos - h * L.out_w;
  const int d0 = blockIdx.y * 64;
  if (!dt.force) {  // any input position of the receptive field changed this round? (block-uniform)
    bool any = false;
    for (int fy = 0; fy < L.fh && !any; ++fy) {
      const int iy = h * L.sh - L.ph + fy;
      if (iy < 0 || iy >= L.in_h) continue;
      for (int fx = 0; fx < L.fw; ++fx) {
        const int ix = w * L.sw - L.pw + fx;
        if (ix < 0 || ix >= L.in_w) continue;
        if (dt.gen_pos[pofs_in + (long long)iy * L.in_w + ix] == dt.g) {
          any = true;
          break;
        }
      }
    }
    if (!any) return;
  }
  double lo, hi, ab, rlo, rhi;
  long long terms, dterms;
  const bool bad = fwd_conv_staged<true>(L, h, w, d0, xlo, xhi, xrlo, xrhi, sw, sx, lo, hi, ab, rlo, rhi, terms,
                                         dterms);
  if (__syncthreads_or(bad))  // operands outside the proven band: the literal restatement
    fwd_conv_staged<false>(L, h, w, d0, xlo, xhi, xrlo, xrhi, sw, sx, lo, hi, ab, rlo, rhi, terms, dterms);
  const long long jj = (long long)pos * L.out_c + d0 + threadIdx.x;
  const double slack = __dmul_rn(__dmul_rn(2.0, (double)(terms + 1)), ulp_above(ab));
  const Iv y{add_down(lo, -slack), add_up(hi, slack)};
  store_bounds(ylo, yhi, yrlo, yrhi, jj, y, rlo, rhi, dt, gofs, pofs_out + pos, layer);
  dev[jj] = __dmul_rn(__dmul_rn(2.0, (double)(dterms + 1)), ulp_above(ab));  // analyzer.hpp:140
  if (relax) store_relax(relax, jj, y);
}

__global__ void k_fwd_relu(long long n, int C, int layer, const double* xlo, const double* xhi,
                           const double* xrlo, const double* xrhi, double* ylo, double* yhi,
                           double* yrlo, double* yrhi, Dirty dt, long long gofs_in, long long gofs,
                           long long pofs_out) {
  PC_FWD_IMAGE(xlo += pc_zo; xhi += pc_zo; xrlo += pc_zo; xrhi += pc_zo; ylo += pc_zo; yhi += pc_zo;
               yrlo += pc_zo; yrhi += pc_zo;)
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (!dt.force && dt.gen_n[gofs_in + i] != dt.g) return;
  const Iv y{xlo[i] > 0.0 ? xlo[i] : 0.0, xhi[i] > 0.0 ? xhi[i] : 0.0};  // eval.hpp:210-217
  store_bounds(ylo, yhi, yrlo, yrhi, i, y, xrlo[i] > 0.0 ? xrlo[i] : 0.0,
               xrhi[i] > 0.0 ? xrhi[i] : 0.0, dt, gofs, pofs_out + i / C, layer);
}

__global__ void k_fwd_join(long long n, int C, int layer, const double* alo, const double* ahi,
                           const double* arlo, const double* arhi, const double* blo,
                           const double* bhi, const double* brlo, const double* brhi, double* ylo,
                           double* yhi, double* yrlo, double* yrhi, double* dev, double* relax,
                           Dirty dt, long long gofs_a, long long gofs_b, long long gofs,
                           long long pofs_out) {
  PC_FWD_IMAGE(alo += pc_zo; ahi += pc_zo; arlo += pc_zo; arhi += pc_zo; blo += pc_zo; bhi += pc_zo;
               brlo += pc_zo; brhi += pc_zo; ylo += pc_zo; yhi += pc_zo; yrlo += pc_zo; yrhi += pc_zo;
               dev += pc_zo; if (relax) relax += 8 * pc_zo;)
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (!dt.force && dt.gen_n[gofs_a + i] != dt.g && dt.gen_n[gofs_b + i] != dt.g) return;
  const Iv a{alo[i], ahi[i]}, b{blo[i], bhi[i]};
  const Iv y = iv_add(a, b);  // eval.hpp:219-223
  store_bounds(ylo, yhi, yrlo, yrhi, i, y, add_down(arlo[i], brlo[i]), add_up(arhi[i], brhi[i]),
               dt, gofs, pofs_out + i / C, layer);
  dev[i] = __dmul_rn(2.0, ulp_above(add_up(iv_mag(a), iv_mag(b))));  // analyzer.hpp:144-150
  if (relax) store_relax(relax, i, y);
}

__global__ void k_relax(long long n, const double* blo, const double* bhi, double* relax) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  store_relax(relax, i, Iv{blo[i], bhi[i]});
}

void launch_forward_layer(cudaStream_t s, const LayerDev& L, int feeds_relu, const double* blo,
                          const double* bhi, const double* rlo, const double* rhi,
                          const long long* offs, const long long* pofs, int k, int p0, int p1,
                          double* dev, double* relax, int* gen_n, int* gen_pos, int* gen_l, int g,
                          int force, int nimg, long long zs, long long zp, int zl) {
  if (debug_skip("forward")) return;
  const long long o = offs[k], a = offs[p0];
  double* ylo = const_cast<double*>(blo) + o;
  double* yhi = const_cast<double*>(bhi) + o;
  double* yrlo = const_cast<double*>(rlo) + o;
  double* yrhi = const_cast<double*>(rhi) + o;
  double* rx = feeds_relu ? relax + 8 * o : nullptr;
  const long long n = (long long)L.out_w * L.out_h * L.out_c;
  Dirty dt{gen_n, gen_pos, gen_l, g, force};
  dt.zs = zs;
  dt.zp = zp;
  dt.zl = zl;
  switch (L.kind) {
    case KIND_DENSE:
      k_fwd_dense<<<dim3(cdiv(n, kFDN), 1, nimg), 2 * kFDN, 0, s>>>(L, k, blo + a, bhi + a, rlo + a, rhi + a, ylo,
                                                     yhi, yrlo, yrhi, dev + o, rx, dt, o);
      break;
    case KIND_CONV: {
      static const int staged = env_int("PC_FWD_STAGED", 1);
      if (staged && L.out_c % 64 == 0)
        k_fwd_conv_staged<<<dim3(L.out_w * L.out_h, L.out_c / 64, nimg), 64, 0, s>>>(
            L, k, blo + a, bhi + a, rlo + a, rhi + a, ylo, yhi, yrlo, yrhi, dev + o, rx, dt, o, pofs[p0], pofs[k]);
      else
        k_fwd_conv<<<dim3(cdiv(n, 64), 1, nimg), 64, 0, s>>>(L, k, blo + a, bhi + a, rlo + a, rhi + a, ylo, yhi,
                                                            yrlo, yrhi, dev + o, rx, dt, o, pofs[p0], pofs[k]);
      break;
    }
    case KIND_RELU:
      k_fwd_relu<<<dim3(cdiv(n, 256), 1, nimg), 256, 0, s>>>(n, L.out_c, k, blo + a, bhi + a, rlo + a, rhi + a,
                                              ylo, yhi, yrlo, yrhi, dt, a, o, pofs[k]);
      break;
    case KIND_JOIN: {
      const long long b = offs[p1];
      k_fwd_join<<<dim3(cdiv(n, 256), 1, nimg), 256, 0, s>>>(n, L.out_c, k, blo + a, bhi + a, rlo + a, rhi + a,
                                              blo + b, bhi + b, rlo + b, rhi + b, ylo, yhi, yrlo,
                                              yrhi, dev + o, rx, dt, a, b, o, pofs[k]);
      break;
    }
    default:
      return;
  }
  ++g_launches;
}

void launch_relax(cudaStream_t s, const double* blo, const double* bhi, long long n,
                  double* relax) {
  k_relax<<<cdiv(n, 256), 256, 0, s>>>(n, blo, bhi, relax);
  ++g_launches;
}

// ===========================================================================
// Pass seeding: CandidateSet::seed + pre-freeze + live-row list
// (backsub.hpp:1000-1015). One block; stable row compaction by block scan.
// cand[q] = {lo, hi, raw_lo, raw_hi}.
// ===========================================================================

constexpr int kScanThreads = 1024;

__global__ void __launch_bounds__(kScanThreads)
    k_seed(int n, const double* blo, const double* bhi, const double* rlo, const double* rhi,
           int allow_freeze, int early_term, double* cand, char* frozen, int* live, int* n_live,
           unsigned long long* n_prefrozen, long long sst, long long kq, int pstride) {
  if (blockIdx.x) {  // image-batched: block b seeds image b
    const long long b = blockIdx.x;
    blo += b * sst; bhi += b * sst; rlo += b * sst; rhi += b * sst;
    cand += 4 * b * kq; frozen += b * kq; live += b * kq; n_live += b; n_prefrozen += b * pstride;
  }
  using Scan = cub::BlockScan<int, kScanThreads>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int s_base;
  if (threadIdx.x == 0) s_base = 0;
  int froze = 0;
  __syncthreads();
  for (int start = 0; start < n; start += kScanThreads) {
    const int q = start + threadIdx.x;
    int keep = 0;
    if (q < n) {
      const double l = blo[q], h = bhi[q], rl = rlo[q], rh = rhi[q];
      cand[4 * q + 0] = l;
      cand[4 * q + 1] = h;
      cand[4 * q + 2] = rl;
      cand[4 * q + 3] = rh;
      const bool st = allow_freeze && (!(rl < 0.0) || !(rh > 0.0));  // stable() :814-817
      frozen[q] = st ? 1 : 0;
      if (st && early_term) ++froze;
      keep = !(early_term && st);
    }
    int pos, total;
    Scan(tmp).ExclusiveSum(keep, pos, total);
    if (keep) live[s_base + pos] = q;
    __syncthreads();
    if (threadIdx.x == 0) s_base += total;
    __syncthreads();
  }
  if (froze) atomicAdd(n_prefrozen, (unsigned long long)froze);
  if (threadIdx.x == 0) *n_live = s_base;
}

void launch_seed(cudaStream_t s, int n, const double* blo, const double* bhi, const double* rlo,
                 const double* rhi, int allow_freeze, int early_term, double* cand, char* frozen,
                 int* live, int* n_live, unsigned long long* n_prefrozen, int nimg, long long sst,
                 long long kq, int pstride) {
  k_seed<<<nimg, kScanThreads, 0, s>>>(n, blo, bhi, rlo, rhi, allow_freeze, early_term, cand, frozen,
                                       live, n_live, n_prefrozen, sst, kq, pstride);
  ++g_launches;
}

// Write the best candidates back (backsub.hpp:1060-1064) and refresh the
// relaxation of the refined layer (analyzer.hpp:229-231); mark changed
// neurons for the refresh round g.
__global__ void k_writeback(int n, int C, int layer, const double* cand, double* blo, double* bhi,
                            double* rlo, double* rhi, double* relax, Dirty dt, long long gofs,
                            long long pofs, long long kq) {
  PC_FWD_IMAGE(blo += pc_zo; bhi += pc_zo; rlo += pc_zo; rhi += pc_zo; if (relax) relax += 8 * pc_zo;
               cand += 4 * (long long)blockIdx.z * kq;)
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const Iv b{cand[4 * q + 0], cand[4 * q + 1]};
  const bool ch = bits_differ(blo[q], b.lo) || bits_differ(bhi[q], b.hi) ||
                  bits_differ(rlo[q], cand[4 * q + 2]) || bits_differ(rhi[q], cand[4 * q + 3]);
  blo[q] = b.lo;
  bhi[q] = b.hi;
  rlo[q] = cand[4 * q + 2];
  rhi[q] = cand[4 * q + 3];
  if (relax) store_relax(relax, q, b);
  if (ch) mark_changed(dt, gofs + q, pofs + q / C, layer);
}

void launch_writeback(cudaStream_t s, int n, int C, int layer, const double* cand, double* blo,
                      double* bhi, double* rlo, double* rhi, double* relax, int* gen_n,
                      int* gen_pos, int* gen_l, int g, long long gofs, long long pofs, int nimg,
                      long long zs, long long zp, int zl, long long kq) {
  Dirty dt{gen_n, gen_pos, gen_l, g, 0};
  dt.zs = zs;
  dt.zp = zp;
  dt.zl = zl;
  k_writeback<<<dim3(cdiv(n, 256), 1, nimg), 256, 0, s>>>(n, C, layer, cand, blo, bhi, rlo, rhi, relax,
                                                          dt, gofs, pofs, kq);
  ++g_launches;
}

// ===========================================================================
// Row initialisation (backsub.hpp:205-336)
// ===========================================================================

// init_affine_rows: the query neuron's own weights / filter taps as point
// coefficients over its predecessor; constant = bias (raw) and bias widened
// by dev[q] (padded).
__global__ void k_init_affine(LayerDev Q, RowsDev rows, FrameDev f, const double* dev_q,
                              MatDev out) {
  int i;
  if (!rows_resolve(rows, blockIdx.y, i)) return;
  bool upper;
  int img;
  const int q = row_query(rows, i, upper, img);
  dev_q += img * rows.sst;
  const long long cells = out.cells;
  double* lo = out.lo + (size_t)i * cells;
  double* hi = out.hi + (size_t)i * cells;
  MagAcc mag;
  if (Q.kind == KIND_DENSE) {
    const long long n_in = cells;
    for (long long t = blockIdx.x * blockDim.x + threadIdx.x; t < n_in;
         t += (long long)gridDim.x * blockDim.x) {
      const double w = Q.W[(size_t)q * n_in + t];
      lo[t] = w;
      hi[t] = w;
      mag.add(w);
    }
  } else {
    const int cq = q % Q.out_c;
    const int qw = (q / Q.out_c) % Q.out_w;
    const int qh = q / (Q.out_c * Q.out_w);
    int bw, bh;
    frame_base(f, q, bw, bh);
    const long long ow = (long long)qw * Q.sw - Q.pw, oh = (long long)qh * Q.sh - Q.ph;
    for (long long c = blockIdx.x * blockDim.x + threadIdx.x; c < cells;
         c += (long long)gridDim.x * blockDim.x) {
      const int ci = (int)(c % f.C);
      const int x = (int)((c / f.C) % f.S_w);
      const int y = (int)(c / ((long long)f.C * f.S_w));
      const long long fx = bw + x - ow, fy = bh + y - oh;
      double v = 0.0;
      if (fx >= 0 && fx < Q.fw && fy >= 0 && fy < Q.fh)
        v = Q.F[((size_t)(fy * Q.fw + fx) * Q.in_c + ci) * Q.out_c + cq];
      lo[c] = v;
      hi[c] = v;
      mag.add(v);
    }
  }
  mag.flush(out.stat);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const double b = Q.bias[Q.kind == KIND_DENSE ? q : q % Q.out_c];
    Iv k{b, b};
    const double dv = dev_q[q];
    if (dv != 0.0) k = Iv{add_down(k.lo, -dv), add_up(k.hi, dv)};  // widen_constant :175-179
    double* K = out.K + 4 * (size_t)i;
    K[0] = k.lo; K[1] = k.hi; K[2] = b; K[3] = b;
  }
}

void launch_init_affine(cudaStream_t s, const LayerDev& Q, const RowsDev& rows, const FrameDev& f,
                        const double* dev_q, MatDev out) {
  dim3 grid(cdiv(out.cells, 256) > 64 ? 64 : cdiv(out.cells, 256), rows.n);
  k_init_affine<<<grid, 256, 0, s>>>(Q, rows, f, dev_q, out);
  ++g_launches;
}

// init_identity_rows: coefficient 1 at the query neuron, constant 0.
__global__ void k_init_identity(RowsDev rows, FrameDev f, MatDev out) {
  int i;
  if (!rows_resolve(rows, blockIdx.y, i)) return;
  bool upper;
  const int q = row_query(rows, i, upper);
  const long long cells = out.cells;
  double* lo = out.lo + (size_t)i * cells;
  double* hi = out.hi + (size_t)i * cells;
  // Dense frame (1x1 grid): cell q; cuboid 1x1 window: cell = channel.
  const long long hot = (f.G_w == 1 && f.G_h == 1) ? q : q % f.C;
  MagAcc mag;
  for (long long c = blockIdx.x * blockDim.x + threadIdx.x; c < cells;
       c += (long long)gridDim.x * blockDim.x) {
    const double v = (c == hot) ? 1.0 : 0.0;
    lo[c] = v;
    hi[c] = v;
    mag.add(v);
  }
  mag.flush(out.stat);
  if (blockIdx.x == 0 && threadIdx.x < 4) out.K[4 * (size_t)i + threadIdx.x] = 0.0;
}

void launch_init_identity(cudaStream_t s, const RowsDev& rows, const FrameDev& f, MatDev out) {
  dim3 grid(cdiv(out.cells, 256) > 64 ? 64 : cdiv(out.cells, 256), rows.n);
  k_init_identity<<<grid, 256, 0, s>>>(rows, f, out);
  ++g_launches;
}

// init_margin_rows: +1 at label, -1 at class j, ascending j != label. Rows
// [first, first + gridDim.x) of the margin rows (a rank's slice when sharded).
// d_label (device-driven walks): the label is read from device memory.
__global__ void k_init_margin(int label, const int* d_label, int n_out, int first, MatDev out) {
  if (d_label) label = *d_label;
  const int r = blockIdx.x;
  const int g = first + r;
  const int j = g < label ? g : g + 1;
  MagAcc mag;
  for (int c = threadIdx.x; c < n_out; c += blockDim.x) {
    const double v = (c == label) ? 1.0 : (c == j ? -1.0 : 0.0);
    out.lo[(size_t)r * n_out + c] = v;
    out.hi[(size_t)r * n_out + c] = v;
    mag.add(v);
  }
  mag.flush(out.stat);
  if (threadIdx.x < 4) out.K[4 * r + threadIdx.x] = 0.0;
}

// The margin pass's query list: classes j != label, ascending (device label).
__global__ void k_margin_rows(const int* d_label, int n_out, int* row_q) {
  const int label = *d_label;
  for (int j = threadIdx.x; j < n_out; j += blockDim.x)
    if (j != label) row_q[j < label ? j : j - 1] = j;
}

void launch_margin_rows(cudaStream_t s, const int* d_label, int n_out, int* row_q) {
  k_margin_rows<<<1, 256, 0, s>>>(d_label, n_out, row_q);
  ++g_launches;
}

void launch_init_margin(cudaStream_t s, int label, const int* d_label, int n_out, int first,
                        int count, MatDev out) {
  if (count <= 0) return;
  k_init_margin<<<count, 128, 0, s>>>(label, d_label, n_out, first, out);
  ++g_launches;
}

// ===========================================================================
// Serial chains. One warp per row: the 32 lanes compute the terms of 32
// consecutive cells in parallel (products, zero skips), stage them in shared
// memory, then one lane per chain folds them into its accumulator in cell
// order. NaN marks a skipped term (real terms are never NaN).
// ===========================================================================

constexpr int kChainWarps = 4;

// Lane fold of one staged group of terms: acc (+)= t for non-NaN t.
template <bool FAST>
__device__ __forceinline__ double fold(double acc, double t, bool up) {
  if (FAST) {
    const double n = f_add_dir(acc, t, up);
    return (t == t) ? n : acc;
  }
  return (t == t) ? add_dir(acc, t, up) : acc;
}

// Constant update of a dense / conv substitution (backsub.hpp:365-389,
// 454-489): k += c*b_j and kraw += c*b_j (iv_acc, zero terms skipped),
// dev += mag(c)*dev_j (DevAccum), then widen_constant(k, dev). Lanes 0..4
// run k.lo, k.hi, kraw.lo, kraw.hi, dev. Also counts the step's multiply-adds
// (dense_madds :386 / gbc_madds :483).
template <bool FAST>
__device__ __forceinline__ bool chain_affine_row(const LayerDev& L, int is_conv, const FrameDev& f,
                                                 int bw, int bh, long long cells, const double* lo,
                                                 const double* hi, const double* dev, double acc,
                                                 double (*s_t)[32], int lane, double& out,
                                                 unsigned long long& madds) {
  const bool up = (lane & 1) || lane == 4;
  const int arr = lane == 4 ? 2 : (lane & 1);
  const int n_in = L.in_w * L.in_h * L.in_c;
  bool bad = FAST && lane < 5 && start_bad(acc);
  for (long long c0 = 0; c0 < cells; c0 += 32) {
    const long long cell = c0 + lane;
    double tl = PC_NAN, th = PC_NAN, td = PC_NAN;
    if (cell < cells) {
      const Iv c{lo[cell], hi[cell]};
      if (!iv_zero(c)) {
        double b;
        long long jd;
        if (is_conv) {
          const int d = (int)(cell % f.C);
          const int x = (int)((cell / f.C) % f.S_w);
          const int y = (int)(cell / ((long long)f.C * f.S_w));
          const int aw = bw + x, ah = bh + y;
          b = L.bias[d];
          jd = ((long long)ah * f.G_w + aw) * f.C + d;
          const int y0 = ah * L.sh - L.ph, x0 = aw * L.sw - L.pw;
          const int ny = min(L.fh, L.in_h - y0) - max(0, -y0);
          const int nx = min(L.fw, L.in_w - x0) - max(0, -x0);
          if (ny > 0 && nx > 0) madds += (unsigned long long)L.in_c * ny * nx;
        } else {
          b = L.bias[cell];
          jd = cell;
          madds += n_in;
        }
        const double dj = dev[jd];
        if (FAST) {
          const bool pos = b > 0.0;
          const double p1 = f_mul_dn(pos ? c.lo : c.hi, b, bad);
          const double p2 = f_mul_up(pos ? c.hi : c.lo, b, bad);
          if (b != 0.0) {
            tl = p1;
            th = p2;
          }
          const double pd = f_mul_up(iv_mag(c), dj, bad);
          if (dj != 0.0) td = pd;
        } else {
          const Iv bt = iv_mul_scalar(c, b);
          if (!iv_zero(bt)) {
            tl = bt.lo;
            th = bt.hi;
          }
          if (dj != 0.0) td = mul_up(iv_mag(c), dj);
        }
      }
    }
    // compact the contributing cells (ascending) so the fold skips the rest
    const bool v = (tl == tl) | (th == th) | (td == td);
    const unsigned mask = __ballot_sync(0xffffffffu, v);
    if (v) {
      const int p = __popc(mask & ((1u << lane) - 1u));
      s_t[0][p] = tl;
      s_t[1][p] = th;
      s_t[2][p] = td;
    }
    __syncwarp();
    if (lane < 5) {
      const int n = __popc(mask);
      for (int k = 0; k < n; ++k) acc = fold<FAST>(acc, s_t[arr][k], up);
    }
    __syncwarp();
  }
  out = acc;
  return __any_sync(0xffffffffu, bad);
}

__global__ void __launch_bounds__(32 * kChainWarps)
    k_chain_affine(LayerDev L, int is_conv, RowsDev rows, FrameDev f, MatDev m, double* Kout,
                   const double* dev, Counters* ctr, const char* frozen) {
  __shared__ double s_t[kChainWarps][3][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int i;
  if (!rows_resolve(rows, blockIdx.x * kChainWarps + warp, i)) return;
  bool upper;
  int img;
  const int q = row_query(rows, i, upper, img);
  if (frozen && frozen[(size_t)img * rows.kq + q]) return;
  dev += img * rows.sst;
  ctr += img;
  if (is_conv && lane == 0)
    atomicAdd(&ctr->gbc_dense_equiv, (unsigned long long)L.out_w * L.out_h * L.out_c *
                                         ((unsigned long long)L.in_w * L.in_h * L.in_c));
  int bw = 0, bh = 0;
  if (is_conv) frame_base(f, q, bw, bh);
  const long long cells = m.cells;
  const size_t pr = phys_row(m, i);
  const double* lo = m.lo + pr * cells;
  const double* hi = m.hi + pr * cells;
  const double acc0 = lane < 4 ? m.K[4 * pr + lane] : 0.0;
  double* K = Kout + 4 * (size_t)i;
  unsigned long long madds = 0;
  double acc;
  if (chain_affine_row<true>(L, is_conv, f, bw, bh, cells, lo, hi, dev, acc0, s_t[warp], lane, acc,
                             madds)) {
    madds = 0;
    chain_affine_row<false>(L, is_conv, f, bw, bh, cells, lo, hi, dev, acc0, s_t[warp], lane, acc,
                            madds);
  }
  const double dtot = __shfl_sync(0xffffffffu, acc, 4);
  if (lane == 0) K[0] = dtot != 0.0 ? add_down(acc, -dtot) : acc;
  if (lane == 1) K[1] = dtot != 0.0 ? add_up(acc, dtot) : acc;
  if (lane == 2 || lane == 3) K[lane] = acc;
  for (int o = 16; o > 0; o >>= 1) madds += __shfl_down_sync(0xffffffffu, madds, o);
  if (lane == 0 && madds) atomicAdd(is_conv ? &ctr->gbc_madds : &ctr->dense_madds, madds);
}

void launch_chain_affine(cudaStream_t s, const LayerDev& L, bool is_conv, const RowsDev& rows,
                         const FrameDev& fin, MatDev m, double* Kout, const double* dev,
                         Counters* ctr, const char* frozen, bool fast) {
  if (use_big_chains(m.cells, rows)) {
    launch_chain_affine_big(s, L, is_conv, rows, fin, m, Kout, dev, ctr, frozen, fast);
    return;
  }
  k_chain_affine<<<cdiv(rows.n, kChainWarps), 32 * kChainWarps, 0, s>>>(L, is_conv ? 1 : 0, rows,
                                                                        fin, m, Kout, dev, ctr, frozen);
  ++g_launches;
}

// Constant update of a relu substitution (backsub.hpp:536-563): per nonzero
// cell one offset term (sign-stable coefficient) or two (straddling: offp
// then offn), each skipped when zero. Lanes 0..3: k.lo, k.hi, kraw.lo, kraw.hi.
template <bool FAST>
__device__ __forceinline__ bool chain_relu_row(const FrameDev& f, int bw, int bh, bool upper,
                                               long long cells, const double* lo, const double* hi,
                                               const double* relax, double acc,
                                               double (*s_t)[2][32], int lane, double& out) {
  const bool up = lane & 1;
  const int arr = lane & 1;
  bool bad = FAST && lane < 4 && start_bad(acc);
  for (long long c0 = 0; c0 < cells; c0 += 32) {
    const long long cell = c0 + lane;
    double t0l = PC_NAN, t0h = PC_NAN, t1l = PC_NAN, t1h = PC_NAN;
    if (cell < cells) {
      const Iv c{lo[cell], hi[cell]};
      if (!iv_zero(c)) {
        const int cc = (int)(cell % f.C);
        const int x = (int)((cell / f.C) % f.S_w);
        const int y = (int)(cell / ((long long)f.C * f.S_w));
        const long long j = ((long long)(bh + y) * f.G_w + (bw + x)) * f.C + cc;
        const double* R = relax + 8 * j;
        const Iv beta{R[2], R[3]}, delta{R[6], R[7]};
        const Iv op = upper ? delta : beta;
        const Iv on = upper ? beta : delta;
        Iv o0{0.0, 0.0}, o1{0.0, 0.0};
        // stable neurons have zero offsets: every product is an exact zero
        if (iv_zero(op) && iv_zero(on)) {
        } else if (!(c.lo < 0.0)) o0 = FAST ? f_iv_mul(c, op, bad) : iv_mul(c, op);
        else if (!(c.hi > 0.0)) o0 = FAST ? f_iv_mul(c, on, bad) : iv_mul(c, on);
        else {
          o0 = FAST ? f_iv_mul(iv_pos_part(c), op, bad) : iv_mul(iv_pos_part(c), op);
          o1 = FAST ? f_iv_mul(iv_neg_part(c), on, bad) : iv_mul(iv_neg_part(c), on);
        }
        if (!iv_zero(o0)) { t0l = o0.lo; t0h = o0.hi; }
        if (!iv_zero(o1)) { t1l = o1.lo; t1h = o1.hi; }
      }
    }
    const bool v = (t0l == t0l) | (t0h == t0h) | (t1l == t1l) | (t1h == t1h);
    const unsigned mask = __ballot_sync(0xffffffffu, v);
    if (v) {
      const int p = __popc(mask & ((1u << lane) - 1u));
      s_t[0][0][p] = t0l;
      s_t[0][1][p] = t0h;
      s_t[1][0][p] = t1l;
      s_t[1][1][p] = t1h;
    }
    __syncwarp();
    if (lane < 4) {
      const int n = __popc(mask);
      for (int k = 0; k < n; ++k) {
        acc = fold<FAST>(acc, s_t[0][arr][k], up);
        acc = fold<FAST>(acc, s_t[1][arr][k], up);
      }
    }
    __syncwarp();
  }
  out = acc;
  return __any_sync(0xffffffffu, bad);
}

__global__ void __launch_bounds__(32 * kChainWarps)
    k_chain_relu(RowsDev rows, FrameDev f, MatDev m, double* Kout, const double* relax,
                 const char* frozen) {
  __shared__ double s_t[kChainWarps][2][2][32];  // [slot][lo/hi][cell]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int i;
  if (!rows_resolve(rows, blockIdx.x * kChainWarps + warp, i)) return;
  bool upper;
  int img;
  const int q = row_query(rows, i, upper, img);
  if (frozen && frozen[(size_t)img * rows.kq + q]) return;
  relax += 8 * img * rows.sst;
  int bw, bh;
  frame_base(f, q, bw, bh);
  const long long cells = m.cells;
  const size_t pr = phys_row(m, i);
  const double* lo = m.lo + pr * cells;
  const double* hi = m.hi + pr * cells;
  const double acc0 = lane < 4 ? m.K[4 * pr + lane] : 0.0;
  double* K = Kout + 4 * (size_t)i;
  double acc;
  if (chain_relu_row<true>(f, bw, bh, upper, cells, lo, hi, relax, acc0, s_t[warp], lane, acc))
    chain_relu_row<false>(f, bw, bh, upper, cells, lo, hi, relax, acc0, s_t[warp], lane, acc);
  if (lane < 4) K[lane] = acc;
}

void launch_chain_relu(cudaStream_t s, const RowsDev& rows, const FrameDev& f, MatDev m,
                       double* Kout, const double* relax, const char* frozen) {
  if (use_big_chains(m.cells, rows)) {
    launch_chain_relu_big(s, rows, f, m, Kout, relax, frozen);
    return;
  }
  k_chain_relu<<<cdiv(rows.n, kChainWarps), 32 * kChainWarps, 0, s>>>(rows, f, m, Kout, relax,
                                                                      frozen);
  ++g_launches;
}

// ---------------------------------------------------------------------------
// relu_step constants from the layer's offset list. Only neurons with a
// nonzero relaxation offset (beta or delta; the unstable ones,
// analyzer.hpp:56-66) add terms (backsub.hpp:536-563: stable neurons' offset
// products are exact zeros, skipped by iv_acc), so the chain visits the
// ascending list of those neurons (k_offset_list, built once per image when
// the layer's bounds are final) instead of scanning the row: same terms, same
// order. Warp per row; lanes 0..3 fold k.lo, k.hi, kraw.lo, kraw.hi.
__global__ void __launch_bounds__(1024)
    k_offset_list(int n, const double* relax, int* list, int* count, long long sst, int cstride) {
  using Scan = cub::BlockScan<int, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int s_base;
  const int img = blockIdx.z;
  relax += 8 * img * sst;
  list += img * sst;
  if (threadIdx.x == 0) s_base = 0;
  __syncthreads();
  for (int start = 0; start < n; start += 1024) {
    const int j = start + threadIdx.x;
    int has = 0;
    if (j < n) {
      const double* R = relax + 8 * (long long)j;
      has = !(bits_zero(R[2]) & bits_zero(R[3]) & bits_zero(R[6]) & bits_zero(R[7]));
    }
    int pos, total;
    Scan(tmp).ExclusiveSum(has, pos, total);
    if (has) list[s_base + pos] = j;
    __syncthreads();
    if (threadIdx.x == 0) s_base += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) count[img * cstride] = s_base;
}

void launch_offset_list(cudaStream_t s, int n, const double* relax, int* list, int* count,
                        int nimg, long long sst, int cstride) {
  k_offset_list<<<dim3(1, 1, nimg), 1024, 0, s>>>(n, relax, list, count, sst, cstride);
  ++g_launches;
}

__global__ void __launch_bounds__(32 * kChainWarps)
    k_chain_relu_list(RowsDev rows, FrameDev f, MatDev m, double* Kout, const double* relax,
                      const int* list, const int* count, int cstride, const char* frozen) {
  __shared__ double s_t[kChainWarps][2][2][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int i;
  if (!rows_resolve(rows, blockIdx.x * kChainWarps + warp, i)) return;
  bool upper;
  int img;
  const int q = row_query(rows, i, upper, img);
  if (frozen && frozen[(size_t)img * rows.kq + q]) return;
  relax += 8 * img * rows.sst;
  list += img * rows.sst;
  const int n = count[img * cstride];
  int bw, bh;
  frame_base(f, q, bw, bh);
  const size_t pr = phys_row(m, i);
  const double* lo = m.lo + pr * m.cells;
  const double* hi = m.hi + pr * m.cells;
  double acc = lane < 4 ? m.K[4 * pr + lane] : 0.0;
  const bool up = lane & 1;
  const int arr = lane & 1;
  const int GC = f.G_w * f.C;
  for (int e0 = 0; e0 < n; e0 += 32) {
    const int e = e0 + lane;
    double t0l = PC_NAN, t0h = PC_NAN, t1l = PC_NAN, t1h = PC_NAN;
    if (e < n) {
      const int j = list[e];
      const int ah = j / GC, rem = j - ah * GC;
      const int aw = rem / f.C, d = rem - aw * f.C;
      const int x = aw - bw, y = ah - bh;
      if (x >= 0 && x < f.S_w && y >= 0 && y < f.S_h) {
        const long long cell = ((long long)y * f.S_w + x) * f.C + d;
        const Iv c{lo[cell], hi[cell]};
        if (!iv_zero(c)) {
          const double* R = relax + 8 * (long long)j;
          const Iv beta{R[2], R[3]}, delta{R[6], R[7]};
          const Iv op = upper ? delta : beta;
          const Iv on = upper ? beta : delta;
          Iv o0{0.0, 0.0}, o1{0.0, 0.0};
          if (!(c.lo < 0.0)) o0 = iv_mul(c, op);
          else if (!(c.hi > 0.0)) o0 = iv_mul(c, on);
          else {
            o0 = iv_mul(iv_pos_part(c), op);
            o1 = iv_mul(iv_neg_part(c), on);
          }
          if (!iv_zero(o0)) { t0l = o0.lo; t0h = o0.hi; }
          if (!iv_zero(o1)) { t1l = o1.lo; t1h = o1.hi; }
        }
      }
    }
    const bool v = (t0l == t0l) | (t0h == t0h) | (t1l == t1l) | (t1h == t1h);
    const unsigned mask = __ballot_sync(0xffffffffu, v);
    if (v) {
      const int p = __popc(mask & ((1u << lane) - 1u));
      s_t[warp][0][0][p] = t0l;
      s_t[warp][0][1][p] = t0h;
      s_t[warp][1][0][p] = t1l;
      s_t[warp][1][1][p] = t1h;
    }
    __syncwarp();
    if (lane < 4) {
      const int k = __popc(mask);
      for (int u = 0; u < k; ++u) {
        const double a = s_t[warp][0][arr][u], b = s_t[warp][1][arr][u];
        if (a == a) acc = up ? add_up(acc, a) : add_down(acc, a);
        if (b == b) acc = up ? add_up(acc, b) : add_down(acc, b);
      }
    }
    __syncwarp();
  }
  if (lane < 4) Kout[4 * (size_t)i + lane] = acc;
}

void launch_chain_relu_list(cudaStream_t s, const RowsDev& rows, const FrameDev& f, MatDev m,
                            double* Kout, const double* relax, const int* list, const int* count,
                            int cstride, const char* frozen) {
  k_chain_relu_list<<<cdiv(rows.n, kChainWarps), 32 * kChainWarps, 0, s>>>(rows, f, m, Kout, relax, list,
                                                                           count, cstride, frozen);
  ++g_launches;
}

// concretize (backsub.hpp:725-764): acc = K.hi (upper) / K.lo (lower), then
// add the corner product with the frame layer's bounds for each nonzero
// cell in ascending order. Lane 0: padded track (constant, bounds); lane 1:
// raw track (constant_raw, raw bounds).
template <bool FAST>
__device__ __forceinline__ bool conc_row(const FrameDev& f, int bw, int bh, bool upper, bool skip0,
                                         long long cells, const double* lo, const double* hi,
                                         const double* blo, const double* bhi, const double* rlo,
                                         const double* rhi, double acc, double (*s_t)[32],
                                         int lane, double& out) {
  bool bad = FAST && lane < 2 && start_bad(acc);
  for (long long c0 = 0; c0 < cells; c0 += 32) {
    const long long cell = c0 + lane;
    double tp = PC_NAN, tr = PC_NAN;
    if (cell < cells) {
      const Iv c{lo[cell], hi[cell]};
      if (!iv_zero(c)) {
        const int cc = (int)(cell % f.C);
        const int x = (int)((cell / f.C) % f.S_w);
        const int y = (int)(cell / ((long long)f.C * f.S_w));
        const long long j = ((long long)(bh + y) * f.G_w + (bw + x)) * f.C + cc;
        const Iv B{blo[j], bhi[j]}, Br{rlo[j], rhi[j]};
        if (FAST) {
          tp = upper ? f_corner_hi(c, B, bad) : f_corner_lo(c, B, bad);
          tr = upper ? f_corner_hi(c, Br, bad) : f_corner_lo(c, Br, bad);
        } else {
          tp = upper ? corner_hi(c, B) : corner_lo(c, B);
          tr = upper ? corner_hi(c, Br) : corner_lo(c, Br);
        }
        // a +0 term leaves a non-(-0) accumulator unchanged: skip it
        if (skip0 && __double_as_longlong(tp) == 0) tp = PC_NAN;
        if (skip0 && __double_as_longlong(tr) == 0) tr = PC_NAN;
      }
    }
    const bool v = (tp == tp) | (tr == tr);
    const unsigned mask = __ballot_sync(0xffffffffu, v);
    if (v) {
      const int p = __popc(mask & ((1u << lane) - 1u));
      s_t[0][p] = tp;
      s_t[1][p] = tr;
    }
    __syncwarp();
    if (lane < 2) {
      const int n = __popc(mask);
      for (int k = 0; k < n; ++k) acc = fold<FAST>(acc, s_t[lane][k], upper);
    }
    __syncwarp();
  }
  out = acc;
  return __any_sync(0xffffffffu, bad);
}

__global__ void __launch_bounds__(32 * kChainWarps)
    k_concretize(RowsDev rows, FrameDev f, MatDev m, const double* blo, const double* bhi,
                 const double* rlo, const double* rhi, double* vals, double* rvals,
                 const char* frozen) {
  __shared__ double s_t[kChainWarps][2][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int i;
  if (!rows_resolve(rows, blockIdx.x * kChainWarps + warp, i)) return;
  bool upper;
  int img;
  const int q = row_query(rows, i, upper, img);
  if (frozen && frozen[(size_t)img * rows.kq + q]) return;
  blo += img * rows.sst;
  bhi += img * rows.sst;
  rlo += img * rows.sst;
  rhi += img * rows.sst;
  int bw, bh;
  frame_base(f, q, bw, bh);
  const long long cells = m.cells;
  const size_t pr = phys_row(m, i);
  const double* lo = m.lo + pr * cells;
  const double* hi = m.hi + pr * cells;
  const double* K = m.K + 4 * pr;
  double acc0 = 0.0;
  if (lane == 0) acc0 = upper ? K[1] : K[0];
  if (lane == 1) acc0 = upper ? K[3] : K[2];
  double acc;
  const double a0 = upper ? K[1] : K[0], a1 = upper ? K[3] : K[2];
  const long long nz = (long long)0x8000000000000000ULL;
  const bool skip0 = __double_as_longlong(a0) != nz && __double_as_longlong(a1) != nz;
  if (conc_row<true>(f, bw, bh, upper, skip0, cells, lo, hi, blo, bhi, rlo, rhi, acc0, s_t[warp], lane, acc))
    conc_row<false>(f, bw, bh, upper, skip0, cells, lo, hi, blo, bhi, rlo, rhi, acc0, s_t[warp], lane, acc);
  if (lane == 0) vals[i] = acc;
  if (lane == 1) rvals[i] = acc;
}

void launch_concretize(cudaStream_t s, const RowsDev& rows, const FrameDev& f, MatDev m,
                       const double* blo, const double* bhi, const double* rlo,
                       const double* rhi, double* vals, double* rvals, const char* frozen, bool fast) {
  if (use_big_chains(m.cells, rows)) {
    launch_concretize_big(s, rows, f, m, blo, bhi, rlo, rhi, vals, rvals, frozen, fast);
    return;
  }
  k_concretize<<<cdiv(rows.n, kChainWarps), 32 * kChainWarps, 0, s>>>(rows, f, m, blo, bhi, rlo,
                                                                      rhi, vals, rvals, frozen);
  ++g_launches;
}

// ===========================================================================
// Coefficient substitution kernels (output-stationary, reduction in the
// reference's ascending order, no split-K).
// ===========================================================================

// dense_step coefficients (backsub.hpp:365-386): M'[r][t] = sum_j M[r][j]*W[j][t]
// over ascending j, skipping zero coefficients and zero weights.
// Output-stationary: a block owns TM rows x 128 columns, each thread TM rows
// of one column (TM independent interval chains for ILP); the frame cells j
// (the reduction) stream through shared memory in ascending slabs. Fast
// branch-free ops; any output whose operands leave the fast band is
// recomputed with the exact ops.
constexpr int kDC = 128, kDK = 16;  // columns per block, frame cells per slab

// Executed interval madds of the dense kernels (rows x live columns x the
// nonzero cells walked), for the roofline report (dense_useful_madds()).
__device__ unsigned long long g_dense_useful;
unsigned long long dense_useful_madds(bool reset) {
  unsigned long long v = 0;
  cudaMemcpyFromSymbol(&v, g_dense_useful, sizeof(v));
  if (reset) {
    const unsigned long long z = 0;
    cudaMemcpyToSymbol(g_dense_useful, &z, sizeof(z));
  }
  return v;
}


__device__ __forceinline__ void madd_fast(double w, double clo, double chi, double& lo, double& hi,
                                          bool& bad) {
  const bool skip = (w == 0.0) | ((clo == 0.0) & (chi == 0.0));
  const bool pos = w > 0.0;
  const double a = pos ? clo : chi, b = pos ? chi : clo;
  const double pl = f_mul_dn(a, w, bad), ph = f_mul_up(b, w, bad);
  const double nl = f_add_dn(lo, pl), nh = f_add_up(hi, ph);
  lo = skip ? lo : nl;
  hi = skip ? hi : nh;
}

__device__ __forceinline__ void madd_exact(double w, double clo, double chi, double& lo,
                                           double& hi) {
  if (w == 0.0 || (clo == 0.0 && chi == 0.0)) return;
  const double a = w > 0.0 ? clo : chi, b = w > 0.0 ? chi : clo;
  lo = add_down(lo, mul_down(a, w));
  hi = add_up(hi, mul_up(b, w));
}

// Live output columns. When the frame after this step is a ReLU layer, the
// relu step maps the coefficient of every stably-negative neuron (relaxation
// alpha = gamma = 0, backsub.hpp:536-563, analyzer.hpp:50-55) to an exact
// zero whatever its value, its offsets add exact zeros, and the checkpoint
// between the two steps multiplies it by that neuron's relu bounds [0, 0]
// (concretize, backsub.hpp:756-759): the reference computes it, but no
// observable result depends on it as long as it is finite, which the band
// proof guarantees. Such columns are written as +0 and not computed. A block
// owns its column range for those zero writes and a kDC-slice of the
// ascending list of columns live in any of its rows for the arithmetic, so
// the warps stay dense. Without relax (frame not a ReLU, or out of band)
// every column is live and the list is the identity.
struct DenseCols {
  int col;    // this thread's output column (>= n_in: none)
  int count;  // live columns of this block
};

template <int TM, int NC = kDC>
__device__ DenseCols dense_live_cols(const RowsDev& rows, int nrows, int r0, int n_in,
                                     const double* relax, MatDev out, int* s_cols, int* s_warp) {
  const int tx = threadIdx.x, lane = tx & 31, wid = tx >> 5;
  const int x0 = blockIdx.x * NC;
  if (!relax) return DenseCols{x0 + tx, min(NC, n_in - x0)};
  const double* rx[TM];
#pragma unroll
  for (int u = 0; u < TM; ++u) {
    rx[u] = nullptr;
    if (r0 + u < nrows) {
      bool upper;
      int img;
      row_query(rows, r0 + u, upper, img);
      rx[u] = relax + 8 * (long long)img * rows.sst;
    }
  }
  int base = 0;
  for (int t0 = 0; t0 < n_in; t0 += NC) {
    const int t = t0 + tx;
    bool live = false;
    if (t < n_in) {
#pragma unroll
      for (int u = 0; u < TM; ++u) {
        if (!rx[u]) continue;
        const double* R = rx[u] + 8 * (long long)t;
        const bool dead = bits_zero(R[0]) & bits_zero(R[1]) & bits_zero(R[4]) & bits_zero(R[5]);
        live |= !dead;
      }
    }
    const unsigned b = __ballot_sync(0xFFFFFFFFu, live);
    __syncthreads();  // s_warp of the previous round consumed
    if (lane == 0) s_warp[wid] = __popc(b);
    __syncthreads();
    int before = base, total = 0;
#pragma unroll
    for (int w2 = 0; w2 < NC / 32; ++w2) {
      const int c = s_warp[w2];
      if (w2 < wid) before += c;
      total += c;
    }
    const int pos = before + __popc(b & ((1u << lane) - 1u));
    if (live && pos >= x0 && pos < x0 + NC) s_cols[pos - x0] = t;
    if (!live && t >= x0 && t < x0 + NC && t < n_in) {
#pragma unroll
      for (int u = 0; u < TM; ++u) {
        if (r0 + u >= nrows) continue;
        out.lo[(size_t)(r0 + u) * n_in + t] = 0.0;
        out.hi[(size_t)(r0 + u) * n_in + t] = 0.0;
      }
    }
    base += total;
  }
  __syncthreads();
  const int count = max(0, min(NC, base - x0));
  return DenseCols{tx < count ? s_cols[tx] : n_in, count};
}

template <int TM, bool BAND>
__device__ __forceinline__ void dense_slab(const double (*s_al)[kDK], const double (*s_ah)[kDK],
                                           const double* w, int kn, double* lo, double* hi,
                                           bool* bad, int& cells) {
  if constexpr (BAND && TM == 1) {
    // One row per thread: the add chain is the critical path. Form the slab's
    // outward-rounded products first (independent of the accumulators), then
    // run the two chains back to back.
    double pl[kDK], ph[kDK];
#pragma unroll
    for (int kk = 0; kk < kDK; ++kk) {
      const double wk = kk < kn ? w[kk] : 0.0;
      const bool neg = __double2hiint(wk) < 0;
      const double cl = s_al[0][kk], ch = s_ah[0][kk];
      const double a = neg ? ch : cl, b = neg ? cl : ch;
      const double p0 = __dmul_rn(a, wk), p1 = __dmul_rn(b, wk);
      pl[kk] = __dadd_rd(p0, -fabs(__fma_rn(a, wk, -p0)));
      ph[kk] = __dadd_ru(p1, fabs(__fma_rn(b, wk, -p1)));
    }
#pragma unroll
    for (int kk = 0; kk < kDK; ++kk) {
      // a zero row coefficient adds the zero interval (skipped by the
      // reference's iv_acc): block-uniform skip, shortens the chain
      if (bits_zero(s_al[0][kk]) && bits_zero(s_ah[0][kk])) continue;
      ++cells;
      const double sl = __dadd_rn(lo[0], pl[kk]), sh = __dadd_rn(hi[0], ph[kk]);
      const bool xl = __dadd_rd(lo[0], pl[kk]) == __dadd_ru(lo[0], pl[kk]);
      const bool xh = __dadd_rd(hi[0], ph[kk]) == __dadd_ru(hi[0], ph[kk]);
      const double tl = __dadd_rd(sl, -4.9406564584124654e-324);
      const double th = __dadd_ru(sh, 4.9406564584124654e-324);
      lo[0] = xl ? sl : tl;  // a zero product (kk >= kn) adds an exact +-0: no-op
      hi[0] = xh ? sh : th;
    }
  } else if constexpr (BAND) {
    // Several rows per thread: skip a cell only when it is zero in every row
    // (block-uniform; ReLU-dead cells are zero in all rows of an image), so
    // the TM madds of a cell form one branch-free block of 2*TM independent
    // chains. A zero cell inside a live group adds an exact +-0: a no-op up
    // to the sign of a zero lower bound, which canon0 restores.
#pragma unroll
    for (int kk = 0; kk < kDK; ++kk) {
      if (kk >= kn) break;
      double cl[TM], ch[TM];
      unsigned nz = 0u;
#pragma unroll
      for (int u = 0; u < TM; ++u) {
        cl[u] = s_al[u][kk];
        ch[u] = s_ah[u][kk];
        nz |= ((unsigned)__double2hiint(cl[u]) << 1) | (unsigned)__double2loint(cl[u]) |
              ((unsigned)__double2hiint(ch[u]) << 1) | (unsigned)__double2loint(ch[u]);
      }
      if (nz == 0u) continue;
      ++cells;
#pragma unroll
      for (int u = 0; u < TM; ++u) madd_band(w[kk], cl[u], ch[u], lo[u], hi[u]);
    }
  } else {
  cells += kn;
#pragma unroll
  for (int kk = 0; kk < kDK; ++kk) {
    if (kk >= kn) break;
#pragma unroll
    for (int u = 0; u < TM; ++u) {
      madd_fast(w[kk], s_al[u][kk], s_ah[u][kk], lo[u], hi[u], bad[u]);
    }
  }
  }
}

// Row slabs (shared by every column of the block) stream through a
// double buffer filled by cp.async one slab ahead; each thread's own weight
// column is prefetched into registers one slab ahead.
template <int TM>
struct DenseSmem {
  double al[2][TM][kDK], ah[2][TM][kDK];
};

template <int TM>
__device__ __forceinline__ void dense_stage(DenseSmem<TM>& sm, int b, int k0, int n_k, int r0,
                                            int nrows, const MatDev& in, int tx) {
  for (int e = tx; e < TM * kDK; e += kDC) {
    const int rr = e / kDK, kk = e % kDK;
    const int r = r0 + rr, k = k0 + kk;
    const bool ok = r < nrows && k < n_k;
    const size_t o = ok ? phys_row(in, r) * (size_t)n_k + k : 0;
    cp_async8(&sm.al[b][rr][kk], in.lo + o, ok);
    cp_async8(&sm.ah[b][rr][kk], in.hi + o, ok);
  }
  cp_async_commit();
}

__device__ __forceinline__ void dense_wload(double* w, const double* __restrict__ W, int k0, int n_k,
                                            int n_in, int col) {
#pragma unroll
  for (int kk = 0; kk < kDK; ++kk) {
    const int k = k0 + kk;
    w[kk] = (k < n_k && col < n_in) ? __ldg(W + (size_t)k * n_in + col) : 0.0;
  }
}

template <int TM>
__global__ void __launch_bounds__(kDC)
    k_dense_coef(const double* __restrict__ W, int n_k, int n_in, RowsDev rows, MatDev in,
                 MatDev out, double wmin, double wmax, const double* relax) {
  __shared__ DenseSmem<TM> sm;
  __shared__ int s_cols[kDC], s_warp[kDC / 32];
  const int tx = threadIdx.x;
  const int r0 = blockIdx.y * TM;
  int i0;
  rows_resolve(rows, 0, i0);  // live row count (physical rows 0..n-1 in order)
  const int nrows = rows.n;
  if (r0 >= nrows) return;
  const bool band = products_in_band(in.stat, wmin, wmax);
  const DenseCols dc = dense_live_cols<TM>(rows, nrows, r0, n_in, band ? relax : nullptr, out,
                                           s_cols, s_warp);
  if (dc.count <= 0) return;
  const int col = dc.col;
  double lo[TM], hi[TM];
  bool bad[TM];
#pragma unroll
  for (int u = 0; u < TM; ++u) {
    lo[u] = hi[u] = 0.0;
    bad[u] = false;
  }
  const int nslab = (n_k + kDK - 1) / kDK;
  int cells = 0;  // cells walked (block-uniform)
  double w[kDK], wn[kDK];
  dense_stage<TM>(sm, 0, 0, n_k, r0, nrows, in, tx);
  dense_wload(w, W, 0, n_k, n_in, col);
  for (int sl = 0; sl < nslab; ++sl) {
    cp_async_wait_all();
    __syncthreads();  // slab sl landed; slab sl-1 consumed
    if (sl + 1 < nslab) {
      dense_stage<TM>(sm, (sl + 1) & 1, (sl + 1) * kDK, n_k, r0, nrows, in, tx);
      dense_wload(wn, W, (sl + 1) * kDK, n_k, n_in, col);
    }
    const int b = sl & 1, kn = min(kDK, n_k - sl * kDK);
    if (band) dense_slab<TM, true>(sm.al[b], sm.ah[b], w, kn, lo, hi, bad, cells);
    else dense_slab<TM, false>(sm.al[b], sm.ah[b], w, kn, lo, hi, bad, cells);
#pragma unroll
    for (int kk = 0; kk < kDK; ++kk) w[kk] = wn[kk];
  }
  if (band) {
#pragma unroll
    for (int u = 0; u < TM; ++u) lo[u] = canon0(lo[u]);
  }
  if (tx == 0)
    atomicAdd(&g_dense_useful, (unsigned long long)cells * dc.count * min(TM, nrows - r0));
  if (col >= n_in) return;
  MagAcc mag;
#pragma unroll
  for (int u = 0; u < TM; ++u) {
    const int r = r0 + u;
    if (r >= nrows) continue;
    if (bad[u]) {
      lo[u] = hi[u] = 0.0;
      for (int k = 0; k < n_k; ++k)
        madd_exact(W[(size_t)k * n_in + col], in.lo[phys_row(in, r) * n_k + k],
                   in.hi[phys_row(in, r) * n_k + k], lo[u], hi[u]);
    }
    out.lo[(size_t)r * n_in + col] = lo[u];
    out.hi[(size_t)r * n_in + col] = hi[u];
    mag.add(lo[u]);
    mag.add(hi[u]);
  }
  mag.flush(out.stat);
}

// Many rows (image batches): TM rows x NC columns per block (the block's live
// columns, dense_live_cols), with the layer's weight slab staged in shared
// memory next to the row slab (2-stage cp.async ring, so no weight registers
// are held across slabs), and the cells of a slab that are zero in every row
// of the block dropped before the arithmetic: each warp ballots the slab's
// nonzero cells and walks them in ascending order in groups of kDG (then 2,
// then 1). A group is one branch-free block of G x TM independent products
// followed by the 2*TM accumulator chains.
#ifndef PC_DENSE2_DG
#define PC_DENSE2_DG 4
#endif
#ifndef PC_DENSE2_DK
#define PC_DENSE2_DK 16
#endif
#ifndef PC_DENSE2_STAGES
#define PC_DENSE2_STAGES 2
#endif
constexpr int kDG = PC_DENSE2_DG;   // cells per branch-free group
// cells per slab (<= 32: one ballot). 16 keeps a block at 37 KB of shared
// memory, so more of the other worker contexts' kernels stay co-resident:
// 5 % faster concurrent throughput than 32-cell slabs, which are 6 % faster
// for a lone launch (fewer barriers per cell)
constexpr int kDK2 = PC_DENSE2_DK;
#ifndef PC_DENSE2_MINB
#define PC_DENSE2_MINB 3  // resident blocks the register budget is sized for
#endif
constexpr int kDStages = PC_DENSE2_STAGES;

template <int TM, int NC>
struct DenseSmem2 {
  double2 c[kDStages][kDK2 + 1][TM];  // (lo, hi); cell kDK2 stays zero
  double w[kDStages][kDK2 + 1][NC];  // weight slab; cell kDK2 stays zero
};

template <int TM, int NC>
__device__ __forceinline__ void dense2_stage(DenseSmem2<TM, NC>& sm, int b, int k0, int n_k, int r0,
                                             int nrows, const MatDev& in,
                                             const double* __restrict__ W, int n_in, int col,
                                             int tx) {
  for (int e = tx; e < TM * kDK2; e += NC) {
    const int kk = e / TM, rr = e % TM;
    const int r = r0 + rr, k = k0 + kk;
    const bool ok = r < nrows && k < n_k;
    const size_t o = ok ? phys_row(in, r) * (size_t)n_k + k : 0;
    cp_async8(&sm.c[b][kk][rr].x, in.lo + o, ok);
    cp_async8(&sm.c[b][kk][rr].y, in.hi + o, ok);
  }
  // weight slab: this thread's column of rows k0.., one pointer step per cell
  const int kn = min(kDK2, n_k - k0);
  const double* p = W + (size_t)k0 * n_in + (col < n_in ? col : 0);
  const unsigned s0 = (unsigned)__cvta_generic_to_shared(&sm.w[b][0][tx]);
  if (col < n_in && kn == kDK2) {
#pragma unroll 8
    for (int kk = 0; kk < kDK2; ++kk, p += n_in)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s0 + kk * NC * 8), "l"(p));
  } else {
    for (int kk = 0; kk < kDK2; ++kk, p += n_in) {
      const bool ok = col < n_in && kk < kn;
      cp_async8(&sm.w[b][kk][tx], ok ? p : W, ok);
    }
  }
}

// G cells of a slab (the next G set bits of m, ascending) x TM rows: all
// products first (independent of the accumulators), then the 2*TM chains.
template <int G, int TM, int NC>
__device__ __forceinline__ void dense2_group(const DenseSmem2<TM, NC>& sm, int b, int tx,
                                             unsigned& m, double* lo, double* hi) {
  int ks[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    ks[g] = __ffs(m) - 1;
    m &= m - 1;
  }
  double pl[G][TM], ph[G][TM];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const double wk = sm.w[b][ks[g]][tx];
    // the factor of each bound is chosen by the weight's sign through the
    // load address, (lo, hi) -> (hi, lo), instead of by selects
    const int sa = __double2hiint(wk) < 0;
    const double* cg = &sm.c[b][ks[g]][0].x;
#pragma unroll
    for (int u = 0; u < TM; ++u)
      band_products_ab(wk, cg[2 * u + sa], cg[2 * u + 1 - sa], pl[g][u], ph[g][u]);
  }
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int u = 0; u < TM; ++u) band_sums(pl[g][u], ph[g][u], lo[u], hi[u]);
}

template <int TM, int NC>
__global__ void __launch_bounds__(NC, PC_DENSE2_MINB * (kDC / NC))
    k_dense_coef2(const double* __restrict__ W, int n_k, int n_in, RowsDev rows, MatDev in,
                  MatDev out, double wmin, double wmax, const double* relax) {
  extern __shared__ __align__(16) unsigned char dense2_raw[];
  DenseSmem2<TM, NC>& sm = *reinterpret_cast<DenseSmem2<TM, NC>*>(dense2_raw);
  __shared__ int s_cols[NC], s_warp[NC / 32];
  const int tx = threadIdx.x, lane = tx & 31;
  const int r0 = blockIdx.y * TM;
  int i0;
  rows_resolve(rows, 0, i0);
  const int nrows = rows.n;
  if (r0 >= nrows) return;
  const bool band = products_in_band(in.stat, wmin, wmax);
  const DenseCols dc = dense_live_cols<TM, NC>(rows, nrows, r0, n_in, band ? relax : nullptr, out,
                                           s_cols, s_warp);
  if (dc.count <= 0) return;
  const int col = dc.col;
  // warps with no live column skip the arithmetic (they still stage and sync)
  const bool warp_live = (tx & ~31) < dc.count;
  for (int b = 0; b < kDStages; ++b) {
    if (tx < TM) sm.c[b][kDK2][tx] = make_double2(0.0, 0.0);
    sm.w[b][kDK2][tx] = 0.0;
  }
  double lo[TM], hi[TM];
  bool bad[TM];
#pragma unroll
  for (int u = 0; u < TM; ++u) {
    lo[u] = hi[u] = 0.0;
    bad[u] = false;
  }
  const int nslab = (n_k + kDK2 - 1) / kDK2;
  int cells = 0;  // cells walked (warp-uniform; warp 0 reports)
#pragma unroll
  for (int p = 0; p < kDStages - 1; ++p) {
    if (p < nslab) dense2_stage<TM, NC>(sm, p, p * kDK2, n_k, r0, nrows, in, W, n_in, col, tx);
    cp_async_commit();
  }
  for (int sl = 0; sl < nslab; ++sl) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(kDStages - 2));
    __syncthreads();  // slab sl landed everywhere; slab sl-1's buffer is free
    if (sl + kDStages - 1 < nslab)
      dense2_stage<TM, NC>(sm, (sl + kDStages - 1) % kDStages, (sl + kDStages - 1) * kDK2, n_k, r0,
                       nrows, in, W, n_in, col, tx);
    cp_async_commit();
    const int b = sl % kDStages;
    if (!warp_live) continue;
    if (band) {
      // lane kk < kDK2: is cell kk nonzero in any row of the block?
      unsigned nz = 0u;
      if (lane < kDK2) {
#pragma unroll
        for (int u = 0; u < TM; ++u) {
          const double2 v = sm.c[b][lane][u];
          nz |= ((unsigned)__double2hiint(v.x) << 1) | (unsigned)__double2loint(v.x) |
                ((unsigned)__double2hiint(v.y) << 1) | (unsigned)__double2loint(v.y);
        }
      }
      unsigned m = __ballot_sync(0xFFFFFFFFu, nz != 0u);
      cells += __popc(m);
      // groups of kDG cells, then one of 2 and one of 1: no padding work
      int left = __popc(m);
      for (; left >= kDG; left -= kDG) dense2_group<kDG, TM, NC>(sm, b, tx, m, lo, hi);
      if (left >= 2) {
        dense2_group<2, TM, NC>(sm, b, tx, m, lo, hi);
        left -= 2;
      }
      if (left) dense2_group<1, TM, NC>(sm, b, tx, m, lo, hi);
    } else {
      const int kn = min(kDK2, n_k - sl * kDK2);
      cells += kn;
      for (int kk = 0; kk < kn; ++kk) {
        const double wk = sm.w[b][kk][tx];
#pragma unroll
        for (int u = 0; u < TM; ++u) {
          const double2 v = sm.c[b][kk][u];
          madd_fast(wk, v.x, v.y, lo[u], hi[u], bad[u]);
        }
      }
    }
  }
  if (band) {
#pragma unroll
    for (int u = 0; u < TM; ++u) lo[u] = canon0(lo[u]);
  }
  if (tx == 0)
    atomicAdd(&g_dense_useful, (unsigned long long)cells * dc.count * min(TM, nrows - r0));
  if (col >= n_in) return;
  MagAcc mag;
#pragma unroll
  for (int u = 0; u < TM; ++u) {
    const int r = r0 + u;
    if (r >= nrows) continue;
    if (bad[u]) {
      lo[u] = hi[u] = 0.0;
      for (int k = 0; k < n_k; ++k)
        madd_exact(W[(size_t)k * n_in + col], in.lo[phys_row(in, r) * n_k + k],
                   in.hi[phys_row(in, r) * n_k + k], lo[u], hi[u]);
    }
    out.lo[(size_t)r * n_in + col] = lo[u];
    out.hi[(size_t)r * n_in + col] = hi[u];
    mag.add(lo[u]);
    mag.add(hi[u]);
  }
  mag.flush(out.stat);
}

// v3 of the batched dense kernel: the union of the block rows' nonzero frame
// cells is listed once (ascending; block scan) in a prologue, and the slabs
// walk that list. Every staged weight row and every walked cell is then
// useful (no per-slab ballot, no partial groups but the last), and full slabs
// run with compile-time cell offsets. Frames longer than kDMaxList cells walk
// every cell (zero cells add exact +-0).
constexpr int kDMaxList = 2048;

template <int TM, int NC>
__device__ int dense3_cells(const RowsDev& rows, int nrows, int r0, int n_k, const MatDev& in,
                            int* s_cells, int* s_warp) {
  const int tx = threadIdx.x, lane = tx & 31, wid = tx >> 5;
  size_t pr[TM];
#pragma unroll
  for (int u = 0; u < TM; ++u) pr[u] = r0 + u < nrows ? phys_row(in, r0 + u) * (size_t)n_k : 0;
  int base = 0;
  for (int k0 = 0; k0 < n_k; k0 += NC) {
    const int k = k0 + tx;
    bool nz = false;
    if (k < n_k) {
#pragma unroll
      for (int u = 0; u < TM; ++u)
        if (r0 + u < nrows) nz |= !(bits_zero(in.lo[pr[u] + k]) && bits_zero(in.hi[pr[u] + k]));
    }
    const unsigned bal = __ballot_sync(0xFFFFFFFFu, nz);
    __syncthreads();  // s_warp of the previous round consumed
    if (lane == 0) s_warp[wid] = __popc(bal);
    __syncthreads();
    int before = base, total = 0;
#pragma unroll
    for (int w2 = 0; w2 < NC / 32; ++w2) {
      const int c = s_warp[w2];
      if (w2 < wid) before += c;
      total += c;
    }
    if (nz) s_cells[before + __popc(bal & ((1u << lane) - 1u))] = k;
    base += total;
  }
  __syncthreads();
  return base;
}

template <int TM, int NC>
__device__ __forceinline__ void dense3_stage(DenseSmem2<TM, NC>& sm, int b, int j0, int nnz,
                                             const int* s_cells, bool listed, int r0, int nrows,
                                             int n_k, const MatDev& in,
                                             const double* __restrict__ W, int n_in, int col,
                                             int tx) {
  for (int e = tx; e < TM * kDK2; e += NC) {
    const int kk = e / TM, rr = e % TM, idx = j0 + kk;
    const bool ok = idx < nnz && r0 + rr < nrows;
    const int cell = ok ? (listed ? s_cells[idx] : idx) : 0;
    const size_t o = ok ? phys_row(in, r0 + rr) * (size_t)n_k + cell : 0;
    cp_async8(&sm.c[b][kk][rr].x, in.lo + o, ok);
    cp_async8(&sm.c[b][kk][rr].y, in.hi + o, ok);
  }
  const unsigned s0 = (unsigned)__cvta_generic_to_shared(&sm.w[b][0][tx]);
  const bool colok = col < n_in;
#pragma unroll 4
  for (int kk = 0; kk < kDK2; ++kk) {
    const int idx = j0 + kk;
    const bool ok = colok && idx < nnz;
    const int row = ok ? (listed ? s_cells[idx] : idx) : 0;
    const double* p = W + (size_t)row * n_in + (colok ? col : 0);
    asm volatile(
        "{ .reg .pred q; setp.ne.b32 q, %2, 0;\n"
        "  @q cp.async.ca.shared.global [%0], [%1], 8;\n"
        "  @!q st.shared.f64 [%0], 0d0000000000000000; }\n" ::"r"(s0 + kk * NC * 8),
        "l"(p), "r"((int)ok));
  }
}

// G consecutive staged cells k0.. x TM rows: products first, then the chains.
template <int G, int TM, int NC>
__device__ __forceinline__ void dense3_group(const DenseSmem2<TM, NC>& sm, int b, int k0, int tx,
                                             double* lo, double* hi) {
  double pl[G][TM], ph[G][TM];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const double wk = sm.w[b][k0 + g][tx];
    const int sa = __double2hiint(wk) < 0;  // factor order by the weight's sign
    const double* cg = &sm.c[b][k0 + g][0].x;
#pragma unroll
    for (int u = 0; u < TM; ++u)
      band_products_ab(wk, cg[2 * u + sa], cg[2 * u + 1 - sa], pl[g][u], ph[g][u]);
  }
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int u = 0; u < TM; ++u) band_sums(pl[g][u], ph[g][u], lo[u], hi[u]);
}

template <int TM, int NC>
__global__ void __launch_bounds__(NC, PC_DENSE2_MINB * (kDC / NC))
    k_dense_coef3(const double* __restrict__ W, int n_k, int n_in, RowsDev rows, MatDev in,
                  MatDev out, double wmin, double wmax, const double* relax) {
  extern __shared__ __align__(16) unsigned char dense3_raw[];
  DenseSmem2<TM, NC>& sm = *reinterpret_cast<DenseSmem2<TM, NC>*>(dense3_raw);
  int* s_cells = reinterpret_cast<int*>(dense3_raw + sizeof(DenseSmem2<TM, NC>));
  __shared__ int s_cols[NC], s_warp[NC / 32];
  const int tx = threadIdx.x;
  const int r0 = blockIdx.y * TM;
  int i0;
  rows_resolve(rows, 0, i0);
  const int nrows = rows.n;
  if (r0 >= nrows) return;
  const bool band = products_in_band(in.stat, wmin, wmax);
  const DenseCols dc = dense_live_cols<TM, NC>(rows, nrows, r0, n_in, band ? relax : nullptr, out,
                                               s_cols, s_warp);
  if (dc.count <= 0) return;
  const int col = dc.col;
  const bool warp_live = (tx & ~31) < dc.count;
  const bool listed = n_k <= kDMaxList;
  const int nnz = listed ? dense3_cells<TM, NC>(rows, nrows, r0, n_k, in, s_cells, s_warp) : n_k;
  double lo[TM], hi[TM];
  bool bad[TM];
#pragma unroll
  for (int u = 0; u < TM; ++u) {
    lo[u] = hi[u] = 0.0;
    bad[u] = false;
  }
  const int nslab = (nnz + kDK2 - 1) / kDK2;
#pragma unroll
  for (int p = 0; p < kDStages - 1; ++p) {
    if (p < nslab)
      dense3_stage<TM, NC>(sm, p, p * kDK2, nnz, s_cells, listed, r0, nrows, n_k, in, W, n_in, col,
                           tx);
    cp_async_commit();
  }
  for (int sl = 0; sl < nslab; ++sl) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(kDStages - 2));
    __syncthreads();  // slab sl landed everywhere; slab sl-1's buffer is free
    if (sl + kDStages - 1 < nslab)
      dense3_stage<TM, NC>(sm, (sl + kDStages - 1) % kDStages, (sl + kDStages - 1) * kDK2, nnz,
                           s_cells, listed, r0, nrows, n_k, in, W, n_in, col, tx);
    cp_async_commit();
    if (!warp_live) continue;
    const int b = sl % kDStages;
    const int n = min(kDK2, nnz - sl * kDK2);
    if (band) {
      if (n == kDK2) {
#pragma unroll
        for (int g = 0; g < kDK2; g += kDG) dense3_group<kDG, TM, NC>(sm, b, g, tx, lo, hi);
      } else {
        int k0 = 0;
        for (; n - k0 >= kDG; k0 += kDG) dense3_group<kDG, TM, NC>(sm, b, k0, tx, lo, hi);
        if (n - k0 >= 2) {
          dense3_group<2, TM, NC>(sm, b, k0, tx, lo, hi);
          k0 += 2;
        }
        if (n - k0) dense3_group<1, TM, NC>(sm, b, k0, tx, lo, hi);
      }
    } else {
      for (int kk = 0; kk < n; ++kk) {
        const double wk = sm.w[b][kk][tx];
#pragma unroll
        for (int u = 0; u < TM; ++u) {
          const double2 v = sm.c[b][kk][u];
          madd_fast(wk, v.x, v.y, lo[u], hi[u], bad[u]);
        }
      }
    }
  }
  if (band) {
#pragma unroll
    for (int u = 0; u < TM; ++u) lo[u] = canon0(lo[u]);
  }
  if (tx == 0)
    atomicAdd(&g_dense_useful, (unsigned long long)nnz * dc.count * min(TM, nrows - r0));
  if (col >= n_in) return;
  MagAcc mag;
#pragma unroll
  for (int u = 0; u < TM; ++u) {
    const int r = r0 + u;
    if (r >= nrows) continue;
    if (bad[u]) {
      lo[u] = hi[u] = 0.0;
      for (int k = 0; k < n_k; ++k)
        madd_exact(W[(size_t)k * n_in + col], in.lo[phys_row(in, r) * n_k + k],
                   in.hi[phys_row(in, r) * n_k + k], lo[u], hi[u]);
    }
    out.lo[(size_t)r * n_in + col] = lo[u];
    out.hi[(size_t)r * n_in + col] = hi[u];
    mag.add(lo[u]);
    mag.add(hi[u]);
  }
  mag.flush(out.stat);
}

// Rows per thread (PC_DENSE_TM; default 4 above 64 rows). PC_DENSE_TM=-1
// picks per launch by a wave model: a launch is one wave set of equal tiles
// (every thread runs the whole n_k chain, so tiles cannot be split along k),
// cost = waves x TM x per-row cost, waves = ceil(tiles / resident tiles) from
// the occupancy queried at init. It wins for a lone stream and loses with
// several worker contexts, whose launches fill each other's last waves.
static int g_dense_tm = 4;
static int g_dense_slots[9] = {0};  // resident blocks per GPU, per TM

static int g_dense_v2 = 1;    // PC_DENSE_V2: staged-weight kernel for TM > 1
static int g_dense_v3 = 1;    // PC_DENSE_V3: listed-cell kernel (default)
static int g_dense_live = 1;  // PC_DENSE_LIVE: skip columns of stably-negative ReLU inputs

template <int TM>
static void dense_launch(cudaStream_t s, const LayerDev& L, const RowsDev& rows, MatDev in,
                         MatDev out, int n_k, int n_in, const double* relax) {
  if constexpr (TM > 1) {
    if (g_dense_v3) {
      constexpr int NC = TM >= 8 ? 64 : kDC;
      dim3 grid(cdiv(n_in, NC), cdiv(rows.n, TM));
      const size_t sm = sizeof(DenseSmem2<TM, NC>) + 4 * (size_t)std::min(n_k, kDMaxList);
      k_dense_coef3<TM, NC><<<grid, NC, sm, s>>>(L.W, n_k, n_in, rows, in, out, L.wmin, L.wmax,
                                                  relax);
      return;
    }
    if (g_dense_v2) {
      // TM = 8: half-width blocks, so the launch keeps as many blocks as TM = 4
      constexpr int NC = TM >= 8 ? 64 : kDC;
      dim3 grid(cdiv(n_in, NC), cdiv(rows.n, TM));
      k_dense_coef2<TM, NC><<<grid, NC, sizeof(DenseSmem2<TM, NC>), s>>>(
          L.W, n_k, n_in, rows, in, out, L.wmin, L.wmax, relax);
      return;
    }
  }
  dim3 grid(cdiv(n_in, kDC), cdiv(rows.n, TM));
  k_dense_coef<TM><<<grid, kDC, 0, s>>>(L.W, n_k, n_in, rows, in, out, L.wmin, L.wmax, relax);
}

static int dense_tm(int nrows, int n_in) {
  // Few rows: one row per thread maximises parallelism (the chain length
  // n_k bounds latency).
  if (nrows <= 64) return 1;
  if (g_dense_tm) return g_dense_tm;
  static const int cand[3] = {4, 3, 2};
  static const double cost[9] = {0, 0, 1.08, 1.0, 1.0, 0, 0, 0, 1.0};  // per-row, relative
  const long long cols = cdiv(n_in, kDC);
  int best = 4;
  double best_t = 1e300;
  for (int TM : cand) {
    const long long tiles = cols * cdiv(nrows, TM);
    const long long slots = g_dense_slots[TM] > 0 ? g_dense_slots[TM] : 444;
    const double t = (double)cdiv(tiles, slots) * TM * cost[TM];
    if (t < best_t - 1e-9) best_t = t, best = TM;
  }
  return best;
}

void launch_dense_coef(cudaStream_t s, const LayerDev& L, const RowsDev& rows, MatDev in,
                       MatDev out, const double* relax, cudaEvent_t ev0, cudaEvent_t ev1) {
  if (!g_dense_live) relax = nullptr;
  const int nrows = rows.n;
  const int n_k = (int)in.cells, n_in = (int)out.cells;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (ev0 || ev1) cudaStreamIsCapturing(s, &cap);
  const unsigned rf = cap == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : 0;
  if (ev0) cudaEventRecordWithFlags(ev0, s, rf);  // external: timeable inside graphs
  switch (dense_tm(nrows, n_in)) {
    case 1: dense_launch<1>(s, L, rows, in, out, n_k, n_in, relax); break;
    case 2: dense_launch<2>(s, L, rows, in, out, n_k, n_in, relax); break;
    case 3: dense_launch<3>(s, L, rows, in, out, n_k, n_in, relax); break;
    case 8: dense_launch<8>(s, L, rows, in, out, n_k, n_in, relax); break;
    default: dense_launch<4>(s, L, rows, in, out, n_k, n_in, relax); break;
  }
  if (ev1) cudaEventRecordWithFlags(ev1, s, rf);
  ++g_launches;
}

// gbc_step coefficients (backsub.hpp:449-485), gather form: each output cell
// (iy, ix, ci) of the new window sums, over the frame cells (ah, aw) whose
// filter window covers it in ascending (ah, aw) order and over ascending
// output channel d, c[ah][aw][d] * filter[fy][fx][ci][d]. That is exactly
// the reference's accumulation order for that coefficient (its scatter loop
// visits frame cells in (ch, cw, d) order).
__device__ __forceinline__ int floordiv(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

// MODE 2: band multiply-add (products proven in band for the launch);
// 1: fast ops with per-product band checks (bad -> recompute with 0);
// 0: the exact ops.
template <int MODE>
__device__ __forceinline__ Iv gbc_gather(const LayerDev& L, const FrameDev& fi, int bw, int bh,
                                         const double* ilo, const double* ihi, int iy, int ix,
                                         int ci, bool& bad) {
  const int cin = L.in_c, cout = L.out_c;
  int ah0 = floordiv(iy + L.ph - L.fh, L.sh) + 1, ah1 = floordiv(iy + L.ph, L.sh);
  int aw0 = floordiv(ix + L.pw - L.fw, L.sw) + 1, aw1 = floordiv(ix + L.pw, L.sw);
  ah0 = max(ah0, bh);
  ah1 = min(ah1, bh + fi.S_h - 1);
  aw0 = max(aw0, bw);
  aw1 = min(aw1, bw + fi.S_w - 1);
  double lo = 0.0, hi = 0.0;
  for (int ah = ah0; ah <= ah1; ++ah) {
    const int fy = iy + L.ph - ah * L.sh;
    for (int aw = aw0; aw <= aw1; ++aw) {
      const int fx = ix + L.pw - aw * L.sw;
      const size_t cb = ((size_t)(ah - bh) * fi.S_w + (aw - bw)) * cout;
      const double* wp = L.FT + ((size_t)(fy * L.fw + fx) * cout) * cin + ci;
      if (MODE > 0) {
        // A zero coefficient adds the zero interval (skipped by the reference's
        // iv_acc). Lanes of a warp share (iy, ix) when cin >= 32, so this
        // branch is warp-uniform and skips the work. Operands are loaded in
        // batches of kGB independent loads so their latency overlaps.
        constexpr int kGB = 8;
        int d = 0;
        for (; d + kGB <= cout; d += kGB) {
          double cl[kGB], ch[kGB], w[kGB];
#pragma unroll
          for (int k = 0; k < kGB; ++k) {
            cl[k] = ilo[cb + d + k];
            ch[k] = ihi[cb + d + k];
            w[k] = wp[(size_t)(d + k) * cin];
          }
#pragma unroll
          for (int k = 0; k < kGB; ++k) {
            if (cl[k] == 0.0 && ch[k] == 0.0) continue;
            if (MODE == 2) madd_band(w[k], cl[k], ch[k], lo, hi);
            else madd_fast(w[k], cl[k], ch[k], lo, hi, bad);
          }
        }
        for (; d < cout; ++d) {
          const double cl = ilo[cb + d], ch = ihi[cb + d];
          if (cl == 0.0 && ch == 0.0) continue;
          if (MODE == 2) madd_band(wp[(size_t)d * cin], cl, ch, lo, hi);
          else madd_fast(wp[(size_t)d * cin], cl, ch, lo, hi, bad);
        }
      } else {
        for (int d = 0; d < cout; ++d) madd_exact(wp[(size_t)d * cin], ilo[cb + d], ihi[cb + d], lo, hi);
      }
    }
  }
  return Iv{lo, hi};
}

// The checked gather out of line (keeps the band loop's register budget).
static __device__ __noinline__ Iv gbc_gather_checked(const LayerDev& L, const FrameDev& fi, int bw, int bh,
                                                     const double* ilo, const double* ihi, int iy, int ix,
                                                     int ci) {
  bool bad = false;
  Iv acc = gbc_gather<1>(L, fi, bw, bh, ilo, ihi, iy, ix, ci, bad);
  if (bad) acc = gbc_gather<0>(L, fi, bw, bh, ilo, ihi, iy, ix, ci, bad);
  return acc;
}


__global__ void __launch_bounds__(256)
    k_gbc_coef(LayerDev L, RowsDev rows, FrameDev fi, FrameDev fo, MatDev in, MatDev out) {
  int i;
  if (!rows_resolve(rows, blockIdx.y, i)) return;
  bool upper;
  const int q = row_query(rows, i, upper);
  int bw, bh, nbw, nbh;
  frame_base(fi, q, bw, bh);
  frame_base(fo, q, nbw, nbh);
  const long long ocells = out.cells, icells = in.cells;
  const double* ilo = in.lo + phys_row(in, i) * icells;
  const double* ihi = in.hi + phys_row(in, i) * icells;
  const int cin = L.in_c;
  const bool band = products_in_band(in.stat, L.wmin, L.wmax);
  MagAcc mag;
  for (long long o = blockIdx.x * blockDim.x + threadIdx.x; o < ocells;
       o += (long long)gridDim.x * blockDim.x) {
    const int ci = (int)(o % cin);
    const int x = (int)((o / cin) % fo.S_w);
    const int y = (int)(o / ((long long)cin * fo.S_w));
    const int iy = nbh + y, ix = nbw + x;
    bool bad = false;
    Iv acc;
    if (band) {
      acc = gbc_gather<2>(L, fi, bw, bh, ilo, ihi, iy, ix, ci, bad);
      acc.lo = canon0(acc.lo);
    } else {
      acc = gbc_gather<1>(L, fi, bw, bh, ilo, ihi, iy, ix, ci, bad);
      if (bad) acc = gbc_gather<0>(L, fi, bw, bh, ilo, ihi, iy, ix, ci, bad);
    }
    out.lo[(size_t)i * ocells + o] = acc.lo;
    out.hi[(size_t)i * ocells + o] = acc.hi;
    mag.add(acc.lo);
    mag.add(acc.hi);
  }
  mag.flush(out.stat);
}

// ---------------------------------------------------------------------------
// Shared-memory tiled gbc_step coefficients (band path). A CTA owns 64 output
// positions (flattened over the row's output window) x 64 input channels of
// one row. The reduction runs tap by tap in the canonical order (fy, fx
// descending = covering cells (ah, aw) ascending for every output) and, within
// a tap, over d in chunks of 32 ascending: exactly each output's reference
// order. Per stage, the 64 positions' covering coefficients c[ah][aw][d-chunk]
// ({lo, hi} pairs, zero when the tap misses the position or the window) and
// the tap's weights W[d-chunk][64 ci] are staged by cp.async into a double
// buffer while the previous stage computes. Warp w owns positions 8w..8w+7,
// lane l channels 2l, 2l+1: coefficient reads are warp-broadcasts, and a zero
// coefficient (a no-op, as in the reference's iv_acc skip) is skipped
// warp-uniformly. Operands outside the proven band fall back to the per-output
// gather with the checked / exact ops.
constexpr int kSC = 64, kSD = 32, kSW = 4;  // ci per CTA, d per stage, warps per CTA

template <int PW>
constexpr size_t gbc_smem_bytes() {  // double buffer of C [4*PW][kSD] {lo,hi} + W [kSD][kSC]
  return 2 * (size_t)(kSW * PW * kSD * 2 + kSD * kSC) * sizeof(double);
}

struct GbcSmemGeom {
  int n_pos, pos_tiles, ci_tiles;
};


// PW positions per warp (CTA: kSW warps = kSW*PW positions x kSC channels;
// lane l owns channels 2l, 2l+1 of the CTA's 64). Work items (row, position
// tile, channel tile) are taken from an atomic queue by a grid sized to the
// resident capacity, so rows whose coefficients are mostly zero (fast items)
// do not leave SMs idle.
template <int PW>
__device__ __forceinline__ void gbc_smem_item(const LayerDev& L, RowsDev rows, const FrameDev& fi,
                                              const FrameDev& fo, const MatDev& in,
                                              const MatDev& out, const GbcSmemGeom& g, int item,
                                              double* sm, MagAcc& mag) {
  constexpr int kSP = kSW * PW;
  constexpr int kCWords = kSP * kSD * 2, kWWords = kSD * kSC, kBuf = kCWords + kWWords;
  const int tiles = g.pos_tiles * g.ci_tiles;
  int i;
  if (!rows_resolve(rows, item / tiles, i)) return;
  const int t = item % tiles;
  const int pt = t % g.pos_tiles, ct = t / g.pos_tiles;
  const int p0 = pt * kSP, ci0 = ct * kSC;
  bool upper;
  const int q = row_query(rows, i, upper);
  int bw, bh, nbw, nbh;
  frame_base(fi, q, bw, bh);
  frame_base(fo, q, nbw, nbh);
  const double* ilo = in.lo + phys_row(in, i) * in.cells;
  const double* ihi = in.hi + phys_row(in, i) * in.cells;
  const int cin = L.in_c, cout = L.out_c;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool band = products_in_band(in.stat, L.wmin, L.wmax);
  double* olo = out.lo + (size_t)i * out.cells;
  double* ohi = out.hi + (size_t)i * out.cells;
  if (!band) {  // checked fast ops, exact recompute on a flagged output
    for (int e = tid; e < kSP * kSC; e += blockDim.x) {
      const int p = p0 + e / kSC, ci = ci0 + e % kSC;
      if (p >= g.n_pos || ci >= cin) continue;
      const int iy = nbh + p / fo.S_w, ix = nbw + p % fo.S_w;
      bool bad = false;
      Iv acc = gbc_gather<1>(L, fi, bw, bh, ilo, ihi, iy, ix, ci, bad);
      if (bad) acc = gbc_gather<0>(L, fi, bw, bh, ilo, ihi, iy, ix, ci, bad);
      const size_t o = (size_t)p * cin + ci;
      olo[o] = acc.lo;
      ohi[o] = acc.hi;
      mag.add(acc.lo);
      mag.add(acc.hi);
    }
    return;
  }
  const int ntaps = L.fh * L.fw;
  const int nchunks = (cout + kSD - 1) / kSD;
  const int nstages = ntaps * nchunks;
  auto stage = [&](int st, int b) {
    const int tap = st / nchunks, d0 = (st % nchunks) * kSD;
    const int fy = L.fh - 1 - tap / L.fw, fx = L.fw - 1 - tap % L.fw;
    double* C = sm + (size_t)b * kBuf;
    double* Wd = C + kCWords;
    for (int e = tid; e < kSP * kSD; e += blockDim.x) {
      const int pp = e / kSD, dd = e % kSD;
      const int p = p0 + pp, d = d0 + dd;
      bool ok = p < g.n_pos && d < cout;
      size_t src = 0;
      if (ok) {
        const int iy = nbh + p / fo.S_w, ix = nbw + p % fo.S_w;
        const int ny = iy + L.ph - fy, nx = ix + L.pw - fx;  // = ah * sh, aw * sw
        ok = ny >= 0 && nx >= 0 && ny % L.sh == 0 && nx % L.sw == 0;
        if (ok) {
          const int ah = ny / L.sh - bh, aw = nx / L.sw - bw;
          ok = ah >= 0 && ah < fi.S_h && aw >= 0 && aw < fi.S_w;
          src = ((size_t)ah * fi.S_w + aw) * cout + d;
        }
      }
      cp_async8(C + 2 * e, ilo + (ok ? src : 0), ok);
      cp_async8(C + 2 * e + 1, ihi + (ok ? src : 0), ok);
    }
    const double* wt = L.FT + ((size_t)(fy * L.fw + fx) * cout) * cin;
    for (int e = tid; e < kSD * kSC; e += blockDim.x) {
      const int dd = e / kSC, cc = e % kSC;
      const bool ok = d0 + dd < cout && ci0 + cc < cin;
      cp_async8(Wd + e, wt + (ok ? (size_t)(d0 + dd) * cin + ci0 + cc : 0), ok);
    }
    cp_async_commit();
  };
  double lo[PW][2], hi[PW][2];
#pragma unroll
  for (int k = 0; k < PW; ++k)
#pragma unroll
    for (int j = 0; j < 2; ++j) lo[k][j] = hi[k][j] = 0.0;
  stage(0, 0);
  for (int st = 0; st < nstages; ++st) {
    cp_async_wait_all();
    __syncthreads();  // stage st landed; stage st-1 consumed
    if (st + 1 < nstages) stage(st + 1, (st + 1) & 1);
    const double* C = sm + (size_t)(st & 1) * kBuf;
    const double2* C2 = reinterpret_cast<const double2*>(C) + (size_t)(warp * PW) * kSD;
    const double2* W2 = reinterpret_cast<const double2*>(C + kCWords) + lane;
#pragma unroll 2
    for (int dd = 0; dd < kSD; ++dd) {
      const double2 w = W2[(size_t)dd * (kSC / 2)];
#pragma unroll
      for (int k = 0; k < PW; ++k) {
        const double2 c = C2[(size_t)k * kSD + dd];
        if (bits_zero(c.x) && bits_zero(c.y)) continue;
        madd_band(w.x, c.x, c.y, lo[k][0], hi[k][0]);
        madd_band(w.y, c.x, c.y, lo[k][1], hi[k][1]);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < PW; ++k) {
    const int p = p0 + warp * PW + k;
    if (p >= g.n_pos) break;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int ci = ci0 + 2 * lane + j;
      if (ci >= cin) continue;
      const double l = canon0(lo[k][j]);
      const size_t o = (size_t)p * cin + ci;
      olo[o] = l;
      ohi[o] = hi[k][j];
      mag.add(l);
      mag.add(hi[k][j]);
    }
  }
}

template <int PW>
__global__ void __launch_bounds__(32 * kSW)
    k_gbc_smem(LayerDev L, RowsDev rows, FrameDev fi, FrameDev fo, MatDev in, MatDev out,
               GbcSmemGeom g, int* queue, int n_items) {
  extern __shared__ double sm[];
  __shared__ int s_item;
  MagAcc mag;
  for (;;) {
    __syncthreads();  // the previous item is done with s_item and the buffers
    if (threadIdx.x == 0) s_item = atomicAdd(queue, 1);
    __syncthreads();
    const int item = s_item;
    if (item >= n_items) break;
    gbc_smem_item<PW>(L, rows, fi, fo, in, out, g, item, sm, mag);
  }
  mag.flush(out.stat);
}

static bool gbc_smem_eligible(const LayerDev& L, const FrameDev& fout) {
  static const int any = env_int("PC_GBC_SMEM_ANY", 0);  // tests: route every conv step here
  return any || (L.in_c >= 32 && (long long)fout.S_w * fout.S_h >= 32);
}

void launch_gbc_smem(cudaStream_t s, const LayerDev& L, const RowsDev& rows, const FrameDev& fin,
                     const FrameDev& fout, MatDev in, MatDev out, int* queue) {
  GbcSmemGeom g;
  g.n_pos = fout.S_w * fout.S_h;
  g.ci_tiles = (L.in_c + kSC - 1) / kSC;
  // positions per warp: the most reuse that still gives >= 4 items per SM
  static const int forced = env_int("PC_GBC_PW", 0);
  int pw = forced;
  if (!pw) {
    pw = 1;
    for (int c : {8, 4, 2}) {
      const long long items = (long long)((g.n_pos + kSW * c - 1) / (kSW * c)) * g.ci_tiles * rows.n;
      if (items >= 4 * 148) { pw = c; break; }
    }
  }
  g.pos_tiles = (g.n_pos + kSW * pw - 1) / (kSW * pw);
  const long long items = (long long)g.pos_tiles * g.ci_tiles * rows.n;
  // resident CTAs per SM for this variant (registers / shared memory), once
  static int occ[9] = {0};
  if (!occ[pw]) {
    int b = 1;
    switch (pw) {
      case 8: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_gbc_smem<8>, 32 * kSW, gbc_smem_bytes<8>()); break;
      case 4: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_gbc_smem<4>, 32 * kSW, gbc_smem_bytes<4>()); break;
      case 2: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_gbc_smem<2>, 32 * kSW, gbc_smem_bytes<2>()); break;
      default: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_gbc_smem<1>, 32 * kSW, gbc_smem_bytes<1>()); break;
    }
    occ[pw] = b > 0 ? b : 1;
  }
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const unsigned grid = (unsigned)std::min<long long>(items, (long long)sms * occ[pw]);
  cudaMemsetAsync(queue, 0, sizeof(int), s);
  const int n_items = (int)items;
  switch (pw) {
    case 8: k_gbc_smem<8><<<grid, 32 * kSW, gbc_smem_bytes<8>(), s>>>(L, rows, fin, fout, in, out, g, queue, n_items); break;
    case 4: k_gbc_smem<4><<<grid, 32 * kSW, gbc_smem_bytes<4>(), s>>>(L, rows, fin, fout, in, out, g, queue, n_items); break;
    case 2: k_gbc_smem<2><<<grid, 32 * kSW, gbc_smem_bytes<2>(), s>>>(L, rows, fin, fout, in, out, g, queue, n_items); break;
    default: k_gbc_smem<1><<<grid, 32 * kSW, gbc_smem_bytes<1>(), s>>>(L, rows, fin, fout, in, out, g, queue, n_items); break;
  }
  ++g_launches;
}

// ---------------------------------------------------------------------------
// Sparse conv back-substitution. About two thirds of a conv step's input
// coefficients are zero on the ResNets (relu steps zero the stable-negative
// neurons), and zero coefficients contribute nothing (the reference skips
// them in iv_acc). k_compact_cells packs each frame cell's nonzero channels
// (ascending, with their index) once; k_gbc_sparse then gathers only those,
// in the reference's (ch, cw, d) order, without per-channel zero tests.

__global__ void __launch_bounds__(256)
    k_compact_cells(RowsDev rows, MatDev m, SparseDev sp) {
  __shared__ unsigned s_mask[16];  // nonzero channels of this block's cells (sp.dmask)
  int i;
  if (!rows_resolve(rows, blockIdx.y, i)) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int C = sp.C;
  if (threadIdx.x < 16) s_mask[threadIdx.x] = 0;
  __syncthreads();
  const double* lo = m.lo + phys_row(m, i) * m.cells;
  const double* hi = m.hi + phys_row(m, i) * m.cells;
  for (int cell = blockIdx.x * 8 + warp; cell < sp.ncell; cell += gridDim.x * 8) {
    const size_t slot = ((size_t)i * sp.ncell + cell) * C;
    int base = 0;
    for (int c0 = 0; c0 < C; c0 += 32) {
      const int c = c0 + lane;
      double a = 0.0, b = 0.0;
      if (c < C) {
        a = lo[(size_t)cell * C + c];
        b = hi[(size_t)cell * C + c];
      }
      const bool nz = c < C && !(bits_zero(a) && bits_zero(b));
      const unsigned mask = __ballot_sync(0xffffffffu, nz);
      if (nz) {
        const int k = base + __popc(mask & ((1u << lane) - 1u));
        sp.idx[slot + k] = (unsigned short)c;
        sp.lo[slot + k] = a;
        sp.hi[slot + k] = b;
      }
      if (sp.dmask && lane == 0 && mask && c0 < 512) atomicOr(&s_mask[c0 >> 5], mask);
      base += __popc(mask);
    }
    if (lane == 0) sp.cnt[(size_t)i * sp.ncell + cell] = base;
  }
  __syncthreads();
  if (sp.dmask && threadIdx.x < 16 && s_mask[threadIdx.x])
    atomicOr(&sp.dmask[(size_t)i * 16 + threadIdx.x], s_mask[threadIdx.x]);
}

void launch_compact_cells(cudaStream_t s, const RowsDev& rows, MatDev m, SparseDev sp) {
  unsigned gx = cdiv(sp.ncell, 8);
  if (gx > 512) gx = 512;
  dim3 grid(gx, rows.n);
  k_compact_cells<<<grid, 256, 0, s>>>(rows, m, sp);
  ++g_launches;
}

__global__ void __launch_bounds__(256)
    k_gbc_sparse(LayerDev L, RowsDev rows, FrameDev fi, FrameDev fo, SparseDev sp, MatDev in,
                 MatDev out) {
  int i;
  if (!rows_resolve(rows, blockIdx.y, i)) return;
  bool upper;
  const int q = row_query(rows, i, upper);
  int bw, bh, nbw, nbh;
  frame_base(fi, q, bw, bh);
  frame_base(fo, q, nbw, nbh);
  const long long ocells = out.cells;
  const double* ilo = in.lo + phys_row(in, i) * in.cells;
  const double* ihi = in.hi + phys_row(in, i) * in.cells;
  const int cin = L.in_c, cout = L.out_c;
  const bool band = products_in_band(in.stat, L.wmin, L.wmax);
  const int* cnt = sp.cnt + (size_t)i * sp.ncell;
  const size_t rbase = (size_t)i * sp.ncell * sp.C;
  MagAcc mag;
  for (long long o = blockIdx.x * blockDim.x + threadIdx.x; o < ocells;
       o += (long long)gridDim.x * blockDim.x) {
    const int ci = (int)(o % cin);
    const int x = (int)((o / cin) % fo.S_w);
    const int y = (int)(o / ((long long)cin * fo.S_w));
    const int iy = nbh + y, ix = nbw + x;
    Iv acc;
    if (!band) {
      acc = gbc_gather_checked(L, fi, bw, bh, ilo, ihi, iy, ix, ci);
    } else {
      int ah0 = floordiv(iy + L.ph - L.fh, L.sh) + 1, ah1 = floordiv(iy + L.ph, L.sh);
      int aw0 = floordiv(ix + L.pw - L.fw, L.sw) + 1, aw1 = floordiv(ix + L.pw, L.sw);
      ah0 = max(ah0, bh);
      ah1 = min(ah1, bh + fi.S_h - 1);
      aw0 = max(aw0, bw);
      aw1 = min(aw1, bw + fi.S_w - 1);
      double lo = 0.0, hi = 0.0;
      for (int ah = ah0; ah <= ah1; ++ah) {
        const int fy = iy + L.ph - ah * L.sh;
        for (int aw = aw0; aw <= aw1; ++aw) {
          const int fx = ix + L.pw - aw * L.sw;
          const int cell = (ah - bh) * fi.S_w + (aw - bw);
          const int n = cnt[cell];
          const size_t sb = rbase + (size_t)cell * sp.C;
          const double* wp = L.FT + ((size_t)(fy * L.fw + fx) * cout) * cin + ci;
          constexpr int kB = 8;
          int e = 0;
          for (; e + kB <= n; e += kB) {
            double cl[kB], ch[kB], w[kB];
#pragma unroll
            for (int k = 0; k < kB; ++k) {
              const int d = sp.idx[sb + e + k];
              cl[k] = sp.lo[sb + e + k];
              ch[k] = sp.hi[sb + e + k];
              w[k] = wp[(size_t)d * cin];
            }
#pragma unroll
            for (int k = 0; k < kB; ++k) madd_band(w[k], cl[k], ch[k], lo, hi);
          }
          for (; e < n; ++e)
            madd_band(wp[(size_t)sp.idx[sb + e] * cin], sp.lo[sb + e], sp.hi[sb + e], lo, hi);
        }
      }
      acc = Iv{canon0(lo), hi};
    }
    out.lo[(size_t)i * ocells + o] = acc.lo;
    out.hi[(size_t)i * ocells + o] = acc.hi;
    mag.add(acc.lo);
    mag.add(acc.hi);
  }
  mag.flush(out.stat);
}

// Two adjacent input channels per thread (even cin, band path only): the
// compacted coefficient (index + interval) is loaded once for two madds and the
// weights as one 16-byte pair.
template <int MINB>
__global__ void __launch_bounds__(256, MINB)
    k_gbc_sparse2(LayerDev L, RowsDev rows, FrameDev fi, FrameDev fo, SparseDev sp, MatDev in,
                  MatDev out) {
  int i;
  if (!rows_resolve(rows, blockIdx.y, i)) return;
  bool upper;
  const int q = row_query(rows, i, upper);
  int bw, bh, nbw, nbh;
  frame_base(fi, q, bw, bh);
  frame_base(fo, q, nbw, nbh);
  const long long ocells = out.cells, opairs = ocells / 2;
  const double* ilo = in.lo + phys_row(in, i) * in.cells;
  const double* ihi = in.hi + phys_row(in, i) * in.cells;
  const int cin = L.in_c, cout = L.out_c, cin2 = cin / 2;
  const bool band = products_in_band(in.stat, L.wmin, L.wmax);
  const int* cnt = sp.cnt + (size_t)i * sp.ncell;
  const size_t rbase = (size_t)i * sp.ncell * sp.C;
  MagAcc mag;
  for (long long o2 = blockIdx.x * blockDim.x + threadIdx.x; o2 < opairs;
       o2 += (long long)gridDim.x * blockDim.x) {
    const int cp = (int)(o2 % cin2);
    const int x = (int)((o2 / cin2) % fo.S_w);
    const int y = (int)(o2 / ((long long)cin2 * fo.S_w));
    const int iy = nbh + y, ix = nbw + x, ci = 2 * cp;
    Iv acc0, acc1;
    if (!band) {
      bool bad = false;
      acc0 = gbc_gather<1>(L, fi, bw, bh, ilo, ihi, iy, ix, ci, bad);
      if (bad) acc0 = gbc_gather<0>(L, fi, bw, bh, ilo, ihi, iy, ix, ci, bad);
      bad = false;
      acc1 = gbc_gather<1>(L, fi, bw, bh, ilo, ihi, iy, ix, ci + 1, bad);
      if (bad) acc1 = gbc_gather<0>(L, fi, bw, bh, ilo, ihi, iy, ix, ci + 1, bad);
    } else {
      int ah0 = floordiv(iy + L.ph - L.fh, L.sh) + 1, ah1 = floordiv(iy + L.ph, L.sh);
      int aw0 = floordiv(ix + L.pw - L.fw, L.sw) + 1, aw1 = floordiv(ix + L.pw, L.sw);
      ah0 = max(ah0, bh);
      ah1 = min(ah1, bh + fi.S_h - 1);
      aw0 = max(aw0, bw);
      aw1 = min(aw1, bw + fi.S_w - 1);
      double lo0 = 0.0, hi0 = 0.0, lo1 = 0.0, hi1 = 0.0;
      for (int ah = ah0; ah <= ah1; ++ah) {
        const int fy = iy + L.ph - ah * L.sh;
        for (int aw = aw0; aw <= aw1; ++aw) {
          const int fx = ix + L.pw - aw * L.sw;
          const int cell = (ah - bh) * fi.S_w + (aw - bw);
          const int n = cnt[cell];
          const size_t sb = rbase + (size_t)cell * sp.C;
          const double2* wp =
              reinterpret_cast<const double2*>(L.FT + ((size_t)(fy * L.fw + fx) * cout) * cin) + cp;
          constexpr int kB = 4;
          int e = 0;
          for (; e + kB <= n; e += kB) {
            double cl[kB], ch[kB];
            double2 w[kB];
#pragma unroll
            for (int k = 0; k < kB; ++k) {
              const int d = sp.idx[sb + e + k];
              cl[k] = sp.lo[sb + e + k];
              ch[k] = sp.hi[sb + e + k];
              w[k] = wp[(size_t)d * cin2];
            }
#pragma unroll
            for (int k = 0; k < kB; ++k) {
              madd_band(w[k].x, cl[k], ch[k], lo0, hi0);
              madd_band(w[k].y, cl[k], ch[k], lo1, hi1);
            }
          }
          for (; e < n; ++e) {
            const double2 w = wp[(size_t)sp.idx[sb + e] * cin2];
            madd_band(w.x, sp.lo[sb + e], sp.hi[sb + e], lo0, hi0);
            madd_band(w.y, sp.lo[sb + e], sp.hi[sb + e], lo1, hi1);
          }
        }
      }
      acc0 = Iv{canon0(lo0), hi0};
      acc1 = Iv{canon0(lo1), hi1};
    }
    const size_t ob = (size_t)i * ocells + 2 * o2;
    out.lo[ob] = acc0.lo;
    out.hi[ob] = acc0.hi;
    out.lo[ob + 1] = acc1.lo;
    out.hi[ob + 1] = acc1.hi;
    mag.add(acc0.lo);
    mag.add(acc0.hi);
    mag.add(acc1.lo);
    mag.add(acc1.hi);
  }
  mag.flush(out.stat);
}

// ---------------------------------------------------------------------------
// Live output cells of a conv step whose frame lands on a ReLU layer P.
//
// The relu step that follows maps the coefficient of every stably-negative
// neuron of P (relaxation all zero, analyzer.hpp:50-55) to an exact zero
// whatever its value and adds no offset for it (backsub.hpp:536-563); the
// checkpoint in between multiplies it by P's padded and raw bounds, both
// [0, 0] for such a neuron, i.e. adds +0 terms (concretize, :756-759), which
// change nothing unless the accumulator is -0 (never, unless a bias is -0:
// the engine then keeps every cell live). In a residual join the branch
// result is added to the other branch before that checkpoint and relu step,
// so the sum at such a cell is just as irrelevant. So these cells (about 60 %
// of the coefficients on the ResNets) are written as +0 and not computed; no
// observable value — bounds, margins, PassStats — depends on them.
//
// k_live_build lists, once per image when P's bounds are final (right after
// its forward refresh), the live channels of every grid position of P:
// cnt[pos], idx[pos * C + k] ascending. Dead = relaxation all zero and P's
// padded and raw bounds exactly zero in value.
__global__ void __launch_bounds__(256)
    k_live_build(int npos, int C, const double* relax, const double* blo, const double* bhi,
                 const double* rlo, const double* rhi, int* cnt, unsigned short* idx,
                 long long sst, long long pst, unsigned* chmask, int mstride) {
  const int img = blockIdx.z;
  if (chmask) chmask += (long long)img * mstride;
  relax += 8 * img * sst;
  blo += img * sst; bhi += img * sst; rlo += img * sst; rhi += img * sst;
  idx += img * sst;
  cnt += img * pst;
  const int lane = threadIdx.x & 31;
  for (int pos = blockIdx.x * 8 + (threadIdx.x >> 5); pos < npos; pos += gridDim.x * 8) {
    int base = 0;
    for (int c0 = 0; c0 < C; c0 += 32) {
      const int c = c0 + lane;
      bool live = false;
      if (c < C) {
        const long long j = (long long)pos * C + c;
        const double* R = relax + 8 * j;
        bool zr = true;
#pragma unroll
        for (int k = 0; k < 8; ++k) zr &= R[k] == 0.0;
        live = !(zr && blo[j] == 0.0 && bhi[j] == 0.0 && rlo[j] == 0.0 && rhi[j] == 0.0);
      }
      const unsigned m = __ballot_sync(0xffffffffu, live);
      if (live) idx[(long long)pos * C + base + __popc(m & ((1u << lane) - 1u))] = (unsigned short)c;
      if (chmask && lane == 0 && m && c0 < 512) atomicOr(&chmask[c0 >> 5], m);  // live at any position
      base += __popc(m);
    }
    if (lane == 0) cnt[pos] = base;
  }
}

void launch_live_build(cudaStream_t s, int npos, int C, const double* relax, const double* blo,
                       const double* bhi, const double* rlo, const double* rhi, int* cnt,
                       unsigned short* idx, int nimg, long long sst, long long pst, unsigned* chmask,
                       int mstride) {
  unsigned gx = cdiv(npos, 8);
  if (gx > 1024) gx = 1024;
  if (chmask)
    for (int b = 0; b < nimg; ++b) cudaMemsetAsync(chmask + (size_t)b * mstride, 0, 16 * sizeof(unsigned), s);
  k_live_build<<<dim3(gx, 1, nimg), 256, 0, s>>>(npos, C, relax, blo, bhi, rlo, rhi, cnt, idx, sst, pst, chmask,
                                                 mstride);
  ++g_launches;
}

// Conv coefficients over the live cells only: one warp per output position of
// the row's window, lanes over that position's live channels (two per lane
// when more than 32 are live, sharing each compacted coefficient load), the
// same gather as k_gbc_sparse2 in the reference's (ch, cw, d) order.
template <int MINB>
__global__ void __launch_bounds__(256, MINB)
    k_gbc_live(LayerDev L, RowsDev rows, FrameDev fi, FrameDev fo, SparseDev sp, MatDev in,
               MatDev out, LiveDev lv, Counters* ctr) {
  int i;
  if (!rows_resolve(rows, blockIdx.y, i)) return;
  bool upper;
  int img;
  const int q = row_query(rows, i, upper, img);
  int bw, bh, nbw, nbh;
  frame_base(fi, q, bw, bh);
  frame_base(fo, q, nbw, nbh);
  const int* lcnt = lv.cnt + (long long)img * lv.pst;
  const unsigned short* lidx = lv.idx + (long long)img * lv.sst;
  const long long ocells = out.cells;
  const double* ilo = in.lo + phys_row(in, i) * in.cells;
  const double* ihi = in.hi + phys_row(in, i) * in.cells;
  double* olo = out.lo + (size_t)i * ocells;
  double* ohi = out.hi + (size_t)i * ocells;
  const int cin = L.in_c, cout = L.out_c;
  const bool band = products_in_band(in.stat, L.wmin, L.wmax);
  const int* cnt = sp.cnt + (size_t)i * sp.ncell;
  const size_t rbase = (size_t)i * sp.ncell * sp.C;
  const int lane = threadIdx.x & 31;
  const int npos = fo.S_w * fo.S_h;
  MagAcc mag;
  unsigned long long exec = 0;  // madds of the live cells (lane 0's tally)
  for (int pos = blockIdx.x * 8 + (threadIdx.x >> 5); pos < npos; pos += gridDim.x * 8) {
    const int y = pos / fo.S_w, x = pos - y * fo.S_w;
    const int iy = nbh + y, ix = nbw + x;
    const int gp = iy * fo.G_w + ix;
    const int nl = lcnt[gp];
    const unsigned short* li = lidx + (size_t)gp * cin;
    double* plo = olo + (size_t)pos * cin;
    double* phi = ohi + (size_t)pos * cin;
    for (int c = lane; c < cin; c += 32) {  // dead cells: +0 (live ones overwritten below)
      plo[c] = 0.0;
      phi[c] = 0.0;
    }
    __syncwarp();
    if (nl == 0) continue;
    int ah0 = floordiv(iy + L.ph - L.fh, L.sh) + 1, ah1 = floordiv(iy + L.ph, L.sh);
    int aw0 = floordiv(ix + L.pw - L.fw, L.sw) + 1, aw1 = floordiv(ix + L.pw, L.sw);
    ah0 = max(ah0, bh);
    ah1 = min(ah1, bh + fi.S_h - 1);
    aw0 = max(aw0, bw);
    aw1 = min(aw1, bw + fi.S_w - 1);
    if (ctr && lane == 0) {
      int terms = 0;
      for (int ah = ah0; ah <= ah1; ++ah)
        for (int aw = aw0; aw <= aw1; ++aw) terms += cnt[(ah - bh) * fi.S_w + (aw - bw)];
      exec += (unsigned long long)terms * nl;
    }
    for (int k0 = 0; k0 < nl; k0 += 64) {
      const int ka = k0 + lane, kb = k0 + 32 + lane;
      const bool va = ka < nl, vb = kb < nl;
      const bool two = k0 + 32 < nl;  // warp-uniform
      const int ca = li[va ? ka : 0];
      const int cb = vb ? li[kb] : ca;
      Iv acc0{0.0, 0.0}, acc1{0.0, 0.0};
      if (!band) {
        bool bad = false;
        acc0 = gbc_gather<1>(L, fi, bw, bh, ilo, ihi, iy, ix, ca, bad);
        if (bad) acc0 = gbc_gather<0>(L, fi, bw, bh, ilo, ihi, iy, ix, ca, bad);
        if (two) {
          bad = false;
          acc1 = gbc_gather<1>(L, fi, bw, bh, ilo, ihi, iy, ix, cb, bad);
          if (bad) acc1 = gbc_gather<0>(L, fi, bw, bh, ilo, ihi, iy, ix, cb, bad);
        }
      } else {
        double lo0 = 0.0, hi0 = 0.0, lo1 = 0.0, hi1 = 0.0;
        for (int ah = ah0; ah <= ah1; ++ah) {
          const int fy = iy + L.ph - ah * L.sh;
          for (int aw = aw0; aw <= aw1; ++aw) {
            const int fx = ix + L.pw - aw * L.sw;
            const int cell = (ah - bh) * fi.S_w + (aw - bw);
            const int n = cnt[cell];
            const size_t sb = rbase + (size_t)cell * sp.C;
            const double* wa = L.FT + ((size_t)(fy * L.fw + fx) * cout) * cin + ca;
            const double* wb = wa + (cb - ca);
            constexpr int kB = 4;
            int e = 0;
            if (two) {
              for (; e + kB <= n; e += kB) {
                double cl[kB], ch[kB], w0[kB], w1[kB];
#pragma unroll
                for (int k = 0; k < kB; ++k) {
                  const size_t d = sp.idx[sb + e + k];
                  cl[k] = sp.lo[sb + e + k];
                  ch[k] = sp.hi[sb + e + k];
                  w0[k] = wa[d * cin];
                  w1[k] = wb[d * cin];
                }
#pragma unroll
                for (int k = 0; k < kB; ++k) {
                  madd_band(w0[k], cl[k], ch[k], lo0, hi0);
                  madd_band(w1[k], cl[k], ch[k], lo1, hi1);
                }
              }
              for (; e < n; ++e) {
                const size_t d = sp.idx[sb + e];
                const double cl = sp.lo[sb + e], ch = sp.hi[sb + e];
                madd_band(wa[d * cin], cl, ch, lo0, hi0);
                madd_band(wb[d * cin], cl, ch, lo1, hi1);
              }
            } else {
              for (; e + kB <= n; e += kB) {
                double cl[kB], ch[kB], w0[kB];
#pragma unroll
                for (int k = 0; k < kB; ++k) {
                  const size_t d = sp.idx[sb + e + k];
                  cl[k] = sp.lo[sb + e + k];
                  ch[k] = sp.hi[sb + e + k];
                  w0[k] = wa[d * cin];
                }
#pragma unroll
                for (int k = 0; k < kB; ++k) madd_band(w0[k], cl[k], ch[k], lo0, hi0);
              }
              for (; e < n; ++e)
                madd_band(wa[(size_t)sp.idx[sb + e] * cin], sp.lo[sb + e], sp.hi[sb + e], lo0, hi0);
            }
          }
        }
        acc0 = Iv{canon0(lo0), hi0};
        acc1 = Iv{canon0(lo1), hi1};
      }
      if (va) {
        plo[ca] = acc0.lo;
        phi[ca] = acc0.hi;
        mag.add(acc0.lo);
        mag.add(acc0.hi);
      }
      if (vb) {
        plo[cb] = acc1.lo;
        phi[cb] = acc1.hi;
        mag.add(acc1.lo);
        mag.add(acc1.hi);
      }
    }
  }
  mag.flush(out.stat);
  if (ctr && lane == 0 && exec) atomicAdd(&ctr[img].conv_exec, exec);
}

// ---------------------------------------------------------------------------
// The live cells of a ReLU layer as one flat ascending list (position-major,
// channel ascending): pref[pos] = live cells before grid position pos,
// fpos / fch = position and channel of each. Built from k_live_build's
// per-position lists once per image (k_live_flat: one block scan).
__global__ void __launch_bounds__(1024)
    k_live_flat(int npos, int C, const int* cnt, const unsigned short* idx, int* pref,
                unsigned short* fpos, unsigned short* fch, long long sst, long long pst, long long fst) {
  using Scan = cub::BlockScan<int, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int s_base;
  const int img = blockIdx.z;
  cnt += img * pst;
  idx += img * sst;
  pref += img * fst;
  fpos += img * sst;
  fch += img * sst;
  if (threadIdx.x == 0) s_base = 0;
  __syncthreads();
  for (int start = 0; start < npos; start += 1024) {
    const int p = start + threadIdx.x;
    const int c = p < npos ? cnt[p] : 0;
    int off, total;
    Scan(tmp).ExclusiveSum(c, off, total);
    off += s_base;
    if (p < npos) {
      pref[p] = off;
      for (int k = 0; k < c; ++k) {
        fpos[off + k] = (unsigned short)p;
        fch[off + k] = idx[(long long)p * C + k];
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) s_base += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) pref[npos] = s_base;
}

void launch_live_flat(cudaStream_t s, int npos, int C, const int* cnt, const unsigned short* idx,
                      int* pref, unsigned short* fpos, unsigned short* fch, int nimg, long long sst,
                      long long pst, long long fst) {
  k_live_flat<<<dim3(1, 1, nimg), 1024, 0, s>>>(npos, C, cnt, idx, pref, fpos, fch, sst, pst, fst);
  ++g_launches;
}

// Conv coefficients over the flat list of live cells: one output (a live
// cell of the row's window) per thread, the gather of k_gbc_sparse2 in the
// reference's (ch, cw, d) order. Threads of a warp take consecutive live
// cells (one or two grid positions), so coefficient loads are broadcasts and
// no lane computes a dead cell. The output rows are zeroed beforehand (dead
// cells). A block takes FlatDev::opb consecutive live cells of its row's window:
// the window's grid rows are consecutive runs of the flat list.
static int flat_opb() {  // live cells per block (PC_GBC_FLAT_OPB)
  static const int v = env_int("PC_GBC_FLAT_OPB", 512);
  return v;
}
template <int MINB, bool FAST = false, int KB = 4, bool CHECKED = false>
__global__ void __launch_bounds__(256, MINB)
    k_gbc_flat(LayerDev L, RowsDev rows_in, FrameDev fi, FrameDev fo, SparseDev sp, MatDev in,
               MatDev out, FlatDev fl, Counters* ctr) {
  __shared__ int s_seg[65];  // live cells before each window row (S_h <= 64)
  // Two instantiations per launch: the band one (no call in its loop, so a
  // lean register budget) returns when the operands are not proven in band,
  // the CHECKED one only works in that (rare) case. The CHECKED one is
  // launched one block row only (gridDim.y == 1) and loops over the rows,
  // so its blocks that return cost little.
  const bool band = FAST || products_in_band(in.stat, L.wmin, L.wmax);
  if (band == CHECKED) return;
  const int nblk = CHECKED ? rows_in.n : 1;
  for (int rb = CHECKED ? 0 : (int)blockIdx.y; rb < (CHECKED ? nblk : (int)blockIdx.y + 1); ++rb) {
  RowsDev rows = rows_in;
  int i;
  if (!rows_resolve(rows, rb, i)) continue;
  bool upper;
  int img;
  const int q = row_query(rows, i, upper, img);
  int bw, bh, nbw, nbh;
  frame_base(fi, q, bw, bh);
  frame_base(fo, q, nbw, nbh);
  const int* pref = fl.pref + (long long)img * fl.fst;
  const unsigned short* fpos = fl.fpos + (long long)img * fl.sst;
  const unsigned short* fch = fl.fch + (long long)img * fl.sst;
  if (threadIdx.x <= fo.S_h) {
    int c = 0;
    for (int y = 0; y < (int)threadIdx.x; ++y) {
      const int g0 = (nbh + y) * fo.G_w + nbw;
      c += pref[g0 + fo.S_w] - pref[g0];
    }
    s_seg[threadIdx.x] = c;
  }
  __syncthreads();
  const int total = s_seg[fo.S_h];
  const int t0 = blockIdx.x * fl.opb;
  double* part = fl.part ? fl.part + ((size_t)i * gridDim.x + blockIdx.x) * 3 : nullptr;
  if (t0 >= total) {
    if (part && threadIdx.x < 3) part[threadIdx.x] = 0.0;
    __syncthreads();  // s_seg is rewritten by the next row
    continue;
  }
  const int t1 = min(total, t0 + fl.opb);
  const long long ocells = out.cells;
  const double* ilo = in.lo + phys_row(in, i) * in.cells;
  const double* ihi = in.hi + phys_row(in, i) * in.cells;
  double* olo = out.lo + (size_t)i * ocells;
  double* ohi = out.hi + (size_t)i * ocells;
  const int cin = L.in_c, cout = L.out_c;
  double pS = 0.0, pA = 0.0, pN = 0.0;  // predicted compaction partials (FlatDev::part)
  const long long pso = (long long)img * rows.sst;
  const int* cnt = sp.cnt + (size_t)i * sp.ncell;
  const size_t rbase = (size_t)i * sp.ncell * sp.C;
  MagAcc mag;
  unsigned long long exec = 0;
  int y = 0;
  for (int t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
    while (t >= s_seg[y + 1]) ++y;
    const int e = pref[(nbh + y) * fo.G_w + nbw] + (t - s_seg[y]);
    const int gp = fpos[e], ci = fch[e];
    const int iy = nbh + y, ix = gp - iy * fo.G_w;
    Iv acc;
    if (CHECKED) {
      acc = gbc_gather_checked(L, fi, bw, bh, ilo, ihi, iy, ix, ci);
    } else {
      int ah0 = floordiv(iy + L.ph - L.fh, L.sh) + 1, ah1 = floordiv(iy + L.ph, L.sh);
      int aw0 = floordiv(ix + L.pw - L.fw, L.sw) + 1, aw1 = floordiv(ix + L.pw, L.sw);
      ah0 = max(ah0, bh);
      ah1 = min(ah1, bh + fi.S_h - 1);
      aw0 = max(aw0, bw);
      aw1 = min(aw1, bw + fi.S_w - 1);
      double lo = 0.0, hi = 0.0;
      for (int ah = ah0; ah <= ah1; ++ah) {
        const int fy = iy + L.ph - ah * L.sh;
        for (int aw = aw0; aw <= aw1; ++aw) {
          const int fx = ix + L.pw - aw * L.sw;
          const int cell = (ah - bh) * fi.S_w + (aw - bw);
          const int n = cnt[cell];
          exec += n;
          const size_t sb = rbase + (size_t)cell * sp.C;
          const double* wp = L.FT + ((size_t)(fy * L.fw + fx) * cout) * cin + ci;
          constexpr int kB = KB;
          int k = 0;
          for (; k + kB <= n; k += kB) {
            double cl[kB], ch[kB], w[kB];
#pragma unroll
            for (int u = 0; u < kB; ++u) {
              cl[u] = sp.lo[sb + k + u];
              ch[u] = sp.hi[sb + k + u];
              w[u] = wp[(size_t)sp.idx[sb + k + u] * cin];
            }
#pragma unroll
            for (int u = 0; u < kB; ++u) {
              if (FAST) madd_dir(w[u], cl[u], ch[u], lo, hi);
              else madd_band(w[u], cl[u], ch[u], lo, hi);
            }
          }
          for (; k < n; ++k) {
            if (FAST) madd_dir(wp[(size_t)sp.idx[sb + k] * cin], sp.lo[sb + k], sp.hi[sb + k], lo, hi);
            else madd_band(wp[(size_t)sp.idx[sb + k] * cin], sp.lo[sb + k], sp.hi[sb + k], lo, hi);
          }
        }
      }
      acc = Iv{canon0(lo), hi};
    }
    const size_t o = ((size_t)y * fo.S_w + (ix - nbw)) * cin + ci;
    olo[o] = acc.lo;
    ohi[o] = acc.hi;
    mag.add(acc.lo);
    mag.add(acc.hi);
    if (part && !iv_zero(acc)) {  // the raw concretisation's corner term (k_pred_terms)
      const long long j = ((long long)iy * fo.G_w + ix) * fo.C + ci;
      const Iv Br{fl.prlo[pso + j], fl.prhi[pso + j]};
      const double tt = upper ? corner_hi(acc, Br) : corner_lo(acc, Br);
      pS += tt;
      pA += fabs(tt);
      pN += 1.0;
    }
  }
  mag.flush(out.stat);
  if (ctr) {
    for (int o = 16; o > 0; o >>= 1) exec += __shfl_down_sync(__activemask(), exec, o);
    if ((threadIdx.x & 31) == 0 && exec) atomicAdd(&ctr[img].conv_exec, exec);
  }
  if (part) {
    __shared__ double s_pr[3][8];
    for (int o = 16; o > 0; o >>= 1) {
      pS += __shfl_down_sync(0xffffffffu, pS, o);
      pA += __shfl_down_sync(0xffffffffu, pA, o);
      pN += __shfl_down_sync(0xffffffffu, pN, o);
    }
    if ((threadIdx.x & 31) == 0) {
      s_pr[0][threadIdx.x >> 5] = pS;
      s_pr[1][threadIdx.x >> 5] = pA;
      s_pr[2][threadIdx.x >> 5] = pN;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
      double v = 0.0;
      for (int w = 0; w < 8; ++w) v += s_pr[threadIdx.x][w];
      part[threadIdx.x] = v;
    }
  }
  __syncthreads();  // s_seg / s_pr are rewritten by the next row
  }
}

// k_gbc_flat with two consecutive live cells per thread: they are (almost
// always) two channels of one grid position, so they share every compacted
// coefficient load and give the thread two independent interval chains.
template <int MINB>
__global__ void __launch_bounds__(256, MINB)
    k_gbc_flat2(LayerDev L, RowsDev rows, FrameDev fi, FrameDev fo, SparseDev sp, MatDev in,
                MatDev out, FlatDev fl, Counters* ctr) {
  __shared__ int s_seg[65];
  int i;
  if (!rows_resolve(rows, blockIdx.y, i)) return;
  bool upper;
  int img;
  const int q = row_query(rows, i, upper, img);
  int bw, bh, nbw, nbh;
  frame_base(fi, q, bw, bh);
  frame_base(fo, q, nbw, nbh);
  const int* pref = fl.pref + (long long)img * fl.fst;
  const unsigned short* fpos = fl.fpos + (long long)img * fl.sst;
  const unsigned short* fch = fl.fch + (long long)img * fl.sst;
  if (threadIdx.x <= fo.S_h) {
    int c = 0;
    for (int y = 0; y < (int)threadIdx.x; ++y) {
      const int g0 = (nbh + y) * fo.G_w + nbw;
      c += pref[g0 + fo.S_w] - pref[g0];
    }
    s_seg[threadIdx.x] = c;
  }
  __syncthreads();
  const int total = s_seg[fo.S_h];
  const int t0b = blockIdx.x * fl.opb;
  if (t0b >= total) return;
  const int t1b = min(total, t0b + fl.opb);
  const long long ocells = out.cells;
  const double* ilo = in.lo + phys_row(in, i) * in.cells;
  const double* ihi = in.hi + phys_row(in, i) * in.cells;
  double* olo = out.lo + (size_t)i * ocells;
  double* ohi = out.hi + (size_t)i * ocells;
  const int cin = L.in_c, cout = L.out_c;
  const bool band = products_in_band(in.stat, L.wmin, L.wmax);
  const int* cnt = sp.cnt + (size_t)i * sp.ncell;
  const size_t rbase = (size_t)i * sp.ncell * sp.C;
  MagAcc mag;
  unsigned long long exec = 0;
  auto locate = [&](int t, int& y, int& ix, int& ci) {
    while (t >= s_seg[y + 1]) ++y;
    const int e = pref[(nbh + y) * fo.G_w + nbw] + (t - s_seg[y]);
    const int gp = fpos[e];
    ci = fch[e];
    ix = gp - (nbh + y) * fo.G_w;
  };
  auto put = [&](int y, int ix, int ci, Iv acc) {
    const size_t o = ((size_t)y * fo.S_w + (ix - nbw)) * cin + ci;
    olo[o] = acc.lo;
    ohi[o] = acc.hi;
    mag.add(acc.lo);
    mag.add(acc.hi);
  };
  int ya = 0;
  for (int t = t0b + 2 * threadIdx.x; t < t1b; t += 2 * blockDim.x) {
    int ixa, ca, yb, ixb = -1, cb = -1;
    locate(t, ya, ixa, ca);
    const bool has_b = t + 1 < t1b;
    yb = ya;
    if (has_b) locate(t + 1, yb, ixb, cb);
    const bool pair = has_b && yb == ya && ixb == ixa;
    const int iy = nbh + ya;
    if (!band || !pair) {  // checked path, or two positions: one output at a time
      for (int u = 0; u < (has_b ? 2 : 1); ++u) {
        const int yy = u ? yb : ya, xx = u ? ixb : ixa, cc = u ? cb : ca;
        Iv acc;
        if (!band) {
          acc = gbc_gather_checked(L, fi, bw, bh, ilo, ihi, nbh + yy, xx, cc);
        } else {
          const int py = nbh + yy;
          int ah0 = floordiv(py + L.ph - L.fh, L.sh) + 1, ah1 = floordiv(py + L.ph, L.sh);
          int aw0 = floordiv(xx + L.pw - L.fw, L.sw) + 1, aw1 = floordiv(xx + L.pw, L.sw);
          ah0 = max(ah0, bh);
          ah1 = min(ah1, bh + fi.S_h - 1);
          aw0 = max(aw0, bw);
          aw1 = min(aw1, bw + fi.S_w - 1);
          double lo = 0.0, hi = 0.0;
          for (int ah = ah0; ah <= ah1; ++ah) {
            const int fy = py + L.ph - ah * L.sh;
            for (int aw = aw0; aw <= aw1; ++aw) {
              const int fx = xx + L.pw - aw * L.sw;
              const int cell = (ah - bh) * fi.S_w + (aw - bw);
              const int n = cnt[cell];
              exec += n;
              const size_t sb = rbase + (size_t)cell * sp.C;
              const double* wp = L.FT + ((size_t)(fy * L.fw + fx) * cout) * cin + cc;
              for (int k = 0; k < n; ++k)
                madd_band(wp[(size_t)sp.idx[sb + k] * cin], sp.lo[sb + k], sp.hi[sb + k], lo, hi);
            }
          }
          acc = Iv{canon0(lo), hi};
        }
        put(yy, xx, cc, acc);
      }
      continue;
    }
    int ah0 = floordiv(iy + L.ph - L.fh, L.sh) + 1, ah1 = floordiv(iy + L.ph, L.sh);
    int aw0 = floordiv(ixa + L.pw - L.fw, L.sw) + 1, aw1 = floordiv(ixa + L.pw, L.sw);
    ah0 = max(ah0, bh);
    ah1 = min(ah1, bh + fi.S_h - 1);
    aw0 = max(aw0, bw);
    aw1 = min(aw1, bw + fi.S_w - 1);
    double lo0 = 0.0, hi0 = 0.0, lo1 = 0.0, hi1 = 0.0;
    for (int ah = ah0; ah <= ah1; ++ah) {
      const int fy = iy + L.ph - ah * L.sh;
      for (int aw = aw0; aw <= aw1; ++aw) {
        const int fx = ixa + L.pw - aw * L.sw;
        const int cell = (ah - bh) * fi.S_w + (aw - bw);
        const int n = cnt[cell];
        exec += 2 * n;
        const size_t sb = rbase + (size_t)cell * sp.C;
        const double* wa = L.FT + ((size_t)(fy * L.fw + fx) * cout) * cin + ca;
        const double* wb = wa + (cb - ca);
        constexpr int kB = 4;
        int k = 0;
        for (; k + kB <= n; k += kB) {
          double cl[kB], ch[kB], w0[kB], w1[kB];
#pragma unroll
          for (int u = 0; u < kB; ++u) {
            const size_t d = sp.idx[sb + k + u];
            cl[u] = sp.lo[sb + k + u];
            ch[u] = sp.hi[sb + k + u];
            w0[u] = wa[d * cin];
            w1[u] = wb[d * cin];
          }
#pragma unroll
          for (int u = 0; u < kB; ++u) {
            madd_band(w0[u], cl[u], ch[u], lo0, hi0);
            madd_band(w1[u], cl[u], ch[u], lo1, hi1);
          }
        }
        for (; k < n; ++k) {
          const size_t d = sp.idx[sb + k];
          const double cl = sp.lo[sb + k], ch = sp.hi[sb + k];
          madd_band(wa[d * cin], cl, ch, lo0, hi0);
          madd_band(wb[d * cin], cl, ch, lo1, hi1);
        }
      }
    }
    put(ya, ixa, ca, Iv{canon0(lo0), hi0});
    put(yb, ixb, cb, Iv{canon0(lo1), hi1});
  }
  mag.flush(out.stat);
  if (ctr) {
    for (int o = 16; o > 0; o >>= 1) exec += __shfl_down_sync(__activemask(), exec, o);
    if ((threadIdx.x & 31) == 0 && exec) atomicAdd(&ctr[img].conv_exec, exec);
  }
}

int gbc_flat_blocks(const FrameDev& fout, const LayerDev& L) {
  return (int)cdiv((long long)fout.S_w * fout.S_h * L.in_c, flat_opb());
}

void launch_gbc_flat(cudaStream_t s, const LayerDev& L, const RowsDev& rows, const FrameDev& fin,
                     const FrameDev& fout, SparseDev sp, MatDev in, MatDev out, FlatDev fl, Counters* ctr,
                     bool fast) {
  if (debug_skip("conv")) return;
  static const int minb = env_int("PC_GBC_FLAT_MINB", 3);
  // dead cells: +0 (the live ones are overwritten)
  cudaMemsetAsync(out.lo, 0, sizeof(double) * (size_t)rows.n * out.cells, s);
  cudaMemsetAsync(out.hi, 0, sizeof(double) * (size_t)rows.n * out.cells, s);
  const long long cells = (long long)fout.S_w * fout.S_h * L.in_c;
  fl.opb = flat_opb();
  dim3 grid(cdiv(cells, fl.opb), rows.n);
  static const int pairs = env_int("PC_GBC_FLAT_PAIRS", 0);
  static const int kb = env_int("PC_GBC_FLAT_KB", 4);
  static const int minb2 = env_int("PC_GBC_FLAT2_MINB", 2);
  if (pairs) {
    if (minb2 >= 3) k_gbc_flat2<3><<<grid, 256, 0, s>>>(L, rows, fin, fout, sp, in, out, fl, ctr);
    else k_gbc_flat2<2><<<grid, 256, 0, s>>>(L, rows, fin, fout, sp, in, out, fl, ctr);
  } else if (fast) {
    k_gbc_flat<3, true><<<grid, 256, 0, s>>>(L, rows, fin, fout, sp, in, out, fl, ctr);
  } else {
    if (kb == 2 && minb >= 4) k_gbc_flat<4, false, 2><<<grid, 256, 0, s>>>(L, rows, fin, fout, sp, in, out, fl, ctr);
    else if (kb == 2) k_gbc_flat<3, false, 2><<<grid, 256, 0, s>>>(L, rows, fin, fout, sp, in, out, fl, ctr);
    else if (kb == 8) k_gbc_flat<2, false, 8><<<grid, 256, 0, s>>>(L, rows, fin, fout, sp, in, out, fl, ctr);
    else if (minb >= 4) k_gbc_flat<4><<<grid, 256, 0, s>>>(L, rows, fin, fout, sp, in, out, fl, ctr);
    else if (minb == 3) k_gbc_flat<3><<<grid, 256, 0, s>>>(L, rows, fin, fout, sp, in, out, fl, ctr);
    else k_gbc_flat<2><<<grid, 256, 0, s>>>(L, rows, fin, fout, sp, in, out, fl, ctr);
    k_gbc_flat<2, false, 4, true><<<dim3(grid.x, 1), 256, 0, s>>>(L, rows, fin, fout, sp, in, out, fl, ctr);
    ++g_launches;
  }
  ++g_launches;
}

// ---------------------------------------------------------------------------
// Dense-tile conv over compacted channel sets. On the residual nets the zero
// pattern of a conv step is (nearly) channel-uniform: a ReLU layer's dead
// neurons are whole channels at almost every position (scripts/live_stats.py),
// so the input coefficients are nonzero on a channel set D (the row's union,
// sp.dmask) and the live outputs on a channel set CI (the layer's union,
// k_live_build's chmask). The step is then a dense product over D x CI per
// filter tap, done as a shared-memory tiled loop: a CTA owns 32 output
// positions (one stride-parity class) x 64 channels of CI; per (tap, 16-wide
// chunk of D) it stages the 32 positions' covering coefficients and the
// 16 x 64 weights by cp.async (double buffered) and every thread runs 8
// interval chains (1 position x 8 channels: the coefficient is reused 8 times,
// the weights are warp broadcasts). Taps run in descending (fy, fx) and D
// ascending, i.e. covering cells ascending then d ascending: the reference's
// (ch, cw, d) order for every output (backsub.hpp:449-489). Terms outside
// the sets are exact zeros (zero coefficient, or a cell no result reads) and a
// zero term leaves the accumulators unchanged, so results are the flat
// kernel's bit for bit.
constexpr int kTP = 32, kTCH = 64, kTD = 16;
struct TileSmem {
  double c[2][kTD][kTP][2];   // coefficients (lo, hi) per d-slot, position
  double w[2][kTD][kTCH];     // weights per d-slot, channel
  unsigned short dl[512], cl[512];
  int nd, nc;
};

__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }

__global__ void __launch_bounds__(256, 2)
    k_gbc_tile(LayerDev L, RowsDev rows, FrameDev fi, FrameDev fo, SparseDev sp, MatDev in, MatDev out,
               const unsigned* chmask, long long mstride, Counters* ctr) {
  extern __shared__ __align__(16) unsigned char tsm_raw[];
  TileSmem& S = *reinterpret_cast<TileSmem*>(tsm_raw);
  int i;
  if (!rows_resolve(rows, blockIdx.z, i)) return;
  bool upper;
  int img;
  const int q = row_query(rows, i, upper, img);
  int bw, bh, nbw, nbh;
  frame_base(fi, q, bw, bh);
  frame_base(fo, q, nbw, nbh);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cin = L.in_c, cout = L.out_c;
  // channel lists: D from the row's nonzero-channel mask, CI from the layer's
  if (tid == 0) {
    const unsigned* dm = sp.dmask + (size_t)i * 16;
    const unsigned* cm = chmask + (long long)img * mstride;
    int nd = 0, nc = 0;
    for (int w = 0; w < 16 && 32 * w < cout; ++w)
      for (unsigned b = dm[w]; b; b &= b - 1) S.dl[nd++] = (unsigned short)(32 * w + __ffs(b) - 1);
    for (int w = 0; w < 16 && 32 * w < cin; ++w)
      for (unsigned b = cm[w]; b; b &= b - 1) S.cl[nc++] = (unsigned short)(32 * w + __ffs(b) - 1);
    S.nd = nd;
    S.nc = nc;
  }
  __syncthreads();
  const int nd = S.nd, nc = S.nc;
  const int ch0 = blockIdx.y * kTCH;
  if (ch0 >= nc) return;
  // stride-parity class and tile of positions
  const int sh = L.sh, sw = L.sw;
  int cls = 0, tile = blockIdx.x, ncy = 0, ncx = 0, y0 = 0, x0 = 0;
  for (;; ++cls) {
    if (cls >= sh * sw) return;
    const int cy = cls / sw, cx = cls - cy * sw;
    y0 = ((cy - nbh) % sh + sh) % sh;  // first window row with (nbh + y) % sh == cy
    x0 = ((cx - nbw) % sw + sw) % sw;
    ncy = y0 < fo.S_h ? (fo.S_h - y0 + sh - 1) / sh : 0;
    ncx = x0 < fo.S_w ? (fo.S_w - x0 + sw - 1) / sw : 0;
    const int nt = (ncy * ncx + kTP - 1) / kTP;
    if (tile < nt) break;
    tile -= nt;
  }
  const int cy = cls / sw, cx = cls - cy * sw;
  const int npos = ncy * ncx;
  // this thread's output: position lane of the tile, channels ch0 + 8*warp .. +8
  const int li = tile * kTP + lane;
  const bool pvalid = li < npos;
  const int y = y0 + sh * (pvalid ? li / ncx : 0), x = x0 + sw * (pvalid ? li % ncx : 0);
  const int iy = nbh + y, ix = nbw + x;
  const int cg = ch0 + 8 * warp;  // first channel slot of this warp
  const bool wvalid = cg < nc;
  const bool band = products_in_band(in.stat, L.wmin, L.wmax);
  const double* ilo = in.lo + phys_row(in, i) * in.cells;
  const double* ihi = in.hi + phys_row(in, i) * in.cells;
  double* olo = out.lo + (size_t)i * out.cells;
  double* ohi = out.hi + (size_t)i * out.cells;
  if (!band) {  // operands not proven in band: the checked gather per output
    if (pvalid && wvalid)
      for (int k = 0; k < 8 && cg + k < nc; ++k) {
        const int ci = S.cl[cg + k];
        const Iv a = gbc_gather_checked(L, fi, bw, bh, ilo, ihi, iy, ix, ci);
        const size_t o = ((size_t)y * fo.S_w + x) * cin + ci;
        olo[o] = a.lo;
        ohi[o] = a.hi;
      }
    return;
  }
  // taps of this parity class, descending: fy = fy_hi, fy_hi - sh, ... (same for x)
  const int fyp = ((cy + L.ph) % sh + sh) % sh, fxp = ((cx + L.pw) % sw + sw) % sw;
  const int nfy = fyp < L.fh ? (L.fh - fyp + sh - 1) / sh : 0;
  const int nfx = fxp < L.fw ? (L.fw - fxp + sw - 1) / sw : 0;
  const int ntap = nfy * nfx, nch = (nd + kTD - 1) / kTD, nit = ntap * nch;
  auto stage = [&](int it, int buf) {
    const int tp = it / nch, dc = (it - tp * nch) * kTD;
    const int fy = fyp + sh * (nfy - 1 - tp / nfx), fx = fxp + sw * (nfx - 1 - tp % nfx);
    // coefficients: 16 d-slots x 32 positions x (lo, hi) = 1024 8-byte copies, 4 per thread
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int e = tid + 256 * r;              // (d-slot, position, half)
      const int half = e & 1, p = (e >> 1) & 31, ds = e >> 6;
      const int lp = tile * kTP + p;
      bool ok = lp < npos && dc + ds < nd;
      const double* src = ilo;
      if (ok) {
        const int py = nbh + y0 + sh * (lp / ncx), px = nbw + x0 + sw * (lp % ncx);
        const int ah = (py + L.ph - fy) / sh, aw = (px + L.pw - fx) / sw;  // exact: parity class
        ok = ah >= bh && ah < bh + fi.S_h && aw >= bw && aw < bw + fi.S_w;
        if (ok) src = (half ? ihi : ilo) + ((size_t)(ah - bh) * fi.S_w + (aw - bw)) * cout + S.dl[dc + ds];
      }
      cp_async8(&S.c[buf][ds][p][half], src, ok);
    }
    // weights: 16 d-slots x 64 channels, 4 per thread
    const double* wt = L.FT + (size_t)(fy * L.fw + fx) * cout * cin;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int e = tid + 256 * r;
      const int c = e & 63, ds = e >> 6;
      const bool ok = dc + ds < nd && ch0 + c < nc;
      const double* src = ok ? wt + (size_t)S.dl[dc + ds] * cin + S.cl[ch0 + c] : wt;
      cp_async8(&S.w[buf][ds][c], src, ok);
    }
    cp_async_commit();
  };
  double lo[8], hi[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) lo[k] = hi[k] = 0.0;
  if (nit > 0) stage(0, 0);
  for (int it = 0; it < nit; ++it) {
    const int buf = it & 1;
    if (it + 1 < nit) {
      stage(it + 1, buf ^ 1);
      cp_async_wait1();
    } else {
      cp_async_wait_all();
    }
    __syncthreads();
    if (wvalid) {
#pragma unroll 4
      for (int ds = 0; ds < kTD; ++ds) {
        const double2 cv = *reinterpret_cast<const double2*>(&S.c[buf][ds][lane][0]);
        const double4* wp = reinterpret_cast<const double4*>(&S.w[buf][ds][8 * warp]);
        const double4 w0 = wp[0], w1 = wp[1];
        madd_band(w0.x, cv.x, cv.y, lo[0], hi[0]);
        madd_band(w0.y, cv.x, cv.y, lo[1], hi[1]);
        madd_band(w0.z, cv.x, cv.y, lo[2], hi[2]);
        madd_band(w0.w, cv.x, cv.y, lo[3], hi[3]);
        madd_band(w1.x, cv.x, cv.y, lo[4], hi[4]);
        madd_band(w1.y, cv.x, cv.y, lo[5], hi[5]);
        madd_band(w1.z, cv.x, cv.y, lo[6], hi[6]);
        madd_band(w1.w, cv.x, cv.y, lo[7], hi[7]);
      }
    }
    __syncthreads();  // buffer `buf` is restaged two iterations on
  }
  MagAcc mag;
  if (pvalid && wvalid) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (cg + k >= nc) break;
      const int ci = S.cl[cg + k];
      const size_t o = ((size_t)y * fo.S_w + x) * cin + ci;
      const double a = canon0(lo[k]);
      olo[o] = a;
      ohi[o] = hi[k];
      mag.add(a);
      mag.add(hi[k]);
    }
  }
  mag.flush(out.stat);
  if (ctr && tid == 0)  // interval madds issued (zero terms included): positions x channels x taps x |D|
    atomicAdd(&ctr[img].conv_exec,
              (unsigned long long)min(kTP, npos - tile * kTP) * min(kTCH, nc - ch0) * ntap * nd);
}

void launch_gbc_tile(cudaStream_t s, const LayerDev& L, const RowsDev& rows, const FrameDev& fin,
                     const FrameDev& fout, SparseDev sp, MatDev in, MatDev out, const unsigned* chmask,
                     long long mstride, Counters* ctr) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_gbc_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(TileSmem));
    attr = true;
  }
  cudaMemsetAsync(out.lo, 0, sizeof(double) * (size_t)rows.n * out.cells, s);  // channels outside CI
  cudaMemsetAsync(out.hi, 0, sizeof(double) * (size_t)rows.n * out.cells, s);
  const int npos = fout.S_w * fout.S_h;
  const unsigned gx = cdiv(npos, kTP) + L.sh * L.sw;  // parity classes round up separately
  dim3 grid(gx, cdiv(L.in_c, kTCH), rows.n);
  k_gbc_tile<<<grid, 256, sizeof(TileSmem), s>>>(L, rows, fin, fout, sp, in, out, chmask, mstride, ctr);
  ++g_launches;
}

void launch_gbc_live(cudaStream_t s, const LayerDev& L, const RowsDev& rows, const FrameDev& fin,
                     const FrameDev& fout, SparseDev sp, MatDev in, MatDev out, LiveDev lv, Counters* ctr) {
  static const int minb = env_int("PC_GBC_LIVE_MINB", 2);
  unsigned gx = cdiv(fout.S_w * fout.S_h, 8);
  if (gx > 1024) gx = 1024;
  dim3 grid(gx, rows.n);
  if (minb >= 3) k_gbc_live<3><<<grid, 256, 0, s>>>(L, rows, fin, fout, sp, in, out, lv, ctr);
  else if (minb == 2) k_gbc_live<2><<<grid, 256, 0, s>>>(L, rows, fin, fout, sp, in, out, lv, ctr);
  else k_gbc_live<1><<<grid, 256, 0, s>>>(L, rows, fin, fout, sp, in, out, lv, ctr);
  ++g_launches;
}

void launch_gbc_sparse(cudaStream_t s, const LayerDev& L, const RowsDev& rows, const FrameDev& fin,
                       const FrameDev& fout, SparseDev sp, MatDev in, MatDev out) {
  static const int pairs = env_int("PC_GBC_PAIRS", 1);
  static const int minb = env_int("PC_GBC_MINB", 3);
  if (pairs && L.in_c % 2 == 0) {
    unsigned gx = cdiv(out.cells / 2, 256);
    if (gx > 1024) gx = 1024;
    dim3 grid(gx, rows.n);
    if (minb >= 4) k_gbc_sparse2<4><<<grid, 256, 0, s>>>(L, rows, fin, fout, sp, in, out);
    else if (minb == 3) k_gbc_sparse2<3><<<grid, 256, 0, s>>>(L, rows, fin, fout, sp, in, out);
    else if (minb == 2) k_gbc_sparse2<2><<<grid, 256, 0, s>>>(L, rows, fin, fout, sp, in, out);
    else k_gbc_sparse2<1><<<grid, 256, 0, s>>>(L, rows, fin, fout, sp, in, out);
    ++g_launches;
    return;
  }
  unsigned gx = cdiv(out.cells, 256);
  if (gx > 1024) gx = 1024;
  dim3 grid(gx, rows.n);
  k_gbc_sparse<<<grid, 256, 0, s>>>(L, rows, fin, fout, sp, in, out);
  ++g_launches;
}

bool gbc_sparse_wanted(const LayerDev& L) {
  static const int variant = env_int("PC_GBC", 3);
  return variant == 3 && L.in_c >= 32 && L.out_c <= 65535;
}

void launch_gbc_coef(cudaStream_t s, const LayerDev& L, const RowsDev& rows, const FrameDev& fin,
                     const FrameDev& fout, MatDev in, MatDev out, int* queue) {
  // PC_GBC: 2 (default) shared-memory tiled kernel where eligible, 1 the
  // register-blocked gather, 0 the one-output-per-thread gather
  static const int variant = env_int("PC_GBC", 3);
  if (variant >= 2 && gbc_smem_eligible(L, fout) && queue) {
    launch_gbc_smem(s, L, rows, fin, fout, in, out, queue);
    return;
  }
  if (variant == 1) {
    launch_gbc_tile(s, L, rows, fin, fout, in, out);
    return;
  }
  unsigned gx = cdiv(out.cells, 256);
  if (gx > 1024) gx = 1024;
  dim3 grid(gx, rows.n);
  k_gbc_coef<<<grid, 256, 0, s>>>(L, rows, fin, fout, in, out);
  ++g_launches;
}

// relu_step coefficients (backsub.hpp:536-563): per nonzero cell, slope by
// sign (upper rows: gamma for c>=0, alpha for c<=0; lower rows mirrored);
// straddling cells split into positive and negative parts.
template <bool FAST>
__device__ __forceinline__ Iv relu_map(const Iv& c, const Iv& sp, const Iv& sn, bool& bad) {
  if (FAST) {
    const bool pos = !(c.lo < 0.0), neg = !(c.hi > 0.0);
    // sign-stable: iv_mul(c, slope); straddling: iv_add of the two parts
    const Iv s1 = (neg && !pos) ? sn : sp;
    const Iv a = pos || neg ? c : iv_pos_part(c);
    const Iv m1 = f_iv_mul(a, s1, bad);
    const Iv m2 = f_iv_mul(iv_neg_part(c), sn, bad);  // products are band-checked
    const Iv sum{f_add_dn(m1.lo, m2.lo), f_add_up(m1.hi, m2.hi)};
    return (pos || neg) ? m1 : sum;
  }
  if (!(c.lo < 0.0)) return iv_mul(c, sp);
  if (!(c.hi > 0.0)) return iv_mul(c, sn);
  return iv_add(iv_mul(iv_pos_part(c), sp), iv_mul(iv_neg_part(c), sn));
}

__global__ void __launch_bounds__(256)
    k_relu_coef(RowsDev rows, FrameDev f, MatDev in, MatDev out, const double* relax) {
  int i;
  if (!rows_resolve(rows, blockIdx.y, i)) return;
  bool upper;
  int img;
  const int q = row_query(rows, i, upper, img);
  relax += 8 * img * rows.sst;
  int bw, bh;
  frame_base(f, q, bw, bh);
  const long long cells = in.cells;
  const double* lo = in.lo + phys_row(in, i) * cells;
  const double* hi = in.hi + phys_row(in, i) * cells;
  MagAcc mag;
  for (long long cell = blockIdx.x * blockDim.x + threadIdx.x; cell < cells;
       cell += (long long)gridDim.x * blockDim.x) {
    const Iv c{lo[cell], hi[cell]};
    Iv r = c;
    if (!iv_zero(c)) {
      const int cc = (int)(cell % f.C);
      const int x = (int)((cell / f.C) % f.S_w);
      const int y = (int)(cell / ((long long)f.C * f.S_w));
      const long long j = ((long long)(bh + y) * f.G_w + (bw + x)) * f.C + cc;
      const double* R = relax + 8 * j;
      const Iv alpha{R[0], R[1]}, gamma{R[4], R[5]};
      // stably positive (alpha = gamma = [1, 1]): every corner product c*1
      // is exact — for |c| at or above the reference's 2^-500 floor, below
      // which it widens anyway (interval.hpp:71-83) — so the map is the
      // identity on a coefficient with two nonzero ends (the straddling split
      // re-adds exact parts); anything else, including signed-zero ends,
      // takes the general map
      const bool ident = alpha.lo == 1.0 && alpha.hi == 1.0 && gamma.lo == 1.0 &&
                         gamma.hi == 1.0 && fabs(c.lo) >= kFloor && fabs(c.hi) >= kFloor;
      if (!ident) {
        const Iv sp = upper ? gamma : alpha;
        const Iv sn = upper ? alpha : gamma;
        bool bad = false;
        r = relu_map<true>(c, sp, sn, bad);
        if (bad) r = relu_map<false>(c, sp, sn, bad);
      }
    }
    out.lo[(size_t)i * cells + cell] = r.lo;
    out.hi[(size_t)i * cells + cell] = r.hi;
    mag.add(r.lo);
    mag.add(r.hi);
  }
  mag.flush(out.stat);
}

void launch_relu_coef(cudaStream_t s, const RowsDev& rows, const FrameDev& f, MatDev in,
                      MatDev out, const double* relax) {
  if (debug_skip("relu")) return;
  unsigned gx = cdiv(in.cells, 256);
  if (gx > 1024) gx = 1024;
  dim3 grid(gx, rows.n);
  k_relu_coef<<<grid, 256, 0, s>>>(rows, f, in, out, relax);
  ++g_launches;
}

// align_add / densify (backsub.hpp:578-688): union frame, branch a then b.
// dense_path mirrors the reference's densify branch: a's coefficients are
// copied (a dense from the start: verbatim; densified: zero cells -> +0)
// instead of accumulated into +0; the constants add K_b into K_a.
__global__ void __launch_bounds__(256)
    k_merge(RowsDev rows, FrameDev fa, FrameDev fb, FrameDev fu, int dense_path, MatDev a,
            MatDev b, MatDev out, int part) {
  int i;
  if (!rows_resolve(rows, blockIdx.y, i)) return;
  bool upper;
  const int q = row_query(rows, i, upper);
  int abw, abh, bbw, bbh, ubw, ubh;
  frame_base(fa, q, abw, abh);
  frame_base(fb, q, bbw, bbh);
  frame_base(fu, q, ubw, ubh);
  const long long cells = out.cells;
  const int C = fu.C;
  MagAcc mag;
  for (long long cell = blockIdx.x * blockDim.x + threadIdx.x; (part & 1) && cell < cells;
       cell += (long long)gridDim.x * blockDim.x) {
    const int cc = (int)(cell % C);
    const int x = (int)((cell / C) % fu.S_w);
    const int y = (int)(cell / ((long long)C * fu.S_w));
    const int aw = ubw + x, ah = ubh + y;
    Iv ca{0.0, 0.0}, cb{0.0, 0.0};
    bool ina = aw >= abw && aw < abw + fa.S_w && ah >= abh && ah < abh + fa.S_h;
    bool inb = aw >= bbw && aw < bbw + fb.S_w && ah >= bbh && ah < bbh + fb.S_h;
    if (ina) {
      const size_t o = phys_row(a, i) * a.cells + ((size_t)(ah - abh) * fa.S_w + (aw - abw)) * C + cc;
      ca = Iv{a.lo[o], a.hi[o]};
    }
    if (inb) {
      const size_t o = phys_row(b, i) * b.cells + ((size_t)(ah - bbh) * fb.S_w + (aw - bbw)) * C + cc;
      cb = Iv{b.lo[o], b.hi[o]};
    }
    Iv n{0.0, 0.0};
    if (dense_path == 2) n = ca;                    // a was dense: kept verbatim
    else if (dense_path == 1) { if (!iv_zero(ca)) n = ca; }  // densified a
    else iv_acc(n, ca);                              // union scatter
    iv_acc(n, cb);
    out.lo[(size_t)i * cells + cell] = n.lo;
    out.hi[(size_t)i * cells + cell] = n.hi;
    mag.add(n.lo);
    mag.add(n.hi);
  }
  if (part & 1) mag.flush(out.stat);
  if ((part & 2) && blockIdx.x == 0 && threadIdx.x == 0) {
    const double* Ka = a.K + 4 * phys_row(a, i);
    const double* Kb = b.K + 4 * phys_row(b, i);
    Iv k{Ka[0], Ka[1]}, kr{Ka[2], Ka[3]};
    iv_acc(k, Iv{Kb[0], Kb[1]});
    iv_acc(kr, Iv{Kb[2], Kb[3]});
    double* Ko = out.K + 4 * (size_t)i;
    Ko[0] = k.lo; Ko[1] = k.hi; Ko[2] = kr.lo; Ko[3] = kr.hi;
  }
}

void launch_merge(cudaStream_t s, const RowsDev& rows, const FrameDev& fa, const FrameDev& fb,
                  const FrameDev& fu, int dense_path, MatDev a, MatDev b, MatDev out, int part) {
  if (debug_skip("merge")) return;
  unsigned gx = (part & 1) ? cdiv(out.cells, 256) : 1;
  if (gx > 1024) gx = 1024;
  dim3 grid(gx, rows.n);
  k_merge<<<grid, (part & 1) ? 256 : 32, 0, s>>>(rows, fa, fb, fu, dense_path, a, b, out, part);
  ++g_launches;
}

// ===========================================================================
// Checkpoint bookkeeping: CandidateSet offers + freeze (backsub.hpp:798-817,
// 1036-1053) and the stable row compaction of compact_rows (:820-845) as a
// block scan producing the new row order.
// ===========================================================================
__global__ void __launch_bounds__(kScanThreads)
    k_offer(RowsDev rows, int R, const double* vals, const double* rvals, double* cand,
            char* frozen, int allow_freeze, int early_term, int* map, int* new_R,
            int* new_row_q, Counters* ctr, double* ckat, int ck_index) {
  using Scan = cub::BlockScan<int, kScanThreads>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int s_base;
  if (rows.dR) R = *rows.dR;  // device-driven walk: the live rows of this checkpoint
  if (threadIdx.x == 0) s_base = 0;
  int froze = 0;
  __syncthreads();
  for (int start = 0; start < R; start += kScanThreads) {
    const int r = start + threadIdx.x;
    int keep = 0, q = 0;
    if (r < R) {
      q = rows.row_q[r];  // a key (img * kq + neuron) in batched walks: cand / frozen are keyed alike
      double* cd = cand + 4 * (size_t)q;
      if (!frozen[q]) {
        const double v = vals[r], rv = rvals[r];  // offer_hi
        if (v < cd[1]) cd[1] = v;
        if (rv < cd[3]) cd[3] = rv;
        const double v2 = vals[R + r], rv2 = rvals[R + r];  // offer_lo
        if (v2 > cd[0]) cd[0] = v2;
        if (rv2 > cd[2]) cd[2] = rv2;
        if (allow_freeze && (!(cd[2] < 0.0) || !(cd[3] > 0.0))) {
          frozen[q] = 1;
          if (early_term) {
            ckat[q] = ck_index;  // the checkpoint that retires this row (k_ck_count)
            if (rows.kq) atomicAdd(&ctr[q / rows.kq].frozen, 1ull);
            else ++froze;
          }
        }
      }
      keep = !(early_term && frozen[q]);
    }
    int pos, total;
    Scan(tmp).ExclusiveSum(keep, pos, total);
    if (keep) {
      map[s_base + pos] = r;
      new_row_q[s_base + pos] = q;
    }
    __syncthreads();
    if (threadIdx.x == 0) s_base += total;
    __syncthreads();
  }
  if (froze) atomicAdd(&ctr->frozen, (unsigned long long)froze);
  const int nR = s_base;
  for (int p = threadIdx.x; p < nR; p += blockDim.x) map[nR + p] = R + map[p];  // lower rows
  if (threadIdx.x == 0) *new_R = nR;
}

void launch_offer(cudaStream_t s, const RowsDev& rows, int R, const double* vals,
                  const double* rvals, double* cand, char* frozen, int allow_freeze,
                  int early_term, int* map, int* new_R, int* new_row_q, Counters* ctr, double* ckat,
                  int ck_index) {
  k_offer<<<1, kScanThreads, 0, s>>>(rows, R, vals, rvals, cand, frozen, allow_freeze, early_term,
                                     map, new_R, new_row_q, ctr, ckat, ck_index);
  ++g_launches;
}

// Row sharding (engine.cu run_pass / run_margin). width doubles per row;
// live == nullptr: rows are identity-indexed.
__global__ void k_shard_pack(const int* live, int b, int cnt, int width, const double* src,
                             double* send) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= cnt * width) return;
  const int k = e / width, c = e % width;
  const int row = live ? live[b + k] : b + k;
  send[e] = src[(size_t)row * width + c];
}

__global__ void k_shard_unpack(const int* live, int n_live, int world, int per, int width,
                               const double* recv, double* dst) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)world * per * width) return;
  const int c = (int)(e % width);
  const long long rk = e / width;
  const int r = (int)(rk / per), k = (int)(rk % per);
  const int b = (int)((long long)n_live * r / world), nb = (int)((long long)n_live * (r + 1) / world);
  if (k >= nb - b) return;
  const int row = live ? live[b + k] : b + k;
  dst[(size_t)row * width + c] = recv[e];
}

void launch_shard_pack(cudaStream_t s, const int* live, int b, int cnt, int width,
                       const double* src, double* send) {
  if (cnt <= 0) return;
  k_shard_pack<<<cdiv((long long)cnt * width, 256), 256, 0, s>>>(live, b, cnt, width, src, send);
  ++g_launches;
}

void launch_shard_unpack(cudaStream_t s, const int* live, int n_live, int world, int per,
                         int width, const double* recv, double* dst) {
  k_shard_unpack<<<cdiv((long long)world * per * width, 256), 256, 0, s>>>(live, n_live, world, per,
                                                                          width, recv, dst);
  ++g_launches;
}

// PassStats.checkpoints as the reference counts it (backsub.hpp:1018-1063):
// the live rows of a pass are walked in chunks of `chunk` rows (its
// rows_per_chunk, from the memory budget; engine.cu ref_rows_per_chunk), and a
// chunk's walk runs checkpoints until its last row froze and was compacted
// (walk_back's rows() == 0 exit, :859) or the walk ends (T checkpoints). A
// row's freeze checkpoint (1-based, ckat; 0 = never froze) is chunk-invariant,
// so each chunk contributes the max over its rows. keys: the pass's live rows
// in the reference's order (image-major keys img * kq + neuron when batched;
// one block per image). all_full: no row ever leaves its walk early (early
// termination off, or the output pass).
__global__ void k_ck_fill(const int* keys, const int* n_keys, double* ckat) {
  const int n = *n_keys;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    ckat[keys[i]] = 0.0;
}

__device__ __forceinline__ int lower_bound_key(const int* keys, int n, long long v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (keys[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void k_ck_count(const int* keys, const int* n_keys, int kq, long long chunk, int T,
                           int all_full, const double* ckat, Counters* ctr) {
  const int n = *n_keys;
  const int b = blockIdx.x;
  const int lo = kq ? lower_bound_key(keys, n, (long long)b * kq) : 0;
  const int hi = kq ? lower_bound_key(keys, n, (long long)(b + 1) * kq) : n;
  const long long nchunks = hi > lo ? (hi - lo + chunk - 1) / chunk : 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  unsigned long long sum = 0;
  for (long long c = warp; c < nchunks; c += nwarps) {
    int mx = 0;
    if (all_full) {
      mx = T;
    } else {
      const long long e = min((long long)hi, lo + (c + 1) * chunk);
      for (long long i = lo + c * chunk + lane; i < e; i += 32) {
        const int v = (int)ckat[keys[i]];
        mx = max(mx, v == 0 ? T : v);
      }
      for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (lane == 0) sum += (unsigned long long)mx;
  }
  if (lane == 0 && sum) atomicAdd(&ctr[b].checkpoints, sum);
}

void launch_ck_fill(cudaStream_t s, const int* keys, const int* n_keys, int cap, double* ckat) {
  k_ck_fill<<<cdiv(cap > 0 ? cap : 1, 256) > 1024 ? 1024 : cdiv(cap > 0 ? cap : 1, 256), 256, 0, s>>>(keys, n_keys, ckat);
  ++g_launches;
}

void launch_ck_count(cudaStream_t s, const int* keys, const int* n_keys, int kq, int nimg,
                     long long chunk, int T, int all_full, const double* ckat, Counters* ctr) {
  k_ck_count<<<nimg, 256, 0, s>>>(keys, n_keys, kq, chunk, T, all_full, ckat, ctr);
  ++g_launches;
}

// Image-batched seed: per-image live lists (live + img * kq, counts n_live[img])
// concatenated into one key list (img * kq + neuron), image-major; total count.
constexpr int kGatherThreads = 256;
static_assert(kMaxBatch <= kGatherThreads, "one scan element per image");
__global__ void __launch_bounds__(kGatherThreads)
    k_gather_keys(const int* live, const int* n_live, int nimg, int kq, int* keys, int* total) {
  using Scan = cub::BlockScan<int, kGatherThreads>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int s_off[kMaxBatch + 1];
  const int t = threadIdx.x;
  const int cnt = t < nimg ? n_live[t] : 0;
  int off, all;
  Scan(tmp).ExclusiveSum(cnt, off, all);  // image-major offsets
  if (t < nimg) s_off[t] = off;
  if (t == 0) {
    s_off[nimg] = all;
    *total = all;
  }
  __syncthreads();
  // one warp per image (strided), lanes over its keys
  const int lane = t & 31, warp = t >> 5;
  for (int b = warp; b < nimg; b += kGatherThreads / 32) {
    const int o = s_off[b], n = s_off[b + 1] - o;
    for (int k = lane; k < n; k += 32) keys[o + k] = b * kq + live[(size_t)b * kq + k];
  }
}

void launch_gather_keys(cudaStream_t s, const int* live, const int* n_live, int nimg, int kq,
                        int* keys, int* total) {
  k_gather_keys<<<1, kGatherThreads, 0, s>>>(live, n_live, nimg, kq, keys, total);
  ++g_launches;
}

// Image-batched margin rows: row key img * kq + class j; +1 at labels[img].
__global__ void k_init_margin_keys(RowsDev rows, const int* labels, int n_out, MatDev out) {
  int i;
  if (!rows_resolve(rows, blockIdx.x, i)) return;
  bool upper;
  int img;
  const int j = row_query(rows, i, upper, img);
  const int label = labels[img];
  MagAcc mag;
  for (int c = threadIdx.x; c < n_out; c += blockDim.x) {
    const double v = (c == label) ? 1.0 : (c == j ? -1.0 : 0.0);
    out.lo[(size_t)i * n_out + c] = v;
    out.hi[(size_t)i * n_out + c] = v;
    mag.add(v);
  }
  mag.flush(out.stat);
  if (threadIdx.x < 4) out.K[4 * (size_t)i + threadIdx.x] = 0.0;
}

void launch_init_margin_keys(cudaStream_t s, const RowsDev& rows, const int* labels, int n_out,
                             MatDev out) {
  k_init_margin_keys<<<rows.n, 128, 0, s>>>(rows, labels, n_out, out);
  ++g_launches;
}

// run_margin_pass checkpoint (backsub.hpp:1082-1091): best = max.
__global__ void k_margin_offer(int n, const double* vals, double* best, char* has) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  if (!has[r] || vals[r] > best[r]) {
    best[r] = vals[r];
    has[r] = 1;
  }
}

void launch_margin_offer(cudaStream_t s, int n, const double* vals, double* best, char* has) {
  k_margin_offer<<<cdiv(n, 128), 128, 0, s>>>(n, vals, best, has);
  ++g_launches;
}

// One shared-memory carveout for every kernel of a walk: the coefficient and
// constants streams run concurrently, and an SM can only co-host CTAs of
// kernels whose carveout it is configured for; mixed carveouts force SMs to
// drain and reconfigure between them.
template <class K>
static void carve(K k) {
  cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}
void init_kernel_attrs_kernels() {
  carve(k_fwd_dense); carve(k_fwd_conv); carve(k_fwd_relu); carve(k_fwd_join); carve(k_relax);
  carve(k_seed); carve(k_writeback); carve(k_init_affine); carve(k_init_identity);
  carve(k_init_margin); carve(k_chain_affine); carve(k_chain_relu); carve(k_concretize);
  carve(k_dense_coef<1>); carve(k_dense_coef<2>); carve(k_dense_coef<3>);
  carve(k_dense_coef<4>); carve(k_dense_coef<8>); carve(k_gbc_coef); carve(k_compact_cells);
  {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    auto slots = [&](auto k, int tm, size_t smem, int nc = kDC) {
      int b = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k, nc, smem);
      g_dense_slots[tm] = b * sms;
    };
    g_dense_v2 = env_int("PC_DENSE_V2", 1);
    g_dense_live = env_int("PC_DENSE_LIVE", 1);
    auto big = [](auto k, size_t bytes) {
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
      carve(k);
    };
    big(k_dense_coef2<2, kDC>, sizeof(DenseSmem2<2, kDC>));
    big(k_dense_coef2<3, kDC>, sizeof(DenseSmem2<3, kDC>));
    big(k_dense_coef2<4, kDC>, sizeof(DenseSmem2<4, kDC>));
    big(k_dense_coef2<8, 64>, sizeof(DenseSmem2<8, 64>));
    g_dense_v3 = env_int("PC_DENSE_V3", 1);
    big(k_dense_coef3<2, kDC>, sizeof(DenseSmem2<2, kDC>) + 4 * kDMaxList);
    big(k_dense_coef3<3, kDC>, sizeof(DenseSmem2<3, kDC>) + 4 * kDMaxList);
    big(k_dense_coef3<4, kDC>, sizeof(DenseSmem2<4, kDC>) + 4 * kDMaxList);
    big(k_dense_coef3<8, 64>, sizeof(DenseSmem2<8, 64>) + 4 * kDMaxList);
    slots(k_dense_coef<1>, 1, 0);
    if (g_dense_v2) {
      slots(k_dense_coef2<2, kDC>, 2, sizeof(DenseSmem2<2, kDC>));
      slots(k_dense_coef2<3, kDC>, 3, sizeof(DenseSmem2<3, kDC>));
      slots(k_dense_coef2<4, kDC>, 4, sizeof(DenseSmem2<4, kDC>));
      slots(k_dense_coef2<8, 64>, 8, sizeof(DenseSmem2<8, 64>), 64);
    } else {
      slots(k_dense_coef<2>, 2, 0); slots(k_dense_coef<3>, 3, 0);
      slots(k_dense_coef<4>, 4, 0); slots(k_dense_coef<8>, 8, 0);
    }
    // Default 4: with several worker contexts per GPU the launches of other
    // streams fill a launch's last wave, so per-row efficiency wins over the
    // single-launch wave model (PC_DENSE_TM=-1).
    const int f = env_int("PC_DENSE_TM", 4);
    g_dense_tm = (f == 1 || f == 2 || f == 3 || f == 4 || f == 8) ? f : 0;
  }
  {
    // the sparse conv kernels use no shared memory; PC_GBC_L1=1 gives them
    // the largest L1 (weights are re-read by every position of a tap)
    const int l1 = env_int("PC_GBC_L1", 1) ? 0 : 100;
    cudaFuncSetAttribute(k_gbc_sparse, cudaFuncAttributePreferredSharedMemoryCarveout, l1);
    cudaFuncSetAttribute(k_gbc_sparse2<1>, cudaFuncAttributePreferredSharedMemoryCarveout, l1);
    cudaFuncSetAttribute(k_gbc_sparse2<2>, cudaFuncAttributePreferredSharedMemoryCarveout, l1);
    cudaFuncSetAttribute(k_gbc_sparse2<3>, cudaFuncAttributePreferredSharedMemoryCarveout, l1);
    cudaFuncSetAttribute(k_gbc_sparse2<4>, cudaFuncAttributePreferredSharedMemoryCarveout, l1);
  }
  carve(k_relu_coef); carve(k_merge); carve(k_offer); carve(k_shard_pack); carve(k_shard_unpack);
  carve(k_margin_offer); carve(k_margin_rows); carve(k_gather_keys); carve(k_init_margin_keys);
  carve(k_gbc_smem<1>); carve(k_gbc_smem<2>); carve(k_gbc_smem<4>); carve(k_gbc_smem<8>);
  cudaFuncSetAttribute(k_gbc_smem<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gbc_smem_bytes<1>());
  cudaFuncSetAttribute(k_gbc_smem<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gbc_smem_bytes<2>());
  cudaFuncSetAttribute(k_gbc_smem<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gbc_smem_bytes<4>());
  cudaFuncSetAttribute(k_gbc_smem<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gbc_smem_bytes<8>());
}

// input_box (network.hpp:160-177): iv_add(point(c), [-eps, eps]) then the
// optional [0, 1] clamp with std::max/std::min semantics.
__global__ void k_input_box(const double* c, int n, double eps, int clamp01, double* lo,
                            double* up) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double l = add_down(c[i], -eps), h = add_up(c[i], eps);
  if (clamp01) {
    l = smax(l, 0.0);
    h = smin(h, 1.0);
  }
  lo[i] = l;
  up[i] = h;
}

cudaError_t input_box_device(const double* center, int n, double eps, int clamp01, double* lo,
                             double* up) {
  double* d = nullptr;
  cudaError_t e = cudaMalloc(&d, sizeof(double) * 3 * (size_t)(n > 0 ? n : 1));
  if (e != cudaSuccess) return e;
  e = cudaMemcpy(d, center, sizeof(double) * n, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && n > 0) {
    k_input_box<<<cdiv(n, 256), 256>>>(d, n, eps, clamp01, d + n, d + 2 * (size_t)n);
    ++g_launches;
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpy(lo, d + n, sizeof(double) * n, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(up, d + 2 * (size_t)n, sizeof(double) * n, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return e;
}

// ===========================================================================
// Concrete forward evaluation (eval.hpp:39-102): round-to-nearest, bias first
// then ascending inputs, separate multiply and add roundings (no FMA), all
// weights including zeros. Used for the candidate label (tools/main.cpp:86-100).
// ===========================================================================
__global__ void k_eval_layer(LayerDev L, const double* x, const double* x2, double* y) {
  const long long n = (long long)L.out_w * L.out_h * L.out_c;
  const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  switch (L.kind) {
    case KIND_DENSE: {
      const int n_in = L.in_w * L.in_h * L.in_c;
      double acc = L.bias[j];
      for (int t = 0; t < n_in; ++t) acc = __dadd_rn(acc, __dmul_rn(L.WT[(size_t)t * n + j], x[t]));
      y[j] = acc;
      break;
    }
    case KIND_CONV: {
      const int d = (int)(j % L.out_c);
      const int w = (int)((j / L.out_c) % L.out_w);
      const int h = (int)(j / ((long long)L.out_c * L.out_w));
      double acc = L.bias[d];
      for (int fy = 0; fy < L.fh; ++fy) {
        const int iy = h * L.sh - L.ph + fy;
        if (iy < 0 || iy >= L.in_h) continue;
        for (int fx = 0; fx < L.fw; ++fx) {
          const int ix = w * L.sw - L.pw + fx;
          if (ix < 0 || ix >= L.in_w) continue;
          for (int ci = 0; ci < L.in_c; ++ci)
            acc = __dadd_rn(acc, __dmul_rn(L.F[((size_t)(fy * L.fw + fx) * L.in_c + ci) * L.out_c + d],
                                           x[((size_t)iy * L.in_w + ix) * L.in_c + ci]));
        }
      }
      y[j] = acc;
      break;
    }
    case KIND_RELU:
      y[j] = x[j] > 0.0 ? x[j] : 0.0;
      break;
    case KIND_JOIN:
      y[j] = __dadd_rn(x[j], x2[j]);
      break;
  }
}

void launch_eval_layer(cudaStream_t s, const LayerDev& L, const double* x, const double* x2,
                       double* y) {
  const long long n = (long long)L.out_w * L.out_h * L.out_c;
  k_eval_layer<<<cdiv(n, 128), 128, 0, s>>>(L, x, x2, y);
  ++g_launches;
}

// Numeric-core self test: one scalar op per element (0 add_down, 1 add_up,
// 2 mul_down, 3 mul_up, 4 div_down, 5 div_up, 6 ulp_above(a), 7 add_dir up,
// 8 add_dir down, 9 nextup_bits(a), 10 nextdown_bits(a)).
__global__ void k_scalar_ops(int op, const double* a, const double* b, double* out, long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double x = a[i], y = b[i];
  double r;
  switch (op) {
    case 0: r = add_down(x, y); break;
    case 1: r = add_up(x, y); break;
    case 2: r = mul_down(x, y); break;
    case 3: r = mul_up(x, y); break;
    case 4: r = div_down(x, y); break;
    case 5: r = div_up(x, y); break;
    case 6: r = ulp_above(x); break;
    case 7: r = add_dir(x, y, true); break;
    case 8: r = add_dir(x, y, false); break;
    case 9: r = nextup_bits(x); break;
    case 10: r = nextdown_bits(x); break;
    // band forms used by madd_band (valid for in-band operands only)
    case 11: { const double p = __dmul_rn(x, y); r = __dadd_rd(p, -fabs(__fma_rn(x, y, -p))); break; }
    case 12: { const double p = __dmul_rn(x, y); r = __dadd_ru(p, fabs(__fma_rn(x, y, -p))); break; }
    case 13: r = canon0(__fma_rd(__dsub_rn(__dadd_ru(x, y), __dadd_rd(x, y)), -0.5, __dadd_rn(x, y))); break;
    default: r = __fma_ru(__dsub_rn(__dadd_ru(x, y), __dadd_rd(x, y)), 0.5, __dadd_rn(x, y)); break;
  }
  out[i] = r;
}

cudaError_t scalar_ops_device(int op, const double* a, const double* b, double* out, long long n) {
  double* d = nullptr;
  cudaError_t e = cudaMalloc(&d, sizeof(double) * 3 * (size_t)(n > 0 ? n : 1));
  if (e != cudaSuccess) return e;
  e = cudaMemcpy(d, a, sizeof(double) * n, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d + n, b, sizeof(double) * n, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && n > 0) {
    k_scalar_ops<<<cdiv(n, 256), 256>>>(op, d, d + n, d + 2 * n, n);
    ++g_launches;
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpy(out, d + 2 * n, sizeof(double) * n, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return e;
}

// Chain-fold self test: chain c folds terms[c * len .. +len) into acc0[c]
// with add_up (up[c]) or add_down, by the warp scan of scanfold.cuh (the
// chain kernels' fold). One warp per chain.
__global__ void k_chain_fold(int n_chains, int len, const double* acc0, const double* terms,
                             const int* up, double* out) {
  const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= n_chains) return;
  const double* t = terms + (size_t)c * len;
  const bool dir = up[c] & 1;  // bit 1 set: the 32-link fold (scan_fold) instead of scan_fold4
  const double r = (up[c] & 2)   ? scan_fold(acc0[c], len, dir, [&](int j) { return t[j]; })
                   : (up[c] & 8) ? scan_fold4_pf(acc0[c], len, dir, t)
                                 : scan_fold4(acc0[c], len, dir, [&](int j) { return t[j]; });
  if ((threadIdx.x & 31) == 0) out[c] = r;
}

__global__ void __launch_bounds__(512) k_chain_fold_block(int len, const double* acc0, const double* terms,
                                                          const int* up, double* out) {
  __shared__ long long sm[2 * 512 / 32 + 8];
  const int c = blockIdx.x;
  const double* t = terms + (size_t)c * len;
  const double r = (up[c] & 16) ? block_scan_fold_rt<512>(acc0[c], len, (up[c] & 1) != 0, [&](int j) { return t[j]; }, sm)
                                : block_scan_fold<512>(acc0[c], len, (up[c] & 1) != 0, [&](int j) { return t[j]; }, sm);
  if (threadIdx.x == 0) out[c] = r;
}

cudaError_t scan_stats_device(int on, unsigned long long* out4) {
  cudaError_t e = cudaSuccess;
  if (out4) e = cudaMemcpyFromSymbol(out4, g_scan_stats, sizeof(unsigned long long) * 8);
  const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_scan_stats, z, sizeof(z));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_scan_stats_on, &on, sizeof(int));
  return e;
}

cudaError_t chain_fold_device(int n_chains, int len, const double* acc0, const double* terms,
                              const int* up, double* out) {
  const size_t nt = (size_t)n_chains * len;
  char* d = nullptr;
  const size_t bytes = 8 * (2 * (size_t)n_chains + nt) + 4 * (size_t)n_chains + 64;
  cudaError_t e = cudaMalloc(&d, bytes);
  if (e != cudaSuccess) return e;
  double* da = reinterpret_cast<double*>(d);
  double* dt = da + n_chains;
  double* dout = dt + nt;
  int* du = reinterpret_cast<int*>(dout + n_chains);
  e = cudaMemcpy(da, acc0, 8 * (size_t)n_chains, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && nt) e = cudaMemcpy(dt, terms, 8 * nt, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(du, up, 4 * (size_t)n_chains, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && n_chains > 0) {
    int u0 = 0;
    cudaMemcpy(&u0, du, sizeof(int), cudaMemcpyDeviceToHost);
    if (u0 & 4) k_chain_fold_block<<<n_chains, 512>>>(len, da, dt, du, dout);  // CTA-wide fold
    else k_chain_fold<<<cdiv(n_chains, 4), 128>>>(n_chains, len, da, dt, du, dout);
    ++g_launches;
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpy(out, dout, 8 * (size_t)n_chains, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return e;
}

}  // namespace pc

namespace pc {

// ---------------------------------------------------------------------------
// FP64 pipe peak (the roofline denominator of the FP64-bound kernels): every
// thread runs 8 independent register-resident DFMA chains; 4 blocks of 256
// threads per SM.
__global__ void __launch_bounds__(256) k_dfma_peak(double* out, double x, double y, int iters) {
  double a[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) a[u] = x + u + threadIdx.x;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = __fma_rn(a[u], x, y);
  double s = 0;
#pragma unroll
  for (int u = 0; u < 8; ++u) s += a[u];
  if (s == 12345.0) out[blockIdx.x] = s;  // keep the chains live
}

cudaError_t fp64_peak_device(double* fma_per_s) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out = nullptr;
  cudaError_t e = cudaMalloc(&out, sizeof(double) * 4 * sms);
  if (e != cudaSuccess) return e;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 1 << 14, blocks = 4 * sms;
  k_dfma_peak<<<blocks, 256>>>(out, 0.999999, 1e-7, iters);  // warm-up (clocks up)
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k_dfma_peak<<<blocks, 256>>>(out, 0.999999, 1e-7, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  e = cudaGetLastError();
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  *fma_per_s = (double)blocks * 256 * 8 * iters / (best * 1e-3);
  return e;
}

}  // namespace pc
