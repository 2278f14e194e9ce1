// kernels.cuh — device data structures and kernel launchers shared by the
// host engine (engine.cu) and the kernels (kernels.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace pc {

enum Kind { KIND_INPUT = 0, KIND_DENSE = 1, KIND_CONV = 2, KIND_RELU = 3, KIND_JOIN = 4 };

// Device-side view of one layer (immutable after pc_net_create).
struct LayerDev {
  int kind, pred0, pred1;
  int in_w, in_h, in_c, out_w, out_h, out_c;
  int fw, fh, sw, sh, pw, ph;
  const double* W;   // dense [out][in] (reference layout)
  const double* WT;  // dense [in][out] (forward kernel layout)
  const double* F;   // conv filter ((fy*fw+fx)*cin+ci)*cout+co (reference layout)
  const double* FT;  // conv filter ((fy*fw+fx)*cout+co)*cin+ci (back-substitution layout)
  const double* bias;
  double wmin, wmax;  // smallest / largest nonzero |weight| (1, 1 if none)
};

// A frame = which cells of a layer a bound matrix row stores.
//
// The reference stores per-row cuboid windows of unclamped width, with dead
// out-of-grid cells (backsub.hpp:85-96). Here every row stores only the
// in-grid STORAGE WINDOW of size S = min(W, G) per axis, based at
// clamp(origin, 0, G - S), so dense frames (S = G, base 0) and cuboid frames
// share one layout and deep residual frames never hold dead cells. Row origins
// are affine in the query neuron's grid position (origin = q_pos * M + A): the
// reference's recurrences (depsets.hpp:27-34) compose affinely, so the host
// tracks (M, A, W) symbolically and kernels derive each row's base on the fly.
// Cells inside the storage window but outside the row's true frame are kept
// exactly zero and zero coefficients are skipped everywhere, as dead cells are
// in the reference; cell order within the window is (y, x, c), i.e. ascending
// absolute order, which is the reference's accumulation order.
struct FrameDev {
  int G_w, G_h, C;           // layer grid
  int S_w, S_h;              // storage window (cells per row = S_w*S_h*C)
  long long M_w, M_h, A_w, A_h;
  int q_w, q_c;              // query layer width / channels (decode row query index)
};

__host__ __device__ inline long long frame_cells(const FrameDev& f) {
  return (long long)f.S_w * f.S_h * f.C;
}

__device__ __forceinline__ void frame_base(const FrameDev& f, int q, int& bw, int& bh) {
  const int qw = (q / f.q_c) % f.q_w;
  const int qh = q / (f.q_c * f.q_w);
  long long ow = (long long)qw * f.M_w + f.A_w;
  long long oh = (long long)qh * f.M_h + f.A_h;
  const long long mw = f.G_w - f.S_w, mh = f.G_h - f.S_h;
  ow = ow < 0 ? 0 : (ow > mw ? mw : ow);
  oh = oh < 0 ? 0 : (oh > mh ? mh : oh);
  bw = (int)ow;
  bh = (int)oh;
}

// Row set of a bound matrix: rows [0, n_up) are upper-polarity rows for
// queries row_q[0..n_up), rows [n_up, n) lower rows for row_q[i - n_up]
// (margin passes: n_up = 0). Coefficients are SoA planes lo[n][cells],
// hi[n][cells]; K[n][4] = {k.lo, k.hi, kraw.lo, kraw.hi}.
// src (nullable): after an early-termination compaction the surviving rows
// are not moved; logical row i lives at physical row src[i] until the next
// step consumes the matrix and writes a compact output.
struct MatDev {
  double* lo;
  double* hi;
  double* K;
  long long cells;
  const int* src = nullptr;
  // Magnitude statistics of the nonzero coefficients (see MagStat below);
  // written by the kernel that produces the matrix, read by its consumer.
  unsigned* stat = nullptr;
};

// ---------------------------------------------------------------------------
// Magnitude statistics. key(x) = high 32 bits of |x| (exponent and top 20
// mantissa bits), so keys order like magnitudes. stat[0] = min key over the
// nonzero entries, stat[1] = ~(max key); both are reduced with atomicMin from
// an initial 0xFFFFFFFF. A consumer proves from them (and the layer's weight
// range) that every nonzero product |c*w| lies in [2^-499, 2^999]; then the
// reference's exactness tests reduce to residual == 0 / RD == RU and the lean
// "band" multiply-add below is bit-identical to the exact ops.
struct MagAcc {
  unsigned kmin = 0xFFFFFFFFu, kmaxinv = 0xFFFFFFFFu;
  __device__ __forceinline__ void add(double x) {
    const unsigned hi = (unsigned)__double2hiint(x) & 0x7FFFFFFFu;
    if (hi | (unsigned)__double2loint(x)) {
      kmin = min(kmin, hi);
      kmaxinv = min(kmaxinv, ~hi);
    }
  }
  // Warp-reduce, then one shared-memory atomic per warp (block-level stat).
  __device__ __forceinline__ void flush_shared(unsigned* s_stat) {
    const unsigned mask = __activemask();
    const unsigned a = __reduce_min_sync(mask, kmin), b = __reduce_min_sync(mask, kmaxinv);
    if ((threadIdx.x & 31) == (unsigned)(__ffs(mask) - 1)) {
      atomicMin(s_stat, a);
      atomicMin(s_stat + 1, b);
    }
  }
  // Warp-reduce over the lanes that reach this call, one atomic per warp.
  __device__ __forceinline__ void flush(unsigned* stat) {
    if (!stat) return;
    const unsigned mask = __activemask();
    const unsigned a = __reduce_min_sync(mask, kmin), b = __reduce_min_sync(mask, kmaxinv);
    if ((threadIdx.x & 31) == (unsigned)(__ffs(mask) - 1) && (a != 0xFFFFFFFFu || b != 0xFFFFFFFFu)) {
      // The stats only decrease, so a value already <= ours needs no atomic:
      // after the first warps, most of a launch's thousands of warps skip
      // them (same-address atomics serialise in L2).
      if (a < *(volatile const unsigned*)stat) atomicMin(stat, a);
      if (b < *(volatile const unsigned*)(stat + 1)) atomicMin(stat + 1, b);
    }
  }
};

__device__ __forceinline__ bool products_in_band(const unsigned* stat, double wmin, double wmax) {
  if (!stat) return false;
  const unsigned kmin = stat[0], kmax = ~stat[1];
  if (kmin == 0xFFFFFFFFu) return true;  // no nonzero coefficient: every product is 0
  const double cmin = __hiloint2double((int)kmin, 0);           // <= min |c|
  const double cmax = __hiloint2double((int)kmax, (int)0xFFFFFFFFu);  // >= max |c|
  return __dmul_rn(cmin, wmin) >= 0x1p-499 && __dmul_rn(cmax, wmax) <= 0x1p999;
}

// interval += c * w (backsub.hpp:385 / :481-482) for in-band operands (see
// products_in_band), accumulators starting at +0 and fewer than 2^20 terms:
// bit-identical to add_down(lo, mul_down(.)) / add_up(hi, mul_up(.)) with the
// reference's zero skips (a zero factor adds an exact +-0, a no-op because the
// accumulators are never -0). Exactness tests are the residual (integer test
// on its bits) and RD == RU; outward steps are predicated.
__device__ __forceinline__ bool bits_zero(double x) {
  return (((unsigned)__double2hiint(x) << 1) | (unsigned)__double2loint(x)) == 0u;
}
// Outward steps without compares or selects (valid in the band):
//  * product: with RN product p and exact residual r = a*w - p (FMA),
//    0 < |r| <= ulp(p)/2 when inexact, so RD(p - |r|) = nextafter(p, -inf)
//    and RU(p + |r|) = nextafter(p, +inf); r = 0 leaves p (the reference's
//    "exact iff residual == 0", interval.hpp:71-83);
//  * sum: with s = RN, d = RD, u = RU of a + b, t = u - d is 0 (exact) or one
//    ulp, so RD(s - t/2) = nextafter(s, -inf) and RU(s + t/2) =
//    nextafter(s, +inf) when inexact and s otherwise (interval.hpp:59-68).
//    The lower form can turn an exact +0 into -0; value-equal, and the
//    accumulators are canonicalised (+0) when stored.
__device__ __forceinline__ void madd_band(double w, double cl, double ch, double& lo, double& hi) {
  const bool neg = __double2hiint(w) < 0;
  const double a = neg ? ch : cl, b = neg ? cl : ch;
  const double pl0 = __dmul_rn(a, w), ph0 = __dmul_rn(b, w);
  const double pl = __dadd_rd(pl0, -fabs(__fma_rn(a, w, -pl0)));
  const double ph = __dadd_ru(ph0, fabs(__fma_rn(b, w, -ph0)));
  const double sl = __dadd_rn(lo, pl), dl = __dadd_rd(lo, pl), ul = __dadd_ru(lo, pl);
  const double sh = __dadd_rn(hi, ph), dh = __dadd_rd(hi, ph), uh = __dadd_ru(hi, ph);
  lo = __fma_rd(__dsub_rn(ul, dl), -0.5, sl);
  hi = __fma_ru(__dsub_rn(uh, dh), 0.5, sh);
}
// Fast numeric mode (pc_options.numeric_mode = 1): the interval
// multiply-add as two directed-rounding FMAs, RD for the lower end and RU for
// the upper — each the correctly rounded exact result, so sound (outward) but
// not the reference's RN-then-step bits. Zero terms add exactly nothing.
__device__ __forceinline__ void madd_dir(double w, double cl, double ch, double& lo, double& hi) {
  const bool neg = __double2hiint(w) < 0;
  lo = __fma_rd(neg ? ch : cl, w, lo);
  hi = __fma_ru(neg ? cl : ch, w, hi);
}
// madd_band split into its accumulator-independent products and the two
// accumulator steps, for kernels that schedule the products of several terms
// ahead of the (latency-bound) sum chains.
__device__ __forceinline__ void band_products(double w, double cl, double ch, double& pl,
                                              double& ph) {
  const bool neg = __double2hiint(w) < 0;
  const double a = neg ? ch : cl, b = neg ? cl : ch;
  const double pl0 = __dmul_rn(a, w), ph0 = __dmul_rn(b, w);
  pl = __dadd_rd(pl0, -fabs(__fma_rn(a, w, -pl0)));
  ph = __dadd_ru(ph0, fabs(__fma_rn(b, w, -ph0)));
}
// band_products with the factors already ordered by the weight's sign
// (a multiplies into the lower bound, b into the upper).
__device__ __forceinline__ void band_products_ab(double w, double a, double b, double& pl,
                                                 double& ph) {
  const double pl0 = __dmul_rn(a, w), ph0 = __dmul_rn(b, w);
  pl = __dadd_rd(pl0, -fabs(__fma_rn(a, w, -pl0)));
  ph = __dadd_ru(ph0, fabs(__fma_rn(b, w, -ph0)));
}
__device__ __forceinline__ void band_sums(double pl, double ph, double& lo, double& hi) {
  const double sl = __dadd_rn(lo, pl), dl = __dadd_rd(lo, pl), ul = __dadd_ru(lo, pl);
  const double sh = __dadd_rn(hi, ph), dh = __dadd_rd(hi, ph), uh = __dadd_ru(hi, ph);
  lo = __fma_rd(__dsub_rn(ul, dl), -0.5, sl);
  hi = __fma_ru(__dsub_rn(uh, dh), 0.5, sh);
}
// Same result as madd_band with a shorter dependency chain through the
// accumulators (2 FP64 latencies + a select instead of 3): for latency-bound
// chains with little independent work per thread.
__device__ __forceinline__ void madd_band_lat(double w, double cl, double ch, double& lo,
                                              double& hi) {
  const bool neg = __double2hiint(w) < 0;
  const double a = neg ? ch : cl, b = neg ? cl : ch;
  const double pl0 = __dmul_rn(a, w), ph0 = __dmul_rn(b, w);
  const double pl = __dadd_rd(pl0, -fabs(__fma_rn(a, w, -pl0)));
  const double ph = __dadd_ru(ph0, fabs(__fma_rn(b, w, -ph0)));
  const double sl = __dadd_rn(lo, pl), sh = __dadd_rn(hi, ph);
  const bool xl = __dadd_rd(lo, pl) == __dadd_ru(lo, pl), xh = __dadd_rd(hi, ph) == __dadd_ru(hi, ph);
  const double tl = __dadd_rd(sl, -4.9406564584124654e-324), th = __dadd_ru(sh, 4.9406564584124654e-324);
  lo = xl ? sl : tl;
  hi = xh ? sh : th;
}

// cp.async (sm_80+): 8-byte global -> shared copies, zero-filled when !valid.
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 8 : 0;  // src-size 0: zero fill
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }
__device__ __forceinline__ void cp_async_wait_one() { asm volatile("cp.async.wait_group 1;\n" ::); }

// -0 -> +0 (RN: -0 + +0 = +0), everything else unchanged.
__device__ __forceinline__ double canon0(double x) { return __dadd_rn(x, 0.0); }

__host__ __device__ __forceinline__ size_t phys_row(const MatDev& m, int i) {
  return (size_t)(m.src ? m.src[i] : i);
}

struct RowsDev {
  const int* row_q;
  int n;     // total rows (launch bound when dR is set)
  int n_up;  // upper rows come first (launch bound when dR is set)
  // Device-driven walks (graph mode): the live rows per polarity are read from
  // device memory (written by the pass seed and by each checkpoint's offers);
  // launches are sized for the bound above and surplus blocks exit.
  const int* dR = nullptr;
  // Image-batched walks: row_q holds keys img * kq + q; per-neuron state
  // arrays (bounds, deviations, relaxations) are strided by sst per image,
  // candidate / freeze arrays by kq, counters by one Counters. kq = 0: one image.
  int kq = 0;
  long long sst = 0;
  int nimg = 1;
};
constexpr int kMaxBatch = 128;  // images per batched walk

// Resolve the block-row index b of a launch into logical row i of the rows
// actually live (upper rows [0, R), lower rows [R, 2R)); false: no such row.
// Updates r.n / r.n_up to the live values.
__device__ __forceinline__ bool rows_resolve(RowsDev& r, int b, int& i) {
  if (!r.dR) {
    i = b;
    return b < r.n;
  }
  const int R = *r.dR;
  if (r.n_up == 0) {  // one polarity (margin rows)
    r.n = R;
    i = b;
    return b < R;
  }
  const int Rmax = r.n_up;
  r.n = 2 * R;
  r.n_up = R;
  if (b < Rmax) {
    i = b;
    return b < R;
  }
  i = R + (b - Rmax);
  return b - Rmax < R;
}

__device__ __forceinline__ int row_query(const RowsDev& r, int i, bool& upper, int& img) {
  upper = i < r.n_up;
  const int key = r.row_q[upper ? i : i - r.n_up];
  img = r.kq ? key / r.kq : 0;
  return r.kq ? key - img * r.kq : key;
}
__device__ __forceinline__ int row_query(const RowsDev& r, int i, bool& upper) {
  int img;
  return row_query(r, i, upper, img);
}

struct Counters {  // device-side PassStats accumulators
  unsigned long long dense_madds;
  unsigned long long gbc_madds;
  unsigned long long frozen;  // rows_terminated_early (checkpoint freezes)
  unsigned long long pad;
  unsigned long long gbc_dense_equiv;
  unsigned long long checkpoints;  // non-margin checkpoints the reference would run
  unsigned long long conv_exec;    // interval madds executed by k_gbc_live (live cells only)
};

// Timing ablation (PC_DEBUG_SKIP=conv,folds,relu,merge,forward): the named
// kernels are not launched. Results are WRONG; only for attributing the
// critical path (with early termination off the work does not depend on
// the values). Never set in tests or the bench.
bool debug_skip(const char* what);

// ----- launchers (kernels.cu) -----
// Forward bounds of layer k (padded + raw + dev + relaxation), skipping
// neurons whose inputs did not change in refresh round g (force: all).
void launch_forward_layer(cudaStream_t s, const LayerDev& L, int feeds_relu, const double* blo,
                          const double* bhi, const double* rlo, const double* rhi,
                          const long long* offs, const long long* pofs, int k, int pred0,
                          int pred1, double* dev, double* relax, int* gen_n, int* gen_pos,
                          int* gen_l, int g, int force, int nimg = 1, long long zs = 0,
                          long long zp = 0, int zl = 0);  // nimg images (blockIdx.z), strided
void launch_relax(cudaStream_t s, const double* blo, const double* bhi, long long n, double* relax);

void launch_seed(cudaStream_t s, int n, const double* blo, const double* bhi, const double* rlo,
                 const double* rhi, int allow_freeze, int early_term, double* cand, char* frozen,
                 int* live, int* n_live, unsigned long long* n_prefrozen, int nimg = 1,
                 long long sst = 0, long long kq = 0, int pstride = 0);
void launch_writeback(cudaStream_t s, int n, int C, int layer, const double* cand, double* blo,
                      double* bhi, double* rlo, double* rhi, double* relax, int* gen_n,
                      int* gen_pos, int* gen_l, int g, long long gofs, long long pofs,
                      int nimg = 1, long long zs = 0, long long zp = 0, int zl = 0,
                      long long kq = 0);

void launch_init_affine(cudaStream_t s, const LayerDev& Q, const RowsDev& rows, const FrameDev& f,
                        const double* dev_q, MatDev out);
void launch_init_identity(cudaStream_t s, const RowsDev& rows, const FrameDev& f, MatDev out);
void launch_init_margin(cudaStream_t s, int label, const int* d_label, int n_out, int first,
                        int count, MatDev out);
void launch_margin_rows(cudaStream_t s, const int* d_label, int n_out, int* row_q);
void launch_gather_keys(cudaStream_t s, const int* live, const int* n_live, int nimg, int kq,
                        int* keys, int* total);
void launch_init_margin_keys(cudaStream_t s, const RowsDev& rows, const int* labels, int n_out,
                             MatDev out);

// Chains read the constants of m (through m.src) and write compact ones to Kout.
// frozen (nullable): rows whose query neuron froze at an earlier checkpoint
// are skipped — the reference has compacted them away by then (early
// termination, backsub.hpp:1040-1054); their results are never read.
// fast: the fast numeric mode (directed-rounding terms and folds) where the
// long-row kernels run; every other path stays exact (also sound).
void launch_chain_affine(cudaStream_t s, const LayerDev& L, bool is_conv, const RowsDev& rows,
                         const FrameDev& fin, MatDev m, double* Kout, const double* dev,
                         Counters* ctr, const char* frozen, bool fast = false);
void launch_chain_relu(cudaStream_t s, const RowsDev& rows, const FrameDev& f, MatDev m,
                       double* Kout, const double* relax, const char* frozen);
void launch_concretize(cudaStream_t s, const RowsDev& rows, const FrameDev& f, MatDev m,
                       const double* blo, const double* bhi, const double* rlo,
                       const double* rhi, double* vals, double* rvals, const char* frozen,
                       bool fast = false);

// Long-row variants (chains.cu): one CTA per row, producer warps compact the
// contributing terms, one consumer warp folds them in order.
void launch_chain_affine_big(cudaStream_t s, const LayerDev& L, bool is_conv, const RowsDev& rows,
                             const FrameDev& fin, MatDev m, double* Kout, const double* dev,
                             Counters* ctr, const char* frozen, bool fast = false);
void launch_chain_relu_big(cudaStream_t s, const RowsDev& rows, const FrameDev& f, MatDev m,
                           double* Kout, const double* relax, const char* frozen);
void launch_concretize_big(cudaStream_t s, const RowsDev& rows, const FrameDev& f, MatDev m,
                           const double* blo, const double* bhi, const double* rlo,
                           const double* rhi, double* vals, double* rvals, const char* frozen,
                           bool fast = false);
// Rows at least this long use the CTA-per-row chains (env PC_BIG_CHAIN_CELLS
// overrides, read once; the tests force 1 to run the corpus through them).
long long big_chain_cells();

// relax: relaxations of the ReLU whose output is the frame after this step
// (per image, strided by rows.sst), or nullptr: see dense_live_cols.
// Executed dense madds since the last reset (device counter; synchronous).
unsigned long long dense_useful_madds(bool reset);
void launch_dense_coef(cudaStream_t s, const LayerDev& L, const RowsDev& rows, MatDev in,
                       MatDev out, const double* relax, cudaEvent_t ev0, cudaEvent_t ev1);
// Compacted nonzero coefficients of a conv step's input, per frame cell of
// each (logical) row: cnt[row*ncell + cell] entries, channel idx and values
// at ((row*ncell + cell)*C + k), ascending channel.
struct SparseDev {
  int* cnt;
  unsigned short* idx;
  double* lo;
  double* hi;
  int ncell, C;
  unsigned* dmask = nullptr;  // optional: per row, the channels nonzero in any cell (16 words)
};
void launch_compact_cells(cudaStream_t s, const RowsDev& rows, MatDev m, SparseDev sp);
// Live channels per grid position of a ReLU layer (k_live_build, kernels.cu):
// cnt at the layer's position offset, idx at its neuron offset; strided per
// image by pst / sst.
struct LiveDev {
  const int* cnt;
  const unsigned short* idx;
  long long pst, sst;
};
void launch_live_build(cudaStream_t s, int npos, int C, const double* relax, const double* blo,
                       const double* bhi, const double* rlo, const double* rhi, int* cnt,
                       unsigned short* idx, int nimg, long long sst, long long pst,
                       unsigned* chmask = nullptr, int mstride = 0);  // chmask: live-anywhere channels
// Ascending list of the neurons of a ReLU layer with a nonzero relaxation
// offset (k_offset_list) and the relu_step constant chains over it.
void launch_offset_list(cudaStream_t s, int n, const double* relax, int* list, int* count,
                        int nimg, long long sst, int cstride);
void launch_chain_relu_list(cudaStream_t s, const RowsDev& rows, const FrameDev& f, MatDev m,
                            double* Kout, const double* relax, const int* list, const int* count,
                            int cstride, const char* frozen);
// The live cells of a ReLU layer as one flat list (k_live_flat): pref per
// grid position (npos + 1 entries), position / channel per live cell.
struct FlatDev {
  const int* pref;
  const unsigned short* fpos;
  const unsigned short* fch;
  long long fst, sst;  // per-image strides of pref and of fpos / fch
  // predicted compaction (optional): the output frame layer's raw bounds;
  // each block writes the (sum, sum of magnitudes, count) of its outputs'
  // raw concretisation corner terms to part[(row * gridDim.x + block) * 3]
  const double* prlo = nullptr;
  const double* prhi = nullptr;
  double* part = nullptr;
  int opb = 512;  // live cells per block (set by launch_gbc_flat)
};
void launch_live_flat(cudaStream_t s, int npos, int C, const int* cnt, const unsigned short* idx,
                      int* pref, unsigned short* fpos, unsigned short* fch, int nimg, long long sst,
                      long long pst, long long fst);
int gbc_flat_blocks(const FrameDev& fout, const LayerDev& L);  // blocks per row of k_gbc_flat
void launch_gbc_flat(cudaStream_t s, const LayerDev& L, const RowsDev& rows, const FrameDev& fin,
                     const FrameDev& fout, SparseDev sp, MatDev in, MatDev out, FlatDev fl, Counters* ctr,
                     bool fast = false);
// CTA-per-chain scan-fold kernels (chains.cu): the conv steps' constant
// chains from the compacted coefficients (tmp: 5 doubles per row), the
// checkpoints' concretisations.
void launch_chain_affine_scan(cudaStream_t s, const LayerDev& L, const RowsDev& rows, const FrameDev& fin,
                              MatDev m, SparseDev sp, double* tmp, double* Kout, const double* dev,
                              Counters* ctr, const char* frozen);
void launch_concretize_scan(cudaStream_t s, const RowsDev& rows, const FrameDev& f, MatDev m,
                            const double* blo, const double* bhi, const double* rlo, const double* rhi,
                            double* vals, double* rvals, const char* frozen);
// Predicted compaction (chains.cu): rows whose raw concretisation provably
// freezes them at this checkpoint (parallel sum + rigorous bound on the
// reference chain's distance from it) are dropped; map / new_R / new_row_q
// like launch_offer's.
// P (nullable): the predicted raw constants (S, E) per physical row, else m.K.
void launch_pred_offer(cudaStream_t s, const RowsDev& rows, int R, const FrameDev& f, MatDev m,
                       const double* P, const double* rlo, const double* rhi, const char* frozen, int* map,
                       int* new_R, int* new_row_q);
void launch_pred_offer_parts(cudaStream_t s, const RowsDev& rows, int R, MatDev m, const double* P,
                             const double* part, int nparts, const char* frozen, int* map, int* new_R,
                             int* new_row_q);
// Predicted raw constants (chains.cu): (S, E) per row, |chain value - S| <= E;
// Pin read through the input matrix's row map, Pout compact.
void launch_pk_affine(cudaStream_t s, const LayerDev& L, bool is_conv, const RowsDev& rows, const FrameDev& f,
                      MatDev m, const double* Pin, double* Pout);
void launch_pk_relu(cudaStream_t s, const RowsDev& rows, const FrameDev& f, MatDev m, const double* Pin,
                    double* Pout, const double* relax, const int* list, const int* count, int cstride);
void launch_pk_merge(cudaStream_t s, const RowsDev& rows, MatDev a, const double* Pa, MatDev b, const double* Pb,
                     double* Pout);
void launch_pk_init(cudaStream_t s, const RowsDev& rows, MatDev m, double* P);
// PassStats dense_madds / gbc_madds / gbc_dense_equiv of an affine step for
// the rows not frozen (the chain kernels' counting, run behind the exact offers)
void launch_count_affine(cudaStream_t s, const LayerDev& L, bool is_conv, const RowsDev& rows, const FrameDev& f,
                         MatDev m, const char* frozen, Counters* ctr);
// Dense-tile conv over the row's nonzero input channels x the layer's
// live-anywhere output channels (needs sp.dmask; chmask per image, 16 words).
void launch_gbc_tile(cudaStream_t s, const LayerDev& L, const RowsDev& rows, const FrameDev& fin,
                     const FrameDev& fout, SparseDev sp, MatDev in, MatDev out, const unsigned* chmask,
                     long long mstride, Counters* ctr);
// Conv coefficients of the live cells of a ReLU frame (dead ones written +0).
void launch_gbc_live(cudaStream_t s, const LayerDev& L, const RowsDev& rows, const FrameDev& fin,
                     const FrameDev& fout, SparseDev sp, MatDev in, MatDev out, LiveDev lv, Counters* ctr);
// Conv coefficients from the compacted input (band path; falls back to the
// checked gather on `in` when the launch's operands are not proven in band).
void launch_gbc_sparse(cudaStream_t s, const LayerDev& L, const RowsDev& rows, const FrameDev& fin,
                       const FrameDev& fout, SparseDev sp, MatDev in, MatDev out);
bool gbc_sparse_wanted(const LayerDev& L);
// queue: a device int the work-queue variant resets and consumes (per stream).
void launch_gbc_coef(cudaStream_t s, const LayerDev& L, const RowsDev& rows, const FrameDev& fin,
                     const FrameDev& fout, MatDev in, MatDev out, int* queue);
void launch_gbc_tile(cudaStream_t s, const LayerDev& L, const RowsDev& rows, const FrameDev& fin,
                     const FrameDev& fout, MatDev in, MatDev out);
// Engine switches from the environment (read once): PC_GBC selects the conv
// kernel: 3 (default) sparse gather where >= 32 channels, 2 shared-memory
// tiled, 1 register-blocked gather, 0 one output per thread.
int env_int(const char* name, int dflt);
void launch_relu_coef(cudaStream_t s, const RowsDev& rows, const FrameDev& f, MatDev in,
                      MatDev out, const double* relax);
void launch_merge(cudaStream_t s, const RowsDev& rows, const FrameDev& fa, const FrameDev& fb,
                  const FrameDev& fu, int dense_path, MatDev a, MatDev b, MatDev out,
                  int part);  // part: 1 coefficients, 2 constants, 3 both

// Offers + freeze; writes the compaction map (2 * new_R entries: upper then
// lower physical rows) and the compacted query list.
void launch_offer(cudaStream_t s, const RowsDev& rows, int R, const double* vals,
                  const double* rvals, double* cand, char* frozen, int allow_freeze,
                  int early_term, int* map, int* new_R, int* new_row_q, Counters* ctr, double* ckat,
                  int ck_index);  // ckat[q] = ck_index when row q freezes
// PassStats.checkpoints of a pass under the reference's chunking (kernels.cu).
void launch_ck_fill(cudaStream_t s, const int* keys, const int* n_keys, int cap, double* ckat);
void launch_ck_count(cudaStream_t s, const int* keys, const int* n_keys, int kq, int nimg,
                     long long chunk, int T, int all_full, const double* ckat, Counters* ctr);
void launch_margin_offer(cudaStream_t s, int n, const double* vals, double* best, char* has);

// Row sharding: pack this rank's slice of candidates (4 doubles per row, in
// live order) / scatter every rank's slice back into cand.
void launch_shard_pack(cudaStream_t s, const int* live, int b, int cnt, int width,
                       const double* src, double* send);
void launch_shard_unpack(cudaStream_t s, const int* live, int n_live, int world, int per,
                         int width, const double* recv, double* dst);

cudaError_t input_box_device(const double* center, int n, double eps, int clamp01, double* lo,
                             double* up);

void launch_eval_layer(cudaStream_t s, const LayerDev& L, const double* x, const double* x2,
                       double* y);

cudaError_t scalar_ops_device(int op, const double* a, const double* b, double* out, long long n);
cudaError_t fp64_peak_device(double* fma_per_s);
cudaError_t scan_stats_device(int on, unsigned long long* out4);         // kernels.cu's folds
cudaError_t scan_stats_device_chains(int on, unsigned long long* out4);  // chains.cu's folds
cudaError_t chain_fold_device(int n_chains, int len, const double* acc0, const double* terms,
                              const int* up, double* out);

extern thread_local long long g_launches;

// Per-kernel attributes (shared-memory carveout, dynamic smem limits), once per process.
void init_kernel_attrs_kernels();
void init_kernel_attrs_chains();
void init_kernel_attrs_gbc();
// Call with the device current (attributes are per device); idempotent.
void init_kernel_attrs(int device);

}  // namespace pc
