// gbc.cu — conv back-substitution coefficients (gbc_step, backsub.hpp:401-499),
// register-blocked gather form.
//
// Output coefficient (iy, ix, ci) of the new frame = sum over the frame cells
// (ah, aw) whose filter window covers (iy, ix), ascending (ah, aw), and over
// ascending output channel d, of c[ah][aw][d] * filter[fy][fx][ci][d] — the
// reference's accumulation order (its scatter loop visits (ch, cw, d)
// lexicographically, :449-485). No split-K.
//
// Blocking: a thread owns P output positions of one output row that share a
// stride-parity class ((ix + pw) mod sw), so they see the same taps in the same
// order and consecutive covering cells aw0 + k, times Q consecutive input
// channels ci. Per (tap, d) it loads P coefficient intervals and Q weights and
// runs P*Q independent interval chains (ILP), each in the reference order.
// Lanes of a warp take consecutive ci groups, so coefficient loads are
// broadcasts and weight loads coalesce. A d whose P coefficients are all zero
// is skipped: adding the zero interval is a no-op in the reference (iv_acc
// skips it) and here (the accumulators are never -0).
#include "kernels.cuh"
#include "numeric.cuh"

namespace pc {

constexpr int kGP = 4;  // positions per thread
constexpr int kGQ = 2;  // input channels per thread

__device__ __forceinline__ int fdiv(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

__device__ __forceinline__ void madd_f(double w, double clo, double chi, double& lo, double& hi,
                                       bool& bad) {
  const bool skip = (w == 0.0) | ((clo == 0.0) & (chi == 0.0));
  const bool pos = w > 0.0;
  const double a = pos ? clo : chi, b = pos ? chi : clo;
  const double pl = f_mul_dn(a, w, bad), ph = f_mul_up(b, w, bad);
  const double nl = f_add_dn(lo, pl), nh = f_add_up(hi, ph);
  lo = skip ? lo : nl;
  hi = skip ? hi : nh;
}

__device__ __forceinline__ void madd_x(double w, double clo, double chi, double& lo, double& hi) {
  if (w == 0.0 || (clo == 0.0 && chi == 0.0)) return;
  const double a = w > 0.0 ? clo : chi, b = w > 0.0 ? chi : clo;
  lo = add_down(lo, mul_down(a, w));
  hi = add_up(hi, mul_up(b, w));
}

// Geometry of one row-task decomposition (host-computed, uniform per launch).
struct GbcGeom {
  int cin, cout, fw, fh, sw, sh, pw, ph;
  int Si_w, Si_h;   // input (frame) window
  int So_w, So_h;   // output window
  int nq;           // ci groups = ceil(cin / Q)
  int ncls_x;       // position groups per output row (over all parity classes)
  long long tasks;  // per row = So_h * ncls_x * nq
};

template <bool FAST>
__device__ __forceinline__ bool gbc_task(const GbcGeom& g, const double* __restrict__ FT,
                                         const double* __restrict__ ilo,
                                         const double* __restrict__ ihi, int bw, int bh, int iy,
                                         int ix0, int npos, int ci0, double (&lo)[kGP][kGQ],
                                         double (&hi)[kGP][kGQ]) {
  bool bad = false;
#pragma unroll
  for (int k = 0; k < kGP; ++k)
#pragma unroll
    for (int j = 0; j < kGQ; ++j) lo[k][j] = hi[k][j] = 0.0;
  const int cout = g.cout, cin = g.cin;
  const int nq = min(kGQ, cin - ci0);
  // covering rows ah ascending <=> fy descending
  int ah0 = fdiv(iy + g.ph - g.fh, g.sh) + 1, ah1 = fdiv(iy + g.ph, g.sh);
  ah0 = max(ah0, bh);
  ah1 = min(ah1, bh + g.Si_h - 1);
  // covering columns of the first position; position k covers aw + k
  int aw0 = fdiv(ix0 + g.pw - g.fw, g.sw) + 1, aw1 = fdiv(ix0 + g.pw, g.sw);
  for (int ah = ah0; ah <= ah1; ++ah) {
    const int fy = iy + g.ph - ah * g.sh;
    for (int aw = aw0; aw <= aw1; ++aw) {
      // position k uses cell (ah, aw + k); skip the tap if no position's cell is in the window
      const int kmin = max(0, bw - aw), kmax = min(npos, bw + g.Si_w - aw);
      if (kmin >= kmax) continue;
      const int fx = ix0 + g.pw - aw * g.sw;
      const double* wp = FT + ((size_t)(fy * g.fw + fx) * cout) * cin + ci0;
      const size_t cb = ((size_t)(ah - bh) * g.Si_w + (aw - bw)) * cout;
      for (int d = 0; d < cout; ++d) {
        double cl[kGP], ch[kGP];
        bool any = false;
#pragma unroll
        for (int k = 0; k < kGP; ++k) {
          const bool in = k >= kmin && k < kmax;
          cl[k] = in ? ilo[cb + (size_t)k * cout + d] : 0.0;
          ch[k] = in ? ihi[cb + (size_t)k * cout + d] : 0.0;
          any |= (cl[k] != 0.0) | (ch[k] != 0.0);
        }
        if (!any) continue;
        double w[kGQ];
#pragma unroll
        for (int j = 0; j < kGQ; ++j) w[j] = j < nq ? wp[(size_t)d * cin + j] : 0.0;
#pragma unroll
        for (int k = 0; k < kGP; ++k)
#pragma unroll
          for (int j = 0; j < kGQ; ++j) {
            if (FAST) madd_f(w[j], cl[k], ch[k], lo[k][j], hi[k][j], bad);
            else madd_x(w[j], cl[k], ch[k], lo[k][j], hi[k][j]);
          }
      }
    }
  }
  return bad;
}

// Store one task's outputs.
__device__ __forceinline__ void gbc_store(const GbcGeom& g, double* olo, double* ohi, int y,
                                          int So_w, int first, int npos, int ci0,
                                          const double (&lo)[kGP][kGQ],
                                          const double (&hi)[kGP][kGQ]) {
#pragma unroll
  for (int k = 0; k < kGP; ++k) {
    if (k >= npos) break;
    const size_t o = ((size_t)y * So_w + first + (size_t)k * g.sw) * g.cin + ci0;
#pragma unroll
    for (int j = 0; j < kGQ; ++j)
      if (ci0 + j < g.cin) {
        olo[o + j] = lo[k][j];
        ohi[o + j] = hi[k][j];
      }
  }
}

// Exact-ops recomputation of one task (an operand left the fast band); kept
// out of line so the fast path's register allocation is unaffected.
__device__ __noinline__ void gbc_task_exact(const GbcGeom& g, const double* FT, const double* ilo,
                                            const double* ihi, int bw, int bh, int iy, int ix0,
                                            int npos, int ci0, double* olo, double* ohi, int y,
                                            int So_w, int first) {
  double lo[kGP][kGQ], hi[kGP][kGQ];
  gbc_task<false>(g, FT, ilo, ihi, bw, bh, iy, ix0, npos, ci0, lo, hi);
  gbc_store(g, olo, ohi, y, So_w, first, npos, ci0, lo, hi);
}

__global__ void __launch_bounds__(256)
    k_gbc_tile(GbcGeom g, const double* __restrict__ FT, RowsDev rows, FrameDev fi, FrameDev fo,
               MatDev in, MatDev out) {
  int i;
  if (!rows_resolve(rows, blockIdx.y, i)) return;
  bool upper;
  const int q = row_query(rows, i, upper);
  int bw, bh, nbw, nbh;
  frame_base(fi, q, bw, bh);
  frame_base(fo, q, nbw, nbh);
  const double* ilo = in.lo + phys_row(in, i) * in.cells;
  const double* ihi = in.hi + phys_row(in, i) * in.cells;
  double* olo = out.lo + (size_t)i * out.cells;
  double* ohi = out.hi + (size_t)i * out.cells;
  MagAcc mag;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < g.tasks;
       t += (long long)gridDim.x * blockDim.x) {
    const int cg = (int)(t % g.nq);
    const long long r = t / g.nq;
    const int xg = (int)(r % g.ncls_x);
    const int y = (int)(r / g.ncls_x);
    // position group xg -> parity class and first member
    int rem = xg, first = 0, n_c = 0;
    bool found = false;
    for (int cls = 0; cls < g.sw; ++cls) {
      // members x in [0, So_w) with (nbw + x + pw) mod sw == cls
      const int x0 = ((cls - (nbw + g.pw)) % g.sw + g.sw) % g.sw;
      n_c = x0 < g.So_w ? (g.So_w - 1 - x0) / g.sw + 1 : 0;
      const int ng = (n_c + kGP - 1) / kGP;
      if (rem < ng) {
        first = x0 + rem * kGP * g.sw;
        n_c -= rem * kGP;
        found = true;
        break;
      }
      rem -= ng;
    }
    if (!found) continue;  // this row's classes have fewer groups than the bound
    const int npos = min(kGP, n_c);
    const int iy = nbh + y, ix0 = nbw + first;
    const int ci0 = cg * kGQ;
    double lo[kGP][kGQ], hi[kGP][kGQ];
    if (gbc_task<true>(g, FT, ilo, ihi, bw, bh, iy, ix0, npos, ci0, lo, hi))
      gbc_task_exact(g, FT, ilo, ihi, bw, bh, iy, ix0, npos, ci0, olo, ohi, y, fo.S_w, first);
    else
      gbc_store(g, olo, ohi, y, fo.S_w, first, npos, ci0, lo, hi);
    // statistics of this task's outputs (read back: the exact path stores directly)
    for (int k = 0; k < npos; ++k) {
      const size_t o = ((size_t)y * fo.S_w + first + (size_t)k * g.sw) * g.cin + ci0;
      for (int j = 0; j < kGQ && ci0 + j < g.cin; ++j) {
        mag.add(olo[o + j]);
        mag.add(ohi[o + j]);
      }
    }
  }
  mag.flush(out.stat);
}

void init_kernel_attrs_gbc() {
  cudaFuncSetAttribute(k_gbc_tile, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}

void launch_gbc_tile(cudaStream_t s, const LayerDev& L, const RowsDev& rows, const FrameDev& fin,
                     const FrameDev& fout, MatDev in, MatDev out) {
  GbcGeom g;
  g.cin = L.in_c; g.cout = L.out_c;
  g.fw = L.fw; g.fh = L.fh; g.sw = L.sw; g.sh = L.sh; g.pw = L.pw; g.ph = L.ph;
  g.Si_w = fin.S_w; g.Si_h = fin.S_h;
  g.So_w = fout.S_w; g.So_h = fout.S_h;
  g.nq = (g.cin + kGQ - 1) / kGQ;
  // position groups per output row: parity classes split into groups of P
  int ncls = 0;
  for (int c = 0; c < g.sw; ++c) {
    // the class sizes depend on the row's window base only through (nbw + pw) mod sw,
    // which varies per row; bound the group count by the largest class size
    const int n_c = (g.So_w + g.sw - 1) / g.sw;
    ncls += (n_c + kGP - 1) / kGP;
    (void)c;
  }
  g.ncls_x = ncls;
  g.tasks = (long long)g.So_h * g.ncls_x * g.nq;
  unsigned gx = (unsigned)((g.tasks + 255) / 256);
  if (gx > 4096) gx = 4096;
  dim3 grid(gx, rows.n);
  k_gbc_tile<<<grid, 256, 0, s>>>(g, L.FT, rows, fin, fout, in, out);
  ++g_launches;
}

}  // namespace pc
