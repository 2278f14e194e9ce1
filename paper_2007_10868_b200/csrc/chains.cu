// chains.cu — serial constant / concretisation chains for long rows.
//
// The reference accumulates each row constant and each concretisation as an
// ascending serial chain of directed-rounded adds (backsub.hpp:365-389,
// 454-489, 536-563, 740-760): term j is added only for nonzero coefficient
// cells, and the chain cannot be split or reassociated in floating point.
// One CTA per row splits the work:
//
//   producer warps  compute the terms of a tile of cells in parallel and
//                   write the cells that contribute (in ascending order, by a
//                   block scan) into a shared-memory buffer — skipped cells
//                   cost nothing downstream;
//   consumer warps  one per chain (k.lo, k.hi, kraw.lo, kraw.hi, dev; or the
//                   padded / raw concretisation) fold the previous tile's
//                   compacted terms in order with the warp-scan fold of
//                   scanfold.cuh: 32 links per step as an exact integer
//                   prefix sum inside the accumulator's binade, the scalar
//                   op for the rare link that leaves it.
//
// Tiles are double-buffered, so term generation runs one tile ahead of the
// fold. Results are identical to the reference's chains (same terms, same
// order, same add_up / add_down), tested against serial folds on adversarial
// chains (tests/test_gpu_numeric.py) and on whole networks.
#include "kernels.cuh"
#include "numeric.cuh"
#include "scanfold.cuh"

namespace pc {

#define PC_NAN __longlong_as_double(0x7ff8000000000000ULL)

constexpr int kCT = 512;  // threads per CTA
constexpr int kCPT = 2;   // cells per producer thread per tile

// Warp roles per generator: G::NF consumer warps (one per chain), the rest
// producers.
template <class G>
struct Roles {
  static constexpr int kProd = kCT - 32 * G::NF;  // producer threads
  static constexpr int kTile = kProd * kCPT;       // cells per tile
};

// Frame cell -> (channel, absolute grid column, row). 32-bit (a row holds
// fewer than 2^31 cells); the channel split is a shift for the power-of-two
// channel counts of the residual nets.
__device__ __forceinline__ void cell_pos(const FrameDev& f, long long cell64, int bw, int bh, int& d,
                                         int& aw, int& ah) {
  const unsigned cell = (unsigned)cell64, C = (unsigned)f.C;
  unsigned pos;
  if ((C & (C - 1)) == 0) {
    d = (int)(cell & (C - 1));
    pos = cell >> (__ffs(C) - 1);
  } else {
    pos = cell / C;
    d = (int)(cell - pos * C);
  }
  const unsigned y = pos / (unsigned)f.S_w;
  aw = bw + (int)(pos - y * (unsigned)f.S_w);
  ah = bh + (int)y;
}

// ---------------------------------------------------------------------------
// Term generators. gen() returns true iff the cell contributes; t[a] = NaN
// marks an array without a term for this cell. Terms use the exact ops.

// dense_step / gbc_step constants: k += c*b_j, kraw += c*b_j, dev += mag(c)*dev_j
// (backsub.hpp:365-389, 454-489). Arrays: 0 lo term, 1 hi term, 2 dev term.
struct AffineGen {
  static constexpr int NA = 3, NF = 5;
  LayerDev L;
  int is_conv;
  FrameDev f;
  int bw, bh;
  const double* dev;
  unsigned long long madds = 0;
  __device__ bool gen(const double* lo, const double* hi, long long cell, double* t) {
    const Iv c{lo[cell], hi[cell]};
    if (iv_zero(c)) return false;
    double b;
    long long jd;
    if (is_conv) {
      int d, aw, ah;
      cell_pos(f, cell, bw, bh, d, aw, ah);
      b = L.bias[d];
      jd = ((long long)ah * f.G_w + aw) * f.C + d;
      const int y0 = ah * L.sh - L.ph, x0 = aw * L.sw - L.pw;
      const int ny = min(L.fh, L.in_h - y0) - max(0, -y0);
      const int nx = min(L.fw, L.in_w - x0) - max(0, -x0);
      if (ny > 0 && nx > 0) madds += (unsigned long long)L.in_c * ny * nx;
    } else {
      b = L.bias[cell];
      jd = cell;
      madds += (unsigned long long)L.in_w * L.in_h * L.in_c;
    }
    const Iv bt = iv_mul_scalar(c, b);
    t[0] = iv_zero(bt) ? PC_NAN : bt.lo;
    t[1] = iv_zero(bt) ? PC_NAN : bt.hi;
    const double dj = dev[jd];
    t[2] = dj != 0.0 ? mul_up(iv_mag(c), dj) : PC_NAN;
    return true;
  }
  // fold lanes: k.lo, k.hi, kraw.lo, kraw.hi, dev
  __device__ static int arr(int lane, int) { return lane == 4 ? 2 : (lane & 1); }
  __device__ static bool up(int lane) { return (lane & 1) || lane == 4; }
  static constexpr int TPE = 1;  // terms per entry per lane
};

// relu_step constants (backsub.hpp:536-563): per nonzero cell one offset (sign
// stable) or two (straddling: offp then offn). Arrays: 0/1 first term lo/hi,
// 2/3 second term lo/hi.
struct ReluGen {
  static constexpr int NA = 4, NF = 4;
  FrameDev f;
  int bw, bh;
  bool upper;
  const double* relax;
  unsigned long long madds = 0;
  __device__ bool gen(const double* lo, const double* hi, long long cell, double* t) {
    const Iv c{lo[cell], hi[cell]};
    if (iv_zero(c)) return false;
    int d, aw, ah;
    cell_pos(f, cell, bw, bh, d, aw, ah);
    const double* R = relax + 8 * (((long long)ah * f.G_w + aw) * f.C + d);
    const Iv beta{R[2], R[3]}, delta{R[6], R[7]};
    const Iv op = upper ? delta : beta;
    const Iv on = upper ? beta : delta;
    if (iv_zero(op) && iv_zero(on)) return false;  // stable neuron: exact zero terms
    Iv o0, o1{0.0, 0.0};
    if (!(c.lo < 0.0)) o0 = iv_mul(c, op);
    else if (!(c.hi > 0.0)) o0 = iv_mul(c, on);
    else {
      o0 = iv_mul(iv_pos_part(c), op);
      o1 = iv_mul(iv_neg_part(c), on);
    }
    const bool z0 = iv_zero(o0), z1 = iv_zero(o1);
    t[0] = z0 ? PC_NAN : o0.lo;
    t[1] = z0 ? PC_NAN : o0.hi;
    t[2] = z1 ? PC_NAN : o1.lo;
    t[3] = z1 ? PC_NAN : o1.hi;
    return !(z0 && z1);
  }
  // fold lanes: k.lo, k.hi, kraw.lo, kraw.hi; each folds term 0 then term 1
  __device__ static int arr(int lane, int k) { return 2 * k + (lane & 1); }
  __device__ static bool up(int lane) { return lane & 1; }
  static constexpr int TPE = 2;
};

// concretize (backsub.hpp:725-764): acc (+)= corner(c_j, B_j) over nonzero
// cells, padded track (bounds) and raw track (raw bounds). A +0 term leaves a
// non-(-0) accumulator unchanged, so it is skipped unless the start value is -0.
struct ConcGen {
  static constexpr int NA = 2, NF = 2;
  FrameDev f;
  int bw, bh;
  bool upper, skip0;
  const double *blo, *bhi, *rlo, *rhi;
  unsigned long long madds = 0;
  __device__ bool gen(const double* lo, const double* hi, long long cell, double* t) {
    const Iv c{lo[cell], hi[cell]};
    if (iv_zero(c)) return false;
    int d, aw, ah;
    cell_pos(f, cell, bw, bh, d, aw, ah);
    const long long j = ((long long)ah * f.G_w + aw) * f.C + d;
    const Iv B{blo[j], bhi[j]}, Br{rlo[j], rhi[j]};
    const double tp = upper ? corner_hi(c, B) : corner_lo(c, B);
    const double tr = upper ? corner_hi(c, Br) : corner_lo(c, Br);
    const bool zp = skip0 && __double_as_longlong(tp) == 0, zr = skip0 && __double_as_longlong(tr) == 0;
    t[0] = zp ? PC_NAN : tp;
    t[1] = zr ? PC_NAN : tr;
    return !(zp && zr);
  }
  __device__ static int arr(int lane, int) { return lane; }
  __device__ bool up_of(int) const { return upper; }
  __device__ static bool up(int) { return false; }  // unused (direction per row)
  static constexpr int TPE = 1;
};

// Consumer warp w folds chain w: the terms of array G::arr(w, k) (k < TPE:
// entry e contributes its TPE terms in order), direction G::up(w) (the row's
// polarity for concretisations).
template <class G>
__device__ __forceinline__ bool chain_up(const G& g, int w) {
  return G::up(w);
}
template <>
__device__ __forceinline__ bool chain_up<ConcGen>(const ConcGen& g, int) {
  return g.upper;
}

struct ChainShared {
  int cnt[2];
  int wsum[kCT / 32];
  double acc[8];  // each chain's result (consumer warp w -> acc[w])
};

// Shared layout: buf[2][NA][kTile] doubles. acc: the chain's start value in
// consumer warp w (all lanes); returns its result there (sh.acc[w] too).
template <class G>
__device__ __forceinline__ double fold_row(G& g, const double* lo, const double* hi,
                                           long long cells, double acc, double* buf,
                                           ChainShared& sh) {
  constexpr int kProd = Roles<G>::kProd, kTile = Roles<G>::kTile;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ntiles = (int)((cells + kTile - 1) / kTile);
  const bool consumer = warp < G::NF;
  const bool up = consumer && chain_up(g, warp);
  for (int it = 0; it <= ntiles; ++it) {
    if (consumer) {
      if (it > 0) {
        const int b = (it - 1) & 1;
        const int n = sh.cnt[b];
        const double* B = buf + (size_t)b * G::NA * kTile;
        if (G::TPE == 1) {
          const double* T = B + G::arr(warp, 0) * kTile;
          acc = scan_fold4(acc, n, up, [&](int j) { return T[j]; });
        } else {
          const double* T0 = B + G::arr(warp, 0) * kTile;
          const double* T1 = B + G::arr(warp, 1) * kTile;
          acc = scan_fold4(acc, G::TPE * n, up, [&](int j) { return (j & 1) ? T1[j >> 1] : T0[j >> 1]; });
        }
      }
    } else if (it < ntiles) {
      const int p = tid - 32 * G::NF;
      const int b = it & 1;
      double* B = buf + (size_t)b * G::NA * kTile;
      double t[kCPT][G::NA];
      bool v[kCPT];
      int nv = 0;
      const long long c0 = (long long)it * kTile + (long long)p * kCPT;
#pragma unroll
      for (int k = 0; k < kCPT; ++k) {
        v[k] = false;
        if (c0 + k < cells) v[k] = g.gen(lo, hi, c0 + k, t[k]);
        if (v[k]) ++nv;
      }
      // exclusive scan of nv over the producer threads (ascending cells)
      int inc = nv;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      const int pw = warp - G::NF;
      if (lane == 31) sh.wsum[pw] = inc;
      asm volatile("bar.sync 1, %0;" ::"r"(kProd));
      int base = 0, tot = 0;
#pragma unroll
      for (int w = 0; w < kProd / 32; ++w) {
        const int s = sh.wsum[w];
        base += w < pw ? s : 0;
        tot += s;
      }
      int pos = base + inc - nv;
#pragma unroll
      for (int k = 0; k < kCPT; ++k)
        if (v[k]) {
#pragma unroll
          for (int a = 0; a < G::NA; ++a) B[a * kTile + pos] = t[k][a];
          ++pos;
        }
      if (p == 0) sh.cnt[b] = tot;
      asm volatile("bar.sync 1, %0;" ::"r"(kProd));
    }
    __syncthreads();
  }
  if (consumer && lane == 0) sh.acc[warp] = acc;
  __syncthreads();
  return acc;
}

// ----- kernels: one CTA per row -----

__global__ void __launch_bounds__(kCT)
    k_chain_affine_big(LayerDev L, int is_conv, RowsDev rows, FrameDev f, MatDev m, double* Kout,
                       const double* dev, Counters* ctr, const char* frozen) {
  extern __shared__ double buf[];
  __shared__ ChainShared sh;
  int i;
  if (!rows_resolve(rows, blockIdx.x, i)) return;
  bool upper;
  int img;
  const int q = row_query(rows, i, upper, img);
  if (frozen && frozen[(size_t)img * rows.kq + q]) return;
  dev += img * rows.sst;
  ctr += img;
  if (is_conv && threadIdx.x == 0)
    atomicAdd(&ctr->gbc_dense_equiv, (unsigned long long)L.out_w * L.out_h * L.out_c *
                                         ((unsigned long long)L.in_w * L.in_h * L.in_c));
  AffineGen g{L, is_conv, f, 0, 0, dev};
  if (is_conv) frame_base(f, q, g.bw, g.bh);
  const size_t pr = phys_row(m, i);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double acc0 = warp < 4 ? m.K[4 * pr + warp] : 0.0;  // warp 4: dev, from 0
  fold_row(g, m.lo + pr * m.cells, m.hi + pr * m.cells, m.cells, acc0, buf, sh);
  if (threadIdx.x < 4) {
    const double dtot = sh.acc[4], a = sh.acc[threadIdx.x];
    double* K = Kout + 4 * (size_t)i;
    if (threadIdx.x == 0) K[0] = dtot != 0.0 ? add_down(a, -dtot) : a;  // widen_constant :175-179
    else if (threadIdx.x == 1) K[1] = dtot != 0.0 ? add_up(a, dtot) : a;
    else K[threadIdx.x] = a;
  }
  unsigned long long md = g.madds;
  for (int o = 16; o > 0; o >>= 1) md += __shfl_down_sync(0xffffffffu, md, o);
  if (lane == 0 && md) atomicAdd(is_conv ? &ctr->gbc_madds : &ctr->dense_madds, md);
}

__global__ void __launch_bounds__(kCT)
    k_chain_relu_big(RowsDev rows, FrameDev f, MatDev m, double* Kout, const double* relax,
                     const char* frozen) {
  extern __shared__ double buf[];
  __shared__ ChainShared sh;
  int i;
  if (!rows_resolve(rows, blockIdx.x, i)) return;
  bool upper;
  int img;
  const int q = row_query(rows, i, upper, img);
  if (frozen && frozen[(size_t)img * rows.kq + q]) return;
  ReluGen g{f, 0, 0, upper, relax + 8 * img * rows.sst};
  frame_base(f, q, g.bw, g.bh);
  const size_t pr = phys_row(m, i);
  const int warp = threadIdx.x >> 5;
  const double acc0 = warp < 4 ? m.K[4 * pr + warp] : 0.0;
  fold_row(g, m.lo + pr * m.cells, m.hi + pr * m.cells, m.cells, acc0, buf, sh);
  if (threadIdx.x < 4) Kout[4 * (size_t)i + threadIdx.x] = sh.acc[threadIdx.x];
}

__global__ void __launch_bounds__(kCT)
    k_concretize_big(RowsDev rows, FrameDev f, MatDev m, const double* blo, const double* bhi,
                     const double* rlo, const double* rhi, double* vals, double* rvals,
                     const char* frozen) {
  extern __shared__ double buf[];
  __shared__ ChainShared sh;
  int i;
  if (!rows_resolve(rows, blockIdx.x, i)) return;
  bool upper;
  int img;
  const int q = row_query(rows, i, upper, img);
  if (frozen && frozen[(size_t)img * rows.kq + q]) return;
  const long long so = img * rows.sst;
  blo += so;
  bhi += so;
  rlo += so;
  rhi += so;
  const size_t pr = phys_row(m, i);
  const double* K = m.K + 4 * pr;
  const double a0 = upper ? K[1] : K[0], a1 = upper ? K[3] : K[2];
  const bool neg0 = (__double_as_longlong(a0) == (long long)0x8000000000000000ULL) ||
                    (__double_as_longlong(a1) == (long long)0x8000000000000000ULL);
  ConcGen g{f, 0, 0, upper, !neg0, blo, bhi, rlo, rhi};
  frame_base(f, q, g.bw, g.bh);
  const int warp = threadIdx.x >> 5;
  const double acc0 = warp == 0 ? a0 : (warp == 1 ? a1 : 0.0);
  fold_row(g, m.lo + pr * m.cells, m.hi + pr * m.cells, m.cells, acc0, buf, sh);
  if (threadIdx.x == 0) vals[i] = sh.acc[0];
  if (threadIdx.x == 1) rvals[i] = sh.acc[1];
}

template <class G>
constexpr size_t chain_smem() {
  return (size_t)2 * G::NA * Roles<G>::kTile * sizeof(double);
}

static void set_attrs() {
  cudaFuncSetAttribute(k_chain_affine_big, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaFuncSetAttribute(k_chain_relu_big, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaFuncSetAttribute(k_concretize_big, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaFuncSetAttribute(k_chain_affine_big, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)chain_smem<AffineGen>());
  cudaFuncSetAttribute(k_chain_relu_big, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)chain_smem<ReluGen>());
  cudaFuncSetAttribute(k_concretize_big, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)chain_smem<ConcGen>());
}

void init_kernel_attrs_chains() { set_attrs(); }

void launch_chain_affine_big(cudaStream_t s, const LayerDev& L, bool is_conv, const RowsDev& rows,
                             const FrameDev& fin, MatDev m, double* Kout, const double* dev,
                             Counters* ctr, const char* frozen) {
  k_chain_affine_big<<<rows.n, kCT, chain_smem<AffineGen>(), s>>>(L, is_conv ? 1 : 0, rows, fin, m,
                                                                   Kout, dev, ctr, frozen);
  ++g_launches;
}

void launch_chain_relu_big(cudaStream_t s, const RowsDev& rows, const FrameDev& f, MatDev m,
                           double* Kout, const double* relax, const char* frozen) {
  k_chain_relu_big<<<rows.n, kCT, chain_smem<ReluGen>(), s>>>(rows, f, m, Kout, relax, frozen);
  ++g_launches;
}

void launch_concretize_big(cudaStream_t s, const RowsDev& rows, const FrameDev& f, MatDev m,
                           const double* blo, const double* bhi, const double* rlo,
                           const double* rhi, double* vals, double* rvals, const char* frozen) {
  k_concretize_big<<<rows.n, kCT, chain_smem<ConcGen>(), s>>>(rows, f, m, blo, bhi, rlo, rhi, vals,
                                                               rvals, frozen);
  ++g_launches;
}

}  // namespace pc
