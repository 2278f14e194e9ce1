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
#include <cub/block/block_scan.cuh>

#include <mutex>
#include <unordered_map>

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
  // index-only operands of a cell, loaded a tile ahead of its coefficient
  struct Pre {
    double b, dj;
    unsigned taps;
  };
  __device__ void pre(long long cell, Pre& p) const {
    long long jd;
    if (is_conv) {
      int d, aw, ah;
      cell_pos(f, cell, bw, bh, d, aw, ah);
      p.b = L.bias[d];
      jd = ((long long)ah * f.G_w + aw) * f.C + d;
      const int y0 = ah * L.sh - L.ph, x0 = aw * L.sw - L.pw;
      const int ny = min(L.fh, L.in_h - y0) - max(0, -y0);
      const int nx = min(L.fw, L.in_w - x0) - max(0, -x0);
      p.taps = (ny > 0 && nx > 0) ? (unsigned)(L.in_c * ny * nx) : 0u;
    } else {
      p.b = L.bias[cell];
      jd = cell;
      p.taps = (unsigned)(L.in_w * L.in_h * L.in_c);
    }
    p.dj = dev[jd];
  }
  bool fast = false;  // fast numeric mode: directed-rounding products
  __device__ bool gen(Iv c, const Pre& p, double* t) {
    if (iv_zero(c)) return false;
    madds += p.taps;
    if (fast) {
      const double b = p.b;
      if (b == 0.0) {
        t[0] = t[1] = PC_NAN;
      } else {
        t[0] = __dmul_rd(b > 0.0 ? c.lo : c.hi, b);
        t[1] = __dmul_ru(b > 0.0 ? c.hi : c.lo, b);
      }
      t[2] = p.dj != 0.0 ? __dmul_ru(iv_mag(c), p.dj) : PC_NAN;
      return true;
    }
    const Iv bt = iv_mul_scalar(c, p.b);
    t[0] = iv_zero(bt) ? PC_NAN : bt.lo;
    t[1] = iv_zero(bt) ? PC_NAN : bt.hi;
    t[2] = p.dj != 0.0 ? mul_up(iv_mag(c), p.dj) : PC_NAN;
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
  struct Pre {
    Iv beta, delta;
  };
  __device__ void pre(long long cell, Pre& p) const {
    int d, aw, ah;
    cell_pos(f, cell, bw, bh, d, aw, ah);
    const double* R = relax + 8 * (((long long)ah * f.G_w + aw) * f.C + d);
    p.beta = Iv{R[2], R[3]};
    p.delta = Iv{R[6], R[7]};
  }
  __device__ bool gen(Iv c, const Pre& p, double* t) {
    if (iv_zero(c)) return false;
    const Iv beta = p.beta, delta = p.delta;
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
  struct Pre {
    Iv B, Br;
  };
  __device__ void pre(long long cell, Pre& p) const {
    int d, aw, ah;
    cell_pos(f, cell, bw, bh, d, aw, ah);
    const long long j = ((long long)ah * f.G_w + aw) * f.C + d;
    p.B = Iv{blo[j], bhi[j]};
    p.Br = Iv{rlo[j], rhi[j]};
  }
  bool fast = false;  // fast numeric mode: directed-rounding corner products
  __device__ static double fcorner(Iv c, Iv B, bool up) {
    if (up)
      return fmax(fmax(__dmul_ru(c.lo, B.lo), __dmul_ru(c.lo, B.hi)), fmax(__dmul_ru(c.hi, B.lo), __dmul_ru(c.hi, B.hi)));
    return fmin(fmin(__dmul_rd(c.lo, B.lo), __dmul_rd(c.lo, B.hi)), fmin(__dmul_rd(c.hi, B.lo), __dmul_rd(c.hi, B.hi)));
  }
  __device__ bool gen(Iv c, const Pre& p, double* t) {
    if (iv_zero(c)) return false;
    const double tp = fast ? fcorner(c, p.B, upper) : upper ? corner_hi(c, p.B) : corner_lo(c, p.B);
    const double tr = fast ? fcorner(c, p.Br, upper) : upper ? corner_hi(c, p.Br) : corner_lo(c, p.Br);
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

// 1-D bulk copies (TMA, cp.async.bulk) global -> shared, completing on an
// mbarrier with a transaction count.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra "
      "WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

constexpr int kStages = 4;  // coefficient tiles in flight (TMA ring)

struct ChainShared {
  unsigned long long bar[kStages];  // coefficient tile staged (TMA) per ring slot
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
  // The row's coefficients stream through shared memory by TMA bulk copies
  // (a kStages ring, issued kStages tiles ahead of the producers), when the
  // row is 16-byte aligned; the index-only operands of the next tile (bounds,
  // deviations, biases) are loaded into registers one tile ahead.
  double* cbuf = buf + 2 * G::NA * kTile;  // [kStages][lo, hi][kTile]
  const bool tma = ((reinterpret_cast<unsigned long long>(lo) | reinterpret_cast<unsigned long long>(hi)) & 15) == 0;
  const int p0 = 32 * G::NF;  // first producer thread
  auto issue = [&](int it) {  // by thread p0
    const int b = it % kStages;
    const long long c0 = (long long)it * kTile;
    const long long n = cells - c0 < kTile ? cells - c0 : kTile;
    const unsigned bytes = (unsigned)(((n * 8) + 15) & ~15LL);  // the arena rounds rows' ends to 256 B
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // earlier generic reads of the buffer
    mbar_expect_tx(&sh.bar[b], 2 * bytes);
    bulk_g2s(cbuf + (size_t)b * 2 * kTile, lo + c0, bytes, &sh.bar[b]);
    bulk_g2s(cbuf + (size_t)b * 2 * kTile + kTile, hi + c0, bytes, &sh.bar[b]);
  };
  if (tma && tid == p0) {
    for (int k = 0; k < kStages; ++k) mbar_init(&sh.bar[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tma && tid == p0)
    for (int k = 0; k < kStages && k < ntiles; ++k) issue(k);
  typename G::Pre pre[kCPT];
  if (!consumer) {
    const long long c0 = (long long)(tid - p0) * kCPT;
#pragma unroll
    for (int k = 0; k < kCPT; ++k)
      if (c0 + k < cells) g.pre(c0 + k, pre[k]);
  }
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
      const int p = tid - p0;
      const int b = it & 1, cb = it % kStages;
      double* B = buf + (size_t)b * G::NA * kTile;
      const double* C = cbuf + (size_t)cb * 2 * kTile;
      const long long c0 = (long long)it * kTile + (long long)p * kCPT;
      Iv cv[kCPT];
      if (tma) {
        mbar_wait(&sh.bar[cb], (unsigned)((it / kStages) & 1));
#pragma unroll
        for (int k = 0; k < kCPT; ++k) cv[k] = Iv{C[p * kCPT + k], C[kTile + p * kCPT + k]};
      } else {
#pragma unroll
        for (int k = 0; k < kCPT; ++k)
          cv[k] = c0 + k < cells ? Iv{lo[c0 + k], hi[c0 + k]} : Iv{0.0, 0.0};
      }
      double t[kCPT][G::NA];
      bool v[kCPT];
      int nv = 0;
#pragma unroll
      for (int k = 0; k < kCPT; ++k) {
        v[k] = c0 + k < cells && g.gen(cv[k], pre[k], t[k]);
        if (v[k]) ++nv;
      }
      // next tile's index-only operands, in flight during the scan and barriers
      const long long c1 = c0 + kTile;
#pragma unroll
      for (int k = 0; k < kCPT; ++k)
        if (c1 + k < cells) g.pre(c1 + k, pre[k]);
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
      // every producer has read coefficient buffer cb: refill it kStages tiles ahead
      if (tma && tid == p0 && it + kStages < ntiles) issue(it + kStages);
    }
    __syncthreads();
  }
  if (consumer && lane == 0) sh.acc[warp] = acc;
  __syncthreads();
  return acc;
}

// ----- kernels: one CTA per row -----

__global__ void __launch_bounds__(kCT, 2)
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

__global__ void __launch_bounds__(kCT, 2)
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

__global__ void __launch_bounds__(kCT, 2)
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

// ---------------------------------------------------------------------------
// CTA-per-chain kernels: every chain of a row is folded by its own CTA with
// the block-wide scan fold (4 * kSF links per step); terms are computed on the
// fly by all threads. Used for the conv steps' constant chains (from the
// compacted nonzero coefficients k_compact_cells already wrote: no second
// pass over the dense row) and for the checkpoints' concretisations, so a
// pass with few rows still spreads over many SMs and a row's chain costs
// microseconds.
constexpr int kSF = 512;

// gbc_step constants (backsub.hpp:449-489) of one row, one chain per CTA
// (blockIdx.y: 0 k.lo, 1 k.hi, 2 kraw.lo, 3 kraw.hi, 4 dev); terms in the
// compacted layout [cell][slot < cnt] = ascending (cell, d). Results go to
// tmp[5 * i + chain]; k_affine_finish widens and stores K.
__global__ void __launch_bounds__(kSF)
    k_chain_affine_scan(LayerDev L, RowsDev rows, FrameDev f, MatDev m, SparseDev sp,
                        const double* dev, double* tmp, Counters* ctr, const char* frozen) {
  __shared__ long long sm[2 * kSF / 32 + 4];
  int i;
  if (!rows_resolve(rows, blockIdx.x, i)) return;
  bool upper;
  int img;
  const int q = row_query(rows, i, upper, img);
  if (frozen && frozen[(size_t)img * rows.kq + q]) return;
  dev += img * rows.sst;
  ctr += img;
  const int chain = blockIdx.y;
  int bw, bh;
  frame_base(f, q, bw, bh);
  const int C = sp.C;
  const int* cnt = sp.cnt + (size_t)i * sp.ncell;
  const size_t rb = (size_t)i * sp.ncell * C;
  const size_t pr = phys_row(m, i);
  if (chain == 0) {  // PassStats: madds of the in-grid taps per nonzero coefficient, dense-equivalent work
    unsigned long long md = 0;
    for (int cell = threadIdx.x; cell < sp.ncell; cell += kSF) {
      const int n = cnt[cell];
      if (!n) continue;
      const int y = cell / f.S_w, x = cell - y * f.S_w;
      const int y0 = (bh + y) * L.sh - L.ph, x0 = (bw + x) * L.sw - L.pw;
      const int ny = min(L.fh, L.in_h - y0) - max(0, -y0);
      const int nx = min(L.fw, L.in_w - x0) - max(0, -x0);
      if (ny > 0 && nx > 0) md += (unsigned long long)n * L.in_c * ny * nx;
    }
    for (int o = 16; o > 0; o >>= 1) md += __shfl_down_sync(0xffffffffu, md, o);
    if ((threadIdx.x & 31) == 0 && md) atomicAdd(&ctr->gbc_madds, md);
    if (threadIdx.x == 0)
      atomicAdd(&ctr->gbc_dense_equiv, (unsigned long long)L.out_w * L.out_h * L.out_c *
                                           ((unsigned long long)L.in_w * L.in_h * L.in_c));
  }
  const bool up = chain == 1 || chain == 3 || chain == 4;
  const double acc0 = chain < 4 ? m.K[4 * pr + chain] : 0.0;
  const int cs = (C & (C - 1)) == 0 ? __ffs(C) - 1 : -1;
  auto term = [&](int j) -> double {
    const int cell = cs >= 0 ? (j >> cs) : j / C;
    const int k = j - cell * C;
    if (k >= cnt[cell]) return PC_NAN;
    const size_t e = rb + (size_t)j;
    const Iv c{sp.lo[e], sp.hi[e]};
    const int d = sp.idx[e];
    if (chain < 4) {
      const Iv bt = iv_mul_scalar(c, L.bias[d]);
      if (iv_zero(bt)) return PC_NAN;
      return (chain & 1) ? bt.hi : bt.lo;
    }
    const int y = cell / f.S_w, x = cell - y * f.S_w;
    const double dj = dev[((long long)(bh + y) * f.G_w + (bw + x)) * f.C + d];
    return dj != 0.0 ? mul_up(iv_mag(c), dj) : PC_NAN;
  };
  const double acc = block_scan_fold<kSF>(acc0, sp.ncell * C, up, term, sm);
  if (threadIdx.x == 0) tmp[5 * (size_t)i + chain] = acc;
}

// widen_constant (backsub.hpp:175-179) with the dev total, store K.
__global__ void k_affine_finish(RowsDev rows, const double* tmp, double* Kout, const char* frozen) {
  int i;
  if (!rows_resolve(rows, blockIdx.x * blockDim.x + threadIdx.x, i)) return;
  bool upper;
  int img;
  const int q = row_query(rows, i, upper, img);
  if (frozen && frozen[(size_t)img * rows.kq + q]) return;
  const double* t = tmp + 5 * (size_t)i;
  const double dtot = t[4];
  double* K = Kout + 4 * (size_t)i;
  K[0] = dtot != 0.0 ? add_down(t[0], -dtot) : t[0];
  K[1] = dtot != 0.0 ? add_up(t[1], dtot) : t[1];
  K[2] = t[2];
  K[3] = t[3];
}

// concretize (backsub.hpp:725-764) of one row and one track per CTA
// (blockIdx.y: 0 padded vs bounds, 1 raw vs raw bounds).
__global__ void __launch_bounds__(kSF)
    k_concretize_scan(RowsDev rows, FrameDev f, MatDev m, const double* blo, const double* bhi,
                      const double* rlo, const double* rhi, double* vals, double* rvals,
                      const char* frozen) {
  __shared__ long long sm[2 * kSF / 32 + 4];
  int i;
  if (!rows_resolve(rows, blockIdx.x, i)) return;
  bool upper;
  int img;
  const int q = row_query(rows, i, upper, img);
  if (frozen && frozen[(size_t)img * rows.kq + q]) return;
  const int track = blockIdx.y;
  const long long so = img * rows.sst;
  const double* BL = (track ? rlo : blo) + so;
  const double* BH = (track ? rhi : bhi) + so;
  int bw, bh;
  frame_base(f, q, bw, bh);
  const size_t pr = phys_row(m, i);
  const double* lo = m.lo + pr * m.cells;
  const double* hi = m.hi + pr * m.cells;
  const double* K = m.K + 4 * pr;
  const double a0 = track ? (upper ? K[3] : K[2]) : (upper ? K[1] : K[0]);
  const bool skip0 = __double_as_longlong(a0) != (long long)0x8000000000000000ULL;
  const unsigned C = (unsigned)f.C;
  const int cs = (C & (C - 1)) == 0 ? __ffs(C) - 1 : -1;
  auto term = [&](int cell) -> double {
    const Iv c{lo[cell], hi[cell]};
    if (iv_zero(c)) return PC_NAN;
    unsigned pos, d;
    if (cs >= 0) {
      pos = (unsigned)cell >> cs;
      d = (unsigned)cell & (C - 1);
    } else {
      pos = (unsigned)cell / C;
      d = (unsigned)cell - pos * C;
    }
    const unsigned y = pos / (unsigned)f.S_w;
    const long long j = ((long long)(bh + (int)y) * f.G_w + (bw + (int)(pos - y * f.S_w))) * f.C + d;
    const Iv B{BL[j], BH[j]};
    const double t = upper ? corner_hi(c, B) : corner_lo(c, B);
    return (skip0 && __double_as_longlong(t) == 0) ? PC_NAN : t;
  };
  const double acc = block_scan_fold<kSF>(a0, (int)m.cells, upper, term, sm);
  if (threadIdx.x == 0) (track ? rvals : vals)[i] = acc;
}

void launch_chain_affine_scan(cudaStream_t s, const LayerDev& L, const RowsDev& rows, const FrameDev& fin,
                              MatDev m, SparseDev sp, double* tmp, double* Kout, const double* dev,
                              Counters* ctr, const char* frozen) {
  k_chain_affine_scan<<<dim3(rows.n, 5), kSF, 0, s>>>(L, rows, fin, m, sp, dev, tmp, ctr, frozen);
  k_affine_finish<<<(rows.n + 127) / 128, 128, 0, s>>>(rows, tmp, Kout, frozen);
  g_launches += 2;
}

void launch_concretize_scan(cudaStream_t s, const RowsDev& rows, const FrameDev& f, MatDev m,
                            const double* blo, const double* bhi, const double* rlo, const double* rhi,
                            double* vals, double* rvals, const char* frozen) {
  k_concretize_scan<<<dim3(rows.n, 2), kSF, 0, s>>>(rows, f, m, blo, bhi, rlo, rhi, vals, rvals, frozen);
  ++g_launches;
}

// ---------------------------------------------------------------------------
// Split chains: a term kernel spreads a row's cells over many CTAs (each
// computes and compacts the terms of one 1024-cell tile into a per-stream
// scratch buffer), then a fold kernel runs one warp per chain over the
// compacted tiles in order. The fold warps hold few resources, so the conv
// kernels stay resident beside them; the term kernel is short and wide.
constexpr int kTT = 256;           // term-kernel threads
constexpr int kTCP = 4;            // cells per thread
constexpr int kTTile = kTT * kTCP;  // cells per tile

struct StreamScratch {
  void* p = nullptr;
  size_t cap = 0;
};
static std::mutex g_scr_mu;
static std::unordered_map<cudaStream_t, StreamScratch> g_scr;
// Grow-only scratch per stream (its kernels run in order, so consecutive
// chains on one stream reuse it).
static void* stream_scratch(cudaStream_t s, size_t bytes) {
  std::lock_guard<std::mutex> lk(g_scr_mu);
  StreamScratch& e = g_scr[s];
  if (bytes > e.cap) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
      cudaGetLastError();
      return nullptr;  // no allocation inside a graph capture: the caller takes the in-CTA fold
    }
    if (e.p) {
      cudaStreamSynchronize(s);
      cudaFree(e.p);
    }
    e.p = nullptr;
    e.cap = 0;
    const size_t want = bytes + bytes / 4;
    if (cudaMalloc(&e.p, want) != cudaSuccess) return nullptr;
    e.cap = want;
  }
  return e.p;
}

template <class G>
__device__ __forceinline__ void tile_terms(G& g, const double* lo, const double* hi, long long cells,
                                           double* tb, long long tstride, int* tcnt) {
  using Scan = cub::BlockScan<int, kTT>;
  __shared__ typename Scan::TempStorage tmp;
  const int tile = blockIdx.x;
  const long long c0 = (long long)tile * kTTile + (long long)threadIdx.x * kTCP;
  typename G::Pre pre[kTCP];
  Iv cv[kTCP];
#pragma unroll
  for (int k = 0; k < kTCP; ++k)
    if (c0 + k < cells) {
      g.pre(c0 + k, pre[k]);
      cv[k] = Iv{lo[c0 + k], hi[c0 + k]};
    }
  double t[kTCP][G::NA];
  bool v[kTCP];
  int nv = 0;
#pragma unroll
  for (int k = 0; k < kTCP; ++k) {
    v[k] = c0 + k < cells && g.gen(cv[k], pre[k], t[k]);
    nv += v[k];
  }
  int pos, tot;
  Scan(tmp).ExclusiveSum(nv, pos, tot);
  double* T = tb + (long long)tile * kTTile;
#pragma unroll
  for (int k = 0; k < kTCP; ++k)
    if (v[k]) {
#pragma unroll
      for (int a = 0; a < G::NA; ++a) T[a * tstride + pos] = t[k][a];
      ++pos;
    }
  if (threadIdx.x == 0) tcnt[tile] = tot;
}

__global__ void __launch_bounds__(kTT)
    k_affine_terms(LayerDev L, int is_conv, RowsDev rows, FrameDev f, MatDev m, const double* dev,
                   double* tbuf, int* tcnt, long long tstride, int ntiles, Counters* ctr, const char* frozen,
                   int fast) {
  int i;
  if (!rows_resolve(rows, blockIdx.y, i)) return;
  bool upper;
  int img;
  const int q = row_query(rows, i, upper, img);
  if (frozen && frozen[(size_t)img * rows.kq + q]) return;
  ctr += img;
  AffineGen g{L, is_conv, f, 0, 0, dev + img * rows.sst};
  g.fast = fast != 0;
  if (is_conv) frame_base(f, q, g.bw, g.bh);
  const size_t pr = phys_row(m, i);
  tile_terms(g, m.lo + pr * m.cells, m.hi + pr * m.cells, m.cells, tbuf + (size_t)i * 3 * tstride, tstride,
             tcnt + (size_t)i * ntiles);
  unsigned long long md = g.madds;
  for (int o = 16; o > 0; o >>= 1) md += __shfl_down_sync(0xffffffffu, md, o);
  if ((threadIdx.x & 31) == 0 && md) atomicAdd(is_conv ? &ctr->gbc_madds : &ctr->dense_madds, md);
  if (is_conv && blockIdx.x == 0 && threadIdx.x == 0)
    atomicAdd(&ctr->gbc_dense_equiv, (unsigned long long)L.out_w * L.out_h * L.out_c *
                                         ((unsigned long long)L.in_w * L.in_h * L.in_c));
}

// Fold one chain over the row's compacted tiles with the warp scan, each tile
// staged into the warp's shared-memory buffer by cp.async one tile ahead
// (16-byte copies; the scratch tiles are 16-byte aligned, kTTile doubles
// apart), so every scan step reads shared memory.
template <bool FAST>
__device__ __forceinline__ double fold_tiles(double acc, bool up, const double* T, const int* cnt,
                                             int ntiles, double* buf /* [2][kTTile] */) {
  const int lane = threadIdx.x & 31;
  auto stage = [&](int t, int b) {
    const int n = cnt[t];
    const double* src = T + (long long)t * kTTile;
    double* dst = buf + b * kTTile;
    for (int e = 2 * lane; e < n; e += 64) {
      const unsigned sa = (unsigned)__cvta_generic_to_shared(dst + e);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src + e));
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  if (ntiles > 0) stage(0, 0);
  for (int t = 0; t < ntiles; ++t) {
    const int b = t & 1;
    if (t + 1 < ntiles) {
      stage(t + 1, b ^ 1);
      asm volatile("cp.async.wait_group 1;\n" ::);
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::);
    }
    __syncwarp();
    const double* B = buf + b * kTTile;
    acc = scan_fold4m<FAST>(acc, cnt[t], up, [&](int j) { return B[j]; });
    __syncwarp();  // buffer b is restaged by the next iteration's stage(t + 2)
  }
  return acc;
}

__global__ void __launch_bounds__(160)
    k_affine_fold(RowsDev rows, MatDev m, double* Kout, const double* tbuf, const int* tcnt,
                  long long tstride, int ntiles, const char* frozen, int fast) {
  __shared__ double s_acc[5];
  int i;
  if (!rows_resolve(rows, blockIdx.x, i)) return;
  bool upper;
  int img;
  const int q = row_query(rows, i, upper, img);
  if (frozen && frozen[(size_t)img * rows.kq + q]) return;
  const int warp = threadIdx.x >> 5;  // chain: k.lo, k.hi, kraw.lo, kraw.hi, dev
  const size_t pr = phys_row(m, i);
  double acc = warp < 4 ? m.K[4 * pr + warp] : 0.0;
  const bool up = AffineGen::up(warp);
  const double* T = tbuf + (size_t)i * 3 * tstride + AffineGen::arr(warp, 0) * tstride;
  const int* cnt = tcnt + (size_t)i * ntiles;
  extern __shared__ __align__(16) double fbuf[];
  acc = fast ? fold_tiles<true>(acc, up, T, cnt, ntiles, fbuf + (size_t)warp * 2 * kTTile)
             : fold_tiles<false>(acc, up, T, cnt, ntiles, fbuf + (size_t)warp * 2 * kTTile);
  if ((threadIdx.x & 31) == 0) s_acc[warp] = acc;
  __syncthreads();
  if (threadIdx.x < 4) {
    const double dtot = s_acc[4], a = s_acc[threadIdx.x];
    double* K = Kout + 4 * (size_t)i;
    if (threadIdx.x == 0) K[0] = dtot != 0.0 ? add_down(a, -dtot) : a;  // widen_constant :175-179
    else if (threadIdx.x == 1) K[1] = dtot != 0.0 ? add_up(a, dtot) : a;
    else K[threadIdx.x] = a;
  }
}

__global__ void __launch_bounds__(kTT)
    k_conc_terms(RowsDev rows, FrameDev f, MatDev m, const double* blo, const double* bhi,
                 const double* rlo, const double* rhi, double* tbuf, int* tcnt, long long tstride,
                 int ntiles, const char* frozen, int fast) {
  int i;
  if (!rows_resolve(rows, blockIdx.y, i)) return;
  bool upper;
  int img;
  const int q = row_query(rows, i, upper, img);
  if (frozen && frozen[(size_t)img * rows.kq + q]) return;
  const long long so = img * rows.sst;
  const size_t pr = phys_row(m, i);
  const double* K = m.K + 4 * pr;
  const double a0 = upper ? K[1] : K[0], a1 = upper ? K[3] : K[2];
  const bool neg0 = (__double_as_longlong(a0) == (long long)0x8000000000000000ULL) ||
                    (__double_as_longlong(a1) == (long long)0x8000000000000000ULL);
  ConcGen g{f, 0, 0, upper, !neg0, blo + so, bhi + so, rlo + so, rhi + so};
  g.fast = fast != 0;
  frame_base(f, q, g.bw, g.bh);
  tile_terms(g, m.lo + pr * m.cells, m.hi + pr * m.cells, m.cells, tbuf + (size_t)i * 2 * tstride, tstride,
             tcnt + (size_t)i * ntiles);
}

__global__ void __launch_bounds__(64)
    k_conc_fold(RowsDev rows, MatDev m, double* vals, double* rvals, const double* tbuf, const int* tcnt,
                long long tstride, int ntiles, const char* frozen, int fast) {
  int i;
  if (!rows_resolve(rows, blockIdx.x, i)) return;
  bool upper;
  int img;
  const int q = row_query(rows, i, upper, img);
  if (frozen && frozen[(size_t)img * rows.kq + q]) return;
  const int warp = threadIdx.x >> 5;  // 0: padded track, 1: raw track
  const size_t pr = phys_row(m, i);
  const double* K = m.K + 4 * pr;
  double acc = warp == 0 ? (upper ? K[1] : K[0]) : (upper ? K[3] : K[2]);
  const double* T = tbuf + (size_t)i * 2 * tstride + warp * tstride;
  const int* cnt = tcnt + (size_t)i * ntiles;
  extern __shared__ __align__(16) double fbuf[];
  acc = fast ? fold_tiles<true>(acc, upper, T, cnt, ntiles, fbuf + (size_t)warp * 2 * kTTile)
             : fold_tiles<false>(acc, upper, T, cnt, ntiles, fbuf + (size_t)warp * 2 * kTTile);
  if ((threadIdx.x & 31) == 0) (warp ? rvals : vals)[i] = acc;
}

// Few-row passes: one CTA per chain with the block fold (local retry), terms
// read from the compacted tiles through a tile prefix in shared memory.
constexpr int kFB = 512;
constexpr int kMaxFoldTiles = 128;

template <bool FAST>
__device__ __forceinline__ double fold_tiles_block(double acc, bool up, const double* T, const int* cnt,
                                                   int ntiles) {
  __shared__ int s_pref[kMaxFoldTiles + 1];
  __shared__ long long sm[2 * kFB / 32 + 8];
  if (threadIdx.x == 0) {
    int c = 0;
    for (int t = 0; t < ntiles; ++t) {
      s_pref[t] = c;
      c += cnt[t];
    }
    s_pref[ntiles] = c;
  }
  __syncthreads();
  const int n = s_pref[ntiles];
  auto term = [&](int j) -> double {
    int a = 0, b = ntiles;  // largest t with s_pref[t] <= j
    while (b - a > 1) {
      const int mid = (a + b) >> 1;
      if (s_pref[mid] <= j) a = mid;
      else b = mid;
    }
    return T[(long long)a * kTTile + (j - s_pref[a])];
  };
  return block_scan_fold_rtm<kFB, FAST>(acc, n, up, term, sm);
}

__global__ void __launch_bounds__(kFB)
    k_affine_fold_block(RowsDev rows, MatDev m, double* tmp, const double* tbuf, const int* tcnt,
                        long long tstride, int ntiles, const char* frozen, int fast) {
  int i;
  if (!rows_resolve(rows, blockIdx.x, i)) return;
  bool upper;
  int img;
  const int q = row_query(rows, i, upper, img);
  if (frozen && frozen[(size_t)img * rows.kq + q]) return;
  const int chain = blockIdx.y;
  const size_t pr = phys_row(m, i);
  const double acc0 = chain < 4 ? m.K[4 * pr + chain] : 0.0;
  const double* T = tbuf + (size_t)i * 3 * tstride + AffineGen::arr(chain, 0) * tstride;
  const double acc = fast ? fold_tiles_block<true>(acc0, AffineGen::up(chain), T, tcnt + (size_t)i * ntiles, ntiles)
                          : fold_tiles_block<false>(acc0, AffineGen::up(chain), T, tcnt + (size_t)i * ntiles, ntiles);
  if (threadIdx.x == 0) tmp[5 * (size_t)i + chain] = acc;
}

__global__ void __launch_bounds__(kFB)
    k_conc_fold_block(RowsDev rows, MatDev m, double* vals, double* rvals, const double* tbuf,
                      const int* tcnt, long long tstride, int ntiles, const char* frozen, int fast) {
  int i;
  if (!rows_resolve(rows, blockIdx.x, i)) return;
  bool upper;
  int img;
  const int q = row_query(rows, i, upper, img);
  if (frozen && frozen[(size_t)img * rows.kq + q]) return;
  const int track = blockIdx.y;
  const size_t pr = phys_row(m, i);
  const double* K = m.K + 4 * pr;
  const double acc0 = track == 0 ? (upper ? K[1] : K[0]) : (upper ? K[3] : K[2]);
  const double* T = tbuf + (size_t)i * 2 * tstride + track * tstride;
  const double acc = fast ? fold_tiles_block<true>(acc0, upper, T, tcnt + (size_t)i * ntiles, ntiles)
                          : fold_tiles_block<false>(acc0, upper, T, tcnt + (size_t)i * ntiles, ntiles);
  if (threadIdx.x == 0) (track ? rvals : vals)[i] = acc;
}

static int block_fold_rows() {
  static const int v = [] {
    const char* e = getenv("PC_BLOCK_FOLD_ROWS");
    return e && *e ? atoi(e) : 16;
  }();
  return v;
}

// ---------------------------------------------------------------------------
// Predicted compaction. Early termination drops a row once a checkpoint's
// exact raw concretisation freezes it, and the next step waits for that
// decision. The decision only needs the sign of the raw value, and the
// reference's chain lies provably close to a plain parallel sum: with
// B = |K| + sum |t_j| over the n terms, every add_up / add_down link moves
// the partial result by its exact sum plus at most 2 ulp outward, so the
// chain value v satisfies
//   add_up:   K + sum t <= v <= K + sum t + 3 n 2^-52 B
//   add_down: K + sum t - 3 n 2^-52 B <= v <= K + sum t
// and a round-to-nearest parallel sum S is within 1.01 n 2^-53 B of
// K + sum t. So with E = 4 (n + 2) 2^-52 B (rounded up), S + E <= 0 proves
// the row's raw upper value is <= 0 and S - E >= 0 its raw lower value >= 0
// (per link at most 2.5 ulp of the exact partial sum: RN's half ulp plus one
// step, which can be twice as wide across a binade boundary; ulps never drop
// below 2^-1074, so E also carries that absolute floor per link):
// the row certainly freezes at this checkpoint (backsub.hpp:814-817). Such
// rows are dropped before the next step without waiting for the exact folds;
// rows not proven (vanishingly rare) simply stay in the walk until the exact
// offers freeze them, which costs work but never changes a result. The exact
// concretisations and offers (candidates, freeze flags, counters) still run,
// on a third stream, off the critical path.
constexpr int kPT = 256;
constexpr int kPredScan = 1024;  // threads of the predicted-offer scan
__global__ void __launch_bounds__(kPT)
    k_pred_terms(RowsDev rows, FrameDev f, MatDev m, const double* rlo, const double* rhi, double* part,
                 int ntiles, const char* frozen) {
  __shared__ double s_red[3][kPT / 32];
  int i;
  if (!rows_resolve(rows, blockIdx.y, i)) return;
  bool upper;
  int img;
  const int q = row_query(rows, i, upper, img);
  double S = 0.0, A = 0.0, N = 0.0;
  if (!(frozen && frozen[(size_t)img * rows.kq + q])) {
    const long long so = img * rows.sst;
    int bw, bh;
    frame_base(f, q, bw, bh);
    const size_t pr = phys_row(m, i);
    const double* lo = m.lo + pr * m.cells;
    const double* hi = m.hi + pr * m.cells;
    const long long c0 = (long long)blockIdx.x * (kPT * 4);
    for (int k = 0; k < 4; ++k) {
      const long long cell = c0 + (long long)k * kPT + threadIdx.x;
      if (cell >= m.cells) break;
      const Iv c{lo[cell], hi[cell]};
      if (iv_zero(c)) continue;
      int d, aw, ah;
      cell_pos(f, cell, bw, bh, d, aw, ah);
      const long long j = ((long long)ah * f.G_w + aw) * f.C + d;
      const Iv Br{rlo[so + j], rhi[so + j]};
      const double t = upper ? corner_hi(c, Br) : corner_lo(c, Br);
      S += t;
      A += fabs(t);
      N += 1.0;
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) {
    S += __shfl_down_sync(0xffffffffu, S, o);
    A += __shfl_down_sync(0xffffffffu, A, o);
    N += __shfl_down_sync(0xffffffffu, N, o);
  }
  if (lane == 0) {
    s_red[0][warp] = S;
    s_red[1][warp] = A;
    s_red[2][warp] = N;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0, a = 0.0, nn = 0.0;
    for (int w = 0; w < kPT / 32; ++w) {
      s += s_red[0][w];
      a += s_red[1][w];
      nn += s_red[2][w];
    }
    double* P = part + ((size_t)i * ntiles + blockIdx.x) * 3;
    P[0] = s;
    P[1] = a;
    P[2] = nn;
  }
}

// The predicted offers: certain freezes dropped, the survivors' row map,
// query list and count written like k_offer's (stable order). Phase 1: a
// thread per row pair (upper r, lower R + r) sums the partials and decides;
// phase 2: block scan over the decisions (dynamic shared memory: one flag
// per row of the launch bound).
__device__ __forceinline__ int pred_decide(double S, double A, double N, double k0, double pe, bool upper) {
  S += k0;
  A = __dadd_ru(A, __dadd_ru(fabs(k0), pe));
  if (!(fabs(S) < 1e300) || !(A < 1e300)) return 0;
  const double B = __dmul_ru(A, 1.0 + 0x1p-30);
  // 2.5 ulp per outward link + the parallel sum's error, relative to B,
  // plus an absolute ulp floor per link for the subnormal range
  const double E = __dadd_ru(pe, __dmul_ru(4.0 * (N + 2.0), __dadd_ru(__dmul_ru(0x1p-52, B), 0x1p-1074)));
  if (!(E < 1e300)) return 0;
  const double up = __dadd_ru(S, E), dn = __dadd_rd(S, -E);
  // +1: the raw value is proven to freeze the row (upper <= 0 / lower >= 0),
  // -1: proven not to, 0: undecided
  if (upper) return up <= 0.0 ? 1 : dn > 0.0 ? -1 : 0;
  return dn >= 0.0 ? 1 : up < 0.0 ? -1 : 0;
}

__global__ void __launch_bounds__(kPredScan)
    k_pred_offer(RowsDev rows, int R, MatDev m, const double* P, const double* part, int ntiles,
                 const char* frozen, int* map, int* new_R, int* new_row_q) {
  using Scan = cub::BlockScan<int, kPredScan>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int s_base;
  extern __shared__ unsigned char s_keep[];
  if (rows.dR) R = *rows.dR;  // device-applied compaction: the live rows of this checkpoint
  if (threadIdx.x == 0) s_base = 0;
  // a thread per row pair: the loads of a row are independent (row list,
  // freeze flag, partials, predicted constants), so each thread's latency is
  // about one memory round trip
  for (int r = threadIdx.x; r < R; r += kPredScan) {
    const int q = rows.row_q[r];
    const size_t p0 = phys_row(m, r), p1 = phys_row(m, R + r);
    double k0, e0 = 0.0, k1, e1 = 0.0;
    if (P) {  // predicted raw constants and their error radii (k_pk_*)
      k0 = P[2 * p0];
      e0 = P[2 * p0 + 1];
      k1 = P[2 * p1];
      e1 = P[2 * p1 + 1];
    } else {
      k0 = m.K[4 * p0 + 3];  // kraw.hi
      k1 = m.K[4 * p1 + 2];  // kraw.lo
    }
    double S0 = 0.0, A0 = 0.0, N0 = 0.0, S1 = 0.0, A1 = 0.0, N1 = 0.0;
    const double* q0 = part + (size_t)r * ntiles * 3;
    const double* q1 = part + (size_t)(R + r) * ntiles * 3;
#pragma unroll 4
    for (int t = 0; t < ntiles; ++t) {
      S0 += q0[3 * t];
      A0 += q0[3 * t + 1];
      N0 += q0[3 * t + 2];
      S1 += q1[3 * t];
      A1 += q1[3 * t + 1];
      N1 += q1[3 * t + 2];
    }
    // undecided rows stay; should the exact offers freeze them, their later
    // work is not counted (launch_count_affine reads the exact freezes in
    // stream order) and their results are ignored
    const bool gone = (frozen && frozen[q]) || pred_decide(S0, A0, N0, k0, e0, true) == 1 ||
                      pred_decide(S1, A1, N1, k1, e1, false) == 1;
    s_keep[r] = gone ? 0 : 1;
  }
  __syncthreads();
  for (int start = 0; start < R; start += kPredScan) {
    const int r = start + threadIdx.x;
    int keep = 0, q = 0;
    if (r < R) {
      q = rows.row_q[r];
      keep = s_keep[r];
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
  const int nR = s_base;
  for (int p = threadIdx.x; p < nR; p += blockDim.x) map[nR + p] = R + map[p];  // lower rows
  if (threadIdx.x == 0) *new_R = nR;
}

void launch_pred_offer(cudaStream_t s, const RowsDev& rows, int R, const FrameDev& f, MatDev m,
                       const double* P, const double* rlo, const double* rhi, const char* frozen, int* map,
                       int* new_R, int* new_row_q) {
  const int ntiles = (int)((m.cells + kPT * 4 - 1) / (kPT * 4));
  double* part = static_cast<double*>(stream_scratch(s, (size_t)rows.n * ntiles * 3 * sizeof(double)));
  k_pred_terms<<<dim3(ntiles, rows.n), kPT, 0, s>>>(rows, f, m, rlo, rhi, part, ntiles, frozen);
  k_pred_offer<<<1, kPredScan, rows.n_up + 16, s>>>(rows, R, m, P, part, ntiles, frozen, map, new_R, new_row_q);
  g_launches += 2;
}

// The predicted offers from partial sums a conv kernel already produced
// (k_gbc_flat with FlatDev::part: nparts per row).
void launch_pred_offer_parts(cudaStream_t s, const RowsDev& rows, int R, MatDev m, const double* P,
                             const double* part, int nparts, const char* frozen, int* map, int* new_R,
                             int* new_row_q) {
  k_pred_offer<<<1, kPredScan, rows.n_up + 16, s>>>(rows, R, m, P, part, nparts, frozen, map, new_R, new_row_q);
  ++g_launches;
}

// ---------------------------------------------------------------------------
// Predicted raw constants. The predicted offers need each row's raw constant
// (kraw.hi of an upper row, kraw.lo of a lower one), which the serial chain
// folds produce last. To keep the coefficient stream from waiting on them,
// a prediction stream carries P = (S, E) per row through the walk: a
// parallel sum S of the same terms the chain adds and a radius E with
// |exact chain value - S| <= E. Each step with n terms t_j (the affine
// step's bias products, the relu step's offset products, a join's branch
// constant) widens it, with B = |S_in| + E_in + sum |t_j| bounding every
// partial result of the chain, by the bound of k_pred_offer:
//   E_out = E_in + 4 (n + 2) (2^-52 B + 2^-1074).
// Rows are never skipped here (a row frozen by the exact offers may still
// sit in the map; its prediction stays valid).
__device__ __forceinline__ void pk_widen(const double* Pin, double S, double A, double N, double* Pout) {
  const double ps = Pin ? Pin[0] : 0.0, pe = Pin ? Pin[1] : 0.0;
  const double s = ps + S;
  const double B = __dmul_ru(__dadd_ru(__dadd_ru(fabs(ps), pe), A), 1.0 + 0x1p-30);
  const double e = __dadd_ru(pe, __dmul_ru(4.0 * (N + 2.0), __dadd_ru(__dmul_ru(0x1p-52, B), 0x1p-1074)));
  const bool ok = fabs(s) < 1e300 && e < 1e300 && N < 0x1p22;
  Pout[0] = ok ? s : 0.0;
  Pout[1] = ok ? e : INFINITY;
}

template <int NT>
__device__ __forceinline__ void block_sum3(double& S, double& A, double& N, double (*red)[NT / 32]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) {
    S += __shfl_down_sync(0xffffffffu, S, o);
    A += __shfl_down_sync(0xffffffffu, A, o);
    N += __shfl_down_sync(0xffffffffu, N, o);
  }
  if (lane == 0) {
    red[0][warp] = S;
    red[1][warp] = A;
    red[2][warp] = N;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    S = A = N = 0.0;
    for (int w = 0; w < NT / 32; ++w) {
      S += red[0][w];
      A += red[1][w];
      N += red[2][w];
    }
  }
}

// affine step (dense_step / gbc_step constants, backsub.hpp:375-392, 469-486):
// raw track terms iv_mul_scalar(c, bias).hi (upper rows) / .lo (lower rows)
__global__ void __launch_bounds__(kPT)
    k_pk_affine_terms(LayerDev L, int is_conv, RowsDev rows, FrameDev f, MatDev m, double* part, int ntiles) {
  __shared__ double s_red[3][kPT / 32];
  int i;
  if (!rows_resolve(rows, blockIdx.y, i)) return;
  bool upper;
  int img;
  const int q = row_query(rows, i, upper, img);
  int bw, bh;
  frame_base(f, q, bw, bh);
  const size_t pr = phys_row(m, i);
  const double* lo = m.lo + pr * m.cells;
  const double* hi = m.hi + pr * m.cells;
  double S = 0.0, A = 0.0, N = 0.0;
  const long long c0 = (long long)blockIdx.x * (kPT * 4);
  for (int k = 0; k < 4; ++k) {
    const long long cell = c0 + (long long)k * kPT + threadIdx.x;
    if (cell >= m.cells) break;
    const Iv c{lo[cell], hi[cell]};
    if (iv_zero(c)) continue;
    double b;
    if (is_conv) {
      int d, aw, ah;
      cell_pos(f, cell, bw, bh, d, aw, ah);
      b = L.bias[d];
    } else {
      b = L.bias[cell];
    }
    const Iv bt = iv_mul_scalar(c, b);
    if (iv_zero(bt)) continue;
    const double t = upper ? bt.hi : bt.lo;
    S += t;
    A += fabs(t);
    N += 1.0;
  }
  block_sum3<kPT>(S, A, N, s_red);
  if (threadIdx.x == 0) {
    double* Pp = part + ((size_t)i * ntiles + blockIdx.x) * 3;
    Pp[0] = S;
    Pp[1] = A;
    Pp[2] = N;
  }
}

__global__ void k_pk_affine_fin(RowsDev rows, MatDev m, const double* Pin, const double* part, int ntiles,
                                double* Pout) {
  int i;
  if (!rows_resolve(rows, blockIdx.x * blockDim.x + threadIdx.x, i)) return;
  double S = 0.0, A = 0.0, N = 0.0;
  for (int t = 0; t < ntiles; ++t) {
    const double* Pp = part + ((size_t)i * ntiles + t) * 3;
    S += Pp[0];
    A += Pp[1];
    N += Pp[2];
  }
  pk_widen(Pin + 2 * phys_row(m, i), S, A, N, Pout + 2 * (size_t)i);
}

void launch_pk_affine(cudaStream_t s, const LayerDev& L, bool is_conv, const RowsDev& rows, const FrameDev& f,
                      MatDev m, const double* Pin, double* Pout) {
  const int ntiles = (int)((m.cells + kPT * 4 - 1) / (kPT * 4));
  double* part = static_cast<double*>(stream_scratch(s, (size_t)rows.n * ntiles * 3 * sizeof(double)));
  k_pk_affine_terms<<<dim3(ntiles, rows.n), kPT, 0, s>>>(L, is_conv ? 1 : 0, rows, f, m, part, ntiles);
  k_pk_affine_fin<<<(rows.n + 127) / 128, 128, 0, s>>>(rows, m, Pin, part, ntiles, Pout);
  g_launches += 2;
}

// relu step (backsub.hpp:536-563) over the layer's offset list, like
// k_chain_relu_list: raw track terms o0 then o1 (.hi upper / .lo lower)
constexpr int kPkWarps = 4;
__global__ void __launch_bounds__(32 * kPkWarps)
    k_pk_relu(RowsDev rows, FrameDev f, MatDev m, const double* Pin, double* Pout, const double* relax,
              const int* list, const int* count, int cstride) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int i;
  if (!rows_resolve(rows, blockIdx.x * kPkWarps + warp, i)) return;
  bool upper;
  int img;
  const int q = row_query(rows, i, upper, img);
  relax += 8 * img * rows.sst;
  list += img * rows.sst;
  const int n = count[img * cstride];
  int bw, bh;
  frame_base(f, q, bw, bh);
  const size_t pr = phys_row(m, i);
  const double* lo = m.lo + pr * m.cells;
  const double* hi = m.hi + pr * m.cells;
  const int GC = f.G_w * f.C;
  double S = 0.0, A = 0.0, N = 0.0;
  for (int e = lane; e < n; e += 32) {
    const int j = list[e];
    const int ah = j / GC, rem = j - ah * GC;
    const int aw = rem / f.C, d = rem - aw * f.C;
    const int x = aw - bw, y = ah - bh;
    if (x < 0 || x >= f.S_w || y < 0 || y >= f.S_h) continue;
    const long long cell = ((long long)y * f.S_w + x) * f.C + d;
    const Iv c{lo[cell], hi[cell]};
    if (iv_zero(c)) continue;
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
    if (!iv_zero(o0)) {
      const double t = upper ? o0.hi : o0.lo;
      S += t;
      A += fabs(t);
      N += 1.0;
    }
    if (!iv_zero(o1)) {
      const double t = upper ? o1.hi : o1.lo;
      S += t;
      A += fabs(t);
      N += 1.0;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    S += __shfl_down_sync(0xffffffffu, S, o);
    A += __shfl_down_sync(0xffffffffu, A, o);
    N += __shfl_down_sync(0xffffffffu, N, o);
  }
  if (lane == 0) pk_widen(Pin + 2 * pr, S, A, N, Pout + 2 * (size_t)i);
}

void launch_pk_relu(cudaStream_t s, const RowsDev& rows, const FrameDev& f, MatDev m, const double* Pin,
                    double* Pout, const double* relax, const int* list, const int* count, int cstride) {
  k_pk_relu<<<(rows.n + kPkWarps - 1) / kPkWarps, 32 * kPkWarps, 0, s>>>(rows, f, m, Pin, Pout, relax, list,
                                                                       count, cstride);
  ++g_launches;
}

// join (align_add, backsub.hpp:610-688): one link, branch a's constant plus b's
__global__ void k_pk_merge(RowsDev rows, MatDev a, const double* Pa, MatDev b, const double* Pb, double* Pout) {
  int i;
  if (!rows_resolve(rows, blockIdx.x * blockDim.x + threadIdx.x, i)) return;
  const double* pb = Pb + 2 * phys_row(b, i);
  double* po = Pout + 2 * (size_t)i;
  pk_widen(Pa + 2 * phys_row(a, i), pb[0], __dadd_ru(fabs(pb[0]), pb[1]), 1.0, po);
  po[1] = __dadd_ru(po[1], pb[1]);
  if (!(po[1] < 1e300)) {
    po[0] = 0.0;
    po[1] = INFINITY;
  }
}

void launch_pk_merge(cudaStream_t s, const RowsDev& rows, MatDev a, const double* Pa, MatDev b, const double* Pb,
                     double* Pout) {
  k_pk_merge<<<(rows.n + 127) / 128, 128, 0, s>>>(rows, a, Pa, b, Pb, Pout);
  ++g_launches;
}

// a walk's first rows: the exact constants, radius 0
__global__ void k_pk_init(RowsDev rows, MatDev m, double* Pout) {
  int i;
  if (!rows_resolve(rows, blockIdx.x * blockDim.x + threadIdx.x, i)) return;
  bool upper;
  int img;
  row_query(rows, i, upper, img);
  const double* K = m.K + 4 * phys_row(m, i);
  const double k = upper ? K[3] : K[2];
  double* po = Pout + 2 * (size_t)phys_row(m, i);
  const bool ok = fabs(k) < 1e300;
  po[0] = ok ? k : 0.0;
  po[1] = ok ? 0.0 : INFINITY;
}

void launch_pk_init(cudaStream_t s, const RowsDev& rows, MatDev m, double* P) {
  k_pk_init<<<(rows.n + 127) / 128, 128, 0, s>>>(rows, m, P);
  ++g_launches;
}

// PassStats work of an affine step (dense_madds / gbc_madds: the in-grid
// taps of every nonzero coefficient, backsub.hpp:386,483; gbc_dense_equiv)
// for the rows the reference still walks. With predicted compaction the
// chain kernels on s2 cannot know whether the exact offers (s3) froze a
// row the prediction kept, so the counting runs here, on s3, in stream
// order behind those offers.
__global__ void __launch_bounds__(kPT)
    k_count_affine(LayerDev L, int is_conv, RowsDev rows, FrameDev f, MatDev m, const char* frozen,
                   Counters* ctr) {
  int i;
  if (!rows_resolve(rows, blockIdx.y, i)) return;
  bool upper;
  int img;
  const int q = row_query(rows, i, upper, img);
  if (frozen && frozen[(size_t)img * rows.kq + q]) return;
  ctr += img;
  int bw = 0, bh = 0;
  if (is_conv) frame_base(f, q, bw, bh);
  const size_t pr = phys_row(m, i);
  const double* lo = m.lo + pr * m.cells;
  const double* hi = m.hi + pr * m.cells;
  unsigned long long md = 0;
  const long long c0 = (long long)blockIdx.x * (kPT * 4);
  for (int k = 0; k < 4; ++k) {
    const long long cell = c0 + (long long)k * kPT + threadIdx.x;
    if (cell >= m.cells) break;
    if (iv_zero(Iv{lo[cell], hi[cell]})) continue;
    if (is_conv) {
      int d, aw, ah;
      cell_pos(f, cell, bw, bh, d, aw, ah);
      const int y0 = ah * L.sh - L.ph, x0 = aw * L.sw - L.pw;
      const int ny = min(L.fh, L.in_h - y0) - max(0, -y0);
      const int nx = min(L.fw, L.in_w - x0) - max(0, -x0);
      if (ny > 0 && nx > 0) md += (unsigned long long)L.in_c * ny * nx;
    } else {
      md += (unsigned long long)L.in_w * L.in_h * L.in_c;
    }
  }
  for (int o = 16; o > 0; o >>= 1) md += __shfl_down_sync(0xffffffffu, md, o);
  if ((threadIdx.x & 31) == 0 && md) atomicAdd(is_conv ? &ctr->gbc_madds : &ctr->dense_madds, md);
  if (is_conv && blockIdx.x == 0 && threadIdx.x == 0)
    atomicAdd(&ctr->gbc_dense_equiv, (unsigned long long)L.out_w * L.out_h * L.out_c *
                                         ((unsigned long long)L.in_w * L.in_h * L.in_c));
}

void launch_count_affine(cudaStream_t s, const LayerDev& L, bool is_conv, const RowsDev& rows, const FrameDev& f,
                         MatDev m, const char* frozen, Counters* ctr) {
  const int ntiles = (int)((m.cells + kPT * 4 - 1) / (kPT * 4));
  k_count_affine<<<dim3(ntiles, rows.n), kPT, 0, s>>>(L, is_conv ? 1 : 0, rows, f, m, frozen, ctr);
  ++g_launches;
}

static void set_attrs_split() {
  cudaFuncSetAttribute(k_affine_fold, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(5 * 2 * kTTile * sizeof(double)));
  cudaFuncSetAttribute(k_conc_fold, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(2 * 2 * kTTile * sizeof(double)));
}

static bool split_chains(cudaStream_t s, long long cells, int nrows, int na, double** tb, int** tc,
                         long long* tstride, int* ntiles) {
  static const int on = [] {
    const char* e = getenv("PC_SPLIT_CHAINS");
    return e && *e ? atoi(e) : 1;
  }();
  // rows shorter than a few tiles fold faster in one CTA-per-row kernel
  static const long long min_cells = [] {
    const char* e = getenv("PC_SPLIT_MIN_CELLS");
    return e && *e ? atoll(e) : 1024ll;
  }();
  if (!on || cells < min_cells) return false;
  *ntiles = (int)((cells + kTTile - 1) / kTTile);
  *tstride = (long long)*ntiles * kTTile;
  const size_t tb_bytes = (size_t)nrows * na * (size_t)*tstride * sizeof(double);
  const size_t tc_bytes = (size_t)nrows * *ntiles * sizeof(int);
  char* p = static_cast<char*>(stream_scratch(s, tb_bytes + tc_bytes + 512 + (size_t)nrows * 5 * sizeof(double)));
  if (!p) return false;
  *tb = reinterpret_cast<double*>(p);
  *tc = reinterpret_cast<int*>(p + ((tb_bytes + 255) & ~(size_t)255));
  return true;
}

template <class G>
constexpr size_t chain_smem() {
  return (size_t)(2 * G::NA + 2 * kStages) * Roles<G>::kTile * sizeof(double);  // terms + coefficient ring
}

static void set_attrs_split();
static void set_attrs() {
  set_attrs_split();
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

cudaError_t scan_stats_device_chains(int on, unsigned long long* out4) {
  cudaError_t e = cudaSuccess;
  if (out4) e = cudaMemcpyFromSymbol(out4, g_scan_stats, sizeof(unsigned long long) * 8);
  const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_scan_stats, z, sizeof(z));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_scan_stats_on, &on, sizeof(int));
  return e;
}

void launch_chain_affine_big(cudaStream_t s, const LayerDev& L, bool is_conv, const RowsDev& rows,
                             const FrameDev& fin, MatDev m, double* Kout, const double* dev,
                             Counters* ctr, const char* frozen, bool fast) {
  if (debug_skip("folds")) return;
  double* tb;
  int* tc;
  long long ts;
  int nt;
  if (split_chains(s, m.cells, rows.n, 3, &tb, &tc, &ts, &nt)) {
    k_affine_terms<<<dim3(nt, rows.n), kTT, 0, s>>>(L, is_conv ? 1 : 0, rows, fin, m, dev, tb, tc, ts, nt, ctr,
                                                   frozen, fast ? 1 : 0);
    if (rows.n <= block_fold_rows() && nt <= kMaxFoldTiles) {
      double* tmp = reinterpret_cast<double*>(reinterpret_cast<char*>(tc) + (((size_t)rows.n * nt * sizeof(int) + 255) & ~(size_t)255));
      k_affine_fold_block<<<dim3(rows.n, 5), kFB, 0, s>>>(rows, m, tmp, tb, tc, ts, nt, frozen, fast ? 1 : 0);
      k_affine_finish<<<(rows.n + 127) / 128, 128, 0, s>>>(rows, tmp, Kout, frozen);
      g_launches += 3;
      return;
    }
    k_affine_fold<<<rows.n, 160, 5 * 2 * kTTile * sizeof(double), s>>>(rows, m, Kout, tb, tc, ts, nt, frozen,
                                                                       fast ? 1 : 0);
    g_launches += 2;
    return;
  }
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
                           const double* rhi, double* vals, double* rvals, const char* frozen, bool fast) {
  if (debug_skip("folds")) return;
  double* tb;
  int* tc;
  long long ts;
  int nt;
  if (split_chains(s, m.cells, rows.n, 2, &tb, &tc, &ts, &nt)) {
    k_conc_terms<<<dim3(nt, rows.n), kTT, 0, s>>>(rows, f, m, blo, bhi, rlo, rhi, tb, tc, ts, nt, frozen,
                                                 fast ? 1 : 0);
    if (rows.n <= block_fold_rows() && nt <= kMaxFoldTiles)
      k_conc_fold_block<<<dim3(rows.n, 2), kFB, 0, s>>>(rows, m, vals, rvals, tb, tc, ts, nt, frozen, fast ? 1 : 0);
    else
      k_conc_fold<<<rows.n, 64, 2 * 2 * kTTile * sizeof(double), s>>>(rows, m, vals, rvals, tb, tc, ts, nt, frozen,
                                                                      fast ? 1 : 0);
    g_launches += 2;
    return;
  }
  k_concretize_big<<<rows.n, kCT, chain_smem<ConcGen>(), s>>>(rows, f, m, blo, bhi, rlo, rhi, vals,
                                                               rvals, frozen);
  ++g_launches;
}

}  // namespace pc
