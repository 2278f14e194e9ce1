// numeric.cuh — device restatement of the reference's WidenedFloat64 scalar
// mode and interval helpers (proj/include/polycert/interval.hpp:38-267,
// backsub.hpp:151-194), bit-exact.
//
// Rule being reproduced (interval.hpp:23-37): every op returns the
// round-to-nearest result, stepped one representable value outward
// (std::nextafter) iff the op was inexact; exactness is decided by TwoSum for
// sums and by an FMA residual (with a 2^-500 floor) for products/quotients.
//
// Fast paths use sm_100a directed-rounding adds: for finite operands below
// 2^1020, TwoSum is exact (no intermediate overflow), so "exact" is
// equivalent to __dadd_rd == __dadd_ru, and an inexact sum is never
// subnormal, so nextafter(s, ±inf) == s ± denorm_min rounded outward. Every
// other case takes a slow path that restates the reference operation by
// operation. tests/test_gpu_numeric.py checks both paths against the
// reference on edge-case and random operands.
#pragma once
#include <cstdint>

namespace pc {

constexpr double kTiny = 4.9406564584124654e-324;  // denorm_min
constexpr double kFloor = 0x1p-500;                 // interval.hpp:48
constexpr double kBig = 0x1p1020;
constexpr double kInf = __builtin_huge_val();

// std::nextafter(x, +inf) / (x, -inf) on the bit pattern.
__device__ __forceinline__ double nextup_bits(double x) {
  if (x != x || x == kInf) return x;
  if (x == 0.0) return kTiny;
  long long b = __double_as_longlong(x);
  b += (b < 0) ? -1 : 1;
  return __longlong_as_double(b);
}
__device__ __forceinline__ double nextdown_bits(double x) {
  if (x != x || x == -kInf) return x;
  if (x == 0.0) return -kTiny;
  long long b = __double_as_longlong(x);
  b += (b < 0) ? 1 : -1;
  return __longlong_as_double(b);
}

// interval.hpp:50-57, restated with non-contracted ops.
__device__ __forceinline__ bool sum_exact_ref(double a, double b, double s) {
  if (!isfinite(s)) return false;
  const double a1 = __dsub_rn(s, b);
  const double b1 = __dsub_rn(s, a1);
  const double da = __dsub_rn(a, a1);
  const double db = __dsub_rn(b, b1);
  return __dadd_rn(da, db) == 0.0;
}

static __device__ __noinline__ double add_up_slow(double a, double b) {
  const double s = __dadd_rn(a, b);
  if (s != s) return kInf;
  return sum_exact_ref(a, b, s) ? s : nextup_bits(s);
}
static __device__ __noinline__ double add_down_slow(double a, double b) {
  const double s = __dadd_rn(a, b);
  if (s != s) return -kInf;
  return sum_exact_ref(a, b, s) ? s : nextdown_bits(s);
}

// add_up / add_down (interval.hpp:59-68)
__device__ __forceinline__ double add_up(double a, double b) {
  if (fabs(a) < kBig && fabs(b) < kBig) {
    const double s = __dadd_rn(a, b);
    const double rd = __dadd_rd(a, b);
    const double ru = __dadd_ru(a, b);
    return (rd == ru) ? s : __dadd_ru(s, kTiny);
  }
  return add_up_slow(a, b);
}
__device__ __forceinline__ double add_down(double a, double b) {
  if (fabs(a) < kBig && fabs(b) < kBig) {
    const double s = __dadd_rn(a, b);
    const double rd = __dadd_rd(a, b);
    const double ru = __dadd_ru(a, b);
    return (rd == ru) ? s : __dadd_rd(s, -kTiny);
  }
  return add_down_slow(a, b);
}
// Direction-generic (branch-free fast path) for chains whose lanes mix
// add_up and add_down: identical results to add_up / add_down.
__device__ __forceinline__ double add_dir(double a, double b, bool up) {
  if (fabs(a) < kBig && fabs(b) < kBig) {
    const double s = __dadd_rn(a, b);
    const double rd = __dadd_rd(a, b);
    const double ru = __dadd_ru(a, b);
    const double st = up ? __dadd_ru(s, kTiny) : __dadd_rd(s, -kTiny);
    return (rd == ru) ? s : st;
  }
  return up ? add_up_slow(a, b) : add_down_slow(a, b);
}

// mul_up / mul_down (interval.hpp:74-83)
__device__ __forceinline__ double mul_up(double a, double b) {
  if (a == 0.0 || b == 0.0) return 0.0;
  const double p = __dmul_rn(a, b);
  const double r = __fma_rn(a, b, -p);
  const double ap = fabs(p);
  if (ap >= kFloor && ap < kInf) return (r == 0.0) ? p : __dadd_ru(p, kTiny);
  return nextup_bits(p);  // non-finite or below the residual floor: always inexact
}
__device__ __forceinline__ double mul_down(double a, double b) {
  if (a == 0.0 || b == 0.0) return 0.0;
  const double p = __dmul_rn(a, b);
  const double r = __fma_rn(a, b, -p);
  const double ap = fabs(p);
  if (ap >= kFloor && ap < kInf) return (r == 0.0) ? p : __dadd_rd(p, -kTiny);
  return nextdown_bits(p);
}

// div_up / div_down (interval.hpp:84-96); only the relaxation uses these.
__device__ __forceinline__ double div_up(double a, double b) {
  if (a == 0.0) return 0.0;
  const double q = __ddiv_rn(a, b);
  const bool exact = isfinite(q) && fabs(a) >= kFloor && __fma_rn(q, b, -a) == 0.0;
  return exact ? q : nextup_bits(q);
}
__device__ __forceinline__ double div_down(double a, double b) {
  if (a == 0.0) return 0.0;
  const double q = __ddiv_rn(a, b);
  const bool exact = isfinite(q) && fabs(a) >= kFloor && __fma_rn(q, b, -a) == 0.0;
  return exact ? q : nextdown_bits(q);
}

// ulp_above (interval.hpp:98-102)
__device__ __forceinline__ double ulp_above(double x) {
  const double m = fabs(x);
  if (!isfinite(m)) return kInf;
  return __dsub_rn(nextup_bits(m), m);
}

// std::max / std::min argument-order semantics (first operand on ties).
__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }
__device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }

struct Iv {
  double lo, hi;
};

__device__ __forceinline__ bool iv_zero(const Iv& a) { return a.lo == 0.0 && a.hi == 0.0; }
__device__ __forceinline__ double iv_mag(const Iv& a) { return smax(fabs(a.lo), fabs(a.hi)); }

// iv_acc (interval.hpp:185-195)
__device__ __forceinline__ void iv_acc(Iv& a, const Iv& b) {
  if (iv_zero(b)) return;
  a.lo = add_down(a.lo, b.lo);
  a.hi = add_up(a.hi, b.hi);
}
__device__ __forceinline__ Iv iv_add(const Iv& a, const Iv& b) {
  return Iv{add_down(a.lo, b.lo), add_up(a.hi, b.hi)};
}
// iv_mul_scalar (interval.hpp:197-208)
__device__ __forceinline__ Iv iv_mul_scalar(const Iv& a, double w) {
  if (w == 0.0 || iv_zero(a)) return Iv{0.0, 0.0};
  if (w > 0.0) return Iv{mul_down(a.lo, w), mul_up(a.hi, w)};
  return Iv{mul_down(a.hi, w), mul_up(a.lo, w)};
}
// iv_mul (interval.hpp:210-226)
__device__ __forceinline__ Iv iv_mul(const Iv& a, const Iv& b) {
  if (iv_zero(a) || iv_zero(b)) return Iv{0.0, 0.0};
  const double l1 = mul_down(a.lo, b.lo), l2 = mul_down(a.lo, b.hi);
  const double l3 = mul_down(a.hi, b.lo), l4 = mul_down(a.hi, b.hi);
  const double u1 = mul_up(a.lo, b.lo), u2 = mul_up(a.lo, b.hi);
  const double u3 = mul_up(a.hi, b.lo), u4 = mul_up(a.hi, b.hi);
  return Iv{smin(smin(l1, l2), smin(l3, l4)), smax(smax(u1, u2), smax(u3, u4))};
}
// Upper endpoint only of iv_mul (for chains that track one endpoint).
__device__ __forceinline__ double iv_mul_hi(const Iv& a, const Iv& b) {
  const double u1 = mul_up(a.lo, b.lo), u2 = mul_up(a.lo, b.hi);
  const double u3 = mul_up(a.hi, b.lo), u4 = mul_up(a.hi, b.hi);
  return smax(smax(u1, u2), smax(u3, u4));
}
__device__ __forceinline__ double iv_mul_lo(const Iv& a, const Iv& b) {
  const double l1 = mul_down(a.lo, b.lo), l2 = mul_down(a.lo, b.hi);
  const double l3 = mul_down(a.hi, b.lo), l4 = mul_down(a.hi, b.hi);
  return smin(smin(l1, l2), smin(l3, l4));
}
// iv_div (interval.hpp:230-247), divisor > 0 by construction.
__device__ __forceinline__ Iv iv_div(const Iv& a, const Iv& b) {
  if (iv_zero(a)) return Iv{0.0, 0.0};
  const double l1 = div_down(a.lo, b.lo), l2 = div_down(a.lo, b.hi);
  const double l3 = div_down(a.hi, b.lo), l4 = div_down(a.hi, b.hi);
  const double u1 = div_up(a.lo, b.lo), u2 = div_up(a.lo, b.hi);
  const double u3 = div_up(a.hi, b.lo), u4 = div_up(a.hi, b.hi);
  return Iv{smin(smin(l1, l2), smin(l3, l4)), smax(smax(u1, u2), smax(u3, u4))};
}
__device__ __forceinline__ Iv iv_pos_part(const Iv& a) { return Iv{smax(a.lo, 0.0), smax(a.hi, 0.0)}; }
__device__ __forceinline__ Iv iv_neg_part(const Iv& a) { return Iv{smin(a.lo, 0.0), smin(a.hi, 0.0)}; }

// detail::corner_hi / corner_lo (backsub.hpp:151-171)
__device__ __forceinline__ double corner_hi(const Iv& a, const Iv& b) {
  double v = mul_up(a.lo, b.lo);
  v = smax(v, mul_up(a.lo, b.hi));
  v = smax(v, mul_up(a.hi, b.lo));
  v = smax(v, mul_up(a.hi, b.hi));
  return v;
}
__device__ __forceinline__ double corner_lo(const Iv& a, const Iv& b) {
  double v = mul_down(a.lo, b.lo);
  v = smin(v, mul_down(a.lo, b.hi));
  v = smin(v, mul_down(a.hi, b.lo));
  v = smin(v, mul_down(a.hi, b.hi));
  return v;
}

// Relaxation record (backsub.hpp:61-64): alpha, beta, gamma, delta.
struct Relax {
  Iv alpha, beta, gamma, delta;
};

// relu_relaxation (analyzer.hpp:38-70), from PADDED bounds.
__device__ __forceinline__ Relax relu_relaxation(const Iv& b) {
  Relax r;
  const Iv one{1.0, 1.0}, zero{0.0, 0.0};
  if (!(b.lo < 0.0)) {
    r.alpha = one; r.beta = zero; r.gamma = one; r.delta = zero;
  } else if (!(b.hi > 0.0)) {
    r.alpha = zero; r.beta = zero; r.gamma = zero; r.delta = zero;
  } else {
    const Iv den = iv_add(Iv{b.hi, b.hi}, Iv{-b.lo, -b.lo});  // iv_sub(point(hi), point(lo))
    r.gamma = iv_div(Iv{b.hi, b.hi}, den);
    const Iv num = iv_mul(Iv{-b.lo, -b.lo}, Iv{b.hi, b.hi});
    r.delta = iv_div(num, den);
    r.alpha = b.hi > -b.lo ? one : zero;
    r.beta = zero;
  }
  return r;
}

// ---------------------------------------------------------------------------
// Branch-free fast paths ("f_" ops) for hot loops.
//
// Valid (bit-identical to the exact ops above) while every product magnitude
// lies in [2^-1020, 2^980) and every sum operand below 2^1020. In that band
// nextafter(p, -inf) == RM(p - denorm_min) and nextafter(p, +inf) ==
// RP(p + denorm_min) exactly, and TwoSum cannot overflow. Callers accumulate a
// `bad` flag from f_mul_* and verify chain starting values; when it is set,
// the affected output is recomputed with the exact ops (same order), so the
// result is always the reference's. Sums are safe when the terms are checked
// and chains start below 2^1000: partial sums then stay below 2^1020 for
// any chain shorter than 2^39 terms.
// ---------------------------------------------------------------------------
constexpr double kSafeHi = 0x1p980;
constexpr double kSafeLo = 0x1p-1020;
constexpr double kStartHi = 0x1p1000;

__device__ __forceinline__ double f_add_up(double a, double b) {
  const double s = __dadd_rn(a, b);
  const double rd = __dadd_rd(a, b), ru = __dadd_ru(a, b);
  const double st = __dadd_ru(s, kTiny);
  return (rd == ru) ? s : st;
}
__device__ __forceinline__ double f_add_dn(double a, double b) {
  const double s = __dadd_rn(a, b);
  const double rd = __dadd_rd(a, b), ru = __dadd_ru(a, b);
  const double st = __dadd_rd(s, -kTiny);
  return (rd == ru) ? s : st;
}
__device__ __forceinline__ double f_add_dir(double a, double b, bool up) {
  const double s = __dadd_rn(a, b);
  const double rd = __dadd_rd(a, b), ru = __dadd_ru(a, b);
  const double st = up ? __dadd_ru(s, kTiny) : __dadd_rd(s, -kTiny);
  return (rd == ru) ? s : st;
}
__device__ __forceinline__ bool out_of_band(double p) {
  const double ap = fabs(p);
  return !(ap < kSafeHi) | (ap < kSafeLo);
}
// Products where either factor may be zero (zero short-circuit, exact 0).
__device__ __forceinline__ double f_mul_up(double a, double b, bool& bad) {
  const double p = __dmul_rn(a, b);
  const double r = __fma_rn(a, b, -p);
  const bool z = (a == 0.0) | (b == 0.0);
  bad |= !z & out_of_band(p);
  const double v = ((r == 0.0) & (fabs(p) >= kFloor)) ? p : __dadd_ru(p, kTiny);
  return z ? 0.0 : v;
}
__device__ __forceinline__ double f_mul_dn(double a, double b, bool& bad) {
  const double p = __dmul_rn(a, b);
  const double r = __fma_rn(a, b, -p);
  const bool z = (a == 0.0) | (b == 0.0);
  bad |= !z & out_of_band(p);
  const double v = ((r == 0.0) & (fabs(p) >= kFloor)) ? p : __dadd_rd(p, -kTiny);
  return z ? 0.0 : v;
}
// Products of two nonzero factors.
__device__ __forceinline__ double f_mul_up_nz(double a, double b, bool& bad) {
  const double p = __dmul_rn(a, b);
  const double r = __fma_rn(a, b, -p);
  bad |= out_of_band(p);
  return ((r == 0.0) & (fabs(p) >= kFloor)) ? p : __dadd_ru(p, kTiny);
}
__device__ __forceinline__ double f_mul_dn_nz(double a, double b, bool& bad) {
  const double p = __dmul_rn(a, b);
  const double r = __fma_rn(a, b, -p);
  bad |= out_of_band(p);
  return ((r == 0.0) & (fabs(p) >= kFloor)) ? p : __dadd_rd(p, -kTiny);
}
__device__ __forceinline__ double f_corner_hi(const Iv& a, const Iv& b, bool& bad) {
  double v = f_mul_up(a.lo, b.lo, bad);
  v = smax(v, f_mul_up(a.lo, b.hi, bad));
  v = smax(v, f_mul_up(a.hi, b.lo, bad));
  v = smax(v, f_mul_up(a.hi, b.hi, bad));
  return v;
}
__device__ __forceinline__ double f_corner_lo(const Iv& a, const Iv& b, bool& bad) {
  double v = f_mul_dn(a.lo, b.lo, bad);
  v = smin(v, f_mul_dn(a.lo, b.hi, bad));
  v = smin(v, f_mul_dn(a.hi, b.lo, bad));
  v = smin(v, f_mul_dn(a.hi, b.hi, bad));
  return v;
}
// iv_mul with both intervals known nonzero... or either zero (returns [0,0]).
__device__ __forceinline__ Iv f_iv_mul(const Iv& a, const Iv& b, bool& bad) {
  const bool z = iv_zero(a) | iv_zero(b);
  const Iv r{f_corner_lo(a, b, bad), f_corner_hi(a, b, bad)};
  return z ? Iv{0.0, 0.0} : r;
}
__device__ __forceinline__ bool start_bad(double x) { return !(fabs(x) < kStartHi); }

}  // namespace pc
