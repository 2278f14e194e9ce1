// scanfold.cuh — the reference's serial directed-rounded chains, folded by a
// warp-wide integer prefix sum, bit-exact.
//
// Every row constant and every concretisation of the reference is a chain
//     acc = add_dir(acc, t_0);  acc = add_dir(acc, t_1);  ...
// of WidenedFloat64 adds (interval.hpp:59-68: round to nearest, then one ulp
// outward iff inexact) in a fixed order (backsub.hpp:365-389, 454-489,
// 536-563, 740-760). Run link by link, the chain costs two dependent FP64
// latencies per term (~39 cycles on B200) — the critical path of a
// single-image walk.
//
// Inside one binade the chain is an integer sum. Write acc = M * 2^E with
// 2^52 <= |M| < 2^53 (E = the ulp exponent of acc) and a term t = y * 2^E,
// y = T + f with T = floor(y), f in [0, 1). As long as every partial result
// stays strictly inside the same binade, the grid there has spacing 2^E, so
//     add_down(acc, t) = (M + T + delta_dn(f)) * 2^E,
//     add_up  (acc, t) = (M + T + delta_up(f)) * 2^E,
//     delta_dn = 0 (f = 0), -1 (0 < f < 1/2), 0 (1/2 < f < 1)
//     delta_up = 0 (f = 0), +1 (0 < f < 1/2), +2 (1/2 < f < 1)
// (RN rounds x = M + y to the nearest integer; the outward step adds one
// more unit iff x was not an integer). The increment depends on the term
// alone — except at a tie (f = 1/2, where RN's tie-to-even reads the parity
// of M + T) — so a warp computes 32 increments in parallel, prefix-sums them
// and checks that every partial result kept the binade (with a 2-unit margin,
// so the exact sum and its RN neighbour did too) and its sign. The first link
// that breaks an assumption (a tie, a huge or non-finite term, a binade
// change, a zero or subnormal accumulator) and every link before a usable
// frame exists runs as the exact scalar op (add_up / add_down of
// numeric.cuh), then the scan resumes from its result. So the fold is the
// reference's chain bit for bit, whatever the data; on the ResNets almost
// every link takes the scan.
#pragma once
#include "numeric.cuh"

namespace pc {

constexpr long long kScanLo = (1LL << 52) + 2;  // |M| range of a scanned partial result
constexpr long long kScanHi = (1LL << 53) - 3;

// acc = M * 2^E with the 2^-E scale as a double; false when acc is zero,
// subnormal, tiny (2^-E not a normal double) or huge (huge terms could
// overflow the scaled domain): those links run as scalar ops.
__device__ __forceinline__ bool scan_frame(double acc, int& ex, double& inv, long long& M) {
  const long long b = __double_as_longlong(acc);
  ex = (int)((b >> 52) & 0x7FF);  // biased exponent: E = ex - 1075
  if (ex < 200 || ex > 2000) return false;
  inv = __longlong_as_double((long long)(2098 - ex) << 52);  // 2^-E = 2^(1075 - ex)
  const long long mant = (b & ((1LL << 52) - 1)) | (1LL << 52);
  M = b < 0 ? -mant : mant;
  return true;
}

// m * 2^E for |m| in [2^52, 2^53): sign | biased exponent | fraction bits.
__device__ __forceinline__ double scan_compose(long long m, int ex) {
  const unsigned long long am = (unsigned long long)(m < 0 ? -m : m);
  const unsigned long long bits = ((unsigned long long)(m < 0) << 63) |
                                  ((unsigned long long)ex << 52) | (am - (1ULL << 52));
  return __longlong_as_double((long long)bits);
}

// Integer increment of one link (see the header); ok = false when the link
// must run as a scalar op. NaN = no term (increment 0).
__device__ __forceinline__ long long scan_delta(double t, double inv, bool up, bool& ok) {
  if (!(t == t) || t == 0.0) return 0;  // no term / adding +-0 leaves a nonzero acc as is
  const double y = t * inv;  // exact when |y| >= 1/4 (normal); only classified below that
  const double ay = fabs(y);
  if (ay < 0.25) return up ? 1 : -1;  // 0 < |y| < 1/4: f in (0, 1/4) or (3/4, 1)
  if (!(ay < 0x1p60)) {
    ok = false;
    return 0;
  }
  const double T = floor(y);
  const double f = y - T;  // a rounded f can only land on 1/2, which falls back
  if (f == 0.5) {
    ok = false;
    return 0;
  }
  long long d = __double2ll_rz(T);
  if (f != 0.0) d += up ? (f < 0.5 ? 1 : 2) : (f < 0.5 ? -1 : 0);
  return d;
}

// Fold n terms term(j) (j ascending) into acc. Called by all 32 lanes of a
// warp with the same acc; returns the same acc in every lane.
template <class TermFn>
__device__ __forceinline__ double scan_fold(double acc, int n, bool up, const TermFn& term) {
  const int lane = threadIdx.x & 31;
  int base = 0;
  while (base < n) {
    int ex;
    double inv;
    long long M;
    if (!scan_frame(acc, ex, inv, M)) {
      const double t = term(base);
      if (t == t) acc = up ? add_up(acc, t) : add_down(acc, t);
      ++base;
      continue;
    }
    const int cnt = min(32, n - base);
    bool ok = true;
    long long d = 0;
    if (lane < cnt) d = scan_delta(term(base + lane), inv, up, ok);
    long long s = d;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long v = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += v;
    }
    const long long m = M + s;
    const long long am = m < 0 ? -m : m;
    ok = ok && ((m < 0) == (M < 0)) && am >= kScanLo && am <= kScanHi;
    const unsigned bad = __ballot_sync(0xffffffffu, lane < cnt && !ok);
    const int k = bad ? __ffs(bad) - 1 : cnt;
    if (k > 0) acc = scan_compose(__shfl_sync(0xffffffffu, m, k - 1), ex);
    base += k;
    if (bad) {  // the link that left the scan's domain, as the scalar op
      const double t = term(base);
      if (t == t) acc = up ? add_up(acc, t) : add_down(acc, t);
      ++base;
    }
  }
  return acc;
}

// The same fold, 4 links per lane (128 per warp step): lane l takes links
// 4l .. 4l+3 of the group, prefix-sums them locally and the lane totals across
// the warp, so a step costs one warp scan for 128 links.
template <class TermFn>
__device__ __forceinline__ double scan_fold4(double acc, int n, bool up, const TermFn& term) {
  const int lane = threadIdx.x & 31;
  int base = 0;
  while (base < n) {
    int ex;
    double inv;
    long long M;
    if (!scan_frame(acc, ex, inv, M)) {
      const double t = term(base);
      if (t == t) acc = up ? add_up(acc, t) : add_down(acc, t);
      ++base;
      continue;
    }
    const int cnt = min(128, n - base);
    const int j0 = 4 * lane;
    long long part[4];
    int first = 4;  // first link of this lane that leaves the scan (4: none)
    long long run = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      bool ok = true;
      long long d = 0;
      if (j0 + k < cnt) d = scan_delta(term(base + j0 + k), inv, up, ok);
      run += d;
      part[k] = run;
      if (!ok && j0 + k < cnt && first == 4) first = k;
    }
    long long incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const long long excl = incl - run;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const long long m = M + excl + part[k];
      const long long am = m < 0 ? -m : m;
      if (k < first && j0 + k < cnt && !(((m < 0) == (M < 0)) && am >= kScanLo && am <= kScanHi)) first = k;
    }
    const unsigned bad = __ballot_sync(0xffffffffu, first < 4);
    int k = cnt;  // links committed by the scan
    if (bad) {
      const int bl = __ffs(bad) - 1;
      k = 4 * bl + __shfl_sync(0xffffffffu, first, bl);
    }
    if (k > 0) {
      const int src = (k - 1) >> 2, slot = (k - 1) & 3;
      const long long mine = M + excl + (slot == 0 ? part[0] : slot == 1 ? part[1] : slot == 2 ? part[2] : part[3]);
      acc = scan_compose(__shfl_sync(0xffffffffu, mine, src), ex);
    }
    base += k;
    if (bad) {  // the link that left the scan's domain, as the scalar op
      const double t = term(base);
      if (t == t) acc = up ? add_up(acc, t) : add_down(acc, t);
      ++base;
    }
  }
  return acc;
}

}  // namespace pc
