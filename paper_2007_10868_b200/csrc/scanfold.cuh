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

#define PC_SCAN_NAN __longlong_as_double(0x7ff8000000000000ULL)

// Diagnostics (pc_scan_stats): [0] scan steps, [1] links committed by scans,
// [2] scalar links after a failed step, [3] frame-less scalar links.
// One copy per translation unit (no relocatable device code); each .cu that
// folds exposes its own accessor (scan_stats_device*).
static __device__ unsigned long long g_scan_stats[8];
static __device__ int g_scan_stats_on;
__device__ __forceinline__ void scan_stat(int k, unsigned long long v) {
  if (g_scan_stats_on) atomicAdd(&g_scan_stats[k], v);
}

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
    scan_stat(5, 1);
    return 0;
  }
  const double T = floor(y);
  const double f = y - T;  // a rounded f can only land on 1/2, which falls back
  if (f == 0.5) {
    ok = false;
    scan_stat(4, 1);
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
      // no binade frame (zero / subnormal / extreme acc): skip to the next
      // term (NaN = none) in one step and apply it as the scalar op
      const int cnt = min(32, n - base);
      const double tl = lane < cnt ? term(base + lane) : PC_SCAN_NAN;
      const unsigned has = __ballot_sync(0xffffffffu, tl == tl);
      if (!has) {
        base += cnt;
        continue;
      }
      const int k = __ffs(has) - 1;
      const double t = __shfl_sync(0xffffffffu, tl, k);
      acc = up ? add_up(acc, t) : add_down(acc, t);
      base += k + 1;
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

// Tie-aware increments: a link whose term sits exactly half way between two
// grid points (f = 1/2) rounds to the even neighbour, so its increment
// depends on the parity p of the incoming partial result: the link maps p to
// (d0, d1)[p]. A run of links composes as such a pair — A then B maps p to
// A(p) + B(p ^ (A(p) & 1)) — and the composition is associative, so the warp
// prefix-sums pairs instead of integers and ties stay inside the scan.
// FAST: plain directed rounding (fast numeric mode): RD(M + T + f) = M + T,
// RU = M + T + [f > 0]; no ties.
template <bool FAST = false>
__device__ __forceinline__ void scan_delta2(double t, double inv, bool up, bool& ok, long long& d0,
                                            long long& d1) {
  d0 = d1 = 0;
  if (!(t == t) || t == 0.0) return;
  const double y = t * inv;
  const double ay = fabs(y);
  if (ay < 0.25) {
    if (FAST) d0 = d1 = up ? (t > 0.0 ? 1 : 0) : (t < 0.0 ? -1 : 0);
    else d0 = d1 = up ? 1 : -1;
    return;
  }
  if (!(ay < 0x1p60)) {
    ok = false;
    scan_stat(5, 1);
    return;
  }
  const double T = floor(y);
  const double f = y - T;
  const long long Ti = __double2ll_rz(T);
  if (FAST) {
    d0 = d1 = Ti + ((up && f != 0.0) ? 1 : 0);
    return;
  }
  if (f == 0.5) {  // RN(m + T + 1/2) = the even one of m + T, m + T + 1
    const long long q = Ti & 1, base = Ti + (up ? 1 : -1);
    d0 = base + q;
    d1 = base + (1 - q);
    scan_stat(4, 1);
    return;
  }
  long long d = Ti;
  if (f != 0.0) d += up ? (f < 0.5 ? 1 : 2) : (f < 0.5 ? -1 : 0);
  d0 = d1 = d;
}

// One link as the scalar op of the mode.
template <bool FAST>
__device__ __forceinline__ double link_op(double acc, double t, bool up) {
  if (FAST) return up ? __dadd_ru(acc, t) : __dadd_rd(acc, t);
  return up ? add_up(acc, t) : add_down(acc, t);
}

// a then b, as parity-indexed pairs
__device__ __forceinline__ void scan_compose2(long long a0, long long a1, long long b0, long long b1,
                                              long long& c0, long long& c1) {
  const long long x0 = a0 + ((a0 & 1) ? b1 : b0);
  const long long x1 = a1 + ((a1 & 1) ? b0 : b1);
  c0 = x0;
  c1 = x1;
}

// The same fold, 4 links per lane (128 per warp step): lane l takes links
// 4l .. 4l+3 of the group, composes them locally and scans the lane pairs
// across the warp, so a step costs one warp scan for 128 links.
template <class TermFn, bool FAST = false>
__device__ __forceinline__ double scan_fold4(double acc, int n, bool up, const TermFn& term) {
  const int lane = threadIdx.x & 31;
  int base = 0;
  while (base < n) {
    int ex;
    double inv;
    long long M;
    if (!scan_frame(acc, ex, inv, M)) {  // skip to the next term, apply it as the scalar op
      const int cnt = min(32, n - base);
      const double tl = lane < cnt ? term(base + lane) : PC_SCAN_NAN;
      const unsigned has = __ballot_sync(0xffffffffu, tl == tl);
      if (!has) {
        base += cnt;
        continue;
      }
      const int k = __ffs(has) - 1;
      const double t = __shfl_sync(0xffffffffu, tl, k);
      acc = link_op<FAST>(acc, t, up);
      base += k + 1;
      if (lane == 0) scan_stat(3, 1);
      continue;
    }
    const int cnt = min(128, n - base);
    const int j0 = 4 * lane;
    // A run of links as (v, e): increment v for an incoming partial result of
    // even parity, v + e for odd (the parity pair (v, v + e), scan_compose2);
    // e is 0 except after ties and stays small. a then b:
    //   v = a.v + b.v + [a.v odd] * b.e,   e = a.e odd ? a.e : a.e + (a.v odd ? -b.e : b.e)
    long long pv[4];  // lane-local inclusive runs
    int pe[4];
    int first = 4;    // first link of this lane that leaves the scan (4: none)
    long long rv = 0;
    int re = 0;
    bool small = true;  // every increment below 2^23: the warp scan runs in 32 bits
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      bool ok = true;
      long long d0 = 0, d1 = 0;
      if (j0 + k < cnt) scan_delta2<FAST>(term(base + j0 + k), inv, up, ok, d0, d1);
      small &= (d0 < (1LL << 23)) & (d0 > -(1LL << 23));
      const int de = (int)(d1 - d0);
      const bool odd = rv & 1;
      rv += d0 + (odd ? de : 0);
      re = (re & 1) ? re : re + (odd ? -de : de);
      pv[k] = rv;
      pe[k] = re;
      if (!ok && j0 + k < cnt && first == 4) first = k;
    }
    long long xv;  // increments before this lane (even incoming parity), and their e
    int xe;
    if (__all_sync(0xffffffffu, small)) {
      int iv = (int)rv, ie = re;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int uv = __shfl_up_sync(0xffffffffu, iv, o), ue = __shfl_up_sync(0xffffffffu, ie, o);
        if (lane >= o) {
          const bool odd = uv & 1;
          const int nv = uv + iv + (odd ? ie : 0);
          ie = (ue & 1) ? ue : ue + (odd ? -ie : ie);
          iv = nv;
        }
      }
      int ev = __shfl_up_sync(0xffffffffu, iv, 1), ee = __shfl_up_sync(0xffffffffu, ie, 1);
      if (lane == 0) ev = ee = 0;
      xv = ev;
      xe = ee;
    } else {
      long long iv = rv;
      int ie = re;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long uv = __shfl_up_sync(0xffffffffu, iv, o);
        const int ue = __shfl_up_sync(0xffffffffu, ie, o);
        if (lane >= o) {
          const bool odd = uv & 1;
          const long long nv = uv + iv + (odd ? ie : 0);
          ie = (ue & 1) ? ue : ue + (odd ? -ie : ie);
          iv = nv;
        }
      }
      long long ev = __shfl_up_sync(0xffffffffu, iv, 1);
      int ee = __shfl_up_sync(0xffffffffu, ie, 1);
      if (lane == 0) ev = ee = 0;
      xv = ev;
      xe = ee;
    }
    const long long P = xv + ((M & 1) ? xe : 0);  // increments before this lane, from M's parity
    const bool pl = (M + P) & 1;                   // parity entering this lane
    long long mk[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      mk[k] = M + P + pv[k] + (pl ? pe[k] : 0);
      const long long am = mk[k] < 0 ? -mk[k] : mk[k];
      if (k < first && j0 + k < cnt && !(((mk[k] < 0) == (M < 0)) && am >= kScanLo && am <= kScanHi)) first = k;
    }
    const unsigned bad = __ballot_sync(0xffffffffu, first < 4);
    int k = cnt;  // links committed by the scan
    if (bad) {
      const int bl = __ffs(bad) - 1;
      k = 4 * bl + __shfl_sync(0xffffffffu, first, bl);
    }
    if (lane == 0) {
      scan_stat(0, 1);
      scan_stat(1, k);
      if (bad) scan_stat(2, 1);
    }
    if (k > 0) {
      const int src = (k - 1) >> 2, slot = (k - 1) & 3;
      const long long mine = slot == 0 ? mk[0] : slot == 1 ? mk[1] : slot == 2 ? mk[2] : mk[3];
      acc = scan_compose(__shfl_sync(0xffffffffu, mine, src), ex);
    }
    base += k;
    if (bad) {  // the link that left the scan's domain, as the scalar op
      const double t = term(base);
      if (t == t) acc = link_op<FAST>(acc, t, up);
      ++base;
    }
  }
  return acc;
}

template <bool FAST, class TermFn>
__device__ __forceinline__ double scan_fold4m(double acc, int n, bool up, const TermFn& term) {
  return scan_fold4<TermFn, FAST>(acc, n, up, term);
}

// scan_fold4 over a contiguous term array in global memory, with the next
// group's terms loaded while the current group is scanned (the loads of a
// group depend only on where it starts, which a failed link rarely moves).
__device__ __forceinline__ double scan_fold4_pf(double acc, int n, bool up, const double* T) {
  const int lane = threadIdx.x & 31;
  auto load = [&](int b, double* v) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int j = b + 4 * lane + k;
      v[k] = j < n ? __ldg(T + j) : PC_SCAN_NAN;
    }
  };
  double cur[4], nxt[4];
  int base = 0;
  load(0, cur);
  while (base < n) {
    int ex;
    double inv;
    long long M;
    if (!scan_frame(acc, ex, inv, M)) {  // next term (NaN = none) as the scalar op
      const int lane_first = (cur[0] == cur[0]) ? 0 : (cur[1] == cur[1]) ? 1 : (cur[2] == cur[2]) ? 2 : (cur[3] == cur[3]) ? 3 : 4;
      const unsigned has = __ballot_sync(0xffffffffu, lane_first < 4);
      if (!has) {
        base += 128;
        load(base, cur);
        continue;
      }
      const int bl = __ffs(has) - 1;
      const int k = 4 * bl + __shfl_sync(0xffffffffu, lane_first, bl);
      const double t = __shfl_sync(0xffffffffu, (k & 3) == 0 ? cur[0] : (k & 3) == 1 ? cur[1] : (k & 3) == 2 ? cur[2] : cur[3], bl);
      acc = up ? add_up(acc, t) : add_down(acc, t);
      base += k + 1;
      if (lane == 0) scan_stat(3, 1);
      load(base, cur);
      continue;
    }
    load(base + 128, nxt);
    const int cnt = min(128, n - base);
    const int j0 = 4 * lane;
    long long p0[4], p1[4];
    int first = 4;
    long long r0 = 0, r1 = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      bool ok = true;
      long long d0 = 0, d1 = 0;
      if (j0 + k < cnt) scan_delta2(cur[k], inv, up, ok, d0, d1);
      scan_compose2(r0, r1, d0, d1, r0, r1);
      p0[k] = r0;
      p1[k] = r1;
      if (!ok && j0 + k < cnt && first == 4) first = k;
    }
    long long i0 = r0, i1 = r1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long u0 = __shfl_up_sync(0xffffffffu, i0, o), u1 = __shfl_up_sync(0xffffffffu, i1, o);
      if (lane >= o) scan_compose2(u0, u1, i0, i1, i0, i1);
    }
    long long e0 = __shfl_up_sync(0xffffffffu, i0, 1), e1 = __shfl_up_sync(0xffffffffu, i1, 1);
    if (lane == 0) e0 = e1 = 0;
    const long long P = (M & 1) ? e1 : e0;
    const int pl = (int)((M + P) & 1);
    long long mk[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      mk[k] = M + P + (pl ? p1[k] : p0[k]);
      const long long am = mk[k] < 0 ? -mk[k] : mk[k];
      if (k < first && j0 + k < cnt && !(((mk[k] < 0) == (M < 0)) && am >= kScanLo && am <= kScanHi)) first = k;
    }
    const unsigned bad = __ballot_sync(0xffffffffu, first < 4);
    int k = cnt;
    if (bad) {
      const int bl = __ffs(bad) - 1;
      k = 4 * bl + __shfl_sync(0xffffffffu, first, bl);
      if (g_scan_stats_on && lane == bl) {  // why the link left the scan: 6 grew past the binade, 7 shrank / flipped
        const int f = k & 3;
        const long long mf = f == 0 ? mk[0] : f == 1 ? mk[1] : f == 2 ? mk[2] : mk[3];
        const long long am = mf < 0 ? -mf : mf;
        if (am > kScanHi && ((mf < 0) == (M < 0))) scan_stat(6, 1);
        else if (am < kScanLo || ((mf < 0) != (M < 0))) scan_stat(7, 1);
      }
    }
    if (lane == 0) {
      scan_stat(0, 1);
      scan_stat(1, k);
      if (bad) scan_stat(2, 1);
    }
    if (k > 0) {
      const int src = (k - 1) >> 2, slot = (k - 1) & 3;
      const long long mine = slot == 0 ? mk[0] : slot == 1 ? mk[1] : slot == 2 ? mk[2] : mk[3];
      acc = scan_compose(__shfl_sync(0xffffffffu, mine, src), ex);
    }
    if (!bad) {
      base += cnt;
#pragma unroll
      for (int u = 0; u < 4; ++u) cur[u] = nxt[u];
    } else {
      base += k;
      const double t = __ldg(T + base);  // the link that left the scan's domain, as the scalar op
      if (t == t) acc = up ? add_up(acc, t) : add_down(acc, t);
      ++base;
      load(base, cur);
    }
  }
  return acc;
}

// The same fold by a whole CTA of NT threads, 4 links per thread (4*NT per
// step): lane-local pairs, a warp scan of the pairs, warp 0 composing the
// warp totals, and a block-wide minimum of the first link that leaves the
// scan's domain. All NT threads call it with the same acc; returns it in
// every thread. sm: at least 2*NT/32 + 4 long longs of shared memory.
template <int NT, class TermFn>
__device__ __forceinline__ double block_scan_fold(double acc, int n, bool up, const TermFn& term,
                                                  long long* sm) {
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  long long* s_w0 = sm;                              // [NW] warp totals -> exclusive prefixes
  long long* s_w1 = sm + NW;
  int* s_first = reinterpret_cast<int*>(sm + 2 * NW);  // first failing link of the step
  long long* s_m = sm + 2 * NW + 1;                  // committed partial result
  double* s_t = reinterpret_cast<double*>(sm + 2 * NW + 2);
  int base = 0;
  while (base < n) {
    int ex;
    double inv;
    long long M;
    if (!scan_frame(acc, ex, inv, M)) {  // skip to the next term, apply it as the scalar op
      const int cnt = min(NT, n - base);
      const double tl = tid < cnt ? term(base + tid) : PC_SCAN_NAN;
      if (tid == 0) *s_first = NT;
      __syncthreads();
      if (tl == tl) atomicMin(s_first, tid);
      __syncthreads();
      const int k = *s_first;
      if (k == tid) *s_t = tl;
      __syncthreads();
      if (k < NT) {
        const double t = *s_t;
        acc = up ? add_up(acc, t) : add_down(acc, t);
        base += k + 1;
        if (tid == 0) scan_stat(3, 1);
      } else {
        base += cnt;
      }
      __syncthreads();
      continue;
    }
    const int cnt = min(4 * NT, n - base);
    const int j0 = 4 * tid;
    long long p0[4], p1[4];
    int first = 4 * NT;
    long long r0 = 0, r1 = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      bool ok = true;
      long long d0 = 0, d1 = 0;
      if (j0 + k < cnt) scan_delta2(term(base + j0 + k), inv, up, ok, d0, d1);
      scan_compose2(r0, r1, d0, d1, r0, r1);
      p0[k] = r0;
      p1[k] = r1;
      if (!ok && j0 + k < cnt && first == 4 * NT) first = j0 + k;
    }
    long long i0 = r0, i1 = r1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long u0 = __shfl_up_sync(0xffffffffu, i0, o), u1 = __shfl_up_sync(0xffffffffu, i1, o);
      if (lane >= o) scan_compose2(u0, u1, i0, i1, i0, i1);
    }
    long long e0 = __shfl_up_sync(0xffffffffu, i0, 1), e1 = __shfl_up_sync(0xffffffffu, i1, 1);
    if (lane == 0) e0 = e1 = 0;
    if (tid == 0) *s_first = 4 * NT;
    if (lane == 31) {
      s_w0[warp] = i0;
      s_w1[warp] = i1;
    }
    __syncthreads();
    if (tid == 0) {  // exclusive prefixes of the warp totals (NW compositions)
      long long a0 = 0, a1 = 0;
      for (int w = 0; w < NW; ++w) {
        const long long b0 = s_w0[w], b1 = s_w1[w];
        s_w0[w] = a0;
        s_w1[w] = a1;
        scan_compose2(a0, a1, b0, b1, a0, a1);
      }
    }
    __syncthreads();
    long long x0, x1;  // increments before this thread: warp prefix, then lane prefix
    scan_compose2(s_w0[warp], s_w1[warp], e0, e1, x0, x1);
    const long long P = (M & 1) ? x1 : x0;
    const int pl = (int)((M + P) & 1);
    long long mk[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      mk[k] = M + P + (pl ? p1[k] : p0[k]);
      const long long am = mk[k] < 0 ? -mk[k] : mk[k];
      if (j0 + k < first && j0 + k < cnt && !(((mk[k] < 0) == (M < 0)) && am >= kScanLo && am <= kScanHi))
        first = j0 + k;
    }
    if (first < 4 * NT) atomicMin(s_first, first);
    __syncthreads();
    const int k = min(*s_first, cnt);  // links committed by the scan
    if (tid == 0) {
      scan_stat(0, 1);
      scan_stat(1, k);
      if (k < cnt) scan_stat(2, 1);
    }
    if (k > 0 && (k - 1) >> 2 == tid) {
      const int slot = (k - 1) & 3;
      *s_m = slot == 0 ? mk[0] : slot == 1 ? mk[1] : slot == 2 ? mk[2] : mk[3];
    }
    __syncthreads();
    if (k > 0) acc = scan_compose(*s_m, ex);
    base += k;
    if (k < cnt) {  // the link that left the scan's domain, as the scalar op (every thread alike)
      const double t = term(base);
      if (t == t) acc = up ? add_up(acc, t) : add_down(acc, t);
      ++base;
    }
    __syncthreads();  // shared scratch reused by the next step
  }
  return acc;
}

// CTA-wide fold with local retry: a window of 4*NT links is loaded into
// registers once; the block scans it, and after a link that leaves the scan's
// domain (applied as the scalar op) it rescans only the rest of the window in
// the new frame, without reloading or recomputing terms. For long chains of
// few rows, where one warp's step latency would be the critical path.
// sm: at least 2*NT/32 + 8 long longs of shared memory.
template <int NT, class TermFn, bool FAST = false>
__device__ __forceinline__ double block_scan_fold_rt(double acc, int n, bool up, const TermFn& term,
                                                     long long* sm) {
  constexpr int NW = NT / 32, WIN = 4 * NT;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  long long* s_w0 = sm;
  long long* s_w1 = sm + NW;
  int* s_first = reinterpret_cast<int*>(sm + 2 * NW);
  long long* s_m = sm + 2 * NW + 1;
  double* s_t = reinterpret_cast<double*>(sm + 2 * NW + 2);
  for (int wb = 0; wb < n; wb += WIN) {
    const int cnt = min(WIN, n - wb);
    const int j0 = 4 * tid;
    double tv[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) tv[k] = j0 + k < cnt ? term(wb + j0 + k) : PC_SCAN_NAN;
    int lo = 0;  // first link of the window not yet folded
    while (lo < cnt) {
      int ex;
      double inv;
      long long M;
      if (!scan_frame(acc, ex, inv, M)) {  // next term as the scalar op
        int mine = WIN;
#pragma unroll
        for (int k = 3; k >= 0; --k)
          if (j0 + k >= lo && j0 + k < cnt && tv[k] == tv[k]) mine = j0 + k;
        if (tid == 0) *s_first = WIN;
        __syncthreads();
        if (mine < WIN) atomicMin(s_first, mine);
        __syncthreads();
        const int f = *s_first;
        if (f < WIN && f >> 2 == tid) *s_t = (f & 3) == 0 ? tv[0] : (f & 3) == 1 ? tv[1] : (f & 3) == 2 ? tv[2] : tv[3];
        __syncthreads();
        if (f < WIN) {
          const double t = *s_t;
          acc = link_op<FAST>(acc, t, up);
          lo = f + 1;
          if (tid == 0) scan_stat(3, 1);
        } else {
          lo = cnt;
        }
        __syncthreads();
        continue;
      }
      long long p0[4], p1[4];
      int first = WIN;
      long long r0 = 0, r1 = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        bool ok = true;
        long long d0 = 0, d1 = 0;
        const int j = j0 + k;
        if (j >= lo && j < cnt) scan_delta2<FAST>(tv[k], inv, up, ok, d0, d1);
        scan_compose2(r0, r1, d0, d1, r0, r1);
        p0[k] = r0;
        p1[k] = r1;
        if (!ok && j >= lo && j < cnt && first == WIN) first = j;
      }
      long long i0 = r0, i1 = r1;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long u0 = __shfl_up_sync(0xffffffffu, i0, o), u1 = __shfl_up_sync(0xffffffffu, i1, o);
        if (lane >= o) scan_compose2(u0, u1, i0, i1, i0, i1);
      }
      long long e0 = __shfl_up_sync(0xffffffffu, i0, 1), e1 = __shfl_up_sync(0xffffffffu, i1, 1);
      if (lane == 0) e0 = e1 = 0;
      if (tid == 0) *s_first = WIN;
      if (lane == 31) {
        s_w0[warp] = i0;
        s_w1[warp] = i1;
      }
      __syncthreads();
      if (warp == 0) {  // exclusive prefixes of the warp totals, by one warp
        long long a0 = lane < NW ? s_w0[lane] : 0, a1 = lane < NW ? s_w1[lane] : 0;
        long long q0 = a0, q1 = a1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const long long u0 = __shfl_up_sync(0xffffffffu, q0, o), u1 = __shfl_up_sync(0xffffffffu, q1, o);
          if (lane >= o) scan_compose2(u0, u1, q0, q1, q0, q1);
        }
        long long x0 = __shfl_up_sync(0xffffffffu, q0, 1), x1 = __shfl_up_sync(0xffffffffu, q1, 1);
        if (lane == 0) x0 = x1 = 0;
        if (lane < NW) {
          s_w0[lane] = x0;
          s_w1[lane] = x1;
        }
      }
      __syncthreads();
      long long x0, x1;
      scan_compose2(s_w0[warp], s_w1[warp], e0, e1, x0, x1);
      const long long P = (M & 1) ? x1 : x0;
      const int pl = (int)((M + P) & 1);
      long long mk[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        mk[k] = M + P + (pl ? p1[k] : p0[k]);
        const long long am = mk[k] < 0 ? -mk[k] : mk[k];
        const int j = j0 + k;
        if (j < first && j >= lo && j < cnt && !(((mk[k] < 0) == (M < 0)) && am >= kScanLo && am <= kScanHi))
          first = j;
      }
      if (first < WIN) atomicMin(s_first, first);
      __syncthreads();
      const int f = min(*s_first, cnt);  // links lo .. f-1 committed by the scan
      if (tid == 0) {
        scan_stat(0, 1);
        scan_stat(1, f - lo);
        if (f < cnt) scan_stat(2, 1);
      }
      if (f > lo && (f - 1) >> 2 == tid) {
        const int slot = (f - 1) & 3;
        *s_m = slot == 0 ? mk[0] : slot == 1 ? mk[1] : slot == 2 ? mk[2] : mk[3];
      }
      if (f < cnt && f >> 2 == tid) *s_t = (f & 3) == 0 ? tv[0] : (f & 3) == 1 ? tv[1] : (f & 3) == 2 ? tv[2] : tv[3];
      __syncthreads();
      if (f > lo) acc = scan_compose(*s_m, ex);
      if (f < cnt) {  // the link that left the scan's domain, as the scalar op
        const double t = *s_t;
        if (t == t) acc = link_op<FAST>(acc, t, up);
        lo = f + 1;
      } else {
        lo = cnt;
      }
      __syncthreads();
    }
  }
  return acc;
}

template <int NT, bool FAST, class TermFn>
__device__ __forceinline__ double block_scan_fold_rtm(double acc, int n, bool up, const TermFn& term,
                                                      long long* sm) {
  return block_scan_fold_rt<NT, TermFn, FAST>(acc, n, up, term, sm);
}

}  // namespace pc
