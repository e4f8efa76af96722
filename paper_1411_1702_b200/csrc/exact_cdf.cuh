// Exact parallel reproduction of the reference's SEQUENTIAL resampling CDF
//   acc = 0; for i: acc += g[i]; cdf[i] = acc          (filter.cpp:162-167)
// so that multinomial ancestors are bit-identical to the reference for any
// fitness vector g, not just "equal up to near-ties".
//
// Why it can be parallel. While the running sum s stays inside one binade
// [2^e, 2^(e+1)) (ulp u = 2^(e-52)), s = m*u with an integer m < 2^53 and
//   fl(s + g) = u * (m + rn(g/u)),
// where the rounding of g/u = q + f is q (f < 1/2), q + 1 (f > 1/2) or, on an
// exact tie f = 1/2, the even neighbour, i.e. depends only on the parity of m.
// An element is therefore the integer map  b = m mod 2  ->  delta(b), and a
// run of elements composes exactly in the monoid
//   (A then B)(b) = A(b) + B((b + A(b)) mod 2),
// represented by the pair (delta(0), delta(1)) -- a parallel scan.
// Binade crossings (where rounding changes scale) are located with a
// double-double approximate prefix P_k and a rigorous bound E_k >= |s_k - P_k|
// (<= cnt_k ulp/2, cnt_k = inexact additions so far). Every element whose
// before/after values are not certainly in one binade becomes a "window":
// the resolver applies it with a real IEEE add, fl(s + g), in order. Windows
// are ~log2(N) per scan (one per binade crossing), so the serial part is tiny.
// Elements with g == 0 are the identity and never need a window.
#pragma once
#include <cstdint>

namespace pfsmc_gpu {

// ---------------- double-double helpers (error-free transforms) ----------
struct DD {
  double hi, lo;
};
__device__ __forceinline__ DD two_sum(double a, double b) {
  const double s = __dadd_rn(a, b);
  const double bb = __dsub_rn(s, a);
  const double err = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
  return {s, err};
}
__device__ __forceinline__ DD dd_add(DD a, double b) {
  DD s = two_sum(a.hi, b);
  s.lo = __dadd_rn(s.lo, a.lo);
  return two_sum(s.hi, s.lo);
}
__device__ __forceinline__ DD dd_add(DD a, DD b) {
  DD s = two_sum(a.hi, b.hi);
  s.lo = __dadd_rn(s.lo, __dadd_rn(a.lo, b.lo));
  return two_sum(s.hi, s.lo);
}

// Binade index with the subnormal range folded into e = -1022
// (ulp 2^-1074 on [0, 2^-1021)).
__device__ __forceinline__ int binade_of(double v) {
  if (!(v >= 0x1.0p-1021)) return -1022;
  return ilogb(v);
}

constexpr int kNoBinade = -100000;

// Monoid element for the segmented scan. flag = segment head (a window or
// the element right after one starts a new segment); e = the binade of the
// segment (kNoBinade while the segment holds only g == 0 elements).
struct Piece {
  long long d0, d1;
  int e;
  int flag;
};

__device__ __forceinline__ Piece piece_identity() { return {0, 0, kNoBinade, 0}; }

// a then b, with b's head flag cutting a off.
__device__ __forceinline__ Piece piece_combine(const Piece& a, const Piece& b) {
  if (b.flag) return b;
  Piece r;
  r.d0 = a.d0 + (((a.d0) & 1) ? b.d1 : b.d0);
  r.d1 = a.d1 + (((1 + a.d1) & 1) ? b.d1 : b.d0);
  r.e = b.e != kNoBinade ? b.e : a.e;
  r.flag = a.flag;
  return r;
}

// Rigorous |s - P| bound. cnt = nonzero g's so far; the first nonzero add
// (onto 0) is exact, and a one-term double-double sum is exact, so cnt <= 1
// gives 0. Otherwise (cnt - 1) roundings of <= 2^-53 s each, doubled plus a
// margin that also covers rounding P.hi +- E itself.
__device__ __forceinline__ double sum_bound(double p_hi, long long cnt) {
  if (cnt <= 1) return 0.0;
  return (static_cast<double>(cnt - 1) + 4.0) * 0x1.0p-51 * p_hi + 0x1.0p-1060;
}

// Per-element kind: 0 = neutral (g == 0), 1 = run element, 2 = window.
// For run elements fills the monoid piece at binade e.
__device__ __forceinline__ int classify(double g, DD p_prev, long long cnt_prev, DD p_cur,
                                        long long cnt_cur, Piece& out) {
  out = piece_identity();
  if (g == 0.0) return 0;
  const double lo = p_prev.hi - sum_bound(p_prev.hi, cnt_prev);
  const double hi = p_cur.hi + sum_bound(p_cur.hi, cnt_cur);
  const int e_lo = binade_of(lo);
  const int e_hi = binade_of(hi);
  if (e_lo != e_hi) {
    out.flag = 1;
    return 2;
  }
  const double v = ldexp(g, 52 - e_lo);  // exact scaling, v < 2^53
  const double q = floor(v);
  const double f = v - q;
  const long long qi = static_cast<long long>(q);
  if (f < 0.5) {
    out.d0 = out.d1 = qi;
  } else if (f > 0.5) {
    out.d0 = out.d1 = qi + 1;
  } else {  // exact tie: round half to even on m + q
    out.d0 = qi + ((0 + qi) & 1);
    out.d1 = qi + ((1 + qi) & 1);
  }
  out.e = e_lo;
  return 1;
}

// Apply a segment aggregate to the exact running sum s (which the
// classification guarantees lies in binade a.e). Returns false on an
// internal inconsistency (never expected; reported as INTERNAL).
__device__ __forceinline__ bool piece_apply(const Piece& a, double& s) {
  if (a.e == kNoBinade) return true;
  if (binade_of(s) != a.e) return false;
  const double ms = ldexp(s, 52 - a.e);
  const long long m = static_cast<long long>(ms);
  if (static_cast<double>(m) != ms) return false;
  const long long m2 = m + ((m & 1) ? a.d1 : a.d0);
  s = ldexp(static_cast<double>(m2), a.e - 52);
  return true;
}

}  // namespace pfsmc_gpu
