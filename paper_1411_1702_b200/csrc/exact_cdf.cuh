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
//
// Binade crossings (where rounding changes scale) are located with an
// approximate parallel prefix P_k (any summation tree, tile offsets from the
// predict kernel's block partials) and a rigorous bound |s_k - P_k| <= E_k
// (sum_bound below). Every
// element whose before/after values are not CERTAINLY in one binade becomes a
// "window": the resolver applies it with a real IEEE add, fl(s + g), in
// order. Windows are ~log2(N) per scan (one per binade crossing), so the
// serial part is tiny. Elements with g == 0 are the identity.
#pragma once
#include "variant.cuh"
#include <cstdint>

PFSMC_BEGIN

// Binade index with the subnormal range folded into e = -1022
// (ulp 2^-1074 on [0, 2^-1021)).
__device__ __forceinline__ int binade_of(double v) {
  if (!(v >= 0x1.0p-1021)) return -1022;
  return static_cast<int>((__double_as_longlong(v) >> 52) & 0x7ff) - 1023;
}

// x * 2^k, exact whenever the result is representable: a single multiply by
// a bit-built power of two on the normal range, ldexp() beyond it.
__device__ __forceinline__ double scale2(double x, int k) {
  if (k >= -1000 && k <= 1000) return x * __longlong_as_double(static_cast<long long>(k + 1023) << 52);
  return ldexp(x, k);
}

constexpr int kNoBinade = -100000;

// Monoid element for the segmented scan. flag = segment head (a window
// starts a new segment); e = the binade of the segment (kNoBinade while the
// segment holds only g == 0 elements).
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
  r.d0 = a.d0 + ((a.d0 & 1) ? b.d1 : b.d0);
  r.d1 = a.d1 + (((1 + a.d1) & 1) ? b.d1 : b.d0);
  r.e = b.e != kNoBinade ? b.e : a.e;
  r.flag = a.flag;
  return r;
}

__device__ __forceinline__ Piece shfl_up_piece(const Piece& p, int o) {
  Piece r;
  r.d0 = __shfl_up_sync(0xffffffffu, p.d0, o);
  r.d1 = __shfl_up_sync(0xffffffffu, p.d1, o);
  r.e = __shfl_up_sync(0xffffffffu, p.e, o);
  r.flag = __shfl_up_sync(0xffffffffu, p.flag, o);
  return r;
}

// Rigorous |s - P| bound. P = (tile prefix from the K1 block partials) +
// (in-tile tree prefix of the exact g). Error sources, u = 2^-53, cnt =
// nonzero (finite) terms so far:
//  * the sequential s and every tree/partial sum: <= cnt rounding nodes each
//    (nodes adding a zero are exact), each <= u of a value <= P(1+tiny);
//  * tile sums = sum_b S_b exp(M_b - lse): per-block product and sum
//    roundings (<= cnt), CUDA exp <= 2 ulp on S_b terms and the scale;
//  * argument roundings fl(lg - M_b), fl(M_b - lse), fl(lg - lse): absolute
//    <= u * 3 * g |ln g| <= u * 3/e per nonzero term (g |ln g| <= 1/e).
// => |s - P| <= u ((5 cnt + 16) P + 2 cnt); used with a 2x margin. cnt <= 1:
// a one-term sum is exact on every path (exp(0) = 1), so both are exact.
__device__ __forceinline__ double sum_bound(double p, long long cnt) {
  if (cnt <= 1) return 0.0;
  const double n = static_cast<double>(cnt);
  return ((12.0 * n + 64.0) * p + 4.0 * n) * 0x1.0p-53 + 0x1.0p-1060;
}

// Per-element kind: 0 = neutral (g == 0), 1 = run element, 2 = window.
// For run elements fills the monoid piece at binade e.
__device__ __forceinline__ int classify(double g, double p_prev, long long cnt_prev, double p_cur,
                                        long long cnt_cur, Piece& out) {
  out = piece_identity();
  if (g == 0.0) return 0;
  const int e_lo = binade_of(p_prev - sum_bound(p_prev, cnt_prev));
  const int e_hi = binade_of(p_cur + sum_bound(p_cur, cnt_cur));
  if (e_lo != e_hi) {
    out.flag = 1;
    return 2;
  }
  const double v = scale2(g, 52 - e_lo);  // exact scaling, v < 2^53
  const double q = floor(v);
  const double f = v - q;
  const long long qi = static_cast<long long>(q);
  if (f < 0.5) {
    out.d0 = out.d1 = qi;
  } else if (f > 0.5) {
    out.d0 = out.d1 = qi + 1;
  } else {  // exact tie: round half to even on m + q
    out.d0 = qi + (qi & 1);
    out.d1 = qi + ((1 + qi) & 1);
  }
  out.e = e_lo;
  return 1;
}

// Apply a segment aggregate to the exact running sum s (which the
// classification guarantees lies in binade a.e). In that binade s = m u with
// u = 2^(e-52), and the parity of m is the lowest significand bit of s, so
// the update is one exact IEEE add: s + delta u is representable (it stays in
// the binade, or lands exactly on 2^(e+1)). Returns false on an internal
// inconsistency (never expected; reported as INTERNAL).
__device__ __forceinline__ bool piece_apply(const Piece& a, double& s) {
  if (a.e == kNoBinade) return true;
  if (binade_of(s) != a.e) return false;
  const long long delta = (__double_as_longlong(s) & 1) ? a.d1 : a.d0;
  s = s + scale2(static_cast<double>(delta), a.e - 52);
  return true;
}

PFSMC_END  // namespace pfsmc_gpu::PFSMC_VNS
