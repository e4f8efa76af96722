// Psi: fixed-step LMM interval propagation for ONE particle, entirely in
// registers (state history, f history, Newton iterate and the d x d LU).
//
// Restates /root/reference/proj/src/lmm.cpp:
//   coefficient tables          lmm.cpp:18-60   (same decimal-rational literals)
//   explicit / implicit terms   lmm.cpp:108-144 (alpha terms first, then h*beta_i f)
//   extrapolation predictor     lmm.cpp:146-165
//   DenseLu factor / solve      linalg.cpp:201-258 (first strict max pivot,
//                                inv = 1/pivot, zero-multiplier skip)
//   newton_solve                lmm.cpp:219-266 (J rebuilt each iteration;
//                                ||dx|| <= tol (1 + ||x||) after the update)
//   LTE factors / finish_step   lmm.cpp:307-342, 438-452
//   ramped interval loop        lmm.cpp:468-503 (order p = min(k, order),
//                                fresh history every interval)
// The order ramp makes steps k = 1, 2, 3 special (avail = min(k, 4) history
// entries); for small d each is a separate compile-time instantiation, so
// every history index is static and nothing touches local memory; for large d
// (the 8-species chain) one runtime-order body keeps the code in the I-cache.
#pragma once
#include "variant.cuh"
#include "models.cuh"

PFSMC_BEGIN

enum Family : int { kAB = 0, kAM = 1, kBDF = 2 };
enum ParticleStatus : int { kOk = 0, kInvalidRhs = 1, kNewtonDivergence = 2, kSingular = 3, kStiffness = 4 };
// Step attempts per interval of the adaptive BDF(1,2) before it reports
// stiffness. The reference's loop (lmm.cpp:918-1016) has no such bound and
// does not terminate in some cases (e.g. its own advdiff generator at n = 4,
// 5); on the GPU an unbounded loop would hang the device.
constexpr long long kAdaptiveMaxAttempts = 1LL << 24;

// ---- coefficient tables (lmm.cpp:18-60) ----------------------------------
__host__ __device__ constexpr double ab_beta(int order, int i) {
  return order == 1   ? (i == 1 ? 1.0 : 0.0)
         : order == 2 ? (i == 1 ? 3.0 / 2.0 : i == 2 ? -1.0 / 2.0 : 0.0)
         : order == 3 ? (i == 1 ? 23.0 / 12.0 : i == 2 ? -16.0 / 12.0 : i == 3 ? 5.0 / 12.0 : 0.0)
                      : (i == 1 ? 55.0 / 24.0 : i == 2 ? -59.0 / 24.0 : i == 3 ? 37.0 / 24.0
                                                : i == 4 ? -9.0 / 24.0 : 0.0);
}
__host__ __device__ constexpr double ab_C(int order) {
  return order == 1 ? 1.0 / 2.0 : order == 2 ? 5.0 / 12.0 : order == 3 ? 3.0 / 8.0 : 251.0 / 720.0;
}
__host__ __device__ constexpr double am_beta(int order, int i) {
  return order == 1   ? (i == 0 ? 1.0 : 0.0)
         : order == 2 ? (i == 0 ? 1.0 / 2.0 : i == 1 ? 1.0 / 2.0 : 0.0)
                      : (i == 0 ? 5.0 / 12.0 : i == 1 ? 8.0 / 12.0 : i == 2 ? -1.0 / 12.0 : 0.0);
}
__host__ __device__ constexpr double am_C(int order) {
  return order == 1 ? -1.0 / 2.0 : order == 2 ? -1.0 / 12.0 : -1.0 / 24.0;
}
__host__ __device__ constexpr double bdf_alpha(int order, int i) {
  return order == 1   ? (i == 0 ? 1.0 : 0.0)
         : order == 2 ? (i == 0 ? 4.0 / 3.0 : i == 1 ? -1.0 / 3.0 : 0.0)
                      : (i == 0 ? 18.0 / 11.0 : i == 1 ? -9.0 / 11.0 : i == 2 ? 2.0 / 11.0 : 0.0);
}
__host__ __device__ constexpr double bdf_beta0(int order) {
  return order == 1 ? 1.0 : order == 2 ? 2.0 / 3.0 : 6.0 / 11.0;
}
__host__ __device__ constexpr double bdf_C(int order) {
  return order == 1 ? -1.0 / 2.0 : order == 2 ? -2.0 / 9.0 : -3.0 / 22.0;
}
__host__ __device__ constexpr int cmin(int a, int b) { return a < b ? a : b; }

// std::max / std::min / std::clamp as the reference uses them.
__device__ __forceinline__ double ref_max(double a, double b) { return (a < b) ? b : a; }
__device__ __forceinline__ double ref_min(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double ref_clamp(double v, double lo, double hi) {
  return (v < lo) ? lo : (hi < v) ? hi : v;
}

// max(0, |v_0|, ..., |v_{N-1}|) with NaN entries skipped, as a fmax tree.
template <int N>
__device__ __forceinline__ double max_abs_tree(const double (&v)[N]) {
  double t[N];
#pragma unroll
  for (int j = 0; j < N; ++j) t[j] = fabs(v[j]);
#pragma unroll
  for (int w = 1; w < N; w <<= 1)
#pragma unroll
    for (int j = 0; j + w < N; j += 2 * w) t[j] = fmax(t[j], t[j + w]);
  return fmax(0.0, t[0]);
}

// ---- LU with partial pivoting, in registers (linalg.cpp:201-258) --------
template <int D>
__device__ __forceinline__ bool lu_solve_inplace(double (&A)[D][D], double (&b)[D]) {
  int piv[D];
#if PFSMC_FAST
  double invd[D];  // fast variant: back substitution multiplies by the pivot reciprocals
#endif
#pragma unroll
  for (int col = 0; col < D; ++col) {
    int pivot = col;
    double best = fabs(A[col][col]);
#pragma unroll
    for (int r = col + 1; r < D; ++r) {
      const double v = fabs(A[r][col]);
      if (v > best) {
        best = v;
        pivot = r;
      }
    }
    if (best == 0.0) return false;
    piv[col] = pivot;
#pragma unroll
    for (int r = col + 1; r < D; ++r) {
      if (pivot == r) {
#pragma unroll
        for (int j = 0; j < D; ++j) {
          const double t = A[col][j];
          A[col][j] = A[r][j];
          A[r][j] = t;
        }
      }
    }
    const double inv = 1.0 / A[col][col];
#if PFSMC_FAST
    invd[col] = inv;
#endif
#pragma unroll
    for (int r = col + 1; r < D; ++r) {
      const double f = A[r][col] * inv;
      A[r][col] = f;
      if (f != 0.0) {
#pragma unroll
        for (int j = col + 1; j < D; ++j) A[r][j] -= f * A[col][j];
      }
    }
  }
#pragma unroll
  for (int i = 0; i < D; ++i) {
#pragma unroll
    for (int r = i + 1; r < D; ++r) {
      if (piv[i] == r) {
        const double t = b[i];
        b[i] = b[r];
        b[r] = t;
      }
    }
#pragma unroll
    for (int j = 0; j < i; ++j) b[i] -= A[i][j] * b[j];
  }
#pragma unroll
  for (int ii = D - 1; ii >= 0; --ii) {
#pragma unroll
    for (int j = ii + 1; j < D; ++j) b[ii] -= A[ii][j] * b[j];
#if PFSMC_FAST
    b[ii] *= invd[ii];
#else
    b[ii] /= A[ii][ii];
#endif
  }
  return true;
}

// Structured path for models whose Jacobian (hence I - h b0 J) is lower
// bidiagonal (M::jac_band gives the diagonal and subdiagonal). When no
// partial-pivoting swap is triggered (the reference's rule: first strictly
// larger |.|) and every band entry is finite with a normal diagonal, the
// dense elimination (linalg.cpp:201-258) performs on the band exactly the
// operations done here; the ones it adds only combine structural zeros (+-0)
// with finite values, leaving every band entry bit-identical. Anything else
// takes the dense path below, which rebuilds J with M::jac; it is kept out of
// line so the 8x8 matrix never lives in the hot loop's registers.
template <class M>
__device__ __forceinline__ bool dense_newton_solve(const typename M::K& mk, double tn, const double* th_p,
                                                   const double* x_p, double hb0, double* r_p) {
  constexpr int D = M::D;
  double th[M::P], x[D], r[D], A[D][D];
  for (int j = 0; j < M::P; ++j) th[j] = th_p[j];
  for (int j = 0; j < D; ++j) x[j] = x_p[j], r[j] = r_p[j];
  M::jac(mk, tn, th, x, A);  // finite: jac_band (same entries) was checked
  for (int i = 0; i < D; ++i)
    for (int j = 0; j < D; ++j) A[i][j] = -hb0 * A[i][j];
  for (int i = 0; i < D; ++i) A[i][i] += 1.0;
  const bool ok = lu_solve_inplace<D>(A, r);
  for (int j = 0; j < D; ++j) r_p[j] = r[j];
  return ok;
}

template <class M>
__device__ __forceinline__ bool band_solve(const typename M::K& mk, double tn, const double (&th)[M::P],
                                           const double (&x)[M::D],
                                           double hb0, const double (&jd)[M::D],
                                           const double (&js)[M::D - 1], double (&b)[M::D]) {
  constexpr int D = M::D;
  double dg[D], sb[D - 1];
  bool fast = true;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    dg[i] = -hb0 * jd[i];
    dg[i] += 1.0;
    // DBL_MIN <= |dg| <= DBL_MAX (not NaN), decided by the high word alone
    const unsigned ha = static_cast<unsigned>(__double2hiint(dg[i])) & 0x7fffffffu;
    fast &= ha - 0x00100000u < 0x7ff00000u - 0x00100000u;
  }
#pragma unroll
  for (int c = 0; c + 1 < D; ++c) {
    sb[c] = -hb0 * js[c];
    fast &= !(fabs(sb[c]) > fabs(dg[c]));
  }
  if (!fast) return dense_newton_solve<M>(mk, tn, th, x, hb0, b);
#if PFSMC_FAST
  // fast variant: the D pivot reciprocals in one batch; forward elimination
  // and back substitution multiply by them (no division)
  {
    double inv[D];
    drcp_batch<D>(dg, inv);
#pragma unroll
    for (int i = 1; i < D; ++i) b[i] -= (sb[i - 1] * inv[i - 1]) * b[i - 1];
#pragma unroll
    for (int i = 0; i < D; ++i) b[i] *= inv[i];
    return true;
  }
#endif
  // the D - 1 pivot reciprocals (inv = 1 / pivot, linalg.cpp:215) and the D
  // back-substitution divisions are independent: batched IEEE divisions
  double one[D - 1], inv[D - 1];
#pragma unroll
  for (int i = 0; i + 1 < D; ++i) one[i] = 1.0;
  double dgl[D - 1];
#pragma unroll
  for (int i = 0; i + 1 < D; ++i) dgl[i] = dg[i];
  ddiv_batch<D - 1>(one, dgl, inv);
#pragma unroll
  for (int i = 1; i < D; ++i) {
    const double l = sb[i - 1] * inv[i - 1];
    b[i] -= l * b[i - 1];
  }
  double bb[D];
#pragma unroll
  for (int i = 0; i < D; ++i) bb[i] = b[i];
  ddiv_batch<D>(bb, dg, b);
  return true;
}

// ---- Newton on G(x) = x - h b0 f(x) - c (lmm.cpp:219-266) ---------------
template <class M>
__device__ __forceinline__ int newton_solve(const typename M::K& mk, double tn, const double (&th)[M::P],
                                            double hb0,
                                            const double (&c)[M::D], double (&x)[M::D],
                                            double tol, int max_iter, int& iters) {
  constexpr int D = M::D;
  for (int iter = 1; iter <= max_iter; ++iter) {
    double f[D], r[D];
    bool solved;
    if constexpr (M::kLowerBidiagonal) {
      // rhs and the Jacobian band from one pass over x (their divisions in one
      // batch); the verdicts are checked in the reference's order (rhs first)
      double jd[D], js[D - 1];
      bool ok_f, ok_j;
      M::rhs_jac_band(mk, tn, th, x, f, ok_f, jd, js, ok_j);
      if (!ok_f || !ok_j) {
        iters += iter;
        return kInvalidRhs;
      }
#pragma unroll
      for (int j = 0; j < D; ++j) r[j] = x[j] - hb0 * f[j] - c[j];
      solved = band_solve<M>(mk, tn, th, x, hb0, jd, js, r);
    } else {
      if (!M::rhs(mk, tn, th, x, f)) {
        iters += iter;
        return kInvalidRhs;
      }
#pragma unroll
      for (int j = 0; j < D; ++j) r[j] = x[j] - hb0 * f[j] - c[j];
      double A[D][D];
      if (!M::jac(mk, tn, th, x, A)) {
        iters += iter;
        return kInvalidRhs;
      }
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) A[i][j] = -hb0 * A[i][j];
#pragma unroll
      for (int i = 0; i < D; ++i) A[i][i] += 1.0;
      solved = lu_solve_inplace<D>(A, r);
    }
    if (!solved) {
      iters += iter;
      return kSingular;
    }
    // the max-norms (lmm.cpp:250-256: a std::max pass from 0 over |.|, which
    // skips NaN entries) as fmax trees: fmax also skips NaN and max is exact,
    // so the values are the reference's, with a log-depth dependency chain
#pragma unroll
    for (int j = 0; j < D; ++j) x[j] -= r[j];
    const double dn = max_abs_tree<D>(r), xn = max_abs_tree<D>(x);
    if (!isfinite(xn) || !isfinite(dn)) {
      iters += iter;
      return kInvalidRhs;
    }
    if (dn <= tol * (1.0 + xn)) {
      iters += iter;
      return kOk;
    }
  }
  iters += max_iter;
  return kNewtonDivergence;
}

// ---- the ramped interval propagator ------------------------------------
template <class M, int FAM, int ORD>
struct Propagator {
  static constexpr int D = M::D;
  static constexpr int P = M::P;
  // ORD == 0: the adaptive BDF(1,2) integrator (run_adaptive only)
  static constexpr int SD = FAM == kBDF ? ORD + 1 : 1;              // states kept
  static constexpr int FD = ORD == 0 ? 1 : FAM == kAB ? ORD + 1 : ORD;  // f values kept

  // History storage: registers, or (models with kSmemHistory: the 8-species
  // chain) a per-thread column of dynamic shared memory bound by the kernel
  // (bind_history), entry (slot, j) at hist_[(slot * D + j) * kHistStride], as
  // ring buffers. Same values, same arithmetic; the registers it frees let
  // three CTAs share an SM instead of one.
  static constexpr bool kSmemHist = SmemHistOf<M>::value;
  static constexpr int kHistStride = BlockOf<M>::value;
  static constexpr int kHistDoubles = (SD + FD) * D;  // per thread
  double xs[kSmemHist ? 1 : SD][D];
  double fs[kSmemHist ? 1 : FD][D];
  double* hist_ = nullptr;
  int hx = 0, hf = 0;
  __device__ __forceinline__ void bind_history(double* column) { hist_ = column; }
  __device__ __forceinline__ double& X(int i, int j) {
    if constexpr (kSmemHist) {
      const int sl = hx + i < SD ? hx + i : hx + i - SD;
      return hist_[(sl * D + j) * kHistStride];
    } else {
      return xs[i][j];
    }
  }
  __device__ __forceinline__ double X(int i, int j) const { return const_cast<Propagator*>(this)->X(i, j); }
  __device__ __forceinline__ double& F(int i, int j) {
    if constexpr (kSmemHist) {
      const int sl = hf + i < FD ? hf + i : hf + i - FD;
      return hist_[((SD + sl) * D + j) * kHistStride];
    } else {
      return fs[i][j];
    }
  }
  __device__ __forceinline__ double F(int i, int j) const { return const_cast<Propagator*>(this)->F(i, j); }
  typename M::K mk;  // model constants (the bound OdeModel's state, models.hpp:20-55)

  // AB(q) explicit combination: 0 + 1.0*x_n, then (h*beta_i) f_{n+1-i}.
  template <int Q>
  __device__ __forceinline__ void ab_step(double h, double (&out)[D]) const {
#pragma unroll
    for (int j = 0; j < D; ++j) out[j] = 0.0 + 1.0 * X(0, j);
#pragma unroll
    for (int i = 1; i <= Q; ++i) {
      const double hb = h * ab_beta(Q, i);
#pragma unroll
      for (int j = 0; j < D; ++j) out[j] += hb * F(i - 1, j);
    }
  }

  // implicit_history_terms for AM(p) / BDF(p) (lmm.cpp:130-144).
  template <int PA>
  __device__ __forceinline__ void implicit_terms(double h, double (&c)[D]) const {
    if constexpr (FAM == kAM) {
#pragma unroll
      for (int j = 0; j < D; ++j) c[j] = 0.0 + 1.0 * X(0, j);
#pragma unroll
      for (int i = 1; i < PA; ++i) {
        const double hb = h * am_beta(PA, i);
#pragma unroll
        for (int j = 0; j < D; ++j) c[j] += hb * F(i - 1, j);
      }
    } else {
#pragma unroll
      for (int j = 0; j < D; ++j) c[j] = 0.0;
#pragma unroll
      for (int i = 0; i < PA; ++i) {
        const double a = bdf_alpha(PA, i);
#pragma unroll
        for (int j = 0; j < D; ++j) c[j] += a * X(i, j);
      }
    }
  }

  // extrapolate_predictor(q) (lmm.cpp:146-165); the binomials are exact.
  template <int Q>
  __device__ __forceinline__ void extrapolate(double (&out)[D]) const {
#pragma unroll
    for (int j = 0; j < D; ++j) out[j] = 0.0;
    double binom = static_cast<double>(Q) + 1.0;
    double sign = 1.0;
#pragma unroll
    for (int i = 0; i <= Q; ++i) {
      const double coef = sign * binom;
#pragma unroll
      for (int j = 0; j < D; ++j) out[j] += coef * X(i, j);
      sign = -sign;
      binom = binom * static_cast<double>(Q + 1 - (i + 1)) / static_cast<double>(i + 2);
    }
  }

  __device__ __forceinline__ void push(const double (&x)[D], const double (&f)[D]) {
    if constexpr (kSmemHist) {
      // ring buffers: the newest entry moves one slot down, nothing is copied
      hx = hx == 0 ? SD - 1 : hx - 1;
      hf = hf == 0 ? FD - 1 : hf - 1;
    } else {
#pragma unroll
      for (int i = SD - 1; i > 0; --i)
#pragma unroll
        for (int j = 0; j < D; ++j) xs[i][j] = xs[i - 1][j];
#pragma unroll
      for (int i = FD - 1; i > 0; --i)
#pragma unroll
        for (int j = 0; j < D; ++j) fs[i][j] = fs[i - 1][j];
    }
#pragma unroll
    for (int j = 0; j < D; ++j) {
      X(0, j) = x[j];
      F(0, j) = f[j];
    }
  }

  // One ramp step at compile-time active order PA with AV history entries.
  // Returns the particle status (kOk keeps going).
  template <int PA, int AV>
  __device__ __forceinline__ int step(const double (&th)[P], double tn, double h, double tol, int max_iter,
                                      double (&gamma)[D], int& iters) {
    double xnew[D], ref[D];
    double factor;
    if constexpr (FAM == kAB) {
      ab_step<PA>(h, xnew);
      if constexpr (AV >= PA + 1) {
        ab_step<PA + 1>(h, ref);
      } else if constexpr (PA >= 2) {
        ab_step<PA - 1>(h, ref);
      } else {
#pragma unroll
        for (int j = 0; j < D; ++j) ref[j] = X(0, j);
      }
      factor = 1.0;
    } else {
      double c[D];
      implicit_terms<PA>(h, c);
      ab_step<PA>(h, xnew);  // Newton's initial guess: explicit AB(q), q = PA
      if constexpr (FAM == kAM) {
#pragma unroll
        for (int j = 0; j < D; ++j) ref[j] = xnew[j];
        factor = fabs(am_C(PA)) / fabs(ab_C(PA) - am_C(PA));
      } else if constexpr (AV >= PA + 1) {
        extrapolate<PA>(ref);
        factor = fabs(bdf_C(PA)) / fabs(1.0 - bdf_C(PA));
      } else if constexpr (AV < 2) {
#pragma unroll
        for (int j = 0; j < D; ++j) ref[j] = xnew[j];
        factor = fabs(bdf_C(PA)) / fabs(ab_C(PA) - bdf_C(PA));
      } else {
        extrapolate<AV - 1>(ref);
        factor = fabs(bdf_C(PA)) / fabs(1.0 - bdf_C(PA));
      }
      const double b0 = FAM == kAM ? am_beta(PA, 0) : bdf_beta0(PA);
      const int st = newton_solve<M>(mk, tn, th, h * b0, c, xnew, tol, max_iter, iters);
      if (st != kOk) return st;
    }
    // finish_step (lmm.cpp:438-452)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const double est = factor * fabs(xnew[j] - ref[j]);
      gamma[j] += est * est;
    }
    double fnew[D];
    if (!M::rhs(mk, tn, th, xnew, fnew)) return kInvalidRhs;
    push(xnew, fnew);
    return kOk;
  }

  // ---- runtime-order forms (large d) -------------------------------------
  // For large state dimensions the four compile-time ramp instantiations
  // (each with its own inlined Newton + LU) blow the kernel past the
  // instruction cache. These forms run ONE step body for every ramp step:
  // loops go to the compile-time maximum under a warp-uniform predicate, so
  // history indices stay static (registers) and the floating-point operation
  // sequence is exactly that of the templates above.
  __device__ __forceinline__ void ab_step_rt(int q, double h, double (&out)[D]) const {
#pragma unroll
    for (int j = 0; j < D; ++j) out[j] = 0.0 + 1.0 * X(0, j);
#pragma unroll
    for (int i = 1; i <= FD; ++i) {
      if (i <= q) {
        const double hb = h * ab_beta(q, i);
#pragma unroll
        for (int j = 0; j < D; ++j) out[j] += hb * F(i - 1, j);
      }
    }
  }
  __device__ __forceinline__ void implicit_terms_rt(int pa, double h, double (&c)[D]) const {
    if constexpr (FAM == kAM) {
#pragma unroll
      for (int j = 0; j < D; ++j) c[j] = 0.0 + 1.0 * X(0, j);
#pragma unroll
      for (int i = 1; i < FD + 1; ++i) {
        if (i < pa) {
          const double hb = h * am_beta(pa, i);
#pragma unroll
          for (int j = 0; j < D; ++j) c[j] += hb * F(i - 1, j);
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < D; ++j) c[j] = 0.0;
#pragma unroll
      for (int i = 0; i < SD; ++i) {
        if (i < pa) {
          const double a = bdf_alpha(pa, i);
#pragma unroll
          for (int j = 0; j < D; ++j) c[j] += a * X(i, j);
        }
      }
    }
  }
  __device__ __forceinline__ void extrapolate_rt(int q, double (&out)[D]) const {
#pragma unroll
    for (int j = 0; j < D; ++j) out[j] = 0.0;
    double binom = static_cast<double>(q) + 1.0;
    double sign = 1.0;
#pragma unroll
    for (int i = 0; i < SD; ++i) {
      if (i <= q) {
        const double coef = sign * binom;
#pragma unroll
        for (int j = 0; j < D; ++j) out[j] += coef * X(i, j);
        sign = -sign;
        binom = binom * static_cast<double>(q + 1 - (i + 1)) / static_cast<double>(i + 2);
      }
    }
  }
  __device__ __forceinline__ int step_rt(int pa, int av, const double (&th)[P], double tn, double h, double tol,
                                         int max_iter, double (&gamma)[D], int& iters) {
    double xnew[D], ref[D];
    double factor;
    if constexpr (FAM == kAB) {
      ab_step_rt(pa, h, xnew);
      if (av >= pa + 1) {
        ab_step_rt(pa + 1, h, ref);
      } else if (pa >= 2) {
        ab_step_rt(pa - 1, h, ref);
      } else {
#pragma unroll
        for (int j = 0; j < D; ++j) ref[j] = X(0, j);
      }
      factor = 1.0;
    } else {
      double c[D];
      implicit_terms_rt(pa, h, c);
      ab_step_rt(pa, h, xnew);
      if constexpr (FAM == kAM) {
#pragma unroll
        for (int j = 0; j < D; ++j) ref[j] = xnew[j];
        factor = fabs(am_C(pa)) / fabs(ab_C(pa) - am_C(pa));
      } else {
        if (av >= pa + 1) {
          extrapolate_rt(pa, ref);
          factor = fabs(bdf_C(pa)) / fabs(1.0 - bdf_C(pa));
        } else if (av < 2) {
#pragma unroll
          for (int j = 0; j < D; ++j) ref[j] = xnew[j];
          factor = fabs(bdf_C(pa)) / fabs(ab_C(pa) - bdf_C(pa));
        } else {
          extrapolate_rt(av - 1, ref);
          factor = fabs(bdf_C(pa)) / fabs(1.0 - bdf_C(pa));
        }
      }
      const double b0 = FAM == kAM ? am_beta(pa, 0) : bdf_beta0(pa);
      const int st = newton_solve<M>(mk, tn, th, h * b0, c, xnew, tol, max_iter, iters);
      if (st != kOk) return st;
    }
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const double est = factor * fabs(xnew[j] - ref[j]);
      gamma[j] += est * est;
    }
    double fnew[D];
    if (!M::rhs(mk, tn, th, xnew, fnew)) return kInvalidRhs;
    push(xnew, fnew);
    return kOk;
  }

  // propagate_interval (lmm.cpp:468-503): m fixed steps of size h from x.
  // On return x holds the last accepted state (the reference's run.x).
  // adaptive_bdf_interval (lmm.cpp:894-1019): variable-step BDF(1,2), the
  // step size driven per particle by the predictor error estimate; Newton as
  // in the fixed-step path; gamma = rtol * accepted steps in every component.
  // The history is three accepted points (x, x_{-1}, x_{-2}) in registers.
  __device__ __forceinline__ int run_adaptive(const double (&th)[P], double (&x)[D], double t0, double t1,
                                              double rtol, double tol, int max_iter, double (&gamma)[D],
                                              int& iters) {
#pragma unroll
    for (int j = 0; j < D; ++j) gamma[j] = 0.0;
    const double total = t1 - t0;
    const double h_min = total * 1e-10;
    double fcur[D], xm1[D], xm2[D];
#pragma unroll
    for (int j = 0; j < D; ++j) xm1[j] = xm2[j] = 0.0;
    double tm1 = 0.0, tm2 = 0.0;
    int npoints = 1;
    long long steps = 0;
    if (!M::rhs(mk, t0, th, x, fcur)) return kInvalidRhs;
    double t = t0;
    double h = total * 1e-2;
    long long attempts = 0;
    while (t < t1 - total * 1e-12) {
      h = ref_min(h, t1 - t);
      if (h < h_min) return kStiffness;
      // no such bound in the reference (see kAdaptiveMaxAttempts)
      if (++attempts > kAdaptiveMaxAttempts) return kStiffness;
      const int p = npoints >= 2 ? 2 : 1;
      const double t_next = t + h;
      double hb0, factor, c[D], pred[D];
      if (p == 1) {
#pragma unroll
        for (int j = 0; j < D; ++j) {
          c[j] = x[j];
          pred[j] = x[j] + h * fcur[j];
        }
        hb0 = h;
        factor = 0.5;
      } else {
        const double h_prev = t - tm1;
        const double omega = h / h_prev;
        const double a2 = -(omega * omega) / (1.0 + 2.0 * omega);
        hb0 = h * (1.0 + omega) / (1.0 + 2.0 * omega);
#pragma unroll
        for (int j = 0; j < D; ++j) c[j] = x[j] + a2 * (xm1[j] - x[j]);
        if (npoints >= 3) {
          const double dt1 = t - tm1;
          const double dt2 = tm1 - tm2;
#pragma unroll
          for (int j = 0; j < D; ++j) {
            const double dd1 = (x[j] - xm1[j]) / dt1;
            const double dd1p = (xm1[j] - xm2[j]) / dt2;
            const double dd2 = (dd1 - dd1p) / (t - tm2);
            pred[j] = x[j] + h * dd1 + h * (h + dt1) * dd2;
          }
        } else {
#pragma unroll
          for (int j = 0; j < D; ++j) pred[j] = x[j] + omega * (x[j] - xm1[j]);
        }
        factor = 2.0 / 11.0;
      }
      double xnew[D];
#pragma unroll
      for (int j = 0; j < D; ++j) xnew[j] = pred[j];
      if (newton_solve<M>(mk, t_next, th, hb0, c, xnew, tol, max_iter, iters) != kOk) {
        h *= 0.25;
        continue;
      }
      double err = 0.0, xn = 0.0;
#pragma unroll
      for (int j = 0; j < D; ++j) {
        err = ref_max(err, factor * fabs(xnew[j] - pred[j]));
        xn = ref_max(xn, fabs(xnew[j]));
      }
      const double est_rel = err / (1.0 + xn);
      double growth;
      if (est_rel == 0.0) {
        growth = 4.0;
      } else {
        growth = 0.9 * pow(rtol / est_rel, 1.0 / (static_cast<double>(p) + 1.0));
        growth = ref_clamp(growth, 0.25, 4.0);
      }
      if (est_rel <= rtol) {
        if (!M::rhs(mk, t_next, th, xnew, fcur)) return kInvalidRhs;
#pragma unroll
        for (int j = 0; j < D; ++j) {
          xm2[j] = xm1[j];
          xm1[j] = x[j];
          x[j] = xnew[j];
        }
        tm2 = tm1;
        tm1 = t;
        t = t_next;
        npoints = npoints + 1 < 3 ? npoints + 1 : 3;
        ++steps;
      }
      h *= growth;
    }
    const double g = rtol * static_cast<double>(steps);
#pragma unroll
    for (int j = 0; j < D; ++j) gamma[j] = g;
    return kOk;
  }

  // t_next = t0 + k h (lmm.cpp:482), not an accumulated sum.
  __device__ __forceinline__ int run(const double (&th)[P], double (&x)[D], double t0, double h, int m,
                                     double tol, int max_iter, double (&gamma)[D], int& iters) {
#pragma unroll
    for (int j = 0; j < D; ++j) gamma[j] = 0.0;
    double f0[D];
    if (!M::rhs(mk, t0, th, x, f0)) return kInvalidRhs;
    hx = hf = 0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      X(0, j) = x[j];
      F(0, j) = f0[j];
    }
    int st = kOk;
    if constexpr (D >= 6) {
      for (int k = 1; k <= m && st == kOk; ++k)
        st = step_rt(cmin(k, ORD), cmin(k, 4), th, t0 + static_cast<double>(k) * h, h, tol, max_iter, gamma,
                     iters);
      if (true) {
#pragma unroll
        for (int j = 0; j < D; ++j) x[j] = X(0, j);
        return st;
      }
    }
    for (int k = 1; k <= m && st == kOk; ++k) {
      if (k == 1)
        st = step<1, 1>(th, t0 + static_cast<double>(k) * h, h, tol, max_iter, gamma, iters);
      else if (k == 2)
        st = step<cmin(2, ORD), 2>(th, t0 + static_cast<double>(k) * h, h, tol, max_iter, gamma, iters);
      else if (k == 3)
        st = step<cmin(3, ORD), 3>(th, t0 + static_cast<double>(k) * h, h, tol, max_iter, gamma, iters);
      else
        st = step<ORD, 4>(th, t0 + static_cast<double>(k) * h, h, tol, max_iter, gamma, iters);
    }
#pragma unroll
    for (int j = 0; j < D; ++j) x[j] = X(0, j);
    return st;
  }
};

PFSMC_END  // namespace pfsmc_gpu::PFSMC_VNS
