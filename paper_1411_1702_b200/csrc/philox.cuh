// Counter-based RNG shared by every kernel: Philox4x64-10 with the
// reference's key constant and counter layout, so a draw is a pure function
// of (seed, time index j, slot n, purpose, block#) exactly as in
// /root/reference/proj/src/rng.cpp:9-75 (pinned by
// tests/data/philox_vectors.csv there; tests/golden/philox_vectors.json here).
//
// 64x64->128 multiplies use the native IMAD.WIDE.U32-based __umul64hi plus a
// plain 64-bit multiply; everything is integer, so device words are
// bit-identical to the reference. Uniforms/normals follow rng.cpp:57-75; the
// normals go through CUDA's log and sincospi (a few ulp from glibc's log/sin/cos
// of fl(2 pi u)) and are the one
// place device streams are not bitwise equal to the host's.
#pragma once
#include <cstdint>

#ifdef __CUDACC__
#define PF_HD __host__ __device__ __forceinline__
#else
#define PF_HD inline
#endif

namespace pfsmc_gpu {

enum Purpose : uint64_t { kInit = 0, kProliferate = 1, kInnovate = 2, kResample = 3 };

constexpr uint64_t kMult0 = 0xD2E7470EE14C6C93ULL;
constexpr uint64_t kMult1 = 0xCA5A826395121157ULL;
constexpr uint64_t kWeyl0 = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t kWeyl1 = 0xBB67AE8584CAA73BULL;
constexpr uint64_t kKeyConstant = 0x7066736D632D3031ULL;  // "pfsmc-01"

PF_HD void mulhilo64(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
#ifdef __CUDA_ARCH__
  // mul.lo.u64 + mul.hi.u64 (measured cheaper in SASS than a hand-split
  // 4 x IMAD.WIDE.U32 product, profiles/r01_notes.md)
  lo = a * b;
  hi = __umul64hi(a, b);
#else
  const unsigned __int128 p = static_cast<unsigned __int128>(a) * b;
  hi = static_cast<uint64_t>(p >> 64);
  lo = static_cast<uint64_t>(p);
#endif
}

struct U64x4 {
  uint64_t v[4];
};

// rng.cpp:28-41
PF_HD U64x4 philox4x64(uint64_t c0, uint64_t c1, uint64_t c2, uint64_t c3,
                       uint64_t k0, uint64_t k1) {
#pragma unroll
  for (int round = 0; round < 10; ++round) {
    if (round > 0) {
      k0 += kWeyl0;
      k1 += kWeyl1;
    }
    uint64_t hi0, lo0, hi1, lo1;
    mulhilo64(kMult0, c0, hi0, lo0);
    mulhilo64(kMult1, c2, hi1, lo1);
    const uint64_t n0 = hi1 ^ c1 ^ k0;
    const uint64_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  return {{c0, c1, c2, c3}};
}

PF_HD double u64_to_uniform(uint64_t w) {
  return static_cast<double>(w >> 11) * 0x1.0p-53;
}

#ifdef __CUDACC__
// Box-Muller's two transcendental steps on their restricted domains, cheaper
// than the general libm routines (whose dynamic paths are ~65 and ~75
// instructions here, ~15% of k_update). Accuracy: a few ulp (measured by
// profiles/probe_fastmath.cu against CUDA's log / sincospi), far inside the
// 1e-10 state tolerance; the reference's own glibc values already differ from
// CUDA's by up to 2 ulp.
//
// log(u) for u in [2^-53, 1]: u = 2^e m, m in [sqrt(1/2), sqrt(2)),
// log(m) = 2 atanh(s), s = (m - 1) / (m + 1), |s| <= 0.1716, the atanh series
// to s^21 (truncation < 2^-60 relative), e ln2 in two parts.
__device__ __forceinline__ double log_unit(double u) {
  const long long bits = __double_as_longlong(u);
  int e = static_cast<int>((bits >> 52) & 0x7ff) - 1023;
  double m = __longlong_as_double((bits & 0x000FFFFFFFFFFFFFLL) | 0x3FF0000000000000LL);
  if (m > 1.4142135623730951) {
    m *= 0.5;
    e += 1;
  }
  const double f = m - 1.0;
  const double den = m + 1.0;
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(den));
  r = fma(r, fma(-den, r, 1.0), r);
  r = fma(r, fma(-den, r, 1.0), r);
  const double s = f * r;
  const double s2 = s * s;
  double p = 0x1.642c8590b2164p-5;  // 1/21
  p = fma(p, s2, 0x1.8618618618618p-5);
  p = fma(p, s2, 0x1.af286bca1af28p-5);
  p = fma(p, s2, 0x1.e1e1e1e1e1e1ep-5);
  p = fma(p, s2, 0x1.1111111111111p-4);
  p = fma(p, s2, 0x1.3b13b13b13b14p-4);
  p = fma(p, s2, 0x1.745d1745d1746p-4);
  p = fma(p, s2, 0x1.c71c71c71c71cp-4);
  p = fma(p, s2, 0x1.2492492492492p-3);
  p = fma(p, s2, 0x1.999999999999ap-3);
  p = fma(p, s2, 0x1.5555555555555p-2);  // 1/3
  const double t = 2.0 * s;
  const double lm = fma(t * s2, p, t);  // 2 atanh(s)
  const double de = static_cast<double>(e);
  return fma(de, 0x1.62e42fefa39efp-1, fma(de, 0x1.abc9e3b39803fp-56, lm));
}

// sqrt(a) for a >= 0 (the Box-Muller radius): hardware rsqrt estimate, two
// Newton steps and one correction of the square root (<= 1 ulp measured).
__device__ __forceinline__ double sqrt_nonneg(double a) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
  const double ha = 0.5 * a;
  y = y * fma(-ha * y, y, 1.5);
  y = y * fma(-ha * y, y, 1.5);
  const double r = a * y;
  return a == 0.0 ? 0.0 : fma(0.5 * y, fma(-r, r, a), r);
}

// sin(pi x), cos(pi x) for x in [0, 2): x = q/2 + t exactly (x is a multiple
// of 2^-52), |t| <= 1/4, Taylor polynomials of sin(pi t) to t^17 and cos(pi t)
// to t^18 (truncation < 2^-58), then the quadrant q mod 4.
__device__ __forceinline__ void sincospi_unit(double x, double* sp, double* cp) {
  const double q = rint(2.0 * x);
  const double t = fma(-0.5, q, x);
  const double t2 = t * t;
  double ps = 0x1.aaec32af93359p-21;
  ps = fma(ps, t2, -0x1.6fadb9f155744p-16);
  ps = fma(ps, t2, 0x1.e8f434d018d63p-12);
  ps = fma(ps, t2, -0x1.e3074fde8871fp-8);
  ps = fma(ps, t2, 0x1.50783487ee782p-4);
  ps = fma(ps, t2, -0x1.32d2cce62bd86p-1);
  ps = fma(ps, t2, 0x1.466bc6775aae2p+1);
  ps = fma(ps, t2, -0x1.4abbce625be53p+2);
  ps = fma(ps, t2, 0x1.921fb54442d18p+1);
  const double sn = ps * t;
  double pc = -0x1.2a0c591af8314p-23;
  pc = fma(pc, t2, 0x1.20c62c2f2d7f5p-18);
  pc = fma(pc, t2, -0x1.b6e24f44b128fp-14);
  pc = fma(pc, t2, 0x1.f9d38a3763cc3p-10);
  pc = fma(pc, t2, -0x1.a6d1f2a204a8cp-6);
  pc = fma(pc, t2, 0x1.e1f506891babbp-3);
  pc = fma(pc, t2, -0x1.55d3c7e3cbffap+0);
  pc = fma(pc, t2, 0x1.03c1f081b5ac4p+2);
  pc = fma(pc, t2, -0x1.3bd3cc9be45dep+2);
  const double cs = fma(pc, t2, 1.0);
  const int qi = static_cast<int>(q) & 3;
  const double s0 = (qi & 1) ? cs : sn;
  const double c0 = (qi & 1) ? sn : cs;
  *sp = (qi & 2) ? -s0 : s0;
  *cp = ((qi + 1) & 2) ? -c0 : c0;
}
#endif

// One keyed stream, consumed in lane order (rng.cpp:43-75). With the draw
// counts of every call site known at compile time and the loops unrolled,
// block/lane/spare live in registers.
struct Stream {
  uint64_t seed, j, n, purpose;
  uint64_t block_index;
  int lane;
  bool have_spare;
  double spare;
  U64x4 block;

  PF_HD Stream(uint64_t seed_, uint64_t j_, uint64_t n_, uint64_t purpose_)
      : seed(seed_), j(j_), n(n_), purpose(purpose_), block_index(0), lane(4),
        have_spare(false), spare(0.0), block{{0, 0, 0, 0}} {}

  PF_HD uint64_t next_u64() {
    if (lane == 4) {
      block = philox4x64(block_index++, j, n, purpose, seed, kKeyConstant);
      lane = 0;
    }
    const uint64_t w = block.v[lane];
    ++lane;
    return w;
  }
  PF_HD double next_uniform() { return u64_to_uniform(next_u64()); }
  PF_HD double next_normal() {
    if (have_spare) {
      have_spare = false;
      return spare;
    }
    const double u1 = (static_cast<double>(next_u64() >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = next_uniform();
#ifdef __CUDA_ARCH__
    const double r = sqrt_nonneg(-2.0 * log_unit(u1));
    double s, c;
    sincospi_unit(2.0 * u2, &s, &c);  // as stream_normals below
#else
    const double r = sqrt(-2.0 * log(u1));
    double s, c;
    const double angle = 2.0 * 3.14159265358979323846 * u2;
    s = sin(angle);
    c = cos(angle);
#endif
    spare = r * s;
    have_spare = true;
    return r * c;
  }
};


// The first K normals of stream (seed, j, n, purpose), in the order
// RngStream::next_normal returns them (rng.cpp:61-75): pair q uses words 2q
// (u1) and 2q+1 (u2) and yields r cos, then the cached r sin. All indices are
// compile-time, so nothing spills to local memory.
template <int K>
PF_HD void stream_normals(uint64_t seed, uint64_t j, uint64_t n, uint64_t purpose,
                          double (&out)[K]) {
  constexpr int kPairs = (K + 1) / 2;
  constexpr int kBlocks = (2 * kPairs + 3) / 4;
  uint64_t w[kBlocks * 4];
#pragma unroll
  for (int b = 0; b < kBlocks; ++b) {
    const U64x4 blk = philox4x64(static_cast<uint64_t>(b), j, n, purpose, seed, kKeyConstant);
#pragma unroll
    for (int l = 0; l < 4; ++l) w[4 * b + l] = blk.v[l];
  }
#pragma unroll
  for (int q = 0; q < kPairs; ++q) {
    const double u1 = (static_cast<double>(w[2 * q] >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = u64_to_uniform(w[2 * q + 1]);
    double s, c;
#ifdef __CUDA_ARCH__
    const double r = sqrt_nonneg(-2.0 * log_unit(u1));
    // sin/cos(2 pi u2) without the range reduction (2 u2 is exact); differs
    // from sin(fl(2 pi u2)) by the rounding of the product, <= 4.4e-16 absolute
    sincospi_unit(2.0 * u2, &s, &c);
#else
    const double r = sqrt(-2.0 * log(u1));
    const double angle = 2.0 * 3.14159265358979323846 * u2;
    s = sin(angle);
    c = cos(angle);
#endif
    out[2 * q] = r * c;
    if (2 * q + 1 < K) out[2 * q + 1] = r * s;
  }
}

// The resampling uniform of slot n at time j (filter.cpp:171-172).
PF_HD double resample_uniform(uint64_t seed, uint64_t j, uint64_t n) {
  return u64_to_uniform(philox4x64(0, j, n, kResample, seed, kKeyConstant).v[0]);
}

}  // namespace pfsmc_gpu
