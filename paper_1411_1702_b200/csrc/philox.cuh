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
#include "variant.cuh"
#include <cstdint>

#ifdef __CUDACC__
#define PF_HD __host__ __device__ __forceinline__
#else
#define PF_HD inline
#endif

PFSMC_BEGIN

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

// rng.cpp:28-41. ROLL: the ten rounds as a loop (kernels whose code size
// matters more than the loop overhead); same words.
PF_HD void philox_round(uint64_t& c0, uint64_t& c1, uint64_t& c2, uint64_t& c3, uint64_t k0, uint64_t k1) {
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
template <bool ROLL = false>
PF_HD U64x4 philox4x64(uint64_t c0, uint64_t c1, uint64_t c2, uint64_t c3,
                       uint64_t k0, uint64_t k1) {
  if constexpr (ROLL) {
    philox_round(c0, c1, c2, c3, k0, k1);
#pragma unroll 1
    for (int round = 1; round < 10; ++round) {
      k0 += kWeyl0;
      k1 += kWeyl1;
      philox_round(c0, c1, c2, c3, k0, k1);
    }
  } else {
#pragma unroll
    for (int round = 0; round < 10; ++round) {
      if (round > 0) {
        k0 += kWeyl0;
        k1 += kWeyl1;
      }
      philox_round(c0, c1, c2, c3, k0, k1);
    }
  }
  return {{c0, c1, c2, c3}};
}

PF_HD double u64_to_uniform(uint64_t w) {
  return static_cast<double>(w >> 11) * 0x1.0p-53;
}

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
    const double r = sqrt(-2.0 * log(u1));
    double s, c;
#ifdef __CUDA_ARCH__
    sincospi(2.0 * u2, &s, &c);  // as stream_normals below
#else
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
template <int K, bool ROLL = false>
PF_HD void stream_normals(uint64_t seed, uint64_t j, uint64_t n, uint64_t purpose,
                          double (&out)[K]) {
  constexpr int kPairs = (K + 1) / 2;
  constexpr int kBlocks = (2 * kPairs + 3) / 4;
  uint64_t w[kBlocks * 4];
#pragma unroll
  for (int b = 0; b < kBlocks; ++b) {
    const U64x4 blk = philox4x64<ROLL>(static_cast<uint64_t>(b), j, n, purpose, seed, kKeyConstant);
#pragma unroll
    for (int l = 0; l < 4; ++l) w[4 * b + l] = blk.v[l];
  }
#pragma unroll
  for (int q = 0; q < kPairs; ++q) {
    const double u1 = (static_cast<double>(w[2 * q] >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = u64_to_uniform(w[2 * q + 1]);
    const double r = sqrt(-2.0 * log(u1));
    double s, c;
#ifdef __CUDA_ARCH__
    // sin/cos(2 pi u2) without the range reduction (2 u2 is exact); differs
    // from sin(fl(2 pi u2)) by the rounding of the product, <= 4.4e-16 absolute
    sincospi(2.0 * u2, &s, &c);
#else
    const double angle = 2.0 * 3.14159265358979323846 * u2;
    s = sin(angle);
    c = cos(angle);
#endif
    out[2 * q] = r * c;
    if (2 * q + 1 < K) out[2 * q + 1] = r * s;
  }
}

// stream_normals written to a strided buffer (out[k * stride]), the Philox
// blocks and the Box-Muller pairs as a loop: one instance of the
// transcendental code instead of one per pair (kernels whose instruction
// footprint matters; the buffer is a shared-memory column). Same values.
#ifdef __CUDACC__
template <int K>
__device__ __forceinline__ void stream_normals_strided(uint64_t seed, uint64_t j, uint64_t n, uint64_t purpose,
                                                       double* out, int stride) {
  constexpr int kPairs = (K + 1) / 2;
  constexpr int kBlocks = (2 * kPairs + 3) / 4;
#pragma unroll 1
  for (int b = 0; b < kBlocks; ++b) {
    const U64x4 blk = philox4x64<true>(static_cast<uint64_t>(b), j, n, purpose, seed, kKeyConstant);
#pragma unroll 1
    for (int l = 0; l < 2; ++l) {
      const int q = 2 * b + l;
      if (q >= kPairs) break;
      const uint64_t w1 = l ? blk.v[2] : blk.v[0], w2 = l ? blk.v[3] : blk.v[1];
      const double u1 = (static_cast<double>(w1 >> 11) + 1.0) * 0x1.0p-53;
      const double u2 = u64_to_uniform(w2);
      const double r = sqrt(-2.0 * log(u1));
      double sn, cs;
      sincospi(2.0 * u2, &sn, &cs);
      out[(2 * q) * stride] = r * cs;
      if (2 * q + 1 < K) out[(2 * q + 1) * stride] = r * sn;
    }
  }
}
#endif

// The resampling uniform of slot n at time j (filter.cpp:171-172).
PF_HD double resample_uniform(uint64_t seed, uint64_t j, uint64_t n) {
  return u64_to_uniform(philox4x64(0, j, n, kResample, seed, kKeyConstant).v[0]);
}

PFSMC_END  // namespace pfsmc_gpu::PFSMC_VNS
