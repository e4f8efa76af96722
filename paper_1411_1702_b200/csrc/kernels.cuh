// Device side shared by every kernel translation unit (one arithmetic
// variant per build, variant.cuh): the templated K1 (k_predict), K3
// (k_update), moments / init kernels, the ancestor search, and the KernelSet
// implementation the host driver dispatches through (types.cuh).
#pragma once
#include "types.cuh"
#include "exact_cdf.cuh"
#include "lmm.cuh"
#include "reduce.cuh"

PFSMC_BEGIN

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}


// ---------------------------------------------------------------- helpers
template <class M>
__device__ __forceinline__ void load_record(const double* __restrict__ rec, int R, long long n,
                                            double (&x)[M::D], double (&th)[M::P]) {
  const double2* p = reinterpret_cast<const double2*>(rec + n * R);
  double v[M::D + M::P + 1];
#pragma unroll
  for (int i = 0; i < (M::D + M::P + 1) / 2; ++i) {
    const double2 q = __ldg(p + i);
    v[2 * i] = q.x;
    v[2 * i + 1] = q.y;
  }
#pragma unroll
  for (int i = 0; i < M::D; ++i) x[i] = v[i];
#pragma unroll
  for (int i = 0; i < M::P; ++i) th[i] = v[M::D + i];
}

template <class M>
__device__ __forceinline__ void store_record(double* __restrict__ rec, int R, long long n,
                                             const double (&x)[M::D], const double (&th)[M::P]) {
  double2* p = reinterpret_cast<double2*>(rec + n * R);
  double v[M::D + M::P + 1];
#pragma unroll
  for (int i = 0; i < M::D; ++i) v[i] = x[i];
#pragma unroll
  for (int i = 0; i < M::P; ++i) v[M::D + i] = th[i];
  v[M::D + M::P] = 0.0;
#pragma unroll
  for (int i = 0; i < (M::D + M::P + 1) / 2; ++i) p[i] = make_double2(v[2 * i], v[2 * i + 1]);
}

// filter::log_likelihood (filter.cpp:124-141): ll_const - ss / (2 s2);
// lognormal extension: (ll_const' - ss/(2 s2)) with r = log y - log x, -inf for x <= 0.
template <class M>
__device__ __forceinline__ double loglik(const Ctx& c, const StepParams& sp,
                                         const double (&x)[M::D]) {
  // all indices compile-time (no local-memory copies of c / sp)
  double ss = 0.0;
  const bool lognormal = c.likelihood == PFSMC_GPU_LIK_LOGNORMAL;
  bool dead = false;
#pragma unroll
  for (int k = 0; k < kMaxObs; ++k) {
    if (k < c.m_y) {
      const int idx = c.obs_idx[k];
      double xv = x[0];
#pragma unroll
      for (int i = 1; i < M::D; ++i) xv = (i == idx) ? x[i] : xv;
      double r;
      if (lognormal) {
        dead |= !(xv > 0.0);
        r = sp.y[k] - log(xv);
      } else {
        r = sp.y[k] - xv;
      }
      ss += r * r;
    }
  }
  if (lognormal) return dead ? kNegInf : (sp.ll_const - ss / c.two_s2) - sp.sly;
  return sp.ll_const - ss / c.two_s2;
}

// L2 eviction-priority hints (createpolicy + ld/st .L2::cache_hint): the
// ancestor search keeps its small tables (guide, segment ends) resident
// while the one-shot traffic (CDF segments, record gathers) is evicted first.
__device__ __forceinline__ uint64_t l2_policy_keep() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_stream() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double ld_hint(const double* a, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ unsigned ld_hint(const unsigned* a, uint64_t pol) {
  unsigned v;
  asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ double2 ld_hint(const double2* a, uint64_t pol) {
  double2 v;
  asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_hint(double2* a, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" :: "l"(a), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
}

__device__ __forceinline__ bool grid_error(const Ctx& c) {
  return *reinterpret_cast<volatile int*>(&c.st->error) != 0;
}

// Approximate fitness mass per exact-CDF tile, straight from the K1 block
// partials (M_b, S_b = sum exp(lg - M_b)), in two levels so no single block
// walks every partial:
//  * group hook (last block of each 64-block group, before lse is known):
//    trel_t = sum_b S_b exp(M_b - M_g) and the finite count of each tile in
//    the group (a tile is 8 or 16 K1 blocks; groups hold whole tiles);
//  * tile_prefixes (final block): T_t = trel_t exp(M_g - lse), exclusive
//    prefix over tiles.
// Only the exact scan's classification reads these, through the rigorous
// bound of exact_cdf.cuh (sum_bound); no pass over the fitness vector and no
// look-back is needed.
__host__ __device__ constexpr int ilog2(int v) { return v <= 1 ? 0 : 1 + ilog2(v >> 1); }

struct TileGroupHook {
  const Ctx* c;
  __device__ void operator()(int g, int gsize) const {
    const int bpt_log2 = c->tile_log2 - c->k1_block_log2;  // K1 blocks per tile (<= 32)
    const double mg = __ldcg(&c->gpart[2 * g]);
    const int b0 = g * kGroup;
    double w = 0.0;
    int n = 0;
    if (threadIdx.x < gsize) {
      const int b = b0 + threadIdx.x;
      const double mb = __ldcg(&c->part[2 * b]);
      if (mb != -INFINITY) w = __ldcg(&c->part[2 * b + 1]) * exp(mb - mg);
      n = __ldcg(&c->blk_cnt[b]);
    }
    // fixed-order sums over the bpt lanes of each tile (butterfly inside aligned lane groups)
    for (int o = 1; o < (1 << bpt_log2); o <<= 1) {
      w += __shfl_xor_sync(0xffffffffu, w, o);
      n += __shfl_xor_sync(0xffffffffu, n, o);
    }
    if (threadIdx.x < gsize && (threadIdx.x & ((1 << bpt_log2) - 1)) == 0) {
      const int t = (b0 + threadIdx.x) >> bpt_log2;
      c->trel[t] = w;
      c->tile_cnt_pre[t] = n;  // per-tile count; tile_prefixes turns it into the prefix
    }
  }
};

// tile_m (C5 path): per-tile maxima instead of the group maxima. NT: the
// calling kernel's block size; the groups are kGroup K1 blocks of
// 2^k1_block_log2 particles.
template <int NT = kThreads>
__device__ __forceinline__ void tile_prefixes(const Ctx& c, double lse, const double* tile_m = nullptr) {
  __shared__ SumCnt sw[2 * (NT / 32)];
  const int tpg_log2 = 6 - (c.tile_log2 - c.k1_block_log2);  // tiles per group
  const int per = (c.ntiles + NT - 1) / NT;
  const int t0 = threadIdx.x * per, t1 = min(t0 + per, c.ntiles);
  double s[8];
  long long n[8];
  SumCnt acc{0.0, 0};
  for (int t = t0; t < t1; ++t) {
    const double mg = tile_m ? __ldcg(&tile_m[t]) : __ldcg(&c.gpart[2 * (t >> tpg_log2)]);
    const double v = mg == -INFINITY ? 0.0 : __ldcg(&c.trel[t]) * exp(mg - lse);
    const long long k = __ldcg(&c.tile_cnt_pre[t]);
    if (t - t0 < 8) {
      s[t - t0] = v;
      n[t - t0] = k;
    }
    acc.s += v;
    acc.c += k;
  }
  SumCnt tot;
  SumCnt ex = block_excl_scan_sc<NT>(acc, tot, sw);
  for (int t = t0; t < t1; ++t) {
    double v;
    long long k;
    if (t - t0 < 8) {
      v = s[t - t0];
      k = n[t - t0];
    } else {
      const double mg = tile_m ? __ldcg(&tile_m[t]) : __ldcg(&c.gpart[2 * (t >> tpg_log2)]);
      v = mg == -INFINITY ? 0.0 : __ldcg(&c.trel[t]) * exp(mg - lse);
      k = __ldcg(&c.tile_cnt_pre[t]);
    }
    c.tile_pre[t] = ex.s;
    c.tile_cnt_pre[t] = ex.c;
    ex.s += v;
    ex.c += k;
  }
  if (threadIdx.x == NT - 1) {
    c.shard_sum[0] = tot.s;
    c.shard_sum[1] = static_cast<double>(tot.c);
  }
}

// ---------------------------------------------------------------- K1
// CTAs per SM the model's K1 / K3 are built for (launch bounds)
// (measured per model at 256 threads, scaled to the model's CTA size; the
// shared-memory-history chain: 3 CTAs of 128)
template <class M>
constexpr int k1_min_blocks() {
  return MinBlocksOf<M>::k1 ? MinBlocksOf<M>::k1
                            : (M::ID == 5 ? 2 : M::D <= 2 ? 6 : M::D <= 3 ? 4 : 1) * (kThreads / BlockOf<M>::value);
}
template <class M>
constexpr int k3_min_blocks() {
  return MinBlocksOf<M>::k3 ? MinBlocksOf<M>::k3
                            : (M::ID == 5 ? 2 : M::D <= 2 ? 4 : M::D <= 3 ? 3 : 1) * (kThreads / BlockOf<M>::value);
}
// Dynamic shared memory of a K1 / K3 CTA: the LMM history columns.
// (+ P + D doubles per thread: the K3 proliferation / innovation normals)
template <class M, int FAM, int ORD>
constexpr int hist_smem_bytes() {
  using Pr = Propagator<M, FAM, ORD>;
  return Pr::kSmemHist ? (Pr::kHistDoubles + M::P + M::D) * BlockOf<M>::value * static_cast<int>(sizeof(double))
                       : 0;
}

template <class M, int FAM, int ORD>
__global__ void __launch_bounds__(BlockOf<M>::value, k1_min_blocks<M>()) k_predict(Ctx c) {
  constexpr int D = M::D, P = M::P;
  constexpr int KT = BlockOf<M>::value;
  __shared__ double scratch[KT / 32 * 2];
  __shared__ double fin[2];
  extern __shared__ double hist_smem[];
  if (grid_error(c)) return;
  const StepParams& sp = *c.sp;  // read fields in place (no local copy)
  const DevState& st = *c.st;
  const long long n = static_cast<long long>(blockIdx.x) * KT + threadIdx.x;
  double lgv = kNegInf;
  int iters = 0;
  if (n < c.N) {
    double x[D], tu[P], th[P], gamma[D];
    load_record<M>(c.rec[st.cur], c.R, n, x, tu);
    const double logw = c.lw[n] - st.lse_w;
    // shrink (filter.cpp:118) + natural_params (models.cpp:18-25)
#pragma unroll
    for (int k = 0; k < P; ++k) th[k] = exp(c.a * tu[k] + c.one_minus_a * st.mu[k]);
    Propagator<M, FAM, ORD> prop;
    prop.mk = M::load_k(c.mconst);
    prop.bind_history(hist_smem + threadIdx.x);
    int status;
    if constexpr (ORD == 0)
      status = prop.run_adaptive(th, x, sp.t_prev, sp.t_obs, c.rtol, c.tol, c.max_iter, gamma, iters);
    else
      status = prop.run(th, x, sp.t_prev, sp.h, sp.m, c.tol, c.max_iter, gamma, iters);
    const double ll = status == kOk ? loglik<M>(c, sp, x) : kNegInf;
    c.llbar[n] = ll;
    lgv = logw + ll;
    c.lg[n] = lgv;
  }
  if (FAM != kAB) {
    int it = iters;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) it += __shfl_xor_sync(0xffffffffu, it, o);
    if ((threadIdx.x & 31) == 0 && it) atomicAdd(&c.st->newton_iters, static_cast<unsigned long long>(it));
  }
  const double one[1] = {1.0};
  const int nfin = __syncthreads_count(isfinite(lgv) != 0);
  if (threadIdx.x == 0) c.blk_cnt[blockIdx.x] = nfin;
  block_partial<1, false, KT>(lgv, one, c.part + blockIdx.x * 2, scratch);
  if (tree_reduce_last<1, false, TileGroupHook, KT>(c.part, c.gpart, c.cnt_pred, fin, scratch, !c.sharded,
                                                     TileGroupHook{&c})) {
    __shared__ double s_lse;
    if (threadIdx.x == 0) {
      // logsumexp (filter.cpp:16-23) + the degeneracy check (filter.cpp:149-152)
      const double mx = fin[0];
      const double lse = isfinite(mx) ? mx + log(fin[1]) : kNegInf;
      c.st->lse_g = lse;
      if (!isfinite(lse)) atomicOr(&c.st->error, kErrPredict);
      s_lse = lse;
    }
    __syncthreads();
    if (isfinite(s_lse)) tile_prefixes<KT>(c, s_lse);
  }
}

// Ancestor search: first k with cdf_k > u (std::upper_bound, filter.cpp:173),
// clamped to N-1 (filter.cpp:175), in two parts:
//  find_segment: guide bucket -> segment bracket [lo, hi] (guide entries and
//    segment ends are L2-resident) -> binary search / walk over seg_end ->
//    the segment whose end first exceeds u;
//  the count of CDF values <= u inside that aligned segment (the CDF is
//    non-decreasing, so the count is the offset of the first value above u).
__device__ __forceinline__ long long find_segment(const Ctx& c, double u) {
  const uint64_t keep = l2_policy_keep();
  constexpr int seg_log2 = kSegLog2;
  const long long nseg = (static_cast<long long>(c.N) + (1 << seg_log2) - 1) >> seg_log2;
  const long long nb = 1LL << c.coarse_bits;
  long long b = static_cast<long long>(scale2(u, c.coarse_bits));
  b = min(max(b, 0LL), nb - 1);
  long long lo = ld_hint(&c.coarse[b], keep);
  long long hi = nseg - 1;
  if (b + 1 < nb) {
    // the next bucket belongs to this handle only if its edge is below our end
    const double edge = scale2(static_cast<double>(b + 1), -c.coarse_bits);
    if (edge < __ldg(&c.tile_info[c.ntiles - 1]).y) hi = min(hi, static_cast<long long>(ld_hint(&c.coarse[b + 1], keep)));
  }
  lo = min(lo, hi);
  while (hi - lo > 4) {
    const long long mid = (lo + hi) >> 1;
    if (ld_hint(&c.seg_end[mid], keep) > u)
      hi = mid;
    else
      lo = mid + 1;
  }
  while (lo < hi && ld_hint(&c.seg_end[lo], keep) <= u) ++lo;
  return lo;
}

// The search tables of one shard, possibly on a peer GPU (NVLink peer memory).
struct SearchView {
  const unsigned* coarse;
  const double* seg_end;
  const double* cdf;
  double end;  // the shard's exact CDF end (its last tile's end)
};

// The rank whose exact-CDF range [start_r, end_r) holds u (sharded filter;
// gtile_info holds every rank's tiles' exact (start, end)).
__device__ __forceinline__ int serving_rank(const Ctx& c, double u) {
  const int ntl = c.ntiles;
  for (int r = 0; r < c.world; ++r) {
    const double lo = c.gtile_info[r * ntl].x;
    const double hi = c.gtile_info[(r + 1) * ntl - 1].y;
    if (u >= lo && u < hi) return r;
  }
  return c.world - 1;  // unreachable: the last range ends at the guarded cdf >= 1 > u
}

// find_segment + the segment count over an explicit view (scalar form).
__device__ __forceinline__ unsigned find_ancestor_view(const Ctx& c, const SearchView& v, double u) {
  constexpr int seg_log2 = kSegLog2;
  const long long nseg = (static_cast<long long>(c.N) + (1 << seg_log2) - 1) >> seg_log2;
  const long long nb = 1LL << c.coarse_bits;
  long long b = static_cast<long long>(scale2(u, c.coarse_bits));
  b = min(max(b, 0LL), nb - 1);
  long long lo = __ldcg(&v.coarse[b]);
  long long hi = nseg - 1;
  if (b + 1 < nb) {
    const double edge = scale2(static_cast<double>(b + 1), -c.coarse_bits);
    if (edge < v.end) hi = min(hi, static_cast<long long>(__ldcg(&v.coarse[b + 1])));
  }
  lo = min(lo, hi);
  while (hi - lo > 4) {
    const long long mid = (lo + hi) >> 1;
    if (__ldcg(&v.seg_end[mid]) > u)
      hi = mid;
    else
      lo = mid + 1;
  }
  while (lo < hi && __ldcg(&v.seg_end[lo]) <= u) ++lo;
  const long long k0 = lo << seg_log2;
  const long long k1 = min(k0 + (1LL << seg_log2), static_cast<long long>(c.N));
  int cnt = 0;
  for (long long k = k0; k < k1; ++k) cnt += __ldcg(&v.cdf[k]) <= u;
  return static_cast<unsigned>(min(k0 + cnt, static_cast<long long>(c.N) - 1));
}

// Warp-cooperative search over per-lane views (each lane's serving shard,
// possibly a peer GPU): the segment bracket per lane as find_ancestor_view,
// then the 64-byte segment counts spread over four lanes per segment as in
// find_ancestor_warp. Every lane must call it (lanes without a slot: u < 0).
__device__ __forceinline__ unsigned find_ancestor_warp_view(const Ctx& c, const SearchView& v, double u) {
  constexpr int SEGL2 = kSegLog2;
  constexpr int P = 1 << (SEGL2 - 1);
  constexpr int S = 32 / P;
  const int lane = threadIdx.x & 31;
  const long long N = c.N;
  long long k0 = 0;
  if (u >= 0.0) {
    const long long nseg = (N + (1 << SEGL2) - 1) >> SEGL2;
    const long long nb = 1LL << c.coarse_bits;
    long long b = static_cast<long long>(scale2(u, c.coarse_bits));
    b = min(max(b, 0LL), nb - 1);
    long long lo = __ldcg(&v.coarse[b]);
    long long hi = nseg - 1;
    if (b + 1 < nb) {
      const double edge = scale2(static_cast<double>(b + 1), -c.coarse_bits);
      if (edge < v.end) hi = min(hi, static_cast<long long>(__ldcg(&v.coarse[b + 1])));
    }
    lo = min(lo, hi);
    while (hi - lo > 4) {
      const long long mid = (lo + hi) >> 1;
      if (__ldcg(&v.seg_end[mid]) > u)
        hi = mid;
      else
        lo = mid + 1;
    }
    while (lo < hi && __ldcg(&v.seg_end[lo]) <= u) ++lo;
    k0 = lo << SEGL2;
  }
  const unsigned long long cdf_bits = reinterpret_cast<unsigned long long>(v.cdf);
  int mine = 0;
#pragma unroll
  for (int q = 0; q < 32; q += S) {
    const int src = q + lane / P;
    const long long ks = __shfl_sync(0xffffffffu, k0, src);
    const double us = __shfl_sync(0xffffffffu, u, src);
    const double* cdf = reinterpret_cast<const double*>(__shfl_sync(0xffffffffu, cdf_bits, src));
    const long long kk = ks + 2 * (lane % P);
    int cnt = 0;
    if (us >= 0.0) {
      if (kk + 1 < N) {
        const double2 w = __ldcg(reinterpret_cast<const double2*>(cdf + kk));
        cnt = (w.x <= us) + (w.y <= us);
      } else if (kk < N) {
        cnt = __ldcg(&cdf[kk]) <= us;
      }
    }
#pragma unroll
    for (int o = P / 2; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    const int got = __shfl_sync(0xffffffffu, cnt, ((lane - q) & (S - 1)) * P);
    if (lane >= q && lane < q + S) mine = got;
  }
  return static_cast<unsigned>(min(k0 + mine, N - 1));
}

// Scalar form (one thread, one slot).
__device__ __forceinline__ unsigned find_ancestor(const Ctx& c, double u) {
  constexpr int seg_log2 = kSegLog2;
  const long long k0 = find_segment(c, u) << seg_log2;
  const long long k1 = min(k0 + (1LL << seg_log2), static_cast<long long>(c.N));
  int cnt = 0;
  for (long long k = k0; k < k1; ++k) cnt += __ldg(&c.cdf[k]) <= u;
  return static_cast<unsigned>(min(k0 + cnt, static_cast<long long>(c.N) - 1));
}

// Warp-cooperative form: every lane of the warp must call it (lanes without
// a slot pass u = -1). The segment reads are spread so that each load
// instruction covers whole 64-byte segments (four lanes each), i.e. one L1
// wavefront per segment instead of one per lane and per 16 bytes. The CDF
// segments are read evict-first (slot order: one-shot random reads) unless
// the caller searches value-bucketed uniforms (LOCAL: neighbouring lanes and
// warps read the same segments, so they stay cached).
template <bool LOCAL = false>
__device__ __forceinline__ unsigned find_ancestor_warp(const Ctx& c, double u) {
  constexpr int SEGL2 = kSegLog2;
  constexpr int P = 1 << (SEGL2 - 1);  // lanes per segment (16-byte parts)
  constexpr int S = 32 / P;            // segments per load instruction
  const int lane = threadIdx.x & 31;
  const long long N = c.N;
  const long long k0 = u >= 0.0 ? (find_segment(c, u) << SEGL2) : 0;
  int mine = 0;
#pragma unroll
  for (int q = 0; q < 32; q += S) {
    const int src = q + lane / P;
    const long long ks = __shfl_sync(0xffffffffu, k0, src);
    const double us = __shfl_sync(0xffffffffu, u, src);
    const long long kk = ks + 2 * (lane % P);
    int cnt = 0;
    if (kk + 1 < N) {
      const double2 v = LOCAL ? __ldg(reinterpret_cast<const double2*>(c.cdf + kk))
                              : ld_hint(reinterpret_cast<const double2*>(c.cdf + kk), l2_policy_stream());
      cnt = (v.x <= us) + (v.y <= us);
    } else if (kk < N) {
      cnt = __ldg(&c.cdf[kk]) <= us;
    }
#pragma unroll
    for (int o = P / 2; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    const int got = __shfl_sync(0xffffffffu, cnt, ((lane - q) & (S - 1)) * P);
    if (lane >= q && lane < q + S) mine = got;
  }
  return static_cast<unsigned>(min(k0 + mine, N - 1));
}

// ---------------------------------------------------------------- K3
template <class M>
struct MomentLayout {
  static constexpr int P = M::P, D = M::D;
  static constexpr int NA = P, NB = P * (P + 1) / 2, NX = D;
  static constexpr int V = 1 + NA + NB + NX + 1;  // values: S, A, B, X, Q (partial = M + V)
};

// Finalise (M, S, A, B, X, Q) into lse_w, mean, cov, trace, chol for the
// next step; K is the shift the partials were taken about.
template <class M>
__device__ __noinline__ void finalize_moments(const Ctx& c, const double* fin, const double (&K)[M::P],
                                 bool set_lse, bool set_cov) {
  using ML = MomentLayout<M>;
  constexpr int P = M::P, D = M::D;
  DevState& st = *c.st;
  const double Mx = fin[0];
  const double S = fin[1];
  const double lse = isfinite(Mx) ? Mx + log(S) : kNegInf;
  if (set_lse) {
    // update_weights degeneracy check (filter.cpp:215-219)
    if (!isfinite(lse)) {
      atomicOr(&st.error, kErrUpdate);
      return;
    }
    st.lse_w = lse;
  }
  double mu[P], dm[P];
#pragma unroll
  for (int k = 0; k < P; ++k) {
    dm[k] = fin[2 + k] / S;
    mu[k] = K[k] + dm[k];
    st.mu[k] = mu[k];
  }
  if (set_cov) {
    int idx = 0;
#pragma unroll
    for (int r = 0; r < P; ++r)
#pragma unroll
      for (int q = r; q < P; ++q) {
        const double v = fin[2 + ML::NA + idx] / S - dm[r] * dm[q];
        st.cov[r * P + q] = v;
        st.cov[q * P + r] = v;
        ++idx;
      }
  }
  // TraceRow (filter.cpp:379-391)
#pragma unroll
  for (int k = 0; k < P; ++k) st.trace[k] = exp(mu[k]);
#pragma unroll
  for (int k = 0; k < P; ++k) st.trace[P + k] = st.cov[k * P + k];
#pragma unroll
  for (int k = 0; k < D; ++k) st.trace[2 * P + k] = fin[2 + ML::NA + ML::NB + k] / S;
  st.trace[2 * P + D] = S * S / fin[2 + ML::NA + ML::NB + ML::NX];
}

// chol_psd with the jitter ladder (linalg.cpp:439-500), one thread. Same
// operation order as the reference; sqrt and division are IEEE-exact, so L
// is bitwise the reference's for the same C.
template <int P>
__device__ __noinline__ void chol_psd_device(DevState& st) {
  const double* C = st.cov;
  double trace = 0.0;
  for (int i = 0; i < P; ++i) trace += C[i * P + i];
  const double unit = trace / static_cast<double>(P);
  const double au = fabs(unit);
  const double pivot_tol = 1e-14 * ((1.0 < au) ? au : 1.0);
  const double ladder[6] = {0.0, 1e-12, 1e-10, 1e-8, 1e-6, 1e-4};
  for (int r = 0; r < 6; ++r) {
    const double eps = ladder[r] * unit;
    double A[P * P], L[P * P];
    for (int i = 0; i < P * P; ++i) {
      A[i] = C[i];
      L[i] = 0.0;
    }
    if (eps != 0.0)
      for (int i = 0; i < P; ++i) A[i * P + i] += eps;
    bool ok = true;
    for (int i = 0; i < P && ok; ++i) {
      double d = A[i * P + i];
      for (int k = 0; k < i; ++k) d -= L[i * P + k] * L[i * P + k];
      if (d < -pivot_tol) {
        ok = false;
        break;
      }
      if (d <= pivot_tol) {
        for (int j = i + 1; j < P; ++j) {
          double s = A[j * P + i];
          for (int k = 0; k < i; ++k) s -= L[j * P + k] * L[i * P + k];
          if (fabs(s) > pivot_tol) ok = false;
        }
        L[i * P + i] = 0.0;
        continue;
      }
      const double root = sqrt(d);
      L[i * P + i] = root;
      for (int j = i + 1; j < P; ++j) {
        double s = A[j * P + i];
        for (int k = 0; k < i; ++k) s -= L[j * P + k] * L[i * P + k];
        L[j * P + i] = s / root;
      }
    }
    if (ok) {
      for (int i = 0; i < P * P; ++i) st.L[i] = L[i];
      st.jitter = eps;
      st.chol_failed = 0;
      return;
    }
  }
  st.chol_failed = 1;
}

template <class M, int FAM, int ORD>
__global__ void __launch_bounds__(BlockOf<M>::value, k3_min_blocks<M>()) k_update(Ctx c) {
  constexpr int D = M::D, P = M::P;
  constexpr int KT = BlockOf<M>::value;
  using ML = MomentLayout<M>;
  constexpr int V = ML::V;
  __shared__ double scratch[KT / 32 * V];
  __shared__ double fin[V + 1];  // M + V values

  constexpr int kTsc = V <= 12 ? V * KT : 1;
  __shared__ double tsc[kTsc];
  extern __shared__ double hist_smem[];
  if (grid_error(c)) return;
  DevState& st = *c.st;
  if (st.chol_failed) {
    // proliferate's chol_psd throws (linalg.cpp:499) after the resample phase
    if (threadIdx.x == 0) atomicOr(&st.error, kErrChol);
    return;
  }
  // the shrink mean and chol(C) of the previous step: every thread reads the
  // same few words (L1 broadcast), no block barrier before the work starts;
  // only the last block rewrites them, after every block's reads
  const double* sL = st.L;
  const double* sK = st.mu;
  const StepParams& sp = *c.sp;  // read fields in place (no local copy)
  const int cur = st.cur;
  const long long n = static_cast<long long>(blockIdx.x) * KT + threadIdx.x;
  double lwv = kNegInf;
  double vals[V];  // moment leaf
#pragma unroll
  for (int k = 0; k < V; ++k) vals[k] = 0.0;
  int iters = 0;
  if (n < c.N) {
    // survival of the fittest (filter.cpp:169-176): the ancestor's record and
    // ll_bar were gathered into slot order by k_serve (coalesced read here)
    // xr: the ancestor's state, propagated in place (on failure it is read
    // again rather than kept live through the propagation)
    double xr[D], tu[P], tb[P], th[P], gamma[D];
    load_record<M>(c.payload, c.R + 2, n, xr, tu);
    const double llb = __ldg(&c.payload[n * (c.R + 2) + c.R]);
    // shrink of the ancestor (filter.cpp:118), proliferation (filter.cpp:185-196)
    double z[P];
    // large models (d >= 6): Philox rounds as a loop (code size, not speed)
    constexpr bool kRoll = D >= 6;
    using Pr = Propagator<M, FAM, ORD>;
    // shared-memory-history models: both normal sets drawn up front into a
    // shared-memory column (one instance of the Box-Muller code, nothing live
    // in registers through the propagation)
    double* zcol = hist_smem + (Pr::kSmemHist ? Pr::kHistDoubles * KT : 0) + threadIdx.x;
    if constexpr (Pr::kSmemHist) {
      stream_normals_strided<P>(c.seed, sp.j, c.n0 + n, kProliferate, zcol, KT);
      stream_normals_strided<D>(c.seed, sp.j, c.n0 + n, kInnovate, zcol + P * KT, KT);
#pragma unroll
      for (int q = 0; q < P; ++q) z[q] = zcol[q * KT];
    } else {
      stream_normals<P, kRoll>(c.seed, sp.j, c.n0 + n, kProliferate, z);
    }
#pragma unroll
    for (int r = 0; r < P; ++r) {
      tb[r] = c.a * tu[r] + c.one_minus_a * sK[r];
      double dot = 0.0;
#pragma unroll
      for (int q = 0; q <= r; ++q) dot += sL[r * P + q] * z[q];
      tb[r] += c.s_prolif * dot;
      th[r] = exp(tb[r]);
    }
    // repropagate + innovate + log-lik (filter.cpp:351-365)
    Propagator<M, FAM, ORD> prop;
    prop.mk = M::load_k(c.mconst);
    prop.bind_history(hist_smem + threadIdx.x);
    int status;
    if constexpr (ORD == 0)
      status = prop.run_adaptive(th, xr, sp.t_prev, sp.t_obs, c.rtol, c.tol, c.max_iter, gamma, iters);
    else
      status = prop.run(th, xr, sp.t_prev, sp.h, sp.m, c.tol, c.max_iter, gamma, iters);
    double ll = kNegInf;
    if (status == kOk) {
      double zi[D];
      if constexpr (Pr::kSmemHist) {
#pragma unroll
        for (int k = 0; k < D; ++k) zi[k] = zcol[(P + k) * KT];
      } else {
        stream_normals<D, kRoll>(c.seed, sp.j, c.n0 + n, kInnovate, zi);
      }
#pragma unroll
      for (int k = 0; k < D; ++k) xr[k] += sqrt(gamma[k]) * zi[k];
      ll = loglik<M>(c, sp, xr);
    } else {
      load_record<M>(c.payload, c.R + 2, n, xr, tu);  // the particle keeps its state
    }
    lwv = ll - llb;  // update_weights (filter.cpp:214)
    store_record<M>(c.rec[cur ^ 1], c.R, n, xr, tb);
    c.lw[n] = lwv;
    // moment leaf: theta about K, outer product, state, ESS
    double dv[P];
#pragma unroll
    for (int k = 0; k < P; ++k) dv[k] = tb[k] - sK[k];
    vals[0] = 1.0;
#pragma unroll
    for (int k = 0; k < P; ++k) vals[1 + k] = dv[k];
    int idx = 0;
#pragma unroll
    for (int r = 0; r < P; ++r)
#pragma unroll
      for (int q = r; q < P; ++q) vals[1 + ML::NA + idx++] = dv[r] * dv[q];
#pragma unroll
    for (int k = 0; k < D; ++k) vals[1 + ML::NA + ML::NB + k] = xr[k];
    vals[V - 1] = 1.0;
  }
  if (FAM != kAB) {
    int it = iters;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) it += __shfl_xor_sync(0xffffffffu, it, o);
    if ((threadIdx.x & 31) == 0 && it) atomicAdd(&st.newton_iters, static_cast<unsigned long long>(it));
  }
  block_partial<V, true, KT>(lwv, vals, c.part + static_cast<size_t>(blockIdx.x) * (V + 1), scratch,
                             V <= 12 ? tsc : nullptr);
  if (tree_reduce_last<V, true, NoGroupHook, KT>(c.part, c.gpart, c.cnt_upd, fin, scratch, !c.sharded)) {
    if (threadIdx.x == 0) {
      double K[P];
#pragma unroll
      for (int k = 0; k < P; ++k) K[k] = sK[k];
      finalize_moments<M>(c, fin, K, true, true);
      if (!(st.error & kErrUpdate)) {
        chol_psd_device<P>(st);
        st.cur = cur ^ 1;
      }
    }
  }
}

// Moments of the resident ensemble (after injection / initialisation):
// refreshes the shrink mean (and, for init, cov + chol); lse_w untouched.
template <class M>
__global__ void __launch_bounds__(BlockOf<M>::value) k_moments(Ctx c, int set_cov) {
  constexpr int D = M::D, P = M::P;
  constexpr int KT = BlockOf<M>::value;  // the partial layout of k_update
  using ML = MomentLayout<M>;
  constexpr int V = ML::V;
  __shared__ double scratch[KT / 32 * V];
  __shared__ double fin[V + 1];  // M + V values
  DevState& st = *c.st;
  const long long n = static_cast<long long>(blockIdx.x) * KT + threadIdx.x;
  double lwv = kNegInf;
  double vals[V];
#pragma unroll
  for (int k = 0; k < V; ++k) vals[k] = 0.0;
  double K[P];
#pragma unroll
  for (int k = 0; k < P; ++k) K[k] = st.mu[k];  // shift: caller-provided guess
  if (n < c.N) {
    double x[D], tu[P];
    load_record<M>(c.rec[st.cur], c.R, n, x, tu);
    lwv = c.lw[n] - st.lse_w;
    vals[0] = 1.0;
#pragma unroll
    for (int k = 0; k < P; ++k) vals[1 + k] = tu[k] - K[k];
    int idx = 0;
#pragma unroll
    for (int r = 0; r < P; ++r)
#pragma unroll
      for (int q = r; q < P; ++q) vals[1 + ML::NA + idx++] = (tu[r] - K[r]) * (tu[q] - K[q]);
#pragma unroll
    for (int k = 0; k < D; ++k) vals[1 + ML::NA + ML::NB + k] = x[k];
    vals[V - 1] = 1.0;
  }
  block_partial<V, true, KT>(lwv, vals, c.part + static_cast<size_t>(blockIdx.x) * (V + 1), scratch);
  if (tree_reduce_last<V, true, NoGroupHook, KT>(c.part, c.gpart, c.cnt_upd, fin, scratch, !c.sharded)) {
    if (threadIdx.x == 0) {
      finalize_moments<M>(c, fin, K, false, set_cov != 0);
      chol_psd_device<P>(st);
    }
  }
}

// Sharded finishers: the same final combine as the single-handle tree
// (combine_partials over the group partials in global order), over the
// allgathered group partials of every shard => bitwise identical results.
// flags: 1 = set lse_w (+ degeneracy check), 2 = set cov, 4 = chol + flip the
// record buffer (a completed step); 0/2 are the injection / init refreshes.
template <class M>
__global__ void __launch_bounds__(kThreads) k_finish_moments(Ctx c, const double* gp, int ngroups,
                                                             int flags) {
  constexpr int P = M::P;
  constexpr int V = MomentLayout<M>::V;
  __shared__ double scratch[kWarps * V];
  __shared__ double fin[V + 1];
  if (grid_error(c)) return;
  DevState& st = *c.st;
  double K[P];
#pragma unroll
  for (int k = 0; k < P; ++k) K[k] = st.mu[k];
  __syncthreads();
  // the single handle's final level (tree_reduce_last): one warp, same order
  if (threadIdx.x < 32) combine_partials_warp<V, true>(gp, ngroups, fin);
  __syncthreads();
  if (threadIdx.x == 0) {
    finalize_moments<M>(c, fin, K, (flags & 1) != 0, (flags & 2) != 0);
    if (!(st.error & kErrUpdate)) {
      chol_psd_device<P>(st);
      if (flags & 4) st.cur ^= 1;
    }
  }
}

template <int P>
__global__ void k_chol(DevState* st) {
  if (threadIdx.x == 0 && blockIdx.x == 0) chol_psd_device<P>(*st);
}

// Initialisation: stream (seed, 0, i, init), theta then x (filter.cpp:87-100).
template <class M>
__global__ void __launch_bounds__(kThreads) k_init(Ctx c, int kind, const double* prm, double lw0) {
  constexpr int D = M::D, P = M::P;
  const long long n = static_cast<long long>(blockIdx.x) * kThreads + threadIdx.x;
  if (n >= c.N) return;
  // prm: gaussian: th_mu[P], th_sigma[P], x_mean[D], x_std[D], x_clamp[D]
  //      uniform : th_lo[P], th_hi[P], x_lo[D], x_hi[D]
  Stream s(c.seed, 0, c.n0 + n, kInit);
  double x[D], tu[P];
  if (kind == 0) {
#pragma unroll
    for (int k = 0; k < P; ++k) tu[k] = prm[k] + prm[P + k] * s.next_normal();
#pragma unroll
    for (int k = 0; k < D; ++k) {
      double v = prm[2 * P + k] + prm[2 * P + D + k] * s.next_normal();
      if (prm[2 * P + 2 * D + k] != 0.0 && v < 0.0) v = 0.0;
      x[k] = v;
    }
  } else {
#pragma unroll
    for (int k = 0; k < P; ++k) tu[k] = log(prm[k] + (prm[P + k] - prm[k]) * s.next_uniform());
#pragma unroll
    for (int k = 0; k < D; ++k) x[k] = prm[2 * P + k] + (prm[2 * P + D + k] - prm[2 * P + k]) * s.next_uniform();
  }
  store_record<M>(c.rec[c.st->cur], c.R, n, x, tu);
  c.lw[n] = lw0;
}

// ---------------------------------------------------------------- host side
// One noise-free truth trajectory (the data generator's reference_observations,
// bench.cpp:296-317): adaptive BDF(1,2) at rtol from x0 through every
// observation time, one thread. prm = model constants[8], theta_nat[P], x0[D];
// out = T x D states; status[0] = first non-ok particle status (0 if none).
template <class M>
__global__ void k_trajectory(const double* prm, const double* times, int T, double t0, double rtol,
                             double tol, int max_iter, double* out, int* status) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  Propagator<M, kBDF, 0> prop;
  prop.mk = M::load_k(prm);
  double th[M::P], x[M::D], gamma[M::D];
#pragma unroll
  for (int k = 0; k < M::P; ++k) th[k] = prm[8 + k];
#pragma unroll
  for (int k = 0; k < M::D; ++k) x[k] = prm[8 + M::P + k];
  double tp = t0;
  int iters = 0;
  status[0] = 0;
  for (int r = 0; r < T; ++r) {
    const int st = prop.run_adaptive(th, x, tp, times[r], rtol, tol, max_iter, gamma, iters);
    if (st != kOk) {
      status[0] = st;
      return;
    }
#pragma unroll
    for (int k = 0; k < M::D; ++k) out[static_cast<long long>(r) * M::D + k] = x[k];
    tp = times[r];
  }
}

template <class M, int FAM, int ORD>
struct KernelSetT final : KernelSet {
  static constexpr int KT = BlockOf<M>::value;
  static constexpr int kHist = hist_smem_bytes<M, FAM, ORD>();
  int attr_device = -1;  // the device whose kernels got the dynamic-smem attribute
  KernelSetT() {
    d = M::D;
    p = M::P;
    kt = KT;
  }
  void set_attributes() {
    if constexpr (kHist > 0) {
      int dev = 0;
      cudaGetDevice(&dev);
      if (dev == attr_device) return;
      cudaFuncSetAttribute(k_predict<M, FAM, ORD>, cudaFuncAttributeMaxDynamicSharedMemorySize, kHist);
      cudaFuncSetAttribute(k_update<M, FAM, ORD>, cudaFuncAttributeMaxDynamicSharedMemorySize, kHist);
      attr_device = dev;
    }
  }
  void trajectory(const double* prm, const double* times, int T, double t0, double rtol, double tol,
                  int max_iter, double* out, int* status, cudaStream_t s) override {
    k_trajectory<M><<<1, 32, 0, s>>>(prm, times, T, t0, rtol, tol, max_iter, out, status);
  }
  void predict(const Ctx& c, int grid, cudaStream_t s) override {
    set_attributes();
    k_predict<M, FAM, ORD><<<grid, KT, kHist, s>>>(c);
  }
  void update(const Ctx& c, int grid, cudaStream_t s) override {
    set_attributes();
    k_update<M, FAM, ORD><<<grid, KT, kHist, s>>>(c);
  }
  void moments(const Ctx& c, int grid, cudaStream_t s, int set_cov) override {
    k_moments<M><<<grid, KT, 0, s>>>(c, set_cov);
  }
  void chol(const Ctx& c, cudaStream_t s) override { k_chol<M::P><<<1, 32, 0, s>>>(c.st); }
  void init(const Ctx& c, int grid, cudaStream_t s, int kind, const double* prm, double lw0) override {
    k_init<M><<<grid, kThreads, 0, s>>>(c, kind, prm, lw0);
  }
  void finish_moments(const Ctx& c, const double* gp, int ngroups, int flags, cudaStream_t s) override {
    k_finish_moments<M><<<1, kThreads, 0, s>>>(c, gp, ngroups, flags);
  }
  int moment_width() const override { return MomentLayout<M>::V + 1; }
};

template <class M, int FAM>
std::unique_ptr<KernelSet> make_order(int order) {
  if constexpr (FAM == kBDF)
    if (order == 0) return std::make_unique<KernelSetT<M, FAM, 0>>();  // adaptive BDF(1,2)
  switch (order) {
    case 1: return std::make_unique<KernelSetT<M, FAM, 1>>();
    case 2: return std::make_unique<KernelSetT<M, FAM, 2>>();
    case 3: return std::make_unique<KernelSetT<M, FAM, 3>>();
  }
  return nullptr;
}
template <class M>
std::unique_ptr<KernelSet> make_family(int fam, int order) {
  switch (fam) {
    case kAB: return make_order<M, kAB>(order);
    case kAM: return make_order<M, kAM>(order);
    case kBDF: return make_order<M, kBDF>(order);
  }
  return nullptr;
}
PFSMC_END  // namespace pfsmc_gpu::PFSMC_VNS
// The per-model entry point of the variant being compiled (types.cuh).
#if PFSMC_FAST
#define PFSMC_ENTRY(name) make_kernels_##name##_fast
#else
#define PFSMC_ENTRY(name) make_kernels_##name
#endif
