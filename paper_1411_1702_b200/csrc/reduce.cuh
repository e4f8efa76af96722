// Deterministic reductions for the log-sum-exp and weighted-moment epilogues.
//
// A "weighted partial" is (M, v[V]): M the max of the leaf log-weights
// (NaN excluded, as the reference's std::max pass, filter.cpp:18), v the sums
// of leaf quantities weighted by e = exp(x - M); the last value may be
// weighted by e^2 (the ESS sum). NaN leaves poison the sums exactly as a NaN
// poisons the reference's exp-sum (filter.cpp:21). Every tree below has a
// fixed shape, so results are bitwise reproducible run to run; no FP atomics.
//
// Cross-block combination uses the "last block done" pattern in two levels
// (groups of kGroup blocks, then the groups), so no launch is spent on it.
#pragma once
#include "variant.cuh"
#include <cstdint>

PFSMC_BEGIN

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kGroup = 64;

__device__ __forceinline__ double nan_free_max(double a, double b) {
  // operands already NaN-free; (a < b) ? b : a like std::max
  return (a < b) ? b : a;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = nan_free_max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide max (all threads get the result). scratch >= NT / 32 doubles.
// NT: threads per block (kThreads unless a model's kernels use another size).
template <int NT = kThreads>
__device__ __forceinline__ double block_max(double v, double* scratch) {
  v = warp_max(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) scratch[w] = v;
  __syncthreads();
  double r = scratch[0];
#pragma unroll
  for (int i = 1; i < NT / 32; ++i) r = nan_free_max(r, scratch[i]);
  return r;
}

// Block-wide sums of V values; result valid in thread 0. scratch >= NT/32*V.
template <int V, int NT = kThreads>
__device__ __forceinline__ void block_sums(double (&v)[V], double* scratch) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < V; ++k) v[k] = warp_sum(v[k]);
  __syncthreads();
  if (l == 0)
#pragma unroll
    for (int k = 0; k < V; ++k) scratch[w * V + k] = v[k];
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < V; ++k) {
      double s = scratch[k];
      for (int i = 1; i < NT / 32; ++i) s += scratch[i * V + k];
      v[k] = s;
    }
  }
}

// Block-wide sums through a shared-memory transpose (fewer instructions
// than V shuffle trees): each thread stores its V values, then V*NW threads
// each fold 32 entries of one value in order, then V threads fold the NW
// chunk sums in order. Fixed shape => bitwise reproducible. Result in
// thread 0's v[]. tsc >= V * NT doubles (V * NW <= NT).
template <int V, int NT = kThreads>
__device__ __forceinline__ void block_sums_smem(double (&v)[V], double* tsc) {
  constexpr int NW = NT / 32;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < V; ++k) tsc[k * NT + threadIdx.x] = v[k];
  __syncthreads();
  double part = 0.0;
  if (threadIdx.x < V * NW) {
    const int k = threadIdx.x / NW, ch = threadIdx.x % NW;
    const double* src = tsc + k * NT + ch * 32;
#pragma unroll 8
    for (int i = 0; i < 32; ++i) part += src[i];
  }
  __syncthreads();
  if (threadIdx.x < V * NW) tsc[threadIdx.x] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < V; ++k) {
      double s = tsc[k * NW];
      for (int i = 1; i < NW; ++i) s += tsc[k * NW + i];
      v[k] = s;
    }
  }
}

// Leaf -> block partial. x: leaf log-weight; vals: leaf quantities (weighted
// by e = exp(x - M) inside, the last one by e^2 when SQ). Thread 0 writes
// (M, sums[V]) to out[0..V]. tsc: V * kThreads doubles of shared scratch
// (null: shuffle trees, scratch >= kWarps * V).
template <int V, bool SQ, int NT = kThreads>
__device__ __forceinline__ void block_partial(double x, const double (&vals)[V], double* out,
                                              double* scratch, double* tsc = nullptr) {
  const bool is_nan = isnan(x);
  const double leaf_max = is_nan ? -INFINITY : x;
  const double M = block_max<NT>(leaf_max, scratch);
  double e;
  if (is_nan)
    e = NAN;
  else if (x == -INFINITY)
    e = 0.0;
  else
    e = exp(x - M);  // M finite here unless every leaf is -inf (then x==-inf)
  double v[V];
#pragma unroll
  for (int k = 0; k < V; ++k) v[k] = ((SQ && k == V - 1) ? e * e : e) * vals[k];
  if (tsc)
    block_sums_smem<V, NT>(v, tsc);
  else
    block_sums<V, NT>(v, scratch);
  if (threadIdx.x == 0) {
    out[0] = M;
#pragma unroll
    for (int k = 0; k < V; ++k) out[1 + k] = v[k];
  }
}

// Combine `count` partials (stride V+1) into one, by one block, fixed order:
// thread t folds partials t, t+256, ... sequentially (rescaled), then a fixed
// warp/block tree. Result in out[0..V] (thread 0 writes).
template <int V, bool SQ, int NT = kThreads>
__device__ __forceinline__ void combine_partials(const double* in, int count, double* out,
                                                 double* scratch) {
  double m = -INFINITY;
  for (int i = threadIdx.x; i < count; i += NT) m = nan_free_max(m, __ldcg(in + i * (V + 1)));
  const double M = block_max<NT>(m, scratch);
  double v[V];
#pragma unroll
  for (int k = 0; k < V; ++k) v[k] = 0.0;
  for (int i = threadIdx.x; i < count; i += NT) {
    const double mi = __ldcg(in + i * (V + 1));
    const double c = (mi == -INFINITY) ? 0.0 : exp(mi - M);
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const double w = (SQ && k == V - 1) ? c * c : c;
      v[k] += w * __ldcg(in + i * (V + 1) + 1 + k);
    }
  }
  block_sums<V, NT>(v, scratch);
  if (threadIdx.x == 0) {
    out[0] = M;
#pragma unroll
    for (int k = 0; k < V; ++k) out[1 + k] = v[k];
  }
}

// combine_partials by ONE warp (the tree levels below run on the critical
// tail of their kernel: the last block's combine is the only work left on the
// GPU, so fewer barriers and no idle warps shorten the step): lane l folds
// partials l, l + 32, ... in order (rescaled to the common max), then a fixed
// butterfly. Lane 0 writes out[]. Fixed shape => bitwise reproducible.
template <int V, bool SQ>
__device__ __noinline__ void combine_partials_warp(const double* in, int count, double* out) {
  const int lane = threadIdx.x & 31;
  double m = -INFINITY;
  for (int i = lane; i < count; i += 32) m = nan_free_max(m, __ldcg(in + i * (V + 1)));
  const double M = warp_max(m);
  double v[V];
#pragma unroll
  for (int k = 0; k < V; ++k) v[k] = 0.0;
  for (int i = lane; i < count; i += 32) {
    const double mi = __ldcg(in + i * (V + 1));
    const double c = (mi == -INFINITY) ? 0.0 : exp(mi - M);
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const double w = (SQ && k == V - 1) ? c * c : c;
      v[k] += w * __ldcg(in + i * (V + 1) + 1 + k);
    }
  }
#pragma unroll
  for (int k = 0; k < V; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0) {
    out[0] = M;
#pragma unroll
    for (int k = 0; k < V; ++k) out[1 + k] = v[k];
  }
}

// Two-level last-block-done tree. Every block calls this after writing its
// partial at part[blockIdx.x*(V+1)]; returns true in exactly one block (the
// last), where `final_out` holds the grand partial (thread 0 wrote it, and a
// __syncthreads() has been issued). counters: [0..ngroups) group counters,
// [ngroups] the final counter; all reset to 0 by their last user.
struct NoGroupHook {
  __device__ void operator()(int, int) const {}
};

// hook(g, gsize) runs in the last block of group g after its group partial
// is written (all of the group's block partials are visible).
template <int V, bool SQ, class Hook = NoGroupHook, int NT = kThreads>
__device__ __forceinline__ bool tree_reduce_last(double* part, double* group_part,
                                                 unsigned* counters, double* final_out,
                                                 double* scratch, bool final_level = true,
                                                 const Hook& hook = Hook()) {
  __shared__ int s_flag;
  const int nblocks = gridDim.x;
  const int ngroups = (nblocks + kGroup - 1) / kGroup;
  const int g = blockIdx.x / kGroup;
  const int gsize = min(kGroup, nblocks - g * kGroup);
  // the block partial was written by thread 0 only: its arrival is one
  // acquire-release atomic (publishes the partial, and the last arriver
  // acquires everyone's), cheaper than a full fence before a relaxed atomic
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(&counters[g]) : "memory");
    s_flag = (old == static_cast<unsigned>(gsize - 1));
    if (s_flag) counters[g] = 0;
  }
  __syncthreads();
  if (!s_flag) return false;
  __threadfence();
  if (threadIdx.x < 32)
    combine_partials_warp<V, SQ>(part + static_cast<size_t>(g) * kGroup * (V + 1), gsize, group_part + g * (V + 1));
  __syncthreads();
  hook(g, gsize);
  if (!final_level) return false;  // sharded: the group partials are exported
  __threadfence();  // the hook's writes (any thread) and the group partial
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned old = atomicAdd(&counters[ngroups], 1u);
    s_flag = (old == static_cast<unsigned>(ngroups - 1));
    if (s_flag) counters[ngroups] = 0;
  }
  __syncthreads();
  if (!s_flag) return false;
  __threadfence();
  if (threadIdx.x < 32) combine_partials_warp<V, SQ>(group_part, ngroups, final_out);
  __syncthreads();
  return true;
}

// Per-thread running values for a block-wide scan.
struct SumCnt {
  double s;
  long long c;
};

// Block-wide exclusive scan of (sum, count) in a fixed shape: warp shuffle
// scan, warp totals through smem, scanned by warp 0. Approximate sums only
// (the bound in exact_cdf.cuh covers any tree); counts exact.
template <int NT = kThreads>
__device__ __forceinline__ SumCnt block_excl_scan_sc(SumCnt v, SumCnt& total, SumCnt* sw) {
  constexpr int kWarps = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  SumCnt x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double ys = __shfl_up_sync(0xffffffffu, x.s, o);
    const long long yc = __shfl_up_sync(0xffffffffu, x.c, o);
    if (lane >= o) {
      x.s = ys + x.s;
      x.c += yc;
    }
  }
  if (lane == 31) sw[w] = x;
  __syncthreads();
  if (w == 0) {
    SumCnt t = lane < kWarps ? sw[lane] : SumCnt{0.0, 0};
#pragma unroll
    for (int o = 1; o < kWarps; o <<= 1) {
      const double ys = __shfl_up_sync(0xffffffffu, t.s, o);
      const long long yc = __shfl_up_sync(0xffffffffu, t.c, o);
      if (lane >= o) {
        t.s = ys + t.s;
        t.c += yc;
      }
    }
    if (lane < kWarps) sw[kWarps + lane] = t;  // inclusive warp prefixes
  }
  __syncthreads();
  const SumCnt pre = w ? sw[kWarps + w - 1] : SumCnt{0.0, 0};
  total = sw[2 * kWarps - 1];
  const double es = __shfl_up_sync(0xffffffffu, x.s, 1);
  const long long ec = __shfl_up_sync(0xffffffffu, x.c, 1);
  SumCnt ex = lane ? SumCnt{es, ec} : SumCnt{0.0, 0};
  ex.s = pre.s + ex.s;
  ex.c += pre.c;
  __syncthreads();
  return ex;
}

PFSMC_END  // namespace pfsmc_gpu::PFSMC_VNS
