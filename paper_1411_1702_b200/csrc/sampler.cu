// B200-native per-step LMM PF-SMC update: the device kernels, the host step
// driver (CUDA graph per step) and the C ABI declared in include/pfsmc_gpu.h.
//
// One step (reference: filter::pf_step, filter.cpp:292-394) is five launches:
//   K1 k_predict      shrink + Psi + log-lik + fitness lse   (filter.cpp:300-324, 143-156)
//   S1 k_scan_sums    fitness g, per-tile double-double sums  \
//   S2 k_scan_pieces  exact-CDF run/window decomposition,      > exact sequential CDF
//                     last block resolves the serial chain    /  (filter.cpp:158-168)
//   S3 k_scan_cdf     exact CDF + per-tile guide tables
//   K3 k_update       ancestor search + gather + proliferate + Psi + innovate +
//                     reweight + moment partials; last block finalises lse,
//                     (theta_bar, C), trace row and chol_psd for the next step
//                     (filter.cpp:169-222, 338-392; linalg.cpp:389-500)
// Particles live in HBM as fixed-stride records {x[d], theta_u[p]} (16-B
// aligned, double-buffered) plus SoA lw / ll_bar / lg / cdf arrays: streamed
// kernels read records with vector loads and the random ancestor gather
// touches ceil(8R/32) sectors instead of d+p+1.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "kernels.cuh"

namespace pfsmc_gpu {
// ---------------------------------------------------------------- exact CDF
__device__ __forceinline__ double fitness_of(const Ctx& c, long long k, double lse) {
  if (k >= c.N) return 0.0;
  if (c.gin) return c.gin[k];
  return exp(c.lg[k] - lse);  // fitness_weights (filter.cpp:154)
}

// smem layout with one pad double per 16 to keep the per-thread contiguous
// reads conflict-free.
__device__ __forceinline__ int sidx(int e) { return e + (e >> 4); }
constexpr int kSmemTile = kTile + kTile / 16;

__device__ __forceinline__ void load_tile_g(const Ctx& c, int t, double* sg) {
  const double lse = c.st->lse_g;
  const long long base = static_cast<long long>(t) * kTile;
#pragma unroll 4
  for (int i = 0; i < kItems; ++i) {
    const int e = i * kThreads + threadIdx.x;
    sg[sidx(e)] = fitness_of(c, base + e, lse);
  }
  __syncthreads();
}

// Block exclusive scan of (DD, count) pairs: approximate prefix only.
__device__ __forceinline__ void block_excl_scan_dd(DD v, long long cnt, DD& excl, long long& cexcl,
                                                   DD* sdd, long long* scnt) {
  sdd[threadIdx.x] = v;
  scnt[threadIdx.x] = cnt;
  __syncthreads();
  if (threadIdx.x < 32) {
    // warp 0 scans 8 chunks of 32 sequentially in dd (deterministic)
    const int l = threadIdx.x;
    DD run = {0.0, 0.0};
    long long crun = 0;
    for (int chunk = 0; chunk < kThreads / 32; ++chunk) {
      const int i = chunk * 32 + l;
      DD x = sdd[i];
      long long cx = scnt[i];
      // inclusive warp scan (Hillis-Steele)
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        DD y;
        y.hi = __shfl_up_sync(0xffffffffu, x.hi, o);
        y.lo = __shfl_up_sync(0xffffffffu, x.lo, o);
        const long long cy = __shfl_up_sync(0xffffffffu, cx, o);
        if (l >= o) {
          x = dd_add(y, x);
          cx += cy;
        }
      }
      DD ex;
      ex.hi = __shfl_up_sync(0xffffffffu, x.hi, 1);
      ex.lo = __shfl_up_sync(0xffffffffu, x.lo, 1);
      long long cex = __shfl_up_sync(0xffffffffu, cx, 1);
      if (l == 0) {
        ex = {0.0, 0.0};
        cex = 0;
      }
      sdd[i] = dd_add(run, ex);
      scnt[i] = crun + cex;
      DD tot;
      tot.hi = __shfl_sync(0xffffffffu, x.hi, 31);
      tot.lo = __shfl_sync(0xffffffffu, x.lo, 31);
      run = dd_add(run, tot);
      crun += __shfl_sync(0xffffffffu, cx, 31);
    }
  }
  __syncthreads();
  excl = sdd[threadIdx.x];
  cexcl = scnt[threadIdx.x];
  __syncthreads();
}

// S1: per-tile double-double sums + nonzero counts; last block: exclusive
// prefix over tiles.
__global__ void __launch_bounds__(kThreads) k_scan_sums(Ctx c) {
  __shared__ double sg[kSmemTile];
  __shared__ DD sdd[kThreads];
  __shared__ long long scnt[kThreads];
  __shared__ int s_last;
  if (grid_error(c)) return;
  const int t = blockIdx.x;
  load_tile_g(c, t, sg);
  DD s = {0.0, 0.0};
  long long cnt = 0;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const double g = sg[sidx(threadIdx.x * kItems + i)];
    s = dd_add(s, g);
    cnt += (g != 0.0);
  }
  DD ex;
  long long cex;
  block_excl_scan_dd(s, cnt, ex, cex, sdd, scnt);
  if (threadIdx.x == kThreads - 1) {
    c.tile_sum[t] = dd_add(ex, s);
    c.tile_cnt[t] = cex + cnt;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned old = atomicAdd(&c.cnt_scan[0], 1u);
    s_last = (old == gridDim.x - 1);
    if (s_last) c.cnt_scan[0] = 0;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // exclusive prefix over tiles: thread-contiguous chunks, then block scan
  const int per = (c.ntiles + kThreads - 1) / kThreads;
  const int t0 = threadIdx.x * per;
  DD ts = {0.0, 0.0};
  long long tc = 0;
  for (int k = t0; k < min(t0 + per, c.ntiles); ++k) {
    DD v;
    v.hi = __ldcg(&c.tile_sum[k].hi);
    v.lo = __ldcg(&c.tile_sum[k].lo);
    ts = dd_add(ts, v);
    tc += __ldcg(&c.tile_cnt[k]);
  }
  block_excl_scan_dd(ts, tc, ex, cex, sdd, scnt);
  for (int k = t0; k < min(t0 + per, c.ntiles); ++k) {
    c.tile_pre[k] = ex;
    c.tile_cnt_pre[k] = cex;
    DD v;
    v.hi = __ldcg(&c.tile_sum[k].hi);
    v.lo = __ldcg(&c.tile_sum[k].lo);
    ex = dd_add(ex, v);
    cex += __ldcg(&c.tile_cnt[k]);
  }
}

// Block-wide exclusive segmented scan of Piece (Hillis-Steele, fixed shape).
__device__ __forceinline__ Piece block_excl_scan_piece(Piece v, Piece* sp) {
  sp[threadIdx.x] = v;
  __syncthreads();
  for (int o = 1; o < kThreads; o <<= 1) {
    Piece mine = sp[threadIdx.x];
    Piece left = threadIdx.x >= o ? sp[threadIdx.x - o] : piece_identity();
    __syncthreads();
    if (threadIdx.x >= o) sp[threadIdx.x] = piece_combine(left, mine);
    __syncthreads();
  }
  Piece ex = threadIdx.x ? sp[threadIdx.x - 1] : piece_identity();
  __syncthreads();
  return ex;
}

__device__ __forceinline__ int block_excl_scan_int(int v, int* si, int& total) {
  si[threadIdx.x] = v;
  __syncthreads();
  for (int o = 1; o < kThreads; o <<= 1) {
    const int x = si[threadIdx.x];
    const int y = threadIdx.x >= o ? si[threadIdx.x - o] : 0;
    __syncthreads();
    si[threadIdx.x] = x + y;
    __syncthreads();
  }
  total = si[kThreads - 1];
  const int ex = threadIdx.x ? si[threadIdx.x - 1] : 0;
  __syncthreads();
  return ex;
}

// Shared per-tile analysis used by S2 and S3 (identical code => identical
// classification in both).
struct TileScan {
  Piece carry;      // exclusive segmented prefix for this thread
  int win_excl;     // windows before this thread's first element
  int win_total;    // windows in the tile
  DD p0;            // approximate prefix before this thread's first element
  long long c0;
};

__device__ __forceinline__ void analyse_tile(const Ctx& c, int t, const double* sg, TileScan& ts,
                                             DD* sdd, long long* scnt, Piece* spc, int* si) {
  DD s = {0.0, 0.0};
  long long cnt = 0;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const double g = sg[sidx(threadIdx.x * kItems + i)];
    s = dd_add(s, g);
    cnt += (g != 0.0);
  }
  DD ex;
  long long cex;
  block_excl_scan_dd(s, cnt, ex, cex, sdd, scnt);
  DD tp;
  tp.hi = __ldcg(&c.tile_pre[t].hi);
  tp.lo = __ldcg(&c.tile_pre[t].lo);
  ts.p0 = dd_add(tp, ex);
  ts.c0 = __ldcg(&c.tile_cnt_pre[t]) + cex;
  // thread-local pass: aggregate piece + window count
  DD P = ts.p0;
  long long C = ts.c0;
  Piece agg = piece_identity();
  int nw = 0;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const double g = sg[sidx(threadIdx.x * kItems + i)];
    const DD pp = P;
    const long long cp = C;
    P = dd_add(P, g);
    C += (g != 0.0);
    Piece pc;
    const int kind = classify(g, pp, cp, P, C, pc);
    nw += (kind == 2);
    agg = piece_combine(agg, pc);
  }
  ts.carry = block_excl_scan_piece(agg, spc);
  ts.win_excl = block_excl_scan_int(nw, si, ts.win_total);
}

// S2: tile records (window list + segment aggregates); last block resolves
// the exact chain over tiles (serial over windows, exact integer runs).
__global__ void __launch_bounds__(kThreads) k_scan_pieces(Ctx c) {
  __shared__ double sg[kSmemTile];
  __shared__ DD sdd[kThreads];
  __shared__ long long scnt[kThreads];
  __shared__ Piece spc[kThreads];
  __shared__ int si[kThreads];
  __shared__ int s_last;
  if (grid_error(c)) return;
  const int t = blockIdx.x;
  load_tile_g(c, t, sg);
  TileScan ts;
  analyse_tile(c, t, sg, ts, sdd, scnt, spc, si);
  const bool overflow = ts.win_total > kMaxWin;
  // second local pass: emit windows with the aggregate preceding each
  DD P = ts.p0;
  long long C = ts.c0;
  Piece acc = ts.carry;
  int w = ts.win_excl;
  for (int i = 0; i < kItems; ++i) {
    const int e = threadIdx.x * kItems + i;
    const double g = sg[sidx(e)];
    const DD pp = P;
    const long long cp = C;
    P = dd_add(P, g);
    C += (g != 0.0);
    Piece pc;
    const int kind = classify(g, pp, cp, P, C, pc);
    if (kind == 2 && !overflow) {
      TileWin tw;
      tw.g = g;
      tw.e = acc.e;
      tw.local = e;
      tw.d0 = acc.d0;
      tw.d1 = acc.d1;
      c.win[static_cast<size_t>(t) * kMaxWin + w] = tw;
      ++w;
    }
    acc = piece_combine(acc, pc);
  }
  if (threadIdx.x == kThreads - 1) {
    TileHdr h;
    h.nwin = overflow ? -1 : ts.win_total;
    h.tail_e = acc.e;
    h.tail_d0 = acc.d0;
    h.tail_d1 = acc.d1;
    c.hdr[t] = h;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned old = atomicAdd(&c.cnt_scan[1], 1u);
    s_last = (old == gridDim.x - 1);
    if (s_last) c.cnt_scan[1] = 0;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // ---- resolver: one thread walks the tiles in order -----------------
  if (threadIdx.x == 0) {
    const double lse = c.st->lse_g;
    double s = 0.0;
    bool ok = true;
    for (int tt = 0; tt < c.ntiles; ++tt) {
      c.tile_start[tt] = s;
      const int nwin = __ldcg(&c.hdr[tt].nwin);
      if (nwin < 0) {
        // serial tile: plain IEEE sequential sum, writes the CDF directly
        const long long base = static_cast<long long>(tt) * kTile;
        for (int e = 0; e < kTile && base + e < c.N; ++e) {
          s = s + fitness_of(c, base + e, lse);
          c.cdf[base + e] = s;
        }
      } else {
        for (int wi = 0; wi < nwin; ++wi) {
          const TileWin* tw = c.win + static_cast<size_t>(tt) * kMaxWin + wi;
          Piece a;
          a.e = __ldcg(&tw->e);
          a.d0 = __ldcg(&tw->d0);
          a.d1 = __ldcg(&tw->d1);
          a.flag = 0;
          ok &= piece_apply(a, s);
          s = s + __ldcg(&tw->g);
          c.win_after[static_cast<size_t>(tt) * kMaxWin + wi] = s;
        }
        Piece a;
        a.e = __ldcg(&c.hdr[tt].tail_e);
        a.d0 = __ldcg(&c.hdr[tt].tail_d0);
        a.d1 = __ldcg(&c.hdr[tt].tail_d1);
        a.flag = 0;
        ok &= piece_apply(a, s);
      }
      c.tile_end[tt] = s;
    }
    c.st->total_mass = s;
    // guard the last bin (filter.cpp:168)
    c.tile_end[c.ntiles - 1] = (s < 1.0) ? 1.0 : s;
    if (!ok) atomicOr(&c.st->error, kErrInternal);
  }
}

// S3: exact per-element CDF, per-tile local guide and the coarse guide.
__global__ void __launch_bounds__(kThreads) k_scan_cdf(Ctx c) {
  __shared__ double sg[kSmemTile];
  __shared__ DD sdd[kThreads];
  __shared__ long long scnt[kThreads];
  __shared__ Piece spc[kThreads];
  __shared__ int si[kThreads];
  if (grid_error(c)) return;
  const int t = blockIdx.x;
  const long long base = static_cast<long long>(t) * kTile;
  load_tile_g(c, t, sg);
  const int nwin = __ldcg(&c.hdr[t].nwin);
  const double c_start = __ldcg(&c.tile_start[t]);
  const double c_end = __ldcg(&c.tile_end[t]);
  if (nwin >= 0) {
    TileScan ts;
    analyse_tile(c, t, sg, ts, sdd, scnt, spc, si);
    DD P = ts.p0;
    long long C = ts.c0;
    Piece acc = ts.carry;
    int w = ts.win_excl;
    double seg = w > 0 ? __ldcg(&c.win_after[static_cast<size_t>(t) * kMaxWin + w - 1]) : c_start;
    double vals[kItems];
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const int e = threadIdx.x * kItems + i;
      const double g = sg[sidx(e)];
      const DD pp = P;
      const long long cp = C;
      P = dd_add(P, g);
      C += (g != 0.0);
      Piece pc;
      const int kind = classify(g, pp, cp, P, C, pc);
      acc = piece_combine(acc, pc);
      double sk;
      if (kind == 2) {
        seg = __ldcg(&c.win_after[static_cast<size_t>(t) * kMaxWin + w]);
        ++w;
        sk = seg;
      } else {
        sk = seg;
        piece_apply(acc, sk);
      }
      vals[i] = sk;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kItems; ++i) sg[sidx(threadIdx.x * kItems + i)] = vals[i];
    __syncthreads();
  } else {
    __syncthreads();
#pragma unroll 4
    for (int i = 0; i < kItems; ++i) {
      const int e = i * kThreads + threadIdx.x;
      sg[sidx(e)] = base + e < c.N ? __ldcg(&c.cdf[base + e]) : 0.0;
    }
    __syncthreads();
  }
  // guard + padding beyond N, then write the CDF (coalesced)
  const int valid = static_cast<int>(min(static_cast<long long>(kTile), c.N - base));
#pragma unroll 4
  for (int i = 0; i < kItems; ++i) {
    const int e = i * kThreads + threadIdx.x;
    double v = sg[sidx(e)];
    if (base + e == c.N - 1) v = (v < 1.0) ? 1.0 : v;  // filter.cpp:168
    if (e >= valid) v = INFINITY;
    sg[sidx(e)] = v;
  }
  __syncthreads();
#pragma unroll 4
  for (int i = 0; i < kItems; ++i) {
    const int e = i * kThreads + threadIdx.x;
    if (e < valid) c.cdf[base + e] = sg[sidx(e)];
  }
  // local guide: bucket i edge x_i = c_start + i*w; first local k with cdf > x_i
  const double wdt = (c_end - c_start) * (1.0 / kTile);
  for (int i = threadIdx.x; i < kTile; i += kThreads) {
    const double x = c_start + static_cast<double>(i) * wdt;
    int lo = 0, len = valid;
    while (len > 0) {
      const int half = len >> 1;
      if (!(x < sg[sidx(lo + half)])) {
        lo += half + 1;
        len -= half + 1;
      } else {
        len = half;
      }
    }
    c.lguide[base + i] = static_cast<unsigned short>(min(lo, valid - 1));
  }
  // coarse guide: buckets b with c_start <= b/B1 < c_end point at this tile
  const double B1 = ldexp(1.0, c.coarse_bits);
  const long long nb = 1LL << c.coarse_bits;
  long long b_lo = static_cast<long long>(ceil(c_start * B1));
  long long b_hi = static_cast<long long>(ceil(fmin(c_end, 1.0) * B1)) - 1;
  if (c_end >= 1.0) b_hi = nb - 1;
  b_lo = max(b_lo, 0LL);
  b_hi = min(b_hi, nb - 1);
  for (long long b = b_lo + threadIdx.x; b <= b_hi; b += kThreads) c.coarse[b] = t;
}

__global__ void __launch_bounds__(kThreads) k_search_only(Ctx c) {
  if (grid_error(c)) return;
  const long long n = static_cast<long long>(blockIdx.x) * kThreads + threadIdx.x;
  if (n >= c.N) return;
  const double u = resample_uniform(c.seed, c.sp->j, n);
  c.anc[n] = find_ancestor(c, u);
}

// Record pack/unpack for the AoS boundary (filter::Ensemble layout).
__global__ void k_pack(Ctx c, int d, int p, const double* states, const double* params, int dir) {
  const long long n = static_cast<long long>(blockIdx.x) * kThreads + threadIdx.x;
  if (n >= c.N) return;
  double* r = c.rec[c.st->cur] + n * c.R;
  if (dir == 0) {
    for (int k = 0; k < d; ++k) r[k] = states[n * d + k];
    for (int k = 0; k < p; ++k) r[d + k] = params[n * p + k];
    for (int k = d + p; k < c.R; ++k) r[k] = 0.0;
  } else {
    double* so = const_cast<double*>(states);
    double* po = const_cast<double*>(params);
    for (int k = 0; k < d; ++k) so[n * d + k] = r[k];
    for (int k = 0; k < p; ++k) po[n * p + k] = r[d + k];
  }
}

__global__ void k_flush(double* buf, long long n) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    buf[i] = static_cast<double>(i);
}

struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NumericalError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define CK(x)                                                                            \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess)                                                               \
      throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e_) + " at " + \
                               #x);                                                      \
  } while (0)

static const char* kKernelNames = "k_predict,k_scan_sums,k_scan_pieces,k_scan_cdf,k_update";
constexpr int kNumKernels = 5;

}  // namespace pfsmc_gpu

using namespace pfsmc_gpu;

struct pfsmc_gpu_sampler {
  pfsmc_gpu_config cfg{};
  std::vector<uint64_t> obs;
  std::unique_ptr<KernelSet> ks;
  int d = 0, p = 0;
  long long N = 0;
  int grid = 0, ntiles = 0;
  Ctx ctx{};
  cudaStream_t stream = nullptr;
  // device buffers
  std::vector<void*> allocs;
  DevState* st = nullptr;
  StepParams* sp_dev = nullptr;
  StepParams* sp_host = nullptr;     // pinned
  double* trace_host = nullptr;      // pinned
  DevState* st_host = nullptr;       // pinned
  double* flush_buf = nullptr;
  long long flush_n = 0;
  // resident observations
  std::vector<StepParams> resident;
  StepParams* resident_dev = nullptr;
  double t0_resident = 0.0;
  // graph
  cudaGraphExec_t graph = nullptr;
  bool timing = false;
  cudaEvent_t ev[kNumKernels + 1] = {};
  double kernel_ms[kNumKernels] = {};
  std::vector<cudaEvent_t> pending;  // (kNumKernels+1) per timed step
  bool have_ensemble = false;

  template <typename T>
  T* dalloc(size_t count) {
    void* p = nullptr;
    CK(cudaMalloc(&p, sizeof(T) * std::max<size_t>(count, 1)));
    allocs.push_back(p);
    return static_cast<T*>(p);
  }
  ~pfsmc_gpu_sampler() {
    if (graph) cudaGraphExecDestroy(graph);
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
    for (auto e : pending) cudaEventDestroy(e);
    for (void* a : allocs) cudaFree(a);
    if (sp_host) cudaFreeHost(sp_host);
    if (trace_host) cudaFreeHost(trace_host);
    if (st_host) cudaFreeHost(st_host);
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace {
thread_local std::string g_last_error;

template <typename F>
pfsmc_gpu_status guarded(F&& f) {
  try {
    return f();
  } catch (const ConfigError& e) {
    g_last_error = e.what();
    return PFSMC_GPU_ERR_CONFIG;
  } catch (const NumericalError& e) {
    g_last_error = e.what();
    return PFSMC_GPU_ERR_NUMERICAL;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return PFSMC_GPU_ERR_INTERNAL;
  }
}

// interval_step_count (lmm.cpp:350-362)
int step_count(double t0, double t1, double h) {
  if (!(t1 > t0) || !(h > 0.0)) throw ConfigError("propagate_interval: need t1 > t0 and h > 0");
  const double ratio = (t1 - t0) / h;
  const long long m = std::llround(ratio);
  if (m < 1 || std::abs(ratio - static_cast<double>(m)) > 1e-9 * std::max(1.0, ratio))
    throw ConfigError("propagate_interval: (t1 - t0)/h must be an integer step count");
  if (m > (1LL << 30)) throw ConfigError("propagate_interval: too many steps");
  return static_cast<int>(m);
}

StepParams make_params(pfsmc_gpu_sampler* s, const double* y, uint64_t j, double t_prev,
                       double t_obs, double h) {
  StepParams sp{};
  sp.j = j;
  sp.t_prev = t_prev;
  sp.h = h;
  sp.m = step_count(t_prev, t_obs, h);
  const double m = static_cast<double>(s->cfg.n_obs);
  const double s2 = s->cfg.sigma * s->cfg.sigma;
  constexpr double kLog2Pi = 1.8378770664093453;
  sp.ll_const = -0.5 * m * (kLog2Pi + std::log(s2));
  if (s->cfg.likelihood == PFSMC_GPU_LIK_LOGNORMAL) {
    double sly = 0.0;
    for (uint64_t k = 0; k < s->cfg.n_obs; ++k) {
      if (!(y[k] > 0.0)) throw ConfigError("lognormal likelihood needs positive observations");
      sp.y[k] = std::log(y[k]);
      sly += sp.y[k];
    }
    sp.sly = sly;
  } else {
    for (uint64_t k = 0; k < s->cfg.n_obs; ++k) sp.y[k] = y[k];
  }
  return sp;
}

void check_error(pfsmc_gpu_sampler* s) {
  const DevState& st = *s->st_host;
  if (st.error & kErrPredict)
    throw NumericalError("total degeneracy: every particle has zero predictive likelihood");
  if (st.error & kErrChol) throw NumericalError("chol_psd: degenerate covariance");
  if (st.error & kErrUpdate)
    throw NumericalError("total degeneracy: every repropagated particle has zero likelihood");
  if (st.error & kErrInternal) throw std::runtime_error("exact CDF: internal inconsistency");
}

void enqueue_kernels(pfsmc_gpu_sampler* s, bool timed) {
  const Ctx& c = s->ctx;
  cudaStream_t st = s->stream;
  cudaEvent_t* ev = nullptr;
  if (timed) {
    for (int i = 0; i <= kNumKernels; ++i) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      s->pending.push_back(e);
    }
    ev = s->pending.data() + s->pending.size() - (kNumKernels + 1);
    CK(cudaEventRecord(ev[0], st));
  }
  s->ks->predict(c, s->grid, st);
  if (timed) CK(cudaEventRecord(ev[1], st));
  k_scan_sums<<<s->ntiles, kThreads, 0, st>>>(c);
  if (timed) CK(cudaEventRecord(ev[2], st));
  k_scan_pieces<<<s->ntiles, kThreads, 0, st>>>(c);
  if (timed) CK(cudaEventRecord(ev[3], st));
  k_scan_cdf<<<s->ntiles, kThreads, 0, st>>>(c);
  if (timed) CK(cudaEventRecord(ev[4], st));
  s->ks->update(c, s->grid, st);
  if (timed) CK(cudaEventRecord(ev[5], st));
  CK(cudaGetLastError());
}

// Step prologue: clear per-step error/iteration counters (device memsets).
void enqueue_prologue(pfsmc_gpu_sampler* s) {
  CK(cudaMemsetAsync(&s->st->error, 0, sizeof(int), s->stream));
  CK(cudaMemsetAsync(&s->st->newton_iters, 0, sizeof(unsigned long long), s->stream));
}

void build_graph(pfsmc_gpu_sampler* s) {
  cudaGraph_t g;
  CK(cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal));
  enqueue_prologue(s);
  enqueue_kernels(s, false);
  CK(cudaMemcpyAsync(s->st_host, s->st, sizeof(DevState), cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamEndCapture(s->stream, &g));
  CK(cudaGraphInstantiate(&s->graph, g, 0));
  CK(cudaGraphDestroy(g));
}

void harvest_timing(pfsmc_gpu_sampler* s) {
  if (s->pending.empty()) return;
  CK(cudaStreamSynchronize(s->stream));
  const size_t steps = s->pending.size() / (kNumKernels + 1);
  for (size_t i = 0; i < steps; ++i) {
    cudaEvent_t* e = s->pending.data() + i * (kNumKernels + 1);
    for (int k = 0; k < kNumKernels; ++k) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, e[k], e[k + 1]));
      s->kernel_ms[k] += ms;
    }
  }
  for (auto e : s->pending) cudaEventDestroy(e);
  s->pending.clear();
}

// Params come either from the pinned host slot (blocking drop-in step; the
// previous step has completed, so the slot is free) or from the resident
// device array (no host involvement).
void enqueue_step(pfsmc_gpu_sampler* s, const StepParams* host_sp, const StepParams* dev_sp) {
  if (!s->have_ensemble) throw ConfigError("step: no ensemble (call set_ensemble or init_*)");
  if (dev_sp) {
    CK(cudaMemcpyAsync(s->sp_dev, dev_sp, sizeof(StepParams), cudaMemcpyDeviceToDevice, s->stream));
  } else {
    *s->sp_host = *host_sp;
    CK(cudaMemcpyAsync(s->sp_dev, s->sp_host, sizeof(StepParams), cudaMemcpyHostToDevice, s->stream));
  }
  if (s->timing) {
    enqueue_prologue(s);
    enqueue_kernels(s, true);
    CK(cudaMemcpyAsync(s->st_host, s->st, sizeof(DevState), cudaMemcpyDeviceToHost, s->stream));
  } else {
    CK(cudaGraphLaunch(s->graph, s->stream));
  }
}

}  // namespace

extern "C" {

const char* pfsmc_gpu_version(void) { return "pfsmc_gpu 0.1 (sm_100a)"; }
const char* pfsmc_gpu_last_error(void) { return g_last_error.c_str(); }

pfsmc_gpu_status pfsmc_gpu_create(const pfsmc_gpu_config* cfg, pfsmc_gpu_sampler** out) {
  return guarded([&] {
    *out = nullptr;
    if (!cfg) throw ConfigError("null config");
    // PfConfig::validate (filter.cpp:45-74)
    if (cfg->particles == 0) throw ConfigError("config: particles must be >= 1");
    if (cfg->particles > (1ULL << 31)) throw ConfigError("config: particles must be < 2^31 per handle");
    if (!(cfg->shrink_a > 0.0 && cfg->shrink_a < 1.0))
      throw ConfigError("config: shrink factor a must lie in (0, 1)");
    if (!(cfg->sigma > 0.0)) throw ConfigError("config: observation noise sigma must be positive");
    if (cfg->order < 1 || cfg->order > 3)
      throw ConfigError("scheme_coefficients: order must be 1, 2 or 3");
    if (cfg->family < 0 || cfg->family > 2) throw ConfigError("scheme_coefficients: unknown family");
    if (cfg->n_obs > static_cast<uint64_t>(kMaxObs)) throw ConfigError("config: at most 8 observed components");
    auto s = std::make_unique<pfsmc_gpu_sampler>();
    s->cfg = *cfg;
    s->ks = make_kernels(cfg->model, cfg->family, cfg->order);
    if (!s->ks) throw ConfigError("unknown model id");
    s->d = s->ks->d;
    s->p = s->ks->p;
    std::vector<bool> seen(s->d, false);
    for (uint64_t k = 0; k < cfg->n_obs; ++k) {
      const uint64_t idx = cfg->obs_indices[k];
      if (idx >= static_cast<uint64_t>(s->d) || seen[idx])
        throw ConfigError("config: observation indices must be distinct and in range");
      seen[idx] = true;
      s->obs.push_back(idx);
    }
    s->cfg.obs_indices = s->obs.data();
    CK(cudaSetDevice(cfg->device));
    CK(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
    s->N = static_cast<long long>(cfg->particles);
    s->grid = static_cast<int>((s->N + kThreads - 1) / kThreads);
    s->ntiles = static_cast<int>((s->N + kTile - 1) / kTile);
    Ctx& c = s->ctx;
    c.N = static_cast<int>(s->N);
    c.R = ((s->d + s->p + 1) / 2) * 2;
    c.ntiles = s->ntiles;
    c.m_y = static_cast<int>(cfg->n_obs);
    c.likelihood = cfg->likelihood;
    for (int k = 0; k < kMaxObs; ++k) c.obs_idx[k] = k < c.m_y ? static_cast<int>(s->obs[k]) : -1;
    c.a = cfg->shrink_a;
    c.one_minus_a = 1.0 - cfg->shrink_a;
    c.s_prolif = std::sqrt(1.0 - cfg->shrink_a * cfg->shrink_a);
    c.tol = cfg->newton_tol;
    c.max_iter = cfg->newton_max_iter;
    c.seed = cfg->seed;
    c.two_s2 = 2.0 * (cfg->sigma * cfg->sigma);
    int cb = 6;
    while ((1LL << cb) < 4LL * s->ntiles) ++cb;
    c.coarse_bits = cb;
    const size_t N = static_cast<size_t>(s->N);
    const size_t NT = static_cast<size_t>(s->ntiles);
    c.rec[0] = s->dalloc<double>(N * c.R);
    c.rec[1] = s->dalloc<double>(N * c.R);
    c.lw = s->dalloc<double>(N);
    c.llbar = s->dalloc<double>(N);
    c.lg = s->dalloc<double>(N);
    c.cdf = s->dalloc<double>(N);
    c.anc = s->dalloc<unsigned>(N);
    c.lguide = s->dalloc<unsigned short>(NT * kTile);
    c.coarse = s->dalloc<unsigned>(size_t(1) << cb);
    c.tile_start = s->dalloc<double>(NT);
    c.tile_end = s->dalloc<double>(NT);
    c.tile_sum = s->dalloc<DD>(NT);
    c.tile_cnt = s->dalloc<long long>(NT);
    c.tile_pre = s->dalloc<DD>(NT);
    c.tile_cnt_pre = s->dalloc<long long>(NT);
    c.hdr = s->dalloc<TileHdr>(NT);
    c.win = s->dalloc<TileWin>(NT * kMaxWin);
    c.win_after = s->dalloc<double>(NT * kMaxWin);
    const int vmax = 1 + 4 + 10 + 8 + 1 + 1;
    c.part = s->dalloc<double>(static_cast<size_t>(s->grid) * vmax + 64);
    c.gpart = s->dalloc<double>(static_cast<size_t>(s->grid / kGroup + 2) * vmax + 64);
    const int ngroups = (s->grid + kGroup - 1) / kGroup;
    unsigned* cnts = s->dalloc<unsigned>(2 * (ngroups + 1) + 8);
    CK(cudaMemset(cnts, 0, (2 * (ngroups + 1) + 8) * sizeof(unsigned)));
    c.cnt_pred = cnts;
    c.cnt_upd = cnts + (ngroups + 1);
    c.cnt_scan = cnts + 2 * (ngroups + 1);
    c.gin = nullptr;
    s->st = s->dalloc<DevState>(1);
    CK(cudaMemset(s->st, 0, sizeof(DevState)));
    c.st = s->st;
    s->sp_dev = s->dalloc<StepParams>(1);
    c.sp = s->sp_dev;
    CK(cudaMallocHost(&s->sp_host, sizeof(StepParams)));
    CK(cudaMallocHost(&s->st_host, sizeof(DevState)));
    CK(cudaMallocHost(&s->trace_host, 64 * sizeof(double)));
    build_graph(s.get());
    *out = s.release();
    return PFSMC_GPU_OK;
  });
}

void pfsmc_gpu_destroy(pfsmc_gpu_sampler* s) { delete s; }

void* pfsmc_gpu_stream(pfsmc_gpu_sampler* s) { return s ? s->stream : nullptr; }

pfsmc_gpu_status pfsmc_gpu_set_ensemble(pfsmc_gpu_sampler* s, const double* states,
                                        const double* params_u, const double* logw,
                                        const double* mean_u, const double* cov_u) {
  return guarded([&] {
    const size_t N = static_cast<size_t>(s->N);
    const int d = s->d, p = s->p;
    double* tmp_x = s->dalloc<double>(N * d);
    double* tmp_t = s->dalloc<double>(N * p);
    CK(cudaMemcpyAsync(tmp_x, states, sizeof(double) * N * d, cudaMemcpyHostToDevice, s->stream));
    CK(cudaMemcpyAsync(tmp_t, params_u, sizeof(double) * N * p, cudaMemcpyHostToDevice, s->stream));
    CK(cudaMemcpyAsync(s->ctx.lw, logw, sizeof(double) * N, cudaMemcpyHostToDevice, s->stream));
    DevState h{};
    CK(cudaMemcpyAsync(&h, s->st, sizeof(DevState), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    h.lse_w = 0.0;
    h.error = 0;
    h.chol_failed = 0;
    for (int k = 0; k < p; ++k) h.mu[k] = mean_u[k];  // shift only; recomputed below
    for (int k = 0; k < p * p; ++k) h.cov[k] = cov_u[k];
    CK(cudaMemcpyAsync(s->st, &h, sizeof(DevState), cudaMemcpyHostToDevice, s->stream));
    k_pack<<<s->grid, kThreads, 0, s->stream>>>(s->ctx, d, p, tmp_x, tmp_t, 0);
    s->ks->moments(s->ctx, s->grid, s->stream, 0);  // shrink mean + chol(cov_u)
    CK(cudaStreamSynchronize(s->stream));
    CK(cudaGetLastError());
    cudaFree(tmp_x);
    cudaFree(tmp_t);
    s->allocs.resize(s->allocs.size() - 2);
    s->have_ensemble = true;
    return PFSMC_GPU_OK;
  });
}

pfsmc_gpu_status pfsmc_gpu_get_ensemble(pfsmc_gpu_sampler* s, double* states, double* params_u,
                                        double* logw, double* mean_u, double* cov_u) {
  return guarded([&] {
    const size_t N = static_cast<size_t>(s->N);
    const int d = s->d, p = s->p;
    double* tmp_x = s->dalloc<double>(N * d);
    double* tmp_t = s->dalloc<double>(N * p);
    k_pack<<<s->grid, kThreads, 0, s->stream>>>(s->ctx, d, p, tmp_x, tmp_t, 1);
    if (states) CK(cudaMemcpyAsync(states, tmp_x, sizeof(double) * N * d, cudaMemcpyDeviceToHost, s->stream));
    if (params_u) CK(cudaMemcpyAsync(params_u, tmp_t, sizeof(double) * N * p, cudaMemcpyDeviceToHost, s->stream));
    DevState h{};
    CK(cudaMemcpyAsync(&h, s->st, sizeof(DevState), cudaMemcpyDeviceToHost, s->stream));
    if (logw) CK(cudaMemcpyAsync(logw, s->ctx.lw, sizeof(double) * N, cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    if (logw)
      for (size_t i = 0; i < N; ++i) logw[i] = logw[i] - h.lse_w;  // update_weights: lw -= lse
    if (mean_u)
      for (int k = 0; k < p; ++k) mean_u[k] = h.mu[k];
    if (cov_u)
      for (int k = 0; k < p * p; ++k) cov_u[k] = h.cov[k];
    cudaFree(tmp_x);
    cudaFree(tmp_t);
    s->allocs.resize(s->allocs.size() - 2);
    return PFSMC_GPU_OK;
  });
}

static pfsmc_gpu_status do_init(pfsmc_gpu_sampler* s, int kind, const std::vector<double>& prm) {
  return guarded([&] {
    double* dprm = s->dalloc<double>(prm.size());
    CK(cudaMemcpyAsync(dprm, prm.data(), sizeof(double) * prm.size(), cudaMemcpyHostToDevice, s->stream));
    DevState h{};
    CK(cudaMemcpyAsync(&h, s->st, sizeof(DevState), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    h.lse_w = 0.0;
    h.error = 0;
    h.chol_failed = 0;
    for (int k = 0; k < 4; ++k) h.mu[k] = 0.0;
    CK(cudaMemcpyAsync(s->st, &h, sizeof(DevState), cudaMemcpyHostToDevice, s->stream));
    const double lw0 = -std::log(static_cast<double>(s->N));  // filter.cpp:86
    s->ks->init(s->ctx, s->grid, s->stream, kind, dprm, lw0);
    // first pass: mean about 0; second pass: cov about that mean
    s->ks->moments(s->ctx, s->grid, s->stream, 1);
    s->ks->moments(s->ctx, s->grid, s->stream, 1);
    CK(cudaStreamSynchronize(s->stream));
    CK(cudaGetLastError());
    cudaFree(dprm);
    s->allocs.pop_back();
    s->have_ensemble = true;
    return PFSMC_GPU_OK;
  });
}

pfsmc_gpu_status pfsmc_gpu_init_gaussian(pfsmc_gpu_sampler* s, const double* th_mu,
                                         const double* th_sigma, const double* x_mean,
                                         const double* x_std, const int* x_clamp) {
  std::vector<double> prm;
  for (int k = 0; k < s->p; ++k) prm.push_back(th_mu[k]);
  for (int k = 0; k < s->p; ++k) prm.push_back(th_sigma[k]);
  for (int k = 0; k < s->d; ++k) prm.push_back(x_mean[k]);
  for (int k = 0; k < s->d; ++k) prm.push_back(x_std[k]);
  for (int k = 0; k < s->d; ++k) prm.push_back(x_clamp ? static_cast<double>(x_clamp[k]) : 0.0);
  return do_init(s, 0, prm);
}

pfsmc_gpu_status pfsmc_gpu_init_uniform(pfsmc_gpu_sampler* s, const double* th_lo, const double* th_hi,
                                        const double* x_lo, const double* x_hi) {
  std::vector<double> prm;
  for (int k = 0; k < s->p; ++k) prm.push_back(th_lo[k]);
  for (int k = 0; k < s->p; ++k) prm.push_back(th_hi[k]);
  for (int k = 0; k < s->d; ++k) prm.push_back(x_lo[k]);
  for (int k = 0; k < s->d; ++k) prm.push_back(x_hi[k]);
  return do_init(s, 1, prm);
}

pfsmc_gpu_status pfsmc_gpu_step(pfsmc_gpu_sampler* s, const double* y, uint64_t j, double t_prev,
                                double t_obs, double h, double* trace_out) {
  return guarded([&] {
    const StepParams sp = make_params(s, y, j, t_prev, t_obs, h);
    enqueue_step(s, &sp, nullptr);
    CK(cudaStreamSynchronize(s->stream));
    harvest_timing(s);
    check_error(s);
    if (trace_out) {
      const int n = 2 * s->p + s->d + 1;
      for (int k = 0; k < n; ++k) trace_out[k] = s->st_host->trace[k];
    }
    return PFSMC_GPU_OK;
  });
}

pfsmc_gpu_status pfsmc_gpu_upload_observations(pfsmc_gpu_sampler* s, const double* ys,
                                               const double* t_obs, uint64_t T, double t0, double h) {
  return guarded([&] {
    s->resident.clear();
    double tp = t0;
    for (uint64_t j = 0; j < T; ++j) {
      s->resident.push_back(make_params(s, ys + j * s->cfg.n_obs, j + 1, tp, t_obs[j], h));
      tp = t_obs[j];
    }
    s->t0_resident = t0;
    if (s->resident_dev) {
      cudaFree(s->resident_dev);
      s->allocs.erase(std::find(s->allocs.begin(), s->allocs.end(), static_cast<void*>(s->resident_dev)));
    }
    s->resident_dev = s->dalloc<StepParams>(s->resident.size());
    CK(cudaMemcpy(s->resident_dev, s->resident.data(), sizeof(StepParams) * s->resident.size(),
                  cudaMemcpyHostToDevice));
    return PFSMC_GPU_OK;
  });
}

pfsmc_gpu_status pfsmc_gpu_step_resident(pfsmc_gpu_sampler* s, uint64_t j) {
  return guarded([&] {
    if (j < 1 || j > s->resident.size()) throw ConfigError("step_resident: j out of range");
    enqueue_step(s, nullptr, s->resident_dev + (j - 1));
    return PFSMC_GPU_OK;
  });
}

pfsmc_gpu_status pfsmc_gpu_synchronize(pfsmc_gpu_sampler* s, double* trace_out) {
  return guarded([&] {
    CK(cudaStreamSynchronize(s->stream));
    harvest_timing(s);
    check_error(s);
    if (trace_out) {
      const int n = 2 * s->p + s->d + 1;
      for (int k = 0; k < n; ++k) trace_out[k] = s->st_host->trace[k];
    }
    return PFSMC_GPU_OK;
  });
}

pfsmc_gpu_status pfsmc_gpu_run(pfsmc_gpu_sampler* s, double* rows, int* warn) {
  return guarded([&] {
    const int w = 2 * s->p + s->d + 1;
    // row 0 from the current ensemble (filter.cpp:409-426)
    s->ks->moments(s->ctx, s->grid, s->stream, 0);
    DevState h{};
    CK(cudaMemcpyAsync(&h, s->st, sizeof(DevState), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    for (int k = 0; k < w; ++k) rows[k] = h.trace[k];
    if (warn) warn[0] = 0;
    int streak = 0;
    for (size_t j = 1; j <= s->resident.size(); ++j) {
      enqueue_step(s, nullptr, s->resident_dev + (j - 1));
      CK(cudaStreamSynchronize(s->stream));
      harvest_timing(s);
      check_error(s);
      for (int k = 0; k < w; ++k) rows[j * w + k] = s->st_host->trace[k];
      const double ess = s->st_host->trace[w - 1];
      int flag = 0;
      if (ess < 1.0 + 1e-6) {
        if (++streak >= 3) flag = 1;
      } else {
        streak = 0;
      }
      if (warn) warn[j] = flag;
    }
    return PFSMC_GPU_OK;
  });
}

pfsmc_gpu_status pfsmc_gpu_get_step_diagnostics(pfsmc_gpu_sampler* s, uint32_t* ancestors,
                                                double* loglik_bar, uint64_t* newton_iters) {
  return guarded([&] {
    const size_t N = static_cast<size_t>(s->N);
    if (ancestors) CK(cudaMemcpyAsync(ancestors, s->ctx.anc, sizeof(uint32_t) * N, cudaMemcpyDeviceToHost, s->stream));
    if (loglik_bar) CK(cudaMemcpyAsync(loglik_bar, s->ctx.llbar, sizeof(double) * N, cudaMemcpyDeviceToHost, s->stream));
    DevState h{};
    CK(cudaMemcpyAsync(&h, s->st, sizeof(DevState), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    if (newton_iters) *newton_iters = h.newton_iters;
    return PFSMC_GPU_OK;
  });
}

pfsmc_gpu_status pfsmc_gpu_resample_from_g(pfsmc_gpu_sampler* s, const double* g, uint64_t j,
                                           uint32_t* ancestors_out, double* cdf_out) {
  return guarded([&] {
    const size_t N = static_cast<size_t>(s->N);
    for (size_t i = 0; i < N; ++i)
      if (!(g[i] >= 0.0) || !std::isfinite(g[i])) throw ConfigError("resample: g must be finite and >= 0");
    double* dg = s->dalloc<double>(N);
    CK(cudaMemcpyAsync(dg, g, sizeof(double) * N, cudaMemcpyHostToDevice, s->stream));
    StepParams sp{};
    sp.j = j;
    *s->sp_host = sp;
    CK(cudaMemcpyAsync(s->sp_dev, s->sp_host, sizeof(StepParams), cudaMemcpyHostToDevice, s->stream));
    CK(cudaMemsetAsync(&s->st->error, 0, sizeof(int), s->stream));
    Ctx c = s->ctx;
    c.gin = dg;
    k_scan_sums<<<s->ntiles, kThreads, 0, s->stream>>>(c);
    k_scan_pieces<<<s->ntiles, kThreads, 0, s->stream>>>(c);
    k_scan_cdf<<<s->ntiles, kThreads, 0, s->stream>>>(c);
    k_search_only<<<s->grid, kThreads, 0, s->stream>>>(c);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(ancestors_out, c.anc, sizeof(uint32_t) * N, cudaMemcpyDeviceToHost, s->stream));
    if (cdf_out) CK(cudaMemcpyAsync(cdf_out, c.cdf, sizeof(double) * N, cudaMemcpyDeviceToHost, s->stream));
    CK(cudaMemcpyAsync(s->st_host, s->st, sizeof(DevState), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    cudaFree(dg);
    s->allocs.pop_back();
    if (s->st_host->error & kErrInternal) throw std::runtime_error("exact CDF: internal inconsistency");
    return PFSMC_GPU_OK;
  });
}

pfsmc_gpu_status pfsmc_gpu_set_kernel_timing(pfsmc_gpu_sampler* s, int enable) {
  return guarded([&] {
    harvest_timing(s);
    s->timing = enable != 0;
    for (double& v : s->kernel_ms) v = 0.0;
    return PFSMC_GPU_OK;
  });
}

pfsmc_gpu_status pfsmc_gpu_kernel_times(pfsmc_gpu_sampler* s, double* ms_out, int* n_kernels,
                                        const char** names_out) {
  return guarded([&] {
    harvest_timing(s);
    if (ms_out)
      for (int k = 0; k < kNumKernels; ++k) ms_out[k] = s->kernel_ms[k];
    if (n_kernels) *n_kernels = kNumKernels;
    if (names_out) *names_out = kKernelNames;
    return PFSMC_GPU_OK;
  });
}

pfsmc_gpu_status pfsmc_gpu_flush_l2(pfsmc_gpu_sampler* s) {
  return guarded([&] {
    if (!s->flush_buf) {
      s->flush_n = (256LL << 20) / 8;  // 256 MiB > 126 MB L2
      s->flush_buf = s->dalloc<double>(static_cast<size_t>(s->flush_n));
    }
    k_flush<<<148 * 4, 256, 0, s->stream>>>(s->flush_buf, s->flush_n);
    CK(cudaGetLastError());
    return PFSMC_GPU_OK;
  });
}

}  // extern "C"
