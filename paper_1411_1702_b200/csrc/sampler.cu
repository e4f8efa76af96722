// B200-native per-step LMM PF-SMC update: the device kernels, the host step
// driver (CUDA graph per step) and the C ABI declared in include/pfsmc_gpu.h.
//
// One step (reference: filter::pf_step, filter.cpp:292-394) is five launches:
//   K1 k_predict      shrink + Psi + log-lik + fitness lse   (filter.cpp:300-324, 143-156)
//   S1 (merged into S2: fitness g, look-back approximate tile prefixes)     \
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
#include <dlfcn.h>
#include <nccl.h>  // types only: NCCL is bound at run time (dlopen), see NcclApi

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
// Tiles of ITEMS * 256 elements (thread t owns elements ITEMS*t .. +ITEMS-1).
// ITEMS = 4 (1024-element tiles) keeps the per-thread serial chains short
// and the grid wide for N <= 2^22; ITEMS = 16 bounds the tile count (and the
// resolver's work) at larger N. One pad double per thread chunk keeps the
// per-thread contiguous shared-memory reads conflict-free.
template <int ITEMS>
struct TileCfg {
  static constexpr int kTileT = ITEMS * kThreads;
  static constexpr int kSmem = kTileT + kThreads;
  __device__ static __forceinline__ int sidx(int e) { return e + e / ITEMS; }
};

// Block-wide exclusive segmented scan of Piece, fixed shape.
__device__ __forceinline__ Piece block_excl_scan_piece(Piece v, Piece* sw) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  Piece x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const Piece y = shfl_up_piece(x, o);
    if (lane >= o) x = piece_combine(y, x);
  }
  if (lane == 31) sw[w] = x;
  __syncthreads();
  if (w == 0) {
    Piece t = lane < kWarps ? sw[lane] : piece_identity();
#pragma unroll
    for (int o = 1; o < kWarps; o <<= 1) {
      const Piece y = shfl_up_piece(t, o);
      if (lane >= o) t = piece_combine(y, t);
    }
    if (lane < kWarps) sw[kWarps + lane] = t;
  }
  __syncthreads();
  Piece ex = shfl_up_piece(x, 1);
  if (lane == 0) ex = piece_identity();
  if (w) ex = piece_combine(sw[kWarps + w - 1], ex);
  __syncthreads();
  return ex;
}

// Block-wide exclusive scan of ints.
__device__ __forceinline__ int block_excl_scan_int(int v, int& total, int* sw) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sw[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = lane < kWarps ? sw[lane] : 0;
#pragma unroll
    for (int o = 1; o < kWarps; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < kWarps) sw[kWarps + lane] = t;
  }
  __syncthreads();
  total = sw[2 * kWarps - 1];
  const int ex = x - v + (w ? sw[kWarps + w - 1] : 0);
  __syncthreads();
  return ex;
}

// Per-thread view of one tile, shared by S2 and S3 (identical code =>
// identical classification in both).
template <int ITEMS>
struct ThreadTile {
  double g[ITEMS];
  double p[ITEMS + 1];  // approximate prefix before each element (p[ITEMS]: after the last)
  int lc[ITEMS + 1];    // nonzero count before each element, relative to cnt0
  long long cnt0;       // nonzero count before the first element
  int uniform_e;        // binade of the whole chunk (fast path) or kNoBinade
  Piece agg;            // the chunk's aggregate piece
  int nwin;             // windows in the chunk
};

struct ScanScratch {
  SumCnt sc[2 * kWarps];
  Piece pc[2 * kWarps];
  int si[2 * kWarps];
};

// Fast-path rounding of one element in a known binade: delta for even /
// odd m (identical unless g/u ends in exactly one half).
// The scale 2^(52-e) is passed as two exact factors: for the subnormal
// binade (e = -1022) 2^1074 itself overflows, 2^537 * 2^537 does not.
struct UlpScale {
  double s1, s2;
};
__device__ __forceinline__ UlpScale ulp_scale(int e) {
  const int k = 52 - e;
  return k <= 1000 ? UlpScale{scale2(1.0, k), 1.0} : UlpScale{scale2(1.0, k - k / 2), scale2(1.0, k / 2)};
}

__device__ __forceinline__ void run_delta(double g, UlpScale scale, long long& d0, long long& d1) {
  const double v = (g * scale.s1) * scale.s2;  // exact: g < 2^(e+1)
  const double q = floor(v);
  const double f = v - q;
  const long long qi = static_cast<long long>(q);
  if (f < 0.5) {
    d0 = d1 = qi;
  } else if (f > 0.5) {
    d0 = d1 = qi + 1;
  } else {
    d0 = qi + (qi & 1);
    d1 = qi + ((1 + qi) & 1);
  }
}

// Classification of element i against the approximate prefix (general path).
template <int ITEMS>
__device__ __forceinline__ int classify_at(const ThreadTile<ITEMS>& tt, int i, Piece& pc) {
  return classify(tt.g[i], tt.p[i], tt.cnt0 + tt.lc[i], tt.p[i + 1], tt.cnt0 + tt.lc[i + 1], pc);
}

// Chunk analysis given p[0] and cnt0: prefix, fast-path test, aggregate.
// Fast path: when [p0 - E, p_end + E] lies in one binade, every nonzero
// element is a run element of that binade (the per-element bounds are
// nested inside), so the per-element classification would agree.
template <int ITEMS>
__device__ __forceinline__ void chunk_analyse(ThreadTile<ITEMS>& tt) {
  tt.lc[0] = 0;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    tt.p[i + 1] = tt.p[i] + tt.g[i];
    tt.lc[i + 1] = tt.lc[i] + (tt.g[i] != 0.0);
  }
  tt.uniform_e = kNoBinade;
  tt.agg = piece_identity();
  tt.nwin = 0;
  if (tt.lc[ITEMS] == 0) return;  // all zero: identity
  const double E = sum_bound(tt.p[ITEMS], tt.cnt0 + tt.lc[ITEMS]);
  const int e_lo = binade_of(tt.p[0] - E);
  const int e_hi = binade_of(tt.p[ITEMS] + E);
  if (e_lo == e_hi) {
    tt.uniform_e = e_lo;
    const UlpScale scale = ulp_scale(e_lo);
    long long s0 = 0, s1 = 0;
    bool tie = false;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      long long d0, d1;
      run_delta(tt.g[i], scale, d0, d1);
      tie |= (d0 != d1);
      s0 += d0;
      s1 += d1;
    }
    if (!tie) {
      tt.agg = Piece{s0, s1, e_lo, 0};
      return;
    }
    Piece a = piece_identity();
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      Piece pc = piece_identity();
      if (tt.g[i] != 0.0) {
        run_delta(tt.g[i], scale, pc.d0, pc.d1);
        pc.e = e_lo;
      }
      a = piece_combine(a, pc);
    }
    tt.agg = a;
    return;
  }
  Piece a = piece_identity();
  int nw = 0;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    Piece pc;
    nw += (classify_at(tt, i, pc) == 2);
    a = piece_combine(a, pc);
  }
  tt.agg = a;
  tt.nwin = nw;
}

// Composite resolver scan element: the segmented piece over window-free
// tiles, the windowed-tile rank and the staged-window offset, in one scan.
struct ResScan {
  Piece pc;
  int rank, wofs;
};

__device__ __forceinline__ ResScan res_combine(const ResScan& a, const ResScan& b) {
  return ResScan{piece_combine(a.pc, b.pc), a.rank + b.rank, a.wofs + b.wofs};
}

__device__ __forceinline__ ResScan shfl_up_res(const ResScan& v, int o) {
  return ResScan{shfl_up_piece(v.pc, o), __shfl_up_sync(0xffffffffu, v.rank, o),
                 __shfl_up_sync(0xffffffffu, v.wofs, o)};
}

// Block-wide exclusive scan of ResScan (fixed shape); total in `tot`.
__device__ __forceinline__ ResScan block_excl_scan_res(ResScan v, ResScan& tot, ResScan* sw) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const ResScan id{piece_identity(), 0, 0};
  ResScan x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const ResScan y = shfl_up_res(x, o);
    if (lane >= o) x = res_combine(y, x);
  }
  if (lane == 31) sw[w] = x;
  __syncthreads();
  if (w == 0) {
    ResScan t = lane < kWarps ? sw[lane] : id;
#pragma unroll
    for (int o = 1; o < kWarps; o <<= 1) {
      const ResScan y = shfl_up_res(t, o);
      if (lane >= o) t = res_combine(y, t);
    }
    if (lane < kWarps) sw[kWarps + lane] = t;
  }
  __syncthreads();
  ResScan ex = shfl_up_res(x, 1);
  if (lane == 0) ex = id;
  if (w) ex = res_combine(sw[kWarps + w - 1], ex);
  tot = sw[2 * kWarps - 1];
  __syncthreads();
  return ex;
}

constexpr int kResolveWin = 256;    // windows staged in smem by the resolver
constexpr int kMaxSuper = 16;       // tiles per resolver thread (super-tile)
constexpr int kStageSuper = 32;     // windowed super-tiles whose headers are staged

struct ResolverSmem {
  TileWin win[kResolveWin];
  const TileWin* wsrc[kResolveWin];
  TileHdr hdr[kStageSuper * kMaxSuper];
  Piece excl[kThreads];
  double out[kThreads];
  int wlist[kThreads];
  ResScan rsw[2 * kWarps];
  double carry;
  int bad;
};

__device__ __forceinline__ TileHdr load_hdr(const TileHdr* hdr, int ti) {
  TileHdr h;
  h.nwin = __ldcg(&hdr[ti].nwin);
  h.tail_e = __ldcg(&hdr[ti].tail_e);
  h.tail_d0 = __ldcg(&hdr[ti].tail_d0);
  h.tail_d1 = __ldcg(&hdr[ti].tail_d1);
  return h;
}

struct WinSmem {
  Piece wp[kResolveWin];   // piece from the previous window (or chain start) to this window
  double wg[kResolveWin];  // the window element
  double sa[kResolveWin];  // exact sum after the window
  int wt[kResolveWin], wk[kResolveWin];
  ResScan rsw[2 * kWarps];
  int bad;
};

// The exact chain at WINDOW granularity, one block (the common case). Each
// thread owns K consecutive tiles; a tile is the segmented element
// (tail piece, head flag = has windows), so one block scan gives every
// thread the piece from the last window before its tiles. Then: (1) threads
// lay out every window's piece-since-the-previous-window in shared memory,
// in global order; (2) ONE thread applies the windows serially (one exact
// piece application and one real IEEE add each, ~log2 N of them); (3) every
// thread derives its tiles' exact (start, end) from the window sums. Returns
// false, having written nothing, when a tile overflowed its window list or
// the windows exceed the staging area: the caller then runs resolve_chain.
template <int ITEMS>
__device__ bool resolve_windows(const Ctx& c, const TileHdr* hdr, const TileWin* win, double* win_after,
                                double2* tile_info, int ntiles, WinSmem& ws) {
  const int K = (ntiles + kThreads - 1) / kThreads;
  const int tb = min(static_cast<int>(threadIdx.x) * K, ntiles), te = min(tb + K, ntiles);
  Piece agg = piece_identity();
  int nw = 0, ovf = 0;
  for (int t0 = tb; t0 < te; t0 += 8) {
    TileHdr h[8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (t0 + i < te) h[i] = load_hdr(hdr, t0 + i);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (t0 + i < te) {
        ovf += h[i].nwin < 0;
        nw += max(h[i].nwin, 0);
        agg = piece_combine(agg, Piece{h[i].tail_d0, h[i].tail_d1, h[i].tail_e, h[i].nwin != 0});
      }
    }
  }
  ResScan tot;
  const ResScan ex = block_excl_scan_res(ResScan{agg, ovf, nw}, tot, ws.rsw);
  if (tot.rank > 0 || tot.wofs > kResolveWin) return false;  // uniform
  if (threadIdx.x == 0) {
    ws.bad = 0;
    c.st->tstamp[3] = c.st->tstamp[4] = global_ns();
    c.st->tstamp[7] = static_cast<unsigned long long>(tot.wofs);
  }
  {
    Piece E = ex.pc;
    int wo = ex.wofs;
    for (int t = tb; t < te; ++t) {
      const TileHdr h = load_hdr(hdr, t);
      for (int k = 0; k < h.nwin; ++k) {
        const TileWin* gw = win + static_cast<size_t>(t) * kMaxWin + k;
        Piece pc{__ldcg(&gw->d0), __ldcg(&gw->d1), __ldcg(&gw->e), 0};
        if (k == 0) pc = piece_combine(E, pc);
        ws.wp[wo] = pc;
        ws.wg[wo] = __ldcg(&gw->g);
        ws.wt[wo] = t;
        ws.wk[wo] = k;
        ++wo;
      }
      E = piece_combine(E, Piece{h.tail_d0, h.tail_d1, h.tail_e, h.nwin != 0});
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    c.st->tstamp[5] = global_ns();
    double s = 0.0;
    bool ok = true;
    for (int w = 0; w < tot.wofs; ++w) {
      ok &= piece_apply(ws.wp[w], s);
      s = s + ws.wg[w];  // the window element: a real IEEE add, as acc += g[i]
      ws.sa[w] = s;
    }
    if (!ok) ws.bad = 1;
    c.st->tstamp[6] = global_ns();
  }
  __syncthreads();
  for (int w = threadIdx.x; w < tot.wofs; w += kThreads)
    win_after[static_cast<size_t>(ws.wt[w]) * kMaxWin + ws.wk[w]] = ws.sa[w];
  {
    double s = ex.wofs > 0 ? ws.sa[ex.wofs - 1] : 0.0;
    bool ok = piece_apply(ex.pc, s);
    int wo = ex.wofs;
    for (int t = tb; t < te; ++t) {
      const TileHdr h = load_hdr(hdr, t);
      const double s_in = s;
      if (h.nwin > 0) {
        wo += h.nwin;
        s = ws.sa[wo - 1];
      }
      ok &= piece_apply(Piece{h.tail_d0, h.tail_d1, h.tail_e, 0}, s);
      double s_end = s;
      if (t == ntiles - 1) {
        c.st->total_mass = s_end;
        s_end = (s_end < 1.0) ? 1.0 : s_end;  // guard the last bin (filter.cpp:168)
      }
      tile_info[t] = make_double2(s_in, s_end);
    }
    if (!ok) ws.bad = 1;
  }
  __syncthreads();
  if (threadIdx.x == 0 && ws.bad) atomicOr(&c.st->error, kErrInternal);
  return true;
}

// Fallback (a tile overflowed its window list, or > kResolveWin windows):
// the exact chain over tiles, one block. Each thread owns a run of K
// consecutive tiles (a super-tile); window-free super-tiles compose in a
// segmented monoid scan, the windowed ones are walked in order by one
// thread with real IEEE adds at the windows; everything that walk touches
// is staged in shared memory. Used for the single handle (own tiles) and,
// sharded, for all shards' tiles on every rank.
template <int ITEMS>
__device__ void resolve_chain(const Ctx& c, const TileHdr* hdr, const TileWin* win, double* win_after,
                              double2* tile_info, int ntiles, bool own_g, ResolverSmem& rs) {
  using TC = TileCfg<ITEMS>;
  const int K = min(kMaxSuper, (ntiles + kThreads - 1) / kThreads);
  if (threadIdx.x == 0) {
    rs.carry = 0.0;
    rs.bad = 0;
  }
  __syncthreads();
  for (int b0 = 0; b0 < ntiles; b0 += kThreads * K) {
    const int tb = b0 + threadIdx.x * K;
    const int te = min(tb + K, ntiles);
    // compose the super-tile (pure if none of its tiles has a window)
    Piece agg = piece_identity();
    bool windowed = false;
    int nw = 0;
    for (int ti = tb; ti < te; ++ti) {
      const TileHdr h = load_hdr(hdr, ti);
      if (h.nwin != 0) {
        windowed = true;
        nw += h.nwin > 0 ? h.nwin : 0;
      } else {
        agg = piece_combine(agg, Piece{h.tail_d0, h.tail_d1, h.tail_e, 0});
      }
    }
    ResScan mine{windowed ? Piece{0, 0, kNoBinade, 1} : agg, windowed ? 1 : 0, windowed ? nw : 0};
    ResScan tot;
    if (threadIdx.x == 0 && b0 == 0) c.st->tstamp[3] = global_ns();
    const ResScan ex = block_excl_scan_res(mine, tot, rs.rsw);
    const int nwt = tot.rank;
    if (threadIdx.x == 0 && b0 == 0) {
      c.st->tstamp[4] = global_ns();
      c.st->tstamp[7] = static_cast<unsigned long long>(nwt) * 100000ull + tot.wofs;
    }
    if (windowed) {
      rs.wlist[ex.rank] = threadIdx.x;
      rs.excl[ex.rank] = ex.pc;
      if (ex.rank < kStageSuper)
        for (int ti = tb; ti < te; ++ti) rs.hdr[ex.rank * kMaxSuper + (ti - tb)] = load_hdr(hdr, ti);
      int w = ex.wofs;  // record where the windows live; loaded cooperatively below
      for (int ti = tb; ti < te; ++ti) {
        const int n = __ldcg(&hdr[ti].nwin);
        for (int k = 0; k < n && w < kResolveWin; ++k, ++w) rs.wsrc[w] = win + static_cast<size_t>(ti) * kMaxWin + k;
      }
    }
    __syncthreads();
    for (int w = threadIdx.x; w < min(tot.wofs, kResolveWin); w += kThreads) rs.win[w] = *rs.wsrc[w];
    __syncthreads();
    if (threadIdx.x == 0 && b0 == 0) c.st->tstamp[5] = global_ns();
    if (threadIdx.x == 0) {
      // in-order walk over the windowed super-tiles of this chunk
      double seg = rs.carry;
      int wo = 0;
      bool ok = true;
      for (int r = 0; r < nwt; ++r) {
        const int st0 = b0 + rs.wlist[r] * K;
        const int st1 = min(st0 + K, ntiles);
        double s = seg;
        ok &= piece_apply(rs.excl[r], s);
        for (int ti = st0; ti < st1; ++ti) {
          const TileHdr wh = r < kStageSuper ? rs.hdr[r * kMaxSuper + (ti - st0)] : load_hdr(hdr, ti);
          const double s_in = s;
          if (wh.nwin < 0 && !own_g) {
            ok = false;  // window overflow in a remote tile: unsupported when sharded
          } else if (wh.nwin < 0) {
            // serial tile (window overflow): plain sequential sum, CDF written here
            const long long tbase = static_cast<long long>(ti) * TC::kTileT;
            const double lse = c.st->lse_g;
            for (int e = 0; e < TC::kTileT && tbase + e < c.N; ++e) {
              s = s + (c.gin ? __ldcg(&c.gin[tbase + e]) : exp(__ldcg(&c.lg[tbase + e]) - lse));
              c.cdf[tbase + e] = s;
            }
          } else {
            for (int k = 0; k < wh.nwin; ++k, ++wo) {
              TileWin tw;
              if (wo < kResolveWin) {
                tw = rs.win[wo];
              } else {
                const TileWin* gw = win + static_cast<size_t>(ti) * kMaxWin + k;
                tw.g = __ldcg(&gw->g);
                tw.e = __ldcg(&gw->e);
                tw.d0 = __ldcg(&gw->d0);
                tw.d1 = __ldcg(&gw->d1);
              }
              ok &= piece_apply(Piece{tw.d0, tw.d1, tw.e, 0}, s);
              s = s + tw.g;  // the window element: a real IEEE add, as acc += g[i]
              win_after[static_cast<size_t>(ti) * kMaxWin + k] = s;
            }
            ok &= piece_apply(Piece{wh.tail_d0, wh.tail_d1, wh.tail_e, 0}, s);
          }
          double s_end = s;
          if (ti == ntiles - 1) {
            c.st->total_mass = s_end;
            s_end = (s_end < 1.0) ? 1.0 : s_end;  // guard the last bin (filter.cpp:168)
          }
          tile_info[ti] = make_double2(s_in, s_end);
        }
        rs.out[r] = s;
        seg = s;
      }
      if (!ok) rs.bad = 1;
      if (b0 == 0) c.st->tstamp[6] = global_ns();
    }
    __syncthreads();
    if (tb < te && !windowed) {
      double s = ex.rank > 0 ? rs.out[ex.rank - 1] : rs.carry;
      bool ok = piece_apply(ex.pc, s);
      for (int ti = tb; ti < te; ++ti) {
        const TileHdr h = load_hdr(hdr, ti);
        const double s_in = s;
        ok &= piece_apply(Piece{h.tail_d0, h.tail_d1, h.tail_e, 0}, s);
        double s_end = s;
        if (ti == ntiles - 1) {
          c.st->total_mass = s_end;
          s_end = (s_end < 1.0) ? 1.0 : s_end;  // guard the last bin (filter.cpp:168)
        }
        tile_info[ti] = make_double2(s_in, s_end);
      }
      if (!ok) rs.bad = 1;
    }
    __syncthreads();
    // the chunk's exact end value: the last super-tile's end
    if (threadIdx.x == 0) {
      const int last = min(b0 + kThreads * K, ntiles) - 1;
      const double2 v = __ldcg(&tile_info[last]);
      rs.carry = (last == ntiles - 1) ? c.st->total_mass : v.y;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && rs.bad) atomicOr(&c.st->error, kErrInternal);
}

template <int ITEMS>
union PiecesSmem {
  double g[TileCfg<ITEMS>::kSmem];
  ResolverSmem rs;
  WinSmem ws;
};

// S2: fitness g = exp(lg - lse) (fitness_weights, filter.cpp:154), written
// once; the approximate prefix from the tile offsets computed in the predict
// kernel's tail (no look-back); classification, windows and tile records;
// the per-thread handoff for S3. SHARDED = 0: the last block resolves the
// exact chain (single handle); 1: records only (every rank resolves all
// shards' records after the allgather, k_resolve_global).
template <int ITEMS, int SHARDED>
__global__ void __launch_bounds__(kThreads) k_scan_pieces(Ctx c) {
  using TC = TileCfg<ITEMS>;
  __shared__ PiecesSmem<ITEMS> sm;
  __shared__ ScanScratch sw;
  __shared__ int s_last;
  if (grid_error(c)) return;
  if (!SHARDED && threadIdx.x == 0 && blockIdx.x == 0) c.st->tstamp[0] = global_ns();
  const int t = blockIdx.x;
  const long long base = static_cast<long long>(t) * TC::kTileT;
  const double lse = c.st->lse_g;
  const double pre = c.shard_off[0] + __ldcg(&c.tile_pre[t]);
  const long long cpre = static_cast<long long>(c.shard_off[1]) + __ldcg(&c.tile_cnt_pre[t]);
  ThreadTile<ITEMS> tt;
  {
    // all ITEMS loads in flight first, then the exps
    const double* src = c.gin ? c.gin : c.lg;
    double x[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const long long k = base + i * kThreads + threadIdx.x;
      x[i] = k < c.N ? __ldcs(&src[k]) : 0.0;
    }
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int e = i * kThreads + threadIdx.x;
      const long long k = base + e;
      double g = 0.0;
      if (k < c.N) g = c.gin ? x[i] : exp(x[i] - lse);  // S3 recomputes it (bitwise)
      sm.g[TC::sidx(e)] = g;
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) tt.g[i] = sm.g[TC::sidx(threadIdx.x * ITEMS + i)];
  SumCnt mine{0.0, 0};
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    mine.s += tt.g[i];
    mine.c += (tt.g[i] != 0.0);
  }
  SumCnt tot;
  const SumCnt ex = block_excl_scan_sc(mine, tot, sw.sc);
  tt.p[0] = pre + ex.s;
  tt.cnt0 = cpre + ex.c;
  chunk_analyse<ITEMS>(tt);
  const Piece carry = block_excl_scan_piece(tt.agg, sw.pc);
  int win_total;
  const int win_excl = block_excl_scan_int(tt.nwin, win_total, sw.si);
  const bool overflow = win_total > kMaxWin;
  c.trec[static_cast<size_t>(t) * kThreads + threadIdx.x] =
      ThreadRec{tt.p[0], tt.cnt0, carry.d0, carry.d1, carry.e, carry.flag, win_excl, 0};
  if (tt.nwin > 0 && !overflow) {
    Piece acc = carry;
    int w = win_excl;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      Piece pc;
      const int kind = classify_at(tt, i, pc);
      if (kind == 2) {
        TileWin tw;
        tw.g = tt.g[i];
        tw.e = acc.e;
        tw.local = threadIdx.x * ITEMS + i;
        tw.d0 = acc.d0;
        tw.d1 = acc.d1;
        c.win[static_cast<size_t>(t) * kMaxWin + w] = tw;
        ++w;
      }
      acc = piece_combine(acc, pc);
    }
  }
  if (threadIdx.x == kThreads - 1) {
    const Piece acc = piece_combine(carry, tt.agg);
    c.hdr[t] = TileHdr{overflow ? -1 : win_total, acc.e, acc.d0, acc.d1};
  }
  if (SHARDED) return;
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
  if (threadIdx.x == 0) c.st->tstamp[1] = global_ns();
  if (!resolve_windows<ITEMS>(c, c.hdr, c.win, c.win_after, c.tile_info, c.ntiles, sm.ws))
    resolve_chain<ITEMS>(c, c.hdr, c.win, c.win_after, c.tile_info, c.ntiles, true, sm.rs);
  if (threadIdx.x == 0) c.st->tstamp[2] = global_ns();
}

// Sharded: every rank resolves the exact chain over ALL shards' tiles.
template <int ITEMS>
__global__ void __launch_bounds__(kThreads) k_resolve_global(Ctx c) {
  __shared__ union {
    ResolverSmem rs;
    WinSmem ws;
  } sm;
  if (grid_error(c)) return;
  if (!resolve_windows<ITEMS>(c, c.ghdr, c.gwin, c.gwin_after, c.gtile_info, c.gntiles, sm.ws))
    resolve_chain<ITEMS>(c, c.ghdr, c.gwin, c.gwin_after, c.gtile_info, c.gntiles, false, sm.rs);
}

// S3: exact per-element CDF (from the S2 per-thread handoff: no block
// scans), per-tile local guide and the coarse guide.
template <int ITEMS>
__global__ void __launch_bounds__(kThreads, (ITEMS == 8 ? 4 : 2)) k_scan_cdf(Ctx c) {
  using TC = TileCfg<ITEMS>;
  __shared__ double sg[TC::kSmem];
  if (grid_error(c)) return;
  const int t = blockIdx.x;
  const long long base = static_cast<long long>(t) * TC::kTileT;
  const int nwin = __ldcg(&c.hdr[t].nwin);
  const double2 ti = __ldcg(&c.tile_info[t]);
  const int valid = static_cast<int>(min(static_cast<long long>(TC::kTileT), c.N - base));
  double vals[ITEMS];
  if (nwin >= 0) {
    ThreadTile<ITEMS> tt;
    // g = exp(lg - lse) recomputed exactly as S2 did (same inputs, same op)
    const double lse = c.st->lse_g;
    const double2* gsrc = reinterpret_cast<const double2*>((c.gin ? c.gin : c.lg) + base + threadIdx.x * ITEMS);
#pragma unroll
    for (int i = 0; i < ITEMS / 2; ++i) {
      const double2 v = __ldcs(gsrc + i);
      const int e = threadIdx.x * ITEMS + 2 * i;
      tt.g[2 * i] = e < valid ? v.x : 0.0;
      tt.g[2 * i + 1] = e + 1 < valid ? v.y : 0.0;
    }
    if (!c.gin) {
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        const int e = threadIdx.x * ITEMS + i;
        tt.g[i] = e < valid ? exp(tt.g[i] - lse) : 0.0;
      }
    }
    const ThreadRec tr = c.trec[static_cast<size_t>(t) * kThreads + threadIdx.x];
    tt.p[0] = tr.p0;
    tt.cnt0 = tr.cnt0;
    chunk_analyse<ITEMS>(tt);
    const Piece carry{tr.d0, tr.d1, tr.e, tr.flag};
    int w = tr.win_excl;
    double seg = w > 0 ? __ldcg(&c.win_after[static_cast<size_t>(t) * kMaxWin + w - 1]) : ti.x;
    bool ok = true;
    if (tt.uniform_e != kNoBinade || tt.lc[ITEMS] == 0) {
      // no window in this chunk: one exact base value, then integer steps
      double s0 = seg;
      ok &= piece_apply(carry, s0);
      if (tt.lc[ITEMS] == 0) {
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) vals[i] = s0;
      } else {
        const int e = tt.uniform_e;
        const UlpScale scale = ulp_scale(e);
        long long m = static_cast<long long>(scale2(s0, 52 - e));
        const long long m_hi = 1LL << 53;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
          if (tt.g[i] != 0.0) {
            long long d0, d1;
            run_delta(tt.g[i], scale, d0, d1);
            m += (m & 1) ? d1 : d0;
          }
          vals[i] = scale2(static_cast<double>(m), e - 52);
        }
        ok &= m < m_hi && binade_of(s0) == e;  // self-check of the bound
      }
    } else {
      Piece acc = carry;
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        Piece pc;
        const int kind = classify_at(tt, i, pc);
        acc = piece_combine(acc, pc);
        double sk = seg;
        if (kind == 2) {
          seg = __ldcg(&c.win_after[static_cast<size_t>(t) * kMaxWin + w]);
          ++w;
          sk = seg;
        } else {
          ok &= piece_apply(acc, sk);
        }
        vals[i] = sk;
      }
    }
    if (!ok) atomicOr(&c.st->error, kErrInternal);
  } else {
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int e = threadIdx.x * ITEMS + i;
      vals[i] = e < valid ? __ldcg(&c.cdf[base + e]) : 0.0;
    }
  }
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int e = threadIdx.x * ITEMS + i;
    double v = vals[i];
    if (c.n0 + base + e == c.n_glob - 1) v = (v < 1.0) ? 1.0 : v;  // filter.cpp:168
    if (e >= valid) v = INFINITY;
    sg[TC::sidx(e)] = v;
  }
  __syncthreads();
#pragma unroll 4
  for (int i = 0; i < ITEMS; ++i) {
    const int e = i * kThreads + threadIdx.x;
    if (e < valid) c.cdf[base + e] = sg[TC::sidx(e)];
  }
  // Segment ends (a segment = 8 elements, one 64-byte burst): seg_end[j] is
  // the exact CDF at the segment's last element. They and the guide below
  // are small enough to stay in L2, so the ancestor search reads HBM once
  // (the one 64/128-byte CDF segment) before the record gather.
  constexpr int SPT = ITEMS >> kSegLog2;  // segments per thread
  constexpr int SPB = SPT * kThreads;     // segments per tile
  __shared__ double send[SPB];
#pragma unroll
  for (int q = 0; q < SPT; ++q) {
    const int i0 = threadIdx.x * ITEMS + (q << kSegLog2);
    const double v = i0 < valid ? sg[TC::sidx(min(i0 + (1 << kSegLog2) - 1, valid - 1))] : INFINITY;
    send[threadIdx.x * SPT + q] = v;
    if (i0 < valid) c.seg_end[static_cast<long long>(t) * SPB + threadIdx.x * SPT + q] = v;
  }
  __syncthreads();
  // guide: bucket b (edge b/B) -> first segment whose end exceeds b/B, for
  // the buckets with start <= b/B < end of this tile (binary search over the
  // tile's 256 segment ends in shared memory; bucket work spread over threads)
  const double B1 = scale2(1.0, c.coarse_bits);
  const long long nb = 1LL << c.coarse_bits;
  long long b_lo = static_cast<long long>(ceil(ti.x * B1));
  long long b_hi = ti.y >= 1.0 ? nb - 1 : static_cast<long long>(ceil(ti.y * B1)) - 1;
  b_lo = max(b_lo, 0LL);
  b_hi = min(b_hi, nb - 1);
  if (t == 0) b_lo = static_cast<long long>(floor(ti.x * B1));  // a shard's first tile also owns
                                                              // the bucket its range starts in
  for (long long b = b_lo + threadIdx.x; b <= b_hi; b += kThreads) {
    const double x = scale2(static_cast<double>(b), -c.coarse_bits);
    int lo = 0, len = SPB;
    while (len > 0) {
      const int half = len >> 1;
      if (!(x < send[lo + half])) {
        lo += half + 1;
        len -= half + 1;
      } else {
        len = half;
      }
    }
    c.coarse[b] = static_cast<unsigned>(t) * SPB + static_cast<unsigned>(min(lo, SPB - 1));
  }
}

void launch_scan(const Ctx& c, int ntiles, cudaStream_t st, int which) {
  const bool small = c.tile_log2 == 11;
  switch (which) {
    case 1:
      if (small) k_scan_pieces<8, 0><<<ntiles, kThreads, 0, st>>>(c);
      else k_scan_pieces<16, 0><<<ntiles, kThreads, 0, st>>>(c);
      break;
    case 2:
      if (small) k_scan_cdf<8><<<ntiles, kThreads, 0, st>>>(c);
      else k_scan_cdf<16><<<ntiles, kThreads, 0, st>>>(c);
      break;
    case 4:
      if (small) k_scan_pieces<8, 1><<<ntiles, kThreads, 0, st>>>(c);
      else k_scan_pieces<16, 1><<<ntiles, kThreads, 0, st>>>(c);
      break;
    case 5:
      if (small) k_resolve_global<8><<<1, kThreads, 0, st>>>(c);
      else k_resolve_global<16><<<1, kThreads, 0, st>>>(c);
      break;
  }
}

// Survival of the fittest (filter.cpp:169-176, 330-335): slot n draws its
// uniform, finds its ancestor in the exact CDF and gathers the ancestor's
// record and predictor log-likelihood into slot order, so K3 streams them
// coalesced. Latency-bound (dependent random loads), so it runs as its own
// small-footprint, high-occupancy kernel.
template <int H>  // 16-byte parts per payload (R / 2 + 1)
__global__ void __launch_bounds__(kThreads) k_serve(Ctx c) {
  if (grid_error(c)) return;
  const long long n = static_cast<long long>(blockIdx.x) * kThreads + threadIdx.x;
  const double u = n < c.N ? resample_uniform(c.seed, c.sp->j, n) : -1.0;
  const unsigned a = find_ancestor_warp(c, u);
  if (n < c.N) c.anc[n] = a;
  // warp-cooperative gather: consecutive lanes move consecutive 16-byte
  // parts of the warp's 32 payloads (coalesced stores, whole-record loads)
  const int lane = threadIdx.x & 31;
  const long long wbase = n - lane;
  const double2* rec = reinterpret_cast<const double2*>(c.rec[c.st->cur]);
  double2* pay = reinterpret_cast<double2*>(c.payload);
#pragma unroll
  for (int it = 0; it < H; ++it) {
    const int idx = lane + 32 * it;
    const int slot = idx / H, part = idx - slot * H;
    const unsigned as = __shfl_sync(0xffffffffu, a, slot);
    const long long ns = wbase + slot;
    if (ns < c.N) {
      double2 v;
      if (part < H - 1)
        v = __ldg(rec + static_cast<long long>(as) * (H - 1) + part);
      else
        v = make_double2(__ldg(&c.llbar[as]), static_cast<double>(as));
      pay[ns * H + part] = v;
    }
  }
}

void launch_serve(const Ctx& c, int grid, cudaStream_t st) {
  switch (c.R / 2 + 1) {
    case 2: k_serve<2><<<grid, kThreads, 0, st>>>(c); break;
    case 3: k_serve<3><<<grid, kThreads, 0, st>>>(c); break;
    case 4: k_serve<4><<<grid, kThreads, 0, st>>>(c); break;
    case 5: k_serve<5><<<grid, kThreads, 0, st>>>(c); break;
    case 7: k_serve<7><<<grid, kThreads, 0, st>>>(c); break;
    default: break;
  }
}

__global__ void __launch_bounds__(kThreads) k_finish_lse(Ctx c, const double* gp, int ngroups) {
  __shared__ double scratch[kWarps * 2];
  __shared__ double fin[2];
  if (grid_error(c)) return;
  __shared__ double s_lse;
  combine_partials<1, false>(gp, ngroups, fin, scratch);
  __syncthreads();
  if (threadIdx.x == 0) {
    const double mx = fin[0];
    const double lse = isfinite(mx) ? mx + log(fin[1]) : kNegInf;
    c.st->lse_g = lse;
    if (!isfinite(lse)) atomicOr(&c.st->error, kErrPredict);
    s_lse = lse;
  }
  __syncthreads();
  // local tile prefixes + this shard's total (allgathered next, phase B)
  if (isfinite(s_lse)) tile_prefixes(c, s_lse);
}

// ---- sharded ancestor migration (pull model) ---------------------------
// Rank r owns the exact-CDF range [start_r, end_r) of its tiles; the global
// upper_bound(cdf, u) lands on rank r iff u is in that range. Every rank draws
// the uniforms of ALL global slots (keyed streams: identical numbers on every
// rank), serves those in its range from its own exact CDF, and ships
// {record, ll_bar, ancestor, destination slot} to the slot's owner.
constexpr int kShardPW = 4;  // extra doubles of a migration payload beyond the record

__device__ __forceinline__ int serving_rank(const Ctx& c, double u) {
  const int ntl = c.ntiles;
  for (int r = 0; r < c.world; ++r) {
    const double lo = c.gtile_info[r * ntl].x;
    const double hi = c.gtile_info[(r + 1) * ntl - 1].y;
    if (u >= lo && u < hi) return r;
  }
  return c.world - 1;  // unreachable: the last range ends at the guarded cdf >= 1 > u
}

// Every rank walks all global slots (a warp = 32 consecutive slots, all of one
// destination since N_local is a multiple of 16384): the slot's serving rank
// from the allgathered exact shard ranges feeds the migration count matrix
// (identical on every rank: cnt[r * W + d] = slots of rank d served by r;
// one atomic per group of lanes with the same server), and the slots this
// rank serves are searched and their payloads written (one atomic per warp).
__global__ void __launch_bounds__(kThreads) k_serve_sharded(Ctx c, double* sendbuf, unsigned* send_cnt,
                                                            unsigned* cnt) {
  if (grid_error(c)) return;
  const int W = c.R + kShardPW;
  const long long cap = c.N;  // per destination: at most its N_local slots
  const int lane = threadIdx.x & 31;
  for (long long ng = static_cast<long long>(blockIdx.x) * kThreads + threadIdx.x; ng < c.n_glob;
       ng += static_cast<long long>(gridDim.x) * kThreads) {
    const double u = resample_uniform(c.seed, c.sp->j, ng);
    const int r = serving_rank(c, u);
    const int dest = static_cast<int>(ng / c.N);
    const unsigned grp = __match_any_sync(0xffffffffu, r);
    if (lane == __ffs(grp) - 1) atomicAdd(&cnt[r * c.world + dest], static_cast<unsigned>(__popc(grp)));
    const bool mine = r == c.rank;
    const unsigned m = __ballot_sync(0xffffffffu, mine);
    if (!m) continue;
    const int leader = __ffs(m) - 1;
    unsigned base = 0;
    if (lane == leader) base = atomicAdd(&send_cnt[dest], static_cast<unsigned>(__popc(m)));
    base = __shfl_sync(0xffffffffu, base, leader);
    const unsigned pos = base + static_cast<unsigned>(__popc(m & ((1u << lane) - 1u)));
    // warp-cooperative search (lanes not served here pass u = -1) and gather:
    // consecutive lanes move consecutive 16-byte parts of the served payloads
    const unsigned a = find_ancestor_warp(c, mine ? u : -1.0);
    const int H = c.R / 2 + kShardPW / 2;  // 16-byte parts per payload
    const double2* rec = reinterpret_cast<const double2*>(c.rec[c.st->cur]);
    for (int idx = lane; idx < 32 * H; idx += 32) {
      const int src_lane = idx / H, part = idx - src_lane * H;
      const unsigned as = __shfl_sync(0xffffffffu, a, src_lane);
      const unsigned ps = __shfl_sync(0xffffffffu, pos, src_lane);
      if (!((m >> src_lane) & 1u)) continue;
      double2 v;
      if (part < c.R / 2)
        v = __ldg(rec + static_cast<long long>(as) * (c.R / 2) + part);
      else if (part == c.R / 2)
        v = make_double2(__ldg(&c.llbar[as]), static_cast<double>(c.n0 + as));
      else
        v = make_double2(static_cast<double>(ng - lane + src_lane - dest * c.N), 0.0);
      reinterpret_cast<double2*>(sendbuf + (dest * cap + ps) * W)[part] = v;
    }
  }
}

__global__ void __launch_bounds__(kThreads) k_place(Ctx c, const double* recvbuf, long long count) {
  if (grid_error(c)) return;
  const long long i = static_cast<long long>(blockIdx.x) * kThreads + threadIdx.x;
  if (i >= count) return;
  const int W = c.R + kShardPW;
  const double2* src = reinterpret_cast<const double2*>(recvbuf + i * W);
  const long long slot = static_cast<long long>(recvbuf[i * W + c.R + 2]);
  double2* dst = reinterpret_cast<double2*>(c.payload + slot * (c.R + 2));
  for (int k = 0; k < c.R / 2 + 1; ++k) dst[k] = src[k];
  c.anc[slot] = static_cast<unsigned>(recvbuf[i * W + c.R + 1]);
}

// Global approximate offset of this shard (rank order) from the allgathered
// (sum, count) pairs.
// Every rank's search tables and records, as seen from this GPU: local
// pointers for itself, CUDA IPC mappings (NVLink peer memory) for the others.
constexpr int kMaxRanks = 8;
struct PeerTable {
  const double* rec0[kMaxRanks];
  const double* rec1[kMaxRanks];
  const double* llbar[kMaxRanks];
  const double* cdf[kMaxRanks];
  const double* seg_end[kMaxRanks];
  const unsigned* coarse[kMaxRanks];
};

// The migration as one pull kernel over peer memory (no count exchange, no
// host sync): slot n's uniform, its serving rank from the exact global shard
// ranges, the exact search in that rank's CDF tables and the gather of that
// rank's record and ll_bar straight into this rank's slot-ordered payload.
__global__ void __launch_bounds__(kThreads) k_pull(Ctx c, PeerTable pt) {
  if (grid_error(c)) return;
  const long long n = static_cast<long long>(blockIdx.x) * kThreads + threadIdx.x;
  if (n >= c.N) return;
  const double u = resample_uniform(c.seed, c.sp->j, c.n0 + n);
  const int r = serving_rank(c, u);
  const int ntl = c.ntiles;
  SearchView v{pt.coarse[r], pt.seg_end[r], pt.cdf[r], c.gtile_info[(r + 1) * ntl - 1].y};
  const unsigned a = find_ancestor_view(c, v, u);
  const double* rec = (c.st->cur ? pt.rec1[r] : pt.rec0[r]) + static_cast<long long>(a) * c.R;
  const int H = c.R / 2;
  const double2* src = reinterpret_cast<const double2*>(rec);
  double2* dst = reinterpret_cast<double2*>(c.payload + n * (c.R + 2));
  for (int i = 0; i < H; ++i) dst[i] = __ldcg(src + i);
  const long long ga = static_cast<long long>(r) * c.N + a;
  dst[H] = make_double2(__ldcg(&pt.llbar[r][a]), static_cast<double>(ga));
  c.anc[n] = static_cast<unsigned>(ga);
}

__global__ void k_shard_offset(Ctx c, const double* gathered) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double s = 0.0, n = 0.0;
  for (int r = 0; r < c.rank; ++r) {
    s += gathered[2 * r];
    n += gathered[2 * r + 1];
  }
  c.shard_off[0] = s;
  c.shard_off[1] = n;
}

// Injected-fitness parity path (pfsmc_gpu_resample_from_g): tile sums of
// the given g (in place of the predict kernel's block partials), then the
// same tile prefixes with lse = 0.
__global__ void __launch_bounds__(kThreads) k_gin_tiles(Ctx c) {
  __shared__ double scratch[kWarps * 2];
  const long long base = static_cast<long long>(blockIdx.x) << c.tile_log2;
  const int tile = 1 << c.tile_log2;
  double s = 0.0;
  int n = 0;
  for (int e = threadIdx.x; e < tile; e += kThreads) {
    const long long k = base + e;
    const double g = k < c.N ? c.gin[k] : 0.0;
    s += g;
    n += (g != 0.0);
  }
  double v[2] = {s, static_cast<double>(n)};
  block_sums<2>(v, scratch);  // fixed-order tree; counts are exact small integers
  if (threadIdx.x == 0) {
    c.trel[blockIdx.x] = v[0];
    c.tile_cnt_pre[blockIdx.x] = static_cast<long long>(v[1]);
  }
  const int ngroups = (c.ntiles * (tile / kThreads) + kGroup - 1) / kGroup;
  for (int g = blockIdx.x * kThreads + threadIdx.x; g < ngroups; g += gridDim.x * kThreads) c.gpart[2 * g] = 0.0;
}

__global__ void __launch_bounds__(kThreads) k_gin_prefix(Ctx c) {
  if (threadIdx.x == 0) c.st->lse_g = 0.0;
  tile_prefixes(c, 0.0);
}

// ---- BASELINE config 5: resample / reduction bandwidth microbenchmark ----
// One iteration over the resident 64-byte records {x[4], h[2], theta[2]}:
// log-sum-exp of lw (+ the exact scan's tile offsets), the weighted 2x2
// parameter covariance, the exact multinomial resampling and the gather of
// the ancestors' records into the next buffer.
__global__ void __launch_bounds__(kThreads) k_c5_weights(Ctx c, double sigma, unsigned long long key) {
  const long long n = static_cast<long long>(blockIdx.x) * kThreads + threadIdx.x;
  if (n >= c.N) return;
  double z[1];
  stream_normals<1>(c.seed, key, c.n0 + n, kInit, z);
  c.lw[n] = sigma * z[0];
}

// One pass over the resident particles computes everything the iteration
// reduces: the log-sum-exp of lw, the weighted 2x2 parameter covariance
// (weighted_mean_cov, linalg.cpp:389-432, about the previous mean) and the
// exact scan's tile offsets. A grid of a few blocks per SM loops over the
// exact-CDF tiles; each thread's ITEMS (lw, theta) loads are all in flight
// before the tile's partial: M_t = max lw, then sums of e = exp(lw - M_t)
// times (1, d0, d1, d0 d0, d0 d1, d1 d1) and the finite count. The block
// folds its tiles in order (combine_partials' rescaling rule); the last block
// combines the block partials in a fixed order. Bitwise reproducible.
template <int ITEMS>
__global__ void __launch_bounds__(kThreads) k_c5_stats(Ctx c) {
  constexpr int kTileT = ITEMS * kThreads;
  constexpr int V = 7;  // S, A0, A1, B00, B01, B11, finite count
  __shared__ double scratch[kWarps * V];
  __shared__ double fin[V];
  __shared__ int s_last;
  if (grid_error(c)) return;
  DevState& st = *c.st;
  const double k0 = st.mu[0], k1 = st.mu[1];
  const double* rec = c.rec[st.cur];
  for (int t = blockIdx.x; t < c.ntiles; t += gridDim.x) {
    const long long base = static_cast<long long>(t) * kTileT;
    double x[ITEMS];
    double2 th[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const long long k = base + i * kThreads + threadIdx.x;
      x[i] = k < c.N ? __ldcs(&c.lw[k]) : -INFINITY;
      th[i] = k < c.N ? __ldcs(reinterpret_cast<const double2*>(rec + k * c.R + 6)) : make_double2(0.0, 0.0);
    }
    double m = -INFINITY;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i)
      if (!isnan(x[i])) m = nan_free_max(m, x[i]);
    const double M = block_max(m, scratch);
    double v[V] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const double e = isnan(x[i]) ? NAN : (x[i] == -INFINITY ? 0.0 : exp(x[i] - M));
      const double d0 = th[i].x - k0, d1 = th[i].y - k1;
      v[0] += e;
      v[1] += e * d0;
      v[2] += e * d1;
      v[3] += e * (d0 * d0);
      v[4] += e * (d0 * d1);
      v[5] += e * (d1 * d1);
      v[6] += isfinite(x[i]) ? 1.0 : 0.0;
    }
    block_sums<V>(v, scratch);
    if (threadIdx.x == 0) {
      double* tp = c.part + static_cast<size_t>(c.ntiles + t) * V;  // per-tile partial (after the block slots)
      tp[0] = M;
#pragma unroll
      for (int k = 0; k < 6; ++k) tp[1 + k] = v[k];
      c.trel[t] = v[0];
      c.tile_m[t] = M;
      c.tile_cnt_pre[t] = static_cast<long long>(v[6]);
    }
  }
  if (threadIdx.x == 0) {
    // this block's partial over its tiles, in tile order
    double M = -INFINITY;
    for (int t = blockIdx.x; t < c.ntiles; t += gridDim.x) M = nan_free_max(M, c.tile_m[t]);
    double acc[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    for (int t = blockIdx.x; t < c.ntiles; t += gridDim.x) {
      const double* tp = c.part + static_cast<size_t>(c.ntiles + t) * V;
      const double w = tp[0] == -INFINITY ? 0.0 : exp(tp[0] - M);
#pragma unroll
      for (int k = 0; k < 6; ++k) acc[k] += w * tp[1 + k];
    }
    double* bp = c.part + static_cast<size_t>(blockIdx.x) * V;
    bp[0] = M;
#pragma unroll
    for (int k = 0; k < 6; ++k) bp[1 + k] = acc[k];
    __threadfence();
    const unsigned old = atomicAdd(&c.cnt_scan[3], 1u);
    s_last = (old == gridDim.x - 1);
    if (s_last) c.cnt_scan[3] = 0;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  combine_partials<6, false>(c.part, gridDim.x, fin, scratch);
  __syncthreads();
  __shared__ double s_lse;
  if (threadIdx.x == 0) {
    const double lse = isfinite(fin[0]) ? fin[0] + log(fin[1]) : kNegInf;
    st.lse_g = lse;
    if (!isfinite(lse)) atomicOr(&st.error, kErrPredict);
    s_lse = lse;
    const double S = fin[1];
    const double m0 = fin[2] / S, m1 = fin[3] / S;
    st.mu[0] = k0 + m0;
    st.mu[1] = k1 + m1;
    st.cov[0] = fin[4] / S - m0 * m0;
    st.cov[1] = st.cov[2] = fin[5] / S - m0 * m1;
    st.cov[3] = fin[6] / S - m1 * m1;
  }
  __syncthreads();
  if (isfinite(s_lse)) tile_prefixes(c, s_lse, c.tile_m);
}

// Survival of the fittest straight into the next record buffer (64-byte
// records: four lanes per record, eight records per load instruction).
__global__ void __launch_bounds__(kThreads) k_c5_serve(Ctx c, unsigned long long j) {
  if (grid_error(c)) return;
  const long long n = static_cast<long long>(blockIdx.x) * kThreads + threadIdx.x;
  const double u = n < c.N ? resample_uniform(c.seed, j, c.n0 + n) : -1.0;
  const unsigned a = find_ancestor_warp(c, u);
  if (n < c.N) c.anc[n] = a;
  const int lane = threadIdx.x & 31;
  const long long wbase = n - lane;
  const int cur = c.st->cur;
  const double2* src = reinterpret_cast<const double2*>(c.rec[cur]);
  double2* dst = reinterpret_cast<double2*>(c.rec[cur ^ 1]);
  const uint64_t pol = l2_policy_stream();
#pragma unroll
  for (int q = 0; q < 32; q += 8) {
    const int slot = q + lane / 4, part = lane & 3;
    const unsigned as = __shfl_sync(0xffffffffu, a, slot);
    const long long ns = wbase + slot;
    if (ns < c.N) st_hint(dst + ns * 4 + part, ld_hint(src + static_cast<long long>(as) * 4 + part, pol), pol);
  }
}

__global__ void k_flip(DevState* st) { st->cur ^= 1; }

// FP64 roofline denominator: 8 independent DFMA chains per thread.
__global__ void __launch_bounds__(kThreads) k_dfma_peak(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double acc = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc += x[i];
  if (acc == 12345.678) out[0] = acc;  // keeps the chains live
}

// Random-gather roofline: dst[n] = src[h(n)] for 64-byte records, h a
// bijective-free integer hash (splitmix64) — the same access shape as the
// resampling gather, without the search. Same warp-cooperative layout.
__global__ void __launch_bounds__(kThreads) k_gather_peak(const double2* __restrict__ src, double2* __restrict__ dst,
                                                          long long n_rec) {
  const long long n = static_cast<long long>(blockIdx.x) * kThreads + threadIdx.x;
  uint64_t z = static_cast<uint64_t>(n) + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  z ^= z >> 31;
  const unsigned a = static_cast<unsigned>(z % static_cast<uint64_t>(n_rec));
  const int lane = threadIdx.x & 31;
  const long long wbase = n - lane;
  const uint64_t pol = l2_policy_stream();
#pragma unroll
  for (int q = 0; q < 32; q += 8) {
    const int slot = q + lane / 4, part = lane & 3;
    const unsigned as = __shfl_sync(0xffffffffu, a, slot);
    const long long ns = wbase + slot;
    if (ns < n_rec) st_hint(dst + ns * 4 + part, ld_hint(src + static_cast<long long>(as) * 4 + part, pol), pol);
  }
}

__global__ void __launch_bounds__(kThreads) k_search_only(Ctx c) {
  if (grid_error(c)) return;
  const long long n = static_cast<long long>(blockIdx.x) * kThreads + threadIdx.x;
  const double u = n < c.N ? resample_uniform(c.seed, c.sp->j, n) : -1.0;
  const unsigned a = find_ancestor_warp(c, u);
  if (n < c.N) c.anc[n] = a;
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

static const char* kKernelNames = "k_predict,k_scan_pieces,k_scan_cdf,k_serve,k_update";
constexpr int kNumKernels = 5;

}  // namespace pfsmc_gpu

using namespace pfsmc_gpu;

// NCCL bound at run time: the process's already-loaded libnccl.so.2 (torch's)
// when there is one, so one NCCL instance serves both; nothing links it.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

const NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    auto sym = [&](auto& f, const char* name) { f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name)); };
    sym(a.GetUniqueId, "ncclGetUniqueId");
    sym(a.CommInitRank, "ncclCommInitRank");
    sym(a.CommDestroy, "ncclCommDestroy");
    sym(a.AllGather, "ncclAllGather");
    sym(a.Send, "ncclSend");
    sym(a.Recv, "ncclRecv");
    sym(a.GroupStart, "ncclGroupStart");
    sym(a.GroupEnd, "ncclGroupEnd");
    sym(a.GetErrorString, "ncclGetErrorString");
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllGather && a.Send && a.Recv && a.GroupStart &&
           a.GroupEnd && a.GetErrorString;
    return a;
  }();
  return api;
}

void NCK(ncclResult_t r) {
  if (r != ncclSuccess) throw std::runtime_error(std::string("nccl: ") + nccl_api().GetErrorString(r));
}

struct pfsmc_gpu_sampler {
  pfsmc_gpu_config cfg{};
  std::vector<uint64_t> obs;
  std::unique_ptr<KernelSet> ks;
  int d = 0, p = 0;
  long long N = 0;
  int grid = 0, ntiles = 0;
  int num_sms = 148;
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
  // sharding (pfsmc_gpu_create_shard)
  int rank = 0, world = 1;
  bool shard_api = false;  // created by pfsmc_gpu_create_shard
  ncclComm_t nccl = nullptr;  // pfsmc_gpu_shard_attach_nccl (native sharded step)
  PeerTable peers{};          // pfsmc_gpu_shard_attach_peers (migration over peer memory)
  bool have_peers = false;
  cudaGraphExec_t shard_graph = nullptr;  // the peer-memory step (graph with NCCL nodes)
  bool shard_graph_refused = false;
  std::vector<void*> ipc_opened;
  int ngroups_pred = 0, ngroups_upd = 0;
  double* gp_pred_all = nullptr;   // allgathered K1 group partials (world * ngroups * 2)
  double* gp_mom_all = nullptr;    // allgathered K3 group partials (world * ngroups * W)
  double* sums_all = nullptr;      // allgathered shard (sum, count) pairs
  double* sendbuf = nullptr;       // world * N_local payloads
  double* recvbuf = nullptr;       // N_local payloads
  unsigned* counts_dev = nullptr;  // [world] send + [world] recv
  unsigned* counts_all = nullptr;  // the W x W migration count matrix (k_serve_sharded)
  unsigned* counts_host = nullptr; // pinned mirror

  template <typename T>
  T* dalloc(size_t count) {
    void* p = nullptr;
    CK(cudaMalloc(&p, sizeof(T) * std::max<size_t>(count, 1)));
    allocs.push_back(p);
    return static_cast<T*>(p);
  }
  ~pfsmc_gpu_sampler() {
    if (shard_graph) cudaGraphExecDestroy(shard_graph);
    if (nccl) nccl_api().CommDestroy(nccl);
    for (void* p : ipc_opened) cudaIpcCloseMemHandle(p);
    if (graph) cudaGraphExecDestroy(graph);
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
    for (auto e : pending) cudaEventDestroy(e);
    for (void* a : allocs) cudaFree(a);
    if (sp_host) cudaFreeHost(sp_host);
    if (trace_host) cudaFreeHost(trace_host);
    if (st_host) cudaFreeHost(st_host);
    if (counts_host) cudaFreeHost(counts_host);
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
  sp.t_obs = t_obs;
  sp.h = h;
  if (s->cfg.adaptive) {
    if (!(t_obs > t_prev)) throw ConfigError("adaptive_bdf_interval: need t1 > t0");  // lmm.cpp:902-904
    sp.m = 0;
  } else {
    sp.m = step_count(t_prev, t_obs, h);
  }
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
  launch_scan(c, s->ntiles, st, 1);
  if (timed) CK(cudaEventRecord(ev[2], st));
  launch_scan(c, s->ntiles, st, 2);
  if (timed) CK(cudaEventRecord(ev[3], st));
  launch_serve(c, s->grid, st);
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

static pfsmc_gpu_status create_impl(const pfsmc_gpu_config* cfg, int rank, int world,
                                    pfsmc_gpu_sampler** out, bool shard_api = false) {
  return guarded([&] {
    *out = nullptr;
    if (world < 1 || rank < 0 || rank >= world) throw ConfigError("shard: need 0 <= rank < world");
    if (shard_api && cfg && cfg->particles % (static_cast<uint64_t>(world) * kGroup * kThreads) != 0)
      throw ConfigError("shard: particles must be a multiple of world * 16384");
    if (!cfg) throw ConfigError("null config");
    // PfConfig::validate (filter.cpp:45-74)
    if (cfg->particles == 0) throw ConfigError("config: particles must be >= 1");
    if (cfg->particles > (1ULL << 31)) throw ConfigError("config: particles must be < 2^31 per handle");
    if (!(cfg->shrink_a > 0.0 && cfg->shrink_a < 1.0))
      throw ConfigError("config: shrink factor a must lie in (0, 1)");
    if (!(cfg->sigma > 0.0)) throw ConfigError("config: observation noise sigma must be positive");
    if (cfg->adaptive) {
      if (!(cfg->rtol > 0.0)) throw ConfigError("config: rtol must be positive");  // filter.cpp:54-56
    } else {
      if (cfg->order < 1 || cfg->order > 3)
        throw ConfigError("scheme_coefficients: order must be 1, 2 or 3");
      if (cfg->family < 0 || cfg->family > 2) throw ConfigError("scheme_coefficients: unknown family");
    }
    if (cfg->n_obs > static_cast<uint64_t>(kMaxObs)) throw ConfigError("config: at most 8 observed components");
    auto s = std::make_unique<pfsmc_gpu_sampler>();
    s->cfg = *cfg;
    // adaptive: the variable-step BDF(1,2) kernels (order slot 0)
    s->ks = cfg->adaptive ? make_kernels(cfg->model, PFSMC_GPU_BDF, 0)
                          : make_kernels(cfg->model, cfg->family, cfg->order);
    if (!s->ks) throw ConfigError("unknown model id");
    if (cfg->model == MetabolicModel::ID && !(cfg->model_consts[5] > 0.0))
      throw ConfigError("metabolic model: tau must be positive");  // MetabolicModel ctor, models.cpp:104-108
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
    CK(cudaDeviceGetAttribute(&s->num_sms, cudaDevAttrMultiProcessorCount, cfg->device));
    CK(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
    s->rank = rank;
    s->world = world;
    s->N = static_cast<long long>(cfg->particles / world);
    s->grid = static_cast<int>((s->N + kThreads - 1) / kThreads);
    const int tile_log2 = s->N <= (1LL << 22) ? 11 : 12;
    s->ntiles = static_cast<int>((s->N + (1LL << tile_log2) - 1) >> tile_log2);
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
    for (int k = 0; k < 8; ++k) c.mconst[k] = cfg->model_consts[k];
    c.rtol = cfg->rtol;
    // guide buckets: about one per CDF segment (of the whole filter), <= 2^22
    const long long nseg_glob = std::max<long long>(1, static_cast<long long>(cfg->particles) >> kSegLog2);
    int cb = 6;
    while ((1LL << cb) < nseg_glob && cb < 22) ++cb;
    c.coarse_bits = cb;
    const size_t N = static_cast<size_t>(s->N);
    const size_t NT = static_cast<size_t>(s->ntiles);
    c.rec[0] = s->dalloc<double>(N * c.R);
    c.rec[1] = s->dalloc<double>(N * c.R);
    c.payload = s->dalloc<double>(N * (c.R + 2));
    c.lw = s->dalloc<double>(N);
    c.llbar = s->dalloc<double>(N);
    c.lg = s->dalloc<double>(N);
    c.cdf = s->dalloc<double>(N);
    c.anc = s->dalloc<unsigned>(N);
    c.tile_log2 = tile_log2;
    // the ancestor search's tables (segment ends, guide): small, read with
    // an L2 evict-last policy so the one-shot gathers stream past them. (A
    // persisting access-policy window was measured: it cost the streaming
    // kernels more than it saved, profiles/r01_notes.md.)
    c.seg_end = s->dalloc<double>((NT << tile_log2) >> kSegLog2);
    c.coarse = s->dalloc<unsigned>(size_t(1) << cb);
    const size_t GNT = NT * world;  // tile arrays cover every shard (aliased at tile0)
    c.n0 = static_cast<long long>(rank) * s->N;
    c.n_glob = static_cast<long long>(cfg->particles);
    c.sharded = shard_api;  // a shard handle (any world size, 1 included) exports its partials
    c.rank = rank;
    c.world = world;
    c.gntiles = static_cast<int>(GNT);
    c.tile0 = static_cast<int>(NT) * rank;
    c.gtile_info = s->dalloc<double2>(GNT);
    c.tile_info = c.gtile_info + c.tile0;
    c.blk_cnt = s->dalloc<int>(static_cast<size_t>(s->grid));
    c.trel = s->dalloc<double>(NT);
    c.tile_m = s->dalloc<double>(NT);
    c.trec = s->dalloc<ThreadRec>(NT * kThreads);
    c.tile_pre = s->dalloc<double>(NT);
    c.tile_cnt_pre = s->dalloc<long long>(NT);
    c.ghdr = s->dalloc<TileHdr>(GNT);
    c.gwin = s->dalloc<TileWin>(GNT * kMaxWin);
    c.gwin_after = s->dalloc<double>(GNT * kMaxWin);
    c.hdr = c.ghdr + c.tile0;
    c.win = c.gwin + static_cast<size_t>(c.tile0) * kMaxWin;
    c.win_after = c.gwin_after + static_cast<size_t>(c.tile0) * kMaxWin;
    c.shard_sum = s->dalloc<double>(2);
    c.shard_off = s->dalloc<double>(2);
    CK(cudaMemset(c.shard_off, 0, 2 * sizeof(double)));
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
    s->ngroups_pred = (s->grid + kGroup - 1) / kGroup;
    s->ngroups_upd = s->ngroups_pred;
    s->shard_api = shard_api;
    if (shard_api) {
      const int W = s->ks->moment_width();
      s->gp_pred_all = s->dalloc<double>(static_cast<size_t>(world) * s->ngroups_pred * 2);
      s->gp_mom_all = s->dalloc<double>(static_cast<size_t>(world) * s->ngroups_upd * W);
      s->sums_all = s->dalloc<double>(2 * world);
      s->sendbuf = s->dalloc<double>(static_cast<size_t>(world) * N * (c.R + kShardPW));
      s->recvbuf = s->dalloc<double>(N * (c.R + kShardPW));
      s->counts_dev = s->dalloc<unsigned>(2 * world);
      s->counts_all = s->dalloc<unsigned>(static_cast<size_t>(world) * world);
      CK(cudaMallocHost(&s->counts_host, (2 * world + world * world) * sizeof(unsigned)));
    }
    build_graph(s.get());
    *out = s.release();
    return PFSMC_GPU_OK;
  });
}

pfsmc_gpu_status pfsmc_gpu_create(const pfsmc_gpu_config* cfg, pfsmc_gpu_sampler** out) {
  return create_impl(cfg, 0, 1, out);
}

pfsmc_gpu_status pfsmc_gpu_create_shard(const pfsmc_gpu_config* cfg, int rank, int world,
                                        pfsmc_gpu_sampler** out) {
  return create_impl(cfg, rank, world, out, true);
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
    // shrink mean + chol(cov_u); sharded: the caller finishes it globally
    // (pfsmc_gpu_shard_moments + allgather + pfsmc_gpu_shard_finish_moments(0))
    if (!s->shard_api) s->ks->moments(s->ctx, s->grid, s->stream, 0);
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
    const double lw0 = -std::log(static_cast<double>(s->cfg.particles));  // filter.cpp:86
    s->ks->init(s->ctx, s->grid, s->stream, kind, dprm, lw0);
    // first pass: mean about 0; second pass: cov about that mean (sharded:
    // the caller runs both passes globally)
    if (!s->shard_api) {
      s->ks->moments(s->ctx, s->grid, s->stream, 1);
      s->ks->moments(s->ctx, s->grid, s->stream, 1);
    }
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

pfsmc_gpu_status pfsmc_gpu_debug_timestamps(pfsmc_gpu_sampler* s, uint64_t* out8) {
  return guarded([&] {
    DevState h{};
    CK(cudaMemcpyAsync(&h, s->st, sizeof(DevState), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    for (int i = 0; i < 8; ++i) out8[i] = h.tstamp[i];
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
    k_gin_tiles<<<s->ntiles, kThreads, 0, s->stream>>>(c);
    k_gin_prefix<<<1, kThreads, 0, s->stream>>>(c);
    launch_scan(c, s->ntiles, s->stream, 1);
    launch_scan(c, s->ntiles, s->stream, 2);
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


// ---------------------------------------------------------------- sharded phases
// One handle per GPU, each owning global slots [rank*N/world, (rank+1)*N/world).
// The host orchestrator (paper_1411_1702_b200/sharded.py) runs the phases in
// order and performs the collectives on the exposed buffers between them.

pfsmc_gpu_status pfsmc_gpu_shard_buffer(pfsmc_gpu_sampler* s, int which, void** ptr, uint64_t* bytes) {
  return guarded([&] {
    const Ctx& c = s->ctx;
    const size_t W = static_cast<size_t>(s->ks->moment_width());
    const size_t PW = static_cast<size_t>(c.R + kShardPW);
    switch (which) {
      case 0: *ptr = c.gpart; *bytes = sizeof(double) * 2 * s->ngroups_pred; break;
      case 1: *ptr = s->gp_pred_all; *bytes = sizeof(double) * 2 * s->ngroups_pred * s->world; break;
      case 2: *ptr = c.shard_sum; *bytes = sizeof(double) * 2; break;
      case 3: *ptr = s->sums_all; *bytes = sizeof(double) * 2 * s->world; break;
      case 4: *ptr = c.ghdr; *bytes = sizeof(TileHdr) * c.gntiles; break;
      case 5: *ptr = c.gwin; *bytes = sizeof(TileWin) * static_cast<size_t>(c.gntiles) * kMaxWin; break;
      case 6: *ptr = c.gpart; *bytes = sizeof(double) * W * s->ngroups_upd; break;
      case 7: *ptr = s->gp_mom_all; *bytes = sizeof(double) * W * s->ngroups_upd * s->world; break;
      case 8: *ptr = s->sendbuf; *bytes = sizeof(double) * PW * s->N * s->world; break;
      case 9: *ptr = s->recvbuf; *bytes = sizeof(double) * PW * s->N; break;
      case 10: *ptr = s->counts_dev; *bytes = sizeof(unsigned) * 2 * s->world; break;
      case 11: *ptr = s->counts_all; *bytes = sizeof(unsigned) * s->world * s->world; break;
      default: throw ConfigError("shard_buffer: unknown buffer id");
    }
    if (!s->shard_api && (which == 1 || which == 3 || which >= 7)) throw ConfigError("not a sharded handle");
    return PFSMC_GPU_OK;
  });
}

static void shard_predict_impl(pfsmc_gpu_sampler* s, const double* y, uint64_t j, double t_prev, double t_obs,
                               double h) {
  if (!s->have_ensemble) throw ConfigError("step: no ensemble (call set_ensemble or init_*)");
  const StepParams sp = make_params(s, y, j, t_prev, t_obs, h);
  CK(cudaStreamSynchronize(s->stream));  // the pinned params slot is free
  *s->sp_host = sp;
  CK(cudaMemcpyAsync(s->sp_dev, s->sp_host, sizeof(StepParams), cudaMemcpyHostToDevice, s->stream));
  enqueue_prologue(s);
  s->ks->predict(s->ctx, s->grid, s->stream);
  CK(cudaGetLastError());
}

pfsmc_gpu_status pfsmc_gpu_shard_predict(pfsmc_gpu_sampler* s, const double* y, uint64_t j,
                                         double t_prev, double t_obs, double h) {
  return guarded([&] {
    shard_predict_impl(s, y, j, t_prev, t_obs, h);
    return PFSMC_GPU_OK;
  });
}

pfsmc_gpu_status pfsmc_gpu_shard_finish_lse(pfsmc_gpu_sampler* s) {
  return guarded([&] {
    k_finish_lse<<<1, kThreads, 0, s->stream>>>(s->ctx, s->gp_pred_all, s->ngroups_pred * s->world);
    CK(cudaGetLastError());
    return PFSMC_GPU_OK;
  });
}

pfsmc_gpu_status pfsmc_gpu_shard_scan_records(pfsmc_gpu_sampler* s) {
  return guarded([&] {
    k_shard_offset<<<1, 32, 0, s->stream>>>(s->ctx, s->sums_all);
    launch_scan(s->ctx, s->ntiles, s->stream, 4);
    CK(cudaGetLastError());
    return PFSMC_GPU_OK;
  });
}

pfsmc_gpu_status pfsmc_gpu_shard_resolve(pfsmc_gpu_sampler* s) {
  return guarded([&] {
    launch_scan(s->ctx, s->ntiles, s->stream, 5);
    launch_scan(s->ctx, s->ntiles, s->stream, 2);
    CK(cudaGetLastError());
    return PFSMC_GPU_OK;
  });
}

// counts_out: [world] payloads this rank sends to each rank, then [world]
// payloads it receives from each rank. Blocking (the exchange needs them).
static void shard_serve_impl(pfsmc_gpu_sampler* s, uint32_t* counts_out) {
  {
    const int W = s->world;
    // counts_dev: [W] actual sends of this rank; counts_all: the W x W matrix
    CK(cudaMemsetAsync(s->counts_dev, 0, 2 * W * sizeof(unsigned), s->stream));
    CK(cudaMemsetAsync(s->counts_all, 0, static_cast<size_t>(W) * W * sizeof(unsigned), s->stream));
    const long long nglob = s->ctx.n_glob;
    const int g = static_cast<int>(std::min<long long>((nglob + kThreads - 1) / kThreads, 148LL * 16));
    k_serve_sharded<<<g, kThreads, 0, s->stream>>>(s->ctx, s->sendbuf, s->counts_dev, s->counts_all);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(s->counts_host, s->counts_dev, W * sizeof(unsigned), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaMemcpyAsync(s->counts_host + 2 * W, s->counts_all, static_cast<size_t>(W) * W * sizeof(unsigned),
                       cudaMemcpyDeviceToHost, s->stream));
    CK(cudaMemcpyAsync(s->st_host, s->st, sizeof(DevState), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    check_error(s);
    const unsigned* mat = s->counts_host + 2 * W;
    for (int d = 0; d < W; ++d)  // the served counts must be the matrix row (self-check)
      if (s->counts_host[d] != mat[s->rank * W + d]) throw std::runtime_error("shard_serve: count mismatch");
    for (int i = 0; i < W; ++i) counts_out[i] = mat[s->rank * W + i];      // sends
    for (int i = 0; i < W; ++i) counts_out[W + i] = mat[i * W + s->rank];  // receives
  }
}

pfsmc_gpu_status pfsmc_gpu_shard_serve(pfsmc_gpu_sampler* s, uint32_t* counts_out) {
  return guarded([&] {
    shard_serve_impl(s, counts_out);
    return PFSMC_GPU_OK;
  });
}

// The W x W migration count matrix of the last shard_serve (row r: rank r's sends).
pfsmc_gpu_status pfsmc_gpu_shard_count_matrix(pfsmc_gpu_sampler* s, uint32_t* out) {
  return guarded([&] {
    if (!s->shard_api) throw ConfigError("not a sharded handle");
    const int W = s->world;
    for (int i = 0; i < W * W; ++i) out[i] = s->counts_host[2 * W + i];
    return PFSMC_GPU_OK;
  });
}

pfsmc_gpu_status pfsmc_gpu_shard_update(pfsmc_gpu_sampler* s, uint64_t n_recv) {
  return guarded([&] {
    if (n_recv != static_cast<uint64_t>(s->N)) throw std::runtime_error("shard_update: payload count mismatch");
    k_place<<<s->grid, kThreads, 0, s->stream>>>(s->ctx, s->recvbuf, static_cast<long long>(n_recv));
    s->ks->update(s->ctx, s->grid, s->stream);
    CK(cudaGetLastError());
    return PFSMC_GPU_OK;
  });
}

pfsmc_gpu_status pfsmc_gpu_shard_moments(pfsmc_gpu_sampler* s) {
  return guarded([&] {
    s->ks->moments(s->ctx, s->grid, s->stream, 1);
    CK(cudaGetLastError());
    return PFSMC_GPU_OK;
  });
}

// flags: 7 = a completed step (lse_w, cov, chol, flip); 2 = init refresh;
// 0 = injection (shrink mean only). Blocking; trace_out optional.
static void shard_finish_moments_impl(pfsmc_gpu_sampler* s, int flags, double* trace_out) {
  s->ks->finish_moments(s->ctx, s->gp_mom_all, s->ngroups_upd * s->world, flags, s->stream);
  CK(cudaMemcpyAsync(s->st_host, s->st, sizeof(DevState), cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  CK(cudaGetLastError());
  check_error(s);
  if (trace_out) {
    const int n = 2 * s->p + s->d + 1;
    for (int k = 0; k < n; ++k) trace_out[k] = s->st_host->trace[k];
  }
}

pfsmc_gpu_status pfsmc_gpu_shard_finish_moments(pfsmc_gpu_sampler* s, int flags, double* trace_out) {
  return guarded([&] {
    shard_finish_moments_impl(s, flags, trace_out);
    return PFSMC_GPU_OK;
  });
}


// ---- native sharded step over NCCL (one call per observation) ------------
pfsmc_gpu_status pfsmc_gpu_nccl_unique_id(uint8_t* out128) {
  return guarded([&] {
    if (!nccl_api().ok) throw std::runtime_error("nccl: libnccl.so.2 not available");
    ncclUniqueId id;
    NCK(nccl_api().GetUniqueId(&id));
    std::memcpy(out128, &id, sizeof(id));
    return PFSMC_GPU_OK;
  });
}

pfsmc_gpu_status pfsmc_gpu_shard_attach_nccl(pfsmc_gpu_sampler* s, const uint8_t* id128) {
  return guarded([&] {
    if (!s->shard_api) throw ConfigError("not a sharded handle");
    if (!nccl_api().ok) throw std::runtime_error("nccl: libnccl.so.2 not available");
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    CK(cudaSetDevice(s->cfg.device));
    if (s->nccl) NCK(nccl_api().CommDestroy(s->nccl));
    NCK(nccl_api().CommInitRank(&s->nccl, s->world, id, s->rank));
    return PFSMC_GPU_OK;
  });
}

// ---- migration over NVLink peer memory --------------------------------------
// The six buffers a peer reads (record buffers, ll_bar, the exact CDF, the
// segment ends, the guide), as CUDA IPC handles: 6 x 64 bytes.
constexpr int kPeerBufs = 6;

pfsmc_gpu_status pfsmc_gpu_shard_ipc_handles(pfsmc_gpu_sampler* s, uint8_t* out) {
  return guarded([&] {
    if (!s->shard_api) throw ConfigError("not a sharded handle");
    const Ctx& c = s->ctx;
    const void* bufs[kPeerBufs] = {c.rec[0], c.rec[1], c.llbar, c.cdf, c.seg_end, c.coarse};
    for (int i = 0; i < kPeerBufs; ++i) {
      cudaIpcMemHandle_t h;
      CK(cudaIpcGetMemHandle(&h, const_cast<void*>(bufs[i])));
      std::memcpy(out + i * sizeof(h), &h, sizeof(h));
    }
    return PFSMC_GPU_OK;
  });
}

// all_handles: world x kPeerBufs IPC handles in rank order (this rank's own
// entry is ignored: local pointers).
pfsmc_gpu_status pfsmc_gpu_shard_attach_peers(pfsmc_gpu_sampler* s, const uint8_t* all_handles) {
  return guarded([&] {
    if (!s->shard_api) throw ConfigError("not a sharded handle");
    if (s->world > kMaxRanks) throw ConfigError("attach_peers: at most 8 ranks");
    CK(cudaSetDevice(s->cfg.device));
    const Ctx& c = s->ctx;
    PeerTable t{};
    for (int r = 0; r < s->world; ++r) {
      const void* p[kPeerBufs];
      if (r == s->rank) {
        p[0] = c.rec[0], p[1] = c.rec[1], p[2] = c.llbar, p[3] = c.cdf, p[4] = c.seg_end, p[5] = c.coarse;
      } else {
        for (int i = 0; i < kPeerBufs; ++i) {
          cudaIpcMemHandle_t h;
          std::memcpy(&h, all_handles + (static_cast<size_t>(r) * kPeerBufs + i) * sizeof(h), sizeof(h));
          void* q = nullptr;
          CK(cudaIpcOpenMemHandle(&q, h, cudaIpcMemLazyEnablePeerAccess));
          s->ipc_opened.push_back(q);
          p[i] = q;
        }
      }
      t.rec0[r] = static_cast<const double*>(p[0]);
      t.rec1[r] = static_cast<const double*>(p[1]);
      t.llbar[r] = static_cast<const double*>(p[2]);
      t.cdf[r] = static_cast<const double*>(p[3]);
      t.seg_end[r] = static_cast<const double*>(p[4]);
      t.coarse[r] = static_cast<const unsigned*>(p[5]);
    }
    s->peers = t;
    s->have_peers = true;
    return PFSMC_GPU_OK;
  });
}

// The device part of one peer-memory sharded step (everything between the
// step-parameter upload and the DevState read-back), for eager launch or
// capture into a CUDA graph (NCCL collectives capture).
static void enqueue_shard_pull_step(pfsmc_gpu_sampler* s) {
  const NcclApi& N = nccl_api();
  const Ctx& c = s->ctx;
  cudaStream_t st = s->stream;
  const int W = s->world;
  enqueue_prologue(s);
  s->ks->predict(c, s->grid, st);
  NCK(N.AllGather(c.gpart, s->gp_pred_all, 2 * static_cast<size_t>(s->ngroups_pred), ncclDouble, s->nccl, st));
  k_finish_lse<<<1, kThreads, 0, st>>>(c, s->gp_pred_all, s->ngroups_pred * W);
  NCK(N.AllGather(c.shard_sum, s->sums_all, 2, ncclDouble, s->nccl, st));
  k_shard_offset<<<1, 32, 0, st>>>(c, s->sums_all);
  launch_scan(c, s->ntiles, st, 4);
  NCK(N.AllGather(c.hdr, c.ghdr, sizeof(TileHdr) * static_cast<size_t>(s->ntiles), ncclUint8, s->nccl, st));
  NCK(N.AllGather(c.win, c.gwin, sizeof(TileWin) * static_cast<size_t>(s->ntiles) * kMaxWin, ncclUint8,
                  s->nccl, st));
  launch_scan(c, s->ntiles, st, 5);
  launch_scan(c, s->ntiles, st, 2);
  NCK(N.AllGather(c.shard_sum, s->sums_all, 2, ncclDouble, s->nccl, st));  // tables complete everywhere
  k_pull<<<s->grid, kThreads, 0, st>>>(c, s->peers);
  s->ks->update(c, s->grid, st);
  const size_t Wm = static_cast<size_t>(s->ks->moment_width());
  NCK(N.AllGather(c.gpart, s->gp_mom_all, Wm * s->ngroups_upd, ncclDouble, s->nccl, st));
  s->ks->finish_moments(c, s->gp_mom_all, s->ngroups_upd * W, 7, st);
  CK(cudaMemcpyAsync(s->st_host, s->st, sizeof(DevState), cudaMemcpyDeviceToHost, st));
}

// The peer-memory step: one CUDA graph per step (built on first use; eager
// launches if capture is refused), one host sync for the trace row.
static void shard_pull_step(pfsmc_gpu_sampler* s, const double* y, uint64_t j, double t_prev, double t_obs,
                            double h, double* trace_out) {
  if (!s->have_ensemble) throw ConfigError("step: no ensemble (call set_ensemble or init_*)");
  const StepParams sp = make_params(s, y, j, t_prev, t_obs, h);
  CK(cudaStreamSynchronize(s->stream));  // the pinned params slot is free
  *s->sp_host = sp;
  CK(cudaMemcpyAsync(s->sp_dev, s->sp_host, sizeof(StepParams), cudaMemcpyHostToDevice, s->stream));
  if (!s->shard_graph && !s->shard_graph_refused) {
    cudaGraph_t g = nullptr;
    bool ok = cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    if (ok) {
      try {
        enqueue_shard_pull_step(s);
      } catch (const std::exception&) {
        ok = false;
      }
      const cudaError_t e = cudaStreamEndCapture(s->stream, &g);
      ok = ok && e == cudaSuccess && g != nullptr &&
           cudaGraphInstantiate(&s->shard_graph, g, 0) == cudaSuccess;
      if (g) cudaGraphDestroy(g);
    }
    if (!ok) {
      s->shard_graph = nullptr;
      s->shard_graph_refused = true;
      cudaGetLastError();  // clear
    }
  }
  if (s->shard_graph)
    CK(cudaGraphLaunch(s->shard_graph, s->stream));
  else
    enqueue_shard_pull_step(s);
  CK(cudaStreamSynchronize(s->stream));
  CK(cudaGetLastError());
  check_error(s);
  if (trace_out) {
    const int n = 2 * s->p + s->d + 1;
    for (int k = 0; k < n; ++k) trace_out[k] = s->st_host->trace[k];
  }
}

// One pf_step of the global filter: the five exchanges as NCCL
// collectives on the sampler stream between the phase kernels, host syncs
// only where the host needs data (the migration counts, the trace row).
pfsmc_gpu_status pfsmc_gpu_shard_step(pfsmc_gpu_sampler* s, const double* y, uint64_t j, double t_prev,
                                      double t_obs, double h, double* trace_out) {
  return guarded([&] {
    if (!s->nccl) throw ConfigError("shard_step: no NCCL communicator (pfsmc_gpu_shard_attach_nccl)");
    if (s->have_peers) {
      shard_pull_step(s, y, j, t_prev, t_obs, h, trace_out);
      return PFSMC_GPU_OK;
    }
    const NcclApi& N = nccl_api();
    const Ctx& c = s->ctx;
    cudaStream_t st = s->stream;
    const int W = s->world, me = s->rank;
    shard_predict_impl(s, y, j, t_prev, t_obs, h);
    // A: predict-kernel group partials -> global LSE
    NCK(N.AllGather(c.gpart, s->gp_pred_all, 2 * static_cast<size_t>(s->ngroups_pred), ncclDouble, s->nccl, st));
    k_finish_lse<<<1, kThreads, 0, st>>>(c, s->gp_pred_all, s->ngroups_pred * W);
    // B: shard (approximate total, nonzero count) -> global prefix for the classification
    NCK(N.AllGather(c.shard_sum, s->sums_all, 2, ncclDouble, s->nccl, st));
    k_shard_offset<<<1, 32, 0, st>>>(c, s->sums_all);
    launch_scan(c, s->ntiles, st, 4);
    // C: tile records, in place (this rank's slice of the global arrays)
    NCK(N.AllGather(c.hdr, c.ghdr, sizeof(TileHdr) * static_cast<size_t>(s->ntiles), ncclUint8, s->nccl, st));
    NCK(N.AllGather(c.win, c.gwin, sizeof(TileWin) * static_cast<size_t>(s->ntiles) * kMaxWin, ncclUint8,
                    s->nccl, st));
    launch_scan(c, s->ntiles, st, 5);
    launch_scan(c, s->ntiles, st, 2);
    CK(cudaGetLastError());

    // D: exact-mode migration; the counts are the locally derived matrix
    std::vector<uint32_t> cnt(2 * static_cast<size_t>(W));
    shard_serve_impl(s, cnt.data());
    const unsigned* mat = s->counts_host + 2 * W;
    const size_t item = sizeof(double) * static_cast<size_t>(c.R + kShardPW);
    const size_t cap = static_cast<size_t>(s->N);
    char* send = reinterpret_cast<char*>(s->sendbuf);
    char* recv = reinterpret_cast<char*>(s->recvbuf);
    size_t off = 0;
    NCK(N.GroupStart());
    for (int r = 0; r < W; ++r) {
      const size_t k_in = mat[r * W + me], k_out = mat[me * W + r];
      if (r == me) {
        if (k_in)
          CK(cudaMemcpyAsync(recv + off * item, send + r * cap * item, k_in * item, cudaMemcpyDeviceToDevice, st));
      } else {
        if (k_out) NCK(N.Send(send + r * cap * item, k_out * item, ncclUint8, r, s->nccl, st));
        if (k_in) NCK(N.Recv(recv + off * item, k_in * item, ncclUint8, r, s->nccl, st));
      }
      off += k_in;
    }
    NCK(N.GroupEnd());
    if (off != cap) throw std::runtime_error("shard_step: payload count mismatch");
    k_place<<<s->grid, kThreads, 0, st>>>(c, s->recvbuf, static_cast<long long>(off));
    s->ks->update(c, s->grid, st);
    // E: update-kernel moment partials -> global lse_w, moments, trace row, chol
    const size_t Wm = static_cast<size_t>(s->ks->moment_width());
    NCK(N.AllGather(c.gpart, s->gp_mom_all, Wm * s->ngroups_upd, ncclDouble, s->nccl, st));
    CK(cudaGetLastError());
    shard_finish_moments_impl(s, 7, trace_out);
    return PFSMC_GPU_OK;
  });
}

// ---- BASELINE config 5 microbenchmark entry points (model PAYLOAD64) -----
pfsmc_gpu_status pfsmc_gpu_c5_set_logweights(pfsmc_gpu_sampler* s, double sigma, uint64_t key) {
  return guarded([&] {
    if (s->cfg.model != Payload64Model::ID) throw ConfigError("c5: needs the PAYLOAD64 model");
    k_c5_weights<<<s->grid, kThreads, 0, s->stream>>>(s->ctx, sigma, key);
    CK(cudaGetLastError());
    return PFSMC_GPU_OK;
  });
}

// One resample/reduction iteration (enqueue only): LSE + tile offsets, the
// weighted 2x2 covariance, the exact CDF, the ancestor search and gather.
pfsmc_gpu_status pfsmc_gpu_c5_iteration(pfsmc_gpu_sampler* s, uint64_t j) {
  return guarded([&] {
    if (s->cfg.model != Payload64Model::ID) throw ConfigError("c5: needs the PAYLOAD64 model");
    Ctx c = s->ctx;
    c.lg = c.lw;  // the fitness log-weights are the log-weights here
    CK(cudaMemsetAsync(&s->st->error, 0, sizeof(int), s->stream));
    // one wave: 126 (ITEMS 16) / 74 (ITEMS 8) registers => 2 / 3 blocks per SM
    if (c.tile_log2 == 11)
      k_c5_stats<8><<<std::min(s->ntiles, s->num_sms * 3), kThreads, 0, s->stream>>>(c);
    else
      k_c5_stats<16><<<std::min(s->ntiles, s->num_sms * 2), kThreads, 0, s->stream>>>(c);
    launch_scan(c, s->ntiles, s->stream, 1);
    launch_scan(c, s->ntiles, s->stream, 2);
    k_c5_serve<<<s->grid, kThreads, 0, s->stream>>>(c, j);
    k_flip<<<1, 1, 0, s->stream>>>(s->st);
    CK(cudaGetLastError());
    return PFSMC_GPU_OK;
  });
}


// Measured FP64 FMA throughput of this device (TFLOP/s, 2 flops per DFMA).
pfsmc_gpu_status pfsmc_gpu_fp64_peak(int device, double* tflops) {
  return guarded([&] {
    CK(cudaSetDevice(device));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    double* out;
    CK(cudaMalloc(&out, sizeof(double)));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const int blocks = sms * 8, iters = 4096;
    k_dfma_peak<<<blocks, kThreads>>>(out, 256, 0.999999, 1e-7);  // warm-up
    CK(cudaEventRecord(e0));
    k_dfma_peak<<<blocks, kThreads>>>(out, iters, 0.999999, 1e-7);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    *tflops = 2.0 * 8.0 * iters * static_cast<double>(blocks) * kThreads / (ms * 1e-3) / 1e12;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    return PFSMC_GPU_OK;
  });
}

// One noise-free trajectory of a compiled-in model through the observation
// times with the adaptive BDF(1,2) integrator (the data generator's truth
// path, bench.cpp:296-317 with lmm::adaptive_bdf_interval). Blocking.
pfsmc_gpu_status pfsmc_gpu_model_trajectory(int model, const double* model_consts, const double* theta_nat,
                                            const double* x0, const double* times, uint64_t T, double t0,
                                            double rtol, int device, double* states_out) {
  return guarded([&] {
    auto ks = make_kernels(model, PFSMC_GPU_BDF, 0);
    if (!ks) throw ConfigError("unknown model id");
    if (!(rtol > 0.0)) throw ConfigError("adaptive_bdf_interval: rtol must be positive");
    if (T == 0) return PFSMC_GPU_OK;
    double tp = t0;
    for (uint64_t r = 0; r < T; ++r) {
      if (!(times[r] > tp)) throw ConfigError("adaptive_bdf_interval: need t1 > t0");
      tp = times[r];
    }
    if (model == MetabolicModel::ID && !(model_consts[5] > 0.0))
      throw ConfigError("metabolic model: tau must be positive");
    CK(cudaSetDevice(device));
    const int d = ks->d, p = ks->p;
    std::vector<double> prm(8 + p + d);
    for (int k = 0; k < 8; ++k) prm[k] = model_consts ? model_consts[k] : 0.0;
    for (int k = 0; k < p; ++k) prm[8 + k] = theta_nat[k];
    for (int k = 0; k < d; ++k) prm[8 + p + k] = x0[k];
    double *dprm, *dt, *dout;
    int* dst;
    CK(cudaMalloc(&dprm, sizeof(double) * prm.size()));
    CK(cudaMalloc(&dt, sizeof(double) * T));
    CK(cudaMalloc(&dout, sizeof(double) * T * d));
    CK(cudaMalloc(&dst, sizeof(int)));
    CK(cudaMemcpy(dprm, prm.data(), sizeof(double) * prm.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dt, times, sizeof(double) * T, cudaMemcpyHostToDevice));
    ks->trajectory(dprm, dt, static_cast<int>(T), t0, rtol, 1e-9, 20, dout, dst, nullptr);  // NewtonOpts{}
    CK(cudaGetLastError());
    int st = 0;
    CK(cudaMemcpy(&st, dst, sizeof(int), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(states_out, dout, sizeof(double) * T * d, cudaMemcpyDeviceToHost));
    cudaFree(dprm);
    cudaFree(dt);
    cudaFree(dout);
    cudaFree(dst);
    if (st != 0) throw NumericalError("reference trajectory integration failed (stiffness)");
    return PFSMC_GPU_OK;
  });
}

// Measured random 64-byte-record gather throughput (GB/s of record bytes
// read + written), over n_rec records (> L2), median-free: best of 5.
pfsmc_gpu_status pfsmc_gpu_gather_peak(int device, long long n_rec, double* gbs) {
  return guarded([&] {
    CK(cudaSetDevice(device));
    double2 *src, *dst;
    CK(cudaMalloc(&src, static_cast<size_t>(n_rec) * 64));
    CK(cudaMalloc(&dst, static_cast<size_t>(n_rec) * 64));
    CK(cudaMemset(src, 0, static_cast<size_t>(n_rec) * 64));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const int blocks = static_cast<int>((n_rec + kThreads - 1) / kThreads);
    float best = 1e30f;
    for (int r = 0; r < 6; ++r) {
      CK(cudaEventRecord(e0));
      k_gather_peak<<<blocks, kThreads>>>(src, dst, n_rec);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (r > 0) best = std::min(best, ms);
    }
    *gbs = 128.0 * static_cast<double>(n_rec) / (best * 1e-3) / 1e9;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(src);
    cudaFree(dst);
    return PFSMC_GPU_OK;
  });
}

}  // extern "C"
