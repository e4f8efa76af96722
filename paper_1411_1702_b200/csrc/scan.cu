// The exact sequential CDF (filter.cpp:158-168) and the ancestor search +
// gather (filter.cpp:169-176, 330-335): tile decomposition, window resolver,
// S3 CDF values and search tables, k_serve. See DESIGN.md §4.
#include "sampler_internal.cuh"

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
__device__ bool resolve_windows(const Ctx& c, const TileHdr* hdr, const WinSrc& win, double* win_after,
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
        const TileWin* gw = win.at(t, k);
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
__device__ void resolve_chain(const Ctx& c, const TileHdr* hdr, const WinSrc& win, double* win_after,
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
        for (int k = 0; k < n && w < kResolveWin; ++k, ++w) rs.wsrc[w] = win.at(ti, k);
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
                const TileWin* gw = win.at(ti, k);
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
      if (k < c.N) g = c.gin ? x[i] : exp(x[i] - lse);  // S3 recomputes it (bitwise) or reads it back
      sm.g[TC::sidx(e)] = g;
      if (c.store_g && k < c.N) __stcg(&c.cdf[k], g);  // L2-resident sizes: S3 reads g instead of exp
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
  WinSrc own{};
  own.base[0] = c.win;
  own.tiles_per_rank = c.ntiles;
  if (!resolve_windows<ITEMS>(c, c.hdr, own, c.win_after, c.tile_info, c.ntiles, sm.ws))
    resolve_chain<ITEMS>(c, c.hdr, own, c.win_after, c.tile_info, c.ntiles, true, sm.rs);
  if (threadIdx.x == 0) c.st->tstamp[2] = global_ns();
}

// Sharded: every rank resolves the exact chain over ALL shards' tiles.
template <int ITEMS>
__global__ void __launch_bounds__(kThreads) k_resolve_global(Ctx c, WinSrc ws) {
  __shared__ union {
    ResolverSmem rs;
    WinSmem ws;
  } sm;
  if (grid_error(c)) return;
  if (!resolve_windows<ITEMS>(c, c.ghdr, ws, c.gwin_after, c.gtile_info, c.gntiles, sm.ws))
    resolve_chain<ITEMS>(c, c.ghdr, ws, c.gwin_after, c.gtile_info, c.gntiles, false, sm.rs);
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

void launch_resolve_global(const Ctx& c, int ntiles, cudaStream_t st, const WinSrc& ws) {
  if (c.tile_log2 == 11) k_resolve_global<8><<<1, kThreads, 0, st>>>(c, ws);
  else k_resolve_global<16><<<1, kThreads, 0, st>>>(c, ws);
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
    case 5: {  // windows from the allgathered copy of every shard's lists
      WinSrc ws{};
      for (int r = 0; r < c.world && r < kMaxRanks; ++r) ws.base[r] = c.gwin + static_cast<size_t>(r) * ntiles * kMaxWin;
      ws.tiles_per_rank = ntiles;
      launch_resolve_global(c, ntiles, st, ws);
      break;
    }
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
  const int ngroups = (c.ntiles * (tile >> c.k1_block_log2) + kGroup - 1) / kGroup;
  for (int g = blockIdx.x * kThreads + threadIdx.x; g < ngroups; g += gridDim.x * kThreads) c.gpart[2 * g] = 0.0;
}

__global__ void __launch_bounds__(kThreads) k_gin_prefix(Ctx c) {
  if (threadIdx.x == 0) c.st->lse_g = 0.0;
  tile_prefixes(c, 0.0);
}

void launch_gin(const Ctx& c, int ntiles, cudaStream_t st) {
  k_gin_tiles<<<ntiles, kThreads, 0, st>>>(c);
  k_gin_prefix<<<1, kThreads, 0, st>>>(c);
}

__global__ void __launch_bounds__(kThreads) k_search_only(Ctx c) {
  if (grid_error(c)) return;
  const long long n = static_cast<long long>(blockIdx.x) * kThreads + threadIdx.x;
  const double u = n < c.N ? resample_uniform(c.seed, c.sp->j, n) : -1.0;
  const unsigned a = find_ancestor_warp(c, u);
  if (n < c.N) c.anc[n] = a;
}

void launch_search_only(const Ctx& c, int grid, cudaStream_t st) {
  k_search_only<<<grid, kThreads, 0, st>>>(c);
}

}  // namespace pfsmc_gpu
