// The exact sequential CDF (filter.cpp:158-168) and the ancestor search +
// gather (filter.cpp:169-176, 330-335): the tile analysis, the single-pass
// look-back scan, the two-pass form with its window resolver, the search
// tables, k_serve. See DESIGN.md §4.
#include "sampler_internal.cuh"

namespace pfsmc_gpu {

// ---------------------------------------------------------------- exact CDF
// Tiles of ITEMS * 256 elements (thread t owns elements ITEMS*t .. +ITEMS-1).
// ITEMS = 8 (2048-element tiles) keeps the per-thread chunks short and the
// grid wide for N <= 2^22; ITEMS = 16 bounds the tile count (and the chain of
// tiles) at larger N. One pad double per thread chunk keeps the
// per-thread contiguous shared-memory reads conflict-free.
template <int ITEMS>
struct TileCfg {
  static constexpr int kTileT = ITEMS * kThreads;
  static constexpr int kSmem = kTileT + kThreads;
  __device__ static __forceinline__ int sidx(int e) { return e + e / ITEMS; }
};

// The scale 2^(52-e) that turns an element into units of binade e's ulp,
// as two exact factors: for the subnormal binade (e = -1022) 2^1074 itself
// overflows, 2^537 * 2^537 does not.
struct UlpScale {
  double s1, s2;
};
__device__ __forceinline__ UlpScale ulp_scale(int e) {
  const int k = 52 - e;
  return k <= 1000 ? UlpScale{scale2(1.0, k), 1.0} : UlpScale{scale2(1.0, k - k / 2), scale2(1.0, k / 2)};
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

// One tile's outputs from its per-thread exact values: the CDF (coalesced
// through shared memory), the segment ends and the tile's guide buckets.
// ti = the exact CDF (before the tile, at its last element incl. the guard).
template <int ITEMS>
__device__ __forceinline__ void tile_emit(const Ctx& c, int t, long long base, int valid, const double (&vals)[ITEMS],
                                          double2 ti, double* sg, double* send) {
  using TC = TileCfg<ITEMS>;
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

// ------------------------------------------------- single-pass exact scan
// The same exact CDF in ONE kernel (single handle): a tile classifies its
// elements as k_scan_pieces does, then learns the exact sum before it by a
// decoupled look-back instead of a resolver pass:
//  * a window-free tile publishes its aggregate piece at once (LookAgg);
//  * every tile publishes the exact CDF at its last element (LookPre) as soon
//    as it knows the exact value before it; a tile with windows applies them
//    in order with real IEEE adds (one thread, ~log2 N windows in the whole
//    scan) before publishing;
//  * the look-back (one warp) composes the aggregate pieces of the predecessors
//    back to the nearest published exact value, oldest first (the monoid is
//    not commutative).
// Tiles are handed out by ticket, so every predecessor of a running tile is
// running or done (forward progress); the flags carry a launch epoch, so no
// reset pass is needed. The values, tables and the guard are then produced by
// the code k_scan_cdf uses (real IEEE adds from the chunk's exact start,
// tile_emit): bitwise the two-pass result, which stays the sharded path (its
// records cross GPUs).
// 16-byte words of the look-back records. An aligned 16-byte access is one
// transaction, so a record's value and its tag are seen together: relaxed
// gpu-scope loads and stores suffice, no fence on either side.
__device__ __forceinline__ void ld_relaxed_v2(const void* p, unsigned long long& a, unsigned long long& b) {
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
__device__ __forceinline__ void st_relaxed_v2(void* p, unsigned long long a, unsigned long long b) {
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void publish_pre(LookPre* r, double v, unsigned tag) {
  st_relaxed_v2(r, static_cast<unsigned long long>(__double_as_longlong(v)), static_cast<unsigned long long>(tag));
}
// The aggregate piece of a window-free tile in one 16-byte word. A composed
// piece has d1 - d0 in {-1, 0, 1} (two running sums that start one apart end
// 0, 1 or 2 apart: a tie moves them apart or together by one, and
// equal-parity sums move together), so the piece and the tag fit.
__device__ __forceinline__ void publish_agg(LookAgg* r, const Piece& pc, unsigned tag, int* err) {
  if (static_cast<unsigned long long>(pc.d1 - pc.d0 + 1) > 2ull) atomicOr(err, kErrInternal);  // never expected
  const unsigned ecode = pc.e == kNoBinade ? 0u : static_cast<unsigned>(pc.e + 2048);
  const unsigned long long meta =
      (static_cast<unsigned long long>(tag) << 32) | (ecode << 16) | static_cast<unsigned>(pc.d1 - pc.d0 + 1);
  st_relaxed_v2(r, static_cast<unsigned long long>(pc.d0), meta);
}
__device__ __forceinline__ Piece unpack_agg(unsigned long long d0, unsigned long long meta) {
  const unsigned lo = static_cast<unsigned>(meta);
  const unsigned ecode = lo >> 16;
  Piece pc;
  pc.d0 = static_cast<long long>(d0);
  pc.d1 = pc.d0 + static_cast<long long>(lo & 0xffu) - 1;
  pc.e = ecode ? static_cast<int>(ecode) - 2048 : kNoBinade;
  pc.flag = 0;
  return pc;
}

constexpr unsigned kLookSpinLimit = 1u << 21;  // polls (~1 s) before a tile gives up (INTERNAL)

// Composition of the warp's pieces, lane 31 (oldest) first, lane 0 last; every lane gets the result.
// Common case: no rounding tie, one binade => the pieces are plain integer steps and compose by a sum
// (any order); otherwise the ordered tree (the monoid is not commutative).
__device__ __forceinline__ Piece warp_compose(Piece x) {
  const int lane = threadIdx.x & 31;
  const int emax = __reduce_max_sync(0xffffffffu, x.e);  // kNoBinade (all-zero tiles) is below every binade
  const bool plain = emax != kNoBinade && !__any_sync(0xffffffffu, x.d0 != x.d1 || (x.e != emax && x.e != kNoBinade));
  if (plain) {
    long long sum = x.d0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    return Piece{sum, sum, emax, 0};
  }
  // ordered tree: lane l ends with lanes (l + o - 1 .. l), older first
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    Piece y;
    y.d0 = __shfl_down_sync(0xffffffffu, x.d0, o);
    y.d1 = __shfl_down_sync(0xffffffffu, x.d1, o);
    y.e = __shfl_down_sync(0xffffffffu, x.e, o);
    y.flag = 0;
    if (lane + o < 32) x = piece_combine(y, x);
  }
  Piece r;
  r.d0 = __shfl_sync(0xffffffffu, x.d0, 0);
  r.d1 = __shfl_sync(0xffffffffu, x.d1, 0);
  r.e = __shfl_sync(0xffffffffu, x.e, 0);
  r.flag = 0;
  return r;
}

// Warp-wide: the exact CDF value before tile t. `bail`: gave up (error word
// set elsewhere, or the spin limit): the caller skips its outputs.
// The walk goes back 32 tiles a round, composing the aggregate pieces of the
// window-free tiles (oldest first: the monoid is not commutative), until it
// meets a published exact value (or the start of the chain). A tile with
// windows publishes only its exact end value, so the ~log2 N such tiles form
// the one serial chain of the scan (one L2 round trip per link).
// (Measured and not kept, profiles/r02_notes.md: replaying through window
// tiles from their published window lists instead of waiting for their exact
// values, and loading the records several rounds ahead.)
__device__ __forceinline__ double look_back(const Ctx& c, int t, unsigned tag, bool& ok, bool& bail) {
  const int lane = threadIdx.x & 31;
  Piece acc = piece_identity();  // tiles [hi, t) composed, oldest first
  double base = 0.0;
  bail = false;
  int hi = t;
  while (hi > 0) {
    const int q = hi - 1 - lane;  // lane 0 looks at the nearest predecessor
    int state = 0;                // 1: aggregate piece seen, 2: exact value seen
    Piece x = piece_identity();
    double pv = 0.0;
    unsigned spins = 0;
    int fp;
    int pre_lane = -1;  // the one tile the round waited for (its later tiles pre-composed), or -1
    Piece pre_chunk = piece_identity();
    for (;;) {
      if (q >= 0 && state != 2) {
        // both records polled at once (independent loads, one 16-byte word each)
        unsigned long long v0, v1, a0 = 0, a1 = 0;
        ld_relaxed_v2(&c.look_pre[q], v0, v1);
        if (state == 0) ld_relaxed_v2(&c.look_agg[q], a0, a1);
        if (static_cast<unsigned>(v1) == tag) {
          state = 2;
          pv = __longlong_as_double(static_cast<long long>(v0));
        } else if (state == 0 && static_cast<unsigned>(a1 >> 32) == tag) {
          x = unpack_agg(a0, a1);
          state = 1;
        }
      }
      const unsigned valid = __ballot_sync(0xffffffffu, q >= 0);
      const unsigned pm = __ballot_sync(0xffffffffu, state == 2);
      const unsigned am = __ballot_sync(0xffffffffu, state != 0);
      fp = pm ? __ffs(pm) - 1 : 32;
      const unsigned need = (fp >= 32 ? 0xffffffffu : ((1u << fp) - 1u)) & valid;  // tiles after the exact value
      const unsigned miss = need & ~am;
      if (miss == 0) break;
      if (pre_lane < 0 && (miss & (miss - 1)) == 0) {
        // waiting for one tile only (a tile with windows: it publishes nothing but its exact value):
        // compose the tiles after it now, so its value is the only thing left on the chain
        pre_lane = __ffs(miss) - 1;
        pre_chunk = warp_compose(lane < pre_lane ? x : piece_identity());
      }
      ++spins;
      const bool stop = spins > kLookSpinLimit || ((spins & 63u) == 0 && grid_error(c));
      if (__any_sync(0xffffffffu, stop)) {
        if (spins > kLookSpinLimit && lane == 0) atomicOr(&c.st->error, kErrInternal);
        bail = true;
        return 0.0;
      }
    }
    // only the tiles after the exact value compose; when the round waited for exactly one tile, the
    // composition of the tiles after it was made while waiting
    const Piece chunk = (pre_lane >= 0 && fp == pre_lane) ? pre_chunk : warp_compose(lane < fp ? x : piece_identity());
    acc = piece_combine(chunk, acc);
    if (fp < 32) {
      base = __shfl_sync(0xffffffffu, pv, fp);
      break;
    }
    hi -= 32;
  }
  double s = base;  // hi <= 0 without an exact value: the chain starts at 0
  ok &= piece_apply(acc, s);
  return s;
}

// Composite element of the fused kernel's second block scan: the segmented
// piece and the window count.
struct PieceWin {
  Piece pc;
  int nwin;
};
__device__ __forceinline__ PieceWin pw_combine(const PieceWin& a, const PieceWin& b) {
  return PieceWin{piece_combine(a.pc, b.pc), a.nwin + b.nwin};
}

template <int ITEMS>
struct alignas(16) FusedSmem {
  double g[TileCfg<ITEMS>::kSmem];
  double send[(ITEMS >> kSegLog2) * kThreads];
  SumCnt wsc[kWarps];   // warp totals of the (sum, count) scan
  PieceWin wpw[kWarps];  // warp totals of the (piece, windows) scan
  Piece wp[kMaxWin];    // piece from the previous window (or the tile start) to each window
  double wg[kMaxWin];   // the window elements
  double wa[kMaxWin];   // exact sums after the windows
  Piece tail;           // piece after the tile's last window (the whole tile if it has none)
  double s_in, s_end;
  int tile, bail;
};

// Where a staging pass puts window w of the tile: the fused kernel's shared
// lists, or the two-pass scan's global tile records.
struct SmemWinSink {
  Piece* wp;
  double* wg;
  __device__ __forceinline__ void put(int w, const Piece& pc, double g) const {
    wp[w] = Piece{pc.d0, pc.d1, pc.e, 0};
    wg[w] = g;
  }
};
struct GlobalWinSink {
  TileWin* tw;
  __device__ __forceinline__ void put(int w, const Piece& pc, double g) const {
    tw[w] = TileWin{g, pc.e, 0, pc.d0, pc.d1};
  }
};
struct NoWinSink {
  __device__ __forceinline__ void put(int, const Piece&, double) const {}
};

// The general per-chunk path of the tile analysis (chunks that hold a window
// or an exact rounding tie: ~log2 N chunks per scan, but they sit on the
// critical path - the first tile's successors wait for it): element by
// element with running scalars, no arrays. STAGE = false: the chunk's
// aggregate piece and window count; STAGE = true (after the block scan): the
// chunk's windows handed to the sink in tile order, each with the piece since
// the previous window. The per-element rule is classify() of exact_cdf.cuh: the
// bound at the element's start is the bound at the previous element's end.
template <int ITEMS, bool STAGE, class Sink>
__device__ __forceinline__ void chunk_general(const double* my, double p0, long long cnt0, Piece carry, int win_excl,
                                              const Sink& sink, Piece& agg, int& nwin) {
  Piece acc = STAGE ? carry : piece_identity();
  int nw = 0;
  double p = p0;
  long long cnt = cnt0;
  double lo = p - sum_bound(p, cnt);
#pragma unroll 1
  for (int i = 0; i < ITEMS; ++i) {
    const double g = my[i];
    if (g == 0.0) continue;  // identity
    const double pn = p + g;
    ++cnt;
    const double En = sum_bound(pn, cnt);
    const int e_lo = binade_of(lo), e_hi = binade_of(pn + En);
    if (e_lo != e_hi) {  // window: applied with a real IEEE add by the tile's resolver
      if (STAGE) sink.put(win_excl + nw, acc, g);
      ++nw;
      acc = Piece{0, 0, kNoBinade, 1};
    } else {
      const UlpScale scale = ulp_scale(e_lo);
      const double v = (g * scale.s1) * scale.s2;  // exact: g < 2^(e+1)
      const double q = rint(v);                    // ties to the even neighbour
      const double diff = v - q;                   // exact
      Piece pc{static_cast<long long>(q), 0, e_lo, 0};
      pc.d1 = pc.d0 + (fabs(diff) == 0.5 ? static_cast<long long>(diff + diff) : 0);  // odd running sum: the odd neighbour
      acc = piece_combine(acc, pc);
    }
    p = pn;
    lo = pn - En;
  }
  agg = acc;
  nwin = nw;
}

// What a thread knows about its chunk after the tile's two block scans.
struct TileChunk {
  double p0;        // approximate prefix before the chunk
  long long cnt0;   // nonzero elements before the chunk
  Piece agg;        // the chunk's aggregate piece (cut at its windows)
  Piece carry;      // the piece since the last window before the chunk (since the tile start if none)
  int nwin;         // windows in the chunk
  int win_excl;     // windows in the tile before the chunk
};

// The tile analysis shared by the single-pass scan and the two-pass records
// kernel: stage g = exp(lg - lse) in shared memory, scan (sum, nonzero count)
// for the chunks' approximate prefixes, classify each chunk (common path:
// integer steps; else chunk_general), scan (piece, windows). Two barriers
// after the staging one.
template <int ITEMS>
__device__ __forceinline__ void tile_analyse(const Ctx& c, int t, long long base, int valid, double* sg, SumCnt* wsc,
                                             PieceWin* wpw, TileChunk& out, int& win_total) {
  using TC = TileCfg<ITEMS>;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  {
    // stage g = exp(lg - lse) (fitness_weights, filter.cpp:154): all loads in flight, then the exps
    const double lse = c.st->lse_g;
    const double* src = c.gin ? c.gin : c.lg;
    double x[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int e = i * kThreads + threadIdx.x;
      x[i] = e < valid ? __ldcs(&src[base + e]) : 0.0;
    }
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int e = i * kThreads + threadIdx.x;
      double g = 0.0;
      if (e < valid) g = c.gin ? x[i] : exp(x[i] - lse);
      sg[TC::sidx(e)] = g;
    }
  }
  __syncthreads();
  // ---- approximate prefix of the thread's chunk (block scan of (sum, nonzero count), one barrier)
  const double* my = &sg[TC::sidx(threadIdx.x * ITEMS)];  // the chunk is contiguous (one pad per chunk)
  SumCnt mine{0.0, 0};
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const double g = my[i];
    mine.s += g;
    mine.c += (g != 0.0);
  }
  SumCnt inc = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double ys = __shfl_up_sync(0xffffffffu, inc.s, o);
    const long long yc = __shfl_up_sync(0xffffffffu, inc.c, o);
    if (lane >= o) {
      inc.s = ys + inc.s;
      inc.c += yc;
    }
  }
  if (lane == 31) wsc[wid] = inc;
  __syncthreads();
  double p0 = c.shard_off[0] + __ldcg(&c.tile_pre[t]);
  long long cnt0 = static_cast<long long>(c.shard_off[1]) + __ldcg(&c.tile_cnt_pre[t]);
  {
    SumCnt pre{0.0, 0};
    for (int w = 0; w < wid; ++w) {
      pre.s = pre.s + wsc[w].s;
      pre.c += wsc[w].c;
    }
    p0 += pre.s + (inc.s - mine.s);
    cnt0 += pre.c + (inc.c - mine.c);
  }
  // ---- chunk analysis. Common path: the whole chunk certainly inside one
  // binade and no exact tie => element i is the integer step rint(g / ulp);
  // anything else goes through the general element-by-element code.
  const int lcn = static_cast<int>(mine.c);
  Piece agg = piece_identity();
  int nwin = 0;
  if (lcn != 0) {
    double pend = p0;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) pend = pend + my[i];
    const double E = sum_bound(pend, cnt0 + lcn);
    const int e_lo = binade_of(p0 - E), e_hi = binade_of(pend + E);
    bool general = e_lo != e_hi;
    if (!general) {
      const UlpScale scale = ulp_scale(e_lo);
      long long acc = 0;
      bool tie = false;
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        const double v = (my[i] * scale.s1) * scale.s2;  // exact: g < 2^(e+1)
        const double q = rint(v);
        tie |= fabs(v - q) == 0.5;  // v - q is exact
        acc += static_cast<long long>(q);
      }
      general = tie;
      agg = Piece{acc, acc, e_lo, 0};
    }
    if (general) chunk_general<ITEMS, false>(my, p0, cnt0, piece_identity(), 0, NoWinSink{}, agg, nwin);
  }
  // ---- segmented scan of the chunk pieces + window counts (one barrier)
  PieceWin pinc{agg, nwin};
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    PieceWin y;
    y.pc = shfl_up_piece(pinc.pc, o);
    y.nwin = __shfl_up_sync(0xffffffffu, pinc.nwin, o);
    if (lane >= o) pinc = pw_combine(y, pinc);
  }
  if (lane == 31) wpw[wid] = pinc;
  PieceWin pex;
  pex.pc = shfl_up_piece(pinc.pc, 1);
  pex.nwin = __shfl_up_sync(0xffffffffu, pinc.nwin, 1);
  if (lane == 0) pex = PieceWin{piece_identity(), 0};
  __syncthreads();
  win_total = 0;
  {
    PieceWin pre{piece_identity(), 0};
    for (int w = 0; w < kWarps; ++w) {
      const PieceWin x = wpw[w];
      if (w < wid) pre = pw_combine(pre, x);
      win_total += x.nwin;
    }
    pex = pw_combine(pre, pex);
  }
  out.p0 = p0;
  out.cnt0 = cnt0;
  out.agg = agg;
  out.carry = pex.pc;
  out.nwin = nwin;
  out.win_excl = pex.nwin;
}

template <int ITEMS, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_scan_fused(Ctx c) {
  using TC = TileCfg<ITEMS>;
  __shared__ FusedSmem<ITEMS> sm;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const bool err = grid_error(c);
  if (threadIdx.x == 0) {
    sm.tile = static_cast<int>(atomicAdd(&c.cnt_scan[2], 1u));
    sm.bail = 0;
  }
  const unsigned tag = __ldcg(&c.cnt_scan[3]) + 1u;  // launch epoch (bumped by the block that finishes last)
  __syncthreads();
  const int t = sm.tile;
  if (!err) {
    const bool last_tile = t == static_cast<int>(gridDim.x) - 1;
    if (threadIdx.x == 0 && t == 0) c.st->tstamp[0] = global_ns();
    if (threadIdx.x == 0 && last_tile) c.st->tstamp[1] = global_ns();
#ifdef PFSMC_SCAN_TRACE
    unsigned long long* ttr = reinterpret_cast<unsigned long long*>(c.trec) + 8 * static_cast<size_t>(t);
    if (threadIdx.x == 0) {
      unsigned smid;
      asm("mov.u32 %0, %%smid;" : "=r"(smid));
      ttr[0] = global_ns();
      ttr[5] = smid;
    }
#endif
    const long long base = static_cast<long long>(t) * TC::kTileT;
    const int valid = static_cast<int>(min(static_cast<long long>(TC::kTileT), c.N - base));
    const double* my = &sm.g[TC::sidx(threadIdx.x * ITEMS)];  // the thread's chunk is contiguous (one pad per chunk)
    TileChunk ch;
    int win_total;
    tile_analyse<ITEMS>(c, t, base, valid, sm.g, sm.wsc, sm.wpw, ch, win_total);
    const double p0 = ch.p0;
    const long long cnt0 = ch.cnt0;
    const Piece agg = ch.agg, carry = ch.carry;
    const int nwin = ch.nwin, win_excl = ch.win_excl;
    const bool overflow = win_total > kMaxWin;
    if (threadIdx.x == kThreads - 1) {
      const Piece tail = piece_combine(carry, agg);
      sm.tail = tail;
      if (win_total == 0) publish_agg(&c.look_agg[t], tail, tag, &c.st->error);  // window-free: successors compose through it at once
    }
    if (nwin > 0 && !overflow) {
      Piece a2;
      int n2;
      chunk_general<ITEMS, true>(my, p0, cnt0, carry, win_excl, SmemWinSink{sm.wp, sm.wg}, a2, n2);
    }
    __syncthreads();
    // the look-back warp differs from tile to tile (tiles sharing an SM arrive 148 apart; warp w issues on
    // scheduler w % 4), so co-resident tiles' look-backs do not share an issue port
    const int lbw = (t / 37) & 3;  // 148 = 4 * 37
    if (wid == lbw) {
      bool ok = true, bail = false;
      if (lane == 0 && last_tile) c.st->tstamp[3] = global_ns();
#ifdef PFSMC_SCAN_TRACE
      if (lane == 0) ttr[1] = global_ns();
#endif
      double s = look_back(c, t, tag, ok, bail);
      if (lane == 0 && last_tile) c.st->tstamp[4] = global_ns();
#ifdef PFSMC_SCAN_TRACE
      if (lane == 0) ttr[2] = global_ns();
#endif
      if (lane == 0) {
        const double s_in = s;
        if (!bail) {
          if (overflow) {
            // serial tile (window overflow): the plain sequential sum, in place
            for (int e = 0; e < valid; ++e) {
              s = s + sm.g[TC::sidx(e)];
              sm.g[TC::sidx(e)] = s;
            }
          } else {
            for (int w = 0; w < win_total; ++w) {
              ok &= piece_apply(sm.wp[w], s);
              s = s + sm.wg[w];  // the window element: a real IEEE add, as acc += g[i]
              sm.wa[w] = s;
            }
            ok &= piece_apply(sm.tail, s);
          }
          if (!last_tile) {
            publish_pre(&c.look_pre[t], s, tag);
          } else {
            c.st->total_mass = s;
            s = (s < 1.0) ? 1.0 : s;  // guard the last bin (filter.cpp:168)
          }
          if (!ok) atomicOr(&c.st->error, kErrInternal);
          c.tile_info[t] = make_double2(s_in, s);  // the search reads the last tile's end (find_segment)
        }
        sm.s_in = s_in;
        sm.s_end = s;
        sm.bail = bail;
      }
    }
    __syncthreads();
    if (!sm.bail) {
      const double2 ti = make_double2(sm.s_in, sm.s_end);
      double vals[ITEMS];
      bool ok = true;
      if (overflow) {
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) vals[i] = threadIdx.x * ITEMS + i < valid ? my[i] : 0.0;
      } else {
        // the exact sum before the chunk (the carry piece applied to the exact
        // value after the last window before it), then the chunk's elements
        // with real IEEE adds: the sequential CDF itself (filter.cpp:162-167)
        double sk = win_excl > 0 ? sm.wa[win_excl - 1] : ti.x;
        ok = piece_apply(carry, sk);
        double chk = sk;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
          sk = sk + my[i];
          vals[i] = sk;
        }
        // self-check of the piece algebra against the real adds (window-free chunks)
        if (nwin == 0) ok &= piece_apply(agg, chk) && chk == sk;
      }
      if (!ok) atomicOr(&c.st->error, kErrInternal);
      // (each thread rewrites only the staged positions it read: no barrier needed here)
      tile_emit<ITEMS>(c, t, base, valid, vals, ti, sm.g, sm.send);
      if (threadIdx.x == 0 && last_tile) c.st->tstamp[2] = global_ns();
      if (threadIdx.x == 0 && t == 0) c.st->tstamp[5] = global_ns();
#ifdef PFSMC_SCAN_TRACE
      if (threadIdx.x == 0) ttr[3] = global_ns();
#endif
    }
  }
  // launch epilogue: the block that finishes last re-arms the ticket and bumps
  // the epoch (every block read the epoch before its own count, so none of
  // this launch can see the bump)
  if (threadIdx.x == 0) {
    const unsigned old = atomicAdd(&c.cnt_scan[1], 1u);
    if (old == gridDim.x - 1) {
      c.cnt_scan[1] = 0;
      c.cnt_scan[2] = 0;
      c.cnt_scan[3] = tag;
    }
  }
}

// ------------------------------------------------- two-pass exact scan
// The form the sharded step uses (the tile records cross GPUs between the
// passes) and PFSMC_GPU_SCAN_TWO_PASS: the same tile analysis as the fused
// kernel, then the tile's records instead of a look-back.
template <int ITEMS>
struct PiecesSmem {
  union {
    struct {
      double g[TileCfg<ITEMS>::kSmem];
      SumCnt wsc[kWarps];
      PieceWin wpw[kWarps];
    } a;
    ResolverSmem rs;
    WinSmem ws;
  };
};

// S2: the tile analysis; the tile's windows (each with the piece since the
// previous window), its header (window count, tail piece) and the per-thread
// handoff for S3 (carry piece, window rank, the chunk's aggregate piece).
// SHARDED = 0: the last block resolves the exact chain (single handle); 1:
// records only (every rank resolves all shards' records after the allgather,
// k_resolve_global).
template <int ITEMS, int SHARDED>
__global__ void __launch_bounds__(kThreads, (ITEMS == 8 ? 3 : 2)) k_scan_pieces(Ctx c) {
  using TC = TileCfg<ITEMS>;
  __shared__ PiecesSmem<ITEMS> sm;
  __shared__ int s_last;
  if (grid_error(c)) return;
  if (!SHARDED && threadIdx.x == 0 && blockIdx.x == 0) c.st->tstamp[0] = global_ns();
  const int t = blockIdx.x;
  const long long base = static_cast<long long>(t) * TC::kTileT;
  const int valid = static_cast<int>(min(static_cast<long long>(TC::kTileT), c.N - base));
  const double* my = &sm.a.g[TC::sidx(threadIdx.x * ITEMS)];
  TileChunk ch;
  int win_total;
  tile_analyse<ITEMS>(c, t, base, valid, sm.a.g, sm.a.wsc, sm.a.wpw, ch, win_total);
  if (c.store_g) {  // L2-resident sizes: S3 reads g back instead of the exps
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int e = i * kThreads + threadIdx.x;
      if (e < valid) __stcg(&c.cdf[base + e], sm.a.g[TC::sidx(e)]);
    }
  }
  const bool overflow = win_total > kMaxWin;
  c.trec[static_cast<size_t>(t) * kThreads + threadIdx.x] =
      ThreadRec{ch.carry.d0, ch.carry.d1, ch.agg.d0, ch.agg.d1, ch.carry.e, ch.agg.e, ch.win_excl, ch.nwin};
  if (ch.nwin > 0 && !overflow) {
    Piece a2;
    int n2;
    chunk_general<ITEMS, true>(my, ch.p0, ch.cnt0, ch.carry, ch.win_excl,
                               GlobalWinSink{c.win + static_cast<size_t>(t) * kMaxWin}, a2, n2);
  }
  if (threadIdx.x == kThreads - 1) {
    const Piece acc = piece_combine(ch.carry, ch.agg);
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

// S3: the exact per-element CDF from the S2 handoff: the exact value before
// the chunk (the carry piece applied to the exact value after the last window
// before it, or to the tile's exact start), then the chunk's elements by real
// IEEE adds - the sequential CDF itself (filter.cpp:162-167); the chunk's
// aggregate piece is checked against those adds. Then the search tables.
template <int ITEMS>
__global__ void __launch_bounds__(kThreads, (ITEMS == 8 ? 4 : 2)) k_scan_cdf(Ctx c) {
  using TC = TileCfg<ITEMS>;
  __shared__ double sg[TC::kSmem];
  __shared__ double send[(ITEMS >> kSegLog2) * kThreads];
  if (grid_error(c)) return;
  const int t = blockIdx.x;
  const long long base = static_cast<long long>(t) * TC::kTileT;
  const int nwin = __ldcg(&c.hdr[t].nwin);
  const double2 ti = __ldcg(&c.tile_info[t]);
  const int valid = static_cast<int>(min(static_cast<long long>(TC::kTileT), c.N - base));
  double vals[ITEMS];
  if (nwin >= 0) {
    // g = exp(lg - lse) recomputed exactly as S2 did (same inputs, same op), or read back
    const double lse = c.st->lse_g;
    const double2* gsrc = reinterpret_cast<const double2*>((c.gin ? c.gin : c.lg) + base + threadIdx.x * ITEMS);
    double g[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS / 2; ++i) {
      const double2 v = __ldcs(gsrc + i);
      const int e = threadIdx.x * ITEMS + 2 * i;
      g[2 * i] = e < valid ? v.x : 0.0;
      g[2 * i + 1] = e + 1 < valid ? v.y : 0.0;
    }
    if (!c.gin) {
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        const int e = threadIdx.x * ITEMS + i;
        g[i] = e < valid ? exp(g[i] - lse) : 0.0;
      }
    }
    const ThreadRec tr = c.trec[static_cast<size_t>(t) * kThreads + threadIdx.x];
    double sk = tr.win_excl > 0 ? __ldcg(&c.win_after[static_cast<size_t>(t) * kMaxWin + tr.win_excl - 1]) : ti.x;
    bool ok = piece_apply(Piece{tr.d0, tr.d1, tr.e, 0}, sk);
    double chk = sk;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      sk = sk + g[i];
      vals[i] = sk;
    }
    if (tr.nwin == 0) ok &= piece_apply(Piece{tr.a0, tr.a1, tr.ae, 0}, chk) && chk == sk;
    if (!ok) atomicOr(&c.st->error, kErrInternal);
  } else {
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int e = threadIdx.x * ITEMS + i;
      vals[i] = e < valid ? __ldcg(&c.cdf[base + e]) : 0.0;
    }
  }
  tile_emit<ITEMS>(c, t, base, valid, vals, ti, sg, send);
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
    case 3:  // single pass (single handle)
      // 4 CTAs per SM (64 registers) for both tile sizes: measured faster than 3 / 2 (profiles/r02_notes.md)
      if (small) k_scan_fused<8, 4><<<ntiles, kThreads, 0, st>>>(c);
      else k_scan_fused<16, 4><<<ntiles, kThreads, 0, st>>>(c);
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
