// One global filter sharded over GPUs: the sharded kernels,
// NCCL bound at run time, the phase-by-phase C ABI, the native step with the
// counted NCCL exchange or the pull over NVLink peer memory.
#include <dlfcn.h>

#include "sampler_internal.cuh"

namespace pfsmc_gpu {

__global__ void __launch_bounds__(kThreads) k_finish_lse(Ctx c, const double* gp, int ngroups) {
  __shared__ double scratch[kWarps * 2];
  __shared__ double fin[2];
  if (grid_error(c)) return;
  __shared__ double s_lse;
  if (threadIdx.x < 32) combine_partials_warp<1, false>(gp, ngroups, fin);  // as tree_reduce_last
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
// {record, ll_bar, ancestor, destination slot} to the slot's owner
// (serving_rank: kernels.cuh).

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

void launch_shard_offset(const Ctx& c, const double* gathered, cudaStream_t st) {
  k_shard_offset<<<1, 32, 0, st>>>(c, gathered);
}

// ---- offspring-allocation mode (north_star) ----------------
// The single handle's multinomial gives slot n the ancestor
// l_n = upper_bound(CDF, u_n) (filter.cpp:169-176); particle i's offspring
// count is o_i = #{n : l_n = i}. Every rank walks the keyed uniforms of ALL
// global slots (identical numbers everywhere, no exchange): the serving rank
// of each u (allgathered exact shard ranges) gives every rank's child total,
// and the uniforms this rank serves are searched in its exact CDF tables, so
// o_i is bitwise the single handle's count. The children are then laid out
// in ancestor order, rank by rank: rank r's children occupy global positions
// [P_r, P_r + O_r), P the exclusive prefix of the totals. Position p belongs
// to rank p / N_local, so a rank builds its own children from its own
// ancestors and only the imbalance (children outside its slot range) crosses
// GPUs.
__global__ void __launch_bounds__(kThreads) k_offspring_walk(Ctx c, unsigned* ocnt, unsigned long long* otot) {
  if (grid_error(c)) return;
  const int lane = threadIdx.x & 31;
  for (long long ng = static_cast<long long>(blockIdx.x) * kThreads + threadIdx.x; ng < c.n_glob;
       ng += static_cast<long long>(gridDim.x) * kThreads) {
    const double u = resample_uniform(c.seed, c.sp->j, ng);
    const int r = serving_rank(c, u);
    const unsigned grp = __match_any_sync(0xffffffffu, r);
    if (lane == __ffs(grp) - 1) atomicAdd(&otot[r], static_cast<unsigned long long>(__popc(grp)));
    const bool mine = r == c.rank;
    if (!__any_sync(0xffffffffu, mine)) continue;
    const unsigned a = find_ancestor_warp(c, mine ? u : -1.0);
    if (mine) atomicAdd(&ocnt[a], 1u);
  }
}

// Exclusive prefix of the per-particle counts (N_local + 1 entries), three
// passes over 2048-element blocks (counts and totals are exact integers).
constexpr int kOffItems = 8;
constexpr int kOffBlock = kOffItems * kThreads;
__global__ void __launch_bounds__(kThreads) k_off_blocksum(const unsigned* cnt, long long n, unsigned* bsum) {
  __shared__ int sw[2 * kWarps];
  const long long base = static_cast<long long>(blockIdx.x) * kOffBlock + threadIdx.x * kOffItems;
  unsigned v = 0;
#pragma unroll
  for (int i = 0; i < kOffItems; ++i) v += base + i < n ? cnt[base + i] : 0u;
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = static_cast<int>(v);
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = 0;
    for (int w = 0; w < kWarps; ++w) t += static_cast<unsigned>(sw[w]);
    bsum[blockIdx.x] = t;
  }
}
__global__ void __launch_bounds__(1024) k_off_scan_blocks(unsigned* bsum, int nb) {
  // one block: exclusive scan of nb block sums (serial per thread chunk + warp scans)
  __shared__ unsigned sw[32];
  const int per = (nb + 1023) / 1024;
  const int b0 = threadIdx.x * per, b1 = min(b0 + per, nb);
  unsigned s = 0;
  for (int b = b0; b < b1; ++b) s += bsum[b];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned x = s;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sw[w] = x;
  __syncthreads();
  if (w == 0) {
    unsigned t = sw[lane];
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    sw[lane] = t;
  }
  __syncthreads();
  unsigned ex = x - s + (w ? sw[w - 1] : 0u);
  for (int b = b0; b < b1; ++b) {
    const unsigned v = bsum[b];
    bsum[b] = ex;
    ex += v;
  }
}
__global__ void __launch_bounds__(kThreads) k_off_apply(const unsigned* cnt, long long n, const unsigned* bsum,
                                                        unsigned* off) {
  __shared__ int sw[2 * kWarps];
  const long long base = static_cast<long long>(blockIdx.x) * kOffBlock + threadIdx.x * kOffItems;
  unsigned v[kOffItems], s = 0;
#pragma unroll
  for (int i = 0; i < kOffItems; ++i) {
    v[i] = base + i < n ? cnt[base + i] : 0u;
    s += v[i];
  }
  int total;
  // block-exclusive scan of the per-thread sums
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned x = s;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sw[w] = static_cast<int>(x);
  __syncthreads();
  if (w == 0) {
    unsigned t = lane < kWarps ? static_cast<unsigned>(sw[lane]) : 0u;
    for (int o = 1; o < kWarps; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < kWarps) sw[kWarps + lane] = static_cast<int>(t);
  }
  __syncthreads();
  total = sw[2 * kWarps - 1];
  (void)total;
  unsigned ex = bsum[blockIdx.x] + x - s + (w ? static_cast<unsigned>(sw[kWarps + w - 1]) : 0u);
#pragma unroll
  for (int i = 0; i < kOffItems; ++i) {
    if (base + i <= n) off[base + i] = ex;  // off[n] = the total
    ex += v[i];
  }
}

// Children of this rank and their global positions from the walk totals.
__device__ __forceinline__ long long offspring_prefix(const Ctx& c, const unsigned long long* otot, int r) {
  long long p = 0;
  for (int q = 0; q < r; ++q) p += static_cast<long long>(otot[q]);
  return p;
}

// The ancestor of local child k: the last i with off[i] <= k (off is the
// exclusive prefix of the counts, so children of i are off[i] .. off[i+1]-1).
__device__ __forceinline__ unsigned child_ancestor(const unsigned* off, long long n, unsigned k) {
  long long lo = 0, hi = n - 1;  // off[lo] <= k < off[hi + 1]
  while (lo < hi) {
    const long long mid = (lo + hi + 1) >> 1;
    if (__ldcg(&off[mid]) <= k) lo = mid;
    else hi = mid - 1;
  }
  return static_cast<unsigned>(lo);
}

// Counted path: this rank's children, packed per destination rank into the
// send regions (dest d at d * cap) as {record, ll_bar, global ancestor,
// local slot on d} — the k_place payload layout.
__global__ void __launch_bounds__(kThreads) k_offspring_pack(Ctx c, const unsigned* off,
                                                             const unsigned long long* otot, double* sendbuf,
                                                             long long cap) {
  if (grid_error(c)) return;
  const long long P = offspring_prefix(c, otot, c.rank);
  const long long O = static_cast<long long>(otot[c.rank]);
  const int W = c.R + kShardPW;
  const double* rec = c.rec[c.st->cur];
  for (long long k = static_cast<long long>(blockIdx.x) * kThreads + threadIdx.x; k < O;
       k += static_cast<long long>(gridDim.x) * kThreads) {
    const long long p = P + k;             // global position of the child
    const int d = static_cast<int>(p / c.N);
    const long long first = max(P, static_cast<long long>(d) * c.N);  // this rank's first child on d
    const unsigned a = child_ancestor(off, c.N, static_cast<unsigned>(k));
    double* dst = sendbuf + (static_cast<long long>(d) * cap + (p - first)) * W;
    const double2* src = reinterpret_cast<const double2*>(rec + static_cast<long long>(a) * c.R);
    for (int i = 0; i < c.R / 2; ++i) reinterpret_cast<double2*>(dst)[i] = __ldg(src + i);
    reinterpret_cast<double2*>(dst)[c.R / 2] = make_double2(__ldg(&c.llbar[a]), static_cast<double>(c.n0 + a));
    reinterpret_cast<double2*>(dst)[c.R / 2 + 1] = make_double2(static_cast<double>(p - static_cast<long long>(d) * c.N), 0.0);
  }
}

// Offspring counts without the global walk (peer memory): each rank draws
// only ITS slots' uniforms, finds the serving rank and the ancestor in that
// rank's tables (warp-cooperative search over peer memory) and increments the
// ancestor's count on its owner with a peer atomic; its slots per serving rank
// go to its own `ocount`. O(N_local) per rank instead of O(N_global); the
// counts are the same integers as the walk's (every slot counted once).
__global__ void __launch_bounds__(kThreads) k_offspring_count_peer(Ctx c, PeerTable pt, unsigned long long* ocount) {
  __shared__ unsigned s_cnt[kMaxRanks];
  if (grid_error(c)) return;
  if (threadIdx.x < kMaxRanks) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  const long long n = static_cast<long long>(blockIdx.x) * kThreads + threadIdx.x;
  const bool mine = n < c.N;
  const double u = mine ? resample_uniform(c.seed, c.sp->j, c.n0 + n) : -1.0;
  const int r = mine ? serving_rank(c, u) : 0;
  const int ntl = c.ntiles;
  const SearchView v{pt.coarse[r], pt.seg_end[r], pt.cdf[r], c.gtile_info[(r + 1) * ntl - 1].y};
  const unsigned a = find_ancestor_warp_view(c, v, u);
  if (mine) atomicAdd(pt.ocnt[r] + a, 1u);
  // slots per serving rank: per warp, then per block in shared memory, one global atomic per
  // (block, rank) - a global atomic per warp on the same word serialises in L2
  const unsigned grp = __match_any_sync(0xffffffffu, mine ? r : -1);
  if (mine && (threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(&s_cnt[r], static_cast<unsigned>(__popc(grp)));
  __syncthreads();
  if (threadIdx.x < kMaxRanks && s_cnt[threadIdx.x])
    atomicAdd(&ocount[threadIdx.x], static_cast<unsigned long long>(s_cnt[threadIdx.x]));
}

// Children per rank, identical on every rank: otot[q] = sum over ranks of
// their slots served by q (every rank's ocount, read over peer memory).
__global__ void k_offspring_totals_peer(Ctx c, PeerTable pt, unsigned long long* otot) {
  const int q = threadIdx.x;
  if (q >= c.world) return;
  unsigned long long t = 0;
  for (int r = 0; r < c.world; ++r) t += __ldcg(&pt.ocount[r][q]);
  otot[q] = t;
}

// Peer-memory path: each slot of this rank pulls its child's ancestor from
// the rank whose children cover that position (mostly itself).
__global__ void __launch_bounds__(kThreads) k_offspring_pull(Ctx c, PeerTable pt, const unsigned long long* otot) {
  if (grid_error(c)) return;
  const long long n = static_cast<long long>(blockIdx.x) * kThreads + threadIdx.x;
  const bool live = n < c.N;
  const long long p = c.n0 + min(n, static_cast<long long>(c.N) - 1);
  int q = 0;
  long long P = 0;
  while (q + 1 < c.world && P + static_cast<long long>(otot[q]) <= p) {
    P += static_cast<long long>(otot[q]);
    ++q;
  }
  const unsigned a = child_ancestor(pt.ooff[q], c.N, static_cast<unsigned>(p - P));
  const long long ga = static_cast<long long>(q) * c.N + a;
  if (live) c.anc[n] = static_cast<unsigned>(ga);
  // warp-cooperative copy (as k_serve): consecutive lanes move consecutive 16-byte parts of the warp's 32
  // payloads, so the stores are coalesced and a record's parts are read together
  const int lane = threadIdx.x & 31;
  const long long wbase = n - lane;
  const int H = c.R / 2 + 1;  // 16-byte parts per payload {record, (ll_bar, global ancestor)}
  const int cur = c.st->cur;
  double2* pay = reinterpret_cast<double2*>(c.payload);
  for (int it = 0; it < H; ++it) {
    const int idx = lane + 32 * it;
    const int slot = idx / H, part = idx - slot * H;
    const unsigned as = __shfl_sync(0xffffffffu, a, slot);
    const int qs = __shfl_sync(0xffffffffu, q, slot);
    const long long ns = wbase + slot;
    if (ns < c.N) {
      double2 v;
      if (part < H - 1)
        v = __ldcg(reinterpret_cast<const double2*>(cur ? pt.rec1[qs] : pt.rec0[qs]) + static_cast<long long>(as) * (H - 1) + part);
      else
        v = make_double2(__ldcg(&pt.llbar[qs][as]), static_cast<double>(static_cast<long long>(qs) * c.N + as));
      pay[ns * H + part] = v;
    }
  }
}

// The resolver's windows read straight from every shard's own list over
// peer memory (phase C without the window allgather: only the tile headers
// are exchanged, and only the windows that exist cross NVLink).
WinSrc peer_winsrc(const pfsmc_gpu_sampler* s) {
  WinSrc ws{};
  for (int r = 0; r < s->world && r < kMaxRanks; ++r) ws.base[r] = s->peers.win[r];
  ws.tiles_per_rank = s->ntiles;
  return ws;
}

}  // namespace pfsmc_gpu

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


// The counted exchange's payload buffers (world x N_local send slots, N_local
// receive slots), allocated on first use: the peer-memory pull and the
// offspring-allocation mode never touch them, so weak scaling does not pay
// world x N_local payloads per GPU for a path it does not run.
void ensure_exchange_buffers(pfsmc_gpu_sampler* s) {
  if (s->sendbuf) return;
  if (!s->shard_api) throw ConfigError("not a sharded handle");
  const size_t PW = static_cast<size_t>(s->ctx.R + kShardPW);
  const size_t N = static_cast<size_t>(s->N);
  s->sendbuf = s->dalloc<double>(static_cast<size_t>(s->world) * N * PW);
  s->recvbuf = s->dalloc<double>(N * PW);
}

// Offspring mode, device part: the global walk (per-particle counts of this
// rank, children per rank) and the prefix of the counts. Enqueued only.
// Exclusive prefix of this rank's per-particle offspring counts (ooff).
static void enqueue_offspring_prefix(pfsmc_gpu_sampler* s) {
  const long long N = s->N;
  const int nb = static_cast<int>(N / kOffBlock + 1);
  k_off_blocksum<<<nb, kThreads, 0, s->stream>>>(s->ocnt, N, s->oblk);
  k_off_scan_blocks<<<1, 1024, 0, s->stream>>>(s->oblk, nb);
  k_off_apply<<<nb, kThreads, 0, s->stream>>>(s->ocnt, N, s->oblk, s->ooff);
}

// Counts by the walk of every global slot (no peer memory needed).
static void enqueue_offspring(pfsmc_gpu_sampler* s) {
  const long long N = s->N;
  CK(cudaMemsetAsync(s->ocnt, 0, sizeof(unsigned) * (N + 1), s->stream));
  CK(cudaMemsetAsync(s->otot, 0, sizeof(unsigned long long) * s->world, s->stream));
  const long long nglob = s->ctx.n_glob;
  const int g = static_cast<int>(std::min<long long>((nglob + kThreads - 1) / kThreads, 148LL * 16));
  k_offspring_walk<<<g, kThreads, 0, s->stream>>>(s->ctx, s->ocnt, s->otot);
  enqueue_offspring_prefix(s);
  CK(cudaGetLastError());
}

// Counts over peer memory, three phases separated by barriers across ranks:
// 0 zero this rank's counts (before the barrier that precedes any rank's
// counting), 1 count this rank's slots into the ancestors' owners (every
// rank's CDF tables complete), 2 (every increment done) the totals and the
// prefix of this rank's counts.
static void enqueue_offspring_peer(pfsmc_gpu_sampler* s, int phase) {
  if (phase == 0) {
    CK(cudaMemsetAsync(s->ocnt, 0, sizeof(unsigned) * (s->N + 1), s->stream));
    CK(cudaMemsetAsync(s->ocount, 0, sizeof(unsigned long long) * s->world, s->stream));
  } else if (phase == 1) {
    k_offspring_count_peer<<<s->grid, kThreads, 0, s->stream>>>(s->ctx, s->peers, s->ocount);
  } else {
    k_offspring_totals_peer<<<1, 32, 0, s->stream>>>(s->ctx, s->peers, s->otot);
    enqueue_offspring_prefix(s);
  }
  CK(cudaGetLastError());
}

// The offspring-mode migration matrix from the children per rank (identical
// on every rank): S[q][d] = |[P_q, P_q + O_q) n [d N, (d + 1) N)|.
static std::vector<uint64_t> offspring_matrix(const unsigned long long* tot, int W, long long N) {
  std::vector<uint64_t> S(static_cast<size_t>(W) * W, 0);
  long long P = 0;
  for (int q = 0; q < W; ++q) {
    const long long a = P, b = P + static_cast<long long>(tot[q]);
    for (int d = 0; d < W; ++d) {
      const long long lo = std::max(a, d * N), hi = std::min(b, (d + 1) * N);
      if (hi > lo) S[static_cast<size_t>(q) * W + d] = static_cast<uint64_t>(hi - lo);
    }
    P = b;
  }
  return S;
}

static void offspring_totals_impl(pfsmc_gpu_sampler* s) {
  enqueue_offspring(s);
  CK(cudaMemcpyAsync(s->otot_host, s->otot, sizeof(unsigned long long) * s->world, cudaMemcpyDeviceToHost,
                     s->stream));
  CK(cudaMemcpyAsync(s->st_host, s->st, sizeof(DevState), cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  check_error(s);
  unsigned long long tot = 0;
  for (int q = 0; q < s->world; ++q) tot += s->otot_host[q];
  if (tot != static_cast<unsigned long long>(s->ctx.n_glob)) throw std::runtime_error("offspring: child total mismatch");
}

static void offspring_pack_impl(pfsmc_gpu_sampler* s) {
  ensure_exchange_buffers(s);
  const long long O = static_cast<long long>(s->otot_host[s->rank]);
  const int g = static_cast<int>(std::max<long long>(1, std::min<long long>((O + kThreads - 1) / kThreads, 148LL * 16)));
  k_offspring_pack<<<g, kThreads, 0, s->stream>>>(s->ctx, s->ooff, s->otot, s->sendbuf, s->N);
  CK(cudaGetLastError());
}

extern "C" {

// ---------------------------------------------------------------- offspring mode
pfsmc_gpu_status pfsmc_gpu_shard_set_mode(pfsmc_gpu_sampler* s, int mode) {
  return guarded([&] {
    if (!s->shard_api) throw ConfigError("not a sharded handle");
    if (mode != PFSMC_GPU_SHARD_EXACT && mode != PFSMC_GPU_SHARD_OFFSPRING)
      throw ConfigError("shard_set_mode: unknown migration mode");
    CK(cudaStreamSynchronize(s->stream));
    if (s->shard_graph) cudaGraphExecDestroy(s->shard_graph);  // captured for the other mode
    s->shard_graph = nullptr;
    s->shard_graph_refused = false;
    s->shard_mode = mode;
    return PFSMC_GPU_OK;
  });
}

pfsmc_gpu_status pfsmc_gpu_shard_offspring(pfsmc_gpu_sampler* s, uint64_t* totals_out) {
  return guarded([&] {
    if (!s->shard_api) throw ConfigError("not a sharded handle");
    offspring_totals_impl(s);
    if (totals_out)
      for (int q = 0; q < s->world; ++q) totals_out[q] = s->otot_host[q];
    return PFSMC_GPU_OK;
  });
}

// Offspring counts over peer memory, phase by phase (see enqueue_offspring_peer;
// the caller puts a barrier across ranks between the phases). Phase 2 also
// returns the children of every rank (world entries, blocking).
pfsmc_gpu_status pfsmc_gpu_shard_offspring_peer(pfsmc_gpu_sampler* s, int phase, uint64_t* totals_out) {
  return guarded([&] {
    if (!s->shard_api) throw ConfigError("not a sharded handle");
    if (!s->have_peers) throw ConfigError("shard_offspring_peer: no peer table (attach_peers / attach_peers_local)");
    if (phase < 0 || phase > 2) throw ConfigError("shard_offspring_peer: phase must be 0, 1 or 2");
    enqueue_offspring_peer(s, phase);
    if (phase == 2) {
      CK(cudaMemcpyAsync(s->otot_host, s->otot, sizeof(unsigned long long) * s->world, cudaMemcpyDeviceToHost,
                         s->stream));
      CK(cudaMemcpyAsync(s->st_host, s->st, sizeof(DevState), cudaMemcpyDeviceToHost, s->stream));
      CK(cudaStreamSynchronize(s->stream));
      check_error(s);
      unsigned long long tot = 0;
      for (int q = 0; q < s->world; ++q) tot += s->otot_host[q];
      if (tot != static_cast<unsigned long long>(s->ctx.n_glob)) throw std::runtime_error("offspring: child total mismatch");
      if (totals_out)
        for (int q = 0; q < s->world; ++q) totals_out[q] = s->otot_host[q];
    }
    return PFSMC_GPU_OK;
  });
}

pfsmc_gpu_status pfsmc_gpu_shard_offspring_counts(pfsmc_gpu_sampler* s, uint32_t* counts_out) {
  return guarded([&] {
    if (!s->shard_api) throw ConfigError("not a sharded handle");
    CK(cudaMemcpyAsync(counts_out, s->ocnt, sizeof(unsigned) * s->N, cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    return PFSMC_GPU_OK;
  });
}

pfsmc_gpu_status pfsmc_gpu_shard_offspring_pack(pfsmc_gpu_sampler* s, uint32_t* matrix_out) {
  return guarded([&] {
    if (!s->shard_api) throw ConfigError("not a sharded handle");
    offspring_pack_impl(s);
    if (matrix_out) {
      const auto S = offspring_matrix(s->otot_host, s->world, s->N);
      for (size_t i = 0; i < S.size(); ++i) matrix_out[i] = static_cast<uint32_t>(S[i]);
    }
    return PFSMC_GPU_OK;
  });
}

pfsmc_gpu_status pfsmc_gpu_shard_offspring_pull(pfsmc_gpu_sampler* s) {
  return guarded([&] {
    if (!s->have_peers) throw ConfigError("shard_offspring_pull: no peer table (attach_peers / attach_peers_local)");
    k_offspring_pull<<<s->grid, kThreads, 0, s->stream>>>(s->ctx, s->peers, s->otot);
    s->ks->update(s->ctx, s->grid_m, s->stream);
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
    if (which == 8 || which == 9) ensure_exchange_buffers(s);
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
      case 12: *ptr = c.gpart; *bytes = sizeof(double) * 7 * c5_shard_groups(s); break;  // config 5
      case 13: *ptr = c5_group_all(s); *bytes = sizeof(double) * 7 * c5_shard_groups(s) * s->world; break;
      default: throw ConfigError("shard_buffer: unknown buffer id");
    }
    if (!s->shard_api && (which == 1 || which == 3 || which >= 7)) throw ConfigError("not a sharded handle");
    return PFSMC_GPU_OK;
  });
}

static void shard_predict_impl(pfsmc_gpu_sampler* s, const double* y, uint64_t j, double t_prev, double t_obs,
                               double h) {
  if (!s->have_ensemble) throw ConfigError("step: no ensemble (call set_ensemble or init_*)");
  raise_pending(s);
  s->c5_fitness_is_lw = false;
  const StepParams sp = make_params(s, y, j, t_prev, t_obs, h);
  CK(cudaStreamSynchronize(s->stream));  // the pinned params slot is free
  *s->sp_host = sp;
  CK(cudaMemcpyAsync(s->sp_dev, s->sp_host, sizeof(StepParams), cudaMemcpyHostToDevice, s->stream));
  enqueue_prologue(s);
  s->ks->predict(s->ctx, s->grid_m, s->stream);
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

// The scan phases' context: the fitness log-weights are lg after a predict
// phase, the log-weights themselves in a config-5 iteration (shard_c5_stats).
static Ctx scan_ctx(const pfsmc_gpu_sampler* s) {
  Ctx c = s->ctx;
  if (s->c5_fitness_is_lw) c.lg = c.lw;
  return c;
}

pfsmc_gpu_status pfsmc_gpu_shard_scan_records(pfsmc_gpu_sampler* s) {
  return guarded([&] {
    const Ctx c = scan_ctx(s);
    k_shard_offset<<<1, 32, 0, s->stream>>>(c, s->sums_all);
    launch_scan(c, s->ntiles, s->stream, 4);
    CK(cudaGetLastError());
    return PFSMC_GPU_OK;
  });
}

pfsmc_gpu_status pfsmc_gpu_shard_resolve(pfsmc_gpu_sampler* s) {
  return guarded([&] {
    const Ctx c = scan_ctx(s);
    launch_scan(c, s->ntiles, s->stream, 5);
    launch_scan(c, s->ntiles, s->stream, 2);
    CK(cudaGetLastError());
    return PFSMC_GPU_OK;
  });
}

// counts_out: [world] payloads this rank sends to each rank, then [world]
// payloads it receives from each rank. Blocking (the exchange needs them).
static void shard_serve_impl(pfsmc_gpu_sampler* s, uint32_t* counts_out) {
  ensure_exchange_buffers(s);
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
    ensure_exchange_buffers(s);
    k_place<<<s->grid, kThreads, 0, s->stream>>>(s->ctx, s->recvbuf, static_cast<long long>(n_recv));
    s->ks->update(s->ctx, s->grid_m, s->stream);
    CK(cudaGetLastError());
    return PFSMC_GPU_OK;
  });
}

pfsmc_gpu_status pfsmc_gpu_shard_moments(pfsmc_gpu_sampler* s) {
  return guarded([&] {
    s->ks->moments(s->ctx, s->grid_m, s->stream, 1);
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

// Drops a previous peer table: the peer-memory step graph captured it by
// value (k_pull's arguments), and its IPC mappings are closed.
static void drop_peers(pfsmc_gpu_sampler* s) {
  CK(cudaStreamSynchronize(s->stream));
  if (s->shard_graph) cudaGraphExecDestroy(s->shard_graph);
  s->shard_graph = nullptr;
  s->shard_graph_refused = false;
  for (void* q : s->ipc_opened) cudaIpcCloseMemHandle(q);
  s->ipc_opened.clear();
  s->peers = PeerTable{};
  s->have_peers = false;
}

// ---- migration over NVLink peer memory --------------------------------------
// The six buffers a peer reads (record buffers, ll_bar, the exact CDF, the
// segment ends, the guide), as CUDA IPC handles: 6 x 64 bytes.
constexpr int kPeerBufs = 10;  // + the offspring prefix and counts (offspring mode), the tile windows

pfsmc_gpu_status pfsmc_gpu_shard_ipc_handles(pfsmc_gpu_sampler* s, uint8_t* out) {
  return guarded([&] {
    if (!s->shard_api) throw ConfigError("not a sharded handle");
    const Ctx& c = s->ctx;
    const void* bufs[kPeerBufs] = {c.rec[0], c.rec[1], c.llbar, c.cdf, c.seg_end, c.coarse, s->ooff, c.win,
                                   s->ocnt, s->ocount};
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
    drop_peers(s);
    const Ctx& c = s->ctx;
    PeerTable t{};
    for (int r = 0; r < s->world; ++r) {
      const void* p[kPeerBufs];
      if (r == s->rank) {
        p[0] = c.rec[0], p[1] = c.rec[1], p[2] = c.llbar, p[3] = c.cdf, p[4] = c.seg_end, p[5] = c.coarse;
        p[6] = s->ooff;
        p[7] = c.win;
        p[8] = s->ocnt;
        p[9] = s->ocount;
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
      t.ooff[r] = static_cast<const unsigned*>(p[6]);
      t.win[r] = static_cast<const TileWin*>(p[7]);
      t.ocnt[r] = static_cast<unsigned*>(const_cast<void*>(p[8]));
      t.ocount[r] = static_cast<unsigned long long*>(const_cast<void*>(p[9]));
    }
    s->peers = t;
    s->have_peers = true;
    return PFSMC_GPU_OK;
  });
}

// Same-process shards (one GPU or P2P-capable GPUs of one process): the peer
// table from the other handles' own device pointers, no IPC. Used to run the
// pull migration phase by phase (pfsmc_gpu_shard_pull) with R shards on one
// GPU, the single-GPU check of the multi-rank pull path.
pfsmc_gpu_status pfsmc_gpu_shard_attach_peers_local(pfsmc_gpu_sampler* s, pfsmc_gpu_sampler* const* shards) {
  return guarded([&] {
    if (!s->shard_api) throw ConfigError("not a sharded handle");
    if (s->world > kMaxRanks) throw ConfigError("attach_peers: at most 8 ranks");
    drop_peers(s);
    PeerTable t{};
    for (int r = 0; r < s->world; ++r) {
      const pfsmc_gpu_sampler* o = shards[r];
      if (!o || !o->shard_api || o->rank != r || o->world != s->world || o->N != s->N || o->ctx.R != s->ctx.R)
        throw ConfigError("attach_peers_local: shards[] must be this filter's handles in rank order");
      const Ctx& c = o->ctx;
      t.rec0[r] = c.rec[0];
      t.rec1[r] = c.rec[1];
      t.llbar[r] = c.llbar;
      t.cdf[r] = c.cdf;
      t.seg_end[r] = c.seg_end;
      t.coarse[r] = c.coarse;
      t.ooff[r] = o->ooff;
      t.win[r] = c.win;
      t.ocnt[r] = o->ocnt;
      t.ocount[r] = o->ocount;
    }
    s->peers = t;
    s->have_peers = true;
    return PFSMC_GPU_OK;
  });
}

// Back to the counted send / receive (e.g. when another rank failed to map
// its peers): unmaps the IPC mappings and drops the peer-memory step graph.
pfsmc_gpu_status pfsmc_gpu_shard_detach_peers(pfsmc_gpu_sampler* s) {
  return guarded([&] {
    CK(cudaSetDevice(s->cfg.device));
    drop_peers(s);
    return PFSMC_GPU_OK;
  });
}

// shard_resolve with the windows read over peer memory (peers attached; every
// shard's scan_records done and the headers allgathered).
pfsmc_gpu_status pfsmc_gpu_shard_resolve_peers(pfsmc_gpu_sampler* s) {
  return guarded([&] {
    if (!s->have_peers) throw ConfigError("shard_resolve_peers: no peer table (attach_peers / attach_peers_local)");
    const Ctx c = scan_ctx(s);
    launch_resolve_global(c, s->ntiles, s->stream, peer_winsrc(s));
    launch_scan(c, s->ntiles, s->stream, 2);
    CK(cudaGetLastError());
    return PFSMC_GPU_OK;
  });
}

// Phase D over peer memory plus the update kernel (replaces shard_serve, the
// payload exchange and shard_update): every peer's tables must be complete
// (the caller orders this after every rank's resolve / CDF phase).
pfsmc_gpu_status pfsmc_gpu_shard_pull(pfsmc_gpu_sampler* s) {
  return guarded([&] {
    if (!s->have_peers) throw ConfigError("shard_pull: no peer table (attach_peers / attach_peers_local)");
    k_pull<<<s->grid, kThreads, 0, s->stream>>>(s->ctx, s->peers);
    s->ks->update(s->ctx, s->grid_m, s->stream);
    CK(cudaGetLastError());
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
  s->ks->predict(c, s->grid_m, st);
  NCK(N.AllGather(c.gpart, s->gp_pred_all, 2 * static_cast<size_t>(s->ngroups_pred), ncclDouble, s->nccl, st));
  k_finish_lse<<<1, kThreads, 0, st>>>(c, s->gp_pred_all, s->ngroups_pred * W);
  NCK(N.AllGather(c.shard_sum, s->sums_all, 2, ncclDouble, s->nccl, st));
  k_shard_offset<<<1, 32, 0, st>>>(c, s->sums_all);
  launch_scan(c, s->ntiles, st, 4);
  // phase C: the headers only; the windows are read over peer memory
  NCK(N.AllGather(c.hdr, c.ghdr, sizeof(TileHdr) * static_cast<size_t>(s->ntiles), ncclUint8, s->nccl, st));
  launch_resolve_global(c, s->ntiles, st, peer_winsrc(s));
  launch_scan(c, s->ntiles, st, 2);
  if (s->shard_mode == PFSMC_GPU_SHARD_OFFSPRING) {
    // counts over peer memory: O(N_local) per rank (k_offspring_count_peer)
    enqueue_offspring_peer(s, 0);
    NCK(N.AllGather(c.shard_sum, s->sums_all, 2, ncclDouble, s->nccl, st));  // tables complete, counts zeroed
    enqueue_offspring_peer(s, 1);
    NCK(N.AllGather(c.shard_sum, s->sums_all, 2, ncclDouble, s->nccl, st));  // every increment done
    enqueue_offspring_peer(s, 2);
    NCK(N.AllGather(c.shard_sum, s->sums_all, 2, ncclDouble, s->nccl, st));  // every rank's prefix complete
    k_offspring_pull<<<s->grid, kThreads, 0, st>>>(c, s->peers, s->otot);
  } else {
    NCK(N.AllGather(c.shard_sum, s->sums_all, 2, ncclDouble, s->nccl, st));  // tables complete everywhere
    k_pull<<<s->grid, kThreads, 0, st>>>(c, s->peers);
  }
  s->ks->update(c, s->grid_m, st);
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
  raise_pending(s);
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

    // D: migration. Exact mode: every slot's ancestor payload from its
    // serving rank (the locally derived count matrix). Offspring mode: this
    // rank's children in ancestor order, only the imbalance to other ranks.
    std::vector<unsigned> omat;
    const unsigned* mat;
    if (s->shard_mode == PFSMC_GPU_SHARD_OFFSPRING) {
      offspring_totals_impl(s);
      offspring_pack_impl(s);
      const auto S = offspring_matrix(s->otot_host, W, s->N);
      omat.assign(S.begin(), S.end());
      mat = omat.data();
    } else {
      std::vector<uint32_t> cnt(2 * static_cast<size_t>(W));
      shard_serve_impl(s, cnt.data());
      mat = s->counts_host + 2 * W;
    }
    const size_t item = sizeof(double) * static_cast<size_t>(c.R + kShardPW);
    const size_t cap = static_cast<size_t>(s->N);
    ensure_exchange_buffers(s);
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
    s->ks->update(c, s->grid_m, st);
    // E: update-kernel moment partials -> global lse_w, moments, trace row, chol
    const size_t Wm = static_cast<size_t>(s->ks->moment_width());
    NCK(N.AllGather(c.gpart, s->gp_mom_all, Wm * s->ngroups_upd, ncclDouble, s->nccl, st));
    CK(cudaGetLastError());
    shard_finish_moments_impl(s, 7, trace_out);
    return PFSMC_GPU_OK;
  });
}

}  // extern "C"
