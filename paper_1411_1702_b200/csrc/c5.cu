// BASELINE config 5 (resample / reduction bandwidth microbenchmark on 64-byte
// records) and the measured-peak helpers (FP64 DFMA, random gather), plus the
// truth-trajectory entry point of the data generator.
#include "sampler_internal.cuh"

namespace pfsmc_gpu {

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
// times (1, d0, d1, d0 d0, d0 d1, d1 d1) and the finite count. The partials
// combine in a fixed two-level tree that does not depend on the grid: groups
// of kC5Group consecutive tiles (combined by the block that finishes a
// group's last tile), then the groups in order (by the block that finishes
// the last group). Bitwise reproducible, and a shard whose range is whole
// groups exports exactly the single handle's group partials (SHARDED: the
// final level runs in k_c5_finish over every rank's groups).
constexpr int kC5Group = 64;  // tiles per group partial
constexpr int kC5V = 6;       // S, A0, A1, B00, B01, B11 (partial = M + 6)

__device__ __forceinline__ void c5_finalize(const Ctx& c, const double* fin, double k0, double k1,
                                            double* s_lse) {
  DevState& st = *c.st;
  const double lse = isfinite(fin[0]) ? fin[0] + log(fin[1]) : kNegInf;
  st.lse_g = lse;
  if (!isfinite(lse)) atomicOr(&st.error, kErrPredict);
  *s_lse = lse;
  const double S = fin[1];
  const double m0 = fin[2] / S, m1 = fin[3] / S;
  st.mu[0] = k0 + m0;
  st.mu[1] = k1 + m1;
  st.cov[0] = fin[4] / S - m0 * m0;
  st.cov[1] = st.cov[2] = fin[5] / S - m0 * m1;
  st.cov[3] = fin[6] / S - m1 * m1;
}

// MOM = 0 (single handle, PFSMC_GPU_C5_SEARCH_SPLIT, second iteration on with unchanged log-weights):
// the pass reads lw only; each tile's five moment sums were made by the previous iteration's gather
// (k_c5_gather_moments: same tile, same thread layout, same tree => the same bits) and are spliced
// into the tile partial here, so each record's theta line is read once per iteration, not twice.
template <int ITEMS, int SHARDED, int MOM = 1>
__global__ void __launch_bounds__(kThreads) k_c5_stats(Ctx c, const double* mpart = nullptr) {
  constexpr int kTileT = ITEMS * kThreads;
  constexpr int V = 7;  // S, A0, A1, B00, B01, B11, finite count
  __shared__ double scratch[kWarps * V];
  __shared__ double fin[kC5V + 1];
  __shared__ int s_flag;
  __shared__ double s_lse;
  if (grid_error(c)) return;
  DevState& st = *c.st;
  const double k0 = st.mu[0], k1 = st.mu[1];
  const double* rec = c.rec[st.cur];
  const int ngroups = (c.ntiles + kC5Group - 1) / kC5Group;
  double* tpart = c.part + static_cast<size_t>(c.ntiles) * (kC5V + 1);  // per-tile partials
  unsigned* gcnt = c.cnt_upd;                                            // [ngroups] + [final]
  for (int t = blockIdx.x; t < c.ntiles; t += gridDim.x) {
    const long long base = static_cast<long long>(t) * kTileT;
    double x[ITEMS];
    double2 th[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const long long k = base + i * kThreads + threadIdx.x;
      x[i] = k < c.N ? __ldcs(&c.lw[k]) : -INFINITY;
      th[i] = (MOM && k < c.N) ? __ldcs(reinterpret_cast<const double2*>(rec + k * c.R + 6))
                               : make_double2(0.0, 0.0);
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
      v[0] += e;
      if (MOM) {
        const double d0 = th[i].x - k0, d1 = th[i].y - k1;
        v[1] += e * d0;
        v[2] += e * d1;
        v[3] += e * (d0 * d0);
        v[4] += e * (d0 * d1);
        v[5] += e * (d1 * d1);
      }
      v[6] += isfinite(x[i]) ? 1.0 : 0.0;
    }
    if (MOM) {
      block_sums<V>(v, scratch);
    } else {  // only the mass and the finite count are summed here (the same per-component tree)
      double v2[2] = {v[0], v[6]};
      block_sums<2>(v2, scratch);
      if (threadIdx.x == 0) {
        v[0] = v2[0];
        v[6] = v2[1];
#pragma unroll
        for (int k = 0; k < 5; ++k) v[1 + k] = __ldcg(&mpart[static_cast<size_t>(t) * 5 + k]);
      }
    }
    const int g = t / kC5Group;
    const int gsize = min(kC5Group, c.ntiles - g * kC5Group);
    if (threadIdx.x == 0) {
      double* tp = tpart + static_cast<size_t>(t) * (kC5V + 1);
      tp[0] = M;
#pragma unroll
      for (int k = 0; k < kC5V; ++k) tp[1 + k] = v[k];
      c.trel[t] = v[0];
      c.tile_m[t] = M;
      c.tile_cnt_pre[t] = static_cast<long long>(v[6]);
      __threadfence();
      const unsigned old = atomicAdd(&gcnt[g], 1u);
      s_flag = old == static_cast<unsigned>(gsize - 1);
      if (s_flag) gcnt[g] = 0;
    }
    __syncthreads();
    if (s_flag) {  // block-uniform: this block completed group g
      __threadfence();
      combine_partials<kC5V, false>(tpart + static_cast<size_t>(g) * kC5Group * (kC5V + 1), gsize,
                                    c.gpart + static_cast<size_t>(g) * (kC5V + 1), scratch);
      __syncthreads();
      if (!SHARDED) {
        if (threadIdx.x == 0) {
          __threadfence();
          const unsigned old = atomicAdd(&gcnt[ngroups], 1u);
          s_flag = old == static_cast<unsigned>(ngroups - 1);
          if (s_flag) gcnt[ngroups] = 0;
        }
        __syncthreads();
        if (s_flag) {  // the last group: the final level, then the tile offsets
          __threadfence();
          combine_partials<kC5V, false>(c.gpart, ngroups, fin, scratch);
          __syncthreads();
          if (threadIdx.x == 0) c5_finalize(c, fin, k0, k1, &s_lse);
          __syncthreads();
          if (isfinite(s_lse)) tile_prefixes(c, s_lse, c.tile_m);
        }
      }
    }
    __syncthreads();
  }
}

// Sharded: every rank combines every rank's group partials (global group
// order = rank order) exactly as the single handle's final level, then its
// own tiles' offsets and its approximate total (phase B).
__global__ void __launch_bounds__(kThreads) k_c5_finish(Ctx c, const double* gall, int ngroups_all) {
  __shared__ double scratch[kWarps * 7];
  __shared__ double fin[kC5V + 1];
  __shared__ double s_lse;
  if (grid_error(c)) return;
  const double k0 = c.st->mu[0], k1 = c.st->mu[1];
  __syncthreads();
  combine_partials<kC5V, false>(gall, ngroups_all, fin, scratch);
  __syncthreads();
  if (threadIdx.x == 0) c5_finalize(c, fin, k0, k1, &s_lse);
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

// PFSMC_GPU_C5_SEARCH_SPLIT: the same search as k_c5_serve writing only the
// ancestors (k_search_only), then this gather: while the search runs, the
// only large random stream is the CDF segments, so the search tables stay in
// L2; the gather is then the bare random-record gather.
__global__ void __launch_bounds__(kThreads) k_c5_gather(Ctx c) {
  if (grid_error(c)) return;
  const long long n = static_cast<long long>(blockIdx.x) * kThreads + threadIdx.x;
  const unsigned a = n < c.N ? __ldcs(&c.anc[n]) : 0u;
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

// The same gather with the NEXT iteration's weighted-moment sums made on the way (the gathered record
// passes through registers): one CTA per exact-CDF tile, thread j visits the tile's slots
// i * 256 + j in order - the stats pass's thread layout - so with e = exp(lw - M_t) (M_t: the tile
// maximum the stats pass of this iteration left in tile_m; lw does not change until the next stats
// pass or the host invalidates) and the same block tree the five sums are bitwise the stats pass's.
template <int ITEMS>
__global__ void __launch_bounds__(kThreads) k_c5_gather_moments(Ctx c, double* mpart) {
  constexpr int kTileT = ITEMS * kThreads;
  constexpr int V = 7;
  __shared__ double scratch[kWarps * V];
  if (grid_error(c)) return;
  const int t = blockIdx.x;
  const long long base = static_cast<long long>(t) * kTileT;
  const int lane = threadIdx.x & 31;
  const int cur = c.st->cur;
  const double k0 = c.st->mu[0], k1 = c.st->mu[1];  // this iteration's mean: what the next stats pass centres on
  const double M = __ldcg(&c.tile_m[t]);
  const double2* src = reinterpret_cast<const double2*>(c.rec[cur]);
  double2* dst = reinterpret_cast<double2*>(c.rec[cur ^ 1]);
  const uint64_t pol = l2_policy_stream();
  double v[V] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll 2
  for (int i = 0; i < ITEMS; ++i) {
    const long long n = base + i * kThreads + threadIdx.x;
    const unsigned a = n < c.N ? __ldcs(&c.anc[n]) : 0u;
    const double x = n < c.N ? __ldcs(&c.lw[n]) : -INFINITY;
    const long long wbase = n - lane;
    double2 th = make_double2(0.0, 0.0);  // theta of THIS lane's slot
#pragma unroll
    for (int q = 0; q < 32; q += 8) {
      const int slot = q + lane / 4, part = lane & 3;
      const unsigned as = __shfl_sync(0xffffffffu, a, slot);
      const long long ns = wbase + slot;
      double2 r = make_double2(0.0, 0.0);
      if (ns < c.N) {
        r = ld_hint(src + static_cast<long long>(as) * 4 + part, pol);
        st_hint(dst + ns * 4 + part, r, pol);
      }
      // the record's last 16 bytes (theta) sit in lane 4 * (slot % 8) + 3 of this sub-round: hand
      // them to the slot's own lane
      const int from = 4 * (lane & 7) + 3;
      const double tx = __shfl_sync(0xffffffffu, r.x, from), ty = __shfl_sync(0xffffffffu, r.y, from);
      if ((lane >> 3) == (q >> 3)) th = make_double2(tx, ty);
    }
    const double e = isnan(x) ? NAN : (x == -INFINITY ? 0.0 : exp(x - M));
    const double d0 = th.x - k0, d1 = th.y - k1;
    v[1] += e * d0;
    v[2] += e * d1;
    v[3] += e * (d0 * d0);
    v[4] += e * (d0 * d1);
    v[5] += e * (d1 * d1);
  }
  block_sums<V>(v, scratch);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < 5; ++k) mpart[static_cast<size_t>(t) * 5 + k] = v[1 + k];
  }
}

// ---- bucketed ancestor search (PFSMC_GPU_C5_SEARCH_BUCKETED) ----
// The slot-order search above reads, per slot, a guide entry, a few segment
// ends and one 64-byte CDF segment at random, then the ancestor's record at
// random: at 2^25 the tables fall out of L2 under the streaming traffic
// (285 B of DRAM reads per slot for 128 B of compulsory random reads,
// profiles/r01_notes.md). Here the uniforms are first partitioned by value
// into 2^k equal ranges of [0, 1) (a counting partition: per-block shared
// histogram, one global reservation per (block, bucket), the items written at
// their reserved positions), then searched and gathered bucket by bucket:
// neighbouring threads search neighbouring uniforms, so the guide, the segment
// ends, the CDF segments and the ancestor records are each read from DRAM
// about once, in a narrow window that stays in L2 (and L1) while the bucket
// is served; the records are written to their slots as 64-byte stores. The
// search itself is unchanged (find_ancestor_warp: upper_bound over the exact
// CDF), so every ancestor is the slot-order one bit for bit; only the order
// in which slots are served changes. Items beyond a bucket's capacity (cap is
// mean + 8 sigma of the binomial count, so essentially never) go to a spill
// list served after the buckets; a spill-list overflow raises kErrInternal.
constexpr int kBucketItems = 16;              // uniforms per thread in the partition pass
constexpr int kSpillCap = 1 << 16;            // spill-list entries
constexpr int kMaxBucketBits = 12;            // <= 4096 buckets (shared histogram)

struct C5Buckets {
  int nb_bits;
  long long cap;
  unsigned* count;  // [NB] fill, [NB] spill count, [NB + 1] spill overflow flag
  double* u;        // NB * cap + kSpillCap
  unsigned* n;
  unsigned* anc;
};

__global__ void __launch_bounds__(kThreads) k_c5_bucket(Ctx c, unsigned long long j, C5Buckets b) {
  __shared__ unsigned hist[1 << kMaxBucketBits];
  __shared__ unsigned base[1 << kMaxBucketBits];
  if (grid_error(c)) return;
  const int nb = 1 << b.nb_bits;
  for (int i = threadIdx.x; i < nb; i += kThreads) hist[i] = 0;
  __syncthreads();
  const long long n0 = static_cast<long long>(blockIdx.x) * (kThreads * kBucketItems);
  double u[kBucketItems];
  unsigned key[kBucketItems];  // bucket << 16 | rank inside this block's bucket run
#pragma unroll
  for (int i = 0; i < kBucketItems; ++i) {
    const long long n = n0 + i * kThreads + threadIdx.x;
    u[i] = -1.0;
    key[i] = 0xffffffffu;
    if (n < c.N) {
      u[i] = resample_uniform(c.seed, j, c.n0 + n);
      const int k = min(static_cast<int>(scale2(u[i], b.nb_bits)), nb - 1);
      key[i] = (static_cast<unsigned>(k) << 16) | atomicAdd(&hist[k], 1u);
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < nb; k += kThreads)
    base[k] = hist[k] ? atomicAdd(&b.count[k], hist[k]) : 0u;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kBucketItems; ++i) {
    if (key[i] == 0xffffffffu) continue;
    const long long n = n0 + i * kThreads + threadIdx.x;
    const int k = static_cast<int>(key[i] >> 16);
    const long long pos = static_cast<long long>(base[k]) + (key[i] & 0xffffu);
    long long at;
    if (pos < b.cap) {
      at = static_cast<long long>(k) * b.cap + pos;
    } else {
      const unsigned s = atomicAdd(&b.count[nb], 1u);
      if (s >= static_cast<unsigned>(kSpillCap)) {
        atomicOr(&c.st->error, kErrInternal);
        continue;
      }
      at = static_cast<long long>(nb) * b.cap + s;
    }
    b.u[at] = u[i];
    b.n[at] = static_cast<unsigned>(n);
  }
}

// Block -> its run of bucket positions: blocks_per_bucket blocks per bucket
// (consecutive, so the grid walks [0, 1) in increasing u), then the spill
// list. Returns false when the whole block lies past the fill (block-uniform);
// else `at` = the block's first position and `rem` = valid positions from it.
__device__ __forceinline__ bool bucket_run(const C5Buckets& b, int blocks_per_bucket, long long& at,
                                           unsigned& rem) {
  const int nb = 1 << b.nb_bits;
  const int k = blockIdx.x / blocks_per_bucket;
  long long i0;
  unsigned filled;
  if (k < nb) {
    i0 = static_cast<long long>(blockIdx.x % blocks_per_bucket) * kThreads;
    filled = min(static_cast<unsigned>(b.cap), __ldcg(&b.count[k]));
    at = static_cast<long long>(k) * b.cap + i0;
  } else {
    i0 = static_cast<long long>(blockIdx.x - nb * blocks_per_bucket) * kThreads;
    filled = min(static_cast<unsigned>(kSpillCap), __ldcg(&b.count[nb]));
    at = static_cast<long long>(nb) * b.cap + i0;
  }
  if (i0 >= filled) return false;
  rem = filled - static_cast<unsigned>(i0);
  return true;
}

__global__ void __launch_bounds__(kThreads) k_c5_bucket_serve(Ctx c, C5Buckets b, int blocks_per_bucket) {
  if (grid_error(c)) return;
  long long at;
  unsigned rem;
  if (!bucket_run(b, blocks_per_bucket, at, rem)) return;
  const bool mine = threadIdx.x < rem;  // valid threads are a prefix of the block
  const double u = mine ? __ldcs(&b.u[at + threadIdx.x]) : -1.0;
  const unsigned n = mine ? __ldcs(&b.n[at + threadIdx.x]) : 0u;
  const unsigned a = find_ancestor_warp<true>(c, u);
  if (mine) b.anc[at + threadIdx.x] = a;
  const int lane = threadIdx.x & 31;
  const int cur = c.st->cur;
  const double2* src = reinterpret_cast<const double2*>(c.rec[cur]);
  double2* dst = reinterpret_cast<double2*>(c.rec[cur ^ 1]);
  const uint64_t wpol = l2_policy_stream();
  const int nvalid = __popc(__ballot_sync(0xffffffffu, mine));
  // four lanes per 64-byte record: the ancestor's record (read through L2,
  // where its bucket neighbours find it) to the slot (one-shot stores)
#pragma unroll
  for (int q = 0; q < 32; q += 8) {
    const int slot = q + lane / 4, part = lane & 3;
    const unsigned as = __shfl_sync(0xffffffffu, a, slot);
    const unsigned ns = __shfl_sync(0xffffffffu, n, slot);
    if (slot < nvalid)
      st_hint(dst + static_cast<long long>(ns) * 4 + part, __ldg(src + static_cast<long long>(as) * 4 + part), wpol);
  }
}

// ctx.anc[n] from the bucket-major (slot, ancestor) pairs: only when the
// step diagnostics are read (pfsmc_gpu_get_step_diagnostics).
__global__ void __launch_bounds__(kThreads) k_c5_bucket_anc(Ctx c, C5Buckets b, int blocks_per_bucket) {
  long long at;
  unsigned rem;
  if (!bucket_run(b, blocks_per_bucket, at, rem) || threadIdx.x >= rem) return;
  c.anc[b.n[at + threadIdx.x]] = b.anc[at + threadIdx.x];
}

// Sharded config 5, exact migration over NVLink peer memory: slot n (global
// n0 + n) draws its uniform, finds its serving rank from the exact global
// shard ranges, searches that rank's CDF tables and copies that rank's
// 64-byte record straight into this rank's next record buffer (four lanes per
// record). remote counts the records that crossed GPUs (NVLink bytes).
__global__ void __launch_bounds__(kThreads) k_c5_pull(Ctx c, PeerTable pt, unsigned long long j,
                                                      unsigned long long* remote) {
  if (grid_error(c)) return;
  const long long n = static_cast<long long>(blockIdx.x) * kThreads + threadIdx.x;
  const bool mine = n < c.N;
  const double u = mine ? resample_uniform(c.seed, j, c.n0 + n) : -1.0;
  const int r = mine ? serving_rank(c, u) : 0;
  const int ntl = c.ntiles;
  const SearchView v{pt.coarse[r], pt.seg_end[r], pt.cdf[r], c.gtile_info[(r + 1) * ntl - 1].y};
  const unsigned a = find_ancestor_warp_view(c, v, u);
  if (mine) c.anc[n] = static_cast<unsigned>(static_cast<long long>(r) * c.N + a);
  const unsigned far = __ballot_sync(0xffffffffu, mine && r != c.rank);
  if ((threadIdx.x & 31) == 0 && far) atomicAdd(remote, static_cast<unsigned long long>(__popc(far)));
  const int lane = threadIdx.x & 31;
  const long long wbase = n - lane;
  const int cur = c.st->cur;
  double2* dst = reinterpret_cast<double2*>(c.rec[cur ^ 1]);
#pragma unroll
  for (int q = 0; q < 32; q += 8) {
    const int slot = q + lane / 4, part = lane & 3;
    const unsigned as = __shfl_sync(0xffffffffu, a, slot);
    const int rs = __shfl_sync(0xffffffffu, r, slot);
    const long long ns = wbase + slot;
    if (ns < c.N) {
      const double2* src = reinterpret_cast<const double2*>(cur ? pt.rec1[rs] : pt.rec0[rs]);
      dst[ns * 4 + part] = __ldcg(src + static_cast<long long>(as) * 4 + part);
    }
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

// ---- sharded config 5 (one global iteration over every GPU's records) ----
int c5_shard_groups(const pfsmc_gpu_sampler* s) { return (s->ntiles + kC5Group - 1) / kC5Group; }
double* c5_group_all(pfsmc_gpu_sampler* s) {
  if (!s->c5_gall) {
    s->c5_gall = s->dalloc<double>(static_cast<size_t>(7) * c5_shard_groups(s) * s->world);
    s->c5_remote = s->dalloc<unsigned long long>(1);
    CK(cudaMemset(s->c5_remote, 0, sizeof(unsigned long long)));
  }
  return s->c5_gall;
}

static void c5_shard_check(pfsmc_gpu_sampler* s) {
  if (s->cfg.model != Payload64Model::ID) throw ConfigError("c5: needs the PAYLOAD64 model");
  if (!s->shard_api) throw ConfigError("c5 shard phases: not a sharded handle");
  if (s->ntiles % kC5Group != 0)
    throw ConfigError("c5 sharded: particles per shard must be a multiple of 64 exact-CDF tiles");
  c5_group_all(s);
}

static void c5_launch_stats(pfsmc_gpu_sampler* s, const Ctx& c, bool sharded) {
  // one wave: 126 (ITEMS 16) / 74 (ITEMS 8) registers => 2 / 3 blocks per SM
  if (c.tile_log2 == 11) {
    const int g = std::min(s->ntiles, s->num_sms * 3);
    if (sharded) k_c5_stats<8, 1><<<g, kThreads, 0, s->stream>>>(c);
    else k_c5_stats<8, 0><<<g, kThreads, 0, s->stream>>>(c);
  } else {
    const int g = std::min(s->ntiles, s->num_sms * 2);
    if (sharded) k_c5_stats<16, 1><<<g, kThreads, 0, s->stream>>>(c);
    else k_c5_stats<16, 0><<<g, kThreads, 0, s->stream>>>(c);
  }
}

static Ctx c5_ctx(pfsmc_gpu_sampler* s) {
  Ctx c = s->ctx;
  c.lg = c.lw;  // the fitness log-weights are the log-weights here
  return c;
}

// The device part of one sharded iteration with NCCL collectives and the
// peer pull.
static void enqueue_c5_shard_iteration(pfsmc_gpu_sampler* s, uint64_t j) {
  const NcclApi& N = nccl_api();
  const Ctx c = c5_ctx(s);
  cudaStream_t st = s->stream;
  const size_t G = static_cast<size_t>(c5_shard_groups(s));
  CK(cudaMemsetAsync(&s->st->error, 0, sizeof(int), st));
  c5_launch_stats(s, c, true);
  NCK(N.AllGather(c.gpart, s->c5_gall, 7 * G, ncclDouble, s->nccl, st));                      // A
  k_c5_finish<<<1, kThreads, 0, st>>>(c, s->c5_gall, static_cast<int>(G) * s->world);
  NCK(N.AllGather(c.shard_sum, s->sums_all, 2, ncclDouble, s->nccl, st));                      // B
  launch_shard_offset(c, s->sums_all, st);
  launch_scan(c, s->ntiles, st, 4);
  NCK(N.AllGather(c.hdr, c.ghdr, sizeof(TileHdr) * static_cast<size_t>(s->ntiles), ncclUint8, s->nccl, st));  // C
  launch_resolve_global(c, s->ntiles, st, peer_winsrc(s));  // windows read over peer memory
  launch_scan(c, s->ntiles, st, 2);
  NCK(N.AllGather(c.shard_sum, s->sums_all, 2, ncclDouble, s->nccl, st));  // every rank's tables complete
  k_c5_pull<<<s->grid, kThreads, 0, st>>>(c, s->peers, j, s->c5_remote);                      // D
  NCK(N.AllGather(c.shard_sum, s->sums_all, 2, ncclDouble, s->nccl, st));  // every pull done before the flip
  k_flip<<<1, 1, 0, st>>>(s->st);
  CK(cudaMemcpyAsync(&s->st_host->error, &s->st->error, sizeof(int), cudaMemcpyDeviceToHost, st));
}

int c5_bpb(const C5Buckets& b) { return static_cast<int>((b.cap + kThreads - 1) / kThreads); }

// Bucket buffers, allocated on the first bucketed iteration: 2^k buckets of
// about 2^16 uniforms each (at most 2^12 buckets), capacity mean + 8 sigma.
C5Buckets c5_buckets(pfsmc_gpu_sampler* s) {
  if (!s->c5_u) {
    int bits = 0;
    while (bits < kMaxBucketBits && (s->N >> (bits + 1)) >= (1LL << 16)) ++bits;
    const double lam = std::ceil(static_cast<double>(s->N) / static_cast<double>(1LL << bits));
    long long cap = static_cast<long long>(lam + 8.0 * std::sqrt(lam)) + kThreads;
    cap = (cap + kThreads - 1) / kThreads * kThreads;
    if (s->c5_cap_override > 0) cap = s->c5_cap_override;
    const size_t slots = (static_cast<size_t>(cap) << bits) + kSpillCap;
    s->c5_nb_bits = bits;
    s->c5_cap = cap;
    s->c5_count = s->dalloc<unsigned>((size_t(1) << bits) + 2);
    s->c5_u = s->dalloc<double>(slots);
    s->c5_n = s->dalloc<unsigned>(slots);
    s->c5_anc = s->dalloc<unsigned>(slots);
  }
  return C5Buckets{s->c5_nb_bits, s->c5_cap, s->c5_count, s->c5_u, s->c5_n, s->c5_anc};
}

// The bucketed iteration leaves its ancestors in bucket order; slot order on
// demand (step diagnostics).
void c5_flush_ancestors(pfsmc_gpu_sampler* s) {
  if (!s->c5_anc_pending) return;
  const C5Buckets b = c5_buckets(s);
  k_c5_bucket_anc<<<(1 << b.nb_bits) * c5_bpb(b) + kSpillCap / kThreads, kThreads, 0, s->stream>>>(s->ctx, b,
                                                                                                      c5_bpb(b));
  CK(cudaGetLastError());
  s->c5_anc_pending = false;
}

}  // namespace pfsmc_gpu

extern "C" {

// ---- BASELINE config 5 microbenchmark entry points (model PAYLOAD64) -----
pfsmc_gpu_status pfsmc_gpu_c5_set_logweights(pfsmc_gpu_sampler* s, double sigma, uint64_t key) {
  return guarded([&] {
    if (s->cfg.model != Payload64Model::ID) throw ConfigError("c5: needs the PAYLOAD64 model");
    s->c5_moments_ready = false;
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
    const bool fuse = s->c5_fuse_moments && s->c5_search == PFSMC_GPU_C5_SEARCH_SPLIT;
    if (fuse && !s->c5_mpart) s->c5_mpart = s->dalloc<double>(static_cast<size_t>(s->ntiles) * 5);
    if (fuse && s->c5_moments_ready) {  // the previous iteration's gather left this ensemble's moment sums
      if (c.tile_log2 == 11)
        k_c5_stats<8, 0, 0><<<std::min(s->ntiles, s->num_sms * 6), kThreads, 0, s->stream>>>(c, s->c5_mpart);
      else
        k_c5_stats<16, 0, 0><<<std::min(s->ntiles, s->num_sms * 6), kThreads, 0, s->stream>>>(c, s->c5_mpart);
    } else if (c.tile_log2 == 11) {
      k_c5_stats<8, 0><<<std::min(s->ntiles, s->num_sms * 3), kThreads, 0, s->stream>>>(c);
    } else {
      k_c5_stats<16, 0><<<std::min(s->ntiles, s->num_sms * 2), kThreads, 0, s->stream>>>(c);
    }
    s->c5_moments_ready = false;
    launch_scan_single(s, c, s->stream);
    if (s->c5_search == PFSMC_GPU_C5_SEARCH_BUCKETED) {
      const C5Buckets b = c5_buckets(s);
      const int nb = 1 << b.nb_bits;
      // the partition pass draws the uniforms; it only needs lse-free data, but
      // runs after the scan so the CDF tables are complete when serving starts
      CK(cudaMemsetAsync(b.count, 0, sizeof(unsigned) * (nb + 1), s->stream));
      const int pgrid = static_cast<int>((s->N + kThreads * kBucketItems - 1) / (kThreads * kBucketItems));
      k_c5_bucket<<<pgrid, kThreads, 0, s->stream>>>(c, j, b);
      k_c5_bucket_serve<<<nb * c5_bpb(b) + kSpillCap / kThreads, kThreads, 0, s->stream>>>(c, b, c5_bpb(b));
      s->c5_anc_pending = true;
    } else if (s->c5_search == PFSMC_GPU_C5_SEARCH_SPLIT) {
      StepParams sp{};
      sp.j = j;
      *s->sp_host = sp;
      CK(cudaMemcpyAsync(s->sp_dev, s->sp_host, sizeof(StepParams), cudaMemcpyHostToDevice, s->stream));
      launch_search_only(c, s->grid, s->stream);
      if (fuse) {
        if (c.tile_log2 == 11) k_c5_gather_moments<8><<<s->ntiles, kThreads, 0, s->stream>>>(c, s->c5_mpart);
        else k_c5_gather_moments<16><<<s->ntiles, kThreads, 0, s->stream>>>(c, s->c5_mpart);
        s->c5_moments_ready = true;  // until the log-weights, the records or the mean change on the host's side
      } else {
        k_c5_gather<<<s->grid, kThreads, 0, s->stream>>>(c);
      }
      s->c5_anc_pending = false;
    } else {
      k_c5_serve<<<s->grid, kThreads, 0, s->stream>>>(c, j);
      s->c5_anc_pending = false;
    }
    k_flip<<<1, 1, 0, s->stream>>>(s->st);
    // the error word reaches the host with the next pfsmc_gpu_synchronize
    CK(cudaMemcpyAsync(&s->st_host->error, &s->st->error, sizeof(int), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaGetLastError());
    return PFSMC_GPU_OK;
  });
}

// ---- sharded config 5: phases (any orchestration) and the native iteration
pfsmc_gpu_status pfsmc_gpu_shard_c5_stats(pfsmc_gpu_sampler* s) {
  return guarded([&] {
    c5_shard_check(s);
    s->c5_fitness_is_lw = true;
    CK(cudaMemsetAsync(&s->st->error, 0, sizeof(int), s->stream));
    c5_launch_stats(s, c5_ctx(s), true);
    CK(cudaGetLastError());
    return PFSMC_GPU_OK;
  });
}

pfsmc_gpu_status pfsmc_gpu_shard_c5_finish(pfsmc_gpu_sampler* s) {
  return guarded([&] {
    c5_shard_check(s);
    k_c5_finish<<<1, kThreads, 0, s->stream>>>(c5_ctx(s), s->c5_gall, c5_shard_groups(s) * s->world);
    CK(cudaGetLastError());
    return PFSMC_GPU_OK;
  });
}

// Phase D of the sharded iteration over peer memory (every rank's CDF tables
// complete, peers attached), then the buffer flip. The caller orders the flip
// after every rank's pull before the next iteration overwrites a record buffer.
pfsmc_gpu_status pfsmc_gpu_shard_c5_pull(pfsmc_gpu_sampler* s, uint64_t j) {
  return guarded([&] {
    c5_shard_check(s);
    if (!s->have_peers) throw ConfigError("shard_c5_pull: no peer table (attach_peers / attach_peers_local)");
    k_c5_pull<<<s->grid, kThreads, 0, s->stream>>>(c5_ctx(s), s->peers, j, s->c5_remote);
    CK(cudaGetLastError());
    return PFSMC_GPU_OK;
  });
}

pfsmc_gpu_status pfsmc_gpu_shard_c5_flip(pfsmc_gpu_sampler* s) {
  return guarded([&] {
    c5_shard_check(s);
    k_flip<<<1, 1, 0, s->stream>>>(s->st);
    CK(cudaMemcpyAsync(&s->st_host->error, &s->st->error, sizeof(int), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaGetLastError());
    return PFSMC_GPU_OK;
  });
}

// Records this rank pulled from other GPUs since the handle was created
// (NVLink traffic of the migration = 64 bytes each, plus the searches).
pfsmc_gpu_status pfsmc_gpu_shard_c5_remote_pulls(pfsmc_gpu_sampler* s, uint64_t* out) {
  return guarded([&] {
    c5_shard_check(s);
    unsigned long long v = 0;
    CK(cudaMemcpyAsync(&v, s->c5_remote, sizeof(v), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    *out = v;
    return PFSMC_GPU_OK;
  });
}

// One config-5 iteration of the global ensemble (enqueue only; errors at the
// next pfsmc_gpu_synchronize): the five phases with NCCL collectives in
// between and the migration pulled over NVLink peer memory.
pfsmc_gpu_status pfsmc_gpu_shard_c5_iteration(pfsmc_gpu_sampler* s, uint64_t j) {
  return guarded([&] {
    c5_shard_check(s);
    if (!s->nccl) throw ConfigError("shard_c5_iteration: attach_nccl first");
    if (!s->have_peers) throw ConfigError("shard_c5_iteration: attach_peers first");
    enqueue_c5_shard_iteration(s, j);  // eager: 9 launches + 7 collectives per ~ms iteration
    CK(cudaGetLastError());
    return PFSMC_GPU_OK;
  });
}

pfsmc_gpu_status pfsmc_gpu_c5_set_search(pfsmc_gpu_sampler* s, int mode) {
  return guarded([&] {
    if (s->cfg.model != Payload64Model::ID) throw ConfigError("c5: needs the PAYLOAD64 model");
    if (mode < PFSMC_GPU_C5_SEARCH_GUIDE || mode > PFSMC_GPU_C5_SEARCH_SPLIT)
      throw ConfigError("c5_set_search: mode must be PFSMC_GPU_C5_SEARCH_GUIDE, _BUCKETED or _SPLIT");
    s->c5_search = mode;
    s->c5_moments_ready = false;
    return PFSMC_GPU_OK;
  });
}

// Test / A-B knob (not in the public header): 0 = every iteration's stats pass reads theta itself.
pfsmc_gpu_status pfsmc_gpu_c5_debug_fuse_moments(pfsmc_gpu_sampler* s, int on) {
  return guarded([&] {
    s->c5_fuse_moments = on != 0;
    s->c5_moments_ready = false;
    return PFSMC_GPU_OK;
  });
}

// Test knob (not in the public header): bucket capacity override, to drive
// items into the spill list; 0 restores the default.
pfsmc_gpu_status pfsmc_gpu_c5_debug_bucket_cap(pfsmc_gpu_sampler* s, long long cap) {
  return guarded([&] {
    if (s->c5_u) throw ConfigError("c5_debug_bucket_cap: set before the first bucketed iteration");
    s->c5_cap_override = cap;
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
    CK(cudaSetDevice(device));
    int grid_n = 0;
    if (model == PFSMC_GPU_MODEL_ADVDIFF) {
      const double gn = model_consts ? model_consts[0] : 0.0;
      if (!(gn == std::floor(gn)) || gn < 4.0 || gn > 33.0)
        throw ConfigError("advdiff model: the GPU path supports 4 <= n <= 33");
      grid_n = static_cast<int>(gn);
    }
    auto ks = make_kernels(model, PFSMC_GPU_BDF, 0, grid_n);
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
