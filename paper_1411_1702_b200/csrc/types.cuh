// Host-visible types shared by the host driver and every device-code variant
// (variant.cuh): launch context, per-step parameters, device state, the
// KernelSet interface the host dispatches through, and the per-model
// instantiation entry points (exact and fast arithmetic).
#pragma once
#include <cuda_runtime.h>
#include <cmath>
#include <memory>
#include <vector>

#include "../../include/pfsmc_gpu.h"

namespace pfsmc_gpu {


constexpr int kMaxObs = 8;               // register models (loglik<M> unrolls to this)
constexpr int kMaxObsAdv = 32;           // the advection-diffusion model (20 sites in the reference)
constexpr int kMaxWin = 64;              // windows per tile before serial fallback
constexpr double kNegInf = -INFINITY;

enum ErrBits : int { kErrPredict = 1, kErrChol = 2, kErrUpdate = 4, kErrInternal = 8 };

// Per-step scalars, copied host->device before each step (graph memcpy node).
struct StepParams {
  unsigned long long j;
  double t_prev, h;
  int m;
  int pad;
  double t_obs;       // interval end (the adaptive integrator's t1)
  double y[kMaxObsAdv];  // observations (log y for the lognormal kind)
  double ll_const;    // -0.5 m (log 2pi + log s2)   (filter.cpp:140, host glibc log)
  double sly;         // sum log y (lognormal extension only)
};

// Device-resident sampler state.
struct DevState {
  int cur;            // which record buffer holds the ensemble
  int error;          // ErrBits of the current step
  int chol_failed;    // chol_psd of cov failed (raised at the next proliferation)
  int pad;
  double lse_w;       // logw_n = lw_n - lse_w
  double lse_g;       // fitness log-normaliser of the current step
  double mu[8];       // shrink mean = weighted mean of the current params
  double cov[64];     // cov_u (p x p), p <= 8
  double L[64];       // chol_psd(cov_u), consumed by the next proliferation
  double jitter;
  double trace[2 * 8 + 8 + 1];  // theta mean/var, state mean (d <= 8; larger d: Ctx::xmean), ess
  unsigned long long newton_iters;
  double total_mass;  // exact CDF total (diagnostic)
  unsigned long long tstamp[8];  // %globaltimer probes (diagnostics)
};

struct TileHdr {
  int nwin;  // -1: overflow (serial tile)
  int tail_e;
  long long tail_d0, tail_d1;
};
struct TileWin {
  double g;
  int e;
  int local;  // element index inside the tile
  long long d0, d1;
};

// Where the resolver finds tile t's windows: rank r = t / tiles_per_rank
// holds them at base[r] + (t - r * tiles_per_rank) * kMaxWin (the handle's own
// list, the allgathered copy of every shard's, or the shards' own lists read
// over peer memory).
constexpr int kMaxRanks = 8;
struct WinSrc {
  const TileWin* base[kMaxRanks];
  int tiles_per_rank;
#ifdef __CUDACC__
  __device__ __forceinline__ const TileWin* at(int t, int k) const {
    const int r = t / tiles_per_rank;
    return base[r] + static_cast<size_t>(t - r * tiles_per_rank) * kMaxWin + k;
  }
#endif
};

// Single-pass exact scan (k_scan_fused): what a tile publishes for the
// look-back of its successors. flag = launch epoch + 1 when valid.
struct alignas(16) LookAgg {  // a tile's piece in ONE 16-byte word (value and flag travel together):
  long long d0;               // delta for an even running sum
  unsigned long long meta;    // epoch tag << 32 | binade code << 16 | (d1 - d0 + 1)
};
struct alignas(16) LookPre {  // exact CDF at the tile's last element: one 16-byte word
  double v;                   // (value and flag travel together)
  unsigned flag, pad;
};

// Per-thread handoff from the records phase to the CDF phase of the two-pass
// exact scan: the piece since the last window before the thread's chunk (the
// tile start if none), the chunk's own aggregate piece (checked against the
// real adds), the windows before the chunk and inside it.
struct ThreadRec {
  long long d0, d1;  // carry piece
  long long a0, a1;  // the chunk's aggregate piece
  int e, ae;         // their binades
  int win_excl, nwin;
};

// Immutable launch context (pointers + constants), passed by value.
struct Ctx {
  int N, R, ntiles;
  int m_y, likelihood;
  int obs_idx[kMaxObsAdv];
  double a, one_minus_a, s_prolif;  // s = sqrt(1 - a^2)
  double tol;
  int max_iter;
  unsigned long long seed;
  double two_s2;
  double mconst[8];  // model constants (METABOLIC: lambda, c0, A0, A, t0_input, tau)
  double rtol;       // adaptive BDF(1,2) tolerance (IntegratorSpec.rtol)
  int coarse_bits;  // coarse guide has 2^coarse_bits buckets
  int tile_log2;    // exact-CDF tile = 2^tile_log2 elements (10 or 12)
  int store_g;      // k_scan_pieces also stores g = exp(lg - lse) into cdf (read back by k_scan_cdf as gin)
  int k1_block_log2;  // particles per predict CTA (KernelSet::kt), log2
  // ---- advection-diffusion model (grid m x m, d = m^2; kernels_advdiff.cu) ----
  int adv_m, adv_d;
  const double2* adv_tw;  // (cos, sin)(2 pi k / m), k < m
  const double2* adv_W;   // the DFT matrix e^{-2 pi i k j / m}, m x m
  double* xmean;          // state mean of the trace row (d doubles)
  double* xmean_part;     // its per-chunk partials
  double* rec[2];
  double* payload;     // slot-ordered ancestor payloads {record, ll_bar, index} (R + 2 doubles)
  double* lw;
  double* llbar;
  double* lg;
  double* cdf;
  unsigned* anc;
  double* seg_end;     // exact CDF at the end of each 8-element segment (L2-resident)
  unsigned* coarse;    // guide: bucket b -> first segment with seg_end > b / 2^coarse_bits
  double2* tile_info;  // exact CDF (value before the tile, value at its last element;
                       // the last tile's end carries the guard, filter.cpp:168)
  double* tile_pre;    // approximate exclusive tile prefixes (from the K1 block partials)
  int* blk_cnt;        // K1 blocks: number of finite fitness log-weights
  double* trel;        // per tile: fitness mass relative to its K1 group max
  double* tile_m;      // per tile max (C5 tile-loop LSE), or unused
  struct ThreadRec* trec;  // S2 -> S3 handoff: per-thread prefix and segment carry
  long long* tile_cnt_pre;
  TileHdr* hdr;
  TileWin* win;        // kMaxWin per tile
  double* win_after;   // exact sum after each window (kMaxWin per tile)
  double* part;        // block partials
  double* gpart;       // group partials
  unsigned* cnt_pred;  // last-block counters of k_predict (ngroups + 1)
  unsigned* cnt_upd;   // ... of k_update / k_moments (ngroups + 1)
  unsigned* cnt_scan;  // [1] scan blocks done, [2] k_scan_fused tile ticket, [3] its launch epoch
  LookAgg* look_agg;   // k_scan_fused look-back records (ntiles each)
  LookPre* look_pre;
  const double* gin;   // injected fitness (parity mode) or null
  DevState* st;
  const StepParams* sp;
  // ---- sharding (one handle = one contiguous range of global slots) ----
  long long n0;        // global index of this shard's first slot (keys every stream)
  long long n_glob;    // global particle count
  int sharded;         // 0: the handle is the whole filter
  int rank, world;
  int gntiles;         // tiles over all shards
  int tile0;           // global index of this shard's first tile
  TileHdr* ghdr;       // all shards' tile headers (allgathered)
  TileWin* gwin;       // all shards' tile windows (allgathered, kMaxWin per tile)
  double* gwin_after;  // exact sums after every window (global resolver)
  double2* gtile_info; // exact (start, end) of every global tile
  double* shard_sum;   // [2]: this shard's approximate g total and nonzero count (K1 tail)
  double* shard_off;   // [2]: global approximate offset and count before this shard
};

constexpr int kSegLog2 = 3;  // ancestor-search segment: 8 CDF values = one 64-byte burst

struct KernelSet {
  virtual ~KernelSet() = default;
  virtual void trajectory(const double* prm, const double* times, int T, double t0, double rtol, double tol,
                          int max_iter, double* out, int* status, cudaStream_t s) = 0;
  virtual void predict(const Ctx& c, int grid, cudaStream_t s) = 0;
  virtual void update(const Ctx& c, int grid, cudaStream_t s) = 0;
  virtual void moments(const Ctx& c, int grid, cudaStream_t s, int set_cov) = 0;
  virtual void chol(const Ctx& c, cudaStream_t s) = 0;
  virtual void init(const Ctx& c, int grid, cudaStream_t s, int kind, const double* prm, double lw0) = 0;
  virtual void finish_moments(const Ctx& c, const double* gp, int ngroups, int flags, cudaStream_t s) = 0;
  virtual int moment_width() const = 0;
  // block-per-particle models: ancestors only from the serve pass (the
  // update kernel gathers the ancestor record itself) and the state mean of
  // the trace row in Ctx::xmean
  virtual bool block_model() const { return false; }
  int d = 0, p = 0;
  int kt = 256;  // threads per CTA (= particles per CTA) of predict / update / moments
};

// One translation unit per model instantiates its 9 (family, order) kernel
// sets (kernels_<model>.cu), so the builds run in parallel.
std::unique_ptr<KernelSet> make_kernels_decay(int fam, int order);
std::unique_ptr<KernelSet> make_kernels_lv(int fam, int order);
std::unique_ptr<KernelSet> make_kernels_robertson(int fam, int order);
std::unique_ptr<KernelSet> make_kernels_chain(int fam, int order);
std::unique_ptr<KernelSet> make_kernels_payload(int fam, int order);
std::unique_ptr<KernelSet> make_kernels_metabolic(int fam, int order);
// the same units built with -DPFSMC_FAST=1 --fmad=true (variant.cuh)
std::unique_ptr<KernelSet> make_kernels_decay_fast(int fam, int order);
std::unique_ptr<KernelSet> make_kernels_lv_fast(int fam, int order);
std::unique_ptr<KernelSet> make_kernels_robertson_fast(int fam, int order);
std::unique_ptr<KernelSet> make_kernels_chain_fast(int fam, int order);
std::unique_ptr<KernelSet> make_kernels_metabolic_fast(int fam, int order);
// AdvDiffModel (models.cpp:158-266): one CTA per particle (kernels_advdiff.cu)
std::unique_ptr<KernelSet> make_kernels_advdiff(int fam, int order, int grid_n);
std::vector<double2> adv_twiddles(int m);    // (cos, sin)(2 pi k / m)
std::vector<double2> adv_dft_matrix(int m);  // e^{-2 pi i k j / m}, row-major m x m

// Caller-defined models (include/pfsmc_gpu_model.cuh): a plugin library
// registers, per model id, the factory of its (family, order) kernel sets
// (exact and optionally fast variant) when it is loaded.
using KernelFactory = std::unique_ptr<KernelSet> (*)(int fam, int order);
KernelFactory registered_factory(int model, bool fast);

inline std::unique_ptr<KernelSet> make_kernels(int model, int fam, int order, int grid_n = 0, bool fast = false) {
  if (model >= PFSMC_GPU_MODEL_USER_BASE) {
    KernelFactory f = registered_factory(model, fast);
    return f ? f(fam, order) : nullptr;
  }
  if (fast) {
    switch (model) {
      case PFSMC_GPU_MODEL_DECAY: return make_kernels_decay_fast(fam, order);
      case PFSMC_GPU_MODEL_LOTKA_VOLTERRA: return make_kernels_lv_fast(fam, order);
      case PFSMC_GPU_MODEL_ROBERTSON: return make_kernels_robertson_fast(fam, order);
      case PFSMC_GPU_MODEL_CHAIN8: return make_kernels_chain_fast(fam, order);
      case PFSMC_GPU_MODEL_METABOLIC: return make_kernels_metabolic_fast(fam, order);
    }
    // no separate fast build (the resample microbenchmark has no arithmetic to
    // contract; the advection-diffusion kernels already use explicit fma in
    // their transforms): the exact set serves both
  }
  switch (model) {
    case PFSMC_GPU_MODEL_ADVDIFF: return make_kernels_advdiff(fam, order, grid_n);
    case PFSMC_GPU_MODEL_DECAY: return make_kernels_decay(fam, order);
    case PFSMC_GPU_MODEL_LOTKA_VOLTERRA: return make_kernels_lv(fam, order);
    case PFSMC_GPU_MODEL_ROBERTSON: return make_kernels_robertson(fam, order);
    case PFSMC_GPU_MODEL_CHAIN8: return make_kernels_chain(fam, order);
    case PFSMC_GPU_MODEL_PAYLOAD64: return make_kernels_payload(fam, order);
    case PFSMC_GPU_MODEL_METABOLIC: return make_kernels_metabolic(fam, order);
  }
  return nullptr;
}

}  // namespace pfsmc_gpu
