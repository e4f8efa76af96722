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
#include "sampler_internal.cuh"

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges for nsys / ncu --nvtx

namespace pfsmc_gpu {

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

// The injected weights' gate (weighted_mean_cov, linalg.cpp:395-409): every
// w = exp(logw) finite and >= 0, and their sum; per-thread compensated sums
// over a grid-stride range, then a fixed-order combine by the last block
// (deterministic; within ~1e-15 of the reference's sequential Kahan sum, far
// inside the 1e-12 gate). out[0] = sum, out[1] = 1 if any weight is invalid.
__global__ void __launch_bounds__(kThreads) k_weight_gate(const double* logw, long long n, double* part,
                                                          unsigned* cnt, double* out) {
  __shared__ double ss[kThreads];
  __shared__ int s_last;
  double sum = 0.0, comp = 0.0;
  int bad = 0;
  for (long long i = static_cast<long long>(blockIdx.x) * kThreads + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * kThreads) {
    const double w = exp(logw[i]);
    bad |= !(w >= 0.0) || !isfinite(w);
    const double y = w - comp, t = sum + y;
    comp = (t - sum) - y;
    sum = t;
  }
  bad = __syncthreads_or(bad);
  ss[threadIdx.x] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0, cb = 0.0;
    for (int k = 0; k < kThreads; ++k) {
      const double y = ss[k] - cb, t = b + y;
      cb = (t - b) - y;
      b = t;
    }
    part[2 * blockIdx.x] = b;
    part[2 * blockIdx.x + 1] = bad;
    __threadfence();
    const unsigned old = atomicAdd(cnt, 1u);
    s_last = old == gridDim.x - 1;
    if (s_last) *cnt = 0;
  }
  __syncthreads();
  if (!s_last || threadIdx.x != 0) return;
  __threadfence();
  double b = 0.0, cb = 0.0, anybad = 0.0;
  for (unsigned k = 0; k < gridDim.x; ++k) {
    const double y = __ldcg(&part[2 * k]) - cb, t = b + y;
    cb = (t - b) - y;
    b = t;
    anybad += __ldcg(&part[2 * k + 1]);
  }
  out[0] = b;
  out[1] = anybad;
}

// logw_n = lw_n - lse_w (update_weights' normalisation, filter.cpp:220) into
// a staging buffer for the read-back.
__global__ void k_normalized_logw(const double* lw, const DevState* st, long long n, double* out) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = lw[i] - st->lse_w;
}

__global__ void k_flush(double* buf, long long n) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    buf[i] = static_cast<double>(i);
}

}  // namespace pfsmc_gpu

thread_local std::string g_last_error;

// ---- caller-defined model registry (include/pfsmc_gpu_model.cuh) ----
namespace {
struct UserModel {
  int id, d, p;
  std::string name;
  pfsmc_gpu::KernelFactory exact = nullptr, fast = nullptr;
};
std::vector<UserModel>& user_models() {
  static std::vector<UserModel> v;
  return v;
}
}  // namespace

pfsmc_gpu::KernelFactory pfsmc_gpu::registered_factory(int model, bool fast) {
  for (const UserModel& m : user_models())
    if (m.id == model) return fast && m.fast ? m.fast : m.exact;
  return nullptr;
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

// The device error word is sticky: once a step fails, every later step's
// kernels early-exit (grid_error) until the host has reported it, so a queued
// run of non-blocking steps surfaces the FIRST failure at the next
// synchronize (the reference throws out of filter::run at that step). The
// host clears it after reading it.
void clear_error(pfsmc_gpu_sampler* s) {
  CK(cudaMemsetAsync(&s->st->error, 0, sizeof(int), s->stream));
  CK(cudaStreamSynchronize(s->stream));
  s->st_host->error = 0;
}

void check_error(pfsmc_gpu_sampler* s) {
  const int err = s->st_host->error;
  if (err) clear_error(s);
  if (err & kErrPredict)
    throw NumericalError("total degeneracy: every particle has zero predictive likelihood");
  if (err & kErrChol) throw NumericalError("chol_psd: degenerate covariance");
  if (err & kErrUpdate)
    throw NumericalError("total degeneracy: every repropagated particle has zero likelihood");
  if (err & kErrInternal) throw std::runtime_error("exact CDF: internal inconsistency");
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
  // NVTX ranges name the PhaseTimings phases (filter.hpp:93-99) the kernels replace
  nvtxRangePushA("propagate (k_predict)");
  s->ks->predict(c, s->grid_m, st);
  nvtxRangePop();
  if (timed) CK(cudaEventRecord(ev[1], st));
  nvtxRangePushA("resample (exact CDF scan + ancestor search)");
  {
    // up to 2^22 particles the fitness vector fits L2: the records pass stores
    // g into the CDF buffer and the CDF pass reads it back instead of
    // recomputing the exps (each tile only reads and then rewrites its own range)
    if (s->scan_mode == PFSMC_GPU_SCAN_FUSED) {
      launch_scan(c, s->ntiles, st, 3);  // single pass; the k_scan_cdf slot of the kernel times stays ~0
      if (timed) CK(cudaEventRecord(ev[2], st));
    } else {
      Ctx cp = c, cc = c;
      cp.store_g = s->N <= (1LL << 22) && !c.gin;
      if (cp.store_g) cc.gin = c.cdf;
      launch_scan(cp, s->ntiles, st, 1);
      if (timed) CK(cudaEventRecord(ev[2], st));
      launch_scan(cc, s->ntiles, st, 2);
    }
  }
  if (timed) CK(cudaEventRecord(ev[3], st));
  if (s->ks->block_model())
    launch_search_only(c, s->grid, st);  // the update CTAs gather their ancestor themselves
  else
    launch_serve(c, s->grid, st);
  nvtxRangePop();
  if (timed) CK(cudaEventRecord(ev[4], st));
  nvtxRangePushA("proliferate + repropagate + weights (k_update)");
  s->ks->update(c, s->grid_m, st);
  nvtxRangePop();
  if (timed) CK(cudaEventRecord(ev[5], st));
  CK(cudaGetLastError());
}

// Step prologue: clear the per-step Newton-iteration counter. (The error
// word is NOT cleared here: it is sticky, see check_error.)
void enqueue_prologue(pfsmc_gpu_sampler* s) {
  CK(cudaMemsetAsync(&s->st->newton_iters, 0, sizeof(unsigned long long), s->stream));
}

// The step's host-visible state: DevState (+ the trace row's state mean for
// the block-per-particle models, Ctx::xmean).
void enqueue_readback(pfsmc_gpu_sampler* s) {
  CK(cudaMemcpyAsync(s->st_host, s->st, sizeof(DevState), cudaMemcpyDeviceToHost, s->stream));
  if (s->xmean_host)
    CK(cudaMemcpyAsync(s->xmean_host, s->ctx.xmean, sizeof(double) * s->d, cudaMemcpyDeviceToHost, s->stream));
}

// TraceRow (filter.hpp:67-75): theta_mean[p], theta_var[p], state_mean[d], ess.
void fill_trace(const pfsmc_gpu_sampler* s, const DevState& h, const double* xmean, double* out) {
  const int p = s->p, d = s->d;
  if (!s->ks->block_model()) {
    for (int k = 0; k < 2 * p + d + 1; ++k) out[k] = h.trace[k];
    return;
  }
  // to_natural of the mean (filter.cpp:381-382): AdvDiffModel's k3, c1, c2 are not log-space
  for (int k = 0; k < p; ++k) out[k] = k < 2 ? h.trace[k] : h.mu[k];
  for (int k = p; k < 2 * p; ++k) out[k] = h.trace[k];
  for (int k = 0; k < d; ++k) out[2 * p + k] = xmean[k];
  out[2 * p + d] = h.trace[2 * p + 1];  // AdvThetaView: one placeholder state slot, then ess
}

void build_graph(pfsmc_gpu_sampler* s) {
  cudaGraph_t g;
  CK(cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal));
  enqueue_prologue(s);
  enqueue_kernels(s, false);
  enqueue_readback(s);
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
// The reference's checks on the Ensemble handed to pf_step that the device
// path would not repeat (it normalises weights itself and keeps cov_u
// symmetric by construction): weighted_mean_cov's weight gate in shrink
// (linalg.cpp:395-409, filter.cpp:107-122) and chol_psd's symmetry check in
// proliferate (linalg.cpp:474-480, filter.cpp:185-187). Run on the host at
// injection; the failure is raised by the next step, where the reference
// raises it.
void ensure_staging(pfsmc_gpu_sampler* s) {
  if (s->stage_x) return;
  const size_t N = static_cast<size_t>(s->N);
  s->stage_x = s->dalloc<double>(N * s->d);
  s->stage_t = s->dalloc<double>(N * s->p);
  s->stage_w = s->dalloc<double>(N);
  s->gate_part = s->dalloc<double>(2 * static_cast<size_t>(s->num_sms) * 4 + 2);
  s->gate_cnt = s->dalloc<unsigned>(1);
  CK(cudaMemset(s->gate_cnt, 0, sizeof(unsigned)));
  s->gate_out = s->dalloc<double>(2);
}

// dev_logw: the injected log-weights already on the device (ctx.lw).
void check_injected(pfsmc_gpu_sampler* s, const double* dev_logw, const double* cov_u) {
  s->pending_code = 0;
  s->pending_msg.clear();
  ensure_staging(s);
  const int g = static_cast<int>(std::min<long long>((s->N + kThreads - 1) / kThreads, s->num_sms * 4LL));
  k_weight_gate<<<g, kThreads, 0, s->stream>>>(dev_logw, s->N, s->gate_part, s->gate_cnt, s->gate_out);
  CK(cudaGetLastError());
  double res[2];
  CK(cudaMemcpyAsync(res, s->gate_out, sizeof(res), cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  const double wsum = res[0];
  if (res[1] != 0.0) {
    s->pending_code = PFSMC_GPU_ERR_CONFIG;
    s->pending_msg = "weighted_mean_cov: weights must be nonnegative";
    return;
  }
  // a shard holds part of the weights: the gate is the global filter's (the
  // caller's, ShardedFilter.set_ensemble)
  if (!s->shard_api && std::abs(wsum - 1.0) > 1e-12) {
    s->pending_code = PFSMC_GPU_ERR_CONFIG;
    s->pending_msg = "weighted_mean_cov: weights must sum to 1";
    return;
  }
  const int p = s->p;
  for (int i = 0; i < p; ++i)
    for (int j = i + 1; j < p; ++j)
      if (std::abs(cov_u[i * p + j] - cov_u[j * p + i]) > 1e-12) {
        s->pending_code = PFSMC_GPU_ERR_INTERNAL;  // std::invalid_argument in the reference
        s->pending_msg = "chol_psd: matrix must be symmetric";
        return;
      }
}

struct InternalError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void raise_pending(pfsmc_gpu_sampler* s) {
  if (!s->pending_code) return;
  const int code = s->pending_code;
  const std::string msg = s->pending_msg;
  if (code == PFSMC_GPU_ERR_CONFIG) throw ConfigError(msg);
  throw InternalError(msg);
}

void enqueue_step(pfsmc_gpu_sampler* s, const StepParams* host_sp, const StepParams* dev_sp) {
  s->c5_moments_ready = false;
  if (s->shard_api)
    throw ConfigError("step: a shard handle runs only the sharded phases (pfsmc_gpu_shard_step / shard_*)");
  if (!s->have_ensemble) throw ConfigError("step: no ensemble (call set_ensemble or init_*)");
  raise_pending(s);
  s->c5_anc_pending = false;  // this step writes ctx.anc in slot order
  if (dev_sp) {
    CK(cudaMemcpyAsync(s->sp_dev, dev_sp, sizeof(StepParams), cudaMemcpyDeviceToDevice, s->stream));
  } else {
    *s->sp_host = *host_sp;
    CK(cudaMemcpyAsync(s->sp_dev, s->sp_host, sizeof(StepParams), cudaMemcpyHostToDevice, s->stream));
  }
  if (s->timing) {
    enqueue_prologue(s);
    enqueue_kernels(s, true);
    enqueue_readback(s);
  } else {
    CK(cudaGraphLaunch(s->graph, s->stream));
  }
}

extern "C" {

const char* pfsmc_gpu_version(void) { return "pfsmc_gpu 0.2 (sm_100a)"; }

pfsmc_gpu_status pfsmc_gpu_register_model(int id, const char* name, int d, int p, int fast, void* make) {
  return guarded([&] {
    if (id < PFSMC_GPU_MODEL_USER_BASE) throw ConfigError("register_model: ids below PFSMC_GPU_MODEL_USER_BASE are built in");
    if (!make || d < 1 || p < 1 || d > 8 || p > 8) throw ConfigError("register_model: need a factory, 1 <= d, p <= 8");
    auto f = reinterpret_cast<pfsmc_gpu::KernelFactory>(make);
    for (UserModel& m : user_models()) {
      if (m.id != id) continue;
      if (m.d != d || m.p != p) throw ConfigError("register_model: id already registered with other dimensions");
      (fast ? m.fast : m.exact) = f;
      return PFSMC_GPU_OK;
    }
    UserModel m{id, d, p, name ? name : "", nullptr, nullptr};
    (fast ? m.fast : m.exact) = f;
    user_models().push_back(m);
    return PFSMC_GPU_OK;
  });
}

pfsmc_gpu_status pfsmc_gpu_registered_model(int index, int* id, const char** name, int* d, int* p) {
  return guarded([&] {
    if (index < 0 || index >= static_cast<int>(user_models().size())) throw ConfigError("registered_model: no such index");
    const UserModel& m = user_models()[static_cast<size_t>(index)];
    if (id) *id = m.id;
    if (name) *name = m.name.c_str();
    if (d) *d = m.d;
    if (p) *p = m.p;
    return PFSMC_GPU_OK;
  });
}
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
    if (cfg->particles / static_cast<uint64_t>(world) >= (1ULL << 31))
      throw ConfigError("config: particles must be < 2^31 per handle");
    if (cfg->particles >= (1ULL << 32)) throw ConfigError("config: particles must be < 2^32 in total");
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
    const bool adv = cfg->model == PFSMC_GPU_MODEL_ADVDIFF;
    if (cfg->n_obs > static_cast<uint64_t>(adv ? kMaxObsAdv : kMaxObs))
      throw ConfigError(adv ? "config: at most 32 observed components" : "config: at most 8 observed components");
    int grid_n = 0;
    if (adv) {
      // AdvDiffModel(n) (models.cpp:185-188): n >= 3; the GPU path needs a
      // grid side m = n - 1 >= 3 (distinct stencil columns) and <= 32
      const double gn = cfg->model_consts[0];
      if (!(gn == std::floor(gn)) || gn < 3.0) throw ConfigError("advdiff model: grid parameter n must be >= 3");
      if (gn < 4.0 || gn > 33.0) throw ConfigError("advdiff model: the GPU path supports 4 <= n <= 33");
      grid_n = static_cast<int>(gn);
      if (shard_api) throw ConfigError("advdiff model: sharded handles are not supported");
    }
    auto s = std::make_unique<pfsmc_gpu_sampler>();
    s->cfg = *cfg;
    CK(cudaSetDevice(cfg->device));
    // adaptive: the variable-step BDF(1,2) kernels (order slot 0)
    if (cfg->arithmetic != PFSMC_GPU_ARITH_EXACT && cfg->arithmetic != PFSMC_GPU_ARITH_FAST)
      throw ConfigError("config: arithmetic must be PFSMC_GPU_ARITH_EXACT or PFSMC_GPU_ARITH_FAST");
    const bool fast = cfg->arithmetic == PFSMC_GPU_ARITH_FAST;
    s->ks = cfg->adaptive ? make_kernels(cfg->model, PFSMC_GPU_BDF, 0, grid_n, fast)
                          : make_kernels(cfg->model, cfg->family, cfg->order, grid_n, fast);
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
    s->grid_m = static_cast<int>((s->N + s->ks->kt - 1) / s->ks->kt);
    // 2048-element tiles up to 2^22 (4096 at 2^20 measured 10% slower: the
    // per-thread serial chains double, profiles/r02_notes.md)
    const int tile_log2 = s->N <= (1LL << 22) ? 11 : 12;
    s->ntiles = static_cast<int>((s->N + (1LL << tile_log2) - 1) >> tile_log2);
    Ctx& c = s->ctx;
    c.N = static_cast<int>(s->N);
    c.R = ((s->d + s->p + 1) / 2) * 2;
    c.ntiles = s->ntiles;
    c.m_y = static_cast<int>(cfg->n_obs);
    c.likelihood = cfg->likelihood;
    for (int k = 0; k < kMaxObsAdv; ++k) c.obs_idx[k] = k < c.m_y ? static_cast<int>(s->obs[k]) : -1;
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
    // slot-ordered ancestor payloads (k_serve); the block-per-particle
    // models gather inside their update CTAs instead
    c.payload = s->ks->block_model() ? nullptr : s->dalloc<double>(N * (c.R + 2));
    if (adv) {
      const int m = grid_n - 1;
      std::vector<double2> tw = adv_twiddles(m);
      std::vector<double2> W = adv_dft_matrix(m);
      double2* dtw = s->dalloc<double2>(static_cast<size_t>(m) + m * m);
      CK(cudaMemcpy(dtw, tw.data(), sizeof(double2) * m, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(dtw + m, W.data(), sizeof(double2) * m * m, cudaMemcpyHostToDevice));
      c.adv_m = m;
      c.adv_d = m * m;
      c.adv_tw = dtw;
      c.adv_W = dtw + m;
      c.xmean = s->dalloc<double>(static_cast<size_t>(c.adv_d));
      c.xmean_part = s->dalloc<double>(static_cast<size_t>(c.adv_d) * 64);
      CK(cudaMemset(c.xmean, 0, sizeof(double) * c.adv_d));
      CK(cudaMallocHost(&s->xmean_host, sizeof(double) * c.adv_d));
    }
    c.lw = s->dalloc<double>(N);
    c.llbar = s->dalloc<double>(N);
    c.lg = s->dalloc<double>(N);
    c.cdf = s->dalloc<double>(N);
    c.anc = s->dalloc<unsigned>(N);
    c.tile_log2 = tile_log2;
    c.store_g = 0;
    c.k1_block_log2 = ilog2(s->ks->kt);
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
    c.blk_cnt = s->dalloc<int>(static_cast<size_t>(s->grid_m));
    c.trel = s->dalloc<double>(NT);
    c.tile_m = s->dalloc<double>(NT);
    c.trec = s->dalloc<ThreadRec>(NT * kThreads);
    c.tile_pre = s->dalloc<double>(NT);
    c.tile_cnt_pre = s->dalloc<long long>(NT);
    c.look_agg = s->dalloc<LookAgg>(NT);
    c.look_pre = s->dalloc<LookPre>(NT);
    CK(cudaMemset(c.look_agg, 0, sizeof(LookAgg) * NT));
    CK(cudaMemset(c.look_pre, 0, sizeof(LookPre) * NT));
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
    c.part = s->dalloc<double>(static_cast<size_t>(s->grid_m) * vmax + 64);
    c.gpart = s->dalloc<double>(static_cast<size_t>(s->grid_m / kGroup + 2) * vmax + 64);
    const int ngroups = (s->grid_m + kGroup - 1) / kGroup;
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
    s->ngroups_pred = (s->grid_m + kGroup - 1) / kGroup;
    s->ngroups_upd = s->ngroups_pred;
    s->shard_api = shard_api;
    if (shard_api) {
      const int W = s->ks->moment_width();
      s->gp_pred_all = s->dalloc<double>(static_cast<size_t>(world) * s->ngroups_pred * 2);
      s->gp_mom_all = s->dalloc<double>(static_cast<size_t>(world) * s->ngroups_upd * W);
      s->sums_all = s->dalloc<double>(2 * world);
      // sendbuf / recvbuf (counted NCCL exchange only): allocated on first use
      s->counts_dev = s->dalloc<unsigned>(2 * world);
      s->counts_all = s->dalloc<unsigned>(static_cast<size_t>(world) * world);
      CK(cudaMallocHost(&s->counts_host, (2 * world + world * world) * sizeof(unsigned)));
      // offspring-allocation mode (shard.cu)
      s->ocnt = s->dalloc<unsigned>(N + 1);
      s->ooff = s->dalloc<unsigned>(N + 1);
      s->oblk = s->dalloc<unsigned>(N / 2048 + 2);
      s->otot = s->dalloc<unsigned long long>(world);
      s->ocount = s->dalloc<unsigned long long>(world);
      CK(cudaMallocHost(&s->otot_host, world * sizeof(unsigned long long)));
    }
    if (!shard_api) build_graph(s.get());  // shard handles step through the sharded phases only
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
    ensure_staging(s);  // persistent device staging (no allocation per call)
    double* tmp_x = s->stage_x;
    double* tmp_t = s->stage_t;
    CK(cudaMemcpyAsync(tmp_x, states, sizeof(double) * N * d, cudaMemcpyHostToDevice, s->stream));
    CK(cudaMemcpyAsync(tmp_t, params_u, sizeof(double) * N * p, cudaMemcpyHostToDevice, s->stream));
    CK(cudaMemcpyAsync(s->ctx.lw, logw, sizeof(double) * N, cudaMemcpyHostToDevice, s->stream));
    check_injected(s, s->ctx.lw, cov_u);
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
    if (!s->shard_api) s->ks->moments(s->ctx, s->grid_m, s->stream, 0);
    CK(cudaStreamSynchronize(s->stream));
    CK(cudaGetLastError());
    s->have_ensemble = true;
    s->c5_moments_ready = false;
    return PFSMC_GPU_OK;
  });
}

pfsmc_gpu_status pfsmc_gpu_get_ensemble(pfsmc_gpu_sampler* s, double* states, double* params_u,
                                        double* logw, double* mean_u, double* cov_u) {
  return guarded([&] {
    const size_t N = static_cast<size_t>(s->N);
    const int d = s->d, p = s->p;
    ensure_staging(s);
    double* tmp_x = s->stage_x;
    double* tmp_t = s->stage_t;
    k_pack<<<s->grid, kThreads, 0, s->stream>>>(s->ctx, d, p, tmp_x, tmp_t, 1);
    if (states) CK(cudaMemcpyAsync(states, tmp_x, sizeof(double) * N * d, cudaMemcpyDeviceToHost, s->stream));
    if (params_u) CK(cudaMemcpyAsync(params_u, tmp_t, sizeof(double) * N * p, cudaMemcpyDeviceToHost, s->stream));
    DevState h{};
    CK(cudaMemcpyAsync(&h, s->st, sizeof(DevState), cudaMemcpyDeviceToHost, s->stream));
    if (logw) {  // update_weights' lw -= lse (filter.cpp:220) on the device
      k_normalized_logw<<<s->grid, kThreads, 0, s->stream>>>(s->ctx.lw, s->st, s->N, s->stage_w);
      CK(cudaMemcpyAsync(logw, s->stage_w, sizeof(double) * N, cudaMemcpyDeviceToHost, s->stream));
    }
    CK(cudaStreamSynchronize(s->stream));
    CK(cudaGetLastError());
    if (mean_u)
      for (int k = 0; k < p; ++k) mean_u[k] = h.mu[k];
    if (cov_u)
      for (int k = 0; k < p * p; ++k) cov_u[k] = h.cov[k];
    return PFSMC_GPU_OK;
  });
}

static pfsmc_gpu_status do_init(pfsmc_gpu_sampler* s, int kind, const std::vector<double>& prm) {
  return guarded([&] {
    s->pending_code = 0;
    s->pending_msg.clear();
    double* dprm = s->dalloc<double>(prm.size());
    CK(cudaMemcpyAsync(dprm, prm.data(), sizeof(double) * prm.size(), cudaMemcpyHostToDevice, s->stream));
    DevState h{};
    CK(cudaMemcpyAsync(&h, s->st, sizeof(DevState), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    h.lse_w = 0.0;
    h.error = 0;
    h.chol_failed = 0;
    for (int k = 0; k < 8; ++k) h.mu[k] = 0.0;
    CK(cudaMemcpyAsync(s->st, &h, sizeof(DevState), cudaMemcpyHostToDevice, s->stream));
    const double lw0 = -std::log(static_cast<double>(s->cfg.particles));  // filter.cpp:86
    s->ks->init(s->ctx, s->grid, s->stream, kind, dprm, lw0);
    // first pass: mean about 0; second pass: cov about that mean (sharded:
    // the caller runs both passes globally)
    if (!s->shard_api) {
      s->ks->moments(s->ctx, s->grid_m, s->stream, 1);
      s->ks->moments(s->ctx, s->grid_m, s->stream, 1);
    }
    CK(cudaStreamSynchronize(s->stream));
    CK(cudaGetLastError());
    cudaFree(dprm);
    s->allocs.pop_back();
    s->have_ensemble = true;
    s->c5_moments_ready = false;
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
  struct Range {  // NVTX range over the drop-in step
    Range() { nvtxRangePushA("pfsmc_gpu_step (filter::pf_step)"); }
    ~Range() { nvtxRangePop(); }
  } range;
  return guarded([&] {
    const StepParams sp = make_params(s, y, j, t_prev, t_obs, h);
    enqueue_step(s, &sp, nullptr);
    CK(cudaStreamSynchronize(s->stream));
    harvest_timing(s);
    check_error(s);
    if (trace_out) fill_trace(s, *s->st_host, s->xmean_host, trace_out);
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
    if (trace_out) fill_trace(s, *s->st_host, s->xmean_host, trace_out);
    return PFSMC_GPU_OK;
  });
}

pfsmc_gpu_status pfsmc_gpu_run(pfsmc_gpu_sampler* s, double* rows, int* warn) {
  return guarded([&] {
    if (s->shard_api) throw ConfigError("run: a shard handle runs only the sharded phases");
    const int w = 2 * s->p + s->d + 1;
    // row 0 from the current ensemble (filter.cpp:409-426)
    s->ks->moments(s->ctx, s->grid_m, s->stream, 0);
    enqueue_readback(s);
    CK(cudaStreamSynchronize(s->stream));
    fill_trace(s, *s->st_host, s->xmean_host, rows);
    if (warn) warn[0] = 0;
    int streak = 0;
    for (size_t j = 1; j <= s->resident.size(); ++j) {
      enqueue_step(s, nullptr, s->resident_dev + (j - 1));
      CK(cudaStreamSynchronize(s->stream));
      harvest_timing(s);
      check_error(s);
      fill_trace(s, *s->st_host, s->xmean_host, rows + j * w);
      const double ess = rows[j * w + w - 1];
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
    if (ancestors) c5_flush_ancestors(s);
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

// Diagnostics (not in the public header): per-tile timeline of the last
// k_scan_fused launch (start, classification done, look-back done, end; ns,
// plus the SM id), written into the two-pass scan's idle handoff buffer.
pfsmc_gpu_status pfsmc_gpu_debug_tile_times(pfsmc_gpu_sampler* s, uint64_t* out, int ntiles) {
  return guarded([&] {
    CK(cudaMemcpyAsync(out, s->ctx.trec, sizeof(uint64_t) * 8 * std::min(ntiles, s->ntiles), cudaMemcpyDeviceToHost,
                       s->stream));
    CK(cudaStreamSynchronize(s->stream));
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
    s->c5_anc_pending = false;
    launch_gin(c, s->ntiles, s->stream);
    launch_scan_single(s, c, s->stream);
    launch_search_only(c, s->grid, s->stream);
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
    // five event slots in both scan modes; the fused scan leaves the second scan slot empty ("-")
    if (names_out) *names_out = s->scan_mode == PFSMC_GPU_SCAN_FUSED ? kKernelNamesFused : kKernelNames;
    return PFSMC_GPU_OK;
  });
}

pfsmc_gpu_status pfsmc_gpu_set_scan_mode(pfsmc_gpu_sampler* s, int mode) {
  return guarded([&] {
    if (mode != PFSMC_GPU_SCAN_FUSED && mode != PFSMC_GPU_SCAN_TWO_PASS)
      throw ConfigError("set_scan_mode: mode must be PFSMC_GPU_SCAN_FUSED or PFSMC_GPU_SCAN_TWO_PASS");
    if (mode == s->scan_mode) return PFSMC_GPU_OK;
    CK(cudaStreamSynchronize(s->stream));
    s->scan_mode = mode;

    if (s->graph) {  // the blocking step's graph holds the scan launches
      CK(cudaGraphExecDestroy(s->graph));
      s->graph = nullptr;
      build_graph(s);
    }
    return PFSMC_GPU_OK;
  });
}

// Bytes one blocking pfsmc_gpu_step moves between host and device: the step
// parameters up (observations, times, constants), the device state down
// (trace row, error word, moments) and, for block models, the state mean.
pfsmc_gpu_status pfsmc_gpu_step_transfer_bytes(pfsmc_gpu_sampler* s, uint64_t* h2d, uint64_t* d2h) {
  return guarded([&] {
    if (h2d) *h2d = sizeof(StepParams);
    if (d2h) *d2h = sizeof(DevState) + (s && s->xmean_host ? sizeof(double) * s->d : 0);
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
