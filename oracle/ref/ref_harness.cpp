// C-ABI harness over the UNMODIFIED reference sampler, compiled from the
// sources where they lie under /root/reference/proj/src (oracle/Makefile).
//
// TEST INFRASTRUCTURE ONLY. The product never links or loads this library:
// only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
// legs do, as the checker or as the timed CPU baseline.
//
// Entry points mirror the reference's public API:
//   ref_pf_step              -> filter::pf_step         (filter.cpp:292-394)
//   ref_initialize_gaussian  -> filter::initialize      (filter.cpp:76-105)
//   ref_propagate_interval   -> lmm::propagate_interval (lmm.cpp:468-503)
//   ref_fitness_weights      -> filter::fitness_weights (filter.cpp:143-156)
//   ref_resample_multinomial -> filter::resample_multinomial (filter.cpp:158-178)
//   ref_weighted_mean_cov    -> linalg::weighted_mean_cov (linalg.cpp:389-432)
//   ref_chol_psd             -> linalg::chol_psd (linalg.cpp:470-500)
//   ref_philox / ref_stream_draws -> rng (rng.cpp:28-75)
// plus ref_pf_step_ancestors, which replays the first half of pf_step from
// the same public building blocks to expose the ancestor vector that pf_step
// itself keeps internal (filter.cpp:327-336).
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "pfsmc/errors.hpp"
#include "pfsmc/exec.hpp"
#include "pfsmc/filter.hpp"
#include "pfsmc/linalg.hpp"
#include "pfsmc/lmm.hpp"
#include "pfsmc/models.hpp"
#include "pfsmc/rng.hpp"
#include "ref_models.hpp"

using namespace pfsmc;

namespace {
thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const NumericalError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

lmm::Family family_of(int f) {
  switch (f) {
    case 0:
      return lmm::Family::ab;
    case 1:
      return lmm::Family::am;
    default:
      return lmm::Family::bdf;
  }
}
}  // namespace

extern "C" {

// Mirrors the fields of filter::PfConfig / ObservationModel that pf_step
// reads (filter.hpp:30-65), flattened to plain C.
typedef struct ref_cfg {
  int model;        // 0 decay, 1 Lotka-Volterra, 2 Robertson, 3 chain, 5 metabolic
  int family;       // 0 ab, 1 am, 2 bdf
  int order;        // 1..3
  double h;         // fixed LMM step
  double a;         // shrink factor
  uint64_t seed;
  double newton_tol;
  int newton_max_iter;
  const uint64_t* obs_idx;
  uint64_t m_y;
  double sigma;
  int workers;      // 0 sequential, >0 parallel(workers), <0 batched(-workers)
  int adaptive;     // IntegratorSpec.adaptive (variable-step BDF(1,2))
  double rtol;      // IntegratorSpec.rtol
} ref_cfg;

typedef struct ref_ens {
  uint64_t n, d, p;
  double* states;    // n*d
  double* params_u;  // n*p
  double* logw;      // n
  double* mean_u;    // p
  double* cov_u;     // p*p
} ref_ens;

const char* ref_last_error(void) { return g_err.c_str(); }

// Constants of the bound MetabolicModel for the next model construction.
void ref_set_model_consts(const double* k) {
  for (int i = 0; i < 8; ++i) pfsmc_oracle_ref::g_model_consts[i] = k[i];
}

int ref_philox(const uint64_t* ctr, const uint64_t* key, uint64_t* out) {
  return guarded([&] {
    const auto r = rng::philox4x64({ctr[0], ctr[1], ctr[2], ctr[3]},
                                   {key[0], key[1]});
    for (int i = 0; i < 4; ++i) out[i] = r[i];
  });
}

// kind 0: u64, 1: uniform, 2: normal
int ref_stream_draws(uint64_t seed, uint64_t j, uint64_t n, int purpose,
                     int kind, uint64_t count, void* out) {
  return guarded([&] {
    rng::RngStream s(seed, j, n, static_cast<rng::Purpose>(purpose));
    for (uint64_t i = 0; i < count; ++i) {
      if (kind == 0)
        static_cast<uint64_t*>(out)[i] = s.next_u64();
      else if (kind == 1)
        static_cast<double*>(out)[i] = s.next_uniform();
      else
        static_cast<double*>(out)[i] = s.next_normal();
    }
  });
}

}  // extern "C"

namespace {

filter::PfConfig to_pf(const ref_cfg& c, std::size_t n, const models::OdeModel& m) {
  filter::PfConfig cfg;
  cfg.particles = n;
  cfg.shrink_a = c.a;
  cfg.h = c.h;
  cfg.integrator.adaptive = c.adaptive != 0;
  cfg.integrator.family = family_of(c.family);
  cfg.integrator.order = c.order;
  cfg.integrator.rtol = c.rtol;
  cfg.seed = c.seed;
  cfg.newton.tol = c.newton_tol;
  cfg.newton.max_iter = c.newton_max_iter;
  cfg.theta_prior.assign(m.param_dim(), {});
  cfg.x0_prior.assign(m.dim(), {});
  return cfg;
}

filter::ObservationModel to_obs(const ref_cfg& c) {
  filter::ObservationModel o;
  for (uint64_t k = 0; k < c.m_y; ++k) o.indices.push_back(c.obs_idx[k]);
  o.sigma = c.sigma;
  return o;
}

filter::Ensemble load(const ref_ens& e) {
  filter::Ensemble ens;
  ens.n = e.n;
  ens.d = e.d;
  ens.p = e.p;
  ens.states.assign(e.states, e.states + e.n * e.d);
  ens.params_u.assign(e.params_u, e.params_u + e.n * e.p);
  ens.logw.assign(e.logw, e.logw + e.n);
  ens.mean_u.assign(e.mean_u, e.mean_u + e.p);
  ens.cov_u = linalg::DenseMatrix(e.p, e.p);
  ens.cov_u.values.assign(e.cov_u, e.cov_u + e.p * e.p);
  return ens;
}

void store(const filter::Ensemble& ens, ref_ens& e) {
  std::memcpy(e.states, ens.states.data(), sizeof(double) * e.n * e.d);
  std::memcpy(e.params_u, ens.params_u.data(), sizeof(double) * e.n * e.p);
  std::memcpy(e.logw, ens.logw.data(), sizeof(double) * e.n);
  std::memcpy(e.mean_u, ens.mean_u.data(), sizeof(double) * e.p);
  std::memcpy(e.cov_u, ens.cov_u.values.data(), sizeof(double) * e.p * e.p);
}

exec::Backend backend_of(int workers) {
  if (workers > 0) return exec::Backend::parallel(workers);
  if (workers < 0) return exec::Backend::batched(-workers);
  return exec::Backend::sequential();
}

}  // namespace

extern "C" {

// One filter::pf_step on an injected ensemble (in/out). trace_out receives
// theta_mean[p], theta_var[p], state_mean[d], ess (2p+d+1 doubles).
int ref_pf_step(const ref_cfg* c, ref_ens* e, const double* y, uint64_t j,
                double t_prev, double t_obs, double* trace_out,
                double* phase_seconds /* 5 or NULL */) {
  return guarded([&] {
    auto model = pfsmc_oracle_ref::make_model(c->model);
    if (!model) throw ConfigError("unknown model id");
    filter::PfConfig cfg = to_pf(*c, e->n, *model);
    filter::ObservationModel obs = to_obs(*c);
    exec::Backend backend = backend_of(c->workers);
    backend.start();
    filter::Ensemble ens = load(*e);
    filter::PhaseTimings t;
    const auto res = filter::pf_step(ens, {y, c->m_y}, j, t_prev, t_obs, cfg,
                                     backend, *model, obs, &t);
    store(ens, *e);
    const std::size_t p = e->p, d = e->d;
    for (std::size_t k = 0; k < p; ++k) trace_out[k] = res.trace.theta_mean[k];
    for (std::size_t k = 0; k < p; ++k)
      trace_out[p + k] = res.trace.theta_var[k];
    for (std::size_t k = 0; k < d; ++k)
      trace_out[2 * p + k] = res.trace.state_mean[k];
    trace_out[2 * p + d] = res.trace.ess;
    if (phase_seconds) {
      phase_seconds[0] = t.propagate;
      phase_seconds[1] = t.resample;
      phase_seconds[2] = t.proliferate;
      phase_seconds[3] = t.repropagate;
      phase_seconds[4] = t.weights;
    }
  });
}

// Replays shrink -> predict -> log-lik -> fitness -> resample with the public
// building blocks (filter.cpp:301-331) and returns the ancestors pf_step would
// draw, plus the predictor log-likelihoods and the fitness vector g.
int ref_pf_step_ancestors(const ref_cfg* c, const ref_ens* e, const double* y,
                          uint64_t j, double t_prev, double t_obs,
                          int64_t* ancestors, double* loglik_bar, double* g_out) {
  return guarded([&] {
    auto model = pfsmc_oracle_ref::make_model(c->model);
    if (!model) throw ConfigError("unknown model id");
    const std::size_t n = e->n, d = e->d, p = e->p;
    filter::ObservationModel obs = to_obs(*c);
    std::vector<double> params(e->params_u, e->params_u + n * p);
    std::vector<double> logw(e->logw, e->logw + n);
    std::vector<double> tb = filter::shrink(params, n, p, logw, c->a);
    const lmm::LmmScheme scheme =
        lmm::scheme_coefficients(family_of(c->family), c->order);
    lmm::NewtonOpts opts{c->newton_tol, c->newton_max_iter};
    std::vector<double> ll(n);
    std::vector<double> nat(p);
    for (std::size_t i = 0; i < n; ++i) {
      models::to_natural(*model, {tb.data() + i * p, p}, nat);
      // the integrator the config selects (filter.cpp:242-264)
      const auto r = c->adaptive
                         ? lmm::adaptive_bdf_interval(*model, nat, {e->states + i * d, d}, t_prev, t_obs,
                                                      c->rtol, opts)
                         : lmm::propagate_interval(*model, nat, {e->states + i * d, d}, t_prev, t_obs,
                                                   c->h, scheme, opts);
      ll[i] = r.status == lmm::ParticleStatus::ok
                  ? filter::log_likelihood({y, c->m_y}, r.state, obs)
                  : -std::numeric_limits<double>::infinity();
    }
    const std::vector<double> g = filter::fitness_weights(logw, ll);
    const auto anc = filter::resample_multinomial(g, c->seed, j);
    for (std::size_t i = 0; i < n; ++i) {
      ancestors[i] = static_cast<int64_t>(anc[i]);
      if (loglik_bar) loglik_bar[i] = ll[i];
      if (g_out) g_out[i] = g[i];
    }
  });
}

int ref_initialize_gaussian(const ref_cfg* c, uint64_t n, const double* th_mu,
                            const double* th_sigma, const double* x_mean,
                            const double* x_std, const int* x_clamp,
                            ref_ens* e) {
  return guarded([&] {
    auto model = pfsmc_oracle_ref::make_model(c->model);
    if (!model) throw ConfigError("unknown model id");
    filter::PfConfig cfg = to_pf(*c, n, *model);
    for (std::size_t k = 0; k < model->param_dim(); ++k)
      cfg.theta_prior[k] = {th_mu[k], th_sigma[k]};
    for (std::size_t k = 0; k < model->dim(); ++k)
      cfg.x0_prior[k] = {x_mean[k], x_std[k], x_clamp[k] != 0};
    const filter::Ensemble ens = filter::initialize(cfg, *model);
    store(ens, *e);
  });
}

int ref_propagate_interval(int model_id, const double* theta_nat,
                           const double* x0, double t0, double t1, double h,
                           int family, int order, double tol, int max_iter,
                           double* state_out, double* gamma_out,
                           int* status_out, int* iters_out) {
  return guarded([&] {
    auto model = pfsmc_oracle_ref::make_model(model_id);
    if (!model) throw ConfigError("unknown model id");
    const std::size_t d = model->dim(), p = model->param_dim();
    const auto r = lmm::propagate_interval(
        *model, {theta_nat, p}, {x0, d}, t0, t1, h,
        lmm::scheme_coefficients(family_of(family), order), {tol, max_iter});
    for (std::size_t k = 0; k < d; ++k) {
      state_out[k] = r.state[k];
      gamma_out[k] = r.gamma_diag[k];
    }
    *status_out = static_cast<int>(r.status);
    *iters_out = r.total_newton_iterations;
  });
}

int ref_fitness_weights(const double* logw, const double* loglik, uint64_t n,
                        double* g) {
  return guarded([&] {
    const auto r = filter::fitness_weights({logw, n}, {loglik, n});
    std::memcpy(g, r.data(), sizeof(double) * n);
  });
}

int ref_resample_multinomial(const double* g, uint64_t n, uint64_t seed,
                             uint64_t j, int64_t* out) {
  return guarded([&] {
    const auto r = filter::resample_multinomial({g, n}, seed, j);
    for (std::size_t i = 0; i < n; ++i) out[i] = static_cast<int64_t>(r[i]);
  });
}

int ref_weighted_mean_cov(const double* params, uint64_t n, uint64_t p,
                          const double* w, double* mean, double* cov) {
  return guarded([&] {
    linalg::DenseMatrix C;
    linalg::weighted_mean_cov({params, n * p}, n, p, {w, n}, {mean, p}, C);
    std::memcpy(cov, C.values.data(), sizeof(double) * p * p);
  });
}

int ref_chol_psd(const double* cov, uint64_t p, double* lower, double* jitter) {
  return guarded([&] {
    linalg::DenseMatrix C(p, p);
    C.values.assign(cov, cov + p * p);
    const auto r = linalg::chol_psd(C);
    std::memcpy(lower, r.lower.values.data(), sizeof(double) * p * p);
    *jitter = r.jitter;
  });
}

double ref_log_likelihood(const double* y, const double* x, uint64_t d,
                          const uint64_t* idx, uint64_t m, double sigma) {
  filter::ObservationModel o;
  for (uint64_t k = 0; k < m; ++k) o.indices.push_back(idx[k]);
  o.sigma = sigma;
  std::vector<double> xv(x, x + d);
  return filter::log_likelihood({y, m}, xv, o);
}

// Times `steps` consecutive pf_step calls (observations y[j-1], times
// t0 + j*dt) on the injected ensemble with the configured backend, exactly
// as bench::run_experiment times filter::run (bench.cpp:565-571): the
// steady_clock window covers the step loop only.
int ref_time_steps(const ref_cfg* c, ref_ens* e, const double* y,
                   const double* t_obs, uint64_t j0, uint64_t steps,
                   double t_prev0, double* seconds) {
  return guarded([&] {
    auto model = pfsmc_oracle_ref::make_model(c->model);
    if (!model) throw ConfigError("unknown model id");
    filter::PfConfig cfg = to_pf(*c, e->n, *model);
    filter::ObservationModel obs = to_obs(*c);
    exec::Backend backend = backend_of(c->workers);
    backend.start();
    filter::Ensemble ens = load(*e);
    double t_prev = t_prev0;
    const auto t0 = std::chrono::steady_clock::now();
    for (uint64_t s = 0; s < steps; ++s) {
      filter::pf_step(ens, {y + s * c->m_y, c->m_y}, j0 + s, t_prev, t_obs[s],
                      cfg, backend, *model, obs);
      t_prev = t_obs[s];
    }
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() -
                                             t0)
                   .count();
    store(ens, *e);
  });
}

}  // extern "C"
