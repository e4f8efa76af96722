// C++ host mirror of the reference sampler API over the pfsmc_gpu C ABI.
//
// The reference (C++20) exposes, in namespace pfsmc::filter
// (/root/reference/proj/include/pfsmc/filter.hpp:19-160):
//   struct Ensemble { n, d, p, states, params_u, logw, mean_u, cov_u };
//   StepResult pf_step(Ensemble&, std::span<const double> y, std::size_t j,
//                      double t_prev, double t_obs, const PfConfig&,
//                      exec::Backend&, const models::OdeModel&,
//                      const ObservationModel&, PhaseTimings*);
// This header gives the same names and argument meaning with the ensemble
// resident on a B200: pfsmc_gpu::pf_step(ens, y, j, t_prev, t_obs, cfg, obs)
// is the call-site replacement (the Backend and the OdeModel are replaced by
// the device and the compiled-in model id). Errors are thrown as the
// reference throws them (ConfigError / NumericalError, errors.hpp:9-25).
//
// Header-only; link against paper_1411_1702_b200/libpfsmc_gpu.so.
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "pfsmc_gpu.h"

namespace pfsmc_gpu {

struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NumericalError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(pfsmc_gpu_status st) {
  if (st == PFSMC_GPU_OK) return;
  const std::string msg = pfsmc_gpu_last_error();
  if (st == PFSMC_GPU_ERR_CONFIG) throw ConfigError(msg);
  if (st == PFSMC_GPU_ERR_NUMERICAL) throw NumericalError(msg);
  throw std::runtime_error(msg);
}

// filter::Ensemble (filter.hpp:19-28): row-major AoS, log-space params.
struct Ensemble {
  std::size_t n = 0, d = 0, p = 0;
  std::vector<double> states, params_u, logw, mean_u, cov_u;
};

// filter::ObservationModel (filter.hpp:30-33) + the likelihood kind.
struct ObservationModel {
  std::vector<std::uint64_t> indices;
  double sigma = 0.0;
  int likelihood = PFSMC_GPU_LIK_GAUSSIAN;
};

// The PfConfig fields pf_step reads (filter.hpp:50-65) + the model id that
// stands in for the OdeModel plugin.
struct PfConfig {
  int model = PFSMC_GPU_MODEL_LOTKA_VOLTERRA;
  std::size_t particles = 1000;
  double shrink_a = 0.98;
  double h = 0.05;
  int family = PFSMC_GPU_BDF;
  int order = 2;
  std::uint64_t seed = 0;
  double newton_tol = 1e-9;
  int newton_max_iter = 20;
  int device = 0;
  // the bound model's constants; METABOLIC: models::MetabolicConstants
  // (lambda, c0, A0, A, t0_input, tau), reference defaults (models.hpp:67-74);
  // ADVDIFF: {n}, the AdvDiffModel grid parameter (set model_consts[0])
  double model_consts[8] = {1.0, 1.0, 1.0, 5.0, 2.0, 1.0, 0.0, 0.0};
  bool adaptive = false;  // IntegratorSpec.adaptive (variable-step BDF(1,2))
  double rtol = 1e-3;     // IntegratorSpec.rtol
  bool fast_arithmetic = false;  // PFSMC_GPU_ARITH_FAST: FMA + shared reciprocals (within tolerance)
};

// filter::TraceRow (filter.hpp:67-75).
struct TraceRow {
  std::size_t j = 0;
  double t = 0.0;
  std::vector<double> theta_mean, theta_var, state_mean;
  double ess = 0.0;
  bool degeneracy_warning = false;
};

class Sampler {
 public:
  Sampler(const PfConfig& cfg, const ObservationModel& obs) : cfg_(cfg), obs_(obs) {
    pfsmc_gpu_config c{};
    c.model = cfg.model;
    c.family = cfg.family;
    c.order = cfg.order;
    c.shrink_a = cfg.shrink_a;
    c.seed = cfg.seed;
    c.newton_tol = cfg.newton_tol;
    c.newton_max_iter = cfg.newton_max_iter;
    c.particles = cfg.particles;
    c.obs_indices = obs_.indices.data();
    c.n_obs = obs_.indices.size();
    c.sigma = obs.sigma;
    c.likelihood = obs.likelihood;
    c.device = cfg.device;
    for (int k = 0; k < 8; ++k) c.model_consts[k] = cfg.model_consts[k];
    c.adaptive = cfg.adaptive ? 1 : 0;
    c.rtol = cfg.rtol;
    c.arithmetic = cfg.fast_arithmetic ? PFSMC_GPU_ARITH_FAST : PFSMC_GPU_ARITH_EXACT;
    check(pfsmc_gpu_create(&c, &h_));
  }
  ~Sampler() { pfsmc_gpu_destroy(h_); }
  Sampler(const Sampler&) = delete;
  Sampler& operator=(const Sampler&) = delete;

  void set_ensemble(const Ensemble& e) {
    check(pfsmc_gpu_set_ensemble(h_, e.states.data(), e.params_u.data(), e.logw.data(),
                                 e.mean_u.data(), e.cov_u.data()));
  }
  void get_ensemble(Ensemble& e) const {
    check(pfsmc_gpu_get_ensemble(h_, e.states.data(), e.params_u.data(), e.logw.data(),
                                 e.mean_u.data(), e.cov_u.data()));
  }
  // One step on the resident ensemble (the hot loop never copies it).
  TraceRow step(std::span<const double> y, std::size_t j, double t_prev, double t_obs,
                std::size_t d, std::size_t p) {
    std::vector<double> row(2 * p + d + 1);
    check(pfsmc_gpu_step(h_, y.data(), j, t_prev, t_obs, cfg_.h, row.data()));
    TraceRow r;
    r.j = j;
    r.t = t_obs;
    r.theta_mean.assign(row.begin(), row.begin() + p);
    r.theta_var.assign(row.begin() + p, row.begin() + 2 * p);
    r.state_mean.assign(row.begin() + 2 * p, row.begin() + 2 * p + d);
    r.ess = row[2 * p + d];
    return r;
  }
  pfsmc_gpu_sampler* handle() const { return h_; }

 private:
  PfConfig cfg_;
  ObservationModel obs_;
  pfsmc_gpu_sampler* h_ = nullptr;
};

// The literal call-site replacement for filter::pf_step: ensemble in host
// memory in, ensemble out (filter.cpp:292-394 mutates ens in place).
inline TraceRow pf_step(Ensemble& ens, std::span<const double> y, std::size_t j, double t_prev,
                        double t_obs, Sampler& dev) {
  dev.set_ensemble(ens);
  TraceRow r = dev.step(y, j, t_prev, t_obs, ens.d, ens.p);
  dev.get_ensemble(ens);
  return r;
}

}  // namespace pfsmc_gpu
