// Drop-in usage of the C++ mirror (include/pfsmc_gpu.hpp): a caller of
// pfsmc::filter::pf_step swaps the call site for pfsmc_gpu::pf_step /
// Sampler::step. Runs Lotka-Volterra from a uniform box prior for a few
// observations and prints the trace rows (a GPU test checks the output
// against the host oracle).
//   usage: drop_in_lv N T seed  < observations (T lines "y1 y2")
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "pfsmc_gpu.hpp"

int main(int argc, char** argv) {
  const std::size_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 4096;
  const int T = argc > 2 ? std::atoi(argv[2]) : 5;
  const std::uint64_t seed = argc > 3 ? std::strtoull(argv[3], nullptr, 10) : 1;
  pfsmc_gpu::PfConfig cfg;
  cfg.model = PFSMC_GPU_MODEL_LOTKA_VOLTERRA;
  cfg.particles = n;
  cfg.shrink_a = 0.98;
  cfg.h = 0.1;
  cfg.family = PFSMC_GPU_AM;
  cfg.order = 2;
  cfg.seed = seed;
  pfsmc_gpu::ObservationModel obs{{0, 1}, 0.05, PFSMC_GPU_LIK_GAUSSIAN};
  try {
    pfsmc_gpu::Sampler dev(cfg, obs);
    const double lo[2] = {0.5, 0.5}, hi[2] = {1.5, 1.5};
    pfsmc_gpu::check(pfsmc_gpu_init_uniform(dev.handle(), lo, hi, lo, hi));
    pfsmc_gpu::Ensemble ens{n, 2, 2, std::vector<double>(2 * n), std::vector<double>(2 * n),
                            std::vector<double>(n), std::vector<double>(2), std::vector<double>(4)};
    dev.get_ensemble(ens);
    double t_prev = 0.0;
    for (int j = 1; j <= T; ++j) {
      double y[2];
      if (std::scanf("%lf %lf", &y[0], &y[1]) != 2) return 4;
      const double t_obs = 0.1 * j;
      // the reference call site: pf_step(ens, y, j, t_prev, t_obs, cfg, backend, model, obs)
      const pfsmc_gpu::TraceRow r = pfsmc_gpu::pf_step(ens, y, j, t_prev, t_obs, dev);
      std::printf("%d %.17g %.17g %.17g %.17g %.17g %.17g %.17g\n", j, r.theta_mean[0], r.theta_mean[1],
                  r.theta_var[0], r.theta_var[1], r.state_mean[0], r.state_mean[1], r.ess);
      t_prev = t_obs;
    }
  } catch (const pfsmc_gpu::NumericalError& e) {
    std::fprintf(stderr, "numerical: %s\n", e.what());
    return 3;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}
