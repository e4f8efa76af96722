// A caller-defined model plugin (include/pfsmc_gpu_model.cuh): two models
// registered with libpfsmc_gpu.so when this library is loaded.
//
//   UserLotkaVolterra (id 100): the Lotka-Volterra right-hand side written
//     as a plugin, term for term the built-in model's, so the sampler run
//     through the plugin path is checked against the C oracle's LV at the
//     same bars as the built-in model (tests/test_plugin_gpu.py);
//   SirModel (id 101): a model the library does not ship, the SIR epidemic
//     S' = -b S I, I' = b S I - g I, R' = g I, theta = (b, g).
//
// Built twice by paper_1411_1702_b200/build.py (exact: --fmad=false; fast:
// -DPFSMC_FAST=1 --fmad=true) into examples/user_model/libuser_models.so.
#include "pfsmc_gpu_model.cuh"

struct UserLotkaVolterra {
  static constexpr int D = 2, P = 2, ID = 100;
  static constexpr bool kLowerBidiagonal = false;
  using K = pfsmc_gpu::NoConsts;
  __device__ static K load_k(const double*) { return {}; }
  __device__ static bool rhs(const K&, double, const double (&th)[P], const double (&x)[D], double (&o)[D]) {
    o[0] = th[0] * x[0] - x[0] * x[1];
    o[1] = x[0] * x[1] - th[1] * x[1];
    return isfinite(o[0]) && isfinite(o[1]);
  }
  __device__ static bool jac(const K&, double, const double (&th)[P], const double (&x)[D], double (&J)[D][D]) {
    J[0][0] = th[0] - x[1];
    J[0][1] = -x[0];
    J[1][0] = x[1];
    J[1][1] = x[0] - th[1];
    return isfinite(J[0][0]) && isfinite(J[0][1]) && isfinite(J[1][0]) && isfinite(J[1][1]);
  }
};

struct SirModel {
  static constexpr int D = 3, P = 2, ID = 101;
  static constexpr bool kLowerBidiagonal = false;
  using K = pfsmc_gpu::NoConsts;
  __device__ static K load_k(const double*) { return {}; }
  __device__ static bool rhs(const K&, double, const double (&th)[P], const double (&x)[D], double (&o)[D]) {
    const double inf = th[0] * x[0] * x[1];
    const double rec = th[1] * x[1];
    o[0] = -inf;
    o[1] = inf - rec;
    o[2] = rec;
    return isfinite(o[0]) && isfinite(o[1]) && isfinite(o[2]);
  }
  __device__ static bool jac(const K&, double, const double (&th)[P], const double (&x)[D], double (&J)[D][D]) {
    J[0][0] = -th[0] * x[1];
    J[0][1] = -th[0] * x[0];
    J[0][2] = 0.0;
    J[1][0] = th[0] * x[1];
    J[1][1] = th[0] * x[0] - th[1];
    J[1][2] = 0.0;
    J[2][0] = 0.0;
    J[2][1] = th[1];
    J[2][2] = 0.0;
    return isfinite(J[0][0]) && isfinite(J[0][1]) && isfinite(J[1][1]);
  }
};

PFSMC_GPU_REGISTER_MODEL(UserLotkaVolterra)
PFSMC_GPU_REGISTER_MODEL(SirModel)
