// Reference-side OdeModel plugins for the BASELINE.json problems.
//
// TEST INFRASTRUCTURE (oracle side). These classes implement the reference's
// own plugin interface (/root/reference/proj/include/pfsmc/models.hpp:20-55:
// ModelEval::rhs/jacobian, OdeModel::dim/params/bind) so the UNMODIFIED
// reference sampler (filter.cpp:292-394) can run the three BASELINE models,
// none of which ship with the reference.
//
// The arithmetic of every right-hand side and Jacobian is written in a fixed
// evaluation order that the C restatement (oracle/pfsmc_oracle.c) and the
// device functors (paper_1411_1702_b200/csrc/models.cuh) repeat term for
// term, so propagation is bitwise comparable when built without FMA
// contraction (the reference's own build has none: CMakeLists.txt:7-9).
#pragma once

#include <cmath>
#include <memory>
#include <span>
#include <vector>

#include "pfsmc/models.hpp"

namespace pfsmc_oracle_ref {

using pfsmc::linalg::DenseMatrix;
using pfsmc::models::ModelEval;
using pfsmc::models::OdeModel;
using pfsmc::models::ParamSpec;

inline bool all_finite(std::span<const double> v) {
  for (double x : v)
    if (!std::isfinite(x)) return false;
  return true;
}

// x' = -theta x (test_filter.cpp:23-52 ScalarDecayModel, used by the
// scripted 3-particle oracle at test_filter.cpp:363-453).
class DecayModel : public OdeModel {
 public:
  std::size_t dim() const override { return 1; }
  const std::vector<ParamSpec>& params() const override {
    static const std::vector<ParamSpec> s = {{"theta", true}};
    return s;
  }
  std::unique_ptr<ModelEval> bind(std::span<const double> th) const override {
    struct E : ModelEval {
      double t0;
      explicit E(double v) : t0(v) {}
      bool rhs(double, std::span<const double> x,
               std::span<double> o) const override {
        o[0] = -t0 * x[0];
        return true;
      }
      bool jacobian(double, std::span<const double>,
                    DenseMatrix& J) const override {
        J = DenseMatrix(1, 1);
        J.at(0, 0) = -t0;
        return true;
      }
    };
    return std::make_unique<E>(th[0]);
  }
};

// Lotka-Volterra (BASELINE configs 1-2):
//   x0' = th0 x0 - x0 x1,  x1' = x0 x1 - th1 x1.
class LotkaVolterraModel : public OdeModel {
 public:
  std::size_t dim() const override { return 2; }
  const std::vector<ParamSpec>& params() const override {
    static const std::vector<ParamSpec> s = {{"theta1", true},
                                             {"theta2", true}};
    return s;
  }
  std::unique_ptr<ModelEval> bind(std::span<const double> th) const override {
    struct E : ModelEval {
      double a, b;
      E(double x, double y) : a(x), b(y) {}
      bool rhs(double, std::span<const double> x,
               std::span<double> o) const override {
        o[0] = a * x[0] - x[0] * x[1];
        o[1] = x[0] * x[1] - b * x[1];
        return all_finite(o);
      }
      bool jacobian(double, std::span<const double> x,
                    DenseMatrix& J) const override {
        J = DenseMatrix(2, 2);
        J.at(0, 0) = a - x[1];
        J.at(0, 1) = -x[0];
        J.at(1, 0) = x[1];
        J.at(1, 1) = x[0] - b;
        return all_finite(J.values);
      }
    };
    return std::make_unique<E>(th[0], th[1]);
  }
};

// Robertson kinetics (BASELINE config 3), theta = (k1, k2, k3):
//   x0' = -k1 x0 + k3 x1 x2, x1' = k1 x0 - k2 x1^2 - k3 x1 x2, x2' = k2 x1^2.
class RobertsonModel : public OdeModel {
 public:
  std::size_t dim() const override { return 3; }
  const std::vector<ParamSpec>& params() const override {
    static const std::vector<ParamSpec> s = {
        {"k1", true}, {"k2", true}, {"k3", true}};
    return s;
  }
  std::unique_ptr<ModelEval> bind(std::span<const double> th) const override {
    struct E : ModelEval {
      double k1, k2, k3;
      E(double a, double b, double c) : k1(a), k2(b), k3(c) {}
      bool rhs(double, std::span<const double> x,
               std::span<double> o) const override {
        const double ra = k1 * x[0];
        const double rb = k2 * x[1] * x[1];
        const double rc = k3 * x[1] * x[2];
        o[0] = rc - ra;
        o[1] = ra - rb - rc;
        o[2] = rb;
        return all_finite(o);
      }
      bool jacobian(double, std::span<const double> x,
                    DenseMatrix& J) const override {
        J = DenseMatrix(3, 3);
        J.at(0, 0) = -k1;
        J.at(0, 1) = k3 * x[2];
        J.at(0, 2) = k3 * x[1];
        J.at(1, 0) = k1;
        J.at(1, 1) = -(2.0 * k2 * x[1]) - k3 * x[2];
        J.at(1, 2) = -(k3 * x[1]);
        J.at(2, 0) = 0.0;
        J.at(2, 1) = 2.0 * k2 * x[1];
        J.at(2, 2) = 0.0;
        return all_finite(J.values);
      }
    };
    return std::make_unique<E>(th[0], th[1], th[2]);
  }
};

// 8-compartment saturating reaction chain (BASELINE config 4), u = 1:
//   flux_i = th0 x_i / (1 + x_i)
//   x0' = u - flux_0
//   x_i' = flux_{i-1} - th1 x_i - th2 x_i^2     (i = 1..6)
//   x7' = th1 x6 - th3 x7
// Undefined (particle invalid) when a denominator 1 + x_i <= 0, mirroring
// the reference metabolic model's convention (models.cpp:44-58).
class ChainModel : public OdeModel {
 public:
  std::size_t dim() const override { return 8; }
  const std::vector<ParamSpec>& params() const override {
    static const std::vector<ParamSpec> s = {
        {"theta1", true}, {"theta2", true}, {"theta3", true}, {"theta4", true}};
    return s;
  }
  std::unique_ptr<ModelEval> bind(std::span<const double> th) const override {
    struct E : ModelEval {
      double t0, t1, t2, t3;
      E(double a, double b, double c, double d) : t0(a), t1(b), t2(c), t3(d) {}
      bool rhs(double, std::span<const double> x,
               std::span<double> o) const override {
        double flux[7];
        for (int i = 0; i < 7; ++i) {
          const double den = 1.0 + x[i];
          if (den <= 0.0) return false;
          flux[i] = t0 * x[i] / den;
        }
        o[0] = 1.0 - flux[0];
        for (int i = 1; i < 7; ++i) {
          o[i] = flux[i - 1] - t1 * x[i] - t2 * x[i] * x[i];
        }
        o[7] = t1 * x[6] - t3 * x[7];
        return all_finite(o);
      }
      bool jacobian(double, std::span<const double> x,
                    DenseMatrix& J) const override {
        J = DenseMatrix(8, 8);
        double dflux[7];
        for (int i = 0; i < 7; ++i) {
          const double den = 1.0 + x[i];
          if (den <= 0.0) return false;
          dflux[i] = t0 / (den * den);
        }
        J.at(0, 0) = -dflux[0];
        for (int i = 1; i < 7; ++i) {
          J.at(i, i - 1) = dflux[i - 1];
          J.at(i, i) = -t1 - 2.0 * t2 * x[i];
        }
        J.at(7, 6) = t1;
        J.at(7, 7) = -t3;
        return all_finite(J.values);
      }
    };
    return std::make_unique<E>(th[0], th[1], th[2], th[3]);
  }
};

enum ModelId { kDecay = 0, kLotkaVolterra = 1, kRobertson = 2, kChain = 3, kMetabolic = 5, kAdvDiff = 6 };

// Constants for the reference's own MetabolicModel (models.hpp:67-74), set
// through the harness (ref_set_model_consts): lambda, c0, A0, A, t0_input, tau.
inline double g_model_consts[8] = {1.0, 1.0, 1.0, 5.0, 2.0, 1.0, 0.0, 0.0};

inline std::unique_ptr<OdeModel> make_model(int id) {
  switch (id) {
    case kMetabolic: {  // the reference's own plugin, unmodified (models.cpp:37-119)
      pfsmc::models::MetabolicConstants k;
      k.lambda = g_model_consts[0];
      k.c0 = g_model_consts[1];
      k.A0 = g_model_consts[2];
      k.A = g_model_consts[3];
      k.t0_input = g_model_consts[4];
      k.tau = g_model_consts[5];
      return std::make_unique<pfsmc::models::MetabolicModel>(k);
    }
    case kAdvDiff:  // the reference's problem 2, unmodified (models.cpp:185-266); n = grid parameter
      return std::make_unique<pfsmc::models::AdvDiffModel>(static_cast<std::size_t>(g_model_consts[0]));
    case kDecay:
      return std::make_unique<DecayModel>();
    case kLotkaVolterra:
      return std::make_unique<LotkaVolterraModel>();
    case kRobertson:
      return std::make_unique<RobertsonModel>();
    case kChain:
      return std::make_unique<ChainModel>();
    default:
      return nullptr;
  }
}

}  // namespace pfsmc_oracle_ref
