/* pfsmc_gpu_model.cuh — caller-defined ODE models for the GPU sampler.
 *
 * The device form of the reference plugin contract
 *   models::OdeModel::bind(theta) -> ModelEval::{rhs, jacobian}
 * (/root/reference/proj/include/pfsmc/models.hpp:20-55). A model is a struct
 *
 *   struct MyModel {
 *     static constexpr int D = ..., P = ...;   // state dim, parameter count (<= 8)
 *     static constexpr int ID = ...;           // >= PFSMC_GPU_MODEL_USER_BASE
 *     static constexpr bool kLowerBidiagonal = false;  // true: J is lower
 *                                              // bidiagonal and the model
 *                                              // provides rhs_jac_band (banded Newton)
 *     // optional, for large states: threads per CTA of the model's kernels
 *     // and the LMM history in shared memory (as the 8-species chain)
 *     //   static constexpr int kBlock = 128;
 *     //   static constexpr bool kSmemHistory = true;
 *     using K = pfsmc_gpu::NoConsts;           // or a struct of bound constants
 *     __device__ static K load_k(const double* consts);  // pfsmc_gpu_config.model_consts
 *     __device__ static bool rhs(const K&, double t, const double (&th)[P],
 *                                const double (&x)[D], double (&f)[D]);
 *     __device__ static bool jac(const K&, double t, const double (&th)[P],
 *                                const double (&x)[D], double (&J)[D][D]);
 *   };
 *
 * theta arrives in natural space (exp of the sampler's log-space params, as
 * filter::natural_params, filter.cpp:267-276). `false` from rhs / jac marks
 * the particle invalid, never an exception (ModelEval contract,
 * models.hpp:24-27). Then, in a .cu file compiled for sm_100a:
 *
 *   #include <pfsmc_gpu_model.cuh>
 *   PFSMC_GPU_REGISTER_MODEL(MyModel)
 *
 * instantiates every kernel of the per-step update (predict, update, moments,
 * init, trajectory) for every (family, order) of the fixed-step LMM set and
 * the adaptive BDF(1,2), and registers them with libpfsmc_gpu.so when the
 * plugin library is loaded; pfsmc_gpu_create then accepts model = MyModel::ID.
 * Build exact (reference operation order) with --fmad=false; the same file
 * compiled again with -DPFSMC_FAST=1 --fmad=true registers the FAST variant
 * (pfsmc_gpu_config.arithmetic = PFSMC_GPU_ARITH_FAST). The model's
 * operation order is what the sampler's Psi reproduces bit for bit in the
 * exact build. See examples/user_model/ for a complete plugin.
 */
#ifndef PFSMC_GPU_MODEL_CUH
#define PFSMC_GPU_MODEL_CUH

#include "../paper_1411_1702_b200/csrc/kernels.cuh"
#include "pfsmc_gpu.h"

#define PFSMC_GPU_MODEL_CAT_(a, b) a##b
#define PFSMC_GPU_MODEL_CAT(a, b) PFSMC_GPU_MODEL_CAT_(a, b)

#define PFSMC_GPU_REGISTER_MODEL(Model)                                                              \
  static_assert(Model::ID >= PFSMC_GPU_MODEL_USER_BASE, "plugin model ids start at PFSMC_GPU_MODEL_USER_BASE"); \
  namespace {                                                                                        \
  struct PFSMC_GPU_MODEL_CAT(pfsmc_gpu_registrar_, Model) {                                          \
    PFSMC_GPU_MODEL_CAT(pfsmc_gpu_registrar_, Model)() {                                             \
      pfsmc_gpu::KernelFactory f = &pfsmc_gpu::make_family<Model>;                                   \
      pfsmc_gpu_register_model(Model::ID, #Model, Model::D, Model::P, PFSMC_FAST,                    \
                               reinterpret_cast<void*>(f));                                          \
    }                                                                                                \
  } PFSMC_GPU_MODEL_CAT(pfsmc_gpu_registrar_instance_, Model);                                       \
  }

#endif
