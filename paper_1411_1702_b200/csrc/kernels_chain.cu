// Kernel instantiations for ChainModel: every (family, order) of the reference's
// fixed-step integrator set (lmm.cpp:64-77: AB/AM/BDF x orders 1-3).
// Built twice: exact (reference operation order) and fast (-DPFSMC_FAST=1
// --fmad=true), see variant.cuh.
#include "kernels.cuh"

namespace pfsmc_gpu {
std::unique_ptr<KernelSet> PFSMC_ENTRY(chain)(int fam, int order) {
  return make_family<ChainModel>(fam, order);
}
}  // namespace pfsmc_gpu
