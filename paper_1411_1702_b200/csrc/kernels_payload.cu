// Kernel set for the resample/reduction microbenchmark record (BASELINE
// config 5): only init / moments are used; one (family, order) instance.
#include "kernels.cuh"

namespace pfsmc_gpu {
std::unique_ptr<KernelSet> make_kernels_payload(int, int) {
  return std::make_unique<KernelSetT<Payload64Model, kAB, 1>>();
}
}  // namespace pfsmc_gpu
