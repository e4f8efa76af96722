// AdvDiffModel kernel sets with E = 3 state element(s) per thread (d <= 3 x 128).
#include "advdiff_set.cuh"

namespace pfsmc_gpu {
// the reference's default grid (n = 20, m = 19) with a compile-time grid side
std::unique_ptr<KernelSet> adv_family_e3(int fam, int order, int n) {
  return n == 20 ? adv_family<3, 19>(fam, order, n) : adv_family<3>(fam, order, n);
}
}  // namespace pfsmc_gpu
