// AdvDiffModel kernel sets with E = 1 state element(s) per thread (d <= 1 x 128).
#include "advdiff_set.cuh"

namespace pfsmc_gpu {
// n = 10 (m = 9): the grid of the reference's acceptance run (acceptance_main.cpp:466-480)
// with a compile-time grid side
std::unique_ptr<KernelSet> adv_family_e1(int fam, int order, int n) {
  return n == 10 ? adv_family<1, 9>(fam, order, n) : adv_family<1>(fam, order, n);
}
}  // namespace pfsmc_gpu
