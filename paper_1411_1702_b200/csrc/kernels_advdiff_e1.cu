// AdvDiffModel kernel sets with E = 1 state element(s) per thread (d <= 1 x 128).
#include "advdiff_set.cuh"

namespace pfsmc_gpu {
std::unique_ptr<KernelSet> adv_family_e1(int fam, int order, int n) { return adv_family<1>(fam, order, n); }
}  // namespace pfsmc_gpu
