// AdvDiffModel kernel sets with E = 8 state element(s) per thread (d <= 8 x 128).
#include "advdiff_set.cuh"

namespace pfsmc_gpu {
std::unique_ptr<KernelSet> adv_family_e8(int fam, int order, int n) { return adv_family<8>(fam, order, n); }
}  // namespace pfsmc_gpu
