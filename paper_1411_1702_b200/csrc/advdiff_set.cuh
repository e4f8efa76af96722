// The AdvDiffModel kernel set (KernelSet over the particle-CTA kernels of
// advdiff.cuh); instantiated per register width E in kernels_advdiff_e*.cu.
#pragma once
#include <stdexcept>
#include <vector>

#include "advdiff.cuh"

namespace pfsmc_gpu {

template <int FAM, int ORD, int E, int MT = 0>
struct AdvKernelSet final : KernelSet {
  int m;
  size_t smem;
  explicit AdvKernelSet(int grid_n) {
    m = grid_n - 1;
    d = m * m;
    p = kAdvP;
    smem = adv_smem_bytes(m);
    cudaFuncSetAttribute(k_adv_predict<FAM, ORD, E, MT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    cudaFuncSetAttribute(k_adv_update<FAM, ORD, E, MT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    cudaFuncSetAttribute(k_adv_trajectory<E>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
  }
  bool block_model() const override { return true; }
  void xmean(const Ctx& c, cudaStream_t s) { adv_launch_xmean(c, d, s); }
  void trajectory(const double* prm, const double* times, int T, double t0, double rtol, double tol,
                  int max_iter, double* out, int* status, cudaStream_t s) override {
    // prm layout of the register models: consts[8], theta[P], x0[d]
    std::vector<double2> tw = adv_twiddles(m);
    std::vector<double2> W = adv_dft_matrix(m);
    double2* dtw = nullptr;
    if (cudaMalloc(&dtw, sizeof(double2) * (m + d)) != cudaSuccess) throw std::runtime_error("advdiff: cudaMalloc");
    cudaMemcpyAsync(dtw, tw.data(), sizeof(double2) * m, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(dtw + m, W.data(), sizeof(double2) * d, cudaMemcpyHostToDevice, s);
    Ctx c{};
    c.adv_m = m;
    c.adv_d = d;
    c.adv_tw = dtw;
    c.adv_W = dtw + m;
    c.tol = tol;
    c.max_iter = max_iter;
    k_adv_trajectory<E><<<1, kAT, smem, s>>>(c, prm + 8, times, T, t0, rtol, out, status);
    cudaStreamSynchronize(s);
    cudaFree(dtw);
  }
  void predict(const Ctx& c, int grid, cudaStream_t s) override {
    k_adv_predict<FAM, ORD, E, MT><<<c.N, kAT, smem, s>>>(c);
    adv_launch_lg_reduce(c, grid, s);
  }
  void update(const Ctx& c, int grid, cudaStream_t s) override {
    k_adv_update<FAM, ORD, E, MT><<<c.N, kAT, smem, s>>>(c);
    adv_launch_moments(c, grid, s, 2);
    xmean(c, s);
  }
  void moments(const Ctx& c, int grid, cudaStream_t s, int set_cov) override {
    adv_launch_moments(c, grid, s, set_cov ? 1 : 0);
    xmean(c, s);
  }
  void chol(const Ctx& c, cudaStream_t s) override { k_chol<kAdvP><<<1, 32, 0, s>>>(c.st); }
  void init(const Ctx& c, int grid, cudaStream_t s, int kind, const double* prm, double lw0) override {
    (void)grid;
    adv_launch_init(c, s, kind, prm, lw0);
  }
  void finish_moments(const Ctx&, const double*, int, int, cudaStream_t) override {
    throw std::runtime_error("advdiff: sharded moments are not supported");
  }
  int moment_width() const override { return MomentLayout<AdvThetaView>::V + 1; }
};

template <int FAM, int E, int MT>
std::unique_ptr<KernelSet> adv_order(int order, int n) {
  if constexpr (FAM == kBDF)
    if (order == 0) return std::make_unique<AdvKernelSet<FAM, 0, E, MT>>(n);
  switch (order) {
    case 1: return std::make_unique<AdvKernelSet<FAM, 1, E, MT>>(n);
    case 2: return std::make_unique<AdvKernelSet<FAM, 2, E, MT>>(n);
    case 3: return std::make_unique<AdvKernelSet<FAM, 3, E, MT>>(n);
  }
  return nullptr;
}
template <int E, int MT = 0>
std::unique_ptr<KernelSet> adv_family(int fam, int order, int n) {
  switch (fam) {
    case kAB: return adv_order<kAB, E, MT>(order, n);
    case kAM: return adv_order<kAM, E, MT>(order, n);
    case kBDF: return adv_order<kBDF, E, MT>(order, n);
  }
  return nullptr;
}

}  // namespace pfsmc_gpu
