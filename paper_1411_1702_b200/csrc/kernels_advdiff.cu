// Kernel set for the reference's AdvDiffModel (models.cpp:158-266): the
// particle-per-CTA propagation kernels of advdiff.cuh plus the
// particle-per-thread passes around them (fitness log-sum-exp over lg, the
// theta moments, the state mean of the trace row, initialisation).
#include <cmath>
#include <stdexcept>
#include <vector>

#include "advdiff.cuh"

namespace pfsmc_gpu {

std::vector<double2> adv_dft_matrix(int m) {
  const std::vector<double2> tw = adv_twiddles(m);
  std::vector<double2> W(static_cast<size_t>(m) * m);
  for (int k = 0; k < m; ++k)
    for (int j = 0; j < m; ++j) {
      const double2 t = tw[(k * j) % m];
      W[static_cast<size_t>(k) * m + j] = make_double2(t.x, -t.y);
    }
  return W;
}

std::vector<double2> adv_twiddles(int m) {
  std::vector<double2> tw(m);
  const double two_pi = 6.283185307179586476925286766559;
  for (int k = 0; k < m; ++k) {
    // exact at the symmetric points; libm cos / sin elsewhere
    const double a = two_pi * static_cast<double>(k) / static_cast<double>(m);
    tw[k] = make_double2(std::cos(a), std::sin(a));
    if (4 * k == m) tw[k] = make_double2(0.0, 1.0);
    if (2 * k == m) tw[k] = make_double2(-1.0, 0.0);
    if (4 * k == 3 * m) tw[k] = make_double2(0.0, -1.0);
  }
  return tw;
}

// The tail of k_predict over a stored lg (filter.cpp:143-156 + the exact-CDF
// tile partials): per-block (max, sum exp) partials, finite counts, the
// last-block tree -> lse_g, tile prefixes.
__global__ void __launch_bounds__(kThreads) k_lg_reduce(Ctx c) {
  __shared__ double scratch[kWarps * 2];
  __shared__ double fin[2];
  if (grid_error(c)) return;
  const long long n = static_cast<long long>(blockIdx.x) * kThreads + threadIdx.x;
  const double lgv = n < c.N ? c.lg[n] : kNegInf;
  const double one[1] = {1.0};
  const int nfin = __syncthreads_count(isfinite(lgv) != 0);
  if (threadIdx.x == 0) c.blk_cnt[blockIdx.x] = nfin;
  block_partial<1, false>(lgv, one, c.part + blockIdx.x * 2, scratch);
  if (tree_reduce_last<1, false>(c.part, c.gpart, c.cnt_pred, fin, scratch, !c.sharded,
                                 TileGroupHook{&c})) {
    __shared__ double s_lse;
    if (threadIdx.x == 0) {
      const double mx = fin[0];
      const double lse = isfinite(mx) ? mx + log(fin[1]) : kNegInf;
      c.st->lse_g = lse;
      if (!isfinite(lse)) atomicOr(&c.st->error, kErrPredict);
      s_lse = lse;
    }
    __syncthreads();
    if (isfinite(s_lse)) tile_prefixes(c, s_lse);
  }
}

// The theta moments read through the fixed-size machinery: a view with
// P = 5 and one (unused) state component; the trace's state mean comes from
// k_adv_xmean.

// mode 0: injected ensemble (shrink mean + chol of the given cov);
// mode 1: initialisation (mean and cov);
// mode 2: a completed step over the new record buffer (lse_w, mean, cov,
//         chol, flip) — the epilogue of k_update.
template <int MODE>
__global__ void __launch_bounds__(kThreads) k_adv_moments(Ctx c) {
  using ML = MomentLayout<AdvThetaView>;
  constexpr int P = kAdvP, V = ML::V;
  __shared__ double scratch[kWarps * V];
  __shared__ double fin[V + 1];
  if (MODE == 2 && grid_error(c)) return;
  DevState& st = *c.st;
  if (MODE == 2 && st.chol_failed) return;
  const int cur = st.cur;
  const double* recs = c.rec[MODE == 2 ? cur ^ 1 : cur];
  const long long n = static_cast<long long>(blockIdx.x) * kThreads + threadIdx.x;
  double K[P];
#pragma unroll
  for (int k = 0; k < P; ++k) K[k] = st.mu[k];
  double lwv = kNegInf;
  double vals[V];
#pragma unroll
  for (int k = 0; k < V; ++k) vals[k] = 0.0;
  if (n < c.N) {
    const double* r = recs + n * c.R;
    lwv = MODE == 2 ? c.lw[n] : c.lw[n] - st.lse_w;
    double dv[P];
#pragma unroll
    for (int k = 0; k < P; ++k) dv[k] = r[c.adv_d + k] - K[k];
    vals[0] = 1.0;
#pragma unroll
    for (int k = 0; k < P; ++k) vals[1 + k] = dv[k];
    int idx = 0;
#pragma unroll
    for (int a = 0; a < P; ++a)
#pragma unroll
      for (int b = a; b < P; ++b) vals[1 + ML::NA + idx++] = dv[a] * dv[b];
    vals[1 + ML::NA + ML::NB] = r[0];
    vals[V - 1] = 1.0;
  }
  block_partial<V, true>(lwv, vals, c.part + static_cast<size_t>(blockIdx.x) * (V + 1), scratch);
  if (tree_reduce_last<V, true>(c.part, c.gpart, c.cnt_upd, fin, scratch, true)) {
    if (threadIdx.x == 0) {
      finalize_moments<AdvThetaView>(c, fin, K, MODE == 2, MODE != 0);
      if (!(st.error & kErrUpdate)) {
        chol_psd_device<P>(st);
        if (MODE == 2) st.cur = cur ^ 1;
      }
    }
  }
}

// State mean of the trace row (filter.cpp:383-389: sum_i w_i x_i with
// w = exp(logw)), after the moments (lse_w final): per chunk of particles a
// partial per component, then a fixed-order sum of the chunk partials.
constexpr int kXmChunks = 64;
__global__ void __launch_bounds__(kThreads) k_adv_xmean_part(Ctx c) {
  if (grid_error(c)) return;
  const int k = blockIdx.x * kThreads + threadIdx.x;
  const long long per = (c.N + kXmChunks - 1) / kXmChunks;
  const long long n0 = blockIdx.y * per, n1 = min(n0 + per, static_cast<long long>(c.N));
  if (k >= c.adv_d) return;
  const double lse = c.st->lse_w;
  const double* recs = c.rec[c.st->cur];
  double s = 0.0;
  for (long long n = n0; n < n1; ++n) s += exp(c.lw[n] - lse) * recs[n * c.R + k];
  c.xmean_part[static_cast<size_t>(blockIdx.y) * c.adv_d + k] = s;
}
__global__ void __launch_bounds__(kThreads) k_adv_xmean_sum(Ctx c) {
  if (grid_error(c)) return;
  const int k = blockIdx.x * kThreads + threadIdx.x;
  if (k >= c.adv_d) return;
  double s = 0.0;
  for (int q = 0; q < kXmChunks; ++q) s += c.xmean_part[static_cast<size_t>(q) * c.adv_d + k];
  c.xmean[k] = s;
}

// filter::initialize (filter.cpp:76-105) / the uniform box prior: stream
// (seed, 0, i, init), theta then x; one CTA per particle, draw k computed
// directly from its Philox block.
__global__ void __launch_bounds__(kAT) k_adv_init(Ctx c, int kind, const double* prm, double lw0) {
  constexpr int P = kAdvP;
  const long long n = blockIdx.x;
  const int d = c.adv_d;
  double* r = c.rec[c.st->cur] + n * c.R;
  const uint64_t nn = c.n0 + n;
  for (int k = threadIdx.x; k < P + d; k += kAT) {
    double v;
    if (kind == 0) {
      // prm: th_mu[P], th_sigma[P], x_mean[d], x_std[d], x_clamp[d]
      const double z = normal_at(c.seed, 0, nn, kInit, k);
      if (k < P) {
        v = prm[k] + prm[P + k] * z;
      } else {
        const int e = k - P;
        v = prm[2 * P + e] + prm[2 * P + d + e] * z;
        if (prm[2 * P + 2 * d + e] != 0.0 && v < 0.0) v = 0.0;
      }
    } else {
      // prm: th_lo[P], th_hi[P], x_lo[d], x_hi[d]
      const double u = uniform_at(c.seed, 0, nn, kInit, k);
      if (k < P) {
        v = log(prm[k] + (prm[P + k] - prm[k]) * u);
      } else {
        const int e = k - P;
        v = prm[2 * P + e] + (prm[2 * P + d + e] - prm[2 * P + e]) * u;
      }
    }
    r[k < P ? d + k : k - P] = v;
  }
  if (threadIdx.x == 0) {
    for (int k = d + P; k < c.R; ++k) r[k] = 0.0;
    c.lw[n] = lw0;
  }
}

void adv_launch_lg_reduce(const Ctx& c, int grid, cudaStream_t s) { k_lg_reduce<<<grid, kThreads, 0, s>>>(c); }
void adv_launch_moments(const Ctx& c, int grid, cudaStream_t s, int mode) {
  if (mode == 2)
    k_adv_moments<2><<<grid, kThreads, 0, s>>>(c);
  else if (mode == 1)
    k_adv_moments<1><<<grid, kThreads, 0, s>>>(c);
  else
    k_adv_moments<0><<<grid, kThreads, 0, s>>>(c);
}
void adv_launch_xmean(const Ctx& c, int d, cudaStream_t s) {
  const dim3 g((d + kThreads - 1) / kThreads, kXmChunks);
  k_adv_xmean_part<<<g, kThreads, 0, s>>>(c);
  k_adv_xmean_sum<<<(d + kThreads - 1) / kThreads, kThreads, 0, s>>>(c);
}
void adv_launch_init(const Ctx& c, cudaStream_t s, int kind, const double* prm, double lw0) {
  k_adv_init<<<c.N, kAT, 0, s>>>(c, kind, prm, lw0);
}

std::unique_ptr<KernelSet> adv_family_e1(int fam, int order, int n);
std::unique_ptr<KernelSet> adv_family_e3(int fam, int order, int n);
std::unique_ptr<KernelSet> adv_family_e8(int fam, int order, int n);

std::unique_ptr<KernelSet> make_kernels_advdiff(int fam, int order, int grid_n) {
  if (grid_n < 4 || grid_n > kAdvMaxM + 1) return nullptr;
  const int d = (grid_n - 1) * (grid_n - 1);
  if (d <= kAT) return adv_family_e1(fam, order, grid_n);
  if (d <= 3 * kAT) return adv_family_e3(fam, order, grid_n);
  return adv_family_e8(fam, order, grid_n);
}

}  // namespace pfsmc_gpu
