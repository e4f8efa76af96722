// Accuracy of philox.cuh's log_unit / sincospi_unit against CUDA's log /
// sincospi over the Box-Muller input grid (u = (k + 1) 2^-53, x = 2 k 2^-53):
// max |difference| in ulps of the libm result, over 2^26 hashed inputs plus
// the domain edges. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
//   -o profiles/probe_fastmath profiles/probe_fastmath.cu
#include <cstdio>
#include <cstdint>
#include "../paper_1411_1702_b200/csrc/philox.cuh"

using namespace pfsmc_gpu;

__device__ double ulps(double a, double b) {
  if (a == b) return 0.0;
  const double u = fabs(b) > 0 ? fabs(b) * 0x1.0p-52 : 0x1.0p-1074;
  return fabs(a - b) / u;
}

__global__ void k(uint64_t n, unsigned long long* out) {
  double ml = 0, ms = 0, mc = 0, mabs = 0, mq = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const U64x4 b = philox4x64(i, 7, 3, 1, 12345, kKeyConstant);
    double u1 = (static_cast<double>(b.v[0] >> 11) + 1.0) * 0x1.0p-53;
    double u2 = static_cast<double>(b.v[1] >> 11) * 0x1.0p-53;
    if (i < 64) { u1 = (static_cast<double>(i) + 1.0) * 0x1.0p-53; u2 = static_cast<double>(i) * 0x1.0p-53; }
    if (i >= 64 && i < 128) { u1 = 1.0 - static_cast<double>(i - 64) * 0x1.0p-53; u2 = 1.0 - static_cast<double>(i - 63) * 0x1.0p-53; }
    const double l0 = log(u1), l1 = log_unit(u1);
    ml = fmax(ml, ulps(l1, l0));
    const double a = -2.0 * l0;
    mq = fmax(mq, ulps(sqrt_nonneg(a), sqrt(a)));
    double s0, c0, s1, c1;
    sincospi(2.0 * u2, &s0, &c0);
    sincospi_unit(2.0 * u2, &s1, &c1);
    ms = fmax(ms, ulps(s1, s0));
    mc = fmax(mc, ulps(c1, c0));
    mabs = fmax(mabs, fmax(fabs(s1 - s0), fabs(c1 - c0)));
  }
  atomicMax(&out[0], __double_as_longlong(ml));
  atomicMax(&out[1], __double_as_longlong(ms));
  atomicMax(&out[2], __double_as_longlong(mc));
  atomicMax(&out[3], __double_as_longlong(mabs));
  atomicMax(&out[4], __double_as_longlong(mq));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 40);
  cudaMemset(d, 0, 40);
  k<<<1184, 256>>>(1ull << 26, d);
  unsigned long long h[5];
  cudaMemcpy(h, d, 40, cudaMemcpyDeviceToHost);
  double v[5];
  for (int i = 0; i < 5; ++i) v[i] = *reinterpret_cast<double*>(&h[i]);
  printf("{\"log_unit_max_ulps\": %.3f, \"sinpi_max_ulps\": %.3f, \"cospi_max_ulps\": %.3f, \"sincos_max_abs\": %.3e, "
         "\"sqrt_nonneg_max_ulps\": %.3f}\n", v[0], v[1], v[2], v[3], v[4]);
  return 0;
}
