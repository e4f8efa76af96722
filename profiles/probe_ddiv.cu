// Bitwise check of models.cuh ddiv_seq against CUDA's a / b over 2^28 hashed
// operand pairs: mantissas uniform, exponents spread over [-60, 60] (the
// chain's flux / Jacobian / band-solve divisions live well inside), plus the
// special cases the batch guard keeps on the slow path. Prints mismatches.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o profiles/probe_ddiv profiles/probe_ddiv.cu
#include <cstdio>
#include "../paper_1411_1702_b200/csrc/philox.cuh"
#include "../paper_1411_1702_b200/csrc/models.cuh"

using namespace pfsmc_gpu;

__global__ void k(unsigned long long n, unsigned long long* bad, unsigned long long* unsafe) {
  unsigned long long nb = 0, nu = 0;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const U64x4 w = philox4x64(i, 1, 2, 3, 99, kKeyConstant);
    const double ma = 1.0 + static_cast<double>(w.v[0] >> 12) * 0x1.0p-52;
    const double mb = 1.0 + static_cast<double>(w.v[1] >> 12) * 0x1.0p-52;
    const int ea = static_cast<int>(w.v[2] % 121) - 60, eb = static_cast<int>(w.v[3] % 121) - 60;
    double a = ldexp(ma, ea) * ((w.v[2] >> 40) & 1 ? -1.0 : 1.0);
    const double b = ldexp(mb, eb) * ((w.v[3] >> 40) & 1 ? -1.0 : 1.0);
    if ((i & 1023) == 0) a = 0.0;
    if (!ddiv_safe(a, b)) { ++nu; continue; }  // (|exponent| <= 60: never, zero dividends: safe)
    const double q0 = a / b, q1 = ddiv_seq(a, b);
    nb += __double_as_longlong(q0) != __double_as_longlong(q1);
  }
  atomicAdd(bad, nb);
  atomicAdd(unsafe, nu);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  cudaMemset(d, 0, 16);
  const unsigned long long n = 1ull << 28;
  k<<<1184, 256>>>(n, d, d + 1);
  unsigned long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("{\"pairs\": %llu, \"mismatches\": %llu, \"guarded\": %llu}\n", n, h[0], h[1]);
  return 0;
}
