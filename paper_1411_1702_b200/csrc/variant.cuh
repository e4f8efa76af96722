// Arithmetic variants of the device code. Every device header wraps its code
// in an inline namespace named after the variant, so one library can hold the
// same kernels built twice with different floating-point rules:
//   exact (default): the reference's operation order, no FMA contraction
//           (--fmad=false; CMakeLists.txt:7-9), divisions where the reference
//           divides — Psi bitwise equal to the CPU reference;
//   fast  (-DPFSMC_FAST=1 --fmad=true): FMA contraction and reciprocal
//           multiplies for shared denominators; within the north_star
//           tolerances (states 1e-10, trace 1e-8, ancestors exact up to
//           classified near-ties), not bitwise.
// The host-visible types (Ctx, DevState, KernelSet, ...) live outside the
// variant namespace (types.cuh), so the host driver dispatches to either set.
#pragma once
#ifndef PFSMC_FAST
#define PFSMC_FAST 0
#endif
#if PFSMC_FAST
#define PFSMC_VNS fast
#else
#define PFSMC_VNS exact
#endif
#define PFSMC_BEGIN \
  namespace pfsmc_gpu { \
  inline namespace PFSMC_VNS {
#define PFSMC_END \
  } \
  }
