// fastmath.cuh — instruction-lean fp64 building blocks for the element passes.
//
// The element kernels are issue-bound, not HBM-bound, when they use the CUDA
// library division and sin: a correctly rounded fp64 division is a ~45
// instruction subroutine plus a ~16 instruction special-case path that every
// warp enters whenever one lane divides 0 (axis-aligned edges make that the
// common case on the refined meshes), and each inlined sin is ~70
// instructions.  This header replaces them with
//
//  * div_rcp(a, b, y): a / b from y = RN(1/b) by two Newton corrections of
//    the quotient (Markstein): q0 = a y, q1 = q0 + (a - b q0) y is within
//    1/2 ulp + tiny of a/b (faithful), and q2 = RN(q1 + (a - b q1) y) equals
//    RN(a / b) whenever y = RN(1/b) and nothing over/underflows (Markstein's
//    theorem, IA-64 division).  So the result is BIT-IDENTICAL to the IEEE
//    division the reference performs; callers check the safe range
//    (div_safe) once per element and fall back to '/' otherwise.  One
//    correctly rounded reciprocal (__drcp_rn) serves the 6 divisions by the
//    element's twice-area (assembly.cpp:23-25); the divisions by the constant
//    3.0 (centroid, |T|/3) use the constant RN(1/3).
//  * sin_fast(x): Cody-Waite reduction by pi/2 (3-part constant, fma) and
//    degree-17 / degree-16 Taylor polynomials on [-pi/4, pi/4]; max error
//    about 1 ulp, like CUDA's sin (2 ulp) and glibc's — the loads are compared
//    with a 1e-12 relative bound (BASELINE.json north_star), never bit-exact.
//    |x| > 2^20 or non-finite falls back to sin().
#pragma once

#include <math.h>

namespace phfem {

// exponent window in which the Markstein division is exact (no subnormal
// quotient, residual or product): |b| and nonzero |a| in [2^-480, 2^480]
__device__ __forceinline__ bool div_safe(double v) {
  const double av = fabs(v);
  return av == 0.0 || (av >= 0x1p-480 && av <= 0x1p480);
}

__device__ __forceinline__ double div_rcp(double a, double b, double y) {
  const double q0 = a * y;
  const double r0 = fma(-b, q0, a);
  const double q1 = fma(r0, y, q0);
  const double r1 = fma(-b, q1, a);
  const double q2 = fma(r1, y, q1);
  return a == 0.0 ? q0 : q2;  // a = -0: the residual path would return +0
}

// RN(1/3) and the division by the constant 3.0 (same theorem; a/3 and the
// residual stay normal for |a| in [2^-900, 2^900])
__device__ __forceinline__ double div3(double a) {
  const double y = 0x1.5555555555555p-2;  // RN(1/3)
  if (!(fabs(a) >= 0x1p-900) || !(fabs(a) <= 0x1p900)) return a / 3.0;
  return div_rcp(a, 3.0, y);
}

// Coefficients in the constant bank: DFMA takes c[bank][offset] operands
// directly, where an fp64 literal would cost two UMOVs per use (measured:
// 190 of 1,211 instructions per 32 elements in k_volume).
__constant__ double kSinPoly[8] = {2.8114572543455206e-15,  -7.647163731819816e-13,  // 1/17!, -1/15!
                                   1.6059043836821613e-10,  -2.505210838544172e-08,  // 1/13!, -1/11!
                                   2.7557319223985893e-06,  -1.984126984126984e-04,  // 1/9!,  -1/7!
                                   8.333333333333333e-03,   -1.6666666666666666e-01}; // 1/5!,  -1/3!
__constant__ double kCosPoly[8] = {4.779477332387385e-14,   -1.1470745597729725e-11, // 1/16!, -1/14!
                                   2.08767569878681e-09,    -2.755731922398589e-07,  // 1/12!, -1/10!
                                   2.48015873015873e-05,    -1.388888888888889e-03,  // 1/8!,  -1/6!
                                   4.1666666666666664e-02,  -0.5};                   // 1/4!,  -1/2!
__constant__ double kPio2[3] = {1.5707963267948966, 6.123233995736766e-17, -1.4973849048591698e-33};

// sin for |x| <= 2^20 (callers check the range, once per element)
__device__ __forceinline__ double sin_fast_core(double x) {
  const double kd = rint(x * 0.6366197723675814);  // x * 2/pi
  // pi/2 = P1 + P2 + P3 (P1 = RN(pi/2))
  double r = fma(-kd, kPio2[0], x);
  r = fma(-kd, kPio2[1], r);
  r = fma(-kd, kPio2[2], r);
  const int n = (int)kd;
  const double z = r * r;
  // sin r = r + r z (-1/3! + z/5! - ... + z^7/17!)
  double s = kSinPoly[0];
#pragma unroll
  for (int k = 1; k < 8; ++k) s = fma(s, z, kSinPoly[k]);
  s = fma(r * z, s, r);
  // cos r = 1 + z (-1/2! + z/4! - ... + z^7/16!)
  double c = kCosPoly[0];
#pragma unroll
  for (int k = 1; k < 8; ++k) c = fma(c, z, kCosPoly[k]);
  c = fma(z, c, 1.0);
  const double v = (n & 1) ? c : s;
  return (n & 2) ? -v : v;
}

__device__ __forceinline__ bool sin_fast_ok(double x) { return fabs(x) <= 1048576.0; }

__device__ __forceinline__ double sin_fast(double x) {
  if (!sin_fast_ok(x)) return sin(x);
  return sin_fast_core(x);
}

}  // namespace phfem
