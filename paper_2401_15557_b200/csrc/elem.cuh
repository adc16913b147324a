// elem.cuh — device restatements of the per-element formulas of
// include/phfem_fields.h, specialised at compile time on the coefficient and
// field kinds and built on fastmath.cuh.
//
// Bit-identical to the shared formulas for everything the reference compares
// exactly (geometry, B, D, M, M0 blocks): the divisions by the twice-area and
// by 3.0 are correctly rounded (Markstein, fastmath.cuh) and every other
// operation is the same expression in the same order.  Field samples use
// sin_fast (~1 ulp), inside the 1e-12 relative bound of the load vectors.
#pragma once

#include "common.cuh"
#include "fastmath.cuh"

namespace phfem {

constexpr int kKindGeneric = -1;
constexpr int kKindSamples = -2;  // field values sampled on the host (drop-in std::function path)

// phfem_geometry (assembly.cpp:17-27) with one reciprocal for the 6 divisions
__device__ __forceinline__ phfem_geom geometry_dev(double x0, double y0, double x1, double y1,
                                                   double x2, double y2) {
  phfem_geom g;
  g.t2 = (x1 - x0) * (y2 - y0) - (y1 - y0) * (x2 - x0);  // mesh.cpp:104-106
  g.area = 0.5 * g.t2;
  const double n0 = y1 - y2, n1 = x2 - x1, n2 = y2 - y0, n3 = x0 - x2, n4 = y0 - y1, n5 = x1 - x0;
  const bool ok = g.t2 != 0.0 && div_safe(g.t2) && div_safe(n0) && div_safe(n1) && div_safe(n2) &&
                  div_safe(n3) && div_safe(n4) && div_safe(n5);
  if (ok) {
    const double y = __drcp_rn(g.t2);
    g.gx[0] = div_rcp(n0, g.t2, y);
    g.gy[0] = div_rcp(n1, g.t2, y);
    g.gx[1] = div_rcp(n2, g.t2, y);
    g.gy[1] = div_rcp(n3, g.t2, y);
    g.gx[2] = div_rcp(n4, g.t2, y);
    g.gy[2] = div_rcp(n5, g.t2, y);
  } else {
    g.gx[0] = n0 / g.t2;
    g.gy[0] = n1 / g.t2;
    g.gx[1] = n2 / g.t2;
    g.gy[1] = n3 / g.t2;
    g.gx[2] = n4 / g.t2;
    g.gy[2] = n5 / g.t2;
  }
  return g;
}

// phfem_coeffs_eval (assembly.hpp:24-31 + the per-element BASELINE extension)
template <int CK>
__device__ __forceinline__ phfem_coeff_values coeffs_dev(const phfem_coeffs& c, double2 v0,
                                                         double2 v1, double2 v2) {
  if (CK == PHFEM_COEFF_CENTROID_POLY) {
    phfem_coeff_values v;
    const double xc = div3(v0.x + v1.x + v2.x);
    const double yc = div3(v0.y + v1.y + v2.y);
    v.a00 = 1.0 + xc * xc;
    v.a01 = 0.5 * xc * yc;
    v.a10 = v.a01;
    v.a11 = 1.0 + yc * yc;
    v.px = c.p[4];
    v.py = c.p[5];
    v.delta = 1.0 + xc + yc;
    return v;
  } else if (CK == PHFEM_COEFF_CONST) {
    phfem_coeff_values v;
    v.a00 = c.p[0];
    v.a01 = c.p[1];
    v.a10 = c.p[2];
    v.a11 = c.p[3];
    v.px = c.p[4];
    v.py = c.p[5];
    v.delta = c.p[6];
    return v;
  } else {
    return phfem_coeffs_eval(&c, v0.x, v0.y, v1.x, v1.y, v2.x, v2.y);
  }
}

// phfem_field_eval for the kinds the configs use; others go through the
// shared runtime switch
template <int FK>
__device__ __forceinline__ double field_dev(const phfem_field& f, double x, double y, double t) {
  if (FK == PHFEM_FIELD_SINSIN) return f.p[0] * sin_fast(PHFEM_PI * x) * sin_fast(PHFEM_PI * y);
  if (FK == PHFEM_FIELD_EXP_SINSIN)
    return exp(-t) * f.p[0] * sin_fast(PHFEM_PI * x) * sin_fast(PHFEM_PI * y);
  if (FK == PHFEM_FIELD_ZERO) return 0.0;
  return phfem_field_eval(&f, x, y, t);
}

// convection block (assembly.cpp:68-71) with the division by 3.0 of fastmath
__device__ __forceinline__ void convection_dev(const phfem_geom* g, const phfem_coeff_values* c,
                                               double* Dk) {
  const double a3 = div3(g->area);
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const double dj = a3 * (c->px * g->gx[j] + c->py * g->gy[j]);
    Dk[3 * j + 0] = dj;
    Dk[3 * j + 1] = dj;
    Dk[3 * j + 2] = dj;
  }
}

// assemble_load's per-element rule (assembly.cpp:185-201): f at the three edge
// midpoints, b_i = 0.0 + (|T|/3 * 0.5) * (f_{i+1} + f_{i+2}) (the 0.0 + is
// scatter_add's zero-initialised accumulation, sparse.cpp:112-118).
template <int FK>
__device__ __forceinline__ void element_load_dev(double2 v0, double2 v1, double2 v2,
                                                 const phfem_field& f, double t, double bl[3],
                                                 bool valid, int64_t m, phfem_dev_errors* err,
                                                 const double* __restrict__ samples = nullptr) {
  const double mx[3] = {0.5 * (v1.x + v2.x), 0.5 * (v2.x + v0.x), 0.5 * (v0.x + v1.x)};
  const double my[3] = {0.5 * (v1.y + v2.y), 0.5 * (v2.y + v0.y), 0.5 * (v0.y + v1.y)};
  const double area = 0.5 * ((v1.x - v0.x) * (v2.y - v0.y) - (v1.y - v0.y) * (v2.x - v0.x));
  double fm[3];
  if (FK == PHFEM_FIELD_SINSIN || FK == PHFEM_FIELD_EXP_SINSIN) {
    // one range check for the element's 6 sines instead of one branch each
    bool ok = true;
#pragma unroll
    for (int i = 0; i < 3; ++i) ok = ok && sin_fast_ok(PHFEM_PI * mx[i]) && sin_fast_ok(PHFEM_PI * my[i]);
    const double c = FK == PHFEM_FIELD_EXP_SINSIN ? exp(-t) * f.p[0] : f.p[0];
#pragma unroll
    for (int i = 0; i < 3; ++i)
      fm[i] = ok ? c * sin_fast_core(PHFEM_PI * mx[i]) * sin_fast_core(PHFEM_PI * my[i])
                 : field_dev<FK>(f, mx[i], my[i], t);
  } else {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      if (FK == kKindSamples) fm[i] = valid ? samples[3 * m + i] : 0.0;
      else fm[i] = field_dev<FK>(f, mx[i], my[i], t);
    }
  }
#pragma unroll
  for (int i = 0; i < 3; ++i)
    if (valid && !isfinite(fm[i])) atomicMin(&err->load_nan, (unsigned long long)m);
  const double w = div3(area) * 0.5;
#pragma unroll
  for (int i = 0; i < 3; ++i) bl[i] = 0.0 + w * (fm[(i + 1) % 3] + fm[(i + 2) % 3]);
}

// dispatch helper: the field kinds with a compiled specialisation
inline int field_kind_spec(const phfem_field& f) {
  return (f.kind == PHFEM_FIELD_SINSIN || f.kind == PHFEM_FIELD_EXP_SINSIN ||
          f.kind == PHFEM_FIELD_ZERO)
             ? f.kind
             : kKindGeneric;
}

}  // namespace phfem
