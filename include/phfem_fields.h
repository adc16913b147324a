/*
 * phfem_fields.h — closed descriptors for the data fields and coefficients of
 * the primal hybrid FEM hot path, plus the ONE inline formula per kind that
 * every side evaluates (CUDA kernels, the C-ABI host code, the C oracle and the
 * lambdas handed to the reference build).
 *
 * Why: the reference passes data as std::function (proj/include/phfem/
 * assembly.hpp:15-19, ScalarField / FluxField), which cannot cross to the
 * device.  The drop-in boundary therefore takes a tagged union; both the GPU
 * path and the CPU oracle call the same expression below, so any difference
 * between them is the libm-vs-CUDA sin/cos/exp ulp, nothing else.
 *
 * Every expression is written in the exact left-to-right operation order the
 * reference / BASELINE formula uses; kernels are compiled with --fmad=false so
 * no contraction changes the rounding.
 */
#ifndef PHFEM_FIELDS_H
#define PHFEM_FIELDS_H

#include <stdint.h>
#include <math.h>

#if defined(__CUDACC__)
#define PHFEM_HD __host__ __device__ __forceinline__
#else
#define PHFEM_HD static inline
#endif

#ifndef PHFEM_PI
#define PHFEM_PI 3.14159265358979323846
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- scalar fields f(x, t), u_D(x, t) (reference ScalarField) ------------ */
enum phfem_field_kind {
  PHFEM_FIELD_ZERO = 0,       /* 0                                           */
  PHFEM_FIELD_CONST = 1,      /* p0                                          */
  PHFEM_FIELD_SINSIN = 2,     /* p0 * sin(pi x) * sin(pi y)   (cfg 1/2: p0 = 2 pi^2) */
  PHFEM_FIELD_EXP_SINSIN = 3, /* exp(-t) * p0 * sin(pi x) * sin(pi y) (cfg 3: p0 = 2 pi^2 - 1) */
  PHFEM_FIELD_AFFINE = 4,     /* p0 + p1 x + p2 y + p3 t                     */
  PHFEM_FIELD_SIN3X = 5,      /* sin(3x) (1 + y^2)  (test_assembly.cpp:295-297 KAT) */
  PHFEM_FIELD_NAN = 6         /* quiet NaN (error-path tests, test_assembly.cpp:286-289) */
};

/* ---- Neumann fluxes g(x, nu, t) (reference FluxField) -------------------- */
enum phfem_flux_kind {
  PHFEM_FLUX_ZERO = 0,        /* 0                                           */
  PHFEM_FLUX_CONST = 1,       /* p0                                          */
  PHFEM_FLUX_GRAD_SINSIN = 2, /* grad(p0 sin(pi x) sin(pi y)) . nu   (cfg 1) */
  PHFEM_FLUX_VEC_KAT = 3      /* (cos y + x, x y - 1) . nu  (test_assembly.cpp:353-358) */
};

/* ---- coefficients A, p, delta (reference ProblemCoefficients) ------------ */
enum phfem_coeff_kind {
  PHFEM_COEFF_CONST = 0,         /* A = [[p0,p1],[p2,p3]], p = (p4,p5), delta = p6 */
  PHFEM_COEFF_CENTROID_POLY = 1  /* cfg 2/4: at centroid xc: A = [[1+x^2, 0.5xy],[0.5xy, 1+y^2]],
                                    p = (p4, p5), delta = 1 + x + y          */
};

typedef struct phfem_field {
  int32_t kind;
  int32_t reserved;
  double p[6];
} phfem_field;

typedef struct phfem_coeffs {
  int32_t kind;
  int32_t reserved;
  double p[8];
} phfem_coeffs;

/* Per-element coefficient values after evaluation. */
typedef struct phfem_coeff_values {
  double a00, a01, a10, a11, px, py, delta;
} phfem_coeff_values;

PHFEM_HD double phfem_field_eval(const phfem_field* f, double x, double y, double t) {
  switch (f->kind) {
    case PHFEM_FIELD_CONST: return f->p[0];
    case PHFEM_FIELD_SINSIN: return f->p[0] * sin(PHFEM_PI * x) * sin(PHFEM_PI * y);
    case PHFEM_FIELD_EXP_SINSIN: return exp(-t) * f->p[0] * sin(PHFEM_PI * x) * sin(PHFEM_PI * y);
    case PHFEM_FIELD_AFFINE: return f->p[0] + f->p[1] * x + f->p[2] * y + f->p[3] * t;
    case PHFEM_FIELD_SIN3X: return sin(3.0 * x) * (1.0 + y * y);
    case PHFEM_FIELD_NAN: return NAN;
    default: return 0.0;
  }
}

PHFEM_HD double phfem_flux_eval(const phfem_field* g, double x, double y, double nx, double ny,
                                double t) {
  (void)t;
  switch (g->kind) {
    case PHFEM_FLUX_CONST: return g->p[0];
    case PHFEM_FLUX_GRAD_SINSIN: {
      const double gx = g->p[0] * PHFEM_PI * cos(PHFEM_PI * x) * sin(PHFEM_PI * y);
      const double gy = g->p[0] * PHFEM_PI * sin(PHFEM_PI * x) * cos(PHFEM_PI * y);
      return gx * nx + gy * ny; /* Eigen dot: x*x' + y*y' */
    }
    case PHFEM_FLUX_VEC_KAT: {
      const double vx = cos(y) + x;
      const double vy = x * y - 1.0;
      return vx * nx + vy * ny;
    }
    default: return 0.0;
  }
}

/* Coefficients of element with vertices (x0,y0),(x1,y1),(x2,y2). */
PHFEM_HD phfem_coeff_values phfem_coeffs_eval(const phfem_coeffs* c, double x0, double y0,
                                              double x1, double y1, double x2, double y2) {
  phfem_coeff_values v;
  if (c->kind == PHFEM_COEFF_CENTROID_POLY) {
    const double xc = (x0 + x1 + x2) / 3.0;
    const double yc = (y0 + y1 + y2) / 3.0;
    v.a00 = 1.0 + xc * xc;
    v.a01 = 0.5 * xc * yc;
    v.a10 = v.a01;
    v.a11 = 1.0 + yc * yc;
    v.px = c->p[4];
    v.py = c->p[5];
    v.delta = 1.0 + xc + yc;
  } else {
    v.a00 = c->p[0];
    v.a01 = c->p[1];
    v.a10 = c->p[2];
    v.a11 = c->p[3];
    v.px = c->p[4];
    v.py = c->p[5];
    v.delta = c->p[6];
  }
  return v;
}

/*
 * Local element matrices in the reference's exact operation order
 * (proj/src/assembly.cpp:17-27 element_geometry, :53-78 local_element_matrices,
 * :134-140 unit mass).  Blocks are column-major 3x3 (out[3*j+i] = X(i,j)),
 * i.e. exactly the 9 values assemble_block_diagonal writes per element
 * (assembly.cpp:106-114).  The pieces are separate so a kernel can emit one
 * block at a time; phfem_local_blocks composes them.
 */
typedef struct phfem_geom {
  double t2, area;
  double gx[3], gy[3]; /* grad lambda_i */
} phfem_geom;

PHFEM_HD phfem_geom phfem_geometry(double x0, double y0, double x1, double y1, double x2,
                                   double y2) {
  phfem_geom g;
  /* mesh.cpp:104-106 signed_area2 */
  g.t2 = (x1 - x0) * (y2 - y0) - (y1 - y0) * (x2 - x0);
  g.area = 0.5 * g.t2;
  /* assembly.cpp:23-25: Vec2(...) / twice_area (component-wise division) */
  g.gx[0] = (y1 - y2) / g.t2;
  g.gy[0] = (x2 - x1) / g.t2;
  g.gx[1] = (y2 - y0) / g.t2;
  g.gy[1] = (x0 - x2) / g.t2;
  g.gx[2] = (y0 - y1) / g.t2;
  g.gy[2] = (x1 - x0) / g.t2;
  return g;
}

/* :59-64 stiffness from the upper triangle: area * (A g_i) . g_j */
PHFEM_HD void phfem_stiffness(const phfem_geom* g, const phfem_coeff_values* c, double* Bk) {
  for (int i = 0; i < 3; ++i) {
    const double rx = c->a00 * g->gx[i] + c->a01 * g->gy[i];
    const double ry = c->a10 * g->gx[i] + c->a11 * g->gy[i];
    for (int j = i; j < 3; ++j) {
      const double v = g->area * (rx * g->gx[j] + ry * g->gy[j]);
      Bk[3 * j + i] = v;
      Bk[3 * i + j] = v;
    }
  }
}

/* :68-71 convection: column-constant area/3 * p . g_j */
PHFEM_HD void phfem_convection(const phfem_geom* g, const phfem_coeff_values* c, double* Dk) {
  for (int j = 0; j < 3; ++j) {
    const double dj = g->area / 3.0 * (c->px * g->gx[j] + c->py * g->gy[j]);
    Dk[3 * j + 0] = dj;
    Dk[3 * j + 1] = dj;
    Dk[3 * j + 2] = dj;
  }
}

/* :73-75 mass, delta-scaled: delta * area * {1/6, 1/12} */
PHFEM_HD void phfem_mass(const phfem_geom* g, double delta, double* Mk) {
  const double md = delta * g->area * (1.0 / 6.0);
  const double mo = delta * g->area * (1.0 / 12.0);
  for (int j = 0; j < 3; ++j)
    for (int i = 0; i < 3; ++i) Mk[3 * j + i] = (i == j) ? md : mo;
}

/* :134-140 unit mass: area * {1/6, 1/12} */
PHFEM_HD void phfem_unit_mass(const phfem_geom* g, double* M0k) {
  const double ud = g->area * (1.0 / 6.0);
  const double uo = g->area * (1.0 / 12.0);
  for (int j = 0; j < 3; ++j)
    for (int i = 0; i < 3; ++i) M0k[3 * j + i] = (i == j) ? ud : uo;
}

/* All four blocks; returns twice the signed area (!(t2 > 0) is the
 * reference's "degenerate or non-CCW triangle" error, assembly.cpp:19-20). */
PHFEM_HD double phfem_local_blocks(double x0, double y0, double x1, double y1, double x2,
                                   double y2, const phfem_coeff_values* c, double* Bk,
                                   double* Dk, double* Mk, double* M0k) {
  const phfem_geom g = phfem_geometry(x0, y0, x1, y1, x2, y2);
  phfem_stiffness(&g, c, Bk);
  phfem_convection(&g, c, Dk);
  phfem_mass(&g, c->delta, Mk);
  phfem_unit_mass(&g, M0k);
  return g.t2;
}

/*
 * ---- manufactured problems (verification) ----------------
 * The exact solution u and its gradient, for the error norms and the exact
 * multiplier (analysis.cpp:26-95).  The two registry problems restate
 * problems.cpp:85-150 in the lambdas' own operation order; SINSIN is the
 * config-1 solution u = sin(pi x) sin(pi y) behind FLUX_GRAD_SINSIN (not in
 * the reference's registry).
 */
enum phfem_problem_kind {
  PHFEM_PROBLEM_ELLIPTIC_POLY = 1,  /* u = mu(x) mu(y), mu(s) = s - s s          */
  PHFEM_PROBLEM_PARABOLIC_POLY = 2, /* u = t mu(x) mu(y)                         */
  PHFEM_PROBLEM_SINSIN = 3          /* u = sin(pi x) sin(pi y)                   */
};

typedef struct phfem_problem {
  int32_t kind;
  int32_t reserved;
  phfem_coeffs coeffs; /* problem.coeffs (constant): A, p for exact_multiplier */
} phfem_problem;

PHFEM_HD double phfem_mu(double s) { return s - s * s; }      /* problems.cpp:91 */
PHFEM_HD double phfem_dmu(double s) { return 1.0 - 2.0 * s; } /* problems.cpp:92 */

PHFEM_HD double phfem_problem_u(const phfem_problem* p, double x, double y, double t) {
  switch (p->kind) {
    case PHFEM_PROBLEM_ELLIPTIC_POLY: return phfem_mu(x) * phfem_mu(y);
    case PHFEM_PROBLEM_PARABOLIC_POLY: return t * phfem_mu(x) * phfem_mu(y);
    case PHFEM_PROBLEM_SINSIN: return sin(PHFEM_PI * x) * sin(PHFEM_PI * y);
    default: return 0.0;
  }
}

PHFEM_HD void phfem_problem_grad(const phfem_problem* p, double x, double y, double t, double* gx,
                                 double* gy) {
  switch (p->kind) {
    case PHFEM_PROBLEM_ELLIPTIC_POLY:
      *gx = phfem_dmu(x) * phfem_mu(y);
      *gy = phfem_mu(x) * phfem_dmu(y);
      return;
    case PHFEM_PROBLEM_PARABOLIC_POLY:
      *gx = t * phfem_dmu(x) * phfem_mu(y);
      *gy = t * phfem_mu(x) * phfem_dmu(y);
      return;
    case PHFEM_PROBLEM_SINSIN:
      *gx = PHFEM_PI * cos(PHFEM_PI * x) * sin(PHFEM_PI * y);
      *gy = PHFEM_PI * sin(PHFEM_PI * x) * cos(PHFEM_PI * y);
      return;
    default:
      *gx = 0.0;
      *gy = 0.0;
  }
}

/* The 25-point Duffy rule of quadrature.cpp:9-53 (TriangleQuadrature::
 * default_rule): barycentric points b[q][3], weights w[q] summing to 1.     */
typedef struct phfem_quad_rule {
  double b[25][3];
  double w[25];
} phfem_quad_rule;

PHFEM_HD void phfem_default_rule(phfem_quad_rule* r) {
  const double a = sqrt(5.0 - 2.0 * sqrt(10.0 / 7.0)) / 3.0;
  const double bb = sqrt(5.0 + 2.0 * sqrt(10.0 / 7.0)) / 3.0;
  const double wa = (322.0 + 13.0 * sqrt(70.0)) / 900.0;
  const double wb = (322.0 - 13.0 * sqrt(70.0)) / 900.0;
  const double xs[5] = {-bb, -a, 0.0, a, bb};
  const double ws[5] = {wb, wa, 128.0 / 225.0, wa, wb};
  double gx[5], gw[5];
  for (int i = 0; i < 5; ++i) {
    gx[i] = 0.5 * (xs[i] + 1.0);
    gw[i] = 0.5 * ws[i];
  }
  for (int i = 0; i < 5; ++i)
    for (int j = 0; j < 5; ++j) {
      const double xi = gx[i], eta = gx[j];
      const double x = xi, y = eta * (1.0 - xi);
      r->b[5 * i + j][0] = 1.0 - x - y;
      r->b[5 * i + j][1] = x;
      r->b[5 * i + j][2] = y;
      r->w[5 * i + j] = 2.0 * gw[i] * gw[j] * (1.0 - xi);
    }
}

/* Per-element terms of error_l2 (analysis.cpp:62-80: area * sum_q w (u - uh)^2)
 * and error_h1 (analysis.cpp:44-58: TriangleQuadrature::integrate of
 * |grad u - grad uh|^2, quadrature.hpp:25-35).                              */
PHFEM_HD double phfem_l2_term(const phfem_problem* p, const phfem_quad_rule* r, double x0,
                              double y0, double x1, double y1, double x2, double y2, double u0,
                              double u1, double u2, double t) {
  const double area = 0.5 * ((x1 - x0) * (y2 - y0) - (y1 - y0) * (x2 - x0));
  double local = 0.0;
  for (int q = 0; q < 25; ++q) {
    const double* bc = r->b[q];
    const double x = bc[0] * x0 + bc[1] * x1 + bc[2] * x2;
    const double y = bc[0] * y0 + bc[1] * y1 + bc[2] * y2;
    const double uh = bc[0] * u0 + bc[1] * u1 + bc[2] * u2;
    const double diff = phfem_problem_u(p, x, y, t) - uh;
    local += r->w[q] * diff * diff;
  }
  return area * local;
}

PHFEM_HD double phfem_h1_term(const phfem_problem* p, const phfem_quad_rule* r, double x0,
                              double y0, double x1, double y1, double x2, double y2, double u0,
                              double u1, double u2, double t) {
  /* barycentric_gradients (analysis.cpp:16-21): Vec2(...) / twice_area */
  const double t2 = (x1 - x0) * (y2 - y0) - (y1 - y0) * (x2 - x0);
  const double g0x = (y1 - y2) / t2, g0y = (x2 - x1) / t2;
  const double g1x = (y2 - y0) / t2, g1y = (x0 - x2) / t2;
  const double g2x = (y0 - y1) / t2, g2y = (x1 - x0) / t2;
  const double ghx = 0.0 + u0 * g0x + u1 * g1x + u2 * g2x; /* grad_h += U_i * grads[i] */
  const double ghy = 0.0 + u0 * g0y + u1 * g1y + u2 * g2y;
  const double area = 0.5 * ((x1 - x0) * (y2 - y0) - (y1 - y0) * (x2 - x0));
  double sum = 0.0;
  for (int q = 0; q < 25; ++q) {
    const double* bc = r->b[q];
    const double x = bc[0] * x0 + bc[1] * x1 + bc[2] * x2;
    const double y = bc[0] * y0 + bc[1] * y1 + bc[2] * y2;
    double gx, gy;
    phfem_problem_grad(p, x, y, t, &gx, &gy);
    const double dx = gx - ghx, dy = gy - ghy;
    sum += r->w[q] * (dx * dx + dy * dy);
  }
  return area * sum;
}

/* exact_multiplier value of edge (a -> b) (analysis.cpp:26-39 with
 * edge_normal, edge_topology.cpp:188-192): (A grad u + u p) . nu at the
 * midpoint, nu = (dy, -dx) / |d|.                                           */
PHFEM_HD double phfem_exact_multiplier_value(const phfem_problem* p, double ax, double ay,
                                             double bx, double by, double t) {
  const double mx = 0.5 * (ax + bx), my = 0.5 * (ay + by);
  const double dx = bx - ax, dy = by - ay;
  const double n = sqrt(dx * dx + dy * dy);
  const double nux = dy / n, nuy = -dx / n;
  double gx, gy;
  phfem_problem_grad(p, mx, my, t, &gx, &gy);
  const double u = phfem_problem_u(p, mx, my, t);
  const double* c = p->coeffs.p; /* A = [[c0, c1], [c2, c3]], p = (c4, c5) */
  const double sx = (c[0] * gx + c[1] * gy) + u * c[4];
  const double sy = (c[2] * gx + c[3] * gy) + u * c[5];
  return sx * nux + sy * nuy;
}

#ifdef __cplusplus
}
#endif

#endif /* PHFEM_FIELDS_H */
