// ref_runner.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" front end over the reference's OWN hot-path sources
// (/root/reference/proj/src/{mesh,edge_topology,refine,sparse,assembly,
// parabolic,elliptic,analysis,problems,quadrature}.cpp, compiled unmodified against shim/Eigen by
// oracle/ref.mk into oracle/_ref/libphfem_ref.so).  Used to pin the C oracle
// (tests/test_oracle_vs_ref.py), to generate tests/golden, and as the
// "reference" CPU baseline of bench.py.  Never linked by the product.
#include <chrono>
#include <cstdio>
#include <sstream>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "phfem/analysis.hpp"
#include "phfem/assembly.hpp"
#include "phfem/edge_topology.hpp"
#include "phfem/elliptic.hpp"
#include "phfem/mesh.hpp"
#include "phfem/parabolic.hpp"
#include "phfem/problems.hpp"
#include "phfem/refine.hpp"
#include "phfem/sparse.hpp"

#include "../include/phfem_fields.h"

using namespace phfem;

namespace {

int fail(const std::exception& ex, char* err, size_t n, int code) {
  if (err && n) {
    std::strncpy(err, ex.what(), n - 1);
    err[n - 1] = 0;
  }
  return code;
}

#define REF_TRY(...)                                                      \
  try {                                                                   \
    __VA_ARGS__;                                                          \
  } catch (const std::invalid_argument& ex) {                             \
    return fail(ex, err, errlen, 7);                                      \
  } catch (const std::out_of_range& ex) {                                 \
    return fail(ex, err, errlen, 8);                                      \
  } catch (const std::exception& ex) {                                    \
    return fail(ex, err, errlen, 1);                                      \
  }                                                                       \
  return 0;

ScalarField scalar(const phfem_field* f) {
  const phfem_field ff = *f;
  return [ff](const Vec2& x, double t) { return phfem_field_eval(&ff, x.x(), x.y(), t); };
}

FluxField flux(const phfem_field* g) {
  const phfem_field gg = *g;
  return [gg](const Vec2& x, const Vec2& nu, double t) {
    return phfem_flux_eval(&gg, x.x(), x.y(), nu.x(), nu.y(), t);
  };
}

ProblemCoefficients coeffs_of(const phfem_coeffs* c, const std::array<Vec2, 3>& v) {
  const phfem_coeff_values cv =
      phfem_coeffs_eval(c, v[0].x(), v[0].y(), v[1].x(), v[1].y(), v[2].x(), v[2].y());
  Eigen::Matrix2d A;
  A(0, 0) = cv.a00;
  A(0, 1) = cv.a01;
  A(1, 0) = cv.a10;
  A(1, 1) = cv.a11;
  return ProblemCoefficients(A, Eigen::Vector2d(cv.px, cv.py), cv.delta);
}

void copy_block_values(const SparseMatrix& s, double* out) {
  const auto& m = s.eigen();
  std::memcpy(out, m.valuePtr(), sizeof(double) * (size_t)m.nonZeros());
}

}  // namespace

extern "C" {

void* ref_mesh_new(const double* coords, int nC, const int* elems, int nE, const int* D, int nD,
                   const int* N, int nN) {
  Mesh* m = new Mesh();
  m->coordinates.reserve(nC);
  for (int i = 0; i < nC; ++i) m->coordinates.emplace_back(coords[2 * i], coords[2 * i + 1]);
  m->elements.resize(nE);
  for (int i = 0; i < nE; ++i) m->elements[i] = {elems[3 * i], elems[3 * i + 1], elems[3 * i + 2]};
  m->dirichlet_edges.resize(nD);
  for (int i = 0; i < nD; ++i) m->dirichlet_edges[i] = {D[2 * i], D[2 * i + 1]};
  m->neumann_edges.resize(nN);
  for (int i = 0; i < nN; ++i) m->neumann_edges[i] = {N[2 * i], N[2 * i + 1]};
  return m;
}

void ref_mesh_free(void* m) { delete static_cast<Mesh*>(m); }

void ref_mesh_sizes(const void* mp, int* sz) {
  const Mesh* m = static_cast<const Mesh*>(mp);
  sz[0] = m->node_count();
  sz[1] = m->element_count();
  sz[2] = (int)m->dirichlet_edges.size();
  sz[3] = (int)m->neumann_edges.size();
}

void ref_mesh_copy(const void* mp, double* coords, int* elems, int* D, int* N) {
  const Mesh* m = static_cast<const Mesh*>(mp);
  for (size_t i = 0; i < m->coordinates.size(); ++i) {
    coords[2 * i] = m->coordinates[i].x();
    coords[2 * i + 1] = m->coordinates[i].y();
  }
  for (size_t i = 0; i < m->elements.size(); ++i)
    for (int k = 0; k < 3; ++k) elems[3 * i + k] = m->elements[i][k];
  for (size_t i = 0; i < m->dirichlet_edges.size(); ++i)
    for (int k = 0; k < 2; ++k) D[2 * i + k] = m->dirichlet_edges[i][k];
  for (size_t i = 0; i < m->neumann_edges.size(); ++i)
    for (int k = 0; k < 2; ++k) N[2 * i + k] = m->neumann_edges[i][k];
}

int ref_build_topology(const void* mp, void** out, char* err, size_t errlen) {
  REF_TRY(*out = new EdgeTopology(build_topology(*static_cast<const Mesh*>(mp))))
}

void ref_topology_free(void* t) { delete static_cast<EdgeTopology*>(t); }

void ref_topology_sizes(const void* tp, int* sz) {
  const EdgeTopology* t = static_cast<const EdgeTopology*>(tp);
  sz[0] = t->edge_count();
  sz[1] = (int)t->interior_edges.size();
  sz[2] = (int)t->boundary_edges.size();
}

void ref_topology_copy(const void* tp, int* edge_nodes, int* edge_elements, int* ltp, int* ltm,
                       int* interior, int* boundary) {
  const EdgeTopology* t = static_cast<const EdgeTopology*>(tp);
  for (int e = 0; e < t->edge_count(); ++e) {
    edge_nodes[2 * e] = t->edge_nodes[e][0];
    edge_nodes[2 * e + 1] = t->edge_nodes[e][1];
    edge_elements[2 * e] = t->edge_elements[e][0];
    edge_elements[2 * e + 1] = t->edge_elements[e][1];
    ltp[e] = t->local_in_tplus[e];
    ltm[e] = t->local_in_tminus[e];
  }
  std::memcpy(interior, t->interior_edges.data(), sizeof(int) * t->interior_edges.size());
  std::memcpy(boundary, t->boundary_edges.data(), sizeof(int) * t->boundary_edges.size());
}

int ref_node_pair_to_edge(const void* tp, int k, int l) {
  return static_cast<const EdgeTopology*>(tp)->node_pair_to_edge(k, l);
}

int ref_directed_pair_to_element(const void* tp, int k, int l) {
  return static_cast<const EdgeTopology*>(tp)->directed_pair_to_element(k, l);
}

int ref_classify_edges(const void* tp, const void* mp, void** out, char* err, size_t errlen) {
  REF_TRY(*out = new EdgeClassification(classify_edges(*static_cast<const EdgeTopology*>(tp),
                                                       *static_cast<const Mesh*>(mp))))
}

void ref_classification_free(void* c) { delete static_cast<EdgeClassification*>(c); }

void ref_classification_sizes(const void* cp, int* sz) {
  const EdgeClassification* c = static_cast<const EdgeClassification*>(cp);
  sz[0] = (int)c->dirichlet_edge_ids.size();
  sz[1] = (int)c->neumann_edge_ids.size();
  sz[2] = c->multiplier_count();
  sz[3] = (int)c->retained_pos.size();
}

void ref_classification_copy(const void* cp, int* dids, int* nids, int* redges, int* rpos) {
  const EdgeClassification* c = static_cast<const EdgeClassification*>(cp);
  std::memcpy(dids, c->dirichlet_edge_ids.data(), sizeof(int) * c->dirichlet_edge_ids.size());
  std::memcpy(nids, c->neumann_edge_ids.data(), sizeof(int) * c->neumann_edge_ids.size());
  std::memcpy(redges, c->retained_edges.data(), sizeof(int) * c->retained_edges.size());
  std::memcpy(rpos, c->retained_pos.data(), sizeof(int) * c->retained_pos.size());
}

int ref_red_refine(const void* mp, const void* tp, void** out, char* err, size_t errlen) {
  REF_TRY(*out = new Mesh(red_refine(*static_cast<const Mesh*>(mp),
                                     *static_cast<const EdgeTopology*>(tp))))
}

int ref_edge_lengths(const void* mp, const void* tp, double* out) {
  const auto L = edge_lengths(*static_cast<const Mesh*>(mp), *static_cast<const EdgeTopology*>(tp));
  std::memcpy(out, L.data(), sizeof(double) * L.size());
  return 0;
}

// B, D, M, M0 values (Eigen valuePtr of the block-diagonal CSC matrices).
// Constant coefficients go through assemble_volume_operators itself; the
// per-element (centroid) coefficients of BASELINE configs 2/4 have no
// reference API, so each element calls the reference's local_element_matrices
// with its own ProblemCoefficients and the block layout of
// assemble_block_diagonal (assembly.cpp:97-116).
int ref_assemble_volume(const void* mp, const phfem_coeffs* c, double* B, double* D, double* M,
                        double* M0, char* err, size_t errlen) {
  const Mesh& mesh = *static_cast<const Mesh*>(mp);
  REF_TRY({
    if (c->kind == PHFEM_COEFF_CONST) {
      const std::array<Vec2, 3> dummy = {Vec2(0, 0), Vec2(1, 0), Vec2(0, 1)};
      const GlobalOperators ops = assemble_volume_operators(mesh, coeffs_of(c, dummy));
      copy_block_values(ops.stiffness, B);
      copy_block_values(ops.convection, D);
      copy_block_values(ops.mass, M);
      copy_block_values(ops.mass_unit, M0);
    } else {
      for (int m = 0; m < mesh.element_count(); ++m) {
        const auto& t = mesh.elements[m];
        const std::array<Vec2, 3> v = {mesh.coordinates[t[0]], mesh.coordinates[t[1]],
                                       mesh.coordinates[t[2]]};
        const LocalMatrices lm = local_element_matrices(v, coeffs_of(c, v));
        const double area = element_area(mesh, m);
        for (int j = 0; j < 3; ++j)
          for (int i = 0; i < 3; ++i) {
            const size_t q = 9 * (size_t)m + 3 * j + i;
            B[q] = lm.stiffness(i, j);
            D[q] = lm.convection(i, j);
            M[q] = lm.mass(i, j);
            M0[q] = area * (i == j ? 1.0 / 6.0 : 1.0 / 12.0);
          }
      }
    }
  })
}

// C (L x N) from assemble_constraint: sizes first (outer may be NULL)
int ref_assemble_constraint(const void* mp, const void* tp, const void* cp, int* rows, int* cols,
                            long long* nnz, int* outer, int* inner, double* vals, char* err,
                            size_t errlen) {
  REF_TRY({
    const SparseMatrix C = assemble_constraint(*static_cast<const Mesh*>(mp),
                                               *static_cast<const EdgeTopology*>(tp),
                                               *static_cast<const EdgeClassification*>(cp));
    const auto& m = C.eigen();
    *rows = C.rows();
    *cols = C.cols();
    *nnz = C.nonzeros();
    if (outer) {
      std::memcpy(outer, m.outerIndexPtr(), sizeof(int) * (size_t)(m.outerSize() + 1));
      std::memcpy(inner, m.innerIndexPtr(), sizeof(int) * (size_t)m.nonZeros());
      std::memcpy(vals, m.valuePtr(), sizeof(double) * (size_t)m.nonZeros());
    }
  })
}

int ref_assemble_load(const void* mp, const phfem_field* f, double t, double* out, char* err,
                      size_t errlen) {
  REF_TRY({
    const Eigen::VectorXd b = assemble_load(*static_cast<const Mesh*>(mp), scalar(f), t);
    std::memcpy(out, b.data(), sizeof(double) * (size_t)b.size());
  })
}

int ref_assemble_neumann(const void* mp, const void* tp, const void* cp, const phfem_field* g,
                         double t, double* out, char* err, size_t errlen) {
  REF_TRY({
    const Eigen::VectorXd b = assemble_neumann(*static_cast<const Mesh*>(mp),
                                               *static_cast<const EdgeTopology*>(tp),
                                               *static_cast<const EdgeClassification*>(cp), flux(g), t);
    std::memcpy(out, b.data(), sizeof(double) * (size_t)b.size());
  })
}

int ref_assemble_dirichlet(const void* mp, const void* tp, const void* cp, const phfem_field* uD,
                           double t, double* out, char* err, size_t errlen) {
  REF_TRY({
    const Eigen::VectorXd b = assemble_dirichlet(*static_cast<const Mesh*>(mp),
                                                 *static_cast<const EdgeTopology*>(tp),
                                                 *static_cast<const EdgeClassification*>(cp), scalar(uD), t);
    std::memcpy(out, b.data(), sizeof(double) * (size_t)b.size());
  })
}

// The CN right-hand side exactly as solve_parabolic forms it for the step
// n -> n+1 (parabolic.cpp:78, 92-103), constant coefficients.
int ref_cn_rhs(const void* mp, const void* tp, const void* cp, const phfem_coeffs* c,
               const phfem_field* f, const phfem_field* g, const phfem_field* uD, double k, int n,
               const double* state, double* rhs, char* err, size_t errlen) {
  const Mesh& mesh = *static_cast<const Mesh*>(mp);
  const EdgeTopology& topo = *static_cast<const EdgeTopology*>(tp);
  const EdgeClassification& cls = *static_cast<const EdgeClassification*>(cp);
  REF_TRY({
    const std::array<Vec2, 3> dummy = {Vec2(0, 0), Vec2(1, 0), Vec2(0, 1)};
    const GlobalOperators ops = assemble_operators(mesh, topo, cls, coeffs_of(c, dummy));
    const auto mats = step_matrices(ops, k);
    const int n_dofs = ops.primal_dofs, n_mult = ops.multipliers;
    Eigen::VectorXd W(n_dofs + n_mult);
    for (int i = 0; i < n_dofs + n_mult; ++i) W[i] = state[i];
    const auto loads = load_at_time(mesh, topo, cls, scalar(f), flux(g), n, k);
    const auto loads_next = load_at_time(mesh, topo, cls, scalar(f), flux(g), n + 1, k);
    const Eigen::VectorXd bd_prev = assemble_dirichlet(mesh, topo, cls, scalar(uD), n * k);
    const Eigen::VectorXd bd_next = assemble_dirichlet(mesh, topo, cls, scalar(uD), (n + 1) * k);
    Eigen::VectorXd r = mats.second.eigen() * W;
    r.head(n_dofs) += k * 0.5 * (loads.first + loads.second + loads_next.first + loads_next.second);
    r.tail(n_mult) += 0.5 * (bd_prev + bd_next);
    std::memcpy(rhs, r.data(), sizeof(double) * (size_t)r.size());
  })
}

// SparseMatrix::from_triplets on a raw buffer: sizes first (outer may be NULL)
int ref_from_triplets(int rows, int cols, const int* ri, const int* ci, const double* v, long long n,
                      long long* nnz, int* outer, int* inner, double* vals, char* err, size_t errlen) {
  REF_TRY({
    TripletBuffer buf(rows, cols);
    for (long long k = 0; k < n; ++k) buf.add(ri[k], ci[k], v[k]);
    const SparseMatrix m = SparseMatrix::from_triplets(buf);
    const auto& e = m.eigen();
    *nnz = m.nonzeros();
    if (outer) {
      std::memcpy(outer, e.outerIndexPtr(), sizeof(int) * (size_t)(e.outerSize() + 1));
      std::memcpy(inner, e.innerIndexPtr(), sizeof(int) * (size_t)e.nonZeros());
      std::memcpy(vals, e.valuePtr(), sizeof(double) * (size_t)e.nonZeros());
    }
  })
}

// build_saddle_matrix (which = 0) / step_matrices(k).first (1) / .second (2)
// of assemble_operators with constant coefficients: sizes first
int ref_operator_matrix(const void* mp, const void* tp, const void* cp, const phfem_coeffs* c,
                        int which, double k, int* dim, long long* nnz, int* outer, int* inner,
                        double* vals, char* err, size_t errlen) {
  REF_TRY({
    const std::array<Vec2, 3> dummy = {Vec2(0, 0), Vec2(1, 0), Vec2(0, 1)};
    const GlobalOperators ops =
        assemble_operators(*static_cast<const Mesh*>(mp), *static_cast<const EdgeTopology*>(tp),
                           *static_cast<const EdgeClassification*>(cp), coeffs_of(c, dummy));
    SparseMatrix m;
    if (which == 0) m = build_saddle_matrix(ops);
    else m = which == 1 ? step_matrices(ops, k).first : step_matrices(ops, k).second;
    const auto& e = m.eigen();
    *dim = m.rows();
    *nnz = m.nonzeros();
    if (outer) {
      std::memcpy(outer, e.outerIndexPtr(), sizeof(int) * (size_t)(e.outerSize() + 1));
      std::memcpy(inner, e.innerIndexPtr(), sizeof(int) * (size_t)e.nonZeros());
      std::memcpy(vals, e.valuePtr(), sizeof(double) * (size_t)e.nonZeros());
    }
  })
}

// CPU baseline: one bench step on the reference — build_topology, red_refine,
// build_topology, classify_edges, B/D/M/M0, C, load + Neumann, Dirichlet.
// Returns wall seconds; the produced triangle count in *n_out.
double ref_pipeline_seconds(const void* mp, int levels, const phfem_coeffs* c, const phfem_field* f,
                            const phfem_field* g, const phfem_field* uD, long long* n_out) {
  const auto t0 = std::chrono::steady_clock::now();
  try {
    Mesh mesh = *static_cast<const Mesh*>(mp);
    for (int l = 0; l < levels; ++l) mesh = red_refine(mesh, build_topology(mesh));
    const EdgeTopology topo = build_topology(mesh);
    const EdgeClassification cls = classify_edges(topo, mesh);
    const size_t n9 = 9 * (size_t)mesh.element_count();
    std::vector<double> B(n9), D(n9), M(n9), M0(n9);
    char err[256];
    ref_assemble_volume(&mesh, c, B.data(), D.data(), M.data(), M0.data(), err, sizeof err);
    const SparseMatrix C = assemble_constraint(mesh, topo, cls);
    const Eigen::VectorXd load = assemble_load(mesh, scalar(f)) + assemble_neumann(mesh, topo, cls, flux(g));
    const Eigen::VectorXd bd = assemble_dirichlet(mesh, topo, cls, scalar(uD));
    *n_out = mesh.element_count() + (load.size() == 0 && bd.size() < 0 ? C.nonzeros() : 0);
  } catch (const std::exception&) {
    *n_out = -1;
  }
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// ---- verification around the solve (analysis.cpp; tools/main.cpp:205-207),
// with the reference's OWN registry problems ("elliptic-poly",
// "parabolic-poly", problems.cpp) ----------------------------------------------
int ref_error_norms(const void* mp, const char* problem, const double* primal, double t, double* l2,
                    double* h1, char* err, size_t errlen) {
  const Mesh& mesh = *static_cast<const Mesh*>(mp);
  REF_TRY({
    const ManufacturedProblem& p = find_problem(problem);
    DiscreteSolution sol;
    sol.primal = Eigen::VectorXd(3 * mesh.element_count());
    for (int i = 0; i < 3 * mesh.element_count(); ++i) sol.primal[i] = primal[i];
    *l2 = error_l2(mesh, sol, p, t);
    *h1 = error_h1(mesh, sol, p, t);
  })
}

int ref_exact_multiplier(const void* mp, const void* tp, const void* cp, const char* problem, double t,
                         double* out, char* err, size_t errlen) {
  REF_TRY({
    const Eigen::VectorXd k =
        exact_multiplier(*static_cast<const Mesh*>(mp), *static_cast<const EdgeTopology*>(tp),
                         *static_cast<const EdgeClassification*>(cp), find_problem(problem), t);
    std::memcpy(out, k.data(), sizeof(double) * (size_t)k.size());
  })
}

// error_multiplier(exact, discrete, constraint, stiffness): constraint =
// assemble_constraint, stiffness = the block-diagonal matrix of the given
// blocks B [nE][9] (column-major, as assemble_block_diagonal stores them)
int ref_error_multiplier(const void* mp, const void* tp, const void* cp, const double* B,
                         const double* exact, const double* discrete, int n_exact, int n_discrete,
                         double* out, char* err, size_t errlen) {
  REF_TRY({
    const Mesh& mesh = *static_cast<const Mesh*>(mp);
    const int ne = mesh.element_count();
    const SparseMatrix Cm = assemble_constraint(mesh, *static_cast<const EdgeTopology*>(tp),
                                                *static_cast<const EdgeClassification*>(cp));
    TripletBuffer buf(3 * ne, 3 * ne);
    for (int m = 0; m < ne; ++m)
      for (int j = 0; j < 3; ++j)
        for (int i = 0; i < 3; ++i) buf.add(3 * m + i, 3 * m + j, B[9 * (size_t)m + 3 * j + i]);
    const SparseMatrix stiffness = SparseMatrix::from_triplets(buf);
    Eigen::VectorXd ex(n_exact), di(n_discrete);
    for (int i = 0; i < n_exact; ++i) ex[i] = exact[i];
    for (int i = 0; i < n_discrete; ++i) di[i] = discrete[i];
    *out = error_multiplier(ex, di, Cm, stiffness);
  })
}

int ref_midpoint_traces(const void* tp, const double* primal, int n, double* out) {
  Eigen::VectorXd U(n);
  for (int i = 0; i < n; ++i) U[i] = primal[i];
  const Eigen::VectorXd tr = hybrid_midpoint_traces(*static_cast<const EdgeTopology*>(tp), U);
  std::memcpy(out, tr.data(), sizeof(double) * (size_t)tr.size());
  return 0;
}

// the CLI's residual check: (C U + bD(t)).lpNorm<Infinity>() (main.cpp:205-207)
int ref_constraint_residual(const void* mp, const void* tp, const void* cp, const phfem_field* uD,
                            double t, const double* primal, double* out, char* err, size_t errlen) {
  const Mesh& mesh = *static_cast<const Mesh*>(mp);
  const EdgeTopology& topo = *static_cast<const EdgeTopology*>(tp);
  const EdgeClassification& cls = *static_cast<const EdgeClassification*>(cp);
  REF_TRY({
    const SparseMatrix Cm = assemble_constraint(mesh, topo, cls);
    const Eigen::VectorXd bd = assemble_dirichlet(mesh, topo, cls, scalar(uD), t);
    Eigen::VectorXd U(3 * mesh.element_count());
    for (int i = 0; i < 3 * mesh.element_count(); ++i) U[i] = primal[i];
    *out = (Cm.eigen() * U + bd).lpNorm<Eigen::Infinity>();
  })
}

// y = A x for A = build_saddle_matrix (which 0) / step_matrices(k).first (1) /
// .second (2) with constant coefficients (Eigen ColMajor SpMV)
int ref_operator_spmv(const void* mp, const void* tp, const void* cp, const phfem_coeffs* c, int which,
                      double k, const double* x, double* y, char* err, size_t errlen) {
  REF_TRY({
    const std::array<Vec2, 3> dummy = {Vec2(0, 0), Vec2(1, 0), Vec2(0, 1)};
    const GlobalOperators ops =
        assemble_operators(*static_cast<const Mesh*>(mp), *static_cast<const EdgeTopology*>(tp),
                           *static_cast<const EdgeClassification*>(cp), coeffs_of(c, dummy));
    SparseMatrix m;
    if (which == 0) m = build_saddle_matrix(ops);
    else m = which == 1 ? step_matrices(ops, k).first : step_matrices(ops, k).second;
    Eigen::VectorXd xv(m.rows());
    for (int i = 0; i < m.rows(); ++i) xv[i] = x[i];
    const Eigen::VectorXd r = m.eigen() * xv;
    std::memcpy(y, r.data(), sizeof(double) * (size_t)r.size());
  })
}

// ---- on-disk formats: load_mesh / save_mesh (mesh.cpp:114-180) on in-memory
// streams, and the CLI's topology CSV (tools/main.cpp:302-323) restated with
// the reference's build_topology / edge_lengths and its fmt ("%.10g") --------
int ref_load_mesh_text(const char* c, size_t nc, const char* e, size_t ne, const char* d, size_t nd,
                       const char* n, size_t nn, void** out, char* err, size_t errlen) {
  REF_TRY({
    std::istringstream cs(std::string(c, nc)), es(std::string(e, ne)), ds(std::string(d, nd)),
        ns(std::string(n, nn));
    *out = new Mesh(load_mesh(cs, es, ds, ns));
  })
}

// which: 0 coordinates, 1 elements, 2 dirichlet, 3 neumann; buf NULL -> size
int ref_save_mesh_text(const void* mp, int which, char* buf, size_t cap, size_t* len) {
  std::ostringstream s[4];
  save_mesh(*static_cast<const Mesh*>(mp), s[0], s[1], s[2], s[3]);
  const std::string t = s[which].str();
  *len = t.size();
  if (buf && cap >= t.size()) std::memcpy(buf, t.data(), t.size());
  return 0;
}

int ref_topology_csv(const void* mp, char* buf, size_t cap, size_t* len, char* err, size_t errlen) {
  const Mesh& mesh = *static_cast<const Mesh*>(mp);
  REF_TRY({
    const EdgeTopology topo = build_topology(mesh);
    const std::vector<double> lengths = edge_lengths(mesh, topo);
    std::ostringstream out;
    out << "edge,node_start,node_end,t_plus,t_minus,led,led_tn,length\n";
    for (int e = 0; e < topo.edge_count(); ++e) {
      const auto& [a, b] = topo.edge_nodes[e];
      const auto& [tp, tm] = topo.edge_elements[e];
      char f[64];
      std::snprintf(f, sizeof f, "%.10g", lengths[e]);
      out << e + 1 << ',' << a + 1 << ',' << b + 1 << ',' << tp + 1 << ',' << tm + 1 << ','
          << topo.local_in_tplus[e] + 1 << ',' << (tm >= 0 ? topo.local_in_tminus[e] + 1 : 0) << ','
          << f << '\n';
    }
    const std::string t = out.str();
    *len = t.size();
    if (buf && cap >= t.size()) std::memcpy(buf, t.data(), t.size());
  })
}

}  // extern "C"
