// assembly_b200.cpp — drop-in for proj/src/assembly.cpp: the functions of
// proj/include/phfem/assembly.hpp on the device.
//
//   ProblemCoefficients ctor   assembly.hpp:30      (argument validation, host)
//   local_element_matrices     assembly.hpp:44-45   -> phfem_assemble_volume (one element)
//   local_constraint_row       assembly.hpp:50      (3 products, host)
//   assemble_volume_operators  assembly.hpp:68      -> phfem_assemble_volume
//   assemble_constraint        assembly.hpp:73-74   -> phfem_constraint_csc
//   assemble_operators         assembly.hpp:77-79
//   assemble_load              assembly.hpp:84      -> phfem_field_points + phfem_assemble_load_sampled
//   assemble_neumann           assembly.hpp:87-89   -> ... + phfem_assemble_neumann_sampled
//   assemble_dirichlet         assembly.hpp:93-95   -> ... + phfem_assemble_dirichlet_sampled
//
// ScalarField / FluxField are std::function and cannot run on the device:
// the kernels produce the sample points (same expressions as the reference),
// the callback is evaluated there on the host, and the kernels finish the
// assembly with the sampled values.  Block values are bit-identical to the
// reference; the sparse layouts are the reference's
// Eigen ColMajor ones (assembly.cpp:97-116, sparse.cpp:30-97).
#include "phfem/assembly.hpp"

#include <cmath>
#include <cstring>

#include "device.hpp"

namespace phfem {

using b200::check;
using b200::context;
using b200::DeviceBuffer;

namespace {

phfem_coeffs const_coeffs(const ProblemCoefficients& c) {
  phfem_coeffs d;
  std::memset(&d, 0, sizeof d);
  d.kind = PHFEM_COEFF_CONST;
  d.p[0] = c.A(0, 0);
  d.p[1] = c.A(0, 1);
  d.p[2] = c.A(1, 0);
  d.p[3] = c.A(1, 1);
  d.p[4] = c.p[0];
  d.p[5] = c.p[1];
  d.p[6] = c.delta;
  return d;
}

// block-diagonal N x N matrix, column 3m+j holding rows 3m..3m+2
SparseMatrix block_diagonal(int ne, const std::vector<double>& vals) {
  const int n = 3 * ne;
  Eigen::SparseMatrix<double> m(n, n);
  int* outer = m.outerIndexPtr();
  for (int c = 0; c <= n; ++c) outer[c] = 3 * c;
  m.resizeNonZeros(static_cast<Eigen::Index>(9) * ne);
  int* inner = m.innerIndexPtr();
  double* v = m.valuePtr();
  for (int e = 0; e < ne; ++e)
    for (int k = 0; k < 9; ++k) inner[9 * static_cast<std::size_t>(e) + k] = 3 * e + k % 3;
  if (!vals.empty()) std::memcpy(v, vals.data(), sizeof(double) * vals.size());
  return SparseMatrix(std::move(m));
}

Eigen::VectorXd to_vector(const std::vector<double>& v) {
  Eigen::VectorXd out(static_cast<Eigen::Index>(v.size()));
  for (std::size_t i = 0; i < v.size(); ++i) out[static_cast<Eigen::Index>(i)] = v[i];
  return out;
}

}  // namespace

ProblemCoefficients::ProblemCoefficients(const Eigen::Matrix2d& A_, const Eigen::Vector2d& p_,
                                         double delta_)
    : A(A_), p(p_), delta(delta_) {
  const double amax =
      std::fmax(std::fmax(std::fabs(A(0, 0)), std::fabs(A(0, 1))), std::fmax(std::fabs(A(1, 0)), std::fabs(A(1, 1))));
  if (std::fabs(A(0, 1) - A(1, 0)) > 1e-14 * (1.0 + amax))
    throw std::invalid_argument("ProblemCoefficients: A is not symmetric");
  if (A(0, 0) <= 0.0 || A.determinant() <= 0.0)
    throw std::invalid_argument("ProblemCoefficients: A is not positive definite");
}

LocalMatrices local_element_matrices(const std::array<Vec2, 3>& vertices,
                                     const ProblemCoefficients& coeffs) {
  Mesh one;
  one.coordinates = {vertices[0], vertices[1], vertices[2]};
  one.elements = {{0, 1, 2}};
  const b200::DeviceMesh dm(one);
  DeviceBuffer<double> b(9), d(9), m(9);
  const phfem_coeffs c = const_coeffs(coeffs);
  check(phfem_assemble_volume(context(), dm.get(), &c, b.get(), d.get(), m.get(), nullptr));
  const auto hb = b.download(9), hd = d.download(9), hm = m.download(9);
  LocalMatrices local;
  for (int j = 0; j < 3; ++j)
    for (int i = 0; i < 3; ++i) {  // column-major 3x3 blocks
      local.stiffness(i, j) = hb[3 * j + i];
      local.convection(i, j) = hd[3 * j + i];
      local.mass(i, j) = hm[3 * j + i];
    }
  return local;
}

Eigen::RowVector3d local_constraint_row(double edge_length, int sign, int local_index) {
  if (local_index < 0 || local_index > 2)
    throw std::invalid_argument("local_constraint_row: local_index must be 0, 1 or 2");
  if (edge_length <= 0.0)
    throw std::invalid_argument("local_constraint_row: edge length must be positive");
  Eigen::RowVector3d row;
  for (int c = 0; c < 3; ++c) row[c] = sign * edge_length * (c == local_index ? 0.0 : 0.5);
  return row;
}

GlobalOperators assemble_volume_operators(const Mesh& mesh, const ProblemCoefficients& coeffs) {
  const int ne = mesh.element_count();
  const b200::DeviceMesh dm(mesh);
  const std::size_t n9 = 9 * static_cast<std::size_t>(ne);
  DeviceBuffer<double> b(n9), d(n9), m(n9), m0(n9);
  const phfem_coeffs c = const_coeffs(coeffs);
  check(phfem_assemble_volume(context(), dm.get(), &c, b.get(), d.get(), m.get(), m0.get()));
  GlobalOperators ops;
  ops.primal_dofs = 3 * ne;
  ops.stiffness = block_diagonal(ne, b.download(n9));
  ops.convection = block_diagonal(ne, d.download(n9));
  ops.mass = block_diagonal(ne, m.download(n9));
  ops.mass_unit = block_diagonal(ne, m0.download(n9));
  return ops;
}

SparseMatrix assemble_constraint(const Mesh& mesh, const EdgeTopology& topology,
                                 const EdgeClassification& classification) {
  if (static_cast<int>(classification.retained_pos.size()) != topology.edge_count())
    throw std::runtime_error("assemble_constraint: classification does not match topology");
  const b200::DeviceMesh dm(mesh);
  const b200::DeviceTopology dt(dm, topology, "assemble_constraint");
  const b200::DeviceClassification dc(dm, dt, classification);
  phfem_csc csc;
  check(phfem_constraint_csc(context(), dm.get(), dt.get(), dc.get(), &csc));
  const std::size_t nnz = static_cast<std::size_t>(csc.nnz);
  const int rows = csc.rows, cols = csc.cols;
  const auto outer = DeviceBuffer<int32_t>::to_host(csc.outer, static_cast<std::size_t>(csc.cols) + 1);
  const auto inner = DeviceBuffer<int32_t>::to_host(csc.inner, nnz);
  const auto vals = DeviceBuffer<double>::to_host(csc.values, nnz);
  phfem_csc_release(context(), &csc);
  Eigen::SparseMatrix<double> m(rows, cols);
  std::memcpy(m.outerIndexPtr(), outer.data(), sizeof(int) * outer.size());
  m.resizeNonZeros(static_cast<Eigen::Index>(nnz));
  if (nnz) {
    std::memcpy(m.innerIndexPtr(), inner.data(), sizeof(int) * nnz);
    std::memcpy(m.valuePtr(), vals.data(), sizeof(double) * nnz);
  }
  return SparseMatrix(std::move(m));
}

GlobalOperators assemble_operators(const Mesh& mesh, const EdgeTopology& topology,
                                   const EdgeClassification& classification,
                                   const ProblemCoefficients& coeffs) {
  GlobalOperators ops = assemble_volume_operators(mesh, coeffs);
  ops.constraint = assemble_constraint(mesh, topology, classification);
  ops.multipliers = classification.multiplier_count();
  return ops;
}

Eigen::VectorXd assemble_load(const Mesh& mesh, const ScalarField& f, double time) {
  const std::size_t n = 3 * mesh.elements.size();
  const b200::DeviceMesh dm(mesh);
  DeviceBuffer<double> pts(2 * n), samples(n), out(n);
  check(phfem_field_points(context(), dm.get(), nullptr, nullptr, PHFEM_POINTS_LOAD, pts.get()));
  const auto xy = pts.download(2 * n);
  std::vector<double> s(n);
  for (std::size_t i = 0; i < n; ++i) s[i] = f(Vec2(xy[2 * i], xy[2 * i + 1]), time);
  samples.upload(s.data(), n);
  check(phfem_assemble_load_sampled(context(), dm.get(), samples.get(), out.get()));
  return to_vector(out.download(n));
}

Eigen::VectorXd assemble_neumann(const Mesh& mesh, const EdgeTopology& topology,
                                 const EdgeClassification& classification,
                                 const FluxField& flux, double time) {
  const std::size_t n3 = 3 * mesh.elements.size(), nn = classification.neumann_edge_ids.size();
  const b200::DeviceMesh dm(mesh);
  const b200::DeviceTopology dt(dm, topology, "assemble_neumann");
  const b200::DeviceClassification dc(dm, dt, classification);
  DeviceBuffer<double> pts(4 * nn), samples(nn), out(n3);
  check(phfem_field_points(context(), dm.get(), dt.get(), dc.get(), PHFEM_POINTS_NEUMANN, pts.get()));
  const auto p = pts.download(4 * nn);
  std::vector<double> s(nn);
  for (std::size_t i = 0; i < nn; ++i)
    s[i] = flux(Vec2(p[4 * i], p[4 * i + 1]), Vec2(p[4 * i + 2], p[4 * i + 3]), time);
  samples.upload(s.data(), nn);
  check(phfem_assemble_neumann_sampled(context(), dm.get(), dt.get(), dc.get(), samples.get(),
                                       out.get(), 0));
  return to_vector(out.download(n3));
}

Eigen::VectorXd assemble_dirichlet(const Mesh& mesh, const EdgeTopology& topology,
                                   const EdgeClassification& classification,
                                   const ScalarField& u_D, double time) {
  const std::size_t L = classification.retained_edges.size(),
                    nd = classification.dirichlet_edge_ids.size();
  const b200::DeviceMesh dm(mesh);
  const b200::DeviceTopology dt(dm, topology, "assemble_dirichlet");
  const b200::DeviceClassification dc(dm, dt, classification);
  DeviceBuffer<double> pts(2 * nd), samples(nd), out(L);
  check(phfem_field_points(context(), dm.get(), dt.get(), dc.get(), PHFEM_POINTS_DIRICHLET, pts.get()));
  const auto p = pts.download(2 * nd);
  std::vector<double> s(nd);
  for (std::size_t i = 0; i < nd; ++i) s[i] = u_D(Vec2(p[2 * i], p[2 * i + 1]), time);
  samples.upload(s.data(), nd);
  check(phfem_assemble_dirichlet_sampled(context(), dm.get(), dt.get(), dc.get(), samples.get(),
                                         out.get()));
  return to_vector(out.download(L));
}

}  // namespace phfem
