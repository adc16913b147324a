// device.cpp — context, exception mapping and host<->HBM mirrors of the
// reference's Mesh / EdgeTopology / EdgeClassification for the drop-in layer.
#include "device.hpp"

#include <cstdlib>
#include <memory>

namespace phfem::b200 {

namespace {
struct CtxHolder {
  phfem_ctx* ctx = nullptr;
  ~CtxHolder() {
    if (ctx) phfem_ctx_destroy(ctx);
  }
};
}  // namespace

phfem_ctx* context() {
  thread_local CtxHolder holder;
  if (!holder.ctx) {
    const char* dev = std::getenv("PHFEM_DEVICE");
    const int device = dev ? std::atoi(dev) : 0;
    phfem_ctx* c = nullptr;
    const phfem_status st = phfem_ctx_create(device, nullptr, &c);
    if (st != PHFEM_OK)
      throw std::runtime_error("phfem (B200): no usable sm_100 device " + std::to_string(device) +
                               " (status " + std::to_string(static_cast<int>(st)) + ")");
    holder.ctx = c;
  }
  return holder.ctx;
}

void raise(phfem_status st, const std::string& prefix) {
  const std::string msg = prefix + phfem_ctx_message(context());
  switch (st) {
    case PHFEM_ERR_INVALID_ARGUMENT:
      throw std::invalid_argument(msg);
    case PHFEM_ERR_OUT_OF_RANGE:
      throw std::out_of_range(msg);
    default:
      throw std::runtime_error(msg);
  }
}

DeviceMesh::DeviceMesh(const Mesh& mesh) {
  const std::size_t nc = mesh.coordinates.size(), ne = mesh.elements.size();
  const std::size_t nd = mesh.dirichlet_edges.size(), nn = mesh.neumann_edges.size();
  std::vector<double> xy(2 * nc);
  for (std::size_t i = 0; i < nc; ++i) {
    xy[2 * i] = mesh.coordinates[i].x();
    xy[2 * i + 1] = mesh.coordinates[i].y();
  }
  auto flat = [](const auto& rows, std::size_t w) {
    std::vector<int32_t> v(rows.size() * w);
    for (std::size_t i = 0; i < rows.size(); ++i)
      for (std::size_t k = 0; k < w; ++k) v[w * i + k] = rows[i][k];
    return v;
  };
  coords_ = DeviceBuffer<double>(xy);
  elements_ = DeviceBuffer<int32_t>(flat(mesh.elements, 3));
  dirichlet_ = DeviceBuffer<int32_t>(flat(mesh.dirichlet_edges, 2));
  neumann_ = DeviceBuffer<int32_t>(flat(mesh.neumann_edges, 2));
  m_.coords = coords_.get();
  m_.elements = elements_.get();
  m_.dirichlet = dirichlet_.get();
  m_.neumann = neumann_.get();
  m_.nC = static_cast<int32_t>(nc);
  m_.nE = static_cast<int32_t>(ne);
  m_.nD = static_cast<int32_t>(nd);
  m_.nN = static_cast<int32_t>(nn);
  m_.owned = 0;
}

DeviceTopology::DeviceTopology(const DeviceMesh& mesh, const EdgeTopology& topo, const char* who) {
  const std::size_t E = topo.edge_nodes.size();
  if (topo.edge_elements.size() != E || topo.local_in_tplus.size() != E ||
      topo.local_in_tminus.size() != E)
    throw std::runtime_error(std::string(who) + ": topology does not match mesh");
  std::vector<int32_t> en(2 * E), el(2 * E);
  for (std::size_t e = 0; e < E; ++e) {
    en[2 * e] = topo.edge_nodes[e][0];
    en[2 * e + 1] = topo.edge_nodes[e][1];
    el[2 * e] = topo.edge_elements[e][0];
    el[2 * e + 1] = topo.edge_elements[e][1];
  }
  en_ = DeviceBuffer<int32_t>(en);
  el_ = DeviceBuffer<int32_t>(el);
  ltp_ = DeviceBuffer<int32_t>(topo.local_in_tplus);
  ltm_ = DeviceBuffer<int32_t>(topo.local_in_tminus);
  in_ = DeviceBuffer<int32_t>(topo.interior_edges);
  bn_ = DeviceBuffer<int32_t>(topo.boundary_edges);
  t_.nC = mesh.get()->nC;
  t_.nE = mesh.get()->nE;
  t_.E = static_cast<int32_t>(E);
  t_.n_interior = static_cast<int32_t>(topo.interior_edges.size());
  t_.n_boundary = static_cast<int32_t>(topo.boundary_edges.size());
  t_.edge_nodes = en_.get();
  t_.edge_elements = el_.get();
  t_.local_in_tplus = ltp_.get();
  t_.local_in_tminus = ltm_.get();
  t_.interior_edges = in_.get();
  t_.boundary_edges = bn_.get();
  const phfem_status st = phfem_topology_derive(context(), mesh.get(), &t_);
  if (st == PHFEM_ERR_MISMATCH)
    throw std::runtime_error(std::string(who) + ": topology does not match mesh");
  check(st);
}

DeviceTopology::~DeviceTopology() {
  // only the derived arrays belong to the library; the rest are DeviceBuffers
  if (t_.elem_edge) phfem_free(context(), t_.elem_edge);
  if (t_.node_edge_start) phfem_free(context(), t_.node_edge_start);
}

DeviceClassification::DeviceClassification(const DeviceMesh& mesh, const DeviceTopology& topo,
                                           const EdgeClassification& cls) {
  check(phfem_classify_edges(context(), topo.get(), mesh.get(), &c_));
  const auto same = [](const int32_t* dev, int n, const std::vector<int>& host) {
    if (static_cast<std::size_t>(n) != host.size()) return false;
    const std::vector<int32_t> d = DeviceBuffer<int32_t>::to_host(dev, static_cast<std::size_t>(n));
    for (int i = 0; i < n; ++i)
      if (d[i] != host[i]) return false;
    return true;
  };
  if (!same(c_.retained_pos, c_.E, cls.retained_pos) ||
      !same(c_.dirichlet_edge_ids, c_.nD, cls.dirichlet_edge_ids) ||
      !same(c_.neumann_edge_ids, c_.nN, cls.neumann_edge_ids)) {
    phfem_classification_release(context(), &c_);
    throw std::runtime_error("classification does not match topology");
  }
}

DeviceClassification::~DeviceClassification() { phfem_classification_release(context(), &c_); }

Mesh download_mesh(const phfem_mesh& m) {
  Mesh out;
  const std::vector<double> xy = DeviceBuffer<double>::to_host(m.coords, 2 * static_cast<std::size_t>(m.nC));
  const std::vector<int32_t> el = DeviceBuffer<int32_t>::to_host(m.elements, 3 * static_cast<std::size_t>(m.nE));
  const std::vector<int32_t> d = DeviceBuffer<int32_t>::to_host(m.dirichlet, 2 * static_cast<std::size_t>(m.nD));
  const std::vector<int32_t> n = DeviceBuffer<int32_t>::to_host(m.neumann, 2 * static_cast<std::size_t>(m.nN));
  out.coordinates.resize(m.nC);
  for (int i = 0; i < m.nC; ++i) out.coordinates[i] = Vec2(xy[2 * i], xy[2 * i + 1]);
  out.elements.resize(m.nE);
  for (int i = 0; i < m.nE; ++i) out.elements[i] = {el[3 * i], el[3 * i + 1], el[3 * i + 2]};
  out.dirichlet_edges.resize(m.nD);
  for (int i = 0; i < m.nD; ++i) out.dirichlet_edges[i] = {d[2 * i], d[2 * i + 1]};
  out.neumann_edges.resize(m.nN);
  for (int i = 0; i < m.nN; ++i) out.neumann_edges[i] = {n[2 * i], n[2 * i + 1]};
  return out;
}

}  // namespace phfem::b200
