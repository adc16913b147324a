// edge_topology_b200.cpp — drop-in for proj/src/edge_topology.cpp: the
// functions declared in proj/include/phfem/edge_topology.hpp, computed by the
// sm_100a kernels of libphfem_b200.so.
//
//   build_topology      edge_topology.hpp:49  -> phfem_build_topology + phfem_topology_tables
//   classify_edges      edge_topology.hpp:64  -> phfem_classify_edges
//   edge_lengths        edge_topology.hpp:67  -> phfem_edge_lengths
//   edge_normal         edge_topology.hpp:71  (one edge: host arithmetic, same expression)
//   node_pair_to_edge / directed_pair_to_element (edge_topology.hpp:29-35):
//                       row scans of the tables the device built
#include "phfem/edge_topology.hpp"

#include "device.hpp"

namespace phfem {

using b200::check;
using b200::context;
using b200::DeviceBuffer;

int EdgeTopology::node_pair_to_edge(int k, int l) const {
  const int a = k < l ? k : l, b = k < l ? l : k;
  if (a < 0 || b >= node_count) return -1;
  for (int s = pair_offsets[a], t = pair_offsets[a + 1]; s < t; ++s)
    if (pair_entries[s].first == b) return pair_entries[s].second;
  return -1;
}

int EdgeTopology::directed_pair_to_element(int k, int l) const {
  if (k < 0 || k >= node_count) return -1;
  for (int s = directed_offsets[k], t = directed_offsets[k + 1]; s < t; ++s)
    if (directed_entries[s].first == l) return directed_entries[s].second;
  return -1;
}

EdgeTopology build_topology(const Mesh& mesh) {
  const b200::DeviceMesh dm(mesh);
  b200::OwnedTopology t;
  check(phfem_build_topology(context(), dm.get(), &t.t));
  const std::size_t E = static_cast<std::size_t>(t.t.E), nc = mesh.coordinates.size(),
                    nd = 3 * mesh.elements.size();
  const auto en = DeviceBuffer<int32_t>::to_host(t.t.edge_nodes, 2 * E);
  const auto el = DeviceBuffer<int32_t>::to_host(t.t.edge_elements, 2 * E);

  EdgeTopology topo;
  topo.node_count = static_cast<int>(nc);
  topo.edge_nodes.resize(E);
  topo.edge_elements.resize(E);
  for (std::size_t e = 0; e < E; ++e) {
    topo.edge_nodes[e] = {en[2 * e], en[2 * e + 1]};
    topo.edge_elements[e] = {el[2 * e], el[2 * e + 1]};
  }
  topo.local_in_tplus = DeviceBuffer<int32_t>::to_host(t.t.local_in_tplus, E);
  topo.local_in_tminus = DeviceBuffer<int32_t>::to_host(t.t.local_in_tminus, E);
  topo.interior_edges = DeviceBuffer<int32_t>::to_host(t.t.interior_edges, t.t.n_interior);
  topo.boundary_edges = DeviceBuffer<int32_t>::to_host(t.t.boundary_edges, t.t.n_boundary);

  // the flat lookup tables (edge_topology.cpp:117-140), built on the device
  DeviceBuffer<int32_t> po(nc + 1), pe(2 * E), dof(nc + 1), de(2 * nd);
  check(phfem_topology_tables(context(), dm.get(), &t.t, po.get(), pe.get(), dof.get(), de.get()));
  topo.pair_offsets = po.download(nc + 1);
  topo.directed_offsets = dof.download(nc + 1);
  const auto pev = pe.download(2 * E);
  const auto dev = de.download(2 * nd);
  topo.pair_entries.resize(E);
  for (std::size_t i = 0; i < E; ++i) topo.pair_entries[i] = {pev[2 * i], pev[2 * i + 1]};
  topo.directed_entries.resize(nd);
  for (std::size_t i = 0; i < nd; ++i) topo.directed_entries[i] = {dev[2 * i], dev[2 * i + 1]};
  return topo;
}

EdgeClassification classify_edges(const EdgeTopology& topology, const Mesh& mesh) {
  const b200::DeviceMesh dm(mesh);
  const b200::DeviceTopology dt(dm, topology, "classify_edges");
  b200::OwnedClassification c;
  check(phfem_classify_edges(context(), dt.get(), dm.get(), &c.c));
  EdgeClassification cls;
  cls.dirichlet_edge_ids = DeviceBuffer<int32_t>::to_host(c.c.dirichlet_edge_ids, c.c.nD);
  cls.neumann_edge_ids = DeviceBuffer<int32_t>::to_host(c.c.neumann_edge_ids, c.c.nN);
  cls.retained_edges = DeviceBuffer<int32_t>::to_host(c.c.retained_edges, c.c.L);
  cls.retained_pos = DeviceBuffer<int32_t>::to_host(c.c.retained_pos, c.c.E);
  return cls;
}

std::vector<double> edge_lengths(const Mesh& mesh, const EdgeTopology& topology) {
  const b200::DeviceMesh dm(mesh);
  const b200::DeviceTopology dt(dm, topology, "edge_lengths");
  DeviceBuffer<double> out(static_cast<std::size_t>(topology.edge_count()));
  check(phfem_edge_lengths(context(), dm.get(), dt.get(), out.get()));
  return out.download(out.size());
}

// A single edge: the same expression as the kernels (Vec2(dy, -dx) / |d|).
Vec2 edge_normal(const Mesh& mesh, const EdgeTopology& topology, int edge_id) {
  const auto& ab = topology.edge_nodes[edge_id];
  const Vec2 d = mesh.coordinates[ab[1]] - mesh.coordinates[ab[0]];
  return Vec2(d.y(), -d.x()) / d.norm();
}

}  // namespace phfem
