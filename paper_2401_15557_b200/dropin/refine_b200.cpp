// refine_b200.cpp — drop-in for proj/src/refine.cpp: red_refine
// (refine.hpp:15) on the device.  The topology is checked against the mesh
// on the device (phfem_topology_derive), which is where the reference's
// midpoint lookups throw "red_refine: topology does not match mesh"
// (refine.cpp:21-25).
#include "phfem/refine.hpp"

#include "device.hpp"

namespace phfem {

Mesh red_refine(const Mesh& mesh, const EdgeTopology& topology) {
  const b200::DeviceMesh dm(mesh);
  const b200::DeviceTopology dt(dm, topology, "red_refine");
  b200::OwnedMesh fine;
  b200::check(phfem_red_refine(b200::context(), dm.get(), dt.get(), &fine.m));
  return b200::download_mesh(fine.m);
}

}  // namespace phfem
