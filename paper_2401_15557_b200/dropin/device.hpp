// device.hpp — plumbing of the C++ drop-in layer: the reference's C++ entry
// points (proj/include/phfem/{edge_topology,refine,assembly}.hpp) implemented
// on the B200 C ABI (include/phfem_gpu.h).  Each call uploads its host
// arguments, runs the sm_100a kernels and returns host objects by value, the
// reference's ownership convention; failures rethrow the
// reference's exception type with the reference's message.
//
// Only the ABI is used here (no CUDA runtime headers): device memory comes
// from phfem_alloc / phfem_free, copies from phfem_memcpy_h2d / _d2h.
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "phfem/edge_topology.hpp"
#include "phfem/mesh.hpp"
#include "phfem_gpu.h"

namespace phfem::b200 {

// One context per host thread (the reference is single-threaded and keeps no
// global state; one ctx per thread keeps concurrent callers independent).
// Device: $PHFEM_DEVICE, default 0.
phfem_ctx* context();

// The reference exception for a status: runtime_error (topology, boundary,
// geometry, non-finite data, mismatch), invalid_argument, out_of_range;
// CUDA / no-device failures are runtime_error as well ("no CPU fallback").
[[noreturn]] void raise(phfem_status st, const std::string& prefix = std::string());
inline void check(phfem_status st) {
  if (st != PHFEM_OK) raise(st);
}

// RAII device buffer from the ctx pool.
template <typename T>
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(std::size_t n) : n_(n) {
    void* p = nullptr;
    check(phfem_alloc(context(), (n ? n : 1) * sizeof(T), &p));
    p_ = static_cast<T*>(p);
  }
  DeviceBuffer(const T* host, std::size_t n) : DeviceBuffer(n) { upload(host, n); }
  explicit DeviceBuffer(const std::vector<T>& host) : DeviceBuffer(host.data(), host.size()) {}
  ~DeviceBuffer() {
    if (p_) phfem_free(context(), p_);
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept : p_(std::exchange(o.p_, nullptr)), n_(o.n_) {}
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    std::swap(p_, o.p_);
    std::swap(n_, o.n_);
    return *this;
  }
  T* get() const { return p_; }
  std::size_t size() const { return n_; }
  void upload(const T* host, std::size_t n) {
    if (n) check(phfem_memcpy_h2d(context(), p_, host, n * sizeof(T)));
  }
  std::vector<T> download(std::size_t n) const { return to_host(p_, n); }
  static std::vector<T> to_host(const T* dev, std::size_t n) {
    std::vector<T> h(n);
    if (n) check(phfem_memcpy_d2h(context(), h.data(), dev, n * sizeof(T)));
    return h;
  }

 private:
  T* p_ = nullptr;
  std::size_t n_ = 0;
};

// Mesh in HBM (coords AoS double2, elements int[3], boundary pairs int[2]).
class DeviceMesh {
 public:
  explicit DeviceMesh(const Mesh& mesh);
  const phfem_mesh* get() const { return &m_; }
  phfem_mesh* get() { return &m_; }

 private:
  DeviceBuffer<double> coords_;
  DeviceBuffer<int32_t> elements_, dirichlet_, neumann_;
  phfem_mesh m_{};
};

// A host EdgeTopology in HBM, with the device-only companions (element->edge
// map, max-node grouping table) derived and checked against the mesh.
class DeviceTopology {
 public:
  DeviceTopology(const DeviceMesh& mesh, const EdgeTopology& topo, const char* who);
  ~DeviceTopology();
  DeviceTopology(const DeviceTopology&) = delete;
  DeviceTopology& operator=(const DeviceTopology&) = delete;
  const phfem_topology* get() const { return &t_; }

 private:
  DeviceBuffer<int32_t> en_, el_, ltp_, ltm_, in_, bn_;
  phfem_topology t_{};
};

// A host EdgeClassification in HBM (plus the Neumann bitmap and block
// prefixes the C / Neumann kernels use), re-derived on the device from the
// mesh's boundary lists and checked against the host object.
class DeviceClassification {
 public:
  DeviceClassification(const DeviceMesh& mesh, const DeviceTopology& topo,
                       const EdgeClassification& cls);
  ~DeviceClassification();
  DeviceClassification(const DeviceClassification&) = delete;
  DeviceClassification& operator=(const DeviceClassification&) = delete;
  const phfem_classification* get() const { return &c_; }

 private:
  phfem_classification c_{};
};

// Library-owned ABI results, released on scope exit.
struct OwnedTopology {
  phfem_topology t{};
  ~OwnedTopology() { phfem_topology_release(context(), &t); }
};
struct OwnedClassification {
  phfem_classification c{};
  ~OwnedClassification() { phfem_classification_release(context(), &c); }
};
struct OwnedMesh {
  phfem_mesh m{};
  ~OwnedMesh() { phfem_mesh_release(context(), &m); }
};

Mesh download_mesh(const phfem_mesh& m);

}  // namespace phfem::b200
