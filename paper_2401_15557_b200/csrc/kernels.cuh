// kernels.cuh — internal interfaces shared by the assembly, CN-RHS and
// pipeline translation units.
#pragma once

#include "common.cuh"

namespace phfem {

struct VolArgs {
  const double2* coords;
  const int32_t* elements;
  int nE;
  int vec;  // outputs 16-byte aligned -> vector stores
  phfem_coeffs coeffs;
  phfem_field f;
  double t;
  double* B;
  double* D;
  double* M;
  double* M0;
  double* load;
  const double* samples;  // host-sampled field values [3nE] (kind kKindSamples), else null
  // non-null: `elements` are red_refine's children of these parent elements
  // [3 nE/4] (refine.cpp:27-37: child 4p = (m0, m1, m2), 4p+1 = (p0, m2, m1),
  // 4p+2 = (p1, m0, m2), 4p+3 = (p2, m1, m0)) and coords[0, parent nC) are the
  // parent's nodes: k_volume gathers the 3 parent vertices and recomputes the
  // midpoints 0.5 * (a + b) (refine.cpp:18, the same bits) instead of reading
  // 12 B of elements and 3 coordinates per child
  const int32_t* parents;
};

VolArgs make_vol_args(const phfem_mesh* mesh);
phfem_status launch_volume(phfem_ctx* ctx, const VolArgs& a, bool blocks, bool load);
phfem_status volume_errors(phfem_ctx* ctx, bool blocks, bool load);

// assemble_load's per-element rule (assembly.cpp:185-201): f at the three edge
// midpoints, b_i = 0.0 + (|T|/3 * 0.5) * (f_{i+1} + f_{i+2}) (the 0.0 + is
// scatter_add's zero-initialised accumulation, sparse.cpp:112-118).
__device__ __forceinline__ void element_load(double2 v0, double2 v1, double2 v2,
                                             const phfem_field* f, double t, double bl[3],
                                             bool valid, int64_t m, phfem_dev_errors* err) {
  const double mx[3] = {0.5 * (v1.x + v2.x), 0.5 * (v2.x + v0.x), 0.5 * (v0.x + v1.x)};
  const double my[3] = {0.5 * (v1.y + v2.y), 0.5 * (v2.y + v0.y), 0.5 * (v0.y + v1.y)};
  const double area = 0.5 * ((v1.x - v0.x) * (v2.y - v0.y) - (v1.y - v0.y) * (v2.x - v0.x));
  double fm[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    fm[i] = phfem_field_eval(f, mx[i], my[i], t);
    if (valid && !isfinite(fm[i])) atomicMin(&err->load_nan, (unsigned long long)m);
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) bl[i] = 0.0 + area / 3.0 * 0.5 * (fm[(i + 1) % 3] + fm[(i + 2) % 3]);
}

// Fibonacci hashing: the HIGH bits of m * 2^32/phi (element ids of boundary
// elements are highly structured -- low bits alone collide).
__device__ __forceinline__ uint32_t neu_hash(int m, int cap) {
  return (uint32_t)(((uint64_t)(uint32_t)m * 11400714819323198485ull) >> 32) & (uint32_t)(cap - 1);
}

struct NeuArgs {
  const double2* coords;
  const int32_t* edge_nodes;
  const int32_t* ltp;
  const int32_t* neu_ids;
  const int32_t* slot_of;
  int nN;
  phfem_field g;
  const double* samples;  // host-sampled flux values [nN] (drop-in std::function path), else null
  double* vals;
};

struct NeuTable {
  int nN = 0, cap = 0, seq = 0;
  int32_t* keys = nullptr;     // element id per slot, -1 empty
  int32_t* slot_of = nullptr;  // slot of each Neumann list entry
  double* vals = nullptr;      // [cap][3] LN values of the slot's element
};

phfem_status neu_table_build(phfem_ctx* ctx, const phfem_topology* topo,
                             const phfem_classification* cls, NeuTable* tab);
void neu_table_free(phfem_ctx* ctx, NeuTable* tab);
phfem_status neu_table_eval(phfem_ctx* ctx, const NeuTable* tab, const phfem_mesh* mesh,
                            const phfem_topology* topo, const phfem_classification* cls,
                            const phfem_field* g, double t, double* vals,
                            const double* samples = nullptr);
phfem_status neu_flux_error(phfem_ctx* ctx, const phfem_mesh* mesh, const phfem_topology* topo,
                            const phfem_classification* cls);
phfem_status neumann_into(phfem_ctx* ctx, const phfem_mesh* mesh, const phfem_topology* topo,
                          const phfem_classification* cls, const phfem_field* g, double t,
                          double* out, int accumulate, bool check, const double* samples = nullptr);
phfem_status dirichlet_into(phfem_ctx* ctx, const phfem_mesh* mesh, const phfem_topology* topo,
                            const phfem_classification* cls, const phfem_field* uD, double t,
                            double* out, const double* samples = nullptr, int32_t r_off = 0);
phfem_status constraint_csr_into(phfem_ctx* ctx, const phfem_mesh* mesh,
                                 const phfem_topology* topo, const phfem_classification* cls,
                                 phfem_csr* out);

// refine.cu / refine_topo.cu internals of the fused pipeline (mid / write_mid:
// who writes the midpoint nodes of the refined mesh)
// defer_elements: the children rows are left to the refined-level pass
// (write_elems below), which writes them together with the fine elem_edge
phfem_status red_refine_impl(phfem_ctx* ctx, const phfem_mesh* mesh, const phfem_topology* topo,
                             phfem_mesh* out, bool write_mid, bool defer_elements = false, phfem_dev_errors* deferred = nullptr);
phfem_status refine_topology_impl(phfem_ctx* ctx, const phfem_mesh* parent,
                                  const phfem_topology* ptopo, const phfem_mesh* fine,
                                  phfem_topology* out, double* mid, bool write_elems = false);
// build_topology + classify_edges + assemble_constraint in one edge pass (edge_gen.cu)
phfem_status build_topology_fused(phfem_ctx* ctx, const phfem_mesh* mesh, phfem_topology* out,
                                  phfem_classification* cls, phfem_csr* C);
phfem_status refine_level_impl(phfem_ctx* ctx, const phfem_mesh* parent,
                               const phfem_topology* ptopo, const phfem_classification* pcls,
                               const phfem_mesh* fine, phfem_topology* topo,
                               phfem_classification* cls, phfem_csr* C, double* mid,
                               bool write_elems = false);

}  // namespace phfem
