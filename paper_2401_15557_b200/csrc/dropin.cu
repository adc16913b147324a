// dropin.cu — device support for the C++ drop-in layer (paper_2401_15557_b200/
// dropin/*.cpp), which implements the reference's own C++ signatures
// (proj/include/phfem/{edge_topology,refine,assembly}.hpp) on top of this ABI:
//
//  * phfem_topology_derive: a host EdgeTopology uploaded by the caller gets its
//    device-only companions (element->edge map, max-node grouping table) and
//    is validated against the mesh (the reference's red_refine throws
//    "topology does not match mesh", refine.cpp:21-25).
//  * phfem_topology_tables: the reference's flat lookup tables behind
//    node_pair_to_edge / directed_pair_to_element (edge_topology.cpp:117-140,
//    SURVEY §8 a5): CSR by smaller node of (larger node, edge id) ascending id,
//    and CSR by initial node of (end node, element) in emission order.
//  * sample points of the std::function fields (the reference's ScalarField /
//    FluxField cannot run on the device): load midpoints (assembly.cpp:33-37),
//    Neumann midpoints + outward normals (:211-215), Dirichlet midpoints
//    (:236) — the drop-in evaluates the callback there on the host and hands
//    the values back to the *_sampled assembly calls.
#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"

namespace phfem {

constexpr int32_t kUnset = INT32_MIN;

__global__ void k_fill_i32(int32_t* __restrict__ p, int64_t n, int32_t v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// elem_edge from the per-edge incidence; every (element, local) slot must be
// written exactly once and carry the element's own vertex pair
__global__ void k_derive_elem_edge(const int32_t* __restrict__ edge_nodes,
                                   const int32_t* __restrict__ edge_elements,
                                   const int32_t* __restrict__ ltp, const int32_t* __restrict__ ltm,
                                   const int32_t* __restrict__ elements, int E, int nE,
                                   int32_t* __restrict__ elem_edge, phfem_dev_errors* err) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int a = edge_nodes[2 * e], b = edge_nodes[2 * e + 1];
    const int tp = edge_elements[2 * e], tm = edge_elements[2 * e + 1];
    const int l = ltp[e], l2 = ltm[e];
    bool ok = tp >= 0 && tp < nE && l >= 0 && l < 3;
    if (ok) {  // t_plus traverses a -> b: vertices l+1, l+2
      ok = elements[3 * (int64_t)tp + (l + 1) % 3] == a && elements[3 * (int64_t)tp + (l + 2) % 3] == b;
      if (ok) ok = atomicExch(&elem_edge[3 * (int64_t)tp + l], (int32_t)e) == kUnset;
    }
    if (ok && tm >= 0) {
      ok = tm < nE && l2 >= 0 && l2 < 3 && elements[3 * (int64_t)tm + (l2 + 1) % 3] == b &&
           elements[3 * (int64_t)tm + (l2 + 2) % 3] == a;
      if (ok) ok = atomicExch(&elem_edge[3 * (int64_t)tm + l2], ~(int32_t)e) == kUnset;
    } else if (ok && l2 != -1) {
      ok = false;
    }
    if (!ok) atomicMin(&err->misc, (unsigned long long)e);
  }
}

// canonical order check (max node, then min node, strictly ascending) and the
// max-node grouping table: node_edge_start[v] = first edge with max node >= v
__global__ void k_derive_nes(const int32_t* __restrict__ edge_nodes, int E, int nC,
                             const int32_t* __restrict__ elem_edge, int nE,
                             int32_t* __restrict__ nes, phfem_dev_errors* err) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e <= E;
       e += (int64_t)gridDim.x * blockDim.x) {
    int hi_prev = -1, lo_prev = -1;
    if (e > 0) {
      const int a = edge_nodes[2 * (e - 1)], b = edge_nodes[2 * (e - 1) + 1];
      hi_prev = max(a, b);
      lo_prev = min(a, b);
    }
    int hi = nC;  // sentinel past the last node
    if (e < E) {
      const int a = edge_nodes[2 * e], b = edge_nodes[2 * e + 1];
      hi = max(a, b);
      const int lo = min(a, b);
      if (lo < 0 || hi >= nC || hi < hi_prev || (hi == hi_prev && lo <= lo_prev))
        atomicMin(&err->classify, (unsigned long long)e);
    }
    for (int v = hi_prev + 1; v <= hi && v <= nC; ++v) nes[v] = (int32_t)e;
  }
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < 3 * (int64_t)nE;
       s += (int64_t)gridDim.x * blockDim.x)
    if (elem_edge[s] == kUnset) atomicMin(&err->misc, (unsigned long long)E);
}

// ---- lookup tables -----------------------------------------------------------
__global__ void k_tab_count(const int32_t* __restrict__ edge_nodes, int E,
                            const int32_t* __restrict__ elements, int nE,
                            int32_t* __restrict__ pcnt, int32_t* __restrict__ dcnt) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += stride)
    atomicAdd(&pcnt[min(edge_nodes[2 * e], edge_nodes[2 * e + 1])], 1);
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < 3 * (int64_t)nE; o += stride)
    atomicAdd(&dcnt[elements[o]], 1);
}

__global__ void k_tab_place(const int32_t* __restrict__ edge_nodes, int E,
                            const int32_t* __restrict__ elements, int nE,
                            int32_t* __restrict__ pcur, int32_t* __restrict__ dcur,
                            int2* __restrict__ pent, int2* __restrict__ dent) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += stride) {
    const int a = edge_nodes[2 * e], b = edge_nodes[2 * e + 1];
    pent[atomicAdd(&pcur[min(a, b)], 1)] = make_int2(max(a, b), (int)e);
  }
  // directed occurrence 3m+s: v_s -> v_{s+1} of element m (edge_topology.cpp:61-68)
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < 3 * (int64_t)nE; o += stride) {
    const int64_t m = o / 3;
    const int s = (int)(o - 3 * m);
    const int from = elements[o], to = elements[3 * m + (s + 1) % 3];
    dent[atomicAdd(&dcur[from], 1)] = make_int2(to, (int)m);
  }
}

// rows are short (node valence); order each by its second field — edge id for
// the pair table (the reference scatters in ascending id), element id for the
// directed table (emission is element-major and a node occurs once per element)
__global__ void k_tab_sort_rows(const int32_t* __restrict__ off, int n, int2* __restrict__ ent) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int s = off[v], t = off[v + 1];
    for (int i = s + 1; i < t; ++i) {
      const int2 x = ent[i];
      int j = i - 1;
      while (j >= s && ent[j].y > x.y) {
        ent[j + 1] = ent[j];
        --j;
      }
      ent[j + 1] = x;
    }
  }
}

// edge_lengths (edge_topology.cpp:179-186): |c[b] - c[a]| (Eigen norm)
__global__ void k_edge_lengths(const double2* __restrict__ coords, const int32_t* __restrict__ edge_nodes,
                               int E, double* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double2 pa = coords[edge_nodes[2 * e]], pb = coords[edge_nodes[2 * e + 1]];
    const double dx = pb.x - pa.x, dy = pb.y - pa.y;
    out[e] = sqrt(dx * dx + dy * dy);
  }
}

// ---- sample points -----------------------------------------------------------
__global__ void k_load_points(const double2* __restrict__ coords, const int32_t* __restrict__ elements,
                              int nE, double2* __restrict__ pts) {
  for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < nE;
       m += (int64_t)gridDim.x * blockDim.x) {
    const double2 v0 = coords[elements[3 * m]], v1 = coords[elements[3 * m + 1]],
                  v2 = coords[elements[3 * m + 2]];
    // 0.5 * (v[k+1] + v[k+2]) (assembly.cpp:36)
    pts[3 * m] = make_double2(0.5 * (v1.x + v2.x), 0.5 * (v1.y + v2.y));
    pts[3 * m + 1] = make_double2(0.5 * (v2.x + v0.x), 0.5 * (v2.y + v0.y));
    pts[3 * m + 2] = make_double2(0.5 * (v0.x + v1.x), 0.5 * (v0.y + v1.y));
  }
}

__global__ void k_edge_points(const double2* __restrict__ coords, const int32_t* __restrict__ edge_nodes,
                              const int32_t* __restrict__ ids, int n, int with_normal,
                              double* __restrict__ pts) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int e = ids[i];
    const double2 pa = coords[edge_nodes[2 * e]], pb = coords[edge_nodes[2 * e + 1]];
    const double mx = 0.5 * (pa.x + pb.x), my = 0.5 * (pa.y + pb.y);
    if (with_normal) {  // Vec2(d.y(), -d.x()) / d.norm()  (assembly.cpp:213-215)
      const double dx = pb.x - pa.x, dy = pb.y - pa.y;
      const double len = sqrt(dx * dx + dy * dy);
      pts[4 * i] = mx;
      pts[4 * i + 1] = my;
      pts[4 * i + 2] = dy / len;
      pts[4 * i + 3] = -dx / len;
    } else {
      pts[2 * i] = mx;
      pts[2 * i + 1] = my;
    }
  }
}

}  // namespace phfem

using namespace phfem;

PHFEM_API phfem_status phfem_topology_derive(phfem_ctx* ctx, const phfem_mesh* mesh,
                                             phfem_topology* topo) {
  if (!ctx || !mesh || !topo) return PHFEM_ERR_INVALID_ARGUMENT;
  topo->nC = mesh->nC;
  topo->nE = mesh->nE;
  dfree(ctx, topo->elem_edge);
  dfree(ctx, topo->node_edge_start);
  PHFEM_TRY(dalloc(ctx, &topo->elem_edge, 3 * (int64_t)mesh->nE));
  PHFEM_TRY(dalloc(ctx, &topo->node_edge_start, (int64_t)mesh->nC + 1));
  PHFEM_TRY(errors_reset(ctx));
  const int64_t n3 = 3 * (int64_t)mesh->nE;
  if (n3 > 0)
    PHFEM_LAUNCH(ctx, "k_fill", (k_fill_i32<<<grid_for(n3, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
        topo->elem_edge, n3, kUnset)));
  if (topo->E > 0)
    PHFEM_LAUNCH(ctx, "k_derive_elem_edge", k_derive_elem_edge<<<grid_for(topo->E, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
        topo->edge_nodes, topo->edge_elements, topo->local_in_tplus, topo->local_in_tminus,
        mesh->elements, topo->E, mesh->nE, topo->elem_edge, ctx->derr));
  PHFEM_LAUNCH(ctx, "k_derive_nes", k_derive_nes<<<grid_for((int64_t)topo->E + 1, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
      topo->edge_nodes, topo->E, mesh->nC, topo->elem_edge, mesh->nE, topo->node_edge_start, ctx->derr));
  PHFEM_TRY(errors_fetch(ctx));
  if (ctx->herr->misc != ~0ull)
    return set_error(ctx, PHFEM_ERR_MISMATCH, "topology does not match mesh");
  if (ctx->herr->classify != ~0ull)
    return set_error(ctx, PHFEM_ERR_MISMATCH, "topology is not in canonical edge order");
  return PHFEM_OK;
}

PHFEM_API phfem_status phfem_topology_tables(phfem_ctx* ctx, const phfem_mesh* mesh,
                                             const phfem_topology* topo, int32_t* pair_offsets,
                                             int32_t* pair_entries, int32_t* directed_offsets,
                                             int32_t* directed_entries) {
  if (!ctx || !mesh || !topo || !pair_offsets || !directed_offsets) return PHFEM_ERR_INVALID_ARGUMENT;
  const int nC = mesh->nC, nE = mesh->nE, E = topo->E;
  PHFEM_CUDA(ctx, cudaMemsetAsync(pair_offsets, 0, sizeof(int32_t) * ((int64_t)nC + 1), ctx->stream));
  PHFEM_CUDA(ctx, cudaMemsetAsync(directed_offsets, 0, sizeof(int32_t) * ((int64_t)nC + 1), ctx->stream));
  if (nC == 0) return PHFEM_OK;
  const int64_t work = std::max<int64_t>(E, 3 * (int64_t)nE);
  int32_t* cur = nullptr;
  PHFEM_TRY(dalloc(ctx, &cur, 2 * ((int64_t)nC + 1)));
  if (work > 0)
    PHFEM_LAUNCH(ctx, "k_tab_count", k_tab_count<<<grid_for(work, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
        topo->edge_nodes, E, mesh->elements, nE, pair_offsets, directed_offsets));
  PHFEM_TRY(scan_exclusive_i32(ctx, pair_offsets, pair_offsets, (int64_t)nC + 1, nullptr));
  PHFEM_TRY(scan_exclusive_i32(ctx, directed_offsets, directed_offsets, (int64_t)nC + 1, nullptr));
  PHFEM_CUDA(ctx, cudaMemcpyAsync(cur, pair_offsets, sizeof(int32_t) * nC, cudaMemcpyDeviceToDevice, ctx->stream));
  PHFEM_CUDA(ctx, cudaMemcpyAsync(cur + nC + 1, directed_offsets, sizeof(int32_t) * nC,
                                  cudaMemcpyDeviceToDevice, ctx->stream));
  if (work > 0)
    PHFEM_LAUNCH(ctx, "k_tab_place", k_tab_place<<<grid_for(work, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
        topo->edge_nodes, E, mesh->elements, nE, cur, cur + nC + 1, (int2*)pair_entries,
        (int2*)directed_entries));
  PHFEM_LAUNCH(ctx, "k_tab_sort_rows", k_tab_sort_rows<<<grid_for(nC, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
      pair_offsets, nC, (int2*)pair_entries));
  PHFEM_LAUNCH(ctx, "k_tab_sort_rows", k_tab_sort_rows<<<grid_for(nC, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
      directed_offsets, nC, (int2*)directed_entries));
  dfree(ctx, cur);
  return PHFEM_OK;
}

PHFEM_API phfem_status phfem_edge_lengths(phfem_ctx* ctx, const phfem_mesh* mesh,
                                          const phfem_topology* topo, double* out) {
  if (!ctx || !mesh || !topo || (!out && topo->E)) return PHFEM_ERR_INVALID_ARGUMENT;
  if (topo->E > 0)
    PHFEM_LAUNCH(ctx, "k_edge_lengths", k_edge_lengths<<<grid_for(topo->E, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
        (const double2*)mesh->coords, topo->edge_nodes, topo->E, out));
  return PHFEM_OK;
}

PHFEM_API phfem_status phfem_field_points(phfem_ctx* ctx, const phfem_mesh* mesh,
                                          const phfem_topology* topo,
                                          const phfem_classification* cls, int which,
                                          double* out) {
  if (!ctx || !mesh || !out) return PHFEM_ERR_INVALID_ARGUMENT;
  if (which == PHFEM_POINTS_LOAD) {
    if (mesh->nE > 0)
      PHFEM_LAUNCH(ctx, "k_load_points", k_load_points<<<grid_for(mesh->nE, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
          (const double2*)mesh->coords, mesh->elements, mesh->nE, (double2*)out));
    return PHFEM_OK;
  }
  if (!topo || !cls) return PHFEM_ERR_INVALID_ARGUMENT;
  const bool neu = which == PHFEM_POINTS_NEUMANN;
  if (!neu && which != PHFEM_POINTS_DIRICHLET) return PHFEM_ERR_INVALID_ARGUMENT;
  const int n = neu ? cls->nN : cls->nD;
  if (n > 0)
    PHFEM_LAUNCH(ctx, "k_edge_points", k_edge_points<<<grid_for(n, 256, ctx->num_sms * 4), 256, 0, ctx->stream>>>(
        (const double2*)mesh->coords, topo->edge_nodes, neu ? cls->neumann_edge_ids : cls->dirichlet_edge_ids,
        n, neu ? 1 : 0, out));
  return PHFEM_OK;
}

PHFEM_API phfem_status phfem_assemble_load_sampled(phfem_ctx* ctx, const phfem_mesh* mesh,
                                                   const double* samples, double* out) {
  if (!ctx || !mesh || ((!samples || !out) && mesh->nE)) return PHFEM_ERR_INVALID_ARGUMENT;
  VolArgs a = make_vol_args(mesh);
  a.samples = samples;
  a.load = out;
  a.vec = ((uintptr_t)out & 15u) == 0;
  PHFEM_TRY(errors_reset(ctx));
  PHFEM_TRY(launch_volume(ctx, a, false, true));
  PHFEM_TRY(errors_fetch(ctx));
  return volume_errors(ctx, false, true);
}

PHFEM_API phfem_status phfem_assemble_neumann_sampled(phfem_ctx* ctx, const phfem_mesh* mesh,
                                                      const phfem_topology* topo,
                                                      const phfem_classification* cls,
                                                      const double* samples, double* out,
                                                      int accumulate) {
  if (!ctx || !mesh || !topo || !cls || (!samples && cls->nN)) return PHFEM_ERR_INVALID_ARGUMENT;
  if (!accumulate && mesh->nE > 0)
    PHFEM_CUDA(ctx, cudaMemsetAsync(out, 0, sizeof(double) * 3 * (int64_t)mesh->nE, ctx->stream));
  phfem_field zero;
  memset(&zero, 0, sizeof zero);
  return neumann_into(ctx, mesh, topo, cls, &zero, 0.0, out, accumulate, true, samples);
}

PHFEM_API phfem_status phfem_assemble_dirichlet_sampled(phfem_ctx* ctx, const phfem_mesh* mesh,
                                                        const phfem_topology* topo,
                                                        const phfem_classification* cls,
                                                        const double* samples, double* out) {
  if (!ctx || !mesh || !topo || !cls || (!samples && cls->nD)) return PHFEM_ERR_INVALID_ARGUMENT;
  phfem_field zero;
  memset(&zero, 0, sizeof zero);
  return dirichlet_into(ctx, mesh, topo, cls, &zero, 0.0, out, samples);
}
