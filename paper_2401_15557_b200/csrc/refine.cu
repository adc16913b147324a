// refine.cu — red_refine and the config-4 orientation pre-pass on sm_100a.
//
// Reference: proj/src/refine.cpp:7-53.  The reference looks the three
// midpoints of every parent up with node_pair_to_edge (row scans); here the
// element->edge map written by build_topology gives them directly, the t_plus
// element of every edge writes that edge's midpoint from its own (already
// gathered) vertices, and the four children of parent m are stored as 48
// contiguous bytes (rows 4m..4m+3).
#include "common.cuh"
#include "kernels.cuh"

namespace phfem {

__global__ void __launch_bounds__(256) k_refine_elements(const double2* __restrict__ coords,
                                                         const int32_t* __restrict__ elements,
                                                         const int32_t* __restrict__ elem_edge,
                                                         int nE, int nC, double2* __restrict__ out_coords,
                                                         int4* __restrict__ out_elems, int write_mid) {
  // children rows staged per warp, stored as contiguous 512-byte warp writes
  __shared__ int4 stage[8][96];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int4* so = stage[warp];
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + warp * 32; base < nE;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = base + lane;
    if (m < nE) {
      const int p0 = __ldg(elements + 3 * m), p1 = __ldg(elements + 3 * m + 1),
                p2 = __ldg(elements + 3 * m + 2);
      const int s0 = __ldg(elem_edge + 3 * m), s1 = __ldg(elem_edge + 3 * m + 1),
                s2 = __ldg(elem_edge + 3 * m + 2);
      const int m0 = nC + (s0 >= 0 ? s0 : ~s0);  // midpoint opposite p0
      const int m1 = nC + (s1 >= 0 ? s1 : ~s1);
      const int m2 = nC + (s2 >= 0 ? s2 : ~s2);
      // children rows 4m..4m+3 (refine.cpp:33-36): (M0,M1,M2),(P0,M2,M1),(P1,M0,M2),(P2,M1,M0)
      so[3 * lane] = make_int4(m0, m1, m2, p0);
      so[3 * lane + 1] = make_int4(m2, m1, p1, m0);
      so[3 * lane + 2] = make_int4(m2, p2, m1, m0);
      // midpoints 0.5 * (c[a] + c[b]) (refine.cpp:16-19), written once by t_plus
      if (write_mid && (s0 >= 0 || s1 >= 0 || s2 >= 0)) {
        const double2 c0 = __ldg(coords + p0), c1 = __ldg(coords + p1), c2 = __ldg(coords + p2);
        if (s0 >= 0) out_coords[m0] = make_double2(0.5 * (c1.x + c2.x), 0.5 * (c1.y + c2.y));
        if (s1 >= 0) out_coords[m1] = make_double2(0.5 * (c2.x + c0.x), 0.5 * (c2.y + c0.y));
        if (s2 >= 0) out_coords[m2] = make_double2(0.5 * (c0.x + c1.x), 0.5 * (c0.y + c1.y));
      }
    }
    __syncwarp();
    const int64_t rem = nE - base;
    const int n4 = 3 * (int)(rem < 32 ? rem : 32);
    for (int i = lane; i < n4; i += 32) out_elems[3 * base + i] = so[i];
    __syncwarp();
  }
}

// refine.cpp:39-50: each pair (a,b) -> (a,mid),(mid,b), consecutive, list order.
__global__ void k_refine_boundary(const int32_t* __restrict__ dpairs, int nD,
                                  const int32_t* __restrict__ npairs, int nN,
                                  const int32_t* __restrict__ nes,
                                  const int32_t* __restrict__ edge_nodes, int nC,
                                  int4* __restrict__ dout, int4* __restrict__ nout,
                                  phfem_dev_errors* err, int4* __restrict__ cdst = nullptr,
                                  const int4* __restrict__ csrc = nullptr, int64_t ncopy = 0) {
  pdl_wait();
  pdl_trigger();
  // the parent coordinates into the refined array (refine.cpp:16), in the
  // same launch as the boundary pairs (one launch less per level)
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ncopy;
       i += (int64_t)gridDim.x * blockDim.x)
    cdst[i] = __ldcs(csrc + i);
  const int64_t total = (int64_t)nD + nN;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool is_d = i < nD;
    const int64_t j = is_d ? i : i - nD;
    const int32_t* pr = is_d ? dpairs : npairs;
    const int a = pr[2 * j], b = pr[2 * j + 1];
    const int e = find_edge(nes, edge_nodes, nC, a, b);
    if (e < 0) {
      atomicMin(&err->misc, (unsigned long long)i);
      continue;
    }
    const int mid = nC + e;
    (is_d ? dout : nout)[j] = make_int4(a, mid, mid, b);
  }
}

__global__ void k_orient(const double2* __restrict__ coords, int32_t* __restrict__ elements,
                         int nE) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < nE; m += stride) {
    const int a = elements[3 * m], b = elements[3 * m + 1], c = elements[3 * m + 2];
    const double2 pa = __ldg(coords + a), pb = __ldg(coords + b), pc = __ldg(coords + c);
    const double t2 = (pb.x - pa.x) * (pc.y - pa.y) - (pb.y - pa.y) * (pc.x - pa.x);
    if (t2 < 0.0) {
      elements[3 * m + 1] = c;
      elements[3 * m + 2] = b;
    }
  }
}

}  // namespace phfem

using namespace phfem;

PHFEM_API void phfem_mesh_release(phfem_ctx* ctx, phfem_mesh* m) {
  if (!m || !m->owned) return;
  dfree(ctx, m->coords);
  dfree(ctx, m->elements);
  dfree(ctx, m->dirichlet);
  dfree(ctx, m->neumann);
  m->owned = 0;
}

namespace phfem {
// write_mid = false: the midpoint nodes nc..nc+E-1 are left to the fused
// refined-level kernel (refine_topo.cu), which writes them coalesced.
// deferred != nullptr (pipeline): the boundary-pair mismatch goes to that
// error block, checked once at the end of the pipeline — no host sync here
phfem_status red_refine_impl(phfem_ctx* ctx, const phfem_mesh* mesh, const phfem_topology* topo,
                             phfem_mesh* out, bool write_mid, bool defer_elements, phfem_dev_errors* deferred) {
  memset(out, 0, sizeof(*out));
  if (!ctx || !mesh || !topo) return PHFEM_ERR_INVALID_ARGUMENT;
  if (topo->nE != mesh->nE || topo->nC != mesh->nC)
    return set_error(ctx, PHFEM_ERR_MISMATCH, "red_refine: topology does not match mesh");
  const int64_t nC = mesh->nC, nE = mesh->nE, E = topo->E;
  if (nC + E >= (int64_t(1) << 31) || 4 * nE >= (int64_t(1) << 31))
    return set_error(ctx, PHFEM_ERR_INVALID_ARGUMENT, "red_refine: refined mesh too large for int ids");
  out->nC = (int32_t)(nC + E);
  out->nE = (int32_t)(4 * nE);
  out->nD = 2 * mesh->nD;
  out->nN = 2 * mesh->nN;
  out->owned = 1;
  PHFEM_TRY(dalloc(ctx, &out->coords, 2 * (nC + E)));
  PHFEM_TRY(dalloc(ctx, &out->elements, 12 * nE));
  PHFEM_TRY(dalloc(ctx, &out->dirichlet, 4 * (int64_t)mesh->nD));
  PHFEM_TRY(dalloc(ctx, &out->neumann, 4 * (int64_t)mesh->nN));
  const int64_t nb = (int64_t)mesh->nD + mesh->nN;
  // pipeline path: the coordinate copy rides in the boundary-pair launch
  const bool fuse_copy = nb > 0 && deferred && nC > 0 &&
                         (((uintptr_t)out->coords | (uintptr_t)mesh->coords) & 15u) == 0;
  if (nC > 0 && !fuse_copy) PHFEM_TRY(copy_d2d(ctx, out->coords, mesh->coords, sizeof(double) * 2 * nC));
  if (nE > 0 && !defer_elements) {
    PHFEM_LAUNCH(ctx, "k_refine_elements", k_refine_elements<<<grid_for(nE, 256, ctx->num_sms * 16), 256, 0, ctx->stream>>>(
        (const double2*)mesh->coords, mesh->elements, topo->elem_edge, (int)nE, (int)nC,
        (double2*)out->coords, (int4*)out->elements, write_mid ? 1 : 0));
  }
  if (nb > 0 && deferred) {
    const int64_t ncopy = fuse_copy ? (int64_t)nC : 0;  // 16-byte coordinate pairs
    PHFEM_LAUNCH_PDL(ctx, "k_refine_boundary", k_refine_boundary,
        grid_for(std::max<int64_t>(nb, ncopy), 256, ctx->num_sms * 32), 256, 0,
        (const int32_t*)mesh->dirichlet, (int)mesh->nD, (const int32_t*)mesh->neumann, (int)mesh->nN,
        (const int32_t*)topo->node_edge_start, (const int32_t*)topo->edge_nodes, (int)nC, (int4*)out->dirichlet,
        (int4*)out->neumann, deferred, (int4*)out->coords, (const int4*)mesh->coords, ncopy);
  } else if (nb > 0) {
    PHFEM_TRY(errors_reset(ctx));
    PHFEM_LAUNCH(ctx, "k_refine_boundary", k_refine_boundary<<<grid_for(nb, 256, ctx->num_sms * 4), 256, 0, ctx->stream>>>(
        mesh->dirichlet, mesh->nD, mesh->neumann, mesh->nN, topo->node_edge_start,
        topo->edge_nodes, (int)nC, (int4*)out->dirichlet, (int4*)out->neumann, ctx->derr));
    PHFEM_TRY(errors_fetch(ctx));
    if (ctx->herr->misc != ~0ull) {
      phfem_mesh_release(ctx, out);
      return set_error(ctx, PHFEM_ERR_MISMATCH, "red_refine: topology does not match mesh");
    }
  }
  return PHFEM_OK;
}
}  // namespace phfem

PHFEM_API phfem_status phfem_red_refine(phfem_ctx* ctx, const phfem_mesh* mesh,
                                        const phfem_topology* topo, phfem_mesh* out) {
  return red_refine_impl(ctx, mesh, topo, out, true);
}

PHFEM_API phfem_status phfem_orient_ccw(phfem_ctx* ctx, phfem_mesh* mesh) {
  if (!ctx || !mesh) return PHFEM_ERR_INVALID_ARGUMENT;
  if (mesh->nE == 0) return PHFEM_OK;
  PHFEM_LAUNCH(ctx, "k_orient", k_orient<<<grid_for(mesh->nE, 256, ctx->num_sms * 16), 256, 0, ctx->stream>>>(
      (const double2*)mesh->coords, mesh->elements, mesh->nE));
  return PHFEM_OK;
}
