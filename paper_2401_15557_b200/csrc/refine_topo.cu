// refine_topo.cu — topology of the red-refined mesh straight from the parent
// topology, no sort.
//
// Result is bit-identical to build_topology(red_refine(M)) (reference
// edge_topology.cpp:52-143 applied to refine.cpp:7-53's output):
//  * every fine edge has a midpoint node mu(e) = nc + e as its larger node, so
//    the canonical (max, min) order groups fine edges by parent edge e;
//  * group e = [half at min(a,b), half at max(a,b), then the interior edges
//    mu(e')-mu(e) for the e' < e that share a parent element with e, by e'];
//  * halves of e = (a,b): a->mu in child 4tp+1+(l+1)%3 (local 2) / child
//    4tm+1+(l'+2)%3 (local 1); mu->b in 4tp+1+(l+2)%3 (local 1) / 4tm+1+(l'+1)%3
//    (local 2); interior edge opposite M_k of parent m: M_{k+1}->M_{k+2},
//    t_plus = 4m (local k), t_minus = 4m+1+k (local 0).
// (Derived from the child layout refine.cpp:33-36 and the emission order
// edge_topology.cpp:61-68; tests/test_gpu_parity.py checks it against the
// oracle's sort-based build_topology.)
//
// Two streaming passes over parent edges: count (group sizes) -> scan -> emit.
#include "common.cuh"

namespace phfem {

struct RtArgs {
  const int32_t* edge_nodes;     // parent
  const int32_t* edge_elements;  // parent
  const int32_t* ltp;            // parent
  const int32_t* ltm;            // parent
  const int32_t* elem_edge;      // parent
  const int32_t* boundary;       // parent ascending boundary list
  int nB;
  int E;
  int nc;
};

__device__ __forceinline__ int abs_edge(int s) { return s >= 0 ? s : ~s; }

// partners of e inside parent element m (its other two edges), with the local
// index of the third edge (the M_k the interior fine edge is opposite to)
__device__ __forceinline__ void partners_in(const int32_t* __restrict__ elem_edge, int m, int e,
                                            int pe[2], int pk[2], int ee[3]) {
  ee[0] = abs_edge(__ldg(elem_edge + 3 * (int64_t)m));
  ee[1] = abs_edge(__ldg(elem_edge + 3 * (int64_t)m + 1));
  ee[2] = abs_edge(__ldg(elem_edge + 3 * (int64_t)m + 2));
  const int i = ee[0] == e ? 0 : (ee[1] == e ? 1 : 2);
  const int j1 = (i + 1) % 3, j2 = (i + 2) % 3;
  pe[0] = ee[j1];
  pk[0] = 3 - i - j1;
  pe[1] = ee[j2];
  pk[1] = 3 - i - j2;
}

__global__ void k_rt_count(RtArgs a, int32_t* __restrict__ cnt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < a.E;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int2 el = reinterpret_cast<const int2*>(a.edge_elements)[e];
    int c = 2;
    int pe[2], pk[2], ee[3];
    partners_in(a.elem_edge, el.x, (int)e, pe, pk, ee);
    c += (pe[0] < e) + (pe[1] < e);
    if (el.y >= 0) {
      partners_in(a.elem_edge, el.y, (int)e, pe, pk, ee);
      c += (pe[0] < e) + (pe[1] < e);
    }
    cnt[e] = c;
  }
}

struct RtOut {
  int32_t* edge_nodes;
  int32_t* edge_elements;
  int32_t* ltp;
  int32_t* ltm;
  int32_t* interior;
  int32_t* boundary;
  int32_t* elem_edge;
  int32_t* node_edge_start;
};

__device__ __forceinline__ void rt_write(const RtOut& o, int f, int from, int to, int tp, int lp,
                                         int tm, int lm) {
  reinterpret_cast<int2*>(o.edge_nodes)[f] = make_int2(from, to);
  reinterpret_cast<int2*>(o.edge_elements)[f] = make_int2(tp, tm);
  o.ltp[f] = lp;
  o.ltm[f] = tm >= 0 ? lm : -1;
  o.elem_edge[3 * (int64_t)tp + lp] = f;
  if (tm >= 0) o.elem_edge[3 * (int64_t)tm + lm] = ~f;
}

// 256 parent edges per CTA; boundary prefix = lower_bound(parent boundary
// list, block start) + in-block scan.
__global__ void __launch_bounds__(256) k_rt_emit(RtArgs a, const int32_t* __restrict__ base_of,
                                                 int total, RtOut o) {
  __shared__ int32_t sm[33];
  __shared__ int32_t s_bpre;
  const int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x;
  const bool valid = e < a.E;
  int2 el = make_int2(0, 0);
  if (valid) el = reinterpret_cast<const int2*>(a.edge_elements)[e];
  const int isB = (valid && el.y < 0) ? 1 : 0;
  if (threadIdx.x == 0) {
    const int key = blockIdx.x * 256;
    int lo = 0, hi = a.nB;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(a.boundary + mid) < key) lo = mid + 1;
      else hi = mid;
    }
    s_bpre = lo;
  }
  int tot;
  const int bex = block_exclusive_scan(isB, sm, &tot);
  if (!valid) return;
  const int bpre = s_bpre + bex;  // parent boundary edges before e
  const int base = base_of[e];
  const int mu = a.nc + (int)e;
  o.node_edge_start[mu] = base;
  if (e == a.E - 1) o.node_edge_start[a.nc + a.E] = total;

  const int2 ab = reinterpret_cast<const int2*>(a.edge_nodes)[e];
  const int l = __ldg(a.ltp + e);
  const int tp = el.x, tm = el.y;
  const int l2 = tm >= 0 ? __ldg(a.ltm + e) : 0;
  // halves
  const int fa = ab.x < ab.y ? base : base + 1;
  const int fb = ab.x < ab.y ? base + 1 : base;
  rt_write(o, fa, ab.x, mu, 4 * tp + 1 + (l + 1) % 3, 2, tm >= 0 ? 4 * tm + 1 + (l2 + 2) % 3 : -1, 1);
  rt_write(o, fb, mu, ab.y, 4 * tp + 1 + (l + 2) % 3, 1, tm >= 0 ? 4 * tm + 1 + (l2 + 1) % 3 : -1, 2);
  if (isB) {
    o.boundary[2 * bpre] = base;
    o.boundary[2 * bpre + 1] = base + 1;
  } else {
    o.interior[base - 2 * bpre] = base;
    o.interior[base + 1 - 2 * bpre] = base + 1;
  }
  // interior fine edges mu(e')-mu(e), e' < e, ascending e'
  int pe[4], pk[4], pm[4], ee[2][3];
  int np = 0;
  {
    int q[2], k[2];
    partners_in(a.elem_edge, tp, (int)e, q, k, ee[0]);
    for (int t = 0; t < 2; ++t)
      if (q[t] < e) {
        pe[np] = q[t];
        pk[np] = k[t];
        pm[np] = 0;
        ++np;
      }
    if (tm >= 0) {
      partners_in(a.elem_edge, tm, (int)e, q, k, ee[1]);
      for (int t = 0; t < 2; ++t)
        if (q[t] < e) {
          pe[np] = q[t];
          pk[np] = k[t];
          pm[np] = 1;
          ++np;
        }
    }
  }
  const int ipos0 = base + 2 - 2 * bpre - (isB ? 2 : 0);  // f - #fine boundary edges before f
  for (int t = 0; t < np; ++t) {
    int rank = 0;
    for (int u = 0; u < np; ++u) rank += pe[u] < pe[t];
    const int f = base + 2 + rank;
    const int m = pm[t] == 0 ? tp : tm;
    const int kk = pk[t];
    const int* E3 = ee[pm[t]];
    rt_write(o, f, a.nc + E3[(kk + 1) % 3], a.nc + E3[(kk + 2) % 3], 4 * m, kk, 4 * m + 1 + kk, 0);
    o.interior[ipos0 + rank] = f;
  }
}

}  // namespace phfem

using namespace phfem;

PHFEM_API phfem_status phfem_refine_topology(phfem_ctx* ctx, const phfem_mesh* parent,
                                             const phfem_topology* ptopo, const phfem_mesh* fine,
                                             phfem_topology* out) {
  memset(out, 0, sizeof(*out));
  if (!ctx || !parent || !ptopo || !fine) return PHFEM_ERR_INVALID_ARGUMENT;
  if (ptopo->nE != parent->nE || ptopo->nC != parent->nC || fine->nE != 4 * parent->nE ||
      fine->nC != parent->nC + ptopo->E)
    return set_error(ctx, PHFEM_ERR_MISMATCH, "refine_topology: meshes do not match the topology");
  const int64_t E = ptopo->E, nc = parent->nC;
  // exact count: two halves per parent edge + three interior edges per parent element
  const int64_t Ef_cap = 2 * E + 3 * (int64_t)parent->nE;
  if (Ef_cap >= (int64_t(1) << 31))
    return set_error(ctx, PHFEM_ERR_INVALID_ARGUMENT, "refine_topology: mesh too large for int ids");
  out->nC = fine->nC;
  out->nE = fine->nE;
  const int64_t Ef = Ef_cap;  // exact: every half (2 per parent edge) + 3 interior per parent element
  const int64_t nBf = 2 * (int64_t)ptopo->n_boundary;
  PHFEM_TRY(dalloc(ctx, &out->edge_nodes, 2 * Ef));
  PHFEM_TRY(dalloc(ctx, &out->edge_elements, 2 * Ef));
  PHFEM_TRY(dalloc(ctx, &out->local_in_tplus, Ef));
  PHFEM_TRY(dalloc(ctx, &out->local_in_tminus, Ef));
  PHFEM_TRY(dalloc(ctx, &out->interior_edges, Ef - nBf));
  PHFEM_TRY(dalloc(ctx, &out->boundary_edges, nBf));
  PHFEM_TRY(dalloc(ctx, &out->elem_edge, 3 * (int64_t)fine->nE));
  PHFEM_TRY(dalloc(ctx, &out->node_edge_start, (int64_t)fine->nC + 1));
  PHFEM_CUDA(ctx, cudaMemsetAsync(out->node_edge_start, 0, sizeof(int32_t) * (nc + 1), ctx->stream));
  if (E == 0) return PHFEM_OK;
  RtArgs a{ptopo->edge_nodes, ptopo->edge_elements, ptopo->local_in_tplus, ptopo->local_in_tminus,
           ptopo->elem_edge, ptopo->boundary_edges, ptopo->n_boundary, (int)E, (int)nc};
  int32_t* base = nullptr;
  PHFEM_TRY(dalloc(ctx, &base, E + 1));
  PHFEM_LAUNCH(ctx, "k_rt_count", k_rt_count<<<grid_for(E, 256, ctx->num_sms * 16), 256, 0, ctx->stream>>>(a, base));
  PHFEM_CUDA(ctx, cudaMemsetAsync(base + E, 0, sizeof(int32_t), ctx->stream));
  PHFEM_TRY(scan_exclusive_i32(ctx, base, base, E + 1, nullptr));
  RtOut o{out->edge_nodes, out->edge_elements, out->local_in_tplus, out->local_in_tminus,
          out->interior_edges, out->boundary_edges, out->elem_edge, out->node_edge_start};
  PHFEM_LAUNCH(ctx, "k_rt_emit", k_rt_emit<<<(unsigned)((E + 255) / 256), 256, 0, ctx->stream>>>(a, base, (int)Ef, o));
  dfree(ctx, base);
  out->E = (int32_t)Ef;
  out->n_boundary = (int32_t)nBf;
  out->n_interior = (int32_t)(Ef - nBf);
  return PHFEM_OK;
}
