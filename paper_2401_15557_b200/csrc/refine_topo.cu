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

// ---------------------------------------------------------------------------
// Group enumeration: the fine edges whose larger node is mu(e), in canonical
// order (halves by smaller old node, then interior edges by partner e').
struct FineEdge {
  int from, to, tp, lp, tm, lm;
};

__device__ __forceinline__ int rt_group(const RtArgs& a, int e, int2 el, FineEdge fe[6]) {
  const int2 ab = reinterpret_cast<const int2*>(a.edge_nodes)[e];
  const int l = __ldg(a.ltp + e);
  const int tp = el.x, tm = el.y;
  const int l2 = tm >= 0 ? __ldg(a.ltm + e) : 0;
  const int mu = a.nc + e;
  const int ia = ab.x < ab.y ? 0 : 1;  // the half at the smaller old node comes first
  fe[ia] = FineEdge{ab.x, mu, 4 * tp + 1 + (l + 1) % 3, 2, tm >= 0 ? 4 * tm + 1 + (l2 + 2) % 3 : -1, 1};
  fe[1 - ia] = FineEdge{mu, ab.y, 4 * tp + 1 + (l + 2) % 3, 1, tm >= 0 ? 4 * tm + 1 + (l2 + 1) % 3 : -1, 2};
  int pe[4], pk[4], pm[4], ee[2][3];
  int np = 0;
  int q[2], k[2];
  partners_in(a.elem_edge, tp, e, q, k, ee[0]);
#pragma unroll
  for (int t = 0; t < 2; ++t)
    if (q[t] < e) {
      pe[np] = q[t];
      pk[np] = k[t];
      pm[np] = 0;
      ++np;
    }
  if (tm >= 0) {
    partners_in(a.elem_edge, tm, e, q, k, ee[1]);
#pragma unroll
    for (int t = 0; t < 2; ++t)
      if (q[t] < e) {
        pe[np] = q[t];
        pk[np] = k[t];
        pm[np] = 1;
        ++np;
      }
  }
  for (int t = 0; t < np; ++t) {
    int rank = 0;
    for (int u = 0; u < np; ++u) rank += pe[u] < pe[t];
    const int m = pm[t] == 0 ? tp : tm;
    const int kk = pk[t];
    const int* E3 = ee[pm[t]];
    fe[2 + rank] = FineEdge{a.nc + E3[(kk + 1) % 3], a.nc + E3[(kk + 2) % 3], 4 * m, kk, 4 * m + 1 + kk, 0};
  }
  return 2 + np;
}

// counts per parent edge: fine edges, retained fine edges, retained boundary fine edges
__global__ void k_rl_count(RtArgs a, const int32_t* __restrict__ prpos, int32_t* __restrict__ cnt,
                           int32_t* __restrict__ rcnt, int32_t* __restrict__ brcnt) {
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
    if (rcnt) {
      const bool neu = prpos[e] < 0;  // halves of a Neumann edge are Neumann
      rcnt[e] = c - (neu ? 2 : 0);
      brcnt[e] = (el.y < 0 && !neu) ? 2 : 0;
    }
  }
}

struct RlOut {
  int32_t* edge_nodes;
  int32_t* edge_elements;
  int32_t* ltp;
  int32_t* ltm;
  int32_t* interior;
  int32_t* boundary;
  int32_t* elem_edge;
  int32_t* node_edge_start;
  // kFull only
  const double2* fcoords;
  const int32_t* prpos;
  const int32_t* base_r;
  const int32_t* base_br;
  int32_t* rpos;
  int32_t* redges;
  int32_t* row_ptr;
  int32_t* col;
  double* val;
  int L;
};

constexpr int kRlEdges = 128;              // parent edges per CTA
constexpr int kRlFine = 6 * kRlEdges;      // max fine edges per CTA

// One CTA per 128 parent edges.  Fine-edge records are staged in SMEM and
// written back with coalesced stores; in the kFull variant every retained
// fine edge also gets its retained position and its C row, and the block's C
// entries (a contiguous range) are produced entry-parallel.
template <bool kFull>
__global__ void __launch_bounds__(kRlEdges) k_rl_emit(RtArgs a, const int32_t* __restrict__ base_f,
                                                       int total, RlOut o) {
  __shared__ int2 s_en[kRlFine];
  __shared__ int2 s_el[kRlFine];
  __shared__ int32_t s_lt[kRlFine];
  __shared__ int32_t s_rp[kFull ? kRlFine : 1];
  __shared__ int32_t s_rs[kFull ? kRlFine : 1];
  __shared__ int16_t s_ri[kFull ? kRlFine : 1];
  __shared__ double s_len[kFull ? kRlFine : 1];
  __shared__ int16_t s_owner[kFull ? 4 * kRlFine : 1];
  __shared__ int32_t sm[33];
  __shared__ int32_t s_bpre;
  const int tid = threadIdx.x;
  const int64_t e0 = (int64_t)blockIdx.x * kRlEdges;
  const int64_t e = e0 + tid;
  const bool valid = e < a.E;
  const int64_t e_end = e0 + kRlEdges < a.E ? e0 + kRlEdges : a.E;
  int2 el = make_int2(0, 0);
  if (valid) el = reinterpret_cast<const int2*>(a.edge_elements)[e];
  const int isB = (valid && el.y < 0) ? 1 : 0;
  if (tid == 0) {
    int lo = 0, hi = a.nB;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(a.boundary + mid) < e0) lo = mid + 1;
      else hi = mid;
    }
    s_bpre = lo;
  }
  int tot;
  const int bex = block_exclusive_scan(isB, sm, &tot);
  const int F0 = base_f[e0];
  const int nf = base_f[e_end] - F0;
  if (valid) {
    const int bpre = s_bpre + bex;  // parent boundary edges before e
    const int base = base_f[e];
    o.node_edge_start[a.nc + e] = base;
    if (e == a.E - 1) o.node_edge_start[a.nc + a.E] = total;
    FineEdge fe[6];
    const int cnt = rt_group(a, (int)e, el, fe);
    int rbase = 0, brbase = 0;
    bool neu = false;
    if (kFull) {
      rbase = o.base_r[e];
      brbase = o.base_br[e];
      neu = o.prpos[e] < 0;
    }
    const int R0 = kFull ? o.base_r[e0] : 0;
    int rk = 0;
    for (int j = 0; j < cnt; ++j) {
      const int f = base + j;
      const int i = f - F0;
      const FineEdge& x = fe[j];
      s_en[i] = make_int2(x.from, x.to);
      s_el[i] = make_int2(x.tp, x.tm);
      s_lt[i] = x.lp | ((x.tm >= 0 ? x.lm : -1) << 8);
      o.elem_edge[3 * (int64_t)x.tp + x.lp] = f;
      if (x.tm >= 0) o.elem_edge[3 * (int64_t)x.tm + x.lm] = ~f;
      const bool fbnd = j < 2 && isB;
      if (fbnd) o.boundary[2 * bpre + j] = f;
      else o.interior[f - 2 * bpre - (j >= 2 && isB ? 2 : 0)] = f;
      if (kFull) {
        const bool ret = j >= 2 || !neu;
        int rp = -1;
        if (ret) {
          rp = rbase + rk;
          const int bret = brbase + ((fbnd && j == 1) ? 1 : 0) + ((j >= 2 && isB && !neu) ? 2 : 0);
          const int rs = 4 * rp - 2 * bret;
          const double2 pa = __ldg(o.fcoords + x.from), pb = __ldg(o.fcoords + x.to);
          const double dx = pb.x - pa.x, dy = pb.y - pa.y;
          const int jr = rp - R0;
          s_rs[jr] = rs;
          s_ri[jr] = (int16_t)i;
          s_len[jr] = sqrt(dx * dx + dy * dy);  // edge_topology.cpp:183
          o.row_ptr[rp] = rs;
          o.redges[rp] = f;
          if (rp == o.L - 1) o.row_ptr[o.L] = rs + (x.tm >= 0 ? 4 : 2);
          ++rk;
        }
        s_rp[i] = rp;
      }
    }
  }
  __syncthreads();
  for (int i = tid; i < nf; i += kRlEdges) {
    const int f = F0 + i;
    reinterpret_cast<int2*>(o.edge_nodes)[f] = s_en[i];
    reinterpret_cast<int2*>(o.edge_elements)[f] = s_el[i];
    const int lt = s_lt[i];
    o.ltp[f] = lt & 0xff;
    o.ltm[f] = lt >> 8;
    if (kFull) o.rpos[f] = s_rp[i];
  }
  if (kFull) {
    // the block's C entries are one contiguous range [K0, K1): map entry -> row
    // in SMEM, then write entry-parallel (coalesced col / value stores)
    const int R0 = o.base_r[e0], R1 = o.base_r[e_end];
    const int K0 = 4 * R0 - 2 * o.base_br[e0];
    const int K1 = 4 * R1 - 2 * o.base_br[e_end];
    for (int j = tid; j < R1 - R0; j += kRlEdges) {
      const int n = s_el[s_ri[j]].y >= 0 ? 4 : 2;
      const int k0 = s_rs[j] - K0;
      for (int q = 0; q < n; ++q) s_owner[k0 + q] = (int16_t)j;
    }
    __syncthreads();
    for (int k = tid; k < K1 - K0; k += kRlEdges) {
      const int j = s_owner[k];
      const int q = k + K0 - s_rs[j];
      const int i = s_ri[j];
      const int2 tt = s_el[i];
      const int lt = s_lt[i];
      const int l = q < 2 ? (lt & 0xff) : (lt >> 8);
      const int c = (q & 1) == 0 ? (l == 0 ? 1 : 0) : (l == 2 ? 1 : 2);  // q-th of {0,1,2} \ {l}
      const double len = s_len[j];
      o.col[K0 + k] = 3 * (q < 2 ? tt.x : tt.y) + c;
      __stcs(o.val + K0 + k, q < 2 ? len * 0.5 : -len * 0.5);  // assembly.cpp:160 / :164
    }
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
  PHFEM_LAUNCH(ctx, "k_rl_count", k_rl_count<<<grid_for(E, 256, ctx->num_sms * 16), 256, 0, ctx->stream>>>(
      a, nullptr, base, nullptr, nullptr));
  PHFEM_CUDA(ctx, cudaMemsetAsync(base + E, 0, sizeof(int32_t), ctx->stream));
  PHFEM_TRY(scan_exclusive_i32(ctx, base, base, E + 1, nullptr));
  RlOut o;
  memset(&o, 0, sizeof o);
  o.edge_nodes = out->edge_nodes;
  o.edge_elements = out->edge_elements;
  o.ltp = out->local_in_tplus;
  o.ltm = out->local_in_tminus;
  o.interior = out->interior_edges;
  o.boundary = out->boundary_edges;
  o.elem_edge = out->elem_edge;
  o.node_edge_start = out->node_edge_start;
  PHFEM_LAUNCH(ctx, "k_rl_emit", k_rl_emit<false><<<(unsigned)((E + kRlEdges - 1) / kRlEdges), kRlEdges, 0,
                                                    ctx->stream>>>(a, base, (int)Ef, o));
  dfree(ctx, base);
  out->E = (int32_t)Ef;
  out->n_boundary = (int32_t)nBf;
  out->n_interior = (int32_t)(Ef - nBf);
  return PHFEM_OK;
}

namespace phfem {
// defined in classify.cu
phfem_status classify_lists(phfem_ctx* ctx, const phfem_topology* topo, const phfem_mesh* mesh,
                            phfem_classification* out, bool with_retained);
}  // namespace phfem

PHFEM_API phfem_status phfem_refine_level(phfem_ctx* ctx, const phfem_mesh* parent,
                                          const phfem_topology* ptopo,
                                          const phfem_classification* pcls,
                                          const phfem_mesh* fine, phfem_topology* topo,
                                          phfem_classification* cls, phfem_csr* C) {
  memset(topo, 0, sizeof(*topo));
  memset(cls, 0, sizeof(*cls));
  memset(C, 0, sizeof(*C));
  if (!ctx || !parent || !ptopo || !pcls || !fine) return PHFEM_ERR_INVALID_ARGUMENT;
  if (ptopo->nE != parent->nE || ptopo->nC != parent->nC || fine->nE != 4 * parent->nE ||
      fine->nC != parent->nC + ptopo->E || pcls->E != ptopo->E ||
      fine->nD != 2 * parent->nD || fine->nN != 2 * parent->nN)
    return set_error(ctx, PHFEM_ERR_MISMATCH, "refine_level: meshes do not match the topology");
  const int64_t E = ptopo->E, nc = parent->nC;
  const int64_t Ef = 2 * E + 3 * (int64_t)parent->nE;
  if (Ef >= (int64_t(1) << 31) || 4 * Ef >= (int64_t(1) << 31))
    return set_error(ctx, PHFEM_ERR_INVALID_ARGUMENT, "refine_level: mesh too large for int ids");
  const int64_t nneu_p = E - pcls->L;                   // Neumann parent edges
  const int64_t nBf = 2 * (int64_t)ptopo->n_boundary;
  const int64_t L = Ef - 2 * nneu_p;                    // their halves are the fine Neumann edges
  const int64_t BR = 2 * ((int64_t)ptopo->n_boundary - nneu_p);
  topo->nC = fine->nC;
  topo->nE = fine->nE;
  PHFEM_TRY(dalloc(ctx, &topo->edge_nodes, 2 * Ef));
  PHFEM_TRY(dalloc(ctx, &topo->edge_elements, 2 * Ef));
  PHFEM_TRY(dalloc(ctx, &topo->local_in_tplus, Ef));
  PHFEM_TRY(dalloc(ctx, &topo->local_in_tminus, Ef));
  PHFEM_TRY(dalloc(ctx, &topo->interior_edges, Ef - nBf));
  PHFEM_TRY(dalloc(ctx, &topo->boundary_edges, nBf));
  PHFEM_TRY(dalloc(ctx, &topo->elem_edge, 3 * (int64_t)fine->nE));
  PHFEM_TRY(dalloc(ctx, &topo->node_edge_start, (int64_t)fine->nC + 1));
  topo->E = (int32_t)Ef;
  topo->n_boundary = (int32_t)nBf;
  topo->n_interior = (int32_t)(Ef - nBf);
  PHFEM_TRY(dalloc(ctx, &cls->retained_pos, Ef));
  PHFEM_TRY(dalloc(ctx, &cls->retained_edges, L));
  C->rows = (int32_t)L;
  C->cols = 3 * fine->nE;
  C->nnz = 4 * L - 2 * BR;
  PHFEM_TRY(dalloc(ctx, &C->row_ptr, L + 1));
  PHFEM_TRY(dalloc(ctx, &C->col_idx, C->nnz));
  PHFEM_TRY(dalloc(ctx, &C->values, C->nnz));
  PHFEM_CUDA(ctx, cudaMemsetAsync(topo->node_edge_start, 0, sizeof(int32_t) * (nc + 1), ctx->stream));
  if (L == 0) PHFEM_CUDA(ctx, cudaMemsetAsync(C->row_ptr, 0, sizeof(int32_t), ctx->stream));
  if (E > 0) {
    RtArgs a{ptopo->edge_nodes, ptopo->edge_elements, ptopo->local_in_tplus, ptopo->local_in_tminus,
             ptopo->elem_edge, ptopo->boundary_edges, ptopo->n_boundary, (int)E, (int)nc};
    int32_t *bf = nullptr, *br = nullptr, *bb = nullptr;
    PHFEM_TRY(dalloc(ctx, &bf, E + 1));
    PHFEM_TRY(dalloc(ctx, &br, E + 1));
    PHFEM_TRY(dalloc(ctx, &bb, E + 1));
    PHFEM_LAUNCH(ctx, "k_rl_count", k_rl_count<<<grid_for(E, 256, ctx->num_sms * 16), 256, 0, ctx->stream>>>(
        a, pcls->retained_pos, bf, br, bb));
    PHFEM_CUDA(ctx, cudaMemsetAsync(bf + E, 0, sizeof(int32_t), ctx->stream));
    PHFEM_CUDA(ctx, cudaMemsetAsync(br + E, 0, sizeof(int32_t), ctx->stream));
    PHFEM_CUDA(ctx, cudaMemsetAsync(bb + E, 0, sizeof(int32_t), ctx->stream));
    PHFEM_TRY(scan_exclusive_i32(ctx, bf, bf, E + 1, nullptr));
    PHFEM_TRY(scan_exclusive_i32(ctx, br, br, E + 1, nullptr));
    PHFEM_TRY(scan_exclusive_i32(ctx, bb, bb, E + 1, nullptr));
    RlOut o;
    memset(&o, 0, sizeof o);
    o.edge_nodes = topo->edge_nodes;
    o.edge_elements = topo->edge_elements;
    o.ltp = topo->local_in_tplus;
    o.ltm = topo->local_in_tminus;
    o.interior = topo->interior_edges;
    o.boundary = topo->boundary_edges;
    o.elem_edge = topo->elem_edge;
    o.node_edge_start = topo->node_edge_start;
    o.fcoords = (const double2*)fine->coords;
    o.prpos = pcls->retained_pos;
    o.base_r = br;
    o.base_br = bb;
    o.rpos = cls->retained_pos;
    o.redges = cls->retained_edges;
    o.row_ptr = C->row_ptr;
    o.col = C->col_idx;
    o.val = C->values;
    o.L = (int)L;
    PHFEM_LAUNCH(ctx, "k_rl_emit_full", k_rl_emit<true><<<(unsigned)((E + kRlEdges - 1) / kRlEdges), kRlEdges, 0,
                                                         ctx->stream>>>(a, bf, (int)Ef, o));
    dfree(ctx, bf);
    dfree(ctx, br);
    dfree(ctx, bb);
  }
  // boundary lists -> ids, Neumann bitmap, block prefixes (retained arrays already written)
  phfem_status st = classify_lists(ctx, topo, fine, cls, false);
  if (st != PHFEM_OK) return st;
  if (cls->L != L)
    return set_error(ctx, PHFEM_ERR_MISMATCH, "refine_level: classification does not match the parent's");
  return PHFEM_OK;
}
