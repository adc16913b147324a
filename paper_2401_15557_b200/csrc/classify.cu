// classify.cu — classify_edges on sm_100a.
//
// Reference: proj/src/edge_topology.cpp:145-177.  Boundary pairs are resolved
// through the max-node grouping table written by build_topology (edges of one
// max node are a contiguous id range sorted by min node -> binary search),
// the Neumann set becomes a bitmap, and retained_pos / retained_edges come
// from per-1024-edge block prefixes of that bitmap (the reference's E-length
// flag loop, :166-174).  Per-block boundary prefixes (from the ascending
// boundary list) are kept for the CSR row pointers of C.
#include <algorithm>

#include "common.cuh"

namespace phfem {

constexpr int kEdgeBlock = 1024;

__global__ void k_cls_pairs(const int32_t* __restrict__ dir_pairs, int nD,
                            const int32_t* __restrict__ neu_pairs, int nN,
                            const int32_t* __restrict__ nes, const int32_t* __restrict__ edge_nodes,
                            const int32_t* __restrict__ edge_elements, int nC,
                            int32_t* __restrict__ dir_ids, int32_t* __restrict__ neu_ids,
                            uint32_t* __restrict__ bits, phfem_dev_errors* err) {
  pdl_wait();
  pdl_trigger();
  const int64_t total = (int64_t)nD + nN;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool is_d = i < nD;
    const int64_t j = is_d ? i : i - nD;
    const int32_t* pr = is_d ? dir_pairs : neu_pairs;
    const int a = pr[2 * j], b = pr[2 * j + 1];
    const int e = find_edge(nes, edge_nodes, nC, a, b);
    if (e < 0) {
      atomicMin(&err->classify, ((unsigned long long)i << 2) | 0ull);
      continue;
    }
    if (edge_elements[2 * e + 1] >= 0) {
      atomicMin(&err->classify, ((unsigned long long)i << 2) | 1ull);
      continue;
    }
    if (is_d) {
      dir_ids[j] = e;
    } else {
      neu_ids[j] = e;
      const uint32_t bit = 1u << (e & 31);
      const uint32_t old = atomicOr(&bits[e >> 5], bit);
      if (old & bit) err->counters[5] = 1;  // duplicate Neumann pair
    }
  }
}

// One thread per 1024-edge block: Neumann count (bitmap popcount) and boundary
// count (two lower_bounds into the ascending boundary list, whose ids start at
// `base`: 0, or the global id of a rank part's first edge).
__global__ void k_cls_block_counts(const uint32_t* __restrict__ bits,
                                   const int32_t* __restrict__ boundary, int nB, int E, int nblk, int base,
                                   int32_t* __restrict__ cnt_bnd, int32_t* __restrict__ cnt_neu) {
  pdl_wait();
  pdl_trigger();
  const int blk = blockIdx.x * blockDim.x + threadIdx.x;
  if (blk > nblk) return;
  if (blk == nblk) {
    cnt_bnd[blk] = 0;
    cnt_neu[blk] = 0;
    return;
  }
  const int nwords = (E + 31) >> 5;
  int nn = 0;
  for (int w = blk * 32; w < min(nwords, blk * 32 + 32); ++w) nn += __popc(bits[w]);
  auto lower = [&](int key) {
    int l = 0, r = nB;
    while (l < r) {
      const int mid = (l + r) >> 1;
      if (boundary[mid] < key) l = mid + 1;
      else r = mid;
    }
    return l;
  };
  cnt_bnd[blk] = lower(base + min(E, (blk + 1) * kEdgeBlock)) - lower(base + blk * kEdgeBlock);
  cnt_neu[blk] = nn;
}

// CTA of 256 threads per block of 1024 edges; thread t owns 4 consecutive
// edges, all inside bitmap word t/8.
// r_off / e_off: the rank's first retained row / first global edge id
// (distributed final level with the offsets known up front; 0 otherwise)
__global__ void __launch_bounds__(256) k_cls_retained(const uint32_t* __restrict__ bits,
                                                      const int32_t* __restrict__ pre_neu,
                                                      int E, int32_t* __restrict__ rpos,
                                                      int32_t* __restrict__ redges, int r_off, int e_off) {
  pdl_wait();
  pdl_trigger();
  __shared__ int32_t wpre[32];
  const int blk = blockIdx.x;
  const int nwords = (E + 31) >> 5;
  if (threadIdx.x < 32) {
    const int64_t wi = (int64_t)blk * 32 + threadIdx.x;
    const int c = wi < nwords ? __popc(bits[wi]) : 0;
    wpre[threadIdx.x] = warp_inclusive_scan(c) - c;
  }
  __syncthreads();
  const int t = threadIdx.x;
  const int64_t e0 = (int64_t)blk * kEdgeBlock + 4 * t;
  if (e0 >= E) return;
  const int w = t >> 3;
  const int64_t wi = (int64_t)blk * 32 + w;
  const uint32_t word = bits[wi];
  const int bit0 = (4 * t) & 31;
  int before = pre_neu[blk] + wpre[w] + __popc(word & ((1u << bit0) - 1u));
  int r[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const bool neu = (word >> (bit0 + q)) & 1u;
    r[q] = neu ? -1 : (int)(e0 + q) - before;
    before += neu;
  }
  int g[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) g[q] = r[q] < 0 ? -1 : r[q] + r_off;
  if (e0 + 3 < E) {
    *reinterpret_cast<int4*>(rpos + e0) = make_int4(g[0], g[1], g[2], g[3]);
  } else {
    for (int q = 0; q < 4 && e0 + q < E; ++q) rpos[e0 + q] = g[q];
  }
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (r[q] >= 0 && e0 + q < E) redges[r[q]] = (int)(e0 + q) + e_off;
}

}  // namespace phfem

using namespace phfem;

PHFEM_API void phfem_classification_release(phfem_ctx* ctx, phfem_classification* c) {
  if (!c) return;
  dfree(ctx, c->dirichlet_edge_ids);
  dfree(ctx, c->neumann_edge_ids);
  dfree(ctx, c->retained_edges);
  dfree(ctx, c->retained_pos);
  dfree(ctx, c->neumann_bits);
  dfree(ctx, c->block_prefix);
  c->L = 0;
}

namespace phfem {
// per-1024-edge-block (boundary, Neumann) prefixes from the Neumann bitmap and
// the ascending boundary list; with_retained also retained_pos / _edges
static phfem_status block_prefix_and_retained(phfem_ctx* ctx, const phfem_topology* topo,
                                              phfem_classification* out, int nblk,
                                              bool with_retained, int bnd_base = 0, int r_off = 0,
                                              int e_off = 0) {
  const int E = topo->E;
  int32_t* pre_bnd = out->block_prefix;
  int32_t* pre_neu = out->block_prefix + nblk + 1;
  PHFEM_LAUNCH_PDL(ctx, "k_cls_block_counts", k_cls_block_counts, grid_for(nblk + 1, 256, 1 << 20), 256, 0,
      out->neumann_bits, topo->boundary_edges, topo->n_boundary, E, nblk, bnd_base, pre_bnd, pre_neu);
  {
    const int32_t* in[2] = {pre_bnd, pre_neu};
    int32_t* io[2] = {pre_bnd, pre_neu};
    PHFEM_TRY(scan_exclusive_i32_set(ctx, 2, in, io, nblk + 1, nullptr));
  }
  if (nblk > 0 && with_retained) {
    PHFEM_LAUNCH_PDL(ctx, "k_cls_retained", k_cls_retained, nblk, 256, 0, out->neumann_bits, pre_neu, E,
                     out->retained_pos, out->retained_edges, r_off, e_off);
  }
  return PHFEM_OK;
}

// Boundary pairs -> ids, the Neumann bitmap and the per-block prefixes; with
// with_retained also retained_pos / retained_edges (else the caller wrote them
// and allocated out->retained_pos / retained_edges already).
phfem_status classify_lists(phfem_ctx* ctx, const phfem_topology* topo, const phfem_mesh* mesh,
                            phfem_classification* out, bool with_retained) {
  const int E = topo->E, nD = mesh->nD, nN = mesh->nN;
  out->nD = nD;
  out->nN = nN;
  out->E = E;
  const int nblk = (E + kEdgeBlock - 1) / kEdgeBlock;
  const int nwords = (E + 31) / 32;
  PHFEM_TRY(dalloc(ctx, &out->dirichlet_edge_ids, nD));
  PHFEM_TRY(dalloc(ctx, &out->neumann_edge_ids, nN));
  if (with_retained) {
    PHFEM_TRY(dalloc(ctx, &out->retained_pos, E));
    PHFEM_TRY(dalloc(ctx, &out->retained_edges, E));
  }
  PHFEM_TRY(dalloc(ctx, &out->neumann_bits, nwords));
  PHFEM_TRY(dalloc(ctx, &out->block_prefix, 2 * ((int64_t)nblk + 1)));
  PHFEM_CUDA(ctx, cudaMemsetAsync(out->neumann_bits, 0, sizeof(uint32_t) * std::max(nwords, 1),
                                  ctx->stream));
  PHFEM_TRY(errors_reset(ctx));
  if ((int64_t)nD + nN > 0) {
    PHFEM_LAUNCH_PDL(ctx, "k_cls_pairs", k_cls_pairs, grid_for((int64_t)nD + nN, 256, ctx->num_sms * 4), 256, 0,
        mesh->dirichlet, nD, mesh->neumann, nN, topo->node_edge_start, topo->edge_nodes,
        topo->edge_elements, topo->nC, out->dirichlet_edge_ids, out->neumann_edge_ids,
        out->neumann_bits, ctx->derr);
  }
  PHFEM_TRY(block_prefix_and_retained(ctx, topo, out, nblk, with_retained));
  // total Neumann count rides back with the error words (one sync)
  PHFEM_CUDA(ctx, cudaMemcpyAsync(&ctx->derr->counters[8], out->block_prefix + nblk + 1 + nblk, sizeof(int32_t),
                                  cudaMemcpyDeviceToDevice, ctx->stream));
  PHFEM_TRY(errors_fetch(ctx));
  const uint64_t ce = ctx->herr->classify;
  if (ce != ~0ull) {
    const int64_t pos = (int64_t)(ce >> 2);
    const bool interior = ce & 1ull;
    const bool is_d = pos < nD;
    const int32_t* src = is_d ? mesh->dirichlet + 2 * pos : mesh->neumann + 2 * (pos - nD);
    int32_t pr[2] = {0, 0};
    PHFEM_CUDA(ctx, cudaMemcpyAsync(pr, src, sizeof pr, cudaMemcpyDeviceToHost, ctx->stream));
    PHFEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    phfem_classification_release(ctx, out);
    return set_error(ctx, interior ? PHFEM_ERR_INTERIOR_BOUNDARY : PHFEM_ERR_NOT_AN_EDGE,
                     interior ? "%s pair (%d,%d) resolves to an interior edge"
                              : "%s pair (%d,%d) is not an edge",
                     is_d ? "dirichlet" : "neumann", pr[0] + 1, pr[1] + 1);
  }
  out->L = E - (int32_t)(ctx->herr->counters[8] & 0xffffffffu);
  out->flags = ctx->herr->counters[5] ? PHFEM_CLS_DUP_NEUMANN : 0;
  return PHFEM_OK;
}
}  // namespace phfem

namespace phfem {
// Distributed ranks (dist.cu): the Neumann bitmap and the owned id lists are
// set; block prefixes, retained_pos / retained_edges and L follow.
phfem_status classify_lists_from_bits(phfem_ctx* ctx, const phfem_topology* topo,
                                      phfem_classification* out, int bnd_base, int r_off, int e_off) {
  const int E = topo->E;
  const int nblk = (E + kEdgeBlock - 1) / kEdgeBlock;
  PHFEM_TRY(dalloc(ctx, &out->retained_pos, E));
  PHFEM_TRY(dalloc(ctx, &out->retained_edges, E));
  PHFEM_TRY(dalloc(ctx, &out->block_prefix, 2 * ((int64_t)nblk + 1)));
  PHFEM_TRY(block_prefix_and_retained(ctx, topo, out, nblk, true, bnd_base, r_off, e_off));
  int32_t nneu = 0;
  PHFEM_CUDA(ctx, cudaMemcpyAsync(&nneu, out->block_prefix + nblk + 1 + nblk, sizeof(int32_t),
                                  cudaMemcpyDeviceToHost, ctx->stream));
  PHFEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  out->L = E - nneu;
  return PHFEM_OK;
}
}  // namespace phfem

PHFEM_API phfem_status phfem_classify_edges(phfem_ctx* ctx, const phfem_topology* topo,
                                            const phfem_mesh* mesh, phfem_classification* out) {
  memset(out, 0, sizeof(*out));
  if (!ctx || !topo || !mesh) return PHFEM_ERR_INVALID_ARGUMENT;
  return classify_lists(ctx, topo, mesh, out, true);
}
