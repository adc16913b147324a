// pipeline.cu — the fused edge-generation -> red-refinement -> assembly step
// (the bench workload) and its host-buffer (drop-in, e2e) variant.
//
// Reference composition: the refinement chain mesh = red_refine(mesh,
// build_topology(mesh)) (tools/main.cpp:159,394; acceptance.cpp:70), then
// build_topology + classify_edges + assemble_operators + the elliptic load
// b + LN (elliptic.cpp:53-56) and the Dirichlet vector.
#include <algorithm>
#include <chrono>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace phfem {

// PHFEM_TRACE=1: synchronising per-phase wall-clock trace on stderr (debug only)
struct Trace {
  bool on;
  phfem_ctx* ctx;
  std::chrono::steady_clock::time_point t0, last;
  explicit Trace(phfem_ctx* c) : on(getenv("PHFEM_TRACE") != nullptr), ctx(c) {
    t0 = last = std::chrono::steady_clock::now();
  }
  void operator()(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(ctx->stream);
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[phfem] %-28s %9.3f ms (t=%9.3f)\n", what,
            std::chrono::duration<double, std::milli>(now - last).count(),
            std::chrono::duration<double, std::milli>(now - t0).count());
    last = now;
  }
};

static phfem_status pipeline_impl(phfem_ctx* ctx, phfem_mesh cur, int levels,
                                  const phfem_coeffs* c, const phfem_field* f,
                                  const phfem_field* g, const phfem_field* uD, double t, int flags,
                                  phfem_pipeline_out* out) {
  // edge generation on the input mesh (sort-based); every refined mesh gets its
  // topology from the parent's (no sort) unless the generic path is forced
  Trace tr(ctx);
  tr("start");
  // red_refine's boundary-pair checks of every level land in dderr, read once
  // with the pipeline's final error fetch (one host sync less per level)
  PHFEM_CUDA(ctx, cudaMemsetAsync(ctx->dderr, 0xff, sizeof(phfem_dev_errors), ctx->stream));
  phfem_topology topo;
  bool have_cls_C = false;
  // the last level's parent mesh stays alive until the element pass: its
  // elements and nodes let k_volume rebuild the children's vertices (3
  // parent gathers per 4 children, VolArgs::parents); PHFEM_VOL_PARENTS=0
  // reads the refined mesh instead
  struct ParentKeep {
    phfem_ctx* ctx;
    phfem_mesh m;
    bool live = false;
    ~ParentKeep() {
      if (live) phfem_mesh_release(ctx, &m);
    }
  } parent{ctx, {}};
  const char* pv = getenv("PHFEM_VOL_PARENTS");
  const bool vol_parents = !(pv && pv[0] == '0');
  phfem_status st;
  if (levels == 0) {  // the given mesh is the final one: classification + C fused into its edge pass
    st = build_topology_fused(ctx, &cur, &topo, &out->cls, &out->C);
    have_cls_C = st == PHFEM_OK;
  } else {
    st = phfem_build_topology(ctx, &cur, &topo);
  }
  tr("build_topology");
  if (st != PHFEM_OK) {
    phfem_mesh_release(ctx, &cur);
    return st;
  }
  for (int l = 0; l < levels; ++l) {
    const bool last_fused = (l == levels - 1) && !(flags & PHFEM_PIPE_GENERIC_EG);
    phfem_classification pcls;
    memset(&pcls, 0, sizeof pcls);
    if (last_fused) st = phfem_classify_edges(ctx, &topo, &cur, &pcls);
    tr("classify parent");
    phfem_mesh next;
    memset(&next, 0, sizeof next);
    // the sort-free paths write the midpoint nodes themselves (coalesced)
    const bool generic = (flags & PHFEM_PIPE_GENERIC_EG) != 0;
    // sort-free levels: children rows + fine elem_edge come from the level pass
    if (st == PHFEM_OK) st = red_refine_impl(ctx, &cur, &topo, &next, generic, !generic, ctx->dderr);
    double* mid = next.coords;  // the level kernels write nodes nc..nc+E-1
    tr("red_refine");
    phfem_topology fine_topo;
    memset(&fine_topo, 0, sizeof fine_topo);
    if (st == PHFEM_OK) {
      if (flags & PHFEM_PIPE_GENERIC_EG) {
        if (l == levels - 1) {  // final level, sort-built: classification + C fused too
          st = build_topology_fused(ctx, &next, &fine_topo, &out->cls, &out->C);
          have_cls_C = st == PHFEM_OK;
        } else {
          st = phfem_build_topology(ctx, &next, &fine_topo);
        }
      } else if (last_fused) {
        st = refine_level_impl(ctx, &cur, &topo, &pcls, &next, &fine_topo, &out->cls, &out->C, mid, true);
        have_cls_C = st == PHFEM_OK;
      } else {
        st = refine_topology_impl(ctx, &cur, &topo, &next, &fine_topo, mid, true);
      }
      if (st != PHFEM_OK) phfem_mesh_release(ctx, &next);
    }
    tr("fine topology");
    phfem_classification_release(ctx, &pcls);
    phfem_topology_release(ctx, &topo);
    if (st == PHFEM_OK && l == levels - 1 && vol_parents) {
      parent.m = cur;
      parent.live = true;
    } else {
      phfem_mesh_release(ctx, &cur);
    }
    tr("release parent");
    if (st != PHFEM_OK) return st;
    cur = next;
    topo = fine_topo;
  }
  out->mesh = cur;
  out->topo = topo;
  if (!have_cls_C) PHFEM_TRY(phfem_classify_edges(ctx, &out->topo, &out->mesh, &out->cls));
  tr("classify");
  const int64_t nE = out->mesh.nE;
  PHFEM_TRY(dalloc(ctx, &out->B, 9 * nE));
  PHFEM_TRY(dalloc(ctx, &out->D, 9 * nE));
  PHFEM_TRY(dalloc(ctx, &out->M, 9 * nE));
  PHFEM_TRY(dalloc(ctx, &out->M0, 9 * nE));
  PHFEM_TRY(dalloc(ctx, &out->load, 3 * nE));
  PHFEM_TRY(dalloc(ctx, &out->bd, std::max(out->cls.L, 1)));
  tr("alloc outputs");
  PHFEM_TRY(errors_reset(ctx));
  VolArgs a = make_vol_args(&out->mesh);
  a.coeffs = *c;
  a.f = *f;
  a.t = t;
  a.B = out->B;
  a.D = out->D;
  a.M = out->M;
  a.M0 = out->M0;
  a.load = out->load;
  a.vec = 2;  // pool allocations are 256-byte aligned (32-byte stores allowed)
  if (parent.live && (int64_t)4 * parent.m.nE == nE) a.parents = parent.m.elements;
  PHFEM_TRY(launch_volume(ctx, a, true, true));
  tr("volume+load");
  PHFEM_TRY(neumann_into(ctx, &out->mesh, &out->topo, &out->cls, g, t, out->load, 1, false));
  if (!have_cls_C) PHFEM_TRY(constraint_csr_into(ctx, &out->mesh, &out->topo, &out->cls, &out->C));
  // (measured: zeroing bD on a side stream beside the input edge pass instead
  // of the 1.6 GB memset here — the fill slows the scatter / tile kernels it
  // shares HBM with by about as much as it saves: 13.95 -> 13.92-13.97 ms)
  PHFEM_TRY(dirichlet_into(ctx, &out->mesh, &out->topo, &out->cls, uD, t, out->bd));
  tr("neumann+C+dirichlet");
  unsigned long long dmisc = ~0ull;
  PHFEM_CUDA(ctx, cudaMemcpyAsync(&dmisc, &ctx->dderr->misc, sizeof dmisc, cudaMemcpyDeviceToHost, ctx->stream));
  PHFEM_TRY(errors_fetch(ctx));
  if (dmisc != ~0ull) return set_error(ctx, PHFEM_ERR_MISMATCH, "red_refine: topology does not match mesh");
  PHFEM_TRY(volume_errors(ctx, true, true));
  PHFEM_TRY(neu_flux_error(ctx, &out->mesh, &out->topo, &out->cls));
  return PHFEM_OK;
}

}  // namespace phfem

using namespace phfem;

PHFEM_API void phfem_pipeline_release(phfem_ctx* ctx, phfem_pipeline_out* out) {
  if (!out) return;
  phfem_csr_release(ctx, &out->C);
  phfem_classification_release(ctx, &out->cls);
  phfem_topology_release(ctx, &out->topo);
  phfem_mesh_release(ctx, &out->mesh);
  dfree(ctx, out->B);
  dfree(ctx, out->D);
  dfree(ctx, out->M);
  dfree(ctx, out->M0);
  dfree(ctx, out->load);
  dfree(ctx, out->bd);
}

PHFEM_API phfem_status phfem_pipeline(phfem_ctx* ctx, const phfem_mesh* mesh_in, int levels,
                                      const phfem_coeffs* c, const phfem_field* f,
                                      const phfem_field* g, const phfem_field* uD, double t,
                                      phfem_pipeline_out* out) {
  return phfem_pipeline_ex(ctx, mesh_in, levels, c, f, g, uD, t, 0, out);
}

PHFEM_API phfem_status phfem_pipeline_ex(phfem_ctx* ctx, const phfem_mesh* mesh_in, int levels,
                                         const phfem_coeffs* c, const phfem_field* f,
                                         const phfem_field* g, const phfem_field* uD, double t,
                                         int flags, phfem_pipeline_out* out) {
  memset(out, 0, sizeof(*out));
  if (!ctx || !mesh_in || !c || !f || !g || !uD || levels < 0) return PHFEM_ERR_INVALID_ARGUMENT;
  phfem_mesh cur = *mesh_in;
  cur.owned = 0;  // the caller's mesh is never freed here
  phfem_status st = pipeline_impl(ctx, cur, levels, c, f, g, uD, t, flags, out);
  if (st != PHFEM_OK) {
    const std::string msg = ctx->message;
    phfem_pipeline_release(ctx, out);
    ctx->message = msg;
  }
  return st;
}

PHFEM_API phfem_status phfem_pipeline_from_host(phfem_ctx* ctx, const double* coords,
                                                const int32_t* elements, const int32_t* dirichlet,
                                                const int32_t* neumann, int32_t nC, int32_t nE,
                                                int32_t nD, int32_t nN, int levels,
                                                const phfem_coeffs* c, const phfem_field* f,
                                                const phfem_field* g, const phfem_field* uD,
                                                double t, phfem_pipeline_out* out) {
  memset(out, 0, sizeof(*out));
  if (!ctx || !c || !f || !g || !uD || levels < 0 || nC < 0 || nE < 0 || nD < 0 || nN < 0)
    return PHFEM_ERR_INVALID_ARGUMENT;
  phfem_mesh m;
  memset(&m, 0, sizeof m);
  m.nC = nC;
  m.nE = nE;
  m.nD = nD;
  m.nN = nN;
  m.owned = 1;
  PHFEM_TRY(dalloc(ctx, &m.coords, 2 * (int64_t)nC));
  PHFEM_TRY(dalloc(ctx, &m.elements, 3 * (int64_t)nE));
  PHFEM_TRY(dalloc(ctx, &m.dirichlet, 2 * (int64_t)nD));
  PHFEM_TRY(dalloc(ctx, &m.neumann, 2 * (int64_t)nN));
  if (nC) PHFEM_CUDA(ctx, cudaMemcpyAsync(m.coords, coords, 16 * (size_t)nC, cudaMemcpyHostToDevice, ctx->stream));
  if (nE) PHFEM_CUDA(ctx, cudaMemcpyAsync(m.elements, elements, 12 * (size_t)nE, cudaMemcpyHostToDevice, ctx->stream));
  if (nD) PHFEM_CUDA(ctx, cudaMemcpyAsync(m.dirichlet, dirichlet, 8 * (size_t)nD, cudaMemcpyHostToDevice, ctx->stream));
  if (nN) PHFEM_CUDA(ctx, cudaMemcpyAsync(m.neumann, neumann, 8 * (size_t)nN, cudaMemcpyHostToDevice, ctx->stream));
  phfem_status st = pipeline_impl(ctx, m, levels, c, f, g, uD, t, 0, out);
  if (st != PHFEM_OK) {
    const std::string msg = ctx->message;
    phfem_pipeline_release(ctx, out);
    ctx->message = msg;
  }
  return st;
}

// phfem_pipeline_download / _download_bytes: download.cu
