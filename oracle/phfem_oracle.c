/*
 * phfem_oracle.c — TEST INFRASTRUCTURE ONLY (see phfem_oracle.h).
 *
 * Single-threaded C restatement of the reference algorithm, function by
 * function, with the reference line numbers beside each step.  Floating-point
 * expressions are written in the reference's evaluation order (SURVEY.md
 * Appendix A) and this file is compiled with -ffp-contract=off, like the
 * reference build (x86-64 -O3, no -march: no FMA).
 */
#include "phfem_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../include/phfem_gpu.h"

#define SETERR(...)                                  \
  do {                                               \
    if (err && errlen) snprintf(err, errlen, __VA_ARGS__); \
  } while (0)

static const double kR[3][3] = {{0.0, 0.5, 0.5}, {0.5, 0.0, 0.5}, {0.5, 0.5, 0.0}}; /* assembly.cpp:39 */

static void* xmalloc(size_t n) {
  void* p = malloc(n ? n : 1);
  if (!p) {
    fprintf(stderr, "oracle: out of memory (%zu bytes)\n", n);
    abort();
  }
  return p;
}
static void* xcalloc(size_t n, size_t s) {
  void* p = calloc(n ? n : 1, s ? s : 1);
  if (!p) {
    fprintf(stderr, "oracle: out of memory\n");
    abort();
  }
  return p;
}

void orc_free(void* p) { free(p); }

void orc_mesh_free(orc_mesh* m) {
  if (!m) return;
  free(m->coords);
  free(m->elements);
  free(m->dirichlet);
  free(m->neumann);
  memset(m, 0, sizeof(*m));
}

void orc_topology_free(orc_topology* t) {
  if (!t) return;
  free(t->edge_nodes);
  free(t->edge_elements);
  free(t->local_in_tplus);
  free(t->local_in_tminus);
  free(t->interior_edges);
  free(t->boundary_edges);
  free(t->elem_edge);
  free(t->node_edge_start);
  free(t->pair_offsets);
  free(t->pair_entries);
  free(t->directed_offsets);
  free(t->directed_entries);
  memset(t, 0, sizeof(*t));
}

void orc_classification_free(orc_classification* c) {
  if (!c) return;
  free(c->dirichlet_edge_ids);
  free(c->neumann_edge_ids);
  free(c->retained_edges);
  free(c->retained_pos);
  memset(c, 0, sizeof(*c));
}

void orc_sparse_free(orc_sparse* s) {
  if (!s) return;
  free(s->ptr);
  free(s->idx);
  free(s->val);
  memset(s, 0, sizeof(*s));
}

/* ------------------------------------------------------------------------ */
/* edge_topology.cpp:36-43 */
int orc_node_pair_to_edge(const orc_topology* t, int k, int l) {
  const int lo = k < l ? k : l;
  const int hi = k < l ? l : k;
  if (lo < 0 || hi >= t->nC) return -1;
  for (int s = t->pair_offsets[lo]; s < t->pair_offsets[lo + 1]; ++s)
    if (t->pair_entries[2 * s] == hi) return t->pair_entries[2 * s + 1];
  return -1;
}

/* edge_topology.cpp:45-50 */
int orc_directed_pair_to_element(const orc_topology* t, int k, int l) {
  if (k < 0 || k >= t->nC) return -1;
  for (int s = t->directed_offsets[k]; s < t->directed_offsets[k + 1]; ++s)
    if (t->directed_entries[2 * s] == l) return t->directed_entries[2 * s + 1];
  return -1;
}

typedef struct {
  int from, to, elem, local;
} directed_t; /* edge_topology.cpp:12-17 */

static inline int d_lo(const directed_t* d) { return d->from < d->to ? d->from : d->to; }
static inline int d_hi(const directed_t* d) { return d->from < d->to ? d->to : d->from; }

/* edge_topology.cpp:19-32: stable counting sort of `order` by key in [0,bins) */
static void counting_sort(int32_t** order, int32_t** scratch, int64_t n, int bins,
                          const directed_t* entries, int by_hi) {
  int64_t* counts = (int64_t*)xcalloc((size_t)bins + 1, sizeof(int64_t));
  int32_t* o = *order;
  int32_t* s = *scratch;
  for (int64_t i = 0; i < n; ++i) {
    const directed_t* d = &entries[o[i]];
    ++counts[(by_hi ? d_hi(d) : d_lo(d)) + 1];
  }
  for (int b = 0; b < bins; ++b) counts[b + 1] += counts[b];
  for (int64_t i = 0; i < n; ++i) {
    const directed_t* d = &entries[o[i]];
    s[counts[by_hi ? d_hi(d) : d_lo(d)]++] = o[i];
  }
  *order = s;
  *scratch = o;
  free(counts);
}

/* edge_topology.cpp:52-143 build_topology (+ the derived a6 map and the
 * max-node grouping table the device path exposes). */
int orc_build_topology(const orc_mesh* mesh, orc_topology* out, char* err, size_t errlen) {
  memset(out, 0, sizeof(*out));
  const int ne = mesh->nE;
  const int nc = mesh->nC;
  const int64_t nd = 3 * (int64_t)ne;
  out->nC = nc;
  out->nE = ne;

  /* :61-68 directed emission, local indices (2, 0, 1) */
  directed_t* directed = (directed_t*)xmalloc(sizeof(directed_t) * (size_t)nd);
  for (int m = 0; m < ne; ++m) {
    const int32_t* t = mesh->elements + 3 * (size_t)m;
    directed[3 * (size_t)m + 0] = (directed_t){t[0], t[1], m, 2};
    directed[3 * (size_t)m + 1] = (directed_t){t[1], t[2], m, 0};
    directed[3 * (size_t)m + 2] = (directed_t){t[2], t[0], m, 1};
  }

  /* :74-77 two stable counting passes: by min, then by max */
  int32_t* order = (int32_t*)xmalloc(sizeof(int32_t) * (size_t)nd);
  int32_t* scratch = (int32_t*)xmalloc(sizeof(int32_t) * (size_t)nd);
  for (int64_t i = 0; i < nd; ++i) order[i] = (int32_t)i;
  counting_sort(&order, &scratch, nd, nc, directed, 0);
  counting_sort(&order, &scratch, nd, nc, directed, 1);

  /* :82-115 run loop (vectors sized to the upper bound, trimmed below) */
  int32_t* en = (int32_t*)xmalloc(sizeof(int32_t) * 2 * (size_t)(nd + 1));
  int32_t* ee = (int32_t*)xmalloc(sizeof(int32_t) * 2 * (size_t)(nd + 1));
  int32_t* ltp = (int32_t*)xmalloc(sizeof(int32_t) * (size_t)(nd + 1));
  int32_t* ltm = (int32_t*)xmalloc(sizeof(int32_t) * (size_t)(nd + 1));
  int32_t* inter = (int32_t*)xmalloc(sizeof(int32_t) * (size_t)(nd + 1));
  int32_t* bound = (int32_t*)xmalloc(sizeof(int32_t) * (size_t)(nd + 1));
  int E = 0, ni = 0, nb = 0;
  int status = PHFEM_OK;
  for (int64_t g = 0; g < nd;) {
    const int lo = d_lo(&directed[order[g]]);
    const int hi = d_hi(&directed[order[g]]);
    int64_t end = g + 1;
    while (end < nd && d_lo(&directed[order[end]]) == lo && d_hi(&directed[order[end]]) == hi)
      ++end;
    if (end - g > 2) {
      SETERR("build_topology: non-manifold edge (%d,%d) shared by more than two elements",
             lo + 1, hi + 1);
      status = PHFEM_ERR_NONMANIFOLD;
      break;
    }
    const directed_t* first = &directed[order[g]];
    if (end - g == 2) {
      const directed_t* second = &directed[order[g + 1]];
      if (second->from == first->from) {
        SETERR("build_topology: duplicate directed edge %d->%d", first->from + 1, first->to + 1);
        status = PHFEM_ERR_DUP_DIRECTED;
        break;
      }
    }
    const int e = E++;
    en[2 * e] = first->from;
    en[2 * e + 1] = first->to;
    ltp[e] = first->local;
    if (end - g == 2) {
      const directed_t* second = &directed[order[g + 1]];
      ee[2 * e] = first->elem;
      ee[2 * e + 1] = second->elem;
      ltm[e] = second->local;
      inter[ni++] = e;
    } else {
      ee[2 * e] = first->elem;
      ee[2 * e + 1] = -1;
      ltm[e] = -1;
      bound[nb++] = e;
    }
    g = end;
  }
  free(order);
  free(scratch);
  if (status != PHFEM_OK) {
    free(directed);
    free(en); free(ee); free(ltp); free(ltm); free(inter); free(bound);
    return status;
  }
  out->E = E;
  out->n_interior = ni;
  out->n_boundary = nb;
  out->edge_nodes = en;
  out->edge_elements = ee;
  out->local_in_tplus = ltp;
  out->local_in_tminus = ltm;
  out->interior_edges = inter;
  out->boundary_edges = bound;

  /* :117-131 pair lookup table by min node, entries in ascending edge id */
  out->pair_offsets = (int32_t*)xcalloc((size_t)nc + 1, sizeof(int32_t));
  for (int e = 0; e < E; ++e) {
    const int a = en[2 * e], b = en[2 * e + 1];
    ++out->pair_offsets[(a < b ? a : b) + 1];
  }
  for (int v = 0; v < nc; ++v) out->pair_offsets[v + 1] += out->pair_offsets[v];
  out->pair_entries = (int32_t*)xmalloc(sizeof(int32_t) * 2 * (size_t)(E + 1));
  {
    int32_t* cursor = (int32_t*)xmalloc(sizeof(int32_t) * ((size_t)nc + 1));
    memcpy(cursor, out->pair_offsets, sizeof(int32_t) * (size_t)nc);
    for (int e = 0; e < E; ++e) {
      const int a = en[2 * e], b = en[2 * e + 1];
      const int lo = a < b ? a : b, hi = a < b ? b : a;
      const int p = cursor[lo]++;
      out->pair_entries[2 * p] = hi;
      out->pair_entries[2 * p + 1] = e;
    }
    free(cursor);
  }
  /* :133-140 directed lookup table by initial node, emission order */
  out->directed_offsets = (int32_t*)xcalloc((size_t)nc + 1, sizeof(int32_t));
  for (int64_t i = 0; i < nd; ++i) ++out->directed_offsets[directed[i].from + 1];
  for (int v = 0; v < nc; ++v) out->directed_offsets[v + 1] += out->directed_offsets[v];
  out->directed_entries = (int32_t*)xmalloc(sizeof(int32_t) * 2 * (size_t)(nd + 1));
  {
    int32_t* cursor = (int32_t*)xmalloc(sizeof(int32_t) * ((size_t)nc + 1));
    memcpy(cursor, out->directed_offsets, sizeof(int32_t) * (size_t)nc);
    for (int64_t i = 0; i < nd; ++i) {
      const int p = cursor[directed[i].from]++;
      out->directed_entries[2 * p] = directed[i].to;
      out->directed_entries[2 * p + 1] = directed[i].elem;
    }
    free(cursor);
  }
  free(directed);

  /* Max-node grouping: canonical ids are ordered by (max, min), so the edges
   * whose larger node is v form the contiguous id range [start[v], start[v+1]). */
  out->node_edge_start = (int32_t*)xcalloc((size_t)nc + 1, sizeof(int32_t));
  for (int e = 0; e < E; ++e) {
    const int a = en[2 * e], b = en[2 * e + 1];
    ++out->node_edge_start[(a < b ? b : a) + 1];
  }
  for (int v = 0; v < nc; ++v) out->node_edge_start[v + 1] += out->node_edge_start[v];

  /* a6: element -> edge map with signs, as the reference derives it per element
   * (refine.cpp:30-32 / analysis.cpp:171-177: node_pair_to_edge of the edge
   * opposite vertex k; sign +1 iff edge_elements[e][0] == m). */
  out->elem_edge = (int32_t*)xmalloc(sizeof(int32_t) * 3 * (size_t)(ne + 1));
  for (int m = 0; m < ne; ++m) {
    const int32_t* t = mesh->elements + 3 * (size_t)m;
    for (int k = 0; k < 3; ++k) {
      const int e = orc_node_pair_to_edge(out, t[(k + 1) % 3], t[(k + 2) % 3]);
      out->elem_edge[3 * (size_t)m + k] = (ee[2 * e] == m) ? e : ~e;
    }
  }
  return PHFEM_OK;
}

/* edge_topology.cpp:145-177 classify_edges */
int orc_classify_edges(const orc_topology* topo, const orc_mesh* mesh, orc_classification* out,
                       char* err, size_t errlen) {
  memset(out, 0, sizeof(*out));
  const int E = topo->E;
  out->nD = mesh->nD;
  out->nN = mesh->nN;
  out->E = E;
  out->dirichlet_edge_ids = (int32_t*)xmalloc(sizeof(int32_t) * ((size_t)mesh->nD + 1));
  out->neumann_edge_ids = (int32_t*)xmalloc(sizeof(int32_t) * ((size_t)mesh->nN + 1));
  for (int list = 0; list < 2; ++list) {
    const int n = list == 0 ? mesh->nD : mesh->nN;
    const int32_t* pairs = list == 0 ? mesh->dirichlet : mesh->neumann;
    const char* what = list == 0 ? "dirichlet" : "neumann";
    int32_t* ids = list == 0 ? out->dirichlet_edge_ids : out->neumann_edge_ids;
    for (int i = 0; i < n; ++i) {
      const int a = pairs[2 * i], b = pairs[2 * i + 1];
      const int e = orc_node_pair_to_edge(topo, a, b); /* :150 */
      if (e < 0) {
        SETERR("%s pair (%d,%d) is not an edge", what, a + 1, b + 1);
        orc_classification_free(out);
        return PHFEM_ERR_NOT_AN_EDGE;
      }
      if (topo->edge_elements[2 * e + 1] >= 0) {
        SETERR("%s pair (%d,%d) resolves to an interior edge", what, a + 1, b + 1);
        orc_classification_free(out);
        return PHFEM_ERR_INTERIOR_BOUNDARY;
      }
      ids[i] = e;
    }
  }
  char* is_neumann = (char*)xcalloc((size_t)E + 1, 1); /* :166-167 */
  for (int i = 0; i < mesh->nN; ++i) is_neumann[out->neumann_edge_ids[i]] = 1;
  out->retained_pos = (int32_t*)xmalloc(sizeof(int32_t) * ((size_t)E + 1));
  out->retained_edges = (int32_t*)xmalloc(sizeof(int32_t) * ((size_t)E + 1));
  int L = 0;
  for (int e = 0; e < E; ++e) { /* :169-174 */
    if (!is_neumann[e]) {
      out->retained_pos[e] = L;
      out->retained_edges[L++] = e;
    } else {
      out->retained_pos[e] = -1;
    }
  }
  free(is_neumann);
  out->L = L;
  return PHFEM_OK;
}

/* edge_topology.cpp:179-186: (c[b] - c[a]).norm() */
int orc_edge_lengths(const orc_mesh* mesh, const orc_topology* topo, double* out) {
  for (int e = 0; e < topo->E; ++e) {
    const int a = topo->edge_nodes[2 * e], b = topo->edge_nodes[2 * e + 1];
    const double dx = mesh->coords[2 * (size_t)b] - mesh->coords[2 * (size_t)a];
    const double dy = mesh->coords[2 * (size_t)b + 1] - mesh->coords[2 * (size_t)a + 1];
    out[e] = sqrt(dx * dx + dy * dy);
  }
  return PHFEM_OK;
}

/* refine.cpp:7-53 red_refine */
int orc_red_refine(const orc_mesh* mesh, const orc_topology* topo, orc_mesh* out, char* err,
                   size_t errlen) {
  memset(out, 0, sizeof(*out));
  const int nc = mesh->nC, ne = mesh->nE, E = topo->E;
  out->nC = nc + E;
  out->nE = 4 * ne;
  out->nD = 2 * mesh->nD;
  out->nN = 2 * mesh->nN;
  out->coords = (double*)xmalloc(sizeof(double) * 2 * ((size_t)nc + E + 1));
  memcpy(out->coords, mesh->coords, sizeof(double) * 2 * (size_t)nc); /* :13 */
  for (int e = 0; e < E; ++e) {                                      /* :16-19 */
    const int a = topo->edge_nodes[2 * e], b = topo->edge_nodes[2 * e + 1];
    out->coords[2 * ((size_t)nc + e)] = 0.5 * (mesh->coords[2 * (size_t)a] + mesh->coords[2 * (size_t)b]);
    out->coords[2 * ((size_t)nc + e) + 1] =
        0.5 * (mesh->coords[2 * (size_t)a + 1] + mesh->coords[2 * (size_t)b + 1]);
  }
  out->elements = (int32_t*)xmalloc(sizeof(int32_t) * 12 * ((size_t)ne + 1));
  for (int m = 0; m < ne; ++m) { /* :27-37 */
    const int32_t* t = mesh->elements + 3 * (size_t)m;
    const int p0 = t[0], p1 = t[1], p2 = t[2];
    const int e0 = orc_node_pair_to_edge(topo, p1, p2);
    const int e1 = orc_node_pair_to_edge(topo, p2, p0);
    const int e2 = orc_node_pair_to_edge(topo, p0, p1);
    if (e0 < 0 || e1 < 0 || e2 < 0) {
      SETERR("red_refine: topology does not match mesh");
      orc_mesh_free(out);
      return PHFEM_ERR_MISMATCH;
    }
    const int m0 = nc + e0, m1 = nc + e1, m2 = nc + e2;
    int32_t* c = out->elements + 12 * (size_t)m;
    c[0] = m0; c[1] = m1; c[2] = m2;
    c[3] = p0; c[4] = m2; c[5] = m1;
    c[6] = p1; c[7] = m0; c[8] = m2;
    c[9] = p2; c[10] = m1; c[11] = m0;
  }
  for (int list = 0; list < 2; ++list) { /* :39-50 bisect */
    const int n = list == 0 ? mesh->nD : mesh->nN;
    const int32_t* in = list == 0 ? mesh->dirichlet : mesh->neumann;
    int32_t* h = (int32_t*)xmalloc(sizeof(int32_t) * 4 * ((size_t)n + 1));
    for (int i = 0; i < n; ++i) {
      const int a = in[2 * i], b = in[2 * i + 1];
      const int e = orc_node_pair_to_edge(topo, a, b);
      if (e < 0) {
        free(h);
        SETERR("red_refine: topology does not match mesh");
        orc_mesh_free(out);
        return PHFEM_ERR_MISMATCH;
      }
      const int mid = nc + e;
      h[4 * i] = a; h[4 * i + 1] = mid;
      h[4 * i + 2] = mid; h[4 * i + 3] = b;
    }
    if (list == 0) out->dirichlet = h; else out->neumann = h;
  }
  return PHFEM_OK;
}

/* Config-4 orientation normalisation (not in the reference): swap v1 <-> v2
 * of every element with negative signed area (mesh.cpp:104-106 formula). */
int orc_orient_ccw(orc_mesh* mesh) {
  for (int m = 0; m < mesh->nE; ++m) {
    int32_t* t = mesh->elements + 3 * (size_t)m;
    const double* a = mesh->coords + 2 * (size_t)t[0];
    const double* b = mesh->coords + 2 * (size_t)t[1];
    const double* c = mesh->coords + 2 * (size_t)t[2];
    const double t2 = (b[0] - a[0]) * (c[1] - a[1]) - (b[1] - a[1]) * (c[0] - a[0]);
    if (t2 < 0.0) {
      const int32_t s = t[1];
      t[1] = t[2];
      t[2] = s;
    }
  }
  return PHFEM_OK;
}

/* assembly.cpp:97-142 assemble_volume_operators: 4 block-diagonal matrices,
 * value layout vals[9m + 3j + i] = X(i,j). */
int orc_assemble_volume(const orc_mesh* mesh, const phfem_coeffs* c, double* B, double* D,
                        double* M, double* M0, char* err, size_t errlen) {
  for (int m = 0; m < mesh->nE; ++m) {
    const int32_t* t = mesh->elements + 3 * (size_t)m;
    const double* v0 = mesh->coords + 2 * (size_t)t[0];
    const double* v1 = mesh->coords + 2 * (size_t)t[1];
    const double* v2 = mesh->coords + 2 * (size_t)t[2];
    const phfem_coeff_values cv = phfem_coeffs_eval(c, v0[0], v0[1], v1[0], v1[1], v2[0], v2[1]);
    double b[9], d[9], mm[9], m0[9];
    const double t2 = phfem_local_blocks(v0[0], v0[1], v1[0], v1[1], v2[0], v2[1], &cv, b, d, mm, m0);
    if (!(t2 > 0.0)) { /* assembly.cpp:19-20 */
      SETERR("local_element_matrices: degenerate or non-CCW triangle");
      return PHFEM_ERR_DEGENERATE;
    }
    if (B) memcpy(B + 9 * (size_t)m, b, sizeof b);
    if (D) memcpy(D + 9 * (size_t)m, d, sizeof d);
    if (M) memcpy(M + 9 * (size_t)m, mm, sizeof mm);
    if (M0) memcpy(M0 + 9 * (size_t)m, m0, sizeof m0);
  }
  return PHFEM_OK;
}

/* assembly.cpp:144-168 assemble_constraint: triplets in edge order (rows
 * ascending, columns ascending inside a row -> sorted-unique fast path of
 * from_triplets, sparse.cpp:43-53), then the stable column scatter into CSC
 * (sparse.cpp:82-96).  The triplet stream itself is the CSR form. */
int orc_assemble_constraint(const orc_mesh* mesh, const orc_topology* topo,
                            const orc_classification* cls, orc_sparse* csr, orc_sparse* csc,
                            char* err, size_t errlen) {
  const int n_dofs = 3 * mesh->nE;
  const int L = cls->L;
  if (cls->E != topo->E) {
    SETERR("assemble_constraint: classification does not match topology");
    return PHFEM_ERR_MISMATCH;
  }
  double* lengths = (double*)xmalloc(sizeof(double) * ((size_t)topo->E + 1));
  orc_edge_lengths(mesh, topo, lengths);
  const size_t cap = 4 * (size_t)L + 1;
  int32_t* ri = (int32_t*)xmalloc(sizeof(int32_t) * cap);
  int32_t* ci = (int32_t*)xmalloc(sizeof(int32_t) * cap);
  double* vv = (double*)xmalloc(sizeof(double) * cap);
  int64_t n = 0;
  for (int e = 0; e < topo->E; ++e) {
    const int row = cls->retained_pos[e];
    if (row < 0) continue;
    const int tp = topo->edge_elements[2 * e], tm = topo->edge_elements[2 * e + 1];
    const int led = topo->local_in_tplus[e];
    for (int c = 0; c < 3; ++c)
      if (kR[led][c] != 0.0) {
        ri[n] = row; ci[n] = 3 * tp + c; vv[n] = lengths[e] * kR[led][c]; ++n;
      }
    if (tm >= 0) {
      const int ledtn = topo->local_in_tminus[e];
      for (int c = 0; c < 3; ++c)
        if (kR[ledtn][c] != 0.0) {
          ri[n] = row; ci[n] = 3 * tm + c; vv[n] = -lengths[e] * kR[ledtn][c]; ++n;
        }
    }
  }
  free(lengths);
  /* sparse.cpp:18-27 check_indices (never fires for a consistent topology) */
  for (int64_t k = 0; k < n; ++k)
    if (ri[k] < 0 || ri[k] >= L || ci[k] < 0 || ci[k] >= n_dofs) {
      SETERR("TripletBuffer: entry %lld at (%d,%d) outside %dx%d", (long long)k, ri[k], ci[k], L,
             n_dofs);
      free(ri); free(ci); free(vv);
      return PHFEM_ERR_OUT_OF_RANGE;
    }
  if (csr) {
    csr->rows = L;
    csr->cols = n_dofs;
    csr->nnz = n;
    csr->ptr = (int32_t*)xcalloc((size_t)L + 1, sizeof(int32_t));
    for (int64_t k = 0; k < n; ++k) ++csr->ptr[ri[k] + 1];
    for (int r = 0; r < L; ++r) csr->ptr[r + 1] += csr->ptr[r];
    csr->idx = (int32_t*)xmalloc(sizeof(int32_t) * (size_t)(n + 1));
    csr->val = (double*)xmalloc(sizeof(double) * (size_t)(n + 1));
    memcpy(csr->idx, ci, sizeof(int32_t) * (size_t)n);
    /* from_triplets keeps the buffer as-is (sorted-unique) -> values 1:1 */
    memcpy(csr->val, vv, sizeof(double) * (size_t)n);
  }
  if (csc) { /* sparse.cpp:82-96 */
    csc->rows = L;
    csc->cols = n_dofs;
    csc->nnz = n;
    csc->ptr = (int32_t*)xcalloc((size_t)n_dofs + 1, sizeof(int32_t));
    for (int64_t k = 0; k < n; ++k) ++csc->ptr[ci[k] + 1];
    for (int c = 0; c < n_dofs; ++c) csc->ptr[c + 1] += csc->ptr[c];
    csc->idx = (int32_t*)xmalloc(sizeof(int32_t) * (size_t)(n + 1));
    csc->val = (double*)xmalloc(sizeof(double) * (size_t)(n + 1));
    int32_t* cursor = (int32_t*)xmalloc(sizeof(int32_t) * ((size_t)n_dofs + 1));
    memcpy(cursor, csc->ptr, sizeof(int32_t) * (size_t)n_dofs);
    for (int64_t k = 0; k < n; ++k) {
      const int p = cursor[ci[k]]++;
      csc->idx[p] = ri[k];
      csc->val[p] = vv[k];
    }
    free(cursor);
  }
  free(ri); free(ci); free(vv);
  return PHFEM_OK;
}

/* assembly.cpp:179-203 assemble_load; scatter_add (sparse.cpp:108-120) adds
 * each value once into a zero vector: out = 0.0 + value. */
int orc_assemble_load(const orc_mesh* mesh, const phfem_field* f, double t, double* out,
                      char* err, size_t errlen) {
  for (int m = 0; m < mesh->nE; ++m) {
    const int32_t* tr = mesh->elements + 3 * (size_t)m;
    const double* v0 = mesh->coords + 2 * (size_t)tr[0];
    const double* v1 = mesh->coords + 2 * (size_t)tr[1];
    const double* v2 = mesh->coords + 2 * (size_t)tr[2];
    /* :35-37 midpoints opposite each vertex */
    const double mx[3] = {0.5 * (v1[0] + v2[0]), 0.5 * (v2[0] + v0[0]), 0.5 * (v0[0] + v1[0])};
    const double my[3] = {0.5 * (v1[1] + v2[1]), 0.5 * (v2[1] + v0[1]), 0.5 * (v0[1] + v1[1])};
    const double area =
        0.5 * ((v1[0] - v0[0]) * (v2[1] - v0[1]) - (v1[1] - v0[1]) * (v2[0] - v0[0]));
    double fm[3];
    for (int i = 0; i < 3; ++i) {
      fm[i] = phfem_field_eval(f, mx[i], my[i], t);
      if (!isfinite(fm[i])) {
        SETERR("assemble_load: non-finite load sample in element %d", m + 1);
        return PHFEM_ERR_NONFINITE;
      }
    }
    for (int i = 0; i < 3; ++i)
      out[3 * (size_t)m + i] = 0.0 + area / 3.0 * 0.5 * (fm[(i + 1) % 3] + fm[(i + 2) % 3]);
  }
  return PHFEM_OK;
}

/* assembly.cpp:205-228 assemble_neumann (scatter_add in list order) */
int orc_assemble_neumann(const orc_mesh* mesh, const orc_topology* topo,
                         const orc_classification* cls, const phfem_field* g, double t,
                         double* out, char* err, size_t errlen) {
  memset(out, 0, sizeof(double) * 3 * (size_t)mesh->nE);
  for (int i = 0; i < cls->nN; ++i) {
    const int e = cls->neumann_edge_ids[i];
    const int a = topo->edge_nodes[2 * e], b = topo->edge_nodes[2 * e + 1];
    const double* pa = mesh->coords + 2 * (size_t)a;
    const double* pb = mesh->coords + 2 * (size_t)b;
    const double midx = 0.5 * (pa[0] + pb[0]), midy = 0.5 * (pa[1] + pb[1]);
    const double dx = pb[0] - pa[0], dy = pb[1] - pa[1];
    const double length = sqrt(dx * dx + dy * dy);
    const double nx = dy / length, ny = -dx / length;
    const double value = phfem_flux_eval(g, midx, midy, nx, ny, t);
    if (!isfinite(value)) {
      SETERR("assemble_neumann: non-finite flux sample on edge (%d,%d)", a + 1, b + 1);
      return PHFEM_ERR_NONFINITE;
    }
    const int elem = topo->edge_elements[2 * e];
    const int led = topo->local_in_tplus[e];
    for (int c = 0; c < 3; ++c) out[3 * (size_t)elem + c] += length * value * kR[led][c];
  }
  return PHFEM_OK;
}

/* assembly.cpp:230-242 assemble_dirichlet */
int orc_assemble_dirichlet(const orc_mesh* mesh, const orc_topology* topo,
                           const orc_classification* cls, const phfem_field* uD, double t,
                           double* out, char* err, size_t errlen) {
  (void)err;
  (void)errlen;
  memset(out, 0, sizeof(double) * (size_t)cls->L);
  for (int i = 0; i < cls->nD; ++i) {
    const int e = cls->dirichlet_edge_ids[i];
    const int a = topo->edge_nodes[2 * e], b = topo->edge_nodes[2 * e + 1];
    const double* pa = mesh->coords + 2 * (size_t)a;
    const double* pb = mesh->coords + 2 * (size_t)b;
    const double midx = 0.5 * (pa[0] + pb[0]), midy = 0.5 * (pa[1] + pb[1]);
    const double dx = pb[0] - pa[0], dy = pb[1] - pa[1];
    const double length = sqrt(dx * dx + dy * dy);
    out[cls->retained_pos[e]] = -length * phfem_field_eval(uD, midx, midy, t);
  }
  return PHFEM_OK;
}

/* solve_parabolic's right-hand side for the step t_n -> t_{n+1}
 * (parabolic.cpp:92-103), with M_minus built the reference's way:
 * step_matrix(ops, k, -1) (parabolic.cpp:21-37) -> triplets -> from_triplets
 * (unsorted path: stable sort by (row, col), run sums 0.0 + v; sparse.cpp:53-78)
 * -> CSC; then the column-major SpMV res[i] += a_ij x_j (Eigen ColMajor sparse
 * x dense) and the two vector updates. */
int orc_cn_rhs(const orc_mesh* mesh, const orc_topology* topo, const orc_classification* cls,
               const phfem_coeffs* c, const phfem_field* f, const phfem_field* g,
               const phfem_field* uD, double k, int n, const double* state, double* rhs,
               char* err, size_t errlen) {
  if (!(k > 0.0)) {
    SETERR("step_matrices: k must be positive");
    return PHFEM_ERR_INVALID_ARGUMENT;
  }
  const int ne = mesh->nE;
  const int N = 3 * ne;
  const int L = cls->L;
  const size_t n9 = 9 * (size_t)ne;
  double* B = (double*)xmalloc(sizeof(double) * (n9 + 1));
  double* D = (double*)xmalloc(sizeof(double) * (n9 + 1));
  double* M = (double*)xmalloc(sizeof(double) * (n9 + 1));
  double* M0 = (double*)xmalloc(sizeof(double) * (n9 + 1));
  int st = orc_assemble_volume(mesh, c, B, D, M, M0, err, errlen);
  orc_sparse C = {0};
  if (st == PHFEM_OK) st = orc_assemble_constraint(mesh, topo, cls, NULL, &C, err, errlen);
  if (st != PHFEM_OK) {
    free(B); free(D); free(M); free(M0);
    orc_sparse_free(&C);
    return st;
  }
  const double sign = -1.0;
  const double s = sign * (k / 2.0);        /* parabolic.cpp:26 */
  const double sct = -sign * (k / 2.0);     /* :34 */
  const double scc = -sign * 0.5;           /* :35 */

  /* CSC of M_minus: column j < N holds the element block rows 3m..3m+2 then
   * the coupling rows N + r (C column j, ascending r); column N + r holds the
   * transposed coupling rows (ascending primal DOF). */
  const int ncol = N + L;
  int64_t* outer = (int64_t*)xcalloc((size_t)ncol + 1, sizeof(int64_t));
  for (int j = 0; j < N; ++j) outer[j + 1] = 3 + (C.ptr[j + 1] - C.ptr[j]);
  int32_t* rcnt = (int32_t*)xcalloc((size_t)L + 1, sizeof(int32_t));
  for (int64_t q = 0; q < C.nnz; ++q) ++rcnt[C.idx[q]];
  for (int r = 0; r < L; ++r) outer[N + r + 1] = rcnt[r];
  for (int j = 0; j < ncol; ++j) outer[j + 1] += outer[j];
  const int64_t nnz = outer[ncol];
  int32_t* inner = (int32_t*)xmalloc(sizeof(int32_t) * (size_t)(nnz + 1));
  double* val = (double*)xmalloc(sizeof(double) * (size_t)(nnz + 1));
  int64_t* cur = (int64_t*)xmalloc(sizeof(int64_t) * ((size_t)ncol + 1));
  memcpy(cur, outer, sizeof(int64_t) * (size_t)ncol);
  for (int m = 0; m < ne; ++m)
    for (int jj = 0; jj < 3; ++jj) {
      const int j = 3 * m + jj;
      for (int i = 0; i < 3; ++i) {
        const size_t q = 9 * (size_t)m + 3 * jj + i;
        /* top = M0 + s * ((B + D) + M); stored as 0.0 + 1.0 * top */
        const double top = M0[q] + s * ((B[q] + D[q]) + M[q]);
        inner[cur[j]] = 3 * m + i;
        val[cur[j]++] = 0.0 + 1.0 * top;
      }
      for (int q = C.ptr[j]; q < C.ptr[j + 1]; ++q) {
        inner[cur[j]] = N + C.idx[q];
        val[cur[j]++] = 0.0 + scc * C.val[q];
      }
    }
  /* transposed coupling block: column N + r gets (row j, sct * C(r, j)) with j
   * ascending — iterate C by column j ascending */
  for (int j = 0; j < N; ++j)
    for (int q = C.ptr[j]; q < C.ptr[j + 1]; ++q) {
      const int col = N + C.idx[q];
      inner[cur[col]] = j;
      val[cur[col]++] = 0.0 + sct * C.val[q];
    }
  free(cur);
  free(rcnt);

  /* rhs = M_minus * state (parabolic.cpp:100) */
  for (int i = 0; i < ncol; ++i) rhs[i] = 0.0;
  for (int j = 0; j < ncol; ++j) {
    const double xj = state[j];
    for (int64_t q = outer[j]; q < outer[j + 1]; ++q) rhs[inner[q]] += val[q] * xj;
  }
  free(outer); free(inner); free(val);

  /* loads at t_n and t_{n+1} (load_at_time, parabolic.cpp:56-64) */
  double* b0 = (double*)xmalloc(sizeof(double) * ((size_t)N + 1));
  double* b1 = (double*)xmalloc(sizeof(double) * ((size_t)N + 1));
  double* l0 = (double*)xmalloc(sizeof(double) * ((size_t)N + 1));
  double* l1 = (double*)xmalloc(sizeof(double) * ((size_t)N + 1));
  double* d0 = (double*)xmalloc(sizeof(double) * ((size_t)L + 1));
  double* d1 = (double*)xmalloc(sizeof(double) * ((size_t)L + 1));
  const double t0 = n * k;
  const double t1 = (n + 1) * k;
  st = orc_assemble_load(mesh, f, t0, b0, err, errlen);
  if (st == PHFEM_OK) st = orc_assemble_neumann(mesh, topo, cls, g, t0, l0, err, errlen);
  if (st == PHFEM_OK) st = orc_assemble_load(mesh, f, t1, b1, err, errlen);
  if (st == PHFEM_OK) st = orc_assemble_neumann(mesh, topo, cls, g, t1, l1, err, errlen);
  if (st == PHFEM_OK) st = orc_assemble_dirichlet(mesh, topo, cls, uD, t0, d0, err, errlen);
  if (st == PHFEM_OK) st = orc_assemble_dirichlet(mesh, topo, cls, uD, t1, d1, err, errlen);
  if (st == PHFEM_OK) {
    const double kh = k * 0.5;
    for (int i = 0; i < N; ++i) rhs[i] += kh * (((b0[i] + l0[i]) + b1[i]) + l1[i]); /* :101-102 */
    for (int r = 0; r < L; ++r) rhs[N + r] += 0.5 * (d0[r] + d1[r]);             /* :103 */
  }
  free(b0); free(b1); free(l0); free(l1); free(d0); free(d1);
  free(B); free(D); free(M); free(M0);
  orc_sparse_free(&C);
  return st;
}


/* ---- SparseMatrix::from_triplets (proj/src/sparse.cpp:30-97) ---------------
 * Index check with the first offending entry (:14-27); a buffer already in
 * strictly increasing (row, col) order is stored as-is (:41-45, :53);
 * otherwise a stable sort by (row, col) and left-to-right run sums starting
 * from 0.0 (:55-76); then the compressed-column fill, rows ascending in each
 * column (:80-96).  The stable sort is a merge sort of the entry indices.   */
static const int32_t* g_ri;
static const int32_t* g_ci;

static int trip_less(int64_t a, int64_t b) {
  if (g_ri[a] != g_ri[b]) return g_ri[a] < g_ri[b];
  return g_ci[a] < g_ci[b];
}

static void merge_sort_idx(int64_t* a, int64_t* tmp, int64_t n) {
  if (n < 2) return;
  const int64_t h = n / 2;
  merge_sort_idx(a, tmp, h);
  merge_sort_idx(a + h, tmp, n - h);
  int64_t i = 0, j = h, k = 0;
  while (i < h && j < n) tmp[k++] = trip_less(a[j], a[i]) ? a[j++] : a[i++];  /* stable */
  while (i < h) tmp[k++] = a[i++];
  while (j < n) tmp[k++] = a[j++];
  memcpy(a, tmp, sizeof(int64_t) * (size_t)n);
}

int orc_from_triplets(int32_t rows, int32_t cols, const int32_t* ri, const int32_t* ci,
                      const double* v, int64_t n, orc_sparse* out, char* err, size_t errlen) {
  memset(out, 0, sizeof(*out));
  for (int64_t k = 0; k < n; ++k)
    if (ri[k] < 0 || ri[k] >= rows || ci[k] < 0 || ci[k] >= cols) {
      snprintf(err, errlen, "TripletBuffer: entry %lld at (%d,%d) outside %dx%d", (long long)k, ri[k],
               ci[k], rows, cols);
      return 8; /* std::out_of_range */
    }
  g_ri = ri;
  g_ci = ci;
  int sorted_unique = 1;
  for (int64_t k = 1; k < n && sorted_unique; ++k)
    if (!trip_less(k - 1, k)) sorted_unique = 0;
  int32_t* mi = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  int32_t* mj = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  double* mv = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
  int64_t nnz = 0;
  if (sorted_unique) {
    for (int64_t k = 0; k < n; ++k) {
      mi[k] = ri[k];
      mj[k] = ci[k];
      mv[k] = v[k];
    }
    nnz = n;
  } else {
    int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    int64_t* tmp = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    for (int64_t k = 0; k < n; ++k) perm[k] = k;
    merge_sort_idx(perm, tmp, n);
    int64_t k = 0;
    while (k < n) {
      const int32_t i = ri[perm[k]], j = ci[perm[k]];
      double sum = 0.0;
      while (k < n && ri[perm[k]] == i && ci[perm[k]] == j) sum += v[perm[k++]];
      mi[nnz] = i;
      mj[nnz] = j;
      mv[nnz] = sum;
      ++nnz;
    }
    free(perm);
    free(tmp);
  }
  out->rows = rows;
  out->cols = cols;
  out->nnz = nnz;
  out->ptr = (int32_t*)calloc((size_t)cols + 1, sizeof(int32_t));
  out->idx = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nnz ? nnz : 1));
  out->val = (double*)malloc(sizeof(double) * (size_t)(nnz ? nnz : 1));
  for (int64_t e = 0; e < nnz; ++e) ++out->ptr[mj[e] + 1];
  for (int32_t c2 = 0; c2 < cols; ++c2) out->ptr[c2 + 1] += out->ptr[c2];
  int32_t* cursor = (int32_t*)malloc(sizeof(int32_t) * (size_t)(cols ? cols : 1));
  memcpy(cursor, out->ptr, sizeof(int32_t) * (size_t)cols);
  for (int64_t e = 0; e < nnz; ++e) {
    const int32_t p = cursor[mj[e]]++;
    out->idx[p] = mi[e];
    out->val[p] = mv[e];
  }
  free(cursor);
  free(mi);
  free(mj);
  free(mv);
  return 0;
}

/* ======================================================================
 * Verification around the solve.
 * ====================================================================== */

/* ||C U + bD||_inf (tools/main.cpp:205-207): the ColMajor SpMV of the CSC C
 * (res = 0; res[i] += a_ij U_j, columns ascending), + bD, lpNorm<Infinity>. */
int orc_constraint_residual(const orc_sparse* csc, const double* U, const double* bd, double* out) {
  const int L = csc->rows;
  double* res = (double*)xcalloc((size_t)L + 1, sizeof(double));
  for (int j = 0; j < csc->cols; ++j) {
    const double xj = U[j];
    for (int p = csc->ptr[j]; p < csc->ptr[j + 1]; ++p) res[csc->idx[p]] += csc->val[p] * xj;
  }
  double worst = 0.0;
  for (int l = 0; l < L; ++l) {
    const double r = bd ? res[l] + bd[l] : res[l];
    const double a = fabs(r);
    if (a > worst || a != a) worst = a;
  }
  free(res);
  *out = worst;
  return PHFEM_OK;
}

/* exact_multiplier (analysis.cpp:26-39): for each retained edge, in edge
 * order, (A grad u + u p) . nu at the midpoint (phfem_fields.h formula). */
int orc_exact_multiplier(const orc_mesh* mesh, const orc_topology* topo,
                         const orc_classification* cls, const phfem_problem* p, double t,
                         double* out) {
  for (int k = 0; k < cls->L; ++k) {
    const int e = cls->retained_edges[k];
    const int a = topo->edge_nodes[2 * e], b = topo->edge_nodes[2 * e + 1];
    out[cls->retained_pos[e]] =
        phfem_exact_multiplier_value(p, mesh->coords[2 * a], mesh->coords[2 * a + 1],
                                     mesh->coords[2 * b], mesh->coords[2 * b + 1], t);
  }
  return PHFEM_OK;
}

/* error_l2 / error_h1 (analysis.cpp:41-80): sum of the per-element terms in
 * element order, then sqrt.  terms (nullable) receives every term. */
static int error_norm(const orc_mesh* mesh, const double* U, const phfem_problem* p, double t,
                      double* out, double* terms, int h1) {
  phfem_quad_rule rule;
  phfem_default_rule(&rule);
  double sum = 0.0;
  for (int m = 0; m < mesh->nE; ++m) {
    const int* tv = mesh->elements + 3 * m;
    const double* c = mesh->coords;
    const double x0 = c[2 * tv[0]], y0 = c[2 * tv[0] + 1], x1 = c[2 * tv[1]], y1 = c[2 * tv[1] + 1];
    const double x2 = c[2 * tv[2]], y2 = c[2 * tv[2] + 1];
    const double term = h1 ? phfem_h1_term(p, &rule, x0, y0, x1, y1, x2, y2, U[3 * m], U[3 * m + 1],
                                           U[3 * m + 2], t)
                           : phfem_l2_term(p, &rule, x0, y0, x1, y1, x2, y2, U[3 * m], U[3 * m + 1],
                                           U[3 * m + 2], t);
    if (terms) terms[m] = term;
    sum += term;
  }
  *out = sqrt(sum);
  return PHFEM_OK;
}

int orc_error_l2(const orc_mesh* mesh, const double* U, const phfem_problem* p, double t,
                 double* out, double* terms) {
  return error_norm(mesh, U, p, t, out, terms, 0);
}

int orc_error_h1(const orc_mesh* mesh, const double* U, const phfem_problem* p, double t,
                 double* out, double* terms) {
  return error_norm(mesh, U, p, t, out, terms, 1);
}

/* error_multiplier (analysis.cpp:82-98): w = C' (exact - discrete) through
 * the CSC columns (rows ascending, from 0), max |w_i| / sqrt(B_ii) over the
 * B_ii > 0 (B = stiffness blocks [nE][9], diagonal at 9m + 4i). */
int orc_error_multiplier(const orc_sparse* csc, const double* B, const double* exact,
                         const double* discrete, int64_t n_exact, int64_t n_discrete, double* out,
                         char* err, size_t errlen) {
  if (n_exact != n_discrete || n_exact != csc->rows) {
    SETERR("error_multiplier: size mismatch");
    return PHFEM_ERR_INVALID_ARGUMENT;
  }
  double worst = 0.0;
  int any = 0;
  for (int j = 0; j < csc->cols; ++j) {
    double w = 0.0;
    for (int p = csc->ptr[j]; p < csc->ptr[j + 1]; ++p) {
      const int l = csc->idx[p];
      w += csc->val[p] * (exact[l] - discrete[l]);
    }
    const double diag = B[9 * (size_t)(j / 3) + 4 * (j % 3)];
    if (diag <= 0.0) continue;
    any = 1;
    const double r = fabs(w) / sqrt(diag);
    if (worst < r) worst = r; /* std::max(worst, r) */
  }
  if (!any) {
    SETERR("error_multiplier: all diagonal entries of B vanish");
    return PHFEM_ERR_RUNTIME;
  }
  *out = worst;
  return PHFEM_OK;
}

/* hybrid_midpoint_traces (analysis.cpp:113-125) */
int orc_midpoint_traces(const orc_topology* topo, const double* U, double* out) {
  for (int e = 0; e < topo->E; ++e) {
    const int m = topo->edge_elements[2 * e];
    const int led = topo->local_in_tplus[e];
    out[e] = 0.5 * (U[3 * m + (led + 1) % 3] + U[3 * m + (led + 2) % 3]);
  }
  return PHFEM_OK;
}

/* y = A x, Eigen ColMajor sparse x dense (res = 0; res[i] += a_ij x_j) */
int orc_csc_spmv(const orc_sparse* csc, const double* x, double* y) {
  for (int i = 0; i < csc->rows; ++i) y[i] = 0.0;
  for (int j = 0; j < csc->cols; ++j) {
    const double xj = x[j];
    for (int p = csc->ptr[j]; p < csc->ptr[j + 1]; ++p) y[csc->idx[p]] += csc->val[p] * xj;
  }
  return PHFEM_OK;
}
