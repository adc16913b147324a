/*
 * phfem_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, single-threaded restatement of the reference C++ algorithm for the
 * edge-generation / red-refinement / assembly path (arXiv 2401.15557,
 * /root/reference/proj/src/{edge_topology,refine,assembly,sparse,parabolic}.cpp).
 * Each function cites the reference lines it restates.  It is the CHECKER for
 * the CUDA path: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load it.  The product library never
 * links or calls it.
 *
 * Pinned by (a) the reference's own known-answer tests re-encoded in
 * tests/test_oracle_kat.py (test_topology.cpp, test_assembly.cpp,
 * test_refine.cpp, test_parabolic.cpp) and (b) bit-for-bit comparison against
 * the reference sources themselves compiled in oracle/_ref (see Makefile,
 * tests/test_oracle_vs_ref.py).
 *
 * All outputs are malloc'd; free them with orc_free / the *_free helpers.
 * Status codes are the phfem_status values of include/phfem_gpu.h and `err`
 * receives the reference's exception text.
 */
#ifndef PHFEM_ORACLE_H
#define PHFEM_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#include "../include/phfem_fields.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_mesh {
  double* coords;     /* [nC][2] */
  int32_t* elements;  /* [nE][3] */
  int32_t* dirichlet; /* [nD][2] */
  int32_t* neumann;   /* [nN][2] */
  int32_t nC, nE, nD, nN;
} orc_mesh;

typedef struct orc_topology {
  int32_t nC, nE, E, n_interior, n_boundary, reserved;
  int32_t* edge_nodes;      /* [E][2] */
  int32_t* edge_elements;   /* [E][2] */
  int32_t* local_in_tplus;  /* [E] */
  int32_t* local_in_tminus; /* [E] */
  int32_t* interior_edges;
  int32_t* boundary_edges;
  int32_t* elem_edge;       /* [nE][3] e or ~e (t_minus) — a6 derived map   */
  int32_t* node_edge_start; /* [nC+1] edges grouped by max node             */
  int32_t* pair_offsets;    /* [nC+1] reference lookup table (by min node)  */
  int32_t* pair_entries;    /* [E][2] (max node, edge id)                   */
  int32_t* directed_offsets;/* [nC+1] by initial node                       */
  int32_t* directed_entries;/* [3nE][2] (end node, element)                 */
} orc_topology;

typedef struct orc_classification {
  int32_t nD, nN, E, L;
  int32_t* dirichlet_edge_ids;
  int32_t* neumann_edge_ids;
  int32_t* retained_edges;
  int32_t* retained_pos;
} orc_classification;

typedef struct orc_sparse {      /* CSR or CSC, by context */
  int32_t rows, cols;
  int64_t nnz;
  int32_t* ptr;                  /* [rows+1] (CSR) or [cols+1] (CSC) */
  int32_t* idx;
  double* val;
} orc_sparse;

void orc_free(void* p);
void orc_mesh_free(orc_mesh* m);
void orc_topology_free(orc_topology* t);
void orc_classification_free(orc_classification* c);
void orc_sparse_free(orc_sparse* s);

int orc_node_pair_to_edge(const orc_topology* t, int k, int l);
int orc_directed_pair_to_element(const orc_topology* t, int k, int l);

int orc_build_topology(const orc_mesh* mesh, orc_topology* out, char* err, size_t errlen);
/* SparseMatrix::from_triplets (sparse.cpp:30-97) -> Eigen ColMajor CSC       */
int orc_from_triplets(int32_t rows, int32_t cols, const int32_t* ri, const int32_t* ci,
                      const double* v, int64_t n, orc_sparse* out, char* err, size_t errlen);
int orc_classify_edges(const orc_topology* topo, const orc_mesh* mesh, orc_classification* out,
                       char* err, size_t errlen);
int orc_edge_lengths(const orc_mesh* mesh, const orc_topology* topo, double* out);
int orc_red_refine(const orc_mesh* mesh, const orc_topology* topo, orc_mesh* out, char* err,
                   size_t errlen);
int orc_orient_ccw(orc_mesh* mesh);
int orc_assemble_volume(const orc_mesh* mesh, const phfem_coeffs* c, double* B, double* D,
                        double* M, double* M0, char* err, size_t errlen);
/* C as the reference's triplet stream (row-major, = CSR) and as Eigen CSC. */
int orc_assemble_constraint(const orc_mesh* mesh, const orc_topology* topo,
                            const orc_classification* cls, orc_sparse* csr, orc_sparse* csc,
                            char* err, size_t errlen);
int orc_assemble_load(const orc_mesh* mesh, const phfem_field* f, double t, double* out,
                      char* err, size_t errlen);
int orc_assemble_neumann(const orc_mesh* mesh, const orc_topology* topo,
                         const orc_classification* cls, const phfem_field* g, double t,
                         double* out, char* err, size_t errlen);
int orc_assemble_dirichlet(const orc_mesh* mesh, const orc_topology* topo,
                           const orc_classification* cls, const phfem_field* uD, double t,
                           double* out, char* err, size_t errlen);
/* rhs for step n -> n+1 of solve_parabolic: M_minus W + [k/2 (...); (...)/2] */
int orc_cn_rhs(const orc_mesh* mesh, const orc_topology* topo, const orc_classification* cls,
               const phfem_coeffs* c, const phfem_field* f, const phfem_field* g,
               const phfem_field* uD, double k, int n, const double* state, double* rhs,
               char* err, size_t errlen);

/* ---- verification around the solve ---------------------- */
int orc_constraint_residual(const orc_sparse* csc, const double* U, const double* bd, double* out);
int orc_exact_multiplier(const orc_mesh* mesh, const orc_topology* topo,
                         const orc_classification* cls, const phfem_problem* p, double t,
                         double* out);
int orc_error_l2(const orc_mesh* mesh, const double* U, const phfem_problem* p, double t,
                 double* out, double* terms);
int orc_error_h1(const orc_mesh* mesh, const double* U, const phfem_problem* p, double t,
                 double* out, double* terms);
int orc_error_multiplier(const orc_sparse* csc, const double* B, const double* exact,
                         const double* discrete, int64_t n_exact, int64_t n_discrete, double* out,
                         char* err, size_t errlen);
int orc_midpoint_traces(const orc_topology* topo, const double* U, double* out);
int orc_csc_spmv(const orc_sparse* csc, const double* x, double* y);

#ifdef __cplusplus
}
#endif

#endif
