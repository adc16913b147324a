/*
 * phfem_gpu.h — the C ABI of the B200-native edge-generation / red-refinement /
 * assembly path of the lowest-order primal hybrid FEM (arXiv 2401.15557).
 *
 * Plain pointers and sizes only (no torch, no Eigen, no C++ types), so it can
 * be bound from C++, ctypes, cgo or JNI.  Every entry point replaces one
 * reference C++ function from /root/reference/proj/include/phfem (cited per
 * function); the C++ drop-in layer in include/phfem/ headers re-exposes the
 * reference signatures on top of this ABI.
 *
 * Conventions
 *  - ids are int32, 0-based, values IEEE fp64 — as in the reference.
 *  - "device" pointers live in HBM of the ctx's device; calls are asynchronous
 *    on the ctx stream except where a data-dependent size must come back
 *    (E, L, nnz), in which case the call synchronises the stream once.
 *  - Errors: every call returns a phfem_status.  The message retrievable with
 *    phfem_ctx_message() is the reference's exception text (1-based ids), so a
 *    wrapper rethrows the same exception type with the same what().
 *  - Library-owned outputs (data-dependent sizes) are released with the
 *    matching *_release(); fixed-size outputs (N = 3 nE blocks, vectors) are
 *    written into caller-provided device buffers.
 *  - There is no CPU fallback: without a usable sm_100 device every call
 *    returns PHFEM_ERR_NO_DEVICE / PHFEM_ERR_CUDA.
 */
#ifndef PHFEM_GPU_H
#define PHFEM_GPU_H

#include <stddef.h>
#include <stdint.h>

#include "phfem_fields.h"

#ifdef __cplusplus
extern "C" {
#endif

#define PHFEM_ABI_VERSION 1

typedef enum phfem_status {
  PHFEM_OK = 0,
  PHFEM_ERR_NONMANIFOLD = 1,        /* runtime_error     edge_topology.cpp:88-91   */
  PHFEM_ERR_DUP_DIRECTED = 2,       /* runtime_error     edge_topology.cpp:93-99   */
  PHFEM_ERR_NOT_AN_EDGE = 3,        /* runtime_error     edge_topology.cpp:151-153 */
  PHFEM_ERR_INTERIOR_BOUNDARY = 4,  /* runtime_error     edge_topology.cpp:154-157 */
  PHFEM_ERR_DEGENERATE = 5,         /* runtime_error     assembly.cpp:19-20        */
  PHFEM_ERR_NONFINITE = 6,          /* runtime_error     assembly.cpp:192-194,217-219 */
  PHFEM_ERR_INVALID_ARGUMENT = 7,   /* invalid_argument  assembly.cpp:46-50,81-84; parabolic.cpp:52 */
  PHFEM_ERR_OUT_OF_RANGE = 8,       /* out_of_range      sparse.cpp:21-24,114-116  */
  PHFEM_ERR_MISMATCH = 9,           /* runtime_error     assembly.cpp:148-149; refine.cpp:23 */
  PHFEM_ERR_OOM = 10,
  PHFEM_ERR_CUDA = 11,
  PHFEM_ERR_NO_DEVICE = 12,
  PHFEM_ERR_RUNTIME = 13            /* runtime_error (other) analysis.cpp:96      */
} phfem_status;

typedef struct phfem_ctx phfem_ctx;

/* ---- context ------------------------------------------------------------- */
int phfem_abi_version(void);
/* stream: a cudaStream_t (NULL = a new non-blocking stream owned by the ctx;
 * pass cudaStreamLegacy (0x1) for the legacy default stream). */
phfem_status phfem_ctx_create(int device, void* stream, phfem_ctx** out);
void phfem_ctx_destroy(phfem_ctx* ctx);
const char* phfem_ctx_message(const phfem_ctx* ctx);
void* phfem_ctx_stream(const phfem_ctx* ctx);
phfem_status phfem_ctx_sync(phfem_ctx* ctx);
/* stream-ordered device memory from the ctx pool */
phfem_status phfem_alloc(phfem_ctx* ctx, size_t bytes, void** out);
void phfem_free(phfem_ctx* ctx, void* ptr);
/* number of kernels this ctx launched so far (bench evidence) */
int64_t phfem_ctx_launches(const phfem_ctx* ctx);
/* Test knob: cap the edge pass's bucket width (bits of max node per bucket,
 * 1..8; default 8, or env PHFEM_EG_MAX_BS at ctx creation).  A cap below 8
 * makes every 256-node tile span several buckets (the multi-sub-bucket tile
 * path that meshes with > 56 packed key bits, e.g. the L13 square, take).
 * Outputs do not depend on it.                                              */
phfem_status phfem_ctx_set_eg_max_bs(phfem_ctx* ctx, int max_bs);
/* Per-launch CUDA-event timing on the ctx stream.  enable != 0 clears the
 * records and starts recording an event pair around every kernel launch;
 * read synchronises and returns the number of distinct kernel names with the
 * summed milliseconds and launch counts (names are static strings).        */
phfem_status phfem_ctx_profile(phfem_ctx* ctx, int enable);
int phfem_ctx_profile_read(phfem_ctx* ctx, int max_names, const char** names, double* ms,
                           int64_t* counts);

/* ---- mesh (reference Mesh, mesh.hpp:22-30; coords AoS like Vec2) --------- */
typedef struct phfem_mesh {
  double* coords;     /* [nC][2]  (x, y)                                     */
  int32_t* elements;  /* [nE][3]  CCW node triples                           */
  int32_t* dirichlet; /* [nD][2]  boundary pairs                             */
  int32_t* neumann;   /* [nN][2]                                             */
  int32_t nC, nE, nD, nN;
  int32_t owned;      /* 1 = library-owned (phfem_mesh_release frees it)     */
  int32_t reserved;
} phfem_mesh;
void phfem_mesh_release(phfem_ctx* ctx, phfem_mesh* mesh);

/* ---- topology (reference EdgeTopology, edge_topology.hpp:21-45) ---------- */
typedef struct phfem_topology {
  int32_t nC, nE, E, n_interior, n_boundary, reserved;
  int32_t* edge_nodes;      /* [E][2] directed (initial, end) of the t_plus cycle */
  int32_t* edge_elements;   /* [E][2] {t_plus, t_minus or -1}                     */
  int32_t* local_in_tplus;  /* [E]                                                */
  int32_t* local_in_tminus; /* [E]  -1 on boundary                                */
  int32_t* interior_edges;  /* [n_interior] ascending                             */
  int32_t* boundary_edges;  /* [n_boundary] ascending                             */
  /* a6: element -> edge map with orientation, elem_edge[3m+k] = id of the edge
   * opposite vertex k, encoded e (m is t_plus, sign +1) or ~e (m is t_minus,
   * sign -1).  Equivalent to node_pair_to_edge(t[(k+1)%3], t[(k+2)%3])
   * (refine.cpp:30-32, analysis.cpp:171-177) with the SPEC.md:393 sign.       */
  int32_t* elem_edge;       /* [nE][3]                                            */
  /* node_edge_start[v] = first id of the edges whose larger node is v (edge ids
   * are grouped by max node, ascending by min node inside a group): the device
   * lookup table behind node_pair_to_edge.                                      */
  int32_t* node_edge_start; /* [nC+1]                                             */
} phfem_topology;

/* build_topology (edge_topology.hpp:49; edge_topology.cpp:52-143) */
phfem_status phfem_build_topology(phfem_ctx* ctx, const phfem_mesh* mesh, phfem_topology* out);
void phfem_topology_release(phfem_ctx* ctx, phfem_topology* topo);

/* ---- classification (EdgeClassification, edge_topology.hpp:53-64) -------- */
#define PHFEM_CLS_DUP_NEUMANN 1 /* a Neumann pair is listed more than once */
typedef struct phfem_classification {
  int32_t nD, nN, E, L;
  int32_t flags, reserved;
  int32_t* dirichlet_edge_ids; /* [nD] mesh list order            */
  int32_t* neumann_edge_ids;   /* [nN] mesh list order            */
  int32_t* retained_edges;     /* [L] ascending                   */
  int32_t* retained_pos;       /* [E] position or -1 (Neumann)    */
  uint32_t* neumann_bits;      /* [ceil(E/32)] Neumann flag bitmap */
  int32_t* block_prefix;       /* internal: per-1024-edge-block (boundary, neumann) prefixes */
} phfem_classification;

/* classify_edges (edge_topology.hpp:64; edge_topology.cpp:145-177) */
phfem_status phfem_classify_edges(phfem_ctx* ctx, const phfem_topology* topo,
                                  const phfem_mesh* mesh, phfem_classification* out);
void phfem_classification_release(phfem_ctx* ctx, phfem_classification* cls);

/* ---- refinement (red_refine, refine.hpp:15; refine.cpp:7-53) -------------
 * out is library-owned: coords [nC+E], elements [4nE] (children 4m..4m+3),
 * boundary lists bisected in order (pairs resolved like midpoint_id,
 * refine.cpp:15-19: an unknown pair is the reference's mismatch error).      */
phfem_status phfem_red_refine(phfem_ctx* ctx, const phfem_mesh* mesh, const phfem_topology* topo,
                              phfem_mesh* out);

/* build_topology(red_refine(mesh)) computed from the parent topology with
 * two streaming passes and no sort; `fine` must be the
 * phfem_red_refine output of (parent, parent_topo).  Bit-identical to
 * phfem_build_topology(fine).                                               */
phfem_status phfem_refine_topology(phfem_ctx* ctx, const phfem_mesh* parent,
                                   const phfem_topology* parent_topo, const phfem_mesh* fine,
                                   phfem_topology* out);

/* One refinement level fused: given red_refine's output `fine` of (parent,
 * parent_topo) and the parent's classification, produce the fine mesh's
 * topology, classification and coupling matrix C (CSR) in one streaming
 * pass over the parent edges (fine Neumann edges are the halves of the
 * parent's).  Bit-identical to build_topology + classify_edges +
 * assemble_constraint on the fine mesh.                                     */
typedef struct phfem_csr phfem_csr;
phfem_status phfem_refine_level(phfem_ctx* ctx, const phfem_mesh* parent,
                                const phfem_topology* parent_topo,
                                const phfem_classification* parent_cls, const phfem_mesh* fine,
                                phfem_topology* topo, phfem_classification* cls, phfem_csr* C);

/* ---- orientation normalisation (config 4; not in the reference) ----------
 * Swaps v1<->v2 of every element with negative signed area, in place.       */
phfem_status phfem_orient_ccw(phfem_ctx* ctx, phfem_mesh* mesh);

/* ---- element blocks (assemble_volume_operators, assembly.hpp:68;
 * assembly.cpp:97-142).  Each output is [nE][9] fp64, the column-major 3x3
 * block of element m = exactly Eigen valuePtr()[9m .. 9m+8] of the
 * reference's block-diagonal CSC matrix (outer[c] = 3c, inner = 3m+i are
 * structural).  Any output pointer may be NULL to skip it.                   */
phfem_status phfem_assemble_volume(phfem_ctx* ctx, const phfem_mesh* mesh, const phfem_coeffs* c,
                                   double* B, double* D, double* M, double* M0);

/* ---- coupling matrix C (assemble_constraint, assembly.hpp:73-74;
 * assembly.cpp:144-168).  CSR L x N: rows = retained positions, 2 entries
 * (boundary) or 4 (interior), columns ascending.                            */
typedef struct phfem_csr {
  int32_t rows, cols;
  int64_t nnz;
  int32_t* row_ptr; /* [rows+1] */
  int32_t* col_idx; /* [nnz]    */
  double* values;   /* [nnz]    */
} phfem_csr;
phfem_status phfem_assemble_constraint(phfem_ctx* ctx, const phfem_mesh* mesh,
                                       const phfem_topology* topo,
                                       const phfem_classification* cls, phfem_csr* out);
void phfem_csr_release(phfem_ctx* ctx, phfem_csr* m);

/* Same matrix in the reference's Eigen ColMajor layout (from_triplets
 * sparse.cpp:30-97): outer [N+1], inner [nnz] (rows ascending per column).  */
typedef struct phfem_csc {
  int32_t rows, cols;
  int64_t nnz;
  int32_t* outer;
  int32_t* inner;
  double* values;
} phfem_csc;
phfem_status phfem_constraint_csc(phfem_ctx* ctx, const phfem_mesh* mesh,
                                  const phfem_topology* topo, const phfem_classification* cls,
                                  phfem_csc* out);
void phfem_csc_release(phfem_ctx* ctx, phfem_csc* m);

/* ---- generic COO -> CSC and the solve's operators ---------
 * SparseMatrix::from_triplets (sparse.hpp:55; sparse.cpp:30-97) on device
 * triplets [n]: first out-of-range entry -> PHFEM_ERR_OUT_OF_RANGE with the
 * reference's message; a strictly (row, col)-increasing buffer is stored
 * as-is, otherwise runs are summed in insertion order from 0.0; Eigen
 * ColMajor CSC out (library-owned, phfem_csc_release).  n < 2^31.          */
phfem_status phfem_from_triplets(phfem_ctx* ctx, int32_t rows, int32_t cols, const int32_t* ri,
                                 const int32_t* ci, const double* v, int64_t n, phfem_csc* out);
/* build_saddle_matrix (elliptic.hpp; elliptic.cpp:22-36): [[B+D+M, -C'],
 * [-C, 0]] from the device blocks ([nE][9]) and C in CSC.                  */
phfem_status phfem_saddle_matrix(phfem_ctx* ctx, int32_t nE, const double* B, const double* D,
                                 const double* M, const phfem_csc* C, phfem_csc* out);
/* step_matrix (parabolic.cpp:21-37): [[M0 + sign k/2 (B+D+M), -sign k/2 C'],
 * [-sign/2 C, 0]]; step_matrices = sign +1 (M_plus) and -1 (M_minus).       */
phfem_status phfem_step_matrix(phfem_ctx* ctx, int32_t nE, const double* B, const double* D,
                               const double* M, const double* M0, const phfem_csc* C, double k,
                               double sign, phfem_csc* out);

/* ---- load vectors --------------------------------------------------------
 * assemble_volume_operators + assemble_load (assembly.cpp:120-142, 179-203)
 * fused in one element pass: identical values, one read of the mesh.       */
phfem_status phfem_assemble_volume_load(phfem_ctx* ctx, const phfem_mesh* mesh,
                                        const phfem_coeffs* c, const phfem_field* f, double t,
                                        double* B, double* D, double* M, double* M0, double* load);
/* assemble_load (assembly.hpp:84; assembly.cpp:179-203) -> out[3nE]         */
phfem_status phfem_assemble_load(phfem_ctx* ctx, const phfem_mesh* mesh, const phfem_field* f,
                                 double t, double* out);
/* assemble_neumann (assembly.hpp:87-89; assembly.cpp:205-228).
 * accumulate = 0: out[3nE] is overwritten with LN (zeros elsewhere).
 * accumulate = 1: out += LN in the reference's elementwise "b + LN" order
 * (elliptic.cpp:54-55) — touching only the DOFs that carry a Neumann term.  */
phfem_status phfem_assemble_neumann(phfem_ctx* ctx, const phfem_mesh* mesh,
                                    const phfem_topology* topo, const phfem_classification* cls,
                                    const phfem_field* g, double t, double* out, int accumulate);
/* assemble_dirichlet (assembly.hpp:93-95; assembly.cpp:230-242) -> out[L]   */
phfem_status phfem_assemble_dirichlet(phfem_ctx* ctx, const phfem_mesh* mesh,
                                      const phfem_topology* topo,
                                      const phfem_classification* cls, const phfem_field* uD,
                                      double t, double* out);

/* ---- Crank-Nicolson right-hand side --------------------------------------
 * The reference forms it inline in solve_parabolic (parabolic.cpp:100-103):
 *   rhs = M_minus * [U; Lambda];  rhs.head += k/2 (b^n + LN^n + b^n+1 + LN^n+1);
 *   rhs.tail += (bD^n + bD^n+1)/2
 * with M_minus from step_matrices (parabolic.cpp:21-54).  The device path
 * recomputes the M_minus blocks from the geometry (bit-identical values) and
 * evaluates f, g, u_D at t_n = n k and t_{n+1}.  state = [U (3nE); Lambda (L)],
 * rhs same length.                                                            */
typedef struct phfem_cn_plan phfem_cn_plan;
phfem_status phfem_cn_plan_create(phfem_ctx* ctx, const phfem_mesh* mesh,
                                  const phfem_topology* topo, const phfem_classification* cls,
                                  const phfem_coeffs* c, const phfem_field* f,
                                  const phfem_field* g, const phfem_field* uD, double k,
                                  phfem_cn_plan** out);
/* rhs for the step t_n -> t_{n+1} (the reference's loop index n+1).         */
phfem_status phfem_cn_rhs(phfem_ctx* ctx, phfem_cn_plan* plan, int n, const double* state,
                          double* rhs);
void phfem_cn_plan_destroy(phfem_ctx* ctx, phfem_cn_plan* plan);

/* ---- fused pipeline (the bench step) --------------------------------------
 * input mesh -> [build_topology -> classify -> red_refine] x levels ->
 * build_topology -> classify -> B, D, M, M0, C (CSR), load = b + LN
 * (elliptic.cpp:54-55), bD.  All outputs library-owned in `out`.           */
typedef struct phfem_pipeline_out {
  phfem_mesh mesh;             /* final (refined) mesh                      */
  phfem_topology topo;
  phfem_classification cls;
  phfem_csr C;
  double* B;                   /* [nE][9] */
  double* D;
  double* M;
  double* M0;
  double* load;                /* [3nE] b + LN */
  double* bd;                  /* [L]         */
} phfem_pipeline_out;
phfem_status phfem_pipeline(phfem_ctx* ctx, const phfem_mesh* mesh_in, int levels,
                            const phfem_coeffs* c, const phfem_field* f, const phfem_field* g,
                            const phfem_field* uD, double t, phfem_pipeline_out* out);
/* flags: PHFEM_PIPE_GENERIC_EG = run the sort-based build_topology on every
 * refined mesh instead of phfem_refine_topology (same results).            */
#define PHFEM_PIPE_GENERIC_EG 1
phfem_status phfem_pipeline_ex(phfem_ctx* ctx, const phfem_mesh* mesh_in, int levels,
                               const phfem_coeffs* c, const phfem_field* f, const phfem_field* g,
                               const phfem_field* uD, double t, int flags, phfem_pipeline_out* out);
void phfem_pipeline_release(phfem_ctx* ctx, phfem_pipeline_out* out);

/* Host-buffer variant (what a reference caller sees): the input mesh comes
 * from HOST memory (copied in by the call), outputs land in `out` on the
 * device; phfem_pipeline_download then copies every output into caller-owned
 * HOST buffers sized from `out` (any destination may be NULL to skip it).   */
phfem_status phfem_pipeline_from_host(phfem_ctx* ctx, const double* coords,
                                      const int32_t* elements, const int32_t* dirichlet,
                                      const int32_t* neumann, int32_t nC, int32_t nE, int32_t nD,
                                      int32_t nN, int levels, const phfem_coeffs* c,
                                      const phfem_field* f, const phfem_field* g,
                                      const phfem_field* uD, double t, phfem_pipeline_out* out);
typedef struct phfem_pipeline_host {
  double* coords; int32_t* elements; int32_t* dirichlet; int32_t* neumann;
  int32_t* edge_nodes; int32_t* edge_elements; int32_t* local_in_tplus; int32_t* local_in_tminus;
  int32_t* interior_edges; int32_t* boundary_edges; int32_t* elem_edge;
  int32_t* dirichlet_edge_ids; int32_t* neumann_edge_ids; int32_t* retained_edges;
  int32_t* retained_pos;
  int32_t* C_row_ptr; int32_t* C_col_idx; double* C_values;
  double* B; double* D; double* M; double* M0; double* load; double* bd;
} phfem_pipeline_host;
phfem_status phfem_pipeline_download(phfem_ctx* ctx, const phfem_pipeline_out* out,
                                     const phfem_pipeline_host* dst);
/* bytes phfem_pipeline_download moves for a given `out` and selection */
int64_t phfem_pipeline_download_bytes(const phfem_pipeline_out* out, const phfem_pipeline_host* dst);

/* ---- support of the C++ drop-in layer (paper_2401_15557_b200/dropin, see
 * INTEGRATION.md): host-built reference objects -> device, the reference's
 * lookup tables, and the std::function field path ------------------------
 *
 * A topology whose edge_nodes / edge_elements / local_in_tplus /
 * local_in_tminus / interior / boundary arrays (and E, n_interior,
 * n_boundary) the caller filled in device memory gets elem_edge and
 * node_edge_start computed and is checked against the mesh: every element
 * slot covered exactly once by an edge with the element's own vertex pair
 * (else PHFEM_ERR_MISMATCH, the reference's "topology does not match mesh",
 * refine.cpp:21-25), edges in canonical (max, min) order.                  */
phfem_status phfem_topology_derive(phfem_ctx* ctx, const phfem_mesh* mesh, phfem_topology* topo);

/* EdgeTopology::pair_offsets / pair_entries / directed_offsets /
 * directed_entries (edge_topology.hpp:38-44; built at edge_topology.cpp:
 * 117-140): CSR by smaller node of (larger node, edge id), ids ascending;
 * CSR by initial node of (end node, element), emission (element) order.
 * Device buffers: offsets [nC+1], pair_entries [E][2], directed_entries
 * [3nE][2].                                                                 */
phfem_status phfem_topology_tables(phfem_ctx* ctx, const phfem_mesh* mesh,
                                   const phfem_topology* topo, int32_t* pair_offsets,
                                   int32_t* pair_entries, int32_t* directed_offsets,
                                   int32_t* directed_entries);

/* edge_lengths (edge_topology.hpp:67; edge_topology.cpp:179-186) -> out[E] */
phfem_status phfem_edge_lengths(phfem_ctx* ctx, const phfem_mesh* mesh, const phfem_topology* topo,
                                double* out);

/* Sample points of the reference's std::function fields, which cannot run on
 * the device.  LOAD: [3nE][2] edge midpoints per element (assembly.cpp:36);
 * NEUMANN: [nN][4] (midpoint, outward unit normal) in Neumann-list order
 * (:211-215); DIRICHLET: [nD][2] midpoints in Dirichlet-list order (:236).
 * The caller evaluates f / g / u_D there and passes the values to:          */
#define PHFEM_POINTS_LOAD 0
#define PHFEM_POINTS_NEUMANN 1
#define PHFEM_POINTS_DIRICHLET 2
phfem_status phfem_field_points(phfem_ctx* ctx, const phfem_mesh* mesh, const phfem_topology* topo,
                                const phfem_classification* cls, int which, double* out);
/* assemble_load / assemble_neumann / assemble_dirichlet with the field given
 * as sampled values (same kernels, same operation order, same errors).      */
phfem_status phfem_assemble_load_sampled(phfem_ctx* ctx, const phfem_mesh* mesh,
                                         const double* samples, double* out);
phfem_status phfem_assemble_neumann_sampled(phfem_ctx* ctx, const phfem_mesh* mesh,
                                            const phfem_topology* topo,
                                            const phfem_classification* cls,
                                            const double* samples, double* out, int accumulate);
phfem_status phfem_assemble_dirichlet_sampled(phfem_ctx* ctx, const phfem_mesh* mesh,
                                              const phfem_topology* topo,
                                              const phfem_classification* cls,
                                              const double* samples, double* out);

/* ---- multi-GPU (host orchestration paper_2401_15557_b200/dist.py)
 * Elements are split into contiguous ranges, max nodes into contiguous key
 * ranges (so every rank owns a contiguous range of canonical edge ids).
 * Not in the reference (single-threaded); the concatenation of the ranks'
 * outputs equals the single-GPU outputs bit for bit.
 *
 * Directed occurrences of elements [elo, ehi) as records {max, min, 3m+s,
 * dir}, grouped by the rank owning the max node (splits [W+1], device):
 * counts[W] always; with send != NULL also offsets[W+1] and the records. */
phfem_status phfem_dist_occurrences(phfem_ctx* ctx, const int32_t* elements, int32_t elo,
                                    int32_t ehi, const int32_t* splits, int32_t W, int32_t* counts,
                                    int32_t* offsets, int32_t* send);
/* red_refine of the rank's elements (local arrays [n][3] + their elem_edge):
 * children 4m..4m+3 (refine.cpp:28-37) -> children[4n][3]; the midpoints of
 * a range of edges (refine.cpp:16-19) -> out[E][2] (all-gathered by dist.py) */
phfem_status phfem_dist_children(phfem_ctx* ctx, const int32_t* elements, const int32_t* elem_edge,
                                 int32_t n, int32_t nC, int32_t* children);
phfem_status phfem_dist_midpoints(phfem_ctx* ctx, const double* coords, const int32_t* edge_nodes,
                                  int32_t E, double* out);
/* build_topology of the records of one max-node range [node_lo, node_hi):
 * out gets the range's edges (rank-local ids, global node / element ids),
 * node_edge_start for the range's nodes; pairs[2E][2] the (element slot
 * 3m+l, edge or ~edge) of every occurrence (slot -1 = none) instead of
 * elem_edge.                                                                */
phfem_status phfem_dist_dedup(phfem_ctx* ctx, const int32_t* recs, int64_t n, int32_t node_lo,
                              int32_t node_hi, int32_t nC_all, int32_t nE_all, phfem_topology* out,
                              int32_t* pairs);
/* The same with the rank's own element range [self_lo, self_hi): their
 * entries go straight into self_elem_edge ([self_hi - self_lo][3], LOCAL ids
 * e / ~e: re-base with phfem_dist_add_offset(..., 2)); pairs then holds only
 * the *n_pairs entries of other ranks' elements (compact, any order).       */
phfem_status phfem_dist_dedup_ex(phfem_ctx* ctx, const int32_t* recs, int64_t n, int32_t node_lo,
                                 int32_t node_hi, int32_t nC_all, int32_t nE_all, int32_t self_lo,
                                 int32_t self_hi, int32_t* self_elem_edge, phfem_topology* out,
                                 int32_t* pairs, int64_t* n_pairs);
/* pairs -> global edge ids (+E0) routed to the element owner (esplits[W+1]);
 * the receiver writes them into its elem_edge ([3(ehi-elo)]).  Pairs of the
 * caller's own elements [self_lo, self_hi) are written to self_elem_edge
 * directly and not sent (self_lo = self_hi: route everything).            */
phfem_status phfem_dist_route_pairs(phfem_ctx* ctx, const int32_t* pairs, int64_t n, int32_t E0,
                                    const int32_t* esplits, int32_t W, int32_t* counts,
                                    int32_t* offsets, int32_t* send, int32_t self_lo,
                                    int32_t self_hi, int32_t* self_elem_edge);
phfem_status phfem_dist_apply_pairs(phfem_ctx* ctx, const int32_t* recv, int64_t n, int32_t elo,
                                    int32_t* elem_edge);
/* a[i] += off (only_nonneg 1: where a[i] >= 0; 2: signed ids e / ~e, i.e.
 * e + off or ~(~a[i] + off)) — re-basing local ids                          */
phfem_status phfem_dist_add_offset(phfem_ctx* ctx, int32_t* a, int64_t n, int32_t off,
                                   int only_nonneg);
/* boundary pairs (global list, positions list_base..) whose max node this
 * rank owns -> global edge ids (else -1); the first error as (position << 2
 * | 0 not an edge / 1 interior) via atomicMin on *err (init ~0).            */
phfem_status phfem_dist_resolve(phfem_ctx* ctx, const phfem_topology* part, int32_t node_lo,
                                int32_t E0, const int32_t* pairs, int32_t n, int32_t list_base,
                                int32_t* ids, unsigned long long* err);
/* classification of the rank's edges from its Dirichlet / Neumann edges
 * (LOCAL ids, list order): rank-local retained_pos / retained_edges / id
 * lists / bitmap.  E0 = global id of the part's first edge (the part's
 * boundary list holds global ids after phfem_dist_add_offset).              */
phfem_status phfem_dist_classify(phfem_ctx* ctx, const phfem_topology* part, int32_t E0,
                                 const int32_t* dir_ids, int32_t nD, const int32_t* neu_ids,
                                 int32_t nN, phfem_classification* out);
/* Neumann edges: the owner writes rows {a, b, t_plus, led} of table[nN][4]
 * (others zero; a sum all-reduce completes it), then every rank adds the
 * Neumann load of its elements [elo, ehi) to its local load vector.         */
phfem_status phfem_dist_neumann_table(phfem_ctx* ctx, const phfem_topology* part, int32_t E0,
                                      const int32_t* neu_ids, int32_t nN, int32_t* table);
phfem_status phfem_dist_neumann_apply(phfem_ctx* ctx, const phfem_mesh* mesh, const int32_t* table,
                                      int32_t nN, int32_t dup, int32_t elo, int32_t ehi,
                                      const phfem_field* g, double t, double* load_local);

/* ---- verification around the solve (csrc/verify.cu) ------
 * Values bit-identical to the reference's; the two error norms sum their
 * per-element terms in a fixed device tree instead of element order (the
 * optional `terms` [nE] output is bit-identical, the norm agrees to
 * rounding).  Scalar results are returned through host pointers (the call
 * synchronises the ctx stream).
 * ||C U + bD||_inf (tools/main.cpp:205-207); bd may be NULL (no addition).  */
phfem_status phfem_constraint_residual(phfem_ctx* ctx, const phfem_csr* C, const double* primal,
                                       const double* bd, double* out);
/* exact_multiplier (analysis.hpp; analysis.cpp:26-39) -> out[L]; the problem's
 * coefficients must be PHFEM_COEFF_CONST (ProblemCoefficients).            */
phfem_status phfem_exact_multiplier(phfem_ctx* ctx, const phfem_mesh* mesh,
                                    const phfem_topology* topo, const phfem_classification* cls,
                                    const phfem_problem* problem, double t, double* out);
/* error_l2 / error_h1 (analysis.cpp:41-80) of primal[3nE] at time t.        */
phfem_status phfem_error_l2(phfem_ctx* ctx, const phfem_mesh* mesh, const double* primal,
                            const phfem_problem* problem, double t, double* out, double* terms);
phfem_status phfem_error_h1(phfem_ctx* ctx, const phfem_mesh* mesh, const double* primal,
                            const phfem_problem* problem, double t, double* out, double* terms);
/* error_multiplier(exact, discrete, C, B) (analysis.cpp:82-98): C from the
 * classification (assemble_constraint), B the stiffness blocks [nE][9];
 * sizes differ or != L -> INVALID_ARGUMENT "size mismatch"; no B_ii > 0 ->
 * RUNTIME "all diagonal entries of B vanish".                               */
phfem_status phfem_error_multiplier(phfem_ctx* ctx, const phfem_mesh* mesh,
                                    const phfem_topology* topo, const phfem_classification* cls,
                                    const double* B, const double* exact, const double* discrete,
                                    int64_t n_exact, int64_t n_discrete, double* out);
/* hybrid_midpoint_traces (analysis.cpp:113-125) -> out[E].                  */
phfem_status phfem_midpoint_traces(phfem_ctx* ctx, const phfem_topology* topo,
                                   const double* primal, double* out);
/* CSC -> CSR (columns ascending per row; library-owned, phfem_csr_release)
 * and y = A x with Eigen's ColMajor SpMV bits (each y_i summed from 0.0 over
 * ascending columns) — e.g. M_minus W on phfem_step_matrix's output.        */
phfem_status phfem_csc_to_csr(phfem_ctx* ctx, const phfem_csc* A, phfem_csr* out);
phfem_status phfem_csr_spmv(phfem_ctx* ctx, const phfem_csr* A, const double* x, double* y);

/* ---- on-disk formats (csrc/io.cu) --------------------------
 * load_mesh (mesh.hpp; mesh.cpp:114-150) from the four text files' bytes
 * (dirichlet / neumann may be empty) -> a library-owned device mesh, with the
 * reference's validation order and messages (PHFEM_ERR_RUNTIME, 1-based
 * rows); boundary pairs normalised to their element-cycle direction.
 * load_mesh_dir reads DIR/{coordinates,elements,dirichlet,neumann}.dat (the
 * last two optional, "cannot open DIR/name" otherwise).                    */
phfem_status phfem_mesh_load_text(phfem_ctx* ctx, const char* coordinates, size_t coordinates_len,
                                  const char* elements, size_t elements_len, const char* dirichlet,
                                  size_t dirichlet_len, const char* neumann, size_t neumann_len,
                                  phfem_mesh* out);
phfem_status phfem_mesh_load_dir(phfem_ctx* ctx, const char* dir, phfem_mesh* out);
/* save_mesh (mesh.cpp:170-180): which 0 coordinates ("%.17g %.17g"), 1
 * elements, 2 dirichlet, 3 neumann (1-based ids) -> *out (malloc'd, free with
 * phfem_text_free), *len bytes.  save_mesh_dir writes the files.           */
phfem_status phfem_mesh_format(phfem_ctx* ctx, const phfem_mesh* mesh, int which, char** out,
                               size_t* len);
void phfem_text_free(char* text);
phfem_status phfem_mesh_save_dir(phfem_ctx* ctx, const phfem_mesh* mesh, const char* dir);
/* The CLI's topology CSV (tools/main.cpp:302-323): header, then per edge
 * "e,a,b,t_plus,t_minus,led,led_tn,length" (1-based, 0 for no t_minus,
 * length "%.10g").                                                          */
phfem_status phfem_topology_csv(phfem_ctx* ctx, const phfem_mesh* mesh, const phfem_topology* topo,
                                char** out, size_t* len);
phfem_status phfem_topology_csv_file(phfem_ctx* ctx, const phfem_mesh* mesh,
                                     const phfem_topology* topo, const char* path);
/* printf("%.<precision>g") of n device doubles on the device (the formatter
 * behind the two calls above; precision 1..17): out = n 32-byte slots,
 * lens = bytes used per slot.  Test entry point.                           */
phfem_status phfem_format_g(phfem_ctx* ctx, const double* vals, int64_t n, int precision,
                            char* out, int32_t* lens);
/* the same formatter on the host (out >= 32 bytes): returns the length.     */
int phfem_format_g_host(double v, int precision, char* out);

/* Distributed refined level (§8(e) with SURVEY f1): the rank's part of the
 * fine topology straight from its parent part `ppart` (parent edges
 * [E0p, E0p + ppart->E), lists with global ids) and the all-gathered parent
 * elem_edge / elements — no sort, no occurrence exchange.  Fine node range
 * [node_lo, node_hi) with node_hi = nc + E0p + E; local fine ids (re-base as
 * for phfem_dist_dedup); *pairs_out (ctx memory, 2 x out->E int2, free with
 * phfem_free) = (fine slot, f / ~f) per fine edge for
 * phfem_dist_route_pairs; mids (nullable, [E][2]) = the rank's midpoints.
 * C (nullable): also the rank's rows of the fine C in CSR (local rows and
 * row pointers, global columns; re-base by the rank's row / nnz offsets),
 * fused as on one GPU, from the parent Neumann edges neu_parent_ids (global
 * ids, all ranks' list).                                                   */
phfem_status phfem_dist_refine_level(phfem_ctx* ctx, const phfem_topology* ppart, int32_t E0p,
                                     const int32_t* elem_edge_all, const int32_t* elements_all,
                                     int32_t nE_all, const double* coords, int32_t nc,
                                     int32_t node_lo, int32_t node_hi,
                                     const int32_t* neu_parent_ids, int32_t nN_parent,
                                     phfem_topology* out, int32_t** pairs_out, double* mids,
                                     phfem_csr* C);
/* The same with the rank's own FINE element range [self_lo, self_hi): their
 * elem_edge entries are written straight into self_elem_edge
 * ([self_hi - self_lo][3], LOCAL ids f / ~f: re-base with
 * phfem_dist_add_offset(..., 2) once the rank's fine edge offset is known);
 * *pairs_out then holds only the *n_pairs pairs of other ranks' elements
 * (compact, any order) for phfem_dist_route_pairs.                          */
phfem_status phfem_dist_refine_level_ex(phfem_ctx* ctx, const phfem_topology* ppart, int32_t E0p,
                                        const int32_t* elem_edge_all, const int32_t* elements_all,
                                        int32_t nE_all, const double* coords, int32_t nc,
                                        int32_t node_lo, int32_t node_hi,
                                        const int32_t* neu_parent_ids, int32_t nN_parent,
                                        int32_t self_lo, int32_t self_hi, int32_t* self_elem_edge,
                                        phfem_topology* out, int32_t** pairs_out, int64_t* n_pairs,
                                        double* mids, phfem_csr* C);

/* Distributed refined level, halo form (dist.py _refine_sort_free; replaces
 * the all-gathers of the parent arrays and midpoints of the _ex variant):
 *  1. element owner: phfem_dist_side_records — for every slot k of its n
 *     elements one 16-byte record {e << 1 | (element is t_minus of e), the
 *     partner edges at local k+1 / k+2 (signed), vertex k} routed by parent
 *     edge id to its owner (esplits: first global edge id per rank, W + 1);
 *     counts / offsets / send as phfem_dist_occurrences (send NULL: counts);
 *  2. edge owner: phfem_dist_side_apply — recv -> side[2 (e - E0) + s]
 *     ([2 E][4] int32, s = 0 t_plus / 1 t_minus);
 *  3. edge owner: phfem_dist_refine_level_side — the fine topology part (as
 *     phfem_dist_refine_level, local fine ids), rk[E] (in-group rank bytes of
 *     each owned parent edge), the owned midpoints into coords_fine[nc + E0p
 *     + le] (coords_fine: the rank's fine coordinate array; coords = the
 *     replicated parent coordinates), C's rows when C != NULL;
 *  4. edge owner: phfem_dist_start_records — for each owned parent edge and
 *     each of its elements a 12-byte record {slot 3 m + l, group start
 *     fine_nes[le + nes_off] (global once re-based), rank byte} routed by
 *     element to its owner (psplits: first parent element per rank);
 *  5. element owner: phfem_dist_start_apply — recv -> gs / grk per slot
 *     ([3 n] int32 / uint8, elements from elo);
 *  6. element owner: phfem_dist_children_slots — children rows and their
 *     elem_edge (global ids) as k_refine_children, from gs / grk, plus the
 *     midpoints of its elements' edges into coords_fine (same bits as 3.). */
phfem_status phfem_dist_side_records(phfem_ctx* ctx, const int32_t* elements, const int32_t* elem_edge,
                                     int32_t n, const int32_t* esplits, int32_t W, int32_t* counts,
                                     int32_t* offsets, int32_t* send);
phfem_status phfem_dist_side_apply(phfem_ctx* ctx, const int32_t* recv, int64_t n, int32_t E0, int32_t E,
                                   int32_t* side);
phfem_status phfem_dist_refine_level_side(phfem_ctx* ctx, const phfem_topology* ppart, int32_t E0p,
                                          const int32_t* side, const double* coords, int32_t nc,
                                          int32_t node_lo, int32_t node_hi, int32_t nE_all,
                                          const int32_t* neu_parent_ids, int32_t nN_parent,
                                          phfem_topology* out, uint8_t* rk, double* coords_fine, phfem_csr* C);
/* phfem_dist_refine_level_side in two halves, so that the rank's fine
 * offsets are known before the level kernel writes: _count (tile counts from
 * the side records; Ef = the rank's fine edges, nneu = its parent Neumann
 * edges when with_C; synchronises; *plan for _run) and _run (f_off = the
 * rank's first global fine edge id, nnz_off = its first C entry, written
 * straight into the fine lists, node_edge_start and C's row pointers; frees
 * the plan).  phfem_dist_classify_ex: retained_pos / retained_edges with the
 * rank's first retained row r_off and first edge id e_off added.           */
phfem_status phfem_dist_level_count(phfem_ctx* ctx, const phfem_topology* ppart, int32_t E0p, const int32_t* side,
                                    const int32_t* neu_parent_ids, int32_t nN_parent, int with_C, int32_t* Ef,
                                    int32_t* nneu, void** plan);
phfem_status phfem_dist_level_run(phfem_ctx* ctx, void* plan, const double* coords, int32_t nc, int32_t node_lo,
                                  int32_t node_hi, int32_t nE_all, int32_t f_off, int32_t nnz_off,
                                  phfem_topology* out, uint8_t* rk, double* coords_fine, phfem_csr* C);
/* _run_ex: also the rank's rows of the classification on the last level —
 * retained_pos [Ef] (global rows from r_off, -1 for Neumann) and
 * retained_edges [Ef - 2 nneu] (global fine ids), ctx memory, both or
 * neither, C required; phfem_dist_classify_given then completes the
 * classification around them (Neumann bitmap, the rank's id lists, flags)
 * and takes ownership.  phfem_dist_children_slots_ex: midpoints of the parent
 * edges [own_lo, own_hi) are skipped (the rank's level kernel wrote them).  */
/* Local mode of the halo exchanges (the C++ orchestration's default): the
 * side record / group start of an element slot whose edge AND element belong
 * to the same rank is not stored at all — the level kernel / children pass
 * gather it from the rank's own arrays instead (at W = 1 no record moves).
 * phfem_dist_local names those arrays: the rank's elements and elem_edge
 * (global signed ids) for its global element range [elo, ehi).            */
typedef struct phfem_dist_local {
  const int32_t* elements;
  const int32_t* elem_edge;
  int32_t elo, ehi;
  int32_t no_remote; /* 1: no other rank holds elements (W = 1): no side record exists */
  int32_t reserved;
} phfem_dist_local;
phfem_status phfem_dist_side_p2p_ex(phfem_ctx* ctx, const int32_t* elements, const int32_t* elem_edge, int32_t n,
                                    const int32_t* esplits, int32_t W, int32_t self, int32_t* const* peer_side,
                                    int32_t* remote, int skip_self);
phfem_status phfem_dist_start_p2p_ex(phfem_ctx* ctx, const phfem_topology* ppart, const int32_t* fine_nes,
                                     int32_t nes_off, const uint8_t* rk, const int32_t* psplits, int32_t W,
                                     int32_t self, int32_t* const* peer_gs, uint8_t* const* peer_grk,
                                     int32_t* remote, int skip_self);
phfem_status phfem_dist_level_count_ex(phfem_ctx* ctx, const phfem_topology* ppart, int32_t E0p, const int32_t* side,
                                       const phfem_dist_local* local, const int32_t* neu_parent_ids,
                                       int32_t nN_parent, int with_C, int32_t* Ef, int32_t* nneu, void** plan);
phfem_status phfem_dist_level_run_ex(phfem_ctx* ctx, void* plan, const double* coords, int32_t nc, int32_t node_lo,
                                     int32_t node_hi, int32_t nE_all, int32_t f_off, int32_t nnz_off, int32_t r_off,
                                     phfem_topology* out, uint8_t* rk, double* coords_fine, phfem_csr* C,
                                     int32_t* retained_pos, int32_t* retained_edges);
phfem_status phfem_dist_classify_given(phfem_ctx* ctx, const phfem_topology* part, const int32_t* dir_ids_local,
                                       int32_t nD, const int32_t* neu_ids_local, int32_t nN, int32_t* retained_pos,
                                       int32_t* retained_edges, int32_t L, phfem_classification* out);
/* children_slots_ex: fine_nes != NULL (local mode): the group starts / rank
 * bytes of the slots whose parent edge is the rank's own (own_lo..own_hi)
 * come from its fine node_edge_start (fine_nes[e - own_lo + nes_off], as
 * phfem_dist_start_p2p) and rk[e - own_lo], not from gs / grk.             */
phfem_status phfem_dist_children_slots_ex(phfem_ctx* ctx, const int32_t* elements, const int32_t* elem_edge,
                                          int32_t n, const int32_t* gs, const uint8_t* grk, int32_t nc,
                                          int32_t own_lo, int32_t own_hi, const int32_t* fine_nes, int32_t nes_off,
                                          const uint8_t* rk, double* coords_fine, int32_t* children,
                                          int32_t* fine_elem_edge);
/* phfem_assemble_volume_load in two halves (_start: reset the ctx error block
 * and launch, no synchronisation; _finish: fetch it and raise the reference's
 * errors) so the caller can enqueue other work while the element pass runs;
 * nothing in between may use the ctx error block.                          */
phfem_status phfem_dist_volume_start(phfem_ctx* ctx, const phfem_mesh* mesh, const phfem_coeffs* c,
                                     const phfem_field* f, double t, double* B, double* D, double* M, double* M0,
                                     double* load);
phfem_status phfem_dist_volume_finish(phfem_ctx* ctx);
/* assemble_dirichlet of a rank whose retained positions start at r_off:
 * out[0 .. L) holds rows r_off .. r_off + L                               */
phfem_status phfem_dist_dirichlet(phfem_ctx* ctx, const phfem_mesh* mesh, const phfem_topology* part,
                                  const phfem_classification* cls, const phfem_field* uD, double t, int32_t r_off,
                                  double* out);
phfem_status phfem_dist_classify_ex(phfem_ctx* ctx, const phfem_topology* part, int32_t E0,
                                    const int32_t* dir_ids_local, int32_t nD, const int32_t* neu_ids_local,
                                    int32_t nN, int32_t r_off, int32_t e_off, phfem_classification* out);
phfem_status phfem_dist_start_records(phfem_ctx* ctx, const phfem_topology* ppart, const int32_t* fine_nes,
                                      int32_t nes_off, const uint8_t* rk, const int32_t* psplits, int32_t W,
                                      int32_t* counts, int32_t* offsets, int32_t* send);
phfem_status phfem_dist_start_apply(phfem_ctx* ctx, const int32_t* recv, int64_t n, int32_t elo, int32_t* gs,
                                    uint8_t* grk);
phfem_status phfem_dist_children_slots(phfem_ctx* ctx, const int32_t* elements, const int32_t* elem_edge,
                                       int32_t n, const int32_t* gs, const uint8_t* grk, int32_t nc,
                                       double* coords_fine, int32_t* children, int32_t* fine_elem_edge);

/* Peer-window forms of steps 1-2 and 4-5 above (one kernel each: the record
 * is computed and stored straight into its final slot of the owner's array,
 * mapped into this rank — CUDA IPC across GPUs over NVLink, or the emulated
 * ranks' arrays on one GPU): peer_side[d] = rank d's side array ([2 E_d][4]),
 * peer_gs[d] / peer_grk[d] = rank d's per-slot arrays; W device pointers
 * each, in device memory.  remote[W] (device) receives the number of records
 * this rank stored into each other rank's window.  The caller fences (kernel
 * completion on every rank) before the owners read.                        */
phfem_status phfem_dist_side_p2p(phfem_ctx* ctx, const int32_t* elements, const int32_t* elem_edge, int32_t n,
                                 const int32_t* esplits, int32_t W, int32_t self, int32_t* const* peer_side,
                                 int32_t* remote);
phfem_status phfem_dist_start_p2p(phfem_ctx* ctx, const phfem_topology* ppart, const int32_t* fine_nes,
                                  int32_t nes_off, const uint8_t* rk, const int32_t* psplits, int32_t W,
                                  int32_t self, int32_t* const* peer_gs, uint8_t* const* peer_grk,
                                  int32_t* remote);

/* Distributed input level with peer windows (dist.py _edge_generation): key
 * ranges aligned to 256-node tiles so that bucket b = max >> bs (bs =
 * phfem_dist_bucket_bits, the same on every rank) has one owner (bsplits:
 * first bucket per rank, W + 1, last = NB = ceil(nC / 2^bs)).
 *  phfem_dist_bucket_hist    own occurrences per global bucket -> hist[NB]
 *                            (the reference's node-range error, global ids);
 *  phfem_dist_bucket_cursors from the all-gathered hist_all[W][NB]: this
 *                            rank's cursor in every bucket (owner-local slot
 *                            of its first item), its own bucket offsets
 *                            boff_me[nb + 1] and item count (synchronises);
 *  phfem_dist_scatter_p2p    packs every own occurrence and stores it into
 *                            the owner's item array (peer_items[W], device
 *                            pointer array) at its cursor — MSD bucket
 *                            scatter fused with the exchange;
 *  phfem_dist_dedup_items    the owner's tile / emit passes over its
 *                            bucketed items (as phfem_dist_dedup_ex).       */
int phfem_dist_bucket_bits(int32_t nC_all, int32_t nE_all);
/* the dedup's pairs of other ranks' elements, re-based by E0, stored straight
 * into the element owners' elem_edge (peer_ee[W]; esplits: first element per
 * rank) — phfem_dist_route_pairs + the all-to-all + phfem_dist_apply_pairs
 * in one kernel                                                             */
phfem_status phfem_dist_pairs_p2p(phfem_ctx* ctx, const int32_t* pairs, int64_t n, int32_t E0,
                                  const int32_t* esplits, int32_t W, int32_t self, int32_t* const* peer_ee,
                                  int32_t* remote);
phfem_status phfem_dist_bucket_hist(phfem_ctx* ctx, const int32_t* elements, int32_t n, int32_t elo,
                                    int32_t nC_all, int32_t nE_all, int32_t* hist);
phfem_status phfem_dist_bucket_cursors(phfem_ctx* ctx, const int32_t* hist_all, int32_t W, int64_t NB, int32_t me,
                                       const int32_t* bsplits, int32_t* cursor, int32_t* boff_me,
                                       int64_t* n_items_me);
phfem_status phfem_dist_scatter_p2p(phfem_ctx* ctx, const int32_t* elements, int32_t n, int32_t elo,
                                    int32_t nC_all, int32_t nE_all, int32_t* cursor, const int32_t* bsplits,
                                    int32_t W, int32_t me, uint64_t* const* peer_items, int32_t* remote);
phfem_status phfem_dist_dedup_items(phfem_ctx* ctx, uint64_t* items, int64_t n, const int32_t* boff,
                                    int32_t node_lo, int32_t node_hi, int32_t nC_all, int32_t nE_all,
                                    int32_t self_lo, int32_t self_hi, int32_t* self_elem_edge,
                                    phfem_topology* out, int32_t* pairs, int64_t* n_pairs);

/* ---- sharded pipeline, host orchestration in C++ (csrc/dist_run.cu) -------
 * The whole distributed step (dist.py distributed_pipeline: peer-window input
 * level, `levels` sort-free halo-form refinements, classification, C, bD,
 * blocks, load = b + LN) in one call, with no Python between the kernels.
 * Communicator: _local(W) emulates W ranks in this process on one device
 * (ctxs[0..W) — may all be the same context; meshes[r] = rank r's view);
 * _nccl makes this process rank `rank` of `world` (one GPU each; unique id
 * from rank 0's phfem_dist_nccl_unique_id, 128 bytes, shared out of band;
 * ctxs[0] / meshes[0] only): bulk exchanges are peer-window kernels into
 * CUDA-IPC-mapped buffers of the owners, NCCL (resolved at run time from the
 * process's libnccl.so.2) carries the small collectives and the fences.
 * Rank r's mesh: replicated coords [nC_all] and boundary lists, its elements
 * [nE_all r / W, nE_all (r+1) / W).  hist_sample > 1: the key-range histogram
 * over every hist_sample-th element (ranges only balance work).  Outputs: one
 * phfem_dist_rank_out per driven rank, global ids; concatenating the ranks'
 * slices gives the single-GPU pipeline's arrays bit for bit.               */
typedef struct phfem_dist_comm phfem_dist_comm;
typedef struct phfem_dist_rank_out {
  phfem_topology part;          /* the rank's edges (global ids); node_edge_start of its key range */
  phfem_classification cls;     /* retained_pos [part.E] / retained_edges [cls.L], global */
  phfem_csr C;                  /* the rank's rows (global row pointers and columns) */
  double *bd, *B, *D, *M, *M0, *load;  /* [cls.L], [n][9] x 4, [n][3]; n = ehi - elo */
  int32_t* elem_edge;           /* [n][3] */
  int32_t* elements;            /* [n][3] */
  double* coords;               /* [nC][2]: all valid when coords_all, else [0, nc_parent) and [mid_lo, mid_hi) */
  int32_t* dirichlet;           /* [nD][2] final boundary lists (replicated) */
  int32_t* neumann;             /* [nN][2] */
  int64_t mid_lo, mid_hi;
  int32_t elo, ehi, E0, R0, E, n_boundary, L, nC, nE, nD, nN, nc_parent, coords_all, reserved;
} phfem_dist_rank_out;
phfem_status phfem_dist_comm_local(int32_t W, phfem_dist_comm** out);
phfem_status phfem_dist_nccl_unique_id(void* uid128);
phfem_status phfem_dist_comm_nccl(const void* uid128, int32_t rank, int32_t world, int32_t device,
                                  phfem_dist_comm** out);
void phfem_dist_comm_destroy(phfem_dist_comm* comm);
const char* phfem_dist_comm_message(const phfem_dist_comm* comm);
/* Exchange statistics (cost model, tools/dist_model_cpp.py): enable (and
 * clear); read returns the number of phases, names[k] (valid until the next
 * pipeline call) and bytes[k][W] = bytes each rank received in phase k
 * (peer-window records stored into it, the other ranks' parts of
 * all-gathers, 2 (W-1)/W of all-reduced buffers; NCCL: what this rank sent
 * to each).  Enabled statistics synchronise after every exchange.           */
phfem_status phfem_dist_comm_set_stats(phfem_dist_comm* comm, int enable);
int phfem_dist_comm_stats(const phfem_dist_comm* comm, int max_phases, const char** names, int64_t* bytes);
#define PHFEM_DIST_NO_LOCAL 1 /* flags: every slot's side record / group start through the windows */
phfem_status phfem_dist_pipeline(phfem_dist_comm* comm, phfem_ctx** ctxs, const phfem_mesh* meshes, int32_t nC_all,
                                 int32_t nE_all, int32_t levels, const phfem_coeffs* coeffs, const phfem_field* f,
                                 const phfem_field* g, const phfem_field* uD, double t, int32_t hist_sample,
                                 int32_t flags, phfem_dist_rank_out* outs);
void phfem_dist_rank_out_release(phfem_ctx* ctx, phfem_dist_rank_out* out);

/* ---- device self-test of the fast-math building blocks (csrc/fastmath.cuh):
 * n random operand pairs; out[0] = fast divisions that differ from IEEE '/'
 * (must be 0: the element kernels rely on it for bit-exact blocks), out[1] =
 * max ulp distance of the fast sin from CUDA's sin, out[2] = divisions by 3.0
 * that differ.  Test infrastructure; no reference counterpart.             */
phfem_status phfem_selftest_fastmath(phfem_ctx* ctx, int64_t n, uint64_t seed,
                                     unsigned long long* out);

/* ---- host <-> device helpers for bindings without a CUDA runtime --------- */
phfem_status phfem_memcpy_h2d(phfem_ctx* ctx, void* dst, const void* src, size_t bytes);
phfem_status phfem_memcpy_d2h(phfem_ctx* ctx, void* dst, const void* src, size_t bytes);
/* device -> device, asynchronous on the ctx stream */
phfem_status phfem_memcpy_d2d(phfem_ctx* ctx, void* dst, const void* src, size_t bytes);

#ifdef __cplusplus
}
#endif

#endif /* PHFEM_GPU_H */
