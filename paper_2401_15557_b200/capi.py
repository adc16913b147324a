"""ctypes binding of the C ABI in include/phfem_gpu.h (libphfem_b200.so).

This is the Python-side mirror of the reference's C++ entry points for the
edge-generation / red-refinement / assembly path (proj/include/phfem/*.hpp):
same names, same argument meaning, same exceptions (std::runtime_error ->
RuntimeError, std::invalid_argument -> ValueError, std::out_of_range ->
IndexError) with the reference's message text.  Device memory for inputs comes
from torch (plumbing only); every computation runs in the sm_100a kernels of
the library.  There is no CPU fallback: without the library or a B200 the
calls raise.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# PHFEM_LIB: an alternative in-tree build of the same library (kernel-variant
# experiments, tools/variants.sh); the default is the one build() makes
LIB_PATH = os.environ.get("PHFEM_LIB") or os.path.join(_HERE, "libphfem_b200.so")

# ---- status codes (phfem_status) -------------------------------------------
OK = 0
ERR_NONMANIFOLD = 1
ERR_DUP_DIRECTED = 2
ERR_NOT_AN_EDGE = 3
ERR_INTERIOR_BOUNDARY = 4
ERR_DEGENERATE = 5
ERR_NONFINITE = 6
ERR_INVALID_ARGUMENT = 7
ERR_OUT_OF_RANGE = 8
ERR_MISMATCH = 9
ERR_OOM = 10
ERR_CUDA = 11
ERR_NO_DEVICE = 12
ERR_RUNTIME = 13

# ---- field / coefficient kinds (phfem_fields.h) ------------------------------
FIELD_ZERO, FIELD_CONST, FIELD_SINSIN, FIELD_EXP_SINSIN, FIELD_AFFINE, FIELD_SIN3X, FIELD_NAN = range(7)
FLUX_ZERO, FLUX_CONST, FLUX_GRAD_SINSIN, FLUX_VEC_KAT = range(4)
COEFF_CONST, COEFF_CENTROID_POLY = range(2)
PROBLEM_ELLIPTIC_POLY, PROBLEM_PARABOLIC_POLY, PROBLEM_SINSIN = 1, 2, 3


class phfem_field(C.Structure):
    _fields_ = [("kind", C.c_int32), ("reserved", C.c_int32), ("p", C.c_double * 6)]


class phfem_coeffs(C.Structure):
    _fields_ = [("kind", C.c_int32), ("reserved", C.c_int32), ("p", C.c_double * 8)]


class phfem_problem(C.Structure):
    _fields_ = [("kind", C.c_int32), ("reserved", C.c_int32), ("coeffs", phfem_coeffs)]


def problem(kind: int, coeffs: "phfem_coeffs | None" = None) -> phfem_problem:
    """Manufactured problem descriptor (phfem_fields.h).  The registry problems
    (problems.cpp:85-150) carry A = I, p = (1, 1), delta = 1; SINSIN (config 1)
    A = I, p = 0, delta = 0."""
    pr = phfem_problem()
    pr.kind = kind
    if coeffs is None:
        coeffs = (coeffs_const(p=(1.0, 1.0), delta=1.0) if kind != PROBLEM_SINSIN else coeffs_const())
    pr.coeffs = coeffs
    return pr


def field(kind: int, *params: float) -> phfem_field:
    f = phfem_field()
    f.kind = kind
    for i, v in enumerate(params):
        f.p[i] = float(v)
    return f


def coeffs_const(A=((1.0, 0.0), (0.0, 1.0)), p=(0.0, 0.0), delta=0.0) -> phfem_coeffs:
    c = phfem_coeffs()
    c.kind = COEFF_CONST
    vals = [A[0][0], A[0][1], A[1][0], A[1][1], p[0], p[1], delta]
    for i, v in enumerate(vals):
        c.p[i] = float(v)
    return c


def coeffs_centroid_poly(p=(0.1, -0.1)) -> phfem_coeffs:
    c = phfem_coeffs()
    c.kind = COEFF_CENTROID_POLY
    c.p[4] = float(p[0])
    c.p[5] = float(p[1])
    return c


TWO_PI2 = 2.0 * math.pi * math.pi          # 2 pi^2, evaluated (2 pi) pi like the C literal
TWO_PI2_M1 = 2.0 * math.pi * math.pi - 1.0


class phfem_mesh(C.Structure):
    _fields_ = [("coords", C.c_void_p), ("elements", C.c_void_p), ("dirichlet", C.c_void_p),
                ("neumann", C.c_void_p), ("nC", C.c_int32), ("nE", C.c_int32), ("nD", C.c_int32),
                ("nN", C.c_int32), ("owned", C.c_int32), ("reserved", C.c_int32)]


class phfem_topology(C.Structure):
    _fields_ = [("nC", C.c_int32), ("nE", C.c_int32), ("E", C.c_int32), ("n_interior", C.c_int32),
                ("n_boundary", C.c_int32), ("reserved", C.c_int32),
                ("edge_nodes", C.c_void_p), ("edge_elements", C.c_void_p),
                ("local_in_tplus", C.c_void_p), ("local_in_tminus", C.c_void_p),
                ("interior_edges", C.c_void_p), ("boundary_edges", C.c_void_p),
                ("elem_edge", C.c_void_p), ("node_edge_start", C.c_void_p)]


class phfem_classification(C.Structure):
    _fields_ = [("nD", C.c_int32), ("nN", C.c_int32), ("E", C.c_int32), ("L", C.c_int32),
                ("flags", C.c_int32), ("reserved", C.c_int32),
                ("dirichlet_edge_ids", C.c_void_p), ("neumann_edge_ids", C.c_void_p),
                ("retained_edges", C.c_void_p), ("retained_pos", C.c_void_p),
                ("neumann_bits", C.c_void_p), ("block_prefix", C.c_void_p)]


class phfem_csr(C.Structure):
    _fields_ = [("rows", C.c_int32), ("cols", C.c_int32), ("nnz", C.c_int64),
                ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p), ("values", C.c_void_p)]


class phfem_csc(C.Structure):
    _fields_ = [("rows", C.c_int32), ("cols", C.c_int32), ("nnz", C.c_int64),
                ("outer", C.c_void_p), ("inner", C.c_void_p), ("values", C.c_void_p)]


class phfem_pipeline_out(C.Structure):
    _fields_ = [("mesh", phfem_mesh), ("topo", phfem_topology), ("cls", phfem_classification),
                ("C", phfem_csr), ("B", C.c_void_p), ("D", C.c_void_p), ("M", C.c_void_p),
                ("M0", C.c_void_p), ("load", C.c_void_p), ("bd", C.c_void_p)]


class phfem_dist_rank_out(C.Structure):
    _fields_ = [("part", phfem_topology), ("cls", phfem_classification), ("C", phfem_csr),
                ("bd", C.c_void_p), ("B", C.c_void_p), ("D", C.c_void_p), ("M", C.c_void_p), ("M0", C.c_void_p),
                ("load", C.c_void_p), ("elem_edge", C.c_void_p), ("elements", C.c_void_p), ("coords", C.c_void_p),
                ("dirichlet", C.c_void_p), ("neumann", C.c_void_p), ("mid_lo", C.c_int64), ("mid_hi", C.c_int64)] + \
        [(n, C.c_int32) for n in ("elo", "ehi", "E0", "R0", "E", "n_boundary", "L", "nC", "nE", "nD", "nN",
                                  "nc_parent", "coords_all", "reserved")]


_HOST_FIELDS = ["coords", "elements", "dirichlet", "neumann", "edge_nodes", "edge_elements",
                "local_in_tplus", "local_in_tminus", "interior_edges", "boundary_edges",
                "elem_edge", "dirichlet_edge_ids", "neumann_edge_ids", "retained_edges",
                "retained_pos", "C_row_ptr", "C_col_idx", "C_values", "B", "D", "M", "M0",
                "load", "bd"]


class phfem_pipeline_host(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in _HOST_FIELDS]


# Every exported symbol of include/phfem_gpu.h (checked by tests/test_abi.py).
EXPORTED = [
    "phfem_abi_version", "phfem_ctx_create", "phfem_ctx_destroy", "phfem_ctx_message",
    "phfem_ctx_stream", "phfem_ctx_sync", "phfem_alloc", "phfem_free", "phfem_ctx_launches",
    "phfem_ctx_set_eg_max_bs", "phfem_mesh_release", "phfem_build_topology", "phfem_topology_release",
    "phfem_classify_edges", "phfem_classification_release", "phfem_red_refine",
    "phfem_orient_ccw", "phfem_assemble_volume", "phfem_assemble_constraint",
    "phfem_csr_release", "phfem_constraint_csc", "phfem_csc_release", "phfem_assemble_load",
    "phfem_assemble_neumann", "phfem_assemble_dirichlet", "phfem_cn_plan_create",
    "phfem_cn_rhs", "phfem_cn_plan_destroy", "phfem_pipeline", "phfem_pipeline_release",
    "phfem_pipeline_from_host", "phfem_pipeline_download", "phfem_pipeline_download_bytes",
    "phfem_memcpy_h2d", "phfem_memcpy_d2h", "phfem_memcpy_d2d", "phfem_ctx_profile", "phfem_ctx_profile_read",
    "phfem_refine_topology", "phfem_pipeline_ex", "phfem_refine_level", "phfem_selftest_fastmath",
    "phfem_topology_derive", "phfem_topology_tables", "phfem_field_points", "phfem_edge_lengths",
    "phfem_assemble_load_sampled", "phfem_assemble_neumann_sampled", "phfem_assemble_dirichlet_sampled",
    "phfem_dist_occurrences", "phfem_dist_dedup", "phfem_dist_route_pairs", "phfem_dist_apply_pairs",
    "phfem_dist_add_offset", "phfem_dist_resolve", "phfem_dist_classify", "phfem_dist_neumann_table",
    "phfem_dist_neumann_apply", "phfem_dist_children", "phfem_dist_midpoints",
    "phfem_dist_side_records", "phfem_dist_side_apply", "phfem_dist_refine_level_side",
    "phfem_dist_start_records", "phfem_dist_start_apply", "phfem_dist_children_slots",
    "phfem_dist_side_p2p", "phfem_dist_start_p2p", "phfem_dist_bucket_bits", "phfem_dist_bucket_hist",
    "phfem_dist_pairs_p2p", "phfem_dist_dirichlet", "phfem_dist_level_count", "phfem_dist_level_run", "phfem_dist_classify_ex",
    "phfem_dist_bucket_cursors", "phfem_dist_scatter_p2p", "phfem_dist_dedup_items",
    "phfem_from_triplets", "phfem_saddle_matrix", "phfem_step_matrix",
    "phfem_constraint_residual", "phfem_exact_multiplier", "phfem_error_l2", "phfem_error_h1",
    "phfem_error_multiplier", "phfem_midpoint_traces", "phfem_csc_to_csr", "phfem_csr_spmv",
    "phfem_mesh_load_text", "phfem_mesh_load_dir", "phfem_mesh_format", "phfem_mesh_save_dir",
    "phfem_topology_csv", "phfem_topology_csv_file", "phfem_text_free", "phfem_dist_refine_level",
    "phfem_assemble_volume_load", "phfem_format_g", "phfem_format_g_host", "phfem_dist_refine_level_ex",
    "phfem_dist_dedup_ex", "phfem_dist_comm_local", "phfem_dist_nccl_unique_id", "phfem_dist_comm_nccl",
    "phfem_dist_comm_destroy", "phfem_dist_comm_message", "phfem_dist_pipeline", "phfem_dist_rank_out_release",
    "phfem_dist_level_run_ex", "phfem_dist_classify_given", "phfem_dist_children_slots_ex",
    "phfem_dist_side_p2p_ex", "phfem_dist_start_p2p_ex", "phfem_dist_level_count_ex",
    "phfem_dist_volume_start", "phfem_dist_volume_finish", "phfem_dist_comm_set_stats", "phfem_dist_comm_stats",
]
DIST_NO_LOCAL = 1
PIPE_GENERIC_EG = 1

_lib = None


def load_library(path: str = LIB_PATH):
    """Load libphfem_b200.so; raises (never falls back) when it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"phfem: CUDA library {path} is not built (run __graft_entry__.build())")
    lib = C.CDLL(path)
    P = C.POINTER
    vp, i32, i64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    sig = {
        "phfem_abi_version": (C.c_int, []),
        "phfem_ctx_create": (C.c_int, [C.c_int, vp, P(vp)]),
        "phfem_ctx_destroy": (None, [vp]),
        "phfem_ctx_message": (C.c_char_p, [vp]),
        "phfem_ctx_stream": (vp, [vp]),
        "phfem_ctx_sync": (C.c_int, [vp]),
        "phfem_alloc": (C.c_int, [vp, C.c_size_t, P(vp)]),
        "phfem_free": (None, [vp, vp]),
        "phfem_ctx_launches": (i64, [vp]),
        "phfem_ctx_set_eg_max_bs": (C.c_int, [vp, C.c_int]),
        "phfem_mesh_release": (None, [vp, P(phfem_mesh)]),
        "phfem_build_topology": (C.c_int, [vp, P(phfem_mesh), P(phfem_topology)]),
        "phfem_topology_release": (None, [vp, P(phfem_topology)]),
        "phfem_classify_edges": (C.c_int, [vp, P(phfem_topology), P(phfem_mesh), P(phfem_classification)]),
        "phfem_classification_release": (None, [vp, P(phfem_classification)]),
        "phfem_red_refine": (C.c_int, [vp, P(phfem_mesh), P(phfem_topology), P(phfem_mesh)]),
        "phfem_orient_ccw": (C.c_int, [vp, P(phfem_mesh)]),
        "phfem_assemble_volume": (C.c_int, [vp, P(phfem_mesh), P(phfem_coeffs), vp, vp, vp, vp]),
        "phfem_assemble_constraint": (C.c_int, [vp, P(phfem_mesh), P(phfem_topology),
                                                P(phfem_classification), P(phfem_csr)]),
        "phfem_csr_release": (None, [vp, P(phfem_csr)]),
        "phfem_constraint_csc": (C.c_int, [vp, P(phfem_mesh), P(phfem_topology),
                                           P(phfem_classification), P(phfem_csc)]),
        "phfem_csc_release": (None, [vp, P(phfem_csc)]),
        "phfem_assemble_load": (C.c_int, [vp, P(phfem_mesh), P(phfem_field), dbl, vp]),
        "phfem_assemble_neumann": (C.c_int, [vp, P(phfem_mesh), P(phfem_topology),
                                             P(phfem_classification), P(phfem_field), dbl, vp, C.c_int]),
        "phfem_assemble_dirichlet": (C.c_int, [vp, P(phfem_mesh), P(phfem_topology),
                                               P(phfem_classification), P(phfem_field), dbl, vp]),
        "phfem_cn_plan_create": (C.c_int, [vp, P(phfem_mesh), P(phfem_topology), P(phfem_classification),
                                           P(phfem_coeffs), P(phfem_field), P(phfem_field),
                                           P(phfem_field), dbl, P(vp)]),
        "phfem_cn_rhs": (C.c_int, [vp, vp, C.c_int, vp, vp]),
        "phfem_cn_plan_destroy": (None, [vp, vp]),
        "phfem_pipeline": (C.c_int, [vp, P(phfem_mesh), C.c_int, P(phfem_coeffs), P(phfem_field),
                                     P(phfem_field), P(phfem_field), dbl, P(phfem_pipeline_out)]),
        "phfem_pipeline_release": (None, [vp, P(phfem_pipeline_out)]),
        "phfem_pipeline_from_host": (C.c_int, [vp, vp, vp, vp, vp, i32, i32, i32, i32, C.c_int,
                                               P(phfem_coeffs), P(phfem_field), P(phfem_field),
                                               P(phfem_field), dbl, P(phfem_pipeline_out)]),
        "phfem_pipeline_download": (C.c_int, [vp, P(phfem_pipeline_out), P(phfem_pipeline_host)]),
        "phfem_pipeline_download_bytes": (i64, [P(phfem_pipeline_out), P(phfem_pipeline_host)]),
        "phfem_memcpy_h2d": (C.c_int, [vp, vp, vp, C.c_size_t]),
        "phfem_memcpy_d2h": (C.c_int, [vp, vp, vp, C.c_size_t]),
        "phfem_memcpy_d2d": (C.c_int, [vp, vp, vp, C.c_size_t]),
        "phfem_ctx_profile": (C.c_int, [vp, C.c_int]),
        "phfem_refine_topology": (C.c_int, [vp, P(phfem_mesh), P(phfem_topology), P(phfem_mesh),
                                            P(phfem_topology)]),
        "phfem_refine_level": (C.c_int, [vp, P(phfem_mesh), P(phfem_topology), P(phfem_classification),
                                         P(phfem_mesh), P(phfem_topology), P(phfem_classification),
                                         P(phfem_csr)]),
        "phfem_pipeline_ex": (C.c_int, [vp, P(phfem_mesh), C.c_int, P(phfem_coeffs), P(phfem_field),
                                        P(phfem_field), P(phfem_field), dbl, C.c_int, P(phfem_pipeline_out)]),
        "phfem_ctx_profile_read": (C.c_int, [vp, C.c_int, P(C.c_char_p), P(C.c_double), P(C.c_int64)]),
        "phfem_selftest_fastmath": (C.c_int, [vp, i64, C.c_uint64, P(C.c_ulonglong)]),
        "phfem_topology_derive": (C.c_int, [vp, P(phfem_mesh), P(phfem_topology)]),
        "phfem_topology_tables": (C.c_int, [vp, P(phfem_mesh), P(phfem_topology), vp, vp, vp, vp]),
        "phfem_field_points": (C.c_int, [vp, P(phfem_mesh), P(phfem_topology), P(phfem_classification),
                                         C.c_int, vp]),
        "phfem_assemble_load_sampled": (C.c_int, [vp, P(phfem_mesh), vp, vp]),
        "phfem_edge_lengths": (C.c_int, [vp, P(phfem_mesh), P(phfem_topology), vp]),
        "phfem_dist_occurrences": (C.c_int, [vp, vp, i32, i32, vp, i32, vp, vp, vp]),
        "phfem_dist_children": (C.c_int, [vp, vp, vp, i32, i32, vp]),
        "phfem_from_triplets": (C.c_int, [vp, i32, i32, vp, vp, vp, i64, P(phfem_csc)]),
        "phfem_saddle_matrix": (C.c_int, [vp, i32, vp, vp, vp, P(phfem_csc), P(phfem_csc)]),
        "phfem_step_matrix": (C.c_int, [vp, i32, vp, vp, vp, vp, P(phfem_csc), dbl, dbl, P(phfem_csc)]),
        "phfem_dist_midpoints": (C.c_int, [vp, vp, vp, i32, vp]),
        "phfem_dist_dedup": (C.c_int, [vp, vp, i64, i32, i32, i32, i32, P(phfem_topology), vp]),
        "phfem_dist_route_pairs": (C.c_int, [vp, vp, i64, i32, vp, i32, vp, vp, vp, i32, i32, vp]),
        "phfem_dist_apply_pairs": (C.c_int, [vp, vp, i64, i32, vp]),
        "phfem_dist_add_offset": (C.c_int, [vp, vp, i64, i32, C.c_int]),
        "phfem_dist_resolve": (C.c_int, [vp, P(phfem_topology), i32, i32, vp, i32, i32, vp, vp]),
        "phfem_dist_classify": (C.c_int, [vp, P(phfem_topology), i32, vp, i32, vp, i32,
                                          P(phfem_classification)]),
        "phfem_dist_neumann_table": (C.c_int, [vp, P(phfem_topology), i32, vp, i32, vp]),
        "phfem_dist_neumann_apply": (C.c_int, [vp, P(phfem_mesh), vp, i32, i32, i32, i32, P(phfem_field),
                                               dbl, vp]),
        "phfem_assemble_neumann_sampled": (C.c_int, [vp, P(phfem_mesh), P(phfem_topology),
                                                     P(phfem_classification), vp, vp, C.c_int]),
        "phfem_assemble_dirichlet_sampled": (C.c_int, [vp, P(phfem_mesh), P(phfem_topology),
                                                       P(phfem_classification), vp, vp]),
        "phfem_constraint_residual": (C.c_int, [vp, P(phfem_csr), vp, vp, P(dbl)]),
        "phfem_exact_multiplier": (C.c_int, [vp, P(phfem_mesh), P(phfem_topology), P(phfem_classification),
                                             P(phfem_problem), dbl, vp]),
        "phfem_error_l2": (C.c_int, [vp, P(phfem_mesh), vp, P(phfem_problem), dbl, P(dbl), vp]),
        "phfem_error_h1": (C.c_int, [vp, P(phfem_mesh), vp, P(phfem_problem), dbl, P(dbl), vp]),
        "phfem_error_multiplier": (C.c_int, [vp, P(phfem_mesh), P(phfem_topology), P(phfem_classification),
                                             vp, vp, vp, i64, i64, P(dbl)]),
        "phfem_midpoint_traces": (C.c_int, [vp, P(phfem_topology), vp, vp]),
        "phfem_csc_to_csr": (C.c_int, [vp, P(phfem_csc), P(phfem_csr)]),
        "phfem_csr_spmv": (C.c_int, [vp, P(phfem_csr), vp, vp]),
        "phfem_mesh_load_text": (C.c_int, [vp, C.c_char_p, C.c_size_t, C.c_char_p, C.c_size_t, C.c_char_p,
                                           C.c_size_t, C.c_char_p, C.c_size_t, P(phfem_mesh)]),
        "phfem_mesh_load_dir": (C.c_int, [vp, C.c_char_p, P(phfem_mesh)]),
        "phfem_mesh_format": (C.c_int, [vp, P(phfem_mesh), C.c_int, P(vp), P(C.c_size_t)]),
        "phfem_text_free": (None, [vp]),
        "phfem_format_g": (C.c_int, [vp, vp, i64, C.c_int, vp, vp]),
        "phfem_format_g_host": (C.c_int, [dbl, C.c_int, C.c_char_p]),
        "phfem_assemble_volume_load": (C.c_int, [vp, P(phfem_mesh), P(phfem_coeffs), P(phfem_field), dbl,
                                                 vp, vp, vp, vp, vp]),
        "phfem_dist_refine_level": (C.c_int, [vp, P(phfem_topology), i32, vp, vp, i32, vp, i32, i32, i32,
                                              vp, i32, P(phfem_topology), P(vp), vp, P(phfem_csr)]),
        "phfem_dist_dedup_ex": (C.c_int, [vp, vp, i64, i32, i32, i32, i32, i32, i32, vp, P(phfem_topology),
                                          vp, P(i64)]),
        "phfem_dist_refine_level_ex": (C.c_int, [vp, P(phfem_topology), i32, vp, vp, i32, vp, i32, i32, i32,
                                                 vp, i32, i32, i32, vp, P(phfem_topology), P(vp), P(i64), vp,
                                                 P(phfem_csr)]),
        "phfem_mesh_save_dir": (C.c_int, [vp, P(phfem_mesh), C.c_char_p]),
        "phfem_dist_side_records": (C.c_int, [vp, vp, vp, i32, vp, i32, vp, vp, vp]),
        "phfem_dist_side_apply": (C.c_int, [vp, vp, i64, i32, i32, vp]),
        "phfem_dist_refine_level_side": (C.c_int, [vp, P(phfem_topology), i32, vp, vp, i32, i32, i32, i32, vp, i32,
                                                   P(phfem_topology), vp, vp, P(phfem_csr)]),
        "phfem_dist_start_records": (C.c_int, [vp, P(phfem_topology), vp, i32, vp, vp, i32, vp, vp, vp]),
        "phfem_dist_start_apply": (C.c_int, [vp, vp, i64, i32, vp, vp]),
        "phfem_dist_children_slots": (C.c_int, [vp, vp, vp, i32, vp, vp, i32, vp, vp, vp]),
        "phfem_dist_side_p2p": (C.c_int, [vp, vp, vp, i32, vp, i32, i32, vp, vp]),
        "phfem_dist_bucket_bits": (C.c_int, [i32, i32]),
        "phfem_dist_dirichlet": (C.c_int, [vp, P(phfem_mesh), P(phfem_topology), P(phfem_classification),
                                           P(phfem_field), dbl, i32, vp]),
        "phfem_dist_level_count": (C.c_int, [vp, P(phfem_topology), i32, vp, vp, i32, C.c_int, P(i32), P(i32),
                                             P(vp)]),
        "phfem_dist_level_run": (C.c_int, [vp, vp, vp, i32, i32, i32, i32, i32, i32, P(phfem_topology), vp, vp,
                                           P(phfem_csr)]),
        "phfem_dist_classify_ex": (C.c_int, [vp, P(phfem_topology), i32, vp, i32, vp, i32, i32, i32,
                                             P(phfem_classification)]),
        "phfem_dist_pairs_p2p": (C.c_int, [vp, vp, i64, i32, vp, i32, i32, vp, vp]),
        "phfem_dist_bucket_hist": (C.c_int, [vp, vp, i32, i32, i32, i32, vp]),
        "phfem_dist_bucket_cursors": (C.c_int, [vp, vp, i32, i64, i32, vp, vp, vp, P(i64)]),
        "phfem_dist_scatter_p2p": (C.c_int, [vp, vp, i32, i32, i32, i32, vp, vp, i32, i32, vp, vp]),
        "phfem_dist_dedup_items": (C.c_int, [vp, vp, i64, vp, i32, i32, i32, i32, i32, i32, vp,
                                             P(phfem_topology), vp, P(i64)]),
        "phfem_dist_start_p2p": (C.c_int, [vp, P(phfem_topology), vp, i32, vp, vp, i32, i32, vp, vp, vp]),
        "phfem_topology_csv": (C.c_int, [vp, P(phfem_mesh), P(phfem_topology), P(vp), P(C.c_size_t)]),
        "phfem_topology_csv_file": (C.c_int, [vp, P(phfem_mesh), P(phfem_topology), C.c_char_p]),
        "phfem_dist_comm_local": (C.c_int, [i32, P(vp)]),
        "phfem_dist_nccl_unique_id": (C.c_int, [vp]),
        "phfem_dist_comm_nccl": (C.c_int, [vp, i32, i32, i32, P(vp)]),
        "phfem_dist_comm_destroy": (None, [vp]),
        "phfem_dist_comm_message": (C.c_char_p, [vp]),
        "phfem_dist_pipeline": (C.c_int, [vp, vp, P(phfem_mesh), i32, i32, i32, P(phfem_coeffs), P(phfem_field),
                                          P(phfem_field), P(phfem_field), dbl, i32, i32, P(phfem_dist_rank_out)]),
        "phfem_dist_volume_start": (C.c_int, [vp, P(phfem_mesh), P(phfem_coeffs), P(phfem_field), dbl, vp, vp, vp,
                                              vp, vp]),
        "phfem_dist_volume_finish": (C.c_int, [vp]),
        "phfem_dist_comm_set_stats": (C.c_int, [vp, C.c_int]),
        "phfem_dist_comm_stats": (C.c_int, [vp, C.c_int, P(C.c_char_p), P(i64)]),
        "phfem_dist_side_p2p_ex": (C.c_int, [vp, vp, vp, i32, vp, i32, i32, vp, vp, C.c_int]),
        "phfem_dist_start_p2p_ex": (C.c_int, [vp, P(phfem_topology), vp, i32, vp, vp, i32, i32, vp, vp, vp,
                                              C.c_int]),
        "phfem_dist_level_count_ex": (C.c_int, [vp, P(phfem_topology), i32, vp, vp, vp, i32, C.c_int, P(i32),
                                                P(i32), P(vp)]),
        "phfem_dist_rank_out_release": (None, [vp, P(phfem_dist_rank_out)]),
        "phfem_dist_level_run_ex": (C.c_int, [vp, vp, vp, i32, i32, i32, i32, i32, i32, i32, P(phfem_topology), vp,
                                              vp, P(phfem_csr), vp, vp]),
        "phfem_dist_classify_given": (C.c_int, [vp, P(phfem_topology), vp, i32, vp, i32, vp, vp, i32,
                                                P(phfem_classification)]),
        "phfem_dist_children_slots_ex": (C.c_int, [vp, vp, vp, i32, vp, vp, i32, i32, i32, vp, i32, vp, vp, vp,
                                                   vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class PhfemError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status


def _raise(status: int, message: str):
    if status == ERR_INVALID_ARGUMENT:
        raise ValueError(message)
    if status == ERR_OUT_OF_RANGE:
        raise IndexError(message)
    raise PhfemError(status, message)


class Context:
    """phfem_ctx: one device + stream.  Uses torch's current stream when torch
    is imported and a device is present, so torch-allocated inputs are ordered."""

    def __init__(self, device: int = 0, stream: Optional[int] = None):
        self.lib = load_library()
        self.ptr = C.c_void_p()
        # stream None: the ctx creates its own non-blocking stream.  An explicit
        # handle 0 is torch's legacy default stream: pass cudaStreamLegacy (0x1),
        # because a null handle would make the ctx create its own (unordered) one.
        handle = None if stream is None else C.c_void_p(stream if stream != 0 else 1)
        st = self.lib.phfem_ctx_create(device, handle, C.byref(self.ptr))
        if st != OK:
            raise PhfemError(st, f"phfem_ctx_create failed with status {st} (no usable sm_100 device?)")
        self.device = device

    def check(self, st: int):
        if st != OK:
            _raise(st, self.lib.phfem_ctx_message(self.ptr).decode())

    def sync(self):
        self.check(self.lib.phfem_ctx_sync(self.ptr))

    @property
    def launches(self) -> int:
        return int(self.lib.phfem_ctx_launches(self.ptr))

    def profile(self, enable: bool):
        """Start (and clear) / stop per-launch CUDA-event timing on the ctx stream."""
        self.check(self.lib.phfem_ctx_profile(self.ptr, 1 if enable else 0))

    def profile_read(self) -> dict:
        """{kernel name: (total ms, launches)} recorded since profile(True)."""
        n = 64
        names = (C.c_char_p * n)()
        ms = (C.c_double * n)()
        cnt = (C.c_int64 * n)()
        k = self.lib.phfem_ctx_profile_read(self.ptr, n, names, ms, cnt)
        if k < 0:
            raise PhfemError(ERR_CUDA, "phfem_ctx_profile_read failed")
        return {names[i].decode(): (ms[i], int(cnt[i])) for i in range(k)}

    def set_eg_max_bs(self, bs: int):
        """Test knob: cap the edge pass's bucket width (1..8, default 8) so
        small meshes take the multi-sub-bucket tile path (outputs unchanged)."""
        self.check(self.lib.phfem_ctx_set_eg_max_bs(self.ptr, int(bs)))

    @property
    def stream(self) -> int:
        return int(self.lib.phfem_ctx_stream(self.ptr) or 0)

    def close(self):
        if self.ptr:
            self.lib.phfem_ctx_destroy(self.ptr)
            self.ptr = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- device memory helpers ------------------------------------------------
    def alloc(self, nbytes: int) -> int:
        p = C.c_void_p()
        self.check(self.lib.phfem_alloc(self.ptr, max(int(nbytes), 1), C.byref(p)))
        return int(p.value)

    def free(self, ptr: int):
        if ptr and self.ptr:
            self.lib.phfem_free(self.ptr, C.c_void_p(ptr))

    def to_device(self, arr: np.ndarray) -> int:
        arr = np.ascontiguousarray(arr)
        p = self.alloc(arr.nbytes)
        if arr.nbytes:
            self.check(self.lib.phfem_memcpy_h2d(self.ptr, C.c_void_p(p), arr.ctypes.data_as(C.c_void_p), arr.nbytes))
        return p

    def to_host(self, ptr, shape, dtype) -> np.ndarray:
        out = np.empty(shape, dtype=dtype)
        if out.nbytes and ptr:
            self.check(self.lib.phfem_memcpy_d2h(self.ptr, out.ctypes.data_as(C.c_void_p), C.c_void_p(ptr), out.nbytes))
        return out


@dataclass
class HostMesh:
    """Reference Mesh (mesh.hpp:22-30) in numpy: 0-based ids."""
    coords: np.ndarray      # [nC, 2] float64
    elements: np.ndarray    # [nE, 3] int32
    dirichlet: np.ndarray   # [nD, 2] int32
    neumann: np.ndarray     # [nN, 2] int32

    def __post_init__(self):
        self.coords = np.ascontiguousarray(self.coords, dtype=np.float64).reshape(-1, 2)
        self.elements = np.ascontiguousarray(self.elements, dtype=np.int32).reshape(-1, 3)
        self.dirichlet = np.ascontiguousarray(self.dirichlet, dtype=np.int32).reshape(-1, 2)
        self.neumann = np.ascontiguousarray(self.neumann, dtype=np.int32).reshape(-1, 2)

    @property
    def nC(self):
        return self.coords.shape[0]

    @property
    def nE(self):
        return self.elements.shape[0]


class DeviceMesh:
    """phfem_mesh over device buffers (caller-owned unless `owned`)."""

    def __init__(self, ctx: Context, m: phfem_mesh, keep=None):
        self.ctx, self.m, self._keep = ctx, m, keep

    @classmethod
    def upload(cls, ctx: Context, hm: HostMesh) -> "DeviceMesh":
        m = phfem_mesh()
        m.coords = ctx.to_device(hm.coords)
        m.elements = ctx.to_device(hm.elements)
        m.dirichlet = ctx.to_device(hm.dirichlet)
        m.neumann = ctx.to_device(hm.neumann)
        m.nC, m.nE, m.nD, m.nN = hm.nC, hm.nE, hm.dirichlet.shape[0], hm.neumann.shape[0]
        m.owned = 1  # allocated from the ctx pool -> released by phfem_mesh_release
        return cls(ctx, m)

    def download(self) -> HostMesh:
        c, m = self.ctx, self.m
        return HostMesh(c.to_host(m.coords, (m.nC, 2), np.float64),
                        c.to_host(m.elements, (m.nE, 3), np.int32),
                        c.to_host(m.dirichlet, (m.nD, 2), np.int32),
                        c.to_host(m.neumann, (m.nN, 2), np.int32))

    def release(self):
        if self.m.owned and self.ctx.ptr:
            self.ctx.lib.phfem_mesh_release(self.ctx.ptr, C.byref(self.m))

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


class Topology:
    def __init__(self, ctx: Context, t: phfem_topology, owner: bool = True):
        self.ctx, self.t, self.owner = ctx, t, owner

    @property
    def E(self):
        return self.t.E

    def download(self) -> dict:
        c, t = self.ctx, self.t
        return {
            "edge_nodes": c.to_host(t.edge_nodes, (t.E, 2), np.int32),
            "edge_elements": c.to_host(t.edge_elements, (t.E, 2), np.int32),
            "local_in_tplus": c.to_host(t.local_in_tplus, (t.E,), np.int32),
            "local_in_tminus": c.to_host(t.local_in_tminus, (t.E,), np.int32),
            "interior_edges": c.to_host(t.interior_edges, (t.n_interior,), np.int32),
            "boundary_edges": c.to_host(t.boundary_edges, (t.n_boundary,), np.int32),
            "elem_edge": c.to_host(t.elem_edge, (t.nE, 3), np.int32),
            "node_edge_start": c.to_host(t.node_edge_start, (t.nC + 1,), np.int32),
        }

    def release(self):
        if self.owner and self.ctx.ptr:
            self.ctx.lib.phfem_topology_release(self.ctx.ptr, C.byref(self.t))
            self.owner = False

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


class Classification:
    def __init__(self, ctx: Context, c: phfem_classification, owner: bool = True):
        self.ctx, self.c, self.owner = ctx, c, owner

    @property
    def L(self):
        return self.c.L

    def download(self) -> dict:
        x, c = self.ctx, self.c
        return {
            "dirichlet_edge_ids": x.to_host(c.dirichlet_edge_ids, (c.nD,), np.int32),
            "neumann_edge_ids": x.to_host(c.neumann_edge_ids, (c.nN,), np.int32),
            "retained_edges": x.to_host(c.retained_edges, (c.L,), np.int32),
            "retained_pos": x.to_host(c.retained_pos, (c.E,), np.int32),
        }

    def release(self):
        if self.owner and self.ctx.ptr:
            self.ctx.lib.phfem_classification_release(self.ctx.ptr, C.byref(self.c))
            self.owner = False

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


def build_topology(ctx: Context, mesh: DeviceMesh) -> Topology:
    t = phfem_topology()
    ctx.check(ctx.lib.phfem_build_topology(ctx.ptr, C.byref(mesh.m), C.byref(t)))
    return Topology(ctx, t)


def classify_edges(ctx: Context, topo: Topology, mesh: DeviceMesh) -> Classification:
    c = phfem_classification()
    ctx.check(ctx.lib.phfem_classify_edges(ctx.ptr, C.byref(topo.t), C.byref(mesh.m), C.byref(c)))
    return Classification(ctx, c)


def red_refine(ctx: Context, mesh: DeviceMesh, topo: Topology) -> DeviceMesh:
    out = phfem_mesh()
    ctx.check(ctx.lib.phfem_red_refine(ctx.ptr, C.byref(mesh.m), C.byref(topo.t), C.byref(out)))
    return DeviceMesh(ctx, out)


def refine_topology(ctx: Context, parent: DeviceMesh, ptopo: Topology, fine: DeviceMesh) -> Topology:
    """build_topology(red_refine(parent)) from the parent topology, no sort."""
    t = phfem_topology()
    ctx.check(ctx.lib.phfem_refine_topology(ctx.ptr, C.byref(parent.m), C.byref(ptopo.t), C.byref(fine.m),
                                            C.byref(t)))
    return Topology(ctx, t)


def refine_level(ctx: Context, parent: DeviceMesh, ptopo: Topology, pcls: Classification,
                 fine: DeviceMesh):
    """Fused refined level: (topology, classification, C CSR host arrays) of
    `fine` = red_refine(parent) from the parent's topology/classification."""
    t, c, m = phfem_topology(), phfem_classification(), phfem_csr()
    ctx.check(ctx.lib.phfem_refine_level(ctx.ptr, C.byref(parent.m), C.byref(ptopo.t), C.byref(pcls.c),
                                         C.byref(fine.m), C.byref(t), C.byref(c), C.byref(m)))
    try:
        csr = (ctx.to_host(m.row_ptr, (m.rows + 1,), np.int32), ctx.to_host(m.col_idx, (m.nnz,), np.int32),
               ctx.to_host(m.values, (m.nnz,), np.float64))
    finally:
        ctx.lib.phfem_csr_release(ctx.ptr, C.byref(m))
    return Topology(ctx, t), Classification(ctx, c), csr


def orient_ccw(ctx: Context, mesh: DeviceMesh):
    ctx.check(ctx.lib.phfem_orient_ccw(ctx.ptr, C.byref(mesh.m)))


def assemble_volume(ctx: Context, mesh: DeviceMesh, coeffs: phfem_coeffs):
    """Returns host arrays B, D, M, M0 of shape [nE, 9] (column-major blocks)."""
    nE = mesh.m.nE
    ptrs = [ctx.alloc(72 * nE) for _ in range(4)]
    try:
        ctx.check(ctx.lib.phfem_assemble_volume(ctx.ptr, C.byref(mesh.m), C.byref(coeffs),
                                                *[C.c_void_p(p) for p in ptrs]))
        return [ctx.to_host(p, (nE, 9), np.float64) for p in ptrs]
    finally:
        for p in ptrs:
            ctx.free(p)


def assemble_load(ctx: Context, mesh: DeviceMesh, f: phfem_field, t: float = 0.0) -> np.ndarray:
    nE = mesh.m.nE
    p = ctx.alloc(24 * nE)
    try:
        ctx.check(ctx.lib.phfem_assemble_load(ctx.ptr, C.byref(mesh.m), C.byref(f), t, C.c_void_p(p)))
        return ctx.to_host(p, (3 * nE,), np.float64)
    finally:
        ctx.free(p)


def assemble_neumann(ctx: Context, mesh: DeviceMesh, topo: Topology, cls: Classification,
                     g: phfem_field, t: float = 0.0) -> np.ndarray:
    nE = mesh.m.nE
    p = ctx.alloc(24 * nE)
    try:
        ctx.check(ctx.lib.phfem_assemble_neumann(ctx.ptr, C.byref(mesh.m), C.byref(topo.t), C.byref(cls.c),
                                                 C.byref(g), t, C.c_void_p(p), 0))
        return ctx.to_host(p, (3 * nE,), np.float64)
    finally:
        ctx.free(p)


def assemble_dirichlet(ctx: Context, mesh: DeviceMesh, topo: Topology, cls: Classification,
                       uD: phfem_field, t: float = 0.0) -> np.ndarray:
    p = ctx.alloc(8 * max(cls.L, 1))
    try:
        ctx.check(ctx.lib.phfem_assemble_dirichlet(ctx.ptr, C.byref(mesh.m), C.byref(topo.t), C.byref(cls.c),
                                                   C.byref(uD), t, C.c_void_p(p)))
        return ctx.to_host(p, (cls.L,), np.float64)
    finally:
        ctx.free(p)


def assemble_constraint(ctx: Context, mesh: DeviceMesh, topo: Topology, cls: Classification):
    """C in CSR -> (row_ptr, col_idx, values) host arrays."""
    m = phfem_csr()
    ctx.check(ctx.lib.phfem_assemble_constraint(ctx.ptr, C.byref(mesh.m), C.byref(topo.t), C.byref(cls.c), C.byref(m)))
    try:
        return (ctx.to_host(m.row_ptr, (m.rows + 1,), np.int32),
                ctx.to_host(m.col_idx, (m.nnz,), np.int32),
                ctx.to_host(m.values, (m.nnz,), np.float64))
    finally:
        ctx.lib.phfem_csr_release(ctx.ptr, C.byref(m))


def constraint_csc(ctx: Context, mesh: DeviceMesh, topo: Topology, cls: Classification):
    """C in the reference's Eigen CSC layout -> (outer, inner, values)."""
    m = phfem_csc()
    ctx.check(ctx.lib.phfem_constraint_csc(ctx.ptr, C.byref(mesh.m), C.byref(topo.t), C.byref(cls.c), C.byref(m)))
    try:
        return (ctx.to_host(m.outer, (m.cols + 1,), np.int32),
                ctx.to_host(m.inner, (m.nnz,), np.int32),
                ctx.to_host(m.values, (m.nnz,), np.float64))
    finally:
        ctx.lib.phfem_csc_release(ctx.ptr, C.byref(m))


# ---- on-disk formats (csrc/io.cu) ------------------------------
def load_mesh_text(ctx: Context, coordinates: bytes, elements: bytes, dirichlet: bytes = b"",
                   neumann: bytes = b"") -> "DeviceMesh":
    """load_mesh (mesh.cpp:114-150) of the four files' contents."""
    m = phfem_mesh()
    ctx.check(ctx.lib.phfem_mesh_load_text(ctx.ptr, coordinates, len(coordinates), elements, len(elements),
                                           dirichlet, len(dirichlet), neumann, len(neumann), C.byref(m)))
    return DeviceMesh(ctx, m)


def load_mesh_dir(ctx: Context, path: str) -> "DeviceMesh":
    m = phfem_mesh()
    ctx.check(ctx.lib.phfem_mesh_load_dir(ctx.ptr, path.encode(), C.byref(m)))
    return DeviceMesh(ctx, m)


def save_mesh_text(ctx: Context, mesh: "DeviceMesh") -> tuple:
    """save_mesh (mesh.cpp:170-180): (coordinates, elements, dirichlet, neumann) bytes."""
    out = []
    for which in range(4):
        p, n = C.c_void_p(), C.c_size_t()
        ctx.check(ctx.lib.phfem_mesh_format(ctx.ptr, C.byref(mesh.m), which, C.byref(p), C.byref(n)))
        out.append(_take_text(ctx, p, n))
    return tuple(out)


def _take_text(ctx: Context, p, n) -> bytes:
    try:
        # (string_at takes a C int size: texts pass 2 GB at L12)
        return (C.c_char * n.value).from_address(p.value).raw if n.value else b""
    finally:
        ctx.lib.phfem_text_free(p)


def save_mesh_dir(ctx: Context, mesh: "DeviceMesh", path: str):
    ctx.check(ctx.lib.phfem_mesh_save_dir(ctx.ptr, C.byref(mesh.m), path.encode()))


def topology_csv(ctx: Context, mesh: "DeviceMesh", topo: "Topology") -> bytes:
    """The CLI's topology CSV (tools/main.cpp:302-323)."""
    p, n = C.c_void_p(), C.c_size_t()
    ctx.check(ctx.lib.phfem_topology_csv(ctx.ptr, C.byref(mesh.m), C.byref(topo.t), C.byref(p), C.byref(n)))
    return _take_text(ctx, p, n)


# ---- verification around the solve (csrc/verify.cu) ----------
def exact_multiplier(ctx: Context, mesh: DeviceMesh, topo: Topology, cls: Classification,
                     prob: phfem_problem, t: float = 0.0) -> np.ndarray:
    p = ctx.alloc(8 * max(cls.L, 1))
    try:
        ctx.check(ctx.lib.phfem_exact_multiplier(ctx.ptr, C.byref(mesh.m), C.byref(topo.t), C.byref(cls.c),
                                                 C.byref(prob), t, C.c_void_p(p)))
        return ctx.to_host(p, (cls.L,), np.float64)
    finally:
        ctx.free(p)


def error_norm(ctx: Context, mesh: DeviceMesh, primal: np.ndarray, prob: phfem_problem, t: float = 0.0,
               h1: bool = False):
    """(error_h1 or error_l2, per-element terms) of a host primal vector."""
    nE = mesh.m.nE
    U = ctx.to_device(np.ascontiguousarray(primal, dtype=np.float64))
    terms = ctx.alloc(8 * max(nE, 1))
    out = C.c_double()
    try:
        fn = ctx.lib.phfem_error_h1 if h1 else ctx.lib.phfem_error_l2
        ctx.check(fn(ctx.ptr, C.byref(mesh.m), C.c_void_p(U), C.byref(prob), t, C.byref(out), C.c_void_p(terms)))
        return out.value, ctx.to_host(terms, (nE,), np.float64)
    finally:
        ctx.free(U)
        ctx.free(terms)


def error_multiplier(ctx: Context, mesh: DeviceMesh, topo: Topology, cls: Classification, B: np.ndarray,
                     exact: np.ndarray, discrete: np.ndarray) -> float:
    dB = ctx.to_device(np.ascontiguousarray(B, dtype=np.float64))
    de = ctx.to_device(np.ascontiguousarray(exact, dtype=np.float64))
    dd = ctx.to_device(np.ascontiguousarray(discrete, dtype=np.float64))
    out = C.c_double()
    try:
        ctx.check(ctx.lib.phfem_error_multiplier(ctx.ptr, C.byref(mesh.m), C.byref(topo.t), C.byref(cls.c),
                                                 C.c_void_p(dB), C.c_void_p(de), C.c_void_p(dd), len(exact),
                                                 len(discrete), C.byref(out)))
        return out.value
    finally:
        for p in (dB, de, dd):
            ctx.free(p)


def midpoint_traces(ctx: Context, topo: Topology, primal: np.ndarray) -> np.ndarray:
    U = ctx.to_device(np.ascontiguousarray(primal, dtype=np.float64))
    out = ctx.alloc(8 * max(topo.E, 1))
    try:
        ctx.check(ctx.lib.phfem_midpoint_traces(ctx.ptr, C.byref(topo.t), C.c_void_p(U), C.c_void_p(out)))
        return ctx.to_host(out, (topo.E,), np.float64)
    finally:
        ctx.free(U)
        ctx.free(out)


def constraint_residual(ctx: Context, mesh: DeviceMesh, topo: Topology, cls: Classification,
                        primal: np.ndarray, bd: Optional[np.ndarray]) -> float:
    """||C U + bD||_inf with C assembled on the device (assemble_constraint)."""
    m = phfem_csr()
    ctx.check(ctx.lib.phfem_assemble_constraint(ctx.ptr, C.byref(mesh.m), C.byref(topo.t), C.byref(cls.c),
                                                C.byref(m)))
    U = ctx.to_device(np.ascontiguousarray(primal, dtype=np.float64))
    b = ctx.to_device(np.ascontiguousarray(bd, dtype=np.float64)) if bd is not None else 0
    out = C.c_double()
    try:
        ctx.check(ctx.lib.phfem_constraint_residual(ctx.ptr, C.byref(m), C.c_void_p(U), C.c_void_p(b or None),
                                                    C.byref(out)))
        return out.value
    finally:
        ctx.lib.phfem_csr_release(ctx.ptr, C.byref(m))
        ctx.free(U)
        if b:
            ctx.free(b)


class CNPlan:
    """Crank-Nicolson right-hand side (parabolic.cpp:95-103) on the device."""

    def __init__(self, ctx: Context, mesh: DeviceMesh, topo: Topology, cls: Classification,
                 coeffs: phfem_coeffs, f: phfem_field, g: phfem_field, uD: phfem_field, k: float):
        self.ctx, self._keep = ctx, (mesh, topo, cls)
        self.ptr = C.c_void_p()
        ctx.check(ctx.lib.phfem_cn_plan_create(ctx.ptr, C.byref(mesh.m), C.byref(topo.t), C.byref(cls.c),
                                               C.byref(coeffs), C.byref(f), C.byref(g), C.byref(uD), k,
                                               C.byref(self.ptr)))
        self.n_state = 3 * mesh.m.nE + cls.L

    def rhs_device(self, n: int, state_ptr: int, rhs_ptr: int):
        self.ctx.check(self.ctx.lib.phfem_cn_rhs(self.ctx.ptr, self.ptr, n, C.c_void_p(state_ptr), C.c_void_p(rhs_ptr)))

    def rhs(self, n: int, state: np.ndarray) -> np.ndarray:
        s = self.ctx.to_device(np.asarray(state, dtype=np.float64))
        r = self.ctx.alloc(8 * self.n_state)
        try:
            self.rhs_device(n, s, r)
            return self.ctx.to_host(r, (self.n_state,), np.float64)
        finally:
            self.ctx.free(s)
            self.ctx.free(r)

    def close(self):
        if self.ptr and self.ctx.ptr:
            self.ctx.lib.phfem_cn_plan_destroy(self.ctx.ptr, self.ptr)
            self.ptr = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class PipelineResult:
    def __init__(self, ctx: Context, out: phfem_pipeline_out):
        self.ctx, self.out = ctx, out

    def download(self) -> dict:
        c, o = self.ctx, self.out
        nE, E, L = o.mesh.nE, o.topo.E, o.cls.L
        mview = phfem_mesh.from_buffer_copy(o.mesh)
        mview.owned = 0  # a view: the result owns the buffers
        res = {
            "mesh": DeviceMesh(c, mview).download(),
            "topo": Topology(c, o.topo, owner=False).download(),
            "cls": Classification(c, o.cls, owner=False).download(),
            "C_row_ptr": c.to_host(o.C.row_ptr, (L + 1,), np.int32),
            "C_col_idx": c.to_host(o.C.col_idx, (o.C.nnz,), np.int32),
            "C_values": c.to_host(o.C.values, (o.C.nnz,), np.float64),
            "B": c.to_host(o.B, (nE, 9), np.float64),
            "D": c.to_host(o.D, (nE, 9), np.float64),
            "M": c.to_host(o.M, (nE, 9), np.float64),
            "M0": c.to_host(o.M0, (nE, 9), np.float64),
            "load": c.to_host(o.load, (3 * nE,), np.float64),
            "bd": c.to_host(o.bd, (L,), np.float64),
        }
        return res

    def mesh_view(self) -> "DeviceMesh":
        mview = phfem_mesh.from_buffer_copy(self.out.mesh)
        mview.owned = 0
        return DeviceMesh(self.ctx, mview)

    def topo_view(self) -> "Topology":
        return Topology(self.ctx, self.out.topo, owner=False)

    def cls_view(self) -> "Classification":
        return Classification(self.ctx, self.out.cls, owner=False)

    def release(self):
        if self.ctx is not None and self.ctx.ptr:
            self.ctx.lib.phfem_pipeline_release(self.ctx.ptr, C.byref(self.out))
            self.ctx = None

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


def pipeline(ctx: Context, mesh: DeviceMesh, levels: int, coeffs: phfem_coeffs, f: phfem_field,
             g: phfem_field, uD: phfem_field, t: float = 0.0, flags: int = 0) -> PipelineResult:
    out = phfem_pipeline_out()
    ctx.check(ctx.lib.phfem_pipeline_ex(ctx.ptr, C.byref(mesh.m), levels, C.byref(coeffs), C.byref(f),
                                        C.byref(g), C.byref(uD), t, flags, C.byref(out)))
    res = PipelineResult(ctx, out)
    # with levels = 0 the result's mesh is the input's buffers: keep the input
    # alive as long as the result (a temporary DeviceMesh would otherwise be
    # released underneath it — found by guard mode, tests/test_guard.py)
    res._input = mesh
    return res


# ---- sharded pipeline, C++ orchestration (csrc/dist_run.cu) -------------------------
class DistComm:
    """phfem_dist_comm: `local(W)` emulates W ranks in this process (one
    device); `nccl(uid, rank, world, device)` makes this process one rank of
    an NCCL communicator (uid = `nccl_unique_id()` of rank 0, shared out of
    band, e.g. with torch.distributed.broadcast_object_list)."""

    def __init__(self, ptr, world: int, local: bool):
        self.lib, self.ptr, self.world, self.local = load_library(), ptr, world, local

    @classmethod
    def local_ranks(cls, W: int) -> "DistComm":
        lib = load_library()
        p = C.c_void_p()
        if lib.phfem_dist_comm_local(W, C.byref(p)) != OK:
            raise ValueError(f"phfem_dist_comm_local({W}) failed")
        return cls(p, W, True)

    @staticmethod
    def nccl_unique_id() -> bytes:
        lib = load_library()
        buf = C.create_string_buffer(128)
        if lib.phfem_dist_nccl_unique_id(buf) != OK:
            raise PhfemError(ERR_CUDA, "ncclGetUniqueId failed (libnccl.so.2 not loadable?)")
        return buf.raw

    @classmethod
    def nccl(cls, uid: bytes, rank: int, world: int, device: int) -> "DistComm":
        lib = load_library()
        p = C.c_void_p()
        buf = C.create_string_buffer(bytes(uid), 128)
        st = lib.phfem_dist_comm_nccl(buf, rank, world, device, C.byref(p))
        if st != OK:
            raise PhfemError(st, f"phfem_dist_comm_nccl(rank {rank} of {world}) failed with status {st}")
        return cls(p, world, False)

    def set_stats(self, enable: bool):
        self.lib.phfem_dist_comm_set_stats(self.ptr, 1 if enable else 0)

    def stats(self) -> dict:
        """{phase: [bytes received per rank]} since set_stats(True)"""
        n = 64
        names = (C.c_char_p * n)()
        b = (C.c_int64 * (n * self.world))()
        k = self.lib.phfem_dist_comm_stats(self.ptr, n, names, b)
        return {names[i].decode(): [int(b[i * self.world + r]) for r in range(self.world)] for i in range(k)}

    def close(self):
        if self.ptr:
            self.lib.phfem_dist_comm_destroy(self.ptr)
            self.ptr = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DistRankOut:
    """One rank's outputs of dist_pipeline (device memory of its ctx)."""

    def __init__(self, ctx: Context, o: phfem_dist_rank_out):
        self.ctx, self.o = ctx, o

    def rank_slice(self) -> dict:
        """dist.rank_slice's layout (host arrays, global ids): dist.concat_slices
        of the ranks' slices is the single-GPU pipeline's output."""
        x, o = self.ctx, self.o
        d = Topology(x, o.part, owner=False).download()
        d.pop("elem_edge")
        n = o.ehi - o.elo
        d["elem_edge"] = x.to_host(o.elem_edge, (n, 3), np.int32)
        d["retained_pos"] = x.to_host(o.cls.retained_pos, (o.cls.E,), np.int32)
        d["retained_edges"] = x.to_host(o.cls.retained_edges, (o.cls.L,), np.int32)
        d["C_row_ptr"] = x.to_host(o.C.row_ptr, (o.C.rows + 1,), np.int32)
        d["C_col_idx"] = x.to_host(o.C.col_idx, (o.C.nnz,), np.int32)
        d["C_values"] = x.to_host(o.C.values, (o.C.nnz,), np.float64)
        d["bd"] = x.to_host(o.bd, (o.cls.L,), np.float64)
        for k in ("B", "D", "M", "M0"):
            d[k] = x.to_host(getattr(o, k), (9 * n,), np.float64)
        d["load"] = x.to_host(o.load, (3 * n,), np.float64)
        if o.coords_all:
            d["coords"] = x.to_host(o.coords, (o.nC, 2), np.float64)
        else:
            d["coords_parent"] = x.to_host(o.coords, (o.nc_parent, 2), np.float64)
            d["mid_own"] = x.to_host((o.coords or 0) + 16 * o.mid_lo, (o.mid_hi - o.mid_lo, 2), np.float64)
        d["elements"] = x.to_host(o.elements, (n, 3), np.int32)
        d["dirichlet"] = x.to_host(o.dirichlet, (o.nD, 2), np.int32)
        d["neumann"] = x.to_host(o.neumann, (o.nN, 2), np.int32)
        return d

    def release(self):
        if self.ctx.ptr:
            self.ctx.lib.phfem_dist_rank_out_release(self.ctx.ptr, C.byref(self.o))

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


def dist_pipeline(comm: DistComm, ctxs, meshes, nC: int, nE: int, levels: int, coeffs: phfem_coeffs,
                  f: phfem_field, g: phfem_field, uD: phfem_field, t: float = 0.0,
                  hist_sample: int = 1, flags: int = 0) -> list:
    """phfem_dist_pipeline: the sharded step with the orchestration in C++.
    ctxs / meshes: one per driven rank (local: W, NCCL: 1); meshes[r] is a
    phfem_mesh (replicated coords / boundary lists, rank r's elements)."""
    n = comm.world if comm.local else 1
    assert len(ctxs) == n and len(meshes) == n
    ca = (C.c_void_p * n)(*[c.ptr.value for c in ctxs])
    ma = (phfem_mesh * n)(*meshes)
    outs = (phfem_dist_rank_out * n)()
    st = ctxs[0].lib.phfem_dist_pipeline(comm.ptr, ca, ma, nC, nE, levels, C.byref(coeffs), C.byref(f), C.byref(g),
                                         C.byref(uD), t, hist_sample, flags, outs)
    ctxs[0].check(st)
    return [DistRankOut(c, outs[i]) for i, c in enumerate(ctxs)]
