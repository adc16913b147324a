"""TEST INFRASTRUCTURE ONLY — ctypes front end of the C oracle (phfem_oracle.c).

The oracle is the single-threaded CPU restatement of the reference algorithm
(/root/reference/proj/src/{edge_topology,refine,assembly,sparse,parabolic}.cpp)
used to check the CUDA path.  Only tests/, __graft_entry__.smoke() and bench.py
(cpu_baseline / --impl reference) import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(_HERE, "_build", "libphfem_oracle.so")

import sys as _sys
_sys.path.insert(0, os.path.dirname(_HERE))
from paper_2401_15557_b200.capi import HostMesh, phfem_coeffs, phfem_field, phfem_problem  # noqa: E402


class orc_mesh(C.Structure):
    _fields_ = [("coords", C.c_void_p), ("elements", C.c_void_p), ("dirichlet", C.c_void_p),
                ("neumann", C.c_void_p), ("nC", C.c_int32), ("nE", C.c_int32), ("nD", C.c_int32),
                ("nN", C.c_int32)]


class orc_topology(C.Structure):
    _fields_ = [("nC", C.c_int32), ("nE", C.c_int32), ("E", C.c_int32), ("n_interior", C.c_int32),
                ("n_boundary", C.c_int32), ("reserved", C.c_int32)] + [
        (n, C.c_void_p) for n in ["edge_nodes", "edge_elements", "local_in_tplus", "local_in_tminus",
                                  "interior_edges", "boundary_edges", "elem_edge", "node_edge_start",
                                  "pair_offsets", "pair_entries", "directed_offsets", "directed_entries"]]


class orc_classification(C.Structure):
    _fields_ = [("nD", C.c_int32), ("nN", C.c_int32), ("E", C.c_int32), ("L", C.c_int32),
                ("dirichlet_edge_ids", C.c_void_p), ("neumann_edge_ids", C.c_void_p),
                ("retained_edges", C.c_void_p), ("retained_pos", C.c_void_p)]


class orc_sparse(C.Structure):
    _fields_ = [("rows", C.c_int32), ("cols", C.c_int32), ("nnz", C.c_int64), ("ptr", C.c_void_p),
                ("idx", C.c_void_p), ("val", C.c_void_p)]


class OracleError(RuntimeError):
    def __init__(self, status, message):
        super().__init__(message)
        self.status = status


_lib = None


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = C.CDLL(LIB)
        P, vp, cp, sz = C.POINTER, C.c_void_p, C.c_char_p, C.c_size_t
        L.orc_build_topology.argtypes = [P(orc_mesh), P(orc_topology), cp, sz]
        L.orc_classify_edges.argtypes = [P(orc_topology), P(orc_mesh), P(orc_classification), cp, sz]
        L.orc_red_refine.argtypes = [P(orc_mesh), P(orc_topology), P(orc_mesh), cp, sz]
        L.orc_orient_ccw.argtypes = [P(orc_mesh)]
        L.orc_assemble_volume.argtypes = [P(orc_mesh), P(phfem_coeffs), vp, vp, vp, vp, cp, sz]
        L.orc_assemble_constraint.argtypes = [P(orc_mesh), P(orc_topology), P(orc_classification),
                                              P(orc_sparse), P(orc_sparse), cp, sz]
        L.orc_assemble_load.argtypes = [P(orc_mesh), P(phfem_field), C.c_double, vp, cp, sz]
        L.orc_assemble_neumann.argtypes = [P(orc_mesh), P(orc_topology), P(orc_classification),
                                           P(phfem_field), C.c_double, vp, cp, sz]
        L.orc_assemble_dirichlet.argtypes = [P(orc_mesh), P(orc_topology), P(orc_classification),
                                             P(phfem_field), C.c_double, vp, cp, sz]
        L.orc_cn_rhs.argtypes = [P(orc_mesh), P(orc_topology), P(orc_classification), P(phfem_coeffs),
                                 P(phfem_field), P(phfem_field), P(phfem_field), C.c_double, C.c_int,
                                 vp, vp, cp, sz]
        L.orc_edge_lengths.argtypes = [P(orc_mesh), P(orc_topology), vp]
        L.orc_node_pair_to_edge.argtypes = [P(orc_topology), C.c_int, C.c_int]
        L.orc_directed_pair_to_element.argtypes = [P(orc_topology), C.c_int, C.c_int]
        L.orc_constraint_residual.argtypes = [P(orc_sparse), vp, vp, P(C.c_double)]
        L.orc_exact_multiplier.argtypes = [P(orc_mesh), P(orc_topology), P(orc_classification),
                                           P(phfem_problem), C.c_double, vp]
        L.orc_error_l2.argtypes = [P(orc_mesh), vp, P(phfem_problem), C.c_double, P(C.c_double), vp]
        L.orc_error_h1.argtypes = [P(orc_mesh), vp, P(phfem_problem), C.c_double, P(C.c_double), vp]
        L.orc_error_multiplier.argtypes = [P(orc_sparse), vp, vp, vp, C.c_int64, C.c_int64, P(C.c_double), cp, sz]
        L.orc_midpoint_traces.argtypes = [P(orc_topology), vp, vp]
        L.orc_csc_spmv.argtypes = [P(orc_sparse), vp, vp]
        for n in ["orc_topology_free", "orc_classification_free", "orc_sparse_free", "orc_mesh_free"]:
            getattr(L, n).restype = None
        L.orc_topology_free.argtypes = [P(orc_topology)]
        L.orc_classification_free.argtypes = [P(orc_classification)]
        L.orc_sparse_free.argtypes = [P(orc_sparse)]
        L.orc_mesh_free.argtypes = [P(orc_mesh)]
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def _arr(ptr, n, dtype):
    if n == 0 or not ptr:
        return np.zeros(0, dtype=dtype)
    ct = {np.int32: C.c_int32, np.float64: C.c_double}[dtype]
    return np.ctypeslib.as_array((ct * n).from_address(ptr)).copy()


def _view(ptr, n, dtype):
    """No-copy numpy view of oracle-owned C memory (valid while its owner lives)."""
    if n == 0 or not ptr:
        return np.zeros(0, dtype=dtype)
    ct = {np.int32: C.c_int32, np.float64: C.c_double}[dtype]
    return np.ctypeslib.as_array((ct * n).from_address(ptr))


def _check(st, err):
    if st != 0:
        msg = err.value.decode()
        if st == 7:
            raise ValueError(msg)
        if st == 8:
            raise IndexError(msg)
        raise OracleError(st, msg)


class OMesh:
    """orc_mesh view over numpy arrays (kept alive by this object)."""

    def __init__(self, hm: HostMesh):
        self.hm = hm
        self.m = orc_mesh(_ptr(hm.coords), _ptr(hm.elements), _ptr(hm.dirichlet), _ptr(hm.neumann),
                          hm.nC, hm.nE, hm.dirichlet.shape[0], hm.neumann.shape[0])


class OTopology:
    def __init__(self, om: OMesh):
        self.om = om
        self.t = orc_topology()
        err = C.create_string_buffer(512)
        _check(lib().orc_build_topology(C.byref(om.m), C.byref(self.t), err, 512), err)

    def arrays(self) -> dict:
        t = self.t
        return {
            "edge_nodes": _arr(t.edge_nodes, 2 * t.E, np.int32).reshape(-1, 2),
            "edge_elements": _arr(t.edge_elements, 2 * t.E, np.int32).reshape(-1, 2),
            "local_in_tplus": _arr(t.local_in_tplus, t.E, np.int32),
            "local_in_tminus": _arr(t.local_in_tminus, t.E, np.int32),
            "interior_edges": _arr(t.interior_edges, t.n_interior, np.int32),
            "boundary_edges": _arr(t.boundary_edges, t.n_boundary, np.int32),
            "elem_edge": _arr(t.elem_edge, 3 * t.nE, np.int32).reshape(-1, 3),
            "node_edge_start": _arr(t.node_edge_start, t.nC + 1, np.int32),
        }

    def views(self) -> dict:
        """arrays() without the copies (large meshes): views of the C buffers."""
        t = self.t
        return {
            "edge_nodes": _view(t.edge_nodes, 2 * t.E, np.int32).reshape(-1, 2),
            "edge_elements": _view(t.edge_elements, 2 * t.E, np.int32).reshape(-1, 2),
            "local_in_tplus": _view(t.local_in_tplus, t.E, np.int32),
            "local_in_tminus": _view(t.local_in_tminus, t.E, np.int32),
            "interior_edges": _view(t.interior_edges, t.n_interior, np.int32),
            "boundary_edges": _view(t.boundary_edges, t.n_boundary, np.int32),
            "elem_edge": _view(t.elem_edge, 3 * t.nE, np.int32).reshape(-1, 3),
            "node_edge_start": _view(t.node_edge_start, t.nC + 1, np.int32),
        }

    def node_pair_to_edge(self, k, l):
        return lib().orc_node_pair_to_edge(C.byref(self.t), k, l)

    def directed_pair_to_element(self, k, l):
        return lib().orc_directed_pair_to_element(C.byref(self.t), k, l)

    def __del__(self):
        try:
            lib().orc_topology_free(C.byref(self.t))
        except Exception:
            pass


class OClassification:
    def __init__(self, topo: OTopology, om: OMesh):
        self.c = orc_classification()
        err = C.create_string_buffer(512)
        _check(lib().orc_classify_edges(C.byref(topo.t), C.byref(om.m), C.byref(self.c), err, 512), err)

    @property
    def L(self):
        return self.c.L

    def arrays(self) -> dict:
        c = self.c
        return {
            "dirichlet_edge_ids": _arr(c.dirichlet_edge_ids, c.nD, np.int32),
            "neumann_edge_ids": _arr(c.neumann_edge_ids, c.nN, np.int32),
            "retained_edges": _arr(c.retained_edges, c.L, np.int32),
            "retained_pos": _arr(c.retained_pos, c.E, np.int32),
        }

    def views(self) -> dict:
        c = self.c
        return {
            "dirichlet_edge_ids": _view(c.dirichlet_edge_ids, c.nD, np.int32),
            "neumann_edge_ids": _view(c.neumann_edge_ids, c.nN, np.int32),
            "retained_edges": _view(c.retained_edges, c.L, np.int32),
            "retained_pos": _view(c.retained_pos, c.E, np.int32),
        }

    def __del__(self):
        try:
            lib().orc_classification_free(C.byref(self.c))
        except Exception:
            pass


def build_topology(hm: HostMesh):
    om = OMesh(hm)
    return om, OTopology(om)


def classify_edges(om: OMesh, topo: OTopology) -> OClassification:
    return OClassification(topo, om)


def red_refine(hm: HostMesh, topo: OTopology | None = None) -> HostMesh:
    om = OMesh(hm)
    if topo is None:
        topo = OTopology(om)
    out = orc_mesh()
    err = C.create_string_buffer(512)
    _check(lib().orc_red_refine(C.byref(om.m), C.byref(topo.t), C.byref(out), err, 512), err)
    res = HostMesh(_arr(out.coords, 2 * out.nC, np.float64).reshape(-1, 2),
                   _arr(out.elements, 3 * out.nE, np.int32).reshape(-1, 3),
                   _arr(out.dirichlet, 2 * out.nD, np.int32).reshape(-1, 2),
                   _arr(out.neumann, 2 * out.nN, np.int32).reshape(-1, 2))
    lib().orc_mesh_free(C.byref(out))
    return res


def refine_levels(hm: HostMesh, levels: int) -> HostMesh:
    for _ in range(levels):
        hm = red_refine(hm)
    return hm


def orient_ccw(hm: HostMesh) -> HostMesh:
    hm2 = HostMesh(hm.coords.copy(), hm.elements.copy(), hm.dirichlet.copy(), hm.neumann.copy())
    om = OMesh(hm2)
    lib().orc_orient_ccw(C.byref(om.m))
    return hm2


def assemble_volume(hm: HostMesh, coeffs: phfem_coeffs):
    om = OMesh(hm)
    outs = [np.zeros((hm.nE, 9)) for _ in range(4)]
    err = C.create_string_buffer(512)
    _check(lib().orc_assemble_volume(C.byref(om.m), C.byref(coeffs), *[_ptr(o) for o in outs], err, 512), err)
    return outs


class OCsr:
    """C in CSR as oracle-owned C memory (no copies): .ptr / .idx / .val views."""

    def __init__(self, om: OMesh, topo: OTopology, cls: OClassification):
        self.s = orc_sparse()
        err = C.create_string_buffer(512)
        _check(lib().orc_assemble_constraint(C.byref(om.m), C.byref(topo.t), C.byref(cls.c), C.byref(self.s),
                                             None, err, 512), err)
        s = self.s
        self.ptr = _view(s.ptr, s.rows + 1, np.int32)
        self.idx = _view(s.idx, s.nnz, np.int32)
        self.val = _view(s.val, s.nnz, np.float64)

    def __del__(self):
        try:
            lib().orc_sparse_free(C.byref(self.s))
        except Exception:
            pass


def assemble_constraint(om: OMesh, topo: OTopology, cls: OClassification):
    csr, csc = orc_sparse(), orc_sparse()
    err = C.create_string_buffer(512)
    _check(lib().orc_assemble_constraint(C.byref(om.m), C.byref(topo.t), C.byref(cls.c), C.byref(csr),
                                         C.byref(csc), err, 512), err)
    r = {
        "csr": (_arr(csr.ptr, csr.rows + 1, np.int32), _arr(csr.idx, csr.nnz, np.int32),
                _arr(csr.val, csr.nnz, np.float64)),
        "csc": (_arr(csc.ptr, csc.cols + 1, np.int32), _arr(csc.idx, csc.nnz, np.int32),
                _arr(csc.val, csc.nnz, np.float64)),
    }
    lib().orc_sparse_free(C.byref(csr))
    lib().orc_sparse_free(C.byref(csc))
    return r


def assemble_load(hm: HostMesh, f: phfem_field, t: float = 0.0):
    om = OMesh(hm)
    out = np.zeros(3 * hm.nE)
    err = C.create_string_buffer(512)
    _check(lib().orc_assemble_load(C.byref(om.m), C.byref(f), t, _ptr(out), err, 512), err)
    return out


def assemble_neumann(om: OMesh, topo: OTopology, cls: OClassification, g: phfem_field, t: float = 0.0):
    out = np.zeros(3 * om.hm.nE)
    err = C.create_string_buffer(512)
    _check(lib().orc_assemble_neumann(C.byref(om.m), C.byref(topo.t), C.byref(cls.c), C.byref(g), t,
                                      _ptr(out), err, 512), err)
    return out


def assemble_dirichlet(om: OMesh, topo: OTopology, cls: OClassification, uD: phfem_field, t: float = 0.0):
    out = np.zeros(max(cls.L, 0))
    err = C.create_string_buffer(512)
    _check(lib().orc_assemble_dirichlet(C.byref(om.m), C.byref(topo.t), C.byref(cls.c), C.byref(uD), t,
                                        _ptr(out) if cls.L else None, err, 512), err)
    return out


def edge_lengths(om: OMesh, topo: OTopology):
    out = np.zeros(topo.t.E)
    lib().orc_edge_lengths(C.byref(om.m), C.byref(topo.t), _ptr(out))
    return out


def cn_rhs(om: OMesh, topo: OTopology, cls: OClassification, coeffs, f, g, uD, k, n, state):
    state = np.ascontiguousarray(state, dtype=np.float64)
    out = np.zeros_like(state)
    err = C.create_string_buffer(512)
    _check(lib().orc_cn_rhs(C.byref(om.m), C.byref(topo.t), C.byref(cls.c), C.byref(coeffs), C.byref(f),
                            C.byref(g), C.byref(uD), k, n, _ptr(state), _ptr(out), err, 512), err)
    return out


def pipeline(hm: HostMesh, levels: int, coeffs, f, g, uD, t: float = 0.0) -> dict:
    """The bench step on the CPU: refine chain, topology, classification,
    blocks, C (CSR), load = b + LN (elliptic.cpp:54-55), bD."""
    for _ in range(levels):
        hm = red_refine(hm)
    om, topo = build_topology(hm)
    cls = classify_edges(om, topo)
    B, D, M, M0 = assemble_volume(hm, coeffs)
    Cm = assemble_constraint(om, topo, cls)
    b = assemble_load(hm, f, t)
    ln = assemble_neumann(om, topo, cls, g, t)
    bd = assemble_dirichlet(om, topo, cls, uD, t)
    return {"mesh": hm, "topo": topo.arrays(), "cls": cls.arrays(), "C_csr": Cm["csr"],
            "C_csc": Cm["csc"], "B": B, "D": D, "M": M, "M0": M0, "load": b + ln, "bd": bd}


def all_outputs(hm: HostMesh, coeffs, f, g, uD, t: float = 0.0) -> dict:
    """Every hot-path output on one mesh, keyed like reference.all_outputs
    (the parity tests compare the two dicts entry by entry)."""
    om, ot = build_topology(hm)
    oc = classify_edges(om, ot)
    B, D, M, M0 = assemble_volume(hm, coeffs)
    Cm = assemble_constraint(om, ot, oc)
    return {"topo": ot.arrays(), "cls": oc.arrays(), "B": B, "D": D, "M": M, "M0": M0, "C_csc": Cm["csc"],
            "C_csr": Cm["csr"], "b": assemble_load(hm, f, t), "ln": assemble_neumann(om, ot, oc, g, t),
            "bd": assemble_dirichlet(om, ot, oc, uD, t), "refined": red_refine(hm, ot)}


def from_triplets(rows: int, cols: int, ri, ci, v):
    """SparseMatrix::from_triplets (sparse.cpp:30-97) -> (outer, inner, values)."""
    ri = np.ascontiguousarray(ri, dtype=np.int32)
    ci = np.ascontiguousarray(ci, dtype=np.int32)
    v = np.ascontiguousarray(v, dtype=np.float64)
    out = orc_sparse()
    err = C.create_string_buffer(512)
    L = lib()
    L.orc_from_triplets.argtypes = [C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                    C.POINTER(orc_sparse), C.c_char_p, C.c_size_t]
    _check(L.orc_from_triplets(rows, cols, _ptr(ri), _ptr(ci), _ptr(v), len(v), C.byref(out), err, 512), err)
    r = (_arr(out.ptr, cols + 1, np.int32), _arr(out.idx, out.nnz, np.int32), _arr(out.val, out.nnz, np.float64))
    L.orc_sparse_free(C.byref(out))
    return r


def operator_matrix(B, D, M, M0, C_csc, nE: int, L: int, which: int, k: float = 0.0):
    """build_saddle_matrix (which 0, elliptic.cpp:22-36) / step_matrix sign +1
    (which 1) / -1 (which 2) (parabolic.cpp:21-37): triplets in the
    reference's append order -> from_triplets.  Blocks [nE][9] column-major."""
    N = 3 * nE
    Bf, Df, Mf = (np.asarray(x, np.float64).reshape(-1) for x in (B, D, M))
    kk = (Bf + Df) + Mf
    if which == 0:
        top, s_ct, s_c = kk, -1.0, -1.0
    else:
        sign = 1.0 if which == 1 else -1.0
        top = np.asarray(M0, np.float64).reshape(-1) + (sign * (k / 2.0)) * kk
        s_ct, s_c = -sign * (k / 2.0), -sign * 0.5
    t = np.arange(9 * nE)
    e, q = t // 9, t % 9
    ri_b, ci_b = 3 * e + q % 3, 3 * e + q // 3
    outer, inner, val = C_csc
    cols = np.repeat(np.arange(N), np.diff(outer))
    ri = np.concatenate([ri_b, cols, N + inner])
    ci = np.concatenate([ci_b, N + inner, cols])
    v = np.concatenate([1.0 * top, s_ct * val, s_c * val])
    return from_triplets(N + L, N + L, ri, ci, v)


# ---- verification around the solve ---------------------------
class _CSC:
    """orc_sparse view of an Eigen ColMajor CSC (outer, inner, values) tuple."""

    def __init__(self, csc, rows: int, cols: int):
        self.keep = [np.ascontiguousarray(csc[0], dtype=np.int32), np.ascontiguousarray(csc[1], dtype=np.int32),
                     np.ascontiguousarray(csc[2], dtype=np.float64)]
        self.s = orc_sparse(rows, cols, len(self.keep[2]), _ptr(self.keep[0]), _ptr(self.keep[1]),
                            _ptr(self.keep[2]))


def constraint_residual(C_csc, L: int, N: int, primal, bd=None) -> float:
    """||C U + bD||_inf (tools/main.cpp:205-207)."""
    cs = _CSC(C_csc, L, N)
    U = np.ascontiguousarray(primal, dtype=np.float64)
    b = None if bd is None else np.ascontiguousarray(bd, dtype=np.float64)
    out = C.c_double()
    lib().orc_constraint_residual(C.byref(cs.s), _ptr(U), None if b is None else _ptr(b), C.byref(out))
    return out.value


def exact_multiplier(om: OMesh, topo: OTopology, cls: OClassification, prob, t: float = 0.0):
    out = np.zeros(cls.L)
    lib().orc_exact_multiplier(C.byref(om.m), C.byref(topo.t), C.byref(cls.c), C.byref(prob), t, _ptr(out))
    return out


def error_norm(hm: HostMesh, primal, prob, t: float = 0.0, h1: bool = False):
    """(norm, per-element terms) of error_h1 / error_l2 (analysis.cpp:41-80)."""
    om = OMesh(hm)
    U = np.ascontiguousarray(primal, dtype=np.float64)
    terms = np.zeros(hm.nE)
    out = C.c_double()
    fn = lib().orc_error_h1 if h1 else lib().orc_error_l2
    fn(C.byref(om.m), _ptr(U), C.byref(prob), t, C.byref(out), _ptr(terms))
    return out.value, terms


def error_multiplier(C_csc, L: int, N: int, B, exact, discrete) -> float:
    cs = _CSC(C_csc, L, N)
    Bv = np.ascontiguousarray(B, dtype=np.float64)
    ex = np.ascontiguousarray(exact, dtype=np.float64)
    di = np.ascontiguousarray(discrete, dtype=np.float64)
    out = C.c_double()
    err = C.create_string_buffer(512)
    _check(lib().orc_error_multiplier(C.byref(cs.s), _ptr(Bv), _ptr(ex), _ptr(di), len(ex), len(di),
                                      C.byref(out), err, 512), err)
    return out.value


def midpoint_traces(topo: OTopology, primal):
    U = np.ascontiguousarray(primal, dtype=np.float64)
    out = np.zeros(topo.t.E)
    lib().orc_midpoint_traces(C.byref(topo.t), _ptr(U), _ptr(out))
    return out


def csc_spmv(A_csc, rows: int, cols: int, x):
    cs = _CSC(A_csc, rows, cols)
    xx = np.ascontiguousarray(x, dtype=np.float64)
    y = np.zeros(rows)
    lib().orc_csc_spmv(C.byref(cs.s), _ptr(xx), _ptr(y))
    return y
