"""TEST INFRASTRUCTURE ONLY — ctypes front end of oracle/_ref/libphfem_ref.so,
the reference's own hot-path sources (/root/reference/proj/src) compiled
unmodified against shim/Eigen (see oracle/ref.mk).  Used to pin the C oracle,
to generate tests/golden and as bench.py's "reference" CPU baseline.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(_HERE, "_ref", "libphfem_ref.so")
# the same extern "C" runner linked against the C++ drop-in layer instead of
# the reference's edge_topology / refine / assembly TUs (oracle/dropin.mk)
DROPIN_LIB = os.path.join(_HERE, "_ref", "dropin", "libphfem_dropin_runner.so")

import sys as _sys
_sys.path.insert(0, os.path.dirname(_HERE))
from paper_2401_15557_b200.capi import HostMesh, phfem_coeffs, phfem_field  # noqa: E402

_lib = None


class ReferenceError_(RuntimeError):
    def __init__(self, status, message):
        super().__init__(message)
        self.status = status


def available() -> bool:
    if os.path.exists(LIB):
        return True
    if os.path.isdir("/root/reference/proj/src"):
        try:
            subprocess.run(["make", "-s", "-j8", "-C", _HERE, "-f", "ref.mk"], check=True)
        except Exception:
            return False
        return os.path.exists(LIB)
    return False


def use_library(path: str) -> None:
    """Point every function of this module at another build of the runner
    (LIB = the reference's sources, DROPIN_LIB = the drop-in layer)."""
    global _lib, LIB
    LIB = path
    _lib = None


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError("oracle/_ref/libphfem_ref.so not built (needs /root/reference)")
        L = C.CDLL(LIB)
        vp, cp, sz, P = C.c_void_p, C.c_char_p, C.c_size_t, C.POINTER
        L.ref_mesh_new.restype = vp
        L.ref_mesh_new.argtypes = [vp, C.c_int, vp, C.c_int, vp, C.c_int, vp, C.c_int]
        L.ref_mesh_free.argtypes = [vp]
        L.ref_mesh_sizes.argtypes = [vp, vp]
        L.ref_mesh_copy.argtypes = [vp, vp, vp, vp, vp]
        L.ref_build_topology.argtypes = [vp, P(vp), cp, sz]
        L.ref_topology_free.argtypes = [vp]
        L.ref_topology_sizes.argtypes = [vp, vp]
        L.ref_topology_copy.argtypes = [vp, vp, vp, vp, vp, vp, vp]
        L.ref_node_pair_to_edge.argtypes = [vp, C.c_int, C.c_int]
        L.ref_directed_pair_to_element.argtypes = [vp, C.c_int, C.c_int]
        L.ref_classify_edges.argtypes = [vp, vp, P(vp), cp, sz]
        L.ref_classification_free.argtypes = [vp]
        L.ref_classification_sizes.argtypes = [vp, vp]
        L.ref_classification_copy.argtypes = [vp, vp, vp, vp, vp]
        L.ref_red_refine.argtypes = [vp, vp, P(vp), cp, sz]
        L.ref_edge_lengths.argtypes = [vp, vp, vp]
        L.ref_assemble_volume.argtypes = [vp, P(phfem_coeffs), vp, vp, vp, vp, cp, sz]
        L.ref_assemble_constraint.argtypes = [vp, vp, vp, P(C.c_int), P(C.c_int), P(C.c_longlong), vp, vp, vp,
                                              cp, sz]
        L.ref_assemble_load.argtypes = [vp, P(phfem_field), C.c_double, vp, cp, sz]
        L.ref_assemble_neumann.argtypes = [vp, vp, vp, P(phfem_field), C.c_double, vp, cp, sz]
        L.ref_assemble_dirichlet.argtypes = [vp, vp, vp, P(phfem_field), C.c_double, vp, cp, sz]
        L.ref_cn_rhs.argtypes = [vp, vp, vp, P(phfem_coeffs), P(phfem_field), P(phfem_field), P(phfem_field),
                                 C.c_double, C.c_int, vp, vp, cp, sz]
        L.ref_pipeline_seconds.restype = C.c_double
        L.ref_pipeline_seconds.argtypes = [vp, C.c_int, P(phfem_coeffs), P(phfem_field), P(phfem_field),
                                           P(phfem_field), P(C.c_longlong)]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _check(st, err):
    if st != 0:
        msg = err.value.decode()
        if st == 7:
            raise ValueError(msg)
        if st == 8:
            raise IndexError(msg)
        raise ReferenceError_(st, msg)


class RMesh:
    def __init__(self, hm: HostMesh = None, handle=None):
        self.h = handle if handle is not None else lib().ref_mesh_new(
            _p(hm.coords), hm.nC, _p(hm.elements), hm.nE, _p(hm.dirichlet), hm.dirichlet.shape[0],
            _p(hm.neumann), hm.neumann.shape[0])

    def host(self) -> HostMesh:
        sz = np.zeros(4, np.int32)
        lib().ref_mesh_sizes(self.h, _p(sz))
        c = np.zeros((sz[0], 2))
        e = np.zeros((sz[1], 3), np.int32)
        d = np.zeros((sz[2], 2), np.int32)
        n = np.zeros((sz[3], 2), np.int32)
        lib().ref_mesh_copy(self.h, _p(c), _p(e), _p(d), _p(n))
        return HostMesh(c, e, d, n)

    def __del__(self):
        try:
            lib().ref_mesh_free(self.h)
        except Exception:
            pass


class RTopology:
    def __init__(self, rm: RMesh):
        self.rm = rm
        h = C.c_void_p()
        err = C.create_string_buffer(512)
        _check(lib().ref_build_topology(rm.h, C.byref(h), err, 512), err)
        self.h = h.value

    def arrays(self) -> dict:
        sz = np.zeros(3, np.int32)
        lib().ref_topology_sizes(self.h, _p(sz))
        E, ni, nb = (int(x) for x in sz)
        out = {"edge_nodes": np.zeros((E, 2), np.int32), "edge_elements": np.zeros((E, 2), np.int32),
               "local_in_tplus": np.zeros(E, np.int32), "local_in_tminus": np.zeros(E, np.int32),
               "interior_edges": np.zeros(ni, np.int32), "boundary_edges": np.zeros(nb, np.int32)}
        lib().ref_topology_copy(self.h, *[_p(out[k]) for k in ["edge_nodes", "edge_elements", "local_in_tplus",
                                                               "local_in_tminus", "interior_edges",
                                                               "boundary_edges"]])
        return out

    def node_pair_to_edge(self, k, l):
        return lib().ref_node_pair_to_edge(self.h, k, l)

    def directed_pair_to_element(self, k, l):
        return lib().ref_directed_pair_to_element(self.h, k, l)

    def __del__(self):
        try:
            lib().ref_topology_free(self.h)
        except Exception:
            pass


class RClassification:
    def __init__(self, rt: RTopology, rm: RMesh):
        h = C.c_void_p()
        err = C.create_string_buffer(512)
        _check(lib().ref_classify_edges(rt.h, rm.h, C.byref(h), err, 512), err)
        self.h = h.value

    @property
    def L(self):
        sz = np.zeros(4, np.int32)
        lib().ref_classification_sizes(self.h, _p(sz))
        return int(sz[2])

    def arrays(self) -> dict:
        sz = np.zeros(4, np.int32)
        lib().ref_classification_sizes(self.h, _p(sz))
        out = {"dirichlet_edge_ids": np.zeros(sz[0], np.int32), "neumann_edge_ids": np.zeros(sz[1], np.int32),
               "retained_edges": np.zeros(sz[2], np.int32), "retained_pos": np.zeros(sz[3], np.int32)}
        lib().ref_classification_copy(self.h, *[_p(out[k]) for k in ["dirichlet_edge_ids", "neumann_edge_ids",
                                                                     "retained_edges", "retained_pos"]])
        return out

    def __del__(self):
        try:
            lib().ref_classification_free(self.h)
        except Exception:
            pass


def red_refine(rm: RMesh, rt: RTopology) -> RMesh:
    h = C.c_void_p()
    err = C.create_string_buffer(512)
    _check(lib().ref_red_refine(rm.h, rt.h, C.byref(h), err, 512), err)
    return RMesh(handle=h.value)


def assemble_volume(rm: RMesh, nE: int, coeffs: phfem_coeffs):
    outs = [np.zeros((nE, 9)) for _ in range(4)]
    err = C.create_string_buffer(512)
    _check(lib().ref_assemble_volume(rm.h, C.byref(coeffs), *[_p(o) for o in outs], err, 512), err)
    return outs


def assemble_constraint_csc(rm: RMesh, rt: RTopology, rc: RClassification):
    rows, cols, nnz = C.c_int(), C.c_int(), C.c_longlong()
    err = C.create_string_buffer(512)
    _check(lib().ref_assemble_constraint(rm.h, rt.h, rc.h, C.byref(rows), C.byref(cols), C.byref(nnz),
                                         None, None, None, err, 512), err)
    outer = np.zeros(cols.value + 1, np.int32)
    inner = np.zeros(nnz.value, np.int32)
    vals = np.zeros(nnz.value)
    _check(lib().ref_assemble_constraint(rm.h, rt.h, rc.h, C.byref(rows), C.byref(cols), C.byref(nnz),
                                         _p(outer), _p(inner), _p(vals), err, 512), err)
    return outer, inner, vals


def csc_to_csr(csc, nrows):
    outer, inner, vals = csc
    ncols = len(outer) - 1
    cols = np.repeat(np.arange(ncols, dtype=np.int32), np.diff(outer))
    order = np.lexsort((cols, inner))  # row-major, columns ascending
    row_ptr = np.zeros(nrows + 1, np.int32)
    np.add.at(row_ptr, inner + 1, 1)
    return np.cumsum(row_ptr).astype(np.int32), cols[order], vals[order]


def assemble_load(rm: RMesh, nE: int, f: phfem_field, t=0.0):
    out = np.zeros(3 * nE)
    err = C.create_string_buffer(512)
    _check(lib().ref_assemble_load(rm.h, C.byref(f), t, _p(out), err, 512), err)
    return out


def assemble_neumann(rm, rt, rc, nE, g, t=0.0):
    out = np.zeros(3 * nE)
    err = C.create_string_buffer(512)
    _check(lib().ref_assemble_neumann(rm.h, rt.h, rc.h, C.byref(g), t, _p(out), err, 512), err)
    return out


def assemble_dirichlet(rm, rt, rc, uD, t=0.0):
    out = np.zeros(max(rc.L, 1))
    err = C.create_string_buffer(512)
    _check(lib().ref_assemble_dirichlet(rm.h, rt.h, rc.h, C.byref(uD), t, _p(out), err, 512), err)
    return out[:rc.L]


def cn_rhs(rm, rt, rc, coeffs, f, g, uD, k, n, state):
    state = np.ascontiguousarray(state, dtype=np.float64)
    out = np.zeros_like(state)
    err = C.create_string_buffer(512)
    _check(lib().ref_cn_rhs(rm.h, rt.h, rc.h, C.byref(coeffs), C.byref(f), C.byref(g), C.byref(uD), k, n,
                            _p(state), _p(out), err, 512), err)
    return out


def pipeline_seconds(hm: HostMesh, levels: int, coeffs, f, g, uD):
    rm = RMesh(hm)
    n = C.c_longlong()
    s = lib().ref_pipeline_seconds(rm.h, levels, C.byref(coeffs), C.byref(f), C.byref(g), C.byref(uD), C.byref(n))
    return s, int(n.value)


def all_outputs(hm: HostMesh, coeffs, f, g, uD, t=0.0) -> dict:
    """Everything the reference computes on one mesh (for parity / goldens)."""
    rm = RMesh(hm)
    rt = RTopology(rm)
    rc = RClassification(rt, rm)
    B, D, M, M0 = assemble_volume(rm, hm.nE, coeffs)
    csc = assemble_constraint_csc(rm, rt, rc)
    fine = red_refine(rm, rt).host()
    return {"topo": rt.arrays(), "cls": rc.arrays(), "B": B, "D": D, "M": M, "M0": M0, "C_csc": csc,
            "C_csr": csc_to_csr(csc, rc.L), "b": assemble_load(rm, hm.nE, f, t),
            "ln": assemble_neumann(rm, rt, rc, hm.nE, g, t), "bd": assemble_dirichlet(rm, rt, rc, uD, t),
            "refined": fine}


def from_triplets(rows, cols, ri, ci, v):
    ri = np.ascontiguousarray(ri, dtype=np.int32)
    ci = np.ascontiguousarray(ci, dtype=np.int32)
    v = np.ascontiguousarray(v, dtype=np.float64)
    L = lib()
    L.ref_from_triplets.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_longlong,
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_char_p, C.c_size_t]
    nnz = C.c_longlong()
    err = C.create_string_buffer(512)
    _check(L.ref_from_triplets(rows, cols, _p(ri), _p(ci), _p(v), len(v), C.byref(nnz), None, None, None,
                               err, 512), err)
    outer = np.zeros(cols + 1, np.int32)
    inner = np.zeros(max(nnz.value, 1), np.int32)
    vals = np.zeros(max(nnz.value, 1), np.float64)
    _check(L.ref_from_triplets(rows, cols, _p(ri), _p(ci), _p(v), len(v), C.byref(nnz), _p(outer), _p(inner),
                               _p(vals), err, 512), err)
    return outer, inner[:nnz.value], vals[:nnz.value]


def operator_matrix(rm, rt, rc, coeffs, which: int, k: float = 0.0):
    """build_saddle_matrix (0) / step_matrices(k).first (1) / .second (2)."""
    L = lib()
    L.ref_operator_matrix.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_double,
                                      C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_char_p,
                                      C.c_size_t]
    dim = C.c_int()
    nnz = C.c_longlong()
    err = C.create_string_buffer(512)
    _check(L.ref_operator_matrix(rm.h, rt.h, rc.h, C.byref(coeffs), which, k, C.byref(dim), C.byref(nnz), None,
                                 None, None, err, 512), err)
    outer = np.zeros(dim.value + 1, np.int32)
    inner = np.zeros(nnz.value, np.int32)
    vals = np.zeros(nnz.value, np.float64)
    _check(L.ref_operator_matrix(rm.h, rt.h, rc.h, C.byref(coeffs), which, k, C.byref(dim), C.byref(nnz),
                                 _p(outer), _p(inner), _p(vals), err, 512), err)
    return outer, inner, vals


# ---- verification around the solve (analysis.cpp; tools/main.cpp:205-207) ----
_vp, _cp, _sz, _dbl = C.c_void_p, C.c_char_p, C.c_size_t, C.c_double


def error_norms(rm: RMesh, problem: str, primal, t: float = 0.0):
    """(error_l2, error_h1) with the reference's registry problem `problem`."""
    L = lib()
    L.ref_error_norms.argtypes = [_vp, _cp, _vp, _dbl, C.POINTER(_dbl), C.POINTER(_dbl), _cp, _sz]
    U = np.ascontiguousarray(primal, dtype=np.float64)
    l2, h1 = _dbl(), _dbl()
    err = C.create_string_buffer(512)
    _check(L.ref_error_norms(rm.h, problem.encode(), _p(U), t, C.byref(l2), C.byref(h1), err, 512), err)
    return l2.value, h1.value


def exact_multiplier(rm, rt, rc, problem: str, L_: int, t: float = 0.0):
    L = lib()
    L.ref_exact_multiplier.argtypes = [_vp, _vp, _vp, _cp, _dbl, _vp, _cp, _sz]
    out = np.zeros(L_)
    err = C.create_string_buffer(512)
    _check(L.ref_exact_multiplier(rm.h, rt.h, rc.h, problem.encode(), t, _p(out), err, 512), err)
    return out


def error_multiplier(rm, rt, rc, B, exact, discrete) -> float:
    L = lib()
    L.ref_error_multiplier.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, C.c_int, C.c_int, C.POINTER(_dbl), _cp, _sz]
    ex = np.ascontiguousarray(exact, dtype=np.float64)
    di = np.ascontiguousarray(discrete, dtype=np.float64)
    out = _dbl()
    err = C.create_string_buffer(512)
    Bv = np.ascontiguousarray(B, dtype=np.float64)
    _check(L.ref_error_multiplier(rm.h, rt.h, rc.h, _p(Bv), _p(ex), _p(di), len(ex), len(di),
                                  C.byref(out), err, 512), err)
    return out.value


def midpoint_traces(rt, primal, E: int):
    L = lib()
    L.ref_midpoint_traces.argtypes = [_vp, _vp, C.c_int, _vp]
    U = np.ascontiguousarray(primal, dtype=np.float64)
    out = np.zeros(E)
    L.ref_midpoint_traces(rt.h, _p(U), len(U), _p(out))
    return out


def constraint_residual(rm, rt, rc, uD, t, primal) -> float:
    L = lib()
    L.ref_constraint_residual.argtypes = [_vp, _vp, _vp, _vp, _dbl, _vp, C.POINTER(_dbl), _cp, _sz]
    U = np.ascontiguousarray(primal, dtype=np.float64)
    out = _dbl()
    err = C.create_string_buffer(512)
    _check(L.ref_constraint_residual(rm.h, rt.h, rc.h, C.byref(uD), t, _p(U), C.byref(out), err, 512), err)
    return out.value


def operator_spmv(rm, rt, rc, coeffs, which: int, k: float, x):
    L = lib()
    L.ref_operator_spmv.argtypes = [_vp, _vp, _vp, _vp, C.c_int, _dbl, _vp, _vp, _cp, _sz]
    xx = np.ascontiguousarray(x, dtype=np.float64)
    y = np.zeros(len(xx))
    err = C.create_string_buffer(512)
    _check(L.ref_operator_spmv(rm.h, rt.h, rc.h, C.byref(coeffs), which, k, _p(xx), _p(y), err, 512), err)
    return y


# ---- on-disk formats (mesh.cpp:114-180; tools/main.cpp:302-323) ---------------
def load_mesh_text(coordinates: bytes, elements: bytes, dirichlet: bytes = b"", neumann: bytes = b"") -> RMesh:
    L = lib()
    L.ref_load_mesh_text.argtypes = [_cp, _sz, _cp, _sz, _cp, _sz, _cp, _sz, C.POINTER(_vp), _cp, _sz]
    h = _vp()
    err = C.create_string_buffer(1024)
    _check(L.ref_load_mesh_text(coordinates, len(coordinates), elements, len(elements), dirichlet, len(dirichlet),
                                neumann, len(neumann), C.byref(h), err, 1024), err)
    return RMesh(handle=h.value)


def save_mesh_text(rm: RMesh) -> tuple:
    L = lib()
    L.ref_save_mesh_text.argtypes = [_vp, C.c_int, _vp, _sz, C.POINTER(_sz)]
    out = []
    for which in range(4):
        n = _sz()
        L.ref_save_mesh_text(rm.h, which, None, 0, C.byref(n))
        buf = C.create_string_buffer(max(n.value, 1))
        L.ref_save_mesh_text(rm.h, which, buf, n.value, C.byref(n))
        out.append(buf.raw[:n.value])
    return tuple(out)


def topology_csv(rm: RMesh) -> bytes:
    L = lib()
    L.ref_topology_csv.argtypes = [_vp, _vp, _sz, C.POINTER(_sz), _cp, _sz]
    n = _sz()
    err = C.create_string_buffer(512)
    _check(L.ref_topology_csv(rm.h, None, 0, C.byref(n), err, 512), err)
    buf = C.create_string_buffer(max(n.value, 1))
    _check(L.ref_topology_csv(rm.h, buf, n.value, C.byref(n), err, 512), err)
    return buf.raw[:n.value]
