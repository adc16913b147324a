"""verification around the solve — the constraint residual
(tools/main.cpp:205-207), exact_multiplier / error_h1 / error_l2 /
error_multiplier / hybrid_midpoint_traces (analysis.cpp), and the
Eigen-ordered SpMV of the stored step / saddle matrices.

not gpu: the C oracle against the reference's OWN analysis.cpp /
problems.cpp / quadrature.cpp (oracle/_ref, the registry problems
"elliptic-poly" and "parabolic-poly" themselves) — bit for bit, including the
element-order sums of the two norms and the exception texts.
gpu: csrc/verify.cu against the oracle: per-entry values and per-element
error terms bit for bit; the norms (a fixed device tree instead of element
order) within 1e-12 relative; max-reductions exact.
"""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O
from oracle import reference as R
from paper_2401_15557_b200 import capi, meshgen as G


def jittered_square():
    hm = G.stress_transform(O.refine_levels(G.square_2tri(), 4), 4)
    return O.orient_ccw(hm)


MESHES = [("crisscross-L2", lambda: O.refine_levels(G.crisscross_square(), 2)),
          ("lshape-L2", lambda: O.refine_levels(G.lshape_6tri(), 2)),
          ("square-L4-jittered", jittered_square)]
PROBLEMS = [("elliptic-poly", capi.PROBLEM_ELLIPTIC_POLY, 0.0),
            ("parabolic-poly", capi.PROBLEM_PARABOLIC_POLY, 0.37)]
COEFFS = capi.coeffs_const(((2.0, 0.3), (0.3, 1.0)), (1.0, -0.5), 0.7)
needs_ref = pytest.mark.skipif(not R.available(), reason="reference build unavailable")


def bits_equal(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    assert a.shape == b.shape
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


def ocase(hm):
    om, ot = O.build_topology(hm)
    return om, ot, O.classify_edges(om, ot)


def rcase(hm):
    rm = R.RMesh(hm)
    rt = R.RTopology(rm)
    return rm, rt, R.RClassification(rt, rm)


def primal_of(hm, seed=3):
    return 0.1 * G.uniform_pm1(seed, 3 * hm.nE)


# ---------------------------------------------------------------- oracle pins
@needs_ref
@pytest.mark.parametrize("mname,make", MESHES, ids=[m[0] for m in MESHES])
@pytest.mark.parametrize("pname,kind,t", PROBLEMS, ids=[p[0] for p in PROBLEMS])
def test_error_norms_equal_reference(mname, make, pname, kind, t):
    hm = make()
    U = primal_of(hm)
    pr = capi.problem(kind)
    l2, _ = O.error_norm(hm, U, pr, t)
    h1, _ = O.error_norm(hm, U, pr, t, h1=True)
    rl2, rh1 = R.error_norms(R.RMesh(hm), pname, U, t)
    bits_equal(l2, rl2)
    bits_equal(h1, rh1)


@needs_ref
@pytest.mark.parametrize("mname,make", MESHES, ids=[m[0] for m in MESHES])
@pytest.mark.parametrize("pname,kind,t", PROBLEMS, ids=[p[0] for p in PROBLEMS])
def test_exact_multiplier_equals_reference(mname, make, pname, kind, t):
    hm = make()
    om, ot, oc = ocase(hm)
    rm, rt, rc = rcase(hm)
    bits_equal(O.exact_multiplier(om, ot, oc, capi.problem(kind), t),
               R.exact_multiplier(rm, rt, rc, pname, oc.L, t))


@needs_ref
@pytest.mark.parametrize("mname,make", MESHES, ids=[m[0] for m in MESHES])
def test_error_multiplier_equals_reference(mname, make):
    hm = make()
    om, ot, oc = ocase(hm)
    rm, rt, rc = rcase(hm)
    exact = O.exact_multiplier(om, ot, oc, capi.problem(capi.PROBLEM_ELLIPTIC_POLY))
    discrete = exact + 1e-3 * G.uniform_pm1(5, oc.L)
    B = O.assemble_volume(hm, COEFFS)[0]
    Cc = O.assemble_constraint(om, ot, oc)["csc"]
    bits_equal(O.error_multiplier(Cc, oc.L, 3 * hm.nE, B, exact, discrete),
               R.error_multiplier(rm, rt, rc, B, exact, discrete))


@needs_ref
def test_error_multiplier_errors_match_reference():
    hm = O.refine_levels(G.crisscross_square(), 1)
    om, ot, oc = ocase(hm)
    rm, rt, rc = rcase(hm)
    Cc = O.assemble_constraint(om, ot, oc)["csc"]
    x = np.ones(oc.L)
    B = O.assemble_volume(hm, COEFFS)[0]
    with pytest.raises(ValueError) as eo:
        O.error_multiplier(Cc, oc.L, 3 * hm.nE, B, x, x[:-1])
    with pytest.raises(ValueError) as er:
        R.error_multiplier(rm, rt, rc, B, x, x[:-1])
    assert str(eo.value) == str(er.value) == "error_multiplier: size mismatch"
    # a stiffness without a positive diagonal entry (B_ii <= 0 are skipped)
    Bz = -np.abs(B)
    with pytest.raises(RuntimeError) as eo:
        O.error_multiplier(Cc, oc.L, 3 * hm.nE, Bz, x, 0.5 * x)
    with pytest.raises(RuntimeError) as er:
        R.error_multiplier(rm, rt, rc, Bz, x, 0.5 * x)
    assert str(eo.value) == str(er.value) == "error_multiplier: all diagonal entries of B vanish"


@needs_ref
@pytest.mark.parametrize("mname,make", MESHES, ids=[m[0] for m in MESHES])
def test_midpoint_traces_and_residual_equal_reference(mname, make):
    hm = make()
    om, ot, oc = ocase(hm)
    rm, rt, rc = rcase(hm)
    U = primal_of(hm)
    bits_equal(O.midpoint_traces(ot, U), R.midpoint_traces(rt, U, ot.t.E))
    uD = capi.field(capi.FIELD_AFFINE, 0.5, 1.0, -2.0, 3.0)
    bd = O.assemble_dirichlet(om, ot, oc, uD, 0.3)
    Cc = O.assemble_constraint(om, ot, oc)["csc"]
    bits_equal(O.constraint_residual(Cc, oc.L, 3 * hm.nE, U, bd), R.constraint_residual(rm, rt, rc, uD, 0.3, U))


@needs_ref
@pytest.mark.parametrize("which", [0, 1, 2])
def test_operator_spmv_equals_reference(which):
    hm = O.refine_levels(G.lshape_6tri(), 2)
    om, ot, oc = ocase(hm)
    rm, rt, rc = rcase(hm)
    B, D, M, M0 = O.assemble_volume(hm, COEFFS)
    Cc = O.assemble_constraint(om, ot, oc)["csc"]
    A = O.operator_matrix(B, D, M, M0, Cc, hm.nE, oc.L, which, 0.125)
    n = 3 * hm.nE + oc.L
    x = G.uniform_pm1(8, n)
    bits_equal(O.csc_spmv(A, n, n, x), R.operator_spmv(rm, rt, rc, COEFFS, which, 0.125, x))


# ------------------------------------------------------------------ device
@pytest.fixture(scope="module")
def ctx():
    c = capi.Context(0)
    yield c
    c.close()


def dcase(ctx, hm):
    dm = capi.DeviceMesh.upload(ctx, hm)
    topo = capi.build_topology(ctx, dm)
    return dm, topo, capi.classify_edges(ctx, topo, dm)


ALL_PROBLEMS = PROBLEMS + [("sinsin", capi.PROBLEM_SINSIN, 0.0)]


@pytest.mark.gpu
@pytest.mark.parametrize("mname,make", MESHES, ids=[m[0] for m in MESHES])
@pytest.mark.parametrize("pname,kind,t", ALL_PROBLEMS, ids=[p[0] for p in ALL_PROBLEMS])
def test_gpu_error_norms_and_exact_multiplier(ctx, mname, make, pname, kind, t):
    hm = make()
    om, ot, oc = ocase(hm)
    dm, topo, cls = dcase(ctx, hm)
    pr = capi.problem(kind)
    U = primal_of(hm)
    for h1 in (False, True):
        on, oterms = O.error_norm(hm, U, pr, t, h1=h1)
        dn, dterms = capi.error_norm(ctx, dm, U, pr, t, h1=h1)
        if kind == capi.PROBLEM_SINSIN:  # CUDA sin/cos vs libm: ulps
            np.testing.assert_allclose(dterms, oterms, rtol=1e-12, atol=1e-300)
        else:
            bits_equal(dterms, oterms)
        assert abs(dn - on) <= 1e-12 * abs(on)
    om_ = O.exact_multiplier(om, ot, oc, pr, t)
    dm_ = capi.exact_multiplier(ctx, dm, topo, cls, pr, t)
    if kind == capi.PROBLEM_SINSIN:
        np.testing.assert_allclose(dm_, om_, rtol=1e-12, atol=1e-14)
    else:
        bits_equal(dm_, om_)


@pytest.mark.gpu
@pytest.mark.parametrize("mname,make", MESHES, ids=[m[0] for m in MESHES])
def test_gpu_error_multiplier_traces_residual(ctx, mname, make):
    hm = make()
    om, ot, oc = ocase(hm)
    dm, topo, cls = dcase(ctx, hm)
    exact = O.exact_multiplier(om, ot, oc, capi.problem(capi.PROBLEM_ELLIPTIC_POLY))
    discrete = exact + 1e-3 * G.uniform_pm1(5, oc.L)
    B = O.assemble_volume(hm, COEFFS)[0]
    Cc = O.assemble_constraint(om, ot, oc)["csc"]
    bits_equal(capi.error_multiplier(ctx, dm, topo, cls, B, exact, discrete),
               O.error_multiplier(Cc, oc.L, 3 * hm.nE, B, exact, discrete))
    U = primal_of(hm)
    bits_equal(capi.midpoint_traces(ctx, topo, U), O.midpoint_traces(ot, U))
    uD = capi.field(capi.FIELD_AFFINE, 0.5, 1.0, -2.0, 3.0)
    bd = O.assemble_dirichlet(om, ot, oc, uD, 0.3)
    bits_equal(capi.constraint_residual(ctx, dm, topo, cls, U, bd), O.constraint_residual(Cc, oc.L, 3 * hm.nE, U, bd))
    bits_equal(capi.constraint_residual(ctx, dm, topo, cls, U, None), O.constraint_residual(Cc, oc.L, 3 * hm.nE, U))


@pytest.mark.gpu
def test_gpu_error_multiplier_errors(ctx):
    hm = O.refine_levels(G.crisscross_square(), 1)
    om, ot, oc = ocase(hm)
    dm, topo, cls = dcase(ctx, hm)
    x = np.ones(oc.L)
    B = O.assemble_volume(hm, COEFFS)[0]
    with pytest.raises(ValueError, match="error_multiplier: size mismatch"):
        capi.error_multiplier(ctx, dm, topo, cls, B, x, x[:-1])
    with pytest.raises(capi.PhfemError, match="error_multiplier: all diagonal entries of B vanish"):
        capi.error_multiplier(ctx, dm, topo, cls, -np.abs(B), x, 0.5 * x)
    # some non-positive diagonals: skipped, the rest decide (oracle)
    Bp = B.copy()
    Bp[::2, 0] = -1.0
    ex = O.exact_multiplier(om, ot, oc, capi.problem(capi.PROBLEM_ELLIPTIC_POLY))
    Cc = O.assemble_constraint(om, ot, oc)["csc"]
    bits_equal(capi.error_multiplier(ctx, dm, topo, cls, Bp, ex, 0.9 * ex),
               O.error_multiplier(Cc, oc.L, 3 * hm.nE, Bp, ex, 0.9 * ex))


def host_csr_of(csc, rows):
    outer, inner, vals = csc
    cols = np.repeat(np.arange(len(outer) - 1, dtype=np.int32), np.diff(outer))
    order = np.argsort(inner, kind="stable")
    row_ptr = np.zeros(rows + 1, np.int32)
    np.add.at(row_ptr, inner + 1, 1)
    return np.cumsum(row_ptr).astype(np.int32), cols[order], vals[order]


@pytest.mark.gpu
@pytest.mark.parametrize("which", [0, 1, 2])
def test_gpu_csc_to_csr_and_spmv(ctx, which):
    """M_plus / M_minus / saddle matrix built on the device (f2), converted to
    CSR, multiplied: bit-identical to Eigen's ColMajor SpMV (the oracle)."""
    hm = O.refine_levels(G.lshape_6tri(), 3)
    om, ot, oc = ocase(hm)
    B, D, M, M0 = O.assemble_volume(hm, COEFFS)
    Cc = O.assemble_constraint(om, ot, oc)["csc"]
    A = O.operator_matrix(B, D, M, M0, Cc, hm.nE, oc.L, which, 0.125)
    n = 3 * hm.nE + oc.L
    dev = capi.phfem_csc()
    dev.rows, dev.cols, dev.nnz = n, n, len(A[2])
    dev.outer, dev.inner, dev.values = (ctx.to_device(np.ascontiguousarray(a)) for a in A)
    csr = capi.phfem_csr()
    ctx.check(ctx.lib.phfem_csc_to_csr(ctx.ptr, C.byref(dev), C.byref(csr)))
    want = host_csr_of(A, n)
    got = (ctx.to_host(csr.row_ptr, (n + 1,), np.int32), ctx.to_host(csr.col_idx, (csr.nnz,), np.int32),
           ctx.to_host(csr.values, (csr.nnz,), np.float64))
    for g, w in zip(got, want):
        assert np.array_equal(g.view(np.uint8), np.ascontiguousarray(w).view(np.uint8))
    x = G.uniform_pm1(8, n)
    dx = ctx.to_device(x)
    dy = ctx.alloc(8 * n)
    ctx.check(ctx.lib.phfem_csr_spmv(ctx.ptr, C.byref(csr), C.c_void_p(dx), C.c_void_p(dy)))
    bits_equal(ctx.to_host(dy, (n,), np.float64), O.csc_spmv(A, n, n, x))
    ctx.lib.phfem_csr_release(ctx.ptr, C.byref(csr))
    for p in (dev.outer, dev.inner, dev.values, dx, dy):
        ctx.free(p)


@pytest.mark.gpu
def test_gpu_error_norms_large(ctx):
    """Square L9 (524 K triangles): per-element terms bit-identical, norms
    within 1e-12 of the element-order sum."""
    hm = O.refine_levels(G.square_2tri(), 9)
    dm = capi.DeviceMesh.upload(ctx, hm)
    U = primal_of(hm, seed=11)
    pr = capi.problem(capi.PROBLEM_PARABOLIC_POLY)
    for h1 in (False, True):
        on, oterms = O.error_norm(hm, U, pr, 0.5, h1=h1)
        dn, dterms = capi.error_norm(ctx, dm, U, pr, 0.5, h1=h1)
        bits_equal(dterms, oterms)
        assert abs(dn - on) <= 1e-12 * abs(on)
