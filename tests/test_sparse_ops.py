"""from_triplets (sparse.cpp:30-97) and the solve's operators
(build_saddle_matrix, elliptic.cpp:22-36; step_matrices, parabolic.cpp:21-54).

not gpu: the C oracle's from_triplets and the numpy operator triplets are
pinned BIT FOR BIT to the reference's own sources (oracle/_ref).
gpu: phfem_from_triplets / phfem_saddle_matrix / phfem_step_matrix against
the oracle, bit for bit (patterns and values, -0.0 handling included).
"""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O
from oracle import reference as R
from paper_2401_15557_b200 import capi, meshgen as G


def buffers():
    rng = np.random.default_rng(7)  # test_sparse.cpp:31 uses seed 7 for its own random buffer
    out = []
    for n, rows, cols, dup in ((0, 3, 4, False), (1, 1, 1, False), (200, 9, 7, True), (5000, 60, 50, True),
                               (3000, 2000, 2000, False)):
        ri = rng.integers(0, rows, n).astype(np.int32)
        ci = rng.integers(0, cols, n).astype(np.int32)
        v = rng.standard_normal(n)
        if n > 3:
            v[::17] = -0.0
        out.append((f"random-{n}", rows, cols, ri, ci, v))
    # already row-major sorted and unique: stored as-is (no 0.0 +, -0.0 kept)
    ri = np.array([0, 0, 1, 2, 2], np.int32)
    ci = np.array([0, 3, 1, 0, 2], np.int32)
    out.append(("sorted-unique", 3, 4, ri, ci, np.array([1.5, -0.0, 2.0, -3.0, -0.0])))
    # duplicates: summed in insertion order from 0.0 (test_sparse.cpp:9-16 pattern)
    out.append(("duplicates", 2, 2, np.array([1, 0, 1, 1], np.int32), np.array([1, 0, 1, 1], np.int32),
                np.array([0.1, -0.0, 0.2, 0.3])))
    return out


BUFS = buffers()


def same(a, b):
    for x, y in zip(a, b):
        assert x.shape == y.shape
        assert np.array_equal(x.view(np.uint8) if x.dtype == np.float64 else x,
                              y.view(np.uint8) if y.dtype == np.float64 else y)


@pytest.mark.skipif(not R.available(), reason="reference build unavailable")
@pytest.mark.parametrize("name,rows,cols,ri,ci,v", BUFS, ids=[b[0] for b in BUFS])
def test_oracle_from_triplets_equals_reference(name, rows, cols, ri, ci, v):
    same(O.from_triplets(rows, cols, ri, ci, v), R.from_triplets(rows, cols, ri, ci, v))


@pytest.mark.skipif(not R.available(), reason="reference build unavailable")
def test_from_triplets_out_of_range_message():
    ri, ci, v = np.array([0, 5], np.int32), np.array([0, 1], np.int32), np.array([1.0, 2.0])
    with pytest.raises(IndexError) as eo:
        O.from_triplets(3, 3, ri, ci, v)
    with pytest.raises(IndexError) as er:
        R.from_triplets(3, 3, ri, ci, v)
    assert str(eo.value) == str(er.value) == "TripletBuffer: entry 1 at (5,1) outside 3x3"


def operator_case(hm, coeffs):
    om, ot = O.build_topology(hm)
    oc = O.classify_edges(om, ot)
    B, D, M, M0 = O.assemble_volume(hm, coeffs)
    Cm = O.assemble_constraint(om, ot, oc)
    return om, ot, oc, (B, D, M, M0), Cm["csc"]


OP_MESHES = [("crisscross-L2", lambda: O.refine_levels(G.crisscross_square(), 2)),
             ("lshape-L2", lambda: O.refine_levels(G.lshape_6tri(), 2))]


@pytest.mark.skipif(not R.available(), reason="reference build unavailable")
@pytest.mark.parametrize("name,make", OP_MESHES, ids=[m[0] for m in OP_MESHES])
@pytest.mark.parametrize("which", [0, 1, 2])
def test_oracle_operator_matrices_equal_reference(name, make, which):
    hm = make()
    coeffs = capi.coeffs_const(((2.0, 0.3), (0.3, 1.0)), (1.0, -0.5), 0.7)
    om, ot, oc, (B, D, M, M0), Ccsc = operator_case(hm, coeffs)
    got = O.operator_matrix(B, D, M, M0, Ccsc, hm.nE, oc.L, which, 0.125)
    rm = R.RMesh(hm)
    rt = R.RTopology(rm)
    rc = R.RClassification(rt, rm)
    same(got, R.operator_matrix(rm, rt, rc, coeffs, which, 0.125))


def dev_csc(ctx, csc):
    c = capi.phfem_csc()
    c.rows, c.cols, c.nnz = csc[3], csc[4], len(csc[2])
    c.outer = ctx.to_device(csc[0])
    c.inner = ctx.to_device(csc[1])
    c.values = ctx.to_device(csc[2])
    return c


def host_csc(ctx, c):
    return (ctx.to_host(c.outer, (c.cols + 1,), np.int32), ctx.to_host(c.inner, (c.nnz,), np.int32),
            ctx.to_host(c.values, (c.nnz,), np.float64))


@pytest.mark.gpu
@pytest.mark.parametrize("name,rows,cols,ri,ci,v", BUFS, ids=[b[0] for b in BUFS])
def test_gpu_from_triplets(ctx, name, rows, cols, ri, ci, v):
    out = capi.phfem_csc()
    ctx.check(ctx.lib.phfem_from_triplets(ctx.ptr, rows, cols, C.c_void_p(ctx.to_device(ri)),
                                          C.c_void_p(ctx.to_device(ci)), C.c_void_p(ctx.to_device(v)), len(v),
                                          C.byref(out)))
    same(host_csc(ctx, out), O.from_triplets(rows, cols, ri, ci, v))
    ctx.lib.phfem_csc_release(ctx.ptr, C.byref(out))


@pytest.mark.gpu
def test_gpu_from_triplets_out_of_range(ctx):
    ri, ci, v = np.array([0, 5], np.int32), np.array([0, 1], np.int32), np.array([1.0, 2.0])
    out = capi.phfem_csc()
    with pytest.raises(IndexError, match=r"TripletBuffer: entry 1 at \(5,1\) outside 3x3"):
        ctx.check(ctx.lib.phfem_from_triplets(ctx.ptr, 3, 3, C.c_void_p(ctx.to_device(ri)),
                                              C.c_void_p(ctx.to_device(ci)), C.c_void_p(ctx.to_device(v)), 2,
                                              C.byref(out)))


@pytest.mark.gpu
@pytest.mark.parametrize("name,make", OP_MESHES + [("square-L5", lambda: O.refine_levels(G.square_2tri(), 5))],
                         ids=[m[0] for m in OP_MESHES] + ["square-L5"])
@pytest.mark.parametrize("which", [0, 1, 2])
def test_gpu_operator_matrices(ctx, name, make, which):
    hm = make()
    coeffs = capi.coeffs_const(((2.0, 0.3), (0.3, 1.0)), (1.0, -0.5), 0.7)
    om, ot, oc, (B, D, M, M0), Ccsc = operator_case(hm, coeffs)
    want = O.operator_matrix(B, D, M, M0, Ccsc, hm.nE, oc.L, which, 0.125)
    dB, dD, dM, dM0 = (ctx.to_device(np.ascontiguousarray(x, np.float64)) for x in (B, D, M, M0))
    Cd = dev_csc(ctx, (*Ccsc, oc.L, 3 * hm.nE))
    out = capi.phfem_csc()
    if which == 0:
        ctx.check(ctx.lib.phfem_saddle_matrix(ctx.ptr, hm.nE, C.c_void_p(dB), C.c_void_p(dD), C.c_void_p(dM),
                                              C.byref(Cd), C.byref(out)))
    else:
        ctx.check(ctx.lib.phfem_step_matrix(ctx.ptr, hm.nE, C.c_void_p(dB), C.c_void_p(dD), C.c_void_p(dM),
                                            C.c_void_p(dM0), C.byref(Cd), 0.125, 1.0 if which == 1 else -1.0,
                                            C.byref(out)))
    same(host_csc(ctx, out), want)
    ctx.lib.phfem_csc_release(ctx.ptr, C.byref(out))


def big_buffers():
    """Multi-tile, multi-digit inputs for the hand-written radix sort
    (csrc/radix_sort.cu): heavy duplicates (stability decides the run sums),
    wide keys (5 digit passes), one hot column, reversed order."""
    rng = np.random.default_rng(2024)
    out = []
    n = 3_000_000
    out.append(("dups-3M", 3000, 2500, rng.integers(0, 3000, n).astype(np.int32),
                rng.integers(0, 2500, n).astype(np.int32), rng.standard_normal(n)))
    n = 2_000_000
    out.append(("wide-2M", 1 << 20, 1 << 20, rng.integers(0, 1 << 20, n).astype(np.int32),
                rng.integers(0, 1 << 20, n).astype(np.int32), rng.standard_normal(n)))
    n = 500_000
    out.append(("hot-column", 100_000, 64, rng.integers(0, 100_000, n).astype(np.int32),
                np.where(rng.random(n) < 0.9, 7, rng.integers(0, 64, n)).astype(np.int32), rng.standard_normal(n)))
    r = np.repeat(np.arange(999, -1, -1, dtype=np.int32), 700)
    c = np.tile(np.arange(699, -1, -1, dtype=np.int32), 1000)
    out.append(("reversed-unique", 1000, 700, r, c, rng.standard_normal(r.size)))
    return out


BIG = big_buffers()


@pytest.mark.gpu
@pytest.mark.parametrize("name,rows,cols,ri,ci,v", BIG, ids=[b[0] for b in BIG])
def test_gpu_from_triplets_large(ctx, name, rows, cols, ri, ci, v):
    out = capi.phfem_csc()
    ctx.check(ctx.lib.phfem_from_triplets(ctx.ptr, rows, cols, C.c_void_p(ctx.to_device(ri)),
                                          C.c_void_p(ctx.to_device(ci)), C.c_void_p(ctx.to_device(v)), len(v),
                                          C.byref(out)))
    same(host_csc(ctx, out), O.from_triplets(rows, cols, ri, ci, v))
    ctx.lib.phfem_csc_release(ctx.ptr, C.byref(out))


@pytest.mark.gpu
@pytest.mark.parametrize("which", [0, 2])
def test_gpu_operator_matrices_L9(ctx, which):
    """Saddle / CN step matrix of the square at L9 (524,288 triangles, ~11 M
    triplets, 3 digit passes): the device-resident inputs of the excluded solve."""
    hm = O.refine_levels(G.square_2tri(), 9)
    coeffs = capi.coeffs_const(((2.0, 0.3), (0.3, 1.0)), (1.0, -0.5), 0.7)
    om, ot, oc, (B, D, M, M0), Ccsc = operator_case(hm, coeffs)
    want = O.operator_matrix(B, D, M, M0, Ccsc, hm.nE, oc.L, which, 1e-3)
    dB, dD, dM, dM0 = (ctx.to_device(np.ascontiguousarray(x, np.float64)) for x in (B, D, M, M0))
    Cd = dev_csc(ctx, (*Ccsc, oc.L, 3 * hm.nE))
    out = capi.phfem_csc()
    if which == 0:
        ctx.check(ctx.lib.phfem_saddle_matrix(ctx.ptr, hm.nE, C.c_void_p(dB), C.c_void_p(dD), C.c_void_p(dM),
                                              C.byref(Cd), C.byref(out)))
    else:
        ctx.check(ctx.lib.phfem_step_matrix(ctx.ptr, hm.nE, C.c_void_p(dB), C.c_void_p(dD), C.c_void_p(dM),
                                            C.c_void_p(dM0), C.byref(Cd), 1e-3, -1.0, C.byref(out)))  # M_minus
    same(host_csc(ctx, out), want)
    ctx.lib.phfem_csc_release(ctx.ptr, C.byref(out))
