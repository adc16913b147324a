"""Parity of the CUDA path (through the C ABI) against the CPU oracle on the same
seeded inputs.  Integer outputs (edges, maps, signs, refined meshes, CSR/CSC
patterns) must be bit-exact; fp64 values bit-exact where the expression is
+-*/sqrt only, and within 1e-12 relative (BASELINE north_star) where libm
sin/cos/exp enter (load, Neumann, CN data terms)."""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_2401_15557_b200 import capi, meshgen as G

pytestmark = pytest.mark.gpu

REL_TOL = 1e-12  # north_star: fp64 values within 1e-12 relative per entry


def rel_close(a, b, tol=REL_TOL, floor=0.0):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape
    scale = np.maximum(np.abs(b), floor)
    err = np.abs(a - b)
    ok = (err <= tol * scale) | (a == b)
    if not ok.all():
        i = np.argmax(np.where(ok, 0, err / np.maximum(scale, 1e-300)))
        raise AssertionError(f"{(~ok).sum()} entries off, worst {a.flat[i]!r} vs {b.flat[i]!r}")


def check_topology(gt: dict, ot: dict):
    for k in ["edge_nodes", "edge_elements", "local_in_tplus", "local_in_tminus", "interior_edges",
              "boundary_edges", "elem_edge", "node_edge_start"]:
        assert np.array_equal(gt[k], ot[k]), k


def check_cls(gc: dict, oc: dict):
    for k in ["dirichlet_edge_ids", "neumann_edge_ids", "retained_edges", "retained_pos"]:
        assert np.array_equal(gc[k], oc[k]), k


def gpu_all(ctx, hm, coeffs, f, g, uD, t=0.0):
    dm = capi.DeviceMesh.upload(ctx, hm)
    topo = capi.build_topology(ctx, dm)
    cls = capi.classify_edges(ctx, topo, dm)
    B, D, M, M0 = capi.assemble_volume(ctx, dm, coeffs)
    res = {
        "topo": topo.download(), "cls": cls.download(), "B": B, "D": D, "M": M, "M0": M0,
        "C_csr": capi.assemble_constraint(ctx, dm, topo, cls),
        "C_csc": capi.constraint_csc(ctx, dm, topo, cls),
        "b": capi.assemble_load(ctx, dm, f, t),
        "ln": capi.assemble_neumann(ctx, dm, topo, cls, g, t),
        "bd": capi.assemble_dirichlet(ctx, dm, topo, cls, uD, t),
        "refined": capi.red_refine(ctx, dm, topo).download(),
    }
    return res


def oracle_all(hm, coeffs, f, g, uD, t=0.0):
    om, topo = O.build_topology(hm)
    cls = O.classify_edges(om, topo)
    B, D, M, M0 = O.assemble_volume(hm, coeffs)
    C = O.assemble_constraint(om, topo, cls)
    return {
        "topo": topo.arrays(), "cls": cls.arrays(), "B": B, "D": D, "M": M, "M0": M0,
        "C_csr": C["csr"], "C_csc": C["csc"], "b": O.assemble_load(hm, f, t),
        "ln": O.assemble_neumann(om, topo, cls, g, t), "bd": O.assemble_dirichlet(om, topo, cls, uD, t),
        "refined": O.red_refine(hm, topo),
    }


def compare_all(gr, orr, exact_loads=False):
    check_topology(gr["topo"], orr["topo"])
    check_cls(gr["cls"], orr["cls"])
    for k in ["B", "D", "M", "M0"]:
        assert np.array_equal(gr[k], orr[k]), k  # +-*/ only: bit-exact
    for k in ["C_csr", "C_csc"]:
        for a, b in zip(gr[k], orr[k]):
            assert np.array_equal(a, b), k
    rg, ro = gr["refined"], orr["refined"]
    assert np.array_equal(rg.coords, ro.coords)
    assert np.array_equal(rg.elements, ro.elements)
    assert np.array_equal(rg.dirichlet, ro.dirichlet)
    assert np.array_equal(rg.neumann, ro.neumann)
    for k in ["b", "ln", "bd"]:
        if exact_loads:
            assert np.array_equal(gr[k], orr[k]), k
        else:
            rel_close(gr[k], orr[k])


# ------------------------------------------------------------------ KATs on GPU
def test_crisscross_kat_gpu(ctx):
    hm = G.crisscross_square()
    dm = capi.DeviceMesh.upload(ctx, hm)
    t = capi.build_topology(ctx, dm).download()
    expected = [(0, 1, 0, -1), (2, 0, 1, -1), (1, 3, 3, -1), (3, 2, 2, -1),
                (4, 0, 0, 1), (1, 4, 0, 3), (4, 2, 1, 2), (4, 3, 2, 3)]
    assert [tuple(t["edge_nodes"][e]) + tuple(t["edge_elements"][e]) for e in range(8)] == expected
    assert t["local_in_tplus"].tolist() == [0, 0, 0, 0, 2, 1, 2, 2]
    assert t["local_in_tminus"].tolist() == [-1, -1, -1, -1, 1, 2, 1, 1]
    assert t["interior_edges"].tolist() == [4, 5, 6, 7]
    assert t["boundary_edges"].tolist() == [0, 1, 2, 3]


@pytest.mark.parametrize("mesh_fn", [G.crisscross_square, G.unit_right_triangle, G.square_2tri,
                                     G.lshape_6tri])
def test_small_meshes_all_outputs(ctx, mesh_fn):
    hm = mesh_fn()
    for level in range(4):
        args = G.config_fields(2)
        compare_all(gpu_all(ctx, hm, *args), oracle_all(hm, *args))
        hm = O.red_refine(hm)


@pytest.mark.parametrize("k,last", [(40, True), (40, False), (700, True), (3000, True), (3000, False)])
def test_high_valence_fans(ctx, k, last):
    """Nodes with > 32 occurrences / tiles beyond SMEM take the fallback paths."""
    hm = G.fan(k, last)
    args = G.config_fields(2)
    compare_all(gpu_all(ctx, hm, *args), oracle_all(hm, *args))


def test_permuted_node_ids(ctx):
    """Random node relabelling + element permutation of a refined L-shape."""
    hm = O.refine_levels(G.lshape_6tri(), 4)
    perm = np.argsort(G.splitmix64(11, hm.nC), kind="stable")
    inv = np.empty_like(perm)
    inv[perm] = np.arange(hm.nC)
    coords = hm.coords[perm]
    m = capi.HostMesh(coords, inv[hm.elements], inv[hm.dirichlet], inv[hm.neumann])
    m = capi.HostMesh(m.coords, m.elements[np.argsort(G.splitmix64(12, m.nE), kind="stable")],
                      m.dirichlet, m.neumann)
    args = G.config_fields(2)
    compare_all(gpu_all(ctx, m, *args), oracle_all(m, *args))


@pytest.mark.parametrize("name", ["crisscross", "square", "lshape", "stress", "fan", "permuted"])
def test_refine_topology_equals_sorted_build(ctx, name):
    """the sort-free topology of the refined mesh is bit-identical
    to the reference's sort-based build_topology(red_refine(M)) (oracle) and to
    the device's generic build_topology."""
    if name == "crisscross":
        hm = O.refine_levels(G.crisscross_square(), 2)
    elif name == "square":
        hm = O.refine_levels(G.square_2tri(), 5)
    elif name == "lshape":
        hm = O.refine_levels(G.lshape_6tri(), 4)
    elif name == "stress":
        hm = O.orient_ccw(G.stress_transform(O.refine_levels(G.square_2tri(), 5), 5))
    elif name == "fan":
        hm = G.fan(50, True)
    else:
        base = O.refine_levels(G.lshape_6tri(), 3)
        perm = np.argsort(G.splitmix64(21, base.nC), kind="stable")
        inv = np.empty_like(perm)
        inv[perm] = np.arange(base.nC)
        hm = capi.HostMesh(base.coords[perm], inv[base.elements][np.argsort(G.splitmix64(22, base.nE))],
                           inv[base.dirichlet], inv[base.neumann])
    dm = capi.DeviceMesh.upload(ctx, hm)
    topo = capi.build_topology(ctx, dm)
    fine = capi.red_refine(ctx, dm, topo)
    fast = capi.refine_topology(ctx, dm, topo, fine).download()
    generic = capi.build_topology(ctx, fine).download()
    _, ot = O.build_topology(O.red_refine(hm))
    check_topology(fast, ot.arrays())
    check_topology(generic, ot.arrays())


@pytest.mark.parametrize("name", ["crisscross", "square", "lshape", "stress", "alldirichlet"])
def test_refine_level_fused(ctx, name):
    """Fused refined level (topology + classification + C) == oracle on the fine mesh."""
    if name == "crisscross":
        hm = O.refine_levels(G.crisscross_square(), 2)
    elif name == "square":
        hm = O.refine_levels(G.square_2tri(), 5)
    elif name == "lshape":
        hm = O.refine_levels(G.lshape_6tri(), 4)
    elif name == "stress":
        hm = O.orient_ccw(G.stress_transform(O.refine_levels(G.square_2tri(), 5), 5))
    else:
        base = O.refine_levels(G.crisscross_square(), 2)
        hm = capi.HostMesh(base.coords, base.elements, np.vstack([base.dirichlet, base.neumann]),
                           np.zeros((0, 2)))
    dm = capi.DeviceMesh.upload(ctx, hm)
    topo = capi.build_topology(ctx, dm)
    cls = capi.classify_edges(ctx, topo, dm)
    fine = capi.red_refine(ctx, dm, topo)
    ft, fc, fC = capi.refine_level(ctx, dm, topo, cls, fine)
    fh = O.red_refine(hm)
    om, ot = O.build_topology(fh)
    oc = O.classify_edges(om, ot)
    check_topology(ft.download(), ot.arrays())
    check_cls(fc.download(), oc.arrays())
    for a, b in zip(fC, O.assemble_constraint(om, ot, oc)["csr"]):
        assert np.array_equal(a, b)


def test_pipeline_generic_and_fused_agree(ctx):
    hm = G.lshape_6tri()
    args = G.config_fields(2)
    a = capi.pipeline(ctx, capi.DeviceMesh.upload(ctx, hm), 4, *args).download()
    b = capi.pipeline(ctx, capi.DeviceMesh.upload(ctx, hm), 4, *args, flags=capi.PIPE_GENERIC_EG).download()
    check_topology(a["topo"], b["topo"])
    for k in ["B", "C_row_ptr", "C_col_idx", "C_values", "load", "bd"]:
        assert np.array_equal(a[k], b[k]), k


def test_error_paths_match_reference(ctx):
    tri = G.unit_right_triangle()
    bad = capi.HostMesh(np.vstack([tri.coords, [[1, 1]]]), np.vstack([tri.elements, [[0, 1, 3]]]),
                        tri.dirichlet, tri.neumann)
    pinched = capi.HostMesh(np.vstack([tri.coords, [[1, 1], [-1, 1]]]),
                            np.vstack([tri.elements, [[1, 0, 3], [0, 1, 4]]]), tri.dirichlet, tri.neumann)
    for m in (bad, pinched):
        with pytest.raises(RuntimeError) as eo:
            O.build_topology(m)
        with pytest.raises(RuntimeError) as eg:
            capi.build_topology(ctx, capi.DeviceMesh.upload(ctx, m))
        assert str(eg.value) == str(eo.value)
    cc = G.crisscross_square()
    for m in (capi.HostMesh(cc.coords, cc.elements, cc.dirichlet, np.vstack([cc.neumann, [[0, 3]]])),
              capi.HostMesh(cc.coords, cc.elements, np.vstack([cc.dirichlet, [[4, 0]]]), cc.neumann)):
        om, ot = O.build_topology(m)
        with pytest.raises(RuntimeError) as eo:
            O.classify_edges(om, ot)
        dm = capi.DeviceMesh.upload(ctx, m)
        with pytest.raises(RuntimeError) as eg:
            capi.classify_edges(ctx, capi.build_topology(ctx, dm), dm)
        assert str(eg.value) == str(eo.value)
    degen = capi.HostMesh(np.array([[0, 0], [1, 0], [2, 0]], float), np.array([[0, 1, 2]]),
                          np.zeros((0, 2)), np.zeros((0, 2)))
    with pytest.raises(RuntimeError, match="degenerate or non-CCW"):
        capi.assemble_volume(ctx, capi.DeviceMesh.upload(ctx, degen), capi.coeffs_const())
    big = O.red_refine(cc)
    with pytest.raises(RuntimeError) as eo:
        O.assemble_load(big, capi.field(capi.FIELD_NAN))
    with pytest.raises(RuntimeError) as eg:
        capi.assemble_load(ctx, capi.DeviceMesh.upload(ctx, big), capi.field(capi.FIELD_NAN))
    assert str(eg.value) == str(eo.value) == "assemble_load: non-finite load sample in element 1"


def test_empty_mesh(ctx):
    hm = capi.HostMesh(np.zeros((0, 2)), np.zeros((0, 3)), np.zeros((0, 2)), np.zeros((0, 2)))
    dm = capi.DeviceMesh.upload(ctx, hm)
    t = capi.build_topology(ctx, dm)
    assert t.E == 0
    c = capi.classify_edges(ctx, t, dm)
    assert c.L == 0


# ------------------------------------------------------------------ configs
def test_config1_l6_full_parity(ctx):
    """BASELINE configs[0]: square, 6 refinements -> 8192 triangles, A=I, f=2pi^2 sin sin,
    D on x=0,y=0, N on x=1,y=1 (g = grad u . nu)."""
    hm = G.square_2tri()
    args = G.config_fields(1)
    for level in range(6):
        hmo = O.red_refine(hm)
        dm = capi.DeviceMesh.upload(ctx, hm)
        hmg = capi.red_refine(ctx, dm, capi.build_topology(ctx, dm)).download()
        assert np.array_equal(hmg.coords, hmo.coords) and np.array_equal(hmg.elements, hmo.elements)
        hm = hmo
    assert hm.nE == 8192
    compare_all(gpu_all(ctx, hm, *args), oracle_all(hm, *args))


def test_config2_lshape_variable_coefficients(ctx):
    hm = O.refine_levels(G.lshape_6tri(), 5)
    args = G.config_fields(2)
    compare_all(gpu_all(ctx, hm, *args), oracle_all(hm, *args))


def test_config4_stress_mesh(ctx):
    """jitter / permutation / rotation / +-orientation, normalised (a18), then
    edge generation, one refinement and full assembly — reduced to L6 -> L7."""
    level = 6
    hm = G.stress_transform(O.refine_levels(G.square_2tri(), level), level)
    assert (G.signed_area2(hm) < 0).any()
    hmo = O.orient_ccw(hm)
    dm = capi.DeviceMesh.upload(ctx, hm)
    capi.orient_ccw(ctx, dm)
    hmg = dm.download()
    assert np.array_equal(hmg.elements, hmo.elements)
    assert (G.signed_area2(hmo) > 0).all()
    args = G.config_fields(4)
    compare_all(gpu_all(ctx, hmo, *args), oracle_all(hmo, *args))
    fine = O.red_refine(hmo)
    compare_all(gpu_all(ctx, fine, *args), oracle_all(fine, *args))


def test_pipeline_equals_pieces(ctx):
    hm = G.lshape_6tri()
    args = G.config_fields(2)
    dm = capi.DeviceMesh.upload(ctx, hm)
    r = capi.pipeline(ctx, dm, 4, *args).download()
    o = O.pipeline(hm, 4, *args)
    assert np.array_equal(r["mesh"].coords, o["mesh"].coords)
    assert np.array_equal(r["mesh"].elements, o["mesh"].elements)
    check_topology(r["topo"], o["topo"])
    check_cls(r["cls"], o["cls"])
    for k in ["B", "D", "M", "M0"]:
        assert np.array_equal(r[k], o[k])
    for a, b in zip((r["C_row_ptr"], r["C_col_idx"], r["C_values"]), o["C_csr"]):
        assert np.array_equal(a, b)
    rel_close(r["load"], o["load"])
    rel_close(r["bd"], o["bd"])


@pytest.mark.parametrize("case", ["lshape_l3", "stress_l5_l2", "square_l1"])
def test_pipeline_volume_from_parents(ctx, monkeypatch, case):
    """The pipeline's element pass rebuilds the refined children's vertices
    from the last parent mesh (VolArgs::parents: 3 parent gathers per 4
    children, midpoints 0.5 * (a + b) recomputed, refine.cpp:18,27-37).  Its
    blocks and load must equal the oracle and the path that reads the refined
    mesh (PHFEM_VOL_PARENTS=0) bit for bit: a partial last chunk (6 x 4^k
    children), the permuted / jittered stress mesh, and a 2-parent level."""
    if case == "lshape_l3":
        hm, levels, cfg = G.lshape_6tri(), 3, 2
    elif case == "stress_l5_l2":
        hm, levels, cfg = O.orient_ccw(G.stress_transform(O.refine_levels(G.square_2tri(), 5), 5)), 2, 2
    else:
        hm, levels, cfg = G.square_2tri(), 1, 1
    args = G.config_fields(cfg)
    outs = []
    for flag in ("1", "0"):
        monkeypatch.setenv("PHFEM_VOL_PARENTS", flag)
        outs.append(capi.pipeline(ctx, capi.DeviceMesh.upload(ctx, hm), levels, *args).download())
    o = O.pipeline(hm, levels, *args)
    for k in ["B", "D", "M", "M0", "load"]:
        assert np.array_equal(outs[0][k], outs[1][k]), k
    for k in ["B", "D", "M", "M0"]:
        assert np.array_equal(outs[0][k], o[k]), k
    rel_close(outs[0]["load"], o["load"])


def test_pipeline_config1_neumann(ctx):
    hm = G.square_2tri()
    args = G.config_fields(1)
    r = capi.pipeline(ctx, capi.DeviceMesh.upload(ctx, hm), 5, *args).download()
    o = O.pipeline(hm, 5, *args)
    rel_close(r["load"], o["load"])


@pytest.mark.parametrize("lam", ["random", "zero"])
def test_cn_rhs_config3(ctx, lam):
    """Config 3 (reduced to L6): W ~ U[-1,1] seed 5, k = 1e-3, every 10th step."""
    hm = O.refine_levels(G.square_2tri(), 6)
    coeffs, f, g, uD = G.config_fields(3)
    om, ot = O.build_topology(hm)
    oc = O.classify_edges(om, ot)
    N, L = 3 * hm.nE, oc.L
    W = G.uniform_pm1(5, N + L)
    if lam == "zero":
        W[N:] = 0.0
    dm = capi.DeviceMesh.upload(ctx, hm)
    topo = capi.build_topology(ctx, dm)
    cls = capi.classify_edges(ctx, topo, dm)
    plan = capi.CNPlan(ctx, dm, topo, cls, coeffs, f, g, uD, 1e-3)
    for n in range(0, 100, 10):
        rg = plan.rhs(n, W)
        ro = O.cn_rhs(om, ot, oc, coeffs, f, g, uD, 1e-3, n, W)
        rel_close(rg, ro)


def test_cn_rhs_with_boundary_data(ctx):
    """Neumann + Dirichlet data and a convective / reactive operator."""
    hm = O.refine_levels(G.crisscross_square(), 3)
    coeffs = capi.coeffs_const(((2.0, 0.3), (0.3, 1.0)), (1.0, -0.5), 0.7)
    f = capi.field(capi.FIELD_EXP_SINSIN, capi.TWO_PI2_M1)
    g = capi.field(capi.FLUX_GRAD_SINSIN, 1.0)
    uD = capi.field(capi.FIELD_AFFINE, 0.5, 1.0, -2.0, 3.0)
    om, ot = O.build_topology(hm)
    oc = O.classify_edges(om, ot)
    W = G.uniform_pm1(9, 3 * hm.nE + oc.L)
    dm = capi.DeviceMesh.upload(ctx, hm)
    topo = capi.build_topology(ctx, dm)
    cls = capi.classify_edges(ctx, topo, dm)
    plan = capi.CNPlan(ctx, dm, topo, cls, coeffs, f, g, uD, 0.125)
    for n in (0, 3):
        rel_close(plan.rhs(n, W), O.cn_rhs(om, ot, oc, coeffs, f, g, uD, 0.125, n, W), floor=1e-300)


@pytest.mark.parametrize("aligned", [True, False])
def test_cn_rhs_tail_tile_and_unaligned_state(ctx, aligned):
    """832 triangles = 6.5 TMA tiles (bulk-copy tiles + the plain-load tail),
    Dirichlet data on the ring; unaligned state / rhs pointers take the
    plain-load kernel for every element.  Same bits either way."""
    hm = O.refine_levels(G.fan(13), 3)
    coeffs, f, g, _ = G.config_fields(3)
    uD = capi.field(capi.FIELD_AFFINE, 0.5, 1.0, -2.0, 3.0)
    om, ot = O.build_topology(hm)
    oc = O.classify_edges(om, ot)
    n_state = 3 * hm.nE + oc.L
    W = G.uniform_pm1(11, n_state)
    dm = capi.DeviceMesh.upload(ctx, hm)
    topo = capi.build_topology(ctx, dm)
    cls = capi.classify_edges(ctx, topo, dm)
    plan = capi.CNPlan(ctx, dm, topo, cls, coeffs, f, g, uD, 1e-3)
    off = 0 if aligned else 1
    s = ctx.to_device(np.concatenate([np.zeros(off), W]))
    r = ctx.alloc(8 * (n_state + off))
    try:
        for n in (0, 7):
            plan.rhs_device(n, s + 8 * off, r + 8 * off)
            rg = ctx.to_host(r + 8 * off, (n_state,), np.float64)
            rel_close(rg, O.cn_rhs(om, ot, oc, coeffs, f, g, uD, 1e-3, n, W), floor=1e-300)
    finally:
        ctx.free(s)
        ctx.free(r)


# ------------------------------------------------------------------ large sizes
def test_large_refinement_properties(ctx):
    """Square L11 (8.4 M triangles, config 3's mesh) on the device only:
    size-independent properties of the outputs."""
    hm = G.square_2tri()
    dm = capi.DeviceMesh.upload(ctx, hm)
    r = capi.pipeline(ctx, dm, 11, *G.config_fields(1))
    o = r.out
    nE, nC, E = o.mesh.nE, o.mesh.nC, o.topo.E
    assert nE == 2 * 4 ** 11
    assert E == nE + nC - 1                              # Euler, simply connected
    assert 3 * nE == 2 * o.topo.n_interior + o.topo.n_boundary
    t = r.topo_view().download()
    en = t["edge_nodes"]
    hi, lo = en.max(axis=1).astype(np.int64), en.min(axis=1).astype(np.int64)
    key = hi * nC + lo
    assert (np.diff(key) > 0).all()                      # canonical (max, min) order, unique
    assert (t["node_edge_start"][hi] <= np.arange(E)).all()
    ee = t["elem_edge"]
    e_abs = np.where(ee >= 0, ee, ~ee)
    tp = t["edge_elements"][:, 0]
    assert (tp[e_abs[ee >= 0]] == np.nonzero(ee >= 0)[0]).all()      # sign +1 <=> t_plus
    rp = r.out.C
    row_ptr = r.ctx.to_host(rp.row_ptr, (r.out.cls.L + 1,), np.int32)
    assert row_ptr[-1] == rp.nnz and (np.diff(row_ptr) >= 2).all()
    r.release()


@pytest.mark.gpu
def test_fastmath_selftest(ctx):
    """The element kernels divide through one correctly rounded reciprocal per
    element (csrc/fastmath.cuh, Markstein); the blocks are bit-exact only if
    that division equals IEEE '/' on every operand — 2^28 random pairs in three
    families (wide exponents, quotients at binade boundaries, mesh-like
    geometry) must show zero mismatches.  The fast sin stays within 2 ulp of
    CUDA's sin."""
    import ctypes as C
    out = (C.c_ulonglong * 3)()
    ctx.check(ctx.lib.phfem_selftest_fastmath(ctx.ptr, 1 << 28, 20241015, out))
    assert out[0] == 0, f"{out[0]} fast divisions differ from IEEE division"
    assert out[2] == 0, f"{out[2]} divisions by 3 differ"
    assert out[1] <= 2, f"sin_fast off by {out[1]} ulp"


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["square-L4-1", "lshape-L3-1", "crisscross-L2-0"])
def test_host_buffer_pipeline_equals_device_outputs(ctx, case):
    """phfem_pipeline_from_host + phfem_pipeline_download (the drop-in / e2e
    path: compact PCIe encodings expanded on the host) reproduce every device
    output bit for bit, for full and partial selections of outputs."""
    import ctypes as Cc
    name, lv, levels = case.rsplit("-", 2)[0], int(case.split("-")[1][1:]), int(case.rsplit("-", 1)[1])
    base = {"square": G.square_2tri, "lshape": G.lshape_6tri, "crisscross": G.crisscross_square}[name.split("-")[0]]
    hm = O.refine_levels(base(), lv)
    args = G.config_fields(2 if name != "crisscross" else 1)
    ref = capi.pipeline(ctx, capi.DeviceMesh.upload(ctx, hm), levels, *args).download()
    out = capi.phfem_pipeline_out()
    ctx.check(ctx.lib.phfem_pipeline_from_host(
        ctx.ptr, hm.coords.ctypes.data_as(Cc.c_void_p), hm.elements.ctypes.data_as(Cc.c_void_p),
        hm.dirichlet.ctypes.data_as(Cc.c_void_p), hm.neumann.ctypes.data_as(Cc.c_void_p), hm.nC, hm.nE,
        len(hm.dirichlet), len(hm.neumann), levels, Cc.byref(args[0]), Cc.byref(args[1]), Cc.byref(args[2]),
        Cc.byref(args[3]), 0.0, Cc.byref(out)))
    o = out
    shapes = {"coords": ((o.mesh.nC, 2), np.float64), "elements": ((o.mesh.nE, 3), np.int32),
              "edge_nodes": ((o.topo.E, 2), np.int32), "edge_elements": ((o.topo.E, 2), np.int32),
              "local_in_tplus": ((o.topo.E,), np.int32), "local_in_tminus": ((o.topo.E,), np.int32),
              "elem_edge": ((o.mesh.nE, 3), np.int32), "retained_edges": ((o.cls.L,), np.int32),
              "retained_pos": ((o.topo.E,), np.int32), "C_row_ptr": ((o.cls.L + 1,), np.int32),
              "C_col_idx": ((o.C.nnz,), np.int32), "C_values": ((o.C.nnz,), np.float64),
              "B": ((o.mesh.nE, 9), np.float64), "D": ((o.mesh.nE, 9), np.float64),
              "M": ((o.mesh.nE, 9), np.float64), "M0": ((o.mesh.nE, 9), np.float64),
              "load": ((3 * o.mesh.nE,), np.float64), "bd": ((o.cls.L,), np.float64)}
    for sel in (list(shapes), ["B", "M0", "C_values", "local_in_tminus", "load"]):
        bufs = {k: np.full(shapes[k][0], -7, dtype=shapes[k][1]) for k in sel}
        dst = capi.phfem_pipeline_host(**{k: bufs[k].ctypes.data for k in sel})
        ctx.check(ctx.lib.phfem_pipeline_download(ctx.ptr, Cc.byref(out), Cc.byref(dst)))
        want = {"coords": ref["mesh"].coords, "elements": ref["mesh"].elements, **ref["topo"], **ref["cls"],
                **{k: ref[k] for k in ("C_row_ptr", "C_col_idx", "C_values", "B", "D", "M", "M0", "load", "bd")}}
        for k in sel:
            a, b = bufs[k].reshape(-1), np.asarray(want[k]).reshape(-1)
            assert a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8)), k
    ctx.lib.phfem_pipeline_release(ctx.ptr, Cc.byref(out))
