"""Pins the CPU oracle (oracle/phfem_oracle.c) to the reference's own
known-answer tests for the hot path, re-encoded from
/root/reference/proj/tests/{test_topology,test_refine,test_assembly,test_sparse}.cpp
and the paper's Example 1.  No GPU needed."""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_2401_15557_b200 import capi, meshgen as G


def crisscross():
    return G.crisscross_square()


# ---------------------------------------------------------------- topology
def test_crisscross_edge_table():  # test_topology.cpp:15-47
    om, t = O.build_topology(crisscross())
    a = t.arrays()
    expected = [(0, 1, 0, -1), (2, 0, 1, -1), (1, 3, 3, -1), (3, 2, 2, -1),
                (4, 0, 0, 1), (1, 4, 0, 3), (4, 2, 1, 2), (4, 3, 2, 3)]
    got = [tuple(a["edge_nodes"][e]) + tuple(a["edge_elements"][e]) for e in range(8)]
    assert got == expected
    assert a["interior_edges"].tolist() == [4, 5, 6, 7]
    assert a["boundary_edges"].tolist() == [0, 1, 2, 3]
    assert a["local_in_tplus"].tolist() == [0, 0, 0, 0, 2, 1, 2, 2]
    assert a["local_in_tminus"].tolist() == [-1, -1, -1, -1, 1, 2, 1, 1]


def test_example1_lookup_matrices():  # PAPER.md:245-264 (1-based, 0 = none)
    om, t = O.build_topology(crisscross())
    n2el = [[0, 1, 0, 0, 2], [0, 0, 0, 4, 1], [2, 0, 0, 0, 3], [0, 0, 3, 0, 4], [1, 4, 2, 3, 0]]
    n2ed = [[0, 1, 2, 0, 5], [1, 0, 0, 3, 6], [2, 0, 0, 4, 7], [0, 3, 4, 0, 8], [5, 6, 7, 8, 0]]
    for k in range(5):
        for l in range(5):
            assert t.directed_pair_to_element(k, l) + 1 == n2el[k][l]
            assert t.node_pair_to_edge(k, l) + 1 == n2ed[k][l]
    e2el = [[1, 2, 1, 0], [3, 1, 2, 0], [2, 4, 4, 0], [4, 3, 3, 0],
            [5, 1, 1, 2], [2, 5, 1, 4], [5, 3, 2, 3], [5, 4, 3, 4]]
    a = t.arrays()
    for e in range(8):
        row = list(a["edge_nodes"][e] + 1) + list(a["edge_elements"][e] + 1)
        assert row == e2el[e]


def test_lookups():  # test_topology.cpp:49-63
    om, t = O.build_topology(crisscross())
    assert t.directed_pair_to_element(0, 1) == 0
    assert t.directed_pair_to_element(2, 0) == 1
    assert t.directed_pair_to_element(1, 0) == -1
    assert t.directed_pair_to_element(0, 3) == -1
    assert t.node_pair_to_edge(0, 1) == 0 and t.node_pair_to_edge(1, 0) == 0
    assert t.node_pair_to_edge(0, 4) == 4 and t.node_pair_to_edge(4, 0) == 4
    assert t.node_pair_to_edge(0, 3) == -1


def test_single_triangle():  # test_topology.cpp:65-72
    om, t = O.build_topology(G.unit_right_triangle())
    a = t.arrays()
    assert t.t.E == 3 and len(a["boundary_edges"]) == 3 and len(a["interior_edges"]) == 0
    assert a["local_in_tplus"].tolist() == [2, 1, 0]


def test_topology_errors():  # test_topology.cpp:74-88
    bad = G.unit_right_triangle()
    bad = capi.HostMesh(np.vstack([bad.coords, [[1, 1]]]), np.vstack([bad.elements, [[0, 1, 3]]]),
                        bad.dirichlet, bad.neumann)
    with pytest.raises(RuntimeError, match="duplicate directed"):
        O.build_topology(bad)
    p = G.unit_right_triangle()
    pinched = capi.HostMesh(np.vstack([p.coords, [[1, 1], [-1, 1]]]),
                            np.vstack([p.elements, [[1, 0, 3], [0, 1, 4]]]), p.dirichlet, p.neumann)
    with pytest.raises(RuntimeError, match="non-manifold"):
        O.build_topology(pinched)


def test_classification():  # test_topology.cpp:90-126
    hm = crisscross()
    om, t = O.build_topology(hm)
    c = O.classify_edges(om, t).arrays()
    assert c["dirichlet_edge_ids"].tolist() == [0, 2]
    assert c["neumann_edge_ids"].tolist() == [3, 1]
    assert c["retained_edges"].tolist() == [0, 2, 4, 5, 6, 7]
    assert c["retained_pos"][0] == 0 and c["retained_pos"][1] == -1 and c["retained_pos"][7] == 5
    alld = capi.HostMesh(hm.coords, hm.elements, np.vstack([hm.dirichlet, hm.neumann]), np.zeros((0, 2)))
    om2, t2 = O.build_topology(alld)
    assert O.classify_edges(om2, t2).L == t2.t.E
    m1 = capi.HostMesh(hm.coords, hm.elements, hm.dirichlet, np.vstack([hm.neumann, [[0, 3]]]))
    om3, t3 = O.build_topology(m1)
    with pytest.raises(RuntimeError, match="not an edge"):
        O.classify_edges(om3, t3)
    m2 = capi.HostMesh(hm.coords, hm.elements, np.vstack([hm.dirichlet, [[4, 0]]]), hm.neumann)
    om4, t4 = O.build_topology(m2)
    with pytest.raises(RuntimeError, match="interior"):
        O.classify_edges(om4, t4)


def test_lengths_normals_euler():  # test_topology.cpp:128-187
    hm = crisscross()
    om, t = O.build_topology(hm)
    L = O.edge_lengths(om, t)
    assert abs(L[0] - 1.0) <= 1e-15 and abs(L[4] - math.sqrt(0.5)) <= 1e-15
    for level in range(4):
        om, t = O.build_topology(hm)
        a = t.arrays()
        assert 3 * hm.nE == 2 * len(a["interior_edges"]) + len(a["boundary_edges"])
        if level < 3:
            for e in range(t.t.E):
                p, q = a["edge_nodes"][e]
                d = hm.coords[q] - hm.coords[p]
                nu = np.array([d[1], -d[0]]) / np.hypot(*d)
                tp = a["edge_elements"][e][0]
                opp = hm.elements[tp][a["local_in_tplus"][e]]
                mid = 0.5 * (hm.coords[p] + hm.coords[q])
                assert nu @ (mid - hm.coords[opp]) > 0
        hm = O.red_refine(hm)


# ---------------------------------------------------------------- refine
def areas(hm):
    return 0.5 * G.signed_area2(hm)


def test_refine_counts_and_areas():  # test_refine.cpp:24-113
    hm = crisscross()
    fine = O.red_refine(hm)
    assert (fine.nE, fine.nC, len(fine.dirichlet), len(fine.neumann)) == (16, 13, 4, 4)
    assert abs(areas(fine).sum() - 1.0) < 1e-12
    for m in range(hm.nE):
        parent = areas(hm)[m]
        assert np.all(np.abs(areas(fine)[4 * m:4 * m + 4] - parent / 4) <= 1e-14 * parent)
    tri = O.red_refine(G.unit_right_triangle())
    assert {frozenset(map(tuple, tri.coords[e])) for e in tri.elements}.__contains__(
        frozenset({(0.5, 0.5), (0.0, 0.5), (0.5, 0.0)}))
    hm = crisscross()
    for level in range(1, 5):
        om, t = O.build_topology(hm)
        nb, eb, db = hm.nC, hm.nE, len(hm.dirichlet)
        hm = O.red_refine(hm, t)
        assert hm.nC == nb + t.t.E and hm.nE == 4 * eb and len(hm.dirichlet) == 2 * db
        assert np.all(areas(hm) > 0)
        on = [(hm.coords[v][1] == 0.0 or hm.coords[v][0] == 1.0) for p in hm.dirichlet for v in p]
        assert all(on)
    assert hm.nE == 4 ** 5


# ---------------------------------------------------------------- assembly
def test_unit_triangle_local_matrices():  # test_assembly.cpp:59-78
    c = capi.coeffs_const(((1, 0), (0, 1)), (1.0, 1.0), 1.0)
    B, D, M, M0 = [x.reshape(3, 3).T for x in O.assemble_volume(G.unit_right_triangle(), c)]
    assert np.abs(B - 0.5 * np.array([[2, -1, -1], [-1, 1, 0], [-1, 0, 1]])).max() < 1e-15
    assert np.abs(D - np.array([[-2, 1, 1]] * 3) / 6.0).max() < 1e-15
    assert np.abs(M - np.array([[2, 1, 1], [1, 2, 1], [1, 1, 2]]) * (0.5 / 12.0)).max() < 1e-15


def test_degenerate_rejected():  # test_assembly.cpp:80-87
    c = capi.coeffs_const()
    for pts in ([[0, 0], [1, 0], [2, 0]], [[0, 0], [0, 1], [1, 0]]):
        hm = capi.HostMesh(np.array(pts, float), np.array([[0, 1, 2]]), np.zeros((0, 2)), np.zeros((0, 2)))
        with pytest.raises(RuntimeError, match="degenerate"):
            O.assemble_volume(hm, c)


def _oracle_integrate(v, fn):  # support.hpp:33-55 (degree-4, 6 points)
    a1, w1, a2, w2 = 0.445948490915965, 0.223381589678011, 0.091576213509771, 0.109951743655322
    rule = [(a1, a1, 1 - 2 * a1, w1), (a1, 1 - 2 * a1, a1, w1), (1 - 2 * a1, a1, a1, w1),
            (a2, a2, 1 - 2 * a2, w2), (a2, 1 - 2 * a2, a2, w2), (1 - 2 * a2, a2, a2, w2)]
    area = 0.5 * ((v[1][0] - v[0][0]) * (v[2][1] - v[0][1]) - (v[1][1] - v[0][1]) * (v[2][0] - v[0][0]))
    return area * sum(q[3] * fn(q[0] * v[0] + q[1] * v[1] + q[2] * v[2], q) for q in rule)


def test_local_matrices_vs_quadrature():  # test_assembly.cpp:89-129 (own RNG, same bar)
    rng = np.random.default_rng(42)
    tested = 0
    while tested < 100:
        v = rng.uniform(-2, 2, (3, 2))
        t2 = (v[1, 0] - v[0, 0]) * (v[2, 1] - v[0, 1]) - (v[1, 1] - v[0, 1]) * (v[2, 0] - v[0, 0])
        if t2 < 0.05:
            continue
        tested += 1
        off = 0.3 * rng.uniform(0.2, 2)
        A = np.array([[rng.uniform(0.2, 2) + 1, off], [off, rng.uniform(0.2, 2) + 1]])
        p = rng.uniform(-2, 2, 2)
        delta = rng.uniform(0.2, 2)
        c = capi.coeffs_const(A, p, delta)
        hm = capi.HostMesh(v, np.array([[0, 1, 2]]), np.zeros((0, 2)), np.zeros((0, 2)))
        B, D, M, _ = [x.reshape(3, 3).T for x in O.assemble_volume(hm, c)]
        grads = [np.array([v[(i + 1) % 3][1] - v[(i + 2) % 3][1], v[(i + 2) % 3][0] - v[(i + 1) % 3][0]]) / t2
                 for i in range(3)]
        for i in range(3):
            for j in range(3):
                assert abs(B[i, j] - _oracle_integrate(v, lambda x, q: (A @ grads[i]) @ grads[j])) < 1e-12
                assert abs(D[i, j] - _oracle_integrate(v, lambda x, q: q[i] * (p @ grads[j]))) < 1e-12
                assert abs(M[i, j] - _oracle_integrate(v, lambda x, q: delta * q[i] * q[j])) < 1e-12


def csr_dense(csr, shape):
    rp, ci, vv = csr
    out = np.zeros(shape)
    for r in range(shape[0]):
        for k in range(rp[r], rp[r + 1]):
            out[r, ci[k]] += vv[k]
    return out


def test_constraint_single_element_and_crisscross():  # test_assembly.cpp:166-231
    tri = G.unit_right_triangle()
    tri = capi.HostMesh(tri.coords, tri.elements, np.array([[0, 1], [1, 2], [2, 0]]), np.zeros((0, 2)))
    om, t = O.build_topology(tri)
    cls = O.classify_edges(om, t)
    Cd = csr_dense(O.assemble_constraint(om, t, cls)["csr"], (3, 3))
    s2 = math.sqrt(2.0) / 2.0
    assert np.allclose(Cd, [[0.5, 0.5, 0.0], [0.5, 0.0, 0.5], [0.0, s2, s2]], rtol=0, atol=1e-15)
    hm = crisscross()
    om, t = O.build_topology(hm)
    cls = O.classify_edges(om, t)
    C = O.assemble_constraint(om, t, cls)
    Cd = csr_dense(C["csr"], (cls.L, 12))
    row = cls.arrays()["retained_pos"][4]
    h = 0.5 * math.sqrt(0.5)
    assert np.allclose(Cd[row, :6], [h, h, 0, -h, 0, -h], rtol=0, atol=1e-16)
    rp = C["csr"][0]
    nnz = np.diff(rp)
    ca = cls.arrays()
    for e in ca["dirichlet_edge_ids"]:
        assert nnz[ca["retained_pos"][e]] == 2
    for e in t.arrays()["interior_edges"]:
        assert nnz[ca["retained_pos"][e]] == 4
        assert abs(Cd[ca["retained_pos"][e]].sum()) < 1e-15
    # CSC is the same matrix
    outer, inner, vals = C["csc"]
    Dc = np.zeros_like(Cd)
    for j in range(12):
        for k in range(outer[j], outer[j + 1]):
            Dc[inner[k], j] = vals[k]
    assert np.array_equal(Dc, Cd)


def test_symmetry_and_mass_rows():  # test_assembly.cpp:233-275
    hm = O.red_refine(crisscross())
    c = capi.coeffs_const(((2.0, 0.4), (0.4, 1.5)), (0.7, -0.3), 0.9)
    B, D, M, M0 = O.assemble_volume(hm, c)
    for X in (B, M):
        blocks = X.reshape(-1, 3, 3)
        assert np.array_equal(blocks, blocks.transpose(0, 2, 1))
    ar = areas(hm)
    assert np.allclose(M.reshape(-1, 3, 3).sum(axis=1), (0.9 * ar / 3.0)[:, None], rtol=1e-13, atol=0)
    _, Dz, _, _ = O.assemble_volume(crisscross(), capi.coeffs_const(p=(0.0, 0.0), delta=1.0))
    assert np.all(Dz == 0.0)


def test_load_vector():  # test_assembly.cpp:277-317
    tri = G.unit_right_triangle()
    b = O.assemble_load(tri, capi.field(capi.FIELD_CONST, 1.0))
    assert np.allclose(b, 0.5 / 3.0, rtol=1e-15, atol=0)
    assert np.all(O.assemble_load(tri, capi.field(capi.FIELD_ZERO)) == 0.0)
    with pytest.raises(RuntimeError, match="element 1"):
        O.assemble_load(tri, capi.field(capi.FIELD_NAN))
    hm = O.red_refine(O.red_refine(crisscross()))
    b = O.assemble_load(hm, capi.field(capi.FIELD_SIN3X))
    f = lambda x: math.sin(3.0 * x[0]) * (1.0 + x[1] * x[1])
    for m in range(hm.nE):
        v = hm.coords[hm.elements[m]]
        area = 0.5 * G.signed_area2(capi.HostMesh(v, np.array([[0, 1, 2]]), np.zeros((0, 2)), np.zeros((0, 2))))[0]
        for j in range(3):
            exp = sum(area / 3.0 * 0.5 * f(0.5 * (v[(i + 1) % 3] + v[(i + 2) % 3])) for i in range(3) if i != j)
            assert abs(b[3 * m + j] - exp) <= 1e-14


def test_neumann_and_dirichlet():  # test_assembly.cpp:319-403
    tri = G.unit_right_triangle()
    tri = capi.HostMesh(tri.coords, tri.elements, np.array([[1, 2], [2, 0]]), np.array([[0, 1]]))
    om, t = O.build_topology(tri)
    cls = O.classify_edges(om, t)
    ln = O.assemble_neumann(om, t, cls, capi.field(capi.FLUX_CONST, 1.0))
    assert np.allclose(ln, [0.5, 0.5, 0.0], rtol=0, atol=1e-15)
    hm = O.red_refine(O.red_refine(crisscross()))
    om, t = O.build_topology(hm)
    cls = O.classify_edges(om, t)
    ln = O.assemble_neumann(om, t, cls, capi.field(capi.FLUX_VEC_KAT))
    a, ca = t.arrays(), cls.arrays()
    exp = np.zeros(3 * hm.nE)
    for e in ca["neumann_edge_ids"]:
        p, q = a["edge_nodes"][e]
        pa, pb = hm.coords[p], hm.coords[q]
        mid, d = 0.5 * (pa + pb), pb - pa
        ln_ = np.hypot(*d)
        g = np.array([math.cos(mid[1]) + mid[0], mid[0] * mid[1] - 1.0]) @ (np.array([d[1], -d[0]]) / ln_)
        el, led = a["edge_elements"][e][0], a["local_in_tplus"][e]
        for c in range(3):
            if c != led:
                exp[3 * el + c] += ln_ * g * 0.5
    assert np.abs(ln - exp).max() <= 1e-14
    hm = crisscross()
    om, t = O.build_topology(hm)
    cls = O.classify_edges(om, t)
    assert np.all(O.assemble_dirichlet(om, t, cls, capi.field(capi.FIELD_ZERO)) == 0)
    bd = O.assemble_dirichlet(om, t, cls, capi.field(capi.FIELD_AFFINE, 0.0, 1.0, 0.0, 0.0))
    assert abs(bd[cls.arrays()["retained_pos"][0]] + 0.5) < 1e-15
    for e in t.arrays()["interior_edges"]:
        assert bd[cls.arrays()["retained_pos"][e]] == 0.0


def test_cn_rhs_matches_dense_restatement():
    """parabolic.cpp:100-103 with M_minus from step_matrix (parabolic.cpp:21-37),
    restated densely with numpy (independent of the oracle's CSC path)."""
    hm = O.red_refine(crisscross())
    om, t = O.build_topology(hm)
    cls = O.classify_edges(om, t)
    c = capi.coeffs_const(((1, 0), (0, 1)), (1.0, 1.0), 1.0)
    f = capi.field(capi.FIELD_AFFINE, 1.0, 0.5, -0.25, 2.0)
    g = capi.field(capi.FLUX_CONST, 0.75)
    uD = capi.field(capi.FIELD_AFFINE, 0.1, 1.0, 0.0, 1.0)
    k, n = 0.25, 2
    N, L = 3 * hm.nE, cls.L
    state = G.uniform_pm1(5, N + L)
    rhs = O.cn_rhs(om, t, cls, c, f, g, uD, k, n, state)
    B, D, M, M0 = O.assemble_volume(hm, c)
    Cd = csr_dense(O.assemble_constraint(om, t, cls)["csr"], (L, N))
    top = np.zeros((N, N))
    for m in range(hm.nE):
        blk = (M0[m] + (-(k / 2.0)) * ((B[m] + D[m]) + M[m])).reshape(3, 3).T
        top[3 * m:3 * m + 3, 3 * m:3 * m + 3] = blk
    Mm = np.block([[top, (k / 2.0) * Cd.T], [0.5 * Cd, np.zeros((L, L))]])
    loads = [O.assemble_load(hm, f, tt) + O.assemble_neumann(om, t, cls, g, tt) for tt in (n * k, (n + 1) * k)]
    bds = [O.assemble_dirichlet(om, t, cls, uD, tt) for tt in (n * k, (n + 1) * k)]
    exp = Mm @ state
    exp[:N] += k * 0.5 * (loads[0] + loads[1])
    exp[N:] += 0.5 * (bds[0] + bds[1])
    assert np.allclose(rhs, exp, rtol=1e-13, atol=1e-15)
