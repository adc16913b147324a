"""Pins the C oracle to the reference itself: the reference's own sources
(/root/reference/proj/src, compiled unmodified against shim/Eigen into
oracle/_ref) and the oracle must agree BIT-FOR-BIT on every hot-path output.
Skipped where the reference sources are absent (the GPU box)."""
import numpy as np
import pytest

from oracle import oracle as O
from oracle import reference as R
from paper_2401_15557_b200 import capi, meshgen as G

pytestmark = pytest.mark.skipif(not R.available(), reason="reference build (oracle/_ref) unavailable")


def meshes():
    out = []
    for lv in range(4):
        out.append((f"crisscross-L{lv}", O.refine_levels(G.crisscross_square(), lv)))
    for lv in (0, 3, 6):
        out.append((f"square-L{lv}", O.refine_levels(G.square_2tri(), lv)))
    for lv in (0, 2, 4):
        out.append((f"lshape-L{lv}", O.refine_levels(G.lshape_6tri(), lv)))
    out.append(("stress-L4", O.orient_ccw(G.stress_transform(O.refine_levels(G.square_2tri(), 4), 4))))
    out.append(("fan-40", G.fan(40, True)))
    out.append(("triangle", G.unit_right_triangle()))
    return out


CASES = meshes()


def oracle_outputs(hm, coeffs, f, g, uD, t=0.0):
    return O.all_outputs(hm, coeffs, f, g, uD, t)


@pytest.mark.parametrize("name,hm", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_oracle_equals_reference(name, hm, cfg):
    args = G.config_fields(cfg)
    o = oracle_outputs(hm, *args, t=0.25)
    r = R.all_outputs(hm, *args, t=0.25)
    for k in r["topo"]:
        assert np.array_equal(o["topo"][k], r["topo"][k]), k
    for k in r["cls"]:
        assert np.array_equal(o["cls"][k], r["cls"][k]), k
    for k in ["B", "D", "M", "M0", "b", "ln", "bd"]:
        assert np.array_equal(o[k], r[k]), k
    for k in ["C_csc", "C_csr"]:
        for a, b in zip(o[k], r[k]):
            assert np.array_equal(a, b), k
    for a, b in zip((o["refined"].coords, o["refined"].elements, o["refined"].dirichlet, o["refined"].neumann),
                    (r["refined"].coords, r["refined"].elements, r["refined"].dirichlet, r["refined"].neumann)):
        assert np.array_equal(a, b)


def test_oracle_lookups_equal_reference():
    hm = O.refine_levels(G.crisscross_square(), 2)
    om, ot = O.build_topology(hm)
    rt = R.RTopology(R.RMesh(hm))
    for k in range(hm.nC):
        for l in range(hm.nC):
            assert ot.node_pair_to_edge(k, l) == rt.node_pair_to_edge(k, l)
            assert ot.directed_pair_to_element(k, l) == rt.directed_pair_to_element(k, l)


def test_error_messages_equal_reference():
    tri = G.unit_right_triangle()
    bad = capi.HostMesh(np.vstack([tri.coords, [[1, 1]]]), np.vstack([tri.elements, [[0, 1, 3]]]),
                        tri.dirichlet, tri.neumann)
    pinched = capi.HostMesh(np.vstack([tri.coords, [[1, 1], [-1, 1]]]),
                            np.vstack([tri.elements, [[1, 0, 3], [0, 1, 4]]]), tri.dirichlet, tri.neumann)
    for m in (bad, pinched):
        with pytest.raises(RuntimeError) as eo:
            O.build_topology(m)
        with pytest.raises(RuntimeError) as er:
            R.RTopology(R.RMesh(m))
        assert str(eo.value) == str(er.value)
    cc = G.crisscross_square()
    for m in (capi.HostMesh(cc.coords, cc.elements, cc.dirichlet, np.vstack([cc.neumann, [[0, 3]]])),
              capi.HostMesh(cc.coords, cc.elements, np.vstack([cc.dirichlet, [[4, 0]]]), cc.neumann)):
        om, ot = O.build_topology(m)
        with pytest.raises(RuntimeError) as eo:
            O.classify_edges(om, ot)
        rm = R.RMesh(m)
        with pytest.raises(RuntimeError) as er:
            R.RClassification(R.RTopology(rm), rm)
        assert str(eo.value) == str(er.value)
    with pytest.raises(RuntimeError) as eo:
        O.assemble_load(O.red_refine(cc), capi.field(capi.FIELD_NAN))
    with pytest.raises(RuntimeError) as er:
        R.assemble_load(R.RMesh(O.red_refine(cc)), 16, capi.field(capi.FIELD_NAN))
    assert str(eo.value) == str(er.value)


@pytest.mark.parametrize("lam", ["random", "zero"])
def test_cn_rhs_equals_reference(lam):
    """The oracle's CN right-hand side vs solve_parabolic's own three lines."""
    hm = O.refine_levels(G.crisscross_square(), 2)
    coeffs = capi.coeffs_const(((2.0, 0.3), (0.3, 1.0)), (1.0, -0.5), 0.7)
    f = capi.field(capi.FIELD_EXP_SINSIN, capi.TWO_PI2_M1)
    g = capi.field(capi.FLUX_GRAD_SINSIN, 1.0)
    uD = capi.field(capi.FIELD_AFFINE, 0.5, 1.0, -2.0, 3.0)
    om, ot = O.build_topology(hm)
    oc = O.classify_edges(om, ot)
    W = G.uniform_pm1(9, 3 * hm.nE + oc.L)
    if lam == "zero":
        W[3 * hm.nE:] = 0.0
    rm = R.RMesh(hm)
    rt = R.RTopology(rm)
    rc = R.RClassification(rt, rm)
    for n in (0, 3, 7):
        assert np.array_equal(O.cn_rhs(om, ot, oc, coeffs, f, g, uD, 0.125, n, W),
                              R.cn_rhs(rm, rt, rc, coeffs, f, g, uD, 0.125, n, W))
