"""The C++ drop-in layer (paper_2401_15557_b200/dropin): the
reference's own C++ entry points (proj/include/phfem) implemented on the B200
C ABI.

* The reference's OWN unit tests (proj/tests/test_{topology,refine,assembly,
  parabolic}.cpp, unmodified, built by oracle/dropin.mk against the drop-in
  instead of proj/src/{edge_topology,refine,assembly}.cpp) must pass on the
  GPU.  Excluded: the test cases that need the global sparse LU solve, which
  BASELINE.json puts outside the product path (the Eigen shim has no LU).
* The same extern "C" runner that drives the reference's sources
  (oracle/ref_runner.cpp) linked against the drop-in must reproduce the C
  oracle bit for bit — including the load vectors: through the drop-in the
  std::function fields are evaluated on the host, like the reference does.
The binaries are built where /root/reference exists and travel with the
snapshot; without them these tests skip.
"""
import os
import subprocess

import numpy as np
import pytest

from oracle import oracle as O
from oracle import reference as R
from paper_2401_15557_b200 import meshgen as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin")

# reference test cases that factorise / solve the saddle or CN system
SOLVER_CASES = ",".join([
    "M_plus factorizes*", "zero data keeps the zero state", "stationary data is a fixed point*",
    "constraint rows hold at every step", "blow-up is reported*", "halving h and k*",
])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["test_topology", "test_refine", "test_assembly", "test_parabolic"])
def test_reference_unit_tests_pass_on_the_dropin(name):
    exe = os.path.join(BIN, name)
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (oracle/dropin.mk needs /root/reference)")
    r = subprocess.run([exe, "-s", f"-tce={SOLVER_CASES}"], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:])
    print(r.stderr[-4000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "Status: SUCCESS" in r.stdout
    assert "| 0 failed" in r.stdout


def dropin_cases():
    out = [("crisscross-L2", O.refine_levels(G.crisscross_square(), 2)),
           ("square-L4", O.refine_levels(G.square_2tri(), 4)),
           ("lshape-L3", O.refine_levels(G.lshape_6tri(), 3)),
           ("stress-L4", O.orient_ccw(G.stress_transform(O.refine_levels(G.square_2tri(), 4), 4))),
           ("fan-40", G.fan(40, True)),
           ("triangle", G.unit_right_triangle())]
    return out


@pytest.fixture
def dropin_runner():
    if not os.path.exists(R.DROPIN_LIB):
        pytest.skip("oracle/_ref/dropin/libphfem_dropin_runner.so not built")
    saved = R.LIB
    R.use_library(R.DROPIN_LIB)
    yield R
    R.use_library(saved)


@pytest.mark.gpu
@pytest.mark.parametrize("name,hm", dropin_cases(), ids=[c[0] for c in dropin_cases()])
@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_dropin_equals_oracle(dropin_runner, name, hm, cfg):
    args = G.config_fields(cfg)
    o = O.all_outputs(hm, *args, t=0.25)
    r = dropin_runner.all_outputs(hm, *args, t=0.25)
    for k in r["topo"]:
        assert np.array_equal(o["topo"][k], r["topo"][k]), k
    for k in r["cls"]:
        assert np.array_equal(o["cls"][k], r["cls"][k]), k
    for k in ["B", "D", "M", "M0", "b", "ln", "bd"]:  # bit-exact, loads included
        assert np.array_equal(o[k], r[k]), k
    for k in ["C_csc", "C_csr"]:
        for a, b in zip(o[k], r[k]):
            assert np.array_equal(a, b), k
    for a, b in zip((o["refined"].coords, o["refined"].elements, o["refined"].dirichlet, o["refined"].neumann),
                    (r["refined"].coords, r["refined"].elements, r["refined"].dirichlet, r["refined"].neumann)):
        assert np.array_equal(a, b)


@pytest.mark.gpu
def test_dropin_lookups_and_errors(dropin_runner):
    hm = O.refine_levels(G.crisscross_square(), 2)
    om, ot = O.build_topology(hm)
    rt = dropin_runner.RTopology(dropin_runner.RMesh(hm))
    for k in range(hm.nC):
        for l in range(hm.nC):
            assert ot.node_pair_to_edge(k, l) == rt.node_pair_to_edge(k, l)
            assert ot.directed_pair_to_element(k, l) == rt.directed_pair_to_element(k, l)


@pytest.mark.gpu
def test_dropin_cn_rhs(dropin_runner):
    """solve_parabolic's RHS lines (reference parabolic.cpp, unchanged) over the
    drop-in's operators and loads == the oracle, bit for bit."""
    from paper_2401_15557_b200 import capi
    hm = O.refine_levels(G.crisscross_square(), 2)
    coeffs = capi.coeffs_const(((2.0, 0.3), (0.3, 1.0)), (1.0, -0.5), 0.7)
    f = capi.field(capi.FIELD_EXP_SINSIN, capi.TWO_PI2_M1)
    g = capi.field(capi.FLUX_GRAD_SINSIN, 1.0)
    uD = capi.field(capi.FIELD_AFFINE, 0.5, 1.0, -2.0, 3.0)
    om, ot = O.build_topology(hm)
    oc = O.classify_edges(om, ot)
    W = G.uniform_pm1(9, 3 * hm.nE + oc.L)
    rm = dropin_runner.RMesh(hm)
    rt = dropin_runner.RTopology(rm)
    rc = dropin_runner.RClassification(rt, rm)
    for n in (0, 3, 7):
        assert np.array_equal(O.cn_rhs(om, ot, oc, coeffs, f, g, uD, 0.125, n, W),
                              dropin_runner.cn_rhs(rm, rt, rc, coeffs, f, g, uD, 0.125, n, W))
