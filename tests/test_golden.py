"""Golden vectors from the reference itself (tests/golden, made by
tools/make_golden.py from oracle/_ref).  The C oracle (CPU) and the CUDA path
(GPU, through the C ABI) must reproduce them: integers and +-*/sqrt values
bit-exactly, libm-dependent values (load, Neumann, CN RHS) within 1e-12
relative on the GPU (CUDA sin/exp vs glibc) and bit-exactly on the CPU."""
import glob
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2401_15557_b200 import capi, meshgen as G

HERE = os.path.dirname(os.path.abspath(__file__))
FILES = sorted(glob.glob(os.path.join(HERE, "golden", "*.npz")))
IDS = [os.path.basename(f)[:-4] for f in FILES]
TOPO = ["edge_nodes", "edge_elements", "local_in_tplus", "local_in_tminus", "interior_edges", "boundary_edges"]
CLS = ["dirichlet_edge_ids", "neumann_edge_ids", "retained_edges", "retained_pos"]


def load(path):
    z = dict(np.load(path))
    hm = capi.HostMesh(z["in_coords"], z["in_elements"], z["in_dirichlet"], z["in_neumann"])
    return z, hm, G.config_fields(int(z["cfg"]))


def rel_ok(a, b, tol):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and bool(np.all((a == b) | (np.abs(a - b) <= tol * np.abs(b))))


@pytest.mark.parametrize("path", FILES, ids=IDS)
def test_oracle_reproduces_golden(path):
    z, hm, (coeffs, f, g, uD) = load(path)
    om, ot = O.build_topology(hm)
    oc = O.classify_edges(om, ot)
    t, c = ot.arrays(), oc.arrays()
    for k in TOPO:
        assert np.array_equal(t[k], z["topo_" + k]), k
    for k in CLS:
        assert np.array_equal(c[k], z["cls_" + k]), k
    for k, v in zip(["B", "D", "M", "M0"], O.assemble_volume(hm, coeffs)):
        assert np.array_equal(v, z[k]), k
    C = O.assemble_constraint(om, ot, oc)
    for k, v in zip(["outer", "inner", "values"], C["csc"]):
        assert np.array_equal(v, z["csc_" + k])
    for k, v in zip(["row_ptr", "col_idx", "values"], C["csr"]):
        assert np.array_equal(v, z["csr_" + k])
    assert np.array_equal(O.assemble_load(hm, f), z["b"])
    assert np.array_equal(O.assemble_neumann(om, ot, oc, g), z["ln"])
    assert np.array_equal(O.assemble_dirichlet(om, ot, oc, uD), z["bd"])
    fm = O.red_refine(hm, ot)
    for k in ["coords", "elements", "dirichlet", "neumann"]:
        assert np.array_equal(getattr(fm, k), z["ref_" + k]), k
    if "cn_state" in z:
        for n in (0, 5):
            assert np.array_equal(O.cn_rhs(om, ot, oc, coeffs, f, g, uD, 1e-3, n, z["cn_state"]), z[f"cn_rhs_{n}"])


@pytest.mark.gpu
@pytest.mark.parametrize("path", FILES, ids=IDS)
def test_cuda_reproduces_golden(ctx, path):
    z, hm, (coeffs, f, g, uD) = load(path)
    dm = capi.DeviceMesh.upload(ctx, hm)
    topo = capi.build_topology(ctx, dm)
    cls = capi.classify_edges(ctx, topo, dm)
    t, c = topo.download(), cls.download()
    for k in TOPO:
        assert np.array_equal(t[k], z["topo_" + k]), k
    for k in CLS:
        assert np.array_equal(c[k], z["cls_" + k]), k
    for k, v in zip(["B", "D", "M", "M0"], capi.assemble_volume(ctx, dm, coeffs)):
        assert np.array_equal(v, z[k]), k
    for k, v in zip(["row_ptr", "col_idx", "values"], capi.assemble_constraint(ctx, dm, topo, cls)):
        assert np.array_equal(v, z["csr_" + k])
    for k, v in zip(["outer", "inner", "values"], capi.constraint_csc(ctx, dm, topo, cls)):
        assert np.array_equal(v, z["csc_" + k])
    assert rel_ok(capi.assemble_load(ctx, dm, f), z["b"], 1e-12)
    assert rel_ok(capi.assemble_neumann(ctx, dm, topo, cls, g), z["ln"], 1e-12)
    assert rel_ok(capi.assemble_dirichlet(ctx, dm, topo, cls, uD), z["bd"], 1e-12)
    fm = capi.red_refine(ctx, dm, topo).download()
    for k in ["coords", "elements", "dirichlet", "neumann"]:
        assert np.array_equal(getattr(fm, k), z["ref_" + k]), k
    if "cn_state" in z:
        plan = capi.CNPlan(ctx, dm, topo, cls, coeffs, f, g, uD, 1e-3)
        for n in (0, 5):
            assert rel_ok(plan.rhs(n, z["cn_state"]), z[f"cn_rhs_{n}"], 1e-12)
