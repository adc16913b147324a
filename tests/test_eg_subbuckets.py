"""The edge pass's multi-sub-bucket tiles (bs < 8) on small meshes.

The sort-based edge generation (csrc/edge_gen.cu, reference
proj/src/edge_topology.cpp:52-143) buckets the directed occurrences by
max node >> bs; bs = min(8, 64 - packed key bits).  Meshes whose packed item
needs more than 56 bits — the L13 square (27 + 29 + 1 = 57 bits, bs = 7) —
make every 256-node tile span several buckets, which changes the tile's node
decode and the rank sort's compares at sub-bucket boundaries.  The ctx knob
phfem_ctx_set_eg_max_bs forces that path on meshes the oracle checks in
milliseconds; outputs must not depend on it."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2401_15557_b200 import capi, meshgen as G

from test_gpu_parity import check_cls, check_topology, compare_all, gpu_all, oracle_all

pytestmark = pytest.mark.gpu

BS = [1, 3, 4, 5, 6, 7]


@pytest.fixture(scope="module")
def ctx_bs():
    c = capi.Context(0)
    yield c
    c.close()


def permuted(base, seed):
    perm = np.argsort(G.splitmix64(seed, base.nC), kind="stable")
    inv = np.empty_like(perm)
    inv[perm] = np.arange(base.nC)
    return capi.HostMesh(base.coords[perm], inv[base.elements][np.argsort(G.splitmix64(seed + 1, base.nE))],
                         inv[base.dirichlet], inv[base.neumann])


def meshes():
    return {
        "square_L6": O.refine_levels(G.square_2tri(), 6),
        "lshape_L5": O.refine_levels(G.lshape_6tri(), 5),
        "stress_L6": O.orient_ccw(G.stress_transform(O.refine_levels(G.square_2tri(), 6), 6)),
        "permuted_L4": permuted(O.refine_levels(G.lshape_6tri(), 4), 31),
        "crisscross_L5": O.refine_levels(G.crisscross_square(), 5),
    }


@pytest.mark.parametrize("bs", BS)
def test_build_topology_any_bucket_width(ctx_bs, bs):
    ctx_bs.set_eg_max_bs(bs)
    try:
        for name, hm in meshes().items():
            dm = capi.DeviceMesh.upload(ctx_bs, hm)
            t = capi.build_topology(ctx_bs, dm).download()
            _, ot = O.build_topology(hm)
            check_topology(t, ot.arrays())
    finally:
        ctx_bs.set_eg_max_bs(8)


@pytest.mark.parametrize("bs", [3, 5, 7])
@pytest.mark.parametrize("k,last", [(40, True), (700, True), (3000, False)])
def test_fans_any_bucket_width(ctx_bs, bs, k, last):
    """High-valence nodes (> 32 occurrences, oversized tiles) with several
    sub-buckets per tile: the general tile path's node decode."""
    ctx_bs.set_eg_max_bs(bs)
    try:
        hm = G.fan(k, last)
        args = G.config_fields(2)
        compare_all(gpu_all(ctx_bs, hm, *args), oracle_all(hm, *args))
    finally:
        ctx_bs.set_eg_max_bs(8)


@pytest.mark.parametrize("bs", [4, 7])
def test_fused_final_level_any_bucket_width(ctx_bs, bs):
    """The given-mesh pipeline (sort-built final level with classification and
    C fused into the emit pass) — the given-L13 bench line's code path."""
    ctx_bs.set_eg_max_bs(bs)
    try:
        for hm in (O.refine_levels(G.square_2tri(), 6), O.refine_levels(G.lshape_6tri(), 5)):
            args = G.config_fields(2)
            r = capi.pipeline(ctx_bs, capi.DeviceMesh.upload(ctx_bs, hm), 0, *args).download()
            o = O.pipeline(hm, 0, *args)
            check_topology(r["topo"], o["topo"])
            check_cls(r["cls"], o["cls"])
            for a, b in zip((r["C_row_ptr"], r["C_col_idx"], r["C_values"]), o["C_csr"]):
                assert np.array_equal(a, b)
            for k in ["B", "D", "M", "M0"]:
                assert np.array_equal(r[k], o[k]), k
    finally:
        ctx_bs.set_eg_max_bs(8)


def test_bucket_width_rejects_out_of_range(ctx_bs):
    for bad in (0, 9, -1):
        with pytest.raises(ValueError):
            ctx_bs.set_eg_max_bs(bad)
