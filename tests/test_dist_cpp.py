"""The sharded step with its orchestration in C++ (csrc/dist_run.cu,
phfem_dist_pipeline) — the same phases as dist.py's peer-window / halo form,
no Python between the kernels.

gpu: W ranks emulated in one process (phfem_dist_comm_local) reproduce the
single-GPU pipeline BIT FOR BIT after concatenating the rank slices, for
W = 1..5, refinement in the loop, the sampled key histogram, the reference's
boundary-pair errors, the L10 -> L11 step at W = 8, and one NCCL rank
(phfem_dist_comm_nccl, world 1: NCCL initialised through the library).
not gpu: the library exports the entry points (tests/test_abi.py checks every
symbol of capi.EXPORTED) and the communicator objects are plain host state.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2401_15557_b200 import meshgen as G

from test_dist import CASES, check_equal


def _rank_meshes(capi, dm, W):
    """rank r's phfem_mesh: the replicated arrays of `dm`, its element range"""
    m = dm.m
    out = []
    for r in range(W):
        lo, hi = m.nE * r // W, m.nE * (r + 1) // W
        v = capi.phfem_mesh()
        v.coords, v.dirichlet, v.neumann = m.coords, m.dirichlet, m.neumann
        v.elements = (m.elements or 0) + 12 * lo
        v.nC, v.nE, v.nD, v.nN, v.owned = m.nC, hi - lo, m.nD, m.nN, 0
        out.append(v)
    return out


def run_cpp(ctx, hm, W, levels, args, hist_sample=1, flags=0):
    from paper_2401_15557_b200 import capi, dist
    dm = capi.DeviceMesh.upload(ctx, hm)
    comm = capi.DistComm.local_ranks(W)
    try:
        outs = capi.dist_pipeline(comm, [ctx] * W, _rank_meshes(capi, dm, W), hm.nC, hm.nE, levels, *args,
                                  hist_sample=hist_sample, flags=flags)
        got = dist.concat_slices([o.rank_slice() for o in outs])
        for o in outs:
            o.release()
    finally:
        comm.close()
        dm.release()
    return got


@pytest.mark.gpu
@pytest.mark.parametrize("W", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("name,make,levels", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("mode", ["local", "windows"])
def test_cpp_emulated_ranks_equal_single_gpu(ctx, W, name, make, levels, mode):
    """local: slots whose element and edge share a rank are gathered from its
    own arrays (the default); windows: every slot's record through the peer
    windows (PHFEM_DIST_NO_LOCAL)"""
    from paper_2401_15557_b200 import capi
    hm = make()
    args = G.config_fields(2)
    ref = capi.pipeline(ctx, capi.DeviceMesh.upload(ctx, hm), levels, *args, flags=capi.PIPE_GENERIC_EG).download()
    check_equal(run_cpp(ctx, hm, W, levels, args, flags=0 if mode == "local" else capi.DIST_NO_LOCAL), ref)


@pytest.mark.gpu
@pytest.mark.parametrize("W", [2, 3])
def test_cpp_sampled_histogram_and_neumann_load(ctx, W):
    """every 3rd element in the key-range histogram; g != 0 (Neumann load
    through the all-reduced table)"""
    from paper_2401_15557_b200 import capi
    hm = O.refine_levels(G.lshape_6tri(), 3)
    args = G.config_fields(1)
    ref = capi.pipeline(ctx, capi.DeviceMesh.upload(ctx, hm), 2, *args, flags=capi.PIPE_GENERIC_EG).download()
    check_equal(run_cpp(ctx, hm, W, 2, args, hist_sample=3), ref)


@pytest.mark.gpu
@pytest.mark.parametrize("levels", [0, 1])
def test_cpp_boundary_errors(ctx, levels):
    """the reference's first boundary-pair error, raised from the rank
    holding it, the library left usable"""
    from paper_2401_15557_b200 import capi
    cc = G.crisscross_square()
    bad = capi.HostMesh(cc.coords, cc.elements, np.vstack([cc.dirichlet, [[4, 0]]]), cc.neumann)
    with pytest.raises(capi.PhfemError, match="resolves to an interior edge"):
        run_cpp(ctx, bad, 2, levels, G.config_fields(2))
    nonedge = capi.HostMesh(cc.coords, cc.elements, cc.dirichlet, np.vstack([cc.neumann, [[0, 3]]]))
    with pytest.raises(capi.PhfemError, match=r"neumann pair \(1,4\) is not an edge"):
        run_cpp(ctx, nonedge, 3, levels, G.config_fields(2))
    hm = O.refine_levels(G.square_2tri(), 2)
    ref = capi.pipeline(ctx, capi.DeviceMesh.upload(ctx, hm), 1, *G.config_fields(2)).download()
    check_equal(run_cpp(ctx, hm, 2, 1, G.config_fields(2)), ref)


@pytest.mark.gpu
def test_cpp_repeated_calls_reuse_windows(ctx):
    """the communicator's peer windows persist across calls (grown on
    demand): a smaller and a larger mesh after each other"""
    from paper_2401_15557_b200 import capi, dist
    args = G.config_fields(2)
    comm = capi.DistComm.local_ranks(3)
    try:
        for hm in (O.refine_levels(G.square_2tri(), 5), O.refine_levels(G.square_2tri(), 3),
                   O.refine_levels(G.lshape_6tri(), 5)):
            dm = capi.DeviceMesh.upload(ctx, hm)
            outs = capi.dist_pipeline(comm, [ctx] * 3, _rank_meshes(capi, dm, 3), hm.nC, hm.nE, 1, *args)
            got = dist.concat_slices([o.rank_slice() for o in outs])
            for o in outs:
                o.release()
            ref = capi.pipeline(ctx, dm, 1, *args).download()
            check_equal(got, ref)
    finally:
        comm.close()


@pytest.mark.gpu
def test_cpp_nccl_single_rank(ctx):
    """phfem_dist_comm_nccl with world 1 (NCCL resolved from the process's
    libnccl.so.2 and initialised by the library) == the single-GPU pipeline"""
    import torch  # noqa: F401  (its libnccl.so.2 is the one the library resolves)
    from paper_2401_15557_b200 import capi, dist
    hm = O.refine_levels(G.lshape_6tri(), 4)
    args = G.config_fields(2)
    ref = capi.pipeline(ctx, capi.DeviceMesh.upload(ctx, hm), 1, *args).download()
    uid = capi.DistComm.nccl_unique_id()
    comm = capi.DistComm.nccl(uid, 0, 1, 0)
    dm = capi.DeviceMesh.upload(ctx, hm)
    try:
        outs = capi.dist_pipeline(comm, [ctx], _rank_meshes(capi, dm, 1), hm.nC, hm.nE, 1, *args)
        got = dist.concat_slices([o.rank_slice() for o in outs])
        outs[0].release()
    finally:
        comm.close()
        dm.release()
    check_equal(got, ref)


@pytest.mark.gpu
@pytest.mark.parametrize("W", [8])
@pytest.mark.parametrize("mode", ["local", "windows"])
def test_cpp_emulated_ranks_at_scale(ctx, W, mode):
    """the L10 -> L11 sharded step (8.4 M triangles, sampled key histogram) over
    W emulated ranks == the single-GPU pipeline, every output bit for bit"""
    from paper_2401_15557_b200 import capi
    base = capi.DeviceMesh.upload(ctx, G.square_2tri())
    for _ in range(10):
        t = capi.build_topology(ctx, base)
        nxt = capi.red_refine(ctx, base, t)
        t.release()
        base.release()
        base = nxt
    hm = base.download()
    base.release()
    args = G.config_fields(5)
    res = capi.pipeline(ctx, capi.DeviceMesh.upload(ctx, hm), 1, *args)
    ref = res.download()
    res.release()
    check_equal(run_cpp(ctx, hm, W, 1, args, hist_sample=8, flags=0 if mode == "local" else capi.DIST_NO_LOCAL), ref)


def test_cpp_local_comm_host_state():
    from paper_2401_15557_b200 import capi
    c = capi.DistComm.local_ranks(4)
    assert c.world == 4 and c.local
    c.close()
    with pytest.raises(ValueError):
        capi.DistComm.local_ranks(0)


@pytest.mark.gpu
@pytest.mark.parametrize("W,levels", [(1, 0), (1, 1), (2, 1)])
def test_cpp_degenerate_element_error(ctx, W, levels):
    """the element pass's error (deferred past the classification / bD /
    Neumann-table enqueue) is the reference's: two nodes of an element at one
    point"""
    from paper_2401_15557_b200 import capi
    hm = O.refine_levels(G.square_2tri(), 2)
    a, b = int(hm.elements[3][0]), int(hm.elements[3][1])
    coords = hm.coords.copy()
    coords[b] = coords[a]
    bad = capi.HostMesh(coords, hm.elements, hm.dirichlet, hm.neumann)
    with pytest.raises(capi.PhfemError, match="degenerate"):
        run_cpp(ctx, bad, W, levels, G.config_fields(2))
    ref = capi.pipeline(ctx, capi.DeviceMesh.upload(ctx, hm), levels, *G.config_fields(2)).download()
    check_equal(run_cpp(ctx, hm, W, levels, G.config_fields(2)), ref)
