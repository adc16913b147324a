"""Multi-GPU path (paper_2401_15557_b200/dist.py).

* gpu: W ranks emulated in one process on one B200 (LocalComm: the real
  kernels of every rank run one after another, never waiting on each other)
  must reproduce the single-GPU pipeline BIT FOR BIT after concatenating the
  rank slices — topology, element->edge map, classification, C in CSR, bD,
  blocks and load — for W = 1..4 and refinement in the loop.
* not gpu: the same orchestration with 2 gloo processes on CPU and the numpy
  restatement of the per-rank operations (tests/dist_cpu_backend.py) against
  the C oracle — the exchange logic (key ranges, all-to-alls, id re-basing,
  boundary-pair resolution, Neumann table) under a real process group.
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2401_15557_b200 import meshgen as G

CASES = [("crisscross-L1", lambda: O.refine_levels(G.crisscross_square(), 1), 1),
         ("square-L3", lambda: O.refine_levels(G.square_2tri(), 3), 1),
         ("lshape-L2", lambda: O.refine_levels(G.lshape_6tri(), 2), 1),
         ("lshape-L3-nolevel", lambda: O.refine_levels(G.lshape_6tri(), 3), 0),
         ("stress-L3", lambda: O.orient_ccw(G.stress_transform(O.refine_levels(G.square_2tri(), 3), 3)), 1),
         ("fan-30", lambda: G.fan(30, True), 1),
         ("crisscross-L1-2levels", lambda: O.refine_levels(G.crisscross_square(), 1), 2),
         ("lshape-L1-3levels", lambda: O.refine_levels(G.lshape_6tri(), 1), 3),
         # > 256 W nodes: the tile-aligned key ranges of the peer-window input
         # level give every rank edges of its own (smaller meshes: one owner)
         ("square-L6", lambda: O.refine_levels(G.square_2tri(), 6), 1),
         ("stress-L6", lambda: O.orient_ccw(G.stress_transform(O.refine_levels(G.square_2tri(), 6), 6)), 1)]


def check_equal(d, ref):
    r = ref
    for k in ("edge_nodes", "edge_elements", "local_in_tplus", "local_in_tminus", "interior_edges",
              "boundary_edges", "node_edge_start", "elem_edge"):
        assert np.array_equal(d[k].reshape(-1), r["topo"][k].reshape(-1)), k
    for k in ("retained_pos", "retained_edges"):
        assert np.array_equal(d[k], r["cls"][k]), k
    for k in ("C_row_ptr", "C_col_idx", "C_values", "bd"):
        assert np.array_equal(d[k], r[k]), k
    for k in ("B", "D", "M", "M0", "load"):
        assert np.array_equal(d[k], r[k].reshape(-1)), k
    assert np.array_equal(d["coords"], r["mesh"].coords)
    assert np.array_equal(d["elements"], r["mesh"].elements)
    assert np.array_equal(d["dirichlet"], r["mesh"].dirichlet)
    assert np.array_equal(d["neumann"], r["mesh"].neumann)


@pytest.mark.gpu
@pytest.mark.parametrize("W", [1, 2, 3, 4])
@pytest.mark.parametrize("name,make,levels", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("sort_free", ["p2p", "a2a", False], ids=["sortfree", "sortfree-a2a", "sorted"])
def test_emulated_ranks_equal_single_gpu(ctx, monkeypatch, W, name, make, levels, sort_free):
    """sortfree: the halo exchanges through peer windows (the CUDA default);
    sortfree-a2a: the same through all-to-alls; sorted: a sort per level."""
    import torch
    from paper_2401_15557_b200 import capi, dist
    if not sort_free and (levels > 1 or W == 3):
        pytest.skip("sorted-level path: covered by the other cases")
    if sort_free == "a2a" and W in (1, 3):
        pytest.skip("all-to-all halo form: W = 2, 4")
    monkeypatch.setattr(dist, "P2P", sort_free != "a2a")
    sort_free = bool(sort_free)
    hm = make()
    args = G.config_fields(2)
    ref = capi.pipeline(ctx, capi.DeviceMesh.upload(ctx, hm), levels, *args, flags=capi.PIPE_GENERIC_EG).download()
    tctx = capi.Context(0, stream=torch.cuda.current_stream().cuda_stream)
    comm = dist.LocalComm(W)
    states = dist.make_states(hm, comm, lambda r: dist.CudaRankOps(tctx, "cuda:0"))
    states, nC, nE = dist.distributed_pipeline(states, comm, hm.nC, hm.nE, levels, *args, sort_free=sort_free)
    check_equal(dist.collect(states), ref)


@pytest.mark.gpu
def test_emulated_ranks_boundary_errors(ctx):
    import torch
    from paper_2401_15557_b200 import capi, dist
    cc = G.crisscross_square()
    bad = capi.HostMesh(cc.coords, cc.elements, np.vstack([cc.dirichlet, [[4, 0]]]), cc.neumann)
    tctx = capi.Context(0, stream=torch.cuda.current_stream().cuda_stream)
    comm = dist.LocalComm(2)
    states = dist.make_states(bad, comm, lambda r: dist.CudaRankOps(tctx, "cuda:0"))
    with pytest.raises(RuntimeError, match="resolves to an interior edge"):
        dist.distributed_pipeline(states, comm, bad.nC, bad.nE, 0, *G.config_fields(2))


def _gloo_worker(rank, world, port, tmp, case, levels):
    import torch.distributed as tdist
    from paper_2401_15557_b200 import dist
    from dist_cpu_backend import NumpyRankOps
    tdist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        hm = dict((c[0], c[1]) for c in CASES)[case]()
        comm = dist.TorchComm()
        states = dist.make_states(hm, comm, lambda r: NumpyRankOps())
        states, nC, nE = dist.distributed_pipeline(states, comm, hm.nC, hm.nE, levels, *G.config_fields(1))
        np.savez(os.path.join(tmp, f"rank{rank}.npz"), **dist.rank_slice(states[0]))
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("case,levels", [("square-L3", 1), ("lshape-L2", 1), ("stress-L3", 0),
                                         ("crisscross-L1-2levels", 2), ("lshape-L1-3levels", 3)])
def test_gloo_two_ranks_equal_oracle(tmp_path, case, levels):
    """2 gloo processes on CPU: the concatenated rank slices == the C oracle
    run on the whole mesh (topology, maps, classification, C, bD, blocks,
    load = b + LN)."""
    import socket
    import torch.multiprocessing as mp
    from paper_2401_15557_b200 import dist
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.start_processes(_gloo_worker, args=(2, port, str(tmp_path), case, levels), nprocs=2, join=True,
                       start_method="fork")
    got = dist.concat_slices([dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(2)])
    hm = dict((c[0], c[1]) for c in CASES)[case]()
    fine = O.refine_levels(hm, levels)
    args = G.config_fields(1)
    om, ot = O.build_topology(fine)
    oc = O.classify_edges(om, ot)
    topo, cls = ot.arrays(), oc.arrays()
    for k in ("edge_nodes", "edge_elements", "local_in_tplus", "local_in_tminus", "interior_edges",
              "boundary_edges"):
        assert np.array_equal(got[k].reshape(-1), topo[k].reshape(-1)), k
    for k in ("retained_pos", "retained_edges"):
        assert np.array_equal(got[k], cls[k]), k
    Cm = O.assemble_constraint(om, ot, oc)
    for a, b in zip((got["C_row_ptr"], got["C_col_idx"], got["C_values"]), Cm["csr"]):
        assert np.array_equal(a, b)
    assert np.array_equal(got["bd"], O.assemble_dirichlet(om, ot, oc, args[3], 0.0))
    B, D, M, M0 = O.assemble_volume(fine, args[0])
    for k, v in zip(("B", "D", "M", "M0"), (B, D, M, M0)):
        assert np.array_equal(got[k], v.reshape(-1)), k
    load = O.assemble_load(fine, args[1], 0.0) + O.assemble_neumann(om, ot, oc, args[2], 0.0)
    assert np.array_equal(got["load"], load)
    assert np.array_equal(got["coords"], fine.coords)
    assert np.array_equal(got["elements"], fine.elements)


@pytest.mark.parametrize("W", [2, 3])
def test_sampled_key_histogram_local_ranks(monkeypatch, W):
    """The key ranges come from a SAMPLED coarse histogram on large meshes
    (dist.HIST_SAMPLE); forced on a small mesh here: W emulated NumPy ranks
    (one process, LocalComm) still reproduce the C oracle bit for bit — the
    ranges only balance work."""
    from paper_2401_15557_b200 import dist
    from dist_cpu_backend import NumpyRankOps
    monkeypatch.setattr(dist, "HIST_SAMPLE", 3)
    monkeypatch.setattr(dist, "HIST_SAMPLE_MIN_ELEMENTS", 0)
    hm = O.refine_levels(G.lshape_6tri(), 2)
    comm = dist.LocalComm(W)
    states = dist.make_states(hm, comm, lambda r: NumpyRankOps())
    states, nC, nE = dist.distributed_pipeline(states, comm, hm.nC, hm.nE, 1, *G.config_fields(1))
    got = dist.collect(states)
    fine = O.refine_levels(hm, 1)
    om, ot = O.build_topology(fine)
    topo = ot.arrays()
    for k in ("edge_nodes", "edge_elements", "local_in_tplus", "local_in_tminus", "elem_edge"):
        assert np.array_equal(np.asarray(got[k]).reshape(-1), topo[k].reshape(-1)), k


@pytest.mark.parametrize("W,case,levels", [(3, "lshape-L1-3levels", 3), (5, "square-L3", 1),
                                           (4, "stress-L3", 1)])
def test_halo_refine_local_ranks_equal_oracle(W, case, levels):
    """The halo form of the sort-free refinement (side records -> edge owners,
    group starts -> element owners, coordinates only where referenced after
    the last level) with W emulated NumPy ranks: every output == the C oracle
    on the whole mesh, coordinates included (parent nodes + the ranks' owned
    midpoints)."""
    from paper_2401_15557_b200 import dist
    from dist_cpu_backend import NumpyRankOps
    hm = dict((c[0], c[1]) for c in CASES)[case]()
    comm = dist.LocalComm(W)
    states = dist.make_states(hm, comm, lambda r: NumpyRankOps())
    args = G.config_fields(1)
    states, nC, nE = dist.distributed_pipeline(states, comm, hm.nC, hm.nE, levels, *args)
    got = dist.collect(states)
    fine = O.refine_levels(hm, levels)
    om, ot = O.build_topology(fine)
    oc = O.classify_edges(om, ot)
    topo = ot.arrays()
    for k in ("edge_nodes", "edge_elements", "local_in_tplus", "local_in_tminus", "elem_edge",
              "interior_edges", "boundary_edges"):
        assert np.array_equal(np.asarray(got[k]).reshape(-1), topo[k].reshape(-1)), k
    for a, b in zip((got["C_row_ptr"], got["C_col_idx"], got["C_values"]), O.assemble_constraint(om, ot, oc)["csr"]):
        assert np.array_equal(a, b)
    load = O.assemble_load(fine, args[1], 0.0) + O.assemble_neumann(om, ot, oc, args[2], 0.0)
    assert np.array_equal(got["load"], load)
    assert np.array_equal(got["coords"], fine.coords)
    assert np.array_equal(got["elements"], fine.elements)


def _ipc_worker(rank, world, port, tmp, case, levels):
    """One of 2 processes on the SAME GPU: collectives over gloo (CPU staging,
    test-only), peer windows through CUDA IPC (torch storage sharing) — the
    plumbing of the multi-GPU peer-window path, on the one GPU available."""
    import torch
    import torch.distributed as tdist
    from paper_2401_15557_b200 import capi, dist

    class StagedComm(dist.TorchComm):
        def all_reduce(self, ts, op):
            c = ts[0].cpu()
            super().all_reduce([c], op)
            ts[0].copy_(c)

        def all_gather(self, ts):
            out = super().all_gather([ts[0].cpu()])
            return [[x.to(ts[0].device) for x in out[0]]]

        def all_to_all_v(self, sends, counts):
            return [super().all_to_all_v([sends[0].cpu()], counts)[0].to(sends[0].device)]

    torch.cuda.set_device(0)
    tdist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        hm = dict((c[0], c[1]) for c in CASES)[case]()
        comm = StagedComm()
        tctx = capi.Context(0, stream=torch.cuda.current_stream().cuda_stream)
        states = dist.make_states(hm, comm, lambda r: dist.CudaRankOps(tctx, "cuda:0"))
        states, nC, nE = dist.distributed_pipeline(states, comm, hm.nC, hm.nE, levels, *G.config_fields(2))
        np.savez(os.path.join(tmp, f"rank{rank}.npz"), **dist.rank_slice(states[0]))
        tdist.barrier()
    finally:
        tdist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("case,levels", [("square-L3", 1), ("lshape-L1-3levels", 3)])
def test_peer_windows_two_processes_one_gpu(ctx, tmp_path, case, levels):
    """2 processes share the B200: the side / group-start records go through
    CUDA-IPC peer windows (no kernel waits on another rank: the fences are
    host barriers); the concatenated slices == the single-GPU pipeline."""
    import socket
    import torch.multiprocessing as mp
    from paper_2401_15557_b200 import capi, dist
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.start_processes(_ipc_worker, args=(2, port, str(tmp_path), case, levels), nprocs=2, join=True,
                       start_method="spawn")
    got = dist.concat_slices([dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(2)])
    hm = dict((c[0], c[1]) for c in CASES)[case]()
    dm = capi.DeviceMesh.upload(ctx, hm)
    ref = capi.pipeline(ctx, dm, levels, *G.config_fields(2), flags=capi.PIPE_GENERIC_EG).download()
    check_equal(got, ref)


@pytest.mark.gpu
@pytest.mark.parametrize("W", [1, 3])
def test_volume_on_side_stream_equal_single_gpu(ctx, W):
    """The last level's blocks + load on a side stream (overlapping the
    host-synchronised classification / resolve / Neumann phases, the NCCL
    default) give the same bits; Neumann data joins the side stream first."""
    import torch
    from paper_2401_15557_b200 import capi, dist
    hm = O.refine_levels(G.square_2tri(), 6)
    args = G.config_fields(1)   # g != 0: the Neumann update must wait for the side-stream load
    ref = capi.pipeline(ctx, capi.DeviceMesh.upload(ctx, hm), 1, *args, flags=capi.PIPE_GENERIC_EG).download()
    tctx = capi.Context(0, stream=torch.cuda.current_stream().cuda_stream)
    comm = dist.LocalComm(W)
    comm.overlap_volume = True
    states = dist.make_states(hm, comm, lambda r: dist.CudaRankOps(tctx, "cuda:0"))
    states, nC, nE = dist.distributed_pipeline(states, comm, hm.nC, hm.nE, 1, *args)
    torch.cuda.synchronize()
    check_equal(dist.collect(states), ref)


@pytest.mark.gpu
@pytest.mark.parametrize("W", [3, 8])
def test_emulated_ranks_at_scale(ctx, W):
    """The sharded L10 -> L11 step (8.4 M triangles; the peer-window input
    level, halo-form refinement with global ids written directly) over W
    emulated ranks == the single-GPU pipeline, every output bit for bit."""
    import torch
    from paper_2401_15557_b200 import capi, dist
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
    tctx = capi.Context(0, stream=torch.cuda.current_stream().cuda_stream)
    comm = dist.LocalComm(W)
    states = dist.make_states(hm, comm, lambda r: dist.CudaRankOps(tctx, "cuda:0"))
    states, nC, nE = dist.distributed_pipeline(states, comm, hm.nC, hm.nE, 1, *args)
    got = dist.collect(states)
    for s in states:
        s.ops.release()
    check_equal(got, ref)
