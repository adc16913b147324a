import sys, numpy as np, torch
sys.path.insert(0, '.')
from oracle import oracle as O
from paper_2401_15557_b200 import capi, dist, meshgen as G
ctx = capi.Context(0)
for lv0, levels in ((0, 0), (1, 0), (0, 1)):
    hm = O.refine_levels(G.crisscross_square(), lv0)
    args = G.config_fields(2)
    ref = capi.pipeline(ctx, capi.DeviceMesh.upload(ctx, hm), levels, *args, flags=capi.PIPE_GENERIC_EG).download()
    tctx = capi.Context(0, stream=torch.cuda.current_stream().cuda_stream)
    comm = dist.LocalComm(3)
    states = dist.make_states(hm, comm, lambda r: dist.CudaRankOps(tctx, "cuda:0"))
    states, nC, nE = dist.distributed_pipeline(states, comm, hm.nC, hm.nE, levels, *args)
    d = dist.collect(states)
    print("case", lv0, levels, "ranges", [(s.elo, s.ehi) for s in states])
    for k in ("edge_nodes", "edge_elements", "elem_edge", "node_edge_start"):
        a, b = d[k].reshape(-1), ref["topo"][k].reshape(-1)
        print(k, np.array_equal(a, b))
        if not np.array_equal(a, b):
            print(" dist", a.tolist()); print(" ref ", b.tolist())
