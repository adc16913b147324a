"""Per-rank cost model of the sharded step with the C++
orchestration (phfem_dist_pipeline, local mode by default): W ranks emulated
on one GPU, each with its own phfem ctx on one stream (per-rank CUDA-event
kernel times), the communicator's statistics give the bytes every rank
RECEIVES per phase (peer-window records stored into it by the other ranks,
the other ranks' parts of all-gathers, 2 (W-1)/W of all-reduces).
Model: T_W = max_r kernel_ms(r) + max_r recv_bytes(r) / BW (no overlap),
BW = 900 GB/s per direction (NVLink 5 / NVSwitch).
usage: python tools/dist_model_cpp.py [W] [final level] [--windows]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from bench import build_input  # noqa: E402
from paper_2401_15557_b200 import capi, dist, meshgen as G  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 8
level = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 13
flags = capi.DIST_NO_LOCAL if "--windows" in sys.argv else 0
BW = 900e9

stream = torch.cuda.current_stream().cuda_stream
ctx0 = capi.Context(0, stream=stream)
dm = build_input(ctx0, level - 1)
hm_nC, hm_nE = dm.m.nC, dm.m.nE
fields = G.config_fields(5)
ctxs = [capi.Context(0, stream=stream) for _ in range(W)]
meshes = []
for r in range(W):
    lo, hi = hm_nE * r // W, hm_nE * (r + 1) // W
    v = capi.phfem_mesh()
    v.coords, v.dirichlet, v.neumann = dm.m.coords, dm.m.dirichlet, dm.m.neumann
    v.elements = dm.m.elements + 12 * lo
    v.nC, v.nE, v.nD, v.nN, v.owned = dm.m.nC, hi - lo, dm.m.nD, dm.m.nN, 0
    meshes.append(v)
comm = capi.DistComm.local_ranks(W)
hs = dist.HIST_SAMPLE if hm_nE >= dist.HIST_SAMPLE_MIN_ELEMENTS else 1
for o in capi.dist_pipeline(comm, ctxs, meshes, hm_nC, hm_nE, 1, *fields, hist_sample=hs, flags=flags):
    o.release()   # warm-up (windows, pool growth)
torch.cuda.synchronize()
comm.set_stats(True)
for c in ctxs:
    c.profile(True)
outs = capi.dist_pipeline(comm, ctxs, meshes, hm_nC, hm_nE, 1, *fields, hist_sample=hs, flags=flags)
torch.cuda.synchronize()
nE = outs[0].o.nE
for o in outs:
    o.release()
kms, top = [], []
for c in ctxs:
    prof = c.profile_read()
    kms.append(sum(v[0] for v in prof.values()))
    top.append(sorted(((k, round(v[0], 3), v[1]) for k, v in prof.items()), key=lambda kv: -kv[1])[:30])
st = comm.stats()
recv_tot = [sum(v[r] for v in st.values()) for r in range(W)]
out = {
    "W": W, "orchestration": "C++ (phfem_dist_pipeline)", "mode": "windows" if flags else "local",
    "step": f"square L{level - 1} -> L{level} ({nE} triangles), config-5 fields",
    "kernel_ms_per_rank": [round(x, 3) for x in kms],
    "recv_bytes_per_rank": recv_tot,
    "recv_bytes_by_phase_max_rank": {k: max(v) for k, v in st.items()},
    "model_ms_no_overlap": round(max(kms) + max(recv_tot) / BW * 1e3, 3),
    "nvlink_ms": round(max(recv_tot) / BW * 1e3, 3),
    "top_kernels_slowest_rank": top[max(range(W), key=lambda r: kms[r])],
}
print(json.dumps(out, indent=1))
