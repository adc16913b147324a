"""Per-rank cost model of the sharded step from W ranks
emulated on one GPU: every rank has its own phfem ctx (per-rank CUDA-event
kernel times), the exchanges go through LocalComm wrapped to count the bytes
each rank RECEIVES per phase (all-to-all: the other ranks' slices for it;
all-gather: every other rank's tensor; all-reduce: 2 (W-1)/W of the tensor,
ring).  Model: T_W = max_r kernel_ms(r) + max_r recv_bytes(r) / BW (no overlap),
BW = 900 GB/s per direction (NVLink 5 / NVSwitch).
usage: python tools/dist_model.py [W] [final level]"""
import json
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from bench import build_input  # noqa: E402
from paper_2401_15557_b200 import capi, dist, meshgen as G  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 8
level = int(sys.argv[2]) if len(sys.argv) > 2 else 13
if "--a2a" in sys.argv:   # the all-to-all form of the halo exchanges instead of peer windows
    dist.P2P = False
BW = 900e9


class CountingComm(dist.LocalComm):
    def __init__(self, world):
        super().__init__(world)
        self.recv = defaultdict(lambda: [0] * world)   # phase -> bytes received per rank
        self.phase = "start"

    @staticmethod
    def nb(t):
        return t.numel() * t.element_size()

    def all_reduce(self, ts, op):
        for r in range(self.world):
            self.recv[self.phase][r] += int(2 * (self.world - 1) / self.world * self.nb(ts[r]))
        super().all_reduce(ts, op)

    def all_gather(self, ts):
        tot = sum(self.nb(t) for t in ts)
        for r in range(self.world):
            self.recv[self.phase][r] += tot - self.nb(ts[r])
        return super().all_gather(ts)

    def account(self, remote, rec_bytes):
        """peer-window stores: rank d receives what the others stored into it"""
        for rem in remote:
            r = rem.cpu().tolist()
            for d in range(self.world):
                self.recv[self.phase][d] += int(r[d]) * rec_bytes

    def all_to_all_v(self, sends, counts):
        out = super().all_to_all_v(sends, counts)
        for d in range(self.world):
            own = int(counts[d][d]) * (self.nb(sends[d]) // max(sends[d].shape[0], 1))
            self.recv[self.phase][d] += self.nb(out[d]) - own
        return out


ctx0 = capi.Context(0, stream=torch.cuda.current_stream().cuda_stream)
hm = build_input(ctx0, level - 1).download()
fields = G.config_fields(5)
ctxs = [capi.Context(0, stream=torch.cuda.current_stream().cuda_stream) for _ in range(W)]
# warm-up run (pool growth, first-touch), then the measured one
comm = dist.LocalComm(W)
states = dist.make_states(hm, comm, lambda r: dist.CudaRankOps(ctxs[r], "cuda:0"))
dist.distributed_pipeline(states, comm, hm.nC, hm.nE, 1, *fields)
for s in states:
    s.ops.release()
del states
torch.cuda.synchronize()
comm = CountingComm(W)
states = dist.make_states(hm, comm, lambda r: dist.CudaRankOps(ctxs[r], "cuda:0"))


class PhaseTrace(dist._Trace):
    def __call__(self, what):
        super().__call__(what)
        comm.phase = f"after {what}"


for c in ctxs:
    c.profile(True)
orig = dist._Trace
dist._Trace = PhaseTrace
states, nC, nE = dist.distributed_pipeline(states, comm, hm.nC, hm.nE, 1, *fields)
dist._Trace = orig
torch.cuda.synchronize()
kms = []
top = []
for r, c in enumerate(ctxs):
    prof = c.profile_read()
    kms.append(sum(v[0] for v in prof.values()))
    top.append(sorted(((k, round(v[0], 3), v[1]) for k, v in prof.items()), key=lambda kv: -kv[1])[:30])
recv_tot = [sum(v[r] for v in comm.recv.values()) for r in range(W)]
out = {
    "W": W, "step": f"square L{level - 1} -> L{level} ({nE} triangles), config-5 fields",
    "kernel_ms_per_rank": [round(x, 3) for x in kms],
    "recv_bytes_per_rank": recv_tot,
    "recv_bytes_by_phase_max_rank": {k: max(v) for k, v in comm.recv.items()},
    "model_ms_no_overlap": round(max(kms) + max(recv_tot) / BW * 1e3, 3),
    "nvlink_ms": round(max(recv_tot) / BW * 1e3, 3),
    "top_kernels_slowest_rank": top[max(range(W), key=lambda r: kms[r])],
}
print(json.dumps(out, indent=1))
