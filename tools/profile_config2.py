"""Config 2 (L-shape, 10 refinements from the 6-triangle mesh): per-step time
(CUDA events on the ctx stream, L2 flushed between steps) and per-kernel
totals of one step.  PHFEM_PROF_TIMELINE=1 adds the launch timeline."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2401_15557_b200 import capi, meshgen as G  # noqa: E402

ctx = capi.Context(0)
f = G.config_fields(2)
dm = capi.DeviceMesh.upload(ctx, G.lshape_6tri())
for _ in range(3):
    capi.pipeline(ctx, dm, 10, *f).release()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
stream = torch.cuda.ExternalStream(ctx.stream)
evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
ctx.sync()
for i in range(10):
    flush.fill_(i)
    evs[i][0].record(stream)
    capi.pipeline(ctx, dm, 10, *f).release()
    evs[i][1].record(stream)
ctx.sync()
print(f"config2 step {sum(a.elapsed_time(b) for a, b in evs) / 10:.3f} ms")
ctx.profile(True)
capi.pipeline(ctx, dm, 10, *f).release()
ctx.sync()
p = ctx.profile_read()
print(f"{sum(v[0] for v in p.values()):.3f} ms kernel sum, {sum(v[1] for v in p.values())} launches")
for k, v in sorted(p.items(), key=lambda kv: -kv[1][0])[:10]:
    print(f"  {k:22s} {v[0]:.4f} ms x{v[1]}")
