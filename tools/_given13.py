"""Config 5 as SURVEY §8(d) reads it: the L13 mesh given, EG + AS (levels = 0)."""
import sys, json
sys.path.insert(0, '.')
import bench, torch
from paper_2401_15557_b200 import capi, meshgen as G
ctx = capi.Context(0)
dm = bench.build_input(ctx, 13)
f = G.config_fields(5)
for _ in range(2):
    capi.pipeline(ctx, dm, 0, *f).release()
ctx.sync()
ctx.profile(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s = torch.cuda.ExternalStream(ctx.stream)
e0.record(s)
for _ in range(3):
    capi.pipeline(ctx, dm, 0, *f).release()
e1.record(s)
ctx.sync()
ms = e0.elapsed_time(e1) / 3
print("given-L13 EG+AS: %.2f ms/step, %.3e tri/s" % (ms, dm.m.nE / ms * 1e3))
for k, (kms, kn) in sorted(ctx.profile_read().items(), key=lambda kv: -kv[1][0])[:14]:
    print(f"  {k:28s} {kms / 3:8.3f} ms")
