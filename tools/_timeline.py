"""One profiled L12 -> L13 pipeline step with the per-launch timeline
(PHFEM_PROF_TIMELINE=1): where the step's non-kernel time goes."""
import os, sys
sys.path.insert(0, '.')
os.environ["PHFEM_PROF_TIMELINE"] = "1"
import bench
from paper_2401_15557_b200 import capi, meshgen as G
ctx = capi.Context(0)
dm = bench.build_input(ctx, 12)
f = G.config_fields(5)
for _ in range(3):
    capi.pipeline(ctx, dm, 1, *f).release()
ctx.sync()
ctx.profile(True)
capi.pipeline(ctx, dm, 1, *f).release()
ctx.profile_read()
ctx.profile(False)
