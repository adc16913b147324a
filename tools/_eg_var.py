"""k_eg_tile / emit times of the generic L12 -> L13 path (sort on both levels), per library."""
import os, sys
sys.path.insert(0, '.')
import bench
from paper_2401_15557_b200 import capi, meshgen as G
ctx = capi.Context(0)
dm = bench.build_input(ctx, 12)
f = G.config_fields(5)
for _ in range(2):
    capi.pipeline(ctx, dm, 1, *f, flags=capi.PIPE_GENERIC_EG).release()
ctx.sync()
ctx.profile(True)
for _ in range(3):
    capi.pipeline(ctx, dm, 1, *f, flags=capi.PIPE_GENERIC_EG).release()
ctx.sync()
p = ctx.profile_read()
print(os.environ.get("PHFEM_LIB", "default"), {k: round(v[0] / 3, 3) for k, v in sorted(p.items(), key=lambda kv: -kv[1][0])[:7]})
