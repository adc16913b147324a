"""One given-L13 pipeline call (levels = 0) for ncu captures."""
import sys
sys.path.insert(0, '.')
import bench
from paper_2401_15557_b200 import capi, meshgen as G
ctx = capi.Context(0)
dm = bench.build_input(ctx, int(sys.argv[1]) if len(sys.argv) > 1 else 13)
capi.pipeline(ctx, dm, 0, *G.config_fields(5)).release()
ctx.sync()
print("ok")
