"""Generic (sort-based) L12 -> L13 pipeline once: k_constraint_csr for ncu."""
import sys
sys.path.insert(0, '.')
import bench
from paper_2401_15557_b200 import capi, meshgen as G
ctx = capi.Context(0)
dm = bench.build_input(ctx, int(sys.argv[1]) if len(sys.argv) > 1 else 12)
r = capi.pipeline(ctx, dm, 1, *G.config_fields(5), flags=capi.PIPE_GENERIC_EG)
ctx.sync()
print("ok", r.out.topo.E)
