import sys
sys.path.insert(0, '.')
import bench
from paper_2401_15557_b200 import capi, meshgen as G
ctx = capi.Context(0)
coeffs, f, g, uD = G.config_fields(3)
dm = bench.build_input(ctx, 11)
topo = capi.build_topology(ctx, dm)
cls = capi.classify_edges(ctx, topo, dm)
plan = capi.CNPlan(ctx, dm, topo, cls, coeffs, f, g, uD, 1e-3)
W = G.uniform_pm1(5, plan.n_state)
dW = ctx.to_device(W); dr = ctx.alloc(8 * plan.n_state)
for n in range(3):
    plan.rhs_device(n, dW, dr)
ctx.sync()
print("ok")
