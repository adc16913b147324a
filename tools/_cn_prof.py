"""CN RHS per-kernel times (ctx event profile) at config 3 (L11); with
--once it runs 3 steps only (for ncu captures)."""
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
if "--once" not in sys.argv:
    ctx.profile(True)
    for n in range(20):
        plan.rhs_device(n, dW, dr)
    ctx.sync()
    for k, (ms, cnt) in sorted(ctx.profile_read().items(), key=lambda kv: -kv[1][0]):
        print(f"{k:24s} {ms / 20:.4f} ms/step  ({cnt // 20} launches/step)")
print("ok")
