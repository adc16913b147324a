"""Config-3 CN right-hand side at level L (default 11): per-kernel event times
over 20 steps (L2 flushed between steps), or --once: one rhs after the plan,
for ncu:  ncu -k regex:'k_cn_tma|k_cn_rows' -c 2 python tools/profile_cn.py 11 --once"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from bench import build_input  # noqa: E402
from paper_2401_15557_b200 import capi, meshgen as G  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 11
ctx = capi.Context(0)
coeffs, f, g, uD = G.config_fields(3)
dm = build_input(ctx, level)
topo = capi.build_topology(ctx, dm)
cls = capi.classify_edges(ctx, topo, dm)
plan = capi.CNPlan(ctx, dm, topo, cls, coeffs, f, g, uD, 1e-3)
W = G.uniform_pm1(5, plan.n_state)
dW, dr = ctx.to_device(W), ctx.alloc(8 * plan.n_state)
ctx.sync()
if "--once" in sys.argv:
    plan.rhs_device(0, dW, dr)
    ctx.sync()
    print("cn rhs once ok")
    sys.exit(0)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
stream = torch.cuda.ExternalStream(ctx.stream)
for n in range(3):
    plan.rhs_device(n, dW, dr)
ctx.sync()
evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
with torch.cuda.stream(stream):
    for n in range(20):
        flush.fill_(n)
        evs[n][0].record(stream)
        plan.rhs_device(n, dW, dr)
        evs[n][1].record(stream)
ctx.sync()
print(f"CN rhs L{level}: step (events on the ctx stream, L2 flushed) "
      f"{sum(a.elapsed_time(b) for a, b in evs) / 20:.4f} ms")
ctx.profile(True)
with torch.cuda.stream(stream):
    for n in range(20):
        flush.fill_(n)
        plan.rhs_device(n, dW, dr)
ctx.sync()
prof = ctx.profile_read()
tot = sum(v[0] for k, v in prof.items() if k.startswith("k_cn"))
print(f"CN rhs L{level} ({dm.m.nE} triangles): kernels {tot / 20:.4f} ms/step")
for k, (ms, n) in sorted(prof.items(), key=lambda kv: -kv[1][0]):
    print(f"  {k:16s} {ms / 20:8.4f} ms x{n // 20}")
