"""The given-mesh pipeline (SURVEY §8(d)'s reading of config 5: L13 mesh given
-> sort-based edge generation + classification + C + blocks / load / bD).
Without --once: per-kernel CUDA-event times over 3 steps after 2 warm-ups.
With --once: one pipeline call after building the input, for ncu:
  the input build launches 13 x (k_eg_tile, k_eg_emit), so
  ncu -k regex:'k_eg_tile$|k_eg_emit' -s 26 -c 2 python tools/profile_given.py 13 --once"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import build_input  # noqa: E402
from paper_2401_15557_b200 import capi, meshgen as G  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 13
ctx = capi.Context(0)
if "--bs" in sys.argv:
    ctx.set_eg_max_bs(int(sys.argv[sys.argv.index("--bs") + 1]))
dm = build_input(ctx, level)
fields = G.config_fields(5)
if "--once" in sys.argv:
    capi.pipeline(ctx, dm, 0, *fields).release()
    ctx.sync()
    print("given pipeline once ok")
    sys.exit(0)
for _ in range(2):
    capi.pipeline(ctx, dm, 0, *fields).release()
ctx.sync()
ctx.profile(True)
import torch  # noqa: E402
stream = torch.cuda.ExternalStream(ctx.stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for _ in range(3):
    capi.pipeline(ctx, dm, 0, *fields).release()
e1.record(stream)
ctx.sync()
ms = e0.elapsed_time(e1) / 3
prof = ctx.profile_read()
print(f"given L{level}: {ms:.3f} ms/step ({dm.m.nE / (ms * 1e-3):.3e} tri/s)")
for k, (kms, kn) in sorted(prof.items(), key=lambda kv: -kv[1][0]):
    print(f"  {k:24s} {kms / 3:8.3f} ms  x{kn // 3}")
