"""Per-launch timeline of one single-GPU config-5 step (L12 resident -> L13),
gaps included (run with PHFEM_PROF_TIMELINE=1: the ctx prints start / duration
/ gap of every launch; gaps are host work, memsets and copies)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import build_input  # noqa: E402
from paper_2401_15557_b200 import capi, meshgen as G  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 else 13
levels = 0 if "--given" in sys.argv else 1
ctx = capi.Context(0)
dm = build_input(ctx, level - levels)
fields = G.config_fields(5)
for _ in range(3):
    capi.pipeline(ctx, dm, levels, *fields).release()
ctx.sync()
ctx.profile(True)
capi.pipeline(ctx, dm, levels, *fields).release()
prof = ctx.profile_read()
tot = sum(v[0] for v in prof.values())
print(f"L{level} {'given' if levels == 0 else 'step'}: kernels {tot:.3f} ms")
