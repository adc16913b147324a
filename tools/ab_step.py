"""A/B of library builds on the config-5 step (L12 resident -> L13 outputs):
per-kernel CUDA-event times (ctx profiling) and the step time, per variant,
interleaved rounds so clock / thermal drift hits every variant alike.

  python tools/ab_step.py [--level 13] [--rounds 3] [--steps 4] LIB [LIB ...]
  (LIB: a path to a build of libphfem_b200.so, e.g. from tools/variants.sh,
   optionally followed by @VAR=VAL[,VAR=VAL] environment settings, e.g.
   paper_2401_15557_b200/libphfem_b200.so@PHFEM_VOL_PARENTS=0)
  --config4: the config-4 step instead (stress L12 -> normalise -> ... -> L13)
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, os, sys, time
sys.path.insert(0, %r)
from bench import build_input
from paper_2401_15557_b200 import capi, meshgen as G
level, steps, levels = %d, %d, %d
ctx = capi.Context(0)
dm = build_input(ctx, level - levels)
f = G.config_fields(5)
for _ in range(2):
    capi.pipeline(ctx, dm, levels, *f).release()
ctx.sync()
ctx.profile(True)
ts = []
for _ in range(steps):
    ctx.sync(); t0 = time.perf_counter()
    r = capi.pipeline(ctx, dm, levels, *f)
    ctx.sync(); ts.append((time.perf_counter() - t0) * 1e3)
    r.release()
prof = ctx.profile_read()
ctx.profile(False)
print("RESULT " + json.dumps({"wall_ms": sorted(ts)[len(ts) // 2],
      "kernels": {k: v[0] / steps for k, v in prof.items()}}))
"""


CHILD4 = r"""
import ctypes as C, json, os, sys, time
sys.path.insert(0, %r)
from bench import config4_input
from paper_2401_15557_b200 import capi, meshgen as G
level, steps = %d, %d
ctx = capi.Context(0)
dm, keep, nflip = config4_input(ctx, level - 1)
f = G.config_fields(4)
def step():
    ctx.check(ctx.lib.phfem_memcpy_d2d(ctx.ptr, C.c_void_p(dm.m.elements), C.c_void_p(keep), 12 * dm.m.nE))
    capi.orient_ccw(ctx, dm)
    capi.pipeline(ctx, dm, 1, *f).release()
for _ in range(2):
    step()
ctx.sync()
ctx.profile(True)
ts = []
for _ in range(steps):
    ctx.sync(); t0 = time.perf_counter()
    step()
    ctx.sync(); ts.append((time.perf_counter() - t0) * 1e3)
prof = ctx.profile_read()
ctx.profile(False)
print("RESULT " + json.dumps({"wall_ms": sorted(ts)[len(ts) // 2],
      "kernels": {k: v[0] / steps for k, v in prof.items()}}))
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--level", type=int, default=13)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--given", action="store_true", help="the L13 mesh given (levels = 0)")
    ap.add_argument("--config4", action="store_true", help="the config-4 stress step")
    ap.add_argument("libs", nargs="+")
    a = ap.parse_args()
    res = {lib: [] for lib in a.libs}
    for _ in range(a.rounds):
        for lib in a.libs:
            path, _, kv = lib.partition("@")
            env = dict(os.environ, PHFEM_LIB=os.path.abspath(path))
            env.update(x.split("=", 1) for x in kv.split(",") if x)
            code = (CHILD4 % (ROOT, a.level, a.steps) if a.config4 else
                    CHILD % (ROOT, a.level, a.steps, 0 if a.given else 1))
            out = subprocess.run([sys.executable, "-c", code], env=env,
                                 capture_output=True, text=True, timeout=600)
            line = [x for x in out.stdout.splitlines() if x.startswith("RESULT ")]
            if not line:
                print(lib, "FAILED", out.stderr[-2000:], flush=True)
                continue
            res[lib].append(json.loads(line[0][7:]))
    for lib, rs in res.items():
        if not rs:
            continue
        ks = {}
        for r in rs:
            for k, v in r["kernels"].items():
                ks.setdefault(k, []).append(v)
        kern = {k: min(v) for k, v in ks.items()}
        tot = sum(kern.values())
        top = sorted(kern.items(), key=lambda kv: -kv[1])[:8]
        print(f"{os.path.basename(lib):32s} wall {min(r['wall_ms'] for r in rs):7.3f} ms  kernels {tot:7.3f} ms  " +
              "  ".join(f"{k} {v:.3f}" for k, v in top), flush=True)


if __name__ == "__main__":
    main()
