"""Host-synchronised per-step wall times of the pipeline + memory-pool state."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import build_input  # noqa: E402
from paper_2401_15557_b200 import capi, meshgen as G  # noqa: E402

try:
    from cuda.bindings import runtime as rt
except Exception:  # older cuda-python
    from cuda import cudart as rt


def pool_state():
    return ""
    err, pool = rt.cudaDeviceGetDefaultMemPool(0)
    out = []
    for a in (rt.cudaMemPoolAttr.cudaMemPoolAttrReservedMemCurrent, rt.cudaMemPoolAttr.cudaMemPoolAttrUsedMemCurrent):
        err, v = rt.cudaMemPoolGetAttribute(pool, a)
        out.append(int(v) / 1e9)
    return "reserved %.1f GB used %.1f GB" % tuple(out)


level = int(sys.argv[1]) if len(sys.argv) > 1 else 13
if "--torch" in sys.argv:
    import torch
    torch.cuda.init()
    _ev = torch.cuda.Event(enable_timing=True)
flags = capi.PIPE_GENERIC_EG if "--generic" in sys.argv else 0
ctx = capi.Context(0)
dm = build_input(ctx, level - 1)
f = G.config_fields(5)
if "--profile" in sys.argv:
    ctx.profile(True)
for i in range(int(os.environ.get("STEPS", "6"))):
    ctx.sync()
    t0 = time.perf_counter()
    r = capi.pipeline(ctx, dm, 1, *f, flags=flags)
    ctx.sync()
    t1 = time.perf_counter()
    r.release()
    ctx.sync()
    t2 = time.perf_counter()
    print(f"step {i}: pipeline {1e3 * (t1 - t0):.2f} ms release {1e3 * (t2 - t1):.2f} ms  {pool_state()}", flush=True)
dm.release()
ctx.close()
