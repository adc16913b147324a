"""Time phfem_step_matrix (generic from_triplets: hand-written radix sort +
run sums) on the square at level L (default 11: 8.4 M triangles, 176 M
triplets); per-kernel event times from the ctx profiler."""
import ctypes as C
import sys
import time

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2401_15557_b200 import capi, meshgen as G  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 else 11
ctx = capi.Context(0)
dm = capi.DeviceMesh.upload(ctx, G.square_2tri())
for _ in range(level):
    t = capi.build_topology(ctx, dm)
    dm = capi.red_refine(ctx, dm, t)
topo = capi.build_topology(ctx, dm)
cls = capi.classify_edges(ctx, topo, dm)
coeffs = capi.coeffs_const(((2.0, 0.3), (0.3, 1.0)), (1.0, -0.5), 0.7)
nE = dm.m.nE
bufs = [ctx.alloc(72 * nE) for _ in range(4)]
ctx.check(ctx.lib.phfem_assemble_volume(ctx.ptr, C.byref(dm.m), C.byref(coeffs), *[C.c_void_p(b) for b in bufs]))
csc = capi.phfem_csc()
ctx.check(ctx.lib.phfem_constraint_csc(ctx.ptr, C.byref(dm.m), C.byref(topo.t), C.byref(cls.c), C.byref(csc)))
ntrip = 9 * nE + 2 * csc.nnz
for it in range(4):
    out = capi.phfem_csc()
    if it == 3:
        ctx.profile(True)
    ctx.sync()
    t0 = time.perf_counter()
    ctx.check(ctx.lib.phfem_step_matrix(ctx.ptr, nE, *[C.c_void_p(b) for b in bufs], C.byref(csc), 1e-3, -1.0,
                                        C.byref(out)))
    ctx.sync()
    dt = time.perf_counter() - t0
    ctx.lib.phfem_csc_release(ctx.ptr, C.byref(out))
print(f"L{level}: {nE} triangles, {ntrip} triplets, step_matrix {dt * 1e3:.2f} ms (host wall, last of 4)")
for k, (ms, n) in sorted(ctx.profile_read().items(), key=lambda kv: -kv[1][0]):
    print(f"  {k:20s} {ms:8.3f} ms x{n}")
