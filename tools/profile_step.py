"""One config-5 step (L12 input resident -> L13 outputs) for ncu captures,
plus a host-synchronised per-API-call breakdown when run without ncu.

Launch order of the filtered kernels: 12 x k_eg_bucket while building the L12
input, then the step: k_eg_bucket (L12), k_eg_bucket (L13), k_volume,
k_constraint_csr  ->  ncu -k regex:'k_eg_bucket|k_volume|k_constraint_csr' -s 13 -c 3
"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import build_input  # noqa: E402
from paper_2401_15557_b200 import capi, meshgen as G  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 else 13
phases = "--phases" in sys.argv
ctx = capi.Context(0)
dm = build_input(ctx, level - 1)
coeffs, f, g, uD = G.config_fields(5)
r = capi.pipeline(ctx, dm, 1, coeffs, f, g, uD)
ctx.sync()
print("step ok", r.out.mesh.nE, r.out.topo.E)
r.release()
if phases:
    for rep in range(3):
        T = {}

        def tick(name, fn):
            ctx.sync()
            t0 = time.perf_counter()
            out = fn()
            ctx.sync()
            T[name] = T.get(name, 0.0) + (time.perf_counter() - t0) * 1e3
            return out
        t0 = time.perf_counter()
        topo = tick("build_topology L12", lambda: capi.build_topology(ctx, dm))
        fine = tick("red_refine", lambda: capi.red_refine(ctx, dm, topo))
        if "--fused" in sys.argv:
            topo2 = tick("refine_topology L13", lambda: capi.refine_topology(ctx, dm, topo, fine))
        else:
            topo2 = tick("build_topology L13", lambda: capi.build_topology(ctx, fine))
        tick("release L12 topo", topo.release)
        cls = tick("classify_edges", lambda: capi.classify_edges(ctx, topo2, fine))
        nE = fine.m.nE
        bufs = [ctx.alloc(72 * nE) for _ in range(4)]
        tick("assemble_volume", lambda: ctx.check(ctx.lib.phfem_assemble_volume(
            ctx.ptr, C.byref(fine.m), C.byref(coeffs), *[C.c_void_p(b) for b in bufs])))
        lb = ctx.alloc(24 * nE)
        tick("assemble_load", lambda: ctx.check(ctx.lib.phfem_assemble_load(
            ctx.ptr, C.byref(fine.m), C.byref(f), 0.0, C.c_void_p(lb))))
        csr = capi.phfem_csr()
        tick("assemble_constraint", lambda: ctx.check(ctx.lib.phfem_assemble_constraint(
            ctx.ptr, C.byref(fine.m), C.byref(topo2.t), C.byref(cls.c), C.byref(csr))))
        tot = (time.perf_counter() - t0) * 1e3
        ctx.lib.phfem_csr_release(ctx.ptr, C.byref(csr))
        for b in bufs + [lb]:
            ctx.free(b)
        cls.release()
        topo2.release()
        fine.release()
        print(f"rep {rep}: total {tot:.2f} ms  " + "  ".join(f"{k}={v:.2f}" for k, v in T.items()))
dm.release()
ctx.close()
