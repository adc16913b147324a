import sys, time
sys.path.insert(0, '.')
import bench
from paper_2401_15557_b200 import capi
ctx = capi.Context(0)
dm = bench.build_input(ctx, 12)
capi.save_mesh_text(ctx, dm)
ctx.sync()
ctx.profile(True)
t0 = time.perf_counter()
import ctypes as C
for w in range(4):
    p, n = C.c_void_p(), C.c_size_t()
    t1 = time.perf_counter()
    ctx.check(ctx.lib.phfem_mesh_format(ctx.ptr, C.byref(dm.m), w, C.byref(p), C.byref(n)))
    t2 = time.perf_counter()
    ctx.lib.phfem_text_free(p)
    print(f"format {w}: {n.value / 1e6:.1f} MB in {(t2 - t1) * 1e3:.1f} ms", flush=True)
for k, (ms, cnt) in sorted(ctx.profile_read().items(), key=lambda kv: -kv[1][0])[:8]:
    print(f"  {k:24s} {ms:8.3f} ms x{cnt}")
