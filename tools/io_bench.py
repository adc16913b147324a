"""Timing of the on-disk formats on in-memory text (no disk):
device mesh -> save_mesh text, text -> load_mesh device mesh, topology CSV,
against the reference's own load_mesh / save_mesh / CLI CSV on a smaller
mesh (oracle/_ref, one thread).  usage: python tools/io_bench.py [level] [ref_level]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import build_input  # noqa: E402
from oracle import reference as R  # noqa: E402
from paper_2401_15557_b200 import capi  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 else 12
ref_level = int(sys.argv[2]) if len(sys.argv) > 2 else 9
ctx = capi.Context(0)


def timed(fn, reps=3):
    best, out = 1e30, None
    for _ in range(reps):
        ctx.sync()
        t0 = time.perf_counter()
        out = fn()
        ctx.sync()
        best = min(best, time.perf_counter() - t0)
    return best, out


for lv, is_ref in ((level, False), (ref_level, True)):
    dm = build_input(ctx, lv)
    nE = dm.m.nE
    ts, text = timed(lambda: capi.save_mesh_text(ctx, dm), 2)
    nbytes = sum(len(t) for t in text)
    tl, m2 = timed(lambda: capi.load_mesh_text(ctx, *text), 2)
    topo = capi.build_topology(ctx, m2)
    tc, csv = timed(lambda: capi.topology_csv(ctx, m2, topo), 2)
    import tempfile
    with tempfile.TemporaryDirectory(dir="/dev/shm" if os.path.isdir("/dev/shm") else None) as td:
        tsd, _ = timed(lambda: capi.save_mesh_dir(ctx, dm, td), 2)
        tld, _ = timed(lambda: capi.load_mesh_dir(ctx, td), 2)
    print(f"device L{lv}: {nE} triangles, text {nbytes / 1e9:.2f} GB: save {ts:.3f} s "
          f"({nE / ts / 1e6:.1f} M tri/s), load {tl:.3f} s ({nE / tl / 1e6:.1f} M tri/s), "
          f"topology CSV {len(csv) / 1e9:.2f} GB in {tc:.3f} s (Python bytes); files in /dev/shm: "
          f"save_mesh_dir {tsd:.3f} s, load_mesh_dir {tld:.3f} s", flush=True)
    if is_ref and R.available():
        t0 = time.perf_counter()
        rm = R.load_mesh_text(*text)
        trl = time.perf_counter() - t0
        t0 = time.perf_counter()
        R.save_mesh_text(rm)
        trs = time.perf_counter() - t0
        t0 = time.perf_counter()
        R.topology_csv(rm)
        trc = time.perf_counter() - t0
        print(f"reference L{lv} (1 thread): save {trs:.3f} s ({nE / trs / 1e6:.2f} M tri/s), "
              f"load {trl:.3f} s ({nE / trl / 1e6:.2f} M tri/s), topology CSV (incl. build_topology) "
              f"{trc:.3f} s", flush=True)
    topo.release()
    m2.release()
    dm.release()
