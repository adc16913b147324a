#!/usr/bin/env python3
"""Bench: triangles/s of the fused edge-generation -> red-refinement -> assembly
step (fp64) on B200, with the HBM-roofline fraction, the end-to-end (host
buffers through the C ABI) number and the CPU baseline.

Workload (BASELINE.json configs[4], "config 5"): unit square (2-triangle coarse
mesh), the L12 mesh (33.5 M triangles) resident in HBM; one step =
build_topology(L12) -> red_refine -> build_topology(L13) -> classify_edges ->
B, D, M, M0 blocks + load (b + LN) + C in CSR + bD on the 134 M-triangle L13
mesh, config-2 coefficients (per-element A(x_c), delta(x_c), p = (0.1,-0.1)).
Inputs are far larger than L2 (126 MB), so no flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "triangles/sec for edge-gen+refine+assembly (fp64), % of HBM roofline, 1/2/4/8 GPU"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---- algorithmic (compulsory) bytes, SURVEY.md §8(d) -------------------------
def eg_bytes(nE, E):
    return 27 * nE + 32 * E


def rf_bytes(nC, nE, E):  # parent sizes
    return 32 * nC + 72 * nE + 24 * E


def as_bytes(nC, nE, E, L, nnz):
    return 16 * nC + 324 * nE + 28 * E + 12 * L + 12 * nnz


def kernel_bytes(name, s, p):
    """Algorithmic bytes of ONE launch of a step kernel (inputs read once,
    outputs written once).  s = final (L13) sizes, p = parent
    (L12) sizes.  None for kernels without a model."""
    nC, nE, E, L, nnz = s["nC"], s["nE"], s["E"], s["L"], s["nnz"]
    pC, pE, pEd = p["nC"], p["nE"], p["E"]
    return {
        # B, D, M, M0 (4 x 72 B) + load (24 B) written; the parent elements +
        # parent coords read (the children's vertices are rebuilt from the
        # parent, VolArgs::parents; PHFEM_VOL_PARENTS=0: 12 nE + 16 nC read)
        "k_volume": (12 * nE + 16 * nC if os.environ.get("PHFEM_VOL_PARENTS") == "0"
                     else 12 * pE + 16 * pC) + 312 * nE,
        # parent build_topology, sort pass: packed items in (3 x 8 B / element),
        # one 16-B edge record per edge + node_edge_start (4 B / node) out
        "k_eg_tile": 24 * pE + 16 * pEd + 4 * pC,
        # emit pass: records in; edge_nodes, edge_elements, ltp, ltm, list slot
        # (28 B / edge) + elem_edge (12 B / element) out
        "k_eg_emit": 16 * pEd + 28 * pEd + 12 * pE,
        "k_eg_scatter": 12 * pE + 24 * pE,
        "k_eg_count": 12 * pE,
        # red_refine without midpoints: elements + elem_edge in, 4 children out
        "k_refine_elements": 24 * pE + 48 * pE,
        # fused refined level: parent edge records + elem_edge / opposite-vertex /
        # coordinate gathers in; fine topology (32 B/edge incl. list slot and
        # retained_pos), node_edge_start + midpoints + partner ranks (21 B per
        # parent edge), retained list + row_ptr (8 B/row), C entries (12 B) out
        "k_rl_level_full": (24 * pEd + pEd // 8 + 24 * pE + 16 * pC) +
                           (32 * E + 21 * pEd + 8 * L + 12 * nnz),
        # element pass: parent elements + elem_edge in, group starts + ranks
        # gathered (5 B per parent edge), children rows + fine elem_edge out
        "k_refine_children": 24 * pE + 5 * pEd + 96 * pE,
        "k_cls_retained": pEd // 8 + 4 * pEd + 4 * pEd,  # parent classification (retained_pos / retained_edges)
    }.get(name)


# ---- clocks during the timed region -------------------------------------------
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int, period_ms: int = 200):
        self.index, self.rows, self.proc, self.period = index, [], None, period_ms

    def __enter__(self):
        if self.period <= 0:
            return self
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", str(self.period)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi takes a while to start: wait for its first row, then
            # keep only the rows sampled while the timed region runs
            t_end = time.time() + 5.0
            while not self.rows and time.time() < t_end and self.proc.poll() is None:
                time.sleep(0.005)
            self.rows.clear()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            t_end = time.time() + 1.0  # a region shorter than the period: take the next row
            while not self.rows and time.time() < t_end and self.proc.poll() is None:
                time.sleep(0.005)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if len(r) > 2 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 2 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, n in enumerate(names):
                if len(r) > 5 + i and r[5 + i].lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# ---- distributed plumbing (torchrun) -------------------------------------------
def dist_init(n_gpus):
    import torch
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def dist_max(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def dist_barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ---- CPU side -------------------------------------------------------------------
def cpu_impl():
    """'reference' = the reference's own sources (oracle/_ref, built from
    /root/reference against shim/Eigen); 'port' = the C restatement."""
    from oracle import reference as R
    return "reference" if os.path.exists(R.LIB) else "port"


def cpu_sample_worker(args):
    level, steps, warmup, kind = args
    from oracle import oracle as O
    from paper_2401_15557_b200 import meshgen as G
    hm = O.refine_levels(G.square_2tri(), level)     # input generation, untimed
    fields = G.config_fields(5)
    times = []
    nE = 0
    for i in range(warmup + steps):
        if kind == "reference":
            from oracle import reference as R
            dt, nE = R.pipeline_seconds(hm, 1, *fields)
        else:
            t0 = time.perf_counter()
            r = O.pipeline(hm, 1, *fields)
            dt = time.perf_counter() - t0
            nE = r["mesh"].nE
            del r
        if i >= warmup:
            times.append(dt)
    return nE, times


def cpu_workers_available(per_worker_gb: float) -> int:
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    try:
        with open("/proc/meminfo") as f:
            mem = {l.split(":")[0]: int(l.split()[1]) for l in f}
        avail_gb = mem.get("MemAvailable", 0) / 1e6
    except Exception:
        avail_gb = 8.0
    return max(1, min(cores, int(avail_gb * 0.6 / per_worker_gb)))


def cpu_baseline_single(level=11):
    """One bounded sample on one core (about 10-30 s of CPU work): square
    L11 -> L12 pipeline (33.5 M triangles) by default."""
    kind = cpu_impl()
    nE, times = cpu_sample_worker((level, 1, 0, kind))
    what = ("reference sources (oracle/_ref, /root/reference/proj/src via shim/Eigen)" if kind == "reference"
            else "oracle/phfem_oracle.c (C restatement)")
    return {"value": nE / times[0], "unit": "triangles/s", "cores": 1, "kind": kind,
            "sample": f"square L{level} -> L{level + 1} pipeline ({nE} triangles): build_topology, red_refine, "
                      f"build_topology, classify_edges, B/D/M/M0, C, load+Neumann, Dirichlet; {what}; "
                      f"1 thread, {times[0]:.2f} s"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import multiprocessing as mp
    level = args.ref_level
    kind = cpu_impl()
    if kind == "reference":     # load oracle/_ref in the parent: the forked workers inherit the mapping
        from oracle import reference as R
        R.lib()
    P = cpu_workers_available(per_worker_gb=1.5)
    with mp.get_context("fork").Pool(P) as pool:
        res = pool.map(cpu_sample_worker, [(level, args.steps, args.warmup, kind)] * P)
    nE = res[0][0]
    per_step = [max(r[1][i] for r in res) for i in range(args.steps)]
    t = statistics.mean(per_step)
    value = P * nE / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "triangles/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"config5 pipeline sample: square L{level} -> L{level + 1}, "
                               f"{P} concurrent single-threaded samples", "triangles_per_sample": nE},
        "cpu_baseline": {"value": value, "unit": "triangles/s", "cores": P, "kind": kind,
                         "sample": f"{P} concurrent single-threaded samples (the reference has no threading), "
                                   f"each square L{level}->L{level + 1} ({nE} tri): build_topology, red_refine, "
                                   "build_topology, classify_edges, B/D/M/M0, C, load+Neumann, Dirichlet"},
        "e2e": {"value": value, "unit": "triangles/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---- GPU side ---------------------------------------------------------------------
def ncu_traffic(level, kernel):
    """Per-launch DRAM bytes of `kernel` at `level` from the committed ncu
    capture (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            return json.load(fh).get(f"L{level}:{kernel}")
    except (OSError, ValueError):
        return None


def build_input(ctx, level):
    from paper_2401_15557_b200 import capi, meshgen as G
    dm = capi.DeviceMesh.upload(ctx, G.square_2tri())
    for _ in range(level):
        t = capi.build_topology(ctx, dm)
        nxt = capi.red_refine(ctx, dm, t)
        t.release()
        dm.release()
        dm = nxt
    ctx.sync()
    return dm


def run_ours_sharded(args, rank, world, local):
    """N > 1: the same step (L12 resident -> L13 outputs) sharded over the
    ranks: element ranges x tile-aligned key ranges, the bulk
    exchanges as peer-window kernels storing into the owners' arrays (CUDA IPC
    over NVLink), NCCL for the small collectives and the fences; the refined
    level sort-free in halo form.  --orch cpp (default): the host orchestration
    in C++ (csrc/dist_run.cu, phfem_dist_pipeline, its own NCCL communicator);
    --orch python: dist.py's.  Every rank keeps its slices; value = total L13
    triangles / max-over-ranks time."""
    import torch
    from paper_2401_15557_b200 import capi, dist, meshgen as G
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    ctx = capi.Context(local, stream=torch.cuda.current_stream(dev).cuda_stream)
    fields = G.config_fields(5)
    hm = build_input(ctx, args.level - 1).download()   # L12 input (untimed), replicated
    es = dist.element_splits(hm.nE, world)
    inp = dict(coords=torch.as_tensor(hm.coords).to(dev), elements=torch.as_tensor(hm.elements[es[rank]:es[rank + 1]]).to(dev),
               dirichlet=torch.as_tensor(hm.dirichlet).to(dev), neumann=torch.as_tensor(hm.neumann).to(dev))
    hist_sample = dist.HIST_SAMPLE if hm.nE >= dist.HIST_SAMPLE_MIN_ELEMENTS else 1
    if args.orch == "cpp":
        import torch.distributed as tdist
        uid = [capi.DistComm.nccl_unique_id() if rank == 0 else None]
        if world > 1:
            tdist.broadcast_object_list(uid, src=0)
        ccomm = capi.DistComm.nccl(uid[0], rank, world, local)
        mv = capi.phfem_mesh()
        mv.coords, mv.elements = inp["coords"].data_ptr(), inp["elements"].data_ptr()
        mv.dirichlet, mv.neumann = inp["dirichlet"].data_ptr(), inp["neumann"].data_ptr()
        mv.nC, mv.nE, mv.nD, mv.nN, mv.owned = hm.nC, int(es[rank + 1] - es[rank]), hm.dirichlet.shape[0], \
            hm.neumann.shape[0], 0

        def step():
            o = capi.dist_pipeline(ccomm, [ctx], [mv], hm.nC, hm.nE, 1, *fields, hist_sample=hist_sample)[0]
            x = o.o
            step.stats = {"E": x.E, "L": x.L, "nnz": 4 * x.L - 2 * (x.n_boundary - (x.E - x.L))}
            res = x.nC, x.nE, x.ehi - x.elo
            o.release()
            return res
    else:
        comm = dist.TorchComm()
        ops = dist.CudaRankOps(ctx, dev)

        def step():
            st = [dist.RankState(rank=rank, ops=ops, coords=inp["coords"], elements=inp["elements"],
                                 elo=int(es[rank]), ehi=int(es[rank + 1]), dirichlet=inp["dirichlet"],
                                 neumann=inp["neumann"])]
            st, nC, nE = dist.distributed_pipeline(st, comm, hm.nC, hm.nE, 1, *fields)
            n_own = st[0].ehi - st[0].elo
            step.stats = st[0].stats
            ops.release()
            return nC, nE, n_own

    for _ in range(args.warmup):
        nC, nE, n_own = step()
    if os.environ.get("PHFEM_DIST_KPROF"):  # per-kernel times of one step (debug)
        ctx.profile(True)
        step()
        for k, (kms, kn) in sorted(ctx.profile_read().items(), key=lambda kv: -kv[1][0])[:25]:
            print(f"[kprof] {k:28s} {kms:8.3f} ms  x{kn}", file=sys.stderr, flush=True)
        ctx.profile(False)
    stream = torch.cuda.current_stream(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist_barrier(world)
    torch.cuda.synchronize()
    launches0 = ctx.launches
    with ClockSampler(local, args.clock_ms) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            nC, nE, n_own = step()
        ev1.record(stream)
        torch.cuda.synchronize()
    ms_local = ev0.elapsed_time(ev1) / args.steps
    ms = dist_max(ms_local, world)
    dist_barrier(world)
    launches = (ctx.launches - launches0) // args.steps
    value = nE / (ms * 1e-3)
    peak, peak_kind = peaks()
    # whole-job compulsory bytes of the workload (as N = 1) against N x peak
    nE0, nC0 = hm.nE, hm.nC
    E0 = nC - nC0                          # one midpoint per parent edge
    E1, L1, nnz1 = step.stats["E"], step.stats["L"], step.stats["nnz"]
    compulsory = (eg_bytes(nE0, E0) + rf_bytes(nC0, nE0, E0) + eg_bytes(nE, E1) +
                  as_bytes(nC, nE, E1, L1, nnz1))
    gbs = compulsory / (ms * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": "triangles/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"config5: square L{args.level - 1} -> L{args.level} ({nE} triangles): "
                               "EG+RF+EG+AS, config-2 coefficients, sharded",
                   "parallelism": f"element-range x key-range sharding over {world} GPUs (peer-window "
                                  "exchange kernels over CUDA IPC / NVLink; NCCL for small collectives + fences)",
                   "orchestration": "C++ (phfem_dist_pipeline)" if args.orch == "cpp" else "Python (dist.py)",
                   "refined_edge_generation": "input level: occurrences stored into the key owners' buckets, "
                                              "owner dedup; refined level: sort-free from the parent topology "
                                              "(SURVEY f1), halo form (side records / group starts)",
                   "triangles": nE, "own_triangles_rank0": n_own, "l2": "inputs larger than L2 (no flush)"},
        "pipeline_roofline": {"compulsory_bytes_per_step": compulsory, "achieved_gbs": round(gbs, 1),
                              "peak": peak * world, "peak_kind": peak_kind, "frac": round(gbs / (peak * world), 4)},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_ours(args):
    from paper_2401_15557_b200 import capi, meshgen as G
    rank, world, local = dist_init(args.gpus)
    if world > 1 and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE = {world}")
    if (world > 1 and not args.replicas) or args.sharded:
        if world == 1:  # --sharded at N = 1: a one-rank NCCL group (exercises the collectives)
            import torch
            import torch.distributed as tdist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29517")
            torch.cuda.set_device(local)
            tdist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", local))
        return run_ours_sharded(args, rank, world, local)
    ctx = capi.Context(local)
    fields = G.config_fields(5)
    dm = build_input(ctx, args.level - 1)          # L12 input, resident in HBM
    # sizes at both levels (one untimed run)
    r = capi.pipeline(ctx, dm, 1, *fields, flags=capi.PIPE_GENERIC_EG if args.generic_eg else 0)
    o = r.out
    s = {"nC": o.mesh.nC, "nE": o.mesh.nE, "E": o.topo.E, "L": o.cls.L, "nnz": o.C.nnz}
    r.release()
    t0 = capi.build_topology(ctx, dm)
    s0 = {"nC": dm.m.nC, "nE": dm.m.nE, "E": t0.E}
    t0.release()
    compulsory = (eg_bytes(s0["nE"], s0["E"]) + rf_bytes(s0["nC"], s0["nE"], s0["E"]) +
                  eg_bytes(s["nE"], s["E"]) + as_bytes(s["nC"], s["nE"], s["E"], s["L"], s["nnz"]))

    flags = capi.PIPE_GENERIC_EG if args.generic_eg else 0
    for _ in range(args.warmup):
        capi.pipeline(ctx, dm, 1, *fields, flags=flags).release()
    ctx.sync()

    import torch
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local))
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist_barrier(world)
    ctx.sync()
    launches0 = ctx.launches
    ctx.profile(True)
    with ClockSampler(local, args.clock_ms) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            capi.pipeline(ctx, dm, 1, *fields, flags=flags).release()
        ev1.record(stream)
        ctx.sync()
    ms_local = ev0.elapsed_time(ev1) / args.steps
    prof = ctx.profile_read()
    ctx.profile(False)
    launches = (ctx.launches - launches0) // args.steps
    ms = dist_max(ms_local, world)
    dist_barrier(world)
    value = world * s["nE"] / (ms * 1e-3)

    peak, peak_kind = peaks()
    # dominant kernel -> roofline
    named = {k: v for k, v in prof.items() if kernel_bytes(k, s, s0) is not None}
    dom = max(named, key=lambda k: named[k][0])
    dom_ms, dom_n = named[dom]
    per_step_bytes = kernel_bytes(dom, s, s0) * (dom_n // args.steps)
    achieved = per_step_bytes / (dom_ms / args.steps * 1e-3) / 1e9
    per_kernel = {}
    for k, (kms, kn) in sorted(named.items(), key=lambda kv: -kv[1][0]):
        b = kernel_bytes(k, s, s0) * (kn // args.steps)
        gbs = b / (kms / args.steps * 1e-3) / 1e9
        per_kernel[k] = {"ms": round(kms / args.steps, 4), "GB/s": round(gbs, 1), "frac": round(gbs / peaks()[0], 4)}
    step_share = {k: round(v[0] / args.steps / ms_local, 4) for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0])}
    traffic = ncu_traffic(args.level, dom)
    roofline = {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "peak_kind": peak_kind,
                "traffic": traffic["bytes"] if traffic else None,
                "traffic_source": traffic["source"] if traffic else None,
                "algorithmic_bytes_per_step": per_step_bytes,
                "kernel_ms_per_step": round(dom_ms / args.steps, 4)}
    if dom == "k_volume":
        roofline["note"] = ("k_volume's stream is ~98 % writes (blocks + load out, parent mesh in): a frac near 1.0 "
                            "means it runs at the measured copy bandwidth (the peak is a read+write copy; a "
                            "write-only stream can reach slightly more)")
    pipeline_gbs = compulsory / (ms_local * 1e-3) / 1e9

    line = {
        "metric": METRIC, "value": value, "unit": "triangles/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak" if world > 1 else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"config5: square L{args.level - 1} -> L{args.level} "
                               f"({s['nE']} triangles): EG+RF+EG+AS, config-2 coefficients",
                   "refined_edge_generation": "sort-based (generic)" if args.generic_eg
                   else "from parent topology (SURVEY f1, bit-identical)",
                   "triangles": s["nE"], "edges": s["E"], "multipliers": s["L"], "nnz_C": s["nnz"],
                   "parallelism": "replicas" if world > 1 else "single",
                   "l2": "inputs larger than L2 (no flush)"},
        "roofline": roofline,
        "pipeline_roofline": {"compulsory_bytes_per_step": compulsory, "achieved_gbs": round(pipeline_gbs, 1),
                              "peak": peak, "frac": round(pipeline_gbs / peak, 4)},
        "kernel_share": step_share,
        "kernel_roofline": per_kernel,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }

    if rank == 0 and world == 1 and not args.no_given:
        dm.release()
        dm = None
        line["config5_given_mesh"] = run_given(ctx, args, fields)
    if rank == 0 and world == 1 and not args.no_configs:
        line["config4_stress"] = run_config4(ctx, args, G.config_fields(4))
        line["config2_lshape"] = run_config2(ctx, args)
    if rank == 0 and world == 1 and not args.no_cn:
        line["cn_rhs"] = run_cn_rhs(ctx, args)
    if rank == 0 and world == 1 and not args.no_e2e:
        line["e2e"] = run_e2e(ctx, args, fields)
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline_single(args.cpu_level)
    if dm is not None:
        dm.release()
    ctx.close()
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_given(ctx, args, fields):
    """SURVEY §8(d)'s reading of config 5: the L13 mesh GIVEN (no parent, so
    the sort-based edge generation) -> classification -> C -> blocks / load /
    bD; same metric, compulsory bytes eg_bytes + as_bytes (72.3 GB @ L13)."""
    import torch
    from paper_2401_15557_b200 import capi
    dm = build_input(ctx, args.level)
    r = capi.pipeline(ctx, dm, 0, *fields)
    o = r.out
    s = {"nC": o.mesh.nC, "nE": o.mesh.nE, "E": o.topo.E, "L": o.cls.L, "nnz": o.C.nnz}
    r.release()
    for _ in range(max(1, args.warmup - 1)):
        capi.pipeline(ctx, dm, 0, *fields).release()
    stream = torch.cuda.ExternalStream(ctx.stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.sync()
    steps = max(3, args.steps)
    e0.record(stream)
    for _ in range(steps):
        capi.pipeline(ctx, dm, 0, *fields).release()
    e1.record(stream)
    ctx.sync()
    ms = e0.elapsed_time(e1) / steps
    dm.release()
    compulsory = eg_bytes(s["nE"], s["E"]) + as_bytes(s["nC"], s["nE"], s["E"], s["L"], s["nnz"])
    peak, kind = peaks()
    gbs = compulsory / (ms * 1e-3) / 1e9
    return {"workload": f"config5 as SURVEY 8(d) reads it: square L{args.level} mesh given "
                        f"({s['nE']} triangles): EG (sort-based: no parent) + classification + C + "
                        "B/D/M/M0/load/bD, config-2 coefficients",
            "ms_per_step": round(ms, 3), "value": s["nE"] / (ms * 1e-3), "unit": "triangles/s", "steps": steps,
            "pipeline_roofline": {"compulsory_bytes_per_step": compulsory, "achieved_gbs": round(gbs, 1),
                                  "peak": peak, "peak_kind": kind, "frac": round(gbs / peak, 4)}}


def step_events(ctx, steps, before, step):
    """Per-step CUDA events on the ctx stream around `step` (`before` runs
    outside the events, e.g. restoring an input the step modifies).
    Returns the mean ms per step."""
    import torch
    stream = torch.cuda.ExternalStream(ctx.stream)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    ctx.sync()
    for i in range(steps):
        before()
        evs[i][0].record(stream)
        step()
        evs[i][1].record(stream)
    ctx.sync()
    return sum(a.elapsed_time(b) for a, b in evs) / steps


def config4_input(ctx, level):
    """Config 4's stress mesh at `level` (the square refined on the device,
    then jittered U[-0.2h, 0.2h] (seed 1), permuted (2), rotated (3) and
    flipped (4) on the host — input generation, untimed) uploaded raw; plus a
    device copy of the raw elements to restore before every step (the
    normalisation rewrites them in place)."""
    from paper_2401_15557_b200 import capi, meshgen as G
    base = build_input(ctx, level)
    hm = base.download()
    base.release()
    raw = G.stress_transform(hm, level)
    dm = capi.DeviceMesh.upload(ctx, raw)
    keep = ctx.to_device(raw.elements)
    nflip = int((G.signed_area2(raw) < 0).sum())
    return dm, keep, nflip


def run_config4(ctx, args, fields4):
    """BASELINE config 4: jittered / permuted / rotated / flipped L12 stress
    mesh -> orientation normalisation (a18) -> build_topology(L12) ->
    red_refine -> L13 topology + classification + C -> B/D/M/M0/load/bD with
    config-2 coefficients.  Compulsory bytes: the normalisation (elements read,
    coordinates read once, flipped rows rewritten) + the config-5 step's."""
    import ctypes as C
    from paper_2401_15557_b200 import capi
    dm, keep, nflip = config4_input(ctx, args.level - 1)
    nE0, nC0 = dm.m.nE, dm.m.nC
    restore = lambda: ctx.check(ctx.lib.phfem_memcpy_d2d(ctx.ptr, C.c_void_p(dm.m.elements), C.c_void_p(keep),
                                                          12 * nE0))

    def step():
        capi.orient_ccw(ctx, dm)
        capi.pipeline(ctx, dm, 1, *fields4).release()
    # sizes (one untimed step)
    restore()
    capi.orient_ccw(ctx, dm)
    r = capi.pipeline(ctx, dm, 1, *fields4)
    o = r.out
    s = {"nC": o.mesh.nC, "nE": o.mesh.nE, "E": o.topo.E, "L": o.cls.L, "nnz": o.C.nnz}
    r.release()
    t0 = capi.build_topology(ctx, dm)
    E0 = t0.E
    t0.release()
    for _ in range(max(1, args.warmup - 1)):
        restore()
        step()
    steps = max(3, args.steps)
    ms = step_events(ctx, steps, restore, step)
    ctx.free(keep)
    dm.release()
    normalise = 12 * nE0 + 16 * nC0 + 12 * nflip
    compulsory = (normalise + eg_bytes(nE0, E0) + rf_bytes(nC0, nE0, E0) + eg_bytes(s["nE"], s["E"]) +
                  as_bytes(s["nC"], s["nE"], s["E"], s["L"], s["nnz"]))
    peak, kind = peaks()
    gbs = compulsory / (ms * 1e-3) / 1e9
    return {"workload": f"config4: stress square L{args.level - 1} ({nE0} triangles; jitter U[-0.2h,0.2h] seed 1, "
                        f"permuted seed 2, rotated seed 3, {nflip} flipped seed 4) -> normalise -> EG -> RF -> "
                        f"L{args.level} EG + AS ({s['nE']} triangles), config-2 coefficients",
            "ms_per_step": round(ms, 3), "value": s["nE"] / (ms * 1e-3), "unit": "triangles/s", "steps": steps,
            "l2": "inputs larger than L2 (no flush); raw elements restored outside the per-step events",
            "pipeline_roofline": {"compulsory_bytes_per_step": compulsory, "achieved_gbs": round(gbs, 1),
                                  "peak": peak, "peak_kind": kind, "frac": round(gbs / peak, 4)},
            "ncu": ncu_traffic(args.level, "config4_sectors")}


def run_config2(ctx, args):
    """BASELINE config 2: the 6-triangle L-shape refined 10 times on the device
    (Σ10 (EG + RF) + EG + AS) -> 6,291,456 triangles, per-element
    A(x_c), delta(x_c), p = (0.1, -0.1).  Compulsory bytes summed over the levels."""
    from paper_2401_15557_b200 import capi, meshgen as G
    fields = G.config_fields(2)
    levels = 10
    dm = capi.DeviceMesh.upload(ctx, G.lshape_6tri())
    # per-level sizes for the byte count (untimed)
    compulsory = 0
    cur = capi.DeviceMesh.upload(ctx, G.lshape_6tri())
    for _ in range(levels):
        t = capi.build_topology(ctx, cur)
        compulsory += eg_bytes(cur.m.nE, t.E) + rf_bytes(cur.m.nC, cur.m.nE, t.E)
        nxt = capi.red_refine(ctx, cur, t)
        t.release()
        cur.release()
        cur = nxt
    cur.release()
    r = capi.pipeline(ctx, dm, levels, *fields)
    o = r.out
    s = {"nC": o.mesh.nC, "nE": o.mesh.nE, "E": o.topo.E, "L": o.cls.L, "nnz": o.C.nnz}
    r.release()
    compulsory += eg_bytes(s["nE"], s["E"]) + as_bytes(s["nC"], s["nE"], s["E"], s["L"], s["nnz"])
    step = lambda: capi.pipeline(ctx, dm, levels, *fields).release()
    for _ in range(max(1, args.warmup)):
        step()
    import torch
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=torch.device("cuda", torch.cuda.current_device()))
    it = [0]

    def before():
        it[0] += 1
        flush.fill_(it[0] & 0xff)
    ms = step_events(ctx, max(10, args.steps), before, step)
    del flush
    dm.release()
    peak, kind = peaks()
    gbs = compulsory / (ms * 1e-3) / 1e9
    return {"workload": f"config2: L-shape 6 triangles -> 10 refinements ({s['nE']} triangles): "
                        "sum of 10 x (EG + RF) + EG + AS, config-2 coefficients",
            "ms_per_step": round(ms, 3), "value": s["nE"] / (ms * 1e-3), "unit": "triangles/s",
            "steps": max(10, args.steps), "l2": "flushed between steps (512 MB write outside the per-step events)",
            "pipeline_roofline": {"compulsory_bytes_per_step": compulsory, "achieved_gbs": round(gbs, 1),
                                  "peak": peak, "peak_kind": kind, "frac": round(gbs / peak, 4)}}


def run_cn_rhs(ctx, args):
    """BASELINE config 3 (secondary line): square L11 (8.4 M triangles), B/D/M/M0
    and C assembled once, then the Crank-Nicolson right-hand side for 100 steps
    (k = 1e-3), state W ~ U[-1,1] (seed 5), solve excluded.  Bytes per step:
    SURVEY §8(d) stored-operator variant 16 nC + 147 nE + 4 E + 16 L (the
    recompute-from-geometry figure 16 nC + 75 nE + 4 E + 16 L is reported too)."""
    import torch
    from paper_2401_15557_b200 import capi, meshgen as G
    coeffs, f, g, uD = G.config_fields(3)
    dm = build_input(ctx, args.cn_level)
    topo = capi.build_topology(ctx, dm)
    cls = capi.classify_edges(ctx, topo, dm)
    plan = capi.CNPlan(ctx, dm, topo, cls, coeffs, f, g, uD, 1e-3)
    n_state = plan.n_state
    W = G.uniform_pm1(5, n_state)
    dW = ctx.to_device(W)
    dr = ctx.alloc(8 * n_state)
    for n in range(3):
        plan.rhs_device(n, dW, dr)
    stream = torch.cuda.ExternalStream(ctx.stream)
    # L2 flushed between steps (a 512 MB write, outside the timed events):
    # every step starts cold, as it would after a solve
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=torch.device("cuda", torch.cuda.current_device()))
    steps = 100
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    ctx.sync()
    with torch.cuda.stream(stream):
        for n in range(steps):
            flush.fill_(n & 0xff)
            evs[n][0].record(stream)
            plan.rhs_device(n, dW, dr)
            evs[n][1].record(stream)
    ctx.sync()
    ms = sum(a.elapsed_time(b) for a, b in evs) / steps
    del flush
    nC, nE, E, L = dm.m.nC, dm.m.nE, topo.E, cls.L
    bytes_recompute = 16 * nC + 75 * nE + 4 * E + 16 * L
    bytes_step = bytes_recompute + 72 * nE   # stored-operator variant
    peak, kind = peaks()
    gbs = bytes_step / (ms * 1e-3) / 1e9
    plan.close()
    ctx.free(dW)
    ctx.free(dr)
    cls.release()
    topo.release()
    dm.release()
    gbs_rc = bytes_recompute / (ms * 1e-3) / 1e9
    return {"workload": f"config3: square L{args.cn_level} ({nE} triangles), 100 CN right-hand sides, k=1e-3",
            "l2": "flushed between steps (512 MB write outside the per-step events)",
            "ms_per_step": round(ms, 4), "triangles_per_s": nE / (ms * 1e-3),
            "design": "k_cn_hyb: M_minus top block + coupling recomputed per step from the (L2-resident) "
                      "coordinates with the plan's expressions (bit-identical); streamed per element: "
                      "elements 12 + load factors 24 + U 24 + row codes 12 B through a 4-stage TMA ring, "
                      "rhs 24 B out; k_cn_rows: 16-B row records + U gathers, 8 B out",
            "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(gbs / peak, 4), "algorithmic_bytes_per_step": bytes_step,
                         "variant": "stored operator: 16 nC + 147 nE + 4 E + 16 L (SURVEY §8(d) "
                                    "recompute bytes + the 72 nE stored top block)",
                         "recompute_variant_bytes": bytes_recompute,
                         "frac_recompute_variant": round(gbs_rc / peak, 4),
                         "traffic": (ncu_traffic(args.cn_level, "cn_rhs_step") or {}).get("bytes"),
                         "peak_kind": kind}}


def run_e2e(ctx, args, fields):
    """Same step through the host-buffer C-ABI calls: pinned host mesh in,
    every output copied back into pinned host buffers, copies timed."""
    import ctypes as C
    import torch
    from paper_2401_15557_b200 import capi
    hm = build_input(ctx, args.e2e_level - 1).download()
    out = capi.phfem_pipeline_out()
    lib = ctx.lib

    def pinned(n, dt):
        return torch.empty(int(n), dtype=dt, pin_memory=True)

    inp = {"coords": pinned(hm.coords.size, torch.float64), "elements": pinned(hm.elements.size, torch.int32),
           "dirichlet": pinned(max(hm.dirichlet.size, 1), torch.int32),
           "neumann": pinned(max(hm.neumann.size, 1), torch.int32)}
    inp["coords"].numpy()[:] = hm.coords.ravel()
    inp["elements"].numpy()[:] = hm.elements.ravel()
    inp["dirichlet"].numpy()[:hm.dirichlet.size] = hm.dirichlet.ravel()
    inp["neumann"].numpy()[:hm.neumann.size] = hm.neumann.ravel()
    h2d = 16 * hm.nC + 12 * hm.nE + 8 * (len(hm.dirichlet) + len(hm.neumann))

    def run_once(dst):
        ctx.check(lib.phfem_pipeline_from_host(
            ctx.ptr, C.c_void_p(inp["coords"].data_ptr()), C.c_void_p(inp["elements"].data_ptr()),
            C.c_void_p(inp["dirichlet"].data_ptr()), C.c_void_p(inp["neumann"].data_ptr()), hm.nC, hm.nE,
            len(hm.dirichlet), len(hm.neumann), 1, C.byref(fields[0]), C.byref(fields[1]), C.byref(fields[2]),
            C.byref(fields[3]), 0.0, C.byref(out)))
        if dst is not None:
            ctx.check(lib.phfem_pipeline_download(ctx.ptr, C.byref(out), C.byref(dst)))
            run_once.wire = int(lib.phfem_pipeline_download_bytes(C.byref(out), C.byref(dst)))
        lib.phfem_pipeline_release(ctx.ptr, C.byref(out))

    # sizes -> pinned destination buffers
    ctx.check(lib.phfem_pipeline_from_host(
        ctx.ptr, C.c_void_p(inp["coords"].data_ptr()), C.c_void_p(inp["elements"].data_ptr()),
        C.c_void_p(inp["dirichlet"].data_ptr()), C.c_void_p(inp["neumann"].data_ptr()), hm.nC, hm.nE,
        len(hm.dirichlet), len(hm.neumann), 1, C.byref(fields[0]), C.byref(fields[1]), C.byref(fields[2]),
        C.byref(fields[3]), 0.0, C.byref(out)))
    o = out
    sizes = {"coords": (2 * o.mesh.nC, torch.float64), "elements": (3 * o.mesh.nE, torch.int32),
             "dirichlet": (2 * o.mesh.nD, torch.int32), "neumann": (2 * o.mesh.nN, torch.int32),
             "edge_nodes": (2 * o.topo.E, torch.int32), "edge_elements": (2 * o.topo.E, torch.int32),
             "local_in_tplus": (o.topo.E, torch.int32), "local_in_tminus": (o.topo.E, torch.int32),
             "interior_edges": (o.topo.n_interior, torch.int32), "boundary_edges": (o.topo.n_boundary, torch.int32),
             "elem_edge": (3 * o.mesh.nE, torch.int32), "dirichlet_edge_ids": (o.cls.nD, torch.int32),
             "neumann_edge_ids": (o.cls.nN, torch.int32), "retained_edges": (o.cls.L, torch.int32),
             "retained_pos": (o.topo.E, torch.int32), "C_row_ptr": (o.cls.L + 1, torch.int32),
             "C_col_idx": (o.C.nnz, torch.int32), "C_values": (o.C.nnz, torch.float64),
             "B": (9 * o.mesh.nE, torch.float64), "D": (9 * o.mesh.nE, torch.float64),
             "M": (9 * o.mesh.nE, torch.float64), "M0": (9 * o.mesh.nE, torch.float64),
             "load": (3 * o.mesh.nE, torch.float64), "bd": (o.cls.L, torch.float64)}
    nE_final = o.mesh.nE
    need = sum(n * (8 if dt == torch.float64 else 4) for n, dt in sizes.values())
    lib.phfem_pipeline_release(ctx.ptr, C.byref(out))
    try:
        with open("/proc/meminfo") as f:
            avail = {l.split(":")[0]: int(l.split()[1]) for l in f}.get("MemAvailable", 0) * 1024
    except Exception:
        avail = 0
    if need > 0.7 * avail:
        return {"value": None, "unit": "triangles/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": need,
                "skipped": f"host RAM {avail / 1e9:.0f} GB < 1.4 x {need / 1e9:.0f} GB of pinned outputs"}
    bufs = {k: pinned(max(n, 1), dt) for k, (n, dt) in sizes.items()}
    dst = capi.phfem_pipeline_host(**{k: bufs[k].data_ptr() for k in bufs})
    steps = max(1, min(args.steps, args.e2e_steps))
    run_once(dst)
    ctx.sync()
    t0 = time.perf_counter()
    for _ in range(steps):
        run_once(dst)
    dt = (time.perf_counter() - t0) / steps
    wire = run_once.wire
    return {"value": nE_final / dt, "unit": "triangles/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": wire, "delivered_bytes_per_step": need, "ms_per_step": dt * 1e3,
            "steps": steps,
            "note": "phfem_pipeline_from_host + phfem_pipeline_download (every output, reference layouts, "
                    "in pinned host buffers; compact PCIe encodings of the blocks / C / locals expanded "
                    "on the host)"}


def relaunch_under_torchrun(args) -> int:
    """`python bench.py --gpus N` (N > 1, no torchrun around it): start the N
    ranks ourselves — one process per GPU, the driver's own launch form — and
    return their exit code.  Rank 0 prints the one JSON line."""
    import socket
    if not args.dry_run:
        import torch
        if torch.cuda.device_count() < args.gpus:
            print(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs, this node has "
                  f"{torch.cuda.device_count()}", file=sys.stderr, flush=True)
            return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")        # NCCL's init lines show nranks / NVLS
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node",
           str(args.gpus), "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    print(f"[bench] launching {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd, env=env)


def run_dry(args):
    """--dry-run: the multi-rank harness alone (rendezvous, barrier, device
    max-over-ranks timing, rank 0's JSON line) over gloo on the CPU, no
    kernels — checks that `bench.py --gpus N` really starts N ranks."""
    import torch
    import torch.distributed as tdist
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        tdist.init_process_group("gloo")
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    if world > 1:
        tdist.barrier()
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": None, "unit": "triangles/s", "n_gpus": world,
                          "dry_run": True, "max_over_ranks": float(t.item()), "steps": args.steps,
                          "warmup": args.warmup}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--level", type=int, default=13, help="final refinement level (config 5: 13)")
    ap.add_argument("--e2e-level", type=int, default=13)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-level", type=int, default=11)
    ap.add_argument("--ref-level", type=int, default=8)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-cn", action="store_true", help="skip the config-3 CN right-hand-side line")
    ap.add_argument("--no-given", action="store_true", help="skip the given-L13-mesh (EG + AS) line")
    ap.add_argument("--cn-level", type=int, default=11)
    ap.add_argument("--no-configs", action="store_true", help="skip the config-4 / config-2 lines")
    ap.add_argument("--clock-ms", type=int, default=50, help="nvidia-smi sampling period (0 = off)")
    ap.add_argument("--sharded", action="store_true",
                    help="run the sharded (multi-GPU) pipeline even at N = 1")
    ap.add_argument("--orch", default="cpp", choices=["cpp", "python"],
                    help="sharded pipeline: host orchestration in C++ (phfem_dist_pipeline) or dist.py")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: N independent single-GPU replicas instead of the sharded pipeline")
    ap.add_argument("--generic-eg", action="store_true",
                    help="sort-based edge generation on the refined mesh too (no SURVEY f1 shortcut)")
    ap.add_argument("--dry-run", action="store_true",
                    help="multi-rank launch / timing harness only (gloo, CPU, no kernels)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        sys.exit(relaunch_under_torchrun(args))
    if args.dry_run:
        return run_dry(args)
    try:
        if args.impl == "reference":
            run_reference(args)
        else:
            run_ours(args)
    finally:
        if "torch.distributed" in sys.modules:
            import torch.distributed as tdist
            if tdist.is_available() and tdist.is_initialized():
                tdist.destroy_process_group()


if __name__ == "__main__":
    main()
