"""Parity at the BASELINE sizes: the CUDA path against the C
oracle on the benchmarked meshes themselves, not reduced levels.

* config 5 — the bench step (square L12 resident -> red_refine -> L13
  topology + classification + C + blocks + load + bD, 134,217,728 triangles)
  and the GIVEN L13 mesh (sort-based edge generation on 402.6 M occurrences:
  its packed items need 27 + 29 + 1 = 57 bits, so bs = 7 and every tile spans
  two buckets — the multi-sub-bucket tile path at full size);
* config 4 — the jittered / permuted / rotated / flipped L12 stress mesh,
  normalised on the device, refined to L13 and assembled;
* config 2 — the L-shape pipeline, 10 refinements from the 6-triangle mesh;
* config 3 — the Crank-Nicolson right-hand side at L11, every 10th step.

Integer outputs (mesh, topology, classification, C pattern) and the +-*/sqrt
values (blocks, C values, bD with u_D = 0) are compared bit for bit; the load
(device sin vs glibc) within 1e-12 relative per entry (BASELINE north_star).
Element-local outputs are compared in element-range chunks: the oracle
assembles each chunk on its own host thread (ctypes drops the GIL) while the
device slices are copied back, so host memory stays ~40 GB at L13.

Reference semantics: proj/src/edge_topology.cpp:52-177, refine.cpp:7-53,
assembly.cpp:97-242, elliptic.cpp:54-55, parabolic.cpp:21-37,56-64,95-103."""
import concurrent.futures as cf
import os
import time

import numpy as np
import pytest

from oracle import oracle as O
from paper_2401_15557_b200 import capi, meshgen as G

pytestmark = pytest.mark.gpu

REL_TOL = 1e-12
THREADS = max(1, min(16, os.cpu_count() or 1))
CHUNK = 1 << 25          # entries per device -> host copy
ELEM_CHUNK = 1 << 21     # elements per oracle assembly task


def log(msg):
    print(f"[scale {time.strftime('%H:%M:%S')}] {msg}", flush=True)


def _first_bad(ok):
    return int(np.argmin(ok))


def dev_equal(ctx, ptr, ref, dtype, what):
    """Device array at ptr == ref bit for bit, copied back in chunks."""
    ref = np.ascontiguousarray(ref).reshape(-1)
    assert ref.dtype == np.dtype(dtype), (what, ref.dtype)
    item = ref.dtype.itemsize
    bits = np.uint64 if item == 8 else np.uint32
    for a in range(0, ref.size, CHUNK):
        b = min(ref.size, a + CHUNK)
        got = ctx.to_host(ptr + a * item, (b - a,), dtype)
        g, e = got.view(bits), ref[a:b].view(bits)
        if not np.array_equal(g, e):
            bad = np.flatnonzero(g != e)
            i = int(bad[0])
            raise AssertionError(f"{what}: {bad.size} entries differ, first at {a + i}: "
                                 f"{got[i]!r} vs {ref[a + i]!r}")


def rel_close(got, exp, what, tol=REL_TOL):
    err = np.abs(got - exp)
    ok = (err <= tol * np.abs(exp)) | (got == exp)
    if not ok.all():
        i = _first_bad(ok)
        raise AssertionError(f"{what}: {int((~ok).sum())} entries off, first at {i}: {got[i]!r} vs {exp[i]!r}")
    return float(np.max(err / np.maximum(np.abs(exp), 1e-300))) if err.size else 0.0


class OracleL:
    """The oracle's outputs for one final mesh (topology, classification, C,
    Neumann / Dirichlet vectors); blocks and load are recomputed per chunk."""

    def __init__(self, hm, fields):
        self.hm, self.fields = hm, fields
        coeffs, f, g, uD = fields
        t0 = time.time()
        self.om, self.ot = O.build_topology(hm)
        self.oc = O.classify_edges(self.om, self.ot)
        log(f"oracle topology + classification ({hm.nE} triangles, E = {self.ot.t.E}): {time.time() - t0:.1f} s")
        t0 = time.time()
        self.csr = O.OCsr(self.om, self.ot, self.oc)
        self.ln = O.assemble_neumann(self.om, self.ot, self.oc, g)
        self.bd = O.assemble_dirichlet(self.om, self.ot, self.oc, uD)
        log(f"oracle C (nnz {self.csr.s.nnz}) + Neumann + Dirichlet: {time.time() - t0:.1f} s")


def check_pipeline(ctx, res, ref: OracleL, check_mesh=True):
    """Every output of a device pipeline result against the oracle."""
    o = res.out
    hm = ref.hm
    t0 = time.time()
    if check_mesh:
        assert (o.mesh.nC, o.mesh.nE, o.mesh.nD, o.mesh.nN) == (hm.nC, hm.nE, len(hm.dirichlet), len(hm.neumann))
        dev_equal(ctx, o.mesh.coords, hm.coords, np.float64, "coords")
        dev_equal(ctx, o.mesh.elements, hm.elements, np.int32, "elements")
        dev_equal(ctx, o.mesh.dirichlet, hm.dirichlet, np.int32, "dirichlet pairs")
        dev_equal(ctx, o.mesh.neumann, hm.neumann, np.int32, "neumann pairs")
    t = ref.ot.t
    assert (o.topo.E, o.topo.n_interior, o.topo.n_boundary) == (t.E, t.n_interior, t.n_boundary)
    tv = ref.ot.views()
    for k, ptr in [("edge_nodes", o.topo.edge_nodes), ("edge_elements", o.topo.edge_elements),
                   ("local_in_tplus", o.topo.local_in_tplus), ("local_in_tminus", o.topo.local_in_tminus),
                   ("interior_edges", o.topo.interior_edges), ("boundary_edges", o.topo.boundary_edges),
                   ("elem_edge", o.topo.elem_edge), ("node_edge_start", o.topo.node_edge_start)]:
        dev_equal(ctx, ptr, tv[k], np.int32, k)
    cv = ref.oc.views()
    assert o.cls.L == ref.oc.L
    for k, ptr in [("dirichlet_edge_ids", o.cls.dirichlet_edge_ids), ("neumann_edge_ids", o.cls.neumann_edge_ids),
                   ("retained_edges", o.cls.retained_edges), ("retained_pos", o.cls.retained_pos)]:
        dev_equal(ctx, ptr, cv[k], np.int32, k)
    assert o.C.nnz == ref.csr.s.nnz
    dev_equal(ctx, o.C.row_ptr, ref.csr.ptr, np.int32, "C row_ptr")
    dev_equal(ctx, o.C.col_idx, ref.csr.idx, np.int32, "C col_idx")
    dev_equal(ctx, o.C.values, ref.csr.val, np.float64, "C values")
    dev_equal(ctx, o.bd, ref.bd, np.float64, "bD")
    log(f"mesh / topology / classification / C / bD bit-exact: {time.time() - t0:.1f} s")

    # element-local outputs: oracle chunks on host threads, device slices copied back
    t0 = time.time()
    coeffs, f, _, _ = ref.fields
    nE = hm.nE
    none = np.zeros((0, 2), np.int32)

    def work(a):
        b = min(nE, a + ELEM_CHUNK)
        sub = capi.HostMesh(hm.coords, hm.elements[a:b], none, none)
        blocks = O.assemble_volume(sub, coeffs)
        load = O.assemble_load(sub, f) + ref.ln[3 * a:3 * b]   # elliptic.cpp:54-55: b + LN
        return a, b, blocks, load

    worst = 0.0
    starts = list(range(0, nE, ELEM_CHUNK))
    with cf.ThreadPoolExecutor(THREADS) as ex:
        pending = [ex.submit(work, a) for a in starts[:2 * THREADS]]
        nxt = 2 * THREADS
        while pending:
            a, b, blocks, load = pending.pop(0).result()
            if nxt < len(starts):
                pending.append(ex.submit(work, starts[nxt]))
                nxt += 1
            for name, exp, ptr in zip(("B", "D", "M", "M0"), blocks, (o.B, o.D, o.M, o.M0)):
                got = ctx.to_host(ptr + 72 * a, (b - a, 9), np.float64)
                if not np.array_equal(got, exp):
                    bad = np.argwhere(got != exp)[0]
                    raise AssertionError(f"{name}: element {a + bad[0]} entry {bad[1]}: "
                                         f"{got[tuple(bad)]!r} vs {exp[tuple(bad)]!r}")
            worst = max(worst, rel_close(ctx.to_host(o.load + 24 * a, (3 * (b - a),), np.float64), load,
                                         f"load elements [{a}, {b})"))
    log(f"B / D / M / M0 bit-exact, load (b + LN) max rel err {worst:.2e}: {time.time() - t0:.1f} s")
    return worst


# ---------------------------------------------------------------- config 5
@pytest.fixture(scope="module")
def square_l12_l13():
    t0 = time.time()
    hm12 = O.refine_levels(G.square_2tri(), 12)
    hm13 = O.red_refine(hm12)
    log(f"oracle square L12 ({hm12.nE}) and L13 ({hm13.nE}) meshes: {time.time() - t0:.1f} s")
    ref = OracleL(hm13, G.config_fields(5))
    yield hm12, ref
    del ref


def test_config5_step_L12_to_L13(ctx, square_l12_l13):
    """The bench step itself: L12 resident -> L13 outputs (134,217,728 triangles)."""
    hm12, ref = square_l12_l13
    assert ref.hm.nE == 134217728
    dm = capi.DeviceMesh.upload(ctx, hm12)
    t0 = time.time()
    res = capi.pipeline(ctx, dm, 1, *G.config_fields(5))
    ctx.sync()
    log(f"device pipeline L12 -> L13: {time.time() - t0:.2f} s (first call)")
    try:
        check_pipeline(ctx, res, ref)
    finally:
        res.release()
        dm.release()


def test_config5_given_L13(ctx, square_l12_l13):
    """SURVEY §8(d)'s reading of config 5: the L13 mesh given, so the sort-based
    edge generation runs on 402.6 M occurrences with two buckets per tile
    (57-bit items, bs = 7) and classification + C fused into its emit pass."""
    _, ref = square_l12_l13
    hm = ref.hm
    lo_bits = int(hm.nC - 1).bit_length()
    occ_bits = int(3 * hm.nE - 1).bit_length()
    assert (lo_bits, occ_bits) == (27, 29)  # 57 packed bits -> bs = min(8, 64 - 57) = 7
    dm = capi.DeviceMesh.upload(ctx, hm)
    res = capi.pipeline(ctx, dm, 0, *G.config_fields(5))
    try:
        check_pipeline(ctx, res, ref, check_mesh=False)
    finally:
        res.release()
        dm.release()


# ---------------------------------------------------------------- config 4
def test_config4_stress_L12_to_L13(ctx):
    """Jittered (U[-0.2h, 0.2h], seed 1), permuted (seed 2), rotated (seed 3)
    and flipped (seed 4) L12 square; orientation normalised on the device
    (a18), then the bench step with config-2 coefficients."""
    level = 12
    t0 = time.time()
    raw = G.stress_transform(O.refine_levels(G.square_2tri(), level), level)
    assert (G.signed_area2(raw) < 0).any()
    hm12 = O.orient_ccw(raw)
    hm13 = O.red_refine(hm12)
    log(f"oracle stress L12 mesh, normalised, refined to L13: {time.time() - t0:.1f} s")
    dm = capi.DeviceMesh.upload(ctx, raw)
    capi.orient_ccw(ctx, dm)
    dev_equal(ctx, dm.m.elements, hm12.elements, np.int32, "normalised elements")
    dev_equal(ctx, dm.m.coords, hm12.coords, np.float64, "jittered coords")
    del raw
    fields = G.config_fields(4)
    res = capi.pipeline(ctx, dm, 1, *fields)
    ref = OracleL(hm13, fields)
    try:
        check_pipeline(ctx, res, ref)
    finally:
        res.release()
        dm.release()


# ---------------------------------------------------------------- config 2
def test_config2_lshape_L10_pipeline(ctx):
    """The full config: 6-triangle L-shape, 10 refinements (6,291,456
    triangles), per-element A(x_c), delta(x_c), p = (0.1, -0.1)."""
    fields = G.config_fields(2)
    hm10 = O.refine_levels(G.lshape_6tri(), 10)
    assert hm10.nE == 6291456
    ref = OracleL(hm10, fields)
    dm = capi.DeviceMesh.upload(ctx, G.lshape_6tri())
    res = capi.pipeline(ctx, dm, 10, *fields)
    try:
        check_pipeline(ctx, res, ref)
    finally:
        res.release()
        dm.release()


# ---------------------------------------------------------------- config 3
@pytest.mark.parametrize("lam", ["state", "zero"])
def test_config3_cn_rhs_L11(ctx, lam):
    """Square L11 (8,388,608 triangles): B/D/M/M0/C once, then the CN
    right-hand side for steps 0, 10, ..., 90 (k = 1e-3), W ~ U[-1,1] (seed 5);
    lam = "zero": Lambda = 0 (the BASELINE's primal-only formula)."""
    hm = O.refine_levels(G.square_2tri(), 11)
    assert hm.nE == 8388608
    coeffs, f, g, uD = G.config_fields(3)
    om, ot = O.build_topology(hm)
    oc = O.classify_edges(om, ot)
    N, L = 3 * hm.nE, oc.L
    W = G.uniform_pm1(5, N + L)
    if lam == "zero":
        W[N:] = 0.0
    dm = capi.DeviceMesh.upload(ctx, hm)
    topo = capi.build_topology(ctx, dm)
    cls = capi.classify_edges(ctx, topo, dm)
    plan = capi.CNPlan(ctx, dm, topo, cls, coeffs, f, g, uD, 1e-3)
    steps = list(range(0, 100, 10))
    t0 = time.time()
    with cf.ThreadPoolExecutor(min(THREADS, 5)) as ex:   # ~6 GB of oracle operators per call
        refs = list(ex.map(lambda n: O.cn_rhs(om, ot, oc, coeffs, f, g, uD, 1e-3, n, W), steps))
    log(f"oracle CN rhs x{len(steps)} at L11: {time.time() - t0:.1f} s")
    worst = 0.0
    try:
        for n, ro in zip(steps, refs):
            worst = max(worst, rel_close(plan.rhs(n, W), ro, f"CN rhs step {n}"))
    finally:
        plan.close()
    log(f"CN rhs steps 0..90 max rel err {worst:.2e}")
