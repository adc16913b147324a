"""the reference's on-disk formats — load_mesh / save_mesh
(mesh.cpp:114-180) and the CLI's topology CSV (tools/main.cpp:302-323).

The checker is the reference itself: its own mesh.cpp (load_mesh on
istringstreams, save_mesh on ostringstreams) and edge_topology.cpp compiled
in oracle/_ref.  not gpu: committed fixtures (tests/golden/io/io_golden.npz,
made by tools/make_golden_io.py from the reference) are reproduced by the
reference build.  gpu: csrc/io.cu against the reference — parsed arrays bit
for bit, written text byte for byte, and every validation error with the
reference's message and precedence.
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from oracle import reference as R
from paper_2401_15557_b200 import capi, meshgen as G

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden", "io", "io_golden.npz")
needs_ref = pytest.mark.skipif(not R.available(), reason="reference build unavailable")


def io_meshes():
    return [("square-L3", O.refine_levels(G.square_2tri(), 3)),
            ("lshape-L2", O.refine_levels(G.lshape_6tri(), 2)),
            ("crisscross-L2", O.refine_levels(G.crisscross_square(), 2)),
            ("jittered-L4", O.orient_ccw(G.stress_transform(O.refine_levels(G.square_2tri(), 4), 4)))]


# Malformed / unusual inputs: (name, coordinates, elements, dirichlet, neumann)
SQ_C = b"0 0\n1 0\n1 1\n0 1\n"
SQ_E = b"1 2 3\n1 3 4\n"
CASES = [
    ("ok-plain", SQ_C, SQ_E, b"1 2\n", b"3 2\n"),
    ("ok-crlf-blank-lines-no-final-newline", b"\n0 0\r\n  1\t0 \r\n\n1 1\r\n0 1", b"1 2 3\n\n 1 3 4 ", b"", b""),
    ("ok-signs-hex-exponents", b"+0 -0\n0x1p0 0.0e5\n1.000000000000000000000001 1E0\n0 .1e1\n", b"+1 +2 +03\n1 3 4\n",
     b"", b""),
    ("ok-flipped-and-foreign-pairs", SQ_C, SQ_E, b"2 1\n4 3\n2 4\n", b"1 4\n"),
    ("coords-count", b"0 0\n1 0 7\n1 1\n0 1\n", SQ_E, b"", b""),
    ("coords-one-entry", b"0 0\n1\n", SQ_E, b"", b""),
    ("coords-not-number", b"0 0\n1 zero\n1 1\n0 1\n", SQ_E, b"", b""),
    ("coords-trailing-junk", b"0 0\n1.5x 0\n", SQ_E, b"", b""),
    ("coords-nan", b"0 0\nnan 0\n", SQ_E, b"", b""),
    ("coords-inf", b"0 0\n1 -inf\n", SQ_E, b"", b""),
    ("coords-overflow", b"0 0\n1e400 0\n", SQ_E, b"", b""),
    ("coords-underflow", b"0 0\n1e-400 0\n", SQ_E, b"", b""),
    ("coords-subnormal", b"0 0\n1e-310 0\n", SQ_E, b"", b""),
    ("elements-count", SQ_C, b"1 2 3\n1 3\n", b"", b""),
    ("elements-not-index", SQ_C, b"1 2 3\n1 3 x\n", b"", b""),
    ("elements-float-index", SQ_C, b"1 2 3.0\n", b"", b""),
    ("elements-zero", SQ_C, b"0 2 3\n", b"", b""),
    ("elements-negative", SQ_C, b"1 2 3\n-1 3 4\n", b"", b""),
    ("elements-too-large", SQ_C, b"1 2 5\n", b"", b""),
    ("elements-long-overflow", SQ_C, b"1 2 99999999999999999999\n", b"", b""),
    ("elements-sign-only", SQ_C, b"1 2 +\n", b"", b""),
    ("elements-clockwise", SQ_C, b"1 3 2\n1 3 4\n", b"", b""),
    ("elements-degenerate", b"0 0\n1 0\n2 0\n", b"1 2 3\n", b"", b""),
    ("elements-area-before-parse", SQ_C, b"1 3 2\n1 3 x\n", b"", b""),
    ("elements-parse-before-area", SQ_C, b"1 3 x\n1 3 2\n", b"", b""),
    ("dirichlet-count", SQ_C, SQ_E, b"1 2\n3\n", b""),
    ("dirichlet-range", SQ_C, SQ_E, b"1 2\n3 9\n", b""),
    ("neumann-not-index", SQ_C, SQ_E, b"1 2\n", b"3 four\n"),
    ("elements-before-dirichlet", SQ_C, b"1 2 3\n1 3 9\n", b"1 x\n", b""),
]


def ref_load(c, e, d, n):
    try:
        rm = R.load_mesh_text(c, e, d, n)
    except RuntimeError as ex:
        return None, str(ex)
    return rm.host(), None


def arrays(hm):
    return [np.asarray(hm.coords), np.asarray(hm.elements), np.asarray(hm.dirichlet).reshape(-1, 2),
            np.asarray(hm.neumann).reshape(-1, 2)]


def same_mesh(a, b):
    for x, y in zip(arrays(a), arrays(b)):
        assert x.shape == y.shape
        assert np.array_equal(x.view(np.uint8), y.view(np.uint8))


# ---------------------------------------------------------------- fixtures (CPU)
@needs_ref
def test_reference_reproduces_io_fixtures():
    z = np.load(GOLDEN)
    for name, hm in io_meshes():
        rm = R.RMesh(hm)
        for w, part in enumerate(R.save_mesh_text(rm)):
            assert part == z[f"{name}_save{w}"].tobytes(), (name, w)
        assert R.topology_csv(rm) == z[f"{name}_csv"].tobytes(), name
    for name, c, e, d, n in CASES:
        hm, msg = ref_load(c, e, d, n)
        if msg is not None:
            assert msg == str(z[f"case_{name}_error"]), name
        else:
            for k, x in enumerate(arrays(hm)):
                assert np.array_equal(x, z[f"case_{name}_{k}"]), name


# ------------------------------------------------------------------ device
@pytest.fixture(scope="module")
def ctx():
    c = capi.Context(0)
    yield c
    c.close()


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("name,c,e,d,n", CASES, ids=[x[0] for x in CASES])
def test_gpu_load_mesh_text_matches_reference(ctx, name, c, e, d, n):
    want, msg = ref_load(c, e, d, n)
    if msg is not None:
        with pytest.raises(capi.PhfemError) as ex:
            capi.load_mesh_text(ctx, c, e, d, n)
        assert str(ex.value) == msg
    else:
        same_mesh(capi.load_mesh_text(ctx, c, e, d, n).download(), want)


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("idx", range(4))
def test_gpu_save_load_and_topology_csv_match_reference(ctx, idx):
    name, hm = io_meshes()[idx]
    rm = R.RMesh(hm)
    text = R.save_mesh_text(rm)
    dm = capi.DeviceMesh.upload(ctx, hm)
    assert capi.save_mesh_text(ctx, dm) == text
    loaded = capi.load_mesh_text(ctx, *text)
    same_mesh(loaded.download(), R.load_mesh_text(*text).host())
    topo = capi.build_topology(ctx, loaded)
    assert capi.topology_csv(ctx, loaded, topo) == R.topology_csv(R.load_mesh_text(*text))


@pytest.mark.gpu
@needs_ref
def test_gpu_mesh_dir_round_trip(ctx, tmp_path):
    hm = O.refine_levels(G.lshape_6tri(), 3)
    dm = capi.DeviceMesh.upload(ctx, hm)
    capi.save_mesh_dir(ctx, dm, str(tmp_path))
    names = ["coordinates.dat", "elements.dat", "dirichlet.dat", "neumann.dat"]
    files = [(tmp_path / f).read_bytes() for f in names]
    assert tuple(files) == R.save_mesh_text(R.RMesh(hm))
    same_mesh(capi.load_mesh_dir(ctx, str(tmp_path)).download(), R.load_mesh_text(*files).host())
    (tmp_path / "neumann.dat").unlink()  # optional file
    same_mesh(capi.load_mesh_dir(ctx, str(tmp_path)).download(), R.load_mesh_text(*files[:3]).host())
    with pytest.raises(capi.PhfemError, match=f"cannot open {tmp_path}/missing/coordinates.dat"):
        capi.load_mesh_dir(ctx, str(tmp_path / "missing"))
    with pytest.raises(capi.PhfemError, match="cannot write"):
        capi.save_mesh_dir(ctx, dm, str(tmp_path / "no" / "such" / "dir"))


@pytest.mark.gpu
@needs_ref
def test_gpu_io_large_round_trip(ctx):
    """Jittered square L9 (524 K triangles, full-precision coordinates):
    save -> load is the identity on the device, and the text equals the
    reference's save_mesh byte for byte."""
    hm = O.orient_ccw(G.stress_transform(O.refine_levels(G.square_2tri(), 9), 9))
    dm = capi.DeviceMesh.upload(ctx, hm)
    text = capi.save_mesh_text(ctx, dm)
    assert text == R.save_mesh_text(R.RMesh(hm))
    back = capi.load_mesh_text(ctx, *text).download()
    same_mesh(back, R.load_mesh_text(*text).host())
    assert np.array_equal(back.coords, hm.coords) and np.array_equal(back.elements, hm.elements)


@pytest.mark.gpu
def test_gpu_io_text_offsets_past_one_scan_block(ctx):
    """Square L11 (8.4 M element rows = 2049 scan tiles): the 64-bit line
    offset scan (k_scan64_*) carries across more than one 1024-tile block.
    The element text equals numpy's rendering of the 1-based ids (save_mesh,
    mesh.cpp:170-180) and save -> load is the identity."""
    hm = O.refine_levels(G.square_2tri(), 11)
    dm = capi.DeviceMesh.upload(ctx, hm)
    text = capi.save_mesh_text(ctx, dm)
    ids = (hm.elements.astype(np.int64) + 1)
    want = np.char.add(np.char.add(np.char.add(ids[:, 0].astype("S8"), b" "),
                                   np.char.add(ids[:, 1].astype("S8"), b" ")),
                       np.char.add(ids[:, 2].astype("S8"), b"\n"))
    assert text[1] == b"".join(want.tolist())
    back = capi.load_mesh_text(ctx, *text).download()
    assert np.array_equal(back.coords, hm.coords) and np.array_equal(back.elements, hm.elements)


# ---- the device "%.<P>g" formatter against glibc's printf ---------------------
def _fmt_cases():
    import struct
    rng = np.random.default_rng(17)
    bits = rng.integers(0, 2**63, 200000, dtype=np.uint64) | (rng.integers(0, 2, 200000, dtype=np.uint64) << 63)
    v = bits.view(np.float64)
    special = [0.0, -0.0, 1.0, -1.0, 0.1, 0.5, 1e-5, 1e-4, 9.9999e-5, 123456789012345678.0, 1e16, 1e17,
               9.999999999999999e16, 1e22, 1e23, 5e-324, 2.2250738585072014e-308, 1.7976931348623157e308,
               1125899906842624.5, 2.0**60, 2.0**64, 0.3, 2.0 / 3.0, float("inf"), -float("inf"), float("nan"),
               -float("nan"), 1.5, 2.5, 0.125, 1e-310, 4.35e-320, 999999999.5, 99999.999999999999]
    # exact ties at 17 and 10 digits: k / 2 with 17 / 10 significant digits before the .5
    ties = [float(k) + 0.5 for k in (1125899906842624, 1125899906842623, 99999999.0, 123456789.0)]
    grid = [m * 10.0 ** k for k in range(-30, 31) for m in (1.0, 0.5, 0.25, 0.999999, 7.0)]
    uni = list(rng.uniform(-2.0, 2.0, 20000)) + list(np.ldexp(rng.uniform(0.5, 1.0, 2000), rng.integers(-1074, 1024, 2000)))
    return np.concatenate([v, np.array(special + ties + grid + uni, dtype=np.float64)])


@pytest.mark.gpu
@pytest.mark.parametrize("prec", [17, 10, 1, 6, 15, 16])
def test_gpu_format_g_equals_glibc(ctx, prec):
    import ctypes as C
    libc = C.CDLL(None)
    vals = _fmt_cases()
    n = len(vals)
    dv = ctx.to_device(vals)
    out = ctx.alloc(32 * n)
    lens = ctx.alloc(4 * n)
    ctx.check(ctx.lib.phfem_format_g(ctx.ptr, C.c_void_p(dv), n, prec, C.c_void_p(out), C.c_void_p(lens)))
    txt = ctx.to_host(out, (n, 32), np.uint8)
    ln = ctx.to_host(lens, (n,), np.int32)
    for p in (dv, out, lens):
        ctx.free(p)
    buf = C.create_string_buffer(64)
    fmt = f"%.{prec}g".encode()
    bad = []
    for i in range(n):
        libc.snprintf(buf, 64, fmt, C.c_double(vals[i]))
        if bytes(txt[i, :ln[i]]) != buf.value:
            bad.append((vals[i], bytes(txt[i, :ln[i]]), buf.value))
            if len(bad) > 5:
                break
    assert not bad, bad


@pytest.mark.parametrize("prec", [17, 10, 1, 6, 15, 16])
def test_format_g_host_equals_glibc(prec):
    """The formatter the kernels use (fmt.cuh), run on the host: the same
    bytes as glibc's printf("%.Pg") for random bit patterns, subnormals,
    powers of ten and their neighbours, exact ties, infinities and NaNs."""
    import ctypes as C
    lib = capi.load_library()
    libc = C.CDLL(None)
    buf, out = C.create_string_buffer(64), C.create_string_buffer(64)
    fmt = f"%.{prec}g".encode()
    bad = []
    for v in _fmt_cases()[::4]:
        libc.snprintf(buf, 64, fmt, C.c_double(v))
        n = lib.phfem_format_g_host(float(v), prec, out)
        if out.raw[:n] != buf.value:
            bad.append((v, out.raw[:n], buf.value))
            if len(bad) > 5:
                break
    assert not bad, bad
