"""Guard mode (PHFEM_GUARD=1): the device-side memory check that stands in for
compute-sanitizer (closed on this GPU pool).  Every library block carries
4 KB red zones on both sides, checked on the device when it is freed, and a
poisoned payload (so reads of never-written memory change results that the
parity tests compare bit for bit).  The whole GPU suite is run under it
(tools/guard_run.sh); this test proves the detector fires."""
import ctypes as C

import numpy as np
import pytest

from paper_2401_15557_b200 import capi

pytestmark = pytest.mark.gpu


def test_guard_detects_out_of_bounds_write(monkeypatch):
    monkeypatch.setenv("PHFEM_GUARD", "1")
    ctx = capi.Context(0)
    try:
        p = ctx.alloc(100)
        # 100 bytes asked: payload rounded to 256, so 600 bytes reach into the red zone
        src = np.arange(600, dtype=np.uint8)
        ctx.check(ctx.lib.phfem_memcpy_h2d(ctx.ptr, C.c_void_p(p), src.ctypes.data_as(C.c_void_p), 600))
        ctx.free(p)
        with pytest.raises(capi.PhfemError, match="out-of-bounds write into the red zone"):
            ctx.sync()
    finally:
        ctx.close()


def test_guard_clean_pipeline(monkeypatch):
    """A small pipeline under guard mode: no red-zone hit, results unchanged."""
    from paper_2401_15557_b200 import meshgen as G
    monkeypatch.setenv("PHFEM_GUARD", "1")
    ref_ctx = capi.Context(0)
    ctx = capi.Context(0)
    try:
        args = G.config_fields(2)
        a = capi.pipeline(ctx, capi.DeviceMesh.upload(ctx, G.lshape_6tri()), 3, *args).download()
        ctx.sync()
        b = capi.pipeline(ref_ctx, capi.DeviceMesh.upload(ref_ctx, G.lshape_6tri()), 3, *args).download()
        for k in ("B", "C_values", "load", "bd"):
            assert np.array_equal(a[k], b[k]), k
    finally:
        ctx.close()
        ref_ctx.close()
