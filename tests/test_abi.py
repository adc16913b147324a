"""The C-ABI library loads here (no GPU) and exports every symbol that
include/phfem_gpu.h declares; without a device the calls fail loudly."""
import ctypes
import os
import re

from paper_2401_15557_b200 import capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "phfem_gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(phfem_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    assert declared_functions() == sorted(capi.EXPORTED)


def test_library_exports_every_declared_symbol():
    lib = capi.load_library()
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.phfem_abi_version() == 1


def test_no_silent_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        return
    lib = capi.load_library()
    p = ctypes.c_void_p()
    st = lib.phfem_ctx_create(0, None, ctypes.byref(p))
    assert st == capi.ERR_NO_DEVICE
    try:
        capi.Context(0)
    except capi.PhfemError:
        pass
    else:
        raise AssertionError("Context() must raise without a B200")


def test_missing_library_raises(tmp_path, monkeypatch):
    monkeypatch.setattr(capi, "_lib", None)
    try:
        capi.load_library(str(tmp_path / "nope.so"))
    except RuntimeError as e:
        assert "not built" in str(e)
    else:
        raise AssertionError
    finally:
        monkeypatch.setattr(capi, "_lib", None)
