"""CPU: the C-ABI library loads (no GPU needed to load it) and exports every
entry point include/skr.h declares; the Python binding covers all of them."""
import ctypes
import os
import re

import pytest

from paper_1602_02350_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "skr.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(skr_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ["skr_lanczos", "skr_problem_create", "skr_full_gradient", "skr_component_gradient",
                 "skr_svrg", "skr_epoch", "skr_ctx_create_dist", "skr_last_error"]:
        assert must in syms
    assert len(syms) >= 35


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_python_binding_covers_the_header():
    assert set(declared_symbols()) == set(_lib.SIGNATURES)


def test_binding_loads_and_reports_abi():
    lib = _lib.load()
    assert lib.skr_abi_version() == 1
    assert isinstance(lib.skr_last_error(), bytes)


def test_no_cuda_device_is_a_loud_error():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1602_02350_b200 import skridge
    with pytest.raises(skridge.DeviceError):
        skridge.Context(0)
