"""libpsd.so loads and exports every symbol include/psd.h declares (no GPU)."""

import ctypes
import os

import pytest

from paper_2603_18016_b200 import native


def test_header_declares_signatures():
    declared = native.header_symbols()
    assert declared, "no psd_* declarations found in include/psd.h"
    exp = native.header_symbols(os.path.join(os.path.dirname(native.HEADER),
                                             "psd_experimental.h"))
    assert sorted(exp) == sorted(native.EXPERIMENTAL)
    assert sorted(native.SIGNATURES) == sorted(declared + exp)


def test_library_exports_every_header_symbol():
    if not os.path.exists(native.LIB_PATH):
        pytest.fail("libpsd.so not built: run python -m paper_2603_18016_b200.build_native")
    lib = ctypes.CDLL(native.LIB_PATH)
    for name in native.header_symbols():
        assert hasattr(lib, name), name
    native.load()


def test_workspace_size_is_pure_host_logic():
    lib = native.load()
    a = lib.psd_verify_workspace_bytes(32, 5, 128256, 128256, 1)
    b = lib.psd_verify_workspace_bytes(32, 5, 128256, 0, 0)
    assert a > b > 0
    assert a % 256 == 0
