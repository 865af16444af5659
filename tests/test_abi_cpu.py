"""CPU-only checks of the boundary: librmips.so loads, exports every symbol include/rmips.h
declares, and argument validation answers without touching the GPU."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rmips.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"RMIPS_API[^;]*?\b(rmips_\w+)\s*\(", src, flags=re.S)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__ as g
    g.build()
    from paper_2110_07131_b200 import rmips
    return rmips


def test_header_declares_the_abi():
    names = _declared()
    for n in ("rmips_build_index", "rmips_query", "rmips_query_stats", "rmips_free_index", "rmips_status_string"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    so = ctypes.CDLL(lib.LIB_PATH)
    for n in _declared():
        assert hasattr(so, n), n
    assert sorted(lib.EXPORTED) == _declared()


def test_status_strings_and_version(lib):
    assert lib.lib.rmips_status_string(0) == b"ok"
    assert b"capacity" in lib.lib.rmips_status_string(4)
    assert b"sm_100a" in lib.lib.rmips_version()


def test_validation_without_gpu(lib):
    L = lib.lib
    h = ctypes.c_void_p()
    # NULL out handle
    assert L.rmips_build_index(None, 0, None, 1, 1, 1, None, None) == lib.RMIPS_ERR_INVALID
    # m < 1, d < 1
    assert L.rmips_build_index(None, 0, None, 0, 4, 1, None, ctypes.byref(h)) == lib.RMIPS_ERR_INVALID
    assert L.rmips_build_index(None, 0, ctypes.c_void_p(8), 3, 0, 1, None, ctypes.byref(h)) == lib.RMIPS_ERR_INVALID
    # d > 1024 unsupported (the tensor-core path covers 1..1024); the SIMT build d <= 256
    assert L.rmips_build_index(None, 0, ctypes.c_void_p(8), 3, 1025, 1, None, ctypes.byref(h)) == lib.RMIPS_ERR_INVALID
    assert L.rmips_build_index_ex(None, 0, ctypes.c_void_p(8), 3, 300, 1, 1, None, ctypes.byref(h)) == lib.RMIPS_ERR_INVALID
    # k_max < 1
    assert L.rmips_build_index(None, 0, ctypes.c_void_p(8), 3, 4, 0, None, ctypes.byref(h)) == lib.RMIPS_ERR_K_RANGE
    # query on a NULL index
    tot = ctypes.c_int64()
    assert L.rmips_query(None, None, 0, 1, None, None, 0, ctypes.byref(tot), None) == lib.RMIPS_ERR_INVALID
    assert L.rmips_query_stats(None, None) == lib.RMIPS_ERR_INVALID
    assert b"NULL" in L.rmips_last_error()


def test_product_does_not_import_oracle():
    """The product package never references oracle/ (DESIGN.md §4)."""
    pkg = os.path.join(ROOT, "paper_2110_07131_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "liboracle" not in txt, f
