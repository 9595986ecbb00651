"""The C-ABI library loads and exports every symbol include/*.h declares
(no compute calls: runs without a GPU)."""

import ctypes
import glob
import os
import re

import pytest

from paper_1804_09666_b200 import _lib, build


def declared_symbols():
    syms = set()
    for h in glob.glob(os.path.join(build.INCLUDE, "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        syms |= set(re.findall(r"\b(bx_\w+)\s*\(", src))
    return sorted(syms)


@pytest.fixture(scope="module")
def lib():
    build.build()
    return ctypes.CDLL(build.LIB)


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ("bx_ntdm_f64", "bx_npdm_f64", "bx_mnpdm_f64", "bx_residual_inf_f64",
              "bx_workspace_bytes", "bx_last_error", "bx_version"):
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, f"missing exports: {missing}"


def test_binding_table_covers_header():
    assert set(declared_symbols()) <= set(_lib.exported_symbols())


def test_version_and_workspace_query(lib):
    L = _lib.lib()
    assert b"sm_100a" in L.bx_version()
    assert L.bx_workspace_bytes(_lib.SOLVER["npdm"], 8, 16, 0, 0) == 2 * 8 * 16 * 8
    assert L.bx_workspace_bytes(_lib.SOLVER["ntdm"], 8, 16, 0, 0) == 8 * 16 * 8


def test_argument_errors_without_gpu(lib):
    L = _lib.lib()
    # n below the minimum is rejected before any CUDA call
    rc = L.bx_ntdm_f64(None, None, None, None, None, None, None, 4, 1, 4, 0, 0, None, 0, None)
    assert rc == 1 and b"minimum" in L.bx_last_error()
    rc = L.bx_npdm_f64(*([None] * 9), 4, 8, 2, 0, 0, None, 0, None)
    assert rc == 1 and b"ld" in L.bx_last_error()
