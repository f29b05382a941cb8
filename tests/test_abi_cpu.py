"""C-ABI library: loads, exports every declared symbol, and its compiled constants are the
reference's.  Runs without a GPU (no compute calls)."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest
import torch

from common import bits_equal
from paper_1501_04784_b200 import _native as N
from paper_1501_04784_b200.element import compiled_dn_table

HEADER = Path(__file__).resolve().parent.parent / "include" / "hexfem_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hx_[a-z0-9_]+)\s*\(", text)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = N.lib()
    names = declared_symbols()
    assert len(names) >= 14
    for name in names:
        assert hasattr(lib, name), name
    assert sorted(N.EXPORTED) == names


def test_abi_version():
    assert N.lib().hx_abi_version() == 4


def test_compiled_dn_table_is_the_reference_table(golden):
    assert bits_equal(compiled_dn_table(), golden["dn_table"])


def test_compiled_pack_tables(golden):
    rows = np.empty(36, dtype=np.int32)
    cols = np.empty(36, dtype=np.int32)
    N.lib().hx_pack_tables(rows.ctypes.data_as(ctypes.c_void_p), cols.ctypes.data_as(ctypes.c_void_p))
    assert np.array_equal(rows, golden["pack_rows"]) and np.array_equal(cols, golden["pack_cols"])


def test_workspace_queries():
    L = N.lib()
    small = L.hx_mesh_csc_workspace_bytes(1000, 1331)
    big = L.hx_mesh_csc_workspace_bytes(1_000_000, 1_030_301)
    assert 0 < small < big
    assert big >= 4 * 8 * 1_000_000  # adjacency alone
    assert L.hx_mesh_csc_workspace_bytes(-1, 5) == -1
    assert L.hx_triplet_csc_workspace_bytes(36_000, 1331) > 36_000 * 24
    assert L.hx_triplet_csc_workspace_bytes(-1, 5) == -1


def test_bad_arguments_are_value_errors_without_touching_the_gpu():
    L = N.lib()
    fail = N.HxFailInfo()
    rc = L.hx_integrate_mesh(None, 0, None, None, 5, 2, None, None, None, 0, ctypes.byref(fail), None)
    assert rc == N.HX_ERR_VALUE
    assert b"bad arguments" in L.hx_last_error()
    with pytest.raises(ValueError):
        N.check(rc, "hx_integrate_mesh")


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_product_path_fails_loudly_without_a_gpu():
    import paper_1501_04784_b200 as hx

    with pytest.raises(hx.NativeLibraryError):
        hx.stiffness_batch(np.zeros((1, 8, 3)), np.ones(1))


def test_rows_widen_host_threads():
    """hx_rows_widen (host code): int32 -> int64 sign extension, any thread count, empty input."""
    import numpy as np

    a = np.concatenate([np.array([0, -1, 2**31 - 1, -2**31], np.int32),
                        np.random.default_rng(0).integers(-2**31, 2**31, 3_000_001, dtype=np.int64).astype(np.int32)])
    for threads in (1, 3, 0):
        b = np.full(a.size, 7, np.int64)
        N.check(N.lib().hx_rows_widen(a.ctypes.data, b.ctypes.data, a.size, threads), "widen")
        assert np.array_equal(b, a.astype(np.int64))
    N.check(N.lib().hx_rows_widen(None, None, 0, 0), "widen empty")
