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


# ---- row-index codec (hx_rows_encode / hx_rows_decode): the format's executable spec -------------
def encode_rows_ref(col_ptr, rows, col_lo):
    """Per column: deltas d_0 = r_0 - c, d_i = r_i - r_(i-1), padded with zeros to a multiple of 4;
    per group of 4 one control byte (2 bits per delta: byte length - 1), all control bytes first,
    then the deltas' little-endian bytes.  Returns (counts u8, lens u8, stream bytes)."""
    import numpy as np

    counts, lens, out = [], [], bytearray()
    for j in range(len(col_ptr) - 1):
        r = [int(x) for x in rows[col_ptr[j]:col_ptr[j + 1]]]
        prev, deltas = col_lo + j, []
        for x in r:
            deltas.append(x - prev)
            prev = x
        deltas += [0] * ((4 - len(deltas) % 4) % 4)
        ctrl, data = bytearray(), bytearray()
        for g in range(len(deltas) // 4):
            c = 0
            for k in range(4):
                d = deltas[4 * g + k]
                nb = 1 if d < 1 << 8 else 2 if d < 1 << 16 else 3 if d < 1 << 24 else 4
                c |= (nb - 1) << (2 * k)
                data += d.to_bytes(nb, "little")
            ctrl.append(c)
        counts.append(len(r))
        lens.append(len(ctrl) + len(data))
        out += ctrl + data
    return np.array(counts, np.uint8), np.array(lens, np.uint8), np.frombuffer(bytes(out), np.uint8)


def _codec_case(seed, ncols, col_lo):
    import numpy as np

    rng = np.random.default_rng(seed)
    counts = rng.integers(0, 34, ncols)
    counts[rng.random(ncols) < 0.1] = 0
    cp = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    rows = []
    for j, m in enumerate(counts):
        c = col_lo + j
        if m == 0:
            continue
        gaps = rng.choice([1, 2, 399, 401, 160_801, 2**20 + 3, 2**27], size=m - 1)
        col = np.concatenate([[c], c + np.cumsum(gaps)])
        rows.append(np.minimum(col, 2**31 - 1 - (m - 1 - np.arange(m))))  # stay below 2^31, ascending
    rows = np.concatenate(rows).astype(np.int64) if rows else np.empty(0, np.int64)
    return cp, rows


@pytest.mark.parametrize("seed,ncols,col_lo,threads", [(1, 1, 0, 1), (2, 7, 5, 1), (3, 5000, 1234, 4),
                                                        (4, 70000, 10, 0), (5, 3, 2**30, 2)])
def test_row_codec_host_decoder_matches_format(seed, ncols, col_lo, threads):
    """hx_rows_decode (host C++, SSSE3) inverts the reference encoding of the format, any thread
    count, empty / single-row columns and deltas up to 2^27; col_ptr ends are offset by row_base."""
    import numpy as np

    from paper_1501_04784_b200.transfer import decode_rows

    cp, rows = _codec_case(seed, ncols, col_lo)
    counts, lens, data = encode_rows_ref(cp, rows, col_lo)
    buf = np.zeros(data.size + 16, np.uint8)
    buf[:data.size] = data
    out = np.full(rows.size + 4, -7, np.int64)
    ends = np.zeros(ncols, np.int64)
    decode_rows(counts, lens, buf, data.size, col_lo, 1000, ends, out, threads)
    assert np.array_equal(out[:rows.size], rows) and np.all(out[rows.size:] == -7)
    assert np.array_equal(ends, 1000 + cp[1:])


def test_row_codec_rejects_inconsistent_stream():
    import numpy as np

    from paper_1501_04784_b200.errors import ConfigurationError
    from paper_1501_04784_b200.transfer import decode_rows

    cp, rows = _codec_case(9, 100, 0)
    counts, lens, data = encode_rows_ref(cp, rows, 0)
    buf = np.zeros(data.size + 16, np.uint8)
    buf[:data.size] = data
    with pytest.raises((ValueError, ConfigurationError)):
        decode_rows(counts, lens, buf, data.size - 1, 0, 0, np.zeros(100, np.int64), np.zeros(rows.size + 4, np.int64), 1)
