"""Matrix Market export (native, hx_mm_write) is byte-identical to the reference writer
(sparseio.py:73-87) -- host code, runs without a GPU."""

import numpy as np
import pytest

import oracle
from paper_1501_04784_b200.assemble import LowerCscMatrix
from paper_1501_04784_b200.sparseio import export_matrix_market


def random_lower_csc(rng, dim, special=True):
    cols = []
    for c in range(dim):
        k = rng.integers(0, 6)
        rows = np.unique(rng.integers(c, dim, size=k))
        cols.append(rows)
    col_ptr = np.concatenate([[0], np.cumsum([len(r) for r in cols])]).astype(np.int64)
    row_idx = np.concatenate(cols).astype(np.int64) if cols else np.empty(0, np.int64)
    n = len(row_idx)
    vals = rng.standard_normal(n) * np.exp(rng.uniform(-300, 300, size=n))
    if special and n > 12:
        vals[:12] = [0.0, -0.0, np.inf, -np.inf, np.nan, 1e-320, 5e-324, 1.7976931348623157e308, 1.0, -3.0,
                     0.1, 1e16]
    return LowerCscMatrix(col_ptr, row_idx, vals, dim)


@pytest.mark.parametrize("dim,threads", [(0, 1), (1, 1), (37, 3), (500, 4), (2000, 0)])
def test_export_byte_identical(tmp_path, dim, threads):
    rng = np.random.default_rng(dim + 7)
    m = random_lower_csc(rng, dim)
    path = tmp_path / "k.mtx"
    export_matrix_market(m, path, threads=threads)
    assert path.read_text() == oracle.export_matrix_market_text(m.col_ptr, m.row_idx, m.vals, m.dim)


def test_export_golden_matrix(tmp_path, golden):
    m = LowerCscMatrix(golden["m345_col_ptr"], golden["m345_row_idx"], golden["m345_vals"],
                       golden["m345_coords"].shape[0])
    path = tmp_path / "m345.mtx"
    export_matrix_market(m, path)
    assert path.read_bytes() == oracle.export_matrix_market_text(m.col_ptr, m.row_idx, m.vals, m.dim).encode()


def test_export_negative_nan_spelled_like_python(tmp_path):
    neg_nan = np.frombuffer(np.uint64(0xFFF8000000000000).tobytes(), dtype=np.float64)[0]
    m = LowerCscMatrix(np.array([0, 2], np.int64), np.array([0, 0], np.int64), np.array([neg_nan, 1.0]), 1)
    m = LowerCscMatrix(np.array([0, 1], np.int64), np.array([0], np.int64), np.array([neg_nan]), 1)
    path = tmp_path / "n.mtx"
    export_matrix_market(m, path)
    assert path.read_text() == oracle.export_matrix_market_text(m.col_ptr, m.row_idx, m.vals, m.dim)


def _native_parse(path):
    import ctypes

    from paper_1501_04784_b200 import _native as N

    n, nnz, err = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int64(0)
    rc = N.lib().hx_mm_read(str(path).encode(), ctypes.byref(n), ctypes.byref(nnz), None, None, None,
                            ctypes.byref(err))
    if rc != 0:
        return rc, None
    r = np.empty(nnz.value, np.int32)
    c = np.empty(nnz.value, np.int32)
    v = np.empty(nnz.value)
    rc = N.lib().hx_mm_read(str(path).encode(), ctypes.byref(n), ctypes.byref(nnz), r.ctypes.data if r.size else None,
                            c.ctypes.data if c.size else None, v.ctypes.data if v.size else None, ctypes.byref(err))
    return rc, (n.value, r, c, v, err.value)


def test_native_reader_parses_the_writer_output_exactly(tmp_path):
    rng = np.random.default_rng(3)
    m = random_lower_csc(rng, 300)
    path = tmp_path / "k.mtx"
    export_matrix_market(m, path)
    rc, out = _native_parse(path)
    assert rc == 0
    n, r, c, v, _ = out
    col_of = np.repeat(np.arange(m.dim), np.diff(m.col_ptr))
    assert n == m.dim and np.array_equal(r, m.row_idx) and np.array_equal(c, col_of)
    same = (v == m.vals) | (np.isnan(v) & np.isnan(m.vals))
    assert same.all() and np.array_equal(np.signbit(v[~np.isnan(v)]), np.signbit(m.vals[~np.isnan(m.vals)]))


@pytest.mark.parametrize("text,rc", [
    ("%%MatrixMarket matrix coordinate real symmetric\n3 3 1\n1 2 4.0\n", 2),       # above the diagonal
    ("%%MatrixMarket matrix coordinate real symmetric\n3 3 1\n4 1 4.0\n", 2),       # outside
    ("%%MatrixMarket matrix coordinate real symmetric\n3 3 1\n+2 1 4.0\n", 1),      # sign: reference rules
    ("%%MatrixMarket matrix coordinate real symmetric\r\n3 3 1\r\n2 1 4.0\r\n", 1),  # CRLF: reference rules
    ("%%MatrixMarket matrix coordinate real symmetric\n3 3 2\n2 1 4.0\n", 1),       # too few entries
    ("%%MatrixMarket matrix coordinate real symmetric\n% c\n3 3 1\n2 1 1_0.5\n", 1),  # underscore
    ("%%MatrixMarket matrix coordinate real symmetric\n% c\n3 3 1\n2 1 -1.5e-3\n", 0),
])
def test_native_reader_strict_subset(tmp_path, text, rc):
    path = tmp_path / "t.mtx"
    path.write_text(text)
    assert _native_parse(path)[0] == rc
