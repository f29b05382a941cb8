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
