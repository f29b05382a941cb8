"""CPU restatement of the reference hot path -- TEST INFRASTRUCTURE ONLY (the checker).

Every function cites the reference file:line it restates (paths under
/root/reference/pkg/src/hexfem/).  The element kernel lives in ``hx_oracle.c`` (plain C,
``-ffp-contract=off``); the assembly is numpy, the same library calls the reference uses,
so the summation rule (``np.add.reduceat``) is numpy's own.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "_build" / "libhxoracle.so"
_lib = None

# element.py:59-62 -- row-major lower triangle incl. diagonal.
PACK_ROWS, PACK_COLS = np.tril_indices(8)


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists():
        subprocess.run(["make", "-C", str(_HERE)], check=True, capture_output=True)
    lib = ctypes.CDLL(str(_LIB_PATH))
    P = ctypes.c_void_p
    lib.hxo_dn_table.argtypes = [P]
    lib.hxo_dn_table.restype = None
    lib.hxo_stiffness_batch.argtypes = [P, P, ctypes.c_int64, P, P, P, ctypes.c_int]
    lib.hxo_stiffness_batch.restype = ctypes.c_int64
    lib.hxo_stiffness_mesh.argtypes = [P, P, P, ctypes.c_int64, ctypes.c_int64, P, P, P, P, P,
                                       ctypes.c_int]
    lib.hxo_stiffness_mesh.restype = ctypes.c_int64
    _lib = lib
    return lib


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


def _threads(threads):
    return int(threads) if threads else (os.cpu_count() or 1)


def dn_table() -> np.ndarray:
    """_DN_AT_GP (8, 3, 8): element.py:104-113 evaluated at the points of element.py:116-124."""
    out = np.empty((8, 3, 8))
    _load().hxo_dn_table(_ptr(out))
    return out


def stiffness_batch(coords, coeff, threads=None):
    """element.py:213-297 on pre-gathered coords (n, 8, 3).

    Returns ``(values (n, 36), first_failing_index or -1, fail_gp (n,), fail_det (n,))``.
    """
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    coeff = np.ascontiguousarray(coeff, dtype=np.float64)
    n = coords.shape[0]
    assert coords.shape == (n, 8, 3) and coeff.shape == (n,)
    out = np.empty((n, 36))
    fail_gp = np.empty(n, dtype=np.int32)
    fail_det = np.empty(n)
    first = _load().hxo_stiffness_batch(_ptr(coords), _ptr(coeff), n, _ptr(out), _ptr(fail_gp),
                                        _ptr(fail_det), _threads(threads))
    return out, int(first), fail_gp, fail_det


def stiffness_mesh(coords, conn, coeff, lo=0, hi=None, with_index=True, threads=None):
    """integrate_all's gather + kernel (integrate.py:146-149, element.py:248-297) fused with
    connectivity_index_arrays (assemble.py:86-93), for elements [lo, hi).

    Returns ``(values, rows, cols, first_failing_global_id or -1, fail_gp, fail_det)``.
    """
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    conn = np.ascontiguousarray(conn, dtype=np.int32)
    coeff = np.ascontiguousarray(coeff, dtype=np.float64)
    hi = conn.shape[0] if hi is None else hi
    n = hi - lo
    out = np.empty((n, 36))
    rows = np.empty(36 * n, dtype=np.int32) if with_index else None
    cols = np.empty(36 * n, dtype=np.int32) if with_index else None
    fail_gp = np.empty(n, dtype=np.int32)
    fail_det = np.empty(n)
    first = _load().hxo_stiffness_mesh(_ptr(coords), _ptr(conn), _ptr(coeff), lo, hi, _ptr(out),
                                       _ptr(rows), _ptr(cols), _ptr(fail_gp), _ptr(fail_det),
                                       _threads(threads))
    return out, rows, cols, int(first), fail_gp, fail_det


def connectivity_index_arrays(conn, lo=0, hi=None):
    """assemble.py:86-93: rows = max, cols = min over the packed pairs, element-major, int32."""
    c = np.asarray(conn)[lo:hi].astype(np.int32, copy=False)
    gr = c[:, PACK_ROWS]
    gc = c[:, PACK_COLS]
    return np.maximum(gr, gc).reshape(-1), np.minimum(gr, gc).reshape(-1)


def dof_index_arrays(conn, dofxn, lo=0, hi=None):
    """assemble.py:65-83 map_local_to_global applied to every element of [lo, hi), element-major:
    dofs = node * dofxn + k (node-major blocks), pairs in np.tril_indices(8 dofxn) order, swapped to
    (max, min); int32 like connectivity_index_arrays (assemble.py:86-93)."""
    c = np.asarray(conn)[lo:hi].astype(np.int64)
    ndof = 8 * dofxn
    dofs = (c[:, :, None] * dofxn + np.arange(dofxn)[None, None, :]).reshape(c.shape[0], ndof)
    li, lj = np.tril_indices(ndof)
    gr, gc = dofs[:, li], dofs[:, lj]
    return (np.maximum(gr, gc).reshape(-1).astype(np.int32), np.minimum(gr, gc).reshape(-1).astype(np.int32))


class OracleValidationError(ValueError):
    """Raised where the reference raises MeshValidationError (assemble.py:143-149)."""


def triplet_to_csc(rows, cols, vals, dim):
    """assemble.py:110-149: validate, stable lexsort by (col, row), add.reduceat, bincount+cumsum.

    Returns ``(col_ptr int64 (dim+1), row_idx int64 (nnz), vals float64 (nnz))``.
    """
    rows = np.asarray(rows)
    cols = np.asarray(cols)
    vals = np.asarray(vals, dtype=np.float64)
    if rows.size:
        if rows.min() < 0 or rows.max() >= dim or cols.min() < 0:
            raise OracleValidationError(f"triplet index outside [0, {dim})")
        if (rows < cols).any():
            raise OracleValidationError("triplet entry above the diagonal")
    if rows.size == 0:
        return np.zeros(dim + 1, dtype=np.int64), np.empty(0, dtype=np.int64), np.empty(0)
    order = np.lexsort((rows, cols))
    r = rows[order]
    c = cols[order]
    v = vals[order]
    is_start = np.empty(r.shape[0], dtype=bool)
    is_start[0] = True
    is_start[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
    starts = np.flatnonzero(is_start)
    summed = np.add.reduceat(v, starts)
    row_idx = r[starts].astype(np.int64)
    col_counts = np.bincount(c[starts], minlength=dim)
    col_ptr = np.zeros(dim + 1, dtype=np.int64)
    np.cumsum(col_counts, out=col_ptr[1:])
    return col_ptr, row_idx, summed


def triplet_to_csc_columns(rows, cols, vals, col_lo, col_hi):
    """assemble.py:110-140 on a column window: the triplets whose column lies in [col_lo, col_hi)
    (given in the reference's element-major order), the same stable lexsort by (col, row) and
    add.reduceat; col_ptr covers only the window (starts at 0).  Equal to the window of the
    full triplet_to_csc because the stable sort keeps every column's triplets in input order."""
    rows = np.asarray(rows)
    cols = np.asarray(cols)
    vals = np.asarray(vals, dtype=np.float64)
    n = col_hi - col_lo
    if rows.size == 0:
        return np.zeros(n + 1, dtype=np.int64), np.empty(0, dtype=np.int64), np.empty(0)
    assert cols.min() >= col_lo and cols.max() < col_hi and (rows >= cols).all()
    order = np.lexsort((rows, cols))
    r = rows[order]
    c = cols[order]
    v = vals[order]
    is_start = np.empty(r.shape[0], dtype=bool)
    is_start[0] = True
    is_start[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
    starts = np.flatnonzero(is_start)
    summed = np.add.reduceat(v, starts)
    col_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(c[starts] - col_lo, minlength=n), out=col_ptr[1:])
    return col_ptr, r[starts].astype(np.int64), summed


def pairwise_sum(a):
    """Pure-Python model of numpy's pairwise summation (numpy/_core/src/umath/loops_utils.h.src
    ``@TYPE@_pairwise_sum``), used to pin the rule the GPU numeric phase implements."""
    n = len(a)
    if n < 8:
        res = -0.0
        for x in a:
            res = res + float(x)
        return res
    if n <= 128:
        r = [float(x) for x in a[:8]]
        i = 8
        while i < n - (n % 8):
            for j in range(8):
                r[j] = r[j] + float(a[i + j])
            i += 8
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            res = res + float(a[i])
            i += 1
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return pairwise_sum(a[:n2]) + pairwise_sum(a[n2:])


def reduceat_model(run):
    """np.add.reduceat on one run: ``v0 + pairwise(v[1:])``."""
    if len(run) == 1:
        return float(run[0])
    return float(run[0]) + pairwise_sum(run[1:])


def export_matrix_market_text(col_ptr, row_idx, vals, dim) -> str:
    """sparseio.py:73-87 restated: the reference writer's exact text."""
    out = ["%%MatrixMarket matrix coordinate real symmetric", f"{dim} {dim} {len(row_idx)}"]
    for col in range(dim):
        for k in range(col_ptr[col], col_ptr[col + 1]):
            out.append(f"{row_idx[k] + 1} {col + 1} {vals[k]:.17g}")
    return "\n".join(out) + "\n"
