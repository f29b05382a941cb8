"""Local-to-global mapping and lower-triangular CSC assembly on the GPU.

Mirrors reference assemble.py:37-244 (TripletMatrix, LowerCscMatrix, map_local_to_global,
connectivity_index_arrays, build_triplet, triplet_to_csc, DirectAssembler, assemble_direct,
nnz_compression) with the same dtypes and the same bits:

* triplet_to_csc      -> hx_triplet_csc_* (stable radix sort + numpy's reduceat rule)
* DirectAssembler     -> values streamed into HBM in element order, then hx_mesh_csc_* (node
                         adjacency symbolic + deterministic column numeric)
* connectivity_index_arrays -> hx_connectivity_index_arrays
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import device as D
from .element import PACK_COLS, PACK_ROWS
from .integrate import LocalValuesBatch

__all__ = [
    "TripletMatrix", "LowerCscMatrix", "map_local_to_global", "connectivity_index_arrays", "build_triplet",
    "triplet_to_csc", "DirectAssembler", "assemble_direct", "nnz_compression", "csc_to_host", "dof_index_arrays",
    "assemble_dof",
]


@dataclass(frozen=True)
class TripletMatrix:
    rows: np.ndarray  # (36 * n_el,) int32
    cols: np.ndarray  # (36 * n_el,) int32
    vals: np.ndarray  # (36 * n_el,) float64
    dim: int

    @property
    def nnz(self) -> int:
        return self.rows.shape[0]


@dataclass(frozen=True)
class LowerCscMatrix:
    col_ptr: np.ndarray  # (dim + 1,) int64
    row_idx: np.ndarray  # (nnz,) int64, strictly increasing within a column
    vals: np.ndarray  # (nnz,) float64
    dim: int

    @property
    def nnz(self) -> int:
        return self.row_idx.shape[0]


def map_local_to_global(element_nodes, dofxn: int = 1):
    """Global (max, min) targets of one element's packed entries (assemble.py:65-83)."""
    nodes = np.asarray(element_nodes, dtype=np.int64)
    if nodes.shape != (8,):
        raise ValueError(f"expected 8 node ids, got shape {nodes.shape}")
    if dofxn < 1:
        raise ValueError(f"dofxn must be at least 1, got {dofxn}")
    ndof = 8 * dofxn
    dofs = (nodes[:, None] * dofxn + np.arange(dofxn)[None, :]).reshape(ndof)
    li, lj = np.tril_indices(ndof)
    gr, gc = dofs[li], dofs[lj]
    return np.stack([np.maximum(gr, gc), np.minimum(gr, gc)], axis=1)


def _device_conn(mesh):
    dev = D.require_device()
    conn = mesh.connectivity
    if isinstance(conn, torch.Tensor):
        return conn.to(dev)
    return torch.from_numpy(np.ascontiguousarray(conn, dtype=np.int32)).to(dev)


def connectivity_index_arrays(mesh, lo: int = 0, hi: int | None = None):
    """(rows, cols) int32 of elements [lo, hi) in packed order (assemble.py:86-93), on the GPU."""
    n_el = mesh.n_el
    hi = n_el if hi is None else min(hi, n_el)
    lo = max(0, lo)
    if hi <= lo:
        return np.empty(0, dtype=np.int32), np.empty(0, dtype=np.int32)
    rows, cols = D.connectivity_index_arrays(_device_conn(mesh), lo, hi)
    return rows.cpu().numpy(), cols.cpu().numpy()


def dof_index_arrays(mesh, dofxn: int = 1, lo: int = 0, hi: int | None = None):
    """map_local_to_global (assemble.py:65-83) of elements [lo, hi), element-major, on the GPU ->
    (rows, cols) int32 ((8 dofxn)(8 dofxn + 1)/2 per element, node-major dof blocks); dofxn = 1
    equals connectivity_index_arrays."""
    if dofxn < 1:
        raise ValueError(f"dofxn must be at least 1, got {dofxn}")
    n_el = mesh.n_el
    hi = n_el if hi is None else min(hi, n_el)
    lo = max(0, lo)
    if hi <= lo:
        return np.empty(0, dtype=np.int32), np.empty(0, dtype=np.int32)
    rows, cols = D.dof_index_arrays(_device_conn(mesh), mesh.n_nodes, dofxn, lo, hi)
    return rows.cpu().numpy(), cols.cpu().numpy()


def assemble_dof(mesh, values, dofxn: int) -> LowerCscMatrix:
    """Lower K (dim n_nodes * dofxn) of per-element packed matrices values (n_el, P) f64, P =
    (8 dofxn)(8 dofxn + 1)/2 in map_local_to_global order: build_triplet + triplet_to_csc
    (assemble.py:96-140) on the GPU, numpy's summation rule."""
    P = (8 * dofxn) * (8 * dofxn + 1) // 2
    values = np.ascontiguousarray(values, dtype=np.float64)
    if values.shape != (mesh.n_el, P):
        raise ValueError(f"values must be ({mesh.n_el}, {P}), got {values.shape}")
    conn = _device_conn(mesh)
    csc = D.assemble_dof(conn, torch.from_numpy(values).to(conn.device), mesh.n_nodes, dofxn)
    return csc_to_host(csc)


def build_triplet(mesh, values: LocalValuesBatch, rows=None, cols=None) -> TripletMatrix:
    """Entry 36e+p carries the p-th packed pair and value of element e (assemble.py:96-107)."""
    if values.values.shape != (mesh.n_el, 36):
        raise ValueError(f"values must be ({mesh.n_el}, 36), got {values.values.shape}")
    if rows is None or cols is None:
        rows, cols = connectivity_index_arrays(mesh)
    return TripletMatrix(rows=rows, cols=cols, vals=values.values.reshape(-1), dim=mesh.n_nodes)


def csc_to_host(csc: D.DeviceCsc) -> LowerCscMatrix:
    return LowerCscMatrix(col_ptr=csc.col_ptr.cpu().numpy(), row_idx=csc.row_idx.cpu().numpy(),
                          vals=csc.vals.cpu().numpy(), dim=csc.dim)


def triplet_to_csc(t: TripletMatrix) -> LowerCscMatrix:
    """Stable (col, row) sort + duplicate summation in entry order (assemble.py:110-149), on the GPU.
    Structural zeros stay stored; empty input gives an all-zero col_ptr."""
    dev = D.require_device()
    rows = torch.from_numpy(np.ascontiguousarray(t.rows, dtype=np.int32)).to(dev)
    cols = torch.from_numpy(np.ascontiguousarray(t.cols, dtype=np.int32)).to(dev)
    vals = torch.from_numpy(np.ascontiguousarray(t.vals, dtype=np.float64)).to(dev)
    return csc_to_host(D.triplet_csc(rows, cols, vals, int(t.dim)))


class DirectAssembler:
    """Connectivity-driven assembly that streams integrated values (assemble.py:152-230).

    Groups must arrive in ascending element order; each consumed group is copied into an HBM
    value buffer, and finish() runs the node-adjacency symbolic + column numeric kernels.  The
    index arrays are never materialised.
    """

    def __init__(self, mesh):
        self._mesh = mesh
        self.dim = mesh.n_nodes
        self._dev = D.require_device()
        self._conn = _device_conn(mesh)
        self._ke = torch.empty((mesh.n_el, 36), dtype=torch.float64, device=self._dev)
        self._next_element = 0

    def consume(self, element_range, values) -> None:
        lo, hi = element_range
        if lo != self._next_element:
            raise ValueError(f"groups must arrive in order; expected {self._next_element}, got {lo}")
        self._next_element = hi
        src = values if isinstance(values, torch.Tensor) else torch.from_numpy(
            np.ascontiguousarray(values, dtype=np.float64))
        self._ke[lo:hi].copy_(src.reshape(hi - lo, 36))

    def finish(self) -> LowerCscMatrix:
        if self._next_element != self._mesh.n_el:
            raise ValueError(f"only {self._next_element} of {self._mesh.n_el} elements were consumed")
        if self._mesh.n_el == 0:
            return LowerCscMatrix(col_ptr=np.zeros(self.dim + 1, dtype=np.int64),
                                  row_idx=np.empty(0, dtype=np.int64), vals=np.empty(0), dim=self.dim)
        return csc_to_host(D.mesh_csc([(self._conn, self._ke)], self.dim))


def assemble_direct(mesh, values: LocalValuesBatch) -> LowerCscMatrix:
    """Lower-triangular CSC straight from connectivity (assemble.py:233-239)."""
    if values.values.shape != (mesh.n_el, 36):
        raise ValueError(f"values must be ({mesh.n_el}, 36), got {values.values.shape}")
    assembler = DirectAssembler(mesh)
    assembler.consume((0, mesh.n_el), values.values)
    return assembler.finish()


def nnz_compression(t: TripletMatrix, m: LowerCscMatrix) -> float:
    return 1.0 - m.nnz / t.nnz
