"""Hexahedral meshes: the data model and the structured cube producer.

The mesh is the INPUT of the hot path (mesh generation / text I/O are out of scope);
this module provides only what the path needs: the ``Mesh`` container with the reference's
field names and dtypes (mesh.py:22-49), the structured generator with the reference's exact
numbering (mesh.py:73-98: node id i + j(nx+1) + k(nx+1)(ny+1), x-fastest elements, local
order [0, 1, 1+sx, sx, L, 1+L, 1+sx+L, sx+L]) and the validation rules (mesh.py:101-120).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import MeshValidationError

__all__ = ["Mesh", "StructuredGridSpec", "generate_cube_mesh", "validate_mesh"]


@dataclass(frozen=True)
class Mesh:
    """coords (n_nodes, 3) f64, connectivity (n_el, 8) i32, coefficient (n_el,) f64."""

    coords: np.ndarray
    connectivity: np.ndarray
    coefficient: np.ndarray

    @property
    def n_nodes(self) -> int:
        return self.coords.shape[0]

    @property
    def n_el(self) -> int:
        return self.connectivity.shape[0]


@dataclass(frozen=True)
class StructuredGridSpec:
    nx: int
    ny: int
    nz: int
    h: float = 1.0
    c0: float = 1.0

    def __post_init__(self):
        for name in ("nx", "ny", "nz"):
            v = getattr(self, name)
            if int(v) != v or v < 1:
                raise MeshValidationError(f"{name} must be a positive integer, got {v!r}")
        if not self.h > 0:
            raise MeshValidationError(f"edge length h must be positive, got {self.h!r}")
        if not self.c0 > 0:
            raise MeshValidationError(f"coefficient c0 must be positive, got {self.c0!r}")


def structured_connectivity(nx: int, ny: int, nz: int) -> np.ndarray:
    """(nx*ny*nz, 8) int32 connectivity of the structured box, built without int64 temporaries."""
    sx, sy = nx + 1, ny + 1
    layer = sx * sy
    if (nz + 1) * layer >= 2**31:
        raise MeshValidationError("mesh too large for int32 node ids")
    ex = np.arange(nx, dtype=np.int32)
    row = (np.arange(ny, dtype=np.int32) * sx)[:, None] + ex[None, :]          # (ny, nx)
    origin = (np.arange(nz, dtype=np.int32) * layer)[:, None, None] + row[None]  # (nz, ny, nx)
    local = np.array([0, 1, 1 + sx, sx, layer, 1 + layer, 1 + sx + layer, sx + layer], dtype=np.int32)
    conn = np.empty((nx * ny * nz, 8), dtype=np.int32)
    flat = origin.reshape(-1)
    for a in range(8):
        np.add(flat, local[a], out=conn[:, a])
    return conn


def generate_cube_mesh(spec: StructuredGridSpec) -> Mesh:
    """Structured box of nx*ny*nz axis-aligned hexes (same numbering as mesh.py:73-98)."""
    nx, ny, nz, h = spec.nx, spec.ny, spec.nz, spec.h
    sx, sy = nx + 1, ny + 1
    n_nodes = sx * sy * (nz + 1)
    coords = np.empty((n_nodes, 3), dtype=np.float64)
    c3 = coords.reshape(nz + 1, sy, sx, 3)
    c3[..., 0] = (np.arange(sx) * h)[None, None, :]
    c3[..., 1] = (np.arange(sy) * h)[None, :, None]
    c3[..., 2] = (np.arange(nz + 1) * h)[:, None, None]
    connectivity = structured_connectivity(nx, ny, nz)
    coefficient = np.full(nx * ny * nz, float(spec.c0))
    return Mesh(coords=coords, connectivity=connectivity, coefficient=coefficient)


def validate_mesh(mesh: Mesh) -> None:
    """Index bounds, per-element node distinctness, coefficient signs (mesh.py:101-120)."""
    conn = mesh.connectivity
    if conn.ndim != 2 or conn.shape[1] != 8:
        raise MeshValidationError(f"connectivity must be (n_el, 8), got {conn.shape}")
    if conn.size and (conn.min() < 0 or conn.max() >= mesh.n_nodes):
        bad = int(np.flatnonzero((conn < 0).any(axis=1) | (conn >= mesh.n_nodes).any(axis=1))[0])
        raise MeshValidationError(f"element {bad} references node outside [0, {mesh.n_nodes})")
    if conn.size:
        dup = (np.diff(np.sort(conn, axis=1), axis=1) == 0).any(axis=1)
        if dup.any():
            raise MeshValidationError(f"element {int(np.flatnonzero(dup)[0])} has repeated nodes")
    if mesh.coefficient.shape != (mesh.n_el,):
        raise MeshValidationError("coefficient array length must equal n_el")
    if mesh.coefficient.size and not (mesh.coefficient > 0).all():
        bad = int(np.flatnonzero(~(mesh.coefficient > 0))[0])
        raise MeshValidationError(f"element {bad} has non-positive coefficient")
