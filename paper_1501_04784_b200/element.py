"""Element-level API: reference constants and the batched stiffness kernel on the GPU.

Mirrors reference element.py:24-245 for the hot-path symbols (NODE_NATURAL_COORDS, PACK_ROWS,
PACK_COLS, stiffness_batch, local_stiffness, pack/unpack_lower, set_worker_threads).  The
element math runs in libhexfem_b200.so; numpy arrays in, numpy arrays out.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import device as D
from ._native import lib as _lib

__all__ = [
    "NODE_NATURAL_COORDS", "PACK_ROWS", "PACK_COLS", "ElementGeometry", "PackedLowerStiffness",
    "stiffness_batch", "local_stiffness", "pack_lower", "unpack_lower", "set_worker_threads",
    "element_geometry",
]

# element.py:45-56
NODE_NATURAL_COORDS = np.array(
    [(-1.0, -1.0, -1.0), (1.0, -1.0, -1.0), (1.0, 1.0, -1.0), (-1.0, 1.0, -1.0),
     (-1.0, -1.0, 1.0), (1.0, -1.0, 1.0), (1.0, 1.0, 1.0), (-1.0, 1.0, 1.0)])
NODE_NATURAL_COORDS.setflags(write=False)
# element.py:59-62
PACK_ROWS, PACK_COLS = np.tril_indices(8)
PACK_ROWS.setflags(write=False)
PACK_COLS.setflags(write=False)


@dataclass(frozen=True)
class ElementGeometry:
    node_coords: np.ndarray  # (8, 3)

    def __post_init__(self):
        pts = np.asarray(self.node_coords, dtype=np.float64)
        if pts.shape != (8, 3):
            raise ValueError(f"node_coords must be (8, 3), got {pts.shape}")
        if np.unique(pts, axis=0).shape[0] != 8:
            raise ValueError("element nodes must be 8 distinct points")
        object.__setattr__(self, "node_coords", pts)


@dataclass(frozen=True)
class PackedLowerStiffness:
    values: np.ndarray  # (36,)

    def unpack(self) -> np.ndarray:
        return unpack_lower(self.values)


def pack_lower(matrix: np.ndarray) -> np.ndarray:
    m = np.asarray(matrix)
    if m.shape != (8, 8):
        raise ValueError(f"expected an 8x8 matrix, got {m.shape}")
    return m[PACK_ROWS, PACK_COLS].copy()


def unpack_lower(values: np.ndarray) -> np.ndarray:
    v = np.asarray(values, dtype=np.float64)
    if v.shape != (36,):
        raise ValueError(f"expected 36 packed values, got shape {v.shape}")
    full = np.zeros((8, 8))
    full[PACK_ROWS, PACK_COLS] = v
    full[PACK_COLS, PACK_ROWS] = v
    return full


def set_worker_threads(workers: int) -> int:
    """Host-thread count of the reference kernel (element.py:202-210).  On the GPU the
    parallelism is the grid; the value is accepted as a hint and does not change results."""
    return max(1, int(workers))


def stiffness_batch(coords, coeff, element_offset: int = 0, out=None, mode: str = "exact"):
    """Element stiffness for a batch: coords (n, 8, 3), coeff (n,) -> (n, 36) (element.py:213-245).

    Runs the sm_100a kernel; raises DegenerateElementError for the lowest failing element
    (labelled element_offset + index).  ``out`` (host, float64 (n, 36)) is filled in place.
    """
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    coeff = np.ascontiguousarray(coeff, dtype=np.float64)
    n = coords.shape[0]
    if coords.shape != (n, 8, 3) or coeff.shape != (n,):
        raise ValueError(f"bad batch shapes {coords.shape}, {coeff.shape}")
    if out is None:
        out = np.empty((n, 36))
    elif out.shape != (n, 36) or out.dtype != np.float64:
        raise ValueError(f"out must be float64 ({n}, 36), got {out.dtype} {out.shape}")
    if n == 0:
        return out
    dev = D.require_device()
    d_out, fail = D.stiffness_batch(torch.from_numpy(coords).to(dev), torch.from_numpy(coeff).to(dev), mode=mode)
    host = d_out.cpu()
    D.raise_if_failed(fail, element_offset)
    out[...] = host.numpy()
    return out


def local_stiffness(geom: ElementGeometry, c: float) -> PackedLowerStiffness:
    """One element's packed stiffness (element.py:180-193); rejects c <= 0 like the reference."""
    if not c > 0:
        raise ValueError(f"coefficient must be positive, got {c!r}")
    values = stiffness_batch(np.asarray(geom.node_coords)[None, :, :], np.array([float(c)]))
    return PackedLowerStiffness(values=values[0])


def element_geometry(mesh, e: int) -> ElementGeometry:
    return ElementGeometry(node_coords=mesh.coords[mesh.connectivity[e]])


def compiled_dn_table() -> np.ndarray:
    """_DN_AT_GP (8, 3, 8) exactly as compiled into the kernels (host introspection)."""
    out = np.empty(192)
    _lib().hx_dn_table(out.ctypes.data_as(__import__("ctypes").c_void_p))
    return out.reshape(8, 3, 8)
