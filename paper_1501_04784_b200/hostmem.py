"""Page-locked host memory for the host <-> HBM copies of the path.

A mesh whose arrays live in pinned memory is copied to the GPU by DMA at PCIe rate, asynchronously,
so ``run_build`` overlaps the connectivity upload with the integration kernel; pageable arrays
(plain numpy) are staged by the driver and the copy blocks the host.  Results come back into pinned
arrays from torch's caching host allocator (recycled once the caller drops the previous result).
"""

from __future__ import annotations

import numpy as np
import torch

from .mesh import Mesh

__all__ = ["pinned_empty", "pinned_copy", "pinned_mesh", "is_pinned"]

_TORCH = {np.dtype(np.float64): torch.float64, np.dtype(np.int32): torch.int32, np.dtype(np.int64): torch.int64,
          np.dtype(np.uint8): torch.uint8}


def pinned_empty(shape, dtype) -> np.ndarray:
    """numpy view of a page-locked host buffer (kept alive by the array)."""
    return torch.empty(tuple(shape), dtype=_TORCH[np.dtype(dtype)], pin_memory=True).numpy()


def pinned_copy(a: np.ndarray) -> np.ndarray:
    out = pinned_empty(a.shape, a.dtype)
    np.copyto(out, a)
    return out


def is_pinned(a) -> bool:
    t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
    try:
        return bool(t.is_pinned())
    except RuntimeError:  # no CUDA runtime
        return False


def pinned_mesh(mesh) -> Mesh:
    """The same mesh with coords / connectivity / coefficient in pinned host memory (reference
    dtypes: f64, int32, f64)."""
    return Mesh(coords=pinned_copy(np.ascontiguousarray(mesh.coords, dtype=np.float64)),
                connectivity=pinned_copy(np.ascontiguousarray(mesh.connectivity, dtype=np.int32)),
                coefficient=pinned_copy(np.ascontiguousarray(mesh.coefficient, dtype=np.float64)))
