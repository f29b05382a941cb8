"""Shared test helpers."""

import hashlib

import numpy as np

from paper_1501_04784_b200.mesh import Mesh

SMALL_MESHES = ("m345", "aniso", "perm5", "unit6")


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def bits_equal(a, b) -> bool:
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    if a.shape != b.shape or a.dtype != b.dtype:
        return False
    return a.tobytes() == b.tobytes()


def golden_mesh(golden, name) -> Mesh:
    return Mesh(coords=golden[f"{name}_coords"], connectivity=golden[f"{name}_conn"],
                coefficient=golden[f"{name}_coeff"])
