"""Synthetic inputs of the BASELINE.json configurations; all seeded.

  C1  20^3 unit cube, c0 = 1                                   (8,000 elements)
  C2  100^3, coords + U(-0.15, 0.15) per component, c ~ U(0.5, 2), default_rng(0)
  C3  200^3 unit cube, c ~ U(0.5, 2), default_rng(2)           (8M elements)
  C4  400^3 as C3                                             (64M elements)
  C5  256^3 perturbed as C2, node numbering permuted by default_rng(5).permutation

The perturbation mirrors the reference's random_valid_hexahedron distortion (oracles.py:121-124);
the coefficient range mirrors test_acceptance.py:66-73.
"""

from __future__ import annotations

import numpy as np

from .mesh import Mesh, StructuredGridSpec, generate_cube_mesh

__all__ = ["WORKLOADS", "make_workload", "perturbed_mesh", "permuted_mesh", "random_coefficient_mesh"]

WORKLOADS = {
    "C1": dict(n=20, desc="hex8 Poisson 20^3 unit cube (8k elements), c0=1"),
    "C2": dict(n=100, desc="hex8 100^3 (1M elements), perturbed coords, random conductivity"),
    "C3": dict(n=200, desc="hex8 200^3 (8M elements), full pipeline"),
    "C4": dict(n=400, desc="hex8 400^3 (64M elements)"),
    "C5": dict(n=256, desc="hex8 256^3, randomly permuted node numbering, perturbed coords"),
}


def perturbed_mesh(n: int, seed: int = 0, distortion: float = 0.15) -> Mesh:
    base = generate_cube_mesh(StructuredGridSpec(n, n, n))
    rng = np.random.default_rng(seed)
    coords = base.coords + rng.uniform(-distortion, distortion, size=base.coords.shape)
    coefficient = rng.uniform(0.5, 2.0, size=base.n_el)
    return Mesh(coords=coords, connectivity=base.connectivity, coefficient=coefficient)


def random_coefficient_mesh(n: int, seed: int) -> Mesh:
    base = generate_cube_mesh(StructuredGridSpec(n, n, n))
    rng = np.random.default_rng(seed)
    return Mesh(coords=base.coords, connectivity=base.connectivity,
                coefficient=rng.uniform(0.5, 2.0, size=base.n_el))


def permuted_mesh(mesh: Mesh, seed: int = 5) -> Mesh:
    """Relabel nodes with a random permutation p: coords_new[p] = coords, conn_new = p[conn]."""
    p = np.random.default_rng(seed).permutation(mesh.n_nodes)
    coords = np.empty_like(mesh.coords)
    coords[p] = mesh.coords
    conn = p.astype(np.int32)[mesh.connectivity]
    return Mesh(coords=coords, connectivity=conn, coefficient=mesh.coefficient)


def make_workload(name: str, n: int | None = None) -> Mesh:
    """Mesh of configuration ``name`` (C1..C5); ``n`` overrides the cube side (tests)."""
    name = name.upper()
    side = WORKLOADS[name]["n"] if n is None else n
    if name == "C1":
        return generate_cube_mesh(StructuredGridSpec(side, side, side))
    if name == "C2":
        return perturbed_mesh(side, seed=0)
    if name in ("C3", "C4"):
        return random_coefficient_mesh(side, seed=2)
    if name == "C5":
        return permuted_mesh(perturbed_mesh(side, seed=0), seed=5)
    raise KeyError(name)
