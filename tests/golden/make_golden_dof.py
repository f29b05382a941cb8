"""Golden vectors for dofxn > 1, made by running the REFERENCE itself (build
container only):

    PYTHONPATH=/root/reference/pkg/src:. PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/nc \\
        python tests/golden/make_golden_dof.py

For a small permuted, perturbed mesh and dofxn in {2, 3}: the reference's map_local_to_global of
every element (assemble.py:65-83) stacked element-major, and the reference's triplet_to_csc
(assemble.py:110-140) of those triplets with seeded random values -> tests/golden/dof.npz.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

import hexfem  # noqa: E402  (the reference, via PYTHONPATH)
from hexfem import assemble as ref_assemble  # noqa: E402

from paper_1501_04784_b200.workloads import permuted_mesh, perturbed_mesh  # noqa: E402


def main():
    mesh = permuted_mesh(perturbed_mesh(3, seed=11), seed=12)
    out = {"conn": mesh.connectivity, "n_nodes": np.int64(mesh.n_nodes)}
    rng = np.random.default_rng(13)
    for d in (2, 3):
        pairs = np.concatenate([ref_assemble.map_local_to_global(g, dofxn=d) for g in mesh.connectivity])
        rows = pairs[:, 0].astype(np.int32)
        cols = pairs[:, 1].astype(np.int32)
        P = (8 * d) * (8 * d + 1) // 2
        vals = rng.standard_normal(mesh.n_el * P)
        csc = hexfem.triplet_to_csc(hexfem.TripletMatrix(rows=rows, cols=cols, vals=vals, dim=mesh.n_nodes * d))
        out.update({f"d{d}_pairs": pairs, f"d{d}_vals": vals, f"d{d}_col_ptr": csc.col_ptr,
                    f"d{d}_row_idx": csc.row_idx, f"d{d}_csc_vals": csc.vals})
    np.savez_compressed(HERE / "dof.npz", **out)
    print("wrote", HERE / "dof.npz", {k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
