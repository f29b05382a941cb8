"""Generate the golden fixtures by running the REFERENCE package itself (build container only).

    PYTHONPATH=/root/reference/pkg/src:. PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/nc \
        python tests/golden/make_golden.py [--big | --add C5]

Writes
  tests/golden/small.npz     small arrays: dn table, element batches, meshes, CSC outputs, errors
  tests/golden/digests.json  SHA-256 of the reference outputs (KE, rows, cols, col_ptr, row_idx,
                             vals) for the BASELINE configs C1, C2 (and C3 / P64 with --big)

Inputs come from paper_1501_04784_b200.workloads (seeded numpy), so the GPU box regenerates the
identical inputs and compares its outputs against these digests bit for bit.  The reference is
imported read-only; nothing under /root/reference is written (bytecode and numba caches are
redirected).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

import hexfem  # noqa: E402  (the reference, via PYTHONPATH)
from hexfem import element as ref_element  # noqa: E402

from paper_1501_04784_b200.workloads import make_workload, perturbed_mesh, permuted_mesh  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ref_pipeline(mesh, workers=8):
    """Reference hot path, component by component (cli.py:112-120, triplet assembler)."""
    plan = hexfem.plan_batches(hexfem.required_bytes(mesh.n_el), 10**13, mesh.n_el)
    with hexfem.HostBackend(workers=workers) as backend:
        batch = hexfem.integrate_all(hexfem.Mesh(mesh.coords, mesh.connectivity, mesh.coefficient), backend, plan)
    ref_mesh = hexfem.Mesh(mesh.coords, mesh.connectivity, mesh.coefficient)
    rows, cols = hexfem.connectivity_index_arrays(ref_mesh)
    csc = hexfem.triplet_to_csc(hexfem.build_triplet(ref_mesh, batch, rows=rows, cols=cols))
    return batch.values, rows, cols, csc


def digests_of(name, mesh):
    t0 = time.time()
    values, rows, cols, csc = ref_pipeline(mesh)
    d = {
        "n_el": int(mesh.n_el), "n_nodes": int(mesh.n_nodes), "nnz": int(csc.nnz),
        "ke": sha(values), "rows": sha(rows), "cols": sha(cols),
        "col_ptr": sha(csc.col_ptr), "row_idx": sha(csc.row_idx), "vals": sha(csc.vals),
        "ke_sum": float(values.sum()), "vals_absmax": float(np.abs(csc.vals).max()),
        "seconds_reference": round(time.time() - t0, 2),
    }
    print(name, d, flush=True)
    return d


def main(big: bool):
    out = {}
    rng = np.random.default_rng(20240517)
    corners = (ref_element.NODE_NATURAL_COORDS + 1.0) / 2.0

    out["dn_table"] = np.array(ref_element._DN_AT_GP)
    out["pack_rows"] = np.array(ref_element.PACK_ROWS)
    out["pack_cols"] = np.array(ref_element.PACK_COLS)

    # element batches: unit cube, scaled cubes, random valid hexes (oracles.py:121-124 style),
    # random parallelepipeds and large/small coordinate magnitudes
    hexes = [corners, corners * 0.5, corners * 2.0, corners * 1e-3 + 7.0, corners * 1e4]
    for _ in range(200):
        hexes.append(corners + rng.uniform(-0.15, 0.15, size=(8, 3)))
    for _ in range(40):
        while True:
            A = rng.uniform(-1.0, 1.0, size=(3, 3)) + 2.0 * np.eye(3)
            if np.linalg.det(A) > 0.5:
                break
        hexes.append(ref_element.NODE_NATURAL_COORDS @ A.T + rng.uniform(-5, 5, size=3))
    batch_coords = np.stack(hexes)
    batch_coeff = rng.uniform(0.5, 2.0, size=batch_coords.shape[0])
    batch_coeff[:5] = 1.0
    out["batch_coords"] = batch_coords
    out["batch_coeff"] = batch_coeff
    out["batch_ke"] = hexfem.stiffness_batch(batch_coords, batch_coeff)

    # small meshes through the full reference pipeline
    meshes = {
        "m345": perturbed_mesh(3, seed=11),
        "aniso": hexfem.generate_cube_mesh(hexfem.StructuredGridSpec(4, 3, 5, h=0.3, c0=1.7)),
        "perm5": permuted_mesh(perturbed_mesh(5, seed=3), seed=9),
        "unit6": make_workload("C1", n=6),
    }
    for name, m in meshes.items():
        values, rows, cols, csc = ref_pipeline(m)
        out[f"{name}_coords"] = m.coords
        out[f"{name}_conn"] = m.connectivity
        out[f"{name}_coeff"] = m.coefficient
        out[f"{name}_ke"] = values
        out[f"{name}_rows"] = rows
        out[f"{name}_cols"] = cols
        out[f"{name}_col_ptr"] = csc.col_ptr
        out[f"{name}_row_idx"] = csc.row_idx
        out[f"{name}_vals"] = csc.vals
        direct = hexfem.assemble_direct(hexfem.Mesh(m.coords, m.connectivity, m.coefficient),
                                        hexfem.LocalValuesBatch(values))
        assert np.array_equal(direct.vals, csc.vals) and np.array_equal(direct.row_idx, csc.row_idx)

    # degenerate elements: flipped faces (test_integrate.py:183-208 style)
    base = hexfem.generate_cube_mesh(hexfem.StructuredGridSpec(3, 3, 3))
    conn = base.connectivity.copy()
    flip = [4, 5, 6, 7, 0, 1, 2, 3]
    conn[20] = conn[20][flip]
    conn[7] = conn[7][flip]
    out["degen_conn"] = conn
    out["degen_coords"] = base.coords
    try:
        hexfem.stiffness_batch(base.coords[conn], base.coefficient)
        raise AssertionError("expected a degenerate element")
    except hexfem.DegenerateElementError as exc:
        out["degen_expect"] = np.array([exc.element_id, exc.gauss_point])
        out["degen_det"] = np.array([exc.det])

    # generic triplets with long duplicate runs (exercise numpy's pairwise rule, runs up to 300)
    n_t, dim = 6000, 12
    r = rng.integers(0, dim, size=n_t).astype(np.int32)
    c = rng.integers(0, dim, size=n_t).astype(np.int32)
    rows_t, cols_t = np.maximum(r, c), np.minimum(r, c)
    vals_t = rng.standard_normal(n_t) * np.exp(rng.uniform(-20, 20, size=n_t))
    t = hexfem.TripletMatrix(rows=rows_t, cols=cols_t, vals=vals_t, dim=dim)
    csc = hexfem.triplet_to_csc(t)
    out.update(trip_rows=rows_t, trip_cols=cols_t, trip_vals=vals_t, trip_dim=np.array([dim]),
               trip_col_ptr=csc.col_ptr, trip_row_idx=csc.row_idx, trip_out=csc.vals)

    np.savez_compressed(HERE / "small.npz", **out)

    digests = {"numpy": np.__version__, "numba": __import__("numba").__version__,
               "reference": "hexfem " + hexfem.__version__, "configs": {}}
    digests["configs"]["C1"] = digests_of("C1", make_workload("C1"))
    digests["configs"]["C2"] = digests_of("C2", make_workload("C2"))
    if big:
        digests["configs"]["P64"] = digests_of("P64", permuted_mesh(perturbed_mesh(64, seed=0), seed=5))
        digests["configs"]["C3"] = digests_of("C3", make_workload("C3"))
    (HERE / "digests.json").write_text(json.dumps(digests, indent=1) + "\n")


def add_config(name: str):
    """Append one BASELINE config's reference digests to digests.json (C5: 16.8M elements,
    permuted numbering -- about 7 minutes and ~40 GB of RAM for the reference's lexsort)."""
    path = HERE / "digests.json"
    digests = json.loads(path.read_text())
    digests["configs"][name] = digests_of(name, make_workload(name))
    path.write_text(json.dumps(digests, indent=1) + "\n")


if __name__ == "__main__":
    assert os.environ.get("PYTHONDONTWRITEBYTECODE"), "set PYTHONDONTWRITEBYTECODE=1 (reference is read-only)"
    if "--add" in sys.argv:
        add_config(sys.argv[sys.argv.index("--add") + 1])
    else:
        main(big="--big" in sys.argv)
