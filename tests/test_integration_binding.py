"""The reference-side binding of INTEGRATION.md (integration/hexfem_cuda_backend.py) as code that runs.

CPU: imported against the reference package itself (PYTHONPATH=/root/reference/pkg/src, in the
build container only; skipped elsewhere) -- the plugin subclasses hexfem's own ComputeBackend and
raises hexfem's own exception type, and the library it binds loads.  GPU: the same module (on a box
without hexfem it binds to this package's identical interface) drives integrate_all; KE bitwise the
oracle's, the degenerate-element report as element.py:237-244.
"""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
REF_SRC = Path("/root/reference/pkg/src")


@pytest.mark.skipif(not REF_SRC.is_dir(), reason="the reference package is only present in the build container")
def test_binding_imports_against_the_reference_package(tmp_path):
    code = (
        "import hexfem.integrate as hi, hexfem.errors as he\n"
        "import integration.hexfem_cuda_backend as b\n"
        "assert issubclass(b.CudaBackend, hi.ComputeBackend)\n"
        "assert b.DegenerateElementError is he.DegenerateElementError\n"
        "assert b._lib.hx_stiffness_batch.restype is not None\n"
        "be = b.CudaBackend(workers=2)\n"
        "with be:\n"
        "    assert be.workers == 2\n"
        "print('binding ok')\n")
    env = dict(os.environ, PYTHONPATH=f"{REF_SRC}:{ROOT}", PYTHONDONTWRITEBYTECODE="1",
               NUMBA_CACHE_DIR=str(tmp_path / "numba"))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, cwd=tmp_path,
                         timeout=600)
    assert out.returncode == 0 and "binding ok" in out.stdout, out.stderr[-2000:]


@pytest.mark.gpu
def test_binding_drives_integrate_all_bitwise():
    import oracle
    from integration.hexfem_cuda_backend import CudaBackend
    from paper_1501_04784_b200 import DegenerateElementError, Mesh, integrate_all, plan_batches, required_bytes
    from paper_1501_04784_b200.workloads import perturbed_mesh

    mesh = perturbed_mesh(12, seed=21)
    ke_ref, _, _, _, _, _ = oracle.stiffness_mesh(mesh.coords, mesh.connectivity, mesh.coefficient)
    with CudaBackend() as be:
        for mode in ("sequential", "overlapped"):
            plan = plan_batches(required_bytes(mesh.n_el), required_bytes(mesh.n_el) // 3 + 1, mesh.n_el)
            assert len(plan.ranges) > 1
            vals = integrate_all(mesh, be, plan, mode=mode)
            assert vals.values.tobytes() == ke_ref.tobytes()
        conn = mesh.connectivity.copy()
        conn[777] = conn[777][[4, 5, 6, 7, 0, 1, 2, 3]]  # inverted: degenerate
        with pytest.raises(DegenerateElementError) as ei:
            integrate_all(Mesh(mesh.coords, conn, mesh.coefficient), be,
                          plan_batches(required_bytes(mesh.n_el), required_bytes(mesh.n_el) // 3 + 1, mesh.n_el))
    assert ei.value.element_id == 777 and ei.value.gauss_point == 0 and ei.value.det < 0
