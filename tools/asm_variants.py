"""Time the mesh-path assembly (hx_mesh_csc_build) of alternate library builds (HEXFEM_B200_LIB)."""
import hashlib
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
if len(sys.argv) > 2 and sys.argv[1] == "--one":
    sys.path.insert(0, str(ROOT))
    import torch
    from paper_1501_04784_b200 import device as D
    from paper_1501_04784_b200.workloads import make_workload
    wl = sys.argv[2]
    dm = D.DeviceMesh.from_host(make_workload(wl))
    ke, _, _, fail = D.integrate_mesh(dm, with_index=False)
    D.raise_if_failed(fail)
    ts = []
    for it in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        csc = D.mesh_csc([(dm.conn, ke)], dm.n_nodes, order=dm.assembly_order())
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    h = hashlib.sha256(csc.vals.cpu().numpy().tobytes()).hexdigest()[:16]
    ts = sorted(ts[2:])
    print(f"{Path(os.environ.get('HEXFEM_B200_LIB', 'default')).name}: {wl} assembly median {ts[len(ts)//2]:.3f} ms "
          f"min {ts[0]:.3f} ms  vals sha {h}", flush=True)
else:
    wl = sys.argv[1] if len(sys.argv) > 1 else "C3"
    libs = sorted((ROOT / "paper_1501_04784_b200" / "_lib" / "variants").glob("*.so"))
    for lib in [None, *libs]:
        env = dict(os.environ)
        if lib is not None:
            env["HEXFEM_B200_LIB"] = str(lib)
        subprocess.run([sys.executable, __file__, "--one", wl], env=env)
