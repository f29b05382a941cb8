"""Time the integration kernel of alternate library builds (HEXFEM_B200_LIB) on one workload."""
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
    n = dm.n_el
    ke = torch.empty((n, 36), dtype=torch.float64, device="cuda")
    rows = torch.empty(36 * n, dtype=torch.int32, device="cuda")
    cols = torch.empty(36 * n, dtype=torch.int32, device="cuda")
    ts = []
    for it in range(8):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _, _, _, fail = D.integrate_mesh(dm, ke=ke, rows=rows, cols=cols, mode=os.environ.get("KE_MODE", "exact"))
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    D.raise_if_failed(fail)
    import hashlib
    h = hashlib.sha256(ke.cpu().numpy().tobytes()).hexdigest()[:16]
    ts = sorted(ts[2:])
    print(f"{os.environ.get('HEXFEM_B200_LIB', 'default')}: {wl} median {ts[len(ts)//2]:.3f} ms min {ts[0]:.3f} ms "
          f"-> {n / ts[0] / 1e6:.3f} G el/s  ke sha {h}", flush=True)
else:
    wl = sys.argv[1] if len(sys.argv) > 1 else "C3"
    libs = sorted((ROOT / "paper_1501_04784_b200" / "_lib" / "variants").glob("*.so"))
    for lib in [None, *libs]:
        env = dict(os.environ)
        if lib is not None:
            env["HEXFEM_B200_LIB"] = str(lib)
        subprocess.run([sys.executable, __file__, "--one", wl], env=env)
