"""Assembly pass kernel times (pattern + scan + emit, cold build) per library variant
(HEXFEM_B200_LIB), CUDA events around build_device minus the integration kernel."""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
if len(sys.argv) > 2 and sys.argv[1] == "--one":
    sys.path.insert(0, str(ROOT))
    import torch
    from paper_1501_04784_b200 import device as D
    from paper_1501_04784_b200.pipeline import build_device
    from paper_1501_04784_b200.workloads import make_workload
    dm = D.DeviceMesh.from_host(make_workload(sys.argv[2]))
    ts = []
    for it in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        bd = build_device(dm)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
        del bd
    ts = sorted(ts[2:])
    print(f"{Path(os.environ.get('HEXFEM_B200_LIB', 'default')).name}: {sys.argv[2]} cold build median {ts[len(ts)//2]:.3f} ms "
          f"min {ts[0]:.3f} ms", flush=True)
else:
    wl = sys.argv[1] if len(sys.argv) > 1 else "C3"
    libs = sorted((ROOT / "paper_1501_04784_b200" / "_lib" / "variants").glob("*.so"))
    for lib in [None, *libs]:
        env = dict(os.environ)
        if lib is not None:
            env["HEXFEM_B200_LIB"] = str(lib)
        subprocess.run([sys.executable, __file__, "--one", wl], env=env)
