"""Fused integrate+emit probe: kernel time of hx_integrate_emit per HX_FUSED_VARIANT against the
separate integration + emit kernels (CUDA events, same plan)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_1501_04784_b200 import device as D  # noqa: E402
from paper_1501_04784_b200.workloads import make_workload  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "C3"
dm = D.DeviceMesh.from_host(make_workload(wl))
n = dm.n_el
plan = D.plan_assembly(dm)
ke = torch.empty((n, 36), dtype=torch.float64, device="cuda")
rows = torch.empty(36 * n, dtype=torch.int32, device="cuda")
cols = torch.empty(36 * n, dtype=torch.int32, device="cuda")


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts)


def separate():
    D.integrate_mesh(dm, ke=ke, rows=rows, cols=cols)
    D.mesh_emit(plan, ke)


t_sep = timed(separate)
t_ke = timed(lambda: D.integrate_mesh(dm, ke=ke, rows=rows, cols=cols))
print(f"{wl} separate {t_sep:.3f} ms (integration {t_ke:.3f})", flush=True)
for v in (sys.argv[2:] or ["1", "2", "3", "0"]):
    os.environ["HX_FUSED_VARIANT"] = v
    t = timed(lambda: D.integrate_emit(dm, plan, ke, rows, cols))
    print(f"{wl} fused variant {v}: {t:.3f} ms", flush=True)
