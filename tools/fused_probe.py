"""Fused integrate+emit probe: kernel time of hx_integrate_emit against the separate integration +
emit kernels (CUDA events, same plan).  Round-2 measurements, C3 / C4 ms: separate
4.24 / 34.99; fused 21.7 / 152+ ; completion counters + fences only (no emit) 3.34 / 26.6; every
emit after the warp's own quads 6.37 / 58.3 (the emit on 16 x 128-register warps per SM runs 3x
slower than the standalone kernel's 48 x 40-register warps)."""
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
t = timed(lambda: D.integrate_emit(dm, plan, ke, rows, cols))
print(f"{wl} fused {t:.3f} ms", flush=True)
