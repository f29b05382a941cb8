"""Fast-mode integration kernel time (HX_FAST_DMMA toggles the tensor-core variant) on one workload."""
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
ke = torch.empty((n, 36), dtype=torch.float64, device="cuda")
rows = torch.empty(36 * n, dtype=torch.int32, device="cuda")
cols = torch.empty(36 * n, dtype=torch.int32, device="cuda")
ts = []
for it in range(8):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    _, _, _, fail = D.integrate_mesh(dm, ke=ke, rows=rows, cols=cols, mode="fast")
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
D.raise_if_failed(fail)
ts = sorted(ts[2:])
ref, _, _, _ = D.integrate_mesh(dm, mode="exact")
err = ((ke - ref).abs().max(dim=1).values / ref.abs().max(dim=1).values).max().item()
print(f"{wl} HX_FAST_DMMA={os.environ.get('HX_FAST_DMMA', '1')}: fast KE median {ts[len(ts)//2]:.3f} ms "
      f"-> {n / ts[0] / 1e6:.3f} G el/s; max row-scaled |dKE| vs exact {err:.2e}", flush=True)
