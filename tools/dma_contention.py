"""D2H DMA throughput alone vs while the GPU runs cold builds (is PCIe slowed by HBM-saturating kernels?)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_1501_04784_b200 import device as D  # noqa: E402
from paper_1501_04784_b200.pipeline import build_device  # noqa: E402
from paper_1501_04784_b200.workloads import make_workload  # noqa: E402

dm = D.DeviceMesh.from_host(make_workload("C4"))
n = 898_402_401
d = torch.empty(n, dtype=torch.float64, device="cuda")
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
cs = torch.cuda.Stream()
ke = torch.empty((dm.n_el, 36), dtype=torch.float64, device="cuda")
rows = torch.empty(36 * dm.n_el, dtype=torch.int32, device="cuda")
cols = torch.empty(36 * dm.n_el, dtype=torch.int32, device="cuda")
b = build_device(dm, ke=ke, rows=rows, cols=cols)
del b


def d2h_ms():
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(cs):
        a.record()
        h.copy_(d, non_blocking=True)
        e.record()
    return a, e


torch.cuda.synchronize()
a, e = d2h_ms()
torch.cuda.synchronize()
print(f"D2H 7.19 GB alone: {a.elapsed_time(e):.1f} ms", flush=True)
a, e = d2h_ms()
k = 0
while not e.query():
    b = build_device(dm, ke=ke, rows=rows, cols=cols)
    del b
    k += 1
torch.cuda.synchronize()
print(f"D2H 7.19 GB during {k} back-to-back cold builds: {a.elapsed_time(e):.1f} ms", flush=True)
# during the integration kernel only
a, e = d2h_ms()
k = 0
while not e.query():
    D.integrate_mesh(dm, ke=ke, rows=rows, cols=cols)
    torch.cuda.synchronize()
    k += 1
torch.cuda.synchronize()
print(f"D2H 7.19 GB during {k} integration kernels: {a.elapsed_time(e):.1f} ms", flush=True)
