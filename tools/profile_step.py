"""Profiling driver: one warm-up build + one profiled build of a workload (used under ncu)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_1501_04784_b200 import device as D  # noqa: E402
from paper_1501_04784_b200.pipeline import build_device  # noqa: E402
from paper_1501_04784_b200.workloads import make_workload  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "C3"
mode = sys.argv[2] if len(sys.argv) > 2 else "exact"
dm = D.DeviceMesh.from_host(make_workload(wl))
for _ in range(2):
    b = build_device(dm, mode=mode)
    torch.cuda.synchronize()
    del b
print("profiled", wl, mode)
