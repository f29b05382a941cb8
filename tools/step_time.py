"""Median device time of build_device steps (overlapped and serial) on one workload."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_1501_04784_b200 import device as D  # noqa: E402
from paper_1501_04784_b200.pipeline import build_device  # noqa: E402
from paper_1501_04784_b200.workloads import make_workload  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "C3"
dm = D.DeviceMesh.from_host(make_workload(wl))
for overlap in (True, False):
    ts = []
    for it in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        r = build_device(dm, overlap=overlap)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
        del r
    ts = sorted(ts[2:])
    print(f"{wl} overlap={overlap} KE_BLOCKS_PER_SM={os.environ.get('HX_KE_BLOCKS_PER_SM', '-')}: "
          f"median {ts[len(ts)//2]:.3f} ms  min {ts[0]:.3f} ms -> {dm.n_el / ts[0] / 1e6:.3f} G el/s", flush=True)
