"""Per-step timeline of the pipelined e2e (C4): host submit / result times and the copy stream's
D2H windows, to see where a step's time goes beyond the PCIe transfer."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1501_04784_b200 import device as D  # noqa: E402
from paper_1501_04784_b200.pipeline import build_device  # noqa: E402
from paper_1501_04784_b200.transfer import CscHostTransfer  # noqa: E402
from paper_1501_04784_b200.workloads import make_workload  # noqa: E402

mesh = make_workload(sys.argv[1] if len(sys.argv) > 1 else "C4")
dev = torch.device("cuda")


def pinned(a):
    t = torch.empty(a.shape, dtype={np.float64: torch.float64, np.int32: torch.int32}[a.dtype.type], pin_memory=True)
    t.numpy()[...] = a
    return t


h = [pinned(mesh.coords), pinned(mesh.connectivity), pinned(mesh.coefficient)]
b0 = build_device(D.DeviceMesh.from_host(mesh))
nnz = b0.csc.nnz
del b0
xfer = CscHostTransfer(mesh.n_nodes, nnz, depth=2)
main = torch.cuda.Stream()
T0 = time.perf_counter()
log = []


def now():
    return (time.perf_counter() - T0) * 1e3


futs = []
for i in range(8):
    t_a = now()
    with torch.cuda.stream(main):
        dm = D.DeviceMesh(*(t.to(dev, non_blocking=True) for t in h))
        t_b = now()
        b = build_device(dm)
        t_c = now()
        f = xfer.submit(b.csc, stream=main)
        t_d = now()
    f.add_done_callback(lambda _f, i=i: log.append((i, "done", now())))
    futs.append(f)
    log.append((i, f"enqueue-h2d {t_a:.0f} build-start {t_b:.0f} build-returned {t_c:.0f} submitted {t_d:.0f}", t_d))
    del b, dm
for f in futs:
    f.result()
torch.cuda.synchronize()
for e in sorted(log, key=lambda x: x[2]):
    print(e[0], e[1], f"{e[2]:.0f}" if e[1] == "done" else "")
for t in (xfer.trace or []):
    print("step %d: D2H %.1f ms, widen %.1f ms" % t[:3])
xfer.close()
