"""run_build (C4, pinned host mesh) call time against the streamed path's knobs: stream blocks K and
decode threads (HX_DECODE_THREADS).  Median of 3 calls after 3 warm-up calls per setting."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1501_04784_b200 import pipeline  # noqa: E402
from paper_1501_04784_b200.hostmem import pinned_mesh  # noqa: E402
from paper_1501_04784_b200.workloads import make_workload  # noqa: E402

host_mesh = make_workload(sys.argv[1] if len(sys.argv) > 1 else "C4")
if os.environ.get("PRE"):  # bench-like: a device-resident mesh and builds before the e2e calls
    import torch

    from paper_1501_04784_b200 import device as D
    from paper_1501_04784_b200.pipeline import build_device
    dm = D.DeviceMesh.from_host(host_mesh)
    for _ in range(3):
        b = build_device(dm)
        torch.cuda.synchronize()
        del b
    torch.cuda.empty_cache()
mesh = pinned_mesh(host_mesh)
keep = []


def call():
    global keep
    t = time.perf_counter()
    keep.append(pipeline.run_build(mesh, budget_bytes=10**13)[0])
    keep = keep[-2:]
    return 1e3 * (time.perf_counter() - t)


for _ in range(3):
    call()
for K in (int(k) for k in os.environ.get("KS", "10").split()):
    for th in os.environ.get("THREADS", "0 4 6 8 12 16").split():
        pipeline.STREAM_BLOCKS = K
        os.environ["HX_DECODE_THREADS"] = th
        for _ in range(2):
            call()
        ts = sorted(call() for _ in range(3))
        print(f"K={K:3d} decode_threads={th:>2s}  call median {ts[1]:7.1f} ms  min {ts[0]:7.1f} ms", flush=True)
