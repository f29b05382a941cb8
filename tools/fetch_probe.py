"""fetch_csc variants at C4: ordering of the row / value chunks, widen threads, no widening."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_1501_04784_b200 import device as D  # noqa: E402
from paper_1501_04784_b200 import transfer  # noqa: E402
from paper_1501_04784_b200.pipeline import build_device, run_build  # noqa: E402
from paper_1501_04784_b200.hostmem import pinned_mesh  # noqa: E402
from paper_1501_04784_b200.workloads import make_workload  # noqa: E402

mesh = make_workload(sys.argv[1] if len(sys.argv) > 1 else "C4")
b = build_device(D.DeviceMesh.from_host(mesh))
torch.cuda.synchronize()
n = b.csc.nnz
keep = []


def timeit(name, fn, reps=4):
    ts = []
    for i in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = fn()
        ts.append(time.perf_counter() - t)
        keep.append(r)
        if len(keep) > 2:
            keep.pop(0)
    print(f"{name}: " + " ".join(f"{x * 1e3:.0f}" for x in ts) + " ms", flush=True)


for kw in ({}, {"rows_first": True}, {"threads": 12}, {"threads": 8}, {"chunk": 1 << 23}, {"chunk": 1 << 27},
           {"rows_first": True, "threads": 8}):
    timeit(f"fetch_csc {kw}", lambda: transfer.fetch_csc(b.csc, **kw))

r32 = D.rows_narrow(b.csc.row_idx)
hv = torch.empty(n, dtype=torch.float64, pin_memory=True)
hr = torch.empty(n, dtype=torch.int32, pin_memory=True)
hc = torch.empty(b.csc.col_ptr.shape[0], dtype=torch.int64, pin_memory=True)


def plain():
    hr.copy_(r32, non_blocking=True)
    hv.copy_(b.csc.vals, non_blocking=True)
    hc.copy_(b.csc.col_ptr, non_blocking=True)
    torch.cuda.synchronize()


timeit("plain D2H rows32+vals+col_ptr, no widen", plain)
pm = pinned_mesh(mesh)
del b
torch.cuda.empty_cache()
keep.clear()
timeit("run_build", lambda: run_build(pm, budget_bytes=10**13), reps=5)
