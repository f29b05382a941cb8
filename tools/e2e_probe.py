"""Where the e2e step goes: pinned D2H of one C4-sized CSC (int32 rows + f64 values + col_ptr) alone,
concurrent with a 4.1 GB H2D, the host widening alone, and the pipelined bench e2e (both row modes)."""
import os
import subprocess
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1501_04784_b200 import _native as N  # noqa: E402
from paper_1501_04784_b200.transfer import host_threads  # noqa: E402

nnz, ncols = 898_402_401, 64_481_201
dev = torch.device("cuda")
d_rows = torch.empty(nnz, dtype=torch.int32, device=dev)
d_vals = torch.empty(nnz, dtype=torch.float64, device=dev)
d_cp = torch.empty(ncols + 1, dtype=torch.int64, device=dev)
h_rows = torch.empty(nnz, dtype=torch.int32, pin_memory=True)
h_vals = torch.empty(nnz, dtype=torch.float64, pin_memory=True)
h_cp = torch.empty(ncols + 1, dtype=torch.int64, pin_memory=True)
h_in = torch.empty(4_107_548_824 // 8, dtype=torch.float64, pin_memory=True)
d_in = torch.empty_like(h_in, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def d2h():
    with torch.cuda.stream(s1):
        h_rows.copy_(d_rows, non_blocking=True)
        h_vals.copy_(d_vals, non_blocking=True)
        h_cp.copy_(d_cp, non_blocking=True)


def h2d():
    with torch.cuda.stream(s2):
        d_in.copy_(h_in, non_blocking=True)


def timed(fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) * 1e3


d2h()
h2d()
for _ in range(2):
    print(f"D2H 11.3 GB alone: {timed(d2h):.1f} ms; with concurrent 4.1 GB H2D: {timed(lambda: (d2h(), h2d())):.1f} ms",
          flush=True)
out = np.empty(nnz, dtype=np.int64)
out.fill(0)
th = host_threads()
for t in (th, th // 2):
    t0 = time.perf_counter()
    N.check(N.lib().hx_rows_widen(h_rows.data_ptr(), out.ctypes.data, nnz, t), "widen")
    print(f"host widen {nnz} rows, {t} threads: {(time.perf_counter() - t0) * 1e3:.1f} ms", flush=True)
t0 = time.perf_counter()
d2h()
N.check(N.lib().hx_rows_widen(h_rows.data_ptr(), out.ctypes.data, nnz, th), "widen")
torch.cuda.synchronize()
print(f"D2H while widening: {(time.perf_counter() - t0) * 1e3:.1f} ms", flush=True)
del d_rows, d_vals, d_cp, d_in
torch.cuda.empty_cache()
for rows in ("i32", "i64", "i32"):
    r = subprocess.run([sys.executable, "bench.py", "--no-cpu-baseline", "--e2e-rows", rows, "--steps", "10"],
                       capture_output=True, text=True)
    import json
    d = json.loads(r.stdout.strip().splitlines()[-1])
    print(f"bench e2e rows={rows}: {d['e2e']['ms_per_step']:.1f} ms/step -> {d['e2e']['value'] / 1e6:.1f} M el/s", flush=True)
