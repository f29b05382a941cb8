"""Where a synchronous run_build call spends its time at C4 (host clock per phase)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1501_04784_b200 import device as D  # noqa: E402
from paper_1501_04784_b200 import transfer  # noqa: E402
from paper_1501_04784_b200.hostmem import pinned_mesh  # noqa: E402
from paper_1501_04784_b200.pipeline import build_device, run_build  # noqa: E402
from paper_1501_04784_b200.workloads import make_workload  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "C4"
mesh = make_workload(wl)
t = time.perf_counter()
pm = pinned_mesh(mesh)
print(f"pinned_mesh {time.perf_counter() - t:.3f}s", flush=True)
dm = D.DeviceMesh.from_host(pm)
b = build_device(dm)
torch.cuda.synchronize()
n = b.csc.nnz
for i in range(4):
    t = time.perf_counter()
    a = torch.empty(n, dtype=torch.float64, pin_memory=True)
    t1 = time.perf_counter()
    print(f"pinned alloc {8 * n / 1e9:.1f} GB: {t1 - t:.3f}s", flush=True)
    del a
for i in range(4):
    torch.cuda.synchronize()
    t = time.perf_counter()
    m = transfer.fetch_csc(b.csc)
    print(f"fetch_csc #{i}: {time.perf_counter() - t:.3f}s", flush=True)
for i in range(3):
    t = time.perf_counter()
    m, rep = run_build(pm, budget_bytes=10**13)
    print(f"run_build #{i}: {time.perf_counter() - t:.3f}s  int {rep.time_integration_s*1e3:.1f} ms asm {rep.time_assembly_s*1e3:.1f} ms", flush=True)
# pieces of fetch_csc
vals_h = torch.empty(n, dtype=torch.float64, pin_memory=True)
for i in range(2):
    torch.cuda.synchronize()
    t = time.perf_counter()
    vals_h.copy_(b.csc.vals, non_blocking=True)
    torch.cuda.synchronize()
    print(f"D2H vals {8*n/1e9:.2f} GB: {time.perf_counter() - t:.3f}s", flush=True)
r32 = D.rows_narrow(b.csc.row_idx)
r32_h = torch.empty(n, dtype=torch.int32, pin_memory=True)
r64_h = torch.empty(n, dtype=torch.int64, pin_memory=True)
r32_h.copy_(r32)
for th in (4, 8, 16):
    t = time.perf_counter()
    D.N.check(D.N.lib().hx_rows_widen(r32_h.data_ptr(), r64_h.data_ptr(), n, th), "w")
    print(f"widen {n} threads {th}: {time.perf_counter() - t:.3f}s", flush=True)
r64_np = np.empty(n, dtype=np.int64)
t = time.perf_counter()
D.N.check(D.N.lib().hx_rows_widen(r32_h.data_ptr(), r64_np.ctypes.data, n, 16), "w")
print(f"widen into fresh numpy 16 threads: {time.perf_counter() - t:.3f}s", flush=True)
t = time.perf_counter()
D.N.check(D.N.lib().hx_rows_widen(r32_h.data_ptr(), r64_np.ctypes.data, n, 16), "w")
print(f"widen into touched numpy 16 threads: {time.perf_counter() - t:.3f}s", flush=True)
