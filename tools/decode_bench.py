"""Host row-decode throughput (hx_rows_decode) on a real build's encoded rows, per thread count."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1501_04784_b200 import device as D  # noqa: E402
from paper_1501_04784_b200.pipeline import build_device  # noqa: E402
from paper_1501_04784_b200.transfer import RowEncoder, decode_rows, host_threads  # noqa: E402
from paper_1501_04784_b200.workloads import make_workload  # noqa: E402

mesh = make_workload(sys.argv[1] if len(sys.argv) > 1 else "C3")
b = build_device(D.DeviceMesh.from_host(mesh))
counts, lens, data, total = RowEncoder().encode(b.csc.col_ptr, b.csc.row_idx, 0)
n = int(total.item())
c, l = counts.cpu().numpy(), lens.cpu().numpy()
buf = np.zeros(n + 16, np.uint8)
buf[:n] = data[:n].cpu().numpy()
nnz = b.csc.nnz
out = np.empty(nnz, np.int64)
out.fill(0)
ends = np.empty(len(c), np.int64)
print(f"{nnz / 1e6:.1f}M rows, {n / nnz:.2f} bytes/row, host threads {host_threads()}", flush=True)
for th in (1, 4, 8, 16, 32, 0):
    ts = []
    for _ in range(3):
        t = time.perf_counter()
        decode_rows(c, l, buf, n, 0, 0, ends, out, th)
        ts.append(time.perf_counter() - t)
    print(f"threads {th}: {1e3 * min(ts):.1f} ms -> {nnz / min(ts) / 1e9:.2f} G rows/s", flush=True)
assert np.array_equal(out, b.csc.row_idx.cpu().numpy())
