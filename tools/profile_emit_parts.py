"""Profiling driver: the rows-only emit (symbolic with row_capacity) and the full build's emit on one
workload, to split the emit pass's DRAM traffic between the record stream and the KE gathers."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_1501_04784_b200 import _native as N  # noqa: E402
from paper_1501_04784_b200 import device as D  # noqa: E402
from paper_1501_04784_b200.workloads import make_workload  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "C3"
dm = D.DeviceMesh.from_host(make_workload(wl))
ke, _, _, fail = D.integrate_mesh(dm, with_index=False)
csc = D.mesh_csc([(dm.conn, ke)], dm.n_nodes)  # full build (emit with values)
nnz = csc.nnz
ws_bytes = N.lib().hx_mesh_csc_workspace_bytes(dm.n_el, dm.n_nodes)
ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
status = torch.zeros(1, dtype=torch.int32, device="cuda")
col_ptr = torch.empty(dm.n_nodes + 1, dtype=torch.int64, device="cuda")
segs = N.segments([(dm.conn.data_ptr(), 0, dm.n_el)])
N.check(N.lib().hx_mesh_csc_symbolic(segs, 1, dm.n_nodes, 0, dm.n_nodes, ctypes.c_void_p(col_ptr.data_ptr()),
                                     ctypes.c_void_p(csc.row_idx.data_ptr()), nnz, ctypes.c_void_p(ws.data_ptr()),
                                     ws_bytes, ctypes.c_void_p(status.data_ptr()), 0, None), "symbolic")
torch.cuda.synchronize()
print("profiled", wl, "status", int(status.item()))
