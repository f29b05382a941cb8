"""Break one rank's unpack + assemble (sharded build) into its calls: CUDA-event time of each with
a sync before and after, and host time of the calls themselves (launch overhead)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1501_04784_b200 import distributed as X  # noqa: E402
from paper_1501_04784_b200.workloads import make_workload  # noqa: E402

wl, world, r = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
mesh = make_workload(wl)
ops0 = X.CudaOps()
whole = ops0.upload(mesh.coords, mesh.connectivity, mesh.coefficient)
hist = ops0.column_weights(whole, mesh.n_nodes, X.histogram_bins(mesh.n_nodes))
bounds = X.balanced_bounds(hist.cpu().numpy(), mesh.n_nodes, world)
del whole
ranks = [X.ShardedBuild(mesh, q, world, ops=X.CudaOps(), exchange=X.LoopbackExchange(), bounds=bounds)
         for q in range(world)]
metas = [rk.phase_local().cpu().numpy() for rk in ranks]
C = ranks[0].check_meta(np.stack(metas))
chunk = 4 * C[:, :, 0] + C[:, :, 1]
sends = []
for q, rk in enumerate(ranks):
    send = rk.ops.alloc_words(int(chunk[q].sum()))
    offs = np.concatenate([[0], np.cumsum(chunk[q])[:-1]])
    rk.pack(*rk.ops.pointers([send.data_ptr()] * world, offs))
    sends.append((send, offs))
recv = torch.cat([sends[s][0][int(sends[s][1][r]):int(sends[s][1][r] + chunk[s, r])] for s in range(world)])
rk = ranks[r]
rk.nnz_hint = None
del sends
for q in range(world):
    if q != r:
        ranks[q] = None
torch.cuda.empty_cache()


def timed(name, fn):
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record()
    out = fn()
    b.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"  {name:28s} gpu {a.elapsed_time(b):7.3f} ms  host {1e3 * (t1 - t0):7.3f} ms", flush=True)
    return out


def wrap(obj, name):
    fn = getattr(obj, name)

    def w(*a, **k):
        return timed(name, lambda: fn(*a, **k))
    setattr(obj, name, w)


for name in ("integrate", "halo_count", "halo_unpack", "assemble"):
    wrap(rk.ops, name)
for rep in range(5):
    print(f"rep {rep}")
    timed("phase_local", rk.phase_local)
    send = rk.ops.alloc_words(int(chunk[r].sum()))
    offs = np.concatenate([[0], np.cumsum(chunk[r])[:-1]])
    timed("pack", lambda: rk.pack(*rk.ops.pointers([send.data_ptr()] * world, offs)))
    timed("phase_assemble", lambda: rk.phase_assemble(recv, C))
    print(f"  mem allocated {torch.cuda.memory_allocated() / 1e9:.2f} GB reserved {torch.cuda.memory_reserved() / 1e9:.2f} GB")
