"""Co-execution probe: the integration kernel and a planned emit pass on two streams at once vs one
after the other (is there slack to overlap the FP64-bound and the DRAM-bound kernels?)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_1501_04784_b200 import device as D  # noqa: E402
from paper_1501_04784_b200.workloads import make_workload  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "C3"
dm = D.DeviceMesh.from_host(make_workload(wl))
n = dm.n_el
plan = D.plan_assembly(dm)
ke0, _, _, f = D.integrate_mesh(dm, with_index=False)
D.raise_if_failed(f)
ke = torch.empty((n, 36), dtype=torch.float64, device="cuda")
rows = torch.empty(36 * n, dtype=torch.int32, device="cuda")
cols = torch.empty(36 * n, dtype=torch.int32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts)


def ke_only():
    D.integrate_mesh(dm, ke=ke, rows=rows, cols=cols)


def emit_only():
    D.mesh_emit(plan, ke0)


def both():
    e = torch.cuda.current_stream().record_event()
    s1.wait_event(e)
    s2.wait_event(e)
    with torch.cuda.stream(s1):
        D.integrate_mesh(dm, ke=ke, rows=rows, cols=cols, stream=s1)
    with torch.cuda.stream(s2):
        D.mesh_emit(plan, ke0, stream=s2)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


tk, te, tb = timed(ke_only), timed(emit_only), timed(both)
print(f"{wl} KE_BLOCKS_PER_SM={os.environ.get('HX_KE_BLOCKS_PER_SM', '-')}: ke {tk:.3f} ms, emit {te:.3f} ms, "
      f"sum {tk + te:.3f} ms, concurrent {tb:.3f} ms", flush=True)
