"""Per-call host time of run_build (the e2e drop-in) at a workload, plus one traced call."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_1501_04784_b200.hostmem import pinned_mesh  # noqa: E402
from paper_1501_04784_b200.pipeline import run_build  # noqa: E402
from paper_1501_04784_b200.workloads import make_workload  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "C4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
mesh = make_workload(wl)
pm = pinned_mesh(mesh)
m = None
for i in range(steps):
    t = time.perf_counter()
    m, rep = run_build(pm, budget_bytes=10**13)
    torch.cuda.synchronize()
    print(f"{wl} run_build #{i}: {1e3 * (time.perf_counter() - t):.1f} ms  int {rep.time_integration_s*1e3:.1f} "
          f"asm {rep.time_assembly_s*1e3:.1f}", flush=True)
os.environ["HX_TRACE_STREAM"] = "1"
m, rep = run_build(pm, budget_bytes=10**13)
