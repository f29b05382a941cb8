"""run_build at C4: streamed column blocks vs one-shot, pinned mesh; out-of-core budgets."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_1501_04784_b200 import pipeline, stream  # noqa: E402
from paper_1501_04784_b200.hostmem import pinned_mesh  # noqa: E402
from paper_1501_04784_b200.workloads import make_workload  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "C4"
mesh = pinned_mesh(make_workload(wl))
t = time.perf_counter()
sp = stream.plan(mesh, 8)
print(f"plan (host scan) {1e3 * (time.perf_counter() - t):.1f} ms; overlap {(sp.e_hi - sp.e_lo).sum() / mesh.n_el:.3f}",
      flush=True)
keep = []
for blocks in (4, 8, 16, 32):
    pipeline.STREAM_BLOCKS = blocks
    ts = []
    for i in range(5):
        t = time.perf_counter()
        m, rep = pipeline.run_build(mesh, budget_bytes=10**13)
        ts.append(time.perf_counter() - t)
        keep.append(m)
        if len(keep) > 2:
            keep.pop(0)
    print(f"streamed K={blocks}: " + " ".join(f"{1e3 * x:.0f}" for x in ts) + f" ms  (int {rep.time_integration_s*1e3:.1f}, asm {rep.time_assembly_s*1e3:.1f})", flush=True)
os.environ["HX_STREAMED"] = "0"
ts = []
for i in range(4):
    t = time.perf_counter()
    m, rep = pipeline.run_build(mesh, budget_bytes=10**13)
    ts.append(time.perf_counter() - t)
    keep.append(m)
    keep.pop(0)
print("one-shot: " + " ".join(f"{1e3 * x:.0f}" for x in ts) + " ms", flush=True)
os.environ["HX_STREAMED"] = "1"
need = pipeline.device_bytes(mesh.n_el, mesh.n_nodes)
for frac in (4, 8):
    ts = []
    for i in range(3):
        t = time.perf_counter()
        m, rep = pipeline.run_build(mesh, budget_bytes=10**13, device_budget_bytes=need // frac)
        ts.append(time.perf_counter() - t)
        keep.append(m)
        keep.pop(0)
    print(f"out-of-core budget 1/{frac}: " + " ".join(f"{1e3 * x:.0f}" for x in ts) + " ms", flush=True)
