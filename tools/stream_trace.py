import os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1501_04784_b200 import pipeline, stream
from paper_1501_04784_b200.hostmem import pinned_mesh
from paper_1501_04784_b200.workloads import make_workload
mesh = pinned_mesh(make_workload(sys.argv[1] if len(sys.argv) > 1 else "C4"))
keep = []
for i in range(3):
    keep.append(pipeline.run_build(mesh, budget_bytes=10**13)[0]); keep = keep[-2:]
os.environ["HX_TRACE_STREAM"] = "1"
for K in (8,):
    pipeline.STREAM_BLOCKS = K
    for i in range(2):
        t = time.perf_counter()
        keep.append(pipeline.run_build(mesh, budget_bytes=10**13)[0]); keep = keep[-2:]
        print(f"K={K} call {1e3*(time.perf_counter()-t):.1f} ms", flush=True)
