"""Profiling driver: one cold build of an n^3 unit-cube mesh generated on the device (used under ncu
to see how a kernel's DRAM traffic scales with the mesh size)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_1501_04784_b200 import device as D  # noqa: E402
from paper_1501_04784_b200.mesh import StructuredGridSpec  # noqa: E402
from paper_1501_04784_b200.pipeline import build_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
dm = D.generate_cube_mesh(StructuredGridSpec(n, n, n))
b = build_device(dm)
torch.cuda.synchronize()
print("profiled cube", n, "nnz", b.csc.nnz)
