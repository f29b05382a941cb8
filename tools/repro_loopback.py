import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from paper_1501_04784_b200.distributed import CudaOps, run_loopback, concat_blocks
from paper_1501_04784_b200.workloads import permuted_mesh, perturbed_mesh
mesh = permuted_mesh(perturbed_mesh(9, seed=8), seed=18)
res = run_loopback(mesh, 8, lambda: CudaOps())
print(concat_blocks(res)[0][-1])
