"""Multi-process check of the sharded build (torchrun): every rank builds its column block through
the real exchange (HX_EXCHANGE=nccl|p2p over HX_DIST_BACKEND=nccl|gloo); rank 0 gathers the blocks
and compares them bit for bit with the single-GPU build.  Prints one PASS/FAIL line per mesh."""
import hashlib
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1501_04784_b200 import device as D  # noqa: E402
from paper_1501_04784_b200 import distributed as X  # noqa: E402
from paper_1501_04784_b200.pipeline import build_device  # noqa: E402
from paper_1501_04784_b200.workloads import make_workload, permuted_mesh, perturbed_mesh  # noqa: E402

backend = os.environ.get("HX_DIST_BACKEND", "nccl")
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1)
torch.cuda.set_device(local)
if backend == "nccl":
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
else:
    dist.init_process_group("gloo")
use_p2p = os.environ.get("HX_EXCHANGE", "nccl") == "p2p"


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


ok_all = True
for name, mesh in [("perturbed 12^3", perturbed_mesh(12, seed=3)),
                   ("permuted 12^3", permuted_mesh(perturbed_mesh(12, seed=4), seed=5)),
                   ("C2", make_workload("C2"))]:
    runner = X.ShardedBuild(mesh, rank, world, exchange=X.P2PExchange() if use_p2p else None)
    for _ in range(2):  # second step reuses the mapped receive buffers
        res = runner.step()
    runner.global_nnz()
    part = (res.col_ptr.cpu().numpy(), res.row_idx.cpu().numpy(), res.vals.cpu().numpy(), res.nnz_offset)
    parts = [None] * world
    dist.all_gather_object(parts, part)
    if rank == 0:
        cp = np.concatenate([[0]] + [p[0][1:] + p[3] for p in parts])
        ri = np.concatenate([p[1] for p in parts])
        vv = np.concatenate([p[2] for p in parts])
        b = build_device(D.DeviceMesh.from_host(mesh))
        ref = digest(b.csc.col_ptr.cpu().numpy(), b.csc.row_idx.cpu().numpy(), b.csc.vals.cpu().numpy())
        ok = digest(cp, ri, vv) == ref
        ok_all &= ok
        print(f"{'PASS' if ok else 'FAIL'} {name}: world {world}, backend {backend}, exchange "
              f"{'p2p' if use_p2p else 'all_to_all'}, nnz {len(ri)}", flush=True)
    del runner
dist.barrier()
dist.destroy_process_group()
sys.exit(0 if ok_all else 1)
