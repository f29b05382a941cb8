"""Multi-process (world_size 2 and 3) sharded build over torch.distributed/gloo on CPU.

The distributed host logic of paper_1501_04784_b200.distributed (element-range shards,
column-block ownership, count exchange, the all-to-all of element-halo records with split
sizes, the [lower ranks | own | higher ranks] segment order, the global nnz all-gather) runs
unchanged; only the per-rank compute is swapped for the CPU oracle (``OracleOps``, test
infrastructure).  The concatenated column blocks must be bitwise equal to the single-process
reference CSC -- the same bar the GPU loopback tests apply to the CUDA kernels.
"""

import os
import socket
import sys
from pathlib import Path
from types import SimpleNamespace

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent
RECORD_DOUBLES = 40


class OracleOps:
    """CPU stand-in for distributed.CudaOps with the same call contract (oracle arithmetic)."""

    def upload(self, coords, conn, coeff):
        return SimpleNamespace(coords=np.ascontiguousarray(coords), conn=torch.from_numpy(np.ascontiguousarray(conn)),
                               coeff=np.ascontiguousarray(coeff))

    def integrate(self, dm):
        import oracle

        ke, rows, cols, first, _, _ = oracle.stiffness_mesh(dm.coords, dm.conn.numpy(), dm.coeff, threads=1)
        return torch.from_numpy(ke), torch.from_numpy(rows), torch.from_numpy(cols), first

    def check_fail(self, fail, offset):
        assert fail == -1

    def bounds(self, bounds_np):
        return bounds_np

    def halo(self, dm, ke, bounds, world, rank):
        """Restatement of hx_halo_count/hx_halo_pack: every local element, in ascending order, to
        every other rank owning one of its nodes; destination-major record buffer."""
        conn = dm.conn.numpy()
        owner = np.searchsorted(bounds, conn, side="right") - 1  # (n, 8)
        buckets = [[] for _ in range(world)]
        for e in range(conn.shape[0]):
            for d in sorted(set(owner[e].tolist()) - {rank}):
                rec = np.empty(RECORD_DOUBLES)
                rec[:36] = ke[e].numpy()
                rec.view(np.int32)[72:80] = conn[e]
                buckets[d].append(rec)
        counts = [len(b) for b in buckets]
        recs = [r for b in buckets for r in b]
        records = torch.from_numpy(np.array(recs).reshape(-1, RECORD_DOUBLES)) if recs else \
            torch.empty((0, RECORD_DOUBLES), dtype=torch.float64)
        return records, counts

    def assemble(self, segments, n_nodes, c_lo, c_hi):
        import oracle

        rows, cols, vals = [], [], []
        for conn, ke in segments:
            r, c = oracle.connectivity_index_arrays(conn.contiguous().numpy())
            rows.append(r)
            cols.append(c)
            vals.append(ke.contiguous().numpy().reshape(-1))
        rows, cols, vals = np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)
        keep = (cols >= c_lo) & (cols < c_hi)
        cp, ri, vv = oracle.triplet_to_csc(rows[keep], cols[keep], vals[keep], n_nodes)
        block = cp[c_lo:c_hi + 1] - cp[c_lo]
        return SimpleNamespace(col_ptr=torch.from_numpy(block), row_idx=torch.from_numpy(ri),
                               vals=torch.from_numpy(vv))


def _mesh(kind):
    from paper_1501_04784_b200.workloads import permuted_mesh, perturbed_mesh

    mesh = perturbed_mesh(5, seed=3)
    return permuted_mesh(mesh, seed=4) if kind == "permuted" else mesh


def _worker(rank, world, port, kind, outdir):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_1501_04784_b200.distributed import ShardedBuild, TorchExchange

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        runner = ShardedBuild(_mesh(kind), rank, world, ops=OracleOps(), exchange=TorchExchange())
        res = runner.step()
        total = runner.global_nnz()
        np.savez(Path(outdir) / f"rank{rank}.npz", col_ptr=res.col_ptr.numpy(), row_idx=res.row_idx.numpy(),
                 vals=res.vals.numpy(), nnz_offset=res.nnz_offset, total=total)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("kind", ["structured", "permuted"])
def test_gloo_sharded_build_bitwise_equal_to_reference(tmp_path, world, kind):
    import oracle

    mp.start_processes(_worker, args=(world, _free_port(), kind, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    blocks = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    col_ptr = np.concatenate([[0]] + [b["col_ptr"][1:] + int(b["nnz_offset"]) for b in blocks])
    row_idx = np.concatenate([b["row_idx"] for b in blocks])
    vals = np.concatenate([b["vals"] for b in blocks])
    mesh = _mesh(kind)
    ke, rows, cols, first, _, _ = oracle.stiffness_mesh(mesh.coords, mesh.connectivity, mesh.coefficient)
    cp, ri, vv = oracle.triplet_to_csc(rows, cols, ke.reshape(-1), mesh.n_nodes)
    assert all(int(b["total"]) == len(ri) for b in blocks)
    assert np.array_equal(col_ptr, cp) and np.array_equal(row_idx, ri)
    assert vals.tobytes() == vv.tobytes()
