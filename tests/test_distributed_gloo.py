"""Multi-process (world_size 2 and 3) sharded build over torch.distributed/gloo on CPU.

The distributed host logic of paper_1501_04784_b200.distributed (element-range shards,
column-block ownership, count exchange, the all-to-all of element-halo records with split
sizes, the [lower ranks | own | higher ranks] segment order, the global nnz all-gather) runs
unchanged; only the per-rank compute is swapped for the CPU oracle (``OracleOps``, test
infrastructure).  The concatenated column blocks must be bitwise equal to the single-process
reference CSC -- the same bar the GPU loopback tests apply to the CUDA kernels.
"""

import ctypes
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


def _words_at(ptr: int, n: int) -> np.ndarray:
    return np.ctypeslib.as_array((ctypes.c_int64 * max(n, 1)).from_address(ptr))[:n]


class OracleOps:
    """CPU stand-in for distributed.CudaOps with the same call contract (oracle arithmetic and the
    numpy restatement of the exchange kernels, oracle/halo.py)."""

    def upload(self, coords, conn, coeff):
        conn = np.ascontiguousarray(conn)
        return SimpleNamespace(coords=np.ascontiguousarray(coords), conn=torch.from_numpy(conn),
                               coeff=np.ascontiguousarray(coeff), n_el=conn.shape[0])

    def integrate(self, dm):
        import oracle

        ke, rows, cols, first, _, _ = oracle.stiffness_mesh(dm.coords, dm.conn.numpy(), dm.coeff, threads=1)
        fail = torch.tensor([-1, -1, 0], dtype=torch.int64)
        if first >= 0:
            fail[0] = first
            fail[1] = 0
        return torch.from_numpy(ke), torch.from_numpy(rows), torch.from_numpy(cols), fail

    def column_weights(self, dm, n_nodes, n_bins):
        from oracle import halo

        return torch.from_numpy(halo.column_weights(dm.conn.numpy(), n_nodes, n_bins))

    def bounds(self, bounds_np):
        return bounds_np

    def halo_count(self, dm, bounds, world, rank):
        from oracle import halo

        return torch.from_numpy(halo.count(dm.conn.numpy(), bounds, world, rank)), None

    def alloc_words(self, n):
        return torch.empty(n, dtype=torch.int64)

    def pointers(self, bases, offsets):
        return [int(b) for b in bases], [int(o) for o in offsets]

    def halo_pack(self, dm, ke, bounds, world, rank, ptrs, offsets, ws):
        from oracle import halo

        for d, chunk in enumerate(halo.pack(dm.conn.numpy(), ke.numpy(), bounds, world, rank)):
            if chunk.size:
                _words_at(ptrs[d] + 8 * offsets[d], chunk.size)[:] = chunk

    def halo_unpack(self, recv, desc, bounds, world, rank, n_rec):
        from oracle import halo

        out = halo.unpack(recv.numpy(), desc, bounds, world, rank)
        assert out.shape[0] == n_rec
        return torch.from_numpy(out)

    def digest(self, t, pos0, add=0):
        from paper_1501_04784_b200.distributed import digest_words

        v = digest_words(t.contiguous().numpy(), pos0, add)
        return torch.tensor([np.uint64(v).astype(np.int64)], dtype=torch.int64)

    def assemble(self, segments, n_nodes, c_lo, c_hi, nnz_hint=None, order="auto"):
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
        digest = runner.exchange.sum_(runner.block_digest())
        np.savez(Path(outdir) / f"rank{rank}.npz", col_ptr=res.col_ptr.numpy(), row_idx=res.row_idx.numpy(),
                 vals=res.vals.numpy(), nnz_offset=res.nnz_offset, total=total, digest=digest.numpy(),
                 bounds=runner.bounds_np, xbytes=runner.exchange_bytes()["bytes"])
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
    # every rank holds the same bounds, and the summed block digests are the whole matrix's
    assert all(np.array_equal(b["bounds"], blocks[0]["bounds"]) for b in blocks)
    from paper_1501_04784_b200.distributed import csc_digest

    want = np.array(csc_digest(cp, ri, vv), dtype=np.uint64).astype(np.int64)
    assert all(np.array_equal(b["digest"], want) for b in blocks)


def _fail_worker(rank, world, port, outdir):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_1501_04784_b200.distributed import ShardedBuild, TorchExchange
    from paper_1501_04784_b200.errors import DegenerateElementError
    from paper_1501_04784_b200.mesh import Mesh

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mesh = _mesh("structured")
        conn = mesh.connectivity.copy()
        conn[[90, 110]] = conn[[90, 110]][:, [4, 5, 6, 7, 0, 1, 2, 3]]  # inverted: degenerate, in the last range
        runner = ShardedBuild(Mesh(mesh.coords, np.ascontiguousarray(conn), mesh.coefficient), rank, world,
                              ops=OracleOps(), exchange=TorchExchange())
        try:
            runner.step()
            got = -1
        except DegenerateElementError as e:
            got = e.element_id
        # every rank raised, so every rank reaches this collective (no rank left waiting in the step)
        dist.barrier()
        np.save(Path(outdir) / f"fail{rank}.npy", np.array([got]))
    finally:
        dist.destroy_process_group()


def test_gloo_sharded_build_raises_the_same_error_on_every_rank(tmp_path):
    """A degenerate element in one rank's range: every rank raises DegenerateElementError for the
    lowest failing global element (element.py:237-244) and none is left inside a collective."""
    world = 2
    mp.start_processes(_fail_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    got = [int(np.load(tmp_path / f"fail{r}.npy")[0]) for r in range(world)]
    assert got == [90, 90]
