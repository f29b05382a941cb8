"""Multi-GPU construction: element-range shards, column blocks, one all-to-all of element halos.

Rank r of G (one process per GPU, torch.distributed over NCCL):

1. integrates its contiguous element range E_r = [n_el*r/G, n_el*(r+1)/G) -- KE + fused iK/jK,
   exactly the single-GPU kernel on a slice of the mesh;
2. owns the lower-CSC column block C_r = [n_nodes*r/G, n_nodes*(r+1)/G) (a column block of the
   lower triangle is a row block of K by symmetry).  Column nnz is <= 27 and near-uniform on
   conforming hex meshes, so an equal node split is an equal nnz split;
3. sends every owned element that has a node in another rank's block to that rank -- one
   all-to-all of 320-byte records (36 KE values + 8 node ids), packed destination-major in
   ascending element order by hx_halo_pack;
4. assembles its block from the segments [received from lower ranks | own | received from
   higher ranks], which are in ascending global element order, so every duplicate position is
   summed in the single-GPU order: the concatenated blocks are bitwise equal to G = 1.

The global K is the concatenation of the blocks; global col_ptr = block col_ptr + exclusive
scan of the block nnz (one all-gather of G int64).

The collective is behind a small ``Exchange`` interface (torch.distributed for NCCL/gloo, a
loopback for simulating G ranks in one process) and the per-rank compute behind ``Ops`` (the
CUDA ops by default), so the host logic is tested with gloo on CPU and the CUDA path with the
loopback on one GPU.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

__all__ = ["element_ranges", "column_bounds", "ShardedBuild", "TorchExchange", "LoopbackExchange", "CudaOps",
           "run_loopback", "run_loopback_p2p", "P2PExchange", "RECORD_DOUBLES", "all_reduce", "barrier"]

RECORD_DOUBLES = 40  # 36 packed KE values + 8 int32 node ids


def element_ranges(n_el: int, world: int):
    return [(n_el * r // world, n_el * (r + 1) // world) for r in range(world)]


def column_bounds(n_nodes: int, world: int) -> np.ndarray:
    return np.array([n_nodes * r // world for r in range(world + 1)], dtype=np.int64)


# ------------------------------------------------------------------------------------------
# collectives
# ------------------------------------------------------------------------------------------
def _host_staged(group=None) -> bool:
    """gloo collectives take host tensors: CUDA buffers are staged through host memory (the
    single-GPU multi-rank test mode); NCCL moves device buffers directly over NVLink."""
    import torch.distributed as dist

    return dist.get_backend(group) == "gloo"


def all_reduce(t: torch.Tensor, op=None, group=None) -> torch.Tensor:
    """In-place all-reduce of ``t`` (any device) over the group's backend; returns ``t``."""
    import torch.distributed as dist

    op = dist.ReduceOp.SUM if op is None else op
    if t.is_cuda and _host_staged(group):
        h = t.cpu()
        dist.all_reduce(h, op=op, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=op, group=group)
    return t


def barrier(group=None, device_index=None) -> None:
    import torch.distributed as dist

    if dist.get_backend(group) == "nccl" and device_index is not None:
        dist.barrier(group=group, device_ids=[device_index])
    else:
        dist.barrier(group=group)


class TorchExchange:
    """torch.distributed all-to-all: NCCL over NVLink on GPUs (device buffers), gloo on CPU (and
    host-staged CUDA buffers when several ranks share one GPU for testing)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group

    def _a2a(self, recv, send, **kw):
        if send.is_cuda and _host_staged(self.group):
            r = torch.empty(recv.shape, dtype=recv.dtype)
            self.dist.all_to_all_single(r, send.cpu(), group=self.group, **kw)
            recv.copy_(r)
        else:
            self.dist.all_to_all_single(recv, send, group=self.group, **kw)
        return recv

    def counts(self, send_counts: torch.Tensor) -> torch.Tensor:
        return self._a2a(torch.empty_like(send_counts), send_counts)

    def records(self, send: torch.Tensor, send_splits, recv_splits) -> torch.Tensor:
        recv = torch.empty((sum(recv_splits), RECORD_DOUBLES), dtype=send.dtype, device=send.device)
        return self._a2a(recv, send, output_split_sizes=list(recv_splits), input_split_sizes=list(send_splits))

    def allgather_int(self, value: int, device) -> list:
        t = torch.tensor([value], dtype=torch.int64, device="cpu" if _host_staged(self.group) else device)
        out = [torch.empty_like(t) for _ in range(self.dist.get_world_size(self.group))]
        self.dist.all_gather(out, t, group=self.group)
        return [int(x.item()) for x in out]


class P2PExchange:
    """The all-to-all done by the producer: every rank maps every other rank's receive buffer
    (CUDA IPC through torch's storage sharing -- NVLink peer memory between GPUs, the same memory
    between processes sharing a GPU) and hx_halo_send writes the records straight into them.  Only
    the G x G count matrix goes through the process group (one all-gather); a stream-ordered
    barrier (an NCCL all-reduce of one word; a host barrier under gloo) orders the receivers'
    reads after every sender's kernel."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.buf = None        # own receive buffer (records, 40 doubles each)
        self.peers = None      # tensors mapping every rank's buffer (own included)
        self.ptrs = None       # device int64 array of the peer base pointers

    def _ensure_capacity(self, need: int, device):
        """Grow the receive buffer when needed; whenever any rank grows, all ranks re-map."""
        grow = self.buf is None or self.buf.shape[0] < need
        flag = torch.tensor([1 if grow else 0], dtype=torch.int64)
        if self.dist.get_backend(self.group) != "gloo":
            flag = flag.to(device)
        self.dist.all_reduce(flag, op=self.dist.ReduceOp.MAX, group=self.group)
        if int(flag.item()) == 0:
            return
        if grow:
            self.buf = torch.empty((max(need + need // 4, 1024), RECORD_DOUBLES), dtype=torch.float64, device=device)
        meta = self.buf.untyped_storage()._share_cuda_()
        metas = [None] * self.world
        self.dist.all_gather_object(metas, meta, group=self.group)
        self.peers = []
        for r, m in enumerate(metas):
            if r == self.rank:
                self.peers.append(self.buf)
            else:
                st = torch.UntypedStorage._new_shared_cuda(*m)
                self.peers.append(torch.empty(0, dtype=torch.float64, device=device).set_(st))
        self.ptrs = torch.tensor([p.data_ptr() for p in self.peers], dtype=torch.int64, device=device)

    def prepare(self, send_counts, device):
        """-> (dest_ptrs, dest_offsets (device int64), recv_counts host list, receive view)"""
        mine = torch.tensor(send_counts, dtype=torch.int64)
        rows = [torch.empty_like(mine) for _ in range(self.world)]
        if self.dist.get_backend(self.group) == "gloo":
            self.dist.all_gather(rows, mine, group=self.group)
        else:
            dev_rows = [torch.empty(self.world, dtype=torch.int64, device=device) for _ in range(self.world)]
            self.dist.all_gather(dev_rows, mine.to(device), group=self.group)
            rows = [r.cpu() for r in dev_rows]
        C = torch.stack(rows).numpy()  # C[s][d] records s -> d
        recv_counts = [int(C[s][self.rank]) for s in range(self.world)]
        self._ensure_capacity(int(sum(recv_counts)), device)
        offsets = torch.tensor([int(C[:self.rank, d].sum()) for d in range(self.world)], dtype=torch.int64,
                               device=device)
        return self.ptrs, offsets, recv_counts, self.buf[:sum(recv_counts)]

    def barrier(self, device):
        if self.dist.get_backend(self.group) == "gloo":
            torch.cuda.synchronize(device)
            self.dist.barrier(group=self.group)
        else:
            t = torch.zeros(1, dtype=torch.int32, device=device)
            self.dist.all_reduce(t, group=self.group)  # stream-ordered: after every rank's send kernel

    def counts(self, send_counts):  # the ShardedBuild e2e helpers use the process group directly
        raise NotImplementedError

    def allgather_int(self, value: int, device) -> list:
        t = torch.tensor([value], dtype=torch.int64)
        out = [torch.empty_like(t) for _ in range(self.world)]
        if self.dist.get_backend(self.group) == "gloo":
            self.dist.all_gather(out, t, group=self.group)
            return [int(x.item()) for x in out]
        dev_out = [torch.empty(1, dtype=torch.int64, device=device) for _ in range(self.world)]
        self.dist.all_gather(dev_out, t.to(device), group=self.group)
        return [int(x.item()) for x in dev_out]


# ------------------------------------------------------------------------------------------
# per-rank compute (CUDA)
# ------------------------------------------------------------------------------------------
class CudaOps:
    """The device kernels of libhexfem_b200.so."""

    def __init__(self, device=None, mode="exact"):
        from . import device as D

        self.D = D
        self.device = D.require_device(device)
        self.mode = mode

    def upload(self, coords, conn, coeff):
        def up(a, dt):
            return torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(self.device)

        return self.D.DeviceMesh(up(coords, np.float64), up(conn, np.int32), up(coeff, np.float64))

    def integrate(self, dm):
        ke, rows, cols, fail = self.D.integrate_mesh(dm, mode=self.mode)
        return ke, rows, cols, fail

    def check_fail(self, fail, offset):
        self.D.raise_if_failed(fail, offset)

    def halo_count(self, dm, bounds_dev, world, rank):
        """-> (per_dest (world,) int64 host list, workspace) -- hx_halo_count."""
        from . import _native as N

        n = dm.n_el
        ws_bytes = N.lib().hx_halo_workspace_bytes(n, world)
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device=self.device)
        per_dest = torch.empty(world, dtype=torch.int64, device=self.device)
        N.check(N.lib().hx_halo_count(self.D._ptr(dm.conn), n, self.D._ptr(bounds_dev), world, rank,
                                      self.D._ptr(per_dest), self.D._ptr(ws), ws_bytes, self.D.stream_handle()),
                "hx_halo_count")
        return per_dest.cpu().tolist(), ws

    def halo(self, dm, ke, bounds_dev, world, rank):
        """-> (records (S, 40) f64 destination-major send buffer, per_dest host list)"""
        from . import _native as N

        counts, ws = self.halo_count(dm, bounds_dev, world, rank)
        records = torch.empty((max(sum(counts), 0), RECORD_DOUBLES), dtype=torch.float64, device=self.device)
        N.check(N.lib().hx_halo_pack(self.D._ptr(dm.conn), self.D._ptr(ke), dm.n_el, self.D._ptr(bounds_dev), world,
                                     rank, self.D._ptr(records), self.D._ptr(ws), self.D.stream_handle()),
                "hx_halo_pack")
        return records, counts

    def halo_send(self, dm, ke, bounds_dev, world, rank, dest_ptrs, dest_offsets, ws):
        """Fused pack-and-send: records straight into the destinations' receive buffers."""
        from . import _native as N

        N.check(N.lib().hx_halo_send(self.D._ptr(dm.conn), self.D._ptr(ke), dm.n_el, self.D._ptr(bounds_dev), world,
                                     rank, self.D._ptr(dest_ptrs), self.D._ptr(dest_offsets), self.D._ptr(ws),
                                     self.D.stream_handle()), "hx_halo_send")

    def bounds(self, bounds_np):
        return torch.from_numpy(bounds_np).to(self.device)

    def assemble(self, segments, n_nodes, c_lo, c_hi):
        return self.D.mesh_csc(segments, n_nodes, c_lo, c_hi)


def record_segment(records: torch.Tensor):
    """(n, 40) f64 records -> (conn (n, 8) int32 view, ke (n, 36) f64 view), no copy."""
    as_i32 = records.view(torch.int32)
    return as_i32[:, 72:80], records[:, :36]


@dataclass
class ShardResult:
    col_ptr: torch.Tensor  # local, starts at 0
    row_idx: torch.Tensor
    vals: torch.Tensor
    col_lo: int
    col_hi: int
    nnz_offset: int = 0


class ShardedBuild:
    """One rank's share of the global build (see module docstring)."""

    def __init__(self, mesh, rank: int, world: int, mode: str = "exact", ops=None, exchange=None):
        self.rank, self.world = rank, world
        self.ops = ops if ops is not None else CudaOps(mode=mode)
        self.exchange = exchange if exchange is not None else TorchExchange()
        self.n_el, self.n_nodes = mesh.n_el, mesh.n_nodes
        self.e_lo, self.e_hi = element_ranges(mesh.n_el, world)[rank]
        self.bounds_np = column_bounds(mesh.n_nodes, world)
        self.c_lo, self.c_hi = int(self.bounds_np[rank]), int(self.bounds_np[rank + 1])
        self.dm = self.ops.upload(mesh.coords, mesh.connectivity[self.e_lo:self.e_hi],
                                  mesh.coefficient[self.e_lo:self.e_hi])
        self.bounds = self.ops.bounds(self.bounds_np)
        self.last = None
        self.last_index = None

    # -- phases (so a loopback driver can interleave G ranks in one process) --
    def phase_local(self):
        ke, rows, cols, fail = self.ops.integrate(self.dm)
        records, send_counts = self.ops.halo(self.dm, ke, self.bounds, self.world, self.rank)
        self._pending = (ke, rows, cols, fail)
        return records, send_counts

    def phase_assemble(self, recv: torch.Tensor, recv_counts):
        ke, rows, cols, fail = self._pending
        self._pending = None
        n_lower = int(sum(recv_counts[:self.rank]))
        segments = []
        if n_lower:
            segments.append(record_segment(recv[:n_lower]))
        segments.append((self.dm.conn, ke))
        if recv.shape[0] > n_lower:
            segments.append(record_segment(recv[n_lower:]))
        self.ops.check_fail(fail, self.e_lo)
        csc = self.ops.assemble(segments, self.n_nodes, self.c_lo, self.c_hi)
        self.last = ShardResult(csc.col_ptr, csc.row_idx, csc.vals, self.c_lo, self.c_hi)
        self.last_index = (ke, rows, cols)
        return self.last

    def step(self):
        if isinstance(self.exchange, P2PExchange):
            return self.step_p2p()
        records, send_counts = self.phase_local()
        dev = records.device
        recv_counts = self.exchange.counts(torch.tensor(send_counts, dtype=torch.int64, device=dev)).cpu().tolist()
        recv = self.exchange.records(records, send_counts, recv_counts)
        return self.phase_assemble(recv, recv_counts)

    def step_p2p(self):
        """Integrate, count, map the destinations, fused pack-and-send, barrier, assemble."""
        dev = self.ops.device
        ke, rows, cols, fail = self.ops.integrate(self.dm)
        send_counts, ws = self.ops.halo_count(self.dm, self.bounds, self.world, self.rank)
        ptrs, offsets, recv_counts, recv = self.exchange.prepare(send_counts, dev)
        self.ops.halo_send(self.dm, ke, self.bounds, self.world, self.rank, ptrs, offsets, ws)
        self.exchange.barrier(dev)
        self._pending = (ke, rows, cols, fail)
        return self.phase_assemble(recv, recv_counts)

    def global_nnz(self) -> int:
        nnzs = self.exchange.allgather_int(int(self.last.row_idx.shape[0]), self.last.row_idx.device)
        self.last.nnz_offset = int(sum(nnzs[:self.rank]))
        return int(sum(nnzs))

    # -- benchmark helpers --
    def stage_times(self, repeats=3):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        acc = {"ke_ms": 0.0, "halo_exchange_ms": 0.0, "assembly_ms": 0.0}
        for _ in range(repeats):
            ev[0].record()
            ke, rows, cols, fail = self.ops.integrate(self.dm)
            ev[1].record()
            if isinstance(self.exchange, P2PExchange):
                dev = self.ops.device
                send_counts, ws = self.ops.halo_count(self.dm, self.bounds, self.world, self.rank)
                ptrs, offsets, recv_counts, recv = self.exchange.prepare(send_counts, dev)
                self.ops.halo_send(self.dm, ke, self.bounds, self.world, self.rank, ptrs, offsets, ws)
                self.exchange.barrier(dev)
            else:
                records, send_counts = self.ops.halo(self.dm, ke, self.bounds, self.world, self.rank)
                dev = records.device
                recv_counts = self.exchange.counts(torch.tensor(send_counts, dtype=torch.int64,
                                                                device=dev)).cpu().tolist()
                recv = self.exchange.records(records, send_counts, recv_counts)
            ev[2].record()
            self._pending = (ke, rows, cols, fail)
            self.phase_assemble(recv, recv_counts)
            ev[3].record()
            torch.cuda.synchronize()
            acc["ke_ms"] += ev[0].elapsed_time(ev[1]) / repeats
            acc["halo_exchange_ms"] += ev[1].elapsed_time(ev[2]) / repeats
            acc["assembly_ms"] += ev[2].elapsed_time(ev[3]) / repeats
        acc["launches_per_step"] = 7 + 5  # single-GPU set + halo count/scan(2)/totals/pack
        return acc

    def measure_e2e(self, steps, barrier):
        """Host shard in (pinned) -> build -> host CSC block (reference dtypes), pipelined like the
        single-GPU e2e (transfer.CscHostTransfer: int32 rows over PCIe, widened on the host while
        the next step builds); host clock per rank, max over ranks."""
        import time

        import torch.distributed as dist

        from .transfer import CscHostTransfer, host_threads

        D = self.ops.D
        h = [t.cpu().pin_memory() for t in (self.dm.coords, self.dm.conn, self.dm.coeff)]
        self.step()
        nnz = int(self.last.row_idx.shape[0])
        dev = self.ops.device
        keep = self.dm
        ncols = self.c_hi - self.c_lo
        # the ranks of one node share its cores (and host memory bandwidth) for the widening
        xfer = CscHostTransfer(ncols, nnz, depth=2, device=dev,
                               threads=max(1, host_threads() // (2 * max(1, self.world))))
        futures = []

        def one():
            self.dm = D.DeviceMesh(*(t.to(dev, non_blocking=True) for t in h))
            r = self.step()
            futures.append(xfer.submit(D.DeviceCsc(r.col_ptr, r.row_idx, r.vals, ncols, self.c_lo)))

        def drain():
            for f in futures:
                f.result()
            futures.clear()
            torch.cuda.synchronize()

        one()
        drain()
        barrier()
        t0 = time.perf_counter()
        for _ in range(steps):
            one()
        drain()
        ms = torch.tensor([(time.perf_counter() - t0) * 1e3 / steps], dtype=torch.float64, device=dev)
        xfer.close()
        all_reduce(ms, op=dist.ReduceOp.MAX)
        self.dm = keep
        h2d = sum(t.numel() * t.element_size() for t in h)
        d2h = xfer.bytes_per_transfer(nnz)
        tot = torch.tensor([h2d, d2h], dtype=torch.int64, device=dev)
        all_reduce(tot)
        return {"value": self.n_el / (float(ms.item()) / 1e3), "unit": "elements/s",
                "h2d_bytes_per_step": int(tot[0]), "d2h_bytes_per_step": int(tot[1]),
                "ms_per_step": float(ms.item()), "steps": steps,
                "pipelined": "step i's D2H (+ host widening) overlaps step i+1's H2D + build",
                "api": "per-rank shard (pinned host -> HBM) + ShardedBuild.step + transfer.CscHostTransfer -> host CSC block"}


# ------------------------------------------------------------------------------------------
# loopback: G virtual ranks in one process (tests the CUDA sharded path on one GPU)
# ------------------------------------------------------------------------------------------
class LoopbackExchange:
    def allgather_int(self, value, device):
        raise NotImplementedError("use run_loopback")


def run_loopback(mesh, world: int, ops_factory):
    """Run all G ranks' phases in one process; returns the list of ShardResult (rank order)."""
    ranks = [ShardedBuild(mesh, r, world, ops=ops_factory(), exchange=LoopbackExchange()) for r in range(world)]
    sends = [rk.phase_local() for rk in ranks]
    results = []
    for r, rk in enumerate(ranks):
        parts, recv_counts = [], []
        for s, (records, counts) in enumerate(sends):
            off = int(sum(counts[:r]))
            parts.append(records[off:off + counts[r]])
            recv_counts.append(int(counts[r]))
        recv = torch.cat(parts) if parts else sends[r][0][:0]
        results.append(rk.phase_assemble(recv, recv_counts))
    off = 0
    for res in results:
        res.nnz_offset = off
        off += int(res.row_idx.shape[0])
    return results


def run_loopback_p2p(mesh, world: int, ops_factory):
    """G virtual ranks in one process with the fused pack-and-send: each rank's hx_halo_send writes
    into the other ranks' receive buffers (local memory here, peer memory across GPUs)."""
    ranks = [ShardedBuild(mesh, r, world, ops=ops_factory(), exchange=LoopbackExchange()) for r in range(world)]
    local = []
    C = np.zeros((world, world), dtype=np.int64)
    for r, rk in enumerate(ranks):
        ke, rows, cols, fail = rk.ops.integrate(rk.dm)
        counts, ws = rk.ops.halo_count(rk.dm, rk.bounds, world, r)
        C[r] = counts
        local.append((ke, rows, cols, fail, ws))
    dev = ranks[0].ops.device
    bufs = [torch.full((max(int(C[:, d].sum()), 1), RECORD_DOUBLES), float("nan"), dtype=torch.float64, device=dev)
            for d in range(world)]
    ptrs = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device=dev)
    for r, rk in enumerate(ranks):
        offsets = torch.tensor([int(C[:r, d].sum()) for d in range(world)], dtype=torch.int64, device=dev)
        ke, _, _, _, ws = local[r]
        rk.ops.halo_send(rk.dm, ke, rk.bounds, world, r, ptrs, offsets, ws)
    results = []
    for r, rk in enumerate(ranks):
        ke, rows, cols, fail, _ = local[r]
        rk._pending = (ke, rows, cols, fail)
        recv_counts = [int(C[s][r]) for s in range(world)]
        results.append(rk.phase_assemble(bufs[r][:sum(recv_counts)], recv_counts))
    off = 0
    for res in results:
        res.nnz_offset = off
        off += int(res.row_idx.shape[0])
    return results


def concat_blocks(results):
    """Global (col_ptr, row_idx, vals) from the rank blocks (host numpy)."""
    col_ptr = [np.zeros(1, dtype=np.int64)]
    rows, vals = [], []
    for res in results:
        cp = res.col_ptr.cpu().numpy()
        col_ptr.append(cp[1:] + res.nnz_offset)
        rows.append(res.row_idx.cpu().numpy())
        vals.append(res.vals.cpu().numpy())
    return np.concatenate(col_ptr), np.concatenate(rows), np.concatenate(vals)
