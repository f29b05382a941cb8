"""Multi-GPU construction: element-range shards, nnz-balanced column blocks, one exchange of
compact element records.

The reference is single-process; the sharded build produces its LowerCscMatrix
(assemble.py:51-62) cut into column blocks, bitwise equal to the single-GPU build.

Rank r of G (one process per GPU, torch.distributed over NCCL):

1. integrates its contiguous element range E_r = [n_el*r/G, n_el*(r+1)/G) -- KE + fused iK/jK,
   exactly the single-GPU kernel on a slice of the mesh;
2. owns the lower-CSC column block C_r = [b_r, b_r+1) (a column block of the lower triangle is a
   row block of K by symmetry).  The bounds cut a global per-column nnz estimate at equal prefix
   sums (``hx_column_weights`` on each rank's elements, one all-reduce of a 64K-bin histogram, the
   same integer cut on every rank): columns are min(node) (assemble.py:86-93), so on a randomly
   numbered mesh low ids own far more lower-triangle entries than high ids and an equal node split
   is off by up to 1.8x;
3. sends every owned element with a node in another rank's block to that rank as a compact record:
   its 8 node ids + only the KE entries whose column the destination owns (entry (i, j) lands in
   column min(g_i, g_j), owned by min(owner(g_i), owner(g_j))).  One all-gather carries the G x G
   (records, values) count matrix and every rank's fail record; one all-to-all (NCCL) moves the
   records -- or, with ``P2PExchange``, the pack kernel writes them straight into the destinations'
   receive buffers (CUDA IPC peer memory over NVLink) and a one-word all-reduce orders the reads;
4. unpacks the received records into 40-word segments and assembles its block from [received from
   lower ranks | own | received from higher ranks], which are in ascending global element order,
   so every duplicate position is summed in the single-GPU order: bitwise equal to G = 1.

The global K is the concatenation of the blocks; global col_ptr = block col_ptr + exclusive scan of
the block nnz (one all-gather of G int64).  ``block_digest`` gives position-keyed checksums whose sum
over the ranks equals the single-GPU build's (the bench's parity check at N > 1).

The collectives are behind a small exchange interface (torch.distributed for NCCL/gloo; the
loopback drivers simulate G ranks in one process) and the per-rank compute behind ``Ops`` (the CUDA
ops by default), so the host logic is tested with gloo on CPU and the CUDA path with the loopback
and multi-process runs on one GPU.
"""

from __future__ import annotations

import contextlib
import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from .errors import MeshValidationError, NodeIndexError

__all__ = ["element_ranges", "column_bounds", "balanced_bounds", "histogram_bins", "ShardedBuild", "TorchExchange",
           "small_h2d", "block_cost_histograms", "touch_weight",
           "P2PExchange", "CudaOps", "run_loopback", "run_loopback_p2p", "RECORD_DOUBLES", "all_reduce", "barrier",
           "digest_words", "concat_blocks", "csc_digest"]

RECORD_DOUBLES = 40  # unpacked record: 36 packed KE values + 8 int32 node ids
FAIL_WORDS = 3       # hx_fail_info as int64 words
MAX_BINS = 1 << 16   # column histogram bins of the balanced bounds


def element_ranges(n_el: int, world: int):
    return [(n_el * r // world, n_el * (r + 1) // world) for r in range(world)]


def column_bounds(n_nodes: int, world: int) -> np.ndarray:
    """Equal node split (the out-of-core build's blocks)."""
    return np.array([n_nodes * r // world for r in range(world + 1)], dtype=np.int64)


def histogram_bins(n_nodes: int) -> int:
    return int(max(1, min(MAX_BINS, n_nodes)))


def balanced_bounds(hist: np.ndarray, n_nodes: int, world: int) -> np.ndarray:
    """Column bounds at equal prefix sums of a per-bin weight histogram (bin b = nodes with
    node * B // n_nodes == b, i.e. starting at ceil(b * n_nodes / B)).  Bound r is the first node
    of the first bin whose exclusive prefix reaches r/G of the total; integer arithmetic only, so
    every rank computes the same bounds from the same all-reduced histogram.  Every block keeps at
    least one column when n_nodes >= world."""
    hist = np.asarray(hist, dtype=np.int64)
    B = hist.shape[0]
    prefix = np.concatenate([[0], np.cumsum(hist)])  # prefix[b] = weight of bins < b
    total = int(prefix[-1])
    bounds = np.zeros(world + 1, dtype=np.int64)
    bounds[world] = n_nodes
    for r in range(1, world):
        if total > 0:
            b = int(np.searchsorted(prefix * world, r * total, side="left"))  # first b: prefix[b]*G >= r*total
            b = min(b, B)
            node = -(-b * n_nodes // B)
        else:
            node = n_nodes * r // world
        bounds[r] = node
    if n_nodes >= world:  # strictly increasing: no empty block
        for r in range(1, world):
            bounds[r] = min(max(bounds[r], bounds[r - 1] + 1), n_nodes - (world - r))
    return bounds


# ------------------------------------------------------------------------------------------
# position-keyed digest (hx_digest restated for the host; test and bench checker)
# ------------------------------------------------------------------------------------------
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _mix(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def digest_words(words: np.ndarray, pos0: int = 0, add: int = 0) -> int:
    """sum_i mix(mix(pos0 + i) ^ (word_i + add)) mod 2^64 over the 8-byte words of ``words``."""
    w = np.ascontiguousarray(words).view(np.uint64)
    pos = np.arange(pos0, pos0 + w.shape[0], dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = _mix(_mix(pos) ^ (w + np.uint64(add & 0xFFFFFFFFFFFFFFFF)))
    return int(np.sum(h, dtype=np.uint64))


def csc_digest(col_ptr, row_idx, vals) -> tuple:
    """(col_ptr, row_idx, vals) digests of a whole lower CSC (host arrays)."""
    return (digest_words(np.asarray(col_ptr, np.int64)), digest_words(np.asarray(row_idx, np.int64)),
            digest_words(np.asarray(vals, np.float64)))


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
    """torch.distributed collectives: NCCL over NVLink on GPUs (device buffers), gloo on CPU (and
    host-staged CUDA buffers when several ranks share one GPU for testing)."""

    p2p = False

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def allgather(self, t: torch.Tensor) -> np.ndarray:
        """All-gather of a 1-D int64 tensor -> host (world, k) array (one host sync)."""
        if t.is_cuda and _host_staged(self.group):
            t = t.cpu()
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return torch.stack(out).cpu().numpy()

    def allgather_async(self, t: torch.Tensor):
        """All-gather of a 1-D int64 tensor whose host copy is read later: returns a callable giving
        the (world, k) host array (it waits only for the collective, not for work enqueued after it
        on the stream -- the host prepares the next launches while the GPU keeps computing)."""
        if not t.is_cuda or _host_staged(self.group):
            out = self.allgather(t)
            return lambda: out
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        host = torch.empty((self.world, t.numel()), dtype=t.dtype, pin_memory=True)
        host.copy_(torch.stack(out), non_blocking=True)
        ev = torch.cuda.current_stream(t.device).record_event()

        def result():
            ev.synchronize()
            return host.numpy()
        return result

    def sum_(self, t: torch.Tensor) -> torch.Tensor:
        return all_reduce(t, group=self.group)

    def alltoall(self, send: torch.Tensor, send_splits, recv_splits) -> torch.Tensor:
        n = int(sum(recv_splits))
        buf = getattr(self, "_recv", None)  # reused across steps (stream-ordered)
        if buf is None or buf.dtype != send.dtype or buf.device != send.device or buf.numel() < n:
            self._recv = buf = torch.empty(max(int(n * 1.05), 1), dtype=send.dtype, device=send.device)
        recv = buf[:n]
        kw = dict(output_split_sizes=[int(x) for x in recv_splits], input_split_sizes=[int(x) for x in send_splits])
        if send.is_cuda and _host_staged(self.group):
            r = torch.empty(recv.shape, dtype=recv.dtype)
            self.dist.all_to_all_single(r, send.cpu(), group=self.group, **kw)
            recv.copy_(r)
        else:
            self.dist.all_to_all_single(recv, send, group=self.group, **kw)
        return recv


class P2PExchange(TorchExchange):
    """The all-to-all done by the producer: every rank maps every other rank's receive buffer and
    hx_halo_pack writes the records straight into them.

    Receive buffers are allocated by the library (``hx_ipc_alloc``: cudaMalloc + IPC handle); the
    handles are all-gathered and opened with ``hx_ipc_open`` in THIS process's device context with
    lazy peer access, so the pack kernel's stores reach another GPU's HBM over NVLink (and the same
    GPU's memory when ranks share a device in tests).  Buffers grow (and every rank re-maps) only
    when a rank needs more room.  Ordering: the count all-gather that precedes the pack is stream-
    ordered after each rank's previous assembly, so no peer overwrites records still being read; a
    one-word all-reduce after the pack orders the receivers' reads after every sender's kernel."""

    p2p = True

    def __init__(self, group=None, device=None):
        super().__init__(group)
        from . import _native as N

        self.N = N
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.own = None        # (ptr, words) of this rank's receive buffer
        self.peers = None      # raw pointers of every rank's buffer as seen from this process
        self.opened = []
        self.ptrs = None       # device int64 array of the peer base pointers

    def _on_device(self):
        return torch.cuda.device(self.device) if self.device.type == "cuda" else contextlib.nullcontext()

    def _sync(self):
        if self.device.type == "cuda":
            torch.cuda.synchronize(self.device)

    def _release(self):
        for p in self.opened:
            self.N.lib().hx_ipc_close(ctypes.c_void_p(p))
        self.opened = []
        if self.own is not None:
            self._sync()
            self.N.lib().hx_ipc_free(ctypes.c_void_p(self.own[0]))
            self.own = None

    def close(self):
        self._release()

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self._release()
        except Exception:
            pass

    def _ensure_capacity(self, need_words: int):
        grow = self.own is None or self.own[1] < need_words
        flag = torch.tensor([1 if grow else 0], dtype=torch.int64,
                            device="cpu" if _host_staged(self.group) else self.device)
        self.dist.all_reduce(flag, op=self.dist.ReduceOp.MAX, group=self.group)
        if int(flag.item()) == 0:
            return
        N = self.N
        for p in self.opened:
            N.check(N.lib().hx_ipc_close(ctypes.c_void_p(p)), "hx_ipc_close")
        self.opened = []
        if grow:
            if self.own is not None:
                self._sync()
                N.check(N.lib().hx_ipc_free(ctypes.c_void_p(self.own[0])), "hx_ipc_free")
                self.own = None
            words = max(need_words + need_words // 4, 1024)
            ptr = ctypes.c_void_p()
            handle = ctypes.create_string_buffer(N.IPC_HANDLE_BYTES)
            with self._on_device():
                N.check(N.lib().hx_ipc_alloc(8 * words, ctypes.byref(ptr), handle), "hx_ipc_alloc")
            self.own = (ptr.value, words, handle.raw)
        metas = [None] * self.world
        self.dist.all_gather_object(metas, self.own[2], group=self.group)
        peers = []
        with self._on_device():
            for r, h in enumerate(metas):
                if r == self.rank:
                    peers.append(self.own[0])
                    continue
                p = ctypes.c_void_p()
                N.check(N.lib().hx_ipc_open(ctypes.create_string_buffer(h, N.IPC_HANDLE_BYTES), ctypes.byref(p)),
                        "hx_ipc_open")
                self.opened.append(p.value)
                peers.append(p.value)
        self.peers = peers
        self.ptrs = torch.tensor(peers, dtype=torch.int64, device=self.device)

    def prepare(self, chunk: np.ndarray):
        """chunk[s, d] = words source s sends to d -> (dest_ptrs, dest_offsets (device int64),
        receive view (int64 words))."""
        need = int(chunk[:, self.rank].sum())
        self._ensure_capacity(need)
        self._staging = getattr(self, "_staging", [])
        offsets = small_h2d(p2p_offsets(chunk, self.rank), self.device, self._staging)
        recv = _words_view(self.own[0], need, self.device)
        return self.ptrs, offsets, recv

    def fence(self):
        """Stream-ordered barrier: the receivers read after every sender's pack kernel."""
        if _host_staged(self.group):
            torch.cuda.synchronize(self.device)
            self.dist.barrier(group=self.group)
        else:
            t = torch.zeros(1, dtype=torch.int32, device=self.device)
            self.dist.all_reduce(t, group=self.group)


def p2p_offsets(chunk: np.ndarray, rank: int) -> list:
    """Where ``rank``'s chunk for each destination d starts in d's receive buffer (words): after
    the chunks of every lower source -- the layout all_to_all_single produces."""
    return [int(chunk[:rank, d].sum()) for d in range(chunk.shape[1])]


def _words_view(ptr: int, words: int, device) -> torch.Tensor:
    """An int64 tensor over raw device memory owned elsewhere (no copy, no ownership)."""
    if words == 0:
        return torch.empty(0, dtype=torch.int64, device=device)

    class _Arr:
        __cuda_array_interface__ = {"shape": (words,), "typestr": "<i8", "data": (ptr, False), "version": 3,
                                    "strides": None}

    return torch.as_tensor(_Arr(), device=device)


def small_h2d(values, device, keep: list | None = None) -> torch.Tensor:
    """A small int64 array on ``device`` without a host sync: staged in pinned memory and copied
    asynchronously (a pageable tensor.to(device) waits for the stream, idling the GPU while the host
    prepares the next launches).  ``keep`` holds the pinned staging tensor until the copy is done
    (the caller's next stream synchronisation)."""
    h = torch.tensor(np.ascontiguousarray(values, dtype=np.int64).reshape(-1), dtype=torch.int64).pin_memory()
    if keep is not None:
        keep.append(h)
        del keep[:-8]
    return h.to(device, non_blocking=True)


# ------------------------------------------------------------------------------------------
# per-rank compute (CUDA)
# ------------------------------------------------------------------------------------------
class CudaOps:
    """The device kernels of libhexfem_b200.so."""

    def __init__(self, device=None, mode="exact"):
        from . import _native as N
        from . import device as D

        self.D, self.N = D, N
        self.device = D.require_device(device)
        self.mode = mode
        self._staging = []  # pinned sources of in-flight small copies (small_h2d)
        self._bufs = {}     # step-to-step scratch (records, workspaces): reused, grown on demand

    def scratch(self, name: str, n: int, dtype) -> torch.Tensor:
        """A reusable device buffer of >= n elements (stream-ordered reuse across steps): the large
        per-step buffers are not re-allocated, so the caching allocator never has to free and
        re-map gigabytes between steps (which synchronises the device)."""
        b = self._bufs.get(name)
        if b is None or b.dtype != dtype or b.numel() < n:
            self._bufs.pop(name, None)
            b = torch.empty(max(int(n * 1.05), 1), dtype=dtype, device=self.device)
            self._bufs[name] = b
        return b[:n]

    def _p(self, t):
        return self.D._ptr(t)

    def _s(self):
        return self.D.stream_handle()

    def upload(self, coords, conn, coeff):
        def up(a, dt):
            return torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(self.device)

        return self.D.DeviceMesh(up(coords, np.float64), up(conn, np.int32), up(coeff, np.float64))

    def integrate(self, dm):
        """-> (ke, rows, cols, fail record (3,) int64 device)"""
        return self.D.integrate_mesh(dm, mode=self.mode)

    def column_weights(self, dm, n_nodes: int, n_bins: int) -> torch.Tensor:
        hist = torch.zeros(n_bins, dtype=torch.int64, device=self.device)
        self.N.check(self.N.lib().hx_column_weights(self._p(dm.conn), dm.n_el, n_nodes, n_bins, self._p(hist),
                                                    self._s()), "hx_column_weights")
        return hist

    def column_touch(self, dm, n_nodes: int, n_bins: int) -> torch.Tensor:
        hist = torch.zeros(n_bins, dtype=torch.int64, device=self.device)
        self.N.check(self.N.lib().hx_column_touch(self._p(dm.conn), dm.n_el, n_nodes, n_bins, self._p(hist),
                                                  self._s()), "hx_column_touch")
        return hist

    def bounds(self, bounds_np):
        return torch.from_numpy(np.ascontiguousarray(bounds_np, dtype=np.int64)).to(self.device)

    def halo_count(self, dm, bounds_dev, world, rank):
        """-> (per_dest (world, 2) int64 device: records, values per destination; workspace)"""
        ws_bytes = self.N.lib().hx_halo_workspace_bytes(dm.n_el, world)
        ws = self.scratch("halo_ws", max(ws_bytes, 1), torch.uint8)
        per_dest = torch.empty((world, 2), dtype=torch.int64, device=self.device)
        self.N.check(self.N.lib().hx_halo_count(self._p(dm.conn), dm.n_el, self._p(bounds_dev), world, rank,
                                                self._p(per_dest), self._p(ws), ws_bytes, self._s()), "hx_halo_count")
        return per_dest, ws

    def alloc_words(self, n: int) -> torch.Tensor:
        """The step's send buffer (reused across steps)."""
        return self.scratch("send", n, torch.int64)

    def halo_pack(self, dm, ke, bounds_dev, world, rank, dest_ptrs, dest_offsets, ws):
        """dest_ptrs: device int64 (world,) base addresses; dest_offsets: device int64 (world,) words."""
        self.N.check(self.N.lib().hx_halo_pack(self._p(dm.conn), self._p(ke), dm.n_el, self._p(bounds_dev), world,
                                               rank, self._p(dest_ptrs), self._p(dest_offsets), self._p(ws),
                                               self._s()), "hx_halo_pack")

    def pointers(self, bases, offsets):
        return (small_h2d([int(b) for b in bases], self.device, self._staging),
                small_h2d([int(o) for o in offsets], self.device, self._staging))

    def halo_unpack(self, recv, src_desc: np.ndarray, bounds_dev, world, rank, n_rec):
        records = self.scratch("records", n_rec * RECORD_DOUBLES, torch.float64).view(n_rec, RECORD_DOUBLES)
        if n_rec == 0:
            return records
        desc = small_h2d(src_desc, self.device, self._staging).reshape(-1, 3)
        ws_bytes = self.N.lib().hx_halo_unpack_workspace_bytes(n_rec)
        ws = self.scratch("unpack_ws", ws_bytes, torch.uint8)
        self.N.check(self.N.lib().hx_halo_unpack(self._p(recv), self._p(desc), world, rank, self._p(bounds_dev), n_rec,
                                                 self._p(records), self._p(ws), ws_bytes, self._s()),
                     "hx_halo_unpack")
        return records

    def halo_index(self, recv, src_desc: np.ndarray, bounds_dev, world, rank, n_rec):
        """The received records as compact element segments (hx_halo_index): their ids as
        connectivity rows, their values left in ``recv`` and addressed per record (first value word,
        owned-entry mask) -- 48 bytes per record written instead of unpacking 320-byte rows."""
        conn = self.scratch("rec_conn", 8 * n_rec, torch.int32).view(n_rec, 8)
        koff = self.scratch("rec_koff", n_rec, torch.int64)
        kmask = self.scratch("rec_kmask", n_rec, torch.int64)
        seg = self.D.CompactSegment(conn, recv.view(torch.float64), koff, kmask)
        if n_rec == 0:
            return seg
        desc = small_h2d(src_desc, self.device, self._staging).reshape(-1, 3)
        ws_bytes = self.N.lib().hx_halo_unpack_workspace_bytes(n_rec)
        ws = self.scratch("unpack_ws", ws_bytes, torch.uint8)
        self.N.check(self.N.lib().hx_halo_index(self._p(recv), self._p(desc), world, rank, self._p(bounds_dev), n_rec,
                                                self._p(conn), self._p(koff), self._p(kmask), self._p(ws), ws_bytes,
                                                self._s()), "hx_halo_index")
        return seg

    def assemble(self, segments, n_nodes, c_lo, c_hi, nnz_hint=None, order="auto"):
        return self.D.mesh_csc(segments, n_nodes, c_lo, c_hi, nnz_hint=nnz_hint, order=order)

    def column_order(self, dm, n_nodes) -> str:
        """Column processing order of this rank's assemblies, decided once (one small reduction)."""
        return "column" if self.D.numbering_is_local(dm.conn, n_nodes) else "element"

    def digest(self, t: torch.Tensor, pos0: int, add: int = 0) -> torch.Tensor:
        """Device u64 (as int64) accumulator of hx_digest over ``t``'s 8-byte words."""
        out = torch.zeros(1, dtype=torch.int64, device=self.device)
        self.N.check(self.N.lib().hx_digest(self._p(t), t.numel() * t.element_size() // 8, pos0,
                                            ctypes.c_uint64(add & 0xFFFFFFFFFFFFFFFF), self._p(out), self._s()),
                     "hx_digest")
        return out


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


def _fail_error(meta: np.ndarray, e_starts, n_nodes):
    """The exception every rank raises: the lowest element with a bad node id, else the lowest
    degenerate element (global ids) over all ranks' fail records (hx_fail_info words)."""
    from .device import fail_error

    best = None
    for r in range(meta.shape[0]):
        err = fail_error(meta[r, :FAIL_WORDS], int(e_starts[r]), n_nodes)
        if err is None:
            continue
        key = (not isinstance(err, NodeIndexError), err.element_id)
        if best is None or key < best[0]:
            best = (key, err)
    return None if best is None else best[1]


def touch_weight() -> float:
    """Weight of the element-touch histogram against the nnz weights in the block cost
    (HX_BALANCE_TOUCH; measured on C5 at G = 8)."""
    import os

    return float(os.environ.get("HX_BALANCE_TOUCH", "4.0"))


def block_cost_histograms(ops, exchange, dm, n_nodes):
    """(nnz histogram, cost histogram) summed over the ranks (one all-reduce of both): cost = nnz
    weights + touch_weight() x element touches, so the cut balances the assembly's per-entry AND
    per-element work (an nnz-only cut gives the wide high-id blocks of a permuted mesh 2.3x the
    records of the low-id ones)."""
    bins = histogram_bins(n_nodes)
    nnz = ops.column_weights(dm, n_nodes, bins)
    lam = touch_weight()
    touch_fn = getattr(ops, "column_touch", None)
    if lam == 0.0 or touch_fn is None:
        nnz = exchange.sum_(nnz)
        h = nnz.cpu().numpy()
        return h, h
    both = exchange.sum_(torch.cat([nnz, touch_fn(dm, n_nodes, bins).to(nnz.device)]))
    h = both.cpu().numpy()
    return h[:bins], h[:bins] + lam * h[bins:]


class ShardedBuild:
    """One rank's share of the global build (see module docstring)."""

    def __init__(self, mesh, rank: int, world: int, mode: str = "exact", ops=None, exchange=None, bounds=None):
        self.rank, self.world = rank, world
        self.ops = ops if ops is not None else CudaOps(mode=mode)
        self.exchange = exchange if exchange is not None else TorchExchange()
        self.n_el, self.n_nodes = mesh.n_el, mesh.n_nodes
        self.ranges = element_ranges(mesh.n_el, world)
        self.e_lo, self.e_hi = self.ranges[rank]
        self.dm = self.ops.upload(mesh.coords, mesh.connectivity[self.e_lo:self.e_hi],
                                  mesh.coefficient[self.e_lo:self.e_hi])
        hist = None
        if bounds is None:
            hist, cost = block_cost_histograms(self.ops, self.exchange, self.dm, self.n_nodes)
            bounds = balanced_bounds(cost, self.n_nodes, world)
        self.bounds_np = np.asarray(bounds, dtype=np.int64)
        self.c_lo, self.c_hi = int(self.bounds_np[rank]), int(self.bounds_np[rank + 1])
        # the block's nnz: estimated from the column-weight histogram (units of 1/8 entry) until the
        # first step measured it; sizes the assembly's buffers so no step re-runs its pattern pass
        self.nnz_hint = None
        if hist is not None:
            h = hist.cpu().numpy() if isinstance(hist, torch.Tensor) else np.asarray(hist)
            nb = h.shape[0]
            b_lo, b_hi = self.c_lo * nb // max(self.n_nodes, 1), max(self.c_hi - 1, 0) * nb // max(self.n_nodes, 1)
            self.nnz_hint = int(1.1 * h[b_lo:b_hi + 1].sum() / 8) + (self.c_hi - self.c_lo)
        order_fn = getattr(self.ops, "column_order", None)
        self.order = order_fn(self.dm, self.n_nodes) if order_fn is not None else "auto"
        self.bounds = self.ops.bounds(self.bounds_np)
        self.last = None
        self.last_index = None
        self.last_counts = None

    # -- phases (so a loopback driver can interleave G ranks in one process) --
    def phase_local(self):
        """Integrate the owned elements and count the records per destination -> the row this
        rank contributes to the metadata all-gather: fail record (3) + (records, values) x G
        (the in-process drivers' single-gather form of step)."""
        ke, rows, cols, fail = self.ops.integrate(self.dm)
        per_dest, ws = self.ops.halo_count(self.dm, self.bounds, self.world, self.rank)
        self._pending = (ke, rows, cols, ws)
        return torch.cat([fail.reshape(-1).to(per_dest.device), per_dest.reshape(-1)])

    def check_meta(self, meta: np.ndarray) -> np.ndarray:
        """Raise the global failure on every rank; -> C (world, world, 2): C[s, d] = (records, values)."""
        err = _fail_error(meta, [lo for lo, _ in self.ranges], self.n_nodes)
        if err is not None:
            self._pending = None
            raise err
        return meta[:, FAIL_WORDS:].reshape(self.world, self.world, 2)

    def pack(self, dest_ptrs, dest_offsets):
        ke, _, _, ws = self._pending
        self.ops.halo_pack(self.dm, ke, self.bounds, self.world, self.rank, dest_ptrs, dest_offsets, ws)

    def phase_assemble(self, recv: torch.Tensor, C: np.ndarray):
        """recv: int64 words, the chunks of every source in ascending source order."""
        ke, rows, cols, _ = self._pending
        self._pending = None
        chunk = 4 * C[:, :, 0] + C[:, :, 1]
        r = self.rank
        desc = np.zeros((self.world, 3), dtype=np.int64)
        desc[:, 0] = np.concatenate([[0], np.cumsum(chunk[:, r])[:-1]])
        desc[:, 1:] = C[:, r, :]
        n_rec = int(C[:, r, 0].sum())
        n_lower = int(C[:r, r, 0].sum())
        segments = []
        if hasattr(self.ops, "halo_index"):  # compact segments over the received words (no unpacking)
            rec = self.ops.halo_index(recv, desc, self.bounds, self.world, r, n_rec)
            lower, upper = (rec.slice(0, n_lower), rec.slice(n_lower, n_rec))
        else:  # CPU stand-ins: 40-word records
            records = self.ops.halo_unpack(recv, desc, self.bounds, self.world, r, n_rec)
            lower, upper = record_segment(records[:n_lower]), record_segment(records[n_lower:])
        if n_lower:
            segments.append(lower)
        segments.append((self.dm.conn, ke))
        if n_rec > n_lower:
            segments.append(upper)
        csc = self.ops.assemble(segments, self.n_nodes, self.c_lo, self.c_hi, nnz_hint=self.nnz_hint, order=self.order)
        self.nnz_hint = int(csc.row_idx.shape[0])  # exact from now on (same mesh every step)
        self.last = ShardResult(csc.col_ptr, csc.row_idx, csc.vals, self.c_lo, self.c_hi)
        self.last_index = (ke, rows, cols)
        self.last_counts = C
        return self.last

    def phase_count(self) -> torch.Tensor:
        """Records / values this rank sends each destination (connectivity only, no KE)."""
        per_dest, ws = self.ops.halo_count(self.dm, self.bounds, self.world, self.rank)
        self._count_ws = ws
        return per_dest.reshape(-1)

    def phase_integrate(self) -> torch.Tensor:
        ke, rows, cols, fail = self.ops.integrate(self.dm)
        self._pending = (ke, rows, cols, self._count_ws)
        return fail.reshape(-1)

    def step(self):
        """One sharded build.  The count all-gather needs only the connectivity, so it runs before
        the integration kernel and the host reads it while the GPU integrates; the fail records
        (one more small all-gather) are checked with the assembly's status read at the end, every
        rank raising the same error for the lowest failing element."""
        async_gather = getattr(self.exchange, "allgather_async", None)
        if async_gather is None:  # in-process drivers / CPU stand-ins: the one-gather form
            return self._step_gathered()
        counts = async_gather(self.phase_count())
        fails = async_gather(self.phase_integrate())
        C = counts().reshape(self.world, self.world, 2)
        err = None
        try:
            res = self._exchange_assemble(C)
        except MeshValidationError as e:  # out-of-range node ids: reported as the element's error below
            err, res = e, None
        meta_fail = fails()
        fe = _fail_error(meta_fail, [lo for lo, _ in self.ranges], self.n_nodes)
        if fe is not None:
            self._pending = None
            raise fe
        if err is not None:
            raise err
        return res

    def _step_gathered(self):
        meta = self.exchange.allgather(self.phase_local())
        C = self.check_meta(meta)
        return self._exchange_assemble(C)

    def _exchange_assemble(self, C):
        chunk = 4 * C[:, :, 0] + C[:, :, 1]
        r = self.rank
        if self.exchange.p2p:
            ptrs, offsets, recv = self.exchange.prepare(chunk)
            self.pack(ptrs, offsets)
            self.exchange.fence()
        else:
            send_splits = chunk[r, :]
            send = self.ops.alloc_words(int(send_splits.sum()))
            offs = np.concatenate([[0], np.cumsum(send_splits)[:-1]])
            ptrs, offsets = self.ops.pointers([send.data_ptr()] * self.world, offs)
            self.pack(ptrs, offsets)
            recv = self.exchange.alltoall(send, send_splits, chunk[:, r])
        return self.phase_assemble(recv, C)

    def global_nnz(self) -> int:
        nnz = torch.tensor([int(self.last.row_idx.shape[0])], dtype=torch.int64, device=self.last.row_idx.device)
        nnzs = self.exchange.allgather(nnz)[:, 0]
        self.last.nnz_offset = int(nnzs[:self.rank].sum())
        return int(nnzs.sum())

    def exchange_bytes(self) -> dict:
        """Bytes of the last step's record exchange over all ranks (wire format: 8-byte words)."""
        C = self.last_counts
        off = ~np.eye(self.world, dtype=bool)
        recs, vals = int(C[:, :, 0][off].sum()), int(C[:, :, 1][off].sum())
        return {"records": recs, "values": vals, "bytes": 8 * (4 * recs + vals),
                "bytes_per_element": 8 * (4 * recs + vals) / max(self.n_el, 1),
                "records_per_element": recs / max(self.n_el, 1)}

    def block_digest(self) -> torch.Tensor:
        """(col_ptr, row_idx, vals) digests of this rank's block at their global positions (call
        global_nnz first); summed over ranks they equal csc_digest of the whole matrix."""
        res, ops = self.last, self.ops
        ncols = self.c_hi - self.c_lo
        d_cp = ops.digest(res.col_ptr[:ncols], self.c_lo, res.nnz_offset)
        if self.rank == self.world - 1:
            d_cp = d_cp + ops.digest(res.col_ptr[ncols:], self.n_nodes, res.nnz_offset)
        return torch.cat([d_cp, ops.digest(res.row_idx, res.nnz_offset), ops.digest(res.vals, res.nnz_offset)])

    # -- benchmark helpers --
    def stage_times(self, repeats=3):
        """Per-stage device times of step() (CUDA events; the exchange includes its host syncs)."""
        acc = {"ke_ms": 0.0, "halo_exchange_ms": 0.0, "assembly_ms": 0.0}
        for _ in range(repeats):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            ev[0].record()
            ke, rows, cols, fail = self.ops.integrate(self.dm)
            ev[1].record()
            per_dest, ws = self.ops.halo_count(self.dm, self.bounds, self.world, self.rank)
            self._pending = (ke, rows, cols, ws)
            meta = self.exchange.allgather(torch.cat([fail.reshape(-1), per_dest.reshape(-1)]))
            C = self.check_meta(meta)
            chunk = 4 * C[:, :, 0] + C[:, :, 1]
            if self.exchange.p2p:
                ptrs, offsets, recv = self.exchange.prepare(chunk)
                self.pack(ptrs, offsets)
                self.exchange.fence()
            else:
                send_splits = chunk[self.rank, :]
                send = self.ops.alloc_words(int(send_splits.sum()))
                offs = np.concatenate([[0], np.cumsum(send_splits)[:-1]])
                ptrs, offsets = self.ops.pointers([send.data_ptr()] * self.world, offs)
                self.pack(ptrs, offsets)
                recv = self.exchange.alltoall(send, send_splits, chunk[:, self.rank])
            ev[2].record()
            self.phase_assemble(recv, C)
            ev[3].record()
            torch.cuda.synchronize()
            acc["ke_ms"] += ev[0].elapsed_time(ev[1]) / repeats
            acc["halo_exchange_ms"] += ev[1].elapsed_time(ev[2]) / repeats
            acc["assembly_ms"] += ev[2].elapsed_time(ev[3]) / repeats
        # integration + fail resolve, halo count (+2 CUB scans x 2 kernels + totals), pack, unpack
        # (count + 2 scan kernels + expand), mesh assembly (adjacency, pattern, scan x2, emit, peek)
        acc["launches_per_step"] = 2 + 6 + 1 + 4 + 6
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
class _LocalSum:
    """The single-process stand-in of the histogram all-reduce."""

    @staticmethod
    def sum_(t):
        return t


class LoopbackExchange:
    """Placeholder exchange of the in-process drivers (they move the chunks themselves)."""

    p2p = False

    def __getattr__(self, name):
        raise NotImplementedError(f"loopback ranks have no collective {name!r}: use run_loopback")


def _loopback_ranks(mesh, world, ops_factory):
    ops0 = ops_factory()
    whole = ops0.upload(mesh.coords, mesh.connectivity, mesh.coefficient)
    _, cost = block_cost_histograms(ops0, _LocalSum(), whole, mesh.n_nodes)
    bounds = balanced_bounds(cost, mesh.n_nodes, world)
    del whole
    ranks = [ShardedBuild(mesh, r, world, ops=ops_factory(), exchange=LoopbackExchange(), bounds=bounds)
             for r in range(world)]
    meta = np.stack([rk.phase_local().cpu().numpy() for rk in ranks])
    C = ranks[0].check_meta(meta)
    return ranks, C, 4 * C[:, :, 0] + C[:, :, 1]


def _finish(ranks, recvs, C):
    results = [rk.phase_assemble(recvs[r], C) for r, rk in enumerate(ranks)]
    off = 0
    for res in results:
        res.nnz_offset = off
        off += int(res.row_idx.shape[0])
    return results


def run_loopback(mesh, world: int, ops_factory):
    """All-to-all layout: each rank packs into its own send buffer, the driver moves the chunks
    like all_to_all_single; returns the ShardResults (rank order)."""
    ranks, C, chunk = _loopback_ranks(mesh, world, ops_factory)
    sends = []
    for r, rk in enumerate(ranks):
        send = rk.ops.alloc_words(int(chunk[r].sum()))
        offs = np.concatenate([[0], np.cumsum(chunk[r])[:-1]])
        rk.pack(*rk.ops.pointers([send.data_ptr()] * world, offs))
        sends.append((send, offs))
    recvs = []
    for d in range(world):
        parts = [sends[s][0][int(sends[s][1][d]):int(sends[s][1][d] + chunk[s, d])] for s in range(world)]
        recvs.append(torch.cat(parts))
    return _finish(ranks, recvs, C)


def run_loopback_p2p(mesh, world: int, ops_factory):
    """Fused pack-and-send layout: every rank's pack kernel writes straight into the destinations'
    receive buffers (local memory here, peer memory across GPUs)."""
    ranks, C, chunk = _loopback_ranks(mesh, world, ops_factory)
    ops = ranks[0].ops
    recvs = [torch.full((max(int(chunk[:, d].sum()), 1),), -1, dtype=torch.int64, device=ops.device)
             for d in range(world)]
    for r, rk in enumerate(ranks):
        offs = p2p_offsets(chunk, r)
        rk.pack(*rk.ops.pointers([b.data_ptr() for b in recvs], offs))
    recvs = [recvs[d][:int(chunk[:, d].sum())] for d in range(world)]
    return _finish(ranks, recvs, C)


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
