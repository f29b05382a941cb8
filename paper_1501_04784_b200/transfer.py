"""Device lower CSC -> host ``LowerCscMatrix`` with the reference's dtypes (assemble.py:51-62: int64
col_ptr / row_idx, float64 vals), pipelined for back-to-back builds.

PCIe (~57 GB/s device -> host) bounds the end-to-end build of a large mesh: its 16-byte entries
are ~14.9 GB at 400^3.  Row indices are node ids (int32 in the reference's meshes), so they cross
as int32 (``hx_rows_narrow`` on the device) and are sign-extended back to int64 on the host by all
host cores (``hx_rows_widen``) while the next build's transfers run: 12 bytes per entry cross the
bus.  Values and col_ptr cross unchanged into pinned buffers.

A ``CscHostTransfer`` owns ``depth`` result slots (pinned values / col_ptr / int32 rows, a host
int64 row array); ``submit`` enqueues the copies of a device CSC on a copy stream ordered after the
producing stream and returns a future of the host matrix, whose arrays stay valid until the slot
is reused ``depth`` submissions later.
"""

from __future__ import annotations

import os
import time
from concurrent.futures import Future, ThreadPoolExecutor

import numpy as np
import torch

from . import _native as N
from . import device as D
from .assemble import LowerCscMatrix

__all__ = ["CscHostTransfer", "host_threads", "fetch_csc", "RowEncoder", "decode_rows", "row_codec_enabled"]


def row_codec_enabled() -> bool:
    """Row indices cross PCIe delta-encoded (hx_rows_encode / hx_rows_decode) unless HX_ROW_CODEC=0
    (then as int32, widened on the host)."""
    return os.environ.get("HX_ROW_CODEC", "1") != "0"


class RowEncoder:
    """Device half of the row-index codec with reusable buffers: encode(col_ptr, row_idx, col_lo)
    launches hx_rows_encode on ``stream`` and returns (counts u8, lens u8, stream bytes u8, total
    int64 (1,)) device tensors; total is -1 when a column is outside the codec."""

    def __init__(self, device=None):
        self.dev = D.require_device(device)
        self._bufs = {}

    def _buf(self, name, n, dtype):
        b = self._bufs.get(name)
        if b is None or b.numel() < n:
            b = self._bufs[name] = torch.empty(max(int(n * 1.05), 16), dtype=dtype, device=self.dev)
        return b[:n]

    def encode(self, col_ptr: torch.Tensor, row_idx: torch.Tensor, col_lo: int, stream=None):
        ncols = col_ptr.shape[0] - 1
        nnz = row_idx.shape[0]
        counts = self._buf("counts", max(ncols, 1), torch.uint8)
        lens = self._buf("lens", max(ncols, 1), torch.uint8)
        cap = 5 * nnz + 17 * ncols
        data = self._buf("bytes", max(cap, 1), torch.uint8)
        total = self._buf("total", 1, torch.int64)
        ws_bytes = N.lib().hx_rows_encode_workspace_bytes(ncols)
        ws = self._buf("ws", max(ws_bytes, 1), torch.uint8)
        N.check(N.lib().hx_rows_encode(D._ptr(col_ptr), D._ptr(row_idx), ncols, col_lo, D._ptr(counts), D._ptr(lens),
                                       D._ptr(data), cap, D._ptr(total), D._ptr(ws), ws_bytes,
                                       D.stream_handle(stream)), "hx_rows_encode")
        return counts[:ncols], lens[:ncols], data, total


def decode_rows(counts: np.ndarray, lens: np.ndarray, data: np.ndarray, nbytes: int, col_lo: int, row_base: int,
                col_ptr_out: np.ndarray, rows_out: np.ndarray, threads: int) -> None:
    """Host half (hx_rows_decode): int64 rows into rows_out and col_ptr ends (row_base + running
    count) into col_ptr_out; ``data`` must hold 16 readable bytes past nbytes."""
    ncols = counts.shape[0]
    if ncols == 0:
        return
    N.check(N.lib().hx_rows_decode(counts.ctypes.data, lens.ctypes.data, data.ctypes.data, int(nbytes), ncols,
                                   int(col_lo), int(row_base), col_ptr_out.ctypes.data,
                                   rows_out.ctypes.data if rows_out.size else 0, int(threads)),
            "hx_rows_decode")


def host_threads() -> int:
    """Host cores this process may use (the widening pass runs one thread per core)."""
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:  # pragma: no cover - non-Linux
        return max(1, os.cpu_count() or 1)


class _Slot:
    def __init__(self, n_cols: int, nnz: int, codec: bool = False, device=None):
        self.col_ptr = torch.empty(n_cols + 1, dtype=torch.int64, pin_memory=True)
        self.vals = torch.empty(max(nnz, 1), dtype=torch.float64, pin_memory=True)
        self.rows32 = torch.empty(max(nnz, 1), dtype=torch.int32, pin_memory=True)
        if codec:  # delta-encoded rows: per-column counts / lengths + the byte stream (16 B read slack)
            self.enc = RowEncoder(device)
            self.counts = torch.empty(max(n_cols, 1), dtype=torch.uint8, pin_memory=True)
            self.lens = torch.empty(max(n_cols, 1), dtype=torch.uint8, pin_memory=True)
            self.bytes = torch.empty(3 * max(nnz, 1) + 64, dtype=torch.uint8, pin_memory=True)
        self.row_idx = np.empty(max(nnz, 1), dtype=np.int64)
        self.row_idx.fill(0)  # fault the pages in now, not inside a timed transfer
        self.pending: Future | None = None


class CscHostTransfer:
    """Pipelined compact transfer of device CSC blocks with a fixed shape (n_cols, nnz capacity)."""

    def __init__(self, n_cols: int, nnz_capacity: int, depth: int = 2, threads: int | None = None,
                 device=None):
        if depth < 1:
            raise ValueError("depth must be at least 1")
        self.dev = D.require_device(device)
        self.n_cols, self.capacity = int(n_cols), int(nnz_capacity)
        if threads is None:  # half the cores: the widening shares host memory bandwidth with the DMA
            threads = int(os.environ.get("HX_WIDEN_THREADS", "0")) or max(1, host_threads() // 2)
        self.threads = int(threads)
        self.codec = row_codec_enabled()
        self.slots = [_Slot(self.n_cols, self.capacity, self.codec, self.dev) for _ in range(depth)]
        self.last_bytes = None  # PCIe bytes of the last transfer
        self.copy = torch.cuda.Stream(device=self.dev)
        self.pool = ThreadPoolExecutor(max_workers=depth)
        self.k = 0
        self.trace = [] if os.environ.get("HX_TRACE_TRANSFER") else None

    def bytes_per_transfer(self, nnz: int) -> int:
        """PCIe bytes of one transfer: the last transfer's when known (codec: counts + lengths + the
        row stream + values), else col_ptr int64 + row indices int32 + values float64."""
        if self.last_bytes is not None:
            return self.last_bytes
        return 8 * (self.n_cols + 1) + 12 * nnz

    def submit(self, csc: D.DeviceCsc, stream=None) -> Future:
        nnz = csc.nnz
        if csc.col_ptr.shape[0] != self.n_cols + 1 or nnz > self.capacity:
            raise ValueError("CSC block does not fit this transfer's buffers")
        slot = self.slots[self.k % len(self.slots)]
        self.k += 1
        if slot.pending is not None:  # its previous result must be finished (widened) first
            slot.pending.result()
        producer = torch.cuda.current_stream(self.dev) if stream is None else stream
        if self.codec:
            fut = self._submit_codec(slot, csc, producer)
            if fut is not None:
                return fut
        rows32 = D.rows_narrow(csc.row_idx, stream=producer)
        ready = producer.record_event()
        self.copy.wait_event(ready)
        with torch.cuda.stream(self.copy):
            started = self.copy.record_event(torch.cuda.Event(enable_timing=self.trace is not None))
            slot.rows32[:nnz].copy_(rows32, non_blocking=True)
            rows_landed = self.copy.record_event(torch.cuda.Event(enable_timing=self.trace is not None))
            slot.vals[:nnz].copy_(csc.vals, non_blocking=True)
            slot.col_ptr.copy_(csc.col_ptr, non_blocking=True)
            done = self.copy.record_event(torch.cuda.Event(enable_timing=self.trace is not None))
            for t in (rows32, csc.row_idx, csc.vals, csc.col_ptr):
                t.record_stream(self.copy)  # keep the device blocks alive until the copies ran
        if csc.readers is not None:  # plan-owned buffers: the next emit into them waits for these copies
            csc.readers.append(done)
        dim, threads = csc.dim, self.threads

        trace, k = self.trace, self.k - 1

        def finish() -> LowerCscMatrix:
            rows_landed.synchronize()
            t0 = time.perf_counter()
            N.check(N.lib().hx_rows_widen(slot.rows32.data_ptr(), slot.row_idx.ctypes.data, nnz, threads),
                    "hx_rows_widen")
            t1 = time.perf_counter()
            done.synchronize()
            if trace is not None:  # (submission, D2H ms on the copy stream, host widening ms)
                trace.append((k, started.elapsed_time(done), (t1 - t0) * 1e3))
            return LowerCscMatrix(col_ptr=slot.col_ptr.numpy(), row_idx=slot.row_idx[:nnz],
                                  vals=slot.vals.numpy()[:nnz], dim=dim)

        self.last_bytes = 8 * (self.n_cols + 1) + 12 * nnz
        slot.pending = self.pool.submit(finish)
        return slot.pending

    def _submit_codec(self, slot, csc, producer):
        """Delta-encoded rows (hx_rows_encode on the producer stream, one status read for the stream
        length); None when a column is outside the codec or the stream outgrows the slot."""
        nnz, n_cols = csc.nnz, self.n_cols
        counts_d, lens_d, bytes_d, total_d = slot.enc.encode(csc.col_ptr, csc.row_idx, csc.col_lo, stream=producer)
        nbytes = D.peek(total_d, stream=producer)[0]
        if nbytes < 0 or nbytes + 16 > slot.bytes.numel():
            return None
        self.copy.wait_event(producer.record_event())
        with torch.cuda.stream(self.copy):
            started = self.copy.record_event(torch.cuda.Event(enable_timing=self.trace is not None))
            slot.counts[:n_cols].copy_(counts_d, non_blocking=True)
            slot.lens[:n_cols].copy_(lens_d, non_blocking=True)
            if nbytes:
                slot.bytes[:nbytes].copy_(bytes_d[:nbytes], non_blocking=True)
            rows_ready = self.copy.record_event()
            slot.vals[:nnz].copy_(csc.vals, non_blocking=True)
            done = self.copy.record_event(torch.cuda.Event(enable_timing=self.trace is not None))
            for t in (counts_d, lens_d, bytes_d, csc.vals):
                t.record_stream(self.copy)
        if csc.readers is not None:
            csc.readers.append(done)
        dim, threads, trace, k = csc.dim, self.threads, self.trace, self.k - 1
        col_lo = csc.col_lo

        def finish() -> LowerCscMatrix:
            rows_ready.synchronize()  # decode while the values are still crossing
            t0 = time.perf_counter()
            slot.col_ptr[0] = 0
            decode_rows(slot.counts.numpy()[:n_cols], slot.lens.numpy()[:n_cols], slot.bytes.numpy(), nbytes, col_lo,
                        0, slot.col_ptr.numpy()[1:], slot.row_idx[:nnz], threads)
            t1 = time.perf_counter()
            done.synchronize()
            if trace is not None:
                trace.append((k, started.elapsed_time(done), (t1 - t0) * 1e3))
            return LowerCscMatrix(col_ptr=slot.col_ptr.numpy(), row_idx=slot.row_idx[:nnz],
                                  vals=slot.vals.numpy()[:nnz], dim=dim)

        self.last_bytes = 2 * n_cols + nbytes + 8 * nnz
        slot.pending = self.pool.submit(finish)
        return slot.pending

    def close(self) -> None:
        for s in self.slots:
            if s.pending is not None:
                s.pending.result()
        self.pool.shutdown()


_COPY_STREAMS: dict = {}


def copy_stream(dev) -> torch.cuda.Stream:
    """The device's host-transfer stream (one per device, shared by fetch_csc and uploads)."""
    key = torch.device(dev).index
    if key not in _COPY_STREAMS:
        _COPY_STREAMS[key] = torch.cuda.Stream(device=dev)
    return _COPY_STREAMS[key]


def fetch_csc(csc: D.DeviceCsc, stream=None, threads: int | None = None, chunk: int = 1 << 25,
              rows_first: bool | None = None) -> LowerCscMatrix:
    """Device lower CSC -> host LowerCscMatrix (reference dtypes) for one synchronous call.

    Row indices cross as int32 (hx_rows_narrow) in chunks interleaved with the value chunks on the
    copy stream; each row chunk is sign-extended to int64 by the host cores (hx_rows_widen) as soon
    as it lands, while the next chunks are in flight, so only the last chunk's widening is exposed.
    Outputs are pinned arrays from torch's caching host allocator (recycled when dropped)."""
    dev = csc.row_idx.device
    producer = torch.cuda.current_stream(dev) if stream is None else stream
    copy = copy_stream(dev)
    n = csc.nnz
    threads = host_threads() if threads is None else int(threads)
    col_ptr = torch.empty(csc.col_ptr.shape[0], dtype=torch.int64, pin_memory=True)
    vals = torch.empty(n, dtype=torch.float64, pin_memory=True)
    row_idx = torch.empty(n, dtype=torch.int64, pin_memory=True)
    rows32 = torch.empty(max(n, 1), dtype=torch.int32, pin_memory=True)
    narrow = D.rows_narrow(csc.row_idx, stream=producer) if n else None
    copy.wait_event(producer.record_event())
    if rows_first is None:
        rows_first = os.environ.get("HX_FETCH_ROWS_FIRST", "0") == "1"
    landed = []
    with torch.cuda.stream(copy):
        col_ptr.copy_(csc.col_ptr, non_blocking=True)
        for lo in range(0, n, chunk):
            hi = min(n, lo + chunk)
            rows32[lo:hi].copy_(narrow[lo:hi], non_blocking=True)
            landed.append((lo, hi, copy.record_event()))
            if not rows_first:
                vals[lo:hi].copy_(csc.vals[lo:hi], non_blocking=True)
        if rows_first:
            vals.copy_(csc.vals, non_blocking=True)
        done = copy.record_event()
        for t in (narrow, csc.row_idx, csc.vals, csc.col_ptr):
            if t is not None:
                t.record_stream(copy)
    if csc.readers is not None:
        csc.readers.append(done)
    base32, base64 = rows32.data_ptr(), row_idx.data_ptr()
    for lo, hi, ev in landed:
        ev.synchronize()
        N.check(N.lib().hx_rows_widen(base32 + 4 * lo, base64 + 8 * lo, hi - lo, threads), "hx_rows_widen")
    done.synchronize()
    return LowerCscMatrix(col_ptr=col_ptr.numpy(), row_idx=row_idx.numpy(), vals=vals.numpy(), dim=csc.dim)
