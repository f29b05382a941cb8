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

__all__ = ["CscHostTransfer", "host_threads", "fetch_csc"]


def host_threads() -> int:
    """Host cores this process may use (the widening pass runs one thread per core)."""
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:  # pragma: no cover - non-Linux
        return max(1, os.cpu_count() or 1)


class _Slot:
    def __init__(self, n_cols: int, nnz: int):
        self.col_ptr = torch.empty(n_cols + 1, dtype=torch.int64, pin_memory=True)
        self.vals = torch.empty(max(nnz, 1), dtype=torch.float64, pin_memory=True)
        self.rows32 = torch.empty(max(nnz, 1), dtype=torch.int32, pin_memory=True)
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
        self.slots = [_Slot(self.n_cols, self.capacity) for _ in range(depth)]
        self.copy = torch.cuda.Stream(device=self.dev)
        self.pool = ThreadPoolExecutor(max_workers=depth)
        self.k = 0
        self.trace = [] if os.environ.get("HX_TRACE_TRANSFER") else None

    def bytes_per_transfer(self, nnz: int) -> int:
        """PCIe bytes of one transfer: col_ptr int64 + row indices int32 + values float64."""
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
