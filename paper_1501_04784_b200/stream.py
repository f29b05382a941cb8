"""Streamed column-block build: host mesh -> host LowerCscMatrix with copies in both directions
overlapping the kernels (run_build's in-core path for locally numbered meshes, and its beyond-HBM
path -- Eq. 10 batching, integrate.py:55-81 / PAPER.md:192-199).

The lower CSC is cut into K column blocks [B_k, B_k+1).  On a locally numbered mesh (structured
generators, RCM-ordered inputs) the elements that can hold a block's columns form a short element
range [e_lo(k), e_hi(k)) -- found on the host cores (``hx_block_ranges``) while the coordinates
are in flight.  Block k then runs as

    H2D stream   conn / coeff of range k+1 (pinned host -> HBM)          } PCIe is full duplex:
    main stream  integrate range k, assemble columns of block k           } these three overlap
    D2H stream   block k-1's rows (int32) / values / col_ptr -> pinned    }
    host pool    widen block k-1's rows to int64, shift its col_ptr

so the call costs ~max(H2D, D2H) + one block, instead of H2D + build + D2H.  Elements on a block
boundary are integrated once per block they touch (a halo recompute instead of a halo exchange);
each block sums its duplicates in ascending global element order, so the concatenated blocks are
bitwise the one-shot build (and the reference).

Meshes without locality (the ranges would cover most elements for every block) are left to the
one-shot path: ``plan`` returns None for them.
"""

from __future__ import annotations

import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

from . import _native as N
from . import device as D
from .assemble import LowerCscMatrix
from .errors import MeshValidationError, NodeIndexError
from .transfer import RowEncoder, copy_stream, decode_rows, host_threads, row_codec_enabled

__all__ = ["block_element_ranges", "StreamPlan", "plan", "streamed_build", "blocks_for_budget"]

# a block layout is streamed only when the summed element ranges stay within this factor of n_el
MAX_RANGE_OVERLAP = 1.25


def block_element_ranges(conn: np.ndarray, bounds: np.ndarray, threads: int | None = None):
    """(e_lo, e_hi) int64 (K,) per column block (hx_block_ranges on the host cores)."""
    conn = np.ascontiguousarray(conn, dtype=np.int32)
    bounds = np.ascontiguousarray(bounds, dtype=np.int64)
    k = bounds.shape[0] - 1
    e_lo, e_hi, n_lo, n_hi = (np.zeros(k, dtype=np.int64) for _ in range(4))
    N.check(N.lib().hx_block_ranges_nodes(conn.ctypes.data, conn.shape[0], bounds.ctypes.data, k, e_lo.ctypes.data,
                                          e_hi.ctypes.data, n_lo.ctypes.data, n_hi.ctypes.data,
                                          host_threads() if threads is None else int(threads)),
            "hx_block_ranges_nodes")
    return e_lo, e_hi, n_lo, n_hi


class StreamPlan:
    def __init__(self, bounds, e_lo, e_hi, node_hi=None):
        self.bounds, self.e_lo, self.e_hi = bounds, e_lo, e_hi
        # coordinates block k's element range may gather lie below node_hi[k] (prefix uploads)
        self.node_hi = node_hi

    @property
    def n_blocks(self) -> int:
        return self.bounds.shape[0] - 1

    def max_block_elements(self) -> int:
        return int((self.e_hi - self.e_lo).max()) if self.n_blocks else 0


def stream_bounds(n_nodes: int, n_blocks: int) -> np.ndarray:
    """Column bounds with quarter-size first and last blocks (K >= 3): the copy-out pipeline
    starts after a short first block and ends with a short widening tail."""
    if n_blocks < 3:
        from .distributed import column_bounds

        return column_bounds(n_nodes, n_blocks)
    w = np.array([0.25] + [1.0] * (n_blocks - 2) + [0.25])
    b = np.floor(np.concatenate([[0.0], np.cumsum(w)]) / w.sum() * n_nodes).astype(np.int64)
    b[-1] = n_nodes
    for r in range(1, n_blocks):  # strictly increasing
        b[r] = min(max(b[r], b[r - 1] + 1), n_nodes - (n_blocks - r))
    return b


def looks_local(conn: np.ndarray, n_nodes: int, sample: int = 4096) -> bool:
    """Host-side twin of device.numbering_is_local: sampled elements' node-id spans are a small
    fraction of the id range on locally numbered meshes."""
    n = conn.shape[0]
    if n == 0 or n_nodes < 1 << 16:
        return True
    idx = np.linspace(0, n - 1, min(sample, n)).astype(np.int64)
    rows = np.asarray(conn[idx], dtype=np.int64)
    return float((rows.max(axis=1) - rows.min(axis=1)).mean()) < n_nodes / 64


def plan(mesh, n_blocks: int, threads: int | None = None) -> StreamPlan | None:
    """Column blocks and their element ranges; None when the numbering has no locality."""
    n_nodes, n_el = mesh.n_nodes, mesh.n_el
    n_blocks = int(max(1, min(n_blocks, n_nodes)))
    if not looks_local(mesh.connectivity, n_nodes):
        return None
    bounds = stream_bounds(n_nodes, n_blocks)
    e_lo, e_hi, _, n_hi = block_element_ranges(mesh.connectivity, bounds, threads)
    if n_el and (e_hi - e_lo).sum() > MAX_RANGE_OVERLAP * n_el + n_blocks:
        return None
    return StreamPlan(bounds, e_lo, e_hi, np.maximum.accumulate(np.minimum(n_hi, n_nodes)))


SAMPLE_STEP = 256  # the sampled plan reads every 256th element's connectivity row


def sampled_plan(mesh, n_blocks: int, step: int | None = None, threads: int | None = None) -> StreamPlan | None:
    """A predicted plan from every step-th element (hx_block_ranges_sampled): ~1/step of the host
    scan's reads.  The streamed build checks it on the device (hx_block_verify) and rebuilds with
    the exact plan when an element falls outside it.  None when it does not cover every element or
    the numbering has no locality."""
    n_nodes, n_el = mesh.n_nodes, mesh.n_el
    n_blocks = int(max(1, min(n_blocks, n_nodes)))
    if n_el == 0 or not looks_local(mesh.connectivity, n_nodes):
        return None
    if step is None:  # a few steps of slack per block stay a small fraction of the block
        step = int(max(1, min(SAMPLE_STEP, n_el // (64 * n_blocks))))
    bounds = stream_bounds(n_nodes, n_blocks)
    conn = np.ascontiguousarray(mesh.connectivity, dtype=np.int32)
    e_lo, e_hi, n_hi = (np.zeros(n_blocks, dtype=np.int64) for _ in range(3))
    N.check(N.lib().hx_block_ranges_sampled(conn.ctypes.data, n_el, bounds.ctypes.data, n_blocks, int(step),
                                            e_lo.ctypes.data, e_hi.ctypes.data, n_hi.ctypes.data,
                                            host_threads() if threads is None else int(threads)),
            "hx_block_ranges_sampled")
    spans = sorted((int(a), int(b)) for a, b in zip(e_lo, e_hi) if b > a)
    reach = 0
    for a, b in spans:  # every element must be uploaded (and so checked) by some block
        if a > reach:
            return None
        reach = max(reach, b)
    if reach < n_el or (e_hi - e_lo).sum() > MAX_RANGE_OVERLAP * n_el + n_blocks:
        return None
    sp = StreamPlan(bounds, e_lo, e_hi, np.maximum.accumulate(np.minimum(n_hi, n_nodes)))
    sp.verify = True
    return sp


def blocks_for_budget(n_el: int, n_nodes: int, budget_bytes: int) -> int:
    """Column blocks so that the coordinates plus three blocks in flight (next upload, current
    build, pending copy-out) fit ``budget_bytes`` of HBM: per block ~344 B per element (conn,
    coeff, KE, halo slack) and ~464 B per column (CSC at the rows estimate, symbolic workspace)."""
    free = budget_bytes - 24 * n_nodes
    if free <= 0:
        return max(1, n_nodes)
    return int(max(1, min(n_nodes, -(-3 * (344 * n_el + 464 * n_nodes) // free))))


def _host(a, dtype):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=dtype))


def streamed_build(mesh, sp, mode: str = "exact", device=None, capacity: int | None = None,
                   stats: dict | None = None):
    """Run the streamed build of ``mesh``; returns the host LowerCscMatrix, or None when the mesh
    has no locality or the result outgrows ``capacity`` entries (default: the rows-per-column
    estimate) -- the caller then takes the one-shot path.  ``sp`` is a StreamPlan, or a block
    count: the plan's host scan then runs while the coordinates are in flight.  Raises
    NodeIndexError / DegenerateElementError for the lowest failing element like the one-shot
    build."""
    dev = D.require_device(device)
    n_nodes, n_el = mesh.n_nodes, mesh.n_el
    if not isinstance(sp, StreamPlan) and not looks_local(mesh.connectivity, n_nodes):
        return None
    cap = D.ROWS_PER_COLUMN_ESTIMATE * n_nodes if capacity is None else int(capacity)
    t0 = time.perf_counter()
    with torch.cuda.device(dev):
        main = torch.cuda.current_stream(dev)
        h2d = _h2d_stream(dev)
        d2h = copy_stream(dev)
        coords_h, conn_h, coeff_h = (_host(mesh.coords, np.float64), _host(mesh.connectivity, np.int32),
                                     _host(mesh.coefficient, np.float64))
        h2d.wait_stream(main)
        # buffers written on the H2D stream are allocated on it and marked as used by the main
        # stream, so the caching allocator never hands their memory to the next upload while a
        # kernel still reads it
        with torch.cuda.stream(h2d):
            coords = torch.empty(tuple(coords_h.shape), dtype=torch.float64, device=dev)
        coords.record_stream(main)
        if not isinstance(sp, StreamPlan):  # element and node ranges of the blocks
            k_req = int(sp)
            sp = sampled_plan(mesh, k_req) if os.environ.get("HX_SAMPLED_PLAN", "1") != "0" else None
            if sp is None:
                sp = plan(mesh, k_req)  # the exact host scan
            if sp is None:
                return None
        K = sp.n_blocks
        t_plan = time.perf_counter()
        # the coordinates go up as prefixes just ahead of the blocks that gather them (block 0 starts
        # after its slice instead of after the whole array)
        node_hi = sp.node_hi if sp.node_hi is not None else np.full(K, n_nodes, dtype=np.int64)
        coords_up = [0]
        tops = [n_nodes] * K  # coordinate prefix uploaded when block k computes
        verify = getattr(sp, "verify", False)
        if verify:  # the predicted plan is checked element by element on the device
            vflag = torch.zeros(1, dtype=torch.int32, device=dev)
            v_bounds = torch.from_numpy(np.ascontiguousarray(sp.bounds, dtype=np.int64)).to(dev)
            v_lo = torch.from_numpy(np.ascontiguousarray(sp.e_lo, dtype=np.int64)).to(dev)
            v_hi = torch.from_numpy(np.ascontiguousarray(sp.e_hi, dtype=np.int64)).to(dev)
        out_cp = torch.empty(n_nodes + 1, dtype=torch.int64, pin_memory=True)
        out_rows = torch.empty(max(cap, 1), dtype=torch.int64, pin_memory=True)
        out_vals = torch.empty(max(cap, 1), dtype=torch.float64, pin_memory=True)
        codec = row_codec_enabled()
        if codec:  # delta-encoded rows (~2 bytes per row on local meshes) + per-column counts / lengths
            encs = [RowEncoder(dev), RowEncoder(dev)]  # alternate: block k encodes while k-1 copies out
            enc_done = [None, None]
            counts_h = torch.empty(max(n_nodes, 1), dtype=torch.uint8, pin_memory=True)
            lens_h = torch.empty(max(n_nodes, 1), dtype=torch.uint8, pin_memory=True)
            bytes_h = torch.empty(3 * max(cap, 1) + 64, dtype=torch.uint8, pin_memory=True)
            boff = 0
        rows32 = torch.empty(max(cap, 1), dtype=torch.int32, pin_memory=True)
        out_cp[0] = 0
        cp_np = out_cp.numpy()
        # host workers of the row decode / widening: half the cores while copies stream in (they share
        # host memory bandwidth with the DMA), HX_DECODE_THREADS to override
        threads = int(os.environ.get("HX_DECODE_THREADS", "0")) or max(1, host_threads() // 2)
        tail_threads = max(threads, host_threads())  # the last blocks' decode has the host to itself
        pool = ThreadPoolExecutor(max_workers=1)

        def upload(k):
            lo, hi = int(sp.e_lo[k]), int(sp.e_hi[k])
            with torch.cuda.stream(h2d):
                conn = torch.empty((hi - lo, 8), dtype=torch.int32, device=dev)
                coeff = torch.empty(hi - lo, dtype=torch.float64, device=dev)
                mark(f"h2d {k} start", h2d)
                top = int(min(max(node_hi[k], coords_up[0]), n_nodes)) if k < K - 1 else n_nodes
                if top > coords_up[0]:
                    coords[coords_up[0]:top].copy_(coords_h[coords_up[0]:top], non_blocking=True)
                    coords_up[0] = top
                tops[k] = coords_up[0]
                conn.copy_(conn_h[lo:hi], non_blocking=True)
                coeff.copy_(coeff_h[lo:hi], non_blocking=True)
                ev = h2d.record_event()
                mark(f"h2d {k} end", h2d)
            conn.record_stream(main)
            coeff.record_stream(main)
            return conn, coeff, ev

        def finish_codec(k, off, nnz, b0, nbytes, rows_ready, done):
            rows_ready.synchronize()  # decode while the block's values are still crossing
            td = time.perf_counter()
            a, z = int(sp.bounds[k]), int(sp.bounds[k + 1])
            decode_rows(counts_h.numpy()[a:z], lens_h.numpy()[a:z], bytes_h.numpy()[b0:], nbytes, a, off,
                        cp_np[a + 1:z + 1], out_rows.numpy()[off:off + nnz], tail_threads if k >= K - 2 else threads)
            if trace is not None:
                trace.append((f"decode {k} {nnz / 1e6:.0f}M rows {1e3 * (time.perf_counter() - td):.1f} ms", None,
                              time.perf_counter()))
            done.synchronize()

        def finish(k, off, nnz, cp_stage, rows_landed, done):
            rows_landed.synchronize()
            if nnz:
                N.check(N.lib().hx_rows_widen(rows32.data_ptr() + 4 * off, out_rows.data_ptr() + 8 * off, nnz,
                                              threads), "hx_rows_widen")
            done.synchronize()
            a, z = int(sp.bounds[k]), int(sp.bounds[k + 1])
            np.add(cp_stage.numpy()[1:], off, out=cp_np[a + 1:z + 1])

        trace = [] if os.environ.get("HX_TRACE_STREAM") else None

        def mark(name, stream):
            if trace is not None:
                e = torch.cuda.Event(enable_timing=True)
                e.record(stream)
                trace.append((name, e, time.perf_counter()))

        fails, futures, stage_events = [], [], []
        offset = 0
        d2h_bytes, coded_blocks = 0, 0
        t_gpu = [torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)]
        mark("start", main)
        if trace is not None:
            print(f"  plan done at host {1e3 * (t_plan - t0):.2f} ms, buffers at {1e3 * (time.perf_counter() - t0):.2f} ms",
                  flush=True)
        t_gpu[0].record(main)
        pending = upload(0) if K else None
        overflow = False
        try:
            for k in range(K):
                conn, coeff, ready = pending
                if k + 1 < K:
                    pending = upload(k + 1)  # next range in flight while this block computes
                main.wait_event(ready)
                a, z = int(sp.bounds[k]), int(sp.bounds[k + 1])
                if verify and conn.shape[0]:
                    N.check(N.lib().hx_block_verify(D._ptr(conn), conn.shape[0], int(sp.e_lo[k]), n_nodes,
                                                    D._ptr(v_bounds), K, D._ptr(v_lo), D._ptr(v_hi), tops[k],
                                                    D._ptr(vflag), D.stream_handle(main)), "hx_block_verify")
                if conn.shape[0] == 0:
                    cp_np[a + 1:z + 1] = offset
                    continue
                dm = D.DeviceMesh(coords, conn, coeff)
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                ev[0].record(main)
                ke, _, _, fail = D.integrate_mesh(dm, with_index=False, mode=mode, stream=main)
                ev[1].record(main)
                fails.append((int(sp.e_lo[k]), fail))
                try:
                    csc = D.mesh_csc([(conn, ke)], n_nodes, a, z, stream=main, order="column")
                except MeshValidationError:
                    _raise_lowest(fails, n_nodes)
                    raise
                ev[2].record(main)
                stage_events.append(ev)
                nnz = csc.nnz
                if offset + nnz > cap:
                    overflow = True
                    break
                if codec:
                    if enc_done[k & 1] is not None:  # block k-2's copies out of these buffers are done
                        main.wait_event(enc_done[k & 1])
                    counts_d, lens_d, bytes_d, total_d = encs[k & 1].encode(csc.col_ptr, csc.row_idx, a, stream=main)
                    nbytes = D.peek(total_d, stream=main)[0]
                    if 0 <= nbytes and boff + nbytes + 16 <= bytes_h.numel():
                        d2h.wait_event(main.record_event())
                        with torch.cuda.stream(d2h):
                            mark(f"d2h {k} start", d2h)
                            counts_h[a:z].copy_(counts_d, non_blocking=True)
                            lens_h[a:z].copy_(lens_d, non_blocking=True)
                            if nbytes:
                                bytes_h[boff:boff + nbytes].copy_(bytes_d[:nbytes], non_blocking=True)
                            rows_ready = d2h.record_event()
                            if nnz:
                                out_vals[offset:offset + nnz].copy_(csc.vals, non_blocking=True)
                            done = d2h.record_event()
                            mark(f"d2h {k} end", d2h)
                        enc_done[k & 1] = done
                        for t in (counts_d, lens_d, bytes_d, csc.vals):
                            t.record_stream(d2h)
                        futures.append(pool.submit(finish_codec, k, offset, nnz, boff, nbytes, rows_ready, done))
                        d2h_bytes += 2 * (z - a) + nbytes + 8 * nnz
                        coded_blocks += 1
                        boff += nbytes
                        offset += nnz
                        del dm, ke, csc
                        continue
                narrow = D.rows_narrow(csc.row_idx, stream=main) if nnz else None
                cp_stage = torch.empty(z - a + 1, dtype=torch.int64, pin_memory=True)
                d2h.wait_event(main.record_event())
                mark(f"asm {k} done (host)", main)
                with torch.cuda.stream(d2h):
                    mark(f"d2h {k} start", d2h)
                    if nnz:
                        rows32[offset:offset + nnz].copy_(narrow, non_blocking=True)
                    rows_landed = d2h.record_event()
                    if nnz:
                        out_vals[offset:offset + nnz].copy_(csc.vals, non_blocking=True)
                    cp_stage.copy_(csc.col_ptr, non_blocking=True)
                    done = d2h.record_event()
                    mark(f"d2h {k} end", d2h)
                for t in (narrow, csc.row_idx, csc.vals, csc.col_ptr):
                    if t is not None:
                        t.record_stream(d2h)
                futures.append(pool.submit(finish, k, offset, nnz, cp_stage, rows_landed, done))
                d2h_bytes += 8 * (z - a + 1) + 12 * nnz
                offset += nnz
                del dm, ke, csc, narrow
            t_gpu[1].record(main)
            for f in futures:
                f.result()
            torch.cuda.synchronize(dev)
            if trace:
                z = trace[0][1]
                for name, e, th in trace:
                    g = f"{z.elapsed_time(e):8.2f}" if e is not None else "       -"
                    print(f"  {name:24s} gpu {g} ms   host {1e3 * (th - t0):8.2f} ms", flush=True)
                print(f"  total host {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
        finally:
            pool.shutdown(wait=True)
        if overflow:
            return None
        if verify and D.peek(vflag, stream=main)[0] != 0:  # the prediction missed an element: exact plan
            exact = plan(mesh, K)
            if exact is None:
                return None
            if stats is not None:
                stats["sampled_plan_fallback"] = True
            return streamed_build(mesh, exact, mode=mode, device=device, capacity=capacity, stats=stats)
        _raise_lowest(fails, n_nodes)
        if stats is not None:
            stats.update(gpu_s=t_gpu[0].elapsed_time(t_gpu[1]) / 1e3, wall_s=time.perf_counter() - t0, blocks=K,
                         integrated_elements=int((sp.e_hi - sp.e_lo).sum()),
                         integration_s=sum(e[0].elapsed_time(e[1]) for e in stage_events) / 1e3,
                         assembly_s=sum(e[1].elapsed_time(e[2]) for e in stage_events) / 1e3,
                         d2h_bytes=d2h_bytes, h2d_bytes=coords_h.numel() * 8 + conn_h.numel() * 4 + coeff_h.numel() * 8,
                         row_codec_blocks=coded_blocks)
    return LowerCscMatrix(col_ptr=cp_np, row_idx=out_rows.numpy()[:offset], vals=out_vals.numpy()[:offset],
                          dim=n_nodes)


def _raise_lowest(fails, n_nodes):
    best = None
    for lo, f in fails:
        err = D.fail_error(f.cpu().numpy(), lo, n_nodes)
        if err is None:
            continue
        key = (not isinstance(err, NodeIndexError), err.element_id)
        if best is None or key < best[0]:
            best = (key, err)
    if best is not None:
        raise best[1]


_H2D: dict = {}


def _h2d_stream(dev) -> torch.cuda.Stream:
    key = torch.device(dev).index
    if key not in _H2D:
        _H2D[key] = torch.cuda.Stream(device=dev)
    return _H2D[key]
