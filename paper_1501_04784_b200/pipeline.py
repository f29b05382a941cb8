"""Global matrix construction pipeline (mesh -> KE + iK/jK -> lower CSC) on the GPU.

``run_build`` mirrors reference cli.py:38-149 (same signature plus ``integration`` and
``device``, same BuildReport fields); stage times come from CUDA events on the launch stream
instead of perf_counter.  ``build_device`` is the device-resident step the benchmark times:
inputs already in HBM, outputs left in HBM.
"""

from __future__ import annotations

import os

import time
from dataclasses import asdict, dataclass

import numpy as np
import torch

from . import device as D
from .assemble import LowerCscMatrix, csc_to_host
from .errors import ConfigurationError, DegenerateElementError, MeshValidationError, NodeIndexError
from .integrate import plan_batches, required_bytes

__all__ = ["BuildReport", "DeviceBuild", "build_device", "run_build", "build_out_of_core", "device_bytes", "triplet_memory", "csc_memory",
           "memory_saving", "format_mb", "format_percent"]

# sparseio.py:26-38 memory model: 16 B per triplet, 16 B per CSC entry + 8 B per column pointer.
_MB = 10**6


def triplet_memory(nnz_triplet: int) -> float:
    if nnz_triplet < 0:
        raise ValueError("nnz must be non-negative")
    return nnz_triplet * 16 / _MB


def csc_memory(nnz_csc: int, dim: int) -> float:
    if nnz_csc < 0 or dim < 0:
        raise ValueError("nnz and dim must be non-negative")
    return (nnz_csc * 16 + (dim + 1) * 8) / _MB


def memory_saving(triplet_mb: float, csc_mb: float) -> float:
    if not triplet_mb > 0:
        raise ValueError(f"triplet memory must be positive, got {triplet_mb!r}")
    return 1.0 - csc_mb / triplet_mb


def format_mb(mb: float) -> str:
    return f"{mb:.2f}" if mb < 10 else f"{mb:.1f}"


def format_percent(fraction: float) -> str:
    return f"{fraction * 100:.1f}%"


@dataclass(frozen=True)
class BuildReport:
    n_el: int
    n_nodes: int
    nnz_triplet: int
    nnz_csc: int
    nnz_compression: float
    triplet_mb: float
    csc_mb: float
    memory_saving: float
    time_integration_s: float
    time_index_s: float | None
    time_assembly_s: float
    time_total_s: float
    pct_integration: float
    pct_assembly: float
    group_count: int
    workers: int
    mode: str
    assembler: str

    def as_dict(self) -> dict:
        return asdict(self)


@dataclass
class DeviceBuild:
    ke: torch.Tensor          # (n_el, 36) f64
    rows: torch.Tensor | None  # (36 n_el,) i32
    cols: torch.Tensor | None  # (36 n_el,) i32
    csc: D.DeviceCsc
    fails: list | None = None  # hx_fail_info records of the integration launches

    def check(self) -> "DeviceBuild":
        """Raise DegenerateElementError for the lowest failing element (synchronises)."""
        for f in self.fails or []:
            D.raise_if_failed(f)
        return self


_SIDE_STREAMS: dict = {}


def _side_stream(dev) -> torch.cuda.Stream:
    key = torch.device(dev).index
    if key not in _SIDE_STREAMS:
        _SIDE_STREAMS[key] = torch.cuda.Stream(device=dev)
    return _SIDE_STREAMS[key]


def build_device(dm: D.DeviceMesh, mode: str = "exact", with_index: bool = True, ranges=None,
                 ke=None, rows=None, cols=None, stream=None, overlap: bool = False,
                 plan: D.MeshPlan | None = None) -> DeviceBuild:
    """KE (+ fused iK/jK) for every element, then the lower CSC, all in HBM.

    Cold build (no ``plan``, no ``overlap``): the integration kernel also records the node adjacency
    that the assembly's symbolic pass starts from (fixed slots, ``device.new_assembly_prep`` /
    ``hx_integrate_mesh_adjacency``), so the assembly runs pattern + scan + emit only; meshes whose
    elements hold a node at the same local index fall back to the atomic adjacency pass inside
    ``mesh_csc`` (detected on the device).  ``HX_FUSED_ADJACENCY=0`` disables the fusion.

    The symbolic assembly reads only the connectivity, so with ``overlap`` it runs on a side
    stream concurrently with the FP64-bound integration kernel and the emit pass (row indices +
    values, which needs KE) follows on the main stream.  Measured neutral to -1% on B200 (the
    integration kernel occupies the whole register file), so the default is one stream.  ``ranges`` is an optional BatchPlan-style
    list of element groups (each one kernel launch into the same output buffers); results are
    bitwise independent of both.  ``plan`` (device.plan_assembly) reuses a verified symbolic plan of
    the same connectivity: the rebuild is the integration kernel plus one emit pass, no host sync.
    """
    dev = dm.conn.device
    n = dm.n_el
    main = torch.cuda.current_stream(dev) if stream is None else stream
    if ke is None:
        ke = torch.empty((n, 36), dtype=torch.float64, device=dev)
    if with_index:
        rows = torch.empty(36 * n, dtype=torch.int32, device=dev) if rows is None else rows
        cols = torch.empty(36 * n, dtype=torch.int32, device=dev) if cols is None else cols
    cached = plan
    plan = None
    if cached is None and overlap and n > 0:
        side = _side_stream(dev)
        side.wait_stream(main)  # inputs and the buffers below are ordered before the plan
        plan = D.mesh_plan_async(dm.conn, dm.n_nodes, stream=side, order=dm.assembly_order())
        plan_done = side.record_event()
    spans = sorted(ranges or [(0, n)])
    covers = spans[0][0] == 0 and spans[-1][1] == n and all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    # HX_FUSED_EMIT=1 (opt-in, measured slower -- DESIGN.md 4.3): symbolic phase first (fixed-slot
    # adjacency, pattern, scan), then ONE launch that integrates every element and runs each column
    # tile's emit on the same warps once its elements are done (hx_integrate_emit).  A verified plan
    # (warm rebuild) skips the symbolic phase.
    fused_emit = (plan is None and covers and len(spans) == 1 and 0 < n and 8 * n < 2**31 - 1
                  and os.environ.get("HX_FUSED_EMIT", "0") == "1")
    if fused_emit:
        if cached is not None and cached.conn is not dm.conn:
            raise ConfigurationError("the assembly plan belongs to another mesh")
        fplan = cached if cached is not None else D.mesh_plan_async(dm.conn, dm.n_nodes, stream=main,
                                                                     order=dm.assembly_order(), fixed=True)
        fail = D.integrate_emit(dm, fplan, ke, rows if with_index else None, cols if with_index else None,
                                mode=mode, stream=main)
        try:
            csc = D.plan_result(fplan, ke, stream=main)
        except MeshValidationError:  # an out-of-range node id is reported as the element's NodeIndexError
            D.raise_if_failed(fail, n_nodes=dm.n_nodes)
            raise
        if cached is None:  # a planned rebuild stays asynchronous: check the fail record later
            D.raise_if_failed(fail, n_nodes=dm.n_nodes)
        return DeviceBuild(ke, rows if with_index else None, cols if with_index else None, csc, [fail])
    # cold single-stream build: the integration kernel also records the node adjacency (the
    # assembly's first pass), so the connectivity is read once and the atomics hide under FP64 work
    fuse = cached is None and plan is None and covers and 0 < n and 8 * n < 2**31 - 1
    prep = D.new_assembly_prep(dm) if fuse and os.environ.get("HX_FUSED_ADJACENCY", "1") != "0" else None
    fails = []
    for lo, hi in (ranges or [(0, n)]):
        _, _, _, fail = D.integrate_mesh(dm, lo, hi, ke=ke[lo:hi],
                                         rows=rows[36 * lo:36 * hi] if with_index else None,
                                         cols=cols[36 * lo:36 * hi] if with_index else None,
                                         with_index=with_index, mode=mode, stream=main, adjacency=prep)
        fails.append(fail)
    if cached is not None and cached.conn is not dm.conn:
        raise ConfigurationError("the assembly plan belongs to another mesh")
    try:
        if cached is not None:
            csc = D.mesh_emit(cached, ke, stream=main)
        elif plan is not None:
            main.wait_event(plan_done)
            csc = D.mesh_emit(plan, ke, stream=main)
        else:
            csc = D.mesh_csc([(dm.conn, ke)], dm.n_nodes, stream=main, order=dm.assembly_order(), prep=prep)
    except MeshValidationError:
        for f in fails:  # an out-of-range node id is reported as the element's NodeIndexError
            D.raise_if_failed(f, n_nodes=dm.n_nodes)
        raise
    if cached is None:  # a planned rebuild stays asynchronous: check the fail records later
        for f in fails:
            D.raise_if_failed(f, n_nodes=dm.n_nodes)
    return DeviceBuild(ke, rows if with_index else None, cols if with_index else None, csc, fails)


def device_bytes(n_el: int, n_nodes: int, with_index: bool = True) -> int:
    """HBM footprint of an in-core build_device: inputs, KE (+ iK/jK), the CSC output buffers at the
    rows-per-column estimate and the symbolic workspace."""
    inputs = 40 * n_el + 24 * n_nodes
    ke = 288 * n_el + (288 * n_el if with_index else 0)
    csc = 16 * D.ROWS_PER_COLUMN_ESTIMATE * n_nodes + 8 * (n_nodes + 1)
    workspace = 156 * n_nodes
    return inputs + ke + csc + workspace


def build_out_of_core(mesh, n_blocks: int, mode: str = "exact", device=None, return_values: bool = False):
    """Global matrix of a mesh whose build does not fit in HBM (Eq. 10 batching, integrate.py:55-81 /
    PAPER.md:192-199): the lower CSC is built one column block at a time on one GPU.

    Block r = columns [N r / B, N (r+1) / B): its elements (those with a node in the block, selected
    in ascending order on the device) are integrated and assembled, the block is copied to the host
    and its device memory released.  Elements on a block boundary are integrated once per block they
    touch (a halo recompute instead of a halo store).  Duplicates are summed in global element order,
    so the result is bitwise equal to the one-shot build.  Returns (LowerCscMatrix, values or None,
    stage times); values (n_el, 36) come from each element's first block.
    """
    from .distributed import column_bounds

    if n_blocks < 1:
        raise ConfigurationError(f"block count must be at least 1, got {n_blocks}")
    dev = D.require_device(device)
    n_el, n_nodes = mesh.n_el, mesh.n_nodes
    with torch.cuda.device(dev):
        dm = D.DeviceMesh.from_host(mesh, dev)
        bounds = column_bounds(n_nodes, n_blocks)
        ids_buf = torch.empty(max(n_el, 1), dtype=torch.int64, device=dev)
        sel_ws = torch.empty(max(D.N.lib().hx_block_select_workspace_bytes(n_el), 1), dtype=torch.uint8, device=dev)
        col_ptr = np.zeros(n_nodes + 1, dtype=np.int64)
        rows, vals = [], []
        values = np.empty((n_el, 36)) if return_values else None
        done = np.zeros(n_el, dtype=bool) if return_values else None
        order = dm.assembly_order()
        worst = None  # (global element id, gauss point, det) of the lowest failing element
        nnz = 0
        t_int = t_asm = 0.0
        for r in range(n_blocks):
            lo, hi = int(bounds[r]), int(bounds[r + 1])
            ids, conn, coeff = D.block_elements(dm, lo, hi, ids=ids_buf, ws=sel_ws)
            if conn.shape[0] == 0:
                continue
            sub = D.DeviceMesh(dm.coords, conn, coeff)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            ev[0].record()
            ke, _, _, fail = D.integrate_mesh(sub, with_index=False, mode=mode)
            ev[1].record()
            f = fail.cpu().numpy()
            if f[0] >= 0:
                gid = int(ids[int(f[0])].item())
                err = D.fail_error(f, n_nodes=n_nodes)
                err.element_id = gid
                # the lowest bad-node element wins over every degenerate one (hx_fail_info)
                key = (not isinstance(err, NodeIndexError), gid)
                if worst is None or key < worst[0]:
                    worst = (key, err)
                continue
            csc = D.mesh_csc([(conn, ke)], n_nodes, lo, hi, order=order)
            ev[2].record()
            torch.cuda.synchronize(dev)
            t_int += ev[0].elapsed_time(ev[1]) / 1e3
            t_asm += ev[1].elapsed_time(ev[2]) / 1e3
            col_ptr[lo + 1:hi + 1] = csc.col_ptr[1:].cpu().numpy() + nnz
            nnz += csc.nnz
            rows.append(csc.row_idx.cpu().numpy())
            vals.append(csc.vals.cpu().numpy())
            if return_values:
                ids_h = ids.cpu().numpy()
                new = ~done[ids_h]
                values[ids_h[new]] = ke.cpu().numpy()[new]
                done[ids_h] = True
            del ids, conn, coeff, sub, ke, csc
        if worst is not None:
            err = worst[1]
            if isinstance(err, NodeIndexError):
                raise NodeIndexError(element_id=err.element_id, node=err.node, n_nodes=n_nodes)
            raise DegenerateElementError(element_id=err.element_id, gauss_point=err.gauss_point, det=err.det)
        # columns of nodes no element references keep col_ptr flat
        np.maximum.accumulate(col_ptr, out=col_ptr)
    matrix = LowerCscMatrix(col_ptr=col_ptr, row_idx=np.concatenate(rows) if rows else np.empty(0, np.int64),
                            vals=np.concatenate(vals) if vals else np.empty(0), dim=n_nodes)
    return matrix, values, {"time_integration_s": t_int, "time_assembly_s": t_asm, "blocks": n_blocks}


# run_build uploads the connectivity in this many element ranges (meshes of at least
# UPLOAD_RANGES_MIN_ELEMENTS elements), so the integration of range k overlaps the copy of range k+1
UPLOAD_RANGES = 8
UPLOAD_RANGES_MIN_ELEMENTS = 1 << 22
# locally numbered meshes of at least STREAM_MIN_ELEMENTS elements take the streamed column-block
# build (stream.py): STREAM_BLOCKS blocks, copies in both directions overlapping the kernels
# transfer statistics of the last streamed run_build (d2h_bytes, row codec use, stage times)
LAST_RUN_STATS: dict = {}
STREAM_BLOCKS: int | None = None  # None: 10 blocks, 20 from 32M elements (C4: 231 vs 238 ms per call,
                                  # profiles/r02/e2e_knobs_c4.txt)


def stream_blocks(n_el: int) -> int:
    return int(STREAM_BLOCKS) if STREAM_BLOCKS is not None else (20 if n_el >= 1 << 25 else 10)

STREAM_MIN_ELEMENTS = 1 << 22


def _host_tensor(a, dtype):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=dtype))


def upload_overlapped(mesh, dev, chunks: int, stream=None):
    """Host mesh -> DeviceMesh on the copy stream: coordinates first, then the connectivity and
    coefficients in ``chunks`` element ranges, one event per range.  Pinned host arrays (hostmem)
    copy asynchronously, so the integration of range k can start while range k+1 is in flight;
    pageable arrays are staged by the driver (the copy blocks the host).  Returns (dm, [(lo, hi,
    event)]); the consumer stream must wait on each event before reading its range."""
    from .transfer import copy_stream

    main = torch.cuda.current_stream(dev) if stream is None else stream
    n = mesh.n_el
    coords_h, conn_h, coeff_h = (_host_tensor(mesh.coords, np.float64), _host_tensor(mesh.connectivity, np.int32),
                                 _host_tensor(mesh.coefficient, np.float64))
    dm = D.DeviceMesh(torch.empty(tuple(coords_h.shape), dtype=torch.float64, device=dev),
                      torch.empty(tuple(conn_h.shape), dtype=torch.int32, device=dev),
                      torch.empty(tuple(coeff_h.shape), dtype=torch.float64, device=dev))
    copy = copy_stream(dev)
    copy.wait_stream(main)  # the buffers' allocation (and anything the caller queued before)
    parts = []
    with torch.cuda.stream(copy):
        dm.coords.copy_(coords_h, non_blocking=True)
        k = max(1, min(chunks, n))
        for i in range(k):
            lo, hi = n * i // k, n * (i + 1) // k
            dm.conn[lo:hi].copy_(conn_h[lo:hi], non_blocking=True)
            dm.coeff[lo:hi].copy_(coeff_h[lo:hi], non_blocking=True)
            parts.append((lo, hi, copy.record_event()))
        if not parts:
            parts.append((0, 0, copy.record_event()))
    return dm, parts


def run_build(mesh, budget_bytes: int, workers: int = 1, mode: str = "sequential", assembler: str = "direct",
              integration: str = "exact", device=None, device_budget_bytes: int | None = None):
    """cli.py:65-149 run_build on the GPU: integrate and assemble one host mesh, return the host
    (LowerCscMatrix, BuildReport) with the reference's dtypes and report fields.

    One call = mesh upload + KE (+ fused iK/jK and the assembly's node adjacency) + lower CSC +
    transfer back.  The connectivity uploads in element ranges on the copy stream while the
    integration kernel consumes the ranges already in HBM (asynchronous when the mesh is in pinned
    memory, ``hostmem.pinned_mesh``); the CSC returns through ``transfer.fetch_csc`` (int32 rows over
    PCIe, widened on the host cores chunk by chunk while the values are still in flight).  Stage
    times come from CUDA events; the host clock brackets the whole call.

    ``device_budget_bytes``: HBM the build may use.  When the in-core footprint (device_bytes)
    exceeds it, the matrix is built in ceil(footprint / budget) column blocks (build_out_of_core).
    """
    from .transfer import fetch_csc

    if assembler not in ("direct", "triplet"):
        raise ConfigurationError(f"assembler must be 'direct' or 'triplet', got {assembler!r}")
    if mode not in ("sequential", "overlapped"):
        raise ConfigurationError(f"mode must be 'sequential' or 'overlapped', got {mode!r}")
    if workers < 1:
        raise ConfigurationError(f"worker count must be at least 1, got {workers}")
    plan = plan_batches(required_bytes(mesh.n_el), budget_bytes, mesh.n_el)
    dev = D.require_device(device)
    with_index = assembler == "triplet"
    need = device_bytes(mesh.n_el, mesh.n_nodes, with_index=with_index)
    if device_budget_bytes is not None and need > device_budget_bytes:
        return _run_build_blocks(mesh, plan, device_budget_bytes, -(-need // device_budget_bytes), workers, mode,
                                 assembler, integration, dev)
    wall0 = time.perf_counter()
    if mesh.n_el >= STREAM_MIN_ELEMENTS and os.environ.get("HX_STREAMED", "1") != "0":
        from . import stream

        st: dict = {}
        matrix = stream.streamed_build(mesh, stream_blocks(mesh.n_el), mode=integration, device=dev, stats=st)
        LAST_RUN_STATS.clear()
        LAST_RUN_STATS.update(st)
        if matrix is not None:
            return matrix, _report(mesh, matrix, plan, st["integration_s"], st["assembly_s"],
                                   time.perf_counter() - wall0, workers, mode, assembler)
    with torch.cuda.device(dev):
        main = torch.cuda.current_stream(dev)
        n = mesh.n_el
        # upload ranges: enough to overlap the connectivity copy with the integration kernel
        chunks = UPLOAD_RANGES if n >= UPLOAD_RANGES_MIN_ELEMENTS else 1
        dm, parts = upload_overlapped(mesh, dev, chunks, stream=main)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ke = torch.empty((n, 36), dtype=torch.float64, device=dev)
        rows = torch.empty(36 * n, dtype=torch.int32, device=dev) if with_index else None
        cols = torch.empty(36 * n, dtype=torch.int32, device=dev) if with_index else None
        fuse = 0 < n and 8 * n < 2**31 - 1 and os.environ.get("HX_FUSED_ADJACENCY", "1") != "0"
        prep = D.new_assembly_prep(dm) if fuse else None
        main.wait_event(parts[0][2])  # the coordinates (and the first range)
        ev[0].record(main)
        fails = []
        for lo, hi, landed in parts:
            main.wait_event(landed)
            if hi > lo:
                _, _, _, fail = D.integrate_mesh(dm, lo, hi, ke=ke[lo:hi],
                                                 rows=rows[36 * lo:36 * hi] if with_index else None,
                                                 cols=cols[36 * lo:36 * hi] if with_index else None,
                                                 with_index=with_index, mode=integration, stream=main,
                                                 adjacency=prep)
                fails.append(fail)
        ev[1].record(main)
        try:
            csc = D.mesh_csc([(dm.conn, ke)], dm.n_nodes, stream=main, order=dm.assembly_order(), prep=prep)
        except MeshValidationError:
            for f in fails:  # an out-of-range node id is the element's NodeIndexError
                D.raise_if_failed(f, n_nodes=dm.n_nodes)
            raise
        for f in fails:
            D.raise_if_failed(f, n_nodes=dm.n_nodes)
        ev[2].record(main)
        matrix: LowerCscMatrix = fetch_csc(csc, stream=main)
        time_integration = ev[0].elapsed_time(ev[1]) / 1e3
        time_assembly = ev[1].elapsed_time(ev[2]) / 1e3
        del dm, ke, rows, cols, csc, prep
    return matrix, _report(mesh, matrix, plan, time_integration, time_assembly, time.perf_counter() - wall0,
                           workers, mode, assembler)


def _report(mesh, matrix, plan, time_integration, time_assembly, time_total, workers, mode, assembler):
    nnz_triplet = 36 * mesh.n_el
    trip_mb = triplet_memory(nnz_triplet)
    matrix_mb = csc_memory(matrix.nnz, matrix.dim)
    stage_sum = time_integration + time_assembly
    pct_integration = 100.0 * time_integration / stage_sum if stage_sum > 0 else 100.0
    return BuildReport(
        n_el=mesh.n_el, n_nodes=mesh.n_nodes, nnz_triplet=nnz_triplet, nnz_csc=matrix.nnz,
        nnz_compression=1.0 - matrix.nnz / nnz_triplet, triplet_mb=trip_mb, csc_mb=matrix_mb,
        memory_saving=memory_saving(trip_mb, matrix_mb), time_integration_s=time_integration,
        # iK/jK are produced inside the integration kernel (fused), so no separate index stage.
        time_index_s=0.0 if assembler == "triplet" else None,
        time_assembly_s=time_assembly, time_total_s=time_total, pct_integration=pct_integration,
        pct_assembly=100.0 - pct_integration, group_count=plan.group_count, workers=workers, mode=mode,
        assembler=assembler)


def _run_build_blocks(mesh, plan, budget, n_blocks, workers, mode, assembler, integration, dev):
    """Beyond the HBM budget: the streamed column-block build when the numbering is local (blocks
    sized for three in flight, copies overlapped), else build_out_of_core's per-block selection."""
    from . import stream

    wall0 = time.perf_counter()
    st: dict = {}
    matrix = stream.streamed_build(mesh, max(3, stream.blocks_for_budget(mesh.n_el, mesh.n_nodes, budget)),
                                   mode=integration, device=dev, stats=st)
    if matrix is not None:
        return matrix, _report(mesh, matrix, plan, st["integration_s"], st["assembly_s"],
                               time.perf_counter() - wall0, workers, mode, assembler)
    matrix, _, st = build_out_of_core(mesh, int(min(n_blocks, max(mesh.n_nodes, 1))), mode=integration, device=dev)
    return matrix, _report(mesh, matrix, plan, st["time_integration_s"], st["time_assembly_s"],
                           time.perf_counter() - wall0, workers, mode, assembler)


def host_csc_equal(a: LowerCscMatrix, b: LowerCscMatrix) -> bool:
    return (a.dim == b.dim and np.array_equal(a.col_ptr, b.col_ptr) and np.array_equal(a.row_idx, b.row_idx)
            and np.array_equal(a.vals.view(np.uint64), b.vals.view(np.uint64)))
