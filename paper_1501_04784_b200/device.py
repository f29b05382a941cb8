"""Device-resident hot path: torch CUDA tensors in, torch CUDA tensors out.

Torch is plumbing here (device memory from its caching allocator, the current stream); every
compute step is a call into libhexfem_b200.so.  The host-facing API in element.py /
integrate.py / assemble.py / pipeline.py is built on these functions.
"""

from __future__ import annotations

import ctypes
import os
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .errors import ConfigurationError, DegenerateElementError, MeshValidationError, NativeLibraryError, NodeIndexError

__all__ = [
    "DeviceMesh", "DeviceCsc", "CompactSegment", "AssemblyPrep", "new_assembly_prep", "rows_narrow", "require_device", "stream_handle", "integrate_mesh", "stiffness_batch",
    "connectivity_index_arrays", "dof_index_arrays", "assemble_dof", "raise_if_failed", "mesh_csc", "triplet_csc", "MeshPlan", "mesh_plan_async",
    "mesh_emit", "integrate_emit", "plan_result", "plan_assembly", "block_elements", "generate_cube_mesh",
]

_FAIL_WORDS = 3  # hx_fail_info = {int64 element, int32 gp, int32 pad, double det} = 24 bytes


def require_device(device=None) -> torch.device:
    """The CUDA device to run on; raises (no CPU fallback) when there is none."""
    N.lib()
    if not torch.cuda.is_available():
        raise NativeLibraryError("hexfem_b200 needs a CUDA device (B200, sm_100a); none is available")
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    if dev.type != "cuda":
        raise ConfigurationError(f"hexfem_b200 runs on CUDA devices only, got {dev}")
    return dev


def stream_handle(stream=None) -> ctypes.c_void_p:
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _check_tensor(t, dtype, shape, name):
    if not isinstance(t, torch.Tensor) or t.device.type != "cuda":
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


@dataclass
class DeviceMesh:
    """Mesh arrays resident in HBM: coords (n_nodes,3) f64, conn (n_el,8) i32, coeff (n_el,) f64."""

    coords: torch.Tensor
    conn: torch.Tensor
    coeff: torch.Tensor

    @property
    def n_nodes(self) -> int:
        return self.coords.shape[0]

    @property
    def n_el(self) -> int:
        return self.conn.shape[0]

    @classmethod
    def from_host(cls, mesh, device=None, non_blocking: bool = False) -> "DeviceMesh":
        dev = require_device(device)

        def up(a, dt):
            t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a, dtype=dt))
            return t.to(dev, non_blocking=non_blocking)

        return cls(up(mesh.coords, np.float64), up(mesh.connectivity, np.int32), up(mesh.coefficient, np.float64))

    def h2d_bytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in (self.coords, self.conn, self.coeff))

    def assembly_order(self) -> str:
        """Column processing order for this mesh's assembly ("column" or "element"), decided once
        per mesh by numbering_is_local (one small device reduction + host read)."""
        if getattr(self, "_order", None) is None:
            self._order = "column" if numbering_is_local(self.conn, self.n_nodes) else "element"
        return self._order


def generate_cube_mesh(spec, device=None, stream=None) -> DeviceMesh:
    """mesh.py:73-98 generate_cube_mesh straight into HBM (hx_generate_cube_mesh): bitwise the
    reference generator's coords / connectivity / coefficient, without the host arrays or the copy."""
    dev = require_device(device)
    nx, ny, nz = int(spec.nx), int(spec.ny), int(spec.nz)
    n_nodes, n_el = (nx + 1) * (ny + 1) * (nz + 1), nx * ny * nz
    coords = torch.empty((n_nodes, 3), dtype=torch.float64, device=dev)
    conn = torch.empty((n_el, 8), dtype=torch.int32, device=dev)
    coeff = torch.empty(n_el, dtype=torch.float64, device=dev)
    N.check(N.lib().hx_generate_cube_mesh(nx, ny, nz, float(spec.h), float(spec.c0), _ptr(coords), _ptr(conn),
                                          _ptr(coeff), stream_handle(stream)), "hx_generate_cube_mesh")
    return DeviceMesh(coords, conn, coeff)


def new_fail_record(device) -> torch.Tensor:
    return torch.empty(_FAIL_WORDS, dtype=torch.int64, device=device)


_PEEK = {}
_PEEK_LOCK = threading.Lock()


def peek(*words: torch.Tensor, stream=None) -> list:
    """Synchronising read of up to 8 small device words (one-element int32 / int64 tensors; int32
    comes back sign-extended) through hx_peek: a kernel writes them into mapped pinned host memory,
    so the read does not wait behind bulk copies queued on the copy engines (the previous build's
    result streaming to the host).  Synchronises ``stream`` (default: the current stream)."""
    if not 0 < len(words) <= N.PEEK_MAX:
        raise ValueError("peek reads 1..8 words")
    if os.environ.get("HX_PEEK", "1") == "0":  # plain copies (they queue on the copy engines)
        return [int(w.reshape(()).to(torch.int64).item()) for w in words]
    dev = words[0].device
    s = torch.cuda.current_stream(dev) if stream is None else stream
    args = N.HxPeekArgs()
    args.n = len(words)
    for i, w in enumerate(words):
        if w.device != dev or w.numel() != 1 or w.element_size() not in (4, 8):
            raise ValueError("peek words must be one-element 4- or 8-byte tensors on one device")
        args.src[i] = w.data_ptr()
        args.bytes[i] = w.element_size()
    with _PEEK_LOCK:
        buf = _PEEK.get(dev.index)
        if buf is None:
            buf = _PEEK[dev.index] = torch.zeros(N.PEEK_MAX, dtype=torch.int64, pin_memory=True)
        N.check(N.lib().hx_peek(ctypes.byref(args), ctypes.c_void_p(buf.data_ptr()), ctypes.c_void_p(s.cuda_stream)),
                "hx_peek")
        s.synchronize()
        return [int(v) for v in buf.numpy()[:len(words)]]


FAIL_BAD_NODE = -2  # hx_fail_info.gauss_point of an element with a node id outside [0, n_nodes)


def fail_error(host: np.ndarray, element_offset: int = 0, n_nodes: int | None = None):
    """The exception an hx_fail_info record (3 int64 words, host) stands for, or None."""
    element = int(host[0])
    if element < 0:
        return None
    gp = int(np.int32(host[1] & 0xFFFFFFFF))
    det = float(host[2:3].view(np.float64)[0])
    if gp == FAIL_BAD_NODE:
        return NodeIndexError(element_id=element_offset + element, node=int(det), n_nodes=n_nodes)
    return DegenerateElementError(element_id=element_offset + element, gauss_point=gp, det=det)


def raise_if_failed(fail: torch.Tensor, element_offset: int = 0, n_nodes: int | None = None) -> None:
    """Synchronising read of an hx_fail_info record; raises NodeIndexError for the lowest element
    with an out-of-range node id, else DegenerateElementError (element.py:237-244) for the lowest
    failing element."""
    if peek(fail[0:1])[0] < 0:
        return
    err = fail_error(fail.cpu().numpy(), element_offset, n_nodes)
    if err is not None:
        raise err


def _mode_id(mode: str) -> int:
    if mode == "exact":
        return N.MODE_EXACT
    if mode == "fast":
        return N.MODE_FAST
    raise ConfigurationError(f"integration mode must be 'exact' or 'fast', got {mode!r}")


def integrate_mesh(dm: DeviceMesh, lo: int = 0, hi: int | None = None, *, ke=None, rows=None, cols=None,
                   with_index: bool = True, mode: str = "exact", fail=None, stream=None, adjacency=None):
    """KE (+ fused iK/jK) for elements [lo, hi) of a device mesh.  Asynchronous: returns
    ``(ke, rows, cols, fail)``; call raise_if_failed(fail) after the stream is done.

    ``adjacency`` = an AssemblyPrep (new_assembly_prep): the kernel also records the node adjacency
    of the mesh-path assembly in its workspace (hx_integrate_mesh_adjacency), which mesh_csc(...,
    prep=) then skips.  The first range of a build resets it."""
    hi = dm.n_el if hi is None else hi
    if not 0 <= lo <= hi <= dm.n_el:
        raise ValueError(f"element range [{lo}, {hi}) outside [0, {dm.n_el})")
    n = hi - lo
    dev = dm.conn.device
    if ke is None:
        ke = torch.empty((n, 36), dtype=torch.float64, device=dev)
    _check_tensor(ke, torch.float64, (n, 36), "ke")
    if with_index:
        if rows is None:
            rows = torch.empty(36 * n, dtype=torch.int32, device=dev)
        if cols is None:
            cols = torch.empty(36 * n, dtype=torch.int32, device=dev)
        _check_tensor(rows, torch.int32, (36 * n,), "rows")
        _check_tensor(cols, torch.int32, (36 * n,), "cols")
    else:
        rows = cols = None
    if fail is None:
        fail = new_fail_record(dev)
    if adjacency is None:
        N.check(N.lib().hx_integrate_mesh(_ptr(dm.coords), dm.n_nodes, _ptr(dm.conn), _ptr(dm.coeff), lo, hi,
                                          _ptr(ke), _ptr(rows), _ptr(cols), _mode_id(mode), _ptr(fail),
                                          stream_handle(stream)), "hx_integrate_mesh")
    else:
        if adjacency.conn is not dm.conn:
            raise ConfigurationError("the assembly workspace belongs to another mesh")
        N.check(N.lib().hx_integrate_mesh_adjacency(
            _ptr(dm.coords), dm.n_nodes, _ptr(dm.conn), _ptr(dm.coeff), lo, hi, _ptr(ke), _ptr(rows), _ptr(cols),
            _mode_id(mode), _ptr(fail), _ptr(adjacency.ws), adjacency.ws.numel(), _ptr(adjacency.status),
            0 if adjacency.started else 1, stream_handle(stream)), "hx_integrate_mesh_adjacency")
        adjacency.started = True
    return ke, rows, cols, fail


@dataclass
class AssemblyPrep:
    """Mesh-CSC workspace + status word whose node adjacency the integration kernel fills
    (hx_integrate_mesh_adjacency) so the assembly skips its first pass."""

    conn: torch.Tensor
    ws: torch.Tensor
    status: torch.Tensor
    started: bool = False


def new_assembly_prep(dm: DeviceMesh) -> AssemblyPrep:
    ws_bytes = N.lib().hx_mesh_csc_workspace_bytes(dm.n_el, dm.n_nodes)
    if ws_bytes < 0 or 8 * dm.n_el >= 2**31 - 1:
        raise ValueError("mesh too large for one assembly plan")
    dev = dm.conn.device
    return AssemblyPrep(dm.conn, torch.empty(ws_bytes, dtype=torch.uint8, device=dev),
                        torch.zeros(1, dtype=torch.int32, device=dev))


def stiffness_batch(coords: torch.Tensor, coeff: torch.Tensor, out=None, mode: str = "exact", fail=None,
                    stream=None):
    """element.py:213-245 on device: coords (n,8,3) f64, coeff (n,) f64 -> (out (n,36), fail)."""
    n = coords.shape[0]
    _check_tensor(coords, torch.float64, (n, 8, 3), "coords")
    _check_tensor(coeff, torch.float64, (n,), "coeff")
    if out is None:
        out = torch.empty((n, 36), dtype=torch.float64, device=coords.device)
    _check_tensor(out, torch.float64, (n, 36), "out")
    if fail is None:
        fail = new_fail_record(coords.device)
    N.check(N.lib().hx_stiffness_batch(_ptr(coords), _ptr(coeff), n, _ptr(out), _mode_id(mode), _ptr(fail),
                                       stream_handle(stream)), "hx_stiffness_batch")
    return out, fail


def connectivity_index_arrays(conn: torch.Tensor, lo: int = 0, hi: int | None = None, stream=None):
    """assemble.py:86-93 on device -> (rows, cols) int32 (36*(hi-lo),)."""
    hi = conn.shape[0] if hi is None else hi
    _check_tensor(conn, torch.int32, (conn.shape[0], 8), "conn")
    n = hi - lo
    rows = torch.empty(36 * n, dtype=torch.int32, device=conn.device)
    cols = torch.empty(36 * n, dtype=torch.int32, device=conn.device)
    N.check(N.lib().hx_connectivity_index_arrays(_ptr(conn), lo, hi, _ptr(rows), _ptr(cols),
                                                 stream_handle(stream)), "hx_connectivity_index_arrays")
    return rows, cols


def dof_index_arrays(conn: torch.Tensor, n_nodes: int, dofxn: int = 1, lo: int = 0, hi: int | None = None,
                     stream=None):
    """map_local_to_global (assemble.py:65-83) for every element of [lo, hi) on device ->
    (rows, cols) int32 (P * (hi-lo),), P = (8 dofxn)(8 dofxn + 1)/2, element-major, each element's
    pairs in np.tril_indices(8 dofxn) order; dofxn = 1 equals connectivity_index_arrays."""
    hi = conn.shape[0] if hi is None else hi
    _check_tensor(conn, torch.int32, (conn.shape[0], 8), "conn")
    if dofxn < 1:
        raise ValueError(f"dofxn must be at least 1, got {dofxn}")
    P = (8 * dofxn) * (8 * dofxn + 1) // 2
    n = hi - lo
    rows = torch.empty(P * n, dtype=torch.int32, device=conn.device)
    cols = torch.empty(P * n, dtype=torch.int32, device=conn.device)
    N.check(N.lib().hx_dof_index_arrays(_ptr(conn), lo, hi, n_nodes, dofxn, _ptr(rows), _ptr(cols),
                                        stream_handle(stream)), "hx_dof_index_arrays")
    return rows, cols


def assemble_dof(conn: torch.Tensor, values: torch.Tensor, n_nodes: int, dofxn: int, stream=None) -> "DeviceCsc":
    """Lower CSC of a dofxn-per-node element matrix set: values (n_el, P) f64 in packed
    np.tril_indices(8 dofxn) order -> K of dim n_nodes * dofxn, through the generic triplet path
    (build_triplet + triplet_to_csc, assemble.py:96-140, numpy's summation rule for any run)."""
    P = (8 * dofxn) * (8 * dofxn + 1) // 2
    _check_tensor(values, torch.float64, (conn.shape[0], P), "values")
    rows, cols = dof_index_arrays(conn, n_nodes, dofxn, stream=stream)
    return triplet_csc(rows, cols, values.reshape(-1), n_nodes * dofxn, stream=stream)


@dataclass
class CompactSegment:
    """An element segment whose KE rows are compact (received halo records, hx_halo_index): element
    e's owned packed entries (bit p of kmask[e]) at values[koff[e] + rank of p] -- see
    hx_elem_segment.ke_offset / ke_mask.  conn (n, 8) int32, koff / kmask (n,) int64."""

    conn: torch.Tensor
    values: torch.Tensor
    koff: torch.Tensor
    kmask: torch.Tensor

    def slice(self, a: int, b: int) -> "CompactSegment":
        return CompactSegment(self.conn[a:b], self.values, self.koff[a:b], self.kmask[a:b])

    @property
    def n_el(self) -> int:
        return self.conn.shape[0]


@dataclass
class DeviceCsc:
    """Lower-triangular CSC block in HBM: col_ptr (ncols+1) i64, row_idx (nnz) i64, vals (nnz) f64."""

    col_ptr: torch.Tensor
    row_idx: torch.Tensor
    vals: torch.Tensor
    dim: int
    col_lo: int = 0
    path: str = "mesh"
    # events of asynchronous readers (e.g. a CscHostTransfer copy) that must complete before the
    # buffers are overwritten -- set when the buffers belong to a reusable MeshPlan
    readers: list | None = None

    @property
    def nnz(self) -> int:
        return self.row_idx.shape[0]


def _status_error(st: int):
    if st & N.ST_BAD_INDEX:
        raise MeshValidationError("triplet index outside [0, dim)")
    if st & N.ST_UPPER:
        raise MeshValidationError("triplet entry above the diagonal")


def _row_stride(t: torch.Tensor, width: int) -> int:
    """Row stride of an (n, width) tensor; a single row's stride is meaningless (numpy's [None]
    gives it 0), so it is the dense width there."""
    return t.stride(0) if t.shape[0] > 1 else width


def _check_segment(conn, ke):
    n = conn.shape[0]
    if conn.dtype != torch.int32 or tuple(conn.shape) != (n, 8) or conn.device.type != "cuda":
        raise ValueError("segment conn must be a CUDA int32 (n, 8) tensor")
    if ke.dtype != torch.float64 or tuple(ke.shape) != (n, 36) or ke.device.type != conn.device.type:
        raise ValueError("segment ke must be a CUDA float64 (n, 36) tensor")
    if n and (conn.stride(1) != 1 or _row_stride(conn, 8) % 4 or _row_stride(conn, 8) < 8 or conn.data_ptr() % 16):
        raise ValueError("segment conn rows must be 16-byte aligned with unit inner stride")
    if n and (ke.stride(1) != 1 or _row_stride(ke, 36) < 36):
        raise ValueError("segment ke rows must have unit inner stride")


# Conforming hex meshes have <= 14 lower rows per column on average (27-point stencil); the
# symbolic pass writes rows into a buffer of this many per column and retries exactly if short.
ROWS_PER_COLUMN_ESTIMATE = 16


def numbering_is_local(conn: torch.Tensor, n_nodes: int, sample: int = 4096) -> bool:
    """Heuristic for the assembly processing order: on meshes numbered with locality (structured
    generators, RCM-ordered inputs) an element's node ids span a small fraction of the id range;
    on randomly numbered meshes they span most of it.  One small device reduction + host read."""
    n = conn.shape[0]
    if n == 0 or n_nodes < 1 << 16:
        return True
    k = min(sample, n)
    idx = torch.arange(k, dtype=torch.int64, device=conn.device) * (n - 1) // max(k - 1, 1)
    rows = conn[idx]
    span = (rows.max(dim=1).values - rows.min(dim=1).values).double().mean()
    return bool(peek((span < n_nodes / 64).to(torch.int32).reshape(1))[0])


def _order_flags(order, conn, n_nodes) -> int:
    if order == "element":
        return N.CSC_ORDER_BY_ELEMENT
    if order == "column":
        return 0
    if order != "auto":
        raise ConfigurationError(f"assembly order must be 'auto', 'element' or 'column', got {order!r}")
    return 0 if numbering_is_local(conn, n_nodes) else N.CSC_ORDER_BY_ELEMENT


def mesh_csc(parts, n_nodes: int, col_lo: int = 0, col_hi: int | None = None, stream=None,
             row_capacity: int | None = None, order: str = "auto", prep: AssemblyPrep | None = None,
             nnz_hint: int | None = None) -> DeviceCsc:
    """Assemble columns [col_lo, col_hi) of the lower CSC from element segments.

    ``parts`` is a list of (conn (n,8) i32, ke (n,36) f64) CUDA tensor views in ascending global
    element order (one pair for a single GPU; halo record views for the multi-GPU path -- rows
    may be strided).  Meshes outside the node-adjacency fast path's limits fall through to the
    generic triplet path with identical results.  ``order`` picks the column processing order
    (results are identical; "auto" uses element order for numberings without locality).  ``prep``:
    the workspace whose adjacency the integration kernel already recorded (one segment, every
    column) -- the first attempt skips the adjacency pass; retries rebuild it.  ``nnz_hint``: expected
    nnz of the block (e.g. the previous step's); sizes the output buffers and the pattern scratch so
    blocks with more rows per column than average (the low columns of a permuted mesh) need no retry.
    """
    col_hi = n_nodes if col_hi is None else col_hi
    if not 1 <= len(parts) <= N.MAX_SEGMENTS:
        raise ValueError(f"1..{N.MAX_SEGMENTS} element segments required")
    def seg_conn(p):
        return p.conn if isinstance(p, CompactSegment) else p[0]

    dev = seg_conn(parts[0]).device
    descs = []
    for p in parts:
        if isinstance(p, CompactSegment):
            n = p.conn.shape[0]
            if (p.conn.dtype != torch.int32 or tuple(p.conn.shape) != (n, 8) or p.conn.stride(1) != 1
                    or p.koff.shape[0] != n or p.kmask.shape[0] != n or p.values.dtype != torch.float64):
                raise ValueError("compact segment: conn (n, 8) int32, koff / kmask (n,), float64 values")
            descs.append((p.conn.data_ptr(), p.values.data_ptr(), n, _row_stride(p.conn, 8), 0, p.koff.data_ptr(),
                          p.kmask.data_ptr()))
        else:
            c, k = p
            _check_segment(c, k)
            descs.append((c.data_ptr(), k.data_ptr(), int(c.shape[0]), _row_stride(c, 8), _row_stride(k, 36)))
    n_total = sum(int(d[2]) for d in descs)
    ncols = col_hi - col_lo
    segs = N.segments(descs)
    flags = _order_flags(order, seg_conn(parts[0]), n_nodes)
    ws_bytes = N.lib().hx_mesh_csc_workspace_bytes(n_total, ncols)
    if ws_bytes < 0:
        raise ValueError("bad mesh size")
    if prep is not None:
        if not prep.started or len(parts) != 1 or parts[0][0] is not prep.conn or col_lo != 0 or col_hi != n_nodes:
            raise ConfigurationError("assembly prep must cover the whole single-segment mesh it was made for")
        status, ws, ws_bytes = prep.status, prep.ws, prep.ws.numel()
        flags |= N.CSC_ADJACENCY_READY
    else:
        status = torch.zeros(1, dtype=torch.int32, device=dev)
    col_ptr = torch.empty(ncols + 1, dtype=torch.int64, device=dev)
    sh = stream_handle(stream)
    capacity = ROWS_PER_COLUMN_ESTIMATE * ncols if row_capacity is None else row_capacity
    if nnz_hint is not None and prep is None:
        capacity = max(capacity, int(nnz_hint))
        extra = int(nnz_hint) - ncols - 15 * ncols  # off-diagonal records beyond the default scratch
        if extra > 0:
            ws_bytes += 8 * extra
    while True:
        if not flags & N.CSC_ADJACENCY_READY:
            ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
        row_buf = torch.empty(max(capacity, 1), dtype=torch.int64, device=dev)
        val_buf = torch.empty(max(capacity, 1), dtype=torch.float64, device=dev)
        N.check(N.lib().hx_mesh_csc_build(segs, len(parts), n_nodes, col_lo, col_hi, _ptr(col_ptr), _ptr(row_buf),
                                          _ptr(val_buf), capacity, _ptr(ws), ws_bytes, _ptr(status), flags, sh),
                "hx_mesh_csc_build")
        st, nnz = peek(status[0:1], col_ptr[-1:], stream=stream)  # one sync: status + nnz
        _status_error(st)
        flags &= ~N.CSC_ADJACENCY_READY  # a retry recomputes the adjacency in a fresh workspace
        if st & N.ST_SLOT_COLLISION:
            continue  # fixed-slot adjacency lost an entry (inconsistent element orientation)
        if st & N.ST_SCRATCH and not st & (N.ST_FASTPATH_LIMITS & ~N.ST_SCRATCH):
            # more off-diagonal records than the default scratch (e.g. the first column block of a
            # permuted mesh): the counts are complete, re-run with room for all of them
            ws_bytes = N.lib().hx_mesh_csc_workspace_bytes(n_total, ncols) + 8 * nnz
            capacity = max(capacity, nnz)
            continue
        if st & N.ST_FASTPATH_LIMITS:
            return _mesh_csc_generic(parts, n_nodes, col_lo, col_hi, stream)
        if nnz <= capacity:
            break
        capacity = nnz  # rare: more rows than the estimate -> exact-size retry
    row_idx = row_buf[:nnz]
    vals = val_buf[:nnz]
    return DeviceCsc(col_ptr, row_idx, vals, n_nodes, col_lo, "mesh")


@dataclass
class MeshPlan:
    """Symbolic assembly launched asynchronously (hx_mesh_csc_symbolic without row emission):
    col_ptr, the workspace holding the sorted adjacency and the off-diagonal records, the status
    word and the output buffers sized by the rows-per-column estimate."""

    conn: torch.Tensor
    n_nodes: int
    col_ptr: torch.Tensor
    ws: torch.Tensor
    status: torch.Tensor
    row_buf: torch.Tensor
    val_buf: torch.Tensor
    capacity: int
    flags: int = 0
    nnz: int = -1  # known once the plan is verified (plan_assembly): emits then need no host sync
    readers: list = None  # events of pending readers of row_buf / val_buf (see DeviceCsc.readers)


def mesh_plan_async(conn: torch.Tensor, n_nodes: int, stream=None, order: str = "auto", ws_bytes: int | None = None,
                    capacity: int | None = None, fixed: bool = False) -> MeshPlan:
    """Launch the symbolic phase of a single-segment mesh assembly on ``stream`` (no host sync).
    It reads only the connectivity, so it can run concurrently with the integration kernel.
    ``fixed``: fixed-slot adjacency (HX_CSC_FIXED_ADJACENCY, no atomic counters); a mesh whose
    elements hold a node at the same local index reports a slot collision (plan_result re-assembles)."""
    n = conn.shape[0]
    if conn.dtype != torch.int32 or tuple(conn.shape) != (n, 8) or not conn.is_contiguous():
        raise ValueError("conn must be a contiguous CUDA int32 (n, 8) tensor")
    dev = conn.device
    if ws_bytes is None:
        ws_bytes = N.lib().hx_mesh_csc_workspace_bytes(n, n_nodes)
    if ws_bytes < 0:
        raise ValueError("bad mesh size")
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    col_ptr = torch.empty(n_nodes + 1, dtype=torch.int64, device=dev)
    capacity = ROWS_PER_COLUMN_ESTIMATE * n_nodes if capacity is None else capacity
    row_buf = torch.empty(max(capacity, 1), dtype=torch.int64, device=dev)
    val_buf = torch.empty(max(capacity, 1), dtype=torch.float64, device=dev)
    segs = N.segments([(conn.data_ptr(), 0, n)])
    flags = _order_flags(order, conn, n_nodes) | (N.CSC_FIXED_ADJACENCY if fixed else 0)
    N.check(N.lib().hx_mesh_csc_symbolic(segs, 1, n_nodes, 0, n_nodes, _ptr(col_ptr), ctypes.c_void_p(0), 0,
                                         _ptr(ws), ws_bytes, _ptr(status), flags, stream_handle(stream)),
            "hx_mesh_csc_symbolic")
    return MeshPlan(conn, n_nodes, col_ptr, ws, status, row_buf, val_buf, capacity, flags)


def plan_assembly(dm: "DeviceMesh", order: str | None = None, stream=None):
    """Verified symbolic plan of a mesh's assembly (pattern, sorted adjacency, contribution records),
    reusable for rebuilds while the connectivity is unchanged -- new coordinates or coefficients
    only need the integration kernel and one emit pass (``build_device(dm, plan=...)``).  Returns
    None when the mesh is outside the node-adjacency fast path (rebuilds then use mesh_csc)."""
    order = dm.assembly_order() if order is None else order
    ws_bytes, capacity = None, None
    while True:
        plan = mesh_plan_async(dm.conn, dm.n_nodes, stream=stream, order=order, ws_bytes=ws_bytes, capacity=capacity)
        st, nnz = peek(plan.status[0:1], plan.col_ptr[-1:], stream=stream)
        _status_error(st)
        if st & N.ST_SCRATCH and not st & (N.ST_FASTPATH_LIMITS & ~N.ST_SCRATCH):
            ws_bytes = N.lib().hx_mesh_csc_workspace_bytes(dm.n_el, dm.n_nodes) + 8 * nnz
            continue
        if st & N.ST_FASTPATH_LIMITS:
            return None
        if nnz > plan.capacity:
            capacity = nnz
            continue
        plan.nnz = nnz
        return plan


def mesh_emit(plan: MeshPlan, ke: torch.Tensor, stream=None) -> DeviceCsc:
    """Row indices and values of a planned assembly (one pass over the KE rows).  A verified plan
    (plan_assembly) returns without a host sync -- the outputs live in the plan's buffers and are
    overwritten by the next emit; otherwise one sync checks the status word and nnz and falls back
    to mesh_csc when the plan hit a limit."""
    _check_segment(plan.conn, ke)
    if plan.readers is None:
        plan.readers = []
    s = torch.cuda.current_stream(ke.device) if stream is None else stream
    for ev in plan.readers:  # a previous result still being read (host transfer): do not overwrite it
        s.wait_event(ev)
    plan.readers.clear()
    segs = N.segments([(plan.conn.data_ptr(), ke.data_ptr(), plan.conn.shape[0])])
    N.check(N.lib().hx_mesh_csc_emit(segs, 1, 0, plan.n_nodes, _ptr(plan.col_ptr), _ptr(plan.row_buf),
                                     _ptr(plan.val_buf), plan.capacity, _ptr(plan.ws), _ptr(plan.status),
                                     stream_handle(stream)), "hx_mesh_csc_emit")
    return plan_result(plan, ke, stream=stream)


def integrate_emit(dm: "DeviceMesh", plan: MeshPlan, ke: torch.Tensor, rows=None, cols=None, mode: str = "exact",
                   stream=None) -> torch.Tensor:
    """KE (+ iK/jK) of every element and the plan's emit pass in one launch (hx_integrate_emit): the
    emit tiles run on the integration kernel's warps as soon as their elements are integrated.
    Returns the fail record; the CSC is read with plan_result."""
    n = dm.n_el
    _check_tensor(ke, torch.float64, (n, 36), "ke")
    if (rows is None) != (cols is None):
        raise ValueError("rows and cols go together")
    if rows is not None:
        _check_tensor(rows, torch.int32, (36 * n,), "rows")
        _check_tensor(cols, torch.int32, (36 * n,), "cols")
    if plan.conn is not dm.conn:
        raise ConfigurationError("the assembly plan belongs to another mesh")
    dev = ke.device
    if plan.readers is None:
        plan.readers = []
    s = torch.cuda.current_stream(dev) if stream is None else stream
    for ev in plan.readers:  # a previous result still being read (host transfer): do not overwrite it
        s.wait_event(ev)
    plan.readers.clear()
    fail = new_fail_record(dev)
    sched_bytes = N.lib().hx_integrate_emit_workspace_bytes(n)
    sched = torch.empty(sched_bytes, dtype=torch.uint8, device=dev)
    N.check(N.lib().hx_integrate_emit(_ptr(dm.coords), dm.n_nodes, _ptr(dm.conn), _ptr(dm.coeff), n, _ptr(ke),
                                      _ptr(rows), _ptr(cols), _mode_id(mode), _ptr(fail), _ptr(plan.col_ptr),
                                      _ptr(plan.row_buf), _ptr(plan.val_buf), plan.capacity, _ptr(plan.ws),
                                      _ptr(plan.status), _ptr(sched), sched_bytes, stream_handle(stream)),
            "hx_integrate_emit")
    return fail


def plan_result(plan: MeshPlan, ke: torch.Tensor, stream=None) -> DeviceCsc:
    """The CSC an emit into ``plan``'s buffers produced (mesh_emit / integrate_emit): a verified plan
    returns without a host sync; otherwise one sync checks the status word and nnz and re-assembles
    with mesh_csc when the plan hit a limit (or its fixed-slot adjacency collided)."""
    if plan.nnz >= 0:
        return DeviceCsc(plan.col_ptr, plan.row_buf[:plan.nnz], plan.val_buf[:plan.nnz], plan.n_nodes, 0, "mesh",
                         readers=plan.readers)
    st, nnz = peek(plan.status[0:1], plan.col_ptr[-1:], stream=stream)
    _status_error(st)
    if st & (N.ST_FASTPATH_LIMITS | N.ST_SLOT_COLLISION) or nnz > plan.capacity:
        order = "element" if plan.flags & N.CSC_ORDER_BY_ELEMENT else "column"
        return mesh_csc([(plan.conn, ke)], plan.n_nodes, stream=stream, order=order)
    return DeviceCsc(plan.col_ptr, plan.row_buf[:nnz], plan.val_buf[:nnz], plan.n_nodes, 0, "mesh",
                     readers=plan.readers)


def rows_narrow(row_idx: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """int32 copy of an int64 row-index array on the device (hx_rows_narrow): the compact form the
    host transfer sends over PCIe."""
    if row_idx.dtype != torch.int64 or row_idx.dim() != 1 or not row_idx.is_contiguous():
        raise ValueError("row_idx must be a contiguous 1-D int64 tensor")
    if out is None:
        out = torch.empty(row_idx.shape[0], dtype=torch.int32, device=row_idx.device)
    _check_tensor(out, torch.int32, (row_idx.shape[0],), "out")
    N.check(N.lib().hx_rows_narrow(_ptr(row_idx), _ptr(out), row_idx.shape[0], stream_handle(stream)),
            "hx_rows_narrow")
    return out


def block_elements(dm: DeviceMesh, col_lo: int, col_hi: int, ids=None, ws=None, stream=None):
    """Elements with a node in columns [col_lo, col_hi), ascending (hx_block_select + gather):
    returns (global ids (m,) i64, conn (m, 8) i32, coeff (m,) f64) on the device."""
    n = dm.n_el
    dev = dm.conn.device
    if ids is None:
        ids = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    if ws is None:
        ws = torch.empty(max(N.lib().hx_block_select_workspace_bytes(n), 1), dtype=torch.uint8, device=dev)
    count = torch.empty(1, dtype=torch.int64, device=dev)
    sh = stream_handle(stream)
    N.check(N.lib().hx_block_select(_ptr(dm.conn), n, col_lo, col_hi, _ptr(ids), _ptr(count), _ptr(ws),
                                    ws.numel(), sh), "hx_block_select")
    m = int(count.item())
    conn = torch.empty((m, 8), dtype=torch.int32, device=dev)
    coeff = torch.empty(m, dtype=torch.float64, device=dev)
    N.check(N.lib().hx_block_gather(_ptr(dm.conn), _ptr(dm.coeff), _ptr(ids), _ptr(count), m, _ptr(conn),
                                    _ptr(coeff), sh), "hx_block_gather")
    return ids[:m], conn, coeff


def _dense_rows(seg: CompactSegment) -> torch.Tensor:
    """(n, 36) float64 rows of a compact segment (entries it does not hold are 0)."""
    bits = (seg.kmask[:, None] >> torch.arange(36, device=seg.kmask.device)) & 1
    idx = seg.koff[:, None] + torch.cumsum(bits, dim=1) - 1
    return torch.where(bits.bool(), seg.values[idx.clamp(min=0)], torch.zeros((), dtype=torch.float64,
                                                                              device=seg.values.device))


def _mesh_csc_generic(parts, n_nodes, col_lo, col_hi, stream) -> DeviceCsc:
    rows_l, cols_l, vals_l = [], [], []
    parts = [(p.conn, _dense_rows(p)) if isinstance(p, CompactSegment) else p for p in parts]
    for conn, ke in parts:
        r, c = connectivity_index_arrays(conn.contiguous(), stream=stream)
        rows_l.append(r)
        cols_l.append(c)
        vals_l.append(ke.contiguous().reshape(-1))
    rows, cols, vals = torch.cat(rows_l), torch.cat(cols_l), torch.cat(vals_l)
    if col_lo != 0 or col_hi != n_nodes:
        keep = (cols >= col_lo) & (cols < col_hi)
        rows, cols, vals = rows[keep], cols[keep], vals[keep]
    full = triplet_csc(rows, cols, vals, n_nodes, stream=stream)
    cp = full.col_ptr[col_lo:col_hi + 1]
    return DeviceCsc(cp - cp[0], full.row_idx, full.vals, n_nodes, col_lo, "triplet")


def triplet_csc(rows: torch.Tensor, cols: torch.Tensor, vals: torch.Tensor, dim: int, stream=None) -> DeviceCsc:
    """Generic triplet -> lower CSC (assemble.py:110-149) on device."""
    n = rows.shape[0]
    _check_tensor(rows, torch.int32, (n,), "rows")
    _check_tensor(cols, torch.int32, (n,), "cols")
    _check_tensor(vals, torch.float64, (n,), "vals")
    dev = rows.device
    ws_bytes = N.lib().hx_triplet_csc_workspace_bytes(n, dim)
    if ws_bytes < 0:
        raise ConfigurationError(f"{n} triplets exceed one device sort")
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    col_ptr = torch.empty(dim + 1, dtype=torch.int64, device=dev)
    row_buf = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    sh = stream_handle(stream)
    N.check(N.lib().hx_triplet_csc_symbolic(_ptr(rows), _ptr(cols), n, dim, _ptr(col_ptr), _ptr(row_buf),
                                            _ptr(ws), ws_bytes, _ptr(status), sh), "hx_triplet_csc_symbolic")
    st, nnz = peek(status[0:1], col_ptr[-1:], stream=stream)
    _status_error(st)
    out = torch.empty(nnz, dtype=torch.float64, device=dev)
    N.check(N.lib().hx_triplet_csc_numeric(_ptr(vals), n, dim, _ptr(col_ptr), _ptr(out), _ptr(ws), sh),
            "hx_triplet_csc_numeric")
    return DeviceCsc(col_ptr, row_buf[:nnz], out, dim, 0, "triplet")
