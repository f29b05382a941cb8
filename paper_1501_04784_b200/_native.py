"""ctypes binding of libhexfem_b200.so (include/hexfem_b200.h).

The library is loaded from the package tree (built in place by build.py / __graft_entry__.build).
There is no fallback: if the library is missing or the device is unavailable, every compute
entry point raises NativeLibraryError.  ctypes releases the GIL during foreign calls, so the
overlapped integration mode can call the ABI from two host threads.
"""

from __future__ import annotations

import ctypes
from pathlib import Path

from .errors import ConfigurationError, NativeLibraryError

import os

# HEXFEM_B200_LIB: alternate build of the same library (kernel experiments only).
LIB_PATH = Path(os.environ.get("HEXFEM_B200_LIB") or Path(__file__).resolve().parent / "_lib" / "libhexfem_b200.so")

HX_OK, HX_ERR_VALUE, HX_ERR_CONFIG, HX_ERR_CUDA, HX_ERR_WORKSPACE = 0, 1, 2, 3, 4
ST_DEG_OVERFLOW, ST_ROW_OVERFLOW, ST_REPEATED_NODE, ST_BAD_INDEX, ST_UPPER, ST_SCRATCH = 1, 2, 4, 8, 16, 32
ST_SLOT_COLLISION = 64
ST_FASTPATH_LIMITS = ST_DEG_OVERFLOW | ST_ROW_OVERFLOW | ST_REPEATED_NODE | ST_SCRATCH
MODE_EXACT, MODE_FAST = 0, 1
CSC_ORDER_BY_ELEMENT = 1
CSC_ADJACENCY_READY = 2
CSC_FIXED_ADJACENCY = 4
MAX_SEGMENTS = 4

# Every symbol declared in include/hexfem_b200.h (checked by tests/test_abi_cpu.py).
EXPORTED = (
    "hx_abi_version", "hx_last_error", "hx_dn_table", "hx_pack_tables", "hx_device_sm_count",
    "hx_selftest_division",
    "hx_stiffness_batch", "hx_integrate_mesh", "hx_integrate_mesh_adjacency", "hx_connectivity_index_arrays",
    "hx_dof_index_arrays",
    "hx_mesh_csc_workspace_bytes", "hx_mesh_csc_symbolic", "hx_mesh_csc_build", "hx_mesh_csc_numeric",
    "hx_mesh_csc_emit", "hx_integrate_emit_workspace_bytes", "hx_integrate_emit",
    "hx_triplet_csc_workspace_bytes", "hx_triplet_csc_symbolic", "hx_triplet_csc_numeric",
    "hx_column_weights", "hx_column_touch", "hx_halo_workspace_bytes", "hx_halo_count", "hx_halo_pack",
    "hx_halo_unpack_workspace_bytes", "hx_halo_unpack", "hx_halo_index", "hx_digest",
    "hx_ipc_alloc", "hx_ipc_open", "hx_ipc_close", "hx_ipc_free",
    "hx_block_select_workspace_bytes", "hx_block_select", "hx_block_gather", "hx_block_ranges", "hx_block_ranges_nodes", "hx_block_ranges_sampled", "hx_block_verify",
    "hx_mm_write", "hx_mm_read", "hx_generate_cube_mesh", "hx_rows_narrow", "hx_rows_widen", "hx_peek",
    "hx_rows_encode_workspace_bytes", "hx_rows_encode", "hx_rows_decode",
)


PEEK_MAX = 8
IPC_HANDLE_BYTES = 64


class HxPeekArgs(ctypes.Structure):
    _fields_ = [("src", ctypes.c_void_p * PEEK_MAX), ("bytes", ctypes.c_int32 * PEEK_MAX), ("n", ctypes.c_int32)]


class HxFailInfo(ctypes.Structure):
    _fields_ = [("element", ctypes.c_int64), ("gauss_point", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("det", ctypes.c_double)]


class HxElemSegment(ctypes.Structure):
    _fields_ = [("conn", ctypes.c_void_p), ("ke", ctypes.c_void_p), ("n_el", ctypes.c_int64),
                ("conn_stride", ctypes.c_int64), ("ke_stride", ctypes.c_int64),
                ("ke_offset", ctypes.c_void_p), ("ke_mask", ctypes.c_void_p)]


_lib = None


def lib():
    """Load (once) and return the native library; raises NativeLibraryError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise NativeLibraryError(
            f"{LIB_PATH} not found: build it with `python -m paper_1501_04784_b200.build` "
            "(there is no CPU fallback)")
    try:
        L = ctypes.CDLL(str(LIB_PATH))
    except OSError as exc:  # pragma: no cover - broken build
        raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
    P, I32, I64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    sig = {
        "hx_abi_version": ([], ctypes.c_int),
        "hx_last_error": ([], ctypes.c_char_p),
        "hx_dn_table": ([P], None),
        "hx_pack_tables": ([P, P], None),
        "hx_device_sm_count": ([], ctypes.c_int),
        "hx_selftest_division": ([ctypes.c_uint64, ctypes.c_uint64, P, P], ctypes.c_int),
        "hx_stiffness_batch": ([P, P, I64, P, I32, P, P], ctypes.c_int),
        "hx_integrate_mesh": ([P, I64, P, P, I64, I64, P, P, P, I32, P, P], ctypes.c_int),
        "hx_integrate_mesh_adjacency": ([P, I64, P, P, I64, I64, P, P, P, I32, P, P, I64, P, I32, P], ctypes.c_int),
        "hx_connectivity_index_arrays": ([P, I64, I64, P, P, P], ctypes.c_int),
        "hx_dof_index_arrays": ([P, I64, I64, I64, I32, P, P, P], ctypes.c_int),
        "hx_mesh_csc_workspace_bytes": ([I64, I64], I64),
        "hx_integrate_emit_workspace_bytes": ([I64], I64),
        "hx_integrate_emit": ([P, I64, P, P, I64, P, P, P, I32, P, P, P, P, I64, P, P, P, I64, P], ctypes.c_int),
        "hx_mesh_csc_symbolic": ([P, I32, I64, I64, I64, P, P, I64, P, I64, P, I32, P], ctypes.c_int),
        "hx_mesh_csc_build": ([P, I32, I64, I64, I64, P, P, P, I64, P, I64, P, I32, P], ctypes.c_int),
        "hx_mesh_csc_numeric": ([P, I32, I64, I64, P, P, P, P, P, P], ctypes.c_int),
        "hx_mesh_csc_emit": ([P, I32, I64, I64, P, P, P, I64, P, P, P], ctypes.c_int),
        "hx_triplet_csc_workspace_bytes": ([I64, I64], I64),
        "hx_triplet_csc_symbolic": ([P, P, I64, I64, P, P, P, I64, P, P], ctypes.c_int),
        "hx_triplet_csc_numeric": ([P, I64, I64, P, P, P, P], ctypes.c_int),
        "hx_column_weights": ([P, I64, I64, I64, P, P], ctypes.c_int),
        "hx_column_touch": ([P, I64, I64, I64, P, P], ctypes.c_int),
        "hx_halo_workspace_bytes": ([I64, I32], I64),
        "hx_halo_count": ([P, I64, P, I32, I32, P, P, I64, P], ctypes.c_int),
        "hx_halo_pack": ([P, P, I64, P, I32, I32, P, P, P, P], ctypes.c_int),
        "hx_halo_unpack_workspace_bytes": ([I64], I64),
        "hx_halo_unpack": ([P, P, I32, I32, P, I64, P, P, I64, P], ctypes.c_int),
        "hx_halo_index": ([P, P, I32, I32, P, I64, P, P, P, P, I64, P], ctypes.c_int),
        "hx_digest": ([P, I64, I64, ctypes.c_uint64, P, P], ctypes.c_int),
        "hx_ipc_alloc": ([I64, ctypes.POINTER(ctypes.c_void_p), P], ctypes.c_int),
        "hx_ipc_open": ([P, ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
        "hx_ipc_close": ([P], ctypes.c_int),
        "hx_ipc_free": ([P], ctypes.c_int),
        "hx_mm_write": ([P, P, P, I64, ctypes.c_char_p, I32], ctypes.c_int),
        "hx_rows_narrow": ([P, P, I64, P], ctypes.c_int),
        "hx_rows_widen": ([P, P, I64, I32], ctypes.c_int),
        "hx_rows_encode_workspace_bytes": ([I64], I64),
        "hx_rows_encode": ([P, P, I64, I64, P, P, P, I64, P, P, I64, P], ctypes.c_int),
        "hx_rows_decode": ([P, P, P, I64, I64, I64, I64, P, P, I32], ctypes.c_int),
        "hx_peek": ([P, P, P], ctypes.c_int),
        "hx_mm_read": ([ctypes.c_char_p, P, P, P, P, P, P], ctypes.c_int),
        "hx_generate_cube_mesh": ([I64, I64, I64, ctypes.c_double, ctypes.c_double, P, P, P, P], ctypes.c_int),
        "hx_block_select_workspace_bytes": ([I64], I64),
        "hx_block_select": ([P, I64, I64, I64, P, P, P, I64, P], ctypes.c_int),
        "hx_block_gather": ([P, P, P, P, I64, P, P, P], ctypes.c_int),
        "hx_block_ranges": ([P, I64, P, I32, P, P, I32], ctypes.c_int),
        "hx_block_ranges_nodes": ([P, I64, P, I32, P, P, P, P, I32], ctypes.c_int),
        "hx_block_ranges_sampled": ([P, I64, P, I32, I64, P, P, P, I32], ctypes.c_int),
        "hx_block_verify": ([P, I64, I64, I64, P, I32, P, P, I64, P, P], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def check(rc: int, what: str) -> None:
    """Map an ABI status onto the reference exception hierarchy."""
    if rc == HX_OK:
        return
    msg = (lib().hx_last_error() or b"").decode(errors="replace")
    if rc == HX_ERR_VALUE:
        raise ValueError(f"{what}: {msg}")
    if rc == HX_ERR_CONFIG:
        raise ConfigurationError(f"{what}: {msg}")
    raise NativeLibraryError(f"{what} failed ({rc}): {msg}")


def segments(parts) -> ctypes.Array:
    """Build an hx_elem_segment[] from (conn_ptr, ke_ptr, n_el[, conn_stride, ke_stride[, ke_offset_ptr,
    ke_mask_ptr]]) tuples."""
    arr = (HxElemSegment * len(parts))()
    for i, part in enumerate(parts):
        conn, ke, n = part[:3]
        arr[i].conn = conn
        arr[i].ke = ke
        arr[i].n_el = n
        arr[i].conn_stride = part[3] if len(part) > 3 else 0
        arr[i].ke_stride = part[4] if len(part) > 4 else 0
        arr[i].ke_offset = part[5] if len(part) > 5 else None
        arr[i].ke_mask = part[6] if len(part) > 6 else None
    return arr
