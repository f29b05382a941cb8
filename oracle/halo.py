"""TEST INFRASTRUCTURE ONLY -- numpy restatement of the multi-GPU exchange step (hx_halo.cu).

The reference has no multi-GPU code; what pins the sharded build is that the
concatenated column blocks equal the single-process triplet_to_csc (assemble.py:110-140) bit for
bit.  This module restates the wire format so the host logic can run over gloo on CPU and the CUDA
pack/unpack kernels can be checked word for word:

  owner(node)             largest r with bounds[r] <= node
  entry p = (i, j) of e   lands in column min(g_i, g_j), owned by min(owner(g_i), owner(g_j))
  record for d            8 node ids (4 int64 words) + the owned entries' bit patterns, ascending p
  chunk s -> d            [ids of all records][values of all records], ascending element order
  column weights          entry (i, j) adds 1 << popcount(code_i ^ code_j) to bin(min(g_i, g_j))
"""

from __future__ import annotations

import numpy as np

PACK_I = np.array([i for i in range(8) for _ in range(i + 1)])
PACK_J = np.array([j for i in range(8) for j in range(i + 1)])
# natural-coordinate codes of the local nodes (element.py:45-56: ccw bottom face, then top face)
_NAT = np.array([[-1, -1, -1], [1, -1, -1], [1, 1, -1], [-1, 1, -1], [-1, -1, 1], [1, -1, 1], [1, 1, 1], [-1, 1, 1]])
_CODE = (_NAT[:, 0] > 0) | ((_NAT[:, 1] > 0) << 1) | ((_NAT[:, 2] > 0) << 2)
PAIR_WEIGHT = np.array([1 << bin(int(_CODE[i] ^ _CODE[j])).count("1") for i, j in zip(PACK_I, PACK_J)],
                       dtype=np.int64)


def owners(conn: np.ndarray, bounds: np.ndarray) -> np.ndarray:
    return np.searchsorted(np.asarray(bounds), np.asarray(conn), side="right") - 1


def owned_mask(conn, bounds, d) -> np.ndarray:
    o = owners(conn, bounds)
    return np.minimum(o[:, PACK_I], o[:, PACK_J]) == d  # (n, 36)


def column_weights(conn: np.ndarray, n_nodes: int, n_bins: int) -> np.ndarray:
    conn = np.asarray(conn, dtype=np.int64)
    col = np.minimum(conn[:, PACK_I], conn[:, PACK_J])
    b = col * n_bins // n_nodes
    w = np.broadcast_to(PAIR_WEIGHT, col.shape)
    return np.bincount(b.ravel(), weights=w.ravel(), minlength=n_bins).astype(np.int64)


def column_touch(conn: np.ndarray, n_nodes: int, n_bins: int) -> np.ndarray:
    """hx_column_touch restated: 8 per (element, distinct bin of its nodes)."""
    conn = np.asarray(conn, dtype=np.int64)
    b = conn * n_bins // n_nodes
    hist = np.zeros(n_bins, dtype=np.int64)
    for e in range(b.shape[0]):
        for x in set(b[e].tolist()):
            hist[x] += 8
    return hist


def count(conn, bounds, world, self_rank) -> np.ndarray:
    """(world, 2) int64: records, values per destination (0 for self)."""
    out = np.zeros((world, 2), dtype=np.int64)
    for d in range(world):
        if d == self_rank:
            continue
        m = owned_mask(conn, bounds, d)
        out[d] = (int(m.any(axis=1).sum()), int(m.sum()))
    return out


def pack(conn, ke, bounds, world, self_rank) -> list:
    """Per destination: the int64 word chunk [ids | values]."""
    conn = np.ascontiguousarray(conn, dtype=np.int32)
    ke_bits = np.ascontiguousarray(ke, dtype=np.float64).view(np.int64)
    chunks = []
    for d in range(world):
        if d == self_rank:
            chunks.append(np.empty(0, dtype=np.int64))
            continue
        m = owned_mask(conn, bounds, d)
        rec = m.any(axis=1)
        ids = np.ascontiguousarray(conn[rec]).view(np.int64).reshape(-1)
        chunks.append(np.concatenate([ids, ke_bits[m]]))  # boolean indexing is row-major: element, then p
    return chunks


def index(recv: np.ndarray, desc: np.ndarray, bounds, world, self_rank):
    """hx_halo_index restated: (conn (n, 8) int32, ke_offset (n,) int64 = word of each record's first
    value in recv, ke_mask (n,) uint64 = its owned packed entries)."""
    conns, offs, masks = [], [], []
    for s in range(world):
        off, nr, nv = (int(x) for x in desc[s])
        if nr == 0:
            continue
        conn = np.ascontiguousarray(recv[off:off + 4 * nr]).view(np.int32).reshape(nr, 8)
        m = owned_mask(conn, bounds, self_rank)
        conns.append(conn)
        offs.append(off + 4 * nr + np.concatenate([[0], np.cumsum(m.sum(axis=1))[:-1]]).astype(np.int64))
        masks.append((m.astype(np.uint64) << np.arange(36, dtype=np.uint64)).sum(axis=1).astype(np.uint64))
    if not conns:
        return np.empty((0, 8), np.int32), np.empty(0, np.int64), np.empty(0, np.uint64)
    return np.concatenate(conns), np.concatenate(offs), np.concatenate(masks)


def unpack(recv: np.ndarray, desc: np.ndarray, bounds, world, self_rank) -> np.ndarray:
    """recv int64 words, desc (world, 3) = (offset, records, values) per source -> (n, 40) f64 records."""
    out = []
    for s in range(world):
        off, nr, nv = (int(x) for x in desc[s])
        if nr == 0:
            continue
        ids = recv[off:off + 4 * nr].reshape(nr, 4)
        vals = recv[off + 4 * nr:off + 4 * nr + nv]
        conn = np.ascontiguousarray(ids).view(np.int32).reshape(nr, 8)
        m = owned_mask(conn, bounds, self_rank)
        rec = np.zeros((nr, 40), dtype=np.float64)
        ke = np.zeros((nr, 36), dtype=np.int64)
        ke[m] = vals
        rec[:, :36] = ke.view(np.float64)
        rec.view(np.int64)[:, 36:] = ids
        out.append(rec)
    return np.concatenate(out) if out else np.empty((0, 40), dtype=np.float64)
