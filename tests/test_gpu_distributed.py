"""Sharded build on one GPU: G virtual ranks (loopback exchange) through the real CUDA kernels
must be bitwise equal to the single-GPU build and to the reference."""

import numpy as np
import pytest
import torch

from common import bits_equal, golden_mesh
from paper_1501_04784_b200 import device as D
from paper_1501_04784_b200 import distributed as X
from paper_1501_04784_b200.distributed import CudaOps, concat_blocks, run_loopback, run_loopback_p2p
from paper_1501_04784_b200.pipeline import build_device
from paper_1501_04784_b200.workloads import make_workload, permuted_mesh, perturbed_mesh

pytestmark = pytest.mark.gpu


def single(mesh):
    b = build_device(D.DeviceMesh.from_host(mesh))
    return b.csc.col_ptr.cpu().numpy(), b.csc.row_idx.cpu().numpy(), b.csc.vals.cpu().numpy()


@pytest.mark.parametrize("world", [2, 3, 4, 8])
@pytest.mark.parametrize("kind", ["structured", "permuted"])
def test_loopback_shards_bitwise_equal_to_single_gpu(world, kind):
    mesh = perturbed_mesh(9, seed=world)
    if kind == "permuted":
        mesh = permuted_mesh(mesh, seed=world + 10)
    results = run_loopback(mesh, world, lambda: CudaOps())
    cp, ri, vv = concat_blocks(results)
    cp1, ri1, vv1 = single(mesh)
    assert bits_equal(cp, cp1) and bits_equal(ri, ri1) and bits_equal(vv, vv1)


def test_loopback_matches_reference_golden(golden):
    mesh = golden_mesh(golden, "perm5")
    cp, ri, vv = concat_blocks(run_loopback(mesh, 4, lambda: CudaOps()))
    assert bits_equal(cp, golden["perm5_col_ptr"])
    assert bits_equal(ri, golden["perm5_row_idx"])
    assert bits_equal(vv, golden["perm5_vals"])


def test_loopback_c2_scale():
    mesh = make_workload("C2")
    cp, ri, vv = concat_blocks(run_loopback(mesh, 8, lambda: CudaOps()))
    cp1, ri1, vv1 = single(mesh)
    assert bits_equal(cp, cp1) and bits_equal(ri, ri1) and bits_equal(vv, vv1)
    torch.cuda.empty_cache()


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("kind", ["structured", "permuted"])
def test_loopback_fused_send_bitwise(world, kind):
    """hx_halo_send (pack-and-send into the destinations' buffers) == the NCCL-path layout, bitwise."""
    mesh = perturbed_mesh(9, seed=world + 40)
    if kind == "permuted":
        mesh = permuted_mesh(mesh, seed=world + 50)
    cp, ri, vv = concat_blocks(run_loopback_p2p(mesh, world, lambda: CudaOps()))
    cp1, ri1, vv1 = single(mesh)
    assert bits_equal(cp, cp1) and bits_equal(ri, ri1) and bits_equal(vv, vv1)


def _dev_mesh(mesh):
    return D.DeviceMesh.from_host(mesh)


@pytest.mark.parametrize("kind", ["structured", "permuted"])
def test_column_weights_match_oracle(kind):
    from oracle import halo
    from paper_1501_04784_b200.distributed import histogram_bins

    mesh = perturbed_mesh(11, seed=7)
    if kind == "permuted":
        mesh = permuted_mesh(mesh, seed=8)
    ops = CudaOps()
    dm = _dev_mesh(mesh)
    for bins in (histogram_bins(mesh.n_nodes), 97, 20000 if mesh.n_nodes > 20000 else mesh.n_nodes):
        got = ops.column_weights(dm, mesh.n_nodes, bins).cpu().numpy()
        assert np.array_equal(got, halo.column_weights(mesh.connectivity, mesh.n_nodes, bins))


def test_column_weights_global_atomics_path():
    """> 16384 bins: the kernel accumulates in global memory instead of shared memory."""
    from oracle import halo

    mesh = permuted_mesh(perturbed_mesh(30, seed=1), seed=2)
    ops = CudaOps()
    got = ops.column_weights(_dev_mesh(mesh), mesh.n_nodes, 25000).cpu().numpy()
    assert np.array_equal(got, halo.column_weights(mesh.connectivity, mesh.n_nodes, 25000))


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("kind", ["structured", "permuted"])
def test_halo_pack_unpack_words_match_oracle(world, kind):
    """hx_halo_count / hx_halo_pack / hx_halo_unpack word for word against oracle/halo.py."""
    from oracle import halo
    from paper_1501_04784_b200.distributed import balanced_bounds, element_ranges, histogram_bins

    mesh = perturbed_mesh(9, seed=world)
    if kind == "permuted":
        mesh = permuted_mesh(mesh, seed=world + 3)
    ops = CudaOps()
    hist = halo.column_weights(mesh.connectivity, mesh.n_nodes, histogram_bins(mesh.n_nodes))
    bounds = balanced_bounds(hist, mesh.n_nodes, world)
    bdev = ops.bounds(bounds)
    rng = np.random.default_rng(world)
    ke = rng.standard_normal((mesh.n_el, 36))
    ke[:, 3] = -0.0
    for r, (lo, hi) in enumerate(element_ranges(mesh.n_el, world)):
        dm = ops.upload(mesh.coords, mesh.connectivity[lo:hi], mesh.coefficient[lo:hi])
        ke_d = torch.from_numpy(ke[lo:hi]).to(ops.device)
        per_dest, ws = ops.halo_count(dm, bdev, world, r)
        want = halo.count(mesh.connectivity[lo:hi], bounds, world, r)
        assert np.array_equal(per_dest.cpu().numpy(), want)
        chunks = 4 * want[:, 0] + want[:, 1]
        send = ops.alloc_words(int(chunks.sum())).fill_(-7)
        offs = np.concatenate([[0], np.cumsum(chunks)[:-1]])
        ops.halo_pack(dm, ke_d, bdev, world, r, *ops.pointers([send.data_ptr()] * world, offs), ws)
        got = send.cpu().numpy()
        for d, c in enumerate(halo.pack(mesh.connectivity[lo:hi], ke[lo:hi], bounds, world, r)):
            assert np.array_equal(got[offs[d]:offs[d] + chunks[d]], c)
        # this rank's chunks, unpacked by each receiver as if it were the only source
        for d in range(world):
            if d == r or chunks[d] == 0:
                continue
            desc = np.zeros((world, 3), np.int64)
            desc[r] = (offs[d], want[d, 0], want[d, 1])
            recs = ops.halo_unpack(send, desc, bdev, world, d, int(want[d, 0])).cpu().numpy()
            ref = halo.unpack(got, desc, bounds, world, d)
            assert recs.tobytes() == ref.tobytes()
            seg = ops.halo_index(send, desc, bdev, world, d, int(want[d, 0]))
            c_ref, o_ref, m_ref = halo.index(got, desc, bounds, world, d)
            assert np.array_equal(seg.conn.cpu().numpy(), c_ref) and np.array_equal(seg.koff.cpu().numpy(), o_ref)
            assert np.array_equal(seg.kmask.cpu().numpy().view(np.uint64), m_ref)
            # the compact view holds exactly the unpacked records' KE rows
            from paper_1501_04784_b200.device import _dense_rows

            assert _dense_rows(seg).cpu().numpy().tobytes() == ref[:, :36].tobytes()


def test_digest_matches_host_restatement():
    from paper_1501_04784_b200.distributed import digest_words

    ops = CudaOps()
    rng = np.random.default_rng(3)
    a = rng.standard_normal(100_003)
    t = torch.from_numpy(a).to(ops.device)
    got = int(np.int64(ops.digest(t, 12345, 99).item()).astype(np.uint64))
    assert got == digest_words(a, 12345, 99)


@pytest.mark.parametrize("world", [2, 8])
def test_block_digests_sum_to_single_gpu_digest(world):
    from paper_1501_04784_b200.distributed import csc_digest

    mesh = permuted_mesh(perturbed_mesh(10, seed=4), seed=6)
    results = run_loopback(mesh, world, lambda: CudaOps())
    cp, ri, vv = single(mesh)
    want = csc_digest(cp, ri, vv)
    # recompute block digests the way ShardedBuild.block_digest does
    ops = CudaOps()
    tot = np.zeros(3, dtype=np.uint64)
    for r, res in enumerate(results):
        ncols = res.col_hi - res.col_lo
        d = [ops.digest(res.col_ptr[:ncols], res.col_lo, res.nnz_offset)]
        if r == world - 1:
            d[0] = d[0] + ops.digest(res.col_ptr[ncols:], mesh.n_nodes, res.nnz_offset)
        d += [ops.digest(res.row_idx, res.nnz_offset), ops.digest(res.vals, res.nnz_offset)]
        with np.errstate(over="ignore"):
            tot += np.array([int(np.int64(x.item()).astype(np.uint64)) for x in d], dtype=np.uint64)
    assert tuple(int(x) for x in tot) == want


def test_loopback_bad_node_id_raises_node_index_error():
    from paper_1501_04784_b200.errors import MeshValidationError, NodeIndexError

    mesh = perturbed_mesh(6, seed=1)
    conn = mesh.connectivity.copy()
    conn[150, 3] = mesh.n_nodes + 5
    conn[20, 1] = -1  # element 20 < 150: reported
    from paper_1501_04784_b200.mesh import Mesh

    bad = Mesh(coords=mesh.coords, connectivity=conn, coefficient=mesh.coefficient)
    with pytest.raises(NodeIndexError) as ei:
        run_loopback(bad, 3, lambda: CudaOps())
    assert ei.value.element_id == 20 and ei.value.node == -1
    assert isinstance(ei.value, MeshValidationError) and isinstance(ei.value, IndexError)


@pytest.mark.parametrize("kind", ["structured", "permuted"])
def test_column_touch_matches_oracle(kind):
    """hx_column_touch: 8 per (element, distinct histogram bin of its nodes) -- the oracle restatement."""
    from oracle import halo

    mesh = perturbed_mesh(10, seed=3) if kind == "structured" else permuted_mesh(perturbed_mesh(10, seed=3), seed=4)
    ops = X.CudaOps()
    dm = ops.upload(mesh.coords, mesh.connectivity, mesh.coefficient)
    for bins in (1, 7, 300, mesh.n_nodes):
        got = ops.column_touch(dm, mesh.n_nodes, bins).cpu().numpy()
        assert np.array_equal(got, halo.column_touch(mesh.connectivity, mesh.n_nodes, bins))


def test_compact_segments_assemble_like_dense_records():
    """mesh_csc over compact received segments (ke_offset / ke_mask) equals the same assembly over
    unpacked 40-word records, bitwise -- the fast path and the generic fallback (forced by a node of
    valence > 8)."""
    from oracle import halo
    from paper_1501_04784_b200.distributed import balanced_bounds, element_ranges, histogram_bins, record_segment

    for mesh in (permuted_mesh(perturbed_mesh(10, seed=5), seed=6), _valence9_mesh()):
        world = 3
        ops = CudaOps()
        hist = halo.column_weights(mesh.connectivity, mesh.n_nodes, histogram_bins(mesh.n_nodes))
        bounds = balanced_bounds(hist, mesh.n_nodes, world)
        bdev = ops.bounds(bounds)
        ke = np.random.default_rng(1).standard_normal((mesh.n_el, 36))
        lo, hi = element_ranges(mesh.n_el, world)[0]
        dm = ops.upload(mesh.coords, mesh.connectivity[lo:hi], mesh.coefficient[lo:hi])
        per_dest, ws = ops.halo_count(dm, bdev, world, 0)
        want = halo.count(mesh.connectivity[lo:hi], bounds, world, 0)
        chunks = 4 * want[:, 0] + want[:, 1]
        send = ops.alloc_words(int(chunks.sum()))
        offs = np.concatenate([[0], np.cumsum(chunks)[:-1]])
        ops.halo_pack(dm, torch.from_numpy(ke[lo:hi]).cuda(), bdev, world, 0,
                      *ops.pointers([send.data_ptr()] * world, offs), ws)
        d = 2
        desc = np.zeros((world, 3), np.int64)
        desc[0] = (offs[d], want[d, 0], want[d, 1])
        n = int(want[d, 0])
        recs = ops.halo_unpack(send, desc, bdev, world, d, n).clone()
        seg = ops.halo_index(send, desc, bdev, world, d, n)
        c_lo, c_hi = int(bounds[d]), int(bounds[d + 1])
        a = D.mesh_csc([record_segment(recs)], mesh.n_nodes, c_lo, c_hi)
        b = D.mesh_csc([seg], mesh.n_nodes, c_lo, c_hi)
        for x, y in ((a.col_ptr, b.col_ptr), (a.row_idx, b.row_idx), (a.vals, b.vals)):
            assert x.cpu().numpy().tobytes() == y.cpu().numpy().tobytes()


def _valence9_mesh():
    """A perturbed mesh whose element 0 is duplicated: its nodes get valence 9 (generic path)."""
    from paper_1501_04784_b200.mesh import Mesh

    m = perturbed_mesh(6, seed=8)
    conn = np.concatenate([m.connectivity, m.connectivity[:1]])
    return Mesh(m.coords, conn, np.concatenate([m.coefficient, m.coefficient[:1]]))
