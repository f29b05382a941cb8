"""Host-side logic mirrored from the reference (no GPU): batching plan, mesh producer, types."""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from common import bits_equal
from paper_1501_04784_b200 import (
    BatchPlan,
    ConfigurationError,
    MeshValidationError,
    StructuredGridSpec,
    generate_cube_mesh,
    map_local_to_global,
    plan_batches,
    required_bytes,
)
from paper_1501_04784_b200.element import PACK_COLS, PACK_ROWS, pack_lower, unpack_lower
from paper_1501_04784_b200.mesh import validate_mesh
from paper_1501_04784_b200.pipeline import csc_memory, format_mb, format_percent, memory_saving, triplet_memory


def test_required_bytes():
    assert required_bytes(0) == 0
    assert required_bytes(1) == 520
    assert required_bytes(1_000_000) == 520_000_000
    with pytest.raises(ValueError):
        required_bytes(-1)


def test_plan_examples():
    assert plan_batches(4_608_000_000, 2_048_000_000, 8_000_000).group_count == 3
    assert plan_batches(520_000, 10**9, 1000).ranges == ((0, 1000),)
    assert [hi - lo for lo, hi in plan_batches(30, 10, 10).ranges] == [4, 3, 3]
    plan = plan_batches(10**9, 1, 5)
    assert plan.group_count == 5 and all(hi - lo == 1 for lo, hi in plan.ranges)
    with pytest.raises(ConfigurationError):
        plan_batches(100, 0, 10)


@settings(max_examples=200, deadline=None)
@given(mem_required=st.integers(0, 10**12), mem_available=st.integers(1, 10**12), n_el=st.integers(1, 10**4))
def test_plan_invariants(mem_required, mem_available, n_el):
    plan = plan_batches(mem_required, mem_available, n_el)
    r = plan.ranges
    assert r[0][0] == 0 and r[-1][1] == n_el
    assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
    sizes = {hi - lo for lo, hi in r}
    assert max(sizes) - min(sizes) <= 1
    assert plan.group_count == max(1, min(n_el, -(-mem_required // mem_available)))


def test_generator_matches_reference_generator(golden):
    m = generate_cube_mesh(StructuredGridSpec(4, 3, 5, h=0.3, c0=1.7))
    assert bits_equal(m.coords, golden["aniso_coords"])
    assert bits_equal(m.connectivity, golden["aniso_conn"])
    assert bits_equal(m.coefficient, golden["aniso_coeff"])
    validate_mesh(m)


def test_validate_mesh_rejects_bad_meshes():
    m = generate_cube_mesh(StructuredGridSpec(2, 1, 1))
    conn = m.connectivity.copy()
    conn[1, 3] = conn[1, 2]
    with pytest.raises(MeshValidationError):
        validate_mesh(type(m)(m.coords, conn, m.coefficient))
    with pytest.raises(MeshValidationError):
        StructuredGridSpec(0, 1, 1)


def test_map_local_to_global():
    pairs = map_local_to_global(np.arange(8))
    assert np.array_equal(pairs[:, 0], PACK_ROWS) and np.array_equal(pairs[:, 1], PACK_COLS)
    assert tuple(map_local_to_global(np.arange(8)[::-1])[1]) == (7, 6)
    assert map_local_to_global(np.arange(8), dofxn=2).shape == (136, 2)


def test_pack_round_trip():
    v = np.arange(36.0)
    assert np.array_equal(pack_lower(unpack_lower(v)), v)


def test_memory_model_table_rows():
    # test_acceptance.py:46-58 published table, 10^3 and 200^3 rows
    assert format_mb(triplet_memory(36_000)) == "0.58"
    assert format_mb(csc_memory(15_561, 1331)) == "0.26"
    assert format_mb(triplet_memory(288_000_000)) == "4608.0"
    assert format_mb(csc_memory(112_601_201, 201**3)) == "1866.6"
    assert format_percent(memory_saving(triplet_memory(288_000_000), csc_memory(112_601_201, 201**3))) == "59.5%"


def test_batchplan_type():
    assert BatchPlan(ranges=((0, 3),)).group_count == 1


def test_block_ranges_host_scan_matches_numpy():
    """hx_block_ranges (host C++): per column block, the element range whose node span covers it."""
    from paper_1501_04784_b200.distributed import column_bounds
    from paper_1501_04784_b200.stream import block_element_ranges
    from paper_1501_04784_b200.workloads import permuted_mesh, perturbed_mesh

    for mesh in (perturbed_mesh(9, seed=1), permuted_mesh(perturbed_mesh(6, seed=2), seed=3)):
        conn = mesh.connectivity.copy()
        conn[5, 2] = mesh.n_nodes + 7  # out-of-range ids clamp to the last / first block
        conn[11, 0] = -4
        for k in (1, 3, 8, 50):
            bounds = column_bounds(mesh.n_nodes, k)
            lo, hi, n_lo, n_hi = block_element_ranges(conn, bounds, threads=3)
            bmin = np.clip(np.searchsorted(bounds, conn.min(axis=1), side="right") - 1, 0, k - 1)
            bmax = np.clip(np.searchsorted(bounds, conn.max(axis=1), side="right") - 1, 0, k - 1)
            for b in range(k):
                cover = np.flatnonzero((bmin <= b) & (bmax >= b))
                want = (cover.min(), cover.max() + 1) if cover.size else (0, 0)
                assert (lo[b], hi[b]) == want
                if hi[b] > lo[b]:  # the node range covers every node the element range gathers
                    sub = conn[lo[b]:hi[b]]
                    assert n_lo[b] <= max(sub.min(), 0) and n_hi[b] >= sub.max() + 1


def test_sampled_plan_covers_the_exact_plan_on_local_meshes():
    """hx_block_ranges_sampled (every step-th element): on locally numbered meshes the predicted
    element and node ranges contain the exact scan's; a numbering without locality gets None."""
    from paper_1501_04784_b200.stream import plan, sampled_plan
    from paper_1501_04784_b200.workloads import permuted_mesh, perturbed_mesh

    for n, k in ((12, 3), (20, 4), (9, 1)):
        mesh = perturbed_mesh(n, seed=n)
        ex, sm = plan(mesh, k), sampled_plan(mesh, k, step=16)
        assert sm is not None and sm.verify and np.array_equal(sm.bounds, ex.bounds)
        assert np.all(sm.e_lo <= ex.e_lo) and np.all(sm.e_hi >= ex.e_hi)
        assert np.all(sm.node_hi <= mesh.n_nodes)
        for b in range(k):  # the coordinate prefix covers every node the exact range gathers
            assert sm.node_hi[b] >= mesh.connectivity[ex.e_lo[b]:ex.e_hi[b]].max() + 1
        assert sm.e_lo.min() == 0 and sm.e_hi.max() == mesh.n_el
    assert sampled_plan(permuted_mesh(perturbed_mesh(10, seed=1), seed=2), 8) is None


def test_stream_bounds_quarter_end_blocks():
    from paper_1501_04784_b200.stream import stream_bounds

    for n, k in ((1000, 10), (17, 5), (5, 5), (100, 3)):
        b = stream_bounds(n, k)
        assert b[0] == 0 and b[-1] == n and len(b) == k + 1 and np.all(np.diff(b) > 0)
    b = stream_bounds(10_000, 10)
    w = np.diff(b)
    assert abs(w[0] / w[1] - 0.25) < 0.01 and abs(w[-1] / w[-2] - 0.25) < 0.01
