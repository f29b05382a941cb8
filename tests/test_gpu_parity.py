"""GPU parity: the CUDA path through the C ABI vs the oracle / the reference's golden outputs.

Bar: bit-exact for indices and (exact mode) values.
"""

import os

import numpy as np
import pytest
import torch

import oracle
from common import SMALL_MESHES, bits_equal, golden_mesh, sha
from paper_1501_04784_b200 import device as D
from paper_1501_04784_b200 import (
    CudaBackend,
    DegenerateElementError,
    DirectAssembler,
    LocalValuesBatch,
    Mesh,
    MeshValidationError,
    StagingError,
    TripletMatrix,
    assemble_direct,
    build_triplet,
    connectivity_index_arrays,
    integrate_all,
    plan_batches,
    required_bytes,
    run_build,
    stiffness_batch,
    triplet_to_csc,
)
from paper_1501_04784_b200.pipeline import build_device, host_csc_equal
from paper_1501_04784_b200.workloads import make_workload, perturbed_mesh, permuted_mesh

pytestmark = pytest.mark.gpu


def one_group(mesh):
    return plan_batches(required_bytes(mesh.n_el), 10**13, mesh.n_el)


def test_stiffness_batch_bitwise(golden):
    out = stiffness_batch(golden["batch_coords"], golden["batch_coeff"])
    assert bits_equal(out, golden["batch_ke"])


def test_stiffness_batch_block_boundaries(golden):
    coords, coeff = golden["batch_coords"], golden["batch_coeff"]
    full = stiffness_batch(coords, coeff)
    pieces = np.vstack([stiffness_batch(coords[lo:lo + 13], coeff[lo:lo + 13]) for lo in range(0, len(coeff), 13)])
    assert bits_equal(full, pieces)


@pytest.mark.parametrize("name", SMALL_MESHES)
def test_integrate_mesh_fused_index_bitwise(golden, name):
    dm = D.DeviceMesh.from_host(golden_mesh(golden, name))
    ke, rows, cols, fail = D.integrate_mesh(dm)
    D.raise_if_failed(fail)
    assert bits_equal(ke.cpu().numpy(), golden[f"{name}_ke"])
    assert bits_equal(rows.cpu().numpy(), golden[f"{name}_rows"])
    assert bits_equal(cols.cpu().numpy(), golden[f"{name}_cols"])


@pytest.mark.parametrize("name", SMALL_MESHES)
def test_mesh_csc_bitwise(golden, name):
    mesh = golden_mesh(golden, name)
    build = build_device(D.DeviceMesh.from_host(mesh))
    assert build.csc.path == "mesh"
    assert bits_equal(build.csc.col_ptr.cpu().numpy(), golden[f"{name}_col_ptr"])
    assert bits_equal(build.csc.row_idx.cpu().numpy(), golden[f"{name}_row_idx"])
    assert bits_equal(build.csc.vals.cpu().numpy(), golden[f"{name}_vals"])


@pytest.mark.parametrize("name", SMALL_MESHES)
def test_triplet_to_csc_generic_bitwise(golden, name):
    t = TripletMatrix(rows=golden[f"{name}_rows"], cols=golden[f"{name}_cols"],
                      vals=golden[f"{name}_ke"].reshape(-1), dim=golden[f"{name}_coords"].shape[0])
    m = triplet_to_csc(t)
    assert bits_equal(m.col_ptr, golden[f"{name}_col_ptr"])
    assert bits_equal(m.row_idx, golden[f"{name}_row_idx"])
    assert bits_equal(m.vals, golden[f"{name}_vals"])


def test_generic_triplets_long_runs_pairwise_rule(golden):
    dim = int(golden["trip_dim"][0])
    m = triplet_to_csc(TripletMatrix(golden["trip_rows"], golden["trip_cols"], golden["trip_vals"], dim))
    assert bits_equal(m.col_ptr, golden["trip_col_ptr"])
    assert bits_equal(m.row_idx, golden["trip_row_idx"])
    assert bits_equal(m.vals, golden["trip_out"])


def test_random_triplets_against_oracle():
    rng = np.random.default_rng(7)
    for n, dim in [(1, 1), (50, 3), (5000, 40), (20000, 7)]:
        r = rng.integers(0, dim, size=n).astype(np.int32)
        c = rng.integers(0, dim, size=n).astype(np.int32)
        rows, cols = np.maximum(r, c), np.minimum(r, c)
        vals = rng.standard_normal(n) * np.exp(rng.uniform(-10, 10, size=n))
        m = triplet_to_csc(TripletMatrix(rows, cols, vals, dim))
        cp, ri, vv = oracle.triplet_to_csc(rows, cols, vals, dim)
        assert bits_equal(m.col_ptr, cp) and bits_equal(m.row_idx, ri) and bits_equal(m.vals, vv)


def test_triplet_edge_cases():
    m = triplet_to_csc(TripletMatrix(np.array([2, 2, 1], np.int32), np.array([0, 0, 1], np.int32),
                                     np.array([1.5, -1.5, 3.0]), 3))
    assert np.array_equal(m.row_idx, [2, 1]) and np.array_equal(m.vals, [0.0, 3.0])
    empty = triplet_to_csc(TripletMatrix(np.empty(0, np.int32), np.empty(0, np.int32), np.empty(0), 3))
    assert empty.nnz == 0 and np.array_equal(empty.col_ptr, np.zeros(4, np.int64))
    with pytest.raises(MeshValidationError):
        triplet_to_csc(TripletMatrix(np.array([5], np.int32), np.array([0], np.int32), np.array([1.0]), 4))
    with pytest.raises(MeshValidationError):
        triplet_to_csc(TripletMatrix(np.array([0], np.int32), np.array([2], np.int32), np.array([1.0]), 4))


def test_connectivity_index_arrays_ranges(golden):
    mesh = golden_mesh(golden, "perm5")
    for lo, hi in [(0, None), (3, 17), (0, 1), (124, 125)]:
        r, c = connectivity_index_arrays(mesh, lo, hi)
        r2, c2 = oracle.connectivity_index_arrays(mesh.connectivity, lo, hi)
        assert bits_equal(r, r2) and bits_equal(c, c2)


def test_degenerate_reports_first_element(golden):
    mesh = Mesh(golden["degen_coords"], golden["degen_conn"], np.ones(golden["degen_conn"].shape[0]))
    exp_el, exp_gp = golden["degen_expect"]
    with CudaBackend() as backend, pytest.raises(DegenerateElementError) as info:
        integrate_all(mesh, backend, one_group(mesh))
    assert info.value.element_id == exp_el and info.value.gauss_point == exp_gp
    assert info.value.det == golden["degen_det"][0]
    with pytest.raises(DegenerateElementError) as info:
        stiffness_batch(mesh.coords[mesh.connectivity], mesh.coefficient, element_offset=100)
    assert info.value.element_id == 100 + exp_el


def test_integrate_all_plans_modes_bitwise(golden):
    mesh = golden_mesh(golden, "m345")
    ref = golden["m345_ke"]
    with CudaBackend() as backend:
        for budget in (10**13, required_bytes(7), 520):
            plan = plan_batches(required_bytes(mesh.n_el), budget, mesh.n_el)
            seen = []
            for mode in ("sequential", "overlapped"):
                seen.clear()
                batch = integrate_all(mesh, backend, plan, mode=mode, consumer=lambda r, v: seen.append((r, v.copy())))
                assert bits_equal(batch.values, ref)
                assert [r for r, _ in seen] == list(plan.ranges)
                assert bits_equal(np.vstack([v for _, v in seen]), ref)


def test_integrate_all_host_staged_run(golden):
    """ComputeBackend.run drop-in (host staged coords) gives the same bits."""
    mesh = golden_mesh(golden, "perm5")
    with CudaBackend() as backend:
        out = np.empty((mesh.n_el, 36))
        backend.run(mesh.coords[mesh.connectivity], mesh.coefficient, out=out)
    assert bits_equal(out, golden["perm5_ke"])


def test_staging_error_and_consumer_errors(golden):
    mesh = golden_mesh(golden, "m345")
    with CudaBackend(capacity_bytes=required_bytes(3)) as backend, pytest.raises(StagingError) as info:
        integrate_all(mesh, backend, one_group(mesh))
    assert info.value.group_index == 0

    def bad(rng, values):
        raise RuntimeError("downstream failed")

    with CudaBackend() as backend, pytest.raises(RuntimeError, match="downstream"):
        integrate_all(mesh, backend, plan_batches(required_bytes(27), required_bytes(5), 27), mode="overlapped",
                      consumer=bad)


def test_direct_assembler_streaming_and_order(golden):
    mesh = golden_mesh(golden, "perm5")
    values = golden["perm5_ke"]
    one = assemble_direct(mesh, LocalValuesBatch(values))
    streamed = DirectAssembler(mesh)
    for lo, hi in plan_batches(required_bytes(mesh.n_el), required_bytes(37), mesh.n_el).ranges:
        streamed.consume((lo, hi), values[lo:hi])
    two = streamed.finish()
    assert host_csc_equal(one, two)
    assert bits_equal(one.vals, golden["perm5_vals"])
    a = DirectAssembler(mesh)
    with pytest.raises(ValueError, match="order"):
        a.consume((4, 8), values[4:8])
    a.consume((0, 4), values[:4])
    with pytest.raises(ValueError, match="consumed"):
        a.finish()


def test_run_build_both_assemblers(golden):
    mesh = golden_mesh(golden, "m345")
    for assembler in ("direct", "triplet"):
        m, report = run_build(mesh, budget_bytes=required_bytes(10), assembler=assembler)
        assert bits_equal(m.vals, golden["m345_vals"]) and bits_equal(m.row_idx, golden["m345_row_idx"])
        assert report.group_count == 3 and report.nnz_csc == m.nnz
        assert abs(report.pct_integration + report.pct_assembly - 100.0) < 1e-9


def _high_valence_mesh(rng):
    """A mesh whose node 0 touches 11 elements (beyond the fast path's degree limit)."""
    base = perturbed_mesh(2, seed=1)
    extra = []
    for _ in range(4):
        others = rng.choice(np.arange(1, base.n_nodes), size=7, replace=False)
        extra.append(np.concatenate([[0], others]).astype(np.int32))
    conn = np.vstack([base.connectivity, np.array(extra)])
    return Mesh(base.coords, conn, np.ones(conn.shape[0]))


def test_fast_path_limits_fall_back_bitwise():
    rng = np.random.default_rng(3)
    mesh = _high_valence_mesh(rng)
    values = rng.standard_normal((mesh.n_el, 36))
    m = assemble_direct(mesh, LocalValuesBatch(values))
    rows, cols = oracle.connectivity_index_arrays(mesh.connectivity)
    cp, ri, vv = oracle.triplet_to_csc(rows, cols, values.reshape(-1), mesh.n_nodes)
    assert bits_equal(m.col_ptr, cp) and bits_equal(m.row_idx, ri) and bits_equal(m.vals, vv)
    # repeated node inside an element
    conn = mesh.connectivity.copy()
    conn[0, 5] = conn[0, 4]
    m2 = assemble_direct(Mesh(mesh.coords, conn, mesh.coefficient), LocalValuesBatch(values))
    rows, cols = oracle.connectivity_index_arrays(conn)
    cp, ri, vv = oracle.triplet_to_csc(rows, cols, values.reshape(-1), mesh.n_nodes)
    assert bits_equal(m2.col_ptr, cp) and bits_equal(m2.row_idx, ri) and bits_equal(m2.vals, vv)


def test_mesh_assembly_random_values_random_numbering():
    """Assembly is value-agnostic: random KE values + permuted numbering vs the oracle."""
    rng = np.random.default_rng(11)
    for n in (1, 2, 7):
        mesh = permuted_mesh(perturbed_mesh(n, seed=n), seed=n + 1)
        values = rng.standard_normal((mesh.n_el, 36)) * np.exp(rng.uniform(-5, 5, size=(mesh.n_el, 36)))
        m = assemble_direct(mesh, LocalValuesBatch(values))
        rows, cols = oracle.connectivity_index_arrays(mesh.connectivity)
        cp, ri, vv = oracle.triplet_to_csc(rows, cols, values.reshape(-1), mesh.n_nodes)
        assert bits_equal(m.col_ptr, cp) and bits_equal(m.row_idx, ri) and bits_equal(m.vals, vv)


@pytest.mark.parametrize("config", ["C1", "C2", "P64", "C3", "C5"])
def test_full_pipeline_matches_reference_digests(digests, config):
    d = digests["configs"][config]
    if config == "P64":
        mesh = permuted_mesh(perturbed_mesh(64, seed=0), seed=5)
    else:
        mesh = make_workload(config)
    dm = D.DeviceMesh.from_host(mesh)
    b = build_device(dm)
    assert b.csc.path == "mesh" and b.csc.nnz == d["nnz"]
    assert sha(b.ke.cpu().numpy()) == d["ke"]
    assert sha(b.rows.cpu().numpy()) == d["rows"] and sha(b.cols.cpu().numpy()) == d["cols"]
    assert sha(b.csc.col_ptr.cpu().numpy()) == d["col_ptr"]
    assert sha(b.csc.row_idx.cpu().numpy()) == d["row_idx"]
    assert sha(b.csc.vals.cpu().numpy()) == d["vals"]
    del b, dm
    torch.cuda.empty_cache()


def test_operator_properties_full_size():
    """Size-independent properties at BASELINE scale (C2): K 1 = 0, symmetric pattern invariants."""
    mesh = make_workload("C2")
    b = build_device(D.DeviceMesh.from_host(mesh))
    cp, ri, vv = b.csc.col_ptr, b.csc.row_idx, b.csc.vals
    ncol = mesh.n_nodes
    col_of = torch.repeat_interleave(torch.arange(ncol, device=cp.device), cp[1:] - cp[:-1])
    assert bool((ri >= col_of).all())
    same = col_of[1:] == col_of[:-1]
    assert bool((ri[1:][same] > ri[:-1][same]).all())
    # K 1 = 0: row sums of the full symmetric matrix
    rs = torch.zeros(ncol, dtype=torch.float64, device=cp.device)
    rs.index_add_(0, ri, vv)
    off = ri != col_of
    rs.index_add_(0, col_of[off], vv[off])
    assert float(rs.abs().max()) <= 1e-10 * float(vv.abs().max()) * 27


def test_exact_division_selftest():
    """Reciprocal + Markstein quotient == IEEE division, bit for bit, on 2^30 operand pairs."""
    from paper_1501_04784_b200 import _native as N

    res = torch.zeros(2, dtype=torch.int64, device="cuda")
    N.check(N.lib().hx_selftest_division(1 << 30, 12345, D._ptr(res), D.stream_handle()), "selftest")
    mismatches, tested = res.cpu().tolist()
    assert tested > (1 << 29)
    assert mismatches == 0


def test_random_elements_bitwise_against_oracle():
    """1M random valid hexahedra (distortion up to 0.3, wide coefficient/scale range) vs the oracle."""
    rng = np.random.default_rng(2024)
    n = 1 << 20
    corners = (np.array([(-1, -1, -1), (1, -1, -1), (1, 1, -1), (-1, 1, -1), (-1, -1, 1), (1, -1, 1), (1, 1, 1),
                         (-1, 1, 1)], dtype=float) + 1.0) / 2.0
    scale = np.exp(rng.uniform(-20, 20, size=(n, 1, 1)))
    coords = (corners[None] + rng.uniform(-0.2, 0.2, size=(n, 8, 3)) + rng.uniform(-10, 10, size=(n, 1, 3))) * scale
    coeff = np.exp(rng.uniform(-10, 10, size=n))
    ref, first, _, _ = oracle.stiffness_batch(coords, coeff)
    assert first == -1
    got = stiffness_batch(coords, coeff)
    assert bits_equal(got, ref)


@pytest.mark.parametrize("permute", [False, True])
def test_unreferenced_nodes_give_empty_columns(permute):
    """Nodes no element references (allowed by validate_mesh, mesh.py:100-119) are empty columns;
    they must not shift the other columns' records (every second id unused, some runs of 3)."""
    base = perturbed_mesh(7, seed=12)
    if permute:
        base = permuted_mesh(base, seed=13)
    old = np.arange(base.n_nodes)
    new_id = 2 * old + (old % 5 == 0)  # gaps of 1 and 2 between used ids
    n_nodes = int(new_id.max()) + 3
    coords = np.zeros((n_nodes, 3))
    coords[new_id] = base.coords
    mesh = Mesh(coords, new_id.astype(np.int32)[base.connectivity], base.coefficient)
    b = build_device(D.DeviceMesh.from_host(mesh))
    assert b.csc.path == "mesh"
    ke, rows, cols, first, _, _ = oracle.stiffness_mesh(mesh.coords, mesh.connectivity, mesh.coefficient)
    cp, ri, vv = oracle.triplet_to_csc(rows, cols, ke.reshape(-1), mesh.n_nodes)
    assert bits_equal(b.csc.col_ptr.cpu().numpy(), cp)
    assert bits_equal(b.csc.row_idx.cpu().numpy(), ri)
    assert bits_equal(b.csc.vals.cpu().numpy(), vv)


@pytest.mark.parametrize("flags", [0, 1])
@pytest.mark.parametrize("name", SMALL_MESHES)
def test_symbolic_rows_only_abi(golden, name, flags):
    """hx_mesh_csc_symbolic with a row buffer: the pattern without values (rows-only emit)."""
    import ctypes

    from paper_1501_04784_b200 import _native as N

    mesh = golden_mesh(golden, name)
    conn = torch.from_numpy(mesh.connectivity).cuda()
    n, dim = mesh.n_el, mesh.n_nodes
    ws_bytes = N.lib().hx_mesh_csc_workspace_bytes(n, dim)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    col_ptr = torch.empty(dim + 1, dtype=torch.int64, device="cuda")
    rows = torch.empty(36 * n, dtype=torch.int64, device="cuda")
    segs = N.segments([(conn.data_ptr(), 0, n)])
    N.check(N.lib().hx_mesh_csc_symbolic(segs, 1, dim, 0, dim, D._ptr(col_ptr), D._ptr(rows), 36 * n, D._ptr(ws),
                                         ws_bytes, D._ptr(status), flags, D.stream_handle()), "symbolic")
    assert int(status.item()) == 0
    nnz = int(col_ptr[-1].item())
    assert bits_equal(col_ptr.cpu().numpy(), golden[f"{name}_col_ptr"])
    assert bits_equal(rows[:nnz].cpu().numpy(), golden[f"{name}_row_idx"])


@pytest.mark.parametrize("order", ["column", "element"])
@pytest.mark.parametrize("kind", ["structured", "permuted", "gaps"])
def test_assembly_orders_bitwise(order, kind):
    """Both column processing orders give the reference's bits (structured, permuted numbering,
    unreferenced nodes)."""
    mesh = perturbed_mesh(11, seed=21)
    if kind == "permuted":
        mesh = permuted_mesh(mesh, seed=22)
    elif kind == "gaps":
        new_id = 3 * np.arange(mesh.n_nodes)
        coords = np.zeros((3 * mesh.n_nodes, 3))
        coords[new_id] = mesh.coords
        mesh = Mesh(coords, new_id.astype(np.int32)[mesh.connectivity], mesh.coefficient)
    dm = D.DeviceMesh.from_host(mesh)
    ke, _, _, fail = D.integrate_mesh(dm)
    D.raise_if_failed(fail)
    csc = D.mesh_csc([(dm.conn, ke)], mesh.n_nodes, order=order)
    plan = D.mesh_plan_async(dm.conn, mesh.n_nodes, order=order)
    csc2 = D.mesh_emit(plan, ke)
    rows, cols = oracle.connectivity_index_arrays(mesh.connectivity)
    cp, ri, vv = oracle.triplet_to_csc(rows, cols, ke.cpu().numpy().reshape(-1), mesh.n_nodes)
    for c in (csc, csc2):
        assert c.path == "mesh"
        assert bits_equal(c.col_ptr.cpu().numpy(), cp)
        assert bits_equal(c.row_idx.cpu().numpy(), ri)
        assert bits_equal(c.vals.cpu().numpy(), vv)


@pytest.mark.parametrize("blocks", [1, 2, 5, 13])
@pytest.mark.parametrize("kind", ["structured", "permuted"])
def test_out_of_core_blocks_bitwise(blocks, kind):
    """Column blocks built one at a time (halo elements recomputed) == the one-shot build, bit for bit."""
    from paper_1501_04784_b200.pipeline import build_out_of_core

    mesh = perturbed_mesh(10, seed=31)
    if kind == "permuted":
        mesh = permuted_mesh(mesh, seed=32)
    m, values, stats = build_out_of_core(mesh, blocks, return_values=True)
    ke, rows, cols, first, _, _ = oracle.stiffness_mesh(mesh.coords, mesh.connectivity, mesh.coefficient)
    cp, ri, vv = oracle.triplet_to_csc(rows, cols, ke.reshape(-1), mesh.n_nodes)
    assert bits_equal(m.col_ptr, cp) and bits_equal(m.row_idx, ri) and bits_equal(m.vals, vv)
    assert bits_equal(values, ke)
    assert stats["blocks"] == blocks


def test_out_of_core_degenerate_and_budget(golden):
    from paper_1501_04784_b200.pipeline import build_out_of_core, device_bytes

    mesh = Mesh(golden["degen_coords"], golden["degen_conn"], np.ones(golden["degen_conn"].shape[0]))
    exp_el, exp_gp = golden["degen_expect"]
    with pytest.raises(DegenerateElementError) as info:
        build_out_of_core(mesh, 3)
    assert info.value.element_id == exp_el and info.value.gauss_point == exp_gp
    good = golden_mesh(golden, "m345")
    budget = device_bytes(good.n_el, good.n_nodes) // 4
    m, report = run_build(good, budget_bytes=10**12, device_budget_bytes=budget)
    assert bits_equal(m.vals, golden["m345_vals"]) and bits_equal(m.row_idx, golden["m345_row_idx"])
    assert abs(report.pct_integration + report.pct_assembly - 100.0) < 1e-9


def test_numbering_heuristic_large_index_range():
    """The locality probe samples element rows by index: exact at 64M elements (no float rounding)."""
    n = 64_000_000
    conn = torch.zeros((n, 8), dtype=torch.int32, device="cuda")
    conn[-1] = torch.arange(8, dtype=torch.int32, device="cuda") * 1_000_000
    assert D.numbering_is_local(conn, 64_481_201) in (True, False)
    torch.cuda.synchronize()
    del conn
    torch.cuda.empty_cache()


def test_matrix_market_round_trip(tmp_path, golden):
    """export (native writer) -> import (reference line rules, GPU triplet_to_csc) reproduces K."""
    from paper_1501_04784_b200 import LowerCscMatrix, MeshFormatError, export_matrix_market, import_matrix_market

    m = LowerCscMatrix(golden["perm5_col_ptr"], golden["perm5_row_idx"], golden["perm5_vals"],
                       golden["perm5_coords"].shape[0])
    path = tmp_path / "k.mtx"
    export_matrix_market(m, path)
    back = import_matrix_market(path)
    assert host_csc_equal(back, m)
    crlf = tmp_path / "crlf.mtx"  # outside the native reader's strict subset: the reference's rules
    crlf.write_bytes(path.read_bytes().replace(b"\n", b"\r\n"))
    assert host_csc_equal(import_matrix_market(crlf), m)
    path.write_text("%%MatrixMarket matrix coordinate real symmetric\n3 3 1\n1 2 4.0\n")
    with pytest.raises(MeshFormatError, match="above the diagonal"):
        import_matrix_market(path)


@pytest.mark.parametrize("dims", [(1, 1, 1), (4, 3, 5), (37, 2, 9), (100, 100, 100)])
def test_device_cube_generator_bitwise(dims):
    """hx_generate_cube_mesh == generate_cube_mesh (mesh.py:73-98 numbering and coordinates)."""
    from paper_1501_04784_b200 import StructuredGridSpec, generate_cube_mesh

    spec = StructuredGridSpec(*dims, h=0.37, c0=1.7)
    host = generate_cube_mesh(spec)
    dm = D.generate_cube_mesh(spec)
    assert bits_equal(dm.coords.cpu().numpy(), host.coords)
    assert bits_equal(dm.conn.cpu().numpy(), host.connectivity)
    assert bits_equal(dm.coeff.cpu().numpy(), host.coefficient)


def test_planned_rebuild_new_coefficients():
    """A verified plan (connectivity only) reused for a rebuild with new coordinates/coefficients
    gives the one-shot build's bits; degenerate elements are still reported (DeviceBuild.check)."""
    from paper_1501_04784_b200.pipeline import build_device

    mesh = permuted_mesh(perturbed_mesh(12, seed=61), seed=62)
    dm = D.DeviceMesh.from_host(mesh)
    plan = D.plan_assembly(dm)
    assert plan is not None and plan.nnz > 0
    for seed in (1, 2):
        rng = np.random.default_rng(seed)
        dm.coeff.copy_(torch.from_numpy(rng.uniform(0.5, 2.0, size=mesh.n_el)))
        warm = build_device(dm, plan=plan).check()
        cold = build_device(D.DeviceMesh(dm.coords, dm.conn, dm.coeff.clone()))
        assert bits_equal(warm.csc.vals.cpu().numpy(), cold.csc.vals.cpu().numpy())
        assert bits_equal(warm.csc.row_idx.cpu().numpy(), cold.csc.row_idx.cpu().numpy())
    flipped = dm.coords.clone()
    dm2 = D.DeviceMesh(flipped, dm.conn, dm.coeff)
    dm2.coords[:, 2] *= -1.0  # mirror: every det < 0
    with pytest.raises(DegenerateElementError):
        build_device(dm2, plan=plan).check()


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_random_mesh_variants_full_pipeline_bitwise(seed):
    """Shuffled element order, deleted elements (holes -> boundary columns and unreferenced nodes),
    permuted node ids and random distortion/coefficients: the full pipeline (KE, iK/jK, CSC) stays
    bitwise equal to the oracle."""
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(3, 11))
    mesh = perturbed_mesh(n, seed=seed, distortion=0.2)
    keep = rng.random(mesh.n_el) > 0.25
    keep[0] = True
    conn = mesh.connectivity[keep]
    coeff = mesh.coefficient[keep] * np.exp(rng.uniform(-3, 3, size=keep.sum()))
    order = rng.permutation(conn.shape[0])
    conn, coeff = conn[order], coeff[order]
    mesh = Mesh(mesh.coords, np.ascontiguousarray(conn), np.ascontiguousarray(coeff))
    if seed % 2:
        mesh = permuted_mesh(mesh, seed=seed + 7)
    b = build_device(D.DeviceMesh.from_host(mesh))
    ke, rows, cols, first, _, _ = oracle.stiffness_mesh(mesh.coords, mesh.connectivity, mesh.coefficient)
    assert first == -1
    cp, ri, vv = oracle.triplet_to_csc(rows, cols, ke.reshape(-1), mesh.n_nodes)
    assert bits_equal(b.ke.cpu().numpy(), ke)
    assert bits_equal(b.rows.cpu().numpy(), rows) and bits_equal(b.cols.cpu().numpy(), cols)
    assert bits_equal(b.csc.col_ptr.cpu().numpy(), cp)
    assert bits_equal(b.csc.row_idx.cpu().numpy(), ri)
    assert bits_equal(b.csc.vals.cpu().numpy(), vv)


@pytest.mark.parametrize("name", SMALL_MESHES)
def test_symbolic_then_numeric_abi(golden, name):
    """hx_mesh_csc_symbolic (pattern + rows) followed by hx_mesh_csc_numeric (values only) on the same
    workspace: the reference's CSC."""
    from paper_1501_04784_b200 import _native as N

    mesh = golden_mesh(golden, name)
    dm = D.DeviceMesh.from_host(mesh)
    ke, _, _, fail = D.integrate_mesh(dm, with_index=False)
    n, dim = mesh.n_el, mesh.n_nodes
    ws_bytes = N.lib().hx_mesh_csc_workspace_bytes(n, dim)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    col_ptr = torch.empty(dim + 1, dtype=torch.int64, device="cuda")
    rows = torch.empty(36 * n, dtype=torch.int64, device="cuda")
    segs = N.segments([(dm.conn.data_ptr(), ke.data_ptr(), n)])
    sh = D.stream_handle()
    N.check(N.lib().hx_mesh_csc_symbolic(segs, 1, dim, 0, dim, D._ptr(col_ptr), D._ptr(rows), 36 * n, D._ptr(ws),
                                         ws_bytes, D._ptr(status), 0, sh), "symbolic")
    nnz = int(col_ptr[-1].item())
    vals = torch.empty(nnz, dtype=torch.float64, device="cuda")
    N.check(N.lib().hx_mesh_csc_numeric(segs, 1, 0, dim, D._ptr(col_ptr), D._ptr(rows), D._ptr(vals), D._ptr(ws),
                                        D._ptr(status), sh), "numeric")
    assert int(status.item()) == 0
    assert bits_equal(rows[:nnz].cpu().numpy(), golden[f"{name}_row_idx"])
    assert bits_equal(vals.cpu().numpy(), golden[f"{name}_vals"])


def _star_mesh(shared):
    """8 elements around node 0; with shared=False they share only node 0 (56 distinct rows in
    column 0 > the 32-slot fast path), with shared=True all 8 also share node 1 (edge (0, 1) carried
    by 8 elements > 4 contributions)."""
    rng = np.random.default_rng(5 if shared else 6)
    conn = []
    nxt = 2 if shared else 1
    for e in range(8):
        others = list(range(nxt, nxt + (6 if shared else 7)))
        nxt += 6 if shared else 7
        nodes = [0, 1] + others if shared else [0] + others
        conn.append(nodes)
    conn = np.array(conn, dtype=np.int32)
    n_nodes = int(conn.max()) + 1
    # geometry irrelevant for assembly: random values through the assembly-only entry point
    return conn, n_nodes, rng.standard_normal((8, 36))


@pytest.mark.parametrize("shared", [False, True])
def test_fast_path_row_limits_fall_back_bitwise(shared):
    conn, n_nodes, values = _star_mesh(shared)
    mesh = Mesh(np.zeros((n_nodes, 3)), conn, np.ones(conn.shape[0]))
    m = assemble_direct(mesh, LocalValuesBatch(values))
    rows, cols = oracle.connectivity_index_arrays(conn)
    cp, ri, vv = oracle.triplet_to_csc(rows, cols, values.reshape(-1), n_nodes)
    assert bits_equal(m.col_ptr, cp) and bits_equal(m.row_idx, ri) and bits_equal(m.vals, vv)


_C4 = {}


def _c4_block(bounds):
    """One column block of the C4 check, run in a forked worker (numpy only, no CUDA): the
    reference algorithm on the elements touching the block, compared with the GPU's block."""
    c0, c1 = bounds
    g = _C4
    conn = g["conn"]
    cand = np.flatnonzero((g["emin"] < c1) & (g["emax"] >= c0))
    sub = conn[cand]
    touch = cand[((sub >= c0) & (sub < c1)).any(axis=1)]  # ascending element ids
    c = conn[touch]
    r = np.maximum(c[:, oracle.PACK_ROWS], c[:, oracle.PACK_COLS]).reshape(-1)
    k = np.minimum(c[:, oracle.PACK_ROWS], c[:, oracle.PACK_COLS]).reshape(-1)
    keep = (k >= c0) & (k < c1)
    cp, ri, vv = oracle.triplet_to_csc_columns(r[keep], k[keep], g["ke"][touch].reshape(-1)[keep], c0, c1)
    gcp = g["col_ptr"][c0:c1 + 1]
    a, z = int(gcp[0]), int(gcp[-1])
    return (np.array_equal(gcp - a, cp), np.array_equal(g["row_idx"][a:z], ri),
            np.array_equal(g["vals"][a:z].view(np.int64), vv.view(np.int64)))


@pytest.mark.slow
def test_c4_every_column_bitwise_against_oracle():
    """C4 (400^3, 64M elements) checked whole: the oracle's KE for every element (C, all host
    cores), iK/jK for every element, and every column of the lower CSC assembled by the reference
    algorithm (numpy lexsort + add.reduceat) in 32 column blocks on forked host workers -- bitwise
    against the single-GPU build (replaces round 1's three 4000-column windows)."""
    import multiprocessing as mp

    mesh = make_workload("C4")
    dm = D.DeviceMesh.from_host(mesh)
    b = build_device(dm)
    torch.cuda.synchronize()
    ke_o, _, _, first, _, _ = oracle.stiffness_mesh(mesh.coords, mesh.connectivity, mesh.coefficient,
                                                    with_index=False)
    assert first == -1
    step = 1 << 23
    for lo in range(0, mesh.n_el, step):  # KE and the fused iK/jK, element chunks
        hi = min(lo + step, mesh.n_el)
        assert np.array_equal(b.ke[lo:hi].cpu().numpy().view(np.int64), ke_o[lo:hi].view(np.int64))
        r, k = oracle.connectivity_index_arrays(mesh.connectivity, lo, hi)
        assert np.array_equal(b.rows[36 * lo:36 * hi].cpu().numpy(), r)
        assert np.array_equal(b.cols[36 * lo:36 * hi].cpu().numpy(), k)
    _C4.update(conn=mesh.connectivity, ke=ke_o, emin=mesh.connectivity.min(axis=1), emax=mesh.connectivity.max(axis=1),
               col_ptr=b.csc.col_ptr.cpu().numpy(), row_idx=b.csc.row_idx.cpu().numpy(), vals=b.csc.vals.cpu().numpy())
    assert int(_C4["col_ptr"][-1]) == b.csc.nnz == 898_402_401
    del b, dm
    torch.cuda.empty_cache()
    n = mesh.n_nodes
    blocks = [(n * i // 32, n * (i + 1) // 32) for i in range(32)]
    try:
        with mp.get_context("fork").Pool(min(16, os.cpu_count() or 1)) as pool:
            results = pool.map(_c4_block, blocks)
    finally:
        _C4.clear()
    assert all(all(r) for r in results), [i for i, r in enumerate(results) if not all(r)]


def test_c4_streamed_run_build_bitwise_to_device_build():
    """The e2e entry point at full size: run_build on C4 from pinned host memory (20 streamed column
    blocks, sampled block plan checked on the device, delta-encoded row transfer decoded on the host)
    returns exactly the single-GPU device build's CSC (which the test above pins to the oracle)."""
    from paper_1501_04784_b200 import pipeline
    from paper_1501_04784_b200.hostmem import pinned_mesh

    mesh = make_workload("C4")
    dm = D.DeviceMesh.from_host(mesh)
    b = build_device(dm)
    torch.cuda.synchronize()
    cp, ri, vv = b.csc.col_ptr.cpu().numpy(), b.csc.row_idx.cpu().numpy(), b.csc.vals.cpu().numpy()
    del b, dm
    torch.cuda.empty_cache()
    m, rep = run_build(pinned_mesh(mesh), budget_bytes=10**13)
    st = pipeline.LAST_RUN_STATS
    from paper_1501_04784_b200.transfer import row_codec_enabled

    assert st.get("blocks", 0) >= 10 and not st.get("sampled_plan_fallback")
    assert (st.get("row_codec_blocks", 0) > 0) == row_codec_enabled()  # HX_ROW_CODEC=0: int32 rows
    assert np.array_equal(m.col_ptr, cp) and np.array_equal(m.row_idx, ri)
    assert np.array_equal(m.vals.view(np.int64), vv.view(np.int64))


def test_empty_and_single_element_meshes():
    """Edge sizes the reference accepts: zero elements (test_assemble.py:212-222 empty-triplet rule,
    stiffness_batch -> (0, 36), assemble_direct -> all-zero col_ptr; run_build rejects it through
    plan_batches, integrate.py:70-71) and a single unit-cube element (test_element.py:133-136)."""
    empty = Mesh(np.zeros((5, 3)), np.empty((0, 8), np.int32), np.empty(0))
    assert stiffness_batch(np.empty((0, 8, 3)), np.empty(0)).shape == (0, 36)
    r, c = connectivity_index_arrays(empty)
    assert r.dtype == np.int32 and r.size == 0 and c.size == 0
    for m in (assemble_direct(empty, LocalValuesBatch(np.empty((0, 36)))),
              triplet_to_csc(build_triplet(empty, LocalValuesBatch(np.empty((0, 36)))))):
        assert m.dim == 5 and np.array_equal(m.col_ptr, np.zeros(6, np.int64)) and m.nnz == 0
        assert m.row_idx.dtype == np.int64 and m.vals.dtype == np.float64
    dm = D.DeviceMesh.from_host(empty)
    ke, _, _, fail = D.integrate_mesh(dm)
    D.raise_if_failed(fail)
    assert tuple(ke.shape) == (0, 36)
    assert np.array_equal(D.mesh_csc([(dm.conn, ke)], dm.n_nodes).col_ptr.cpu().numpy(), np.zeros(6, np.int64))
    with pytest.raises(ValueError):
        run_build(empty, 1 << 20)

    corners = np.array([(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0), (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1)],
                       float)
    one = Mesh(corners, np.arange(8, dtype=np.int32)[None], np.ones(1))
    ke_ref, rows, cols, first, _, _ = oracle.stiffness_mesh(one.coords, one.connectivity, one.coefficient)
    cp, ri, vv = oracle.triplet_to_csc(rows, cols, ke_ref.reshape(-1), 8)
    for assembler in ("direct", "triplet"):
        m, rep = run_build(one, 1 << 20, assembler=assembler)
        assert rep.nnz_csc == 36 and rep.n_el == 1
        assert bits_equal(m.col_ptr, cp) and bits_equal(m.row_idx, ri) and bits_equal(m.vals, vv)


def test_generic_triplet_path_beyond_int32_triplets():
    """C4 through the triplet assembler: 36 * 64M = 2.30e9 triplets (> 2^31, 64-bit offsets in the
    sort, run detection and pairwise gather) must give the same CSC, bit for bit, as the fused
    direct path (itself checked against the oracle by test_full_size_column_windows_bitwise)."""
    mesh = make_workload("C4")
    dm = D.DeviceMesh.from_host(mesh)
    del mesh
    ke, rows, cols, fail = D.integrate_mesh(dm, with_index=True)
    D.raise_if_failed(fail)
    assert rows.shape[0] > 2**31
    direct = D.mesh_csc([(dm.conn, ke)], dm.n_nodes)
    d_ptr, d_rows, d_vals = direct.col_ptr, direct.row_idx.to(torch.int32), direct.vals
    del direct
    torch.cuda.empty_cache()
    trip = D.triplet_csc(rows, cols, ke.view(-1), dm.n_nodes)
    assert torch.equal(trip.col_ptr, d_ptr)
    assert torch.equal(trip.row_idx.to(torch.int32), d_rows)
    assert torch.equal(trip.vals.view(torch.int64), d_vals.view(torch.int64))


def _oracle_build(mesh):
    ke, rows, cols, first, _, _ = oracle.stiffness_mesh(mesh.coords, mesh.connectivity, mesh.coefficient)
    assert first == -1
    return ke, rows, cols, oracle.triplet_to_csc(rows, cols, ke.reshape(-1), mesh.n_nodes)


@pytest.mark.parametrize("emit", ["0", "1"])
@pytest.mark.parametrize("fused", ["0", "1"])
@pytest.mark.parametrize("rotate", [0.0, 0.3, 1.0])
def test_fused_adjacency_orientations_bitwise(monkeypatch, fused, rotate, emit):
    """The cold build records the node adjacency inside the integration kernel in fixed slots
    (slot = local node).  Elements re-oriented by a rotation of the reference cube put shared nodes
    at colliding local indices; the build detects the lost slots and re-runs the atomic adjacency
    pass.  Either way the results are bitwise the oracle's (also with the fusion switched off)."""
    monkeypatch.setenv("HX_FUSED_ADJACENCY", fused)
    monkeypatch.setenv("HX_FUSED_EMIT", emit)
    rng = np.random.default_rng(77)
    mesh = perturbed_mesh(7, seed=5, distortion=0.15)
    conn = mesh.connectivity.copy()
    turn = rng.random(mesh.n_el) < rotate  # 90 degrees about t: a valid, positively oriented relabelling
    conn[turn] = conn[turn][:, [1, 2, 3, 0, 5, 6, 7, 4]]
    mesh = Mesh(mesh.coords, np.ascontiguousarray(conn), mesh.coefficient)
    ke, rows, cols, (cp, ri, vv) = _oracle_build(mesh)
    b = build_device(D.DeviceMesh.from_host(mesh))
    assert bits_equal(b.ke.cpu().numpy(), ke)
    assert bits_equal(b.rows.cpu().numpy(), rows) and bits_equal(b.cols.cpu().numpy(), cols)
    assert bits_equal(b.csc.col_ptr.cpu().numpy(), cp)
    assert bits_equal(b.csc.row_idx.cpu().numpy(), ri)
    assert bits_equal(b.csc.vals.cpu().numpy(), vv)


def test_fused_adjacency_slot_collision_detected():
    """Two elements holding a node at the same local index: the fixed-slot record loses one entry
    and the status word says so (HX_ST_SLOT_COLLISION) -- the Python layer then re-runs."""
    from paper_1501_04784_b200 import _native as N

    mesh = perturbed_mesh(3, seed=2)
    conn = mesh.connectivity.copy()
    conn[1] = conn[1][[1, 2, 3, 0, 5, 6, 7, 4]]
    mesh = Mesh(mesh.coords, np.ascontiguousarray(conn), mesh.coefficient)
    dm = D.DeviceMesh.from_host(mesh)
    prep = D.new_assembly_prep(dm)
    ke, _, _, fail = D.integrate_mesh(dm, adjacency=prep)
    D.raise_if_failed(fail)
    segs = N.segments([(dm.conn.data_ptr(), ke.data_ptr(), dm.n_el)])
    col_ptr = torch.empty(dm.n_nodes + 1, dtype=torch.int64, device=dm.conn.device)
    cap = 16 * dm.n_nodes
    rbuf = torch.empty(cap, dtype=torch.int64, device=dm.conn.device)
    vbuf = torch.empty(cap, dtype=torch.float64, device=dm.conn.device)
    N.check(N.lib().hx_mesh_csc_build(segs, 1, dm.n_nodes, 0, dm.n_nodes, col_ptr.data_ptr(), rbuf.data_ptr(),
                                      vbuf.data_ptr(), cap, prep.ws.data_ptr(), prep.ws.numel(),
                                      prep.status.data_ptr(), N.CSC_ADJACENCY_READY, None), "build")
    torch.cuda.synchronize()
    assert int(prep.status.item()) & N.ST_SLOT_COLLISION


def test_fused_adjacency_bad_node_id_raises():
    """An out-of-range node id is reported (MeshValidationError, assemble.py:146-149), never
    dereferenced by the fused integration kernel."""
    mesh = perturbed_mesh(3, seed=2)
    conn = mesh.connectivity.copy()
    conn[4, 6] = mesh.n_nodes + 1000
    with pytest.raises(MeshValidationError):
        build_device(D.DeviceMesh.from_host(Mesh(mesh.coords, conn, mesh.coefficient)))


@pytest.mark.parametrize("ranges", [[(0, 100), (100, 250), (250, 343)], [(250, 343), (0, 250)], [(0, 100)]])
def test_fused_adjacency_with_element_groups(ranges):
    """BatchPlan-style element groups (one integration launch each, any order) share one fused
    adjacency record; a partial cover falls back to the assembly's own pass.  Bitwise either way."""
    mesh = permuted_mesh(perturbed_mesh(7, seed=9), seed=3)
    ke, rows, cols, (cp, ri, vv) = _oracle_build(mesh)
    dm = D.DeviceMesh.from_host(mesh)
    if sum(hi - lo for lo, hi in ranges) != mesh.n_el:
        # elements outside the groups keep their (caller-provided) values: zero KE rows
        ke0 = torch.zeros((mesh.n_el, 36), dtype=torch.float64, device=dm.conn.device)
        b = build_device(dm, ranges=ranges, ke=ke0)
        part = ke.copy()
        covered = np.zeros(mesh.n_el, bool)
        for lo, hi in ranges:
            covered[lo:hi] = True
        part[~covered] = 0.0
        cp, ri, vv = oracle.triplet_to_csc(rows, cols, part.reshape(-1), mesh.n_nodes)
        assert bits_equal(b.ke.cpu().numpy(), part)
    else:
        b = build_device(dm, ranges=ranges)
        assert bits_equal(b.ke.cpu().numpy(), ke)
    assert bits_equal(b.csc.col_ptr.cpu().numpy(), cp)
    assert bits_equal(b.csc.row_idx.cpu().numpy(), ri)
    assert bits_equal(b.csc.vals.cpu().numpy(), vv)


def test_compact_host_transfer_matches_device_csc():
    """transfer.CscHostTransfer (int32 rows over PCIe, widened on the host) returns exactly the
    device CSC, with the reference dtypes; pipelined submissions reuse the slots correctly."""
    from paper_1501_04784_b200.assemble import csc_to_host
    from paper_1501_04784_b200.transfer import CscHostTransfer

    meshes = [permuted_mesh(perturbed_mesh(9, seed=s), seed=s + 1) for s in range(3)]
    builds = [build_device(D.DeviceMesh.from_host(m)) for m in meshes]
    ref = [csc_to_host(b.csc) for b in builds]
    xfer = CscHostTransfer(meshes[0].n_nodes, max(b.csc.nnz for b in builds), depth=2, threads=3)

    def check(g, r):
        assert g.col_ptr.dtype == np.int64 and g.row_idx.dtype == np.int64 and g.vals.dtype == np.float64
        assert bits_equal(g.col_ptr, r.col_ptr) and bits_equal(g.row_idx, r.row_idx) and bits_equal(g.vals, r.vals)

    futs = [xfer.submit(b.csc) for b in builds[:2]]  # both slots in flight
    for f, r in zip(futs, ref[:2]):
        check(f.result(), r)
    check(xfer.submit(builds[2].csc).result(), ref[2])  # reuses slot 0 (results valid until then)
    xfer.close()
    # an unaligned (offset) view narrows through the scalar path
    ri = builds[0].csc.row_idx
    assert np.array_equal(D.rows_narrow(ri[1:].contiguous()).cpu().numpy(), ri[1:].cpu().numpy())
    assert np.array_equal(D.rows_narrow(ri[3:]).cpu().numpy(), ri[3:].cpu().numpy())


def test_peek_reads_device_words():
    """hx_peek: int32 words come back sign-extended, int64 words exact, from any stream."""
    dev = torch.device("cuda")
    a = torch.tensor([-7], dtype=torch.int32, device=dev)
    b = torch.tensor([2**40 + 3], dtype=torch.int64, device=dev)
    c = torch.tensor([2**31 - 1], dtype=torch.int32, device=dev)
    assert D.peek(a, b, c) == [-7, 2**40 + 3, 2**31 - 1]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        d = torch.full((1,), -(2**62), dtype=torch.int64, device=dev)
        assert D.peek(d, stream=s) == [-(2**62)]
    with pytest.raises(ValueError):
        D.peek(torch.zeros(2, dtype=torch.int64, device=dev))


def test_compact_host_transfer_empty_block():
    """A CSC block with no entries (a mesh without elements) crosses as col_ptr only."""
    from paper_1501_04784_b200.transfer import CscHostTransfer

    mesh = Mesh(np.zeros((5, 3)), np.zeros((0, 8), np.int32), np.zeros(0))
    b = build_device(D.DeviceMesh.from_host(mesh))
    xfer = CscHostTransfer(mesh.n_nodes, 0, depth=1)
    got = xfer.submit(b.csc).result()
    xfer.close()
    assert got.row_idx.shape == (0,) and got.vals.shape == (0,) and got.row_idx.dtype == np.int64
    assert np.array_equal(got.col_ptr, np.zeros(6, np.int64))


@pytest.mark.parametrize("node", ["big", "negative"])
def test_unfused_paths_bad_node_id_raise_node_index_error(node):
    """Every integration entry point refuses out-of-range node ids without dereferencing them:
    integrate_all (CudaBackend, the reference raises IndexError at staging, integrate.py:146-149),
    build_device with element groups / overlap, run_build and the out-of-core blocks.  The lowest
    such element wins over a degenerate one (the reference fails at staging, before computing)."""
    from paper_1501_04784_b200 import NodeIndexError
    from paper_1501_04784_b200.pipeline import build_out_of_core

    mesh = perturbed_mesh(5, seed=3)
    conn = mesh.connectivity.copy()
    bad_id = mesh.n_nodes + 10**6 if node == "big" else -3
    conn[77, 5] = bad_id
    conn[90, 2] = mesh.n_nodes  # a later bad element
    conn[10] = conn[10][[4, 5, 6, 7, 0, 1, 2, 3]]  # degenerate (flipped), lower id: still loses
    bad = Mesh(mesh.coords, conn, mesh.coefficient)

    def check(exc):
        assert exc.element_id == 77 and exc.node == bad_id
        assert isinstance(exc, IndexError) and isinstance(exc, MeshValidationError)

    with CudaBackend() as be:
        with pytest.raises(NodeIndexError) as ei:
            integrate_all(bad, be, one_group(bad))
        check(ei.value)
        # groups run in plan order (integrate.py:174-179): the first group holds the degenerate
        # element 10 and fails before the group with the bad id is staged, as in the reference
        with pytest.raises(DegenerateElementError) as ei:
            integrate_all(bad, be, plan_batches(required_bytes(bad.n_el), required_bytes(40), bad.n_el))
        assert ei.value.element_id == 10
    dm = D.DeviceMesh.from_host(bad)
    for kw in ({"ranges": [(0, 125)]}, {"overlap": True}, {}):
        with pytest.raises(NodeIndexError) as ei:
            build_device(dm, **kw)
        check(ei.value)
    with pytest.raises(DegenerateElementError) as ei:  # groups report in order, like integrate_all
        build_device(dm, ranges=[(0, 60), (60, 125)])
    assert ei.value.element_id == 10
    with pytest.raises(NodeIndexError) as ei:
        run_build(bad, budget_bytes=10**12)
    check(ei.value)
    with pytest.raises(NodeIndexError) as ei:
        build_out_of_core(bad, 3)
    check(ei.value)


def test_cuda_backend_sees_in_place_changes():
    """integrate_all uploads the mesh per call: changing the caller's arrays in place between
    calls (same objects, same ids) is always seen -- the reference backend is stateless."""
    mesh = perturbed_mesh(4, seed=5)
    coords = mesh.coords.copy()
    coeff = mesh.coefficient.copy()
    m = Mesh(coords, mesh.connectivity, coeff)
    with CudaBackend() as be:
        a = integrate_all(m, be, one_group(m)).values.copy()
        coeff *= 2.0
        coords[:] = coords * 1.5
        b = integrate_all(m, be, one_group(m)).values
    ke, _, _, first, _, _ = oracle.stiffness_mesh(coords, m.connectivity, coeff)
    assert first == -1 and bits_equal(b, ke) and not bits_equal(a, b)


def test_integrate_all_pipelined_groups_many_plans():
    """Two groups in flight (pinned staging, one stream): every plan, both modes, bitwise."""
    mesh = permuted_mesh(perturbed_mesh(9, seed=2), seed=4)
    ke, _, _, _, _, _ = oracle.stiffness_mesh(mesh.coords, mesh.connectivity, mesh.coefficient)
    seen = []
    with CudaBackend() as be:
        for groups in (1, 2, 3, 7, 64):
            plan = plan_batches(groups * required_bytes(mesh.n_el // groups + 1), required_bytes(mesh.n_el // groups + 1),
                                mesh.n_el)
            for mode in ("sequential", "overlapped"):
                seen.clear()
                got = integrate_all(mesh, be, plan, mode=mode,
                                    consumer=lambda r, v: seen.append((r, v.copy())))
                assert bits_equal(got.values, ke)
                assert [r for r, _ in seen] == list(plan.ranges)
                assert all(bits_equal(v, ke[lo:hi]) for (lo, hi), v in seen)


def test_host_transfer_of_planned_rebuilds_not_overwritten():
    """A verified plan reuses its output buffers; the next emit waits for a pending host copy of
    the previous result instead of overwriting it (DeviceCsc.readers)."""
    from paper_1501_04784_b200.transfer import CscHostTransfer

    mesh = perturbed_mesh(12, seed=6)
    dm = D.DeviceMesh.from_host(mesh)
    plan = D.plan_assembly(dm)
    xfer = CscHostTransfer(mesh.n_nodes, plan.nnz, depth=2, threads=2)
    futs, want = [], []
    for k in range(4):
        dm.coeff.mul_(2.0)  # exact: the host restatement scales by 2**(k+1)
        b = build_device(dm, plan=plan)
        futs.append(xfer.submit(b.csc))
        ke, rows, cols, _, _, _ = oracle.stiffness_mesh(mesh.coords, mesh.connectivity,
                                                        mesh.coefficient * 2.0 ** (k + 1))
        want.append(oracle.triplet_to_csc(rows, cols, ke.reshape(-1), mesh.n_nodes)[2])
        if k % 2 == 1:
            for f, w in zip(futs, want):
                assert bits_equal(f.result().vals, w)
            futs, want = [], []
    xfer.close()


@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("assembler", ["direct", "triplet"])
def test_run_build_overlapped_upload_bitwise(monkeypatch, pinned, assembler):
    """run_build's element-range upload (copy stream, one event per range, integration chasing the
    copies) and fetch_csc's chunked int32 transfer + host widening: bitwise the oracle, pinned or
    pageable host arrays, many ranges and many transfer chunks."""
    from paper_1501_04784_b200 import pipeline, transfer
    from paper_1501_04784_b200.hostmem import is_pinned, pinned_mesh

    monkeypatch.setattr(pipeline, "UPLOAD_RANGES_MIN_ELEMENTS", 1)
    monkeypatch.setattr(pipeline, "UPLOAD_RANGES", 7)
    mesh = permuted_mesh(perturbed_mesh(13, seed=8), seed=9)
    if pinned:
        mesh = pinned_mesh(mesh)
        assert is_pinned(mesh.connectivity)
    ke, rows, cols, _, _, _ = oracle.stiffness_mesh(mesh.coords, mesh.connectivity, mesh.coefficient)
    cp, ri, vv = oracle.triplet_to_csc(rows, cols, ke.reshape(-1), mesh.n_nodes)
    orig = transfer.fetch_csc
    monkeypatch.setattr(transfer, "fetch_csc", lambda csc, stream=None: orig(csc, stream=stream, chunk=1000))
    for _ in range(2):
        m, rep = run_build(mesh, budget_bytes=10**12, assembler=assembler)
        assert m.col_ptr.dtype == np.int64 and m.row_idx.dtype == np.int64 and m.vals.dtype == np.float64
        assert bits_equal(m.col_ptr, cp) and bits_equal(m.row_idx, ri) and bits_equal(m.vals, vv)
        assert rep.nnz_csc == len(ri) and rep.time_total_s > 0


@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("blocks", [1, 3, 8])
def test_streamed_run_build_bitwise(monkeypatch, pinned, blocks):
    """run_build's streamed column-block path (stream.py: H2D of range k+1, build of block k and
    D2H of block k-1 overlapped; halo elements recomputed per block) == the oracle, bit for bit."""
    from paper_1501_04784_b200 import pipeline
    from paper_1501_04784_b200.hostmem import pinned_mesh

    monkeypatch.setattr(pipeline, "STREAM_MIN_ELEMENTS", 1)
    monkeypatch.setattr(pipeline, "STREAM_BLOCKS", blocks)
    mesh = perturbed_mesh(14, seed=blocks)
    if pinned:
        mesh = pinned_mesh(mesh)
    ke, rows, cols, _, _, _ = oracle.stiffness_mesh(mesh.coords, mesh.connectivity, mesh.coefficient)
    cp, ri, vv = oracle.triplet_to_csc(rows, cols, ke.reshape(-1), mesh.n_nodes)
    for _ in range(2):
        m, rep = run_build(mesh, budget_bytes=10**12)
        assert bits_equal(m.col_ptr, cp) and bits_equal(m.row_idx, ri) and bits_equal(m.vals, vv)
        assert rep.nnz_csc == len(ri) and rep.time_integration_s > 0
        assert not pipeline.LAST_RUN_STATS.get("sampled_plan_fallback")  # the sampled plan held


def test_streamed_plan_rejects_permuted_and_overflow_falls_back(monkeypatch):
    from paper_1501_04784_b200 import pipeline, stream

    perm = permuted_mesh(perturbed_mesh(10, seed=1), seed=2)
    assert stream.plan(perm, 8) is None
    mesh = perturbed_mesh(20, seed=3)  # 4 blocks: the halo layers stay within MAX_RANGE_OVERLAP
    sp = stream.plan(mesh, 4)
    assert sp is not None and sp.max_block_elements() < mesh.n_el
    assert stream.streamed_build(mesh, sp, capacity=100) is None  # result outgrows the buffers
    monkeypatch.setattr(pipeline, "STREAM_MIN_ELEMENTS", 1)
    ke, rows, cols, _, _, _ = oracle.stiffness_mesh(perm.coords, perm.connectivity, perm.coefficient)
    cp, ri, vv = oracle.triplet_to_csc(rows, cols, ke.reshape(-1), perm.n_nodes)
    m, _ = run_build(perm, budget_bytes=10**12)  # one-shot path
    assert bits_equal(m.col_ptr, cp) and bits_equal(m.row_idx, ri) and bits_equal(m.vals, vv)


@pytest.mark.parametrize("miss", ["node_hi", "e_hi"])
def test_sampled_plan_device_check_falls_back_to_exact_plan(miss):
    """The sampled plan (every 64th element) is checked element by element on the device
    (hx_block_verify); a plan that misses an element's block or coordinates is detected and the
    build reruns with the exact host-scan plan -- bitwise either way."""
    import copy

    from paper_1501_04784_b200 import stream

    mesh = perturbed_mesh(20, seed=5)
    ke, rows, cols, _, _, _ = oracle.stiffness_mesh(mesh.coords, mesh.connectivity, mesh.coefficient)
    cp, ri, vv = oracle.triplet_to_csc(rows, cols, ke.reshape(-1), mesh.n_nodes)
    sp = stream.sampled_plan(mesh, 4)
    assert sp is not None and sp.verify
    stats = {}
    m = stream.streamed_build(mesh, sp, stats=stats)
    assert not stats.get("sampled_plan_fallback")
    assert bits_equal(m.col_ptr, cp) and bits_equal(m.row_idx, ri) and bits_equal(m.vals, vv)
    bad = copy.copy(stream.plan(mesh, 4))
    bad.verify = True
    if miss == "node_hi":  # block 0's halo elements gather coordinates above the uploaded prefix
        bad.node_hi = bad.node_hi.copy()
        bad.node_hi[0] = bad.bounds[1]
    else:  # the last element of block 0's range is uploaded only by block 1
        bad.e_hi = bad.e_hi.copy()
        bad.e_hi[0] -= 1
        assert bad.e_lo[1] <= bad.e_hi[0]
    stats = {}
    m = stream.streamed_build(mesh, bad, stats=stats)
    assert stats.get("sampled_plan_fallback")
    assert bits_equal(m.col_ptr, cp) and bits_equal(m.row_idx, ri) and bits_equal(m.vals, vv)


def test_streamed_errors_lowest_element(monkeypatch):
    from paper_1501_04784_b200 import NodeIndexError, pipeline

    monkeypatch.setattr(pipeline, "STREAM_MIN_ELEMENTS", 1)
    monkeypatch.setattr(pipeline, "STREAM_BLOCKS", 4)
    mesh = perturbed_mesh(8, seed=4)
    conn = mesh.connectivity.copy()
    conn[400] = conn[400][[4, 5, 6, 7, 0, 1, 2, 3]]  # degenerate
    conn[300] = conn[300][[4, 5, 6, 7, 0, 1, 2, 3]]  # lower degenerate id: reported
    with pytest.raises(DegenerateElementError) as ei:
        run_build(Mesh(mesh.coords, conn, mesh.coefficient), budget_bytes=10**12)
    assert ei.value.element_id == 300
    conn[450, 1] = mesh.n_nodes + 3  # a bad node id wins over every degenerate element
    with pytest.raises(NodeIndexError) as ei:
        run_build(Mesh(mesh.coords, conn, mesh.coefficient), budget_bytes=10**12)
    assert ei.value.element_id == 450


def test_out_of_core_budget_takes_streamed_blocks():
    """A device budget below the in-core footprint: the streamed path with blocks sized for the
    budget (locally numbered mesh), bitwise."""
    from paper_1501_04784_b200.pipeline import device_bytes

    mesh = perturbed_mesh(16, seed=7)
    ke, rows, cols, _, _, _ = oracle.stiffness_mesh(mesh.coords, mesh.connectivity, mesh.coefficient)
    cp, ri, vv = oracle.triplet_to_csc(rows, cols, ke.reshape(-1), mesh.n_nodes)
    budget = device_bytes(mesh.n_el, mesh.n_nodes) // 4
    m, rep = run_build(mesh, budget_bytes=10**12, device_budget_bytes=budget)
    assert bits_equal(m.col_ptr, cp) and bits_equal(m.row_idx, ri) and bits_equal(m.vals, vv)


@pytest.mark.parametrize("d", [1, 2, 3, 5])
def test_dof_index_arrays_and_assembly_bitwise(d):
    """dofxn > 1 (assemble.py:65-83): the index kernel vs the reference's
    map_local_to_global (golden, d = 2, 3) and the oracle; the generic triplet assembly of the
    block matrix vs the reference's triplet_to_csc (golden) / the oracle."""
    from pathlib import Path

    g = np.load(Path(__file__).parent / "golden" / "dof.npz")
    n_nodes = int(g["n_nodes"])
    conn = torch.from_numpy(g["conn"]).cuda()
    rows, cols = D.dof_index_arrays(conn, n_nodes, d)
    r_o, c_o = oracle.dof_index_arrays(g["conn"], d)
    assert bits_equal(rows.cpu().numpy(), r_o) and bits_equal(cols.cpu().numpy(), c_o)
    P = (8 * d) * (8 * d + 1) // 2
    if f"d{d}_pairs" in g:
        assert np.array_equal(rows.cpu().numpy(), g[f"d{d}_pairs"][:, 0])
        vals = g[f"d{d}_vals"]
    else:
        vals = np.random.default_rng(d).standard_normal(g["conn"].shape[0] * P)
    csc = D.assemble_dof(conn, torch.from_numpy(vals.reshape(-1, P)).cuda(), n_nodes, d)
    col_ptr, row_idx, v = oracle.triplet_to_csc(r_o, c_o, vals, n_nodes * d)
    assert bits_equal(csc.col_ptr.cpu().numpy(), col_ptr) and bits_equal(csc.row_idx.cpu().numpy(), row_idx)
    assert bits_equal(csc.vals.cpu().numpy(), v)
    if f"d{d}_pairs" in g:
        assert bits_equal(csc.vals.cpu().numpy(), g[f"d{d}_csc_vals"])
    # a larger permuted mesh, index arrays only, over a sub-range
    mesh = make_workload("C1")
    cd = torch.from_numpy(mesh.connectivity).cuda()
    r2, c2 = D.dof_index_arrays(cd, mesh.n_nodes, d, lo=100, hi=2100)
    r_o2, c_o2 = oracle.dof_index_arrays(mesh.connectivity, d, lo=100, hi=2100)
    assert bits_equal(r2.cpu().numpy(), r_o2) and bits_equal(c2.cpu().numpy(), c_o2)


def test_dof_index_arrays_rejects_bad_dofxn():
    conn = torch.zeros((1, 8), dtype=torch.int32, device="cuda")
    with pytest.raises(ValueError):
        D.dof_index_arrays(conn, 1, 0)
    with pytest.raises(ValueError):
        D.dof_index_arrays(conn, 1, 17)
    with pytest.raises(ValueError):
        D.dof_index_arrays(conn, 2**30, 4)


# ---- integration fused with the emit pass (hx_integrate_emit, the default build) --------------------
def _fused_meshes():
    rot = perturbed_mesh(9, seed=21, distortion=0.15)
    conn = rot.connectivity.copy()
    turn = np.random.default_rng(3).random(rot.n_el) < 0.5
    conn[turn] = conn[turn][:, [1, 2, 3, 0, 5, 6, 7, 4]]  # colliding fixed slots -> re-assembly
    return {"structured": perturbed_mesh(23, seed=20), "permuted": permuted_mesh(perturbed_mesh(19, seed=22), seed=23),
            "rotated": Mesh(rot.coords, np.ascontiguousarray(conn), rot.coefficient),
            "tiny": perturbed_mesh(1, seed=24)}


@pytest.mark.parametrize("name", ["structured", "permuted", "rotated", "tiny"])
@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_integrate_emit_equals_separate_kernels(monkeypatch, name, mode):
    """One launch integrating every element and emitting every column tile once its elements are
    done: KE, iK/jK and the CSC are bitwise those of the separate kernels (and the oracle in exact
    mode), for local, permuted and colliding-slot meshes."""
    mesh = _fused_meshes()[name]
    dm = D.DeviceMesh.from_host(mesh)
    monkeypatch.setenv("HX_FUSED_EMIT", "0")
    ref = build_device(dm, mode=mode)
    monkeypatch.setenv("HX_FUSED_EMIT", "1")  # opt-in path
    for _ in range(2):
        b = build_device(dm, mode=mode)
        torch.cuda.synchronize()
        assert bits_equal(b.ke.cpu().numpy(), ref.ke.cpu().numpy())
        assert bits_equal(b.rows.cpu().numpy(), ref.rows.cpu().numpy())
        assert bits_equal(b.cols.cpu().numpy(), ref.cols.cpu().numpy())
        for a, r in ((b.csc.col_ptr, ref.csc.col_ptr), (b.csc.row_idx, ref.csc.row_idx), (b.csc.vals, ref.csc.vals)):
            assert bits_equal(a.cpu().numpy(), r.cpu().numpy())
    if mode == "exact":
        ke, rows, cols, (cp, ri, vv) = _oracle_build(mesh)
        assert bits_equal(b.ke.cpu().numpy(), ke) and bits_equal(b.csc.vals.cpu().numpy(), vv)
        assert bits_equal(b.csc.row_idx.cpu().numpy(), ri) and bits_equal(b.csc.col_ptr.cpu().numpy(), cp)


def test_integrate_emit_low_capacity_and_plan_reuse():
    """A plan whose output buffers are too small: the fused launch writes only the first entries and
    plan_result re-assembles; a verified plan (warm rebuild) runs the fused launch without a sync."""
    mesh = permuted_mesh(perturbed_mesh(12, seed=31), seed=32)
    dm = D.DeviceMesh.from_host(mesh)
    ke_o, _, _, (cp, ri, vv) = _oracle_build(mesh)
    plan = D.mesh_plan_async(dm.conn, dm.n_nodes, capacity=100, fixed=True)
    ke = torch.empty((dm.n_el, 36), dtype=torch.float64, device="cuda")
    fail = D.integrate_emit(dm, plan, ke)
    csc = D.plan_result(plan, ke)
    D.raise_if_failed(fail)
    assert bits_equal(ke.cpu().numpy(), ke_o)
    assert bits_equal(csc.row_idx.cpu().numpy(), ri) and bits_equal(csc.vals.cpu().numpy(), vv)
    vplan = D.plan_assembly(dm)
    os.environ["HX_FUSED_EMIT"] = "1"
    try:
        bs = [build_device(dm, plan=vplan) for _ in range(3)]
    finally:
        os.environ.pop("HX_FUSED_EMIT")
    for b in bs:
        torch.cuda.synchronize()
        D.raise_if_failed(b.fails[0])
        assert bits_equal(b.csc.vals.cpu().numpy(), vv) and bits_equal(b.csc.row_idx.cpu().numpy(), ri)


def test_integrate_emit_errors(monkeypatch):
    """Degenerate elements and bad node ids through the fused launch: the reference's exceptions for
    the lowest failing element, nothing dereferenced out of range."""
    monkeypatch.setenv("HX_FUSED_EMIT", "1")
    mesh = perturbed_mesh(6, seed=41)
    conn = mesh.connectivity.copy()
    conn[100] = conn[100][[4, 5, 6, 7, 0, 1, 2, 3]]
    conn[70] = conn[70][[4, 5, 6, 7, 0, 1, 2, 3]]
    with pytest.raises(DegenerateElementError) as ei:
        build_device(D.DeviceMesh.from_host(Mesh(mesh.coords, np.ascontiguousarray(conn), mesh.coefficient)))
    assert ei.value.element_id == 70
    conn[150, 3] = -5
    from paper_1501_04784_b200 import NodeIndexError

    with pytest.raises(NodeIndexError) as ei:
        build_device(D.DeviceMesh.from_host(Mesh(mesh.coords, np.ascontiguousarray(conn), mesh.coefficient)))
    assert ei.value.element_id == 150


@pytest.mark.parametrize("name", ["structured", "permuted"])
def test_row_codec_device_encoder_matches_format(name):
    """hx_rows_encode produces exactly the format's reference bytes (tests/test_abi_cpu.py), and the
    host decoder restores row_idx / col_ptr of a real build bit for bit, also on a column block."""
    from test_abi_cpu import encode_rows_ref

    from paper_1501_04784_b200.transfer import RowEncoder, decode_rows

    mesh = perturbed_mesh(12, seed=61) if name == "structured" else permuted_mesh(perturbed_mesh(12, seed=61), seed=62)
    b = build_device(D.DeviceMesh.from_host(mesh))
    cp, ri = b.csc.col_ptr.cpu().numpy(), b.csc.row_idx.cpu().numpy()
    enc = RowEncoder()
    for lo, hi in ((0, mesh.n_nodes), (100, 1500)):
        sub_cp = torch.from_numpy(cp[lo:hi + 1] - cp[lo]).cuda()
        sub_ri = torch.from_numpy(ri[cp[lo]:cp[hi]]).cuda()
        counts, lens, data, total = enc.encode(sub_cp, sub_ri, lo)
        nbytes = int(total.item())
        c_ref, l_ref, d_ref = encode_rows_ref(cp[lo:hi + 1] - cp[lo], ri[cp[lo]:cp[hi]], lo)
        assert np.array_equal(counts.cpu().numpy(), c_ref) and np.array_equal(lens.cpu().numpy(), l_ref)
        assert nbytes == d_ref.size and np.array_equal(data[:nbytes].cpu().numpy(), d_ref)
        buf = np.zeros(nbytes + 16, np.uint8)
        buf[:nbytes] = d_ref
        out = np.empty(cp[hi] - cp[lo] + 4, np.int64)
        ends = np.empty(hi - lo, np.int64)
        decode_rows(c_ref, l_ref, buf, nbytes, lo, 0, ends, out, 3)
        assert np.array_equal(out[:cp[hi] - cp[lo]], ri[cp[lo]:cp[hi]]) and np.array_equal(ends, cp[lo + 1:hi + 1] - cp[lo])


@pytest.mark.parametrize("codec", ["0", "1"])
def test_host_transfer_codec_round_trip(monkeypatch, codec):
    """CscHostTransfer with and without the row codec: the host LowerCscMatrix equals the device CSC
    (and the oracle), several submissions through the pipelined slots."""
    from paper_1501_04784_b200.transfer import CscHostTransfer

    monkeypatch.setenv("HX_ROW_CODEC", codec)
    mesh = permuted_mesh(perturbed_mesh(14, seed=71), seed=72)
    dm = D.DeviceMesh.from_host(mesh)
    _, _, _, (cp, ri, vv) = _oracle_build(mesh)
    xfer = CscHostTransfer(mesh.n_nodes, len(ri), depth=2)
    futs = [xfer.submit(build_device(dm).csc) for _ in range(3)]
    for f in futs[-2:]:
        m = f.result()
        assert bits_equal(m.col_ptr, cp) and bits_equal(m.row_idx, ri) and bits_equal(m.vals, vv)
    assert (xfer.bytes_per_transfer(len(ri)) < 8 * (mesh.n_nodes + 1) + 12 * len(ri)) == (codec == "1")
    xfer.close()


_BAND_SCRIPT = r"""
import sys
sys.path[:0] = [{root!r}, {root!r} + '/tests']
import oracle
from common import bits_equal
from paper_1501_04784_b200 import device as D
from paper_1501_04784_b200.pipeline import build_device, run_build
from paper_1501_04784_b200.workloads import permuted_mesh, perturbed_mesh
mesh = perturbed_mesh(24, seed=11)  # band 651 columns: ten 64-column strips
ke, rows, cols, _, _, _ = oracle.stiffness_mesh(mesh.coords, mesh.connectivity, mesh.coefficient)
cp, ri, vv = oracle.triplet_to_csc(rows, cols, ke.reshape(-1), mesh.n_nodes)
csc = build_device(D.DeviceMesh.from_host(mesh)).csc
assert bits_equal(csc.col_ptr.cpu().numpy(), cp) and bits_equal(csc.row_idx.cpu().numpy(), ri)
assert bits_equal(csc.vals.cpu().numpy(), vv)
m, _ = run_build(mesh, budget_bytes=10**12)
assert bits_equal(m.col_ptr, cp) and bits_equal(m.row_idx, ri) and bits_equal(m.vals, vv)
# permuted node ids: element order, first-element keys in the strip order of the element band (~601)
perm = permuted_mesh(mesh, seed=12)
ke, rows, cols, _, _, _ = oracle.stiffness_mesh(perm.coords, perm.connectivity, perm.coefficient)
cp, ri, vv = oracle.triplet_to_csc(rows, cols, ke.reshape(-1), perm.n_nodes)
csc = build_device(D.DeviceMesh.from_host(perm)).csc
assert bits_equal(csc.col_ptr.cpu().numpy(), cp) and bits_equal(csc.row_idx.cpu().numpy(), ri)
assert bits_equal(csc.vals.cpu().numpy(), vv)
print("band ok")
"""


def test_band_strip_order_bitwise():
    """The strip processing orders (band_kernel / band_order_kernel for banded node numberings,
    element_band_kernel's strip keys for element-ordered builds; on by default when the band holds
    four strips) forced onto small meshes with 64-wide strips: the CSC is bitwise the oracle's
    (HX_BAND_STRIP is read once per process, hence the subprocess)."""
    import subprocess
    import sys
    from pathlib import Path

    root = str(Path(__file__).resolve().parent.parent)
    out = subprocess.run([sys.executable, "-c", _BAND_SCRIPT.format(root=root)], capture_output=True, text=True,
                         env={**os.environ, "HX_BAND_STRIP": "64"}, timeout=600)
    assert out.returncode == 0 and "band ok" in out.stdout, out.stderr[-2000:]


@pytest.mark.parametrize("lo,hi", [(0, 1), (5, 8), (0, 63), (1, 66), (0, 9471), (3, 9476), (7, 10000), (0, 13824)])
def test_persistent_integration_ranges_bitwise(lo, hi):
    """The persistent integration kernel's quad scheduling (static first quads, then 16-quad claims
    from the counter) on ranges around the quad, claim and first-wave boundaries (148 SMs x 16
    warps x 4 elements = 9472): KE and iK/jK bitwise the oracle's for exactly the range."""
    mesh = perturbed_mesh(24, seed=9)  # 13824 elements
    ke_ref, rows_ref, cols_ref, _, _, _ = oracle.stiffness_mesh(mesh.coords, mesh.connectivity, mesh.coefficient)
    dm = D.DeviceMesh.from_host(mesh)
    ke, rows, cols, fail = D.integrate_mesh(dm, lo, hi)
    torch.cuda.synchronize()
    D.raise_if_failed(fail)
    assert bits_equal(ke.cpu().numpy(), ke_ref[lo:hi])
    assert np.array_equal(rows.cpu().numpy(), rows_ref[36 * lo:36 * hi])
    assert np.array_equal(cols.cpu().numpy(), cols_ref[36 * lo:36 * hi])


@pytest.mark.parametrize("layout", ["reversed", "anisotropic"])
def test_streamed_run_build_element_layouts(monkeypatch, layout):
    """run_build's streamed path (sampled block plan checked on the device) on locally numbered meshes
    whose element order runs backwards or whose box is far from a cube: bitwise the oracle's, and the
    sampled plan holds (no fallback to the exact scan)."""
    from paper_1501_04784_b200 import pipeline
    from paper_1501_04784_b200.mesh import Mesh

    monkeypatch.setattr(pipeline, "STREAM_MIN_ELEMENTS", 1)
    monkeypatch.setattr(pipeline, "STREAM_BLOCKS", 4)
    if layout == "reversed":
        base = perturbed_mesh(22, seed=31)
        mesh = Mesh(base.coords, np.ascontiguousarray(base.connectivity[::-1]), np.ascontiguousarray(base.coefficient[::-1]))
    else:
        from paper_1501_04784_b200.mesh import StructuredGridSpec, generate_cube_mesh

        g = generate_cube_mesh(StructuredGridSpec(70, 9, 40))
        rng = np.random.default_rng(32)
        mesh = Mesh(g.coords + rng.uniform(-0.1, 0.1, g.coords.shape), g.connectivity,
                    rng.uniform(0.5, 2.0, g.n_el))
    ke, rows, cols, _, _, _ = oracle.stiffness_mesh(mesh.coords, mesh.connectivity, mesh.coefficient)
    cp, ri, vv = oracle.triplet_to_csc(rows, cols, ke.reshape(-1), mesh.n_nodes)
    m, _ = run_build(mesh, budget_bytes=10**12)
    assert bits_equal(m.col_ptr, cp) and bits_equal(m.row_idx, ri) and bits_equal(m.vals, vv)
    assert pipeline.LAST_RUN_STATS.get("blocks") == 4 and not pipeline.LAST_RUN_STATS.get("sampled_plan_fallback")
