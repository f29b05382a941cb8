"""Pin the CPU oracle against the reference's own outputs (golden vectors + digests)."""

from pathlib import Path

import numpy as np
import pytest

import oracle
from common import SMALL_MESHES, bits_equal, sha
from paper_1501_04784_b200.workloads import make_workload


def test_dn_table_is_the_reference_table(golden):
    assert bits_equal(oracle.dn_table(), golden["dn_table"])


def test_pack_tables(golden):
    assert np.array_equal(oracle.PACK_ROWS, golden["pack_rows"])
    assert np.array_equal(oracle.PACK_COLS, golden["pack_cols"])


@pytest.mark.parametrize("threads", [1, 4])
def test_element_batch_bitwise(golden, threads):
    ke, first, _, _ = oracle.stiffness_batch(golden["batch_coords"], golden["batch_coeff"], threads=threads)
    assert first == -1
    assert bits_equal(ke, golden["batch_ke"])


@pytest.mark.parametrize("name", SMALL_MESHES)
def test_small_mesh_pipeline_bitwise(golden, name):
    ke, rows, cols, first, _, _ = oracle.stiffness_mesh(golden[f"{name}_coords"], golden[f"{name}_conn"],
                                                        golden[f"{name}_coeff"])
    assert first == -1
    assert bits_equal(ke, golden[f"{name}_ke"])
    assert bits_equal(rows, golden[f"{name}_rows"])
    assert bits_equal(cols, golden[f"{name}_cols"])
    r2, c2 = oracle.connectivity_index_arrays(golden[f"{name}_conn"])
    assert bits_equal(r2, rows) and bits_equal(c2, cols)
    col_ptr, row_idx, vals = oracle.triplet_to_csc(rows, cols, ke.reshape(-1), golden[f"{name}_coords"].shape[0])
    assert bits_equal(col_ptr, golden[f"{name}_col_ptr"])
    assert bits_equal(row_idx, golden[f"{name}_row_idx"])
    assert bits_equal(vals, golden[f"{name}_vals"])


def test_degenerate_first_element_wins(golden):
    coords = golden["degen_coords"][golden["degen_conn"]]
    _, first, gp, det = oracle.stiffness_batch(coords, np.ones(coords.shape[0]), threads=4)
    exp_el, exp_gp = golden["degen_expect"]
    assert first == exp_el
    assert gp[first] == exp_gp
    assert det[first] == golden["degen_det"][0]


def test_generic_triplets_with_long_runs(golden):
    col_ptr, row_idx, vals = oracle.triplet_to_csc(golden["trip_rows"], golden["trip_cols"], golden["trip_vals"],
                                                   int(golden["trip_dim"][0]))
    assert bits_equal(col_ptr, golden["trip_col_ptr"])
    assert bits_equal(row_idx, golden["trip_row_idx"])
    assert bits_equal(vals, golden["trip_out"])


def test_reduceat_rule_model_matches_numpy():
    """The rule the GPU numeric phases implement: out = v0 + pairwise(v[1:])."""
    rng = np.random.default_rng(5)
    for length in list(range(1, 40)) + [127, 128, 129, 130, 200, 257, 300, 1000]:
        for _ in range(5):
            v = rng.standard_normal(length) * np.exp(rng.uniform(-30, 30, size=length))
            got = oracle.reduceat_model(v)
            ref = np.add.reduceat(v, [0])[0]
            assert np.float64(got).tobytes() == np.float64(ref).tobytes(), length


def test_oracle_triplet_validation():
    with pytest.raises(ValueError):
        oracle.triplet_to_csc(np.array([5], np.int32), np.array([0], np.int32), np.array([1.0]), 4)
    with pytest.raises(ValueError):
        oracle.triplet_to_csc(np.array([0], np.int32), np.array([2], np.int32), np.array([1.0]), 4)


@pytest.mark.parametrize("config", ["C1", "C2"])
def test_oracle_matches_reference_digests(digests, config):
    d = digests["configs"][config]
    mesh = make_workload(config)
    ke, rows, cols, first, _, _ = oracle.stiffness_mesh(mesh.coords, mesh.connectivity, mesh.coefficient)
    assert first == -1
    assert sha(ke) == d["ke"]
    assert sha(rows) == d["rows"] and sha(cols) == d["cols"]
    col_ptr, row_idx, vals = oracle.triplet_to_csc(rows, cols, ke.reshape(-1), mesh.n_nodes)
    assert len(row_idx) == d["nnz"]
    assert sha(col_ptr) == d["col_ptr"] and sha(row_idx) == d["row_idx"] and sha(vals) == d["vals"]


def test_column_window_restatement_equals_full_assembly(golden):
    """oracle.triplet_to_csc_columns (the reference algorithm on a column window, used by the C4
    every-column GPU check) == the window of the full triplet_to_csc, on the reference's outputs."""
    for name in ("perm5", "m345"):
        conn, ke = golden[f"{name}_conn"], golden[f"{name}_ke"]
        cp, ri, vv = golden[f"{name}_col_ptr"], golden[f"{name}_row_idx"], golden[f"{name}_vals"]
        n = cp.shape[0] - 1
        for c0, c1 in ((0, n // 3), (n // 3, n // 2), (n // 2, n)):
            touch = np.flatnonzero(((conn >= c0) & (conn < c1)).any(axis=1))
            c = conn[touch]
            r = np.maximum(c[:, oracle.PACK_ROWS], c[:, oracle.PACK_COLS]).reshape(-1)
            k = np.minimum(c[:, oracle.PACK_ROWS], c[:, oracle.PACK_COLS]).reshape(-1)
            keep = (k >= c0) & (k < c1)
            a, b, v = oracle.triplet_to_csc_columns(r[keep], k[keep], ke[touch].reshape(-1)[keep], c0, c1)
            assert np.array_equal(a, cp[c0:c1 + 1] - cp[c0])
            assert np.array_equal(b, ri[cp[c0]:cp[c1]])
            assert v.tobytes() == vv[cp[c0]:cp[c1]].tobytes()


@pytest.mark.parametrize("d", [2, 3])
def test_dof_index_arrays_match_reference_mapping(d):
    """oracle.dof_index_arrays == the reference's map_local_to_global, element by element
    (tests/golden/dof.npz, made by tests/golden/make_golden_dof.py), and its triplet_to_csc."""
    g = np.load(Path(__file__).parent / "golden" / "dof.npz")
    rows, cols = oracle.dof_index_arrays(g["conn"], d)
    assert np.array_equal(rows, g[f"d{d}_pairs"][:, 0]) and np.array_equal(cols, g[f"d{d}_pairs"][:, 1])
    col_ptr, row_idx, vals = oracle.triplet_to_csc(rows, cols, g[f"d{d}_vals"], int(g["n_nodes"]) * d)
    assert bits_equal(col_ptr, g[f"d{d}_col_ptr"]) and bits_equal(row_idx, g[f"d{d}_row_idx"])
    assert bits_equal(vals, g[f"d{d}_csc_vals"])


def test_dof_index_arrays_dofxn1_is_connectivity_index_arrays():
    conn = make_workload("C1").connectivity[:500]
    r1, c1 = oracle.dof_index_arrays(conn, 1)
    r0, c0 = oracle.connectivity_index_arrays(conn)
    assert bits_equal(r1, r0) and bits_equal(c1, c0)
