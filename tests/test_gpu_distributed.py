"""Sharded build on one GPU: G virtual ranks (loopback exchange) through the real CUDA kernels
must be bitwise equal to the single-GPU build and to the reference."""

import numpy as np
import pytest
import torch

from common import bits_equal, golden_mesh
from paper_1501_04784_b200 import device as D
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
