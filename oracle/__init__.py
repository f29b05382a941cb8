"""CPU parity oracle for the hexfem hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline leg and
``--impl reference``) may import this package, and only as the checker / CPU baseline.
The product package ``paper_1501_04784_b200`` never imports it.

Parity status: pinned against golden vectors and SHA-256 digests produced by running the
reference package itself in the build container (``tests/golden/make_golden.py``).
"""

from .oracle import (  # noqa: F401
    PACK_COLS,
    PACK_ROWS,
    connectivity_index_arrays,
    dn_table,
    dof_index_arrays,
    export_matrix_market_text,
    pairwise_sum,
    reduceat_model,
    stiffness_batch,
    stiffness_mesh,
    triplet_to_csc,
    triplet_to_csc_columns,
)
