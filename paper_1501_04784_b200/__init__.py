"""B200-native global finite-element matrix construction for 3D Poisson on hex8 meshes
(arXiv 1501.04784), a drop-in for the reference package ``hexfem``'s hot path:

    mesh + coefficient -> packed lower KE (36/element) -> iK/jK -> lower-triangular CSC K

All compute runs in hand-written sm_100a CUDA kernels behind the C ABI of libhexfem_b200.so
(include/hexfem_b200.h); there is no CPU fallback.
"""

from .assemble import (
    DirectAssembler,
    LowerCscMatrix,
    TripletMatrix,
    assemble_direct,
    assemble_dof,
    dof_index_arrays,
    build_triplet,
    connectivity_index_arrays,
    map_local_to_global,
    nnz_compression,
    triplet_to_csc,
)
from .element import (
    NODE_NATURAL_COORDS,
    PACK_COLS,
    PACK_ROWS,
    ElementGeometry,
    PackedLowerStiffness,
    element_geometry,
    local_stiffness,
    pack_lower,
    set_worker_threads,
    stiffness_batch,
    unpack_lower,
)
from .errors import (
    ConfigurationError,
    DegenerateElementError,
    HexFemError,
    MeshFormatError,
    MeshValidationError,
    NativeLibraryError,
    NodeIndexError,
    StagingError,
)
from .integrate import (
    BYTES_PER_ELEMENT,
    BatchPlan,
    ComputeBackend,
    CudaBackend,
    LocalValuesBatch,
    integrate_all,
    plan_batches,
    required_bytes,
)
from .mesh import Mesh, StructuredGridSpec, generate_cube_mesh, validate_mesh
from .sparseio import export_matrix_market, import_matrix_market
from .pipeline import (
    BuildReport,
    build_device,
    csc_memory,
    format_mb,
    format_percent,
    memory_saving,
    run_build,
    triplet_memory,
)
from .transfer import CscHostTransfer

__version__ = "0.1.0"
