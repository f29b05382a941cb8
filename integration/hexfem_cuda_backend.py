"""hexfem/cuda_backend.py -- the reference-side binding a `hexfem` maintainer adds:
a `ComputeBackend` plugin (integrate.py:84-112) over the C ABI of libhexfem_b200.so, via ctypes.
torch is used only for device memory and the current stream.

Imports `hexfem` when it is installed; otherwise the identical interface of
`paper_1501_04784_b200` (so the binding itself is exercised by this repo's GPU tests on a box that
has no `hexfem`).  The library path comes from HEXFEM_B200_LIB, else the in-tree build.
"""
import ctypes
import os
from pathlib import Path

import numpy as np
import torch

try:  # the reference package
    from hexfem.errors import DegenerateElementError
    from hexfem.integrate import ComputeBackend
except ImportError:  # same names, same contract
    from paper_1501_04784_b200.errors import DegenerateElementError
    from paper_1501_04784_b200.integrate import ComputeBackend

_DEFAULT = Path(__file__).resolve().parent.parent / "paper_1501_04784_b200" / "_lib" / "libhexfem_b200.so"
_lib = ctypes.CDLL(os.environ.get("HEXFEM_B200_LIB", str(_DEFAULT)))
_P, _I32, _I64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
_lib.hx_stiffness_batch.argtypes = [_P, _P, _I64, _P, _I32, _P, _P]
_lib.hx_stiffness_batch.restype = ctypes.c_int
_lib.hx_last_error.restype = ctypes.c_char_p
HX_MODE_EXACT = 0


class CudaBackend(ComputeBackend):
    """integrate.py:84-112 contract: run(coords (n,8,3), coeff (n,), element_offset, out) -> (n,36)."""

    def __init__(self, workers=1, capacity_bytes=None):
        self.workers, self.capacity_bytes = workers, capacity_bytes

    def run(self, coords, coeff, element_offset=0, out=None):
        n = coords.shape[0]
        d_coords = torch.from_numpy(np.ascontiguousarray(coords, np.float64)).cuda()
        d_coeff = torch.from_numpy(np.ascontiguousarray(coeff, np.float64)).cuda()
        d_out = torch.empty((n, 36), dtype=torch.float64, device="cuda")
        d_fail = torch.empty(3, dtype=torch.int64, device="cuda")  # hx_fail_info, 24 bytes
        stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        rc = _lib.hx_stiffness_batch(d_coords.data_ptr(), d_coeff.data_ptr(), n, d_out.data_ptr(),
                                     HX_MODE_EXACT, d_fail.data_ptr(), stream)
        if rc != 0:
            raise RuntimeError(_lib.hx_last_error().decode())
        fail = d_fail.cpu().numpy()
        if fail[0] >= 0:
            raise DegenerateElementError(element_id=element_offset + int(fail[0]),
                                         gauss_point=int(np.int32(fail[1] & 0xFFFFFFFF)),
                                         det=float(fail[2:3].view(np.float64)[0]))
        if out is None:
            out = np.empty((n, 36))
        out[...] = d_out.cpu().numpy()
        return out

    def close(self):
        pass
