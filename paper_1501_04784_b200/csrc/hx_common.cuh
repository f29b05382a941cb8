// hx_common.cuh -- element constants, error plumbing and small device helpers shared by the
// hexfem B200 kernels.  Constants are compile-time so fully unrolled kernels fold them into
// instruction immediates (no constant-bank traffic on the FP64 critical path).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/hexfem_b200.h"

namespace hx {

// Fail-record key of an integration call (atomicMin): a degenerate element e is
// HX_FAIL_DEGENERATE_KEY | e, an element with an out-of-range node id is plain e, so the lowest
// bad-node element wins over every degenerate one (see hx_fail_info).
constexpr unsigned long long HX_FAIL_DEGENERATE_KEY = 1ull << 62;

// ---------------------------------------------------------------------------------------
// Reference element tables (element.py:43-62, 104-135).
//
// _DN_AT_GP[gp][d][a] = 0.125 * r_a * (1 + s_a s)(1 + t_a t) (and the two rotations), at
// gp = 4*ir + 2*is + it with r = (ir ? +g : -g), g = 1/sqrt(3).  Every entry is +-one of
// three magnitudes, M[k] = 0.125 (1+g)^k (1-g)^(2-k) with k = number of "(1+g)" factors;
// the two mixed products are bitwise equal because 0.125*x is exact.  The hex values are
// pinned against the reference's own table by tests/test_abi_cpu.py (hx_dn_table).
// ---------------------------------------------------------------------------------------
__host__ __device__ constexpr double dn_magnitude(int k) {
    return k == 0 ? 0x1.6dd707e2911c6p-6 : (k == 1 ? 0x1.5555555555554p-4 : 0x1.3e77e4d72c439p-2);
}
// NODE_NATURAL_COORDS (element.py:45-56): ccw bottom face (t=-1), then ccw top face.
__host__ __device__ constexpr int nat_r(int a) { return (a == 1 || a == 2 || a == 5 || a == 6) ? 1 : -1; }
__host__ __device__ constexpr int nat_s(int a) { return (a == 2 || a == 3 || a == 6 || a == 7) ? 1 : -1; }
__host__ __device__ constexpr int nat_t(int a) { return a >= 4 ? 1 : -1; }
__host__ __device__ constexpr int gp_r(int gp) { return (gp >> 2) & 1 ? 1 : -1; }
__host__ __device__ constexpr int gp_s(int gp) { return (gp >> 1) & 1 ? 1 : -1; }
__host__ __device__ constexpr int gp_t(int gp) { return gp & 1 ? 1 : -1; }

// sign and magnitude index of _DN_AT_GP[gp][d][a]
__host__ __device__ constexpr int dn_sign(int gp, int d, int a) {
    return d == 0 ? nat_r(a) : (d == 1 ? nat_s(a) : nat_t(a));
}
__host__ __device__ constexpr int dn_mag(int gp, int d, int a) {
    return d == 0 ? (nat_s(a) * gp_s(gp) > 0) + (nat_t(a) * gp_t(gp) > 0)
         : d == 1 ? (nat_r(a) * gp_r(gp) > 0) + (nat_t(a) * gp_t(gp) > 0)
                  : (nat_r(a) * gp_r(gp) > 0) + (nat_s(a) * gp_s(gp) > 0);
}
__host__ __device__ constexpr double dn_value(int gp, int d, int a) {
    return dn_sign(gp, d, a) > 0 ? dn_magnitude(dn_mag(gp, d, a)) : -dn_magnitude(dn_mag(gp, d, a));
}

// Packing (element.py:59-62): p -> (i, j), row-major lower triangle, i >= j.
__host__ __device__ constexpr int pack_i(int p) {
    return p < 1 ? 0 : p < 3 ? 1 : p < 6 ? 2 : p < 10 ? 3 : p < 15 ? 4 : p < 21 ? 5 : p < 28 ? 6 : 7;
}
__host__ __device__ constexpr int pack_j(int p) { return p - pack_i(p) * (pack_i(p) + 1) / 2; }
__host__ __device__ constexpr int pack_index(int i, int j) {  // i >= j
    return i * (i + 1) / 2 + j;
}

// ---------------------------------------------------------------------------------------
// Error plumbing
// ---------------------------------------------------------------------------------------
void set_last_error(const char *fmt, ...);
int cuda_status(cudaError_t err, const char *where);

#define HX_TRY_CUDA(expr)                                                        \
    do {                                                                         \
        cudaError_t _e = (expr);                                                 \
        if (_e != cudaSuccess) return ::hx::cuda_status(_e, #expr);              \
    } while (0)
#define HX_CHECK_LAUNCH(where) HX_TRY_CUDA(cudaGetLastError())

// Adjacency section (deg (ncols) i32, adj (8 ncols) i32) of a mesh-CSC workspace (hx_assemble.cu),
// filled by the integration kernel in the fused build (hx_integrate_mesh_adjacency).
int mesh_ws_adjacency(void *workspace, int64_t workspace_bytes, int64_t ncols, int32_t **deg, int32_t **adj);

// Resolve an integration launch's fail key into the hx_fail_info record (hx_ke.cu).
int integrate_fail_resolve(const double *coords, int64_t n_nodes, const int32_t *conn, hx_fail_info *fail,
                           cudaStream_t s);

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace hx
