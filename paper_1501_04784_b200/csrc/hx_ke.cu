// hx_ke.cu -- numerical integration (the paper's Algorithm 2) for hex8 Poisson elements on
// sm_100a, fused with the iK/jK triplet index generation.
//
// One thread per element.  The 8 node coordinates are gathered straight from the mesh via two
// 16-byte connectivity loads per element (no host-side staging, integrate.py:146-149 is gone),
// the 2x2x2 Gauss quadrature runs in FP64 registers, and the 36 packed lower-triangular values
// are staged in shared memory so the global stores of the element-major (n_el, 36) f64 array and
// of the (36 n_el) i32 row/col arrays are fully coalesced.  Tensor cores are deliberately not
// used: the contractions are 8x3 and FP64.
//
// HX_MODE_EXACT reproduces element.py:255-297 operation for operation with explicitly rounded
// intrinsics (__dmul_rn/__dadd_rn/__ddiv_rn cannot be contracted into FMA), so the output is
// bitwise equal to the reference.  Two bit-preserving restructurings are applied:
//   * dn = +-M_k: (-M)*x == -(M*x) exactly, so products are formed from the 3 magnitudes and
//     the sign becomes add/sub;
//   * B[r][a] = (i_r0 dn0a + i_r1 dn1a) + i_r2 dn2a uses the same identity.
#include <algorithm>
#include <cstdio>

#include "hx_common.cuh"

namespace hx {

constexpr int KE_BLOCK = 128;
constexpr int KE_PAD = 37;  // odd stride (in doubles) -> conflict-free smem staging

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
// acc + dn*x with dn = sign * M_k  (bitwise equal to acc + (dn*x))
__device__ __forceinline__ double acc_signed(double acc, int sign, double prod) {
    return sign > 0 ? dadd(acc, prod) : dsub(acc, prod);
}

// element.py:255-297 for one element, bitwise.  Returns failing gauss point or -1.
__device__ __forceinline__ int ke_exact(const double (&x)[8][3], double coeff, double (&ke)[36],
                                        double &fail_det) {
#pragma unroll
    for (int p = 0; p < 36; ++p) ke[p] = 0.0;
    int fail = -1;
#pragma unroll
    for (int gp = 0; gp < 8; ++gp) {
        // J = dn @ x (element.py:262-269): accumulate from 0.0 over a = 0..7
        double j[3][3];
#pragma unroll
        for (int d = 0; d < 3; ++d)
#pragma unroll
            for (int k = 0; k < 3; ++k) j[d][k] = 0.0;
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int d = 0; d < 3; ++d)
#pragma unroll
                for (int k = 0; k < 3; ++k)
                    j[d][k] = acc_signed(j[d][k], dn_sign(gp, d, a),
                                         dmul(dn_magnitude(dn_mag(gp, d, a)), x[a][k]));
        // cofactors of the first row and det (element.py:271-275)
        const double c00 = dsub(dmul(j[1][1], j[2][2]), dmul(j[1][2], j[2][1]));
        const double c01 = dsub(dmul(j[1][2], j[2][0]), dmul(j[1][0], j[2][2]));
        const double c02 = dsub(dmul(j[1][0], j[2][1]), dmul(j[1][1], j[2][0]));
        const double det = dadd(dadd(dmul(j[0][0], c00), dmul(j[0][1], c01)), dmul(j[0][2], c02));
        if (!(det > 0.0)) {  // element.py:276-279 (also catches NaN)
            fail = gp;
            fail_det = det;
            break;
        }
        // adjugate / det (element.py:281-284), true IEEE division
        double inv[3][3];
        inv[0][0] = __ddiv_rn(c00, det);
        inv[0][1] = __ddiv_rn(dsub(dmul(j[0][2], j[2][1]), dmul(j[0][1], j[2][2])), det);
        inv[0][2] = __ddiv_rn(dsub(dmul(j[0][1], j[1][2]), dmul(j[0][2], j[1][1])), det);
        inv[1][0] = __ddiv_rn(c01, det);
        inv[1][1] = __ddiv_rn(dsub(dmul(j[0][0], j[2][2]), dmul(j[0][2], j[2][0])), det);
        inv[1][2] = __ddiv_rn(dsub(dmul(j[0][2], j[1][0]), dmul(j[0][0], j[1][2])), det);
        inv[2][0] = __ddiv_rn(c02, det);
        inv[2][1] = __ddiv_rn(dsub(dmul(j[0][1], j[2][0]), dmul(j[0][0], j[2][1])), det);
        inv[2][2] = __ddiv_rn(dsub(dmul(j[0][0], j[1][1]), dmul(j[0][1], j[1][0])), det);
        // B = J^-1 dn (element.py:286-290): (i_r0*dn0a + i_r1*dn1a) + i_r2*dn2a
        double B[3][8];
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            double q[3][3];  // q[d][m] = inv[r][d] * M_m
#pragma unroll
            for (int d = 0; d < 3; ++d)
#pragma unroll
                for (int m = 0; m < 3; ++m) q[d][m] = dmul(inv[r][d], dn_magnitude(m));
#pragma unroll
            for (int a = 0; a < 8; ++a) {
                const double t0 = dn_sign(gp, 0, a) > 0 ? q[0][dn_mag(gp, 0, a)] : -q[0][dn_mag(gp, 0, a)];
                const double t01 = acc_signed(t0, dn_sign(gp, 1, a), q[1][dn_mag(gp, 1, a)]);
                B[r][a] = acc_signed(t01, dn_sign(gp, 2, a), q[2][dn_mag(gp, 2, a)]);
            }
        }
        // ke[p] += (c*det) * ((B0i B0j + B1i B1j) + B2i B2j)  (element.py:293-297)
        const double scale = dmul(coeff, det);
#pragma unroll
        for (int p = 0; p < 36; ++p) {
            const int i = pack_i(p), jj = pack_j(p);
            const double s = dadd(dadd(dmul(B[0][i], B[0][jj]), dmul(B[1][i], B[1][jj])),
                                  dmul(B[2][i], B[2][jj]));
            ke[p] = dadd(ke[p], dmul(scale, s));
        }
    }
    return fail;
}

// Recompute one element to report (gauss point, det) of a failure -- single thread.
__device__ void fail_detail(const double (&x)[8][3], double coeff, int64_t element, hx_fail_info *fail) {
    double ke[36];
    double det = 0.0;
    const int gp = ke_exact(x, coeff, ke, det);
    fail->element = element;
    fail->gauss_point = gp;
    fail->det = det;
}

__device__ __forceinline__ void load_node(const double *__restrict__ coords, int32_t node, double (&xa)[3]) {
    const double *p = coords + 3 * (int64_t)node;
    xa[0] = __ldg(p);
    xa[1] = __ldg(p + 1);
    xa[2] = __ldg(p + 2);
}

__device__ __forceinline__ void load_conn(const int32_t *__restrict__ conn, int64_t e, int32_t (&g)[8]) {
    const int4 *c4 = reinterpret_cast<const int4 *>(conn) + 2 * e;
    const int4 lo = __ldg(c4), hi = __ldg(c4 + 1);
    g[0] = lo.x; g[1] = lo.y; g[2] = lo.z; g[3] = lo.w;
    g[4] = hi.x; g[5] = hi.y; g[6] = hi.z; g[7] = hi.w;
}

// Packed pair tables in shared memory for the coalesced copy-out (dynamic p per lane).
__device__ __forceinline__ void init_pack_smem(uint8_t *pi, uint8_t *pj) {
    if (threadIdx.x < 36) {
        const int p = threadIdx.x;
        int i = 0;
        while ((i + 1) * (i + 2) / 2 <= p) ++i;
        pi[p] = (uint8_t)i;
        pj[p] = (uint8_t)(p - i * (i + 1) / 2);
    }
}

// Mesh kernel: elements [lo, lo+n) of the mesh; outputs indexed from 0 (= element lo).
template <int MODE>
__global__ void __launch_bounds__(KE_BLOCK)
integrate_mesh_kernel(const double *__restrict__ coords, const int32_t *__restrict__ conn,
                      const double *__restrict__ coeff, int64_t lo, int64_t n,
                      double *__restrict__ ke_out, int32_t *__restrict__ rows_out,
                      int32_t *__restrict__ cols_out, unsigned long long *__restrict__ fail_min) {
    __shared__ double s_ke[KE_BLOCK * KE_PAD];
    __shared__ int32_t s_conn[KE_BLOCK * 8];
    __shared__ uint8_t s_pi[36], s_pj[36];
    init_pack_smem(s_pi, s_pj);

    const int64_t first = (int64_t)blockIdx.x * KE_BLOCK;
    const int t = threadIdx.x;
    const int64_t k = first + t;
    if (k < n) {
        const int64_t e = lo + k;
        int32_t g[8];
        load_conn(conn, e, g);
#pragma unroll
        for (int a = 0; a < 8; ++a) s_conn[t * 8 + a] = g[a];
        double x[8][3];
#pragma unroll
        for (int a = 0; a < 8; ++a) load_node(coords, g[a], x[a]);
        double ke[36];
        double det = 0.0;
        const int gp = ke_exact(x, __ldg(coeff + e), ke, det);
        if (gp >= 0) atomicMin(fail_min, (unsigned long long)e);
#pragma unroll
        for (int p = 0; p < 36; ++p) s_ke[t * KE_PAD + p] = ke[p];
    }
    __syncthreads();
    const int nvalid = (int)(n - first < KE_BLOCK ? n - first : KE_BLOCK);
    const int total = nvalid * 36;
    double *kdst = ke_out + first * 36;
    for (int w = t; w < total; w += KE_BLOCK) {
        const int el = w / 36, p = w - el * 36;
        kdst[w] = s_ke[el * KE_PAD + p];
    }
    if (rows_out != nullptr) {
        int32_t *rdst = rows_out + first * 36;
        int32_t *cdst = cols_out + first * 36;
        for (int w = t; w < total; w += KE_BLOCK) {
            const int el = w / 36, p = w - el * 36;
            const int32_t gi = s_conn[el * 8 + s_pi[p]], gj = s_conn[el * 8 + s_pj[p]];
            rdst[w] = max(gi, gj);
            cdst[w] = min(gi, gj);
        }
    }
}

// Batch kernel: pre-gathered coords (n, 8, 3) (stiffness_batch, element.py:213-245).
template <int MODE>
__global__ void __launch_bounds__(KE_BLOCK)
stiffness_batch_kernel(const double *__restrict__ coords, const double *__restrict__ coeff, int64_t n,
                       double *__restrict__ out, unsigned long long *__restrict__ fail_min) {
    __shared__ double s_ke[KE_BLOCK * KE_PAD];
    const int64_t first = (int64_t)blockIdx.x * KE_BLOCK;
    const int t = threadIdx.x;
    const int64_t e = first + t;
    if (e < n) {
        double x[8][3];
        const double *src = coords + 24 * e;
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int d = 0; d < 3; ++d) x[a][d] = __ldg(src + 3 * a + d);
        double ke[36];
        double det = 0.0;
        const int gp = ke_exact(x, __ldg(coeff + e), ke, det);
        if (gp >= 0) atomicMin(fail_min, (unsigned long long)e);
#pragma unroll
        for (int p = 0; p < 36; ++p) s_ke[t * KE_PAD + p] = ke[p];
    }
    __syncthreads();
    const int nvalid = (int)(n - first < KE_BLOCK ? n - first : KE_BLOCK);
    const int total = nvalid * 36;
    double *kdst = out + first * 36;
    for (int w = t; w < total; w += KE_BLOCK) {
        const int el = w / 36, p = w - el * 36;
        kdst[w] = s_ke[el * KE_PAD + p];
    }
}

// Resolve the lowest failing element into the hx_fail_info record (element.py:237-244).
__global__ void fail_resolve_mesh_kernel(const double *__restrict__ coords, const int32_t *__restrict__ conn,
                                         const double *__restrict__ coeff, hx_fail_info *fail) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const unsigned long long key = *reinterpret_cast<unsigned long long *>(fail);
    if (key == ~0ull) {
        fail->element = -1;
        fail->gauss_point = -1;
        fail->det = 0.0;
        return;
    }
    const int64_t e = (int64_t)key;
    int32_t g[8];
    load_conn(conn, e, g);
    double x[8][3];
    for (int a = 0; a < 8; ++a) load_node(coords, g[a], x[a]);
    fail_detail(x, coeff[e], e, fail);
}

__global__ void fail_resolve_batch_kernel(const double *__restrict__ coords, const double *__restrict__ coeff,
                                          hx_fail_info *fail) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const unsigned long long key = *reinterpret_cast<unsigned long long *>(fail);
    if (key == ~0ull) {
        fail->element = -1;
        fail->gauss_point = -1;
        fail->det = 0.0;
        return;
    }
    const int64_t e = (int64_t)key;
    double x[8][3];
    for (int a = 0; a < 8; ++a)
        for (int d = 0; d < 3; ++d) x[a][d] = coords[24 * e + 3 * a + d];
    fail_detail(x, coeff[e], e, fail);
}

// connectivity_index_arrays alone (assemble.py:86-93), 4 outputs per thread.
__global__ void index_kernel(const int32_t *__restrict__ conn, int64_t lo, int64_t n,
                             int32_t *__restrict__ rows, int32_t *__restrict__ cols) {
    __shared__ uint8_t s_pi[36], s_pj[36];
    init_pack_smem(s_pi, s_pj);
    __syncthreads();
    const int64_t total = 36 * n;
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < total;
         w += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = w / 36;
        const int p = (int)(w - k * 36);
        const int32_t *c = conn + 8 * (lo + k);
        const int32_t gi = __ldg(c + s_pi[p]), gj = __ldg(c + s_pj[p]);
        rows[w] = max(gi, gj);
        cols[w] = min(gi, gj);
    }
}

}  // namespace hx

using namespace hx;

extern "C" int hx_integrate_mesh(const double *coords, int64_t n_nodes, const int32_t *conn,
                                 const double *coeff, int64_t lo, int64_t hi, double *ke,
                                 int32_t *rows, int32_t *cols, int32_t mode, hx_fail_info *fail,
                                 void *stream) {
    (void)n_nodes;
    if (lo < 0 || hi < lo || ke == nullptr || fail == nullptr || (rows == nullptr) != (cols == nullptr)) {
        set_last_error("hx_integrate_mesh: bad arguments (lo=%lld hi=%lld)", (long long)lo, (long long)hi);
        return HX_ERR_VALUE;
    }
    if (mode != HX_MODE_EXACT && mode != HX_MODE_FAST) {
        set_last_error("hx_integrate_mesh: unknown mode %d", mode);
        return HX_ERR_CONFIG;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t n = hi - lo;
    HX_TRY_CUDA(cudaMemsetAsync(fail, 0xff, sizeof(unsigned long long), s));
    if (n > 0) {
        const int64_t blocks = ceil_div(n, KE_BLOCK);
        integrate_mesh_kernel<HX_MODE_EXACT><<<(unsigned)blocks, KE_BLOCK, 0, s>>>(
            coords, conn, coeff, lo, n, ke, rows, cols, reinterpret_cast<unsigned long long *>(fail));
        HX_CHECK_LAUNCH("integrate_mesh_kernel");
    }
    fail_resolve_mesh_kernel<<<1, 1, 0, s>>>(coords, conn, coeff, fail);
    HX_CHECK_LAUNCH("fail_resolve_mesh_kernel");
    return HX_OK;
}

extern "C" int hx_stiffness_batch(const double *coords, const double *coeff, int64_t n, double *out,
                                  int32_t mode, hx_fail_info *fail, void *stream) {
    if (n < 0 || out == nullptr || fail == nullptr) {
        set_last_error("hx_stiffness_batch: bad arguments (n=%lld)", (long long)n);
        return HX_ERR_VALUE;
    }
    if (mode != HX_MODE_EXACT && mode != HX_MODE_FAST) {
        set_last_error("hx_stiffness_batch: unknown mode %d", mode);
        return HX_ERR_CONFIG;
    }
    cudaStream_t s = (cudaStream_t)stream;
    HX_TRY_CUDA(cudaMemsetAsync(fail, 0xff, sizeof(unsigned long long), s));
    if (n > 0) {
        const int64_t blocks = ceil_div(n, KE_BLOCK);
        stiffness_batch_kernel<HX_MODE_EXACT><<<(unsigned)blocks, KE_BLOCK, 0, s>>>(
            coords, coeff, n, out, reinterpret_cast<unsigned long long *>(fail));
        HX_CHECK_LAUNCH("stiffness_batch_kernel");
    }
    fail_resolve_batch_kernel<<<1, 1, 0, s>>>(coords, coeff, fail);
    HX_CHECK_LAUNCH("fail_resolve_batch_kernel");
    return HX_OK;
}

extern "C" int hx_connectivity_index_arrays(const int32_t *conn, int64_t lo, int64_t hi, int32_t *rows,
                                            int32_t *cols, void *stream) {
    if (lo < 0 || hi < lo || rows == nullptr || cols == nullptr) {
        set_last_error("hx_connectivity_index_arrays: bad arguments");
        return HX_ERR_VALUE;
    }
    const int64_t n = hi - lo;
    if (n == 0) return HX_OK;
    const int threads = 256;
    const int64_t blocks = std::min<int64_t>(ceil_div(36 * n, threads), 148 * 16);
    index_kernel<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(conn, lo, n, rows, cols);
    HX_CHECK_LAUNCH("index_kernel");
    return HX_OK;
}
