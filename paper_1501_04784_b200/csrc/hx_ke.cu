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

// IEEE round-to-nearest a/b from y = RN(1/b): q0 = RN(a*y) is within 2 ulp of a/b; one
// correction q1 = RN(q0 + (a - b q0) y) lands within 1 ulp (the residual is exact via FMA and
// the correction error is ~2^-52 ulp); Markstein's theorem (y = RN(1/b), q within 1 ulp, exact
// residual) then makes q2 = RN(q1 + (a - b q1) y) the correctly rounded quotient, i.e. bitwise
// __ddiv_rn(a, b).  Valid while nothing over/underflows: the caller guards exponents and zero.
__device__ __forceinline__ double div_markstein(double a, double b, double y) {
    const double q0 = __dmul_rn(a, y);
    const double r0 = __fma_rn(-q0, b, a);
    const double q1 = __fma_rn(r0, y, q0);
    const double r1 = __fma_rn(-q1, b, a);
    const double q2 = __fma_rn(r1, y, q1);
    return a == 0.0 ? q0 : q2;  // signed zero: 0*y keeps the sign of a (b > 0)
}

// |x| in [2^-800, 2^800] (or x == 0): Markstein path safe for these operands.
__device__ __forceinline__ bool div_safe(double x) {
    const int e = (__double2hiint(x) >> 20) & 0x7ff;
    return (e >= 1023 - 800 && e <= 1023 + 800) || x == 0.0;
}

// element.py:255-297 for one element, bitwise.  Coordinates are read from shared memory with
// volatile loads (xs[(3a+k)*stride]) once per Gauss point: products M_k*x are recomputed per
// point instead of being kept live across all eight (register pressure -> occupancy).
// Returns the failing gauss point or -1.
__device__ __forceinline__ int ke_exact(const volatile double *xs, int stride, double coeff, double (&ke)[36],
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
        for (int a = 0; a < 8; ++a) {
            double xa[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) xa[k] = xs[(3 * a + k) * stride];
#pragma unroll
            for (int d = 0; d < 3; ++d)
#pragma unroll
                for (int k = 0; k < 3; ++k)
                    j[d][k] = acc_signed(j[d][k], dn_sign(gp, d, a), dmul(dn_magnitude(dn_mag(gp, d, a)), xa[k]));
        }
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
        // adjugate / det (element.py:281-284): IEEE-exact quotients
        double num[9];
        num[0] = c00;
        num[1] = dsub(dmul(j[0][2], j[2][1]), dmul(j[0][1], j[2][2]));
        num[2] = dsub(dmul(j[0][1], j[1][2]), dmul(j[0][2], j[1][1]));
        num[3] = c01;
        num[4] = dsub(dmul(j[0][0], j[2][2]), dmul(j[0][2], j[2][0]));
        num[5] = dsub(dmul(j[0][2], j[1][0]), dmul(j[0][0], j[1][2]));
        num[6] = c02;
        num[7] = dsub(dmul(j[0][1], j[2][0]), dmul(j[0][0], j[2][1]));
        num[8] = dsub(dmul(j[0][0], j[1][1]), dmul(j[0][1], j[1][0]));
        bool safe = div_safe(det) && det != 0.0;
#pragma unroll
        for (int i = 0; i < 9; ++i) safe &= div_safe(num[i]);
        double inv[3][3];
        if (safe) {
            const double y = __drcp_rn(det);
#pragma unroll
            for (int i = 0; i < 9; ++i) inv[i / 3][i % 3] = div_markstein(num[i], det, y);
        } else {
#pragma unroll
            for (int i = 0; i < 9; ++i) inv[i / 3][i % 3] = __ddiv_rn(num[i], det);
        }
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
    const int gp = ke_exact(&x[0][0], 1, coeff, ke, det);
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
    __shared__ double s_ke[KE_BLOCK * KE_PAD];  // also holds the staged coordinates (24 x KE_BLOCK)
    __shared__ int32_t s_conn[KE_BLOCK * 8];
    __shared__ uint8_t s_pi[36], s_pj[36];
    init_pack_smem(s_pi, s_pj);

    const int64_t first = (int64_t)blockIdx.x * KE_BLOCK;
    const int t = threadIdx.x;
    const int64_t k = first + t;
    double ke[36];
    if (k < n) {
        const int64_t e = lo + k;
        int32_t g[8];
        load_conn(conn, e, g);
#pragma unroll
        for (int a = 0; a < 8; ++a) s_conn[t * 8 + a] = g[a];
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            double xa[3];
            load_node(coords, g[a], xa);
#pragma unroll
            for (int d = 0; d < 3; ++d) s_ke[(3 * a + d) * KE_BLOCK + t] = xa[d];
        }
        double det = 0.0;
        const int gp = ke_exact(s_ke + t, KE_BLOCK, __ldg(coeff + e), ke, det);
        if (gp >= 0) atomicMin(fail_min, (unsigned long long)e);
    }
    __syncthreads();  // every thread is done with its staged coordinates
    if (k < n) {
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
    double ke[36];
    if (e < n) {
        const double *src = coords + 24 * e;
#pragma unroll
        for (int i = 0; i < 24; ++i) s_ke[i * KE_BLOCK + t] = __ldg(src + i);
        double det = 0.0;
        const int gp = ke_exact(s_ke + t, KE_BLOCK, __ldg(coeff + e), ke, det);
        if (gp >= 0) atomicMin(fail_min, (unsigned long long)e);
    }
    __syncthreads();
    if (e < n) {
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

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

// Self-test of div_markstein against __ddiv_rn: random mantissas, exponents spread over the
// guarded range, cancellation-like numerators, exact multiples and neighbours of exact
// quotients (the hardest rounding cases).  Counts mismatching bit patterns.
__global__ void division_selftest_kernel(uint64_t n, uint64_t seed, unsigned long long *mismatches,
                                         unsigned long long *tested) {
    unsigned long long bad = 0, cnt = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r1 = splitmix64(seed ^ (2 * i)), r2 = splitmix64(seed ^ (2 * i + 1));
        const int kind = (int)(r1 & 3);
        const int ea = (int)((r1 >> 2) & 1023) - 512, eb = (int)((r2 >> 2) & 1023) - 512;
        double b = __hiloint2double(0x3ff00000 | (int)((r2 >> 12) & 0xfffff), (int)(r2 >> 32));
        b = ldexp(b, kind == 0 ? eb : (eb & 63) - 32);
        double a = __hiloint2double(0x3ff00000 | (int)((r1 >> 12) & 0xfffff), (int)(r1 >> 32));
        a = ldexp(a, kind == 0 ? ea : (ea & 63) - 32);
        if (r1 & (1ull << 62)) a = -a;
        if (kind == 2) {  // a = exact-ish multiple of b, nudged by a few ulps
            const double q = __hiloint2double(0x3ff00000 | (int)((r2 >> 40) & 0xfffff), (int)r1);
            a = __dmul_rn(q, b);
            const long long bits = __double_as_longlong(a) + (long long)((r2 >> 60) & 7) - 3;
            a = __longlong_as_double(bits);
        } else if (kind == 3) {  // small-integer ratios (cancellation zeros and halves)
            a = (double)((long long)(r1 >> 40) % 97 - 48);
            b = (double)((r2 >> 40) % 13 + 1);
        }
        if (!(b > 0.0) || !div_safe(a) || !div_safe(b)) continue;
        const double y = __drcp_rn(b);
        const double q = div_markstein(a, b, y), ref = __ddiv_rn(a, b);
        bad += __double_as_longlong(q) != __double_as_longlong(ref);
        ++cnt;
    }
    atomicAdd(mismatches, bad);
    atomicAdd(tested, cnt);
}

}  // namespace hx

using namespace hx;

extern "C" int hx_selftest_division(uint64_t n, uint64_t seed, unsigned long long *result2, void *stream) {
    if (result2 == nullptr) {
        set_last_error("hx_selftest_division: null result");
        return HX_ERR_VALUE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    HX_TRY_CUDA(cudaMemsetAsync(result2, 0, 2 * sizeof(unsigned long long), s));
    division_selftest_kernel<<<148 * 8, 256, 0, s>>>(n, seed, result2, result2 + 1);
    HX_CHECK_LAUNCH("division_selftest_kernel");
    return HX_OK;
}

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
