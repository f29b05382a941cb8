// hx_ke_device.cuh -- device side of the integration kernel (hx_ke.cu): the per-(element, Gauss
// point) arithmetic in reference operation order, the warp's shared staging, the output stores and
// the persistent per-warp element-quad loop.  Included by hx_ke.cu (the integration kernels) and
// hx_assemble.cu (the integration kernel fused with the assembly's emit pass).
#pragma once
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "hx_common.cuh"

namespace hx {

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
// acc + dn*x with dn = sign * M_k  (bitwise equal to acc + (dn*x))
__device__ __forceinline__ double acc_signed(double acc, int sign, double prod) {
    return sign > 0 ? dadd(acc, prod) : dsub(acc, prod);
}

__device__ __forceinline__ double dabs_bits(double x) {
    return __hiloint2double(__double2hiint(x) & 0x7fffffff, __double2loint(x));
}
// x with the sign bit of s (x >= +0)
__device__ __forceinline__ double dsign_bits(double x, double s) {
    return __hiloint2double(__double2hiint(x) | (__double2hiint(s) & (int)0x80000000), __double2loint(x));
}

// IEEE round-to-nearest a/b (b > 0) from y = RN(1/b).  For A = |a|: q0 = RN(A y) is within 2 ulp
// of A/b; q1 = RN(q0 + (A - b q0) y) lands within 1 ulp (the FMA residual is exact); Markstein's
// theorem (y = RN(1/b), q1 within 1 ulp, exact residual) makes q2 = RN(q1 + (A - b q1) y) the
// correctly rounded quotient.  RN is odd-symmetric, so copysign(q2, a) == RN(a/b) -- including
// a = -0.  Valid while no intermediate over/underflows (the callers guarantee the operand range).
__device__ __forceinline__ double div_exact(double a, double b, double y) {
    const double A = dabs_bits(a);
    const double q0 = __dmul_rn(A, y);
    const double r0 = __fma_rn(-q0, b, A);
    const double q1 = __fma_rn(r0, y, q0);
    const double r1 = __fma_rn(-q1, b, A);
    const double q2 = __fma_rn(r1, y, q1);
    return dsign_bits(q2, a);
}

// det > 0 (element.py:276: `not det > 0` fails; NaN fails) on the integer pipe.
__device__ __forceinline__ bool positive(double x) {
    const long long b = __double_as_longlong(x);
    return b > 0 && b <= 0x7ff0000000000000ll;
}

// Coordinates 0 or with |x| in [2^-100, 2^100]: every J entry, cofactor and det of the element
// then stays within [2^-600, 2^320] or is exactly 0, so the Markstein quotients are exact.
__device__ __forceinline__ bool coord_in_range(double x) {
    const unsigned hi = (unsigned)__double2hiint(x) & 0x7fffffffu, lo = (unsigned)__double2loint(x);
    return (hi | lo) == 0u || hi - (unsigned)((1023 - 100) << 20) < (201u << 20);
}

// First failing Gauss point of one element and its det (reference order for J and det), or -1.
// Only the degenerate-element report needs it (element.py:237-244), so it runs single-threaded.
static __device__ int first_failing_gp(const double (&x)[8][3], double &fail_det) {
    for (int gp = 0; gp < 8; ++gp) {
        double dn[3][8];
        for (int a = 0; a < 8; ++a)
            for (int d = 0; d < 3; ++d) dn[d][a] = dn_value(gp, d, a);
        double j[3][3];
        for (int d = 0; d < 3; ++d)
            for (int k = 0; k < 3; ++k) {
                double acc = 0.0;
                for (int a = 0; a < 8; ++a) acc = dadd(acc, dmul(dn[d][a], x[a][k]));
                j[d][k] = acc;
            }
        const double c00 = dsub(dmul(j[1][1], j[2][2]), dmul(j[1][2], j[2][1]));
        const double c01 = dsub(dmul(j[1][2], j[2][0]), dmul(j[1][0], j[2][2]));
        const double c02 = dsub(dmul(j[1][0], j[2][1]), dmul(j[1][1], j[2][0]));
        const double det = dadd(dadd(dmul(j[0][0], c00), dmul(j[0][1], c01)), dmul(j[0][2], c02));
        if (!(det > 0.0)) {
            fail_det = det;
            return gp;
        }
    }
    return -1;
}

static __device__ void fail_detail(const double (&x)[8][3], int64_t element, hx_fail_info *fail) {
    double det = 0.0;
    const int gp = first_failing_gp(x, det);
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

// Packed pair tables in shared memory (lane-dependent p -> (i, j) lookups).
__device__ __forceinline__ void init_pack_smem(uint8_t *pi, uint8_t *pj) {
    for (int p = threadIdx.x; p < 36; p += blockDim.x) {
        int i = 0;
        while ((i + 1) * (i + 2) / 2 <= p) ++i;
        pi[p] = (uint8_t)i;
        pj[p] = (uint8_t)(p - i * (i + 1) / 2);
    }
}

// __launch_bounds__ minimum blocks: 15 gives ptxas a 136-register budget; it still allocates 128,
// so 16 one-warp blocks stay resident, but schedules better than under the exact 128 cap of 16:
// C4 KE kernel 21.1 -> 20.4 ms (13: 20.9, 14: 20.6; profiles/r02/ke_min_blocks.txt).
#ifndef HX_KE_MIN_BLOCKS
#define HX_KE_MIN_BLOCKS 15
#endif
#ifndef HX_KE_BLOCK
#define HX_KE_BLOCK 32
#endif
constexpr int GP_BLOCK = HX_KE_BLOCK;  // one warp (4 elements x 8 Gauss points) per block, 16 per SM at 128
                                       // regs: measured 0.6-0.9% faster than 4 x 128-thread blocks, 2% than 2 x 256
constexpr int GP_WARPS = GP_BLOCK / 32;
constexpr int GP_EL_PER_BLOCK = GP_BLOCK / 8;
constexpr int GP_EL_PER_WARP = 4;
// Shared products P[el][m][a][k] = M_m x[a][k]: m stride 25, element stride 76 (doubles) keep the
// <= 12 distinct (el, m) words of one warp-wide load in distinct bank pairs.
constexpr int P_M_STRIDE = 25;
constexpr int P_EL_STRIDE = 76;
// HX_KE_LANE_PRODUCTS (exact mode): the warp stages the raw coordinates X[el][k][a] instead of the
// 72 products, and every Gauss-point lane forms its own dN x products (the same roundings: M x with
// M the lane's magnitude, signs folded into the add/sub).  The integration kernel is bound by the
// LSU data pipe (ncu: 95% of its wavefronts, shared memory 77%): a lane's 72 product loads cost 24
// wavefronts per element, its 24 coordinates 3 (element-wide broadcast, 16-byte pairs), for +504
// DMUL per element.  Element stride 24 doubles (= 8 mod 16): the two elements of a half-warp hit
// distinct banks for both the 8-byte stores and the 16-byte pair loads.
#ifndef HX_KE_LANE_PRODUCTS
#define HX_KE_LANE_PRODUCTS 1
#endif
constexpr int X_EL_STRIDE = 24;
// Contribution buffer t[el][j][g]: g contiguous (the reducing lane reads 8 doubles with 4 x 16-B
// loads), j stride 10 and element stride 88 make both the stores and the loads conflict-free.
constexpr int T_J_STRIDE = 10;
constexpr int T_EL_STRIDE = 88;
// HX_KE_FULL_T: all 36 contributions of a Gauss point are staged at once (t[el][p][g], p stride 10,
// element stride 376 -- conflict-free 64-bit stores and 128-bit loads), so a lane reduces its up to
// five entries as independent chains after a single __syncwarp instead of five store/sync/reduce
// passes with one serial 8-add chain each.  The product table P aliases the buffer (it is dead once
// J is formed; a __syncwarp separates the last P read from the first contribution store).
// Measured: exact mode -0.5% with 4 x 128-thread blocks per SM and +0.6% with one-warp blocks x 16
// (the 12 KB per warp take L1 space from the coordinate gathers); fast mode -7% either way -- so the
// default is 1.
#ifndef HX_KE_FULL_T
#define HX_KE_FULL_T 1
#endif
constexpr int TF_EL_STRIDE = 376;

__host__ __device__ constexpr int bit_r(int a) { return nat_r(a) > 0; }
__host__ __device__ constexpr int bit_s(int a) { return nat_s(a) > 0; }
__host__ __device__ constexpr int bit_t(int a) { return nat_t(a) > 0; }

struct __align__(16) GpWarpSmem {
#if HX_KE_FULL_T
    union {
        double t[GP_EL_PER_WARP * TF_EL_STRIDE];
        double P[GP_EL_PER_WARP * P_EL_STRIDE];
    };
#else
    double t[GP_EL_PER_WARP * T_EL_STRIDE];
    double P[GP_EL_PER_WARP * P_EL_STRIDE];
#endif
    double coeff[GP_EL_PER_WARP];
    int32_t conn[GP_EL_PER_WARP * 8];
};

// Output stores of the integration kernel.  HX_KE_STREAM_STORES: evict-first (st.global.cs) -- KE,
// iK and jK are not re-read by this kernel, so they should not push the partially written adjacency
// slot sectors out of L2 (each slot sector collects 8 stores from elements up to a layer apart).
#ifndef HX_KE_STREAM_STORES
#define HX_KE_STREAM_STORES 1
#endif
template <typename T>
__device__ __forceinline__ void st_out(T *p, T v) {
#if HX_KE_STREAM_STORES
    __stcs(p, v);
#else
    *p = v;
#endif
}
// KE stores: evict-first like st_out, or (KE_KEEP, the build fused with the emit pass) plain
// write-back stores -- the emit tiles read the KE rows back from L2 shortly after.
template <bool KE_KEEP>
__device__ __forceinline__ void st_ke(double *p, double v) {
    if (KE_KEEP) *p = v;
    else st_out(p, v);
}

// All 36 staged contributions of element el (t[el][p][g]) reduced by its 8 lanes -- lane gp takes
// entries gp, gp + 8, ..., as independent chains -- and KE / iK / jK stored (HX_KE_FULL_T).  Exact
// mode sums in Gauss-point order, fast mode as a fixed depth-3 tree.
template <int MODE, bool WITH_INDEX, bool KE_KEEP = false>
__device__ __forceinline__ void reduce_store_all(const GpWarpSmem &sm, const double *tb, int el, int gp,
                                                 int64_t out_el, bool valid, double *__restrict__ ke_out,
                                                 int32_t *__restrict__ rows_out, int32_t *__restrict__ cols_out,
                                                 uint32_t pcode) {
    double acc[5];
#pragma unroll
    for (int c = 0; c < 5; ++c) {
        const int p = 8 * c + gp;
        acc[c] = 0.0;
        if (c < 4 || gp < 4) {
            const double2 *src = reinterpret_cast<const double2 *>(tb + p * T_J_STRIDE);
            const double2 v0 = src[0], v1 = src[1], v2 = src[2], v3 = src[3];
            if (MODE == HX_MODE_EXACT) {
                double a = dadd(0.0, v0.x);
                a = dadd(a, v0.y);
                a = dadd(a, v1.x);
                a = dadd(a, v1.y);
                a = dadd(a, v2.x);
                a = dadd(a, v2.y);
                a = dadd(a, v3.x);
                acc[c] = dadd(a, v3.y);
            } else {
                acc[c] = ((v0.x + v0.y) + (v1.x + v1.y)) + ((v2.x + v2.y) + (v3.x + v3.y));
            }
        }
    }
    if (valid) {
#pragma unroll
        for (int c = 0; c < 5; ++c) {
            const int p = 8 * c + gp;
            if (c < 4 || gp < 4) {
                st_ke<KE_KEEP>(ke_out + out_el * 36 + p, acc[c]);
                if (WITH_INDEX) {
                    const int pi = (pcode >> (6 * c)) & 7u, pj = (pcode >> (6 * c + 3)) & 7u;
                    const int32_t gi = sm.conn[el * 8 + pi], gj = sm.conn[el * 8 + pj];
                    st_out(rows_out + out_el * 36 + p, max(gi, gj));
                    st_out(cols_out + out_el * 36 + p, min(gi, gj));
                }
            }
        }
    }
}

__device__ __forceinline__ double mag_select(int k) {
    return k == 0 ? dn_magnitude(0) : (k == 1 ? dn_magnitude(1) : dn_magnitude(2));
}


// Lane (el, a): publish node a's id and, in exact mode, its products M_m x[a][k] (fast mode: the
// raw coordinates); the element's coefficient from a = 0.
template <int MODE>
__device__ __forceinline__ void publish_node(GpWarpSmem &sm, int el, int a, int32_t node, double x0, double x1,
                                             double x2, double c) {
    if (MODE == HX_MODE_EXACT && HX_KE_LANE_PRODUCTS) {
        double *X = sm.P + el * X_EL_STRIDE + a;
        X[0] = x0;
        X[8] = x1;
        X[16] = x2;
        sm.conn[el * 8 + a] = node;
        if (a == 0) sm.coeff[el] = c;
        return;
    }
    double *P = sm.P + el * P_EL_STRIDE + 3 * a;
    if (MODE == HX_MODE_EXACT) {
#pragma unroll
        for (int m = 0; m < 3; ++m) {
            P[m * P_M_STRIDE] = dmul(dn_magnitude(m), x0);
            P[m * P_M_STRIDE + 1] = dmul(dn_magnitude(m), x1);
            P[m * P_M_STRIDE + 2] = dmul(dn_magnitude(m), x2);
        }
    } else {
        P[0] = x0;
        P[1] = x1;
        P[2] = x2;
    }
    sm.conn[el * 8 + a] = node;
    if (a == 0) sm.coeff[el] = c;
}

// Reduce the element's 8 lanes' contributions of pass c and store KE / iK / jK (shared by both
// modes; exact mode sums in Gauss-point order, fast mode as a fixed depth-3 tree).
template <int MODE, bool WITH_INDEX>
__device__ __forceinline__ void reduce_store(const GpWarpSmem &sm, const double *tb, int el, int gp, int c,
                                             int64_t out_el, bool valid, double *__restrict__ ke_out,
                                             int32_t *__restrict__ rows_out, int32_t *__restrict__ cols_out,
                                             uint32_t pcode) {
    const int p = 8 * c + gp;  // this lane reduces packed entry p of its element
    if (p >= 36) return;
    const double2 *src = reinterpret_cast<const double2 *>(tb + gp * T_J_STRIDE);
    const double2 v0 = src[0], v1 = src[1], v2 = src[2], v3 = src[3];
    double acc;
    if (MODE == HX_MODE_EXACT) {
        acc = dadd(0.0, v0.x);
        acc = dadd(acc, v0.y);
        acc = dadd(acc, v1.x);
        acc = dadd(acc, v1.y);
        acc = dadd(acc, v2.x);
        acc = dadd(acc, v2.y);
        acc = dadd(acc, v3.x);
        acc = dadd(acc, v3.y);
    } else {
        acc = ((v0.x + v0.y) + (v1.x + v1.y)) + ((v2.x + v2.y) + (v3.x + v3.y));
    }
    if (valid) {
        ke_out[out_el * 36 + p] = acc;
        if (WITH_INDEX) {
            const int pi = (pcode >> (6 * c)) & 7u, pj = (pcode >> (6 * c + 3)) & 7u;
            const int32_t gi = sm.conn[el * 8 + pi], gj = sm.conn[el * 8 + pj];
            rows_out[out_el * 36 + p] = max(gi, gj);
            cols_out[out_el * 36 + p] = min(gi, gj);
        }
    }
}

// Fast mode (HX_MODE_FAST): the same quadrature restructured for FMA,
//   ke_ij += dN_i^T G dN_j,  G = (c / det) adj(J)^T adj(J)  (= c det J^-1 J^-T),
// about 300 FP64 operations per Gauss point instead of ~500 in reference order.  Not bitwise:
// |KE - KE_ref| <= 1e-12 max_j |KE_ref[e, j]| per element (tests/test_gpu_fast_mode.py), and the
// degenerate-element test uses this det (differs from the reference only for |det| at rounding
// level of 0).
template <bool WITH_INDEX, bool KE_KEEP = false>
__device__ __forceinline__ bool ke_gauss_point_fast(GpWarpSmem &sm, int el, int gp, int64_t out_el, bool valid,
                                                    double *__restrict__ ke_out, int32_t *__restrict__ rows_out,
                                                    int32_t *__restrict__ cols_out, uint32_t pcode) {
    const int ir = (gp >> 2) & 1, is = (gp >> 1) & 1, it = gp & 1;
    const double *X = sm.P + el * P_EL_STRIDE;
    double Mr[4], Ms[4], Mt[4];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
            Mr[2 * u + v] = mag_select((u == is) + (v == it));
            Ms[2 * u + v] = mag_select((u == ir) + (v == it));
            Mt[2 * u + v] = mag_select((u == ir) + (v == is));
        }
    // dN[d][a] = sign(d, a) * M (register-resident for this lane's Gauss point)
    auto dn = [&](int d, int a) -> double {
        const double m = d == 0 ? Mr[2 * bit_s(a) + bit_t(a)] : d == 1 ? Ms[2 * bit_r(a) + bit_t(a)]
                                                               : Mt[2 * bit_r(a) + bit_s(a)];
        const int sg = d == 0 ? nat_r(a) : d == 1 ? nat_s(a) : nat_t(a);
        return sg > 0 ? m : -m;
    };
    double j[3][3];
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            double acc = dn(d, 0) * X[k];
#pragma unroll
            for (int a = 1; a < 8; ++a) acc = fma(dn(d, a), X[3 * a + k], acc);
            j[d][k] = acc;
        }
    // adjugate: a[r][d] = det * inv[r][d]
    double ad[3][3];
    ad[0][0] = fma(j[1][1], j[2][2], -j[1][2] * j[2][1]);
    ad[0][1] = fma(j[0][2], j[2][1], -j[0][1] * j[2][2]);
    ad[0][2] = fma(j[0][1], j[1][2], -j[0][2] * j[1][1]);
    ad[1][0] = fma(j[1][2], j[2][0], -j[1][0] * j[2][2]);
    ad[1][1] = fma(j[0][0], j[2][2], -j[0][2] * j[2][0]);
    ad[1][2] = fma(j[0][2], j[1][0], -j[0][0] * j[1][2]);
    ad[2][0] = fma(j[1][0], j[2][1], -j[1][1] * j[2][0]);
    ad[2][1] = fma(j[0][1], j[2][0], -j[0][0] * j[2][1]);
    ad[2][2] = fma(j[0][0], j[1][1], -j[0][1] * j[1][0]);
    const double det = fma(j[0][0], ad[0][0], fma(j[0][1], ad[1][0], j[0][2] * ad[2][0]));
    const bool ok = positive(det);
    const double f = sm.coeff[el] * __drcp_rn(det);
    // G = f adj^T adj (symmetric)
    double G[3][3];
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
        for (int e = d; e < 3; ++e) {
            G[d][e] = f * fma(ad[0][d], ad[0][e], fma(ad[1][d], ad[1][e], ad[2][d] * ad[2][e]));
            G[e][d] = G[d][e];
        }
    // H = G dN (3 x 8)
    double H[3][8];
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
        for (int a = 0; a < 8; ++a) H[d][a] = fma(G[d][0], dn(0, a), fma(G[d][1], dn(1, a), G[d][2] * dn(2, a)));
#if HX_KE_FULL_T
    __syncwarp();  // every lane has read the coordinates, which the contribution buffer overwrites
    {
        double *tf = sm.t + el * TF_EL_STRIDE;
#pragma unroll
        for (int p = 0; p < 36; ++p) {
            const int i = pack_i(p), q = pack_j(p);
            tf[p * T_J_STRIDE + gp] = fma(dn(0, i), H[0][q], fma(dn(1, i), H[1][q], dn(2, i) * H[2][q]));
        }
        __syncwarp();
        reduce_store_all<HX_MODE_FAST, WITH_INDEX, KE_KEEP>(sm, tf, el, gp, out_el, valid, ke_out, rows_out, cols_out, pcode);
    }
    return ok;
#endif
    double *tb = sm.t + el * T_EL_STRIDE;
#pragma unroll
    for (int c = 0; c < 5; ++c) {
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
            const int p = 8 * c + jj;
            if (p < 36) {
                const int i = pack_i(p), q = pack_j(p);
                tb[jj * T_J_STRIDE + gp] = fma(dn(0, i), H[0][q], fma(dn(1, i), H[1][q], dn(2, i) * H[2][q]));
            }
        }
        __syncwarp();
        reduce_store<HX_MODE_FAST, WITH_INDEX>(sm, tb, el, gp, c, out_el, valid, ke_out, rows_out, cols_out, pcode);
        __syncwarp();
    }
    return ok;
}

// Gauss point gp of element el (products published in sm), reference operation order; then the
// cooperative reduction and the KE / iK / jK stores of element out_el.  Returns det > 0.
template <bool WITH_INDEX, bool KE_KEEP = false>
__device__ __forceinline__ bool ke_gauss_point(GpWarpSmem &sm, int el, int gp, bool fast_div,
                                               int64_t out_el, bool valid, double *__restrict__ ke_out,
                                               int32_t *__restrict__ rows_out, int32_t *__restrict__ cols_out,
                                               uint32_t pcode) {
    const int ir = (gp >> 2) & 1, is = (gp >> 1) & 1, it = gp & 1;
    // This lane's dN magnitudes per direction, indexed by the node's other two natural coordinates
    // (dN_r,a = sign * Mr[2 s_a + t_a], cyclically for s and t).
    double Mr[4], Ms[4], Mt[4];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
            Mr[2 * u + v] = mag_select((u == is) + (v == it));  // (s_a, t_a)
            Ms[2 * u + v] = mag_select((u == ir) + (v == it));  // (r_a, t_a)
            Mt[2 * u + v] = mag_select((u == ir) + (v == is));  // (r_a, s_a)
        }
    // J = dn @ x (element.py:262-269), accumulated from 0.0 over a = 0..7.
    double j[3][3];
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
        for (int k = 0; k < 3; ++k) j[d][k] = 0.0;
#if HX_KE_LANE_PRODUCTS
    const double *X = sm.P + el * X_EL_STRIDE;
#pragma unroll
    for (int a2 = 0; a2 < 8; a2 += 2)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double2 xv = *reinterpret_cast<const double2 *>(X + 8 * k + a2);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int a = a2 + h;
                const double x = h ? xv.y : xv.x;
                j[0][k] = acc_signed(j[0][k], nat_r(a), dmul(Mr[2 * bit_s(a) + bit_t(a)], x));
                j[1][k] = acc_signed(j[1][k], nat_s(a), dmul(Ms[2 * bit_r(a) + bit_t(a)], x));
                j[2][k] = acc_signed(j[2][k], nat_t(a), dmul(Mt[2 * bit_r(a) + bit_s(a)], x));
            }
        }
#else
    // dN_r,a at this point has magnitude index (s_a == s_gp) + (t_a == t_gp), and cyclically for s
    // and t: the published products P[m][a][k] = M_m x[a][k].
    const double *P = sm.P + el * P_EL_STRIDE;
#pragma unroll
    for (int a = 0; a < 8; ++a) {
        const int mr = (bit_s(a) == is) + (bit_t(a) == it);
        const int ms = (bit_r(a) == ir) + (bit_t(a) == it);
        const int mt = (bit_r(a) == ir) + (bit_s(a) == is);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            j[0][k] = acc_signed(j[0][k], nat_r(a), P[mr * P_M_STRIDE + 3 * a + k]);
            j[1][k] = acc_signed(j[1][k], nat_s(a), P[ms * P_M_STRIDE + 3 * a + k]);
            j[2][k] = acc_signed(j[2][k], nat_t(a), P[mt * P_M_STRIDE + 3 * a + k]);
        }
    }
#endif
    // cofactors, det (element.py:271-275)
    const double c00 = dsub(dmul(j[1][1], j[2][2]), dmul(j[1][2], j[2][1]));
    const double c01 = dsub(dmul(j[1][2], j[2][0]), dmul(j[1][0], j[2][2]));
    const double c02 = dsub(dmul(j[1][0], j[2][1]), dmul(j[1][1], j[2][0]));
    const double det = dadd(dadd(dmul(j[0][0], c00), dmul(j[0][1], c01)), dmul(j[0][2], c02));
    const bool ok = positive(det);
    // adjugate / det (element.py:281-284): true divisions
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
    double inv[3][3];
    if (fast_div && ok) {
        const double y = __drcp_rn(det);
#pragma unroll
        for (int i = 0; i < 9; ++i) inv[i / 3][i % 3] = div_exact(num[i], det, y);
    } else {
#pragma unroll
        for (int i = 0; i < 9; ++i) inv[i / 3][i % 3] = __ddiv_rn(num[i], det);
    }
    // B = J^-1 dn (element.py:286-290): (i_r0 dn0a + i_r1 dn1a) + i_r2 dn2a with dn = sign * M.
    double B[3][8];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        double q0[4], q1[4], q2[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            q0[c] = dmul(inv[r][0], Mr[c]);
            q1[c] = dmul(inv[r][1], Ms[c]);
            q2[c] = dmul(inv[r][2], Mt[c]);
        }
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            const double p0 = q0[2 * bit_s(a) + bit_t(a)];
            const double t0 = nat_r(a) > 0 ? p0 : -p0;
            const double t01 = acc_signed(t0, nat_s(a), q1[2 * bit_r(a) + bit_t(a)]);
            B[r][a] = acc_signed(t01, nat_t(a), q2[2 * bit_r(a) + bit_s(a)]);
        }
    }
    const double scale = dmul(sm.coeff[el], det);
#if HX_KE_FULL_T
    __syncwarp();  // every lane has read its J from P, which the contribution buffer overwrites
    {
        double *tf = sm.t + el * TF_EL_STRIDE;
#pragma unroll
        for (int p = 0; p < 36; ++p) {
            const int i = pack_i(p), q = pack_j(p);
            const double s = dadd(dadd(dmul(B[0][i], B[0][q]), dmul(B[1][i], B[1][q])), dmul(B[2][i], B[2][q]));
            tf[p * T_J_STRIDE + gp] = dmul(scale, s);
        }
        __syncwarp();
        reduce_store_all<HX_MODE_EXACT, WITH_INDEX, KE_KEEP>(sm, tf, el, gp, out_el, valid, ke_out, rows_out, cols_out, pcode);
    }
    return ok;
#endif
    // 36 contributions, 8 per pass, reduced across the element's 8 lanes in Gauss-point order
    double *tb = sm.t + el * T_EL_STRIDE;
#pragma unroll
    for (int c = 0; c < 5; ++c) {
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
            const int p = 8 * c + jj;
            if (p < 36) {
                const int i = pack_i(p), q = pack_j(p);
                const double s = dadd(dadd(dmul(B[0][i], B[0][q]), dmul(B[1][i], B[1][q])), dmul(B[2][i], B[2][q]));
                tb[jj * T_J_STRIDE + gp] = dmul(scale, s);
            }
        }
        __syncwarp();
        reduce_store<HX_MODE_EXACT, WITH_INDEX>(sm, tb, el, gp, c, out_el, valid, ke_out, rows_out, cols_out, pcode);
        __syncwarp();
    }
    return ok;
}

// Mesh kernel: elements [lo, lo+n) of the mesh; outputs indexed from 0 (= element lo).
// Persistent warps, each prefetching the next quad's node ids, coordinates and coefficients into
// registers before integrating the current one, so the gather latency hides under the FP64 work.
// Work distribution: warps take element quads from a global counter (self-balancing, also when the
// kernel shares the GPU with a concurrently running symbolic phase).  HX_KE_STATIC=1 assigns quads
// w, w + W, w + 2W, ... instead (no counter atomic): measured 1% slower at C3/C4 although ncu
// attributes 15% of the stall samples to waiting on the atomic's result -- other warps fill those
// cycles, so the default stays dynamic.
#ifndef HX_KE_STATIC
#define HX_KE_STATIC 0
#endif
// HX_KE_CLAIM: quads per counter claim (ptxas turns the lane-0 atomicAdd into a warp-aggregated
// atomic whose result SHFL follows the ATOM directly, so every claim stalls its warp for a round trip).
#ifndef HX_KE_CLAIM
#define HX_KE_CLAIM 16  // 8-64 measured equal, 3.5% faster than 1 at C4 and C5 (profiles/r02/ke_claim_batch.txt)
#endif
#ifndef HX_KE_LATE_GRAB
#define HX_KE_LATE_GRAB 1
#endif
// Adjacency output of the fused symbolic first pass (WITH_ADJ): adj (8 n_nodes) i32 fixed slots
// (emptied to -1 by the caller), status bit HX_ST_BAD_INDEX.
struct AdjOut {
    int32_t *adj;
    uint32_t *status;
};

// The persistent warp loop of the integration kernel: element quads from a global counter, each
// warp prefetching the next quad's node ids, coordinates and coefficients into registers before
// integrating the current one.  hook.after_quad(quad) runs after every integrated quad (its KE rows
// are stored) and hook.drain() once the warp's last quad is done -- no-ops for the plain
// integration kernel; the kernel fused with the emit pass signals quad completion and runs ready
// emit tiles there.
struct NoHook {
    __device__ __forceinline__ void after_quad(int64_t) {}
    __device__ __forceinline__ void drain() {}
};

template <int MODE, bool WITH_INDEX, bool WITH_ADJ, bool KE_KEEP, typename Hook>
__device__ __forceinline__ void integrate_quads(GpWarpSmem &sm, const uint8_t *s_pi, const uint8_t *s_pj,
                                                const double *__restrict__ coords, int64_t n_nodes,
                                                const int32_t *__restrict__ conn, const double *__restrict__ coeff,
                                                int64_t lo, int64_t n, double *__restrict__ ke_out,
                                                int32_t *__restrict__ rows_out, int32_t *__restrict__ cols_out,
                                                unsigned long long *__restrict__ fail_min,
                                                unsigned *__restrict__ quad_counter, AdjOut adj_out, Hook &hook) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int el = lane >> 3, gp = lane & 7;
    // the (i, j) local nodes of this lane's packed entries p = gp + 8c, 3 + 3 bits per c, in a register
    uint32_t pcode = 0;
#pragma unroll
    for (int c = 0; c < 5; ++c)
        if (8 * c + gp < 36) pcode |= (uint32_t)(s_pi[8 * c + gp] | (s_pj[8 * c + gp] << 3)) << (6 * c);
    const int64_t n_quads = (n + GP_EL_PER_WARP - 1) / GP_EL_PER_WARP;
    const int64_t first_dynamic = (int64_t)gridDim.x * GP_WARPS;
    int64_t static_next = (int64_t)blockIdx.x * GP_WARPS + warp;
    int64_t spare = 0;  // the rest of the last claim: quads spare .. spare + spare_n - 1
    int spare_n = 0;
    auto grab = [&]() -> int64_t {
        if (HX_KE_STATIC) {
            (void)quad_counter;
            static_next += first_dynamic;
            return static_next;
        }
        if (spare_n > 0) {
            --spare_n;
            return spare++;
        }
        unsigned q = 0;
        if (lane == 0) q = atomicAdd(quad_counter, (unsigned)HX_KE_CLAIM);
        const int64_t base = first_dynamic + (int64_t)__shfl_sync(0xffffffffu, q, 0);
        spare = base + 1;
        spare_n = HX_KE_CLAIM - 1;
        return base;
    };
    auto node_id = [&](int64_t q) -> int32_t {
        const int64_t k = q * GP_EL_PER_WARP + el;
        return k < n ? __ldg(conn + (lo + k) * 8 + gp) : -1;
    };
    // padding lanes integrate a unit cube (keeps them off the slow paths; never stored)
    const double u0 = nat_r(gp) > 0, u1 = nat_s(gp) > 0, u2 = nat_t(gp) > 0;
    int64_t quad = (int64_t)blockIdx.x * GP_WARPS + warp;  // being published / integrated
    int64_t quad1 = quad < n_quads ? grab() : n_quads;      // coordinates in flight
    int64_t quad2 = quad1 < n_quads ? grab() : n_quads;     // node ids in flight
    int32_t node = node_id(quad), node_next = node_id(quad1);
    double x0 = u0, x1 = u1, x2 = u2, c = 1.0;
    // node ids outside [0, n_nodes) are never dereferenced: the element is reported through the
    // fail record (bad-node key, below) and, fused, the assembly status (HX_ST_BAD_INDEX)
    if (node >= 0 && node < n_nodes) {
        const double *p = coords + 3 * (int64_t)node;
        x0 = __ldg(p); x1 = __ldg(p + 1); x2 = __ldg(p + 2);
        c = __ldg(coeff + lo + quad * GP_EL_PER_WARP + el);
    }
    while (quad < n_quads) {
        const int64_t k = quad * GP_EL_PER_WARP + el;
        const bool valid = k < n;
        const unsigned in_range = __ballot_sync(0xffffffffu, coord_in_range(x0) && coord_in_range(x1) &&
                                                               coord_in_range(x2));
        const bool fast_div = ((in_range >> (8 * el)) & 0xffu) == 0xffu;
        // fixed-slot adjacency: (element, local node gp) -> slot gp of its node (fire and forget)
        if (valid && (node < 0 || node >= n_nodes)) {
            atomicMin(fail_min, (unsigned long long)(lo + k));  // bad-node key: below every degenerate key
            if (WITH_ADJ) atomicOr(adj_out.status, HX_ST_BAD_INDEX);
        } else if (WITH_ADJ && valid) {
            adj_out.adj[8 * (int64_t)node + gp] = (int32_t)(((lo + k) << 3) | gp);
        }
        __syncwarp();
        publish_node<MODE>(sm, el, gp, node, x0, x1, x2, c);
        __syncwarp();
        // prefetch: coordinates of quad1, node ids of quad2, claim the quad after
        node = node_next;
        node_next = node_id(quad2);
        x0 = u0; x1 = u1; x2 = u2; c = 1.0;
        if (node >= 0 && node < n_nodes) {
            const double *p = coords + 3 * (int64_t)node;
            x0 = __ldg(p); x1 = __ldg(p + 1); x2 = __ldg(p + 2);
            c = __ldg(coeff + lo + quad1 * GP_EL_PER_WARP + el);
        }
#if HX_KE_LATE_GRAB
        // claim the quad after next now, read the claim after this quad's FP64 work: the atomic's
        // round trip overlaps the Gauss-point arithmetic instead of stalling the warp here
        unsigned claim = 0;
        const bool claiming = !HX_KE_STATIC && quad2 < n_quads && spare_n == 0;
        if (claiming && lane == 0) claim = atomicAdd(quad_counter, (unsigned)HX_KE_CLAIM);
#else
        const int64_t quad3 = quad2 < n_quads ? grab() : n_quads;
#endif
        bool ok;
        if constexpr (MODE == HX_MODE_EXACT)
            ok = ke_gauss_point<WITH_INDEX, KE_KEEP>(sm, el, gp, fast_div, k, valid, ke_out, rows_out, cols_out, pcode);
        else
            ok = ke_gauss_point_fast<WITH_INDEX, KE_KEEP>(sm, el, gp, k, valid, ke_out, rows_out, cols_out, pcode);
        if (valid && !ok) atomicMin(fail_min, HX_FAIL_DEGENERATE_KEY | (unsigned long long)(lo + k));
#if HX_KE_LATE_GRAB
        int64_t quad3 = n_quads;
        if (quad2 < n_quads) {
            if (HX_KE_STATIC) {
                static_next += first_dynamic;
                quad3 = static_next;
            } else if (claiming) {
                quad3 = first_dynamic + (int64_t)__shfl_sync(0xffffffffu, claim, 0);
                spare = quad3 + 1;
                spare_n = HX_KE_CLAIM - 1;
            } else {
                --spare_n;
                quad3 = spare++;
            }
        }
#endif
        hook.after_quad(quad);
        quad = quad1;
        quad1 = quad2;
        quad2 = quad3;
    }
    hook.drain();
}

}  // namespace hx
