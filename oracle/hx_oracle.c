/*
 * hx_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * Plain-C restatement of the reference hexfem element kernel so the CUDA path can be
 * checked bit-for-bit.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.
 *
 * Reference followed (file:line under /root/reference/pkg/src/hexfem/):
 *   element.py:43-56    NODE_NATURAL_COORDS (ccw bottom face, then ccw top face)
 *   element.py:104-113  shape_gradients: 0.125 * ra * (1 + sa*s) * (1 + ta*t), left-assoc
 *   element.py:116-124  Gauss points r slowest, t fastest, g = 1/sqrt(3)
 *   element.py:59-62    packing = np.tril_indices(8), row-major lower
 *   element.py:248-297  _stiffness_kernel: J accumulation from 0.0 over a = 0..7,
 *                       first-row cofactors, det, `not det > 0` failure, adjugate/det
 *                       (true division), B = J^-1 dN, ke[p] += (c*det)*((b0+b1)+b2)
 *   element.py:213-245  stiffness_batch: lowest failing element wins
 *   integrate.py:146-149 _stage_group: coords[conn] gather (fused here for the mesh variant)
 *
 * Build with -ffp-contract=off (see oracle/Makefile): the numba kernel is strict IEEE with
 * no FMA contraction, and this restatement matches it bitwise (tests/test_oracle.py pins it
 * against golden vectors produced by the reference itself, tests/golden/make_golden.py).
 *
 * Parity status: PINNED (golden vectors + digests from the reference run in the build
 * container; see tests/golden/README.md).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <pthread.h>

/* Minimal static-schedule parallel-for over [0, n) (numba prange analogue, element.py:252). */
typedef void (*hxo_body_fn)(int64_t lo, int64_t hi, void *ctx);
typedef struct { hxo_body_fn fn; void *ctx; int64_t lo, hi; } hxo_task;
static void *hxo_run_task(void *arg) {
    hxo_task *t = (hxo_task *)arg;
    t->fn(t->lo, t->hi, t->ctx);
    return NULL;
}
static void hxo_parallel_for(int64_t n, int threads, hxo_body_fn fn, void *ctx) {
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    if (n < 1024 || threads == 1) { fn(0, n, ctx); return; }
    pthread_t tid[256];
    hxo_task task[256];
    const int64_t base = n / threads, extra = n % threads;
    int64_t lo = 0;
    for (int t = 0; t < threads; ++t) {
        const int64_t hi = lo + base + (t < extra ? 1 : 0);
        task[t] = (hxo_task){fn, ctx, lo, hi};
        lo = hi;
    }
    for (int t = 1; t < threads; ++t) pthread_create(&tid[t], NULL, hxo_run_task, &task[t]);
    hxo_run_task(&task[0]);
    for (int t = 1; t < threads; ++t) pthread_join(tid[t], NULL);
}

static const double NAT[8][3] = {
    {-1.0, -1.0, -1.0}, {+1.0, -1.0, -1.0}, {+1.0, +1.0, -1.0}, {-1.0, +1.0, -1.0},
    {-1.0, -1.0, +1.0}, {+1.0, -1.0, +1.0}, {+1.0, +1.0, +1.0}, {-1.0, +1.0, +1.0},
};

static double DN[8][3][8];
static int PI_[36], PJ_[36];
static int tables_ready = 0;

/* element.py:104-113 and element.py:116-130 */
static void build_tables(void) {
    if (tables_ready) return;
    const double g = 1.0 / sqrt(3.0);
    int gp = 0;
    for (int ir = 0; ir < 2; ++ir)
        for (int is = 0; is < 2; ++is)
            for (int it = 0; it < 2; ++it, ++gp) {
                const double r = ir ? g : -g, s = is ? g : -g, t = it ? g : -g;
                for (int a = 0; a < 8; ++a) {
                    const double ra = NAT[a][0], sa = NAT[a][1], ta = NAT[a][2];
                    DN[gp][0][a] = 0.125 * ra * (1.0 + sa * s) * (1.0 + ta * t);
                    DN[gp][1][a] = 0.125 * sa * (1.0 + ra * r) * (1.0 + ta * t);
                    DN[gp][2][a] = 0.125 * ta * (1.0 + ra * r) * (1.0 + sa * s);
                }
            }
    int p = 0;
    for (int i = 0; i < 8; ++i)
        for (int j = 0; j <= i; ++j, ++p) { PI_[p] = i; PJ_[p] = j; }
    tables_ready = 1;
}

void hxo_dn_table(double *out /* 8*3*8 */) {
    build_tables();
    memcpy(out, DN, sizeof(DN));
}

/* element.py:255-297 for one element; returns failing gauss point or -1. */
static int element_ke(const double x[8][3], double c, double *ke, double *fail_det) {
    double B[3][8];
    for (int p = 0; p < 36; ++p) ke[p] = 0.0;
    for (int gp = 0; gp < 8; ++gp) {
        const double (*dn)[8] = DN[gp];
        double j00 = 0.0, j01 = 0.0, j02 = 0.0;
        double j10 = 0.0, j11 = 0.0, j12 = 0.0;
        double j20 = 0.0, j21 = 0.0, j22 = 0.0;
        for (int a = 0; a < 8; ++a) {
            j00 += dn[0][a] * x[a][0]; j01 += dn[0][a] * x[a][1]; j02 += dn[0][a] * x[a][2];
            j10 += dn[1][a] * x[a][0]; j11 += dn[1][a] * x[a][1]; j12 += dn[1][a] * x[a][2];
            j20 += dn[2][a] * x[a][0]; j21 += dn[2][a] * x[a][1]; j22 += dn[2][a] * x[a][2];
        }
        const double c00 = j11 * j22 - j12 * j21;
        const double c01 = j12 * j20 - j10 * j22;
        const double c02 = j10 * j21 - j11 * j20;
        const double det = j00 * c00 + j01 * c01 + j02 * c02;
        if (!(det > 0.0)) { *fail_det = det; return gp; }
        const double i00 = c00 / det, i01 = (j02 * j21 - j01 * j22) / det, i02 = (j01 * j12 - j02 * j11) / det;
        const double i10 = c01 / det, i11 = (j00 * j22 - j02 * j20) / det, i12 = (j02 * j10 - j00 * j12) / det;
        const double i20 = c02 / det, i21 = (j01 * j20 - j00 * j21) / det, i22 = (j00 * j11 - j01 * j10) / det;
        for (int a = 0; a < 8; ++a) {
            B[0][a] = i00 * dn[0][a] + i01 * dn[1][a] + i02 * dn[2][a];
            B[1][a] = i10 * dn[0][a] + i11 * dn[1][a] + i12 * dn[2][a];
            B[2][a] = i20 * dn[0][a] + i21 * dn[1][a] + i22 * dn[2][a];
        }
        const double scale = c * det;
        for (int p = 0; p < 36; ++p) {
            const int i = PI_[p], j = PJ_[p];
            ke[p] += scale * (B[0][i] * B[0][j] + B[1][i] * B[1][j] + B[2][i] * B[2][j]);
        }
    }
    return -1;
}

typedef struct { const double *coords, *coeff; double *out; int32_t *fail_gp; double *fail_det; } batch_ctx;
static void batch_body(int64_t lo, int64_t hi, void *vctx) {
    batch_ctx *c = (batch_ctx *)vctx;
    for (int64_t e = lo; e < hi; ++e) {
        double det = 0.0;
        const int gp = element_ke((const double (*)[3])(c->coords + 24 * e), c->coeff[e], c->out + 36 * e, &det);
        c->fail_gp[e] = gp;
        c->fail_det[e] = gp >= 0 ? det : 0.0;
    }
}

/* stiffness_batch (element.py:213-245) on pre-gathered coords (n,8,3).
 * Returns the lowest failing element index (0-based, batch-local) or -1. */
int64_t hxo_stiffness_batch(const double *coords, const double *coeff, int64_t n, double *out,
                            int32_t *fail_gp, double *fail_det, int threads) {
    build_tables();
    batch_ctx ctx = {coords, coeff, out, fail_gp, fail_det};
    hxo_parallel_for(n, threads, batch_body, &ctx);
    for (int64_t e = 0; e < n; ++e)
        if (fail_gp[e] >= 0) return e;
    return -1;
}

typedef struct {
    const double *coords; const int32_t *conn; const double *coeff; int64_t lo;
    double *out; int32_t *rows, *cols; int32_t *fail_gp; double *fail_det;
} mesh_ctx;
static void mesh_body(int64_t klo, int64_t khi, void *vctx) {
    mesh_ctx *c = (mesh_ctx *)vctx;
    for (int64_t k = klo; k < khi; ++k) {
        const int64_t e = c->lo + k;
        double x[8][3];
        const int32_t *g = c->conn + 8 * e;
        for (int a = 0; a < 8; ++a)
            for (int d = 0; d < 3; ++d) x[a][d] = c->coords[3 * (int64_t)g[a] + d];
        double det = 0.0;
        const int gp = element_ke((const double (*)[3])x, c->coeff[e], c->out + 36 * k, &det);
        c->fail_gp[k] = gp;
        c->fail_det[k] = gp >= 0 ? det : 0.0;
        if (c->rows) {
            for (int p = 0; p < 36; ++p) {
                const int32_t gr = g[PI_[p]], gc = g[PJ_[p]];
                c->rows[36 * k + p] = gr > gc ? gr : gc;
                c->cols[36 * k + p] = gr > gc ? gc : gr;
            }
        }
    }
}

/* Mesh variant: integrate_all's gather (integrate.py:146-149) fused with the kernel, plus
 * connectivity_index_arrays (assemble.py:86-93) when rows/cols are non-NULL.
 * Elements [lo, hi) of the mesh; outputs are indexed from lo. */
int64_t hxo_stiffness_mesh(const double *coords, const int32_t *conn, const double *coeff,
                           int64_t lo, int64_t hi, double *out, int32_t *rows, int32_t *cols,
                           int32_t *fail_gp, double *fail_det, int threads) {
    build_tables();
    const int64_t n = hi - lo;
    mesh_ctx ctx = {coords, conn, coeff, lo, out, rows, cols, fail_gp, fail_det};
    hxo_parallel_for(n, threads, mesh_body, &ctx);
    for (int64_t k = 0; k < n; ++k)
        if (fail_gp[k] >= 0) return lo + k;
    return -1;
}
