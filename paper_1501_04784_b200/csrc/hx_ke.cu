// hx_ke.cu -- numerical integration (the paper's Algorithm 2) for hex8 Poisson elements on
// sm_100a, fused with the iK/jK triplet index generation.
//
// Exact mode (the only arithmetic this file ships) reproduces element.py:255-297 operation for
// operation with explicitly rounded intrinsics (__dmul_rn/__dadd_rn cannot be contracted into
// FMA), so KE is bitwise equal to the reference's numba kernel.  Tensor cores are deliberately
// not used: the contractions are 8x3 and FP64, and the kernel is FP64-pipe bound.
//
// Work decomposition: one thread per (element, Gauss point).  A warp holds 4 elements x 8 Gauss
// points (lane = 8 el + gp):
//   * lane (el, a) gathers node a of its element (connectivity row read 8-wide across lanes) and
//     stores the 9 products M_m * x[a][k] (m = the 3 dN magnitudes) to shared memory -- the only
//     distinct products of J = dN @ X over all eight Gauss points (72 per element instead of 576);
//   * lane (el, gp) then runs Gauss point gp in reference order: J (signed sums of the shared
//     products), cofactors, det, the 9 true divisions, B, and its 36 contributions
//     t_gp[p] = (c det) ((B0i B0j + B1i B1j) + B2i B2j);
//   * the element's 8 lanes reduce ke[p] = ((((0 + t_0) + t_1) + ...) + t_7) in Gauss-point order
//     through a per-warp shared buffer (8 entries per pass) -- the reference's accumulation -- and
//     store KE and the fused iK/jK as 8-wide element-major runs.
// Warps are persistent and prefetch the next element quad's connectivity and coordinates into
// registers while integrating the current one.
// With WITH_ADJ the kernel also records the node adjacency of the mesh-path assembly (the symbolic
// phase's first pass): lane (el, a) already holds node a of its element and stores (element << 3 |
// a) into slot a of that node -- a fixed slot, so no atomic and no returned value stalls the FP64
// work; the connectivity is read once for both.  Meshes whose elements put one node at the same
// local index twice (inconsistent orientation) lose a slot; the pattern pass counts the filled
// slots and the build then re-runs the atomic adjacency (HX_ST_SLOT_COLLISION).
//
// Bit-preserving rewrites:
//   * dN = sign * M_k with M_k one of three magnitudes; (-M)*x == -(M*x) exactly, so the sign is
//     folded into add/sub and the products are shared between Gauss points;
//   * a/b = copysign(Markstein(|a|, b, RN(1/b)), a): reciprocal + two FMA corrections, bitwise
//     __ddiv_rn(a, b) while nothing over/underflows.  That is guaranteed for every element whose
//     coordinates are 0 or within [2^-100, 2^100] in magnitude (checked per element; other
//     elements take __ddiv_rn).  hx_selftest_division checks the quotient on 2^30 operand pairs.
#include "hx_ke_device.cuh"

namespace hx {

template <int MODE, bool WITH_INDEX, bool WITH_ADJ>
__global__ void __launch_bounds__(GP_BLOCK, HX_KE_MIN_BLOCKS)
integrate_mesh_kernel(const double *__restrict__ coords, int64_t n_nodes, const int32_t *__restrict__ conn,
                      const double *__restrict__ coeff, int64_t lo, int64_t n,
                      double *__restrict__ ke_out, int32_t *__restrict__ rows_out,
                      int32_t *__restrict__ cols_out, unsigned long long *__restrict__ fail_min,
                      unsigned *__restrict__ quad_counter, AdjOut adj_out) {
    extern __shared__ __align__(16) unsigned char s_dyn[];
    GpWarpSmem *s_warp = reinterpret_cast<GpWarpSmem *>(s_dyn);
    __shared__ uint8_t s_pi[36], s_pj[36];
    init_pack_smem(s_pi, s_pj);
    __syncthreads();
    NoHook hook;
    integrate_quads<MODE, WITH_INDEX, WITH_ADJ, false>(s_warp[threadIdx.x >> 5], s_pi, s_pj, coords, n_nodes, conn,
                                                       coeff, lo, n, ke_out, rows_out, cols_out, fail_min,
                                                       quad_counter, adj_out, hook);
}

// Batch kernel: pre-gathered coords (n, 8, 3) (stiffness_batch, element.py:213-245).
template <int MODE>
__global__ void __launch_bounds__(GP_BLOCK, HX_KE_MIN_BLOCKS)
stiffness_batch_kernel(const double *__restrict__ coords, const double *__restrict__ coeff, int64_t n,
                       double *__restrict__ out, unsigned long long *__restrict__ fail_min) {
    extern __shared__ __align__(16) unsigned char s_dyn[];
    GpWarpSmem *s_warp = reinterpret_cast<GpWarpSmem *>(s_dyn);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int el = lane >> 3, gp = lane & 7;
    GpWarpSmem &sm = s_warp[warp];
    const int64_t e = (int64_t)blockIdx.x * GP_EL_PER_BLOCK + warp * GP_EL_PER_WARP + el;
    const bool valid = e < n;
    double x[3];
#pragma unroll
    for (int d = 0; d < 3; ++d)
        x[d] = valid ? __ldg(coords + 24 * e + 3 * gp + d)
                     : (double)((d == 0 ? nat_r(gp) : d == 1 ? nat_s(gp) : nat_t(gp)) > 0);
    const unsigned in_range =
        __ballot_sync(0xffffffffu, coord_in_range(x[0]) && coord_in_range(x[1]) && coord_in_range(x[2]));
    const bool fast_div = ((in_range >> (8 * el)) & 0xffu) == 0xffu;
    publish_node<MODE>(sm, el, gp, 0, x[0], x[1], x[2], valid ? __ldg(coeff + e) : 1.0);
    __syncwarp();
    bool ok;
    if constexpr (MODE == HX_MODE_EXACT)
        ok = ke_gauss_point<false>(sm, el, gp, fast_div, e, valid, out, nullptr, nullptr, 0u);
    else
        ok = ke_gauss_point_fast<false>(sm, el, gp, e, valid, out, nullptr, nullptr, 0u);
    if (valid && !ok) atomicMin(fail_min, HX_FAIL_DEGENERATE_KEY | (unsigned long long)e);
}

// Resolve the lowest failing element into the hx_fail_info record (element.py:237-244).
__global__ void fail_resolve_mesh_kernel(const double *__restrict__ coords, int64_t n_nodes,
                                         const int32_t *__restrict__ conn, hx_fail_info *fail) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const unsigned long long key = *reinterpret_cast<unsigned long long *>(fail);
    if (key == ~0ull) {
        fail->element = -1;
        fail->gauss_point = -1;
        fail->det = 0.0;
        return;
    }
    int32_t g[8];
    if (!(key & HX_FAIL_DEGENERATE_KEY)) {  // lowest element with a node id outside [0, n_nodes)
        const int64_t e = (int64_t)key;
        load_conn(conn, e, g);
        int a = 0;
        while (a < 7 && g[a] >= 0 && g[a] < n_nodes) ++a;
        fail->element = e;
        fail->gauss_point = HX_FAIL_BAD_NODE;
        fail->det = (double)g[a];  // the offending node id
        return;
    }
    const int64_t e = (int64_t)(key & ~HX_FAIL_DEGENERATE_KEY);
    load_conn(conn, e, g);
    double x[8][3];
    for (int a = 0; a < 8; ++a) load_node(coords, g[a], x[a]);
    fail_detail(x, e, fail);
}

__global__ void fail_resolve_batch_kernel(const double *__restrict__ coords, hx_fail_info *fail) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const unsigned long long key = *reinterpret_cast<unsigned long long *>(fail);
    if (key == ~0ull) {
        fail->element = -1;
        fail->gauss_point = -1;
        fail->det = 0.0;
        return;
    }
    const int64_t e = (int64_t)(key & ~HX_FAIL_DEGENERATE_KEY);
    double x[8][3];
    for (int a = 0; a < 8; ++a)
        for (int d = 0; d < 3; ++d) x[a][d] = coords[24 * e + 3 * a + d];
    fail_detail(x, e, fail);
}

// connectivity_index_arrays alone (assemble.py:86-93).
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

// map_local_to_global for dofxn >= 1 (assemble.py:65-83), element-major over a range: local dof
// i = a * dofxn + k of node a is global dof g[a] * dofxn + k (node-major blocks); element e's
// (8 dofxn)(8 dofxn + 1)/2 pairs follow np.tril_indices(8 dofxn) (row-major lower triangle,
// li >= lj) and are swapped to (max, min).  dofxn = 1 is connectivity_index_arrays.
__global__ void dof_index_kernel(const int32_t *__restrict__ conn, int64_t lo, int64_t n, int32_t dofxn,
                                 int32_t *__restrict__ rows, int32_t *__restrict__ cols) {
    const int64_t P = (int64_t)(8 * dofxn) * (8 * dofxn + 1) / 2;
    const int64_t total = P * n;
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < total;
         w += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = w / P;
        const int p = (int)(w - k * P);
        // row li of the packed lower triangle: li (li + 1) / 2 <= p < (li + 1)(li + 2) / 2
        int li = (int)((sqrt(8.0 * p + 1.0) - 1.0) * 0.5);
        while (li * (li + 1) / 2 > p) --li;
        while ((li + 1) * (li + 2) / 2 <= p) ++li;
        const int lj = p - li * (li + 1) / 2;
        const int32_t *c = conn + 8 * (lo + k);
        const int32_t gi = __ldg(c + li / dofxn) * dofxn + li % dofxn;
        const int32_t gj = __ldg(c + lj / dofxn) * dofxn + lj % dofxn;
        rows[w] = max(gi, gj);
        cols[w] = min(gi, gj);
    }
}

constexpr size_t GP_SMEM = GP_WARPS * sizeof(GpWarpSmem);  // dynamic shared memory per block

// Opt the integration kernels into dynamic shared memory beyond the default (once per device).
template <int MODE>
static void configure_mode() {
    cudaFuncSetAttribute(integrate_mesh_kernel<MODE, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)GP_SMEM);
    cudaFuncSetAttribute(integrate_mesh_kernel<MODE, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)GP_SMEM);
    cudaFuncSetAttribute(integrate_mesh_kernel<MODE, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)GP_SMEM);
    cudaFuncSetAttribute(integrate_mesh_kernel<MODE, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)GP_SMEM);
    cudaFuncSetAttribute(stiffness_batch_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GP_SMEM);
}
static void configure_ke_kernels() {
    static bool done[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && done[dev]) return;
    configure_mode<HX_MODE_EXACT>();
    configure_mode<HX_MODE_FAST>();
    if (dev < 64) done[dev] = true;
}

// Resident blocks of the persistent integration kernel on the current device (queried once per mode).
template <int MODE>
static int64_t persistent_blocks() {
    static int64_t cached = 0;
    configure_ke_kernels();
    if (cached == 0) {
        int dev = 0, sms = 148, per_sm = HX_KE_MIN_BLOCKS;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, integrate_mesh_kernel<MODE, true, false>, GP_BLOCK, GP_SMEM);
        if (const char *env = getenv("HX_KE_BLOCKS_PER_SM")) per_sm = std::min(per_sm, atoi(env));  // experiments
        cached = (int64_t)sms * std::max(per_sm, 1);
    }
    return cached;
}

template <int MODE>
static void launch_integrate(int64_t blocks, cudaStream_t s, const double *coords, int64_t n_nodes, const int32_t *conn,
                             const double *coeff, int64_t lo, int64_t n, double *ke, int32_t *rows, int32_t *cols,
                             hx_fail_info *fail, AdjOut adj) {
    unsigned *counter = reinterpret_cast<unsigned *>(&fail->reserved);
    auto *fmin = reinterpret_cast<unsigned long long *>(fail);
    auto go = [&](auto kernel) {
        kernel<<<(unsigned)blocks, GP_BLOCK, GP_SMEM, s>>>(coords, n_nodes, conn, coeff, lo, n, ke, rows, cols, fmin,
                                                           counter, adj);
    };
    if (adj.adj != nullptr) {
        if (rows != nullptr) go(integrate_mesh_kernel<MODE, true, true>);
        else go(integrate_mesh_kernel<MODE, false, true>);
    } else {
        if (rows != nullptr) go(integrate_mesh_kernel<MODE, true, false>);
        else go(integrate_mesh_kernel<MODE, false, false>);
    }
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

// Self-test of div_exact against __ddiv_rn over the operand range the kernel guarantees
// (|a| = 0 or in [2^-420, 2^260], b in [2^-600, 2^330]): random mantissas, signed zeros,
// cancellation-like small integers, exact multiples and their ulp neighbours (the hardest rounding
// cases).  Counts mismatching bit patterns.
__global__ void division_selftest_kernel(uint64_t n, uint64_t seed, unsigned long long *mismatches,
                                         unsigned long long *tested) {
    unsigned long long bad = 0, cnt = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r1 = splitmix64(seed ^ (2 * i)), r2 = splitmix64(seed ^ (2 * i + 1));
        const int kind = (int)(r1 & 3);
        const int ea = (int)((r1 >> 2) % 681) - 420, eb = (int)((r2 >> 2) % 931) - 600;
        double b = __hiloint2double(0x3ff00000 | (int)((r2 >> 12) & 0xfffff), (int)(r2 >> 32));
        b = ldexp(b, kind == 0 ? eb : (eb & 63) - 32);
        double a = __hiloint2double(0x3ff00000 | (int)((r1 >> 12) & 0xfffff), (int)(r1 >> 32));
        a = ldexp(a, kind == 0 ? ea : (ea & 63) - 32);
        if (kind == 2) {  // a = exact-ish multiple of b, nudged by a few ulps
            const double q = __hiloint2double(0x3ff00000 | (int)((r2 >> 40) & 0xfffff), (int)r1);
            a = __dmul_rn(q, b);
            const long long bits = __double_as_longlong(a) + (long long)((r2 >> 60) & 7) - 3;
            a = __longlong_as_double(bits);
        } else if (kind == 3) {  // small-integer ratios (cancellation zeros and halves)
            a = (double)((long long)(r1 >> 40) % 97 - 48);
            b = (double)((r2 >> 40) % 13 + 1);
        }
        if (r1 & (1ull << 62)) a = -a;
        const double y = __drcp_rn(b);
        const double q = div_exact(a, b, y), ref = __ddiv_rn(a, b);
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

static int integrate_mesh_impl(const double *coords, int64_t n_nodes, const int32_t *conn, const double *coeff,
                               int64_t lo, int64_t hi, double *ke, int32_t *rows, int32_t *cols, int32_t mode,
                               hx_fail_info *fail, AdjOut adj, cudaStream_t s) {
    const int64_t n = hi - lo;
    HX_TRY_CUDA(cudaMemsetAsync(fail, 0xff, sizeof(unsigned long long), s));
    HX_TRY_CUDA(cudaMemsetAsync(&fail->reserved, 0, sizeof(int32_t), s));  // quad counter
    if (n > 0) {
        if (n > (int64_t)UINT32_MAX * GP_EL_PER_WARP / 2) {
            set_last_error("hx_integrate_mesh: %lld elements exceed one launch", (long long)n);
            return HX_ERR_CONFIG;
        }
        if (mode == HX_MODE_EXACT)
            launch_integrate<HX_MODE_EXACT>(std::min<int64_t>(ceil_div(n, GP_EL_PER_BLOCK), persistent_blocks<HX_MODE_EXACT>()),
                                            s, coords, n_nodes, conn, coeff, lo, n, ke, rows, cols, fail, adj);
        else
            launch_integrate<HX_MODE_FAST>(std::min<int64_t>(ceil_div(n, GP_EL_PER_BLOCK), persistent_blocks<HX_MODE_FAST>()),
                                           s, coords, n_nodes, conn, coeff, lo, n, ke, rows, cols, fail, adj);
        HX_CHECK_LAUNCH("integrate_mesh_kernel");
    }
    fail_resolve_mesh_kernel<<<1, 1, 0, s>>>(coords, n_nodes, conn, fail);
    HX_CHECK_LAUNCH("fail_resolve_mesh_kernel");
    return HX_OK;
}

namespace hx {
// The fail-record epilogue of an integration launch (also used by hx_integrate_emit).
int integrate_fail_resolve(const double *coords, int64_t n_nodes, const int32_t *conn, hx_fail_info *fail,
                           cudaStream_t s) {
    fail_resolve_mesh_kernel<<<1, 1, 0, s>>>(coords, n_nodes, conn, fail);
    HX_CHECK_LAUNCH("fail_resolve_mesh_kernel");
    return HX_OK;
}
}  // namespace hx

static bool integrate_args_ok(int64_t lo, int64_t hi, const double *ke, const int32_t *rows, const int32_t *cols,
                              const hx_fail_info *fail, int32_t mode, int &rc) {
    if (lo < 0 || hi < lo || (hi > lo && ke == nullptr) || fail == nullptr || (rows == nullptr) != (cols == nullptr)) {
        set_last_error("hx_integrate_mesh: bad arguments (lo=%lld hi=%lld)", (long long)lo, (long long)hi);
        rc = HX_ERR_VALUE;
        return false;
    }
    if (mode != HX_MODE_EXACT && mode != HX_MODE_FAST) {
        set_last_error("hx_integrate_mesh: unknown mode %d", mode);
        rc = HX_ERR_CONFIG;
        return false;
    }
    return true;
}

extern "C" int hx_integrate_mesh(const double *coords, int64_t n_nodes, const int32_t *conn,
                                 const double *coeff, int64_t lo, int64_t hi, double *ke,
                                 int32_t *rows, int32_t *cols, int32_t mode, hx_fail_info *fail,
                                 void *stream) {
    int rc = HX_OK;
    if (!integrate_args_ok(lo, hi, ke, rows, cols, fail, mode, rc)) return rc;
    return integrate_mesh_impl(coords, n_nodes, conn, coeff, lo, hi, ke, rows, cols, mode, fail,
                               AdjOut{nullptr, nullptr}, (cudaStream_t)stream);
}

extern "C" int hx_integrate_mesh_adjacency(const double *coords, int64_t n_nodes, const int32_t *conn,
                                           const double *coeff, int64_t lo, int64_t hi, double *ke, int32_t *rows,
                                           int32_t *cols, int32_t mode, hx_fail_info *fail, void *csc_workspace,
                                           int64_t workspace_bytes, uint32_t *csc_status, int32_t reset,
                                           void *stream) {
    int rc = HX_OK;
    if (!integrate_args_ok(lo, hi, ke, rows, cols, fail, mode, rc)) return rc;
    if (csc_status == nullptr || n_nodes < 0 || n_nodes >= INT32_MAX || 8 * hi >= (int64_t)INT32_MAX) {
        set_last_error("hx_integrate_mesh_adjacency: bad arguments (n_nodes=%lld hi=%lld)", (long long)n_nodes,
                       (long long)hi);
        return HX_ERR_VALUE;
    }
    AdjOut adj{nullptr, csc_status};
    int32_t *deg = nullptr;
    rc = mesh_ws_adjacency(csc_workspace, workspace_bytes, n_nodes, &deg, &adj.adj);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    if (reset) {  // status 0, every adjacency slot empty (-1)
        HX_TRY_CUDA(cudaMemsetAsync(csc_status, 0, sizeof(uint32_t), s));
        if (n_nodes > 0) HX_TRY_CUDA(cudaMemsetAsync(adj.adj, 0xff, sizeof(int32_t) * 8 * n_nodes, s));
    }
    return integrate_mesh_impl(coords, n_nodes, conn, coeff, lo, hi, ke, rows, cols, mode, fail, adj, s);
}

extern "C" int hx_stiffness_batch(const double *coords, const double *coeff, int64_t n, double *out,
                                  int32_t mode, hx_fail_info *fail, void *stream) {
    if (n < 0 || (n > 0 && out == nullptr) || fail == nullptr) {
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
        const int64_t blocks = ceil_div(n, GP_EL_PER_BLOCK);
        configure_ke_kernels();
        if (mode == HX_MODE_EXACT)
            stiffness_batch_kernel<HX_MODE_EXACT><<<(unsigned)blocks, GP_BLOCK, GP_SMEM, s>>>(
                coords, coeff, n, out, reinterpret_cast<unsigned long long *>(fail));
        else
            stiffness_batch_kernel<HX_MODE_FAST><<<(unsigned)blocks, GP_BLOCK, GP_SMEM, s>>>(
                coords, coeff, n, out, reinterpret_cast<unsigned long long *>(fail));
        HX_CHECK_LAUNCH("stiffness_batch_kernel");
    }
    fail_resolve_batch_kernel<<<1, 1, 0, s>>>(coords, fail);
    HX_CHECK_LAUNCH("fail_resolve_batch_kernel");
    return HX_OK;
}

extern "C" int hx_connectivity_index_arrays(const int32_t *conn, int64_t lo, int64_t hi, int32_t *rows,
                                            int32_t *cols, void *stream) {
    if (lo < 0 || hi < lo || (hi > lo && (rows == nullptr || cols == nullptr))) {
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

extern "C" int hx_dof_index_arrays(const int32_t *conn, int64_t lo, int64_t hi, int64_t n_nodes, int32_t dofxn,
                                   int32_t *rows, int32_t *cols, void *stream) {
    if (lo < 0 || hi < lo || dofxn < 1 || dofxn > HX_MAX_DOFXN || (hi > lo && (rows == nullptr || cols == nullptr))) {
        set_last_error("hx_dof_index_arrays: bad arguments (dofxn must be in [1, %d])", HX_MAX_DOFXN);
        return HX_ERR_VALUE;
    }
    if (n_nodes * (int64_t)dofxn > INT32_MAX) {
        set_last_error("hx_dof_index_arrays: %lld nodes x %d dofs exceed the int32 index range",
                       (long long)n_nodes, dofxn);
        return HX_ERR_VALUE;
    }
    const int64_t n = hi - lo;
    if (n == 0) return HX_OK;
    const int64_t P = (int64_t)(8 * dofxn) * (8 * dofxn + 1) / 2;
    const int threads = 256;
    const int64_t blocks = std::min<int64_t>(ceil_div(P * n, threads), 148 * 16);
    dof_index_kernel<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(conn, lo, n, dofxn, rows, cols);
    HX_CHECK_LAUNCH("dof_index_kernel");
    return HX_OK;
}
