// hx_shard.cu -- column blocks of one GPU (the out-of-core build: elements touching a column
// block, selected in ascending order) and the structured mesh producer on the device.
#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <cstring>

#include "hx_common.cuh"

namespace hx {

// ---- column-block element selection (out-of-core build: one column block at a time) ----------
// Element e belongs to block [col_lo, col_hi) when one of its nodes does; the selection keeps
// ascending element order (a stable compaction), so the block's single segment sums duplicates in
// the global element order.
struct TouchesBlock {
    const int32_t *conn;
    int64_t lo, hi;
    __device__ __forceinline__ bool operator()(const int64_t &e) const {
        const int4 *c4 = reinterpret_cast<const int4 *>(conn) + 2 * e;
        const int4 a = __ldg(c4), b = __ldg(c4 + 1);
        const int32_t g[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        bool in = false;
#pragma unroll
        for (int k = 0; k < 8; ++k) in |= g[k] >= lo && g[k] < hi;
        return in;
    }
};

__global__ void block_gather_kernel(const int32_t *__restrict__ conn, const double *__restrict__ coeff,
                                    const int64_t *__restrict__ ids, const int64_t *__restrict__ count,
                                    int32_t *__restrict__ conn_out, double *__restrict__ coeff_out) {
    const int64_t n = *count;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = ids[i];
        const int4 *src = reinterpret_cast<const int4 *>(conn) + 2 * e;
        int4 *dst = reinterpret_cast<int4 *>(conn_out) + 2 * i;
        dst[0] = __ldg(src);
        dst[1] = __ldg(src + 1);
        coeff_out[i] = __ldg(coeff + e);
    }
}

// Check of a sampled streaming plan (hx_block_ranges_sampled) on the device: every element of block
// k's uploaded range (global ids e0 + i) must lie inside the predicted element range of every column
// block its node span covers, and its nodes below the block's coordinate prefix -- else *flag != 0 and
// the caller rebuilds with the exact host scan.  bounds (K + 1), e_lo / e_hi (K) device int64.
__global__ void block_verify_kernel(const int32_t *__restrict__ conn, int64_t n, int64_t e0, int64_t n_nodes,
                                    const int64_t *__restrict__ bounds, int K, const int64_t *__restrict__ e_lo,
                                    const int64_t *__restrict__ e_hi, int64_t node_top,
                                    unsigned *__restrict__ flag) {
    unsigned bad = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int4 *c4 = reinterpret_cast<const int4 *>(conn + 8 * i);
        const int4 lo = __ldg(c4), hi = __ldg(c4 + 1);
        const int mn = min(min(min(lo.x, lo.y), min(lo.z, lo.w)), min(min(hi.x, hi.y), min(hi.z, hi.w)));
        const int mx = max(max(max(lo.x, lo.y), max(lo.z, lo.w)), max(max(hi.x, hi.y), max(hi.z, hi.w)));
        if ((int64_t)mx >= node_top && (int64_t)mx < n_nodes) bad |= 2u;  // a coordinate not uploaded yet
        int b0 = 0, b1 = 0;  // blocks of mn / mx, clamped like hx_block_ranges
        for (int b = 1; b < K; ++b) {
            b0 += (int64_t)mn >= __ldg(bounds + b);
            b1 += (int64_t)mx >= __ldg(bounds + b);
        }
        const int64_t e = e0 + i;
        for (int b = b0; b <= b1; ++b)
            if (e < __ldg(e_lo + b) || e >= __ldg(e_hi + b)) bad |= 1u;
    }
    if (bad) atomicOr(flag, bad);
}

}  // namespace hx

using namespace hx;

extern "C" int64_t hx_block_select_workspace_bytes(int64_t n_el) {
    if (n_el < 0 || n_el > INT32_MAX) return -1;
    size_t b = 0;
    cub::DeviceSelect::If(nullptr, b, thrust::counting_iterator<int64_t>(0), (int64_t *)nullptr, (int64_t *)nullptr,
                          (int)std::max<int64_t>(n_el, 1), TouchesBlock{nullptr, 0, 0});
    return (int64_t)b;
}

extern "C" int hx_block_select(const int32_t *conn, int64_t n_el, int64_t col_lo, int64_t col_hi, int64_t *ids,
                               int64_t *count, void *workspace, int64_t workspace_bytes, void *stream) {
    if (n_el < 0 || n_el > INT32_MAX || col_lo < 0 || col_hi < col_lo || ids == nullptr || count == nullptr ||
        (n_el > 0 && conn == nullptr)) {
        set_last_error("hx_block_select: bad arguments");
        return HX_ERR_VALUE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    if (n_el == 0) {
        HX_TRY_CUDA(cudaMemsetAsync(count, 0, sizeof(int64_t), s));
        return HX_OK;
    }
    size_t b = (size_t)workspace_bytes;
    if (workspace == nullptr || workspace_bytes < hx_block_select_workspace_bytes(n_el)) {
        set_last_error("hx_block_select: workspace too small");
        return HX_ERR_WORKSPACE;
    }
    HX_TRY_CUDA(cub::DeviceSelect::If(workspace, b, thrust::counting_iterator<int64_t>(0), ids, count, (int)n_el,
                                      TouchesBlock{conn, col_lo, col_hi}, s));
    return HX_OK;
}

extern "C" int hx_block_gather(const int32_t *conn, const double *coeff, const int64_t *ids, const int64_t *count,
                               int64_t capacity, int32_t *conn_out, double *coeff_out, void *stream) {
    if (conn == nullptr || coeff == nullptr || ids == nullptr || count == nullptr || capacity < 0 ||
        (capacity > 0 && (conn_out == nullptr || coeff_out == nullptr))) {
        set_last_error("hx_block_gather: bad arguments");
        return HX_ERR_VALUE;
    }
    if (capacity == 0) return HX_OK;
    block_gather_kernel<<<(unsigned)std::min<int64_t>(ceil_div(capacity, 256), 148 * 16), 256, 0,
                          (cudaStream_t)stream>>>(conn, coeff, ids, count, conn_out, coeff_out);
    HX_CHECK_LAUNCH("block_gather_kernel");
    return HX_OK;
}

// ---- structured box on the device (mesh.py:73-98: the mesh producer before the path) ------------
namespace hx {
__global__ void cube_nodes_kernel(int64_t sx, int64_t sy, int64_t n_nodes, double h, double *__restrict__ coords) {
    for (int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; id < n_nodes;
         id += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = id % sx, j = (id / sx) % sy, k = id / (sx * sy);
        coords[3 * id] = __dmul_rn((double)i, h);  // node (i, j, k) at (i h, j h, k h)
        coords[3 * id + 1] = __dmul_rn((double)j, h);
        coords[3 * id + 2] = __dmul_rn((double)k, h);
    }
}

__global__ void cube_elements_kernel(int64_t nx, int64_t ny, int64_t n_el, double c0, int32_t *__restrict__ conn,
                                     double *__restrict__ coeff) {
    const int64_t sx = nx + 1, layer = sx * (ny + 1);
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n_el; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t ex = e % nx, ey = (e / nx) % ny, ez = e / (nx * ny);  // x-fastest element numbering
        const int32_t o = (int32_t)(ex + ey * sx + ez * layer);
        const int32_t s = (int32_t)sx, l = (int32_t)layer;
        int4 *dst = reinterpret_cast<int4 *>(conn) + 2 * e;
        dst[0] = make_int4(o, o + 1, o + 1 + s, o + s);               // ccw bottom face
        dst[1] = make_int4(o + l, o + 1 + l, o + 1 + s + l, o + s + l);  // ccw top face
        coeff[e] = c0;
    }
}
}  // namespace hx

extern "C" int hx_generate_cube_mesh(int64_t nx, int64_t ny, int64_t nz, double h, double c0, double *coords,
                                     int32_t *conn, double *coeff, void *stream) {
    if (nx < 1 || ny < 1 || nz < 1 || !(h > 0.0) || !(c0 > 0.0) || coords == nullptr || conn == nullptr ||
        coeff == nullptr) {
        set_last_error("hx_generate_cube_mesh: bad arguments");
        return HX_ERR_VALUE;
    }
    const int64_t n_nodes = (nx + 1) * (ny + 1) * (nz + 1), n_el = nx * ny * nz;
    if (n_nodes >= INT32_MAX) {
        set_last_error("hx_generate_cube_mesh: %lld nodes exceed int32 ids", (long long)n_nodes);
        return HX_ERR_CONFIG;
    }
    cudaStream_t s = (cudaStream_t)stream;
    cube_nodes_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n_nodes, 256), 148 * 32), 256, 0, s>>>(nx + 1, ny + 1,
                                                                                                  n_nodes, h, coords);
    HX_CHECK_LAUNCH("cube_nodes_kernel");
    cube_elements_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n_el, 256), 148 * 32), 256, 0, s>>>(nx, ny, n_el, c0,
                                                                                                  conn, coeff);
    HX_CHECK_LAUNCH("cube_elements_kernel");
    return HX_OK;
}

extern "C" int hx_block_verify(const int32_t *conn, int64_t n, int64_t e0, int64_t n_nodes, const int64_t *bounds,
                               int32_t n_blocks, const int64_t *e_lo, const int64_t *e_hi, int64_t node_top,
                               uint32_t *flag, void *stream) {
    if (n < 0 || n_blocks < 1 || bounds == nullptr || e_lo == nullptr || e_hi == nullptr || flag == nullptr ||
        (n > 0 && conn == nullptr)) {
        set_last_error("hx_block_verify: bad arguments");
        return HX_ERR_VALUE;
    }
    if (n == 0) return HX_OK;
    const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(n, 256), 148 * 8);
    block_verify_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(conn, n, e0, n_nodes, bounds, n_blocks, e_lo, e_hi,
                                                                  node_top, flag);
    HX_CHECK_LAUNCH("block_verify_kernel");
    return HX_OK;
}
