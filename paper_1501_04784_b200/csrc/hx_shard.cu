// hx_shard.cu -- multi-GPU element-halo exchange plan (element-range shards, column blocks).
//
// Rank r owns elements [E_r, E_r+1) (it integrates them) and lower-CSC columns
// [C_r, C_r+1).  An owned element must also reach every other rank whose column block holds one
// of its nodes (each node's column receives that element's contributions).  This file builds the
// send buffer of one all-to-all: records of 40 doubles per (element, destination) -- the 36
// packed KE values followed by the 8 int32 node ids -- grouped destination-major and, within a
// destination, in ascending element order (a stable multi-split), so that the receiver's
// [lower ranks | own | higher ranks] element segments are in ascending global element order and
// duplicate positions are summed in exactly the single-GPU order.
//
//   pass 1  tile_counts[d][tile]  per-destination counts of a tile (warp ballots)
//   scan    exclusive scan over the destination-major (d, tile) table (CUB)
//   pass 2  each tile writes its records at offset(d, tile) + intra-tile rank (ballots again)
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <cstring>

#include "hx_common.cuh"

namespace hx {

constexpr int SHARD_TILE = 256;  // elements per tile (one block of 256 threads)
constexpr int MAX_WORLD = 32;

__device__ __forceinline__ int owner_of(int32_t node, const int64_t *__restrict__ bounds, int world) {
    int lo = 0, hi = world;  // largest r with bounds[r] <= node
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (bounds[mid] <= node) lo = mid; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ uint32_t dest_mask(const int32_t *__restrict__ conn, int64_t e,
                                              const int64_t *__restrict__ bounds, int world, int self) {
    const int4 *c4 = reinterpret_cast<const int4 *>(conn) + 2 * e;
    const int4 lo = __ldg(c4), hi = __ldg(c4 + 1);
    const int32_t g[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    uint32_t m = 0;
#pragma unroll
    for (int a = 0; a < 8; ++a) m |= 1u << owner_of(g[a], bounds, world);
    return m & ~(1u << self);
}

// per-(destination, tile) counts; table is destination-major: counts[d * n_tiles + tile]
__global__ void __launch_bounds__(SHARD_TILE)
halo_count_kernel(const int32_t *__restrict__ conn, int64_t n_el, const int64_t *__restrict__ bounds, int world,
                  int self, int64_t n_tiles, int64_t *__restrict__ counts) {
    __shared__ int32_t s_cnt[MAX_WORLD];
    const int t = threadIdx.x;
    if (t < MAX_WORLD) s_cnt[t] = 0;
    __syncthreads();
    const int64_t e = (int64_t)blockIdx.x * SHARD_TILE + t;
    const uint32_t m = e < n_el ? dest_mask(conn, e, bounds, world, self) : 0u;
    const int lane = t & 31;
    for (int d = 0; d < world; ++d) {
        const uint32_t ballot = __ballot_sync(0xffffffffu, (m >> d) & 1u);
        if (lane == 0 && ballot) atomicAdd(&s_cnt[d], __popc(ballot));
    }
    __syncthreads();
    if (t < world) counts[(int64_t)t * n_tiles + blockIdx.x] = s_cnt[t];
}

__global__ void __launch_bounds__(SHARD_TILE)
halo_pack_kernel(const int32_t *__restrict__ conn, const double *__restrict__ ke, int64_t n_el,
                 const int64_t *__restrict__ bounds, int world, int self, int64_t n_tiles,
                 const int64_t *__restrict__ offsets, double *__restrict__ records) {
    __shared__ int32_t s_warp[MAX_WORLD][SHARD_TILE / 32];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int64_t e = (int64_t)blockIdx.x * SHARD_TILE + t;
    const uint32_t m = e < n_el ? dest_mask(conn, e, bounds, world, self) : 0u;
    uint32_t ballots[MAX_WORLD];
    for (int d = 0; d < world; ++d) {
        ballots[d] = __ballot_sync(0xffffffffu, (m >> d) & 1u);
        if (lane == 0) s_warp[d][warp] = __popc(ballots[d]);
    }
    __syncthreads();
    for (int d = 0; d < world; ++d) {
        if (!((m >> d) & 1u)) continue;
        int before = 0;
        for (int w = 0; w < warp; ++w) before += s_warp[d][w];
        before += __popc(ballots[d] & ((1u << lane) - 1u));
        const int64_t slot = offsets[(int64_t)d * n_tiles + blockIdx.x] + before;
        double *dst = records + 40 * slot;
        const double *src = ke + 36 * e;
#pragma unroll
        for (int p = 0; p < 36; ++p) dst[p] = src[p];
        const int4 *c4 = reinterpret_cast<const int4 *>(conn) + 2 * e;
        int4 *d4 = reinterpret_cast<int4 *>(dst + 36);
        d4[0] = __ldg(c4);
        d4[1] = __ldg(c4 + 1);
    }
}

__global__ void halo_totals_kernel(const int64_t *__restrict__ offsets, const int64_t *__restrict__ counts,
                                   int world, int64_t n_tiles, int64_t *__restrict__ per_dest) {
    const int d = threadIdx.x;
    if (d < world) {
        const int64_t first = offsets[(int64_t)d * n_tiles];
        const int64_t last = offsets[(int64_t)d * n_tiles + n_tiles - 1] + counts[(int64_t)d * n_tiles + n_tiles - 1];
        per_dest[d] = last - first;
    }
}

// Fused pack-and-send (the dispatch of the all-to-all done by the producer over NVLink): each warp
// takes its 32 elements one destination at a time, and the warp's records for that destination --
// contiguous at the receiver -- are written cooperatively with coalesced 8-byte stores straight into
// the destination rank's receive buffer (a peer pointer opened from its IPC handle, or a local
// buffer in the loopback).  The receiver's buffer layout is the one the NCCL all-to-all produces:
// source ranks in ascending order, ascending element order within each source.
__global__ void __launch_bounds__(SHARD_TILE)
halo_send_kernel(const int32_t *__restrict__ conn, const double *__restrict__ ke, int64_t n_el,
                 const int64_t *__restrict__ bounds, int world, int self, int64_t n_tiles,
                 const int64_t *__restrict__ offsets, double *const *__restrict__ dest_ptrs,
                 const int64_t *__restrict__ dest_offsets) {
    __shared__ int32_t s_warp[MAX_WORLD][SHARD_TILE / 32];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int64_t e = (int64_t)blockIdx.x * SHARD_TILE + t;
    const uint32_t m = e < n_el ? dest_mask(conn, e, bounds, world, self) : 0u;
    uint32_t ballots[MAX_WORLD];
    for (int d = 0; d < world; ++d) {
        ballots[d] = __ballot_sync(0xffffffffu, (m >> d) & 1u);
        if (lane == 0) s_warp[d][warp] = __popc(ballots[d]);
    }
    __syncthreads();
    const int64_t e0 = (int64_t)blockIdx.x * SHARD_TILE + warp * 32;
    for (int d = 0; d < world; ++d) {
        const uint32_t b = ballots[d];
        const int k = __popc(b);
        if (k == 0) continue;
        int before = 0;
        for (int w = 0; w < warp; ++w) before += s_warp[d][w];
        // record slot of this warp's first record for d, in d's receive buffer
        const int64_t slot0 = dest_offsets[d] + (offsets[(int64_t)d * n_tiles + blockIdx.x] - offsets[(int64_t)d * n_tiles]) + before;
        double *dst = dest_ptrs[d] + 40 * slot0;
        for (int f = lane; f < 40 * k; f += 32) {
            const int i = f / 40, word = f - 40 * i;
            const int64_t el = e0 + __fns(b, 0, i + 1);  // the warp's i-th record: (i+1)-th set bit
            double v;
            if (word < 36) {
                v = __ldg(ke + 36 * el + word);
            } else {
                const int2 ids = __ldg(reinterpret_cast<const int2 *>(conn + 8 * el) + (word - 36));
                v = __hiloint2double(ids.y, ids.x);  // bit copy of two int32 node ids
            }
            dst[f] = v;
        }
    }
}

struct ShardWs {
    int64_t *counts, *offsets;
    void *cub_tmp;
    size_t cub_bytes, total;
};

static ShardWs shard_ws_layout(void *base, int64_t n_el, int world) {
    ShardWs w{};
    const int64_t n_tiles = std::max<int64_t>(1, ceil_div(n_el, SHARD_TILE));
    const int64_t n = n_tiles * world;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off = align_up(off + bytes, 256);
        return o;
    };
    const size_t o_c = take(sizeof(int64_t) * n), o_o = take(sizeof(int64_t) * n);
    cub::DeviceScan::ExclusiveSum(nullptr, w.cub_bytes, (int64_t *)nullptr, (int64_t *)nullptr, (int)n);
    const size_t o_t = take(w.cub_bytes);
    w.total = off;
    if (base) {
        char *b = (char *)base;
        w.counts = (int64_t *)(b + o_c);
        w.offsets = (int64_t *)(b + o_o);
        w.cub_tmp = b + o_t;
    }
    return w;
}

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

extern "C" int64_t hx_halo_workspace_bytes(int64_t n_el, int32_t world) {
    if (n_el < 0 || world < 1 || world > MAX_WORLD) return -1;
    return (int64_t)shard_ws_layout(nullptr, n_el, world).total;
}

extern "C" int hx_halo_count(const int32_t *conn, int64_t n_el, const int64_t *col_bounds, int32_t world,
                             int32_t self, int64_t *per_dest, void *workspace, int64_t workspace_bytes,
                             void *stream) {
    if (n_el < 0 || world < 1 || world > MAX_WORLD || self < 0 || self >= world || col_bounds == nullptr ||
        per_dest == nullptr) {
        set_last_error("hx_halo_count: bad arguments");
        return HX_ERR_VALUE;
    }
    ShardWs w = shard_ws_layout(workspace, n_el, world);
    if (workspace == nullptr || workspace_bytes < (int64_t)w.total) {
        set_last_error("hx_halo_count: workspace too small");
        return HX_ERR_WORKSPACE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t n_tiles = std::max<int64_t>(1, ceil_div(n_el, SHARD_TILE));
    HX_TRY_CUDA(cudaMemsetAsync(w.counts, 0, sizeof(int64_t) * n_tiles * world, s));
    if (n_el > 0) {
        halo_count_kernel<<<(unsigned)n_tiles, SHARD_TILE, 0, s>>>(conn, n_el, col_bounds, world, self, n_tiles,
                                                                  w.counts);
        HX_CHECK_LAUNCH("halo_count_kernel");
    }
    size_t cb = w.cub_bytes;
    HX_TRY_CUDA(cub::DeviceScan::ExclusiveSum(w.cub_tmp, cb, w.counts, w.offsets, (int)(n_tiles * world), s));
    halo_totals_kernel<<<1, MAX_WORLD, 0, s>>>(w.offsets, w.counts, world, n_tiles, per_dest);
    HX_CHECK_LAUNCH("halo_totals_kernel");
    return HX_OK;
}

extern "C" int hx_halo_send(const int32_t *conn, const double *ke, int64_t n_el, const int64_t *col_bounds,
                            int32_t world, int32_t self, double *const *dest_ptrs, const int64_t *dest_offsets,
                            const void *workspace, void *stream) {
    if (n_el < 0 || world < 1 || world > MAX_WORLD || workspace == nullptr || dest_ptrs == nullptr ||
        dest_offsets == nullptr) {
        set_last_error("hx_halo_send: bad arguments");
        return HX_ERR_VALUE;
    }
    if (n_el == 0) return HX_OK;
    ShardWs w = shard_ws_layout(const_cast<void *>(workspace), n_el, world);
    const int64_t n_tiles = ceil_div(n_el, SHARD_TILE);
    halo_send_kernel<<<(unsigned)n_tiles, SHARD_TILE, 0, (cudaStream_t)stream>>>(
        conn, ke, n_el, col_bounds, world, self, n_tiles, w.offsets, dest_ptrs, dest_offsets);
    HX_CHECK_LAUNCH("halo_send_kernel");
    return HX_OK;
}

extern "C" int hx_halo_pack(const int32_t *conn, const double *ke, int64_t n_el, const int64_t *col_bounds,
                            int32_t world, int32_t self, double *records, const void *workspace, void *stream) {
    if (n_el < 0 || world < 1 || world > MAX_WORLD || workspace == nullptr || (n_el > 0 && records == nullptr)) {
        set_last_error("hx_halo_pack: bad arguments");
        return HX_ERR_VALUE;
    }
    if (n_el == 0) return HX_OK;
    ShardWs w = shard_ws_layout(const_cast<void *>(workspace), n_el, world);
    const int64_t n_tiles = ceil_div(n_el, SHARD_TILE);
    halo_pack_kernel<<<(unsigned)n_tiles, SHARD_TILE, 0, (cudaStream_t)stream>>>(
        conn, ke, n_el, col_bounds, world, self, n_tiles, w.offsets, records);
    HX_CHECK_LAUNCH("halo_pack_kernel");
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
