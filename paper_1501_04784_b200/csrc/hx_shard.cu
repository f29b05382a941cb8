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

#include <algorithm>

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

}  // namespace hx

using namespace hx;

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
