// hx_triplet.cu -- generic triplet -> lower-triangular CSC (assemble.py:110-149) for arbitrary
// (row, col, val) triplets, e.g. imported matrices or meshes outside the node-adjacency fast
// path's limits.
//
//   symbolic: validate (_check_indices, assemble.py:143-149) -> pack (col, row) into one key of
//             2*ceil(log2 dim) bits -> stable LSD radix sort of (key, original index) (CUB; the
//             stable order reproduces np.lexsort((rows, cols)), assemble.py:125) -> run starts
//             (assemble.py:130-133) -> row_idx and col_ptr (assemble.py:136-139).
//   numeric:  one thread per run, gathering the run's values in stable order and reducing
//             them with numpy add.reduceat's exact rule out = v0 + pairwise(v[1:]) (numpy's
//             pairwise summation: sequential below 8 terms, 8 accumulators up to 128,
//             recursive halving above), so the result is bitwise np.add.reduceat
//             (assemble.py:135) for any run length.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include <algorithm>

#include "hx_common.cuh"

namespace hx {

__global__ void triplet_keys_kernel(const int32_t *__restrict__ rows, const int32_t *__restrict__ cols, int64_t n,
                                    int64_t dim, int nb, uint64_t *__restrict__ keys, uint32_t *__restrict__ idx,
                                    uint32_t *__restrict__ status) {
    uint32_t st = 0;
    const uint64_t mask = (nb >= 64) ? ~0ull : ((1ull << nb) - 1);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t r = rows[i], c = cols[i];
        if (r < 0 || (int64_t)r >= dim || c < 0) st |= HX_ST_BAD_INDEX;
        else if (r < c) st |= HX_ST_UPPER;
        const uint64_t rr = (uint64_t)(uint32_t)max(r, 0) & mask;
        const uint64_t cc = (uint64_t)(uint32_t)max(c, 0) & mask;
        keys[i] = (cc << nb) | rr;
        idx[i] = (uint32_t)i;
    }
    if (st) atomicOr(status, st);
}

__global__ void run_flags_kernel(const uint64_t *__restrict__ keys, int64_t n, uint8_t *__restrict__ flags) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        flags[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

// row_idx[r], col_ptr (dense over [0, dim]) and the end sentinel of the run table.
__global__ void runs_kernel(const uint64_t *__restrict__ keys, int64_t n, int64_t dim, int nb,
                            int64_t *__restrict__ starts, const int64_t *__restrict__ num_runs_dev,
                            int64_t *__restrict__ row_idx, int64_t *__restrict__ col_ptr) {
    const int64_t nr = *num_runs_dev;
    const uint64_t mask = (1ull << nb) - 1;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nr; r += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t key = keys[starts[r]];
        const int64_t row = (int64_t)(key & mask);
        int64_t col = (int64_t)(key >> nb);
        if (col >= dim) col = dim - 1;  // invalid input (status already flagged): stay in bounds
        row_idx[r] = row;
        int64_t prev = -1;
        if (r > 0) {
            prev = (int64_t)(keys[starts[r - 1]] >> nb);
            if (prev >= dim) prev = dim - 1;
        }
        for (int64_t cc = prev + 1; cc <= col; ++cc) col_ptr[cc] = r;
        if (r == nr - 1) {
            for (int64_t cc = col + 1; cc <= dim; ++cc) col_ptr[cc] = nr;
            starts[nr] = n;
        }
    }
}

// numpy's pairwise summation (loops_utils.h.src @TYPE@_pairwise_sum) over v(i) = vals[idx[off+i]].
__device__ double pairwise_gather(const double *__restrict__ vals, const uint32_t *__restrict__ idx, int64_t off,
                                  int64_t n) {
    if (n < 8) {
        double res = -0.0;
        for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, vals[idx[off + i]]);
        return res;
    }
    if (n <= 128) {
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = vals[idx[off + j]];
        int64_t i = 8;
        for (; i < n - (n % 8); i += 8) {
#pragma unroll
            for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], vals[idx[off + i + j]]);
        }
        double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                               __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; i < n; ++i) res = __dadd_rn(res, vals[idx[off + i]]);
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return __dadd_rn(pairwise_gather(vals, idx, off, n2), pairwise_gather(vals, idx, off + n2, n - n2));
}

__global__ void run_sum_kernel(const double *__restrict__ vals, const uint32_t *__restrict__ idx,
                               const int64_t *__restrict__ starts, const int64_t *__restrict__ num_runs_dev,
                               double *__restrict__ out) {
    const int64_t nr = *num_runs_dev;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nr; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = starts[r], e = starts[r + 1];
        const double v0 = vals[idx[s]];
        out[r] = (e - s == 1) ? v0 : __dadd_rn(v0, pairwise_gather(vals, idx, s + 1, e - s - 1));
    }
}

struct TripletWs {
    uint64_t *keys_in, *keys_out;
    uint32_t *idx_in, *idx_out;
    uint8_t *flags;
    int64_t *starts;
    int64_t *num_runs;
    void *cub_tmp;
    size_t cub_bytes, total;
};

static int key_bits(int64_t dim) {
    int nb = 1;
    while (nb < 62 && (int64_t(1) << nb) < dim) ++nb;
    return nb;
}

static TripletWs triplet_ws_layout(void *base, int64_t n, int64_t dim) {
    TripletWs w{};
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off = align_up(off + bytes, 256);
        return o;
    };
    const int64_t nn = std::max<int64_t>(n, 1);
    const size_t o_ki = take(sizeof(uint64_t) * nn), o_ko = take(sizeof(uint64_t) * nn);
    const size_t o_ii = take(sizeof(uint32_t) * nn), o_io = take(sizeof(uint32_t) * nn);
    const size_t o_fl = take(nn), o_st = take(sizeof(int64_t) * (nn + 1)), o_nr = take(sizeof(int64_t));
    size_t b_sort = 0, b_sel = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b_sort, (uint64_t *)nullptr, (uint64_t *)nullptr,
                                    (uint32_t *)nullptr, (uint32_t *)nullptr, nn, 0, 2 * key_bits(dim));
    cub::DeviceSelect::Flagged(nullptr, b_sel, cub::CountingInputIterator<int64_t>(0), (uint8_t *)nullptr,
                               (int64_t *)nullptr, (int64_t *)nullptr, nn);
    w.cub_bytes = std::max(b_sort, b_sel);
    const size_t o_cub = take(w.cub_bytes);
    w.total = off;
    char *b = (char *)base;
    if (b) {
        w.keys_in = (uint64_t *)(b + o_ki);
        w.keys_out = (uint64_t *)(b + o_ko);
        w.idx_in = (uint32_t *)(b + o_ii);
        w.idx_out = (uint32_t *)(b + o_io);
        w.flags = (uint8_t *)(b + o_fl);
        w.starts = (int64_t *)(b + o_st);
        w.num_runs = (int64_t *)(b + o_nr);
        w.cub_tmp = b + o_cub;
    }
    return w;
}

static unsigned grid_1d(int64_t n, int threads) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, threads), 148 * 32));
}

}  // namespace hx

using namespace hx;

extern "C" int64_t hx_triplet_csc_workspace_bytes(int64_t n, int64_t dim) {
    if (n < 0 || dim < 0 || n >= (int64_t)UINT32_MAX) return -1;
    return (int64_t)triplet_ws_layout(nullptr, n, dim).total;
}

extern "C" int hx_triplet_csc_symbolic(const int32_t *rows, const int32_t *cols, int64_t n, int64_t dim,
                                       int64_t *col_ptr, int64_t *row_idx, void *workspace, int64_t workspace_bytes,
                                       uint32_t *status, void *stream) {
    if (n < 0 || dim < 0 || col_ptr == nullptr || status == nullptr || (n > 0 && (rows == nullptr || cols == nullptr))) {
        set_last_error("hx_triplet_csc_symbolic: bad arguments");
        return HX_ERR_VALUE;
    }
    if (n >= (int64_t)UINT32_MAX) {
        set_last_error("hx_triplet_csc_symbolic: %lld triplets exceed one sort (2^32)", (long long)n);
        return HX_ERR_CONFIG;
    }
    cudaStream_t s = (cudaStream_t)stream;
    TripletWs w = triplet_ws_layout(workspace, n, dim);
    if (workspace == nullptr || workspace_bytes < (int64_t)w.total) {
        set_last_error("hx_triplet_csc_symbolic: workspace %lld < %lld bytes", (long long)workspace_bytes,
                       (long long)w.total);
        return HX_ERR_WORKSPACE;
    }
    HX_TRY_CUDA(cudaMemsetAsync(status, 0, sizeof(uint32_t), s));
    HX_TRY_CUDA(cudaMemsetAsync(w.num_runs, 0, sizeof(int64_t), s));
    if (n == 0 || dim == 0) {  // assemble.py:118-124
        HX_TRY_CUDA(cudaMemsetAsync(col_ptr, 0, sizeof(int64_t) * (dim + 1), s));
        if (n > 0) {  // dim == 0 with entries: every index is out of range
            triplet_keys_kernel<<<grid_1d(n, 256), 256, 0, s>>>(rows, cols, n, dim, 1, w.keys_in, w.idx_in, status);
            HX_CHECK_LAUNCH("triplet_keys_kernel");
        }
        return HX_OK;
    }
    const int nb = key_bits(dim);
    triplet_keys_kernel<<<grid_1d(n, 256), 256, 0, s>>>(rows, cols, n, dim, nb, w.keys_in, w.idx_in, status);
    HX_CHECK_LAUNCH("triplet_keys_kernel");
    size_t cb = w.cub_bytes;
    HX_TRY_CUDA(cub::DeviceRadixSort::SortPairs(w.cub_tmp, cb, w.keys_in, w.keys_out, w.idx_in, w.idx_out, n, 0,
                                                2 * nb, s));
    run_flags_kernel<<<grid_1d(n, 256), 256, 0, s>>>(w.keys_out, n, w.flags);
    HX_CHECK_LAUNCH("run_flags_kernel");
    cb = w.cub_bytes;
    HX_TRY_CUDA(cub::DeviceSelect::Flagged(w.cub_tmp, cb, cub::CountingInputIterator<int64_t>(0), w.flags, w.starts,
                                           w.num_runs, n, s));
    runs_kernel<<<grid_1d(n, 256), 256, 0, s>>>(w.keys_out, n, dim, nb, w.starts, w.num_runs, row_idx, col_ptr);
    HX_CHECK_LAUNCH("runs_kernel");
    return HX_OK;
}

extern "C" int hx_triplet_csc_numeric(const double *vals, int64_t n, int64_t dim, const int64_t *col_ptr,
                                      double *out_vals, const void *workspace, void *stream) {
    (void)col_ptr;
    if (n < 0 || workspace == nullptr || (n > 0 && (vals == nullptr || out_vals == nullptr))) {
        set_last_error("hx_triplet_csc_numeric: bad arguments");
        return HX_ERR_VALUE;
    }
    if (n == 0 || dim == 0) return HX_OK;
    TripletWs w = triplet_ws_layout(const_cast<void *>(workspace), n, dim);
    run_sum_kernel<<<grid_1d(n, 256), 256, 0, (cudaStream_t)stream>>>(vals, w.idx_out, w.starts, w.num_runs,
                                                                     out_vals);
    HX_CHECK_LAUNCH("run_sum_kernel");
    return HX_OK;
}
