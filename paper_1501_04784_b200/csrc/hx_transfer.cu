// hx_transfer.cu -- compact device -> host transfer of the lower CSC.
//
// The host result of the path is the reference's LowerCscMatrix (assemble.py:51-62): int64 col_ptr
// and row_idx, float64 vals, 16 bytes per entry.  Over PCIe (~57 GB/s device -> host, the
// end-to-end bound of a 64M-element build) the row indices do not need 64 bits: node ids are int32
// in the reference (mesh.py connectivity), so they cross as int32 -- hx_rows_narrow on the device,
// then hx_rows_widen on the host, sign-extending back to the reference dtype with all host cores
// while the next build's transfers run.  12 bytes per entry instead of 16; values and col_ptr cross
// unchanged.
#include <algorithm>

#include <cub/device/device_scan.cuh>
#include <cub/iterator/transform_input_iterator.cuh>

#include "hx_common.cuh"

namespace hx {

// 4 entries per thread per iteration: two 16-byte loads, one 16-byte store (streaming: read once).
// Unaligned buffers (views into a larger allocation) take the scalar loop only.
__global__ void rows_narrow_kernel(const int64_t *__restrict__ src, int32_t *__restrict__ dst, int64_t n,
                                   bool vector) {
    const int64_t n4 = vector ? n / 4 : 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
        const longlong2 a = __ldcs(reinterpret_cast<const longlong2 *>(src) + 2 * i);
        const longlong2 b = __ldcs(reinterpret_cast<const longlong2 *>(src) + 2 * i + 1);
        __stcs(reinterpret_cast<int4 *>(dst) + i, make_int4((int)a.x, (int)a.y, (int)b.x, (int)b.y));
    }
    for (int64_t i = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        dst[i] = (int32_t)src[i];
}

// Small device words -> mapped pinned host memory, written by a kernel: the host's status / nnz /
// fail-record reads of a build then do not queue behind a multi-gigabyte copy of the previous
// build's result on the copy engine (a cudaMemcpy of 16 bytes would wait ~200 ms there).
__global__ void peek_kernel(hx_peek_args a, int64_t *__restrict__ host) {
    const int i = threadIdx.x;
    if (i >= a.n) return;
    const unsigned char *src = static_cast<const unsigned char *>(a.src[i]);
    int64_t v = 0;
    if (a.bytes[i] == 4) v = *reinterpret_cast<const int32_t *>(src);  // sign-extended
    else v = *reinterpret_cast<const int64_t *>(src);                   // raw 8 bytes
    host[i] = v;
}

// ---- row-index codec: per-column delta stream, Stream-VByte groups --------------------------------
// Rows of a lower-CSC column are ascending node ids starting at the diagonal, so the column is sent
// as deltas d_0 = r_0 - c, d_i = r_i - r_{i-1}: in groups of 4, one control byte (2 bits per delta:
// byte length - 1) followed by the deltas' little-endian bytes; a partial last group is padded with
// 1-byte zero deltas.  Per column: count m (uint8, the col_ptr difference) and byte length (uint8).
// ~26 bytes for a 14-row interior column of a structured mesh instead of 56 (int32) -- the host
// decodes with one byte shuffle per 4 rows (hx_rows_decode).
constexpr int CODEC_BLOCK = 128;
constexpr int CODEC_MAX_COL_BYTES = 9 + 4 * 36;  // <= 36 rows per column (fast path: 33)

__device__ __forceinline__ int delta_bytes(uint32_t d) { return d < (1u << 8) ? 1 : d < (1u << 16) ? 2 : d < (1u << 24) ? 3 : 4; }

__global__ void __launch_bounds__(CODEC_BLOCK)
rows_codec_size_kernel(const int64_t *__restrict__ col_ptr, const int64_t *__restrict__ row_idx, int64_t ncols,
                       int64_t col_lo, uint8_t *__restrict__ counts, uint8_t *__restrict__ lens,
                       uint32_t *__restrict__ bad) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < ncols; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = col_ptr[j], b = col_ptr[j + 1];
        const int64_t m = b - a;
        if (m < 0 || m > 36) {  // not a fast-path column: the caller sends int32 rows instead
            atomicOr(bad, 1u);
            counts[j] = 0;
            lens[j] = 0;
            continue;
        }
        uint32_t prev = (uint32_t)(col_lo + j);
        int bytes = (int)((m + 3) / 4);
        for (int64_t i = a; i < b; ++i) {
            const uint32_t r = (uint32_t)__ldg(row_idx + i);
            bytes += delta_bytes(r - prev);
            prev = r;
        }
        bytes += (int)((4 - (m & 3)) & 3);  // pad deltas, 1 byte each
        counts[j] = (uint8_t)m;
        lens[j] = (uint8_t)bytes;
    }
}

struct U8ToI64 {
    __host__ __device__ __forceinline__ int64_t operator()(uint8_t x) const { return (int64_t)x; }
};

// one block = CODEC_BLOCK consecutive columns: each thread encodes its column into shared memory at
// its block-local offset, then the block's bytes are copied out coalesced
__global__ void __launch_bounds__(CODEC_BLOCK)
rows_codec_pack_kernel(const int64_t *__restrict__ col_ptr, const int64_t *__restrict__ row_idx, int64_t ncols,
                       int64_t col_lo, const uint8_t *__restrict__ lens, const int64_t *__restrict__ offsets,
                       uint8_t *__restrict__ out, int64_t capacity) {
    __shared__ uint8_t s_buf[CODEC_BLOCK * CODEC_MAX_COL_BYTES];
    const int64_t first = (int64_t)blockIdx.x * CODEC_BLOCK;
    const int64_t last = first + CODEC_BLOCK < ncols ? first + CODEC_BLOCK : ncols;
    const int64_t base = offsets[first], end = offsets[last];
    if (end > capacity) return;  // the caller sees total > capacity and falls back
    const int64_t j = first + threadIdx.x;
    if (j < last) {
        const int64_t a = col_ptr[j], b = col_ptr[j + 1];
        const int m = (int)(b - a);
        uint8_t *p = s_buf + (offsets[j] - base);
        const int groups = (m + 3) / 4;
        uint8_t *data = p + groups;
        uint32_t prev = (uint32_t)(col_lo + j);
        for (int g = 0; g < groups; ++g) {
            uint32_t ctrl = 0;
            for (int k = 0; k < 4; ++k) {
                const int i = 4 * g + k;
                uint32_t d = 0;
                if (i < m) {
                    const uint32_t r = (uint32_t)__ldg(row_idx + a + i);
                    d = r - prev;
                    prev = r;
                }
                const int nb = delta_bytes(d);
                ctrl |= (uint32_t)(nb - 1) << (2 * k);
                for (int q = 0; q < nb; ++q) *data++ = (uint8_t)(d >> (8 * q));
            }
            p[g] = (uint8_t)ctrl;
        }
    }
    __syncthreads();
    for (int64_t q = threadIdx.x; q < end - base; q += CODEC_BLOCK) out[base + q] = s_buf[q];
}

// total bytes, or -1 when a column is outside the codec (the caller sends int32 rows instead)
__global__ void rows_codec_total_kernel(const int64_t *__restrict__ end, const uint32_t *__restrict__ bad,
                                        int64_t *__restrict__ total) {
    *total = *bad ? -1 : *end;
}

}  // namespace hx

using namespace hx;

extern "C" int64_t hx_rows_encode_workspace_bytes(int64_t ncols) {
    if (ncols < 0) return -1;
    size_t cb = 0;
    cub::TransformInputIterator<int64_t, U8ToI64, const uint8_t *> it(nullptr, U8ToI64{});
    cub::DeviceScan::ExclusiveSum(nullptr, cb, it, (int64_t *)nullptr, (int)(ncols + 1));
    return (int64_t)(align_up(8 * (size_t)(ncols + 1), 256) + 256 + cb);
}

extern "C" int hx_rows_encode(const int64_t *col_ptr, const int64_t *row_idx, int64_t ncols, int64_t col_lo,
                              uint8_t *counts, uint8_t *lens, uint8_t *bytes, int64_t capacity, int64_t *total,
                              void *workspace, int64_t workspace_bytes, void *stream) {
    if (ncols < 0 || col_ptr == nullptr || total == nullptr || (ncols > 0 && (counts == nullptr || lens == nullptr)) ||
        capacity < 0 || (capacity > 0 && bytes == nullptr) || workspace == nullptr ||
        workspace_bytes < hx_rows_encode_workspace_bytes(ncols) || ncols >= INT32_MAX) {
        set_last_error("hx_rows_encode: bad arguments");
        return HX_ERR_VALUE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    char *w = (char *)workspace;
    int64_t *offsets = (int64_t *)w;  // ncols + 1
    uint32_t *bad = (uint32_t *)(w + align_up(8 * (size_t)(ncols + 1), 256));
    void *cub_tmp = w + align_up(8 * (size_t)(ncols + 1), 256) + 256;
    size_t cb = (size_t)workspace_bytes - align_up(8 * (size_t)(ncols + 1), 256) - 256;
    HX_TRY_CUDA(cudaMemsetAsync(bad, 0, sizeof(uint32_t), s));
    if (ncols == 0) {
        HX_TRY_CUDA(cudaMemsetAsync(total, 0, sizeof(int64_t), s));
        return HX_OK;
    }
    const int64_t blocks = ceil_div(ncols, CODEC_BLOCK);
    rows_codec_size_kernel<<<(unsigned)std::min<int64_t>(blocks, 148 * 16), CODEC_BLOCK, 0, s>>>(
        col_ptr, row_idx, ncols, col_lo, counts, lens, bad);
    HX_CHECK_LAUNCH("rows_codec_size_kernel");
    // offsets[j] = bytes before column j, offsets[ncols] = total: inclusive scan into offsets + 1
    cub::TransformInputIterator<int64_t, U8ToI64, const uint8_t *> it(lens, U8ToI64{});
    HX_TRY_CUDA(cub::DeviceScan::InclusiveSum(cub_tmp, cb, it, offsets + 1, (int)ncols, s));
    HX_TRY_CUDA(cudaMemsetAsync(offsets, 0, sizeof(int64_t), s));
    rows_codec_pack_kernel<<<(unsigned)blocks, CODEC_BLOCK, 0, s>>>(col_ptr, row_idx, ncols, col_lo, lens, offsets,
                                                                    bytes, capacity);
    HX_CHECK_LAUNCH("rows_codec_pack_kernel");
    rows_codec_total_kernel<<<1, 1, 0, s>>>(offsets + ncols, bad, total);
    HX_CHECK_LAUNCH("rows_codec_total_kernel");
    return HX_OK;
}


extern "C" int hx_peek(const hx_peek_args *args, int64_t *host_dst, void *stream) {
    if (args == nullptr || host_dst == nullptr || args->n < 0 || args->n > HX_PEEK_MAX) {
        set_last_error("hx_peek: bad arguments");
        return HX_ERR_VALUE;
    }
    for (int i = 0; i < args->n; ++i)
        if (args->src[i] == nullptr || (args->bytes[i] != 4 && args->bytes[i] != 8)) {
            set_last_error("hx_peek: word %d must be a 4- or 8-byte device word", i);
            return HX_ERR_VALUE;
        }
    if (args->n == 0) return HX_OK;
    peek_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(*args, host_dst);
    HX_CHECK_LAUNCH("peek_kernel");
    return HX_OK;
}

extern "C" int hx_rows_narrow(const int64_t *row_idx, int32_t *rows32, int64_t n, void *stream) {
    if (n < 0 || (n > 0 && (row_idx == nullptr || rows32 == nullptr))) {
        set_last_error("hx_rows_narrow: bad arguments");
        return HX_ERR_VALUE;
    }
    if (n == 0) return HX_OK;
    const bool vector = !(reinterpret_cast<uintptr_t>(row_idx) & 15) && !(reinterpret_cast<uintptr_t>(rows32) & 15);
    const int64_t blocks = std::min<int64_t>(ceil_div(std::max<int64_t>(vector ? n / 4 : n, 1), 256), 148 * 8);
    rows_narrow_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(row_idx, rows32, n, vector);
    HX_CHECK_LAUNCH("rows_narrow_kernel");
    return HX_OK;
}


