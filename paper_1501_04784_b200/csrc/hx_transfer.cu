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

}  // namespace hx

using namespace hx;

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


