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
#include <thread>
#include <vector>

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

}  // namespace hx

using namespace hx;

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

extern "C" int hx_rows_widen(const int32_t *rows32, int64_t *row_idx, int64_t n, int32_t threads) {
    if (n < 0 || (n > 0 && (rows32 == nullptr || row_idx == nullptr))) {
        set_last_error("hx_rows_widen: bad arguments");
        return HX_ERR_VALUE;
    }
    const int nt = (int)std::max<int64_t>(1, std::min<int64_t>(threads > 0 ? threads : (int)std::thread::hardware_concurrency(),
                                                              n / (1 << 20) + 1));
    auto work = [&](int t) {
        const int64_t lo = n * t / nt, hi = n * (t + 1) / nt;
        for (int64_t i = lo; i < hi; ++i) row_idx[i] = rows32[i];
    };
    if (nt == 1) {
        work(0);
        return HX_OK;
    }
    std::vector<std::thread> pool;
    pool.reserve(nt - 1);
    for (int t = 1; t < nt; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto &th : pool) th.join();
    return HX_OK;
}
