// hx_host.cpp -- host-side halves of the CSC transfer (plain C++, compiled by the host compiler).
//
// hx_rows_widen sign-extends the int32 row indices that crossed PCIe back to the reference's int64
// row_idx (assemble.py:51-62) with all host cores.  It runs while the value array is still in
// flight, so it shares host memory bandwidth with the DMA engine: on AVX-512 hosts the stores are
// non-temporal (no read-for-ownership of the 8-byte destination: 12 instead of 20 bytes of memory
// traffic per entry).
#include <immintrin.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <thread>
#include <vector>

#include "../../include/hexfem_b200.h"

namespace hx {
void set_last_error(const char *fmt, ...);
}

namespace {

void widen_scalar(const int32_t *src, int64_t *dst, int64_t n) {
    for (int64_t i = 0; i < n; ++i) dst[i] = src[i];
}

__attribute__((target("avx512f"))) void widen_avx512(const int32_t *src, int64_t *dst, int64_t n) {
    int64_t i = 0;
    while (i < n && (reinterpret_cast<uintptr_t>(dst + i) & 63)) {  // align the stores to 64 bytes
        dst[i] = src[i];
        ++i;
    }
    for (; i + 16 <= n; i += 16) {
        const __m512i v = _mm512_loadu_si512(reinterpret_cast<const void *>(src + i));
        _mm512_stream_si512(reinterpret_cast<__m512i *>(dst + i), _mm512_cvtepi32_epi64(_mm512_castsi512_si256(v)));
        _mm512_stream_si512(reinterpret_cast<__m512i *>(dst + i + 8),
                            _mm512_cvtepi32_epi64(_mm512_extracti64x4_epi64(v, 1)));
    }
    for (; i < n; ++i) dst[i] = src[i];
    _mm_sfence();
}

}  // namespace

extern "C" int hx_rows_widen(const int32_t *rows32, int64_t *row_idx, int64_t n, int32_t threads) {
    if (n < 0 || (n > 0 && (rows32 == nullptr || row_idx == nullptr))) {
        hx::set_last_error("hx_rows_widen: bad arguments");
        return HX_ERR_VALUE;
    }
    static const bool avx512 = __builtin_cpu_supports("avx512f");
    auto widen = avx512 ? widen_avx512 : widen_scalar;
    // chunks of 2^20 entries taken from a shared counter: a core that is busy elsewhere (the
    // caller's stream synchronisation spins on one) delays only the chunks it holds
    constexpr int64_t CHUNK = int64_t(1) << 20;
    const int64_t chunks = (n + CHUNK - 1) / CHUNK;
    const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
    const int nt = (int)std::max<int64_t>(1, std::min<int64_t>(threads > 0 ? threads : hw, chunks));
    std::atomic<int64_t> next{0};
    auto work = [&]() {
        for (int64_t c = next.fetch_add(1); c < chunks; c = next.fetch_add(1)) {
            const int64_t lo = c * CHUNK, hi = std::min(n, lo + CHUNK);
            widen(rows32 + lo, row_idx + lo, hi - lo);
        }
    };
    std::vector<std::thread> pool;
    pool.reserve(nt - 1);
    for (int t = 1; t < nt; ++t) pool.emplace_back(work);
    work();
    for (auto &th : pool) th.join();
    return HX_OK;
}
