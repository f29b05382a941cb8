// hx_host.cpp -- host-side halves of the CSC transfer (plain C++, compiled by the host compiler).
//
// hx_rows_widen sign-extends the int32 row indices that crossed PCIe back to the reference's int64
// row_idx (assemble.py:51-62) with all host cores.  It runs while the value array is still in
// flight, so it shares host memory bandwidth with the DMA engine: on AVX-512 hosts the stores are
// non-temporal (no read-for-ownership of the 8-byte destination: 12 instead of 20 bytes of memory
// traffic per entry).
#include <immintrin.h>
#include <stdint.h>

#include <climits>

#include <algorithm>
#include <atomic>
#include <thread>
#include <vector>

#include "../../include/hexfem_b200.h"

namespace hx {
void set_last_error(const char *fmt, ...);
}

namespace {

// min and max of an element's 8 node ids (one 256-bit load on AVX2 hosts)
__attribute__((target("avx2"))) inline void minmax8_avx2(const int32_t *g, int32_t &mn, int32_t &mx) {
    const __m256i v = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(g));
    __m128i lo = _mm_min_epi32(_mm256_castsi256_si128(v), _mm256_extracti128_si256(v, 1));
    __m128i hi = _mm_max_epi32(_mm256_castsi256_si128(v), _mm256_extracti128_si256(v, 1));
    lo = _mm_min_epi32(lo, _mm_shuffle_epi32(lo, 0x4E));
    hi = _mm_max_epi32(hi, _mm_shuffle_epi32(hi, 0x4E));
    lo = _mm_min_epi32(lo, _mm_shuffle_epi32(lo, 0xB1));
    hi = _mm_max_epi32(hi, _mm_shuffle_epi32(hi, 0xB1));
    mn = _mm_cvtsi128_si32(lo);
    mx = _mm_cvtsi128_si32(hi);
}

inline void minmax8_scalar(const int32_t *g, int32_t &mn, int32_t &mx) {
    mn = mx = g[0];
    for (int k = 1; k < 8; ++k) {
        mn = std::min(mn, g[k]);
        mx = std::max(mx, g[k]);
    }
}

// Elements [a, z) of the block-range scan: per block the first / one-past-last element whose node
// span covers it (L / H), and the chunk's node range.  The same body twice: AVX2 min / max of the 8
// ids, and scalar.
__attribute__((target("avx2"))) void scan_chunk_avx2(const int32_t *conn, int64_t a, int64_t z,
                                                     const int64_t *bounds, int K, int64_t *L, int64_t *H,
                                                     int32_t &chunk_min, int32_t &chunk_max) {
    auto block_of = [&](int64_t node) -> int {
        const int64_t *it = std::upper_bound(bounds + 1, bounds + K, node);
        return (int)(it - (bounds + 1));
    };
    // consecutive elements of a locally numbered mesh stay in one block span: cache the last
    // element's block bounds and binary-search only when a node leaves them
    int b0 = 0, b1 = 0;
    int64_t lo0 = INT64_MAX, hi0 = INT64_MIN, lo1 = INT64_MAX, hi1 = INT64_MIN;
    // runs of consecutive elements with the same block span update L / H once per run
    int rb0 = -1, rb1 = -1;
    int64_t run_start = a;
    auto close_run = [&](int64_t run_end) {
        for (int b = rb0; b <= rb1 && rb0 >= 0; ++b) {
            if (L[b] == INT64_MAX) L[b] = run_start;  // elements of a chunk come in ascending order
            H[b] = run_end;
        }
    };
    for (int64_t e = a; e < z; ++e) {
        int32_t mn, mx;
        minmax8_avx2(conn + 8 * e, mn, mx);
        chunk_min = std::min(chunk_min, mn);
        chunk_max = std::max(chunk_max, mx);
        if (mn < lo0 || mn >= hi0) {
            b0 = block_of(mn);
            lo0 = b0 == 0 ? INT64_MIN : bounds[b0];
            hi0 = b0 == K - 1 ? INT64_MAX : bounds[b0 + 1];
        }
        if (mx < lo1 || mx >= hi1) {
            b1 = block_of(mx);
            lo1 = b1 == 0 ? INT64_MIN : bounds[b1];
            hi1 = b1 == K - 1 ? INT64_MAX : bounds[b1 + 1];
        }
        if (b0 != rb0 || b1 != rb1) {
            close_run(e);
            rb0 = b0;
            rb1 = b1;
            run_start = e;
        }
    }
    close_run(z);
}

void scan_chunk_scalar(const int32_t *conn, int64_t a, int64_t z, const int64_t *bounds, int K, int64_t *L,
                       int64_t *H, int32_t &chunk_min, int32_t &chunk_max) {
    auto block_of = [&](int64_t node) -> int {
        const int64_t *it = std::upper_bound(bounds + 1, bounds + K, node);
        return (int)(it - (bounds + 1));
    };
    // consecutive elements of a locally numbered mesh stay in one block span: cache the last
    // element's block bounds and binary-search only when a node leaves them
    int b0 = 0, b1 = 0;
    int64_t lo0 = INT64_MAX, hi0 = INT64_MIN, lo1 = INT64_MAX, hi1 = INT64_MIN;
    // runs of consecutive elements with the same block span update L / H once per run
    int rb0 = -1, rb1 = -1;
    int64_t run_start = a;
    auto close_run = [&](int64_t run_end) {
        for (int b = rb0; b <= rb1 && rb0 >= 0; ++b) {
            if (L[b] == INT64_MAX) L[b] = run_start;  // elements of a chunk come in ascending order
            H[b] = run_end;
        }
    };
    for (int64_t e = a; e < z; ++e) {
        int32_t mn, mx;
        minmax8_scalar(conn + 8 * e, mn, mx);
        chunk_min = std::min(chunk_min, mn);
        chunk_max = std::max(chunk_max, mx);
        if (mn < lo0 || mn >= hi0) {
            b0 = block_of(mn);
            lo0 = b0 == 0 ? INT64_MIN : bounds[b0];
            hi0 = b0 == K - 1 ? INT64_MAX : bounds[b0 + 1];
        }
        if (mx < lo1 || mx >= hi1) {
            b1 = block_of(mx);
            lo1 = b1 == 0 ? INT64_MIN : bounds[b1];
            hi1 = b1 == K - 1 ? INT64_MAX : bounds[b1 + 1];
        }
        if (b0 != rb0 || b1 != rb1) {
            close_run(e);
            rb0 = b0;
            rb1 = b1;
            run_start = e;
        }
    }
    close_run(z);
}


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

// ---- row-index codec, host half (hx_rows_encode's format, hx_transfer.cu) ------------------------
struct CodecTables {
    alignas(16) uint8_t shuf[256][16];
    uint8_t len[256];
    CodecTables() {
        for (int c = 0; c < 256; ++c) {
            int off = 0;
            for (int k = 0; k < 4; ++k) {
                const int nb = ((c >> (2 * k)) & 3) + 1;
                for (int q = 0; q < 4; ++q) shuf[c][4 * k + q] = q < nb ? (uint8_t)(off + q) : 0x80;
                off += nb;
            }
            len[c] = (uint8_t)off;
        }
    }
};
const CodecTables &codec_tables() {
    static const CodecTables t;
    return t;
}

// Columns [j0, j1) of a block: rows_out / bytes at this range's first row / byte.  Groups decode 4
// rows at a time into a cache-resident staging buffer (the 0..3 rows past a column's end are
// rewritten by the next column), which is flushed to rows_out with non-temporal stores: the int64
// rows are the host's largest write, and regular stores would first read every destination line
// (read-for-ownership), doubling the memory traffic the decode shares with the incoming DMA.
// Returns the bytes consumed.
__attribute__((target("sse2"))) void stream_out(int64_t *dst, const int64_t *src, int64_t n) {
    if (n > 0 && (reinterpret_cast<uintptr_t>(dst) & 15)) {
        _mm_stream_si64(reinterpret_cast<long long *>(dst), src[0]);
        ++dst;
        ++src;
        --n;
    }
    for (; n >= 2; n -= 2, dst += 2, src += 2)
        _mm_stream_si128(reinterpret_cast<__m128i *>(dst), _mm_loadu_si128(reinterpret_cast<const __m128i *>(src)));
    if (n > 0) _mm_stream_si64(reinterpret_cast<long long *>(dst), src[0]);
}

__attribute__((target("ssse3,sse4.1"))) int64_t decode_columns(const uint8_t *counts, const uint8_t *bytes,
                                                                 int64_t j0, int64_t j1, int64_t col_lo,
                                                                 int64_t *rows_out) {
    const CodecTables &T = codec_tables();
    constexpr int STAGE = 2048;
    alignas(64) int64_t stage[STAGE + 8];
    int pos = 0;
    const uint8_t *p = bytes;
    int64_t *out = rows_out;
    for (int64_t j = j0; j < j1; ++j) {
        const int m = counts[j];
        if (pos + m + 4 > STAGE) {
            stream_out(out, stage, pos);
            out += pos;
            pos = 0;
        }
        const int groups = (m + 3) >> 2;
        const uint8_t *ctrl = p;
        const uint8_t *data = p + groups;
        __m128i base = _mm_set1_epi32((int)(uint32_t)(col_lo + j));
        int64_t *st = stage + pos;
        for (int g = 0; g < groups; ++g) {
            const uint8_t c = ctrl[g];
            __m128i v = _mm_shuffle_epi8(_mm_loadu_si128(reinterpret_cast<const __m128i *>(data)),
                                         _mm_load_si128(reinterpret_cast<const __m128i *>(T.shuf[c])));
            v = _mm_add_epi32(v, _mm_slli_si128(v, 4));
            v = _mm_add_epi32(v, _mm_slli_si128(v, 8));
            v = _mm_add_epi32(v, base);
            _mm_storeu_si128(reinterpret_cast<__m128i *>(st + 4 * g), _mm_cvtepu32_epi64(v));
            _mm_storeu_si128(reinterpret_cast<__m128i *>(st + 4 * g + 2), _mm_cvtepu32_epi64(_mm_srli_si128(v, 8)));
            base = _mm_shuffle_epi32(v, 0xFF);
            data += T.len[c];
        }
        pos += m;
        p = data;
    }
    stream_out(out, stage, pos);
    _mm_sfence();
    return p - bytes;
}

}  // namespace

// Decode hx_rows_encode's stream into int64 rows (the reference's row_idx dtype) and col_ptr ends
// (col_ptr_out[j] = row_base + rows of columns 0..j), all host cores: each worker takes a range of
// columns, whose first row / byte come from a first parallel pass over the counts and lengths.
extern "C" int hx_rows_decode(const uint8_t *counts, const uint8_t *lens, const uint8_t *bytes, int64_t nbytes,
                              int64_t ncols, int64_t col_lo, int64_t row_base, int64_t *col_ptr_out,
                              int64_t *rows_out, int32_t threads) {
    if (ncols < 0 || nbytes < 0 || (ncols > 0 && (counts == nullptr || lens == nullptr || col_ptr_out == nullptr)) ||
        (nbytes > 0 && (bytes == nullptr || rows_out == nullptr))) {
        hx::set_last_error("hx_rows_decode: bad arguments");
        return HX_ERR_VALUE;
    }
    if (ncols == 0) return HX_OK;
    if (!__builtin_cpu_supports("ssse3") || !__builtin_cpu_supports("sse4.1")) {
        hx::set_last_error("hx_rows_decode: the host CPU lacks SSSE3 / SSE4.1");
        return HX_ERR_CONFIG;
    }
    const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
    constexpr int64_t MIN_COLS = int64_t(1) << 15;
    const int nt = (int)std::max<int64_t>(1, std::min<int64_t>(threads > 0 ? threads : hw, ncols / MIN_COLS + 1));
    std::vector<int64_t> jb(nt + 1), rows_before(nt + 1, 0), bytes_before(nt + 1, 0);
    for (int t = 0; t <= nt; ++t) jb[t] = ncols * t / nt;
    auto run = [&](auto &&fn) {
        std::vector<std::thread> pool;
        pool.reserve(nt - 1);
        for (int t = 1; t < nt; ++t) pool.emplace_back(fn, t);
        fn(0);
        for (auto &th : pool) th.join();
    };
    run([&](int t) {  // per range: rows and bytes
        int64_t r = 0, b = 0;
        for (int64_t j = jb[t]; j < jb[t + 1]; ++j) {
            r += counts[j];
            b += lens[j];
        }
        rows_before[t + 1] = r;
        bytes_before[t + 1] = b;
    });
    for (int t = 0; t < nt; ++t) {
        rows_before[t + 1] += rows_before[t];
        bytes_before[t + 1] += bytes_before[t];
    }
    if (bytes_before[nt] != nbytes) {
        hx::set_last_error("hx_rows_decode: the stream holds %lld bytes, the lengths say %lld", (long long)nbytes,
                           (long long)bytes_before[nt]);
        return HX_ERR_VALUE;
    }
    std::atomic<int> bad{0};
    run([&](int t) {
        const int64_t j0 = jb[t], j1 = jb[t + 1];
        if (j0 == j1) return;
        const int64_t used = decode_columns(counts, bytes + bytes_before[t], j0, j1, col_lo, rows_out + rows_before[t]);
        if (used != bytes_before[t + 1] - bytes_before[t]) bad.store(1);
        int64_t acc = row_base + rows_before[t];
        for (int64_t j = j0; j < j1; ++j) {
            acc += counts[j];
            col_ptr_out[j] = acc;
        }
    });
    if (bad.load()) {
        hx::set_last_error("hx_rows_decode: corrupt stream (byte lengths do not match the control bytes)");
        return HX_ERR_VALUE;
    }
    return HX_OK;
}

namespace {

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

// Element range of each column block for the streamed build: block k = columns [bounds[k],
// bounds[k+1]); an element with node ids spanning blocks [b(min), b(max)] may hold columns of each
// of them, so e_lo[k] / e_hi[k] = the lowest element / one past the highest element whose span
// covers k (a superset of the elements touching k -- extra elements contribute nothing to the
// block).  Ids outside [0, n_nodes) clamp to the first / last block (the integration kernel reports
// them).  Empty blocks get e_lo = e_hi = 0.  Host code, `threads` workers over element chunks.
extern "C" int hx_block_ranges_nodes(const int32_t *conn, int64_t n_el, const int64_t *bounds, int32_t n_blocks,
                                     int64_t *e_lo, int64_t *e_hi, int64_t *node_lo, int64_t *node_hi,
                                     int32_t threads);

extern "C" int hx_block_ranges(const int32_t *conn, int64_t n_el, const int64_t *bounds, int32_t n_blocks,
                               int64_t *e_lo, int64_t *e_hi, int32_t threads) {
    return hx_block_ranges_nodes(conn, n_el, bounds, n_blocks, e_lo, e_hi, nullptr, nullptr, threads);
}

extern "C" int hx_block_ranges_nodes(const int32_t *conn, int64_t n_el, const int64_t *bounds, int32_t n_blocks,
                                     int64_t *e_lo, int64_t *e_hi, int64_t *node_lo, int64_t *node_hi,
                                     int32_t threads) {
    if (n_el < 0 || n_blocks < 1 || bounds == nullptr || e_lo == nullptr || e_hi == nullptr ||
        (n_el > 0 && conn == nullptr) || ((node_lo == nullptr) != (node_hi == nullptr))) {
        hx::set_last_error("hx_block_ranges: bad arguments");
        return HX_ERR_VALUE;
    }
    const int K = n_blocks;
    auto block_of = [&](int64_t node) -> int {
        // largest k with bounds[k] <= node, clamped to [0, K-1]
        const int64_t *it = std::upper_bound(bounds + 1, bounds + K, node);
        return (int)(it - (bounds + 1));
    };
    const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
    static const bool avx2 = __builtin_cpu_supports("avx2");
    const int64_t per = int64_t(1) << 20;
    const int64_t chunks = (n_el + per - 1) / per;
    const int nt = (int)std::max<int64_t>(1, std::min<int64_t>(threads > 0 ? threads : hw, chunks));
    struct Acc {
        std::vector<int64_t> L, H;
    };
    std::vector<Acc> acc(nt);
    // per element chunk: its smallest / largest node (the node range of a block's element range is
    // bounded by the chunks it overlaps -- a superset of what the block gathers)
    std::vector<int64_t> cmin(chunks, INT64_MAX), cmax(chunks, INT64_MIN);
    std::atomic<int64_t> next{0};
    auto work = [&](int t) {
        // thread-local accumulators (the per-element updates must not share cache lines)
        std::vector<int64_t> Lv(K, INT64_MAX), Hv(K, 0);
        int64_t *L = Lv.data(), *H = Hv.data();
        for (int64_t c = next.fetch_add(1); c < chunks; c = next.fetch_add(1)) {
            const int64_t a = c * per, z = std::min(n_el, a + per);
            int32_t chunk_min = INT32_MAX, chunk_max = INT32_MIN;
            if (avx2) scan_chunk_avx2(conn, a, z, bounds, K, L, H, chunk_min, chunk_max);
            else scan_chunk_scalar(conn, a, z, bounds, K, L, H, chunk_min, chunk_max);
            cmin[c] = chunk_min;
            cmax[c] = chunk_max;
        }
        acc[t] = Acc{std::move(Lv), std::move(Hv)};
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto &th : pool) th.join();
    for (int b = 0; b < K; ++b) {
        int64_t l = INT64_MAX, h = 0;
        for (int t = 0; t < nt; ++t) {
            l = std::min(l, acc[t].L[b]);
            h = std::max(h, acc[t].H[b]);
        }
        e_lo[b] = h > 0 ? l : 0;
        e_hi[b] = h;
        if (node_lo != nullptr) {  // nodes the block's element range may gather: [node_lo, node_hi)
            int64_t nl = INT64_MAX, nh = INT64_MIN;
            for (int64_t c = h > 0 ? e_lo[b] / per : 0; h > 0 && c <= (h - 1) / per; ++c) {
                nl = std::min(nl, cmin[c]);
                nh = std::max(nh, cmax[c]);
            }
            node_lo[b] = h > 0 ? std::max<int64_t>(nl, 0) : 0;
            node_hi[b] = h > 0 ? nh + 1 : 0;
        }
    }
    return HX_OK;
}

// A streaming plan from every step-th element (the streamed run_build's fast start: ~1/step of the
// connectivity read instead of all of it).  Block k's predicted element range extends one sample
// before its first touching sample and two after its last; its coordinate prefix covers those
// samples' nodes.  A prediction, not a superset: hx_block_verify checks every element on the device
// and the caller falls back to hx_block_ranges_nodes when it fails.  HOST code.
extern "C" int hx_block_ranges_sampled(const int32_t *conn, int64_t n_el, const int64_t *bounds, int32_t n_blocks,
                                       int64_t step, int64_t *e_lo, int64_t *e_hi, int64_t *node_hi,
                                       int32_t threads) {
    if (n_el < 0 || n_blocks < 1 || step < 1 || bounds == nullptr || e_lo == nullptr || e_hi == nullptr ||
        node_hi == nullptr || (n_el > 0 && conn == nullptr)) {
        hx::set_last_error("hx_block_ranges_sampled: bad arguments");
        return HX_ERR_VALUE;
    }
    const int K = n_blocks;
    const int64_t ns = n_el > 0 ? (n_el - 1) / step + 1 : 0;  // samples 0, step, 2 step, ..., and n_el - 1
    std::vector<int32_t> smax(ns + 1, INT32_MIN);
    // each sample is one cache line (and usually one page walk) away from the last: latency-bound, so
    // the samples are split over threads, each with its own first / last sample per block
    const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
    const int T = (int)std::max<int64_t>(1, std::min<int64_t>({threads > 0 ? threads : hw, hw, (ns + 1) / 4096 + 1}));
    std::vector<int64_t> first((size_t)T * K, -1), last((size_t)T * K, -1);
    auto work = [&](int t) {
        const int64_t i_lo = (ns + 1) * t / T, i_hi = (ns + 1) * (t + 1) / T;
        int64_t *f = first.data() + (size_t)t * K, *l = last.data() + (size_t)t * K;
        for (int64_t i = i_lo; i < i_hi && n_el > 0; ++i) {
            const int64_t e = std::min(i * step, n_el - 1);
            const int32_t *g = conn + 8 * e;
            int32_t mn = g[0], mx = g[0];
            for (int k = 1; k < 8; ++k) {
                mn = std::min(mn, g[k]);
                mx = std::max(mx, g[k]);
            }
            smax[i] = mx;
            const int b0 = (int)(std::upper_bound(bounds + 1, bounds + K, (int64_t)mn) - (bounds + 1));
            const int b1 = (int)(std::upper_bound(bounds + 1, bounds + K, (int64_t)mx) - (bounds + 1));
            for (int b = b0; b <= b1; ++b) {
                if (f[b] < 0) f[b] = i;
                l[b] = i;
            }
        }
    };
    if (T == 1) {
        work(0);
    } else {
        std::vector<std::thread> pool;
        for (int t = 0; t < T; ++t) pool.emplace_back(work, t);
        for (auto &th : pool) th.join();
    }
    for (int b = 0; b < K; ++b) {
        int64_t fb = -1, lb = -1;
        for (int t = 0; t < T; ++t) {  // threads hold ascending sample ranges
            const int64_t f = first[(size_t)t * K + b], l = last[(size_t)t * K + b];
            if (f >= 0 && fb < 0) fb = f;
            if (l >= 0) lb = l;
        }
        if (fb < 0) {
            e_lo[b] = e_hi[b] = node_hi[b] = 0;
            continue;
        }
        const int64_t i0 = std::max<int64_t>(fb - 1, 0), i1 = std::min<int64_t>(lb + 2, ns);
        e_lo[b] = std::min(i0 * step, n_el);
        e_hi[b] = std::min((i1 + 1) * step, n_el);
        // nodes up to the sample after the range (elements between the last two samples lie below it
        // on a locally numbered mesh; hx_block_verify checks the rest)
        int32_t top = INT32_MIN;
        for (int64_t i = i0; i <= std::min(i1 + 1, ns); ++i) top = std::max(top, smax[i]);
        node_hi[b] = (int64_t)top + 1;
    }
    return HX_OK;
}
