// hx_mmio.cu -- Matrix Market export of the lower CSC (sparseio.py:73-87) as multi-threaded native
// host code: the reference formats every entry in a Python loop (`f"{r} {c} {v:.17g}"`), minutes
// for the 900M entries of the 64M-element mesh.  Here worker threads format disjoint column ranges
// with snprintf("%.17g") -- glibc's correctly rounded conversion and C99's %g rules, which are the
// same digits, exponent form ("e-05"), trailing-zero removal and inf/nan spelling as Python's
// format(v, ".17g") -- and the buffers are written in column order, so the file is byte-identical.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "hx_common.cuh"

namespace hx {

static void format_columns(const int64_t *col_ptr, const int64_t *row_idx, const double *vals, int64_t c0,
                           int64_t c1, std::string &out) {
    char line[96];
    out.clear();
    out.reserve((size_t)(col_ptr[c1] - col_ptr[c0]) * 36);
    for (int64_t c = c0; c < c1; ++c)
        for (int64_t k = col_ptr[c]; k < col_ptr[c + 1]; ++k) {
            const int n = snprintf(line, sizeof(line), "%lld %lld %.17g\n", (long long)(row_idx[k] + 1),
                                   (long long)(c + 1), vals[k]);
            out.append(line, (size_t)n);
        }
}

}  // namespace hx

using namespace hx;

extern "C" int hx_mm_write(const int64_t *col_ptr, const int64_t *row_idx, const double *vals, int64_t dim,
                           const char *path, int32_t threads) {
    if (dim < 0 || col_ptr == nullptr || path == nullptr || (col_ptr[dim] > 0 && (row_idx == nullptr || vals == nullptr))) {
        set_last_error("hx_mm_write: bad arguments");
        return HX_ERR_VALUE;
    }
    FILE *f = fopen(path, "wb");
    if (f == nullptr) {
        set_last_error("hx_mm_write: cannot open %s", path);
        return HX_ERR_VALUE;
    }
    const int64_t nnz = col_ptr[dim];
    fprintf(f, "%%%%MatrixMarket matrix coordinate real symmetric\n%lld %lld %lld\n", (long long)dim, (long long)dim,
            (long long)nnz);
    const int nt = std::max(1, threads > 0 ? threads : (int)std::thread::hardware_concurrency());
    // rounds of nt column ranges of ~2M entries each: bounded memory, file order preserved
    const int64_t per_task = 1 << 21;
    std::vector<std::string> bufs(nt);
    int64_t c = 0;
    int rc = HX_OK;
    while (c < dim && rc == HX_OK) {
        std::vector<int64_t> starts(nt + 1, dim);
        starts[0] = c;
        for (int t = 0; t < nt; ++t) {
            const int64_t target = col_ptr[starts[t]] + per_task;
            int64_t e = std::upper_bound(col_ptr + starts[t], col_ptr + dim + 1, target) - col_ptr - 1;
            starts[t + 1] = std::min<int64_t>(dim, std::max<int64_t>(e, starts[t] + 1));
            if (starts[t] >= dim) starts[t + 1] = dim;
        }
        std::vector<std::thread> pool;
        for (int t = 0; t < nt; ++t)
            if (starts[t] < starts[t + 1])
                pool.emplace_back(format_columns, col_ptr, row_idx, vals, starts[t], starts[t + 1], std::ref(bufs[t]));
        for (auto &th : pool) th.join();
        for (int t = 0; t < nt; ++t)
            if (starts[t] < starts[t + 1] && fwrite(bufs[t].data(), 1, bufs[t].size(), f) != bufs[t].size()) {
                set_last_error("hx_mm_write: short write to %s", path);
                rc = HX_ERR_VALUE;
                break;
            }
        c = starts[nt];
    }
    if (fclose(f) != 0 && rc == HX_OK) {
        set_last_error("hx_mm_write: close failed for %s", path);
        rc = HX_ERR_VALUE;
    }
    return rc;
}
