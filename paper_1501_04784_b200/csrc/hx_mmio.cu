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
            // Python formats every NaN as "nan"; glibc prints a negative NaN as "-nan"
            const double v = vals[k];
            const int n = v != v ? snprintf(line, sizeof(line), "%lld %lld nan\n", (long long)(row_idx[k] + 1),
                                             (long long)(c + 1))
                                 : snprintf(line, sizeof(line), "%lld %lld %.17g\n", (long long)(row_idx[k] + 1),
                                             (long long)(c + 1), v);
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

// ---- Matrix Market import (sparseio.py:90-138), strict fast path ------------------------------------
// The reference splits the text with str.splitlines()/str.split() and converts with int()/float().
// This parser accepts the strict subset those produce identically for files like the writer's: '\n'
// line ends, ' ' / '\t' separators, decimal integers, and decimal/exponent floats or inf/nan (strtod
// is correctly rounded, as float() is).  Anything else -- other whitespace or line breaks, signs on
// indices, underscores, hex floats, ... -- returns HX_MM_FALLBACK and the caller re-reads the file
// with the reference's own rules, so semantics (and error messages) never differ.
#include <cerrno>
#include <cmath>
#include <cstdlib>

namespace hx {
enum { MM_OK = 0, MM_FALLBACK = 1, MM_ERROR = 2 };

static bool is_sep(char c) { return c == ' ' || c == '\t'; }

// next token of [p, end) (within one line); returns false at the end of the line
static bool next_token(const char *&p, const char *end, const char *&tb, const char *&te) {
    while (p < end && is_sep(*p)) ++p;
    if (p >= end) return false;
    tb = p;
    while (p < end && !is_sep(*p)) ++p;
    te = p;
    return true;
}

static bool strict_int(const char *b, const char *e, long long &v) {
    if (b >= e || e - b > 18) return false;
    long long x = 0;
    for (const char *q = b; q < e; ++q) {
        if (*q < '0' || *q > '9') return false;
        x = 10 * x + (*q - '0');
    }
    v = x;
    return true;
}

static bool strict_double(const char *b, const char *e, double &v) {
    char buf[64];
    const size_t n = (size_t)(e - b);
    if (n == 0 || n >= sizeof(buf)) return false;
    memcpy(buf, b, n);
    buf[n] = '\0';
    // accepted alphabet: digits . e E + - and the words inf / nan (as the writer emits them)
    const char *s = buf + ((buf[0] == '-' || buf[0] == '+') ? 1 : 0);
    if (strcmp(s, "inf") != 0 && strcmp(s, "nan") != 0) {
        for (const char *q = s; *q; ++q)
            if (!((*q >= '0' && *q <= '9') || *q == '.' || *q == 'e' || *q == 'E' || *q == '+' || *q == '-'))
                return false;
        if (!((s[0] >= '0' && s[0] <= '9') || s[0] == '.')) return false;
    }
    char *endp = nullptr;
    errno = 0;
    v = strtod(buf, &endp);
    return endp == buf + n;
}
}  // namespace hx

// Parse `path`.  First call with rows == NULL to get the sizes (n_rows, nnz); then with buffers of
// nnz entries.  Returns 0 (ok), 1 (fall back to the reference parser), 2 (format error at *err_line,
// message in hx_last_error, mirroring sparseio.py's MeshFormatError).
extern "C" int hx_mm_read(const char *path, int64_t *n_rows, int64_t *nnz, int32_t *rows, int32_t *cols, double *vals,
                          int64_t *err_line) {
    if (path == nullptr || n_rows == nullptr || nnz == nullptr || err_line == nullptr) return MM_FALLBACK;
    FILE *f = fopen(path, "rb");
    if (f == nullptr) return MM_FALLBACK;
    std::string text;
    {
        char chunk[1 << 16];
        size_t got;
        while ((got = fread(chunk, 1, sizeof(chunk), f)) > 0) text.append(chunk, got);
        fclose(f);
    }
    for (char c : text)
        if (c == '\r' || c == '\v' || c == '\f' || (unsigned char)c >= 0x1c && (unsigned char)c <= 0x1e ||
            (unsigned char)c >= 0x80)
            return MM_FALLBACK;  // other line breaks / non-ASCII: the reference's splitlines rules
    const char *p = text.data(), *end = p + text.size();
    int64_t line_no = 0;
    auto next_line = [&](const char *&lb, const char *&le) -> bool {
        if (p >= end) return false;
        lb = p;
        const char *nl = (const char *)memchr(p, '\n', (size_t)(end - p));
        le = nl ? nl : end;
        p = nl ? nl + 1 : end;
        ++line_no;
        return true;
    };
    const char *lb, *le, *tb, *te;
    if (!next_line(lb, le)) return MM_FALLBACK;  // empty file: the reference's error path
    {  // banner, case-insensitive tokens
        static const char *want[5] = {"%%matrixmarket", "matrix", "coordinate", "real", "symmetric"};
        const char *q = lb;
        for (int k = 0; k < 5; ++k) {
            if (!next_token(q, le, tb, te) || (size_t)(te - tb) != strlen(want[k])) return MM_FALLBACK;
            for (size_t i = 0; i < strlen(want[k]); ++i)
                if (tolower((unsigned char)tb[i]) != want[k][i]) return MM_FALLBACK;
        }
        if (next_token(q, le, tb, te)) return MM_FALLBACK;
    }
    // comments, then the size line
    do {
        if (!next_line(lb, le)) return MM_FALLBACK;
    } while (le > lb && lb[0] == '%');
    long long nr, nc, nz;
    {
        const char *q = lb;
        if (!next_token(q, le, tb, te) || !strict_int(tb, te, nr)) return MM_FALLBACK;
        if (!next_token(q, le, tb, te) || !strict_int(tb, te, nc)) return MM_FALLBACK;
        if (!next_token(q, le, tb, te) || !strict_int(tb, te, nz)) return MM_FALLBACK;
        if (next_token(q, le, tb, te)) return MM_FALLBACK;
    }
    if (nr != nc || nr > INT32_MAX) return MM_FALLBACK;
    *n_rows = nr;
    *nnz = nz;
    if (rows == nullptr) return MM_OK;  // size query
    for (long long k = 0; k < nz; ++k) {
        if (!next_line(lb, le)) return MM_FALLBACK;  // too few entries: reference error path
        const char *q = lb;
        long long r, c;
        double v;
        if (!next_token(q, le, tb, te) || !strict_int(tb, te, r)) return MM_FALLBACK;
        if (!next_token(q, le, tb, te) || !strict_int(tb, te, c)) return MM_FALLBACK;
        if (!next_token(q, le, tb, te) || !strict_double(tb, te, v)) return MM_FALLBACK;
        if (next_token(q, le, tb, te)) return MM_FALLBACK;
        if (!(1 <= r && r <= nr && 1 <= c && c <= nc)) {
            *err_line = line_no;
            set_last_error("entry (%lld, %lld) outside the matrix", r, c);
            return MM_ERROR;
        }
        if (r < c) {
            *err_line = line_no;
            set_last_error("entry (%lld, %lld) lies above the diagonal; symmetric storage is lower-triangular", r, c);
            return MM_ERROR;
        }
        rows[k] = (int32_t)(r - 1);
        cols[k] = (int32_t)(c - 1);
        vals[k] = v;
    }
    return MM_OK;
}
