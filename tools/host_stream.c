// Host memory bandwidth probe (the e2e roofline's host side): non-temporal write, read, and NT copy
// over 4 GiB buffers with every core.  Build: gcc -O3 -march=native -fopenmp tools/host_stream.c
#include <immintrin.h>
#include <omp.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static double now(void) { return omp_get_wtime(); }

int main(int argc, char **argv) {
    const size_t n = (size_t)(argc > 1 ? atof(argv[1]) : 4.0) * (1ull << 30);
    const size_t m = n / 64;
    __m512i *a = aligned_alloc(64, n), *b = aligned_alloc(64, n);
    memset(a, 1, n);
    memset(b, 2, n);
    for (int rep = 0; rep < 3; ++rep) {
        double t = now();
#pragma omp parallel for schedule(static)
        for (size_t i = 0; i < m; ++i) _mm512_stream_si512(a + i, _mm512_set1_epi64((long long)i));
        _mm_sfence();
        const double tw = now() - t;
        t = now();
        __m512i acc = _mm512_setzero_si512();
#pragma omp parallel
        {
            __m512i s = _mm512_setzero_si512();
#pragma omp for schedule(static)
            for (size_t i = 0; i < m; ++i) s = _mm512_add_epi64(s, _mm512_load_si512(a + i));
#pragma omp critical
            acc = _mm512_add_epi64(acc, s);
        }
        const double tr = now() - t;
        t = now();
#pragma omp parallel for schedule(static)
        for (size_t i = 0; i < m; ++i) _mm512_stream_si512(b + i, _mm512_load_si512(a + i));
        _mm_sfence();
        const double tc = now() - t;
        long long v[8];
        _mm512_storeu_si512(v, acc);
        printf("threads %d  NT write %.1f GB/s  read %.1f GB/s  NT copy %.1f GB/s (read+write)  [%lld]\n",
               omp_get_max_threads(), n / tw / 1e9, n / tr / 1e9, 2.0 * n / tc / 1e9, v[0] & 1);
    }
    return 0;
}
