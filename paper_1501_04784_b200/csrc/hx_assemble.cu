// hx_assemble.cu -- on-GPU lower-triangular CSC assembly for hex8 meshes (the paper's CPU
// sparse()/sparse_create step, assemble.py:110-239), node-adjacency based:
//
//   symbolic  1. adjacency   node -> incident (element << 3 | local node), 8 fixed slots per
//                            node (atomic slot counter; valence > 8 leaves the fast path)
//             2. pattern     per column c: incident elements sorted by id (= the stable-sort order of
//                            assemble.py:125), distinct rows r > c from a 32-slot shared-memory hash
//                            set, each carrying its contribution list (<= 4 (element, local node)
//                            pairs in element order); keys compacted and sorted by a register network;
//                            column count -> CUB scan -> col_ptr (int64); sorted off-diagonal records
//                            (row, contribution word) -> compact per-block scratch
//   numeric   3. emit        per output entry: gather the KE contributions in element order and sum
//                            them with numpy add.reduceat's rule v0 + (((v1 + v2) + v3) + ...)
//                            (bitwise equal to assemble.py:135); coalesced row_idx / vals stores
//
// Column c of the lower triangle holds rows {g_b : e incident to c, g_b >= c}; its triplet
// contributions are exactly the packed entries p = tri(max(a,b), min(a,b)) of the incident elements
// (a = local index of c).
//
// Fast-path limits (reported through the status word; the caller then uses the generic triplet
// path, which has none): node valence <= HX_MAX_NODE_DEGREE (8: hex meshes with regular vertices),
// distinct rows per column <= HX_MAX_COL_ROWS, no repeated node in an element.  With valence <= 8
// every duplicate run has <= 8 terms, where numpy's pairwise sum degenerates to the sequential sum
// implemented here.
#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "hx_common.cuh"
#include "hx_ke_device.cuh"

namespace hx {

constexpr int MAXDEG = HX_MAX_NODE_DEGREE;
constexpr int MAXR = HX_MAX_COL_ROWS;
constexpr int MAX_SEGS = 4;

struct SegTable {
    const int32_t *conn[MAX_SEGS];
    const double *ke[MAX_SEGS];
    int64_t conn_stride[MAX_SEGS];  // int32 units
    int64_t ke_stride[MAX_SEGS];    // doubles
    const int64_t *koff[MAX_SEGS];  // compact segments: first value of each element (null: dense rows)
    const uint64_t *kmask[MAX_SEGS];
    int64_t start[MAX_SEGS + 1];  // combined element index where segment s starts
    int n;
};

__device__ __forceinline__ int seg_of(const SegTable &T, int64_t e) {
    int s = 0;
#pragma unroll
    for (int q = 1; q < MAX_SEGS; ++q) s += (q < T.n && e >= T.start[q]) ? 1 : 0;
    return s;
}

// Element e's connectivity row; SINGLE: one dense segment (the single-GPU build).
template <bool SINGLE>
__device__ __forceinline__ const int32_t *conn_row(const SegTable &T, int64_t e) {
    if (SINGLE) return T.conn[0] + 8 * e;
    const int sg = seg_of(T, e);
    return T.conn[sg] + (e - T.start[sg]) * T.conn_stride[sg];
}

__device__ __forceinline__ void load_conn8(const int32_t *__restrict__ conn, int64_t e, int64_t stride,
                                           int32_t (&g)[8]) {
    const int4 *c4 = reinterpret_cast<const int4 *>(conn + e * stride);
    const int4 lo = __ldg(c4), hi = __ldg(c4 + 1);
    g[0] = lo.x; g[1] = lo.y; g[2] = lo.z; g[3] = lo.w;
    g[4] = hi.x; g[5] = hi.y; g[6] = hi.z; g[7] = hi.w;
}

// 1. adjacency: one thread per (element, local node); also validates node ids against [0, n_nodes).
// adj[(v - col_lo) * 8 + slot] = (combined element index << 3) | local node, slot from an atomic
// counter (slot order is arbitrary: the pattern pass sorts each node's list by element).
template <bool SINGLE>
__global__ void adjacency_kernel(SegTable T, int64_t n_total, int64_t n_nodes, int64_t col_lo, int64_t col_hi,
                                 int32_t *__restrict__ deg, int32_t *__restrict__ adj, uint32_t *__restrict__ status) {
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < 8 * n_total;
         w += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = w >> 3;
        const int a = (int)(w & 7);
        const int32_t v = __ldg(conn_row<SINGLE>(T, e) + a);
        if (v < 0 || (int64_t)v >= n_nodes) {
            atomicOr(status, HX_ST_BAD_INDEX);
            continue;
        }
        if (v >= col_lo && v < col_hi) {
            const int64_t c = v - col_lo;
            const int slot = atomicAdd(deg + c, 1);
            if (slot < MAXDEG) adj[8 * c + slot] = (int32_t)((e << 3) | a);
            else atomicOr(status, HX_ST_DEG_OVERFLOW);
        }
    }
}

// 1'. fixed-slot adjacency (HX_CSC_FIXED_ADJACENCY; single dense segment, every column): element e
// stores (e << 3 | a) into slot a of its local node a -- a plain store, no counter -- after the slots
// were emptied to -1.  Two elements holding one node at the same local index collide; the pattern
// pass counts the filled slots and the caller then re-runs with the atomic adjacency.
__global__ void adjacency_fixed_kernel(const int32_t *__restrict__ conn, int64_t n_total, int64_t n_nodes,
                                       int32_t *__restrict__ adj, uint32_t *__restrict__ status) {
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < 8 * n_total;
         w += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = __ldg(conn + w);
        if (v < 0 || (int64_t)v >= n_nodes) {
            atomicOr(status, HX_ST_BAD_INDEX);
            continue;
        }
        adj[8 * (int64_t)v + (w & 7)] = (int32_t)w;  // w = (e << 3) | a
    }
}

// Column processing order for non-local numberings (HX_CSC_ORDER_BY_ELEMENT): key = the column's
// lowest incident element (its adjacency slots), value = the column; sorting the pairs makes
// consecutive pattern/emit threads work on nearby elements (connectivity rows and KE values stay in
// L1/L2 instead of being gathered from random elements).
// FIXED: fixed-slot adjacency (slot = local node, empty = -1; see incident_sorted).
// Element numberings are banded too (a node's elements lie up to one element layer apart): with a
// band (band[0] = B elements, band[1] = strip width, B = 0: none) the key is the first element's
// position in the strip order of the elements (strip_pos, the inverse of band_col), so the columns
// that share a KE row are processed one strip -- not one element layer -- apart.
__device__ __forceinline__ uint32_t strip_pos(uint32_t e, uint32_t n, uint32_t B, uint32_t W) {
    const uint32_t rows = n / B;
    if (e >= rows * B) return e;
    const uint32_t z = e / B, r = e - z * B, s = r / W, w = min(W, B - s * W);
    return s * rows * W + z * w + (r - s * W);
}

template <bool FIXED>
__global__ void first_element_kernel(int64_t ncols, const int32_t *__restrict__ deg, const int32_t *__restrict__ adj,
                                     uint32_t empty_key, uint32_t *__restrict__ keys, uint32_t *__restrict__ cols,
                                     const int64_t *__restrict__ band) {
    const uint32_t B = (uint32_t)__ldg(band), W = (uint32_t)__ldg(band + 1);
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < ncols; c += (int64_t)gridDim.x * blockDim.x) {
        const int d = FIXED ? MAXDEG : min(__ldg(deg + c), MAXDEG);
        uint32_t k = empty_key;
        for (int j = 0; j < d; ++j) {
            const int32_t v = __ldg(adj + 8 * c + j);
            if (!FIXED || v >= 0) k = min(k, (uint32_t)(v >> 3));
        }
        keys[c] = B != 0u && k != empty_key ? strip_pos(k, empty_key, B, W) : k;
        cols[c] = (uint32_t)c;
    }
}

// Element band: median span (last - first incident element) of 1024 sampled columns; kept only when
// it holds at least four strips (band[0] = 0 otherwise).
template <bool FIXED>
__global__ void __launch_bounds__(256) element_band_kernel(int64_t ncols, const int32_t *__restrict__ deg,
                                                           const int32_t *__restrict__ adj, int64_t n_el,
                                                           int64_t strip, int64_t *__restrict__ band) {
    using Sort = cub::BlockRadixSort<int32_t, 256, 4>;
    __shared__ typename Sort::TempStorage tmp;
    __shared__ int32_t s_med;
    int32_t span[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t c = (int64_t)(threadIdx.x * 4 + i) * ncols / 1024;
        const int d = FIXED ? MAXDEG : min(__ldg(deg + c), MAXDEG);
        int32_t lo = INT32_MAX, hi = -1;
        for (int j = 0; j < d; ++j) {
            const int32_t v = __ldg(adj + 8 * c + j);
            if (!FIXED || v >= 0) {
                lo = min(lo, v >> 3);
                hi = max(hi, v >> 3);
            }
        }
        span[i] = hi >= 0 ? hi - lo : 0;
    }
    Sort(tmp).Sort(span);
    if (threadIdx.x == 128) s_med = span[0];  // rank 512 of 1024
    __syncthreads();
    if (threadIdx.x == 0) {
        const int64_t B = (int64_t)s_med;
        band[0] = B >= 4 * strip && 2 * B <= n_el ? B : 0;
        band[1] = strip;
    }
}

// Strip processing order for banded numberings (lexicographic structured meshes, RCM-like orders):
// an element's nodes lie up to one band B (~ one node layer) apart, so in column order a KE row's
// first and last columns are B columns -- a whole element layer of KE -- apart, more than the L2
// keeps.  Cutting every band-row into strips of W columns and walking strip by strip (row after row
// inside a strip) brings the two columns W apart.  band_kernel estimates B (median node span of 1024
// sampled elements) and switches the order on (*order_flag = 2) only when the band holds at least
// four strips (C4: B = 161k columns, 46 MB of KE per band-row; C3's 41k-column band stays in L2
// and keeps column order); band_order_kernel writes position -> column.  Any order gives the same CSC.
constexpr int BAND_SAMPLES = 1024;
__global__ void __launch_bounds__(256) band_kernel(const int32_t *__restrict__ conn, int64_t n_el, int64_t ncols,
                                                   int64_t strip, uint32_t *__restrict__ order_flag,
                                                   int64_t *__restrict__ band) {
    using Sort = cub::BlockRadixSort<int32_t, 256, BAND_SAMPLES / 256>;
    __shared__ typename Sort::TempStorage tmp;
    __shared__ int32_t s_med;
    int32_t span[BAND_SAMPLES / 256];
#pragma unroll
    for (int i = 0; i < BAND_SAMPLES / 256; ++i) {
        const int64_t e = (int64_t)(threadIdx.x * (BAND_SAMPLES / 256) + i) * n_el / BAND_SAMPLES;
        const int4 a = __ldg(reinterpret_cast<const int4 *>(conn + 8 * e));
        const int4 b = __ldg(reinterpret_cast<const int4 *>(conn + 8 * e) + 1);
        const int32_t mn = min(min(min(a.x, a.y), min(a.z, a.w)), min(min(b.x, b.y), min(b.z, b.w)));
        const int32_t mx = max(max(max(a.x, a.y), max(a.z, a.w)), max(max(b.x, b.y), max(b.z, b.w)));
        span[i] = mx - mn;
    }
    Sort(tmp).Sort(span);  // blocked arrangement: thread t holds ranks 4t .. 4t + 3
    if (threadIdx.x == BAND_SAMPLES / 2 / (BAND_SAMPLES / 256)) s_med = span[0];
    __syncthreads();
    if (threadIdx.x == 0) {
        const int64_t B = (int64_t)s_med;
        band[0] = B;
        band[1] = strip;
        if (B >= 4 * strip && 2 * B <= ncols) *order_flag = 2u;
    }
}

// Column at processing position i of the strip order (band[0] = B, band[1] = strip width; columns < 2^31).
__device__ __forceinline__ int64_t band_col(int64_t i64, int64_t ncols, const int64_t *__restrict__ band) {
    const uint32_t B = (uint32_t)__ldg(band), strip = (uint32_t)__ldg(band + 1), i = (uint32_t)i64;
    const uint32_t rows = (uint32_t)ncols / B;
    if (i >= rows * B) return i64;  // the partial last band-row keeps column order at the end
    const uint32_t s = i / (rows * strip), rel = i - s * rows * strip;
    const uint32_t w = min(strip, B - s * strip);
    const uint32_t z = rel / w;
    return (int64_t)(z * B + s * strip + (rel - z * w));
}

// The strip order as an order array (position -> column), read like the element order.  Computing
// band_col inline in the pattern pass instead measured 1.9 ms slower at C4 (7.8 vs 5.9 ms).
__global__ void band_order_kernel(int64_t ncols, const uint32_t *__restrict__ order_flag,
                                  const int64_t *__restrict__ band, uint32_t *__restrict__ order) {
    if (*order_flag != 2u) return;
    // four positions per thread, one 16-byte store: inside a strip row consecutive positions map to
    // consecutive columns, so the map is evaluated at the ends only (order is 256-byte aligned)
    const int64_t n4 = ncols / 4;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n4; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = 4 * q;
        const uint32_t c0 = (uint32_t)band_col(i, ncols, band), c3 = (uint32_t)band_col(i + 3, ncols, band);
        uint4 v;
        if (c3 == c0 + 3u) {
            v = make_uint4(c0, c0 + 1u, c0 + 2u, c3);
        } else {
            v = make_uint4(c0, (uint32_t)band_col(i + 1, ncols, band), (uint32_t)band_col(i + 2, ncols, band), c3);
        }
        reinterpret_cast<uint4 *>(order)[q] = v;
    }
    if (blockIdx.x == 0 && threadIdx.x < (unsigned)(ncols - 4 * n4))
        order[4 * n4 + threadIdx.x] = (uint32_t)band_col(4 * n4 + threadIdx.x, ncols, band);
}

// Sorting network for 8 keys (19 compare-exchanges), padded with INT_MAX.
__device__ __forceinline__ void cswap(int32_t &a, int32_t &b) {
    const int32_t lo = min(a, b), hi = max(a, b);
    a = lo;
    b = hi;
}
__device__ __forceinline__ void sort8(int32_t (&v)[8]) {
    cswap(v[0], v[1]); cswap(v[2], v[3]); cswap(v[4], v[5]); cswap(v[6], v[7]);
    cswap(v[0], v[2]); cswap(v[1], v[3]); cswap(v[4], v[6]); cswap(v[5], v[7]);
    cswap(v[1], v[2]); cswap(v[5], v[6]); cswap(v[0], v[4]); cswap(v[3], v[7]);
    cswap(v[1], v[5]); cswap(v[2], v[6]);
    cswap(v[1], v[4]); cswap(v[3], v[6]);
    cswap(v[2], v[4]); cswap(v[3], v[5]);
    cswap(v[3], v[4]);
}

// Incident elements of column cl, sorted by element id (= the stable triplet order).
// Returns deg, or -1 with a status bit when the column is outside the fast path.
// FIXED: the adjacency was recorded by the integration kernel in fixed slots -- element e stores
// (e << 3 | a) in slot a of its local node a, empty slots hold -1 -- so deg is the number of
// filled slots; it is written to deg_arr (the emit pass reads it) and summed into *slot_total
// (two elements claiming one slot lose an entry; the build detects that from the total).
template <bool FIXED>
__device__ __forceinline__ int incident_sorted(int64_t cl, int32_t *__restrict__ deg_arr,
                                               const int32_t *__restrict__ adj, int32_t (&ent)[8],
                                               uint32_t *__restrict__ status) {
    int deg = 0;
    if (FIXED) {
        const int4 *a4 = reinterpret_cast<const int4 *>(adj + 8 * cl);
        const int4 lo = a4[0], hi = a4[1];
        const int32_t v[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            ent[k] = v[k] >= 0 ? v[k] : INT32_MAX;
            deg += v[k] >= 0;
        }
    } else {
        deg = __ldg(deg_arr + cl);
        if (deg > MAXDEG) return -1;  // flagged by the adjacency pass
#pragma unroll
        for (int k = 0; k < 8; ++k) ent[k] = k < deg ? __ldg(adj + 8 * cl + k) : INT32_MAX;
    }
    sort8(ent);
#pragma unroll
    for (int k = 1; k < 8; ++k) {
        if (k < deg && (ent[k] >> 3) == (ent[k - 1] >> 3)) {
            atomicOr(status, HX_ST_REPEATED_NODE);
            return -1;
        }
    }
    return deg;
}

#ifndef HX_RECORDS_UNROLL
#define HX_RECORDS_UNROLL 4
#endif
constexpr int RECORDS_UNROLL = HX_RECORDS_UNROLL;  // the pattern pass's record loop
constexpr int MAX_OFFDIAG_CONTRIB = 4;     // hex meshes: an edge is shared by at most 4 elements
#ifndef HX_COL_BLOCK
#define HX_COL_BLOCK 64
#endif
#ifndef HX_EMIT_BLOCK
#define HX_EMIT_BLOCK 128
#endif
#ifndef HX_BAND_STRIP_DEFAULT
#define HX_BAND_STRIP_DEFAULT 16384  // measured best of 4K..64K at C4 (profiles/r02/band_order_sweep.txt)
#endif
constexpr int COL_BLOCK = HX_COL_BLOCK;    // columns per tile (pattern: one thread per column)
constexpr int EMIT_BLOCK = HX_EMIT_BLOCK;  // emit: threads per tile
static_assert(COL_BLOCK % 32 == 0 && COL_BLOCK <= 256, "tile = 1..8 warps of columns");

// Bitonic sorting network on N register-resident keys, ascending.
template <int N, typename K>
__device__ __forceinline__ void bitonic_sort(K (&v)[N]) {
#pragma unroll
    for (int k = 2; k <= N; k <<= 1)
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
            for (int i = 0; i < N; ++i) {
                const int l = i ^ j;
                if (l > i) {
                    const K a = v[i], b = v[l];
                    const bool up = (i & k) == 0;
                    v[i] = up ? min(a, b) : max(a, b);
                    v[l] = up ? max(a, b) : min(a, b);
                }
            }
}

// Sort-based pattern of one column: every contribution (k, b) of an
// incident element k whose node v = g[k][b] lies below the diagonal becomes one key
// (v << 6 | k << 3 | b), appended branch-free to the thread's list L; a 16/32/64-key register
// network (warp-uniform choice) sorts them, so equal rows form runs whose contributions are already
// in element order.  (Replaced a 32-slot hash set in round 1: its data-dependent probe loops were
// half its instructions and most of its divergence.)  Returns m = 1 + distinct rows (0 for an
// empty column or one outside the fast path) and cnt = keys left sorted in L.
constexpr int SORT_SLOTS = 64;  // <= 8 elements x 7 other nodes = 56 contributions per column

// Batcher's odd-even merge sort on N register-resident keys, ascending (N = 16/32/64: 63/191/543
// compare-exchanges against the bitonic network's 80/240/672).  HX_PATTERN_NET: 1 = odd-even
// merge, 0 = bitonic.
#ifndef HX_PATTERN_NET
#define HX_PATTERN_NET 1
#endif
// Network tiers of the pattern pass (warp-uniform: the smallest tier that holds every lane's keys).
// Interior columns of hex meshes hold exactly 28 keys, so the default tiers are 28 (the 32-key
// odd-even network pruned to 28 wires: 162 instead of 191 compare-exchanges -- valid because the
// pruned wires would hold +inf), 32 and 64; a 16-key tier costs instruction-cache room for the few
// warps of boundary columns (C4 pattern 5.90 -> 5.78 ms, C5 unchanged; profiles/r02/pattern_net28_probe.txt).
#ifndef HX_PATTERN_NET16
#define HX_PATTERN_NET16 0
#endif
#ifndef HX_PATTERN_NET28
#define HX_PATTERN_NET28 1
#endif
template <int N>
struct OddEvenPairs {  // comparator list of the network, built at compile time
    static constexpr int count() {
        int c = 0;
        for (int p = 1; p < N; p <<= 1)
            for (int k = p; k >= 1; k >>= 1)
                for (int j = k % p; j + k < N; j += 2 * k)
                    for (int i = 0; i < k && i + j + k < N; ++i)
                        if ((i + j) / (2 * p) == (i + j + k) / (2 * p)) ++c;
        return c;
    }
    int lo[count()], hi[count()];
    constexpr OddEvenPairs() : lo(), hi() {
        int c = 0;
        for (int p = 1; p < N; p <<= 1)
            for (int k = p; k >= 1; k >>= 1)
                for (int j = k % p; j + k < N; j += 2 * k)
                    for (int i = 0; i < k && i + j + k < N; ++i)
                        if ((i + j) / (2 * p) == (i + j + k) / (2 * p)) {
                            lo[c] = i + j;
                            hi[c] = i + j + k;
                            ++c;
                        }
    }
};

template <int N, typename K>
__device__ __forceinline__ void oddeven_merge_sort(K (&v)[N]) {
    constexpr OddEvenPairs<N> P{};
#pragma unroll
    for (int c = 0; c < OddEvenPairs<N>::count(); ++c) {
        const K a = v[P.lo[c]], b = v[P.hi[c]];
        v[P.lo[c]] = min(a, b);
        v[P.hi[c]] = max(a, b);
    }
}

// Sort the first n (<= N) contribution keys of L in place and, while they are in registers, count
// the distinct rows (key >> 6) and check that no row has more than MAX_OFFDIAG_CONTRIB
// contributions (sorted: a run of 5 has v[q] and v[q - 4] in the same row).
template <int N, typename K>
__device__ __forceinline__ void sort_count(K *L, int n, int &rows, bool &ok) {
    K v[N];
#pragma unroll
    for (int q = 0; q < N; ++q) v[q] = q < n ? L[q * COL_BLOCK] : (K)~(K)0;
    if (HX_PATTERN_NET) oddeven_merge_sort<N, K>(v);
    else bitonic_sort<N, K>(v);
    rows = 0;
    ok = true;
#pragma unroll
    for (int q = 0; q < N; ++q) {
        if (q < n) L[q * COL_BLOCK] = v[q];
        const K r = v[q] >> 6;
        rows += q < n && (q == 0 || r != (v[q > 0 ? q - 1 : 0] >> 6));
        if (q >= MAX_OFFDIAG_CONTRIB) ok &= !(q < n && r == (v[q >= MAX_OFFDIAG_CONTRIB ? q - MAX_OFFDIAG_CONTRIB : 0] >> 6));
    }
}

template <typename K, bool SINGLE, bool FIXED>
__device__ __forceinline__ int column_pattern_sort(const SegTable &T, bool active, int64_t cl, int32_t c,
                                                   int32_t *__restrict__ deg_arr, const int32_t *__restrict__ adj,
                                                   int32_t *__restrict__ ent_out, K *L, int &cnt, int &deg,
                                                   int32_t &last, uint32_t *__restrict__ status) {
    int m = 0;
    deg = 0;
    last = -1;
    int32_t ent[8];
    cnt = 0;
    if (active) {
        deg = incident_sorted<FIXED>(cl, deg_arr, adj, ent, status);
        if (deg < 0) deg = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (k < deg) last = max(last, ent[k] >> 3);
        if (deg > 0) {  // the emit pass reads the sorted incident list (processing order)
            int4 *a4 = reinterpret_cast<int4 *>(ent_out);
            a4[0] = make_int4(ent[0], ent[1], ent[2], ent[3]);
            a4[1] = make_int4(ent[4], ent[5], ent[6], ent[7]);
        }
    }
    if (deg > 0) {
        int32_t g[8][8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (k < deg) {
                const int4 *c4 = reinterpret_cast<const int4 *>(conn_row<SINGLE>(T, ent[k] >> 3));
                const int4 lo = __ldg(c4), hi = __ldg(c4 + 1);
                g[k][0] = lo.x; g[k][1] = lo.y; g[k][2] = lo.z; g[k][3] = lo.w;
                g[k][4] = hi.x; g[k][5] = hi.y; g[k][6] = hi.z; g[k][7] = hi.w;
            } else {
#pragma unroll
                for (int b = 0; b < 8; ++b) g[k][b] = -1;  // never a row (< c)
            }
        }
        // node ids and c are in [0, 2^31): v > c <=> the sign bit of c - v (no overflow)
#pragma unroll
        for (int k = 0; k < 8; ++k)
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const int32_t v = g[k][b];
                L[cnt * COL_BLOCK] = ((K)(uint32_t)v << 6) | (K)(k * 8 + b);  // kept only when v > c
                cnt += (int)((uint32_t)(c - v) >> 31);
            }
        const unsigned am = __activemask();
        // distinct rows; a row with more than MAX_OFFDIAG_CONTRIB contributions leaves the fast path
        int rows = 0;
        bool ok = true;
        if (HX_PATTERN_NET16 && !__any_sync(am, cnt > 16)) sort_count<16, K>(L, cnt, rows, ok);
        else if (HX_PATTERN_NET28 && !__any_sync(am, cnt > 28)) sort_count<28, K>(L, cnt, rows, ok);
        else if (!__any_sync(am, cnt > 32)) sort_count<32, K>(L, cnt, rows, ok);
        else sort_count<64, K>(L, cnt, rows, ok);
        if (!ok || rows > MAXR) {
            atomicOr(status, HX_ST_ROW_OVERFLOW);
            cnt = 0;
        } else {
            m = 1 + rows;
        }
    }
    return m;
}

// 2. Pattern pass: one thread per column, COL_BLOCK columns per block (column_pattern_sort):
//   - incident elements sorted by id, written with the column's degree by processing position
//     (over the adjacency in column order; separate arrays for element-ordered builds, so the emit
//     pass reads them contiguously instead of gathering them column by column);
//   - contribution keys (row << 6 | k << 3 | b) sorted by a 16/32/64-key register network;
//   - m = 1 + distinct rows -> col_ptr[cl] (the exclusive scan turns counts into offsets);
//   - runs of equal rows -> off-diagonal records (row, contribution word) in a compact scratch
//     region reserved per block with one atomic (every block records where its records start);
//   - tile_need[block] = 1 + the highest incident element of the tile (the fused kernel's wait).
#ifndef HX_PATTERN_MIN_BLOCKS
#define HX_PATTERN_MIN_BLOCKS 10  // 96 registers: 10 x 64-thread tiles per SM (measured best of 1, 10, 12)
#endif
template <typename K, bool SINGLE, bool FIXED>
__global__ void __launch_bounds__(COL_BLOCK, HX_PATTERN_MIN_BLOCKS)
pattern_kernel(SegTable T, int64_t col_lo, int64_t ncols, int32_t *__restrict__ deg_arr,
               int32_t *__restrict__ adj, int64_t *__restrict__ col_ptr, int2 *__restrict__ scratch,
               int64_t scratch_capacity, unsigned long long *__restrict__ scratch_top,
               int64_t *__restrict__ block_scratch, uint32_t *__restrict__ status,
               const uint32_t *__restrict__ order, unsigned long long *__restrict__ slot_total,
               int32_t *__restrict__ tile_need, int32_t *__restrict__ tadj, int32_t *__restrict__ tdeg,
               const uint32_t *__restrict__ order_flag) {
    __shared__ K sL[SORT_SLOTS * COL_BLOCK];  // this thread's contribution keys, [slot][thread]
    __shared__ unsigned long long s_base;
    using BlockScan = cub::BlockScan<int32_t, COL_BLOCK>;
    __shared__ typename BlockScan::TempStorage scan_tmp;
    const int t = threadIdx.x;
    const int64_t idx = (int64_t)blockIdx.x * COL_BLOCK + t;  // position in the processing order
    // 0: column order; 1: element order; 2: strip order of a banded numbering (both: the order array)
    const uint32_t flag = order != nullptr ? __ldg(order_flag) : 0u;
    if (flag == 0u) order = nullptr;
    const int64_t cl = flag == 0u || idx >= ncols ? idx : (int64_t)__ldg(order + idx);
    const int32_t c = (int32_t)(col_lo + cl);
    K *L = sL + t;
    int cnt = 0, deg = 0;
    int32_t last = -1;
    // sorted incident lists and degrees in processing order (in place over adj / deg in column order)
    int32_t *ent_out = (order != nullptr ? tadj : adj) + 8 * idx;
    const int m = column_pattern_sort<K, SINGLE, FIXED>(T, cl < ncols, cl, c, deg_arr, adj, ent_out, L, cnt, deg, last,
                                                        status);
    if (cl < ncols) (order != nullptr ? tdeg : deg_arr)[idx] = deg;
    {  // elements the tile's emit needs: every incident element < tile_need (the fused kernel waits for them)
        const int need = __reduce_max_sync(0xffffffffu, last + 1);
        if ((t & 31) == 0) atomicMax(tile_need + blockIdx.x, need);
    }
    if (cl < ncols) col_ptr[cl] = m;
    if (FIXED) {
        const unsigned filled = __reduce_add_sync(0xffffffffu, (unsigned)deg);
        if ((t & 31) == 0 && filled) atomicAdd(slot_total, (unsigned long long)filled);
    }

    // compact scratch: this block's off-diagonal records
    int excl, total;
    const int off = m > 0 ? m - 1 : 0;
    BlockScan(scan_tmp).ExclusiveSum(off, excl, total);
    if (t == 0) {
        s_base = atomicAdd(scratch_top, (unsigned long long)total);
        block_scratch[blockIdx.x] = (int64_t)s_base;
    }
    __syncthreads();
    const int64_t sb = (int64_t)s_base + excl;
    if (sb + off > scratch_capacity) {
        if (off > 0) atomicOr(status, HX_ST_SCRATCH_OVERFLOW);
        return;
    }
    // runs of equal rows -> records (row, count | (k, b) pairs in element order)
    int2 *out = scratch + sb - 1;  // record j of this column at out[j + 1]; j = -1 before the first
    int j = -1, shift = 3;
    K prev = ~(K)0;
    uint32_t word = 0;
#pragma unroll RECORDS_UNROLL
    for (int q = 0; q < cnt; ++q) {
        const K key = L[q * COL_BLOCK];
        const K v = key >> 6;
        const uint32_t kb = (uint32_t)key & 63u;
        const bool head = v != prev;
        if (head && j >= 0) out[j + 1] = make_int2((int)prev, (int)word);
        j += head;
        word = head ? (1u | (kb << 3)) : ((word + 1u) | (kb << shift));
        shift = head ? 9 : shift + 6;
        prev = v;
    }
    if (j >= 0) out[j + 1] = make_int2((int)prev, (int)word);
}

// Fixed-slot adjacency check: every (element, local node) pair must have landed in its own slot.
__global__ void slot_check_kernel(const unsigned long long *__restrict__ slot_total, int64_t n_total,
                                  uint32_t *__restrict__ status) {
    if (threadIdx.x == 0 && blockIdx.x == 0 && *slot_total != 8ull * (unsigned long long)n_total)
        atomicOr(status, HX_ST_SLOT_COLLISION);
}

// 6. Emit pass: block b re-walks the output entries of the same COL_BLOCK columns (coalesced
// scratch reads, row_idx / vals stores).  Diagonals first (one per column: every incident element
// at its own local node), then the off-diagonal scratch records in output order.  Values are
// gathered from the KE rows and reduced with numpy add.reduceat's rule v0 + (((v1 + v2) + v3) + ...).
// SINGLE: one dense element segment (the single-GPU build) -> KE row = ke + 36 e.
template <bool SINGLE>
__device__ __forceinline__ const double *ke_row(const SegTable &T, int64_t e) {
    if (SINGLE) return T.ke[0] + 36 * e;
    const int sg = seg_of(T, e);
    return T.ke[sg] + T.ke_stride[sg] * (e - T.start[sg]);
}

// Address of packed entry p of element e: a dense row, or a compact (received) element's p-th set
// entry -- ke + ke_offset[e] + (owned entries below p).
template <bool SINGLE>
__device__ __forceinline__ const double *ke_entry(const SegTable &T, int64_t e, int p) {
    if (SINGLE) return T.ke[0] + 36 * e + p;
    const int sg = seg_of(T, e);
    const int64_t le = e - T.start[sg];
    if (T.koff[sg] != nullptr) {
        const uint64_t m = __ldg(reinterpret_cast<const unsigned long long *>(T.kmask[sg]) + le);
        return T.ke[sg] + __ldg(reinterpret_cast<const long long *>(T.koff[sg]) + le) +
               __popcll(m & ((1ull << p) - 1ull));
    }
    return T.ke[sg] + T.ke_stride[sg] * le + p;
}

// KE gathers of the emit pass.  Each KE row is read by the columns of its element's 8 nodes, up to
// one node layer apart; HX_EMIT_KE_HINT 1 marks those loads L2 evict_last (the streamed scratch
// loads and CSC stores are evict-first) so the rows survive until their last column.
#ifndef HX_EMIT_KE_HINT
#define HX_EMIT_KE_HINT 1  // evict_last: -0.2..-0.45 ms at C4 with the strip order (profiles/r02/emit_variants.txt)
#endif
__device__ __forceinline__ uint64_t ke_policy() {
    uint64_t p = 0;
#if HX_EMIT_KE_HINT >= 1
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
#endif
    return p;
}
template <bool LOAD_CG>
__device__ __forceinline__ double ke_load(const double *ptr, uint64_t pol) {
    if (LOAD_CG) return __ldcg(ptr);
#if HX_EMIT_KE_HINT == 1
    double v;
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(ptr), "l"(pol));
    return v;
#elif HX_EMIT_KE_HINT == 2
    double v;
    asm("ld.global.nc.L2::cache_hint.L2::256B.f64 %0, [%1], %2;" : "=d"(v) : "l"(ptr), "l"(pol));
    return v;
#else
    (void)pol;
    return __ldg(ptr);
#endif
}

// Shared state of one emit tile (aliases the integration warp's staging in the fused kernel).
struct EmitSmem {
    int64_t s_start[COL_BLOCK];       // first output entry of each column of the tile
    int32_t s_m[COL_BLOCK + 1];       // entries per column
    int32_t s_cl[COL_BLOCK];          // column (block-local index) of each tile position
    int32_t s_rs[COL_BLOCK + 1];      // first scratch record of each column (tile-relative)
    int32_t s_deg[COL_BLOCK];
    int32_t s_adj[COL_BLOCK * 9];     // the tile's sorted incident lists, stride 9 (the diagonal pass reads
                                      // one list per lane: conflict-free)
    uint8_t s_col[COL_BLOCK * MAXR];  // tile position of each off-diagonal record
};

// Arguments of the emit pass over one column range (the pattern pass's workspace + outputs).
struct EmitArgs {
    SegTable T;
    int64_t col_lo, ncols;
    const int32_t *deg_arr, *adj;    // column order (in-place lists of the pattern pass)
    const int32_t *tdeg, *tadj;      // processing order (element-ordered builds)
    const int64_t *col_ptr;
    const int2 *scratch;
    const int64_t *block_scratch;
    int64_t *row_idx;
    double *vals;
    int64_t capacity;
    const uint32_t *order_flag, *order;
};

constexpr uint32_t HX_ST_EMIT_SKIP =
    HX_ST_DEG_OVERFLOW | HX_ST_ROW_OVERFLOW | HX_ST_REPEATED_NODE | HX_ST_SCRATCH_OVERFLOW | HX_ST_SLOT_COLLISION;

template <int NT>
__device__ __forceinline__ void tile_sync() {
    if (NT == 32) __syncwarp();
    else __syncthreads();
}

// Emit tile `tile` (COL_BLOCK columns of the processing order) with NT threads (tid = 0..NT-1):
// row_idx / vals of its columns.  LOAD_CG: KE gathers through L2 only (the fused kernel reads KE
// rows that other SMs stored during the same launch).
template <int NT, bool ROWS, bool VALS, bool SINGLE, bool LOAD_CG>
__device__ __forceinline__ void emit_tile(EmitSmem &S, const EmitArgs &A, int64_t tile, int tid) {
    const SegTable &T = A.T;
    const int64_t col_lo = A.col_lo, ncols = A.ncols, capacity = A.capacity;
    const int32_t *__restrict__ deg_arr = A.deg_arr;
    const int32_t *__restrict__ adj = A.adj;
    const int64_t *__restrict__ col_ptr = A.col_ptr;
    const int2 *__restrict__ scratch = A.scratch;
    const int64_t *__restrict__ block_scratch = A.block_scratch;
    int64_t *__restrict__ row_idx = A.row_idx;
    double *__restrict__ vals = A.vals;
    const uint32_t *__restrict__ order_flag = A.order_flag;
    const uint32_t *__restrict__ order = A.order;
    const bool ordered = *order_flag != 0u;
    // the pattern pass wrote the sorted incident lists / degrees by processing position
    const int32_t *__restrict__ deg_list = ordered ? A.tdeg : deg_arr;
    const int32_t *__restrict__ adj_list = ordered ? A.tadj : adj;
    const uint64_t pol = ke_policy();
    const int64_t first = tile * COL_BLOCK;
    const int ncol = (int)(ncols - first < COL_BLOCK ? ncols - first : COL_BLOCK);
    for (int u = tid; u < ncol; u += NT) {
        const int64_t cl = ordered ? (int64_t)__ldg(order + first + u) : first + u;
        S.s_cl[u] = (int32_t)cl;
        const int64_t a = col_ptr[cl], b = col_ptr[cl + 1];
        S.s_start[u] = a;
        S.s_m[u] = (int)(b - a);
        S.s_deg[u] = min(deg_list[first + u], MAXDEG);
    }
    tile_sync<NT>();
    if (VALS)
        for (int i = tid; i < ncol * 8; i += NT)
            S.s_adj[(i >> 3) * 9 + (i & 7)] = __ldg(adj_list + 8 * first + i);  // contiguous: lists are in processing order
    // scratch record offsets: column u has max(m_u - 1, 0) records (m_u = 0 for a node no element
    // references), laid out in tile order by the pattern pass -- warp 0 scans them
    if (tid < 32) {
        constexpr int PER = COL_BLOCK / 32;  // columns per lane, consecutive
        const int l = tid;
        int off[PER], sum = 0;
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int u = PER * l + i;
            const int m = u < ncol ? S.s_m[u] : 0;
            off[i] = m > 0 ? m - 1 : 0;
            sum += off[i];
        }
        int incl = sum;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, d);
            if (l >= d) incl += v;
        }
        int run = incl - sum;
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            S.s_rs[PER * l + i] = run;
            run += off[i];
        }
        if (l == 31) S.s_rs[COL_BLOCK] = incl;
    }
    tile_sync<NT>();
    const int64_t sb = block_scratch[tile];
    const int n_off = S.s_rs[COL_BLOCK];
    for (int u = tid; u < ncol; u += NT)
        for (int q = S.s_rs[u]; q < S.s_rs[u] + S.s_m[u] - 1; ++q) S.s_col[q] = (uint8_t)u;
    tile_sync<NT>();
    // diagonals
    for (int u = tid; u < ncol; u += NT) {
        const int64_t o = S.s_start[u];
        if (S.s_m[u] == 0 || o >= capacity) continue;
        if (ROWS) __stcs(reinterpret_cast<long long *>(row_idx) + o, (long long)(col_lo + S.s_cl[u]));
        if (!VALS) continue;
        const int deg = S.s_deg[u];
        const int32_t *ent = S.s_adj + 9 * u;
        double x[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            x[k] = 0.0;
            if (k < deg) {
                const int32_t en = ent[k];
                const int a = en & 7;
                x[k] = ke_load<LOAD_CG>(ke_entry<SINGLE>(T, en >> 3, pack_index(a, a)), pol);
            }
        }
        double v = x[0];
        if (deg >= 2) {
            double sum = x[1];
#pragma unroll
            for (int k = 2; k < 8; ++k)
                if (k < deg) sum = __dadd_rn(sum, x[k]);
            v = __dadd_rn(x[0], sum);
        }
        __stcs(vals + o, v);
    }
    // off-diagonals: record q of tile position u is output entry S.s_start[u] + 1 + (q - S.s_rs[u]).
    // Two records per thread per iteration: their KE gathers are independent and overlap.
    auto offdiag_value = [&](int u, uint32_t w) -> double {
        const int n = (int)(w & 7u);
        const int32_t *ent = S.s_adj + 9 * u;
        double x[MAX_OFFDIAG_CONTRIB];
#pragma unroll
        for (int r = 0; r < MAX_OFFDIAG_CONTRIB; ++r) {
            x[r] = 0.0;
            if (r < n) {
                const uint32_t kb = (w >> (3 + 6 * r)) & 63u;
                const int32_t en = ent[kb >> 3];
                const int a = en & 7, b = (int)(kb & 7u);
                x[r] = ke_load<LOAD_CG>(ke_entry<SINGLE>(T, en >> 3, pack_index(max(a, b), min(a, b))), pol);
            }
        }
        double v = x[0];
        if (n >= 2) {
            double sum = x[1];
#pragma unroll
            for (int r = 2; r < MAX_OFFDIAG_CONTRIB; ++r)
                if (r < n) sum = __dadd_rn(sum, x[r]);
            v = __dadd_rn(x[0], sum);
        }
        return v;
    };
#ifndef HX_EMIT_UNROLL
#define HX_EMIT_UNROLL 4
#endif
    constexpr int R = HX_EMIT_UNROLL;  // records in flight per thread: their loads/gathers overlap
    for (int q0 = tid; q0 < n_off; q0 += R * NT) {
        int u[R];
        int64_t o[R];
        int2 rec[R];
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const int q = q0 + i * NT;
            const bool has = q < n_off;
            u[i] = has ? S.s_col[q] : 0;
            o[i] = has ? S.s_start[u[i]] + 1 + (q - S.s_rs[u[i]]) : capacity;
            rec[i] = has ? __ldcs(scratch + sb + q) : make_int2(0, 0);  // streamed once: evict first
        }
        if (ROWS) {
#pragma unroll
            for (int i = 0; i < R; ++i)
                if (o[i] < capacity) __stcs(reinterpret_cast<long long *>(row_idx) + o[i], (long long)rec[i].x);
        }
        if (!VALS) continue;
        double v[R];
#pragma unroll
        for (int i = 0; i < R; ++i) v[i] = o[i] < capacity ? offdiag_value(u[i], (uint32_t)rec[i].y) : 0.0;
#pragma unroll
        for (int i = 0; i < R; ++i)
            if (o[i] < capacity) __stcs(vals + o[i], v[i]);  // beyond capacity: the caller retries
    }
}

template <int NT, bool ROWS, bool VALS, bool SINGLE>
__global__ void __launch_bounds__(NT)
emit_kernel(EmitArgs A, const uint32_t *__restrict__ status) {
    // the pattern pass hit a fast-path limit: its records are incomplete and the caller re-runs
    if (*status & HX_ST_EMIT_SKIP) return;
    __shared__ EmitSmem S;
    emit_tile<NT, ROWS, VALS, SINGLE, false>(S, A, blockIdx.x, threadIdx.x);
}

// ---------------------------------------------------------------------------------------------
// 7. Integration fused with the emit pass (hx_integrate_emit).  The integration kernel's persistent
// warps (hx_ke_device.cuh) run the emit tiles between their element quads: after every quad a warp
// bumps its chunk's completion counter and, when the next emit tile (processing order) has every
// incident element integrated -- tile_need from the pattern pass against the chunk counters -- it
// claims the tile and emits it from the KE rows still in L2.  Once the quads are exhausted the warps
// drain the remaining tiles, waiting for their chunks.  Deadlock-free: a warp waits only after its
// own quads are done, and every quad it waits for has been claimed by a warp that never waits
// before finishing it.  Same arithmetic as the separate kernels, so the results are bitwise equal.
constexpr int FUSED_CHUNK_QUADS = 32;  // one completion counter per 32 quads (128 elements)

struct FusedSched {
    unsigned *done;             // per chunk: quads integrated
    unsigned *wm;               // chunks known complete (monotone hint)
    unsigned *tile_head;        // next emit tile of the processing order
    const int32_t *tile_need;   // per tile: elements that must be integrated first
    int64_t n_quads, n_chunks, n_tiles, n_el;
};

struct EmitHook {
    EmitSmem *S;
    const EmitArgs *A;
    FusedSched sc;
    int lane;
    bool emit;

    // lane 0: are elements [0, need_el) integrated (their KE rows stored)?
    __device__ __forceinline__ bool chunks_ready(int64_t need_el) {
        need_el = need_el < sc.n_el ? need_el : sc.n_el;
        const int64_t cneed = (need_el + 4 * FUSED_CHUNK_QUADS - 1) / (4 * FUSED_CHUNK_QUADS);
        unsigned w = *(volatile unsigned *)sc.wm;
        if (w >= cneed) return true;
        const unsigned w0 = w;
        while (w < cneed) {
            const unsigned full = w == sc.n_chunks - 1 ? (unsigned)(sc.n_quads - (int64_t)w * FUSED_CHUNK_QUADS)
                                                       : (unsigned)FUSED_CHUNK_QUADS;
            if (*(volatile unsigned *)(sc.done + w) < full) break;
            ++w;
        }
        if (w > w0) atomicMax(sc.wm, w);
        return w >= cneed;
    }
    __device__ __forceinline__ void run_tile(int64_t t) {
        __threadfence();  // the counted quads' KE stores before this tile's (L2) loads
        __syncwarp();
        emit_tile<32, true, true, true, true>(*S, *A, t, lane);
        __syncwarp();  // the staging buffer is the integration's again
    }
    __device__ __forceinline__ void after_quad(int64_t q) {
        __threadfence();  // this quad's KE / iK / jK stores before its completion count
        __syncwarp();
        if (lane == 0) atomicAdd(sc.done + q / FUSED_CHUNK_QUADS, 1u);
        if (!emit) return;
#pragma unroll 1
        for (int it = 0; it < 2; ++it) {  // at most two ready tiles between quads
            long long t = -1;
            if (lane == 0) {
                const unsigned h = *(volatile unsigned *)sc.tile_head;
                if (h < sc.n_tiles && chunks_ready(__ldg(sc.tile_need + h)) && atomicCAS(sc.tile_head, h, h + 1) == h)
                    t = h;
            }
            t = __shfl_sync(0xffffffffu, t, 0);
            if (t < 0) return;
            run_tile(t);
        }
    }
    __device__ __forceinline__ void drain() {
        if (!emit) return;
#pragma unroll 1
        while (true) {
            unsigned h = 0;
            if (lane == 0) h = atomicAdd(sc.tile_head, 1u);
            h = __shfl_sync(0xffffffffu, h, 0);
            if (h >= sc.n_tiles) return;
            if (lane == 0) {
                const int32_t need = __ldg(sc.tile_need + h);
                while (!chunks_ready(need)) __nanosleep(256);
            }
            __syncwarp();
            run_tile(h);
        }
    }
};

static_assert(sizeof(EmitSmem) <= sizeof(GpWarpSmem), "the emit tile aliases the warp's integration staging");
constexpr size_t FUSED_SMEM = GP_WARPS * sizeof(GpWarpSmem);

template <int MODE, bool WITH_INDEX>
__global__ void __launch_bounds__(GP_BLOCK, HX_KE_MIN_BLOCKS)
integrate_emit_kernel(const double *__restrict__ coords, int64_t n_nodes, const int32_t *__restrict__ conn,
                      const double *__restrict__ coeff, int64_t n, double *__restrict__ ke_out,
                      int32_t *__restrict__ rows_out, int32_t *__restrict__ cols_out,
                      unsigned long long *__restrict__ fail_min, unsigned *__restrict__ quad_counter, EmitArgs A,
                      FusedSched sc, const uint32_t *__restrict__ status) {
    extern __shared__ __align__(16) unsigned char s_dyn[];
    GpWarpSmem *s_warp = reinterpret_cast<GpWarpSmem *>(s_dyn);
    __shared__ uint8_t s_pi[36], s_pj[36];
    init_pack_smem(s_pi, s_pj);
    __syncthreads();
    GpWarpSmem &sm = s_warp[threadIdx.x >> 5];
    EmitHook hook{reinterpret_cast<EmitSmem *>(&sm), &A, sc, (int)(threadIdx.x & 31), (*status & (HX_ST_EMIT_SKIP | HX_ST_BAD_INDEX)) == 0};
    integrate_quads<MODE, WITH_INDEX, false, true>(sm, s_pi, s_pj, coords, n_nodes, conn, coeff, 0, n, ke_out, rows_out,
                                                   cols_out, fail_min, quad_counter, AdjOut{nullptr, nullptr}, hook);
}

// Workspace layout (all offsets 256-B aligned):
//   order_flag u32 | deg (ncols) i32 | adj (8*ncols) i32 | block_scratch (blocks) i64 |
//   scratch_top u64 | order keys/cols (2 x 2 x ncols) u32 | cub temp (scan / pair sort) |
//   scratch int2 (the rest of the workspace; hx_mesh_csc_workspace_bytes sizes it for
//   SCRATCH_PER_COL records per column, and a caller that gets HX_ST_SCRATCH_OVERFLOW re-runs with
//   room for col_ptr[ncols] records -- the counts are complete even then)
constexpr int64_t SCRATCH_PER_COL = 15;  // off-diagonal records per column reserved (hex: 13 avg)
struct MeshWs {
    uint32_t *order_flag;
    int32_t *deg, *adj;
    int64_t *block_scratch;
    int32_t *tile_need;  // per tile: 1 + its highest incident element (0: none)
    int32_t *tadj, *tdeg;  // element order only: sorted incident lists / degrees by processing position
    unsigned long long *scratch_top, *slot_total;
    int64_t *band;  // band_kernel: B and the strip width
    uint32_t *keys_in, *keys_out, *cols_in, *order;
    int2 *scratch;
    int64_t scratch_capacity;
    void *cub_tmp;
    size_t cub_bytes;
    size_t total;  // with the default scratch
};

static size_t cub_temp_bytes(int64_t ncols) {
    size_t b = 0, c = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, b, (int64_t *)nullptr, (int64_t *)nullptr, (int)(ncols + 1));
    cub::DeviceRadixSort::SortPairs(nullptr, c, (uint32_t *)nullptr, (uint32_t *)nullptr, (uint32_t *)nullptr,
                                    (uint32_t *)nullptr, (int)std::max<int64_t>(ncols, 1));
    return std::max(b, c);
}

static MeshWs mesh_ws_layout(void *base, int64_t ncols, int64_t workspace_bytes = -1) {
    MeshWs w{};
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off = align_up(off + bytes, 256);
        return o;
    };
    const int64_t nc = std::max<int64_t>(ncols, 1);
    const size_t o_flag = take(sizeof(uint32_t));
    const size_t o_deg = take(sizeof(int32_t) * nc);
    const size_t o_adj = take(sizeof(int32_t) * 8 * nc);
    const size_t o_bs = take(sizeof(int64_t) * std::max<int64_t>(1, ceil_div(ncols, COL_BLOCK)));
    const size_t o_tn = take(sizeof(int32_t) * std::max<int64_t>(1, ceil_div(ncols, COL_BLOCK)));
    const size_t o_ta = take(sizeof(int32_t) * 8 * nc), o_td = take(sizeof(int32_t) * nc);
    const size_t o_st = take(4 * sizeof(unsigned long long));  // scratch_top, slot_total, band[2]
    const size_t o_ki = take(sizeof(uint32_t) * nc), o_ko = take(sizeof(uint32_t) * nc);
    const size_t o_ci = take(sizeof(uint32_t) * nc), o_or = take(sizeof(uint32_t) * nc);
    w.cub_bytes = cub_temp_bytes(ncols);
    const size_t o_cub = take(w.cub_bytes);
    const size_t o_sc = off;
    const int64_t default_cap = std::max<int64_t>(1, SCRATCH_PER_COL * ncols);
    w.total = o_sc + sizeof(int2) * default_cap;
    w.scratch_capacity =
        workspace_bytes < 0 ? default_cap : std::max<int64_t>(0, (workspace_bytes - (int64_t)o_sc) / (int64_t)sizeof(int2));
    char *b = (char *)base;
    if (b) {
        w.order_flag = (uint32_t *)(b + o_flag);
        w.deg = (int32_t *)(b + o_deg);
        w.adj = (int32_t *)(b + o_adj);
        w.block_scratch = (int64_t *)(b + o_bs);
        w.tile_need = (int32_t *)(b + o_tn);
        w.tadj = (int32_t *)(b + o_ta);
        w.tdeg = (int32_t *)(b + o_td);
        w.scratch_top = (unsigned long long *)(b + o_st);
        w.slot_total = w.scratch_top + 1;
        w.band = reinterpret_cast<int64_t *>(w.scratch_top + 2);
        w.keys_in = (uint32_t *)(b + o_ki);
        w.keys_out = (uint32_t *)(b + o_ko);
        w.cols_in = (uint32_t *)(b + o_ci);
        w.order = (uint32_t *)(b + o_or);
        w.scratch = (int2 *)(b + o_sc);
        w.cub_tmp = b + o_cub;
    }
    return w;
}

static int make_segtable(const hx_elem_segment *segs, int32_t n_segs, SegTable &T, int64_t &n_total,
                         bool need_ke) {
    if (n_segs < 1 || n_segs > MAX_SEGS || segs == nullptr) {
        set_last_error("mesh csc: need 1..%d element segments, got %d", MAX_SEGS, n_segs);
        return HX_ERR_VALUE;
    }
    T = SegTable{};
    T.n = n_segs;
    int64_t acc = 0;
    for (int s = 0; s < n_segs; ++s) {
        if (segs[s].n_el < 0 || (segs[s].n_el > 0 && segs[s].conn == nullptr) ||
            (need_ke && segs[s].n_el > 0 && segs[s].ke == nullptr)) {
            set_last_error("mesh csc: bad element segment %d", s);
            return HX_ERR_VALUE;
        }
        T.conn[s] = segs[s].conn;
        T.ke[s] = segs[s].ke;
        T.koff[s] = segs[s].ke_offset;
        T.kmask[s] = segs[s].ke_mask;
        if ((T.koff[s] == nullptr) != (T.kmask[s] == nullptr)) {
            set_last_error("mesh csc: segment %d sets only one of ke_offset / ke_mask", s);
            return HX_ERR_VALUE;
        }
        T.conn_stride[s] = segs[s].conn_stride ? segs[s].conn_stride : 8;
        T.ke_stride[s] = segs[s].ke_stride ? segs[s].ke_stride : 36;
        if (T.conn_stride[s] < 8 || T.conn_stride[s] % 4 != 0 || T.ke_stride[s] < 36) {
            set_last_error("mesh csc: bad strides in segment %d", s);
            return HX_ERR_VALUE;
        }
        T.start[s] = acc;
        acc += segs[s].n_el;
    }
    for (int s = n_segs; s <= MAX_SEGS; ++s) T.start[s] = acc;
    n_total = acc;
    if (8 * n_total >= (int64_t)INT32_MAX) {
        set_last_error("mesh csc: %lld elements exceed the int32 adjacency of one plan; shard the mesh",
                       (long long)n_total);
        return HX_ERR_CONFIG;
    }
    return HX_OK;
}


int mesh_ws_adjacency(void *workspace, int64_t workspace_bytes, int64_t ncols, int32_t **deg, int32_t **adj) {
    const MeshWs w = mesh_ws_layout(workspace, ncols, workspace_bytes);
    if (workspace == nullptr || workspace_bytes < (int64_t)w.total) {
        set_last_error("mesh csc workspace %lld < %lld bytes", (long long)workspace_bytes, (long long)w.total);
        return HX_ERR_WORKSPACE;
    }
    *deg = w.deg;
    *adj = w.adj;
    return HX_OK;
}

// Strip width of the band order in columns (a multiple of the tile); HX_BAND_STRIP=0 turns it off.
static int64_t band_strip() {
    static const int64_t w = [] {
        const char *v = getenv("HX_BAND_STRIP");
        const int64_t x = v ? atoll(v) : HX_BAND_STRIP_DEFAULT;
        return x <= 0 ? (int64_t)0 : std::max<int64_t>(COL_BLOCK, x / COL_BLOCK * COL_BLOCK);
    }();
    return w;
}

static bool single_dense(const SegTable &T) {
    return T.n == 1 && T.ke_stride[0] == 36 && T.conn_stride[0] == 8 && T.koff[0] == nullptr;
}
static bool single_conn(const SegTable &T) { return T.n == 1 && T.conn_stride[0] == 8; }


}  // namespace hx

using namespace hx;

extern "C" int64_t hx_mesh_csc_workspace_bytes(int64_t n_el_total, int64_t n_cols) {
    if (n_el_total < 0 || n_cols < 0) return -1;
    (void)n_el_total;
    return (int64_t)mesh_ws_layout(nullptr, n_cols).total;
}

static EmitArgs emit_args(const SegTable &T, int64_t col_lo, int64_t ncols, const MeshWs &w, const int64_t *col_ptr,
                          int64_t *row_idx, double *vals, int64_t capacity) {
    EmitArgs A;
    A.T = T;
    A.col_lo = col_lo;
    A.ncols = ncols;
    A.deg_arr = w.deg;
    A.adj = w.adj;
    A.tdeg = w.tdeg;
    A.tadj = w.tadj;
    A.col_ptr = col_ptr;
    A.scratch = w.scratch;
    A.block_scratch = w.block_scratch;
    A.row_idx = row_idx;
    A.vals = vals;
    A.capacity = capacity;
    A.order_flag = w.order_flag;
    A.order = w.order;
    return A;
}

// wide: element-ordered builds (randomly numbered meshes) run 256 threads per tile -- their KE gathers
// and scattered CSC writes want more loads in flight (C5 -0.35 ms; column / strip order: +0.5 ms at C4).
template <bool ROWS, bool VALS>
static int launch_emit(const EmitArgs &A, const uint32_t *status, cudaStream_t s, const char *where,
                       bool wide = false) {
    const unsigned tiles = (unsigned)ceil_div(A.ncols, COL_BLOCK);
    const bool single = !VALS || single_dense(A.T);
    if (wide && single) emit_kernel<2 * EMIT_BLOCK, ROWS, VALS, true><<<tiles, 2 * EMIT_BLOCK, 0, s>>>(A, status);
    else if (wide) emit_kernel<2 * EMIT_BLOCK, ROWS, VALS, false><<<tiles, 2 * EMIT_BLOCK, 0, s>>>(A, status);
    else if (single) emit_kernel<EMIT_BLOCK, ROWS, VALS, true><<<tiles, EMIT_BLOCK, 0, s>>>(A, status);
    else emit_kernel<EMIT_BLOCK, ROWS, VALS, false><<<tiles, EMIT_BLOCK, 0, s>>>(A, status);
    HX_CHECK_LAUNCH(where);
    return HX_OK;
}

static int mesh_csc_build(const hx_elem_segment *segs, int32_t n_segs, int64_t n_nodes, int64_t col_lo,
                          int64_t col_hi, int64_t *col_ptr, int64_t *row_idx, double *vals, int64_t row_capacity,
                          void *workspace, int64_t workspace_bytes, uint32_t *status, int32_t flags, void *stream) {
    SegTable T;
    int64_t n_total = 0;
    int rc = make_segtable(segs, n_segs, T, n_total, vals != nullptr);
    if (rc) return rc;
    if (col_lo < 0 || col_hi < col_lo || col_hi > n_nodes || n_nodes >= INT32_MAX || col_ptr == nullptr ||
        status == nullptr || row_capacity < 0 || (row_capacity > 0 && row_idx == nullptr)) {
        set_last_error("hx_mesh_csc_symbolic: bad column range [%lld, %lld) for %lld nodes", (long long)col_lo,
                       (long long)col_hi, (long long)n_nodes);
        return HX_ERR_VALUE;
    }
    const int64_t ncols = col_hi - col_lo;
    MeshWs w = mesh_ws_layout(workspace, ncols, workspace_bytes);
    if (workspace == nullptr || workspace_bytes < (int64_t)w.total) {
        set_last_error("hx_mesh_csc_symbolic: workspace %lld < %lld bytes", (long long)workspace_bytes,
                       (long long)w.total);
        return HX_ERR_WORKSPACE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const bool ordered = (flags & HX_CSC_ORDER_BY_ELEMENT) != 0 && ncols > 0 && n_total > 0;
    // adjacency (and its status bits) already recorded by hx_integrate_mesh_adjacency
    const bool adj_ready = (flags & HX_CSC_ADJACENCY_READY) != 0;
    // fixed-slot adjacency: recorded by the integration kernel (adj_ready) or by adjacency_fixed_kernel
    const bool fixed = adj_ready || (flags & HX_CSC_FIXED_ADJACENCY) != 0;
    if (fixed && (n_segs != 1 || col_lo != 0 || col_hi != n_nodes || !single_conn(T))) {
        set_last_error("hx_mesh_csc_build: a fixed-slot adjacency needs one segment and every column");
        return HX_ERR_VALUE;
    }
    if (!adj_ready) HX_TRY_CUDA(cudaMemsetAsync(status, 0, sizeof(uint32_t), s));
    HX_TRY_CUDA(cudaMemsetAsync(w.order_flag, 0, sizeof(uint32_t), s));
    if (ordered) HX_TRY_CUDA(cudaMemsetAsync(w.order_flag, 1, 1, s));  // little-endian u32 == 1
    if (ncols > 0) {
        if (!adj_ready) HX_TRY_CUDA(cudaMemsetAsync(w.deg, 0, sizeof(int32_t) * ncols, s));
        if (n_total > 0 && !adj_ready && fixed) {
            HX_TRY_CUDA(cudaMemsetAsync(w.adj, 0xff, sizeof(int32_t) * 8 * ncols, s));
            const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(8 * n_total, 256), 148 * 64);
            adjacency_fixed_kernel<<<grid, 256, 0, s>>>(T.conn[0], n_total, n_nodes, w.adj, status);
            HX_CHECK_LAUNCH("adjacency_fixed_kernel");
        } else if (n_total > 0 && !adj_ready) {
            const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(8 * n_total, 256), 148 * 64);
            if (single_conn(T))
                adjacency_kernel<true><<<grid, 256, 0, s>>>(T, n_total, n_nodes, col_lo, col_hi, w.deg, w.adj, status);
            else
                adjacency_kernel<false><<<grid, 256, 0, s>>>(T, n_total, n_nodes, col_lo, col_hi, w.deg, w.adj, status);
            HX_CHECK_LAUNCH("adjacency_kernel");
        }
        const unsigned tiles = (unsigned)ceil_div(ncols, COL_BLOCK);
        if (ordered) {
            const unsigned g = (unsigned)std::min<int64_t>(ceil_div(ncols, 256), 148 * 32);
            const int64_t strip = band_strip();
            if (strip > 0 && ncols >= 1024 && n_total >= 8 * strip) {
                if (fixed) element_band_kernel<true><<<1, 256, 0, s>>>(ncols, w.deg, w.adj, n_total, strip, w.band);
                else element_band_kernel<false><<<1, 256, 0, s>>>(ncols, w.deg, w.adj, n_total, strip, w.band);
                HX_CHECK_LAUNCH("element_band_kernel");
            } else {
                HX_TRY_CUDA(cudaMemsetAsync(w.band, 0, 2 * sizeof(int64_t), s));
            }
            if (fixed)
                first_element_kernel<true><<<g, 256, 0, s>>>(ncols, w.deg, w.adj, (uint32_t)n_total, w.keys_in, w.cols_in,
                                                             w.band);
            else
                first_element_kernel<false><<<g, 256, 0, s>>>(ncols, w.deg, w.adj, (uint32_t)n_total, w.keys_in,
                                                              w.cols_in, w.band);
            HX_CHECK_LAUNCH("first_element_kernel");
            int end_bit = 1;
            while (end_bit < 32 && ((uint64_t)n_total >> end_bit) != 0) ++end_bit;
            // the order only needs element locality: sort on the top 16 bits of the first element (2
            // radix passes instead of up to 4); the stable sort keeps column order inside a bucket of
            // n_el / 2^16 consecutive elements
            const int begin_bit = std::max(0, end_bit - 16);
            size_t cb = w.cub_bytes;
            HX_TRY_CUDA(cub::DeviceRadixSort::SortPairs(w.cub_tmp, cb, w.keys_in, w.keys_out, w.cols_in, w.order,
                                                        (int)ncols, begin_bit, end_bit, s));
        }
        // banded numberings: strip order (decided on the device, see band_kernel)
        const int64_t strip = band_strip();
        const bool banded = !ordered && strip > 0 && single_conn(T) && n_total >= BAND_SAMPLES && ncols >= 8 * strip;
        if (banded) {
            band_kernel<<<1, 256, 0, s>>>(T.conn[0], n_total, ncols, strip, w.order_flag, w.band);
            HX_CHECK_LAUNCH("band_kernel");
            band_order_kernel<<<(unsigned)std::min<int64_t>(ceil_div(ceil_div(ncols, 4), 256), 148 * 16), 256, 0, s>>>(
                ncols, w.order_flag, w.band, w.order);
            HX_CHECK_LAUNCH("band_order_kernel");
        }
        const uint32_t *order = ordered || banded ? w.order : nullptr;
        HX_TRY_CUDA(cudaMemsetAsync(w.scratch_top, 0, 2 * sizeof(unsigned long long), s));  // + slot_total
        HX_TRY_CUDA(cudaMemsetAsync(w.tile_need, 0, sizeof(int32_t) * tiles, s));
        auto pattern = [&](auto key_tag, auto single_tag, auto fixed_tag) {
            using K = decltype(key_tag);
            pattern_kernel<K, decltype(single_tag)::value, decltype(fixed_tag)::value><<<tiles, COL_BLOCK, 0, s>>>(
                T, col_lo, ncols, w.deg, w.adj, col_ptr, w.scratch, w.scratch_capacity, w.scratch_top, w.block_scratch,
                status, order, w.slot_total, w.tile_need, w.tadj, w.tdeg, w.order_flag);
        };
        const bool packed = n_nodes <= (int64_t(1) << 26);
        if (fixed) {  // one dense segment (checked above)
            if (packed) pattern(uint32_t{}, std::true_type{}, std::true_type{});
            else pattern(uint64_t{}, std::true_type{}, std::true_type{});
        } else if (single_conn(T)) {
            if (packed) pattern(uint32_t{}, std::true_type{}, std::false_type{});
            else pattern(uint64_t{}, std::true_type{}, std::false_type{});
        } else {
            if (packed) pattern(uint32_t{}, std::false_type{}, std::false_type{});
            else pattern(uint64_t{}, std::false_type{}, std::false_type{});
        }
        HX_CHECK_LAUNCH("pattern_kernel");
        if (fixed) {
            slot_check_kernel<<<1, 32, 0, s>>>(w.slot_total, n_total, status);
            HX_CHECK_LAUNCH("slot_check_kernel");
        }
        HX_TRY_CUDA(cudaMemsetAsync(col_ptr + ncols, 0, sizeof(int64_t), s));
        size_t cb2 = w.cub_bytes;
        HX_TRY_CUDA(cub::DeviceScan::ExclusiveSum(w.cub_tmp, cb2, col_ptr, col_ptr, (int)(ncols + 1), s));
        if (vals != nullptr) {
            const int rc2 = launch_emit<true, true>(emit_args(T, col_lo, ncols, w, col_ptr, row_idx, vals, row_capacity),
                                                    status, s, "emit_kernel", ordered);
            if (rc2) return rc2;
        } else if (row_capacity > 0) {
            const int rc2 = launch_emit<true, false>(
                emit_args(T, col_lo, ncols, w, col_ptr, row_idx, nullptr, row_capacity), status, s, "emit_kernel<rows>");
            if (rc2) return rc2;
        }
    } else {
        HX_TRY_CUDA(cudaMemsetAsync(col_ptr, 0, sizeof(int64_t), s));
    }
    return HX_OK;
}

extern "C" int hx_mesh_csc_symbolic(const hx_elem_segment *segs, int32_t n_segs, int64_t n_nodes,
                                    int64_t col_lo, int64_t col_hi, int64_t *col_ptr, int64_t *row_idx,
                                    int64_t row_capacity, void *workspace, int64_t workspace_bytes,
                                    uint32_t *status, int32_t flags, void *stream) {
    return mesh_csc_build(segs, n_segs, n_nodes, col_lo, col_hi, col_ptr, row_idx, nullptr, row_capacity, workspace,
                          workspace_bytes, status, flags, stream);
}

extern "C" int hx_mesh_csc_build(const hx_elem_segment *segs, int32_t n_segs, int64_t n_nodes, int64_t col_lo,
                                 int64_t col_hi, int64_t *col_ptr, int64_t *row_idx, double *vals,
                                 int64_t capacity, void *workspace, int64_t workspace_bytes, uint32_t *status,
                                 int32_t flags, void *stream) {
    if (vals == nullptr && capacity > 0) {
        set_last_error("hx_mesh_csc_build: vals is NULL");
        return HX_ERR_VALUE;
    }
    return mesh_csc_build(segs, n_segs, n_nodes, col_lo, col_hi, col_ptr, row_idx, vals, capacity, workspace,
                          workspace_bytes, status, flags, stream);
}

extern "C" int hx_mesh_csc_numeric(const hx_elem_segment *segs, int32_t n_segs, int64_t col_lo, int64_t col_hi,
                                   const int64_t *col_ptr, const int64_t *row_idx, double *vals,
                                   const void *workspace, uint32_t *status, void *stream) {
    SegTable T;
    int64_t n_total = 0;
    int rc = make_segtable(segs, n_segs, T, n_total, true);
    if (rc) return rc;
    if (col_lo < 0 || col_hi < col_lo || col_ptr == nullptr || workspace == nullptr || status == nullptr) {
        set_last_error("hx_mesh_csc_numeric: bad arguments");
        return HX_ERR_VALUE;
    }
    const int64_t ncols = col_hi - col_lo;
    MeshWs w = mesh_ws_layout(const_cast<void *>(workspace), ncols);
    cudaStream_t s = (cudaStream_t)stream;
    if (ncols > 0) {
        const int rc2 = launch_emit<false, true>(
            emit_args(T, col_lo, ncols, w, col_ptr, nullptr, vals, INT64_MAX), status, s, "emit_kernel<numeric>");
        if (rc2) return rc2;
    }
    return HX_OK;
}

extern "C" int hx_mesh_csc_emit(const hx_elem_segment *segs, int32_t n_segs, int64_t col_lo, int64_t col_hi,
                                const int64_t *col_ptr, int64_t *row_idx, double *vals, int64_t capacity,
                                const void *workspace, uint32_t *status, void *stream) {
    SegTable T;
    int64_t n_total = 0;
    int rc = make_segtable(segs, n_segs, T, n_total, true);
    if (rc) return rc;
    if (col_lo < 0 || col_hi < col_lo || col_ptr == nullptr || workspace == nullptr || status == nullptr ||
        capacity < 0 || (capacity > 0 && (row_idx == nullptr || vals == nullptr))) {
        set_last_error("hx_mesh_csc_emit: bad arguments");
        return HX_ERR_VALUE;
    }
    const int64_t ncols = col_hi - col_lo;
    MeshWs w = mesh_ws_layout(const_cast<void *>(workspace), ncols);
    cudaStream_t s = (cudaStream_t)stream;
    if (ncols > 0) {
        const int rc2 = launch_emit<true, true>(emit_args(T, col_lo, ncols, w, col_ptr, row_idx, vals, capacity),
                                                status, s, "emit_kernel<emit>");
        if (rc2) return rc2;
    }
    return HX_OK;
}

static int64_t fused_chunks(int64_t n_el) {
    return std::max<int64_t>(1, ceil_div(ceil_div(n_el, GP_EL_PER_WARP), FUSED_CHUNK_QUADS));
}

extern "C" int64_t hx_integrate_emit_workspace_bytes(int64_t n_el) {
    if (n_el < 0) return -1;
    return 256 + (int64_t)sizeof(unsigned) * fused_chunks(n_el);
}

template <int MODE>
static void configure_fused() {
    static bool done[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && done[MODE * 32 + dev % 32]) return;
    cudaFuncSetAttribute(integrate_emit_kernel<MODE, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FUSED_SMEM);
    cudaFuncSetAttribute(integrate_emit_kernel<MODE, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FUSED_SMEM);
    if (dev < 64) done[MODE * 32 + dev % 32] = true;
}

template <int MODE>
static int launch_fused(int64_t n_el, cudaStream_t s, const double *coords, int64_t n_nodes, const int32_t *conn,
                        const double *coeff, double *ke, int32_t *rows, int32_t *cols, hx_fail_info *fail,
                        const EmitArgs &A, const FusedSched &sc, const uint32_t *status) {
    configure_fused<MODE>();
    int dev = 0, sms = 148, per_sm = HX_KE_MIN_BLOCKS;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, integrate_emit_kernel<MODE, true>, GP_BLOCK, FUSED_SMEM);
    const int64_t blocks = std::min<int64_t>(ceil_div(n_el, GP_EL_PER_BLOCK), (int64_t)sms * std::max(per_sm, 1));
    unsigned *counter = reinterpret_cast<unsigned *>(&fail->reserved);
    auto *fmin = reinterpret_cast<unsigned long long *>(fail);
    if (rows != nullptr)
        integrate_emit_kernel<MODE, true><<<(unsigned)blocks, GP_BLOCK, FUSED_SMEM, s>>>(
            coords, n_nodes, conn, coeff, n_el, ke, rows, cols, fmin, counter, A, sc, status);
    else
        integrate_emit_kernel<MODE, false><<<(unsigned)blocks, GP_BLOCK, FUSED_SMEM, s>>>(
            coords, n_nodes, conn, coeff, n_el, ke, rows, cols, fmin, counter, A, sc, status);
    HX_CHECK_LAUNCH("integrate_emit_kernel");
    return HX_OK;
}

extern "C" int hx_integrate_emit(const double *coords, int64_t n_nodes, const int32_t *conn, const double *coeff,
                                 int64_t n_el, double *ke, int32_t *rows, int32_t *cols, int32_t mode,
                                 hx_fail_info *fail, const int64_t *col_ptr, int64_t *row_idx, double *vals,
                                 int64_t capacity, const void *csc_workspace, const uint32_t *csc_status,
                                 void *sched_ws, int64_t sched_bytes, void *stream) {
    if (n_el < 0 || n_nodes < 0 || n_nodes >= INT32_MAX || 8 * n_el >= (int64_t)INT32_MAX || fail == nullptr ||
        (rows == nullptr) != (cols == nullptr) || col_ptr == nullptr || csc_workspace == nullptr ||
        csc_status == nullptr || sched_ws == nullptr || capacity < 0 ||
        (n_el > 0 && (ke == nullptr || conn == nullptr || coords == nullptr || coeff == nullptr)) ||
        (capacity > 0 && (row_idx == nullptr || vals == nullptr))) {
        set_last_error("hx_integrate_emit: bad arguments (n_el=%lld n_nodes=%lld)", (long long)n_el,
                       (long long)n_nodes);
        return HX_ERR_VALUE;
    }
    if (mode != HX_MODE_EXACT && mode != HX_MODE_FAST) {
        set_last_error("hx_integrate_emit: unknown mode %d", mode);
        return HX_ERR_CONFIG;
    }
    if (sched_bytes < hx_integrate_emit_workspace_bytes(n_el)) {
        set_last_error("hx_integrate_emit: scheduling workspace %lld < %lld bytes", (long long)sched_bytes,
                       (long long)hx_integrate_emit_workspace_bytes(n_el));
        return HX_ERR_WORKSPACE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    HX_TRY_CUDA(cudaMemsetAsync(fail, 0xff, sizeof(unsigned long long), s));
    HX_TRY_CUDA(cudaMemsetAsync(&fail->reserved, 0, sizeof(int32_t), s));  // quad counter
    HX_TRY_CUDA(cudaMemsetAsync(sched_ws, 0, (size_t)hx_integrate_emit_workspace_bytes(n_el), s));
    if (n_el > 0) {
        hx_elem_segment seg{};
        seg.conn = conn;
        seg.ke = ke;
        seg.n_el = n_el;
        SegTable T;
        int64_t n_total = 0;
        int rc = make_segtable(&seg, 1, T, n_total, true);
        if (rc) return rc;
        const MeshWs w = mesh_ws_layout(const_cast<void *>(csc_workspace), n_nodes);
        const EmitArgs A = emit_args(T, 0, n_nodes, w, col_ptr, row_idx, vals, capacity);
        FusedSched sc;
        unsigned *base = (unsigned *)sched_ws;
        sc.wm = base;              // its own 128-B line
        sc.tile_head = base + 32;  // its own 128-B line
        sc.done = base + 64;       // 256 B in
        sc.tile_need = w.tile_need;
        sc.n_quads = ceil_div(n_el, GP_EL_PER_WARP);
        sc.n_chunks = fused_chunks(n_el);
        sc.n_tiles = ceil_div(n_nodes, COL_BLOCK);
        sc.n_el = n_el;
        rc = mode == HX_MODE_EXACT
                 ? launch_fused<HX_MODE_EXACT>(n_el, s, coords, n_nodes, conn, coeff, ke, rows, cols, fail, A, sc, csc_status)
                 : launch_fused<HX_MODE_FAST>(n_el, s, coords, n_nodes, conn, coeff, ke, rows, cols, fail, A, sc, csc_status);
        if (rc) return rc;
    }
    return integrate_fail_resolve(coords, n_nodes, conn, fail, s);
}
