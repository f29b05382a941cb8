// hx_halo.cu -- the exchange step of the sharded (multi-GPU) build.
//
// Rank r integrates elements [E_r, E_r+1) and owns lower-CSC columns [C_r, C_r+1).  Entry (i, j)
// (i >= j, packed p) of element e lands in column min(g_i, g_j), so rank d needs exactly the
// entries with owner(min(g_i, g_j)) == d -- and because owners are monotone in the node id,
// owner(min(g_i, g_j)) = min(o_i, o_j) with o_a = owner(g_a).  With m_d = #{a : o_a >= d} the
// element holds T(m_d) - T(m_d+1) such entries (T(m) = m (m+1) / 2, diagonal included).
//
//   column weights   nnz estimate per column bin (for nnz-balanced column bounds, one all-reduce)
//   count / pack     compact records per (element, destination): the 8 node ids (4 words) in the
//                    destination's ids region, the owned KE entries (ascending p) in its values
//                    region -- destination-major, ascending element order within a destination,
//                    written warp-cooperatively (coalesced, also over NVLink into peer memory)
//   unpack           receiver: records -> full 40-word records (36 KE words, unowned entries 0,
//                    + the 8 ids), directly an hx_elem_segment (conn_stride 80, ke_stride 40)
//   digest           position-keyed 64-bit sum of an array, additive across ranks (parity)
//   ipc              receive buffers shared between processes (CUDA IPC, lazy peer access)
//
// Wire format: int64 words.  A source's chunk for destination d is [ids: 4 n_rec words][values:
// n_val words]; chunks arrive in ascending source order, so the receiver's [lower ranks | own |
// higher ranks] segments are in ascending global element order and every duplicate position is
// summed in the single-GPU order (bitwise equal to one GPU).
#include <cub/device/device_scan.cuh>

#include <algorithm>

#include "hx_common.cuh"

namespace hx {

constexpr int HALO_TILE = 256;
constexpr int HALO_WARPS = HALO_TILE / 32;
constexpr int HALO_MAX_WORLD = 32;

__device__ __forceinline__ int halo_owner(int32_t node, const int64_t *__restrict__ bounds, int world) {
    int lo = 0, hi = world;  // largest r with bounds[r] <= node
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(bounds + mid) <= node) lo = mid; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ int tri(int m) { return m * (m + 1) >> 1; }

__device__ __forceinline__ void halo_load(const int32_t *__restrict__ conn, int64_t e, int32_t (&g)[8]) {
    const int4 *c4 = reinterpret_cast<const int4 *>(conn) + 2 * e;
    const int4 a = __ldg(c4), b = __ldg(c4 + 1);
    g[0] = a.x; g[1] = a.y; g[2] = a.z; g[3] = a.w;
    g[4] = b.x; g[5] = b.y; g[6] = b.z; g[7] = b.w;
}

// number of entries of an element whose column rank d owns
__device__ __forceinline__ int owned_count(const int (&o)[8], int d) {
    int ge = 0, gt = 0;
#pragma unroll
    for (int a = 0; a < 8; ++a) {
        ge += o[a] >= d;
        gt += o[a] > d;
    }
    return tri(ge) - tri(gt);
}

// ---- nnz-balanced column bounds: per-bin nnz estimate ------------------------------------------
// Entry (i, j) of a hex8 element adds 1/s to its column's nnz where s = the number of elements
// sharing that node pair in a conforming interior neighbourhood: 8 (diagonal), 4 (edge), 2 (face
// diagonal), 1 (body diagonal) -- in units of 1/8: 1, 2, 4, 8 = 1 << (number of differing natural
// coordinates).  Exact away from the boundary; the bounds only need it to be proportional.
__host__ __device__ constexpr int nat_code(int a) {
    return (nat_r(a) > 0) | ((nat_s(a) > 0) << 1) | ((nat_t(a) > 0) << 2);
}

__global__ void __launch_bounds__(256)
column_weights_kernel(const int32_t *__restrict__ conn, int64_t n_el, int64_t n_nodes, int64_t n_bins,
                      unsigned long long *__restrict__ hist, int use_smem) {
    extern __shared__ unsigned s_hist[];
    if (use_smem) {
        for (int64_t b = threadIdx.x; b < n_bins; b += blockDim.x) s_hist[b] = 0u;
        __syncthreads();
    }
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n_el; e += (int64_t)gridDim.x * blockDim.x) {
        int32_t g[8];
        halo_load(conn, e, g);
        unsigned w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j <= i; ++j) {
                const unsigned wt = 1u << __popc(nat_code(i) ^ nat_code(j));
                if (g[j] <= g[i]) w[j] += wt; else w[i] += wt;  // the column is the smaller node
            }
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            if (w[a] == 0u || g[a] < 0 || g[a] >= n_nodes) continue;
            const int64_t b = (int64_t)g[a] * n_bins / n_nodes;
            if (use_smem) atomicAdd(&s_hist[b], w[a]);
            else atomicAdd(&hist[b], (unsigned long long)w[a]);
        }
    }
    if (use_smem) {
        __syncthreads();
        for (int64_t b = threadIdx.x; b < n_bins; b += blockDim.x)
            if (s_hist[b]) atomicAdd(&hist[b], (unsigned long long)s_hist[b]);
    }
}

// ---- per-bin element touches: the records / adjacency work a column block costs ---------------
// hist[b] += 8 for every element with at least one node in bin b (distinct bins of an element).  A
// block's received records and the elements its assembly walks scale with the elements touching it,
// not with its nnz: on a randomly numbered mesh the high-id blocks that an nnz-balanced cut makes
// wide receive twice the records of the low-id ones.
__global__ void __launch_bounds__(256)
column_touch_kernel(const int32_t *__restrict__ conn, int64_t n_el, int64_t n_nodes, int64_t n_bins,
                    unsigned long long *__restrict__ hist) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n_el; e += (int64_t)gridDim.x * blockDim.x) {
        int32_t g[8];
        halo_load(conn, e, g);
        int64_t b[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) b[a] = (g[a] < 0 || g[a] >= n_nodes) ? -1 : (int64_t)g[a] * n_bins / n_nodes;
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            bool first = b[a] >= 0;
#pragma unroll
            for (int q = 0; q < a; ++q) first = first && b[q] != b[a];
            if (first) atomicAdd(&hist[b[a]], 8ull);
        }
    }
}

// ---- count / pack ------------------------------------------------------------------------------
struct HaloWs {
    int64_t *rec_counts, *val_counts, *rec_offsets, *val_offsets, *totals;  // totals: (world, 2)
    void *cub_tmp;
    size_t cub_bytes, total;
};

static HaloWs halo_ws_layout(void *base, int64_t n_el, int world) {
    HaloWs w{};
    const int64_t n_tiles = std::max<int64_t>(1, ceil_div(n_el, HALO_TILE));
    const int64_t n = n_tiles * world;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off = align_up(off + bytes, 256);
        return o;
    };
    const size_t o_rc = take(8 * n), o_vc = take(8 * n), o_ro = take(8 * n), o_vo = take(8 * n);
    const size_t o_t = take(8 * 2 * (size_t)world);
    cub::DeviceScan::ExclusiveSum(nullptr, w.cub_bytes, (int64_t *)nullptr, (int64_t *)nullptr, (int)n);
    const size_t o_c = take(w.cub_bytes);
    w.total = off;
    if (base) {
        char *b = (char *)base;
        w.rec_counts = (int64_t *)(b + o_rc);
        w.val_counts = (int64_t *)(b + o_vc);
        w.rec_offsets = (int64_t *)(b + o_ro);
        w.val_offsets = (int64_t *)(b + o_vo);
        w.totals = (int64_t *)(b + o_t);
        w.cub_tmp = b + o_c;
    }
    return w;
}

__device__ __forceinline__ void element_owners(const int32_t *__restrict__ conn, int64_t e, int64_t n_el,
                                               const int64_t *__restrict__ bounds, int world, int32_t (&g)[8],
                                               int (&o)[8]) {
    if (e < n_el) {
        halo_load(conn, e, g);
#pragma unroll
        for (int a = 0; a < 8; ++a) o[a] = halo_owner(g[a], bounds, world);
    } else {
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            g[a] = 0;
            o[a] = -1;  // owns nothing anywhere
        }
    }
}

__global__ void __launch_bounds__(HALO_TILE)
halo_count_kernel(const int32_t *__restrict__ conn, int64_t n_el, const int64_t *__restrict__ bounds, int world,
                  int self, int64_t n_tiles, int64_t *__restrict__ rec_counts, int64_t *__restrict__ val_counts) {
    __shared__ int s_rec[HALO_MAX_WORLD], s_val[HALO_MAX_WORLD];
    const int t = threadIdx.x, lane = t & 31;
    if (t < HALO_MAX_WORLD) s_rec[t] = s_val[t] = 0;
    __syncthreads();
    const int64_t e = (int64_t)blockIdx.x * HALO_TILE + t;
    int32_t g[8];
    int o[8];
    element_owners(conn, e, n_el, bounds, world, g, o);
    for (int d = 0; d < world; ++d) {
        if (d == self) continue;
        // an element sends to d iff one of its nodes is owned by d (its diagonal entry): skip the
        // destinations no element of this warp touches (most of them on locally numbered meshes)
        bool touches = false;
#pragma unroll
        for (int a = 0; a < 8; ++a) touches |= o[a] == d;
        if (!__any_sync(0xffffffffu, touches)) continue;
        const int k = owned_count(o, d);
        const unsigned ballot = __ballot_sync(0xffffffffu, k > 0);
        int ks = k;
#pragma unroll
        for (int sh = 16; sh > 0; sh >>= 1) ks += __shfl_xor_sync(0xffffffffu, ks, sh);
        if (lane == 0 && ballot) {
            atomicAdd(&s_rec[d], __popc(ballot));
            atomicAdd(&s_val[d], ks);
        }
    }
    __syncthreads();
    if (t < world) {
        rec_counts[(int64_t)t * n_tiles + blockIdx.x] = s_rec[t];
        val_counts[(int64_t)t * n_tiles + blockIdx.x] = s_val[t];
    }
}

__global__ void halo_totals_kernel(const int64_t *__restrict__ rec_offsets, const int64_t *__restrict__ rec_counts,
                                   const int64_t *__restrict__ val_offsets, const int64_t *__restrict__ val_counts,
                                   int world, int64_t n_tiles, int64_t *__restrict__ totals,
                                   int64_t *__restrict__ per_dest) {
    const int d = threadIdx.x;
    if (d < world) {
        const int64_t a = (int64_t)d * n_tiles, z = a + n_tiles - 1;
        const int64_t nr = rec_offsets[z] + rec_counts[z] - rec_offsets[a];
        const int64_t nv = val_offsets[z] + val_counts[z] - val_offsets[a];
        totals[2 * d] = nr;
        totals[2 * d + 1] = nv;
        per_dest[2 * d] = nr;
        per_dest[2 * d + 1] = nv;
    }
}

// one tile = 8 warps x 32 elements; per destination each warp writes its records cooperatively
__global__ void __launch_bounds__(HALO_TILE)
halo_pack_kernel(const int32_t *__restrict__ conn, const double *__restrict__ ke, int64_t n_el,
                 const int64_t *__restrict__ bounds, int world, int self, int64_t n_tiles,
                 const int64_t *__restrict__ rec_counts, const int64_t *__restrict__ rec_offsets,
                 const int64_t *__restrict__ val_offsets, const int64_t *__restrict__ totals,
                 int64_t *const *__restrict__ dest_ptrs, const int64_t *__restrict__ dest_offsets) {
    __shared__ int s_wrec[HALO_WARPS], s_wval[HALO_WARPS];
    __shared__ uint16_t s_list[HALO_WARPS][32 * 36];  // (lane << 8) | p of the warp's values, in order
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int64_t e = (int64_t)blockIdx.x * HALO_TILE + t;
    const int64_t e0 = (int64_t)blockIdx.x * HALO_TILE + warp * 32;
    int32_t g[8];
    int o[8];
    element_owners(conn, e, n_el, bounds, world, g, o);
    const unsigned long long *ke_bits = reinterpret_cast<const unsigned long long *>(ke);
    for (int d = 0; d < world; ++d) {
        // nothing of this tile goes to d (block-uniform, from the count pass): skip the scan and syncs
        if (d == self || rec_counts[(int64_t)d * n_tiles + blockIdx.x] == 0) continue;
        bool touches = false;
#pragma unroll
        for (int a = 0; a < 8; ++a) touches |= o[a] == d;
        const int k = __any_sync(0xffffffffu, touches) ? owned_count(o, d) : 0;
        const unsigned ballot = __ballot_sync(0xffffffffu, k > 0);
        int incl = k;  // inclusive warp scan of k
#pragma unroll
        for (int sh = 1; sh < 32; sh <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, sh);
            if (lane >= sh) incl += v;
        }
        const int warp_val = __shfl_sync(0xffffffffu, incl, 31);
        if (lane == 0) {
            s_wrec[warp] = __popc(ballot);
            s_wval[warp] = warp_val;
        }
        // this lane's owned entries, ascending p, into the warp's list
        if (k > 0) {
            int q = incl - k;
#pragma unroll
            for (int p = 0; p < 36; ++p)
                if (min(o[pack_i(p)], o[pack_j(p)]) == d) s_list[warp][q++] = (uint16_t)((lane << 8) | p);
        }
        __syncthreads();
        int rec_before = 0, val_before = 0;
        for (int w = 0; w < warp; ++w) {
            rec_before += s_wrec[w];
            val_before += s_wval[w];
        }
        const int64_t a = (int64_t)d * n_tiles;
        const int64_t rec0 = rec_offsets[a + blockIdx.x] - rec_offsets[a] + rec_before;  // warp's first record
        const int64_t val0 = val_offsets[a + blockIdx.x] - val_offsets[a] + val_before;
        int64_t *base = dest_ptrs[d] + dest_offsets[d];
        int64_t *ids = base + 4 * rec0;
        int64_t *vals = base + 4 * totals[2 * d] + val0;
        const int nrec = __popc(ballot);
        for (int f = lane; f < 4 * nrec; f += 32) {
            const int i = f >> 2, word = f & 3;
            const int64_t el = e0 + __fns(ballot, 0, i + 1);
            ids[f] = __ldg(reinterpret_cast<const long long *>(conn + 8 * el) + word);
        }
        for (int f = lane; f < warp_val; f += 32) {
            const unsigned w = s_list[warp][f];
            vals[f] = (int64_t)__ldg(ke_bits + 36 * (e0 + (w >> 8)) + (w & 255u));
        }
        __syncthreads();  // s_list / s_w* are rewritten for the next destination
    }
}

// ---- unpack at the receiver -----------------------------------------------------------------------
// src_desc (world, 3) int64: word offset of source s's chunk in recv, its record count, its value count.
struct SrcTable {
    int64_t rec_start[HALO_MAX_WORLD + 1], val_start[HALO_MAX_WORLD + 1], off[HALO_MAX_WORLD], nrec[HALO_MAX_WORLD];
};

__device__ void load_src_table(SrcTable &tb, const int64_t *__restrict__ src_desc, int world) {
    if (threadIdx.x == 0) {
        int64_t r = 0, v = 0;
        for (int s = 0; s < world; ++s) {
            tb.rec_start[s] = r;
            tb.val_start[s] = v;
            tb.off[s] = src_desc[3 * s];
            tb.nrec[s] = src_desc[3 * s + 1];
            r += src_desc[3 * s + 1];
            v += src_desc[3 * s + 2];
        }
        tb.rec_start[world] = r;
        tb.val_start[world] = v;
    }
    __syncthreads();
}

__device__ __forceinline__ int src_of(const SrcTable &tb, int64_t i, int world) {
    int s = 0;
    while (s + 1 < world && tb.rec_start[s + 1] <= i) ++s;
    return s;
}

__global__ void __launch_bounds__(256)
halo_unpack_count_kernel(const int64_t *__restrict__ recv, const int64_t *__restrict__ src_desc, int world, int self,
                         const int64_t *__restrict__ bounds, int64_t n_rec, int64_t *__restrict__ kbuf) {
    __shared__ SrcTable tb;
    load_src_table(tb, src_desc, world);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_rec; i += (int64_t)gridDim.x * blockDim.x) {
        const int s = src_of(tb, i, world);
        const int32_t *g = reinterpret_cast<const int32_t *>(recv + tb.off[s] + 4 * (i - tb.rec_start[s]));
        int o[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) o[a] = halo_owner(g[a], bounds, world);
        kbuf[i] = owned_count(o, self);
    }
}

// 8 lanes per record (4 records per warp and step): lane a of a record owns node a (owner lookup) and
// the packed entries p = a, a + 8, ... (p < 36); the record's owned-entry mask is OR-reduced across
// its 8 lanes, so each lane knows where its entries sit in the compact value list.  Stores are 8
// consecutive doubles per record and instruction (the thread-per-record form wrote 40 scattered
// words per thread: 4x slower at C5, G = 8).
__global__ void __launch_bounds__(256)
halo_unpack_kernel(const int64_t *__restrict__ recv, const int64_t *__restrict__ src_desc, int world, int self,
                   const int64_t *__restrict__ bounds, int64_t n_rec, const int64_t *__restrict__ voff,
                   double *__restrict__ records) {
    __shared__ SrcTable tb;
    load_src_table(tb, src_desc, world);
    const int lane = threadIdx.x & 31, sub = lane & 7, grp = lane >> 3;
    const int64_t stride = ((int64_t)gridDim.x * blockDim.x) >> 3;  // records per grid step
    // warp-uniform loop (shuffles below): the warp's 4 records are base .. base + 3
    for (int64_t base = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 4; base < n_rec; base += stride) {
        const int64_t i = base + grp;
        const bool active = i < n_rec;
        int s = 0;
        int64_t chunk_off = 0, rec_start = 0, val_start = 0, nrec = 0;
        if (active) {
            s = src_of(tb, i, world);
            chunk_off = tb.off[s];
            rec_start = tb.rec_start[s];
            val_start = tb.val_start[s];
            nrec = tb.nrec[s];
        }
        const int64_t *chunk = recv + chunk_off;
        const int32_t *g = reinterpret_cast<const int32_t *>(chunk + 4 * (i - rec_start));
        const int32_t node = active ? __ldg(g + sub) : 0;
        const int own_node = active ? halo_owner(node, bounds, world) : -1;
        int o[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) o[a] = __shfl_sync(0xffffffffu, own_node, 8 * grp + a);
        unsigned long long mine = 0;
#pragma unroll
        for (int m = 0; m < 5; ++m) {
            const int p = sub + 8 * m;
            if (p < 36 && min(o[pack_i(p)], o[pack_j(p)]) == self) mine |= 1ull << p;
        }
#pragma unroll
        for (int sh = 1; sh < 8; sh <<= 1) mine |= __shfl_xor_sync(0xffffffffu, mine, sh);
        if (!active) continue;
        const int64_t *vals = chunk + 4 * nrec + (voff[i] - val_start);
        double *out = records + 40 * i;
#pragma unroll
        for (int m = 0; m < 5; ++m) {
            const int p = sub + 8 * m;
            if (p < 36) {
                const bool own = (mine >> p) & 1ull;
                out[p] = own ? __longlong_as_double(__ldg(vals + __popcll(mine & ((1ull << p) - 1ull)))) : 0.0;
            }
        }
        if (sub < 4) reinterpret_cast<long long *>(out + 36)[sub] = __ldg(reinterpret_cast<const long long *>(g) + sub);
    }
}

// Received records as compact element segments (hx_halo_index): thread per record -- its 8 ids as
// the segment's connectivity row, the word index of its first value in recv, its owned-entry mask.
__global__ void __launch_bounds__(256)
halo_index_kernel(const int64_t *__restrict__ recv, const int64_t *__restrict__ src_desc, int world, int self,
                  const int64_t *__restrict__ bounds, int64_t n_rec, const int64_t *__restrict__ voff,
                  int32_t *__restrict__ conn, int64_t *__restrict__ ke_offset, uint64_t *__restrict__ ke_mask) {
    __shared__ SrcTable tb;
    load_src_table(tb, src_desc, world);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_rec; i += (int64_t)gridDim.x * blockDim.x) {
        const int s = src_of(tb, i, world);
        const int64_t *ids = recv + tb.off[s] + 4 * (i - tb.rec_start[s]);
        // 8-byte loads: a source chunk starts at any word (its value count can be odd)
        const int64_t w0 = ids[0], w1 = ids[1], w2 = ids[2], w3 = ids[3];
        const int32_t g[8] = {(int32_t)(w0 & 0xffffffff), (int32_t)(w0 >> 32), (int32_t)(w1 & 0xffffffff),
                              (int32_t)(w1 >> 32), (int32_t)(w2 & 0xffffffff), (int32_t)(w2 >> 32),
                              (int32_t)(w3 & 0xffffffff), (int32_t)(w3 >> 32)};
        int o[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) o[q] = halo_owner(g[q], bounds, world);
        uint64_t m = 0;
#pragma unroll
        for (int p = 0; p < 36; ++p)
            if (min(o[pack_i(p)], o[pack_j(p)]) == self) m |= 1ull << p;
        int4 *c4 = reinterpret_cast<int4 *>(conn + 8 * i);
        c4[0] = make_int4(g[0], g[1], g[2], g[3]);
        c4[1] = make_int4(g[4], g[5], g[6], g[7]);
        ke_offset[i] = tb.off[s] + 4 * tb.nrec[s] + (voff[i] - tb.val_start[s]);
        ke_mask[i] = m;
    }
}

// ---- digest ----------------------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t digest_mix(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

__global__ void __launch_bounds__(256)
digest_kernel(const uint64_t *__restrict__ data, int64_t n, int64_t pos0, uint64_t add,
              unsigned long long *__restrict__ out) {
    uint64_t acc = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        acc += digest_mix(digest_mix((uint64_t)(pos0 + i)) ^ (__ldg(data + i) + add));
#pragma unroll
    for (int sh = 16; sh > 0; sh >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, sh);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, (unsigned long long)acc);
}

}  // namespace hx

using namespace hx;

extern "C" int hx_column_weights(const int32_t *conn, int64_t n_el, int64_t n_nodes, int64_t n_bins, uint64_t *hist,
                                 void *stream) {
    if (n_el < 0 || n_nodes < 1 || n_bins < 1 || n_bins > n_nodes || hist == nullptr || (n_el > 0 && conn == nullptr)) {
        set_last_error("hx_column_weights: bad arguments");
        return HX_ERR_VALUE;
    }
    if (n_el == 0) return HX_OK;
    const int use_smem = n_bins <= 16384;
    const size_t smem = use_smem ? sizeof(unsigned) * (size_t)n_bins : 0;
    if (use_smem && smem > 48 * 1024)
        HX_TRY_CUDA(cudaFuncSetAttribute(column_weights_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t blocks = std::min<int64_t>(ceil_div(n_el, 256), use_smem ? 148 * 2 : 148 * 16);
    column_weights_kernel<<<(unsigned)blocks, 256, smem, (cudaStream_t)stream>>>(
        conn, n_el, n_nodes, n_bins, reinterpret_cast<unsigned long long *>(hist), use_smem);
    HX_CHECK_LAUNCH("column_weights_kernel");
    return HX_OK;
}

extern "C" int hx_column_touch(const int32_t *conn, int64_t n_el, int64_t n_nodes, int64_t n_bins, uint64_t *hist,
                               void *stream) {
    if (n_el < 0 || n_nodes < 1 || n_bins < 1 || n_bins > n_nodes || hist == nullptr || (n_el > 0 && conn == nullptr)) {
        set_last_error("hx_column_touch: bad arguments");
        return HX_ERR_VALUE;
    }
    if (n_el == 0) return HX_OK;
    const int64_t blocks = std::min<int64_t>(ceil_div(n_el, 256), 148 * 16);
    column_touch_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
        conn, n_el, n_nodes, n_bins, reinterpret_cast<unsigned long long *>(hist));
    HX_CHECK_LAUNCH("column_touch_kernel");
    return HX_OK;
}

extern "C" int64_t hx_halo_workspace_bytes(int64_t n_el, int32_t world) {
    if (n_el < 0 || world < 1 || world > HALO_MAX_WORLD) return -1;
    return (int64_t)halo_ws_layout(nullptr, n_el, world).total;
}

extern "C" int hx_halo_count(const int32_t *conn, int64_t n_el, const int64_t *col_bounds, int32_t world, int32_t self,
                             int64_t *per_dest, void *workspace, int64_t workspace_bytes, void *stream) {
    if (n_el < 0 || world < 1 || world > HALO_MAX_WORLD || self < 0 || self >= world || col_bounds == nullptr ||
        per_dest == nullptr || (n_el > 0 && conn == nullptr)) {
        set_last_error("hx_halo_count: bad arguments");
        return HX_ERR_VALUE;
    }
    HaloWs w = halo_ws_layout(workspace, n_el, world);
    if (workspace == nullptr || workspace_bytes < (int64_t)w.total) {
        set_last_error("hx_halo_count: workspace too small");
        return HX_ERR_WORKSPACE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t n_tiles = std::max<int64_t>(1, ceil_div(n_el, HALO_TILE));
    const int64_t n = n_tiles * world;
    if (n > INT32_MAX) {
        set_last_error("hx_halo_count: %lld elements x %d ranks exceed one scan", (long long)n_el, world);
        return HX_ERR_CONFIG;
    }
    if (n_el == 0) {
        HX_TRY_CUDA(cudaMemsetAsync(w.rec_counts, 0, 8 * n, s));
        HX_TRY_CUDA(cudaMemsetAsync(w.val_counts, 0, 8 * n, s));
    } else {
        halo_count_kernel<<<(unsigned)n_tiles, HALO_TILE, 0, s>>>(conn, n_el, col_bounds, world, self, n_tiles,
                                                                 w.rec_counts, w.val_counts);
        HX_CHECK_LAUNCH("halo_count_kernel");
    }
    size_t cb = w.cub_bytes;
    HX_TRY_CUDA(cub::DeviceScan::ExclusiveSum(w.cub_tmp, cb, w.rec_counts, w.rec_offsets, (int)n, s));
    cb = w.cub_bytes;
    HX_TRY_CUDA(cub::DeviceScan::ExclusiveSum(w.cub_tmp, cb, w.val_counts, w.val_offsets, (int)n, s));
    halo_totals_kernel<<<1, HALO_MAX_WORLD, 0, s>>>(w.rec_offsets, w.rec_counts, w.val_offsets, w.val_counts, world,
                                                    n_tiles, w.totals, per_dest);
    HX_CHECK_LAUNCH("halo_totals_kernel");
    return HX_OK;
}

extern "C" int hx_halo_pack(const int32_t *conn, const double *ke, int64_t n_el, const int64_t *col_bounds,
                            int32_t world, int32_t self, int64_t *const *dest_ptrs, const int64_t *dest_offsets,
                            const void *workspace, void *stream) {
    if (n_el < 0 || world < 1 || world > HALO_MAX_WORLD || self < 0 || self >= world || workspace == nullptr ||
        dest_ptrs == nullptr || dest_offsets == nullptr || col_bounds == nullptr ||
        (n_el > 0 && (conn == nullptr || ke == nullptr))) {
        set_last_error("hx_halo_pack: bad arguments");
        return HX_ERR_VALUE;
    }
    if (n_el == 0) return HX_OK;
    HaloWs w = halo_ws_layout(const_cast<void *>(workspace), n_el, world);
    const int64_t n_tiles = ceil_div(n_el, HALO_TILE);
    halo_pack_kernel<<<(unsigned)n_tiles, HALO_TILE, 0, (cudaStream_t)stream>>>(
        conn, ke, n_el, col_bounds, world, self, n_tiles, w.rec_counts, w.rec_offsets, w.val_offsets, w.totals,
        dest_ptrs, dest_offsets);
    HX_CHECK_LAUNCH("halo_pack_kernel");
    return HX_OK;
}

extern "C" int64_t hx_halo_unpack_workspace_bytes(int64_t n_rec) {
    if (n_rec < 0 || n_rec > INT32_MAX) return -1;
    size_t cb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, cb, (int64_t *)nullptr, (int64_t *)nullptr, (int)std::max<int64_t>(n_rec, 1));
    return (int64_t)(align_up(16 * (size_t)std::max<int64_t>(n_rec, 1), 256) + cb);
}

extern "C" int hx_halo_unpack(const int64_t *recv, const int64_t *src_desc, int32_t world, int32_t self,
                              const int64_t *col_bounds, int64_t n_rec, double *records, void *workspace,
                              int64_t workspace_bytes, void *stream) {
    if (world < 1 || world > HALO_MAX_WORLD || self < 0 || self >= world || n_rec < 0 || src_desc == nullptr ||
        col_bounds == nullptr || (n_rec > 0 && (recv == nullptr || records == nullptr))) {
        set_last_error("hx_halo_unpack: bad arguments");
        return HX_ERR_VALUE;
    }
    if (n_rec == 0) return HX_OK;
    const int64_t need = hx_halo_unpack_workspace_bytes(n_rec);
    if (need < 0 || workspace == nullptr || workspace_bytes < need) {
        set_last_error("hx_halo_unpack: workspace too small");
        return HX_ERR_WORKSPACE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    int64_t *kbuf = (int64_t *)workspace, *voff = kbuf + n_rec;
    void *cub_tmp = (char *)workspace + align_up(16 * (size_t)n_rec, 256);
    size_t cb = (size_t)workspace_bytes - align_up(16 * (size_t)n_rec, 256);
    const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(n_rec, 256), 148 * 8);
    halo_unpack_count_kernel<<<blocks, 256, 0, s>>>(recv, src_desc, world, self, col_bounds, n_rec, kbuf);
    HX_CHECK_LAUNCH("halo_unpack_count_kernel");
    HX_TRY_CUDA(cub::DeviceScan::ExclusiveSum(cub_tmp, cb, kbuf, voff, (int)n_rec, s));
    halo_unpack_kernel<<<blocks, 256, 0, s>>>(recv, src_desc, world, self, col_bounds, n_rec, voff, records);
    HX_CHECK_LAUNCH("halo_unpack_kernel");
    return HX_OK;
}

extern "C" int hx_halo_index(const int64_t *recv, const int64_t *src_desc, int32_t world, int32_t self,
                             const int64_t *col_bounds, int64_t n_rec, int32_t *conn, int64_t *ke_offset,
                             uint64_t *ke_mask, void *workspace, int64_t workspace_bytes, void *stream) {
    if (world < 1 || world > HALO_MAX_WORLD || self < 0 || self >= world || n_rec < 0 || src_desc == nullptr ||
        col_bounds == nullptr ||
        (n_rec > 0 && (recv == nullptr || conn == nullptr || ke_offset == nullptr || ke_mask == nullptr))) {
        set_last_error("hx_halo_index: bad arguments");
        return HX_ERR_VALUE;
    }
    if (n_rec == 0) return HX_OK;
    const int64_t need = hx_halo_unpack_workspace_bytes(n_rec);
    if (need < 0 || workspace == nullptr || workspace_bytes < need) {
        set_last_error("hx_halo_index: workspace too small");
        return HX_ERR_WORKSPACE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    int64_t *kbuf = (int64_t *)workspace, *voff = kbuf + n_rec;
    void *cub_tmp = (char *)workspace + align_up(16 * (size_t)n_rec, 256);
    size_t cb = (size_t)workspace_bytes - align_up(16 * (size_t)n_rec, 256);
    const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(n_rec, 256), 148 * 8);
    halo_unpack_count_kernel<<<blocks, 256, 0, s>>>(recv, src_desc, world, self, col_bounds, n_rec, kbuf);
    HX_CHECK_LAUNCH("halo_unpack_count_kernel");
    HX_TRY_CUDA(cub::DeviceScan::ExclusiveSum(cub_tmp, cb, kbuf, voff, (int)n_rec, s));
    halo_index_kernel<<<blocks, 256, 0, s>>>(recv, src_desc, world, self, col_bounds, n_rec, voff, conn, ke_offset,
                                             ke_mask);
    HX_CHECK_LAUNCH("halo_index_kernel");
    return HX_OK;
}

extern "C" int hx_digest(const void *data, int64_t n_words, int64_t pos0, uint64_t add, uint64_t *out, void *stream) {
    if (n_words < 0 || out == nullptr || (n_words > 0 && data == nullptr)) {
        set_last_error("hx_digest: bad arguments");
        return HX_ERR_VALUE;
    }
    if (n_words == 0) return HX_OK;
    const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(n_words, 256), 148 * 8);
    digest_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>((const uint64_t *)data, n_words, pos0, add,
                                                            reinterpret_cast<unsigned long long *>(out));
    HX_CHECK_LAUNCH("digest_kernel");
    return HX_OK;
}

// ---- CUDA IPC receive buffers -------------------------------------------------------------------------
extern "C" int hx_ipc_alloc(int64_t bytes, void **ptr, void *handle) {
    if (bytes < 1 || ptr == nullptr || handle == nullptr) {
        set_last_error("hx_ipc_alloc: bad arguments");
        return HX_ERR_VALUE;
    }
    static_assert(sizeof(cudaIpcMemHandle_t) == HX_IPC_HANDLE_BYTES, "IPC handle size");
    HX_TRY_CUDA(cudaMalloc(ptr, (size_t)bytes));
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, *ptr);
    if (e != cudaSuccess) {
        cudaFree(*ptr);
        *ptr = nullptr;
        return cuda_status(e, "cudaIpcGetMemHandle");
    }
    memcpy(handle, &h, sizeof(h));
    return HX_OK;
}

extern "C" int hx_ipc_open(const void *handle, void **ptr) {
    if (handle == nullptr || ptr == nullptr) {
        set_last_error("hx_ipc_open: bad arguments");
        return HX_ERR_VALUE;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    // mapped into the CURRENT device's context; lazy peer access lets this device's kernels store
    // into the owner's memory over NVLink when the owner is another GPU
    HX_TRY_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return HX_OK;
}

extern "C" int hx_ipc_close(void *ptr) {
    if (ptr) HX_TRY_CUDA(cudaIpcCloseMemHandle(ptr));
    return HX_OK;
}

extern "C" int hx_ipc_free(void *ptr) {
    if (ptr) HX_TRY_CUDA(cudaFree(ptr));
    return HX_OK;
}
