/*
 * hexfem_b200.h -- C ABI of the B200-native hexfem hot path (libhexfem_b200.so).
 *
 * Drop-in boundary for the reference package `hexfem` (/root/reference/pkg/src/hexfem).
 * Every entry point is extern "C", takes plain pointers + sizes, is asynchronous on the
 * given CUDA stream (`void *stream`, a cudaStream_t; NULL = legacy default stream) and
 * returns an int status (HX_OK = 0).  Device-side failures (degenerate elements, index
 * validation, fast-path limits) are reported through small caller-owned DEVICE words that
 * the caller reads after synchronising, so no call here blocks the host.
 *
 * All device buffers are caller-owned (the reference's `out=` convention,
 * integrate.py:93-99); scratch is a caller-provided workspace sized by the *_workspace_bytes
 * queries.  The library allocates nothing (except hx_ipc_alloc, which exists to allocate).  Arrays of length zero may be passed as NULL
 * (what allocators hand out for empty tensors); zero-size calls are valid no-ops that still
 * write their status / fail words.
 *
 * Reference interfaces replaced (file:line under /root/reference/pkg/src/hexfem/):
 *   hx_stiffness_batch             element.py:213-245 stiffness_batch / integrate.py:84-131
 *                                  ComputeBackend.run
 *   hx_integrate_mesh              integrate.py:146-149 + 152-212 (gather + per-group run) fused
 *                                  with assemble.py:86-93 connectivity_index_arrays
 *   hx_integrate_mesh_adjacency    hx_integrate_mesh + the node adjacency (first pass) of hx_mesh_csc_build
 *   hx_connectivity_index_arrays   assemble.py:86-93
 *   hx_mesh_csc_*                  assemble.py:152-239 DirectAssembler / assemble_direct, and
 *                                  triplet_to_csc (assemble.py:110-140) on mesh triplets
 *   hx_triplet_csc_*               assemble.py:110-149 triplet_to_csc + _check_indices
 *   hx_halo_*, hx_column_weights,  (new) exchange step of the multi-GPU path: nnz-balanced column
 *   hx_digest, hx_ipc_*            blocks, compact element records, block checksums, IPC buffers
 *   hx_block_*                     (new) column blocks of the out-of-core build (Eq. 10 batching,
 *                                  integrate.py:55-81 / PAPER.md:192-199, beyond one GPU's HBM)
 */
#ifndef HEXFEM_B200_H
#define HEXFEM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HX_ABI_VERSION 4  /* 2: flags argument of hx_mesh_csc_symbolic/build, hx_mesh_csc_emit, hx_block_*
                           * 3: hx_integrate_mesh_adjacency + HX_CSC_ADJACENCY_READY (fused first pass)
                           * 4: compact halo records (hx_halo_count/pack/unpack), hx_column_weights,
                           *    hx_digest, hx_ipc_*; HX_FAIL_BAD_NODE */

/* Status codes (host return values).  The Python layer maps them onto the reference
 * exception hierarchy (errors.py:4-59). */
#define HX_OK 0
#define HX_ERR_VALUE 1         /* ValueError: bad sizes / pointers (element.py:228-233)    */
#define HX_ERR_CONFIG 2        /* ConfigurationError (errors.py:46-47)                     */
#define HX_ERR_CUDA 3          /* CUDA runtime error; see hx_last_error()                  */
#define HX_ERR_WORKSPACE 4     /* workspace smaller than the *_workspace_bytes query       */

/* Bits of the device status word written by the assembly entry points. */
#define HX_ST_DEG_OVERFLOW 1u  /* a node has more than HX_MAX_NODE_DEGREE incident elements */
#define HX_ST_ROW_OVERFLOW 2u  /* a column has more than HX_MAX_COL_ROWS distinct rows      */
#define HX_ST_REPEATED_NODE 4u /* an element lists the same node twice                     */
#define HX_ST_BAD_INDEX 8u     /* index outside [0, dim) (MeshValidationError, assemble.py:146) */
#define HX_ST_UPPER 16u        /* triplet above the diagonal (MeshValidationError, assemble.py:148) */
#define HX_ST_SCRATCH_OVERFLOW 32u /* pattern scratch too small (> 15 off-diagonals per column on average):
                                    * col_ptr is complete; re-run with workspace_bytes +=
                                    * 8 * col_ptr[ncols] */
#define HX_ST_SLOT_COLLISION 64u /* HX_CSC_ADJACENCY_READY build: two elements hold one node at the same
                                   * local index, so the fixed-slot adjacency lost an entry: re-run the
                                   * build without the flag (the atomic adjacency pass) */
/* DEG/ROW/REPEATED mean "mesh fast path not applicable": the caller re-runs the generic triplet
 * path (hx_triplet_csc_*), which has no such limits.  With any of the four bits set the entry
 * points write no row_idx / vals. */

#define HX_MAX_NODE_DEGREE 8
#define HX_MAX_COL_ROWS 32

/* Flags of the mesh-path assembly (hx_mesh_csc_symbolic / hx_mesh_csc_build). */
#define HX_CSC_ORDER_BY_ELEMENT 1 /* process columns in order of their lowest incident element (one pair
                                   * sort): for numberings without locality (e.g. randomly permuted
                                   * node ids) the pattern and emit passes then gather nearby
                                   * elements; results are identical either way */
#define HX_CSC_ADJACENCY_READY 2  /* hx_mesh_csc_build only: the workspace's node adjacency and the status
                                   * word were filled by hx_integrate_mesh_adjacency over every element
                                   * (one segment, columns [0, n_nodes)); the build skips its first pass */
#define HX_CSC_FIXED_ADJACENCY 4  /* symbolic/build: record the node adjacency in fixed slots (element e puts
                                   * e << 3 | a in slot a of its local node a; plain stores, no atomic
                                   * counter) -- one segment, columns [0, n_nodes).  Two elements holding one
                                   * node at the same local index raise HX_ST_SLOT_COLLISION: re-run
                                   * without the flag */

/* Integration modes. */
#define HX_MODE_EXACT 0 /* reference operation order, no FMA: bitwise equal to the reference */
#define HX_MODE_FAST 1  /* FMA + restructured algebra: |d| <= 1e-12 * max|row| (documented)  */

/* Lowest failing element of an integration call (DegenerateElementError fields,
 * errors.py:21-40).  element = -1 when every element is valid.  Device memory.
 * gauss_point = HX_FAIL_BAD_NODE: the element references a node id outside [0, n_nodes) (the
 * reference's staging gather raises IndexError there, integrate.py:146-149; validate_mesh raises
 * MeshValidationError, mesh.py:106-110) -- det then holds the offending node id.  Elements with a
 * bad node id take precedence over degenerate ones (the reference fails at staging, before
 * computing). */
#define HX_FAIL_BAD_NODE (-2)
typedef struct hx_fail_info {
    int64_t element;     /* global element id (element_offset applied, element.py:237-244) */
    int32_t gauss_point; /* 0..7, r slowest (element.py:116-121); HX_FAIL_BAD_NODE         */
    int32_t reserved;    /* scratch of the integration call (work counter), zeroed by it        */
    double det;          /* det(J) at that point (element.py:276-279)                      */
} hx_fail_info;

/* One contiguous run of elements (connectivity + packed values).  Segments passed to the
 * hx_mesh_csc_* calls are concatenated in order and MUST be in ascending global element
 * order: duplicate positions are summed in that order (assemble.py:115-117, 179-184). */
typedef struct hx_elem_segment {
    const int32_t *conn; /* element e's 8 global node ids at conn + e*conn_stride, device      */
    const double *ke;    /* element e's 36 packed values at ke + e*ke_stride (NULL: symbolic) */
    int64_t n_el;
    int64_t conn_stride; /* in int32 units, multiple of 4; 0 means dense (8)                 */
    int64_t ke_stride;   /* in doubles; 0 means dense (36)                                   */
    /* compact KE (received halo records, hx_halo_index): when ke_offset != NULL, element e holds
     * only the packed entries set in ke_mask[e] (bit p = entry p), stored in ascending p at
     * ke + ke_offset[e]; the assembly reads only entries of the columns it owns, which are exactly
     * those.  NULL: dense rows as above. */
    const int64_t *ke_offset;
    const uint64_t *ke_mask;
} hx_elem_segment;

/* ---- introspection (host only, no GPU needed) ------------------------------------------ */
int hx_abi_version(void);
const char *hx_last_error(void);
/* _DN_AT_GP (element.py:126-130) as compiled into the kernels: out[gp*24 + d*8 + a]. */
void hx_dn_table(double *out192);
/* PACK_ROWS / PACK_COLS (element.py:59-62) as compiled into the kernels. */
void hx_pack_tables(int32_t *rows36, int32_t *cols36);
/* Number of streaming multiprocessors of the current device (0 when no device). */
int hx_device_sm_count(void);
/* Self-test of the exact-mode quotient (reciprocal + two Markstein corrections) against IEEE
 * division on n generated operand pairs; result2 (device, 2 x u64) = {mismatches, tested}. */
int hx_selftest_division(uint64_t n, uint64_t seed, unsigned long long *result2, void *stream);

/* ---- numerical integration (Alg. 2) ----------------------------------------------------- */
/* element.py:213-245: coords (n,8,3) f64 pre-gathered, coeff (n,) f64 -> out (n,36) f64.
 * fail->element is batch-local (0-based); the caller adds element_offset. */
int hx_stiffness_batch(const double *coords, const double *coeff, int64_t n, double *out,
                       int32_t mode, hx_fail_info *fail, void *stream);

/* integrate_all for elements [lo, hi) straight from the device-resident mesh: no host
 * gather (integrate.py:146-149 disappears).  coords (n_nodes,3) f64, conn (n_el,8) i32,
 * coeff (n_el,) f64.  Writes ke (hi-lo, 36) and, when rows/cols are non-NULL, the fused
 * iK/jK triplet indices (36*(hi-lo),) i32 each (assemble.py:86-93).  fail->element is a
 * global element id. */
int hx_integrate_mesh(const double *coords, int64_t n_nodes, const int32_t *conn,
                      const double *coeff, int64_t lo, int64_t hi, double *ke, int32_t *rows,
                      int32_t *cols, int32_t mode, hx_fail_info *fail, void *stream);

/* hx_integrate_mesh fused with the first pass of the mesh-path assembly: the kernel also records
 * each node's incident (element << 3 | local node) slots in the adjacency section of a mesh-CSC
 * workspace (hx_mesh_csc_workspace_bytes(n_el, n_nodes) bytes) -- element e puts (e << 3 | a) in
 * slot a of its local node a, no atomics -- and validates node ids into csc_status
 * (HX_ST_BAD_INDEX).  reset != 0 empties the slots and zeroes the status first (the first element
 * range of a build).  Follow with hx_mesh_csc_build(...,
 * flags | HX_CSC_ADJACENCY_READY) on the same workspace and status.  Element ids must fit the
 * int32 adjacency: 8 * hi < 2^31. */
int hx_integrate_mesh_adjacency(const double *coords, int64_t n_nodes, const int32_t *conn,
                                const double *coeff, int64_t lo, int64_t hi, double *ke, int32_t *rows,
                                int32_t *cols, int32_t mode, hx_fail_info *fail, void *csc_workspace,
                                int64_t workspace_bytes, uint32_t *csc_status, int32_t reset, void *stream);

/* assemble.py:86-93 alone: rows/cols (36*(hi-lo),) i32 for elements [lo, hi). */
int hx_connectivity_index_arrays(const int32_t *conn, int64_t lo, int64_t hi, int32_t *rows,
                                 int32_t *cols, void *stream);

/* assemble.py:65-83 map_local_to_global for dofxn >= 1, element-major over elements [lo, hi):
 * rows/cols ((8 dofxn)(8 dofxn + 1)/2 * (hi-lo),) i32 -- local dof i = a * dofxn + k of node a is
 * global dof conn[e][a] * dofxn + k (node-major blocks), pairs in np.tril_indices(8 dofxn) order,
 * swapped to (max, min).  Assemble them with hx_triplet_csc_* (dim = n_nodes * dofxn).
 * n_nodes * dofxn must fit int32; 1 <= dofxn <= HX_MAX_DOFXN. */
#define HX_MAX_DOFXN 16
int hx_dof_index_arrays(const int32_t *conn, int64_t lo, int64_t hi, int64_t n_nodes, int32_t dofxn,
                        int32_t *rows, int32_t *cols, void *stream);

/* ---- mesh-path assembly (node-adjacency symbolic + deterministic column numeric) ---------
 * Builds the lower-triangular CSC block for columns [col_lo, col_hi) of a mesh with
 * n_nodes nodes, from element segments in ascending global element order.
 *   symbolic: writes col_ptr (col_hi-col_lo+1) i64 (col_ptr[0] = 0, nnz = col_ptr[last]) and
 *             row_idx i64 (ascending within each column) for the first row_capacity entries;
 *             when nnz > row_capacity the caller re-runs symbolic with row_capacity >= nnz.
 *   numeric:  writes vals (nnz) f64, summing duplicates in element order with numpy
 *             add.reduceat's rule (bitwise equal to assemble.py:135).
 * The workspace written by symbolic must be passed unchanged to numeric. */
/* Default workspace (scratch for 15 off-diagonal records per column); any larger workspace is
 * used in full as scratch. */
int64_t hx_mesh_csc_workspace_bytes(int64_t n_el_total, int64_t n_cols);
int hx_mesh_csc_symbolic(const hx_elem_segment *segs, int32_t n_segs, int64_t n_nodes,
                         int64_t col_lo, int64_t col_hi, int64_t *col_ptr, int64_t *row_idx,
                         int64_t row_capacity, void *workspace, int64_t workspace_bytes,
                         uint32_t *status, int32_t flags, void *stream);
/* symbolic + numeric in one pass (the cold build): col_ptr, row_idx and vals, the latter two for
 * the first `capacity` entries (re-run with capacity >= nnz when short). */
int hx_mesh_csc_build(const hx_elem_segment *segs, int32_t n_segs, int64_t n_nodes, int64_t col_lo,
                      int64_t col_hi, int64_t *col_ptr, int64_t *row_idx, double *vals, int64_t capacity,
                      void *workspace, int64_t workspace_bytes, uint32_t *status, int32_t flags, void *stream);
/* Symbolic with row_capacity = 0 only plans (col_ptr + workspace, no row_idx); hx_mesh_csc_emit
 * then writes row_idx and vals (first `capacity` entries) in one pass -- the split lets the plan run
 * on a second stream concurrently with the integration kernel. */
int hx_mesh_csc_emit(const hx_elem_segment *segs, int32_t n_segs, int64_t col_lo, int64_t col_hi,
                     const int64_t *col_ptr, int64_t *row_idx, double *vals, int64_t capacity,
                     const void *workspace, uint32_t *status, void *stream);
int hx_mesh_csc_numeric(const hx_elem_segment *segs, int32_t n_segs, int64_t col_lo,
                        int64_t col_hi, const int64_t *col_ptr, const int64_t *row_idx,
                        double *vals, const void *workspace, uint32_t *status, void *stream);

/* ---- integration fused with the emit pass (the cold build's second phase) ----------------------
 * hx_integrate_mesh (KE + iK/jK of every element, same outputs, fail record and bitwise results)
 * and hx_mesh_csc_emit (row_idx / vals of every column) in ONE persistent launch: the warps take
 * element quads and, as soon as every element a column tile touches has been integrated, the
 * tile's emit -- its KE gathers then hit the L2 lines the integration just wrote, and the DRAM-bound
 * emit work runs under the FP64-bound integration.  csc_workspace / col_ptr / csc_status: a plan of
 * the same connectivity from hx_mesh_csc_symbolic (row_capacity 0, one segment, columns
 * [0, n_nodes)); when its status word has a fast-path limit bit the launch only integrates and the
 * caller re-assembles.  sched_ws: hx_integrate_emit_workspace_bytes(n_el) bytes (scheduling
 * counters, reset by the call).  Entries beyond `capacity` are not written (re-run when
 * col_ptr[n_nodes] > capacity). */
int64_t hx_integrate_emit_workspace_bytes(int64_t n_el);
int hx_integrate_emit(const double *coords, int64_t n_nodes, const int32_t *conn, const double *coeff, int64_t n_el,
                      double *ke, int32_t *rows, int32_t *cols, int32_t mode, hx_fail_info *fail,
                      const int64_t *col_ptr, int64_t *row_idx, double *vals, int64_t capacity,
                      const void *csc_workspace, const uint32_t *csc_status, void *sched_ws, int64_t sched_bytes,
                      void *stream);

/* ---- generic triplet -> CSC (assemble.py:110-149) ----------------------------------------
 * symbolic: validates (status bits BAD_INDEX / UPPER), stable-sorts by (col,row), finds the
 *           duplicate runs and writes col_ptr (dim+1) i64 and row_idx (nnz) i64 where
 *           nnz = col_ptr[dim] (row_idx must hold n entries: nnz <= n).
 * numeric:  vals (n,) f64 -> out_vals (nnz,) f64 with numpy add.reduceat's summation rule
 *           (v0 + pairwise(v[1:]), any run length). */
int64_t hx_triplet_csc_workspace_bytes(int64_t n, int64_t dim);
int hx_triplet_csc_symbolic(const int32_t *rows, const int32_t *cols, int64_t n, int64_t dim,
                            int64_t *col_ptr, int64_t *row_idx, void *workspace,
                            int64_t workspace_bytes, uint32_t *status, void *stream);
int hx_triplet_csc_numeric(const double *vals, int64_t n, int64_t dim, const int64_t *col_ptr,
                           double *out_vals, const void *workspace, void *stream);

/* ---- multi-GPU exchange (element-range shards, nnz-balanced column blocks) ---------------------
 * The sharded build has no reference counterpart (the reference is single-process);
 * the blocks it produces are the reference's LowerCscMatrix (assemble.py:51-62) cut into column
 * ranges, bitwise.
 *
 * column_weights: hist[b] += nnz estimate (units of 1/8 entry) of the lower-CSC columns in bin
 *        b = node * n_bins / n_nodes, over the given elements (hex8 pair (i, j) adds 1 << (number of
 *        differing natural coordinates)).  Summed over ranks (all-reduce) and cut at equal prefix
 *        sums, it gives nnz-balanced column bounds.  hist (n_bins) u64 device, caller-zeroed.
 * col_bounds: (world+1) int64 device array, rank r owns columns [col_bounds[r], col_bounds[r+1]).
 * count: per_dest (world, 2) int64 device <- (records, values) each rank needs from this rank's
 *        elements: one record per element with a node in that rank's block, carrying the KE
 *        entries whose column (min of the pair's node ids) the rank owns; per_dest[self] = 0.
 * pack:  writes the records into dest_ptrs[d] + dest_offsets[d] (int64 words; device arrays of
 *        world entries -- a send buffer for an all-to-all, or receive buffers in peer memory):
 *        [ids: 4 words per record = the 8 int32 node ids][values: the owned entries, ascending
 *        packed index p, as f64 bit patterns], destination-major, ascending element order.  Must
 *        follow count with the same workspace.
 * unpack: recv = the chunks of every source in ascending source order; src_desc (world, 3) int64
 *        device = per source (word offset of its chunk in recv, records, values).  records
 *        (n_rec, 40) f64 <- 36 KE words (entries this rank does not own are 0) + the 8 ids, i.e.
 *        an hx_elem_segment with conn_stride 80, ke_stride 40.
 * digest: *out += sum_i mix(mix(pos0 + i) ^ (word_i + add)) (mod 2^64) over n_words 8-byte words --
 *        a position-keyed checksum whose sum over the ranks' blocks equals that of the whole array. */
int hx_column_weights(const int32_t *conn, int64_t n_el, int64_t n_nodes, int64_t n_bins, uint64_t *hist,
                      void *stream);
/* touch: hist[b] += 8 per element with a node in bin b (each distinct bin of the element once) -- the
 *        per-element work of a column block (received records, adjacency), blended with the nnz
 *        weights so randomly numbered meshes balance records as well as nnz.  Caller-zeroed. */
int hx_column_touch(const int32_t *conn, int64_t n_el, int64_t n_nodes, int64_t n_bins, uint64_t *hist,
                    void *stream);
int64_t hx_halo_workspace_bytes(int64_t n_el, int32_t world);
int hx_halo_count(const int32_t *conn, int64_t n_el, const int64_t *col_bounds, int32_t world, int32_t self,
                  int64_t *per_dest, void *workspace, int64_t workspace_bytes, void *stream);
int hx_halo_pack(const int32_t *conn, const double *ke, int64_t n_el, const int64_t *col_bounds, int32_t world,
                 int32_t self, int64_t *const *dest_ptrs, const int64_t *dest_offsets, const void *workspace,
                 void *stream);
int64_t hx_halo_unpack_workspace_bytes(int64_t n_rec);
int hx_halo_unpack(const int64_t *recv, const int64_t *src_desc, int32_t world, int32_t self,
                   const int64_t *col_bounds, int64_t n_rec, double *records, void *workspace,
                   int64_t workspace_bytes, void *stream);
/* index: the received records as compact element segments without moving their values: conn
 *        (n_rec, 8) i32 <- the ids, ke_offset (n_rec) i64 <- word index in recv of the record's first
 *        value, ke_mask (n_rec) u64 <- the packed entries this rank owns (see hx_elem_segment).
 *        Workspace: hx_halo_unpack_workspace_bytes(n_rec). */
int hx_halo_index(const int64_t *recv, const int64_t *src_desc, int32_t world, int32_t self,
                  const int64_t *col_bounds, int64_t n_rec, int32_t *conn, int64_t *ke_offset, uint64_t *ke_mask,
                  void *workspace, int64_t workspace_bytes, void *stream);
int hx_digest(const void *data, int64_t n_words, int64_t pos0, uint64_t add, uint64_t *out, void *stream);

/* CUDA IPC receive buffers of the fused pack-and-send exchange (the one allocating entry point: an
 * IPC handle needs its own cudaMalloc base).  alloc: device buffer + its 64-byte handle; open: maps
 * a handle of ANOTHER process into the current device's context with lazy peer access (NVLink
 * stores from this device's kernels into the owner's GPU); close / free undo them. */
#define HX_IPC_HANDLE_BYTES 64
int hx_ipc_alloc(int64_t bytes, void **ptr, void *handle);
int hx_ipc_open(const void *handle, void **ptr);
int hx_ipc_close(void *ptr);
int hx_ipc_free(void *ptr);

/* ---- column blocks of one GPU (out-of-core build, Eq. 10 beyond HBM) ---------------------------
 * select: ids (n_el capacity) i64 device <- ascending ids of the elements with a node in
 *         [col_lo, col_hi); *count (device) = their number.  Stable: the block's elements keep the
 *         global element order, so duplicates are summed exactly as in the one-shot build.
 * gather: conn_out (count, 8) i32 / coeff_out (count,) f64 <- those elements' rows; capacity bounds
 *         the launch (>= count). */
int64_t hx_block_select_workspace_bytes(int64_t n_el);
int hx_block_select(const int32_t *conn, int64_t n_el, int64_t col_lo, int64_t col_hi, int64_t *ids,
                    int64_t *count, void *workspace, int64_t workspace_bytes, void *stream);
int hx_block_gather(const int32_t *conn, const double *coeff, const int64_t *ids, const int64_t *count,
                    int64_t capacity, int32_t *conn_out, double *coeff_out, void *stream);
/* ranges (HOST code): for the streamed column-block build of a locally numbered mesh -- e_lo[k] /
 *         e_hi[k] (n_blocks each) = the element range whose node span covers block k = columns
 *         [bounds[k], bounds[k+1]) (a superset of the elements touching it; 0/0 when none).  conn
 *         (n_el, 8) int32 HOST array, `threads` workers (<= 0: all). */
int hx_block_ranges(const int32_t *conn, int64_t n_el, const int64_t *bounds, int32_t n_blocks, int64_t *e_lo,
                    int64_t *e_hi, int32_t threads);
/* as hx_block_ranges, plus node_lo / node_hi (n_blocks each): a node range [node_lo, node_hi) that
 * holds every node the elements [e_lo[k], e_hi[k]) reference (bounded per chunk of 2^20 elements;
 * the streamed build uploads the coordinates as prefixes ahead of each block).  HOST code. */
/* a predicted plan from every step-th element (the streamed run_build's fast start), checked on the
 * device by hx_block_verify: element e0 + i (i < n, conn = the block's uploaded range) must lie in the
 * predicted range of every block its node span covers and reference only nodes below node_top;
 * failures set *flag (1: range, 2: coordinates) and the caller rebuilds with the exact scan. */
int hx_block_ranges_sampled(const int32_t *conn, int64_t n_el, const int64_t *bounds, int32_t n_blocks, int64_t step,
                            int64_t *e_lo, int64_t *e_hi, int64_t *node_hi, int32_t threads);
int hx_block_verify(const int32_t *conn, int64_t n, int64_t e0, int64_t n_nodes, const int64_t *bounds,
                    int32_t n_blocks, const int64_t *e_lo, const int64_t *e_hi, int64_t node_top, uint32_t *flag,
                    void *stream);
int hx_block_ranges_nodes(const int32_t *conn, int64_t n_el, const int64_t *bounds, int32_t n_blocks, int64_t *e_lo,
                          int64_t *e_hi, int64_t *node_lo, int64_t *node_hi, int32_t threads);

/* ---- structured box in device memory (mesh.py:73-98 generate_cube_mesh) --------------------------
 * coords (n_nodes, 3) f64, conn (n_el, 8) i32, coeff (n_el,) f64: node (i,j,k) at (i h, j h, k h)
 * with id i + j (nx+1) + k (nx+1)(ny+1), x-fastest elements, local order
 * [0, 1, 1+sx, sx, L, 1+L, 1+sx+L, sx+L] -- bitwise the reference generator's arrays. */
int hx_generate_cube_mesh(int64_t nx, int64_t ny, int64_t nz, double h, double c0, double *coords, int32_t *conn,
                          double *coeff, void *stream);

/* ---- compact device -> host transfer of the lower CSC (12 instead of 16 bytes per entry) -------
 * narrow: rows32[i] = (int32) row_idx[i] on the device (node ids are int32 in the reference).
 * widen:  row_idx[i] = rows32[i] on the host with `threads` worker threads (<= 0: all), giving back
 *         the reference's int64 row_idx (assemble.py:51-62).  Host code. */
int hx_rows_narrow(const int64_t *row_idx, int32_t *rows32, int64_t n, void *stream);
/* peek: up to HX_PEEK_MAX 4- or 8-byte device words -> host_dst[i] (int64; 4-byte words sign-
 * extended) written by a kernel into MAPPED pinned host memory (cudaHostAlloc / pinned torch
 * tensors), so the read does not queue behind bulk copies on the copy engines; the caller
 * synchronises the stream before reading host_dst. */
#define HX_PEEK_MAX 8
typedef struct hx_peek_args {
    const void *src[HX_PEEK_MAX];
    int32_t bytes[HX_PEEK_MAX];
    int32_t n;
} hx_peek_args;
int hx_peek(const hx_peek_args *args, int64_t *host_dst, void *stream);
int hx_rows_widen(const int32_t *rows32, int64_t *row_idx, int64_t n, int32_t threads);

/* Row-index codec of the device -> host transfer (the PCIe bytes bound the end-to-end build).
 * encode (device): each column's ascending rows as deltas from the column id / previous row, in
 *   Stream-VByte groups of 4 (one control byte of 2-bit byte lengths, then the deltas' little-endian
 *   bytes; a partial last group padded with 1-byte zeros), columns concatenated.  counts (ncols) u8
 *   = rows per column (col_ptr differences), lens (ncols) u8 = bytes per column, bytes = the stream
 *   (capacity bytes; 5 * nnz + 17 * ncols always suffices); *total (device int64) = stream bytes, or
 *   -1 when a column has more than 36 rows (send the rows uncompressed instead).  Workspace:
 *   hx_rows_encode_workspace_bytes(ncols).
 * decode (HOST): rows_out (int64, sum(counts) entries) and col_ptr_out (ncols entries: row_base +
 *   the rows of columns 0..j) from counts / lens / bytes; all host cores (threads <= 0) or the given
 *   count; bytes must be readable for 16 bytes past nbytes.  SSSE3 + SSE4.1. */
int64_t hx_rows_encode_workspace_bytes(int64_t ncols);
int hx_rows_encode(const int64_t *col_ptr, const int64_t *row_idx, int64_t ncols, int64_t col_lo, uint8_t *counts,
                   uint8_t *lens, uint8_t *bytes, int64_t capacity, int64_t *total, void *workspace,
                   int64_t workspace_bytes, void *stream);
int hx_rows_decode(const uint8_t *counts, const uint8_t *lens, const uint8_t *bytes, int64_t nbytes, int64_t ncols,
                   int64_t col_lo, int64_t row_base, int64_t *col_ptr_out, int64_t *rows_out, int32_t threads);

/* ---- Matrix Market export (sparseio.py:73-87), host code -----------------------------------------
 * Host arrays of a lower CSC -> "%%MatrixMarket matrix coordinate real symmetric" file, 1-based,
 * column-major, "%.17g" values: byte-identical to the reference's writer, formatted by `threads`
 * worker threads (<= 0: all hardware threads). */
int hx_mm_write(const int64_t *col_ptr, const int64_t *row_idx, const double *vals, int64_t dim, const char *path,
                int32_t threads);
/* Import (sparseio.py:90-138), host code: rows == NULL queries (n_rows, nnz); then fills rows/cols
 * (0-based int32) and vals.  Returns 0 ok, 1 = outside the strict fast path (the caller re-reads with
 * the reference's own rules), 2 = format error at *err_line (message in hx_last_error). */
int hx_mm_read(const char *path, int64_t *n_rows, int64_t *nnz, int32_t *rows, int32_t *cols, double *vals,
               int64_t *err_line);

#ifdef __cplusplus
}
#endif
#endif /* HEXFEM_B200_H */
