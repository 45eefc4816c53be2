/*
 * lb.h -- C ABI of liblb.so: CSR SpMV y = A x under a programmable load-balancing
 * schedule, B200-native (sm_100a).  The hot path of arXiv 2212.08964 (Osama, "GPU load
 * balancing"), Ch.3-4.
 *
 * Citations: "P:L" = PAPER.md line L [section / algorithm / listing].
 *
 * Conventions (all entry points)
 *  - Plain pointers and sizes only.  "d_" pointers are CUDA device pointers, "h_" pointers
 *    are host pointers.  A `stream` argument is a cudaStream_t passed as void* (NULL = the
 *    legacy default stream).
 *  - Ownership: every caller array is BORROWED.  A handle (lb_csr_t) keeps the device
 *    pointers given to lb_csr_create; they must outlive the handle and stay unmodified while
 *    calls are in flight.  A handle owns only its scratch (partition cache, carries), which is
 *    allocated at create time so that lb_spmv can be captured in a CUDA graph.
 *  - Asynchrony: every call is stream-ordered and does not synchronise the host, except
 *    lb_csr_create(validate=1) (one sync to read the validation flag), lb_spmv_host and
 *    lb_spmv_host_x (return with y on the host), lb_spmv_host_x_wait, the lb_comm_* setup calls,
 *    and the first LB_SPMV_CHUNKED call per tile length (one sync to read the chunk cuts; in
 *    lb_spmv_multi_ex also to exchange them).
 *  - Errors: a status code is returned; no exception crosses the ABI.  lb_last_error()
 *    returns a thread-local message for the last failing call on this thread.
 *  - Index widths: int32 row offsets and column indices, fp32 values, x and y (P:963-969,
 *    Listing 3).  Sizes are int64; rows + nnz must be <= 2^31 - 2^16 - 1 (int32 indices with headroom
 *    for tile overshoot; reading R13).
 *  - y is OVERWRITTEN (y = A x, not y += A x; "y[row] = sum", Alg.3).
 *  - Empty rows produce y = +0 (P:982 with the zero-initialised sum); rows == 0 is a no-op.
 *  - There is no CPU fallback: every compute call runs CUDA kernels of this library and
 *    fails with LB_ERR_CUDA if no device is usable.
 */
#ifndef LB_H
#define LB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LB_OK = 0,
  LB_ERR_INVALID_ARG = 1,  /* null pointer with non-zero size, negative size, rows+nnz > 2^31-2^16-1,
                              unknown schedule, unsupported items_per_tile, x aliasing y, ... */
  LB_ERR_INVALID_CSR = 2,  /* validation failed: off[0] != 0, off not non-decreasing,
                              off[rows] != nnz, or a column index outside [0, cols) */
  LB_ERR_UNSUPPORTED = 3,  /* feature not available in this build (e.g. NCCL not loadable) */
  LB_ERR_OOM = 4,          /* device or host allocation failed */
  LB_ERR_CUDA = 5,         /* a CUDA runtime call failed (message in lb_last_error) */
  LB_ERR_NCCL = 6          /* an NCCL call failed or reported an asynchronous error */
} lb_status_t;

/*
 * Load-balancing schedules ("update a single C++ enum ... to select the desired load
 * balancing schedule").
 *  THREAD_MAPPED   one row (work tile) per thread, atoms of the row processed sequentially,
 *                  grid-stride over rows; 256 threads per block, ceil(rows/256) blocks
 *                  (P:211-237 [Sec. Thread-Mapped]; Listings 2-3 P:904-990).
 *  GROUP_MAPPED    group of G = 32 lanes (a warp) takes G consecutive rows per round: lanes
 *                  load their row's atom count, the group prefix-sums them, lanes stride the
 *                  group's atom pool by G and find each atom's row by binary search in the
 *                  prefix sum (P:241-281 [Sec. Group-Mapped], Alg.2).  Products
 *                  are summed per row by a deterministic segmented reduction (reading R8).
 *  MERGE_PATH      work-oriented merge-path: rows + nnz merge items split evenly into tiles of
 *                  L items; per tile the (row, nz) start comes from the 2-D diagonal search;
 *                  complete rows are written, the trailing partial row is carried out and
 *                  fixed up after all tiles (P:283-339 [Sec. Work-Oriented], Alg.3;
 *                  P:1018-1028 [Sec. Merge-path load balancing]).
 *  BLOCK_MAPPED    GROUP_MAPPED with G = 256 (a CTA) -- the block-mapped instance the paper gets
 *                  "for free" from the group-mapped schedule (table).
 *  NONZERO_SPLIT   work-oriented with nonzeros as the only work items (table): tiles of
 *                  1016 nonzeros, each tile's first row found by a 1-D binary search of
 *                  row_offsets (lb_partition_nz); rows without nonzeros cost no work, so tiles may
 *                  span arbitrarily many empty rows.  Runs on the merge-path tile processor.
 *  WARP_MAPPED     warp-level load balancing: every warp takes an equal share of rows
 *                  (a contiguous run) and processes them one at a time, the 32 lanes striding the
 *                  row's atoms by 32 ("CSR-vector"); fixed xor-tree sum over the lanes.
 *  BINNING         three-bin schedule (Alg.4; three kernels): rows with >= 256
 *                  nonzeros are processed by a CTA each, rows with >= 32 by a warp each, the rest by
 *                  a thread each; the bins are rebuilt on the device in every call (count, scan,
 *                  stable scatter -- ascending row ids per bin, reading R21), no host sync.
 *  AUTO            the paper's heuristic: merge-path unless (rows < alpha or cols < alpha)
 *                  and nnz < beta (alpha = 500, beta = 10000), then thread-mapped; extended with a
 *                  row-regularity test for B200 (reading R18): thread-mapped when the longest row
 *                  is at most 2 x mean + 8 and the mean is <= 32 nonzeros.  The row-length maximum
 *                  is computed once per handle by a reduction kernel (first AUTO call; one sync).
 */
typedef enum {
  LB_SCHED_THREAD_MAPPED = 0,
  LB_SCHED_GROUP_MAPPED = 1,
  LB_SCHED_MERGE_PATH = 2,
  LB_SCHED_BLOCK_MAPPED = 3,
  LB_SCHED_AUTO = 4,
  LB_SCHED_NONZERO_SPLIT = 5,
  LB_SCHED_WARP_MAPPED = 6,
  LB_SCHED_BINNING = 7
} lb_schedule_t;


typedef struct lb_csr_s* lb_csr_t;   /* opaque CSR handle (borrowed arrays + owned scratch) */
typedef struct lb_comm_s* lb_comm_t; /* opaque multi-GPU communicator (wraps an ncclComm_t) */

/* Merge-path tile length L (merge items per tile).  Supported lengths are 504, 1016, 2040, 3064 and
 * 4088 (= 256*R - 8 or NT*E - 8: a tile's 32-byte-aligned range of nonzeros spans at most L + 7
 * elements, so every lane of the processing warp/CTA gets the same number of slots).  The handle's
 * default is chosen from the shape at lb_csr_create: 2040 when nnz < 8*rows (short rows), else
 * 1016.  LB_DEFAULT_ITEMS_PER_TILE is the long-row default. */
#define LB_DEFAULT_ITEMS_PER_TILE 1016

/*
 * lb_csr_create -- borrow a CSR matrix (P:149 [Sec. CSR]: row offsets = prefix sum of row
 * lengths, column indices and values in row-major order).
 *  rows, cols, nnz     matrix shape and number of stored entries (>= 0; rows + nnz <= 2^31 - 2^16 - 1,
 *                      cols < 2^31 - 1).
 *  d_row_offsets       int32[rows+1], d_col_idx int32[nnz], d_values fp32[nnz] (device).
 *  validate            1: run the validation kernel (off[0] = 0, off non-decreasing,
 *                      off[rows] = nnz, 0 <= col < cols) and synchronise `stream` once to read
 *                      the result; failure returns LB_ERR_INVALID_CSR naming the first
 *                      offending index.  0: trust the caller (no sync).
 *  out                 receives the handle; release with lb_csr_destroy.
 * Duplicate and unsorted column indices are allowed (SpMV is linear in stored entries).
 */
lb_status_t lb_csr_create(int64_t rows, int64_t cols, int64_t nnz, const int32_t* d_row_offsets,
                          const int32_t* d_col_idx, const float* d_values, int32_t validate,
                          void* stream, lb_csr_t* out);

/* lb_csr_destroy -- free the handle's scratch (after all work using it has completed). */
lb_status_t lb_csr_destroy(lb_csr_t A);

/*
 * lb_csr_set_items_per_tile -- choose the merge-path tile length L used by lb_spmv
 * (0 = the shape-based default described at LB_DEFAULT_ITEMS_PER_TILE).  Supported: 504, 1016, 2040, 3064, 4088; anything else returns
 * LB_ERR_INVALID_ARG.
 * Invalidates the cached partition.  Not thread-safe with respect to in-flight lb_spmv.
 */
lb_status_t lb_csr_set_items_per_tile(lb_csr_t A, int32_t items_per_tile);

/*
 * lb_partition_size -- number of merge-path tiles T = ceil((rows + nnz) / L) for tile length
 * L = items_per_tile (0 = the handle's current L).  Host-only, no device work.
 */
lb_status_t lb_partition_size(lb_csr_t A, int32_t items_per_tile, int64_t* num_tiles);

/*
 * lb_partition -- merge-path partition (Alg.3 P:306-311 "2DSearch").
 * For t = 0..T with d_t = min(t*L, rows+nnz), writes the coordinate
 *   (i_t, j_t):  i_t = #{ k < rows : k + off[k+1] < d_t },  j_t = d_t - i_t
 * (the number of row ends and of nonzeros that precede diagonal d_t in the merge of the row
 * ends with the nonzero indices; a row end precedes nonzero off[k+1] -- reading R1).
 *  items_per_tile  L >= 1 (any value; 0 = the handle's current L).
 *  d_coords        int32[(T+1)*2] device buffer, (row, nz) pairs, caller-owned.
 * Bit-exact: integer arithmetic only.
 */
lb_status_t lb_partition(lb_csr_t A, int32_t items_per_tile, int32_t* d_coords, void* stream);

/*
 * lb_partition_nz -- nonzero-splitting partition: T = max(1, ceil(nnz / L)) tiles of L
 * nonzeros (L = items_per_tile >= 1; 0 = 1016); for 0 < t < T writes (i_t, j_t) with
 * j_t = t*L and i_t = #{ r : off[r+1] <= j_t } (every row ending at or before nonzero j_t), plus
 * (0, 0) and (rows, nnz).  d_coords: int32[(T+1)*2] device.  Bit-exact.
 */
lb_status_t lb_partition_nz(lb_csr_t A, int32_t items_per_tile, int32_t* d_coords, void* stream);

/*
 * lb_spmv -- y = A x under schedule `sched` (Listing 3; Alg.3).
 *  d_x  fp32[cols] device; d_y  fp32[rows] device (overwritten); x and y must not alias.
 * MERGE_PATH uses the handle's cached partition at its L, computing it on the first call.
 * Arithmetic: fp32 products and fp32 accumulation (reading R12); deterministic (bitwise
 * identical results for identical inputs and launch configuration).
 */
lb_status_t lb_spmv(lb_csr_t A, lb_schedule_t sched, const float* d_x, float* d_y, void* stream);

/* lb_select_schedule -- the concrete schedule LB_SCHED_AUTO resolves to for this handle (computes
 * and caches the row statistics on first use: one reduction kernel + one sync of `stream`). */
lb_status_t lb_select_schedule(lb_csr_t A, void* stream, lb_schedule_t* out);

/*
 * lb_spmm -- Y = A X for a dense X with n columns (Listing 4: SpMM is SpMV with a loop
 * over the columns of B), on the same merge-path tiles (L = 1016; lb_partition's output at that
 * length is reused).  X: fp32 [cols x n] row-major with leading dimension ldx >= n; Y: fp32
 * [rows x n], leading dimension ldy >= n, overwritten.  Columns are processed in panels: 32 or 16
 * columns with lanes over columns (lane c of a P-lane group gathers X[col, c]; needs 32-byte
 * aligned col_idx/values, ldy a multiple of 4 and a 16-byte aligned Y panel), otherwise 8 columns
 * with one 32-byte gather of X[col, c..c+8) per nonzero (X rows 32-byte aligned), 4 columns with one
 * 16-byte gather (16-byte aligned, ldx and ldy multiples of 4), or one column at a time.  X and Y must not
 * alias.  Errors: LB_ERR_INVALID_ARG for a null handle, n < 0, ldx < n, ldy < n, null X / Y with
 * work to do, or X == Y.
 */
lb_status_t lb_spmm(lb_csr_t A, int64_t n, const float* d_X, int64_t ldx, float* d_Y, int64_t ldy, void* stream);

/*
 * lb_csr_plan_hot_x -- x-reuse plan for MERGE_PATH (B200 extension; not in the paper -- DESIGN.md
 * section 6b).  Background: a merge-path tile reads col/val as a stream but x[col] as random 4-byte
 * gathers (Listing 3 P:980 `x[column_indices[nz]]`).  On B200 every gather that misses L1 costs a
 * 32-byte L2 sector and an L1TEX wavefront, and when x exceeds the L2 a DRAM sector too, while
 * shared memory serves random 4-byte reads several times faster.  The plan orders the columns by
 *   deg(c) = number of stored entries in column c  (candidates: deg(c) >= 2)
 * and builds two tiers:
 *  HOT   fewer than `slots` candidates: all are hot, slots numbered in ascending column order;
 *        otherwise the first `slots` candidates ordered by (deg descending, column ascending); with
 *        tau1 = the smallest degree among them, slots go first to the hot columns with deg > tau1,
 *        then to those with deg == tau1, each in ascending column order.
 *  WARM  (only when the hot tier is full and warm_cols > 0) the non-hot columns with
 *        deg >= tau2, where tau2 is the smallest degree >= 2 with #{deg >= tau2} <= slots +
 *        warm_cols (whole degree levels; warm_cols is an upper bound), provided tau2 <= tau1;
 *        numbered in ascending column order.
 * and a private copy of col_idx in which an entry of hot column c holds ~slot(c) (< 0), an entry
 * of warm column c holds cols + warm_index(c), other entries keep c.  With a plan, every
 * lb_spmv(MERGE_PATH) call (L = 504 or 1016) gathers x of the hot and warm columns once (warm
 * columns ascend, so that gather sweeps x in address order), each CTA stages the hot values in
 * shared memory, and the tile kernel reads warm values from the dense copy (kept in L2 with an
 * evict_last policy; cold x reads use evict_first).  Products and summation order are unchanged:
 * y is bitwise identical to the call without a plan.  Other schedules ignore the plan.
 *  slots          0 = automatic: the default budget (16384: 64 KB of shared memory per SM), and no plan
 *                 where it cannot pay -- the handle's tile length has no plan kernel (only 504 and 1016
 *                 do), or x fits in the L2 (no warm tier) and the hot columns hold < 0.5% of the stored
 *                 entries; 1 .. 45056 = that budget, always built; < 0 drops the plan.
 *  warm_cols      0 = no warm tier; -1 = auto (a 48 MB budget when x (4*cols bytes) is larger
 *                 than the L2, else none); > 0 = budget in columns; -2 = compact x: EVERY
 *                 referenced non-hot column is warm (numbered in ascending column order), its entry
 *                 holds the warm index itself, each call builds x_warm by a mask-driven compaction
 *                 sweep over x (fused into the partition launch) and the tile kernel gathers from
 *                 x_warm as its x -- the gathered footprint shrinks from all of x to the referenced
 *                 columns.  Falls back to no warm tier when the hot set is not full.
 *  hot_cols_out   (optional) number of planned hot columns (0: no plan was kept).
 *  hot_nnz_out    (optional) number of stored entries in hot columns.
 * Cost: device memory 4*nnz + 8*(hot + warm) + 4*cols (temporary); a degree histogram, a few
 * selection passes and a remap of col_idx; synchronises `stream`.  The caller's arrays are not
 * modified.  Errors: LB_ERR_UNSUPPORTED if col_idx/values are not 32-byte aligned; LB_ERR_OOM;
 * LB_ERR_INVALID_ARG for slots > 45056 or warm_cols < -2.  Re-plan (or drop the plan) after
 * modifying col_idx.
 */
lb_status_t lb_csr_plan_hot_x(lb_csr_t A, int32_t slots, int64_t warm_cols, void* stream, int32_t* hot_cols_out,
                              int64_t* hot_nnz_out);

/* lb_csr_hot_plan -- inspect the plan (tests): numbers of hot / warm columns and their stored
 * entries (0: no plan / no warm tier); when a plan exists, copies (stream-ordered, device to device,
 * each pointer optional) the hot slot -> column table into d_hot_cols_out int32[hot_n], the warm
 * index -> column table into d_warm_cols_out int32[warm_n] and the remapped column stream into
 * d_col_out int32[nnz] (caller-owned device buffers). */
lb_status_t lb_csr_hot_plan(lb_csr_t A, int32_t* hot_n, int64_t* hot_nnz, int64_t* warm_n, int64_t* warm_nnz,
                            int32_t* d_hot_cols_out, int32_t* d_warm_cols_out, int32_t* d_col_out, void* stream);

/*
 * lb_sssp -- single-source shortest paths on the graph A (NEXT-4; Listing 5, "Loop until
 * the frontier is empty"): row u of A lists u's out-edges, col_idx = neighbour, values = weight
 * (>= 0).  Every round relaxes the out-edges of the current frontier,
 *   dist[v] = min(dist[v], dist[u] + w)     (fp32 add; atomicMin on the int32 view of non-negative floats)
 * and the vertices whose distance dropped form the next frontier (each vertex at most once per
 * round).  The round's edges are load-balanced by `sched`: THREAD_MAPPED (a thread per frontier
 * vertex), GROUP_MAPPED / BLOCK_MAPPED (a warp takes 32 frontier vertices and strides their pooled
 * edges, Alg.2), MERGE_PATH / AUTO / NONZERO_SPLIT (frontier vertices + edges split evenly, 16 merge
 * items per thread, each thread's start found by the 2-D search of Alg.3 over the frontier's
 * degree prefix).  The result is the least fixed point of the relaxation, identical to Dijkstra
 * with fp32 path sums (tests/test_gpu_sssp.py).
 *  source      0 <= source < rows;   d_dist  fp32[rows] device (output; +inf if unreachable).
 *  rounds_out  (optional) number of frontier rounds.
 * Requires rows == cols.  Synchronises `stream` once per round.  Allocates a 16*rows-byte workspace
 * in the handle on first use.  Errors: LB_ERR_INVALID_ARG for a negative or NaN weight (checked
 * before the first round), a bad source or a non-square matrix.
 */
lb_status_t lb_sssp(lb_csr_t A, int64_t source, lb_schedule_t sched, float* d_dist, void* stream, int32_t* rounds_out);

/*
 * lb_bins -- the three bins of the BINNING schedule (Alg.4): rows with >= 256 nonzeros
 * (CTA bin), >= 32 (warp bin), the rest (thread bin), each in ascending row order (reading R21).
 *  d_ids     int32[rows] device (output): [CTA bin | warp bin | thread bin].
 *  h_sizes   int64[3] host (output): the bin sizes.
 * Synchronises `stream` once (to read the sizes).  Allocates the handle's binning workspace
 * (4*rows bytes + 12 bytes per 1024 rows) on first use.
 */
lb_status_t lb_bins(lb_csr_t A, int32_t* d_ids, int64_t h_sizes[3], void* stream);

/* Flags for lb_spmv_ex. */
#define LB_SPMV_REPARTITION 1u /* MERGE_PATH: recompute the partition inside this call */
#define LB_SPMV_PADDED 4u      /* lb_spmv_multi_ex: padded all-gather layout (see lb_spmv_multi_ex) */
#define LB_SPMV_CHUNKED 2u     /* lb_spmv_host_x, MERGE_PATH with an x-reuse plan: run the tile kernel as
                                  up to 8 launches over tile ranges cut at clean merge-path coordinates
                                  (no row split across a cut) and copy each range's y rows to the host
                                  while the next range computes.  Same products; a row's summation
                                  order can differ from the one-launch call (carries per launch), so
                                  y is within tolerance of it, bit-exact in integer mode.
                                  lb_spmv_multi_ex: the same cuts on every rank's shard; once chunk c is
                                  done, an NCCL group of broadcasts sends every rank's chunk-c rows (on an
                                  exchange stream of the handle) while chunk c+1 computes.  Collective:
                                  all ranks pass it, with the same tile length, and build or drop their
                                  plans together (the cut table is exchanged on the first such call and
                                  after a plan change).  A rank without a plan sends its rows as one
                                  chunk. */

/* lb_spmv_ex -- lb_spmv with flags (LB_SPMV_REPARTITION: the whole merge-path method --
 * partition, tile processing, fix-up -- runs in this call; used by bench.py's step). */
lb_status_t lb_spmv_ex(lb_csr_t A, lb_schedule_t sched, const float* d_x, float* d_y, uint32_t flags,
                       void* stream);

/*
 * lb_spmv_host -- end-to-end y = A x from HOST buffers (ideally pinned): copies the CSR arrays
 * and x host->device into `d_workspace`, builds a transient handle (no validation), partitions,
 * runs `sched`, copies y device->host and synchronises `stream` before returning.
 *  d_workspace      device buffer of at least lb_spmv_host_workspace_size(rows, cols, nnz)
 *                   bytes (caller-owned; reused across calls to avoid allocation).
 */
size_t lb_spmv_host_workspace_size(int64_t rows, int64_t cols, int64_t nnz);
lb_status_t lb_spmv_host(int64_t rows, int64_t cols, int64_t nnz, const int32_t* h_row_offsets,
                         const int32_t* h_col_idx, const float* h_values, const float* h_x, float* h_y,
                         lb_schedule_t sched, void* d_workspace, size_t workspace_bytes, void* stream);

/*
 * lb_spmv_host_x -- end-to-end y = A x for a device-resident matrix with HOST x and y (the
 * iterative-solver call: A is uploaded once, every call moves only x in and y out): copies h_x
 * [cols] host->device into a staging buffer the handle owns (allocated on the first call, freed
 * by lb_csr_destroy), runs `sched` with `flags` (as lb_spmv_ex), copies y [rows] device->host
 * into h_y and synchronises `stream` before returning.  Pinned host buffers give full PCIe
 * bandwidth.  Errors: LB_ERR_INVALID_ARG (null handle, null h_x / h_y with work to do),
 * LB_ERR_OOM (staging allocation), LB_ERR_CUDA; the schedule's own errors as lb_spmv.
 */
lb_status_t lb_spmv_host_x(lb_csr_t A, lb_schedule_t sched, const float* h_x, float* h_y, uint32_t flags,
                           void* stream);

/*
 * lb_spmv_host_x_async / lb_spmv_host_x_wait -- the same y = A x with HOST x and y as lb_spmv_host_x,
 * for a stream of independent right-hand sides (many x vectors against one resident matrix, e.g. a
 * serving batch): the call only ENQUEUES the pinned H2D copy of h_x [cols] into one of three staging
 * slots the handle owns (on an H2D stream of its own), the SpMV of `sched` with `flags` on `stream`
 * (as lb_spmv_ex; it waits for that copy) and the D2H copy of y [rows] into h_y (on a D2H stream of
 * its own, after the SpMV), and returns.  Consecutive calls rotate through the slots, so call k's
 * H2D, call k-1's SpMV and call k-2's D2H can run at once (PCIe is full duplex); a call reuses a slot
 * only after the SpMV and the D2H of the call three back on it (stream-ordered event waits, no host
 * sync).  Ownership: h_x must stay unmodified and h_y untouched until lb_spmv_host_x_wait returns;
 * h_y holds y after lb_spmv_host_x_wait(A), which blocks until every enqueued call's y is on the
 * host.  Pinned host buffers are required for the copies to overlap.  Products and summation order
 * are those of lb_spmv_ex, so y is bitwise equal to lb_spmv_host_x for the same inputs.  Staging,
 * streams and events are allocated on the first call and freed by lb_csr_destroy.  Errors:
 * LB_ERR_INVALID_ARG (null handle, null h_x / h_y with work to do), LB_ERR_OOM, LB_ERR_CUDA; the
 * schedule's own errors as lb_spmv.  Not in the paper: host-side pipelining around P:123's y = A x.
 */
lb_status_t lb_spmv_host_x_async(lb_csr_t A, lb_schedule_t sched, const float* h_x, float* h_y,
                                 uint32_t flags, void* stream);
lb_status_t lb_spmv_host_x_wait(lb_csr_t A);

/*
 * lb_spmv_phase_times -- diagnostics: run `sched` once with CUDA events between its kernels on
 * `stream`, synchronise, and report milliseconds per phase in ms_out[3] = {partition, main
 * kernel, fix-up} (unused phases are 0).  MERGE_PATH recomputes the partition.
 */
lb_status_t lb_spmv_phase_times(lb_csr_t A, lb_schedule_t sched, const float* d_x, float* d_y, void* stream,
                                float* ms_out);

/*
 * lb_csr_trace_phases -- per-call phase timing of the next `capacity` lb_spmv* calls on this handle
 * (0 disables and frees).  Each traced call records four CUDA events on its stream (start, partition
 * done, main kernel done, fix-up done); lb_csr_trace_read synchronises on the last one, writes
 * ms_out[c*3 + {0,1,2}] = (partition, main, fix-up) milliseconds of traced call c (n_out calls) and
 * resets the trace (the capacity stays).  For measuring the dominant kernel inside a timed region of
 * back-to-back calls (bench.py); the event records may defeat the PDL overlap of partition and tile
 * kernel, so the region's own step time is reported beside it.
 */
lb_status_t lb_csr_trace_phases(lb_csr_t A, int32_t capacity);
lb_status_t lb_csr_trace_read(lb_csr_t A, int32_t* n_out, float* ms_out);

/*
 * lb_probe_stream_gather -- diagnostics: time (CUDA events, synchronises `stream`) a kernel that
 * streams A's col_idx/values with the tile processor's 256-bit loads and gathers x[col] with no
 * row structure, `reps` times; ms_out = mean milliseconds per pass.  nnz / ms_out is the
 * stream+gather ceiling for this matrix on this GPU (the bound of the merge-path tile processor
 * on random-column matrices).  With an x-reuse plan (lb_csr_plan_hot_x) the
 * probe streams the plan's column stream and serves hot / warm columns exactly as the tile kernel
 * does (x_hot staged in shared memory, one CTA of 16 warps per SM) -- the ceiling of the plan.
 * Needs 32-byte aligned col_idx/values.
 */
lb_status_t lb_probe_stream_gather(lb_csr_t A, const float* d_x, int32_t reps, void* stream, float* ms_out);

/*
 * lb_probe_stream -- diagnostics: time (CUDA events, synchronises `stream`) a kernel that only
 * streams A's col_idx and values (the tile processor's 256-bit evict-first loads, no x gathers,
 * no rows), `reps` times; ms_out = mean milliseconds per pass.  8 * nnz / ms_out is this GPU's
 * read-only stream rate for the matrix's own arrays -- the in-repo stream microbenchmark that
 * SURVEY 8(d) asks the tile kernel to be reported against.  Needs 32-byte aligned arrays
 * (LB_ERR_UNSUPPORTED otherwise); LB_ERR_INVALID_ARG for a null handle / ms_out or reps < 1.
 */
lb_status_t lb_probe_stream(lb_csr_t A, int32_t reps, void* stream, float* ms_out);

/*
 * lb_shard_bounds -- host-only: row-shard bounds for `nranks` GPUs with equal nonzeros
 * (reading R9; the paper defers multi-GPU to future work):
 *   b_0 = 0, b_G = rows, b_g = min{ r : off[r] >= ceil(g * nnz / G) }   (0 < g < G).
 *  h_row_offsets  int32[rows+1] host;  h_bounds  int64[nranks+1] host (output).
 */
lb_status_t lb_shard_bounds(const int32_t* h_row_offsets, int64_t rows, int32_t nranks, int64_t* h_bounds);

/*
 * Multi-GPU (one process per GPU).  NCCL is loaded at run time (dlopen of libnccl.so.2, the
 * copy already mapped by PyTorch if any); LB_ERR_UNSUPPORTED if it cannot be loaded.
 *  lb_comm_unique_id  rank 0 creates the 128-byte NCCL unique id (ship it to the other ranks
 *                     with any host transport, e.g. torch.distributed.broadcast_object_list).
 *  lb_comm_init       every rank: join communicator `id` as `rank` of `nranks` on CUDA `device`.
 */
lb_status_t lb_comm_unique_id(uint8_t id_out[128]);
lb_status_t lb_comm_init(const uint8_t id[128], int32_t rank, int32_t nranks, int32_t device, lb_comm_t* out);
lb_status_t lb_comm_destroy(lb_comm_t c);

/*
 * lb_spmv_multi -- one iteration of row-sharded SpMV: this rank computes
 *   y_full[b_r .. b_{r+1}) = A_local x_full
 * with `sched`, then all-gathers the shards so every rank holds the whole y_full
 * (NCCL over NVLink, on `stream`, after the compute).
 *  A_local   handle of this rank's row shard (rows b_{r+1}-b_r, GLOBAL column ids, offsets
 *            rebased to start at 0).
 *  h_bounds  int64[nranks+1] host, identical on every rank (from lb_shard_bounds).
 *  d_x_full  fp32[cols] (replicated); d_y_full fp32[b_G] (must not alias d_x_full).
 */
lb_status_t lb_spmv_multi(lb_csr_t A_local, lb_comm_t c, lb_schedule_t sched, const int64_t* h_bounds,
                          const float* d_x_full, float* d_y_full, void* stream);

/* lb_spmv_multi_ex -- lb_spmv_multi with lb_spmv_ex flags (LB_SPMV_REPARTITION: the rank's merge-path
 * partition is recomputed inside the call; bench.py's multi-GPU step), LB_SPMV_CHUNKED (see the flag)
 * or LB_SPMV_PADDED (the padded all-gather layout of lb_allgather_padded: d_x_full and d_y_full are
 * fp32[nranks * P], P = lb_padded_rows, rank r's rows at slot r * P, and A_local's column ids were
 * remapped with lb_remap_cols_padded; exclusive with LB_SPMV_CHUNKED).  Flags must be equal on all
 * ranks (the collectives they select must match). */
lb_status_t lb_spmv_multi_ex(lb_csr_t A_local, lb_comm_t c, lb_schedule_t sched, const int64_t* h_bounds,
                             const float* d_x_full, float* d_y_full, uint32_t flags, void* stream);

/*
 * Fused multi-GPU step (NEXT-1): the all-gather of y is folded into the tile kernel's epilogue.
 * lb_peer_create registers this rank's y buffer (d_y_full, fp32[rows_global], device; any pointer
 * inside a cudaMalloc allocation, e.g. a torch tensor) with every rank of `c`: CUDA IPC handles and
 * offsets are exchanged with NCCL and the other ranks' buffers are mapped into this process
 * (synchronises `stream`; collective: every rank calls it).  Up to 8 ranks (one NVSwitch node).
 * lb_spmv_multi_fused then computes this rank's rows of y = A x with the merge-path tile kernel
 * writing every final y value to its own buffer AND to every peer's buffer over NVLink (rows whose
 * value the fix-up completes are sent by the fix-up), followed by a cross-rank barrier (an NCCL
 * group of 4-byte broadcasts), so that in stream order every rank's buffer holds the whole y.  An
 * entry barrier of the same kind precedes the kernel, so no rank stores into a peer's buffer before
 * that peer's stream has finished the work queued before the call (write-after-read: e.g. copying
 * the previous y into its x); reads of the buffer on OTHER streams must be ordered by the caller.  If
 * no fused kernel applies (schedule other than MERGE_PATH, L other than 504/1016, unaligned
 * arrays) it computes locally and exchanges with lb_allgather_rows.  x must not alias the buffer.
 * flags: LB_SPMV_REPARTITION.  lb_peer_destroy unmaps the peers (after all work completed).
 */
typedef struct lb_peer_s* lb_peer_t;
lb_status_t lb_peer_create(lb_comm_t c, float* d_y_full, int64_t rows_global, void* stream, lb_peer_t* out);
lb_status_t lb_peer_destroy(lb_peer_t p);
lb_status_t lb_spmv_multi_fused(lb_csr_t A_local, lb_peer_t p, lb_schedule_t sched, const int64_t* h_bounds,
                                const float* d_x_full, uint32_t flags, void* stream);

/* lb_spmv_peers -- diagnostics for the fused epilogue on one GPU: y = A x (MERGE_PATH) where the tile
 * kernel also stores every final y value into each of the npeers (<= 7) device buffers h_peer_y[p]
 * (fp32[rows] each, host array of device pointers) exactly as lb_spmv_multi_fused stores into the
 * other ranks' buffers.  LB_ERR_UNSUPPORTED if no fused kernel applies to this handle. */
lb_status_t lb_spmv_peers(lb_csr_t A, const float* d_x, float* d_y, float* const* h_peer_y, int32_t npeers,
                          uint32_t flags, void* stream);

/* lb_allgather_rows -- the exchange step of lb_spmv_multi alone: rank r contributes
 * d_y_full[b_r .. b_{r+1}) and receives every other rank's slice in place (SURVEY 8(e) option 1: one
 * NCCL group of broadcasts with root k sending rank k's slice, scheduled by lb_exchange_schedule;
 * at world size 1 the group holds one in-place broadcast). */
lb_status_t lb_allgather_rows(lb_comm_t c, const int64_t* h_bounds, float* d_y_full, void* stream);

/*
 * lb_exchange_schedule -- host-only: the broadcasts of the y exchange, as every exchange path of this
 * library issues them.  For chunk c (0 <= c < nchunks) and root rank k, rank k broadcasts
 * y_full[h_offsets[c*nranks + k], + h_counts[c*nranks + k]) to every rank (count 0: no call).
 *  h_bounds    int64[nranks+1] shard bounds (b_0 = 0, non-decreasing; from lb_shard_bounds).
 *  h_cut_rows  int64[nranks][nchunks+1]: rank k's chunk c is its LOCAL rows [cut[k][c], cut[k][c+1])
 *              (cut[k][0] = 0, cut[k][nchunks] = b_{k+1} - b_k, non-decreasing), e.g. the table
 *              lb_spmv_multi_ex(LB_SPMV_CHUNKED) exchanges (lb_csr_chunk_rows of every rank);
 *              NULL: one chunk holding every rank's whole slice (lb_allgather_rows).
 * Over all (c, k) the ranges tile [0, b_G) exactly once.  LB_ERR_INVALID_ARG on bounds or cuts that
 * are not monotone or do not span the shard.
 */
lb_status_t lb_exchange_schedule(int32_t nranks, const int64_t* h_bounds, int32_t nchunks, const int64_t* h_cut_rows,
                                 int64_t* h_offsets, int64_t* h_counts);

/* lb_csr_chunk_rows -- the handle's LB_SPMV_CHUNKED cut rows padded to nchunks + 1 entries (nchunks
 * must be 8): what this rank contributes to the chunked exchange's cut table.  Computes the cuts on
 * first use (synchronises `stream`); without a usable x-reuse plan: {0, rows, rows, ...}. */
lb_status_t lb_csr_chunk_rows(lb_csr_t A, int32_t nchunks, int64_t* h_rows_out, void* stream);

/*
 * Padded all-gather layout (SURVEY 8(e) option 2).  P = lb_padded_rows(nranks, h_bounds) = the largest
 * shard; y lives in fp32[nranks * P] with rank k's rows at [k*P, k*P + b_{k+1} - b_k).
 *  lb_remap_cols_padded  global column c (in shard k: b_k <= c < b_{k+1}) -> k*P + (c - b_k), for a
 *                        shard's col_idx (device, nnz entries; in and out may alias).  Synchronises.
 *  lb_allgather_padded   one in-place ncclAllGather of the P-sized slots (every rank's slot r*P).
 */
int64_t lb_padded_rows(int32_t nranks, const int64_t* h_bounds);
lb_status_t lb_remap_cols_padded(int32_t nranks, const int64_t* h_bounds, const int32_t* d_col_in, int64_t nnz,
                                 int32_t* d_col_out, void* stream);
lb_status_t lb_allgather_padded(lb_comm_t c, int64_t padded_rows, float* d_y_pad, void* stream);

/*
 * Replica check (after the exchange every rank's y must match bitwise).
 *  lb_y_checksum           h = sum_i mix64(i * 0x9E3779B97F4A7C15 + bits(y_i)) mod 2^64, mix64 = the
 *                          splitmix64 finaliser, bits = the fp32 bit pattern (so -0 != +0).  Order-free
 *                          and deterministic.  Synchronises `stream`.
 *  lb_comm_check_replicas  the same hash on every rank, NCCL all-reduces of its min and max:
 *                          *h_equal = 1 iff every rank's d_y[0, n) hashes equal.  Collective;
 *                          synchronises `stream`.
 */
lb_status_t lb_y_checksum(const float* d_y, int64_t n, void* stream, uint64_t* h_out);
lb_status_t lb_comm_check_replicas(lb_comm_t c, const float* d_y, int64_t n, void* stream, int32_t* h_equal,
                                   uint64_t* h_hash);

/* Name of the main kernel lb_spmv(A, sched) launches with the handle's current settings
 * (diagnostics / bench reporting); "" for an unknown schedule. */
const char* lb_kernel_name(lb_csr_t A, lb_schedule_t sched);

/* Last error message of the calling thread ("" if none). */
const char* lb_last_error(void);

/* Number of CUDA kernels this library has launched in this process (for bench accounting). */
uint64_t lb_launch_count(void);

/* Library version string. */
const char* lb_version(void);

#ifdef __cplusplus
}
#endif

#endif /* LB_H */
