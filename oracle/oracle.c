/*
 * oracle.c -- plain, slow, obviously-correct CPU reference for the hot path of
 * arXiv 2212.08964 (CSR SpMV y = A x under a load-balancing schedule).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or helper with paper_2212_08964_b200/ (the CUDA product path), and
 * the product never calls it.
 *
 * Citations: "P:L" = /root/reference/PAPER.md line L (section / algorithm in brackets).
 *
 * Precision: every fp32 input is widened to double; a product of two fp32 values is
 * exact in double (24+24 <= 53 significand bits), sums are taken in row order in double.
 *
 * Parity status: every function here is pinned by tests/test_oracle_pins.py
 * (dense brute force, closed forms, invariants, independent derivations); nothing is
 * "parity unpinned".
 */
#include <stdint.h>
#include <stddef.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/*
 * SpMV by definition: y = A x for A in CSR (P:123 [Ch.3 intro]: "SpMV computes the output
 * vector y = Ax"; P:149 [Sec. CSR]; Listing 3: for each row, sum += values[nz] *
 * x[indices[nz]] over the row's nonzeros, then y[row] = sum).
 * Also returns s[i] = sum_k |a_ik x_k| (the tolerance scale of BASELINE.json north_star).
 * Empty rows give y = +0 (P:982 assigns the zero-initialised sum).
 */
void oracle_spmv(int64_t rows, const int32_t *row_offsets, const int32_t *col_idx,
                 const float *values, const float *x, double *y, double *s)
{
    for (int64_t i = 0; i < rows; ++i) {
        double acc = 0.0, mag = 0.0;
        for (int64_t k = row_offsets[i]; k < row_offsets[i + 1]; ++k) {
            double p = (double)values[k] * (double)x[col_idx[k]];
            acc += p;
            mag += fabs(p);
        }
        y[i] = acc;
        if (s) s[i] = mag;
    }
}

/* The same definition, rows split across OpenMP threads (used only to time the CPU
 * baseline on the host's cores; the arithmetic per row is identical). */
void oracle_spmv_omp(int64_t rows, const int32_t *row_offsets, const int32_t *col_idx,
                     const float *values, const float *x, double *y, double *s)
{
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t i = 0; i < rows; ++i) {
        double acc = 0.0, mag = 0.0;
        for (int64_t k = row_offsets[i]; k < row_offsets[i + 1]; ++k) {
            double p = (double)values[k] * (double)x[col_idx[k]];
            acc += p;
            mag += fabs(p);
        }
        y[i] = acc;
        if (s) s[i] = mag;
    }
}

int oracle_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/*
 * SpMV on a set of selected rows whose nonzeros were gathered into a packed CSR
 * (sel_offsets[n_sel+1] indexes sel_cols / sel_vals).  Used for sampled parity at
 * full size, where the whole matrix is too big to evaluate on the host in the test.
 */
void oracle_spmv_packed(int64_t n_sel, const int64_t *sel_offsets, const int32_t *sel_cols,
                        const float *sel_vals, const float *x, double *y, double *s)
{
    for (int64_t r = 0; r < n_sel; ++r) {
        double acc = 0.0, mag = 0.0;
        for (int64_t k = sel_offsets[r]; k < sel_offsets[r + 1]; ++k) {
            double p = (double)sel_vals[k] * (double)x[sel_cols[k]];
            acc += p;
            mag += fabs(p);
        }
        y[r] = acc;
        if (s) s[r] = mag;
    }
}

/*
 * SpMM by definition: Y = A X for A in CSR and X dense, row-major with leading dimension ldx
 * (Listing 4 P:1046-1074 [Sec. Application Space]: "a simple loop wrapped around SpMV": for each
 * row and each column j of X, sum += values[nz] * X(indices[nz], j); C(row, j) = sum).
 * Y[i*ldy + j] = sum_k val[k] * X[col[k]*ldx + j] in row order, in double; S likewise with |.|.
 */
void oracle_spmm(int64_t rows, const int32_t *row_offsets, const int32_t *col_idx, const float *values,
                 int64_t n, const float *X, int64_t ldx, double *Y, int64_t ldy, double *S)
{
    for (int64_t i = 0; i < rows; ++i) {
        for (int64_t j = 0; j < n; ++j) {
            double acc = 0.0, mag = 0.0;
            for (int64_t k = row_offsets[i]; k < row_offsets[i + 1]; ++k) {
                double p = (double)values[k] * (double)X[(int64_t)col_idx[k] * ldx + j];
                acc += p;
                mag += fabs(p);
            }
            Y[i * ldy + j] = acc;
            if (S) S[i * ldy + j] = mag;
        }
    }
}

/*
 * Merge-path partition by brute force: walk the merge of list A = the row ends
 * (row i ends after its off[i+1] nonzeros) and list B = the nonzero indices 0..nnz-1,
 * one merge item per step, exactly as the merge-path schedule defines the work
 * (P:292 [Sec. Work-Oriented]: "a work item as either a nonzero element or an output";
 * "2-D split of the grid created using the row-offsets and the nonzero indices";
 * P:1021 [Sec. Merge-path load balancing]: nnzs + rows work divided evenly).
 * The coordinate (i, j) = (#row ends consumed, #nonzeros consumed) is recorded whenever the
 * step count equals d_t = min(t * L, rows + nnz), t = 0..T, T = ceil((rows+nnz)/L)
 * (Alg.3, with the ceil reading of items_per_thread -- DESIGN.md reading R2).
 * Tie-break (R1): when off[i+1] == j the row end is taken first, because
 * CSR rows are half-open and nonzero j belongs to a later row.
 * coords receives (T+1) pairs (row, nz), row-major.  Returns T, or -1 on bad input.
 */
int64_t oracle_partition(int64_t rows, int64_t nnz, const int32_t *row_offsets, int64_t L,
                         int32_t *coords)
{
    if (L <= 0 || rows < 0 || nnz < 0) return -1;
    int64_t total = rows + nnz;
    int64_t T = (total + L - 1) / L;
    int64_t i = 0, j = 0, t = 0, step = 0;
    for (;;) {
        int64_t d_t = t * L < total ? t * L : total;
        while (t <= T && step == d_t) {
            coords[2 * t] = (int32_t)i;
            coords[2 * t + 1] = (int32_t)j;
            ++t;
            d_t = t * L < total ? t * L : total;
        }
        if (t > T || step == total) break;
        /* one merge item */
        if (i < rows && (j == nnz || row_offsets[i + 1] <= j)) ++i;  /* row end i */
        else ++j;                                                      /* nonzero j */
        ++step;
    }
    return T;
}

/*
 * Nonzero-splitting partition (P:291 [Sec. Work-Oriented]: "non-zero splitting ... considers the
 * total number of nonzero elements ... as the total work"; table): tiles of L nonzeros,
 * T = max(1, ceil(nnz/L)), j_t = min(t*L, nnz); the tile starts after every row whose end lies at
 * or before nonzero j_t: i_t = #{ r : off[r+1] <= j_t } (reading R1: a row end precedes the nonzero
 * at the same position), with i_0 = 0 and i_T = rows so that every row is covered.  By brute force
 * (linear count).  coords receives (T+1) (row, nz) pairs; returns T.
 */
int64_t oracle_partition_nz(int64_t rows, int64_t nnz, const int32_t *row_offsets, int64_t L, int32_t *coords)
{
    if (L <= 0 || rows < 0 || nnz < 0) return -1;
    int64_t T = (nnz + L - 1) / L;
    if (T < 1) T = 1;
    for (int64_t t = 0; t <= T; ++t) {
        int64_t j = t * L < nnz ? t * L : nnz;
        int64_t i = 0;
        if (t == 0) i = 0;
        else if (t == T) i = rows;
        else
            for (int64_t r = 0; r < rows; ++r)
                if (row_offsets[r + 1] <= j) ++i;
        coords[2 * t] = (int32_t)i;
        coords[2 * t + 1] = (int32_t)j;
    }
    return T;
}

/*
 * Row-shard bounds for G ranks by equal nnz (reading R9; the paper has no
 * multi-GPU design, P:784 / P:2187-2192): b_0 = 0, b_G = rows, and for 0 < g < G,
 * b_g = min{ r : off[r] >= ceil(g * nnz / G) }, found by a linear scan.
 */
void oracle_shard_bounds(int64_t rows, const int32_t *row_offsets, int32_t G, int64_t *bounds)
{
    int64_t nnz = rows > 0 ? row_offsets[rows] : 0;
    bounds[0] = 0;
    int64_t r = 0;
    for (int32_t g = 1; g < G; ++g) {
        int64_t target = (g * nnz + G - 1) / G;
        while (r < rows && row_offsets[r] < target) ++r;
        bounds[g] = r;
    }
    bounds[G] = rows;
}

/*
 * Three-bin classification of the binning schedule (Alg.4 P:364-377 [Sec. Binning and
 * Reordering]): num_nonzeros = offsets[row+1] - offsets[row]; >= block_size -> CTA bin, else
 * >= warp_size -> warp bin, else thread bin.  Each bin lists its rows in ascending order (reading
 * R21: Alg.4 appends with bin_size++ in an unspecified order).  Output layout of ids:
 * [CTA bin | warp bin | thread bin]; sizes[0..2] = bin sizes.  One pass per bin over the rows.
 */
void oracle_bins(int64_t rows, const int32_t *row_offsets, int64_t block_size, int64_t warp_size,
                 int32_t *ids, int64_t *sizes)
{
    int64_t n = 0;
    for (int bin = 0; bin < 3; ++bin) {
        int64_t start = n;
        for (int64_t r = 0; r < rows; ++r) {
            int64_t num_nonzeros = (int64_t)row_offsets[r + 1] - row_offsets[r];
            int b = num_nonzeros >= block_size ? 0 : (num_nonzeros >= warp_size ? 1 : 2);
            if (b == bin) ids[n++] = (int32_t)r;
        }
        sizes[bin] = n - start;
    }
}

/*
 * x-reuse plan by definition (B200 extension of the merge-path tile processor -- DESIGN.md section 6b
 * and include/lb.h lb_csr_plan_hot_x; the paper has no such step: it only fixes that the tile
 * processor gathers x[col] per nonzero, Listing 3).
 *   deg(c)  = number of entries k with col_idx[k] == c;  candidates = columns with deg >= 2;
 *   HOT: if fewer than `slots` candidates, all of them, slots in ascending column order; else the
 *   first `slots` candidates in the order (deg descending, column ascending); with tau1 = the
 *   smallest degree among them, slots go first to hot columns with deg > tau1 (ascending column),
 *   then to hot columns with deg == tau1 (ascending column).
 *   WARM (hot tier full and warm > 0): tau2 = the smallest d >= 2 with #{deg >= d} <= slots + warm;
 *   if tau2 <= tau1, the non-hot columns with deg >= tau2 in ascending column order; else none.
 *   remapped[k] = ~slot(c) (hot), cols + warm_index(c) (warm), c otherwise (c = col_idx[k]).
 * Plain counting and selection by repeated maximum search (no sort, no histogram): O(slots*cols +
 * cols*max_deg), for the small matrices the tests use.  Returns the number of hot columns;
 * *n_warm, *hot_nnz, *warm_nnz as named.  deg and tier_of are caller scratch of `cols` entries.
 */
int64_t oracle_x_plan(int64_t cols, int64_t nnz, const int32_t *col_idx, int32_t slots, int64_t warm,
                      int64_t *deg, int32_t *tier_of, int32_t *slot_cols, int32_t *warm_cols,
                      int32_t *remapped, int64_t *n_warm, int64_t *hot_nnz, int64_t *warm_nnz)
{
    for (int64_t c = 0; c < cols; ++c) { deg[c] = 0; tier_of[c] = -1; }
    for (int64_t k = 0; k < nnz; ++k) deg[col_idx[k]] += 1;
    int64_t ncand = 0, maxdeg = 0;
    for (int64_t c = 0; c < cols; ++c) { ncand += deg[c] >= 2; if (deg[c] > maxdeg) maxdeg = deg[c]; }
    int64_t n = 0;
    *hot_nnz = 0; *warm_nnz = 0; *n_warm = 0;
    if (ncand < slots) {
        for (int64_t c = 0; c < cols; ++c)
            if (deg[c] >= 2) { tier_of[c] = (int32_t)n; slot_cols[n++] = (int32_t)c; *hot_nnz += deg[c]; }
    } else {
        /* mark the hot set: `slots` times take the unmarked candidate of largest degree (lowest
         * column on ties); tier_of = -2 marks "chosen" until slots are numbered below */
        int64_t tau1 = 0;
        for (int32_t s = 0; s < slots; ++s) {
            int64_t best = -1;
            for (int64_t c = 0; c < cols; ++c)
                if (deg[c] >= 2 && tier_of[c] == -1 && (best < 0 || deg[c] > deg[best])) best = c;
            tier_of[best] = -2;
            tau1 = deg[best];
        }
        for (int64_t c = 0; c < cols; ++c)
            if (tier_of[c] == -2 && deg[c] > tau1) { tier_of[c] = (int32_t)n; slot_cols[n++] = (int32_t)c; *hot_nnz += deg[c]; }
        for (int64_t c = 0; c < cols; ++c)
            if (tier_of[c] == -2 && deg[c] == tau1) { tier_of[c] = (int32_t)n; slot_cols[n++] = (int32_t)c; *hot_nnz += deg[c]; }
        if (warm > 0) {
            int64_t tau2 = maxdeg + 1;
            for (int64_t d = 2; d <= maxdeg + 1; ++d) {
                int64_t cnt = 0;
                for (int64_t c = 0; c < cols; ++c) cnt += deg[c] >= d;
                if (cnt <= (int64_t)slots + warm) { tau2 = d; break; }
            }
            if (tau2 <= tau1)
                for (int64_t c = 0; c < cols; ++c)
                    if (tier_of[c] == -1 && deg[c] >= tau2) {
                        tier_of[c] = (int32_t)(n + *n_warm);
                        warm_cols[(*n_warm)++] = (int32_t)c;
                        *warm_nnz += deg[c];
                    }
        }
    }
    for (int64_t k = 0; k < nnz; ++k) {
        int32_t c = col_idx[k], t = tier_of[c];
        remapped[k] = t < 0 ? c : (t < n ? ~t : (int32_t)(cols + (t - n)));
    }
    return n;
}

/*
 * Single-source shortest paths by Dijkstra's algorithm (NEXT-4; Listing 5 P:1076-1107 relaxes
 * dist[neighbor] = min(dist[neighbor], dist[source] + weight) with float distances).
 * Graph in CSR: row u lists u's out-edges (col_idx = neighbor, values = weight >= 0).  Distances are
 * fp32 like the paper's `float source_dist`; every tentative distance is the fp32 sum
 * fl(dist[u] + w), the same monotone edge function the GPU relaxation applies, so both reach the
 * same least fixed point exactly.  Unreachable vertices get +inf.  Plain O(n^2) selection of the
 * unsettled vertex with the smallest distance (no heap), for the small graphs the tests use.
 * Returns -1 if a weight is negative, else the number of settled vertices.
 */
int64_t oracle_sssp(int64_t n, const int32_t *row_offsets, const int32_t *col_idx, const float *weights,
                    int64_t source, float *dist, uint8_t *settled)
{
    for (int64_t k = 0; k < row_offsets[n]; ++k)
        if (!(weights[k] >= 0.0f)) return -1;
    for (int64_t v = 0; v < n; ++v) { dist[v] = INFINITY; settled[v] = 0; }
    dist[source] = 0.0f;
    int64_t done = 0;
    for (;;) {
        int64_t u = -1;
        for (int64_t v = 0; v < n; ++v)
            if (!settled[v] && dist[v] < INFINITY && (u < 0 || dist[v] < dist[u])) u = v;
        if (u < 0) break;
        settled[u] = 1;
        ++done;
        for (int64_t k = row_offsets[u]; k < row_offsets[u + 1]; ++k) {
            float nd = dist[u] + weights[k];   /* fp32 add, as on the GPU */
            if (nd < dist[col_idx[k]]) dist[col_idx[k]] = nd;
        }
    }
    return done;
}
