/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the Sinkhorn-WMD hot path.
 *
 * A plain-C restatement of the reference's numba kernels
 * (/root/reference/pkg/src/sinkwmd/_jit.py) and of its solver loop
 * (sinkwmd/solver.py:106-201).  It exists to CHECK the CUDA path (tests/,
 * __graft_entry__.smoke()) and to time the reference algorithm on the host
 * cores (bench.py cpu_baseline leg and `--impl reference`).  Nothing in the
 * product package links or calls it.
 *
 * Numerics follow the reference bit for bit: float64 throughout, sequential
 * accumulation in the reference's loop order, no FMA contraction (build with
 * -ffp-contract=off, matching numba's fastmath=False, _jit.py:8-9), glibc
 * exp()/sqrt().  The pinning tests (tests/test_oracle_golden.py) compare it
 * with outputs of the reference package itself (tests/golden/).
 *
 * Parallelism mirrors the reference's deterministic "columns" mode
 * (_jit.py:164-183, sparse.py:261-276): contiguous column blocks balanced
 * by nonzero count, one OpenMP thread per block, so results are independent
 * of the thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_OK 0
#define ORACLE_ZERO_DENOM 1   /* errpos = (i, j): "zero denominator at nonzero (i, j)" */
#define ORACLE_NONPOS_X 2     /* errpos = (flat index, -1); value in *errval */

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_threads(int p) {
#ifdef _OPENMP
    if (p > 0) omp_set_num_threads(p);
#else
    (void)p;
#endif
}

/* _jit.py:90-102 euclid_rows: cost[i,a] = sqrt(sum_k (vecs[sel[a],k]-vecs[i,k])^2). */
void oracle_euclid_rows(const double* vecs, int64_t n_rows, int64_t dim,
                        const int64_t* sel, int64_t n_sel, double* cost) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n_rows; ++i) {
        const double* vi = vecs + i * dim;
        for (int64_t a = 0; a < n_sel; ++a) {
            const double* vb = vecs + sel[a] * dim;
            double s = 0.0;
            for (int64_t k = 0; k < dim; ++k) {
                double d = vb[k] - vi[k];
                s += d * d;
            }
            cost[i * n_sel + a] = sqrt(s);
        }
    }
}

/* _jit.py:105-114 precompute_mats: kernel=exp(-lam*cost), kor=kernel/w, kcost=kernel*cost. */
void oracle_precompute(const double* cost, int64_t n_rows, int64_t n_sel,
                       const double* weights, double lam, double* kernel,
                       double* kor, double* kcost) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n_rows; ++i) {
        for (int64_t a = 0; a < n_sel; ++a) {
            double c = cost[i * n_sel + a];
            double k = exp(-lam * c);
            kernel[i * n_sel + a] = k;
            if (kor) kor[i * n_sel + a] = k / weights[a];
            if (kcost) kcost[i * n_sel + a] = k * c;
        }
    }
}

static inline void note_err(int64_t* errpos, int64_t i, int64_t j) {
    if (errpos[0] < 0) { errpos[0] = i; errpos[1] = j; }
}

/* _jit.py:120-137 fused_iter_serial (CSR order). x must be zeroed by caller. */
void oracle_fused_iter_serial(const int64_t* row_ptr, const int64_t* col_idx,
                              const double* vals, int64_t n_rows,
                              const double* kernel, const double* kor, int64_t vr,
                              const double* u, double* x, int64_t* errpos) {
    for (int64_t i = 0; i < n_rows; ++i) {
        const double* ki = kernel + i * vr;
        const double* ri = kor + i * vr;
        for (int64_t z = row_ptr[i]; z < row_ptr[i + 1]; ++z) {
            int64_t j = col_idx[z];
            const double* uj = u + j * vr;
            double s = 0.0;
            for (int64_t a = 0; a < vr; ++a) s += ki[a] * uj[a];
            if (s == 0.0) { note_err(errpos, i, j); continue; }
            double t = vals[z] / s;
            double* xj = x + j * vr;
            for (int64_t a = 0; a < vr; ++a) xj[a] += ri[a] * t;
        }
    }
}

/* Smallest (i, j) in row-major order among a column walk's zero denominators;
 * the serial CSR walk reports exactly this pair first. */
static inline void note_err_min(int64_t* best_i, int64_t* best_j, int64_t i, int64_t j) {
    if (*best_i < 0 || i < *best_i || (i == *best_i && j < *best_j)) { *best_i = i; *best_j = j; }
}

static void merge_err(int64_t* errpos, int64_t bi, int64_t bj) {
    if (bi < 0) return;
#pragma omp critical(oracle_err)
    {
        if (errpos[0] < 0 || bi < errpos[0] || (bi == errpos[0] && bj < errpos[1])) {
            errpos[0] = bi; errpos[1] = bj;
        }
    }
}

/* _jit.py:164-183 fused_iter_columns. Column blocks from col_bounds (nblocks+1).
 * The error position reported is the serial walk's (deterministic), a
 * refinement of the reference's first-found race. */
void oracle_fused_iter_columns(const int64_t* col_ptr, const int32_t* rows,
                               const double* vals, const int64_t* col_bounds,
                               int64_t nblocks, const double* kernel,
                               const double* kor, int64_t vr, const double* u,
                               double* x, int64_t* errpos) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t w = 0; w < nblocks; ++w) {
        int64_t bi = -1, bj = -1;
        for (int64_t j = col_bounds[w]; j < col_bounds[w + 1]; ++j) {
            const double* uj = u + j * vr;
            double* xj = x + j * vr;
            for (int64_t q = col_ptr[j]; q < col_ptr[j + 1]; ++q) {
                int64_t i = rows[q];
                const double* ki = kernel + i * vr;
                double s = 0.0;
                for (int64_t a = 0; a < vr; ++a) s += ki[a] * uj[a];
                if (s == 0.0) { note_err_min(&bi, &bj, i, j); continue; }
                double t = vals[q] / s;
                const double* ri = kor + i * vr;
                for (int64_t a = 0; a < vr; ++a) xj[a] += ri[a] * t;
            }
        }
        merge_err(errpos, bi, bj);
    }
}

/* _jit.py:243-262 fused_final_serial. wmd must be zeroed by caller. */
void oracle_fused_final_serial(const int64_t* row_ptr, const int64_t* col_idx,
                               const double* vals, int64_t n_rows,
                               const double* kernel, const double* kcost, int64_t vr,
                               const double* u, double* wmd, int64_t* errpos) {
    for (int64_t i = 0; i < n_rows; ++i) {
        const double* ki = kernel + i * vr;
        const double* mi = kcost + i * vr;
        for (int64_t z = row_ptr[i]; z < row_ptr[i + 1]; ++z) {
            int64_t j = col_idx[z];
            const double* uj = u + j * vr;
            double s = 0.0;
            for (int64_t a = 0; a < vr; ++a) s += ki[a] * uj[a];
            if (s == 0.0) { note_err(errpos, i, j); continue; }
            double v = vals[z] / s;
            double d = 0.0;
            for (int64_t a = 0; a < vr; ++a) d += mi[a] * uj[a];
            wmd[j] += v * d;
        }
    }
}

/* _jit.py:291-312 fused_final_columns. wmd must be zeroed by caller. */
void oracle_fused_final_columns(const int64_t* col_ptr, const int32_t* rows,
                                const double* vals, const int64_t* col_bounds,
                                int64_t nblocks, const double* kernel,
                                const double* kcost, int64_t vr, const double* u,
                                double* wmd, int64_t* errpos) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t w = 0; w < nblocks; ++w) {
        int64_t bi = -1, bj = -1;
        for (int64_t j = col_bounds[w]; j < col_bounds[w + 1]; ++j) {
            const double* uj = u + j * vr;
            double acc = wmd[j];
            for (int64_t q = col_ptr[j]; q < col_ptr[j + 1]; ++q) {
                int64_t i = rows[q];
                const double* ki = kernel + i * vr;
                double s = 0.0;
                for (int64_t a = 0; a < vr; ++a) s += ki[a] * uj[a];
                if (s == 0.0) { note_err_min(&bi, &bj, i, j); continue; }
                double v = vals[q] / s;
                const double* mi = kcost + i * vr;
                double d = 0.0;
                for (int64_t a = 0; a < vr; ++a) d += mi[a] * uj[a];
                acc += v * d;
            }
            wmd[j] = acc;
        }
        merge_err(errpos, bi, bj);
    }
}

/* _jit.py:319-336 sddmm_serial: w_out[z] = vals[z] / (kernel[i,:] . u[j,:]) in CSR order. */
void oracle_sddmm_serial(const int64_t* row_ptr, const int64_t* col_idx,
                         const double* vals, int64_t n_rows, const double* kernel,
                         int64_t vr, const double* u, double* w_out, int64_t* errpos) {
    for (int64_t i = 0; i < n_rows; ++i) {
        const double* ki = kernel + i * vr;
        for (int64_t z = row_ptr[i]; z < row_ptr[i + 1]; ++z) {
            const double* uj = u + col_idx[z] * vr;
            double s = 0.0;
            for (int64_t a = 0; a < vr; ++a) s += ki[a] * uj[a];
            if (s == 0.0) { note_err(errpos, i, col_idx[z]); w_out[z] = 0.0; continue; }
            w_out[z] = vals[z] / s;
        }
    }
}

/* _jit.py:361-370 spmm_serial: x[j,:] += kor[i,:] * w[z] in CSR order. */
void oracle_spmm_serial(const int64_t* row_ptr, const int64_t* col_idx,
                        const double* w_vals, int64_t n_rows, const double* kor,
                        int64_t vr, double* x) {
    for (int64_t i = 0; i < n_rows; ++i) {
        const double* ri = kor + i * vr;
        for (int64_t z = row_ptr[i]; z < row_ptr[i + 1]; ++z) {
            double t = w_vals[z];
            double* xj = x + col_idx[z] * vr;
            for (int64_t a = 0; a < vr; ++a) xj[a] += ri[a] * t;
        }
    }
}

/* sparse.py:261-276 column_blocks: p+1 nnz-balanced column boundaries. */
void oracle_column_blocks(const int64_t* col_ptr, int64_t n_cols, int64_t p,
                          int64_t* bounds) {
    int64_t nnz = col_ptr[n_cols];
    bounds[0] = 0;
    for (int64_t k = 1; k < p; ++k) {
        /* np.searchsorted(col_ptr, k*nnz//p, side="left") */
        int64_t target = (k * nnz) / p;
        int64_t lo = 0, hi = n_cols + 1;
        while (lo < hi) {
            int64_t mid = lo + (hi - lo) / 2;
            if (col_ptr[mid] < target) lo = mid + 1; else hi = mid;
        }
        bounds[k] = lo;
    }
    bounds[p] = n_cols;
    for (int64_t k = 1; k <= p; ++k)       /* np.maximum.accumulate */
        if (bounds[k] < bounds[k - 1]) bounds[k] = bounds[k - 1];
}

/* solver.py:95-103 update_u: u = 1/x after checking min(x) > 0.  Returns
 * ORACLE_NONPOS_X with the first argmin flat index and its value. */
static int update_u(const double* x, double* u, int64_t n, int64_t* flat, double* val) {
    /* np.min propagates NaN (and NaN <= 0 is false), so a NaN anywhere
     * suppresses the check exactly as in the reference. */
    double mn = INFINITY; int64_t at = -1; int has_nan = 0;
    for (int64_t k = 0; k < n; ++k) {
        if (x[k] != x[k]) has_nan = 1;
        else if (x[k] < mn) { mn = x[k]; at = k; }
    }
    if (n > 0 && !has_nan && mn <= 0.0) { *flat = at; *val = mn; return ORACLE_NONPOS_X; }
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < n; ++k) u[k] = 1.0 / x[k];
    return ORACLE_OK;
}

/*
 * solver.py:106-201 sinkhorn_wmd with SolverConfig(deterministic=True,
 * workers=nblocks) and tol=None: distances -> precompute -> init ->
 * max_iter fused iterations -> final.  Scratch: cost,kernel,kor,kcost
 * (V*vr each), x,x_prev,u (N*vr each).  timings[0..4] receive seconds for
 * distances, precompute, iterations, final, total (omp_get_wtime).
 * Returns ORACLE_OK or an error kind with errpos / errval filled.
 */
/* max |a - b| over n entries with numpy's NaN propagation (np.max returns
 * NaN when any entry is NaN; solver.py:180) */
static double max_abs_diff(const double* a, const double* b, int64_t n) {
    double m = 0.0;
    int nan = 0;
    for (int64_t k = 0; k < n; ++k) {
        const double d = fabs(a[k] - b[k]);
        if (d != d) nan = 1;
        else if (d > m) m = d;
    }
    return nan ? NAN : m;
}

/*
 * oracle_solve with SolverConfig.tol (solver.py:170-183): tol < 0 means None.
 * After iteration t, delta = max|x - x_prev| is written to deltas[t] and the
 * loop stops when delta < tol; *iterations / *converged receive the
 * reference's iterations_run / converged.
 */
int oracle_solve_tol(const double* vecs, int64_t n_rows, int64_t dim,
                     const int64_t* sel, const double* weights, int64_t vr,
                     const int64_t* col_ptr, const int32_t* rows, const double* vals,
                     int64_t n_cols, double lam, int64_t max_iter, double tol, int64_t nblocks,
                     double* cost, double* kernel, double* kor, double* kcost,
                     double* x, double* x_prev, double* u, double* wmd,
                     int64_t* errpos, double* errval, double* timings,
                     int64_t* iterations, int32_t* converged, double* deltas);

int oracle_solve(const double* vecs, int64_t n_rows, int64_t dim,
                 const int64_t* sel, const double* weights, int64_t vr,
                 const int64_t* col_ptr, const int32_t* rows, const double* vals,
                 int64_t n_cols, double lam, int64_t max_iter, int64_t nblocks,
                 double* cost, double* kernel, double* kor, double* kcost,
                 double* x, double* x_prev, double* u, double* wmd,
                 int64_t* errpos, double* errval, double* timings) {
    int64_t it = 0;
    int32_t conv = 0;
    return oracle_solve_tol(vecs, n_rows, dim, sel, weights, vr, col_ptr, rows, vals, n_cols,
                            lam, max_iter, -1.0, nblocks, cost, kernel, kor, kcost, x, x_prev,
                            u, wmd, errpos, errval, timings, &it, &conv, NULL);
}

int oracle_solve_tol(const double* vecs, int64_t n_rows, int64_t dim,
                     const int64_t* sel, const double* weights, int64_t vr,
                     const int64_t* col_ptr, const int32_t* rows, const double* vals,
                     int64_t n_cols, double lam, int64_t max_iter, double tol, int64_t nblocks,
                     double* cost, double* kernel, double* kor, double* kcost,
                     double* x, double* x_prev, double* u, double* wmd,
                     int64_t* errpos, double* errval, double* timings,
                     int64_t* iterations, int32_t* converged, double* deltas) {
    double t_start = 0, t0 = 0;
#ifdef _OPENMP
    t_start = omp_get_wtime();
#endif
    int64_t* bounds = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nblocks + 1));
    oracle_column_blocks(col_ptr, n_cols, nblocks, bounds);
    errpos[0] = errpos[1] = -1;
#ifdef _OPENMP
    t0 = omp_get_wtime();
#endif
    oracle_euclid_rows(vecs, n_rows, dim, sel, vr, cost);
#ifdef _OPENMP
    timings[0] = omp_get_wtime() - t0; t0 = omp_get_wtime();
#endif
    oracle_precompute(cost, n_rows, vr, weights, lam, kernel, kor, kcost);
#ifdef _OPENMP
    timings[1] = omp_get_wtime() - t0; t0 = omp_get_wtime();
#endif
    int64_t n = n_cols * vr;
    for (int64_t k = 0; k < n; ++k) x[k] = 1.0 / (double)vr;
    int rc = ORACLE_OK;
    *iterations = 0;
    *converged = 0;
    for (int64_t it = 0; it < max_iter; ++it) {
        rc = update_u(x, u, n, &errpos[0], errval);
        if (rc) { errpos[1] = -1; goto done; }
        double* tmp = x; x = x_prev; x_prev = tmp;
        memset(x, 0, sizeof(double) * (size_t)n);
        oracle_fused_iter_columns(col_ptr, rows, vals, bounds, nblocks, kernel, kor,
                                  vr, u, x, errpos);
        if (errpos[0] >= 0) { rc = ORACLE_ZERO_DENOM; goto done; }
        *iterations = it + 1;
        if (tol >= 0.0) {
            const double delta = max_abs_diff(x, x_prev, n);
            if (deltas) deltas[it] = delta;
            if (delta < tol) { *converged = 1; break; }
        }
    }
#ifdef _OPENMP
    timings[2] = omp_get_wtime() - t0; t0 = omp_get_wtime();
#endif
    rc = update_u(x, u, n, &errpos[0], errval);
    if (rc) { errpos[1] = -1; goto done; }
    memset(wmd, 0, sizeof(double) * (size_t)n_cols);
    oracle_fused_final_columns(col_ptr, rows, vals, bounds, nblocks, kernel, kcost,
                               vr, u, wmd, errpos);
    if (errpos[0] >= 0) { rc = ORACLE_ZERO_DENOM; goto done; }
#ifdef _OPENMP
    timings[3] = omp_get_wtime() - t0;
    timings[4] = omp_get_wtime() - t_start;
#endif
done:
    free(bounds);
    return rc;
}
