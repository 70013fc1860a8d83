/*
 * swmd.h — C ABI of the B200 (sm_100a) Sinkhorn-WMD hot path (libswmd.so).
 *
 * Every entry point replaces one native kernel of the reference package
 * (/root/reference/pkg/src/sinkwmd/_jit.py, called from kernels.py / solver.py)
 * and keeps its calling convention: plain pointers and sizes, caller-owned
 * buffers mutated in place, errors reported through an out-parameter rather
 * than exceptions.  Differences, all forced by the device boundary:
 *
 *   - every pointer except `err` readbacks is DEVICE memory (cudaMalloc /
 *     torch CUDA tensors); every call is asynchronous on the caller's stream
 *     (`stream` is a cudaStream_t, NULL = legacy default stream);
 *   - the corpus arrives column-major (CSC: col_ptr int64, rows int32
 *     ascending inside a column, vals f64), i.e. the reference's
 *     CsrMatrix.csc_index() view (sparse.py:98-120) — the traversal of its
 *     deterministic "columns" mode (_jit.py:164-183);
 *   - the reference's errpos (2,) int64 becomes a device int64[SWMD_ERR_WORDS]
 *     record, reset by swmd_err_reset and read back by the host, which raises
 *     the reference's DegeneracyError messages (kernels.py:170-174,
 *     solver.py:95-103).
 *
 * Return value: 0 on success, a cudaError_t value on a CUDA failure, or one
 * of the SWMD_E* codes below for an argument the kernels cannot take.
 */
#ifndef SWMD_H
#define SWMD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SWMD_ABI_VERSION 2

#define SWMD_EINVAL 1000      /* bad size / null pointer / misaligned buffer */
#define SWMD_EVR 1001         /* v_r outside what this entry point supports */

/*
 * Error record (device int64[SWMD_ERR_WORDS]); "no event" is INT64_MAX.
 *   err[0]  min over zero denominators of (code << 47) | (i * n_key + j)
 *           — the smallest (i, j) in row-major order, i.e. the pair the
 *           reference's serial CSR walk reports first (_jit.py:130-134);
 *           (i * n_key + j) saturates at 2^47-1 (host then re-derives).
 *   err[1]  min event code of a nonpositive iterate entry (update_u check);
 *   err[2]  max |x_new - x_prev| as the bit pattern of a nonnegative double
 *           (tol path; reset to 0);
 *   err[3]  min event code at which an iterate entry was NaN.
 * Event codes order the reference's checks inside one solve: iteration t
 * performs update_u on x^(t) (code 2t) then the fused iteration (2t+1); the
 * final pass is update_u on x^(T) (code 2T) then fused_final (2T+1).
 */
#define SWMD_ERR_WORDS 4

int swmd_abi_version(void);
int swmd_device_sm_count(void);
int swmd_err_reset(int64_t* err, void* stream);
/* error record + solve work counter in one launch; enqueue it before the cost
 * build so the following swmd_solve_f64_reset_done starts right after it */
int swmd_solve_reset(int64_t* err, int32_t* counter, void* stream);

/* Row sums of squares of E (V x dim, row stride ldE) — cached per embedding
 * table for the Gram-form cost build. */
int swmd_row_norms_f64(const double* E, int64_t V, int32_t dim, int64_t ldE,
                       double* norms, void* stream);

/*
 * Cost + Gibbs-kernel build for one query: replaces _jit.euclid_rows
 * (_jit.py:90-102, called by kernels.euclidean_rows, kernels.py:91-111) fused
 * with _jit.precompute_mats (_jit.py:105-114, kernels.precompute,
 * kernels.py:114-141).  For each row i (all V rows, or the n_list rows in
 * row_list) and query word a < v_r:
 *     M[i,a]  = ||E[sel[a]] - E[i]||_2
 *     K[i,a]  = exp(-lam * M[i,a]);  KoR = K / weights[a];  KM = K * M
 * Outputs are (V, ldk) row-major, ldk >= v_r; columns a in [v_r, ldk) are
 * written as 0.  Any of cost / kernel_over_r / kernel_cost may be NULL.
 * mode 0: difference form in the reference's exact operation order
 *         (no FMA): bitwise-identical M.
 * mode 1: Gram form ||e||^2 + ||q||^2 - 2 e.q on FMA (norms required),
 *         M[sel[a],a] forced to exactly 0 and near-zero distances
 *         recomputed in difference form.
 */
int swmd_cost_build_f64(const double* E, int64_t V, int32_t dim, int64_t ldE,
                        const int64_t* sel, int32_t v_r, const double* weights,
                        double lam, int32_t mode, const double* norms,
                        const int32_t* row_list, int64_t n_list,
                        double* cost, double* kernel, double* kernel_over_r,
                        double* kernel_cost, int64_t ldk, void* stream);

/*
 * swmd_cost_build_f64 (Gram mode) for the rows a corpus actually uses, read
 * from their compacted copy E_c (n_c x dim, row stride ldEc, dim and ldEc
 * even): row r of E_c is vocabulary row row_ids[r] (row_ids NULL: identity).
 * E (row stride ldE) supplies the query vectors, norms are per vocabulary row.
 * Streams E_c through TMA tensor copies (cp.async.bulk.tensor, 128-byte
 * swizzle, 4-stage mbarrier ring of 32 KB boxes) into the FP64 tensor pipe (DMMA).
 */
int swmd_cost_build_compact_f64(const double* E, int64_t ldE, const double* E_c, int64_t n_c,
                                int32_t dim, int64_t ldEc, const int32_t* row_ids,
                                const int64_t* sel, int32_t v_r, const double* weights,
                                double lam, const double* norms, double* kernel,
                                double* kernel_cost, int64_t ldk, void* stream);
/* the same build, whose first thread also resets the solve's error record and
 * work counter (swmd_solve_reset folded into the cost launch) */
int swmd_cost_build_compact_reset_f64(const double* E, int64_t ldE, const double* E_c,
                                      int64_t n_c, int32_t dim, int64_t ldEc,
                                      const int32_t* row_ids, const int64_t* sel, int32_t v_r,
                                      const double* weights, double lam, const double* norms,
                                      double* kernel, double* kernel_cost, int64_t ldk,
                                      int64_t* err, int32_t* counter, void* stream);

/* Elementwise precompute from a given cost matrix: replaces
 * _jit.precompute_mats (_jit.py:105-114) behind kernels.precompute
 * (kernels.py:114-141).  kernel_over_r / kernel_cost may be NULL. */
int swmd_precompute_f64(const double* cost, int64_t V, int32_t v_r, int64_t ldk,
                        const double* weights, double lam, double* kernel,
                        double* kernel_over_r, double* kernel_cost, void* stream);

/*
 * The whole Sinkhorn loop for one query over a CSC column range, in ONE
 * persistent launch: replaces the solver loop of solver.py:168-193 —
 * update_u (solver.py:95-103) + _jit.fused_iter_columns (_jit.py:164-183)
 * per iteration and update_u + _jit.fused_final_columns (_jit.py:291-312)
 * at the end.  Columns are independent (test_acceptance.py:212-222), so
 * each column runs all of its iterations with x, u held on chip; v is never
 * stored.  kernel_over_r is folded: x[j,a] = (sum_i K[i,a] t_ij) / r[a].
 *   iterations t_begin <= t < t_end run; x_in (N x v_r) seeds x^(t_begin)
 *   (NULL = the reference's init 1/v_r); x_out (nullable) receives x^(t_end);
 *   wmd (nullable) receives the final pass; delta_out on err[2] when x_in
 *   is given (tol path).  order (nullable) is a column permutation used as
 *   the work order (longest columns first).  counter is a device int32
 *   scratch word (reset inside).  col_key_offset / n_key place the local
 *   columns in the global (i * n_key + j) error key.  group_hint = lanes per
 *   column for the register-only v_r <= 32 kernel (16 or 32); max_len_hint =
 *   longest column (sizes the shared-memory slab of staged K rows; 0 = 96).
 * Supports any v_r >= 1 (v_r <= 32 on the register-resident fast kernel).
 */
int swmd_solve_f64(const int64_t* col_ptr, const int32_t* rows, const double* vals,
                   int64_t n_cols, const int32_t* order,
                   const double* kernel, const double* kernel_cost,
                   const double* weights, int32_t v_r, int64_t ldk,
                   int32_t t_begin, int32_t t_end,
                   const double* x_in, double* x_out, double* wmd,
                   int64_t col_key_offset, int64_t n_key, int32_t group_hint,
                   int32_t max_len_hint, int64_t* err, int32_t* counter, void* stream);
/* swmd_solve_f64 whose counter (and error record) were reset by swmd_solve_reset
 * earlier on the stream: no memset node between the cost build and the solve */
int swmd_solve_f64_reset_done(const int64_t* col_ptr, const int32_t* rows, const double* vals,
                              int64_t n_cols, const int32_t* order,
                              const double* kernel, const double* kernel_cost,
                              const double* weights, int32_t v_r, int64_t ldk,
                              int32_t t_begin, int32_t t_end,
                              const double* x_in, double* x_out, double* wmd,
                              int64_t col_key_offset, int64_t n_key, int32_t group_hint,
                              int32_t max_len_hint, int64_t* err, int32_t* counter, void* stream);
/* swmd_solve_f64 for long queries (32 < v_r <= 256, the per-column gather of
 * _jit.py:164-183 / 291-312 at large v_r, where K no longer fits L2) with the
 * corpus's hot-row index: hot_slot[i] is the rank of vocabulary row i among
 * the corpus's n_hot most frequent rows (-1 when it is not one of them) and
 * hot_ids[s] the row of rank s.  The launch keeps the K rows of as many of
 * those ranks as fit beside its working set in shared memory (one CTA per SM,
 * several columns in flight per CTA sharing the slab), so the Zipf head of
 * the vocabulary is read from L2 once per launch instead of once per nonzero
 * and pass.  Results are bitwise those of swmd_solve_f64 (same rows, same
 * order; only where a row is read from differs).  Both index pointers NULL or
 * n_hot = 0: identical to swmd_solve_f64 / _reset_done (counter_zeroed != 0). */
int swmd_solve_hot_f64(const int64_t* col_ptr, const int32_t* rows, const double* vals,
                       int64_t n_cols, const int32_t* order,
                       const double* kernel, const double* kernel_cost,
                       const double* weights, int32_t v_r, int64_t ldk,
                       int32_t t_begin, int32_t t_end,
                       const double* x_in, double* x_out, double* wmd,
                       int64_t col_key_offset, int64_t n_key, int32_t group_hint,
                       int32_t max_len_hint, int64_t* err, int32_t* counter, void* stream,
                       int32_t counter_zeroed, const int32_t* hot_slot, const int32_t* hot_ids,
                       int32_t n_hot);

/*
 * fp32 multi-query variant (BASELINE config c4; the reference is fp64-only,
 * so these twin the f64 entry points for a batch of queries).
 * swmd_cost_build_batch_f32: one GEMM over the concatenated words of a batch;
 * output column c (of LD, LD % 4 == 0) holds word words[col_word[c]]
 * (col_word[c] == -1: zero padding).  K, K*M are (V, LD) fp32.
 * swmd_solve_f32: swmd_solve_f64 on fp32 K / K*M / weights / x / wmd; a
 * query's K block starts at its first column (16-byte aligned) with row
 * stride ldk = LD and zero padding up to v_r rounded to 8.
 */
int swmd_row_norms_f32(const float* E, int64_t V, int32_t dim, int64_t ldE, float* norms,
                       void* stream);
int swmd_cost_build_batch_f32(const float* E, int64_t V, int32_t dim, int64_t ldE,
                              const int64_t* words, const int32_t* col_word, int32_t LD,
                              float lam, const float* norms, const int32_t* row_list,
                              int64_t n_list, float* kernel, float* kernel_cost, void* stream);
int swmd_solve_f32(const int64_t* col_ptr, const int32_t* rows, const double* vals,
                   int64_t n_cols, const int32_t* order, const float* kernel,
                   const float* kernel_cost, const float* weights, int32_t v_r, int64_t ldk,
                   int32_t t_begin, int32_t t_end, const float* x_in, float* x_out, float* wmd,
                   int64_t col_key_offset, int64_t n_key, int32_t max_len_hint, int64_t* err,
                   int32_t* counter, void* stream);

/*
 * One fused type-1 iteration with explicit u and kernel_over_r, accumulating
 * into x (x[j,a] += sum ...; zero it first for a fresh iteration):
 * replaces _jit.fused_iter_serial / _columns (_jit.py:120-137, 164-183) as
 * called by kernels.fused_iteration (kernels.py:250-310).  Per column the
 * accumulation runs over rows in increasing order (the reference's order).
 * Zero denominators: event code 1.
 */
int swmd_fused_iteration_f64(const int64_t* col_ptr, const int32_t* rows,
                             const double* vals, int64_t n_cols,
                             const double* kernel, const double* kernel_over_r,
                             int32_t v_r, int64_t ldk, const double* u, double* x,
                             int64_t n_key, int64_t* err, void* stream);

/* Type-2 final pass with explicit u: wmd[j] = sum (c/(K_i.u_j)) (KM_i.u_j);
 * replaces _jit.fused_final_* (_jit.py:243-312) behind kernels.fused_final
 * (kernels.py:313-354).  wmd is overwritten.  Zero denominators: code 1. */
int swmd_fused_final_f64(const int64_t* col_ptr, const int32_t* rows,
                         const double* vals, int64_t n_cols,
                         const double* kernel, const double* kernel_cost,
                         int32_t v_r, int64_t ldk, const double* u, double* wmd,
                         int64_t n_key, int64_t* err, void* stream);

/* Unfused SDDMM: w[pos[q]] = vals[q] / (K[rows[q],:] . u[j,:]) with w in CSR
 * storage order (pos = CsrMatrix.csc_index()[2]); replaces _jit.sddmm_*
 * (_jit.py:319-358) behind kernels.sddmm (kernels.py:177-208).  A zero
 * denominator stores 0 and records code 1. */
int swmd_sddmm_f64(const int64_t* col_ptr, const int32_t* rows, const int64_t* pos,
                   const double* vals, int64_t n_cols, const double* kernel,
                   int32_t v_r, int64_t ldk, const double* u, double* w,
                   int64_t n_key, int64_t* err, void* stream);

/* Unfused SpMM: x[j,:] += sum_q kernel_over_r[rows[q],:] * w[pos[q]];
 * replaces _jit.spmm_* (_jit.py:361-398) behind kernels.spmm
 * (kernels.py:211-247).  Rows in increasing order per column. */
int swmd_spmm_f64(const int64_t* col_ptr, const int32_t* rows, const int64_t* pos,
                  const double* w, int64_t n_cols, const double* kernel_over_r,
                  int32_t v_r, int64_t ldk, double* x, void* stream);

/* Multi-query fp32 solve of one group of nq <= 4 queries with the same padded
 * width (v_rs[q] rounded up to 8, v_rs[q] <= 64) on one corpus: the whole
 * loop (max_iter iterations + the final pass, tol unset) in ONE persistent
 * launch that claims columns and solves each claimed column for every query
 * of the group in turn, so the column's CSC entries are read from HBM once
 * per group.  Per query q: kernels[q] / kernel_costs[q] (row stride ldk,
 * 16-byte aligned blocks of the batch K), weights[q] (v_rs[q] floats),
 * wmds[q] (n_cols floats), errs[q] (the 4-word error record, reset by the
 * caller).  Pointer arrays are host arrays of device pointers.  Replaces the
 * per-query loop of sinkhorn_wmd_batch (solver.py:204-223). */
int swmd_solve_group_f32(const int64_t* col_ptr, const int32_t* rows, const double* vals,
                         int64_t n_cols, const int32_t* order, int32_t nq,
                         const float* const* kernels, const float* const* kernel_costs,
                         const float* const* weights, const int32_t* v_rs, int64_t ldk,
                         int32_t max_iter, float* const* wmds, int64_t* const* errs,
                         int64_t col_key_offset, int64_t n_key, int32_t* counter, void* stream);

/* Unfused comparator, one Sinkhorn iteration t (baseline.unfused_sparse_wmd,
 * baseline.py:67-131): an SDDMM launch that applies update_u to x_in while
 * loading each column's row (event code 2t; x_in == NULL means x = 1/v_r,
 * init_x) and stores w[q] = vals[q] / (K[rows[q],:] . u[j,:]) for every
 * nonzero q in CSC order in HBM (zero denominator: w = 0, code 2t+1), then an
 * SpMM launch that reads w back and writes x_out[j,a] = (sum_q K[rows[q],a]
 * w[q]) / r[a] and records max |x_out - x_in| in err[2] (the tol test,
 * solver.py:179-183).  Rows are padded: ldk == ldx == swmd_unfused_row_width
 * (v_r) (pad columns of K zero).  v_r <= 64; SWMD_EVR otherwise. */
int swmd_unfused_row_width(int32_t v_r);
int swmd_unfused_iterate_f64(const int64_t* col_ptr, const int32_t* rows,
                             const double* vals, int64_t n_cols, const double* kernel,
                             const double* r, int32_t v_r, int64_t ldk,
                             const double* x_in, double* x_out, int64_t ldx, double* w,
                             int32_t t, int64_t key_off, int64_t n_key, int64_t* err,
                             void* stream);

/* Unfused comparator, final pass after t_final iterations: update_u on x_in
 * (code 2*t_final) and wmd[j] = sum_q (vals[q] / (K[i,:] . u)) (KM[i,:] . u)
 * (code 2*t_final+1), i.e. kernels.fused_final (kernels.py:313-354). */
int swmd_unfused_final_f64(const int64_t* col_ptr, const int32_t* rows,
                           const double* vals, int64_t n_cols, const double* kernel,
                           const double* kernel_cost, int32_t v_r, int64_t ldk,
                           const double* x_in, int64_t ldx, double* wmd, int32_t t_final,
                           int64_t key_off, int64_t n_key, int64_t* err, void* stream);

/* u = 1/x elementwise with the update_u check (solver.py:95-103): records
 * `code` in err[1] if any entry <= 0 and in err[3] if any entry is NaN. */
int swmd_update_u_f64(const double* x, double* u, int64_t n, int32_t code,
                      int64_t* err, void* stream);

/* HOST function: the query's positive entries (kernels.select_nonzero,
 * kernels.py:74-88) in one pass over the dense histogram r (n doubles).
 * Writes the ascending word ids to stage[0:cnt] and the weights (float64
 * bit patterns) to stage[cnt:2*cnt]; stage holds 2*cap int64.  Returns cnt,
 * -2 if an entry is negative (ValueError), -1 on bad arguments, or the
 * needed cap (> cap) when stage is too small.  cnt == 0 means no positive
 * entry (EmptyQueryError). */
int64_t swmd_select_query(const double* r, int64_t n, int64_t* stage, int64_t cap);

/* HOST function: memcpy of `bytes` from src to dst split over `threads`
 * threads (result buffers of a batch, detached from the pinned workspace). */
int swmd_host_copy(void* dst, const void* src, int64_t bytes, int32_t threads);

/*
 * Native per-query runtime (replaces the Python orchestration of
 * solver.py:106-201 for the common case tol == NULL, v_r <= 32).
 * swmd_plan_create binds the resident buffers once; desc is an int64 array:
 *   [0] E  [1] V  [2] dim  [3] ldE  [4] norms  [5] col_ptr  [6] rows  [7] vals
 *   [8] n_cols  [9] order  [10] present rows (or 0)  [11] n_present
 *   [12] col_key_offset  [13] n_key  [14] max_len  [15] group_hint
 *   [16] K  [17] KM  [18] K/KM capacity (doubles)  [19] device stage (2*q_cap
 *   int64)  [20] pinned host stage (2*q_cap int64)  [21] q_cap
 *   [22] device out (n_cols doubles + 4 int64 error record + 3 int64 device
 *   clock stamps)  [23] pinned host out (same)
 *   [24] int32 counter  [25] stream (optional)  [26] E_c  [27] n_c  [28] ldEc
 *   (optional: compacted corpus rows for the TMA cost build, 0 = none)
 * swmd_plan_run: select (host) -> H2D -> cost build -> solve -> D2H -> sync;
 * copies the distances to wmd_host and the error record to err_host and the
 * cost / solve device times (ms) to times_ms[0..1]; host times (ms, from
 * entry) to times_ms[2] (select done), [3] (all work enqueued), [4] (stream
 * synchronised), [5] (results copied out) — times_ms holds 6 floats or is
 * NULL.  Returns 0, a CUDA
 * error, -2 (negative query entry), -3 (no positive entry) or -4 (query
 * outside the plan's fast path: the caller uses the general entry points).
 */
typedef struct swmd_plan swmd_plan;
int swmd_plan_create(swmd_plan** out, const int64_t* desc, int32_t n);
int swmd_plan_destroy(swmd_plan* plan);
int swmd_plan_run(swmd_plan* plan, const double* query, int64_t V, double lam,
                  int32_t max_iter, int32_t cost_mode, double* wmd_host,
                  int64_t* err_host, float* times_ms, int64_t* v_r_out);

/* swmd_plan_run for a query already in selected form (ascending unique word
 * ids sel[0:v_r] and positive weights — a SparseVector histogram, the
 * reference's ingest output): no dense scan.  -4 when the selection is not
 * valid or too wide for the native path (the caller's general path decides). */
int swmd_plan_run_selected(swmd_plan* p, const int64_t* sel, const double* weights,
                           int64_t v_r, double lam, int32_t max_iter, int32_t cost_mode,
                           double* wmd_host, int64_t* err_host, float* times_ms);

/* swmd_plan_run with the distances (n_cols doubles) and the 4-word error
 * record written to caller device buffers and nothing copied back: the
 * work is only enqueued on the plan's stream (no synchronisation), so the
 * caller's next stream operation — the multi-GPU path's all-gather of the
 * distance slots (distributed.py) — consumes them in place.  Same return
 * codes as swmd_plan_run (-4: outside the native fast path). */
int swmd_plan_run_device(swmd_plan* p, const double* query, int64_t V, double lam,
                         int32_t max_iter, int32_t cost_mode, double* wmd_dev,
                         int64_t* err_dev, int64_t* v_r_out);

/*
 * Device CSR -> CSC transpose (replaces the host argsort of
 * CsrMatrix.csc_index, sparse.py:98-120): from row_ptr (n_rows+1), col_idx,
 * vals (nnz) to col_ptr (n_cols+1), rows (int32), cvals and pos (the CSR
 * position of each CSC slot), rows ascending inside each column — identical
 * to the host transpose.  Columns longer than 1024 entries are left unsorted
 * and the longest such length is written to *longest_unsorted (0: all done);
 * the caller then sorts those on the host.  scratch: device memory of
 * swmd_csr_to_csc_scratch_bytes(n_cols) bytes.
 */
int swmd_csr_to_csc_f64(const int64_t* row_ptr, const int64_t* col_idx, const double* vals,
                        int64_t n_rows, int64_t n_cols, int64_t nnz, int64_t* col_ptr,
                        int32_t* rows, double* cvals, int64_t* pos, void* scratch,
                        int64_t scratch_bytes, int32_t* longest_unsorted, void* stream);
int64_t swmd_csr_to_csc_scratch_bytes(int64_t n_cols);

/*
 * Device top-k of a distance vector (north_star: identical top-k document
 * indices): the k <= 1024 smallest values in ascending order, ties broken
 * toward the lower index — exactly np.argsort(values, kind="stable")[:k]
 * (NaN sorts last).  out_idx receives index + index_offset.  scratch must
 * hold swmd_topk_scratch_bytes(n, k) bytes of device memory.
 */
int swmd_topk_f64(const double* values, int64_t n, int32_t k, int64_t index_offset,
                  int64_t* out_idx, double* out_val, void* scratch, int64_t scratch_bytes,
                  void* stream);
int64_t swmd_topk_scratch_bytes(int64_t n, int32_t k);

/*
 * HOST function: claim order of the persistent solve (DeviceCorpus.order) for
 * `slots` resident warps.  The solve's warps claim columns through one atomic
 * counter in this order; the reference walks columns in index order
 * (_jit.py:164-183, deterministic mode) and results do not depend on the
 * order.  Longest-first when n_cols <= slots or n_cols > max_ratio * slots;
 * otherwise a MULTIFIT plan (first-fit-decreasing under a binary-searched
 * capacity) of the per-column time model (register rounds `reg_rounds`,
 * `slab_rows` shared-memory rows) serialised by planned start time
 * (paper_2107_06433_b200/schedule.py restates it).  Writes n_cols ids.
 */
int swmd_schedule_order(const int64_t* col_ptr, int64_t n_cols, int32_t slots,
                        int32_t reg_rounds, int32_t slab_rows, int32_t max_ratio,
                        int32_t* order);
/* resident warps of the f64 persistent solve for a query of v_r words on the
 * current device (0 for v_r > 32, whose kernels take columns longest-first),
 * and its register-round count */
int swmd_solve_slots_f64(int32_t v_r, int32_t* slots);
int swmd_solve_reg_rounds_f64(int32_t v_r);

/* Flush helper for benchmarks: writes `bytes` of scratch (> L2 evicts
 * everything) and reads it back, leaving L2 clean (no dirty write-back is
 * charged to the next kernel). */
int swmd_l2_flush(void* scratch, int64_t bytes, void* stream);

/* Host helper: a multiply-xorshift hash of 64 strided elements + the last 16 of a host
 * array (n elements of itemsize bytes) — the in-place-edit check of the
 * resident embedding-table cache (device.py). */
int64_t swmd_sample_crc(const void* data, int64_t n, int64_t itemsize);
/* Host helper: a hash of EVERY byte of a host buffer (`threads` host threads)
 * — the edit check of a writeable embedding table (device.py). */
int64_t swmd_content_hash(const void* data, int64_t bytes, int32_t threads);

#ifdef __cplusplus
}
#endif
#endif /* SWMD_H */
