/*
 * svdrec_b200.h -- C ABI of the B200-native adaptive-PCA / CF hot path.
 *
 * Drop-in boundary for the reference package ``svdrec``
 * (/root/reference/pkg/src/svdrec).  The reference is Python; its hot path
 * calls numpy/scipy through the functions cited below.  Each entry point
 * here replaces one of those calls with an sm_100a kernel; the Python host
 * layer (paper_2009_02251_b200/) binds them with ctypes exactly like the
 * stub in INTEGRATION.md and mirrors the reference's function names,
 * argument meaning and errors.
 *
 * Conventions
 *  - plain pointers + sizes, no torch types; every pointer named d_* is
 *    DEVICE memory, every other pointer is host memory;
 *  - dense matrices are ROW-MAJOR with an explicit leading dimension
 *    (elements), float64 unless the name says otherwise;
 *  - ``stream`` is a cudaStream_t passed as void*; every call is
 *    asynchronous on that stream, nothing synchronises the device;
 *  - return value: 0 on success, otherwise a CUDA error code (>0) or a
 *    negative SVDREC_E* code; svdrec_last_error() gives the message;
 *  - data-dependent failures that the reference raises as exceptions
 *    (rank-deficient pivot, near-singular Gram, exhausted raw stream) are
 *    reported through a device int32 status word the caller reads back
 *    when it next synchronises (bit flags SVDREC_STATUS_*).
 *  - scratch memory is supplied by the caller; *_workspace_bytes() sizes it.
 */
#ifndef SVDREC_B200_H
#define SVDREC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SVDREC_E_ARG (-1)       /* invalid argument (shape, ld, size)   */
#define SVDREC_E_WORKSPACE (-2) /* workspace smaller than required      */
#define SVDREC_E_UNSUPPORTED (-3)

#define SVDREC_STATUS_ZERO_PIVOT 1u    /* lu: exactly singular pivot    */
#define SVDREC_STATUS_NEAR_SINGULAR 2u /* eig: Gram eigenvalue <= floor */
#define SVDREC_STATUS_STREAM_SHORT 4u  /* normal: raw window too short  */
#define SVDREC_STATUS_NO_CONVERGE 8u   /* eig: Jacobi sweep cap hit     */
#define SVDREC_STATUS_NS_CHECK 16u     /* inv_sqrt: inconclusive, check
                                          singularity with svdrec_syev   */

int svdrec_abi_version(void);
const char* svdrec_last_error(void);
int svdrec_device_sm_count(void);
/* Number of kernels this library has launched in the process so far. */
long long svdrec_launch_count(void);

/* ---------------------------------------------------------------------
 * Gaussian stream.  Replaces GaussianStream.normal / gaussian_matrix
 * (reference pkg/src/svdrec/linalg.py:28-51), i.e. numpy
 * Generator(Philox(key=seed)).standard_normal((rows, cols)).  Bit-exact:
 * Philox4x64-10 raw words parsed by numpy's 256-layer ziggurat as a
 * 3-state transducer with a parallel chunk-composition scan.
 *
 * Draws ``count`` samples starting at raw-word position *d_pos (device
 * int64, 0 for a fresh seed) and advances *d_pos past them, so successive
 * calls continue the stream exactly as the reference's successive
 * stream.normal() calls do.  out[e] is the e-th sample (C order of the
 * reference's (rows, cols) draw); with ``row_perm`` non-NULL sample
 * (i, j) of a (count/cols, cols) draw lands at out[row_perm[i]*ld + j].
 * ------------------------------------------------------------------- */
size_t svdrec_normal_workspace_bytes(int64_t count);
int svdrec_normal_fill(uint64_t key_lo, uint64_t key_hi, int64_t* d_pos,
                       int64_t count, int64_t cols, const int32_t* d_row_perm,
                       double* d_out, int64_t ld, void* d_work, size_t work_bytes,
                       uint32_t* d_status, void* stream);

/* ---------------------------------------------------------------------
 * Sparse x dense.  Replaces sparse_dense_mul (linalg.py:141-158):
 * Y = A @ X with A in CSR (int64 indptr, int32 indices, float64 values).
 * A.T @ X is the same call on the CSR of A.T (the host keeps both).
 * Rows are described by segments (row, [begin, end) of the CSR arrays);
 * the simplest valid plan is one segment per row (seg_row[i] = i,
 * seg_begin/end = indptr[i]/indptr[i+1], seg_slot = -1, nlong = 0,
 * nwarp = 0).  The Python host cuts long rows into <= 2048-nonzero segments
 * whose partial sums a deterministic fix-up adds in slot order
 * (paper_2009_02251_b200/sparse.py: segment_plan), so results are bitwise
 * reproducible run to run; tests/c_abi/spmm_smoke.c is a plain-C caller.
 *   seg_row/seg_begin/seg_end : nseg segments, row-ordered
 *   seg_slot                  : -1 = segment covers its whole row (direct
 *                               store), else partial slot index
 *   long_row/long_slot0/long_slot1: nlong split rows and their slot range
 *   x_rows                    : rows of X (= columns of A)
 *   nwarp/warp_seg            : optional balanced schedule (nwarp = 0:
 *                               none): warp w owns segments
 *                               [warp_seg[w], warp_seg[w+1]) -- contiguous,
 *                               ~equal nonzeros (svdrec_warp_plan), nwarp =
 *                               SMs x svdrec_spmm_warps_per_sm(b)
 *   warp_chunk/chunks         : the same schedule in chunk records, which
 *                               the pipelined kernel for even b <= 32 reads
 *                               (svdrec_chunk_plan: 16-B records of <= 32
 *                               entries; svdrec_warp_chunks: warp w owns
 *                               records [warp_chunk[w], warp_chunk[w+1])).
 *                               32 < b <= 64 (b % 4 == 0) runs the wide
 *                               kernel on warp_seg; without the matching
 *                               plan the plain row-per-warp kernel runs
 *   slot_long/long_done       : optional, for the pipelined kernel: the
 *                               split rows' partial sums are added inside
 *                               the kernel (by the warp that finishes a
 *                               row's last outstanding segment, in slot
 *                               order: the fix-up kernel's sum bit for bit)
 *                               instead of by a second launch.  slot_long[s]
 *                               = index of slot s's split row; long_done =
 *                               nlong int32 tickets, zero before the first
 *                               call (the kernel leaves them zero).  NULL:
 *                               the fix-up kernel runs
 *   d_partial                 : (nslots x b) scratch
 * ------------------------------------------------------------------- */
int svdrec_spmm(int64_t nseg, const int32_t* d_seg_row, const int64_t* d_seg_begin,
                const int64_t* d_seg_end, const int32_t* d_seg_slot,
                const int32_t* d_indices, const double* d_values,
                const double* d_X, int64_t ldx, int64_t x_rows, double* d_Y, int64_t ldy,
                int32_t b, int64_t nlong, const int32_t* d_long_row, const int32_t* d_long_slot0,
                const int32_t* d_long_slot1, int64_t nwarp, const int32_t* d_warp_seg,
                const int32_t* d_warp_chunk, const void* d_chunks, const int32_t* d_slot_long,
                int32_t* d_long_done, double* d_partial, void* stream);
/* Warps per SM of the schedule (nwarp = SMs x this) that the pipelined
 * kernel for width b runs: 16 for even b <= 32 (two 8-warp CTAs, 2 doubles
 * per lane), fewer for 32 < b <= 64 with b % 4 == 0 (4 doubles per lane,
 * wider gather rings).  Without a schedule (or for odd b / unaligned rows)
 * the plain row-per-warp kernel runs. */
int svdrec_spmm_warps_per_sm(int32_t b);
/* Hot-set variant of A @ X (even b <= 32, or b % 4 == 0 up to 64): the
 * rows X[d_hot_items[rank]] of the nhot most rated items (rank < nhot)
 * are staged in every CTA's shared memory; the CSR is given as its
 * hot-first copy (svdrec_spmm_hot_partition: every row stably partitioned
 * into the hot items' entries, index -(rank + 1), then the others, index
 * = item id; d_rank = item -> popularity rank), with A's row structure.
 * Each 32-entry batch is split by a warp ballot into its hot entries
 * (shared memory) and cold ones (L2 / HBM gathers).  Same segment plan /
 * fix-up as svdrec_spmm, schedule of 16 warps per SM;
 * nhot <= svdrec_spmm_hot_rows(b) (0: width not supported). */
int svdrec_spmm_hot_rows(int32_t b);
int svdrec_spmm_hot_partition(int64_t m, const int64_t* d_indptr, const int32_t* d_indices,
                              const double* d_values, const int32_t* d_rank, int32_t nhot,
                              int32_t* d_out_indices, double* d_out_values, void* stream);
int svdrec_spmm_hot(int64_t nseg, const int32_t* d_seg_row, const int64_t* d_seg_begin,
                    const int64_t* d_seg_end, const int32_t* d_seg_slot, const int32_t* d_hidx,
                    const double* d_hval, const double* d_X, int64_t ldx, int64_t x_rows,
                    const int32_t* d_hot_items,
                    int32_t nhot, double* d_Y, int64_t ldy, int32_t b, int64_t nlong,
                    const int32_t* d_long_row, const int32_t* d_long_slot0, const int32_t* d_long_slot1,
                    int64_t nwarp, const int32_t* d_warp_seg, double* d_partial, void* stream);
/* Hot / cold chunk kernel for A @ X (even b <= 32; the path the headline's
 * b = 20 products A @ Omega and A @ r take).  hot_pack: the PACKED hot-first
 * copy of a CSR -- 16-B entries {int32 id, int32 0, double value}, every row
 * stably partitioned into the entries of the nhot most rated items (id =
 * popularity rank = row of the shared-memory table) and the rest (id =
 * item) -- and d_hot_cnt[r] = row r's hot entries.  The chunk plan is
 * svdrec_chunk_plan with d_indptr / d_hot_cnt (no chunk straddles a row's
 * hot / cold boundary), svdrec_warp_chunks for nwarp = SMs x
 * svdrec_spmm_hc_warps_per_sm().  Hot chunks read X rows from shared memory,
 * cold chunks gather them (LDG) -- only those reach L2.
 * nhot <= svdrec_spmm_hc_rows(b) (0: width not supported). */
int svdrec_spmm_hc_warps_per_sm(void);
int svdrec_spmm_hc_rows(int32_t b);
int svdrec_spmm_hot_pack(int64_t m, const int64_t* d_indptr, const int32_t* d_indices,
                         const double* d_values, const int32_t* d_rank, int32_t nhot, void* d_out,
                         int32_t* d_hot_cnt, void* stream);
int svdrec_spmm_hc(int64_t nseg, const void* d_entries, const double* d_X, int64_t ldx, int64_t x_rows,
                   const int32_t* d_hot_items, int32_t nhot, double* d_Y, int64_t ldy, int32_t b,
                   int64_t nlong, const int32_t* d_long_row, const int32_t* d_long_slot0,
                   const int32_t* d_long_slot1, int64_t nwarp, const int32_t* d_warp_chunk,
                   const void* d_chunks, double* d_partial, void* stream);
/* fp32 variant: X stored as float (half the gathered bytes), values,
 * accumulation and Y in double.  b in {4, 8, ..., 64}, 16-B aligned rows,
 * a schedule of svdrec_spmm_x32_warps_per_sm(b) warps per SM. */
int svdrec_spmm_x32_warps_per_sm(int32_t b);
int svdrec_spmm_x32(int64_t nseg, const int32_t* d_seg_row, const int64_t* d_seg_begin,
                    const int64_t* d_seg_end, const int32_t* d_seg_slot,
                    const int32_t* d_indices, const double* d_values,
                    const float* d_X, int64_t ldx, int64_t x_rows, double* d_Y, int64_t ldy,
                    int32_t b, int64_t nlong, const int32_t* d_long_row, const int32_t* d_long_slot0,
                    const int32_t* d_long_slot1, int64_t nwarp, const int32_t* d_warp_seg,
                    const int32_t* d_warp_chunk, const void* d_chunks, const int32_t* d_slot_long,
                    int32_t* d_long_done, double* d_partial, void* stream);
/* ---------------------------------------------------------------------
 * Dense tall-skinny contractions (the deflation products of
 * rsvd.py:135-142, 179-194: Q @ (B @ X), Q @ (Q.T @ X), B.T @ (Q.T @ X)
 * and the Gram M.T @ M of eig_svd, linalg.py:127).
 *   gemm_tn: C (p x q) = alpha * X.T @ Y + beta * C, X (r x p), Y (r x q);
 *            deterministic split-r reduction through d_work.
 *   gemm_nn: Y (r x q) = alpha * X @ C + beta * Y, X (r x p), C (p x q).
 * ------------------------------------------------------------------- */
size_t svdrec_gemm_tn_workspace_bytes(int64_t r, int64_t p, int64_t q);
int svdrec_gemm_tn(int64_t r, int64_t p, int64_t q, double alpha, const double* d_X,
                   int64_t ldx, const double* d_Y, int64_t ldy, double beta, double* d_C,
                   int64_t ldc, void* d_work, size_t work_bytes, void* stream);
int svdrec_gemm_nn(int64_t r, int64_t p, int64_t q, double alpha, const double* d_X,
                   int64_t ldx, const double* d_C, int64_t ldc, double beta, double* d_Y,
                   int64_t ldy, void* stream);

/* Sum of squares of a strided r x q block, per column (d_colsq, q values,
 * may be NULL) and in total (d_total, 1 value, may be NULL); fixed-order.
 * fro_norm_sq (linalg.py:161-168) and the error-indicator update
 * ||B_i||_F^2 (rsvd.py:146, 197) / row energies (rsvd.py:209). */
size_t svdrec_sumsq_workspace_bytes(int64_t r, int64_t q);
int svdrec_sumsq(int64_t r, int64_t q, const double* d_X, int64_t ldx, double* d_colsq,
                 double* d_total, void* d_work, size_t work_bytes, void* stream);

/* Fixed-order sum of a float64 vector (the global mean of _global_mean,
 * cf.py:102-105). */
size_t svdrec_vec_sum_workspace_bytes(int64_t n);
int svdrec_vec_sum(int64_t n, const double* d_x, double* d_out, void* d_work, size_t work_bytes, void* stream);

/* ---------------------------------------------------------------------
 * orthonormal_basis (linalg.py:54-81): economic Householder QR of the
 * tall r x b block A via a TSQR tree; writes the explicit Q (r x b, may
 * alias A) and R (b x b row-major, upper).  Orthonormal to working
 * precision even for rank-deficient input (the reference's
 * check_rank=False behaviour); the host applies the 1e-12 |R_ii| floor.
 * Supports b <= 80.
 * ------------------------------------------------------------------- */
size_t svdrec_tsqr_workspace_bytes(int64_t r, int32_t b);
int svdrec_tsqr(int64_t r, int32_t b, const double* d_A, int64_t lda, double* d_Q,
                int64_t ldq, double* d_R, void* d_work, size_t work_bytes, void* stream);

/* Orthonormal basis without R, as the QB engines use it (rsvd.py:136-142,
 * 186-193): CholeskyQR2 (two passes of Gram + Cholesky + triangular apply,
 * same Q up to column signs as Householder) with a device-side check --
 * non-positive pivot or kappa > 1e6 -- that gates a Householder TSQR of the
 * untouched input launched behind it.  No host round trip; Q may alias A.
 * b <= 64 takes the fast path, 64 < b <= 80 goes to TSQR directly. */
size_t svdrec_orth_workspace_bytes(int64_t r, int32_t b);
int svdrec_orth(int64_t r, int32_t b, const double* d_A, int64_t lda, double* d_Q, int64_t ldq,
                void* d_work, size_t work_bytes, void* stream);

/* Row-sharded CholeskyQR building blocks (the multi-GPU engine's
 * orthonormalisation; no single reference function -- together they replace
 * orthonormal_basis, linalg.py:54-81, and lu_lower_basis, linalg.py:84-97,
 * when the rows of the block are spread over ranks).  svdrec_gram writes
 * the full symmetric b x b Gram Y.T Y of this rank's r rows (fixed-order
 * sum; r may be 0); the caller all-reduces it over the ranks;
 * svdrec_chol_apply factors R = chol(G + shift_rel * trace(G) * I) (upper)
 * and writes Q = Y R^-1 for this rank's rows (Q may alias Y).  A
 * non-positive pivot sets SVDREC_STATUS_ZERO_PIVOT in d_status.  b <= 64. */
size_t svdrec_gram_workspace_bytes(int64_t r, int32_t b);
int svdrec_gram(int64_t r, int32_t b, const double* d_Y, int64_t ldy, double* d_G, void* d_work,
                size_t work_bytes, void* stream);
size_t svdrec_chol_apply_workspace_bytes(int64_t r, int32_t b);
int svdrec_chol_apply(int64_t r, int32_t b, const double* d_G, int64_t ldg, double shift_rel,
                      const double* d_Y, int64_t ldy, double* d_Q, int64_t ldq, uint32_t* d_status,
                      void* d_work, size_t work_bytes, void* stream);

/* ---------------------------------------------------------------------
 * lu_lower_basis (linalg.py:84-97): partial-pivoting LU of the tall
 * r x b block, in place, returning P.L (original row order, unit
 * diagonal on pivot rows) and U's diagonal in d_udiag (b values).
 * Exactly zero pivot -> SVDREC_STATUS_ZERO_PIVOT.  One cooperative
 * kernel, one grid barrier per column.
 * ------------------------------------------------------------------- */
size_t svdrec_lu_workspace_bytes(int64_t r, int32_t b);
/* 1 if the r x b factorization takes the panel-resident (shared-memory)
 * path -- every CTA's rows on chip, ~0.1 ms at 138k x 20 -- else 0 (the
 * global-memory path: one grid barrier per column over r rows, slow for
 * tall blocks; the QB engines then use a CholeskyQR basis instead, which
 * spans the same columns, see rsvd.py). */
int svdrec_lu_fast_path(int64_t r, int32_t b);
int svdrec_lu_lower(int64_t r, int32_t b, double* d_A, int64_t lda, double* d_udiag,
                    void* d_work, size_t work_bytes, uint32_t* d_status, void* stream);

/* ---------------------------------------------------------------------
 * Symmetric eigendecomposition for eig_svd (linalg.py:108-138): the
 * k x k Gram G (row-major, symmetric PSD) -> eigenvalues ascending in
 * d_w and eigenvectors as columns of d_V (k x k row-major).  Blocked
 * one-sided Jacobi in one cooperative kernel (k <= 760; scalar rounds
 * beyond).  d_V0 (nullable, k x k row-major orthonormal) warm-starts the
 * sweeps, e.g. with the previous block's eigenvectors padded by I.  Flags
 * SVDREC_STATUS_NEAR_SINGULAR when w[0] <= 0 or w[0] < 1e-14 trace(G).
 * ------------------------------------------------------------------- */
size_t svdrec_syev_workspace_bytes(int32_t k);
int svdrec_syev(int32_t k, const double* d_G, int64_t ldg, const double* d_V0, int64_t ldv0,
                double* d_w, double* d_V, int64_t ldv, void* d_work, size_t work_bytes,
                uint32_t* d_status, void* stream);

/* One-sided Jacobi SVD of a tall rows x k block (rows >= k): singular
 * values descending in d_s, left vectors d_U (rows x k), right vectors as
 * columns of d_V (k x k).  Replaces scipy.linalg.svd(b) of basic_rsvd
 * (rsvd.py:263), applied to b.T so no condition number is squared. */
size_t svdrec_gesvj_workspace_bytes(int64_t rows, int32_t k);
int svdrec_gesvj(int64_t rows, int32_t k, const double* d_A, int64_t lda, double* d_s, double* d_U,
                 int64_t ldu, double* d_V, int64_t ldv, void* d_work, size_t work_bytes,
                 uint32_t* d_status, void* stream);

/* ---------------------------------------------------------------------
 * Collaborative filtering (cf.py:77-190).
 *  Item similarity is the cosine of Alg. 4 in a metric M:
 *  cos(l, j) = x_j.y_l / (n_l n_j), y_l = M x_l, n_l = sqrt(x_l.y_l).
 *  With explicit factors T (LatentFactors) x_l = y_l = T[:, l]; per QB
 *  block x_l = B[:, l] and M = (B B.T)^(-1/2) (svdrec_inv_sqrt), which
 *  gives exactly the cosines of latent_from_qb's T without an eig.
 *  svdrec_cf_normalize: unit rows Tn = T.T / |T_l| and norms (x = y = T).
 *  svdrec_cf_normalize_pair: Xn = X / n, Yn = Y / n with n_l =
 *   sqrt(x_l.y_l) (zero rows where n_l = 0, the reference's skipped
 *   zero-norm items).
 *  svdrec_cf_predict: Alg. 4 (_predict, cf.py:108-143) for held-out
 *   (user, item) samples sorted by user.  Per user one warp forms
 *   P_u = sum_l A(u,l) Yn_l and S_u = sum_l Yn_l, then each sample's
 *   raw prediction is (Xn_j . P_u) / (Xn_j . S_u) with the |w| < 1e-9
 *   user-mean / global-mean fallback and clamping.  Writes clamped value,
 *   raw value and fallback flag per sample (in sorted order).  k <= 1024.
 *   The training CSR is passed RANKED: each item id replaced by its
 *   popularity rank (0 = most rated; svdrec_csr_transpose of A.T taken
 *   in popularity order builds it) and each row's
 *   entries ordered by rank, with d_Yr the unit rows Yn in rank order
 *   (Yr[rank(l)] = Yn[l]) plus one zero row at index n_items (the
 *   padding target), rows 16-B aligned (ldy even; float: ldy % 4 == 0) and
 *   zero-padded to that width (16-B vector loads);
 *   d_Xn and d_norm stay indexed by item id, as do
 *   the samples (d_items).  The first rows of Yr that fit in ~208 KB are
 *   staged in every CTA's shared memory, so each user's hot ratings (a
 *   prefix of the ranked row) read shared memory.  Work items -- a user,
 *   or a <= 512-rating chunk of a heavy user -- are claimed dynamically
 *   through d_counter (one device int32, reset here), heaviest first:
 *   item w starts at CSR entry d_work_start[w] and d_work_meta[8w..8w+7]
 *   = (length, user degree, first sample, end sample, chunks of the user,
 *   partial slot or -1, completion counter, chunk index).  Chunks store
 *   (P, S, sum v) in d_partial ((2k+1) doubles per slot) and the warp
 *   completing the user (d_done counters, ndone of them, reset here) adds
 *   the slots in order and scores the user's samples.
 *  svdrec_err_sum: fixed-order sum |pred - truth| and (pred-truth)^2.
 * ------------------------------------------------------------------- */
int svdrec_cf_normalize(int64_t n, int32_t k, const double* d_Tt, int64_t ldt, double* d_Tn,
                        int64_t ldn, double* d_norm, void* stream);
int svdrec_cf_normalize_pair(int64_t n, int32_t k, const double* d_X, int64_t ldx,
                             const double* d_Y, int64_t ldy, double* d_Xn, double* d_Yn,
                             int64_t ldn, double* d_norm, void* stream);
int svdrec_cf_predict(int64_t nwork, const int64_t* d_work_start, const int32_t* d_work_meta,
                      const int32_t* d_items, const int32_t* d_ranked_indices,
                      const double* d_ranked_values, int32_t k, const double* d_Yr, int64_t ldy,
                      const double* d_Xn, int64_t ldn, const double* d_norm, double global_mean,
                      double rating_min, double rating_max, int32_t n_items, int32_t* d_done,
                      int64_t ndone, double* d_partial, int32_t* d_counter, double* d_value,
                      double* d_raw, uint8_t* d_fallback, void* stream);
/* fp32 variant: d_Yr (leading dimension ldy) stored as float -- half the
 * gathered bytes and twice the rows staged on chip; accumulation, the
 * sample rows d_Xn and all outputs stay double. */
int svdrec_cf_predict_f32(int64_t nwork, const int64_t* d_work_start, const int32_t* d_work_meta,
                          const int32_t* d_items, const int32_t* d_ranked_indices,
                          const double* d_ranked_values, int32_t k, const float* d_Yr, int64_t ldy,
                          const double* d_Xn, int64_t ldn, const double* d_norm, double global_mean,
                          double rating_min, double rating_max, int32_t n_items, int32_t* d_done,
                          int64_t ndone, double* d_partial, int32_t* d_counter, double* d_value,
                          double* d_raw, uint8_t* d_fallback, void* stream);
/* Ranked CSR for svdrec_cf_predict: d_out[t] = d_rank[d_indices[t]] (item ->
 * popularity rank, 0 = most rated); the caller then orders each row's
 * entries by rank (ascending), so every user's hot items form a prefix. */
/* Alg. 4 for wide factors (k > 1024, which svdrec_cf_predict rejects): the
 * same outputs, one CTA per user group.  Groups are runs of samples of one
 * user: samples [group_offsets[g], group_offsets[g+1]) belong to user
 * group_users[g]; d_indptr is the training CSR's row pointer (the ranked
 * copy shares it); d_Yr the unit rows in rank order (n_items x ldy). */
int svdrec_cf_predict_wide(int64_t ngroups, const int64_t* d_group_offsets, const int64_t* d_group_users,
                           const int64_t* d_indptr, const int32_t* d_items, const int32_t* d_ranked_indices,
                           const double* d_ranked_values, int32_t k, const double* d_Yr, int64_t ldy,
                           const double* d_Xn, int64_t ldn, const double* d_norm, double global_mean,
                           double rating_min, double rating_max, double* d_value, double* d_raw,
                           uint8_t* d_fallback, void* stream);
/* The scoring kernel's work plan (see svdrec_cf_predict) on the device:
 * groups with degree d_group_deg (int64, ngroups), heaviest-first order
 * d_order (a stable sort of -degree).  plan_scan writes d_first (first
 * work item of the j-th group in that order), d_slot0 / d_done_idx (per
 * group: first partial slot / completion counter of a split group, -1
 * otherwise) and d_stats = (work items, split groups, partial slots,
 * ratings streamed); plan_emit writes d_work_start / d_work_meta
 * (d_stats[0] items; d_group_start: ngroups + 1 sample offsets,
 * d_row_start: CSR offset of each group's user row). */
int svdrec_cf_plan_scan(int64_t ngroups, const int64_t* d_group_deg, const int64_t* d_order, int32_t chunk,
                        int64_t* d_first, int32_t* d_slot0, int32_t* d_done_idx, int64_t* d_stats,
                        void* stream);
int svdrec_cf_plan_emit(int64_t ngroups, const int64_t* d_group_deg, const int64_t* d_order,
                        const int64_t* d_first, const int32_t* d_slot0, const int32_t* d_done_idx,
                        const int64_t* d_group_start, const int64_t* d_row_start, int32_t chunk,
                        int64_t* d_work_start, int32_t* d_work_meta, void* stream);

/* Stable counting-sort transpose of a CSR, on the device (ingest; replaces
 * the reference's scipy transpose behind ``A.T @ X``, linalg.py:141-158,
 * and SparseRatings.transposed, sparse.py).  The nrows input rows are
 * taken in processing order d_perm (nullable: identity) with d_pptr[q] =
 * sum of the lengths of the first q rows in that order (nrows + 1
 * entries; total = d_pptr[nrows], passed by the caller: no device read).  Output row c (c < n_out) lists, in processing order, every
 * input row holding column c: its entries carry the input row's index
 * (relabel = 0) or its processing position (relabel = 1) and the value.
 * Writes d_out_indptr (n_out + 1), d_out_indices / d_out_values (one per
 * entry).  Deterministic; no sort.  Fewer than 2^31 entries.  Scratch:
 * svdrec_csr_transpose_scratch(n_out) + 2 x (entries x 4 B, rounded up to
 * 256 B). */
int64_t svdrec_csr_transpose_scratch(int64_t n_out);
int svdrec_csr_transpose(int64_t nrows, int64_t n_out, int64_t total, const int64_t* d_indptr,
                         const int32_t* d_indices, const double* d_values, const int32_t* d_perm,
                         const int64_t* d_pptr, int32_t relabel,
                         int64_t* d_out_indptr, int32_t* d_out_indices, double* d_out_values, void* d_scratch,
                         int64_t scratch_bytes, void* stream);

/* G^(-1/2) of a k x k SPD Gram by coupled Newton-Schulz iteration (one
 * cooperative kernel, GEMM phases over the whole GPU).  Sets
 * SVDREC_STATUS_NS_CHECK when it cannot certify the reference's
 * near-singularity floor (eigenvalue >= 1e-14 trace); the caller then
 * decides with svdrec_syev.  d_iters (nullable) receives the iterations. */
size_t svdrec_inv_sqrt_workspace_bytes(int32_t k);
int svdrec_inv_sqrt(int32_t k, const double* d_G, int64_t ldg, double* d_Z, int64_t ldz,
                    void* d_work, size_t work_bytes, uint32_t* d_status, int32_t* d_iters,
                    void* stream);
size_t svdrec_err_sum_workspace_bytes(int64_t nsamp);
int svdrec_err_sum(int64_t nsamp, const double* d_pred, const double* d_truth,
                   double* d_out2, void* d_work, size_t work_bytes, void* stream);

/* Popularity-ranked copy of a CSR (m rows, n <= 65536 columns), for
 * svdrec_cf_predict: every entry's column replaced by d_rank[column] and
 * every row reordered by rank (ranks distinct within a row).  One warp per
 * row: a shared-memory bitset over the n ranks gives each entry's position
 * (no sort; row-local writes).  Output has d_indptr's row structure. */
int svdrec_rank_rows(int64_t m, int32_t n, const int64_t* d_indptr, const int32_t* d_indices,
                     const double* d_values, const int32_t* d_rank, int32_t* d_out_indices,
                     double* d_out_values, void* stream);

/* The SpMM row-segment plan on the device (what the Python host's
 * segment_plan / warp_plan define, sparse.py).  seg_plan_count: per row
 * the exclusive scans d_first (first segment), d_sbase (first partial
 * slot of a split row), d_lidx (fix-up record of a split row), all m
 * int64, and d_totals = (segments, partial slots, split rows);
 * seg_plan_emit writes the arrays of svdrec_spmm's plan.  warp_plan: the
 * nwarp + 1 contiguous, cost-balanced range starts (cost = entries +
 * seg_cost per segment; seg_cost < 0: entries rounded up to whole 32-entry
 * chunks, at least one, plus -seg_cost -- what the chunk kernels execute);
 * d_scratch holds nseg + 1 int64. */
int svdrec_seg_plan_count(int64_t m, const int64_t* d_indptr, int32_t seg_max, int64_t* d_first,
                          int64_t* d_sbase, int64_t* d_lidx, int64_t* d_totals, void* stream);
int svdrec_seg_plan_emit(int64_t m, const int64_t* d_indptr, int32_t seg_max, const int64_t* d_first,
                         const int64_t* d_sbase, const int64_t* d_lidx, int32_t* d_seg_row,
                         int64_t* d_seg_begin, int64_t* d_seg_end, int32_t* d_seg_slot,
                         int32_t* d_long_row, int32_t* d_long_s0, int32_t* d_long_s1, void* stream);
int svdrec_warp_plan(int64_t nseg, const int64_t* d_seg_begin, const int64_t* d_seg_end, int64_t nwarp,
                     int32_t seg_cost, int64_t* d_scratch, int32_t* d_out, void* stream);
/* The pipelined SpMMs' chunk plan (linalg.py:141-158 has no counterpart:
 * scipy walks the CSR row by row).  chunk_plan: every segment cut into
 * chunks of <= 32 entries, one 16-B record each (int32 x 4: low word of the
 * first entry's offset; output row, or ~slot for a split row's partial;
 * entries | first-of-segment << 8 | last-of-segment << 9 | hot << 10; high
 * word of the offset).  d_cbase: nseg + 1 int64 (per segment its first
 * record; [nseg] = the record count); d_recs: room for nnz / 32 + 2 nseg
 * records.  With d_indptr / d_hot_cnt (the packed hot-first copy of
 * svdrec_spmm_hot_pack) a chunk is all hot or all cold (svdrec_spmm_hc);
 * both NULL for the plain plan.  warp_chunks: warp_chunk[w] = first record
 * of segment warp_seg[w] (nwarp + 1 int32). */
int svdrec_chunk_plan(int64_t nseg, const int32_t* d_seg_row, const int64_t* d_seg_begin,
                      const int64_t* d_seg_end, const int32_t* d_seg_slot, const int64_t* d_indptr,
                      const int32_t* d_hot_cnt, int64_t* d_cbase, void* d_recs, void* stream);
int svdrec_warp_chunks(int64_t nwarp, const int32_t* d_warp_seg, int64_t nseg, const int64_t* d_cbase,
                       int32_t* d_warp_chunk, void* stream);

/* Exclusive scan of n int64 values (d_in may equal d_out); the total goes
 * to d_total (nullable). */
int svdrec_scan_i64(int64_t n, const int64_t* d_in, int64_t* d_out, int64_t* d_total, void* stream);

/* Count samples whose (user, item) is stored in the CSR (ValidationMae's
 * disjointness check, cf.py:243-254); binary search per sample. */
int svdrec_count_overlap(int64_t nsamp, const int32_t* d_users, const int32_t* d_items,
                         const int64_t* d_indptr, const int32_t* d_indices,
                         int32_t* d_count, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SVDREC_B200_H */
