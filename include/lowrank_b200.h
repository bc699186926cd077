/*
 * lowrank_b200.h -- C ABI of the B200-native SVT / rSVD hot path.
 *
 * Drop-in boundary for the reference package `lowrank`
 * (/root/reference/pkg/src/lowrank).  The reference is pure Python over
 * numpy/scipy/LAPACK, so its "FFI" is the set of module-global kernel calls
 * its algorithms make; each entry point below replaces one of them and cites
 * it.  The host mirror (paper_1810_06860_b200/) binds these through ctypes
 * and re-exposes the reference's own Python names and error behaviour.
 *
 * Conventions
 *   - every pointer is a DEVICE pointer unless the name ends in _host;
 *   - dense blocks are row-major fp64 with an explicit leading dimension
 *     (ld >= columns), matching the reference's C-contiguous arrays;
 *   - sparse patterns use int32 offsets/indices (all BASELINE configs have
 *     nnz < 2^31); the reference stores int64 (sparse.py:47-48);
 *   - `stream` is a cudaStream_t passed as void*; calls are stream-ordered
 *     and never synchronize unless documented;
 *   - no function allocates device memory on the hot path: scratch is
 *     passed in, sized by the *_workspace helpers;
 *   - return value: LR_OK or an lr_status code; lr_last_error() gives the
 *     message of the calling thread's last failure.
 */
#ifndef LOWRANK_B200_H
#define LOWRANK_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LR_OK = 0,
  LR_ERR_ARG = 1,    /* -> ValueError            */
  LR_ERR_RANK = 2,   /* -> RankDeficiencyError   */
  LR_ERR_NOCONV = 3, /* -> NumericalError        */
  LR_ERR_CUDA = 4,   /* -> RuntimeError          */
} lr_status;

int lr_version(void);
const char* lr_last_error(void);
int lr_sm_count(void);
/* Number of kernels this library has launched in the process (all streams). */
long long lr_launch_count(void);

/* ------------------------------------------------------------------ sparse */

/* Y[rows x w] = A * X  for a row-compressed pattern (CSR for Y*X, the CSC copy
 * for Y^T*X).  Replaces scipy csr_matvecs as called by `spmm`
 * (sparse.py:153-158) and by `spmm_t` (sparse.py:161-170, which re-gathers
 * A.data[perm] every call -- here the CSC values are a persistent copy).
 * items: optional (NULL -> one item per row) int4 {row, beg, end, slot}
 *   schedule splitting long rows; slot >= 0 writes a partial row into
 *   scratch[slot*w ...]; splits (int4 {row, slot_beg, slot_end, 0}) then sum
 *   partial rows in slot order (deterministic).  Rows are summed in stored
 *   order (scipy's sequential axpy order) within an item. */
int lr_spmm_f64(const int* ptr, const int* idx, const double* val, int rows,
                const int* items, int n_items, const int* splits, int n_splits,
                const double* X, long long ldx, int w, double* Y, long long ldy,
                double* scratch, void* stream);

/* The same product with shared-memory / TMA staging of the block rows a
 * skewed pattern gathers most (north_star (1): "shared-memory/TMA staging of
 * block rows"; replaces the same scipy csr_matvecs call, sparse.py:153-170).
 * idx_hot: the index stream with the hot_max most frequent indices (rank by
 * occurrence count) stored as -(rank + 1), every other entry as in idx;
 * hot_order[rank] = index.  Per column chunk the H most frequent rows of X
 * that fit shared memory are packed into hot_buf (>= lr_spmm_hot_buf_doubles()
 * doubles) and bulk-copied (cp.async.bulk + mbarrier) into every CTA's shared
 * memory; gathers of those rows never leave the SM.  Results are bit-identical
 * to lr_spmm_f64 (same chunks, lane map and summation order).  hot_max <=
 * lr_spmm_hot_rows_max(). */
int lr_spmm_hot_rows_max(void);
long long lr_spmm_hot_buf_doubles(void);
int lr_spmm_hot_f64(const int* ptr, const int* idx, const int* idx_hot, const int* hot_order, int hot_max,
                    double* hot_buf, long long hot_buf_doubles, const double* val, int rows, const int* items,
                    int n_items, const int* splits, int n_splits, const double* X, long long ldx, int w, double* Y,
                    long long ldy, double* scratch, void* stream);

/* fp32 mode (north_star: "optional fp32 path", singular values within 1e-4):
 * the same SpMM over fp32 values and fp32 dense blocks (float2 per lane and
 * column pair: half the gathered bytes of the fp64 kernel), w >= 2.  The
 * dense linear algebra of the fp32 mode stays fp64 (rsvd.py converts the
 * product blocks with lr_convert_*). */
int lr_spmm_f32(const int* ptr, const int* idx, const float* val, int rows, const int* items, int n_items,
                const int* splits, int n_splits, const float* X, long long ldx, int w, float* Y, long long ldy,
                float* scratch, void* stream);

/* x_e = sum_t U[i,t]*S[t]*V[j,t] for every stored (i,j), CSR order.
 * Replaces `project_pattern` / `_project_entries` (sparse.py:173-191). */
int lr_sddmm_f64(const int* ptr, const int* idx, int rows, const int* items, int n_items,
                 const double* U, long long ldu, const double* S, const double* V, long long ldv,
                 int r, double* x, void* stream);

/* The fused SVT step of completion.py:373-386 in one pass over the pattern:
 *   x_e   = sum_t U[i,t]*S[t]*V[j,t]           (project_pattern)
 *   d_e   = x_e - m_e;  partial sums of d_e^2   (frobenius(x - m), sparse.py:219-228)
 *   if apply: y_e += step*(m_e - x_e) in the CSR copy and, through inv_perm,
 *             in the CSC copy                   (update_pattern_values, sparse.py:205-216)
 * r == 0 is legal (x = 0).  Writes n_blocks partial (sum d^2, max|d|) pairs to
 * partial[]; lr_svt_step_finish reduces them in fixed order into out2[0..1]. */
int lr_svt_step_f64(const int* ptr, const int* idx, int rows, const int* items, int n_items,
                    const double* U, long long ldu, const double* S, const double* V, long long ldv,
                    int r, const double* m_vals, double* y_csr, double* y_csc, const int* inv_perm,
                    double step, int apply, double* partial, int n_partial, double* out2, void* stream);
int lr_svt_step_partials(void);

/* Flat form of the two entry points above (the default product path): the
 * stored entries are cut into tiles of lr_svt_tile_entries() consecutive CSR
 * slots, one warp per tile, whatever the row lengths.  tile_row[t] = the row
 * holding slot t * lr_svt_tile_entries() (lr_svt_tile_rows_i32, once per
 * pattern; lr_svt_tile_count(nnz) ints).  Same results as lr_svt_step_f64 /
 * lr_sddmm_f64 (each entry's sum depends only on its U row, S and V row);
 * y_csc may be NULL: only the CSR copy is updated (the caller refreshes the
 * CSC copy with lr_gather_f64 before it is next read).  partial[] must hold
 * lr_svt_flat_partials() doubles.  Any rank (r > 256 runs in column chunks). */
int lr_svt_tile_entries(void);
long long lr_svt_tile_count(long long nnz);
int lr_svt_tile_rows_i32(const int* ptr, int m, long long nnz, int* tile_row, void* stream);
int lr_svt_flat_partials(void);
int lr_svt_step_flat_f64(const int* ptr, const int* idx, int m, long long nnz, const int* tile_row,
                         const double* U, long long ldu, const double* S, const double* V, long long ldv, int r,
                         const double* m_vals, double* y_csr, double* y_csc, const int* inv_perm, double step,
                         int apply, double* partial, int n_partial, double* out2, void* stream);
int lr_sddmm_flat_f64(const int* ptr, const int* idx, int m, long long nnz, const int* tile_row, const double* U,
                      long long ldu, const double* S, const double* V, long long ldv, int r, double* x,
                      void* stream);

/* y_csr += delta; y_csc[inv_perm[e]] += delta[e]  (update_pattern_values). */
int lr_pattern_axpy_f64(double* y_csr, double* y_csc, const int* inv_perm, const double* delta,
                        double alpha, long long nnz, void* stream);
/* dst[t] = src[perm[t]] : builds/refreshes the CSC value copy. */
int lr_gather_f64(const double* src, const int* perm, double* dst, long long n, void* stream);

/* CSR -> CSC transpose index of a pattern on the device (the reference's
 * SparseMatrix._transpose_index, sparse.py:129-139: stable argsort of the
 * column indices): t_ptr (n+1), t_idx = CSR row of each CSC slot (nnz),
 * perm = CSR slot of each CSC slot, inv_perm = its inverse.  Bit-exact with a
 * stable host argsort.  work: lr_csr_transpose_workspace_ints(m, n) ints. */
long long lr_csr_transpose_workspace_ints(int m, int n);
int lr_csr_transpose_i32(int m, int n, long long nnz, const int* ptr, const int* idx, int* t_ptr,
                         int* t_idx, int* perm, int* inv_perm, int* work, long long work_ints,
                         void* stream);

/* ----------------------------------------------------------- reductions */
/* out[0] = sum x^2, out[1] = max |x|, out[2] = #non-finite  over an
 * rows x cols block (ld); deterministic fixed-order tree.  Backs
 * `frobenius` (sparse.py:219-228) and the finiteness checks of
 * linalg._check_matrix (linalg.py:78-84). */
int lr_block_stats_f64(const double* X, long long rows, long long cols, long long ld,
                       double* partial, double* out3, void* stream);
int lr_stats_partials(void);
/* out[0] = sum_i x_i*y_i (deterministic). */
int lr_dot_f64(const double* x, const double* y, long long n, double* partial, double* out,
               void* stream);
/* Power-iteration helper for spectral_norm_est (sparse.py:231-256):
 * given z (n) and the current x (n): lam = x.z, zn = ||z||; if not done:
 * prev=curr, curr=sqrt(max(lam,0)); x = z/zn; done when |curr-prev| <=
 * tol*max(curr,1e-300) or zn == 0.  state = {prev, curr, done, iters, zero}. */
int lr_power_update_f64(double* x, const double* z, long long n, double tol, double* state,
                        double* partial, void* stream);

/* ---------------------------------------------------------------- dense */
enum {
  LR_GEMM_B_UPPER = 1,    /* B is upper triangular (K == N): skip zero blocks   */
  LR_GEMM_SYRK_UPPER = 2, /* transA, A == B: compute upper tiles, mirror (exactly symmetric) */
};
/* C[MxN] = alpha*op(A)*B + beta*C on fp64 tensor cores (mma.sync f64 ->
 * DMMA.8x8x4).  transA=0: A is MxK; transA=1: A is KxM (C = A^T B, split-K
 * over the long K with a fixed-order partial reduction).  Replaces the BLAS
 * dsyrk/dgemm calls of eig_svd (linalg.py:189,200), the lift products
 * (rsvd.py:195,229; completion.py:217,243) and qb_error (rsvd.py:252). */
long long lr_gemm_workspace_doubles(int transA, int M, int N, int K, int flags);
int lr_gemm_f64(int transA, int M, int N, int K, double alpha, const double* A, long long lda,
                const double* B, long long ldb, double beta, double* C, long long ldc, int flags,
                double* work, long long work_doubles, void* stream);

/* Upper Cholesky A = R^T R (n x n, in place; upper triangle of A receives R,
 * lower triangle zeroed) and R^{-1} (upper, into Rinv).  info_host receives 0
 * or 1 + the first non-positive pivot column (synchronizes). Building block of
 * the CholeskyQR2 / shifted CholeskyQR3 replacement of the Householder QR in
 * `orth` (linalg.py:101-124). shift is added to the diagonal first. */
long long lr_potrf_workspace_doubles(int n);
int lr_potrf_inv_f64(int n, double* A, long long lda, double shift, double* Rinv, long long ldr,
                     double* work, int* info_host, void* stream);
/* Asynchronous variant: info (0, or the 1-based failing column) to device
 * memory *info_dev, no host synchronisation. */
int lr_potrf_inv_async_f64(int n, double* A, long long lda, double shift, double* Rinv, long long ldr,
                           double* work, int* info_dev, void* stream);

/* Partial-pivoting LU of a tall m x n block (m >= n), in place, returning
 * P^T L like scipy.linalg.lu(X, permute_l=True) as used by `lu_pl`
 * (linalg.py:127-150): pivot = first max |x| of the remaining rows, unit
 * entry at the pivot row, zeros to its right, multipliers elsewhere.
 * status_host[0] = -1 on success, else the first column whose |pivot| <
 * 1e-14*max|X| (pivot value in status_host[1], tolerance in status_host[2]),
 * -2 for a zero matrix, -3 for non-finite input. Synchronizes. */
long long lr_lu_workspace_doubles(int m, int n);
int lr_lu_pl_f64(int m, int n, double* X, long long ldx, double* work, double* status_host,
                 void* stream);
/* Asynchronous variant (no host synchronisation): {code, pivot, tol} go to
 * device memory status_dev[0..2] with the codes above (-1 ok, -2 zero
 * matrix, -3 non-finite, j >= 0 zero pivot at column j); the caller checks
 * several calls' statuses with one read (rsvd.py's speculative BKI). */
int lr_lu_pl_async_f64(int m, int n, double* X, long long ldx, double* work, double* status_dev, void* stream);

/* Symmetric eigendecomposition by parallel (block-)Jacobi: eigenvalues
 * ascending in d, orthonormal eigenvectors in V (n x n, ldv).  A (n x n) is
 * overwritten.  Replaces LAPACK dsyevd behind `sym_eig` (linalg.py:153-169).
 * sweeps_host receives the sweep count; LR_ERR_NOCONV after max_sweeps. */
long long lr_syevj_workspace_doubles(int n);
int lr_syevj_f64(int n, double* A, long long lda, double* d, double* V, long long ldv,
                 int max_sweeps, double* work, int* sweeps_host, void* stream);

/* Symmetric eigendecomposition by Householder tridiagonalization (cooperative
 * kernel, rows in shared memory), multisection bisection and inverse
 * iteration (+ MGS inside clusters closer than 1e-8*||A||), then the
 * back-transform.  Eigenvalues ascending in d, eigenvectors in V; A is not
 * modified.  LAPACK-level accuracy (absolute eps*||A||), the default solver
 * behind sym_eig / eig_svd (linalg.py:153-202).  Clusters are found on the
 * device; the call is asynchronous unless clusters_host is non-NULL, in which
 * case it synchronizes the stream and stores the number of re-orthonormalised
 * clusters there. */
long long lr_syevd_workspace_doubles(int n);
int lr_syevd_f64(int n, const double* A, long long lda, double* d, double* V, long long ldv, double* work,
                 int* clusters_host, void* stream);

/* Sign rule of linalg._fix_signs (linalg.py:87-98): flip column j of V (and
 * of U if non-NULL) so V's first nonzero entry in column j is >= 0. */
int lr_fix_signs_f64(double* V, long long ldv, int rows_v, int cols, double* U, long long ldu,
                     int rows_u, void* stream);
/* S[i] = sqrt(max(d[i], 0)): singular values of ascending Gram eigenvalues
 * (linalg.py:196), on the device so eig_svd's lift is queued before the host
 * reads d for the rank checks. */
int lr_gram_spectrum_f64(const double* d, int n, double* S, void* stream);
/* fp32 mode's eigSVD Gram (linalg.py:189, A.T @ A) on the tcgen05 tensor
 * cores: G (n x n, fp64, exactly symmetric) = A^T A of the fp32 block A
 * (K x n, row-major, lda >= n) as 3xTF32 (a = hi + lo, hi.hi + hi.lo +
 * lo.hi) with fp32 TMEM accumulation over chunks of <= 4096 rows and a
 * fixed-order fp64 sum of the chunk partials (deterministic).  work: at least
 * lr_gram_tf32x3_workspace_floats(K, n) floats of device memory. */
long long lr_gram_tf32x3_workspace_floats(int K, int n);
int lr_gram_tf32x3(const float* A, long long lda, int K, int n, double* G, long long ldg, float* work,
                   long long work_floats, void* stream);
/* B[:, j] = V[:, idx_j] * scale_j with scale_j = sgn/S[idx_j]; column gather
 * used by eig_svd's U = A (V / S) for a selected window (linalg.py:199-201). */
int lr_scale_columns_f64(const double* V, long long ldv, int rows, const int* cols_idx, int ncols,
                         const double* S, int invert, double* B, long long ldb, void* stream);

/* ----------------------------------------------------------- COO -> CSR */
/* Coordinate triples (int64 rows/cols, count entries; with split != NULL only
 * the entries tagged `tag`) -> CSR on the device: SparseMatrix.from_coo
 * (sparse.py:84-104; ObservationSet.train_matrix, :259-328).  ptr (m+1),
 * col_out / src_out (int32: column, source index, in CSR order), vals_out
 * (values gathered in CSR order, may be NULL).  Bit-exact with the host
 * lexsort.  status_host[0]: 0 ok, 1 a row / 3 a column out of range, 2 a
 * non-finite value; [1] the CSR slot of the first duplicate cell (-1: none);
 * [2] nnz.  Synchronizes the stream (twice). */
long long lr_coo_to_csr_workspace_ints(int m, long long count);
int lr_coo_to_csr_i32(int m, int n, long long count, const long long* rows, const long long* cols,
                      const unsigned char* split, int tag, const double* vals, int* ptr, int* col_out, int* src_out,
                      double* vals_out, int* work, long long work_ints, int* status_host, void* stream);

/* One-sided Jacobi sweep for the dense SVD fallback (oracle_svd ->
 * dgesdd, linalg.py:205-221): the columns of B are the rows of Bt (n x m),
 * the columns of V the rows of Vt (n x n).  Every column pair (one
 * round-robin sweep, N-1 launches) with |<b_p, b_q>| > tol |b_p| |b_q| is
 * rotated orthogonal, the rotation applied to Vt too, except pairs whose
 * squared norms are both below noise2 (0: none skipped); off[0] (device) =
 * the largest measure rotated (0: converged).  Deterministic. */
int lr_jacobi_sweep_f64(int n, int m, double* Bt, long long ldb, double* Vt, long long ldv, double tol,
                        double noise2, double* off, void* stream);
/* out[i] = ||row i of Bt||_2 (scaled, no overflow), n rows of length m. */
int lr_row_norms_f64(const double* Bt, long long ldb, int n, int m, double* out, void* stream);

/* --------------------------------------------------------------- random */
/* Omega (rows x cols, row-major, ldo) = gaussian_matrix(RngState(seed), rows,
 * cols) of rng.py:77-94 on the device: numpy Philox4x64-10 (key = seed,
 * counter starting at 1), uniforms (x >> 11) * 2^-53, Box-Muller pairs over
 * the whole request, column-major fill.  Uniform stream bit-exact with numpy;
 * normals within a few ulp (log/sincos rounding). */
int lr_gaussian_f64(unsigned long long seed, int rows, int cols, double* omega, long long ldo,
                    void* stream);

/* The parity Omega assembled on the device from host-computed halves
 * (rng.py:38-55's Box-Muller, split as rng.Superset splits it): R[i] =
 * sqrt(-2 log(1 - u[i])) and cs[2j], cs[2j+1] = cos / sin(2 pi u[p_lo + j])
 * computed on the host with numpy's own log and libm's cos / sin and uploaded
 * once for a range of widths; for the width whose pair count is P = ceil(rows
 * cols / 2), off = P - p_lo and z[2i] = R[i] cs[2 (off + i)], z[2i+1] = R[i]
 * cs[2 (off + i) + 1] fill Omega (rows x cols, row-major, ldo) column-major:
 * one IEEE multiply per entry, so bit-identical to the host draw. */
int lr_omega_assemble_f64(const double* R, const double* cs, long long off, int rows, int cols, double* omega,
                          long long ldo, void* stream);

/* Host functions (no device work): the C pieces of the parity Omega's host
 * draw (rng.py:38-55 of the reference).  lr_host_uniforms: out[i] = uniform
 * start + i of numpy's Philox(key=seed) stream ((x >> 11) 2^-53).
 * lr_host_box_muller: z[2i] = sqrt(-2 logs[i]) cos(2 pi u2[i]),
 * z[2i+1] = ... sin(...), logs[i] = log(1 - u[i]) computed by numpy. */
void lr_host_uniforms(unsigned long long seed, long long start, long long count, double* out);
void lr_host_box_muller(const double* logs, const double* u2, long long n, double* z);
/* The same draw split for several widths at once (rng.Superset): cs[2j] =
 * cos(2 pi u[j]), cs[2j+1] = sin(...) over a run of stream positions, and
 * z[2i] = R[i] cs[2i], z[2i+1] = R[i] cs[2i+1] with R[i] = sqrt(-2 log(1 - u[i])). */
void lr_host_cossin(const double* u, long long n, double* cs);
void lr_host_bm_assemble(const double* R, const double* cs, long long n, double* z);

/* ------------------------------------------------------------- utilities */
int lr_copy2d_f64(const double* src, long long lds, double* dst, long long ldd, long long rows,
                  long long cols, int reverse_cols, void* stream);
/* Precision conversion of strided row-major blocks (round to nearest). */
int lr_convert_f64_to_f32(const double* src, long long lds, float* dst, long long ldd, long long rows,
                          long long cols, void* stream);
int lr_convert_f32_to_f64(const float* src, long long lds, double* dst, long long ldd, long long rows,
                          long long cols, void* stream);
int lr_fill_f64(double* dst, long long ld, long long rows, long long cols, double v, void* stream);
/* dst (cols x rows) = src^T */
int lr_transpose_f64(const double* src, long long lds, long long rows, long long cols, double* dst,
                     long long ldd, void* stream);
/* dst = (src + src^T) / 2 : the symmetrization of sym_eig (linalg.py:165) */
int lr_symmetrize_f64(const double* src, long long lds, int n, double* dst, long long ldd, void* stream);
/* d[i] = A[i][i] */
int lr_diag_f64(const double* A, long long lda, int n, double* d, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LOWRANK_B200_H */
