// Internal launcher declarations (not part of the C ABI; see include/tssvd.h).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace tsk {

struct DevInfo {
  int sms = 148;
  size_t smem_optin = 227 * 1024;
};
const DevInfo& dev_info();

// ---- streaming passes over tall row-major matrices (stream_kernels.cu) ----
// Partial Gram (lower triangle) of X[:, :w] over `grid` contiguous row ranges:
// part[p][i*wp + j] (i >= j), wp = pad8(w).  Returns the number of partials.
int syrk_partials_grid(int64_t m, int w);
size_t syrk_partials_doubles(int64_t m, int w);
cudaError_t launch_syrk(const double* X, int64_t ldx, int64_t m, int w, double* part,
                        cudaStream_t s);
// B = sum_p part[p]  (lower), written symmetric into B (ldb); optionally also the
// packed lower triangle (w(w+1)/2, row-major) for a half-size allreduce.
cudaError_t launch_reduce_sym(const double* part, int nparts, int w, double* B, int ldb,
                              double* packed, cudaStream_t s);

// Y[:, :c] = X[:, :k] * M  (M row-major, ld = smem_ld(c), rows padded to mult. of 32
// with zeros; c <= 256).  Optional column sums of squares partials
// norm_part[g][gemm_nn_part_stride(c)].
// In place (Y == X, ldy == ldx) is allowed.
int gemm_nn_grid(int64_t m, int c);
int gemm_nn_part_stride(int c);  // doubles per CTA in norm_part (>= pad8(c))
// scratch (nullable): gemm_nn_scratch_doubles(m, k, c) doubles enable the stream-K work split
// (used only without norm_part; a null scratch runs the row-tile split).
cudaError_t launch_gemm_nn(const double* X, int64_t ldx, int64_t m, int k, const double* M,
                           int c, double* Y, int64_t ldy, double* norm_part, double* scratch,
                           cudaStream_t s);
size_t gemm_nn_m_doubles(int k, int c);  // size of the padded M buffer
size_t gemm_nn_scratch_doubles(int64_t m, int k, int c);
size_t gemm_nn_scratch_max(int k, int c);  // stream-K records for any m (0 if K has one chunk)

// Z (n x l, ld ldz) partials: Zp[split][n_pad x ldz] = X[rows, :n]^T * Y[rows, :l]
// reduced over `splits` row ranges.
struct TnPlan {
  int cb, mi, nbl, xr, colblocks, splits, kr, nst, ldz;  // xr: remainder columns on the FMA pipe
  int64_t rows_per_split;
  size_t part_doubles;
};
TnPlan plan_gemm_tn(int64_t m, int n, int l);
cudaError_t launch_gemm_tn(const TnPlan& p, const double* X, int64_t ldx, int64_t m, int n,
                           const double* Y, int64_t ldy, int l, double* part, cudaStream_t s);
// out[e] = sum_p part[p*stride + e] for e < len (fixed two-level order)
cudaError_t launch_reduce_parts(const double* part, int nparts, int64_t stride, int64_t len,
                                double* out, cudaStream_t s);
// out[row*ldo + col] = sum_p part[p*stride + row*ldi + col], col < cols (zeros up to ldo
// when zero_pad)
cudaError_t launch_reduce_parts_2d(const double* part, int nparts, int64_t stride, int64_t rows,
                                   int ldi, int cols, double* out, int ldo, bool zero_pad, cudaStream_t s,
                                   bool accumulate = false);  // accumulate: out += the sum

// ---- one-sided Jacobi (jacobi.cu) ----
// EIG: B (n x n, ldb, symmetric PSD) -> k <= n eigenpairs: vals[j] descending,
// eigenvector j (unit) contiguous at vecs + j*ldv.  Pivoted-Cholesky
// preconditioned; pivots <= trunc * max(diag B) are dropped (k = info[2]).
// info = {sweeps, converged, k, -, -, rounds, nonfinite}: a non-finite diagonal
// entry (Inf/NaN in the streamed matrix) gives k = 0 and info[6] = 1.  vecs may alias B.
cudaError_t launch_jacobi_eig(const double* B, int ldb, int n, double tol, double trunc,
                              int max_sweeps, double* vecs, int ldv, double* vals, int* info,
                              cudaStream_t s);
// SVD of K given by N columns of length ldot (column j contiguous at cols + j*ldc):
// K J = P diag(vals), vals descending.  Output column r (ld ldout >= ldot + N):
// [P(:, r) unit (ldot) ; J(:, r) (N)].  info = {sweeps, converged, N}.
cudaError_t launch_jacobi_svd(const double* cols, int ldc, int N, int ldot, double tol,
                              int max_sweeps, double* out, int ldout, double* vals, int* info,
                              cudaStream_t s);

// ---- tridiagonal QL eigensolver (tridiag_eig.cu): Alg. 4 step 8 on Z = Y^* Y ~ I ----
// Same contract and info layout as launch_jacobi_eig (info[0] = QL iterations, info[5] =
// rotations); n <= kTridiagMax (one CTA, the matrix in shared memory).
constexpr int kTridiagMax = 160;
cudaError_t launch_tridiag_eig(const double* B, int ldb, int n, double trunc, double* vecs, int ldv, double* vals,
                               int* info, cudaStream_t s);

// ---- wide cores, 256 < n <= 2048 (jacobi_wide.cu): cooperative multi-CTA solvers ----
// Same contracts as launch_jacobi_eig / launch_jacobi_svd, plus a device workspace of
// jacobi_wide_workspace(n, L) doubles (n = order / max(N, dot), L = rows per column).
size_t jacobi_wide_workspace(int n, int L);
cudaError_t launch_jacobi_eig_wide(const double* B, int ldb, int n, double tol, double trunc, int max_sweeps,
                                   double* vecs, int ldv, double* vals, int* info, double* work,
                                   cudaStream_t s);
cudaError_t launch_jacobi_svd_wide(const double* cols, int ldc, int N, int dot, double tol, int max_sweeps,
                                   double* out, int ldout, double* vals, int* info, double* work,
                                   cudaStream_t s);

// ---- Algorithms 1 / 2 (tsqr.cu), n <= 128 ----
// Omega^T (wb x wb, ld ldm; row i = Omega e_i) for width *wdev (device, draws at row w-1 of the
// tables, ld ldp) or wconst (wdev null: the draws at phases / perms); zero past the width.
cudaError_t launch_mix_matrix(const double* phases, const int* perms, int ldp, const int* wdev, int wconst, int wb,
                              double* M, int ldm, cudaStream_t s);
// TSQR in place: X (rows x n, ldx) <- Q, R (n x n, row-major) to R_out; work: tsqr_workspace_doubles.
int tsqr_block_rows(int n);
size_t tsqr_workspace_doubles(int64_t rows, int n);
cudaError_t launch_tsqr(double* X, int64_t ldx, int64_t rows, int n, double* R_out, double* work, cudaStream_t s);
cudaError_t launch_r_discard(double* R, int w, double wp, int* slot, int* mask, cudaStream_t s);
cudaError_t launch_zero_cols(double* X, int64_t ldx, int64_t m, int w, const int* mask, cudaStream_t s);
cudaError_t launch_tri_mul(const double* R2, const double* R1, int w, double* T, cudaStream_t s);
cudaError_t launch_tsqr_out(const double* svo, int w, const double* vals, const double* M0, const int* rr,
                            double* sigma, double* V, int64_t ldv, double* Mg, int ldm, cudaStream_t s);

// ---- LU-based subspace tracking (lu_track.cu) ----
struct LuWork {
  void* rec;
  unsigned char* chosen;
  double* pval;
  long long* pidx;
  double* urow;
  double* gbuf;  // [0]: the column's max |.| (MAX-allreduced across ranks)
  double* lbuf;  // [0]: this rank's max
  int* obuf;     // [0]: owning rank candidate (MIN-allreduced)
};
size_t lu_workspace_bytes(int64_t rows, int w);
LuWork lu_carve(void* ws, int64_t rows, int w);
cudaError_t lu_init(const LuWork& lw, int64_t rows, cudaStream_t s);
cudaError_t lu_colmax(const LuWork& lw, const double* Y, int64_t ldy, int64_t rows, int j, cudaStream_t s);
cudaError_t lu_owner(const LuWork& lw, int rank, cudaStream_t s);
cudaError_t lu_decide(const LuWork& lw, const double* Y, int64_t ldy, int w, int j, const int* wdev, double wp,
                      int rank, cudaStream_t s);
cudaError_t lu_update(const LuWork& lw, double* Y, int64_t ldy, int64_t rows, int w, int j, cudaStream_t s);
cudaError_t lu_finish(const LuWork& lw, double* Y, int64_t ldy, int64_t rows, int w, int* slot, cudaStream_t s);
cudaError_t lu_fused(const LuWork& lw, double* Y, int64_t ldy, int64_t rows, int w, const int* wdev, double wp,
                     int* slot, cudaStream_t s);

}  // namespace tsk
