/*
 * tssvd.h -- C ABI of the B200 (sm_100a) implementation of the Gram-based
 * distributed SVD hot path of Li, Kluger & Tygert, arXiv 1612.08709
 * ("Algorithms for distributed computation of PCA and SVD").
 *
 * Citations: P:n = line n of the paper's LaTeX source.
 *
 * Conventions (all entry points)
 *   - Every matrix is FP64, ROW-MAJOR, with an explicit leading dimension
 *     (elements between consecutive rows).  A tall matrix is ROW-SHARDED:
 *     rank p of the communicator passes its contiguous block of rows A_p
 *     (m_local x n); the global matrix is the concatenation over ranks in rank
 *     order ("IndexedRowMatrix" partitions).
 *   - Pointers are CUDA DEVICE pointers on the communicator's device unless
 *     opts->host_io == 1, in which case A/Omega and U/sigma/V are HOST pointers
 *     (pinned memory recommended) and the library stages them through the
 *     workspace with cudaMemcpyAsync on `stream`.
 *   - `stream` is a cudaStream_t (passed as void* to keep this header free of
 *     CUDA types).  All work is enqueued on it and the call returns with the
 *     outputs complete.  The rank decisions ("Discard ..." steps) stay on the
 *     device: launches are sized by upper bounds and factor columns past a kept
 *     rank are zeros, so lowrank_svd() and tssvd() with n <= 32 make ONE host
 *     round trip (at the end, for the returned rank and the error flags).
 *     tssvd() with n > 32 also reads back the eigensolver's count and the first
 *     discard's rank (they size its dominant GEMMs): three round trips.
 *   - Multi-rank: every replicated decision (kept ranks) is checked across ranks
 *     by a max-allreduce; a rank that disagrees makes EVERY rank return
 *     TSSVD_ENCCL instead of issuing mismatched collectives.
 *   - The caller owns every buffer (workspace included); nothing is allocated
 *     inside tssvd() / lowrank_svd().  A and Omega are never written.
 *   - Errors: every entry point returns a tssvd_status; on failure
 *     tssvd_last_error() returns a thread-local detail string.  In a
 *     multi-rank job every rank returns the same status for argument errors
 *     that depend on global sizes.  Nothing throws across the ABI.
 */
#ifndef TSSVD_H_
#define TSSVD_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSSVD_ABI_VERSION 1

typedef enum {
  TSSVD_OK = 0,
  TSSVD_EINVAL = 1,     /* bad argument: sizes, leading dimensions, alignment, wp, l, k, iters */
  TSSVD_ENONFINITE = 2, /* NaN/Inf in A (or Omega): a non-finite diagonal of the first pass's
                           Gram matrix (also an overflowing column, |a|^2 > DBL_MAX) */
  TSSVD_ENOCONV = 3,    /* a Jacobi eigen/SVD core exceeded max_jacobi_sweeps */
  TSSVD_ECUDA = 4,      /* CUDA runtime error (detail in tssvd_last_error) */
  TSSVD_ENCCL = 5,      /* NCCL error */
  TSSVD_ENOMEM = 6      /* workspace_bytes smaller than *_workspace_size() */
} tssvd_status;

const char* tssvd_status_string(int status);
const char* tssvd_last_error(void);
int tssvd_abi_version(void);

/* ---- communicator -------------------------------------------------------
 * Opaque handle: an NCCL communicator plus rank/size/device.  A NULL comm
 * means a single-GPU job on the current device (no collectives). */
typedef struct tssvd_comm tssvd_comm;

/* Rank 0 creates the 128-byte unique id (host memory) and distributes it
 * out of band (e.g. a torch.distributed broadcast). */
int tssvd_get_unique_id(unsigned char id[128]);
/* Collective over `nranks` processes: ncclCommInitRank on `device`. */
int tssvd_comm_create(int nranks, int rank, const unsigned char id[128], int device,
                      tssvd_comm** out);
/* Borrow an existing NCCL communicator (an ncclComm_t, e.g. the one behind a
 * torch ProcessGroupNCCL: pg._get_backend(torch.device("cuda"))._comm_ptr()).
 * Rank, size and device are queried from NCCL.  The handle does not own the
 * communicator: tssvd_comm_destroy frees only the handle, the caller keeps
 * the communicator alive while the handle is in use.  Same NCCL library
 * required (the process's libnccl.so.2).  Errors: TSSVD_EINVAL for a NULL
 * communicator or out pointer, TSSVD_ENCCL when NCCL rejects the queries. */
int tssvd_comm_wrap_nccl(void* nccl_comm, tssvd_comm** out);
/* Frees the handle; destroys the NCCL communicator only if it was created by
 * tssvd_comm_create. */
int tssvd_comm_destroy(tssvd_comm* comm);
int tssvd_comm_rank(const tssvd_comm* comm, int* rank, int* nranks);
/* Sum-allreduce of `count` doubles in place on `stream` (exposed for tests). */
int tssvd_allreduce_sum(tssvd_comm* comm, void* stream, double* buf, int64_t count);

/* ---- options ------------------------------------------------------------ */
typedef struct {
  int abi_version;           /* must be TSSVD_ABI_VERSION */
  double working_precision;  /* wp in (0,1), default 1e-11 ("could be 10^-11") */
  int orthonormalizations;   /* tssvd: 1 = Algorithm 3, 2 = Algorithm 4 */
  int max_jacobi_sweeps;     /* cap per small core, e.g. 60; exceeded -> TSSVD_ENOCONV */
  int host_io;               /* 0: device pointers; 1: host pointers (see conventions);
                                2 (lowrank_svd only): host pointers and A is never resident --
                                every pass over A streams row chunks of ~256 MB through two
                                device staging buffers on a library-owned copy stream
                                (out-of-core; PCIe-bound; workspace without the m x n copy) */
} tssvd_opts;

/* Fills defaults: wp 1e-11, Algorithm 4, 60 sweeps, device pointers. */
void tssvd_opts_default(tssvd_opts* opts);

/* ---- problem {1}: thin SVD of a tall-skinny matrix ------------
 * A = U diag(sigma) V^T with U (m x r) and V (n x r) orthonormal columns,
 * sigma descending, r = kept rank after the "Discard" steps
 * (Alg. 3 step 5 / Alg. 4 steps 5 and 11: entries below max * sqrt(wp)).
 * Signs: each (u_j, v_j) is flipped so the largest-|.| entry of v_j is positive.
 *
 *   m_local  rows of this rank's shard (>= 0); m = sum over ranks must be >= n
 *   n        columns, 1 <= n <= 2048 (odd n allowed; n > 256 runs the wide core: the
 *            workspace then holds an m_local x n copy of Y~ and the eigen/SVD cores
 *            are the cooperative multi-CTA solvers)
 *   A        m_local x n, lda >= n, lda EVEN, 16-byte aligned (rows move as
 *            16-byte TMA granules); read-only
 *   U        m_local x n capacity, ldu >= n, ldu even, 16-byte aligned: columns
 *            [0, r) receive U_p (sharded like A); the rest is scratch.
 *            U may alias A (same pointer and ldu == lda): then A is overwritten.
 *            host_io == 1: U is a host buffer of m_local x n doubles; ldu >= n
 *            gives row-major U with that leading dimension, ldu == 0 returns U
 *            PACKED with leading dimension (r + 1) & ~1 (one contiguous D2H copy).
 *   sigma    n capacity, [0, r) written, replicated on every rank
 *   V        n x n capacity, ldv >= n: columns [0, r) written, replicated
 *   rank     HOST out: r (identical on every rank)
 *   workspace/workspace_bytes: device scratch of at least tssvd_workspace_size()
 */
int tssvd_workspace_size(const tssvd_comm* comm, int64_t m_local, int64_t n,
                         const tssvd_opts* opts, size_t* bytes);
int tssvd(tssvd_comm* comm, void* stream, int64_t m_local, int64_t n, const double* A,
          int64_t lda, const tssvd_opts* opts, double* U, int64_t ldu, double* sigma, double* V,
          int64_t ldv, int64_t* rank, void* workspace, size_t workspace_bytes);

/* ---- problem {2}: rank-l approximation, Algorithm 8 ----------
 * Algorithm 5 (subspace iteration) with Algorithm 3 in its steps 4
 * and 6 and Algorithm 4 in its last step, fed into Algorithm 6 (P:744-766,
 * whose SVD of B = Q^T A is Algorithm 4 applied to B^T).  Returns the leading
 * k <= l triplets with ||A - U diag(sigma) V^T||_2 ~ sigma_{k+1}.
 *
 *   n        columns of A, n > l (odd n allowed); A: lda >= n, lda EVEN, 16-byte aligned
 *   Omega    n x l start block Q~_0, ldo >= l; must be bit-identical
 *            on every rank (the caller seeds it)
 *   l, iters 0 < l < min(m, n), l <= 128; iters >= 0 (the paper's i)
 *   k        0 < k <= l
 *   U        m_local x k capacity (ldu >= k), sharded like A; device API: ldu EVEN
 *            and U 16-byte aligned (the GEMM epilogue stores 16-byte pairs),
 *            checked before any work is enqueued
 *   sigma    k capacity;  V  n x k capacity (ldv >= k), replicated
 *   rank     HOST out: min(k, kept rank); columns [rank, k) of U, V are zeros
 */
int lowrank_workspace_size(const tssvd_comm* comm, int64_t m_local, int64_t n, int64_t l,
                           const tssvd_opts* opts, size_t* bytes);
int lowrank_svd(tssvd_comm* comm, void* stream, int64_t m_local, int64_t n, const double* A,
                int64_t lda, const double* Omega, int64_t ldo, int64_t l, int iters, int64_t k,
                const tssvd_opts* opts, double* U, int64_t ldu, double* sigma, double* V,
                int64_t ldv, int64_t* rank, void* workspace, size_t workspace_bytes);

/* ---- problem {1} by Algorithms 1 / 2: randomized TSQR-based SVD --
 * B^* = A Omega^* (every row of A mixed by the random orthogonal Omega = D F S D~ F S~
 * of Remark 'randomness'), B^* = Q R by TSQR (Householder QR of row blocks,
 * the stacked R factors QR'd again; multi-rank: the ranks' R all-gathered and factored
 * identically on every rank), rows of R with |R_jj| < |R_11| wp discarded, SVD of R
 * (Alg. 2: of T = R R~ after a second TSQR of the kept Q~), U = Q U~, V = Omega^-1 V~.
 * Same conventions and outputs as tssvd() (signs: largest-|.| entry of v_j positive);
 * device pointers only (opts->host_io must be 0); opts->orthonormalizations 1 = Alg. 1,
 * 2 = Alg. 2.
 *
 *   n        1 <= n <= 128 (odd n: the last coordinate is left unmixed, R17)
 *   phases   DEVICE, 2 * (n / 2) doubles: [theta_D (h) ; theta_D~ (h)], h = n / 2,
 *            D = diag(exp(i theta)); bit-identical on every rank
 *   perms    DEVICE, 2 * (n / 2) ints: [S (h) ; S~ (h)], permutations of 0..h-1 with
 *            (S z)_k = z_{S[k]}; bit-identical on every rank
 *   (F is the unitary DFT of length h acting on the pairs (x_2k, x_2k+1) as complex numbers)
 */
int tsqr_svd_workspace_size(const tssvd_comm* comm, int64_t m_local, int64_t n, const tssvd_opts* opts,
                            size_t* bytes);
int tsqr_svd(tssvd_comm* comm, void* stream, int64_t m_local, int64_t n, const double* A, int64_t lda,
             const double* phases, const int* perms, const tssvd_opts* opts, double* U, int64_t ldu,
             double* sigma, double* V, int64_t ldv, int64_t* rank, void* workspace, size_t workspace_bytes);

/* ---- problem {2} by Algorithm 7 ---------------------------------
 * lowrank_svd() with Algorithm 1 in steps 4 and 6 of Alg. 5 and Algorithm 2 in its
 * last step and in Alg. 6.  Every factorization gets the random Omega of its width w
 * (w = l, or the kept rank of the factorization before it): row w - 1 of the tables
 *   phases   DEVICE, l x l doubles (ld l): row w - 1 = the 2 * (w / 2) phases for width w
 *   perms    DEVICE, l x l ints (ld l):    row w - 1 = the 2 * (w / 2) permutation entries
 * (layouts as tsqr_svd's).  Other arguments as lowrank_svd(); device pointers only.
 */
int lowrank_tsqr_workspace_size(const tssvd_comm* comm, int64_t m_local, int64_t n, int64_t l,
                                const tssvd_opts* opts, size_t* bytes);
int lowrank_svd_tsqr(tssvd_comm* comm, void* stream, int64_t m_local, int64_t n, const double* A,
                     int64_t lda, const double* Omega, int64_t ldo, int64_t l, int iters, int64_t k,
                     const double* phases, const int* perms, const tssvd_opts* opts, double* U, int64_t ldu,
                     double* sigma, double* V, int64_t ldv, int64_t* rank, void* workspace,
                     size_t workspace_bytes);

/* ---- problem {2}, Algorithm 8 with LU-based subspace tracking ---
 * lowrank_svd() with Alg. 5's intermediate steps 4 and 6 taking the L factor of Gaussian
 * elimination with partial (row) pivoting of Y_j / Y~_j instead of Alg. 3's orthonormal Q ("the
 * column space of L is the same as the column space of Q"); the last step (Alg. 4) and Alg. 6
 * unchanged.  Pivots: the largest |.| among the rows not yet chosen, ties to the lowest global
 * row (rank order); elimination stops at the first pivot with |pivot_j| <= |pivot_1| wp.  Every
 * pivot decision stays on the device (multi-rank: three small allreduces per column).  Arguments,
 * outputs and errors as lowrank_svd() (host_io 0 and 1).
 */
int lowrank_lu_workspace_size(const tssvd_comm* comm, int64_t m_local, int64_t n, int64_t l,
                              const tssvd_opts* opts, size_t* bytes);
int lowrank_svd_lu(tssvd_comm* comm, void* stream, int64_t m_local, int64_t n, const double* A,
                   int64_t lda, const double* Omega, int64_t ldo, int64_t l, int iters, int64_t k,
                   const tssvd_opts* opts, double* U, int64_t ldu, double* sigma, double* V,
                   int64_t ldv, int64_t* rank, void* workspace, size_t workspace_bytes);

/* ---- instrumentation ------------------------------------------------------
 * Per-call counters of the last tssvd()/lowrank_svd() on this thread:
 * kernel launches enqueued, Jacobi sweeps of each core, and the kept ranks. */
#define TSSVD_MAX_PASSES 48
typedef enum {
  TSSVD_PASS_GRAM_X = 1, /* B = X^T X            (Alg. 3/4 step 1)            */
  TSSVD_PASS_XV = 2,     /* Y~ = X V~ + norms    (Alg. 3/4 steps 3-4)         */
  TSSVD_PASS_GRAM_Y = 3, /* Z = Y^T Y            (Alg. 4 step 7)              */
  TSSVD_PASS_QNORM = 4,  /* norms of Q~ = Y W    (Alg. 4 steps 9-10)          */
  TSSVD_PASS_UOUT = 5,   /* U = Y~ M (in place)  (Alg. 3 step 6/Alg. 4 st 15) */
  TSSVD_PASS_ALPHA = 6,  /* Y = A Q~             (Alg. 5 steps 3, 8)          */
  TSSVD_PASS_BETA = 7,   /* A^T Q                (Alg. 5 step 5, Alg. 6 st 1) */
  TSSVD_PASS_JACOBI = 8, /* one-sided Jacobi core (eig / SVD)                 */
  TSSVD_PASS_TSQR = 9    /* TSQR, Q formed in place (Alg. 1/2 steps 2, 4)     */
} tssvd_pass_kind;
typedef struct {
  int64_t kernel_launches;
  int64_t a_passes;          /* streaming passes over A */
  int jacobi_sweeps[16];
  int n_jacobi;
  int64_t ranks[8];
  int n_ranks;
  /* filled only while tssvd_set_pass_timing(1): CUDA-event time of each
   * streaming pass / Jacobi core, its kind and its ALGORITHMIC flops and bytes */
  int n_pass;
  int pass_kind[TSSVD_MAX_PASSES];
  double pass_ms[TSSVD_MAX_PASSES];
  double pass_flops[TSSVD_MAX_PASSES];
  double pass_bytes[TSSVD_MAX_PASSES];
} tssvd_stats;
int tssvd_last_stats(tssvd_stats* out);
/* Enable (1) / disable (0) per-pass CUDA-event timing on this thread. */
int tssvd_set_pass_timing(int enable);

/* Low-level building blocks, exported for kernel-level parity tests and
 * benchmarks (device pointers, row-major, `stream` as above). */
/* G = X^T X (n x n, ldg) over the local rows only (Alg. 3 step 1 before aggregation). */
int tssvd_gram(void* stream, int64_t m, int64_t n, const double* X, int64_t ldx, double* G,
               int64_t ldg, void* workspace, size_t workspace_bytes);
size_t tssvd_gram_workspace(int64_t m, int64_t n);
/* Y = X M (m x c, ldy), M is k x c (ldm); optional column sums of squares nsq (c). */
int tssvd_matmul(void* stream, int64_t m, int64_t k, int64_t c, const double* X, int64_t ldx,
                 const double* M, int64_t ldm, double* Y, int64_t ldy, double* nsq,
                 void* workspace, size_t workspace_bytes);
size_t tssvd_matmul_workspace(int64_t m, int64_t k, int64_t c);
/* Z = X^T Y (n x l, ldz) over the local rows (Alg. 5 step 5 before aggregation). */
int tssvd_matmul_tn(void* stream, int64_t m, int64_t n, int64_t l, const double* X, int64_t ldx,
                    const double* Y, int64_t ldy, double* Z, int64_t ldz, void* workspace,
                    size_t workspace_bytes);
size_t tssvd_matmul_tn_workspace(int64_t m, int64_t n, int64_t l);
/* Eigendecomposition of a symmetric POSITIVE SEMIDEFINITE B (n x n, ldb; a
 * Gram matrix; 1 <= n <= 2048, else TSSVD_EINVAL; n > 256 runs the cooperative
 * multi-CTA solver) by one-sided Jacobi on its
 * columns: lambda[j] (descending) and the unit eigenvectors as ROWS of Vt
 * (n x n, ldv): Vt[j, :] = v_j.  (For an indefinite B, lambda holds |eigenvalues|.) */
int tssvd_sym_eig(void* stream, int64_t n, const double* B, int64_t ldb, double* lambda,
                  double* Vt, int64_t ldv, int max_sweeps, int* sweeps, void* workspace,
                  size_t workspace_bytes);
size_t tssvd_sym_eig_workspace(int64_t n);

/* Eigendecomposition of a symmetric PSD matrix by Householder tridiagonalisation and the
 * implicit QL iteration (one CTA; the solver tssvd() uses for Alg. 4 step 8, P:670-672,
 * "Calculate the eigendecomposition Z = W D W^*", where Z = Y^* Y is near the identity and
 * one-sided Jacobi converges only linearly).  Same layout and outputs as tssvd_sym_eig:
 * lambda[j] descending (values <= eps * max diag(B) returned as 0 with a zero row), row j of Vt
 * (ld ldv) = eigenvector j.  1 <= n <= 160.  *iterations (may be NULL) = QL iterations.
 * Workspace: tssvd_sym_eig_workspace(n) bytes.  Errors: TSSVD_EINVAL (n, ld), TSSVD_ENOMEM
 * (workspace), TSSVD_ENONFINITE (Inf/NaN in B), TSSVD_ENOCONV (an eigenvalue not deflated in
 * 30 QL iterations). */
int tssvd_sym_eig_ql(void* stream, int64_t n, const double* B, int64_t ldb, double* lambda,
                     double* Vt, int64_t ldv, int* iterations, void* workspace, size_t workspace_bytes);

/* Plan-only run (no GPU, no CUDA or NCCL call): the steps and collectives that
 * tssvd() (problem = 1; l, iters, k ignored), lowrank_svd() (2), tsqr_svd() (3),
 * lowrank_svd_tsqr() (4) or lowrank_svd_lu() (5) would
 * take on one of `nranks` ranks holding m_local rows, written to buf as
 * "token;token;..." (e.g. "gram:X;allreduce:gram:5050;eig:B;...").  Used by the
 * multi-rank CPU tests, whose replay of the distributed data flow is driven by
 * this trace of the real orchestrator.  TSSVD_ENOMEM if buf_len is too small. */
int tssvd_trace(int problem, int nranks, int64_t m_local, int64_t n, int64_t l, int iters, int64_t k,
                const tssvd_opts* opts, char* buf, size_t buf_len);

#ifdef __cplusplus
}
#endif
#endif /* TSSVD_H_ */
