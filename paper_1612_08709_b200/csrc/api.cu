// Host orchestrator and C ABI (include/tssvd.h).
//
// Sequences the paper's Algorithms 3, 4 (tall-skinny SVD), 5, 6 and 8
// (low-rank SVD) over the sm_100a kernels, with NCCL sum-allreduces of the
// small per-rank partials (Gram matrices, column sums of squares, A^T Q).
// Every arithmetic step runs on the device; the host only sequences launches
// and reads back the kept ranks (the "Discard" decisions).
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/tssvd.h"
#include "common.cuh"
#include "kernels.h"
#include "small_kernels.h"

struct tssvd_comm {
  ncclComm_t nccl = nullptr;
  int rank = 0, nranks = 1, device = 0;
  bool owned = true;  // false: borrowed through tssvd_comm_wrap_nccl
};

namespace {

using namespace tsk;

thread_local std::string g_err;
thread_local tssvd_stats g_stats;
thread_local bool g_timing = false;

struct Fail {
  int code;
};

[[noreturn]] void fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  throw Fail{code};
}

#define CU(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) fail(TSSVD_ECUDA, "%s: %s (%s:%d)", #x, cudaGetErrorString(e_),     \
                                __FILE__, __LINE__);                                           \
  } while (0)
#define NC(x)                                                                                  \
  do {                                                                                         \
    ncclResult_t e_ = (x);                                                                     \
    if (e_ != ncclSuccess) fail(TSSVD_ENCCL, "%s: %s", #x, ncclGetErrorString(e_));            \
  } while (0)
#define KL(x)                                                                                  \
  do {                                                                                         \
    CU(x);                                                                                     \
    ++g_stats.kernel_launches;                                                                 \
  } while (0)
#define KS(x)                                                                                  \
  do {                                                                                         \
    x;                                                                                         \
    CU(cudaGetLastError());                                                                    \
    ++g_stats.kernel_launches;                                                                 \
  } while (0)

template <class F>
int guarded(F&& f) {
  try {
    f();
    return TSSVD_OK;
  } catch (const Fail& e) {
    return e.code;
  } catch (...) {
    g_err = "unexpected C++ exception";
    return TSSVD_ECUDA;
  }
}

// Bump allocator over the caller's workspace; dry mode only measures.
struct Arena {
  char* base = nullptr;
  size_t cap = 0, off = 0;
  bool dry = true;
  template <class T>
  T* get(size_t count) {
    off = (off + 255) & ~size_t(255);
    T* p = dry ? nullptr : reinterpret_cast<T*>(base + off);
    off += std::max<size_t>(count, 1) * sizeof(T);
    if (!dry && off > cap)
      fail(TSSVD_ENOMEM, "workspace too small (%zu bytes given, more needed)", cap);
    return p;
  }
};

int* pinned_ints() {
  static thread_local int* p = nullptr;
  if (!p) CU(cudaHostAlloc(reinterpret_cast<void**>(&p), 16 * sizeof(int), cudaHostAllocDefault));
  return p;
}

struct Ctx {
  tssvd_comm* comm = nullptr;
  cudaStream_t s = nullptr;
  double wp = 1e-11;
  int max_sweeps = 60;
  // Jacobi solves whose convergence is checked after the call's final sync
  // (no host round trip per solve): device info slots of 8 ints each
  int* jinfo = nullptr;
  int njinfo = 0;
  static constexpr int kMaxDeferred = 48;
  bool dist() const { return comm && comm->nranks > 1; }
  int* next_info() {
    if (njinfo >= kMaxDeferred) fail(TSSVD_ECUDA, "too many deferred Jacobi solves");
    return jinfo + 8 * njinfo++;
  }
};

void allreduce(Ctx& c, double* buf, int64_t count) {
  if (!c.dist() || count <= 0) return;
  NC(ncclAllReduce(buf, buf, (size_t)count, ncclDouble, ncclSum, c.comm->nccl, c.s));
}

void read_ints(Ctx& c, const int* dev, int n, int* host) {
  int* h = pinned_ints();
  CU(cudaMemcpyAsync(h, dev, n * sizeof(int), cudaMemcpyDeviceToHost, c.s));
  CU(cudaStreamSynchronize(c.s));
  std::memcpy(host, h, n * sizeof(int));
}

// Per-pass CUDA-event timing (tssvd_set_pass_timing): events recorded on the
// call's stream around each streaming kernel, resolved after the final sync.
struct PassTimer {
  cudaEvent_t ev[2 * TSSVD_MAX_PASSES] = {};
  int open = -1;
  cudaStream_t s = nullptr;
  void begin(cudaStream_t st, int kind, double flops, double bytes) {
    if (!g_timing || g_stats.n_pass >= TSSVD_MAX_PASSES) return;
    const int i = g_stats.n_pass;
    for (int q = 0; q < 2; ++q)
      if (!ev[2 * i + q]) CU(cudaEventCreate(&ev[2 * i + q]));
    g_stats.pass_kind[i] = kind;
    g_stats.pass_flops[i] = flops;
    g_stats.pass_bytes[i] = bytes;
    CU(cudaEventRecord(ev[2 * i], st));
    open = i;
    s = st;
  }
  void end() {
    if (open < 0) return;
    cudaEventRecord(ev[2 * open + 1], s);  // no throw: runs in a destructor
    g_stats.n_pass = open + 1;
    open = -1;
  }
  void resolve() {
    for (int i = 0; i < g_stats.n_pass; ++i) {
      float ms = 0.f;
      CU(cudaEventElapsedTime(&ms, ev[2 * i], ev[2 * i + 1]));
      g_stats.pass_ms[i] = ms;
    }
  }
};
thread_local PassTimer g_timer;

struct Pass {
  Pass(cudaStream_t s, int kind, double flops, double bytes) { g_timer.begin(s, kind, flops, bytes); }
  ~Pass() { g_timer.end(); }
};

inline int mrows_for(int k) { return (int)(gemm_nn_m_doubles(k, 1) / smem_ld(1)); }

// ---------------------------------------------------------------- core ----
// Buffers of one Alg. 3/4 run on an (m_local x w) matrix.
struct Core {
  int64_t m_local = 0;
  int w = 0;
  double *part, *npart, *B, *lam, *nsq, *sig, *M, *G, *Z, *dz, *tsq, *T, *Rt, *sv, *Ps;
  int *idx, *idx2, *iout, *info;
  void alloc(Arena& a, int64_t m, int ww) {
    m_local = m;
    w = ww;
    size_t np = 0;
    for (int q = 1; q <= w; ++q) np = std::max(np, syrk_partials_doubles(std::max<int64_t>(m, 1), q));
    part = a.get<double>(np);
    size_t nn = 0;
    for (int q = 1; q <= w; ++q)
      nn = std::max(nn, (size_t)gemm_nn_grid(std::max<int64_t>(m, 1), q) * gemm_nn_part_stride(q));
    npart = a.get<double>(nn);
    B = a.get<double>((size_t)w * w);
    lam = a.get<double>(w);
    nsq = a.get<double>(w);
    sig = a.get<double>(w);
    M = a.get<double>(gemm_nn_m_doubles(w, w));
    G = a.get<double>((size_t)w * w);
    Z = a.get<double>((size_t)w * w);
    dz = a.get<double>(w);
    tsq = a.get<double>(w);
    T = a.get<double>(w);
    Rt = a.get<double>((size_t)w * (3 * w + 2));
    sv = a.get<double>(w);
    Ps = a.get<double>((size_t)w * w);
    idx = a.get<int>(w);
    idx2 = a.get<int>(w);
    iout = a.get<int>(8);
    info = a.get<int>(8);
  }
};

int jacobi_info(Ctx& c, const int* info, const char* what, int N) {
  int h[3];
  read_ints(c, info, 3, h);
  if (g_stats.n_jacobi < 16) g_stats.jacobi_sweeps[g_stats.n_jacobi++] = h[0];
  if (!h[1]) fail(TSSVD_ENOCONV, "Jacobi %s (N=%d) not converged in %d sweeps", what, N, h[0]);
  return h[2];
}

// After the final sync of a call: every deferred solve must have converged.
void check_deferred(Ctx& c) {
  if (!c.njinfo) return;
  static thread_local int* h = nullptr;
  if (!h) CU(cudaHostAlloc(reinterpret_cast<void**>(&h), 8 * Ctx::kMaxDeferred * sizeof(int), cudaHostAllocDefault));
  CU(cudaMemcpyAsync(h, c.jinfo, 8 * c.njinfo * sizeof(int), cudaMemcpyDeviceToHost, c.s));
  CU(cudaStreamSynchronize(c.s));
  for (int q = 0; q < c.njinfo; ++q) {
    if (g_stats.n_jacobi < 16) g_stats.jacobi_sweeps[g_stats.n_jacobi++] = h[8 * q];
    if (!h[8 * q + 1]) fail(TSSVD_ENOCONV, "Jacobi solve %d not converged in %d sweeps", q, h[8 * q]);
  }
}

// One-sided Jacobi rotation threshold for columns of `rows` dot-product rows:
// |x_p.x_q| > tol |x_p||x_q|, tol = max(8, 2 sqrt(rows)) eps -- LAPACK dgesvj's
// sqrt(M) eps with a factor 2 of margin over the dot products' rounding noise (an
// n eps threshold let the orthonormality of U drift to 1.1e-13 at r = 128).
inline double jacobi_tol(int rows) { return std::max(8.0, 2.0 * std::sqrt((double)rows)) * kEps; }

// Eigendecomposition of the PSD matrix B (n x n, ld n) in place: returns k and
// leaves eigenvector j (unit, descending eigenvalue) at B + j*n.  Pivots below
// trunc_rel * max diag are dropped (numerically null directions; reading R10).
// sync = false: no host round trip -- returns n (the kernel zero-fills the
// eigenvector slots [k, n), which then carry zero norms into the next discard)
// and convergence is checked after the call.
int eig(Ctx& c, Core& b, double* B, int n, double* vals, double trunc_rel, bool sync = true) {
  Pass t(c.s, TSSVD_PASS_JACOBI, 0, 0);
  int* info = sync ? b.info : c.next_info();
  KL(launch_jacobi_eig(B, n, n, jacobi_tol(n), trunc_rel, c.max_sweeps, B, n, vals, info, c.s));
  return sync ? jacobi_info(c, info, "eig", n) : n;
}

void note_rank(int64_t r) {
  if (g_stats.n_ranks < 8) g_stats.ranks[g_stats.n_ranks++] = r;
}

// Alg. 3 (passes = 1) or Alg. 4 (passes = 2) on X
// (m_local x w, ldx; row-sharded over the communicator when dist, replicated
// otherwise).  U (m_local x w capacity, ldu) receives U[:, :r]; may alias X.
// sigma[:r], V (w x r, ldv) replicated.  Returns r.
int64_t core(Ctx& c, Core& b, const double* X, int64_t ldx, int64_t m_local, int w, int passes,
             bool dist, double* U, int64_t ldu, double* sigma, double* V, int64_t ldv,
             double* Upack = nullptr) {
  // Upack: the final U is written there packed, leading dimension (r + 1) & ~1, instead of in place
  cudaStream_t s = c.s;
  Ctx cd = c;
  if (!dist) cd.comm = nullptr;
  // truncation of the eigensolver's pivoted Cholesky (reading R13): directions with
  // lambda <= 0.01 wp lambda_max have Sigma~^2 <= lambda + |E| far below the discard line
  // wp Sigma~_max^2, so they could never be kept; the truncated Schur complement
  // (<= (n-K) trunc lambda_max) moves the kept sigma by ~1e-13 sigma_1 (simulated at c2/c4),
  // three orders below the 1e-10 contract.
  const double trunc = std::max(kEps, 0.01 * c.wp);
  // Step 1 (P:613 / P:646): B = A^* A over the local rows, aggregated across ranks.
  {
    Pass t(s, TSSVD_PASS_GRAM_X, (double)m_local * w * (w + 1), 8.0 * m_local * w);
    KL(launch_syrk(X, ldx, m_local, w, b.part, s));
    KL(launch_reduce_sym(b.part, syrk_partials_grid(m_local, w), w, b.B, w, s));
  }
  if (cd.dist()) {
    allreduce(cd, b.B, (int64_t)w * w);
    KS(symmetrize(b.B, w, w, s));
  }
  // Step 2 (P:615 / P:648): B = V~ D V~^*  -> k eigenvectors (columns of B's buffer).
  const int k = eig(c, b, b.B, w, b.lam, trunc);
  if (k == 0) {  // B == 0 (or non-finite): nothing survives
    note_rank(0);
    return 0;
  }
  // Step 3 (P:619 / P:652): Y~ = A V~ (k columns) written into U;
  // Step 4 (P:621 / P:654): Sigma~ = column norms (sums of squares fused, then reduced).
  KS(cols_to_m(b.B, w, w, k, b.M, smem_ld(k), mrows_for(w), s));
  {
    Pass t(s, TSSVD_PASS_XV, 2.0 * m_local * w * k, 8.0 * m_local * (w + k));
    KL(launch_gemm_nn(X, ldx, m_local, w, b.M, k, U, ldu, b.npart, s));
    KL(launch_reduce_parts(b.npart, gemm_nn_grid(std::max<int64_t>(m_local, 1), k), gemm_nn_part_stride(k), k, b.nsq, s));
  }
  ++g_stats.a_passes;
  allreduce(cd, b.nsq, k);
  // Step 5 (P:625 / P:658): discard below max * sqrt(wp).
  KS(discard(b.nsq, k, c.wp, b.sig, b.idx, b.iout, nullptr, 0, s));
  int h[3];
  read_ints(c, b.iout, 3, h);
  if (h[2]) fail(TSSVD_ENONFINITE, "non-finite entries in the input (column norms)");
  const int r = h[0], nc = h[1];
  note_rank(r);
  if (r == 0) return 0;

  if (passes == 1) {
    // Step 6: U = Y~ Sigma^-1 (kept columns, sorted by Sigma, signs fixed), in place.
    const int ldm = smem_ld(r);
    KS(fill(b.M, (int64_t)mrows_for(nc) * ldm, 0.0, s));
    KS(alg3_out(b.sig, b.idx, r, b.B, w, b.M, ldm, sigma, V, ldv, s));
    {
      Pass t(s, TSSVD_PASS_UOUT, 2.0 * m_local * nc * r, 8.0 * m_local * (nc + r));
      KL(launch_gemm_nn(U, ldu, m_local, nc, b.M, r, Upack ? Upack : U, Upack ? (r + 1) & ~1 : ldu,
                        nullptr, s));
    }
    return r;
  }
  // Steps 6-7: Z = Y^* Y = Sigma~^-1 (Y~^* Y~)_keep Sigma~^-1.
  {
    Pass t(s, TSSVD_PASS_GRAM_Y, (double)m_local * nc * (nc + 1), 8.0 * m_local * nc);
    KL(launch_syrk(U, ldu, m_local, nc, b.part, s));
    KL(launch_reduce_sym(b.part, syrk_partials_grid(m_local, nc), nc, b.G, nc, s));
  }
  if (cd.dist()) {
    allreduce(cd, b.G, (int64_t)nc * nc);
    KS(symmetrize(b.G, nc, nc, s));
  }
  KS(build_z(b.G, nc, b.idx, b.sig, r, b.Z, s));
  // Step 8: Z = W D W^*  (W: r x kz, column-major in b.Z).
  const int kz = eig(c, b, b.Z, r, b.dz, trunc, false);  // Z = Y^T Y ~ I: kz = r
  // Steps 9-10: Q~ = Y W, T = column norms of Q~ (norms only, nothing stored).
  const int ldm_k = smem_ld(kz);
  KS(fill(b.M, (int64_t)mrows_for(nc) * ldm_k, 0.0, s));
  KS(build_m1(b.Z, b.idx, b.sig, r, kz, b.M, ldm_k, s));
  {
    Pass t(s, TSSVD_PASS_QNORM, 2.0 * m_local * nc * kz, 8.0 * m_local * nc);
    KL(launch_gemm_nn(U, ldu, m_local, nc, b.M, kz, nullptr, 0, b.npart, s));
    KL(launch_reduce_parts(b.npart, gemm_nn_grid(std::max<int64_t>(m_local, 1), kz), gemm_nn_part_stride(kz), kz, b.tsq, s));
  }
  allreduce(cd, b.tsq, kz);
  // Step 11: discard T below max(T) sqrt(wp).
  KS(discard(b.tsq, kz, c.wp, b.T, b.idx2, b.iout, nullptr, 0, s));
  read_ints(c, b.iout, 3, h);
  if (h[2]) fail(TSSVD_ENONFINITE, "non-finite column norms in the second orthonormalization");
  const int r2 = h[0];
  note_rank(r2);
  if (r2 == 0) return 0;
  // Steps 12-14: R = T W^* Sigma~ V~^* = K V~_keep^T with K = T W_keep^T Sigma~
  // (r2 x r); SVD of K by one-sided Jacobi on its columns, K J = P Sigma  =>  V = V~_keep J.
  KS(build_k(b.T, b.idx2, r2, b.Z, r, b.sig, b.idx, b.Rt, s));
  {
    Pass t(s, TSSVD_PASS_JACOBI, 0, 0);
    KL(launch_jacobi_svd(b.Rt, r2, r, r2, jacobi_tol(r2), c.max_sweeps, b.Rt + (size_t)r2 * r,
                         r2 + r, b.sv, c.next_info(), s));
  }
  KS(svd_out(b.Rt + (size_t)r2 * r, r2 + r, r2, r, b.sv, b.B, w, b.idx, sigma, V, ldv, b.Ps, s));
  // Step 15: U = Q P = Y~[:, :nc] (S W T^-1 P), in place.
  const int ldm_r2 = smem_ld(r2);
  KS(fill(b.M, (int64_t)mrows_for(nc) * ldm_r2, 0.0, s));
  KS(build_m2(b.Z, r, b.idx, b.sig, b.T, b.idx2, r2, b.Ps, b.M, ldm_r2, s));
  {
    Pass t(s, TSSVD_PASS_UOUT, 2.0 * m_local * nc * r2, 8.0 * m_local * (nc + r2));
    KL(launch_gemm_nn(U, ldu, m_local, nc, b.M, r2, Upack ? Upack : U, Upack ? (r2 + 1) & ~1 : ldu,
                      nullptr, s));
  }
  return r2;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

void check_opts(const tssvd_opts* o) {
  if (!o) fail(TSSVD_EINVAL, "opts is NULL");
  if (o->abi_version != TSSVD_ABI_VERSION) fail(TSSVD_EINVAL, "opts->abi_version %d != %d", o->abi_version, TSSVD_ABI_VERSION);
  if (!(o->working_precision > 0.0 && o->working_precision < 1.0))
    fail(TSSVD_EINVAL, "working precision %g not in (0,1)", o->working_precision);
  if (o->max_jacobi_sweeps < 1) fail(TSSVD_EINVAL, "max_jacobi_sweeps < 1");
  if (o->host_io != 0 && o->host_io != 1) fail(TSSVD_EINVAL, "host_io must be 0 or 1");
}

void set_device(tssvd_comm* comm) {
  if (comm) CU(cudaSetDevice(comm->device));
}

// global m = sum of m_local over ranks (int64 allreduce), used for validation
int64_t global_rows(Ctx& c, int64_t m_local, void* scratch_dev) {
  if (!c.dist()) return m_local;
  int64_t* d = static_cast<int64_t*>(scratch_dev);
  int64_t* h = reinterpret_cast<int64_t*>(pinned_ints());
  *h = m_local;
  CU(cudaMemcpyAsync(d, h, 8, cudaMemcpyHostToDevice, c.s));
  NC(ncclAllReduce(d, d, 1, ncclInt64, ncclSum, c.comm->nccl, c.s));
  CU(cudaMemcpyAsync(h, d, 8, cudaMemcpyDeviceToHost, c.s));
  CU(cudaStreamSynchronize(c.s));
  return *h;
}

struct TsPlan {
  Core core;
  int* jinfo;
  int64_t* m_scratch;
  double* a_stage;  // host_io: device copy of A (also holds Y~)
  double* u_pack;   // host_io: U packed (ld (r+1)&~1) for one contiguous D2H copy
  double* sig_stage;
  double* v_stage;
};

size_t plan_tssvd(Arena& a, TsPlan& p, int64_t m_local, int n, const tssvd_opts* o) {
  p.jinfo = a.get<int>(8 * Ctx::kMaxDeferred);
  p.m_scratch = a.get<int64_t>(2);
  p.core.alloc(a, m_local, n);
  if (o && o->host_io) {
    p.a_stage = a.get<double>((size_t)std::max<int64_t>(m_local, 1) * n);
    p.u_pack = a.get<double>((size_t)std::max<int64_t>(m_local, 1) * ((n + 1) & ~1));
    p.sig_stage = a.get<double>(n);
    p.v_stage = a.get<double>((size_t)n * n);
  }
  return a.off;
}

void validate_tall(int64_t m_local, int64_t n, int64_t lda) {
  if (m_local < 0) fail(TSSVD_EINVAL, "m_local < 0");
  if (n < 1 || n > 256) fail(TSSVD_EINVAL, "n = %lld must be in [1, 256]", (long long)n);
  if (n & 1) fail(TSSVD_EINVAL, "n = %lld must be even (rows move as 16-byte TMA granules)", (long long)n);
  if (lda < n || (lda & 1)) fail(TSSVD_EINVAL, "lda = %lld must be even and >= n", (long long)lda);
}

void tssvd_impl(tssvd_comm* comm, void* stream, int64_t m_local, int64_t n, const double* A,
                int64_t lda, const tssvd_opts* opts, double* U, int64_t ldu, double* sigma,
                double* V, int64_t ldv, int64_t* rank, void* ws, size_t ws_bytes) {
  g_stats = tssvd_stats{};
  check_opts(opts);
  validate_tall(m_local, n, lda);
  if (opts->orthonormalizations != 1 && opts->orthonormalizations != 2)
    fail(TSSVD_EINVAL, "orthonormalizations must be 1 or 2");
  if (!rank) fail(TSSVD_EINVAL, "rank is NULL");
  if (ldv < n) fail(TSSVD_EINVAL, "ldv < n");
  const bool hio = opts->host_io == 1;
  if (!hio) {
    if (ldu < n || (ldu & 1)) fail(TSSVD_EINVAL, "ldu must be even and >= n");
    if ((m_local > 0 && (!aligned16(A) || !aligned16(U)))) fail(TSSVD_EINVAL, "A and U must be 16-byte aligned");
  } else if (ldu != 0 && ldu < n) {
    fail(TSSVD_EINVAL, "ldu must be 0 (packed) or >= n");
  }
  if (!ws || !aligned16(ws)) fail(TSSVD_EINVAL, "workspace NULL or misaligned");
  set_device(comm);
  Ctx c;
  c.comm = comm;
  c.s = static_cast<cudaStream_t>(stream);
  c.wp = opts->working_precision;
  c.max_sweeps = opts->max_jacobi_sweeps;
  Arena a;
  a.base = static_cast<char*>(ws);
  a.cap = ws_bytes;
  a.dry = false;
  TsPlan p;
  plan_tssvd(a, p, m_local, (int)n, opts);
  c.jinfo = p.jinfo;
  const int64_t m = global_rows(c, m_local, p.m_scratch);
  if (m < n) fail(TSSVD_EINVAL, "m = %lld < n = %lld (the matrix must be tall, P:98-104)", (long long)m, (long long)n);
  const double* X = A;
  int64_t ldx = lda;
  double* Ud = U;
  int64_t ldud = ldu;
  double* sigd = sigma;
  double* Vd = V;
  int64_t ldvd = ldv;
  if (hio) {  // stage host A into the workspace (it becomes the in-place U buffer)
    if (m_local > 0) {
      if (lda == n) CU(cudaMemcpyAsync(p.a_stage, A, (size_t)m_local * n * 8, cudaMemcpyHostToDevice, c.s));
      else CU(cudaMemcpy2DAsync(p.a_stage, n * 8, A, lda * 8, n * 8, m_local, cudaMemcpyHostToDevice, c.s));
    }
    X = p.a_stage;
    ldx = n;
    Ud = p.a_stage;
    ldud = n;
    sigd = p.sig_stage;
    Vd = p.v_stage;
    ldvd = n;
  }
  const bool packed = hio && ldu == 0;
  const int64_t r = core(c, p.core, X, ldx, m_local, (int)n, opts->orthonormalizations, true, Ud,
                         ldud, sigd, Vd, ldvd, packed ? p.u_pack : nullptr);
  if (hio && r > 0) {
    if (m_local > 0) {
      if (packed)  // one contiguous copy: U with leading dimension (r + 1) & ~1
        CU(cudaMemcpyAsync(U, p.u_pack, (size_t)m_local * ((r + 1) & ~1) * 8, cudaMemcpyDeviceToHost, c.s));
      else
        CU(cudaMemcpy2DAsync(U, ldu * 8, Ud, ldud * 8, r * 8, m_local, cudaMemcpyDeviceToHost, c.s));
    }
    CU(cudaMemcpyAsync(sigma, sigd, r * 8, cudaMemcpyDeviceToHost, c.s));
    CU(cudaMemcpy2DAsync(V, ldv * 8, Vd, ldvd * 8, r * 8, n, cudaMemcpyDeviceToHost, c.s));
  }
  CU(cudaStreamSynchronize(c.s));
  check_deferred(c);
  g_timer.resolve();
  *rank = r;
}

// ------------------------------------------------------------- low rank --
struct LrPlan {
  Core tall, small;
  int* jinfo;
  int64_t* m_scratch;
  double *Qt, *Y, *Z, *tn, *Ut, *sig_tmp, *v_scr, *sig_scr, *Mfin;
  double *a_stage, *o_stage, *u_stage, *s_stage, *vo_stage;
  int lp, ldzmax;
};

size_t plan_lowrank(Arena& a, LrPlan& p, int64_t m_local, int n, int l, const tssvd_opts* o) {
  p.lp = (l + 1) & ~1;
  p.ldzmax = pad8(l);
  p.jinfo = a.get<int>(8 * Ctx::kMaxDeferred);
  p.m_scratch = a.get<int64_t>(2);
  p.tall.alloc(a, m_local, l);
  p.small.alloc(a, n, l);
  p.Qt = a.get<double>(gemm_nn_m_doubles(n, l));
  p.Y = a.get<double>((size_t)std::max<int64_t>(m_local, 1) * p.lp);
  p.Z = a.get<double>((size_t)n * p.ldzmax);
  size_t tn = 0;
  for (int q = 1; q <= l; ++q) tn = std::max(tn, plan_gemm_tn(std::max<int64_t>(m_local, 1), n, q).part_doubles);
  p.tn = a.get<double>(tn);
  p.Ut = a.get<double>((size_t)l * l);
  p.sig_tmp = a.get<double>(l);
  p.sig_scr = a.get<double>(l);
  p.v_scr = a.get<double>((size_t)std::max(n, l) * l);
  p.Mfin = a.get<double>(gemm_nn_m_doubles(l, l));
  if (o && o->host_io) {
    p.a_stage = a.get<double>((size_t)std::max<int64_t>(m_local, 1) * n);
    p.o_stage = a.get<double>((size_t)n * l);
    p.u_stage = a.get<double>((size_t)std::max<int64_t>(m_local, 1) * l);
    p.s_stage = a.get<double>(l);
    p.vo_stage = a.get<double>((size_t)n * l);
  }
  return a.off;
}

// Z (n x ldz) = sum over ranks of A_p^T Q_p  (Alg. 5 step 5 / Alg. 6 step 1)
int tn_pass(Ctx& c, LrPlan& p, const double* A, int64_t lda, int64_t m_local, int n, int r) {
  const TnPlan tp = plan_gemm_tn(std::max<int64_t>(m_local, 1), n, r);
  if (m_local > 0) {
    Pass t(c.s, TSSVD_PASS_BETA, 2.0 * m_local * n * r, 8.0 * m_local * (n + r));
    KL(launch_gemm_tn(tp, A, lda, m_local, n, p.Y, p.lp, r, p.tn, c.s));
    KL(launch_reduce_parts(p.tn, tp.splits, (int64_t)tp.colblocks * tp.cb * tp.ldz, (int64_t)n * tp.ldz, p.Z, c.s));
  } else {
    KS(fill(p.Z, (int64_t)n * tp.ldz, 0.0, c.s));
  }
  ++g_stats.a_passes;
  allreduce(c, p.Z, (int64_t)n * tp.ldz);
  return tp.ldz;
}

void lowrank_impl(tssvd_comm* comm, void* stream, int64_t m_local, int64_t n, const double* A,
                  int64_t lda, const double* Omega, int64_t ldo, int64_t l, int iters, int64_t k,
                  const tssvd_opts* opts, double* U, int64_t ldu, double* sigma, double* V,
                  int64_t ldv, int64_t* rank, void* ws, size_t ws_bytes) {
  g_stats = tssvd_stats{};
  check_opts(opts);
  if (m_local < 0) fail(TSSVD_EINVAL, "m_local < 0");
  if (n < 2 || (n & 1)) fail(TSSVD_EINVAL, "n = %lld must be even and >= 2", (long long)n);
  if (lda < n || (lda & 1)) fail(TSSVD_EINVAL, "lda must be even and >= n");
  if (l < 1 || l > 128 || l >= n) fail(TSSVD_EINVAL, "need 0 < l < min(m, n) and l <= 128 (l = %lld)", (long long)l);
  if (iters < 0) fail(TSSVD_EINVAL, "iters < 0");
  if (k < 1 || k > l) fail(TSSVD_EINVAL, "need 0 < k <= l");
  if (ldo < l || ldu < k || ldv < k) fail(TSSVD_EINVAL, "ldo < l, ldu < k or ldv < k");
  if (!rank) fail(TSSVD_EINVAL, "rank is NULL");
  const bool hio = opts->host_io == 1;
  if (!hio && m_local > 0 && !aligned16(A)) fail(TSSVD_EINVAL, "A must be 16-byte aligned");
  if (!ws || !aligned16(ws)) fail(TSSVD_EINVAL, "workspace NULL or misaligned");
  set_device(comm);
  Ctx c;
  c.comm = comm;
  c.s = static_cast<cudaStream_t>(stream);
  c.wp = opts->working_precision;
  c.max_sweeps = opts->max_jacobi_sweeps;
  Arena a;
  a.base = static_cast<char*>(ws);
  a.cap = ws_bytes;
  a.dry = false;
  LrPlan p;
  plan_lowrank(a, p, m_local, (int)n, (int)l, opts);
  c.jinfo = p.jinfo;
  const int64_t m = global_rows(c, m_local, p.m_scratch);
  if (l >= std::min<int64_t>(m, n)) fail(TSSVD_EINVAL, "need l < min(m, n) (P:705-707)");
  const int N = (int)n, Lc = (int)l;
  const double* Ad = A;
  int64_t ldad = lda;
  const double* Od = Omega;
  int64_t ldod = ldo;
  if (hio) {
    if (m_local > 0)
      CU(cudaMemcpy2DAsync(p.a_stage, n * 8, A, lda * 8, n * 8, m_local, cudaMemcpyHostToDevice, c.s));
    CU(cudaMemcpy2DAsync(p.o_stage, l * 8, Omega, ldo * 8, l * 8, n, cudaMemcpyHostToDevice, c.s));
    Ad = p.a_stage;
    ldad = n;
    Od = p.o_stage;
    ldod = l;
  }
  // Alg. 5 step 1: Q~_0 = Omega.
  int lj = Lc;
  KS(rows_to_m(Od, ldod, N, lj, p.Qt, smem_ld(lj), mrows_for(N), c.s));
  for (int it = 0; it < iters; ++it) {
    // step 3: Y_j = A Q~_{j-1}
    {
      Pass t(c.s, TSSVD_PASS_ALPHA, 2.0 * m_local * N * lj, 8.0 * m_local * (N + lj));
      KL(launch_gemm_nn(Ad, ldad, m_local, N, p.Qt, lj, p.Y, p.lp, nullptr, c.s));
    }
    ++g_stats.a_passes;
    // step 4: Y_j = Q_j R_j by Alg. 3 (Q_j = U, in place in Y)
    const int64_t r = core(c, p.tall, p.Y, p.lp, m_local, lj, 1, true, p.Y, p.lp, p.sig_scr, p.v_scr, lj);
    if (r == 0) { *rank = 0; CU(cudaStreamSynchronize(c.s)); check_deferred(c); return; }
    // step 5: Y~_j = A^* Q_j
    const int ldz = tn_pass(c, p, Ad, ldad, m_local, N, (int)r);
    // step 6: Y~_j = Q~_j R~_j by Alg. 3 on the replicated n x r matrix
    const int64_t r2 = core(c, p.small, p.Z, ldz, N, (int)r, 1, false, p.Z, ldz, p.sig_scr, p.v_scr, r);
    if (r2 == 0) { *rank = 0; CU(cudaStreamSynchronize(c.s)); check_deferred(c); return; }
    lj = (int)r2;
    KS(rows_to_m(p.Z, ldz, N, lj, p.Qt, smem_ld(lj), mrows_for(N), c.s));
  }
  // step 8: Y = A Q~_i; step 9: Y = Q R by Alg. 4
  {
    Pass t(c.s, TSSVD_PASS_ALPHA, 2.0 * m_local * N * lj, 8.0 * m_local * (N + lj));
    KL(launch_gemm_nn(Ad, ldad, m_local, N, p.Qt, lj, p.Y, p.lp, nullptr, c.s));
  }
  ++g_stats.a_passes;
  const int64_t r3 = core(c, p.tall, p.Y, p.lp, m_local, lj, 2, true, p.Y, p.lp, p.sig_scr, p.v_scr, lj);
  if (r3 == 0) { *rank = 0; CU(cudaStreamSynchronize(c.s)); check_deferred(c); return; }
  // Alg. 6 step 1: B^T = A^* Q
  const int ldz = tn_pass(c, p, Ad, ldad, m_local, N, (int)r3);
  // Alg. 6 step 2: B^T = V Sigma U~^* by Alg. 4 (reading R6); V in place in Z
  const int64_t r4 = core(c, p.small, p.Z, ldz, N, (int)r3, 2, false, p.Z, ldz, p.sig_tmp, p.Ut, Lc);
  if (r4 == 0) { *rank = 0; CU(cudaStreamSynchronize(c.s)); check_deferred(c); return; }
  KS(canon_lowrank(p.Z, ldz, N, p.Ut, Lc, (int)r3, (int)r4, c.s));
  const int kk = (int)std::min<int64_t>(k, r4);
  // Alg. 6 step 3: U = Q U~ (leading kk columns, reading R7)
  KS(rows_to_m(p.Ut, Lc, (int)r3, kk, p.Mfin, smem_ld(kk), mrows_for((int)r3), c.s));
  double* Uo = hio ? p.u_stage : U;
  int64_t lduo = hio ? kk : ldu;
  if (!hio && m_local > 0 && (!aligned16(U) || (ldu & 1))) {
    // unaligned caller U: produce into Y's spare space is not possible; use u via copy
    fail(TSSVD_EINVAL, "U must be 16-byte aligned with an even ldu");
  }
  KL(launch_gemm_nn(p.Y, p.lp, m_local, (int)r3, p.Mfin, kk, Uo, lduo, nullptr, c.s));
  double* So = hio ? p.s_stage : sigma;
  double* Vo = hio ? p.vo_stage : V;
  int64_t ldvo = hio ? kk : ldv;
  KS(copy2d(p.sig_tmp, kk, So, kk, 1, kk, c.s));
  KS(copy2d(p.Z, ldz, Vo, ldvo, N, kk, c.s));
  if (hio) {
    if (m_local > 0)
      CU(cudaMemcpy2DAsync(U, ldu * 8, Uo, lduo * 8, kk * 8, m_local, cudaMemcpyDeviceToHost, c.s));
    CU(cudaMemcpyAsync(sigma, So, kk * 8, cudaMemcpyDeviceToHost, c.s));
    CU(cudaMemcpy2DAsync(V, ldv * 8, Vo, ldvo * 8, kk * 8, N, cudaMemcpyDeviceToHost, c.s));
  }
  CU(cudaStreamSynchronize(c.s));
  check_deferred(c);
  g_timer.resolve();
  *rank = kk;
}

}  // namespace

// ================================================================= C ABI ==
extern "C" {

const char* tssvd_status_string(int st) {
  switch (st) {
    case TSSVD_OK: return "ok";
    case TSSVD_EINVAL: return "invalid argument";
    case TSSVD_ENONFINITE: return "non-finite input";
    case TSSVD_ENOCONV: return "Jacobi did not converge";
    case TSSVD_ECUDA: return "CUDA error";
    case TSSVD_ENCCL: return "NCCL error";
    case TSSVD_ENOMEM: return "workspace too small";
    default: return "unknown status";
  }
}

const char* tssvd_last_error(void) { return g_err.c_str(); }
int tssvd_abi_version(void) { return TSSVD_ABI_VERSION; }

void tssvd_opts_default(tssvd_opts* o) {
  if (!o) return;
  o->abi_version = TSSVD_ABI_VERSION;
  o->working_precision = 1e-11;
  o->orthonormalizations = 2;
  o->max_jacobi_sweeps = 60;
  o->host_io = 0;
}

int tssvd_get_unique_id(unsigned char id[128]) {
  return guarded([&] {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId u;
    NC(ncclGetUniqueId(&u));
    std::memcpy(id, &u, 128);
  });
}

int tssvd_comm_create(int nranks, int rank, const unsigned char id[128], int device,
                      tssvd_comm** out) {
  return guarded([&] {
    if (!out || nranks < 1 || rank < 0 || rank >= nranks) fail(TSSVD_EINVAL, "bad comm arguments");
    CU(cudaSetDevice(device));
    auto* c = new tssvd_comm;
    c->rank = rank;
    c->nranks = nranks;
    c->device = device;
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, u, rank);
    if (r != ncclSuccess) {
      delete c;
      fail(TSSVD_ENCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
    }
    *out = c;
  });
}

int tssvd_comm_wrap_nccl(void* nccl_comm, tssvd_comm** out) {
  return guarded([&] {
    if (!nccl_comm || !out) fail(TSSVD_EINVAL, "tssvd_comm_wrap_nccl: NULL communicator or out pointer");
    auto* c = new tssvd_comm;
    c->nccl = static_cast<ncclComm_t>(nccl_comm);
    c->owned = false;
    ncclResult_t r = ncclCommUserRank(c->nccl, &c->rank);
    if (r == ncclSuccess) r = ncclCommCount(c->nccl, &c->nranks);
    if (r == ncclSuccess) r = ncclCommCuDevice(c->nccl, &c->device);
    if (r != ncclSuccess) {
      delete c;
      fail(TSSVD_ENCCL, "tssvd_comm_wrap_nccl: %s", ncclGetErrorString(r));
    }
    *out = c;
  });
}

int tssvd_comm_destroy(tssvd_comm* c) {
  return guarded([&] {
    if (!c) return;
    if (c->nccl && c->owned) NC(ncclCommDestroy(c->nccl));
    delete c;
  });
}

int tssvd_comm_rank(const tssvd_comm* c, int* rank, int* nranks) {
  return guarded([&] {
    if (rank) *rank = c ? c->rank : 0;
    if (nranks) *nranks = c ? c->nranks : 1;
  });
}

int tssvd_allreduce_sum(tssvd_comm* comm, void* stream, double* buf, int64_t count) {
  return guarded([&] {
    Ctx c;
    c.comm = comm;
    c.s = static_cast<cudaStream_t>(stream);
    allreduce(c, buf, count);
    CU(cudaStreamSynchronize(c.s));
  });
}

int tssvd_workspace_size(const tssvd_comm*, int64_t m_local, int64_t n, const tssvd_opts* opts,
                         size_t* bytes) {
  return guarded([&] {
    check_opts(opts);
    validate_tall(m_local, n, n);
    if (!bytes) fail(TSSVD_EINVAL, "bytes is NULL");
    Arena a;
    TsPlan p;
    *bytes = plan_tssvd(a, p, m_local, (int)n, opts) + 256;
  });
}

int tssvd(tssvd_comm* comm, void* stream, int64_t m_local, int64_t n, const double* A,
          int64_t lda, const tssvd_opts* opts, double* U, int64_t ldu, double* sigma, double* V,
          int64_t ldv, int64_t* rank, void* workspace, size_t workspace_bytes) {
  return guarded([&] {
    tssvd_impl(comm, stream, m_local, n, A, lda, opts, U, ldu, sigma, V, ldv, rank, workspace,
               workspace_bytes);
  });
}

int lowrank_workspace_size(const tssvd_comm*, int64_t m_local, int64_t n, int64_t l,
                           const tssvd_opts* opts, size_t* bytes) {
  return guarded([&] {
    check_opts(opts);
    if (m_local < 0 || n < 2 || l < 1 || l > 128 || l >= n) fail(TSSVD_EINVAL, "bad sizes");
    if (!bytes) fail(TSSVD_EINVAL, "bytes is NULL");
    Arena a;
    LrPlan p;
    *bytes = plan_lowrank(a, p, m_local, (int)n, (int)l, opts) + 256;
  });
}

int lowrank_svd(tssvd_comm* comm, void* stream, int64_t m_local, int64_t n, const double* A,
                int64_t lda, const double* Omega, int64_t ldo, int64_t l, int iters, int64_t k,
                const tssvd_opts* opts, double* U, int64_t ldu, double* sigma, double* V,
                int64_t ldv, int64_t* rank, void* workspace, size_t workspace_bytes) {
  return guarded([&] {
    lowrank_impl(comm, stream, m_local, n, A, lda, Omega, ldo, l, iters, k, opts, U, ldu, sigma, V,
                 ldv, rank, workspace, workspace_bytes);
  });
}

int tssvd_set_pass_timing(int enable) {
  g_timing = enable != 0;
  return TSSVD_OK;
}

int tssvd_last_stats(tssvd_stats* out) {
  if (!out) return TSSVD_EINVAL;
  *out = g_stats;
  return TSSVD_OK;
}

// ---- building blocks ------------------------------------------------------
size_t tssvd_gram_workspace(int64_t m, int64_t n) {
  return (syrk_partials_doubles(std::max<int64_t>(m, 1), (int)n) + 64) * 8;
}

int tssvd_gram(void* stream, int64_t m, int64_t n, const double* X, int64_t ldx, double* G,
               int64_t ldg, void* ws, size_t wsb) {
  return guarded([&] {
    if (m < 0 || n < 1 || n > 256 || ldx < ((n + 1) & ~1) || (ldx & 1) || ldg < n)
      fail(TSSVD_EINVAL, "bad gram arguments");
    if (wsb < tssvd_gram_workspace(m, n)) fail(TSSVD_ENOMEM, "gram workspace too small");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    double* part = static_cast<double*>(ws);
    CU(launch_syrk(X, ldx, m, (int)n, part, s));
    CU(launch_reduce_sym(part, syrk_partials_grid(m, (int)n), (int)n, G, (int)ldg, s));
    CU(cudaStreamSynchronize(s));
  });
}

size_t tssvd_matmul_workspace(int64_t m, int64_t k, int64_t c) {
  return (gemm_nn_m_doubles((int)k, (int)c) + (size_t)gemm_nn_grid(std::max<int64_t>(m, 1), (int)c) * gemm_nn_part_stride((int)c) + 128) * 8;
}

int tssvd_matmul(void* stream, int64_t m, int64_t k, int64_t c, const double* X, int64_t ldx,
                 const double* M, int64_t ldm, double* Y, int64_t ldy, double* nsq, void* ws,
                 size_t wsb) {
  return guarded([&] {
    if (m < 0 || k < 1 || c < 1 || c > 256 || ldx < ((k + 1) & ~1) || (ldx & 1) || ldm < c)
      fail(TSSVD_EINVAL, "bad matmul arguments");
    if (Y && (ldy < c || (ldy & 1))) fail(TSSVD_EINVAL, "ldy must be even and >= c");
    if (wsb < tssvd_matmul_workspace(m, k, c)) fail(TSSVD_ENOMEM, "matmul workspace too small");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    double* Mp = static_cast<double*>(ws);
    double* np = Mp + ((gemm_nn_m_doubles((int)k, (int)c) + 31) & ~size_t(31));
    rows_to_m(M, ldm, (int)k, (int)c, Mp, smem_ld((int)c), mrows_for((int)k), s);
    CU(cudaGetLastError());
    CU(launch_gemm_nn(X, ldx, m, (int)k, Mp, (int)c, Y, ldy, nsq ? np : nullptr, s));
    if (nsq)
      CU(launch_reduce_parts(np, gemm_nn_grid(std::max<int64_t>(m, 1), (int)c), gemm_nn_part_stride((int)c), c, nsq, s));
    CU(cudaStreamSynchronize(s));
  });
}

size_t tssvd_matmul_tn_workspace(int64_t m, int64_t n, int64_t l) {
  return (plan_gemm_tn(std::max<int64_t>(m, 1), (int)n, (int)l).part_doubles + 64) * 8;
}

int tssvd_matmul_tn(void* stream, int64_t m, int64_t n, int64_t l, const double* X, int64_t ldx,
                    const double* Y, int64_t ldy, double* Z, int64_t ldz, void* ws, size_t wsb) {
  return guarded([&] {
    if (m < 1 || n < 2 || (n & 1) || l < 1 || l > 128 || ldx < n || (ldx & 1) ||
        ldy < ((l + 1) & ~1) || (ldy & 1) || ldz < l)
      fail(TSSVD_EINVAL, "bad matmul_tn arguments");
    if (wsb < tssvd_matmul_tn_workspace(m, n, l)) fail(TSSVD_ENOMEM, "matmul_tn workspace too small");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const TnPlan tp = plan_gemm_tn(m, (int)n, (int)l);
    double* part = static_cast<double*>(ws);
    CU(launch_gemm_tn(tp, X, ldx, m, (int)n, Y, ldy, (int)l, part, s));
    // reduce into Z columns [0, l): reduce to a padded temp is avoided by reducing per element
    CU(launch_reduce_parts(part, tp.splits, (int64_t)tp.colblocks * tp.cb * tp.ldz, (int64_t)n * tp.ldz, part, s));  // in place into split 0
    copy2d(part, tp.ldz, Z, ldz, n, (int)l, s);
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(s));
  });
}

size_t tssvd_sym_eig_workspace(int64_t n) { return ((size_t)n * n + 64) * 8; }

int tssvd_sym_eig(void* stream, int64_t n, const double* B, int64_t ldb, double* lambda, double* Vt,
                  int64_t ldv, int max_sweeps, int* sweeps, void* ws, size_t wsb) {
  return guarded([&] {
    if (n < 1 || n > 512 || ldb < n || ldv < n) fail(TSSVD_EINVAL, "bad sym_eig arguments");
    if (wsb < tssvd_sym_eig_workspace(n)) fail(TSSVD_ENOMEM, "sym_eig workspace too small");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    double* vecs = static_cast<double*>(ws);
    int* info = reinterpret_cast<int*>(vecs + (size_t)n * n);
    fill(vecs, (int64_t)n * n, 0.0, s);
    fill(lambda, n, 0.0, s);
    CU(cudaGetLastError());
    // no truncation beyond the noise floor: trunc = eps
    CU(launch_jacobi_eig(B, (int)ldb, (int)n, jacobi_tol((int)n), kEps, max_sweeps,
                         vecs, (int)n, lambda, info, s));
    copy2d(vecs, n, Vt, ldv, n, (int)n, s);  // eigenvector j (contiguous) -> row j of Vt
    CU(cudaGetLastError());
    int h[3];
    CU(cudaMemcpyAsync(h, info, 12, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    if (sweeps) *sweeps = h[0];
    if (!h[1]) fail(TSSVD_ENOCONV, "sym_eig did not converge");
  });
}

}  // extern "C"
