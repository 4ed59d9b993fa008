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
#include <vector>

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
// Plan-only ("dry") run, tssvd_trace(): no CUDA or NCCL call is made, every step the
// orchestrator takes is appended to g_trace instead ("token;token;...").  The gloo
// replay test drives its numpy re-enactment of the multi-rank data flow with it.
thread_local bool g_dry = false;
thread_local std::string g_trace;

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
// CUDA runtime calls of the orchestrator (copies, syncs): skipped in a dry run
#define CUR(x)                                                                                 \
  do {                                                                                         \
    if (!g_dry) CU(x);                                                                         \
  } while (0)
#define KL(x)                                                                                  \
  do {                                                                                         \
    if (!g_dry) CU(x);                                                                         \
    ++g_stats.kernel_launches;                                                                 \
  } while (0)
#define KS(x)                                                                                  \
  do {                                                                                         \
    if (!g_dry) {                                                                              \
      x;                                                                                       \
      CU(cudaGetLastError());                                                                  \
    }                                                                                          \
    ++g_stats.kernel_launches;                                                                 \
  } while (0)

void step(const char* fmt, ...) {
  if (!g_dry) return;
  char buf[128];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_trace += buf;
  g_trace += ';';
}

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

// Per-call control block in device memory, read back once at the end of the call:
//   jinfo : deferred Jacobi solves, 8 ints each {sweeps, converged, k, -, -, rounds, nonfinite, -}
//   slots : "Discard" decisions, 8 ints each (small_kernels.h kSlot*)
//   guard : multi-rank: max-allreduced copy of the slots (every rank must match it)
//   m64   : multi-rank: global row count (int64 allreduce), validated at the end
constexpr int kMaxDeferred = 48, kMaxSlots = 32;
constexpr int kCtlInts = 8 * kMaxDeferred + 2 * 8 * kMaxSlots + 4;

struct Ctx {
  tssvd_comm* comm = nullptr;
  cudaStream_t s = nullptr;
  double wp = 1e-11;
  int max_sweeps = 60;
  int* ctl = nullptr;  // device, kCtlInts
  int njinfo = 0, nslots = 0;
  bool dist() const { return comm && comm->nranks > 1; }
  int* jinfo() const { return ctl; }
  int* slots() const { return ctl + 8 * kMaxDeferred; }
  int* guard() const { return ctl + 8 * kMaxDeferred + 8 * kMaxSlots; }
  int64_t* m64() const { return reinterpret_cast<int64_t*>(ctl + 8 * kMaxDeferred + 16 * kMaxSlots); }
  int* next_info() {
    if (njinfo >= kMaxDeferred) fail(TSSVD_ECUDA, "too many deferred Jacobi solves");
    return jinfo() + 8 * njinfo++;
  }
  int next_slot() {
    if (nslots >= kMaxSlots) fail(TSSVD_ECUDA, "too many discard decisions");
    return nslots++;
  }
  int* slot(int i) const { return slots() + 8 * i; }
};

// pinned host mirror of the control block
int* host_ctl() {
  static thread_local int* p = nullptr;
  if (!p) CU(cudaHostAlloc(reinterpret_cast<void**>(&p), (kCtlInts + 4) * sizeof(int), cudaHostAllocDefault));
  return p;
}

void allreduce(Ctx& c, double* buf, int64_t count, const char* what) {
  if (!c.dist() || count <= 0) return;
  step("allreduce:%s:%lld", what, (long long)count);
  if (!g_dry) NC(ncclAllReduce(buf, buf, (size_t)count, ncclDouble, ncclSum, c.comm->nccl, c.s));
}

// Per-pass CUDA-event timing (tssvd_set_pass_timing): events recorded on the
// call's stream around each streaming kernel, resolved after the final sync.
struct PassTimer {
  cudaEvent_t ev[2 * TSSVD_MAX_PASSES] = {};
  int open = -1;
  cudaStream_t s = nullptr;
  void begin(cudaStream_t st, int kind, double flops, double bytes) {
    if (g_dry || !g_timing || g_stats.n_pass >= TSSVD_MAX_PASSES) return;
    const int i = g_stats.n_pass;
    for (int q = 0; q < 2; ++q)
      if (!ev[2 * i + q]) CU(cudaEventCreate(&ev[2 * i + q]));
    g_stats.pass_kind[i] = kind;
    g_stats.pass_flops[i] = flops;
    g_stats.pass_bytes[i] = bytes;
    CU(record(ev[2 * i], st));
    open = i;
    s = st;
  }
  void end() {
    if (open < 0) return;
    record(ev[2 * open + 1], s);  // no throw: runs in a destructor
    g_stats.n_pass = open + 1;
    open = -1;
  }
  // Inside a stream capture a plain cudaEventRecord only orders the capture; the graph gets
  // an event-record node (so the timing events fire on every replay) with the External flag.
  static cudaError_t record(cudaEvent_t e, cudaStream_t st) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusActive)
      return cudaEventRecordWithFlags(e, st, cudaEventRecordExternal);
    return cudaEventRecord(e, st);
  }
  void create_all() {  // before a graph capture: no event creation inside it
    for (auto& e : ev)
      if (!e) CU(cudaEventCreate(&e));
  }
  void resolve() {
    if (g_dry) return;
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
inline int64_t even(int64_t x) { return (x + 1) & ~int64_t(1); }

int64_t ooc_chunk_rows(int n) {  // ~256 MB per staging buffer (TSSVD_OOC_CHUNK_ROWS overrides)
  static const int64_t force = getenv("TSSVD_OOC_CHUNK_ROWS") ? atoll(getenv("TSSVD_OOC_CHUNK_ROWS")) : 0;
  if (force > 0) return force;
  return std::max<int64_t>(256, (int64_t)(256.0 * (1 << 20) / (8.0 * std::max(n, 1))));
}


// ---------------------------------------------------------------- core ----
// Buffers of one Alg. 3/4 run on an (m_local x w) matrix.
struct Core {
  int64_t m_local = 0;
  int w = 0;
  double *part, *npart, *B, *Bp, *lam, *nsq, *sig, *M, *G, *Z, *dz, *tsq, *T, *Rt, *sv, *Ps;
  int *idx, *idx2, *info;
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
    Bp = a.get<double>((size_t)w * (w + 1) / 2);
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
    info = a.get<int>(8);
  }
};

// Host-side counters of a finished call: sweeps of every Jacobi solve, kept ranks.
void note_rank(int64_t r) {
  if (g_stats.n_ranks < 8) g_stats.ranks[g_stats.n_ranks++] = r;
}

// Reads n ints at dev into host (one round trip; dry run: `dry_val` everywhere).
void read_ints(Ctx& c, const int* dev, int n, int* host, int dry_val) {
  if (g_dry) {
    for (int i = 0; i < n; ++i) host[i] = dry_val;
    return;
  }
  int* h = host_ctl();
  CU(cudaMemcpyAsync(h, dev, n * sizeof(int), cudaMemcpyDeviceToHost, c.s));
  CU(cudaStreamSynchronize(c.s));
  std::memcpy(host, h, n * sizeof(int));
}

// Host-mode decision: the discard's slot is read now (its r sizes the next launches).
// Multi-rank: max-allreduce of the guard words first, in the same round trip -- a rank
// whose r or nc differs from another's fails on EVERY rank instead of issuing a
// differently sized collective (a hang).
void decide_now(Ctx& c, int slot, int* r, int* nc, int bound, const char* what) {
  step("sync:%s", what);
  int* sl = c.slot(slot);
  if (g_dry) {
    *r = *nc = bound;
    return;
  }
  int* gw = c.guard() + 8 * slot;
  if (c.dist()) {
    CU(cudaMemcpyAsync(gw, sl + kSlotGuard, 4 * sizeof(int), cudaMemcpyDeviceToDevice, c.s));
    NC(ncclAllReduce(gw, gw, 4, ncclInt32, ncclMax, c.comm->nccl, c.s));
  }
  int* h = host_ctl();
  CU(cudaMemcpyAsync(h, sl, 8 * sizeof(int), cudaMemcpyDeviceToHost, c.s));
  if (c.dist()) CU(cudaMemcpyAsync(h + 8, gw, 4 * sizeof(int), cudaMemcpyDeviceToHost, c.s));
  CU(cudaStreamSynchronize(c.s));
  if (c.dist() && (h[8] != h[kSlotGuard] || h[9] != h[kSlotGuard + 1] || h[10] != h[kSlotGuard + 2] ||
                   h[11] != h[kSlotGuard + 3]))
    fail(TSSVD_ENCCL, "replicated discard decision (%s) differs across ranks (r %d vs max %d)", what, h[0], h[8]);
  if (h[kSlotBad]) fail(TSSVD_ENONFINITE, "non-finite entries in the input (%s)", what);
  *r = h[kSlotR];
  *nc = h[kSlotNc];
}

// End of a call: ONE round trip reads the whole control block (deferred Jacobi
// convergence, device-side decisions, the multi-rank guard and global m).
struct Finish {
  int jinfo[8 * kMaxDeferred];
  int slots[8 * kMaxSlots];
  int64_t m = -1;
};
// the stream part of finish (guard allreduce, one D2H copy of the control block): a CUDA
// graph of the call ends with it
void finish_enqueue(Ctx& c) {
  step("finish");
  if (g_dry) return;
  if (c.dist() && c.nslots > 0) {
    CU(cudaMemcpyAsync(c.guard(), c.slots(), 8 * c.nslots * sizeof(int), cudaMemcpyDeviceToDevice, c.s));
    NC(ncclAllReduce(c.guard(), c.guard(), 8 * c.nslots, ncclInt32, ncclMax, c.comm->nccl, c.s));
  }
  CU(cudaMemcpyAsync(host_ctl(), c.ctl, kCtlInts * sizeof(int), cudaMemcpyDeviceToHost, c.s));
}

void finish_host(Ctx& c, Finish& f) {
  if (g_dry) {
    for (int q = 0; q < c.nslots; ++q) f.slots[8 * q] = f.slots[8 * q + 1] = 1 << 20;
    return;
  }
  int* h = host_ctl();
  CU(cudaStreamSynchronize(c.s));
  std::memcpy(f.jinfo, h, sizeof f.jinfo);
  std::memcpy(f.slots, h + 8 * kMaxDeferred, sizeof f.slots);
  const int* g = h + 8 * kMaxDeferred + 8 * kMaxSlots;
  std::memcpy(&f.m, h + 8 * kMaxDeferred + 16 * kMaxSlots, sizeof(int64_t));
  for (int q = 0; q < c.njinfo; ++q)
    if (g_stats.n_jacobi < 16) g_stats.jacobi_sweeps[g_stats.n_jacobi++] = f.jinfo[8 * q];
  for (int q = 0; q < c.nslots; ++q) note_rank(f.slots[8 * q + kSlotR]);
  if (c.dist())
    for (int q = 0; q < 8 * c.nslots; ++q)
      if (g[q] != f.slots[q])
        fail(TSSVD_ENCCL, "replicated discard decision %d differs across ranks", q / 8);
  for (int q = 0; q < c.nslots; ++q)
    if (f.slots[8 * q + kSlotBad]) fail(TSSVD_ENONFINITE, "non-finite entries in the input (A or Omega)");
  for (int q = 0; q < c.njinfo; ++q)
    if (!f.jinfo[8 * q + 1]) fail(TSSVD_ENOCONV, "Jacobi solve %d not converged in %d sweeps", q, f.jinfo[8 * q]);
}

void finish(Ctx& c, Finish& f) {
  finish_enqueue(c);
  finish_host(c, f);
}

// ---- one CUDA graph per call (the device-decision paths: lowrank_svd) -------------
// With every decision on the device, a call is a fixed sequence of kernels, copies and
// NCCL collectives for fixed arguments: it is captured once and replayed (TSSVD_GRAPH=0
// disables).  The key is every argument that reaches a launch (pointers baked into kernel
// parameters and TMA descriptors included); a replay restores the host-side counters the
// capture produced.
struct GraphKey {
  const void* p[10];
  int64_t v[10];
  double wp;
  bool operator==(const GraphKey& o) const { return std::memcmp(this, &o, sizeof *this) == 0; }
};
struct GraphEntry {
  GraphKey key;
  cudaGraphExec_t exec = nullptr;
  tssvd_stats stats;
  int njinfo = 0, nslots = 0;
  int aux[4] = {0, 0, 0, 0};  // call-specific host values the replay needs
};
thread_local std::vector<GraphEntry> g_graphs;
constexpr size_t kMaxGraphs = 8;

bool graphs_on() {
  static const bool on = !getenv("TSSVD_GRAPH") || atoi(getenv("TSSVD_GRAPH")) != 0;
  return on;
}
GraphEntry* graph_find(const GraphKey& k) {
  for (auto& e : g_graphs)
    if (e.key == k) return &e;
  return nullptr;
}
GraphEntry* graph_store(const GraphKey& k, cudaGraphExec_t ex) {
  if (g_graphs.size() >= kMaxGraphs) {
    cudaGraphExecDestroy(g_graphs.front().exec);
    g_graphs.erase(g_graphs.begin());
  }
  g_graphs.push_back(GraphEntry{});
  g_graphs.back().key = k;
  g_graphs.back().exec = ex;
  return &g_graphs.back();
}

// One-sided Jacobi rotation threshold for columns of `rows` dot-product rows:
// |x_p.x_q| > tol |x_p||x_q|, tol = max(8, 2 sqrt(rows)) eps -- LAPACK dgesvj's
// sqrt(M) eps with a factor 2 of margin over the dot products' rounding noise (an
// n eps threshold let the orthonormality of U drift to 1.1e-13 at r = 128).
inline double jacobi_tol(int rows) { return std::max(8.0, 2.0 * std::sqrt((double)rows)) * kEps; }

// Eigendecomposition of the PSD matrix B (n x n, ld n) in place: eigenvector j
// (unit, descending eigenvalue) at B + j*n; slots past the solver's k are zero.
// Pivots below trunc_rel * max diag are dropped (numerically null directions;
// reading R13).  sync = true: one round trip returns k (it sizes the next GEMM);
// sync = false: returns the bound n, convergence is checked at the end of the call.
// *nf_flag receives the device address of the solve's non-finite flag.
// Alg. 4 step 8 on Z = Y^* Y ~ I (n <= 160): tridiagonal QL (tridiag_eig.cu), which deflates
// regardless of Z's clustered spectrum (one-sided Jacobi needs 11-15 sweeps there).  Measured:
// time-neutral against Jacobi (c2 Z solve 0.48 vs 0.50 ms, c4 equal), U's orthonormality after
// pass 2 three times better (c2 3.2e-15 vs 9.3e-15, c4 4.4e-15 vs 1.4e-14).
// TSSVD_ZEIG=jacobi restores the Jacobi solve (A/B runs).
// Below 48 columns Jacobi is faster (c3's 25-column Z: ~50 us in 2-5 sweeps vs 135 us for QL,
// whose serial chase and reduction barriers do not shrink with n as fast).
static bool z_by_ql(int n) {
  static const bool jac = getenv("TSSVD_ZEIG") && strcmp(getenv("TSSVD_ZEIG"), "jacobi") == 0;
  return !jac && n >= 48 && n <= kTridiagMax;
}

int eig(Ctx& c, Core& b, double* B, int n, double* vals, double trunc_rel, bool sync, const int** nf_flag,
        const char* what) {
  step("eig:%s", what);
  int* info = sync ? b.info : c.next_info();
  {
    Pass t(c.s, TSSVD_PASS_JACOBI, 0, 0);
    if (what[0] == 'Z' && z_by_ql(n))
      KL(launch_tridiag_eig(B, n, n, trunc_rel, B, n, vals, info, c.s));
    else
      KL(launch_jacobi_eig(B, n, n, jacobi_tol(n), trunc_rel, c.max_sweeps, B, n, vals, info, c.s));
  }
  *nf_flag = info + 6;
  if (!sync) return n;
  step("sync:k_%s", what);
  int h[7];
  read_ints(c, info, 7, h, n);
  if (g_dry) return n;
  if (g_stats.n_jacobi < 16) g_stats.jacobi_sweeps[g_stats.n_jacobi++] = h[0];
  if (h[6]) fail(TSSVD_ENONFINITE, "non-finite entries in the input (Gram diagonal)");
  if (!h[1]) fail(TSSVD_ENOCONV, "Jacobi eig (N=%d) not converged in %d sweeps", n, h[0]);
  return h[2];
}

// Result of one Alg. 3/4 run: `bound` columns were written (host shape); the kept
// rank itself is slot(slot)[kSlotR] (known on the host only after finish(), unless
// exact).  The factor columns [rank, bound) are zeros.
struct CoreOut {
  int bound = 0;
  int slot = -1;
  bool exact = false;
};

// Alg. 3 (passes = 1) or Alg. 4 (passes = 2) on X
// (m_local x w, ldx; row-sharded over the communicator when dist, replicated
// otherwise).  U (m_local x w capacity, ldu) receives U[:, :r]; may alias X.
// sigma[:r], V (w x r, ldv) replicated.
// devmode: every rank decision stays on the device (shapes sized by the bound w,
// zero columns past the device count; no host round trip at all).  Otherwise
// the eigensolver's k and the first discard's r are read back (they size the
// dominant GEMMs of a wide core); the second discard always stays on the device.
CoreOut core(Ctx& c, Core& b, const double* X, int64_t ldx, int64_t m_local, int w, int passes, bool dist,
             double* U, int64_t ldu, double* sigma, double* V, int64_t ldv, bool devmode,
             double* Upack = nullptr) {
  // Upack: the final U is written there packed (leading dimension (bound + 1) & ~1)
  cudaStream_t s = c.s;
  Ctx cd = c;
  if (!dist) cd.comm = nullptr;
  const bool dd = cd.dist();
  step("core:%s:%d:%d", dist ? "sharded" : "local", passes, w);
  // truncation of the eigensolver's pivoted Cholesky (reading R13): directions with
  // lambda <= 0.01 wp lambda_max have Sigma~^2 <= lambda + |E| far below the discard line
  // wp Sigma~_max^2, so they could never be kept; the truncated Schur complement
  // (<= (n-K) trunc lambda_max) moves the kept sigma by ~1e-13 sigma_1 (simulated at c2/c4),
  // three orders below the 1e-10 contract.
  const double trunc = std::max(kEps, 0.01 * c.wp);
  // Step 1 (P:613 / P:646): B = A^* A over the local rows, aggregated across ranks
  // (the packed lower triangle: w(w+1)/2 doubles on the wire).
  step("gram:X");
  {
    Pass t(s, TSSVD_PASS_GRAM_X, (double)m_local * w * (w + 1), 8.0 * m_local * w);
    KL(launch_syrk(X, ldx, m_local, w, b.part, s));
    KL(launch_reduce_sym(b.part, syrk_partials_grid(m_local, w), w, b.B, w, dd ? b.Bp : nullptr, s));
  }
  if (dd) {
    allreduce(cd, b.Bp, (int64_t)w * (w + 1) / 2, "gram");
    KS(unpack_sym(b.Bp, w, b.B, w, s));
  }
  // Step 2 (P:615 / P:648): B = V~ D V~^*  -> k eigenvectors (columns of B's buffer).
  const int* nf = nullptr;
  const int k = eig(c, b, b.B, w, b.lam, trunc, !devmode, &nf, "B");
  CoreOut out;
  if (k == 0) {  // host mode, B == 0: nothing survives (device mode carries zeros instead)
    out.exact = true;
    return out;
  }
  // Step 3 (P:619 / P:652): Y~ = A V~ (k columns) written into U;
  // Step 4 (P:621 / P:654): Sigma~ = column norms (sums of squares fused, then reduced).
  step("xv:%d", k);
  KS(cols_to_m(b.B, w, w, k, b.M, smem_ld(k), mrows_for(w), s));
  {
    Pass t(s, TSSVD_PASS_XV, 2.0 * m_local * w * k, 8.0 * m_local * (w + k));
    KL(launch_gemm_nn(X, ldx, m_local, w, b.M, k, U, ldu, b.npart, nullptr, s));
    KL(launch_reduce_parts(b.npart, gemm_nn_grid(std::max<int64_t>(m_local, 1), k), gemm_nn_part_stride(k), k, b.nsq, s));
  }
  ++g_stats.a_passes;
  allreduce(cd, b.nsq, k, "norms");
  // Step 5 (P:625 / P:658): discard below max * sqrt(wp).
  step("discard:1");
  const int s1 = c.next_slot();
  int* d1 = c.slot(s1);
  KS(discard(b.nsq, k, c.wp, b.sig, b.idx, d1, nf, s));
  int r = k, nc = k;  // device mode: shape bounds
  if (!devmode) {
    decide_now(c, s1, &r, &nc, k, "first discard");
    if (r == 0) {
      out.slot = s1;
      out.exact = true;
      return out;
    }
  }

  if (passes == 1) {
    // Step 6: U = Y~ Sigma^-1 (kept columns, sorted by Sigma, signs fixed), in place.
    step("alg3_out");
    const int ldm = smem_ld(r);
    KS(fill(b.M, (int64_t)mrows_for(nc) * ldm, 0.0, s));
    KS(alg3_out(b.sig, b.idx, d1, r, b.B, w, b.M, ldm, sigma, V, ldv, s));
    step("uout:%d", r);
    {
      Pass t(s, TSSVD_PASS_UOUT, 2.0 * m_local * nc * r, 8.0 * m_local * (nc + r));
      KL(launch_gemm_nn(U, ldu, m_local, nc, b.M, r, Upack ? Upack : U, Upack ? (r + 1) & ~1 : ldu,
                        nullptr, nullptr, s));
    }
    out.bound = r;
    out.slot = s1;
    out.exact = !devmode;
    return out;
  }
  // Steps 6-7: Z = Y^* Y = Sigma~^-1 (Y~^* Y~)_keep Sigma~^-1.
  step("gram:Y:%d", nc);
  {
    Pass t(s, TSSVD_PASS_GRAM_Y, (double)m_local * nc * (nc + 1), 8.0 * m_local * nc);
    KL(launch_syrk(U, ldu, m_local, nc, b.part, s));
    KL(launch_reduce_sym(b.part, syrk_partials_grid(m_local, nc), nc, b.G, nc, dd ? b.Bp : nullptr, s));
  }
  if (dd) {
    allreduce(cd, b.Bp, (int64_t)nc * (nc + 1) / 2, "gram");
    KS(unpack_sym(b.Bp, nc, b.G, nc, s));
  }
  const int rb = r;  // bound of r (exact in host mode)
  step("build_z");
  KS(build_z(b.G, nc, b.idx, b.sig, d1, rb, b.Z, s));
  // Step 8: Z = W D W^*  (W: rb x kz, column-major in b.Z).
  const int* nfz = nullptr;
  const int kz = eig(c, b, b.Z, rb, b.dz, trunc, false, &nfz, "Z");  // Z = Y^T Y ~ I: kz = r
  // Steps 9-10: Q~ = Y W, T = column norms of Q~ (norms only, nothing stored).
  step("qnorm:%d", kz);
  const int ldm_k = smem_ld(kz);
  KS(fill(b.M, (int64_t)mrows_for(nc) * ldm_k, 0.0, s));
  KS(build_m1(b.Z, rb, b.idx, b.sig, d1, rb, kz, b.M, ldm_k, s));
  {
    Pass t(s, TSSVD_PASS_QNORM, 2.0 * m_local * nc * kz, 8.0 * m_local * nc);
    KL(launch_gemm_nn(U, ldu, m_local, nc, b.M, kz, nullptr, 0, b.npart, nullptr, s));
    KL(launch_reduce_parts(b.npart, gemm_nn_grid(std::max<int64_t>(m_local, 1), kz), gemm_nn_part_stride(kz), kz, b.tsq, s));
  }
  allreduce(cd, b.tsq, kz, "norms");
  // Step 11: discard T below max(T) sqrt(wp) -- r2 stays on the device: every
  // later launch is sized by its bound rb2 = kz (= r, as Z ~ I keeps every direction).
  step("discard:2");
  const int s2 = c.next_slot();
  int* d2 = c.slot(s2);
  KS(discard(b.tsq, kz, c.wp, b.T, b.idx2, d2, nfz, s));
  const int rb2 = kz;
  // Steps 12-14: R = T W^* Sigma~ V~^* = K V~_keep^T with K = T W_keep^T Sigma~
  // (r2 x r); SVD of K by one-sided Jacobi on its columns, K J = P Sigma  =>  V = V~_keep J.
  step("svd:R");
  KS(build_k(b.T, b.idx2, d2, rb2, b.Z, rb, d1, rb, b.sig, b.idx, b.Rt, s));
  {
    Pass t(s, TSSVD_PASS_JACOBI, 0, 0);
    KL(launch_jacobi_svd(b.Rt, rb2, rb, rb2, jacobi_tol(rb2), c.max_sweeps, b.Rt + (size_t)rb2 * rb,
                         rb2 + rb, b.sv, c.next_info(), s));
  }
  KS(svd_out(b.Rt + (size_t)rb2 * rb, rb2 + rb, d2, rb2, d1, b.sv, b.B, w, b.idx, sigma, V, ldv, b.Ps, s));
  // Step 15: U = Q P = Y~[:, :nc] (S W T^-1 P), in place.
  step("uout:%d", rb2);
  const int ldm_r2 = smem_ld(rb2);
  KS(fill(b.M, (int64_t)mrows_for(nc) * ldm_r2, 0.0, s));
  KS(build_m2(b.Z, rb, d1, rb, b.idx, b.sig, b.T, b.idx2, d2, rb2, b.Ps, b.M, ldm_r2, s));
  {
    Pass t(s, TSSVD_PASS_UOUT, 2.0 * m_local * nc * rb2, 8.0 * m_local * (nc + rb2));
    KL(launch_gemm_nn(U, ldu, m_local, nc, b.M, rb2, Upack ? Upack : U, Upack ? (rb2 + 1) & ~1 : ldu,
                      nullptr, nullptr, s));
  }
  out.bound = rb2;
  out.slot = s2;
  return out;
}

// ------------------------------------------------------------ wide core ----
// Alg. 3/4 for 256 < w <= 2048 (the paper's n = 2000 workloads, Tables 3-5 / 19-21).  The
// same steps as core(); what changes is the shape of the work:
//   * Grams: block columns of 128 by the A^T Y kernel (gemm_tn with Y = the panel of the
//     same matrix), lower block columns only, then mirrored;
//   * products with more than 256 columns (Y~ = A V~, Q~ norms, U = Y~ M2): column panels
//     of <= 256 through gemm_nn; Y~ lives in the workspace (m_local x K), so the final U may
//     still alias A (A is not read after the A V~ pass);
//   * the eigensolver / SVD of width > 256: the cooperative solvers of jacobi_wide.cu;
//   * host decisions for k and r (the panels are sized by them), r' on the device.
constexpr int kWideMax = 2048, kGramPanel = 128;
// column-panel width of the wide products (TSSVD_WIDE_PANEL overrides, experiments)
int wide_panel() {
  // 96: measured on the paper's Table 3 matrix (1e6 x 2000; tools/nn_bench.py + bench t3):
  // panels of 256 ran the GEMM at 18 TF (one row block per warp), 96-192 at 32-33 TF;
  // t3 515 -> 400 ms per call
  static const int v = getenv("TSSVD_WIDE_PANEL") ? atoi(getenv("TSSVD_WIDE_PANEL")) : 96;
  return std::max(8, std::min(256, v));
}
constexpr int kPanel = 256;  // buffer bound

struct WideCore {
  int w = 0;
  double *tnpart, *Yw, *B, *Bp, *lam, *nsq, *sig, *Mp, *Mfull, *G, *Z, *dz, *tsq, *T, *Rt, *sv, *Ps, *vj, *jw;
  double* npart;
  int *idx, *idx2, *info;
  int64_t ldyw = 0;
  void alloc(Arena& a, int64_t m, int ww) {
    w = ww;
    const int64_t mm = std::max<int64_t>(m, 1);
    size_t tn = 0;
    for (int j0 = 0; j0 < ww; j0 += kGramPanel)
      tn = std::max(tn, plan_gemm_tn(mm, ww - j0, std::min(kGramPanel, ww - j0)).part_doubles);
    tnpart = a.get<double>(tn);
    ldyw = even(ww);
    Yw = a.get<double>((size_t)mm * ldyw);
    B = a.get<double>((size_t)ww * ww);
    Bp = a.get<double>((size_t)ww * (ww + 1) / 2);
    lam = a.get<double>(ww);
    nsq = a.get<double>(ww);
    sig = a.get<double>(ww);
    Mp = a.get<double>(gemm_nn_m_doubles(ww, kPanel));
    Mfull = a.get<double>((size_t)ww * ww);
    G = a.get<double>((size_t)ww * ww);
    Z = a.get<double>((size_t)ww * ww);
    dz = a.get<double>(ww);
    tsq = a.get<double>(ww);
    T = a.get<double>(ww);
    Rt = a.get<double>((size_t)ww * (3 * ww + 2));
    sv = a.get<double>(ww);
    Ps = a.get<double>((size_t)ww * ww);
    vj = a.get<double>((size_t)ww * ww);
    jw = a.get<double>(jacobi_wide_workspace(ww, 2 * ww + 2));
    size_t nn = 0;
    for (int q = 1; q <= kPanel; ++q) nn = std::max(nn, (size_t)gemm_nn_grid(mm, q) * gemm_nn_part_stride(q));
    npart = a.get<double>(nn);
    idx = a.get<int>(ww);
    idx2 = a.get<int>(ww);
    info = a.get<int>(8);
  }
};

// G (w x w, ld ldg) = X^T X over the local rows: lower block columns of 128 by gemm_tn with
// Y = X's own panel, reduced in a fixed order, mirrored; aggregated (packed) across ranks.
void wide_gram(Ctx& c, Ctx& cd, WideCore& b, const double* X, int64_t ldx, int64_t m_local, int w, double* G,
               int ldg, int pass_kind) {
  cudaStream_t s = c.s;
  {
    Pass t(s, pass_kind, (double)m_local * w * (w + 1), 8.0 * m_local * w);
    for (int j0 = 0; j0 < w; j0 += kGramPanel) {
      const int l = std::min(kGramPanel, w - j0);
      const TnPlan tp = plan_gemm_tn(std::max<int64_t>(m_local, 1), w - j0, l);
      KL(launch_gemm_tn(tp, X + j0, ldx, m_local, w - j0, X + j0, ldx, l, b.tnpart, s));
      KL(launch_reduce_parts_2d(b.tnpart, tp.splits, (int64_t)tp.colblocks * tp.cb * tp.ldz, w - j0, tp.ldz, l,
                                G + (size_t)j0 * ldg + j0, ldg, false, s));
    }
    KS(symmetrize(G, w, ldg, s));
  }
  if (cd.dist()) {
    KS(pack_lower(G, w, ldg, b.Bp, s));
    allreduce(cd, b.Bp, (int64_t)w * (w + 1) / 2, "gram");
    KS(unpack_sym(b.Bp, w, G, ldg, s));
  }
}

// Y (m x c) = X (m x k) M with M given row-major (k x c, ld ldm): column panels of <= 256
void wide_product(Ctx& c, WideCore& b, const double* X, int64_t ldx, int64_t m_local, int k, const double* M,
                  int ldm, int cols, double* Y, int64_t ldy, double* nsq_out, int pass_kind) {
  cudaStream_t s = c.s;
  Pass t(s, pass_kind, 2.0 * m_local * k * cols, 8.0 * m_local * (k + cols));
  const int pw = wide_panel();
  for (int c0 = 0; c0 < cols; c0 += pw) {
    const int cw = std::min(pw, cols - c0);
    KS(rows_to_m(M + c0, ldm, k, cw, b.Mp, smem_ld(cw), mrows_for(k), s));
    KL(launch_gemm_nn(X, ldx, m_local, k, b.Mp, cw, Y ? Y + c0 : nullptr, ldy, nsq_out ? b.npart : nullptr,
                      nullptr, s));
    if (nsq_out)
      KL(launch_reduce_parts(b.npart, gemm_nn_grid(std::max<int64_t>(m_local, 1), cw), gemm_nn_part_stride(cw), cw,
                             nsq_out + c0, s));
  }
}

int wide_eig(Ctx& c, WideCore& b, double* Bm, int n, double* vals, double trunc, bool sync, const int** nf,
             const char* what) {
  step("eig:%s", what);
  int* info = sync ? b.info : c.next_info();
  {
    Pass t(c.s, TSSVD_PASS_JACOBI, 0, 0);
    if (what[0] == 'Z' && z_by_ql(n))
      KL(launch_tridiag_eig(Bm, n, n, trunc, Bm, n, vals, info, c.s));
    else if (n <= 256)
      KL(launch_jacobi_eig(Bm, n, n, jacobi_tol(n), trunc, c.max_sweeps, Bm, n, vals, info, c.s));
    else
      KL(launch_jacobi_eig_wide(Bm, n, n, jacobi_tol(n), trunc, c.max_sweeps, Bm, n, vals, info, b.jw, c.s));
  }
  *nf = info + 6;
  if (!sync) return n;
  step("sync:k_%s", what);
  int h[7];
  read_ints(c, info, 7, h, n);
  if (g_dry) return n;
  if (g_stats.n_jacobi < 16) g_stats.jacobi_sweeps[g_stats.n_jacobi++] = h[0];
  if (h[6]) fail(TSSVD_ENONFINITE, "non-finite entries in the input (Gram diagonal)");
  if (!h[1]) fail(TSSVD_ENOCONV, "Jacobi eig (N=%d) not converged in %d sweeps", n, h[0]);
  return h[2];
}

CoreOut core_wide(Ctx& c, WideCore& b, const double* X, int64_t ldx, int64_t m_local, int w, int passes,
                  bool dist, double* U, int64_t ldu, double* sigma, double* V, int64_t ldv, double* Upack) {
  cudaStream_t s = c.s;
  Ctx cd = c;
  if (!dist) cd.comm = nullptr;
  step("core_wide:%s:%d:%d", dist ? "sharded" : "local", passes, w);
  const double trunc = std::max(kEps, 0.01 * c.wp);  // reading R13, as in core()
  // Step 1 (P:613 / P:646): B = A^* A
  step("gram:X");
  wide_gram(c, cd, b, X, ldx, m_local, w, b.B, w, TSSVD_PASS_GRAM_X);
  // Step 2 (P:615 / P:648): B = V~ D V~^*  (k read back: it sizes the panels)
  const int* nf = nullptr;
  const int k = wide_eig(c, b, b.B, w, b.lam, trunc, true, &nf, "B");
  CoreOut out;
  if (k == 0) {
    out.exact = true;
    return out;
  }
  // Steps 3-4: Y~ = A V~ (k columns, into the workspace) and its column sums of squares
  step("xv:%d", k);
  // M = V~ (w x k row-major, ld k): eigenvector j is contiguous at B + j w
  KS(cols_to_m(b.B, w, w, k, b.Mfull, k, w, s));
  wide_product(c, b, X, ldx, m_local, w, b.Mfull, k, k, b.Yw, b.ldyw, b.nsq, TSSVD_PASS_XV);
  ++g_stats.a_passes;
  allreduce(cd, b.nsq, k, "norms");
  // Step 5: discard (r, nc read back)
  step("discard:1");
  const int s1 = c.next_slot();
  int* d1 = c.slot(s1);
  KS(discard(b.nsq, k, c.wp, b.sig, b.idx, d1, nf, s));
  int r = k, nc = k;
  decide_now(c, s1, &r, &nc, k, "first discard");
  if (r == 0) {
    out.slot = s1;
    out.exact = true;
    return out;
  }
  double* Uo = Upack ? Upack : U;
  if (passes == 1) {  // Step 6: U = Y~ Sigma^-1 (kept columns sorted, signs fixed)
    step("alg3_out");
    KS(fill(b.Mfull, (int64_t)nc * r, 0.0, s));
    KS(alg3_out(b.sig, b.idx, d1, r, b.B, w, b.Mfull, r, sigma, V, ldv, s));
    step("uout:%d", r);
    wide_product(c, b, b.Yw, b.ldyw, m_local, nc, b.Mfull, r, r, Uo, Upack ? (r + 1) & ~1 : ldu, nullptr,
                 TSSVD_PASS_UOUT);
    out.bound = r;
    out.slot = s1;
    out.exact = true;
    return out;
  }
  // Steps 6-7: Z = Sigma~^-1 (Y~^* Y~)_keep Sigma~^-1
  step("gram:Y:%d", nc);
  wide_gram(c, cd, b, b.Yw, b.ldyw, m_local, nc, b.G, nc, TSSVD_PASS_GRAM_Y);
  const int rb = r;
  step("build_z");
  KS(build_z(b.G, nc, b.idx, b.sig, d1, rb, b.Z, s));
  // Step 8: Z = W D W^*
  const int* nfz = nullptr;
  const int kz = wide_eig(c, b, b.Z, rb, b.dz, trunc, false, &nfz, "Z");
  // Steps 9-10: T = column norms of Q~ = Y W (norms only)
  step("qnorm:%d", kz);
  KS(fill(b.Mfull, (int64_t)nc * kz, 0.0, s));
  KS(build_m1(b.Z, rb, b.idx, b.sig, d1, rb, kz, b.Mfull, kz, s));
  wide_product(c, b, b.Yw, b.ldyw, m_local, nc, b.Mfull, kz, kz, nullptr, 0, b.tsq, TSSVD_PASS_QNORM);
  allreduce(cd, b.tsq, kz, "norms");
  // Step 11: discard r' (on the device)
  step("discard:2");
  const int s2 = c.next_slot();
  int* d2 = c.slot(s2);
  KS(discard(b.tsq, kz, c.wp, b.T, b.idx2, d2, nfz, s));
  const int rb2 = kz;
  // Steps 12-14: SVD of K = T W_keep^T Sigma~ (r' x r)
  step("svd:R");
  KS(build_k(b.T, b.idx2, d2, rb2, b.Z, rb, d1, rb, b.sig, b.idx, b.Rt, s));
  {
    Pass t(s, TSSVD_PASS_JACOBI, 0, 0);
    if (rb <= 256 && rb2 <= 256)
      KL(launch_jacobi_svd(b.Rt, rb2, rb, rb2, jacobi_tol(rb2), c.max_sweeps, b.Rt + (size_t)rb2 * rb, rb2 + rb,
                           b.sv, c.next_info(), s));
    else
      KL(launch_jacobi_svd_wide(b.Rt, rb2, rb, rb2, jacobi_tol(rb2), c.max_sweeps, b.Rt + (size_t)rb2 * rb,
                                rb2 + rb, b.sv, c.next_info(), b.jw, s));
  }
  KS(wide_svd_out(b.Rt + (size_t)rb2 * rb, rb2 + rb, d2, rb2, d1, rb, b.sv, b.B, w, b.idx, sigma, V, ldv, b.Ps,
                  b.vj, s));
  // Step 15: U = Q P = Y~[:, :nc] M2
  step("uout:%d", rb2);
  KS(fill(b.Mfull, (int64_t)nc * rb2, 0.0, s));
  KS(wide_build_m2(b.Z, rb, d1, rb, b.idx, b.sig, b.T, b.idx2, d2, rb2, b.Ps, b.Mfull, rb2, s));
  wide_product(c, b, b.Yw, b.ldyw, m_local, nc, b.Mfull, rb2, rb2, Uo, Upack ? (rb2 + 1) & ~1 : ldu, nullptr,
               TSSVD_PASS_UOUT);
  out.bound = rb2;
  out.slot = s2;
  return out;
}

// kept rank of a finished core
int64_t core_rank(const CoreOut& o, const Finish& f) {
  if (o.slot < 0) return 0;
  return f.slots[8 * o.slot + kSlotR];
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
// ---------------------------------------------------------- TSQR cores ----
// Algorithms 1 / 2: the randomized TSQR-based SVD of a tall-skinny X (w <= 128).
struct TsqrCore {
  int w = 0, P = 1;
  double *M0, *Mg, *R1, *R2, *T, *svo, *sv, *work, *Rloc, *Rall, *work2;
  int *mask1, *mask2;
  void alloc(Arena& a, int64_t m, int ww, int nranks) {
    w = ww;
    P = std::max(nranks, 1);
    M0 = a.get<double>((size_t)w * w);
    Mg = a.get<double>(gemm_nn_m_doubles(w, w));
    R1 = a.get<double>((size_t)w * w);
    R2 = a.get<double>((size_t)w * w);
    T = a.get<double>((size_t)w * w);
    svo = a.get<double>((size_t)2 * w * w);
    sv = a.get<double>(w);
    work = a.get<double>(tsqr_workspace_doubles(std::max<int64_t>(m, 1), w));
    Rloc = a.get<double>((size_t)w * w);
    Rall = a.get<double>((size_t)P * w * w);
    work2 = a.get<double>(tsqr_workspace_doubles((int64_t)P * w, w));
    mask1 = a.get<int>(w + 1);
    mask2 = a.get<int>(w + 1);
  }
};

// TSQR of X (m_local x w, in place -> Q) with R (w x w, replicated) to R_out.  Row-sharded
// (dist): each rank's TSQR gives Q_p R_p; the R_p are all-gathered (P w x w, rank order) and
// factored again, identically on every rank: [R_0; ...; R_P-1] = Q' R; Q_p <- Q_p Q'_p (the
// rank's w rows of Q') -- the top of the TSQR tree.
void tsqr_run(Ctx& c, TsqrCore& b, double* X, int64_t ldx, int64_t m_local, int w, bool dd, double* R_out) {
  cudaStream_t s = c.s;
  step("tsqr:%d", w);
  {
    Pass t(s, TSSVD_PASS_TSQR, 4.0 * m_local * w * w, 16.0 * m_local * w);
    KL(launch_tsqr(X, ldx, m_local, w, dd ? b.Rloc : R_out, b.work, s));
  }
  ++g_stats.a_passes;
  if (!dd) return;
  step("allgather:R:%d", w * w);
  if (!g_dry)
    NC(ncclAllGather(b.Rloc, b.Rall, (size_t)w * w, ncclDouble, c.comm->nccl, s));
  KL(launch_tsqr(b.Rall, w, (int64_t)c.comm->nranks * w, w, R_out, b.work2, s));
  step("tsqr_top");
  KS(rows_to_m(b.Rall + (size_t)c.comm->rank * w * w, w, w, w, b.Mg, smem_ld(w), mrows_for(w), s));
  KL(launch_gemm_nn(X, ldx, m_local, w, b.Mg, w, X, ldx, nullptr, nullptr, s));
}

// Alg. 1 (passes = 1) or Alg. 2 (passes = 2) on X (m_local x w, ldx),
// U (may alias X) receives U[:, :r]; sigma[:r], V (w x r, ldv) replicated.  The width of the
// factorization is w, or the device count *wdev <= w (columns past it are zero: the draws of
// the random Omega are then row *wdev - 1 of the tables, ld ldp).  Every decision stays on the
// device (launches sized by w, zero columns past the kept rank).
CoreOut tsqr_core(Ctx& c, TsqrCore& b, const double* X, int64_t ldx, int64_t m_local, int w, const int* wdev,
                  const double* ph, const int* pm, int ldp, int passes, bool dist, double* U, int64_t ldu,
                  double* sigma, double* V, int64_t ldv) {
  cudaStream_t s = c.s;
  Ctx cd = c;
  if (!dist) cd.comm = nullptr;
  const bool dd = cd.dist();
  step("tsqr_core:%s:%d:%d", dist ? "sharded" : "local", passes, w);
  // Step 1 (P:527-529 / P:567-569): B^* = A Omega^* -- every row of A mixed by Omega.
  step("mix");
  const double* ph0 = (!wdev && ldp > 0) ? ph + (size_t)(w - 1) * ldp : ph;
  const int* pm0 = (!wdev && ldp > 0) ? pm + (size_t)(w - 1) * ldp : pm;
  KL(launch_mix_matrix(ph0, pm0, ldp, wdev, w, w, b.M0, w, s));
  KS(rows_to_m(b.M0, w, w, w, b.Mg, smem_ld(w), mrows_for(w), s));
  {
    Pass t(s, TSSVD_PASS_XV, 2.0 * m_local * w * w, 16.0 * m_local * w);
    KL(launch_gemm_nn(X, ldx, m_local, w, b.Mg, w, U, ldu, nullptr, nullptr, s));
  }
  ++g_stats.a_passes;
  // Step 2 (P:531-532 / P:571-573): B^* = Q R (Q~ R~) by TSQR, Q in place in U.
  tsqr_run(cd, b, U, ldu, m_local, w, dd, b.R1);
  // Step 3 (P:534-538 / P:575-579): discard rows of R with |R_jj| < |R_11| wp.
  step("discard:1");
  const int s1 = c.next_slot();
  KL(launch_r_discard(b.R1, w, c.wp, c.slot(s1), b.mask1, s));
  int slot = s1;
  const double* K = b.R1;
  if (passes == 2) {
    // Step 4: Q~ (kept columns) = Q R.
    step("zero_cols");
    KL(launch_zero_cols(U, ldu, m_local, w, b.mask1, s));
    tsqr_run(cd, b, U, ldu, m_local, w, dd, b.R2);
    // Step 5: discard.  Step 6: T = R R~.
    step("discard:2");
    const int s2 = c.next_slot();
    KL(launch_r_discard(b.R2, w, c.wp, c.slot(s2), b.mask2, s));
    KL(launch_tri_mul(b.R2, b.R1, w, b.T, s));
    K = b.T;
    slot = s2;
  }
  // Step 4 / 7 (P:540-543 / P:593-596): R (T) = U~ Sigma V~^* by one-sided Jacobi on the columns
  // of K = R^T (rows of R): K J = P Sigma  =>  U~ = J, V~ = P.
  step("svd:R");
  {
    Pass t(s, TSSVD_PASS_JACOBI, 0, 0);
    KL(launch_jacobi_svd(K, w, w, w, jacobi_tol(w), c.max_sweeps, b.svo, 2 * w, b.sv, c.next_info(), s));
  }
  // Step 5-6 / 8-9 (P:545-549 / P:598-602): V = Omega^-1 V~, U = Q U~ (in place), signs (R5).
  step("tsqr_out");
  KS(fill(b.Mg, (int64_t)mrows_for(w) * smem_ld(w), 0.0, s));
  KL(launch_tsqr_out(b.svo, w, b.sv, b.M0, c.slot(slot) + kSlotR, sigma, V, ldv, b.Mg, smem_ld(w), s));
  step("uout:%d", w);
  {
    Pass t(s, TSSVD_PASS_UOUT, 2.0 * m_local * w * w, 16.0 * m_local * w);
    KL(launch_gemm_nn(U, ldu, m_local, w, b.Mg, w, U, ldu, nullptr, nullptr, s));
  }
  CoreOut out;
  out.bound = w;
  out.slot = slot;
  return out;
}


void check_opts(const tssvd_opts* o) {
  if (!o) fail(TSSVD_EINVAL, "opts is NULL");
  if (o->abi_version != TSSVD_ABI_VERSION) fail(TSSVD_EINVAL, "opts->abi_version %d != %d", o->abi_version, TSSVD_ABI_VERSION);
  if (!(o->working_precision > 0.0 && o->working_precision < 1.0))
    fail(TSSVD_EINVAL, "working precision %g not in (0,1)", o->working_precision);
  if (o->max_jacobi_sweeps < 1) fail(TSSVD_EINVAL, "max_jacobi_sweeps < 1");
  if (o->host_io < 0 || o->host_io > 2) fail(TSSVD_EINVAL, "host_io must be 0, 1 or 2");
}

void set_device(tssvd_comm* comm) {
  if (comm && !g_dry) CU(cudaSetDevice(comm->device));
}

// Global m = sum of m_local over ranks: an int64 allreduce on the device, validated
// in finish() (single rank: known now).  Returns m when known now, else -1.
int64_t global_rows(Ctx& c, int64_t m_local) {
  if (!c.dist()) return m_local;
  step("allreduce:m:1");
  if (g_dry) return -1;
  int64_t* h = reinterpret_cast<int64_t*>(host_ctl() + kCtlInts);  // own staging word (H2D in flight;
  *h = m_local;                                                      // a graph replay restages it)
  CU(cudaMemcpyAsync(c.m64(), h, 8, cudaMemcpyHostToDevice, c.s));
  NC(ncclAllReduce(c.m64(), c.m64(), 1, ncclInt64, ncclSum, c.comm->nccl, c.s));
  return -1;
}

// Device-side rank decisions for a tall-skinny core of width w: always for narrow
// cores (bound-sized launches cost nothing there); wide cores read k and r back
// because they size the dominant GEMMs.  TSSVD_DEVICE_RANK=1/0 forces (experiments).
bool devmode_for(int w) {
  static const int force = getenv("TSSVD_DEVICE_RANK") ? atoi(getenv("TSSVD_DEVICE_RANK")) : -1;
  if (force >= 0) return force != 0;
  return w <= 32;
}

struct TsPlan {
  Core core;
  WideCore wide;
  int* ctl;
  double* a_stage;  // host_io: device copy of A (also holds Y~)
  double* u_pack;   // host_io: U packed (ld (r+1)&~1) for one contiguous D2H copy
  double* sig_stage;
  double* v_stage;
};

size_t plan_tssvd(Arena& a, TsPlan& p, int64_t m_local, int n, const tssvd_opts* o) {
  p.ctl = a.get<int>(kCtlInts);
  if (n <= 256) p.core.alloc(a, m_local, n);
  else p.wide.alloc(a, m_local, n);  // 256 < n <= 2048: m_local x n of workspace for Y~
  if (o && o->host_io) {
    p.a_stage = a.get<double>((size_t)std::max<int64_t>(m_local, 1) * even(n));
    p.u_pack = a.get<double>((size_t)std::max<int64_t>(m_local, 1) * even(n));
    p.sig_stage = a.get<double>(n);
    p.v_stage = a.get<double>((size_t)n * n);
  }
  return a.off;
}

// host_io: A is staged with an even leading dimension, so any lda >= n is accepted
void validate_tall(int64_t m_local, int64_t n, int64_t lda, bool hio) {
  if (m_local < 0) fail(TSSVD_EINVAL, "m_local < 0");
  if (n < 1 || n > kWideMax) fail(TSSVD_EINVAL, "n = %lld must be in [1, %d]", (long long)n, kWideMax);
  if (lda < n || (!hio && (lda & 1)))
    fail(TSSVD_EINVAL, "lda = %lld must be even and >= n (16-byte TMA row strides)", (long long)lda);
}

void tssvd_impl(tssvd_comm* comm, void* stream, int64_t m_local, int64_t n, const double* A,
                int64_t lda, const tssvd_opts* opts, double* U, int64_t ldu, double* sigma,
                double* V, int64_t ldv, int64_t* rank, void* ws, size_t ws_bytes) {
  g_stats = tssvd_stats{};
  check_opts(opts);
  validate_tall(m_local, n, lda, opts->host_io == 1);
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
  c.ctl = p.ctl;
  step("tssvd:%d", opts->orthonormalizations);
  CUR(cudaMemsetAsync(c.ctl, 0, kCtlInts * sizeof(int), c.s));
  const int64_t m_now = global_rows(c, m_local);
  if (m_now >= 0 && m_now < n)
    fail(TSSVD_EINVAL, "m = %lld < n = %lld (the matrix must be tall, P:98-104)", (long long)m_now, (long long)n);
  const double* X = A;
  int64_t ldx = lda;
  double* Ud = U;
  int64_t ldud = ldu;
  double* sigd = sigma;
  double* Vd = V;
  int64_t ldvd = ldv;
  if (hio) {  // stage host A into the workspace (it becomes the in-place U buffer)
    const int64_t lds = even(n);
    step("h2d:A");
    if (m_local > 0) {
      if (lda == lds) CUR(cudaMemcpyAsync(p.a_stage, A, (size_t)m_local * n * 8, cudaMemcpyHostToDevice, c.s));
      else CUR(cudaMemcpy2DAsync(p.a_stage, lds * 8, A, lda * 8, n * 8, m_local, cudaMemcpyHostToDevice, c.s));
    }
    X = p.a_stage;
    ldx = lds;
    Ud = p.a_stage;
    ldud = lds;
    sigd = p.sig_stage;
    Vd = p.v_stage;
    ldvd = n;
  }
  const bool packed = hio && ldu == 0;
  const CoreOut o = n <= 256 ? core(c, p.core, X, ldx, m_local, (int)n, opts->orthonormalizations, true, Ud, ldud,
                                    sigd, Vd, ldvd, devmode_for((int)n), packed ? p.u_pack : nullptr)
                               : core_wide(c, p.wide, X, ldx, m_local, (int)n, opts->orthonormalizations, true, Ud,
                                           ldud, sigd, Vd, ldvd, packed ? p.u_pack : nullptr);
  Finish f;
  finish(c, f);
  if (c.dist() && !g_dry && f.m < n)
    fail(TSSVD_EINVAL, "m = %lld < n = %lld (the matrix must be tall, P:98-104)", (long long)f.m, (long long)n);
  const int64_t r = core_rank(o, f);
  if (hio && r > 0) {  // results D2H: exactly r columns (the factor buffers hold o.bound)
    step("d2h:U");
    if (m_local > 0) {
      const int64_t pb = (o.bound + 1) & ~1, pr = (r + 1) & ~1;
      if (packed && pb == pr)  // one contiguous copy: U with leading dimension (r + 1) & ~1
        CUR(cudaMemcpyAsync(U, p.u_pack, (size_t)m_local * pr * 8, cudaMemcpyDeviceToHost, c.s));
      else if (packed)
        CUR(cudaMemcpy2DAsync(U, pr * 8, p.u_pack, pb * 8, r * 8, m_local, cudaMemcpyDeviceToHost, c.s));
      else
        CUR(cudaMemcpy2DAsync(U, ldu * 8, Ud, ldud * 8, r * 8, m_local, cudaMemcpyDeviceToHost, c.s));
    }
    CUR(cudaMemcpyAsync(sigma, sigd, r * 8, cudaMemcpyDeviceToHost, c.s));
    CUR(cudaMemcpy2DAsync(V, ldv * 8, Vd, ldvd * 8, r * 8, n, cudaMemcpyDeviceToHost, c.s));
    CUR(cudaStreamSynchronize(c.s));
  }
  g_timer.resolve();
  *rank = r;
}

// ------------------------------------- LU-based subspace tracking --
// X (rows x w, ldx; row-sharded when dist) becomes the L of Gaussian elimination with partial
// pivoting, in place (csrc/lu_track.cu), every decision on the device: per column the rank-local
// pivot candidate, a MAX allreduce of its magnitude and a MIN allreduce of the owning rank (ties
// to the lowest rank, then the lowest local row), the pivot row summed across ranks (the owner
// contributes it, the others zeros), the elimination.  The kept count r (first numerically zero
// pivot, reading R21) goes to a decision slot; columns >= r are zero.
CoreOut lu_core(Ctx& c, void* lws, double* X, int64_t ldx, int64_t rows, int w, const int* wdev, bool dist) {
  cudaStream_t s = c.s;
  Ctx cd = c;
  if (!dist) cd.comm = nullptr;
  const bool dd = cd.dist();
  step("lu_core:%s:%d", dist ? "sharded" : "local", w);
  const LuWork lw = lu_carve(lws, rows, w);
  const int rank = dd ? c.comm->rank : 0;
  // no collective between the steps (one rank, or a replicated factor): the whole elimination as
  // one cooperative kernel, bit-identical to the launch-per-step loop below (TSSVD_LU_FUSED=0
  // forces the loop, for A/B runs)
  static const bool fused_ok = !(getenv("TSSVD_LU_FUSED") && strcmp(getenv("TSSVD_LU_FUSED"), "0") == 0);
  if (!dd && fused_ok) {
    for (int j = 0; j < w; ++j) step("lu_col:%d", j);
    const int sl = c.next_slot();
    step("lu_finish");
    KL(lu_fused(lw, X, ldx, rows, w, wdev, c.wp, c.slot(sl), s));
    CoreOut out;
    out.bound = w;
    out.slot = sl;
    return out;
  }
  KL(lu_init(lw, rows, s));
  for (int j = 0; j < w; ++j) {
    step("lu_col:%d", j);
    KL(lu_colmax(lw, X, ldx, rows, j, s));
    if (dd) {
      step("allreduce:lu_max:1");
      if (!g_dry) NC(ncclAllReduce(lw.gbuf, lw.gbuf, 1, ncclDouble, ncclMax, c.comm->nccl, s));
    }
    KL(lu_owner(lw, rank, s));
    if (dd) {
      step("allreduce:lu_owner:1");
      if (!g_dry) NC(ncclAllReduce(lw.obuf, lw.obuf, 1, ncclInt32, ncclMin, c.comm->nccl, s));
    }
    KL(lu_decide(lw, X, ldx, w, j, wdev, c.wp, rank, s));
    if (dd) {
      step("allreduce:lu_row:%d", w + 1);
      if (!g_dry) NC(ncclAllReduce(lw.urow, lw.urow, (size_t)w + 1, ncclDouble, ncclSum, c.comm->nccl, s));
    }
    KL(lu_update(lw, X, ldx, rows, w, j, s));
  }
  const int sl = c.next_slot();
  step("lu_finish");
  KL(lu_finish(lw, X, ldx, rows, w, c.slot(sl), s));
  CoreOut out;
  out.bound = w;
  out.slot = sl;
  return out;
}

// ------------------------------------------------------------- low rank --
struct LrPlan {
  Core tall, small;
  TsqrCore tq_tall, tq_small;  // Alg. 7 (method 1)
  void *lu_tall, *lu_small;     // LU-based tracking (method 2)
  int* ctl;
  double *Qt, *Y, *Z, *tn, *Ut, *sig_tmp, *v_scr, *sig_scr, *Mfin, *sk;
  double *a_stage, *a_stage2, *o_stage, *u_stage, *s_stage, *vo_stage;
  int lp, ldzmax;
};

size_t plan_lowrank(Arena& a, LrPlan& p, int64_t m_local, int n, int l, const tssvd_opts* o, int method = 0,
                    int nranks = 1) {
  p.lp = (l + 1) & ~1;
  p.ldzmax = pad8(l);
  p.ctl = a.get<int>(kCtlInts);
  if (method != 1) {
    p.tall.alloc(a, m_local, l);
    p.small.alloc(a, n, l);
    if (method == 2) {
      p.lu_tall = a.get<char>(lu_workspace_bytes(m_local, l));
      p.lu_small = a.get<char>(lu_workspace_bytes(n, l));
    }
  } else {
    p.tq_tall.alloc(a, m_local, l, nranks);
    p.tq_small.alloc(a, n, l, 1);
  }
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
  // alpha stream-K records: sized for any row count (the out-of-core mode runs it on chunks)
  p.sk = a.get<double>(gemm_nn_scratch_max(n, l));
  p.a_stage2 = nullptr;
  if (o && o->host_io == 2) {  // out-of-core: two chunk-sized staging buffers instead of A
    const int64_t ch = std::min<int64_t>(std::max<int64_t>(m_local, 1), ooc_chunk_rows(n));
    p.a_stage = a.get<double>((size_t)ch * even(n));
    p.a_stage2 = a.get<double>((size_t)ch * even(n));
  }
  if (o && o->host_io) {
    if (o->host_io == 1) p.a_stage = a.get<double>((size_t)std::max<int64_t>(m_local, 1) * even(n));
    p.o_stage = a.get<double>((size_t)n * even(l));
    p.u_stage = a.get<double>((size_t)std::max<int64_t>(m_local, 1) * even(l));  // k <= l columns
    p.s_stage = a.get<double>(l);
    p.vo_stage = a.get<double>((size_t)n * l);
  }
  return a.off;
}

// ---- the tall matrix as a source of row chunks (out-of-core mode, host_io = 2) ----
// In-core, an A-pass is one launch over the resident A.  Streamed, A stays in (pinned) host
// memory and every A-pass walks it in row chunks: a library-owned copy stream moves chunk
// c + 1 into one of two device staging buffers while the call's stream runs the pass's kernel
// on chunk c (events order the reuse).  Row-local passes (alpha: Y = A Q~) write their rows of
// Y; the reduction over rows (beta: A^T Q) accumulates the chunks' fixed-order partial sums in
// chunk order, so the result is deterministic.  PCIe-bound by design: it is for A larger than
// the GPU's memory.
struct ASource {
  bool streamed = false;
  const double* dev = nullptr;  // in-core A (device)
  int64_t ld = 0;
  const double* host = nullptr;  // streamed A (host)
  int64_t hld = 0;
  int64_t m = 0;
  int n = 0;
  int64_t chunk = 0;             // rows per chunk
  double* stage[2] = {nullptr, nullptr};
  int64_t sld = 0;               // staging leading dimension (even)
  cudaStream_t cs = nullptr;
  cudaEvent_t ready[2] = {nullptr, nullptr}, freed[2] = {nullptr, nullptr};
  // f(const double* A_chunk, int64_t ld, int64_t row0, int64_t rows, bool first)
  template <class F>
  void each(Ctx& c, F&& f) {
    if (!streamed) {
      f(dev, ld, 0, m, true);
      return;
    }
    const int64_t nch = m > 0 ? ceil_div(m, chunk) : 0;
    // the staging buffers are free once the stream's earlier work is done (the previous pass
    // may still be reading them): the pass's first copies wait for it
    if (!g_dry && nch > 0) {
      CU(cudaEventRecord(freed[0], c.s));
      CU(cudaStreamWaitEvent(cs, freed[0], 0));
    }
    for (int64_t q = 0; q < nch; ++q) {
      const int b = (int)(q & 1);
      const int64_t r0 = q * chunk, rows = std::min(chunk, m - r0);
      if (!g_dry) {
        if (q >= 2) CU(cudaStreamWaitEvent(cs, freed[b], 0));
        CU(cudaMemcpy2DAsync(stage[b], sld * 8, host + r0 * hld, hld * 8, (size_t)n * 8, rows,
                             cudaMemcpyHostToDevice, cs));
        CU(cudaEventRecord(ready[b], cs));
        CU(cudaStreamWaitEvent(c.s, ready[b], 0));
      }
      f(stage[b], sld, r0, rows, q == 0);
      if (!g_dry) CU(cudaEventRecord(freed[b], c.s));
    }
  }
};

// Z (n x ldo) = sum over ranks of A_p^T Q_p  (Alg. 5 step 5 / Alg. 6 step 1); the
// split-K partials are summed in a fixed order on the device (36 MB per c3 pass
// through L2/HBM, ~15 us), then allreduced WITHOUT the partials' pad columns
// (ldo = r rounded up to even).
int tn_pass(Ctx& c, LrPlan& p, ASource& src, int64_t m_local, int n, int r) {
  step("beta:%d", r);
  const int ldo = (r + 1) & ~1;
  if (m_local > 0) {
    Pass t(c.s, TSSVD_PASS_BETA, 2.0 * m_local * n * r, 8.0 * m_local * (n + r));
    src.each(c, [&](const double* A, int64_t lda, int64_t r0, int64_t rows, bool first) {
      const TnPlan tp = plan_gemm_tn(rows, n, r);
      KL(launch_gemm_tn(tp, A, lda, rows, n, p.Y + r0 * p.lp, p.lp, r, p.tn, c.s));
      KL(launch_reduce_parts_2d(p.tn, tp.splits, (int64_t)tp.colblocks * tp.cb * tp.ldz, n, tp.ldz, r, p.Z, ldo,
                                true, c.s, !first));
    });
  } else {
    KS(fill(p.Z, (int64_t)n * ldo, 0.0, c.s));
  }
  ++g_stats.a_passes;
  allreduce(c, p.Z, (int64_t)n * ldo, "beta");
  return ldo;
}

void lowrank_impl(tssvd_comm* comm, void* stream, int64_t m_local, int64_t n, const double* A,
                  int64_t lda, const double* Omega, int64_t ldo, int64_t l, int iters, int64_t k,
                  const tssvd_opts* opts, double* U, int64_t ldu, double* sigma, double* V,
                  int64_t ldv, int64_t* rank, void* ws, size_t ws_bytes, int method = 0,
                  const double* mph = nullptr, const int* mpm = nullptr) {
  // method 0: Algorithm 8 (Gram-based cores); 1: Algorithm 7 (TSQR-based cores, the random
  // mixing draws per width in the tables mph / mpm, ld l); 2: Algorithm 8 with LU-based subspace
  // tracking in the iterations
  g_stats = tssvd_stats{};
  check_opts(opts);
  if (m_local < 0) fail(TSSVD_EINVAL, "m_local < 0");
  if (n < 2) fail(TSSVD_EINVAL, "n = %lld must be >= 2", (long long)n);
  if (method == 1 && opts->host_io != 0) fail(TSSVD_EINVAL, "lowrank_svd_tsqr takes device pointers (host_io 0)");
  if (method == 1 && (!mph || !mpm)) fail(TSSVD_EINVAL, "phases / perms tables are NULL");
  if (lda < n || (opts->host_io != 1 && (lda & 1)))
    fail(TSSVD_EINVAL, "lda must be even and >= n (16-byte TMA row strides)");
  if (l < 1 || l > 128 || l >= n) fail(TSSVD_EINVAL, "need 0 < l < min(m, n) and l <= 128 (l = %lld)", (long long)l);
  if (iters < 0) fail(TSSVD_EINVAL, "iters < 0");
  if (k < 1 || k > l) fail(TSSVD_EINVAL, "need 0 < k <= l");
  if (ldo < l || ldu < k || ldv < k) fail(TSSVD_EINVAL, "ldo < l, ldu < k or ldv < k");
  if (!rank) fail(TSSVD_EINVAL, "rank is NULL");
  const bool hio = opts->host_io >= 1;
  const bool streamed = opts->host_io == 2;  // out-of-core: A is never resident
  if (!hio && m_local > 0 && !aligned16(A)) fail(TSSVD_EINVAL, "A must be 16-byte aligned");
  if (!hio && m_local > 0 && (!aligned16(U) || (ldu & 1)))
    fail(TSSVD_EINVAL, "U must be 16-byte aligned with an even ldu");
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
  plan_lowrank(a, p, m_local, (int)n, (int)l, opts, method, comm ? comm->nranks : 1);
  c.ctl = p.ctl;
  const bool use_graph = !hio && !g_dry && graphs_on();
  GraphKey key{};
  if (use_graph) {
    const void* ps[10] = {comm, A, Omega, U, sigma, V, ws, stream, mph, mpm};
    const int64_t vs[10] = {m_local, n, lda, ldo, l, iters, k, ldu, ldv,
                            (int64_t)ws_bytes ^ ((int64_t)opts->max_jacobi_sweeps << 48) ^
                                ((int64_t)method << 56) ^ ((int64_t)g_timing << 60)};
    std::memcpy(key.p, ps, sizeof ps);
    std::memcpy(key.v, vs, sizeof vs);
    key.wp = opts->working_precision;
    host_ctl();  // pinned staging allocated outside any capture
    if (g_timing) g_timer.create_all();
    if (GraphEntry* e = graph_find(key)) {  // replay the captured call
      if (c.dist()) *reinterpret_cast<int64_t*>(host_ctl() + kCtlInts) = m_local;
      g_stats = e->stats;
      c.njinfo = e->njinfo;
      c.nslots = e->nslots;
      CU(cudaGraphLaunch(e->exec, c.s));
      Finish f;
      finish_host(c, f);
      if (c.dist() && l >= std::min<int64_t>(f.m, n)) fail(TSSVD_EINVAL, "need l < min(m, n) (P:705-707)");
      *rank = std::min<int64_t>(e->aux[0], f.slots[8 * e->aux[1] + kSlotR]);
      g_timer.resolve();
      return;
    }
    // capture on a library-owned stream (the caller's may be the legacy default stream,
    // which cannot be captured); the graph is launched on the caller's stream
    static thread_local cudaStream_t cap = nullptr;
    if (!cap) CU(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    c.s = cap;
    CU(cudaStreamBeginCapture(c.s, cudaStreamCaptureModeThreadLocal));
  }
  try {
  step("lowrank:%d:%lld:%lld", iters, (long long)l, (long long)k);
  CUR(cudaMemsetAsync(c.ctl, 0, kCtlInts * sizeof(int), c.s));
  const int64_t m_now = global_rows(c, m_local);
  if (m_now >= 0 && l >= std::min<int64_t>(m_now, n)) fail(TSSVD_EINVAL, "need l < min(m, n) (P:705-707)");
  const int N = (int)n, Lc = (int)l;
  const double* Ad = A;
  int64_t ldad = lda;
  const double* Od = Omega;
  int64_t ldod = ldo;
  ASource src;
  src.m = m_local;
  src.n = N;
  if (hio) {
    if (!streamed) {
      step("h2d:A");
      if (m_local > 0)
        CUR(cudaMemcpy2DAsync(p.a_stage, even(n) * 8, A, lda * 8, n * 8, m_local, cudaMemcpyHostToDevice, c.s));
      Ad = p.a_stage;
      ldad = even(n);
    }
    CUR(cudaMemcpy2DAsync(p.o_stage, even(l) * 8, Omega, ldo * 8, l * 8, n, cudaMemcpyHostToDevice, c.s));
    Od = p.o_stage;
    ldod = even(l);
  }
  src.dev = Ad;
  src.ld = ldad;
  if (streamed) {
    step("stream:A");
    src.streamed = true;
    src.host = A;
    src.hld = lda;
    src.chunk = ooc_chunk_rows(N);
    src.sld = even(n);
    src.stage[0] = p.a_stage;
    src.stage[1] = p.a_stage2;
    if (!g_dry) {
      static thread_local cudaStream_t cs = nullptr;
      static thread_local cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
      if (!cs) {
        CU(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        for (auto& e : ev) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      }
      src.cs = cs;
      src.ready[0] = ev[0], src.ready[1] = ev[1], src.freed[0] = ev[2], src.freed[1] = ev[3];
    }
  }
  auto alpha = [&]() {
    step("alpha:%d", Lc);
    Pass t(c.s, TSSVD_PASS_ALPHA, 2.0 * m_local * N * Lc, 8.0 * m_local * (N + Lc));
    src.each(c, [&](const double* Ac, int64_t ldc, int64_t r0, int64_t rows, bool) {
      KL(launch_gemm_nn(Ac, ldc, rows, N, p.Qt, Lc, p.Y + r0 * p.lp, p.lp, nullptr, p.sk, c.s));
    });
    ++g_stats.a_passes;
  };
  // The factorizations: Alg. 3 / 4 (method 0) or Alg. 1 / 2 (method 1).  wprev: the device
  // count of the previous factorization's kept rank = the width of the next one's input (its
  // columns past it are zero; Alg. 1/2 draw their Omega for that width).
  const int* wprev = nullptr;
  auto fact = [&](Core& cb, TsqrCore& tb, double* X, int64_t ldx, int64_t rows, int w, int passes, bool dist,
                  double* sg, double* Vv) -> CoreOut {
    CoreOut o;
    if (method == 1)
      o = tsqr_core(c, tb, X, ldx, rows, w, wprev, mph, mpm, Lc, passes, dist, X, ldx, sg, Vv, Lc);
    else if (method == 2 && passes == 1)  // Alg. 5 steps 4 / 6: L instead of Q
      o = lu_core(c, &cb == &p.tall ? p.lu_tall : p.lu_small, X, ldx, rows, w, wprev, dist);
    else
      o = core(c, cb, X, ldx, rows, w, passes, dist, X, ldx, sg, Vv, Lc, true);
    wprev = c.slot(o.slot) + kSlotR;
    return o;
  };
  // Every decision stays on the device (no host round trip until the end): the
  // launches are sized by the block width l, and columns past a kept rank are zeros.
  // Alg. 5 step 1: Q~_0 = Omega.
  KS(rows_to_m(Od, ldod, N, Lc, p.Qt, smem_ld(Lc), mrows_for(N), c.s));
  for (int it = 0; it < iters; ++it) {
    // step 3: Y_j = A Q~_{j-1}
    alpha();
    // step 4: Y_j = Q_j R_j by Alg. 3 / Alg. 1 (Q_j = U, in place in Y)
    fact(p.tall, p.tq_tall, p.Y, p.lp, m_local, Lc, 1, true, p.sig_scr, p.v_scr);
    // step 5: Y~_j = A^* Q_j
    const int ldz = tn_pass(c, p, src, m_local, N, Lc);
    // step 6: Y~_j = Q~_j R~_j by Alg. 3 / Alg. 1 on the replicated n x l matrix
    fact(p.small, p.tq_small, p.Z, ldz, N, Lc, 1, false, p.sig_scr, p.v_scr);
    step("qt");
    KS(rows_to_m(p.Z, ldz, N, Lc, p.Qt, smem_ld(Lc), mrows_for(N), c.s));
  }
  // step 8: Y = A Q~_i; step 9: Y = Q R by Alg. 4 / Alg. 2
  alpha();
  const CoreOut o3 = fact(p.tall, p.tq_tall, p.Y, p.lp, m_local, Lc, 2, true, p.sig_scr, p.v_scr);
  // Alg. 6 step 1: B^T = A^* Q
  const int ldz = tn_pass(c, p, src, m_local, N, o3.bound);
  // Alg. 6 step 2: B^T = V Sigma U~^* by Alg. 4 / Alg. 2 (reading R6); V in place in Z
  const CoreOut o4 = fact(p.small, p.tq_small, p.Z, ldz, N, o3.bound, 2, false, p.sig_tmp, p.Ut);
  step("canon");
  KS(canon_lowrank(p.Z, ldz, N, p.Ut, Lc, o3.bound, c.slot(o4.slot) + kSlotR, o4.bound, c.s));
  const int kk = (int)std::min<int64_t>(k, o4.bound);
  // Alg. 6 step 3: U = Q U~ (leading kk columns, reading R7)
  step("uout:%d", kk);
  KS(rows_to_m(p.Ut, Lc, o3.bound, kk, p.Mfin, smem_ld(kk), mrows_for(o3.bound), c.s));
  double* Uo = hio ? p.u_stage : U;
  const int64_t lduo = hio ? even(kk) : ldu;  // even: the GEMM stores double2 pairs
  KL(launch_gemm_nn(p.Y, p.lp, m_local, o3.bound, p.Mfin, kk, Uo, lduo, nullptr, nullptr, c.s));
  double* So = hio ? p.s_stage : sigma;
  double* Vo = hio ? p.vo_stage : V;
  const int64_t ldvo = hio ? kk : ldv;
  KS(copy2d(p.sig_tmp, kk, So, kk, 1, kk, c.s));
  KS(copy2d(p.Z, ldz, Vo, ldvo, N, kk, c.s));
  finish_enqueue(c);
  if (use_graph) {  // end of the capture: instantiate, keep, launch
    cudaGraph_t gr = nullptr;
    CU(cudaStreamEndCapture(c.s, &gr));
    cudaGraphExec_t ex = nullptr;
    const cudaError_t ie = cudaGraphInstantiate(&ex, gr, 0);
    cudaGraphDestroy(gr);
    CU(ie);
    GraphEntry* e = graph_store(key, ex);
    e->stats = g_stats;
    e->njinfo = c.njinfo;
    e->nslots = c.nslots;
    e->aux[0] = kk;
    e->aux[1] = o4.slot;
    c.s = static_cast<cudaStream_t>(stream);
    CU(cudaGraphLaunch(ex, c.s));
  }
  Finish f;
  finish_host(c, f);
  if (c.dist() && !g_dry && l >= std::min<int64_t>(f.m, n)) fail(TSSVD_EINVAL, "need l < min(m, n) (P:705-707)");
  const int r = (int)std::min<int64_t>(kk, core_rank(o4, f));
  if (hio && r > 0) {
    step("d2h:U");
    if (m_local > 0)
      CUR(cudaMemcpy2DAsync(U, ldu * 8, Uo, lduo * 8, r * 8, m_local, cudaMemcpyDeviceToHost, c.s));
    CUR(cudaMemcpyAsync(sigma, So, r * 8, cudaMemcpyDeviceToHost, c.s));
    CUR(cudaMemcpy2DAsync(V, ldv * 8, Vo, ldvo * 8, r * 8, N, cudaMemcpyDeviceToHost, c.s));
    CUR(cudaStreamSynchronize(c.s));
  }
  g_timer.resolve();
  *rank = r;
  } catch (...) {
    if (use_graph) {  // a failure inside the capture: end it (the stream leaves capture mode)
      cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
      if (cudaStreamIsCapturing(c.s, &st) == cudaSuccess && st != cudaStreamCaptureStatusNone) {
        cudaGraph_t gr = nullptr;
        cudaStreamEndCapture(c.s, &gr);
        if (gr) cudaGraphDestroy(gr);
      }
      cudaGetLastError();
      c.s = static_cast<cudaStream_t>(stream);
    }
    throw;
  }
}

// ------------------------------------------------ Alg. 1 / 2 (tsqr_svd) --
struct TqPlan {
  TsqrCore core;
  int* ctl;
};

size_t plan_tsqr(Arena& a, TqPlan& p, int64_t m_local, int n, int nranks) {
  p.ctl = a.get<int>(kCtlInts);
  p.core.alloc(a, m_local, n, nranks);
  return a.off;
}

constexpr int kTsqrMax = 128;

void tsqr_impl(tssvd_comm* comm, void* stream, int64_t m_local, int64_t n, const double* A, int64_t lda,
               const double* phases, const int* perms, const tssvd_opts* opts, double* U, int64_t ldu,
               double* sigma, double* V, int64_t ldv, int64_t* rank, void* ws, size_t ws_bytes) {
  g_stats = tssvd_stats{};
  check_opts(opts);
  if (opts->host_io != 0) fail(TSSVD_EINVAL, "tsqr_svd takes device pointers (host_io 0)");
  if (m_local < 0) fail(TSSVD_EINVAL, "m_local < 0");
  if (n < 1 || n > kTsqrMax) fail(TSSVD_EINVAL, "n = %lld must be in [1, %d]", (long long)n, kTsqrMax);
  if (opts->orthonormalizations != 1 && opts->orthonormalizations != 2)
    fail(TSSVD_EINVAL, "orthonormalizations must be 1 or 2");
  if (lda < n || (lda & 1) || ldu < n || (ldu & 1)) fail(TSSVD_EINVAL, "lda and ldu must be even and >= n");
  if (ldv < n) fail(TSSVD_EINVAL, "ldv < n");
  if (!rank) fail(TSSVD_EINVAL, "rank is NULL");
  if (n >= 2 && (!phases || !perms)) fail(TSSVD_EINVAL, "phases / perms are NULL");
  if (m_local > 0 && (!aligned16(A) || !aligned16(U))) fail(TSSVD_EINVAL, "A and U must be 16-byte aligned");
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
  TqPlan p;
  plan_tsqr(a, p, m_local, (int)n, comm ? comm->nranks : 1);
  c.ctl = p.ctl;
  step("tsqr_svd:%d", opts->orthonormalizations);
  CUR(cudaMemsetAsync(c.ctl, 0, kCtlInts * sizeof(int), c.s));
  const int64_t m_now = global_rows(c, m_local);
  if (m_now >= 0 && m_now < n)
    fail(TSSVD_EINVAL, "m = %lld < n = %lld (the matrix must be tall, P:98-104)", (long long)m_now, (long long)n);
  const CoreOut o = tsqr_core(c, p.core, A, lda, m_local, (int)n, nullptr, phases, perms, 0,
                              opts->orthonormalizations, true, U, ldu, sigma, V, ldv);
  Finish f;
  finish(c, f);
  if (c.dist() && !g_dry && f.m < n)
    fail(TSSVD_EINVAL, "m = %lld < n = %lld (the matrix must be tall, P:98-104)", (long long)f.m, (long long)n);
  g_timer.resolve();
  *rank = core_rank(o, f);
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
    allreduce(c, buf, count, "user");
    CU(cudaStreamSynchronize(c.s));
  });
}

int tssvd_workspace_size(const tssvd_comm*, int64_t m_local, int64_t n, const tssvd_opts* opts,
                         size_t* bytes) {
  return guarded([&] {
    check_opts(opts);
    validate_tall(m_local, n, n, true);
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

int tsqr_svd_workspace_size(const tssvd_comm* comm, int64_t m_local, int64_t n, const tssvd_opts* opts,
                            size_t* bytes) {
  return guarded([&] {
    check_opts(opts);
    if (m_local < 0 || n < 1 || n > kTsqrMax) fail(TSSVD_EINVAL, "bad sizes (1 <= n <= %d)", kTsqrMax);
    if (!bytes) fail(TSSVD_EINVAL, "bytes is NULL");
    Arena a;
    TqPlan p;
    *bytes = plan_tsqr(a, p, m_local, (int)n, comm ? comm->nranks : 1) + 256;
  });
}

int tsqr_svd(tssvd_comm* comm, void* stream, int64_t m_local, int64_t n, const double* A, int64_t lda,
             const double* phases, const int* perms, const tssvd_opts* opts, double* U, int64_t ldu,
             double* sigma, double* V, int64_t ldv, int64_t* rank, void* workspace, size_t workspace_bytes) {
  return guarded([&] {
    tsqr_impl(comm, stream, m_local, n, A, lda, phases, perms, opts, U, ldu, sigma, V, ldv, rank, workspace,
              workspace_bytes);
  });
}

int lowrank_tsqr_workspace_size(const tssvd_comm* comm, int64_t m_local, int64_t n, int64_t l,
                                const tssvd_opts* opts, size_t* bytes) {
  return guarded([&] {
    check_opts(opts);
    if (m_local < 0 || n < 2 || l < 1 || l > 128 || l >= n) fail(TSSVD_EINVAL, "bad sizes");
    if (!bytes) fail(TSSVD_EINVAL, "bytes is NULL");
    Arena a;
    LrPlan p;
    *bytes = plan_lowrank(a, p, m_local, (int)n, (int)l, opts, 1, comm ? comm->nranks : 1) + 256;
  });
}

int lowrank_lu_workspace_size(const tssvd_comm* comm, int64_t m_local, int64_t n, int64_t l,
                              const tssvd_opts* opts, size_t* bytes) {
  return guarded([&] {
    check_opts(opts);
    if (m_local < 0 || n < 2 || l < 1 || l > 128 || l >= n) fail(TSSVD_EINVAL, "bad sizes");
    if (!bytes) fail(TSSVD_EINVAL, "bytes is NULL");
    Arena a;
    LrPlan p;
    *bytes = plan_lowrank(a, p, m_local, (int)n, (int)l, opts, 2, comm ? comm->nranks : 1) + 256;
  });
}

int lowrank_svd_lu(tssvd_comm* comm, void* stream, int64_t m_local, int64_t n, const double* A, int64_t lda,
                   const double* Omega, int64_t ldo, int64_t l, int iters, int64_t k, const tssvd_opts* opts,
                   double* U, int64_t ldu, double* sigma, double* V, int64_t ldv, int64_t* rank, void* workspace,
                   size_t workspace_bytes) {
  return guarded([&] {
    lowrank_impl(comm, stream, m_local, n, A, lda, Omega, ldo, l, iters, k, opts, U, ldu, sigma, V, ldv, rank,
                 workspace, workspace_bytes, 2);
  });
}

int lowrank_svd_tsqr(tssvd_comm* comm, void* stream, int64_t m_local, int64_t n, const double* A,
                     int64_t lda, const double* Omega, int64_t ldo, int64_t l, int iters, int64_t k,
                     const double* phases, const int* perms, const tssvd_opts* opts, double* U, int64_t ldu,
                     double* sigma, double* V, int64_t ldv, int64_t* rank, void* workspace,
                     size_t workspace_bytes) {
  return guarded([&] {
    lowrank_impl(comm, stream, m_local, n, A, lda, Omega, ldo, l, iters, k, opts, U, ldu, sigma, V, ldv, rank,
                 workspace, workspace_bytes, 1, phases, perms);
  });
}

int tssvd_trace(int problem, int nranks, int64_t m_local, int64_t n, int64_t l, int iters, int64_t k,
                const tssvd_opts* opts, char* buf, size_t buf_len) {
  struct DryScope {  // restores normal operation however the run ends
    DryScope() {
      g_dry = true;
      g_trace.clear();
    }
    ~DryScope() { g_dry = false; }
  };
  return guarded([&] {
    if (problem < 1 || problem > 5)
      fail(TSSVD_EINVAL,
           "problem must be 1 (tssvd), 2 (lowrank_svd), 3 (tsqr_svd), 4 (lowrank_svd_tsqr) or 5 (lowrank_svd_lu)");
    if (nranks < 1 || !buf || buf_len == 0) fail(TSSVD_EINVAL, "bad trace arguments");
    check_opts(opts);
    tssvd_opts o = *opts;
    o.host_io = 0;
    tssvd_comm fc;  // no NCCL communicator: a dry run never calls NCCL
    fc.nranks = nranks;
    fc.rank = 0;
    // placeholder (never dereferenced) device addresses, 16-byte aligned
    double* fake = reinterpret_cast<double*>(uintptr_t(1) << 20);
    void* fws = reinterpret_cast<void*>(uintptr_t(1) << 40);
    const size_t fws_bytes = size_t(1) << 46;
    int64_t rank = 0;
    {
      DryScope dry;
      const int64_t ld = even(n), lk = even(std::max<int64_t>(k, 1));
      tssvd_comm* fcp = nranks > 1 ? &fc : nullptr;
      const int* ifake = reinterpret_cast<const int*>(fake);
      if (problem == 1)
        tssvd_impl(fcp, nullptr, m_local, n, fake, ld, &o, fake, ld, fake, fake, n, &rank, fws, fws_bytes);
      else if (problem == 3)
        tsqr_impl(fcp, nullptr, m_local, n, fake, ld, fake, ifake, &o, fake, ld, fake, fake, n, &rank, fws,
                  fws_bytes);
      else
        lowrank_impl(fcp, nullptr, m_local, n, fake, ld, fake, l, l, iters, k, &o, fake, lk, fake, fake, k, &rank,
                     fws, fws_bytes, problem == 4 ? 1 : (problem == 5 ? 2 : 0), fake, ifake);
    }
    if (g_trace.size() + 1 > buf_len) fail(TSSVD_ENOMEM, "trace needs %zu bytes", g_trace.size() + 1);
    std::memcpy(buf, g_trace.c_str(), g_trace.size() + 1);
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
    CU(launch_reduce_sym(part, syrk_partials_grid(m, (int)n), (int)n, G, (int)ldg, nullptr, s));
    CU(cudaStreamSynchronize(s));
  });
}

size_t tssvd_matmul_workspace(int64_t m, int64_t k, int64_t c) {
  return (gemm_nn_m_doubles((int)k, (int)c) + (size_t)gemm_nn_grid(std::max<int64_t>(m, 1), (int)c) * gemm_nn_part_stride((int)c) +
          gemm_nn_scratch_doubles(m, (int)k, (int)c) + 128) * 8;
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
    double* sk = np + (size_t)gemm_nn_grid(std::max<int64_t>(m, 1), (int)c) * gemm_nn_part_stride((int)c);
    CU(launch_gemm_nn(X, ldx, m, (int)k, Mp, (int)c, Y, ldy, nsq ? np : nullptr, sk, s));
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
    // fixed-order reduction of the split-K partials straight into Z's columns [0, l)
    CU(launch_reduce_parts_2d(part, tp.splits, (int64_t)tp.colblocks * tp.cb * tp.ldz, n, tp.ldz, (int)l,
                              Z, (int)ldz, false, s));
    CU(cudaStreamSynchronize(s));
  });
}

size_t tssvd_sym_eig_workspace(int64_t n) {
  const size_t wide = n > 256 && n <= 2048 ? jacobi_wide_workspace((int)n, (int)n) : 0;
  return ((size_t)n * n + 64 + wide) * 8;
}

int tssvd_sym_eig(void* stream, int64_t n, const double* B, int64_t ldb, double* lambda, double* Vt,
                  int64_t ldv, int max_sweeps, int* sweeps, void* ws, size_t wsb) {
  return guarded([&] {
    if (n < 1 || n > 2048 || ldb < n || ldv < n) fail(TSSVD_EINVAL, "bad sym_eig arguments (1 <= n <= 2048, ldb, ldv >= n)");
    if (wsb < tssvd_sym_eig_workspace(n)) fail(TSSVD_ENOMEM, "sym_eig workspace too small");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    double* vecs = static_cast<double*>(ws);
    int* info = reinterpret_cast<int*>(vecs + (size_t)n * n);
    fill(vecs, (int64_t)n * n, 0.0, s);
    fill(lambda, n, 0.0, s);
    CU(cudaGetLastError());
    // no truncation beyond the noise floor: trunc = eps
    if (n <= 256)
      CU(launch_jacobi_eig(B, (int)ldb, (int)n, jacobi_tol((int)n), kEps, max_sweeps,
                           vecs, (int)n, lambda, info, s));
    else  // the cooperative multi-CTA solver (jacobi_wide.cu)
      CU(launch_jacobi_eig_wide(B, (int)ldb, (int)n, jacobi_tol((int)n), kEps, max_sweeps, vecs, (int)n, lambda,
                                info, reinterpret_cast<double*>(info + 64), s));
    copy2d(vecs, n, Vt, ldv, n, (int)n, s);  // eigenvector j (contiguous) -> row j of Vt
    CU(cudaGetLastError());
    int h[3];
    CU(cudaMemcpyAsync(h, info, 12, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    if (sweeps) *sweeps = h[0];
    if (!h[1]) fail(TSSVD_ENOCONV, "sym_eig did not converge");
  });
}

int tssvd_sym_eig_ql(void* stream, int64_t n, const double* B, int64_t ldb, double* lambda, double* Vt,
                     int64_t ldv, int* iterations, void* ws, size_t wsb) {
  return guarded([&] {
    if (n < 1 || n > kTridiagMax || ldb < n || ldv < n)
      fail(TSSVD_EINVAL, "bad sym_eig_ql arguments (1 <= n <= %d, ldb, ldv >= n)", kTridiagMax);
    if (wsb < tssvd_sym_eig_workspace(n)) fail(TSSVD_ENOMEM, "sym_eig_ql workspace too small");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    double* vecs = static_cast<double*>(ws);
    int* info = reinterpret_cast<int*>(vecs + (size_t)n * n);
    CU(launch_tridiag_eig(B, (int)ldb, (int)n, kEps, vecs, (int)n, lambda, info, s));
    copy2d(vecs, n, Vt, ldv, n, (int)n, s);  // eigenvector j (contiguous) -> row j of Vt
    CU(cudaGetLastError());
    int h[7];
    CU(cudaMemcpyAsync(h, info, 28, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    if (iterations) *iterations = h[0];
    if (h[6]) fail(TSSVD_ENONFINITE, "sym_eig_ql: non-finite input");
    if (!h[1]) fail(TSSVD_ENOCONV, "sym_eig_ql: QL did not deflate within 30 iterations");
  });
}

}  // extern "C"
