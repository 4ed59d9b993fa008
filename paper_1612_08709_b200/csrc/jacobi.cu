// Small replicated cores of Alg. 3/4 on one CTA or one CTA cluster (sm_100a):
//
//   EIG mode -- "Calculate the eigendecomposition B = V D V^*" (PAPER.md:615-617,
//     648-650, 670-672) of a symmetric positive semidefinite Gram matrix:
//       1. diagonally pivoted Cholesky  B = X X^T (X = R^T, n x K), stopped when
//          the largest remaining pivot is <= trunc * max_i B_ii;
//       2. one-sided (Hestenes) Jacobi on the K columns of X:  X J = Y with
//          mutually orthogonal columns, so B = Y Y^T = V diag(|y_j|^2) V^T.
//          Eigenvectors are the normalised columns of Y (no accumulator).
//     The pivoted Cholesky preconditions one-sided Jacobi (Drmac-Veselic):
//     X is graded, Jacobi converges in ~8 sweeps instead of ~20-30 on B, and
//     numerically null directions (which the paper's discard step drops
//     anyway) never enter.
//   SVD mode -- "Calculate the singular value decomposition" of a
//     small matrix K given by columns, rotations accumulated into an appended
//     identity block: K J = P diag(sigma), so K = P diag(sigma) J^T.
//
// Layout.  Every column ("slot") is stored contiguously in shared memory.
// With a cluster of C CTAs the ROWS are split: CTA h holds rows
// [h*Lh, (h+1)*Lh) of every slot.  A Jacobi round rotates all pairs of the
// round-robin (circle) ordering in parallel, one group of G lanes per pair;
// the three dot products of a pair are reduced over the group by an xor
// butterfly (bit-identical in every lane) and, for C > 1, summed over the
// cluster in CTA order through distributed shared memory.  Every reduction has
// a fixed order, so every rank computes bit-identical results from identical
// inputs, and all CTAs of a cluster take identical rotation decisions.
//
// Cost model (B200: 64 FP64 FMA/clk/SM): a round is ~7 L FMAs per pair, spread
// over all 16 warps; C = 1 rounds end in one __syncthreads, C > 1 rounds add one
// DSMEM exchange and one cluster barrier (~600 cycles), so clusters are used
// only when a single CTA's 227 KB cannot hold the columns.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace tsk {

static constexpr int JT = 512;          // threads per CTA
static constexpr int JW = JT / 32;      // warps per CTA
static constexpr int JMAX = 256;        // max slots (columns)
static constexpr int JMAXP = JMAX / 2;  // max pairs per round

struct JacArgs {
  const double* in;
  int ldin;
  int mode;  // 0 = EIG, 1 = SVD
  int n;     // EIG: order of B
  int N;     // SVD: number of columns
  int ldot;  // SVD: rows of K (dot-product rows); EIG: n
  int dpad;  // rows entering dot products, rounded up to even (accumulator starts here)
  int L;     // total rows per slot (EIG: n; SVD: dpad + N)
  int Lh;    // rows per CTA (even)
  int P;     // slot pitch in doubles (= 2 G V >= Lh)
  int V;     // double2 per lane per slot in the sweeps (= template V)
  double tol, trunc;
  int max_sweeps;
  int blk_min;  // warp-block ordering when more than blk_min columns survive the Cholesky
  double* out;
  int ldout;
  double* vals;
  int* info;
};

template <int C>
struct Cl {
  cg::cluster_group c = cg::this_cluster();
  __device__ int rank() const { return C == 1 ? 0 : (int)c.block_rank(); }
  __device__ void sync() {
    if constexpr (C == 1) __syncthreads();
    else c.sync();
  }
  template <class T>
  __device__ T* at(T* p, int q) {
    if constexpr (C == 1) return p;
    else return c.map_shared_rank(p, q);
  }
};

// argmax over a warp of the pivot candidates (v, i), i < 0 = none: larger v wins,
// ties -> lower index.  Positive doubles order like their bit patterns, so the
// max is two 32-bit redux.sync (high word, then low word among the high-word
// winners) and the index a third (min over the winners) -- three reductions
// instead of a 5-level shuffle butterfly over (double, int) pairs.  Candidates
// <= 0 collapse to key 0 (the Cholesky stops there anyway: v = 0 is returned).
__device__ __forceinline__ void warp_argmax(double& v, int& i) {
  const unsigned long long key =
      (i >= 0 && v > 0.0) ? static_cast<unsigned long long>(__double_as_longlong(v)) : 0ull;
  const unsigned hi = static_cast<unsigned>(key >> 32), lo = static_cast<unsigned>(key);
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
  const bool win = i >= 0 && hi == mhi && lo == mlo;
  i = static_cast<int>(__reduce_min_sync(0xffffffffu, win ? static_cast<unsigned>(i) : 0xffffffffu));
  v = __longlong_as_double(static_cast<long long>((static_cast<unsigned long long>(mhi) << 32) | mlo));
}

// DSMEM producer/consumer exchange: remote shared address of `p` in CTA `rank`,
// st.async of one double that signals the remote mbarrier's transaction count.
__device__ __forceinline__ uint32_t mapa_u32(const void* p, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async_f64(uint32_t raddr, double v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];\n" ::"r"(raddr),
               "l"(__double_as_longlong(v)), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITC_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Reciprocal square root: MUFU approximation + two Newton steps.
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const double e = fma(-x * y, y, 1.0);
    y = fma(0.5 * y, e, y);
  }
  return y;
}

// Rotation of the pair (p, q) with Gram entries [[al, ga], [ga, be]], or false
// when the pair is already orthogonal to tolerance (|ga| <= tol sqrt(al be)) or
// both columns are negligible.  With d = be - al:
//   t = tan(theta) = sign(d) 2ga / (|d| + sqrt(d^2 + 4ga^2)),  c = 1/sqrt(1+t^2), s = c t;
// then x_p' = c x_p - s x_q, x_q' = s x_p + c x_q.  d and 2ga are first scaled by
// a power of two (exact) so the squares cannot over/underflow; rsqrt by MUFU +
// two Newton steps (~1 ulp).
__device__ __forceinline__ bool jac_rot(double al, double be, double ga, double tol2, double skip2,
                                        double& c, double& sn) {
  if (!(ga != 0.0 && ga * ga > tol2 * al * be && fmax(al, be) > skip2)) return false;
  double d = be - al, g2 = ga + ga;
  const double big = fmax(fabs(d), fabs(g2));
  const int ex = (int)((__double_as_longlong(big) >> 52) & 0x7ff);        // biased exponent
  const double sc = __longlong_as_double((long long)(2046 - ex) << 52);  // 2^(1023 - ex)
  d *= sc;
  g2 *= sc;
  // With root = sqrt(d^2 + g2^2) and q = |d| + root:  c^2 = q / (2 root) and
  // s = sign(d) g2 / sqrt(2 root q) (the same c, s as t = sign(d) g2 / q,
  // c = 1/sqrt(1+t^2), s = c t), so the two reciprocal square roots run in
  // parallel after the first instead of rsqrt -> rcp -> rsqrt in series.
  const double w = fma(d, d, g2 * g2);
  const double y = rsqrt_nr(w);  // 1 / root
  const double root = w * y;
  const double q = fabs(d) + root;
  const double u = q * (0.5 * y);
  const double v = (root + root) * q;
  c = u * rsqrt_nr(u);
  sn = (d >= 0.0 ? g2 : -g2) * rsqrt_nr(v);
  return true;
}

// Dot products (x.x, y.y, x.y) over this lane's first `elim` double2 rows,
// reduced over an 8-lane group by an xor butterfly (identical in every lane).
template <int V>
__device__ __forceinline__ void dots8(const double2 (&x)[V], const double2 (&y)[V], int elim, double& xx,
                                      double& yy, double& xy) {
  double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0, c0 = 0.0, c1 = 0.0;
#pragma unroll
  for (int e = 0; e < V; ++e)
    if (e < elim) {
      a0 = fma(x[e].x, x[e].x, a0);
      a1 = fma(x[e].y, x[e].y, a1);
      b0 = fma(y[e].x, y[e].x, b0);
      b1 = fma(y[e].y, y[e].y, b1);
      c0 = fma(x[e].x, y[e].x, c0);
      c1 = fma(x[e].y, y[e].y, c1);
    }
  xx = a0 + a1;
  yy = b0 + b1;
  xy = c0 + c1;
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) {
    xx += __shfl_xor_sync(0xffffffffu, xx, o);
    yy += __shfl_xor_sync(0xffffffffu, yy, o);
    xy += __shfl_xor_sync(0xffffffffu, xy, o);
  }
}

#ifdef JAC_PROF  // phase timing of the element rounds (tools/jac_phase.cu only)
__device__ unsigned long long g_jac_phase[8];
#define JP_DECL long long jp_t[5] = {0, 0, 0, 0, 0};
#define JP_T(i) if (threadIdx.x == 0) jp_t[i] = clock64();
#define JP_ACC                                                                     \
  if (threadIdx.x == 0)                                                            \
    for (int i = 1; i < 5; ++i) atomicAdd(&g_jac_phase[i], (unsigned long long)(jp_t[i] - jp_t[i - 1]));
#else
#define JP_DECL
#define JP_T(i)
#define JP_ACC
#endif

template <int C, int G, int V, bool BLK>
__global__ void __launch_bounds__(JT, 1) jacobi_kernel(const JacArgs a) {
  Cl<C> cl;
  const int h = cl.rank();
  extern __shared__ __align__(16) double dsm[];
  __shared__ int s_order[JMAX];  // column k -> slot (EIG: pivot order)
  __shared__ int s_rank[JMAX];
  __shared__ double s_nrm[JMAX];
  __shared__ double s_cand[8][2];  // C > 1: per-CTA pivot candidates (value, index)
  __shared__ double s_red[JW];
  __shared__ __align__(8) uint64_t s_xbar[2];  // C > 1: per-round-parity exchange barriers

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long t_start = clock64();
  if (C > 1 && tid == 0) {
    mbar_init(&s_xbar[0], 1);
    mbar_init(&s_xbar[1], 1);
    fence_mbar_init();
  }
  const int nslots = a.mode == 0 ? a.n : a.N;
  const int P = a.P, Lh = a.Lh;
  TCHECK(nslots <= JMAX && Lh <= P && a.V * 2 * (P / (2 * a.V)) == P);
  const int row0 = h * Lh;                         // first global row held here
  const int nloc = max(0, min(Lh, a.L - row0));    // rows held here
  double* X = dsm;                                 // [nslots][P]
  double* bc = X + (size_t)(nslots + 1) * P;       // [JMAX] pivot row (EIG, C > 1)
  double* xch = bc + JMAX;                         // C > 1: [2][JMAXP][C][4] pair partials
  double* nx = xch + (C > 1 ? 2 * JMAXP * C * 4 : 0);  // [C][JMAX] partial column norms

  // ------------------------------------------------------------ load ----
  for (int r = tid; r < P; r += JT) X[(size_t)nslots * P + r] = 0.0;  // the zero (pad) slot
  if (a.mode == 0) {  // slot i = column i of B (= row i), rows row0..row0+Lh
    for (int s = warp; s < nslots; s += JW)
      for (int r = lane; r < P; r += 32)
        X[s * P + r] = r < nloc ? a.in[(size_t)s * a.ldin + row0 + r] : 0.0;
  } else {  // K's columns, zero rows up to dpad, then the identity accumulator
    for (int s = warp; s < nslots; s += JW)
      for (int r = lane; r < P; r += 32) {
        const int gr = row0 + r;
        double v = 0.0;
        if (r < nloc) v = gr < a.ldot ? a.in[(size_t)s * a.ldin + gr] : (gr - a.dpad == s ? 1.0 : 0.0);
        X[s * P + r] = v;
      }
  }
  __syncthreads();

  int K = nslots;
  bool nonfinite = false;
  if (a.mode == 0) {
    // ---- scale of the truncation: max diagonal of B ----
    const int n = a.n;
    // (a NaN counts as +Inf: a non-finite Gram diagonal -- an Inf/NaN in the streamed matrix,
    // or an overflowing column -- stops the solve with K = 0 and the non-finite flag set)
    double dmax = 0.0;
    for (int i = tid; i < n; i += JT)
      if (i >= row0 && i < row0 + nloc) {
        const double d = X[i * P + (i - row0)];
        dmax = fmax(dmax, isnan(d) ? INFINITY : d);
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    if (lane == 0) s_red[warp] = dmax;
    __syncthreads();
    if (tid == 0) {
      double c = 0.0;
      for (int w = 0; w < JW; ++w) c = fmax(c, s_red[w]);
      for (int q = 0; q < C; ++q) cl.at(&s_cand[0][0], q)[2 * h] = c;
    }
    cl.sync();
    double gmax = 0.0;
    for (int q = 0; q < C; ++q) gmax = fmax(gmax, s_cand[q][0]);
    const double tabs = a.trunc * gmax;
    nonfinite = !(gmax < INFINITY);
    cl.sync();

    bool done = nonfinite;  // non-finite diagonal: K = 0, nothing pivoted
    K = 0;
    if (!done) {
      if (n <= 128) {
        // ---- diagonally pivoted Cholesky with the Schur complement in registers ----
        // (every CTA of a cluster runs it redundantly -- bit-identical -- and keeps its rows)
        // Thread (warp w, lane l) owns S[r][c] for rows r = l + 32 i (i < 4) and
        // slots c = w + 16 j (j < 8).  Step k with pivot p: the owner warp of
        // slot p publishes column p (pcol) and writes X[:, k] = pcol / sqrt(S_pp)
        // (zero on rows pivoted earlier) into slot k; every thread updates its
        // elements S[r][c] -= pcol[r] pcol[c] / S_pp; the owners of diagonal
        // elements publish them for the next argmax.  Two barriers per step.
        double* diag = bc;  // [n]
        double* pcol = nx;  // [n]
        double Sr[8][4];
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int c = warp + JW * j, r = lane + 32 * i;
            Sr[j][i] = (c < n && r < n) ? a.in[(size_t)c * a.ldin + r] : 0.0;  // B symmetric
          }
        // diagonal element r (r = lane + 32 i) lives in slot j = r / 16 of warp r % 16
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int r = lane + 32 * i;
            if (r < n && warp + JW * j == r) diag[r] = Sr[j][i];
          }
        __syncthreads();  // S is in registers: the slots are free for X
        uint32_t rmask = 0, smask = 0;  // pivoted rows (bit i) / slots (bit j) of this thread
        int k = 0;
        for (; k < n; ++k) {
          double bv = -1.0;
          int bi = -1;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int r = lane + 32 * i;
            if (r < n && !((rmask >> i) & 1)) {
              double d = diag[r];
              if (isnan(d)) d = INFINITY;  // non-finite input: pivot it (NaN spreads, caught downstream)
              if (bi < 0 || d > bv) bv = d, bi = r;
            }
          }
          warp_argmax(bv, bi);
          const int p = bi;
          const double dp = bv;
          if (p < 0 || !(dp > tabs)) break;  // uniform over the CTA
          const double rsq = rsqrt_nr(dp);  // MUFU + Newton: no IEEE div / sqrt sequences on the pivot chain
          if ((p % JW) == warp) {  // owner of slot p: publish column p, write X[:, k]
            const int jp = p / JW;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int r = lane + 32 * i;
              double v = 0.0;
#pragma unroll
              for (int j = 0; j < 8; ++j) v = j == jp ? Sr[j][i] : v;
              if (r < n) {
                pcol[r] = v;
                if (r >= row0 && r < row0 + nloc) X[k * P + (r - row0)] = ((rmask >> i) & 1) ? 0.0 : v * rsq;
              }
            }
          }
          if (tid == 0) s_order[k] = k;
          __syncthreads();
          const double inv = rsq * rsq;
          double pr[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int r = lane + 32 * i;
            pr[i] = (r < n && r != p && !((rmask >> i) & 1)) ? pcol[r] * inv : 0.0;
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int c = warp + JW * j;
            if (c < n && c != p && !((smask >> j) & 1)) {
              const double f = pcol[c];
#pragma unroll
              for (int i = 0; i < 4; ++i) Sr[j][i] = fma(-pr[i], f, Sr[j][i]);
            }
          }
          if (((p - lane) & 31) == 0) rmask |= 1u << (p >> 5);
          if ((p % JW) == warp) smask |= 1u << (p / JW);
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const int r = lane + 32 * i;
              if (r < n && warp + JW * j == r && !((rmask >> i) & 1)) diag[r] = Sr[j][i];
            }
          __syncthreads();
        }
        K = k;
        done = true;
      }
    }
    if (!done) {
    // ---- diagonally pivoted Cholesky, right-looking, in place ----
    // Step k with pivot p: X[:, k] := S[:, p] / sqrt(S_pp), stored in slot p
    // (zero on rows pivoted earlier; finalised one step late, when slot p is no
    // longer read), and S[c][c'] -= S[c][p] S[c'][p] / S_pp on the remaining
    // block.  Pivoted rows/slots are tracked in per-thread bit masks: this
    // thread's rows are row0 + lane + 32 j, its warp's slots are warp + JW j'.
    // s_rank[] doubles as the "pivoted" flag per global row during this phase.
    for (int i = tid; i < JMAX; i += JT) s_rank[i] = 0;
    __syncthreads();
    uint32_t rmask = 0, smask = 0;
    int prev = -1;
    int k = 0;
    for (; k < n; ++k) {
      // argmax of the remaining diagonal (ties -> lowest index), every warp redundantly
      double bv = -1.0;
      int bi = -1;
      for (int j = 0; 32 * j < nloc; ++j) {
        const int r = lane + 32 * j;
        if (r < nloc && !((rmask >> j) & 1)) {
          double d = X[(row0 + r) * P + r];
          if (isnan(d)) d = INFINITY;  // non-finite input: pivot it (NaN spreads, caught downstream)
          if (bi < 0 || d > bv) bv = d, bi = row0 + r;
        }
      }
      warp_argmax(bv, bi);
      int p = bi;
      double dp = bv;
      if constexpr (C > 1) {
        if (tid == 0)
          for (int q = 0; q < C; ++q) {
            double* cq = cl.at(&s_cand[0][0], q);
            cq[2 * h] = bv;
            cq[2 * h + 1] = (double)bi;
          }
        cl.sync();
        p = -1, dp = -1.0;
        for (int q = 0; q < C; ++q) {
          const double v = s_cand[q][0];
          const int i = (int)s_cand[q][1];
          if (i >= 0 && (p < 0 || v > dp || (v == dp && i < p))) dp = v, p = i;
        }
      }
      if (p < 0 || !(dp > tabs)) break;  // uniform over the cluster
      const double rsq = rsqrt_nr(dp);
      if (tid == 0) {
        s_order[k] = p;
        s_rank[p] = 1;
        s_nrm[k] = rsq;
      }
      const double inv = rsq * rsq;
      const double* fsrc = X + p * P;  // C == 1: S[s][p] = slot p, row s
      if constexpr (C > 1) {
        // the owner of row p broadcasts S[p][s] (row p of every slot) to the cluster
        if (p >= row0 && p < row0 + nloc)
          for (int s = tid; s < n; s += JT) {
            const double v = X[s * P + (p - row0)];
            for (int q = 0; q < C; ++q) cl.at(bc, q)[s] = v;
          }
        cl.sync();
        fsrc = bc;
      }
      // rank-1 update of the remaining block (slots of this warp, rows of this lane);
      // the pivot column is held in registers, zero on excluded rows (no-op FMA)
      const double* xp = X + p * P;
      double pv[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int r = lane + 32 * j;
        pv[j] = (r < nloc && row0 + r != p && !((rmask >> j) & 1)) ? xp[r] : 0.0;
      }
      for (int jj = 0; warp + JW * jj < n; ++jj) {
        const int s = warp + JW * jj;
        if (s == p || ((smask >> jj) & 1)) continue;
        const double f = fsrc[s] * inv;
        double* xs = X + s * P;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int r = lane + 32 * j;
          if (32 * j < nloc && r < nloc) xs[r] = fma(-pv[j], f, xs[r]);
        }
      }
      // finalise the previous pivot's column: zero on rows pivoted before it, scaled elsewhere
      if (prev >= 0) {
        const double rsq = s_nrm[k - 1];
        double* xs = X + prev * P;
        for (int e = tid; e < nloc; e += JT) {
          const int gr = row0 + e;
          const bool dead = s_rank[gr] != 0 && gr != prev && gr != p;
          xs[e] = dead ? 0.0 : xs[e] * rsq;
        }
      }
      if (p >= row0 && p < row0 + nloc && ((p - row0) & 31) == lane) rmask |= 1u << ((p - row0) >> 5);
      if ((p % JW) == warp) smask |= 1u << (p / JW);
      prev = p;
      __syncthreads();  // (C > 1: the cluster barriers above order the DSMEM traffic)
    }
    K = k;
    if (prev >= 0) {
      const double rsq = s_nrm[K - 1];
      double* xs = X + prev * P;
      for (int e = tid; e < nloc; e += JT) {
        const int gr = row0 + e;
        const bool dead = s_rank[gr] != 0 && gr != prev;
        xs[e] = dead ? 0.0 : xs[e] * rsq;
      }
    }
    }
  } else {
    for (int i = tid; i < nslots; i += JT) s_order[i] = i;
  }
  cl.sync();

  // ---- column norms^2 over the dot rows (partial per CTA, summed in CTA order) ----
  auto col_norms = [&](int ncols) {
    const int dloc = max(0, min(nloc, a.dpad - row0));
    for (int kk = warp; kk < ncols; kk += JW) {
      const double* x = X + s_order[kk] * P;
      double s = 0.0;
      for (int r = lane; r < dloc; r += 32) s = fma(x[r], x[r], s);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0)
        for (int q = 0; q < C; ++q) cl.at(nx, q)[h * JMAX + kk] = s;
    }
    cl.sync();
    for (int kk = tid; kk < ncols; kk += JT) {
      double s = 0.0;
      for (int q = 0; q < C; ++q) s += nx[q * JMAX + kk];
      s_nrm[kk] = s;
    }
    __syncthreads();
  };

  col_norms(K);
  double nu2 = 0.0;
  for (int kk = 0; kk < K; ++kk) nu2 = fmax(nu2, s_nrm[kk]);
  const double skip2 = (kEps * kEps) * nu2;
  const double tol2 = a.tol * a.tol;
  cl.sync();  // s_nrm reads done before it is reused

  // ---------------------------------------------------- Jacobi sweeps ----
  const long long t_chol = clock64();
  int sweep = 0, rounds = 0;
  bool converged = K <= 1;
  if (BLK && C == 1 && K > a.blk_min && K <= 8 * JW) {
    // Warp-block ordering (one CTA).  The K columns are taken four at a time
    // ("blocks", padded to an even number of blocks with the zero slot).  In a
    // block round warp w holds the block pair (T, B) that the circle ordering
    // over blocks assigns it, one column of each per 8-lane group, and rotates
    // the 16 cross pairs (T_g, B_(g+s) mod 4) in four sub-rounds; between
    // sub-rounds the B columns move one group over by a lane shuffle.  The six
    // pairs inside every block are rotated at the first block round of a sweep
    // (three sub-rounds, partner group g xor m).  Every pair is rotated once per
    // sweep (a cyclic ordering, as in the element ordering below), but shared
    // memory is touched only to load and store eight columns per block round,
    // and the CTA synchronises once per block round instead of once per round.
    // Measured on B200 (tools/jac_bench.py): 2x faster than the element
    // ordering at K = 106, ~10% at K = 82, no gain below K ~ 64 (the four
    // sub-rounds' dependency chains, not shared memory, then bound a round).
    static_assert(!BLK || G == 8, "warp-block sweeps use 8-lane groups");
    const int NB = (K + 3) / 4, NBE = NB + (NB & 1), W = NBE / 2;
    for (int k = K + tid; k < 4 * NBE; k += JT) s_order[k] = nslots;
    __syncthreads();
    const int g = lane >> 3, gl = lane & 7;
    const int dloc = min(nloc, a.dpad);
    const int elim = dloc > 2 * gl ? (dloc - 2 * gl + 15) / 16 : 0;
    // the six pairs of the block held in x (group g holds its column g)
    auto inner = [&](double2 (&x)[V]) -> int {
      int r = 0;
#pragma unroll 1
      for (int m = 1; m < 4; ++m) {
        double2 y[V];
#pragma unroll
        for (int e = 0; e < V; ++e) {
          y[e].x = __shfl_xor_sync(0xffffffffu, x[e].x, 8 * m);
          y[e].y = __shfl_xor_sync(0xffffffffu, x[e].y, 8 * m);
        }
        // pair (p, q) = (lower group, higher group): both groups compute the same sums
        const bool lo = g < (g ^ m);
        double xx, yy, xy, c, sn;
        dots8<V>(x, y, elim, xx, yy, xy);
        if (jac_rot(lo ? xx : yy, lo ? yy : xx, xy, tol2, skip2, c, sn)) {
          const double sa = lo ? -sn : sn;  // x_p' = c x_p - s x_q,  x_q' = s x_p + c x_q
#pragma unroll
          for (int e = 0; e < V; ++e)
            x[e] = make_double2(fma(c, x[e].x, sa * y[e].x), fma(c, x[e].y, sa * y[e].y));
          r = 1;
        }
      }
      return r;
    };
    for (; sweep < a.max_sweeps && !converged; ++sweep) {
      int any = 0;
      for (int br = 0; br < NBE - 1; ++br, ++rounds) {
        int rot = 0;
        if (warp < W) {
          const int pT = warp ? 1 + (warp - 1 + br) % (NBE - 1) : 0;
          const int pB = 1 + (NBE - 2 - warp + br) % (NBE - 1);
          if (br == 0) {  // the six pairs inside each of the two blocks
#pragma unroll 1
            for (int hb = 0; hb < 2; ++hb) {
              double2* xc = reinterpret_cast<double2*>(X + s_order[4 * (hb ? pB : pT) + g] * P) + gl;
              double2 x[V];
#pragma unroll
              for (int e = 0; e < V; ++e) x[e] = xc[8 * e];
              if (inner(x)) {
#pragma unroll
                for (int e = 0; e < V; ++e) xc[8 * e] = x[e];
                rot = 1;
              }
            }
            __syncwarp();
          }
          double2* xt = reinterpret_cast<double2*>(X + s_order[4 * pT + g] * P) + gl;
          const double2* xb0 = reinterpret_cast<const double2*>(X + s_order[4 * pB + g] * P) + gl;
          double2 t[V], b[V];
#pragma unroll
          for (int e = 0; e < V; ++e) t[e] = xt[8 * e], b[e] = xb0[8 * e];
#pragma unroll 1
          for (int sr = 0; sr < 4; ++sr) {
            if (sr) {  // group g takes group g+1's B column
              const int src = (lane + 8) & 31;
#pragma unroll
              for (int e = 0; e < V; ++e) {
                b[e].x = __shfl_sync(0xffffffffu, b[e].x, src);
                b[e].y = __shfl_sync(0xffffffffu, b[e].y, src);
              }
            }
            double al, be, ga, c, sn;
            dots8<V>(t, b, elim, al, be, ga);
            if (jac_rot(al, be, ga, tol2, skip2, c, sn)) {
#pragma unroll
              for (int e = 0; e < V; ++e) {
                const double2 tp = t[e], bq = b[e];
                t[e] = make_double2(fma(c, tp.x, -sn * bq.x), fma(c, tp.y, -sn * bq.y));
                b[e] = make_double2(fma(sn, tp.x, c * bq.x), fma(sn, tp.y, c * bq.y));
              }
              rot = 1;
            }
          }
          double2* xb = reinterpret_cast<double2*>(X + s_order[4 * pB + ((g + 3) & 3)] * P) + gl;
#pragma unroll
          for (int e = 0; e < V; ++e) xt[8 * e] = t[e], xb[8 * e] = b[e];
        }
        any |= __syncthreads_or(rot);
      }
      converged = !any;
    }
  } else {
  // Circle (round-robin) ordering on positions 0..NE-1: in round r, pair i is
  // (p, q) = (i ? 1 + (i-1+r) mod (NE-1) : 0, 1 + (NE-2-i+r) mod (NE-1)),
  // advanced incrementally.  An odd K is padded with the all-zero slot
  // `nslots` (it never rotates: its dot products are 0).  Pair i is handled by
  // group i % GPW of warp i / GPW (the launcher guarantees one pass).
  const int NE = K + (K & 1), npairs = NE / 2;
  if (K & 1) s_order[K] = nslots;
  __syncthreads();
  constexpr int GPW = 32 / G;
  const int grp = lane / G, gl = lane % G;
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (grp * G));
  const int gidx = warp * GPW + grp;
  const bool has = gidx < npairs;
  // rows of this lane: 2*gl + 2*G*e (+0, +1), e < V (storage padded with zeros);
  // only rows below dpad (SVD: the matrix part) enter the dot products
  const int dloc = max(0, min(nloc, a.dpad - row0));
  const int elim = dloc > 2 * gl ? (dloc - 2 * gl + 2 * G - 1) / (2 * G) : 0;
  int pos_p = gidx, pos_q = NE - 1 - gidx;  // round 0 (gidx == 0 -> fixed position 0)
  for (; sweep < a.max_sweeps && !converged; ++sweep) {
    int any = 0;
    for (int r = 0; r < NE - 1; ++r, ++rounds) {
      JP_DECL
      JP_T(0)
      int rot = 0;
      double al = 0.0, be = 0.0, ga = 0.0;
      double2 vp[V], vq[V];
      double2* xp = nullptr;
      double2* xq = nullptr;
      if (has) {
        TCHECK(pos_p < NE && pos_q < NE && s_order[pos_p] <= nslots && s_order[pos_q] <= nslots);
        xp = reinterpret_cast<double2*>(X + s_order[pos_p] * P) + gl;
        xq = reinterpret_cast<double2*>(X + s_order[pos_q] * P) + gl;
#pragma unroll
        for (int e = 0; e < V; ++e) vp[e] = xp[G * e], vq[e] = xq[G * e];  // all loads in flight
        double al1 = 0.0, be1 = 0.0, ga1 = 0.0;
#pragma unroll
        for (int e = 0; e < V; ++e) {
          if (e < elim) {
            al = fma(vp[e].x, vp[e].x, al);
            al1 = fma(vp[e].y, vp[e].y, al1);
            be = fma(vq[e].x, vq[e].x, be);
            be1 = fma(vq[e].y, vq[e].y, be1);
            ga = fma(vp[e].x, vq[e].x, ga);
            ga1 = fma(vp[e].y, vq[e].y, ga1);
          }
        }
        al += al1;
        be += be1;
        ga += ga1;
        JP_T(1)
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) {  // xor butterfly: identical sums in every lane
          al += __shfl_xor_sync(gmask, al, o);
          be += __shfl_xor_sync(gmask, be, o);
          ga += __shfl_xor_sync(gmask, ga, o);
        }
        JP_T(2)
      }
      if constexpr (C > 1) {
        // partial dot products to every CTA of the cluster: plain stores locally, st.async
        // to the peers (completing their per-parity exchange mbarrier), then wait for the
        // C-1 remote contributions; summed in CTA order (identical on every CTA)
        const int par = rounds & 1;
        uint64_t* xbar = &s_xbar[par];
        double* xb = xch + ((size_t)par * JMAXP + (has ? gidx : 0)) * C * 4;
        if (tid == 0) mbar_arrive_expect_tx(xbar, (uint32_t)((C - 1) * npairs * 24));
        if (has && gl == 0) {
          xb[h * 4] = al;
          xb[h * 4 + 1] = be;
          xb[h * 4 + 2] = ga;
          for (int qc = 0; qc < C; ++qc) {
            if (qc == h) continue;
            const uint32_t rb = mapa_u32(xbar, qc), rx = mapa_u32(xb + h * 4, qc);
            st_async_f64(rx, al, rb);
            st_async_f64(rx + 8, be, rb);
            st_async_f64(rx + 16, ga, rb);
          }
        }
        __syncthreads();  // local contributions visible
        mbar_wait_cluster(xbar, (uint32_t)((rounds >> 1) & 1));
        al = be = ga = 0.0;
        for (int qc = 0; qc < C; ++qc) al += xb[qc * 4], be += xb[qc * 4 + 1], ga += xb[qc * 4 + 2];
      }
      double c, sn;
      if (has && jac_rot(al, be, ga, tol2, skip2, c, sn)) {
#pragma unroll
        for (int e = 0; e < V; ++e) {
          xp[G * e] = make_double2(fma(c, vp[e].x, -sn * vq[e].x), fma(c, vp[e].y, -sn * vq[e].y));
          xq[G * e] = make_double2(fma(sn, vp[e].x, c * vq[e].x), fma(sn, vp[e].y, c * vq[e].y));
        }
        rot = 1;
      }
      // advance this pair's positions to the next round
      if (pos_p != 0) pos_p = pos_p == NE - 1 ? 1 : pos_p + 1;
      pos_q = pos_q == NE - 1 ? 1 : pos_q + 1;
      JP_T(3)
      any |= __syncthreads_or(rot);
      JP_T(4)
      JP_ACC
    }
    converged = !any;
  }
  }
  const long long t_sweeps = clock64();
  // ------------------------------------------ norms, order, write back ----
  col_norms(K);
  for (int kk = tid; kk < K; kk += JT) {
    const double nj = s_nrm[kk];
    int rk = 0;
    for (int ii = 0; ii < K; ++ii) {
      const double ni = s_nrm[ii];
      rk += (ni > nj) || (ni == nj && ii < kk);
    }
    s_rank[kk] = rk;
  }
  __syncthreads();
  // output column rk: first ldot rows normalised, then the accumulator rows (SVD)
  for (int kk = warp; kk < K; kk += JW) {
    const int rk = s_rank[kk];
    const double n2 = s_nrm[kk];
    const double nj = sqrt(n2);
    const double invn = nj > 0.0 ? 1.0 / nj : 0.0;
    const double* x = X + s_order[kk] * P;
    double* dst = a.out + (size_t)rk * a.ldout;
    for (int r = lane; r < nloc; r += 32) {
      const int gr = row0 + r;
      if (gr < a.ldot) dst[gr] = x[r] * invn;
      else if (gr >= a.dpad) dst[a.ldot + (gr - a.dpad)] = x[r];
    }
    if (lane == 0 && h == 0) a.vals[rk] = a.mode == 0 ? n2 : nj;
  }
  if (a.mode == 0)  // eigenvector slots [K, n) are zero (callers may use all n without reading K)
    for (int e = tid; e < (a.n - K) * nloc; e += JT) {
      const int kk = K + e / nloc, r = e % nloc;
      a.out[(size_t)kk * a.ldout + row0 + r] = 0.0;
      if (r == 0 && h == 0) a.vals[kk] = 0.0;
    }
  if (h == 0 && tid == 0) {
    a.info[0] = sweep;
    a.info[1] = converged ? 1 : 0;
    a.info[2] = K;
    a.info[3] = (int)((t_chol - t_start) >> 4);  // phase timings, units of 16 cycles
    a.info[4] = (int)((t_sweeps - t_chol) >> 4);
    a.info[5] = rounds;
    a.info[6] = nonfinite ? 1 : 0;
  }
  if constexpr (C > 1) cl.sync();  // keep DSMEM alive until every CTA is done with it
}

// ------------------------------------------------------------- launch ----
template <int C, int G, int V, bool BLK>
static cudaError_t jac_go(const JacArgs& a, size_t smem, cudaStream_t s) {
  auto kern = jacobi_kernel<C, G, V, BLK>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(JT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

template <int C, int G, bool BLK = false>
static cudaError_t jac_v(const JacArgs& a, size_t smem, cudaStream_t s) {
  switch (a.V) {
    case 2: return jac_go<C, G, 2, BLK>(a, smem, s);
    case 3: return jac_go<C, G, 3, BLK>(a, smem, s);
    case 4: return jac_go<C, G, 4, BLK>(a, smem, s);
    case 5: return jac_go<C, G, 5, BLK>(a, smem, s);
    case 6: return jac_go<C, G, 6, BLK>(a, smem, s);
    case 7: return jac_go<C, G, 7, BLK>(a, smem, s);
    default: return jac_go<C, G, 8, BLK>(a, smem, s);
  }
}

template <int C>
static cudaError_t jac_g(const JacArgs& a, int g, size_t smem, cudaStream_t s) {
  switch (g) {
    case 4: return jac_v<C, 4>(a, smem, s);
    case 8: return jac_v<C, 8>(a, smem, s);
    default: return jac_v<C, 16>(a, smem, s);
  }
}

// dynamic shared memory (doubles): slots (+ zero slot), pivot row, exchange, norms
static size_t jac_smem(int C, int nslots, int P) {
  return ((size_t)(nslots + 1) * P + JMAX + (C > 1 ? 2 * JMAXP * C * 4 : 0) + (size_t)C * JMAX) * 8;
}

// Round cost model (cycles; B200 measured: DFMA/DADD 7-cycle latency, 2 issue
// cycles per warp-instruction on the 16-lane FP64 unit, SHFL+DADD 35, LDS 29,
// shared-memory bandwidth 128 B/cycle/SM, MUFU f64 ~19; the rotation
// parameters ~230 on the critical path; a cluster round adds an st.async
// exchange through DSMEM and an mbarrier wait that grows with the cluster:
// measured ~1400 cycles at C = 2 and 2100 more at C = 8 than at C = 4
// (n = 200: 6950 vs 4840 cycles per round), modelled as 700 C; so clusters
// only when one CTA cannot hold the columns, and the smallest that can).  A round reads and writes both columns of
// every pair, so one CTA is shared-memory-bandwidth bound.
static double jac_round_cost(int C, int G, int V, int npairs) {
  const int warps = (int)ceil_div(npairs, 32 / G);
  const int per_smsp = (int)ceil_div(warps, 4);
  int lg = 0;
  while ((1 << lg) < G) ++lg;
  const double pipe = 2.0 * per_smsp * (14.0 * V + 3.0 * lg + 35.0);
  const double smem = 2.0 * npairs * (2.0 * G * V) * 16.0 / 128.0 / C;
  const double chain = 60.0 + 9.0 * V + 35.0 * lg + 230.0 + 16.0 * V;
  return std::max(pipe, smem) + chain + (C > 1 ? 700.0 * C : 50.0);  // cluster: calibrated on B200
}

static cudaError_t jac_dispatch(JacArgs a, cudaStream_t s) {
  const int nslots = a.mode == 0 ? a.n : a.N;
  if (nslots <= 0) return cudaSuccess;
  if (nslots > JMAX || a.L > 2 * JMAX) return cudaErrorInvalidValue;
  const size_t budget = dev_info().smem_optin - 8 * 1024;  // static shared + slack
  const int npairs = (nslots + 1) / 2;
  // tuning overrides (experiments only): TSSVD_JAC_G, TSSVD_JAC_C
  static const int force_g = getenv("TSSVD_JAC_G") ? atoi(getenv("TSSVD_JAC_G")) : 0;
  static const int force_c = getenv("TSSVD_JAC_C") ? atoi(getenv("TSSVD_JAC_C")) : 0;
  double best = 1e300;
  int bC = 0, bG = 0, bV = 0, bLh = 0;
  for (int C = 1; C <= 8; C *= 2) {  // 8 = portable cluster limit (SVD of up to 256 x 256)
    const int Lh = (int)((ceil_div(a.L, C) + 1) & ~1);
    for (int G = 4; G <= 16; G *= 2) {
      if (JW * (32 / G) < npairs) continue;  // one pass over the pairs
      if ((force_g && G != force_g) || (force_c && C != force_c)) continue;
      int V = (int)ceil_div(Lh, 2 * G);
      if (V > 8) continue;
      V = std::max(V, 2);
      if (jac_smem(C, nslots, 2 * G * V) > budget) continue;
      const double cost = jac_round_cost(C, G, V, npairs);
      if (cost < best) best = cost, bC = C, bG = G, bV = V, bLh = Lh;
    }
  }
  // warp-block sweeps (one CTA, 8-lane groups) when more than 64 columns may
  // survive the Cholesky, they fit one pass of the 16 warps and one CTA holds
  // them (TSSVD_JAC_BLK=0 disables; K <= 64 falls back to the element ordering)
  static const bool blk_ok = !getenv("TSSVD_JAC_BLK") || atoi(getenv("TSSVD_JAC_BLK")) != 0;
  static const int blk_min = getenv("TSSVD_JAC_BLKMIN") ? atoi(getenv("TSSVD_JAC_BLKMIN")) : 64;
  a.blk_min = blk_min;
  if (blk_ok && !force_g && force_c <= 1 && nslots > blk_min && nslots <= 8 * JW) {
    const int V = std::max(2, (int)ceil_div(a.L, 16));
    if (V <= 8 && jac_smem(1, nslots, 16 * V) <= budget) {
      a.Lh = (a.L + 1) & ~1;
      a.V = V;
      a.P = 16 * V;
      return jac_v<1, 8, true>(a, jac_smem(1, nslots, a.P), s);
    }
  }
  if (!bC) return cudaErrorInvalidValue;
  a.Lh = bLh;
  a.V = bV;
  a.P = 2 * bG * bV;
  const size_t smem = jac_smem(bC, nslots, a.P);
  if (bC == 1) return jac_g<1>(a, bG, smem, s);
  if (bC == 2) return jac_g<2>(a, bG, smem, s);
  if (bC == 4) return jac_g<4>(a, bG, smem, s);
  return jac_g<8>(a, bG, smem, s);
}

cudaError_t launch_jacobi_eig(const double* B, int ldb, int n, double tol, double trunc,
                              int max_sweeps, double* vecs, int ldv, double* vals, int* info,
                              cudaStream_t s) {
  JacArgs a{};
  a.in = B;
  a.ldin = ldb;
  a.mode = 0;
  a.n = n;
  a.N = 0;
  a.ldot = n;
  a.dpad = n;
  a.L = n;
  a.tol = tol;
  a.trunc = trunc;
  a.max_sweeps = max_sweeps;
  a.out = vecs;
  a.ldout = ldv;
  a.vals = vals;
  a.info = info;
  return jac_dispatch(a, s);
}

cudaError_t launch_jacobi_svd(const double* cols, int ldc, int N, int ldot, double tol,
                              int max_sweeps, double* out, int ldout, double* vals, int* info,
                              cudaStream_t s) {
  JacArgs a{};
  a.in = cols;
  a.ldin = ldc;
  a.mode = 1;
  a.n = 0;
  a.N = N;
  a.ldot = ldot;
  a.dpad = (ldot + 1) & ~1;
  a.L = a.dpad + N;
  a.tol = tol;
  a.trunc = 0.0;
  a.max_sweeps = max_sweeps;
  a.out = out;
  a.ldout = ldout;
  a.vals = vals;
  a.info = info;
  return jac_dispatch(a, s);
}

}  // namespace tsk
