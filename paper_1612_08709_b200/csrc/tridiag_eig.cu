// Eigendecomposition of the second-pass Gram Z = Y^* Y (Alg. 4 step 8, P:670-672:
// "Calculate the eigendecomposition Z = W D W^*") by Householder tridiagonalisation and the
// implicit QL iteration with Wilkinson-type shifts, on one CTA (n <= 160, the matrix in
// shared memory).
//
// Why not the one-sided Jacobi of jacobi.cu here: Z = I + E with E graded (its eigenvalues
// spread geometrically from ~1e-15 to ~1e-6 around 1, +/- pairs), and every parallel Jacobi
// ordering converges only linearly on that spectrum -- 11-14 sweeps at c2 (measured on the GPU
// and simulated in numpy for round-robin, odd-even, cyclic and anti-diagonal orderings; only
// the row-cyclic ordering with the graded end first needs 6 sweeps, and it has twice the
// rounds per sweep).  QL deflates an eigenvalue in ~1.3 iterations whatever the clustering;
// on c2's Z (n = 55) it needs 69 iterations / 1875 rotations (numpy model), a chain of
// ~120-cycle FP64 steps on one thread, against ~650 Jacobi rounds of ~1250 cycles.
// Accuracy: backward stable, W^T Z W diagonal to ~n eps ||Z||, W orthonormal to ~n eps --
// what Alg. 4 needs (Q = Y W T^-1 orthonormal to the same level).
//
// Contract (as launch_jacobi_eig): B (n x n, ldb, symmetric PSD) -> k <= n eigenpairs,
// vals[j] descending, eigenvector j (unit) contiguous at vecs + j*ldv; eigenvalues
// <= trunc * max(diag B) are dropped (k = info[2]; slots past k are zero).
// info = {QL iterations, converged, k, -, -, rotations, nonfinite}.  vecs may alias B.
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"

namespace tsk {

static constexpr int TQ_THREADS = 512;

__device__ __forceinline__ double warp_sum_all(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// 1/sqrt(x): MUFU approximation + two Newton steps (no IEEE sqrt/div sequence on the chase)
__device__ __forceinline__ double rsqrt_newton(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
#pragma unroll
  for (int i = 0; i < 2; ++i) y = fma(0.5 * y, fma(-x * y, y, 1.0), y);
  return y;
}

__global__ void __launch_bounds__(TQ_THREADS, 1)
    k_tridiag_eig(const double* B, int ldb, int n, double trunc, double* vecs, int ldv, double* vals, int* info) {
  extern __shared__ __align__(16) double sm[];
  const int LD = n | 1;  // odd row stride: row-strided thread accesses are conflict-light
  double* A = sm;        // the matrix, then Q, then the eigenvectors (row r = component r)
  double* d = A + (size_t)n * LD;
  double* e = d + n;
  double* v = e + n;
  double* p = v + n;
  double* tau = p + n;
  double* rc = tau + n;  // [2][n]: the Givens pairs of a chase, two slots (producer / appliers)
  double* rs = rc + 2 * n;
  __shared__ double s_scale, s_beta[2], s_K;  // s_beta by k parity: warp 0 may run one step ahead
  __shared__ int s_lo[2], s_m[2], s_iters, s_rots, s_conv;
  __shared__ __align__(8) uint64_t s_full[2], s_empty[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long clk0 = clock64();  // phase timing: info[3] / info[4] = kilocycles of the
  long long clk1 = clk0;             // reduction + Q formation / of the QL phase

  // ---- load (lower triangle, mirrored), non-finite check, scale to max diag = 1 ----
  bool bad = false;
  double dmax = 0.0;
  for (int idx = tid; idx < n * n; idx += TQ_THREADS) {
    const int i = idx / n, j = idx - (idx / n) * n;
    const double x = B[(size_t)i * ldb + j];
    bad |= !isfinite(x);  // every entry is checked; the lower triangle is used
    if (j > i) continue;
    A[i * LD + j] = x;
    A[j * LD + i] = x;
    if (i == j) dmax = fmax(dmax, x);
  }
  if (__syncthreads_or(bad)) {
    for (int idx = tid; idx < n * n; idx += TQ_THREADS) vecs[(size_t)(idx / n) * ldv + idx % n] = 0.0;
    for (int j = tid; j < n; j += TQ_THREADS) vals[j] = 0.0;
    if (tid == 0) {
      info[0] = 0, info[1] = 1, info[2] = 0, info[3] = 0, info[4] = 0, info[5] = 0, info[6] = 1;
    }
    return;
  }
  if (tid == 0) s_scale = 0.0;
  __syncthreads();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  if (lane == 0) atomicMax(reinterpret_cast<unsigned long long*>(&s_scale), __double_as_longlong(dmax));
  __syncthreads();
  const double scale = s_scale;  // >= 0: the PSD diagonal (bit order = value order)
  if (scale == 0.0) {            // B == 0 (its diagonal is): nothing survives
    for (int idx = tid; idx < n * n; idx += TQ_THREADS) vecs[(size_t)(idx / n) * ldv + idx % n] = 0.0;
    for (int j = tid; j < n; j += TQ_THREADS) vals[j] = 0.0;
    if (tid == 0) info[0] = 0, info[1] = 1, info[2] = 0, info[3] = 0, info[4] = 0, info[5] = 0, info[6] = 0;
    return;
  }
  const double inv = 1.0 / scale;
  for (int idx = tid; idx < n * LD; idx += TQ_THREADS) A[idx] *= inv;
  __syncthreads();

  // ---- Householder tridiagonalisation: H_k annihilates A[k+2:, k] (k = 0 .. n-3) ----
  for (int k = 0; k + 2 < n; ++k) {
    const int L = n - k - 1;
    double* Ak = A + (size_t)(k + 1) * LD + (k + 1);  // A22 = A[k+1:, k+1:]
    if (warp == 0) {
      double s2 = 0.0;
      for (int i = 1 + lane; i < L; i += 32) {
        const double x = A[(k + 1 + i) * LD + k];
        s2 = fma(x, x, s2);
      }
      s2 = warp_sum_all(s2);  // bit-identical in every lane
      const double x0 = A[(k + 1) * LD + k];
      double beta = 0.0, alpha = x0, v0 = 0.0;
      if (s2 > 0.0) {
        const double nx = sqrt(fma(x0, x0, s2));
        alpha = x0 > 0.0 ? -nx : nx;
        v0 = x0 - alpha;
        beta = 1.0 / (nx * (nx + fabs(x0)));  // 2 / (v^T v)
      }
      for (int i = lane; i < L; i += 32) v[i] = i == 0 ? v0 : A[(k + 1 + i) * LD + k];
      if (lane == 0) {
        s_beta[k & 1] = beta;
        tau[k] = beta;
        e[k] = alpha;
        d[k] = A[k * LD + k];
        A[(k + 1) * LD + k] = v0;  // v_k kept below the diagonal of column k (for Q)
      }
    }
    __syncthreads();
    const double beta = s_beta[k & 1];
    if (beta == 0.0) continue;  // column already reduced (uniform branch)
    // p = beta A22 v: four threads per row; the loop bound is rounded up to whole warps (8 rows)
    // so every lane of a warp reaches the shuffles
    const int L8 = (L + 7) & ~7;
    for (int i = tid >> 2; i < L8; i += TQ_THREADS / 4) {
      double acc = 0.0;
      if (i < L) {
        const double* row = Ak + (size_t)i * LD;
        for (int j = tid & 3; j < L; j += 4) acc = fma(row[j], v[j], acc);
      }
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      if ((tid & 3) == 0 && i < L) p[i] = beta * acc;
    }
    __syncthreads();
    if (warp == 0) {
      double a = 0.0;
      for (int i = lane; i < L; i += 32) a = fma(p[i], v[i], a);
      a = warp_sum_all(a);
      if (lane == 0) s_K = 0.5 * beta * a;
    }
    __syncthreads();
    const double K = s_K;
    // A22 -= v w^T + w v^T, w = p - K v (a warp per row, lanes over the columns)
    for (int i = warp; i < L; i += TQ_THREADS / 32) {
      const double vi = v[i], wi = fma(-K, vi, p[i]);
      double* row = Ak + (size_t)i * LD;
      for (int j = lane; j < L; j += 32) {
        const double vj = v[j], wj = fma(-K, vj, p[j]);
        row[j] -= fma(vi, wj, wi * vj);
      }
    }
    __syncthreads();
  }
  if (tid == 0) {
    if (n >= 2) {
      d[n - 2] = A[(n - 2) * LD + n - 2];
      d[n - 1] = A[(n - 1) * LD + n - 1];
      e[n - 2] = A[(n - 1) * LD + n - 2];
    } else {
      d[0] = A[0];
    }
    e[n - 1] = 0.0;
    if (n < 3) tau[0] = 0.0;
  }
  __syncthreads();

  // ---- Q = H_0 H_1 ... H_{n-3}, accumulated backward in place ----
  if (tid == 0) {
    for (int i = n - 2 < 0 ? 0 : n - 2; i < n; ++i)
      for (int j = n - 2 < 0 ? 0 : n - 2; j < n; ++j) A[i * LD + j] = i == j ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int k = n - 3; k >= 0; --k) {
    const int L = n - k - 1;
    const double beta = tau[k];
    double* Qk = A + (size_t)(k + 1) * LD + (k + 1);
    if (beta != 0.0) {
      // y_j = sum_i v_i Q22[i][j] (v_k in column k below the diagonal)
      const int L8 = (L + 7) & ~7;  // whole warps reach the shuffles
      for (int j = tid >> 2; j < L8; j += TQ_THREADS / 4) {
        double acc = 0.0;
        if (j < L)
          for (int i = tid & 3; i < L; i += 4) acc = fma(A[(k + 1 + i) * LD + k], Qk[(size_t)i * LD + j], acc);
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        acc += __shfl_xor_sync(0xffffffffu, acc, 2);
        if ((tid & 3) == 0 && j < L) p[j] = beta * acc;
      }
      for (int i = tid; i < L; i += TQ_THREADS) v[i] = A[(k + 1 + i) * LD + k];
      __syncthreads();
      for (int i = warp; i < L; i += TQ_THREADS / 32) {
        const double vi = v[i];
        double* row = Qk + (size_t)i * LD;
        for (int j = lane; j < L; j += 32) row[j] = fma(-vi, p[j], row[j]);
      }
      __syncthreads();
    }
    for (int j = tid; j < n - k; j += TQ_THREADS) {  // row and column k of Q: e_k
      A[k * LD + k + j] = j == 0 ? 1.0 : 0.0;
      if (j > 0) A[(k + j) * LD + k] = 0.0;
    }
    __syncthreads();
  }

  clk1 = clock64();
  // ---- implicit QL (tql2) on (d, e); the rotations update Q's columns ----
  // Lane 0 of the last warp computes the chases (a serial chain of Givens steps; every operand it
  // reads is prefetched one step ahead -- a step never reads what the chase wrote before) and
  // hands each chase's Givens pairs to the appliers (the warps holding rows of Q, one row per
  // thread) through two slots with full / empty mbarriers, so applying chase t overlaps
  // computing chase t + 1.
  const int ncons = (n + 31) >> 5;  // applier warps 0 .. ncons - 1 (n <= 160: <= 5)
  constexpr int PW = TQ_THREADS / 32 - 1;
  if (tid == 0) {
    for (int q = 0; q < 2; ++q) {
      mbar_init(&s_full[q], 1);
      mbar_init(&s_empty[q], ncons);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == PW && lane == 0) {
    constexpr double eps = kEps;
    int l = 0, it = 0, t = 0, iters = 0, rots = 0, conv = 1;
    while (l < n) {
      int m = l;
      for (; m < n - 1; ++m)
        if (fabs(e[m]) <= eps * (fabs(d[m]) + fabs(d[m + 1]))) break;
      if (m == l || it >= 30) {
        if (m != l) conv = 0;  // not deflated in 30 iterations (deferred ENOCONV)
        ++l, it = 0;
        continue;
      }
      ++it, ++iters;
      // shift from the leading 2 x 2 block
      double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
      double r = hypot(g, 1.0);
      g = d[m] - d[l] + e[l] / (g + copysign(r, g));
      double s = 1.0, c = 1.0, pp = 0.0;
      const int slot = t & 1;
      if (t >= 2) mbar_wait(&s_empty[slot], (uint32_t)(((t >> 1) - 1) & 1));
      double* crc = rc + slot * n;
      double* crs = rs + slot * n;
      int lo = l, i = m - 1;
      double dip1 = d[m], di = d[m - 1], ei = e[m - 1];  // d[i+1], d[i], e[i] (originals)
      for (; i >= l; --i) {
        const double din = i > l ? d[i - 1] : 0.0, ein = i > l ? e[i - 1] : 0.0;
        const double f = s * ei, b = c * ei;
        const double h = fma(f, f, g * g);
        if (h > 1e-280) {  // the matrix is scaled to max |entry| <= 1: no overflow
          const double ri = rsqrt_newton(h);
          r = h * ri, s = f * ri, c = g * ri;
        } else {
          r = hypot(f, g);
          if (r == 0.0) {  // underflow: rotations m-1 .. i+1 applied, split here
            e[i + 1] = 0.0;
            d[i + 1] = dip1 - pp;
            e[m] = 0.0;
            lo = i + 1;
            break;
          }
          s = f / r, c = g / r;
        }
        e[i + 1] = r;
        crc[i] = c, crs[i] = s;
        g = dip1 - pp;
        const double r2 = fma(di - g, s, 2.0 * c * b);
        pp = s * r2;
        d[i + 1] = g + pp;
        g = fma(c, r2, -b);
        dip1 = di, di = din, ei = ein;
      }
      if (i < l) {
        d[l] = dip1 - pp;
        e[l] = g;
        e[m] = 0.0;
      }
      rots += m - lo;
      if (lo < m) {
        s_lo[slot] = lo, s_m[slot] = m;
        mbar_arrive(&s_full[slot]);
        ++t;
      }
    }
    const int slot = t & 1;  // end marker
    if (t >= 2) mbar_wait(&s_empty[slot], (uint32_t)(((t >> 1) - 1) & 1));
    s_m[slot] = -1;
    mbar_arrive(&s_full[slot]);
    s_iters = iters, s_rots = rots, s_conv = conv;
  } else if (warp < ncons) {
    for (int t = 0;; ++t) {
      const int slot = t & 1;
      mbar_wait(&s_full[slot], (uint32_t)((t >> 1) & 1));
      const int lo = s_lo[slot], m = s_m[slot];
      if (m < 0) break;
      if (tid < n) {  // row tid of Z: rotations m-1 .. lo in order, the next column prefetched
        const double* crc = rc + slot * n;
        const double* crs = rs + slot * n;
        double* zr = A + (size_t)tid * LD;
        double cur = zr[m], gi = zr[m - 1];
        for (int i = m - 1; i >= lo; --i) {
          const double gn = i > lo ? zr[i - 1] : 0.0, c = crc[i], sn = crs[i];
          zr[i + 1] = fma(sn, gi, c * cur);
          cur = fma(c, gi, -sn * cur);
          gi = gn;
        }
        zr[lo] = cur;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[slot]);
    }
  }
  __syncthreads();

  // ---- k, descending order, output ----
  const double thr = trunc;  // scaled: max diag = 1
  int kk = 0;
  for (int j = 0; j < n; ++j) kk += d[j] > thr;
  for (int j = warp; j < n; j += TQ_THREADS / 32) {
    const double lj = d[j];
    int rank = 0;
    for (int i = lane; i < n; i += 32) rank += d[i] > lj || (d[i] == lj && i < j);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
    const bool keep = lj > thr && rank < kk;
    if (lane == 0) vals[rank] = keep ? lj * scale : 0.0;
    double* out = vecs + (size_t)rank * ldv;
    for (int r = lane; r < n; r += 32) out[r] = keep ? A[(size_t)r * LD + j] : 0.0;
  }
  if (tid == 0) {
    const long long clk2 = clock64();
    info[0] = s_iters, info[1] = s_conv, info[2] = kk, info[5] = s_rots, info[6] = 0;
    info[3] = (int)((clk1 - clk0) / 1000), info[4] = (int)((clk2 - clk1) / 1000);
  }
}

size_t tridiag_eig_smem(int n) { return ((size_t)n * (n | 1) + 9 * (size_t)n) * sizeof(double); }

cudaError_t launch_tridiag_eig(const double* B, int ldb, int n, double trunc, double* vecs, int ldv, double* vals,
                               int* info, cudaStream_t s) {
  if (n < 1 || n > kTridiagMax) return cudaErrorInvalidValue;
  const size_t smem = tridiag_eig_smem(n);
  cudaError_t e = cudaFuncSetAttribute(k_tridiag_eig, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_tridiag_eig<<<1, TQ_THREADS, smem, s>>>(B, ldb, n, trunc, vecs, ldv, vals, info);
  return cudaGetLastError();
}

}  // namespace tsk
