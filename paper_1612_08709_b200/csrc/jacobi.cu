// Small replicated cores of Alg. 3/4 on one CTA cluster (sm_100a):
//
//   EIG mode -- "Calculate the eigendecomposition B = V D V^*" (PAPER.md:615-617,
//     648-650, 670-672) of a symmetric positive semidefinite Gram matrix:
//       1. diagonally pivoted Cholesky  B = R^T R, stopped when the largest
//          remaining pivot is <= trunc * max_i B_ii (k <= n rows);
//       2. one-sided (Hestenes) Jacobi on the k columns of R^T:
//          R^T J = X with mutually orthogonal columns, so X = V diag(s) and
//          B = V diag(s^2) V^T on the range kept.  Eigenvectors are the
//          normalised columns of X (no accumulator), eigenvalues s^2.
//     The pivoted Cholesky is the preconditioner of one-sided Jacobi
//     (Drmac-Veselic): R^T is graded, Jacobi converges in ~8 sweeps instead of
//     ~30 on B itself, and columns below trunc (numerically null directions,
//     which the paper's discard step would drop anyway) never enter.
//   SVD mode -- "Calculate the singular value decomposition" of a
//     small matrix given by columns, rotations accumulated into an appended
//     identity block: K J = P diag(sigma), so K = P diag(sigma) J^T.
//
// Storage: all slots (columns) live in the distributed shared memory of a
// cluster of C CTAs (slot s in CTA s % C).  A round of the round-robin
// (circle) ordering rotates N/2 disjoint pairs in parallel, one group of G
// lanes per pair; rounds end with a barrier (cluster barrier when C > 1).
// Rotation test: |x_p^T x_q| > tol ||x_p|| ||x_q||.  Every reduction has a
// fixed order: all ranks compute bit-identical results from identical inputs.
#include <cooperative_groups.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace tsk {

static constexpr int JAC_THREADS = 512;
static constexpr int JAC_WARPS = JAC_THREADS / 32;
static constexpr int JAC_MAXSLOTS = 256;  // per CTA

struct JacShared {
  double red_d[JAC_WARPS];
  int red_i[JAC_WARPS];
  double cta_val[2];  // per-CTA partial results read by the other CTAs
  int cta_idx;
  int flag[3];
  int piv_flag[JAC_MAXSLOTS];
  double nrm[512];
  int rank_out[512];
  int order[512];  // global column index -> slot (EIG: pivot order)
  double bcast[512];  // local copy of the current pivot row
  double mu, thresh, nu2;
  int k;
};

template <int G, int EPG>
__global__ void __launch_bounds__(JAC_THREADS) jacobi_kernel(const double* __restrict__ in,
                                                           int ldin, int mode, int n, int N,
                                                           int ldot, int lacc, double tol,
                                                           double trunc, int max_sweeps,
                                                           double* __restrict__ out, int ldout,
                                                           double* __restrict__ vals,
                                                           int* __restrict__ info) {
  cg::cluster_group cluster = cg::this_cluster();
  const int C = (int)cluster.num_blocks();
  const int me = (int)cluster.block_rank();
  extern __shared__ __align__(16) double jsm[];
  __shared__ JacShared sh;
  auto csync = [&]() {
    if (C == 1) __syncthreads();
    else cluster.sync();
  };
  auto remote = [&](auto* p, int cta) { return C == 1 ? p : cluster.map_shared_rank(p, cta); };

  const int L = ldot + lacc;
  const int lds = (L + 1) & ~1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tid = threadIdx.x;
  // slot s -> CTA s % C, local row s / C
  auto slot_ptr = [&](int s) -> double* { return remote(jsm + (s / C) * lds, s % C); };
  const int nslots = mode == 0 ? n : N;
  const int myslots = (nslots - me + C - 1) / C;

  // ------------------------------------------------------------- load ----
  if (mode == 0) {  // B rows (symmetric): slot i = row i
    for (int ls = warp; ls < myslots; ls += JAC_WARPS) {
      const int i = ls * C + me;
      for (int c = lane; c < lds; c += 32) jsm[ls * lds + c] = c < n ? in[(size_t)i * ldin + c] : 0.0;
    }
  } else {  // given columns + identity accumulator
    for (int ls = warp; ls < myslots; ls += JAC_WARPS) {
      const int j = ls * C + me;
      for (int c = lane; c < lds; c += 32)
        jsm[ls * lds + c] = c < ldot ? in[(size_t)j * ldin + c] : (c - ldot == j ? 1.0 : 0.0);
    }
  }
  for (int i = tid; i < JAC_MAXSLOTS; i += JAC_THREADS) sh.piv_flag[i] = 0;
  if (tid < 3) sh.flag[tid] = 0;
  csync();

  int K = N;
  if (mode == 0) {
    // ---- max diagonal (the scale of the truncation threshold) ----
    double dmax = 0.0;
    for (int ls = tid; ls < myslots; ls += JAC_THREADS) dmax = fmax(dmax, jsm[ls * lds + ls * C + me]);
    for (int o = 16; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    if (lane == 0) sh.red_d[warp] = dmax;
    __syncthreads();
    if (tid == 0) {
      double c = 0.0;
      for (int w = 0; w < JAC_WARPS; ++w) c = fmax(c, sh.red_d[w]);
      sh.cta_val[1] = c;
      sh.k = 0;
      sh.mu = 0.0;
    }
    csync();
    double dgmax = 0.0;
    for (int q = 0; q < C; ++q) dgmax = fmax(dgmax, remote(&sh, q)->cta_val[1]);
    const double tabs = trunc * dgmax;
    csync();

    // ---- diagonally pivoted Cholesky, right-looking, truncated at tabs ----
    for (int step = 0; step < n; ++step) {
      // argmax of the remaining diagonal (ties -> lowest index)
      double bv = -1.0;
      int bi = -1;
      for (int ls = tid; ls < myslots; ls += JAC_THREADS) {
        const int i = ls * C + me;
        if (sh.piv_flag[ls]) continue;
        const double d = jsm[ls * lds + i];
        if (d > bv || (d == bv && i < bi)) bv = d, bi = i;
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi >= 0 && (bi < 0 || oi < bi))) bv = ov, bi = oi;
      }
      if (lane == 0) sh.red_d[warp] = bv, sh.red_i[warp] = bi;
      __syncthreads();
      if (tid == 0) {
        double v = -1.0;
        int ix = -1;
        for (int w = 0; w < JAC_WARPS; ++w)
          if (sh.red_d[w] > v || (sh.red_d[w] == v && sh.red_i[w] >= 0 && (ix < 0 || sh.red_i[w] < ix)))
            v = sh.red_d[w], ix = sh.red_i[w];
        sh.cta_val[0] = v;
        sh.cta_idx = ix;
      }
      csync();
      double v = -1.0;
      int j = -1;
      for (int q = 0; q < C; ++q) {
        JacShared* o = remote(&sh, q);
        const double ov = o->cta_val[0];
        const int oi = o->cta_idx;
        if (ov > v || (ov == v && oi >= 0 && (j < 0 || oi < j))) v = ov, j = oi;
      }
      if (j < 0 || !(v > tabs)) break;  // uniform across the cluster
      // pivot row r = S[j,:] / sqrt(S_jj): copy into every CTA's bcast buffer
      const double* pr = slot_ptr(j);
      const double inv = 1.0 / sqrt(v);
      for (int c = tid; c < n; c += JAC_THREADS) sh.bcast[c] = pr[c] * inv;
      csync();  // all copies done before the owner overwrites its row
      if ((j % C) == me) {
        const int ls = j / C;
        for (int c = tid; c < lds; c += JAC_THREADS) jsm[ls * lds + c] = c < n ? sh.bcast[c] : 0.0;
        if (tid == 0) sh.piv_flag[ls] = 1;
      }
      if (tid == 0) sh.order[step] = j;
      // rank-1 update of the remaining rows: S[i][c] -= r_i r_c
      for (int e = tid; e < myslots * n; e += JAC_THREADS) {
        const int ls = e / n, c = e % n;
        const int i = ls * C + me;
        if (i == j || sh.piv_flag[ls]) continue;
        jsm[ls * lds + c] -= sh.bcast[i] * sh.bcast[c];
      }
      if (tid == 0) sh.k = step + 1;
      csync();
    }
    K = sh.k;
  } else {
    for (int i = tid; i < N; i += JAC_THREADS) sh.order[i] = i;
    if (tid == 0) sh.mu = 0.0;
    __syncthreads();
  }
  // nu2 = max squared column norm (for the noise-pair skip test)
  {
    double mx = 0.0;
    for (int jj = warp; jj < K; jj += JAC_WARPS) {
      const int s = sh.order[jj];
      if (s % C != me) continue;
      const double* x = jsm + (s / C) * lds;
      double a = 0.0;
      for (int c = lane; c < ldot; c += 32) a = fma(x[c], x[c], a);
      mx = fmax(mx, warp_sum_bcast(a));
    }
    if (lane == 0) sh.red_d[warp] = mx;
    __syncthreads();
    if (tid == 0) {
      double a = 0.0;
      for (int w = 0; w < JAC_WARPS; ++w) a = fmax(a, sh.red_d[w]);
      sh.cta_val[1] = a;
    }
    csync();
    double a = 0.0;
    for (int q = 0; q < C; ++q) a = fmax(a, remote(&sh, q)->cta_val[1]);
    sh.nu2 = a;  // identical on every CTA
  }
  csync();

  // ---------------------------------------------------- Jacobi sweeps ----
  const int NE = K + (K & 1);
  constexpr int GPW = 32 / G;  // pair groups per warp
  const int grp = lane / G, gl = lane % G;
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (grp * G));
  const int gw = (me * JAC_WARPS + warp) * GPW + grp;
  const int tg = C * JAC_WARPS * GPW;
  const double skip2 = (kEps * kEps) * sh.nu2;
  int sweep = 0;
  bool converged = K <= 1;
  for (; sweep < max_sweeps && !converged; ++sweep) {
    if (tid == 0) sh.flag[(sweep + 1) % 3] = 0;
    for (int r = 0; r < NE - 1; ++r) {
      for (int i = gw; i < NE / 2; i += tg) {
        const int pp = i, qq = NE - 1 - i;
        const int p = pp == 0 ? 0 : 1 + (pp - 1 + r) % (NE - 1);
        const int q = 1 + (qq - 1 + r) % (NE - 1);
        if (p >= K || q >= K) continue;  // the pad column of an odd K
        double* xp = slot_ptr(sh.order[p]);
        double* xq = slot_ptr(sh.order[q]);
        double vp[EPG], vq[EPG];
        double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
        for (int e = 0; e < EPG; ++e) {
          const int idx = gl + G * e;
          vp[e] = idx < L ? xp[idx] : 0.0;
          vq[e] = idx < L ? xq[idx] : 0.0;
          if (idx < ldot) {
            al = fma(vp[e], vp[e], al);
            be = fma(vq[e], vq[e], be);
            ga = fma(vp[e], vq[e], ga);
          }
        }
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) {
          al += __shfl_xor_sync(gmask, al, o);
          be += __shfl_xor_sync(gmask, be, o);
          ga += __shfl_xor_sync(gmask, ga, o);
        }
        const int src = grp * G;
        al = __shfl_sync(gmask, al, src);
        be = __shfl_sync(gmask, be, src);
        ga = __shfl_sync(gmask, ga, src);
        if (ga != 0.0 && ga * ga > tol * tol * al * be && fmax(al, be) > skip2) {
          const double zeta = (be - al) / (2.0 * ga);
          const double tt = copysign(1.0, zeta) / (fabs(zeta) + hypot(1.0, zeta));
          const double c = 1.0 / sqrt(fma(tt, tt, 1.0));
          const double s = c * tt;
#pragma unroll
          for (int e = 0; e < EPG; ++e) {
            const int idx = gl + G * e;
            if (idx < L) {
              xp[idx] = c * vp[e] - s * vq[e];
              xq[idx] = s * vp[e] + c * vq[e];
            }
          }
          if (gl == 0) sh.flag[sweep % 3] = 1;
        }
      }
      csync();
    }
    int any = 0;
    for (int q = 0; q < C; ++q) any |= remote(&sh, q)->flag[sweep % 3];
    converged = !any;
  }

  // ------------------------------------------ norms, order, write back ----
  for (int jj = warp; jj < K; jj += JAC_WARPS) {
    const int s = sh.order[jj];
    if (s % C != me) continue;
    const double* x = jsm + (s / C) * lds;
    double a = 0.0;
    for (int c = lane; c < ldot; c += 32) a = fma(x[c], x[c], a);
    a = warp_sum_bcast(a);
    if (lane == 0) sh.nrm[jj] = sqrt(a);  // indexed by column (jj), stored where the slot lives
  }
  csync();
  for (int jj = tid; jj < K; jj += JAC_THREADS) {
    const int s = sh.order[jj];
    if (s % C != me) continue;
    const double nj = sh.nrm[jj];
    int rk = 0;
    for (int ii = 0; ii < K; ++ii) {
      const double ni = remote(&sh, sh.order[ii] % C)->nrm[ii];
      rk += (ni > nj) || (ni == nj && ii < jj);
    }
    sh.rank_out[jj] = rk;
  }
  __syncthreads();
  const double mu = sh.mu;
  for (int jj = warp; jj < K; jj += JAC_WARPS) {
    const int s = sh.order[jj];
    if (s % C != me) continue;
    const int rk = sh.rank_out[jj];
    const double nj = sh.nrm[jj];
    const double invn = nj > 0.0 ? 1.0 / nj : 0.0;
    const double* x = jsm + (s / C) * lds;
    double* dst = out + (size_t)rk * ldout;
    for (int c = lane; c < L; c += 32) dst[c] = c < ldot ? x[c] * invn : x[c];
    if (lane == 0) vals[rk] = mode == 0 ? fma(nj, nj, mu) : nj;
  }
  if (me == 0 && tid == 0) {
    info[0] = sweep;
    info[1] = converged ? 1 : 0;
    info[2] = K;
  }
  cluster.sync();  // keep DSMEM alive until every CTA is done reading it
}

template <int G, int EPG>
static cudaError_t jac_go(int C, size_t smem, const double* in, int ldin, int mode, int n, int N,
                          int ldot, int lacc, double tol, double trunc, int max_sweeps,
                          double* out, int ldout, double* vals, int* info, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(jacobi_kernel<G, EPG>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(JAC_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, jacobi_kernel<G, EPG>, in, ldin, mode, n, N, ldot, lacc, tol,
                            trunc, max_sweeps, out, ldout, vals, info);
}

static cudaError_t jac_dispatch(int mode, const double* in, int ldin, int n, int N, int ldot,
                                int lacc, double tol, double trunc, int max_sweeps, double* out,
                                int ldout, double* vals, int* info, cudaStream_t s) {
  const int L = ldot + lacc;
  const int nslots = mode == 0 ? n : N;
  if (nslots <= 0) return cudaSuccess;
  if (L > 512 || nslots > 512) return cudaErrorInvalidValue;
  const int lds = (L + 1) & ~1;
  const size_t budget = std::min<size_t>(dev_info().smem_optin - 16384, 200 * 1024);
  int C = 1;
  while (C < 8 && ((size_t)((nslots + C - 1) / C) * lds * 8 > budget ||
                   (nslots + C - 1) / C > JAC_MAXSLOTS))
    C *= 2;
  const size_t smem = (size_t)((nslots + C - 1) / C) * lds * 8;
  if (smem > budget) return cudaErrorInvalidValue;
#define JGO(G, E) \
  return jac_go<G, E>(C, smem, in, ldin, mode, n, N, ldot, lacc, tol, trunc, max_sweeps, out, ldout, vals, info, s)
  if (L <= 32) JGO(8, 4);
  if (L <= 64) JGO(8, 8);
  if (L <= 128) JGO(8, 16);
  if (L <= 256) JGO(16, 16);
  JGO(32, 16);
#undef JGO
}

cudaError_t launch_jacobi_eig(const double* B, int ldb, int n, double tol, double trunc,
                              int max_sweeps, double* vecs, int ldv, double* vals, int* info,
                              cudaStream_t s) {
  return jac_dispatch(0, B, ldb, n, n, n, 0, tol, trunc, max_sweeps, vecs, ldv, vals, info, s);
}

cudaError_t launch_jacobi_svd(const double* cols, int ldc, int N, int ldot, double tol,
                              int max_sweeps, double* out, int ldout, double* vals, int* info,
                              cudaStream_t s) {
  return jac_dispatch(1, cols, ldc, 0, N, ldot, N, tol, 0.0, max_sweeps, out, ldout, vals, info, s);
}

}  // namespace tsk
