// Algorithms 1 / 2 and the TSQR they use (Demmel-Grigori-Hoemmen-Langou, cited
// at P:531-532), for tall-skinny row-sharded matrices with n <= 128 columns:
//
//   * k_mix_matrix: the random orthogonal Omega = D F S D~ F S~ of Remark 'randomness'
//      as an explicit n x n matrix, built from the caller's random draws (phases of
//     D, D~, permutations S, S~) by a direct DFT of length h = n / 2 (the pairs of reals viewed
//     as complex numbers; for odd n the last coordinate is left unmixed, reading R17).  Row i of
//     the output is Omega e_i, i.e. the output is Omega^T, so B^* = A Omega^T is a GEMM.
//   * TSQR: leaf Householder QR of row blocks of b >= n rows, one CTA per block with the block
//     in shared memory (LAPACK dgeqr2 order: column by column, reflector H = I - tau v v^T with
//     v_j = 1), the explicit Q of the block formed in place (dorg2r order); the blocks' R
//     factors are stacked and factored the same way, recursively, and the final Q of a level
//     is its blocks' Q times the matching rows of the level above (k_block_mul).
//
// Every reduction has a fixed order (bit-identical on every rank for replicated inputs).
#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace tsk {

static constexpr int QT = 512;  // threads per CTA

// ------------------------------------------------------------------ Omega --
// Output row i = Omega e_i (M[i][j], ld ldm): z = complex pairs of e_i; z <- S~ z; z <- F z;
// z <- D~ z; z <- S z; z <- F z; z <- D z (F unitary, (S z)_k = z_{S[k]}, D = diag(e^{i theta})).
// The width w is `wconst`, or the device count *wdev (a kept rank: the factorization's input has
// zero columns past it), whose random draws are row w - 1 of the tables (ld ldp); rows and
// columns of M past w (up to the launch bound wb) are zero.
// Tables: phases[row] = [theta_D (h), theta_D~ (h)], perms[row] = [S (h), S~ (h)], h = w / 2.
__global__ void __launch_bounds__(256) k_mix_matrix(const double* phases, const int* perms, int ldp, const int* wdev,
                                                    int wconst, int wb, double* M, int ldm) {
  extern __shared__ double zm[];  // [2][h] complex (re, im interleaved)
  const int i = blockIdx.x;
  const int w = wdev ? min(*wdev, wb) : wconst;
  if (i >= w || w <= 0) {
    for (int j = threadIdx.x; j < wb; j += blockDim.x) M[(size_t)i * ldm + j] = 0.0;
    return;
  }
  const double* ph0 = wdev ? phases + (size_t)(w - 1) * ldp : phases;
  const int* pm0 = wdev ? perms + (size_t)(w - 1) * ldp : perms;
  const int h = w / 2;
  double* za = zm;          // 2h doubles
  double* zb = zm + 2 * h;  // 2h doubles
  const double inv_sqrt_h = h > 0 ? rsqrt((double)h) : 0.0;
  for (int k = threadIdx.x; k < h; k += blockDim.x) {  // e_i as complex pairs
    za[2 * k] = (2 * k == i) ? 1.0 : 0.0;
    za[2 * k + 1] = (2 * k + 1 == i) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int stage = 0; stage < 2; ++stage) {
    const int* perm = pm0 + (stage == 0 ? h : 0);    // S~ first, then S
    const double* ph = ph0 + (stage == 0 ? h : 0);   // D~ first, then D
    for (int k = threadIdx.x; k < h; k += blockDim.x) {  // zb = S za
      zb[2 * k] = za[2 * perm[k]];
      zb[2 * k + 1] = za[2 * perm[k] + 1];
    }
    __syncthreads();
    for (int f = threadIdx.x; f < h; f += blockDim.x) {  // za = D F zb (direct DFT, fixed order)
      double re = 0.0, im = 0.0;
      for (int k = 0; k < h; ++k) {
        double s, c;  // e^{-2 pi i f k / h}: exact argument reduction of f k mod h
        sincospi(-2.0 * (double)(((long long)f * k) % h) / (double)h, &s, &c);
        const double xr = zb[2 * k], xi = zb[2 * k + 1];
        re = fma(xr, c, fma(-xi, s, re));
        im = fma(xr, s, fma(xi, c, im));
      }
      double s, c;
      sincos(ph[f], &s, &c);
      re *= inv_sqrt_h;
      im *= inv_sqrt_h;
      za[2 * f] = re * c - im * s;  // (re + i im) e^{i theta}
      za[2 * f + 1] = re * s + im * c;
    }
    __syncthreads();
  }
  for (int j = threadIdx.x; j < wb; j += blockDim.x)  // odd w: the last coordinate unmixed (R17)
    M[(size_t)i * ldm + j] = j < 2 * h ? za[j] : (j == i && j < w ? 1.0 : 0.0);
}

// ------------------------------------------------------ leaf Householder QR --
// Block `blk` of X (rows [blk*b, min(rows, (blk+1)*b)) x n, ld ldx): R (kmax x n, upper, row-major,
// ld n) to R + roff(blk) * n, the explicit Q (k x kmax) back into the block, columns past kmax zero.
// roff(blk) = sum of kmax over the earlier blocks = blk * n (every block but the last has >= n rows).
__global__ void __launch_bounds__(QT, 1) k_leaf_qr(double* X, int64_t ldx, int64_t rows, int n, int b,
                                                  double* R) {
  extern __shared__ double xs[];  // [b][n + 1]
  __shared__ double s_red[QT / 32];
  __shared__ double s_tau[128];
  __shared__ double s_par[2];
  const int ldsm = n + 1;
  const int64_t r0 = (int64_t)blockIdx.x * b;
  const int k = (int)min((int64_t)b, rows - r0);
  const int kmax = min(k, n);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < k * n; e += QT) {
    const int i = e / n, c = e % n;
    xs[i * ldsm + c] = X[(r0 + i) * ldx + c];
  }
  __syncthreads();
  // ---- Householder QR (dgeqr2 order)
  for (int j = 0; j < kmax; ++j) {
    double s = 0.0;
    for (int i = j + 1 + tid; i < k; i += QT) s = fma(xs[i * ldsm + j], xs[i * ldsm + j], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) s_red[warp] = s;
    __syncthreads();
    if (tid == 0) {
      double sig2 = 0.0;
      for (int w = 0; w < QT / 32; ++w) sig2 += s_red[w];
      const double alpha = xs[j * ldsm + j];
      double tau = 0.0, scale = 0.0, beta = alpha;
      if (sig2 > 0.0) {  // (dlarfg; sig2 == 0: H = I)
        const double nrm = sqrt(fma(alpha, alpha, sig2));
        beta = alpha >= 0.0 ? -nrm : nrm;
        tau = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
      }
      s_tau[j] = tau;
      s_par[0] = scale;
      s_par[1] = beta;
    }
    __syncthreads();
    const double tau = s_tau[j], scale = s_par[0];
    if (tau != 0.0)
      for (int i = j + 1 + tid; i < k; i += QT) xs[i * ldsm + j] *= scale;  // v (v_j = 1 implicit)
    __syncthreads();
    if (tid == 0) xs[j * ldsm + j] = s_par[1];  // R_jj
    // H_j to the trailing columns: one warp per column (lanes over rows, fixed-order sums)
    if (tau != 0.0)
      for (int c = j + 1 + warp; c < n; c += QT / 32) {
        double w = 0.0;
        for (int i = j + 1 + lane; i < k; i += 32) w = fma(xs[i * ldsm + j], xs[i * ldsm + c], w);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
        w += xs[j * ldsm + c];  // v_j = 1
        const double tw = tau * w;
        if (lane == 0) xs[j * ldsm + c] -= tw;
        for (int i = j + 1 + lane; i < k; i += 32) xs[i * ldsm + c] = fma(-tw, xs[i * ldsm + j], xs[i * ldsm + c]);
      }
    __syncthreads();
  }
  // ---- R out (rows 0..kmax-1, upper triangle; below-diagonal zero)
  double* Rb = R + (size_t)blockIdx.x * n * n;
  for (int e = tid; e < kmax * n; e += QT) {
    const int i = e / n, c = e % n;
    Rb[(size_t)i * n + c] = c >= i ? xs[i * ldsm + c] : 0.0;
  }
  __syncthreads();
  // ---- explicit Q in place (dorg2r order): columns kmax-1 .. 0
  for (int j = kmax - 1; j >= 0; --j) {
    const double tau = s_tau[j];
    if (j < kmax - 1) {  // H_j to Q's columns j+1.., rows j..
      for (int c = j + 1 + warp; c < kmax; c += QT / 32) {
        double w = 0.0;
        for (int i = j + 1 + lane; i < k; i += 32) w = fma(xs[i * ldsm + j], xs[i * ldsm + c], w);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
        w += xs[j * ldsm + c];  // row j of column c is 0 here (set when c was formed), v_j = 1
        const double tw = tau * w;
        if (lane == 0) xs[j * ldsm + c] -= tw;
        for (int i = j + 1 + lane; i < k; i += 32) xs[i * ldsm + c] = fma(-tw, xs[i * ldsm + j], xs[i * ldsm + c]);
      }
      __syncthreads();
    }
    for (int i = j + 1 + tid; i < k; i += QT) xs[i * ldsm + j] *= -tau;
    if (tid == 0) xs[j * ldsm + j] = 1.0 - tau;
    for (int i = tid; i < j; i += QT) xs[i * ldsm + j] = 0.0;
    __syncthreads();
  }
  for (int e = tid; e < k * n; e += QT) {
    const int i = e / n, c = e % n;
    X[(r0 + i) * ldx + c] = c < kmax ? xs[i * ldsm + c] : 0.0;
  }
}

// Q_block (k x n, ld ldx) <- Q_block * Qup[blk*n .. blk*n + kmax, :] (kmax x n, ld ldu), one CTA per
// block, Qup's slice staged in shared memory, one thread per (row, column) output in fixed order.
__global__ void __launch_bounds__(256) k_block_mul(double* X, int64_t ldx, int64_t rows, int n, int b,
                                                   const double* Qup, int64_t ldu) {
  extern __shared__ double qs[];  // [n][n]
  const int64_t r0 = (int64_t)blockIdx.x * b;
  const int k = (int)min((int64_t)b, rows - r0);
  const int kmax = min(k, n);
  const double* qu = Qup + (size_t)blockIdx.x * n * ldu;
  for (int e = threadIdx.x; e < kmax * n; e += blockDim.x) qs[e] = qu[(size_t)(e / n) * ldu + e % n];
  __syncthreads();
  // row by row: the row's kmax values to registers through a shared row buffer
  double* rowbuf = qs + (size_t)n * n;  // [8][n]
  const int sub = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i0 = 0; i0 < k; i0 += 8) {
    const int i = i0 + sub;
    if (i < k)
      for (int c = lane; c < kmax; c += 32) rowbuf[sub * n + c] = X[(r0 + i) * ldx + c];
    __syncwarp();
    if (i < k)
      for (int c = lane; c < n; c += 32) {
        double s = 0.0;
        for (int t = 0; t < kmax; ++t) s = fma(rowbuf[sub * n + t], qs[t * n + c], s);
        X[(r0 + i) * ldx + c] = s;
      }
    __syncwarp();
  }
}

// ------------------------------------------------------ Alg. 1/2 steps 3-9 --
// Discard (Alg. 1 step 3 P:534-538, Alg. 2 steps 3, 5 P:571-589; reading R18): row j of R is kept
// iff |R_jj| >= |R_00| wp (nothing when R_00 == 0 or a diagonal entry is not finite: the
// non-finite flag).  Discarded rows of R are zeroed in place; mask[j] = kept, mask[w] = 1 when
// something was discarded.  Slot ints as k_discard: {r, nc, bad, r, -r, nc, -nc, 0}.
__global__ void k_r_discard(double* R, int w, double wp, int* out, int* mask) {
  __shared__ int s_mask[129];
  if (threadIdx.x == 0) {
    int bad = 0;
    for (int j = 0; j < w; ++j)
      if (!isfinite(R[(size_t)j * w + j])) bad = 1;
    const double d0 = w > 0 ? fabs(R[0]) : 0.0;
    int r = 0, nc = 0;
    for (int j = 0; j < w; ++j) {
      const int keep = !bad && d0 > 0.0 && fabs(R[(size_t)j * w + j]) >= d0 * wp;
      s_mask[j] = keep;
      if (keep) ++r, nc = j + 1;
    }
    s_mask[w] = r < w;
    out[0] = r;
    out[1] = nc;
    out[2] = bad;
    out[3] = r;
    out[4] = -r;
    out[5] = nc;
    out[6] = -nc;
    out[7] = 0;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < w * w; e += blockDim.x)
    if (!s_mask[e / w]) R[e] = 0.0;
  for (int j = threadIdx.x; j <= w; j += blockDim.x) mask[j] = s_mask[j];
}

// Alg. 2 step 3: the discarded columns of Q~ are dropped (zeroed) before Q~ = Q R.
__global__ void k_zero_cols(double* X, int64_t ldx, int64_t m, int w, const int* mask) {
  if (!mask[w]) return;
  __shared__ int s_mask[128];
  for (int j = threadIdx.x; j < w; j += blockDim.x) s_mask[j] = mask[j];
  __syncthreads();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m * w; e += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(e % w);
    if (!s_mask[j]) X[(e / w) * ldx + j] = 0.0;
  }
}

// Alg. 2 step 6: T = R R~ (w x w, row-major, fixed k order).
__global__ void k_tri_mul(const double* R2, const double* R1, int w, double* T) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= w * w) return;
  const int i = e / w, j = e % w;
  double acc = 0.0;
  for (int k = i; k <= j; ++k) acc = fma(R2[(size_t)i * w + k], R1[(size_t)k * w + j], acc);  // both upper
  T[e] = acc;
}

// Alg. 1 steps 4-6 / Alg. 2 steps 7-9 after the Jacobi SVD of K = R^T
// (column a of the solver's output: [P(:, a) (w) ; J(:, a) (w)], K J = P Sigma, so R = J Sigma P^T:
// U~ = J, V~ = P).  One CTA per output column a:
//   V(:, a) = s_a Omega^-1 P(:, a) = s_a M0 P(:, a)   (M0 = Omega^T, row i = Omega e_i)
//   Mg[b][a] = s_a J(b, a)  (the GEMM operand of U = Q U~), sigma[a] = vals[a]
// s_a: the largest-|.| entry of V(:, a) positive, ties to the lowest row (reading R5); a >= r:
// zeros.
__global__ void __launch_bounds__(128) k_tsqr_out(const double* svo, int w, const double* vals, const double* M0,
                                                  const int* rr, double* sigma, double* V, int64_t ldv, double* Mg,
                                                  int ldm) {
  __shared__ double vv[128];
  __shared__ double s_sign;
  const int a = blockIdx.x, tid = threadIdx.x;
  const int r = *rr;
  if (a >= r) {
    for (int i = tid; i < w; i += blockDim.x) {
      V[(size_t)i * ldv + a] = 0.0;
      Mg[(size_t)i * ldm + a] = 0.0;
    }
    if (tid == 0) sigma[a] = 0.0;
    return;
  }
  const double* P = svo + (size_t)a * 2 * w;
  const double* J = P + w;
  for (int i = tid; i < w; i += blockDim.x) {
    double acc = 0.0;
    for (int k = 0; k < w; ++k) acc = fma(M0[(size_t)i * w + k], P[k], acc);
    vv[i] = acc;
  }
  __syncthreads();
  if (tid == 0) {
    int best = 0;
    double bv = -1.0;
    for (int i = 0; i < w; ++i)
      if (fabs(vv[i]) > bv) bv = fabs(vv[i]), best = i;
    s_sign = vv[best] < 0.0 ? -1.0 : 1.0;
    sigma[a] = vals[a];
  }
  __syncthreads();
  const double sg = s_sign;
  for (int i = tid; i < w; i += blockDim.x) {
    V[(size_t)i * ldv + a] = sg * vv[i];
    Mg[(size_t)i * ldm + a] = sg * J[i];
  }
}

// ------------------------------------------------------------- launchers ----
int tsqr_block_rows(int n) {
  int b = (24576 / (n + 1)) / 8 * 8;
  b = b < 256 ? b : 256;
  return b > n ? b : ((n + 7) / 8) * 8;
}

size_t tsqr_workspace_doubles(int64_t rows, int n) {
  const int b = tsqr_block_rows(n);
  size_t tot = 0;
  int64_t r = rows;
  while (r > b) {
    const int64_t nb = ceil_div(r, b);
    const int64_t next = (nb - 1) * n + std::min<int64_t>(n, r - (nb - 1) * b);
    tot += (size_t)nb * n * n;  // R stack of this level (n x n per block, rows used: kmax)
    r = next;
  }
  return tot + (size_t)n * n + 64;
}

cudaError_t launch_mix_matrix(const double* phases, const int* perms, int ldp, const int* wdev, int wconst, int wb,
                              double* M, int ldm, cudaStream_t s) {
  if (wb <= 0) return cudaSuccess;
  k_mix_matrix<<<wb, 256, (size_t)4 * (wb / 2) * 8 + 16, s>>>(phases, perms, ldp, wdev, wconst, wb, M, ldm);
  return cudaGetLastError();
}

// TSQR of X (rows x n, ld ldx) in place: X <- Q (rows x n, orthonormal columns; columns past
// min(rows, n) zero), R (n x n, upper, row-major ld n; rows past min(rows, n) zero) to R_out.
// Recursive over levels: leaf QRs of b-row blocks, R stack factored the same way (its own Q),
// X's blocks multiplied by their rows of that Q.  work: tsqr_workspace_doubles(rows, n).
cudaError_t launch_tsqr(double* X, int64_t ldx, int64_t rows, int n, double* R_out, double* work, cudaStream_t s) {
  if (n < 1 || n > 128) return cudaErrorInvalidValue;
  const int b = tsqr_block_rows(n);
  const size_t smem = (size_t)b * (n + 1) * 8;
  cudaError_t e = cudaFuncSetAttribute(k_leaf_qr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (rows <= b) {  // one block: R straight out (kmax rows), zero rows below
    e = cudaMemsetAsync(R_out, 0, (size_t)n * n * 8, s);
    if (e != cudaSuccess) return e;
    k_leaf_qr<<<1, QT, smem, s>>>(X, ldx, rows, n, b, R_out);
    return cudaGetLastError();
  }
  const int64_t nb = ceil_div(rows, b);
  const int64_t last_k = std::min<int64_t>(n, rows - (nb - 1) * b);
  const int64_t srows = (nb - 1) * n + last_k;  // stacked R rows
  double* Rs = work;  // nb x (n x n): block q's rows at q*n (== the stacking order)
  k_leaf_qr<<<(unsigned)nb, QT, smem, s>>>(X, ldx, rows, n, b, Rs);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  // the stacked R's: rows [q*n, q*n + kmax_q) of Rs (ld n) -- contiguous because every block
  // but the last has kmax = n
  e = launch_tsqr(Rs, n, srows, n, R_out, work + (size_t)nb * n * n, s);
  if (e != cudaSuccess) return e;
  const size_t msmem = ((size_t)n * n + 8 * n) * 8;
  e = cudaFuncSetAttribute(k_block_mul, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)msmem);
  if (e != cudaSuccess) return e;
  k_block_mul<<<(unsigned)nb, 256, msmem, s>>>(X, ldx, rows, n, b, Rs, n);
  return cudaGetLastError();
}

cudaError_t launch_r_discard(double* R, int w, double wp, int* slot, int* mask, cudaStream_t s) {
  k_r_discard<<<1, 256, 0, s>>>(R, w, wp, slot, mask);
  return cudaGetLastError();
}
cudaError_t launch_zero_cols(double* X, int64_t ldx, int64_t m, int w, const int* mask, cudaStream_t s) {
  if (m <= 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>(ceil_div(m * w, 256), 148 * 16);
  k_zero_cols<<<(unsigned)blocks, 256, 0, s>>>(X, ldx, m, w, mask);
  return cudaGetLastError();
}
cudaError_t launch_tri_mul(const double* R2, const double* R1, int w, double* T, cudaStream_t s) {
  k_tri_mul<<<(unsigned)ceil_div((int64_t)w * w, 256), 256, 0, s>>>(R2, R1, w, T);
  return cudaGetLastError();
}
cudaError_t launch_tsqr_out(const double* svo, int w, const double* vals, const double* M0, const int* rr,
                            double* sigma, double* V, int64_t ldv, double* Mg, int ldm, cudaStream_t s) {
  k_tsqr_out<<<w, 128, 0, s>>>(svo, w, vals, M0, rr, sigma, V, ldv, Mg, ldm);
  return cudaGetLastError();
}

}  // namespace tsk
