// Algorithms 1 / 2 and the TSQR they use (Demmel-Grigori-Hoemmen-Langou, cited
// at P:531-532), for tall-skinny row-sharded matrices with n <= 128 columns:
//
//   * k_mix_matrix: the random orthogonal Omega = D F S D~ F S~ of Remark 'randomness'
//      as an explicit n x n matrix, built from the caller's random draws (phases of
//     D, D~, permutations S, S~) by a direct DFT of length h = n / 2 (the pairs of reals viewed
//     as complex numbers; for odd n the last coordinate is left unmixed, reading R17).  Row i of
//     the output is Omega e_i, i.e. the output is Omega^T, so B^* = A Omega^T is a GEMM.
//   * TSQR: leaf Householder QR of row blocks of b >= n rows, one CTA per block with the block
//     in registers (LAPACK dgeqr2 order: column by column, reflector H = I - tau v v^T with
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
// One CTA per block of B = 4 RPT rows, the block REGISTER-resident: thread (c, g) (t = 4 c + g)
// holds column c at the rows i = 4 q + g (q < RPT; interleaved, so every thread keeps the same
// share of active rows as the factorization advances).  The four threads of a column are
// adjacent lanes (column norms and dot products reduce with two shuffles); the four columns of a
// panel [4P, 4P + 4) are one half-warp.
// Blocked Householder (LAPACK dgeqrf / dorgqr with panels of 4, compact WY H_p..H_p+3 =
// I - V T V^T, T upper triangular as dlarft):
//   QR, per panel: its half-warp factors the 4 columns (dgeqr2 order: dlarfg beta =
//   -sign(alpha) ||x||, tau = (beta - alpha) / beta, v = x / (alpha - beta), v_j = 1; each
//   reflector applied to the panel's later columns), builds T and publishes V; one CTA barrier;
//   every later column c: C <- (I - V T^T V^T) C.
//   Q, panels last to first: the panel's columns reset to e_c, then every column c >= 4P:
//   C <- (I - V T V^T) C  (Q = H_0 .. H_kmax-1 [I; 0]; one barrier per panel).
// V in shared memory: vp[g (4 RPT + 4) + 4 q + k] = v_k at row 4q + g (a thread's row: 32 bytes;
// the pad puts the four groups of a warp on different banks).
// Block `blk`: rows [blk B, min(rows, (blk + 1) B)); R (kmax x n, upper, row-major ld n) to
// R + blk n n, the explicit Q (k x kmax) back in place, columns past kmax zero.

// publish slot k of panel V from my column (col): v_i = x (i > col), 1 (i == col), 0 (i < col);
// an absent reflector (col >= kmax) publishes zeros
template <int RPT>
__device__ __forceinline__ void pan_publish(const double (&x)[RPT], int col, bool present, int g, int k,
                                            double* vp) {
  double* row = vp + (size_t)g * (RPT * 4 + 4) + k;
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int i = 4 * q + g;
    row[4 * q] = present ? (i > col ? x[q] : (i == col ? 1.0 : 0.0)) : 0.0;
  }
}

// W = V^T x over my rows, reduced over the column's 4 lanes
template <int RPT>
__device__ __forceinline__ void pan_dots(const double (&x)[RPT], int g, unsigned mask4, const double* vp,
                                         double (&w)[4]) {
  const double* row = vp + (size_t)g * (RPT * 4 + 4);
  w[0] = w[1] = w[2] = w[3] = 0.0;
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const double2 a = *reinterpret_cast<const double2*>(row + 4 * q);
    const double2 b = *reinterpret_cast<const double2*>(row + 4 * q + 2);
    w[0] = fma(a.x, x[q], w[0]);
    w[1] = fma(a.y, x[q], w[1]);
    w[2] = fma(b.x, x[q], w[2]);
    w[3] = fma(b.y, x[q], w[3]);
  }
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    w[h] += __shfl_xor_sync(mask4, w[h], 1);
    w[h] += __shfl_xor_sync(mask4, w[h], 2);
  }
}

// x -= V w
template <int RPT>
__device__ __forceinline__ void pan_update(double (&x)[RPT], int g, const double* vp, const double (&w)[4]) {
  const volatile double* row = vp + (size_t)g * (RPT * 4 + 4);  // re-read (keeps V out of the registers)
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    double acc = x[q];
    acc = fma(-row[4 * q], w[0], acc);
    acc = fma(-row[4 * q + 1], w[1], acc);
    acc = fma(-row[4 * q + 2], w[2], acc);
    acc = fma(-row[4 * q + 3], w[3], acc);
    x[q] = acc;
  }
}

template <int RPT, int MAXT>
__global__ void __launch_bounds__(MAXT, 1) k_leaf_qr(double* X, int64_t ldx, int64_t rows, int n, double* R) {
  constexpr int B = 4 * RPT;
  __shared__ __align__(16) double vpan[2][4 * (RPT * 4 + 4)];  // group g at g (4 RPT + 4): conflict-free
  __shared__ double sT[32][16];  // T of panel P: sT[P][4 i + j] = T(i, j)
  constexpr int PLD = B + 4;  // column stride of the staged panel (bank-conflict-free columns)
  __shared__ __align__(16) double pan[4 * PLD];  // the panel being factored, column-major
  __shared__ double xpark[32 * RPT];              // the panel warp's other columns, parked
  const int t = threadIdx.x, g = t & 3, c = t >> 2, kk = c & 3, P = c >> 2;
  const int lane = t & 31, lane0 = lane & ~3;
  const unsigned mask4 = 0xFu << lane0;
  const unsigned maskP = 0xFFFFu << (lane & 16);
  const int64_t r0 = (int64_t)blockIdx.x * B;
  const int k = (int)min((int64_t)B, rows - r0);
  const int kmax = min(k, n);
  const bool act = c < n;
  double x[RPT];
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int i = 4 * q + g;
    x[q] = (act && i < k) ? X[(r0 + i) * ldx + c] : 0.0;
  }
  if (kmax <= 0) return;
  const int npan = (kmax + 3) / 4;
  // ---- QR
  for (int P0 = 0; P0 < npan; ++P0) {
    const int p = 4 * P0;
    double* vp = vpan[P0 & 1];
    double* T = sT[P0];
    if ((t >> 5) == (P0 >> 1)) {  // the warp holding the panel: factor it in shared memory
      // its half-warp stages the 4 columns (pan[kk PLD + i]); the other half parks its columns, so
      // no resident row stays live in registers across the panel code (which would spill)
      if (P == P0) {
#pragma unroll
        for (int q = 0; q < RPT; ++q) pan[kk * PLD + 4 * q + g] = x[q];
      } else {
#pragma unroll
        for (int q = 0; q < RPT; ++q) xpark[q * 32 + lane] = x[q];
      }
      __syncwarp();
      constexpr int RL = B / 32;  // rows per lane: i = lane + 32 r
#pragma unroll  // kq compile-time: the accumulator slots below stay in registers
      for (int kq = 0; kq < 4; ++kq) {
        const int col = p + kq;
        if (col >= kmax) {  // absent reflector: H = I (tau 0, zero column of T)
          if (lane == 0)
#pragma unroll
            for (int i2 = 0; i2 < 4; ++i2) T[4 * i2 + kq] = 0.0;
          continue;
        }
        // (1) dlarfg on rows >= col of column kq: sum of squares below the diagonal, one reduction
        double val[RL];
        double sq = 0.0;
#pragma unroll
        for (int r = 0; r < RL; ++r) {
          const int i = lane + 32 * r;
          val[r] = pan[kq * PLD + i];
          sq = fma(i > col ? val[r] : 0.0, val[r], sq);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
        const double alpha = pan[kq * PLD + col];
        double tau = 0.0, scale = 0.0, beta = alpha;
        if (sq > 0.0) {
          const double nrm = sqrt(fma(alpha, alpha, sq));
          beta = alpha >= 0.0 ? -nrm : nrm;
          tau = (beta - alpha) / beta;
          scale = 1.0 / (alpha - beta);
        }
        // (2) v (unit at col, zero above) and, in ONE fused reduction of three values: the dots
        //     d_k2 = v^T u_k2 of the panel's later columns (k2 > kq) and z_i2 = v_i2^T v of its
        //     earlier reflectors (i2 < kq) for T
        double acc[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int r = 0; r < RL; ++r) {
          const int i = lane + 32 * r;
          const double v = i > col ? val[r] * scale : (i == col ? 1.0 : 0.0);
          val[r] = v;
          const double u[4] = {pan[i], pan[PLD + i], pan[2 * PLD + i], pan[3 * PLD + i]};
#pragma unroll
          for (int k2 = 0; k2 < 4; ++k2) {
            if (k2 == kq) continue;
            // slot: later columns k2 > kq use acc[k2 - 1 - ... ]; simpler: acc index = k2 < kq ? k2 : k2 - 1
            const int slot = k2 < kq ? k2 : k2 - 1;
            // earlier reflector i2 = k2 < kq: v_i2 = u (i > p + k2), 1 (i == p + k2), 0 above
            const double w = k2 < kq ? (i > p + k2 ? u[k2] : (i == p + k2 ? 1.0 : 0.0)) : u[k2];
            acc[slot] = fma(v, w, acc[slot]);
          }
        }
#pragma unroll
        for (int h = 0; h < 3; ++h)
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) acc[h] += __shfl_xor_sync(0xffffffffu, acc[h], o);
        __syncwarp();  // every lane has read the panel before it is rewritten
        // (3) write v into column kq (beta on the diagonal), apply H to the later columns:
        //     u_k2 -= tau d_k2 v  (rows >= col)
#pragma unroll
        for (int r = 0; r < RL; ++r) {
          const int i = lane + 32 * r;
          if (i < col) continue;
          pan[kq * PLD + i] = i == col ? beta : val[r];
#pragma unroll
          for (int k2 = 0; k2 < 4; ++k2)
            if (k2 > kq) pan[k2 * PLD + i] = fma(-tau * acc[k2 - 1], val[r], pan[k2 * PLD + i]);
        }
        // (4) column kq of T (dlarft): T(0:kq, kq) = -tau T(0:kq, 0:kq) z, T(kq, kq) = tau
        if (lane == 0) {
          T[5 * kq] = tau;
#pragma unroll
          for (int i2 = 0; i2 < 3; ++i2) {
            if (i2 < kq) {
              double s2 = 0.0;
#pragma unroll
              for (int j2 = 0; j2 < 3; ++j2)
                if (j2 >= i2 && j2 < kq) s2 = fma(T[4 * i2 + j2], acc[j2], s2);
              T[4 * i2 + kq] = -tau * s2;
            }
          }
          for (int i2 = kq + 1; i2 < 4; ++i2) T[4 * i2 + kq] = 0.0;
        }
        __syncwarp();
      }
      // publish V for the trailing update: vp[(g RPT + q) 4 + k] = v_k(row 4q + g)
#pragma unroll
      for (int r = 0; r < RL; ++r) {
        const int i = lane + 32 * r;
        double v4[4];
#pragma unroll
        for (int k2 = 0; k2 < 4; ++k2) {
          const int c2 = p + k2;
          v4[k2] = c2 >= kmax ? 0.0 : (i > c2 ? pan[k2 * PLD + i] : (i == c2 ? 1.0 : 0.0));
        }
        double* dst = vp + (size_t)(i & 3) * (RPT * 4 + 4) + (i >> 2) * 4;
        *reinterpret_cast<double2*>(dst) = make_double2(v4[0], v4[1]);
        *reinterpret_cast<double2*>(dst + 2) = make_double2(v4[2], v4[3]);
      }
      __syncwarp();
      if (P == P0) {  // the panel's columns back: R above / on the diagonal, v below
#pragma unroll
        for (int q = 0; q < RPT; ++q) x[q] = pan[kk * PLD + 4 * q + g];
      } else {
#pragma unroll
        for (int q = 0; q < RPT; ++q) x[q] = xpark[q * 32 + lane];
      }
    }
    __syncthreads();
    if (act && c >= p + 4) {  // C <- (I - V T^T V^T) C
      double w[4];
      pan_dots<RPT>(x, g, mask4, vp, w);
      double u[4];
      u[0] = T[0] * w[0];
      u[1] = fma(T[1], w[0], T[5] * w[1]);
      u[2] = fma(T[2], w[0], fma(T[6], w[1], T[10] * w[2]));
      u[3] = fma(T[3], w[0], fma(T[7], w[1], fma(T[11], w[2], T[15] * w[3])));
      pan_update<RPT>(x, g, vp, u);
    }
  }
  // ---- R out (upper triangle; zeros below)
  if (act) {
    double* Rb = R + (size_t)blockIdx.x * n * n;
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int i = 4 * q + g;
      if (i < kmax) Rb[(size_t)i * n + c] = c >= i ? x[q] : 0.0;
    }
  }
  // ---- explicit Q (dorgqr order, panels last to first)
  __syncthreads();
  if (P == npan - 1) {
    pan_publish<RPT>(x, c, c < kmax, g, kk, vpan[(npan - 1) & 1]);
#pragma unroll
    for (int q = 0; q < RPT; ++q) x[q] = (4 * q + g == c) ? 1.0 : 0.0;
  }
  for (int P0 = npan - 1; P0 >= 0; --P0) {
    __syncthreads();
    const double* vp = vpan[P0 & 1];
    const double* T = sT[P0];
    if (act && c >= 4 * P0 && c < kmax) {  // C <- (I - V T V^T) C
      double w[4];
      pan_dots<RPT>(x, g, mask4, vp, w);
      double u[4];
      u[0] = fma(T[0], w[0], fma(T[1], w[1], fma(T[2], w[2], T[3] * w[3])));
      u[1] = fma(T[5], w[1], fma(T[6], w[2], T[7] * w[3]));
      u[2] = fma(T[10], w[2], T[11] * w[3]);
      u[3] = T[15] * w[3];
      pan_update<RPT>(x, g, vp, u);
    } else if (P == P0 - 1) {  // the next panel publishes its V and resets its columns to e_c
      pan_publish<RPT>(x, c, c < kmax, g, kk, vpan[(P0 - 1) & 1]);
#pragma unroll
      for (int q = 0; q < RPT; ++q) x[q] = (4 * q + g == c) ? 1.0 : 0.0;
    }
  }
  if (act) {
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int i = 4 * q + g;
      if (i < k) X[(r0 + i) * ldx + c] = c < kmax ? x[q] : 0.0;
    }
  }
}

// Q_block (k x n, ld ldx) <- Q_block * Qup[blk*n .. blk*n + kmax, :] (kmax x n, ld ldu).  One CTA
// per block: Qup's slice in shared memory, the block in chunks of 32 rows (staged, then
// overwritten); each thread a 4 x 4 output tile, k-loop in fixed order.
static constexpr int BM_ROWS = 32;
__global__ void __launch_bounds__(256) k_block_mul(double* X, int64_t ldx, int64_t rows, int n, int b,
                                                   const double* Qup, int64_t ldu) {
  extern __shared__ double sm[];
  const int ldq = ((n + 3) & ~3);  // Qup rows padded to whole 4-column tiles (zeros)
  double* qs = sm;                              // [n][ldq]
  double* xs = sm + (size_t)n * ldq;            // [BM_ROWS][n + 1]
  const int ldx_s = n + 1;
  const int64_t r0 = (int64_t)blockIdx.x * b;
  const int k = (int)min((int64_t)b, rows - r0);
  const int kmax = min(k, n);
  const double* qu = Qup + (size_t)blockIdx.x * n * ldu;
  for (int e = threadIdx.x; e < n * ldq; e += blockDim.x) {
    const int i = e / ldq, cc = e % ldq;
    qs[e] = (i < kmax && cc < n) ? qu[(size_t)i * ldu + cc] : 0.0;
  }
  const int ncg = ldq / 4;                 // column tiles
  const int tr = threadIdx.x / ncg, tc = threadIdx.x % ncg;  // tr < 8 (rows 4 tr .. 4 tr + 3)
  const bool worker = threadIdx.x < 8 * ncg;
  for (int i0 = 0; i0 < k; i0 += BM_ROWS) {
    const int nr = min(BM_ROWS, k - i0);
    __syncthreads();
    for (int e = threadIdx.x; e < nr * kmax; e += blockDim.x) {
      const int i = e / kmax, cc = e % kmax;
      xs[i * ldx_s + cc] = X[(r0 + i0 + i) * ldx + cc];
    }
    __syncthreads();
    if (worker && 4 * tr < nr) {
      double acc[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int bb = 0; bb < 4; ++bb) acc[a][bb] = 0.0;
      const double* xr = xs + (4 * tr) * ldx_s;
      const double* qc = qs + 4 * tc;
      for (int tt = 0; tt < kmax; ++tt) {
        double av[4], bv[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) av[a] = xr[a * ldx_s + tt];
        const double2 b01 = *reinterpret_cast<const double2*>(qc + (size_t)tt * ldq);
        const double2 b23 = *reinterpret_cast<const double2*>(qc + (size_t)tt * ldq + 2);
        bv[0] = b01.x, bv[1] = b01.y, bv[2] = b23.x, bv[3] = b23.y;
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int bb = 0; bb < 4; ++bb) acc[a][bb] = fma(av[a], bv[bb], acc[a][bb]);
      }
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int i = 4 * tr + a;
        if (i < nr)
#pragma unroll
          for (int bb = 0; bb < 4; ++bb) {
            const int cc = 4 * tc + bb;
            if (cc < n) X[(r0 + i0 + i) * ldx + cc] = acc[a][bb];
          }
      }
    }
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
// rows per thread of the leaf kernel: the block is B = 4 RPT rows (>= n), held in registers
static inline int leaf_rpt(int n) { return n <= 64 ? 64 : 48; }
int tsqr_block_rows(int n) { return 4 * leaf_rpt(n); }

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
static cudaError_t leaf(double* X, int64_t ldx, int64_t rows, int n, double* R, cudaStream_t s) {
  const int64_t nb = ceil_div(rows, tsqr_block_rows(n));
  const int threads = 4 * ((n + 7) & ~7);
  if (leaf_rpt(n) == 64) k_leaf_qr<64, 256><<<(unsigned)nb, threads, 0, s>>>(X, ldx, rows, n, R);
  else k_leaf_qr<48, 512><<<(unsigned)nb, threads, 0, s>>>(X, ldx, rows, n, R);
  return cudaGetLastError();
}

cudaError_t launch_tsqr(double* X, int64_t ldx, int64_t rows, int n, double* R_out, double* work, cudaStream_t s) {
  if (n < 1 || n > 128) return cudaErrorInvalidValue;
  const int b = tsqr_block_rows(n);
  cudaError_t e;
  if (rows <= b) {  // one block: R straight out (kmax rows), zero rows below
    e = cudaMemsetAsync(R_out, 0, (size_t)n * n * 8, s);
    if (e != cudaSuccess) return e;
    return rows > 0 ? leaf(X, ldx, rows, n, R_out, s) : cudaSuccess;
  }
  const int64_t nb = ceil_div(rows, b);
  const int64_t last_k = std::min<int64_t>(n, rows - (nb - 1) * b);
  const int64_t srows = (nb - 1) * n + last_k;  // stacked R rows
  double* Rs = work;  // nb x (n x n): block q's rows at q*n (== the stacking order)
  e = leaf(X, ldx, rows, n, Rs, s);
  if (e != cudaSuccess) return e;
  // the stacked R's: rows [q*n, q*n + kmax_q) of Rs (ld n) -- contiguous because every block
  // but the last has kmax = n
  e = launch_tsqr(Rs, n, srows, n, R_out, work + (size_t)nb * n * n, s);
  if (e != cudaSuccess) return e;
  const size_t msmem = ((size_t)n * ((n + 3) & ~3) + (size_t)BM_ROWS * (n + 1)) * 8;
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
