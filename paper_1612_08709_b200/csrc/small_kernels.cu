// Small replicated-core kernels of Alg. 3/4 (everything between the streaming
// passes that is not the Jacobi solver itself): symmetrisation, the "Discard"
// decisions, and the assembly of the small n x r factors.  All of them run on
// data that is bit-identical on every rank, in a fixed order.
#include <cstdint>

#include "common.cuh"
#include "small_kernels.h"

namespace tsk {

// B[j][i] = B[i][j] for i > j (NCCL sums the two triangles in different orders).
__global__ void k_symmetrize(double* B, int w, int ldb) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= w * w) return;
  const int i = e / w, j = e % w;
  if (i > j) B[(size_t)j * ldb + i] = B[(size_t)i * ldb + j];
}

// Row-major padded M (mrows x ldm, zero outside) from column-major cols (c columns of length k, ldc):
// M[i][j] = cols[j*ldc + i].
__global__ void k_cols_to_m(const double* cols, int ldc, int k, int c, double* M, int ldm,
                            int mrows) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)mrows * ldm) return;
  const int i = (int)(e / ldm), j = (int)(e % ldm);
  M[e] = (i < k && j < c) ? cols[(size_t)j * ldc + i] : 0.0;
}

// Row-major padded M from a row-major source (k x c, lds).
__global__ void k_rows_to_m(const double* src, int64_t lds, int k, int c, double* M, int ldm,
                            int mrows) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)mrows * ldm) return;
  const int i = (int)(e / ldm), j = (int)(e % ldm);
  M[e] = (i < k && j < c) ? src[(size_t)i * lds + j] : 0.0;
}

// Discard rule.  One CTA.
//   sig_j = sqrt(nsq_j); keep j iff sig_j >= max(sig) * sqrt(wp) (and max > 0).
//   idx = kept indices in ascending order.  Decision slot `out` (8 ints):
//     [0] r  [1] nc = max kept + 1  [2] non-finite flag  [3] r [4] -r [5] nc [6] -nc
//   ([3..6] are max-allreduced across ranks by the rank-consistency guard: every
//   rank must see max == own value).  nf (nullable): the eigensolver's non-finite
//   flag for the Gram diagonal (an Inf/NaN in A or Omega, caught by the first pass).
__global__ void k_discard(const double* nsq, int w, double sqrt_wp, double* sig, int* idx,
                          int* out, const int* nf) {
  __shared__ double smax[32];
  __shared__ int bad;
  if (threadIdx.x == 0) bad = nf ? (*nf != 0) : 0;
  __syncthreads();
  double mx = 0.0;
  for (int j = threadIdx.x; j < w; j += blockDim.x) {
    const double v = nsq[j];
    const double s = sqrt(fmax(v, 0.0));
    sig[j] = s;
    if (!isfinite(v)) bad = 1;
    mx = fmax(mx, s);
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) smax[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int q = 0; q < (int)(blockDim.x + 31) / 32; ++q) m = fmax(m, smax[q]);
    const double thr = m * sqrt_wp;
    int r = 0, nc = 0;
    if (m > 0.0 && !bad) {
      for (int j = 0; j < w; ++j)
        if (sig[j] >= thr) {
          idx[r++] = j;
          nc = j + 1;
        }
    }
    out[0] = r;
    out[1] = nc;
    out[2] = bad;
    out[3] = r;
    out[4] = -r;
    out[5] = nc;
    out[6] = -nc;
    out[7] = 0;
  }
}

// Sign of column a: +1/-1 so that its largest-|.| entry (ties -> lowest index) is positive.
__device__ double col_sign(const double* x, int stride, int len) {
  int best = 0;
  double bv = -1.0;
  for (int i = 0; i < len; ++i) {
    const double v = fabs(x[(size_t)i * stride]);
    if (v > bv) bv = v, best = i;
  }
  return x[(size_t)best * stride] < 0.0 ? -1.0 : 1.0;
}

// Alg. 3 outputs with reading R4 (sort by Sigma descending) and R5 (signs).
// Vt: eigenvectors, column-major (column j at Vt + j*w).  One thread per output
// position a < rb (rb = host bound >= r; r = *rr is the kept rank on the device).
//   rank_a = position of kept column a by descending sig (ties by index)
//   M[idx_a][rank_a] = s_a / sig[idx_a];  V[:, rank_a] = s_a * Vt[:, idx_a];  sigma[rank_a] = sig
// Positions [r, rb) get sigma = 0 and V = 0 (M's columns there stay zero).
__global__ void k_alg3_out(const double* sig, const int* idx, const int* rr, int rb, const double* Vt,
                           int w, double* M, int ldm, double* sigma, double* V, int64_t ldv) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= rb) return;
  const int r = *rr;
  if (a >= r) {
    sigma[a] = 0.0;
    for (int i = 0; i < w; ++i) V[(size_t)i * ldv + a] = 0.0;
    return;
  }
  const int ja = idx[a];
  TCHECK(ja >= 0 && ja < w && r <= rb && rb <= ldm);
  const double sa = sig[ja];
  int rk = 0;
  for (int b = 0; b < r; ++b) {
    const double sb = sig[idx[b]];
    rk += (sb > sa) || (sb == sa && b < a);
  }
  const double* v = Vt + (size_t)ja * w;
  const double sg = col_sign(v, 1, w);
  M[(size_t)ja * ldm + rk] = sg / sa;
  sigma[rk] = sa;
  for (int i = 0; i < w; ++i) V[(size_t)i * ldv + rk] = sg * v[i];
}

// Z[a][b] = G[idx_a][idx_b] / (sig_a sig_b) -- Gram of Y = Y~_keep Sigma~^-1;
// rb x rb (ld rb), zero outside the leading r x r block (r = *rr).
__global__ void k_build_z(const double* G, int ldg, const int* idx, const double* sig, const int* rr,
                          int rb, double* Z) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rb * rb) return;
  const int r = *rr;
  const int a = e / rb, b = e % rb;
  if (a >= r || b >= r) {
    Z[e] = 0.0;
    return;
  }
  const int ia = idx[a], ib = idx[b];
  Z[e] = G[(size_t)ia * ldg + ib] / (sig[ia] * sig[ib]);
}

// M1 (nc x kz, row-major padded, pre-zeroed): M1[idx_a][b] = W(a, b) / sig[idx_a] for a < r,
// so that Y~[:, :nc] M1 = Y~_keep Sigma~^-1 W = Y W = Q~.  W column-major (ld ldw).
__global__ void k_build_m1(const double* W, int ldw, const int* idx, const double* sig, const int* rr,
                           int rb, int kz, double* M1, int ldm) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rb * kz) return;
  const int a = e / kz, b = e % kz;
  if (a >= *rr) return;
  const int ia = idx[a];
  M1[(size_t)ia * ldm + b] = W[(size_t)b * ldw + a] / sig[ia];
}

// Columns of K = T_keep W_keep^T Sigma~ (r2 x r) for the SVD of R = K V~_keep^T
// (reading R13): column b (length rb2, zero rows from r2 on) at Kc + b*rb2,
// rb columns (zero from r on):  K[a][b] = T[idx2_a] * W(b, idx2_a) * sig[idx_b].
__global__ void k_build_k(const double* T, const int* idx2, const int* rr2, int rb2, const double* W,
                          int ldw, const int* rr, int rb, const double* sig, const int* idx, double* Kc) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rb2 * rb) return;
  const int b = e / rb2, a = e % rb2;
  if (a >= *rr2 || b >= *rr) {
    Kc[e] = 0.0;
    return;
  }
  const int c2 = idx2[a];
  Kc[e] = T[c2] * W[(size_t)c2 * ldw + b] * sig[idx[b]];
}

// After the Jacobi SVD of K (column a of `cols`: [P(:, a) (rb2) ; J(:, a) (rb)]):
//   V(:, a) = V~_keep J(:, a)  (R = P Sigma (V~_keep J)^T), sign fixed (R5),
//   sigma[a], V (row-major, ldv), Ps = P * signs (column-major rb2 x rb2, zero from r2 on).
// Output columns a in [r2, rb2) (r2 = *rr2, kept rank of the second discard) are zeros.
// One CTA per 8 output columns; thread i computes row i of V(:, a0:a0+8).
static constexpr int SVO_COLS = 8;
__global__ void __launch_bounds__(256) k_svd_out(const double* cols, int ldc, const int* rr2, int rb2,
                                                 const int* rr, const double* vals, const double* Vt,
                                                 int w, const int* idx, double* sigma, double* V,
                                                 int64_t ldv, double* Ps) {
  __shared__ double sJ[256][SVO_COLS];
  __shared__ int sidx[256];
  __shared__ double sbest[8][SVO_COLS];
  __shared__ int sbi[8][SVO_COLS];
  __shared__ double ssign[SVO_COLS];
  const int r2 = *rr2, r = *rr;
  TCHECK(r <= 256 && r2 <= rb2 && w <= 256);  // sJ / sidx rows, one thread per row of V
  const int a0 = blockIdx.x * SVO_COLS, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nall = min(SVO_COLS, rb2 - a0);           // output columns of this CTA
  const int na = max(0, min(SVO_COLS, r2 - a0));      // ... that are real
  for (int e = tid; e < r * SVO_COLS; e += blockDim.x) {
    const int bb = e / SVO_COLS, q = e % SVO_COLS;
    sJ[bb][q] = q < na ? cols[(size_t)(a0 + q) * ldc + rb2 + bb] : 0.0;
  }
  for (int bb = tid; bb < r; bb += blockDim.x) sidx[bb] = idx[bb];
  __syncthreads();
  double v[SVO_COLS];
#pragma unroll
  for (int q = 0; q < SVO_COLS; ++q) v[q] = 0.0;
  const int i = tid;
  if (i < w)
    for (int bb = 0; bb < r; ++bb) {
      const double x = Vt[(size_t)sidx[bb] * w + i];
#pragma unroll
      for (int q = 0; q < SVO_COLS; ++q) v[q] = fma(x, sJ[bb][q], v[q]);
    }
  // sign of each column: its largest-|.| entry positive (ties -> lowest index)
#pragma unroll
  for (int q = 0; q < SVO_COLS; ++q) {
    double bv = i < w ? fabs(v[q]) : -1.0;
    int bi = i < w ? i : (1 << 30);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) bv = ov, bi = oi;
    }
    if (lane == 0) sbest[warp][q] = bv, sbi[warp][q] = bi;
  }
  __syncthreads();
  if (tid < SVO_COLS) {
    double bv = -1.0;
    int bi = 1 << 30;
    for (int ww = 0; ww < (int)(blockDim.x >> 5); ++ww)
      if (sbest[ww][tid] > bv || (sbest[ww][tid] == bv && sbi[ww][tid] < bi)) bv = sbest[ww][tid], bi = sbi[ww][tid];
    ssign[tid] = 1.0;  // resolved below by the owner of row bi
    sbi[0][tid] = bi;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < SVO_COLS; ++q)
    if (i == sbi[0][q] && i < w) ssign[q] = v[q] < 0.0 ? -1.0 : 1.0;
  __syncthreads();
  if (i < w)
#pragma unroll
    for (int q = 0; q < SVO_COLS; ++q)
      if (q < nall) V[(size_t)i * ldv + a0 + q] = q < na ? ssign[q] * v[q] : 0.0;
  for (int e = tid; e < nall * rb2; e += blockDim.x) {
    const int q = e / rb2, c = e % rb2;
    Ps[(size_t)(a0 + q) * rb2 + c] = (q < na && c < r2) ? ssign[q] * cols[(size_t)(a0 + q) * ldc + c] : 0.0;
  }
  if (tid < nall) sigma[a0 + tid] = tid < na ? vals[a0 + tid] : 0.0;
}

// M2 (nc x r2 row-major padded, pre-zeroed): M2[idx_b][a] = sum_c W(b, idx2_c) / (sig[idx_b] T[idx2_c]) Ps(c, a)
// so that Y~[:, :nc] M2 = Q~_keep T^-1 P = Q P = U.  b < r = *rr, a, c < r2 = *rr2.
__global__ void __launch_bounds__(256) k_build_m2(const double* W, int ldw, const int* rr, const int* idx,
                                                   const double* sig, const double* T, const int* idx2,
                                                   const int* rr2, int ldp, const double* Ps, double* M2,
                                                   int ldm) {
  // one CTA per row b: wrow[c] = W(b, idx2_c) / T[idx2_c] staged once, then thread a
  // forms sum_c wrow[c] Ps(c, a) in a fixed order
  __shared__ double wrow[256];
  const int b = blockIdx.x;
  if (b >= *rr) return;
  const int r2 = *rr2;
  TCHECK(r2 <= 256 && r2 <= ldm);
  for (int c = threadIdx.x; c < r2; c += blockDim.x) {
    const int c2 = idx2[c];
    wrow[c] = W[(size_t)c2 * ldw + b] / T[c2];
  }
  __syncthreads();
  const int ib = idx[b];
  const double inv = 1.0 / sig[ib];
  for (int a = threadIdx.x; a < r2; a += blockDim.x) {
    const double* pa = Ps + (size_t)a * ldp;
    double s = 0.0;
#pragma unroll 8
    for (int c = 0; c < r2; ++c) s = fma(wrow[c], pa[c], s);
    M2[(size_t)ib * ldm + a] = s * inv;
  }
}

// Packed lower triangle (w(w+1)/2, row-major (i, j<=i)) -> symmetric B (ldb).  Used after
// the allreduce of the packed Gram (half the bytes of the full matrix).
__global__ void k_unpack_sym(const double* packed, int w, double* B, int ldb) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= w * w) return;
  const int i = e / w, j = e % w;
  const int hi = max(i, j), lo = min(i, j);
  B[(size_t)i * ldb + j] = packed[(size_t)hi * (hi + 1) / 2 + lo];
}

// Low-rank final step: flip (V_A[:, a], Ut(:, a)) so V_A's largest entry is positive (R5),
// V_A row-major (n x ?, ldva), Ut row-major (r3 x r4, ldu_t).  Columns a < r4 = *rr4.
__global__ void __launch_bounds__(256) k_canon_lowrank(double* VA, int64_t ldva, int n, double* Ut, int ldut,
                                                        int r3, const int* rr4) {
  // one CTA per column a: block argmax of |V_A(:, a)| (ties -> lowest row), then a parallel flip
  __shared__ double sv[8];
  __shared__ int si[8];
  __shared__ double sgn;
  const int a = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (a >= *rr4) return;
  double bv = -1.0, val = 0.0;
  int bi = 1 << 30;
  for (int i = tid; i < n; i += blockDim.x) {
    const double v = VA[(size_t)i * ldva + a];
    if (fabs(v) > bv) bv = fabs(v), bi = i, val = v;  // increasing i: ties keep the lowest
  }
  double sv_ = val < 0.0 ? -1.0 : 1.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    const double os = __shfl_xor_sync(0xffffffffu, sv_, o);
    if (ob > bv || (ob == bv && oi < bi)) bv = ob, bi = oi, sv_ = os;
  }
  if (lane == 0) sv[warp] = bv, si[warp] = bi;
  __shared__ double ss[8];
  if (lane == 0) ss[warp] = sv_;
  __syncthreads();
  if (tid == 0) {
    double b = -1.0, g = 1.0;
    int i0 = 1 << 30;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
      if (sv[w] > b || (sv[w] == b && si[w] < i0)) b = sv[w], i0 = si[w], g = ss[w];
    sgn = g;
  }
  __syncthreads();
  if (sgn < 0) {
    for (int i = tid; i < n; i += blockDim.x) VA[(size_t)i * ldva + a] = -VA[(size_t)i * ldva + a];
    for (int i = tid; i < r3; i += blockDim.x) Ut[(size_t)i * ldut + a] = -Ut[(size_t)i * ldut + a];
  }
}

// 2-D strided copy (row-major), rows x cols.
__global__ void k_copy2d(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t rows,
                         int cols) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * cols) return;
  const int64_t i = e / cols;
  const int j = (int)(e % cols);
  dst[i * ldd + j] = src[i * lds + j];
}

__global__ void k_fill(double* p, int64_t n, double v) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) p[e] = v;
}

// ---------------------------------------------------------------- launchers --
static inline unsigned nb(int64_t n, int b = 256) { return (unsigned)((n + b - 1) / b); }

void symmetrize(double* B, int w, int ldb, cudaStream_t s) {
  k_symmetrize<<<nb((int64_t)w * w), 256, 0, s>>>(B, w, ldb);
}
void unpack_sym(const double* packed, int w, double* B, int ldb, cudaStream_t s) {
  k_unpack_sym<<<nb((int64_t)w * w), 256, 0, s>>>(packed, w, B, ldb);
}
void cols_to_m(const double* cols, int ldc, int k, int c, double* M, int ldm, int mrows,
               cudaStream_t s) {
  k_cols_to_m<<<nb((int64_t)mrows * ldm), 256, 0, s>>>(cols, ldc, k, c, M, ldm, mrows);
}
void rows_to_m(const double* src, int64_t lds, int k, int c, double* M, int ldm, int mrows,
               cudaStream_t s) {
  k_rows_to_m<<<nb((int64_t)mrows * ldm), 256, 0, s>>>(src, lds, k, c, M, ldm, mrows);
}
void discard(const double* nsq, int w, double wp, double* sig, int* idx, int* out, const int* nf,
             cudaStream_t s) {
  k_discard<<<1, 256, 0, s>>>(nsq, w, sqrt(wp), sig, idx, out, nf);
}
void alg3_out(const double* sig, const int* idx, const int* rr, int rb, const double* Vt, int w,
              double* M, int ldm, double* sigma, double* V, int64_t ldv, cudaStream_t s) {
  if (rb > 0) k_alg3_out<<<nb(rb, 64), 64, 0, s>>>(sig, idx, rr, rb, Vt, w, M, ldm, sigma, V, ldv);
}
void build_z(const double* G, int ldg, const int* idx, const double* sig, const int* rr, int rb,
             double* Z, cudaStream_t s) {
  if (rb > 0) k_build_z<<<nb((int64_t)rb * rb), 256, 0, s>>>(G, ldg, idx, sig, rr, rb, Z);
}
void build_m1(const double* W, int ldw, const int* idx, const double* sig, const int* rr, int rb,
              int kz, double* M1, int ldm, cudaStream_t s) {
  if (rb > 0 && kz > 0) k_build_m1<<<nb((int64_t)rb * kz), 256, 0, s>>>(W, ldw, idx, sig, rr, rb, kz, M1, ldm);
}
void build_k(const double* T, const int* idx2, const int* rr2, int rb2, const double* W, int ldw,
             const int* rr, int rb, const double* sig, const int* idx, double* Kc, cudaStream_t s) {
  if (rb > 0 && rb2 > 0)
    k_build_k<<<nb((int64_t)rb2 * rb), 256, 0, s>>>(T, idx2, rr2, rb2, W, ldw, rr, rb, sig, idx, Kc);
}
void svd_out(const double* cols, int ldc, const int* rr2, int rb2, const int* rr, const double* vals,
             const double* Vt, int w, const int* idx, double* sigma, double* V, int64_t ldv, double* Ps,
             cudaStream_t s) {
  if (rb2 > 0) k_svd_out<<<nb(rb2, SVO_COLS), 256, 0, s>>>(cols, ldc, rr2, rb2, rr, vals, Vt, w, idx, sigma, V, ldv, Ps);
}
void build_m2(const double* W, int ldw, const int* rr, int rb, const int* idx, const double* sig,
              const double* T, const int* idx2, const int* rr2, int ldp, const double* Ps, double* M2,
              int ldm, cudaStream_t s) {
  if (rb > 0 && ldp > 0) k_build_m2<<<rb, 256, 0, s>>>(W, ldw, rr, idx, sig, T, idx2, rr2, ldp, Ps, M2, ldm);
}
void canon_lowrank(double* VA, int64_t ldva, int n, double* Ut, int ldut, int r3, const int* rr4, int rb4,
                   cudaStream_t s) {
  if (rb4 > 0) k_canon_lowrank<<<rb4, 256, 0, s>>>(VA, ldva, n, Ut, ldut, r3, rr4);
}
void copy2d(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t rows, int cols,
            cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return;
  k_copy2d<<<nb(rows * cols), 256, 0, s>>>(src, lds, dst, ldd, rows, cols);
}
void fill(double* p, int64_t n, double v, cudaStream_t s) {
  if (n <= 0) return;
  k_fill<<<nb(n), 256, 0, s>>>(p, n, v);
}

}  // namespace tsk
