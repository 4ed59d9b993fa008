// Assembly kernels of the wide (256 < n <= 2048) Alg. 3/4 core: the small-core steps whose
// round-1 kernels hold a row of 256 in shared memory (svd_out, build_m2) become tiled FP64
// products over the bound r (<= 2048), plus the packing of the Gram for its allreduce.
//   V = V~_keep J              (Alg. 4 step 14: R = P Sigma (V~_keep J)^T)
//   M2 = S W T^-1 P            (Alg. 4 steps 12 and 15: U = Y~ M2)
// Fixed summation order everywhere (bit-identical on every rank).
#include <cstdint>

#include "common.cuh"
#include "small_kernels.h"

namespace tsk {

// packed lower triangle (row-major (i, j <= i)) of B (ldb) for the allreduce of the Gram
__global__ void k_pack_lower(const double* B, int w, int ldb, double* packed) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)w * (w + 1) / 2) return;
  int i = (int)((sqrt(8.0 * (double)e + 1.0) - 1.0) * 0.5);
  while ((int64_t)i * (i + 1) / 2 > e) --i;
  while ((int64_t)(i + 1) * (i + 2) / 2 <= e) ++i;
  const int j = (int)(e - (int64_t)i * (i + 1) / 2);
  packed[e] = B[(size_t)i * ldb + j];
}

// 16 x 16 output tiles, K in steps of 16, smem staging; C(i, j) = sum_k A(i, k) B(k, j)
// accumulated in k order (one FMA chain per output: deterministic).
static constexpr int TT = 16;

// V~_keep J:  A(i, b) = Vt[idx[b] * w + i] (eigenvector idx_b of B, contiguous),
//             B(b, a) = J(b, a) = cols[a * ldc + rb2 + b]  (accumulator rows of SVD column a)
//             C: out[i * ldo + a], i < w, a < rb2; k = b < r (*rr)
__global__ void __launch_bounds__(TT * TT) k_wide_vj(const double* Vt, int w, const int* idx, const int* rr,
                                                   const double* cols, int ldc, int rb2, double* out, int ldo) {
  __shared__ double As[TT][TT + 1], Bs[TT][TT + 1];
  const int tx = threadIdx.x % TT, ty = threadIdx.x / TT;
  const int i = blockIdx.y * TT + ty, a = blockIdx.x * TT + tx;
  const int r = *rr;
  double acc = 0.0;
  for (int k0 = 0; k0 < r; k0 += TT) {
    const int kb = k0 + tx;  // A tile: row i (ty), column kb (tx)
    As[ty][tx] = (i < w && kb < r) ? Vt[(size_t)idx[kb] * w + i] : 0.0;
    const int kr = k0 + ty;  // B tile: row kr (ty), column a (tx)
    Bs[ty][tx] = (kr < r && a < rb2) ? cols[(size_t)a * ldc + rb2 + kr] : 0.0;
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TT; ++kk) acc = fma(As[ty][kk], Bs[kk][tx], acc);
    __syncthreads();
  }
  if (i < w && a < rb2) out[(size_t)i * ldo + a] = acc;
}

// Signs (reading R5) and outputs of the wide SVD, one CTA per column a < rb2:
//   s_a = sign of the largest-|.| entry of V(:, a) (ties -> lowest row);
//   V[:, a] = s_a VJ(:, a), Ps(:, a) = s_a P(:, a) (rows < r2), sigma[a] = vals[a]; a >= r2: zeros.
__global__ void __launch_bounds__(256) k_wide_svd_sign(const double* VJ, int ldvj, int w, const double* cols, int ldc,
                                                       const int* rr2, int rb2, const double* vals, double* sigma,
                                                       double* V, int64_t ldv, double* Ps) {
  const int a = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r2 = *rr2;
  __shared__ double sb[8];
  __shared__ int si[8];
  __shared__ double ssg;
  if (a >= r2) {
    for (int i = tid; i < w; i += blockDim.x) V[(size_t)i * ldv + a] = 0.0;
    for (int c = tid; c < rb2; c += blockDim.x) Ps[(size_t)a * rb2 + c] = 0.0;
    if (tid == 0) sigma[a] = 0.0;
    return;
  }
  double bv = -1.0, val = 0.0;
  int bi = 1 << 30;
  for (int i = tid; i < w; i += blockDim.x) {
    const double v = VJ[(size_t)i * ldvj + a];
    if (fabs(v) > bv) bv = fabs(v), bi = i, val = v;
  }
  double sg = val < 0.0 ? -1.0 : 1.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    const double os = __shfl_xor_sync(0xffffffffu, sg, o);
    if (ob > bv || (ob == bv && oi < bi)) bv = ob, bi = oi, sg = os;
  }
  __shared__ double ss[8];
  if (lane == 0) sb[warp] = bv, si[warp] = bi, ss[warp] = sg;
  __syncthreads();
  if (tid == 0) {
    double b = -1.0, g = 1.0;
    int i0 = 1 << 30;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q)
      if (sb[q] > b || (sb[q] == b && si[q] < i0)) b = sb[q], i0 = si[q], g = ss[q];
    ssg = g;
  }
  // the column's norm (V~_keep J has unit columns in exact arithmetic; the accumulated
  // rotations drift in norm at the rounding level): fixed-order block sum
  double nn = 0.0;
  for (int i = tid; i < w; i += blockDim.x) nn = fma(VJ[(size_t)i * ldvj + a], VJ[(size_t)i * ldvj + a], nn);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nn += __shfl_xor_sync(0xffffffffu, nn, o);
  __shared__ double snn[8];
  if (lane == 0) snn[warp] = nn;
  __syncthreads();
  double tot = 0.0;
  for (int q = 0; q < (int)(blockDim.x >> 5); ++q) tot += snn[q];
  const double s = ssg / sqrt(tot);
  for (int i = tid; i < w; i += blockDim.x) V[(size_t)i * ldv + a] = s * VJ[(size_t)i * ldvj + a];
  for (int c = tid; c < rb2; c += blockDim.x) Ps[(size_t)a * rb2 + c] = c < r2 ? ssg * cols[(size_t)a * ldc + c] : 0.0;
  if (tid == 0) sigma[a] = vals[a];
}

// M2[idx_b][a] = (sum_{c < r2} W(b, idx2_c) / T[idx2_c] * Ps(c, a)) / sig[idx_b],  b < r, a < r2
// (W column-major, ld ldw: W(b, j) = W[j * ldw + b]; Ps column-major, ld ldp; M2 pre-zeroed)
__global__ void __launch_bounds__(TT * TT) k_wide_m2(const double* W, int ldw, const int* rr, const int* idx,
                                                   const double* sig, const double* T, const int* idx2,
                                                   const int* rr2, int ldp, const double* Ps, double* M2, int ldm,
                                                   int rb) {
  __shared__ double As[TT][TT + 1], Bs[TT][TT + 1];
  const int tx = threadIdx.x % TT, ty = threadIdx.x / TT;
  const int b = blockIdx.y * TT + ty, a = blockIdx.x * TT + tx;
  const int r = *rr, r2 = *rr2;
  double acc = 0.0;
  for (int k0 = 0; k0 < r2; k0 += TT) {
    const int kc = k0 + tx;
    if (b < r && kc < r2) {
      const int c2 = idx2[kc];
      As[ty][tx] = W[(size_t)c2 * ldw + b] / T[c2];
    } else {
      As[ty][tx] = 0.0;
    }
    const int kr = k0 + ty;
    Bs[ty][tx] = (kr < r2 && a < r2) ? Ps[(size_t)a * ldp + kr] : 0.0;
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TT; ++kk) acc = fma(As[ty][kk], Bs[kk][tx], acc);
    __syncthreads();
  }
  if (b < r && a < r2 && b < rb) M2[(size_t)idx[b] * ldm + a] = acc / sig[idx[b]];
}

static inline unsigned nbk(int64_t n, int b = 256) { return (unsigned)((n + b - 1) / b); }

void pack_lower(const double* B, int w, int ldb, double* packed, cudaStream_t s) {
  const int64_t n = (int64_t)w * (w + 1) / 2;
  if (n > 0) k_pack_lower<<<nbk(n), 256, 0, s>>>(B, w, ldb, packed);
}
void wide_svd_out(const double* cols, int ldc, const int* rr2, int rb2, const int* rr, int rb,
                  const double* vals, const double* Vt, int w, const int* idx, double* sigma, double* V,
                  int64_t ldv, double* Ps, double* vj_tmp, cudaStream_t s) {
  if (rb2 <= 0) return;
  dim3 grid((rb2 + TT - 1) / TT, (w + TT - 1) / TT);
  k_wide_vj<<<grid, TT * TT, 0, s>>>(Vt, w, idx, rr, cols, ldc, rb2, vj_tmp, rb2);
  k_wide_svd_sign<<<rb2, 256, 0, s>>>(vj_tmp, rb2, w, cols, ldc, rr2, rb2, vals, sigma, V, ldv, Ps);
  (void)rb;
}
void wide_build_m2(const double* W, int ldw, const int* rr, int rb, const int* idx, const double* sig,
                   const double* T, const int* idx2, const int* rr2, int rb2, const double* Ps, double* M2, int ldm,
                   cudaStream_t s) {
  if (rb <= 0 || rb2 <= 0) return;
  dim3 grid((rb2 + TT - 1) / TT, (rb + TT - 1) / TT);
  k_wide_m2<<<grid, TT * TT, 0, s>>>(W, ldw, rr, idx, sig, T, idx2, rr2, rb2, Ps, M2, ldm, rb);
}

}  // namespace tsk
