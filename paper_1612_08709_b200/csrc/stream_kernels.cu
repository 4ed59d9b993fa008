// Streaming FP64 passes over the row-sharded tall matrix (sm_100a).
//
//   syrk   : B_p = X_p^T X_p            Alg. 3/4 step 1, Alg. 4 step 7
//   gemm_nn: Y = X M (+ column norms)   Alg. 3/4 steps 3-4, steps 9-10
//                                       (P:674-678), step 15; Alg. 5 steps 3, 8
//   gemm_tn: Z_p = X_p^T Y_p            Alg. 5 step 5, Alg. 6 step 1
//
// All three stream row blocks of X from HBM into shared memory with the TMA
// bulk-copy engine (cp.async.bulk, one 16-B-aligned row segment per copy,
// completion on an mbarrier), multi-stage, and run the contraction on the FP64
// tensor pipe (mma.sync m8n8k4 f64 -> DMMA.8x8x4; on B200 this is the only
// FP64 MMA shape -- tcgen05 has no f64 kind).  Reductions over rows are split
// across CTAs into per-CTA partials that are summed in a fixed order by a
// separate kernel, so every result is bitwise deterministic.
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "kernels.h"

namespace tsk {

const DevInfo& dev_info() {
  static DevInfo d = [] {
    DevInfo x;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&x.sms, cudaDevAttrMultiProcessorCount, dev);
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    x.smem_optin = (size_t)v;
    return x;
  }();
  return d;
}

static constexpr int kBarBytes = 128;  // room for up to 16 mbarriers at the start of smem

// ============================================================== SYRK (Gram) ==
// CTA b owns rows [b*rpc, (b+1)*rpc).  Output tiles of B are 8x8 DMMA tiles in
// the lower triangle, grouped in 2x2 "units" (16x16) so each fragment load
// feeds two MMAs.  Because both operands are columns of the same row block,
// the fragment of column block c at k-step kk is Xs[kk*4 + t][c*8 + g] for the
// A role (A = X^T, 8x4) and the B role (4x8) alike.
static constexpr int SYRK_KR = 32;

template <int UPW>
__global__ void __launch_bounds__(512) syrk_kernel(const double* __restrict__ X, int64_t ldx,
                                                   int64_t m, int w, int wc, int64_t rpc,
                                                   double* __restrict__ part, int nst, int ups) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  double* buf = reinterpret_cast<double*>(smem + kBarBytes);
  const int lds = smem_ld(w);
  const int stage_d = SYRK_KR * lds;
  const int nb = (w + 7) >> 3, nu = (nb + 1) >> 1, nunits = nu * (nu + 1) / 2;
  const int wp = nb * 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int nw = blockDim.x >> 5;
  const int64_t r0 = (int64_t)blockIdx.x * rpc;
  const int64_t r1 = min(m, r0 + rpc);
  const int nsteps = r1 > r0 ? (int)ceil_div(r1 - r0, SYRK_KR) : 0;

  for (int i = threadIdx.x; i < nst * stage_d; i += blockDim.x) buf[i] = 0.0;
  fence_proxy_async();
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  // this warp's units (ui >= uj), decoded from the linear lower-triangle index
  int ci0[UPW], ci1[UPW], cj0[UPW], cj1[UPW];
  bool uv[UPW], dg[UPW], vi1[UPW], vj1[UPW];
#pragma unroll
  const int ubase = blockIdx.y * ups, uend = min(nunits, ubase + ups);
  for (int k = 0; k < UPW; ++k) {
    const int u = ubase + warp + k * nw;
    uv[k] = u < uend;
    int ui = 0;
    while ((ui + 1) * (ui + 2) / 2 <= u) ++ui;
    const int uj = u - ui * (ui + 1) / 2;
    dg[k] = ui == uj;
    vi1[k] = 2 * ui + 1 < nb;
    vj1[k] = 2 * uj + 1 < nb;
    ci0[k] = (2 * ui) * 8 + g;
    ci1[k] = vi1[k] ? (2 * ui + 1) * 8 + g : g;
    cj0[k] = (2 * uj) * 8 + g;
    cj1[k] = vj1[k] ? (2 * uj + 1) * 8 + g : g;
    if (!uv[k]) ci0[k] = ci1[k] = cj0[k] = cj1[k] = g;
  }
  double acc[UPW][4][2];
#pragma unroll
  for (int k = 0; k < UPW; ++k)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[k][q][0] = acc[k][q][1] = 0.0;

  auto issue = [&](int s) {  // executed by warp 0
    const int b = s % nst;
    const int64_t rs = r0 + (int64_t)s * SYRK_KR;
    const int nr = (int)min64(SYRK_KR, r1 - rs);
    double* dst = buf + b * stage_d;
    if (lane == 0) mbar_arrive_expect_tx(&bar[b], (uint32_t)(nr * wc * 8));
    __syncwarp();
    for (int i = lane; i < nr; i += 32) bulk_g2s(dst + i * lds, X + (rs + i) * ldx, wc * 8, &bar[b]);
    for (int i = nr; i < SYRK_KR; ++i)
      for (int j = lane; j < wc; j += 32) dst[i * lds + j] = 0.0;
  };

  if (warp == 0)
    for (int s = 0; s < min(nst - 1, nsteps); ++s) issue(s);
  __syncthreads();
  for (int s = 0; s < nsteps; ++s) {
    if (warp == 0 && s + nst - 1 < nsteps) issue(s + nst - 1);
    const int b = s % nst;
    mbar_wait(&bar[b], (uint32_t)((s / nst) & 1));
    const double* base = buf + b * stage_d + t * lds;
#pragma unroll
    for (int kk = 0; kk < SYRK_KR / 4; ++kk) {
      const double* rp = base + kk * 4 * lds;
#pragma unroll
      for (int k = 0; k < UPW; ++k) {
        if (!uv[k]) continue;
        const double fi0 = rp[ci0[k]], fi1 = rp[ci1[k]];
        const double fj0 = rp[cj0[k]], fj1 = rp[cj1[k]];
        dmma(acc[k][0], fi0, fj0);
        if (!dg[k] && vj1[k]) dmma(acc[k][1], fi0, fj1);
        if (vi1[k]) dmma(acc[k][2], fi1, fj0);
        if (vi1[k] && vj1[k]) dmma(acc[k][3], fi1, fj1);
      }
    }
    __syncthreads();
  }

  double* P = part + (size_t)blockIdx.x * wp * wp;
#pragma unroll
  for (int k = 0; k < UPW; ++k) {
    if (!uv[k]) continue;
    const int u = ubase + warp + k * nw;
    int ui = 0;
    while ((ui + 1) * (ui + 2) / 2 <= u) ++ui;
    const int uj = u - ui * (ui + 1) / 2;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int I = 2 * ui + (q >> 1), J = 2 * uj + (q & 1);
      if (I >= nb || J >= nb || J > I) continue;
      double2 v = make_double2(acc[k][q][0], acc[k][q][1]);
      *reinterpret_cast<double2*>(P + (size_t)(I * 8 + g) * wp + J * 8 + 2 * t) = v;
    }
  }
}

// Units per warp (UPW), warps per CTA and unit splits (grid.y): at most 16
// warps and 6 units (48 accumulator doubles) per warp; beyond 96 units
// (n > 208) the units are split over grid.y CTAs that read the same rows.
static int syrk_upw(int w, int* nw_out, int* splits_out = nullptr, int* ups_out = nullptr) {
  const int nb = (w + 7) / 8, nu = (nb + 1) / 2, nunits = nu * (nu + 1) / 2;
  const int splits = (int)ceil_div(nunits, 96);
  const int ups = (int)ceil_div(nunits, splits);
  int upw = (int)ceil_div(ups, 16);
  if (upw == 5) upw = 6;
  *nw_out = (int)ceil_div(ups, upw);
  if (splits_out) *splits_out = splits;
  if (ups_out) *ups_out = ups;
  return upw;
}

static int syrk_nst(int w) {
  const size_t stage = (size_t)SYRK_KR * smem_ld(w) * 8;
  size_t budget = dev_info().smem_optin - kBarBytes;
  int nst = (int)std::min<size_t>(4, budget / stage);
  return std::max(nst, 2);
}

int syrk_partials_grid(int64_t m, int w) {
  int nw;
  syrk_upw(w, &nw);
  const size_t smem = kBarBytes + (size_t)syrk_nst(w) * SYRK_KR * smem_ld(w) * 8;
  int per_sm = (int)std::max<size_t>(1, std::min<size_t>(228 * 1024 / (smem + 1024), 2048 / (32 * nw)));
  per_sm = std::min(per_sm, 4);
  int64_t g = (int64_t)dev_info().sms * per_sm;
  int64_t maxg = std::max<int64_t>(1, ceil_div(m, SYRK_KR));
  return (int)std::max<int64_t>(1, std::min(g, maxg));
}

size_t syrk_partials_doubles(int64_t m, int w) {
  const int wp = pad8(w);
  return (size_t)syrk_partials_grid(m, w) * wp * wp;
}

template <int UPW>
static cudaError_t syrk_go(dim3 grid, int nw, size_t smem, const double* X, int64_t ldx, int64_t m,
                           int w, int wc, int64_t rpc, double* part, int nst, int ups,
                           cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(syrk_kernel<UPW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  syrk_kernel<UPW><<<grid, nw * 32, smem, s>>>(X, ldx, m, w, wc, rpc, part, nst, ups);
  return cudaGetLastError();
}

cudaError_t launch_syrk(const double* X, int64_t ldx, int64_t m, int w, double* part,
                        cudaStream_t s) {
  int nw, splits, ups;
  const int upw = syrk_upw(w, &nw, &splits, &ups);
  const int nst = syrk_nst(w);
  const int gx = syrk_partials_grid(m, w);
  const dim3 grid(gx, splits);
  int64_t rpc = ceil_div(std::max<int64_t>(m, 1), gx);
  rpc = ceil_div(rpc, SYRK_KR) * SYRK_KR;
  const int wc = (w + 1) & ~1;  // bulk copies move whole 16-B granules (ldx >= wc checked by caller)
  const size_t smem = kBarBytes + (size_t)nst * SYRK_KR * smem_ld(w) * 8;
  switch (upw) {
    case 1: return syrk_go<1>(grid, nw, smem, X, ldx, m, w, wc, rpc, part, nst, ups, s);
    case 2: return syrk_go<2>(grid, nw, smem, X, ldx, m, w, wc, rpc, part, nst, ups, s);
    case 3: return syrk_go<3>(grid, nw, smem, X, ldx, m, w, wc, rpc, part, nst, ups, s);
    case 4: return syrk_go<4>(grid, nw, smem, X, ldx, m, w, wc, rpc, part, nst, ups, s);
    default: return syrk_go<6>(grid, nw, smem, X, ldx, m, w, wc, rpc, part, nst, ups, s);
  }
}

// Fixed-order two-level sum over partials: groups of ~sqrt(np) summed
// sequentially, then the group sums sequentially (error ~2 sqrt(np) eps).
__device__ __forceinline__ double sum_parts(const double* p, int np, size_t stride) {
  int gs = 1;
  while (gs * gs < np) ++gs;
  double tot = 0.0;
  for (int p0 = 0; p0 < np; p0 += gs) {
    double s = 0.0;
    const int p1 = min(np, p0 + gs);
    for (int q = p0; q < p1; ++q) s += p[(size_t)q * stride];
    tot += s;
  }
  return tot;
}

__global__ void reduce_sym_kernel(const double* __restrict__ part, int np, int w, int wp,
                                  double* __restrict__ B, int ldb) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= w * w) return;
  const int i = e / w, j = e % w;
  if (j > i) return;
  const double v = sum_parts(part + (size_t)i * wp + j, np, (size_t)wp * wp);
  B[(size_t)i * ldb + j] = v;
  B[(size_t)j * ldb + i] = v;
}

cudaError_t launch_reduce_sym(const double* part, int np, int w, double* B, int ldb,
                              cudaStream_t s) {
  const int n = w * w;
  reduce_sym_kernel<<<(int)ceil_div(n, 256), 256, 0, s>>>(part, np, w, pad8(w), B, ldb);
  return cudaGetLastError();
}

__global__ void reduce_parts_kernel(const double* __restrict__ part, int np, int64_t stride,
                                    int64_t len, double* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= len) return;
  out[e] = sum_parts(part + e, np, (size_t)stride);
}

cudaError_t launch_reduce_parts(const double* part, int np, int64_t stride, int64_t len,
                                double* out, cudaStream_t s) {
  if (len <= 0) return cudaSuccess;
  reduce_parts_kernel<<<(int)ceil_div(len, 256), 256, 0, s>>>(part, np, stride, len, out);
  return cudaGetLastError();
}

// ================================================================= GEMM NN ==
// Y[r, :c] = X[r, :k] M.  A CTA owns row tiles of R = 64*MI rows and ALL c
// columns (so the product may overwrite X in place: every row is read into
// shared memory before it is written).  Warp w computes row blocks
// w*MI .. w*MI+MI-1 against all NI = ceil(c/8) column blocks.  K is streamed in
// chunks of 32: a stage holds X[rows, k0:k0+32] (one bulk copy per row) and
// M[k0:k0+32, :] (one bulk copy; M is stored with ld = smem_ld(c)).
static constexpr int NN_KC = 32;
static constexpr int NN_WARPS = 8;

template <int MI, int NI>
__global__ void __launch_bounds__(256) gemm_nn_kernel(const double* X, int64_t ldx, int64_t m,
                                                      int kc_count, int kcopy,
                                                      const double* __restrict__ M, int c,
                                                      double* Y, int64_t ldy,
                                                      double* __restrict__ norm_part, int nst) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int R = 8 * MI * NN_WARPS;
  constexpr int LDX = NN_KC + 4;  // smem_ld(32)
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  double* buf = reinterpret_cast<double*>(smem + kBarBytes);
  const int ldm = smem_ld(c);
  const int stage_d = R * LDX + NN_KC * ldm;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int64_t ntiles = ceil_div(m, R);
  const int64_t mytiles =
      blockIdx.x < ntiles ? ceil_div(ntiles - blockIdx.x, (int64_t)gridDim.x) : 0;
  const int64_t nsteps = mytiles * kc_count;

  for (int i = threadIdx.x; i < nst * stage_d; i += blockDim.x) buf[i] = 0.0;
  double* red = buf;  // reused after the main loop for the norm reduction
  fence_proxy_async();
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  auto issue = [&](int64_t s) {  // warp 0
    const int b = (int)(s % nst);
    const int64_t tile = blockIdx.x + (s / kc_count) * gridDim.x;
    const int kc = (int)(s % kc_count);
    const int64_t row0 = tile * R;
    const int nr = (int)min64(R, m - row0);
    const int k0 = kc * NN_KC;
    const int kw = min(NN_KC, kcopy - k0);
    double* xs = buf + b * stage_d;
    double* ms = xs + R * LDX;
    if (lane == 0) mbar_arrive_expect_tx(&bar[b], (uint32_t)(nr * kw * 8 + NN_KC * ldm * 8));
    __syncwarp();
    for (int i = lane; i < nr; i += 32) bulk_g2s(xs + i * LDX, X + (row0 + i) * ldx + k0, kw * 8, &bar[b]);
    if (lane == 31) bulk_g2s(ms, M + (size_t)k0 * ldm, NN_KC * ldm * 8, &bar[b]);
    for (int i = nr; i < R; ++i) xs[i * LDX + lane] = 0.0;
  };

  double acc[MI][NI][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  double nacc[NI][2];
#pragma unroll
  for (int j = 0; j < NI; ++j) nacc[j][0] = nacc[j][1] = 0.0;

  if (warp == 0)
    for (int64_t s = 0; s < min64(nst - 1, nsteps); ++s) issue(s);
  __syncthreads();
  for (int64_t s = 0; s < nsteps; ++s) {
    if (warp == 0 && s + nst - 1 < nsteps) issue(s + nst - 1);
    const int b = (int)(s % nst);
    mbar_wait(&bar[b], (uint32_t)((s / nst) & 1));
    const double* xs = buf + b * stage_d + (warp * MI * 8 + g) * LDX + t;
    const double* ms = buf + b * stage_d + R * LDX + t * ldm + g;
    // k-steps in this chunk: the last chunk of a row tile may be partial
    const int kc_here = (int)(s % kc_count);
    const int nks = min(NN_KC / 4, (kcopy - kc_here * NN_KC + 3) / 4);
#pragma unroll
    for (int kk = 0; kk < NN_KC / 4; ++kk) {
      if (kk >= nks) break;
      double a[MI];
#pragma unroll
      for (int i = 0; i < MI; ++i) a[i] = xs[i * 8 * LDX + kk * 4];
#pragma unroll
      for (int j = 0; j < NI; ++j) {
        const double bf = ms[kk * 4 * ldm + j * 8];
#pragma unroll
        for (int i = 0; i < MI; ++i) dmma(acc[i][j], a[i], bf);
      }
    }
    if ((s + 1) % kc_count == 0) {  // tile complete: epilogue
      const int64_t tile = blockIdx.x + (s / kc_count) * gridDim.x;
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const int64_t row = tile * R + (warp * MI + i) * 8 + g;
        const bool rv = row < m;
#pragma unroll
        for (int j = 0; j < NI; ++j) {
          const int col = j * 8 + 2 * t;
          if (rv) {
            if (norm_part) {
              nacc[j][0] += acc[i][j][0] * acc[i][j][0];
              nacc[j][1] += acc[i][j][1] * acc[i][j][1];
            }
            if (Y) {
              if (col + 1 < c)
                *reinterpret_cast<double2*>(Y + row * ldy + col) =
                    make_double2(acc[i][j][0], acc[i][j][1]);
              else if (col < c)
                Y[row * ldy + col] = acc[i][j][0];
            }
          }
          acc[i][j][0] = acc[i][j][1] = 0.0;
        }
      }
    }
    __syncthreads();
  }

  if (norm_part) {
    // rows of this thread -> reduce over g (lanes xor 4, 8, 16), then over warps in order
#pragma unroll
    for (int j = 0; j < NI; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double v = nacc[j][e];
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        if (g == 0) red[warp * NI * 8 + j * 8 + 2 * t + e] = v;
      }
    __syncthreads();
    const int cp = NI * 8;
    for (int col = threadIdx.x; col < cp; col += blockDim.x) {
      double v = 0.0;
      for (int w = 0; w < NN_WARPS; ++w) v += red[w * cp + col];
      norm_part[(size_t)blockIdx.x * cp + col] = v;
    }
  }
}

static int nn_mi_max(int ni) { return std::max(1, std::min(4, 28 / ni)); }

static size_t nn_stage_bytes(int mi, int c) {
  return (size_t)(8 * mi * NN_WARPS * (NN_KC + 4) + NN_KC * smem_ld(c)) * 8;
}

struct NnPlan {
  int mi, ni, nst, grid;
  size_t smem;
};

static NnPlan plan_nn(int64_t m, int c) {
  NnPlan p;
  p.ni = (c + 7) / 8;
  const int sms = dev_info().sms;
  const size_t budget = dev_info().smem_optin - kBarBytes;
  // choose MI (rows per tile = 64*MI) minimising the busiest CTA's row count
  int best_mi = 1;
  int64_t best_cost = INT64_MAX;
  for (int mi = 1; mi <= nn_mi_max(p.ni); ++mi) {
    if (2 * nn_stage_bytes(mi, c) > budget) continue;
    const int64_t R = 64 * mi, tiles = ceil_div(m, R);
    const int64_t cost = ceil_div(tiles, sms) * R;
    if (cost < best_cost || (cost == best_cost && mi > best_mi)) best_cost = cost, best_mi = mi;
  }
  p.mi = best_mi;
  p.nst = (int)std::min<size_t>(4, budget / nn_stage_bytes(p.mi, c));
  p.smem = kBarBytes + (size_t)p.nst * nn_stage_bytes(p.mi, c);
  p.grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(m, 64 * p.mi), sms));
  return p;
}

int gemm_nn_grid(int64_t m, int c) { return plan_nn(m, c).grid; }
size_t gemm_nn_m_doubles(int k, int c) { return (size_t)ceil_div(k + 1, NN_KC) * NN_KC * smem_ld(c); }

template <int MI, int NI>
static cudaError_t nn_go(const NnPlan& p, const double* X, int64_t ldx, int64_t m, int k,
                         const double* M, int c, double* Y, int64_t ldy, double* norm_part,
                         cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(gemm_nn_kernel<MI, NI>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
  if (e != cudaSuccess) return e;
  const int kcopy = (k + 1) & ~1;
  const int kcc = (int)ceil_div(kcopy, NN_KC);
  gemm_nn_kernel<MI, NI><<<p.grid, NN_WARPS * 32, p.smem, s>>>(X, ldx, m, kcc, kcopy, M, c, Y, ldy,
                                                               norm_part, p.nst);
  return cudaGetLastError();
}

template <int NI>
static cudaError_t nn_mi(const NnPlan& p, const double* X, int64_t ldx, int64_t m, int k,
                         const double* M, int c, double* Y, int64_t ldy, double* np,
                         cudaStream_t s) {
  switch (p.mi) {
    case 1: return nn_go<1, NI>(p, X, ldx, m, k, M, c, Y, ldy, np, s);
    case 2: if constexpr (28 / NI >= 2) return nn_go<2, NI>(p, X, ldx, m, k, M, c, Y, ldy, np, s);
            [[fallthrough]];
    case 3: if constexpr (28 / NI >= 3) return nn_go<3, NI>(p, X, ldx, m, k, M, c, Y, ldy, np, s);
            [[fallthrough]];
    default: if constexpr (28 / NI >= 4) return nn_go<4, NI>(p, X, ldx, m, k, M, c, Y, ldy, np, s);
             return nn_go<1, NI>(p, X, ldx, m, k, M, c, Y, ldy, np, s);
  }
}

cudaError_t launch_gemm_nn(const double* X, int64_t ldx, int64_t m, int k, const double* M,
                           int c, double* Y, int64_t ldy, double* norm_part, cudaStream_t s) {
  if (m <= 0 || c <= 0) return cudaSuccess;
  const NnPlan p = plan_nn(m, c);
#define NN_CASE(N) \
  case N: return nn_mi<N>(p, X, ldx, m, k, M, c, Y, ldy, norm_part, s);
  switch (p.ni) {
    NN_CASE(1) NN_CASE(2) NN_CASE(3) NN_CASE(4) NN_CASE(5) NN_CASE(6) NN_CASE(7) NN_CASE(8)
    NN_CASE(9) NN_CASE(10) NN_CASE(11) NN_CASE(12) NN_CASE(13) NN_CASE(14) NN_CASE(15)
    NN_CASE(16) NN_CASE(17) NN_CASE(18) NN_CASE(19) NN_CASE(20) NN_CASE(21) NN_CASE(22)
    NN_CASE(23) NN_CASE(24) NN_CASE(25) NN_CASE(26) NN_CASE(27) NN_CASE(28) NN_CASE(29)
    NN_CASE(30) NN_CASE(31) NN_CASE(32)
    default: return cudaErrorInvalidValue;
  }
#undef NN_CASE
}

// ================================================================= GEMM TN ==
// Zp[split] = X[rows, c0:c0+CB]^T Y[rows, :l] for column block c0 and the
// split's row range.  Warp w owns X-column blocks w*MI..w*MI+MI-1 and all NBL
// column blocks of Y.  Fragments: A = X^T (8x4) -> Xs[k][i0+g], B = Y (4x8)
// -> Ys[k][j0+g], k = kk*4 + t.
static constexpr int TN_WARPS = 8;

template <int MI, int NBL>
__global__ void __launch_bounds__(256) gemm_tn_kernel(const double* __restrict__ X, int64_t ldx,
                                                      int64_t m, int n,
                                                      const double* __restrict__ Y, int64_t ldy,
                                                      int lcopy, int64_t rps,
                                                      double* __restrict__ part, int ldz,
                                                      int64_t n_pad, int KR, int nst) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int CB = 8 * MI * TN_WARPS;
  constexpr int LDXS = CB + 4;
  constexpr int LDYS = NBL * 8 + 4;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  double* buf = reinterpret_cast<double*>(smem + kBarBytes);
  const int stage_d = KR * (LDXS + LDYS);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int c0 = blockIdx.x * CB;
  const int cw = min(CB, n - c0);  // even (n even, CB multiple of 64)
  const int64_t r0 = (int64_t)blockIdx.y * rps;
  const int64_t r1 = min(m, r0 + rps);
  const int nsteps = r1 > r0 ? (int)ceil_div(r1 - r0, KR) : 0;

  for (int i = threadIdx.x; i < nst * stage_d; i += blockDim.x) buf[i] = 0.0;
  fence_proxy_async();
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  auto issue = [&](int s) {
    const int b = s % nst;
    const int64_t rs = r0 + (int64_t)s * KR;
    const int nr = (int)min64(KR, r1 - rs);
    double* xs = buf + b * stage_d;
    double* ys = xs + KR * LDXS;
    if (lane == 0) mbar_arrive_expect_tx(&bar[b], (uint32_t)(nr * (cw + lcopy) * 8));
    __syncwarp();
    for (int i = lane; i < nr; i += 32) {
      bulk_g2s(xs + i * LDXS, X + (rs + i) * ldx + c0, cw * 8, &bar[b]);
      bulk_g2s(ys + i * LDYS, Y + (rs + i) * ldy, lcopy * 8, &bar[b]);
    }
    for (int i = nr; i < KR; ++i) {
      for (int j = lane; j < cw; j += 32) xs[i * LDXS + j] = 0.0;
      for (int j = lane; j < lcopy; j += 32) ys[i * LDYS + j] = 0.0;
    }
  };

  double acc[MI][NBL][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NBL; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  if (warp == 0)
    for (int s = 0; s < min(nst - 1, nsteps); ++s) issue(s);
  __syncthreads();
  for (int s = 0; s < nsteps; ++s) {
    if (warp == 0 && s + nst - 1 < nsteps) issue(s + nst - 1);
    const int b = s % nst;
    mbar_wait(&bar[b], (uint32_t)((s / nst) & 1));
    const double* xs = buf + b * stage_d + t * LDXS + warp * MI * 8 + g;
    const double* ys = buf + b * stage_d + KR * LDXS + t * LDYS + g;
    for (int kk = 0; kk < KR / 4; ++kk) {
      double a[MI], bf[NBL];
#pragma unroll
      for (int i = 0; i < MI; ++i) a[i] = xs[kk * 4 * LDXS + i * 8];
#pragma unroll
      for (int j = 0; j < NBL; ++j) bf[j] = ys[kk * 4 * LDYS + j * 8];
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NBL; ++j) dmma(acc[i][j], a[i], bf[j]);
    }
    __syncthreads();
  }

  double* P = part + (size_t)blockIdx.y * n_pad * ldz;
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const int row = c0 + (warp * MI + i) * 8 + g;
    if (row >= n) continue;
#pragma unroll
    for (int j = 0; j < NBL; ++j)
      *reinterpret_cast<double2*>(P + (size_t)row * ldz + j * 8 + 2 * t) =
          make_double2(acc[i][j][0], acc[i][j][1]);
  }
}

TnPlan plan_gemm_tn(int64_t m, int n, int l) {
  TnPlan p;
  p.nbl = (l + 7) / 8;
  p.mi = p.nbl <= 4 ? 4 : (p.nbl <= 8 ? 2 : 1);
  p.cb = 8 * p.mi * TN_WARPS;
  p.ldz = p.nbl * 8;
  p.colblocks = (int)ceil_div(n, p.cb);
  const size_t row_bytes = (size_t)((p.cb + 4) + (p.nbl * 8 + 4)) * 8;
  const size_t budget = dev_info().smem_optin - kBarBytes;
  p.kr = 32;
  while (p.kr > 8 && 3 * p.kr * row_bytes > budget) p.kr -= 8;
  p.nst = (int)std::min<size_t>(4, budget / (p.kr * row_bytes));
  const int sms = dev_info().sms;
  // split count: best wave efficiency, at least 256 rows per split
  int best = 1;
  double best_eff = -1;
  for (int s = 1; s <= 64; ++s) {
    if (s > 1 && ceil_div(m, s) < 256) break;
    const int64_t tot = (int64_t)p.colblocks * s;
    const double eff = (double)tot / (double)(ceil_div(tot, sms) * sms);
    const double score = eff * std::min(1.0, (double)tot / sms);
    if (score > best_eff + 1e-9) best_eff = score, best = s;
  }
  p.splits = best;
  p.rows_per_split = ceil_div(std::max<int64_t>(m, 1), p.splits);
  p.part_doubles = (size_t)p.splits * p.colblocks * p.cb * p.ldz;
  return p;
}

template <int MI, int NBL>
static cudaError_t tn_go(const TnPlan& p, const double* X, int64_t ldx, int64_t m, int n,
                         const double* Y, int64_t ldy, int l, double* part, cudaStream_t s) {
  const size_t smem = kBarBytes + (size_t)p.nst * p.kr * ((p.cb + 4) + (NBL * 8 + 4)) * 8;
  cudaError_t e = cudaFuncSetAttribute(gemm_tn_kernel<MI, NBL>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(p.colblocks, p.splits);
  gemm_tn_kernel<MI, NBL><<<grid, TN_WARPS * 32, smem, s>>>(
      X, ldx, m, n, Y, ldy, (l + 1) & ~1, p.rows_per_split, part, p.ldz,
      (int64_t)p.colblocks * p.cb, p.kr, p.nst);
  return cudaGetLastError();
}

cudaError_t launch_gemm_tn(const TnPlan& p, const double* X, int64_t ldx, int64_t m, int n,
                           const double* Y, int64_t ldy, int l, double* part, cudaStream_t s) {
#define TN_CASE(MI, NB) \
  if (p.mi == MI && p.nbl == NB) return tn_go<MI, NB>(p, X, ldx, m, n, Y, ldy, l, part, s);
  TN_CASE(4, 1) TN_CASE(4, 2) TN_CASE(4, 3) TN_CASE(4, 4)
  TN_CASE(2, 5) TN_CASE(2, 6) TN_CASE(2, 7) TN_CASE(2, 8)
  TN_CASE(1, 9) TN_CASE(1, 10) TN_CASE(1, 11) TN_CASE(1, 12) TN_CASE(1, 13) TN_CASE(1, 14)
  TN_CASE(1, 15) TN_CASE(1, 16)
#undef TN_CASE
  return cudaErrorInvalidValue;
}

}  // namespace tsk
