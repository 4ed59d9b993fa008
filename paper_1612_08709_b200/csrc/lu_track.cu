// LU-based subspace tracking: in the intermediate steps of
// Alg. 5 the tall factor is the L of Gaussian elimination with partial (row) pivoting instead of
// Alg. 3's orthonormal Q -- "the column space of L is the same as the column space of Q".
//
// Y (rows x w, ld ldy; row-sharded over the ranks for the tall factor) becomes L in place, in
// Y's own row order (the P L of Y = P L U): multipliers below/around, 1 at each pivot row's own
// column, 0 right of it; columns past the kept count r zero.  Per column j (host loop, every
// decision on the device):
//   k_lu_colmax   block partials of max |Y(i, j)| over the rows not yet chosen (ties: lowest row)
//   k_lu_reduce   the rank's max and its row (fixed order), into the pivot record
//   [multi-rank: allreduce MAX of the value, MIN of the owning rank among the maxima]
//   k_lu_decide   stop at the first numerically zero pivot (|pivot_j| <= |pivot_1| wp, reading
//                 R21) or past the device width; else the owner copies its pivot row to urow
//   [multi-rank: allreduce SUM of urow]
//   k_lu_update   multipliers Y(i, j) / pivot, Y(i, c) -= mult * urow(c) for c > j; chosen rows
//                 get 0 (1 at the pivot row itself)
// k_lu_finish zeroes the columns >= r and writes the decision slot.
//
// Single-rank / replicated factors (no collective between the steps): k_lu_fused runs the whole
// elimination as ONE cooperative kernel -- one grid barrier per column instead of six launches.
// Every CTA reduces the previous step's block partials itself (same fixed order: every CTA takes
// the same pivot), reads the pivot row into shared memory, and each thread updates its own rows
// (the same row -> thread map in every column) while it computes the next column's candidate.
// The pivot row's own 1 is written one step late (after the barrier that ends every CTA's read of
// that row).  (max, lowest row) is associative, so the pivot -- and every element of L -- is the
// same as the launch-per-step path's.
#include <cooperative_groups.h>
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace tsk {

struct LuRec {  // device pivot record (one per factorization)
  double gmax;     // |pivot| of the current column (after the cross-rank MAX)
  double p1;       // |pivot_1|
  double pv;       // signed pivot value (broadcast through urow[w])
  long long row;   // local row of the rank's candidate
  int owner;       // rank owning the pivot (after the cross-rank MIN)
  int stopped;     // sticky: elimination finished
  int r;           // columns kept
  int pad;
};

static constexpr int LU_T = 256;
static constexpr int LU_CH = 16;  // k_lu_fused: columns of a row loaded together

__global__ void __launch_bounds__(LU_T) k_lu_colmax(const double* Y, int64_t ldy, int64_t rows, int j,
                                                   const unsigned char* chosen, const LuRec* rec, double* pval,
                                                   long long* pidx) {
  __shared__ double sv[LU_T / 32];
  __shared__ long long si[LU_T / 32];
  double bv = -1.0;
  long long bi = 0x7fffffffffffffffLL;
  if (!rec->stopped) {
    for (int64_t i = (int64_t)blockIdx.x * LU_T + threadIdx.x; i < rows; i += (int64_t)gridDim.x * LU_T) {
      if (chosen[i]) continue;
      const double v = fabs(Y[i * ldy + j]);
      if (v > bv) bv = v, bi = i;  // rows visited in increasing order: ties keep the lowest
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) bv = ov, bi = oi;
  }
  if ((threadIdx.x & 31) == 0) sv[threadIdx.x >> 5] = bv, si[threadIdx.x >> 5] = bi;
  __syncthreads();
  if (threadIdx.x == 0) {
    bv = sv[0], bi = si[0];
    for (int w = 1; w < LU_T / 32; ++w)
      if (sv[w] > bv || (sv[w] == bv && si[w] < bi)) bv = sv[w], bi = si[w];
    pval[blockIdx.x] = bv;
    pidx[blockIdx.x] = bi;
  }
}

// rank-local max over the block partials (fixed order); gbuf[0] = value for the MAX allreduce,
// obuf[0] = my rank if I hold it (set after the MAX by k_lu_owner)
// (max, lowest row) over the block partials by one warp: lanes take strided partials (their
// loads in flight together -- a one-thread loop waited an L2 round trip per partial: ~0.3 ms per
// column at 800 partials), then an xor butterfly.  The pair order is total, so the result does
// not depend on how the partials are split.
__device__ __forceinline__ void lu_warp_best(const double* pval, const long long* pidx, int nparts, double& bv,
                                             long long& bi) {
  bv = -1.0;
  bi = 0x7fffffffffffffffLL;
  for (int q0 = threadIdx.x & 31; q0 < nparts; q0 += 256) {  // 8 partials per lane in flight
    double v[8];
    long long id[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int q = q0 + 32 * k;  // written by other CTAs before a grid barrier: L2, not L1
      v[k] = q < nparts ? __ldcg(pval + q) : -1.0;
      id[k] = q < nparts ? __ldcg(pidx + q) : 0x7fffffffffffffffLL;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (v[k] > bv || (v[k] == bv && id[k] < bi)) bv = v[k], bi = id[k];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) bv = ov, bi = oi;
  }
}

__global__ void k_lu_reduce(const double* pval, const long long* pidx, int nparts, LuRec* rec, double* gbuf) {
  if (threadIdx.x >= 32 || rec->stopped) return;
  double bv;
  long long bi;
  lu_warp_best(pval, pidx, nparts, bv, bi);
  if (threadIdx.x == 0) {
    rec->row = bi;
    gbuf[0] = bv;  // < 0: no candidate row on this rank
  }
}

__global__ void k_lu_owner(const double* gbuf, const LuRec* rec, int* obuf, int rank, const double* lbuf) {
  if (threadIdx.x != 0) return;
  obuf[0] = (!rec->stopped && lbuf[0] >= 0.0 && lbuf[0] == gbuf[0]) ? rank : 0x7fffffff;
}

// decision for column j; the owner copies its pivot row (w values) to urow, others write zeros;
// urow[w] = the signed pivot (summed across ranks with urow)
__global__ void k_lu_decide(const double* Y, int64_t ldy, int w, int j, const int* wdev, double wp,
                            const double* gbuf, const int* obuf, int rank, LuRec* rec, double* urow,
                            unsigned char* chosen) {
  __shared__ int s_go, s_mine;
  if (threadIdx.x == 0) {
    int go = 0, mine = 0;
    if (!rec->stopped) {
      const double g = gbuf[0];
      if (j == 0) rec->p1 = g > 0.0 ? g : 0.0;
      const int width = wdev ? min(*wdev, w) : w;
      go = j < width && rec->p1 > 0.0 && g > rec->p1 * wp;
      if (!go) {
        rec->stopped = 1;
      } else {
        rec->r = j + 1;
        rec->owner = obuf[0];
        mine = rec->owner == rank;
        if (mine) chosen[rec->row] = 2;  // 2: the current pivot (becomes 1 after the update)
      }
    }
    s_go = go;
    s_mine = mine;
  }
  __syncthreads();
  if (!s_go) return;
  for (int c = threadIdx.x; c <= w; c += blockDim.x) {
    double v = 0.0;
    if (s_mine) v = c < w ? Y[rec->row * ldy + c] : Y[rec->row * ldy + j];
    urow[c] = v;
  }
}

__global__ void __launch_bounds__(LU_T) k_lu_update(double* Y, int64_t ldy, int64_t rows, int w, int j,
                                                   unsigned char* chosen, const LuRec* rec, const double* urow) {
  if (rec->stopped && rec->r <= j) return;
  const double inv = 1.0 / urow[w];
  for (int64_t i = (int64_t)blockIdx.x * LU_T + threadIdx.x; i < rows; i += (int64_t)gridDim.x * LU_T) {
    double* y = Y + i * ldy;
    const unsigned char ch = chosen[i];
    if (ch == 1) {  // an earlier pivot row: L is 0 right of its own column
      y[j] = 0.0;
    } else if (ch == 2) {  // the pivot row: 1 on its column (its remaining entries are U's row)
      y[j] = 1.0;
      chosen[i] = 1;
    } else {
      const double mult = y[j] * inv;
      y[j] = mult;
      for (int c0 = j + 1; c0 < w; c0 += LU_CH) {  // chunks of independent loads (as k_lu_fused)
        double u[LU_CH];
#pragma unroll
        for (int k = 0; k < LU_CH; ++k) u[k] = c0 + k < w ? y[c0 + k] : 0.0;
#pragma unroll
        for (int k = 0; k < LU_CH; ++k)
          if (c0 + k < w) y[c0 + k] = fma(-mult, urow[c0 + k], u[k]);
      }
    }
  }
}

// columns >= r zero; pivot rows already hold 0 right of their column for the columns < r; slot
__global__ void k_lu_finish(double* Y, int64_t ldy, int64_t rows, int w, const LuRec* rec, int* slot) {
  const int r = rec->r;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < rows * (int64_t)(w - r);
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / (w - r);
    const int c = r + (int)(e % (w - r));
    Y[i * ldy + c] = 0.0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    slot[0] = r;
    slot[1] = r;
    slot[2] = 0;
    slot[3] = r;
    slot[4] = -r;
    slot[5] = r;
    slot[6] = -r;
    slot[7] = 0;
  }
}

__global__ void k_lu_init(unsigned char* chosen, int64_t rows, LuRec* rec) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x)
    chosen[i] = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    rec->gmax = rec->p1 = rec->pv = 0.0;
    rec->row = 0;
    rec->owner = 0;
    rec->stopped = 0;
    rec->r = 0;
  }
}

// one-pass block reduction of (max |.|, lowest row) into (pv, pi) of block b
__device__ __forceinline__ void lu_block_best(double bv, long long bi, double* sv, long long* si, double* pval,
                                              long long* pidx, int b) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) bv = ov, bi = oi;
  }
  if ((threadIdx.x & 31) == 0) sv[threadIdx.x >> 5] = bv, si[threadIdx.x >> 5] = bi;
  __syncthreads();
  if (threadIdx.x == 0) {
    bv = sv[0], bi = si[0];
    for (int w = 1; w < LU_T / 32; ++w)
      if (sv[w] > bv || (sv[w] == bv && si[w] < bi)) bv = sv[w], bi = si[w];
    pval[b] = bv;
    pidx[b] = bi;
  }
}

// pval / pidx: 2 x gridDim.x entries (double-buffered by column parity)
__global__ void __launch_bounds__(LU_T) k_lu_fused(double* Y, int64_t ldy, int64_t rows, int w, const int* wdev,
                                                  double wp, unsigned char* chosen, double* pval, long long* pidx,
                                                  LuRec* rec, int* slot) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ double sv[LU_T / 32];
  __shared__ long long si[LU_T / 32];
  __shared__ double s_urow[129];
  __shared__ long long s_row;
  __shared__ double s_g;
  const int G = gridDim.x;
  const int64_t stride = (int64_t)G * LU_T;
  const int64_t i0 = (int64_t)blockIdx.x * LU_T + threadIdx.x;
  // column 0 candidates (nothing chosen yet)
  double bv = -1.0;
  long long bi = 0x7fffffffffffffffLL;
  for (int64_t i = i0; i < rows; i += stride) {
    chosen[i] = 0;
    const double v = fabs(Y[i * ldy]);
    if (v > bv) bv = v, bi = i;
  }
  lu_block_best(bv, bi, sv, si, pval, pidx, blockIdx.x);
  const int width = wdev ? min(*wdev, w) : w;
  double p1 = 0.0;
  int r = 0;
  long long prev = -1;  // the previous column's pivot row (its 1 is written one step late)
  grid.sync();
  for (int j = 0; j < w; ++j) {
    const double* pv_ = pval + (j & 1) * G;
    const long long* pi_ = pidx + (j & 1) * G;
    if (threadIdx.x < 32) {  // warp 0 reduces the block partials (the same result in every CTA)
      double g;
      long long row;
      lu_warp_best(pv_, pi_, G, g, row);
      if (threadIdx.x == 0) s_g = g, s_row = row;
    }
    __syncthreads();
    const double g = s_g;
    const long long row = s_row;
    if (j == 0) p1 = g > 0.0 ? g : 0.0;
    if (!(j < width && p1 > 0.0 && g > p1 * wp)) break;  // every CTA takes the same decision
    r = j + 1;
    for (int c = threadIdx.x; c <= w; c += LU_T) s_urow[c] = __ldcg(Y + row * ldy + (c < w ? c : j));
    __syncthreads();
    const double inv = 1.0 / s_urow[w];
    bv = -1.0;
    bi = 0x7fffffffffffffffLL;
    const bool next = j + 1 < w;
    for (int64_t i = i0; i < rows; i += stride) {
      double* y = Y + i * ldy;
      // every load of the row's first chunk is issued before any decision (independent loads: one
      // L2 round trip per chunk -- ncu showed the element-by-element load -> FMA -> store chain
      // stalled on long_scoreboard at every DFMA)
      const unsigned char ch = chosen[i];
      const double yj = y[j];
      double v[LU_CH];
#pragma unroll
      for (int k = 0; k < LU_CH; ++k) v[k] = j + 1 + k < w ? y[j + 1 + k] : 0.0;
      if (i == prev) y[j - 1] = 1.0;  // the previous pivot row's own 1 (every read of it is done)
      if (i == row) {                  // the pivot row: its remaining entries are U's row
        chosen[i] = 1;
        continue;
      }
      if (ch) {  // an earlier pivot row: L is 0 right of its own column
        y[j] = 0.0;
        continue;
      }
      const double mult = yj * inv;
      y[j] = mult;
#pragma unroll
      for (int k = 0; k < LU_CH; ++k)
        if (j + 1 + k < w) y[j + 1 + k] = v[k] = fma(-mult, s_urow[j + 1 + k], v[k]);
      for (int c0 = j + 1 + LU_CH; c0 < w; c0 += LU_CH) {
        double u[LU_CH];
#pragma unroll
        for (int k = 0; k < LU_CH; ++k) u[k] = c0 + k < w ? y[c0 + k] : 0.0;
#pragma unroll
        for (int k = 0; k < LU_CH; ++k)
          if (c0 + k < w) y[c0 + k] = fma(-mult, s_urow[c0 + k], u[k]);
      }
      if (next) {
        const double a = fabs(v[0]);
        if (a > bv) bv = a, bi = i;
      }
    }
    prev = row;
    if (next) lu_block_best(bv, bi, sv, si, pval + ((j + 1) & 1) * G, pidx + ((j + 1) & 1) * G, blockIdx.x);
    grid.sync();
  }
  // the last pivot's 1; columns >= r zero; the decision slot
  for (int64_t i = i0; i < rows; i += stride) {
    double* y = Y + i * ldy;
    if (i == prev) y[r - 1] = 1.0;
    for (int c = r; c < w; ++c) y[c] = 0.0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    rec->r = r;
    rec->stopped = 1;
    slot[0] = r;
    slot[1] = r;
    slot[2] = 0;
    slot[3] = r;
    slot[4] = -r;
    slot[5] = r;
    slot[6] = -r;
    slot[7] = 0;
  }
}

// ------------------------------------------------------------- launchers ----
static inline unsigned lu_grid(int64_t rows) {
  const int64_t b = ceil_div(std::max<int64_t>(rows, 1), LU_T);
  return (unsigned)std::min<int64_t>(b, 148 * 8);
}

// the partial buffers hold 2 x lu_grid entries: k_lu_fused double-buffers them
size_t lu_workspace_bytes(int64_t rows, int w) {
  return 256 + ((size_t)std::max<int64_t>(rows, 1) + 255) / 256 * 256 + (size_t)lu_grid(rows) * 32 +
         (size_t)(w + 1) * 8 + 64 + 64;
}

LuWork lu_carve(void* ws, int64_t rows, int w) {
  char* p = static_cast<char*>(ws);
  LuWork lw;
  lw.rec = p;
  p += 256;
  lw.chosen = reinterpret_cast<unsigned char*>(p);
  p += ((size_t)std::max<int64_t>(rows, 1) + 255) / 256 * 256;
  lw.pval = reinterpret_cast<double*>(p);
  p += (size_t)lu_grid(rows) * 16;
  lw.pidx = reinterpret_cast<long long*>(p);
  p += (size_t)lu_grid(rows) * 16;
  lw.urow = reinterpret_cast<double*>(p);
  p += (size_t)(w + 1) * 8;
  lw.gbuf = reinterpret_cast<double*>(p);
  p += 32;
  lw.lbuf = reinterpret_cast<double*>(p);
  p += 16;
  lw.obuf = reinterpret_cast<int*>(p);
  return lw;
}

cudaError_t lu_init(const LuWork& lw, int64_t rows, cudaStream_t s) {
  k_lu_init<<<lu_grid(rows), LU_T, 0, s>>>(lw.chosen, rows, static_cast<LuRec*>(lw.rec));
  return cudaGetLastError();
}
cudaError_t lu_colmax(const LuWork& lw, const double* Y, int64_t ldy, int64_t rows, int j, cudaStream_t s) {
  const unsigned g = lu_grid(rows);
  LuRec* rec = static_cast<LuRec*>(lw.rec);
  k_lu_colmax<<<g, LU_T, 0, s>>>(Y, ldy, rows, j, lw.chosen, rec, lw.pval, lw.pidx);
  k_lu_reduce<<<1, 32, 0, s>>>(lw.pval, lw.pidx, (int)g, rec, lw.lbuf);
  return cudaMemcpyAsync(lw.gbuf, lw.lbuf, 8, cudaMemcpyDeviceToDevice, s);
}
cudaError_t lu_owner(const LuWork& lw, int rank, cudaStream_t s) {
  k_lu_owner<<<1, 32, 0, s>>>(lw.gbuf, static_cast<LuRec*>(lw.rec), lw.obuf, rank, lw.lbuf);
  return cudaGetLastError();
}
cudaError_t lu_decide(const LuWork& lw, const double* Y, int64_t ldy, int w, int j, const int* wdev, double wp,
                      int rank, cudaStream_t s) {
  k_lu_decide<<<1, 128, 0, s>>>(Y, ldy, w, j, wdev, wp, lw.gbuf, lw.obuf, rank, static_cast<LuRec*>(lw.rec),
                                lw.urow, lw.chosen);
  return cudaGetLastError();
}
cudaError_t lu_update(const LuWork& lw, double* Y, int64_t ldy, int64_t rows, int w, int j, cudaStream_t s) {
  k_lu_update<<<lu_grid(rows), LU_T, 0, s>>>(Y, ldy, rows, w, j, lw.chosen, static_cast<LuRec*>(lw.rec), lw.urow);
  return cudaGetLastError();
}
cudaError_t lu_finish(const LuWork& lw, double* Y, int64_t ldy, int64_t rows, int w, int* slot, cudaStream_t s) {
  k_lu_finish<<<lu_grid(rows * w), LU_T, 0, s>>>(Y, ldy, rows, w, static_cast<LuRec*>(lw.rec), slot);
  return cudaGetLastError();
}

// The whole elimination in one cooperative launch (single rank or a replicated factor; w <= 128).
// Grid: as many CTAs as are co-resident (occupancy x SMs), at most lu_grid(rows).
cudaError_t lu_fused(const LuWork& lw, double* Y, int64_t ldy, int64_t rows, int w, const int* wdev, double wp,
                     int* slot, cudaStream_t s) {
  if (w < 1 || w > 128) return cudaErrorInvalidValue;
  static int per_sm = -1, sms = 0;
  if (per_sm < 0) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_lu_fused, LU_T, 0);
    if (e != cudaSuccess) return e;
  }
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>(lu_grid(rows), (int64_t)per_sm * sms));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)g);
  cfg.blockDim = dim3(LU_T);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_lu_fused, Y, ldy, rows, w, wdev, wp, lw.chosen, lw.pval, lw.pidx,
                            static_cast<LuRec*>(lw.rec), slot);
}

}  // namespace tsk
