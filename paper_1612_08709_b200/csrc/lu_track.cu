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
__global__ void k_lu_reduce(const double* pval, const long long* pidx, int nparts, LuRec* rec, double* gbuf) {
  if (threadIdx.x != 0 || rec->stopped) return;
  double bv = -1.0;
  long long bi = 0x7fffffffffffffffLL;
  for (int q = 0; q < nparts; ++q)
    if (pval[q] > bv || (pval[q] == bv && pidx[q] < bi)) bv = pval[q], bi = pidx[q];
  rec->row = bi;
  gbuf[0] = bv;  // < 0: no candidate row on this rank
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
      for (int c = j + 1; c < w; ++c) y[c] = fma(-mult, urow[c], y[c]);
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

// ------------------------------------------------------------- launchers ----
static inline unsigned lu_grid(int64_t rows) {
  const int64_t b = ceil_div(std::max<int64_t>(rows, 1), LU_T);
  return (unsigned)std::min<int64_t>(b, 148 * 8);
}

size_t lu_workspace_bytes(int64_t rows, int w) {
  return 256 + ((size_t)std::max<int64_t>(rows, 1) + 255) / 256 * 256 + (size_t)lu_grid(rows) * 16 +
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
  p += (size_t)lu_grid(rows) * 8;
  lw.pidx = reinterpret_cast<long long*>(p);
  p += (size_t)lu_grid(rows) * 8;
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

}  // namespace tsk
