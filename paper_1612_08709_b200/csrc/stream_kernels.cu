// Streaming FP64 passes over the row-sharded tall matrix (sm_100a).
//
//   syrk   : B_p = X_p^T X_p            Alg. 3/4 step 1, Alg. 4 step 7
//   gemm_nn: Y = X M (+ column norms)   Alg. 3/4 steps 3-4, steps 9-10
//                                       (P:674-678), step 15; Alg. 5 steps 3, 8
//   gemm_tn: Z_p = X_p^T Y_p            Alg. 5 step 5, Alg. 6 step 1
//
// All three are warp-specialised pipelines: one producer warp streams 2-D
// boxes of the operands from HBM/L2 into a ring of shared-memory stages with
// the tensor TMA engine (cp.async.bulk.tensor.2d -> SASS UTMALDG; out-of-range
// rows/columns arrive as zeros, so ragged tails need no special code), with a
// "full" mbarrier per stage (transaction bytes) and an "empty" mbarrier per
// stage (one arrival per consumer warp).  The consumer warps run the
// contraction on the FP64 tensor pipe (mma.sync m8n8k4 f64 -> DMMA.8x8x4; on
// B200 the only FP64 MMA shape -- tcgen05 has no f64 kind).
//
// Shared-memory rows of every box are `ld = 4 (mod 8)` doubles wide, so the
// DMMA fragment loads (lanes g = lane>>2, t = lane&3 read 4 rows x 8 doubles)
// are bank-conflict free: boxes are loaded exactly that wide (the TMA box is
// the padded width; the tensor map's true width zero-fills the pad columns).
//
// Reductions over rows are split across CTAs into per-CTA partials that are
// summed in a fixed order by a separate kernel, so every result is bitwise
// deterministic run to run.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
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

// ---- tensor maps ------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// L2 promotion (the granule in which an L2 miss of the TMA engine is filled from
// DRAM): 256 B when a box row is a whole contiguous matrix row; when it is only a slice
// of a longer row (the first nc columns of Y~ inside U's ld = n rows) a 256-B fill
// drags in neighbour bytes no one reads (ncu r1: 1.38x DRAM traffic for the Gram of
// Y~), so those use 64 B.  TSSVD_L2PROMO = 0/64/128/256 forces one (experiments).
static CUtensorMapL2promotion l2_promotion(int64_t cols, int64_t ld, int box_cols) {
  static const int force = getenv("TSSVD_L2PROMO") ? atoi(getenv("TSSVD_L2PROMO")) : -1;
  const int v = force >= 0 ? force : (cols == ld || box_cols < cols ? 256 : 64);
  switch (v) {
    case 0: return CU_TENSOR_MAP_L2_PROMOTION_NONE;
    case 64: return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
    case 128: return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    default: return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }
}

// Row-major FP64 matrix (rows x cols, leading dimension ld doubles) as a 2-D
// tensor map with boxes of box_rows x box_cols (box_cols may exceed cols:
// the excess is zero-filled).
static cudaError_t make_tmap(CUtensorMap* map, const double* base, int64_t rows, int64_t cols,
                             int64_t ld, int box_rows, int box_cols) {
  auto fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  if (rows < 1 || cols < 1 || box_cols > 256 || box_rows > 256 || (ld & 1) ||
      (reinterpret_cast<uintptr_t>(base) & 15))
    return cudaErrorInvalidValue;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  const cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  const cuuint32_t es[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box,
                  es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  l2_promotion(cols, ld, box_cols), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

static constexpr int kBarBytes = 256;  // up to 16 stages x (full, empty) mbarriers

struct Ring {  // the pipeline's mbarriers: full[s] at bar[s], empty[s] at bar[16 + s]
  uint64_t* bar;
  __device__ uint64_t* full(int s) const { return bar + s; }
  __device__ uint64_t* empty(int s) const { return bar + 16 + s; }
};

__device__ __forceinline__ void ring_init(Ring r, int nst, int consumers) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(r.full(s), 1);
      mbar_init(r.empty(s), consumers);
    }
    fence_mbar_init();
  }
  __syncthreads();
}

// 8-byte shared-memory load by shared-window address (volatile asm: ordered against the mbarrier
// wait before it and the arrive after it)
__device__ __forceinline__ double lds_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}

// ============================================================== SYRK (Gram) ==
// CTA b owns rows [b*rpc, (b+1)*rpc) (rpc a multiple of KR, so only the last
// CTA's last box can cross m -- and there TMA zero-fills).  The T = nb(nb+1)/2
// lower-triangle 8x8 DMMA tiles of B, in row-major order (0,0), (1,0), (1,1),
// (2,0), ..., are dealt to the consumer warps in contiguous, equal runs of at
// most SYRK_TPW tiles (grid.y splits the list when one CTA cannot hold it), so
// every warp issues the same number of DMMAs per stage and consecutive tiles
// of a run share their row fragment.  Both operands are columns of the same
// row block: the fragment of column block c at k-step kk is Xs[kk*4+t][c*8+g]
// in the A (= X^T) and the B role alike.
// rows per pipeline stage.  64 rows measured 1.4-2.5% faster at w = 92..200 (c2 Gram 0.773 ->
// 0.762 ms, c4 10.84 -> 10.65 ms; profiles/r02s2_gram_kr64_ab.txt) but two 64-row stages of a
// 256-column box exceed the 227 KB of shared memory (w = 256 failed to launch), so the default
// stays 32; A/B builds: build.py -D TSSVD_SYRK_KR=64
#ifdef TSSVD_SYRK_KR
static constexpr int SYRK_KR = TSSVD_SYRK_KR;
#else
static constexpr int SYRK_KR = 32;
#endif
static constexpr int SYRK_TPW = 11;
// CTAs per SM: runs of <= 6 tiles fit 64 registers (two CTAs per SM), longer
// runs need up to 128 (one CTA per SM)
static constexpr int syrk_minb(int tpw) { return tpw <= 6 ? 2 : 1; }

template <int TPW, int MINB>
__global__ void __launch_bounds__(512, MINB) syrk_kernel(const __grid_constant__ CUtensorMap tx, int64_t m,
                                                      int w, int W, int64_t rpc, double* __restrict__ part,
                                                      int nst, int tps, int tpw) {
  extern __shared__ __align__(128) unsigned char smem[];
  const Ring ring{reinterpret_cast<uint64_t*>(smem)};
  double* buf = reinterpret_cast<double*>(smem + kBarBytes);
  const int stage_d = SYRK_KR * W;
  const int nb = (w + 7) >> 3, ntiles = nb * (nb + 1) / 2;
  const int wp = nb * 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int ncw = (blockDim.x >> 5) - 1;  // consumer warps (warp 0 produces)
  // grid = (tile-list splits, row blocks): the splits of one row block are
  // launched together, so the second reads its rows from L2 instead of HBM
  const int rb = blockIdx.y, sp = blockIdx.x;
  const int64_t r0 = (int64_t)rb * rpc;
  const int64_t r1 = min(m, r0 + rpc);
  const int nsteps = r1 > r0 ? (int)ceil_div(r1 - r0, SYRK_KR) : 0;
  ring_init(ring, nst, ncw);

  if (warp == 0) {  // ---- producer
    if (lane == 0) {
      int b = 0;
      uint32_t ph = 0;
      for (int s = 0; s < nsteps; ++s) {
        if (s >= nst) mbar_wait(ring.empty(b), ph ^ 1u);
        mbar_arrive_expect_tx(ring.full(b), (uint32_t)(stage_d * 8));
        tma_load_2d(buf + b * stage_d, &tx, 0, (int)(r0 + (int64_t)s * SYRK_KR), ring.full(b));
        if (++b == nst) b = 0, ph ^= 1u;
      }
    }
    return;
  }
  // this warp's run of tiles [q0, q1) of the row-major lower triangle
  const int q0 = min(ntiles, sp * tps + (warp - 1) * tpw);
  const int q1 = min(ntiles, min(sp * tps + tps, q0 + tpw));
  const int nt = q1 - q0;
  int I0 = 0;
  while ((I0 + 1) * (I0 + 2) / 2 <= q0) ++I0;
  const int J0 = q0 - I0 * (I0 + 1) / 2;
  // Per tile: the shared-memory offsets of its row and column fragments within a
  // k-row, packed (row << 16 | col), and a bit when it starts a new block row.
  // Tiles past the run repeat the last one (computed, never stored), so the
  // DMMA sequence of a k-step is branch-free: all column fragments are loaded
  // first, then each DMMA issues behind at most a predicated row-fragment load.
  uint32_t off[TPW];
  uint32_t newrow = 0;
  {
    int I = I0, J = J0;
#pragma unroll
    for (int k = 0; k < TPW; ++k) {
      off[k] = k < nt || k == 0 ? (uint32_t)(I * 8) << 16 | (uint32_t)(J * 8) : off[k > 0 ? k - 1 : 0];
      if (k > 0 && k < nt && J == 0) newrow |= 1u << k;
      if (++J > I) ++I, J = 0;
    }
  }
  double acc[TPW][2];
#pragma unroll
  for (int k = 0; k < TPW; ++k) acc[k][0] = acc[k][1] = 0.0;

  // Shared-window byte addresses of every tile's column fragment (and of the row fragments where a
  // block row starts) within stage 0, k-row 0: loop invariants in registers.  A load adds only the
  // warp-uniform (stage, k-step) offset -- the element-index arithmetic per load (unpack, scale,
  // add the window base) was ~4 integer instructions in front of every LDS, each DMMA right
  // behind its own load.
  const uint32_t lane0 = smem_u32(buf) + (uint32_t)(t * W + g) * 8u;
  uint32_t ac[TPW], ar[TPW];
#pragma unroll
  for (int k = 0; k < TPW; ++k) ac[k] = lane0 + (off[k] & 0xffffu) * 8u, ar[k] = lane0 + (off[k] >> 16) * 8u;
  const uint32_t kstep_b = (uint32_t)(4 * W) * 8u, stage_b = (uint32_t)stage_d * 8u;

  int b = 0;
  uint32_t ph = 0;
  for (int s = 0; s < nsteps; ++s) {
    mbar_wait(ring.full(b), ph);
    if (nt > 0) {
      uint32_t u = (uint32_t)b * stage_b;
#pragma unroll
      for (int kk = 0; kk < SYRK_KR / 4; ++kk, u += kstep_b) {
        double cf[TPW];
#pragma unroll
        for (int k = 0; k < TPW; ++k) cf[k] = lds_f64(ac[k] + u);
        double fi = lds_f64(ar[0] + u);
#pragma unroll
        for (int k = 0; k < TPW; ++k) {
          if ((newrow >> k) & 1u) fi = lds_f64(ar[k] + u);  // a new block row starts
          dmma(acc[k], fi, cf[k]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(ring.empty(b));
    if (++b == nst) b = 0, ph ^= 1u;
  }

  double* P = part + (size_t)rb * wp * wp;
  TCHECK(rb < (int)gridDim.y && I0 * 8 < wp);
#pragma unroll
  for (int k = 0; k < TPW; ++k)
    if (k < nt)
      TCHECK((int)(off[k] >> 16) + g < wp && (int)(off[k] & 0xffffu) + 2 * t + 1 < wp),
      *reinterpret_cast<double2*>(P + (size_t)((off[k] >> 16) + g) * wp + (off[k] & 0xffffu) + 2 * t) =
          make_double2(acc[k][0], acc[k][1]);
}

// Tiles per warp, consumer warps and tile-list splits over grid.y: equal runs
// of 3..SYRK_TPW tiles, <= 15 consumer warps.  The DMMA pipe belongs to an SM
// sub-partition (warp w runs on SMSP w % 4), and every stage waits for the
// slowest warp, so a CTA's time per stage is ceil(ncw / 4) * tpw DMMA slots on
// its busiest SMSP: the planner maximises
//   (useful tiles / DMMA slots) x min(1, consumer warps per SMSP / 3) x 0.93^(splits-1),
// the second factor for latency hiding (runs of <= 6 tiles fit two CTAs per
// SM), the third for re-streaming the rows once per split.  Measured at
// m = 2e6 (B200, tools/gram_bench.py): it picks the fastest of the measured
// shapes at w = 55, 64, 82, 92, 100 (0.32, 0.35, 0.64, 0.70, 0.81 ms; w = 100
// was 13 x 7 = 0.91 ms).
struct SyrkPlan {
  int splits, tps, tpw, ncw;
};
static SyrkPlan syrk_plan(int w) {
  const int nb = (w + 7) / 8, ntiles = nb * (nb + 1) / 2;
  const int smem_per_sm = (int)std::max<size_t>(
      1, 228 * 1024 / (kBarBytes + (size_t)4 * SYRK_KR * std::min(smem_ld(w), 256) * 8 + 1024));
  SyrkPlan p{};
  double best = -1.0;
  static const int force_splits = getenv("TSSVD_SYRK_SPLITS") ? atoi(getenv("TSSVD_SYRK_SPLITS")) : 0;
  const int s0 = std::max((int)ceil_div(ntiles, 15 * SYRK_TPW), force_splits);
  for (int splits = s0; splits <= (force_splits ? s0 : s0 + 1); ++splits) {
    const int tps = (int)ceil_div(ntiles, splits);
    for (int tpw = SYRK_TPW; tpw >= 3; --tpw) {  // runs of 1-2 tiles: too many loads per DMMA
      const int ncw = (int)ceil_div(tps, tpw);
      if (ncw > 15) break;
      const int per_sm = std::min(syrk_minb(tpw), smem_per_sm);
      const double slots = (double)splits * 4 * ceil_div(ncw, 4) * tpw;
      const double score = ntiles / slots * std::min(1.0, ncw * per_sm / 4.0 / 3.0) *
                           std::pow(0.93, splits - 1);  // every split re-streams the rows
      if (score > best + 1e-9) best = score, p.splits = splits, p.tps = tps, p.ncw = ncw, p.tpw = tpw;
    }
  }
  static const int force_tpw = getenv("TSSVD_SYRK_TPW") ? atoi(getenv("TSSVD_SYRK_TPW")) : 0;  // experiments
  if (force_tpw >= 1 && force_tpw <= SYRK_TPW && ceil_div(p.tps, force_tpw) <= 15)
    p.tpw = force_tpw, p.ncw = (int)ceil_div(p.tps, force_tpw);
  return p;
}

static size_t syrk_stage_bytes(int w) { return (size_t)SYRK_KR * std::min(smem_ld(w), 256) * 8; }

// CTAs per SM: by shared memory (>= 4 stages each) and threads, at most 4
int syrk_partials_grid(int64_t m, int w) {
  const SyrkPlan p = syrk_plan(w);
  const size_t smem = kBarBytes + (size_t)4 * syrk_stage_bytes(w);
  int per_sm = (int)std::max<size_t>(1, std::min<size_t>(228 * 1024 / (smem + 1024), 2048 / (32 * (p.ncw + 1))));
  per_sm = std::min(per_sm, syrk_minb(p.tpw));
  int64_t g = (int64_t)dev_info().sms * per_sm;
  int64_t maxg = std::max<int64_t>(1, ceil_div(m, SYRK_KR));
  return (int)std::max<int64_t>(1, std::min(g, maxg));
}

size_t syrk_partials_doubles(int64_t m, int w) {
  const int wp = pad8(w);
  return (size_t)syrk_partials_grid(m, w) * wp * wp;
}

cudaError_t launch_syrk(const double* X, int64_t ldx, int64_t m, int w, double* part,
                        cudaStream_t s) {
  const SyrkPlan p = syrk_plan(w);
  const int gx = syrk_partials_grid(m, w);
  const int W = std::min(smem_ld(w), 256);  // TMA box limit (w > 248: conflicted but correct)
  const int per_sm = std::max(1, (int)ceil_div(gx, dev_info().sms));
  const size_t budget = (dev_info().smem_optin + 1024) / per_sm - 1024 - kBarBytes;
  const int nst = (int)std::max<size_t>(2, std::min<size_t>(8, budget / syrk_stage_bytes(w)));
  const size_t smem = kBarBytes + (size_t)nst * syrk_stage_bytes(w);
  int64_t rpc = ceil_div(std::max<int64_t>(m, 1), gx);
  rpc = ceil_div(rpc, SYRK_KR) * SYRK_KR;
  if (m <= 0) {  // all partials are zero
    return cudaMemsetAsync(part, 0, (size_t)gx * pad8(w) * pad8(w) * 8, s);
  }
  CUtensorMap tx;
  cudaError_t e = make_tmap(&tx, X, m, w, ldx, SYRK_KR, W);
  if (e != cudaSuccess) return e;
  void (*kern)(CUtensorMap, int64_t, int, int, int64_t, double*, int, int, int) = nullptr;
  switch (p.tpw) {
    case 1: kern = syrk_kernel<1, syrk_minb(1)>; break;
    case 2: kern = syrk_kernel<2, syrk_minb(2)>; break;
    case 3: kern = syrk_kernel<3, syrk_minb(3)>; break;
    case 4: kern = syrk_kernel<4, syrk_minb(4)>; break;
    case 5: kern = syrk_kernel<5, syrk_minb(5)>; break;
    case 6: kern = syrk_kernel<6, syrk_minb(6)>; break;
    case 7: kern = syrk_kernel<7, syrk_minb(7)>; break;
    case 8: kern = syrk_kernel<8, syrk_minb(8)>; break;
    case 9: kern = syrk_kernel<9, syrk_minb(9)>; break;
    case 10: kern = syrk_kernel<10, syrk_minb(10)>; break;
    default: kern = syrk_kernel<SYRK_TPW, syrk_minb(SYRK_TPW)>; break;
  }
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<dim3(p.splits, gx), (p.ncw + 1) * 32, smem, s>>>(tx, m, w, W, rpc, part, nst, p.tps, p.tpw);
  return cudaGetLastError();
}

// Fixed-order sum over partials by one warp per output element: lane l sums
// partials l, l+32, ... sequentially, then an xor butterfly (identical result
// in every lane).  Deterministic; error ~ (np/32 + 5) eps.
__device__ __forceinline__ double warp_sum_parts(const double* p, int np, size_t stride, int lane) {
  double s = 0.0;
  for (int q = lane; q < np; q += 32) s += p[(size_t)q * stride];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

__global__ void reduce_sym_kernel(const double* __restrict__ part, int np, int w, int wp,
                                  double* __restrict__ B, int ldb, double* __restrict__ packed) {
  const int e = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (e >= w * (w + 1) / 2) return;
  int i = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);  // lower-triangle index e -> (i, j), j <= i
  while (i * (i + 1) / 2 > e) --i;
  while ((i + 1) * (i + 2) / 2 <= e) ++i;
  const int j = e - i * (i + 1) / 2;
  const double v = warp_sum_parts(part + (size_t)i * wp + j, np, (size_t)wp * wp, lane);
  if (lane == 0) {
    B[(size_t)i * ldb + j] = v;
    B[(size_t)j * ldb + i] = v;
    if (packed) packed[e] = v;
  }
}

cudaError_t launch_reduce_sym(const double* part, int np, int w, double* B, int ldb, double* packed,
                              cudaStream_t s) {
  const int64_t threads = (int64_t)w * (w + 1) / 2 * 32;
  if (threads == 0) return cudaSuccess;
  reduce_sym_kernel<<<(int)ceil_div(threads, 256), 256, 0, s>>>(part, np, w, pad8(w), B, ldb, packed);
  return cudaGetLastError();
}

__global__ void reduce_parts_kernel(const double* __restrict__ part, int np, int64_t stride,
                                    int64_t len, double* __restrict__ out) {
  const int64_t e = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (e >= len) return;
  const double v = warp_sum_parts(part + e, np, (size_t)stride, lane);
  if (lane == 0) out[e] = v;
}

// Long outputs (the n x l partials of A^T Q): one thread per element, partials
// summed in a fixed two-level order (groups of ~sqrt(np)), coalesced over e.
__global__ void reduce_parts_long_kernel(const double* __restrict__ part, int np, int64_t stride,
                                         int64_t len, double* __restrict__ out) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= len) return;
  int gs = 1;
  while (gs * gs < np) ++gs;
  double tot = 0.0;
  for (int p0 = 0; p0 < np; p0 += gs) {
    double s = 0.0;
    const int p1 = min(np, p0 + gs);
    for (int q = p0; q < p1; ++q) s += part[(size_t)q * stride + e];
    tot += s;
  }
  out[e] = tot;
}

cudaError_t launch_reduce_parts(const double* part, int np, int64_t stride, int64_t len,
                                double* out, cudaStream_t s) {
  if (len <= 0) return cudaSuccess;
  if (len >= 32768)
    reduce_parts_long_kernel<<<(int)ceil_div(len, 256), 256, 0, s>>>(part, np, stride, len, out);
  else
    reduce_parts_kernel<<<(int)ceil_div(len * 32, 256), 256, 0, s>>>(part, np, stride, len, out);
  return cudaGetLastError();
}

// 2-D variant for the n x l partials of A^T Q (ld ldi inside each partial): out[row*ldo + col]
// for col < cols (zeros up to ldo when zero_pad); the partials' pad columns never leave the kernel (the
// allreduce then moves n x ldo doubles, ldo = l rounded up to even, not n x pad8(l)).
__global__ void reduce_parts_2d_kernel(const double* __restrict__ part, int np, int64_t stride,
                                       int64_t rows, int ldi, int cols, double* __restrict__ out,
                                       int ldo, int zero_pad, int accumulate) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= rows * ldo) return;
  const int64_t row = e / ldo;
  const int col = (int)(e % ldo);
  if (col >= cols) {
    if (zero_pad) out[e] = 0.0;
    return;
  }
  const double* p = part + row * ldi + col;
  int gs = 1;
  while (gs * gs < np) ++gs;
  double tot = 0.0;
  for (int p0 = 0; p0 < np; p0 += gs) {
    double sum = 0.0;
    const int p1 = min(np, p0 + gs);
    for (int q = p0; q < p1; ++q) sum += p[(size_t)q * stride];
    tot += sum;
  }
  out[e] = accumulate ? out[e] + tot : tot;
}

cudaError_t launch_reduce_parts_2d(const double* part, int np, int64_t stride, int64_t rows, int ldi,
                                   int cols, double* out, int ldo, bool zero_pad, cudaStream_t s,
                                   bool accumulate) {
  if (rows <= 0) return cudaSuccess;
  reduce_parts_2d_kernel<<<(int)ceil_div(rows * ldo, 256), 256, 0, s>>>(part, np, stride, rows, ldi,
                                                                         cols, out, ldo, zero_pad, accumulate);
  return cudaGetLastError();
}

// ================================================================= GEMM NN ==
// Y[r, :c] = X[r, :k] M.  A CTA owns row tiles of R rows and ALL c columns (so
// the product may overwrite X in place: every row of a tile is read into
// shared memory before any of them is written).  The 8 consumer warps form a
// (8/WC) x WC grid: warp w computes row blocks (w % RW)*MI .. +MI-1 (RW = 8/WC)
// against column blocks (w / RW)*NIW .. +NIW-1 (NIW*WC >= ceil(c/8)).  K is
// streamed in chunks of KC (= 4 mod 8) columns: a stage holds the box
// X[tile rows, k0:k0+KC] and the box M[k0:k0+KC, :] (M row-major,
// ld = smem_ld(c)); columns >= k of X and rows >= k of M arrive as zeros.
// XR > 0 (c = 8 NIW + XR, WC = 1): the last XR columns go to the FP64 FMA pipe
// instead of a DMMA tile that would be (8 - XR)/8 zeros: lane (g, t) already
// holds X[row g][4 kk + t] as its DMMA A fragment, multiplies it by the
// broadcast M[4 kk + t][8 NIW + x] and the four t-partials are summed by an xor
// butterfly at the end of the tile (c = 25 = 3*8 + 1: 25 instead of 32 columns
// of FP64 work).
// Consumer warps: 12 (3 per SMSP) when a warp's accumulators are small
// (MI * NIW <= 12 tiles, one column group: register room for 13 warps), else 8.
__host__ __device__ constexpr int nn_cw(int mi, int niw, int wc) { return mi * niw <= 12 && wc == 1 ? 12 : 8; }

// Stream-K mode (sk_rec != nullptr; only without the norm epilogue): the ntiles x kc_count
// (tile, K-chunk) units are cut into gridDim.x contiguous, equal ranges (tile-major), so
// every CTA streams the same number of chunks whatever ntiles mod gridDim.x is (c3 alpha:
// 521 row tiles on 148 SMs left a 12% tail).  A tile whose chunks are split between CTAs
// leaves partial accumulators in per-CTA records (slot 2b: the CTA's first tile, 2b + 1:
// its last), which gemm_nn_fixup sums in CTA (= K) order and stores.
__host__ __device__ inline int64_t sk_u0(int b, int64_t units, int grid) { return units * b / grid; }

// KCT > 0: the K chunk as a compile-time constant (stream-K launches with the planner's usual
// chunks): every k-step of a stage is unrolled with immediate shared-memory offsets (the
// zero-filled k-steps of the last chunk are computed: 0 x 0 adds nothing).
template <int MI, int NIW, int WC, int XR, bool SK, int KCT = 0, int NN_CW = nn_cw(MI, NIW, WC)>
__global__ void __launch_bounds__(32 * (NN_CW + 1)) gemm_nn_kernel(
    const __grid_constant__ CUtensorMap tx, const __grid_constant__ CUtensorMap tm, int64_t m, int k,
    int KC_rt, int kc_count, int LDM, int c, double* Y, int64_t ldy, double* __restrict__ norm_part,
    int nst, double* __restrict__ sk_rec) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int KC = KCT > 0 ? KCT : KC_rt;
  constexpr int RW = NN_CW / WC;
  constexpr int R = 8 * MI * RW;
  static_assert(XR == 0 || WC == 1, "remainder columns need a single column group");
  constexpr int NB = NIW + (XR > 0);  // column blocks per warp in the norm layout
  constexpr int CP = NB * WC * 8;     // padded output columns (norm_part stride)
  const Ring ring{reinterpret_cast<uint64_t*>(smem)};
  double* buf = reinterpret_cast<double*>(smem + kBarBytes);
  const int xs_d = R * KC, stage_d = xs_d + KC * LDM;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int64_t ntiles = ceil_div(m, R);
  constexpr bool sk = SK;
  const int64_t units = ntiles * kc_count;
  const int64_t u0 = sk ? sk_u0(blockIdx.x, units, gridDim.x) : 0;
  const int64_t mytiles = blockIdx.x < ntiles ? ceil_div(ntiles - blockIdx.x, (int64_t)gridDim.x) : 0;
  const int64_t nsteps = sk ? sk_u0(blockIdx.x + 1, units, gridDim.x) - u0 : mytiles * kc_count;
  const int64_t first_tile = sk ? u0 / kc_count : -1;
  // Step s -> (row tile, K chunk) and (ring slot, phase), advanced incrementally: one
  // division at the start instead of four 64-bit divisions per stage (ncu r2: the integer
  // work of the stage boundaries was 10% of the alpha pass's issue samples).
  struct Cursor {
    int64_t tile;
    int chunk, b;
    uint32_t ph;
  };
  const Cursor cur0{sk ? first_tile : (int64_t)blockIdx.x, sk ? (int)(u0 % kc_count) : 0, 0, 0u};
  auto advance = [&](Cursor& q) {
    if (++q.chunk == kc_count) {
      q.chunk = 0;
      q.tile += sk ? 1 : (int64_t)gridDim.x;
    }
    if (++q.b == nst) q.b = 0, q.ph ^= 1u;
  };
  ring_init(ring, nst, NN_CW);

  if (warp == NN_CW) {  // ---- producer (last warp)
    if (lane == 0) {
      Cursor q = cur0;
      for (int64_t s = 0; s < nsteps; ++s, advance(q)) {
        const int b = q.b;
        if (s >= nst) mbar_wait(ring.empty(b), q.ph ^ 1u);
        const int64_t tile = q.tile;
        const int k0 = q.chunk * KC;
        double* xs = buf + b * stage_d;
        mbar_arrive_expect_tx(ring.full(b), (uint32_t)(stage_d * 8));
        // the X box in TMA boxes of at most 256 rows (R = 384 with 12 consumer warps)
        constexpr int RB = R <= 256 ? R : R / 2;
#pragma unroll
        for (int h = 0; h < R / RB; ++h)
          tma_load_2d(xs + h * RB * KC, &tx, k0, (int)(tile * R + h * RB), ring.full(b));
        tma_load_2d(xs + xs_d, &tm, 0, k0, ring.full(b));
      }
    }
    return;
  }
  const int rg = warp % RW, cg = warp / RW;
  const int col0 = cg * NIW * 8;

  double acc[MI][NIW][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NIW; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  // per-warp column sums of squares (norm epilogue): in registers over the whole
  // run when they fit (NRM), else per tile into a shared-memory row after the stages
  constexpr bool NRM = 2 * MI * NIW + 2 * NIW + MI * XR + XR <= 56;  // (measured: no spills up to 56)
  double nacc[NRM ? NIW : 1][2];
#pragma unroll
  for (int j = 0; j < (NRM ? NIW : 1); ++j) nacc[j][0] = nacc[j][1] = 0.0;
  double ex[MI][XR > 0 ? XR : 1], nx[XR > 0 ? XR : 1];  // remainder-column partials and norms
#pragma unroll
  for (int x = 0; x < (XR > 0 ? XR : 1); ++x) {
    nx[x] = 0.0;
#pragma unroll
    for (int i = 0; i < MI; ++i) ex[i][x] = 0.0;
  }
  double* red = buf + nst * stage_d + warp * NB * 8;
  if (norm_part && !NRM)
    for (int col = lane; col < NB * 8; col += 32) red[col] = 0.0;

  bool partial = false;  // stream-K: this CTA's part of the current tile misses chunks
  Cursor q = cur0;
  for (int64_t s = 0; s < nsteps; ++s, advance(q)) {
    const int b = q.b;
    mbar_wait(ring.full(b), q.ph);
    const double* xs = buf + b * stage_d + (rg * MI * 8 + g) * KC + t;
    const double* ms = buf + b * stage_d + xs_d + t * LDM + col0 + g;
    TCHECK(((rg * MI + MI - 1) * 8 + g) * KC + t + KC - 4 < xs_d && col0 + (NIW - 1) * 8 + g < LDM);
    int64_t tile = q.tile;
    const int kc_here = q.chunk;
    if constexpr (SK)
      if (s == 0 || kc_here == 0) partial = kc_here != 0;
    // k-steps holding real columns (stream-K with KCT: all of them, the zero-filled ones included)
    const int nks = SK && KCT > 0 ? KCT / 4 : min(KC / 4, (k - kc_here * KC + 3) / 4);
    // (software-pipelining the fragment loads, as gemm_tn does, measured slower
    // here: 7.9 -> 9.0 ms per c3 alpha pass.)  SK: the fragments of a k-step are loaded
    // before its first DMMA (c3 alpha 7.2 -> 6.9 ms); the same source order made the
    // row-tile passes slower (c2 A V~ 1.06 -> 1.18 ms), so they keep the per-column-block
    // loads (measured r2, tools/nn_bench.py).
    auto row_tile_step = [&](int kk) {
      double a[MI];
#pragma unroll
      for (int i = 0; i < MI; ++i) a[i] = xs[i * 8 * KC + kk * 4];
#pragma unroll
      for (int j = 0; j < NIW; ++j) {
        const double bf = ms[kk * 4 * LDM + j * 8];
#pragma unroll
        for (int i = 0; i < MI; ++i) dmma(acc[i][j], a[i], bf);
      }
      if constexpr (XR > 0) {
#pragma unroll
        for (int x = 0; x < XR; ++x) {
          const double mv = ms[kk * 4 * LDM - g + NIW * 8 + x];
#pragma unroll
          for (int i = 0; i < MI; ++i) ex[i][x] = fma(a[i], mv, ex[i][x]);
        }
      }
    };
    if constexpr (!SK && KCT > 0) {  // constant chunk: unrolled, the last chunk's padding skipped
#pragma unroll
      for (int kk = 0; kk < KCT / 4; ++kk)
        if (kk < nks) row_tile_step(kk);
    } else if constexpr (!SK) {
      for (int kk = 0; kk < nks; ++kk) row_tile_step(kk);
    } else
#pragma unroll
    for (int kk = 0; kk < nks; ++kk) {
      double a[MI], bfr[NIW], mv[XR > 0 ? XR : 1];
#pragma unroll
      for (int j = 0; j < NIW; ++j) bfr[j] = ms[kk * 4 * LDM + j * 8];
#pragma unroll
      for (int i = 0; i < MI; ++i) a[i] = xs[i * 8 * KC + kk * 4];
      if constexpr (XR > 0)  // M[4kk + t][8 NIW + x]: one broadcast load per t
#pragma unroll
        for (int x = 0; x < XR; ++x) mv[x] = ms[kk * 4 * LDM - g + NIW * 8 + x];
#pragma unroll
      for (int j = 0; j < NIW; ++j)
#pragma unroll
        for (int i = 0; i < MI; ++i) dmma(acc[i][j], a[i], bfr[j]);
      if constexpr (XR > 0)
#pragma unroll
        for (int x = 0; x < XR; ++x)
#pragma unroll
          for (int i = 0; i < MI; ++i) ex[i][x] = fma(a[i], mv[x], ex[i][x]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(ring.empty(b));
    if constexpr (SK)
      if (s == nsteps - 1 && kc_here != kc_count - 1) partial = true;
    if (SK && partial && (kc_here == kc_count - 1 || s == nsteps - 1)) {
      // stream-K partial tile: accumulators to this CTA's record (summed by gemm_nn_fixup)
      double* rec = sk_rec + (size_t)(2 * blockIdx.x + (tile == first_tile ? 0 : 1)) * R * CP;
      TCHECK(tile >= first_tile && tile < ntiles && col0 + NIW * 8 <= CP);
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const int row = (rg * MI + i) * 8 + g;
#pragma unroll
        for (int j = 0; j < NIW; ++j) {
          *reinterpret_cast<double2*>(rec + (size_t)row * CP + col0 + j * 8 + 2 * t) =
              make_double2(acc[i][j][0], acc[i][j][1]);
          acc[i][j][0] = acc[i][j][1] = 0.0;
        }
        if constexpr (XR > 0) {
#pragma unroll
          for (int x = 0; x < XR; ++x) {
            double v = ex[i][x];
            v += __shfl_xor_sync(0xffffffffu, v, 1);
            v += __shfl_xor_sync(0xffffffffu, v, 2);
            ex[i][x] = 0.0;
            if (t == x) rec[(size_t)row * CP + NIW * 8 + x] = v;
          }
        }
      }
    } else if (kc_here == kc_count - 1) {  // tile complete: epilogue
      if (norm_part && NRM) {  // rows beyond m hold zeros (TMA zero fill): no masking needed
#pragma unroll
        for (int j = 0; j < (NRM ? NIW : 1); ++j)
#pragma unroll
          for (int i = 0; i < MI; ++i) {
            nacc[j][0] = fma(acc[i][j][0], acc[i][j][0], nacc[j][0]);
            nacc[j][1] = fma(acc[i][j][1], acc[i][j][1], nacc[j][1]);
          }
      } else if (norm_part) {
#pragma unroll
        for (int j = 0; j < NIW; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            double v = 0.0;
#pragma unroll
            for (int i = 0; i < MI; ++i) v = fma(acc[i][j][e], acc[i][j][e], v);
            v += __shfl_xor_sync(0xffffffffu, v, 4);
            v += __shfl_xor_sync(0xffffffffu, v, 8);
            v += __shfl_xor_sync(0xffffffffu, v, 16);
            if (g == 0) red[j * 8 + 2 * t + e] += v;
          }
      }
      if constexpr (XR > 0) {  // remainder columns: sum the four t-partials, store, norms
#pragma unroll
        for (int i = 0; i < MI; ++i) {
          const int64_t row = tile * R + (rg * MI + i) * 8 + g;
#pragma unroll
          for (int x = 0; x < XR; ++x) {
            double v = ex[i][x];
            v += __shfl_xor_sync(0xffffffffu, v, 1);
            v += __shfl_xor_sync(0xffffffffu, v, 2);
            ex[i][x] = 0.0;
            if (t == x && row < m && Y) Y[row * ldy + NIW * 8 + x] = v;
            nx[x] = fma(v, v, nx[x]);  // rows beyond m are zero
          }
        }
      }
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const int64_t row = tile * R + (rg * MI + i) * 8 + g;
        const bool rv = row < m;
#pragma unroll
        for (int j = 0; j < NIW; ++j) {
          const int col = col0 + j * 8 + 2 * t;
          if (rv && Y) {
            if (col + 1 < c)
              *reinterpret_cast<double2*>(Y + row * ldy + col) = make_double2(acc[i][j][0], acc[i][j][1]);
            else if (col < c)
              Y[row * ldy + col] = acc[i][j][0];
          }
          acc[i][j][0] = acc[i][j][1] = 0.0;
        }
      }
    }
  }

  if (norm_part) {  // sum the row-group warps of each column group in a fixed order
    if constexpr (NRM) {
#pragma unroll
      for (int j = 0; j < (NRM ? NIW : 1); ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          double v = nacc[j][e];
          v += __shfl_xor_sync(0xffffffffu, v, 4);
          v += __shfl_xor_sync(0xffffffffu, v, 8);
          v += __shfl_xor_sync(0xffffffffu, v, 16);
          if (g == 0) red[j * 8 + 2 * t + e] = v;
        }
    }
    if constexpr (XR > 0) {  // every t-lane holds the same sums: sum over g only
#pragma unroll
      for (int x = 0; x < XR; ++x) {
        double v = nx[x];
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        nx[x] = v;
      }
      if (lane < 8) red[NIW * 8 + lane] = lane == 0 ? nx[0] : (XR > 1 && lane == 1 ? nx[XR > 1 ? 1 : 0] : 0.0);
    }
    bar_consumers(NN_CW * 32);
    const double* red0 = buf + nst * stage_d;
    for (int col = threadIdx.x; col < CP; col += NN_CW * 32) {
      const int cgi = col / (NB * 8), cc = col % (NB * 8);
      double v = 0.0;
      for (int r2 = 0; r2 < RW; ++r2) v += red0[(cgi * RW + r2) * NB * 8 + cc];
      norm_part[(size_t)blockIdx.x * CP + col] = v;
    }
  }
}

// Stream-K fixup: one block per CTA boundary b >= 1 that cuts a tile t (and is the first
// boundary inside t): the records of the CTAs covering t are summed in CTA order (= K
// order, fixed) and the rows of t stored (columns < c, rows < m).
__global__ void __launch_bounds__(256) gemm_nn_fixup(const double* __restrict__ rec, int R, int CP, int c,
                                                    int64_t m, int64_t ntiles, int kc_count, int grid,
                                                    double* Y, int64_t ldy) {
  __shared__ int s_slot[1024];  // record slots of the CTAs covering the tile, in CTA (= K) order
  __shared__ int s_n;
  const int b = blockIdx.x + 1;
  const int64_t units = ntiles * kc_count;
  const int64_t ub = sk_u0(b, units, grid);
  if (ub % kc_count == 0 || ub >= units) return;
  const int64_t t = ub / kc_count;
  if (sk_u0(b - 1, units, grid) > t * kc_count) return;  // an earlier boundary cut t already
  if (threadIdx.x == 0) {
    int n = 0;
    for (int q = b - 1; q < grid && n < 1024 && sk_u0(q, units, grid) < (t + 1) * kc_count; ++q)
      s_slot[n++] = 2 * q + (sk_u0(q, units, grid) / kc_count == t ? 0 : 1);
    s_n = n;
  }
  __syncthreads();
  const int nq = s_n;
  const int64_t rows = min((int64_t)R, m - t * R);
  for (int e = threadIdx.x; e < rows * c; e += blockDim.x) {
    const int row = e / c, col = e % c;
    double v = 0.0;
    for (int q = 0; q < nq; ++q) v += rec[((size_t)s_slot[q] * R + row) * CP + col];
    Y[(t * R + row) * ldy + col] = v;
  }
}

// Warp grid and rows per tile from the accumulator budget (<= 24 8x8 tiles,
// <= 16 column blocks per warp); c = 8 ni + 1 or + 2 (1 <= ni <= 4, where the
// extra accumulators still fit without spills) puts the last one or two columns
// on the FMA pipe (xr).
struct NnShape {
  int ni, xr, wc, niw, mi;
};
static int nn_xr(int c) { return (c % 8 == 1 || c % 8 == 2) && c > 8 && c / 8 <= 4 ? c % 8 : 0; }
static NnShape nn_shape(int c) {
  NnShape sh;
  sh.xr = nn_xr(c);
  sh.ni = sh.xr ? c / 8 : (c + 7) / 8;
  // two column groups from 12 column blocks on: each warp then holds 3 x 6..8
  // tiles instead of 1 x 12..16, 0.5 instead of 1.07 fragment loads per DMMA
  // (c4 A V~ 13.36 -> 13.14 ms); below 12 the padded column block costs more
  // (c2, 9 blocks: 1.02 -> 1.09 ms).  TSSVD_NN_WC2 moves the threshold (experiments).
  static const int wc2_from = getenv("TSSVD_NN_WC2") ? atoi(getenv("TSSVD_NN_WC2")) : 12;
  // four column groups from wc4_from column blocks on (experiments: TSSVD_NN_WC4)
  // four column groups from 20 column blocks on (3 x 5..8 tiles per warp instead of 1 x 10..16:
  // c = 160..256 at 29-33 TF instead of 16-30; measured r2, tools/nn_bench.py); TSSVD_NN_WC4
  // moves the threshold (experiments)
  static const int wc4_from = getenv("TSSVD_NN_WC4") ? atoi(getenv("TSSVD_NN_WC4")) : 20;
  sh.wc = sh.ni < wc2_from || sh.xr ? 1 : (sh.ni >= wc4_from && sh.ni >= 20 ? 4 : 2);
  sh.niw = (sh.ni + sh.wc - 1) / sh.wc;
  sh.mi = std::max(1, std::min(4, 24 / sh.niw));
  // remainder-column shapes (c = 8j + 1/2, j <= 4): TSSVD_NN_MI = 2/3/4 row blocks per warp
  // (R = 96 MI rows per tile; experiments)
  static const int force_mi = getenv("TSSVD_NN_MI") ? atoi(getenv("TSSVD_NN_MI")) : 0;
  if (sh.xr && force_mi >= 2 && force_mi <= 4) sh.mi = force_mi;
  return sh;
}

struct NnPlan {
  NnShape sh;
  int ni, R, KC, kcc, nst, grid, ldm, cp;
  bool sk;  // stream-K work split (see gemm_nn_kernel)
  size_t smem;
};

int gemm_nn_part_stride(int c);

// K chunk (= 4 mod 8, <= 252) and stage count from shared memory: fewest
// zero-filled columns, then fewest chunks, with at least 2 stages (3
// preferred).  (Measured at c2: 2 chunks x 2 stages beat 4 chunks x 4 stages.)
static NnPlan plan_nn(int64_t m, int k, int c) {
  NnPlan p;
  p.sh = nn_shape(c);
  p.ni = p.sh.ni;
  const int ncw = nn_cw(p.sh.mi, p.sh.niw, p.sh.wc);
  p.R = 8 * p.sh.mi * (ncw / p.sh.wc);
  // smem row stride of the M box: covers every column block a warp reads (the padded last one
  // included, zero-filled by TMA beyond M's width), TMA box limit 256
  p.ldm = std::min(smem_ld(std::max(c, p.sh.niw * p.sh.wc * 8)), 256);
  const size_t red = (size_t)ncw * (p.sh.niw + (p.sh.xr > 0)) * 8 * 8;
  const size_t budget = dev_info().smem_optin - kBarBytes - red;
  double best = 1e300;
  p.KC = 28;
  for (int kc = 28; kc <= 252; kc += 8) {
    const size_t stage = (size_t)(p.R * kc + kc * p.ldm) * 8;
    const int nst = (int)std::min<size_t>(8, budget / stage);
    if (nst < 2) break;
    const int chunks = (int)ceil_div(k, kc);
    const double waste = (double)(chunks * kc - k) / k;
    const double score = waste + chunks / (double)k + (nst < 3 ? 0.05 : (nst < 4 ? 0.02 : 0.0));
    if (score < best) best = score, p.KC = kc;
  }
  static const int force_kc = getenv("TSSVD_NN_KC") ? atoi(getenv("TSSVD_NN_KC")) : 0;  // experiments
  if (force_kc >= 12 && force_kc % 8 == 4) p.KC = force_kc;
  p.kcc = (int)ceil_div(k, p.KC);
  const size_t stage = (size_t)(p.R * p.KC + p.KC * p.ldm) * 8;
  p.nst = (int)std::max<size_t>(2, std::min<size_t>(8, budget / stage));
  p.smem = kBarBytes + (size_t)p.nst * stage + red;
  const int64_t ntiles = ceil_div(m, p.R);
  p.grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, dev_info().sms));
  p.cp = gemm_nn_part_stride(c);
  // stream-K when the row tiles keep less than 97% of the SMs busy over the waves (a
  // ragged last wave, or fewer tiles than SMs: then it is a split-K) and K has >= 2 chunks
  // (TSSVD_NN_SK=0/1 forces, experiments)
  static const int force_sk = getenv("TSSVD_NN_SK") ? atoi(getenv("TSSVD_NN_SK")) : -1;
  const int sms = dev_info().sms;
  const double tail = (double)ceil_div(ntiles, sms) * sms / (double)ntiles - 1.0;
  p.sk = p.kcc >= 2 && ntiles * p.kcc >= 2 * dev_info().sms && (force_sk >= 0 ? force_sk == 1 : tail > 0.03);
  if (p.sk) p.grid = dev_info().sms;
  return p;
}

int gemm_nn_grid(int64_t m, int c) {
  const NnShape sh = nn_shape(c);
  const int R = 8 * sh.mi * (nn_cw(sh.mi, sh.niw, sh.wc) / sh.wc);
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(m, R), dev_info().sms));
}
int gemm_nn_part_stride(int c) {
  const NnShape sh = nn_shape(c);
  return (sh.niw + (sh.xr > 0)) * sh.wc * 8;
}
size_t gemm_nn_m_doubles(int k, int c) { return (size_t)ceil_div(k + 1, 32) * 32 * smem_ld(c); }
size_t gemm_nn_scratch_max(int k, int c) {  // for any m: the records do not depend on m
  if (c <= 0 || c > 256) return 0;
  NnPlan p = plan_nn(1 << 20, std::max(k, 1), c);
  return p.kcc >= 2 ? (size_t)2 * dev_info().sms * p.R * p.cp : 0;
}
size_t gemm_nn_scratch_doubles(int64_t m, int k, int c) {
  if (c <= 0 || c > 256) return 0;
  const NnPlan p = plan_nn(std::max<int64_t>(m, 1), std::max(k, 1), c);
  return p.sk ? (size_t)2 * p.grid * p.R * p.cp : 0;
}

template <int MI, int NIW, int WC, int XR>
static cudaError_t nn_go(const NnPlan& p, const CUtensorMap& tx, const CUtensorMap& tm, int64_t m,
                         int k, int c, double* Y, int64_t ldy, double* norm_part, double* sk_rec,
                         cudaStream_t s) {
  // the planner's usual K chunks as compile-time constants (stream-K: 20, 28; row tiles: 52;
  // TSSVD_NN_KCT=0: runtime KC, A/B runs)
  static const bool kct = !getenv("TSSVD_NN_KCT") || atoi(getenv("TSSVD_NN_KCT")) != 0;
  // (row tiles with KC = 28 measured 7% slower as a constant -- c2's 55-column passes: 0.471 ->
  // 0.506 ms -- and KC = 52 2% faster: c2 A V~ 1.007 -> 0.988 ms, c4 14.21 -> 13.89 ms)
  auto kern = !sk_rec ? (kct && p.KC == 52 ? gemm_nn_kernel<MI, NIW, WC, XR, false, 52>
                                           : gemm_nn_kernel<MI, NIW, WC, XR, false>)
              : kct && p.KC == 20 ? gemm_nn_kernel<MI, NIW, WC, XR, true, 20>
              : kct && p.KC == 28 ? gemm_nn_kernel<MI, NIW, WC, XR, true, 28>
                                  : gemm_nn_kernel<MI, NIW, WC, XR, true>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
  if (e != cudaSuccess) return e;
  kern<<<p.grid, (nn_cw(MI, NIW, WC) + 1) * 32, p.smem, s>>>(tx, tm, m, k, p.KC, p.kcc, p.ldm, c, Y, ldy, norm_part,
                                                p.nst, sk_rec);
  e = cudaGetLastError();
  if (e != cudaSuccess || !sk_rec) return e;
  gemm_nn_fixup<<<p.grid - 1 > 0 ? p.grid - 1 : 1, 256, 0, s>>>(sk_rec, p.R, p.cp, c, m, ceil_div(m, p.R), p.kcc,
                                                               p.grid, Y, ldy);
  return cudaGetLastError();
}

template <int NI, int XR = 0, int WCF = 0>
static cudaError_t nn_ni_go(const NnPlan& p, const CUtensorMap& tx, const CUtensorMap& tm, int64_t m,
                            int k, int c, double* Y, int64_t ldy, double* np, double* sk_rec, cudaStream_t s) {
  constexpr int WC = WCF ? WCF : (NI <= 16 ? 1 : 2);
  constexpr int NIW = (NI + WC - 1) / WC;
  constexpr int MI = 24 / NIW < 1 ? 1 : (24 / NIW > 4 ? 4 : 24 / NIW);
  if constexpr (XR > 0 && MI == 4) {  // remainder shapes: the planner's row blocks per warp
    if (p.sh.mi == 2) return nn_go<2, NIW, WC, XR>(p, tx, tm, m, k, c, Y, ldy, np, sk_rec, s);
    if (p.sh.mi == 3) return nn_go<3, NIW, WC, XR>(p, tx, tm, m, k, c, Y, ldy, np, sk_rec, s);
  }
  return nn_go<MI, NIW, WC, XR>(p, tx, tm, m, k, c, Y, ldy, np, sk_rec, s);
}

cudaError_t launch_gemm_nn(const double* X, int64_t ldx, int64_t m, int k, const double* M,
                           int c, double* Y, int64_t ldy, double* norm_part, double* scratch,
                           cudaStream_t s) {
  if (c <= 0) return cudaSuccess;
  if (c > 256) return cudaErrorInvalidValue;
  NnPlan p = plan_nn(std::max<int64_t>(m, 1), std::max(k, 1), c);
  // stream-K needs the caller's scratch (gemm_nn_scratch_doubles) and no norm epilogue
  double* sk_rec = p.sk && scratch && !norm_part && Y ? scratch : nullptr;
  if (p.sk && !sk_rec) {
    p.sk = false;
    p.grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(std::max<int64_t>(m, 1), p.R), dev_info().sms));
  }
  if (m <= 0 || k <= 0) {
    if (norm_part) return cudaMemsetAsync(norm_part, 0, (size_t)p.grid * gemm_nn_part_stride(c) * 8, s);
    return cudaSuccess;
  }
  CUtensorMap tx, tm;
  cudaError_t e = make_tmap(&tx, X, m, k, ldx, p.R <= 256 ? p.R : p.R / 2, p.KC);
  if (e != cudaSuccess) return e;
  e = make_tmap(&tm, M, k, smem_ld(c), smem_ld(c), p.KC, p.ldm);
  if (e != cudaSuccess) return e;
#define NN_XCASE(N) \
  case N: return p.sh.xr == 1 ? nn_ni_go<N, 1>(p, tx, tm, m, k, c, Y, ldy, norm_part, sk_rec, s) \
                              : nn_ni_go<N, 2>(p, tx, tm, m, k, c, Y, ldy, norm_part, sk_rec, s);
  if (p.sh.xr) switch (p.ni) {
      NN_XCASE(1) NN_XCASE(2) NN_XCASE(3) NN_XCASE(4)
      default: return cudaErrorInvalidValue;
    }
#undef NN_XCASE
#define NN_WCASE(N) \
  case N: return nn_ni_go<N, 0, 2>(p, tx, tm, m, k, c, Y, ldy, norm_part, sk_rec, s);
  if (p.sh.wc == 2 && p.ni <= 16) switch (p.ni) {
      NN_WCASE(9) NN_WCASE(10) NN_WCASE(11) NN_WCASE(12) NN_WCASE(13) NN_WCASE(14) NN_WCASE(15) NN_WCASE(16)
      default: return cudaErrorInvalidValue;
    }
#undef NN_WCASE
#define NN_W4CASE(N) \
  case N: return nn_ni_go<N, 0, 4>(p, tx, tm, m, k, c, Y, ldy, norm_part, sk_rec, s);
  if (p.sh.wc == 4) switch (p.ni) {
      NN_W4CASE(20) NN_W4CASE(21) NN_W4CASE(22) NN_W4CASE(23) NN_W4CASE(24) NN_W4CASE(25) NN_W4CASE(26)
      NN_W4CASE(27) NN_W4CASE(28) NN_W4CASE(29) NN_W4CASE(30) NN_W4CASE(31) NN_W4CASE(32)
      default: return cudaErrorInvalidValue;
    }
#undef NN_W4CASE
#define NN_CASE(N) \
  case N: return nn_ni_go<N>(p, tx, tm, m, k, c, Y, ldy, norm_part, sk_rec, s);
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
// split's row range (a multiple of KR rows, so only the last split's last box
// can cross m, where TMA zero-fills).  Consumer warp w owns X-column blocks
// w*MI..w*MI+MI-1 and all NBL column blocks of Y.  Fragments: A = X^T (8x4)
// -> Xs[k][i0+g], B = Y (4x8) -> Ys[k][j0+g], k = kk*4 + t.  The X box is
// CB + 4 columns wide (the 4 extra columns only pad the smem rows to = 4 mod 8).
// XR > 0 (l = 8 NBL + XR): the last XR columns of Y on the FMA pipe, as in gemm_nn
// (lane (g, t) holds X[4kk + t][i0 + g] as its A fragment; the four t-partials
// are summed by a butterfly before the store).
static constexpr int TN_CW = 12;  // 3 consumer warps per SMSP: 8 -> 12 took c3 beta 7.7 -> 6.7 ms/pass

// KRT > 0: rows per stage as a compile-time constant (the planner's usual 32): the k-steps of a
// stage unroll with immediate shared-memory offsets.
template <int MI, int NBL, int XR, int KRT = 0>
__global__ void __launch_bounds__(32 * (TN_CW + 1)) gemm_tn_kernel(
    const __grid_constant__ CUtensorMap tx, const __grid_constant__ CUtensorMap ty, int64_t m, int n,
    int64_t rps, double* __restrict__ part, int ldz, int64_t n_pad, int KR_rt, int nst) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int KR = KRT > 0 ? KRT : KR_rt;
  constexpr int CB = 8 * MI * TN_CW;
  constexpr int LDXS = CB + 4;
  constexpr int LDYS = NBL * 8 + 4;
  const Ring ring{reinterpret_cast<uint64_t*>(smem)};
  double* buf = reinterpret_cast<double*>(smem + kBarBytes);
  const int xs_d = KR * LDXS, stage_d = KR * (LDXS + LDYS);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int c0 = blockIdx.x * CB;
  const int64_t r0 = (int64_t)blockIdx.y * rps;
  const int64_t r1 = min(m, r0 + rps);
  const int nsteps = r1 > r0 ? (int)ceil_div(r1 - r0, KR) : 0;
  ring_init(ring, nst, TN_CW);

  if (warp == TN_CW) {  // ---- producer
    if (lane == 0) {
      int b = 0;
      uint32_t ph = 0;
      for (int s = 0; s < nsteps; ++s) {  // ring slot and phase advanced incrementally
        if (s >= nst) mbar_wait(ring.empty(b), ph ^ 1u);
        const int rs = (int)(r0 + (int64_t)s * KR);
        double* xs = buf + b * stage_d;
        mbar_arrive_expect_tx(ring.full(b), (uint32_t)(stage_d * 8));
        tma_load_2d(xs, &tx, c0, rs, ring.full(b));
        tma_load_2d(xs + xs_d, &ty, 0, rs, ring.full(b));
        if (++b == nst) b = 0, ph ^= 1u;
      }
    }
    return;
  }

  double acc[MI][NBL][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NBL; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  double ex[MI][XR > 0 ? XR : 1];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int x = 0; x < (XR > 0 ? XR : 1); ++x) ex[i][x] = 0.0;

  int b = 0;
  uint32_t ph = 0;
  for (int s = 0; s < nsteps; ++s) {
    mbar_wait(ring.full(b), ph);
    const double* xs = buf + b * stage_d + t * LDXS + warp * MI * 8 + g;
    const double* ys = buf + b * stage_d + xs_d + t * LDYS + g;
    // software-pipelined fragment loads, as in gemm_nn
    constexpr int XRA = XR > 0 ? XR : 1;
    const int nkk = KR / 4;
    double a[MI], bf[NBL], yv[XRA];
    auto load = [&](int q, double (&fa)[MI], double (&fb)[NBL], double (&fy)[XRA]) {
#pragma unroll
      for (int i = 0; i < MI; ++i) fa[i] = xs[q * 4 * LDXS + i * 8];
#pragma unroll
      for (int j = 0; j < NBL; ++j) fb[j] = ys[q * 4 * LDYS + j * 8];
      if constexpr (XR > 0)  // Y[4q + t][8 NBL + x]: one broadcast load per t
#pragma unroll
        for (int x = 0; x < XR; ++x) fy[x] = ys[q * 4 * LDYS + NBL * 8 + x - g];
    };
    load(0, a, bf, yv);
#pragma unroll
    for (int kk = 0; kk < nkk; ++kk) {
      double an[MI], bn[NBL], yn[XRA];
      load(min(kk + 1, nkk - 1), an, bn, yn);
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NBL; ++j) dmma(acc[i][j], a[i], bf[j]);
      if constexpr (XR > 0)
#pragma unroll
        for (int x = 0; x < XR; ++x)
#pragma unroll
          for (int i = 0; i < MI; ++i) ex[i][x] = fma(a[i], yv[x], ex[i][x]);
#pragma unroll
      for (int i = 0; i < MI; ++i) a[i] = an[i];
#pragma unroll
      for (int j = 0; j < NBL; ++j) bf[j] = bn[j];
#pragma unroll
      for (int x = 0; x < XRA; ++x) yv[x] = yn[x];
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(ring.empty(b));
    if (++b == nst) b = 0, ph ^= 1u;
  }

  double* P = part + (size_t)blockIdx.y * n_pad * ldz;
  TCHECK(c0 + CB <= n_pad && NBL * 8 <= ldz);
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const int row = c0 + (warp * MI + i) * 8 + g;
    if (row >= n) continue;
#pragma unroll
    for (int j = 0; j < NBL; ++j)
      *reinterpret_cast<double2*>(P + (size_t)row * ldz + j * 8 + 2 * t) =
          make_double2(acc[i][j][0], acc[i][j][1]);
  }
  if constexpr (XR > 0) {  // columns 8 NBL .. 8 NBL + 7 of the partial: remainder sums, then zeros
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      double v0 = ex[i][0], v1 = 0.0;
      v0 += __shfl_xor_sync(0xffffffffu, v0, 1);
      v0 += __shfl_xor_sync(0xffffffffu, v0, 2);
      if constexpr (XR > 1) {
        v1 = ex[i][XR > 1 ? 1 : 0];
        v1 += __shfl_xor_sync(0xffffffffu, v1, 1);
        v1 += __shfl_xor_sync(0xffffffffu, v1, 2);
      }
      const int row = c0 + (warp * MI + i) * 8 + g;
      if (row < n)
        *reinterpret_cast<double2*>(P + (size_t)row * ldz + NBL * 8 + 2 * t) =
            t == 0 ? make_double2(v0, v1) : make_double2(0.0, 0.0);
    }
  }
}

TnPlan plan_gemm_tn(int64_t m, int n, int l) {
  TnPlan p;
  p.xr = (l % 8 == 1 || l % 8 == 2) && l > 8 && l / 8 <= 5 ? l % 8 : 0;  // remainder columns on the FMA pipe
  p.nbl = p.xr ? l / 8 : (l + 7) / 8;
  p.mi = p.nbl <= 8 ? 2 : 1;
  p.cb = 8 * p.mi * TN_CW;
  p.ldz = pad8(l);
  p.colblocks = (int)ceil_div(n, p.cb);
  const size_t row_bytes = (size_t)((p.cb + 4) + (p.nbl * 8 + 4)) * 8;
  const size_t budget = dev_info().smem_optin - kBarBytes;
  p.kr = 32;
  while (p.kr > 8 && 3 * p.kr * row_bytes > budget) p.kr -= 8;
  p.nst = (int)std::min<size_t>(8, budget / (p.kr * row_bytes));
  const int sms = dev_info().sms;
  // split count: wave efficiency x per-CTA amortisation (a CTA's prologue -- ring
  // set-up, first TMA round trip -- and partial write cost ~20 stages, measured)
  int best = 1;
  double best_eff = -1;
  for (int s = 1; s <= 64; ++s) {
    if (s > 1 && ceil_div(m, s) < 256) break;
    const int64_t tot = (int64_t)p.colblocks * s;
    const double eff = (double)tot / (double)(ceil_div(tot, sms) * sms);
    const double steps = (double)ceil_div(ceil_div(m, s), p.kr);
    const double score = eff * std::min(1.0, (double)tot / sms) * steps / (steps + 20.0);
    if (score > best_eff + 1e-9) best_eff = score, best = s;
  }
  p.splits = best;
  p.rows_per_split = ceil_div(ceil_div(std::max<int64_t>(m, 1), p.splits), p.kr) * p.kr;
  p.part_doubles = (size_t)p.splits * p.colblocks * p.cb * p.ldz;
  return p;
}

template <int MI, int NBL, int XR = 0>
static cudaError_t tn_go(const TnPlan& p, const CUtensorMap& tx, const CUtensorMap& ty, int64_t m, int n,
                         double* part, cudaStream_t s) {
  const size_t smem = kBarBytes + (size_t)p.nst * p.kr * ((p.cb + 4) + (NBL * 8 + 4)) * 8;
  static const bool krt = !getenv("TSSVD_TN_KRT") || atoi(getenv("TSSVD_TN_KRT")) != 0;  // experiments
  auto kern = krt && p.kr == 32 ? gemm_tn_kernel<MI, NBL, XR, 32> : gemm_tn_kernel<MI, NBL, XR>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(p.colblocks, p.splits);
  kern<<<grid, (TN_CW + 1) * 32, smem, s>>>(tx, ty, m, n, p.rows_per_split, part, p.ldz,
                                            (int64_t)p.colblocks * p.cb, p.kr, p.nst);
  return cudaGetLastError();
}

cudaError_t launch_gemm_tn(const TnPlan& p, const double* X, int64_t ldx, int64_t m, int n,
                           const double* Y, int64_t ldy, int l, double* part, cudaStream_t s) {
  if (m <= 0) return cudaMemsetAsync(part, 0, p.part_doubles * 8, s);
  CUtensorMap tx, ty;
  cudaError_t e = make_tmap(&tx, X, m, n, ldx, p.kr, p.cb + 4);
  if (e != cudaSuccess) return e;
  e = make_tmap(&ty, Y, m, l, ldy, p.kr, p.nbl * 8 + 4);
  if (e != cudaSuccess) return e;
#define TN_XCASE(MI, NB)                                                                   \
  if (p.xr && p.mi == MI && p.nbl == NB)                                                   \
    return p.xr == 1 ? tn_go<MI, NB, 1>(p, tx, ty, m, n, part, s) : tn_go<MI, NB, 2>(p, tx, ty, m, n, part, s);
  TN_XCASE(2, 1) TN_XCASE(2, 2) TN_XCASE(2, 3) TN_XCASE(2, 4) TN_XCASE(2, 5)
#undef TN_XCASE
  if (p.xr) return cudaErrorInvalidValue;
#define TN_CASE(MI, NB) \
  if (p.mi == MI && p.nbl == NB) return tn_go<MI, NB>(p, tx, ty, m, n, part, s);
  TN_CASE(2, 1) TN_CASE(2, 2) TN_CASE(2, 3) TN_CASE(2, 4)
  TN_CASE(2, 5) TN_CASE(2, 6) TN_CASE(2, 7) TN_CASE(2, 8)
  TN_CASE(1, 9) TN_CASE(1, 10) TN_CASE(1, 11) TN_CASE(1, 12) TN_CASE(1, 13) TN_CASE(1, 14)
  TN_CASE(1, 15) TN_CASE(1, 16)
#undef TN_CASE
  return cudaErrorInvalidValue;
}

}  // namespace tsk
