// Shared device helpers for the sm_100a kernels of the Gram-based SVD hot path.
// (No code here is shared with oracle/ -- the oracle is plain numpy.)
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

// Device-side bounds checks, compiled in only for the checking build
// (`python paper_1612_08709_b200/build.py --out tools/ab/libtssvd_checks.so -D TSSVD_CHECKS`,
// loaded through TSSVD_LIB): compute-sanitizer is closed on this pool, so the GPU test suite
// runs against this build instead -- a failed check traps the kernel and fails the test.
#ifdef TSSVD_CHECKS
#include <cassert>
#define TCHECK(c) assert(c)
#else
#define TCHECK(c) ((void)0)
#endif

namespace tsk {

constexpr double kEps = 2.220446049250313e-16;

// Shared-memory leading dimension (in doubles) for a row of `w` doubles:
// rounded up to a multiple of 8 columns (one DMMA n8/m8 block) plus 4, so that
// ld % 16 == 4 or 12.  A half-warp fragment load (4 rows x 4 consecutive
// doubles, lanes g=lane>>2, t=lane&3) then touches 4 distinct 32-byte bank
// groups: conflict-free for every fragment pattern used below.
__host__ __device__ inline int smem_ld(int w) { return ((w + 7) / 8) * 8 + 4; }
__host__ __device__ inline int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ inline int pad8(int w) { return ((w + 7) / 8) * 8; }
__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// D = A(8x4) * B(4x8) + D on the FP64 tensor pipe (SASS: DMMA.8x8x4).
// Fragments (PTX ISA, mma.m8n8k4 .f64): a = A[g][t], b = B[t][g],
// d = {D[g][2t], D[g][2t+1]} with g = lane>>2, t = lane&3.
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

// ---- mbarrier + bulk async copy (TMA engine, SASS: UBLKCP) -----------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// 2-D tensor TMA load of one box (SASS: UTMALDG); columns c0.., rows r0.. of the
// tensor map; out-of-bounds elements are zero-filled; completion on `bar`.
__device__ __forceinline__ void tma_load_2d(void* dst_smem, const CUtensorMap* map, int c0, int r0,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst_smem)),
      "l"(map), "r"(c0), "r"(r0), "r"(smem_u32(bar))
      : "memory");
}
// named barrier over the consumer warps only (the producer warp never joins)
__device__ __forceinline__ void bar_consumers(int nthreads) {
  asm volatile("bar.sync 1, %0;\n" ::"r"(nthreads) : "memory");
}

// global -> shared bulk copy of `bytes` (multiple of 16, both addresses 16-B aligned)
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---- warp reductions --------------------------------------------------------
__device__ __forceinline__ double warp_sum_bcast(double v) {
  // butterfly, then broadcast lane 0 so every lane holds bit-identical values
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return __shfl_sync(0xffffffffu, v, 0);
}

}  // namespace tsk
