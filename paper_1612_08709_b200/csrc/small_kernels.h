// Launchers of the small replicated-core kernels (small_kernels.cu).
//
// Rank decisions stay on the device: the "Discard" kernel writes a decision slot
// (r, nc, non-finite flag, guard words; see k_discard) and every later kernel
// reads r / r2 from it (`rr`, `rr2`).  Host-side ints (`rb`, `rb2`, `kz`) are
// only SHAPE BOUNDS (grid sizes, leading dimensions): entries past the device
// count are written as zeros, so a launch sized by a bound computes exactly what
// a launch sized by the count would.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tsk {
// decision slot layout (ints)
constexpr int kSlotR = 0, kSlotNc = 1, kSlotBad = 2, kSlotGuard = 3, kSlotInts = 8;

void symmetrize(double* B, int w, int ldb, cudaStream_t s);
void unpack_sym(const double* packed, int w, double* B, int ldb, cudaStream_t s);
void cols_to_m(const double* cols, int ldc, int k, int c, double* M, int ldm, int mrows,
               cudaStream_t s);
void rows_to_m(const double* src, int64_t lds, int k, int c, double* M, int ldm, int mrows,
               cudaStream_t s);
void discard(const double* nsq, int w, double wp, double* sig, int* idx, int* out, const int* nf,
             cudaStream_t s);
void alg3_out(const double* sig, const int* idx, const int* rr, int rb, const double* Vt, int w,
              double* M, int ldm, double* sigma, double* V, int64_t ldv, cudaStream_t s);
void build_z(const double* G, int ldg, const int* idx, const double* sig, const int* rr, int rb,
             double* Z, cudaStream_t s);
void build_m1(const double* W, int ldw, const int* idx, const double* sig, const int* rr, int rb,
              int kz, double* M1, int ldm, cudaStream_t s);
void build_k(const double* T, const int* idx2, const int* rr2, int rb2, const double* W, int ldw,
             const int* rr, int rb, const double* sig, const int* idx, double* Kc, cudaStream_t s);
void svd_out(const double* cols, int ldc, const int* rr2, int rb2, const int* rr, const double* vals,
             const double* Vt, int w, const int* idx, double* sigma, double* V, int64_t ldv, double* Ps,
             cudaStream_t s);
void build_m2(const double* W, int ldw, const int* rr, int rb, const int* idx, const double* sig,
              const double* T, const int* idx2, const int* rr2, int ldp, const double* Ps, double* M2,
              int ldm, cudaStream_t s);
void canon_lowrank(double* VA, int64_t ldva, int n, double* Ut, int ldut, int r3, const int* rr4, int rb4,
                   cudaStream_t s);
void copy2d(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t rows, int cols,
            cudaStream_t s);
// wide core (wide_core.cu): Gram packing, V = V~_keep J with signs, M2 = S W T^-1 P
void pack_lower(const double* B, int w, int ldb, double* packed, cudaStream_t s);
void wide_svd_out(const double* cols, int ldc, const int* rr2, int rb2, const int* rr, int rb,
                  const double* vals, const double* Vt, int w, const int* idx, double* sigma, double* V,
                  int64_t ldv, double* Ps, double* vj_tmp, cudaStream_t s);
void wide_build_m2(const double* W, int ldw, const int* rr, int rb, const int* idx, const double* sig,
                   const double* T, const int* idx2, const int* rr2, int rb2, const double* Ps, double* M2, int ldm,
                   cudaStream_t s);
void fill(double* p, int64_t n, double v, cudaStream_t s);
}  // namespace tsk
