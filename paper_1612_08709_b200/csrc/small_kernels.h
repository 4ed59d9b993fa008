// Launchers of the small replicated-core kernels (small_kernels.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tsk {
void symmetrize(double* B, int w, int ldb, cudaStream_t s);
void cols_to_m(const double* cols, int ldc, int k, int c, double* M, int ldm, int mrows,
               cudaStream_t s);
void rows_to_m(const double* src, int64_t lds, int k, int c, double* M, int ldm, int mrows,
               cudaStream_t s);
void discard(const double* nsq, int w, double wp, double* sig, int* idx, int* out,
             const double* gdiag, int gld, cudaStream_t s);
void alg3_out(const double* sig, const int* idx, int r, const double* Vt, int w, double* M, int ldm,
              double* sigma, double* V, int64_t ldv, cudaStream_t s);
void build_z(const double* G, int ldg, const int* idx, const double* sig, int r, double* Z,
             cudaStream_t s);
void build_m1(const double* W, const int* idx, const double* sig, int r, int kz, double* M1,
              int ldm, cudaStream_t s);
void build_k(const double* T, const int* idx2, int r2, const double* W, int r, const double* sig,
             const int* idx, double* Kc, cudaStream_t s);
void svd_out(const double* cols, int ldc, int r2, int r, const double* vals, const double* Vt,
             int w, const int* idx, double* sigma, double* V, int64_t ldv, double* Ps,
             cudaStream_t s);
void build_m2(const double* W, int r, const int* idx, const double* sig, const double* T,
              const int* idx2, int r2, const double* Ps, double* M2, int ldm, cudaStream_t s);
void canon_lowrank(double* VA, int64_t ldva, int n, double* Ut, int ldut, int r3, int r4,
                   cudaStream_t s);
void copy2d(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t rows, int cols,
            cudaStream_t s);
void fill(double* p, int64_t n, double v, cudaStream_t s);
}  // namespace tsk
