// Cycles per iteration of CTA-synchronous step loops (512 threads, 1 CTA):
// what a pivoted-Cholesky / Jacobi round costs on B200 before any real work.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void warp_argmax(double& v, int& i) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int oi = __shfl_xor_sync(0xffffffffu, i, o);
    if (oi >= 0 && (i < 0 || ov > v || (ov == v && oi < i))) v = ov, i = oi;
  }
}

template <int MODE>
__global__ void k(double* out, long long* cyc, int iters) {
  __shared__ double diag[256], pcol[256];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 256; i += blockDim.x) diag[i] = 1.0 + i, pcol[i] = 0.5 + i;
  double S[8][4];
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) S[j][i] = j + i * 0.1 + tid;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    double bv = -1.0;
    int bi = -1;
    if (MODE >= 1) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double d = diag[lane + 32 * i];
        if (bi < 0 || d > bv) bv = d, bi = lane + 32 * i;
      }
      warp_argmax(bv, bi);
    }
    if (MODE >= 2 && warp == (bi & 15)) {
#pragma unroll
      for (int i = 0; i < 4; ++i) pcol[lane + 32 * i] = S[0][i] * 1e-3;
    }
    __syncthreads();
    if (MODE >= 3) {
      const double inv = MODE == 4 ? 0.5 : 1.0 / (bv + 1.0);
      double pr[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) pr[i] = pcol[lane + 32 * i] * inv;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const double f = pcol[warp + 16 * j];
#pragma unroll
        for (int i = 0; i < (MODE == 6 ? 1 : 4); ++i) S[j][i] = fma(-pr[i], f, S[j][i]);
      }
      if (MODE != 5 && lane < 8) diag[warp * 8 + lane] = S[0][0] * 1e-6 + it + bv;
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) cyc[MODE] = (t1 - t0) / iters;
  double r = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) r += S[j][i];
  out[tid] = r;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * 8);
  cudaMallocManaged(&cyc, 16 * 8);
  for (int threads : {512, 256, 128}) {
    k<0><<<1, threads>>>(out, cyc, 1000);
    k<1><<<1, threads>>>(out, cyc, 1000);
    k<2><<<1, threads>>>(out, cyc, 1000);
    k<3><<<1, threads>>>(out, cyc, 1000);
    k<4><<<1, threads>>>(out, cyc, 1000);
    k<5><<<1, threads>>>(out, cyc, 1000);
    k<6><<<1, threads>>>(out, cyc, 1000);
    cudaDeviceSynchronize();
    printf("threads=%d cycles/iter: 2 barriers %lld | +argmax %lld | +publish %lld | +update %lld | no-div %lld | no-diag-store %lld | 8 fma %lld (%s)\n", threads,
           cyc[0], cyc[1], cyc[2], cyc[3], cyc[4], cyc[5], cyc[6], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
