// Latency microbenchmark of the FP64 / MUFU / shuffle operations on the Jacobi
// critical path (one warp, dependent chains, clock64).  nvcc -arch=sm_100a.
#include <cstdio>
#include <cuda_runtime.h>

#define CHAIN 256

__device__ __forceinline__ double rcp_approx(double x) {
  double y;
  asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}
__device__ __forceinline__ double rsqrt_approx(double x) {
  double y;
  asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

__global__ void lat(double* out, long long* cyc, double seed) {
  double x = seed + threadIdx.x * 1e-3, y = 1.0000001;
  long long t0, t1;
  int k = 0;
#define MEASURE(expr)                       \
  t0 = clock64();                           \
  for (int i = 0; i < CHAIN; ++i) { expr; } \
  t1 = clock64();                           \
  if (threadIdx.x == 0) cyc[k] = (t1 - t0) / CHAIN;  \
  ++k;
  MEASURE(x = fma(x, y, 1e-9))
  MEASURE(x = x + y)
  MEASURE(x = x * y)
  MEASURE(x = rcp_approx(x) + 1e-300)
  MEASURE(x = rsqrt_approx(x + 1.0))
  MEASURE(x = 1.0 / x)
  MEASURE(x = sqrt(x) + 1.0)
  MEASURE(x = x + __shfl_xor_sync(0xffffffffu, x, 1))
  MEASURE(x = fmin(x, y) + 1e-9)
  MEASURE(x = x * rsqrt(x + 1.0))
  out[threadIdx.x] = x;
}

// throughput of independent DFMA streams per warp count (cycles per warp-instruction)
__global__ void thr(double* out, long long* cyc, int iters) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double m = 1.0000001, c = 1e-9;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
    a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

// shuffle throughput: 8 independent 32-bit shuffles per iteration per lane
__global__ void shfl_thr(float* out, long long* cyc, int iters) {
  float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    a0 = __shfl_down_sync(0xffffffffu, a0, 8); a1 = __shfl_down_sync(0xffffffffu, a1, 8);
    a2 = __shfl_down_sync(0xffffffffu, a2, 8); a3 = __shfl_down_sync(0xffffffffu, a3, 8);
    a4 = __shfl_up_sync(0xffffffffu, a4, 8); a5 = __shfl_up_sync(0xffffffffu, a5, 8);
    a6 = __shfl_up_sync(0xffffffffu, a6, 8); a7 = __shfl_up_sync(0xffffffffu, a7, 8);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
// shared-memory LDS.128 + STS.128 throughput
__global__ void smem_thr(double* out, long long* cyc, int iters) {
  __shared__ double2 buf[4096 - 1024];
  for (int i = threadIdx.x; i < 3072; i += blockDim.x) buf[i] = make_double2(i, i);
  __syncthreads();
  double2 acc = make_double2(0, 0);
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    double2 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = buf[(threadIdx.x + 64 * k + i) & 2047];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc.x += v[k].x, acc.y += v[k].y;
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = acc.x + acc.y;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * 8);
  cudaMallocManaged(&cyc, 64 * 8);
  lat<<<1, 32>>>(out, cyc, 1.5);
  cudaDeviceSynchronize();
  lat<<<1, 32>>>(out, cyc, 1.5);
  cudaDeviceSynchronize();
  const char* names[] = {"DFMA", "DADD", "DMUL", "rcp.approx.f64", "rsqrt.approx.f64 (+DADD)", "1.0/x (div)",
                         "sqrt (+DADD)", "SHFL.f64+DADD", "fmin.f64+DADD", "x*rsqrt(x+1)"};
  for (int i = 0; i < 10; ++i) printf("latency %-26s %lld cycles\n", names[i], cyc[i]);
  for (int w = 1; w <= 32; w *= 2) {
    thr<<<1, 32 * w>>>(out, cyc, 4096);
    cudaDeviceSynchronize();
    printf("DFMA throughput: %2d warps/SM: %.2f cycles per warp-instruction per SMSP\n", w,
           (double)cyc[0] / (4096.0 * 8 * w) * 4);
  }
  float* fo;
  cudaMalloc(&fo, 1024 * 4);
  for (int w = 4; w <= 16; w *= 2) {
    shfl_thr<<<1, 32 * w>>>(fo, cyc, 4096);
    cudaDeviceSynchronize();
    printf("SHFL throughput: %2d warps/SM: %.2f SM-cycles per warp-SHFL\n", w, (double)cyc[0] / (4096.0 * 8 * w));
    smem_thr<<<1, 32 * w>>>(out, cyc, 4096);
    cudaDeviceSynchronize();
    printf("LDS.128 throughput: %2d warps/SM: %.2f SM-cycles per warp-LDS.128\n", w, (double)cyc[0] / (4096.0 * 8 * w));
  }
  return 0;
}
