// Box characterisation for the FP64 roofline denominators.
// Measures: DFMA throughput, DMMA (mma.sync m8n8k4 f64) throughput, read-only HBM stream.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

template <int TILES>
__global__ void dmma_kernel(double* out, int iters) {
  double c[TILES][2];
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
#pragma unroll
  for (int t = 0; t < TILES; ++t) { c[t][0] = 0; c[t][1] = t; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < TILES; ++t) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < TILES; ++t) s += c[t][0] + c[t][1];
  if (s == 12345.678) out[0] = s;
}


// Mixed: warps with (warp & 1) == 0 issue DMMA, the others DFMA -- do the two share one pipe?
template <int TILES, int CHAINS>
__global__ void mixed_kernel(double* out, int iters_mma, int iters_fma, double a0, double b0) {
  int warp = threadIdx.x >> 5;
  double s = 0;
  if ((warp & 1) == 0) {
    double c[TILES][2];
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
#pragma unroll
    for (int t = 0; t < TILES; ++t) { c[t][0] = 0; c[t][1] = t; }
    for (int i = 0; i < iters_mma; ++i) {
#pragma unroll
      for (int t = 0; t < TILES; ++t)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
#pragma unroll
    for (int t = 0; t < TILES; ++t) s += c[t][0] + c[t][1];
  } else {
    double acc[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-3 + c;
    for (int i = 0; i < iters_fma; ++i) {
#pragma unroll
      for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a0, b0);
    }
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += acc[c];
  }
  if (s == 12345.678) out[0] = s;
}

__global__ void read_kernel(const double2* __restrict__ p, size_t n, double* out) {
  double s = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double2 v = __ldcs(p + i);
    s += v.x + v.y;
  }
  if (s == 12345.678) out[0] = s;
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  // DFMA
  for (int bpsm : {1, 2, 4}) {
    int blocks = sms * bpsm, threads = 512, iters = 20000;
    dfma_kernel<8><<<blocks, threads>>>(out, 100, 1.0000001, 1e-9);
    CK(cudaEventRecord(e0));
    for (int r = 0; r < 5; ++r) dfma_kernel<8><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 5.0 * blocks * threads * (double)iters * 8 * 2;
    printf("DFMA blocks/SM=%d: %.2f TFLOP/s\n", bpsm, flops / (ms * 1e-3) / 1e12);
  }
  // DMMA
  for (int bpsm : {1, 2, 4}) {
    int blocks = sms * bpsm, threads = 256, iters = 20000;
    dmma_kernel<8><<<blocks, threads>>>(out, 100);
    CK(cudaEventRecord(e0));
    for (int r = 0; r < 5; ++r) dmma_kernel<8><<<blocks, threads>>>(out, iters);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 5.0 * blocks * (threads / 32) * (double)iters * 8 * 512;
    printf("DMMA m8n8k4 blocks/SM=%d: %.2f TFLOP/s\n", bpsm, flops / (ms * 1e-3) / 1e12);
  }
  // sustained DMMA ~3 s
  {
    int blocks = sms * 2, threads = 256, iters = 200000;
    CK(cudaEventRecord(e0));
    for (int r = 0; r < 10; ++r) dmma_kernel<8><<<blocks, threads>>>(out, iters);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 10.0 * blocks * (threads / 32) * (double)iters * 8 * 512;
    printf("DMMA sustained (%.1f s): %.2f TFLOP/s\n", ms * 1e-3, flops / (ms * 1e-3) / 1e12);
  }
  {
    int blocks = sms * 2, threads = 512, iters = 200000;
    CK(cudaEventRecord(e0));
    for (int r = 0; r < 10; ++r) dfma_kernel<8><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 10.0 * blocks * threads * (double)iters * 8 * 2;
    printf("DFMA sustained (%.1f s): %.2f TFLOP/s\n", ms * 1e-3, flops / (ms * 1e-3) / 1e12);
  }

  // Mixed DMMA + DFMA warps in the same CTAs: if the sum exceeds the DMMA peak, the pipes are separate.
  for (int fi : {0, 5000, 10000, 20000, 40000}) {
    int blocks = sms * 2, threads = 512, im = 20000;
    mixed_kernel<8, 8><<<blocks, threads>>>(out, 100, fi ? 100 : 0, 1.0000001, 1e-9);
    CK(cudaEventRecord(e0));
    for (int r = 0; r < 5; ++r) mixed_kernel<8, 8><<<blocks, threads>>>(out, im, fi, 1.0000001, 1e-9);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double fm = 5.0 * blocks * (threads / 64) * (double)im * 8 * 512;
    double ff = 5.0 * blocks * (threads / 2) * (double)fi * 8 * 2;
    printf("MIXED dmma iters=%d dfma iters=%d: %.3f ms, DMMA %.2f + DFMA %.2f = %.2f TFLOP/s\n", im, fi, ms,
           fm / (ms * 1e-3) / 1e12, ff / (ms * 1e-3) / 1e12, (fm + ff) / (ms * 1e-3) / 1e12);
  }
  // HBM read
  size_t bytes = (size_t)8 << 30;
  double2* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 0, bytes));
  for (int bpsm : {2, 4, 8}) {
    int blocks = sms * bpsm, threads = 512;
    read_kernel<<<blocks, threads>>>(buf, bytes / 16, out);
    CK(cudaEventRecord(e0));
    for (int r = 0; r < 5; ++r) read_kernel<<<blocks, threads>>>(buf, bytes / 16, out);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("HBM read blocks/SM=%d: %.1f GB/s\n", bpsm, 5.0 * bytes / (ms * 1e-3) / 1e9);
  }
  CK(cudaDeviceSynchronize());
  printf("done\n");
  return 0;
}
