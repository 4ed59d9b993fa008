// DMMA.8x8x4 throughput with fragments loaded from shared memory (the pattern
// of the streaming kernels): warp tile MI x NI 8x8 tiles, per k-step MI + NI
// LDS.64 and MI*NI DMMAs.  Reports TFLOP/s for several warp counts per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_smem_bench tools/dmma_smem_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

template <int MI, int NI>
__global__ void k(double* out, int iters) {
  __shared__ double s[2 * 64 * 36];
  for (int i = threadIdx.x; i < 2 * 64 * 36; i += blockDim.x) s[i] = 1.0 + i * 1e-9;
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double acc[MI][NI][2] = {};
  for (int it = 0; it < iters; ++it) {
    // the stage alternates between two buffers: the loads cannot be hoisted
    const double* xa = s + (it & 1) * 64 * 36 + g * 36 + t;
    const double* xb = s + (it & 1) * 64 * 36 + t * 36 + g;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      double a[MI], b[NI];
#pragma unroll
      for (int i = 0; i < MI; ++i) a[i] = xa[(i * 8) * 36 + kk * 4];
#pragma unroll
      for (int j = 0; j < NI; ++j) b[j] = xb[kk * 4 * 36 + j * 8 % 32];
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) dmma(acc[i][j], a[i], b[j]);
    }
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) r += acc[i][j][0] + acc[i][j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

// the gemm_nn inner loop shape: runtime k-step count per stage, 13 k-steps
template <int MI, int NI>
__global__ void k_rt(double* out, int iters, int nks) {
  __shared__ double s[2 * 64 * 36];
  for (int i = threadIdx.x; i < 2 * 64 * 36; i += blockDim.x) s[i] = 1.0 + i * 1e-9;
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double acc[MI][NI][2] = {};
  for (int it = 0; it < iters; ++it) {
    const double* xa = s + (it & 1) * 64 * 36 + g * 36 + t;
    const double* xb = s + (it & 1) * 64 * 36 + t * 36 + g;
    for (int kk = 0; kk < nks; ++kk) {
      double a[MI];
#pragma unroll
      for (int i = 0; i < MI; ++i) a[i] = xa[(i * 8) * 36 + (kk & 7) * 4];
#pragma unroll
      for (int j = 0; j < NI; ++j) {
        const double b = xb[(kk & 7) * 4 * 36 + j * 8 % 32];
#pragma unroll
        for (int i = 0; i < MI; ++i) dmma(acc[i][j], a[i], b);
      }
    }
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) r += acc[i][j][0] + acc[i][j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int MI, int NI>
void run_rt(double* out, int warps, int sms, int nks) {
  const int iters = 2000;
  k_rt<MI, NI><<<sms, warps * 32>>>(out, 10, nks);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_rt<MI, NI><<<sms, warps * 32>>>(out, iters, nks);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = (double)sms * warps * iters * nks * MI * NI * 512.0;
  printf("runtime-loop MI=%d NI=%d warps/SM=%2d nks=%d: %.2f TFLOP/s\n", MI, NI, warps, nks, flops / ms / 1e9);
}

template <int MI, int NI>
void run(double* out, int warps, int sms) {
  const int iters = 2000;
  k<MI, NI><<<sms, warps * 32>>>(out, 10);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<MI, NI><<<sms, warps * 32>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = (double)sms * warps * iters * 8 * MI * NI * 512.0;
  printf("MI=%d NI=%d warps/SM=%2d : %.2f TFLOP/s  (%s)\n", MI, NI, warps, flops / ms / 1e9,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 148 * 1024 * 8);
  run_rt<2, 10>(out, 8, sms, 13);
  run_rt<2, 10>(out, 8, sms, 7);
  run_rt<3, 7>(out, 8, sms, 7);
  for (int w : {4, 8, 12, 16}) run<2, 10>(out, w, sms);
  for (int w : {8, 16}) run<3, 7>(out, w, sms);
  for (int w : {8, 16, 24, 32}) run<2, 2>(out, w, sms);
  for (int w : {8, 16}) run<4, 4>(out, w, sms);
  for (int w : {8, 16, 28}) run<1, 7>(out, w, sms);
  return 0;
}
