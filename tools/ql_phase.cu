// Phase timing of the tridiagonal-QL eigensolver (clock64 marks in the kernel, info[3] / info[4]):
// a near-identity graded Z = I + D^-1 F D^-1 (the shape of Alg. 4's second-pass Gram) of order n.
// Build (on the box): nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I include -o /tmp/ql_phase
//   tools/ql_phase.cu -Lpaper_1612_08709_b200/lib -ltssvd_b200 -Xlinker -rpath=$PWD/paper_1612_08709_b200/lib
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
namespace tsk {
cudaError_t launch_tridiag_eig(const double* B, int ldb, int n, double trunc, double* vecs, int ldv, double* vals,
                               int* info, cudaStream_t s);
}
int main() {
  for (int n : {25, 55, 92, 110, 160}) {
    std::vector<double> z((size_t)n * n);
    srand(n);
    std::vector<double> sc(n);
    for (int i = 0; i < n; ++i) sc[i] = std::pow(10.0, -5.0 * i / (n - 1));
    for (int i = 0; i < n; ++i)
      for (int j = 0; j <= i; ++j) {
        const double f = (rand() / (double)RAND_MAX - 0.5) * 2.2e-16 / (sc[i] * sc[j]) * (i != j);
        z[(size_t)i * n + j] = z[(size_t)j * n + i] = (i == j) + f;
      }
    double *dz, *dv, *dl;
    int* di;
    cudaMalloc(&dz, z.size() * 8);
    cudaMalloc(&dv, z.size() * 8);
    cudaMalloc(&dl, n * 8);
    cudaMalloc(&di, 64);
    cudaMemcpy(dz, z.data(), z.size() * 8, cudaMemcpyHostToDevice);
    int h[8];
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    tsk::launch_tridiag_eig(dz, n, n, 2.2e-16, dv, n, dl, di, 0);
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) tsk::launch_tridiag_eig(dz, n, n, 2.2e-16, dv, n, dl, di, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpy(h, di, 28, cudaMemcpyDeviceToHost);
    printf("n=%d: %.3f ms/solve; QL iterations %d, rotations %d; reduction+Q %d kcycles, QL %d kcycles (%s)\n", n,
           ms / 10, h[0], h[5], h[3], h[4], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
