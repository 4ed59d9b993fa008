// Phase timing of the Jacobi element rounds (thread 0): loads + dots, butterfly,
// rotation + update, barrier.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
//   -std=c++17 -DJAC_PROF -I include -o tools/jac_phase tools/jac_phase.cu
//   paper_1612_08709_b200/csrc/stream_kernels.cu -lcuda
#include <cstdio>
#include <random>
#include <vector>

#include "../paper_1612_08709_b200/csrc/jacobi.cu"

int main() {
  for (int n : {55, 100}) {
    // B = X^T X with X = I + 1e-6 N (near identity, like the second-pass Gram) or a graded Gram
    for (int kind = 0; kind < 2; ++kind) {
      std::mt19937_64 g(n + kind);
      std::normal_distribution<double> nd;
      std::vector<double> X(n * n), B(n * n, 0.0);
      for (int i = 0; i < n * n; ++i) X[i] = (i % (n + 1) == 0 ? 1.0 : 0.0) + (kind ? 1.0 : 1e-6) * nd(g);
      if (kind)
        for (int i = 0; i < n; ++i)
          for (int j = 0; j < n; ++j) X[i * n + j] *= std::pow(10.0, -5.0 * j / (n - 1));
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
          double s = 0;
          for (int k = 0; k < n; ++k) s += X[k * n + i] * X[k * n + j];
          B[i * n + j] = s;
        }
      double *dB, *dV, *dl;
      int* di;
      cudaMalloc(&dB, n * n * 8);
      cudaMalloc(&dV, n * n * 8);
      cudaMalloc(&dl, n * 8);
      cudaMalloc(&di, 64);
      cudaMemcpy(dB, B.data(), n * n * 8, cudaMemcpyHostToDevice);
      unsigned long long z[8] = {0};
      for (int rep = 0; rep < 2; ++rep) {
        cudaMemcpyToSymbol(tsk::g_jac_phase, z, sizeof(z));
        cudaError_t e = tsk::launch_jacobi_eig(dB, n, n, 20 * 2.2e-16, 2.2e-16, 60, dV, n, dl, di, 0);
        cudaDeviceSynchronize();
        if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
      }
      unsigned long long ph[8];
      int info[8];
      cudaMemcpyFromSymbol(ph, tsk::g_jac_phase, sizeof(ph));
      cudaMemcpy(info, di, 32, cudaMemcpyDeviceToHost);
      const double r = info[5] > 0 ? info[5] : 1;
      printf("n=%d %s sweeps=%d K=%d rounds=%d cyc/round: dots %.0f butterfly %.0f rot+upd %.0f barrier %.0f (sweep total %.0f)\n",
             n, kind ? "graded" : "near-I", info[0], info[2], info[5], ph[1] / r, ph[2] / r, ph[3] / r, ph[4] / r,
             info[4] * 16.0 / r);
      cudaFree(dB); cudaFree(dV); cudaFree(dl); cudaFree(di);
    }
  }
  return 0;
}
