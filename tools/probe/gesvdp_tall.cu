// Probe: cusolverDnXgesvdp on a tall p x ell matrix vs on its ell x ell R factor.
#include <cstdio>
#include <vector>
#include <random>
#include <cmath>
#include <cuda_runtime.h>
#include <cusolverDn.h>
#define CK(x) do { auto e = (x); if ((int)e) { printf("err %d at line %d\n", (int)e, __LINE__); exit(1);} } while (0)
int main() {
  cusolverDnHandle_t h; CK(cusolverDnCreate(&h));
  cusolverDnParams_t prm; CK(cusolverDnCreateParams(&prm));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (auto [m, n] : std::vector<std::pair<int,int>>{{1185, 100}, {8577, 300}, {33921, 500}}) {
    std::mt19937_64 rng(1); std::normal_distribution<double> N(0, 1);
    std::vector<double> A((size_t)m * n);
    for (size_t i = 0; i < A.size(); ++i) A[i] = N(rng) * pow(10.0, -8.0 * (double)(i / m) / n);
    double *dA, *dA0, *dS, *dU, *dV; int* info;
    CK(cudaMalloc(&dA, 8ull * m * n)); CK(cudaMalloc(&dA0, 8ull * m * n)); CK(cudaMalloc(&dS, 8 * n));
    CK(cudaMalloc(&dU, 8ull * m * n)); CK(cudaMalloc(&dV, 8ull * n * n)); CK(cudaMalloc(&info, 4));
    cudaMemcpy(dA0, A.data(), 8ull * m * n, cudaMemcpyHostToDevice);
    size_t wd = 0, wh = 0;
    CK(cusolverDnXgesvdp_bufferSize(h, prm, CUSOLVER_EIG_MODE_VECTOR, 1, m, n, CUDA_R_64F, dA, m, CUDA_R_64F, dS, CUDA_R_64F, dU, m, CUDA_R_64F, dV, n, CUDA_R_64F, &wd, &wh));
    void* dw; cudaMalloc(&dw, wd + 8); std::vector<char> hw(wh + 8);
    double err = 0;
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemcpy(dA, dA0, 8ull * m * n, cudaMemcpyDeviceToDevice);
      cudaEventRecord(e0);
      CK(cusolverDnXgesvdp(h, prm, CUSOLVER_EIG_MODE_VECTOR, 1, m, n, CUDA_R_64F, dA, m, CUDA_R_64F, dS, CUDA_R_64F, dU, m, CUDA_R_64F, dV, n, CUDA_R_64F, dw, wd, hw.data(), wh, info, &err));
      cudaEventRecord(e1); cudaEventSynchronize(e1);
    }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("gesvdp tall %d x %d: %.3f ms (err %.2e)\n", m, n, ms, err);
  }
  return 0;
}
