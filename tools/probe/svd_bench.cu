// Probe: cost/accuracy of cuSOLVER SVD options for the Nystrom factor (B = Q R, SVD of R).
#include <cstdio>
#include <cmath>
#include <vector>
#include <random>
#include <algorithm>
#include <cuda_runtime.h>
#include <cublas_v2.h>
#include <cusolverDn.h>

#define CK(x) do { auto e = (x); if ((int)e) { printf("err %d at %s:%d\n", (int)e, __FILE__, __LINE__); exit(1);} } while (0)

int main() {
  cusolverDnHandle_t h; CK(cusolverDnCreate(&h));
  cublasHandle_t bl; CK(cublasCreate(&bl));
  cusolverDnParams_t params; CK(cusolverDnCreateParams(&params));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sizes[] = {100, 300, 500, 1000};
  for (int n : sizes) {
    // R = Qa diag(s) Qb^T, s graded 1 .. 1e-8 with a tail cluster near 1e-8
    std::mt19937_64 rng(n);
    std::normal_distribution<double> N(0, 1);
    std::vector<double> A(n * n), Bm(n * n), s(n);
    for (int i = 0; i < n; ++i) s[i] = (i < n / 2) ? pow(10.0, -8.0 * i / (n / 2)) : 1e-8 * (1.0 + 1e-3 * i);
    std::sort(s.begin(), s.end(), std::greater<double>());
    for (auto& x : A) x = N(rng);
    for (auto& x : Bm) x = N(rng);
    double *dA, *dB, *dR, *dS, *dU, *dV, *dwork, *tau; int* info;
    CK(cudaMalloc(&dA, 8 * n * n)); CK(cudaMalloc(&dB, 8 * n * n)); CK(cudaMalloc(&dR, 8 * n * n));
    CK(cudaMalloc(&dS, 8 * n)); CK(cudaMalloc(&dU, 8 * n * n)); CK(cudaMalloc(&dV, 8 * n * n)); CK(cudaMalloc(&tau, 8 * n));
    CK(cudaMalloc(&info, 4));
    cudaMemcpy(dA, A.data(), 8 * n * n, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, Bm.data(), 8 * n * n, cudaMemcpyHostToDevice);
    int lw = 0; CK(cusolverDnDgeqrf_bufferSize(h, n, n, dA, n, &lw)); CK(cudaMalloc(&dwork, 8 * std::max(lw, 1 << 24)));
    CK(cusolverDnDgeqrf(h, n, n, dA, n, tau, dwork, lw, info)); CK(cusolverDnDorgqr(h, n, n, n, dA, n, tau, dwork, lw, info));
    CK(cusolverDnDgeqrf(h, n, n, dB, n, tau, dwork, lw, info)); CK(cusolverDnDorgqr(h, n, n, n, dB, n, tau, dwork, lw, info));
    // R0 = Qa diag(s) Qb^T
    std::vector<double> qa(n * n); cudaMemcpy(qa.data(), dA, 8 * n * n, cudaMemcpyDeviceToHost);
    for (int j = 0; j < n; ++j) for (int i = 0; i < n; ++i) qa[j * n + i] *= s[j];
    cudaMemcpy(dU, qa.data(), 8 * n * n, cudaMemcpyHostToDevice);
    double one = 1, zero = 0;
    CK(cublasDgemm(bl, CUBLAS_OP_N, CUBLAS_OP_T, n, n, n, &one, dU, n, dB, n, &zero, dR, n));
    std::vector<double> R0(n * n); cudaMemcpy(R0.data(), dR, 8 * n * n, cudaMemcpyDeviceToHost);
    auto reset = [&]() { cudaMemcpy(dR, R0.data(), 8 * n * n, cudaMemcpyHostToDevice); };
    auto report = [&](const char* name, float ms) {
      std::vector<double> hs(n); cudaMemcpy(hs.data(), dS, 8 * n, cudaMemcpyDeviceToHost);
      double worst_top = 0, worst_all = 0;
      for (int i = 0; i < n; ++i) {
        double r = fabs(hs[i] - s[i]) / s[i];
        if (s[i] > 1e-4) worst_top = std::max(worst_top, r);
        worst_all = std::max(worst_all, fabs(hs[i] - s[i]) / s[0]);
      }
      printf("n=%4d %-28s %9.3f ms  relerr(s>1e-4)=%.2e  abs/s1=%.2e  s_min=%.3e\n", n, name, ms, worst_top, worst_all, hs[n - 1]);
    };
    for (double tol : {0.0, 1e-10}) {
      gesvdjInfo_t gi; CK(cusolverDnCreateGesvdjInfo(&gi));
      if (tol > 0) { CK(cusolverDnXgesvdjSetTolerance(gi, tol)); }
      int lwj = 0; CK(cusolverDnDgesvdj_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, 0, n, n, dR, n, dS, dU, n, dV, n, &lwj, gi));
      for (int rep = 0; rep < 2; ++rep) {
        reset();
        cudaEventRecord(e0);
        CK(cusolverDnDgesvdj(h, CUSOLVER_EIG_MODE_VECTOR, 0, n, n, dR, n, dS, dU, n, dV, n, dwork, lwj, info, gi));
        cudaEventRecord(e1); cudaEventSynchronize(e1);
      }
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      int sweeps = 0; double resid = 0; cusolverDnXgesvdjGetSweeps(h, gi, &sweeps); cusolverDnXgesvdjGetResidual(h, gi, &resid);
      char nm[64]; snprintf(nm, 64, "gesvdj tol=%g sweeps=%d", tol, sweeps);
      report(nm, ms);
      cusolverDnDestroyGesvdjInfo(gi);
    }
    {
      int lwg = 0; CK(cusolverDnDgesvd_bufferSize(h, n, n, &lwg));
      double* rw; cudaMalloc(&rw, 8 * n);
      for (int rep = 0; rep < 2; ++rep) {
        reset();
        cudaEventRecord(e0);
        CK(cusolverDnDgesvd(h, 'S', 'S', n, n, dR, n, dS, dU, n, dV, n, dwork, lwg, rw, info));
        cudaEventRecord(e1); cudaEventSynchronize(e1);
      }
      float ms; cudaEventElapsedTime(&ms, e0, e1); report("gesvd", ms);
    }
    {
      size_t wd = 0, wh = 0;
      CK(cusolverDnXgesvdp_bufferSize(h, params, CUSOLVER_EIG_MODE_VECTOR, 1, n, n, CUDA_R_64F, dR, n, CUDA_R_64F, dS,
                                      CUDA_R_64F, dU, n, CUDA_R_64F, dV, n, CUDA_R_64F, &wd, &wh));
      void* dw; cudaMalloc(&dw, wd + 8); std::vector<char> hw(wh + 8);
      double err = 0;
      for (int rep = 0; rep < 2; ++rep) {
        reset();
        cudaEventRecord(e0);
        CK(cusolverDnXgesvdp(h, params, CUSOLVER_EIG_MODE_VECTOR, 1, n, n, CUDA_R_64F, dR, n, CUDA_R_64F, dS, CUDA_R_64F,
                             dU, n, CUDA_R_64F, dV, n, CUDA_R_64F, dw, wd, hw.data(), wh, info, &err));
        cudaEventRecord(e1); cudaEventSynchronize(e1);
      }
      float ms; cudaEventElapsedTime(&ms, e0, e1); char nm[64]; snprintf(nm, 64, "gesvdp err=%.1e", err); report(nm, ms);
      cudaFree(dw);
    }
    {
      // syevd of R^T R (squared)
      CK(cublasDgemm(bl, CUBLAS_OP_T, CUBLAS_OP_N, n, n, n, &one, dR, n, dR, n, &zero, dU, n));
      int lwe = 0; CK(cusolverDnDsyevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER, n, dU, n, dS, &lwe));
      std::vector<double> G(n * n); cudaMemcpy(G.data(), dU, 8 * n * n, cudaMemcpyDeviceToHost);
      for (int rep = 0; rep < 2; ++rep) {
        cudaMemcpy(dU, G.data(), 8 * n * n, cudaMemcpyHostToDevice);
        cudaEventRecord(e0);
        CK(cusolverDnDsyevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER, n, dU, n, dS, dwork, lwe, info));
        cudaEventRecord(e1); cudaEventSynchronize(e1);
      }
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("n=%4d %-28s %9.3f ms\n", n, "syevd(R^T R)", ms);
    }
    cudaFree(dA); cudaFree(dB); cudaFree(dR); cudaFree(dS); cudaFree(dU); cudaFree(dV); cudaFree(dwork); cudaFree(tau); cudaFree(info);
  }
  return 0;
}
