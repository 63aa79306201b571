// Accuracy + timing of the block Jacobi SVD vs a reference spectrum (read from a binary file).
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../../paper_2505_11638_b200/csrc/ngd_svd.cu"
namespace ngd {
void probe_before(int, cudaStream_t) {}
void probe_after(int, cudaStream_t) {}
}
int main(int argc, char** argv) {
  // file: int n, then A (n*n col-major), then sigma_ref (n)
  FILE* f = fopen(argv[1], "rb");
  int n;
  if (fread(&n, sizeof(int), 1, f) != 1) return 1;
  std::vector<double> A((size_t)n * n), sref(n), s(n);
  if (fread(A.data(), sizeof(double), A.size(), f) != A.size()) return 1;
  if (fread(sref.data(), sizeof(double), n, f) != (size_t)n) return 1;
  fclose(f);
  double *dA, *dU, *dS;
  int* dinfo;
  cudaMalloc(&dA, sizeof(double) * n * n);
  cudaMalloc(&dU, sizeof(double) * n * n);
  cudaMalloc(&dS, sizeof(double) * n);
  cudaMalloc(&dinfo, sizeof(int));
  cudaMemcpy(dA, A.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice);
  ngd::jacobi_svd_block(dA, n, n, dU, n, dS, dinfo, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < 5; ++i) ngd::jacobi_svd_block(dA, n, n, dU, n, dS, dinfo, 0);
  cudaEventRecord(e1);
  cudaDeviceSynchronize();
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
#ifdef NGD_SVD_TRACE
  unsigned long long t[16];
  cudaMemcpyFromSymbol(t, ngd::g_tr, sizeof(t));
  printf("per exchange (%llu): sync %.0f vwait %.0f apply(incl vwait) %.0f xwait %.0f | rounds %llu work %.0f barrier %.0f\n",
         t[2], (double)t[0] / t[2], (double)t[8] / t[2], (double)t[9] / t[2], (double)t[10] / t[2], t[5],
         (double)t[3] / (t[5] ? t[5] : 1), (double)t[4] / (t[5] ? t[5] : 1));
#endif
  int info;
  cudaMemcpy(&info, dinfo, sizeof(int), cudaMemcpyDeviceToHost);
  cudaMemcpy(s.data(), dS, sizeof(double) * n, cudaMemcpyDeviceToHost);
  double e = 0, er = 0;
  for (int i = 0; i < n; ++i) {
    e = fmax(e, fabs(s[i] - sref[i]));
    er = fmax(er, fabs(s[i] - sref[i]) / sref[i]);
  }
  printf("n=%d %.3f ms/svd sweeps=%d abs_err/s1=%.2e max_rel=%.2e (%s)\n", n, ms / 5, info, e / sref[0], er,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
