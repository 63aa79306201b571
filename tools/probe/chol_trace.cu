// Phase cycles (CTA 0, thread 0) of the cluster Cholesky.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DNGD_CHOL_TRACE tools/probe/chol_trace.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_2505_11638_b200/csrc/ngd_chol.cu"
namespace ngd {
void probe_before(int, cudaStream_t) {}
void probe_after(int, cudaStream_t) {}
}
int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 300;
  std::vector<double> g((size_t)3 * n * n), a((size_t)n * n, 0.0);
  srand(3);
  for (auto& x : g) x = rand() / (double)RAND_MAX - 0.5;
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < n; ++k) {
      double s = 0;
      for (int r = 0; r < 3 * n; ++r) s += g[(size_t)r * n + i] * g[(size_t)r * n + k];
      a[(size_t)k * n + i] = s;
    }
  double* dA; int* di;
  cudaMalloc(&dA, sizeof(double) * n * n);
  cudaMalloc(&di, 16);
  cudaMemcpy(dA, a.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice);
  ngd::chol_upper_cluster(dA, n, n, di, di + 2, 0);
  cudaDeviceSynchronize();
  unsigned long long z[8] = {0};
  cudaMemcpyToSymbol(ngd::g_ctr, z, sizeof(z));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int reps = 10;
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) {
    cudaMemcpyAsync(dA, a.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice);
  }
  cudaEventRecord(e1);
  cudaDeviceSynchronize();
  float copy_ms; cudaEventElapsedTime(&copy_ms, e0, e1);
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) {
    cudaMemcpyAsync(dA, a.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice);
    ngd::chol_upper_cluster(dA, n, n, di, di + 2, 0);
  }
  cudaEventRecord(e1);
  cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long t[8];
  cudaMemcpyFromSymbol(t, ngd::g_ctr, sizeof(t));
  int info; cudaMemcpy(&info, di, 4, cudaMemcpyDeviceToHost);
  printf("n=%d kernel %.1f us info=%d (%s)\n", n, 1e3 * (ms - copy_ms) / reps, info, cudaGetErrorString(cudaGetLastError()));
  const char* nm[] = {"factor (warp 0)", "-", "panel", "sync A", "diag update", "factor|trailing", "sync B", "total"};
  for (int k = 0; k < 8; ++k) printf("  %-18s %10.0f cycles/call\n", nm[k], (double)t[k] / reps);
  return 0;
}
