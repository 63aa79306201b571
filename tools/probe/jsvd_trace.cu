// Standalone timing of the block-exchange Jacobi SVD on a graded triangular matrix.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/probe/jsvd_trace.cu -o /tmp/jsvd_trace
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
  const int n = argc > 1 ? atoi(argv[1]) : 300;
  std::vector<double> A((size_t)n * n);
  srand(1);
  // upper triangular graded matrix (rows decay), column-major
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i)
      A[(size_t)j * n + i] = (i <= j) ? exp(-15.0 * i / n) * ((rand() / (double)RAND_MAX) - 0.5) : 0.0;
  double *dA, *dU, *dS;
  int* dinfo;
  cudaMalloc(&dA, sizeof(double) * n * n);
  cudaMalloc(&dU, sizeof(double) * n * n);
  cudaMalloc(&dS, sizeof(double) * n);
  cudaMalloc(&dinfo, sizeof(int));
  cudaMemcpy(dA, A.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice);
  ngd::jacobi_svd_block(dA, n, n, dU, n, dS, dinfo, 0);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  cudaError_t err = ngd::jacobi_svd_block(dA, n, n, dU, n, dS, dinfo, 0);
  cudaEventRecord(e1);
  cudaDeviceSynchronize();
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int info;
  cudaMemcpy(&info, dinfo, sizeof(int), cudaMemcpyDeviceToHost);
  printf("n=%d err=%s %.3f ms sweeps=%d\n", n, cudaGetErrorString(err), ms, info);
  return 0;
}
