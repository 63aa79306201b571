// Phase split (CTA 0, thread 0) of the FP32 pre-sweep and FP64 finishing Jacobi kernels on the C2 R.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -DNGD_SVD_TRACE \
//   tools/probe/jsvd_f32trace.cu -o tools/probe/jsvd_f32trace.bin ; ./jsvd_f32trace.bin tools/probe/R_c2.bin
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../../paper_2505_11638_b200/csrc/ngd_svd.cu"
namespace ngd {
void probe_before(int, cudaStream_t) {}
void probe_after(int, cudaStream_t) {}
}
static void report(const char* name, float ms, int info) {
  unsigned long long ta[256];
  cudaMemcpyFromSymbol(ta, ngd::g_tr, sizeof(ta));
  const unsigned long long* t = ta;
  for (int c = 0; c < 16; ++c) {
    const unsigned long long* u = ta + 16 * c;
    printf("  cta %2d: barrier %.2f ms copy %.2f ms rounds %.2f ms (work %.2f)\n", c, u[0] / 1.92e6, u[1] / 1.92e6,
           (u[3] + u[4]) / 1.92e6, u[3] / 1.92e6);
  }
  const double ex = t[2] ? (double)t[2] : 1.0, rd = t[5] ? (double)t[5] : 1.0;
  printf("%s: %.3f ms sweeps %d | exchanges %llu: barrier %.0f + copy %.0f cycles | cross rounds %llu: work %.0f + "
         "syncthreads %.0f cycles | totals: exch %.2f ms rounds %.2f ms (at 1.92 GHz)\n",
         name, ms, info, t[2], t[0] / ex, t[1] / ex, t[5], t[3] / rd, t[4] / rd, (t[0] + t[1]) / 1.92e6,
         (t[3] + t[4]) / 1.92e6);
  unsigned long long z[256] = {0};
  cudaMemcpyToSymbol(ngd::g_tr, z, sizeof(z));
}
int main(int argc, char** argv) {
  FILE* f = fopen(argv[1], "rb");
  int n;
  if (fread(&n, sizeof(int), 1, f) != 1) return 1;
  std::vector<double> A((size_t)n * n);
  if (fread(A.data(), sizeof(double), A.size(), f) != A.size()) return 1;
  fclose(f);
  double *dA, *dU, *dS;
  int* dinfo;
  cudaMalloc(&dA, sizeof(double) * n * n);
  cudaMalloc(&dU, sizeof(double) * n * n);
  cudaMalloc(&dS, sizeof(double) * n);
  cudaMalloc(&dinfo, 2 * sizeof(int));
  cudaMemcpy(dA, A.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int pass = 0; pass < 2; ++pass) {
    unsigned long long z[256] = {0};
    cudaMemcpyToSymbol(ngd::g_tr, z, sizeof(z));
    float ms;
    int info;
    cudaEventRecord(e0);
    ngd::jacobi_presweep_f32(dA, n, n, dU, n, 1e-3, dinfo, 0);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpy(&info, dinfo, sizeof(int), cudaMemcpyDeviceToHost);
    if (pass) report("fp32 presweep", ms, info);
    cudaMemcpyToSymbol(ngd::g_tr, z, sizeof(z));
    cudaEventRecord(e0);
    ngd::jacobi_svd_block(dA, n, n, dU, n, dS, dinfo, 0);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpy(&info, dinfo, sizeof(int), cudaMemcpyDeviceToHost);
    if (pass) report("fp64 from I", ms, info);
  }
  printf("(%s)\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
