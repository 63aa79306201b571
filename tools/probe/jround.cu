// Cycles per Jacobi cross round (load partner column, Gram, rotation, store) vs active warps.
#include <cstdio>
#include "../../paper_2505_11638_b200/csrc/ngd_svd.cu"
namespace ngd {
void probe_before(int, cudaStream_t) {}
void probe_after(int, cudaStream_t) {}
template <int RPL, int PART>
__global__ void __launch_bounds__(512, 1) jround(int h, int ldc, int rounds, long long* out, double* sink) {
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nq = ldc >> 1;
  for (int e = tid; e < 2 * h * ldc; e += blockDim.x) sm[e] = 1e-3 * ((e * 7919) % 1000) - 0.5;
  __syncthreads();
  double* X1 = sm + h * ldc;
  double2 xr[RPL];
  if (warp < h) load_col<RPL>(xr, sm + warp * ldc, nq, lane);
  const double tol = 1e-300;
  long long t0 = clock64();
  for (int it = 0; it < rounds; ++it) {
    const int sft = it % h;
    if (warp < h) {
      const int j = (warp + sft >= h) ? warp + sft - h : warp + sft;
      double* yc = X1 + (size_t)j * ldc;
      double2 y[RPL];
      load_col<RPL>(y, yc, nq, lane);
      double al = 1, be = 2, ga = 0.1;
      if (PART >= 1) gram3<RPL>(xr, y, al, be, ga);
      double c = 1, s = 0;
      if (PART >= 2) jacobi_cs(al, be, ga + 1e-3, c, s);
      else { c = al * 1e-9 + 0.9; s = be * 1e-9 + ga * 1e-9; }
      rot2<RPL>(xr, y, c, s);
      store_col<RPL>(yc, y, nq, lane);
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) out[0] = (t1 - t0) / rounds;
  if (warp < h) store_col<RPL>(sink + warp * ldc, xr, nq, lane);
}
}  // namespace ngd
int main() {
  long long* o; double* sink;
  cudaMalloc(&o, 8); cudaMalloc(&sink, 1 << 20);
  const int ldc = 300;
  cudaFuncSetAttribute(ngd::jround<5, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(ngd::jround<5, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(ngd::jround<5, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int part = 0; part < 3; ++part)
    for (int h : {1, 2, 4, 10, 16}) {
      long long c = 0;
      for (int rep = 0; rep < 2; ++rep) {
        size_t smem = sizeof(double) * 2 * 16 * ldc;
        if (part == 0) ngd::jround<5, 0><<<1, 512, smem>>>(h, ldc, 2000, o, sink);
        if (part == 1) ngd::jround<5, 1><<<1, 512, smem>>>(h, ldc, 2000, o, sink);
        if (part == 2) ngd::jround<5, 2><<<1, 512, smem>>>(h, ldc, 2000, o, sink);
        cudaMemcpy(&c, o, 8, cudaMemcpyDeviceToHost);
      }
      printf("part %d (%s) warps %2d: %lld cycles/round (%s)\n", part,
             part == 0 ? "ld+rot+st" : (part == 1 ? "+gram" : "+jacobi_cs"), h, c, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
