// Dissect the Jacobi round latency (single warp): which part of load/rotate/store/barrier costs.
#include <cstdio>
#include "../../paper_2505_11638_b200/csrc/ngd_svd.cu"
namespace ngd {
void probe_before(int, cudaStream_t) {}
void probe_after(int, cudaStream_t) {}
template <int RPL, int V>
__global__ void __launch_bounds__(512, 1) jr(int h, int ldc, int rounds, long long* out, double* sink) {
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nq = ldc >> 1;
  for (int e = tid; e < 2 * 16 * ldc; e += blockDim.x) sm[e] = 1e-3 * ((e * 7919) % 1000) - 0.5;
  __syncthreads();
  double* X1 = sm + 16 * ldc;
  double2 xr[RPL];
  load_col<RPL>(xr, sm + warp * ldc, nq, lane);
  long long t0 = clock64();
  int sft = 0;
  for (int it = 0; it < rounds; ++it) {
    sft = (sft + 1 == h) ? 0 : sft + 1;
    if (warp < h) {
      const int j = (warp + sft >= h) ? warp + sft - h : warp + sft;
      double* yc = X1 + (size_t)j * ldc;
      double2 y[RPL];
      if (V == 5) {  // register-only: no smem traffic
#pragma unroll
        for (int u = 0; u < RPL; ++u) y[u] = make_double2(xr[u].y, xr[u].x);
      } else {
        load_col<RPL>(y, yc, nq, lane);
      }
      double c = 0.9, s = 0.1;
      if (V >= 1) {
        double al, be, ga;
        gram3<RPL>(xr, y, al, be, ga);
        c = 0.9 + 1e-20 * al; s = 0.1 + 1e-20 * (be + ga);
      }
      rot2<RPL>(xr, y, c, s);
      if (V != 3 && V != 5) store_col<RPL>(yc, y, nq, lane);
      if (V == 5) { xr[0].x += y[0].x * 1e-30; }
    }
    if (V != 4) __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) out[0] = (t1 - t0) / rounds;
  store_col<RPL>(sink + warp * ldc, xr, nq, lane);
}
}  // namespace ngd
int main() {
  long long* o; double* sink;
  cudaMalloc(&o, 8); cudaMalloc(&sink, 1 << 20);
  const int ldc = 300;
  const char* nm[] = {"ld+rot+st+bar", "+gram", "", "no store", "no barrier", "regs only (+gram, bar)"};
#define RUN(V)                                                                                   \
  cudaFuncSetAttribute(ngd::jr<5, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);  \
  for (int h : {1, 10}) {                                                                        \
    long long c = 0;                                                                             \
    for (int rep = 0; rep < 2; ++rep) {                                                          \
      ngd::jr<5, V><<<1, 512, sizeof(double) * 32 * ldc>>>(h, ldc, 4000, o, sink);              \
      cudaMemcpy(&c, o, 8, cudaMemcpyDeviceToHost);                                              \
    }                                                                                            \
    printf("%-24s warps %2d: %lld cycles/round\n", nm[V], h, c);                                 \
  }
  RUN(0) RUN(1) RUN(3) RUN(4) RUN(5)
  return 0;
}
