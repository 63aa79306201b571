// Dependent-chain latencies (cycles) of the FP64 operations in the Jacobi rotation (one warp).
#include <cstdio>
__global__ void lat(double* out, long long* cyc, double seed) {
  double x = seed + threadIdx.x * 1e-3, y = 1.0000001;
  long long t0, t1;
  const int N = 256;
#define CHAIN(k, expr)                          \
  __syncwarp();                                 \
  t0 = clock64();                               \
  for (int i = 0; i < N; ++i) { expr; }         \
  t1 = clock64();                               \
  if (threadIdx.x == 0) cyc[k] = (t1 - t0) / N;
  CHAIN(0, x = fma(x, y, 1e-9))
  CHAIN(1, x = x * y)
  CHAIN(2, x = x + __shfl_xor_sync(0xffffffffu, x, 1))
  CHAIN(3, x = sqrt(x) + 0.5)
  CHAIN(4, x = __drcp_rn(x) + 1.5)
  CHAIN(5, x = 1.0 / x + 1.5)
  CHAIN(6, x = rsqrt(x) + 0.5)
  CHAIN(7, x = __dsqrt_rn(x) + 0.5)
  out[threadIdx.x] = x;
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 32 * sizeof(double)); cudaMalloc(&c, 16 * sizeof(long long));
  lat<<<1, 32>>>(o, c, 1.5);
  lat<<<1, 32>>>(o, c, 1.5);
  long long h[16];
  cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  const char* n[] = {"dfma", "dmul", "shfl_xor+dadd", "sqrt+add", "__drcp_rn+add", "1/x+add", "rsqrt+add", "__dsqrt_rn+add"};
  for (int k = 0; k < 8; ++k) printf("%-16s %lld cycles\n", n[k], h[k]);
  return 0;
}
