// DMMA.8x8x4 (FP64 mma.sync) dependent-chain latency and throughput vs independent chains per warp
// and warps per SM: how much accumulator-level parallelism a DMMA kernel needs on B200.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probe/dmma_lat.cu -o tools/probe/dmma_lat.bin
#include <cstdio>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int CH>
__global__ void k(double* out, long long* cyc, int iters) {
  double acc[CH][2];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c][0] = acc[c][1] = 0.0;
  const double a = 1e-3 * threadIdx.x, b = 1.0;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) dmma(acc[c][0], acc[c][1], a, b);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
template <int CH>
void run(int warps, double* o, long long* c) {
  const int iters = 2048;
  k<CH><<<1, 32 * warps>>>(o, c, iters);
  k<CH><<<1, 32 * warps>>>(o, c, iters);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, c, sizeof(h), cudaMemcpyDeviceToHost);
  const double per = (double)h / iters;  // cycles per iteration of CH dependent-chain steps
  printf("chains/warp %2d warps %2d: %6.1f cycles per chain step, %5.2f cycles per DMMA per SM (%.0f FMA/clk/SM)\n", CH,
         warps, per, per / (CH * warps), 256.0 * CH * warps / per);
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 1 << 20); cudaMalloc(&c, 64);
  for (int w : {1, 4, 8, 16, 24, 32}) {
    run<1>(w, o, c);
    run<4>(w, o, c);
    run<8>(w, o, c);
    run<16>(w, o, c);
  }
  return 0;
}
