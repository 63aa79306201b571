// Probe: do DMMA (mma.sync m8n8k4 f64) and DFMA share the FP64 pipe on sm_100a, or do they overlap?
// Runs DMMA-only, DFMA-only and a mix with equal pipe time of each (4 DMMA.884 = 64 cycles, 32 DFMA = 64
// cycles per SM sub-partition); shared units -> the mix takes the sum, separate pipes -> the max.
#include <cstdio>
#include <cuda_runtime.h>

template <int NM, int NF>
__global__ void mix_kernel(double* out, int iters) {
  double acc[8][2];
  double f[16];
#pragma unroll
  for (int u = 0; u < 8; ++u) acc[u][0] = acc[u][1] = 0.0;
#pragma unroll
  for (int u = 0; u < 16; ++u) f[u] = threadIdx.x * 1e-9 + u;
  const double a = 1e-3 * threadIdx.x, b = 1e-3 * (threadIdx.x + 1), m = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
#pragma unroll
      for (int u = 0; u < NM; ++u)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(acc[u][0]), "+d"(acc[u][1]) : "d"(a), "d"(b));
#pragma unroll
      for (int u = 0; u < NF; ++u) f[u % 16] = fma(f[u % 16], m, c);
    }
  }
  double s = 0;
#pragma unroll
  for (int u = 0; u < 8; ++u) s += acc[u][0] + acc[u][1];
#pragma unroll
  for (int u = 0; u < 16; ++u) s += f[u];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NM, int NF>
void run(const char* name, double* out, int sms) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int threads = 256, iters = 4096;
  for (int bps : {1, 2, 4}) {
    dim3 grid(sms * bps);
    mix_kernel<NM, NF><<<grid, threads>>>(out, 16);
    cudaEventRecord(e0);
    mix_kernel<NM, NF><<<grid, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double warps = (double)grid.x * threads / 32, n = 4.0 * iters;
    const double fl_m = warps * n * NM * 512.0, fl_f = warps * n * NF * 64.0;
    printf("%-28s CTAs/SM=%d: %.3f ms  DMMA %.2f TF/s + DFMA %.2f TF/s = %.2f TF/s\n", name, bps, ms, fl_m / ms / 1e9,
           fl_f / ms / 1e9, (fl_m + fl_f) / ms / 1e9);
  }
}

int main() {
  cudaDeviceProp prop; cudaGetDeviceProperties(&prop, 0);
  const int sms = prop.multiProcessorCount;
  double* out; cudaMalloc(&out, sizeof(double) * sms * 8 * 256);
  run<8, 0>("DMMA only (8 per round)", out, sms);
  run<0, 64>("DFMA only (64 per round)", out, sms);
  run<8, 64>("mix 8 DMMA + 64 DFMA", out, sms);
  run<8, 16>("mix 8 DMMA + 16 DFMA", out, sms);
  run<8, 8>("mix 8 DMMA + 8 DFMA", out, sms);
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
