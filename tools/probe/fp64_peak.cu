// Microbenchmark: FP64 vector (DFMA) vs FP64 tensor (DMMA via mma.sync f64) throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

template <int SHAPE>
__global__ void dmma_kernel(double* out, int iters) {
  // SHAPE 0: m8n8k4 ; 1: m16n8k4 ; 2: m16n8k16
  double acc[4][8];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 8; ++v) acc[u][v] = 0.0;
  double a[8], b[4];
#pragma unroll
  for (int v = 0; v < 8; ++v) a[v] = 1e-3 * (threadIdx.x + v);
#pragma unroll
  for (int v = 0; v < 4; ++v) b[v] = 1e-3 * (threadIdx.x - v);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (SHAPE == 0) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(acc[u][0]), "+d"(acc[u][1]) : "d"(a[0]), "d"(b[0]));
      } else if (SHAPE == 1) {
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                     : "+d"(acc[u][0]), "+d"(acc[u][1]), "+d"(acc[u][2]), "+d"(acc[u][3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
      } else {
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                     : "+d"(acc[u][0]), "+d"(acc[u][1]), "+d"(acc[u][2]), "+d"(acc[u][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                       "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 8; ++v) s += acc[u][v];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int dev = 0; cudaDeviceProp prop; cudaGetDeviceProperties(&prop, dev);
  int sms = prop.multiProcessorCount;
  printf("device %s sms %d clock %d kHz\n", prop.name, sms, prop.clockRate);
  double* out; cudaMalloc(&out, sizeof(double) * sms * 16 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int blocksPerSm : {4, 8}) {
    int threads = 256, iters = 4096;
    dim3 grid(sms * blocksPerSm);
    dfma_kernel<<<grid, threads>>>(out, 16);
    cudaEventRecord(e0);
    dfma_kernel<<<grid, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 16 * (double)iters * threads * grid.x;
    printf("DFMA blocks/SM=%d: %.2f TFLOP/s (%.3f ms)\n", blocksPerSm, flops / ms / 1e9, ms);
  }
  for (int shape = 0; shape < 3; ++shape) {
    for (int blocksPerSm : {2, 4, 8}) {
      int threads = 128, iters = 2048;
      dim3 grid(sms * blocksPerSm);
      auto launch = [&](int it) {
        if (shape == 0) dmma_kernel<0><<<grid, threads>>>(out, it);
        else if (shape == 1) dmma_kernel<1><<<grid, threads>>>(out, it);
        else dmma_kernel<2><<<grid, threads>>>(out, it);
      };
      launch(16);
      cudaEventRecord(e0);
      launch(iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      int m = shape == 0 ? 8 : 16, n = 8, k = shape == 2 ? 16 : 4;
      double flops = 2.0 * m * n * k * 4.0 * iters * (threads / 32) * grid.x;
      printf("DMMA m%dn%dk%d blocks/SM=%d: %.2f TFLOP/s (%.3f ms)\n", m, n, k, blocksPerSm, flops / ms / 1e9, ms);
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(err));
  return 0;
}
