// DMMA throughput when operands come from shared memory (the phase-B inner loop shape): 8 warps,
// 32x32 warp tiles (16 accumulator chains), per k-step 4 A + 4 B fragment loads (+ optional DMUL
// scaling of A), vs register-resident operands.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probe/dmma_smem.cu -o tools/probe/dmma_smem.bin
#include <cstdio>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int MODE>  // 0 regs, 1 smem, 2 smem + DMUL scale
__global__ void k(double* out, long long* cyc, int iters) {
  __shared__ double As[64 * 16], Bs[64 * 16], cs[16];
  for (int i = threadIdx.x; i < 64 * 16; i += blockDim.x) { As[i] = 1e-3 * i; Bs[i] = 1.0 - 1e-4 * i; }
  if (threadIdx.x < 16) cs[threadIdx.x] = 1.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) & 1, wn = warp & 1, kg = warp >> 2;
  double acc[4][4][2] = {};
  double ar[4], br[4];
  for (int q = 0; q < 4; ++q) { ar[q] = As[q]; br[q] = Bs[q]; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int kk = kg * 4 + h * 8;
      double a[4], b[4];
      if (MODE == 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) { a[q] = ar[q]; b[q] = br[q]; }
      } else {
        const double cc = MODE == 2 ? cs[kk + t] : 1.0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          a[q] = As[(wm * 32 + q * 8 + g) * 16 + (((kk + t) >> 1) ^ g) * 2 + (t & 1)];
          if (MODE == 2) a[q] *= cc;
          b[q] = Bs[(wn * 32 + q * 8 + g) * 16 + (((kk + t) >> 1) ^ g) * 2 + (t & 1)];
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int r = 0; r < 4; ++r) dmma(acc[q][r][0], acc[q][r][1], a[q], b[r]);
    }
  }
  long long t1 = clock64();
  double s = 0;
  for (int q = 0; q < 4; ++q) for (int r = 0; r < 4; ++r) s += acc[q][r][0] + acc[q][r][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
template <int MODE>
void run(const char* name, double* o, long long* c, int ctas) {
  const int iters = 1000;
  k<MODE><<<ctas, 256>>>(o, c, iters);
  k<MODE><<<ctas, 256>>>(o, c, iters);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, c, sizeof(h), cudaMemcpyDeviceToHost);
  const double dmmas = 8.0 * 2 * 16 * iters;  // per CTA
  printf("%-18s ctas %4d: %.2f cycles per DMMA per CTA (SM peak 4.0) (%s)\n", name, ctas, (double)h / dmmas,
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 1 << 22); cudaMalloc(&c, 64);
  for (int ctas : {1, 148, 296}) {
    run<0>("regs", o, c, ctas);
    run<1>("smem", o, c, ctas);
    run<2>("smem+dmul", o, c, ctas);
  }
  return 0;
}
