// Probe: raw throughput of the Ozaki residue arithmetic (no memory traffic): elements/s for the
// FP64 magic-number scheme used by ngd_ozaki.cu, at several occupancies / ILP widths.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/probe/oz_conv_probe.cu -o tools/probe/oz_conv_probe
#include <cstdio>
#include <cuda_runtime.h>

constexpr double kMagic = 6755399441055744.0;
__host__ __device__ constexpr int mod_of(int j) {
  return j == 0 ? 256 : j == 1 ? 255 : j == 2 ? 253 : j == 3 ? 251 : j == 4 ? 247 : j == 5 ? 241 : j == 6 ? 239
       : j == 7 ? 233 : j == 8 ? 229 : j == 9 ? 227 : j == 10 ? 223 : j == 11 ? 217 : j == 12 ? 211
       : j == 13 ? 199 : j == 14 ? 197 : 193;
}
__constant__ double c26[16];

template <int E, int J = 0>
__device__ __forceinline__ void res(const double (&xh)[E], const double (&xl)[E], unsigned& acc) {
  if constexpr (J < 16) {
    constexpr double m = (double)mod_of(J);
    constexpr double inv = 1.0 / (double)mod_of(J);
    const double c = c26[J];
    double v[E], q[E];
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = fma(xh[e], c, xl[e]);
#pragma unroll
    for (int e = 0; e < E; ++e) q[e] = fma(v[e], inv, kMagic) - kMagic;
#pragma unroll
    for (int e = 0; e < E; ++e) acc ^= (unsigned)__double2loint(fma(-q[e], m, v[e]) + kMagic) << (e & 3);
    res<E, J + 1>(xh, xl, acc);
  }
}

template <int E>
__global__ void probe(int iters, unsigned* out) {
  unsigned acc = 0;
  double base = (double)(blockIdx.x * blockDim.x + threadIdx.x) * 1234567.0;
  for (int it = 0; it < iters; ++it) {
    double xh[E], xl[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const double x = base + (double)(it * E + e) * 7919.0;
      xh[e] = fma(x, 1.0 / 67108864.0, kMagic) - kMagic;
      xl[e] = fma(-xh[e], 67108864.0, x);
    }
    res<E>(xh, xl, acc);
  }
  if (acc == 0x12345u) out[0] = acc;
}

template <int E>
void run(int blocks_per_sm, int threads) {
  unsigned* out;
  cudaMalloc(&out, 4);
  const int grid = 148 * blocks_per_sm, iters = 2048 / E;
  probe<E><<<grid, threads>>>(iters, out);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  probe<E><<<grid, threads>>>(iters, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double elems = (double)grid * threads * iters * E;
  int regs = 0;
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, probe<E>);
  regs = fa.numRegs;
  printf("E=%d blocks/SM=%d threads=%d regs=%d: %.3f ms, %.2f Gelem/s (%.2f clk/elem/SM at 1.965 GHz) [%s]\n", E,
         blocks_per_sm, threads, regs, ms, elems / ms / 1e6, 148 * 1.965e9 / (elems / ms * 1e3),
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  double h[16];
  for (int j = 0; j < 16; ++j) {
    int c = (int)((1ull << 26) % (unsigned long long)mod_of(j));
    if (c > mod_of(j) / 2) c -= mod_of(j);
    h[j] = c;
  }
  cudaMemcpyToSymbol(c26, h, sizeof(h));
  run<4>(2, 256);
  run<4>(4, 256);
  run<4>(8, 256);
  run<8>(2, 256);
  run<8>(4, 256);
  run<8>(8, 256);
  run<16>(2, 256);
  run<16>(4, 256);
  return 0;
}
