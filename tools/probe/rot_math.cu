// Throughput/latency of the Jacobi rotation-parameter chain with W warps per SM.
#include <cstdio>
__device__ __forceinline__ void rot_rutis(double al, double be, double ga, double& c, double& s) {
  const double zeta = 0.5 * (be - al) * __drcp_rn(ga);
  const double az = fabs(zeta);
  const double t = (az > 1e150) ? 0.5 * __drcp_rn(zeta) : copysign(__drcp_rn(az + sqrt(fma(az, az, 1.0))), zeta);
  c = rsqrt(fma(t, t, 1.0));
  s = c * t;
}
__device__ __forceinline__ void rot_rsqrt(double al, double be, double ga, double& c, double& s) {
  const double d = be - al, g2 = 2.0 * ga;
  const double ri = rsqrt(fma(d, d, g2 * g2));
  const double cos2 = fabs(d) * ri;
  const double sin2 = copysign(g2, d) * ri;  // sign: tan(theta) has the sign of zeta = d / (2 ga)
  const double h = fma(0.5, cos2, 0.5);
  const double rh = rsqrt(h);
  c = h * rh;
  s = 0.5 * sin2 * rh;
}
template <int MODE>
__global__ void bench(double* out, long long* cyc, int iters) {
  double al = 1.0 + threadIdx.x * 1e-6, be = 2.0, ga = 0.3, acc = 0.0;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    double c, s;
    if (MODE == 0) rot_rutis(al, be, ga, c, s);
    if (MODE == 1) rot_rsqrt(al, be, ga, c, s);
    if (MODE == 2) {  // lane 0 computes, broadcast
      if ((threadIdx.x & 31) == 0) rot_rsqrt(al, be, ga, c, s);
      c = __shfl_sync(0xffffffffu, c, 0);
      s = __shfl_sync(0xffffffffu, s, 0);
    }
    ga = fma(s, 1e-3, ga) - 1e-3 * s;  // dependency on the previous iteration
    acc += c;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / iters;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 1024 * 148 * sizeof(double)); cudaMalloc(&c, 148 * sizeof(long long));
  for (int mode = 0; mode < 3; ++mode)
    for (int w : {1, 4, 8, 12, 16}) {
      long long h = 0;
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) bench<0><<<1, 32 * w>>>(o, c, 1000);
        if (mode == 1) bench<1><<<1, 32 * w>>>(o, c, 1000);
        if (mode == 2) bench<2><<<1, 32 * w>>>(o, c, 1000);
        cudaMemcpy(&h, c, sizeof(h), cudaMemcpyDeviceToHost);
      }
      printf("mode %d (%s) warps %2d: %lld cycles / rotation\n", mode,
             mode == 0 ? "rutishauser" : (mode == 1 ? "2 rsqrt" : "2 rsqrt lane0"), w, h);
    }
  return 0;
}
