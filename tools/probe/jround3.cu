// Round latency: one pair per warp (current) vs one pair per half-warp (two pairs per warp),
// full round body (partner load, Gram, rotation parameters, X and V updates), 10 pairs per CTA.
#include <cstdio>
#include "../../paper_2505_11638_b200/csrc/ngd_svd.cu"
namespace ngd {
void probe_before(int, cudaStream_t) {}
void probe_after(int, cudaStream_t) {}

template <int RPL>  // half-warp variant: 16 lanes per column
__device__ __forceinline__ void gram3_half(const double2 (&x)[RPL], const double2 (&y)[RPL], double& al, double& be,
                                           double& ga) {
  double a0 = 0, a1 = 0, b0 = 0, b1 = 0, g0 = 0, g1 = 0;
#pragma unroll
  for (int u = 0; u < RPL; u += 2) {
    a0 = fma(x[u].x, x[u].x, a0); a0 = fma(x[u].y, x[u].y, a0);
    b0 = fma(y[u].x, y[u].x, b0); b0 = fma(y[u].y, y[u].y, b0);
    g0 = fma(x[u].x, y[u].x, g0); g0 = fma(x[u].y, y[u].y, g0);
    if (u + 1 < RPL) {
      a1 = fma(x[u + 1].x, x[u + 1].x, a1); a1 = fma(x[u + 1].y, x[u + 1].y, a1);
      b1 = fma(y[u + 1].x, y[u + 1].x, b1); b1 = fma(y[u + 1].y, y[u + 1].y, b1);
      g1 = fma(x[u + 1].x, y[u + 1].x, g1); g1 = fma(x[u + 1].y, y[u + 1].y, g1);
    }
  }
  al = a0 + a1; be = b0 + b1; ga = g0 + g1;
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) {
    al += __shfl_xor_sync(0xffffffffu, al, o);
    be += __shfl_xor_sync(0xffffffffu, be, o);
    ga += __shfl_xor_sync(0xffffffffu, ga, o);
  }
}

template <int RPL, int HALF>
__global__ void __launch_bounds__(HALF ? 256 : 512, 1) jr(int npairs, int ldc, int rounds, long long* out, double* sink) {
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x;
  const int nq = ldc >> 1;
  for (int e = tid; e < 4 * 16 * ldc; e += blockDim.x) sm[e] = 1e-3 * ((e * 7919) % 1000) - 0.5;
  __syncthreads();
  double* X0 = sm;
  double* V0 = sm + 16 * ldc;
  double* X1 = sm + 32 * ldc;
  double* V1 = sm + 48 * ldc;
  const int lanes = HALF ? 16 : 32;
  const int pid = HALF ? (tid >> 4) : (tid >> 5);  // pair slot
  const int ln = tid & (lanes - 1);
  const bool own = pid < npairs;
  double2 xr[RPL], vr[RPL];
  auto ldc2 = [&](double2 (&r)[RPL], const double* col) {
    const double2* c2 = reinterpret_cast<const double2*>(col);
#pragma unroll
    for (int u = 0; u < RPL; ++u) { const int q = ln + lanes * u; r[u] = q < nq ? c2[q] : make_double2(0, 0); }
  };
  auto stc2 = [&](double* col, const double2 (&r)[RPL]) {
    double2* c2 = reinterpret_cast<double2*>(col);
#pragma unroll
    for (int u = 0; u < RPL; ++u) { const int q = ln + lanes * u; if (q < nq) c2[q] = r[u]; }
  };
  if (own) { ldc2(xr, X0 + pid * ldc); ldc2(vr, V0 + pid * ldc); }
  long long t0 = clock64();
  int sft = 0;
  for (int it = 0; it < rounds; ++it) {
    sft = (sft + 1 == npairs) ? 0 : sft + 1;
    if (own) {
      const int j = (pid + sft >= npairs) ? pid + sft - npairs : pid + sft;
      double2 y[RPL];
      ldc2(y, X1 + j * ldc);
      double al, be, ga;
      if (HALF) gram3_half<RPL>(xr, y, al, be, ga); else gram3<RPL>(xr, y, al, be, ga);
      double c, s;
      jacobi_cs(al, be, ga + 1e-3 * al, c, s);
      rot2<RPL>(xr, y, c, s);
      stc2(X1 + j * ldc, y);
      ldc2(y, V1 + j * ldc);
      rot2<RPL>(vr, y, c, s);
      stc2(V1 + j * ldc, y);
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) out[0] = (t1 - t0) / rounds;
  if (own) stc2(sink + pid * ldc, xr);
}
}  // namespace ngd
int main() {
  long long* o; double* sink;
  cudaMalloc(&o, 8); cudaMalloc(&sink, 1 << 21);
  const int ldc = 300;
  const size_t smem = sizeof(double) * 64 * ldc;
  cudaFuncSetAttribute(ngd::jr<5, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(ngd::jr<10, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int np : {2, 10, 16}) {
    long long c0 = 0, c1 = 0;
    for (int rep = 0; rep < 2; ++rep) {
      ngd::jr<5, 0><<<1, 512, smem>>>(np, ldc, 3000, o, sink);
      cudaMemcpy(&c0, o, 8, cudaMemcpyDeviceToHost);
      ngd::jr<10, 1><<<1, 256, smem>>>(np, ldc, 3000, o, sink);
      cudaMemcpy(&c1, o, 8, cudaMemcpyDeviceToHost);
    }
    printf("pairs %2d: warp/pair %lld cycles/round, half-warp/pair %lld cycles/round (%s)\n", np, c0, c1,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
