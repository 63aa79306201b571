// Round latency of the Jacobi cross round (partner load, Gram, rotation, X and V updates) in FP64
// (double2 per lane) vs FP32 (float2 per lane), 10 and 20 pairs per CTA.
#include <cstdio>
#include "../../paper_2505_11638_b200/csrc/ngd_svd.cu"
namespace ngd {
void probe_before(int, cudaStream_t) {}
void probe_after(int, cudaStream_t) {}

template <int RPL>
__device__ __forceinline__ void gram3f(const float2 (&x)[RPL], const float2 (&y)[RPL], float& al, float& be, float& ga) {
  al = be = ga = 0.f;
#pragma unroll
  for (int u = 0; u < RPL; ++u) {
    al = fmaf(x[u].x, x[u].x, al); be = fmaf(y[u].x, y[u].x, be); ga = fmaf(x[u].x, y[u].x, ga);
    al = fmaf(x[u].y, x[u].y, al); be = fmaf(y[u].y, y[u].y, be); ga = fmaf(x[u].y, y[u].y, ga);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    al += __shfl_xor_sync(0xffffffffu, al, o);
    be += __shfl_xor_sync(0xffffffffu, be, o);
    ga += __shfl_xor_sync(0xffffffffu, ga, o);
  }
}
__device__ __forceinline__ void jcs_f(float al, float be, float ga, float& c, float& s) {
  float d = be - al, g2 = 2.f * ga;
  const float ri = rsqrtf(fmaf(d, d, g2 * g2));
  const float cos2 = fabsf(d) * ri, sin2 = (d < 0.f ? -g2 : g2) * ri;
  const float hh = fmaf(0.5f, cos2, 0.5f), rh = rsqrtf(hh);
  c = hh * rh; s = 0.5f * sin2 * rh;
}

template <typename V2, int RPL, bool F32>
__global__ void __launch_bounds__(512, 1) jr(int npairs, int ldc, int rounds, long long* out, double* sink) {
  extern __shared__ __align__(16) unsigned char smraw[];
  using T = typename std::conditional<F32, float, double>::type;
  T* sm = reinterpret_cast<T*>(smraw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nq = ldc >> 1;
  for (int e = tid; e < 4 * 20 * ldc; e += blockDim.x) sm[e] = (T)(1e-3 * ((e * 7919) % 1000) - 0.5);
  __syncthreads();
  T* X1 = sm + 20 * ldc;
  T* V1 = sm + 40 * ldc;
  T* V0 = sm + 60 * ldc;
  const bool own = warp < npairs;
  V2 xr[RPL], vr[RPL];
  auto ld = [&](V2 (&r)[RPL], const T* col) {
    const V2* c2 = reinterpret_cast<const V2*>(col);
#pragma unroll
    for (int u = 0; u < RPL; ++u) { const int q = lane + 32 * u; r[u] = q < nq ? c2[q] : V2{0, 0}; }
  };
  auto st = [&](T* col, const V2 (&r)[RPL]) {
    V2* c2 = reinterpret_cast<V2*>(col);
#pragma unroll
    for (int u = 0; u < RPL; ++u) { const int q = lane + 32 * u; if (q < nq) c2[q] = r[u]; }
  };
  auto rot = [&](V2 (&x)[RPL], V2 (&y)[RPL], T c, T s) {
#pragma unroll
    for (int u = 0; u < RPL; ++u) {
      const V2 a = x[u], b = y[u];
      x[u] = V2{c * a.x - s * b.x, c * a.y - s * b.y};
      y[u] = V2{s * a.x + c * b.x, s * a.y + c * b.y};
    }
  };
  if (own) { ld(xr, sm + warp * ldc); ld(vr, V0 + warp * ldc); }
  long long t0 = clock64();
  int sft = 0;
  for (int it = 0; it < rounds; ++it) {
    sft = (sft + 1 == npairs) ? 0 : sft + 1;
    if (own) {
      const int j = (warp + sft >= npairs) ? warp + sft - npairs : warp + sft;
      V2 y[RPL];
      ld(y, X1 + j * ldc);
      T al, be, ga, c, s;
      if constexpr (F32) { gram3f<RPL>(xr, y, al, be, ga); jcs_f(al, be, ga + 1e-3f * al, c, s); }
      else { gram3<RPL>(xr, y, al, be, ga); jacobi_cs(al, be, ga + 1e-3 * al, c, s); }
      rot(xr, y, c, s);
      st(X1 + j * ldc, y);
      ld(y, V1 + j * ldc);
      rot(vr, y, c, s);
      st(V1 + j * ldc, y);
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) out[0] = (t1 - t0) / rounds;
  if (own) sink[warp] = (double)xr[0].x;
}
}  // namespace ngd
int main() {
  long long* o; double* sink;
  cudaMalloc(&o, 8); cudaMalloc(&sink, 1 << 16);
  const int ldc = 300;
  const size_t sm64 = sizeof(double) * 80 * ldc, sm32 = sizeof(float) * 80 * ldc;
  cudaFuncSetAttribute(ngd::jr<double2, 5, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm64);
  cudaFuncSetAttribute(ngd::jr<float2, 5, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm32);
  for (int np : {2, 10, 16}) {
    long long a = 0, b = 0;
    for (int rep = 0; rep < 2; ++rep) {
      ngd::jr<double2, 5, false><<<1, 512, sm64>>>(np, ldc, 3000, o, sink);
      cudaMemcpy(&a, o, 8, cudaMemcpyDeviceToHost);
      ngd::jr<float2, 5, true><<<1, 512, sm32>>>(np, ldc, 3000, o, sink);
      cudaMemcpy(&b, o, 8, cudaMemcpyDeviceToHost);
    }
    printf("pairs %2d: fp64 %lld cycles/round, fp32 %lld cycles/round (%s)\n", np, a, b, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
