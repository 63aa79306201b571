// Shared device helpers for the B200 NystromNGD inner solve (sm_100a, fp64).
//
// Data layout ("channel-points"):
//   * points are grouped in blocks of PB = 16.  Interior points carry C = d+2
//     Taylor channels (value, d gradient channels, one Laplacian channel --
//     the forward-Laplacian form of autodiff.py:621-666);
//     boundary points carry one channel (value).
//   * a layer quantity is a row-major matrix [rows][S_pad] of fp64 where
//     column = blk*PB*C + c*PB + r%PB for interior point r, channel c, and
//     column = NIB*PB*C + s for boundary point s.  Channel-major inside a
//     point block keeps every channel run 16 doubles (128 B) long and aligned.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <utility>

#ifndef NGD_PB
#define NGD_PB 16
#endif

namespace ngd {

// Programmatic dependent launch for the PCG iteration's kernel chain: each kernel waits for its
// predecessor grid (griddepcontrol.wait: completion + memory visibility) before touching memory, so
// the successor's launch overlaps the predecessor's drain instead of following its completion
// (C2: 80.6 -> 79.7 us per PCG iteration).  Every kernel of the chain waits unconditionally (before
// any early exit), which keeps the ordering transitive.  An explicit early trigger
// (griddepcontrol.launch_dependents at kernel entry, NGD_PDL_TRIGGER) measured slower (90 us per
// iteration: the waiting successor CTAs take SM slots from the predecessor's last wave).  Outside a
// PDL launch the wait is a no-op.
__device__ __forceinline__ void pdl_entry() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
#ifdef NGD_PDL_TRIGGER
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
extern int g_pdl;  // option "pdl" (default 1)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

constexpr int PB = NGD_PB;
constexpr int kThreads = 256;

// ---------------------------------------------------------------------------
// FP64 tensor-core MMA: D(8x8) += A(8x4, row) * B(4x8, col)  -> SASS DMMA.8x8x4
// Fragments (per lane, g = lane>>2, t = lane&3):
//   A: a = A[g][t];  B: b = B[t][g];  C/D: c0 = C[g][2t], c1 = C[g][2t+1]
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// deterministic warp reduction (fixed xor tree)
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// deterministic block reduction for blockDim.x == kThreads; result valid in thread 0
__device__ __forceinline__ double block_sum(double v, double* sh /*[kThreads/32]*/) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < kThreads / 32; ++i) r += sh[i];
  }
  return r;
}

// Geometry of one problem instance, passed by value to kernels.
struct Geom {
  int d;          // input dimension
  int C;          // interior channels = d + 2
  int n_int;      // interior points (real)
  int n_bnd;      // boundary points (real)
  int nib;        // interior point blocks
  int nbb;        // boundary point blocks
  int64_t s_pad;  // columns = nib*PB*C + nbb*PB
  __host__ __device__ int64_t int_cols() const { return (int64_t)nib * PB * C; }
  __host__ __device__ int n_pts_pad() const { return (nib + nbb) * PB; }
};

// column of (interior point r, channel c)
__host__ __device__ __forceinline__ int64_t col_int(int r, int c, int C) {
  return (int64_t)(r / PB) * PB * C + (int64_t)c * PB + (r % PB);
}

}  // namespace ngd
