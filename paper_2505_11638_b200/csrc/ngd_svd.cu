// Small dense SVD for the Nystrom factor: one-sided (Hestenes) Jacobi in a
// thread-block cluster, the matrix resident in (distributed) shared memory.
//
// sketch.py:85 takes the thin SVD of B = Y_nu C^{-1}; after B = Q R (shifted
// Cholesky-QR3) only the ell x ell SVD of R remains.  cuSOLVER's dense SVDs are
// latency-bound at these sizes (gesvdp 9.6 ms, gesvdj 32 ms at ell = 300 on
// B200, tools/probe/svd_bench.cu).  Here the ell columns of R are spread over a
// cluster of CL CTAs (CL * 200 KB of shared memory); every round of the
// round-robin (circle) ordering rotates ell/2 disjoint column pairs in parallel
// -- one warp per pair, columns reached through DSMEM when they live in
// another CTA -- followed by one cluster barrier.  One-sided Jacobi is
// backward stable with high relative accuracy for the small singular values
// (the property the Nystrom shift nu = eps ||Y||_F relies on).
// It runs on X = R^T (Drmac-Veselic preconditioning: the rows of a triangular
// factor are graded, cutting the sweep count about 2x versus R itself) and
// accumulates the rotations V, which are then R's left singular vectors:
// R^T V = U_X S  =>  R = V S U_X^T.
#include <cooperative_groups.h>

#include "ngd_common.cuh"
#include "ngd_kernels.h"

namespace cg = cooperative_groups;

namespace ngd {

// threads per CTA: keep the two register-resident columns (2 x RPL doubles) spill-free
template <int RPL>
constexpr int svd_threads() { return RPL <= 4 ? 1024 : (RPL <= 8 ? 512 : 256); }

// circle-method round robin on n players (n even): round r in [0, n-1), pair k in [0, n/2)
__device__ __forceinline__ void circle_pair(int n, int r, int k, int& a, int& b) {
  const int m = n - 1;
  if (k == 0) {
    a = 0;
    b = 1 + r;
  } else {
    int x = r + k;
    x = (x >= m) ? x - m : x;
    int y = r - k;
    y = (y < 0) ? y + m : y;
    a = 1 + x;
    b = 1 + y;
  }
}

template <int CL>
__device__ __forceinline__ void cluster_barrier() {
  if constexpr (CL == 1) {
    __syncthreads();
  } else {
    cg::this_cluster().sync();
  }
}

template <int CL>
__device__ __forceinline__ double* col_ptr(double* cols, int j, int m, int ldc) {
  if constexpr (CL == 1) {
    return cols + (int64_t)j * ldc;
  } else {
    return cg::this_cluster().map_shared_rank(cols, j / m) + (int64_t)(j % m) * ldc;
  }
}

// A: ell x ell column-major (lda).  Outputs: sigma (descending), U (ell x ell, ldu),
// info[0] = sweeps used (negative if not converged).
template <int CL, int RPL>
__global__ void __launch_bounds__(svd_threads<RPL>(), 1) jsvd_kernel(const double* A, int ell, int lda, double* U, int ldu,
                                                              double* sigma, double tol, int max_sweeps, int* info) {
  extern __shared__ __align__(16) double smem[];
  const int n = (ell + 2 * CL - 1) / (2 * CL) * (2 * CL);  // even, multiple of CL
  const int m = n / CL;                                     // columns per CTA
  const int ldc = ell;
  double* cols = smem;                           // [m][ldc]  X columns
  double* vcols = cols + (int64_t)m * ldc;       // [m][ldc]  accumulated rotations
  double* norms = vcols + (int64_t)m * ldc;      // [m]
  int* flags = reinterpret_cast<int*>(norms + m);  // [2]
  const int q = (CL == 1) ? 0 : (int)cg::this_cluster().block_rank();
  constexpr int kSvdThreads = svd_threads<RPL>();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = kSvdThreads / 32;

  // X = R^T (column j of X = row j of R) and V = I, both [m][ldc] per CTA
  for (int64_t e = tid; e < (int64_t)m * ldc; e += kSvdThreads) {
    const int jl = (int)(e / ldc), r = (int)(e % ldc);
    const int j = q * m + jl;
    cols[e] = (j < ell) ? A[(int64_t)r * lda + j] : 0.0;
    vcols[e] = (j == r) ? 1.0 : 0.0;
  }
  if (tid < 2) flags[tid] = 0;
  cluster_barrier<CL>();

  int sweep = 0;
  bool converged = false;
  for (; sweep < max_sweeps && !converged; ++sweep) {
    const int par = sweep & 1;
    for (int rd = 0; rd < n - 1; ++rd) {
      // pairs k = q, q + CL, ... of this round; one warp per pair
      for (int k = q + CL * warp; k < n / 2; k += CL * NW) {
        int i, j;
        circle_pair(n, rd, k, i, j);
        double* ci = col_ptr<CL>(cols, i, m, ldc);
        double* cj = col_ptr<CL>(cols, j, m, ldc);
        double* vi = col_ptr<CL>(vcols, i, m, ldc);
        double* vj = col_ptr<CL>(vcols, j, m, ldc);
        // both columns and their rotation-accumulator columns into registers up front
        // (all loads in flight at once: one (D)SMEM latency per pair)
        double x[RPL], y[RPL], pv[RPL], qv[RPL];
#pragma unroll
        for (int u = 0; u < RPL; ++u) {
          const int r = lane + 32 * u;
          const bool in = r < ell;
          x[u] = in ? ci[r] : 0.0;
          y[u] = in ? cj[r] : 0.0;
          pv[u] = in ? vi[r] : 0.0;
          qv[u] = in ? vj[r] : 0.0;
        }
        double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
        for (int u = 0; u < RPL; ++u) {
          al = fma(x[u], x[u], al);
          be = fma(y[u], y[u], be);
          ga = fma(x[u], y[u], ga);
        }
        al = warp_sum(al);
        be = warp_sum(be);
        ga = warp_sum(ga);
        // rotate iff |ga| > tol sqrt(al be)  (squared form: no square roots on the test)
        if (ga != 0.0 && ga * ga > tol * tol * al * be) {
          const double zeta = (be - al) / (2.0 * ga);
          const double az = fabs(zeta);
          const double t = (az > 1e150) ? 0.5 / zeta : copysign(1.0 / (az + sqrt(fma(az, az, 1.0))), zeta);
          const double c = rsqrt(fma(t, t, 1.0)), s = c * t;
#pragma unroll
          for (int u = 0; u < RPL; ++u) {
            const int r = lane + 32 * u;
            if (r < ell) {
              ci[r] = c * x[u] - s * y[u];
              cj[r] = s * x[u] + c * y[u];
              vi[r] = c * pv[u] - s * qv[u];
              vj[r] = s * pv[u] + c * qv[u];
            }
          }
          if (lane == 0) flags[par] = 1;
        }
      }
      cluster_barrier<CL>();
    }
    // cluster-wide convergence test (flags double-buffered by sweep parity)
    int any = 0;
    if constexpr (CL == 1) {
      any = flags[par];
    } else {
      for (int o = 0; o < CL; ++o) any |= cg::this_cluster().map_shared_rank(flags, o)[par];
    }
    converged = (any == 0);
    if (tid == 0) flags[par ^ 1] = 0;
    cluster_barrier<CL>();
  }
  // norms of own columns
  for (int jl = warp; jl < m; jl += NW) {
    const double* c = cols + (int64_t)jl * ldc;
    double s = 0.0;
    for (int r = lane; r < ell; r += 32) s = fma(c[r], c[r], s);
    s = warp_sum(s);
    if (lane == 0) norms[jl] = sqrt(s);
  }
  cluster_barrier<CL>();
  // rank of each own column among all n (descending sigma, ties by index), write sigma and U
  for (int jl = warp; jl < m; jl += NW) {
    const int j = q * m + jl;
    const double sj = norms[jl];
    int rank = 0;
    for (int o = lane; o < n; o += 32) {
      const double so = (CL == 1) ? norms[o] : cg::this_cluster().map_shared_rank(norms, o / m)[o % m];
      rank += (so > sj || (so == sj && o < j)) ? 1 : 0;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) rank += __shfl_xor_sync(0xffffffffu, rank, off);
    if (rank < ell) {
      if (lane == 0) sigma[rank] = sj;
      const double* v = vcols + (int64_t)jl * ldc;
      for (int r = lane; r < ell; r += 32) U[(int64_t)rank * ldu + r] = v[r];
    }
  }
  if (q == 0 && tid == 0) info[0] = converged ? sweep : -sweep;
  cluster_barrier<CL>();  // keep shared memory alive until every CTA has finished reading it
}

static size_t jsvd_smem(int ell, int cl) {
  const int n = (ell + 2 * cl - 1) / (2 * cl) * (2 * cl);
  const int m = n / cl;
  return sizeof(double) * (2 * (size_t)m * ell + m) + 2 * sizeof(int) + 16;
}

int jsvd_cluster_size(int ell) {
  for (int cl : {1, 2, 4, 8, 16})
    if (jsvd_smem(ell, cl) <= 200 * 1024) return cl;
  return 0;  // too large: caller falls back
}

template <int CL, int RPL>
static cudaError_t launch_jsvd_r(const double* A, int ell, int lda, double* U, int ldu, double* sigma, double tol,
                                 int max_sweeps, int* info, cudaStream_t st) {
  const size_t smem = jsvd_smem(ell, CL);
  auto kern = jsvd_kernel<CL, RPL>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (CL > 8) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CL, 1, 1);
  cfg.blockDim = dim3(svd_threads<RPL>(), 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  probe_before(K_SVD, st);
  e = cudaLaunchKernelEx(&cfg, kern, A, ell, lda, U, ldu, sigma, tol, max_sweeps, info);
  probe_after(K_SVD, st);
  return e;
}

template <int CL>
static cudaError_t launch_jsvd(const double* A, int ell, int lda, double* U, int ldu, double* sigma, double tol,
                               int max_sweeps, int* info, cudaStream_t st) {
  const int rpl = (ell + 31) / 32;
  if (rpl <= 4) return launch_jsvd_r<CL, 4>(A, ell, lda, U, ldu, sigma, tol, max_sweeps, info, st);
  if (rpl <= 8) return launch_jsvd_r<CL, 8>(A, ell, lda, U, ldu, sigma, tol, max_sweeps, info, st);
  if (rpl <= 12) return launch_jsvd_r<CL, 12>(A, ell, lda, U, ldu, sigma, tol, max_sweeps, info, st);
  if (rpl <= 16) return launch_jsvd_r<CL, 16>(A, ell, lda, U, ldu, sigma, tol, max_sweeps, info, st);
  if (rpl <= 24) return launch_jsvd_r<CL, 24>(A, ell, lda, U, ldu, sigma, tol, max_sweeps, info, st);
  return cudaErrorInvalidValue;
}

cudaError_t jacobi_svd(const double* A, int ell, int lda, double* U, int ldu, double* sigma, int* info,
                       cudaStream_t st) {
  // rotate only when |a_i.a_j| > ell * eps * |a_i||a_j|: tighter thresholds only chase dot-product rounding noise
  const double tol = 2.220446049250313e-16 * (double)ell;
  const int max_sweeps = 40;
  switch (jsvd_cluster_size(ell)) {
    case 1: return launch_jsvd<1>(A, ell, lda, U, ldu, sigma, tol, max_sweeps, info, st);
    case 2: return launch_jsvd<2>(A, ell, lda, U, ldu, sigma, tol, max_sweeps, info, st);
    case 4: return launch_jsvd<4>(A, ell, lda, U, ldu, sigma, tol, max_sweeps, info, st);
    case 8: return launch_jsvd<8>(A, ell, lda, U, ldu, sigma, tol, max_sweeps, info, st);
    case 16: return launch_jsvd<16>(A, ell, lda, U, ldu, sigma, tol, max_sweeps, info, st);
    default: return cudaErrorInvalidValue;
  }
}


// ---------------------------------------------------------------------------
// Block-exchange variant: every rotation touches only LOCAL shared memory.
// The n (padded) columns form 2*CL blocks of h columns; CTA k holds two blocks.
// A sweep = one round-robin tournament of the 2*CL blocks (circle method):
//   super-round 0 also rotates all pairs inside each block (h-1 local rounds),
//   every super-round rotates all cross pairs of the CTA's two blocks (h local
//   rounds of h disjoint pairs), then blocks move to the CTA that pairs them in
//   the next super-round (bulk DSMEM copies into a second buffer, one cluster
//   barrier).  Rounds per sweep ~ n (as for element-wise Jacobi) but each costs a
//   __syncthreads, not a cluster barrier + element-wise remote traffic.
// Columns: X = R^T and V = I, as in jsvd_kernel.
// DSMEM block copy with 8 remote loads in flight per thread (remote latency ~200+ cycles)
__device__ __forceinline__ void copy_remote(double2* dst, const double2* src, size_t n, int tid, int T) {
  size_t e = tid;
  for (; e + 7 * (size_t)T < n; e += 8 * (size_t)T) {
    double2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = src[e + u * (size_t)T];
#pragma unroll
    for (int u = 0; u < 8; ++u) dst[e + u * (size_t)T] = v[u];
  }
  for (; e < n; e += T) dst[e] = src[e];
}

template <int RPL>  // RPL = double2 per lane per column (rows 2q, 2q+1 for q = lane + 32 u)
__device__ __forceinline__ bool rotate_pair(double* ci, double* cj, double* vi, double* vj, int ldc, int lane,
                                            double tol) {
  const int nq = ldc >> 1;  // double2 per column (ldc even; padding rows are zero)
  const double2* ci2 = reinterpret_cast<const double2*>(ci);
  const double2* cj2 = reinterpret_cast<const double2*>(cj);
  double2 x[RPL], y[RPL];
#pragma unroll
  for (int u = 0; u < RPL; ++u) {
    const int q = lane + 32 * u;
    const bool in = q < nq;
    x[u] = in ? ci2[q] : make_double2(0.0, 0.0);
    y[u] = in ? cj2[q] : make_double2(0.0, 0.0);
  }
  double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
  for (int u = 0; u < RPL; ++u) {
    al = fma(x[u].x, x[u].x, al);
    al = fma(x[u].y, x[u].y, al);
    be = fma(y[u].x, y[u].x, be);
    be = fma(y[u].y, y[u].y, be);
    ga = fma(x[u].x, y[u].x, ga);
    ga = fma(x[u].y, y[u].y, ga);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {  // three interleaved butterfly reductions
    al += __shfl_xor_sync(0xffffffffu, al, o);
    be += __shfl_xor_sync(0xffffffffu, be, o);
    ga += __shfl_xor_sync(0xffffffffu, ga, o);
  }
  if (!(ga != 0.0 && ga * ga > tol * tol * al * be)) return false;
  // rotation parameters (Rutishauser); __drcp_rn keeps the divide off the slow path
  const double zeta = 0.5 * (be - al) * __drcp_rn(ga);
  const double az = fabs(zeta);
  const double t = (az > 1e150) ? 0.5 * __drcp_rn(zeta) : copysign(__drcp_rn(az + sqrt(fma(az, az, 1.0))), zeta);
  const double c = rsqrt(fma(t, t, 1.0)), s = c * t;
  double2* wi = reinterpret_cast<double2*>(ci);
  double2* wj = reinterpret_cast<double2*>(cj);
  double2* pi = reinterpret_cast<double2*>(vi);
  double2* pj = reinterpret_cast<double2*>(vj);
#pragma unroll
  for (int u = 0; u < RPL; ++u) {
    const int q = lane + 32 * u;
    if (q < nq) {
      wi[q] = make_double2(c * x[u].x - s * y[u].x, c * x[u].y - s * y[u].y);
      wj[q] = make_double2(s * x[u].x + c * y[u].x, s * x[u].y + c * y[u].y);
      const double2 pv = pi[q], qv = pj[q];
      pi[q] = make_double2(c * pv.x - s * qv.x, c * pv.y - s * qv.y);
      pj[q] = make_double2(s * pv.x + c * qv.x, s * pv.y + c * qv.y);
    }
  }
  return true;
}

// 16 warps: one column pair per warp and local round (h <= 16)
constexpr int kBlockSvdThreads = 512;

template <int RPL>
__global__ void __launch_bounds__(kBlockSvdThreads, 1) jsvd_block_kernel(const double* A, int ell, int lda,
                                                                           double* U, int ldu, double* sigma,
                                                                           double tol, int max_sweeps, int h,
                                                                           int* info) {
  extern __shared__ __align__(16) double smem[];
  constexpr int T = kBlockSvdThreads;
  constexpr int NW = T / 32;
  cg::cluster_group cl = cg::this_cluster();
  const int CL = (int)cl.num_blocks();
  const int k = (int)cl.block_rank();
  const int nb = 2 * CL;  // blocks
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ldc = ell + (ell & 1);             // even column stride: 16-B aligned double2 columns
  const size_t slot_sz = (size_t)h * ldc;  // one block of X (or V)
  // buf[phase][slot][0 = X, 1 = V][h][ell]
  auto bufp = [&](double* base, int phase, int slot, int which) {
    return base + ((size_t)(phase * 2 + slot) * 2 + which) * slot_sz;
  };
  double* norms = smem + 8 * slot_sz;          // [2][h]
  int* flags = reinterpret_cast<int*>(norms + 2 * h);  // [2]
  int phase = 0;
  int blk[2];
  circle_pair(nb, 0, k, blk[0], blk[1]);
  for (int sl = 0; sl < 2; ++sl) {
    double* X = bufp(smem, 0, sl, 0);
    double* V = bufp(smem, 0, sl, 1);
    for (int64_t e = tid; e < (int64_t)slot_sz; e += T) {
      const int i = (int)(e / ldc), r = (int)(e % ldc);
      const int j = blk[sl] * h + i;  // global column id
      X[e] = (j < ell && r < ell) ? A[(int64_t)r * lda + j] : 0.0;
      V[e] = (j == r && r < ell) ? 1.0 : 0.0;
    }
  }
  if (tid < 2) flags[tid] = 0;
  cl.sync();
  int sweep = 0;
  bool converged = false;
  for (; sweep < max_sweeps && !converged; ++sweep) {
    const int par = sweep & 1;
    bool rotated = false;
    for (int r = 0; r < nb - 1; ++r) {
      double* X0 = bufp(smem, phase, 0, 0);
      double* V0 = bufp(smem, phase, 0, 1);
      double* X1 = bufp(smem, phase, 1, 0);
      double* V1 = bufp(smem, phase, 1, 1);
      if (r == 0) {  // pairs inside each of the two blocks (circle method on h columns)
        for (int rr = 0; rr < h - 1; ++rr) {
          for (int q = warp; q < h; q += NW) {  // h/2 pairs per block, two blocks
            const int sl = q / (h / 2), kk = q % (h / 2);
            int i, j;
            circle_pair(h, rr, kk, i, j);
            double* X = sl ? X1 : X0;
            double* V = sl ? V1 : V0;
            rotated |= rotate_pair<RPL>(X + (size_t)i * ldc, X + (size_t)j * ldc, V + (size_t)i * ldc,
                                        V + (size_t)j * ldc, ldc, lane, tol);
          }
          __syncthreads();
        }
      }
      // cross pairs of the two blocks: h rounds of h disjoint pairs
      for (int sft = 0; sft < h; ++sft) {
        for (int i = warp; i < h; i += NW) {
          const int j = (i + sft >= h) ? i + sft - h : i + sft;
          rotated |= rotate_pair<RPL>(X0 + (size_t)i * ldc, X1 + (size_t)j * ldc, V0 + (size_t)i * ldc,
                                      V1 + (size_t)j * ldc, ldc, lane, tol);
        }
        __syncthreads();
      }
      if (r == nb - 2) break;  // sweep ends; the exchange to round 0 happens after the convergence test
      cl.sync();  // every CTA has finished rotating its blocks before anyone pulls them
      // move blocks to their owners of super-round r+1 (pull from remote current buffers)
      int want[2];
      circle_pair(nb, r + 1, k, want[0], want[1]);
      for (int sl = 0; sl < 2; ++sl) {
        int src_cta = 0, src_slot = 0;
        for (int k2 = 0; k2 < CL; ++k2) {
          int a, b;
          circle_pair(nb, r, k2, a, b);
          if (a == want[sl]) { src_cta = k2; src_slot = 0; }
          if (b == want[sl]) { src_cta = k2; src_slot = 1; }
        }
        const double2* srcx = reinterpret_cast<const double2*>(cl.map_shared_rank(bufp(smem, phase, src_slot, 0), src_cta));
        double2* dst = reinterpret_cast<double2*>(bufp(smem, phase ^ 1, sl, 0));
        copy_remote(dst, srcx, slot_sz, tid, T);  // X and V blocks are contiguous: 2*slot_sz doubles
      }
      cl.sync();
      phase ^= 1;
      blk[0] = want[0];
      blk[1] = want[1];
    }
    if (rotated && lane == 0) flags[par] = 1;
    cl.sync();
    int any = 0;
    for (int o = 0; o < CL; ++o) any |= cl.map_shared_rank(flags, o)[par];
    converged = (any == 0);
    if (tid == 0) flags[par ^ 1] = 0;
    if (!converged) {  // back to the round-0 placement
      int want[2];
      circle_pair(nb, 0, k, want[0], want[1]);
      for (int sl = 0; sl < 2; ++sl) {
        int src_cta = 0, src_slot = 0;
        for (int k2 = 0; k2 < CL; ++k2) {
          int a, b;
          circle_pair(nb, nb - 2, k2, a, b);
          if (a == want[sl]) { src_cta = k2; src_slot = 0; }
          if (b == want[sl]) { src_cta = k2; src_slot = 1; }
        }
        const double2* srcx = reinterpret_cast<const double2*>(cl.map_shared_rank(bufp(smem, phase, src_slot, 0), src_cta));
        double2* dst = reinterpret_cast<double2*>(bufp(smem, phase ^ 1, sl, 0));
        copy_remote(dst, srcx, slot_sz, tid, T);
      }
      blk[0] = want[0];
      blk[1] = want[1];
      phase ^= 1;
    }
    cl.sync();
  }
  // norms of the held columns, ranks over the cluster, outputs
  for (int q = warp; q < 2 * h; q += NW) {
    const double* c = bufp(smem, phase, q / h, 0) + (size_t)(q % h) * ldc;
    double sacc = 0.0;
    for (int r = lane; r < ell; r += 32) sacc = fma(c[r], c[r], sacc);
    sacc = warp_sum(sacc);
    if (lane == 0) norms[q] = sqrt(sacc);
  }
  // publish which blocks this CTA holds (flags area reused as ints after the loop)
  __shared__ int held[2];
  if (tid == 0) {
    held[0] = blk[0];
    held[1] = blk[1];
  }
  cl.sync();
  for (int q = warp; q < 2 * h; q += NW) {
    const int gid = blk[q / h] * h + (q % h);
    const double sj = norms[q];
    int rank = 0;
    for (int o = lane; o < 2 * h * CL; o += 32) {
      const int octa = o / (2 * h), oq = o % (2 * h);
      const double so = cl.map_shared_rank(norms, octa)[oq];
      const int ogid = cl.map_shared_rank(held, octa)[oq / h] * h + (oq % h);
      rank += (so > sj || (so == sj && ogid < gid)) ? 1 : 0;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) rank += __shfl_xor_sync(0xffffffffu, rank, off);
    if (rank < ell) {
      if (lane == 0) sigma[rank] = sj;
      const double* v = bufp(smem, phase, q / h, 1) + (size_t)(q % h) * ldc;
      for (int r = lane; r < ell; r += 32) U[(int64_t)rank * ldu + r] = v[r];
    }
  }
  if (k == 0 && tid == 0) info[0] = converged ? sweep : -sweep;
  cl.sync();
}

// cluster size / block size for the block-exchange Jacobi: h <= 16 columns per block
// (one pair per warp and round), 8 blocks of X/V per CTA within 200 KB.
static bool jsvd_block_plan(int ell, int& cl, int& h) {
  for (int c : {2, 4, 8, 16}) {
    int hh = (ell + 2 * c - 1) / (2 * c);
    hh += hh & 1;  // even (circle method inside a block)
    if (hh > 16 && c < 16) continue;
    if (sizeof(double) * (8 * (size_t)hh * (ell + (ell & 1)) + 2 * hh) + 64 > 200 * 1024) continue;
    cl = c;
    h = hh;
    return true;
  }
  return false;
}

int jsvd_block_supported(int ell) {
  int c, h;
  return jsvd_block_plan(ell, c, h) ? c : 0;
}

template <int RPL>
static cudaError_t launch_jsvd_block_r(const double* A, int ell, int lda, double* U, int ldu, double* sigma,
                                       double tol, int max_sweeps, int cl, int h, int* info, cudaStream_t st) {
  const size_t smem = sizeof(double) * (8 * (size_t)h * (ell + (ell & 1)) + 2 * h) + 64;
  auto kern = jsvd_block_kernel<RPL>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (cl > 8) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cl, 1, 1);
  cfg.blockDim = dim3(kBlockSvdThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  probe_before(K_SVD, st);
  e = cudaLaunchKernelEx(&cfg, kern, A, ell, lda, U, ldu, sigma, tol, max_sweeps, h, info);
  probe_after(K_SVD, st);
  return e;
}

cudaError_t jacobi_svd_block(const double* A, int ell, int lda, double* U, int ldu, double* sigma, int* info,
                             cudaStream_t st) {
  int cl, h;
  if (!jsvd_block_plan(ell, cl, h)) return cudaErrorInvalidValue;
  const double tol = 2.220446049250313e-16 * (double)ell;
  const int max_sweeps = 40;
  const int rpl = (ell + 63) / 64;  // double2 per lane
  switch (rpl) {
    case 1: return launch_jsvd_block_r<1>(A, ell, lda, U, ldu, sigma, tol, max_sweeps, cl, h, info, st);
    case 2: return launch_jsvd_block_r<2>(A, ell, lda, U, ldu, sigma, tol, max_sweeps, cl, h, info, st);
    case 3: return launch_jsvd_block_r<3>(A, ell, lda, U, ldu, sigma, tol, max_sweeps, cl, h, info, st);
    case 4: return launch_jsvd_block_r<4>(A, ell, lda, U, ldu, sigma, tol, max_sweeps, cl, h, info, st);
    case 5: return launch_jsvd_block_r<5>(A, ell, lda, U, ldu, sigma, tol, max_sweeps, cl, h, info, st);
    case 6: return launch_jsvd_block_r<6>(A, ell, lda, U, ldu, sigma, tol, max_sweeps, cl, h, info, st);
    case 7: return launch_jsvd_block_r<7>(A, ell, lda, U, ldu, sigma, tol, max_sweeps, cl, h, info, st);
    case 8: return launch_jsvd_block_r<8>(A, ell, lda, U, ldu, sigma, tol, max_sweeps, cl, h, info, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ngd
