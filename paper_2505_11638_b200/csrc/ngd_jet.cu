// Per-layer "jet GEMM" kernels of the factored Gramian (FP64 tensor cores, DMMA.8x8x4).
//
// The metric map theta -> F(theta) (F = Lap u on interior points, u on boundary
// points; problems.py:168-172) is linearised once per NGD step.  For layer k
// with input jets Zin_k (n_{k-1} x S) and adjoints D_k = dF/d(pre-activation jets)
// (n_k x S), the Jacobian row of point r restricted to W_k is
//     J_r[W_k] = sum_c D_k[:, (r,c)] Zin_k[:, (r,c)]^T,    J_r[b_k] = D_k[:, (r,value)]
// so   (J v)_r      = sum_k sum_c <D_k[:,(r,c)], V_k Zin_k[:,(r,c)]> + <D_k[:,(r,0)], vb_k>   (phase A)
//      (J^T c)[W_k] = D_k diag(c) Zin_k^T,  (J^T c)[b_k] = sum_{value cols} c D_k             (phase B)
// which is the reference's tape JVP/VJP (autodiff.py:90-125, gramian.py:48-53)
// restated as dense contractions.  Linearisation itself is a forward jet sweep
// (mode FWD, autodiff.py:643-659) and a reverse sweep over the jets (mode REV).
//
// CTA tile (modes FWD/REV/PHA): 64 rows x one point block (16 points x C channels),
// 8 warps = 4 (rows) x 2 (8-point groups).  Each lane owns 2 rows x 2 points x
// all C channels, so the cross-channel jet nonlinearity is lane-local.
#include "ngd_common.cuh"
#include "ngd_kernels.h"

namespace ngd {



constexpr int BM = 64, BK = 16, APAD = 4;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// forward jet nonlinearity (tanh, forward-Laplacian channels)
template <int C>
__device__ __forceinline__ void jet_act(const double (&a)[C], double (&z)[C]) {
  const double t = tanh(a[0]);
  z[0] = t;
  if constexpr (C > 1) {
    const double s1 = 1.0 - t * t;
    const double s2 = -2.0 * t * s1;
    double q = 0.0;
#pragma unroll
    for (int i = 1; i < C - 1; ++i) {
      z[i] = s1 * a[i];
      q += a[i] * a[i];
    }
    z[C - 1] = s2 * q + s1 * a[C - 1];
  }
}

// reverse of jet_act: adjoints of the outputs -> adjoints of the pre-activations
template <int C>
__device__ __forceinline__ void jet_act_rev(const double (&a)[C], const double (&g)[C], double (&o)[C]) {
  const double t = tanh(a[0]);
  const double s1 = 1.0 - t * t;
  if constexpr (C == 1) {
    o[0] = g[0] * s1;
  } else {
    const double s2 = -2.0 * t * s1;
    const double lb = g[C - 1];
    double q = 0.0, s1b = lb * a[C - 1];
#pragma unroll
    for (int i = 1; i < C - 1; ++i) {
      q += a[i] * a[i];
      s1b += g[i] * a[i];
      o[i] = g[i] * s1 + 2.0 * lb * s2 * a[i];
    }
    o[C - 1] = lb * s1;
    const double s2b = lb * q;
    const double tb = g[0] - 2.0 * t * s1b + (6.0 * t * t - 2.0) * s2b;
    o[0] = tb * s1;
  }
}

template <int C, int MODE>
__global__ void __launch_bounds__(kThreads) jet_gemm_kernel(JetArgs p) {
  constexpr int NC = PB * C;        // columns in one point block
  constexpr int BSTR = NC + 4;      // smem row stride (== 4 mod 16 doubles -> conflict-free B frags)
  constexpr int ASTR = BK + APAD;   // 20 doubles
  extern __shared__ __align__(16) double smem[];
  double* As = smem;                        // [2][BM][ASTR]
  double* Bs = smem + 2 * BM * ASTR;        // [2][BK][BSTR]

  if (p.skip && *p.skip) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp & 3, wn = warp >> 2;
  const int m0 = blockIdx.y * BM;
  const int64_t cblk = p.col0 + (int64_t)blockIdx.x * NC;

  auto load_stage = [&](int stage, int kt) {
    const int k0 = kt * BK;
    double* as = As + stage * BM * ASTR;
    double* bs = Bs + stage * BK * BSTR;
    // A: 64 x 16 doubles = 512 16-B chunks
    for (int i = tid; i < BM * BK / 2; i += kThreads) {
      const int r = i >> 3, c2 = (i & 7) * 2;
      cp_async16(as + r * ASTR + c2, p.A + (int64_t)(m0 + r) * p.Kp + k0 + c2);
    }
    // B: 16 x NC doubles
    for (int i = tid; i < BK * NC / 2; i += kThreads) {
      const int r = i / (NC / 2), c2 = (i % (NC / 2)) * 2;
      cp_async16(bs + r * BSTR + c2, p.B + (int64_t)(k0 + r) * p.s_pad + cblk + c2);
    }
    cp_async_commit();
  };

  double acc[2][C][2];
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int c = 0; c < C; ++c) acc[mi][c][0] = acc[mi][c][1] = 0.0;

  const int ktiles = p.Kp / BK;
  load_stage(0, 0);
  for (int kt = 0; kt < ktiles; ++kt) {
    if (kt + 1 < ktiles) {
      load_stage((kt + 1) & 1, kt + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* as = As + (kt & 1) * BM * ASTR + (wm * 16 + g) * ASTR + t;
    const double* bs = Bs + (kt & 1) * BK * BSTR + t * BSTR + wn * 8 + g;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      const double a0 = as[kk];
      const double a1 = as[8 * ASTR + kk];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const double b = bs[kk * BSTR + c * PB];
        dmma884(acc[0][c][0], acc[0][c][1], a0, b);
        dmma884(acc[1][c][0], acc[1][c][1], a1, b);
      }
    }
    __syncthreads();
  }

  // ---------------------------- epilogues ---------------------------------
  if constexpr (MODE == FWD || MODE == REV) {
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      const int row = m0 + wm * 16 + mi * 8 + g;
      if (row >= p.M) {
        // keep the zero padding rows [M, roundup16(M)) of a reused activation buffer clean
        if (MODE == FWD && p.z_out && row < ((p.M + 15) & ~15)) {
#pragma unroll
          for (int e = 0; e < 2; ++e)
#pragma unroll
            for (int c = 0; c < C; ++c) p.z_out[(int64_t)row * p.s_pad + cblk + wn * 8 + 2 * t + e + c * PB] = 0.0;
        }
        continue;
      }
      const double bias = (MODE == FWD && p.bias) ? p.bias[row] : 0.0;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t cbase = (int64_t)row * p.s_pad + cblk + wn * 8 + 2 * t + e;
        double v[C];
#pragma unroll
        for (int c = 0; c < C; ++c) v[c] = acc[mi][c][e];
        if constexpr (MODE == FWD) {
          v[0] += bias;
          if (p.pre_out) {
#pragma unroll
            for (int c = 0; c < C; ++c) p.pre_out[cbase + c * PB] = v[c];
          }
          if (p.z_out) {
            double z[C];
            jet_act<C>(v, z);
#pragma unroll
            for (int c = 0; c < C; ++c) p.z_out[cbase + c * PB] = z[c];
          }
        } else {
          double a[C], o[C];
#pragma unroll
          for (int c = 0; c < C; ++c) a[c] = p.dbuf[cbase + c * PB];
          jet_act_rev<C>(a, v, o);
#pragma unroll
          for (int c = 0; c < C; ++c) p.dbuf[cbase + c * PB] = o[c];
        }
      }
    }
  } else {  // PHA: per-point partial <D, V Zin>
    __shared__ double red[4][PB];
    double part[2] = {0.0, 0.0};
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      const int row = m0 + wm * 16 + mi * 8 + g;
      if (row >= p.M) continue;
      const double vb = p.bias ? p.bias[row] : 0.0;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t cbase = (int64_t)row * p.s_pad + cblk + wn * 8 + 2 * t + e;
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < C; ++c) {
          const double v = acc[mi][c][e] + (c == 0 ? vb : 0.0);
          s = fma(p.Dk[cbase + c * PB], v, s);
        }
        part[e] += s;
      }
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      part[e] += __shfl_xor_sync(0xffffffffu, part[e], 4);
      part[e] += __shfl_xor_sync(0xffffffffu, part[e], 8);
      part[e] += __shfl_xor_sync(0xffffffffu, part[e], 16);
    }
    if (g == 0) {
      red[wm][wn * 8 + 2 * t] = part[0];
      red[wm][wn * 8 + 2 * t + 1] = part[1];
    }
    __syncthreads();
    if (tid < PB) {
      const double s = (red[0][tid] + red[1][tid]) + (red[2][tid] + red[3][tid]);
      p.partA[(int64_t)blockIdx.y * p.n_pts_pad + p.pt0 + blockIdx.x * PB + tid] = s;
    }
  }
}

template <int C, int MODE>
static cudaError_t launch_jet(const JetArgs& a, int nblocks, int mtiles, cudaStream_t st) {
  constexpr int NC = PB * C;
  const size_t smem = sizeof(double) * (2 * BM * (BK + APAD) + 2 * BK * (NC + 4));
  auto kern = jet_gemm_kernel<C, MODE>;
  static bool attr_set = false;  // per-instantiation
  if (!attr_set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set = true;
  }
  if (nblocks <= 0 || mtiles <= 0) return cudaSuccess;
  probe_before(MODE == FWD ? K_FWD : (MODE == REV ? K_REV : K_PHA), st);
  kern<<<dim3(nblocks, mtiles), kThreads, smem, st>>>(a);
  probe_after(MODE == FWD ? K_FWD : (MODE == REV ? K_REV : K_PHA), st);
  return cudaGetLastError();
}

cudaError_t jet_gemm(int C, int mode, const JetArgs& a, int nblocks, int mtiles, cudaStream_t st) {
#define NGD_JET_CASE(CC)                                              \
  case CC:                                                            \
    if (mode == FWD) return launch_jet<CC, FWD>(a, nblocks, mtiles, st); \
    if (mode == REV) return launch_jet<CC, REV>(a, nblocks, mtiles, st); \
    return launch_jet<CC, PHA>(a, nblocks, mtiles, st);
  switch (C) {
    NGD_JET_CASE(1)
    NGD_JET_CASE(3)
    NGD_JET_CASE(4)
    NGD_JET_CASE(5)
    NGD_JET_CASE(6)
    NGD_JET_CASE(7)
    NGD_JET_CASE(8)
    NGD_JET_CASE(12)
    default:
      return cudaErrorInvalidValue;
  }
#undef NGD_JET_CASE
}

// ---------------------------------------------------------------------------
// Phase B: split-K  out_k = D_k diag(cc) Zin_k^T  (+ bias column), DMMA.
// Tile 64 (a) x 64 (b) x 16 (columns j); 8 warps = 4 (a) x 2 (b), warp 16 x 32.
// Partial of split g goes to part[g][off_k + a*N + b] / part[g][off_k + M*N + a],
// i.e. the flat parameter layout (model.py:41-51); a fixed-order reduction
// (reduce_splits) makes the result bitwise deterministic.
// ---------------------------------------------------------------------------

constexpr int PBM = 64, PBN = 64, PSTR = BK + 4;

__device__ __forceinline__ int point_of_col(int64_t j, int64_t int_cols, int C, int nib) {
  if (j < int_cols) {
    const int64_t blk = j / (PB * C);
    return (int)(blk * PB + (j % PB));
  }
  return nib * PB + (int)(j - int_cols);
}
__device__ __forceinline__ bool is_value_col(int64_t j, int64_t int_cols, int C) {
  return j >= int_cols || ((j % (PB * C)) < PB);
}

__global__ void __launch_bounds__(kThreads) phb_kernel(PhbArgs p) {
  __shared__ __align__(16) double As[2][PBM][PSTR];
  __shared__ __align__(16) double Bs[2][PBN][PSTR];
  __shared__ double ccs[2][BK];
  __shared__ double bias_acc[PBM];
  if (p.skip && *p.skip) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp & 3, wn = warp >> 2;
  const int n0 = blockIdx.x * PBN, m0 = blockIdx.y * PBM;
  const int split = blockIdx.z;
  const int kt0 = split * p.ktiles_per_split;
  const int kt1 = min(p.ktiles_total, kt0 + p.ktiles_per_split);
  const bool do_bias = (blockIdx.x == 0);
  if (tid < PBM) bias_acc[tid] = 0.0;

  auto load_stage = [&](int stage, int kt) {
    const int64_t j0 = (int64_t)kt * BK;
    for (int i = tid; i < PBM * BK / 2; i += kThreads) {
      const int r = i >> 3, c2 = (i & 7) * 2;
      const int row = m0 + r;
      if (row < p.M)
        cp_async16(&As[stage][r][c2], p.D + (int64_t)row * p.s_pad + j0 + c2);
      else
        *reinterpret_cast<double2*>(&As[stage][r][c2]) = make_double2(0.0, 0.0);
    }
    for (int i = tid; i < PBN * BK / 2; i += kThreads) {
      const int r = i >> 3, c2 = (i & 7) * 2;
      const int row = n0 + r;
      if (row < p.N)
        cp_async16(&Bs[stage][r][c2], p.Z + (int64_t)row * p.s_pad + j0 + c2);
      else
        *reinterpret_cast<double2*>(&Bs[stage][r][c2]) = make_double2(0.0, 0.0);
    }
    if (tid < BK) ccs[stage][tid] = p.cvec[point_of_col(j0 + tid, p.int_cols, p.C, p.nib)];
    cp_async_commit();
  };

  double acc[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  if (kt0 < kt1) load_stage(0, kt0);
  for (int kt = kt0; kt < kt1; ++kt) {
    const int st = (kt - kt0) & 1;
    if (kt + 1 < kt1) {
      load_stage(st ^ 1, kt + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      const double cc = ccs[st][kk + t];
      const double a0 = As[st][wm * 16 + g][kk + t] * cc;
      const double a1 = As[st][wm * 16 + 8 + g][kk + t] * cc;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double b = Bs[st][wn * 32 + j * 8 + g][kk + t];
        dmma884(acc[0][j][0], acc[0][j][1], a0, b);
        dmma884(acc[1][j][0], acc[1][j][1], a1, b);
      }
    }
    if (do_bias && tid < PBM) {
      const int64_t j0 = (int64_t)kt * BK;
      double s = bias_acc[tid];
#pragma unroll
      for (int kk = 0; kk < BK; ++kk)
        if (is_value_col(j0 + kk, p.int_cols, p.C)) s = fma(As[st][tid][kk], ccs[st][kk], s);
      bias_acc[tid] = s;
    }
    __syncthreads();
  }
  double* out = p.part + (int64_t)split * p.p + p.off;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int row = m0 + wm * 16 + i * 8 + g;
    if (row >= p.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = n0 + wn * 32 + j * 8 + 2 * t + e;
        if (col < p.N) out[(int64_t)row * p.N + col] = acc[i][j][e];
      }
    }
  }
  if (do_bias && tid < PBM && m0 + tid < p.M) out[(int64_t)p.M * p.N + m0 + tid] = bias_acc[tid];
}

cudaError_t phase_b(const PhbArgs& a, int splits, cudaStream_t st) {
  dim3 grid((a.N + PBN - 1) / PBN, (a.M + PBM - 1) / PBM, splits);
  probe_before(K_PHB, st);
  phb_kernel<<<grid, kThreads, 0, st>>>(a);
  probe_after(K_PHB, st);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Explicit Jacobian rows for the sketch (J-chunk formulation):
//   Jt[q][off_k + a*n_in + b] = sum_c D_k[a][(r,c)] Zin_k[b][(r,c)],  Jt[q][off_bk + a] = D_k[a][(r,0)]
// One CTA per (point, layer); threads stride over b, loop over a.  Write-bound.
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(kThreads) formj_kernel(FormJArgs a) {
  const int q = a.q0 + blockIdx.x;
  const int k = blockIdx.y;
  const int nin = a.n_in[k], nout = a.n_out[k];
  const double* Z = a.Z[k];
  const double* D = a.D[k];
  double* row = a.Jt + (int64_t)blockIdx.x * a.ldj + a.off[k];
  int64_t col0;
  int nch;
  if (q < a.n_int) {
    col0 = col_int(q, 0, a.C);
    nch = a.C;
  } else {
    col0 = a.int_cols + (q - a.n_int);
    nch = 1;
  }
  for (int b = threadIdx.x; b < nin; b += blockDim.x) {
    double z[12];
#pragma unroll
    for (int c = 0; c < 12; ++c) z[c] = (c < nch) ? Z[(int64_t)b * a.s_pad + col0 + c * PB] : 0.0;
    for (int o = 0; o < nout; ++o) {
      const double* drow = D + (int64_t)o * a.s_pad + col0;
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < 12; ++c)
        if (c < nch) s = fma(drow[c * PB], z[c], s);
      row[(int64_t)o * nin + b] = s;
    }
  }
  for (int o = threadIdx.x; o < nout; o += blockDim.x)
    row[(int64_t)nout * nin + o] = D[(int64_t)o * a.s_pad + col0];
}

cudaError_t form_j(const FormJArgs& a, int R, int n_layers, cudaStream_t st) {
  if (R <= 0) return cudaSuccess;
  probe_before(K_FORMJ, st);
  formj_kernel<<<dim3(R, n_layers), kThreads, 0, st>>>(a);
  probe_after(K_FORMJ, st);
  return cudaGetLastError();
}

}  // namespace ngd
