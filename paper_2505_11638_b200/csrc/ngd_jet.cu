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
#include <climits>
#include "ngd_common.cuh"
#include "ngd_kernels.h"

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace ngd {



constexpr int BM = 64, BK = 16, APAD = 4;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// forward jet nonlinearity (tanh, forward-Laplacian channels).
// The last channel carries Lambda_S = sum_{i in S} d_ii of the coordinate subset
// S = lap_mask (all coordinates: the Laplacian; heat1p1d: {x}, problems.py:290-292).
template <int C>
__device__ __forceinline__ void jet_act(const double (&a)[C], double (&z)[C], unsigned mask) {
  const double t = tanh(a[0]);
  z[0] = t;
  if constexpr (C > 1) {
    const double s1 = 1.0 - t * t;
    const double s2 = -2.0 * t * s1;
    double q = 0.0;
#pragma unroll
    for (int i = 1; i < C - 1; ++i) {
      z[i] = s1 * a[i];
      if ((mask >> (i - 1)) & 1u) q += a[i] * a[i];
    }
    z[C - 1] = s2 * q + s1 * a[C - 1];
  }
}

// reverse of jet_act: adjoints of the outputs -> adjoints of the pre-activations
template <int C>
__device__ __forceinline__ void jet_act_rev(const double (&a)[C], const double (&g)[C], double (&o)[C],
                                            unsigned mask) {
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
      const bool in_s = (mask >> (i - 1)) & 1u;
      if (in_s) q += a[i] * a[i];
      s1b += g[i] * a[i];
      o[i] = in_s ? g[i] * s1 + 2.0 * lb * s2 * a[i] : g[i] * s1;
    }
    o[C - 1] = lb * s1;
    const double s2b = lb * q;
    const double tb = g[0] - 2.0 * t * s1b + (6.0 * t * t - 2.0) * s2b;
    o[0] = tb * s1;
  }
}

template <int C, int MODE>
__device__ __forceinline__ void jet_tile(const JetArgs& p, const int bx, const int by) {
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
  const int m0 = by * BM;
  const int64_t cblk = p.col0 + (int64_t)bx * NC;

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
  // skip MMA work on all-padding rows (output layer: M = 1) and all-padding k-steps (input layer: K = d)
  const bool m_active = (m0 + wm * 16) < p.M;
  const int kvalid = p.K > 0 ? p.K : p.Kp;
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
    if (m_active && kt * BK + BK <= kvalid) {
      // full stage: no early exit inside the unrolled k-steps, so the scheduler can interleave the
      // 2 C independent accumulator chains across k-steps (the guarded loop below serialised each
      // chain's four DMMAs back to back: profiles/r02_phab_c5 source page)
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
    } else {
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4) {
        if (!m_active || kt * BK + kk >= kvalid) break;
        const double a0 = as[kk];
        const double a1 = as[8 * ASTR + kk];
#pragma unroll
        for (int c = 0; c < C; ++c) {
          const double b = bs[kk * BSTR + c * PB];
          dmma884(acc[0][c][0], acc[0][c][1], a0, b);
          dmma884(acc[1][c][0], acc[1][c][1], a1, b);
        }
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
            jet_act<C>(v, z, p.lap_mask);
#pragma unroll
            for (int c = 0; c < C; ++c) p.z_out[cbase + c * PB] = z[c];
          }
        } else {
          double a[C], o[C];
#pragma unroll
          for (int c = 0; c < C; ++c) a[c] = p.dbuf[cbase + c * PB];
          jet_act_rev<C>(a, v, o, p.lap_mask);
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
      p.partA[(int64_t)by * p.n_pts_pad + p.pt0 + bx * PB + tid] = s;
    }
  }
}

template <int C, int MODE>
__global__ void __launch_bounds__(kThreads) jet_gemm_kernel(JetArgs p) {
  jet_tile<C, MODE>(p, blockIdx.x, blockIdx.y);
}

// Phase A over ALL layers and both point segments in one launch (tile table).
template <int C>
__global__ void __launch_bounds__(kThreads) pha_all_kernel(PhaAll a) {
  pdl_entry();  // (PCG chain: programmatic dependent launch)
  const int t = blockIdx.x;
  int l = 0;
  while (l + 1 < a.n_layers && t >= a.tile_start[l + 1]) ++l;
  const int local = t - a.tile_start[l];
  const int mt = a.mtiles[l];
  const int n_int_tiles = a.nib * mt;
  JetArgs p = a.L[l];
  // m-tile fastest: the mt CTAs of one point block run back to back and share its Zin slice in L2
  // (block-major order read each slice from DRAM mt times: 55.9 GB per C5 launch for ~17 GB of jets)
  if (local < n_int_tiles) {
    jet_tile<C, PHA>(p, local / mt, local % mt);
  } else {
    const int lb = local - n_int_tiles;
    p.col0 = a.int_cols;
    p.pt0 = a.nib * PB;
    jet_tile<1, PHA>(p, lb / mt, lb % mt);
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

template <int C>
static cudaError_t launch_pha_all(const PhaAll& a, cudaStream_t st) {
  constexpr int NC = PB * C;
  const size_t smem = sizeof(double) * (2 * BM * (BK + APAD) + 2 * BK * (NC + 4));
  auto kern = pha_all_kernel<C>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set = true;
  }
  const int tiles = a.tile_start[a.n_layers];
  if (tiles <= 0) return cudaSuccess;
  probe_before(K_PHA, st);
  const cudaError_t e = launch_pdl(kern, dim3(tiles), dim3(kThreads), smem, st, a);
  probe_after(K_PHA, st);
  return e;
}

cudaError_t pha_all(int C, const PhaAll& a, cudaStream_t st) {
  switch (C) {
    case 3: return launch_pha_all<3>(a, st);
    case 4: return launch_pha_all<4>(a, st);
    case 5: return launch_pha_all<5>(a, st);
    case 6: return launch_pha_all<6>(a, st);
    case 7: return launch_pha_all<7>(a, st);
    case 8: return launch_pha_all<8>(a, st);
    case 12: return launch_pha_all<12>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

// Both point segments of a forward / reverse layer sweep in one launch: CTAs [0, nib) take the
// interior blocks (C channels), CTAs [nib, nib + nbb) the boundary blocks (value channel only).
// one linear grid, m-tile fastest: the m-tiles of one point block are adjacent CTAs and share its
// input slice in L2 (the block-major order re-read every slice from DRAM once per m-tile)
template <int C, int MODE>
__global__ void __launch_bounds__(kThreads) jet_both_kernel(JetArgs p, int nib, int64_t int_cols, int mtiles) {
  const int blk = (int)(blockIdx.x / (unsigned)mtiles), mt = (int)(blockIdx.x % (unsigned)mtiles);
  if (blk < nib) {
    jet_tile<C, MODE>(p, blk, mt);
  } else {
    JetArgs q = p;
    q.col0 = int_cols;
    q.pt0 = nib * PB;
    jet_tile<1, MODE>(q, blk - nib, mt);
  }
}

template <int C, int MODE>
static cudaError_t launch_jet_both(const JetArgs& a, int nib, int nbb, int64_t int_cols, int mtiles, cudaStream_t st) {
  constexpr int NC = PB * C;
  const size_t smem = sizeof(double) * (2 * BM * (BK + APAD) + 2 * BK * (NC + 4));
  auto kern = jet_both_kernel<C, MODE>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set = true;
  }
  if (nib + nbb <= 0 || mtiles <= 0) return cudaSuccess;
  JetArgs b = a;
  b.col0 = 0;
  b.pt0 = 0;
  probe_before(MODE == FWD ? K_FWD : K_REV, st);
  kern<<<dim3((unsigned)((nib + nbb) * mtiles)), kThreads, smem, st>>>(b, nib, int_cols, mtiles);
  probe_after(MODE == FWD ? K_FWD : K_REV, st);
  return cudaGetLastError();
}

cudaError_t jet_gemm_both(int C, int mode, const JetArgs& a, int nib, int nbb, int64_t int_cols, int mtiles,
                          cudaStream_t st) {
#define NGD_JET_BOTH(CC)                                                                          \
  case CC:                                                                                        \
    return mode == FWD ? launch_jet_both<CC, FWD>(a, nib, nbb, int_cols, mtiles, st)              \
                       : launch_jet_both<CC, REV>(a, nib, nbb, int_cols, mtiles, st);
  switch (C) {
    NGD_JET_BOTH(3)
    NGD_JET_BOTH(4)
    NGD_JET_BOTH(5)
    NGD_JET_BOTH(6)
    NGD_JET_BOTH(7)
    NGD_JET_BOTH(8)
    NGD_JET_BOTH(12)
    default:
      return cudaErrorInvalidValue;
  }
#undef NGD_JET_BOTH
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
// Explicit Jacobian rows for the sketch (J-chunk formulation):
//   Jt[pt][off_l + a*n_in + b] = sum_c D_l[a][(pt,c)] Zin_l[b][(pt,c)],  Jt[pt][off_bl + a] = D_l[a][(pt,0)]
// i.e. per point a rank-C outer-product sum: a 64 x 64 tile of J_r[W_l] is an (a x c) . (c x b)
// product with K = C channels (<= 12: three DMMA k-steps of 4).  One CTA per (point block of 16,
// layer, 64 x 64 tile): the block's D and Zin rows of the tile are staged in shared memory
// (coalesced 128-byte channel runs), then every warp owns one 8-row band of the tile for all 16
// points (8 DMMA blocks x k-steps per point) and stores its rows of J straight from the
// accumulators.  Write-bound: 8 p bytes per point (the previous scalar-FMA form issued one shared
// load per FMA and ran at 0.64 TB/s at C5, profiles/r02_launches_c5_summary.txt).
// Shared layout: element (row, channel c, point r) at row * FJ_LD + c * 17 + r -- the channel
// stride 17 and FJ_LD = 4 (mod 16) make every DMMA fragment load two wavefronts.
constexpr int FJ_T = 64;                     // tile rows (a) and columns (b)
constexpr int FJ_CS = 17;                    // channel stride in shared memory (doubles)
constexpr int FJ_LD = 12 * FJ_CS + 8;        // 212 = 4 (mod 16)
constexpr int FJ_THREADS = 256;

__global__ void __launch_bounds__(FJ_THREADS, 1) formj_kernel(FormJArgs a) {
  extern __shared__ __align__(16) double fsm[];
  double* Ds = fsm;                 // [FJ_T][FJ_LD]
  double* Zs = fsm + FJ_T * FJ_LD;  // [FJ_T][FJ_LD]
  const int l = blockIdx.y;
  const int nin = a.n_in[l], nout = a.n_out[l];
  const int tiles_b = (nin + FJ_T - 1) / FJ_T;
  const int a0 = (blockIdx.z / tiles_b) * FJ_T, b0 = (blockIdx.z % tiles_b) * FJ_T;
  if (a0 >= nout) return;
  const int blk = a.blk0 + blockIdx.x * max(a.blk_stride, 1);  // global point block
  const bool interior = blk < a.nib;
  const int Cs = interior ? a.C : 1;
  const int nks = (Cs + 3) / 4;         // DMMA k-steps (channels padded to a multiple of 4 with zeros)
  const int64_t cbase = interior ? (int64_t)blk * PB * a.C : a.int_cols + (int64_t)(blk - a.nib) * PB;
  const double* Z = a.Z[l];
  const double* D = a.D[l];
  const int nb = min(FJ_T, nin - b0), na = min(FJ_T, nout - a0);
  const int ncols = PB * 4 * nks;  // channels 0 .. 4 nks - 1 (zero past Cs)
  // stage with asynchronous 8-byte copies (the channel stride 17 leaves runs 8-byte aligned only):
  // all of a thread's ~96 loads in flight at once -- plain loads stalled on DRAM latency at one CTA
  // per SM (long-scoreboard 15 cycles per issue, 1.07 TB/s of writes)
  for (int e = threadIdx.x; e < FJ_T * ncols; e += FJ_THREADS) {
    const int r = e / ncols, cc = e - r * ncols;  // cc = c * 16 + point
    const int c = cc >> 4, pt = cc & 15;
    const bool on = c < Cs;
    double* zd = Zs + r * FJ_LD + c * FJ_CS + pt;
    double* dd = Ds + r * FJ_LD + c * FJ_CS + pt;
    if (on && r < nb)
      cp_async8(zd, Z + (int64_t)(b0 + r) * a.s_pad + cbase + cc);
    else
      *zd = 0.0;
    if (on && r < na)
      cp_async8(dd, D + (int64_t)(a0 + r) * a.s_pad + cbase + cc);
    else
      *dd = 0.0;
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int64_t prow0 = (int64_t)blockIdx.x * PB;  // chunk-local padded point row
  const int64_t off = a.off[l];
  const int arow = warp * 8 + g;  // this lane's tile row (A fragment / accumulator row)
  const bool row_ok = arow < na;
  const bool vec2 = ((off + (int64_t)(a0 + arow) * nin + b0) & 1) == 0 && (a.ldj & 1) == 0;
  const bool trk_r = a.rmax != nullptr, trk_c = a.cmax != nullptr, store = !a.no_store;
  unsigned long long cm[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) cm[j][0] = cm[j][1] = 0ull;
  unsigned long long bm = 0ull;  // bias column maximum (threads < na)
  // column prescale exponents of this thread's 16 weights and (threads < na) one bias
  int gam[8][2];
  int gamb = 0;
  if (trk_r) {
    const int* ce = a.cexp + off + (int64_t)(a0 + arow) * nin + b0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int col = j * 8 + 2 * t;
      gam[j][0] = (row_ok && col < nb) ? ce[col] : 0;
      gam[j][1] = (row_ok && col + 1 < nb) ? ce[col + 1] : 0;
    }
    if (b0 == 0 && threadIdx.x < na) gamb = a.cexp[off + (int64_t)nout * nin + a0 + threadIdx.x];
  }
  for (int r = 0; r < PB; ++r) {
    double acc[8][2];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < 3; ++ks) {
      if (ks < nks) {
        const int c = ks * 4 + t;
        const double av = Ds[arow * FJ_LD + c * FJ_CS + r];
#pragma unroll
        for (int j = 0; j < 8; ++j) dmma884(acc[j][0], acc[j][1], av, Zs[(j * 8 + g) * FJ_LD + c * FJ_CS + r]);
      }
    }
    if (store) {
      double* row = a.Jt + (prow0 + r) * a.ldj + off + (int64_t)(a0 + arow) * nin + b0;
      if (row_ok) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int col = j * 8 + 2 * t;
          if (vec2 && col + 1 < nb) {
            *reinterpret_cast<double2*>(row + col) = make_double2(acc[j][0], acc[j][1]);
          } else {
            if (col < nb) row[col] = acc[j][0];
            if (col + 1 < nb) row[col + 1] = acc[j][1];
          }
        }
      }
      if (b0 == 0 && threadIdx.x < na)  // bias entries: value channel of D
        a.Jt[(prow0 + r) * a.ldj + off + (int64_t)nout * nin + a0 + threadIdx.x] = Ds[threadIdx.x * FJ_LD + r];
    }
    if (trk_c) {
      if (row_ok) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int col = j * 8 + 2 * t;
          if (col < nb) cm[j][0] = max(cm[j][0], (unsigned long long)__double_as_longlong(fabs(acc[j][0])));
          if (col + 1 < nb) cm[j][1] = max(cm[j][1], (unsigned long long)__double_as_longlong(fabs(acc[j][1])));
        }
      }
      if (b0 == 0 && threadIdx.x < na)
        bm = max(bm, (unsigned long long)__double_as_longlong(fabs(Ds[threadIdx.x * FJ_LD + r])));
    }
    if (trk_r) {
      long long rm = kOzLogEmpty - 1;
      if (row_ok) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int col = j * 8 + 2 * t;
          if (col < nb) rm = max(rm, oz_logbits(acc[j][0], gam[j][0]));
          if (col + 1 < nb) rm = max(rm, oz_logbits(acc[j][1], gam[j][1]));
        }
      }
      if (b0 == 0 && threadIdx.x < na) rm = max(rm, oz_logbits(Ds[threadIdx.x * FJ_LD + r], gamb));
      for (int o = 16; o; o >>= 1) rm = max(rm, __shfl_xor_sync(0xffffffffu, rm, o));
      if (lane == 0 && rm >= kOzLogEmpty) atomicMax(a.rmax + prow0 + r, rm);
    }
  }
  if (trk_c) {
    if (row_ok) {
      unsigned long long* cr = a.cmax + off + (int64_t)(a0 + arow) * nin + b0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int col = j * 8 + 2 * t;
        if (col < nb && cm[j][0]) atomicMax(cr + col, cm[j][0]);
        if (col + 1 < nb && cm[j][1]) atomicMax(cr + col + 1, cm[j][1]);
      }
    }
    if (b0 == 0 && threadIdx.x < na && bm) atomicMax(a.cmax + off + (int64_t)nout * nin + a0 + threadIdx.x, bm);
  }
}

size_t formj_smem(int C) {
  (void)C;
  return sizeof(double) * 2 * FJ_T * FJ_LD;
}

cudaError_t form_j(const FormJArgs& a, int nblocks, int n_layers, int max_nin, int max_nout, cudaStream_t st) {
  if (nblocks <= 0) return cudaSuccess;
  if (a.C > 12) return cudaErrorInvalidValue;
  const size_t smem = formj_smem(a.C);
  static size_t attr = 0;
  if (smem > attr) {
    cudaFuncSetAttribute(formj_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = smem;
  }
  const int tz = ((max_nout + FJ_T - 1) / FJ_T) * ((max_nin + FJ_T - 1) / FJ_T);
  probe_before(K_FORMJ, st);
  formj_kernel<<<dim3(nblocks, n_layers, tz), FJ_THREADS, smem, st>>>(a);
  probe_after(K_FORMJ, st);
  return cudaGetLastError();
}

}  // namespace ngd
