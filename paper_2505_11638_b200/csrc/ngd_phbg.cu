// Phase B of the factored Gramian matvec on the DMMA GEMM core, for the wide layers (both sides
// >= 256: C4 / C5's hidden layers):
//     out_l = D_l diag(c) Zin_l^T   (n_l x n_{l-1}, K = S channel-columns)  + bias column
// (the J^T c half of gramian.py:48-53, autodiff.py:90-125; layout in ngd_common.cuh).
//
// Same pipeline as ngd_gemm.cu -- 128 x 128 CTA tiles, 16-column k-stages streamed by TMA (one
// K-major box of D_l and one of Zin_l, 128-byte swizzle) through a 6-deep mbarrier ring, eight
// DMMA warps with 64 x 32 warp tiles, lane 0 of warp 0 issuing the stage four ahead -- plus the
// stage's 16 cotangents (a 128-byte bulk copy: a stage is one channel run of one point block, so
// its points are consecutive), which scale the Zin fragments, and the bias rows accumulated over
// value-channel stages.  Items are (split, layer, m-tile, n-tile), split-major: the CTAs running
// together read the same column range of D_l / Zin_l (each panel shared by two tiles, L2).  Every
// item writes its partial tile into part[split] in the flat parameter layout (model.py:41-51);
// reduce_splits / pcg_ad sum the splits in fixed order (bitwise deterministic).
//
// Measured at C5 (profiles/r02_phab_c5_summary.txt): the previous 64 x 64-tile kernel (ngd_phb2.cu,
// which keeps the thin input / output layers) ran the DMMA pipe at 80.6% of active cycles on 144
// of 148 SMs; this core ran the sketch GEMM at 95.6% (profiles/r02_gemm_c5_summary.txt).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>

#include "ngd_common.cuh"
#include "ngd_kernels.h"
#include "ngd_tma.cuh"

namespace ngd {

namespace {
constexpr int BBM = 128, BBN = 128, BBK = 16;
constexpr int BNS = 6, BAHEAD = 4;
#ifndef PHBG_CW
#define PHBG_CW 8  // DMMA warps: 8 (64 x 32 warp tiles, 232 registers) or 16 (32 x 32 warp tiles, 112 registers)
#endif
constexpr int kPhbgWarps = PHBG_CW;
constexpr int kMI = 16 / (PHBG_CW / 4);  // 8-row DMMA blocks per warp: 8 or 4

struct __align__(1024) BStage {
  double A[BBM * BBK];  // D_l rows m0 .. m0+127, 16 columns
  double B[BBN * BBK];  // Zin_l rows n0 .. n0+127
  double cc[BBK];       // cotangents of the stage's 16 columns
};
constexpr size_t kPhbgSmem = sizeof(BStage) * BNS + 2 * BNS * sizeof(unsigned long long) + 1024;

struct BItem {
  int h, tm, tn, split, s0, s1;
};
__device__ __forceinline__ BItem decode_b(const PhbgArgs& a, int idx) {
  BItem it;
  const int per = a.item_start[a.n_heavy];
  it.split = idx / per;
  int r = idx - it.split * per;
  int h = 0;
  while (h + 1 < a.n_heavy && r >= a.item_start[h + 1]) ++h;
  r -= a.item_start[h];
  it.h = h;
  it.tm = r / a.tiles_n[h];
  it.tn = r - it.tm * a.tiles_n[h];
  it.s0 = min(a.kstages, it.split * a.kps);
  it.s1 = min(a.kstages, it.s0 + a.kps);
  return it;
}
// first padded point of k-stage u (interior: C channel runs per 16-point block; then boundary blocks)
__device__ __forceinline__ int stage_point(const PhbgArgs& a, int u) {
  return u < a.int_units ? (u / a.C) * PB : a.nib * PB + (u - a.int_units) * PB;
}
__device__ __forceinline__ bool stage_is_value(const PhbgArgs& a, int u) {
  return u >= a.int_units || (u % a.C) == 0;
}
#ifndef PHBG_KORD
// fragment k order: lane t of MMA ks takes column koff[t] ^ 2 ks of the 16-column stage.  A 64-bit shared load
// is served per half-warp (rows g = 0..3 x the four t): with the 128-byte swizzle the 16 lanes cover all 32
// banks iff the four koff differ in (parity, bit 3) -- K-major tiles -- and in bits 1..2 -- MN-major tiles
// (ngd_phag.cu): {0, 10, 5, 15} does both.  The first order {0,4,1,5} + {0,2,8,10} (0) took two wavefronts
// per half-warp (ncu: 2 x the ideal shared wavefronts); 1 = {0,8,1,9} + 2 ks (K-major only).
#define PHBG_KORD 2
#endif
template <bool BIAS>
__device__ __forceinline__ void stage_mma(const double* As, const double* Bs, const double* cc, int wm, int wn, int g,
                                          int koff, double (&acc)[kMI][4][2], double (&bsum)[kMI]) {
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
#if PHBG_KORD == 2
    const int kk = (ks << 1) ^ koff;
#elif PHBG_KORD == 1
    const int kk = (ks << 1) + koff;
#else
    const int kk = ((ks & 1) << 1) + ((ks >> 1) << 3) + koff;
#endif
    const double cv = cc[kk];
    double av[kMI], bv[4];
#pragma unroll
    for (int i = 0; i < kMI; ++i) av[i] = As[tma::kmaj_off(wm * (kMI * 8) + i * 8 + g, kk)];
#pragma unroll
    for (int j = 0; j < 4; ++j) bv[j] = Bs[tma::kmaj_off(wn * 32 + j * 8 + g, kk)] * cv;
#pragma unroll
    for (int i = 0; i < kMI; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], av[i], bv[j]);
    if (BIAS) {
#pragma unroll
      for (int i = 0; i < kMI; ++i) bsum[i] = fma(av[i], cv, bsum[i]);
    }
  }
}
}  // namespace

#ifndef PHBG_WS
#define PHBG_WS 1  // 1: a producer warpgroup issues the TMA ring (setmaxnreg hands its registers to the DMMA warps)
#endif
#if PHBG_WS
constexpr int kPhbgThreads = (kPhbgWarps + 4) * 32;
// Warp-specialised form.  Measured on the single-role kernel (ncu source page, C5): the ring was issued
// by lane 0 of DMMA warp 0 -- ~135 dependent instructions per k-stage (slot wait, three bulk copies,
// the stage -> point division), 21% of that warp's time -- and the other seven warps, limited to the
// ring's lookahead past warp 0, spent 8.5% of theirs waiting on the full barriers (DMMA pipe 86%).
// Here warps 8..11 are a producer warpgroup that gives its registers away (setmaxnreg: 12 warps launch
// at 168 registers, the DMMA warps grow to 232) and one of its lanes runs the whole (item, stage)
// sequence ahead of the consumers, bounded only by the ring depth.
__global__ void __launch_bounds__(kPhbgThreads, 1) phbg_kernel(const __grid_constant__ PhbgArgs a,
                                                               const __grid_constant__ PhbgMaps maps) {
  pdl_entry();  // (PCG chain: programmatic dependent launch)
  if (a.skip && *a.skip) return;
  extern __shared__ unsigned char bsm_raw[];
  unsigned char* base = bsm_raw + ((1024u - (tma::smem(bsm_raw) & 1023u)) & 1023u);
  BStage* st = reinterpret_cast<BStage*>(base);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(st + BNS);
  unsigned long long* empty = full + BNS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < BNS; ++s) {
      tma::mbar_init(&full[s], 1);
      tma::mbar_init(&empty[s], kPhbgWarps);
    }
    tma::fence_init();
  }
  __syncthreads();
  const int n_items = a.item_start[a.n_heavy] * a.G;
  if (warp >= kPhbgWarps) {  // producer warpgroup
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(PHBG_CW == 16 ? 32 : 40));
    if (warp == kPhbgWarps && lane == 0) {
      unsigned qp = 0;
      for (int idx = blockIdx.x; idx < n_items; idx += gridDim.x) {
        const BItem it = decode_b(a, idx);
        const int m0 = it.tm * BBM, n0 = it.tn * BBN;
        for (int s = it.s0; s < it.s1; ++s, ++qp) {
          const int slot = qp % BNS;
          if (qp >= BNS) tma::wait(&empty[slot], ((qp / BNS) - 1) & 1u);
          tma::expect_tx(&full[slot], (2 * BBM * BBK + BBK) * sizeof(double));
          tma::load2d(st[slot].A, &maps.d[it.h], s * BBK, m0, &full[slot]);
          tma::load2d(st[slot].B, &maps.z[it.h], s * BBK, n0, &full[slot]);
          tma::load1d(st[slot].cc, a.cvec + stage_point(a, s), BBK * sizeof(double), &full[slot]);
        }
      }
    }
    return;
  }
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(PHBG_CW == 16 ? 112 : 232));
  const int wm = warp >> 2, wn = warp & 3;
  const int g = lane >> 2, t = lane & 3;
#if PHBG_KORD == 2
  const int koff = ((t & 1) * 10) ^ ((t >> 1) * 5);  // {0, 10, 5, 15}
#elif PHBG_KORD == 1
  const int koff = ((t & 1) << 3) | (t >> 1);  // {0, 8, 1, 9}
#else
  const int koff = ((t & 1) << 2) | (t >> 1);  // {0, 4, 1, 5}: fragment k order (ngd_gemm.cu)
#endif
  unsigned q = 0;
  for (int idx = blockIdx.x; idx < n_items; idx += gridDim.x) {
    const BItem it = decode_b(a, idx);
    const bool do_bias = it.tn == 0 && wn == 0;
    double acc[kMI][4][2], bsum[kMI];
#pragma unroll
    for (int i = 0; i < kMI; ++i) {
      bsum[i] = 0.0;
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    }
    // value-channel stages (bias rows): every C-th interior stage, every boundary stage
    int vc = it.s0 < a.int_units ? it.s0 % a.C : 0;
    for (int s = it.s0; s < it.s1; ++s, ++q) {
      const int slot = q % BNS;
      tma::wait(&full[slot], (q / BNS) & 1u);
      const double* As = st[slot].A;
      const double* Bs = st[slot].B;
      const bool value = s >= a.int_units || vc == 0;
      vc = (vc + 1 == a.C) ? 0 : vc + 1;
      // the n-tile-0 warps also accumulate the bias rows on value-channel stages: a uniform branch
      // between two unrolled bodies (a predicated bias FMA would issue on every stage)
      if (do_bias && value)
        stage_mma<true>(As, Bs, st[slot].cc, wm, wn, g, koff, acc, bsum);
      else
        stage_mma<false>(As, Bs, st[slot].cc, wm, wn, g, koff, acc, bsum);
      tma::fence_proxy_async();  // generic-proxy reads of the slot before the async-proxy refill (ngd_phag.cu)
      __syncwarp();
      if (lane == 0) tma::arrive(&empty[slot]);
    }
    // epilogue: this split's partial of W_l (rows m, cols n) and, from the n-tile 0 warps, of b_l
    const int M = a.M[it.h], N = a.N[it.h];
    double* out = a.part + (int64_t)it.split * a.p + a.off[it.h];
    const int m0 = it.tm * BBM + wm * (kMI * 8) + g, n0 = it.tn * BBN + wn * 32 + 2 * t;
#pragma unroll
    for (int i = 0; i < kMI; ++i) {
      const int m = m0 + i * 8;
      if (m < M) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int n = n0 + j * 8 + e;
            if (n < N) out[(int64_t)m * N + n] = acc[i][j][e];
          }
      }
      if (do_bias) {  // fixed xor tree over the four k-lanes
        double b = bsum[i];
        b += __shfl_xor_sync(0xffffffffu, b, 1);
        b += __shfl_xor_sync(0xffffffffu, b, 2);
        if (t == 0 && m < M) out[(int64_t)M * N + m] = b;
      }
    }
  }
}
#else
constexpr int kPhbgThreads = kPhbgWarps * 32;
__global__ void __maxnreg__(224) phbg_kernel(const __grid_constant__ PhbgArgs a, const __grid_constant__ PhbgMaps maps) {
  pdl_entry();  // (PCG chain: programmatic dependent launch)
  if (a.skip && *a.skip) return;
  extern __shared__ unsigned char bsm_raw[];
  unsigned char* base = bsm_raw + ((1024u - (tma::smem(bsm_raw) & 1023u)) & 1023u);
  BStage* st = reinterpret_cast<BStage*>(base);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(st + BNS);
  unsigned long long* empty = full + BNS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < BNS; ++s) {
      tma::mbar_init(&full[s], 1);
      tma::mbar_init(&empty[s], kPhbgWarps);
    }
    tma::fence_init();
  }
  __syncthreads();
  const int n_items = a.item_start[a.n_heavy] * a.G;
  // producer cursor (thread 0): the (item, stage) sequence of this CTA
  const bool producer = (tid == 0);
  int p_idx = blockIdx.x, p_s = 0, p_s1 = 0, p_h = 0, p_m0 = 0, p_n0 = 0;
  bool p_valid = false;
  auto p_load = [&]() {
    while (p_idx < n_items) {
      const BItem it = decode_b(a, p_idx);
      if (it.s0 < it.s1) {
        p_s = it.s0;
        p_s1 = it.s1;
        p_h = it.h;
        p_m0 = it.tm * BBM;
        p_n0 = it.tn * BBN;
        return true;
      }
      p_idx += gridDim.x;
    }
    return false;
  };
  if (producer) p_valid = p_load();
  unsigned qp = 0;
  const int wm = warp >> 2, wn = warp & 3;
  const int g = lane >> 2, t = lane & 3;
  const int koff = ((t & 1) << 2) | (t >> 1);  // {0, 4, 1, 5}: conflict-free fragment loads (ngd_gemm.cu)
  unsigned q = 0;
  for (int idx = blockIdx.x; idx < n_items; idx += gridDim.x) {
    const BItem it = decode_b(a, idx);
    const bool do_bias = it.tn == 0 && wn == 0;
    double acc[kMI][4][2], bsum[kMI];
#pragma unroll
    for (int i = 0; i < kMI; ++i) {
      bsum[i] = 0.0;
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    }
    for (int s = it.s0; s < it.s1; ++s, ++q) {
      if (producer) {
        while (p_valid && qp < q + BAHEAD) {
          const int slot = qp % BNS;
          if (qp >= BNS) tma::wait(&empty[slot], ((qp / BNS) - 1) & 1u);
          tma::expect_tx(&full[slot], (2 * BBM * BBK + BBK) * sizeof(double));
          const int k0 = p_s * BBK;
          tma::load2d(st[slot].A, &maps.d[p_h], k0, p_m0, &full[slot]);
          tma::load2d(st[slot].B, &maps.z[p_h], k0, p_n0, &full[slot]);
          tma::load1d(st[slot].cc, a.cvec + stage_point(a, p_s), BBK * sizeof(double), &full[slot]);
          ++qp;
          if (++p_s >= p_s1) {
            p_idx += gridDim.x;
            p_valid = p_load();
          }
        }
      }
      __syncwarp();
      const int slot = q % BNS;
      tma::wait(&full[slot], (q / BNS) & 1u);
      const double* As = st[slot].A;
      const double* Bs = st[slot].B;
      // value-channel stages of the n-tile-0 warps also accumulate the bias rows: a uniform branch
      // between two unrolled bodies (a predicated bias FMA would issue on every stage)
      if (do_bias && stage_is_value(a, s))
        stage_mma<true>(As, Bs, st[slot].cc, wm, wn, g, koff, acc, bsum);
      else
        stage_mma<false>(As, Bs, st[slot].cc, wm, wn, g, koff, acc, bsum);
      tma::fence_proxy_async();
      __syncwarp();
      if (lane == 0) tma::arrive(&empty[slot]);
    }
    // epilogue: this split's partial of W_l (rows m, cols n) and, from the n-tile 0 warps, of b_l
    const int M = a.M[it.h], N = a.N[it.h];
    double* out = a.part + (int64_t)it.split * a.p + a.off[it.h];
    const int m0 = it.tm * BBM + wm * (kMI * 8) + g, n0 = it.tn * BBN + wn * 32 + 2 * t;
#pragma unroll
    for (int i = 0; i < kMI; ++i) {
      const int m = m0 + i * 8;
      if (m < M) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int n = n0 + j * 8 + e;
            if (n < N) out[(int64_t)m * N + n] = acc[i][j][e];
          }
      }
      if (do_bias) {  // fixed xor tree over the four k-lanes
        double b = bsum[i];
        b += __shfl_xor_sync(0xffffffffu, b, 1);
        b += __shfl_xor_sync(0xffffffffu, b, 2);
        if (t == 0 && m < M) out[(int64_t)M * N + m] = b;
      }
    }
  }
}

#endif

namespace {
PFN_cuTensorMapEncodeTiled_v12000 enc_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}
// rows x s_pad row-major jets, box 16 columns x 128 rows (rows past `rows` zero-filled)
bool encode_jets(CUtensorMap* m, const double* base, int rows, int64_t s_pad) {
  auto enc = enc_fn();
  if (!enc) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)s_pad, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)s_pad * sizeof(double)};
  const cuuint32_t box[2] = {(cuuint32_t)BBK, (cuuint32_t)BBM};
  const cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace

// wide layers only: at 128 x 128 (C3) the two-launch split (this kernel + the thin pipeline of
// ngd_phb2.cu) measured slower than ngd_phb2.cu alone (C3 phase B 0.35 vs 0.31 ms per matvec);
// at 256 x 256 (C4 / C5) it is faster (C5 22.2 vs 22.6 ms, DMMA pipe 86% vs 81%)
#ifndef NGD_WIDE_MIN
#define NGD_WIDE_MIN 256
#endif
bool phbg_layer_ok(int M, int N) { return M >= NGD_WIDE_MIN && N >= NGD_WIDE_MIN; }

// splits G of the K range so the items fill whole waves of one CTA per SM (>= 64 stages per split)
int phbg_splits(int tiles, int kstages) {
  int best = 1;
  double best_eff = -1.0;
  const int gmax = std::max(1, std::min(148, kstages / 64));
  for (int gs = 1; gs <= gmax; ++gs) {
    const int items = tiles * gs;
    const int waves = (items + 147) / 148;
    const double eff = (double)items / (waves * 148.0) - 0.0005 * gs;
    if (eff > best_eff + 1e-12) {
      best_eff = eff;
      best = gs;
    }
  }
  return best;
}

cudaError_t phase_b_gemm(const PhbgArgs& a, PhbgCache& cache, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(phbg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPhbgSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  for (int h = 0; h < a.n_heavy; ++h) {
    if (cache.kd[h] != cache.src_d[h] || cache.kz[h] != cache.src_z[h] || cache.km[h] != a.M[h] ||
        cache.kn[h] != a.N[h] || cache.ks[h] != cache.s_pad) {
      if (!encode_jets(&cache.maps.d[h], cache.src_d[h], a.M[h], cache.s_pad) ||
          !encode_jets(&cache.maps.z[h], cache.src_z[h], a.N[h], cache.s_pad))
        return cudaErrorInvalidValue;
      cache.kd[h] = cache.src_d[h];
      cache.kz[h] = cache.src_z[h];
      cache.km[h] = a.M[h];
      cache.kn[h] = a.N[h];
      cache.ks[h] = cache.s_pad;
    }
  }
  const int items = a.item_start[a.n_heavy] * a.G;
  if (items <= 0) return cudaSuccess;
  probe_before(K_PHB, st);
  const cudaError_t e = launch_pdl(phbg_kernel, dim3(std::min(items, 148)), dim3(kPhbgThreads), kPhbgSmem, st, a,
                                   cache.maps);
  probe_after(K_PHB, st);
  return e;
}

}  // namespace ngd
