// MEASURED SLOWER, not compiled (round 2): C5 matvec 45.97 ms with this phase A vs 44.4 ms with
// pha_all_kernel (per-layer items: 47.8 ms, 72% DMMA pipe).  The D epilogue per 16 K-stages and
// the per-item reduction idle the SM; kept as evidence.
// Phase A of the factored Gramian matvec on the DMMA GEMM core, for the wide layers (both sides
// >= 256: C4 / C5's hidden layers):
//     (J v)_r += sum_c < D_l[:, (r,c)], V_l Zin_l[:, (r,c)] + vb_l [c = value] >
// (the J v half of gramian.py:48-53, autodiff.py:90-109; layout in ngd_common.cuh).
//
// P = V_l Zin_l is a GEMM with K = n_{l-1}; the per-point result is the column-wise dot of P with
// D_l, summed over the point's channels.  Pipeline of ngd_gemm.cu: 128 x 128 tiles (m = rows of
// V_l, n = channel-point columns), 16-row k-stages streamed by TMA (V_l K-major: one 16 x 128 box;
// Zin_l MN-major: eight 16 x 16 boxes; 128-byte swizzle) through a 6-deep mbarrier ring, eight
// DMMA warps of 64 x 32, lane 0 of warp 0 issuing four stages ahead.  After an item's K stages the
// same ring carries four "D stages" (32 rows x 128 columns of D_l each, eight 16 x 32 boxes), so
// the epilogue's operand arrives like any other stage instead of as a latency-bound global load.
// Each warp dots its accumulators with the D rows it owns, sums over rows by shuffles, the CTA
// combines its two row halves and the channel runs of each point, and writes one partial per point
// into the phase-A partial rows (reduce_pha sums rows in fixed order: deterministic).
// Items: (n-tile, m-tile) over all wide layers, m-tile fastest -- the two m-tiles of a Zin panel
// are adjacent.
// Tiles never straddle the interior / boundary segments; an interior tile covers the channel
// runs of at most two point blocks at C <= 12, whose partials go to row (tile - first tile of
// the block) of the m-tile's group (rows a block never touches stay zero).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>

#include "ngd_common.cuh"
#include "ngd_kernels.h"
#include "ngd_tma.cuh"

namespace ngd {

namespace {
constexpr int ABM = 128, ABN = 128, ABK = 16;
constexpr int ANS = 6, AAHEAD = 4;
constexpr int kPhagWarps = 8;
constexpr int kDStages = ABM / 32;  // D rows per item in 32-row stages

struct __align__(1024) AStage {
  double A[ABM * ABK];  // K stage: V_l rows (K-major box); D stage: with B, 8 boxes of [32 rows][16 cols]
  double B[ABN * ABK];  // K stage: Zin_l rows k0 .. k0+15, 128 columns (8 boxes of [16 k][16 cols])
};
static_assert(sizeof(double) * 32 * ABN == sizeof(double) * (ABM + ABN) * ABK, "a D stage fills one ring slot");
constexpr size_t kPhagSmem = sizeof(AStage) * ANS + 2 * ANS * sizeof(unsigned long long) + 1024;

struct AItem {
  int mt, nt;
};
__device__ __forceinline__ AItem decode_a(const PhagArgs& a, int idx) {
  AItem it;
  it.mt = idx % a.mtiles;
  it.nt = idx / a.mtiles;
  return it;
}
// first column of n-tile nt: interior tiles over [0, int_cols), boundary tiles over [int_cols, s_pad)
__device__ __forceinline__ int64_t tile_col(const PhagArgs& a, int nt) {
  return nt < a.int_tiles ? (int64_t)nt * ABN : a.int_cols + (int64_t)(nt - a.int_tiles) * ABN;
}
__device__ __forceinline__ int tile_cols(const PhagArgs& a, int nt) {
  const int64_t c0 = tile_col(a, nt);
  const int64_t end = nt < a.int_tiles ? a.int_cols : a.s_pad;
  return (int)(end - c0 < ABN ? end - c0 : ABN);
}
// element (row r of a 32-row D stage, column n of the tile) in the 8 boxes of [32][16]
__device__ __forceinline__ int dstage_off(int r, int n) {
  return (n >> 4) * 512 + r * 16 + (((((n & 15) >> 1) ^ (r & 7)) << 1) | (n & 1));
}
__device__ __forceinline__ int mnmaj_off(int mn, int k) {
  return (mn >> 4) * 256 + k * 16 + (((((mn & 15) >> 1) ^ (k & 7)) << 1) | (mn & 1));
}
}  // namespace

// One item = one (n-tile, m-tile) over ALL wide layers: per layer its K stages (P = V_l Zin_l in
// the accumulators) then its D stages (column sums of D_l o P accumulated across layers), then one
// per-point reduction per item -- items of one layer measured 72% of the DMMA pipe (the per-item
// epilogue and barriers idle the SM every 16 stages).
__global__ void __maxnreg__(224) phag_kernel(const __grid_constant__ PhagArgs a, const __grid_constant__ PhagMaps maps) {
  pdl_entry();  // (PCG chain: programmatic dependent launch)
  if (a.skip && *a.skip) return;
  extern __shared__ unsigned char asm_raw[];
  unsigned char* base = asm_raw + ((1024u - (tma::smem(asm_raw) & 1023u)) & 1023u);
  AStage* st = reinterpret_cast<AStage*>(base);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(st + ANS);
  unsigned long long* empty = full + ANS;
  __shared__ double red[2][ABN];  // column sums of the two row halves
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < ANS; ++s) {
      tma::mbar_init(&full[s], 1);
      tma::mbar_init(&empty[s], kPhagWarps);
    }
    tma::fence_init();
  }
  __syncthreads();
  const int n_items = a.n_tiles * a.mtiles;
  const int kst = a.kstages;                   // K stages per layer
  const int per_layer = kst + kDStages;
  const int per_item = a.n_wide * per_layer;
  // producer (thread 0): positions over (item, layer, stage); stage < kst: K stage, else D stage
  const bool producer = (tid == 0);
  int p_idx = blockIdx.x, p_s = 0;
  unsigned qp = 0;
  const int wm = warp >> 2, wn = warp & 3;
  const int g = lane >> 2, t = lane & 3;
  const int koff = ((t & 1) << 2) | (t >> 1);  // {0, 4, 1, 5}: conflict-free fragment loads (ngd_gemm.cu)
  unsigned q = 0;
  auto produce = [&](unsigned upto) {
    while (p_idx < n_items && qp < upto) {
      const int slot = qp % ANS;
      if (qp >= ANS) tma::wait(&empty[slot], ((qp / ANS) - 1) & 1u);
      const AItem it = decode_a(a, p_idx);
      const int c0 = (int)tile_col(a, it.nt);
      const int h = p_s / per_layer, s = p_s - h * per_layer;
      tma::expect_tx(&full[slot], sizeof(AStage));
      if (s < kst) {
        const int k0 = s * ABK;
        tma::load2d(st[slot].A, &maps.v[h], k0, it.mt * ABM, &full[slot]);
#pragma unroll
        for (int b = 0; b < ABN / 16; ++b) tma::load2d(st[slot].B + b * 256, &maps.z[h], c0 + b * 16, k0, &full[slot]);
      } else {
        const int r0 = it.mt * ABM + (s - kst) * 32;
#pragma unroll
        for (int b = 0; b < ABN / 16; ++b) tma::load2d(st[slot].A + b * 512, &maps.d[h], c0 + b * 16, r0, &full[slot]);
      }
      ++qp;
      if (++p_s >= per_item) {
        p_s = 0;
        p_idx += gridDim.x;
      }
    }
  };
  for (int idx = blockIdx.x; idx < n_items; idx += gridDim.x) {
    const AItem it = decode_a(a, idx);
    const int64_t c0 = tile_col(a, it.nt);
    const int ncol = tile_cols(a, it.nt);
    const bool interior = it.nt < a.int_tiles;
    double colsum[4][2];
    bool isval[4][2];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        colsum[j][e] = 0.0;
        const int64_t col = c0 + wn * 32 + j * 8 + 2 * t + e;
        isval[j][e] = !interior || ((col / PB) % a.C) == 0;
      }
    for (int h = 0; h < a.n_wide; ++h) {
      double acc[8][4][2];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      for (int s = 0; s < kst; ++s, ++q) {
        if (producer) produce(q + AAHEAD);
        __syncwarp();
        const int slot = q % ANS;
        tma::wait(&full[slot], (q / ANS) & 1u);
        const double* As = st[slot].A;
        const double* Bs = st[slot].B;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const int kk = ((ks & 1) << 1) + ((ks >> 1) << 3) + koff;
          double av[8], bv[4];
#pragma unroll
          for (int i = 0; i < 8; ++i) av[i] = As[tma::kmaj_off(wm * 64 + i * 8 + g, kk)];
#pragma unroll
          for (int j = 0; j < 4; ++j) bv[j] = Bs[mnmaj_off(wn * 32 + j * 8 + g, kk)];
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], av[i], bv[j]);
        }
        __syncwarp();
        if (lane == 0) tma::arrive(&empty[slot]);
      }
      // this layer's D stages: colsum += D o (P + vb [value column]) over this warp's 64 rows
      double vb[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int m = it.mt * ABM + wm * 64 + i * 8 + g;
        vb[i] = m < a.M ? a.vb[h][m] : 0.0;
      }
#pragma unroll
      for (int ds = 0; ds < kDStages; ++ds, ++q) {
        if (producer) produce(q + AAHEAD);
        __syncwarp();
        const int slot = q % ANS;
        tma::wait(&full[slot], (q / ANS) & 1u);
        if ((ds >> 1) == wm) {  // this 32-row D stage holds rows of this warp's half
          const double* Ds = st[slot].A;
#pragma unroll
          for (int ii = 0; ii < 4; ++ii) {
            const int i = (ds & 1) * 4 + ii;
            const int r = ii * 8 + g;  // row within the D stage
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const double pv = isval[j][e] ? acc[i][j][e] + vb[i] : acc[i][j][e];
                colsum[j][e] = fma(Ds[dstage_off(r, wn * 32 + j * 8 + 2 * t + e)], pv, colsum[j][e]);
              }
          }
        }
        __syncwarp();
        if (lane == 0) tma::arrive(&empty[slot]);
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double v = colsum[j][e];
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        if (g == 0) red[wm][wn * 32 + j * 8 + 2 * t + e] = v;
      }
    __syncthreads();
    // per point: the tile's channel runs of each point block (interior) or one column (boundary)
    double* part = a.part + (int64_t)(a.rowbase + it.mt * a.rows_per_mt) * a.n_pts_pad;
    if (interior) {
      const int bw = PB * a.C;                     // columns per point block
      const int64_t blk0 = c0 / bw;
      const int64_t blk1 = (c0 + ncol - 1) / bw;
      if (tid < (int)(blk1 - blk0 + 1) * PB) {
        const int64_t blk = blk0 + tid / PB;
        const int r = tid % PB;
        double s = 0.0;
        for (int run = 0; run < ncol / PB; ++run) {  // fixed order over the tile's runs
          const int64_t col = c0 + run * PB;
          if (col / bw == blk) s += red[0][run * PB + r] + red[1][run * PB + r];
        }
        const int row = it.nt - (int)((blk * bw) / ABN);  // tile index within the block's tiles
        part[(int64_t)row * a.n_pts_pad + blk * PB + r] = s;
      }
    } else if (tid < ncol) {
      part[a.nib * PB + (c0 - a.int_cols) + tid] = red[0][tid] + red[1][tid];
    }
    __syncthreads();  // red is reused by the next item
  }
}

namespace {
PFN_cuTensorMapEncodeTiled_v12000 enc_a() {
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
bool enc2d(CUtensorMap* m, const double* base, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t b0,
           uint32_t b1) {
  auto enc = enc_a();
  if (!enc) return false;
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {ld * sizeof(double)};
  const cuuint32_t box[2] = {b0, b1};
  const cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace

int phag_rows_per_mtile(int C) { return (112 + PB * C + ABN - 1) / ABN; }

cudaError_t phase_a_gemm(const PhagArgs& a, PhagCache& cache, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(phag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPhagSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  for (int h = 0; h < a.n_wide; ++h) {
    if (cache.kv[h] != cache.src_v[h] || cache.kz[h] != cache.src_z[h] || cache.kd[h] != cache.src_d[h] ||
        cache.ks[h] != a.s_pad) {
      // V_l: packed [Mp][Kp] (K-major, box 16 x 128); Zin_l: [Kp rows][s_pad] (box 16 cols x 16 rows);
      // D_l: [M rows][s_pad] (box 16 cols x 32 rows)
      if (!enc2d(&cache.maps.v[h], cache.src_v[h], a.Kp, a.Mp, a.Kp, 16, 128) ||
          !enc2d(&cache.maps.z[h], cache.src_z[h], a.s_pad, a.Kp, a.s_pad, 16, 16) ||
          !enc2d(&cache.maps.d[h], cache.src_d[h], a.s_pad, a.M, a.s_pad, 16, 32))
        return cudaErrorInvalidValue;
      cache.kv[h] = cache.src_v[h];
      cache.kz[h] = cache.src_z[h];
      cache.kd[h] = cache.src_d[h];
      cache.ks[h] = a.s_pad;
    }
  }
  const int items = a.n_tiles * a.mtiles;
  if (items <= 0) return cudaSuccess;
  probe_before(K_PHA, st);
  const cudaError_t e = launch_pdl(phag_kernel, dim3(std::min(items, 148)), dim3(kPhagWarps * 32), kPhagSmem, st, a,
                                   cache.maps);
  probe_after(K_PHA, st);
  return e;
}

}  // namespace ngd
