// Phase A of the factored Gramian matvec on the DMMA GEMM core, for the wide layers (both sides
// >= 256: C4 / C5's hidden layers):
//     (J v)_r += sum_c < D_l[:, (r,c)], V_l Zin_l[:, (r,c)] + [c = value] vb_l >
// (the J v half of gramian.py:48-53, autodiff.py:90-125; layout in ngd_common.cuh).
//
// T = V_l Zin_l is a GEMM with M = n_l, N = S channel-columns, K = n_{l-1} = 256.  Same pipeline
// as ngd_gemm.cu / ngd_phbg.cu -- persistent CTAs, 128 x 128 tiles, 16-deep k-stages streamed by
// TMA (V_l K-major: one 16 x 128 box; Zin_l MN-major: eight 16 x 16 boxes; 128-byte swizzle)
// through a 6-deep mbarrier ring, eight DMMA warps of 64 x 32, lane 0 of warp 0 issuing four
// stages ahead.  The epilogue operand D_l travels through the same ring: after an item's 16
// k-stages come four "D stages" (two 16 x 128 boxes each = 32 columns of the tile's 128 rows), so
// the adjoint tile is in shared memory when the accumulators are done and the next item's operands
// are already in flight.  Warp (wm, wn) dots its 64 x 32 accumulator block with D on D stage wn
// and writes the 32 column sums of its 64 rows into colpart[(layer, m tile, wm)][column]; the
// reduction kernel (reduce_pha_cols, ngd_vec.cu) sums the point's channel columns and the rows in
// fixed order (bitwise deterministic, no atomics).  Items run m-tile fastest: the two m tiles of
// one column range are adjacent CTAs and share the Zin panel in L2.
//
// Replaces the 64-row x one-point-block tiles of pha_all_kernel (ngd_jet.cu: cp.async double
// buffer, D read from global memory in the epilogue) on these layers; the thin input / output
// layers stay there.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>

#include "ngd_common.cuh"
#include "ngd_kernels.h"
#include "ngd_tma.cuh"

namespace ngd {

namespace {
constexpr int ABM = 128, ABN = 128, ABK = 16;
#ifndef PHAG_NS
#define PHAG_NS 6
#endif
#ifndef PHAG_AHEAD
#define PHAG_AHEAD 4
#endif
#ifndef PHAG_PF
#define PHAG_PF 0  // bit 0: L2 prefetch of the item's D tile, bit 1: of the next item's first Zin stages
#endif
#ifndef PHAG_DG
#define PHAG_DG 0  // 1: the epilogue reads D from global memory (L2) instead of ring D stages
#endif
constexpr int ANS = PHAG_NS, AAHEAD = PHAG_AHEAD;
constexpr int kPhagWarps = 8;
constexpr int kDStages = PHAG_DG ? 0 : ABN / 32;  // D stages per item (one per warp column)

struct __align__(1024) AStage {
  double A[ABM * ABK];  // k-stage: V_l rows m0 .. m0+127, 16 k     | D stage: D_l columns +0 .. +15
  double B[ABN * ABK];  // k-stage: Zin_l k rows, 128 columns (MN) | D stage: D_l columns +16 .. +31
};
constexpr size_t kPhagSmem = sizeof(AStage) * ANS + 2 * ANS * sizeof(unsigned long long) + 1024;

// element (mn, k) of the MN-major stage tile: eight [16 k][16 mn] boxes, 128-byte swizzle
__device__ __forceinline__ int mn_off(int mn, int k) {
  return (mn >> 4) * 256 + k * 16 + (((((mn & 15) >> 1) ^ (k & 7)) << 1) | (mn & 1));
}

// L2 prefetch of one TMA box (no shared-memory destination, no completion)
__device__ __forceinline__ void prefetch2d(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1)
               : "memory");
}

struct AItem {
  int h, tm, tn;
};
__device__ __forceinline__ AItem decode_a(const PhagArgs& a, int idx) {
  AItem it;
  int h = 0;
  while (h + 1 < a.n_heavy && idx >= a.item_start[h + 1]) ++h;
  const int r = idx - a.item_start[h];
  it.h = h;
  it.tn = r / a.tiles_m[h];
  it.tm = r - it.tn * a.tiles_m[h];
  return it;
}
}  // namespace

#ifndef PHAG_KORD
#define PHAG_KORD 2  // fragment k order (see ngd_phbg.cu)
#endif
#ifndef PHAG_WS
#define PHAG_WS 1  // 1: a producer warpgroup issues the TMA ring (setmaxnreg; see ngd_phbg.cu)
#endif
#if PHAG_WS
constexpr int kPhagThreads = (kPhagWarps + 4) * 32;
static_assert(!PHAG_DG && !PHAG_PF, "the warp-specialised form streams D through the ring");
// The producer refills a slot as soon as its eighth consumer warp has arrived, so the consumers order
// their shared-memory reads (generic proxy) before the refill (async proxy) with fence.proxy.async ahead
// of the arrive.  Measured without it (tools/ws_stress.py, C5): one stale 16-column box -- one point
// block of J v off by 1e-4 .. 3e-3 -- in ~10% of the launches; with it 0 in 100 (the single-role form
// never refilled a slot less than two stages after its release).
__global__ void __launch_bounds__(kPhagThreads, 1) phag_kernel(const __grid_constant__ PhagArgs a,
                                                               const __grid_constant__ PhagMaps maps) {
  pdl_entry();  // (PCG chain: programmatic dependent launch)
  if (a.skip && *a.skip) return;
  extern __shared__ unsigned char asm_raw[];
  unsigned char* base = asm_raw + ((1024u - (tma::smem(asm_raw) & 1023u)) & 1023u);
  AStage* st = reinterpret_cast<AStage*>(base);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(st + ANS);
  unsigned long long* empty = full + ANS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < ANS; ++s) {
      tma::mbar_init(&full[s], 1);
      tma::mbar_init(&empty[s], kPhagWarps);
    }
    tma::fence_init();
  }
  __syncthreads();
  const int n_items = a.item_start[a.n_heavy];
  if (warp >= kPhagWarps) {  // producer warpgroup: units 0 .. ks-1 of an item are k-stages, then its D stages
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n");
    if (warp == kPhagWarps && lane == 0) {
      unsigned qp = 0;
      for (int idx = blockIdx.x; idx < n_items; idx += gridDim.x) {
        const AItem it = decode_a(a, idx);
        const int ks = a.Kp[it.h] / ABK, m0 = it.tm * ABM, n0 = it.tn * ABN;
        for (int u = 0; u < ks + kDStages; ++u, ++qp) {
          const int slot = qp % ANS;
          if (qp >= ANS) tma::wait(&empty[slot], ((qp / ANS) - 1) & 1u);
          tma::expect_tx(&full[slot], (ABM + ABN) * ABK * sizeof(double));
          if (u < ks) {
            const int k0 = u * ABK;
            tma::load2d(st[slot].A, &maps.v[it.h], k0, m0, &full[slot]);
#pragma unroll
            for (int b = 0; b < ABN / 16; ++b)
              tma::load2d(st[slot].B + b * 256, &maps.z[it.h], n0 + b * 16, k0, &full[slot]);
          } else {
            const int c0 = n0 + (u - ks) * 32;
            tma::load2d(st[slot].A, &maps.d[it.h], c0, m0, &full[slot]);
            tma::load2d(st[slot].B, &maps.d[it.h], c0 + 16, m0, &full[slot]);
          }
        }
      }
    }
    return;
  }
  asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n");
  const int wm = warp >> 2, wn = warp & 3;
  const int g = lane >> 2, t = lane & 3;
#if PHAG_KORD == 2
  const int koff = ((t & 1) * 10) ^ ((t >> 1) * 5);  // {0, 10, 5, 15}: bank-conflict-free half-warps (ngd_phbg.cu)
#else
  const int koff = ((t & 1) << 2) | (t >> 1);  // {0, 4, 1, 5}
#endif
  unsigned q = 0;
  for (int idx = blockIdx.x; idx < n_items; idx += gridDim.x) {
    const AItem it = decode_a(a, idx);
    const int ks = a.Kp[it.h] / ABK;
    double acc[8][4][2];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int s = 0; s < ks; ++s, ++q) {
      const int slot = q % ANS;
      tma::wait(&full[slot], (q / ANS) & 1u);
      const double* As = st[slot].A;
      const double* Bs = st[slot].B;
#pragma unroll
      for (int kq = 0; kq < 4; ++kq) {
#if PHAG_KORD == 2
        const int kk = (kq << 1) ^ koff;
#else
        const int kk = ((kq & 1) << 1) + ((kq >> 1) << 3) + koff;  // kbase {0, 2, 8, 10}
#endif
        double av[8], bv[4];
#pragma unroll
        for (int i = 0; i < 8; ++i) av[i] = As[tma::kmaj_off(wm * 64 + i * 8 + g, kk)];
#pragma unroll
        for (int j = 0; j < 4; ++j) bv[j] = Bs[mn_off(wn * 32 + j * 8 + g, kk)];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], av[i], bv[j]);
      }
      tma::fence_proxy_async();  // generic-proxy reads of the slot before the producer's async-proxy refill
     __syncwarp();
      if (lane == 0) tma::arrive(&empty[slot]);
    }
    // epilogue: bias of the value-channel columns, dot with D over this warp's 64 rows
    const int M = a.M[it.h];
    const int mrow = it.tm * ABM + wm * 64 + g;
    double vb[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) vb[i] = (mrow + i * 8 < M) ? __ldg(&a.vbias[it.h][mrow + i * 8]) : 0.0;
    const int64_t ncol = (int64_t)it.tn * ABN + wn * 32;
    bool val[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t run = (ncol + j * 8) >> 4;
      val[j] = run >= a.int_units || (run % a.C) == 0;
    }
    double cs[4][2];
#pragma unroll
    for (int j = 0; j < 4; ++j) cs[j][0] = cs[j][1] = 0.0;
    if (PHAG_DG) {
      const int64_t s_pad = a.s_pad;
      const double* Dg = a.dptr[it.h] + (int64_t)mrow * s_pad + ncol + 2 * t;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (ncol + j * 8 >= s_pad) break;
        double2 dv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
          dv[i] = (mrow + i * 8 < M) ? __ldcg(reinterpret_cast<const double2*>(Dg + (int64_t)i * 8 * s_pad + j * 8))
                                     : make_double2(0.0, 0.0);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const double b = val[j] ? vb[i] : 0.0;
          cs[j][0] = fma(dv[i].x, acc[i][j][0] + b, cs[j][0]);
          cs[j][1] = fma(dv[i].y, acc[i][j][1] + b, cs[j][1]);
        }
      }
    }
    for (int dq = 0; dq < kDStages; ++dq, ++q) {
      const int slot = q % ANS;
      tma::wait(&full[slot], (q / ANS) & 1u);
      if (dq == wn) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const double* Db = (j < 2) ? st[slot].A : st[slot].B;
          const int kin = (j & 1) * 8 + 2 * t;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const double2 dv = *reinterpret_cast<const double2*>(Db + tma::kmaj_off(wm * 64 + i * 8 + g, kin));
            const double b = val[j] ? vb[i] : 0.0;
            cs[j][0] = fma(dv.x, acc[i][j][0] + b, cs[j][0]);
            cs[j][1] = fma(dv.y, acc[i][j][1] + b, cs[j][1]);
          }
        }
      }
      tma::fence_proxy_async();  // generic-proxy reads of the slot before the producer's async-proxy refill
     __syncwarp();
      if (lane == 0) tma::arrive(&empty[slot]);
    }
    // fixed xor tree over the eight row groups g, then lanes g = 0 store their two columns per j
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double v = cs[j][e];
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        cs[j][e] = v;
      }
    if (g == 0) {
      double* row = a.colpart + (int64_t)(a.slot0[it.h] + it.tm * 2 + wm) * a.s_pad;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t n = ncol + j * 8 + 2 * t;
        if (n + 1 < a.s_pad) {
          *reinterpret_cast<double2*>(row + n) = make_double2(cs[j][0], cs[j][1]);
        } else if (n < a.s_pad) {
          row[n] = cs[j][0];
        }
      }
    }
  }
}

#else
constexpr int kPhagThreads = kPhagWarps * 32;
__global__ void __maxnreg__(224) phag_kernel(const __grid_constant__ PhagArgs a, const __grid_constant__ PhagMaps maps) {
  pdl_entry();  // (PCG chain: programmatic dependent launch)
  if (a.skip && *a.skip) return;
  extern __shared__ unsigned char asm_raw[];
  unsigned char* base = asm_raw + ((1024u - (tma::smem(asm_raw) & 1023u)) & 1023u);
  AStage* st = reinterpret_cast<AStage*>(base);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(st + ANS);
  unsigned long long* empty = full + ANS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < ANS; ++s) {
      tma::mbar_init(&full[s], 1);
      tma::mbar_init(&empty[s], kPhagWarps);
    }
    tma::fence_init();
  }
  __syncthreads();
  const int n_items = a.item_start[a.n_heavy];
  // producer cursor (thread 0): units 0 .. ks-1 are k-stages, ks .. ks+3 the D stages of the item
  const bool producer = (tid == 0);
  int p_idx = blockIdx.x, p_u = 0, p_ks = 0, p_h = 0, p_m0 = 0, p_n0 = 0;
  bool p_valid = false;
  auto p_load = [&]() {
    if (p_idx >= n_items) return false;
    const AItem it = decode_a(a, p_idx);
    p_u = 0;
    p_h = it.h;
    p_ks = a.Kp[it.h] / ABK;
    p_m0 = it.tm * ABM;
    p_n0 = it.tn * ABN;
    return true;
  };
  if (producer) p_valid = p_load();
  unsigned qp = 0;
  auto produce = [&](unsigned q) {
    while (p_valid && qp < q + AAHEAD) {
      const int slot = qp % ANS;
      if (qp >= ANS) tma::wait(&empty[slot], ((qp / ANS) - 1) & 1u);
      tma::expect_tx(&full[slot], (ABM + ABN) * ABK * sizeof(double));
      if ((PHAG_PF & 1) && p_u == 0) {
        // the item's D tile (needed after its k-stages) and, further below, the next item's first
        // Zin stages: the D stages and the next item's start otherwise wait on DRAM right after the
        // ring's lookahead shrank to the few cycles of the epilogue
#pragma unroll
        for (int b = 0; b < ABN / 16; ++b) prefetch2d(&maps.d[p_h], p_n0 + b * 16, p_m0);
      }
      if ((PHAG_PF & 2) && p_u == p_ks / 2 && p_idx + (int)gridDim.x < n_items) {
        const AItem nx = decode_a(a, p_idx + gridDim.x);
#pragma unroll 1
        for (int k = 0; k < 2; ++k)
#pragma unroll
          for (int b = 0; b < ABN / 16; ++b) prefetch2d(&maps.z[nx.h], nx.tn * ABN + b * 16, k * ABK);
      }
      if (p_u < p_ks) {
        const int k0 = p_u * ABK;
        tma::load2d(st[slot].A, &maps.v[p_h], k0, p_m0, &full[slot]);
#pragma unroll
        for (int b = 0; b < ABN / 16; ++b) tma::load2d(st[slot].B + b * 256, &maps.z[p_h], p_n0 + b * 16, k0, &full[slot]);
      } else {
        const int c0 = p_n0 + (p_u - p_ks) * 32;
        tma::load2d(st[slot].A, &maps.d[p_h], c0, p_m0, &full[slot]);
        tma::load2d(st[slot].B, &maps.d[p_h], c0 + 16, p_m0, &full[slot]);
      }
      ++qp;
      if (++p_u >= p_ks + kDStages) {
        p_idx += gridDim.x;
        p_valid = p_load();
      }
    }
  };
  const int wm = warp >> 2, wn = warp & 3;
  const int g = lane >> 2, t = lane & 3;
  const int koff = ((t & 1) << 2) | (t >> 1);  // {0, 4, 1, 5}: conflict-free fragment loads (ngd_gemm.cu)
  unsigned q = 0;
  for (int idx = blockIdx.x; idx < n_items; idx += gridDim.x) {
    const AItem it = decode_a(a, idx);
    const int ks = a.Kp[it.h] / ABK;
    double acc[8][4][2];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int s = 0; s < ks; ++s, ++q) {
      if (producer) produce(q);
      __syncwarp();
      const int slot = q % ANS;
      tma::wait(&full[slot], (q / ANS) & 1u);
      const double* As = st[slot].A;
      const double* Bs = st[slot].B;
#pragma unroll
      for (int kq = 0; kq < 4; ++kq) {
        const int kk = ((kq & 1) << 1) + ((kq >> 1) << 3) + koff;  // kbase {0, 2, 8, 10}
        double av[8], bv[4];
#pragma unroll
        for (int i = 0; i < 8; ++i) av[i] = As[tma::kmaj_off(wm * 64 + i * 8 + g, kk)];
#pragma unroll
        for (int j = 0; j < 4; ++j) bv[j] = Bs[mn_off(wn * 32 + j * 8 + g, kk)];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], av[i], bv[j]);
      }
      tma::fence_proxy_async();
      __syncwarp();
      if (lane == 0) tma::arrive(&empty[slot]);
    }
    // epilogue: bias of the value-channel columns, dot with D over this warp's 64 rows
    const int M = a.M[it.h];
    const int mrow = it.tm * ABM + wm * 64 + g;
    double vb[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) vb[i] = (mrow + i * 8 < M) ? __ldg(&a.vbias[it.h][mrow + i * 8]) : 0.0;
    const int64_t ncol = (int64_t)it.tn * ABN + wn * 32;
    bool val[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t run = (ncol + j * 8) >> 4;
      val[j] = run >= a.int_units || (run % a.C) == 0;
    }
    double cs[4][2];
#pragma unroll
    for (int j = 0; j < 4; ++j) cs[j][0] = cs[j][1] = 0.0;
    if (PHAG_DG) {
      const int64_t s_pad = a.s_pad;
      const double* Dg = a.dptr[it.h] + (int64_t)mrow * s_pad + ncol + 2 * t;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (ncol + j * 8 >= s_pad) break;
        double2 dv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
          dv[i] = (mrow + i * 8 < M) ? __ldcg(reinterpret_cast<const double2*>(Dg + (int64_t)i * 8 * s_pad + j * 8))
                                     : make_double2(0.0, 0.0);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const double b = val[j] ? vb[i] : 0.0;
          cs[j][0] = fma(dv[i].x, acc[i][j][0] + b, cs[j][0]);
          cs[j][1] = fma(dv[i].y, acc[i][j][1] + b, cs[j][1]);
        }
      }
    }
    for (int dq = 0; dq < kDStages; ++dq, ++q) {
      if (producer) produce(q);
      __syncwarp();
      const int slot = q % ANS;
      tma::wait(&full[slot], (q / ANS) & 1u);
      if (dq == wn) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const double* Db = (j < 2) ? st[slot].A : st[slot].B;
          const int kin = (j & 1) * 8 + 2 * t;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const double2 dv = *reinterpret_cast<const double2*>(Db + tma::kmaj_off(wm * 64 + i * 8 + g, kin));
            const double b = val[j] ? vb[i] : 0.0;
            cs[j][0] = fma(dv.x, acc[i][j][0] + b, cs[j][0]);
            cs[j][1] = fma(dv.y, acc[i][j][1] + b, cs[j][1]);
          }
        }
      }
      tma::fence_proxy_async();
      __syncwarp();
      if (lane == 0) tma::arrive(&empty[slot]);
    }
    // fixed xor tree over the eight row groups g, then lanes g = 0 store their two columns per j
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double v = cs[j][e];
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        cs[j][e] = v;
      }
    if (g == 0) {
      double* row = a.colpart + (int64_t)(a.slot0[it.h] + it.tm * 2 + wm) * a.s_pad;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t n = ncol + j * 8 + 2 * t;
        if (n + 1 < a.s_pad) {
          *reinterpret_cast<double2*>(row + n) = make_double2(cs[j][0], cs[j][1]);
        } else if (n < a.s_pad) {
          row[n] = cs[j][0];
        }
      }
    }
  }
}

#endif

namespace {
PFN_cuTensorMapEncodeTiled_v12000 enc_fn_a() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}
// row-major [rows][ld] doubles, box (bx columns, by rows), 128-byte swizzle, out-of-range zero-filled
bool encode_rm(CUtensorMap* m, const double* base, int64_t cols, int64_t rows, int64_t ld, int bx, int by) {
  auto enc = enc_fn_a();
  if (!enc) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(double)};
  const cuuint32_t box[2] = {(cuuint32_t)bx, (cuuint32_t)by};
  const cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace

cudaError_t phase_a_gemm(const PhagArgs& a, PhagCache& cache, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(phag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPhagSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  for (int h = 0; h < a.n_heavy; ++h) {
    if (cache.kv[h] != cache.src_v[h] || cache.kz[h] != cache.src_z[h] || cache.kd[h] != cache.src_d[h] ||
        cache.ks[h] != cache.s_pad) {
      if (!encode_rm(&cache.maps.v[h], cache.src_v[h], a.Kp[h], cache.mp[h], a.Kp[h], ABK, ABM) ||
          !encode_rm(&cache.maps.z[h], cache.src_z[h], cache.s_pad, a.Kp[h], cache.s_pad, 16, ABK) ||
          !encode_rm(&cache.maps.d[h], cache.src_d[h], cache.s_pad, a.M[h], cache.s_pad, 16, ABM))
        return cudaErrorInvalidValue;
      cache.kv[h] = cache.src_v[h];
      cache.kz[h] = cache.src_z[h];
      cache.kd[h] = cache.src_d[h];
      cache.ks[h] = cache.s_pad;
    }
  }
  const int items = a.item_start[a.n_heavy];
  if (items <= 0) return cudaSuccess;
  probe_before(K_PHA, st);
  const cudaError_t e =
      launch_pdl(phag_kernel, dim3(std::min(items, 148)), dim3(kPhagThreads), kPhagSmem, st, a, cache.maps);
  probe_after(K_PHA, st);
  return e;
}

}  // namespace ngd
