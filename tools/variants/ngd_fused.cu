// Fused Gramian matvec for narrow networks (all widths <= 64, <= 4 layers, <= 4 jet channels):
//   out = J^T diag(w) J v  computed point block by point block in ONE kernel.
//
// The factored matvec (ngd_jet.cu) runs phase A (J v), a per-point reduction, phase B
// (J^T c) and a split reduction as separate launches; at BASELINE C1/C2 sizes those
// launches are latency-bound (C2: ~65 us for 0.57 GFLOP, C1: ~38 us for 18 MFLOP).  Here a
// persistent CTA takes whole point blocks (16 points x C channels):
//   phase A  for every layer l: T = V_l Zin_l[:, blk] (+ v_b on value channels), column sums
//            of D_l o T  -> s_r (per point, summed over channels) -> c_r = w_r s_r
//   phase B  for every layer l: G_l += D_l diag(c) Zin_l[:, blk]^T (DMMA fragments held in
//            registers across the CTA's blocks), g_b += sum over value columns of D_l c
// and writes one parameter-space partial per CTA; reduce_splits / pcg_ad sum the partials in
// a fixed order (bitwise deterministic).  V_l is read straight from the flat p-vector into
// shared memory once per CTA; each block's jets are staged twice (phase A and phase B, L2 hits
// the second time) with cp.async double buffering.
#include "ngd_common.cuh"
#include "ngd_kernels.h"

namespace ngd {

constexpr int FW = 64;          // max width
constexpr int FNCS = 68;        // staged jet row stride: (4 g + t) distinct banks for DMMA fragments
constexpr int FL = 4;           // max layers
constexpr int FJ = 8;           // max phase-B tiles per warp per layer (64 x 64 / 64 / 8 warps)
constexpr int kFusedThreads = 256;

__device__ __forceinline__ void cpa16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cpa_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

__device__ __forceinline__ int rup8(int x) { return (x + 7) & ~7; }
__device__ __forceinline__ int rup4(int x) { return (x + 3) & ~3; }

// stage Zin_l rows [0, rup8(n_in)) and D_l rows [0, rup8(n_out)) of columns [col0, col0 + nc)
__device__ __forceinline__ void stage_layer(const FusedArgs& a, int l, int64_t col0, int nc, double* Zs, double* Ds) {
  const int zr = rup8(a.n_in[l]), dr = rup8(a.n_out[l]);
  const int per_row = nc >> 1;  // 16-byte chunks per row (<= 32: one per lane)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane < per_row) {
    for (int row = warp; row < zr + dr; row += kFusedThreads / 32) {
      if (row < zr) {
        cpa16(Zs + row * FNCS + 2 * lane, a.Z[l] + (int64_t)row * a.s_pad + col0 + 2 * lane);
      } else {
        const int r = row - zr;
        cpa16(Ds + r * FNCS + 2 * lane, a.D[l] + (int64_t)r * a.s_pad + col0 + 2 * lane);
      }
    }
  }
  cpa_commit();
}

__global__ void __launch_bounds__(kFusedThreads, 1) fused_mv_kernel(FusedArgs a) {
  if (a.skip && *a.skip) return;
  extern __shared__ __align__(16) double fsm[];
  double* Vs = fsm;                          // per layer [rup8(n_out)][vs_l], then biases
  double* stage = fsm + a.v_total;           // 2 x (Zs [FW][FNCS] + Ds [FW][FNCS])
  double* colsum = stage + 4 * FW * FNCS;    // [64]
  double* ccol = colsum + 64;                // [64] cotangent per column
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int NL = a.n_layers;

  // V_l (row-major W-shaped block of v) and v_b into shared memory, zero padded
  for (int l = 0; l < NL; ++l) {
    const int M = a.n_out[l], K = a.n_in[l], vs = a.vs[l], mr = rup8(M);
    double* V = Vs + a.vso[l];
    for (int m = warp; m < mr; m += kFusedThreads / 32) {  // warp per row, lanes over k (coalesced)
      const double* src = a.v + a.woff[l] + (int64_t)m * K;
      for (int k = lane; k < vs; k += 32) V[m * vs + k] = (m < M && k < K) ? __ldg(src + k) : 0.0;
    }
    double* vb = Vs + a.vbo[l];
    for (int m = tid; m < mr; m += kFusedThreads) vb[m] = (m < M) ? a.v[a.boff[l] + m] : 0.0;
  }

  double acc[FL][FJ][2];
#pragma unroll
  for (int l = 0; l < FL; ++l)
#pragma unroll
    for (int j = 0; j < FJ; ++j) acc[l][j][0] = acc[l][j][1] = 0.0;
  double bacc[FL];
#pragma unroll
  for (int l = 0; l < FL; ++l) bacc[l] = 0.0;

  const int nblk = a.nib + a.nbb;
  int buf = 0;
  // prologue: first block, layer 0 (phase A)
  int b = blockIdx.x;
  if (b < nblk) {
    const bool inte = b < a.nib;
    stage_layer(a, 0, inte ? (int64_t)b * PB * a.C : a.int_cols + (int64_t)(b - a.nib) * PB, inte ? PB * a.C : PB,
                stage, stage + FW * FNCS);
  }
  for (; b < nblk; b += gridDim.x) {
    const bool inte = b < a.nib;
    const int nc = inte ? PB * a.C : PB;
    const int64_t col0 = inte ? (int64_t)b * PB * a.C : a.int_cols + (int64_t)(b - a.nib) * PB;
    const int pt0 = b * PB;
    double cs0 = 0.0, cs1 = 0.0;  // phase-A column sums of this warp's two fragment columns
    for (int st = 0; st < 2 * NL; ++st) {
      const bool phase_b = st >= NL;
      const int l = phase_b ? st - NL : st;
      double* Zs = stage + buf * 2 * FW * FNCS;
      double* Ds = Zs + FW * FNCS;
      // prefetch the next stage (the next layer, phase B's reload, or the next block's layer 0)
      {
        const int nst = st + 1;
        double* Zn = stage + (buf ^ 1) * 2 * FW * FNCS;
        if (nst < 2 * NL) {
          stage_layer(a, nst >= NL ? nst - NL : nst, col0, nc, Zn, Zn + FW * FNCS);
        } else if (b + (int)gridDim.x < nblk) {
          const int b2 = b + gridDim.x;
          const bool i2 = b2 < a.nib;
          stage_layer(a, 0, i2 ? (int64_t)b2 * PB * a.C : a.int_cols + (int64_t)(b2 - a.nib) * PB, i2 ? PB * a.C : PB,
                      Zn, Zn + FW * FNCS);
        } else {
          cpa_commit();  // empty group keeps "wait_group 1" meaning "this stage has landed"
        }
      }
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
      __syncthreads();
      const int M = a.n_out[l], K = a.n_in[l];
      const int mr = rup8(M), kr4 = rup4(K), kr8 = rup8(K);
      if (!phase_b) {
        // ---- phase A: warp w owns fragment columns [8w, 8w + 8) of the block
        if (warp * 8 < nc) {
          const double* V = Vs + a.vso[l];
          const double* vb = Vs + a.vbo[l];
          const int vs = a.vs[l];
          const int colb = warp * 8;
          const bool value_cols = !inte || colb < PB;  // channel 0 = value (bias applies)
          // all (<= 8) row tiles at once: independent DMMA chains overlap their latency
          double d[FW / 8][2];
#pragma unroll
          for (int mt = 0; mt < FW / 8; ++mt) d[mt][0] = d[mt][1] = 0.0;
          for (int k0 = 0; k0 < kr4; k0 += 4) {
            const double bz = Zs[(k0 + t) * FNCS + colb + g];
#pragma unroll
            for (int mt = 0; mt < FW / 8; ++mt)
              if (mt * 8 < mr) dmma884(d[mt][0], d[mt][1], V[(mt * 8 + g) * vs + k0 + t], bz);
          }
#pragma unroll
          for (int mt = 0; mt < FW / 8; ++mt) {
            if (mt * 8 < mr) {
              double d0 = d[mt][0], d1 = d[mt][1];
              if (value_cols) {
                const double bb = vb[mt * 8 + g];
                d0 += bb;
                d1 += bb;
              }
              const double* drow = Ds + (mt * 8 + g) * FNCS + colb + 2 * t;
              cs0 = fma(drow[0], d0, cs0);
              cs1 = fma(drow[1], d1, cs1);
            }
          }
        }
        if (l == NL - 1) {
          // column sums over the 8 fragment rows (lanes with equal t), then per point over channels
#pragma unroll
          for (int o = 4; o < 32; o <<= 1) {
            cs0 += __shfl_xor_sync(0xffffffffu, cs0, o);
            cs1 += __shfl_xor_sync(0xffffffffu, cs1, o);
          }
          if (warp * 8 < nc && g == 0) {
            colsum[warp * 8 + 2 * t] = cs0;
            colsum[warp * 8 + 2 * t + 1] = cs1;
          }
          __syncthreads();
          if (tid < PB) {
            const int nch = inte ? a.C : 1;
            double s = 0.0;
            for (int ch = 0; ch < nch; ++ch) s += colsum[ch * PB + tid];
            const double cr = a.w[pt0 + tid] * s;
            for (int ch = 0; ch < nch; ++ch) ccol[ch * PB + tid] = cr;
          }
        }
      } else {
        // ---- phase B: G_l += (D_l diag(c)) Zin_l^T over this block's columns
        const int nmt = mr >> 3, nkt = kr8 >> 3, ntile = nmt * nkt;
        int doff[FJ], zoff[FJ];  // fragment row offsets of this warp's tiles (no division in the loop)
#pragma unroll
        for (int j = 0; j < FJ; ++j) {
          const int tile = min(warp + 8 * j, ntile - 1);
          const int mt = tile / nkt, kt = tile - mt * nkt;
          doff[j] = (mt * 8 + g) * FNCS + t;
          zoff[j] = (kt * 8 + g) * FNCS + t;
        }
#pragma unroll
        for (int ll = 0; ll < FL; ++ll) {
          if (ll != l) continue;
          // columns outer, this warp's (<= 8) tiles inner: independent DMMA chains
          for (int c0 = 0; c0 < nc; c0 += 4) {
            const double cc = ccol[c0 + t];
#pragma unroll
            for (int j = 0; j < FJ; ++j) {
              if (warp + 8 * j < ntile)
                dmma884(acc[ll][j][0], acc[ll][j][1], Ds[doff[j] + c0] * cc, Zs[zoff[j] + c0]);
            }
          }
          if (tid < M) {  // bias: value columns only
            const double* drow = Ds + tid * FNCS;
            double s = bacc[ll];
            for (int cc = 0; cc < PB; ++cc) s = fma(drow[cc], ccol[cc], s);
            bacc[ll] = s;
          }
        }
      }
      __syncthreads();  // stage buffer free for the prefetch two stages ahead
      buf ^= 1;
    }
  }
  cpa_wait_all();
  // per-CTA partial in the flat parameter layout (model.py:41-51)
  double* part = a.part + (int64_t)blockIdx.x * a.p;
#pragma unroll
  for (int l = 0; l < FL; ++l) {
    if (l >= NL) break;
    const int M = a.n_out[l], K = a.n_in[l];
    const int nkt = rup8(K) >> 3, ntile = (rup8(M) >> 3) * nkt;
#pragma unroll
    for (int j = 0; j < FJ; ++j) {
      const int tile = warp + 8 * j;
      if (tile < ntile) {
        const int mt = tile / nkt, kt = tile - mt * nkt;
        const int m = mt * 8 + g, k = kt * 8 + 2 * t;
        if (m < M && k < K) part[a.woff[l] + (int64_t)m * K + k] = acc[l][j][0];
        if (m < M && k + 1 < K) part[a.woff[l] + (int64_t)m * K + k + 1] = acc[l][j][1];
      }
    }
    if (tid < M) part[a.boff[l] + tid] = bacc[l];
  }
}

bool fused_supported(const int* widths, int n_layers, int C) {
  if (n_layers < 1 || n_layers > FL || C > 4) return false;
  for (int l = 0; l <= n_layers; ++l)
    if (widths[l] < 1 || widths[l] > FW) return false;
  return true;
}

size_t fused_smem(const FusedArgs& a) {
  return sizeof(double) * ((size_t)a.v_total + 4 * FW * FNCS + 128);
}

cudaError_t fused_mv(const FusedArgs& a, int grid, cudaStream_t st) {
  const size_t smem = fused_smem(a);
  static size_t attr = 0;
  if (smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(fused_mv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = smem;
  }
  probe_before(K_FUSED, st);
  fused_mv_kernel<<<grid, kFusedThreads, smem, st>>>(a);
  probe_after(K_FUSED, st);
  return cudaGetLastError();
}

}  // namespace ngd
