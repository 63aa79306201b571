// Phase A of the factored Gramian matvec, persistent TMA-pipelined form (option "pha_plan" = 1; NOT the
// default -- measured slower than the first form in ngd_jet.cu, see "Measured" below):
//     partA[(l, m-tile)][pt] = sum_{rows a of the tile} sum_c D_l[a][(pt, c)] (V_l Zin_l + vb_l)[a][(pt, c)]
// i.e. the J v half of gramian.py:48-53 (restated in ngd_jet.cu's header).
//
// The first form launched one 256-thread CTA per (layer, 64-row tile, 16-point block) -- 1152
// CTAs at C2, each loading its 64 x Kp slice of V and a Kp x 16C slice of Zin for only 1024
// DMMAs, so most of its life was pipeline fill (21 us for ~8 us of tensor-core work).  Here one
// persistent CTA per SM walks a contiguous, cost-balanced range of those units:
//   * warp 0 lane 0 streams every (unit, k-chunk) through a 2-deep ring with TMA: one 3-D box of
//     V_l ({16, 64 rows, KC/16}) and one of Zin_l ({16, C channel runs, KC rows}), 128-byte
//     swizzle, completion on "full" mbarriers, refilled once all warps released the slot;
//   * eight consumer warps (2 row halves x 2 point halves x 2 k-groups, all C channels) run the
//     DMMAs and fold each finished unit into per-point partials; the unit's D tile is copied to
//     shared memory by coalesced cp.async while the MMAs run; the partials are summed in
//     fixed order (deterministic) behind one named barrier per unit.
// Measured (C2, B200, ncu --cache-control none): 42-46 us vs 21 us for the first form, and 25-30
// us with the MMAs compiled out -- the kernel is bound by its operand traffic, not the tensor
// pipe: every unit re-streams its 32 KB V tile (37 MB per matvec, as in the first form), plus Zin
// and D (~54 MB), and 148 CTAs sustain ~3.7 TB/s of it where the first form's 1152 small CTAs
// reach ~5.3 TB/s.  Kept as an option for that reason; the route to a faster phase A is to stop
// re-reading D and Zin altogether (fusing phase A and B per point block), not a better pipeline.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <type_traits>

#include "ngd_common.cuh"
#include "ngd_kernels.h"

namespace ngd {

#ifdef NGD_PHA2_TRACE
__device__ unsigned long long g_a2tr[1024][4];  // per CTA: start ns, end ns, units, consumer wait cycles
#endif

namespace {
constexpr int AB = 64;   // rows of a unit (m-tile)
constexpr int AK = 16;   // doubles per 128-byte row of a box
// k-chunk of a stage (rows of Zin / columns of V), by channel count so that two ring slots plus the
// double-buffered D tile fit in shared memory
template <int C>
constexpr int kc_max() { return C <= 4 ? 64 : (C <= 7 ? 32 : 16); }
__host__ __device__ constexpr int kc_max_rt(int C) { return C <= 4 ? 64 : (C <= 7 ? 32 : 16); }
constexpr int ANS = 2;  // ring depth
constexpr int kAConsumers = 8;  // two per SM sub-partition; warp 0 lane 0 also issues the TMA stream
constexpr int kPha2Threads = kAConsumers * 32;
template <int C>
constexpr size_t v_bytes() { return sizeof(double) * AB * kc_max<C>(); }  // V box {16, 64, KC/16}
template <int C>
constexpr size_t z_bytes() { return sizeof(double) * kc_max<C>() * AK * C; }  // Zin box {16, C, KC}
template <int C>
constexpr size_t stage_bytes() { return (v_bytes<C>() + z_bytes<C>() + 1023) & ~size_t(1023); }
template <int C>
constexpr int dstride() { return PB * C + 4; }  // D tile row stride (doubles) in shared memory
template <int C>
constexpr size_t d_bytes() { return sizeof(double) * 2 * AB * dstride<C>(); }  // [2 parity][64][stride]
template <int C>
constexpr size_t pha2_smem_bytes() {
  return 1024 + ANS * stage_bytes<C>() + d_bytes<C>() + 2 * ANS * sizeof(unsigned long long) +
         2 * 4 * PB * sizeof(double);
}

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void minit(unsigned long long* m, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(m)), "r"(c));
}
__device__ __forceinline__ void mexpect(unsigned long long* m, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void marrive(unsigned long long* m) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(m)) : "memory");
}
__device__ __forceinline__ void mwait(unsigned long long* m, unsigned parity) {
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(sa(m)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void tma(void* dst, const CUtensorMap* map, int c0, int c1, unsigned long long* m) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          sa(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(sa(m))
      : "memory");
}
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* map, int c0, int c1, int c2, unsigned long long* m) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          sa(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(sa(m))
      : "memory");
}
// element c (0..15) of 128-byte row r of a box with 128-byte swizzle
__device__ __forceinline__ int sw(int r, int c) { return r * AK + ((((c >> 1) ^ (r & 7))) << 1) + (c & 1); }


struct Unit {
  int l, by, b;  // layer, m-tile, point block (b >= nib: boundary)
};
__device__ __forceinline__ Unit decode_unit(const Pha2Args& a, int u) {
  Unit x{0, 0, 0};
  const int nblk = a.nib + a.nbb;
  for (int l = 0; l < a.n_layers; ++l) {
    const int n = a.mtiles[l] * nblk;
    if (u < n) {
      x.l = l;
      x.by = u / nblk;
      x.b = u % nblk;
      return x;
    }
    u -= n;
  }
  return x;
}
}  // namespace

template <int C>
__global__ void __maxnreg__(255) pha2_kernel(const __grid_constant__ Pha2Args a) {
  constexpr size_t kStage = stage_bytes<C>(), kVBytes = v_bytes<C>();
  constexpr int DS = dstride<C>();
  extern __shared__ unsigned char pha2_smem[];
  unsigned char* base = pha2_smem + ((1024u - (sa(pha2_smem) & 1023u)) & 1023u);
  double* dtile = reinterpret_cast<double*>(base + ANS * kStage);  // [2][64][DS]
  unsigned long long* full = reinterpret_cast<unsigned long long*>(base + ANS * kStage + d_bytes<C>());
  unsigned long long* empty = full + ANS;
  double* red = reinterpret_cast<double*>(empty + ANS);  // [2 parity][4 row groups][PB points]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#ifdef NGD_PHA2_TRACE
  unsigned long long gt0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt0));
  long long wsum = 0;
#endif
  if (a.skip && *a.skip) return;
  const int u0 = a.cta_start[blockIdx.x], u1 = a.cta_start[blockIdx.x + 1];
  if (u0 >= u1) return;
  if (tid == 0) {
    for (int s = 0; s < ANS; ++s) {
      minit(&full[s], 1);
      minit(&empty[s], kAConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int run_int = (int)(a.int_cols / PB);  // first boundary run
  // TMA stream (warp 0, lane 0): stage j = the j-th (unit, k-chunk) of this CTA's range.  The ring
  // is refilled in-loop: after stage j is released by all warps, stage j + ANS goes into its slot.
  int pu = u0, pq = 0;  // producer cursor: unit, k-chunk
  int pj = 0;           // stages issued
  auto issue_next = [&]() {
    if (pu >= u1) return;
    const Unit x = decode_unit(a, pu);
    const int run0 = x.b < a.nib ? x.b * C : run_int + (x.b - a.nib);
    const int kc = a.kchunk[x.l], nk = a.kchunks[x.l];
    const int s = pj % ANS;
    unsigned char* stg = base + s * kStage;
#ifdef NGD_PHA2_NOTMA
    mexpect(&full[s], 0u);
    (void)stg;
    (void)run0;
#else
    mexpect(&full[s], (unsigned)(sizeof(double) * (AB * kc + kc * AK * C)));
    tma3(stg, &a.vmap[x.l], 0, x.by * AB, pq * (kc / AK), &full[s]);
    tma3(stg + kVBytes, &a.zmap[x.l], 0, run0, pq * kc, &full[s]);
#endif
    ++pj;
    if (++pq == nk) {
      pq = 0;
      ++pu;
    }
  };
  if (tid == 0)
    for (int j = 0; j < ANS; ++j) issue_next();
  // consumers: warp (kg, wm, wn): rows wm*32 + 8 mi + g (mi < 4), points wn*8 + {2t, 2t+1}, all C
  // channels, k-steps kk = 8 j + 4 kg (two k-groups; the fold is linear in the accumulators, so each
  // k-group folds its own half and the halves meet in the shared-memory sum).  Eight warps, two per
  // SM sub-partition (one warp alone could not cover its operand-load latency), and no separate
  // producer warp: a ninth warp would put three on one sub-partition and cap registers at 168.
  const int g = lane >> 2, t = lane & 3;
  const int kg = warp >> 2, wm = (warp >> 1) & 1, wn = warp & 1;
  int i = 0, parity = 0;
  for (int u = u0; u < u1; ++u, parity ^= 1) {
    const Unit x = decode_unit(a, u);
    const bool interior = x.b < a.nib;
    const int M = a.M[x.l];
    const int m0 = x.by * AB;
    const int ma = max(0, min(4, (M - m0 - wm * 32 + 7) / 8));  // 8-row blocks holding real rows
    const int col0 = interior ? x.b * PB * C : (int)a.int_cols + (x.b - a.nib) * PB;
    const int pt0 = interior ? x.b * PB : a.nib * PB + (x.b - a.nib) * PB;
    // the unit's adjoint tile D[m0.., col0..] -> shared memory with coalesced 16-byte async copies,
    // overlapping the MMAs (read at the fold after cp.async.wait_group + the unit barrier)
    double* Dt = dtile + parity * AB * DS;
    {
      const double* D = a.D[x.l];
      const int nc = interior ? PB * C : PB;  // columns of the tile
      const int rows = min(AB, M - m0);
      for (int e = tid; e < rows * (nc / 2); e += kAConsumers * 32) {
        const int r = e / (nc / 2), c2 = (e % (nc / 2)) * 2;
        const unsigned dst = sa(Dt + r * DS + c2);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst),
                     "l"(D + (int64_t)(m0 + r) * a.s_pad + col0 + c2));
      }
      asm volatile("cp.async.commit_group;\n" ::);
    }
    double acc[4][C][2];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int c = 0; c < C; ++c) acc[mi][c][0] = acc[mi][c][1] = 0.0;
    const int kc = a.kchunk[x.l], nk = a.kchunks[x.l];
    for (int q = 0; q < nk; ++q, ++i) {
      const int s = i % ANS;
#ifdef NGD_PHA2_TRACE
      long long w0 = clock64();
#endif
      mwait(&full[s], (unsigned)(i / ANS) & 1u);
#ifdef NGD_PHA2_TRACE
      wsum += clock64() - w0;
#endif
      const double* V = reinterpret_cast<const double*>(base + s * kStage);
      const double* Z = reinterpret_cast<const double*>(base + s * kStage + kVBytes);
      // MMA stream without predicates or loops: KC (k-chunk), MA (row blocks: 4, or 1 for the output
      // layer; rows past M are zero in the box) and the point-block kind are compile-time
      auto mma_chunk = [&](auto kc_tag, auto ma_tag, auto int_tag) {
        constexpr int KC = decltype(kc_tag)::value, MA = decltype(ma_tag)::value;
        constexpr int CC = decltype(int_tag)::value ? C : 1;
#pragma unroll
        for (int kk = 0; kk < KC; kk += 8) {
          const int k = kk + kg * 4 + t;
          double av[MA];
#pragma unroll
          for (int mi = 0; mi < MA; ++mi) av[mi] = V[sw((k >> 4) * AB + wm * 32 + mi * 8 + g, k & 15)];
#pragma unroll
          for (int c = 0; c < CC; ++c) {
            const double b = Z[sw(k * C + c, wn * 8 + g)];
#pragma unroll
            for (int mi = 0; mi < MA; ++mi) dmma884(acc[mi][c][0], acc[mi][c][1], av[mi], b);
          }
        }
      };
      using I16 = std::integral_constant<int, 16>;
      using I64 = std::integral_constant<int, 64>;
      using M1 = std::integral_constant<int, 1>;
      using M4 = std::integral_constant<int, 4>;
      using TI = std::integral_constant<int, 1>;
      using TB = std::integral_constant<int, 0>;
#ifdef NGD_PHA2_NOMMA
      if (ma > 1000) {
#else
      if (ma > 0) {
#endif
        if (kc == 64) {
          if (ma == 1)
            interior ? mma_chunk(I64{}, M1{}, TI{}) : mma_chunk(I64{}, M1{}, TB{});
          else
            interior ? mma_chunk(I64{}, M4{}, TI{}) : mma_chunk(I64{}, M4{}, TB{});
        } else if (kc == 32) {
          using I32 = std::integral_constant<int, 32>;
          if (ma == 1)
            interior ? mma_chunk(I32{}, M1{}, TI{}) : mma_chunk(I32{}, M1{}, TB{});
          else
            interior ? mma_chunk(I32{}, M4{}, TI{}) : mma_chunk(I32{}, M4{}, TB{});
        } else if (kc == 48) {
          using I48 = std::integral_constant<int, 48>;
          if (ma == 1)
            interior ? mma_chunk(I48{}, M1{}, TI{}) : mma_chunk(I48{}, M1{}, TB{});
          else
            interior ? mma_chunk(I48{}, M4{}, TI{}) : mma_chunk(I48{}, M4{}, TB{});
        } else {
          if (ma == 1)
            interior ? mma_chunk(I16{}, M1{}, TI{}) : mma_chunk(I16{}, M1{}, TB{});
          else
            interior ? mma_chunk(I16{}, M4{}, TI{}) : mma_chunk(I16{}, M4{}, TB{});
        }
      }
      __syncwarp();
      if (lane == 0) marrive(&empty[s]);
      if (tid == 0) {  // refill this slot once every warp has released it
        mwait(&empty[s], (unsigned)(i / ANS) & 1u);
        issue_next();
      }
    }
    // fold this k-group's half: sum over rows and channels, then over the 8 row lanes g
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    asm volatile("bar.sync 1, %0;" ::"n"(kAConsumers * 32));  // every thread's D copies have landed
    double part[2] = {0.0, 0.0};
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
      const int rl = wm * 32 + mi * 8 + g, row = m0 + rl;
      const bool ok = mi < ma && row < M;
      const double vbm = (kg == 0 && ok) ? a.vb[x.l][row] : 0.0;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double sacc = 0.0;
#pragma unroll
        for (int c = 0; c < C; ++c) {
          const double dd = (ok && (interior || c == 0)) ? Dt[rl * DS + c * PB + wn * 8 + 2 * t + e] : 0.0;
          sacc = fma(dd, acc[mi][c][e] + (c == 0 ? vbm : 0.0), sacc);
        }
        part[e] += sacc;
      }
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      part[e] += __shfl_xor_sync(0xffffffffu, part[e], 4);
      part[e] += __shfl_xor_sync(0xffffffffu, part[e], 8);
      part[e] += __shfl_xor_sync(0xffffffffu, part[e], 16);
    }
    double* rp = red + parity * 4 * PB;  // [kg * 2 + wm][PB]
    if (g == 0) {
      rp[(kg * 2 + wm) * PB + wn * 8 + 2 * t] = part[0];
      rp[(kg * 2 + wm) * PB + wn * 8 + 2 * t + 1] = part[1];
    }
    // red and the D tile are double-buffered by unit parity: the next unit's writes cannot race
    // this unit's reads past the barrier below
    asm volatile("bar.sync 1, %0;" ::"n"(kAConsumers * 32));
    if (tid < PB) {
      a.partA[x.l][(int64_t)x.by * a.n_pts_pad + pt0 + tid] = (rp[tid] + rp[PB + tid]) + (rp[2 * PB + tid] + rp[3 * PB + tid]);
    }
  }
#ifdef NGD_PHA2_TRACE
  if (tid == 0) {
    unsigned long long gt1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt1));
    g_a2tr[blockIdx.x][0] = gt0;
    g_a2tr[blockIdx.x][1] = gt1;
    g_a2tr[blockIdx.x][2] = u1 - u0;
    g_a2tr[blockIdx.x][3] = wsum;
  }
#endif
}

namespace {
PFN_cuTensorMapEncodeTiled_v12000 encoder() {
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
// 3-D view {16 doubles, runs of 16 along a row, rows} of a row-major [rows][cols] matrix; box
// {16, box_runs, box_rows}: one 128-byte-swizzled box per stage
// V_l as {16 doubles, rows, runs}: the box {16, 64 rows, KC/16 runs} lands as [run][row][16], so a
// fragment column of 8 consecutive rows spans 8 distinct swizzle phases (conflict-free A loads)
bool encode3_rows_inner(CUtensorMap* m, const double* base, int64_t cols, int rows, int box_rows, int box_runs) {
  auto enc = encoder();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)AK, (cuuint64_t)rows, (cuuint64_t)(cols / AK)};
  const cuuint64_t strides[2] = {(cuuint64_t)cols * sizeof(double), (cuuint64_t)AK * sizeof(double)};
  const cuuint32_t box[3] = {(cuuint32_t)AK, (cuuint32_t)box_rows, (cuuint32_t)box_runs};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool encode3(CUtensorMap* m, const double* base, int64_t cols, int rows, int box_runs, int box_rows) {
  auto enc = encoder();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)AK, (cuuint64_t)(cols / AK), (cuuint64_t)rows};
  const cuuint64_t strides[2] = {(cuuint64_t)AK * sizeof(double), (cuuint64_t)cols * sizeof(double)};
  const cuuint32_t box[3] = {(cuuint32_t)AK, (cuuint32_t)box_runs, (cuuint32_t)box_rows};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int C>
cudaError_t launch_pha2(const Pha2Args& a, cudaStream_t st) {
  const size_t smem = pha2_smem_bytes<C>();
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(pha2_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  probe_before(K_PHA, st);
  pha2_kernel<C><<<a.n_ctas, kPha2Threads, smem, st>>>(a);
  probe_after(K_PHA, st);
  return cudaGetLastError();
}
}  // namespace

bool pha2_supported(int C) { return C == 3 || C == 4 || C == 5 || C == 6 || C == 7 || C == 8; }

// Fills the tensor maps (cached per layer while the buffers stay put) and the cost-balanced unit
// ranges, then launches.  Units cost ~ k-chunks x (channel boxes + V box) (interior) or x 2
// (boundary).
cudaError_t pha2_all_layers(Pha2Args& a, Pha2Cache& cache, const double* const* vp, const double* const* zin,
                            const int* kp, const int* mp, int C, cudaStream_t st) {
  for (int l = 0; l < a.n_layers; ++l) {
    const int kc = std::min(kp[l], kc_max_rt(C));
    if (cache.kv[l] != vp[l] || cache.kz[l] != zin[l] || cache.kkp[l] != kp[l] || cache.kmp[l] != mp[l] ||
        cache.ks[l] != a.s_pad || cache.kc[l] != C) {  // a.vmap / a.zmap persist with the context's args
      if (!encode3_rows_inner(&a.vmap[l], vp[l], kp[l], mp[l], AB, kc / AK) ||
          !encode3(&a.zmap[l], zin[l], a.s_pad, kp[l], C, kc))
        return cudaErrorInvalidValue;
      cache.kc[l] = C;
      cache.kv[l] = vp[l];
      cache.kz[l] = zin[l];
      cache.kkp[l] = kp[l];
      cache.kmp[l] = mp[l];
      cache.ks[l] = a.s_pad;
    }
    a.kchunk[l] = std::min(kp[l], kc_max_rt(C));
    a.kchunks[l] = kp[l] / a.kchunk[l];
  }
  // cost-balanced contiguous unit ranges over one CTA per SM
  const int nblk = a.nib + a.nbb;
  double total = 0.0;
  for (int l = 0; l < a.n_layers; ++l)
    total += (double)a.mtiles[l] * a.kchunks[l] * ((double)a.nib * (C + 1) + (double)a.nbb * 2);
  const int ctas = 148;
  a.n_ctas = ctas;
  int u = 0, cta = 0;
  double acc = 0.0;
  a.cta_start[0] = 0;
  for (int l = 0; l < a.n_layers; ++l)
    for (int by = 0; by < a.mtiles[l]; ++by)
      for (int b = 0; b < nblk; ++b, ++u) {
        acc += (double)a.kchunks[l] * (b < a.nib ? C + 1 : 2);
        while (cta + 1 < ctas && acc >= total * (cta + 1) / ctas) a.cta_start[++cta] = u + 1;
      }
  while (cta + 1 <= ctas) a.cta_start[++cta] = u;
  switch (C) {
    case 3: return launch_pha2<3>(a, st);
    case 4: return launch_pha2<4>(a, st);
    case 5: return launch_pha2<5>(a, st);
    case 6: return launch_pha2<6>(a, st);
    case 7: return launch_pha2<7>(a, st);
    case 8: return launch_pha2<8>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ngd

#ifdef NGD_PHA2_TRACE
extern "C" void ngd_debug_read_a2tr(unsigned long long* out) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, ngd::g_a2tr, sizeof(ngd::g_a2tr));
}
#endif
