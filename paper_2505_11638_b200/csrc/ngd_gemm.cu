// FP64 tensor-core GEMM (DMMA.8x8x4) with a TMA / mbarrier operand pipeline -- the dense
// contractions of the Nystrom sketch and factorisation (gramian.py:55-61, sketch.py:73-86):
//
//   sketch block  S = J_c Omega          (M = chunk points, N = ell, K = p: split-K)
//                 Y += J_c^T (w o S)     (M = p,            N = ell, K = chunk points)
//   factor        Omega^T Y_nu, tall Grams A^T A, U = Q U_R, R_pass R, Newton-Schulz products,
//                 the off-diagonal updates of the blocked Cholesky / triangular solve (ell > 512)
//
//   C(m, n) = alpha * sum_k A(m, k) B(k, n) [* row_scale(m)] + beta * C(m, n),  C column-major.
//   Operand layouts: K-major  A(m, k) = A[m * lda + k]   (B(k, n) = B[n * ldb + k])
//                    MN-major A(m, k) = A[k * lda + m]   (B(k, n) = B[k * ldb + n])
//
// Design (B200, FP64 has no tcgen05 kind: warp-level DMMA, 64 FMA/clk/SM, 16-cycle issue per
// sub-partition -- tools/probe/dmma_lat.cu):
//   * 128 x 128 CTA tile, k-stages of 16, streamed with TMA (K-major operand: one 16 x 128 box;
//     MN-major operand: eight 16 x 16 boxes) into a 6-deep ring with 128-byte swizzle, completion
//     on a "full" mbarrier; eight MMA warps (2 x 4, 64 x 32 warp tiles = 32 independent DMMA
//     chains, 224 registers) release slots on "empty".  Lane 0 of warp 0 issues the TMA for the
//     stage four ahead: a dedicated ninth producer warp would put three warps on one SM
//     sub-partition, whose 16K-register file then caps every warp at 168 registers (spills);

//   * lane t of k-step ks takes column {0, 10, 5, 15}[t] ^ 2 ks of the 16-column stage.  A 64-bit
//     shared load is served per half-warp (rows g = 0..3 x the four t): with the 128-byte swizzle
//     its 16 lanes cover all 32 banks iff the four k differ in (parity, bit 3) -- K-major tiles --
//     and in bits 1..2 -- MN-major tiles; this order does both (ncu: shared wavefronts at the
//     ideal count; the first order {0,4,1,5} + {0,2,8,10}, checked per full warp, took twice
//     as many, and the plain order makes MN-major loads four-way);
//   * persistent CTAs (one per SM) walk (split, m-tile, n-tile) items n-fastest, so the CTAs
//     sharing an A panel run together (L2 reuse); long-K products are split so the item count
//     fills whole waves, the partials are summed in split order by a second kernel
//     (deterministic: fixed work assignment, no atomics).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>

#include "ngd_common.cuh"
#include "ngd_kernels.h"

namespace ngd {

namespace {
constexpr int GBK = 16;
// ring depth: 6 stages of 32 KB (128 x 128) or 5 of 40 KB (256 x 64); stages in flight ahead of
// the MMA warps: depth - 2 (slack of two stages)
template <int BM, int BN>
constexpr int gemm_ns() { return (BM + BN) * GBK * 8 * 6 <= 200 * 1024 ? 6 : 5; }
constexpr int kGemmConsumers = 8;
constexpr int kGemmThreads = kGemmConsumers * 32;
constexpr int kSms = 148;

// CTA tile BM x BN: 128 x 128 (2 x 4 warps of 64 x 32) or 256 x 64 (4 x 2 warps) -- the latter for
// narrow products (ell = 300: 5 tiles of 64 instead of 3 of 128, 6% padding instead of 28%)
template <int BM, int BN>
struct __align__(1024) GStage {
  double A[BM * GBK];
  double B[BN * GBK];
};
template <int BM, int BN>
constexpr size_t gemm_smem() {
  return sizeof(GStage<BM, BN>) * gemm_ns<BM, BN>() + 2 * gemm_ns<BM, BN>() * sizeof(unsigned long long) + 1024;
}

__device__ __forceinline__ unsigned g_smem(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void g_mbar_init(unsigned long long* m, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(g_smem(m)), "r"(count));
}
__device__ __forceinline__ void g_expect_tx(unsigned long long* m, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(g_smem(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void g_arrive(unsigned long long* m) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(g_smem(m)) : "memory");
}
__device__ __forceinline__ void g_wait(unsigned long long* m, unsigned parity) {
  const unsigned a = g_smem(m);
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void g_tma2d(void* dst, const CUtensorMap* map, int c0, int c1, unsigned long long* m) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          g_smem(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(g_smem(m))
      : "memory");
}

// offset (doubles) of element (mn, k) of a stage tile
template <bool KMAJ>
__device__ __forceinline__ int toff(int mn, int k) {
  if (KMAJ) return mn * 16 + ((((k >> 1) ^ (mn & 7)) << 1) | (k & 1));  // [128 rows mn][16 k]
  return (mn >> 4) * 256 + k * 16 + (((((mn & 15) >> 1) ^ (k & 7)) << 1) | (mn & 1));  // [8][16 k][16 mn]
}

struct GItem {
  int tm, tn, split, s0, s1;
};
__device__ __forceinline__ GItem decode(const GemmArgs& a, int idx) {
  GItem it;
  const int per = a.tiles_m * a.tiles_n;
  it.split = idx / per;
  const int r = idx - it.split * per;
  it.tm = r / a.tiles_n;
  it.tn = r - it.tm * a.tiles_n;
  it.s0 = min(a.kstages, it.split * a.kps);
  it.s1 = min(a.kstages, it.s0 + a.kps);
  return it;
}
}  // namespace

// walks the (item, k-stage) sequence of one CTA: items blockIdx.x, blockIdx.x + gridDim.x, ...
struct GCursor {
  int idx, s, s1, m0, n0;
};
template <int BM, int BN>
__device__ __forceinline__ bool cursor_load(const GemmArgs& a, int n_items, GCursor& c) {
  while (c.idx < n_items) {
    const GItem it = decode(a, c.idx);
    if (it.s0 < it.s1) {
      c.s = it.s0;
      c.s1 = it.s1;
      c.m0 = it.tm * BM;
      c.n0 = it.tn * BN;
      return true;
    }
    c.idx += gridDim.x;
  }
  return false;
}

template <int BM, int BN, bool AK, bool BK>
__device__ __forceinline__ void issue_stage(GStage<BM, BN>& st, const CUtensorMap& mapA, const CUtensorMap& mapB,
                                            const GCursor& c, unsigned long long* full) {
  g_expect_tx(full, sizeof(double) * (BM + BN) * GBK);
  const int k0 = c.s * GBK;
  if (AK) {
    g_tma2d(st.A, &mapA, k0, c.m0, full);
  } else {
#pragma unroll
    for (int b = 0; b < BM / 16; ++b) g_tma2d(st.A + b * 256, &mapA, c.m0 + b * 16, k0, full);
  }
  if (BK) {
    g_tma2d(st.B, &mapB, k0, c.n0, full);
  } else {
#pragma unroll
    for (int b = 0; b < BN / 16; ++b) g_tma2d(st.B + b * 256, &mapB, c.n0 + b * 16, k0, full);
  }
}

template <int BM, int BN, bool AK, bool BK>
__global__ void __maxnreg__(224)
    dgemm_kernel(const __grid_constant__ GemmArgs a, const __grid_constant__ CUtensorMap mapA,
                 const __grid_constant__ CUtensorMap mapB) {
  constexpr int WGN = BN / 32;  // warps along n (64 x 32 warp tiles, 8 warps)
  constexpr int GNS = gemm_ns<BM, BN>(), GAHEAD = GNS - 2;
  static_assert((BM / 64) * WGN == kGemmConsumers, "8 warps of 64 x 32");
  extern __shared__ unsigned char gsm_raw[];
  unsigned char* base = gsm_raw + ((1024u - (g_smem(gsm_raw) & 1023u)) & 1023u);
  GStage<BM, BN>* st = reinterpret_cast<GStage<BM, BN>*>(base);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(st + GNS);
  unsigned long long* empty = full + GNS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < GNS; ++s) {
      g_mbar_init(&full[s], 1);
      g_mbar_init(&empty[s], kGemmConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int n_items = a.tiles_m * a.tiles_n * a.splits;
  const bool producer = (tid == 0);
  GCursor pc{(int)blockIdx.x, 0, 0, 0, 0};
  bool p_valid = producer ? cursor_load<BM, BN>(a, n_items, pc) : false;
  unsigned qp = 0;  // next ring position the producer fills
  // warp (wm, wn) owns rows wm*64 .. +63, cols wn*32 .. +31 of the tile
  const int wm = warp / WGN, wn = warp % WGN;
  const int g = lane >> 2, t = lane & 3;
#ifndef GEMM_KORD
#define GEMM_KORD 2
#endif
#if GEMM_KORD == 2
  const int koff = ((t & 1) * 10) ^ ((t >> 1) * 5);  // {0, 10, 5, 15}
#else
  const int koff = ((t & 1) << 2) | (t >> 1);  // {0, 4, 1, 5} (first order, kept for A/B builds)
#endif
  unsigned q = 0;  // ring position of the next stage consumed
  for (int idx = blockIdx.x; idx < n_items; idx += gridDim.x) {
    const GItem it = decode(a, idx);
    double acc[8][4][2];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int s = it.s0; s < it.s1; ++s, ++q) {
      if (producer) {  // keep GAHEAD stages in flight: the slot of position q + GAHEAD - 1 was freed at q - 2
        while (p_valid && qp < q + GAHEAD) {
          const int slot = qp % GNS;
          if (qp >= GNS) g_wait(&empty[slot], ((qp / GNS) - 1) & 1u);
          issue_stage<BM, BN, AK, BK>(st[slot], mapA, mapB, pc, &full[slot]);
          ++qp;
          if (++pc.s >= pc.s1) {
            pc.idx += gridDim.x;
            p_valid = cursor_load<BM, BN>(a, n_items, pc);
          }
        }
      }
      __syncwarp();
      const int slot = q % GNS;
      g_wait(&full[slot], (q / GNS) & 1u);
      const double* As = st[slot].A;
      const double* Bs = st[slot].B;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
#if GEMM_KORD == 2
        const int kk = (ks << 1) ^ koff;
#else
        const int kk = ((ks & 1) << 1) + ((ks >> 1) << 3) + koff;
#endif
        double av[8], bv[4];
#pragma unroll
        for (int i = 0; i < 8; ++i) av[i] = As[toff<AK>(wm * 64 + i * 8 + g, kk)];
#pragma unroll
        for (int j = 0; j < 4; ++j) bv[j] = Bs[toff<BK>(wn * 32 + j * 8 + g, kk)];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], av[i], bv[j]);
      }
      // a lagging warp's release can be the one the producer is waiting on: order the shared-memory
      // reads (generic proxy) before the TMA refill (async proxy), as in ngd_phag.cu
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) g_arrive(&empty[slot]);
    }
    // epilogue: direct column-major stores (8 consecutive rows per column segment)
    const int m0 = it.tm * BM + wm * 64 + g, n0 = it.tn * BN + wn * 32 + 2 * t;
    double* C = a.C;
    int64_t ldc = a.ldc;
    double alpha = a.alpha, beta = a.beta;
    const double* rs = a.row_scale;
    if (a.splits > 1) {  // partial of this split: dense M x N, no scaling
      C = a.part + (int64_t)it.split * a.M * a.N;
      ldc = a.M;
      alpha = 1.0;
      beta = 0.0;
      rs = nullptr;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int m = m0 + i * 8;
      if (m >= a.M) continue;
      const double sc = rs ? alpha * rs[m] : alpha;
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int n = n0 + j * 8 + e;
          if (n < a.N) {
            double* dst = C + (int64_t)n * ldc + m;
            double v = sc * acc[i][j][e];
            if (beta != 0.0) v = fma(beta, *dst, v);
            *dst = v;
          }
        }
    }
  }
}

// C = alpha * sum_g part[g] (* row_scale) + beta * C  (splits in fixed order)
__global__ void gemm_reduce_kernel(const double* __restrict__ part, int splits, int M, int N, double alpha,
                                   const double* __restrict__ row_scale, double beta, double* C, int64_t ldc) {
  const int64_t total = (int64_t)M * N;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int gidx = 0; gidx < splits; ++gidx) s += part[(int64_t)gidx * total + e];
    const int n = (int)(e / M), m = (int)(e - (int64_t)n * M);
    double v = alpha * s;
    if (row_scale) v *= row_scale[m];
    double* dst = C + (int64_t)n * ldc + m;
    if (beta != 0.0) v = fma(beta, *dst, v);
    *dst = v;
  }
}

namespace {
PFN_cuTensorMapEncodeTiled_v12000 tm_encode() {
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
// K-major: dims {K, MN}, box {16, tile};  MN-major: dims {MN, K}, box {16, 16}
bool encode_operand(CUtensorMap* m, const GemmOperand& o, int MN, int K, int tile) {
  auto enc = tm_encode();
  if (!enc) return false;
  cuuint64_t dims[2];
  cuuint32_t box[2];
  if (o.kmaj) {
    dims[0] = (cuuint64_t)K;
    dims[1] = (cuuint64_t)MN;
    box[0] = 16;
    box[1] = (cuuint32_t)tile;
  } else {
    dims[0] = (cuuint64_t)MN;
    dims[1] = (cuuint64_t)K;
    box[0] = 16;
    box[1] = 16;
  }
  const cuuint64_t strides[1] = {(cuuint64_t)o.ld * sizeof(double)};
  const cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(o.p), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BM, int BN, bool AK, bool BK>
cudaError_t launch(const GemmArgs& a, const CUtensorMap& ma, const CUtensorMap& mb, int grid, cudaStream_t st) {
  static bool attr = false;
  constexpr size_t smem = gemm_smem<BM, BN>();
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(dgemm_kernel<BM, BN, AK, BK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dgemm_kernel<BM, BN, AK, BK><<<grid, kGemmThreads, smem, st>>>(a, ma, mb);
  return cudaGetLastError();
}
template <int BM, int BN>
cudaError_t launch_any(bool ak, bool bk, const GemmArgs& a, const CUtensorMap& ma, const CUtensorMap& mb, int grid,
                       cudaStream_t st) {
  if (ak && bk) return launch<BM, BN, true, true>(a, ma, mb, grid, st);
  if (ak) return launch<BM, BN, true, false>(a, ma, mb, grid, st);
  if (bk) return launch<BM, BN, false, true>(a, ma, mb, grid, st);
  return launch<BM, BN, false, false>(a, ma, mb, grid, st);
}
}  // namespace

bool gemm_operand_ok(const GemmOperand& o, int MN, int K) {
  const int64_t inner = o.kmaj ? K : MN;
  return o.p != nullptr && (reinterpret_cast<uintptr_t>(o.p) & 15u) == 0 && (o.ld & 1) == 0 && o.ld >= inner &&
         o.ld < ((int64_t)1 << 36);
}

GemmPlan gemm_plan(int M, int N, int K) {
  GemmPlan pl;
  // tile shape: the one with the least padded area (ties: 128 x 128)
  const int64_t pad_sq = (int64_t)((M + 127) / 128 * 128) * ((N + 127) / 128 * 128);
  const int64_t pad_tall = (int64_t)((M + 255) / 256 * 256) * ((N + 63) / 64 * 64);
  pl.bm = pad_tall < pad_sq ? 256 : 128;
  pl.bn = pl.bm == 256 ? 64 : 128;
  pl.tiles_m = (M + pl.bm - 1) / pl.bm;
  pl.tiles_n = (N + pl.bn - 1) / pl.bn;
  pl.kstages = (K + GBK - 1) / GBK;
  const int tiles = pl.tiles_m * pl.tiles_n;
  // split long-K products so the items fill whole waves of one CTA per SM; each split keeps >= 32
  // k-stages (the ring prologue and the epilogue amortised) and splits <= 64
  int best = 1;
  double best_score = -1.0;
  const int gmax = std::max(1, std::min(64, pl.kstages / 32));
  for (int gs = 1; gs <= gmax; ++gs) {
    const int items = tiles * gs;
    const int waves = (items + kSms - 1) / kSms;
    const double eff = (double)items / ((double)waves * kSms);
    const double score = eff - 0.004 * (gs - 1);
    if (score > best_score + 1e-12) {
      best_score = score;
      best = gs;
    }
    if (tiles * gs >= 4 * kSms && eff > 0.97) break;
  }
  pl.splits = best;
  pl.kps = (pl.kstages + best - 1) / best;
  pl.splits = (pl.kstages + pl.kps - 1) / pl.kps;  // no empty splits
  pl.work_bytes = pl.splits > 1 ? sizeof(double) * (size_t)pl.splits * M * N : 0;
  return pl;
}

// algorithmic FLOPs (2 M N K) of every GEMM launched so far (bench.py's roofline of this class)
static double g_gemm_flops = 0.0;
double gemm_flops_total() { return g_gemm_flops; }

cudaError_t dgemm(int M, int N, int K, double alpha, const GemmOperand& A, const GemmOperand& B, double beta,
                  double* C, int64_t ldc, const double* row_scale, double* work, size_t work_bytes,
                  cudaStream_t st) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  if (K <= 0) return cudaErrorInvalidValue;
  if (!gemm_operand_ok(A, M, K) || !gemm_operand_ok(B, N, K)) return cudaErrorInvalidValue;
  const GemmPlan pl = gemm_plan(M, N, K);
  if (pl.work_bytes > work_bytes) return cudaErrorInvalidValue;
  GemmArgs a{};
  a.M = M;
  a.N = N;
  a.K = K;
  a.tiles_m = pl.tiles_m;
  a.tiles_n = pl.tiles_n;
  a.kstages = pl.kstages;
  a.splits = pl.splits;
  a.kps = pl.kps;
  a.alpha = alpha;
  a.beta = beta;
  a.C = C;
  a.ldc = ldc;
  a.row_scale = row_scale;
  a.part = work;
  CUtensorMap ma, mb;
  if (!encode_operand(&ma, A, M, K, pl.bm) || !encode_operand(&mb, B, N, K, pl.bn)) return cudaErrorInvalidValue;
  const int items = pl.tiles_m * pl.tiles_n * pl.splits;
  const int grid = std::min(items, kSms);
  g_gemm_flops += 2.0 * M * N * (double)K;
  probe_before(K_GEMM, st);
  const cudaError_t e = pl.bm == 256 ? launch_any<256, 64>(A.kmaj, B.kmaj, a, ma, mb, grid, st)
                                      : launch_any<128, 128>(A.kmaj, B.kmaj, a, ma, mb, grid, st);
  probe_after(K_GEMM, st);
  if (e != cudaSuccess || pl.splits == 1) return e;
  const int64_t total = (int64_t)M * N;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 4 * kSms);
  probe_before(K_GEMM, st);
  gemm_reduce_kernel<<<blocks, 256, 0, st>>>(work, pl.splits, M, N, alpha, row_scale, beta, C, ldc);
  probe_after(K_GEMM, st);
  return cudaGetLastError();
}

// y = G x for a row-major n x n G (one warp per row, fixed-order lane sums): the dense-operator
// PCG of gramian.py:101-120 / krylov.py (the DenseOperator path of the tests and the spectrum)
__global__ void gemv_rows_kernel(const double* __restrict__ G, int64_t n, const double* __restrict__ x,
                                 double* __restrict__ y, const int* skip) {
  if (skip && *skip) return;
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (row >= n) return;
  const double* gr = G + row * n;
  double s = 0.0;
  for (int64_t k = lane; k < n; k += 32) s = fma(gr[k], x[k], s);
  s = warp_sum(s);
  if (lane == 0) y[row] = s;
}

cudaError_t gemv_rows(const double* G, int64_t n, const double* x, double* y, const int* skip, cudaStream_t st) {
  const int blocks = (int)((n + 7) / 8);
  probe_before(K_GEMM, st);
  gemv_rows_kernel<<<blocks, 256, 0, st>>>(G, n, x, y, skip);
  probe_after(K_GEMM, st);
  return cudaGetLastError();
}

}  // namespace ngd
