// FP64-exact GEMM on the INT8 tensor cores (tcgen05.mma kind::i8, TMEM accumulators, TMA ring):
// the Ozaki scheme II (integer modular form, CRT reconstruction) for the two dense contractions of
// the J-chunk Nystrom sketch (gramian.py:55-61 evaluated as Y = G Omega, sketch.py:76):
//
//     S = diag(w) J_c Omega        (M = chunk points, N = ell, K = p)
//     Y += J_c^T S                 (M = p,            N = ell, K = chunk points)
//
// FP64 has no tcgen05 kind on sm_100a; the DMMA pipe peaks at ~37 TF/s while the INT8 tensor
// pipe runs ~3 POPS.  The product is computed exactly in integers and rounded once:
//
//   1. scaling (per row of A, per column of B):  A'(m,k) = rint(A(m,k) 2^alpha_m) with
//      max_k |A'(m,k)| <= 2^t, likewise B'(k,n) = rint(B(k,n) 2^beta_n); t = 53 (the row maximum
//      keeps its full FP64 mantissa) unless K 2^(2t+1) would reach the CRT modulus.
//   2. residues:  A'_j = A' mod m_j for 16 pairwise-coprime moduli m_j <= 256 (symmetric, int8).
//   3. 16 int8 GEMMs  C_j = A'_j B'_j  (exact int32: K <= 131071 per K-split), reduced mod m_j to
//      int8 in the epilogue.
//   4. CRT:  C' = A' B' is the unique integer in (-M/2, M/2), M = prod m_j (2^125.4), congruent to
//      C_j mod m_j:  C'/M = sum_j r_j (y_j / m_j) mod 1, y_j = (M/m_j)^-1 mod m_j, evaluated exactly
//      in three 41-bit slices of y_j / m_j (every partial sum is an exact FP64 integer), then one
//      rounding: C = C' 2^-(alpha_m + beta_n).
//
// Accuracy: the only errors are the rounding of A, B to t-bit integers relative to their row /
// column maxima (2^-54 relative to max_k |A(m,k)| resp. max_k |B(k,n)|) and the final rounding of
// C' (2^-53 relative, plus an absolute 2^-83 M from the CRT slices -- 2^-64 of the largest
// possible product term): |C - AB| <= 2^-53 (max_k|A_mk| sum_k|B_kn| + sum_k|A_mk| max_k|B_kn|)
// + 2^-53 |AB|, the same order as FP64 GEMM's own K-dependent error bound (tests/test_gpu_ozaki.py).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>

#include "ngd_common.cuh"
#include "ngd_kernels.h"

namespace ngd {

namespace {

constexpr int NMOD = kOzMods;
__host__ __device__ constexpr int mod_of(int j) {
  return j == 0    ? 256
         : j == 1  ? 255
         : j == 2  ? 253
         : j == 3  ? 251
         : j == 4  ? 247
         : j == 5  ? 241
         : j == 6  ? 239
         : j == 7  ? 233
         : j == 8  ? 229
         : j == 9  ? 227
         : j == 10 ? 223
         : j == 11 ? 217
         : j == 12 ? 211
         : j == 13 ? 199
         : j == 14 ? 197
                   : 193;
}
constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52: x + kMagic rounds x to an integer
constexpr int kExpNonFinite = kOzNonFinite;     // row / column exponent of a non-finite input

// per-modulus constants of the CRT and the residue generation (host-computed, passed by value)
struct OzTab {
  double h[NMOD], g[NMOD], l[NMOD];  // y_j / m_j = (h 2^-41 + g 2^-82 + l 2^-123) + O(2^-123)
  double c26[NMOD];                  // 2^26 mod m_j, symmetric
  double md;                         // M rounded to FP64
  double log2m;
};

OzTab make_tab() {
  OzTab t{};
  // M = prod m_j as a 128-bit integer (2^125.4 < 2^128)
  unsigned __int128 M = 1;
  for (int j = 0; j < NMOD; ++j) M *= (unsigned)mod_of(j);
  long double md = 1.0L;
  double lg = 0.0;
  for (int j = 0; j < NMOD; ++j) {
    md *= (long double)mod_of(j);
    lg += std::log2((double)mod_of(j));
  }
  t.md = (double)md;
  t.log2m = lg;
  for (int j = 0; j < NMOD; ++j) {
    const int m = mod_of(j);
    const unsigned __int128 Mj = M / (unsigned)m;
    const int mjr = (int)(Mj % (unsigned)m);
    int y = 0;
    for (int k = 1; k < m; ++k)
      if ((mjr * k) % m == 1) {
        y = k;
        break;
      }
    // binary expansion of y / m: 123 bits in three 41-bit slices
    unsigned long long rem = (unsigned long long)y;
    unsigned long long s[3] = {0, 0, 0};
    for (int b = 0; b < 123; ++b) {
      rem <<= 1;
      const unsigned long long bit = rem >= (unsigned long long)m ? 1ull : 0ull;
      if (bit) rem -= (unsigned long long)m;
      s[b / 41] = (s[b / 41] << 1) | bit;
    }
    t.h[j] = (double)s[0];
    t.g[j] = (double)s[1];
    t.l[j] = (double)s[2];
    int c = (int)((1ull << 26) % (unsigned long long)m);
    if (c > m / 2) c -= m;
    t.c26[j] = (double)c;
  }
  return t;
}

const OzTab& tab() {
  static const OzTab t = make_tab();
  return t;
}

// 2^e for |e| <= ~2100 as two exactly representable factors
__device__ __forceinline__ double pow2(int e) { return __longlong_as_double((long long)(e + 1023) << 52); }
__device__ __forceinline__ double scale2(double x, int e) {
  const int e1 = e >> 1;
  return (x * pow2(e1)) * pow2(e - e1);
}

// residue words of 8 elements (two groups of 4 consecutive) for every modulus: w[j][0], w[j][1].
// The 8 elements' chains of one modulus are written as separate passes over arrays so the four
// dependent FP64 steps of each chain interleave across the elements (the per-element form compiled
// to back-to-back dependent DFMA / DADD pairs).
template <int J = 0>
__device__ __forceinline__ void residue_words8(const double (&xh)[8], const double (&xl)[8], const OzTab& tb,
                                               unsigned (&w)[NMOD][2]) {
  if constexpr (J < NMOD) {
    constexpr double m = (double)mod_of(J);
    constexpr double inv = 1.0 / (double)mod_of(J);
    const double c = tb.c26[J];
    double v[8], q[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = fma(xh[e], c, xl[e]);
#pragma unroll
    for (int e = 0; e < 8; ++e) q[e] = fma(v[e], inv, kMagic);
#pragma unroll
    for (int e = 0; e < 8; ++e) q[e] -= kMagic;
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = fma(-q[e], m, v[e]) + kMagic;
    unsigned lo = 0, hi = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      lo |= ((unsigned)__double2loint(v[e]) & 0xFFu) << (8 * e);
      hi |= ((unsigned)__double2loint(v[e + 4]) & 0xFFu) << (8 * e);
    }
    w[J][0] = lo;
    w[J][1] = hi;
    residue_words8<J + 1>(xh, xl, tb, w);
  }
}

__device__ __forceinline__ void split26(double a, double s1, double s2, double& xh, double& xl) {
  const double x = rint((a * s1) * s2);  // |x| <= 2^t <= 2^53
  xh = fma(x, 1.0 / 67108864.0, kMagic) - kMagic;
  xl = fma(-xh, 67108864.0, x);
}

__device__ __forceinline__ int exp_for_max(double mx, int t) {
  if (!(mx <= 1.79769313486231570815e+308)) return kExpNonFinite;  // inf / nan
  if (mx == 0.0) return 0;
  return t - 1 - ilogb(mx);  // mx 2^alpha in [2^(t-1), 2^t)
}


// Exponents from running maxima kept as ordered bit patterns of |x| (formj_kernel's RED.MAX): bit
// patterns at or above +inf's flag a non-finite row / column.
__global__ void oz_exps_kernel(const unsigned long long* __restrict__ mx, int n, int t, int* __restrict__ exps) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long b = mx[i];
  exps[i] = b >= 0x7ff0000000000000ull ? kExpNonFinite : exp_for_max(__longlong_as_double((long long)b), t);
}

// exponent making max |x| 2^g land in [2^(t-1), 2^t), from its log-bit pattern (oz_logbits)
__device__ __forceinline__ int exp_from_logbits(long long v, int t) {
  if (v == 0x7fffffffffffffffll) return kExpNonFinite;
  if (v < kOzLogEmpty) return 0;                    // no entry (all zero)
  return t - 1 - (int)((v >> 51) - 1023);           // floor(log2) of a normal |x| 2^g
}
__global__ void oz_exps_log_kernel(const long long* __restrict__ mx, int n, int t, int* __restrict__ exps) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) exps[i] = exp_from_logbits(mx[i], t);
}

// Row exponents of a K-major FP64 operand, optionally of the column-prescaled |A(r, k)| 2^(sign
// colexp[k]) (two-sided scaling): one CTA per row, log-bit maxima.
__global__ void __launch_bounds__(256) oz_rowmax_kernel(const double* __restrict__ A, int64_t lda, int rows, int K,
                                                        int t, int* __restrict__ exps, const int* __restrict__ colexp,
                                                        int colsign) {
  __shared__ long long sh[8];
  const int r = blockIdx.x;
  if (r >= rows) return;
  const double* a = A + (int64_t)r * lda;
  long long mx = kOzLogEmpty - 1;
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    int g = 0;
    if (colexp) {
      g = colexp[k];
      if (g != kExpNonFinite) g *= colsign;
    }
    mx = max(mx, oz_logbits(a[k], g));
  }
  for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mx = max(mx, sh[w]);
    exps[r] = exp_from_logbits(mx, t);
  }
}

__device__ __forceinline__ void cp16(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"((unsigned)__cvta_generic_to_shared(ssrc)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Row-scaled residues of a K-major FP64 operand A(r, k) = A[r lda + k] (r < rows, k < K; lda even,
// A 16-byte aligned) with the row exponents given: out[j][r][ldo] (int8, k contiguous, zero for
// K <= k < ldo).  Persistent CTAs over tiles of one row x 2048 k.  Compute and memory overlap
// (run back to back they added up: 4.2 ms of arithmetic + ~5 ms of traffic for a C3 chunk):
//   * the next tile streams into shared memory with cp.async while this one is converted;
//   * the 16 residue rows (2 KB each, one per modulus) leave a double-buffered shared-memory stage
//     as asynchronous bulk copies (cp.async.bulk ... bulk_group), drained one tile later.
constexpr int kRowsK = 2048;
constexpr int kConvIn = 3;  // input ring depth (tiles in flight ahead of the arithmetic)
constexpr size_t kRowsSmem = kConvIn * kRowsK * sizeof(double) + 2 * NMOD * kRowsK;
template <bool HASCOL>
__global__ void __launch_bounds__(256) oz_rows_kernel(const double* __restrict__ A, int64_t lda, int rows, int K,
                                                      const int* __restrict__ exps, const int* __restrict__ colexp,
                                                      int colsign, int8_t* __restrict__ out, int64_t ldo,
                                                      int64_t plane, const OzTab tb) {
  extern __shared__ __align__(128) unsigned char rsm[];
  double* in = reinterpret_cast<double*>(rsm);                   // [kConvIn][2048]
  unsigned char* stg = rsm + kConvIn * kRowsK * sizeof(double);  // [2][16][2048]
  const int tiles_k = (int)((ldo + kRowsK - 1) / kRowsK);
  const int ntiles = rows * tiles_k;
  const int tid = threadIdx.x;
  auto issue = [&](int tile, int buf) {
    if (tile < ntiles) {
      const int r = tile / tiles_k, k0 = (tile % tiles_k) * kRowsK;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int kk = k0 + 2 * (tid + 256 * i);
        const bool ok = kk < lda;
        cp16(in + buf * kRowsK + 2 * (tid + 256 * i), ok ? A + (int64_t)r * lda + kk : A, ok ? 16u : 0u);
      }
    }
    cp_commit();
  };
  // the row exponent is fetched one tile ahead; column exponents (HASCOL) are read per element (L2 / L1)
  auto row_exp = [&](int tl) { return tl < ntiles ? exps[tl / tiles_k] : 0; };
  int tile = blockIdx.x;
  issue(tile, 0);
  issue(tile + gridDim.x, 1);
  int e_next = row_exp(tile);
  for (int it = 0; tile < ntiles; ++it, tile += gridDim.x) {
    const int buf = it & 1, ib = it % kConvIn;
    const int e = e_next;
    issue(tile + 2 * gridDim.x, (it + 2) % kConvIn);
    e_next = row_exp(tile + gridDim.x);
    if (tid == 0) bulk_wait_read<1>();  // the stage written two tiles ago has been read out
    cp_wait<2>();
    __syncthreads();
    const int r = tile / tiles_k, k0 = (tile % tiles_k) * kRowsK;
    unsigned wd[NMOD][2];
    {
      double xh[8], xl[8];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int kl = 4 * tid + (kRowsK / 2) * h;
        const double* src = in + ib * kRowsK + kl;
        const double2 d0 = *reinterpret_cast<const double2*>(src), d1 = *reinterpret_cast<const double2*>(src + 2);
        const double v[4] = {d0.x, d0.y, d1.x, d1.y};
        int ce[4] = {0, 0, 0, 0};
        if (HASCOL) {
          if (k0 + kl + 3 < K) {
            const int4 c4 = *reinterpret_cast<const int4*>(colexp + k0 + kl);
            ce[0] = c4.x, ce[1] = c4.y, ce[2] = c4.z, ce[3] = c4.w;
          } else {
#pragma unroll
            for (int e4 = 0; e4 < 4; ++e4) ce[e4] = k0 + kl + e4 < K ? colexp[k0 + kl + e4] : 0;
          }
        }
#pragma unroll
        for (int e4 = 0; e4 < 4; ++e4) {
          const int k = k0 + kl + e4;
          const bool live = e != kExpNonFinite && ce[e4] != kExpNonFinite && k < K;
          const int ek = live ? e + colsign * ce[e4] : 0;
          const int e1 = ek >> 1;
          split26(live ? v[e4] : 0.0, pow2(e1), pow2(ek - e1), xh[4 * h + e4], xl[4 * h + e4]);
        }
      }
      residue_words8(xh, xl, tb, wd);
    }
    unsigned* so = reinterpret_cast<unsigned*>(stg + (size_t)buf * NMOD * kRowsK);
#pragma unroll
    for (int j = 0; j < NMOD; ++j) {
      so[j * (kRowsK / 4) + tid] = wd[j][0];
      so[j * (kRowsK / 4) + tid + kRowsK / 8] = wd[j][1];
    }
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      const unsigned bytes = (unsigned)(ldo - k0 < kRowsK ? ldo - k0 : kRowsK);
      int8_t* dst = out + (int64_t)r * ldo + k0;
      for (int j = 0; j < NMOD; ++j)
        bulk_store(dst + (int64_t)j * plane, stg + ((size_t)buf * NMOD + j) * kRowsK, bytes);
      bulk_commit();
    }
  }
  cp_wait<0>();
  if (tid == 0) bulk_wait_read<0>();
}

// Blocked residues of J' (two-sided exponents): out[j] = [row block][column block][128][128] int8,
// each 128 x 128 block contiguous (16 KB), so the TMA boxes of BOTH products -- K-major for
// S = J' V' and MN-major (as J'^T) for Y = J'^T S' -- are single contiguous blocks (the MN-major reads
// of the row-major layout touched 128 rows 200 kB apart per box).  Tiles of 16 rows x 128 columns:
// thread (q = tid / 16, c = 8 (tid % 16)) converts 8 consecutive elements of row q; the 16 residue
// slabs (16 rows x 128 B, contiguous inside a block) leave as asynchronous bulk copies.  Rows >= rows
// and columns >= K of the last blocks are written as zero residues.
constexpr size_t kBlkSmem = kConvIn * 2048 * sizeof(double) + 2 * NMOD * 2048;
__global__ void __launch_bounds__(256) oz_rows_blocked_kernel(const double* __restrict__ A, int64_t lda, int rows,
                                                              int K, int nrb, int ncb, const int* __restrict__ rexp,
                                                              const int* __restrict__ cexp, int8_t* __restrict__ out,
                                                              int64_t plane, const OzTab tb) {
  extern __shared__ __align__(128) unsigned char bsm[];
  double* in = reinterpret_cast<double*>(bsm);                  // [kConvIn][16][128]
  unsigned char* stg = bsm + kConvIn * 2048 * sizeof(double);   // [2][16][16 x 128]
  const int tiles_c = ncb, ntiles = nrb * 8 * ncb;              // 8 row slabs of 16 per row block
  const int tid = threadIdx.x;
  const int q = tid >> 4, c = (tid & 15) * 8;
  auto issue = [&](int tile, int buf) {
    if (tile < ntiles) {
      const int r0 = (tile / tiles_c) * 16, k0 = (tile % tiles_c) * 128;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int ch = tid + 256 * i;  // row ch / 64, doubles 2 (ch % 64)
        const int rr = r0 + (ch >> 6), kk = k0 + 2 * (ch & 63);
        const bool ok = rr < rows && kk < lda;
        cp16(in + buf * 2048 + ch * 2, ok ? A + (int64_t)rr * lda + kk : A, ok ? 16u : 0u);
      }
    }
    cp_commit();
  };
  auto row_exp = [&](int tl) {
    const int rr = (tl / tiles_c) * 16 + q;
    return (tl < ntiles && rr < rows) ? rexp[rr] : kExpNonFinite;  // rows past `rows`: zero residues
  };
  int tile = blockIdx.x;
  issue(tile, 0);
  issue(tile + gridDim.x, 1);
  int e_next = row_exp(tile);
  for (int it = 0; tile < ntiles; ++it, tile += gridDim.x) {
    const int buf = it & 1, ib = it % kConvIn;
    const int e = e_next;
    issue(tile + 2 * gridDim.x, (it + 2) % kConvIn);
    e_next = row_exp(tile + gridDim.x);
    if (tid == 0) bulk_wait_read<1>();
    cp_wait<2>();
    __syncthreads();
    const int r0 = (tile / tiles_c) * 16, k0 = (tile % tiles_c) * 128;
    unsigned wd[NMOD][2];
    {
      double xh[8], xl[8];
      const double* src = in + ib * 2048 + q * 128 + c;
#pragma unroll
      for (int e8 = 0; e8 < 8; ++e8) {
        const int k = k0 + c + e8;
        const int ce = k < K ? cexp[k] : kExpNonFinite;
        const bool live = e != kExpNonFinite && ce != kExpNonFinite;
        const int ek = live ? e + ce : 0;
        const int e1 = ek >> 1;
        split26(live ? src[e8] : 0.0, pow2(e1), pow2(ek - e1), xh[e8], xl[e8]);
      }
      residue_words8(xh, xl, tb, wd);
    }
    unsigned char* so = stg + (size_t)buf * NMOD * 2048;
#pragma unroll
    for (int j = 0; j < NMOD; ++j)
      *reinterpret_cast<uint2*>(so + j * 2048 + q * 128 + c) = make_uint2(wd[j][0], wd[j][1]);
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      const int rb = r0 >> 7, cb = k0 >> 7;
      int8_t* dst = out + ((int64_t)rb * ncb + cb) * 16384 + (r0 & 127) * 128;
      for (int j = 0; j < NMOD; ++j) bulk_store(dst + (int64_t)j * plane, so + j * 2048, 2048);
      bulk_commit();
    }
  }
  cp_wait<0>();
  if (tid == 0) bulk_wait_read<0>();
}

// ------------------------------------------------------------------------------------------------
// INT8 tensor-core GEMM (tcgen05.mma.cta_group::1.kind::i8): per (K-split s, modulus j, 128 x 256
// output tile) item  C = A_j(m, k) B_j(n, k)^T  over the split's k range, both operands K-major in
// 128-byte swizzled TMA boxes of 128 k; a 4-deep ring (48 KB stages); int32 accumulators in TMEM,
// double-buffered (2 x 256 columns) so the epilogue of one item overlaps the next item's MMAs.
//   warp 0: TMA producer (one lane)   warp 1: TMEM allocation + MMA issue (one lane)
//   warps 2-5: epilogue -- tcgen05.ld 32 columns at a time, reduce mod m_j, store int8 residues
//              res[(s NMOD + j) plane + n ldo + m]   (column-major, coalesced over m)
// Items walk n fastest, then m, then (j, s): the CTAs that share an A panel run together and one
// modulus' B panel stays in L2 while every m-tile reads it.
constexpr int IBM = 128, IBN = 256, IBK = 128, INS = 4;
constexpr int kI8Threads = 192;
struct __align__(1024) I8Stage {
  int8_t A[IBM * IBK];
  int8_t B[IBN * IBK];
};
constexpr size_t kI8Smem = sizeof(I8Stage) * INS + 1024 + 256;

struct I8Args {
  int M, N, splits, tiles_m, tiles_n, kblocks, kb_per_split;
  int8_t* res;
  int64_t ldo, plane;
  int a_blocked;  // A in 128 x 128 blocks (oz_rows_blocked): 5-D boxes {128, 128, block, block, j}
};

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(unsigned long long* m, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(m)), "r"(c));
}
__device__ __forceinline__ void mb_wait(unsigned long long* m, unsigned par) {
  unsigned done = 0;
  while (!done)
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}\n"
        : "=r"(done)
        : "r"(sa(m)), "r"(par)
        : "memory");
}
__device__ __forceinline__ void mb_expect(unsigned long long* m, unsigned b) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(m)), "r"(b) : "memory");
}
__device__ __forceinline__ void mb_arrive(unsigned long long* m) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(m)) : "memory");
}
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* map, int c0, int c1, int c2, unsigned long long* m) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(sa(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(sa(m))
      : "memory");
}
// shared-memory matrix descriptor: K-major, 128-byte swizzle, 8-row core groups 1024 B apart
__device__ __forceinline__ uint64_t sw128(unsigned saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ void mma_i8(unsigned tmem, uint64_t ad, uint64_t bd, unsigned idesc, unsigned acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(
          tmem),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(unsigned long long* m) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(m)) : "memory");
}
__device__ __forceinline__ void tmem_ld32(unsigned taddr, int (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

template <bool AMN>
__global__ void __launch_bounds__(kI8Threads, 1)
    oz_i8gemm_kernel(const __grid_constant__ I8Args a, const __grid_constant__ CUtensorMap mapA,
                     const __grid_constant__ CUtensorMap mapB) {
  extern __shared__ unsigned char raw[];
  unsigned char* base = raw + ((1024u - (sa(raw) & 1023u)) & 1023u);
  I8Stage* st = reinterpret_cast<I8Stage*>(base);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(st + INS);
  unsigned long long* empty = full + INS;
  unsigned long long* tfull = empty + INS;
  unsigned long long* tempty = tfull + 2;
  unsigned* tmem_slot = reinterpret_cast<unsigned*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < INS; ++s) {
      mb_init(&full[s], 1);
      mb_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mb_init(&tfull[b], 1);
      mb_init(&tempty[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tmem = *tmem_slot;
  const int per = a.tiles_m * a.tiles_n;
  const int n_items = per * NMOD * a.splits;
  if (warp == 0) {
    if (lane == 0) {
      unsigned q = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int js = it / per, r = it % per;
        const int j = js % NMOD, s = js / NMOD;
        const int m0 = (r / a.tiles_n) * IBM, n0 = (r % a.tiles_n) * IBN;
        const int kb0 = s * a.kb_per_split, kb1 = min(a.kblocks, kb0 + a.kb_per_split);
        for (int kb = kb0; kb < kb1; ++kb, ++q) {
          const int sl = q % INS;
          if (q >= INS) mb_wait(&empty[sl], ((q / INS) - 1) & 1);
          mb_expect(&full[sl], sizeof(I8Stage));
          if constexpr (AMN)
            tma3(st[sl].A, &mapA, m0, kb * IBK, j, &full[sl]);  // [k rows][128 m] box
          else
            tma3(st[sl].A, &mapA, kb * IBK, m0, j, &full[sl]);
          tma3(st[sl].B, &mapB, kb * IBK, n0, j, &full[sl]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // D s32, A s8, B s8, both K-major, N >> 3 at bit 17, M >> 4 at bit 24
      const unsigned idesc = (2u << 4) | (1u << 7) | (1u << 10) | (AMN ? (1u << 15) : 0u) | ((unsigned)(IBN >> 3) << 17) |
                             ((unsigned)(IBM >> 4) << 24);
      unsigned q = 0, u = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++u) {
        const int js = it / per;
        const int s = js / NMOD;
        const int kb0 = s * a.kb_per_split, kb1 = min(a.kblocks, kb0 + a.kb_per_split);
        const int buf = u & 1;
        if (u >= 2) mb_wait(&tempty[buf], ((u >> 1) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const unsigned d = tmem + buf * IBN;
        for (int kb = kb0; kb < kb1; ++kb, ++q) {
          const int sl = q % INS;
          mb_wait(&full[sl], (q / INS) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t ad = sw128(sa(st[sl].A)), bd = sw128(sa(st[sl].B));
#pragma unroll
          for (int k = 0; k < IBK / 32; ++k)  // K-major: 32 bytes along the row; MN-major: 32 rows of 128 B
            mma_i8(d, ad + (AMN ? 256 : 2) * k, bd + 2 * k, idesc, (kb > kb0 || k) ? 1u : 0u);
          mma_commit(&empty[sl]);
        }
        mma_commit(&tfull[buf]);
      }
    }
  } else {
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    unsigned u = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++u) {
      const int buf = u & 1;
      const int js = it / per, r = it % per;
      const int j = js % NMOD;
      const int m0 = (r / a.tiles_n) * IBM, n0 = (r % a.tiles_n) * IBN;
      double mj = 0.0;
#pragma unroll
      for (int jj = 0; jj < NMOD; ++jj)
        if (jj == j) mj = (double)mod_of(jj);
      const double inv = 1.0 / mj;
      mb_wait(&tfull[buf], (u >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int m = m0 + row;
      int8_t* o = a.res + (int64_t)js * a.plane + m;
      const int ncols = min(IBN, a.N - n0);
#pragma unroll 1
      for (int c = 0; c < IBN; c += 32) {
        if (c >= ncols) break;  // warp-uniform
        int v[32];
        tmem_ld32(tmem + ((unsigned)(quarter * 32) << 16) + buf * IBN + c, v);
        if (m < a.M) {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            if (c + i < ncols) {
              const double x = (double)v[i];
              const double qq = fma(x, inv, kMagic) - kMagic;
              const double rr = fma(-qq, mj, x);
              o[(int64_t)(n0 + c + i) * a.ldo] = (int8_t)(__double2loint(rr + kMagic) & 0xFF);
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mb_arrive(&tempty[buf]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ------------------------------------------------------------------------------------------------
// CTA-pair variant (tcgen05.mma.cta_group::2): a cluster of two CTAs on one TPC computes a 256 x 512
// item (the full TMEM of both SMs: two 128 x 256 int32 accumulators per CTA).  Per k-block of 128
// each CTA stages its own 128 rows of A (16 KB) and its half of the item's 512 B rows (2 x 128 rows,
// 32 KB) -- L2 traffic per MMA is half of the single-CTA 128 x 256 tile, and an A panel is read once
// per 512 output columns instead of once per 256.  Both CTAs' TMA loads complete on the leader's
// "full" barrier; the leader's one elected lane issues the MMAs (M = 256, N = 256, two per k-step)
// and multicasts the completions (stage release, accumulator ready) to both CTAs; the eight epilogue
// warps of the pair free the accumulators on the leader's barrier.  No accumulator double
// buffering (the epilogue of an item waits for its MMAs; <= ~10% of a short-K item).
constexpr int P_BN = 512;  // output columns per item
struct __align__(1024) I8Stage2 {
  int8_t A[IBM * IBK];      // this CTA's 128 rows
  int8_t B[2][128 * IBK];   // this CTA's 128-row halves of the item's two 256-column MMAs
};
constexpr size_t kI8Smem2 = sizeof(I8Stage2) * INS + 1024 + 256;
constexpr int kI8Threads2 = 320;  // producer, MMA, eight epilogue warps

__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma3_pair(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                          unsigned long long* mbar_local) {
  const unsigned bar = sa(mbar_local) & 0xFEFFFFFFu;  // the leader CTA's barrier at the same offset
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
      "%4}], [%5];" ::"r"(sa(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma5_pair(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3, int c4,
                                          unsigned long long* mbar_local) {
  const unsigned bar = sa(mbar_local) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.5d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
      "%4, %5, %6}], [%7];" ::"r"(sa(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void mma_i8_pair(unsigned tmem, uint64_t ad, uint64_t bd, unsigned idesc, unsigned acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(
          tmem),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit_pair(unsigned long long* m) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(sa(m)),
      "h"((unsigned short)3)
      : "memory");
}
__device__ __forceinline__ void mb_wait_cluster(unsigned long long* m, unsigned par) {
  unsigned done = 0;
  while (!done)
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n selp.u32 "
        "%0,1,0,p;\n}\n"
        : "=r"(done)
        : "r"(sa(m)), "r"(par)
        : "memory");
}
__device__ __forceinline__ void mb_arrive_leader(unsigned long long* m) {
  unsigned remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(sa(m)));
  // relaxed: the TMEM reads completed (tcgen05.wait::ld) before it; a release would also wait for
  // the item's global residue stores to drain before the MMAs of the next item may start
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}

template <bool AMN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kI8Threads2, 1)
    oz_i8gemm2_kernel(const __grid_constant__ I8Args a, const __grid_constant__ CUtensorMap mapA,
                      const __grid_constant__ CUtensorMap mapB) {
  extern __shared__ unsigned char raw[];
  unsigned char* base = raw + ((1024u - (sa(raw) & 1023u)) & 1023u);
  I8Stage2* st = reinterpret_cast<I8Stage2*>(base);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(st + INS);
  unsigned long long* empty = full + INS;
  unsigned long long* tfull = empty + INS;
  unsigned long long* tempty = tfull + 1;
  unsigned* tmem_slot = reinterpret_cast<unsigned*>(tempty + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned rank = cluster_rank();
  if (threadIdx.x == 0) {
    for (int s = 0; s < INS; ++s) {
      mb_init(&full[s], 1);
      mb_init(&empty[s], 1);
    }
    mb_init(tfull, 1);
    mb_init(tempty, 16);  // the pair's sixteen epilogue warps (leader's barrier)
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tmem = *tmem_slot;
  const int per = a.tiles_m * a.tiles_n;  // pair m-tiles (256 rows) x n-blocks (512 columns)
  const int n_items = per * NMOD * a.splits;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  if (warp == 0) {
    if (lane == 0) {
      unsigned q = 0;
      for (int it = cid; it < n_items; it += ncl) {
        const int js = it / per, r = it % per;
        const int j = js % NMOD, s = js / NMOD;
        const int m0 = (r / a.tiles_n) * 256 + 128 * rank, n0 = (r % a.tiles_n) * P_BN + 128 * rank;
        const int kb0 = s * a.kb_per_split, kb1 = min(a.kblocks, kb0 + a.kb_per_split);
        for (int kb = kb0; kb < kb1; ++kb, ++q) {
          const int sl = q % INS;
          if (q >= INS) mb_wait(&empty[sl], ((q / INS) - 1) & 1);
          if (rank == 0) mb_expect(&full[sl], 2 * sizeof(I8Stage2));
          if (a.a_blocked)  // K-major: block (m0 / 128, kb); MN-major (J'^T): block (kb, m0 / 128)
            tma5_pair(st[sl].A, &mapA, 0, 0, AMN ? m0 >> 7 : kb, AMN ? kb : m0 >> 7, j, &full[sl]);
          else if constexpr (AMN)
            tma3_pair(st[sl].A, &mapA, m0, kb * IBK, j, &full[sl]);
          else
            tma3_pair(st[sl].A, &mapA, kb * IBK, m0, j, &full[sl]);
          tma3_pair(st[sl].B[0], &mapB, kb * IBK, n0, j, &full[sl]);
          tma3_pair(st[sl].B[1], &mapB, kb * IBK, n0 + 256, j, &full[sl]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // D s32, A/B s8, M = 256 (pair), N = 256 per MMA
      const unsigned idesc =
          (2u << 4) | (1u << 7) | (1u << 10) | (AMN ? (1u << 15) : 0u) | (256u >> 3) << 17 | (256u >> 4) << 24;
      unsigned q = 0, u = 0;
      for (int it = cid; it < n_items; it += ncl, ++u) {
        const int js = it / per, r = it % per;
        const int s = js / NMOD;
        const int two = (r % a.tiles_n) * P_BN + 256 < a.N;  // second 256-column half present
        const int kb0 = s * a.kb_per_split, kb1 = min(a.kblocks, kb0 + a.kb_per_split);
        if (u >= 1) mb_wait_cluster(tempty, (u - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int kb = kb0; kb < kb1; ++kb, ++q) {
          const int sl = q % INS;
          mb_wait(&full[sl], (q / INS) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t ad = sw128(sa(st[sl].A)), bd0 = sw128(sa(st[sl].B[0])), bd1 = sw128(sa(st[sl].B[1]));
#pragma unroll
          for (int k = 0; k < IBK / 32; ++k) {
            const uint64_t ak = ad + (AMN ? 256 : 2) * k;
            const unsigned acc = (kb > kb0 || k) ? 1u : 0u;
            mma_i8_pair(tmem, ak, bd0 + 2 * k, idesc, acc);
            if (two) mma_i8_pair(tmem + 256, ak, bd1 + 2 * k, idesc, acc);
          }
          mma_commit_pair(&empty[sl]);
        }
        mma_commit_pair(tfull);
      }
    }
  } else {
    // eight epilogue warps: TMEM lane quarter (warp % 4) x column half ((warp - 2) / 4)
    const int quarter = warp & 3, half = (warp - 2) >> 2;
    const int row = quarter * 32 + lane;
    unsigned u = 0;
    for (int it = cid; it < n_items; it += ncl, ++u) {
      const int js = it / per, r = it % per;
      const int j = js % NMOD;
      const int m0 = (r / a.tiles_n) * 256 + 128 * rank, n0 = (r % a.tiles_n) * P_BN;
      double mj = 0.0;
#pragma unroll
      for (int jj = 0; jj < NMOD; ++jj)
        if (jj == j) mj = (double)mod_of(jj);
      const double inv = 1.0 / mj;
      mb_wait(tfull, u & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int m = m0 + row;
      int8_t* o = a.res + (int64_t)js * a.plane + m;
      const int ncols = min(P_BN, a.N - n0);
#pragma unroll 1
      for (int c = half * (P_BN / 2); c < (half + 1) * (P_BN / 2); c += 32) {
        if (c >= ncols) break;  // warp-uniform
        int v[32];
        tmem_ld32(tmem + ((unsigned)(quarter * 32) << 16) + c, v);
        if (m < a.M) {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            if (c + i < ncols) {
              const double x = (double)v[i];
              const double qq = fma(x, inv, kMagic) - kMagic;
              const double rr = fma(-qq, mj, x);
              o[(int64_t)(n0 + c + i) * a.ldo] = (int8_t)(__double2loint(rr + kMagic) & 0xFF);
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mb_arrive_leader(tempty);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ------------------------------------------------------------------------------------------------
// CRT reconstruction + scaling: C(m, n) = alpha rw(m) 2^-(ea_m + eb_n) C'(m, n) + beta C(m, n).
// Thread per (n, 4 consecutive m); residues summed over the K-splits.
template <int SPLITS>
__global__ void __launch_bounds__(256) oz_crt_kernel(const int8_t* __restrict__ res, int64_t ldo, int64_t plane,
                                                     int M, int N, const int* __restrict__ ea,
                                                     const int* __restrict__ eb, const double* __restrict__ rw,
                                                     double alpha, double beta, double* __restrict__ C, int64_t ldc,
                                                     const OzTab tb) {
  const int mq = (M + 3) / 4;
  const int64_t total = (int64_t)mq * N;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < total; w += (int64_t)gridDim.x * blockDim.x) {
    const int n = (int)(w / mq);
    const int m0 = (int)(w % mq) * 4;
    double T1[4] = {0, 0, 0, 0}, T2[4] = {0, 0, 0, 0}, T3[4] = {0, 0, 0, 0};
    const int8_t* rp = res + (int64_t)n * ldo + m0;
    // all 16 x SPLITS residue words in flight before the arithmetic
    unsigned wv[SPLITS][NMOD];
#pragma unroll
    for (int sp = 0; sp < SPLITS; ++sp)
#pragma unroll
      for (int j = 0; j < NMOD; ++j) wv[sp][j] = *reinterpret_cast<const unsigned*>(rp + (int64_t)(sp * NMOD + j) * plane);
#pragma unroll
    for (int j = 0; j < NMOD; ++j) {
      int r[4] = {0, 0, 0, 0};
#pragma unroll
      for (int sp = 0; sp < SPLITS; ++sp)
#pragma unroll
        for (int e = 0; e < 4; ++e) r[e] += (int)(int8_t)((wv[sp][j] >> (8 * e)) & 0xFF);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        int x = r[e];
        if (SPLITS > 1) {  // |x| <= 128 splits: bring into [-m/2, m/2]
          const int m = mod_of(j);
          x -= m * __float2int_rn((float)x / (float)m);
        }
        const double xd = (double)x;
        T1[e] = fma(xd, tb.h[j], T1[e]);
        T2[e] = fma(xd, tb.g[j], T2[e]);
        T3[e] = fma(xd, tb.l[j], T3[e]);
      }
    }
    const int ebn = eb[n];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int m = m0 + e;
      if (m >= M) break;
      const int eam = ea[m];
      double v;
      if (eam == kExpNonFinite || ebn == kExpNonFinite) {
        v = __longlong_as_double(0x7ff8000000000000ll);
      } else {
        // C'/M = T1 2^-41 + T2 2^-82 + T3 2^-123  (mod 1, symmetric)
        const double k1 = fma(T1[e], 1.0 / 2199023255552.0, kMagic) - kMagic;  // rint(T1 2^-41)
        const double t1 = fma(-k1, 2199023255552.0, T1[e]);                     // exact, |t1| <= 2^40
        const double lo = T2[e] * (1.0 / 4835703278458516698824704.0) + T3[e] * 9.4039548065783000637e-38;
        const double f = fma(t1, 1.0 / 2199023255552.0, lo);
        v = scale2(f * tb.md, -(eam + ebn));
      }
      if (rw) v *= rw[m];
      v *= alpha;
      double* dst = C + (int64_t)n * ldc + m;
      if (beta != 0.0) v = fma(beta, *dst, v);
      *dst = v;
    }
  }
}

PFN_cuTensorMapEncodeTiled_v12000 oz_encode() {
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

// [NMOD][rows][ld] int8 residues, K = valid row length: box {128 k, box_rows, 1}
bool encode_res(CUtensorMap* m, const int8_t* p, int K, int rows, int64_t ld, int64_t plane, int box_rows) {
  auto enc = oz_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)rows, (cuuint64_t)NMOD};
  cuuint64_t strides[2] = {(cuuint64_t)ld, (cuuint64_t)plane};
  cuuint32_t box[3] = {IBK, (cuuint32_t)box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(p), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

static double g_oz_ops = 0.0;  // INT8 tensor ops (2 M N K per modulus) launched so far
int g_oz_pair = 1;             // option "i8_pair": CTA-pair (cta_group::2) INT8 GEMM
double oz_i8_ops_total() { return g_oz_ops; }
static double g_oz_conv = 0.0;  // FP64 elements converted to residues so far
double oz_conv_elems_total() { return g_oz_conv; }

int oz_bits(int64_t K) {
  const double t = std::floor((tab().log2m - 1.0 - std::log2((double)std::max<int64_t>(K, 1)) - 1e-9) / 2.0);
  return (int)std::min(53.0, t);
}

int oz_splits(int64_t K) {
  const int64_t kb = (K + IBK - 1) / IBK;
  const int64_t max_kb = kOzMaxKSplit / IBK;  // K-blocks per split with an exact int32 accumulator
  return (int)((kb + max_kb - 1) / max_kb);
}

cudaError_t oz_exps(const unsigned long long* maxbits, int n, int t, int* exps, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  probe_before(K_OZCONV, st);
  oz_exps_kernel<<<(n + 255) / 256, 256, 0, st>>>(maxbits, n, t, exps);
  probe_after(K_OZCONV, st);
  return cudaGetLastError();
}

cudaError_t oz_exps_log(const long long* logmax, int n, int t, int* exps, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  probe_before(K_OZCONV, st);
  oz_exps_log_kernel<<<(n + 255) / 256, 256, 0, st>>>(logmax, n, t, exps);
  probe_after(K_OZCONV, st);
  return cudaGetLastError();
}

// persistent grid: resident CTAs per SM x 148 (queried once per kernel; sets the smem attribute)
template <typename Kern>
static cudaError_t persistent_grid(Kern k, size_t smem, int& grid) {
  if (grid > 0) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, 256, smem);
  if (e != cudaSuccess) return e;
  grid = 148 * std::max(per, 1);
  return cudaSuccess;
}

cudaError_t oz_rows(const double* A, int64_t lda, int rows, int K, int t, int8_t* out, int64_t ldo, int64_t plane,
                    int* exps, bool have_exps, cudaStream_t st, const int* colexp, int colsign) {
  if (rows <= 0 || K <= 0) return cudaSuccess;
  if ((ldo & 15) || K > ldo || K > lda || (lda & 1) || (reinterpret_cast<uintptr_t>(A) & 15) ||
      (colexp && (reinterpret_cast<uintptr_t>(colexp) & 15)) || (colsign != 1 && colsign != -1))
    return cudaErrorInvalidValue;
  static int grid[2] = {0, 0};
  const bool hc = colexp != nullptr;
  const cudaError_t ea = hc ? persistent_grid(oz_rows_kernel<true>, kRowsSmem, grid[1])
                            : persistent_grid(oz_rows_kernel<false>, kRowsSmem, grid[0]);
  if (ea != cudaSuccess) return ea;
  if (!have_exps) {
    probe_before(K_OZCONV, st);
    oz_rowmax_kernel<<<rows, 256, 0, st>>>(A, lda, rows, K, t, exps, colexp, colsign);
    probe_after(K_OZCONV, st);
  }
  const int64_t tiles = (int64_t)rows * ((ldo + kRowsK - 1) / kRowsK);
  g_oz_conv += (double)rows * K;
  const int gr = (int)std::min<int64_t>(tiles, grid[hc]);
  probe_before(K_OZCONV, st);
  if (hc)
    oz_rows_kernel<true><<<gr, 256, kRowsSmem, st>>>(A, lda, rows, K, exps, colexp, colsign, out, ldo, plane, tab());
  else
    oz_rows_kernel<false><<<gr, 256, kRowsSmem, st>>>(A, lda, rows, K, exps, nullptr, 1, out, ldo, plane, tab());
  probe_after(K_OZCONV, st);
  return cudaGetLastError();
}

cudaError_t oz_rows_blocked(const double* A, int64_t lda, int rows, int K, int nrb, int ncb, const int* rexp,
                            const int* cexp, int8_t* out, int64_t plane, cudaStream_t st) {
  if (rows <= 0 || K <= 0) return cudaSuccess;
  if ((lda & 1) || (reinterpret_cast<uintptr_t>(A) & 15) || (int64_t)nrb * 128 < rows || (int64_t)ncb * 128 < K ||
      (int64_t)ncb * 128 > lda + 127 || (plane & 15) || plane < (int64_t)nrb * ncb * 16384)
    return cudaErrorInvalidValue;
  static int grid = 0;
  const cudaError_t ea = persistent_grid(oz_rows_blocked_kernel, kBlkSmem, grid);
  if (ea != cudaSuccess) return ea;
  const int64_t tiles = (int64_t)nrb * 8 * ncb;
  g_oz_conv += (double)rows * K;
  probe_before(K_OZCONV, st);
  oz_rows_blocked_kernel<<<(int)std::min<int64_t>(tiles, grid), 256, kBlkSmem, st>>>(A, lda, rows, K, nrb, ncb, rexp,
                                                                                       cexp, out, plane, tab());
  probe_after(K_OZCONV, st);
  return cudaGetLastError();
}

cudaError_t oz_i8gemm(const int8_t* A, int64_t lda, int64_t planeA, bool a_mn, int M, const int8_t* B, int64_t ldb,
                      int64_t planeB, int N, int K, int8_t* res, int64_t ldo, int64_t planeO, cudaStream_t st,
                      int a_nrb, int a_ncb) {
  if (M <= 0 || N <= 0 || K <= 0) return cudaSuccess;
  const bool blocked = a_nrb > 0;
  const int64_t a_inner = a_mn ? M : K, a_outer = a_mn ? K : M;
  if ((lda & 15) || (ldb & 15) || (ldo & 3) || (!blocked && a_inner > lda) || K > ldb || M > ldo || (planeA & 15) ||
      (planeB & 15) || (planeO & 3) || (!blocked && planeA < lda * a_outer) || planeB < ldb * N || planeO < ldo * N)
    return cudaErrorInvalidValue;
  if (blocked && (!g_oz_pair || planeA < (int64_t)a_nrb * a_ncb * 16384 ||
                  (int64_t)(a_mn ? a_ncb : a_nrb) * 128 < M || (int64_t)(a_mn ? a_nrb : a_ncb) * 128 < K))
    return cudaErrorInvalidValue;
  static bool attr[4] = {false, false, false, false};
  const bool pair = g_oz_pair != 0;
  const int ai = (a_mn ? 1 : 0) + (pair ? 2 : 0);
  if (!attr[ai]) {
    const cudaError_t e =
        pair ? cudaFuncSetAttribute(a_mn ? oz_i8gemm2_kernel<true> : oz_i8gemm2_kernel<false>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kI8Smem2)
             : cudaFuncSetAttribute(a_mn ? oz_i8gemm_kernel<true> : oz_i8gemm_kernel<false>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kI8Smem);
    if (e != cudaSuccess) return e;
    attr[ai] = true;
  }
  I8Args a{};
  a.M = M;
  a.N = N;
  a.tiles_m = pair ? (M + 255) / 256 : (M + IBM - 1) / IBM;
  a.tiles_n = pair ? (N + P_BN - 1) / P_BN : (N + IBN - 1) / IBN;
  a.kblocks = (K + IBK - 1) / IBK;
  a.splits = oz_splits(K);
  a.kb_per_split = (a.kblocks + a.splits - 1) / a.splits;
  a.res = res;
  a.ldo = ldo;
  a.plane = planeO;
  a.a_blocked = blocked ? 1 : 0;
  CUtensorMap ma, mb;
  bool ok_a;
  if (blocked) {  // [j][row block][column block][128][128]
    auto enc = oz_encode();
    cuuint64_t dims[5] = {128, 128, (cuuint64_t)a_ncb, (cuuint64_t)a_nrb, (cuuint64_t)NMOD};
    cuuint64_t strides[4] = {128, 16384, (cuuint64_t)a_ncb * 16384, (cuuint64_t)planeA};
    cuuint32_t box[5] = {128, 128, 1, 1, 1};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    ok_a = enc && enc(&ma, CU_TENSOR_MAP_DATA_TYPE_UINT8, 5, const_cast<int8_t*>(A), dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  } else {
    ok_a = a_mn ? encode_res(&ma, A, M, K, lda, planeA, IBK)   // box {128 m, 128 k}
                : encode_res(&ma, A, K, M, lda, planeA, IBM);  // box {128 k, 128 m}
  }
  if (!ok_a || !encode_res(&mb, B, K, N, ldb, planeB, pair ? 128 : IBN)) return cudaErrorInvalidValue;
  const int items = a.tiles_m * a.tiles_n * NMOD * a.splits;
  const int grid = pair ? 2 * std::min(items, 74) : std::min(items, 148);
  g_oz_ops += 2.0 * NMOD * (double)M * N * (double)K;
  probe_before(K_I8GEMM, st);
  if (pair) {
    if (a_mn)
      oz_i8gemm2_kernel<true><<<grid, kI8Threads2, kI8Smem2, st>>>(a, ma, mb);
    else
      oz_i8gemm2_kernel<false><<<grid, kI8Threads2, kI8Smem2, st>>>(a, ma, mb);
  } else if (a_mn) {
    oz_i8gemm_kernel<true><<<grid, kI8Threads, kI8Smem, st>>>(a, ma, mb);
  } else {
    oz_i8gemm_kernel<false><<<grid, kI8Threads, kI8Smem, st>>>(a, ma, mb);
  }
  probe_after(K_I8GEMM, st);
  return cudaGetLastError();
}

cudaError_t oz_crt(const int8_t* res, int64_t ldo, int64_t planeO, int M, int N, int splits, const int* ea,
                   const int* eb, const double* row_w, double alpha, double beta, double* C, int64_t ldc,
                   cudaStream_t st) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  if ((ldo & 3) || (planeO & 3) || splits < 1 || splits > 4) return cudaErrorInvalidValue;
  const int64_t total = (int64_t)((M + 3) / 4) * N;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  probe_before(K_OZCRT, st);
  switch (splits) {
    case 1: oz_crt_kernel<1><<<blocks, 256, 0, st>>>(res, ldo, planeO, M, N, ea, eb, row_w, alpha, beta, C, ldc, tab()); break;
    case 2: oz_crt_kernel<2><<<blocks, 256, 0, st>>>(res, ldo, planeO, M, N, ea, eb, row_w, alpha, beta, C, ldc, tab()); break;
    case 3: oz_crt_kernel<3><<<blocks, 256, 0, st>>>(res, ldo, planeO, M, N, ea, eb, row_w, alpha, beta, C, ldc, tab()); break;
    case 4: oz_crt_kernel<4><<<blocks, 256, 0, st>>>(res, ldo, planeO, M, N, ea, eb, row_w, alpha, beta, C, ldc, tab()); break;
    default: break;  // K > 4 x 130944: rejected above
  }
  probe_after(K_OZCRT, st);
  return cudaGetLastError();
}

}  // namespace ngd
