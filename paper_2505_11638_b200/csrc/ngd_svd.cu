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
#include <cstdlib>
#include <cstring>
#include <vector>
#include <mutex>
#include <map>
#include <memory>
#include <algorithm>

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

// ---------------------------------------------------------------------------
// Block-exchange variant: every rotation touches only LOCAL shared memory.
// The n (padded) columns form 2*CL blocks of h columns; CTA k holds two blocks.
// A sweep = one round-robin tournament of the 2*CL blocks (circle method):
//   super-round 0 also rotates all pairs inside each block (h-1 local rounds),
//   every super-round rotates all cross pairs of the CTA's two blocks (h local
//   rounds of h disjoint pairs), then blocks move to the CTA that pairs them in
//   the next super-round.  Columns: X = R^T and V = I, as in jsvd_kernel.
//
// Measured on B200 (tools/probe/jsvd_acc.cu, jround.cu): a round costs ~1000
// cycles of dependent latency for a single warp (partner-column load, Gram
// butterfly, rotation parameters, update) and ~1500 with 10 warps sharing the
// SM; an exchange was two cluster barriers plus DSMEM pulls.  Hence: in the
// cross rounds warp i keeps column i of block 0 (X and V) in registers so only
// the partner column moves through shared memory; rotation parameters take two
// rsqrt (plus one Newton step for orthogonality) instead of Rutishauser's
// rcp/sqrt/rcp/rsqrt chain; blocks move by bulk-async pushes (cp.async.bulk
// shared::cta -> shared::cluster, completion on the receiver's mbarrier) behind
// a single cluster barrier.  (Keeping V in L2 and applying each super-round's
// accumulated rotation with DMMA was measured slower: at one SM's FP64 rate that
// update costs as much as the direct rotations.)
#ifdef NGD_SVD_TRACE
__device__ unsigned long long g_tr[16 * 16];  // [CTA][counter], thread 0 of each CTA
#define TR_T(v) long long v = clock64()
#define TR_ADD(k, d) do { if (threadIdx.x == 0) g_tr[blockIdx.x * 16 + (k)] += (unsigned long long)(d); } while (0)
#else
#define TR_T(v)
#define TR_ADD(k, d)
#endif
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ unsigned cluster_addr(unsigned a, int rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}

__device__ __forceinline__ void mbar_wait(unsigned mbar, unsigned parity) {
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(mbar), "r"(parity)
        : "memory");
  }
}

// Jacobi rotation (c, s) annihilating the (al, be, ga) Gram pair: tan(2 theta) = 2 ga / (be - al),
// |theta| <= pi/4.  cos(2 theta) = |d| / r, sin(2 theta) = sign(d) 2 ga / r, c = sqrt((1 + cos 2theta)/2),
// s = sin(2 theta) / (2 c): two rsqrt instead of Rutishauser's rcp/sqrt/rcp/rsqrt chain.
__device__ __forceinline__ void jacobi_cs(double al, double be, double ga, double& c, double& s) {
  double d = be - al, g2 = 2.0 * ga;
  const double m = fmax(fabs(d), fabs(g2));
  if (m > 1e150 || m < 1e-150) {  // keep d^2 + g2^2 representable
    const double sc = 1.0 / m;
    d *= sc;
    g2 *= sc;
  }
  const double ri = rsqrt(fma(d, d, g2 * g2));
  const double cos2 = fabs(d) * ri;
  const double sin2 = (d < 0.0 ? -g2 : g2) * ri;
  const double hh = fma(0.5, cos2, 0.5);
  const double rh = rsqrt(hh);
  c = hh * rh;
  s = 0.5 * sin2 * rh;
  // one Newton step on 1/sqrt(c^2 + s^2): rsqrt is not correctly rounded, and a rotation that is
  // off-orthogonal by a few ulp would drift column norms over thousands of rotations
  const double f = fma(-0.5, fma(c, c, fma(s, s, -1.0)), 1.0);
  c *= f;
  s *= f;
}

// FP32 twin for the single-precision pre-sweeps (orthogonality is restored in FP64 afterwards)
__device__ __forceinline__ void jacobi_cs(float al, float be, float ga, float& c, float& s) {
  float d = be - al, g2 = 2.0f * ga;
  const float m = fmaxf(fabsf(d), fabsf(g2));
  if (m > 1e18f || m < 1e-18f) {
    const float sc = 1.0f / m;
    d *= sc;
    g2 *= sc;
  }
  const float ri = rsqrtf(fmaf(d, d, g2 * g2));
  const float cos2 = fabsf(d) * ri;
  const float sin2 = (d < 0.0f ? -g2 : g2) * ri;
  const float hh = fmaf(0.5f, cos2, 0.5f);
  const float rh = rsqrtf(hh);
  c = hh * rh;
  s = 0.5f * sin2 * rh;
  const float f = fmaf(-0.5f, fmaf(c, c, fmaf(s, s, -1.0f)), 1.0f);
  c *= f;
  s *= f;
}

template <typename T> struct Vec2;
template <> struct Vec2<double> { using type = double2; };
template <> struct Vec2<float> { using type = float2; };
template <typename T> using vec2_t = typename Vec2<T>::type;

__device__ __forceinline__ double fmx(double a, double b, double c) { return fma(a, b, c); }
__device__ __forceinline__ float fmx(float a, float b, float c) { return fmaf(a, b, c); }

// warp-wide Gram entries of two register-resident columns
template <int RPL, typename T>
__device__ __forceinline__ void gram3(const vec2_t<T> (&x)[RPL], const vec2_t<T> (&y)[RPL], T& al, T& be, T& ga) {
  al = T(0);
  be = T(0);
  ga = T(0);
#pragma unroll
  for (int u = 0; u < RPL; ++u) {
    al = fmx(x[u].x, x[u].x, al);
    be = fmx(y[u].x, y[u].x, be);
    ga = fmx(x[u].x, y[u].x, ga);
    al = fmx(x[u].y, x[u].y, al);
    be = fmx(y[u].y, y[u].y, be);
    ga = fmx(x[u].y, y[u].y, ga);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {  // three interleaved butterfly reductions
    al += __shfl_xor_sync(0xffffffffu, al, o);
    be += __shfl_xor_sync(0xffffffffu, be, o);
    ga += __shfl_xor_sync(0xffffffffu, ga, o);
  }
}

// CG: a V column in global memory (written by other CTAs of the cluster): bypass L1
template <int RPL, typename T, bool CG = false>
__device__ __forceinline__ void load_col(vec2_t<T> (&x)[RPL], const T* col, int nq, int lane) {
  const vec2_t<T>* c2 = reinterpret_cast<const vec2_t<T>*>(col);
#pragma unroll
  for (int u = 0; u < RPL; ++u) {
    const int q = lane + 32 * u;
    if constexpr (CG)
      x[u] = q < nq ? __ldcg(c2 + q) : vec2_t<T>{T(0), T(0)};
    else
      x[u] = q < nq ? c2[q] : vec2_t<T>{T(0), T(0)};
  }
}

template <int RPL, typename T>
__device__ __forceinline__ void store_col(T* col, const vec2_t<T> (&x)[RPL], int nq, int lane) {
  vec2_t<T>* c2 = reinterpret_cast<vec2_t<T>*>(col);
#pragma unroll
  for (int u = 0; u < RPL; ++u) {
    const int q = lane + 32 * u;
    if (q < nq) c2[q] = x[u];
  }
}

template <int RPL, typename T>
__device__ __forceinline__ void rot2(vec2_t<T> (&x)[RPL], vec2_t<T> (&y)[RPL], T c, T s) {
#pragma unroll
  for (int u = 0; u < RPL; ++u) {
    const vec2_t<T> a = x[u], b = y[u];
    x[u] = vec2_t<T>{c * a.x - s * b.x, c * a.y - s * b.y};
    y[u] = vec2_t<T>{s * a.x + c * b.x, s * a.y + c * b.y};
  }
}

// rotate two column pairs (X in shared memory, V in shared or global memory) in place; one warp.  Rotates when the relative
// coupling |ga| / sqrt(al be) exceeds tol (tol2 = tol^2); 'big' records a coupling^2 >= tbig.
template <int RPL, typename T, bool VG = false>
__device__ __forceinline__ bool rotate_pair(T* ci, T* cj, T* vi, T* vj, int ldc, int lane, T tol2, T tbig,
                                            bool& big) {
  const int nq = ldc >> 1;
  vec2_t<T> x[RPL], y[RPL];
  load_col<RPL, T>(x, ci, nq, lane);
  load_col<RPL, T>(y, cj, nq, lane);
  T al, be, ga;
  gram3<RPL, T>(x, y, al, be, ga);
  if (!(ga != T(0) && ga * ga > tol2 * al * be)) return false;
  big |= ga * ga >= tbig * (al * be);
  T c, s;
  jacobi_cs(al, be, ga, c, s);
  rot2<RPL, T>(x, y, c, s);
  store_col<RPL, T>(ci, x, nq, lane);
  store_col<RPL, T>(cj, y, nq, lane);
  load_col<RPL, T, VG>(x, vi, nq, lane);
  load_col<RPL, T, VG>(y, vj, nq, lane);
  rot2<RPL, T>(x, y, c, s);
  store_col<RPL, T>(vi, x, nq, lane);
  store_col<RPL, T>(vj, y, nq, lane);
  return true;
}

// 16 warps: one column pair per warp and local round (h <= 16)
constexpr int kBlockSvdThreads = 512;
constexpr int kPlanMax = 256;  // exchanges per schedule period (CL = 16, three buffers: 6 sweeps x 31)

// Exchange schedule of the block tournament (circle method on nb = 2 CL blocks), NB = 3 or 4 block
// buffers per CTA (two held, the others free).  Consecutive rounds share no pair, so the graph
// "CTA -- next-round pair containing one of its blocks" is 2-regular and has a perfect matching:
// every CTA keeps one block in place and receives its new partner into a free buffer.  Three
// buffers: into the free one, the buffer it sent from becomes free.  Four: buffers s and s + 2 belong
// to slot s, and the slot that sends receives into its other buffer (a FIFO over the two free
// buffers measured the same).  The placement sequence repeats after a few sweeps (CL = 16: 6 with
// three buffers, 4 with four).
// Word (t, c): bits 0-1 source buffer, 2-5 destination CTA, 6-7 destination buffer, 8-12 / 13-17
// blocks held after the move (slots 0, 1), 18-19 / 20-21 their buffers.
// Point-to-point exchange: a CTA may write its outgoing block into buffer b of CTA d as soon as
// every earlier copy OUT of that buffer has landed -- counted in d's gen[b], incremented by the
// receiver of each copy.  Word2 (t, c): bits 0-7 the count required at the first period, 8-15 its
// increase per period, 16-19 the CTA that sends to c at t, 20-21 that sender's source buffer.  Data
// of consecutive exchanges lands on alternating mbarriers (exchange t + 2 cannot reach a CTA before
// it consumed t).  Verified on random asynchronous schedules (no write into an in-flight source or
// a held block, no stall), as emitted here: tools/probe/jsvd_pool_check.py.
struct JsvdPlan {
  int period = 0;                      // exchanges
  std::vector<unsigned> w, w2;         // [period][CL]
};
// the schedule as a kernel parameter (constant bank: the exchange path is latency bound -- words
// read from global memory measured 2% slower on C2's factor, a shared-memory copy 1%)
constexpr int kPlanWords = 3072;  // >= period * CL (three buffers, CL = 16: 186 x 16)
struct JsvdPlanArg {
  int period;
  int p2p;
  unsigned w[kPlanWords];
  unsigned w2[kPlanWords];
};

static bool jsvd_make_plan(int CL, int NB, JsvdPlan& P) {
  const int nb = 2 * CL, m = nb - 1;
  auto circle = [&](int r, int kk, int& a, int& b) {
    if (kk == 0) {
      a = 0;
      b = 1 + r;
    } else {
      a = 1 + (r + kk) % m;
      b = 1 + ((r - kk) % m + m) % m;
    }
  };
  int blk[16][2] = {}, bf[16][2] = {}, fr[16][2] = {};  // held blocks, their buffers, free buffers (FIFO)
  auto reset = [&] {
    for (int c = 0; c < CL; ++c) {
      circle(0, c, blk[c][0], blk[c][1]);
      bf[c][0] = 0;
      bf[c][1] = 1;
      fr[c][0] = 2;
      fr[c][1] = 3;
    }
  };
  // one exchange (to round r_to) of the current state; fills word row t if w != nullptr
  auto step = [&](int r_to, unsigned* w) {
    int pa[16][2], pair_of[32], hold_c[32], hold_s[32], assigned[16], keep[16], owner[16];
    for (int j = 0; j < CL; ++j) {
      circle(r_to, j, pa[j][0], pa[j][1]);
      pair_of[pa[j][0]] = pair_of[pa[j][1]] = j;
    }
    for (int c = 0; c < CL; ++c) {
      assigned[c] = -1;
      for (int s = 0; s < 2; ++s) {
        hold_c[blk[c][s]] = c;
        hold_s[blk[c][s]] = s;
      }
    }
    for (int c0 = 0; c0 < CL; ++c0) {  // walk each alternating cycle
      if (assigned[c0] >= 0) continue;
      int c = c0, x = blk[c0][0];
      while (true) {
        const int j = pair_of[x];
        assigned[c] = j;
        owner[j] = c;
        keep[c] = hold_s[x];
        const int z = pa[j][0] == x ? pa[j][1] : pa[j][0];
        const int c2 = hold_c[z];
        if (assigned[c2] >= 0) break;
        c = c2;
        x = blk[c2][hold_s[z] ^ 1];
      }
    }
    int nblk[16][2], nbf[16][2], nfr[16][2];  // (rows >= CL: unused, kept equal for the period test)
    memcpy(nblk, blk, sizeof(blk));
    memcpy(nbf, bf, sizeof(bf));
    memcpy(nfr, fr, sizeof(fr));
    for (int c = 0; c < CL; ++c) {
      const int os = keep[c] ^ 1, kept = blk[c][keep[c]], j = assigned[c];
      nblk[c][keep[c]] = kept;
      nbf[c][keep[c]] = bf[c][keep[c]];
      nblk[c][os] = pa[j][0] == kept ? pa[j][1] : pa[j][0];
      if (NB == 4) {  // buffers 2 s + phase belong to slot s: receive into the slot's other phase
        nbf[c][os] = bf[c][os] ^ 2;
      } else {  // receive into the free buffer, the one sent from becomes free
        nbf[c][os] = fr[c][0];
        nfr[c][0] = bf[c][os];
      }
    }
    if (w)
      for (int c = 0; c < CL; ++c) {
        const int os = keep[c] ^ 1, y = blk[c][os];
        const int d = owner[pair_of[y]];
        w[c] = (unsigned)bf[c][os] | ((unsigned)d << 2) | ((unsigned)nbf[d][keep[d] ^ 1] << 6) | ((unsigned)nblk[c][0] << 8) |
               ((unsigned)nblk[c][1] << 13) | ((unsigned)nbf[c][0] << 18) | ((unsigned)nbf[c][1] << 20);
      }
    memcpy(blk, nblk, sizeof(blk));
    memcpy(bf, nbf, sizeof(bf));
    memcpy(fr, nfr, sizeof(fr));
  };
  // period: sweeps until the state at a sweep boundary returns to the initial one
  reset();
  int sweeps = 0;
  int b0[16][2], f0[16][2], r0[16][2];
  memcpy(b0, blk, sizeof(blk));
  memcpy(f0, bf, sizeof(bf));
  memcpy(r0, fr, sizeof(fr));
  for (sweeps = 1; sweeps <= 16; ++sweeps) {
    for (int t = 0; t < m; ++t) step((t + 1) % m, nullptr);
    if (!memcmp(b0, blk, sizeof(blk)) && !memcmp(f0, bf, sizeof(bf)) && !memcmp(r0, fr, sizeof(fr))) break;
  }
  if (sweeps > 16 || sweeps * m > kPlanMax) return false;
  const int period = sweeps * m;
  P.period = period;
  P.w.assign((size_t)period * CL, 0u);
  P.w2.assign((size_t)period * CL, 0u);
  reset();
  for (int t = 0; t < period; ++t) step((t + 1) % m, &P.w[(size_t)t * CL]);
  // point-to-point permissions from three periods of the (periodic) schedule
  const int T = 3 * period;
  auto dec = [&](int t, int c, int& sb, int& dc, int& db) {
    const unsigned w = P.w[(size_t)(t % period) * CL + c];
    sb = w & 3;
    dc = (w >> 2) & 15;
    db = (w >> 6) & 3;
  };
  std::vector<int> uses[16][4];  // source-use exchanges per (cta, buffer)
  for (int t = 0; t < T; ++t)
    for (int c = 0; c < CL; ++c) {
      int sb, dc, db;
      dec(t, c, sb, dc, db);
      uses[c][sb].push_back(t);
    }
  auto req = [&](int t, int c) {
    int sb, dc, db;
    dec(t, c, sb, dc, db);
    int n = 0;
    for (int u : uses[dc][db]) n += (u < t) ? 1 : 0;
    return n;
  };
  for (int t = 0; t < period; ++t)
    for (int c = 0; c < CL; ++c) {
      const int base = req(t, c), upp = req(t + period, c) - base;
      if (base > 255 || upp > 255 || req(t + 2 * period, c) - req(t + period, c) != upp) return false;
      int snd = -1, ssb = 0;
      for (int e = 0; e < CL; ++e) {
        int sb, dc, db;
        dec(t, e, sb, dc, db);
        if (dc == c) {
          snd = e;
          ssb = sb;
        }
      }
      if (snd < 0) return false;
      P.w2[(size_t)t * CL + c] = (unsigned)base | ((unsigned)upp << 8) | ((unsigned)snd << 16) | ((unsigned)ssb << 20);
    }
  return true;
}

// T = double: the FP64 Jacobi (outputs sigma descending and U = V sorted; V starts at V0 when given,
// else I).  T = float: single-precision pre-sweeps on X = s A^T (s a power of two bringing max|A| to
// [0.5, 1)); sigma == nullptr selects the raw output: V (unsorted, as double) into U[j * ldu + r].
// vglobal: V is not kept in shared memory but updated in place in Vg (ldv, column = global column
// id; the FP64 finish for ell > 310, where X alone fills the cluster's shared memory) -- each
// column has exactly one owner CTA at a time, and V never moves between CTAs.
template <typename T, int RPL, bool VG>
__global__ void __launch_bounds__(kBlockSvdThreads, 1) jsvd_block_kernel(const double* A, int ell, int lda,
                                                                           const double* Vin, double* Vg, int ldv,
                                                                           double* U, int ldu, double* sigma,
                                                                           double tol, double tbig_d, int max_sweeps,
                                                                           int h, int* info, int nbuf,
                                                                           const __grid_constant__ JsvdPlanArg plan) {
#ifdef NGD_JSVD_ALIGN1024
  extern __shared__ __align__(1024) unsigned char smem_raw[];
#else
  extern __shared__ __align__(16) unsigned char smem_raw[];
#endif
  T* smem = reinterpret_cast<T*>(smem_raw);
  constexpr int NT = kBlockSvdThreads;
  constexpr int NW = NT / 32;
  cg::cluster_group cl = cg::this_cluster();
  const int CL = (int)cl.num_blocks();
  const int k = (int)cl.block_rank();
  const int nb = 2 * CL;  // blocks
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ldc = ell + (ell & 1);  // even column stride: 8/16-B aligned vector columns
  const int nq = ldc >> 1;
  const size_t slot_sz = (size_t)h * ldc;  // one block of X (or V)
  constexpr int nwh = VG ? 1 : 2;          // X (+ V) per block buffer
  const T tol2 = (T)(tol * tol), tbig = (T)tbig_d;
  // nbuf block buffers: buf[b][0 = X, 1 = V][h][ldc], X and V of one buffer contiguous
  auto bufp = [&](int b, int which) { return smem + ((size_t)b * nwh + which) * slot_sz; };
  double* norms = reinterpret_cast<double*>(smem + (size_t)nbuf * nwh * slot_sz);  // [2][h]
  int* flags = reinterpret_cast<int*>(norms + 2 * h);                   // [4]: rotated / large, by sweep parity
  __shared__ __align__(8) unsigned long long mbars[2];                 // block arrivals, by exchange parity
  __shared__ unsigned gen[4];                                          // copies out of each buffer that landed
  const int period = plan.period, p2p = plan.p2p;
#define pw(t) plan.w[(t) * CL + k]
#define pw2(t) plan.w2[(t) * CL + k]
  __shared__ int p2p_err;
  __shared__ int held[2];
  __shared__ double red[NW];
  const unsigned mbar_a = smem_u32(&mbars[0]);
  const unsigned blk_bytes = (unsigned)(nwh * slot_sz * sizeof(T));  // one block buffer
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar_a));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar_a + 8));
    asm volatile("fence.mbarrier_init.release.cluster;");
    for (int b = 0; b < 4; ++b) gen[b] = 0;
    p2p_err = 0;
  }
  double scale = 1.0;
  if constexpr (sizeof(T) == 4) {  // keep FP32 Gram entries far from overflow / underflow
    double m = 0.0;
    for (int64_t e = tid; e < (int64_t)ell * ell; e += NT) m = fmax(m, fabs(A[(e / ell) * lda + e % ell]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) red[warp] = m;
    __syncthreads();
    m = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) m = fmax(m, red[w]);
    if (m > 0.0) {
      int ex;
      frexp(m, &ex);
      scale = ldexp(1.0, -ex);
    }
  }
  int blk[2], bf[2] = {0, 1};
  circle_pair(nb, 0, k, blk[0], blk[1]);
  for (int sl = 0; sl < 2; ++sl) {
    T* X = bufp(bf[sl], 0);
    T* V = VG ? nullptr : bufp(bf[sl], 1);
    for (int64_t e = tid; e < (int64_t)slot_sz; e += NT) {
      const int i = (int)(e / ldc), r = (int)(e % ldc);
      const int j = blk[sl] * h + i;  // global column id
      const bool in = j < ell && r < ell;
      X[e] = in ? (T)(A[(int64_t)r * lda + j] * scale) : T(0);
      if (V) {
        if (Vin)
          V[e] = in ? (T)Vin[(int64_t)j * ldv + r] : T(0);
        else
          V[e] = (j == r && r < ell) ? T(1) : T(0);
      }
    }
  }
  if (tid < 4) flags[tid] = 0;
  cl.sync();
  // V column of global column gid (shared-memory slot or, vglobal, the in-place global column)
  T* V0s = nullptr;  // this round's V blocks in shared memory (!VG)
  T* V1s = nullptr;
  auto vcol = [&](int sl, int i) -> T* {
    if constexpr (!VG) return (sl ? V1s : V0s) + i * ldc;
    const int gid = blk[sl] * h + i;
    return gid < ell ? reinterpret_cast<T*>(Vg + (int64_t)gid * ldv) : nullptr;
  };

  // Move to the next round's placement: one block per CTA crosses DSMEM, the other stays in place
  // (the exchange is DSMEM-bandwidth bound).
  int xt = 0;  // exchanges so far
  auto exchange = [&]() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> async-proxy reads
    const int tp = xt % period, xi = xt;
    const unsigned e = pw(tp);
    ++xt;
    const int sb = e & 3, dc = (e >> 2) & 15, db = (e >> 6) & 3;
    const unsigned mb_own = mbar_a + 8u * (unsigned)(xi & 1);
    TR_T(e0);
    if (p2p) {
      __syncthreads();  // this CTA's rotations are done: the outgoing block is final
      if (tid == 0) {
        const unsigned w2 = pw2(tp);
        const unsigned need = (w2 & 255u) + (unsigned)(xi / period) * ((w2 >> 8) & 255u);
        const unsigned ga = cluster_addr(smem_u32(&gen[db]), dc);
        unsigned have = 0;
        for (long long spin = 0;; ++spin) {  // the destination buffer's earlier copies out have landed
          asm volatile("ld.acquire.cluster.shared::cluster.u32 %0, [%1];" : "=r"(have) : "r"(ga) : "memory");
          if (have >= need) break;
          if (spin > (1ll << 28)) {  // protocol error: never hang the device
            p2p_err = 1;
            break;
          }
        }
      }
    } else {
      cl.sync();  // all rotations done everywhere; every copy of the previous exchange has landed
    }
    if (tid == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb_own), "r"(blk_bytes) : "memory");
      const unsigned src = smem_u32(bufp(sb, 0));
      const unsigned dst = cluster_addr(smem_u32(bufp(db, 0)), dc);
      const unsigned mb = cluster_addr(mbar_a + 8u * (unsigned)(xi & 1), dc);
      asm volatile(
          "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
          "r"(src), "r"(blk_bytes), "r"(mb)
          : "memory");
    }
    TR_T(e1);
    TR_ADD(0, e1 - e0);
    blk[0] = (e >> 8) & 31;
    blk[1] = (e >> 13) & 31;
    bf[0] = (e >> 18) & 3;
    bf[1] = (e >> 20) & 3;
    mbar_wait(mb_own, (unsigned)(xi >> 1) & 1u);
    if (p2p && tid == 0) {  // the sender's source buffer is free again: count it at its owner
      const unsigned w2 = pw2(tp);
      const unsigned ga = cluster_addr(smem_u32(&gen[(w2 >> 20) & 3u]), (int)((w2 >> 16) & 15u));
      asm volatile("red.release.cluster.shared::cluster.add.u32 [%0], 1;" ::"r"(ga) : "memory");
    }
    TR_T(e2);
    TR_ADD(1, e2 - e1);
    TR_ADD(2, 1);
  };

  // info[0]: sweeps (negative: not converged), or -1000 if any CTA's exchange protocol timed out
  auto report = [&](bool conv, int sweeps) {
    cl.sync();  // every CTA's p2p_err is final
    if (k == 0 && tid == 0) {
      int err = 0;
      for (int o = 0; o < CL; ++o) err |= *cl.map_shared_rank(&p2p_err, o);
      info[0] = err ? -1000 : (conv ? sweeps : -sweeps);
    }
    cl.sync();  // keep every CTA's shared memory alive until CTA 0 has read it
  };
  int sweep = 0;
  bool converged = false;
  for (; sweep < max_sweeps && !converged; ++sweep) {
    const int par = sweep & 1;
    bool rotated = false;
    bool big = false;  // a rotation with coupling^2 >= tbig happened in this sweep
    for (int r = 0; r < nb - 1; ++r) {
      T* X0 = bufp(bf[0], 0);
      T* X1 = bufp(bf[1], 0);
      V0s = bufp(bf[0], 1);
      V1s = bufp(bf[1], 1);
      if (r == 0) {  // pairs inside each of the two blocks (circle method on h columns)
        for (int rr = 0; rr < h - 1; ++rr) {
          for (int q = warp; q < h; q += NW) {  // h/2 pairs per block, two blocks
            const int sl = q / (h / 2), kk = q % (h / 2);
            int i, j;
            circle_pair(h, rr, kk, i, j);
            T* X = sl ? X1 : X0;
            T* vi = vcol(sl, i);
            T* vj = vcol(sl, j);
            // (a padded column -- X zero, no global V -- never rotates: ga == 0)
            if (!VG || (vi && vj))
              rotated |= rotate_pair<RPL, T, VG>(X + (size_t)i * ldc, X + (size_t)j * ldc, vi, vj, ldc, lane, tol2, tbig,
                                             big);
          }
          __syncthreads();
        }
      }
      // cross pairs of the two blocks: h rounds of h disjoint pairs (i, i + sft mod h).  Warp i keeps
      // column i of block 0 (X and V) in registers; the partner columns move through shared memory.
      {
        vec2_t<T> xr[RPL], vr[RPL];
        T* vown = nullptr;
        const bool own = warp < h;
        if (own) {
          load_col<RPL, T>(xr, X0 + (size_t)warp * ldc, nq, lane);
          vown = vcol(0, warp);
          if (!VG || vown)  // (compile-time true with V in shared memory: no generic-pointer test)
            load_col<RPL, T, VG>(vr, vown, nq, lane);
          else
#pragma unroll
            for (int u = 0; u < RPL; ++u) vr[u] = vec2_t<T>{T(0), T(0)};
        }
        for (int sft = 0; sft < h; ++sft) {
          TR_T(c0);
          if (own) {
            const int j = (warp + sft >= h) ? warp + sft - h : warp + sft;
            T* yc = X1 + (size_t)j * ldc;
            vec2_t<T> y[RPL];
            load_col<RPL, T>(y, yc, nq, lane);
            T al, be, ga;
            gram3<RPL, T>(xr, y, al, be, ga);
            if (ga != T(0) && ga * ga > tol2 * al * be) {
              big |= ga * ga >= tbig * (al * be);
              T c, s;
              jacobi_cs(al, be, ga, c, s);
              rot2<RPL, T>(xr, y, c, s);
              store_col<RPL, T>(yc, y, nq, lane);
              T* vc = vcol(1, j);
              if (!VG || vc) {  // (vglobal: both columns real whenever ga != 0)
                load_col<RPL, T, VG>(y, vc, nq, lane);
                rot2<RPL, T>(vr, y, c, s);
                store_col<RPL, T>(vc, y, nq, lane);
              }
              rotated = true;
            }
          }
          TR_T(c1);
          __syncthreads();
          TR_T(c2);
          TR_ADD(3, c1 - c0);
          TR_ADD(4, c2 - c1);
          TR_ADD(5, 1);
        }
        if (own) {
          store_col<RPL, T>(X0 + (size_t)warp * ldc, xr, nq, lane);
          if (!VG || vown) store_col<RPL, T>(vown, vr, nq, lane);
        }
      }
      if (r == nb - 2) break;  // sweep ends; the exchange to round 0 happens after the convergence test
      if (VG) __threadfence();  // this CTA's V writes before the blocks (and columns) change hands
      exchange();
    }
    // Converged when no pair needed a rotation, or when every rotation of the sweep was below
    // sqrt(tbig) in relative coupling.  FP64 (tbig = tol): one-sided Jacobi converges quadratically
    // at the end, so the following sweep would find every coupling ~ coupling^2 < tol and rotate
    // nothing (measured on the C2 sketch's R: 1.7e-8 -> no rotation; tests vs LAPACK).
    if (rotated && lane == 0) flags[par] = 1;
    if (big && lane == 0) flags[2 + par] = 1;
    if (VG) __threadfence();
    cl.sync();
    int any = 0, any_big = 0;
    for (int o = 0; o < CL; ++o) {
      any |= cl.map_shared_rank(flags, o)[par];
      any_big |= cl.map_shared_rank(flags, o)[2 + par];
    }
    converged = (any == 0) || (any_big == 0);
    if (tid == 0) {
      flags[par ^ 1] = 0;
      flags[2 + (par ^ 1)] = 0;
    }
    if (!converged) exchange();  // on to round 0 of the next sweep
  }
  __syncthreads();
  V0s = bufp(bf[0], 1);  // (the last exchange may have moved the blocks)
  V1s = bufp(bf[1], 1);
  if (sigma == nullptr) {  // raw V, column j = global column id
    for (int q = warp; q < 2 * h; q += NW) {
      const int gid = blk[q / h] * h + (q % h);
      if (gid >= ell) continue;
      const T* v = vcol(q / h, q % h);
      for (int r = lane; r < ell; r += 32) U[(int64_t)gid * ldu + r] = (double)v[r];
    }
    report(converged, sweep);
    return;
  }
  // norms of the held columns, ranks over the cluster, outputs
  for (int q = warp; q < 2 * h; q += NW) {
    const T* c = bufp(bf[q / h], 0) + (size_t)(q % h) * ldc;
    double sacc = 0.0;
    for (int r = lane; r < ell; r += 32) sacc = fma((double)c[r], (double)c[r], sacc);
    sacc = warp_sum(sacc);
    if (lane == 0) norms[q] = sqrt(sacc) / scale;
  }
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
      const T* v = vcol(q / h, q % h);
      if (v)
        for (int r = lane; r < ell; r += 32) U[(int64_t)rank * ldu + r] = (double)v[r];
      else
        for (int r = lane; r < ell; r += 32) U[(int64_t)rank * ldu + r] = 0.0;
    }
  }
  report(converged, sweep);
}

#undef pw
#undef pw2

static size_t jsvd_block_smem(int ell, int h, size_t elt, int nwh, int nbuf) {
  return elt * nbuf * nwh * (size_t)h * (ell + (ell & 1)) + sizeof(double) * 2 * h + 64;
}

// cluster size / block size for the block-exchange Jacobi: h <= 16 columns per block (one pair per
// warp and round), nbuf X(+V) block buffers per CTA within 200 KB -- four where they fit, else three;
// vglobal: V in global memory.  NGD_SVD_NBUF=3 forces three buffers (tuning / A-B).
static bool jsvd_block_plan(int ell, size_t elt, bool allow_vglobal, int& cl, int& h, int& vglobal, int& nbuf) {
  static const int max_nbuf = [] {
    const char* e = getenv("NGD_SVD_NBUF");
    return e && atoi(e) == 3 ? 3 : 4;
  }();
  for (int c : {2, 4, 8, 16}) {
    int hh = (ell + 2 * c - 1) / (2 * c);
    hh += hh & 1;  // even (circle method inside a block)
    if (hh > 16) continue;
    for (int nwh = 2; nwh >= (allow_vglobal ? 1 : 2); --nwh)
      for (int nb = max_nbuf; nb >= 3; --nb)
        if (jsvd_block_smem(ell, hh, elt, nwh, nb) <= 200 * 1024) {
          cl = c;
          h = hh;
          vglobal = nwh == 1;
          nbuf = nb;
          return true;
        }
  }
  return false;
}

int jsvd_block_supported(int ell) {
  int c, h, vg, nb;
  return jsvd_block_plan(ell, sizeof(double), false, c, h, vg, nb) ? c : 0;
}

// the mixed FP32 / FP64 factorisation: FP32 pre-sweeps with V in shared memory, FP64 finish with V
// in shared memory or (larger ell) in place in global memory
int jsvd_mixed_supported(int ell) {
  int c, h, vg, nb;
  if (!jsvd_block_plan(ell, sizeof(float), false, c, h, vg, nb)) return 0;
  return jsvd_block_plan(ell, sizeof(double), true, c, h, vg, nb) ? c : 0;
}

namespace {
int p2p_mode() {
  static const int m = [] {
    const char* env = getenv("NGD_SVD_P2P");  // tuning / A-B: 0 = one cluster barrier per exchange
    return env ? atoi(env) : 1;
  }();
  return m;
}
// the schedules as launch parameters, per cluster size and buffer count; built once
const JsvdPlanArg* plan_arg(int cl, int nbuf) {
  static std::mutex mu;
  static std::map<int, std::unique_ptr<JsvdPlanArg>> cache;  // 8 CL + NB
  std::lock_guard<std::mutex> lock(mu);
  auto& slot = cache[8 * cl + nbuf];
  if (!slot) {
    JsvdPlan P;
    if (!jsvd_make_plan(cl, nbuf, P) || P.w.size() > (size_t)kPlanWords) return nullptr;
    auto a = std::make_unique<JsvdPlanArg>();
    memset(a.get(), 0, sizeof(JsvdPlanArg));
    a->period = P.period;
    a->p2p = p2p_mode();
    std::copy(P.w.begin(), P.w.end(), a->w);
    std::copy(P.w2.begin(), P.w2.end(), a->w2);
    slot = std::move(a);
  }
  return slot.get();
}
}  // namespace

template <typename T, int RPL, bool VG>
static cudaError_t launch_jsvd_block_r(const double* A, int ell, int lda, const double* Vin, double* Vg, int ldv,
                                       double* U, int ldu, double* sigma, double tol, double tbig, int max_sweeps,
                                       int cl, int h, int nbuf, int* info, cudaStream_t st) {
  const size_t smem = jsvd_block_smem(ell, h, sizeof(T), VG ? 1 : 2, nbuf);
  auto kern = jsvd_block_kernel<T, RPL, VG>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (cl > 8) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  const JsvdPlanArg* pa = plan_arg(cl, nbuf);
  if (!pa) return cudaErrorInvalidValue;

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
  e = cudaLaunchKernelEx(&cfg, kern, A, ell, lda, Vin, Vg, ldv, U, ldu, sigma, tol, tbig, max_sweeps, h, info, nbuf,
                         *pa);
  probe_after(K_SVD, st);
  return e;
}

template <typename T>
static cudaError_t launch_jsvd_block(const double* A, int ell, int lda, const double* Vin, double* Vg, int ldv,
                                     double* U, int ldu, double* sigma, double tol, double tbig, int max_sweeps,
                                     int* info, bool allow_vglobal, cudaStream_t st) {
  int cl, h, vglobal, nbuf;
  if (!jsvd_block_plan(ell, sizeof(T), allow_vglobal && Vg != nullptr, cl, h, vglobal, nbuf))
    return cudaErrorInvalidValue;
  if (vglobal && ((ldv & 1) || (reinterpret_cast<uintptr_t>(Vg) & 15))) return cudaErrorInvalidValue;  // vector columns
  switch ((ell + 63) / 64) {  // vector pairs per lane
  // V in global memory: FP64 only, ell > 310 (RPL >= 5)
#define NGD_JSVD_CASE(R)                                                                                       \
  case R:                                                                                                      \
    if constexpr (sizeof(T) == 8 && R >= 5)                                                                    \
      if (vglobal)                                                                                             \
        return launch_jsvd_block_r<T, R, true>(A, ell, lda, Vin, Vg, ldv, U, ldu, sigma, tol, tbig, max_sweeps, cl, \
                                               h, nbuf, info, st);                                             \
    if (vglobal) return cudaErrorInvalidValue;                                                                 \
    return launch_jsvd_block_r<T, R, false>(A, ell, lda, Vin, Vg, ldv, U, ldu, sigma, tol, tbig, max_sweeps, cl, h, \
                                            nbuf, info, st);
    NGD_JSVD_CASE(1)
    NGD_JSVD_CASE(2)
    NGD_JSVD_CASE(3)
    NGD_JSVD_CASE(4)
    NGD_JSVD_CASE(5)
    NGD_JSVD_CASE(6)
    NGD_JSVD_CASE(7)
    NGD_JSVD_CASE(8)
#undef NGD_JSVD_CASE
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t jacobi_svd_block(const double* A, int ell, int lda, double* U, int ldu, double* sigma, int* info,
                             cudaStream_t st) {
  const double tol = 2.220446049250313e-16 * (double)ell;
  return launch_jsvd_block<double>(A, ell, lda, nullptr, nullptr, 0, U, ldu, sigma, tol, tol, 40, info, false, st);
}

cudaError_t jacobi_svd_block_from(const double* A, int ell, int lda, double* V0, int ldv, double* U, int ldu,
                                  double* sigma, int* info, cudaStream_t st) {
  // V0 is also the in-place V when the FP64 columns of X fill the cluster's shared memory alone
  // (then ldv must be even and V0 16-byte aligned; rows ell .. ldv - 1 are scratch)
  const double tol = 2.220446049250313e-16 * (double)ell;
  return launch_jsvd_block<double>(A, ell, lda, V0, V0, ldv, U, ldu, sigma, tol, tol, 40, info, true, st);
}

cudaError_t jacobi_presweep_f32(const double* A, int ell, int lda, double* V, int ldv, double coupling, int* info,
                                cudaStream_t st) {
  // rotate above coupling^2 (near FP32 rounding), stop once no rotation of a sweep reached 'coupling'
  return launch_jsvd_block<float>(A, ell, lda, nullptr, nullptr, 0, V, ldv, nullptr, coupling * coupling,
                                  coupling * coupling, 30, info, false, st);
}

}  // namespace ngd
