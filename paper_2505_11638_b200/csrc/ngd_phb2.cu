// Phase B of the factored Gramian matvec, pipelined form (phb_plan = 2, default):
//     out_k = D_k diag(c) Zin_k^T  (+ bias column sum over value columns)   per layer k
// (the J^T c half of gramian.py:48-53; see ngd_jet.cu for the layout and the first form).
//
// Why a second form: measured on B200 (tools/probe/dmma_lat.cu) FP64 DMMA.8x8x4 issues one per
// 16 cycles per SM sub-partition (64 FMA/clk/SM, 26-cycle latency), so a 64 x 64 tile streams
// 16 KB per 256 DMMAs and one CTA per SM can keep the tensor pipe busy -- if the operand stream
// never stalls the math warps.  The first form (8 warps doing both cp.async issue and MMA, one
// __syncthreads per 16-column stage) ran the pipe at ~35% and split the work so unevenly over
// SMs (thin input/output layers padded to full tiles) that C2's phase B took 35 us for 10 us of
// DMMA work.  Here:
//   * one producer thread streams each 16-column k-unit into a 4-deep ring with TMA: a 64 x 16
//     box of D and one of Zin (cp.async.bulk.tensor.2d, 128-byte swizzle, rows past the layer
//     zero-filled) plus the 16 cotangents (1-D bulk copy), completion on a "full" mbarrier;
//     eight consumer warps wait on "full", compute, and release the slot on an "empty"
//     mbarrier -- no CTA-wide barrier in the main loop.  (Per-row 128-byte bulk copies were
//     measured issue-bound: one UBLKCP per lane through the uniform datapath, ~2 us per unit);
//   * consumer warps form 2 (rows) x 2 (cols) x 2 (k-groups) with 32 x 32 warp tiles (16
//     independent accumulator chains, 8 fragment loads per 16 DMMAs); the two k-groups are
//     summed in shared memory at the end (fixed order: deterministic);
//   * 8x8 blocks wholly outside the layer (input layer N = d, output layer M = 1) are skipped,
//     so a thin tile costs its operand stream, not a full tile of MMAs;
//   * one CTA per SM: CTA i owns heavy work item i (a K split of a 64 x 64 tile of a layer with
//     both sides > 16) AND thin item i (a K split of the input layer's 64 x d or the output
//     layer's 1 x 64 tile); the producer interleaves the two unit streams evenly, so the thin
//     tiles' operand stream hides under the heavy tiles' MMAs (two CTAs per SM were measured
//     to run in two waves: the second CTA of many SMs started only after the first ended).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "ngd_common.cuh"
#include "ngd_kernels.h"

namespace ngd {

#ifdef NGD_PHB2_TRACE
__device__ unsigned long long g_p2tr[1024][4];  // per CTA: consumer-0 wait, compute, total; producer empty-wait
#define P2_T(v) long long v = clock64()
#define P2_ADD(k, d) p2acc[k] += (d)
#else
#define P2_T(v)
#define P2_ADD(k, d)
#endif

namespace {
constexpr int HB = 64;                 // tile rows / cols
constexpr int HK = 16;                 // k-unit: one channel run of one point block (128 B per row)
constexpr int HNS = 6;                 // heavy ring depth
constexpr int TNS = 4;                 // thin ring depth
constexpr int kConsumerWarps = 8;      // heavy consumers: 2 (rows) x 2 (cols) x 2 (k-groups)
constexpr int kThinWarps = 4;          // thin consumers: 2 x 2, all four k-steps each
// warps: [0, 8) heavy consumers, 8 heavy producer, [9, 13) thin consumers, 13 thin producer
constexpr int kHeavyProducer = kConsumerWarps, kThin0 = kConsumerWarps + 1, kThinProducer = kThin0 + kThinWarps;
constexpr int kPhb2Threads = (kThinProducer + 1) * 32;
// one ring slot: TMA boxes (row r of 128 B at r * 128, its 16-byte chunks XOR-swizzled by r & 7)
struct __align__(1024) HStage {
  double A[HB * HK];
  double B[HB * HK];
  double cc[HK];
  double pad[128 - HK];
};
constexpr size_t kPhb2Smem = sizeof(HStage) * (HNS + TNS) + 2 * (HNS + TNS) * sizeof(unsigned long long) + 1024;
static_assert(HB * (HB + 1) + 2 * HB <= HNS * (2 * HB * HK), "epilogue staging must fit");

__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* m, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(m)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* m, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* m) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(m)) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(unsigned long long* m, unsigned parity) {
  const unsigned a = smem_addr(m);
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* map, int c0, int c1, unsigned long long* m) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_addr(m))
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* m) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(m))
               : "memory");
}

// first point of k-unit u (interior blocks: C channel runs of PB points each; then one boundary
// point per column) -- 32-bit unit arithmetic, the producer's only per-unit integer work
__device__ __forceinline__ int unit_point(int u, int int_units, int C, int nib) {
  return u < int_units ? (u / C) * PB : nib * PB + (u - int_units) * HK;
}


// one K-split of one tile: layer, tile coordinates, unit range, split index
struct Item {
  int l, bx, by, k0, k1, split;
};

// item `idx` of the heavy (thin = 0) or thin (thin = 1) list: layers in order, tiles x G_l each
__device__ __forceinline__ bool decode_item(const PhbAll& a, int thin, int idx, Item& it) {
  for (int l = 0; l < a.n_layers; ++l) {
    if (a.thin[l] != thin) continue;
    const int nt = a.tiles_n[l] * a.tiles_m[l] * a.G[l];
    if (idx < nt) {
      const int G = a.G[l];
      const int split = idx % G, tile = idx / G;
      const PhbArgs& p = a.L[l];
      it.l = l;
      it.bx = tile % a.tiles_n[l];
      it.by = tile / a.tiles_n[l];
      it.split = split;
      it.k0 = min(p.ktiles_total, split * p.ktiles_per_split);
      it.k1 = min(p.ktiles_total, it.k0 + p.ktiles_per_split);
      return true;
    }
    idx -= nt;
  }
  return false;
}

// real 8 x 8 blocks of a warp's 32 x 32 sub-tile (rows wm*32.., cols wn*32..)
__device__ __forceinline__ int blocks_of(int extent, int w) { return max(0, min(4, (extent - w * 32 + 7) / 8)); }

// one unit (16 columns) for a warp with QA x RA real blocks; acc[q*RA + r]
template <int QA, int RA, int NACC, int KS = 2>
__device__ __forceinline__ void mma_unit(const HStage& S, int arow, int brow, int kg, int g, int t, bool val,
                                         double (&acc)[NACC][2], double (&bs)[4]) {
#pragma unroll
  for (int h = 0; h < KS; ++h) {
    const int kk = KS == 2 ? kg * 4 + h * 8 : h * 4;
    const int sw = ((((kk + t) >> 1) ^ g) << 1) + (t & 1);  // 128-byte swizzle of column kk + t
    const double cc = S.cc[kk + t];
    double a[QA], b[RA];
#pragma unroll
    for (int q = 0; q < QA; ++q) a[q] = S.A[arow + q * 8 * HK + sw] * cc;
#pragma unroll
    for (int r = 0; r < RA; ++r) b[r] = S.B[brow + r * 8 * HK + sw];
#pragma unroll
    for (int q = 0; q < QA; ++q)
#pragma unroll
      for (int r = 0; r < RA; ++r) dmma884(acc[q * RA + r][0], acc[q * RA + r][1], a[q], b[r]);
    if (val) {
#pragma unroll
      for (int q = 0; q < QA; ++q) bs[q] += a[q];
    }
  }
}

// write a tile's partial.  Heavy (KGROUPS = 2): k-group 1 -> staging, k-group 0 adds (fixed order),
// named barrier 1 over the 8 heavy consumer warps.  Thin (KGROUPS = 1): each warp holds its whole
// sum; named barrier 2 over the 4 thin consumer warps (bias rows staged).
template <int QA, int RA, int NACC, int KGROUPS>
__device__ __forceinline__ void epilogue(const PhbArgs& p, const Item& it, double (&acc)[NACC][2],
                                         double (&bs)[4], bool do_bias, double* red, double* redb, int kg, int wm,
                                         int wn, int g, int t, int ltid) {
  constexpr int RS = HB + 1;
  constexpr int NT = KGROUPS == 2 ? kConsumerWarps * 32 : kThinWarps * 32;
  constexpr int BAR = KGROUPS == 2 ? 1 : 2;
  const int m0 = it.by * HB, n0 = it.bx * HB;
  const int mrows = min(HB, p.M - m0), nrows = min(HB, p.N - n0);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    bs[q] += __shfl_xor_sync(0xffffffffu, bs[q], 1);
    bs[q] += __shfl_xor_sync(0xffffffffu, bs[q], 2);
  }
  if (KGROUPS == 2 && kg == 1) {
#pragma unroll
    for (int q = 0; q < QA; ++q)
#pragma unroll
      for (int r = 0; r < RA; ++r)
#pragma unroll
        for (int e = 0; e < 2; ++e) red[(wm * 32 + q * 8 + g) * RS + wn * 32 + r * 8 + 2 * t + e] = acc[q * RA + r][e];
  }
  if (do_bias && t == 0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) redb[kg * HB + wm * 32 + q * 8 + g] = bs[q];
  }
  asm volatile("bar.sync %0, %1;" ::"n"(BAR), "n"(NT));
  double* out = p.part + (int64_t)it.split * p.p + p.off;
  if (kg == 0) {
#pragma unroll
    for (int q = 0; q < QA; ++q)
#pragma unroll
      for (int r = 0; r < RA; ++r)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int row = wm * 32 + q * 8 + g, col = wn * 32 + r * 8 + 2 * t + e;
          if (row < mrows && col < nrows)
            out[(int64_t)(m0 + row) * p.N + n0 + col] =
                KGROUPS == 2 ? acc[q * RA + r][e] + red[row * RS + col] : acc[q * RA + r][e];
        }
  }
  if (it.bx == 0 && ltid < mrows)
    out[(int64_t)p.M * p.N + m0 + ltid] = KGROUPS == 2 ? redb[ltid] + redb[HB + ltid] : redb[ltid];
}
}  // namespace

namespace {
// one thread streams an item's units through an NS-deep ring (TMA boxes + cotangent run)
template <int NS>
__device__ __forceinline__ void produce(const PhbAll& a, const Phb2Maps& maps, const Item& it, HStage* st,
                                        unsigned long long* full, unsigned long long* empty) {
  constexpr unsigned bytes = (2 * HB * HK + HK) * sizeof(double);  // full boxes (OOB rows zero-filled)
  const PhbArgs& p = a.L[it.l];
  const int iu = (int)(p.int_cols / HK);
  for (int i = 0; i < it.k1 - it.k0; ++i) {
    const int s = i % NS;
    if (i >= NS) mbar_wait_parity(&empty[s], (unsigned)((i / NS) - 1) & 1u);
    const int u = it.k0 + i;
    mbar_expect_tx(&full[s], bytes);
    tma2d(st[s].A, &maps.d[it.l], u * HK, it.by * HB, &full[s]);
    tma2d(st[s].B, &maps.z[it.l], u * HK, it.bx * HB, &full[s]);
    bulk_g2s(st[s].cc, p.cvec + unit_point(u, iu, p.C, p.nib), HK * sizeof(double), &full[s]);
  }
}

// consumer loop of one pipeline: QA x RA real blocks per warp, KS k-steps per warp and unit
template <int QA, int RA, int NACC, int KS, int NS>
__device__ __forceinline__ void consume(const PhbArgs& p, const Item& it, const HStage* st, unsigned long long* full,
                                        unsigned long long* empty, bool do_bias, int arow, int brow, int kg, int g,
                                        int t, int lane, double (&acc)[NACC][2], double (&bs)[4]) {
  const int iu = (int)(p.int_cols / HK);
  int ch = it.k0 % max(1, p.C);  // channel of the first unit (interior units cycle through C runs)
  for (int i = 0; i < it.k1 - it.k0; ++i) {
    const int s = i % NS;
    mbar_wait_parity(&full[s], (unsigned)(i / NS) & 1u);
    const bool val = do_bias && (it.k0 + i >= iu || ch == 0);
    ch = (ch + 1 == p.C) ? 0 : ch + 1;
    if (QA > 0 && RA > 0) mma_unit<(QA > 0 ? QA : 1), (RA > 0 ? RA : 1), NACC, KS>(st[s], arow, brow, kg, g, t, val, acc, bs);
    // the producer warp refills the slot as soon as the last consumer has arrived: order this warp's
    // shared-memory reads (generic proxy) before that TMA write (async proxy) -- see ngd_phag.cu
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
}
}  // namespace

// CTA i owns heavy item i and thin item i (either may be absent) and runs them as two independent
// warp-specialised pipelines side by side: the thin tiles' operand stream and MMAs overlap the
// heavy tiles' MMAs on the same SM.
__global__ void __maxnreg__(144) phb2_kernel(const __grid_constant__ PhbAll a,
                                              const __grid_constant__ Phb2Maps maps) {
  pdl_entry();  // (PCG chain: programmatic dependent launch)
  extern __shared__ unsigned char phb2_smem[];
  // 1024-byte aligned rings (128-byte swizzle atoms); offsetting the extern array keeps the
  // accesses in the shared window (LDS) -- an integer round trip through uintptr_t made them generic
  unsigned char* base = phb2_smem + ((1024u - (smem_addr(phb2_smem) & 1023u)) & 1023u);
  HStage* sth = reinterpret_cast<HStage*>(base);
  HStage* stt = sth + HNS;
  unsigned long long* fullh = reinterpret_cast<unsigned long long*>(stt + TNS);
  unsigned long long* emptyh = fullh + HNS;
  unsigned long long* fullt = emptyh + HNS;
  unsigned long long* emptyt = fullt + TNS;
  double* redh = reinterpret_cast<double*>(emptyt + TNS);  // heavy epilogue staging [HB][HB+1] + [2][HB]
  double* redt = redh + HB * (HB + 1) + 2 * HB;          // thin bias staging [HB]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  Item H{}, T{};
  const bool hasH = decode_item(a, 0, blockIdx.x, H);
  const bool hasT = decode_item(a, 1, blockIdx.x, T);
  if (a.L[0].skip && *a.L[0].skip) return;
  if (tid == 0) {
    for (int s = 0; s < HNS; ++s) {
      mbar_init(&fullh[s], 1);
      mbar_init(&emptyh[s], kConsumerWarps);
    }
    for (int s = 0; s < TNS; ++s) {
      mbar_init(&fullt[s], 1);
      mbar_init(&emptyt[s], kThinWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int g = lane >> 2, t = lane & 3;
  if (warp == kHeavyProducer) {
    if (hasH && lane == 0) produce<HNS>(a, maps, H, sth, fullh, emptyh);
    return;
  }
  if (warp == kThinProducer) {
    if (hasT && lane == 0) produce<TNS>(a, maps, T, stt, fullt, emptyt);
    return;
  }
  if (warp < kConsumerWarps) {  // heavy consumers: 2 x 2 x 2 (k-groups)
    if (!hasH) return;
    const PhbArgs& p = a.L[H.l];
    const int kg = warp >> 2, wm = (warp >> 1) & 1, wn = warp & 1;
    const bool do_bias = H.bx == 0 && wn == 0;
    double acc[16][2], bs[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i][0] = acc[i][1] = 0.0;
    consume<4, 4, 16, 2, HNS>(p, H, sth, fullh, emptyh, do_bias, (wm * 32 + g) * HK, (wn * 32 + g) * HK, kg, g, t,
                              lane, acc, bs);
    epilogue<4, 4, 16, 2>(p, H, acc, bs, do_bias, redh, redh + HB * (HB + 1), kg, wm, wn, g, t, tid);
    return;
  }
  // thin consumers: 2 x 2 warps over the 64 x 64 box, all k-steps; dispatch on the real blocks
  if (!hasT) return;
  const PhbArgs& p = a.L[T.l];
  const int w = warp - kThin0, wm = w >> 1, wn = w & 1;
  const bool do_bias = T.bx == 0 && wn == 0;
  const int qa = blocks_of(p.M - T.by * HB, wm), ra = blocks_of(p.N - T.bx * HB, wn);
  double acc[8][2], bs[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
  const int arow = (wm * 32 + g) * HK, brow = (wn * 32 + g) * HK, ltid = tid - kThin0 * 32;
#define NGD_THIN(QA, RA)                                                                                    \
  do {                                                                                                     \
    consume<QA, RA, 8, 4, TNS>(p, T, stt, fullt, emptyt, do_bias, arow, brow, 0, g, t, lane, acc, bs);    \
    epilogue<(QA > 0 ? QA : 1), (RA > 0 ? RA : 1), 8, 1>(p, T, acc, bs, do_bias, nullptr, redt, 0, wm, wn, g, t, \
                                                         ltid);                                            \
  } while (0)
  switch (qa * 8 + ra) {
    case 4 * 8 + 1: NGD_THIN(4, 1); break;
    case 4 * 8 + 2: NGD_THIN(4, 2); break;
    case 3 * 8 + 1: NGD_THIN(3, 1); break;
    case 3 * 8 + 2: NGD_THIN(3, 2); break;
    case 2 * 8 + 1: NGD_THIN(2, 1); break;
    case 2 * 8 + 2: NGD_THIN(2, 2); break;
    case 1 * 8 + 1: NGD_THIN(1, 1); break;
    case 1 * 8 + 2: NGD_THIN(1, 2); break;
    case 1 * 8 + 3: NGD_THIN(1, 3); break;
    case 1 * 8 + 4: NGD_THIN(1, 4); break;
    case 2 * 8 + 3: NGD_THIN(2, 3); break;
    case 2 * 8 + 4: NGD_THIN(2, 4); break;
    default: NGD_THIN(0, 0); break;  // no real block: ring protocol and bias staging only
  }
#undef NGD_THIN
}

// Thin-only form (no heavy tile in this launch -- every layer with both sides >= 256 runs on the GEMM
// core, C4 / C5): five warps (four consumers + the producer) and a TO_NS-deep ring, small enough for
// three CTAs per SM, so the memory-bound thin tiles (the input layer's D_1 and the output layer's
// Zin_L, 2 x 3.3 GB per C5 matvec) stream with three times the bytes in flight of the paired form.
constexpr int TO_NS = 4;
constexpr int kThinOnlyThreads = (kThinWarps + 1) * 32;
constexpr size_t kThinOnlySmem = sizeof(HStage) * TO_NS + 2 * TO_NS * sizeof(unsigned long long) +
                                 sizeof(double) * HB + 1024;
__global__ void __launch_bounds__(kThinOnlyThreads) phb2_thin_kernel(const __grid_constant__ PhbAll a,
                                                                     const __grid_constant__ Phb2Maps maps) {
  pdl_entry();  // (PCG chain: programmatic dependent launch)
  extern __shared__ unsigned char phb2_smem[];
  unsigned char* base = phb2_smem + ((1024u - (smem_addr(phb2_smem) & 1023u)) & 1023u);
  HStage* stt = reinterpret_cast<HStage*>(base);
  unsigned long long* fullt = reinterpret_cast<unsigned long long*>(stt + TO_NS);
  unsigned long long* emptyt = fullt + TO_NS;
  double* redt = reinterpret_cast<double*>(emptyt + TO_NS);  // thin bias staging [HB]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  Item T{};
  const bool hasT = decode_item(a, 1, blockIdx.x, T);
  if (a.L[0].skip && *a.L[0].skip) return;
  if (tid == 0) {
    for (int s = 0; s < TO_NS; ++s) {
      mbar_init(&fullt[s], 1);
      mbar_init(&emptyt[s], kThinWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (!hasT) return;
  const int g = lane >> 2, t = lane & 3;
  if (warp == kThinWarps) {
    if (lane == 0) produce<TO_NS>(a, maps, T, stt, fullt, emptyt);
    return;
  }
  const PhbArgs& p = a.L[T.l];
  const int wm = warp >> 1, wn = warp & 1;
  const bool do_bias = T.bx == 0 && wn == 0;
  const int qa = blocks_of(p.M - T.by * HB, wm), ra = blocks_of(p.N - T.bx * HB, wn);
  double acc[8][2], bs[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
  const int arow = (wm * 32 + g) * HK, brow = (wn * 32 + g) * HK;
#define NGD_THIN(QA, RA)                                                                                     \
  do {                                                                                                      \
    consume<QA, RA, 8, 4, TO_NS>(p, T, stt, fullt, emptyt, do_bias, arow, brow, 0, g, t, lane, acc, bs);   \
    epilogue<(QA > 0 ? QA : 1), (RA > 0 ? RA : 1), 8, 1>(p, T, acc, bs, do_bias, nullptr, redt, 0, wm, wn, g, t, \
                                                         tid);                                              \
  } while (0)
  switch (qa * 8 + ra) {
    case 4 * 8 + 1: NGD_THIN(4, 1); break;
    case 4 * 8 + 2: NGD_THIN(4, 2); break;
    case 3 * 8 + 1: NGD_THIN(3, 1); break;
    case 3 * 8 + 2: NGD_THIN(3, 2); break;
    case 2 * 8 + 1: NGD_THIN(2, 1); break;
    case 2 * 8 + 2: NGD_THIN(2, 2); break;
    case 1 * 8 + 1: NGD_THIN(1, 1); break;
    case 1 * 8 + 2: NGD_THIN(1, 2); break;
    case 1 * 8 + 3: NGD_THIN(1, 3); break;
    case 1 * 8 + 4: NGD_THIN(1, 4); break;
    case 2 * 8 + 3: NGD_THIN(2, 3); break;
    case 2 * 8 + 4: NGD_THIN(2, 4); break;
    default: NGD_THIN(0, 0); break;  // no real block: ring protocol and bias staging only
  }
#undef NGD_THIN
}

namespace {
constexpr size_t kStaging = sizeof(double) * (HB * (HB + 1) + 4 * HB);
}
int phb2_ctas_per_sm() { return 1; }
// thin items of a thin-only launch (every wide layer on the GEMM core): three CTAs per SM
int phb2_thin_only_ctas() { return 3 * 148; }

namespace {
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
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
bool encode_rows(CUtensorMap* m, const double* base, int rows, int64_t s_pad) {
  auto enc = get_encode();
  if (!enc) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)s_pad, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)s_pad * sizeof(double)};
  const cuuint32_t box[2] = {(cuuint32_t)HK, (cuuint32_t)HB};
  const cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace

cudaError_t phase_b2_all_layers(const PhbAll& a, Phb2Cache& cache, cudaStream_t st) {
  const size_t smem = kPhb2Smem + kStaging;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(phb2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  int nh = 0, nt = 0;
  // thin[l] == 2: the layer runs on the GEMM core (ngd_phbg.cu); 3: output layer from its precontracted
  // rows (out_phase_b, ngd_vec.cu)
  for (int l = 0; l < a.n_layers; ++l) {
    if (a.thin[l] == 0) nh += a.tiles_n[l] * a.tiles_m[l] * a.G[l];
    if (a.thin[l] == 1) nt += a.tiles_n[l] * a.tiles_m[l] * a.G[l];
  }
  const int ctas = std::max(nh, nt);
  if (ctas <= 0) return cudaSuccess;
  const bool thin_only = nh == 0;
  static bool attr_thin = false;
  if (thin_only && !attr_thin) {
    cudaError_t e = cudaFuncSetAttribute(phb2_thin_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kThinOnlySmem);
    if (e != cudaSuccess) return e;
    attr_thin = true;
  }
  // tensor maps of every layer's operands (host-side encode, cached in the context while the
  // buffers stay put)
  for (int l = 0; l < a.n_layers; ++l) {
    const PhbArgs& p = a.L[l];
    if (a.thin[l] >= 2) continue;
    if (cache.kd[l] != p.D || cache.kz[l] != p.Z || cache.km[l] != p.M || cache.kn[l] != p.N ||
        cache.ks[l] != p.s_pad) {
      if (!encode_rows(&cache.maps.d[l], p.D, p.M, p.s_pad) || !encode_rows(&cache.maps.z[l], p.Z, p.N, p.s_pad))
        return cudaErrorInvalidValue;
      cache.kd[l] = p.D;
      cache.kz[l] = p.Z;
      cache.km[l] = p.M;
      cache.kn[l] = p.N;
      cache.ks[l] = p.s_pad;
    }
  }
  probe_before(K_PHB, st);
  const cudaError_t e = thin_only ? launch_pdl(phb2_thin_kernel, dim3(ctas), dim3(kThinOnlyThreads), kThinOnlySmem,
                                               st, a, cache.maps)
                                  : launch_pdl(phb2_kernel, dim3(ctas), dim3(kPhb2Threads), smem, st, a, cache.maps);
  probe_after(K_PHB, st);
  return e;
}

}  // namespace ngd
