// Probe: tcgen05 kind::i8 GEMM (both operands K-major, 128-byte swizzle, TMA ring, TMEM
// double-buffered accumulators) -- correctness vs a host int reference and throughput on B200.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lcuda tools/probe/i8gemm.cu -o /tmp/i8gemm
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CKR(x)                                                                       \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);      \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

constexpr int BM = 128, BN = 256, BK = 128, NS = 4;
constexpr int kThreads = 192;
struct __align__(1024) Stage {
  int8_t A[BM * BK];
  int8_t B[BN * BK];
};
constexpr size_t kSmem = sizeof(Stage) * NS + 1024 + 256;

struct Args {
  int M, N, K, nb;       // batch nb of (M x K) . (N x K)^T
  int tiles_m, tiles_n;  // per batch
  int kblocks;
  int32_t* C;  // [nb][M][N] (mode 0)
  int mode;
  unsigned long long* sink;
};

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* m, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(m)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(unsigned long long* m, unsigned par) {
  unsigned done = 0;
  while (!done)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}\n"
                 : "=r"(done)
                 : "r"(sa(m)), "r"(par)
                 : "memory");
}
__device__ __forceinline__ void expect_tx(unsigned long long* m, unsigned b) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(m)), "r"(b) : "memory");
}
__device__ __forceinline__ void arrive(unsigned long long* m) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(m)) : "memory");
}
__device__ __forceinline__ void tma3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, unsigned long long* m) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          sa(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(sa(m))
      : "memory");
}
__device__ __forceinline__ uint64_t sw128_desc(unsigned saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;            // LBO (ignored for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;  // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;            // descriptor version (sm100)
  d |= (uint64_t)2 << 61;            // SWIZZLE_128B
  return d;
}
__device__ __forceinline__ void mma_i8(unsigned tmem, uint64_t ad, uint64_t bd, unsigned idesc, unsigned acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit(unsigned long long* m) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(m)) : "memory");
}

__global__ void __launch_bounds__(kThreads, 1)
    i8gemm(const __grid_constant__ Args a, const __grid_constant__ CUtensorMap mapA,
           const __grid_constant__ CUtensorMap mapB) {
  extern __shared__ unsigned char raw[];
  unsigned char* base = raw + ((1024u - (sa(raw) & 1023u)) & 1023u);
  Stage* st = reinterpret_cast<Stage*>(base);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(st + NS);
  unsigned long long* empty = full + NS;
  unsigned long long* tfull = empty + NS;
  unsigned long long* tempty = tfull + 2;
  unsigned* tmem_slot = reinterpret_cast<unsigned*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
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
  const int n_items = per * a.nb;
  if (warp == 0) {
    if (lane == 0) {
      unsigned q = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int b = it / per, r = it % per;
        const int m0 = (r / a.tiles_n) * BM, n0 = (r % a.tiles_n) * BN;
        for (int kb = 0; kb < a.kblocks; ++kb, ++q) {
          const int s = q % NS;
          if (q >= NS) mbar_wait(&empty[s], ((q / NS) - 1) & 1);
          expect_tx(&full[s], sizeof(Stage));
          tma3d(st[s].A, &mapA, kb * BK, m0, b, &full[s]);
          tma3d(st[s].B, &mapB, kb * BK, n0, b, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const unsigned idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((unsigned)(BN >> 3) << 17) | ((unsigned)(BM >> 4) << 24);
      unsigned q = 0, u = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++u) {
        const int buf = u & 1;
        if (u >= 2) mbar_wait(&tempty[buf], ((u >> 1) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const unsigned d = tmem + buf * BN;
        for (int kb = 0; kb < a.kblocks; ++kb, ++q) {
          const int s = q % NS;
          mbar_wait(&full[s], (q / NS) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t ad = sw128_desc(sa(st[s].A)), bd = sw128_desc(sa(st[s].B));
#pragma unroll
          for (int k = 0; k < BK / 32; ++k) mma_i8(d, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
          commit(&empty[s]);
        }
        commit(&tfull[buf]);
      }
    }
  } else {
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    unsigned long long chk = 0;
    unsigned u = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++u) {
      const int buf = u & 1;
      const int b = it / per, r = it % per;
      const int m0 = (r / a.tiles_n) * BM, n0 = (r % a.tiles_n) * BN;
      mbar_wait(&tfull[buf], (u >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        unsigned v[32];
        const unsigned taddr = tmem + ((unsigned)(quarter * 32) << 16) + buf * BN + c;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%"
            "20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
              "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
              "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
              "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (a.mode == 0) {
          const int m = m0 + row;
          if (m < a.M)
            for (int j = 0; j < 32; ++j)
              if (n0 + c + j < a.N) a.C[((size_t)b * a.M + m) * a.N + n0 + c + j] = (int32_t)v[j];
        } else {
          for (int j = 0; j < 32; ++j) chk += v[j];
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) arrive(&tempty[buf]);
    }
    if (a.mode != 0 && chk == 0x123456789ull) a.sink[0] = chk;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  CKR(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
}
static CUtensorMap make_map(const int8_t* p, int K, int rows, int nb, int ldk, int box_rows) {
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)rows, (cuuint64_t)nb};
  cuuint64_t strides[2] = {(cuuint64_t)ldk, (cuuint64_t)ldk * rows};
  cuuint32_t box[3] = {BK, (cuuint32_t)box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)p, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("encode failed %d\n", (int)r);
    exit(1);
  }
  return m;
}

static void run(int M, int N, int K, int nb, bool check, int reps) {
  const int ldk = (K + 15) / 16 * 16;
  std::vector<int8_t> hA((size_t)nb * M * ldk, 0), hB((size_t)nb * N * ldk, 0);
  uint32_t s = 12345;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return (int8_t)((s >> 24) & 0xff); };
  for (int b = 0; b < nb; ++b)
    for (int i = 0; i < M; ++i)
      for (int k = 0; k < K; ++k) hA[((size_t)b * M + i) * ldk + k] = rnd();
  for (int b = 0; b < nb; ++b)
    for (int i = 0; i < N; ++i)
      for (int k = 0; k < K; ++k) hB[((size_t)b * N + i) * ldk + k] = rnd();
  int8_t *dA, *dB;
  int32_t* dC;
  unsigned long long* sink;
  CKR(cudaMalloc(&dA, hA.size()));
  CKR(cudaMalloc(&dB, hB.size()));
  CKR(cudaMalloc(&dC, sizeof(int32_t) * (size_t)nb * M * N));
  CKR(cudaMalloc(&sink, 8));
  CKR(cudaMemcpy(dA, hA.data(), hA.size(), cudaMemcpyHostToDevice));
  CKR(cudaMemcpy(dB, hB.data(), hB.size(), cudaMemcpyHostToDevice));
  CUtensorMap mA = make_map(dA, K, M, nb, ldk, BM), mB = make_map(dB, K, N, nb, ldk, BN);
  Args a;
  a.M = M;
  a.N = N;
  a.K = K;
  a.nb = nb;
  a.tiles_m = (M + BM - 1) / BM;
  a.tiles_n = (N + BN - 1) / BN;
  a.kblocks = (K + BK - 1) / BK;
  a.C = dC;
  a.mode = check ? 0 : 1;
  a.sink = sink;
  CKR(cudaFuncSetAttribute(i8gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem));
  const int items = a.tiles_m * a.tiles_n * nb;
  const int grid = items < 148 ? items : 148;
  i8gemm<<<grid, kThreads, kSmem>>>(a, mA, mB);
  CKR(cudaGetLastError());
  CKR(cudaDeviceSynchronize());
  if (check) {
    std::vector<int32_t> hC((size_t)nb * M * N);
    CKR(cudaMemcpy(hC.data(), dC, hC.size() * 4, cudaMemcpyDeviceToHost));
    long bad = 0;
    for (int b = 0; b < nb; ++b)
      for (int i = 0; i < M; ++i)
        for (int j = 0; j < N; ++j) {
          int64_t ref = 0;
          for (int k = 0; k < K; ++k)
            ref += (int)hA[((size_t)b * M + i) * ldk + k] * (int)hB[((size_t)b * N + j) * ldk + k];
          if ((int32_t)ref != hC[((size_t)b * M + i) * N + j]) {
            if (bad < 5) printf("  mismatch b%d (%d,%d): got %d want %lld\n", b, i, j, hC[((size_t)b * M + i) * N + j], (long long)ref);
            ++bad;
          }
        }
    printf("check M=%d N=%d K=%d nb=%d: %s (%ld bad)\n", M, N, K, nb, bad ? "FAIL" : "ok", bad);
  } else {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) i8gemm<<<grid, kThreads, kSmem>>>(a, mA, mB);
    cudaEventRecord(e1);
    CKR(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    const double ops = 2.0 * M * N * (double)K * nb;
    printf("perf M=%d N=%d K=%d nb=%d: %.3f ms  %.1f TOPS\n", M, N, K, nb, ms, ops / ms / 1e9);
  }
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dC);
  cudaFree(sink);
}

int main() {
  run(128, 256, 128, 1, true, 0);
  run(128, 256, 512, 1, true, 0);
  run(300, 520, 1000, 2, true, 0);
  run(600, 520, 4100, 2, true, 0);
  run(5344, 1024, 65536, 1, false, 5);
  run(5344, 1024, 131072, 2, false, 3);
  run(8192, 8192, 8192, 1, false, 5);
  run(16384, 1024, 16384, 4, false, 5);
  return 0;
}
