// cuBLAS DGEMM vs the cuBLASLt heuristic candidates for the two sketch GEMMs of C2
// (S = Jt^T V: M=4608 N=300 K=8577 TN; Y = Jt S: M=8577 N=300 K=4608 NN).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probe/lt_gemm.cu -lcublasLt -lcublas -o tools/probe/lt_gemm.bin
#include <cstdio>
#include <vector>
#include <cublasLt.h>
#include <cublas_v2.h>
#include <cuda_runtime.h>
static float time_it(cudaStream_t st, int reps, auto&& fn) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  fn(); cudaStreamSynchronize(st);
  cudaEventRecord(a, st);
  for (int i = 0; i < reps; ++i) fn();
  cudaEventRecord(b, st); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}
int main() {
  const int p = 8577, r = 4608, l = 300;
  double *jt, *V, *S, *Y;
  cudaMalloc(&jt, sizeof(double) * (size_t)p * r); cudaMalloc(&V, sizeof(double) * (size_t)p * l);
  cudaMalloc(&S, sizeof(double) * (size_t)r * l); cudaMalloc(&Y, sizeof(double) * (size_t)p * l);
  cudaMemset(jt, 0, sizeof(double) * (size_t)p * r); cudaMemset(V, 0, sizeof(double) * (size_t)p * l);
  cudaMemset(S, 0, sizeof(double) * (size_t)r * l);
  cudaStream_t st; cudaStreamCreate(&st);
  cublasHandle_t h; cublasCreate(&h); cublasSetStream(h, st);
  cublasLtHandle_t lt; cublasLtCreate(&lt);
  size_t wsz = 64 << 20; void* ws; cudaMalloc(&ws, wsz);
  const double one = 1.0, zero = 0.0;
  struct Shape { const char* name; cublasOperation_t ta, tb; int M, N, K; const double* A; int lda; const double* B; int ldb; double* C; int ldc; };
  Shape shapes[2] = {{"S = Jt^T V (TN)", CUBLAS_OP_T, CUBLAS_OP_N, r, l, p, jt, p, V, p, S, r},
                     {"Y = Jt S (NN)", CUBLAS_OP_N, CUBLAS_OP_N, p, l, r, jt, p, S, r, Y, p}};
  for (auto& sh : shapes) {
    const double flop = 2.0 * sh.M * sh.N * (double)sh.K;
    float t0 = time_it(st, 10, [&] { cublasDgemm(h, sh.ta, sh.tb, sh.M, sh.N, sh.K, &one, sh.A, sh.lda, sh.B, sh.ldb, &zero, sh.C, sh.ldc); });
    printf("%s: cublasDgemm %.1f us (%.1f TF/s)\n", sh.name, 1e3 * t0, flop / t0 / 1e9);
    cublasLtMatmulDesc_t desc; cublasLtMatmulDescCreate(&desc, CUBLAS_COMPUTE_64F, CUDA_R_64F);
    cublasLtMatmulDescSetAttribute(desc, CUBLASLT_MATMUL_DESC_TRANSA, &sh.ta, sizeof(sh.ta));
    cublasLtMatmulDescSetAttribute(desc, CUBLASLT_MATMUL_DESC_TRANSB, &sh.tb, sizeof(sh.tb));
    cublasLtMatrixLayout_t la, lb, lc;
    const int ar = sh.ta == CUBLAS_OP_N ? sh.M : sh.K, ac = sh.ta == CUBLAS_OP_N ? sh.K : sh.M;
    const int br = sh.tb == CUBLAS_OP_N ? sh.K : sh.N, bc = sh.tb == CUBLAS_OP_N ? sh.N : sh.K;
    cublasLtMatrixLayoutCreate(&la, CUDA_R_64F, ar, ac, sh.lda);
    cublasLtMatrixLayoutCreate(&lb, CUDA_R_64F, br, bc, sh.ldb);
    cublasLtMatrixLayoutCreate(&lc, CUDA_R_64F, sh.M, sh.N, sh.ldc);
    cublasLtMatmulPreference_t pref; cublasLtMatmulPreferenceCreate(&pref);
    cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wsz, sizeof(wsz));
    cublasLtMatmulHeuristicResult_t res[32]; int n = 0;
    cublasLtMatmulAlgoGetHeuristic(lt, desc, la, lb, lc, lc, pref, 32, res, &n);
    for (int i = 0; i < n; ++i) {
      float t = time_it(st, 10, [&] { cublasLtMatmul(lt, desc, &one, sh.A, la, sh.B, lb, &zero, sh.C, lc, sh.C, lc, &res[i].algo, ws, wsz, st); });
      printf("   lt algo %2d: %.1f us (%.1f TF/s) ws %zu\n", i, 1e3 * t, flop / t / 1e9, res[i].workspaceSize);
    }
  }
  printf("(%s)\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
