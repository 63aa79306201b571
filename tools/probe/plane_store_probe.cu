// Probe: DRAM write throughput when a CTA writes its tile into P separate planes (residue layout
// of ngd_ozaki.cu) with C contiguous bytes per plane per tile, vs one plane.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/probe/plane_store_probe.cu -o tools/probe/plane_store_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cstdlib>

// tile t: plane j gets bytes [t*C, t*C + C) of plane j (planes `pitch` bytes apart)
__global__ void store_planes(uint8_t* out, int64_t pitch, int planes, int C, int ntiles) {
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    for (int j = 0; j < planes; ++j) {
      uint4* o = reinterpret_cast<uint4*>(out + (int64_t)j * pitch + (int64_t)t * C);
      for (int i = threadIdx.x; i < C / 16; i += blockDim.x) o[i] = make_uint4(t, j, i, 7);
    }
  }
}

// read 8 B per output byte-column (an FP64 tile of C elements) then write 16 planes x C bytes
__global__ void read_store(const double* in, uint8_t* out, int64_t pitch, int planes, int C, int ntiles) {
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    unsigned acc = 0;
    const double2* src = reinterpret_cast<const double2*>(in + (int64_t)t * C);
    for (int i = threadIdx.x; i < C / 2; i += blockDim.x) {
      const double2 v = src[i];
      acc += __double2loint(v.x) ^ __double2loint(v.y);
    }
    for (int j = 0; j < planes; ++j) {
      uint4* o = reinterpret_cast<uint4*>(out + (int64_t)j * pitch + (int64_t)t * C);
      for (int i = threadIdx.x; i < C / 16; i += blockDim.x) o[i] = make_uint4(t, j, i, acc);
    }
  }
}

int main2() {
  const int64_t elems = 600ll << 20;  // FP64 elements read (4.8 GB), 16 x 600 MB written
  double* in;
  uint8_t* out;
  if (cudaMalloc(&in, elems * 8) != cudaSuccess || cudaMalloc(&out, elems * 16 + (64 << 20)) != cudaSuccess) return 1;
  cudaMemset(in, 0, elems * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int C : {512, 2048, 8192})
    for (int grid : {148 * 2, 148 * 8}) {
      const int ntiles = (int)(elems / C);
      const int64_t pitch = elems + 9472;
      read_store<<<grid, 256>>>(in, out, pitch, 16, C, ntiles);
      cudaEventRecord(a);
      read_store<<<grid, 256>>>(in, out, pitch, 16, C, ntiles);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("read+16 planes chunk %5d elems grid %4d: %.2f ms  %.0f GB/s (read+write)\n", C, grid, ms,
             (double)elems * 24 / ms / 1e6);
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

int main() {
  if (getenv("MAIN2")) return main2();
  const int64_t total = 8ll << 30;  // bytes written per run
  uint8_t* buf;
  if (cudaMalloc(&buf, total + (64 << 20)) != cudaSuccess) return 1;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int Ps[] = {1, 4, 16, 32};
  const int Cs[] = {512, 2048, 8192, 32768};
  for (int P : Ps)
    for (int C : Cs) {
      const int64_t pitch = total / P + 9472;
      const int ntiles = (int)((total / P) / C) - 1;
      for (int grid : {148 * 2, 148 * 8}) {
        store_planes<<<grid, 256>>>(buf, pitch, P, C, ntiles);
        cudaEventRecord(a);
        store_planes<<<grid, 256>>>(buf, pitch, P, C, ntiles);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("planes %2d chunk %6d B grid %4d: %.2f ms  %.0f GB/s\n", P, C, grid, ms,
               (double)ntiles * C * P / ms / 1e6);
      }
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
