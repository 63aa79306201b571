#include <cstdio>
int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  printf("l2CacheSize %d persistingL2CacheMaxSize %d accessPolicyMaxWindowSize %d\n", p.l2CacheSize,
         p.persistingL2CacheMaxSize, p.accessPolicyMaxWindowSize);
  return 0;
}
