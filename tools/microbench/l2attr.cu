// L2 persistence capabilities of device 0
#include <cstdio>
#include <cuda_runtime.h>
int main() {
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxPersistingL2CacheSize, 0);
  printf("{\"max_persisting_l2_bytes\": %d, ", v);
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxAccessPolicyWindowSize, 0);
  printf("\"max_access_policy_window_bytes\": %d, ", v);
  cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, 0);
  printf("\"l2_bytes\": %d}\n", v);
  return 0;
}
