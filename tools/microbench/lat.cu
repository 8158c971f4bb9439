// DFMA dependent-chain latency and throughput vs independent chains per warp.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void chain(double* out, int iters, double a, double b, long long* cyc) {
  double x[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) x[i] = threadIdx.x + i;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = fma(x[i], a, b);
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += x[i];
  if (s == 1.2345) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 8); cudaMalloc(&cyc, 8);
  long long h;
  int iters = 4096;
#define RUN(CH, W, B)                                                                          \
  chain<CH><<<B, 32 * W>>>(out, 16, 1.0000001, 1e-9, cyc); cudaDeviceSynchronize();            \
  chain<CH><<<B, 32 * W>>>(out, iters, 1.0000001, 1e-9, cyc); cudaDeviceSynchronize();         \
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);                                              \
  printf("{\"chains\": %d, \"warps_per_block\": %d, \"blocks\": %d, \"cyc_per_iter\": %.2f, \"cyc_per_dfma_per_warp\": %.2f}\n", CH, W, B, (double)h / iters, (double)h / iters / CH);
  RUN(1, 1, 1) RUN(2, 1, 1) RUN(4, 1, 1) RUN(8, 1, 1)
  RUN(1, 4, 1) RUN(1, 8, 1) RUN(1, 16, 1) RUN(2, 8, 1) RUN(4, 4, 1) RUN(4, 8, 1) RUN(8, 8, 1)
  return 0;
}
