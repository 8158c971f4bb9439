// Does DFMA throughput depend on operand values?  Same kernel, different data.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(const double* __restrict__ in, double* out, int iters) {
  double a = in[0], b = in[1];
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = in[2 + i];
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1.2345) out[0] = s;
}
int main() {
  double *d, *o; cudaMalloc(&d, 80); cudaMalloc(&o, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  struct { const char* name; double v[10]; } cases[] = {
    {"normal", {0.999999, 1e-9, 1, 2, 3, 4, 5, 6, 7, 8}},
    {"zeros", {0, 0, 0, 0, 0, 0, 0, 0, 0, 0}},
    {"a=0 x!=0", {0, 1e-9, 1, 2, 3, 4, 5, 6, 7, 8}},
    {"x=0 a!=0 b=0", {0.999999, 0, 0, 0, 0, 0, 0, 0, 0, 0}},
    {"subnormal", {0.5, 1e-310, 1e-310, 2e-310, 3e-310, 4e-310, 5e-310, 6e-310, 7e-310, 8e-310}},
    {"a=1 b=0", {1, 0, 1, 2, 3, 4, 5, 6, 7, 8}},
  };
  int iters = 20000, blocks = 148 * 4, threads = 512;
  for (auto& c : cases) {
    cudaMemcpy(d, c.v, 80, cudaMemcpyHostToDevice);
    k<<<blocks, threads>>>(d, o, 100); cudaDeviceSynchronize();
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); k<<<blocks, threads>>>(d, o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double fl = 2.0 * blocks * threads * iters * 8;
    printf("{\"case\": \"%s\", \"ms\": %.3f, \"tflops\": %.2f}\n", c.name, best, fl / best / 1e9);
  }
  return 0;
}
