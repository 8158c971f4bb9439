// Microbenchmarks that fix the roofline denominators MEASURED_PEAKS.json lacks
// for this FP64 path: DFMA throughput, DMMA throughput
// and whether the two pipes overlap, L2 size and L2-resident read bandwidth,
// HBM read/copy bandwidth on doubles, back-to-back launch gap (plain and in a
// CUDA graph) and a software grid-barrier round trip.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int CHAINS>
__global__ void dmma_kernel(double* out, int iters, double a, double b) {
  double d[CHAINS][2];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { d[i][0] = 0; d[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) dmma(d[i][0], d[i][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += d[i][0] + d[i][1];
  if (s == 12345.678) out[0] = s;
}

// even warps: DFMA, odd warps: DMMA (same iteration counts as the solo kernels)
template <int CHAINS>
__global__ void mixed_kernel(double* out, int iters_f, int iters_m, double a, double b) {
  int w = threadIdx.x / 32;
  double s = 0;
  if (w % 2 == 0) {
    double x[CHAINS];
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters_f; ++it) {
#pragma unroll
      for (int i = 0; i < CHAINS; ++i) x[i] = fma(x[i], a, b);
    }
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) s += x[i];
  } else {
    double d[CHAINS][2];
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) { d[i][0] = 0; d[i][1] = 0; }
    for (int it = 0; it < iters_m; ++it) {
#pragma unroll
      for (int i = 0; i < CHAINS; ++i) dmma(d[i][0], d[i][1], a, b);
    }
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) s += d[i][0] + d[i][1];
  }
  if (s == 12345.678) out[0] = s;
}

__global__ void read_kernel(const double2* __restrict__ in, size_t n2, double* out) {
  double acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += stride) {
    double2 v = in[i];
    acc += v.x + v.y;
  }
  if (acc == 12345.678) out[0] = acc;
}

__global__ void copy_kernel(const double2* __restrict__ in, double2* __restrict__ o, size_t n2) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += stride) o[i] = in[i];
}

__global__ void empty_kernel(int* p) { if (p && threadIdx.x == 1234567) p[0] = 1; }

__global__ void barrier_kernel(unsigned int* ctr, int rounds, double* out) {
  // sense-free monotone counter barrier: round r completes when ctr >= (r+1)*gridDim.x
  __shared__ int dummy;
  for (int r = 0; r < rounds; ++r) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(ctr, 1u);
      unsigned target = (unsigned)(r + 1) * gridDim.x;
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr));
      } while (v < target);
      dummy = r;
    }
    __syncthreads();
  }
  if (dummy == -5) out[0] = 1;
}

static float time_ms(cudaEvent_t a, cudaEvent_t b) { float ms; CK(cudaEventElapsedTime(&ms, a, b)); return ms; }

int main() {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  int l2 = 0, clk = 0, memclk = 0;
  CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  CK(cudaDeviceGetAttribute(&memclk, cudaDevAttrMemoryClockRate, dev));
  int nsm = prop.multiProcessorCount;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_per_sm\": %zu, \"smem_optin_per_block\": %zu, \"regs_per_sm\": %d, \"clock_khz\": %d, \"mem_clock_khz\": %d}\n",
         prop.name, nsm, l2, prop.sharedMemPerMultiprocessor, prop.sharedMemPerBlockOptin, prop.regsPerMultiprocessor, clk, memclk);
  double* out; CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));

  // ---- DFMA peak ----
  {
    const int CH = 8; int iters = 20000; int threads = 512; int blocks = nsm * 4;
    dfma_kernel<CH><<<blocks, threads>>>(out, 100, 1.0000001, 1e-9);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      CK(cudaEventRecord(e0)); dfma_kernel<CH><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9); CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1)); best = fminf(best, time_ms(e0, e1));
    }
    double fma = (double)blocks * threads * iters * CH;
    printf("{\"test\": \"dfma\", \"ms\": %.4f, \"tflops\": %.3f, \"dfma_per_clk_per_sm_at_boost\": %.2f}\n", best,
           2 * fma / (best * 1e-3) / 1e12, fma / (best * 1e-3) / nsm / (clk * 1e3));
  }
  // ---- DMMA peak (m8n8k4: 256 FMA per warp-instr) ----
  float dmma_ms = 0; double dmma_fma = 0;
  {
    const int CH = 4; int iters = 10000; int threads = 512; int blocks = nsm * 4;
    dmma_kernel<CH><<<blocks, threads>>>(out, 100, 1.0, 1e-9);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      CK(cudaEventRecord(e0)); dmma_kernel<CH><<<blocks, threads>>>(out, iters, 1.0, 1e-9); CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1)); best = fminf(best, time_ms(e0, e1));
    }
    double fma = (double)blocks * (threads / 32) * iters * CH * 256.0;
    dmma_ms = best; dmma_fma = fma;
    printf("{\"test\": \"dmma\", \"ms\": %.4f, \"tflops\": %.3f}\n", best, 2 * fma / (best * 1e-3) / 1e12);
  }
  // ---- mixed: do DFMA and DMMA pipes overlap? ----
  {
    const int CH = 4; int itf = 20000, itm = 5000; int threads = 512; int blocks = nsm * 4;
    mixed_kernel<CH><<<blocks, threads>>>(out, 100, 100, 1.0000001, 1e-9);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      CK(cudaEventRecord(e0)); mixed_kernel<CH><<<blocks, threads>>>(out, itf, itm, 1.0000001, 1e-9); CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1)); best = fminf(best, time_ms(e0, e1));
    }
    double ffma = (double)blocks * (threads / 64) * 32 * itf * CH;
    double mfma = (double)blocks * (threads / 64) * itm * CH * 256.0;
    printf("{\"test\": \"mixed_dfma_dmma\", \"ms\": %.4f, \"combined_tflops\": %.3f, \"dfma_part_tflops\": %.3f, \"dmma_part_tflops\": %.3f}\n",
           best, 2 * (ffma + mfma) / (best * 1e-3) / 1e12, 2 * ffma / (best * 1e-3) / 1e12, 2 * mfma / (best * 1e-3) / 1e12);
  }
  // ---- bandwidth: HBM read, HBM copy, L2-resident read ----
  {
    size_t big = (size_t)2 << 30;  // 2 GiB
    double2* a; double2* b; CK(cudaMalloc(&a, big)); CK(cudaMalloc(&b, big));
    CK(cudaMemset(a, 0, big)); CK(cudaMemset(b, 0, big));
    size_t n2 = big / sizeof(double2);
    int blocks = nsm * 8, threads = 512;
    read_kernel<<<blocks, threads>>>(a, n2, out); CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) { CK(cudaEventRecord(e0)); read_kernel<<<blocks, threads>>>(a, n2, out); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); best = fminf(best, time_ms(e0, e1)); }
    printf("{\"test\": \"hbm_read\", \"bytes\": %zu, \"ms\": %.4f, \"gbs\": %.1f}\n", big, best, big / (best * 1e-3) / 1e9);
    best = 1e30f;
    for (int r = 0; r < 5; ++r) { CK(cudaEventRecord(e0)); copy_kernel<<<blocks, threads>>>(a, b, n2 / 2); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); best = fminf(best, time_ms(e0, e1)); }
    printf("{\"test\": \"hbm_copy\", \"bytes_rw\": %zu, \"ms\": %.4f, \"gbs\": %.1f}\n", big, best, big / (best * 1e-3) / 1e9);
    for (size_t mb : {8, 16, 32, 48, 64, 96}) {
      size_t bytes = mb << 20; size_t m2 = bytes / sizeof(double2);
      read_kernel<<<blocks, threads>>>(a, m2, out);
      CK(cudaDeviceSynchronize());
      best = 1e30f;
      for (int r = 0; r < 10; ++r) { CK(cudaEventRecord(e0)); read_kernel<<<blocks, threads>>>(a, m2, out); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); best = fminf(best, time_ms(e0, e1)); }
      printf("{\"test\": \"l2_read\", \"mb\": %zu, \"ms\": %.5f, \"gbs\": %.1f}\n", mb, best, bytes / (best * 1e-3) / 1e9);
    }
    CK(cudaFree(a)); CK(cudaFree(b));
  }
  // ---- launch gap ----
  {
    int n = 2000;
    cudaStream_t s; CK(cudaStreamCreate(&s));
    for (int i = 0; i < 100; ++i) empty_kernel<<<nsm, 256, 0, s>>>(nullptr);
    CK(cudaStreamSynchronize(s));
    CK(cudaEventRecord(e0, s));
    for (int i = 0; i < n; ++i) empty_kernel<<<nsm, 256, 0, s>>>(nullptr);
    CK(cudaEventRecord(e1, s)); CK(cudaEventSynchronize(e1));
    printf("{\"test\": \"launch_stream\", \"us_per_launch\": %.3f}\n", time_ms(e0, e1) * 1e3 / n);
    cudaGraph_t g; cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
    for (int i = 0; i < 400; ++i) empty_kernel<<<nsm, 256, 0, s>>>(nullptr);
    CK(cudaStreamEndCapture(s, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    CK(cudaGraphLaunch(ge, s)); CK(cudaStreamSynchronize(s));
    CK(cudaEventRecord(e0, s));
    for (int i = 0; i < 5; ++i) CK(cudaGraphLaunch(ge, s));
    CK(cudaEventRecord(e1, s)); CK(cudaEventSynchronize(e1));
    printf("{\"test\": \"launch_graph\", \"us_per_launch\": %.3f}\n", time_ms(e0, e1) * 1e3 / 2000);
    // grid barrier
    unsigned int* ctr; CK(cudaMalloc(&ctr, 4));
    int rounds = 2000;
    for (int blocks : {nsm, 2 * nsm}) {
      CK(cudaMemset(ctr, 0, 4));
      barrier_kernel<<<blocks, 256, 0, s>>>(ctr, 10, out); CK(cudaStreamSynchronize(s));
      CK(cudaMemset(ctr, 0, 4));
      CK(cudaEventRecord(e0, s));
      barrier_kernel<<<blocks, 256, 0, s>>>(ctr, rounds, out);
      CK(cudaEventRecord(e1, s)); CK(cudaEventSynchronize(e1));
      printf("{\"test\": \"grid_barrier\", \"blocks\": %d, \"us_per_barrier\": %.3f}\n", blocks, time_ms(e0, e1) * 1e3 / rounds);
    }
  }
  CK(cudaGetLastError());
  return 0;
}
