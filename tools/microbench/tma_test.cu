// Minimal TMA (cp.async.bulk.tensor.4d, fp64, zero-filled halo box) + mbarrier test.
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e_), __LINE__); return 1; } } while (0)
__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
template <int FENCE>
__global__ void k(const __grid_constant__ CUtensorMap tm, double* out, int x0, int y0, int z0) {
  __shared__ __align__(1024) double buf[4 * 600];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&bar)), "r"(1) : "memory");
    if (FENCE == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    else if (FENCE == 1) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(4 * 600 * 8) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(su(buf)),
        "l"(reinterpret_cast<uint64_t>(&tm)), "r"(x0), "r"(y0), "r"(z0), "r"(0), "r"(su(&bar))
        : "memory");
  }
  asm volatile("{\n .reg .pred P;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra W_%=;\n}\n" ::"r"(su(&bar)),
               "r"(0)
               : "memory");
  for (int i = threadIdx.x; i < 2400; i += blockDim.x) out[i] = buf[i];
}
int main(int argc, char** argv) {
  const int var = argc > 1 ? atoi(argv[1]) : 0, dt = argc > 2 ? atoi(argv[2]) : 0;
  const int N = 64, nm = 4;
  const size_t n = (size_t)N * N * N * nm;
  double* h = new double[n];
  for (size_t i = 0; i < n; ++i) h[i] = (double)i;
  double *d, *o;
  CK(cudaMalloc(&d, n * 8));
  CK(cudaMalloc(&o, 2400 * 8));
  CK(cudaMemcpy(d, h, n * 8, cudaMemcpyHostToDevice));
  const int l2 = argc > 3 ? atoi(argv[3]) : 1, bx = argc > 4 ? atoi(argv[4]) : 6, direct = argc > 5 ? atoi(argv[5]) : 0;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  auto enc = direct ? cuTensorMapEncodeTiled : (PFN_cuTensorMapEncodeTiled_v12000)fn;
  CUtensorMap tm;
  cuuint64_t dims[4] = {N, N, N, (cuuint64_t)nm}, str[3] = {N * 8, N * N * 8, (cuuint64_t)N * N * N * 8};
  cuuint32_t box[4] = {(cuuint32_t)bx, 10, 10, 4}, es[4] = {1, 1, 1, 1};
  CUresult r = enc(&tm, dt ? CU_TENSOR_MAP_DATA_TYPE_INT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, l2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  double* ho = new double[2400];
  const int first = argc > 6 ? atoi(argv[6]) : 0;
  for (int f = first; f < 2; ++f) {
    const int x0a = f ? 3 : -1, y0a = f ? 7 : -1, z0a = f ? 7 : -1;
    if (var == 0) k<0><<<1, 128>>>(tm, o, x0a, y0a, z0a);
    else if (var == 1) k<1><<<1, 128>>>(tm, o, x0a, y0a, z0a);
    else k<2><<<1, 128>>>(tm, o, x0a, y0a, z0a);
    cudaError_t e = cudaDeviceSynchronize();
    printf("fence variant %d: %s\n", f, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    CK(cudaMemcpy(ho, o, 2400 * 8, cudaMemcpyDeviceToHost));
    int x0 = f ? 3 : -1, y0 = f ? 7 : -1, z0 = f ? 7 : -1, bad = 0;
    for (int m = 0; m < 4; ++m)
      for (int z = 0; z < 10; ++z)
        for (int y = 0; y < 10; ++y)
          for (int x = 0; x < 6; ++x) {
            int gx = x0 + x, gy = y0 + y, gz = z0 + z;
            double ex = (gx < 0 || gy < 0 || gz < 0 || gx >= N || gy >= N || gz >= N)
                            ? 0.0
                            : (double)(gx + N * (gy + N * (gz + (size_t)N * m)));
            if (ho[x + 6 * (y + 10 * (z + 10 * m))] != ex) bad++;
          }
    printf("variant %d mismatches %d\n", f, bad);
  }
  return 0;
}
