// TMA probe: 2-D fp64 box load at (0,0), encode via the driver API linked directly (-lcuda).
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void k2d(const __grid_constant__ CUtensorMap tm, double* out, int x0, int y0) {
  __shared__ __align__(1024) double buf[16 * 16];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&bar)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(16 * 16 * 8) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(su(buf)),
        "l"(reinterpret_cast<uint64_t>(&tm)), "r"(su(&bar)), "r"(x0), "r"(y0)
        : "memory");
  }
  asm volatile("{\n .reg .pred P;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra W_%=;\n}\n" ::"r"(su(&bar)),
               "r"(0)
               : "memory");
  for (int i = threadIdx.x; i < 256; i += blockDim.x) out[i] = buf[i];
}
int main() {
  const int N = 64;
  double* h = new double[N * N];
  for (int i = 0; i < N * N; ++i) h[i] = i;
  double *d, *o;
  cudaMalloc(&d, N * N * 8);
  cudaMalloc(&o, 256 * 8);
  cudaMemcpy(d, h, N * N * 8, cudaMemcpyHostToDevice);
  CUtensorMap tm;
  cuuint64_t dims[2] = {N, N}, str[1] = {N * 8};
  cuuint32_t box[2] = {16, 16}, es[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, str, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  k2d<<<1, 128>>>(tm, o, 0, 0);
  cudaError_t e = cudaDeviceSynchronize();
  printf("2d load: %s\n", cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  double ho[256];
  cudaMemcpy(ho, o, 256 * 8, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int y = 0; y < 16; ++y)
    for (int x = 0; x < 16; ++x) bad += ho[x + 16 * y] != (double)(x + N * y);
  printf("mismatches %d\n", bad);
  return 0;
}
