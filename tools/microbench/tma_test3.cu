// TMA probe: 2-D fp64 box load at (0,0), encode via the driver API linked directly (-lcuda).
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void k2d(const __grid_constant__ CUtensorMap tm, double* out, int x0, int y0, int z0, int bxw) {
  __shared__ __align__(1024) double buf[32 * 10 * 10];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&bar)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(bxw * 10 * 10 * 8) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(su(buf)),
        "l"(reinterpret_cast<uint64_t>(&tm)), "r"(su(&bar)), "r"(x0), "r"(y0), "r"(z0)
        : "memory");
  }
  asm volatile("{\n .reg .pred P;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra W_%=;\n}\n" ::"r"(su(&bar)),
               "r"(0)
               : "memory");
  for (int i = threadIdx.x; i < bxw * 100; i += blockDim.x) out[i] = buf[i];
}
int main(int argc, char** argv) {
  const int bxw = argc > 1 ? atoi(argv[1]) : 6;
  const int N = 64;
  double* h = new double[N * N * N];
  for (int i = 0; i < N * N * N; ++i) h[i] = i;
  double *d, *o;
  cudaMalloc(&d, N * N * N * 8);
  cudaMalloc(&o, 3200 * 8);
  cudaMemcpy(d, h, N * N * N * 8, cudaMemcpyHostToDevice);
  CUtensorMap tm;
  cuuint64_t dims[3] = {N, N, N}, str[2] = {N * 8, N * N * 8};
  cuuint32_t box[3] = {(cuuint32_t)bxw, 10, 10}, es[3] = {1, 1, 1};
  CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, str, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  for (int f = 0; f < 2; ++f) {
    const int x0 = f ? -2 : (argc > 2 ? atoi(argv[2]) : 3), y0 = f ? -1 : (argc > 3 ? atoi(argv[3]) : 7), z0 = f ? -1 : (argc > 4 ? atoi(argv[4]) : 7);
    k2d<<<1, 128>>>(tm, o, x0, y0, z0, bxw);
    cudaError_t e = cudaDeviceSynchronize();
    printf("3d load (%d,%d,%d): %s\n", x0, y0, z0, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    double ho[3200];
    cudaMemcpy(ho, o, bxw * 100 * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int z = 0; z < 10; ++z) for (int y = 0; y < 10; ++y) for (int x = 0; x < bxw; ++x) {
      int gx = x0 + x, gy = y0 + y, gz = z0 + z;
      double ex = (gx < 0 || gy < 0 || gz < 0 || gx >= N || gy >= N || gz >= N) ? 0.0 : (double)(gx + N * (gy + N * gz));
      bad += ho[x + bxw * (y + 10 * z)] != ex;
    }
    printf("mismatches %d\n", bad);
  }
  return 0;
}
