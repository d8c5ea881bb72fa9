// Does a tiled TMA load accept an inner-dimension box origin that is only
// 8-byte aligned in global memory?
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap m, int c0, float* out) {
  __shared__ __align__(128) float buf[76 * 8];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar)), "r"(76 * 8 * 4));
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(s32(buf)), "l"((uint64_t)&m), "r"(c0), "r"(0), "r"(s32(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(s32(&bar)));
  __syncthreads();
  if (threadIdx.x < 76) out[threadIdx.x] = buf[threadIdx.x];
}
int main() {
  const int W = 256, Hh = 8;
  float* g; cudaMalloc(&g, W * Hh * 4);
  float h[W * Hh]; for (int i = 0; i < W * Hh; ++i) h[i] = (float)i;
  cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap m;
  cuuint64_t dims[2] = {W, Hh}; cuuint64_t str[1] = {W * 4}; cuuint32_t box[2] = {76, 8}, es[2] = {1, 1};
  CUresult r = ((PFN_cuTensorMapEncodeTiled_v12000)fn)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, dims, str, box, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  float* o; cudaMalloc(&o, 76 * 4);
  int origins[4] = {4, 2, -2, -6};
  for (int i = 0; i < 4; ++i) {
    k<<<1, 128>>>(m, origins[i], o);
    cudaError_t e = cudaDeviceSynchronize();
    float ho[76]; cudaMemcpy(ho, o, sizeof(ho), cudaMemcpyDeviceToHost);
    printf("origin %d: %s first=%g\n", origins[i], cudaGetErrorString(e), ho[0]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
