// standalone TMA 2D load probe: ./tma_test <boxw> <boxh> <x> <y> <promo> <dynsmem>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__global__ void k(const __grid_constant__ CUtensorMap tmap, int x, int y, int bytes, int* out, int n) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  unsigned char* al = sm + ((128u - (smem_u32(sm) & 127u)) & 127u);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      :: "r"(smem_u32(al)), "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(x), "r"(y), "r"(smem_u32(&bar)) : "memory");
  }
  uint32_t done = 0;
  do { asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(smem_u32(&bar)), "r"(0) : "memory"); } while (!done);
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = reinterpret_cast<int*>(al)[i];
}
int main(int argc, char** argv) {
  int bw = atoi(argv[1]), bh = atoi(argv[2]), x = atoi(argv[3]), y = atoi(argv[4]), promo = atoi(argv[5]);
  int P = 128;
  std::vector<int> h(P * P); for (int i = 0; i < P * P; ++i) h[i] = i;
  int *d, *o; cudaMalloc(&d, P * P * 4); cudaMalloc(&o, bw * bh * 4);
  cudaMemcpy(d, h.data(), P * P * 4, cudaMemcpyHostToDevice);
  void* fp = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
  CUtensorMap m;
  cuuint64_t gdim[2] = {(cuuint64_t)P, (cuuint64_t)P}; cuuint64_t gs[1] = {(cuuint64_t)P * 4};
  cuuint32_t box[2] = {(cuuint32_t)bw, (cuuint32_t)bh}; cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_INT32, 2, d, gdim, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
    CU_TENSOR_MAP_SWIZZLE_NONE, promo ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode=%d ", (int)r);
  k<<<1, 128, bw * bh * 4 + 256>>>(m, x, y, bw * bh * 4, o, bw * bh);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<int> ho(bw * bh); cudaMemcpy(ho.data(), o, bw * bh * 4, cudaMemcpyDeviceToHost);
  printf("box %dx%d at (%d,%d) promo %d -> %s first %d %d second-row %d\n", bw, bh, x, y, promo, cudaGetErrorString(e), ho[0], ho[1], ho[bw]);
  return 0;
}
