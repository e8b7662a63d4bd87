// Minimal TMA (cp.async.bulk.tensor.3d + mbarrier) probe: loads a 64 x 16
// box of a float32 volume into shared memory and writes it back out.
// Variants (argv[1]): 0 grid_constant map, 1 + __cluster_dims__(1,1,1),
// 2 map in global memory, 3 grid_constant map with cudaLaunchKernelEx
// cluster (1,1,1).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tma_probe tma_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned s32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void body(const CUtensorMap* map, float* out,
                                     int x0, int y0, int z0) {
  __shared__ alignas(128) float tile[16][64];
  __shared__ alignas(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(s32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(s32(&bar)), "r"(4096) : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(s32(&tile[0][0])), "l"(map), "r"(x0), "r"(y0), "r"(z0), "r"(s32(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(s32(&bar)) : "memory");
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) out[i] = tile[i / 64][i % 64];
}

__global__ void k4(float* out) {  // mbarrier only
  __shared__ alignas(8) uint64_t bar;
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(s32(&bar)) : "memory");
  __syncthreads();
  if (threadIdx.x == 0) asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(s32(&bar)) : "memory");
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(s32(&bar)) : "memory");
  if (threadIdx.x == 0) out[0] = 1.f;
}
__global__ void k5(const float* src, float* out) {  // 1D bulk copy
  __shared__ alignas(128) float tile[1024];
  __shared__ alignas(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(s32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(s32(&bar)), "r"(4096) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(s32(&tile[0])), "l"(src), "r"(4096), "r"(s32(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(s32(&bar)) : "memory");
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) out[i] = tile[i];
}
__global__ void k6(const __grid_constant__ CUtensorMap map, float* out) {  // 2D map
  __shared__ alignas(128) float tile[16][64];
  __shared__ alignas(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(s32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(s32(&bar)), "r"(4096) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(s32(&tile[0][0])), "l"(&map), "r"(0), "r"(0), "r"(s32(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(s32(&bar)) : "memory");
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) out[i] = tile[i / 64][i % 64];
}
__global__ void k0(const __grid_constant__ CUtensorMap map, float* out, int x0, int y0, int z0) { body(&map, out, x0, y0, z0); }
__global__ void __cluster_dims__(1, 1, 1) k1(const __grid_constant__ CUtensorMap map, float* out, int x0, int y0, int z0) { body(&map, out, x0, y0, z0); }
__global__ void k2(const CUtensorMap* map, float* out, int x0, int y0, int z0) { body(map, out, x0, y0, z0); }

int main(int argc, char** argv) {
  const int variant = argc > 1 ? atoi(argv[1]) : 0;
  const int nx = 128, ny = 40, nz = 8;
  float* h = new float[nx * ny * nz];
  for (int i = 0; i < nx * ny * nz; i++) h[i] = (float)i;
  float *d, *o;
  cudaMalloc(&d, sizeof(float) * nx * ny * nz);
  cudaMalloc(&o, sizeof(float) * 1024);
  cudaMemcpy(d, h, sizeof(float) * nx * ny * nz, cudaMemcpyHostToDevice);
  PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn, cudaEnableDefault, &q);
  CUtensorMap m;
  cuuint64_t dims[3] = {nx, ny, nz}, str[2] = {nx * 4, nx * ny * 4};
  cuuint32_t box[3] = {64, 16, 1}, es[3] = {1, 1, 1};
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaMemset(o, 0, 4096);
  if (variant == 0) k0<<<1, 128>>>(m, o, -2, -1, 3);
  if (variant == 8) k0<<<1, 128>>>(m, o, 0, 0, 3);
  if (variant == 9) k0<<<1, 128>>>(m, o, 4, 0, 0);
  if (variant == 10) k0<<<1, 128>>>(m, o, 0, -1, 0);
  if (variant == 11) k0<<<1, 128>>>(m, o, -4, 0, 0);
  if (variant == 1) k1<<<1, 128>>>(m, o, -2, -1, 3);
  if (variant == 2) {
    CUtensorMap* dm;
    cudaMalloc(&dm, sizeof(CUtensorMap));
    cudaMemcpy(dm, &m, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
    k2<<<1, 128>>>(dm, o, -2, -1, 3);
  }
  if (variant == 3) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1); cfg.blockDim = dim3(128);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k0, m, o, -2, -1, 3);
  }
  if (variant == 6 || variant == 7) {
    CUtensorMap m2;
    cuuint64_t d2[2] = {nx, ny * nz}, s2[1] = {nx * 4};
    cuuint32_t b2[2] = {64, 16}, e2[2] = {1, 1};
    CUresult r2 = (variant == 6 ? fn : cuTensorMapEncodeTiled)(&m2, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, d2, s2, b2, e2,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("2D encode %d\n", (int)r2);
    k6<<<1, 128>>>(m2, o);
  }
  if (variant == 4) k4<<<1, 128>>>(o);
  if (variant == 5) k5<<<1, 128>>>(d, o);
  cudaError_t e = cudaDeviceSynchronize();
  float ho[1024];
  cudaMemcpy(ho, o, 4096, cudaMemcpyDeviceToHost);
  printf("variant %d encode %d: %s  t[0][0]=%g (want 0)  t[1][2]=%g (want %g)\n",
         variant, (int)r, cudaGetErrorString(e), ho[0], ho[66], (float)(3 * nx * ny + 0));
  return e != cudaSuccess;
}
