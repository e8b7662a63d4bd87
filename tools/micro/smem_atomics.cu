// Microbenchmark: shared-memory deposit mechanisms on B200 (per SM rates).
//   mode 0: LDS+FADD+STS to a thread-private slot (owner RMW)
//   mode 1: atomicAdd(float) on shared, spread addresses (CAS loop on sm_100)
//   mode 2: atomicAdd(int) on shared, spread addresses (native ATOMS.ADD)
//   mode 3: red.global.add.f32, spread addresses (L2)
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float* gout, int iters) {
  __shared__ float sf[4096 + 4096 * 0];
  __shared__ int si[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) { sf[i] = 0; si[i] = 0; }
  __syncthreads();
  unsigned h = threadIdx.x * 2654435761u + blockIdx.x * 97u;
  float acc = 0;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int j = 0; j < 8; j++) {
      h = h * 1664525u + 1013904223u;
      int a;
      if (MODE == 0) a = ((j * 4 + (it & 3)) * 256 + threadIdx.x) & 4095;
      else a = (threadIdx.x * 32 + (h >> 27) + j * 7) & 4095;
      float v = (float)(h & 255) * 1e-3f;
      if (MODE == 0) sf[a] += v;
      else if (MODE == 1) atomicAdd(&sf[a], v);
      else if (MODE == 2) atomicAdd(&si[a], (int)(h & 255));
      else atomicAdd(&gout[(blockIdx.x * 8192 + a) & ((1 << 24) - 1)], v);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) acc += sf[i] + si[i];
  if (acc == 12345.f) gout[0] = acc;
}
int main() {
  float* g; cudaMalloc(&g, sizeof(float) << 24); cudaMemset(g, 0, sizeof(float) << 24);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int iters = 2000; int blocks = sms * 4, threads = 256;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const char* names[] = {"owner LDS+FADD+STS", "atomicAdd f32 smem", "atomicAdd s32 smem", "red.global f32"};
  for (int mode = 0; mode < 4; mode++) {
    for (int rep = 0; rep < 2; rep++) {
      cudaEventRecord(a);
      if (mode == 0) k<0><<<blocks, threads>>>(g, iters);
      if (mode == 1) k<1><<<blocks, threads>>>(g, iters);
      if (mode == 2) k<2><<<blocks, threads>>>(g, iters);
      if (mode == 3) k<3><<<blocks, threads>>>(g, iters / 10);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double ops = (double)blocks * threads * 8 * (mode == 3 ? iters / 10 : iters);
      if (rep) printf("%-22s %8.3f ms  %8.1f Gop/s  %.2f op/clk/SM@1.9GHz\n", names[mode], ms, ops / ms / 1e6, ops / (ms * 1e-3) / sms / 1.9e9);
    }
  }
  return 0;
}
