// Microbenchmark: per-SM fetch rates for the Ax trilinear sample on B200.
// All reads hit L1 / shared memory (each CTA works inside a small window),
// so the numbers are the pipe ceilings the Ax kernel design chooses between:
//   tld4   : tld4.r.a2d (2x2 gather of one layer, 4 values per thread)
//   tex1   : tex.a2d point fetch (1 value per thread)
//   lds32  : LDS.32, conflict-free
//   lds64  : LDS.64, conflict-free
//   lds128 : LDS.128, conflict-free
//   ldg32  : ld.global.nc.f32, L1-hit
//   ldg64  : ld.global.nc.v2.f32, L1-hit
//   mix    : 1 tld4 + 4 LDS.32 per step (do the pipes overlap?)
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a fetch_rates.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float4 g4(cudaTextureObject_t t, int layer, float x,
                                     float y) {
  float4 r;
  asm volatile(
      "tld4.r.a2d.v4.f32.f32 {%0, %1, %2, %3}, [%4, {%5, %6, %7, %8}];"
      : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
      : "l"(t), "r"(layer), "f"(x), "f"(y), "f"(0.f));
  return r;
}
__device__ __forceinline__ float t1(cudaTextureObject_t t, int layer, float x,
                                   float y) {
  float4 r;
  asm volatile(
      "tex.a2d.v4.f32.f32 {%0, %1, %2, %3}, [%4, {%5, %6, %7, %8}];"
      : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
      : "l"(t), "r"(layer), "f"(x), "f"(y), "f"(0.f));
  return r.x;
}

constexpr int UNR = 8;

template <int MODE>
__global__ void __launch_bounds__(256) k(cudaTextureObject_t tex,
                                         cudaTextureObject_t tex4, cudaTextureObject_t tex2,
                                         const float* __restrict__ gv,
                                         const float* __restrict__ g,
                                         float* out, int iters) {
  __shared__ __align__(16) float s[8192];
  for (int i = threadIdx.x; i < 8192; i += 256) s[i] = (float)i * 1e-4f;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // warp = 8u x 4v tile like the Ax kernel; CTA window ~ 48 x 24 texels
  const float bx = (float)((blockIdx.x & 7) * 48 + (lane & 7) + (warp & 1) * 8);
  const float by = (float)(((blockIdx.x >> 3) & 7) * 24 + (lane >> 3) + (warp >> 1) * 4);
  const int layer0 = (blockIdx.x >> 6) & 7;
  const float* gb = g + ((blockIdx.x & 63) * 4096);
  float acc = 0.f;
  for (int it = 0; it < iters; it++) {
    const float f = (float)(it & 15) * 0.53f;
#pragma unroll
    for (int j = 0; j < UNR; j++) {
      const float x = bx + f + (float)j * 0.71f, y = by + f * 0.5f + (float)j * 0.13f;
      if (MODE == 0) {
        float4 r = g4(tex, layer0 + (j & 1), x, y);
        acc += r.x + r.y + r.z + r.w;
      } else if (MODE == 1) {
        acc += t1(tex, layer0 + (j & 1), x, y);
      } else if (MODE == 2) {
        acc += s[((it * 7 + j * 33) & 255) * 32 + lane];
      } else if (MODE == 3) {
        float2 v = reinterpret_cast<const float2*>(s)[((it * 7 + j * 33) & 127) * 32 + lane];
        acc += v.x + v.y;
      } else if (MODE == 4) {
        float4 v = reinterpret_cast<const float4*>(s)[((it * 7 + j * 33) & 63) * 32 + lane];
        acc += v.x + v.y + v.z + v.w;
      } else if (MODE == 5) {
        acc += __ldg(gb + ((it * 7 + j * 33) & 127) * 32 + lane);
      } else if (MODE == 6) {
        float2 v = __ldg(reinterpret_cast<const float2*>(gb) + ((it * 7 + j * 33) & 63) * 32 + lane);
        acc += v.x + v.y;
      } else if (MODE == 8) {  // float4-texel point fetch
        float4 r = tex2DLayered<float4>(tex4, x, y, layer0 + (j & 1));
        acc += r.x + r.y + r.z + r.w;
      } else if (MODE == 9) {  // float2-texel point fetch
        float2 r = tex2DLayered<float2>(tex2, x, y, layer0 + (j & 1));
        acc += r.x + r.y;
      } else if (MODE == 10) {  // ldg32, lanes scattered over 8 rows x 4 planes
        const int xi = (int)x, yi = (int)y;
        acc += __ldg(gv + ((size_t)(layer0 + (j & 3)) * 256 + (lane >> 3) * 8 + yi % 8) * 512 + (xi & 511));
      } else if (MODE == 11) {  // tld4 + 4 scattered ldg32 per step
        if (j & 1) {
          float4 r = g4(tex, layer0, x, y);
          acc += r.x + r.y + r.z + r.w;
        } else {
          const int xi = (int)x, yi = (int)y;
          const float* q = gv + ((size_t)(layer0 + 1) * 256 + yi) * 512 + (xi & 511);
          acc += __ldg(q) + __ldg(q + 1) + __ldg(q + 512) + __ldg(q + 513);
        }
      } else if (MODE == 13) {  // Ax-like: 8u x 4v rays, lanes 1.41 texels apart
        const float xr = (float)((blockIdx.x & 7) * 48) + (float)(lane & 7) * 1.41f + f + (float)j * 0.5f;
        const float yr = (float)(((blockIdx.x >> 3) & 7) * 24) + (float)(lane >> 3) * 1.41f + f * 0.3f;
        float4 r = g4(tex, layer0 + (j & 1), xr, yr);
        acc += r.x + r.y + r.z + r.w;
      } else if (MODE == 14) {  // quad = 4 consecutive samples (0.5 texel) of one ray
        const int ray = lane >> 2, smp = lane & 3;
        const float xr = (float)((blockIdx.x & 7) * 48) + (float)(ray & 7) * 1.41f + f + (float)(j * 4 + smp) * 0.5f;
        const float yr = (float)(((blockIdx.x >> 3) & 7) * 24) + (float)(warp & 3) * 1.41f + f * 0.3f;
        float4 r = g4(tex, layer0 + (j & 1), xr, yr);
        acc += r.x + r.y + r.z + r.w;
      } else if (MODE == 15) {  // 25% of lanes active, one per quad
        if (((lane + j) & 3) == 0) {
          float4 r = g4(tex, layer0 + (j & 1), x, y);
          acc += r.x + r.y + r.z + r.w;
        }
      } else if (MODE == 16) {  // 25% of lanes active, whole quads
        if ((((lane >> 2) + j) & 3) == 0) {
          float4 r = g4(tex, layer0 + (j & 1), x, y);
          acc += r.x + r.y + r.z + r.w;
        }
      } else if (MODE == 17) {  // 25% of lanes active, one warp-quarter (8 lanes)
        if ((((lane >> 3) + j) & 3) == 0) {
          float4 r = g4(tex, layer0 + (j & 1), x, y);
          acc += r.x + r.y + r.z + r.w;
        }
      } else if (MODE == 12) {  // 2 float4 point fetches (one sample's 8 taps)
        float4 r = tex2DLayered<float4>(tex4, x, y, layer0 + (j & 1));
        float4 r2 = tex2DLayered<float4>(tex4, x, y + 1.f, layer0 + (j & 1));
        acc += r.x + r.y + r.z + r.w + r2.x + r2.y + r2.z + r2.w;
      } else {
        if (j & 1) {
          float4 r = g4(tex, layer0, x, y);
          acc += r.x + r.y + r.z + r.w;
        } else {
          const int b = ((it * 7 + j * 33) & 63) * 32 + lane;
          acc += s[b] + s[b + 2048] + s[b + 4096] + s[b + 6144];
        }
      }
    }
  }
  if (acc == 1234.5f) out[0] = acc;
}

int main() {
  const int W = 512, H = 256, L = 16;
  cudaArray_t arr;
  cudaChannelFormatDesc cd = cudaCreateChannelDesc<float>();
  cudaMalloc3DArray(&arr, &cd, make_cudaExtent(W, H, L), cudaArrayLayered);
  float* host = new float[(size_t)W * H * L];
  for (size_t i = 0; i < (size_t)W * H * L; i++) host[i] = (float)(i % 977) * 1e-3f;
  cudaMemcpy3DParms p = {};
  p.srcPtr = make_cudaPitchedPtr(host, W * 4, W, H);
  p.dstArray = arr;
  p.extent = make_cudaExtent(W, H, L);
  p.kind = cudaMemcpyHostToDevice;
  cudaMemcpy3D(&p);
  cudaResourceDesc rd = {};
  rd.resType = cudaResourceTypeArray;
  rd.res.array.array = arr;
  cudaTextureDesc td = {};
  td.addressMode[0] = td.addressMode[1] = cudaAddressModeBorder;
  td.filterMode = cudaFilterModePoint;
  td.readMode = cudaReadModeElementType;
  cudaTextureObject_t tex;
  cudaCreateTextureObject(&tex, &rd, &td, nullptr);
  auto mk = [&](cudaChannelFormatDesc c, size_t esz) {
    cudaArray_t ar;
    cudaMalloc3DArray(&ar, &c, make_cudaExtent(W, H, L), cudaArrayLayered);
    char* hb = new char[(size_t)W * H * L * esz];
    for (size_t i = 0; i < (size_t)W * H * L * esz; i++) hb[i] = (char)(i % 13);
    cudaMemcpy3DParms q = {};
    q.srcPtr = make_cudaPitchedPtr(hb, W * esz, W, H);
    q.dstArray = ar; q.extent = make_cudaExtent(W, H, L); q.kind = cudaMemcpyHostToDevice;
    cudaMemcpy3D(&q);
    cudaResourceDesc r2 = {}; r2.resType = cudaResourceTypeArray; r2.res.array.array = ar;
    cudaTextureObject_t t; cudaCreateTextureObject(&t, &r2, &td, nullptr);
    return t;
  };
  cudaTextureObject_t tex4 = mk(cudaCreateChannelDesc<float4>(), 16);
  cudaTextureObject_t tex2 = mk(cudaCreateChannelDesc<float2>(), 8);
  float* gv; cudaMalloc(&gv, sizeof(float) * W * H * L); cudaMemset(gv, 0, sizeof(float) * W * H * L);
  float* g;
  cudaMalloc(&g, sizeof(float) * 64 * 4096 + 4096 * 4);
  cudaMemset(g, 0, sizeof(float) * 64 * 4096);
  float* out;
  cudaMalloc(&out, 16);
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double ghz = clk * 1e-6;
  const int blocks = sms * 8, iters = 4000;
  const char* names[] = {"tld4 (4 val)", "tex point (1 val)", "lds32", "lds64",
                         "lds128", "ldg32 L1-hit", "ldg64 L1-hit",
                         "mix tld4 + 4 lds32", "tex float4 point", "tex float2 point", "ldg32 scattered 8y4z", "mix tld4 + 4 ldg32", "2x float4 point (8 taps)", "tld4 Ax-like spread rays", "tld4 quad = 4 samples of a ray", "tld4 25% lanes (1/quad)", "tld4 25% lanes (whole quads)", "tld4 25% lanes (8 contiguous)"};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  printf("SMs %d, clock %.3f GHz (nominal max)\n", sms, ghz);
  for (int mode = 0; mode < 18; mode++) {
    for (int rep = 0; rep < 2; rep++) {
      cudaEventRecord(a);
      switch (mode) {
        case 0: k<0><<<blocks, 256>>>(tex, tex4, tex2, gv, g, out, iters); break;
        case 1: k<1><<<blocks, 256>>>(tex, tex4, tex2, gv, g, out, iters); break;
        case 2: k<2><<<blocks, 256>>>(tex, tex4, tex2, gv, g, out, iters); break;
        case 3: k<3><<<blocks, 256>>>(tex, tex4, tex2, gv, g, out, iters); break;
        case 4: k<4><<<blocks, 256>>>(tex, tex4, tex2, gv, g, out, iters); break;
        case 5: k<5><<<blocks, 256>>>(tex, tex4, tex2, gv, g, out, iters); break;
        case 6: k<6><<<blocks, 256>>>(tex, tex4, tex2, gv, g, out, iters); break;
        case 7: k<7><<<blocks, 256>>>(tex, tex4, tex2, gv, g, out, iters); break;
        case 8: k<8><<<blocks, 256>>>(tex, tex4, tex2, gv, g, out, iters); break;
        case 9: k<9><<<blocks, 256>>>(tex, tex4, tex2, gv, g, out, iters); break;
        case 10: k<10><<<blocks, 256>>>(tex, tex4, tex2, gv, g, out, iters); break;
        case 11: k<11><<<blocks, 256>>>(tex, tex4, tex2, gv, g, out, iters); break;
        case 12: k<12><<<blocks, 256>>>(tex, tex4, tex2, gv, g, out, iters); break;
        case 13: k<13><<<blocks, 256>>>(tex, tex4, tex2, gv, g, out, iters); break;
        case 14: k<14><<<blocks, 256>>>(tex, tex4, tex2, gv, g, out, iters); break;
        case 15: k<15><<<blocks, 256>>>(tex, tex4, tex2, gv, g, out, iters); break;
        case 16: k<16><<<blocks, 256>>>(tex, tex4, tex2, gv, g, out, iters); break;
        case 17: k<17><<<blocks, 256>>>(tex, tex4, tex2, gv, g, out, iters); break;
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double insts = (double)blocks * 256 * UNR * iters;  // thread-level fetch instrs
      if (rep)
        printf("%-22s %8.3f ms  %6.2f thread-fetch/clk/SM  (%5.2f warp-inst/clk/SM) err=%s\n",
               names[mode], ms, insts / (ms * 1e-3) / sms / (ghz * 1e9),
               insts / 32 / (ms * 1e-3) / sms / (ghz * 1e9),
               cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
