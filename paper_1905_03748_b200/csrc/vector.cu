// vector.cu -- loop algebra of cgls / os_sart (K11, algorithms.py:204-304)
// on device-resident fp32 vectors with fp64 reductions.  Reductions are
// deterministic: a fixed grid of 4 x SMs CTAs writes fp64 partials that
// one CTA sums in a fixed order.  Scalars (alpha = gamma/delta, beta) stay
// on the device so the loops never round-trip through the host for them.
#include "common.cuh"

namespace cs {

int reduce_into(const double* partial, size_t n, double* out, cudaStream_t s);

__global__ void __launch_bounds__(256)
    dot_kernel(const float* __restrict__ a, const float* __restrict__ b,
               int64_t n, double* __restrict__ partial) {
  __shared__ double sh[8];
  double v = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // 4 independent accumulators for MLP
  double v1 = 0.0, v2 = 0.0, v3 = 0.0;
  for (; i + 3 * stride < n; i += 4 * stride) {
    v += (double)a[i] * b[i];
    v1 += (double)a[i + stride] * b[i + stride];
    v2 += (double)a[i + 2 * stride] * b[i + 2 * stride];
    v3 += (double)a[i + 3 * stride] * b[i + 3 * stride];
  }
  for (; i < n; i += stride) v += (double)a[i] * b[i];
  v = (v + v1) + (v2 + v3);
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < 8; w++) s += sh[w];
    partial[blockIdx.x] = s;
  }
}

__device__ __forceinline__ bool ratio(const double* num, const double* den,
                                      double& r) {
  const double d = *den;
  if (d < 1e-30) return false;  // CG_BREAKDOWN, algorithms.py:50
  r = *num / d;
  return true;
}

__global__ void axpy_ratio_kernel(float* __restrict__ y,
                                  const float* __restrict__ x, int64_t n,
                                  const double* num, const double* den,
                                  double sign) {
  double r;
  if (!ratio(num, den, r)) return;
  const float a = (float)(sign * r);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += stride)
    y[i] = fmaf(a, x[i], y[i]);
}

__global__ void xpay_ratio_kernel(float* __restrict__ p,
                                  const float* __restrict__ s, int64_t n,
                                  const double* num, const double* den) {
  double r;
  if (!ratio(num, den, r)) r = 0.0;
  const float b = (float)r;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += stride)
    p[i] = fmaf(b, p[i], s[i]);
}

__global__ void guarded_inverse_kernel(const float* __restrict__ a,
                                       float* __restrict__ out, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += stride) {
    const float v = a[i];
    out[i] = ((double)v >= 1e-8) ? (float)(1.0 / (double)v) : 0.f;
  }
}

__global__ void sart_update_kernel(float* __restrict__ x,
                                   float* __restrict__ upd,
                                   const float* __restrict__ v, float lam,
                                   int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += stride) {
    x[i] = fmaf(lam * v[i], upd[i], x[i]);
    upd[i] = 0.f;
  }
}

__global__ void weighted_residual_kernel(float* __restrict__ r,
                                         const float* __restrict__ b,
                                         const float* __restrict__ w,
                                         int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += stride) {
    const float d = b[i] - r[i];
    r[i] = w ? w[i] * d : d;
  }
}

// Sum of n_src equally strided slices in slice order (deterministic), and
// optionally the OS-SART residual of the sum: out = w o (b - sum).  The
// owner-side half of the sharded forward's peer exchange (sharded.py): the
// slices are the partial projections the other ranks stored into this
// rank's inbox.  float4 lanes when every base and the stride are 16-byte
// aligned (sheets of n_u n_v floats with n_u n_v % 4 == 0), else scalar.
template <typename T>
__device__ __forceinline__ T ld_slice(const float* p, int64_t i) {
  return reinterpret_cast<const T*>(p)[i];
}

__device__ __forceinline__ float4 f4_add(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}

__device__ __forceinline__ float4 f4_res(float4 b, float4 s) {
  return make_float4(b.x - s.x, b.y - s.y, b.z - s.z, b.w - s.w);
}

__device__ __forceinline__ float4 f4_mul(float4 a, float4 b) {
  return make_float4(a.x * b.x, a.y * b.y, a.z * b.z, a.w * b.w);
}

__global__ void __launch_bounds__(256)
    sum_slices4_kernel(const float* __restrict__ src, int n_src,
                       int64_t stride4, int64_t n4,
                       const float* __restrict__ b,
                       const float* __restrict__ w, float* __restrict__ out) {
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += step) {
    float4 s = ld_slice<float4>(src, i);
    for (int k = 1; k < n_src; k++)
      s = f4_add(s, ld_slice<float4>(src, k * stride4 + i));
    if (b) {
      s = f4_res(ld_slice<float4>(b, i), s);
      if (w) s = f4_mul(ld_slice<float4>(w, i), s);
    }
    reinterpret_cast<float4*>(out)[i] = s;
  }
}

__global__ void sum_slices_kernel(const float* __restrict__ src, int n_src,
                                  int64_t stride, int64_t n,
                                  const float* __restrict__ b,
                                  const float* __restrict__ w,
                                  float* __restrict__ out) {
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += step) {
    float s = src[i];
    for (int k = 1; k < n_src; k++) s += src[k * stride + i];
    if (b) {
      s = b[i] - s;
      if (w) s = w[i] * s;
    }
    out[i] = s;
  }
}

__global__ void fill_kernel(float* __restrict__ x, float value, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += stride)
    x[i] = value;
}

static inline int grid_for(int64_t n) {
  const int64_t want = (n + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 8;
  return (int)(want < cap ? (want < 1 ? 1 : want) : cap);
}

}  // namespace cs

using namespace cs;

extern "C" {

int cs_dot(const float* a, const float* b, int64_t n, double* out_sum,
           cs_stream_t stream) {
  CS_REQUIRE(n >= 0, CS_ERR_ARG, "negative length");
  cudaStream_t s = (cudaStream_t)stream;
  const int nb = num_sms() * 4;
  double* part = nullptr;
  CS_CHECK_CUDA(cudaMallocAsync((void**)&part, nb * sizeof(double), s));
  dot_kernel<<<nb, 256, 0, s>>>(a, b, n, part);
  CS_COUNT_LAUNCH();
  CS_CHECK_CUDA(cudaGetLastError());
  int rc = reduce_into(part, nb, out_sum, s);
  cudaFreeAsync(part, s);
  return rc;
}

int cs_axpy_ratio(float* y, const float* x, int64_t n, const double* num,
                  const double* den, double sign, cs_stream_t stream) {
  if (n <= 0) return CS_OK;
  axpy_ratio_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(
      y, x, n, num, den, sign);
  CS_COUNT_LAUNCH();
  CS_CHECK_CUDA(cudaGetLastError());
  return CS_OK;
}

int cs_xpay_ratio(float* p, const float* s, int64_t n, const double* num,
                  const double* den, cs_stream_t stream) {
  if (n <= 0) return CS_OK;
  xpay_ratio_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(p, s, n,
                                                                   num, den);
  CS_COUNT_LAUNCH();
  CS_CHECK_CUDA(cudaGetLastError());
  return CS_OK;
}

int cs_guarded_inverse(const float* a, float* out, int64_t n,
                       cs_stream_t stream) {
  if (n <= 0) return CS_OK;
  guarded_inverse_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(
      a, out, n);
  CS_COUNT_LAUNCH();
  CS_CHECK_CUDA(cudaGetLastError());
  return CS_OK;
}

int cs_sart_update(float* x, float* upd, const float* v, double lam,
                   int64_t n, cs_stream_t stream) {
  if (n <= 0) return CS_OK;
  sart_update_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(
      x, upd, v, (float)lam, n);
  CS_COUNT_LAUNCH();
  CS_CHECK_CUDA(cudaGetLastError());
  return CS_OK;
}

int cs_weighted_residual(float* r, const float* b, const float* w, int64_t n,
                         cs_stream_t stream) {
  if (n <= 0) return CS_OK;
  weighted_residual_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(
      r, b, w, n);
  CS_COUNT_LAUNCH();
  CS_CHECK_CUDA(cudaGetLastError());
  return CS_OK;
}

int cs_sum_slices(const float* src, int n_src, int64_t stride, int64_t n,
                  const float* b, const float* w, float* out,
                  cs_stream_t stream) {
  if (n <= 0) return CS_OK;
  CS_REQUIRE(n_src >= 1 && src && out && (b || !w), CS_ERR_ARG,
             "sum_slices: need n_src >= 1, src, out (and b with w)");
  auto al = [](const void* p) {
    return ((uintptr_t)p & 15) == 0;
  };
  const cudaStream_t s = (cudaStream_t)stream;
  if (n % 4 == 0 && stride % 4 == 0 && al(src) && al(out) &&
      (!b || al(b)) && (!w || al(w))) {
    sum_slices4_kernel<<<grid_for(n / 4), 256, 0, s>>>(src, n_src, stride / 4,
                                                       n / 4, b, w, out);
  } else {
    sum_slices_kernel<<<grid_for(n), 256, 0, s>>>(src, n_src, stride, n, b, w,
                                                  out);
  }
  CS_COUNT_LAUNCH();
  CS_CHECK_CUDA(cudaGetLastError());
  return CS_OK;
}

int cs_fill(float* x, float value, int64_t n, cs_stream_t stream) {
  if (n <= 0) return CS_OK;
  fill_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(x, value, n);
  CS_COUNT_LAUNCH();
  CS_CHECK_CUDA(cudaGetLastError());
  return CS_OK;
}

}  // extern "C"
