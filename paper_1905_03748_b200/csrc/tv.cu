// tv.cu -- TV regularisation stencils (K6-K10) for sm_100a.
//
// Restates regularization.py:88-182 on a window u[nzw][ny][nx] whose first
// and last planes are faces: forward differences with a zero last plane
// (_grad, :88-95) and the one-sided negative adjoint (_div, :98-110).  Both
// reduce to one rule: p = 0 outside the window and on the face where the
// forward difference is undefined, so -div p at voxel i is
//   -(pz(i) - pz(i - ez) + py(i) - py(i - ey) + px(i) - px(i - ex)).
// GD needs the global norm of g before the update, so it is two passes
// (12 B / voxel-iteration): pass 1 reduces Σg² over the core
// planes in fp64 (deterministic two-stage reduction), pass 2 recomputes g
// and writes u - step g / ||g|| to a second buffer.  ROF is one fused pass
// per iteration (28 B / voxel-iteration).  Stencil neighbours come through
// L1 (__ldg); one thread per voxel, CTA = 32 x 8 (x, y).
#include "common.cuh"

namespace cs {

constexpr double TV_EPS = 1e-8;       // regularization.py:39
constexpr double ROF_TAU = 1.0 / 12;  // regularization.py:40

struct Win {
  int nx, ny, nz;
  __device__ __forceinline__ size_t at(int x, int y, int z) const {
    return ((size_t)z * ny + y) * nx + x;
  }
};

__device__ __forceinline__ float3 fwd_grad(const float* __restrict__ u,
                                           const Win& W, int x, int y,
                                           int z) {
  const float c = __ldg(u + W.at(x, y, z));
  float3 g;
  g.x = (x < W.nx - 1) ? __ldg(u + W.at(x + 1, y, z)) - c : 0.f;
  g.y = (y < W.ny - 1) ? __ldg(u + W.at(x, y + 1, z)) - c : 0.f;
  g.z = (z < W.nz - 1) ? __ldg(u + W.at(x, y, z + 1)) - c : 0.f;
  return g;
}

// normalised gradient p = ∇u / sqrt(|∇u|² + eps), zero outside the window
__device__ __forceinline__ float3 norm_grad(const float* __restrict__ u,
                                            const Win& W, int x, int y,
                                            int z) {
  if (x < 0 || y < 0 || z < 0) return make_float3(0.f, 0.f, 0.f);
  const float3 g = fwd_grad(u, W, x, y, z);
  const float inv =
      rsqrtf(g.x * g.x + g.y * g.y + g.z * g.z + (float)TV_EPS);
  return make_float3(g.x * inv, g.y * inv, g.z * inv);
}

// TV sub-gradient g = -div(∇u/|∇u|_eps), regularization.py:127-130
__device__ __forceinline__ float tv_subgrad(const float* __restrict__ u,
                                            const Win& W, int x, int y,
                                            int z) {
  const float3 p = norm_grad(u, W, x, y, z);
  const float pxm = norm_grad(u, W, x - 1, y, z).x;
  const float pym = norm_grad(u, W, x, y - 1, z).y;
  const float pzm = norm_grad(u, W, x, y, z - 1).z;
  return -((p.z - pzm) + (p.y - pym) + (p.x - pxm));
}

__device__ __forceinline__ double block_reduce(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int tid = threadIdx.x + blockDim.x * threadIdx.y;
  const int nw = (blockDim.x * blockDim.y) >> 5;
  if ((tid & 31) == 0) sh[tid >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (tid == 0)
    for (int i = 0; i < nw; i++) s += sh[i];
  return s;  // valid in thread 0
}

__global__ void __launch_bounds__(256)
    tv_sumsq_kernel(const float* __restrict__ u, Win W, int core_lo,
                    int core_hi, double* __restrict__ partial) {
  __shared__ double sh[8];
  const int x = blockIdx.x * 32 + threadIdx.x;
  const int y = blockIdx.y * 8 + threadIdx.y;
  const int z = core_lo + blockIdx.z;
  double v = 0.0;
  if (x < W.nx && y < W.ny && z < core_hi) {
    const float g = tv_subgrad(u, W, x, y, z);
    v = (double)g * (double)g;
  }
  const double s = block_reduce(v, sh);
  if (threadIdx.x == 0 && threadIdx.y == 0)
    partial[((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x +
            blockIdx.x] = s;
}

__global__ void __launch_bounds__(256)
    tv_step_kernel(const float* __restrict__ u, float* __restrict__ uo, Win W,
                   double step, const double* __restrict__ sumsq,
                   double scale) {
  const int x = blockIdx.x * 32 + threadIdx.x;
  const int y = blockIdx.y * 8 + threadIdx.y;
  const int z = blockIdx.z;
  if (x >= W.nx || y >= W.ny) return;
  const double norm = sqrt(*sumsq) * scale;
  const size_t i = W.at(x, y, z);
  if (norm < 1e-30) {  // regularization.py:148-149 / :258
    uo[i] = u[i];
    return;
  }
  const float g = tv_subgrad(u, W, x, y, z);
  uo[i] = (float)((double)u[i] - step * (double)g / norm);
}

__global__ void __launch_bounds__(256)
    tv_norm_kernel(const float* __restrict__ u, Win W,
                   double* __restrict__ partial) {
  __shared__ double sh[8];
  const int x = blockIdx.x * 32 + threadIdx.x;
  const int y = blockIdx.y * 8 + threadIdx.y;
  const int z = blockIdx.z;
  double v = 0.0;
  if (x < W.nx && y < W.ny) {
    const float3 g = fwd_grad(u, W, x, y, z);
    v = sqrt((double)g.x * g.x + (double)g.y * g.y + (double)g.z * g.z);
  }
  const double s = block_reduce(v, sh);
  if (threadIdx.x == 0 && threadIdx.y == 0)
    partial[((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x +
            blockIdx.x] = s;
}

// ---- ROF (regularization.py:154-182) ------------------------------------

// div p at (x, y, z) with p = 0 outside the window / on the undefined face
__device__ __forceinline__ float divp(const float* __restrict__ p,
                                      const Win& W, size_t vol, int x, int y,
                                      int z) {
  const float* pz = p;
  const float* py = p + vol;
  const float* px = p + 2 * vol;
  const size_t i = W.at(x, y, z);
  float d = 0.f;
  d += (z < W.nz - 1 ? __ldg(pz + i) : 0.f) -
       (z > 0 ? __ldg(pz + i - (size_t)W.nx * W.ny) : 0.f);
  d += (y < W.ny - 1 ? __ldg(py + i) : 0.f) - (y > 0 ? __ldg(py + i - W.nx) : 0.f);
  d += (x < W.nx - 1 ? __ldg(px + i) : 0.f) - (x > 0 ? __ldg(px + i - 1) : 0.f);
  return d;
}

__global__ void __launch_bounds__(256)
    rof_iter_kernel(const float* __restrict__ f, const float* __restrict__ pin,
                    float* __restrict__ pout, Win W, float lam,
                    float tau_over_lam) {
  const int x = blockIdx.x * 32 + threadIdx.x;
  const int y = blockIdx.y * 8 + threadIdx.y;
  const int z = blockIdx.z;
  if (x >= W.nx || y >= W.ny) return;
  const size_t vol = (size_t)W.nx * W.ny * W.nz;
  const size_t i = W.at(x, y, z);
  // u = f + lam div p at i and at the +1 neighbours (forward gradient)
  const float uc = __ldg(f + i) + lam * divp(pin, W, vol, x, y, z);
  float gz = 0.f, gy = 0.f, gx = 0.f;
  if (z < W.nz - 1)
    gz = (__ldg(f + W.at(x, y, z + 1)) + lam * divp(pin, W, vol, x, y, z + 1)) - uc;
  if (y < W.ny - 1)
    gy = (__ldg(f + W.at(x, y + 1, z)) + lam * divp(pin, W, vol, x, y + 1, z)) - uc;
  if (x < W.nx - 1)
    gx = (__ldg(f + W.at(x + 1, y, z)) + lam * divp(pin, W, vol, x + 1, y, z)) - uc;
  float qz = __ldg(pin + i) + tau_over_lam * gz;
  float qy = __ldg(pin + vol + i) + tau_over_lam * gy;
  float qx = __ldg(pin + 2 * vol + i) + tau_over_lam * gx;
  const float mag = fmaxf(sqrtf(qz * qz + qy * qy + qx * qx), 1.f);
  pout[i] = qz / mag;
  pout[vol + i] = qy / mag;
  pout[2 * vol + i] = qx / mag;
}

__global__ void __launch_bounds__(256)
    rof_finish_kernel(const float* __restrict__ f, const float* __restrict__ p,
                      float* __restrict__ u, Win W, float lam) {
  const int x = blockIdx.x * 32 + threadIdx.x;
  const int y = blockIdx.y * 8 + threadIdx.y;
  const int z = blockIdx.z;
  if (x >= W.nx || y >= W.ny) return;
  const size_t vol = (size_t)W.nx * W.ny * W.nz;
  const size_t i = W.at(x, y, z);
  u[i] = f[i] + lam * divp(p, W, vol, x, y, z);
}

// Deterministic single-CTA reduction of the block partials.
__global__ void __launch_bounds__(1024)
    reduce_partials_kernel(const double* __restrict__ partial, size_t n,
                           double* __restrict__ out) {
  __shared__ double sh[32];
  double v = 0.0;
  for (size_t i = threadIdx.x; i < n; i += blockDim.x) v += partial[i];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); i++) s += sh[i];
    *out = s;
  }
}

int reduce_into(const double* partial, size_t n, double* out,
                cudaStream_t s) {
  reduce_partials_kernel<<<1, 1024, 0, s>>>(partial, n, out);
  CS_CHECK_CUDA(cudaGetLastError());
  return CS_OK;
}

static int check_win(int nx, int ny, int nzw) {
  CS_REQUIRE(nx >= 2 && ny >= 2 && nzw >= 2, CS_ERR_ARG,
             "TV needs at least 2 voxels per axis (got %d x %d x %d)", nx, ny,
             nzw);
  CS_REQUIRE(nzw <= 65535, CS_ERR_ARG, "window too tall (%d planes)", nzw);
  return CS_OK;
}

}  // namespace cs

using namespace cs;

extern "C" {

int cs_tv_grad_sumsq(const float* u, int nx, int ny, int nzw, int core_lo,
                     int core_hi, double* out_sum, cs_stream_t stream) {
  int rc = check_win(nx, ny, nzw);
  if (rc) return rc;
  CS_REQUIRE(0 <= core_lo && core_lo < core_hi && core_hi <= nzw, CS_ERR_ARG,
             "bad core [%d, %d) in window of %d", core_lo, core_hi, nzw);
  cudaStream_t s = (cudaStream_t)stream;
  const dim3 grid((nx + 31) / 32, (ny + 7) / 8, core_hi - core_lo);
  const size_t nb = (size_t)grid.x * grid.y * grid.z;
  double* part = nullptr;
  CS_CHECK_CUDA(cudaMallocAsync((void**)&part, nb * sizeof(double), s));
  tv_sumsq_kernel<<<grid, dim3(32, 8), 0, s>>>(u, Win{nx, ny, nzw}, core_lo,
                                               core_hi, part);
  CS_CHECK_CUDA(cudaGetLastError());
  rc = reduce_into(part, nb, out_sum, s);
  cudaFreeAsync(part, s);
  return rc;
}

int cs_tv_step(const float* u, float* u_out, int nx, int ny, int nzw,
               double step, const double* norm_sumsq_dev, double scale,
               cs_stream_t stream) {
  int rc = check_win(nx, ny, nzw);
  if (rc) return rc;
  CS_REQUIRE(u != u_out, CS_ERR_ARG, "cs_tv_step: u and u_out must differ");
  const dim3 grid((nx + 31) / 32, (ny + 7) / 8, nzw);
  tv_step_kernel<<<grid, dim3(32, 8), 0, (cudaStream_t)stream>>>(
      u, u_out, Win{nx, ny, nzw}, step, norm_sumsq_dev, scale);
  CS_CHECK_CUDA(cudaGetLastError());
  return CS_OK;
}

int cs_rof_iter(const float* f, const float* p_in, float* p_out, int nx,
                int ny, int nzw, double lam, cs_stream_t stream) {
  int rc = check_win(nx, ny, nzw);
  if (rc) return rc;
  CS_REQUIRE(p_in != p_out, CS_ERR_ARG, "cs_rof_iter: p_in aliases p_out");
  CS_REQUIRE(lam > 0, CS_ERR_ARG, "lambda must be positive");
  const dim3 grid((nx + 31) / 32, (ny + 7) / 8, nzw);
  rof_iter_kernel<<<grid, dim3(32, 8), 0, (cudaStream_t)stream>>>(
      f, p_in, p_out, Win{nx, ny, nzw}, (float)lam, (float)(ROF_TAU / lam));
  CS_CHECK_CUDA(cudaGetLastError());
  return CS_OK;
}

int cs_rof_finish(const float* f, const float* p, float* u, int nx, int ny,
                  int nzw, double lam, cs_stream_t stream) {
  int rc = check_win(nx, ny, nzw);
  if (rc) return rc;
  const dim3 grid((nx + 31) / 32, (ny + 7) / 8, nzw);
  rof_finish_kernel<<<grid, dim3(32, 8), 0, (cudaStream_t)stream>>>(
      f, p, u, Win{nx, ny, nzw}, (float)lam);
  CS_CHECK_CUDA(cudaGetLastError());
  return CS_OK;
}

int cs_tv_norm(const float* u, int nx, int ny, int nzw, double* out_sum,
               cs_stream_t stream) {
  int rc = check_win(nx, ny, nzw);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  const dim3 grid((nx + 31) / 32, (ny + 7) / 8, nzw);
  const size_t nb = (size_t)grid.x * grid.y * grid.z;
  double* part = nullptr;
  CS_CHECK_CUDA(cudaMallocAsync((void**)&part, nb * sizeof(double), s));
  tv_norm_kernel<<<grid, dim3(32, 8), 0, s>>>(u, Win{nx, ny, nzw}, part);
  CS_CHECK_CUDA(cudaGetLastError());
  rc = reduce_into(part, nb, out_sum, s);
  cudaFreeAsync(part, s);
  return rc;
}

}  // extern "C"
