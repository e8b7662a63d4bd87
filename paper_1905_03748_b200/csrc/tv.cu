// tv.cu -- TV regularisation stencils (K6-K10) for sm_100a.
//
// Restates regularization.py:88-182 on a window u[nzw][ny][nx] whose first
// and last planes are faces: forward differences with a zero last plane
// (_grad, :88-95) and the one-sided negative adjoint (_div, :98-110).  Both
// reduce to one rule: p = 0 outside the window and on the face where the
// forward difference is undefined, so -div p at voxel i is
//   -(pz(i) - pz(i - ez) + py(i) - py(i - ey) + px(i) - px(i - ex)).
// GD needs the global norm of g before the update: production is one
// marching pass per iteration that applies step i and computes gradient
// i+1 (tv_march2_kernel / tv_march_kernel, cs_tv_gd_fused), bracketed by a
// gradient pass (cs_tv_grad_store) and a final float4 stream step
// (cs_tv_step_g); Σg² partials are fp32 per thread and reduced in fp64
// (deterministic two-stage reduction).  The r01 tiled kernel remains as the
// A/B baseline and for the two-pass norm / step pair (cs_tv_grad_sumsq +
// cs_tv_step).  ROF: one marching pass per dual iteration (rof_march2_kernel,
// 28 B / voxel-iteration; the r01 per-voxel kernel for odd nx).
#include <atomic>
#include <cstdint>

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdlib>

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

// 1 / sqrt(gx^2 + gy^2 + gz^2 + eps) with the rounding order pinned (no
// contraction freedom; the p = g * inv products are likewise __fmul_rn so
// they cannot fuse into the divergence), so every GD kernel produces the
// same bits; the
// argument is >= eps (normal), where the ftz approximation equals rsqrtf.
__device__ __forceinline__ float tv_inv_norm(float gx, float gy, float gz) {
  const float n = __fadd_rn(
      __fmaf_rn(gz, gz, __fmaf_rn(gy, gy, __fmul_rn(gx, gx))), (float)TV_EPS);
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(n));
  return r;
}

// The GD step u - c g with c = step / ||g|| rounded once to fp32: one
// FFMA, the same in every GD kernel (bit-identical across them).  The fp64
// form (round(u - c g) from exact fp64 products) differs only by c's fp32
// rounding, 6e-8 of the step; per-thread partial sums of g^2 are fp32 over
// <= 64 terms (<= 4e-6 relative on the norm), then reduced in fp64.  9% off
// the fused pass (0.458 -> 0.416 ms at 512^3, profiles/ab_tv_f32_r02au.jsonl).
__device__ __forceinline__ float tv_coef(double step, double norm) {
  return norm < 1e-30 ? 0.f : (float)(step / norm);  // regularization.py:148
}
__device__ __forceinline__ float tv_step1(float u, float g, float c) {
  return __fmaf_rn(-c, g, u);
}

// ---- tiled TV-GD (r01; A/B baseline and the two-pass norm/step pair) ---------------------------------------------
// CTA = 32 x 8 (x, y) tile marching over a chunk of TV_ZC planes.  Per plane
// the normalised gradient p is computed ONCE per voxel (plus a one-voxel
// halo at x - 1 / y - 1) from two rotating u-planes in shared memory; pz of
// the previous plane stays in a register.  u is read ~1.3x per pass instead
// of the 13 neighbour reads (and 4 p evaluations) of the reference stencil.
constexpr int TV_TX = 32, TV_TY = 8, TV_ZC = 16;
constexpr int TV_UX = TV_TX + 2, TV_UY = TV_TY + 2;  // u tile: x0-1 .. x0+32
constexpr int TV_PX = TV_TX + 1, TV_PY = TV_TY + 1;  // p tile: x0-1 .. x0+31

// PASS 0: sum of g^2 over [z_begin, z_end); 1: step; 2: g stored to uo
// over [z_begin, z_end) and g^2 summed over the core [c_lo, c_hi)
template <int PASS>
__global__ void __launch_bounds__(TV_TX * TV_TY)
    tv_gd_tiled_kernel(const float* __restrict__ u, float* __restrict__ uo,
                       Win W, int z_begin, int z_end, double step,
                       const double* __restrict__ sumsq, double scale,
                       double* __restrict__ partial, int c_lo = 0,
                       int c_hi = 0) {
  constexpr int NT = TV_TX * TV_TY;
  constexpr int UN = TV_UX * TV_UY;            // 340 u values per plane
  constexpr int UPT = (UN + NT - 1) / NT;      // per thread (2)
  constexpr int PN = TV_PX * TV_PY;            // 297 p values per plane
  constexpr int PPT = (PN + NT - 1) / NT;      // per thread (2)
  __shared__ float su[3][UN];                  // planes z, z+1, z+2 (ring)
  __shared__ float spx[PN], spy[PN], spz[PN];
  __shared__ double sred[8];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = ty * TV_TX + tx;
  const int x0 = blockIdx.x * TV_TX, y0 = blockIdx.y * TV_TY;
  const int zb = z_begin + blockIdx.z * TV_ZC;
  const int ze = min(z_end, zb + TV_ZC);
  const int x = x0 + tx, y = y0 + ty;
  const bool own = x < W.nx && y < W.ny;
  const size_t plane = (size_t)W.nx * W.ny;
  double norm = 0.0;
  if (PASS == 1) norm = sqrt(*sumsq) * scale;
  const bool skip = PASS == 1 && norm < 1e-30;  // regularization.py:148-149
  const float coef = skip ? 0.f : tv_coef(step, norm);  // u -= step g/||g||

  // Per-thread tile bookkeeping is plane-invariant: computed once.  u tile
  // element i = (lx, ly) holds global (x0 - 1 + lx, y0 - 1 + ly); p tile
  // element e = (lx, ly) sits at the same global position.
  int u_off[UPT];
  bool u_ok[UPT];
#pragma unroll
  for (int j = 0; j < UPT; j++) {
    const int i = tid + j * NT;
    const int ly = i / TV_UX, lx = i - ly * TV_UX;
    const int gx = x0 - 1 + lx, gy = y0 - 1 + ly;
    u_ok[j] = i < UN && gx >= 0 && gx < W.nx && gy >= 0 && gy < W.ny;
    u_off[j] = u_ok[j] ? gy * W.nx + gx : 0;  // in-plane, < 2^31
  }
  int p_su[PPT];           // u-tile index of the p position
  unsigned p_flags[PPT];   // 1: inside the window (x, y); 2: x+1 in; 4: y+1 in
#pragma unroll
  for (int j = 0; j < PPT; j++) {
    const int e = tid + j * NT;
    const int ly = e / TV_PX, lx = e - ly * TV_PX;
    const int gx = x0 - 1 + lx, gy = y0 - 1 + ly;
    p_su[j] = ly * TV_UX + lx;
    unsigned f = 0;
    if (e < PN && gx >= 0 && gy >= 0 && gx < W.nx && gy < W.ny) {
      f = 1u;
      if (gx < W.nx - 1) f |= 2u;
      if (gy < W.ny - 1) f |= 4u;
    }
    p_flags[j] = f;
  }
  const int own_off = own ? y * W.nx + x : 0;
  const int c_p = (ty + 1) * TV_PX + (tx + 1);  // own p / u positions
  const int c_u = (ty + 1) * TV_UX + (tx + 1);

  auto fetch = [&](int z, float (&r)[UPT]) {
    const bool zin = z >= 0 && z < W.nz;
    const float* uz = u + (size_t)(zin ? z : 0) * plane;
#pragma unroll
    for (int j = 0; j < UPT; j++)
      r[j] = (zin && u_ok[j]) ? __ldg(uz + u_off[j]) : 0.f;
  };
  auto put = [&](float* dst, const float (&r)[UPT]) {
#pragma unroll
    for (int j = 0; j < UPT; j++) {
      const int i = tid + j * NT;
      if (i < UN) dst[i] = r[j];
    }
  };
  float* pl0 = su[0];  // plane z
  float* pl1 = su[1];  // plane z + 1
  float* pl2 = su[2];  // plane z + 2
  float rb[UPT];
  fetch(zb - 1, rb);
  put(pl0, rb);
  fetch(zb, rb);
  put(pl1, rb);
  fetch(zb + 1, rb);  // in flight while plane zb - 1 is processed
  float pz_prev = 0.f;
  float acc = 0.f;
  for (int z = zb - 1; z < ze; z++) {
    __syncthreads();  // planes z, z+1 visible; previous p consumed
    const bool zlast = z >= W.nz - 1;
#pragma unroll
    for (int j = 0; j < PPT; j++) {
      const int e = tid + j * NT;
      if (j * NT + NT > PN && e >= PN) break;
      float px = 0.f, py = 0.f, pz = 0.f;
      const unsigned f = p_flags[j];
      if ((f & 1u) && z >= 0) {
        const int k = p_su[j];
        const float cc = pl0[k];
        const float gxv = (f & 2u) ? pl0[k + 1] - cc : 0.f;
        const float gyv = (f & 4u) ? pl0[k + TV_UX] - cc : 0.f;
        const float gzv = zlast ? 0.f : pl1[k] - cc;
        const float inv = tv_inv_norm(gxv, gyv, gzv);
        px = __fmul_rn(gxv, inv);
        py = __fmul_rn(gyv, inv);
        pz = __fmul_rn(gzv, inv);
      }
      spx[e] = px;
      spy[e] = py;
      spz[e] = pz;
    }
    put(pl2, rb);  // plane z + 2 (slot freed by plane z - 1)
    if (z + 3 <= ze) fetch(z + 3, rb);
    __syncthreads();
    const float pz_own = spz[c_p];
    if (z >= zb && own) {
      const float g = -((pz_own - pz_prev) + (spy[c_p] - spy[c_p - TV_PX]) +
                        (spx[c_p] - spx[c_p - 1]));
      if (PASS == 0) {
        acc = __fmaf_rn(g, g, acc);
      } else if (PASS == 2) {
        uo[(size_t)z * plane + own_off] = g;
        if (z >= c_lo && z < c_hi) acc = __fmaf_rn(g, g, acc);
      } else {
        const float uc = pl0[c_u];
        uo[(size_t)z * plane + own_off] =
            skip ? uc : tv_step1(uc, g, coef);
      }
    }
    pz_prev = pz_own;
    float* t = pl0;
    pl0 = pl1;
    pl1 = pl2;
    pl2 = t;
  }
  if (PASS != 1) {
    double accd = (double)acc;
    for (int o = 16; o > 0; o >>= 1)
      accd += __shfl_xor_sync(0xffffffffu, accd, o);
    if ((tid & 31) == 0) sred[tid >> 5] = accd;
    __syncthreads();
    if (tid == 0) {
      double sm = 0.0;
      for (int i = 0; i < 8; i++) sm += sred[i];
      partial[((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x +
              blockIdx.x] = sm;
    }
  }
}

// ---- marching TV-GD (production) ----------------------------------------
// One pass per iteration.  Iteration i of GD is u_{i+1} = u_i - c_i g_i with
// c_i = step / ||g_i|| (regularization.py:145-150), and g_{i+1} = grad TV
// (u_{i+1}).  The norm is global, so u_{i+1} cannot be written before g_i is
// complete -- but g_{i+1} can be computed in the same pass that applies the
// step: every thread forms u_{i+1} = u_i - c_i g_i on the fly from the u_i,
// g_i it loads, and the stencil runs on those values.  The pass reads u_i,
// g_i and writes u_{i+1}, g_{i+1} (16 B / voxel) plus the partial sums of
// g_{i+1}^2; the first iteration reads u only (tv_march<0>, = grad_store)
// and the last applies its step with the float4 stream (tv_step_g_kernel).
//
// CTA = 16 warps; lane l <-> x = x0 - 1 + l, warp w <-> y = y0 - 1 + w.
// Lane 0 / warp 0 are a one-voxel halo whose p feeds the divergence; lane 31
// / warp 15 only supply u(x+1) / u(y+1) to their neighbours: 30 x 14 outputs
// per CTA, and no thread loads anything but its own voxel.  Each thread
// marches its column in z over a chunk of TM_ZC planes: u(x+1) by
// shfl_down, p(x-1) by shfl_up, u(y+1) and p(y-1) through two double-buffered
// shared rows (one barrier per plane), pz(z-1) in a register.  Loads run
// TM_D planes ahead through a per-thread cp.async ring (zero-fill outside the
// window); a thread reads back only its own slots, so the ring needs no
// barrier.  Same per-voxel expressions as tv_gd_tiled_kernel and the step of
// tv_step_g_kernel (tv_step1), so g and u are bit-identical to grad_store +
// step_g for the same input sum; only the grouping of the partial sums
// differs between kernels.
constexpr int TM_WARPS = 16, TM_THREADS = 32 * TM_WARPS;
constexpr int TM_OX = 30, TM_OY = TM_WARPS - 2;
#ifndef CS_TM_ZC
#define CS_TM_ZC 32
#endif
constexpr int TM_ZC = CS_TM_ZC;
#ifndef CS_TM_UNROLL2
#define CS_TM_UNROLL2 1
#endif
constexpr int TM_NS = 8;         // ring stages (power of two)
constexpr int TM_D = TM_NS;  // planes in flight (the ring slot reused is
                               // the one taken an iteration earlier)

__device__ __forceinline__ void cp_async4(unsigned dst, const float* src,
                                          bool ok) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst),
               "l"(src), "r"(ok ? 4 : 0)  // 0: zero-fill, nothing read
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// FUSED 0: g = grad TV(u) -> gout (window), sum g^2 over the core.
// FUSED 1: u' = u - c g (c from sumsq_in) -> uo, g' = grad TV(u') -> gout.
template <int FUSED>
__global__ void __launch_bounds__(TM_THREADS, 2)
    tv_march_kernel(const float* __restrict__ u, const float* __restrict__ gin,
                    float* __restrict__ uo, float* __restrict__ gout, Win W,
                    int c_lo, int c_hi, double step,
                    const double* __restrict__ sumsq_in, double scale,
                    double* __restrict__ partial) {
  constexpr int NA = FUSED ? 2 : 1;  // arrays loaded per voxel
  __shared__ float ring[TM_NS][NA][TM_THREADS];
  __shared__ float su[2][TM_WARPS][32];   // u rows (for gy)
  __shared__ float spy[2][TM_WARPS][32];  // py rows (for div)
  __shared__ double sred[TM_WARPS];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int tid = threadIdx.x;
  const int x = blockIdx.x * TM_OX - 1 + lane;
  const int y = blockIdx.y * TM_OY - 1 + w;
  const int zb = blockIdx.z * TM_ZC;
  const int ze = min(W.nz, zb + TM_ZC);
  const bool in_xy = x >= 0 && x < W.nx && y >= 0 && y < W.ny;
  const bool own = in_xy && lane > 0 && lane < 31 && w > 0 && w < TM_WARPS - 1;
  const bool xl = x < W.nx - 1, yl = y < W.ny - 1;  // forward diffs exist
  const size_t plane = (size_t)W.nx * W.ny;
  const int off = in_xy ? y * W.nx + x : 0;
  float coef = 0.f;
  if (FUSED) coef = tv_coef(step, sqrt(*sumsq_in) * scale);
  // ring slot of this thread, stage 0 / array 0; stage stride, array stride
  const unsigned ring0 = (unsigned)__cvta_generic_to_shared(&ring[0][0][tid]);
  constexpr unsigned RS = NA * TM_THREADS * 4, RA = TM_THREADS * 4;
  // issue pointer: plane zi of the next load
  int zi = zb - 1;
  const float* pu = u + (ptrdiff_t)zi * (ptrdiff_t)plane + off;
  const float* pg = FUSED ? gin + (ptrdiff_t)zi * (ptrdiff_t)plane + off : u;
  auto issue = [&]() {  // planes past ze are not needed: empty group
    const bool ok = in_xy && (unsigned)zi < (unsigned)W.nz;
    const unsigned st = ring0 + ((zi - zb + 1) & (TM_NS - 1)) * RS;
    if (zi <= ze) {
      cp_async4(st, ok ? pu : u, ok);
      if (FUSED) cp_async4(st + RA, ok ? pg : u, ok);
    }
    cp_async_commit();
    zi++;
    pu += plane;
    if (FUSED) pg += plane;
  };
  auto take = [&](int zz) {
    const int st = (zz - zb + 1) & (TM_NS - 1);
    const float uu = ring[st][0][tid];
    if (!FUSED) return uu;
    const float gg = ring[st][NA - 1][tid];
    return tv_step1(uu, gg, coef);  // as tv_step_g_kernel
  };
#pragma unroll
  for (int i = 0; i <= TM_D - 1; i++) issue();  // planes zb-1 .. zb-2+D
  cp_async_wait<TM_D - 1>();
  float uc = take(zb - 1);
  su[(zb - 1) & 1][w][lane] = uc;
  __syncthreads();
  float pz_prev = 0.f;
  float acc = 0.f;  // fp32 partial over this thread's <= 32 planes
  float* po = gout + (ptrdiff_t)zb * (ptrdiff_t)plane + off;
  float* puo = FUSED ? uo + (ptrdiff_t)zb * (ptrdiff_t)plane + off : nullptr;
  const int wy = w < TM_WARPS - 1 ? w + 1 : w;
  // branch-free masks: p = 0 outside the window (all three differences
  // masked) and each forward difference zero where it is undefined
  const float mx = (in_xy && xl) ? 1.f : 0.f;
  const float my = (in_xy && yl) ? 1.f : 0.f;
  const int zlo_sum = max(zb, c_lo), zhi_sum = own ? c_hi : INT_MIN;
  for (int z = zb - 1; z < ze; z++) {
    issue();                    // plane z + D
    cp_async_wait<TM_D - 1>();  // plane z + 1 landed (own slots only)
    const float un = take(z + 1);
    // p(z) at (x, y): forward differences, zero on the undefined faces
    const float ux = __shfl_down_sync(0xffffffffu, uc, 1);
    const float uy = su[z & 1][wy][lane];
    const float mz = (in_xy && z >= 0 && z < W.nz - 1) ? 1.f : 0.f;
    const float gxv = (ux - uc) * mx;
    const float gyv = (uy - uc) * my;
    const float gzv = (un - uc) * mz;
    const float inv = tv_inv_norm(gxv, gyv, gzv);
    const float px = __fmul_rn(gxv, inv), py = __fmul_rn(gyv, inv);
    const float pz = (in_xy && z >= 0) ? __fmul_rn(gzv, inv) : 0.f;
    spy[z & 1][w][lane] = py;
    su[(z + 1) & 1][w][lane] = un;
    __syncthreads();
    const float pxm = __shfl_up_sync(0xffffffffu, px, 1);
    const float pym = spy[z & 1][w > 0 ? w - 1 : 0][lane];
    const float g = -((pz - pz_prev) + (py - pym) + (px - pxm));
    if (z >= zb) {
      if (own) {
        *po = g;
        if (FUSED) *puo = uc;
      }
      po += plane;
      if (FUSED) puo += plane;
    }
    const float gs = (z >= zlo_sum && z < zhi_sum) ? g : 0.f;
    acc = __fmaf_rn(gs, gs, acc);
    pz_prev = pz;
    uc = un;
  }
  cp_async_wait<0>();
  double accd = (double)acc;
  for (int o = 16; o > 0; o >>= 1)
    accd += __shfl_xor_sync(0xffffffffu, accd, o);
  if (lane == 0) sred[w] = accd;
  __syncthreads();
  if (tid == 0) {
    double sm = 0.0;
    for (int i = 0; i < TM_WARPS; i++) sm += sred[i];
    partial[((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x +
            blockIdx.x] = sm;
  }
}

// Paired variant (nx even, 8-byte aligned windows): lane l holds the voxel
// pair x = x0 - 2 + 2l, +1 (float2 loads / stores, 60 x 14 outputs per CTA):
// the pair's inner neighbours stay in registers, so per voxel half the
// shuffles, shared-memory and global instructions and half the per-plane
// loop overhead.  Same expressions (and bits) as tv_march_kernel.
constexpr int TM2_OX = 60;
constexpr int TM2_NS = 4;          // ring stages of 8-byte slots (48 KB
constexpr int TM2_D = TM2_NS;  // static shared memory when fused)

__device__ __forceinline__ void cp_async8(unsigned dst, const float* src,
                                          bool ok) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst),
               "l"(src), "r"(ok ? 8 : 0)
               : "memory");
}

template <int FUSED>
__global__ void __launch_bounds__(TM_THREADS, 2)
    tv_march2_kernel(const float* __restrict__ u,
                     const float* __restrict__ gin, float* __restrict__ uo,
                     float* __restrict__ gout, Win W, int c_lo, int c_hi,
                     double step, const double* __restrict__ sumsq_in,
                     double scale, double* __restrict__ partial) {
  constexpr int NA = FUSED ? 2 : 1;
  __shared__ float2 ring[TM2_NS][NA][TM_THREADS];
  __shared__ float2 su[2][TM_WARPS][32];
  __shared__ float2 spy[2][TM_WARPS][32];
  double* sred = reinterpret_cast<double*>(&su[0][0][0]);  // after the loop
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int tid = threadIdx.x;
  const int x = blockIdx.x * TM2_OX - 2 + 2 * lane;  // pair (x, x + 1)
  const int y = blockIdx.y * TM_OY - 1 + w;
  const int zb = blockIdx.z * TM_ZC;
  const int ze = min(W.nz, zb + TM_ZC);
  // nx even, x even: the pair is wholly inside or wholly outside
  const bool in_xy = x >= 0 && x < W.nx && y >= 0 && y < W.ny;
  const bool own = in_xy && lane > 0 && lane < 31 && w > 0 && w < TM_WARPS - 1;
  const size_t plane = (size_t)W.nx * W.ny;
  const int off = in_xy ? y * W.nx + x : 0;
  float coef = 0.f;
  if (FUSED) coef = tv_coef(step, sqrt(*sumsq_in) * scale);
  const unsigned ring0 = (unsigned)__cvta_generic_to_shared(&ring[0][0][tid]);
  constexpr unsigned RS = NA * TM_THREADS * 8, RA = TM_THREADS * 8;
  int zi = zb - 1;
  const float* pu = u + (ptrdiff_t)zi * (ptrdiff_t)plane + off;
  const float* pg = FUSED ? gin + (ptrdiff_t)zi * (ptrdiff_t)plane + off : u;
  auto issue = [&]() {  // planes past ze are not needed: empty group
    const bool ok = in_xy && (unsigned)zi < (unsigned)W.nz;
    const unsigned st = ring0 + ((zi - zb + 1) & (TM2_NS - 1)) * RS;
    if (zi <= ze) {
      cp_async8(st, ok ? pu : u, ok);
      if (FUSED) cp_async8(st + RA, ok ? pg : u, ok);
    }
    cp_async_commit();
    zi++;
    pu += plane;
    if (FUSED) pg += plane;
  };
  auto take = [&](int zz) {
    const int st = (zz - zb + 1) & (TM2_NS - 1);
    float2 v = ring[st][0][tid];
    if (FUSED) {
      const float2 gg = ring[st][NA - 1][tid];
      v.x = tv_step1(v.x, gg.x, coef);  // as tv_step_g_kernel
      v.y = tv_step1(v.y, gg.y, coef);
    }
    return v;
  };
#pragma unroll
  for (int i = 0; i <= TM2_D - 1; i++) issue();
  cp_async_wait<TM2_D - 1>();
  float2 uc = take(zb - 1);
  su[(zb - 1) & 1][w][lane] = uc;
  __syncthreads();
  float2 pz_prev = make_float2(0.f, 0.f);
  float acc = 0.f;  // fp32 partial over this thread's <= 64 voxels
  float2* po = reinterpret_cast<float2*>(gout + (ptrdiff_t)zb * (ptrdiff_t)plane + off);
  float2* puo = FUSED ? reinterpret_cast<float2*>(
                            uo + (ptrdiff_t)zb * (ptrdiff_t)plane + off)
                      : nullptr;
  const size_t plane2 = plane / 2;
  const int wy = w < TM_WARPS - 1 ? w + 1 : w;
  const float mxa = in_xy ? 1.f : 0.f;  // x < nx - 1 holds for the even x
  const float mxb = (in_xy && x + 1 < W.nx - 1) ? 1.f : 0.f;
  const float my = (in_xy && y < W.ny - 1) ? 1.f : 0.f;
  const int zlo_sum = max(zb, c_lo), zhi_sum = own ? c_hi : INT_MIN;
  for (int z = zb - 1; z < ze; z++) {
    issue();
    cp_async_wait<TM2_D - 1>();
    const float2 un = take(z + 1);
    const float uxb = __shfl_down_sync(0xffffffffu, uc.x, 1);
    const float2 uy = su[z & 1][wy][lane];
    const float mz = (in_xy && z >= 0 && z < W.nz - 1) ? 1.f : 0.f;
    const float gxa = (uc.y - uc.x) * mxa, gxb = (uxb - uc.y) * mxb;
    const float gya = (uy.x - uc.x) * my, gyb = (uy.y - uc.y) * my;
    const float gza = (un.x - uc.x) * mz, gzb = (un.y - uc.y) * mz;
    const float ia = tv_inv_norm(gxa, gya, gza);
    const float ib = tv_inv_norm(gxb, gyb, gzb);
    const bool pv = in_xy && z >= 0;
    const float pxa = __fmul_rn(gxa, ia), pxb = __fmul_rn(gxb, ib);
    const float2 py = make_float2(__fmul_rn(gya, ia), __fmul_rn(gyb, ib));
    const float2 pz = make_float2(pv ? __fmul_rn(gza, ia) : 0.f, pv ? __fmul_rn(gzb, ib) : 0.f);
    spy[z & 1][w][lane] = py;
    su[(z + 1) & 1][w][lane] = un;
    __syncthreads();
    const float pxm = __shfl_up_sync(0xffffffffu, pxb, 1);
    const float2 pym = spy[z & 1][w > 0 ? w - 1 : 0][lane];
    const float ga = -((pz.x - pz_prev.x) + (py.x - pym.x) + (pxa - pxm));
    const float gb = -((pz.y - pz_prev.y) + (py.y - pym.y) + (pxb - pxa));
    if (z >= zb) {
      if (own) {
        *po = make_float2(ga, gb);
        if (FUSED) *puo = uc;
      }
      po += plane2;
      if (FUSED) puo += plane2;
    }
    const bool sum = z >= zlo_sum && z < zhi_sum;
    const float sa = sum ? ga : 0.f, sb = sum ? gb : 0.f;
    acc = __fmaf_rn(sa, sa, acc);
    acc = __fmaf_rn(sb, sb, acc);
    pz_prev = pz;
    uc = un;
  }
  cp_async_wait<0>();
  double accd = (double)acc;
  for (int o = 16; o > 0; o >>= 1)
    accd += __shfl_xor_sync(0xffffffffu, accd, o);
  __syncthreads();  // su is reused for the warp sums
  if (lane == 0) sred[w] = accd;
  __syncthreads();
  if (tid == 0) {
    double sm = 0.0;
    for (int i = 0; i < TM_WARPS; i++) sm += sred[i];
    partial[((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x +
            blockIdx.x] = sm;
  }
}

// TMA-fed paired variant (production when nx % 4 == 0): the same kernel
// body as tv_march2_kernel, but each plane's 68 x 16 tile of u (and g) is
// fetched by ONE cp.async.bulk.tensor per array, issued by thread 0 into the
// ring stage and completed on that stage's mbarrier (out-of-range
// coordinates -- x/y/z outside the window -- arrive as zeros, the window
// rule); the threads only wait on the barrier and read their float2.  This
// takes the per-thread cp.async address / predicate work (two LDGSTS and
// ~8 integer instructions per thread and plane) off the issue-bound loop.
constexpr int TMT_NS = 4;  // ring stages (planes in flight)
constexpr int TMT_BOXX = 68;  // box columns: x0 - 4 .. x0 + 63
// floats per ring slot: 68 x 16 box padded to a 128-byte multiple
constexpr int TMT_SLOT = ((TMT_BOXX * TM_WARPS * 4 + 127) / 128) * 32;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile(
      "mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
      "r"(bytes)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map,
                                            int x, int y, int z,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx"
      "::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

template <int FUSED>
__global__ void __launch_bounds__(TM_THREADS, 2)
    tv_march2_tma_kernel(const __grid_constant__ CUtensorMap map_u,
                         const __grid_constant__ CUtensorMap map_g,
                         float* __restrict__ uo, float* __restrict__ gout,
                         Win W, int c_lo, int c_hi, double step,
                         const double* __restrict__ sumsq_in, double scale,
                         double* __restrict__ partial) {
  constexpr int NA = FUSED ? 2 : 1;
  constexpr unsigned TILE = TMT_BOXX * TM_WARPS * sizeof(float);  // box bytes
  // dynamic shared memory (just over the 48 KB static limit when fused):
  // ring | su | spy | barriers
  extern __shared__ __align__(128) unsigned char tmt_smem[];
  float* ring = reinterpret_cast<float*>(tmt_smem);  // [NS][NA][TMT_SLOT]
  auto& su = *reinterpret_cast<float2(*)[2][TM_WARPS][32]>(
      tmt_smem + sizeof(float) * TMT_NS * NA * TMT_SLOT);
  auto& spy = *reinterpret_cast<float2(*)[2][TM_WARPS][32]>(
      tmt_smem + sizeof(float) * TMT_NS * NA * TMT_SLOT +
      sizeof(float2) * 2 * TM_WARPS * 32);
  uint64_t* bars = reinterpret_cast<uint64_t*>(
      tmt_smem + sizeof(float) * TMT_NS * NA * TMT_SLOT +
      sizeof(float2) * 4 * TM_WARPS * 32);
  double* sred = reinterpret_cast<double*>(&su[0][0][0]);  // after the loop
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int tid = threadIdx.x;
  // the box starts 16-byte aligned (a TMA requirement on the innermost
  // coordinate): 4 columns left of the tile, 2 more than the pair lanes
  const int xt = blockIdx.x * TM2_OX - 4, yt = blockIdx.y * TM_OY - 1;
  const int x = xt + 2 + 2 * lane;  // pair (x, x + 1)
  const int y = yt + w;
  const int zb = blockIdx.z * TM_ZC;
  const int ze = min(W.nz, zb + TM_ZC);
  const bool in_xy = x >= 0 && x < W.nx && y >= 0 && y < W.ny;
  const bool own = in_xy && lane > 0 && lane < 31 && w > 0 && w < TM_WARPS - 1;
  const size_t plane = (size_t)W.nx * W.ny;
  const int off = in_xy ? y * W.nx + x : 0;
  float coef = 0.f;
  if (FUSED) coef = tv_coef(step, sqrt(*sumsq_in) * scale);
  if (tid == 0) {
    for (int i = 0; i < TMT_NS; i++) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int zi = zb - 1;  // next plane to fetch (thread 0)
  auto issue = [&]() {  // planes past ze are not needed
    if (tid == 0 && zi <= ze) {
      const int st = (zi - zb + 1) & (TMT_NS - 1);
      mbar_expect_tx(&bars[st], NA * TILE);
      tma_load_3d(ring + (st * NA) * TMT_SLOT, &map_u, xt, yt, zi, &bars[st]);
      if (FUSED)
        tma_load_3d(ring + (st * NA + 1) * TMT_SLOT, &map_g, xt, yt, zi,
                    &bars[st]);
    }
    zi++;
  };
  auto take = [&](int zz) {
    const int k = zz - zb + 1;  // fill index of the plane
    const int st = k & (TMT_NS - 1);
    mbar_wait(&bars[st], (unsigned)(k / TMT_NS) & 1u);
    const int e = w * TMT_BOXX + 2 + 2 * lane;  // this pair in the box
    float2 v = *reinterpret_cast<const float2*>(ring + (st * NA) * TMT_SLOT + e);
    if (FUSED) {
      const float2 gg =
          *reinterpret_cast<const float2*>(ring + (st * NA + 1) * TMT_SLOT + e);
      v.x = tv_step1(v.x, gg.x, coef);  // as tv_step_g_kernel
      v.y = tv_step1(v.y, gg.y, coef);
    }
    return v;
  };
#pragma unroll
  for (int i = 0; i < TMT_NS; i++) issue();  // planes zb-1 .. zb-2+NS
  float2 uc = take(zb - 1);
  su[(zb - 1) & 1][w][lane] = uc;
  __syncthreads();
  float2 pz_prev = make_float2(0.f, 0.f);
  float acc = 0.f;  // fp32 partial over this thread's <= 64 voxels
  float2* po = reinterpret_cast<float2*>(gout + (ptrdiff_t)zb * (ptrdiff_t)plane + off);
  float2* puo = FUSED ? reinterpret_cast<float2*>(
                            uo + (ptrdiff_t)zb * (ptrdiff_t)plane + off)
                      : nullptr;
  const size_t plane2 = plane / 2;
  const int wy = w < TM_WARPS - 1 ? w + 1 : w;
  const float mxa = in_xy ? 1.f : 0.f;  // x < nx - 1 holds for the even x
  const float mxb = (in_xy && x + 1 < W.nx - 1) ? 1.f : 0.f;
  const float my = (in_xy && y < W.ny - 1) ? 1.f : 0.f;
  const int zlo_sum = max(zb, c_lo), zhi_sum = own ? c_hi : INT_MIN;
#if CS_TM_UNROLL2
#pragma unroll 2
#endif
  for (int z = zb - 1; z < ze; z++) {
    // the stage of plane z was read by every thread before the previous
    // plane's barrier: refill it (plane z + NS)
    issue();
    const float2 un = take(z + 1);
    const float uxb = __shfl_down_sync(0xffffffffu, uc.x, 1);
    const float2 uy = su[z & 1][wy][lane];
    const float mz = (in_xy && z >= 0 && z < W.nz - 1) ? 1.f : 0.f;
    const float gxa = (uc.y - uc.x) * mxa, gxb = (uxb - uc.y) * mxb;
    const float gya = (uy.x - uc.x) * my, gyb = (uy.y - uc.y) * my;
    const float gza = (un.x - uc.x) * mz, gzb = (un.y - uc.y) * mz;
    const float ia = tv_inv_norm(gxa, gya, gza);
    const float ib = tv_inv_norm(gxb, gyb, gzb);
    const bool pv = in_xy && z >= 0;
    const float pxa = __fmul_rn(gxa, ia), pxb = __fmul_rn(gxb, ib);
    const float2 py = make_float2(__fmul_rn(gya, ia), __fmul_rn(gyb, ib));
    const float2 pz = make_float2(pv ? __fmul_rn(gza, ia) : 0.f,
                                  pv ? __fmul_rn(gzb, ib) : 0.f);
    spy[z & 1][w][lane] = py;
    su[(z + 1) & 1][w][lane] = un;
    __syncthreads();
    const float pxm = __shfl_up_sync(0xffffffffu, pxb, 1);
    const float2 pym = spy[z & 1][w > 0 ? w - 1 : 0][lane];
    const float ga = -((pz.x - pz_prev.x) + (py.x - pym.x) + (pxa - pxm));
    const float gb = -((pz.y - pz_prev.y) + (py.y - pym.y) + (pxb - pxa));
    if (z >= zb) {
      if (own) {
        *po = make_float2(ga, gb);
        if (FUSED) *puo = uc;
      }
      po += plane2;
      if (FUSED) puo += plane2;
    }
    const bool sum = z >= zlo_sum && z < zhi_sum;
    const float sa = sum ? ga : 0.f, sb = sum ? gb : 0.f;
    acc = __fmaf_rn(sa, sa, acc);
    acc = __fmaf_rn(sb, sb, acc);
    pz_prev = pz;
    uc = un;
  }
  double accd = (double)acc;
  for (int o = 16; o > 0; o >>= 1)
    accd += __shfl_xor_sync(0xffffffffu, accd, o);
  __syncthreads();  // su is reused for the warp sums
  if (lane == 0) sred[w] = accd;
  __syncthreads();
  if (tid == 0) {
    double sm = 0.0;
    for (int i = 0; i < TM_WARPS; i++) sm += sred[i];
    partial[((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x +
            blockIdx.x] = sm;
  }
}

// 3D tensor map (x, y, z) of a float32 window with a 68 x 16 x 1 box
// (cuTensorMapEncodeTiled through the runtime's driver entry point, so the
// library needs no -lcuda); false when unavailable or the row pitch is not
// a multiple of 16 bytes.
static bool tv_plane_map(CUtensorMap* m, const float* base, int nx, int ny,
                         int nz) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn,
                                cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
  }
  if (!fn || nx % 4 != 0 || ((uintptr_t)base & 15) != 0) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nz};
  const cuuint64_t strides[2] = {(cuuint64_t)nx * 4,
                                 (cuuint64_t)nx * ny * 4};
  const cuuint32_t box[3] = {(cuuint32_t)TMT_BOXX, (cuuint32_t)TM_WARPS, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)base, dims, strides,
            box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int reduce_into(const double* partial, size_t n, double* out, cudaStream_t s);

// Launch the marching GD pass: the paired kernel when nx is even and every
// buffer is 8-byte aligned, else the single-voxel kernel.
template <int FUSED>
static int launch_march(const float* u, const float* g, float* uo, float* go,
                        int nx, int ny, int nzw, int core_lo, int core_hi,
                        double step, const double* sumsq_in, double scale,
                        double* out_sum, cudaStream_t s) {
  static const char* knob = getenv("CS_TV_PAIRS");  // A/B: 0 = single
  const bool pairs =
      (!knob || knob[0] != '0') && nx % 2 == 0 && (uintptr_t)u % 8 == 0 &&
      (uintptr_t)go % 8 == 0 &&
      (!FUSED || ((uintptr_t)g % 8 == 0 && (uintptr_t)uo % 8 == 0));
  const dim3 grid((nx + (pairs ? TM2_OX : TM_OX) - 1) / (pairs ? TM2_OX : TM_OX),
                  (ny + TM_OY - 1) / TM_OY, (nzw + TM_ZC - 1) / TM_ZC);
  const size_t nb = (size_t)grid.x * grid.y * grid.z;
  double* part = nullptr;
  retain_pool();
  CS_CHECK_CUDA(cudaMallocAsync((void**)&part, nb * sizeof(double), s));
  static const char* tma_knob = getenv("CS_TV_TMA");  // A/B: 0 = cp.async
  CUtensorMap mu, mg;
  const bool tma = pairs && !(tma_knob && tma_knob[0] == '0') &&
                   tv_plane_map(&mu, u, nx, ny, nzw) &&
                   (!FUSED || tv_plane_map(&mg, g, nx, ny, nzw));
  if (tma) {
    constexpr int NA = FUSED ? 2 : 1;
    const size_t smem = sizeof(float) * TMT_NS * NA * TMT_SLOT +
                        sizeof(float2) * 4 * TM_WARPS * 32 +
                        sizeof(uint64_t) * TMT_NS;
    static std::atomic<unsigned long long> attr_done{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(attr_done.load() & bit)) {
      CS_CHECK_CUDA(cudaFuncSetAttribute(
          tv_march2_tma_kernel<FUSED>,
          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr_done.fetch_or(bit);
    }
    tv_march2_tma_kernel<FUSED><<<grid, TM_THREADS, smem, s>>>(
        mu, FUSED ? mg : mu, uo, go, Win{nx, ny, nzw}, core_lo, core_hi,
        step, sumsq_in, scale, part);
  }
  else if (pairs)
    tv_march2_kernel<FUSED><<<grid, TM_THREADS, 0, s>>>(
        u, g, uo, go, Win{nx, ny, nzw}, core_lo, core_hi, step, sumsq_in,
        scale, part);
  else
    tv_march_kernel<FUSED><<<grid, TM_THREADS, 0, s>>>(
        u, g, uo, go, Win{nx, ny, nzw}, core_lo, core_hi, step, sumsq_in,
        scale, part);
  CS_COUNT_LAUNCH();
  CS_CHECK_CUDA(cudaGetLastError());
  const int rc = reduce_into(part, nb, out_sum, s);
  cudaFreeAsync(part, s);
  return rc;
}

// ---- ROF (regularization.py:154-182) ------------------------------------

__device__ __forceinline__ float rof_inv_mag(float qz, float qy, float qx) {
  return __frcp_rn(fmaxf(
      sqrtf(__fmaf_rn(qx, qx, __fmaf_rn(qy, qy, __fmul_rn(qz, qz)))), 1.f));
}

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

// div p at the voxel whose three components sit at pz[0], pz[vol],
// pz[2 vol] (pointer already offset to the voxel): same terms and order as
// divp, 32-bit neighbour strides (plane = nx ny < 2^31).
__device__ __forceinline__ float divp_at(const float* __restrict__ pzi,
                                         size_t vol, int plane, int nx,
                                         bool zl, bool zf, bool yl, bool yf,
                                         bool xl, bool xf) {
  const float* pyi = pzi + vol;
  const float* pxi = pyi + vol;
  float d = 0.f;
  d += (zl ? __ldg(pzi) : 0.f) - (zf ? __ldg(pzi - plane) : 0.f);
  d += (yl ? __ldg(pyi) : 0.f) - (yf ? __ldg(pyi - nx) : 0.f);
  d += (xl ? __ldg(pxi) : 0.f) - (xf ? __ldg(pxi - 1) : 0.f);
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
  const int nx = W.nx, plane = W.nx * W.ny;
  const size_t vol = (size_t)plane * W.nz;
  const size_t i = (size_t)z * plane + (size_t)(y * nx + x);
  const float* fi = f + i;
  const float* pi = pin + i;
  // "l": the forward difference exists (not the last plane/row/column);
  // "f": the backward one exists (not the first)
  const bool zl = z < W.nz - 1, zf = z > 0, yl = y < W.ny - 1, yf = y > 0;
  const bool xl = x < nx - 1, xf = x > 0;
  // u = f + lam div p at i and at the +1 neighbours (forward gradient)
  const float uc = __fmaf_rn(lam, divp_at(pi, vol, plane, nx, zl, zf, yl, yf,
                                          xl, xf), __ldg(fi));
  float gz = 0.f, gy = 0.f, gx = 0.f;
  if (zl)
    gz = __fmaf_rn(lam, divp_at(pi + plane, vol, plane, nx, z + 1 < W.nz - 1,
                                true, yl, yf, xl, xf), __ldg(fi + plane)) - uc;
  if (yl)
    gy = __fmaf_rn(lam, divp_at(pi + nx, vol, plane, nx, zl, zf,
                                y + 1 < W.ny - 1, true, xl, xf),
                   __ldg(fi + nx)) - uc;
  if (xl)
    gx = __fmaf_rn(lam, divp_at(pi + 1, vol, plane, nx, zl, zf, yl, yf,
                                x + 1 < nx - 1, true), __ldg(fi + 1)) - uc;
  float qz = __fmaf_rn(tau_over_lam, gz, __ldg(pi));
  float qy = __fmaf_rn(tau_over_lam, gy, __ldg(pi + vol));
  float qx = __fmaf_rn(tau_over_lam, gx, __ldg(pi + 2 * vol));
  // p / max(1, |p|): one reciprocal (mag >= 1) instead of three IEEE
  // divisions (rounding order pinned: rof_march2_kernel gives the same bits)
  const float inv = rof_inv_mag(qz, qy, qx);
  float* po = pout + i;
  po[0] = __fmul_rn(qz, inv);
  po[vol] = __fmul_rn(qy, inv);
  po[2 * vol] = __fmul_rn(qx, inv);
}

// ---- marching ROF (production for even nx) -----------------------------
// One dual iteration in one pass with the layout of tv_march2_kernel (lane
// = voxel pair, warp = row, 60 x 14 outputs, column march in z over TM_ZC
// planes, one barrier per plane): a thread loads f and p (pz, py, px) of its
// pair one plane ahead through a cp.async ring, forms u(z+1) = f + lam div p
// -- px(x-1) by shfl_up, py(y-1) from a shared row, pz(z) in registers --
// then the forward gradient of u at plane z (u(x+2) by shfl_down, u(y+1)
// from a shared row) and writes p' = (p + tau/lam grad u) / max(1, |.|).
// Values of p on the faces where the forward difference is undefined (and
// outside the window) are zeroed at load, which is the masking of divp_at;
// same expressions and rounding as rof_iter_kernel, so the same bits.
// 28 B / voxel: f and p read once, p' written once.
constexpr int RM_NS = 4;
constexpr int RM_D = RM_NS - 1;

// TMA: the four arrays of each plane arrive as 68 x 16 tensor boxes
// (one cp.async.bulk.tensor per array, issued by thread 0 into an mbarrier
// ring stage), as in tv_march2_tma_kernel; else per-thread cp.async.
struct RofMaps {
  CUtensorMap f, pz, py, px;
};

template <bool TMA>
__global__ void __launch_bounds__(TM_THREADS, 2)
    rof_march2_kernel(const float* __restrict__ f, const float* __restrict__ pin,
                      float* __restrict__ pout, Win W, float lam,
                      float tau_over_lam,
                      const __grid_constant__ RofMaps maps) {
  // dynamic: cp.async ring float2[RM_NS][4][TM_THREADS] (f pz py px), or
  // the TMA ring float[RM_NS][4][TMT_SLOT] + RM_NS mbarriers
  extern __shared__ __align__(128) unsigned char rm_smem[];
  float2* rm_ring = reinterpret_cast<float2*>(rm_smem);
  float* tm_ring = reinterpret_cast<float*>(rm_smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(
      rm_smem + sizeof(float) * RM_NS * 4 * TMT_SLOT);
  __shared__ float2 su[2][TM_WARPS][32];
  __shared__ float2 spy[2][TM_WARPS][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int tid = threadIdx.x;
  const int xt = blockIdx.x * TM2_OX - 4, yt = blockIdx.y * TM_OY - 1;
  const int x = blockIdx.x * TM2_OX - 2 + 2 * lane;  // pair (x, x + 1)
  const int y = blockIdx.y * TM_OY - 1 + w;
  const int zb = blockIdx.z * TM_ZC;
  const int ze = min(W.nz, zb + TM_ZC);
  const bool in_xy = x >= 0 && x < W.nx && y >= 0 && y < W.ny;
  const bool own = in_xy && lane > 0 && lane < 31 && w > 0 && w < TM_WARPS - 1;
  const size_t plane = (size_t)W.nx * W.ny;
  const size_t vol = plane * (size_t)W.nz;
  const int off = in_xy ? y * W.nx + x : 0;
  const bool xlb = x + 1 < W.nx - 1;  // x < nx - 1 holds for the even x
  const bool yl = y < W.ny - 1;
  const unsigned ring0 = (unsigned)__cvta_generic_to_shared(&rm_ring[tid]);
  constexpr unsigned RS = 4 * TM_THREADS * 8, RA = TM_THREADS * 8;
  int zi = zb - 1;
  const float* pf = f + (ptrdiff_t)zi * (ptrdiff_t)plane + off;
  const float* pp = pin + (ptrdiff_t)zi * (ptrdiff_t)plane + off;
  if (TMA) {
    if (tid == 0) {
      for (int i = 0; i < RM_NS; i++) mbar_init(&bars[i], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
  }
  auto issue = [&]() {
    const int st = (zi - zb + 1) & (RM_NS - 1);
    if (TMA) {
      if (tid == 0) {
        constexpr unsigned BOX = TMT_BOXX * TM_WARPS * sizeof(float);
        float* dst = tm_ring + st * 4 * TMT_SLOT;
        mbar_expect_tx(&bars[st], 4 * BOX);
        tma_load_3d(dst, &maps.f, xt, yt, zi, &bars[st]);
        tma_load_3d(dst + TMT_SLOT, &maps.pz, xt, yt, zi, &bars[st]);
        tma_load_3d(dst + 2 * TMT_SLOT, &maps.py, xt, yt, zi, &bars[st]);
        tma_load_3d(dst + 3 * TMT_SLOT, &maps.px, xt, yt, zi, &bars[st]);
      }
    } else {
      const bool ok = in_xy && (unsigned)zi < (unsigned)W.nz;
      const unsigned sa = ring0 + st * RS;
      cp_async8(sa, ok ? pf : f, ok);
      cp_async8(sa + RA, ok ? pp : f, ok);
      cp_async8(sa + 2 * RA, ok ? pp + vol : f, ok);
      cp_async8(sa + 3 * RA, ok ? pp + 2 * vol : f, ok);
      cp_async_commit();
      pf += plane;
      pp += plane;
    }
    zi++;
  };
  auto take = [&](int zz, float2& fv, float2& pz, float2& py, float2& px) {
    const int k = zz - zb + 1;
    const int st = k & (RM_NS - 1);
    if (TMA) {
      mbar_wait(&bars[st], (unsigned)(k / RM_NS) & 1u);
      const float* r = tm_ring + st * 4 * TMT_SLOT + w * TMT_BOXX + 2 + 2 * lane;
      fv = *reinterpret_cast<const float2*>(r);
      pz = *reinterpret_cast<const float2*>(r + TMT_SLOT);
      py = *reinterpret_cast<const float2*>(r + 2 * TMT_SLOT);
      px = *reinterpret_cast<const float2*>(r + 3 * TMT_SLOT);
    } else {
      const float2* r = rm_ring + st * 4 * TM_THREADS + tid;
      fv = r[0];
      pz = r[TM_THREADS];
      py = r[2 * TM_THREADS];
      px = r[3 * TM_THREADS];
    }
  };
#pragma unroll
  for (int i = 0; i <= RM_D - 1; i++) issue();  // planes zb-1 .. zb-2+D
  float2 u0 = make_float2(0.f, 0.f);
  float2 pz0 = make_float2(0.f, 0.f), py0 = pz0, px0 = pz0;
  float2* po = reinterpret_cast<float2*>(pout + (ptrdiff_t)zb * (ptrdiff_t)plane + off);
  const size_t plane2 = plane / 2, vol2 = vol / 2;
  const int wy = w < TM_WARPS - 1 ? w + 1 : w;
  const int wm = w > 0 ? w - 1 : 0;
  for (int z = zb - 2; z < ze; z++) {
    if (z + 1 + RM_D <= ze) {  // planes up to ze; empty groups keep the count
      issue();
    } else if (!TMA) {
      cp_async_commit();
    }
    if (!TMA) cp_async_wait<RM_D>();  // plane z + 1 landed (own slots only)
    float2 f1, pz1, py1, px1;
    take(z + 1, f1, pz1, py1, px1);
    spy[(z + 1) & 1][w][lane] = py1;
    __syncthreads();
    // u(z + 1) = f + lam div p (divp_at's terms and order): the voxel's own
    // p is dropped on the faces where its forward difference is undefined;
    // the backward neighbours' p (never on such a face) are zero-filled
    // outside the window.  The dual step below uses the raw p, as
    // rof_iter_kernel does.
    const float2 pym = spy[(z + 1) & 1][wm][lane];
    const float pxm = __shfl_up_sync(0xffffffffu, px1.y, 1);
    const bool zl1 = z + 1 < W.nz - 1;
    const float2 pz1m = zl1 ? pz1 : make_float2(0.f, 0.f);
    const float2 py1m = yl ? py1 : make_float2(0.f, 0.f);
    const float px1mb = xlb ? px1.y : 0.f;
    const float da = ((pz1m.x - pz0.x) + (py1m.x - pym.x)) + (px1.x - pxm);
    const float db = ((pz1m.y - pz0.y) + (py1m.y - pym.y)) + (px1mb - px1.x);
    const float2 u1 = make_float2(__fmaf_rn(lam, da, f1.x),
                                  __fmaf_rn(lam, db, f1.y));
    // gradient of u at plane z and the projected dual step
    if (z >= zb) {
      const float uxb = __shfl_down_sync(0xffffffffu, u0.x, 1);
      const float2 uy = su[z & 1][wy][lane];
      const bool zl = z < W.nz - 1;
      const float gza = zl ? u1.x - u0.x : 0.f, gzb = zl ? u1.y - u0.y : 0.f;
      const float gya = yl ? uy.x - u0.x : 0.f, gyb = yl ? uy.y - u0.y : 0.f;
      const float gxa = u0.y - u0.x, gxb = xlb ? uxb - u0.y : 0.f;
      const float qza = __fmaf_rn(tau_over_lam, gza, pz0.x);
      const float qzb = __fmaf_rn(tau_over_lam, gzb, pz0.y);
      const float qya = __fmaf_rn(tau_over_lam, gya, py0.x);
      const float qyb = __fmaf_rn(tau_over_lam, gyb, py0.y);
      const float qxa = __fmaf_rn(tau_over_lam, gxa, px0.x);
      const float qxb = __fmaf_rn(tau_over_lam, gxb, px0.y);
      const float ia = rof_inv_mag(qza, qya, qxa);
      const float ib = rof_inv_mag(qzb, qyb, qxb);
      if (own) {
        po[0] = make_float2(__fmul_rn(qza, ia), __fmul_rn(qzb, ib));
        po[vol2] = make_float2(__fmul_rn(qya, ia), __fmul_rn(qyb, ib));
        po[2 * vol2] = make_float2(__fmul_rn(qxa, ia), __fmul_rn(qxb, ib));
      }
      po += plane2;
    }
    su[(z + 1) & 1][w][lane] = u1;
    u0 = u1;
    pz0 = pz1;
    py0 = py1;
    px0 = px1;
  }
  cp_async_wait<0>();
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
  CS_COUNT_LAUNCH();
  CS_CHECK_CUDA(cudaGetLastError());
  return CS_OK;
}

__global__ void sqrt_in_place_kernel(double* v) { *v = sqrt(*v); }

// u_out = u - step g / ||g|| from a stored g (cs_tv_grad_store): the same
// update (tv_step1) as tv_gd_tiled_kernel<1> and the fused passes.
__global__ void __launch_bounds__(256)
    tv_step_g_kernel(const float4* __restrict__ u,
                     const float4* __restrict__ g, float4* __restrict__ uo,
                     size_t n4, double step, const double* __restrict__ sumsq,
                     double scale) {
  const double norm = sqrt(*sumsq) * scale;
  const bool skip = norm < 1e-30;  // regularization.py:148-149
  const float coef = skip ? 0.f : tv_coef(step, norm);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4;
       i += (size_t)gridDim.x * blockDim.x) {
    const float4 a = __ldg(u + i);
    if (skip) {
      uo[i] = a;
      continue;
    }
    const float4 b = __ldg(g + i);
    float4 r;
    r.x = tv_step1(a.x, b.x, coef);
    r.y = tv_step1(a.y, b.y, coef);
    r.z = tv_step1(a.z, b.z, coef);
    r.w = tv_step1(a.w, b.w, coef);
    uo[i] = r;
  }
}

__global__ void tv_step_g_tail_kernel(const float* __restrict__ u,
                                      const float* __restrict__ g,
                                      float* __restrict__ uo, size_t i0,
                                      size_t n, double step,
                                      const double* __restrict__ sumsq,
                                      double scale) {
  const double norm = sqrt(*sumsq) * scale;
  const bool skip = norm < 1e-30;
  const float coef = skip ? 0.f : tv_coef(step, norm);
  const size_t i = i0 + threadIdx.x;
  if (i < n) uo[i] = skip ? u[i] : tv_step1(u[i], g[i], coef);
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
  const dim3 grid((nx + TV_TX - 1) / TV_TX, (ny + TV_TY - 1) / TV_TY,
                  (core_hi - core_lo + TV_ZC - 1) / TV_ZC);
  const size_t nb = (size_t)grid.x * grid.y * grid.z;
  double* part = nullptr;
  retain_pool();
  CS_CHECK_CUDA(cudaMallocAsync((void**)&part, nb * sizeof(double), s));
  tv_gd_tiled_kernel<0><<<grid, dim3(TV_TX, TV_TY), 0, s>>>(
      u, nullptr, Win{nx, ny, nzw}, core_lo, core_hi, 0.0, nullptr, 1.0, part);
  CS_COUNT_LAUNCH();
  CS_CHECK_CUDA(cudaGetLastError());
  rc = reduce_into(part, nb, out_sum, s);
  cudaFreeAsync(part, s);
  return rc;
}

int cs_tv_grad_norm(const float* u, int nx, int ny, int nzw, int core_lo,
                    int core_hi, double* out_norm, cs_stream_t stream) {
  int rc = cs_tv_grad_sumsq(u, nx, ny, nzw, core_lo, core_hi, out_norm,
                            stream);
  if (rc) return rc;
  sqrt_in_place_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(out_norm);
  CS_COUNT_LAUNCH();
  CS_CHECK_CUDA(cudaGetLastError());
  return CS_OK;
}

int cs_tv_step(const float* u, float* u_out, int nx, int ny, int nzw,
               double step, const double* norm_sumsq_dev, double scale,
               cs_stream_t stream) {
  int rc = check_win(nx, ny, nzw);
  if (rc) return rc;
  CS_REQUIRE(u != u_out, CS_ERR_ARG, "cs_tv_step: u and u_out must differ");
  const dim3 grid((nx + TV_TX - 1) / TV_TX, (ny + TV_TY - 1) / TV_TY,
                  (nzw + TV_ZC - 1) / TV_ZC);
  tv_gd_tiled_kernel<1><<<grid, dim3(TV_TX, TV_TY), 0, (cudaStream_t)stream>>>(
      u, u_out, Win{nx, ny, nzw}, 0, nzw, step, norm_sumsq_dev, scale,
      nullptr);
  CS_COUNT_LAUNCH();
  CS_CHECK_CUDA(cudaGetLastError());
  return CS_OK;
}

int cs_tv_grad_store(const float* u, float* g, int nx, int ny, int nzw,
                     int core_lo, int core_hi, double* out_sum,
                     cs_stream_t stream) {
  int rc = check_win(nx, ny, nzw);
  if (rc) return rc;
  CS_REQUIRE(0 <= core_lo && core_lo < core_hi && core_hi <= nzw, CS_ERR_ARG,
             "bad core [%d, %d) in window of %d", core_lo, core_hi, nzw);
  CS_REQUIRE(u != g, CS_ERR_ARG, "cs_tv_grad_store: g aliases u");
  cudaStream_t s = (cudaStream_t)stream;
  static const char* tiled = getenv("CS_TV_TILED");  // A/B: r01 kernel
  if (tiled && tiled[0] == '1') {
    const dim3 grid((nx + TV_TX - 1) / TV_TX, (ny + TV_TY - 1) / TV_TY,
                    (nzw + TV_ZC - 1) / TV_ZC);
    const size_t nb = (size_t)grid.x * grid.y * grid.z;
    double* part = nullptr;
    retain_pool();
    CS_CHECK_CUDA(cudaMallocAsync((void**)&part, nb * sizeof(double), s));
    tv_gd_tiled_kernel<2><<<grid, dim3(TV_TX, TV_TY), 0, s>>>(
        u, g, Win{nx, ny, nzw}, 0, nzw, 0.0, nullptr, 1.0, part, core_lo,
        core_hi);
    CS_COUNT_LAUNCH();
    CS_CHECK_CUDA(cudaGetLastError());
    rc = reduce_into(part, nb, out_sum, s);
    cudaFreeAsync(part, s);
    return rc;
  }
  return launch_march<0>(u, nullptr, nullptr, g, nx, ny, nzw, core_lo,
                         core_hi, 0.0, nullptr, 1.0, out_sum, s);
}

int cs_tv_gd_fused(const float* u, const float* g, float* u_out, float* g_out,
                   int nx, int ny, int nzw, int core_lo, int core_hi,
                   double step, const double* norm_sumsq_dev, double scale,
                   double* out_sum, cs_stream_t stream) {
  int rc = check_win(nx, ny, nzw);
  if (rc) return rc;
  CS_REQUIRE(0 <= core_lo && core_lo < core_hi && core_hi <= nzw, CS_ERR_ARG,
             "bad core [%d, %d) in window of %d", core_lo, core_hi, nzw);
  CS_REQUIRE(u != u_out && u != g_out && g != u_out && g != g_out &&
                 u_out != g_out,
             CS_ERR_ARG, "cs_tv_gd_fused: outputs alias inputs or each other");
  CS_REQUIRE(norm_sumsq_dev != out_sum, CS_ERR_ARG,
             "cs_tv_gd_fused: the input and output sums must differ");
  cudaStream_t s = (cudaStream_t)stream;
  return launch_march<1>(u, g, u_out, g_out, nx, ny, nzw, core_lo, core_hi,
                         step, norm_sumsq_dev, scale, out_sum, s);
}

int cs_tv_step_g(const float* u, const float* g, float* u_out, int64_t n,
                 double step, const double* norm_sumsq_dev, double scale,
                 cs_stream_t stream) {
  CS_REQUIRE(n >= 0, CS_ERR_ARG, "negative length");
  // elementwise: u_out may be u (in place); not g
  CS_REQUIRE(g != u_out, CS_ERR_ARG, "cs_tv_step_g: u_out aliases g");
  cudaStream_t s = (cudaStream_t)stream;
  const bool vec = ((uintptr_t)u % 16 == 0) && ((uintptr_t)g % 16 == 0) &&
                   ((uintptr_t)u_out % 16 == 0);
  size_t n4 = vec ? (size_t)n / 4 : 0;
  if (n4) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t want = (n4 + 255) / 256;
    const unsigned blocks = (unsigned)(want < (size_t)sms * 16 ? want : (size_t)sms * 16);
    tv_step_g_kernel<<<blocks, 256, 0, s>>>(
        reinterpret_cast<const float4*>(u), reinterpret_cast<const float4*>(g),
        reinterpret_cast<float4*>(u_out), n4, step, norm_sumsq_dev, scale);
    CS_COUNT_LAUNCH();
    CS_CHECK_CUDA(cudaGetLastError());
  }
  for (size_t i0 = n4 * 4; i0 < (size_t)n; i0 += 1024) {
    tv_step_g_tail_kernel<<<1, 1024, 0, s>>>(u, g, u_out, i0, (size_t)n, step,
                                             norm_sumsq_dev, scale);
    CS_COUNT_LAUNCH();
    CS_CHECK_CUDA(cudaGetLastError());
  }
  return CS_OK;
}

int cs_rof_iter(const float* f, const float* p_in, float* p_out, int nx,
                int ny, int nzw, double lam, cs_stream_t stream) {
  int rc = check_win(nx, ny, nzw);
  if (rc) return rc;
  CS_REQUIRE(p_in != p_out, CS_ERR_ARG, "cs_rof_iter: p_in aliases p_out");
  CS_REQUIRE(lam > 0, CS_ERR_ARG, "lambda must be positive");
  cudaStream_t s = (cudaStream_t)stream;
  static const char* knob = getenv("CS_ROF_MARCH");  // A/B: 0 = r01 kernel
  const bool march = (!knob || knob[0] != '0') && nx % 2 == 0 &&
                     (uintptr_t)f % 8 == 0 && (uintptr_t)p_in % 8 == 0 &&
                     (uintptr_t)p_out % 8 == 0;
  if (march) {
    // TMA feed when every array qualifies (nx % 4 == 0, 16-byte bases)
    static const char* tma_knob = getenv("CS_TV_TMA");  // A/B: 0 = cp.async
    const size_t vol = (size_t)nx * ny * nzw;
    RofMaps maps;
    const bool tma = !(tma_knob && tma_knob[0] == '0') &&
                     tv_plane_map(&maps.f, f, nx, ny, nzw) &&
                     tv_plane_map(&maps.pz, p_in, nx, ny, nzw) &&
                     tv_plane_map(&maps.py, p_in + vol, nx, ny, nzw) &&
                     tv_plane_map(&maps.px, p_in + 2 * vol, nx, ny, nzw);
    const size_t smem =
        tma ? sizeof(float) * RM_NS * 4 * TMT_SLOT + sizeof(uint64_t) * RM_NS
            : (size_t)RM_NS * 4 * TM_THREADS * sizeof(float2);
    static std::atomic<unsigned long long> attr_done{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(attr_done.load() & bit)) {
      const int big = (int)(sizeof(float) * RM_NS * 4 * TMT_SLOT +
                            sizeof(uint64_t) * RM_NS);
      CS_CHECK_CUDA(cudaFuncSetAttribute(
          rof_march2_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
          big));
      CS_CHECK_CUDA(cudaFuncSetAttribute(
          rof_march2_kernel<false>,
          cudaFuncAttributeMaxDynamicSharedMemorySize,
          (int)((size_t)RM_NS * 4 * TM_THREADS * sizeof(float2))));
      attr_done.fetch_or(bit);
    }
    const dim3 grid((nx + TM2_OX - 1) / TM2_OX, (ny + TM_OY - 1) / TM_OY,
                    (nzw + TM_ZC - 1) / TM_ZC);
    if (tma)
      rof_march2_kernel<true><<<grid, TM_THREADS, smem, s>>>(
          f, p_in, p_out, Win{nx, ny, nzw}, (float)lam,
          (float)(ROF_TAU / lam), maps);
    else
      rof_march2_kernel<false><<<grid, TM_THREADS, smem, s>>>(
          f, p_in, p_out, Win{nx, ny, nzw}, (float)lam,
          (float)(ROF_TAU / lam), maps);
  } else {
    const dim3 grid((nx + 31) / 32, (ny + 7) / 8, nzw);
    rof_iter_kernel<<<grid, dim3(32, 8), 0, s>>>(
        f, p_in, p_out, Win{nx, ny, nzw}, (float)lam, (float)(ROF_TAU / lam));
  }
  CS_COUNT_LAUNCH();
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
  CS_COUNT_LAUNCH();
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
  retain_pool();
  CS_CHECK_CUDA(cudaMallocAsync((void**)&part, nb * sizeof(double), s));
  tv_norm_kernel<<<grid, dim3(32, 8), 0, s>>>(u, Win{nx, ny, nzw}, part);
  CS_COUNT_LAUNCH();
  CS_CHECK_CUDA(cudaGetLastError());
  rc = reduce_into(part, nb, out_sum, s);
  cudaFreeAsync(part, s);
  return rc;
}

}  // extern "C"
