// fwd_dual.cu -- interpolated Ax (K1) on both fetch pipes of every SM.
//
// Measured on B200 (tools/micro/fetch_rates.cu, profiles/): the texture
// path returns 8 floats/clk/SM (tld4 gathers at 2 per clk), shared memory
// 32 floats/clk/SM, and the two pipes run concurrently.  The texture
// kernel (forward.cu) sits at ~85% of the texture ceiling with ~45% of its
// issue slots idle; the shared-memory staged kernel (staged.cu) is bound by
// issue and box-load latency.  Here one persistent CTA runs both:
//   * warps 0..7  ("texture half") trace a 32u x 8v tile of detector rays
//     with two tld4 gathers per trilinear sample (forward.cu's method);
//   * warps 8..15 ("staged half") trace another tile from CTA-staged volume
//     boxes in shared memory (staged.cu's method: chunks of DS planes along
//     the view's main axis), synchronising on their own named barrier.
// Both halves pull work items (tiles, view-major) from one atomic counter,
// so the split between the pipes follows the hardware, and the latency of
// one half's box loads is hidden by the other half's issue.
//
// Each sample is evaluated with the same fp32 operations in the same order
// by both halves (tri_acc below; the texture half's values, zero padding
// and slab masks equal the staged half's box contents), so a ray's result
// does not depend on which half traced it: outputs are deterministic and
// identical to forward.cu's kernel.  Ray set-up is the shared fp64 code of
// common.cuh (_kernels.py:194-246); the march is _kernels.py:248-275.
#include <climits>
#include <cstdlib>
#include <map>
#include <mutex>

#include "common.cuh"

namespace cs {

constexpr int DU = 32;   // item: 32 (u) x 8 (v) rays of one view
constexpr int DV = 8;
constexpr int DS = 8;    // planes per staged chunk along the main axis
constexpr int HALF = 256;
constexpr int BAR_TEX = 1;  // named barriers of the two halves (0 = CTA)
constexpr int BAR_ST = 2;
#ifndef DUAL_MINB
#define DUAL_MINB 2
#endif

struct DualArgs {
  cudaTextureObject_t tex;   // slab [z_lo, z_hi) as a layered texture
  const float* vol;          // the same slab, linear [z][y][x]
  const AngleGeom* geom;
  Grid G;
  double step_max;
  int z_lo, z_hi, n_u, n_v, v_base, v_end;
  int tiles_u, tiles_v, n_items;
  float* out;
  const float* rb;
  const float* rw;
  int* counter;
  int box_cap;
  int vec_ok;
};

__device__ __forceinline__ void half_bar(int id) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(HALF) : "memory");
}

// One trilinear sample added to acc: slice l0 taps a.. and slice l1 taps
// c.. at (i, j), (i+1, j), (i, j+1), (i+1, j+1); m0 / m1 = slab-masked z
// weights.  Identical operation order to forward.cu's kernel.
__device__ __forceinline__ float tri_acc(float acc, float wx, float wy,
                                         float m0, float m1, float a00,
                                         float a10, float a01, float a11,
                                         float c00, float c10, float c01,
                                         float c11) {
  const float r00 = fmaf(wx, a10 - a00, a00);
  const float r01 = fmaf(wx, a11 - a01, a01);
  const float r10 = fmaf(wx, c10 - c00, c00);
  const float r11 = fmaf(wx, c11 - c01, c01);
  const float b0 = fmaf(wy, r01 - r00, r00);
  const float b1 = fmaf(wy, r11 - r10, r10);
  return fmaf(m0, b0, fmaf(m1, b1, acc));
}

template <int MODE>
__device__ __forceinline__ void emit(const DualArgs& P, int a, int u, int v,
                                     float acc, double step) {
  const size_t idx = ((size_t)a * P.n_v + v) * P.n_u + u;
  const float val = acc * (float)step;
  if (MODE == 0) {
    P.out[idx] = val;
  } else if (MODE == 1) {
    P.out[idx] += val;
  } else {
    const float wt = P.rw ? P.rw[idx] : 1.f;
    P.out[idx] = wt * (P.rb[idx] - val);
  }
}

// Eight taps of one sample straight from global memory (zero outside the
// grid / slab): the staged half's fallback for boxes that do not fit.
__device__ __forceinline__ float global_sample(const DualArgs& P, float acc,
                                               float qx, float qy,
                                               float qz) {
  const float fx = floorf(qx), fy = floorf(qy), fz = floorf(qz);
  const float wx = qx - fx, wy = qy - fy, wz = qz - fz;
  const int ix = (int)fx, iy = (int)fy;
  const int l0 = (int)fz - P.z_lo, l1 = l0 + 1;
  const int top = P.z_hi - P.z_lo - 1;
  const int nx = P.G.n[0], ny = P.G.n[1];
  const float m0 = (l0 >= 0 && l0 <= top) ? 1.f - wz : 0.f;
  const float m1 = (l1 >= 0 && l1 <= top) ? wz : 0.f;
  float t[2][4];
#pragma unroll
  for (int c = 0; c < 2; c++) {
    const int l = c ? l1 : l0;
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const int x = ix + (q & 1), y = iy + (q >> 1);
      t[c][q] = (l >= 0 && l <= top && x >= 0 && x < nx && y >= 0 && y < ny)
                    ? __ldg(P.vol + ((size_t)l * ny + y) * nx + x)
                    : 0.f;
    }
  }
  return tri_acc(acc, wx, wy, m0, m1, t[0][0], t[0][1], t[0][2], t[0][3],
                 t[1][0], t[1][1], t[1][2], t[1][3]);
}

// ---------------------------------------------------------------- texture
template <int MODE>
__device__ void tex_item(const DualArgs& P, int a, int tu, int tv, int tid) {
  const int lane = tid & 31, w = tid >> 5;
  // warp = 8u x 4v sub-tile (compact ray frustum -> compact texel set)
  const int u = tu * DU + (w & 3) * 8 + (lane & 7);
  const int v = P.v_base + tv * DV + (w >> 2) * 4 + (lane >> 3);
  if (u >= P.n_u || v >= P.v_end) return;
  Ray r;
  setup_ray(P.geom[a], P.G, P.step_max, u, v, r);
  float acc = 0.f;
  if (r.n > 0) {
    March m;
    march_params(r, P.G, m);
    long long k0l, k1l;
    slab_k_range(r, m, P.G, P.z_lo, P.z_hi, k0l, k1l);
    const int k0 = (int)k0l, k1 = (int)k1l, kc = (int)m.kc;
    const int top = P.z_hi - P.z_lo - 1;
    float cfx = -1e30f, cfy = 0.f, cfz = 0.f;
    float4 s0 = make_float4(0.f, 0.f, 0.f, 0.f), s1 = s0;
#pragma unroll 2
    for (int k = k0; k < k1; ++k) {
      const float kf = (float)(k - kc);
      const float qx = fmaf(kf, m.B[0], m.A[0]);
      const float qy = fmaf(kf, m.B[1], m.A[1]);
      const float qz = fmaf(kf, m.B[2], m.A[2]);
      const float fx = floorf(qx), fy = floorf(qy), fz = floorf(qz);
      const float wx = qx - fx, wy = qy - fy, wz = qz - fz;
      const int l0 = (int)fz - P.z_lo, l1 = l0 + 1;
      const float m0 = (l0 >= 0 && l0 <= top) ? 1.f - wz : 0.f;
      const float m1 = (l1 >= 0 && l1 <= top) ? wz : 0.f;
      if (fx != cfx || fy != cfy || fz != cfz) {
        s0 = gather_a2d(P.tex, min(max(l0, 0), top), fx + 1.f, fy + 1.f);
        s1 = gather_a2d(P.tex, min(max(l1, 0), top), fx + 1.f, fy + 1.f);
        cfx = fx;
        cfy = fy;
        cfz = fz;
      }
      // tld4: w = (i, j), z = (i+1, j), x = (i, j+1), y = (i+1, j+1)
      acc = tri_acc(acc, wx, wy, m0, m1, s0.w, s0.z, s0.x, s0.y, s1.w, s1.z,
                    s1.x, s1.y);
    }
  }
  emit<MODE>(P, a, u, v, acc, r.step);
}

// ----------------------------------------------------------------- staged
__device__ __forceinline__ int dual_qfloor(const March& m, int k, int axis) {
  return (int)floorf(fmaf((float)(k - (int)m.kc), m.B[axis], m.A[axis]));
}

template <int M, int MODE>
__device__ void staged_item(const DualArgs& P, int a, int tu, int tv,
                            int tid, float* box, int* ext, int* ext8) {
  constexpr int T = 1 - M;
  const int lane = tid & 31, warp = tid >> 5;
  const int u = tu * DU + lane;
  const int v = P.v_base + tv * DV + warp;
  const bool valid = u < P.n_u && v < P.v_end;
  const int nx = P.G.n[0], ny = P.G.n[1];
  const size_t plane = (size_t)nx * ny;
  const int top = P.z_hi - P.z_lo - 1;

  Ray r;
  r.n = 0;
  r.step = 0.0;
  if (valid) setup_ray(P.geom[a], P.G, P.step_max, u, v, r);
  March m;
  int k0 = 0, k1 = 0;
  if (r.n > 0) {
    march_params(r, P.G, m);
    long long k0l, k1l;
    slab_k_range(r, m, P.G, P.z_lo, P.z_hi, k0l, k1l);
    k0 = (int)k0l;
    k1 = (int)k1l;
  }
  const bool has = k1 > k0;
  if (tid == 0) {
    ext[0] = INT_MAX;
    ext[1] = INT_MIN;
    ext[6] = 0;
    ext[7] = 0;
  }
  half_bar(BAR_ST);
  if (has) {
    const int fa = dual_qfloor(m, k0, M), fb = dual_qfloor(m, k1 - 1, M);
    atomicMin(&ext[0], min(fa, fb));
    atomicMax(&ext[1], max(fa, fb));
    atomicOr(&ext[m.B[M] >= 0.f ? 7 : 6], 1);
  }
  half_bar(BAR_ST);
  const int mlo = ext[0], mhi = ext[1];
  const int dir = ext[6] ? -1 : 1;
  const bool mixed = ext[6] && ext[7];
  float acc = 0.f;
  if (mlo <= mhi && mixed) {
    // rays of this tile march both ways along M (degenerate geometry):
    // every sample from global memory
    for (int kk = k0; kk < k1; kk++) {
      const float kf = (float)(kk - (int)m.kc);
      acc = global_sample(P, acc, fmaf(kf, m.B[0], m.A[0]),
                          fmaf(kf, m.B[1], m.A[1]), fmaf(kf, m.B[2], m.A[2]));
    }
  }
  int k = k0;
  int cur = dir > 0 ? mlo : mhi;
  const bool run = mlo <= mhi && !mixed;
  while (run && (dir > 0 ? cur <= mhi : cur >= mlo)) {
    // candidate chunks of DS and DS/2 cells along M (march order)
    int kbc[2] = {k, k};
    if (has) {
#pragma unroll
      for (int ci = 0; ci < 2; ci++) {
        const int S = DS >> ci;
        const int c_lo = dir > 0 ? cur : cur - S + 1;
        const int c_hi = c_lo + S - 1;
        const float face = dir > 0 ? (float)(c_hi + 1) : (float)c_lo;
        const float kst = (face - m.A[M]) / m.B[M] + (float)(int)m.kc;
        int ke = (int)fminf(fmaxf(ceilf(kst), (float)k), (float)k1);
        if (dir > 0) {
          while (ke > k && dual_qfloor(m, ke - 1, M) > c_hi) ke--;
          while (ke < k1 && dual_qfloor(m, ke, M) <= c_hi) ke++;
        } else {
          while (ke > k && dual_qfloor(m, ke - 1, M) < c_lo) ke--;
          while (ke < k1 && dual_qfloor(m, ke, M) >= c_lo) ke++;
        }
        kbc[ci] = ke;
      }
    }
    half_bar(BAR_ST);  // previous chunk's box fully consumed
    if (tid < 8) ext8[tid] = (tid & 1) ? INT_MIN : INT_MAX;
    half_bar(BAR_ST);
#pragma unroll
    for (int ci = 0; ci < 2; ci++) {
      if (kbc[ci] > k) {
        const int t0 = dual_qfloor(m, k, T), t1 = dual_qfloor(m, kbc[ci] - 1, T);
        const int z0 = dual_qfloor(m, k, 2), z1 = dual_qfloor(m, kbc[ci] - 1, 2);
        atomicMin(&ext8[4 * ci + 0], min(t0, t1));
        atomicMax(&ext8[4 * ci + 1], max(t0, t1));
        atomicMin(&ext8[4 * ci + 2], min(z0, z1));
        atomicMax(&ext8[4 * ci + 3], max(z0, z1));
      }
    }
    half_bar(BAR_ST);
    auto box_size = [&](int ci, int S) {
      const int c_lo = dir > 0 ? cur : cur - S + 1;
      const int nt = ext8[4 * ci + 1] - ext8[4 * ci] + 2;
      const int nzz = ext8[4 * ci + 3] - ext8[4 * ci + 2] + 2;
      const int xlo = M == 0 ? c_lo : ext8[4 * ci];
      const int xn = M == 0 ? S + 1 : nt;
      const int nbx = ((xlo + xn - (xlo & ~3)) + 3) & ~3;
      const int nby = M == 0 ? nt : S + 1;
      return M == 1 ? nbx * nby * nzz : nbx * (nby | 1) * nzz;
    };
    const int ci = (ext8[0] > ext8[1] || box_size(0, DS) <= P.box_cap) ? 0 : 1;
    const int S = DS >> ci;
    const int c_lo = dir > 0 ? cur : cur - S + 1;
    cur += dir * S;
    const int ka = k, kb = kbc[ci];
    k = kb;
    if (ext8[4 * ci] > ext8[4 * ci + 1]) continue;  // nobody samples it
    // box over taps: cells [lo, hi + 1] per axis; x padded to aligned quads
    int bo[3], bn[3];
    bo[M] = c_lo;
    bn[M] = S + 1;
    bo[T] = ext8[4 * ci];
    bn[T] = ext8[4 * ci + 1] - ext8[4 * ci] + 2;
    bo[2] = ext8[4 * ci + 2];
    bn[2] = ext8[4 * ci + 3] - ext8[4 * ci + 2] + 2;
    {
      const int x0 = bo[0] & ~3;
      bn[0] = ((bo[0] + bn[0] - x0) + 3) & ~3;
      bo[0] = x0;
    }
    // transverse axis innermost (lanes = adjacent T -> distinct banks):
    //   M = y: [z][y][x], x-quads contiguous;  M = x: [z][x][y], odd pitch
    const int sx = M == 1 ? 1 : (bn[1] | 1);
    const int sy = M == 1 ? bn[0] : 1;
    const int sz = M == 1 ? bn[0] * bn[1] : bn[0] * sx;
    const bool fits = sz * bn[2] <= P.box_cap;
    const int qpr = bn[0] >> 2;  // x-quads per (y, z) row
    if (fits) {
      // box load: rows (y, z) walked incrementally, lanes over x-quads
      // (M = y: a warp per row; M = x: 8 rows x 4 quads per warp)
      const int rows = bn[1] * bn[2];
      const int rpw = M == 1 ? 1 : 8;          // rows per warp-iteration
      const int lq = M == 1 ? lane : (lane & 3);
      int row = M == 1 ? warp : warp * 8 + (lane >> 2);
      int by = row, bz = 0;
      while (by >= bn[1]) {
        by -= bn[1];
        bz++;
      }
      const int rstep = 8 * rpw;
      for (; row < rows; row += rstep) {
        const int gy = bo[1] + by, gz = bo[2] + bz;
        const bool row_in = gy >= 0 && gy < ny && gz >= P.z_lo && gz < P.z_hi;
        const float* src = P.vol + (size_t)(gz - P.z_lo) * plane +
                           (size_t)gy * nx;
        for (int xq = lq; xq < qpr; xq += (M == 1 ? 32 : 4)) {
          const int gx = bo[0] + 4 * xq;
          float4 q4 = make_float4(0.f, 0.f, 0.f, 0.f);
          if (row_in) {
            if (P.vec_ok && gx >= 0 && gx + 3 < nx) {
              q4 = __ldg(reinterpret_cast<const float4*>(src + gx));
            } else {
              if (gx >= 0 && gx < nx) q4.x = __ldg(src + gx);
              if (gx + 1 >= 0 && gx + 1 < nx) q4.y = __ldg(src + gx + 1);
              if (gx + 2 >= 0 && gx + 2 < nx) q4.z = __ldg(src + gx + 2);
              if (gx + 3 >= 0 && gx + 3 < nx) q4.w = __ldg(src + gx + 3);
            }
          }
          const int d = bz * sz + by * sy + 4 * xq * sx;
          if (M == 1) {
            *reinterpret_cast<float4*>(box + d) = q4;
          } else {
            box[d] = q4.x;
            box[d + sx] = q4.y;
            box[d + 2 * sx] = q4.z;
            box[d + 3 * sx] = q4.w;
          }
        }
        by += rstep;
        while (by >= bn[1]) {
          by -= bn[1];
          bz++;
        }
      }
      half_bar(BAR_ST);
    }
    for (int kk = ka; kk < kb; kk++) {
      const float kf = (float)(kk - (int)m.kc);
      const float qx = fmaf(kf, m.B[0], m.A[0]);
      const float qy = fmaf(kf, m.B[1], m.A[1]);
      const float qz = fmaf(kf, m.B[2], m.A[2]);
      if (fits) {
        const float fx = floorf(qx), fy = floorf(qy), fz = floorf(qz);
        const float wx = qx - fx, wy = qy - fy, wz = qz - fz;
        const int ix = (int)fx, iy = (int)fy, iz = (int)fz;
        const int l0 = iz - P.z_lo, l1 = l0 + 1;
        const float m0 = (l0 >= 0 && l0 <= top) ? 1.f - wz : 0.f;
        const float m1 = (l1 >= 0 && l1 <= top) ? wz : 0.f;
        const float* b = box + (iz - bo[2]) * sz + (iy - bo[1]) * sy +
                         (ix - bo[0]) * sx;
        acc = tri_acc(acc, wx, wy, m0, m1, b[0], b[sx], b[sy], b[sy + sx],
                      b[sz], b[sz + sx], b[sz + sy], b[sz + sy + sx]);
      } else {
        acc = global_sample(P, acc, qx, qy, qz);
      }
    }
  }
  if (valid) emit<MODE>(P, a, u, v, acc, r.step);
}

// Main axis of a view from its central ray: 0 = x, 1 = y.
__device__ __forceinline__ int dual_view_axis(const AngleGeom& g, int n_u,
                                              int n_v) {
  double d[2];
#pragma unroll
  for (int i = 0; i < 2; i++)
    d[i] = g.det00[i] + 0.5 * (n_u - 1) * g.ustep[i] +
           0.5 * (n_v - 1) * g.vstep[i] - g.src[i];
  return fabs(d[0]) >= fabs(d[1]) ? 0 : 1;
}

template <int MODE>
__global__ void __launch_bounds__(2 * HALF, DUAL_MINB) fwd_dual_kernel(DualArgs P) {
  extern __shared__ float4 dual_smem[];
  float* box = reinterpret_cast<float*>(dual_smem);
  __shared__ int s_item[2];
  __shared__ int ext[8], ext8[8];
  const int half = threadIdx.x / HALF;  // 0 = texture, 1 = staged
  const int tid = threadIdx.x % HALF;
  const int bar = half ? BAR_ST : BAR_TEX;
  const int per_view = P.tiles_u * P.tiles_v;
  for (;;) {
    if (tid == 0) s_item[half] = atomicAdd(P.counter, 1);
    half_bar(bar);
    const int item = s_item[half];
    half_bar(bar);
    if (item >= P.n_items) break;
    const int a = item / per_view;
    const int rem = item - a * per_view;
    const int tv = rem / P.tiles_u, tu = rem - tv * P.tiles_u;
    if (half == 0) {
      tex_item<MODE>(P, a, tu, tv, tid);
    } else if (dual_view_axis(P.geom[a], P.n_u, P.n_v) == 0) {
      staged_item<0, MODE>(P, a, tu, tv, tid, box, ext, ext8);
    } else {
      staged_item<1, MODE>(P, a, tu, tv, tid, box, ext, ext8);
    }
  }
}

// per (device, stream) work counter
static int dual_counter(cudaStream_t s, int** out) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, int*> cache;
  int dev = 0;
  CS_CHECK_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  int*& p = cache[{dev, s}];
  if (!p) CS_CHECK_CUDA(cudaMalloc((void**)&p, sizeof(int)));
  *out = p;
  return CS_OK;
}

bool dual_enabled() {
  static int on = -1;
  if (on < 0) {
    // opt-in A/B (CS_FWD_DUAL=1): measured slower than the texture kernel
    // at config 2 (225 vs 268 GUPS, DESIGN.md experiments)
    const char* k = getenv("CS_FWD_DUAL");
    on = (k && k[0] == '1') ? 1 : 0;
  }
  return on == 1;
}

template <int MODE>
int launch_dual(cudaTextureObject_t tex, const float* vol, const AngleGeom* dgeom,
                const Grid& G, double step_max, int z_lo, int z_hi, int n_a,
                int n_u, int n_v, int v0, int v1, float* out, const float* b,
                const float* w, cudaStream_t s) {
  DualArgs P;
  P.tex = tex;
  P.vol = vol;
  P.geom = dgeom;
  P.G = G;
  P.step_max = step_max;
  P.z_lo = z_lo;
  P.z_hi = z_hi;
  P.n_u = n_u;
  P.n_v = n_v;
  P.v_base = v0;
  P.v_end = v1;
  P.tiles_u = (n_u + DU - 1) / DU;
  P.tiles_v = (v1 - v0 + DV - 1) / DV;
  const long long items = (long long)n_a * P.tiles_u * P.tiles_v;
  CS_REQUIRE(items < INT_MAX, CS_ERR_ARG, "too many work items (%lld)", items);
  P.n_items = (int)items;
  P.out = out;
  P.rb = b;
  P.rw = w;
  static const char* kb = getenv("CS_DUAL_SMEM_KB");
  const size_t smem = (size_t)(kb ? atoi(kb) : 64) * 1024;
  P.box_cap = (int)(smem / sizeof(float));
  P.vec_ok = (G.n[0] % 4 == 0) && (((uintptr_t)vol & 15) == 0);
  int rc = dual_counter(s, &P.counter);
  if (rc) return rc;
  CS_CHECK_CUDA(cudaMemsetAsync(P.counter, 0, sizeof(int), s));
  static bool attr = false;
  if (!attr) {
    CS_CHECK_CUDA(cudaFuncSetAttribute(
        fwd_dual_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
        200 * 1024));
    attr = true;
  }
  int per_sm = 0;
  CS_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &per_sm, fwd_dual_kernel<MODE>, 2 * HALF, smem));
  CS_REQUIRE(per_sm > 0, CS_ERR_UNSUPPORTED, "dual Ax kernel does not fit");
  const long long want = (long long)per_sm * num_sms();
  const int grid = (int)(want < (items + 1) / 2 + 1 ? want : (items + 1) / 2 + 1);
  fwd_dual_kernel<MODE><<<grid, 2 * HALF, smem, s>>>(P);
  CS_CHECK_CUDA(cudaGetLastError());
  return CS_OK;
}

template int launch_dual<0>(cudaTextureObject_t, const float*,
                            const AngleGeom*, const Grid&, double, int, int,
                            int, int, int, int, int, float*, const float*,
                            const float*, cudaStream_t);
template int launch_dual<1>(cudaTextureObject_t, const float*,
                            const AngleGeom*, const Grid&, double, int, int,
                            int, int, int, int, int, float*, const float*,
                            const float*, cudaStream_t);
template int launch_dual<2>(cudaTextureObject_t, const float*,
                            const AngleGeom*, const Grid&, double, int, int,
                            int, int, int, int, int, float*, const float*,
                            const float*, cudaStream_t);

}  // namespace cs
