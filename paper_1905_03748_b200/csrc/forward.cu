// forward.cu -- Ax: interpolated (K1) and Siddon (K4) cone-beam forward
// projectors for sm_100a.
//
// K1 design: one thread per detector ray, a warp per 8u x 4v
// detector tile (a compact ray frustum, so the 32 lanes gather from a
// compact texel neighbourhood), four warps per CTA (16u x 8v).  The ray
// set-up is fp64 and bit-identical to the reference (_kernels.py:194-246);
// positions are exact Q32.32 fixed point (common.cuh).  Each trilinear sample is
// TWO texture gathers (tld4 on a 2D-layered float texture: 2x2 texels of
// two adjacent layers) with fp32 software weights, i.e. exact
// interpolation weights (hardware filtering's 8-bit weights are 100x off
// the parity budget) at a quarter of the point-sample
// fetch count.  Production: fwd_mlayer_kernel (layers = planes along the
// view's main axis, v-adjacent texture quads, pipelined gathers);
// fwd_interp_kernel (layers = z slices) is the A/B baseline and serves
// the residual epilogue when x or y exceeds the layer limit.  Border addressing gives the reference's zero padding in
// x/y; z taps are masked to the slab [z_lo, z_hi) exactly as
// _kernels.py:259-262, and the sample range is clipped to the slab so a
// slab launch costs only its share of the ray.
#include <climits>
#include <cstdlib>
#include <cstring>

#include "common.cuh"

namespace cs {

enum FwdMode { FWD_OVERWRITE = 0, FWD_ACCUMULATE = 1, FWD_RESIDUAL = 2 };

constexpr int FWD_TILE_U = 16;  // per CTA
constexpr int FWD_TILE_V = 8;

// v_base: first detector row of the launch (v-band culling: rows whose rays
// cannot reach the slab are not launched, runtime.cu slab_row_band).
__device__ __forceinline__ void tile_coords(int& u, int& v, int v_base) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  u = blockIdx.x * FWD_TILE_U + (warp & 1) * 8 + (lane & 7);
  v = v_base + blockIdx.y * FWD_TILE_V + (warp >> 1) * 4 + (lane >> 3);
}

#ifndef FWD_MINB
#define FWD_MINB 8  // <= 64 registers: 32 warps/SM keep the tld4 pipe fed
#endif
template <int MODE>
__global__ void __launch_bounds__(128, FWD_MINB)
    fwd_interp_kernel(cudaTextureObject_t tex,
                      const AngleGeom* __restrict__ geom, Grid G,
                      double step_max, int z_lo, int z_hi, int n_u, int n_v,
                      int v_base, int v_end, float* __restrict__ out,
                      const float* __restrict__ b,
                      const float* __restrict__ w) {
  int u, v;
  tile_coords(u, v, v_base);
  const int a = blockIdx.z;
  if (u >= n_u || v >= v_end) return;
  Ray r;
  setup_ray(geom[a], G, step_max, u, v, r);
  float acc = 0.f;
  if (r.n > 0) {
    March m;
    march_params(r, G, m);
    long long k0l, k1l;
    slab_k_range(r, m, G, z_lo, z_hi, k0l, k1l);
    const int k0 = (int)k0l, k1 = (int)k1l;
    const int top = z_hi - z_lo - 1;
    // exact fixed-point positions (common.cuh), advanced by integer adds
    long long qx = q_at(m, k0, 0), qy = q_at(m, k0, 1), qz = q_at(m, k0, 2);
    const long long bx = m.Bq[0], by = m.Bq[1], bz = m.Bq[2];
    // Consecutive samples (step <= half a voxel) often share their 2x2x2
    // texel cell; re-gather only when the cell changes (-10% texture
    // writeback, the measured limiter).
    int cx = INT_MIN, cy = 0, cz = 0;
    float4 s0 = make_float4(0.f, 0.f, 0.f, 0.f), s1 = s0;
#pragma unroll 2
    for (int k = k0; k < k1; ++k, qx += bx, qy += by, qz += bz) {
      const int ix = q_cell(qx), iy = q_cell(qy), iz = q_cell(qz);
      const float wx = q_frac(qx), wy = q_frac(qy), wz = q_frac(qz);
      const int l0 = iz - z_lo, l1 = l0 + 1;
      const float m0 = (l0 >= 0 && l0 <= top) ? 1.f - wz : 0.f;
      const float m1 = (l1 >= 0 && l1 <= top) ? wz : 0.f;
      if (ix != cx || iy != cy || iz != cz) {
        const float tx = int_to_float(ix + 1), ty = int_to_float(iy + 1);
        s0 = gather_a2d(tex, min(max(l0, 0), top), tx, ty);
        s1 = gather_a2d(tex, min(max(l1, 0), top), tx, ty);
        cx = ix;
        cy = iy;
        cz = iz;
      }
      // s.w=(i,j) s.z=(i+1,j) s.x=(i,j+1) s.y=(i+1,j+1)
      const float r00 = fmaf(wx, s0.z - s0.w, s0.w);
      const float r01 = fmaf(wx, s0.y - s0.x, s0.x);
      const float r10 = fmaf(wx, s1.z - s1.w, s1.w);
      const float r11 = fmaf(wx, s1.y - s1.x, s1.x);
      const float b0 = fmaf(wy, r01 - r00, r00);
      const float b1 = fmaf(wy, r11 - r10, r10);
      acc = fmaf(m0, b0, fmaf(m1, b1, acc));
    }
  }
  const float val = acc * (float)r.step;
  const size_t idx = ((size_t)a * n_v + v) * n_u + u;
  if (MODE == FWD_OVERWRITE) {
    out[idx] = val;
  } else if (MODE == FWD_ACCUMULATE) {
    out[idx] += val;
  } else {
    const float wt = w ? w[idx] : 1.f;
    out[idx] = wt * (b[idx] - val);
  }
}

// ---------------------------------------------------------------------------
// K1 on main-axis layers.  For views whose central ray runs mainly along
// M (x or y), the slab is held as a 2D-layered texture with one layer per
// M plane (texel (T, z - s0) of layer iM), and a warp's quads are 4
// v-ADJACENT rays: rays of one detector column share their xy path and,
// with equal sample counts, their x / y sample positions, so their cells
// change together -- the texture pipe charges a tld4 per quad with any
// active lane.  A cell change re-gathers both layers (iM, iM + 1).  T and z
// outside the texture read the border zero (the reference's padding and
// the slab's z range); layers outside [0, n_M) -- or outside the piece of
// layers this launch holds -- are masked in the weights.
#ifndef ML_WU
#define ML_WU 2
#endif
#ifndef ML_WARP_U
#define ML_WARP_U 8
#endif
constexpr int ML_TILE_U = ML_WARP_U * ML_WU,
              ML_TILE_V = (32 / ML_WARP_U) * (4 / ML_WU);
#ifndef FWD_ML_MINB
#define FWD_ML_MINB 8  // 64 registers (two prefetch buffers), 32 warps/SM
#endif
template <int MODE, int M>
__global__ void __launch_bounds__(128, FWD_ML_MINB)
    fwd_mlayer_kernel(cudaTextureObject_t tex,
                      const AngleGeom* __restrict__ geom,
                      const int* __restrict__ view_ids, Grid G,
                      double step_max, int z_lo, int z_hi, int m_lo,
                      int m_hi, int n_u, int n_v, int v_base, int v_end,
                      float* __restrict__ out, const float* __restrict__ b,
                      const float* __restrict__ w) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // warp = ML_WARP_U u x (32 / ML_WARP_U) v rays, v fastest (quads = 4
  // v-adjacent lanes); the CTA's 4 warps tile ML_WU x (4 / ML_WU) along (u, v)
  constexpr int WV = 32 / ML_WARP_U;
  const int u = blockIdx.x * ML_TILE_U + (warp % ML_WU) * ML_WARP_U + lane / WV;
  const int v = v_base + blockIdx.y * ML_TILE_V + (warp / ML_WU) * WV +
                lane % WV;
  const int a = view_ids[blockIdx.z];
  if (u >= n_u || v >= v_end) return;
  Ray r;
  setup_ray(geom[a], G, step_max, u, v, r);
  float acc = 0.f;
  if (r.n > 0) {
    March m;
    march_params(r, G, m);
    long long k0l, k1l, k0m, k1m;
    slab_k_range(r, m, G, z_lo, z_hi, k0l, k1l);
    // the texture holds M planes [m_lo, m_hi) (all of them unless n_M
    // exceeds the layer limit); layer = plane - m_lo
    constexpr int T = 1 - M;
    axis_k_range(r, m, M, G.n[M], m_lo, m_hi, k0m, k1m);
    const int k0 = (int)max(k0l, k0m), k1 = (int)min(k1l, k1m);
    const int top = m_hi - m_lo - 1;
    long long qm = q_at(m, k0, M) - ((long long)m_lo << QF), qt = q_at(m, k0, T),
              qz = q_at(m, k0, 2);
    const long long bm = m.Bq[M], bt = m.Bq[T], bz = m.Bq[2];
    // Software-pipelined over two prefetch buffers: sample k+1's gathers
    // (predicated on its cell change) go to one while sample k's data is
    // taken from the other, gathered one iteration earlier, so the wait for
    // a gather spans a whole iteration.  With the quads skipping together
    // the plain loop was tld4-latency bound.  r01 A/B at config 2 (90-view
    // launches incl. texture fills): re-gather on change 283 GUPS; one-layer
    // M-step reuse through predicated gathers 242 (+38% instructions); one
    // prefetch buffer 309 (56 regs) / 325 (48 regs) -- its rotation waited
    // on the gathers just issued; two buffers 344 (64 regs) / 326 (56) /
    // 283 (48, spills).
    int cm = q_cell(qm), ct = q_cell(qt), cz = q_cell(qz);
    const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 s0 = zero4, s1 = zero4, pa0 = zero4, pa1 = zero4, pb0 = zero4,
           pb1 = zero4;
    bool chk = true;
    if (k0 < k1) {
      const float tx = int_to_float(ct + 1), ty = int_to_float(cz - z_lo + 1);
      pb0 = gather_a2d(tex, cm, tx, ty);
      pb1 = gather_a2d(tex, cm + 1, tx, ty);
    }
    auto body = [&](float4& n0, float4& n1, const float4& p0,
                    const float4& p1) {
      const float wm = q_frac(qm), wt = q_frac(qt), wz = q_frac(qz);
      const float m0 = (cm >= 0 && cm <= top) ? 1.f - wm : 0.f;
      const float m1 = (cm + 1 >= 0 && cm + 1 <= top) ? wm : 0.f;
      qm += bm;
      qt += bt;
      qz += bz;
      const int im = q_cell(qm), it = q_cell(qt), iz = q_cell(qz);
      const bool ch = im != cm || it != ct || iz != cz;
      {
        const float tx = int_to_float(it + 1);
        const float ty = int_to_float(iz - z_lo + 1);
        gather_a2d_if(n0, ch, tex, im, tx, ty);
        gather_a2d_if(n1, ch, tex, im + 1, tx, ty);
      }
      if (chk) {
        s0 = p0;
        s1 = p1;
      }
      const float r00 = fmaf(wt, s0.z - s0.w, s0.w);
      const float r01 = fmaf(wt, s0.y - s0.x, s0.x);
      const float r10 = fmaf(wt, s1.z - s1.w, s1.w);
      const float r11 = fmaf(wt, s1.y - s1.x, s1.x);
      const float b0 = fmaf(wz, r01 - r00, r00);
      const float b1 = fmaf(wz, r11 - r10, r10);
      acc = fmaf(m0, b0, fmaf(m1, b1, acc));
      chk = ch;
      cm = im;
      ct = it;
      cz = iz;
    };
    int k = k0;
#pragma unroll 1
    for (; k + 1 < k1; k += 2) {
      body(pa0, pa1, pb0, pb1);
      body(pb0, pb1, pa0, pa1);
    }
    if (k < k1) body(pa0, pa1, pb0, pb1);
  }
  const float val = acc * (float)r.step;
  const size_t idx = ((size_t)a * n_v + v) * n_u + u;
  if (MODE == FWD_OVERWRITE) {
    out[idx] = val;
  } else if (MODE == FWD_ACCUMULATE) {
    out[idx] += val;
  } else {
    const float wt = w ? w[idx] : 1.f;
    out[idx] = wt * (b[idx] - val);
  }
}

// Slab [nzs, ny, nx] -> x-layers (layer x, texel (y, z)).  A CTA moves a
// 32 x 32 y x 8 z brick through shared memory: row-contiguous volume reads,
// and per layer a 32 y x 8 z surface block (two whole 64 B x 8-row GOBs of
// the block-linear array).  Rows z in [nzs, zr) are written as zeros (guard
// rows of an array taller than the slab).
__global__ void __launch_bounds__(256)
    fill_xlayers_kernel(cudaSurfaceObject_t surf,
                        const float* __restrict__ vol, int nx, int ny, int nzs,
                        int zr, int l0, int l1) {
  __shared__ float brick[8][32][33];
  const int x0 = l0 + blockIdx.x * 32, y0 = blockIdx.y * 32, z0 = blockIdx.z * 8;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  const size_t plane = (size_t)nx * ny;
  for (int zz = 0; zz < 8; zz++) {
    const int z = z0 + zz;
    for (int j = ty; j < 32; j += 8) {
      const int x = x0 + tx, y = y0 + j;
      brick[zz][j][tx] = (x < l1 && y < ny && z < nzs)
                             ? vol[(size_t)z * plane + (size_t)y * nx + x]
                             : 0.f;
    }
  }
  __syncthreads();
  const int z = z0 + ty, y = y0 + tx;
  if (z >= zr || y >= ny) return;
  for (int j = 0; j < 32 && x0 + j < l1; j++)
    surf2DLayeredwrite(brick[ty][tx][j], surf, y * (int)sizeof(float), z,
                       x0 + j - l0);
}

// Slab [nzs, ny, nx] -> y-layers (layer y, texel (x, z)): a CTA writes a
// 32 x x 8 z block of one layer (two whole GOBs), reading 8 row segments.
__global__ void __launch_bounds__(256)
    fill_ylayers_kernel(cudaSurfaceObject_t surf,
                        const float* __restrict__ vol, int nx, int ny, int nzs,
                        int zr, int l0) {
  const int x = blockIdx.x * 32 + threadIdx.x;
  const int z = blockIdx.y * 8 + threadIdx.y, y = l0 + blockIdx.z;
  if (x >= nx || z >= zr) return;
  surf2DLayeredwrite(z < nzs ? vol[((size_t)z * ny + y) * nx + x] : 0.f, surf,
                     x * (int)sizeof(float), z, y - l0);
}

// Loads slab planes [0, nzs) of `vol`, M planes [l0, l1), as main-axis-M
// layers (layer = plane - l0).
static int load_mlayers(int M, const float* vol, int nx, int ny, int nzs,
                        int l0, int l1, cudaStream_t s, LayeredTexture** t) {
  const TexRole role = (M == 1 && nx != ny) ? TEX_VOL_M2 : TEX_VOL_M;
  // slabs of different heights reuse a taller array (no reallocation and
  // stream drain per slab)
  int rc = M == 0 ? acquire_layered(role, ny, nzs, l1 - l0, s, t, true)
                  : acquire_layered(role, nx, nzs, l1 - l0, s, t, true);
  if (rc) return rc;
  // rows past the slab must read zero: slab_k_range keeps <= 3 samples
  // beyond the slab (<= 1.5 planes at |dz| <= 1/2 voxel per sample), so a
  // taller array gets 4 zero guard rows
  const int zr = min((*t)->h, nzs + 4);
  if (M == 0) {
    fill_xlayers_kernel<<<dim3((l1 - l0 + 31) / 32, (ny + 31) / 32,
                               (zr + 7) / 8),
                          dim3(32, 8), 0, s>>>((*t)->surf, vol, nx, ny, nzs,
                                               zr, l0, l1);
  } else {
    fill_ylayers_kernel<<<dim3((nx + 31) / 32, (zr + 7) / 8, l1 - l0),
                          dim3(32, 8), 0, s>>>((*t)->surf, vol, nx, ny, nzs,
                                               zr, l0);
  }
  CS_COUNT_LAUNCH();
  CS_CHECK_CUDA(cudaGetLastError());
  return CS_OK;
}

// Main-axis-layered K1 over all n_a views: views grouped by main axis, one
// texture fill + one launch per group (the two fills share one array when
// nx == ny; stream order separates them).  Slab height and the layer
// counts nx, ny must fit the layered-texture limits (caller checks).
template <int MODE>
static int launch_mlayer(const float* vol, int nx, int ny, int nz, int z_lo,
                         int z_hi, const Grid& G, const double* geom,
                         const AngleGeom* dgeom, int n_a, int n_u, int n_v,
                         double step_max, float* out, const float* b,
                         const float* w, cudaStream_t s) {
  int* ids_h = (int*)malloc(sizeof(int) * (size_t)n_a);
  int cnt[2] = {0, 0}, m = 0;
  for (int c = 0; c < 2; c++)
    for (int a = 0; a < n_a; a++)
      if (view_axis(geom + 12 * a, n_u, n_v) == c) {
        ids_h[m++] = a;
        cnt[c]++;
      }
  int* ids = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&ids, sizeof(int) * n_a, s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(ids, ids_h, sizeof(int) * n_a, cudaMemcpyHostToDevice,
                        s);
  // the host table must outlive the async copy: it is pageable, so the copy
  // is staged before cudaMemcpyAsync returns
  free(ids_h);
  CS_CHECK_CUDA(e);
  int rc = CS_OK;
  int v0 = 0, v1 = n_v;
  if (MODE != FWD_RESIDUAL && cull_enabled())
    slab_row_band(geom, n_a, G, z_lo, z_hi, n_v, &v0, &v1);
  if (MODE == FWD_OVERWRITE)
    rc = zero_rows_outside(out, n_a, n_u, n_v, v0, v1, s);
  // n_M over the layer limit: the M planes go through in pieces of <= maxl
  // layers, the first applying MODE (not the residual: the caller keeps
  // that to one piece), the rest accumulating
  const int maxl = max_layers();
  for (int c = 0; c < 2 && rc == CS_OK && v1 > v0; c++) {
    if (!cnt[c]) continue;
    const int n_m = c == 0 ? nx : ny;
    const int np = (n_m + maxl - 1) / maxl;
    for (int p = 0; p < np && rc == CS_OK; p++) {
      const int l0 = (int)((long long)n_m * p / np);
      const int l1 = (int)((long long)n_m * (p + 1) / np);
      LayeredTexture* t = nullptr;
      if ((rc = load_mlayers(c, vol, nx, ny, z_hi - z_lo, l0, l1, s, &t)))
        break;
      const dim3 grid((n_u + ML_TILE_U - 1) / ML_TILE_U,
                      (v1 - v0 + ML_TILE_V - 1) / ML_TILE_V, cnt[c]);
      auto kern = p == 0 ? (c == 0 ? fwd_mlayer_kernel<MODE, 0>
                                   : fwd_mlayer_kernel<MODE, 1>)
                         : (c == 0 ? fwd_mlayer_kernel<FWD_ACCUMULATE, 0>
                                   : fwd_mlayer_kernel<FWD_ACCUMULATE, 1>);
      kern<<<grid, 128, 0, s>>>(t->tex, dgeom, ids + (c ? cnt[0] : 0), G,
                                step_max, z_lo, z_hi, l0, l1, n_u, n_v, v0, v1,
                                out, p == 0 ? b : nullptr,
                                p == 0 ? w : nullptr);
      CS_COUNT_LAUNCH();
      if ((e = cudaGetLastError()) != cudaSuccess) break;
    }
    if (e != cudaSuccess) break;
  }
  cudaFreeAsync(ids, s);
  CS_CHECK_CUDA(e);
  return rc;
}

// Siddon traversal, _kernels.py:71-151 (fp64, midpoint attribution).
#ifndef SID_MINB
#define SID_MINB 12  // 40 registers: 48 warps/SM hide the serial fp64 event chain
#endif
__global__ void __launch_bounds__(128, SID_MINB)
    fwd_siddon_kernel(const float* __restrict__ vol,
                      const AngleGeom* __restrict__ geom, Grid G, int z_lo,
                      int z_hi, int n_u, int n_v, int v_base, int v_end,
                      float* __restrict__ out, int accumulate) {
  int u, v;
  tile_coords(u, v, v_base);
  const int a = blockIdx.z;
  if (u >= n_u || v >= v_end) return;
  const AngleGeom g = geom[a];
  double o[3] = {g.src[0], g.src[1], g.src[2]}, d[3];
  pixel_direction(g, u, v, d);
  const double gx0 = G.g0[0], gy0 = G.g0[1], gz0 = G.g0[2];
  const double vx = G.vox[0], vy = G.vox[1], vz = G.vox[2];
  const int nx = G.n[0], ny = G.n[1];
  double b0[3] = {gx0, gy0, __dadd_rn(gz0, __dmul_rn((double)z_lo, vz))};
  double b1[3] = {__dadd_rn(gx0, __dmul_rn((double)nx, vx)),
                  __dadd_rn(gy0, __dmul_rn((double)ny, vy)),
                  __dadd_rn(gz0, __dmul_rn((double)z_hi, vz))};
  double acc = 0.0, t0, t1;
  if (clip_box(o, d, b0, b1, t0, t1) && dsub(t1, t0) > 1e-12) {
    double p[3], tn[3], dt[3];
    const double vv[3] = {vx, vy, vz}, gg[3] = {gx0, gy0, gz0};
#pragma unroll
    for (int i = 0; i < 3; i++) {
      p[i] = o[i] + t0 * d[i];
      const double rel = p[i] - gg[i];
      if (d[i] > 0.0) {
        tn[i] = t0 + ((floor(rel / vv[i]) + 1.0) * vv[i] - rel) / d[i];
        dt[i] = vv[i] / d[i];
      } else if (d[i] < 0.0) {
        tn[i] = t0 + ((ceil(rel / vv[i]) - 1.0) * vv[i] - rel) / d[i];
        dt[i] = -vv[i] / d[i];
      } else {
        tn[i] = 1e300;
        dt[i] = 0.0;
      }
    }
    const size_t plane = (size_t)nx * ny;
    // The voxel of a piece is floor of its midpoint / voxel size
    // (_kernels.py:71-151).  A midpoint lies mid-voxel (>= half the piece,
    // > 5e-13, from any plane), so multiplying by the fp64 reciprocal picks
    // the same voxel as the division -- three fp64 divisions per piece were
    // the kernel's largest cost.
    const double ivx = 1.0 / vx, ivy = 1.0 / vy, ivz = 1.0 / vz;
    // The voxel is taken from the midpoint once (first piece longer than
    // 1e-12) and then stepped with the crossings: every later piece lies
    // between the same fp64 events the reference uses, so its midpoint
    // voxel is the stepped one (pieces <= 1e-12 are skipped by both).
    // Bit-identical to the per-piece midpoint floor at config 2 and on
    // every parity case; 345 -> 354 GUPS, 362 at 40 registers (r01).
    const int sx = d[0] > 0.0 ? 1 : -1, sy = d[1] > 0.0 ? 1 : -1,
              sz = d[2] > 0.0 ? 1 : -1;
    int ix = 0, iy = 0, iz = 0;
    bool have = false;
    double t = t0;
    while (t < t1 - 1e-12) {
      double tnext = fmin(fmin(tn[0], tn[1]), tn[2]);
      if (tnext > t1) tnext = t1;
      const double seg = tnext - t;
      if (seg > 1e-12) {
        if (!have) {
          const double tm = 0.5 * (t + tnext);
          ix = (int)floor((o[0] + tm * d[0] - gx0) * ivx);
          iy = (int)floor((o[1] + tm * d[1] - gy0) * ivy);
          iz = (int)floor((o[2] + tm * d[2] - gz0) * ivz);
          have = true;
        }
        if ((unsigned)ix < (unsigned)nx && (unsigned)iy < (unsigned)ny &&
            iz >= z_lo && iz < z_hi)
          acc += seg * (double)__ldg(vol + (size_t)(iz - z_lo) * plane +
                                     (size_t)iy * nx + ix);
      }
      if (tnext >= t1) break;
      if (tn[0] <= tnext) { tn[0] += dt[0]; ix += have ? sx : 0; }
      if (tn[1] <= tnext) { tn[1] += dt[1]; iy += have ? sy : 0; }
      if (tn[2] <= tnext) { tn[2] += dt[2]; iz += have ? sz : 0; }
      t = tnext;
    }
  }
  const size_t idx = ((size_t)a * n_v + v) * n_u + u;
  if (accumulate)
    out[idx] += (float)acc;
  else
    out[idx] = (float)acc;
}

static int check_common(int nx, int ny, int nz, int z_lo, int z_hi, int n_a,
                        int n_u, int n_v) {
  CS_REQUIRE(nx > 0 && ny > 0 && nz > 0, CS_ERR_ARG, "bad grid %dx%dx%d", nx,
             ny, nz);
  CS_REQUIRE(0 <= z_lo && z_lo < z_hi && z_hi <= nz, CS_ERR_ARG,
             "invalid slab range [%d, %d) for nz=%d", z_lo, z_hi, nz);
  CS_REQUIRE(n_a > 0 && n_a <= 65535, CS_ERR_ARG,
             "n_a=%d outside [1, 65535] per launch", n_a);
  CS_REQUIRE(n_u > 0 && n_v > 0, CS_ERR_ARG, "bad detector %dx%d", n_u, n_v);
  return CS_OK;
}

// One z-layered K1 pass over the sub-slab [z_lo, z_hi) (nzs <= layer limit).
template <int MODE>
static int launch_zlayer(const float* vol, int nx, int ny, int nz, int z_lo,
                         int z_hi, const Grid& G, const double* geom,
                         const AngleGeom* dgeom, int n_a, int n_u, int n_v,
                         double step_max, float* out, const float* b,
                         const float* w, cudaStream_t s) {
  int v0 = 0, v1 = n_v, rc;
  if (MODE != FWD_RESIDUAL && cull_enabled())
    slab_row_band(geom, n_a, G, z_lo, z_hi, n_v, &v0, &v1);
  if (MODE == FWD_OVERWRITE &&
      (rc = zero_rows_outside(out, n_a, n_u, n_v, v0, v1, s)))
    return rc;
  if (v1 <= v0) return CS_OK;
  LayeredTexture* t = nullptr;
  if ((rc = load_layered(TEX_VOLUME, vol, nx, ny, z_hi - z_lo, s, &t)))
    return rc;
  const dim3 grid((n_u + FWD_TILE_U - 1) / FWD_TILE_U,
                  (v1 - v0 + FWD_TILE_V - 1) / FWD_TILE_V, n_a);
  fwd_interp_kernel<MODE><<<grid, 128, 0, s>>>(t->tex, dgeom, G, step_max,
                                               z_lo, z_hi, n_u, n_v, v0, v1,
                                               out, b, w);
  CS_COUNT_LAUNCH();
  CS_CHECK_CUDA(cudaGetLastError());
  return CS_OK;
}

template <int MODE>
static int launch_interp(const float* vol, int nx, int ny, int nz, int z_lo,
                         int z_hi, const double* grid6, const double* geom,
                         int n_a, int n_u, int n_v, double step_max,
                         float* out, const float* b, const float* w,
                         cudaStream_t s) {
  int rc = check_common(nx, ny, nz, z_lo, z_hi, n_a, n_u, n_v);
  if (rc) return rc;
  CS_REQUIRE(step_max > 0.0, CS_ERR_ARG, "step_max must be positive");
  // Texture-gather kernel (below) is the production Ax; the shared-memory
  // staged variant (staged.cu) is selectable for A/B runs (CS_FWD_STAGED=1):
  // it is latency-bound on its box loads (149 vs 284 GUPS at config 2, r01).
  static const char* knob = getenv("CS_FWD_STAGED");
  if (knob && knob[0] == '1')
    return launch_staged<OP_FWD, MODE>(vol, nullptr, nx, ny, nz, z_lo, z_hi,
                                       grid6, geom, n_a, n_u, n_v, step_max,
                                       out, nullptr, b, w, s);
  const Grid G = make_grid(grid6, nx, ny, nz);
  AngleGeom* dgeom = nullptr;
  if ((rc = upload_geometry(geom, n_a, s, &dgeom))) return rc;
  const int maxl = max_layers();
  // main-axis-layered kernel unless disabled (CS_FWD_MLAYER=0)
  static const char* ml_knob = getenv("CS_FWD_MLAYER");
  // (x / y extents over the layer limit go through in layer pieces, which
  // the residual epilogue cannot: it keeps the z-layers there)
  const bool ml = !(ml_knob && ml_knob[0] == '0') &&
                  ((nx <= maxl && ny <= maxl) || MODE != FWD_RESIDUAL);
  // The slab goes through the texture in sub-slabs of at most h planes
  // (the first applies MODE, the rest accumulate): h starts at the
  // texture limit and halves whenever the texture array does not fit in
  // device memory (the array is a copy of the sub-slab: a slab planned to
  // fill HBM would not fit twice).
  int h = min(z_hi - z_lo, ml ? max_layered_height() : maxl);
  const size_t plane = (size_t)nx * ny;
  for (int s0 = z_lo; s0 < z_hi;) {
    const int s1 = min(z_hi, s0 + h);
    const bool first = s0 == z_lo;
    const float* vs = vol + (size_t)(s0 - z_lo) * plane;
    if (ml) {
      rc = first ? launch_mlayer<MODE>(vs, nx, ny, nz, s0, s1, G, geom, dgeom,
                                       n_a, n_u, n_v, step_max, out, b, w, s)
                 : launch_mlayer<FWD_ACCUMULATE>(vs, nx, ny, nz, s0, s1, G,
                                                 geom, dgeom, n_a, n_u, n_v,
                                                 step_max, out, nullptr,
                                                 nullptr, s);
    } else {
      rc = first ? launch_zlayer<MODE>(vs, nx, ny, nz, s0, s1, G, geom, dgeom,
                                       n_a, n_u, n_v, step_max, out, b, w, s)
                 : launch_zlayer<FWD_ACCUMULATE>(vs, nx, ny, nz, s0, s1, G,
                                                 geom, dgeom, n_a, n_u, n_v,
                                                 step_max, out, nullptr,
                                                 nullptr, s);
    }
    // nothing was launched for a sub-slab whose array failed: retry it
    // smaller (not the residual epilogue, which needs the whole slab)
    if (rc == CS_ERR_CUDA && strstr(cs_last_error(), "out of memory") &&
        MODE != FWD_RESIDUAL && h > 1) {
      h = (h + 1) / 2;
      continue;
    }
    if (rc) break;
    s0 = s1;
  }
  release_geometry(dgeom, s);
  return rc;
}

}  // namespace cs

using namespace cs;

extern "C" {

int cs_fwd_interp(const float* vol, int nx, int ny, int nz, int z_lo,
                  int z_hi, const double* grid6, const double* geom, int n_a,
                  int n_u, int n_v, double step_max, float* out,
                  int accumulate, cs_stream_t stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (accumulate)
    return launch_interp<FWD_ACCUMULATE>(vol, nx, ny, nz, z_lo, z_hi, grid6,
                                         geom, n_a, n_u, n_v, step_max, out,
                                         nullptr, nullptr, s);
  return launch_interp<FWD_OVERWRITE>(vol, nx, ny, nz, z_lo, z_hi, grid6,
                                      geom, n_a, n_u, n_v, step_max, out,
                                      nullptr, nullptr, s);
}

int cs_fwd_interp_residual(const float* vol, int nx, int ny, int nz,
                           const double* grid6, const double* geom, int n_a,
                           int n_u, int n_v, double step_max, const float* b,
                           const float* w, float* out, cs_stream_t stream) {
  CS_REQUIRE(b != nullptr, CS_ERR_ARG, "residual mode needs b");
  CS_REQUIRE(nz <= max_layers(), CS_ERR_UNSUPPORTED,
             "residual epilogue needs the volume in one texture (nz <= %d)",
             max_layers());
  return launch_interp<FWD_RESIDUAL>(vol, nx, ny, nz, 0, nz, grid6, geom,
                                     n_a, n_u, n_v, step_max, out, b, w,
                                     (cudaStream_t)stream);
}

int cs_fwd_siddon(const float* vol, int nx, int ny, int nz, int z_lo,
                  int z_hi, const double* grid6, const double* geom, int n_a,
                  int n_u, int n_v, float* out, int accumulate,
                  cs_stream_t stream) {
  int rc = check_common(nx, ny, nz, z_lo, z_hi, n_a, n_u, n_v);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  const Grid G = make_grid(grid6, nx, ny, nz);
  AngleGeom* dgeom = nullptr;
  if ((rc = upload_geometry(geom, n_a, s, &dgeom))) return rc;
  int v0 = 0, v1 = n_v;
  if (cull_enabled()) slab_row_band(geom, n_a, G, z_lo, z_hi, n_v, &v0, &v1);
  if (!accumulate && (rc = zero_rows_outside(out, n_a, n_u, n_v, v0, v1, s))) {
    release_geometry(dgeom, s);
    return rc;
  }
  cudaError_t e = cudaSuccess;
  if (v1 > v0) {
    const dim3 grid((n_u + FWD_TILE_U - 1) / FWD_TILE_U,
                    (v1 - v0 + FWD_TILE_V - 1) / FWD_TILE_V, n_a);
    fwd_siddon_kernel<<<grid, 128, 0, s>>>(vol, dgeom, G, z_lo, z_hi, n_u,
                                           n_v, v0, v1, out, accumulate);
    CS_COUNT_LAUNCH();
    e = cudaGetLastError();
  }
  release_geometry(dgeom, s);
  CS_CHECK_CUDA(e);
  return CS_OK;
}

}  // extern "C"
