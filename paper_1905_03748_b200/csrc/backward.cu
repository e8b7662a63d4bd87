// backward.cu -- Atb on sm_100a: the exact (matched) adjoint of the
// interpolated projector (K2) and the voxel-driven FDK backprojector (K3).
//
// K2 replaces the reference's single-threaded scatter
// (_kernels.py:278-337): the staged shared-memory kernel of staged.cu
// replays K1's ray set-up and sample lattice exactly (shared code in
// common.cuh); cs_bwd_matched below is its C-ABI entry.
//
// K3 replaces fdk_backward_chunk (_kernels.py:340-398): one thread per
// (x, y) column and FDK_ZB consecutive z voxels held in registers; the
// column-angle terms (U, magnification, u coordinate, (dso/U)^2) are fp64
// once per column and angle, the z walk is fp32 relative to an integer
// detector row so the v coordinate keeps ~1e-6 px accuracy; the 2x2
// detector footprint comes from one tld4 gather on a 2D-layered texture of
// the projections (layers = angles) with border = 0 (the reference's
// out-of-detector taps, :385-394).
#include <cstdlib>

#include "common.cuh"

namespace cs {

#ifndef CS_FDK_ZB
#define CS_FDK_ZB 16
#endif
constexpr int FDK_ZB = CS_FDK_ZB;  // z voxels per thread (registers)

__global__ void __launch_bounds__(128)
    bwd_fdk_kernel(cudaTextureObject_t tex, const double2* __restrict__ cs,
                   int n_a, double gx0, double gy0, double gz0, double vx,
                   double vy, double vz, int nx, int ny, int z_lo, int n_slab,
                   double dso, double dsd, double inv_du, double inv_dv,
                   double off_u, double off_v, int n_u, int n_v,
                   float* __restrict__ vol) {
  const int ix = blockIdx.x * 32 + threadIdx.x;
  const int iy = blockIdx.y * 4 + threadIdx.y;
  const int zb = blockIdx.z * FDK_ZB;
  if (ix >= nx || iy >= ny) return;
  // voxel centres, _kernels.py:364-368
  const double wx = gx0 + (ix + 0.5) * vx;
  const double wy = gy0 + (iy + 0.5) * vy;
  const double wz0 = gz0 + (z_lo + zb + 0.5) * vz;
  const double cu = 0.5 * (n_u - 1), cv = 0.5 * (n_v - 1);
  float acc[FDK_ZB];
#pragma unroll
  for (int j = 0; j < FDK_ZB; j++) acc[j] = 0.f;

  for (int a = 0; a < n_a; a++) {
    const double2 c_s = __ldg(cs + a);
    const double c = c_s.x, s = c_s.y;
    const double big_u = dso - (wx * c + wy * s);  // :373
    if (big_u <= 1e-9) continue;                   // :374-375
    const double rU = 1.0 / big_u;
    const double mag = dsd * rU;
    const double uf = ((-wx * s + wy * c) * mag - off_u) * inv_du + cu;
    const double vf = (wz0 * mag - off_v) * inv_dv + cv;
    const double wgt = dso * rU;
    const float w2 = (float)(wgt * wgt);
    const double fu0 = floor(uf), fv0 = floor(vf);
    const float fu = (float)(uf - fu0);
    const float xu = (float)fu0 + 1.f;
    const float vfrac = (float)(vf - fv0);
    const float vrow = (float)fv0 + 1.f;
    const float dvz = (float)(vz * mag * inv_dv);
#pragma unroll
    for (int j = 0; j < FDK_ZB; j++) {
      const float vv = fmaf((float)j, dvz, vfrac);
      const float fl = floorf(vv);
      const float fv = vv - fl;
      const float4 t = gather_a2d(tex, a, xu, vrow + fl);
      // t.w=(u0,v0) t.z=(u0+1,v0) t.x=(u0,v0+1) t.y=(u0+1,v0+1)
      const float r0 = fmaf(fu, t.z - t.w, t.w);
      const float r1 = fmaf(fu, t.y - t.x, t.x);
      acc[j] = fmaf(w2, fmaf(fv, r1 - r0, r0), acc[j]);
    }
  }
  const size_t plane = (size_t)nx * ny;
  float* col = vol + (size_t)iy * nx + ix;
#pragma unroll
  for (int j = 0; j < FDK_ZB; j++)
    if (zb + j < n_slab) col[(size_t)(zb + j) * plane] += acc[j];
}

// Staged FDK (production K3): CTA = 16 x 8 voxel columns x FDK_ZB z
// voxels; views are taken in batches of up to FS_NB whose detector
// footprints (the projective image of the CTA's voxel box, extremes at its
// corners, plus a one-pixel margin) are staged in shared memory with
// coalesced loads and zero outside the detector (the reference's border
// rule, _kernels.py:385-394).  The bilinear taps are then 4 shared loads
// instead of one texture gather: the texture path is bound by its 16-byte
// writeback per voxel-view (ncu: tex writeback 99.7%, issue 28%).
// 7 CTAs/SM x 28 KB footprint buffers (r01 A/B at config 2: 6 x 32 KB 892
// GUPS, 7 x 28 KB 917, 8 x 24 / 20 KB 883 / 894 -- spills at 64 registers)
#ifndef FS_MINB
#define FS_MINB 7
#endif
#ifndef CS_FS_CAP
#define CS_FS_CAP 7168
#endif
// (A/B, -DCS_FS_PAIRS=1) footprint staged as column pairs, one LDS.64 per
// bilinear row instead of two LDS: 826 vs 896 GUPS at config 2 (twice the
// staging loads and 8-byte shared rows), not kept
// (profiles/ab_fdk_pairs_r02ci.jsonl)
#ifndef CS_FS_PAIRS
#define CS_FS_PAIRS 0
#endif
constexpr int FS_TX = 16, FS_TY = 8, FS_NB = 16, FS_CAP = CS_FS_CAP;

struct FsBox {
  int u0, v0, nu, nv, off;
};

__global__ void __launch_bounds__(FS_TX * FS_TY, FS_MINB)
    fdk_staged_kernel(const float* __restrict__ proj,
                      const double2* __restrict__ cs, int n_a, double gx0,
                      double gy0, double gz0, double vx, double vy, double vz,
                      int nx, int ny, int z_lo, int n_slab, double dso,
                      double dsd, double inv_du, double inv_dv, double off_u,
                      double off_v, int n_u, int n_v,
                      float* __restrict__ vol) {
#if CS_FS_PAIRS
  // footprint as column pairs (t[v][u], t[v][u + 1]): one LDS.64 per
  // bilinear row instead of two LDS
  __shared__ float2 sbox2[FS_CAP / 2];
#else
  __shared__ float sbox[FS_CAP];
#endif
  __shared__ FsBox sb[FS_NB];
  __shared__ int s_m;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * FS_TX + tx;
  const int bx0 = blockIdx.x * FS_TX, by0 = blockIdx.y * FS_TY;
  const int ix = bx0 + tx, iy = by0 + ty;
  const int zb = blockIdx.z * FDK_ZB;
  const bool own = ix < nx && iy < ny;
  const double wx = gx0 + (ix + 0.5) * vx;
  const double wy = gy0 + (iy + 0.5) * vy;
  const double wz0 = gz0 + (z_lo + zb + 0.5) * vz;
  const double cu = 0.5 * (n_u - 1), cv = 0.5 * (n_v - 1);
  const size_t sheet = (size_t)n_u * n_v;
  // tile corners (voxel centres) for the footprint boxes
  const int xl = min(bx0 + FS_TX, nx) - 1, yl = min(by0 + FS_TY, ny) - 1;
  const int zl = min(zb + FDK_ZB, n_slab) - 1;
  const int nk = zl - zb + 1;  // planes of this CTA inside the slab
  const double cxs[2] = {gx0 + (bx0 + 0.5) * vx, gx0 + (xl + 0.5) * vx};
  const double cys[2] = {gy0 + (by0 + 0.5) * vy, gy0 + (yl + 0.5) * vy};
  const double czs[2] = {wz0, gz0 + (z_lo + zl + 0.5) * vz};
  float acc[FDK_ZB];
#pragma unroll
  for (int j = 0; j < FDK_ZB; j++) acc[j] = 0.f;

  int a0 = 0;
  while (a0 < n_a) {
    __syncthreads();  // previous batch consumed
    if (tid < FS_NB) {
      FsBox b = {0, 0, 0, 0, 0};
      const int a = a0 + tid;
      if (a < n_a) {
        const double2 c_s = __ldg(cs + a);
        double umin = 1e300, umax = -1e300, vmin = 1e300, vmax = -1e300;
        bool ok = true;
        for (int i = 0; i < 4; i++) {
          const double x = cxs[i & 1], y = cys[i >> 1];
          const double U = dso - (x * c_s.x + y * c_s.y);
          if (U <= 1e-9) {
            ok = false;
            break;
          }
          const double mag = dsd / U;
          const double uf = ((-x * c_s.y + y * c_s.x) * mag - off_u) * inv_du + cu;
          umin = fmin(umin, uf);
          umax = fmax(umax, uf);
          for (int k = 0; k < 2; k++) {
            const double vf = (czs[k] * mag - off_v) * inv_dv + cv;
            vmin = fmin(vmin, vf);
            vmax = fmax(vmax, vf);
          }
        }
        if (ok) {
          b.u0 = (int)floor(umin) - 1;
          b.v0 = (int)floor(vmin) - 1;
          b.nu = (int)floor(umax) + 3 - b.u0;
          b.nv = (int)floor(vmax) + 3 - b.v0;
          if (b.nu > 4096 || b.nv > 4096) b.nu = b.nv = 4096;  // too big
        } else {
          b.nu = b.nv = 4096;  // degenerate view: direct path
        }
      }
      sb[tid] = b;
    }
    __syncthreads();
    if (tid == 0) {
      int off = 0, m = 0;
      for (; m < FS_NB && a0 + m < n_a; m++) {
        const int sz = sb[m].nu * sb[m].nv;
        if (off + sz > (CS_FS_PAIRS ? FS_CAP / 2 : FS_CAP)) break;
        sb[m].off = off;
        off += sz;
      }
      s_m = m;  // 0: the next view alone exceeds the buffer
    }
    __syncthreads();
    const int m = s_m;
    if (m > 0) {
      for (int j = 0; j < m; j++) {
        const FsBox b = sb[j];
        const float* pj = proj + (size_t)(a0 + j) * sheet;
        // element e = tid + 128 i -> (row r, column c): one division for
        // the first, then an incremental walk (integer division goes
        // through the XU pipe, the kernel's busiest)
        constexpr int NT = FS_TX * FS_TY;
        int r = tid / b.nu, c = tid - r * b.nu;
        const int dr = NT / b.nu, dc = NT - dr * b.nu;
        for (int e = tid; e < b.nu * b.nv; e += NT) {
          const int u = b.u0 + c, v = b.v0 + r;
#if CS_FS_PAIRS
          const bool vin = v >= 0 && v < n_v;
          const float* rowp = pj + (size_t)v * n_u;
          sbox2[b.off + e] = make_float2(
              (vin && u >= 0 && u < n_u) ? __ldg(rowp + u) : 0.f,
              (vin && u + 1 >= 0 && u + 1 < n_u) ? __ldg(rowp + u + 1) : 0.f);
#else
          sbox[b.off + e] = (u >= 0 && u < n_u && v >= 0 && v < n_v)
                                ? __ldg(pj + (size_t)v * n_u + u)
                                : 0.f;
#endif
          c += dc;
          r += dr;
          if (c >= b.nu) {
            c -= b.nu;
            r++;
          }
        }
      }
      __syncthreads();
      if (own) {
        for (int j = 0; j < m; j++) {
          const double2 c_s = __ldg(cs + a0 + j);
          const double c = c_s.x, s = c_s.y;
          const double big_u = dso - (wx * c + wy * s);  // :373
          if (big_u <= 1e-9) continue;                   // :374-375
          const double rU = 1.0 / big_u;
          const double mag = dsd * rU;
          const double uf = ((-wx * s + wy * c) * mag - off_u) * inv_du + cu;
          const double vf = (wz0 * mag - off_v) * inv_dv + cv;
          const double wgt = dso * rU;
          const float w2 = (float)(wgt * wgt);
          const double fu0 = floor(uf), fv0 = floor(vf);
          const float fu = (float)(uf - fu0);
          const float vfrac = (float)(vf - fv0);
          // rows per plane split into integer rows + fraction, so the fp32
          // walk only carries the fraction (fine pixels: ~9 rows per plane,
          // ulp(16 x 9) would be 1.5e-5 of a row at the 16th plane)
          const double dvd = vz * mag * inv_dv;
          const double dvi = floor(dvd);
          const int di = (int)dvi;
          const float dvz = (float)(dvd - dvi);
          const FsBox b = sb[j];
          const int col = (int)fu0 - b.u0;
          const int row0 = (int)fv0 - b.v0;
#if CS_FS_PAIRS
          const float2* base = sbox2 + b.off + col;
#else
          const float* base = sbox + b.off + col;
#endif
          const f32x2 fu2 = f2(fu, fu);
          auto tap = [&](int k) {
            const float vv = fmaf((float)k, dvz, vfrac);
            // floor by the 1.5 * 2^23 magic add rounded toward -inf (one
            // FADD.RM on the FMA pipe instead of FRND on the conversion
            // pipe): mb = 1.5 * 2^23 + floor(vv) exactly for |vv| < 2^22,
            // its low mantissa bits the integer, mb - 1.5 * 2^23 == floorf
            const float mb = __fadd_rd(vv, 12582912.f);
            const float fl = mb - 12582912.f;
            const float fv = vv - fl;
            const int il = __float_as_int(mb) - 0x4B400000 + k * di;
#if CS_FS_PAIRS
            const float2* q = base + (row0 + il) * b.nu;
            const float2 qa = q[0], qb = q[b.nu];
            const float t00 = qa.x, t01 = qa.y, t10 = qb.x, t11 = qb.y;
#else
            const float* q = base + (row0 + il) * b.nu;
            const float t00 = q[0], t01 = q[1];
            const float t10 = q[b.nu], t11 = q[b.nu + 1];
#endif
            // both row lerps in one FADD2 + FFMA2 (bit-identical to the
            // scalar fmaf(fu, t01 - t00, t00), fmaf(fu, t11 - t10, t10))
            const f32x2 lo = f2(t00, t10);
            float r0, r1;
            f2_split(f2_fma(fu2, f2_sub(f2(t01, t11), lo), lo), r0, r1);
            acc[k] = fmaf(w2, fmaf(fv, r1 - r0, r0), acc[k]);
          };
          if (nk == FDK_ZB) {
#pragma unroll
            for (int k = 0; k < FDK_ZB; k++) tap(k);
          } else {
            // the slab's last z-block: planes past the slab lie outside the
            // staged footprint (its z range is the slab's), so they are
            // not sampled (CTA-uniform branch)
#pragma unroll
            for (int k = 0; k < FDK_ZB; k++)
              if (k < nk) tap(k);
          }
        }
      }
      a0 += m;
    } else {
      // one view whose footprint exceeds the buffer: direct global gather
      if (own) {
        const double2 c_s = __ldg(cs + a0);
        const double c = c_s.x, s = c_s.y;
        const double big_u = dso - (wx * c + wy * s);
        if (big_u > 1e-9) {
          const double rU = 1.0 / big_u;
          const double mag = dsd * rU;
          const double uf = ((-wx * s + wy * c) * mag - off_u) * inv_du + cu;
          const double wgt = dso * rU;
          const float w2 = (float)(wgt * wgt);
          const int u0 = (int)floor(uf);
          const float fu = (float)(uf - floor(uf));
          const float* pj = proj + (size_t)a0 * sheet;
#pragma unroll
          for (int k = 0; k < FDK_ZB; k++) {
            const double vf =
                ((wz0 + k * vz) * mag - off_v) * inv_dv + cv;
            const int v0 = (int)floor(vf);
            const float fv = (float)(vf - floor(vf));
            float t[4];
#pragma unroll
            for (int q = 0; q < 4; q++) {
              const int u = u0 + (q & 1), v = v0 + (q >> 1);
              t[q] = (u >= 0 && u < n_u && v >= 0 && v < n_v)
                         ? __ldg(pj + (size_t)v * n_u + u)
                         : 0.f;
            }
            const float r0 = fmaf(fu, t[1] - t[0], t[0]);
            const float r1 = fmaf(fu, t[3] - t[2], t[2]);
            acc[k] = fmaf(w2, fmaf(fv, r1 - r0, r0), acc[k]);
          }
        }
      }
      a0 += 1;
    }
  }
  if (own) {
    const size_t plane = (size_t)nx * ny;
    float* col = vol + (size_t)iy * nx + ix;
#pragma unroll
    for (int j = 0; j < FDK_ZB; j++)
      if (zb + j < n_slab) col[(size_t)(zb + j) * plane] += acc[j];
  }
}

__global__ void ray_table_kernel(const AngleGeom* __restrict__ geom, Grid G,
                                 double step_max, int n_u, int n_v,
                                 double* t0, double* step, int64_t* n) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y;
  const int a = blockIdx.z;
  if (u >= n_u) return;
  Ray r;
  setup_ray(geom[a], G, step_max, u, v, r);
  const size_t i = ((size_t)a * n_v + v) * n_u + u;
  t0[i] = r.t0;
  step[i] = r.step;
  n[i] = r.n;
}

}  // namespace cs

using namespace cs;

extern "C" {

int cs_bwd_matched(float* vol_acc, int nx, int ny, int nz, int z_lo,
                   int z_hi, const double* grid6, const double* geom, int n_a,
                   int n_u, int n_v, double step_max, const float* proj,
                   cs_stream_t stream) {
  CS_REQUIRE(nx > 0 && ny > 0 && nz > 0, CS_ERR_ARG, "bad grid");
  CS_REQUIRE(0 <= z_lo && z_lo < z_hi && z_hi <= nz, CS_ERR_ARG,
             "invalid slab range [%d, %d) for nz=%d", z_lo, z_hi, nz);
  CS_REQUIRE(n_a > 0 && n_a <= 65535 && n_u > 0 && n_v > 0, CS_ERR_ARG,
             "bad projection shape");
  CS_REQUIRE(step_max > 0.0, CS_ERR_ARG, "step_max must be positive");
  // staged shared-memory boxes (staged.cu)
  return launch_staged<OP_BWD, 0>(nullptr, vol_acc, nx, ny, nz, z_lo, z_hi,
                                  grid6, geom, n_a, n_u, n_v, step_max,
                                  nullptr, proj, nullptr, nullptr,
                                  (cudaStream_t)stream);
}

int cs_bwd_fdk(float* vol_acc, int nx, int ny, int z_lo, int n_slab,
               const double* grid6, const double* cs_host, int n_a,
               double dso, double dsd, double du, double dv, double off_u,
               double off_v, int n_u, int n_v, const float* proj,
               cs_stream_t stream) {
  CS_REQUIRE(nx > 0 && ny > 0 && n_slab > 0 && z_lo >= 0, CS_ERR_ARG,
             "bad slab");
  CS_REQUIRE(n_a > 0 && n_u > 0 && n_v > 0, CS_ERR_ARG,
             "bad projection shape");
  CS_REQUIRE(du > 0 && dv > 0, CS_ERR_ARG, "pixel sizes must be positive");
  cudaStream_t s = (cudaStream_t)stream;
  double2* dcs = nullptr;
  CS_CHECK_CUDA(cudaMallocAsync((void**)&dcs, sizeof(double2) * n_a, s));
  CS_CHECK_CUDA(cudaMemcpyAsync(dcs, cs_host, sizeof(double2) * n_a,
                                cudaMemcpyHostToDevice, s));
  int rc = CS_OK;
  static const char* tex_knob = getenv("CS_FDK_TEX");
  if (!(tex_knob && tex_knob[0] == '1')) {
    const dim3 grid((nx + FS_TX - 1) / FS_TX, (ny + FS_TY - 1) / FS_TY,
                    (n_slab + FDK_ZB - 1) / FDK_ZB);
    fdk_staged_kernel<<<grid, dim3(FS_TX, FS_TY), 0, s>>>(
        proj, dcs, n_a, grid6[0], grid6[1], grid6[2], grid6[3], grid6[4],
        grid6[5], nx, ny, z_lo, n_slab, dso, dsd, 1.0 / du, 1.0 / dv, off_u,
        off_v, n_u, n_v, vol_acc);
    CS_COUNT_LAUNCH();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      set_error("bwd_fdk launch: %s", cudaGetErrorString(e));
      rc = CS_ERR_CUDA;
    }
    cudaFreeAsync(dcs, s);
    return rc;
  }
  // texture-gather variant (A/B: CS_FDK_TEX=1)
  const dim3 block(32, 4);
  const dim3 grid((nx + 31) / 32, (ny + 3) / 4,
                  (n_slab + FDK_ZB - 1) / FDK_ZB);
  const int maxl = max_layers();
  const size_t sheet = (size_t)n_u * n_v;
  for (int a0 = 0; a0 < n_a && rc == CS_OK; a0 += maxl) {
    const int na = min(maxl, n_a - a0);
    LayeredTexture* t = nullptr;
    rc = load_layered(TEX_PROJ, proj + (size_t)a0 * sheet, n_u, n_v, na, s,
                      &t);
    if (rc) break;
    bwd_fdk_kernel<<<grid, block, 0, s>>>(
        t->tex, dcs + a0, na, grid6[0], grid6[1], grid6[2], grid6[3],
        grid6[4], grid6[5], nx, ny, z_lo, n_slab, dso, dsd, 1.0 / du,
        1.0 / dv, off_u, off_v, n_u, n_v, vol_acc);
    CS_COUNT_LAUNCH();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      set_error("bwd_fdk launch: %s", cudaGetErrorString(e));
      rc = CS_ERR_CUDA;
    }
  }
  cudaFreeAsync(dcs, s);
  return rc;
}

int cs_ray_table(int nx, int ny, int nz, const double* grid6,
                 const double* geom, int n_a, int n_u, int n_v,
                 double step_max, double* t0, double* step, int64_t* n,
                 cs_stream_t stream) {
  CS_REQUIRE(n_a > 0 && n_a <= 65535 && n_v <= 65535, CS_ERR_ARG,
             "bad shape");
  cudaStream_t s = (cudaStream_t)stream;
  const Grid G = make_grid(grid6, nx, ny, nz);
  AngleGeom* dgeom = nullptr;
  int rc = upload_geometry(geom, n_a, s, &dgeom);
  if (rc) return rc;
  ray_table_kernel<<<dim3((n_u + 127) / 128, n_v, n_a), 128, 0, s>>>(
      dgeom, G, step_max, n_u, n_v, t0, step, n);
  CS_COUNT_LAUNCH();
  cudaError_t e = cudaGetLastError();
  release_geometry(dgeom, s);
  CS_CHECK_CUDA(e);
  return CS_OK;
}

}  // extern "C"
