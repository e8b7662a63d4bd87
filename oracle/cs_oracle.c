/*
 * cs_oracle.c -- CPU restatement of the reference's projection kernels.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU
 * baseline ("kind": "port") for the B200 build; it is never linked into the
 * product library.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.
 *
 * It restates, operation for operation, the numba kernels of
 * /root/reference/pkg/src/conesplit/_kernels.py with float64 accumulation
 * (the reference's "accumulate in fp64, store in fp32" contract,
 * _kernels.py:3-13).  Every function cites the reference lines it follows.
 * Arithmetic is kept in the reference's evaluation order and compiled
 * without FP contraction (-ffp-contract=off) so that results are the
 * reference's bits (pinned by tests/golden, generated from the reference
 * itself by tests/golden/make_golden.py).
 *
 * Geometry arrives flattened exactly like the reference's _flat_geometry
 * (projectors.py:172-194): per angle 12 doubles
 *     src[3], det00[3], ustep[3], vstep[3]
 * and the grid as 6 doubles gx0, gy0, gz0, vx, vy, vz (projectors.py:197-202).
 *
 * Parallelism: OpenMP over detector rows (forward), over z bands (matched
 * scatter; each thread owns a z band and replays every ray in the
 * reference's fixed (angle, v, u, k, corner) order, so every voxel sees
 * the reference's accumulation order -- _kernels.py:284-285), and over
 * x-y columns (FDK).
 */
#include <math.h>
#include <stdint.h>
#include <omp.h>

#define EPS_LEN 1e-12 /* _kernels.py:25 */

/* _kernels.py:28-68 -- slab-method ray/box clip; miss when t0 > t1. */
static void clip_box(double ox, double oy, double oz, double dx, double dy,
                     double dz, double bx0, double by0, double bz0, double bx1,
                     double by1, double bz1, double *t0o, double *t1o) {
  double t0 = -1e300, t1 = 1e300, ta, tb, tmp;
  if (dx != 0.0) {
    ta = (bx0 - ox) / dx;
    tb = (bx1 - ox) / dx;
    if (ta > tb) { tmp = ta; ta = tb; tb = tmp; }
    if (ta > t0) t0 = ta;
    if (tb < t1) t1 = tb;
  } else if (ox < bx0 || ox > bx1) {
    *t0o = 1.0; *t1o = -1.0; return;
  }
  if (dy != 0.0) {
    ta = (by0 - oy) / dy;
    tb = (by1 - oy) / dy;
    if (ta > tb) { tmp = ta; ta = tb; tb = tmp; }
    if (ta > t0) t0 = ta;
    if (tb < t1) t1 = tb;
  } else if (oy < by0 || oy > by1) {
    *t0o = 1.0; *t1o = -1.0; return;
  }
  if (dz != 0.0) {
    ta = (bz0 - oz) / dz;
    tb = (bz1 - oz) / dz;
    if (ta > tb) { tmp = ta; ta = tb; tb = tmp; }
    if (ta > t0) t0 = ta;
    if (tb < t1) t1 = tb;
  } else if (oz < bz0 || oz > bz1) {
    *t0o = 1.0; *t1o = -1.0; return;
  }
  if (t0 > t1) { *t0o = 1.0; *t1o = -1.0; return; }
  *t0o = t0; *t1o = t1;
}

/* Unit ray direction from the source through pixel (u, v) of angle row g;
 * _kernels.py:234-243 (same in :179-188 and :297-306). */
static void pixel_dir(const double *g, int u, int v, double *dx, double *dy,
                      double *dz) {
  double tx = g[3] + u * g[6] + v * g[9];
  double ty = g[4] + u * g[7] + v * g[10];
  double tz = g[5] + u * g[8] + v * g[11];
  double x = tx - g[0], y = ty - g[1], z = tz - g[2];
  double inv = 1.0 / sqrt(x * x + y * y + z * z);
  *dx = x * inv; *dy = y * inv; *dz = z * inv;
}

/* _kernels.py:194-210 -- sample count and step against the FULL grid box. */
static void ray_steps(double ox, double oy, double oz, double dx, double dy,
                      double dz, const double *grid, int nx, int ny, int nz,
                      double step_max, double *t0o, double *stepo,
                      int64_t *no) {
  double t0, t1;
  clip_box(ox, oy, oz, dx, dy, dz, grid[0], grid[1], grid[2],
           grid[0] + nx * grid[3], grid[1] + ny * grid[4],
           grid[2] + nz * grid[5], &t0, &t1);
  double length = t1 - t0;
  if (t0 > t1 || length <= EPS_LEN) {
    *t0o = 0.0; *stepo = 0.0; *no = 0; return;
  }
  int64_t n = (int64_t)ceil(length / step_max);
  *t0o = t0; *stepo = length / (double)n; *no = n;
}

/* _kernels.py:213-275 -- trilinear-sampled forward projection of a slab.
 * vol is [z_hi - z_lo, ny, nx]; out is [n_a, n_v, n_u] (overwritten). */
int orc_fwd_interp(const float *vol, int nx, int ny, int nz, int z_lo,
                   int z_hi, const double *grid, const double *geom, int n_a,
                   int n_u, int n_v, double step_max, float *out,
                   int nthreads) {
  const double gx0 = grid[0], gy0 = grid[1], gz0 = grid[2];
  const double vx = grid[3], vy = grid[4], vz = grid[5];
  const int64_t plane = (int64_t)nx * ny;
#pragma omp parallel for collapse(2) schedule(dynamic, 1) num_threads(nthreads)
  for (int a = 0; a < n_a; a++)
    for (int v = 0; v < n_v; v++) {
      const double *g = geom + 12 * a;
      const double ox = g[0], oy = g[1], oz = g[2];
      for (int u = 0; u < n_u; u++) {
        double dx, dy, dz, t0, step;
        int64_t n;
        pixel_dir(g, u, v, &dx, &dy, &dz);
        ray_steps(ox, oy, oz, dx, dy, dz, grid, nx, ny, nz, step_max, &t0,
                  &step, &n);
        double acc = 0.0;
        for (int64_t k = 0; k < n; k++) {
          double t = t0 + ((double)k + 0.5) * step;
          double qx = (ox + t * dx - gx0) / vx - 0.5;
          double qy = (oy + t * dy - gy0) / vy - 0.5;
          double qz = (oz + t * dz - gz0) / vz - 0.5;
          double fx0 = floor(qx), fy0 = floor(qy), fz0 = floor(qz);
          int ix0 = (int)fx0, iy0 = (int)fy0, iz0 = (int)fz0;
          double wx = qx - ix0, wy = qy - iy0, wz = qz - iz0;
          for (int cz = 0; cz < 2; cz++) {
            int zi = iz0 + cz;
            if (zi < z_lo || zi >= z_hi) continue;
            double fz = cz == 1 ? wz : 1.0 - wz;
            for (int cy = 0; cy < 2; cy++) {
              int yi = iy0 + cy;
              if (yi < 0 || yi >= ny) continue;
              double fy = cy == 1 ? wy : 1.0 - wy;
              for (int cx = 0; cx < 2; cx++) {
                int xi = ix0 + cx;
                if (xi < 0 || xi >= nx) continue;
                double fx = cx == 1 ? wx : 1.0 - wx;
                acc += fz * fy * fx *
                       (double)vol[(int64_t)(zi - z_lo) * plane +
                                   (int64_t)yi * nx + xi];
              }
            }
          }
        }
        out[((int64_t)a * n_v + v) * n_u + u] = (float)(acc * step);
      }
    }
  return 0;
}

/* _kernels.py:278-337 -- exact adjoint of orc_fwd_interp, scattered into
 * the float64 slab accumulator vol64 [z_hi - z_lo, ny, nx] (accumulates).
 * Each thread owns a z band and walks every ray in the reference's order,
 * so the per-voxel summation order is the reference's single-thread one. */
int orc_bwd_matched(double *vol64, int nx, int ny, int nz, int z_lo, int z_hi,
                    const double *grid, const double *geom, int n_a, int n_u,
                    int n_v, double step_max, const float *proj,
                    int nthreads) {
  const double gx0 = grid[0], gy0 = grid[1], gz0 = grid[2];
  const double vx = grid[3], vy = grid[4], vz = grid[5];
  const int64_t plane = (int64_t)nx * ny;
  const int n_slab = z_hi - z_lo;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > n_slab) nthreads = n_slab;
#pragma omp parallel num_threads(nthreads)
  {
    const int tid = omp_get_thread_num(), nt = omp_get_num_threads();
    const int b0 = z_lo + (int)((int64_t)n_slab * tid / nt);
    const int b1 = z_lo + (int)((int64_t)n_slab * (tid + 1) / nt);
    for (int a = 0; a < n_a; a++) {
      const double *g = geom + 12 * a;
      const double ox = g[0], oy = g[1], oz = g[2];
      for (int v = 0; v < n_v; v++)
        for (int u = 0; u < n_u; u++) {
          float val = proj[((int64_t)a * n_v + v) * n_u + u];
          if (val == 0.0f) continue;
          double dx, dy, dz, t0, step;
          int64_t n;
          pixel_dir(g, u, v, &dx, &dy, &dz);
          ray_steps(ox, oy, oz, dx, dy, dz, grid, nx, ny, nz, step_max, &t0,
                    &step, &n);
          double scaled = (double)val * step;
          for (int64_t k = 0; k < n; k++) {
            double t = t0 + ((double)k + 0.5) * step;
            double qz = (oz + t * dz - gz0) / vz - 0.5;
            double fz0 = floor(qz);
            int iz0 = (int)fz0;
            /* only this thread's band (the reference masks by slab) */
            if (iz0 + 1 < b0 || iz0 >= b1) continue;
            double qx = (ox + t * dx - gx0) / vx - 0.5;
            double qy = (oy + t * dy - gy0) / vy - 0.5;
            int ix0 = (int)floor(qx), iy0 = (int)floor(qy);
            double wx = qx - ix0, wy = qy - iy0, wz = qz - iz0;
            for (int cz = 0; cz < 2; cz++) {
              int zi = iz0 + cz;
              if (zi < b0 || zi >= b1) continue;
              double fz = cz == 1 ? wz : 1.0 - wz;
              for (int cy = 0; cy < 2; cy++) {
                int yi = iy0 + cy;
                if (yi < 0 || yi >= ny) continue;
                double fy = cy == 1 ? wy : 1.0 - wy;
                for (int cx = 0; cx < 2; cx++) {
                  int xi = ix0 + cx;
                  if (xi < 0 || xi >= nx) continue;
                  double fx = cx == 1 ? wx : 1.0 - wx;
                  vol64[(int64_t)(zi - z_lo) * plane + (int64_t)yi * nx +
                        xi] += scaled * fz * fy * fx;
                }
              }
            }
          }
        }
    }
  }
  return 0;
}

/* _kernels.py:340-398 -- voxel-driven FDK backprojection with (dso/U)^2
 * weights into the float64 slab accumulator vol64 [n_slab, ny, nx]
 * (accumulates; every voxel extends its own chain in angle order). */
int orc_bwd_fdk(double *vol64, int nx, int ny, int n_slab, int z_lo,
                const double *grid, const double *cs, int n_a, double dso,
                double dsd, double du, double dv, double off_u, double off_v,
                int n_u, int n_v, const float *proj, int nthreads) {
  const double gx0 = grid[0], gy0 = grid[1], gz0 = grid[2];
  const double vx = grid[3], vy = grid[4], vz = grid[5];
  const int64_t plane = (int64_t)nx * ny;
  const int64_t sheet = (int64_t)n_u * n_v;
#pragma omp parallel for collapse(2) schedule(static) num_threads(nthreads)
  for (int iy = 0; iy < ny; iy++)
    for (int ix = 0; ix < nx; ix++) {
      double wy = gy0 + (iy + 0.5) * vy;
      double wx = gx0 + (ix + 0.5) * vx;
      for (int iz = 0; iz < n_slab; iz++) {
        double wz = gz0 + (z_lo + iz + 0.5) * vz;
        double *cell = vol64 + (int64_t)iz * plane + (int64_t)iy * nx + ix;
        double acc = *cell;
        for (int a = 0; a < n_a; a++) {
          double c = cs[2 * a], s = cs[2 * a + 1];
          double big_u = dso - (wx * c + wy * s);
          if (big_u <= 1e-9) continue;
          double mag = dsd / big_u;
          double uf = ((-wx * s + wy * c) * mag - off_u) / du + 0.5 * (n_u - 1);
          double vf = (wz * mag - off_v) / dv + 0.5 * (n_v - 1);
          int u0 = (int)floor(uf), v0 = (int)floor(vf);
          double fu = uf - u0, fv = vf - v0;
          const float *p = proj + (int64_t)a * sheet;
          double val = 0.0;
          if (0 <= v0 && v0 < n_v) {
            if (0 <= u0 && u0 < n_u)
              val += (1.0 - fv) * (1.0 - fu) * p[(int64_t)v0 * n_u + u0];
            if (0 <= u0 + 1 && u0 + 1 < n_u)
              val += (1.0 - fv) * fu * p[(int64_t)v0 * n_u + u0 + 1];
          }
          if (0 <= v0 + 1 && v0 + 1 < n_v) {
            if (0 <= u0 && u0 < n_u)
              val += fv * (1.0 - fu) * p[(int64_t)(v0 + 1) * n_u + u0];
            if (0 <= u0 + 1 && u0 + 1 < n_u)
              val += fv * fu * p[(int64_t)(v0 + 1) * n_u + u0 + 1];
          }
          if (val != 0.0) {
            double w = dso / big_u;
            acc += w * w * val;
          }
        }
        *cell = acc;
      }
    }
  return 0;
}

/* _kernels.py:71-151 -- exact intersection-length integral of one ray over
 * slab [z_lo, z_hi), midpoint attribution (half-open voxels). */
static double siddon_ray(const float *vol, double ox, double oy, double oz,
                         double dx, double dy, double dz, const double *grid,
                         int nx, int ny, int z_lo, int z_hi) {
  const double gx0 = grid[0], gy0 = grid[1], gz0 = grid[2];
  const double vx = grid[3], vy = grid[4], vz = grid[5];
  double bz_lo = gz0 + z_lo * vz, bz_hi = gz0 + z_hi * vz;
  double t0, t1;
  clip_box(ox, oy, oz, dx, dy, dz, gx0, gy0, bz_lo, gx0 + nx * vx,
           gy0 + ny * vy, bz_hi, &t0, &t1);
  if (t0 > t1 || t1 - t0 <= EPS_LEN) return 0.0;
  double px = ox + t0 * dx, py = oy + t0 * dy, pz = oz + t0 * dz;
  double tnx, dtx, tny, dty, tnz, dtz;
  if (dx > 0.0) {
    tnx = t0 + ((floor((px - gx0) / vx) + 1.0) * vx - (px - gx0)) / dx;
    dtx = vx / dx;
  } else if (dx < 0.0) {
    tnx = t0 + ((ceil((px - gx0) / vx) - 1.0) * vx - (px - gx0)) / dx;
    dtx = -vx / dx;
  } else { tnx = 1e300; dtx = 0.0; }
  if (dy > 0.0) {
    tny = t0 + ((floor((py - gy0) / vy) + 1.0) * vy - (py - gy0)) / dy;
    dty = vy / dy;
  } else if (dy < 0.0) {
    tny = t0 + ((ceil((py - gy0) / vy) - 1.0) * vy - (py - gy0)) / dy;
    dty = -vy / dy;
  } else { tny = 1e300; dty = 0.0; }
  if (dz > 0.0) {
    tnz = t0 + ((floor((pz - gz0) / vz) + 1.0) * vz - (pz - gz0)) / dz;
    dtz = vz / dz;
  } else if (dz < 0.0) {
    tnz = t0 + ((ceil((pz - gz0) / vz) - 1.0) * vz - (pz - gz0)) / dz;
    dtz = -vz / dz;
  } else { tnz = 1e300; dtz = 0.0; }
  const int64_t plane = (int64_t)nx * ny;
  double acc = 0.0, t = t0;
  while (t < t1 - EPS_LEN) {
    double tn = tnx;
    if (tny < tn) tn = tny;
    if (tnz < tn) tn = tnz;
    if (tn > t1) tn = t1;
    double seg = tn - t;
    if (seg > EPS_LEN) {
      double tm = 0.5 * (t + tn);
      int ix = (int)floor((ox + tm * dx - gx0) / vx);
      int iy = (int)floor((oy + tm * dy - gy0) / vy);
      int iz = (int)floor((oz + tm * dz - gz0) / vz);
      if (0 <= ix && ix < nx && 0 <= iy && iy < ny && z_lo <= iz && iz < z_hi)
        acc += seg * (double)vol[(int64_t)(iz - z_lo) * plane +
                                 (int64_t)iy * nx + ix];
    }
    if (tn >= t1) break;
    if (tnx <= tn) tnx += dtx;
    if (tny <= tn) tny += dty;
    if (tnz <= tn) tnz += dtz;
    t = tn;
  }
  return acc;
}

/* _kernels.py:154-191 -- Siddon forward projection of a slab. */
int orc_fwd_siddon(const float *vol, int nx, int ny, int nz, int z_lo,
                   int z_hi, const double *grid, const double *geom, int n_a,
                   int n_u, int n_v, float *out, int nthreads) {
  (void)nz;
#pragma omp parallel for collapse(2) schedule(dynamic, 1) num_threads(nthreads)
  for (int a = 0; a < n_a; a++)
    for (int v = 0; v < n_v; v++) {
      const double *g = geom + 12 * a;
      for (int u = 0; u < n_u; u++) {
        double dx, dy, dz;
        pixel_dir(g, u, v, &dx, &dy, &dz);
        out[((int64_t)a * n_v + v) * n_u + u] = (float)siddon_ray(
            vol, g[0], g[1], g[2], dx, dy, dz, grid, nx, ny, z_lo, z_hi);
      }
    }
  return 0;
}

/* Ray/box set-up exposed for tests: (t0, step, n_steps) per ray of one
 * angle, _kernels.py:194-210. */
int orc_ray_table(const double *grid, int nx, int ny, int nz,
                  const double *geom, int n_a, int n_u, int n_v,
                  double step_max, double *t0_out, double *step_out,
                  int64_t *n_out) {
  for (int a = 0; a < n_a; a++)
    for (int v = 0; v < n_v; v++)
      for (int u = 0; u < n_u; u++) {
        const double *g = geom + 12 * a;
        double dx, dy, dz;
        pixel_dir(g, u, v, &dx, &dy, &dz);
        int64_t i = ((int64_t)a * n_v + v) * n_u + u;
        ray_steps(g[0], g[1], g[2], dx, dy, dz, grid, nx, ny, nz, step_max,
                  &t0_out[i], &step_out[i], &n_out[i]);
      }
  return 0;
}
