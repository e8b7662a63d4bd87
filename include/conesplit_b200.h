/*
 * conesplit_b200.h -- C-ABI of the B200-native cone-beam hot path.
 *
 * Drop-in boundary B1 of SURVEY 8(b): each entry point replaces one numba
 * kernel of the reference package `conesplit`
 * (/root/reference/pkg/src/conesplit/_kernels.py) or one numpy stencil of
 * its regulariser (regularization.py), with the same argument meaning.
 *
 * Conventions
 *   - Array arguments marked "device" are device pointers owned by the
 *     caller (no allocation of caller-visible memory inside the library);
 *     "host" arrays are read synchronously before the call returns.
 *   - Geometry arrives flattened exactly as the reference's _flat_geometry
 *     (projectors.py:172-194): per angle 12 doubles
 *         src[3], det00[3], ustep[3], vstep[3]
 *     and the grid as grid6 = {gx0, gy0, gz0, vx, vy, vz}
 *     (projectors.py:197-202, geometry.py:64-68).
 *   - Volumes are [z][y][x] (x fastest), projections [angle][v][u]
 *     (u fastest), both float32 (projectors.py:81-163).
 *   - Every call is asynchronous on `stream` (a cudaStream_t; 0 = legacy
 *     default stream) and returns 0 on success or a negative CS_ERR_* code;
 *     cs_last_error() returns the thread's last message.
 *   - Accumulation is fp32 on device (the reference accumulates in fp64,
 *     _kernels.py:3-13); per-ray set-up is fp64 with the reference's exact
 *     operation order, so sample counts and positions are the reference's.
 */
#ifndef CONESPLIT_B200_H
#define CONESPLIT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CS_OK 0
#define CS_ERR_ARG -1
#define CS_ERR_CUDA -2
#define CS_ERR_UNSUPPORTED -3

typedef void* cs_stream_t; /* cudaStream_t */

/* Library identity / diagnostics. */
const char* cs_version(void);
const char* cs_last_error(void);
/* Kernels launched by the library since it was loaded (diagnostics; the
 * bench's gpu_launches claim). */
long long cs_launch_count(void);
/* Blocks the host until `stream` drains (the only synchronising call). */
int cs_sync(cs_stream_t stream);
/* Frees the library's cached texture arrays on the current device (one per
 * stream and layout, each the size of the largest slab / stack projected
 * through it); synchronises the device first.  Called by the Python layer
 * before retrying a call that ran out of device memory. */
int cs_release_cache(void);

/* ---------------------------------------------------------------- Ax ---- */

/* Interpolated (trilinear, fixed-step) forward projection of the slab
 * vol = grid slices [z_lo, z_hi) onto n_a angles.
 * Replaces interp_forward_chunk(vol, srcs, det00, ustep, vstep, gx0, gy0,
 * gz0, vx, vy, vz, nx, ny, nz, z_lo, z_hi, step_max, tile_u, tile_v, out)
 * (_kernels.py:213-275); tiles are a CPU scheduling detail and are absent.
 *   vol  device [z_hi-z_lo][ny][nx]     geom host [n_a][12]
 *   out  device [n_a][n_v][n_u]; overwritten (accumulate=0) or added to
 *        (accumulate=1: the partial-projection accumulate of
 *        execution.py:224-235 fused into the kernel epilogue). */
int cs_fwd_interp(const float* vol, int nx, int ny, int nz, int z_lo,
                  int z_hi, const double* grid6, const double* geom, int n_a,
                  int n_u, int n_v, double step_max, float* out,
                  int accumulate, cs_stream_t stream);

/* OS-SART residual epilogue fused into Ax (algorithms.py:294-296):
 *   out[r] = w[r] * (b[r] - (A vol)[r])      (w may be NULL -> 1)
 * Full volume only (z range [0, nz)). */
int cs_fwd_interp_residual(const float* vol, int nx, int ny, int nz,
                           const double* grid6, const double* geom, int n_a,
                           int n_u, int n_v, double step_max, const float* b,
                           const float* w, float* out, cs_stream_t stream);

/* Siddon (exact intersection length) forward projection of a slab.
 * Replaces siddon_forward_chunk (_kernels.py:154-191, ray :71-151). */
int cs_fwd_siddon(const float* vol, int nx, int ny, int nz, int z_lo,
                  int z_hi, const double* grid6, const double* geom, int n_a,
                  int n_u, int n_v, float* out, int accumulate,
                  cs_stream_t stream);

/* --------------------------------------------------------------- Atb ---- */

/* Exact adjoint of cs_fwd_interp, accumulated into the slab
 * vol_acc = grid slices [z_lo, z_hi).
 * Replaces matched_backward_chunk(vol64, proj, srcs, det00, ustep, vstep,
 * gx0.., vx.., nx, ny, nz, z_lo, z_hi, step_max) (_kernels.py:278-337).
 *   vol_acc device [z_hi-z_lo][ny][nx] (added to)   proj device [n_a][n_v][n_u] */
int cs_bwd_matched(float* vol_acc, int nx, int ny, int nz, int z_lo,
                   int z_hi, const double* grid6, const double* geom, int n_a,
                   int n_u, int n_v, double step_max, const float* proj,
                   cs_stream_t stream);
/* Run-to-run determinism of cs_bwd_matched (process-wide; default off, or
 * CS_ST_DETERMINISTIC=1).  Off: CTAs add their (exact, integer) box sums
 * into vol_acc with fp32 reductions, whose order -- and so the last bits of
 * a voxel -- varies from run to run.  On: the contributions are rounded
 * once to a launch-wide fixed point and summed as 64-bit integers in a
 * slab-sized scratch accumulator (8 B per voxel, from CUDA's stream-ordered
 * pool; a second, transposed one when the x-major views run in the
 * transposed frame), then added into vol_acc: bit-identical results every
 * run, as the
 * reference's fp64 host accumulation is (_kernels.py:278-337). */
int cs_set_deterministic(int on);

/* Voxel-driven FDK-weighted backprojection, accumulated into slab
 * vol_acc = grid slices [z_lo, z_lo + n_slab).
 * Replaces fdk_backward_chunk(vol64, proj, coss, sins, dso, dsd, du, dv,
 * off_u, off_v, gx0, gy0, gz0, vx, vy, vz, z_lo, tile_x, tile_y)
 * (_kernels.py:340-398).  cs = host [n_a][2] = (cos, sin). */
int cs_bwd_fdk(float* vol_acc, int nx, int ny, int z_lo, int n_slab,
               const double* grid6, const double* cs, int n_a, double dso,
               double dsd, double du, double dv, double off_u, double off_v,
               int n_u, int n_v, const float* proj, cs_stream_t stream);

/* Per-ray fp64 set-up (t0, step, n_steps), for parity tests of the ray
 * clip of _kernels.py:194-210.  Outputs device [n_a][n_v][n_u]. */
int cs_ray_table(int nx, int ny, int nz, const double* grid6,
                 const double* geom, int n_a, int n_u, int n_v,
                 double step_max, double* t0, double* step, int64_t* n,
                 cs_stream_t stream);

/* ---------------------------------------------------------------- TV ---- */
/* All TV kernels act on a window u[nzw][ny][nx] whose first/last planes are
 * treated as faces (the reference's _grad/_div on a window array,
 * regularization.py:88-110, used per halo window at :241-260).  Reductions
 * are written as fp64 to `out_sum` (device, 1 element) deterministically.
 * Σ over planes [core_lo, core_hi) of the window only. */

/* Σ g^2 over the core, g = -div(∇u / sqrt(|∇u|^2 + 1e-8))
 * (regularization.py:127-130, :245-251 / :147). */
int cs_tv_grad_sumsq(const float* u, int nx, int ny, int nzw, int core_lo,
                     int core_hi, double* out_sum, cs_stream_t stream);
/* ||g||_2 over the core (regularization.py:147: np.linalg.norm(g)); the same
 * pass as cs_tv_grad_sumsq plus a device sqrt.  Multi-GPU callers reduce the
 * sum of squares across ranks first, so they use cs_tv_grad_sumsq. */
int cs_tv_grad_norm(const float* u, int nx, int ny, int nzw, int core_lo,
                    int core_hi, double* out_norm, cs_stream_t stream);

/* u_out = u - step * g / norm with norm = *norm_dev (device fp64 scalar);
 * skipped (u_out = u) when norm < 1e-30 (regularization.py:150, :258-260).
 * `scale` multiplies the norm (LocalApprox extrapolation, :252-257). */
int cs_tv_step(const float* u, float* u_out, int nx, int ny, int nzw,
               double step, const double* norm_sumsq_dev, double scale,
               cs_stream_t stream);

/* The GD iteration in two passes that share g: g stored over the whole
 * window (g[nzw][ny][nx], device) with Σg² over the core into out_sum, then
 * u_out = u - step * g / (sqrt(*norm_sumsq_dev) * scale) elementwise over
 * n voxels -- the same g and the same step arithmetic as cs_tv_grad_sumsq
 * + cs_tv_step (the sums agree to fp32 partial-sum grouping), with the
 * second pass a stream instead of a second stencil.  The step is
 * u - c g with c = step / norm rounded once to fp32 (one FFMA);
 * cs_tv_step_g may write in place (u_out == u), not over g. */
int cs_tv_grad_store(const float* u, float* g, int nx, int ny, int nzw,
                     int core_lo, int core_hi, double* out_sum,
                     cs_stream_t stream);
int cs_tv_step_g(const float* u, const float* g, float* u_out, int64_t n,
                 double step, const double* norm_sumsq_dev, double scale,
                 cs_stream_t stream);
/* One whole GD iteration after the first, in ONE pass (replaces the
 * reference's loop body regularization.py:145-150 for iterations >= 2):
 *   u_out = u - step * g / (sqrt(*norm_sumsq_dev) * scale)   (every voxel)
 *   g_out = TV subgradient of u_out over the window, *out_sum = sum of
 *           g_out^2 over the core planes [core_lo, core_hi)
 * u_out / g_out are bit-identical to cs_tv_step_g followed by
 * cs_tv_grad_store (same kernel family, same sums).  norm_sumsq_dev and out_sum must differ (the kernel reads
 * one while the reduction writes the other). */
int cs_tv_gd_fused(const float* u, const float* g, float* u_out, float* g_out,
                   int nx, int ny, int nzw, int core_lo, int core_hi,
                   double step, const double* norm_sumsq_dev, double scale,
                   double* out_sum, cs_stream_t stream);

/* One Chambolle dual iteration (regularization.py:174-182):
 *   u = f + lam div p; p += (1/12/lam) ∇u; p /= max(1, |p|)
 * p_in/p_out device [3][nzw][ny][nx] (must not alias). */
int cs_rof_iter(const float* f, const float* p_in, float* p_out, int nx,
                int ny, int nzw, double lam, cs_stream_t stream);

/* u = f + lam div p (regularization.py:170, :280). */
int cs_rof_finish(const float* f, const float* p, float* u, int nx, int ny,
                  int nzw, double lam, cs_stream_t stream);

/* Σ sqrt(Δz²+Δy²+Δx²) (regularization.py:119-124), fp64 into out_sum. */
int cs_tv_norm(const float* u, int nx, int ny, int nzw, double* out_sum,
               cs_stream_t stream);

/* --------------------------------------------- loop vector algebra ---- */
/* Building blocks of cgls / os_sart (algorithms.py:204-304). */

/* out_sum = Σ a[i]*b[i] in fp64, deterministic (b may equal a). */
int cs_dot(const float* a, const float* b, int64_t n, double* out_sum,
           cs_stream_t stream);
/* y += alpha * x, alpha read from device fp64 expression alpha = num/den
 * (den < 1e-30 -> no-op); sign = +1/-1.  (CGLS x += αp, r -= αq) */
int cs_axpy_ratio(float* y, const float* x, int64_t n, const double* num,
                  const double* den, double sign, cs_stream_t stream);
/* p = s + (num/den) * p  (CGLS direction update, algorithms.py:243-244) */
int cs_xpay_ratio(float* p, const float* s, int64_t n, const double* num,
                  const double* den, cs_stream_t stream);
/* out = a >= 1e-8 ? 1/a : 0  (algorithms.py:254-258) */
int cs_guarded_inverse(const float* a, float* out, int64_t n,
                       cs_stream_t stream);
/* x += lam * v * upd; upd = 0  (algorithms.py:298 + buffer reset) */
int cs_sart_update(float* x, float* upd, const float* v, double lam,
                   int64_t n, cs_stream_t stream);
/* r = w * (b - r) (w may be NULL: r = b - r) -- OS-SART's weighted
 * residual W_S (b_S - A_S x) on a projection shard (algorithms.py:296-297)
 * when A_S x arrives from the slab-sharded forward pass */
int cs_weighted_residual(float* r, const float* b, const float* w, int64_t n,
                         cs_stream_t stream);
/* x = value */
int cs_fill(float* x, float value, int64_t n, cs_stream_t stream);

/* ------------------------------------------- sharded peer exchange ---- */

/* out[i] = sum_{k < n_src} src[k * stride + i], summed in k order; with b:
 * out = b - sum, with b and w: out = w * (b - sum).  The owner-side half of
 * the slab-sharded forward's peer exchange (sharded.py / peer.py): the
 * other ranks' kernels stored their partial projections of the owner's
 * views into the owner's inbox slices (replaces the reduce-scatter of the
 * partials, the reference's slab-partial sum execution.py:224-235, fused
 * with OS-SART's residual algorithms.py:296-297). */
int cs_sum_slices(const float* src, int n_src, int64_t stride, int64_t n,
                  const float* b, const float* w, float* out,
                  cs_stream_t stream);
/* Lets kernels on the current device load / store device memory of
 * `peer_device` (cudaDeviceEnablePeerAccess; already enabled or
 * peer == current is fine).  CS_ERR_UNSUPPORTED when the pair has no P2P
 * path. */
int cs_peer_enable(int peer_device);

#ifdef __cplusplus
}
#endif
#endif /* CONESPLIT_B200_H */
