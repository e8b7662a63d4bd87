// common.cuh -- shared device/host helpers for the conesplit B200 library.
//
// Error model of the C-ABI (include/conesplit_b200.h): every entry point
// returns 0 on success or a negative code, and records a message readable
// through cs_last_error() (thread-local).  Entry points never synchronise
// the host; all work is enqueued on the caller's stream.
#pragma once

#include <cuda_runtime.h>
#include <atomic>
#include <stdint.h>
#include <cstdio>
#include <string>

#include "../../include/conesplit_b200.h"

namespace cs {

// Packed fp32 pairs (sm_100 FADD2 / FMUL2 / FFMA2: two lanes of fp32 per
// instruction, each rounded exactly as the scalar op): the matched
// deposit's weight products and magic adds (staged.cu), the FDK lerps
// (backward.cu).
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 f2(float a, float b) {
  f32x2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2_split(f32x2 v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ f32x2 f2_mul(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2 f2_sub(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2 f2_fma(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}


void set_error(const char* fmt, ...);

// Kernels launched by this library since load (cs_launch_count()).
extern std::atomic<long long> g_launches;
#define CS_COUNT_LAUNCH() ::cs::g_launches.fetch_add(1, std::memory_order_relaxed)

#define CS_CHECK_CUDA(expr)                                                  \
  do {                                                                       \
    cudaError_t _e = (expr);                                                 \
    if (_e != cudaSuccess) {                                                 \
      ::cs::set_error("%s:%d %s -> %s", __FILE__, __LINE__, #expr,           \
                      cudaGetErrorString(_e));                               \
      return CS_ERR_CUDA;                                                    \
    }                                                                        \
  } while (0)

#define CS_REQUIRE(cond, code, ...)                                          \
  do {                                                                       \
    if (!(cond)) {                                                           \
      ::cs::set_error(__VA_ARGS__);                                          \
      return (code);                                                         \
    }                                                                        \
  } while (0)

// Voxel grid: lower corner, voxel size and counts (projectors.py:197-202).
struct Grid {
  double g0[3];
  double vox[3];
  int n[3];  // nx, ny, nz (FULL grid: ray sampling always uses the full box)
};

// Per-angle flattened geometry, projectors.py:172-194:
//   src[3], det00[3], ustep[3], vstep[3]
struct AngleGeom {
  double src[3], det00[3], ustep[3], vstep[3];
};

// ---------------------------------------------------------------------------
// fp64 ray set-up, IEEE round-to-nearest with NO contraction so that the
// sample count n = ceil(L / step_max) and t0 / step are the reference's bits
// (_kernels.py:28-68, :194-210, :234-246).  SURVEY 0.3: fp32 set-up flips
// n_steps on ~1e-4 of rays at 512^3.

__device__ __forceinline__ double dsub(double a, double b) {
  return __dadd_rn(a, -b);
}

struct Ray {
  double o[3];    // source
  double d[3];    // unit direction
  double t0;      // entry parameter on the full grid box
  double step;    // L / n
  long long n;    // number of samples (0 = miss / graze)
};

// Unit direction through pixel (u, v): _kernels.py:234-243.
__device__ __forceinline__ void pixel_direction(const AngleGeom& g, int u,
                                                int v, double d[3]) {
  double t[3];
#pragma unroll
  for (int i = 0; i < 3; i++)
    t[i] = __dadd_rn(__dadd_rn(g.det00[i], __dmul_rn((double)u, g.ustep[i])),
                     __dmul_rn((double)v, g.vstep[i]));
  double x = dsub(t[0], g.src[0]), y = dsub(t[1], g.src[1]),
         z = dsub(t[2], g.src[2]);
  double ss = __dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)),
                        __dmul_rn(z, z));
  double inv = __ddiv_rn(1.0, __dsqrt_rn(ss));
  d[0] = __dmul_rn(x, inv);
  d[1] = __dmul_rn(y, inv);
  d[2] = __dmul_rn(z, inv);
}

// Slab-method clip against [b0, b1] per axis: _kernels.py:28-68.
// Returns false on a miss.
__device__ __forceinline__ bool clip_box(const double o[3], const double d[3],
                                         const double b0[3],
                                         const double b1[3], double& t0o,
                                         double& t1o) {
  double t0 = -1e300, t1 = 1e300;
#pragma unroll
  for (int i = 0; i < 3; i++) {
    if (d[i] != 0.0) {
      double ta = __ddiv_rn(dsub(b0[i], o[i]), d[i]);
      double tb = __ddiv_rn(dsub(b1[i], o[i]), d[i]);
      if (ta > tb) {
        double tmp = ta;
        ta = tb;
        tb = tmp;
      }
      if (ta > t0) t0 = ta;
      if (tb < t1) t1 = tb;
    } else if (o[i] < b0[i] || o[i] > b1[i]) {
      return false;
    }
  }
  if (t0 > t1) return false;
  t0o = t0;
  t1o = t1;
  return true;
}

// _kernels.py:194-210 (+ the direction of :234-243).
__device__ __forceinline__ void setup_ray(const AngleGeom& g, const Grid& G,
                                          double step_max, int u, int v,
                                          Ray& r) {
  r.o[0] = g.src[0];
  r.o[1] = g.src[1];
  r.o[2] = g.src[2];
  pixel_direction(g, u, v, r.d);
  double b0[3], b1[3];
#pragma unroll
  for (int i = 0; i < 3; i++) {
    b0[i] = G.g0[i];
    b1[i] = __dadd_rn(G.g0[i], __dmul_rn((double)G.n[i], G.vox[i]));
  }
  double t0, t1;
  r.n = 0;
  r.t0 = 0.0;
  r.step = 0.0;
  if (!clip_box(r.o, r.d, b0, b1, t0, t1)) return;
  double length = dsub(t1, t0);
  if (length <= 1e-12) return;  // _EPS_LEN graze
  double nf = ceil(__ddiv_rn(length, step_max));
  r.n = (long long)nf;
  r.t0 = t0;
  r.step = __ddiv_rn(length, nf);
}

// March parameters.  The sample positions of the reference,
//   q(k) = (o + (t0 + (k + 1/2) step) d - g0) / vox - 1/2   (_kernels.py:249-252)
// are evaluated in 64-bit fixed point Q32.32: q(k) = A0 + k Bq exactly in
// integers (A0, Bq rounded once from fp64), so the cell index is the high
// word and the trilinear weight the top 23 bits of the low word (one
// 64-bit add, a shift, a LOP3 and an FADD per axis and sample -- the
// instruction count of the fp32 form it replaces).  Position error
// <= k * 2^-33 voxel (< 1e-6 at 2048^3) independent of the volume size --
// fp32 absolute coordinates carried ulp(N/2) (3e-5 voxel at 512^3, 1.2e-4
// at 2048^3), which put the matched adjoint at relL2 1.6e-5 / 6.5e-5 vs the
// reference at those sizes.  Being exact integers, positions are the same
// function of k in every kernel, chunk and slab launch.
constexpr int QF = 32;

struct March {
  long long A0[3];  // q(0), Q32.32
  long long Bq[3];  // q(k + 1) - q(k), Q32.32
  float A[3], B[3]; // fp32 q(kc) and step: estimates only (chunk bounds)
  double Ad[3], Bd[3];
  long long kc;
};

__device__ __forceinline__ void march_params(const Ray& r, const Grid& G,
                                             March& m) {
  m.kc = r.n >> 1;
  const double t0 = r.t0 + 0.5 * r.step;
  const double tc = r.t0 + ((double)m.kc + 0.5) * r.step;
#pragma unroll
  for (int i = 0; i < 3; i++) {
    const double q0 = (r.o[i] + t0 * r.d[i] - G.g0[i]) / G.vox[i] - 0.5;
    const double b = r.step * r.d[i] / G.vox[i];
    m.A0[i] = __double2ll_rn(ldexp(q0, QF));
    m.Bq[i] = __double2ll_rn(ldexp(b, QF));
    m.Ad[i] = (r.o[i] + tc * r.d[i] - G.g0[i]) / G.vox[i] - 0.5;
    m.Bd[i] = b;
    m.A[i] = (float)m.Ad[i];
    m.B[i] = (float)b;
  }
}

// q(k) along axis i (exact)
__device__ __forceinline__ long long q_at(const March& m, int k, int i) {
  return m.A0[i] + (long long)k * m.Bq[i];
}
// floor(q): the integer part (arithmetic shift: floor for negative q too)
__device__ __forceinline__ int q_cell(long long q) {
  return (int)(q >> QF);
}
// q - floor(q) in [0, 1): the top 23 fraction bits as 1.f... - 1
__device__ __forceinline__ float q_frac(long long q) {
  return __uint_as_float(0x3F800000u |
                         ((unsigned)(q >> (QF - 23)) & 0x7FFFFFu)) - 1.f;
}
// int -> float for |i| < 2^22 without the conversion pipe
__device__ __forceinline__ float int_to_float(int i) {
  return __int_as_float(i + 0x4B400000) - 12582912.f;
}

// Sample range [k0, k1) whose trilinear support along `axis` can touch
// planes [lo, hi): q(axis, k) in [lo - 1, hi) (slab_k_range: z, the slab).
// Conservative by two samples; exact membership is decided per tap in the
// march loop from the same exact positions a monolithic launch computes, so
// slab partial sums add up to the monolithic result.
__device__ __forceinline__ void axis_k_range(const Ray& r, const March& m,
                                             int axis, int n_axis, int lo_i,
                                             int hi_i, long long& k0,
                                             long long& k1) {
  k0 = 0;
  k1 = r.n;
  if (lo_i <= 0 && hi_i >= n_axis) return;
  double B = m.Bd[axis], A = m.Ad[axis];
  double lo = (double)lo_i - 1.0, hi = (double)hi_i;
  if (fabs(B) < 1e-30) {
    if (A < lo - 1.0 || A > hi + 1.0) k1 = 0;
    return;
  }
  double ka = (lo - A) / B + (double)m.kc, kb = (hi - A) / B + (double)m.kc;
  if (ka > kb) {
    double t = ka;
    ka = kb;
    kb = t;
  }
  double fa = floor(ka) - 2.0, fb = ceil(kb) + 3.0;
  if (fa > 0.0) k0 = fa > (double)r.n ? r.n : (long long)fa;
  if (fb < (double)r.n) k1 = fb < 0.0 ? 0 : (long long)fb;
}

__device__ __forceinline__ void slab_k_range(const Ray& r, const March& m,
                                             const Grid& G, int z_lo,
                                             int z_hi, long long& k0,
                                             long long& k1) {
  axis_k_range(r, m, 2, G.n[2], z_lo, z_hi, k0, k1);
}

// tld4 (gather) on a 2D layered float texture: returns the 2x2 footprint a
// bilinear fetch at (x, y) would use.  With x = i + 1, y = j + 1 (unnormalised
// coordinates) the footprint is texels i..i+1 x j..j+1.  Component order
// (PTX tld4): x = (i, j+1), y = (i+1, j+1), z = (i+1, j), w = (i, j).
// Border address mode supplies the reference's zero padding in x and y
// (_kernels.py:264-272; FDK :385-394); layers are clamped by hardware, so
// callers mask layers themselves.
__device__ __forceinline__ float4 gather_a2d(cudaTextureObject_t t, int layer,
                                             float x, float y) {
  float4 r;
  asm volatile(
      "tld4.r.a2d.v4.f32.f32 {%0, %1, %2, %3}, [%4, {%5, %6, %7, %8}];"
      : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
      : "l"(t), "r"(layer), "f"(x), "f"(y), "f"(0.f));
  return r;
}

// gather_a2d into r only where p holds (predicated tld4: a quad whose lanes
// are all off costs the texture pipe nothing; r keeps its value elsewhere)
__device__ __forceinline__ void gather_a2d_if(float4& r, bool p,
                                              cudaTextureObject_t t,
                                              int layer, float x, float y) {
  asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %9, 0;\n\t"
      "@q tld4.r.a2d.v4.f32.f32 {%0, %1, %2, %3}, [%4, {%5, %6, %7, %8}];\n\t}"
      : "+f"(r.x), "+f"(r.y), "+f"(r.z), "+f"(r.w)
      : "l"(t), "r"(layer), "f"(x), "f"(y), "f"(0.f), "r"((int)p));
}

// ---------------------------------------------------------------------------
// Host side: per-(device, stream) layered-texture cache.  A volume slab
// [n_slab, ny, nx] becomes a cudaArray with nx x ny layers; a projection
// stack [n_a, n_v, n_u] becomes n_u x n_v layers.
struct LayeredTexture {
  cudaArray_t array = nullptr;
  cudaTextureObject_t tex = 0;
  cudaSurfaceObject_t surf = 0;
  int w = 0, h = 0, layers = 0;
};

// TEX_VOLUME: a volume slab as z-layers (x, y per layer);
// TEX_PROJ: a projection stack as angle-layers (u, v per layer).
// TEX_VOL_M / TEX_VOL_M2: a volume slab layered along a main axis (x- or
// y-layers, forward.cu's main-axis kernel; M2 when nx != ny).
enum TexRole { TEX_VOLUME = 0, TEX_PROJ = 1, TEX_VOL_M = 2, TEX_VOL_M2 = 3 };

// Main axis of a view (0 = x, 1 = y): the larger |x| / |y| component of the
// central ray.  Host side.
inline int view_axis(const double* g12, int n_u, int n_v) {
  double d[2];
  for (int i = 0; i < 2; i++)
    d[i] = g12[3 + i] + 0.5 * (n_u - 1) * g12[6 + i] +
           0.5 * (n_v - 1) * g12[9 + i] - g12[i];
  return fabs(d[0]) >= fabs(d[1]) ? 0 : 1;
}

// Cached (w, h, >= layers) surface-writable layered array, contents
// undefined; stream-ordered reuse per (device, stream, role).
// taller_ok: an array of height >= h may be reused (the caller zeroes the
// rows past h that its reads can reach).
int acquire_layered(TexRole role, int w, int h, int layers, cudaStream_t s,
                    LayeredTexture** out, bool taller_ok = false);

// Returns a texture whose array is (w, h, >= layers) and loads `layers`
// layers from the linear array `src` ([layers][h][w], device or host
// memory) on stream s.
int load_layered(TexRole role, const float* src, int w, int h, int layers,
                 cudaStream_t s, LayeredTexture** out);

// Max layers of a 2D layered texture on this device (2048 on sm_100).
int max_layers();
// Max width / height of a 2D layered texture on this device.
int max_layered_height();

// Default mempool keeps freed memory (see runtime.cu).
void retain_pool();

// Geometry tables copied to the device (stream-ordered allocation).
int upload_geometry(const double* geom, int n_a, cudaStream_t s,
                    AngleGeom** d_geom);
void release_geometry(AngleGeom* d_geom, cudaStream_t s);

Grid make_grid(const double grid6[6], int nx, int ny, int nz);

// Detector rows [v0, v1) whose rays can touch slices [z_lo, z_hi) in any of
// the n_a views (full range for a full-height slab); runtime.cu.
void slab_row_band(const double* geom, int n_a, const Grid& G, int z_lo,
                   int z_hi, int n_v, int* v0, int* v1);

// Knob: CS_NO_CULL=1 disables v-band culling (A/B runs).
bool cull_enabled();

// Zero rows [0, v0) and [v1, n_v) of every view of out[n_a][n_v][n_u]
// (the overwrite-mode result of the culled rows).
int zero_rows_outside(float* out, int n_a, int n_u, int n_v, int v0, int v1,
                      cudaStream_t s);

// Shared-memory staged Ax / matched Atb (staged.cu).
enum StOpKind { OP_FWD = 0, OP_BWD = 1 };
template <int OP, int MODE>
int launch_staged(const float* vol_in, float* vol_acc, int nx, int ny, int nz,
                  int z_lo, int z_hi, const double* grid6, const double* geom,
                  int n_a, int n_u, int n_v, double step_max, float* out,
                  const float* proj_in, const float* rb, const float* rw,
                  cudaStream_t s);

inline int num_sms() {
  static int sms = -1;
  if (sms < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return sms;
}

}  // namespace cs
