// staged.cu -- shared-memory staged Ax (K1) and matched Atb (K2).
//
// A CTA owns a 32 (u) x 8 (v) tile of detector rays of ONE view; warp w is
// detector row v0 + w, lane l is pixel u0 + l.  The view's rays travel
// mainly along M = x or y (|d_M| >= |d_T|); the CTA walks the volume in
// chunks of ST_S planes along M.  For each chunk it computes the box of
// voxels its rays' trilinear supports touch (block min/max of the first /
// last sample of every ray in the chunk) and stages that box in shared
// memory:
//   * Ax (OP_FWD): the box is loaded from the fp32 slab (zero outside the
//     grid / slab = the reference's masks, _kernels.py:259-272), then every
//     ray samples its chunk from shared memory -- 8 LDS per sample instead of
//     2 texture gathers, lifting the texture-writeback ceiling of the tex
//     kernel (forward.cu);
//   * matched Atb (OP_BWD): the box is zeroed, rays deposit their 8 taps
//     with native int32 shared atomics (ATOMS.ADD; fp32 shared atomics are
//     CAS loops on sm_100) in fixed point, scaled per CTA by its largest
//     |proj| so no voxel sum can overflow; the box is then added to global
//     memory with one 16-byte RED per aligned x-quad.  Where a voxel can
//     be reached only by tiny trilinear weights -- CTAs at the detector
//     border, and chunks where neighbouring rays are >= CS_ST_PRECISE_FP
//     voxels apart -- the chunk's box holds two words per voxel: the tap
//     rounded to the CTA's unit plus its exact rounding residual at 2^-k
//     of that unit ("precise" boxes), so tiny sums keep their relative
//     accuracy (the reference accumulates in fp64, _kernels.py:278-337).
// Samples, weights and masks are exactly those of the texture kernel (same
// fp64 ray set-up, same exact fixed-point positions q(k) = A0 + k Bq), so
// chunking changes only summation order.  Boxes that would not fit the
// shared-memory budget are served from global memory for that chunk.
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "common.cuh"

namespace cs {

constexpr int ST_TU = 32;
constexpr int ST_TV = 8;
constexpr int ST_THREADS = ST_TU * ST_TV;
#ifndef CS_ST_S
#define CS_ST_S 8
#endif
#ifndef CS_ST_ACC
#define CS_ST_ACC 0
#endif
// matched: zero the box words as the flush reads them (one zeroing of the
// whole box per CTA instead of one pass per chunk: 512^3 dense 259.8 -> 265.9
// GUPS, 256^3 188.7 -> 207.9; profiles/ab_matched_zof_r02am.jsonl)
// matched: launch order with the view index fastest (CTAs of neighbouring
// views of one detector tile run together, so their box flushes hit L2):
// 2048^3 x 32 views 262.5 -> 273.8 GUPS dense, 1024^3 265.0 -> 268.9, 512^3
// neutral (profiles/ab_matched_viewfast_r02ar.jsonl)
#ifndef CS_ST_VIEWFAST
#define CS_ST_VIEWFAST 1
#endif
// (A/B, -DCS_ST_UNROLL2=1) the sample loop unrolled by two: dense 512^3
// 255.8 vs 257.5 GUPS, 1024^3 267.7 vs 269.3 -- the kernel is bound by the
// shared-atomic wavefronts, not issue (profiles/ab_matched_unroll2_r02cr.jsonl)
#ifndef CS_ST_UNROLL2
#define CS_ST_UNROLL2 0
#endif
#ifndef CS_ST_ZOF
#define CS_ST_ZOF 1
#endif
constexpr int ST_S = CS_ST_S;  // planes per chunk along the main axis
constexpr int ST_S_DEEP = 14;  // matched on large planes (launch_staged)


// Float -> int without the conversion pipe: for |x| < 2^22, x + 1.5 * 2^23
// holds round-to-nearest(x) in its low mantissa bits.  F2I / FRND run at a
// quarter of the FMA rate on sm_100 and the matched deposit needed 8 of
// them per sample for its fixed-point taps; this is one FFMA + IADD.
constexpr float ST_MAGIC = 12582912.f;
// largest fixed-point tap: |x| < 2^22 keeps the magic add exact
constexpr double ST_BUDGET_CAP = 4.0e6;
__device__ __forceinline__ int magic_int(float biased) {
  return __float_as_int(biased) - 0x4B400000;
}

// a / b for 0 <= a < 2^22, 0 < b < 2^22 without the integer-division
// sequence (~25 instructions): fp32 reciprocal estimate, one correction
__device__ __forceinline__ int small_div(int a, int b, float rb) {
  int q = (int)((float)a * rb);
  const int r = a - q * b;
  q += r >= b ? 1 : (r < 0 ? -1 : 0);
  return q;
}

__device__ __forceinline__ int qfloor(const March& m, int k, int axis) {
  return q_cell(q_at(m, k, axis));  // exact (common.cuh)
}

// Red of a float4 quad (16-byte aligned) -- see backward.cu.
__device__ __forceinline__ void st_red4(float* p, float a, float b, float c,
                                        float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p),
               "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

// Deterministic matched Atb (cs_set_deterministic / CS_ST_DETERMINISTIC=1):
// every contribution that would be an fp32 red into the volume -- a CTA's
// flushed box voxel (itself an exact integer sum: the box is
// order-independent) or a global-path tap -- is rounded once to a launch-wide
// fixed point S = 2^k and added as a 64-bit integer (RED.E.ADD.64: integer
// adds are associative, so the total does not depend on the order in which
// CTAs finish); one pass adds acc / S into the fp32 volume at the end.  S is
// the largest power of two with n_a * max|proj| * step_max * taps * S <
// 2^62 (taps = samples of all rays in one voxel's support per view), from
// the launch's |proj| maximum on the device.
// (S is read from device memory at each use -- the launch computed it --
// so the production path keeps no register for it.)
__device__ __forceinline__ void det_add(long long* p, float v,
                                        const double* S) {
  if (v != 0.f)
    atomicAdd(reinterpret_cast<unsigned long long*>(p),
              (unsigned long long)__double2ll_rn((double)v * __ldg(S)));
}

// Precise boxes (matched only, chosen per chunk, CTA-uniform): every voxel
// holds an int2 (hi, lo): hi sums the taps rounded to the CTA's unit
// (scale = fx_budget / max tap), lo sums their exact rounding residuals
// times lo_scale = 2^k (|residual| <= 1/2, so k is sized to keep the
// per-voxel residual sum below 2^31).  value = (hi + lo / 2^k) / scale.
// Used where a voxel's whole coverage can consist of tiny weights: the
// int32 box resolves a tap only to 2.5e-7 of the CTA's largest tap, and
// OS-SART's V = 1 / A^T 1 (algorithms.py:254-258) turns that into a
// relative error of the update.  Also used everywhere when the int32
// budget falls below the magic-add cap (pixels much finer than voxels:
// many rays per voxel), where the residual word restores the resolution
// the coarse unit gives up.
//
// MINB = CTAs per SM: 3 (72 registers, 72 KB boxes) or 4 (64 registers, 54 KB
// boxes; 4 x 54 KB + the static arrays fit an SM's 228 KB), chosen per launch
// by the slab size (launch_staged).
template <int OP, int M, int MODE, int MINB = 3, int SD = ST_S>
__global__ void __launch_bounds__(ST_THREADS, MINB)
    staged_kernel(const float* __restrict__ vol_in, float* __restrict__ vol_acc,
                  const AngleGeom* __restrict__ geom,
                  const int* __restrict__ view_ids, Grid G, double step_max,
                  int z_lo, int z_hi, int n_u, int n_v, int v_base, int v_end,
                  float* __restrict__ out, const float* __restrict__ proj_in,
                  const float* __restrict__ rb, const float* __restrict__ rw,
                  int box_cap, float fx_budget, int vec_ok, int lane_stride,
                  int prec_mode, float prec_fp, int edge, float lo_scale,
                  int tpad, long long* __restrict__ dacc,
                  const double* __restrict__ dscale, int vpair, int n_ids) {
  constexpr int T = 1 - M;
  // matched in deterministic mode is the MODE = 3 instantiation (MODE is
  // otherwise an Ax epilogue selector): the default kernels carry no trace
  // of it
  constexpr bool DET = OP == OP_BWD && MODE == 3;
  extern __shared__ float4 st_box4[];
  float* st_box = reinterpret_cast<float*>(st_box4);
  int* box_i = reinterpret_cast<int*>(st_box4);
  // one-word deposit (native ATOMS.ADD; sm_100 has no native fp32 or 64-bit
  // shared add -- both compile to ATOMS.CAST.SPIN loops)
  auto deposit = [&](int idx, float y, float w) {
    atomicAdd(box_i + idx, magic_int(fmaf(y, w, ST_MAGIC)));
  };
  // two-word deposit: rounded tap + exact residual (precise boxes)
  auto deposit2 = [&](int idx, float y, float w) {
    const float tb = fmaf(y, w, ST_MAGIC);
    const float hf = tb - ST_MAGIC;   // round(y w), exact for |y w| < 2^22
    const float e = fmaf(y, w, -hf);  // y w - round(y w), |e| <= 1/2
    int* p = box_i + 2 * idx;
    atomicAdd(p, magic_int(tb));
    atomicAdd(p + 1, magic_int(fmaf(e, lo_scale, ST_MAGIC)));
  };
  __shared__ int ext[8];   // mlo, mhi, -, -, -, -, dir flags
  // per chunk candidate: tlo, thi, zlo, zhi (x2); double-buffered by chunk
  // parity, so the next chunk's set is reset while this one is read (two
  // barriers per chunk instead of three)
  __shared__ int ext8s[2][8];
  __shared__ float s_scale;
  __shared__ float s_gap;  // largest neighbouring-ray slope difference
  __shared__ float s_sqm;  // the source's q coordinate along M
  __shared__ int s_pall;   // all chunks precise

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // lane_stride s (power of two <= ST_TV): the CTA covers 32 s columns x
  // 8 / s rows and a warp's lanes are s pixels apart, so with pixels finer
  // than voxels the lanes of one ATOMS instruction seldom hit the same
  // shared word (same-address atomics serialise)
  const bool vf = OP == OP_BWD && CS_ST_VIEWFAST;
  const int bidx = vf ? blockIdx.y : blockIdx.x;   // detector u tile
  const int bidy = vf ? blockIdx.z : blockIdx.y;   // detector v tile
  const int bidv = vf ? blockIdx.x : blockIdx.z;   // view
  // view pairs (matched, lane stride 1): warps 0-3 take 4 detector rows of
  // view 2 bidv, warps 4-7 the same rows of view 2 bidv + 1 -- neighbouring
  // angles whose rays cross nearly the same voxels, so one box of about half
  // the z extent serves 256 rays and the flush per ray roughly halves
  const bool pr = OP == OP_BWD && vpair;
  const int wv = pr ? (warp & 3) : warp;
  const int tv_rows = pr ? ST_TV / 2 : ST_TV / lane_stride;
  const int vi = pr ? 2 * bidv + (warp >> 2) : bidv;
  const int u = bidx * (ST_TU * lane_stride) + lane * lane_stride +
                (wv & (lane_stride - 1));
  const int v = v_base + bidy * tv_rows + (pr ? wv : warp / lane_stride);
  const bool has_view = vi < n_ids;
  const int a = view_ids[has_view ? vi : 0];
  const bool valid = has_view && u < n_u && v < v_end;
  const int nx = G.n[0], ny = G.n[1];
  const size_t plane = (size_t)nx * ny;
  const size_t pix = ((size_t)a * n_v + v) * n_u + u;

  float val = 0.f;
  if (OP == OP_BWD && valid) val = __ldg(proj_in + pix);
  Ray r;
  r.n = 0;
  r.step = 0.0;
  if (valid && (OP == OP_FWD || val != 0.f)) setup_ray(geom[a], G, step_max, u, v, r);
  March m;
  int k0 = 0, k1 = 0;
  if (r.n > 0) {
    march_params(r, G, m);
    long long k0l, k1l;
    slab_k_range(r, m, G, z_lo, z_hi, k0l, k1l);
    k0 = (int)k0l;
    k1 = (int)k1l;
  }
  const bool has = k1 > k0;

  if (threadIdx.x == 0) {
    ext[0] = INT_MAX;
    ext[1] = INT_MIN;
    ext[6] = 0;  // any ray marching -M
    ext[7] = 0;  // any ray marching +M
    s_scale = 0.f;
    s_gap = 0.f;
    s_sqm = 0.f;
  }
  __syncthreads();
  if (has) {
    const int fa = qfloor(m, k0, M), fb = qfloor(m, k1 - 1, M);
    atomicMin(&ext[0], min(fa, fb));
    atomicMax(&ext[1], max(fa, fb));
    atomicOr(&ext[m.B[M] >= 0.f ? 7 : 6], 1);
  }
  if (OP == OP_BWD) {
    // per-CTA fixed-point scale: taps are |val| * step * w, w <= 1
    const float mag = has ? fabsf(val) * (float)r.step : 0.f;
    float wmax = mag;
    // Ray spacing for the precise-box rule: in voxel coordinates a ray is
    // q_T = sq_T + s_T (q_M - sq_M) (sq = the source), so the rays of
    // neighbouring pixels (u + 1, v + 1) sit |delta s| |q_M - sq_M| apart on
    // plane q_M.  gap = the largest such slope difference (T or z).
    float gap = 0.f;
    if (has && prec_mode == 0 && prec_fp < 1e29f) {
      const AngleGeom& ag = geom[a];
      float P[3], Pu[3], Pv[3];
#pragma unroll
      for (int i = 0; i < 3; i++) {
        const float iv = 1.f / (float)G.vox[i];
        const float pi = (float)(ag.det00[i] + (double)u * ag.ustep[i] +
                                 (double)v * ag.vstep[i] - ag.src[i]);
        P[i] = pi * iv;
        Pu[i] = (pi + (float)ag.ustep[i]) * iv;
        Pv[i] = (pi + (float)ag.vstep[i]) * iv;
      }
      const float i0 = 1.f / P[M], iu = 1.f / Pu[M], iv = 1.f / Pv[M];
      gap = fmaxf(fmaxf(fabsf(P[T] * i0 - Pu[T] * iu),
                        fabsf(P[2] * i0 - Pu[2] * iu)),
                  fmaxf(fabsf(P[T] * i0 - Pv[T] * iv),
                        fabsf(P[2] * i0 - Pv[2] * iv)));
    }
    for (int o = 16; o > 0; o >>= 1) {
      wmax = fmaxf(wmax, __shfl_xor_sync(0xffffffffu, wmax, o));
      gap = fmaxf(gap, __shfl_xor_sync(0xffffffffu, gap, o));
    }
    if (lane == 0) {
      atomicMax(reinterpret_cast<int*>(&s_scale),
                __float_as_int(wmax));  // non-negative floats
      atomicMax(reinterpret_cast<int*>(&s_gap), __float_as_int(gap));
    }
  }
  __syncthreads();
  const int mlo = ext[0], mhi = ext[1];
  if (mlo > mhi) {  // no ray of the tile touches the slab
    if (OP == OP_FWD && valid) {
      if (MODE == 0)
        out[pix] = 0.f;
      else if (MODE == 2)
        out[pix] = (rw ? rw[pix] : 1.f) * rb[pix];
    }
    return;
  }
  const int dir = ext[6] ? -1 : 1;  // march direction (uniform per view)
  const bool mixed = ext[6] && ext[7];
  float fscale = 0.f, inv_scale = 0.f;
  if (OP == OP_BWD) {
    const float tmax = s_scale;
    fscale = tmax > 0.f ? fx_budget / tmax : 0.f;
    inv_scale = fscale > 0.f ? 1.f / fscale : 0.f;
  }
  const float sv = OP == OP_BWD ? val * (float)r.step * fscale : 0.f;
  // precise boxes: always (prec_mode 1), never (2), or (0) for CTAs whose
  // tile lies within `edge` pixels of the detector border (voxels just
  // outside the outermost rays see only their weight tails) and for chunks
  // where neighbouring rays are >= prec_fp voxels apart (voxels between
  // them likewise); CTA-uniform
  // (kept in shared memory: read once per chunk, no registers held)
  if (OP == OP_BWD && threadIdx.x == 0) {
    bool pc = prec_mode == 1;
    if (prec_mode == 0) {
      const int tu = ST_TU * lane_stride, tv = tv_rows;
      const int u_first = bidx * tu, v_first = v_base + bidy * tv;
      pc = u_first < edge || u_first + tu > n_u - edge ||
           v_first < edge || v_first + tv > n_v - edge;
      const AngleGeom& ag = geom[a];
      s_sqm = (float)((ag.src[M] - G.g0[M]) / G.vox[M] - 0.5);
    }
    s_pall = pc;  // every chunk precise
    if (prec_mode == 2) s_gap = 0.f;
  }

  float acc = 0.f;
  if (mixed) {
    // rays of this tile march both ways along M (degenerate geometry):
    // serve every sample from global memory, no staging
    for (int kk = k0; kk < k1; kk++) {
      const long long qx = q_at(m, kk, 0), qy = q_at(m, kk, 1),
                      qz = q_at(m, kk, 2);
      const float wx = q_frac(qx), wy = q_frac(qy), wz = q_frac(qz);
      const int ix = q_cell(qx), iy = q_cell(qy), iz = q_cell(qz);
#pragma unroll
      for (int cz = 0; cz < 2; cz++) {
        const int zi = iz + cz;
        if (zi < z_lo || zi >= z_hi) continue;
        const float fz_ = cz ? wz : 1.f - wz;
#pragma unroll
        for (int cy = 0; cy < 2; cy++) {
          const int yi = iy + cy;
          if (yi < 0 || yi >= ny) continue;
          const float fy_ = cy ? wy : 1.f - wy;
#pragma unroll
          for (int cx = 0; cx < 2; cx++) {
            const int xi = ix + cx;
            if (xi < 0 || xi >= nx) continue;
            const float w = fz_ * fy_ * (cx ? wx : 1.f - wx);
            const size_t gi = (size_t)(zi - z_lo) * plane + (size_t)yi * nx + xi;
            if (OP == OP_FWD)
              acc = fmaf(w, __ldg(vol_in + gi), acc);
            else if (DET)
              det_add(dacc + gi, val * (float)r.step * w, dscale);
            else
              atomicAdd(vol_acc + gi, val * (float)r.step * w);
          }
        }
      }
    }
  }
  // samples are consumed in index order in both march directions: chunk c
  // takes the next run of samples whose M-cell lies in it
  // Chunks of ST_S cells along M in march order; a chunk whose box would
  // not fit the shared budget is retried at ST_S / 2 cells (both candidate
  // extents are reduced in one pass), and only then served from global.
  if (OP == OP_BWD && CS_ST_ZOF) {  // the flushes keep it zero afterwards
    for (int i = threadIdx.x; i < box_cap; i += ST_THREADS) box_i[i] = 0;
  }
  if (threadIdx.x < 16)
    ext8s[threadIdx.x >> 3][threadIdx.x & 7] =
        (threadIdx.x & 1) ? INT_MIN : INT_MAX;
  int par = 0;
  int k = k0;
  int cur = dir > 0 ? mlo : mhi;  // next M-cell in march order
  // reciprocal of the M step for the chunk-end estimates (an estimate:
  // the exact cell test settles it), one division per ray
  const float rbm = has ? 1.f / m.B[M] : 0.f;
  const bool run = !mixed;
  while (run && (dir > 0 ? cur <= mhi : cur >= mlo)) {
    // candidate chunks: S = SD (index 0) and, only when its box does not
    // fit the shared budget (a CTA-uniform decision), SD / 2 (index 1)
    int kbc[2] = {k, k};
    // last sample of candidate ci: qM(k) crosses the far face at
    // k* = kc + (face - A_M) / B_M; estimate, then settle on the exact cell
    // test (the same floor the sampling loop uses)
    auto chunk_end = [&](int ci) {
      const int S = SD >> ci;
      const int c_lo = dir > 0 ? cur : cur - S + 1;
      const int c_hi = c_lo + S - 1;
      const float face = dir > 0 ? (float)(c_hi + 1) : (float)c_lo;
      const float kst = (face - m.A[M]) * rbm + (float)(int)m.kc;
      int ke = (int)fminf(fmaxf(ceilf(kst), (float)k), (float)k1);
      if (dir > 0) {
        while (ke > k && qfloor(m, ke - 1, M) > c_hi) ke--;
        while (ke < k1 && qfloor(m, ke, M) <= c_hi) ke++;
      } else {
        while (ke > k && qfloor(m, ke - 1, M) < c_lo) ke--;
        while (ke < k1 && qfloor(m, ke, M) >= c_lo) ke++;
      }
      return ke;
    };
    // this ray's T / z extent over samples [k, ke) into candidate ci's slots
    auto extents = [&](int* e8, int ci) {
      if (kbc[ci] > k) {
        const int t0 = qfloor(m, k, T), t1 = qfloor(m, kbc[ci] - 1, T);
        const int zz0 = qfloor(m, k, 2), zz1 = qfloor(m, kbc[ci] - 1, 2);
        atomicMin(&e8[4 * ci + 0], min(t0, t1));
        atomicMax(&e8[4 * ci + 1], max(t0, t1));
        atomicMin(&e8[4 * ci + 2], min(zz0, zz1));
        atomicMax(&e8[4 * ci + 3], max(zz0, zz1));
      }
    };
    if (has) kbc[0] = chunk_end(0);
    __syncthreads();  // previous chunk's box consumed; ext8 reset
    int* ext8 = ext8s[par];
    extents(ext8, 0);
    __syncthreads();
    if (threadIdx.x < 8)  // the next chunk's set (read after its barrier)
      ext8s[par ^ 1][threadIdx.x] = (threadIdx.x & 1) ? INT_MIN : INT_MAX;
    par ^= 1;
    // box size for a candidate (same formula as the layout below)
    auto box_size = [&](int ci, int S) {
      const int c_lo = dir > 0 ? cur : cur - S + 1;
      const int nt = ext8[4 * ci + 1] - ext8[4 * ci] + 2;
      const int nzz = ext8[4 * ci + 3] - ext8[4 * ci + 2] + 2;
      const int xlo = M == 0 ? c_lo : ext8[4 * ci];
      const int xn = M == 0 ? S + 1 : nt;
      const int nbx = ((xlo + xn - (xlo & ~3)) + 3) & ~3;
      const int nby = M == 0 ? nt : S + 1;
      if (OP == OP_BWD && tpad)  // T pitch padded (layout below)
        return M == 1 ? ((nbx + tpad) & ~tpad) * nby * nzz
                      : nbx * ((nby + tpad) & ~tpad) * nzz;
      return M == 1 ? nbx * nby * nzz : nbx * (nby | 1) * nzz;
    };
    bool prec = false;
    if (OP == OP_BWD) {
      const float c0f = (float)(dir > 0 ? cur : cur - SD + 1);
      const float sq_m = s_sqm;
      prec = s_pall ||
             s_gap * fmaxf(fabsf(c0f - sq_m), fabsf(c0f + SD - sq_m)) >=
                 prec_fp;
    }
    const int cap_eff = prec ? box_cap / 2 : box_cap;  // int2 entries
    const int ci = (ext8[0] > ext8[1] || box_size(0, SD) <= cap_eff) ? 0 : 1;
    if (ci) {  // CTA-uniform: the half-depth candidate, reduced now
      if (has) kbc[1] = chunk_end(1);
      extents(ext8, 1);
      __syncthreads();
    }
    const int S = SD >> ci;
    const int c_lo = dir > 0 ? cur : cur - S + 1;
    cur += dir * S;
    const int ka = k;
    const int kb = ci ? kbc[1] : kbc[0];  // (no local-memory array)
    k = kb;
    const bool any = kb > ka;
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
    // Shared layout: the transverse axis is innermost, so the 32 lanes of a
    // warp (adjacent detector columns = adjacent T) hit distinct banks:
    //   M = y: [z][y][x] (x = T, unit stride; x-quads contiguous)
    //   M = x: [z][x][y] (y = T, unit stride)
    // Matched: the T rows are padded to a multiple of 32 words, so the M and
    // z pitches are multiples of 32 and a warp's deposits (lanes in two M
    // cells / z rows) collide only where their T cells agree mod 32 -- 12%
    // fewer ATOMS wavefronts in the bank model (tools/sim_smem_banks.py:
    // 2.28 vs 2.58 per deposit).  Ax: odd x pitch (its box fill writes
    // x-quads across a warp, which a 32-word pitch would put in one bank).
    const int sx = M == 1 ? 1 : (tpad ? (bn[1] + tpad) & ~tpad : (bn[1] | 1));
    const int sy = M == 1 ? (bn[0] + tpad) & ~tpad : 1;
    const int sz = M == 1 ? sy * bn[1] : bn[0] * sx;
    const int bsize = sz * bn[2];
    const bool fits = !mixed && bsize <= cap_eff;
    const int qpr = bn[0] >> 2;            // x-quads per (y, z) row
    const int nquads = qpr * bn[1] * bn[2];
    const float inv_q = 1.f / (float)qpr, inv_y = 1.f / (float)bn[1];
    // quad qi -> (x0 = 4 xq, y, z) box coordinates
    auto quad_coords = [&](int qi, int& xq, int& by, int& bz) {
      int row = (int)((float)qi * inv_q);
      xq = qi - row * qpr;
      if (xq < 0) { row--; xq += qpr; } else if (xq >= qpr) { row++; xq -= qpr; }
      bz = (int)((float)row * inv_y);
      by = row - bz * bn[1];
      if (by < 0) { bz--; by += bn[1]; } else if (by >= bn[1]) { bz++; by -= bn[1]; }
    };
    // Every thread walks quads tid, tid + 256, ...: decompose the first,
    // then advance incrementally (stride = drow rows + dq quads).
    int drow, dq;
    {
      drow = (int)((float)ST_THREADS * inv_q);
      dq = ST_THREADS - drow * qpr;
      if (dq < 0) { drow--; dq += qpr; } else if (dq >= qpr) { drow++; dq -= qpr; }
    }
    auto quad_next = [&](int& xq, int& by, int& bz) {
      xq += dq;
      int r = drow;
      if (xq >= qpr) { xq -= qpr; r++; }
      by += r;
      while (by >= bn[1]) { by -= bn[1]; bz++; }
    };

    if (fits) {
      if (OP == OP_FWD) {
        int xq, by, bz;
        quad_coords(threadIdx.x, xq, by, bz);
        for (int qi = threadIdx.x; qi < nquads;
             qi += ST_THREADS, quad_next(xq, by, bz)) {
          const int gx = bo[0] + 4 * xq, gy = bo[1] + by, gz = bo[2] + bz;
          float4 q4 = make_float4(0.f, 0.f, 0.f, 0.f);
          if (gy >= 0 && gy < ny && gz >= z_lo && gz < z_hi) {
            const float* src = vol_in + (size_t)(gz - z_lo) * plane +
                               (size_t)gy * nx;
            if ((vec_ok & 1) && gx >= 0 && gx + 3 < nx) {
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
            *reinterpret_cast<float4*>(st_box + d) = q4;
          } else {
            st_box[d] = q4.x;
            st_box[d + sx] = q4.y;
            st_box[d + 2 * sx] = q4.z;
            st_box[d + 3 * sx] = q4.w;
          }
        }
      } else if (!CS_ST_ZOF) {
        const int nw = prec ? 2 * bsize : bsize;
        for (int i = threadIdx.x; i < nw; i += ST_THREADS) box_i[i] = 0;
      }
      if (OP == OP_FWD || !CS_ST_ZOF) __syncthreads();
    }
    // ---- samples of the chunk: one instantiation of the march per box
    // mode (MODE_BOX: one-word box / Ax box reads, MODE_PREC: two-word
    // box, MODE_GLOBAL: no box, straight from / to global memory), so the
    // CTA-uniform mode is not re-tested per sample
    auto march = [&](auto mode_tag) {
      constexpr int BM = decltype(mode_tag)::value;
      // exact fixed-point positions (common.cuh), integer-advanced; on the
      // staged path relative to the box origin (an exact integer shift), so
      // the cells index the box directly
      long long qx = q_at(m, ka, 0), qy = q_at(m, ka, 1), qz = q_at(m, ka, 2);
      if (BM != 2) {
        qx -= (long long)bo[0] << QF;
        qy -= (long long)bo[1] << QF;
        qz -= (long long)bo[2] << QF;
      }
#if CS_ST_ACC
      // (A/B) consecutive samples of a ray in the same cell: their fixed-
      // point taps are summed in registers and deposited when the cell
      // changes (integer sums: the same bits as per-sample deposits)
      int b_cur = -1;
      int a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0, a5 = 0, a6 = 0, a7 = 0;
      auto flush_acc = [&]() {
        atomicAdd(box_i + b_cur, a0);
        atomicAdd(box_i + b_cur + sx, a1);
        atomicAdd(box_i + b_cur + sy, a2);
        atomicAdd(box_i + b_cur + sy + sx, a3);
        atomicAdd(box_i + b_cur + sz, a4);
        atomicAdd(box_i + b_cur + sz + sx, a5);
        atomicAdd(box_i + b_cur + sz + sy, a6);
        atomicAdd(box_i + b_cur + sz + sy + sx, a7);
      };
#endif
#if CS_ST_UNROLL2
#pragma unroll 2
#endif
      for (int kk = ka; kk < kb;
           kk++, qx += m.Bq[0], qy += m.Bq[1], qz += m.Bq[2]) {
        const float wx = q_frac(qx), wy = q_frac(qy), wz = q_frac(qz);
        const int ix = q_cell(qx), iy = q_cell(qy), iz = q_cell(qz);
        if (BM != 2) {
          const int b = iz * sz + iy * sy + ix * sx;
          if (OP == OP_FWD) {
            const float s000 = st_box[b], s001 = st_box[b + sx];
            const float s010 = st_box[b + sy], s011 = st_box[b + sy + sx];
            const float s100 = st_box[b + sz], s101 = st_box[b + sz + sx];
            const float s110 = st_box[b + sz + sy];
            const float s111 = st_box[b + sz + sy + sx];
            const float r00 = fmaf(wx, s001 - s000, s000);
            const float r01 = fmaf(wx, s011 - s010, s010);
            const float r10 = fmaf(wx, s101 - s100, s100);
            const float r11 = fmaf(wx, s111 - s110, s110);
            const float b0 = fmaf(wy, r01 - r00, r00);
            const float b1 = fmaf(wy, r11 - r10, r10);
            acc += fmaf(wz, b1 - b0, b0);
          } else {
            float z0, z1, y00, y01, y10, y11;
            f2_split(f2_mul(f2(sv, sv), f2(1.f - wz, wz)), z0, z1);
            const f32x2 wyp = f2(1.f - wy, wy);
            f2_split(f2_mul(f2(z0, z0), wyp), y00, y01);
            f2_split(f2_mul(f2(z1, z1), wyp), y10, y11);
            const float vx = 1.f - wx;
            if (BM == 1) {
              deposit2(b, y00, vx);
              deposit2(b + sx, y00, wx);
              deposit2(b + sy, y01, vx);
              deposit2(b + sy + sx, y01, wx);
              deposit2(b + sz, y10, vx);
              deposit2(b + sz + sx, y10, wx);
              deposit2(b + sz + sy, y11, vx);
              deposit2(b + sz + sy + sx, y11, wx);
            } else {
              // the same products and magic adds as deposit(), two per
              // FMUL2 / FFMA2 (bit-identical taps)
              const f32x2 wxp = f2(vx, wx), mm = f2(ST_MAGIC, ST_MAGIC);
              float t0, t1;
#if CS_ST_ACC
              if (b != b_cur) {
                if (b_cur >= 0) flush_acc();
                b_cur = b;
                a0 = a1 = a2 = a3 = a4 = a5 = a6 = a7 = 0;
              }
              auto acc2 = [&](float y, int& lo, int& hi) {
                f2_split(f2_fma(f2(y, y), wxp, mm), t0, t1);
                lo += magic_int(t0);
                hi += magic_int(t1);
              };
              acc2(y00, a0, a1);
              acc2(y01, a2, a3);
              acc2(y10, a4, a5);
              acc2(y11, a6, a7);
              continue;
#endif
              auto dep2 = [&](int idx, float y, int dx) {
                f2_split(f2_fma(f2(y, y), wxp, mm), t0, t1);
                atomicAdd(box_i + idx, magic_int(t0));
                atomicAdd(box_i + idx + dx, magic_int(t1));
              };
              dep2(b, y00, sx);
              dep2(b + sy, y01, sx);
              dep2(b + sz, y10, sx);
              dep2(b + sz + sy, y11, sx);
            }
          }
        } else {
          // overflow path: straight from / to global memory
#pragma unroll
          for (int cz = 0; cz < 2; cz++) {
            const int zi = iz + cz;
            if (zi < z_lo || zi >= z_hi) continue;
            const float fz_ = cz ? wz : 1.f - wz;
#pragma unroll
            for (int cy = 0; cy < 2; cy++) {
              const int yi = iy + cy;
              if (yi < 0 || yi >= ny) continue;
              const float fy_ = cy ? wy : 1.f - wy;
#pragma unroll
              for (int cx = 0; cx < 2; cx++) {
                const int xi = ix + cx;
                if (xi < 0 || xi >= nx) continue;
                const float w = fz_ * fy_ * (cx ? wx : 1.f - wx);
                const size_t gi =
                    (size_t)(zi - z_lo) * plane + (size_t)yi * nx + xi;
                if (OP == OP_FWD)
                  acc = fmaf(w, __ldg(vol_in + gi), acc);
                else if (DET)
                  det_add(dacc + gi, val * (float)r.step * w, dscale);
                else
                  atomicAdd(vol_acc + gi, val * (float)r.step * w);
              }
            }
          }
        }
      }
#if CS_ST_ACC
      if (OP == OP_BWD && BM == 0 && b_cur >= 0) flush_acc();
#endif
    };
    if (any) {
      if (!fits)
        march(std::integral_constant<int, 2>());
      else if (OP == OP_BWD && prec)
        march(std::integral_constant<int, 1>());
      else
        march(std::integral_constant<int, 0>());
    }
    if (OP == OP_BWD && !DET && M == 1 && fits && !prec && (vec_ok & 2)) {
      // (A/B, CS_ST_BULK=1) flush through the TMA engine: the box's x-quads
      // are converted to fp32 in place (int 0 and +0.f share their bits, so
      // zero quads stay), then every in-grid (y, z) row of the box is added
      // into the volume by one cp.reduce.async.bulk .add.f32 (UBLKRED) from
      // shared memory -- no per-thread REDs through the LSU -- and the box
      // is zeroed for the next chunk once the engine has read it
      __syncthreads();
      const int qpr_ = bn[0] >> 2;
      const int nrow = bn[1] * bn[2];
      const int nq = qpr_ * nrow;
      const float rq = 1.f / (float)qpr_;
      for (int qi = threadIdx.x; qi < nq; qi += ST_THREADS) {
        const int row = small_div(qi, qpr_, rq);
        int* bp = box_i + row * sy + 4 * (qi - row * qpr_);
        const int4 q = *reinterpret_cast<const int4*>(bp);
        if (q.x | q.y | q.z | q.w)
          *reinterpret_cast<float4*>(bp) =
              make_float4((float)q.x * inv_scale, (float)q.y * inv_scale,
                          (float)q.z * inv_scale, (float)q.w * inv_scale);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      const int gx0 = max(bo[0], 0), gx1 = min(bo[0] + bn[0], nx);
      bool issued = false;
      if (gx1 > gx0) {
        const float rb1 = 1.f / (float)bn[1];
        const unsigned sbase = (unsigned)__cvta_generic_to_shared(
            box_i + (gx0 - bo[0]));
        const unsigned nbytes = (unsigned)(gx1 - gx0) * 4u;
        for (int row = threadIdx.x; row < nrow; row += ST_THREADS) {
          const int bz = small_div(row, bn[1], rb1);
          const int gy = bo[1] + row - bz * bn[1], gz = bo[2] + bz;
          if (gy < 0 || gy >= ny || gz < z_lo || gz >= z_hi) continue;
          float* gp = vol_acc + (size_t)(gz - z_lo) * plane +
                      (size_t)gy * nx + gx0;
          asm volatile(
              "cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 "
              "[%0], [%1], %2;" ::"l"(gp),
              "r"(sbase + 4u * (unsigned)(row * sy)), "r"(nbytes)
              : "memory");
          issued = true;
        }
      }
      if (issued) {
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
      __syncthreads();
      for (int qi = threadIdx.x; qi < nq; qi += ST_THREADS) {
        const int row = small_div(qi, qpr_, rq);
        *reinterpret_cast<int4*>(box_i + row * sy + 4 * (qi - row * qpr_)) =
            make_int4(0, 0, 0, 0);
      }
    } else if (OP == OP_BWD && fits) {
      __syncthreads();
      // flush the box: one 16-byte reduction per aligned x-quad.  A thread
      // owns one (x-quad, y) column of the box and walks it in z with
      // running shared / global pointers (the per-quad index arithmetic
      // was ~25% of the kernel's instructions), over the planes inside the
      // slab only.  Threads are laid along the box's unit-stride axis
      // (x-quads for M = y, y for M = x), so the shared loads of a warp do
      // not conflict.
      const int qpr_ = bn[0] >> 2;
      const int P = qpr_ * bn[1];                  // columns per z-plane
      const bool fold = P <= ST_THREADS;           // several z per pass
      const float rP = 1.f / (float)P;
      const int zstep = fold ? small_div(ST_THREADS, P, rP) : 1;
      const int z_first = fold ? small_div(threadIdx.x, P, rP) : 0;
      const int pstride = fold ? P : ST_THREADS;
      const int bz0 = max(0, z_lo - bo[2]), bz1 = min(bn[2], z_hi - bo[2]);
      int bzs = z_first;
      // zero-on-flush: every plane and row of the box is read (and zeroed);
      // only those inside the grid and slab are reduced into the volume
      if (!CS_ST_ZOF)
        while (bzs < bz0) bzs += zstep;
      const int bze = CS_ST_ZOF ? bn[2] : bz1;
      const float il = inv_scale / lo_scale;
      const int wps = prec ? 2 : 1;                // words per box voxel
      const int bstep = zstep * sz * wps;
      const size_t gstep = (size_t)zstep * plane;
      const float rq = 1.f / (float)(M == 1 ? qpr_ : bn[1]);
      for (int cp = fold ? threadIdx.x - z_first * P : threadIdx.x;
           z_first < zstep && cp < P; cp += pstride) {
        int xq, by;
        if (M == 1) {
          by = small_div(cp, qpr_, rq);
          xq = cp - by * qpr_;
        } else {
          xq = small_div(cp, bn[1], rq);
          by = cp - xq * bn[1];
        }
        const int gx = bo[0] + 4 * xq, gy = bo[1] + by;
        const bool row_in = gy >= 0 && gy < ny;
        if (!CS_ST_ZOF && !row_in) continue;
        const bool vec = (vec_ok & 1) && gx >= 0 && gx + 3 < nx;
        const int* bp = box_i + (by * sy + 4 * xq * sx + bzs * sz) * wps;
        float* gp = vol_acc + (size_t)(bo[2] + bzs - z_lo) * plane +
                    (size_t)gy * nx + gx;
        const int sxw = sx * wps;
        for (int bz = bzs; bz < bze; bz += zstep, bp += bstep, gp += gstep) {
          float f0, f1, f2, f3;
          int* bw = const_cast<int*>(bp);
          if (prec) {
            int2 q0, q1, q2, q3;
            if (M == 1) {
              const int4 a01 = *reinterpret_cast<const int4*>(bp);
              const int4 a23 = *reinterpret_cast<const int4*>(bp + 4);
              q0 = make_int2(a01.x, a01.y); q1 = make_int2(a01.z, a01.w);
              q2 = make_int2(a23.x, a23.y); q3 = make_int2(a23.z, a23.w);
            } else {
              q0 = *reinterpret_cast<const int2*>(bp);
              q1 = *reinterpret_cast<const int2*>(bp + sxw);
              q2 = *reinterpret_cast<const int2*>(bp + 2 * sxw);
              q3 = *reinterpret_cast<const int2*>(bp + 3 * sxw);
            }
            if ((q0.x | q0.y | q1.x | q1.y | q2.x | q2.y | q3.x | q3.y) == 0)
              continue;
            if (CS_ST_ZOF) {
              if (M == 1) {
                *reinterpret_cast<int4*>(bw) = make_int4(0, 0, 0, 0);
                *reinterpret_cast<int4*>(bw + 4) = make_int4(0, 0, 0, 0);
              } else {
                for (int j = 0; j < 4; j++)
                  *reinterpret_cast<int2*>(bw + j * sxw) = make_int2(0, 0);
              }
              if (!row_in || bz < bz0 || bz >= bz1) continue;
            }
            f0 = fmaf((float)q0.y, il, (float)q0.x * inv_scale);
            f1 = fmaf((float)q1.y, il, (float)q1.x * inv_scale);
            f2 = fmaf((float)q2.y, il, (float)q2.x * inv_scale);
            f3 = fmaf((float)q3.y, il, (float)q3.x * inv_scale);
          } else {
            int q0, q1, q2, q3;
            if (M == 1) {
              const int4 q = *reinterpret_cast<const int4*>(bp);
              q0 = q.x; q1 = q.y; q2 = q.z; q3 = q.w;
            } else {
              q0 = bp[0];
              q1 = bp[sxw];
              q2 = bp[2 * sxw];
              q3 = bp[3 * sxw];
            }
            if ((q0 | q1 | q2 | q3) == 0) continue;
            if (CS_ST_ZOF) {
              if (M == 1) {
                *reinterpret_cast<int4*>(bw) = make_int4(0, 0, 0, 0);
              } else {
                for (int j = 0; j < 4; j++) bw[j * sxw] = 0;
              }
              if (!row_in || bz < bz0 || bz >= bz1) continue;
            }
            f0 = (float)q0 * inv_scale; f1 = (float)q1 * inv_scale;
            f2 = (float)q2 * inv_scale; f3 = (float)q3 * inv_scale;
          }
          if (DET) {
            const float f[4] = {f0, f1, f2, f3};
            long long* dp = dacc + (gp - vol_acc);
#pragma unroll
            for (int j = 0; j < 4; j++)
              if (gx + j >= 0 && gx + j < nx) det_add(dp + j, f[j], dscale);
          } else if (vec) {
            st_red4(gp, f0, f1, f2, f3);
          } else {
            const float f[4] = {f0, f1, f2, f3};
#pragma unroll
            for (int j = 0; j < 4; j++)
              if (gx + j >= 0 && gx + j < nx && f[j] != 0.f)
                atomicAdd(gp + j, f[j]);
          }
        }
      }
    }
  }
  if (OP == OP_FWD && valid) {
    const float outv = acc * (float)r.step;
    if (MODE == 0)
      out[pix] = outv;
    else if (MODE == 1)
      out[pix] += outv;
    else
      out[pix] = (rw ? rw[pix] : 1.f) * (rb[pix] - outv);
  }
}

// Smallest footprint of a detector pixel on the grid, in voxels (pixels
// nearest the source are smallest: magnification dsd / (dso - r)).
static double min_pixel_footprint(const double* grid6, int nx, int ny,
                                  int nz, const double* geom, int n_a,
                                  int n_u, int n_v) {
  const double ex = nx * grid6[3], ey = ny * grid6[4], ez = nz * grid6[5];
  const double gc[3] = {grid6[0] + 0.5 * ex, grid6[1] + 0.5 * ey,
                        grid6[2] + 0.5 * ez};
  const double rad = 0.5 * sqrt(ex * ex + ey * ey + ez * ez);
  const double vmax = fmax(grid6[3], fmax(grid6[4], grid6[5]));
  double fp = 1e300;
  for (int a = 0; a < n_a; a++) {
    const double* g = geom + 12 * a;
    const double du = sqrt(g[6] * g[6] + g[7] * g[7] + g[8] * g[8]);
    const double dv = sqrt(g[9] * g[9] + g[10] * g[10] + g[11] * g[11]);
    double c[3], s2c[3];
    for (int i = 0; i < 3; i++) {
      c[i] = g[3 + i] + 0.5 * (n_u - 1) * g[6 + i] +
             0.5 * (n_v - 1) * g[9 + i] - g[i];
      s2c[i] = gc[i] - g[i];
    }
    const double dsd = sqrt(c[0] * c[0] + c[1] * c[1] + c[2] * c[2]);
    const double dso = sqrt(s2c[0] * s2c[0] + s2c[1] * s2c[1] + s2c[2] * s2c[2]);
    const double near = fmax(dso - rad, 1e-6 * dsd);
    fp = fmin(fp, fmin(du, dv) * near / dsd / vmax);
  }
  return fp;
}

// Fixed-point budget for matched deposits: the int32 box must hold the
// largest per-voxel chunk sum.  A voxel's trilinear support (2 voxels per
// axis) is crossed by at most (2 / footprint + 1)^2 rays and each ray puts
// at most (2 / min step + 1) samples of weight <= 1 into it; the footprint
// of a pixel is smallest nearest the source (magnification dsd / (dso - r)).
// Returns the scale numerator: per CTA, scale = budget / max|val * step|.
static float fixed_point_budget(const double* grid6, int nx, int ny, int nz,
                                const double* geom, int n_a, int n_u, int n_v,
                                double step_max, double* taps_bound = nullptr) {
  const double vmax = fmax(grid6[3], fmax(grid6[4], grid6[5]));
  double fp = min_pixel_footprint(grid6, nx, ny, nz, geom, n_a, n_u, n_v);
  fp = fmax(fp, 1e-3);
  const double rays = (2.0 / fp + 1.0) * (2.0 / fp + 1.0);
  const double samples = 2.0 * vmax / (0.5 * step_max) + 1.0;
  const double bound = fmin(rays, (double)ST_THREADS) * samples;
  if (taps_bound) *taps_bound = bound;
  // per-voxel |sum| <= 2e9 < 2^31.  The bound counts every sample of a
  // ray in the 2x2x2 support at weight 1; the weights of one ray through
  // the support sum to at most 1 / step + 1 <= 4 / vmin + 1 voxels' worth
  // (step >= step_max / 2), against the 4 vmax / step_max + 1 = 8 + 1
  // counted here, so the true sum stays under ~1.1e9.
  double b = 2.0e9 / bound;
  // every tap |val * step * w| * scale <= b must stay below 2^22 for the
  // magic-number conversion (ST_MAGIC): resolution 2.5e-7 of the CTA's
  // largest tap
  if (b > ST_BUDGET_CAP) b = ST_BUDGET_CAP;
  return (float)b;
}

}  // namespace cs

using namespace cs;

namespace cs {

static size_t staged_smem_cap() {
  static size_t cap = 0;
  if (!cap) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin,
                           dev);
    cap = optin > 0 ? (size_t)optin : 48 * 1024;
  }
  return cap;
}

// vol[z][y][x] += acc_t[z][x][y] over a slab (32 x 32 tiles through shared
// memory, coalesced on both sides): the x-major views' matched Atb, computed
// in the transposed frame, added into the volume (launch_staged).
__global__ void __launch_bounds__(256)
    transpose_add_kernel(float* __restrict__ vol,
                         const float* __restrict__ acc_t, int nx, int ny) {
  __shared__ float tile[32][33];
  const size_t plane = (size_t)nx * ny;
  const float* src = acc_t + (size_t)blockIdx.z * plane;
  float* dst = vol + (size_t)blockIdx.z * plane;
  const int x0 = blockIdx.y * 32, y0 = blockIdx.x * 32;
  // read acc_t rows x (length ny), columns y
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int x = x0 + i, y = y0 + threadIdx.x;
    tile[i][threadIdx.x] = (x < nx && y < ny) ? src[(size_t)x * ny + y] : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int y = y0 + i, x = x0 + threadIdx.x;
    if (x < nx && y < ny) dst[(size_t)y * nx + x] += tile[threadIdx.x][i];
  }
}

// Deterministic matched Atb (see det_add): the launch's max |proj| (float
// bits of non-negative values order like unsigned ints), and the final
// vol += acc / S.
__global__ void __launch_bounds__(256)
    abs_max_kernel(const float* __restrict__ x, size_t n,
                   unsigned* __restrict__ out) {
  float m = 0.f;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    m = fmaxf(m, fabsf(x[i]));
  for (int o = 16; o > 0; o >>= 1)
    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.f) atomicMax(out, __float_as_uint(m));
}

__global__ void det_scale_kernel(const unsigned* __restrict__ gmax_bits,
                                 double det_c, double* __restrict__ S) {
  const float g = __uint_as_float(*gmax_bits);
  *S = g > 0.f ? exp2(floor(log2(det_c / (double)g))) : 0.0;
}

__global__ void __launch_bounds__(256)
    det_finish_kernel(float* __restrict__ vol, const long long* __restrict__ acc,
                      size_t n, const double* __restrict__ dscale) {
  const double S = *dscale;
  if (S == 0.0) return;
  const double inv = 1.0 / S;   // a power of two: exact
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const long long q = acc[i];
    if (q) vol[i] += (float)((double)q * inv);
  }
}

// Deterministic mode with the transposed frame: vol[z][y][x] += (acc[z][y][x]
// + acc_t[z][x][y]) / S -- the two integer accumulators (same S) summed
// exactly, then rounded once like det_finish_kernel (32 x 32 tiles of acc_t
// through shared memory, coalesced on both sides).
__global__ void __launch_bounds__(256)
    det_finish_t_kernel(float* __restrict__ vol,
                        const long long* __restrict__ acc,
                        const long long* __restrict__ acc_t, int nx, int ny,
                        const double* __restrict__ dscale) {
  __shared__ long long tile[32][33];
  const double S = *dscale;
  const size_t plane = (size_t)nx * ny;
  const long long* src = acc_t + (size_t)blockIdx.z * plane;
  const int x0 = blockIdx.y * 32, y0 = blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int x = x0 + i, y = y0 + threadIdx.x;
    tile[i][threadIdx.x] = (x < nx && y < ny) ? src[(size_t)x * ny + y] : 0;
  }
  __syncthreads();
  if (S == 0.0) return;
  const double inv = 1.0 / S;   // a power of two: exact
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int y = y0 + i, x = x0 + threadIdx.x;
    if (x < nx && y < ny) {
      const size_t gi = (size_t)blockIdx.z * plane + (size_t)y * nx + x;
      const long long q = acc[gi] + tile[threadIdx.x][i];
      if (q) vol[gi] += (float)((double)q * inv);
    }
  }
}

static int g_deterministic = -1;   // -1: CS_ST_DETERMINISTIC decides

static bool deterministic_matched() {
  if (g_deterministic < 0) {
    const char* k = getenv("CS_ST_DETERMINISTIC");
    g_deterministic = (k && k[0] == '1') ? 1 : 0;
  }
  return g_deterministic == 1;
}

// Launch one staged pass over n_a views (OP_FWD: Ax into out with MODE
// epilogue; OP_BWD: matched Atb into vol_acc).
template <int OP, int MODE>
int launch_staged(const float* vol_in, float* vol_acc, int nx, int ny, int nz,
                  int z_lo, int z_hi, const double* grid6, const double* geom,
                  int n_a, int n_u, int n_v, double step_max, float* out,
                  const float* proj_in, const float* rb, const float* rw,
                  cudaStream_t s) {
  const Grid G = make_grid(grid6, nx, ny, nz);
  AngleGeom* dgeom = nullptr;
  int rc = upload_geometry(geom, n_a, s, &dgeom);
  if (rc) return rc;
  int* ids_h = (int*)malloc(sizeof(int) * (size_t)n_a);
  int nxm = 0;
  for (int a = 0; a < n_a; a++)
    if (view_axis(geom + 12 * a, n_u, n_v) == 0) ids_h[nxm++] = a;
  int nall = nxm;
  for (int a = 0; a < n_a; a++)
    if (view_axis(geom + 12 * a, n_u, n_v) == 1) ids_h[nall++] = a;
  int* ids = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&ids, sizeof(int) * n_a, s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(ids, ids_h, sizeof(int) * n_a, cudaMemcpyHostToDevice,
                        s);
  free(ids_h);
  if (e != cudaSuccess) {
    release_geometry(dgeom, s);
    CS_CHECK_CUDA(e);
  }
  // Occupancy by slab size (r01 A/B, matched, 32-360 views): 4 CTAs/SM x
  // 54 KB boxes win up to 512^3 (+2-4%), 3 x 64 KB above (+4% at 768^3, +5%
  // at 1024^3, +10% at 2048^3: the smaller boxes take more half-depth chunks
  // and flushes, which cost more once the slab is far beyond L2).  5 CTAs
  // (48 registers) spill.
  static const char* tp_env = getenv("CS_ST_TPAD");
  const bool padded = OP == OP_BWD && !(tp_env && atoi(tp_env) == 0);
  // Matched, x-major views: run as y-major views of the transposed frame
  // when the device has room for a slab-sized accumulator (see the launch
  // below; knob CS_ST_TRANSPOSE=0 disables).
  bool use_t = false;
  const size_t plane_bytes = (size_t)nx * ny * sizeof(float);
  const size_t slab_bytes = (size_t)(z_hi - z_lo) * plane_bytes;
  const bool det = OP == OP_BWD && deterministic_matched();
  int t_planes = z_hi - z_lo;  // planes per transposed-frame piece
  if (OP == OP_BWD && nxm > 0) {
    // deterministic mode: two int64 accumulators (direct + transposed)
    static const char* tk = getenv("CS_ST_TRANSPOSE");
    size_t free_b = 0, total_b = 0;
    const size_t margin = (size_t)4 << 30;
    if (!(tk && tk[0] == '0') &&
        cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
      if (free_b > (det ? 4 : 1) * slab_bytes + margin) {
        use_t = true;
      } else if (!det && free_b > margin) {
        // no room for a slab-sized accumulator (e.g. a 2048^3 slab beside
        // its cached Ax textures): the x-major views in z pieces of the
        // slab, each into a piece-sized accumulator; pieces of at least
        // 64 planes and 1/8 of the slab (thinner ones re-walk too many
        // rays per plane)
        const size_t fit = (free_b - margin) / plane_bytes;
        const size_t need = (size_t)max(64, (z_hi - z_lo + 7) / 8);
        if (fit >= need) {
          use_t = true;
          t_planes = (int)fit;
        }
      }
      // (test knob) CS_ST_TPIECE=n: z pieces of n planes
      static const char* tp_piece = getenv("CS_ST_TPIECE");
      if (use_t && !det && tp_piece && atoi(tp_piece) > 0)
        t_planes = atoi(tp_piece);
    }
  }
  // Occupancy: with every matched view y-major (transposed frame) 4 CTAs x
  // 54 KB win (512^3: 250.6 vs 243.2 GUPS dense for 3 x 72 KB; 1024^3: 261.9
  // vs 254.4; profiles/ab_matched_occupancy_r02ad.jsonl); x-major boxes in
  // their own frame (y rows padded to 32 words) need 3 x 72 KB.
  static const char* four_knob = getenv("CS_ST_FOUR");  // A/B: 4 CTAs/SM
  bool four =
      four_knob ? four_knob[0] == '1'
                : (padded ? (use_t || nxm == 0)
                          : (double)(z_hi - z_lo) * nx * ny <= 134217728.0);
  static const char* kb_knob = getenv("CS_STAGED_SMEM_KB");
  // (3 CTAs: 72 KB boxes, +1-3% over 64 KB at 1024^3 / 2048^3; 80 KB no
  // longer fits three)
  size_t smem = (kb_knob ? (size_t)atoi(kb_knob) : four ? 54 : 72) * 1024;
  int cap = (int)(smem / sizeof(float));
  double taps = 1.0;
  const float budget =
      OP == OP_BWD ? fixed_point_budget(grid6, nx, ny, nz, geom, n_a, n_u, n_v,
                                        step_max, &taps)
                   : 0.f;
  // Precise (two-word) boxes: everywhere when the int32 budget falls below
  // the magic-add cap (many rays per voxel: the coarse unit gives up
  // resolution that the residual word restores), else per chunk (the
  // kernel's edge / ray-gap rule).  Knobs: CS_ST_PRECISE=0|1|auto,
  // CS_ST_PRECISE_FP (ray gap in voxels; default 1.9 below 8 views).
  static const char* pk = getenv("CS_ST_PRECISE");
  static const char* pf = getenv("CS_ST_PRECISE_FP");
  int prec_mode = 0;
  if (pk && pk[0] == '1') prec_mode = 1;
  if (pk && pk[0] == '0') prec_mode = 2;
  if (OP == OP_BWD && budget < ST_BUDGET_CAP && prec_mode != 2) prec_mode = 1;
  // the ray-gap rule (voxels between rays >= prec_fp voxels apart can get
  // only tiny weights from every view) only matters when few views cover a
  // voxel: on by default for launches of < 8 views (OS-SART blocks of a
  // few views), any launch with the knob
  const float prec_fp = pf ? (float)atof(pf) : (n_a < 8 ? 1.9f : 1e30f);
  // residual scale 2^k: |residual| <= 1/2 per tap and at most `taps` taps
  // per voxel and chunk, so the residual word stays below 2^30
  int lo_k = 16;
  while (lo_k > 0 && taps * ldexp(0.5, lo_k) >= 1073741824.0) lo_k--;
  const float lo_scale = ldexpf(1.f, lo_k);
  int edge = 0;
  if (OP == OP_BWD) {
    const double fp = min_pixel_footprint(grid6, nx, ny, nz, geom, n_a, n_u,
                                          n_v);
    edge = (int)fmin(ceil(1.0 / fmax(fp, 1e-3)) + 1.0, (double)max(n_u, n_v));
  }
  const void* vbase = OP == OP_BWD ? (const void*)vol_acc : (const void*)vol_in;
  // bit 0: 16-byte volume rows; bit 1: matched bulk-reduce flush (A/B knob
  // CS_ST_BULK=1, y-major boxes, see the kernel)
  static const char* bulk_knob = getenv("CS_ST_BULK");
  const int bulk = OP == OP_BWD && bulk_knob && bulk_knob[0] == '1' ? 2 : 0;
  const int vec_ok = (nx % 4 == 0) && (((uintptr_t)vbase & 15) == 0)
                         ? 1 | bulk : 0;
  // v-band culling per main-axis class (runtime.cu slab_row_band); the
  // overwrite-mode Ax zeroes the culled rows
  int band[2][2] = {{0, n_v}, {0, n_v}};
  if (cull_enabled() && MODE != 2) {
    double* gsub = (double*)malloc(sizeof(double) * 12 * (size_t)n_a);
    for (int c = 0; c < 2; c++) {
      const int lo = c == 0 ? 0 : nxm, hi = c == 0 ? nxm : nall;
      ids_h = (int*)malloc(sizeof(int) * (size_t)n_a);
      int m = 0;
      for (int a = 0; a < n_a; a++)
        if (view_axis(geom + 12 * a, n_u, n_v) == c) ids_h[m++] = a;
      for (int i = 0; i < m; i++)
        memcpy(gsub + 12 * i, geom + 12 * ids_h[i], 12 * sizeof(double));
      free(ids_h);
      if (hi > lo)
        slab_row_band(gsub, hi - lo, G, z_lo, z_hi, n_v, &band[c][0],
                      &band[c][1]);
    }
    free(gsub);
    if (OP == OP_FWD && MODE == 0) {
      // rows outside a class's band are zero for that class's views;
      // zero outside the union (rows inside it are written by the kernels
      // of both classes or lie in one class's band)
      int v0 = n_v, v1 = 0;
      for (int c = 0; c < 2; c++)
        if ((c == 0 ? nxm : nall - nxm) > 0) {
          v0 = min(v0, band[c][0]);
          v1 = max(v1, band[c][1]);
        }
      if (v1 < v0) v0 = v1 = 0;
      for (int c = 0; c < 2; c++) {
        // launch rows as the union so every view's rows are written
        band[c][0] = v0;
        band[c][1] = v1;
      }
      rc = zero_rows_outside(out, n_a, n_u, n_v, v0, v1, s);
      if (rc) {
        cudaFreeAsync(ids, s);
        release_geometry(dgeom, s);
        return rc;
      }
    }
  }
  // lane stride from the finest pixel footprint fp (fixed_point_budget's
  // geometry): s fp <= 1/2 voxel between neighbouring lanes.  Measured on
  // 256^3 with 512^2 / 1024^2 / 2048^2 detectors (fp = 0.4 / 0.2 / 0.1):
  // s = 2 loses 8% at fp = 0.4; s = 2 / 4 gain 3% / 55% at fp = 0.2 / 0.1
  int lane_stride = 1;
  if (OP == OP_BWD) {
    const double fp = min_pixel_footprint(grid6, nx, ny, nz, geom, n_a, n_u,
                                          n_v);
    while (lane_stride < ST_TV && fp * lane_stride * 4 <= 1.0)
      lane_stride *= 2;
  }
  static const char* ls_knob = getenv("CS_ST_LANE_STRIDE");  // A/B knob
  if (ls_knob) {
    const int k = atoi(ls_knob);
    if (k == 1 || k == 2 || k == 4 || k == 8) lane_stride = k;
  }
  // matched T-pitch padding (power of two minus one; A/B knob CS_ST_TPAD)
  static const char* tp_knob = getenv("CS_ST_TPAD");
  const int tpad = OP == OP_BWD ? (tp_knob ? atoi(tp_knob) : 31) : 0;
  const unsigned gx = (n_u + ST_TU * lane_stride - 1) / (ST_TU * lane_stride);
  // matched view pairs per CTA (see the kernel; A/B knob CS_ST_PAIR=1, off
  // by default: dense 180 views at 256^3 / 512^3 / 1024^3: 224.4 / 260.4 /
  // 274.7 vs 216.7 / 263.6 / 282.0 GUPS -- the shared box shrinks only to
  // ~0.7x (the views' footprints are shifted, the rays' z drift over a
  // 14-plane chunk remains), profiles/ab_matched_view_pairs_r02bp.jsonl);
  // with lane stride 1 and without the few-view ray-gap rule (its source
  // position is per view)
  static const char* pair_knob = getenv("CS_ST_PAIR");
  const int vpair = OP == OP_BWD && lane_stride == 1 && prec_fp >= 1e29f &&
                    pair_knob && pair_knob[0] == '1';
  auto rows = [&](int c) {
    const int rv = vpair ? ST_TV / 2 : ST_TV / lane_stride;
    return (unsigned)((band[c][1] - band[c][0] + rv - 1) / rv);
  };
  auto nviews = [&](int n) { return (unsigned)(vpair ? (n + 1) / 2 : n); };
  // matched chunk depth: 14 planes with 3 CTAs x 72 KB boxes for planes of
  // >= 512^2 voxels (512^3: 261.6 vs 249.1 GUPS dense for 8 planes at 4 x 54
  // KB, 1024^3: 271.6 vs 262.1, 2048^3 x 32 views: 260.5 vs 263.9), else 8
  // (256^3: 165 vs 189; profiles/ab_matched_depth_r02ai.jsonl)
  static const char* deep_knob = getenv("CS_ST_DEEP");  // A/B: 0 / 1
  const bool deep =
      OP == OP_BWD && padded && !(four_knob || kb_knob) &&
      (deep_knob ? deep_knob[0] == '1'
                 : (use_t || nxm == 0) && (double)nx * ny >= 262144.0);
  if (deep) {
    four = false;
    smem = 72 * 1024;
    cap = (int)(smem / sizeof(float));
  }
  auto grid_of = [&](unsigned tu, unsigned tv, unsigned nv) {
    return (OP == OP_BWD && CS_ST_VIEWFAST) ? dim3(nv, tu, tv) : dim3(tu, tv, nv);
  };
  // DM: the deterministic matched instantiation (MODE 3; == MODE for Ax)
  constexpr int DM = OP == OP_BWD ? 3 : MODE;
  auto k0 = deep ? (det ? staged_kernel<OP, 0, DM, 3, ST_S_DEEP>
                        : staged_kernel<OP, 0, MODE, 3, ST_S_DEEP>)
            : four ? (det ? staged_kernel<OP, 0, DM, 4>
                          : staged_kernel<OP, 0, MODE, 4>)
                   : (det ? staged_kernel<OP, 0, DM, 3>
                          : staged_kernel<OP, 0, MODE, 3>);
  auto k1 = deep ? (det ? staged_kernel<OP, 1, DM, 3, ST_S_DEEP>
                        : staged_kernel<OP, 1, MODE, 3, ST_S_DEEP>)
            : four ? (det ? staged_kernel<OP, 1, DM, 4>
                          : staged_kernel<OP, 1, MODE, 4>)
                   : (det ? staged_kernel<OP, 1, DM, 3>
                          : staged_kernel<OP, 1, MODE, 3>);
  // the dynamic shared-memory opt-in is per device: set it once on each
  // (the executor drives several GPUs from one process)
  static std::atomic<unsigned long long> attr_done{0};
  int dev_ord = 0;
  cudaGetDevice(&dev_ord);
  const unsigned long long bit = 1ull << (dev_ord & 63);
  if (!(attr_done.load() & bit)) {
    for (auto k : {staged_kernel<OP, 0, MODE, 3>, staged_kernel<OP, 1, MODE, 3>,
                   staged_kernel<OP, 0, MODE, 4>, staged_kernel<OP, 1, MODE, 4>,
                   staged_kernel<OP, 0, MODE, 3, ST_S_DEEP>,
                   staged_kernel<OP, 1, MODE, 3, ST_S_DEEP>,
                   staged_kernel<OP, 0, DM, 3>, staged_kernel<OP, 1, DM, 3>,
                   staged_kernel<OP, 0, DM, 4>, staged_kernel<OP, 1, DM, 4>,
                   staged_kernel<OP, 0, DM, 3, ST_S_DEEP>,
                   staged_kernel<OP, 1, DM, 3, ST_S_DEEP>})
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           200 * 1024);
    attr_done.fetch_or(bit);
  }
  // Matched, x-major views: run them as y-major views of the transposed
  // frame (x <-> y swapped in the geometry and grid) into a transposed slab
  // accumulator, then add it back transposed.  The sample positions, taps
  // and box sums are exactly those of the direct launch (the fp64 set-up is
  // symmetric in x and y); only the fp32 summation into the volume is
  // grouped differently.  The y-major layout flushes x-quads with one
  // LDS.128 and contiguous REDs, where the x-major one needs four LDS and
  // spreads a warp's REDs over 32 rows: 34.2 vs 24.3 ms per 45 views at
  // 512^3 (profiles/ncu_r02w.md).  Needs a slab-sized buffer: used when the
  // device has room for it (knob CS_ST_TRANSPOSE=0 disables).
  // deterministic mode: a slab-sized int64 accumulator, plus a transposed
  // one for the x-major views when they run in the transposed frame (both
  // in units of the same S, summed exactly by det_finish_t_kernel)
  long long* dacc = nullptr;
  long long* dacc_t = nullptr;  // deterministic + transposed frame
  unsigned* dgmax = nullptr;   // [0]: max |proj| bits; [2..3]: S (double)
  double* dscale = nullptr;
  double det_c = 0.0;
  if (det) {
    const size_t nvox = (size_t)(z_hi - z_lo) * nx * ny;
    double fp = fmax(min_pixel_footprint(grid6, nx, ny, nz, geom, n_a, n_u,
                                         n_v), 1e-3);
    const double vmax = fmax(grid6[3], fmax(grid6[4], grid6[5]));
    const double taps_all = (2.0 / fp + 1.0) * (2.0 / fp + 1.0) *
                            (2.0 * vmax / (0.5 * step_max) + 1.0);
    det_c = ldexp(1.0, 62) / (2.0 * n_a * step_max * taps_all);
    cudaError_t ed = cudaMallocAsync((void**)&dacc, nvox * sizeof(long long),
                                     s);
    if (ed == cudaSuccess)
      ed = cudaMallocAsync((void**)&dgmax, 4 * sizeof(unsigned), s);
    if (ed == cudaSuccess)
      ed = cudaMemsetAsync(dacc, 0, nvox * sizeof(long long), s);
    if (ed == cudaSuccess) ed = cudaMemsetAsync(dgmax, 0, sizeof(unsigned), s);
    if (ed == cudaSuccess) {
      dscale = reinterpret_cast<double*>(dgmax + 2);
      abs_max_kernel<<<num_sms() * 4, 256, 0, s>>>(
          proj_in, (size_t)n_a * n_u * n_v, dgmax);
      CS_COUNT_LAUNCH();
      det_scale_kernel<<<1, 1, 0, s>>>(dgmax, det_c, dscale);
      CS_COUNT_LAUNCH();
      ed = cudaGetLastError();
    }
    if (ed != cudaSuccess) {
      if (dacc) cudaFreeAsync(dacc, s);
      if (dgmax) cudaFreeAsync(dgmax, s);
      cudaFreeAsync(ids, s);
      release_geometry(dgeom, s);
      CS_CHECK_CUDA(ed);
    }
  }
  bool transposed = false;
  if (use_t && rows(0) > 0) {
    double* geom_t = (double*)malloc(sizeof(double) * 12 * (size_t)n_a);
    memcpy(geom_t, geom, sizeof(double) * 12 * (size_t)n_a);
    for (int a = 0; a < n_a; a++)
      for (int c = 0; c < 12; c += 3) {
        double* g3 = geom_t + 12 * a + c;
        const double t = g3[0];
        g3[0] = g3[1];
        g3[1] = t;
      }
    double grid6_t[6] = {grid6[1], grid6[0], grid6[2],
                         grid6[4], grid6[3], grid6[5]};
    const Grid GT = make_grid(grid6_t, ny, nx, nz);
    AngleGeom* dgeom_t = nullptr;
    float* acc_t = nullptr;
    const size_t acc_bytes =
        det ? 2 * slab_bytes
            : (size_t)min(t_planes, z_hi - z_lo) * plane_bytes;
    rc = upload_geometry(geom_t, n_a, s, &dgeom_t);
    free(geom_t);
    cudaError_t e2 = rc ? cudaErrorUnknown
                        : cudaMallocAsync((void**)&acc_t, acc_bytes, s);
    if (!rc && e2 == cudaSuccess)
      e2 = cudaMemsetAsync(acc_t, 0, acc_bytes, s);
    if (!rc && e2 == cudaSuccess) {
      const int vec_t = (ny % 4 == 0) ? 1 | bulk : 0;
      // deterministic: acc_t is the transposed int64 accumulator (passed as
      // both the offset base and dacc; the kernel never stores floats there)
      // and covers the whole slab; otherwise z pieces of t_planes planes,
      // each accumulated and transposed-added before the next reuses acc_t
      for (int zl = z_lo; zl < z_hi; zl += t_planes) {
        const int zh = min(z_hi, zl + t_planes);
        if (!det && zl > z_lo) {
          e2 = cudaMemsetAsync(acc_t, 0, (size_t)(zh - zl) * plane_bytes, s);
          if (e2 != cudaSuccess) break;
        }
        k1<<<grid_of(gx, rows(0), nviews(nxm)), ST_THREADS, smem, s>>>(
            vol_in, acc_t, dgeom_t, ids, GT, step_max, zl, zh, n_u, n_v,
            band[0][0], band[0][1], out, proj_in, rb, rw, cap, budget, vec_t,
            lane_stride, prec_mode, prec_fp, edge, lo_scale, tpad,
            det ? reinterpret_cast<long long*>(acc_t) : nullptr,
            det ? dscale : nullptr, vpair, nxm);
        CS_COUNT_LAUNCH();
        if (!det) {
          const dim3 tg((ny + 31) / 32, (nx + 31) / 32, zh - zl);
          transpose_add_kernel<<<tg, dim3(32, 8), 0, s>>>(
              vol_acc + (size_t)(zl - z_lo) * nx * ny, acc_t, nx, ny);
          CS_COUNT_LAUNCH();
        }
      }
      if (det) dacc_t = reinterpret_cast<long long*>(acc_t);  // finished below
      const cudaError_t e3 = e2 != cudaSuccess ? e2 : cudaGetLastError();
      if (!det) cudaFreeAsync(acc_t, s);
      release_geometry(dgeom_t, s);
      if (e3 != cudaSuccess) {  // a launch failure is an error, not a
        cudaFreeAsync(ids, s);  // fallback
        release_geometry(dgeom, s);
        if (dacc_t) cudaFreeAsync(dacc_t, s);
        if (dacc) cudaFreeAsync(dacc, s);
        if (dgmax) cudaFreeAsync(dgmax, s);
        CS_CHECK_CUDA(e3);
      }
      transposed = true;
    } else {
      // could not stage the transposed frame: the direct launch below
      if (acc_t) cudaFreeAsync(acc_t, s);
      if (dgeom_t) release_geometry(dgeom_t, s);
      (void)cudaGetLastError();
      rc = 0;
    }
  }
  if (!transposed && nxm > 0 && rows(0) > 0) {
    k0<<<grid_of(gx, rows(0), nviews(nxm)), ST_THREADS, smem, s>>>(
        vol_in, vol_acc, dgeom, ids, G, step_max, z_lo, z_hi, n_u, n_v,
        band[0][0], band[0][1], out, proj_in, rb, rw, cap, budget, vec_ok,
        lane_stride, prec_mode, prec_fp, edge, lo_scale, tpad, dacc, dscale,
        vpair, nxm);
    CS_COUNT_LAUNCH();
  }
  if (nall > nxm && rows(1) > 0) {
    k1<<<grid_of(gx, rows(1), nviews(nall - nxm)), ST_THREADS, smem, s>>>(
        vol_in, vol_acc, dgeom, ids + nxm, G, step_max, z_lo, z_hi, n_u, n_v,
        band[1][0], band[1][1], out, proj_in, rb, rw, cap, budget, vec_ok,
        lane_stride, prec_mode, prec_fp, edge, lo_scale, tpad, dacc, dscale,
        vpair, nall - nxm);
    CS_COUNT_LAUNCH();
  }
  if (det && dacc_t) {
    const dim3 tg((ny + 31) / 32, (nx + 31) / 32, z_hi - z_lo);
    det_finish_t_kernel<<<tg, dim3(32, 8), 0, s>>>(vol_acc, dacc, dacc_t, nx,
                                                   ny, dscale);
    CS_COUNT_LAUNCH();
    cudaFreeAsync(dacc_t, s);
    cudaFreeAsync(dacc, s);
    cudaFreeAsync(dgmax, s);
  } else if (det) {
    det_finish_kernel<<<num_sms() * 8, 256, 0, s>>>(
        vol_acc, dacc, (size_t)(z_hi - z_lo) * nx * ny, dscale);
    CS_COUNT_LAUNCH();
    cudaFreeAsync(dacc, s);
    cudaFreeAsync(dgmax, s);
  }
  e = cudaGetLastError();
  cudaFreeAsync(ids, s);
  release_geometry(dgeom, s);
  CS_CHECK_CUDA(e);
  (void)staged_smem_cap;
  return CS_OK;
}

template int launch_staged<OP_FWD, 0>(const float*, float*, int, int, int,
                                      int, int, const double*, const double*,
                                      int, int, int, double, float*,
                                      const float*, const float*,
                                      const float*, cudaStream_t);
template int launch_staged<OP_FWD, 1>(const float*, float*, int, int, int,
                                      int, int, const double*, const double*,
                                      int, int, int, double, float*,
                                      const float*, const float*,
                                      const float*, cudaStream_t);
template int launch_staged<OP_FWD, 2>(const float*, float*, int, int, int,
                                      int, int, const double*, const double*,
                                      int, int, int, double, float*,
                                      const float*, const float*,
                                      const float*, cudaStream_t);
template int launch_staged<OP_BWD, 0>(const float*, float*, int, int, int,
                                      int, int, const double*, const double*,
                                      int, int, int, double, float*,
                                      const float*, const float*,
                                      const float*, cudaStream_t);

}  // namespace cs

extern "C" int cs_set_deterministic(int on) {
  cs::g_deterministic = on ? 1 : 0;
  return CS_OK;
}
