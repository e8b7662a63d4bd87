// runtime.cu -- error state, texture cache and geometry upload for the
// conesplit B200 C-ABI.
#include <atomic>
#include <cstdarg>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "common.cuh"

namespace cs {

static thread_local char g_err[1024] = "";
std::atomic<long long> g_launches{0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

Grid make_grid(const double grid6[6], int nx, int ny, int nz) {
  Grid G;
  for (int i = 0; i < 3; i++) {
    G.g0[i] = grid6[i];
    G.vox[i] = grid6[3 + i];
  }
  G.n[0] = nx;
  G.n[1] = ny;
  G.n[2] = nz;
  return G;
}

int max_layered_height() {
  static int v = -1;
  if (v < 0) {
    int dev = 0, h = 0, w = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&h, cudaDevAttrMaxTexture2DLayeredHeight,
                               dev) != cudaSuccess)
      h = 16384;
    if (cudaDeviceGetAttribute(&w, cudaDevAttrMaxTexture2DLayeredWidth,
                               dev) != cudaSuccess)
      w = 16384;
    v = h < w ? h : w;
  }
  return v;
}

int max_layers() {
  static int v = -1;
  if (v < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    int dims[2] = {0, 0};
    // cudaDevAttrMaxTexture2DLayeredLayers
    if (cudaDeviceGetAttribute(&dims[0], cudaDevAttrMaxTexture2DLayeredLayers,
                               dev) != cudaSuccess)
      dims[0] = 2048;
    // test knob: a lower limit exercises the layer pieces / sub-slabs
    const char* k = getenv("CS_MAX_LAYERS");
    if (k && atoi(k) > 0 && atoi(k) < dims[0]) dims[0] = atoi(k);
    v = dims[0];
  }
  return v;
}

namespace {
struct Key {
  int device;
  cudaStream_t stream;
  int role;
  bool operator<(const Key& o) const {
    return std::tie(device, stream, role) <
           std::tie(o.device, o.stream, o.role);
  }
};
std::mutex g_mu;
std::map<Key, LayeredTexture> g_cache;

int make_texture(LayeredTexture& t, int w, int h, int layers) {
  cudaChannelFormatDesc fd = cudaCreateChannelDesc<float>();
  cudaExtent ext = make_cudaExtent(w, h, layers);
  CS_CHECK_CUDA(cudaMalloc3DArray(&t.array, &fd, ext,
                                  cudaArrayLayered | cudaArraySurfaceLoadStore));
  cudaResourceDesc rd = {};
  rd.resType = cudaResourceTypeArray;
  rd.res.array.array = t.array;
  cudaTextureDesc td = {};
  td.addressMode[0] = cudaAddressModeBorder;  // zero padding
  td.addressMode[1] = cudaAddressModeBorder;
  td.addressMode[2] = cudaAddressModeBorder;
  td.borderColor[0] = td.borderColor[1] = td.borderColor[2] =
      td.borderColor[3] = 0.f;
  td.filterMode = cudaFilterModePoint;  // weights are computed in software
  td.readMode = cudaReadModeElementType;
  td.normalizedCoords = 0;
  CS_CHECK_CUDA(cudaCreateTextureObject(&t.tex, &rd, &td, nullptr));
  CS_CHECK_CUDA(cudaCreateSurfaceObject(&t.surf, &rd));
  t.w = w;
  t.h = h;
  t.layers = layers;
  return CS_OK;
}
}  // namespace

int acquire_layered(TexRole role, int w, int h, int layers, cudaStream_t s,
                    LayeredTexture** out, bool taller_ok) {
  CS_REQUIRE(layers >= 1 && layers <= max_layers(), CS_ERR_ARG,
             "layered texture: %d layers outside [1, %d]", layers,
             max_layers());
  int dev = 0;
  CS_CHECK_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_mu);
  LayeredTexture& t = g_cache[Key{dev, s, (int)role}];
  if (t.array && (t.w != w || (taller_ok ? t.h < h : t.h != h) ||
                  t.layers < layers)) {
    // shape change: previous launches on this stream may still read the old
    // array, so drain the stream before releasing it.
    CS_CHECK_CUDA(cudaStreamSynchronize(s));
    cudaDestroySurfaceObject(t.surf);
    cudaDestroyTextureObject(t.tex);
    cudaFreeArray(t.array);
    t = LayeredTexture();
  }
  if (!t.array) {
    // test knob: arrays above CS_TEX_MAX_MB fail as out of memory
    static const char* cap_knob = getenv("CS_TEX_MAX_MB");
    if (cap_knob && (double)w * h * layers * sizeof(float) >
                        atof(cap_knob) * 1048576.0) {
      set_error("layered texture %dx%dx%d: out of memory (CS_TEX_MAX_MB)", w,
                h, layers);
      return CS_ERR_CUDA;
    }
    int rc = make_texture(t, w, h, layers);
    if (rc) return rc;
  }
  *out = &t;
  return CS_OK;
}

int load_layered(TexRole role, const float* src, int w, int h, int layers,
                 cudaStream_t s, LayeredTexture** out) {
  int rc = acquire_layered(role, w, h, layers, s, out);
  if (rc) return rc;
  cudaMemcpy3DParms p = {};
  p.srcPtr = make_cudaPitchedPtr((void*)src, (size_t)w * sizeof(float), w, h);
  p.dstArray = (*out)->array;
  p.extent = make_cudaExtent(w, h, layers);
  p.kind = cudaMemcpyDefault;
  CS_CHECK_CUDA(cudaMemcpy3DAsync(&p, s));
  return CS_OK;
}

// Keep memory freed by cudaFreeAsync in the device's default pool instead
// of returning it to the driver at every synchronisation (release threshold
// 0 by default): the per-call geometry tables / reduction partials are then
// sub-allocations, not fresh mappings (ms-scale jitter on small kernels).
void retain_pool() {
  static thread_local int done_dev = -1;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev == done_dev) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done_dev = dev;
}

int upload_geometry(const double* geom, int n_a, cudaStream_t s,
                    AngleGeom** d_geom) {
  retain_pool();
  static_assert(sizeof(AngleGeom) == 12 * sizeof(double), "layout");
  size_t bytes = (size_t)n_a * sizeof(AngleGeom);
  CS_CHECK_CUDA(cudaMallocAsync((void**)d_geom, bytes, s));
  CS_CHECK_CUDA(cudaMemcpyAsync(*d_geom, geom, bytes, cudaMemcpyHostToDevice,
                                s));
  return CS_OK;
}

void release_geometry(AngleGeom* d_geom, cudaStream_t s) {
  if (d_geom) cudaFreeAsync(d_geom, s);
}

bool cull_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* k = getenv("CS_NO_CULL");
    on = (k && k[0] == '1') ? 0 : 1;
  }
  return on == 1;
}

int zero_rows_outside(float* out, int n_a, int n_u, int n_v, int v0, int v1,
                      cudaStream_t s) {
  const size_t row = (size_t)n_u * sizeof(float);
  const size_t pitch = row * n_v;
  if (v1 <= v0) {
    CS_CHECK_CUDA(cudaMemsetAsync(out, 0, pitch * n_a, s));
    return CS_OK;
  }
  if (v0 > 0)
    CS_CHECK_CUDA(cudaMemset2DAsync(out, pitch, 0, row * v0, n_a, s));
  if (v1 < n_v)
    CS_CHECK_CUDA(cudaMemset2DAsync(out + (size_t)v1 * n_u, pitch, 0,
                                    row * (n_v - v1), n_a, s));
  return CS_OK;
}

// Detector-row band of a slab (v-band culling).  A sample
// can put a trilinear tap on a slice of [z_lo, z_hi) only if its z lies in
// (gz0 + (z_lo - 1/2) vz, gz0 + (z_hi + 1/2) vz); every sample lies in the
// grid box.  The rays through that slab box hit the detector inside the
// projective image of its 8 corners (a convex box in front of the source
// maps to the convex hull of its corner images), so rows outside
// [min v - 2, max v + 2] never touch the slab.  Margins: 1.5 voxels in z, 2
// rows on the detector.  Returns the union over the n_a views.
void slab_row_band(const double* geom, int n_a, const Grid& G, int z_lo,
                   int z_hi, int n_v, int* v0, int* v1) {
  *v0 = 0;
  *v1 = n_v;
  if (z_lo <= 0 && z_hi >= G.n[2]) return;
  const double zlo = G.g0[2] + (z_lo - 1.5) * G.vox[2];
  const double zhi = G.g0[2] + (z_hi + 1.5) * G.vox[2];
  const double xlo = G.g0[0] - G.vox[0], xhi = G.g0[0] + (G.n[0] + 1) * G.vox[0];
  const double ylo = G.g0[1] - G.vox[1], yhi = G.g0[1] + (G.n[1] + 1) * G.vox[1];
  double bmin = 1e300, bmax = -1e300;
  for (int a = 0; a < n_a; a++) {
    const double* g = geom + 12 * a;
    const double *S = g, *D = g + 3, *us = g + 6, *vs = g + 9;
    const double nrm[3] = {us[1] * vs[2] - us[2] * vs[1],
                           us[2] * vs[0] - us[0] * vs[2],
                           us[0] * vs[1] - us[1] * vs[0]};
    const double vv = vs[0] * vs[0] + vs[1] * vs[1] + vs[2] * vs[2];
    const double num = nrm[0] * (D[0] - S[0]) + nrm[1] * (D[1] - S[1]) +
                       nrm[2] * (D[2] - S[2]);
    for (int c = 0; c < 8; c++) {
      const double P[3] = {(c & 1) ? xhi : xlo, (c & 2) ? yhi : ylo,
                           (c & 4) ? zhi : zlo};
      const double d[3] = {P[0] - S[0], P[1] - S[1], P[2] - S[2]};
      const double den = nrm[0] * d[0] + nrm[1] * d[1] + nrm[2] * d[2];
      const double t = num / den;
      if (!(den * num > 0.0) || !(t > 0.0)) return;  // corner not in front
      double b = 0.0;
      for (int i = 0; i < 3; i++) b += (S[i] + t * d[i] - D[i]) * vs[i];
      b /= vv;
      bmin = fmin(bmin, b);
      bmax = fmax(bmax, b);
    }
  }
  if (!(bmin <= bmax)) return;
  const double lo = floor(bmin) - 2.0, hi = ceil(bmax) + 3.0;
  *v0 = lo <= 0.0 ? 0 : (lo >= n_v ? n_v : (int)lo);
  *v1 = hi >= n_v ? n_v : (hi <= 0.0 ? 0 : (int)hi);
  if (*v1 < *v0) *v1 = *v0;
}

}  // namespace cs

extern "C" {

const char* cs_version(void) { return "conesplit-b200 0.1.0 sm_100a"; }

const char* cs_last_error(void) { return cs::g_err; }

long long cs_launch_count(void) { return cs::g_launches.load(); }

int cs_sync(cs_stream_t stream) {
  CS_CHECK_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  return CS_OK;
}

int cs_release_cache(void) {
  int dev = 0;
  CS_CHECK_CUDA(cudaGetDevice(&dev));
  // texture reads of queued launches must finish before their arrays go
  CS_CHECK_CUDA(cudaDeviceSynchronize());
  std::lock_guard<std::mutex> lock(cs::g_mu);
  for (auto it = cs::g_cache.begin(); it != cs::g_cache.end();) {
    if (it->first.device != dev) {
      ++it;
      continue;
    }
    cs::LayeredTexture& t = it->second;
    if (t.surf) cudaDestroySurfaceObject(t.surf);
    if (t.tex) cudaDestroyTextureObject(t.tex);
    if (t.array) cudaFreeArray(t.array);
    it = cs::g_cache.erase(it);
  }
  CS_CHECK_CUDA(cudaGetLastError());
  return CS_OK;
}

int cs_peer_enable(int peer_device) {
  int dev = 0, n = 0;
  CS_CHECK_CUDA(cudaGetDevice(&dev));
  CS_CHECK_CUDA(cudaGetDeviceCount(&n));
  CS_REQUIRE(peer_device >= 0 && peer_device < n, CS_ERR_ARG,
             "peer device %d out of range (%d devices)", peer_device, n);
  if (peer_device == dev) return CS_OK;
  int ok = 0;
  CS_CHECK_CUDA(cudaDeviceCanAccessPeer(&ok, dev, peer_device));
  CS_REQUIRE(ok, CS_ERR_UNSUPPORTED, "no P2P path from device %d to %d", dev,
             peer_device);
  const cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return CS_OK;
  }
  CS_CHECK_CUDA(e);
  return CS_OK;
}

}  // extern "C"
