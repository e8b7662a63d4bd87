// runtime.cu -- error state, texture cache and geometry upload for the
// conesplit B200 C-ABI.
#include <cstdarg>
#include <map>
#include <mutex>
#include <tuple>

#include "common.cuh"

namespace cs {

static thread_local char g_err[1024] = "";

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
                    LayeredTexture** out) {
  CS_REQUIRE(layers >= 1 && layers <= max_layers(), CS_ERR_ARG,
             "layered texture: %d layers outside [1, %d]", layers,
             max_layers());
  int dev = 0;
  CS_CHECK_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_mu);
  LayeredTexture& t = g_cache[Key{dev, s, (int)role}];
  if (t.array && (t.w != w || t.h != h || t.layers < layers)) {
    // shape change: previous launches on this stream may still read the old
    // array, so drain the stream before releasing it.
    CS_CHECK_CUDA(cudaStreamSynchronize(s));
    cudaDestroySurfaceObject(t.surf);
    cudaDestroyTextureObject(t.tex);
    cudaFreeArray(t.array);
    t = LayeredTexture();
  }
  if (!t.array) {
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

int upload_geometry(const double* geom, int n_a, cudaStream_t s,
                    AngleGeom** d_geom) {
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

}  // namespace cs

extern "C" {

const char* cs_version(void) { return "conesplit-b200 0.1.0 sm_100a"; }

const char* cs_last_error(void) { return cs::g_err; }

int cs_sync(cs_stream_t stream) {
  CS_CHECK_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  return CS_OK;
}

}  // extern "C"
