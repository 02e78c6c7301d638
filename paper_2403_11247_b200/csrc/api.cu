// api.cu -- the extern "C" boundary of libcsplat (include/csplat.h): argument
// validation, device check, workspace sizing, error reporting, and the kernel
// launches of the other translation units.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>

#include <nvtx3/nvToolsExt.h>

#include "common.cuh"

namespace {

thread_local char g_err[512] = {0};

void set_err(const char *msg) {
  std::snprintf(g_err, sizeof(g_err), "%s", msg);
}

int cuda_status(cudaError_t e, const char *where) {
  if (e == cudaSuccess) return CSPLAT_OK;
  std::snprintf(g_err, sizeof(g_err), "%s: %s (%s)", where, cudaGetErrorName(e),
                cudaGetErrorString(e));
  return CSPLAT_ERR_CUDA;
}

int check_device() {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_status(e, "cudaGetDevice");
  static thread_local int cached_dev = -1, cached_ok = 0;
  if (cached_dev == dev) return cached_ok ? CSPLAT_OK : CSPLAT_ERR_UNSUPPORTED;
  int major = 0;
  e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  if (e != cudaSuccess) return cuda_status(e, "cudaDeviceGetAttribute");
  cached_dev = dev;
  cached_ok = major == 10;
  if (!cached_ok) {
    set_err("csplat requires a compute capability 10.x (B200, sm_100a) device");
    return CSPLAT_ERR_UNSUPPORTED;
  }
  return CSPLAT_OK;
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int invalid(const char *msg) {
  set_err(msg);
  return CSPLAT_ERR_INVALID_ARG;
}

int check_camera(const csplat_camera *c) {
  if (!c) return invalid("camera is NULL");
  if (c->width <= 0 || c->height <= 0 || c->width > 32767 || c->height > 32767)
    return invalid("camera width/height out of range (1..32767)");
  if (!(c->fx > 0) || !(c->fy > 0)) return invalid("fx, fy must be > 0");
  if (!(c->near_z > 0) || !(c->far_z > c->near_z)) return invalid("need 0 < near < far");
  if (!std::isfinite(c->cx) || !std::isfinite(c->cy)) return invalid("cx, cy must be finite");
  return CSPLAT_OK;
}

int check_gaussians(const csplat_gaussians *g, bool need_rgb = true) {
  if (!g) return invalid("gaussians is NULL");
  if (g->n < 0 || g->n > 0xffffffffLL) return invalid("n out of range");
  if (g->n == 0) return CSPLAT_OK;
  if (!g->mean || !g->opacity || !g->mask || (need_rgb && !g->rgb))
    return invalid("a required Gaussian plane is NULL");
  const void *ps[6] = {g->mean, g->opacity, g->rgb, g->log_scale, g->quat, g->mask};
  for (const void *p : ps)
    if (p && !aligned16(p)) {
      set_err("Gaussian planes must be 16-byte aligned");
      return CSPLAT_ERR_ALIGNMENT;
    }
  return CSPLAT_OK;
}

int check_codebook(const csplat_codebook *cb, bool need_codes) {
  if (!cb) return CSPLAT_OK;
  if (cb->stages < 1 || cb->stages > 16) return invalid("codebook stages must be 1..16");
  if (cb->size < 1 || cb->size > 65536) return invalid("codebook size must be 1..65536");
  if (cb->idx_bytes != 1 && cb->idx_bytes != 2) return invalid("idx_bytes must be 1 or 2");
  if (cb->idx_bytes == 1 && cb->size > 256) return invalid("idx_bytes=1 needs size <= 256");
  if (!cb->scale_idx || !cb->rot_idx) return invalid("codebook index planes are NULL");
  if (need_codes) {
    if (!cb->scale_codes || !cb->rot_codes) return invalid("codebook codes are NULL");
    if (!aligned16(cb->rot_codes)) {
      set_err("rot_codes must be 16-byte aligned");
      return CSPLAT_ERR_ALIGNMENT;
    }
  }
  return CSPLAT_OK;
}

csplat::DecodeArgs decode_args(const csplat_codebook *cb) {
  csplat::DecodeArgs d{};
  d.L = cb->stages;
  d.P = cb->size;
  d.idx_bytes = cb->idx_bytes;
  d.scale_codes = cb->scale_codes;
  d.rot_codes = cb->rot_codes;
  d.scale_idx = cb->scale_idx;
  d.rot_idx = cb->rot_idx;
  d.status = cb->status;
  return d;
}

float mask_tau(float eps) {
  // R12: tau = fl32(ln(eps / (1 - eps))) evaluated in double
  const double e = (double)eps;
  return (float)std::log(e / (1.0 - e));
}

#define RET_IF(x)            \
  do {                       \
    const int _s = (x);      \
    if (_s != CSPLAT_OK) return _s; \
  } while (0)

// NVTX ranges per ABI call (SURVEY §5 tracing): pushed only when the
// environment sets CSPLAT_NVTX=1 (read once), so a normal call pays one
// predictable branch.  nvtx3 is header-only: without a tool attached the push
// and pop are no-ops.
bool nvtx_on() {
  static const bool on = [] {
    const char *e = std::getenv("CSPLAT_NVTX");
    return e && e[0] == '1';
  }();
  return on;
}
struct NvtxRange {
  bool on;
  explicit NvtxRange(const char *name) : on(nvtx_on()) {
    if (on) nvtxRangePushA(name);
  }
  ~NvtxRange() {
    if (on) nvtxRangePop();
  }
};
#define CSPLAT_TRACE NvtxRange _nvtx_range(__func__)

}  // namespace

extern "C" {

int csplat_version(void) { return (2 << 16) | 0; }  // 2.0: tile_range status slot, codebook status

int csplat_release_thread_resources(void) {
  CSPLAT_TRACE;
  csplat::release_thread_fork_resources();
  return CSPLAT_OK;
}

const char *csplat_status_string(int s) {
  switch (s) {
    case CSPLAT_OK: return "ok";
    case CSPLAT_ERR_INVALID_ARG: return "invalid argument";
    case CSPLAT_ERR_ALIGNMENT: return "misaligned buffer";
    case CSPLAT_ERR_CAPACITY: return "pair capacity exceeded";
    case CSPLAT_ERR_WORKSPACE: return "workspace too small";
    case CSPLAT_ERR_CUDA: return "CUDA error";
    case CSPLAT_ERR_UNSUPPORTED: return "unsupported device";
    default: return "unknown status";
  }
}

int csplat_last_error(char *buf, size_t len) {
  CSPLAT_TRACE;
  const int n = (int)std::strlen(g_err);
  if (buf && len) {
    std::strncpy(buf, g_err, len - 1);
    buf[len - 1] = 0;
  }
  return n;
}

size_t csplat_workspace_bytes(int op, int64_t n, int64_t pairs, const csplat_camera *cam) {
  switch (op) {
    case CSPLAT_OP_BIN_TILES: return cam ? csplat::bin_workspace_bytes(n, pairs, *cam) : 0;
    case CSPLAT_OP_RENDER_BWD: return csplat::bwd_workspace_bytes(n);
    case CSPLAT_OP_MASK_PRUNE: return csplat::prune_workspace_bytes(n);
    case CSPLAT_OP_TRACKING_LOSS: return 64;
    case CSPLAT_OP_MASK_LOSS: return 64;
    case CSPLAT_OP_KEYFRAME_OVERLAP: return (size_t)(n > 0 ? n : 1) * 48 + 64;
    case CSPLAT_OP_RVQ_UPDATE:  // n = L * P, pairs = d
      return (size_t)n * (size_t)pairs * 4 + (size_t)n * 4 + 17 * 4 + 256;  // L <= 16
    default: return 0;
  }
}

static int project_impl(const csplat_gaussians *g, const csplat_codebook *cb,
                        const csplat_camera *cam, const csplat_view *view, const float *view_dev,
                        const csplat_params *prm, void *rec, int32_t *count, void *stream) {
  RET_IF(check_gaussians(g));
  RET_IF(check_camera(cam));
  RET_IF(check_codebook(cb, true));
  if ((!view && !view_dev) || !prm) return invalid("view/params NULL");
  if (g->n > 0 && (!rec || !count)) return invalid("rec/count NULL");
  if (!cb && g->n > 0 && (!g->log_scale || !g->quat)) return invalid("log_scale/quat NULL");
  if (!aligned16(rec)) {
    set_err("rec must be 16-byte aligned");
    return CSPLAT_ERR_ALIGNMENT;
  }
  if (!(prm->mask_eps > 0.f) || !(prm->mask_eps < 1.f)) return invalid("mask_eps must be in (0,1)");
  RET_IF(check_device());
  csplat::DecodeArgs d;
  if (cb) d = decode_args(cb);
  return cuda_status(csplat::launch_project(*g, cb ? &d : nullptr, *cam, view ? *view : csplat_view{}, view_dev,
                                            mask_tau(prm->mask_eps), prm->dilation, rec, count,
                                            static_cast<cudaStream_t>(stream)),
                     "csplat_project");
}

int csplat_project(const csplat_gaussians *g, const csplat_codebook *cb, const csplat_camera *cam,
                   const csplat_view *view, const csplat_params *prm, void *rec, int32_t *count,
                   void *stream) {
  CSPLAT_TRACE;
  if (!view) return invalid("view NULL");
  return project_impl(g, cb, cam, view, nullptr, prm, rec, count, stream);
}

int csplat_project_dv(const csplat_gaussians *g, const csplat_codebook *cb,
                      const csplat_camera *cam, const float *view_dev, const csplat_params *prm,
                      void *rec, int32_t *count, void *stream) {
  CSPLAT_TRACE;
  if (!view_dev) return invalid("view_dev NULL");
  return project_impl(g, cb, cam, nullptr, view_dev, prm, rec, count, stream);
}

int csplat_project_views(const csplat_gaussians *g, const csplat_codebook *cb,
                         const csplat_camera *cam, const csplat_view *views, int32_t n_views,
                         const csplat_params *prm, void *rec, int32_t *count, void *stream) {
  CSPLAT_TRACE;
  RET_IF(check_gaussians(g));
  RET_IF(check_camera(cam));
  RET_IF(check_codebook(cb, true));
  if (n_views < 0) return invalid("n_views < 0");
  if ((n_views > 0 && !views) || !prm) return invalid("views/params NULL");
  if (g->n > 0 && n_views > 0 && (!rec || !count)) return invalid("rec/count NULL");
  if (!cb && g->n > 0 && (!g->log_scale || !g->quat)) return invalid("log_scale/quat NULL");
  if (!aligned16(rec)) {
    set_err("rec must be 16-byte aligned");
    return CSPLAT_ERR_ALIGNMENT;
  }
  if (!(prm->mask_eps > 0.f) || !(prm->mask_eps < 1.f)) return invalid("mask_eps must be in (0,1)");
  if (n_views == 0) return CSPLAT_OK;
  RET_IF(check_device());
  csplat::DecodeArgs d;
  if (cb) d = decode_args(cb);
  return cuda_status(csplat::launch_project_views(*g, cb ? &d : nullptr, *cam, views, n_views,
                                                  mask_tau(prm->mask_eps), prm->dilation, rec,
                                                  count, nullptr, 0, 0, nullptr, 0, nullptr,
                                                  nullptr, nullptr, nullptr, 0, 0,
                                                  static_cast<cudaStream_t>(stream)),
                     "csplat_project_views");
}

int csplat_project_bin_views(const csplat_gaussians *g, const csplat_codebook *cb,
                             const csplat_camera *cam, const csplat_view *views, int32_t n_views,
                             const csplat_params *prm, const uint32_t *tile_active,
                             const int32_t *tile_lists, int64_t list_stride, int32_t max_list,
                             void *rec, int32_t *count, int64_t pair_capacity, uint32_t *pair_gid,
                             uint32_t *tile_range, int64_t *n_pairs_dev, void *ws,
                             size_t ws_bytes_per_view, void *stream) {
  CSPLAT_TRACE;
  RET_IF(check_gaussians(g));
  RET_IF(check_camera(cam));
  RET_IF(check_codebook(cb, true));
  if (n_views < 0) return invalid("n_views < 0");
  if ((n_views > 0 && !views) || !prm) return invalid("views/params NULL");
  if (g->n > 0 && n_views > 0 && (!rec || !count)) return invalid("rec/count NULL");
  if (!cb && g->n > 0 && (!g->log_scale || !g->quat)) return invalid("log_scale/quat NULL");
  if (!(prm->mask_eps > 0.f) || !(prm->mask_eps < 1.f)) return invalid("mask_eps must be in (0,1)");
  if (pair_capacity < 0 || pair_capacity > 0xffffffffLL) return invalid("capacity out of range");
  if (g->n > (int64_t)csplat::kPairGidMask + 1) return invalid("n must be < 2^28 for binning");
  if (n_views > 0 && (!tile_range || !n_pairs_dev)) return invalid("tile_range/n_pairs NULL");
  if (pair_capacity > 0 && n_views > 0 && !pair_gid) return invalid("pair_gid NULL");
  if (!aligned16(rec)) {
    set_err("rec must be 16-byte aligned");
    return CSPLAT_ERR_ALIGNMENT;
  }
  const size_t need = csplat::bin_workspace_bytes(g->n, pair_capacity, *cam);
  if (n_views > 0 && (!ws || ws_bytes_per_view < need || (ws_bytes_per_view & 255u) ||
                      (reinterpret_cast<uintptr_t>(ws) & 255u))) {
    set_err("project_bin_views: workspace per view too small, or not a multiple of 256 bytes / "
            "256-byte aligned");
    return CSPLAT_ERR_WORKSPACE;
  }
  if (tile_lists && (!tile_active || max_list < 0))
    return invalid("tile_lists needs tile_active and max_list >= 0");
  if (n_views == 0) return CSPLAT_OK;
  RET_IF(check_device());
  csplat::DecodeArgs d;
  if (cb) d = decode_args(cb);
  const csplat::CamInfo ci = csplat::cam_info(*cam);
  const int64_t words = ((int64_t)ci.tiles_x * ci.tiles_y + 31) / 32;
  return cuda_status(csplat::launch_project_views(*g, cb ? &d : nullptr, *cam, views, n_views,
                                                  mask_tau(prm->mask_eps), prm->dilation, rec,
                                                  count, ws, (int64_t)ws_bytes_per_view,
                                                  pair_capacity, tile_active, words, pair_gid,
                                                  tile_range, n_pairs_dev, tile_lists,
                                                  list_stride, max_list,
                                                  static_cast<cudaStream_t>(stream)),
                     "csplat_project_bin_views");
}

int csplat_chain_views(const csplat_gaussians *g, const csplat_codebook *cb,
                       const csplat_camera *cam, const csplat_view *views, int32_t n_views,
                       const csplat_params *prm, const void *rec, void *ws, uint32_t flags,
                       const csplat_grads *out, void *stream) {
  CSPLAT_TRACE;
  RET_IF(check_gaussians(g));
  RET_IF(check_camera(cam));
  RET_IF(check_codebook(cb, true));
  if (n_views < 0) return invalid("n_views < 0");
  if ((n_views > 0 && !views) || !prm || !out) return invalid("views/params/out NULL");
  if (flags & CSPLAT_POSE_ONLY) return invalid("chain_views: POSE_ONLY is not supported");
  if (g->n > 0 && n_views > 0 && (!rec || !ws)) return invalid("rec/ws NULL");
  if (!cb && g->n > 0 && (!g->log_scale || !g->quat)) return invalid("log_scale/quat NULL");
  if (!aligned16(rec) || (reinterpret_cast<uintptr_t>(ws) & 255u)) {
    set_err("rec must be 16-byte aligned, ws 256-byte aligned");
    return CSPLAT_ERR_ALIGNMENT;
  }
  RET_IF(check_device());
  csplat::DecodeArgs d;
  if (cb) d = decode_args(cb);
  return cuda_status(csplat::launch_chain_views(*g, cb ? &d : nullptr, *cam, views, n_views, *prm,
                                                rec, ws, flags, *out,
                                                static_cast<cudaStream_t>(stream)),
                     "csplat_chain_views");
}

static int project_bin_impl(const csplat_gaussians *g, const csplat_codebook *cb,
                            const csplat_camera *cam, const csplat_view *view,
                            const float *view_dev, const csplat_params *prm, void *rec,
                            int32_t *count, const uint32_t *tile_active, int64_t pair_capacity,
                            uint32_t *pair_gid, uint32_t *tile_range,
                            int64_t *n_pairs_dev, uint32_t flags, void *ws, size_t ws_bytes,
                            void *stream) {
  RET_IF(check_gaussians(g));
  RET_IF(check_camera(cam));
  RET_IF(check_codebook(cb, true));
  if ((!view && !view_dev) || !prm) return invalid("view/params NULL");
  if (g->n > 0 && (!rec || !count)) return invalid("rec/count NULL");
  if (!cb && g->n > 0 && (!g->log_scale || !g->quat)) return invalid("log_scale/quat NULL");
  if (!(prm->mask_eps > 0.f) || !(prm->mask_eps < 1.f)) return invalid("mask_eps must be in (0,1)");
  if (pair_capacity < 0 || pair_capacity > 0xffffffffLL) return invalid("capacity out of range");
  if (g->n > (int64_t)csplat::kPairGidMask + 1) return invalid("n must be < 2^28 for binning");
  if (!tile_range || !n_pairs_dev) return invalid("tile_range/n_pairs NULL");
  if (pair_capacity > 0 && !pair_gid) return invalid("pair_gid NULL");
  if (!aligned16(rec)) {
    set_err("rec must be 16-byte aligned");
    return CSPLAT_ERR_ALIGNMENT;
  }
  const size_t need = csplat::bin_workspace_bytes(g->n, pair_capacity, *cam);
  if (!ws || ws_bytes < need) {
    set_err("project_bin workspace too small");
    return CSPLAT_ERR_WORKSPACE;
  }
  RET_IF(check_device());
  csplat::DecodeArgs d;
  if (cb) d = decode_args(cb);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  RET_IF(cuda_status(csplat::launch_project_bin(*g, cb ? &d : nullptr, *cam,
                                                view ? *view : csplat_view{}, view_dev,
                                                mask_tau(prm->mask_eps), prm->dilation, rec, count,
                                                pair_capacity, tile_active, pair_gid,
                                                tile_range, n_pairs_dev, ws, s),
                     "csplat_project_bin"));
  if (flags & CSPLAT_SYNC) {
    int64_t total = 0;
    RET_IF(cuda_status(cudaMemcpyAsync(&total, n_pairs_dev, sizeof(total), cudaMemcpyDeviceToHost, s),
                       "csplat_project_bin readback"));
    RET_IF(cuda_status(cudaStreamSynchronize(s), "csplat_project_bin sync"));
    if (total > pair_capacity) {
      std::snprintf(g_err, sizeof(g_err), "%lld pairs exceed capacity %lld", (long long)total,
                    (long long)pair_capacity);
      return CSPLAT_ERR_CAPACITY;
    }
  }
  return CSPLAT_OK;
}

int csplat_project_bin(const csplat_gaussians *g, const csplat_codebook *cb,
                       const csplat_camera *cam, const csplat_view *view,
                       const csplat_params *prm, void *rec, int32_t *count,
                       const uint32_t *tile_active, int64_t pair_capacity, uint32_t *pair_gid, uint32_t *tile_range, int64_t *n_pairs_dev,
                       uint32_t flags, void *ws, size_t ws_bytes, void *stream) {
  CSPLAT_TRACE;
  if (!view) return invalid("view NULL");
  return project_bin_impl(g, cb, cam, view, nullptr, prm, rec, count, tile_active, pair_capacity,
                          pair_gid, tile_range, n_pairs_dev, flags, ws, ws_bytes, stream);
}

int csplat_project_bin_dv(const csplat_gaussians *g, const csplat_codebook *cb,
                          const csplat_camera *cam, const float *view_dev,
                          const csplat_params *prm, void *rec, int32_t *count,
                          const uint32_t *tile_active, int64_t pair_capacity, uint32_t *pair_gid, uint32_t *tile_range, int64_t *n_pairs_dev,
                          uint32_t flags, void *ws, size_t ws_bytes, void *stream) {
  CSPLAT_TRACE;
  if (!view_dev) return invalid("view_dev NULL");
  return project_bin_impl(g, cb, cam, nullptr, view_dev, prm, rec, count, tile_active,
                          pair_capacity, pair_gid, tile_range, n_pairs_dev, flags, ws,
                          ws_bytes, stream);
}

static int project_bin_render_impl(const csplat_gaussians *g, const csplat_codebook *cb,
                                   const csplat_camera *cam, const csplat_view *view,
                                   const float *view_dev, const csplat_params *prm, void *rec,
                                   int32_t *count, int64_t pair_capacity, uint32_t *pair_gid, uint32_t *tile_range, int64_t *n_pairs_dev,
                                   void *ws, size_t ws_bytes, float *color, float *depth,
                                   float *silhouette, float *t_final, int32_t *n_contrib,
                                   void *stream) {
  RET_IF(check_gaussians(g));
  RET_IF(check_camera(cam));
  RET_IF(check_codebook(cb, true));
  if ((!view && !view_dev) || !prm) return invalid("view/params NULL");
  if (g->n > 0 && (!rec || !count)) return invalid("rec/count NULL");
  if (!cb && g->n > 0 && (!g->log_scale || !g->quat)) return invalid("log_scale/quat NULL");
  if (!(prm->mask_eps > 0.f) || !(prm->mask_eps < 1.f)) return invalid("mask_eps must be in (0,1)");
  if (pair_capacity < 0 || pair_capacity > 0xffffffffLL) return invalid("capacity out of range");
  if (g->n > (int64_t)csplat::kPairGidMask + 1) return invalid("n must be < 2^28 for binning");
  if (!tile_range || !n_pairs_dev) return invalid("tile_range/n_pairs NULL");
  if (pair_capacity > 0 && !pair_gid) return invalid("pair_gid NULL");
  if (!color || !depth || !silhouette || !t_final || !n_contrib)
    return invalid("project_bin_render: image NULL");
  if (!aligned16(rec)) {
    set_err("rec must be 16-byte aligned");
    return CSPLAT_ERR_ALIGNMENT;
  }
  const size_t need = csplat::bin_workspace_bytes(g->n, pair_capacity, *cam);
  if (!ws || ws_bytes < need) {
    set_err("project_bin_render workspace too small");
    return CSPLAT_ERR_WORKSPACE;
  }
  RET_IF(check_device());
  csplat::DecodeArgs d;
  if (cb) d = decode_args(cb);
  return cuda_status(csplat::launch_project_bin_render(
                         *g, cb ? &d : nullptr, *cam, view ? *view : csplat_view{}, view_dev,
                         mask_tau(prm->mask_eps), prm->dilation, *prm, rec, count, pair_capacity,
                         pair_gid, tile_range, n_pairs_dev, ws, color, depth,
                         silhouette, t_final, n_contrib, static_cast<cudaStream_t>(stream)),
                     "csplat_project_bin_render");
}

int csplat_project_bin_render(const csplat_gaussians *g, const csplat_codebook *cb,
                              const csplat_camera *cam, const csplat_view *view,
                              const csplat_params *prm, void *rec, int32_t *count,
                              int64_t pair_capacity, uint32_t *pair_gid,
                              uint32_t *tile_range, int64_t *n_pairs_dev, void *ws,
                              size_t ws_bytes, float *color, float *depth, float *silhouette,
                              float *t_final, int32_t *n_contrib, void *stream) {
  CSPLAT_TRACE;
  if (!view) return invalid("view NULL");
  return project_bin_render_impl(g, cb, cam, view, nullptr, prm, rec, count, pair_capacity,
                                 pair_gid, tile_range, n_pairs_dev, ws, ws_bytes, color,
                                 depth, silhouette, t_final, n_contrib, stream);
}

int csplat_project_bin_render_dv(const csplat_gaussians *g, const csplat_codebook *cb,
                                 const csplat_camera *cam, const float *view_dev,
                                 const csplat_params *prm, void *rec, int32_t *count,
                                 int64_t pair_capacity, uint32_t *pair_gid,
                                 uint32_t *tile_range, int64_t *n_pairs_dev, void *ws,
                                 size_t ws_bytes, float *color, float *depth, float *silhouette,
                                 float *t_final, int32_t *n_contrib, void *stream) {
  CSPLAT_TRACE;
  if (!view_dev) return invalid("view_dev NULL");
  return project_bin_render_impl(g, cb, cam, nullptr, view_dev, prm, rec, count, pair_capacity,
                                 pair_gid, tile_range, n_pairs_dev, ws, ws_bytes, color,
                                 depth, silhouette, t_final, n_contrib, stream);
}

static int render_step_impl(const csplat_gaussians *g, const csplat_codebook *cb,
                            const csplat_camera *cam, const csplat_view *view,
                            const float *view_dev, const csplat_params *prm, void *rec,
                            int32_t *count, int64_t pair_capacity, uint32_t *pair_gid, uint32_t *tile_range, int64_t *n_pairs_dev,
                            void *ws_bin, size_t ws_bin_bytes, float *color, float *depth,
                            float *silhouette, float *t_final, int32_t *n_contrib,
                            const float *d_color, const float *d_depth,
                            const float *d_silhouette, const csplat::TrackingLoss *loss,
                            uint32_t flags, const csplat_grads *out, void *ws_bwd,
                            size_t ws_bwd_bytes, void *stream) {
  RET_IF(check_gaussians(g));
  RET_IF(check_camera(cam));
  RET_IF(check_codebook(cb, true));
  if ((!view && !view_dev) || !prm || !out) return invalid("view/params/grads NULL");
  if (g->n > 0 && (!rec || !count)) return invalid("rec/count NULL");
  if (!cb && g->n > 0 && (!g->log_scale || !g->quat)) return invalid("log_scale/quat NULL");
  if (!(prm->mask_eps > 0.f) || !(prm->mask_eps < 1.f)) return invalid("mask_eps must be in (0,1)");
  if (pair_capacity < 0 || pair_capacity > 0xffffffffLL) return invalid("capacity out of range");
  if (g->n > (int64_t)csplat::kPairGidMask + 1) return invalid("n must be < 2^28 for binning");
  if (!tile_range || !n_pairs_dev) return invalid("tile_range/n_pairs NULL");
  if (pair_capacity > 0 && !pair_gid) return invalid("pair_gid NULL");
  if (!color || !depth || !silhouette || !t_final || !n_contrib)
    return invalid("render_step: image NULL");
  if (!loss && (!d_color || !d_depth || !d_silhouette)) return invalid("render_step: upstream NULL");
  if (!loss && (flags & CSPLAT_POSE_ONLY)) return invalid("render_step: CSPLAT_POSE_ONLY not supported");
  if (!aligned16(rec)) {
    set_err("rec must be 16-byte aligned");
    return CSPLAT_ERR_ALIGNMENT;
  }
  if (!ws_bin || ws_bin_bytes < csplat::bin_workspace_bytes(g->n, pair_capacity, *cam)) {
    set_err("render_step binning workspace too small");
    return CSPLAT_ERR_WORKSPACE;
  }
  if (!ws_bwd || ws_bwd_bytes < csplat::bwd_workspace_bytes(g->n) || !aligned16(ws_bwd)) {
    set_err("render_step backward workspace too small or misaligned");
    return CSPLAT_ERR_WORKSPACE;
  }
  RET_IF(check_device());
  csplat::DecodeArgs d;
  if (cb) d = decode_args(cb);
  const csplat::StepBwd b{d_color, d_depth, d_silhouette, flags, *out, ws_bwd, loss};
  return cuda_status(csplat::launch_render_step(*g, cb ? &d : nullptr, *cam,
                                                view ? *view : csplat_view{}, view_dev,
                                                mask_tau(prm->mask_eps), prm->dilation, *prm, rec,
                                                count, pair_capacity, pair_gid,
                                                tile_range, n_pairs_dev, ws_bin, color, depth,
                                                silhouette, t_final, n_contrib, &b,
                                                static_cast<cudaStream_t>(stream)),
                     "csplat_render_step");
}

int csplat_render_step(const csplat_gaussians *g, const csplat_codebook *cb,
                       const csplat_camera *cam, const csplat_view *view,
                       const csplat_params *prm, void *rec, int32_t *count,
                       int64_t pair_capacity, uint32_t *pair_gid,
                       uint32_t *tile_range, int64_t *n_pairs_dev, void *ws_bin,
                       size_t ws_bin_bytes, float *color, float *depth, float *silhouette,
                       float *t_final, int32_t *n_contrib, const float *d_color,
                       const float *d_depth, const float *d_silhouette, uint32_t flags,
                       const csplat_grads *out, void *ws_bwd, size_t ws_bwd_bytes,
                       void *stream) {
  CSPLAT_TRACE;
  if (!view) return invalid("view NULL");
  return render_step_impl(g, cb, cam, view, nullptr, prm, rec, count, pair_capacity, pair_gid,
                          tile_range, n_pairs_dev, ws_bin, ws_bin_bytes, color, depth,
                          silhouette, t_final, n_contrib, d_color, d_depth, d_silhouette, nullptr,
                          flags, out, ws_bwd, ws_bwd_bytes, stream);
}

int csplat_tracking_step(const csplat_gaussians *g, const csplat_codebook *cb,
                         const csplat_camera *cam, const csplat_view *view,
                         const float *view_dev, const csplat_params *prm, void *rec,
                         int32_t *count, int64_t pair_capacity, uint32_t *pair_gid, uint32_t *tile_range, int64_t *n_pairs_dev,
                         void *ws_bin, size_t ws_bin_bytes, float *color, float *depth,
                         float *silhouette, float *t_final, int32_t *n_contrib,
                         const float *obs_color, const float *obs_depth,
                         const uint64_t *n_valid_dev, float lambda_depth, float sil_gate,
                         uint32_t flags, const csplat_grads *out, float *loss3_dev,
                         void *ws_bwd, size_t ws_bwd_bytes, void *stream) {
  CSPLAT_TRACE;
  if ((view == nullptr) == (view_dev == nullptr)) return invalid("give exactly one of view / view_dev");
  if (!obs_color || !obs_depth || !n_valid_dev || !loss3_dev)
    return invalid("tracking_step: NULL observation argument");
  if (!std::isfinite(lambda_depth) || !std::isfinite(sil_gate))
    return invalid("lambda_depth / sil_gate must be finite");
  const csplat::TrackingLoss tl{color, depth, silhouette, obs_color, obs_depth,
                                reinterpret_cast<const unsigned long long *>(n_valid_dev),
                                lambda_depth, sil_gate, loss3_dev};
  return render_step_impl(g, cb, cam, view, view_dev, prm, rec, count, pair_capacity, pair_gid,
                          tile_range, n_pairs_dev, ws_bin, ws_bin_bytes, color, depth,
                          silhouette, t_final, n_contrib, nullptr, nullptr, nullptr, &tl, flags,
                          out, ws_bwd, ws_bwd_bytes, stream);
}

int csplat_bin_tiles_active(const void *rec, const int32_t *count, int64_t n,
                            const csplat_camera *cam, const uint32_t *tile_active,
                            int64_t pair_capacity, uint32_t *pair_gid,
                     uint32_t *tile_range, int64_t *n_pairs_dev, uint32_t flags, void *ws,
                     size_t ws_bytes, void *stream) {
  CSPLAT_TRACE;
  RET_IF(check_camera(cam));
  if (n < 0 || n > (int64_t)csplat::kPairGidMask + 1 || pair_capacity < 0 ||
      pair_capacity > 0xffffffffLL)
    return invalid("n (< 2^28 for binning) / capacity out of range");
  if (!tile_range || !n_pairs_dev) return invalid("tile_range/n_pairs NULL");
  if (n > 0 && (!rec || !count)) return invalid("rec/count NULL");
  if (pair_capacity > 0 && !pair_gid) return invalid("pair_gid NULL");
  if (!aligned16(rec)) {
    set_err("rec must be 16-byte aligned");
    return CSPLAT_ERR_ALIGNMENT;
  }
  const size_t need = csplat::bin_workspace_bytes(n, pair_capacity, *cam);
  if (!ws || ws_bytes < need) {
    set_err("bin_tiles workspace too small");
    return CSPLAT_ERR_WORKSPACE;
  }
  RET_IF(check_device());
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  RET_IF(cuda_status(csplat::launch_bin(rec, count, n, *cam, pair_capacity, tile_active, pair_gid,
                                        tile_range, n_pairs_dev, ws, s),
                     "csplat_bin_tiles"));
  if (flags & CSPLAT_SYNC) {
    int64_t total = 0;
    RET_IF(cuda_status(cudaMemcpyAsync(&total, n_pairs_dev, sizeof(total), cudaMemcpyDeviceToHost, s),
                       "csplat_bin_tiles readback"));
    RET_IF(cuda_status(cudaStreamSynchronize(s), "csplat_bin_tiles sync"));
    if (total > pair_capacity) {
      std::snprintf(g_err, sizeof(g_err), "%lld pairs exceed capacity %lld", (long long)total,
                    (long long)pair_capacity);
      return CSPLAT_ERR_CAPACITY;
    }
  }
  return CSPLAT_OK;
}

int csplat_bin_tiles(const void *rec, const int32_t *count, int64_t n, const csplat_camera *cam,
                     int64_t pair_capacity, uint32_t *pair_gid,
                     uint32_t *tile_range, int64_t *n_pairs_dev, uint32_t flags, void *ws,
                     size_t ws_bytes, void *stream) {
  CSPLAT_TRACE;
  return csplat_bin_tiles_active(rec, count, n, cam, nullptr, pair_capacity, pair_gid,
                                 tile_range, n_pairs_dev, flags, ws, ws_bytes, stream);
}

int csplat_ba_patches(const float *obs_depth, const csplat_camera *cam, const int32_t *patches,
                      int64_t n_patches, uint32_t *tile_active, uint64_t *n_valid_dev,
                      void *stream) {
  CSPLAT_TRACE;
  RET_IF(check_camera(cam));
  if (n_patches < 0) return invalid("n_patches < 0");
  if (!tile_active || !n_valid_dev || (n_patches > 0 && (!obs_depth || !patches)))
    return invalid("ba_patches: NULL argument");
  RET_IF(check_device());
  return cuda_status(csplat::launch_ba_patches(obs_depth, *cam, patches, n_patches, tile_active,
                                               reinterpret_cast<unsigned long long *>(n_valid_dev),
                                               static_cast<cudaStream_t>(stream)),
                     "csplat_ba_patches");
}

int csplat_ba_patch_loss(const float *color, const float *depth, const float *obs_color,
                         const float *obs_depth, const csplat_camera *cam, const int32_t *patches,
                         int64_t n_patches, int64_t n_rays, const uint64_t *n_valid_dev,
                         float lambda_depth, float lambda_ssim, float *d_color, float *d_depth,
                         float *d_silhouette, float *loss3_dev, void *stream) {
  CSPLAT_TRACE;
  RET_IF(check_camera(cam));
  if (n_patches < 0 || (n_patches > 0 && n_rays <= 0))
    return invalid("need n_patches >= 0 and n_rays > 0");
  if (!d_color || !d_depth || !d_silhouette)
    return invalid("ba_patch_loss: NULL gradient output");
  if (n_patches > 0 && (!color || !depth || !obs_color || !obs_depth || !patches ||
                        !n_valid_dev || !loss3_dev))
    return invalid("ba_patch_loss: NULL argument");
  if (!std::isfinite(lambda_depth) || !std::isfinite(lambda_ssim))
    return invalid("lambda_depth / lambda_ssim must be finite");
  RET_IF(check_device());
  return cuda_status(
      csplat::launch_ba_loss(color, depth, obs_color, obs_depth, *cam, patches, n_patches,
                             n_rays, reinterpret_cast<const unsigned long long *>(n_valid_dev),
                             lambda_depth, lambda_ssim, d_color, d_depth, d_silhouette, loss3_dev,
                             static_cast<cudaStream_t>(stream)),
      "csplat_ba_patch_loss");
}

int csplat_render_fwd_list(const void *rec, const uint32_t *pair_gid, const uint32_t *tile_range,
                           const int32_t *tile_list, int32_t max_tiles, const csplat_camera *cam,
                           const csplat_params *prm, float *color, float *depth, float *silhouette,
                           float *t_final, int32_t *n_contrib, void *stream) {
  CSPLAT_TRACE;
  RET_IF(check_camera(cam));
  if (!prm || !tile_range || !tile_list || !color || !depth || !silhouette || !t_final ||
      !n_contrib || max_tiles < 0)
    return invalid("render_fwd_list: NULL argument / max_tiles < 0");
  if (!aligned16(rec)) {
    set_err("rec must be 16-byte aligned");
    return CSPLAT_ERR_ALIGNMENT;
  }
  RET_IF(check_device());
  return cuda_status(csplat::launch_render_fwd(rec, pair_gid, tile_range, *cam, *prm, color, depth,
                                               silhouette, t_final, n_contrib,
                                               static_cast<cudaStream_t>(stream), 0, max_tiles,
                                               tile_list),
                     "csplat_render_fwd_list");
}

int csplat_render_fwd(const void *rec, const uint32_t *pair_gid, const uint32_t *tile_range,
                      const csplat_camera *cam, const csplat_params *prm, float *color,
                      float *depth, float *silhouette, float *t_final, int32_t *n_contrib,
                      void *stream) {
  CSPLAT_TRACE;
  RET_IF(check_camera(cam));
  if (!prm || !tile_range || !color || !depth || !silhouette || !t_final || !n_contrib)
    return invalid("render_fwd: NULL argument");
  if (!aligned16(rec)) {
    set_err("rec must be 16-byte aligned");
    return CSPLAT_ERR_ALIGNMENT;
  }
  RET_IF(check_device());
  return cuda_status(csplat::launch_render_fwd(rec, pair_gid, tile_range, *cam, *prm, color, depth,
                                               silhouette, t_final, n_contrib,
                                               static_cast<cudaStream_t>(stream)),
                     "csplat_render_fwd");
}

static int render_bwd_impl(const csplat_gaussians *g, const csplat_codebook *cb,
                      const csplat_camera *cam, const csplat_view *view, const float *view_dev,
                      const csplat_params *prm,
                      const void *rec, const uint32_t *pair_gid, const uint32_t *tile_range,
                      const float *t_final, const int32_t *n_contrib, const float *d_color,
                      const float *d_depth, const float *d_silhouette, uint32_t flags,
                      const csplat_grads *out, void *ws, size_t ws_bytes, void *stream,
                      const csplat::TrackingLoss *loss = nullptr, const int32_t *list = nullptr,
                      int max_tiles = 0) {
  RET_IF(check_gaussians(g, false));
  RET_IF(check_camera(cam));
  RET_IF(check_codebook(cb, true));
  if ((!view && !view_dev) || !prm || !out || !tile_range || !t_final || !n_contrib ||
      (!loss && (!d_color || !d_depth || !d_silhouette)))
    return invalid("render_bwd: NULL argument");
  if (g->n > 0 && !rec) return invalid("rec NULL");
  if (!cb && g->n > 0 && (!g->log_scale || !g->quat)) return invalid("log_scale/quat NULL");
  if (!aligned16(rec)) {
    set_err("rec must be 16-byte aligned");
    return CSPLAT_ERR_ALIGNMENT;
  }
  if (!ws || ws_bytes < csplat::bwd_workspace_bytes(g->n) || !aligned16(ws)) {
    set_err("render_bwd workspace too small or misaligned");
    return CSPLAT_ERR_WORKSPACE;
  }
  RET_IF(check_device());
  csplat::DecodeArgs d;
  if (cb) d = decode_args(cb);
  return cuda_status(csplat::launch_render_bwd(*g, cb ? &d : nullptr, *cam,
                                               view ? *view : csplat_view{}, view_dev, loss,
                                               *prm, rec,
                                               pair_gid, tile_range, t_final, n_contrib, d_color,
                                               d_depth, d_silhouette, flags, *out, ws,
                                               static_cast<cudaStream_t>(stream), list, max_tiles),
                     "csplat_render_bwd");
}

int csplat_render_bwd_list(const csplat_gaussians *g, const csplat_codebook *cb,
                           const csplat_camera *cam, const csplat_view *view,
                           const csplat_params *prm, const void *rec, const uint32_t *pair_gid,
                           const uint32_t *tile_range, const int32_t *tile_list,
                           int32_t max_tiles, const float *t_final, const int32_t *n_contrib,
                           const float *d_color, const float *d_depth, const float *d_silhouette,
                           uint32_t flags, const csplat_grads *out, void *ws, size_t ws_bytes,
                           void *stream) {
  CSPLAT_TRACE;
  if (!view) return invalid("view NULL");
  if (!tile_list || max_tiles < 0) return invalid("tile_list NULL / max_tiles < 0");
  return render_bwd_impl(g, cb, cam, view, nullptr, prm, rec, pair_gid, tile_range, t_final,
                         n_contrib, d_color, d_depth, d_silhouette, flags, out, ws, ws_bytes,
                         stream, nullptr, tile_list, max_tiles);
}

int csplat_render_bwd(const csplat_gaussians *g, const csplat_codebook *cb,
                      const csplat_camera *cam, const csplat_view *view, const csplat_params *prm,
                      const void *rec, const uint32_t *pair_gid, const uint32_t *tile_range,
                      const float *t_final, const int32_t *n_contrib, const float *d_color,
                      const float *d_depth, const float *d_silhouette, uint32_t flags,
                      const csplat_grads *out, void *ws, size_t ws_bytes, void *stream) {
  CSPLAT_TRACE;
  if (!view) return invalid("view NULL");
  return render_bwd_impl(g, cb, cam, view, nullptr, prm, rec, pair_gid, tile_range, t_final,
                         n_contrib, d_color, d_depth, d_silhouette, flags, out, ws, ws_bytes,
                         stream);
}

int csplat_render_bwd_dv(const csplat_gaussians *g, const csplat_codebook *cb,
                         const csplat_camera *cam, const float *view_dev,
                         const csplat_params *prm, const void *rec, const uint32_t *pair_gid,
                         const uint32_t *tile_range, const float *t_final,
                         const int32_t *n_contrib, const float *d_color, const float *d_depth,
                         const float *d_silhouette, uint32_t flags, const csplat_grads *out,
                         void *ws, size_t ws_bytes, void *stream) {
  CSPLAT_TRACE;
  if (!view_dev) return invalid("view_dev NULL");
  return render_bwd_impl(g, cb, cam, nullptr, view_dev, prm, rec, pair_gid, tile_range, t_final,
                         n_contrib, d_color, d_depth, d_silhouette, flags, out, ws, ws_bytes,
                         stream);
}

int csplat_count_valid_depth(const float *obs_depth, int32_t width, int32_t height,
                             uint64_t *n_valid_dev, void *stream) {
  CSPLAT_TRACE;
  if (width <= 0 || height <= 0) return invalid("width/height must be > 0");
  if (!obs_depth || !n_valid_dev) return invalid("count_valid_depth: NULL argument");
  RET_IF(check_device());
  return cuda_status(csplat::launch_count_valid(obs_depth, (int64_t)width * height,
                                                reinterpret_cast<unsigned long long *>(n_valid_dev),
                                                static_cast<cudaStream_t>(stream)),
                     "csplat_count_valid_depth");
}

int csplat_tracking_bwd(const csplat_gaussians *g, const csplat_codebook *cb,
                        const csplat_camera *cam, const csplat_view *view, const float *view_dev,
                        const csplat_params *prm, const void *rec, const uint32_t *pair_gid,
                        const uint32_t *tile_range, const float *t_final,
                        const int32_t *n_contrib, const float *color, const float *depth,
                        const float *silhouette, const float *obs_color, const float *obs_depth,
                        const uint64_t *n_valid_dev, float lambda_depth, float sil_gate,
                        uint32_t flags, const csplat_grads *out, float *loss3_dev, void *ws,
                        size_t ws_bytes, void *stream) {
  CSPLAT_TRACE;
  if ((view == nullptr) == (view_dev == nullptr)) return invalid("give exactly one of view / view_dev");
  if (!color || !depth || !silhouette || !obs_color || !obs_depth || !n_valid_dev)
    return invalid("tracking_bwd: NULL image argument");
  if (!std::isfinite(lambda_depth) || !std::isfinite(sil_gate))
    return invalid("lambda_depth / sil_gate must be finite");
  csplat::TrackingLoss tl{color, depth, silhouette, obs_color, obs_depth,
                          reinterpret_cast<const unsigned long long *>(n_valid_dev), lambda_depth,
                          sil_gate, loss3_dev};
  return render_bwd_impl(g, cb, cam, view, view_dev, prm, rec, pair_gid, tile_range, t_final,
                         n_contrib, nullptr, nullptr, nullptr, flags, out, ws, ws_bytes, stream,
                         &tl);
}

int csplat_pose_step(float *view_dev, const float *pose_grad_dev, float lr_rot, float lr_trans,
                     void *stream) {
  CSPLAT_TRACE;
  if (!view_dev || !pose_grad_dev) return invalid("pose_step: NULL argument");
  if (!std::isfinite(lr_rot) || !std::isfinite(lr_trans)) return invalid("lr must be finite");
  RET_IF(check_device());
  return cuda_status(csplat::launch_pose_step(view_dev, pose_grad_dev, lr_rot, lr_trans,
                                              static_cast<cudaStream_t>(stream)),
                     "csplat_pose_step");
}

int csplat_tracking_loss(const float *color, const float *depth, const float *silhouette,
                         const float *obs_color, const float *obs_depth, int32_t width,
                         int32_t height, float lambda_depth, float sil_gate, float *d_color,
                         float *d_depth, float *d_silhouette, float *loss3_dev, void *ws,
                         size_t ws_bytes, void *stream) {
  CSPLAT_TRACE;
  if (width <= 0 || height <= 0) return invalid("width/height must be > 0");
  if (!color || !depth || !silhouette || !obs_color || !obs_depth || !d_color || !d_depth ||
      !d_silhouette)
    return invalid("tracking_loss: NULL argument");
  if (!std::isfinite(lambda_depth) || !std::isfinite(sil_gate))
    return invalid("lambda_depth / sil_gate must be finite");
  if (!ws || ws_bytes < 64) {
    set_err("tracking_loss workspace too small");
    return CSPLAT_ERR_WORKSPACE;
  }
  RET_IF(check_device());
  return cuda_status(csplat::launch_tracking_loss(color, depth, silhouette, obs_color, obs_depth,
                                                  width, height, lambda_depth, sil_gate, d_color,
                                                  d_depth, d_silhouette, loss3_dev, ws,
                                                  static_cast<cudaStream_t>(stream)),
                     "csplat_tracking_loss");
}

int csplat_mask_loss(const csplat_gaussians *g, const int32_t *count, float lambda,
                     float *d_mask, float *loss_dev, void *ws, size_t ws_bytes, void *stream) {
  CSPLAT_TRACE;
  if (!g || g->n < 0) return invalid("gaussians NULL / n < 0");
  if (g->n > 0 && (!g->mask || !count || !d_mask)) return invalid("mask_loss: NULL argument");
  if (!std::isfinite(lambda)) return invalid("lambda must be finite");
  if (!ws || ws_bytes < 64) {
    set_err("mask_loss workspace too small");
    return CSPLAT_ERR_WORKSPACE;
  }
  RET_IF(check_device());
  return cuda_status(csplat::launch_mask_loss(g->n, g->n_dev, g->mask, count, lambda, d_mask,
                                              loss_dev, ws, static_cast<cudaStream_t>(stream)),
                     "csplat_mask_loss");
}

int csplat_keyframe_overlap(const float *depth, const csplat_camera *cam, const csplat_view *cur,
                            const csplat_view *views, int32_t K, int64_t *counts_dev, void *ws,
                            size_t ws_bytes, void *stream) {
  CSPLAT_TRACE;
  RET_IF(check_camera(cam));
  if (K < 0 || K > 256) return invalid("K must be 0..256");
  if (!depth || !cur || (K > 0 && (!views || !counts_dev))) return invalid("overlap: NULL argument");
  if (!ws || ws_bytes < (size_t)(K > 0 ? K : 1) * 48 + 64) {
    set_err("keyframe_overlap workspace too small");
    return CSPLAT_ERR_WORKSPACE;
  }
  if (K == 0) return CSPLAT_OK;
  RET_IF(check_device());
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  float *vd = static_cast<float *>(ws);
  RET_IF(cuda_status(cudaMemcpyAsync(vd, views, (size_t)K * 48, cudaMemcpyHostToDevice, s),
                     "keyframe_overlap views upload"));
  return cuda_status(csplat::launch_overlap(depth, *cam, *cur, vd, K,
                                            reinterpret_cast<unsigned long long *>(counts_dev), s),
                     "csplat_keyframe_overlap");
}

int csplat_rvq_update(const float *x, int64_t n, const int64_t *n_dev, int32_t d,
                      const float *codes, int32_t L, int32_t P, const void *idx, int32_t idx_bytes,
                      float *codes_out, int32_t *counts_out, float *loss_out, void *ws,
                      size_t ws_bytes, void *stream) {
  CSPLAT_TRACE;
  if (n < 0) return invalid("n < 0");
  if (d < 1 || d > 8) return invalid("d must be 1..8");
  if (L < 1 || L > 16) return invalid("L must be 1..16");
  if (P < 1 || P > 65536) return invalid("P must be 1..65536");
  if (idx_bytes != 1 && idx_bytes != 2) return invalid("idx_bytes must be 1 or 2");
  if (!codes || !codes_out || (n > 0 && (!x || !idx))) return invalid("rvq_update: NULL argument");
  if (!ws || ws_bytes < csplat::rvq_update_workspace_bytes(L, P, d)) {
    set_err("rvq_update workspace too small");
    return CSPLAT_ERR_WORKSPACE;
  }
  RET_IF(check_device());
  return cuda_status(csplat::launch_rvq_update(x, n, n_dev, d, codes, L, P, idx, idx_bytes,
                                               codes_out, counts_out, loss_out, ws,
                                               static_cast<cudaStream_t>(stream)),
                     "csplat_rvq_update");
}

int csplat_rvq_code_grad(const float *d_shat, int64_t n, const int64_t *n_dev, int32_t d,
                         const void *idx, int32_t idx_bytes, int32_t L, int32_t P,
                         float *d_codes, uint32_t flags, void *stream) {
  CSPLAT_TRACE;
  if (n < 0) return invalid("n < 0");
  if (d < 1 || d > 8) return invalid("d must be 1..8");
  if (L < 1 || L > 16) return invalid("L must be 1..16");
  if (P < 1 || P > 65536) return invalid("P must be 1..65536");
  if (idx_bytes != 1 && idx_bytes != 2) return invalid("idx_bytes must be 1 or 2");
  if (!d_codes || (n > 0 && (!d_shat || !idx))) return invalid("rvq_code_grad: NULL argument");
  if (d == 4 && (reinterpret_cast<uintptr_t>(d_codes) & 15u)) {
    set_err("rvq_code_grad: d_codes must be 16-byte aligned");
    return CSPLAT_ERR_ALIGNMENT;
  }
  RET_IF(check_device());
  return cuda_status(csplat::launch_rvq_code_grad(d_shat, n, n_dev, d, L, P, idx, idx_bytes,
                                                  d_codes, (flags & CSPLAT_ACCUMULATE) != 0,
                                                  static_cast<cudaStream_t>(stream)),
                     "csplat_rvq_code_grad");
}

int csplat_rvq_init_stage(const float *x, int64_t n, int32_t d, float *codes, int32_t L,
                          int32_t P, int32_t stage, const void *idx, int32_t idx_bytes,
                          const int64_t *sample, void *stream) {
  CSPLAT_TRACE;
  if (n < 1) return invalid("n must be >= 1");
  if (d < 1 || d > 8) return invalid("d must be 1..8");
  if (L < 1 || L > 16) return invalid("L must be 1..16");
  if (P < 1 || P > 65536) return invalid("P must be 1..65536");
  if (stage < 0 || stage >= L) return invalid("stage must be 0..L-1");
  if (idx_bytes != 1 && idx_bytes != 2) return invalid("idx_bytes must be 1 or 2");
  if (!x || !codes || !sample || (stage > 0 && !idx)) return invalid("rvq_init_stage: NULL argument");
  RET_IF(check_device());
  return cuda_status(csplat::launch_rvq_init_stage(x, n, d, codes, P, stage, idx, idx_bytes, sample,
                                                   static_cast<cudaStream_t>(stream)),
                     "csplat_rvq_init_stage");
}

int csplat_rvq_assign(const float *x, int64_t n, const int64_t *n_dev, int32_t d,
                      const float *codes, int32_t L, int32_t P, void *idx_out, int32_t idx_bytes,
                      float *recon_out, void *stream) {
  CSPLAT_TRACE;
  if (n < 0) return invalid("n < 0");
  if (d < 1 || d > 8) return invalid("d must be 1..8");
  if (L < 1 || L > 16) return invalid("L must be 1..16");
  if (P < 1 || P > 65536) return invalid("P must be 1..65536");
  if (idx_bytes != 1 && idx_bytes != 2) return invalid("idx_bytes must be 1 or 2");
  if (idx_bytes == 1 && P > 256) return invalid("idx_bytes=1 needs P <= 256");
  if (n > 0 && (!x || !codes || !idx_out)) return invalid("rvq: NULL argument");
  RET_IF(check_device());
  return cuda_status(csplat::launch_rvq(x, n, n_dev, d, codes, L, P, idx_out, idx_bytes, recon_out,
                                        static_cast<cudaStream_t>(stream)),
                     "csplat_rvq_assign");
}

int csplat_mask_prune(const csplat_gaussians *in, const csplat_codebook *in_idx, float mask_eps,
                      float reset_mask_logit, const csplat_gaussians_out *out,
                      void *out_scale_idx, void *out_rot_idx, int32_t *keep_map,
                      int64_t *n_kept_dev, void *ws, size_t ws_bytes, void *stream) {
  CSPLAT_TRACE;
  RET_IF(check_gaussians(in));
  if (in->n > 0 && (!in->log_scale || !in->quat)) return invalid("log_scale/quat NULL");
  if (!out || !n_kept_dev) return invalid("out/n_kept NULL");
  if (out->capacity < in->n) return invalid("out capacity < n");
  if (in->n > 0 && (!out->mean || !out->opacity || !out->rgb || !out->log_scale || !out->quat ||
                    !out->mask))
    return invalid("an output plane is NULL");
  if (in_idx) {
    RET_IF(check_codebook(in_idx, false));
    if (!out_scale_idx || !out_rot_idx) return invalid("output index planes NULL");
  }
  if (!(mask_eps > 0.f) || !(mask_eps < 1.f)) return invalid("mask_eps must be in (0,1)");
  if (!ws || ws_bytes < csplat::prune_workspace_bytes(in->n)) {
    set_err("mask_prune workspace too small");
    return CSPLAT_ERR_WORKSPACE;
  }
  RET_IF(check_device());
  csplat::DecodeArgs d;
  if (in_idx) d = decode_args(in_idx);
  return cuda_status(csplat::launch_prune(*in, in_idx ? &d : nullptr, mask_tau(mask_eps),
                                          reset_mask_logit, *out, out_scale_idx, out_rot_idx,
                                          keep_map, n_kept_dev, ws,
                                          static_cast<cudaStream_t>(stream)),
                     "csplat_mask_prune");
}

}  // extern "C"
