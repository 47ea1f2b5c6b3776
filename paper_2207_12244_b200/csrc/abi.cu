// abi.cu -- the C-ABI of include/dfuse_cuda.h: argument checks with the
// reference's error codes, host<->device staging, kernel launches, and the
// device-resident keyframe session. No computation happens on the host
// except per-frame-pair geometry (geometry_host.cpp).
#include <stdio.h>
#include <string.h>

#include <atomic>
#include <memory>
#include <mutex>
#include <new>
#include <vector>

#include "common.cuh"
#include "fusion.cuh"
#include "stereo.cuh"

using namespace dfuse_cuda;

namespace dfuse_cuda {

void* scratch(dfuse_ctx* ctx, int slot, size_t bytes) {
  Buffer& b = ctx->scratch[slot];
  if (bytes == 0) bytes = 16;
  if (b.bytes < bytes) {
    if (b.ptr) DF_CUDA(cudaFreeAsync(b.ptr, ctx->stream));
    b.ptr = nullptr;
    b.bytes = 0;
    DF_CUDA(cudaMallocAsync(&b.ptr, bytes, ctx->stream));
    b.bytes = bytes;
  }
  return b.ptr;
}

}  // namespace dfuse_cuda

namespace {

const char* kErrNames[] = {
    "NonPositiveDepth", "BehindCamera", "OutOfBounds", "DegenerateBaseline", "NoMinimum",
    "ZeroBaselineStep", "DegenerateJacobian", "BorderPixel", "BadMagic", "DimensionMismatch",
    "NonPositiveVariance", "TruncatedFile", "NonPositiveFocal", "NonPositiveGroundTruth",
    "MissingFile", "MalformedLine", "NonUnitQuaternion", "BadImageFormat", "NonPositiveScale",
    "CgDivergence", "NoSemiDenseSupport", "NoValidGroundTruth", "MismatchedKeyframeSets",
    "IoError", "UnknownKey", "TypeError", "InvalidArgument"};

template <class F>
int guarded(dfuse_ctx* ctx, F&& f) {
  if (!ctx) return DFUSE_E_INVALID_ARGUMENT;
  try {
    DF_CUDA(cudaSetDevice(ctx->device));
    f();
    ctx->last_error.clear();
    return DFUSE_OK;
  } catch (const RefError& e) {
    ctx->last_error = e.msg;
    return e.code;
  } catch (const CudaFailure& e) {
    ctx->last_error = std::string("CUDA: ") + cudaGetErrorString(e.err) + " in " + e.what;
    return DFUSE_E_CUDA;
  } catch (const std::bad_alloc&) {
    ctx->last_error = "host allocation failed";
    return DFUSE_E_CUDA;
  }
}

void require(bool ok, int code, const char* msg) {
  if (!ok) throw RefError{code, msg};
}

void h2d(dfuse_ctx* ctx, void* dst, const void* src, size_t bytes) {
  if (bytes) DF_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
}
void d2h(dfuse_ctx* ctx, void* dst, const void* src, size_t bytes) {
  if (bytes) DF_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
}
void sync(dfuse_ctx* ctx) { DF_CUDA(cudaStreamSynchronize(ctx->stream)); }

void check_geom(const dfuse_epigeom* g) {
  require(g != nullptr, DFUSE_E_INVALID_ARGUMENT, "null geometry");
  require(g->K.width > 0 && g->K.height > 0, DFUSE_E_INVALID_ARGUMENT,
          "raster dimensions must be positive");
}

struct Sel {
  bool net, grad, scale;
};
Sel terms_for(int mode) {
  Sel s{true, true, true};
  if (mode == DFUSE_MODE_NOPAIRWISE) s.grad = false;
  if (mode == DFUSE_MODE_LSSCALE) s.net = s.scale = false;
  return s;
}

bool any_valid(const uint8_t* v, long P) {
  for (long i = 0; i < P; ++i)
    if (v[i]) return true;
  return false;
}

// huber_weight throws InvalidArgument for delta <= 0 (fusion.hpp:80) on the
// first term it is evaluated for; the kernels do not throw, so the host
// rejects the configurations under which the reference would.
void check_deltas(const dfuse_robust_cfg* cfg, int mode, int w, int h, bool semi_used,
                  bool net_grad_used) {
  const Sel sel = terms_for(mode);
  if (semi_used && cfg->delta_semi <= 0.0)
    throw RefError{DFUSE_E_INVALID_ARGUMENT, "huber delta must be > 0"};
  if (net_grad_used) {
    if (sel.net && cfg->delta_net <= 0.0)
      throw RefError{DFUSE_E_INVALID_ARGUMENT, "huber delta must be > 0"};
    if (sel.grad && (w > 1 || h > 1) && cfg->delta_grad <= 0.0)
      throw RefError{DFUSE_E_INVALID_ARGUMENT, "huber delta must be > 0"};
  }
}

// device workspace of one fusion problem
struct FusionWS {
  double* pred;  // 6P
  double* sd;
  double* sv;
  uint8_t* svalid;
  double* lnsd;
  double* irs;
  double* ivar[3];
  double* ld[2];
  double *diag, *right, *down, *b, *x, *r, *z, *p0, *p1, *q;
  ReduceSlot* slots;
  unsigned long long* halo;
  FusionControl* ctl;
  FusionStateDev* st;  // [2]
};

size_t align_up(size_t v) { return (v + 255) & ~size_t(255); }

FusionWS alloc_fusion_ws(dfuse_ctx* ctx, long P, int grid, int slot) {
  const size_t dP = align_up(sizeof(double) * P);
  const bool resident = fusion_resident_possible(P, grid);
  size_t total = 6 * dP + 7 * dP + align_up(P) + 12 * dP + align_up(fusion_slots_bytes(grid)) +
                 align_up(sizeof(FusionControl)) + align_up(2 * sizeof(FusionStateDev)) +
                 (resident ? align_up(fusion_halo_bytes(P)) : 0);
  char* base = (char*)scratch(ctx, slot, total);
  FusionWS w;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    char* p = base + o;
    o += align_up(bytes);
    return p;
  };
  w.pred = (double*)take(6 * dP);
  w.sd = (double*)take(dP);
  w.sv = (double*)take(dP);
  w.svalid = (uint8_t*)take(P);
  w.lnsd = (double*)take(dP);
  w.irs = (double*)take(dP);
  for (int k = 0; k < 3; ++k) w.ivar[k] = (double*)take(dP);
  w.ld[0] = (double*)take(dP);
  w.ld[1] = (double*)take(dP);
  w.diag = (double*)take(dP);
  w.right = (double*)take(dP);
  w.down = (double*)take(dP);
  w.b = (double*)take(dP);
  w.x = (double*)take(dP);
  w.r = (double*)take(dP);
  w.z = (double*)take(dP);
  w.p0 = (double*)take(dP);
  w.p1 = (double*)take(dP);
  w.q = (double*)take(dP);
  w.slots = (ReduceSlot*)take(fusion_slots_bytes(grid));
  w.ctl = (FusionControl*)take(sizeof(FusionControl));
  w.st = (FusionStateDev*)take(2 * sizeof(FusionStateDev));
  w.halo = resident ? (unsigned long long*)take(fusion_halo_bytes(P)) : nullptr;
  return w;
}

void fill_args(FusionArgs& a, const FusionWS& w, int W, int H) {
  memset(&a, 0, sizeof a);
  a.W = W;
  a.H = H;
  const long P = (long)W * H;
  for (int c = 0; c < 6; ++c) a.pred[c] = w.pred + align_up(sizeof(double) * P) / 8 * c;
  a.sd = w.sd;
  a.sv = w.sv;
  a.svalid = w.svalid;
  a.lnsd = w.lnsd;
  a.irs = w.irs;
  for (int k = 0; k < 3; ++k) a.ivar[k] = w.ivar[k];
  a.ld[0] = w.ld[0];
  a.ld[1] = w.ld[1];
  a.diag = w.diag;
  a.right = w.right;
  a.down = w.down;
  a.b = w.b;
  a.x = w.x;
  a.r = w.r;
  a.z = w.z;
  a.p[0] = w.p0;
  a.p[1] = w.p1;
  a.q = w.q;
  a.slots = w.slots;
  a.halo = w.halo;
  a.ctl = w.ctl;
  a.st_in = w.st;
  a.st_out = w.st + 1;
}

void set_cfg(FusionArgs& a, const dfuse_robust_cfg* cfg, int mode) {
  a.dsemi = cfg->delta_semi;
  a.dnet = cfg->delta_net;
  a.dgrad = cfg->delta_grad;
  a.cg_tol = cfg->cg_tol;
  a.gn = cfg->gn_iterations;
  a.cg_max = cfg->cg_max_iters;
  a.est_scale = cfg->estimate_scale;
  a.mode = mode;
}

void upload_inputs(dfuse_ctx* ctx, const FusionArgs& a, const dfuse_fusion_inputs* in,
                   bool with_pred) {
  const long P = (long)in->width * in->height;
  if (with_pred)
    for (int c = 0; c < 6; ++c) {
      require(in->pred[c] != nullptr, DFUSE_E_INVALID_ARGUMENT, "null prediction plane");
      h2d(ctx, (void*)a.pred[c], in->pred[c], sizeof(double) * P);
    }
  require(in->semi_depth && in->semi_variance && in->semi_valid, DFUSE_E_INVALID_ARGUMENT,
          "null semi-dense map");
  h2d(ctx, (void*)a.sd, in->semi_depth, sizeof(double) * P);
  h2d(ctx, (void*)a.sv, in->semi_variance, sizeof(double) * P);
  h2d(ctx, (void*)a.svalid, in->semi_valid, P);
}

void check_inputs(const dfuse_fusion_inputs* in, int mode) {
  require(in != nullptr, DFUSE_E_INVALID_ARGUMENT, "null fusion inputs");
  require(in->width > 0 && in->height > 0, DFUSE_E_INVALID_ARGUMENT,
          "raster dimensions must be positive");
  require(mode >= 0 && mode <= 2, DFUSE_E_INVALID_ARGUMENT, "unknown fusion mode");
  require((long)in->width * in->height < (1L << 31), DFUSE_E_INVALID_ARGUMENT,
          "raster too large");
}

}  // namespace

// ===========================================================================
extern "C" {

int dfuse_abi_version(void) { return DFUSE_ABI_VERSION; }

const char* dfuse_err_name(int code) {
  if (code == 0) return "Ok";
  if (code >= 1 && code <= (int)(sizeof kErrNames / sizeof kErrNames[0])) return kErrNames[code - 1];
  if (code == DFUSE_E_CUDA) return "Cuda";
  return "UnknownError";
}

int dfuse_ctx_create(int device, dfuse_ctx** out) {
  if (!out) return DFUSE_E_INVALID_ARGUMENT;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n <= 0 || device < 0 || device >= n) {
    cudaGetLastError();
    return DFUSE_E_CUDA;
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return DFUSE_E_CUDA;
  if (prop.major < 10) return DFUSE_E_CUDA;  // built for sm_100a only
  dfuse_ctx* ctx = new (std::nothrow) dfuse_ctx();
  if (!ctx) return DFUSE_E_CUDA;
  ctx->device = device;
  ctx->num_sms = prop.multiProcessorCount;
  const char* tr = getenv("DFUSE_TRACE");
  ctx->trace = tr ? atoi(tr) : 0;
  if (const char* rp = getenv("DFUSE_PCG_REPEAT")) {
    ctx->diag_repeat = atoi(rp);
    ctx->diag_sweep = strchr(rp, ',') ? atoi(strchr(rp, ',') + 1) : 0;
  }
  if (cudaSetDevice(device) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete ctx;
    return DFUSE_E_CUDA;
  }
  for (auto& e : ctx->ev) cudaEventCreate(&e);
  *out = ctx;
  return DFUSE_OK;
}

int dfuse_ctx_destroy(dfuse_ctx* ctx) {
  if (!ctx) return DFUSE_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (auto& b : ctx->scratch)
    if (b.ptr) cudaFreeAsync(b.ptr, ctx->stream);
  cudaStreamSynchronize(ctx->stream);
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  for (auto& t : ctx->tex_cache)
    if (t.tex) cudaDestroyTextureObject(t.tex);
  cudaStreamDestroy(ctx->stream);
  delete ctx;
  return DFUSE_OK;
}

const char* dfuse_last_error(const dfuse_ctx* ctx) {
  return ctx ? ctx->last_error.c_str() : "null context";
}

int dfuse_ctx_set_solver_ctas(dfuse_ctx* ctx, int ctas) {
  if (!ctx || ctas < 0) return DFUSE_E_INVALID_ARGUMENT;
  ctx->solver_ctas = ctas;
  return DFUSE_OK;
}

int dfuse_ctx_set_stereo_texture(dfuse_ctx* ctx, int on) {
  if (!ctx) return DFUSE_E_INVALID_ARGUMENT;
  ctx->stereo_tex = on ? 1 : 0;
  return DFUSE_OK;
}

int64_t dfuse_ctx_texture_launches(const dfuse_ctx* ctx) { return ctx ? ctx->tex_launches : 0; }

int dfuse_ctx_set_fp32_predictions(dfuse_ctx* ctx, int on) {
  if (!ctx) return DFUSE_E_INVALID_ARGUMENT;
  ctx->pred_fp32 = on ? 1 : 0;
  return DFUSE_OK;
}

int dfuse_debug_sync_bench(dfuse_ctx* ctx, int n, int variant, int grid, float* ms) {
  return guarded(ctx, [&] {
    require(ms != nullptr && n >= 0, DFUSE_E_INVALID_ARGUMENT, "bad arguments");
    *ms = sync_bench(ctx, n, variant, grid);
  });
}

int dfuse_ctx_set_solver_path(dfuse_ctx* ctx, int path) {
  if (!ctx || path < 0 || path > 3) return DFUSE_E_INVALID_ARGUMENT;
  ctx->force_streaming = path;
  return DFUSE_OK;
}

int64_t dfuse_ctx_launch_count(const dfuse_ctx* ctx) { return ctx ? ctx->launches : 0; }

void* dfuse_ctx_stream(const dfuse_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

// ---------------------------------------------------------------------------
int dfuse_texture_mask(dfuse_ctx* ctx, const float* img, int w, int h, double threshold,
                       uint8_t* mask) {
  return guarded(ctx, [&] {
    require(threshold > 0.0, DFUSE_E_INVALID_ARGUMENT, "texture threshold must be > 0");
    require(w > 0 && h > 0, DFUSE_E_INVALID_ARGUMENT, "raster dimensions must be positive");
    require(img && mask, DFUSE_E_INVALID_ARGUMENT, "null pointer");
    const long P = (long)w * h;
    float* dimg = (float*)scratch(ctx, S_IMG0, sizeof(float) * P);
    uint8_t* dmask = (uint8_t*)scratch(ctx, S_MASK, P);
    h2d(ctx, dimg, img, sizeof(float) * P);
    launch_texture_mask(ctx, dimg, w, h, threshold, dmask);
    d2h(ctx, mask, dmask, P);
    sync(ctx);
  });
}

int dfuse_search_depth(dfuse_ctx* ctx, const dfuse_epigeom* g, const float* I0, const float* I1,
                       int n, const double* px, const double* prior, const uint8_t* has_prior,
                       const dfuse_search_cfg* cfg, int32_t* status, dfuse_obs* obs, int32_t* best,
                       int32_t* n_steps) {
  // unversioned images: uploaded by this call
  return dfuse_search_depth_gen(ctx, g, I0, 0, I1, 0, n, px, prior, has_prior, cfg, status, obs,
                                best, n_steps);
}

int dfuse_photometric_error_5pt(dfuse_ctx* ctx, const dfuse_epigeom* g, const float* I0,
                                const float* I1, double x, double y, double d, double e[5],
                                int32_t* status) {
  return guarded(ctx, [&] {
    check_geom(g);
    require(I0 && I1 && e && status, DFUSE_E_INVALID_ARGUMENT, "null pointer");
    const long P = (long)g->K.width * g->K.height;
    float* d0 = (float*)scratch(ctx, S_IMG0, sizeof(float) * P);
    float* d1 = (float*)scratch(ctx, S_IMG1, sizeof(float) * P);
    double* out = (double*)scratch(ctx, S_TMP3, 8 * sizeof(double));
    h2d(ctx, d0, I0, sizeof(float) * P);
    h2d(ctx, d1, I1, sizeof(float) * P);
    launch_photometric(ctx, *g, d0, d1, x, y, d, out);
    double h[6];
    d2h(ctx, h, out, sizeof h);
    sync(ctx);
    for (int j = 0; j < 5; ++j) e[j] = h[j];
    *status = (int32_t)h[5];
  });
}

int dfuse_update_semidense(dfuse_ctx* ctx, int w, int h, double* depth, double* variance,
                           uint8_t* valid, int32_t* inlier_count, int n_obs,
                           const dfuse_obs* obs) {
  return guarded(ctx, [&] {
    require(w > 0 && h > 0, DFUSE_E_INVALID_ARGUMENT, "raster dimensions must be positive");
    require(depth && variance && valid && inlier_count && (n_obs == 0 || obs),
            DFUSE_E_INVALID_ARGUMENT, "null pointer");
    const long P = (long)w * h;
    double* dd = (double*)scratch(ctx, S_SEMI_D, sizeof(double) * P);
    double* dv = (double*)scratch(ctx, S_SEMI_V, sizeof(double) * P);
    uint8_t* dval = (uint8_t*)scratch(ctx, S_SEMI_VALID, P);
    int* cnt = (int*)scratch(ctx, S_COUNTERS, 64);
    h2d(ctx, dd, depth, sizeof(double) * P);
    h2d(ctx, dv, variance, sizeof(double) * P);
    h2d(ctx, dval, valid, P);
    if (n_obs > 0) {
      dfuse_obs* dobs = (dfuse_obs*)scratch(ctx, S_OBS, sizeof(dfuse_obs) * n_obs);
      int* head = (int*)scratch(ctx, S_TMP0, sizeof(int) * P);
      int* link = (int*)scratch(ctx, S_TMP1, sizeof(int) * n_obs);
      h2d(ctx, dobs, obs, sizeof(dfuse_obs) * n_obs);
      launch_update_list(ctx, dobs, n_obs, w, h, head, link, cnt + 1, dd, dv, dval);
    }
    launch_count_valid(ctx, dval, P, cnt);  // semidense.hpp:413-415
    d2h(ctx, depth, dd, sizeof(double) * P);
    d2h(ctx, variance, dv, sizeof(double) * P);
    d2h(ctx, valid, dval, P);
    d2h(ctx, inlier_count, cnt, sizeof(int));
    sync(ctx);
  });
}

int dfuse_stereo_update(dfuse_ctx* ctx, const dfuse_epigeom* g, const float* I0, const float* I1,
                        const uint8_t* mask, const dfuse_search_cfg* cfg, double* depth,
                        double* variance, uint8_t* valid, int32_t* inlier_count, int32_t* n_obs,
                        int8_t* status, int32_t* best, int32_t* n_steps, dfuse_obs* obs) {
  return guarded(ctx, [&] {
    check_geom(g);
    require(cfg && I0 && I1 && mask && depth && variance && valid && inlier_count && n_obs,
            DFUSE_E_INVALID_ARGUMENT, "null pointer");
    const int w = g->K.width, h = g->K.height;
    const long P = (long)w * h;
    StereoArgs a;
    memset(&a, 0, sizeof a);
    a.g = *g;
    a.cfg = *cfg;
    float* dI0 = (float*)scratch(ctx, S_IMG0, sizeof(float) * P);
    float* dI1 = (float*)scratch(ctx, S_IMG1, sizeof(float) * P);
    uint8_t* dmask = (uint8_t*)scratch(ctx, S_MASK, P);
    h2d(ctx, dI0, I0, sizeof(float) * P);
    h2d(ctx, dI1, I1, sizeof(float) * P);
    h2d(ctx, dmask, mask, P);
    a.I0 = dI0;
    a.I1 = dI1;
    a.depth = (double*)scratch(ctx, S_SEMI_D, sizeof(double) * P);
    a.variance = (double*)scratch(ctx, S_SEMI_V, sizeof(double) * P);
    a.valid = (uint8_t*)scratch(ctx, S_SEMI_VALID, P);
    h2d(ctx, a.depth, depth, sizeof(double) * P);
    h2d(ctx, a.variance, variance, sizeof(double) * P);
    h2d(ctx, a.valid, valid, P);
    int* counters = (int*)scratch(ctx, S_COUNTERS, 64);  // [0] work [1] n_list [2] n_obs [3] installed [4] count
    DF_CUDA(cudaMemsetAsync(counters, 0, 64, ctx->stream));
    int* list = (int*)scratch(ctx, S_LIST, sizeof(int) * P);
    launch_mask_list(ctx, dmask, P, list, counters + 1);
    int n_list = 0;
    d2h(ctx, &n_list, counters + 1, sizeof(int));
    sync(ctx);
    a.list = list;
    a.n_items = n_list;
    a.work_counter = counters;
    a.n_obs = counters + 2;
    a.n_installed = counters + 3;
    if (status) {
      a.status = scratch(ctx, S_STATUS, P);
      DF_CUDA(cudaMemsetAsync(a.status, 0xff, P, ctx->stream));  // DFUSE_EPI_NOT_SEARCHED
    }
    if (best) {
      a.best = (int32_t*)scratch(ctx, S_BEST, sizeof(int32_t) * P);
      DF_CUDA(cudaMemsetAsync(a.best, 0xff, sizeof(int32_t) * P, ctx->stream));
    }
    if (n_steps) {
      a.n_steps = (int32_t*)scratch(ctx, S_NSTEPS, sizeof(int32_t) * P);
      DF_CUDA(cudaMemsetAsync(a.n_steps, 0xff, sizeof(int32_t) * P, ctx->stream));
    }
    dfuse_obs* dense = nullptr;
    if (obs) {
      dense = (dfuse_obs*)scratch(ctx, S_OBS, sizeof(dfuse_obs) * P);
      a.obs = dense;
      a.obs_flag = (uint8_t*)scratch(ctx, S_TMP0, P);
      DF_CUDA(cudaMemsetAsync(a.obs_flag, 0, P, ctx->stream));
    }
    if (n_list > 0) launch_stereo(ctx, a, false);
    int hc[2] = {0, 0};
    d2h(ctx, hc, counters + 2, 2 * sizeof(int));
    sync(ctx);
    *n_obs = hc[0];
    if (hc[0] > 0) {  // update_semidense runs only when observations exist (pipeline.hpp:209)
      launch_count_valid(ctx, a.valid, P, counters + 4);
      d2h(ctx, inlier_count, counters + 4, sizeof(int));
    }
    d2h(ctx, depth, a.depth, sizeof(double) * P);
    d2h(ctx, variance, a.variance, sizeof(double) * P);
    d2h(ctx, valid, a.valid, P);
    if (status) d2h(ctx, status, a.status, P);
    if (best) d2h(ctx, best, a.best, sizeof(int32_t) * P);
    if (n_steps) d2h(ctx, n_steps, a.n_steps, sizeof(int32_t) * P);
    if (obs && hc[0] > 0) {
      dfuse_obs* compact = (dfuse_obs*)scratch(ctx, S_TMP2, sizeof(dfuse_obs) * hc[0]);
      int* blocks = (int*)scratch(ctx, S_TMP1, sizeof(int) * ((P + 1023) / 1024 + 1));
      launch_compact_obs(ctx, a.obs_flag, dense, P, blocks, compact);
      d2h(ctx, obs, compact, sizeof(dfuse_obs) * hc[0]);
    }
    sync(ctx);
  });
}

// ---------------------------------------------------------------------------
// versioned host images: process-wide device copies
//
// The reference's stereo_scan calls search_depth once per masked pixel from
// an OpenMP loop (pipeline.hpp:167-178), each call with the same two
// images. Per call, the drop-in passes the images' generation
// (dfuse::IntensityImage::generation(), renewed by every mutable access), and
// the device copy is looked up by (device, host pointer, bytes, generation)
// in one cache shared by every context of the process: one upload per image
// version however many threads and pixels use it. Entries are reference
// counted, so evicting one never frees a buffer a queued search still reads.
namespace {

struct CachedImage {
  int device;
  const void* host;
  size_t bytes;
  uint64_t gen;
  std::shared_ptr<void> dev;
  uint64_t tick;
};
constexpr int kImageCachePerDevice = 8;
std::mutex g_img_mu;
std::vector<CachedImage>* g_img = new std::vector<CachedImage>();  // never destroyed (exit order)
uint64_t g_img_tick = 0;
std::atomic<long long> g_uploads{0}, g_upload_bytes{0};

struct ImageRef {
  const float* ptr;
  std::shared_ptr<void> hold;  // keeps a cached copy alive for the call
};

ImageRef device_image(dfuse_ctx* ctx, int slot, const float* host, size_t bytes, uint64_t gen) {
  if (gen == 0) {  // unversioned: a private upload for this call
    float* d = (float*)scratch(ctx, slot, bytes);
    h2d(ctx, d, host, bytes);
    g_uploads += 1;
    g_upload_bytes += (long long)bytes;
    return {d, nullptr};
  }
  std::lock_guard<std::mutex> lk(g_img_mu);
  const uint64_t tick = ++g_img_tick;
  size_t lru = SIZE_MAX;
  int n = 0;
  for (size_t k = 0; k < g_img->size(); ++k) {
    CachedImage& e = (*g_img)[k];
    if (e.device != ctx->device) continue;
    if (e.host == host && e.bytes == bytes && e.gen == gen) {
      e.tick = tick;
      return {(const float*)e.dev.get(), e.dev};
    }
    ++n;
    if (lru == SIZE_MAX || e.tick < (*g_img)[lru].tick) lru = k;
  }
  if (n >= kImageCachePerDevice) g_img->erase(g_img->begin() + (long)lru);
  void* d = nullptr;
  DF_CUDA(cudaMalloc(&d, bytes));
  const int dev = ctx->device;
  std::shared_ptr<void> hold(d, [dev](void* p) {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(dev);
    cudaFree(p);
    cudaSetDevice(cur);
  });
  // complete before the entry is visible to any other context's stream
  DF_CUDA(cudaMemcpyAsync(d, host, bytes, cudaMemcpyHostToDevice, ctx->stream));
  DF_CUDA(cudaStreamSynchronize(ctx->stream));
  g_uploads += 1;
  g_upload_bytes += (long long)bytes;
  g_img->push_back(CachedImage{dev, host, bytes, gen, hold, tick});
  return {(const float*)d, hold};
}

// search_depth over a list of pixels on device images (dfuse_search_depth*)
void search_list(dfuse_ctx* ctx, const dfuse_epigeom* g, const float* dI0, const float* dI1, int n,
                 const double* px, const double* prior, const uint8_t* has_prior,
                 const dfuse_search_cfg* cfg, int32_t* status, dfuse_obs* obs, int32_t* best,
                 int32_t* n_steps) {
  StereoArgs a;
  memset(&a, 0, sizeof a);
  a.g = *g;
  a.cfg = *cfg;
  a.I0 = dI0;
  a.I1 = dI1;
  a.n_items = n;
  a.work_counter = (int*)scratch(ctx, S_COUNTERS, 64);
  a.px = (const double*)scratch(ctx, S_PX, sizeof(double) * 2 * n);
  h2d(ctx, (void*)a.px, px, sizeof(double) * 2 * n);
  if (prior) {
    a.prior = (const double*)scratch(ctx, S_PRIOR, sizeof(double) * 2 * n);
    h2d(ctx, (void*)a.prior, prior, sizeof(double) * 2 * n);
    if (has_prior) {
      a.has_prior = (const uint8_t*)scratch(ctx, S_HASPRIOR, n);
      h2d(ctx, (void*)a.has_prior, has_prior, n);
    }
  }
  a.status = scratch(ctx, S_STATUS, sizeof(int32_t) * n);
  a.obs = (dfuse_obs*)scratch(ctx, S_OBS, sizeof(dfuse_obs) * n);
  a.best = (int32_t*)scratch(ctx, S_BEST, sizeof(int32_t) * n);
  a.n_steps = (int32_t*)scratch(ctx, S_NSTEPS, sizeof(int32_t) * n);
  launch_stereo(ctx, a, true);
  d2h(ctx, status, a.status, sizeof(int32_t) * n);
  d2h(ctx, obs, a.obs, sizeof(dfuse_obs) * n);
  if (best) d2h(ctx, best, a.best, sizeof(int32_t) * n);
  if (n_steps) d2h(ctx, n_steps, a.n_steps, sizeof(int32_t) * n);
  sync(ctx);
}

}  // namespace

extern "C" {

int dfuse_image_uploads(int64_t* count, int64_t* bytes) {
  if (count) *count = g_uploads.load();
  if (bytes) *bytes = g_upload_bytes.load();
  return DFUSE_OK;
}

int dfuse_search_depth_gen(dfuse_ctx* ctx, const dfuse_epigeom* g, const float* I0, uint64_t gen0,
                           const float* I1, uint64_t gen1, int n, const double* px,
                           const double* prior, const uint8_t* has_prior,
                           const dfuse_search_cfg* cfg, int32_t* status, dfuse_obs* obs,
                           int32_t* best, int32_t* n_steps) {
  return guarded(ctx, [&] {
    check_geom(g);
    require(cfg && I0 && I1 && (n == 0 || (px && status && obs)), DFUSE_E_INVALID_ARGUMENT,
            "null pointer");
    if (n <= 0) return;
    const size_t bytes = sizeof(float) * (size_t)g->K.width * g->K.height;
    const ImageRef i0 = device_image(ctx, S_IMG0, I0, bytes, gen0);
    const ImageRef i1 = device_image(ctx, S_IMG1, I1, bytes, gen1);
    search_list(ctx, g, i0.ptr, i1.ptr, n, px, prior, has_prior, cfg, status, obs, best, n_steps);
  });
}

int dfuse_photometric_error_5pt_gen(dfuse_ctx* ctx, const dfuse_epigeom* g, const float* I0,
                                    uint64_t gen0, const float* I1, uint64_t gen1, double x,
                                    double y, double d, double e[5], int32_t* status) {
  return guarded(ctx, [&] {
    check_geom(g);
    require(I0 && I1 && e && status, DFUSE_E_INVALID_ARGUMENT, "null pointer");
    const size_t bytes = sizeof(float) * (size_t)g->K.width * g->K.height;
    const ImageRef i0 = device_image(ctx, S_IMG0, I0, bytes, gen0);
    const ImageRef i1 = device_image(ctx, S_IMG1, I1, bytes, gen1);
    double* out = (double*)scratch(ctx, S_TMP3, 8 * sizeof(double));
    launch_photometric(ctx, *g, i0.ptr, i1.ptr, x, y, d, out);
    double h[6];
    d2h(ctx, h, out, sizeof h);
    sync(ctx);
    for (int j = 0; j < 5; ++j) e[j] = h[j];
    *status = (int32_t)h[5];
  });
}

// stereo_scan (pipeline.hpp:157-190): every masked pixel searched with the
// prior read from the map; the OK observations in raster order. The map is
// not changed: the kernel's fused update runs on a scratch copy (each pixel
// reads only its own prior, so the observations are those of a read-only
// scan) and is dropped.
int dfuse_stereo_scan(dfuse_ctx* ctx, const dfuse_epigeom* g, const float* I0, uint64_t gen0,
                      const float* I1, uint64_t gen1, const uint8_t* mask, const double* depth,
                      const double* variance, const uint8_t* valid, const dfuse_search_cfg* cfg,
                      dfuse_obs* obs, int32_t* n_obs) {
  return guarded(ctx, [&] {
    check_geom(g);
    require(cfg && I0 && I1 && mask && depth && variance && valid && obs && n_obs,
            DFUSE_E_INVALID_ARGUMENT, "null pointer");
    const long P = (long)g->K.width * g->K.height;
    const ImageRef i0 = device_image(ctx, S_IMG0, I0, sizeof(float) * P, gen0);
    const ImageRef i1 = device_image(ctx, S_IMG1, I1, sizeof(float) * P, gen1);
    StereoArgs a;
    memset(&a, 0, sizeof a);
    a.g = *g;
    a.cfg = *cfg;
    a.I0 = i0.ptr;
    a.I1 = i1.ptr;
    uint8_t* dmask = (uint8_t*)scratch(ctx, S_MASK, P);
    h2d(ctx, dmask, mask, P);
    a.depth = (double*)scratch(ctx, S_SEMI_D, sizeof(double) * P);
    a.variance = (double*)scratch(ctx, S_SEMI_V, sizeof(double) * P);
    a.valid = (uint8_t*)scratch(ctx, S_SEMI_VALID, P);
    h2d(ctx, a.depth, depth, sizeof(double) * P);
    h2d(ctx, a.variance, variance, sizeof(double) * P);
    h2d(ctx, a.valid, valid, P);
    int* counters = (int*)scratch(ctx, S_COUNTERS, 64);
    DF_CUDA(cudaMemsetAsync(counters, 0, 64, ctx->stream));
    int* list = (int*)scratch(ctx, S_LIST, sizeof(int) * P);
    launch_mask_list(ctx, dmask, P, list, counters + 1);
    int n_list = 0;
    d2h(ctx, &n_list, counters + 1, sizeof(int));
    sync(ctx);
    a.list = list;
    a.n_items = n_list;
    a.work_counter = counters;
    a.n_obs = counters + 2;
    a.n_installed = counters + 3;
    dfuse_obs* dense = (dfuse_obs*)scratch(ctx, S_OBS, sizeof(dfuse_obs) * P);
    a.obs = dense;
    a.obs_flag = (uint8_t*)scratch(ctx, S_TMP0, P);
    DF_CUDA(cudaMemsetAsync(a.obs_flag, 0, P, ctx->stream));
    if (n_list > 0) launch_stereo(ctx, a, false);
    int nb = 0;
    d2h(ctx, &nb, counters + 2, sizeof(int));
    sync(ctx);
    *n_obs = nb;
    if (nb > 0) {
      dfuse_obs* compact = (dfuse_obs*)scratch(ctx, S_TMP2, sizeof(dfuse_obs) * nb);
      int* blocks = (int*)scratch(ctx, S_TMP1, sizeof(int) * ((P + 1023) / 1024 + 1));
      launch_compact_obs(ctx, a.obs_flag, dense, P, blocks, compact);
      d2h(ctx, obs, compact, sizeof(dfuse_obs) * nb);
      sync(ctx);
    }
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// fusion
namespace {

struct FusionCall {
  FusionArgs a;
  FusionWS w;
  int grid;
};

FusionCall prepare(dfuse_ctx* ctx, const dfuse_fusion_inputs* in, const double* log_depth,
                   double scale, const dfuse_robust_cfg* cfg, int mode, int op, bool with_pred) {
  check_inputs(in, mode);
  require(log_depth != nullptr && cfg != nullptr, DFUSE_E_INVALID_ARGUMENT, "null pointer");
  FusionCall c;
  c.grid = fusion_grid(ctx);
  const long P = (long)in->width * in->height;
  c.w = alloc_fusion_ws(ctx, P, c.grid, S_FUSION_WS);
  fill_args(c.a, c.w, in->width, in->height);
  set_cfg(c.a, cfg, mode);
  c.a.op = op;
  c.a.scale0 = scale;
  c.a.inlier_count = in->inlier_count;
  upload_inputs(ctx, c.a, in, with_pred);
  h2d(ctx, c.w.ld[0], log_depth, sizeof(double) * P);
  return c;
}

}  // namespace

int dfuse_assemble_normal_equations(dfuse_ctx* ctx, const dfuse_fusion_inputs* in,
                                    const double* log_depth, double scale,
                                    const dfuse_robust_cfg* cfg, int mode, double* diag,
                                    double* right, double* down, double* b) {
  return guarded(ctx, [&] {
    check_inputs(in, mode);
    require(cfg && diag && right && down && b, DFUSE_E_INVALID_ARGUMENT, "null pointer");
    const long P = (long)in->width * in->height;
    check_deltas(cfg, mode, in->width, in->height, any_valid(in->semi_valid, P), true);
    FusionCall c = prepare(ctx, in, log_depth, scale, cfg, mode, OP_ASSEMBLE, true);
    launch_fusion(ctx, c.a, c.grid);
    d2h(ctx, diag, c.w.diag, sizeof(double) * P);
    d2h(ctx, right, c.w.right, sizeof(double) * P);
    d2h(ctx, down, c.w.down, sizeof(double) * P);
    d2h(ctx, b, c.w.b, sizeof(double) * P);
    sync(ctx);
  });
}

int dfuse_total_cost(dfuse_ctx* ctx, const dfuse_fusion_inputs* in, const double* log_depth,
                     double scale, const dfuse_robust_cfg* cfg, int mode, double* cost) {
  return guarded(ctx, [&] {
    require(cost != nullptr, DFUSE_E_INVALID_ARGUMENT, "null pointer");
    FusionCall c = prepare(ctx, in, log_depth, scale, cfg, mode, OP_COST, true);
    launch_fusion(ctx, c.a, c.grid);
    d2h(ctx, cost, &c.w.ctl->value[0], sizeof(double));
    sync(ctx);
  });
}

int dfuse_cost_gradient(dfuse_ctx* ctx, const dfuse_fusion_inputs* in, const double* log_depth,
                        double scale, const dfuse_robust_cfg* cfg, int mode, double* cost,
                        double* wrt_log_depth, double* wrt_ln_scale) {
  return guarded(ctx, [&] {
    require(cost && wrt_log_depth && wrt_ln_scale, DFUSE_E_INVALID_ARGUMENT, "null pointer");
    check_inputs(in, mode);
    const long P = (long)in->width * in->height;
    check_deltas(cfg, mode, in->width, in->height, any_valid(in->semi_valid, P), true);
    FusionCall c = prepare(ctx, in, log_depth, scale, cfg, mode, OP_COST, true);
    launch_gradient(ctx, c.a, c.grid, c.w.x);
    d2h(ctx, wrt_log_depth, c.w.x, sizeof(double) * P);
    double v[2];
    d2h(ctx, v, &c.w.ctl->value[0], 2 * sizeof(double));
    sync(ctx);
    *cost = v[0];
    *wrt_ln_scale = v[1];
  });
}

int dfuse_stencil_apply(dfuse_ctx* ctx, int w, int h, const double* diag, const double* right,
                        const double* down, const double* x, double* y) {
  return guarded(ctx, [&] {
    require(w > 0 && h > 0, DFUSE_E_INVALID_ARGUMENT, "raster dimensions must be positive");
    require(diag && right && down && x && y, DFUSE_E_INVALID_ARGUMENT, "null pointer");
    const long P = (long)w * h;
    double* buf = (double*)scratch(ctx, S_FUSION_WS, sizeof(double) * 5 * P);
    h2d(ctx, buf, diag, sizeof(double) * P);
    h2d(ctx, buf + P, right, sizeof(double) * P);
    h2d(ctx, buf + 2 * P, down, sizeof(double) * P);
    h2d(ctx, buf + 3 * P, x, sizeof(double) * P);
    launch_stencil_apply(ctx, w, h, buf, buf + P, buf + 2 * P, buf + 3 * P, buf + 4 * P);
    d2h(ctx, y, buf + 4 * P, sizeof(double) * P);
    sync(ctx);
  });
}

int dfuse_solve_depth_step(dfuse_ctx* ctx, int w, int h, const double* diag, const double* right,
                           const double* down, const double* b, const dfuse_robust_cfg* cfg,
                           double* delta, int32_t* iterations) {
  return guarded(ctx, [&] {
    require(w > 0 && h > 0, DFUSE_E_INVALID_ARGUMENT, "raster dimensions must be positive");
    require(diag && right && down && b && cfg && delta, DFUSE_E_INVALID_ARGUMENT,
            "null pointer");
    const long P = (long)w * h;
    FusionCall c;
    c.grid = fusion_grid(ctx);
    c.w = alloc_fusion_ws(ctx, P, c.grid, S_FUSION_WS);
    fill_args(c.a, c.w, w, h);
    set_cfg(c.a, cfg, DFUSE_MODE_FULL);
    c.a.op = OP_PCG;
    h2d(ctx, c.w.diag, diag, sizeof(double) * P);
    h2d(ctx, c.w.right, right, sizeof(double) * P);
    h2d(ctx, c.w.down, down, sizeof(double) * P);
    h2d(ctx, c.w.b, b, sizeof(double) * P);
    launch_fusion(ctx, c.a, c.grid);
    int st[4];
    d2h(ctx, st, c.w.ctl, sizeof(int) * 4);
    sync(ctx);
    if (iterations) *iterations = st[3];
    if (st[0]) throw RefError{st[0], "PCG diverged (non-positive diagonal, lost curvature or "
                                     "10 consecutive residual increases)"};
    d2h(ctx, delta, c.w.x, sizeof(double) * P);
    sync(ctx);
  });
}

int dfuse_solve_scale_step(dfuse_ctx* ctx, const dfuse_fusion_inputs* in, const double* log_depth,
                           double scale, const dfuse_robust_cfg* cfg, double* scale_out) {
  return guarded(ctx, [&] {
    require(scale_out != nullptr, DFUSE_E_INVALID_ARGUMENT, "null pointer");
    check_inputs(in, DFUSE_MODE_FULL);
    require(in->inlier_count > 0, DFUSE_E_NO_SEMIDENSE_SUPPORT, "no valid semi-dense pixels");
    const long P = (long)in->width * in->height;
    check_deltas(cfg, DFUSE_MODE_FULL, in->width, in->height, any_valid(in->semi_valid, P),
                 false);
    FusionCall c = prepare(ctx, in, log_depth, scale, cfg, DFUSE_MODE_FULL, OP_SCALE, false);
    launch_fusion(ctx, c.a, c.grid);
    d2h(ctx, scale_out, &c.w.ctl->value[0], sizeof(double));
    sync(ctx);
  });
}

int dfuse_optimize(dfuse_ctx* ctx, const dfuse_fusion_inputs* in, double* log_depth,
                   double* scale, int32_t* iteration, const dfuse_robust_cfg* cfg, int mode,
                   dfuse_solver_stats* stats) {
  return guarded(ctx, [&] {
    require(scale && iteration, DFUSE_E_INVALID_ARGUMENT, "null pointer");
    check_inputs(in, mode);
    require(cfg != nullptr, DFUSE_E_INVALID_ARGUMENT, "null pointer");
    const long P = (long)in->width * in->height;
    if (cfg->gn_iterations > 0) {
      const bool ls = mode == DFUSE_MODE_LSSCALE;
      const bool semi = any_valid(in->semi_valid, P);
      const bool scale_block = !ls && cfg->estimate_scale && in->inlier_count > 0;
      const bool depth_block = !ls || in->inlier_count > 0;
      check_deltas(cfg, mode, in->width, in->height, semi && (scale_block || depth_block),
                   depth_block);
    }
    FusionCall c = prepare(ctx, in, log_depth, *scale, cfg, mode, OP_OPTIMIZE, true);
    FusionStateDev st{*scale, *iteration, 0};
    h2d(ctx, c.w.st, &st, sizeof st);
    launch_fusion(ctx, c.a, c.grid);
    FusionControl* hc = (FusionControl*)malloc(sizeof(FusionControl));
    if (!hc) throw std::bad_alloc();
    d2h(ctx, hc, c.w.ctl, sizeof(FusionControl));
    sync(ctx);
    const int status = hc->status;
    if (stats) *stats = hc->stats;
    if (status) {
      free(hc);
      throw RefError{status, "optimize: PCG diverged; state unchanged"};
    }
    d2h(ctx, log_depth, c.w.ld[hc->ld_final], sizeof(double) * P);
    *scale = hc->scale;
    *iteration = hc->iteration;
    free(hc);
    sync(ctx);
  });
}

}  // extern "C"
