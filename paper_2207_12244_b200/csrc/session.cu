// session.cu -- device-resident keyframe session (pipeline.hpp:125-228).
//
// A dfuse_keyframe owns everything make_keyframe builds (I0, texture mask,
// predictions, empty semi-dense map, init_state) in HBM. process_frame for a
// tracked frame is then two kernels -- k_stereo (scan + in-place semi-dense
// update) and k_fusion (the whole optimize()) -- with no host round trip
// between them: the inlier count and the fusion state scalars (scale,
// iteration, live log-depth buffer) stay on the device. One small
// device->host copy per frame returns the ProcessOutcome-like result.
#include <string.h>

#include <new>

#include "common.cuh"
#include "fusion.cuh"
#include "stereo.cuh"

using namespace dfuse_cuda;

struct dfuse_keyframe {
  dfuse_ctx* ctx = nullptr;
  int W = 0, H = 0;
  long P = 0;
  int n_mask = 0;
  int stereo_frames = 0;
  int parity = 0;
  int grid = 0;
  void* block = nullptr;  // one device allocation for everything below
  float* I0 = nullptr;
  float* I1 = nullptr;
  uint8_t* mask = nullptr;
  int* list = nullptr;
  double* semi_d = nullptr;
  double* semi_v = nullptr;
  uint8_t* semi_valid = nullptr;
  int* counters = nullptr;  // [0] work [1] n_list [2] n_obs [3] unused [4] inlier_count
  FusionArgs fa;
  FusionStateDev* st = nullptr;  // [2] ping-pong
  FusionControl* h_ctl = nullptr;  // pinned
  int* h_counters = nullptr;       // pinned
};

namespace {

template <class F>
int kf_guarded(dfuse_keyframe* kf, F&& f) {
  if (!kf || !kf->ctx) return DFUSE_E_INVALID_ARGUMENT;
  dfuse_ctx* ctx = kf->ctx;
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
  }
}

size_t al(size_t v) { return (v + 255) & ~size_t(255); }

void reset_state(dfuse_keyframe* kf) {
  dfuse_ctx* ctx = kf->ctx;
  const long P = kf->P;
  // SemiDenseMap::empty (semidense.hpp:27-30), init_state (fusion.hpp:44-46)
  DF_CUDA(cudaMemsetAsync(kf->semi_d, 0, sizeof(double) * P, ctx->stream));
  DF_CUDA(cudaMemsetAsync(kf->semi_v, 0, sizeof(double) * P, ctx->stream));
  DF_CUDA(cudaMemsetAsync(kf->semi_valid, 0, P, ctx->stream));
  DF_CUDA(cudaMemsetAsync(kf->counters + 4, 0, sizeof(int), ctx->stream));
  DF_CUDA(cudaMemcpyAsync(kf->fa.ld[0], kf->fa.pred[0], sizeof(double) * P,
                          cudaMemcpyDeviceToDevice, ctx->stream));
  FusionStateDev s0{1.0, 0, 0};
  kf->parity = 0;
  DF_CUDA(cudaMemcpyAsync(kf->st, &s0, sizeof s0, cudaMemcpyHostToDevice, ctx->stream));
  DF_CUDA(cudaStreamSynchronize(ctx->stream));
  kf->stereo_frames = 0;
}

void process(dfuse_keyframe* kf, const dfuse_epigeom* g, const float* I1_dev,
             const dfuse_search_cfg* scfg, const dfuse_robust_cfg* rcfg, int mode,
             dfuse_frame_result* res) {
  dfuse_ctx* ctx = kf->ctx;
  if (!g || !scfg || !rcfg || !res) throw RefError{DFUSE_E_INVALID_ARGUMENT, "null pointer"};
  if (g->K.width != kf->W || g->K.height != kf->H)
    throw RefError{DFUSE_E_DIMENSION_MISMATCH, "frame does not match the keyframe raster"};
  if (mode < 0 || mode > 2) throw RefError{DFUSE_E_INVALID_ARGUMENT, "unknown fusion mode"};
  if (rcfg->gn_iterations > 0) {
    const bool ls = mode == DFUSE_MODE_LSSCALE;
    if (rcfg->delta_semi <= 0.0 || (!ls && rcfg->delta_net <= 0.0) ||
        (mode != DFUSE_MODE_NOPAIRWISE && rcfg->delta_grad <= 0.0))
      throw RefError{DFUSE_E_INVALID_ARGUMENT, "huber delta must be > 0"};
  }
  // ---- stereo stage: stereo_scan + update_semidense, pipeline.hpp:205-213
  DF_CUDA(cudaEventRecord(ctx->ev[0], ctx->stream));
  DF_CUDA(cudaMemsetAsync(kf->counters, 0, sizeof(int), ctx->stream));
  DF_CUDA(cudaMemsetAsync(kf->counters + 2, 0, sizeof(int), ctx->stream));
  StereoArgs a;
  memset(&a, 0, sizeof a);
  a.g = *g;
  a.cfg = *scfg;
  a.I0 = kf->I0;
  a.I1 = I1_dev;
  a.n_items = kf->n_mask;
  a.work_counter = kf->counters;
  a.list = kf->list;
  a.depth = kf->semi_d;
  a.variance = kf->semi_v;
  a.valid = kf->semi_valid;
  a.n_obs = kf->counters + 2;
  a.n_installed = kf->counters + 4;  // inlier_count += newly installed pixels
  if (kf->n_mask > 0) launch_stereo(ctx, a, false);
  DF_CUDA(cudaEventRecord(ctx->ev[1], ctx->stream));
  // ---- optimise stage, pipeline.hpp:223-226
  FusionArgs& f = kf->fa;
  f.dsemi = rcfg->delta_semi;
  f.dnet = rcfg->delta_net;
  f.dgrad = rcfg->delta_grad;
  f.cg_tol = rcfg->cg_tol;
  f.gn = rcfg->gn_iterations;
  f.cg_max = rcfg->cg_max_iters;
  f.est_scale = rcfg->estimate_scale;
  f.mode = mode;
  f.op = OP_OPTIMIZE;
  f.st_in = kf->st + kf->parity;
  f.st_out = kf->st + (1 - kf->parity);
  launch_fusion(ctx, f, kf->grid);
  DF_CUDA(cudaEventRecord(ctx->ev[2], ctx->stream));
  DF_CUDA(cudaMemcpyAsync(kf->h_counters, kf->counters, 8 * sizeof(int), cudaMemcpyDeviceToHost,
                          ctx->stream));
  DF_CUDA(cudaMemcpyAsync(kf->h_ctl, f.ctl, sizeof(FusionControl), cudaMemcpyDeviceToHost,
                          ctx->stream));
  DF_CUDA(cudaStreamSynchronize(ctx->stream));
  kf->parity = 1 - kf->parity;
  const int n_obs = kf->h_counters[2];
  if (n_obs > 0) kf->stereo_frames += 1;  // pipeline.hpp:211
  res->observations = n_obs;
  res->inlier_count = kf->h_counters[4];
  res->stereo_frames = kf->stereo_frames;
  res->optimize_status = kf->h_ctl->status;  // CgDivergence: solve skipped, pipeline.hpp:328-331
  DF_CUDA(cudaEventElapsedTime(&res->stereo_ms, ctx->ev[0], ctx->ev[1]));
  DF_CUDA(cudaEventElapsedTime(&res->optimise_ms, ctx->ev[1], ctx->ev[2]));
  res->stats = kf->h_ctl->stats;
}

}  // namespace

extern "C" {

int dfuse_kf_create(dfuse_ctx* ctx, const dfuse_intrinsics* K, const float* I0,
                    const double* const pred[6], double texture_threshold, dfuse_keyframe** out) {
  if (!ctx || !out) return DFUSE_E_INVALID_ARGUMENT;
  *out = nullptr;
  dfuse_keyframe* kf = new (std::nothrow) dfuse_keyframe();
  if (!kf) return DFUSE_E_CUDA;
  kf->ctx = ctx;
  const int rc = kf_guarded(kf, [&] {
    if (!K || !I0 || !pred) throw RefError{DFUSE_E_INVALID_ARGUMENT, "null pointer"};
    for (int c = 0; c < 6; ++c)
      if (!pred[c]) throw RefError{DFUSE_E_INVALID_ARGUMENT, "null prediction plane"};
    if (K->width <= 0 || K->height <= 0)
      throw RefError{DFUSE_E_INVALID_ARGUMENT, "raster dimensions must be positive"};
    if (texture_threshold <= 0.0)
      throw RefError{DFUSE_E_INVALID_ARGUMENT, "texture threshold must be > 0"};
    kf->W = K->width;
    kf->H = K->height;
    const long P = kf->P = (long)kf->W * kf->H;
    kf->grid = fusion_grid(ctx);
    const size_t dP = al(sizeof(double) * P);
    const bool resident = fusion_resident_possible(P, kf->grid);
    const size_t total = 2 * al(sizeof(float) * P) + al(P) + al(sizeof(int) * P) + 2 * dP +
                         al(P) + 256 + 11 * dP + 11 * dP + al(fusion_slots_bytes(kf->grid)) +
                         al(sizeof(FusionControl)) + al(2 * sizeof(FusionStateDev)) +
                         (resident ? al(fusion_halo_bytes(P)) : 0);
    DF_CUDA(cudaMalloc(&kf->block, total));
    char* p = (char*)kf->block;
    auto take = [&](size_t bytes) {
      char* r = p;
      p += al(bytes);
      return (void*)r;
    };
    kf->I0 = (float*)take(sizeof(float) * P);
    kf->I1 = (float*)take(sizeof(float) * P);
    kf->mask = (uint8_t*)take(P);
    kf->list = (int*)take(sizeof(int) * P);
    kf->semi_d = (double*)take(dP);
    kf->semi_v = (double*)take(dP);
    kf->semi_valid = (uint8_t*)take(P);
    kf->counters = (int*)take(256);
    FusionArgs& f = kf->fa;
    memset(&f, 0, sizeof f);
    f.W = kf->W;
    f.H = kf->H;
    for (int c = 0; c < 6; ++c) f.pred[c] = (double*)take(dP);
    f.sd = kf->semi_d;
    f.sv = kf->semi_v;
    f.svalid = kf->semi_valid;
    f.lnsd = (double*)take(dP);
    f.irs = (double*)take(dP);
    for (int k = 0; k < 3; ++k) f.ivar[k] = (double*)take(dP);
    f.inlier_dev = kf->counters + 4;
    f.ld[0] = (double*)take(dP);
    f.ld[1] = (double*)take(dP);
    f.diag = (double*)take(dP);
    f.right = (double*)take(dP);
    f.down = (double*)take(dP);
    f.b = (double*)take(dP);
    f.x = (double*)take(dP);
    f.r = (double*)take(dP);
    f.p[0] = (double*)take(dP);
    f.p[1] = (double*)take(dP);
    f.q = (double*)take(dP);
    f.slots = (ReduceSlot*)take(fusion_slots_bytes(kf->grid));
    f.halo = resident ? (unsigned long long*)take(fusion_halo_bytes(P)) : nullptr;
    f.ctl = (FusionControl*)take(sizeof(FusionControl));
    kf->st = (FusionStateDev*)take(2 * sizeof(FusionStateDev));
    DF_CUDA(cudaMallocHost(&kf->h_ctl, sizeof(FusionControl)));
    DF_CUDA(cudaMallocHost(&kf->h_counters, 8 * sizeof(int)));
    DF_CUDA(cudaMemsetAsync(kf->counters, 0, 256, ctx->stream));
    DF_CUDA(cudaMemcpyAsync(kf->I0, I0, sizeof(float) * P, cudaMemcpyHostToDevice, ctx->stream));
    for (int c = 0; c < 6; ++c)
      DF_CUDA(cudaMemcpyAsync((void*)f.pred[c], pred[c], sizeof(double) * P,
                              cudaMemcpyHostToDevice, ctx->stream));
    // make_keyframe: texture_mask (pipeline.hpp:148) + the masked-pixel list
    launch_texture_mask(ctx, kf->I0, kf->W, kf->H, texture_threshold, kf->mask);
    launch_mask_list(ctx, kf->mask, P, kf->list, kf->counters + 1);
    DF_CUDA(cudaMemcpyAsync(&kf->n_mask, kf->counters + 1, sizeof(int), cudaMemcpyDeviceToHost,
                            ctx->stream));
    reset_state(kf);  // synchronises
  });
  if (rc) {
    dfuse_kf_destroy(kf);
    return rc;
  }
  *out = kf;
  return DFUSE_OK;
}

int dfuse_kf_destroy(dfuse_keyframe* kf) {
  if (!kf) return DFUSE_OK;
  if (kf->ctx) {
    cudaSetDevice(kf->ctx->device);
    cudaStreamSynchronize(kf->ctx->stream);
  }
  if (kf->block) cudaFree(kf->block);
  if (kf->h_ctl) cudaFreeHost(kf->h_ctl);
  if (kf->h_counters) cudaFreeHost(kf->h_counters);
  delete kf;
  return DFUSE_OK;
}

int dfuse_kf_reset(dfuse_keyframe* kf) {
  return kf_guarded(kf, [&] { reset_state(kf); });
}

int dfuse_kf_process_frame(dfuse_keyframe* kf, const dfuse_epigeom* g, const float* I1,
                           const dfuse_search_cfg* scfg, const dfuse_robust_cfg* rcfg, int mode,
                           dfuse_frame_result* res) {
  return kf_guarded(kf, [&] {
    if (!I1) throw RefError{DFUSE_E_INVALID_ARGUMENT, "null image"};
    DF_CUDA(cudaMemcpyAsync(kf->I1, I1, sizeof(float) * kf->P, cudaMemcpyHostToDevice,
                            kf->ctx->stream));
    process(kf, g, kf->I1, scfg, rcfg, mode, res);
  });
}

int dfuse_kf_process_frame_dev(dfuse_keyframe* kf, const dfuse_epigeom* g, const float* I1_dev,
                               const dfuse_search_cfg* scfg, const dfuse_robust_cfg* rcfg,
                               int mode, dfuse_frame_result* res) {
  return kf_guarded(kf, [&] {
    if (!I1_dev) throw RefError{DFUSE_E_INVALID_ARGUMENT, "null image"};
    process(kf, g, I1_dev, scfg, rcfg, mode, res);
  });
}

int dfuse_kf_download(dfuse_keyframe* kf, double* log_depth, double* scale, int32_t* iteration,
                      double* semi_depth, double* semi_variance, uint8_t* semi_valid,
                      int32_t* inlier_count, uint8_t* mask) {
  return kf_guarded(kf, [&] {
    dfuse_ctx* ctx = kf->ctx;
    FusionStateDev st;
    DF_CUDA(cudaMemcpyAsync(&st, kf->st + kf->parity, sizeof st, cudaMemcpyDeviceToHost,
                            ctx->stream));
    DF_CUDA(cudaStreamSynchronize(ctx->stream));
    const long P = kf->P;
    auto cp = [&](void* dst, const void* src, size_t bytes) {
      if (dst) DF_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    };
    cp(log_depth, kf->fa.ld[st.cur], sizeof(double) * P);
    cp(semi_depth, kf->semi_d, sizeof(double) * P);
    cp(semi_variance, kf->semi_v, sizeof(double) * P);
    cp(semi_valid, kf->semi_valid, P);
    cp(inlier_count, kf->counters + 4, sizeof(int));
    cp(mask, kf->mask, P);
    DF_CUDA(cudaStreamSynchronize(ctx->stream));
    if (scale) *scale = st.scale;
    if (iteration) *iteration = st.iteration;
  });
}

}  // extern "C"
