// session.cu -- device-resident keyframe session (pipeline.hpp:125-228).
//
// A dfuse_keyframe owns everything make_keyframe builds (I0, texture mask,
// predictions, empty semi-dense map, init_state) in HBM. process_frame for a
// tracked frame is then two kernels -- k_stereo (scan + in-place semi-dense
// update) and k_fusion (the whole optimize()) -- with no host round trip
// between them: the inlier count and the fusion state scalars (scale,
// iteration, live log-depth buffer) stay on the device. One small
// device->host copy per frame returns the ProcessOutcome-like result.
#include <math.h>
#include <string.h>

#include <cub/device/device_radix_sort.cuh>
#include <new>
#include <string>

#include "common.cuh"
#include "eval.cuh"
#include "fusion.cuh"
#include "stereo.cuh"

using namespace dfuse_cuda;

struct dfuse_keyframe {
  dfuse_ctx* ctx = nullptr;
  int W = 0, H = 0;
  long P = 0;
  int n_mask = 0;
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
  // [0] stereo work counter, [1] n_obs, [2..3] epipolar steps (64-bit): per
  // frame, cleared by one memset; [4] inlier_count, [5] stereo_frames: per
  // keyframe. ([1] holds the masked-pixel count while the keyframe is made.)
  int* counters = nullptr;
  FusionArgs fa;
  FusionStateDev* st = nullptr;  // [2] ping-pong
  FusionControl* h_ctl = nullptr;  // pinned
  int* h_counters = nullptr;       // pinned
  double median_depth = -1.0;      // cached median_predicted_depth (< 0: not computed)
  bool pending = false;            // a frame was enqueued and not yet collected
  FusionStateDev* h_s0 = nullptr;  // pinned: init_state's scalars for reset
  // host-buffer pipeline (dfuse_kf_process_frame_host_async), made on first
  // use: two frame slots and two result slots, a copy-in and a copy-out
  // stream (so that frame n+1's copy-in never queues behind frame n's
  // copy-out), and events ordering slot reuse between the streams
  struct HostPipe {
    float* img[2] = {};
    double* out[2] = {};
    cudaStream_t copy = nullptr, copy_out = nullptr;
    cudaEvent_t in[2] = {}, read[2] = {}, staged[2] = {}, done[2] = {};
    long n = 0;
  } hp;
  bool hp_used = false;
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

// slot and halo words of the all-reduces and the LL counters, cleared once:
// the session's launches then continue the flags (FusionArgs::persist_sync)
void clear_sync(dfuse_keyframe* kf) {
  dfuse_ctx* ctx = kf->ctx;
  FusionArgs& f = kf->fa;
  DF_CUDA(cudaMemsetAsync(f.slots, 0, fusion_slots_bytes(kf->grid), ctx->stream));
  if (f.halo) DF_CUDA(cudaMemsetAsync(f.halo, 0, fusion_halo_bytes(kf->P), ctx->stream));
  DF_CUDA(cudaMemsetAsync(f.ctl, 0, sizeof(FusionControl), ctx->stream));
  f.persist_sync = 1;
}

void reset_state(dfuse_keyframe* kf) {
  dfuse_ctx* ctx = kf->ctx;
  const long P = kf->P;
  // SemiDenseMap::empty (semidense.hpp:27-30), init_state (fusion.hpp:44-46)
  DF_CUDA(cudaMemsetAsync(kf->semi_d, 0, sizeof(double) * P, ctx->stream));
  DF_CUDA(cudaMemsetAsync(kf->semi_v, 0, sizeof(double) * P, ctx->stream));
  DF_CUDA(cudaMemsetAsync(kf->semi_valid, 0, P, ctx->stream));
  DF_CUDA(cudaMemsetAsync(kf->counters + 4, 0, 2 * sizeof(int), ctx->stream));
  DF_CUDA(cudaMemcpyAsync(kf->fa.ld[0], kf->fa.pred[0], sizeof(double) * P,
                          cudaMemcpyDeviceToDevice, ctx->stream));
  kf->parity = 0;
  DF_CUDA(cudaMemcpyAsync(kf->st, kf->h_s0, sizeof(FusionStateDev), cudaMemcpyHostToDevice,
                          ctx->stream));
}

// the fused log-depth (ld[st->cur]) into a staging slot, on the device:
// the host does not know cur without a synchronisation
__global__ void k_copy_state_ld(const FusionStateDev* __restrict__ st,
                                const double* __restrict__ ld0, const double* __restrict__ ld1,
                                double* __restrict__ out, long P) {
  const double* src = st->cur ? ld1 : ld0;
  const long n2 = P / 2;  // 16-byte vectors (the buffers are 256-byte aligned), odd tail below
  const double2* s2 = reinterpret_cast<const double2*>(src);
  double2* o2 = reinterpret_cast<double2*>(out);
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n2;
       i += (long)gridDim.x * blockDim.x)
    o2[i] = s2[i];
  if ((P & 1) && blockIdx.x == 0 && threadIdx.x == 0) out[P - 1] = src[P - 1];
}

void host_pipe_init(dfuse_keyframe* kf) {
  auto& h = kf->hp;
  if (h.copy) return;
  const size_t P = (size_t)kf->P;
  for (int b = 0; b < 2; ++b) {
    DF_CUDA(cudaMalloc(&h.img[b], sizeof(float) * P));
    DF_CUDA(cudaMalloc(&h.out[b], sizeof(double) * P));
    for (cudaEvent_t* e : {&h.in[b], &h.read[b], &h.staged[b], &h.done[b]})
      DF_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  }
  DF_CUDA(cudaStreamCreateWithFlags(&h.copy, cudaStreamNonBlocking));
  DF_CUDA(cudaStreamCreateWithFlags(&h.copy_out, cudaStreamNonBlocking));
}

void host_pipe_free(dfuse_keyframe* kf) {
  auto& h = kf->hp;
  if (!h.copy) return;
  cudaStreamSynchronize(h.copy);
  cudaStreamSynchronize(h.copy_out);
  for (int b = 0; b < 2; ++b) {
    cudaFree(h.img[b]);
    cudaFree(h.out[b]);
    for (cudaEvent_t e : {h.in[b], h.read[b], h.staged[b], h.done[b]}) cudaEventDestroy(e);
  }
  cudaStreamDestroy(h.copy);
  cudaStreamDestroy(h.copy_out);
  h = dfuse_keyframe::HostPipe{};
}

// process_frame, enqueued on the context's stream (no host synchronisation):
// the result lands in pinned host memory, read by collect()
void enqueue(dfuse_keyframe* kf, const dfuse_epigeom* g, const float* I1_dev,
             const dfuse_search_cfg* scfg, const dfuse_robust_cfg* rcfg, int mode) {
  dfuse_ctx* ctx = kf->ctx;
  if (!g || !scfg || !rcfg) throw RefError{DFUSE_E_INVALID_ARGUMENT, "null pointer"};
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
  DF_CUDA(cudaMemsetAsync(kf->counters, 0, 4 * sizeof(int), ctx->stream));
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
  a.n_obs = kf->counters + 1;
  a.n_installed = kf->counters + 4;  // inlier_count += newly installed pixels
  a.step_count = reinterpret_cast<unsigned long long*>(kf->counters + 2);
  if (kf->n_mask > 0) launch_stereo(ctx, a, false, true);  // counters[0] cleared above
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
  kf->parity = 1 - kf->parity;
  kf->pending = true;
}

// wait for the frames enqueued so far; res = the last one's outcome
void collect(dfuse_keyframe* kf, dfuse_frame_result* res) {
  dfuse_ctx* ctx = kf->ctx;
  if (!res) throw RefError{DFUSE_E_INVALID_ARGUMENT, "null pointer"};
  if (!kf->pending) throw RefError{DFUSE_E_INVALID_ARGUMENT, "no frame enqueued"};
  // the last frame's counters and control block (nothing after it on the
  // stream touches them)
  DF_CUDA(cudaMemcpyAsync(kf->h_counters, kf->counters, 8 * sizeof(int), cudaMemcpyDeviceToHost,
                          ctx->stream));
  DF_CUDA(cudaMemcpyAsync(kf->h_ctl, kf->fa.ctl, sizeof(FusionControl), cudaMemcpyDeviceToHost,
                          ctx->stream));
  DF_CUDA(cudaStreamSynchronize(ctx->stream));
  if (kf->hp.copy_out) DF_CUDA(cudaStreamSynchronize(kf->hp.copy_out));  // the results' copies
  kf->pending = false;
  if (kf->h_ctl->sync_phase > (1u << 30) || kf->h_ctl->sync_ll > (1u << 30))
    clear_sync(kf);  // 32-bit LL flags: start over long before they wrap
  res->observations = kf->h_counters[1];
  res->inlier_count = kf->h_counters[4];
  res->stereo_frames = kf->h_counters[5];  // counted on the device, pipeline.hpp:211
  long long steps;
  memcpy(&steps, kf->h_counters + 2, sizeof steps);
  res->epipolar_steps = steps;
  res->optimize_status = kf->h_ctl->status;  // CgDivergence: solve skipped, pipeline.hpp:328-331
  DF_CUDA(cudaEventElapsedTime(&res->stereo_ms, ctx->ev[0], ctx->ev[1]));
  DF_CUDA(cudaEventElapsedTime(&res->optimise_ms, ctx->ev[1], ctx->ev[2]));
  res->stats = kf->h_ctl->stats;
  res->solver_ppt = kf->fa.ppt;  // set by launch_fusion's tile planner
  res->reserved = 0;
}

// the session's one device allocation (make_keyframe's Keyframe, the
// fusion workspace and its control blocks)
void kf_alloc(dfuse_keyframe* kf, const dfuse_intrinsics* K) {
  dfuse_ctx* ctx = kf->ctx;
  kf->W = K->width;
  kf->H = K->height;
  const long P = kf->P = (long)kf->W * kf->H;
  kf->grid = fusion_grid(ctx);
  const size_t dP = al(sizeof(double) * P);
  const bool resident = fusion_resident_possible(P, kf->grid);
  const size_t fP = al(sizeof(float) * P);
  const size_t total = 2 * fP + al(P) + al(sizeof(int) * P) + 2 * dP + al(P) + 256 + 11 * dP +
                       5 * fP + 12 * dP + al(fusion_slots_bytes(kf->grid)) +
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
  for (int c = 1; c < 6; ++c) f.predf[c] = (float*)take(sizeof(float) * P);
  f.pred_f32_ok = 0;
  f.sd = kf->semi_d;
  f.sv = kf->semi_v;
  f.svalid = kf->semi_valid;
  f.lnsd = (double*)take(dP);
  f.irs = (double*)take(dP);
  for (int k = 0; k < 3; ++k) f.ivar[k] = (double*)take(dP);
  f.inlier_dev = kf->counters + 4;
  f.session_counters = kf->counters;
  f.ld[0] = (double*)take(dP);
  f.ld[1] = (double*)take(dP);
  f.diag = (double*)take(dP);
  f.right = (double*)take(dP);
  f.down = (double*)take(dP);
  f.b = (double*)take(dP);
  f.x = (double*)take(dP);
  f.r = (double*)take(dP);
  f.z = (double*)take(dP);
  f.p[0] = (double*)take(dP);
  f.p[1] = (double*)take(dP);
  f.q = (double*)take(dP);
  f.slots = (ReduceSlot*)take(fusion_slots_bytes(kf->grid));
  f.halo = resident ? (unsigned long long*)take(fusion_halo_bytes(P)) : nullptr;
  f.ctl = (FusionControl*)take(sizeof(FusionControl));
  kf->st = (FusionStateDev*)take(2 * sizeof(FusionStateDev));
  DF_CUDA(cudaMallocHost(&kf->h_ctl, sizeof(FusionControl)));
  DF_CUDA(cudaMallocHost(&kf->h_counters, 8 * sizeof(int)));
  DF_CUDA(cudaMallocHost(&kf->h_s0, sizeof(FusionStateDev)));
  *kf->h_s0 = FusionStateDev{1.0, 0, 0};  // init_state, fusion.hpp:44-46
  DF_CUDA(cudaMemsetAsync(kf->counters, 0, 256, ctx->stream));
}

// upload I0, texture mask (pipeline.hpp:148) + the masked-pixel list, empty
// semi-dense map and init_state (pipeline.hpp:149-150)
void kf_finish(dfuse_keyframe* kf, const float* I0, double texture_threshold) {
  dfuse_ctx* ctx = kf->ctx;
  const long P = kf->P;
  // prediction planes 1..5 as float32 when every value is float-exact (the
  // reference keeps them at float precision: predictions.hpp:16-17)
  int* inexact = kf->counters + 6;
  DF_CUDA(cudaMemsetAsync(inexact, 0, sizeof(int), ctx->stream));
  launch_pred_narrow(ctx, kf->fa.pred, const_cast<float* const*>(kf->fa.predf), P, inexact);
  int h_inexact = 0;
  DF_CUDA(cudaMemcpyAsync(&h_inexact, inexact, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  DF_CUDA(cudaMemcpyAsync(kf->I0, I0, sizeof(float) * P, cudaMemcpyHostToDevice, ctx->stream));
  launch_texture_mask(ctx, kf->I0, kf->W, kf->H, texture_threshold, kf->mask);
  launch_mask_list(ctx, kf->mask, P, kf->list, kf->counters + 1);
  DF_CUDA(cudaMemcpyAsync(&kf->n_mask, kf->counters + 1, sizeof(int), cudaMemcpyDeviceToHost,
                          ctx->stream));
  clear_sync(kf);
  reset_state(kf);
  DF_CUDA(cudaStreamSynchronize(ctx->stream));
  kf->fa.pred_f32_ok = (h_inexact == 0 && ctx->pred_fp32) ? 1 : 0;
}

void check_kf_args(const dfuse_intrinsics* K, const float* I0, double texture_threshold) {
  if (!K || !I0) throw RefError{DFUSE_E_INVALID_ARGUMENT, "null pointer"};
  if (K->width <= 0 || K->height <= 0)
    throw RefError{DFUSE_E_INVALID_ARGUMENT, "raster dimensions must be positive"};
  if (texture_threshold <= 0.0)
    throw RefError{DFUSE_E_INVALID_ARGUMENT, "texture threshold must be > 0"};
}

// ---- DFPRED ingest (predictions.hpp:31-123) and focal_adjust (148-157) ----
constexpr size_t kDfpredHeader = 24;
const char* const kDfpredChannel[6] = {"log_depth",  "log_depth_var", "grad_x",
                                       "grad_x_var", "grad_y",        "grad_y_var"};

uint32_t rd_u32_le(const unsigned char* p) {
  return (uint32_t)p[0] | (uint32_t)p[1] << 8 | (uint32_t)p[2] << 16 | (uint32_t)p[3] << 24;
}

struct DfpredHeader {
  int w, h;
  double source_focal;
};

// load_predictions' header checks, same order, codes and byte offsets
// (predictions.hpp:72-95)
DfpredHeader parse_dfpred_header(const unsigned char* b, size_t nbytes) {
  if (!b) throw RefError{DFUSE_E_INVALID_ARGUMENT, "null buffer"};
  if (nbytes < kDfpredHeader)
    throw RefError{DFUSE_E_TRUNCATED_FILE, "dfpred: header, read " + std::to_string(nbytes) +
                                               " of 24 bytes"};
  if (memcmp(b, "DFPR", 4) != 0) throw RefError{DFUSE_E_BAD_MAGIC, "dfpred: bad magic at byte 0"};
  const uint32_t version = rd_u32_le(b + 4);
  if (version != 1)
    throw RefError{DFUSE_E_BAD_MAGIC,
                   "dfpred: unsupported version " + std::to_string(version) + " at byte 4"};
  const uint32_t width = rd_u32_le(b + 8), height = rd_u32_le(b + 12);
  const uint32_t channels = rd_u32_le(b + 16), focal_milli = rd_u32_le(b + 20);
  if (width == 0 || height == 0 || width > 65536 || height > 65536)
    throw RefError{DFUSE_E_DIMENSION_MISMATCH, "dfpred: " + std::to_string(width) + "x" +
                                                   std::to_string(height) + " at byte 8"};
  if (channels != 6)
    throw RefError{DFUSE_E_DIMENSION_MISMATCH,
                   "dfpred: channel_count " + std::to_string(channels) + " at byte 16"};
  if (focal_milli == 0)
    throw RefError{DFUSE_E_NON_POSITIVE_FOCAL, "dfpred: source_focal at byte 20"};
  return DfpredHeader{(int)width, (int)height, (double)focal_milli / 1000.0};
}

// Widen the six fp32 planes to the session's fp64 planes, validate every
// variance (v > 0 and finite, predictions.hpp:112-118; the first failure in
// file order wins, as the reference reads channel by channel) and add the
// focal_adjust shift to log_depth (predictions.hpp:154-155). One thread per
// (pixel, channel pair), float4-wide reads of the raw planes.
__global__ void k_dfpred_ingest(const float* __restrict__ raw, long P, double shift, int do_shift,
                                double* const* __restrict__ planes,
                                unsigned long long* first_bad) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < P;
       i += (long)gridDim.x * blockDim.x) {
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      double v = (double)raw[(long)c * P + i];
      if (c & 1) {
        if (!(v > 0.0 && isfinite(v))) atomicMin(first_bad, (unsigned long long)c * P + i);
      } else if (c == 0 && do_shift) {
        v += shift;
      }
      planes[c][i] = v;
    }
  }
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
    check_kf_args(K, I0, texture_threshold);
    if (!pred) throw RefError{DFUSE_E_INVALID_ARGUMENT, "null pointer"};
    for (int c = 0; c < 6; ++c)
      if (!pred[c]) throw RefError{DFUSE_E_INVALID_ARGUMENT, "null prediction plane"};
    kf_alloc(kf, K);
    for (int c = 0; c < 6; ++c)
      DF_CUDA(cudaMemcpyAsync((void*)kf->fa.pred[c], pred[c], sizeof(double) * kf->P,
                              cudaMemcpyHostToDevice, ctx->stream));
    kf_finish(kf, I0, texture_threshold);
  });
  if (rc) {
    dfuse_kf_destroy(kf);
    return rc;
  }
  *out = kf;
  return DFUSE_OK;
}

int dfuse_dfpred_header(dfuse_ctx* ctx, const void* bytes, size_t nbytes, int32_t* width,
                        int32_t* height, double* source_focal) {
  try {
    const DfpredHeader h = parse_dfpred_header((const unsigned char*)bytes, nbytes);
    if (width) *width = h.w;
    if (height) *height = h.h;
    if (source_focal) *source_focal = h.source_focal;
    if (ctx) ctx->last_error.clear();
    return DFUSE_OK;
  } catch (const RefError& e) {
    if (ctx) ctx->last_error = e.msg;
    return e.code;
  }
}

int dfuse_kf_create_dfpred(dfuse_ctx* ctx, const dfuse_intrinsics* K, const float* I0,
                           const void* dfpred, size_t nbytes, double texture_threshold,
                           dfuse_keyframe** out) {
  if (!ctx || !out) return DFUSE_E_INVALID_ARGUMENT;
  *out = nullptr;
  dfuse_keyframe* kf = new (std::nothrow) dfuse_keyframe();
  if (!kf) return DFUSE_E_CUDA;
  kf->ctx = ctx;
  const int rc = kf_guarded(kf, [&] {
    check_kf_args(K, I0, texture_threshold);
    const unsigned char* b = (const unsigned char*)dfpred;
    const DfpredHeader h = parse_dfpred_header(b, nbytes);  // predictions.hpp:72-95
    const long P = (long)h.w * h.h;
    const size_t need = kDfpredHeader + 24 * (size_t)P;
    if (nbytes < need) {  // predictions.hpp:103-108: the first short channel
      const size_t c = (nbytes - kDfpredHeader) / (4 * (size_t)P);
      throw RefError{DFUSE_E_TRUNCATED_FILE, std::string("dfpred: channel ") +
                                                 kDfpredChannel[c] + ", at byte " +
                                                 std::to_string(nbytes)};
    }
    if (h.w != K->width || h.h != K->height)  // pipeline.hpp:139-141
      throw RefError{DFUSE_E_DIMENSION_MISMATCH,
                     "dfpred does not match the processing resolution"};
    kf_alloc(kf, K);
    // the six fp32 planes go to HBM as they are (24 B/px) and are widened
    // there; the staging buffer is the fusion workspace's PCG vectors
    float* raw = (float*)kf->fa.x;  // x, r, p0, p1, q: 5 x 8P >= 24P bytes, contiguous
    DF_CUDA(cudaMemcpyAsync(raw, b + kDfpredHeader, 24 * (size_t)P, cudaMemcpyHostToDevice,
                            ctx->stream));
    const double test_focal = K->fx;  // focal_adjust(pred, camera.fx), pipeline.hpp:145
    const bool shift_on = test_focal > 0.0 && test_focal != h.source_focal;
    const double shift = shift_on ? log(test_focal / h.source_focal) : 0.0;
    double** planes = (double**)scratch(ctx, S_TMP3, sizeof(double*) * 6 + 64);
    unsigned long long* bad = (unsigned long long*)(planes + 6);
    double* hp[6];
    for (int c = 0; c < 6; ++c) hp[c] = (double*)kf->fa.pred[c];
    const unsigned long long none = ~0ULL;
    DF_CUDA(cudaMemcpyAsync(planes, hp, sizeof hp, cudaMemcpyHostToDevice, ctx->stream));
    DF_CUDA(cudaMemcpyAsync(bad, &none, sizeof none, cudaMemcpyHostToDevice, ctx->stream));
    long blocks = (P + 255) / 256;
    if (blocks > 8L * ctx->num_sms) blocks = 8L * ctx->num_sms;
    k_dfpred_ingest<<<(int)blocks, 256, 0, ctx->stream>>>(raw, P, shift, shift_on ? 1 : 0,
                                                          planes, bad);
    DF_LAUNCHED(ctx);
    unsigned long long first = 0;
    DF_CUDA(cudaMemcpyAsync(&first, bad, sizeof first, cudaMemcpyDeviceToHost, ctx->stream));
    DF_CUDA(cudaStreamSynchronize(ctx->stream));
    if (first != none) {  // predictions.hpp:113-117
      const size_t c = first / P, i = first % P;
      throw RefError{DFUSE_E_NON_POSITIVE_VARIANCE,
                     std::string("dfpred: ") + kDfpredChannel[c] + "[" + std::to_string(i) +
                         "] at byte " + std::to_string(kDfpredHeader + c * P * 4 + i * 4)};
    }
    if (!(test_focal > 0.0))  // focal_adjust, predictions.hpp:149-150
      throw RefError{DFUSE_E_NON_POSITIVE_FOCAL, "focal_adjust requires positive focal lengths"};
    kf_finish(kf, I0, texture_threshold);
  });
  if (rc) {
    dfuse_kf_destroy(kf);
    return rc;
  }
  *out = kf;
  return DFUSE_OK;
}

// median_predicted_depth (pipeline.hpp:94-99): exp of the element
// nth_element puts at n/2, i.e. the (n/2)-th smallest log-depth -- an exact
// device radix sort of the keys, one element read back, exp on the host
// (the reference's std::exp). Cached per keyframe.
int dfuse_kf_median_depth(dfuse_keyframe* kf, double* out) {
  return kf_guarded(kf, [&] {
    if (!out) throw RefError{DFUSE_E_INVALID_ARGUMENT, "null pointer"};
    if (kf->median_depth < 0.0) {
      dfuse_ctx* ctx = kf->ctx;
      const long P = kf->P;
      // keys in / out: the fusion workspace's r and p0 vectors (idle between frames)
      const double* keys_in = kf->fa.pred[0];
      double* keys_out = kf->fa.r;
      size_t temp = 0;
      DF_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, temp, keys_in, keys_out, (int)P, 0, 64,
                                             ctx->stream));
      void* tmp = scratch(ctx, S_TMP4, temp);
      DF_CUDA(cub::DeviceRadixSort::SortKeys(tmp, temp, keys_in, keys_out, (int)P, 0, 64,
                                             ctx->stream));
      DF_LAUNCHED(ctx);
      double mid = 0.0;
      DF_CUDA(cudaMemcpyAsync(&mid, keys_out + P / 2, sizeof mid, cudaMemcpyDeviceToHost,
                              ctx->stream));
      DF_CUDA(cudaStreamSynchronize(ctx->stream));
      kf->median_depth = exp(mid);
    }
    *out = kf->median_depth;
  });
}

int dfuse_kf_destroy(dfuse_keyframe* kf) {
  if (!kf) return DFUSE_OK;
  if (kf->ctx) {
    cudaSetDevice(kf->ctx->device);
    cudaStreamSynchronize(kf->ctx->stream);
  }
  host_pipe_free(kf);
  if (kf->block) cudaFree(kf->block);
  if (kf->h_ctl) cudaFreeHost(kf->h_ctl);
  if (kf->h_counters) cudaFreeHost(kf->h_counters);
  if (kf->h_s0) cudaFreeHost(kf->h_s0);
  delete kf;
  return DFUSE_OK;
}

int dfuse_kf_reset(dfuse_keyframe* kf) {
  // stream-ordered like everything after it: no need to wait here
  return kf_guarded(kf, [&] { reset_state(kf); });
}

int dfuse_kf_process_frame(dfuse_keyframe* kf, const dfuse_epigeom* g, const float* I1,
                           const dfuse_search_cfg* scfg, const dfuse_robust_cfg* rcfg, int mode,
                           dfuse_frame_result* res) {
  return kf_guarded(kf, [&] {
    if (!I1) throw RefError{DFUSE_E_INVALID_ARGUMENT, "null image"};
    DF_CUDA(cudaMemcpyAsync(kf->I1, I1, sizeof(float) * kf->P, cudaMemcpyHostToDevice,
                            kf->ctx->stream));
    enqueue(kf, g, kf->I1, scfg, rcfg, mode);
    collect(kf, res);
  });
}

int dfuse_kf_process_frame_dev(dfuse_keyframe* kf, const dfuse_epigeom* g, const float* I1_dev,
                               const dfuse_search_cfg* scfg, const dfuse_robust_cfg* rcfg,
                               int mode, dfuse_frame_result* res) {
  return kf_guarded(kf, [&] {
    if (!I1_dev) throw RefError{DFUSE_E_INVALID_ARGUMENT, "null image"};
    enqueue(kf, g, I1_dev, scfg, rcfg, mode);
    collect(kf, res);
  });
}

int dfuse_kf_process_frame_async(dfuse_keyframe* kf, const dfuse_epigeom* g,
                                 const float* I1_dev, const dfuse_search_cfg* scfg,
                                 const dfuse_robust_cfg* rcfg, int mode) {
  return kf_guarded(kf, [&] {
    if (!I1_dev) throw RefError{DFUSE_E_INVALID_ARGUMENT, "null image"};
    enqueue(kf, g, I1_dev, scfg, rcfg, mode);
  });
}

// Host-buffer pipeline: frame n's H2D (copy stream) overlaps frame n-1's
// compute; its fused log-depth is staged on the device after the solve and
// copied out on the copy stream while frame n+1 computes.
int dfuse_kf_process_frame_host_async(dfuse_keyframe* kf, const dfuse_epigeom* g,
                                      const float* I1_host, const dfuse_search_cfg* scfg,
                                      const dfuse_robust_cfg* rcfg, int mode,
                                      double* log_depth_host) {
  return kf_guarded(kf, [&] {
    if (!I1_host) throw RefError{DFUSE_E_INVALID_ARGUMENT, "null image"};
    dfuse_ctx* ctx = kf->ctx;
    host_pipe_init(kf);
    auto& h = kf->hp;
    const int b = (int)(h.n & 1);
    const size_t P = (size_t)kf->P;
    // frame slot b: free once frame n-2 (its last reader) is done
    DF_CUDA(cudaStreamWaitEvent(h.copy, h.read[b], 0));
    DF_CUDA(cudaMemcpyAsync(h.img[b], I1_host, sizeof(float) * P, cudaMemcpyHostToDevice, h.copy));
    DF_CUDA(cudaEventRecord(h.in[b], h.copy));
    DF_CUDA(cudaStreamWaitEvent(ctx->stream, h.in[b], 0));
    enqueue(kf, g, h.img[b], scfg, rcfg, mode);
    DF_CUDA(cudaEventRecord(h.read[b], ctx->stream));
    if (log_depth_host) {
      // result slot b: free once frame n-2's copy-out is done
      DF_CUDA(cudaStreamWaitEvent(ctx->stream, h.done[b], 0));
      k_copy_state_ld<<<ctx->num_sms * 4, 256, 0, ctx->stream>>>(
          kf->st + kf->parity, kf->fa.ld[0], kf->fa.ld[1], h.out[b], (long)P);
      DF_LAUNCHED(ctx);
      DF_CUDA(cudaEventRecord(h.staged[b], ctx->stream));
      DF_CUDA(cudaStreamWaitEvent(h.copy_out, h.staged[b], 0));
      DF_CUDA(cudaMemcpyAsync(log_depth_host, h.out[b], sizeof(double) * P,
                              cudaMemcpyDeviceToHost, h.copy_out));
      DF_CUDA(cudaEventRecord(h.done[b], h.copy_out));
    }
    h.n += 1;
  });
}

int dfuse_kf_last_result(dfuse_keyframe* kf, dfuse_frame_result* res) {
  return kf_guarded(kf, [&] { collect(kf, res); });
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

int dfuse_kf_score(dfuse_keyframe* kf, const double* gt_metres, const uint8_t* gt_valid,
                   dfuse_keyframe_score* out) {
  return kf_guarded(kf, [&] {
    if (!gt_metres || !gt_valid || !out) throw RefError{DFUSE_E_INVALID_ARGUMENT, "null pointer"};
    dfuse_ctx* ctx = kf->ctx;
    const long P = kf->P;
    FusionStateDev st;
    DF_CUDA(cudaMemcpyAsync(&st, kf->st + kf->parity, sizeof st, cudaMemcpyDeviceToHost,
                            ctx->stream));
    // ground truth into the idle PCG vectors (q, b) of the fusion workspace
    double* d_gt = kf->fa.q;
    uint8_t* d_gv = (uint8_t*)kf->fa.b;
    DF_CUDA(cudaMemcpyAsync(d_gt, gt_metres, sizeof(double) * P, cudaMemcpyHostToDevice,
                            ctx->stream));
    DF_CUDA(cudaMemcpyAsync(d_gv, gt_valid, P, cudaMemcpyHostToDevice, ctx->stream));
    DF_CUDA(cudaStreamSynchronize(ctx->stream));
    score_device(ctx, P, nullptr, kf->fa.ld[st.cur], nullptr, d_gt, d_gv, out);
  });
}

int dfuse_kf_export_depth_u16(dfuse_keyframe* kf, double depth_scale, uint16_t* out) {
  return kf_guarded(kf, [&] {
    if (!out) throw RefError{DFUSE_E_INVALID_ARGUMENT, "null pointer"};
    dfuse_ctx* ctx = kf->ctx;
    FusionStateDev st;
    DF_CUDA(cudaMemcpyAsync(&st, kf->st + kf->parity, sizeof st, cudaMemcpyDeviceToHost,
                            ctx->stream));
    DF_CUDA(cudaStreamSynchronize(ctx->stream));
    uint16_t* d = (uint16_t*)kf->fa.q;
    export_u16_device(ctx, kf->P, kf->fa.ld[st.cur], depth_scale, d);
    DF_CUDA(cudaMemcpyAsync(out, d, sizeof(uint16_t) * kf->P, cudaMemcpyDeviceToHost,
                            ctx->stream));
    DF_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

}  // extern "C"
