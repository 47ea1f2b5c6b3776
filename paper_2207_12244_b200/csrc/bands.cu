// bands.cu -- a keyframe split into row bands.
//
// Band g owns rows [y0_g, y1_g) of the raster. Everything per pixel that the
// fusion optimiser keeps (predictions, semi-dense map, log-depth buffers,
// normal equations, PCG vectors) lives in the band's own allocation, which
// covers rows [y0 - 1, y1 + 1): one halo row on each side. Plane pointers are
// shifted so that global pixel indices address them, so the sweeps of
// fusion.cu run unchanged on a band; the planes read at i - W or i + W get
// their halo rows from the neighbour band (halo_put / BandNb), and the
// all-reduces are two-level (BandCtx). The stereo stage needs no exchange:
// each band scans its own masked pixels against the full I0 / I1 and updates
// its own semi-dense rows; the inlier count is one shared counter.
//
// On one GPU all bands run in one cooperative launch (this file); the
// multi-GPU layout is the same allocations on different devices, with the
// BandNb pointers and level-2 arrays mapped from the peers.
#include <string.h>

#include <new>
#include <vector>

#include "common.cuh"
#include "fusion.cuh"
#include "stereo.cuh"

using namespace dfuse_cuda;

namespace {

size_t al(size_t v) { return (v + 255) & ~size_t(255); }

enum BandPlane {  // the 25 double planes of a band, in allocation order
  BP_PRED0 = 0, BP_SD = 6, BP_SV, BP_LNSD, BP_IRS, BP_IV0, BP_IV1, BP_IV2, BP_LD0, BP_LD1,
  BP_DIAG, BP_RIGHT, BP_DOWN, BP_B, BP_X, BP_R, BP_Z, BP_P0, BP_P1, BP_Q, BP_COUNT
};
static_assert(BP_COUNT == 25, "plane count");

struct Band {
  int y0 = 0, y1 = 0;
  void* block = nullptr;
  bool owned = false;   // allocated here (else an IPC mapping of a peer's band, or absent)
  bool local = false;   // computed by this process
  int* list = nullptr;
  int* counters = nullptr;  // [0] work counter, [1] list length, [2] n_obs, [3] inlier count
  int n_mask = 0;
  int h_counters[4] = {0, 0, 0, 0};  // n_obs, inliers, steps (64-bit)
  double *semi_d = nullptr, *semi_v = nullptr;
  uint8_t* semi_valid = nullptr;
  unsigned long long* rank_slots = nullptr;
  FusionStateDev* st = nullptr;  // [2]
  BandNb* nb_dev = nullptr;
  FusionArgs fa;  // device pointers, shifted to global pixel indices
  double* plane_base[BP_COUNT];  // unshifted plane starts (for copies)
};

}  // namespace

struct dfuse_banded_keyframe {
  dfuse_ctx* ctx = nullptr;
  int W = 0, H = 0, nband = 0, cpr = 0;
  int rank = -1;      // -1: every band in this process; else the one band it computes
  bool connected = false;  // neighbours and level-2 arrays bound (dfuse_bkf_connect)
  long P = 0;
  void* common = nullptr;  // I0, I1, mask, shared counters, device arg arrays
  float* I0 = nullptr;
  float* I1 = nullptr;
  uint8_t* mask = nullptr;
  int* shared = nullptr;  // unused (per-band counters)
  FusionArgs* d_args = nullptr;
  unsigned long long** d_rank = nullptr;
  std::vector<Band> bands;
  int parity = 0;
  int stereo_frames = 0;
  FusionControl* h_ctl = nullptr;  // pinned
};

namespace {

template <class F>
int bkf_guarded(dfuse_banded_keyframe* kf, F&& f) {
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

// the band's rows, with halo rows clamped to the image
inline int lo_row(const Band& b) { return b.y0 > 0 ? b.y0 - 1 : 0; }
inline int hi_row(const Band& b, int H) { return b.y1 < H ? b.y1 + 1 : H; }



// Byte layout of one band's allocation: a pure function of (W, rows, CTAs
// per band, band count), so a peer can rebuild every pointer of a band it
// maps by IPC from the base address alone.
struct BandLayout {
  size_t plane[BP_COUNT], planef[5], valid, list, counters, slots, rank_slots, ctl, st, nb, total;
};

BandLayout band_layout(int W, int y0, int y1, int cpr, int nband) {
  BandLayout L;
  const long n = (long)(y1 - y0 + 2) * W;  // halo row on both sides
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t r = o;
    o += al(bytes);
    return r;
  };
  for (int k = 0; k < BP_COUNT; ++k) L.plane[k] = take(sizeof(double) * n);
  for (int k = 0; k < 5; ++k) L.planef[k] = take(sizeof(float) * n);  // predf[1..5]
  L.valid = take(n);
  L.list = take(sizeof(int) * (size_t)(y1 - y0) * W);
  L.counters = take(256);
  L.slots = take(fusion_slots_bytes(cpr));
  L.rank_slots = take(band_rank_slots_bytes(nband));
  L.ctl = take(sizeof(FusionControl));
  L.st = take(2 * sizeof(FusionStateDev));
  L.nb = take(sizeof(BandNb));
  L.total = o;
  return L;
}

// point b (and b.fa) into the band allocation at `base`
void bind_band(dfuse_banded_keyframe* kf, Band& b, char* base, int cpr) {
  const int W = kf->W;
  const BandLayout L = band_layout(W, b.y0, b.y1, cpr, kf->nband);
  b.block = base;
  const long shift = (long)(b.y0 - 1) * W;  // plane + shift addresses row y0 - 1 at index 0
  double* sh[BP_COUNT];
  for (int k = 0; k < BP_COUNT; ++k) {
    b.plane_base[k] = (double*)(base + L.plane[k]);
    sh[k] = b.plane_base[k] - shift;
  }
  b.semi_valid = (uint8_t*)(base + L.valid) - shift;
  b.list = (int*)(base + L.list);
  b.counters = (int*)(base + L.counters);
  FusionArgs& f = b.fa;
  memset(&f, 0, sizeof f);
  f.W = kf->W;
  f.H = kf->H;
  for (int c = 0; c < 6; ++c) f.pred[c] = sh[BP_PRED0 + c];
  for (int c = 1; c < 6; ++c) f.predf[c] = (float*)(base + L.planef[c - 1]) - shift;
  b.semi_d = sh[BP_SD];
  b.semi_v = sh[BP_SV];
  f.sd = b.semi_d;
  f.sv = b.semi_v;
  f.svalid = b.semi_valid;
  f.lnsd = sh[BP_LNSD];
  f.irs = sh[BP_IRS];
  for (int k = 0; k < 3; ++k) f.ivar[k] = sh[BP_IV0 + k];
  f.ld[0] = sh[BP_LD0];
  f.ld[1] = sh[BP_LD1];
  f.diag = sh[BP_DIAG];
  f.right = sh[BP_RIGHT];
  f.down = sh[BP_DOWN];
  f.b = sh[BP_B];
  f.x = sh[BP_X];
  f.r = sh[BP_R];
  f.z = sh[BP_Z];
  f.p[0] = sh[BP_P0];
  f.p[1] = sh[BP_P1];
  f.q = sh[BP_Q];
  f.slots = (ReduceSlot*)(base + L.slots);
  b.rank_slots = (unsigned long long*)(base + L.rank_slots);
  f.ctl = (FusionControl*)(base + L.ctl);
  b.st = (FusionStateDev*)(base + L.st);
  b.nb_dev = (BandNb*)(base + L.nb);
  f.inlier_dev = b.counters + 3;  // the band's own inlier count (summed in the kernel)
  f.band_y0 = b.y0;
  f.band_y1 = b.y1;
  f.band_ctas = cpr;
  f.nb = b.nb_dev;
}

void alloc_band(dfuse_banded_keyframe* kf, Band& b) {
  const BandLayout L = band_layout(kf->W, b.y0, b.y1, kf->cpr, kf->nband);
  void* base = nullptr;
  DF_CUDA(cudaMalloc(&base, L.total));
  b.owned = true;
  bind_band(kf, b, (char*)base, kf->cpr);
  DF_CUDA(cudaMemsetAsync(b.counters, 0, 256, kf->ctx->stream));
  // LL words and the control block are cleared once, here, before any peer
  // can know this allocation exists (its IPC handle is exported only after
  // creation returns): launches then continue the flags (persist_sync)
  DF_CUDA(cudaMemsetAsync(b.fa.slots, 0, fusion_slots_bytes(kf->cpr), kf->ctx->stream));
  DF_CUDA(cudaMemsetAsync(b.rank_slots, 0, band_rank_slots_bytes(kf->nband), kf->ctx->stream));
  DF_CUDA(cudaMemsetAsync(b.fa.ctl, 0, sizeof(FusionControl), kf->ctx->stream));
  b.fa.persist_sync = 1;
}

// BandNb of band g: the halo planes of its neighbours (HaloPlane order)
BandNb neighbours(dfuse_banded_keyframe* kf, int g) {
  BandNb nb;
  memset(&nb, 0, sizeof nb);
  auto planes = [](const FusionArgs& f, double** out) {
    out[HP_LD0] = f.ld[0];
    out[HP_LD1] = f.ld[1];
    out[HP_X] = f.x;
    out[HP_Z] = f.z;
    out[HP_DOWN] = f.down;
    out[HP_P0] = f.p[0];
    out[HP_P1] = f.p[1];
    out[HP_IV2] = f.ivar[2];
  };
  if (g > 0) planes(kf->bands[g - 1].fa, nb.up);
  if (g + 1 < kf->nband) planes(kf->bands[g + 1].fa, nb.dn);
  return nb;
}

void reset_bkf(dfuse_banded_keyframe* kf) {
  dfuse_ctx* ctx = kf->ctx;
  const int W = kf->W;
  for (Band& b : kf->bands) {
    if (!b.local) continue;
    const long n = (long)(b.y1 - b.y0 + 2) * W;
    DF_CUDA(cudaMemsetAsync(b.plane_base[BP_SD], 0, sizeof(double) * n, ctx->stream));
    DF_CUDA(cudaMemsetAsync(b.plane_base[BP_SV], 0, sizeof(double) * n, ctx->stream));
    DF_CUDA(cudaMemsetAsync(b.semi_valid + (long)(b.y0 - 1) * W, 0, n, ctx->stream));
    // init_state (fusion.hpp:44-46), halo rows included: they hold the
    // neighbours' rows of the same raster
    DF_CUDA(cudaMemcpyAsync(b.plane_base[BP_LD0], b.plane_base[BP_PRED0], sizeof(double) * n,
                            cudaMemcpyDeviceToDevice, ctx->stream));
    FusionStateDev s0{1.0, 0, 0};
    DF_CUDA(cudaMemcpyAsync(b.st, &s0, sizeof s0, cudaMemcpyHostToDevice, ctx->stream));
    DF_CUDA(cudaMemsetAsync(b.counters + 2, 0, 2 * sizeof(int), ctx->stream));
  }
  DF_CUDA(cudaStreamSynchronize(ctx->stream));
  kf->parity = 0;
  kf->stereo_frames = 0;
}

void process_bkf(dfuse_banded_keyframe* kf, const dfuse_epigeom* g, const float* I1_dev,
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
  // stereo stage: every band scans its own masked pixels (pipeline.hpp:205-213)
  DF_CUDA(cudaEventRecord(ctx->ev[0], ctx->stream));
  if (!kf->connected) throw RefError{DFUSE_E_INVALID_ARGUMENT, "bands not connected"};
  for (Band& b : kf->bands) {
    if (!b.local) continue;
    DF_CUDA(cudaMemsetAsync(b.counters + 2, 0, sizeof(int), ctx->stream));  // n_obs
    DF_CUDA(cudaMemsetAsync(b.counters + 4, 0, 2 * sizeof(int), ctx->stream));  // steps
    if (b.n_mask == 0) continue;
    StereoArgs a;
    memset(&a, 0, sizeof a);
    a.g = *g;
    a.cfg = *scfg;
    a.I0 = kf->I0;
    a.I1 = I1_dev;
    a.n_items = b.n_mask;
    a.work_counter = b.counters;
    a.list = b.list;
    a.depth = b.semi_d;
    a.variance = b.semi_v;
    a.valid = b.semi_valid;
    a.n_obs = b.counters + 2;
    a.n_installed = b.counters + 3;
    a.step_count = reinterpret_cast<unsigned long long*>(b.counters + 4);
    launch_stereo(ctx, a, false);
  }
  DF_CUDA(cudaEventRecord(ctx->ev[1], ctx->stream));
  // optimise stage over all bands (pipeline.hpp:223-226)
  std::vector<FusionArgs> args(kf->nband);
  int first = -1, nlocal = 0;
  for (int k = 0; k < kf->nband; ++k) {
    Band& b = kf->bands[k];
    if (!b.local) continue;
    if (first < 0) first = k;
    FusionArgs f = b.fa;
    f.dsemi = rcfg->delta_semi;
    f.dnet = rcfg->delta_net;
    f.dgrad = rcfg->delta_grad;
    f.cg_tol = rcfg->cg_tol;
    f.gn = rcfg->gn_iterations;
    f.cg_max = rcfg->cg_max_iters;
    f.est_scale = rcfg->estimate_scale;
    f.mode = mode;
    f.op = OP_OPTIMIZE;
    f.st_in = b.st + kf->parity;
    f.st_out = b.st + (1 - kf->parity);
    f.band_cta0 = (k - first) * kf->cpr;
    args[k] = f;
    ++nlocal;
    // no per-launch clearing of the LL arrays: the flags continue from the
    // previous launch (ctl->sync_phase, identical in every band), and every
    // slot is rewritten each time its phase parity comes round, so 32-bit
    // flag wrap-around never meets a stale word of the same value
  }
  DF_CUDA(cudaMemcpyAsync(kf->d_args, args.data(), sizeof(FusionArgs) * kf->nband,
                          cudaMemcpyHostToDevice, ctx->stream));
  launch_fusion_banded(ctx, kf->d_args, kf->d_rank, kf->nband, kf->cpr, first, nlocal,
                       kf->rank >= 0 ? 1 : 0, &args[first]);
  DF_CUDA(cudaEventRecord(ctx->ev[2], ctx->stream));
  for (Band& b : kf->bands)
    if (b.local)
      DF_CUDA(cudaMemcpyAsync(b.h_counters, b.counters + 2, 4 * sizeof(int),
                              cudaMemcpyDeviceToHost, ctx->stream));
  DF_CUDA(cudaMemcpyAsync(kf->h_ctl, kf->bands[first].fa.ctl, sizeof(FusionControl),
                          cudaMemcpyDeviceToHost, ctx->stream));
  DF_CUDA(cudaStreamSynchronize(ctx->stream));
  int n_obs = 0, inliers = 0;
  long long steps = 0;
  for (Band& b : kf->bands)
    if (b.local) {
      n_obs += b.h_counters[0];
      inliers += b.h_counters[1];
      long long st;
      memcpy(&st, b.h_counters + 2, sizeof st);
      steps += st;
    }
  kf->parity = 1 - kf->parity;
  // multi-process: these are this rank's bands (the caller sums over ranks)
  if (n_obs > 0) kf->stereo_frames += 1;  // pipeline.hpp:211
  res->observations = n_obs;
  res->inlier_count = inliers;
  res->stereo_frames = kf->stereo_frames;
  res->optimize_status = kf->h_ctl->status;
  DF_CUDA(cudaEventElapsedTime(&res->stereo_ms, ctx->ev[0], ctx->ev[1]));
  DF_CUDA(cudaEventElapsedTime(&res->optimise_ms, ctx->ev[1], ctx->ev[2]));
  res->stats = kf->h_ctl->stats;
  res->epipolar_steps = steps;
  res->solver_ppt = 0;  // the row-band solve streams
  res->reserved = 0;
}

// the HaloPlane `plane` of a band's FusionArgs (the order of neighbours())
double* halo_plane(const FusionArgs& f, int plane) {
  switch (plane) {
    case HP_LD0: return f.ld[0];
    case HP_LD1: return f.ld[1];
    case HP_X: return f.x;
    case HP_Z: return f.z;
    case HP_DOWN: return f.down;
    case HP_P0: return f.p[0];
    case HP_P1: return f.p[1];
    case HP_IV2: return f.ivar[2];
    default: throw RefError{DFUSE_E_INVALID_ARGUMENT, "unknown halo plane"};
  }
}

// diagnostics: this band's boundary rows into the neighbours' halo rows with
// the solver's halo_put stores (fusion_impl.cuh) -- remote stores when the
// neighbour is a peer mapping -- value base + global pixel index
__global__ void k_band_halo_probe(const BandNb* __restrict__ nb, int W, int y0, int y1, int plane,
                                  double base) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < W; x += gridDim.x * blockDim.x) {
    const long top = (long)y0 * W + x, bot = (long)(y1 - 1) * W + x;
    if (nb->up[plane]) nb->up[plane][top] = base + (double)top;
    if (nb->dn[plane]) nb->dn[plane][bot] = base + (double)bot;
  }
  __threadfence_system();
}

}  // namespace

namespace {

void bind_neighbours(dfuse_banded_keyframe* kf) {
  dfuse_ctx* ctx = kf->ctx;
  std::vector<unsigned long long*> rank(kf->nband);
  for (int g = 0; g < kf->nband; ++g) rank[g] = kf->bands[g].rank_slots;
  for (int g = 0; g < kf->nband; ++g) {
    Band& b = kf->bands[g];
    if (!b.local) continue;
    const BandNb nb = neighbours(kf, g);
    DF_CUDA(cudaMemcpyAsync(b.nb_dev, &nb, sizeof nb, cudaMemcpyHostToDevice, ctx->stream));
  }
  DF_CUDA(cudaMemcpyAsync(kf->d_rank, rank.data(), sizeof(void*) * kf->nband,
                          cudaMemcpyHostToDevice, ctx->stream));
  DF_CUDA(cudaStreamSynchronize(ctx->stream));
  kf->connected = true;
}

// everything up to (not including) the neighbour binding; bands with
// local = true are allocated and initialised here
void create_bkf(dfuse_banded_keyframe* kf, const dfuse_intrinsics* K, const float* I0,
                const double* const pred[6], double texture_threshold, int bands, int rank) {
  dfuse_ctx* ctx = kf->ctx;
  if (!K || !I0 || !pred) throw RefError{DFUSE_E_INVALID_ARGUMENT, "null pointer"};
  for (int c = 0; c < 6; ++c)
    if (!pred[c]) throw RefError{DFUSE_E_INVALID_ARGUMENT, "null prediction plane"};
  if (K->width <= 0 || K->height <= 0)
    throw RefError{DFUSE_E_INVALID_ARGUMENT, "raster dimensions must be positive"};
  if (texture_threshold <= 0.0)
    throw RefError{DFUSE_E_INVALID_ARGUMENT, "texture threshold must be > 0"};
  const int per_process = rank < 0 ? bands : 1;
  if (bands < 1 || bands > K->height || per_process > ctx->num_sms ||
      (rank >= 0 && rank >= bands))
    throw RefError{DFUSE_E_INVALID_ARGUMENT, "bands must be in [1, min(height, SMs)]"};
  kf->W = K->width;
  kf->H = K->height;
  kf->P = (long)kf->W * kf->H;
  kf->nband = bands;
  kf->rank = rank;
  // CTAs per band: two per SM overall, like the streaming kernel (whose
  // reductions a one-band keyframe then reproduces bit for bit)
  kf->cpr = band_ctas_per_sm() * fusion_grid(ctx) / per_process;
  if (kf->cpr > 32 * 5 * 2) kf->cpr = 32 * 5 * 2;
  const long P = kf->P;
  const size_t common = 2 * al(sizeof(float) * P) + al(P) + al(sizeof(int) * bands + 256) +
                        al(sizeof(FusionArgs) * bands) + al(sizeof(void*) * bands);
  DF_CUDA(cudaMalloc(&kf->common, common));
  char* p = (char*)kf->common;
  auto take = [&](size_t bytes) {
    char* r = p;
    p += al(bytes);
    return (void*)r;
  };
  kf->I0 = (float*)take(sizeof(float) * P);
  kf->I1 = (float*)take(sizeof(float) * P);
  kf->mask = (uint8_t*)take(P);
  kf->shared = (int*)take(sizeof(int) * bands + 256);  // per-band scratch counters
  kf->d_args = (FusionArgs*)take(sizeof(FusionArgs) * bands);
  kf->d_rank = (unsigned long long**)take(sizeof(void*) * bands);
  DF_CUDA(cudaMallocHost(&kf->h_ctl, sizeof(FusionControl)));
  kf->bands.resize(bands);
  for (int g = 0; g < bands; ++g) {  // even row split
    Band& b = kf->bands[g];
    b.y0 = (int)((long)kf->H * g / bands);
    b.y1 = (int)((long)kf->H * (g + 1) / bands);
    b.local = rank < 0 || rank == g;
    if (b.local) alloc_band(kf, b);
  }
  for (Band& b : kf->bands) {
    if (!b.local) continue;
    // predictions: the band's rows and its halo rows (pred[4] is read at i - W)
    const int r0 = lo_row(b), r1 = hi_row(b, kf->H);
    for (int c = 0; c < 6; ++c)
      DF_CUDA(cudaMemcpyAsync((double*)b.fa.pred[c] + (long)r0 * kf->W,
                              pred[c] + (long)r0 * kf->W,
                              sizeof(double) * (size_t)(r1 - r0) * kf->W, cudaMemcpyHostToDevice,
                              ctx->stream));
  }
  // prediction planes 1..5 as float32 where every value (halo rows
  // included) is float-exact; a band that is not keeps its fp64 planes
  // (both forms give the same bits, so the bands may differ)
  int* inexact = (int*)kf->shared;
  DF_CUDA(cudaMemsetAsync(inexact, 0, sizeof(int) * bands, ctx->stream));
  for (int g = 0; g < bands; ++g) {
    Band& b = kf->bands[g];
    if (!b.local) continue;
    const long o = (long)lo_row(b) * kf->W;
    const double* p64[6];
    float* p32[6];
    for (int c = 0; c < 6; ++c) {
      p64[c] = b.fa.pred[c] + o;
      p32[c] = c ? const_cast<float*>(b.fa.predf[c]) + o : nullptr;
    }
    launch_pred_narrow(ctx, p64, p32, (long)(hi_row(b, kf->H) - lo_row(b)) * kf->W, inexact + g);
  }
  std::vector<int> h_inexact(bands, 0);
  DF_CUDA(cudaMemcpyAsync(h_inexact.data(), inexact, sizeof(int) * bands, cudaMemcpyDeviceToHost,
                          ctx->stream));
  DF_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int g = 0; g < bands; ++g)
    if (kf->bands[g].local) {
      Band& b = kf->bands[g];
      b.fa.pred_f32_ok = (h_inexact[g] == 0 && ctx->pred_fp32);
      b.fa.pred_f32 = b.fa.pred_f32_ok ? 1 : 0;  // the row-band solve streams: mode 1
    }
  DF_CUDA(cudaMemcpyAsync(kf->I0, I0, sizeof(float) * P, cudaMemcpyHostToDevice, ctx->stream));
  // make_keyframe: texture_mask (pipeline.hpp:148), then each band's list
  launch_texture_mask(ctx, kf->I0, kf->W, kf->H, texture_threshold, kf->mask);
  for (Band& b : kf->bands) {
    if (!b.local) continue;
    const long off = (long)b.y0 * kf->W;
    launch_mask_list(ctx, kf->mask + off, (long)(b.y1 - b.y0) * kf->W, b.list, b.counters + 1,
                     off);
    DF_CUDA(cudaMemcpyAsync(&b.n_mask, b.counters + 1, sizeof(int), cudaMemcpyDeviceToHost,
                            ctx->stream));
  }
  reset_bkf(kf);  // synchronises
}

}  // namespace

extern "C" {

int dfuse_bkf_destroy(dfuse_banded_keyframe* kf) {
  if (!kf) return DFUSE_OK;
  if (kf->ctx) {
    cudaSetDevice(kf->ctx->device);
    cudaStreamSynchronize(kf->ctx->stream);
  }
  for (Band& b : kf->bands) {
    if (b.owned && b.block) cudaFree(b.block);
    else if (b.block) cudaIpcCloseMemHandle(b.block);
  }
  if (kf->common) cudaFree(kf->common);
  if (kf->h_ctl) cudaFreeHost(kf->h_ctl);
  delete kf;
  return DFUSE_OK;
}

int dfuse_bkf_create(dfuse_ctx* ctx, const dfuse_intrinsics* K, const float* I0,
                     const double* const pred[6], double texture_threshold, int bands,
                     dfuse_banded_keyframe** out) {
  if (!ctx || !out) return DFUSE_E_INVALID_ARGUMENT;
  *out = nullptr;
  dfuse_banded_keyframe* kf = new (std::nothrow) dfuse_banded_keyframe();
  if (!kf) return DFUSE_E_CUDA;
  kf->ctx = ctx;
  const int rc = bkf_guarded(kf, [&] {
    create_bkf(kf, K, I0, pred, texture_threshold, bands, -1);
    bind_neighbours(kf);
  });
  if (rc) {
    dfuse_bkf_destroy(kf);
    return rc;
  }
  *out = kf;
  return DFUSE_OK;
}

int dfuse_bkf_create_rank(dfuse_ctx* ctx, const dfuse_intrinsics* K, const float* I0,
                          const double* const pred[6], double texture_threshold, int world,
                          int rank, dfuse_banded_keyframe** out) {
  if (!ctx || !out) return DFUSE_E_INVALID_ARGUMENT;
  *out = nullptr;
  dfuse_banded_keyframe* kf = new (std::nothrow) dfuse_banded_keyframe();
  if (!kf) return DFUSE_E_CUDA;
  kf->ctx = ctx;
  const int rc = bkf_guarded(kf, [&] {
    if (rank < 0) throw RefError{DFUSE_E_INVALID_ARGUMENT, "rank must be >= 0"};
    create_bkf(kf, K, I0, pred, texture_threshold, world, rank);
    if (world == 1) bind_neighbours(kf);
  });
  if (rc) {
    dfuse_bkf_destroy(kf);
    return rc;
  }
  *out = kf;
  return DFUSE_OK;
}

int dfuse_bkf_peer_info(dfuse_banded_keyframe* kf, dfuse_band_peer* out) {
  return bkf_guarded(kf, [&] {
    if (!out || kf->rank < 0) throw RefError{DFUSE_E_INVALID_ARGUMENT, "not a rank keyframe"};
    const Band& b = kf->bands[kf->rank];
    memset(out, 0, sizeof *out);
    cudaIpcMemHandle_t h;
    DF_CUDA(cudaIpcGetMemHandle(&h, b.block));
    static_assert(sizeof h == sizeof out->handle, "IPC handle size");
    memcpy(out->handle, &h, sizeof h);
    out->cpr = kf->cpr;
    out->y0 = b.y0;
    out->y1 = b.y1;
    out->width = kf->W;
  });
}

int dfuse_bkf_connect(dfuse_banded_keyframe* kf, const dfuse_band_peer* peers) {
  return bkf_guarded(kf, [&] {
    if (!peers || kf->rank < 0) throw RefError{DFUSE_E_INVALID_ARGUMENT, "not a rank keyframe"};
    for (int g = 0; g < kf->nband; ++g) {
      Band& b = kf->bands[g];
      const dfuse_band_peer& pi = peers[g];
      if (pi.y0 != b.y0 || pi.y1 != b.y1 || pi.width != kf->W)
        throw RefError{DFUSE_E_DIMENSION_MISMATCH, "peer band layout differs"};
      if (b.local) continue;
      cudaIpcMemHandle_t h;
      memcpy(&h, pi.handle, sizeof h);
      void* base = nullptr;
      DF_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
      bind_band(kf, b, (char*)base, pi.cpr);
    }
    bind_neighbours(kf);
  });
}

int dfuse_bkf_debug_halo_put(dfuse_banded_keyframe* kf, int plane, double base) {
  return bkf_guarded(kf, [&] {
    if (!kf->connected) throw RefError{DFUSE_E_INVALID_ARGUMENT, "bands not connected"};
    if (plane < 0 || plane >= HP_COUNT) throw RefError{DFUSE_E_INVALID_ARGUMENT, "bad plane"};
    dfuse_ctx* ctx = kf->ctx;
    for (Band& b : kf->bands) {
      if (!b.local) continue;
      k_band_halo_probe<<<(kf->W + 255) / 256, 256, 0, ctx->stream>>>(b.nb_dev, kf->W, b.y0,
                                                                       b.y1, plane, base);
      DF_LAUNCHED(ctx);
    }
    DF_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int dfuse_bkf_debug_halo_get(dfuse_banded_keyframe* kf, int plane, double* above,
                             double* below) {
  return bkf_guarded(kf, [&] {
    if (kf->rank < 0) throw RefError{DFUSE_E_INVALID_ARGUMENT, "not a rank keyframe"};
    const Band& b = kf->bands[kf->rank];
    const double* p = halo_plane(b.fa, plane);
    dfuse_ctx* ctx = kf->ctx;
    const size_t row = sizeof(double) * kf->W;
    if (above && b.y0 > 0)
      DF_CUDA(cudaMemcpyAsync(above, p + (long)(b.y0 - 1) * kf->W, row, cudaMemcpyDeviceToHost,
                              ctx->stream));
    if (below && b.y1 < kf->H)
      DF_CUDA(cudaMemcpyAsync(below, p + (long)b.y1 * kf->W, row, cudaMemcpyDeviceToHost,
                              ctx->stream));
    DF_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int dfuse_bkf_reset(dfuse_banded_keyframe* kf) {
  return bkf_guarded(kf, [&] { reset_bkf(kf); });
}

int dfuse_bkf_process_frame(dfuse_banded_keyframe* kf, const dfuse_epigeom* g, const float* I1,
                            const dfuse_search_cfg* scfg, const dfuse_robust_cfg* rcfg, int mode,
                            dfuse_frame_result* res) {
  return bkf_guarded(kf, [&] {
    if (!I1) throw RefError{DFUSE_E_INVALID_ARGUMENT, "null image"};
    DF_CUDA(cudaMemcpyAsync(kf->I1, I1, sizeof(float) * kf->P, cudaMemcpyHostToDevice,
                            kf->ctx->stream));
    process_bkf(kf, g, kf->I1, scfg, rcfg, mode, res);
  });
}

int dfuse_bkf_process_frame_dev(dfuse_banded_keyframe* kf, const dfuse_epigeom* g,
                                const float* I1_dev, const dfuse_search_cfg* scfg,
                                const dfuse_robust_cfg* rcfg, int mode,
                                dfuse_frame_result* res) {
  return bkf_guarded(kf, [&] {
    if (!I1_dev) throw RefError{DFUSE_E_INVALID_ARGUMENT, "null image"};
    process_bkf(kf, g, I1_dev, scfg, rcfg, mode, res);
  });
}

int dfuse_bkf_download(dfuse_banded_keyframe* kf, double* log_depth, double* scale,
                       int32_t* iteration, double* semi_depth, double* semi_variance,
                       uint8_t* semi_valid, int32_t* inlier_count, uint8_t* mask) {
  return bkf_guarded(kf, [&] {
    dfuse_ctx* ctx = kf->ctx;
    int first = 0;
    while (!kf->bands[first].local) ++first;
    FusionStateDev st;
    DF_CUDA(cudaMemcpyAsync(&st, kf->bands[first].st + kf->parity, sizeof st,
                            cudaMemcpyDeviceToHost, ctx->stream));
    DF_CUDA(cudaStreamSynchronize(ctx->stream));
    const int W = kf->W;
    int inliers = 0;
    for (Band& b : kf->bands) {  // each local band's own rows
      if (!b.local) continue;
      const long o = (long)b.y0 * W;
      const size_t n = (size_t)(b.y1 - b.y0) * W;
      auto cp = [&](void* dst, const void* src, size_t elem) {
        if (dst)
          DF_CUDA(cudaMemcpyAsync((char*)dst + o * elem, (const char*)src + o * elem, n * elem,
                                  cudaMemcpyDeviceToHost, ctx->stream));
      };
      cp(log_depth, b.fa.ld[st.cur], sizeof(double));
      cp(semi_depth, b.semi_d, sizeof(double));
      cp(semi_variance, b.semi_v, sizeof(double));
      cp(semi_valid, b.semi_valid, 1);
      DF_CUDA(cudaMemcpyAsync(b.h_counters, b.counters + 2, 2 * sizeof(int),
                              cudaMemcpyDeviceToHost, ctx->stream));
    }
    if (mask) DF_CUDA(cudaMemcpyAsync(mask, kf->mask, kf->P, cudaMemcpyDeviceToHost, ctx->stream));
    DF_CUDA(cudaStreamSynchronize(ctx->stream));
    for (Band& b : kf->bands)
      if (b.local) inliers += b.h_counters[1];
    if (inlier_count) *inlier_count = inliers;
    if (scale) *scale = st.scale;
    if (iteration) *iteration = st.iteration;
  });
}

}  // extern "C"
