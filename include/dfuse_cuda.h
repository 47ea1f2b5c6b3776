/*
 * dfuse_cuda.h -- C-ABI of the B200 implementation of DeepFusion's per-frame
 * dense-depth hot path (texture mask -> epipolar SSD search -> semi-dense
 * update -> alternating Gauss-Newton fusion with Huber IRLS + Jacobi PCG).
 *
 * Every entry point replaces one function of the reference's header-only
 * C++ API (/root/reference/proj/include/dfuse, cited per entry point below as
 * file:line). Conventions:
 *   - plain pointers and sizes only; no C++ or torch types;
 *   - every raster is row-major, index i = y*W + x (raster.hpp:11-12,30);
 *   - pointers are HOST pointers unless the name ends in _dev;
 *   - return value 0 = OK, otherwise (int)dfuse::Err + 1 (errors.hpp:8-42);
 *     dfuse_last_error() returns the message of the last failing call;
 *   - one dfuse_ctx = one device + one stream; not thread-safe; distinct
 *     contexts may run concurrently; every call is synchronous;
 *   - there is no CPU fallback: a context cannot be created without an sm_100
 *     device and every compute call runs a CUDA kernel.
 */
#ifndef DFUSE_CUDA_H
#define DFUSE_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DFUSE_ABI_VERSION 1

/* error codes = (int)dfuse::Err + 1, errors.hpp:8-42 */
enum {
  DFUSE_OK = 0,
  DFUSE_E_NON_POSITIVE_DEPTH = 1,
  DFUSE_E_BEHIND_CAMERA = 2,
  DFUSE_E_OUT_OF_BOUNDS = 3,
  DFUSE_E_DEGENERATE_BASELINE = 4,
  DFUSE_E_NO_MINIMUM = 5,
  DFUSE_E_ZERO_BASELINE_STEP = 6,
  DFUSE_E_DEGENERATE_JACOBIAN = 7,
  DFUSE_E_BORDER_PIXEL = 8,
  DFUSE_E_BAD_MAGIC = 9,
  DFUSE_E_DIMENSION_MISMATCH = 10,
  DFUSE_E_NON_POSITIVE_VARIANCE = 11,
  DFUSE_E_TRUNCATED_FILE = 12,
  DFUSE_E_NON_POSITIVE_FOCAL = 13,
  DFUSE_E_NON_POSITIVE_GROUND_TRUTH = 14,
  DFUSE_E_MISSING_FILE = 15,
  DFUSE_E_MALFORMED_LINE = 16,
  DFUSE_E_NON_UNIT_QUATERNION = 17,
  DFUSE_E_BAD_IMAGE_FORMAT = 18,
  DFUSE_E_NON_POSITIVE_SCALE = 19,
  DFUSE_E_CG_DIVERGENCE = 20,
  DFUSE_E_NO_SEMIDENSE_SUPPORT = 21,
  DFUSE_E_NO_VALID_GROUND_TRUTH = 22,
  DFUSE_E_MISMATCHED_KEYFRAME_SETS = 23,
  DFUSE_E_IO_ERROR = 24,
  DFUSE_E_UNKNOWN_KEY = 25,
  DFUSE_E_TYPE_ERROR = 26,
  DFUSE_E_INVALID_ARGUMENT = 27,
  DFUSE_E_CUDA = 100 /* CUDA runtime failure (not a reference error) */
};

/* EpipolarStatus, semidense.hpp:46-53 */
enum {
  DFUSE_EPI_OK = 0,
  DFUSE_EPI_DEGENERATE_BASELINE = 1,
  DFUSE_EPI_OUT_OF_BOUNDS = 2,
  DFUSE_EPI_BEHIND_CAMERA = 3,
  DFUSE_EPI_NO_MINIMUM = 4,
  DFUSE_EPI_DEGENERATE_JACOBIAN = 5,
  DFUSE_EPI_NOT_SEARCHED = -1 /* pixel outside the texture mask (debug output only) */
};

/* FusionMode, fusion.hpp:33 */
enum { DFUSE_MODE_FULL = 0, DFUSE_MODE_NOPAIRWISE = 1, DFUSE_MODE_LSSCALE = 2 };

/* CameraIntrinsics, geometry.hpp:18-41 */
typedef struct {
  double fx, fy, cx, cy;
  int32_t width, height;
} dfuse_intrinsics;

/* EpipolarGeometry, semidense.hpp:94-99. R_10 row-major. */
typedef struct {
  double R_10[9];
  double t_10[3];
  double t_01[3];
  dfuse_intrinsics K;
} dfuse_epigeom;

/* SearchConfig, semidense.hpp:66-73 (defaults 0.25, 50, 0.05) */
typedef struct {
  double min_depth, max_depth, max_rms_error;
} dfuse_search_cfg;

/* RobustConfig, fusion.hpp:23-31 (defaults 0.3, 0.3, 0.1, 10, 1e-6, 200, 1) */
typedef struct {
  double delta_semi, delta_net, delta_grad;
  double cg_tol;
  int32_t gn_iterations;
  int32_t cg_max_iters;
  int32_t estimate_scale;
  int32_t reserved;
} dfuse_robust_cfg;

/* EpipolarObservation, semidense.hpp:38-44 (112 bytes, same field order) */
typedef struct {
  double x, y;
  double depth;
  double error5[5];
  double jacobian[5];
  double variance;
} dfuse_obs;

/* Dense fusion problem (FusionState inputs other than log_depth/scale,
 * SemiDenseMap semidense.hpp:21-31, PredictionSet predictions.hpp:18-29).
 * pred[c], c = log_depth, log_depth_var, grad_x, grad_x_var, grad_y,
 * grad_y_var. Host pointers, W*H entries each. */
typedef struct {
  int32_t width, height;
  const double* semi_depth;
  const double* semi_variance;
  const uint8_t* semi_valid;
  int32_t inlier_count;
  int32_t reserved;
  const double* pred[6];
} dfuse_fusion_inputs;

/* Solver trace of one optimize() call (fusion.hpp:402-454). Per-GN arrays
 * are recorded for the first DFUSE_STATS_MAX_GN iterations. */
#define DFUSE_STATS_MAX_GN 512
typedef struct {
  int32_t gn_done;      /* GN iterations executed */
  int32_t pcg_total;    /* PCG iterations summed over GN iterations */
  int32_t cost_evals;   /* total_cost sweeps (incl. line-search trials) */
  int32_t grid_syncs;   /* device-wide barriers executed */
  int32_t pcg_iters[DFUSE_STATS_MAX_GN];   /* -1: depth block not run */
  double scale_step[DFUSE_STATS_MAX_GN];   /* accepted step; 0 none; -1 not run */
  double depth_step[DFUSE_STATS_MAX_GN];   /* accepted step; 0 none; -1 not run */
} dfuse_solver_stats;

typedef struct dfuse_ctx dfuse_ctx;
typedef struct dfuse_keyframe dfuse_keyframe;

/* ---- context ---------------------------------------------------------- */
int dfuse_abi_version(void);
const char* dfuse_err_name(int code); /* err_name, errors.hpp:44-75 */
int dfuse_ctx_create(int device, dfuse_ctx** out);
int dfuse_ctx_destroy(dfuse_ctx* ctx);
const char* dfuse_last_error(const dfuse_ctx* ctx);
/* number of persistent CTAs the fusion solver uses (0 = one per SM) */
int dfuse_ctx_set_solver_ctas(dfuse_ctx* ctx, int ctas);
/* PCG data path: 0 = auto (SM-resident tiles, pipelined PCG whose one grid
 * all-reduce per iteration overlaps the SpMV, when the raster fits on chip,
 * else streaming from L2/HBM), 1 = always streaming, 2 = SM-resident with
 * two all-reduces per iteration (the reference's direct p.q), 3 = SM-resident
 * Chronopoulos-Gear (one exposed all-reduce per iteration) */
int dfuse_ctx_set_solver_path(dfuse_ctx* ctx, int path);
/* kernels launched on this context since creation (evidence counter) */
int64_t dfuse_ctx_launch_count(const dfuse_ctx* ctx);
/* the epipolar scan reads the tracked frame through a texture gather (one
 * tld4 per bilinear sample, the same texels: bit-identical results) when the
 * buffer meets the texture alignment; on = 0 forces plain loads (A/B, tests).
 * Default on. */
int dfuse_ctx_set_stereo_texture(dfuse_ctx* ctx, int on);
/* scan launches that used the texture gather (evidence counter) */
int64_t dfuse_ctx_texture_launches(const dfuse_ctx* ctx);
/* keyframes created on this context keep prediction planes 1..5 as float32
 * when every value is float-exact (the reference's own precision,
 * predictions.hpp:16-17): half the prediction bytes per sweep, bit-identical
 * results. on = 0 keeps fp64 planes (A/B, tests). Default on. */
int dfuse_ctx_set_fp32_predictions(dfuse_ctx* ctx, int on);
/* diagnostics: device time (ms) of one cooperative launch running n grid-wide
 * all-reduces of the fusion solver on `grid` CTAs (variant 10 = production LL
 * all-to-all, 2 = atomic arrival counter; 11-16 = two-level over CTA pairs,
 * cluster launch: 11/13 pair stage spinning on a DSMEM LL word, 12/14 the
 * same with only the even CTAs polling, 15 = variant 10 under a cluster
 * launch, 16 = pair stage by st.async on an mbarrier) */
int dfuse_debug_sync_bench(dfuse_ctx* ctx, int n, int variant, int grid, float* ms);
/* the context's cudaStream_t (for timing with events on the launch stream) */
void* dfuse_ctx_stream(const dfuse_ctx* ctx);

/* ---- host-side geometry ------------------------------------------------
 * make_epipolar_geometry(T0, T1, K), semidense.hpp:101-106, with Pose =
 * (quaternion w,x,y,z ; translation), geometry.hpp:44-67. Pure host code:
 * per frame pair, 15 doubles. */
int dfuse_make_epipolar_geometry(const double q0_wxyz[4], const double t0[3],
                                 const double q1_wxyz[4], const double t1[3],
                                 const dfuse_intrinsics* K, dfuse_epigeom* out);

/* ---- stereo front end (semidense.hpp) -------------------------------- */
/* texture_mask(img, threshold), semidense.hpp:77-91 */
int dfuse_texture_mask(dfuse_ctx* ctx, const float* img, int width, int height, double threshold,
                       uint8_t* mask);

/* search_depth(g, I0, I1, x, prior, cfg), semidense.hpp:277-379, for a list
 * of n pixels. px: n (x,y) pairs. prior: n (depth, sigma) pairs or NULL;
 * has_prior: n flags or NULL (NULL with prior != NULL means all have one).
 * Outputs: status[n] (DFUSE_EPI_*), obs[n] (valid where status == OK),
 * optional best[n] / n_steps[n] (search index of the SSD minimum and the
 * number of steps; -1 where the search did not reach that point). */
int dfuse_search_depth(dfuse_ctx* ctx, const dfuse_epigeom* g, const float* I0, const float* I1,
                       int n, const double* px, const double* prior, const uint8_t* has_prior,
                       const dfuse_search_cfg* cfg, int32_t* status, dfuse_obs* obs,
                       int32_t* best, int32_t* n_steps);

/* search_depth for VERSIONED host images (semidense.hpp:277-379): the
 * caller guarantees that the pixels at I0 (I1) do not change while gen0
 * (gen1) does not (the drop-in dfuse::IntensityImage hands out a fresh,
 * process-unique generation on construction, copy and every mutable
 * access). Device copies live in one process-wide cache keyed by (device,
 * host pointer, bytes, generation), shared by every context, so the
 * reference's per-pixel stereo_scan loop (pipeline.hpp:167-178, OpenMP
 * threads each with its own context) uploads each image once. gen = 0:
 * uncached (uploaded by this call). Otherwise as dfuse_search_depth. */
int dfuse_search_depth_gen(dfuse_ctx* ctx, const dfuse_epigeom* g, const float* I0, uint64_t gen0,
                           const float* I1, uint64_t gen1, int n, const double* px,
                           const double* prior, const uint8_t* has_prior,
                           const dfuse_search_cfg* cfg, int32_t* status, dfuse_obs* obs,
                           int32_t* best, int32_t* n_steps);
/* photometric_error_5pt with versioned images (see dfuse_search_depth_gen) */
int dfuse_photometric_error_5pt_gen(dfuse_ctx* ctx, const dfuse_epigeom* g, const float* I0,
                                    uint64_t gen0, const float* I1, uint64_t gen1, double x,
                                    double y, double d, double e[5], int32_t* status);
/* process-wide number of host->device image uploads and their bytes (the
 * evidence that versioned images are uploaded once) */
int dfuse_image_uploads(int64_t* count, int64_t* bytes);
/* stereo_scan(kf, frame, camera, cfg), pipeline.hpp:157-190: every masked
 * pixel searched with the prior (depth, sqrt(variance)) of the map where
 * valid; the OK observations in raster order into obs (capacity W*H),
 * *n_obs of them. The map is read only. One scan launch per frame. Images
 * versioned as in dfuse_search_depth_gen. */
int dfuse_stereo_scan(dfuse_ctx* ctx, const dfuse_epigeom* g, const float* I0, uint64_t gen0,
                      const float* I1, uint64_t gen1, const uint8_t* mask, const double* depth,
                      const double* variance, const uint8_t* valid, const dfuse_search_cfg* cfg,
                      dfuse_obs* obs, int32_t* n_obs);

/* photometric_error_5pt(g, I0, I1, x, d, e), semidense.hpp:227-243: the five
 * stencil residuals at one depth hypothesis; *status = DFUSE_EPI_* */
int dfuse_photometric_error_5pt(dfuse_ctx* ctx, const dfuse_epigeom* g, const float* I0,
                                const float* I1, double x, double y, double d, double e[5],
                                int32_t* status);

/* update_semidense(map, observations), semidense.hpp:393-417. The map is
 * updated in place (depth, variance, valid, inlier_count). Observations are
 * applied in list order (duplicates of one pixel fuse sequentially). */
int dfuse_update_semidense(dfuse_ctx* ctx, int width, int height, double* depth, double* variance,
                           uint8_t* valid, int32_t* inlier_count, int n_obs, const dfuse_obs* obs);

/* stereo_scan + update_semidense fused (pipeline.hpp:157-190,207-212): every
 * masked pixel searched with the prior taken from the map, then fused into
 * the map in place. n_obs = number of OK observations. Optional outputs
 * (NULL to skip): per-pixel status (int8, DFUSE_EPI_NOT_SEARCHED off-mask),
 * best, n_steps, and the observation list in raster order (capacity W*H). */
int dfuse_stereo_update(dfuse_ctx* ctx, const dfuse_epigeom* g, const float* I0, const float* I1,
                        const uint8_t* mask, const dfuse_search_cfg* cfg, double* depth,
                        double* variance, uint8_t* valid, int32_t* inlier_count, int32_t* n_obs,
                        int8_t* status, int32_t* best, int32_t* n_steps, dfuse_obs* obs);

/* ---- fusion optimiser (fusion.hpp) ----------------------------------- */
/* assemble_normal_equations, fusion.hpp:171-222 */
int dfuse_assemble_normal_equations(dfuse_ctx* ctx, const dfuse_fusion_inputs* in,
                                    const double* log_depth, double scale,
                                    const dfuse_robust_cfg* cfg, int mode, double* diag,
                                    double* right, double* down, double* b);
/* total_cost, fusion.hpp:225-253 */
int dfuse_total_cost(dfuse_ctx* ctx, const dfuse_fusion_inputs* in, const double* log_depth,
                     double scale, const dfuse_robust_cfg* cfg, int mode, double* cost);
/* cost_gradient, fusion.hpp:263-308 */
int dfuse_cost_gradient(dfuse_ctx* ctx, const dfuse_fusion_inputs* in, const double* log_depth,
                        double scale, const dfuse_robust_cfg* cfg, int mode, double* cost,
                        double* wrt_log_depth, double* wrt_ln_scale);
/* StencilMatrix::apply, fusion.hpp:120-135 */
int dfuse_stencil_apply(dfuse_ctx* ctx, int width, int height, const double* diag,
                        const double* right, const double* down, const double* x, double* y);
/* solve_depth_step, fusion.hpp:316-368. iterations: PCG iterations run. */
int dfuse_solve_depth_step(dfuse_ctx* ctx, int width, int height, const double* diag,
                           const double* right, const double* down, const double* b,
                           const dfuse_robust_cfg* cfg, double* delta, int32_t* iterations);
/* solve_scale_step, fusion.hpp:373-391 */
int dfuse_solve_scale_step(dfuse_ctx* ctx, const dfuse_fusion_inputs* in, const double* log_depth,
                           double scale, const dfuse_robust_cfg* cfg, double* scale_out);
/* optimize, fusion.hpp:402-454. Transactional: log_depth/scale/iteration are
 * written only when the call returns DFUSE_OK. stats may be NULL. */
int dfuse_optimize(dfuse_ctx* ctx, const dfuse_fusion_inputs* in, double* log_depth,
                   double* scale, int32_t* iteration, const dfuse_robust_cfg* cfg, int mode,
                   dfuse_solver_stats* stats);

/* ---- device-resident keyframe session (pipeline.hpp:125-228) ---------- */
/* Result of one tracked frame through process_frame (pipeline.hpp:194-228)
 * with keyframe retirement disabled. */
typedef struct {
  int32_t observations;   /* ProcessOutcome::observations */
  int32_t inlier_count;   /* SemiDenseMap::inlier_count after the update */
  int32_t stereo_frames;  /* Keyframe::stereo_frames */
  int32_t optimize_status;/* DFUSE_OK, or the error optimize threw (state unchanged) */
  float stereo_ms;        /* device time of the stereo stage */
  float optimise_ms;      /* device time of the optimise stage */
  dfuse_solver_stats stats;
  int64_t epipolar_steps; /* steps of all epipolar searches of the frame
                             (semidense.hpp:323), for the stereo roofline */
  int32_t solver_ppt;     /* PCG data path of the solve: pixels per thread of
                             the SM-resident tiles, 0 = streaming from L2/HBM */
  int32_t reserved;
} dfuse_frame_result;

/* make_keyframe (pipeline.hpp:125-153) minus prediction I/O: uploads I0 and
 * the six prediction planes, computes the texture mask, empties the
 * semi-dense map and sets the fusion state to init_state(pred). */
int dfuse_kf_create(dfuse_ctx* ctx, const dfuse_intrinsics* K, const float* I0,
                    const double* const pred[6], double texture_threshold, dfuse_keyframe** out);
/* make_keyframe with a DFPRED prediction file already in host memory
 * (pipeline.hpp:133-147): load_predictions' checks (predictions.hpp:69-123;
 * header on the host, same codes and byte offsets in the messages; the
 * variance check on the device, first failure in file order), the size check
 * against K (DimensionMismatch), focal_adjust to K->fx (predictions.hpp:148-157)
 * on the device, then as dfuse_kf_create. The six fp32 planes are copied to
 * HBM as they are (24 B/px) and widened there. */
int dfuse_kf_create_dfpred(dfuse_ctx* ctx, const dfuse_intrinsics* K, const float* I0,
                           const void* dfpred, size_t nbytes, double texture_threshold,
                           dfuse_keyframe** out);
/* DFPRED header checks alone (predictions.hpp:72-95); host code, ctx may be
 * NULL (then no message) */
int dfuse_dfpred_header(dfuse_ctx* ctx, const void* bytes, size_t nbytes, int32_t* width,
                        int32_t* height, double* source_focal);
/* median_predicted_depth (pipeline.hpp:94-99) of the keyframe's predictions,
 * computed once on the device (exact selection) and cached: the per-frame
 * should_create_keyframe test (semidense.hpp:419-424) needs only this and
 * the inlier count */
int dfuse_kf_median_depth(dfuse_keyframe* kf, double* median_depth);
int dfuse_kf_destroy(dfuse_keyframe* kf);

/* ---- row-band keyframe ------------------------ */
/* The keyframe split into `bands` row bands, each with its own planes and
 * one halo row on each side; the stereo stage runs per band, and optimize
 * runs over all bands with halo-row exchange and a two-level all-reduce
 * (band level, then across bands). Here every band lives on this context's
 * device and one cooperative launch runs them all: the single-GPU form of
 * the multi-GPU layout. Same semantics as dfuse_kf_* (make_keyframe /
 * process_frame / download), results within the fusion tolerance of the
 * single-band solve; bands in [1, min(height, SMs)]. */
typedef struct dfuse_banded_keyframe dfuse_banded_keyframe;
int dfuse_bkf_create(dfuse_ctx* ctx, const dfuse_intrinsics* K, const float* I0,
                     const double* const pred[6], double texture_threshold, int bands,
                     dfuse_banded_keyframe** out);
int dfuse_bkf_destroy(dfuse_banded_keyframe* kf);
int dfuse_bkf_reset(dfuse_banded_keyframe* kf);
int dfuse_bkf_process_frame(dfuse_banded_keyframe* kf, const dfuse_epigeom* g, const float* I1,
                            const dfuse_search_cfg* scfg, const dfuse_robust_cfg* rcfg, int mode,
                            dfuse_frame_result* res);
int dfuse_bkf_process_frame_dev(dfuse_banded_keyframe* kf, const dfuse_epigeom* g,
                                const float* I1_dev, const dfuse_search_cfg* scfg,
                                const dfuse_robust_cfg* rcfg, int mode, dfuse_frame_result* res);
int dfuse_bkf_download(dfuse_banded_keyframe* kf, double* log_depth, double* scale,
                       int32_t* iteration, double* semi_depth, double* semi_variance,
                       uint8_t* semi_valid, int32_t* inlier_count, uint8_t* mask);

/* Multi-GPU form (one process per GPU, `world` bands, this process computes
 * band `rank`): create the band, exchange dfuse_band_peer records between the
 * ranks (any transport: torch.distributed all_gather_object in
 * paper_2207_12244_b200/bands_dist.py), connect. The neighbours' halo rows
 * and the level-2 all-reduce arrays are then CUDA-IPC mappings of the peers'
 * band allocations over NVLink, written with system-scope fences; every rank
 * calls process_frame for the same frame and the ranks' kernels meet through
 * those mappings. download returns this rank's rows (and its share of the
 * observation / inlier counts); world == 1 needs no connect. */
typedef struct {
  char handle[64];  /* cudaIpcMemHandle_t of the band allocation */
  int32_t cpr;      /* CTAs per band on that rank (sizes its all-reduce slots) */
  int32_t y0, y1;   /* rows of the band */
  int32_t width;
} dfuse_band_peer;
int dfuse_bkf_create_rank(dfuse_ctx* ctx, const dfuse_intrinsics* K, const float* I0,
                          const double* const pred[6], double texture_threshold, int world,
                          int rank, dfuse_banded_keyframe** out);
int dfuse_bkf_peer_info(dfuse_banded_keyframe* kf, dfuse_band_peer* out);
int dfuse_bkf_connect(dfuse_banded_keyframe* kf, const dfuse_band_peer* peers);
/* diagnostics of the multi-process layout, no solve: _put writes base + i
 * (i = global pixel index) for this rank's two boundary rows into the
 * neighbours' halo rows of halo plane `plane` (0..7: ld0, ld1, x, z, down,
 * p0, p1, 1/var_gy) with the solver's halo stores over the peer mappings;
 * _get reads this rank's own halo rows (y0 - 1 and y1; W doubles each,
 * skipped at the raster edge) */
int dfuse_bkf_debug_halo_put(dfuse_banded_keyframe* kf, int plane, double base);
int dfuse_bkf_debug_halo_get(dfuse_banded_keyframe* kf, int plane, double* above,
                             double* below);

/* ---- scoring (eval.hpp:34-68, 221-226; pipeline.hpp:232-247) --------- */
typedef struct {
  double pct_within_10;   /* KeyframeScore::pct_correct */
  int32_t n_evaluated;    /* valid ground-truth pixels (finalize_keyframe's n_gt) */
  double median_abs_rel;  /* KeyframeScore::median_abs_rel */
} dfuse_keyframe_score;
/* pct_within_10 + median_abs_rel of an estimate in metres against ground
 * truth (host buffers; est_valid may be NULL = every estimate defined).
 * NoValidGroundTruth on an empty ground-truth mask (eval.hpp:45). */
int dfuse_score_depth(dfuse_ctx* ctx, int width, int height, const double* est,
                      const uint8_t* est_valid, const double* gt_metres, const uint8_t* gt_valid,
                      dfuse_keyframe_score* out);
/* finalize_keyframe's score of the session's fused state, est = exp(log_depth)
 * computed on the device (pipeline.hpp:234-247); gt on the host */
int dfuse_kf_score(dfuse_keyframe* kf, const double* gt_metres, const uint8_t* gt_valid,
                   dfuse_keyframe_score* out);
/* export_depth_image's 16-bit raster of the session's fused state:
 * round(exp(log_depth) * depth_scale) clamped to [0, 65535]
 * (eval.hpp:221-226, depth_io.hpp:51-63); PNG encoding is the caller's */
int dfuse_kf_export_depth_u16(dfuse_keyframe* kf, double depth_scale, uint16_t* out);
/* restore the just-created state (device-to-device copies, enqueued on the
 * context's stream like every later call) */
int dfuse_kf_reset(dfuse_keyframe* kf);
/* process_frame for a tracked frame: stereo scan + update + optimize.
 * I1 is a host image (copied in); _dev takes a device pointer. */
int dfuse_kf_process_frame(dfuse_keyframe* kf, const dfuse_epigeom* g, const float* I1,
                           const dfuse_search_cfg* scfg, const dfuse_robust_cfg* rcfg, int mode,
                           dfuse_frame_result* res);
int dfuse_kf_process_frame_dev(dfuse_keyframe* kf, const dfuse_epigeom* g, const float* I1_dev,
                               const dfuse_search_cfg* scfg, const dfuse_robust_cfg* rcfg,
                               int mode, dfuse_frame_result* res);
/* The same for a device image, enqueued on the context's stream without
 * waiting: frames can be submitted back to back (the next frame's stereo
 * uses this frame's semi-dense update, stream order keeps that).
 * dfuse_kf_last_result waits for everything enqueued and returns the last
 * frame's result (stereo_frames counts every enqueued frame). */
int dfuse_kf_process_frame_async(dfuse_keyframe* kf, const dfuse_epigeom* g,
                                 const float* I1_dev, const dfuse_search_cfg* scfg,
                                 const dfuse_robust_cfg* rcfg, int mode);
int dfuse_kf_last_result(dfuse_keyframe* kf, dfuse_frame_result* res);
/* The same for a HOST image, pipelined: the image is copied in on a copy
 * stream while the previous frame computes, and, when log_depth_host is not
 * null, the frame's fused log-depth (W*H doubles, what dfuse_kf_download
 * returns after this frame) is copied out while the next frame computes.
 * Both buffers should be pinned (cudaHostAlloc) for the copies to be
 * asynchronous, and must stay untouched until dfuse_kf_last_result (which
 * also waits for the copies). */
int dfuse_kf_process_frame_host_async(dfuse_keyframe* kf, const dfuse_epigeom* g,
                                      const float* I1_host, const dfuse_search_cfg* scfg,
                                      const dfuse_robust_cfg* rcfg, int mode,
                                      double* log_depth_host);
/* copy state back to the host (any pointer may be NULL) */
int dfuse_kf_download(dfuse_keyframe* kf, double* log_depth, double* scale, int32_t* iteration,
                      double* semi_depth, double* semi_variance, uint8_t* semi_valid,
                      int32_t* inlier_count, uint8_t* mask);

#ifdef __cplusplus
}
#endif

#endif /* DFUSE_CUDA_H */
