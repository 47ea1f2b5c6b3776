/*
 * dfuse_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference's hot path, used as the parity checker
 * for the CUDA implementation. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it; the product path
 * (paper_2207_12244_b200/) never links or calls it.
 *
 * Two libraries export this exact function set:
 *   orc_*  oracle/dfuse_oracle.c  -- plain-C restatement, single thread
 *   ref_*  oracle/ref_driver.cpp  -- the reference's own headers from
 *          /root/reference/proj/include compiled unmodified (+ OpenMP)
 *          against include/compat/Eigen; built into oracle/_ref/.
 * tests/test_oracle_pin.py checks orc_* == ref_* bit for bit on seeded
 * inputs, which pins the restatement to the reference.
 *
 * Types and error codes are those of include/dfuse_cuda.h.
 */
#ifndef DFUSE_ORACLE_H
#define DFUSE_ORACLE_H

#include "../include/dfuse_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

#define DFUSE_ORACLE_DECLS(P)                                                                     \
  int P##make_epipolar_geometry(const double q0_wxyz[4], const double t0[3],                     \
                                const double q1_wxyz[4], const double t1[3],                     \
                                const dfuse_intrinsics* K, dfuse_epigeom* out);                  \
  int P##texture_mask(const float* img, int width, int height, double threshold, uint8_t* mask); \
  int P##search_depth(const dfuse_epigeom* g, const float* I0, const float* I1, int n,           \
                      const double* px, const double* prior, const uint8_t* has_prior,          \
                      const dfuse_search_cfg* cfg, int32_t* status, dfuse_obs* obs,             \
                      int32_t* best, int32_t* n_steps);                                          \
  int P##update_semidense(int width, int height, double* depth, double* variance,               \
                          uint8_t* valid, int32_t* inlier_count, int n_obs,                     \
                          const dfuse_obs* obs);                                                 \
  int P##stereo_update(const dfuse_epigeom* g, const float* I0, const float* I1,                 \
                       const uint8_t* mask, const dfuse_search_cfg* cfg, double* depth,         \
                       double* variance, uint8_t* valid, int32_t* inlier_count, int32_t* n_obs, \
                       int8_t* status, int32_t* best, int32_t* n_steps, dfuse_obs* obs);        \
  int P##assemble_normal_equations(const dfuse_fusion_inputs* in, const double* log_depth,      \
                                   double scale, const dfuse_robust_cfg* cfg, int mode,         \
                                   double* diag, double* right, double* down, double* b);       \
  int P##total_cost(const dfuse_fusion_inputs* in, const double* log_depth, double scale,       \
                    const dfuse_robust_cfg* cfg, int mode, double* cost);                       \
  int P##cost_gradient(const dfuse_fusion_inputs* in, const double* log_depth, double scale,    \
                       const dfuse_robust_cfg* cfg, int mode, double* cost,                     \
                       double* wrt_log_depth, double* wrt_ln_scale);                            \
  int P##stencil_apply(int width, int height, const double* diag, const double* right,          \
                       const double* down, const double* x, double* y);                         \
  int P##solve_depth_step(int width, int height, const double* diag, const double* right,       \
                          const double* down, const double* b, const dfuse_robust_cfg* cfg,     \
                          double* delta, int32_t* iterations);                                  \
  int P##solve_scale_step(const dfuse_fusion_inputs* in, const double* log_depth, double scale, \
                          const dfuse_robust_cfg* cfg, double* scale_out);                      \
  int P##optimize(const dfuse_fusion_inputs* in, double* log_depth, double* scale,              \
                  int32_t* iteration, const dfuse_robust_cfg* cfg, int mode,                    \
                  dfuse_solver_stats* stats);

DFUSE_ORACLE_DECLS(orc_)
DFUSE_ORACLE_DECLS(ref_)

/* small helpers the reference exposes for its KATs (semidense.hpp:227-272,
 * fusion.hpp:51-100); same signatures under both prefixes */
#define DFUSE_ORACLE_HELPERS(P)                                                                   \
  int P##photometric_error_5pt(const dfuse_epigeom* g, const float* I0, const float* I1,         \
                               double x, double y, double d, double e[5]);                       \
  int P##jacobian_fd(const double e_lo[5], const double e_hi[5], double d_lo, double d_hi,      \
                     double J[5]);                                                               \
  double P##observation_variance(const double J[5]);                                             \
  int P##huber(double r, double delta, double* weight, double* cost);                           \
  double P##residual_semi(double ln_d, double s, double d_semi);                                 \
  double P##semi_log_variance(double variance, double depth);                                    \
  int P##should_create_keyframe(const double q_kf[4], const double t_kf[3],                     \
                                const double q_cur[4], const double t_cur[3], double median,    \
                                int inlier_count, double lambda_trans, int lambda_inliers,      \
                                int* out);
DFUSE_ORACLE_HELPERS(orc_)
DFUSE_ORACLE_HELPERS(ref_)
double orc_hypot(double x, double y);

/* ref_ only: one tracked frame through the reference's process_frame
 * (pipeline.hpp:194-228) with retirement disabled, timed per stage like
 * StageTimer (pipeline.hpp:101-115). Returns the optimize error code (the
 * fusion state is unchanged on error, as in run_sequence). */
int ref_process_frame(const dfuse_epigeom* g, const float* I0, const float* I1,
                      const uint8_t* mask, const dfuse_search_cfg* scfg,
                      const dfuse_fusion_inputs* in_pred_only, double* semi_depth,
                      double* semi_variance, uint8_t* semi_valid, int32_t* inlier_count,
                      double* log_depth, double* scale, int32_t* iteration,
                      const dfuse_robust_cfg* rcfg, int mode, int32_t* n_obs,
                      double* stereo_ms, double* optimise_ms);
int ref_omp_max_threads(void);

/* focal_adjust (predictions.hpp:148-157), median_predicted_depth
 * (pipeline.hpp:94-99) */
int orc_focal_adjust(int w, int h, double* log_depth, double source_focal, double test_focal);
double orc_median_predicted_depth(const double* log_depth, long n);

/* scoring: pct_within_10, median_abs_rel (eval.hpp:34-68), export_depth_image
 * quantisation (eval.hpp:221-226, depth_io.hpp:51-63) */
int orc_pct_within_10(long n, const double* est, const uint8_t* est_valid, const double* gt,
                      const uint8_t* gt_valid, double* out);
double orc_median_abs_rel(long n, const double* est, const uint8_t* est_valid, const double* gt,
                          const uint8_t* gt_valid);
void orc_export_depth_u16(long n, const double* log_depth, double depth_scale, uint16_t* out);

#ifdef __cplusplus
}
#endif

#endif
