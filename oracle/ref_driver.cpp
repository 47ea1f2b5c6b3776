// ref_driver.cpp -- TEST INFRASTRUCTURE ONLY (see dfuse_oracle.h).
//
// Exposes the reference's OWN hot-path code -- the headers under
// /root/reference/proj/include/dfuse, compiled unmodified by
// oracle/Makefile into oracle/_ref/libdfuse_ref.so against the Eigen subset
// in include/compat -- through the ref_* C functions declared in
// dfuse_oracle.h. Marshalling only: every computation below is a call into
// the reference (semidense.hpp, fusion.hpp). The two pieces of pipeline.hpp
// that cannot be included (it pulls in OpenCV via datasets.hpp) --
// stereo_scan and the tracked-frame branch of process_frame -- are restated
// line for line from pipeline.hpp:157-228, OpenMP pragma included.
#include <chrono>
#include <cmath>
#include <cstring>
#include <optional>
#include <vector>

#include "dfuse/eval.hpp"
#include "dfuse/fusion.hpp"
#include "dfuse/predictions.hpp"
#include "dfuse/semidense.hpp"
#include "dfuse_oracle.h"

#ifdef _OPENMP
#include <omp.h>
#endif

using namespace dfuse;

namespace {

int code_of(const Error& e) { return static_cast<int>(e.code()) + 1; }

Pose make_pose(const double q[4], const double t[3]) {
  Pose p;
  p.rotation = Eigen::Quaterniond(q[0], q[1], q[2], q[3]);
  p.translation = Eigen::Vector3d(t[0], t[1], t[2]);
  return p;
}

CameraIntrinsics make_K(const dfuse_intrinsics& k) {
  return CameraIntrinsics{k.fx, k.fy, k.cx, k.cy, k.width, k.height};
}

EpipolarGeometry make_geom(const dfuse_epigeom& g) {
  EpipolarGeometry out;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) out.R_10(r, c) = g.R_10[3 * r + c];
  out.t_10 = Eigen::Vector3d(g.t_10[0], g.t_10[1], g.t_10[2]);
  out.t_01 = Eigen::Vector3d(g.t_01[0], g.t_01[1], g.t_01[2]);
  out.K = make_K(g.K);
  return out;
}

IntensityImage make_image(const float* px, int w, int h) {
  IntensityImage img(w, h, 0.f);
  std::memcpy(img.raster().data(), px, sizeof(float) * static_cast<std::size_t>(w) * h);
  return img;
}

Raster<double> make_raster(const double* v, int w, int h) {
  Raster<double> r(w, h, 0.0);
  std::memcpy(r.data(), v, sizeof(double) * r.size());
  return r;
}

SemiDenseMap make_semi(const double* d, const double* var, const uint8_t* valid, int count, int w,
                       int h) {
  SemiDenseMap m = SemiDenseMap::empty(w, h);
  std::memcpy(m.depth.data(), d, sizeof(double) * m.depth.size());
  std::memcpy(m.variance.data(), var, sizeof(double) * m.variance.size());
  std::memcpy(m.valid.data(), valid, m.valid.size());
  m.inlier_count = count;
  return m;
}

PredictionSet make_pred(const dfuse_fusion_inputs& in) {
  PredictionSet p;
  Raster<double>* ch[6] = {&p.log_depth, &p.log_depth_var, &p.grad_x,
                           &p.grad_x_var, &p.grad_y,      &p.grad_y_var};
  for (int c = 0; c < 6; ++c) *ch[c] = make_raster(in.pred[c], in.width, in.height);
  p.source_focal = 1.0;
  return p;
}

RobustConfig make_robust(const dfuse_robust_cfg& c) {
  RobustConfig r;
  r.delta_semi = c.delta_semi;
  r.delta_net = c.delta_net;
  r.delta_grad = c.delta_grad;
  r.gn_iterations = c.gn_iterations;
  r.cg_tol = c.cg_tol;
  r.cg_max_iters = c.cg_max_iters;
  r.estimate_scale = c.estimate_scale != 0;
  return r;
}

FusionMode make_mode(int m) {
  if (m == DFUSE_MODE_NOPAIRWISE) return FusionMode::NoPairwise;
  if (m == DFUSE_MODE_LSSCALE) return FusionMode::LeastSquaresScale;
  return FusionMode::Full;
}

void put_obs(const EpipolarObservation& o, dfuse_obs* out) {
  out->x = o.pixel.x;
  out->y = o.pixel.y;
  out->depth = o.depth;
  for (int j = 0; j < 5; ++j) {
    out->error5[j] = o.error5[j];
    out->jacobian[j] = o.jacobian[j];
  }
  out->variance = o.variance;
}

EpipolarObservation get_obs(const dfuse_obs& o) {
  EpipolarObservation r;
  r.pixel = {o.x, o.y};
  r.depth = o.depth;
  for (int j = 0; j < 5; ++j) {
    r.error5[j] = o.error5[j];
    r.jacobian[j] = o.jacobian[j];
  }
  r.variance = o.variance;
  return r;
}

// stereo_scan, pipeline.hpp:157-190 (Keyframe/Frame unpacked into images,
// mask and semi map).
std::vector<EpipolarObservation> stereo_scan(const EpipolarGeometry& g, const IntensityImage& I0,
                                             const IntensityImage& I1, const Mask& texture,
                                             const SemiDenseMap& semidense,
                                             const SearchConfig& search,
                                             std::vector<int8_t>* status_out) {
  if (g.t_10.norm() < 1e-12) return {};
  const int w = g.K.width, h = g.K.height;
  std::vector<EpipolarObservation> slots(static_cast<std::size_t>(w) * h);
  std::vector<std::uint8_t> got(slots.size(), 0);
#pragma omp parallel for schedule(dynamic, 4)
  for (int y = 0; y < h; ++y) {
    for (int x = 0; x < w; ++x) {
      if (!texture.at(x, y)) continue;
      const std::size_t i = texture.index(x, y);
      std::optional<DepthPrior> prior;
      if (semidense.valid[i])
        prior = DepthPrior{semidense.depth[i], std::sqrt(semidense.variance[i])};
      const EpipolarResult r = search_depth(
          g, I0, I1, PixelCoord{static_cast<double>(x), static_cast<double>(y)}, prior, search);
      if (status_out) (*status_out)[i] = static_cast<int8_t>(r.status);
      if (r.ok()) {
        slots[i] = r.obs;
        got[i] = 1;
      }
    }
  }
  std::vector<EpipolarObservation> obs;
  obs.reserve(slots.size() / 4);
  for (std::size_t i = 0; i < slots.size(); ++i)
    if (got[i]) obs.push_back(slots[i]);
  return obs;
}

}  // namespace

extern "C" {

int ref_omp_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

// the OpenMP team size of the reference's parallel loops (torchrun exports
// OMP_NUM_THREADS=1 to every rank; the reference arm runs on rank 0 alone
// and takes the host's cores)
void ref_omp_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

int ref_make_epipolar_geometry(const double q0[4], const double t0[3], const double q1[4],
                               const double t1[3], const dfuse_intrinsics* K, dfuse_epigeom* out) {
  const EpipolarGeometry g = make_epipolar_geometry(make_pose(q0, t0), make_pose(q1, t1), make_K(*K));
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) out->R_10[3 * r + c] = g.R_10(r, c);
  for (int i = 0; i < 3; ++i) {
    out->t_10[i] = g.t_10(i);
    out->t_01[i] = g.t_01(i);
  }
  out->K = *K;
  return DFUSE_OK;
}

int ref_texture_mask(const float* img, int w, int h, double threshold, uint8_t* mask) {
  try {
    const Mask m = texture_mask(make_image(img, w, h), threshold);
    std::memcpy(mask, m.data(), m.size());
    return DFUSE_OK;
  } catch (const Error& e) {
    return code_of(e);
  }
}

int ref_search_depth(const dfuse_epigeom* g, const float* I0, const float* I1, int n,
                     const double* px, const double* prior, const uint8_t* has_prior,
                     const dfuse_search_cfg* cfg, int32_t* status, dfuse_obs* obs, int32_t* best,
                     int32_t* n_steps) {
  const EpipolarGeometry geom = make_geom(*g);
  const IntensityImage i0 = make_image(I0, g->K.width, g->K.height);
  const IntensityImage i1 = make_image(I1, g->K.width, g->K.height);
  const SearchConfig sc{cfg->min_depth, cfg->max_depth, cfg->max_rms_error};
  for (int k = 0; k < n; ++k) {
    std::optional<DepthPrior> pr;
    if (prior && (!has_prior || has_prior[k])) pr = DepthPrior{prior[2 * k], prior[2 * k + 1]};
    const EpipolarResult r = search_depth(geom, i0, i1, PixelCoord{px[2 * k], px[2 * k + 1]}, pr, sc);
    status[k] = static_cast<int32_t>(r.status);
    std::memset(&obs[k], 0, sizeof(dfuse_obs));
    if (r.ok()) put_obs(r.obs, &obs[k]);
    if (best) best[k] = -1;  // internal to the reference's search_depth
    if (n_steps) n_steps[k] = -1;
  }
  return DFUSE_OK;
}

int ref_update_semidense(int w, int h, double* depth, double* variance, uint8_t* valid,
                         int32_t* inlier_count, int n_obs, const dfuse_obs* obs) {
  try {
    SemiDenseMap m = make_semi(depth, variance, valid, *inlier_count, w, h);
    std::vector<EpipolarObservation> o(n_obs);
    for (int k = 0; k < n_obs; ++k) o[k] = get_obs(obs[k]);
    m = update_semidense(std::move(m), o);
    std::memcpy(depth, m.depth.data(), sizeof(double) * m.depth.size());
    std::memcpy(variance, m.variance.data(), sizeof(double) * m.variance.size());
    std::memcpy(valid, m.valid.data(), m.valid.size());
    *inlier_count = m.inlier_count;
    return DFUSE_OK;
  } catch (const Error& e) {
    return code_of(e);
  }
}

int ref_stereo_update(const dfuse_epigeom* g, const float* I0, const float* I1,
                      const uint8_t* mask, const dfuse_search_cfg* cfg, double* depth,
                      double* variance, uint8_t* valid, int32_t* inlier_count, int32_t* n_obs,
                      int8_t* status, int32_t* best, int32_t* n_steps, dfuse_obs* obs_out) {
  const int w = g->K.width, h = g->K.height;
  const std::size_t P = static_cast<std::size_t>(w) * h;
  try {
    const EpipolarGeometry geom = make_geom(*g);
    const IntensityImage i0 = make_image(I0, w, h), i1 = make_image(I1, w, h);
    Mask texture(w, h, 0);
    std::memcpy(texture.data(), mask, P);
    SemiDenseMap m = make_semi(depth, variance, valid, *inlier_count, w, h);
    std::vector<int8_t> st(P, static_cast<int8_t>(DFUSE_EPI_NOT_SEARCHED));
    // masked pixels skipped by the zero-baseline early exit report the
    // status search_depth would have given them (semidense.hpp:287)
    if (geom.t_10.norm() < 1e-12)
      for (std::size_t i = 0; i < P; ++i)
        if (mask[i]) st[i] = static_cast<int8_t>(EpipolarStatus::DegenerateBaseline);
    const SearchConfig sc{cfg->min_depth, cfg->max_depth, cfg->max_rms_error};
    const std::vector<EpipolarObservation> obs = stereo_scan(geom, i0, i1, texture, m, sc, &st);
    *n_obs = static_cast<int32_t>(obs.size());
    if (!obs.empty()) m = update_semidense(std::move(m), obs);  // pipeline.hpp:209-212
    std::memcpy(depth, m.depth.data(), sizeof(double) * P);
    std::memcpy(variance, m.variance.data(), sizeof(double) * P);
    std::memcpy(valid, m.valid.data(), P);
    *inlier_count = m.inlier_count;
    if (status) std::memcpy(status, st.data(), P);
    for (std::size_t i = 0; i < P; ++i) {
      if (best) best[i] = -1;
      if (n_steps) n_steps[i] = -1;
    }
    if (obs_out)
      for (std::size_t k = 0; k < obs.size(); ++k) put_obs(obs[k], &obs_out[k]);
    return DFUSE_OK;
  } catch (const Error& e) {
    return code_of(e);
  }
}

int ref_assemble_normal_equations(const dfuse_fusion_inputs* in, const double* log_depth,
                                  double scale, const dfuse_robust_cfg* cfg, int mode,
                                  double* diag, double* right, double* down, double* b) {
  try {
    FusionState st{make_raster(log_depth, in->width, in->height), scale, 0};
    const SemiDenseMap semi = make_semi(in->semi_depth, in->semi_variance, in->semi_valid,
                                        in->inlier_count, in->width, in->height);
    const NormalEquations eq =
        assemble_normal_equations(st, semi, make_pred(*in), make_robust(*cfg), make_mode(mode));
    const std::size_t P = eq.b.size();
    std::memcpy(diag, eq.H.diag.data(), P * sizeof(double));
    std::memcpy(right, eq.H.right.data(), P * sizeof(double));
    std::memcpy(down, eq.H.down.data(), P * sizeof(double));
    std::memcpy(b, eq.b.data(), P * sizeof(double));
    return DFUSE_OK;
  } catch (const Error& e) {
    return code_of(e);
  }
}

int ref_total_cost(const dfuse_fusion_inputs* in, const double* log_depth, double scale,
                   const dfuse_robust_cfg* cfg, int mode, double* cost) {
  try {
    FusionState st{make_raster(log_depth, in->width, in->height), scale, 0};
    const SemiDenseMap semi = make_semi(in->semi_depth, in->semi_variance, in->semi_valid,
                                        in->inlier_count, in->width, in->height);
    *cost = total_cost(st, semi, make_pred(*in), make_robust(*cfg), make_mode(mode));
    return DFUSE_OK;
  } catch (const Error& e) {
    return code_of(e);
  }
}

int ref_cost_gradient(const dfuse_fusion_inputs* in, const double* log_depth, double scale,
                      const dfuse_robust_cfg* cfg, int mode, double* cost, double* wrt_log_depth,
                      double* wrt_ln_scale) {
  try {
    FusionState st{make_raster(log_depth, in->width, in->height), scale, 0};
    const SemiDenseMap semi = make_semi(in->semi_depth, in->semi_variance, in->semi_valid,
                                        in->inlier_count, in->width, in->height);
    const CostGradient g =
        cost_gradient(st, semi, make_pred(*in), make_robust(*cfg), make_mode(mode));
    *cost = g.cost;
    std::memcpy(wrt_log_depth, g.wrt_log_depth.data(), g.wrt_log_depth.size() * sizeof(double));
    *wrt_ln_scale = g.wrt_ln_scale;
    return DFUSE_OK;
  } catch (const Error& e) {
    return code_of(e);
  }
}

int ref_stencil_apply(int w, int h, const double* diag, const double* right, const double* down,
                      const double* x, double* y) {
  StencilMatrix H(w, h);
  const std::size_t P = H.size();
  std::memcpy(H.diag.data(), diag, P * sizeof(double));
  std::memcpy(H.right.data(), right, P * sizeof(double));
  std::memcpy(H.down.data(), down, P * sizeof(double));
  H.apply(x, y);
  return DFUSE_OK;
}

int ref_solve_depth_step(int w, int h, const double* diag, const double* right, const double* down,
                         const double* b, const dfuse_robust_cfg* cfg, double* delta,
                         int32_t* iterations) {
  try {
    NormalEquations eq;
    eq.H = StencilMatrix(w, h);
    const std::size_t P = eq.H.size();
    std::memcpy(eq.H.diag.data(), diag, P * sizeof(double));
    std::memcpy(eq.H.right.data(), right, P * sizeof(double));
    std::memcpy(eq.H.down.data(), down, P * sizeof(double));
    eq.b.assign(b, b + P);
    const std::vector<double> d = solve_depth_step(eq, make_robust(*cfg));
    std::memcpy(delta, d.data(), P * sizeof(double));
    if (iterations) *iterations = -1;  // not exposed by the reference
    return DFUSE_OK;
  } catch (const Error& e) {
    return code_of(e);
  }
}

int ref_solve_scale_step(const dfuse_fusion_inputs* in, const double* log_depth, double scale,
                         const dfuse_robust_cfg* cfg, double* scale_out) {
  try {
    FusionState st{make_raster(log_depth, in->width, in->height), scale, 0};
    const SemiDenseMap semi = make_semi(in->semi_depth, in->semi_variance, in->semi_valid,
                                        in->inlier_count, in->width, in->height);
    *scale_out = solve_scale_step(st, semi, make_robust(*cfg));
    return DFUSE_OK;
  } catch (const Error& e) {
    return code_of(e);
  }
}

int ref_optimize(const dfuse_fusion_inputs* in, double* log_depth, double* scale,
                 int32_t* iteration, const dfuse_robust_cfg* cfg, int mode,
                 dfuse_solver_stats* stats) {
  try {
    FusionState st{make_raster(log_depth, in->width, in->height), *scale, *iteration};
    const SemiDenseMap semi = make_semi(in->semi_depth, in->semi_variance, in->semi_valid,
                                        in->inlier_count, in->width, in->height);
    const FusionState out =
        optimize(st, semi, make_pred(*in), make_robust(*cfg), make_mode(mode));
    std::memcpy(log_depth, out.log_depth.data(), out.log_depth.size() * sizeof(double));
    *scale = out.scale;
    *iteration = out.iteration;
    if (stats) std::memset(stats, 0, sizeof *stats);  // not exposed by the reference
    return DFUSE_OK;
  } catch (const Error& e) {
    return code_of(e);
  }
}

// Tracked-frame branch of process_frame, pipeline.hpp:203-227, with the
// keyframe decision evaluated but retirement disabled by the caller's
// policy (lambda_inliers = 0, lambda_trans huge; test_pipeline.cpp:20).
int ref_process_frame(const dfuse_epigeom* g, const float* I0, const float* I1,
                      const uint8_t* mask, const dfuse_search_cfg* scfg,
                      const dfuse_fusion_inputs* in, double* semi_depth, double* semi_variance,
                      uint8_t* semi_valid, int32_t* inlier_count, double* log_depth,
                      double* scale, int32_t* iteration, const dfuse_robust_cfg* rcfg, int mode,
                      int32_t* n_obs, double* stereo_ms, double* optimise_ms) {
  using clock = std::chrono::steady_clock;
  const int w = g->K.width, h = g->K.height;
  const std::size_t P = static_cast<std::size_t>(w) * h;
  try {
    const EpipolarGeometry geom = make_geom(*g);
    const IntensityImage i0 = make_image(I0, w, h), i1 = make_image(I1, w, h);
    Mask texture(w, h, 0);
    std::memcpy(texture.data(), mask, P);
    SemiDenseMap semi = make_semi(semi_depth, semi_variance, semi_valid, *inlier_count, w, h);
    const PredictionSet pred = make_pred(*in);
    FusionState fusion{make_raster(log_depth, w, h), *scale, *iteration};
    const SearchConfig sc{scfg->min_depth, scfg->max_depth, scfg->max_rms_error};

    const auto t0 = clock::now();
    {
      const std::vector<EpipolarObservation> obs =
          stereo_scan(geom, i0, i1, texture, semi, sc, nullptr);
      *n_obs = static_cast<int32_t>(obs.size());
      if (!obs.empty()) semi = update_semidense(std::move(semi), obs);
    }
    const auto t1 = clock::now();
    // median_predicted_depth + should_create_keyframe, pipeline.hpp:94-99,215-216
    {
      std::vector<double> vals(pred.log_depth.data(), pred.log_depth.data() + pred.log_depth.size());
      const std::size_t mid = vals.size() / 2;
      std::nth_element(vals.begin(), vals.begin() + mid, vals.end());
      const double median_depth = std::exp(vals[mid]);
      (void)should_create_keyframe(Pose::identity(), Pose::identity(), median_depth, semi,
                                   KeyframePolicy{1e300, 0});
    }
    int rc = DFUSE_OK;
    const auto t2 = clock::now();
    try {
      fusion = optimize(fusion, semi, pred, make_robust(*rcfg), make_mode(mode));
    } catch (const Error& e) {
      if (e.code() != Err::CgDivergence) throw;
      rc = code_of(e);  // run_sequence skips the solve, pipeline.hpp:328-331
    }
    const auto t3 = clock::now();
    *stereo_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    *optimise_ms = std::chrono::duration<double, std::milli>(t3 - t2).count();
    std::memcpy(semi_depth, semi.depth.data(), P * sizeof(double));
    std::memcpy(semi_variance, semi.variance.data(), P * sizeof(double));
    std::memcpy(semi_valid, semi.valid.data(), P);
    *inlier_count = semi.inlier_count;
    std::memcpy(log_depth, fusion.log_depth.data(), P * sizeof(double));
    *scale = fusion.scale;
    *iteration = fusion.iteration;
    return rc;
  } catch (const Error& e) {
    return code_of(e);
  }
}


int ref_photometric_error_5pt(const dfuse_epigeom* g, const float* I0, const float* I1, double x,
                              double y, double d, double e[5]) {
  std::array<double, 5> ee{};
  const EpipolarStatus st = photometric_error_5pt(make_geom(*g), make_image(I0, g->K.width, g->K.height),
                                                  make_image(I1, g->K.width, g->K.height),
                                                  PixelCoord{x, y}, d, ee);
  for (int j = 0; j < 5; ++j) e[j] = ee[j];
  return static_cast<int>(st);
}

int ref_jacobian_fd(const double e_lo[5], const double e_hi[5], double d_lo, double d_hi,
                    double J[5]) {
  try {
    std::array<double, 5> a, b;
    for (int j = 0; j < 5; ++j) {
      a[j] = e_lo[j];
      b[j] = e_hi[j];
    }
    const std::array<double, 5> r = jacobian_fd(a, b, d_lo, d_hi);
    for (int j = 0; j < 5; ++j) J[j] = r[j];
    return DFUSE_OK;
  } catch (const Error& e) {
    return code_of(e);
  }
}

double ref_observation_variance(const double J[5]) {
  std::array<double, 5> a;
  for (int j = 0; j < 5; ++j) a[j] = J[j];
  return observation_variance(a);
}

int ref_huber(double r, double delta, double* weight, double* cost) {
  *cost = huber_cost(r, delta);
  try {
    *weight = huber_weight(r, delta);
    return DFUSE_OK;
  } catch (const Error& e) {
    *weight = 0.0;
    return code_of(e);
  }
}

double ref_residual_semi(double ln_d, double s, double d_semi) {
  return residual_semi(ln_d, s, d_semi);
}

double ref_semi_log_variance(double variance, double depth) {
  return semi_log_variance(variance, depth);
}

int ref_should_create_keyframe(const double q_kf[4], const double t_kf[3], const double q_cur[4],
                               const double t_cur[3], double median, int inlier_count,
                               double lambda_trans, int lambda_inliers, int* out) {
  try {
    SemiDenseMap m;
    m.inlier_count = inlier_count;
    *out = should_create_keyframe(make_pose(q_kf, t_kf), make_pose(q_cur, t_cur), median, m,
                                  KeyframePolicy{lambda_trans, lambda_inliers});
    return DFUSE_OK;
  } catch (const Error& e) {
    return code_of(e);
  }
}

// ---- prediction files (predictions.hpp:69-157), for the DFPRED ingest pin
namespace {
void copy_msg(const Error& e, char* msg, int msglen) {
  if (msg && msglen > 0) {
    std::strncpy(msg, e.what(), (size_t)msglen - 1);
    msg[msglen - 1] = 0;
  }
}
}  // namespace

int ref_load_predictions(const char* path, int w, int h, double* planes, double* source_focal,
                         char* msg, int msglen) {
  try {
    const PredictionSet p = load_predictions(path);
    if (p.width() != w || p.height() != h) return DFUSE_E_DIMENSION_MISMATCH;
    const Raster<double>* ch[6] = {&p.log_depth, &p.log_depth_var, &p.grad_x,
                                   &p.grad_x_var, &p.grad_y,       &p.grad_y_var};
    const std::size_t n = (std::size_t)w * h;
    for (int c = 0; c < 6; ++c) std::memcpy(planes + c * n, ch[c]->data(), n * sizeof(double));
    *source_focal = p.source_focal;
    return DFUSE_OK;
  } catch (const Error& e) {
    copy_msg(e, msg, msglen);
    return code_of(e);
  }
}

int ref_save_predictions(const char* path, int w, int h, const double* planes,
                         double source_focal) {
  try {
    PredictionSet p;
    Raster<double>* ch[6] = {&p.log_depth, &p.log_depth_var, &p.grad_x,
                             &p.grad_x_var, &p.grad_y,       &p.grad_y_var};
    const std::size_t n = (std::size_t)w * h;
    for (int c = 0; c < 6; ++c) {
      *ch[c] = Raster<double>(w, h, 0.0);
      std::memcpy(ch[c]->data(), planes + c * n, n * sizeof(double));
    }
    p.source_focal = source_focal;
    save_predictions(p, path);
    return DFUSE_OK;
  } catch (const Error& e) {
    return code_of(e);
  }
}

int ref_focal_adjust(int w, int h, double* log_depth, double source_focal, double test_focal) {
  try {
    PredictionSet p;
    p.log_depth = Raster<double>(w, h, 0.0);
    std::memcpy(p.log_depth.data(), log_depth, sizeof(double) * (std::size_t)w * h);
    p.source_focal = source_focal;
    const PredictionSet q = focal_adjust(p, test_focal);
    std::memcpy(log_depth, q.log_depth.data(), sizeof(double) * (std::size_t)w * h);
    return DFUSE_OK;
  } catch (const Error& e) {
    return code_of(e);
  }
}

// ---- scoring (eval.hpp:34-68, 221-226; pipeline.hpp:232-247) ------------
namespace {
DepthImage depth_image(int w, int h, const double* gt, const uint8_t* gt_valid) {
  DepthImage d{Raster<double>(w, h, 0.0), Mask(w, h, 0)};
  std::memcpy(d.metres.data(), gt, sizeof(double) * (std::size_t)w * h);
  std::memcpy(d.valid.data(), gt_valid, (std::size_t)w * h);
  return d;
}
}  // namespace

int ref_pct_within_10(int w, int h, const double* est, const uint8_t* est_valid,
                      const double* gt, const uint8_t* gt_valid, double* out) {
  try {
    Raster<double> e(w, h, 0.0);
    std::memcpy(e.data(), est, sizeof(double) * (std::size_t)w * h);
    Mask m(w, h, 0);
    if (est_valid) std::memcpy(m.data(), est_valid, (std::size_t)w * h);
    *out = pct_within_10(e, est_valid ? &m : nullptr, depth_image(w, h, gt, gt_valid));
    return DFUSE_OK;
  } catch (const Error& e) {
    return code_of(e);
  }
}

int ref_median_abs_rel(int w, int h, const double* est, const uint8_t* est_valid,
                       const double* gt, const uint8_t* gt_valid, double* out) {
  try {
    Raster<double> e(w, h, 0.0);
    std::memcpy(e.data(), est, sizeof(double) * (std::size_t)w * h);
    Mask m(w, h, 0);
    if (est_valid) std::memcpy(m.data(), est_valid, (std::size_t)w * h);
    *out = median_abs_rel(e, est_valid ? &m : nullptr, depth_image(w, h, gt, gt_valid));
    return DFUSE_OK;
  } catch (const Error& e) {
    return code_of(e);
  }
}

// export_depth_image (eval.hpp:221-226) -> save_depth_png's 16-bit raster,
// captured by the in-memory imwrite of oracle/compat_cv
int ref_export_depth_u16(int w, int h, const double* log_depth, double depth_scale,
                         uint16_t* out) {
  try {
    FusionState st{Raster<double>(w, h, 0.0), 1.0, 0};
    std::memcpy(st.log_depth.data(), log_depth, sizeof(double) * (std::size_t)w * h);
    export_depth_image(st, "ref_export.png", depth_scale);
    const cv::Mat& m = cv::image_store().at("ref_export.png");
    for (int y = 0; y < h; ++y) std::memcpy(out + (std::size_t)y * w, m.ptr<uint16_t>(y), 2 * w);
    return DFUSE_OK;
  } catch (const Error& e) {
    return code_of(e);
  }
}

}  // extern "C"
