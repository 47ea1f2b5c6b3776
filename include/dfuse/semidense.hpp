// dfuse/semidense.hpp -- drop-in for proj/include/dfuse/semidense.hpp:18-424.
//
// Same types, names and signatures. texture_mask, search_depth,
// photometric_error_5pt and update_semidense run on the GPU through the
// C-ABI (include/dfuse_cuda.h); make_epipolar_geometry, epipolar_segment,
// jacobian_fd, observation_variance and should_create_keyframe are the
// per-frame-pair / per-5-vector scalar helpers and stay inline host math.
// For whole frames use search_depth_batch (one launch for many pixels) or
// the device-resident session in dfuse/session.hpp.
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <optional>
#include <utility>
#include <vector>

#include "dfuse/device.hpp"
#include "dfuse/geometry.hpp"
#include "dfuse/image.hpp"
#include "dfuse/raster.hpp"

namespace dfuse {

struct SemiDenseMap {
  Raster<double> depth;
  Raster<double> variance;
  Mask valid;
  int inlier_count = 0;

  static SemiDenseMap empty(int width, int height) {
    return {Raster<double>(width, height, 0.0), Raster<double>(width, height, 0.0),
            Mask(width, height, 0), 0};
  }
};

struct KeyframePolicy {
  double lambda_trans = 0.07;
  int lambda_inliers = 1500;
};

struct EpipolarObservation {
  PixelCoord pixel;
  double depth = 0.0;
  std::array<double, 5> error5{};
  std::array<double, 5> jacobian{};
  double variance = 0.0;
};
static_assert(sizeof(EpipolarObservation) == sizeof(dfuse_obs), "observation layout");

enum class EpipolarStatus {
  Ok,
  DegenerateBaseline,
  OutOfBounds,
  BehindCamera,
  NoMinimum,
  DegenerateJacobian,
};

struct EpipolarResult {
  EpipolarStatus status = EpipolarStatus::Ok;
  EpipolarObservation obs;
  bool ok() const { return status == EpipolarStatus::Ok; }
};

struct DepthPrior {
  double depth = 0.0;
  double sigma = 0.0;
};

struct SearchConfig {
  double min_depth = 0.25;
  double max_depth = 50.0;
  double max_rms_error = 0.05;
  dfuse_search_cfg c_abi() const { return {min_depth, max_depth, max_rms_error}; }
};

inline Mask texture_mask(const IntensityImage& img, double threshold) {
  Mask m(img.width(), img.height(), 0);
  device::check(dfuse_texture_mask(device::ctx(), img.raster().data(), img.width(), img.height(),
                                   threshold, m.data()),
                "texture_mask");
  return m;
}

struct EpipolarGeometry {
  Eigen::Matrix3d R_10;
  Eigen::Vector3d t_10;
  Eigen::Vector3d t_01;
  CameraIntrinsics K;

  dfuse_epigeom c_abi() const {
    dfuse_epigeom g;
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) g.R_10[3 * r + c] = R_10(r, c);
    for (int i = 0; i < 3; ++i) {
      g.t_10[i] = t_10(i);
      g.t_01[i] = t_01(i);
    }
    g.K = K.c_abi();
    return g;
  }
};

// host-side, with the caller's Eigen: bit-identical to the reference's own
// computation of the per-frame-pair geometry
inline EpipolarGeometry make_epipolar_geometry(const Pose& T0, const Pose& T1,
                                               const CameraIntrinsics& K) {
  const Pose T10 = compose(T1.inverse(), T0);
  const Pose T01 = compose(T0.inverse(), T1);
  return {T10.rotation.toRotationMatrix(), T10.translation, T01.translation, K};
}

inline std::optional<std::pair<PixelCoord, PixelCoord>> epipolar_segment(
    const EpipolarGeometry& g, const PixelCoord& x, double d_lo, double d_hi) {
  const Eigen::Vector3d ray((x.x - g.K.cx) / g.K.fx, (x.y - g.K.cy) / g.K.fy, 1.0);
  const Eigen::Vector3d a = g.R_10 * ray;
  auto proj = [&](double d) -> std::optional<PixelCoord> {
    const Eigen::Vector3d p = d * a + g.t_10;
    if (p.z() <= 0.0) return std::nullopt;
    return PixelCoord{g.K.fx * p.x() / p.z() + g.K.cx, g.K.fy * p.y() / p.z() + g.K.cy};
  };
  const auto lo = proj(d_lo), hi = proj(d_hi);
  if (!lo || !hi) return std::nullopt;
  return std::make_pair(*lo, *hi);
}

namespace detail {
inline std::vector<float> pixels_of(const IntensityImage& img) {
  return std::vector<float>(img.raster().data(), img.raster().data() + img.raster().size());
}
}  // namespace detail

inline EpipolarStatus photometric_error_5pt(const EpipolarGeometry& g, const IntensityImage& I0,
                                            const IntensityImage& I1, const PixelCoord& x,
                                            double d, std::array<double, 5>& e) {
  const dfuse_epigeom cg = g.c_abi();
  int32_t st = 0;
  device::check(dfuse_photometric_error_5pt_gen(device::ctx(), &cg, I0.raster().data(),
                                                I0.generation(), I1.raster().data(),
                                                I1.generation(), x.x, x.y, d, e.data(), &st),
                "photometric_error_5pt");
  return static_cast<EpipolarStatus>(st);
}

inline EpipolarStatus photometric_error_5pt(const IntensityImage& I0, const IntensityImage& I1,
                                            const PixelCoord& x, double d, const Pose& T0,
                                            const Pose& T1, const CameraIntrinsics& K,
                                            std::array<double, 5>& e) {
  return photometric_error_5pt(make_epipolar_geometry(T0, T1, K), I0, I1, x, d, e);
}

inline std::array<double, 5> jacobian_fd(const std::array<double, 5>& e_lo,
                                         const std::array<double, 5>& e_hi, double d_lo,
                                         double d_hi) {
  if (d_hi == d_lo) throw Error(Err::ZeroBaselineStep, "identical depths");
  std::array<double, 5> J;
  const double inv = 1.0 / (d_hi - d_lo);
  for (int j = 0; j < 5; ++j) J[j] = (e_hi[j] - e_lo[j]) * inv;
  return J;
}

inline constexpr double kMinJacobianNormSq = 1e-12;

inline double observation_variance(const std::array<double, 5>& J) {
  double s = 0.0;
  for (double v : J) s += v * v;
  return s < kMinJacobianNormSq ? -1.0 : 1.0 / s;
}

// many pixels in one launch (what stereo_scan does per frame)
inline std::vector<EpipolarResult> search_depth_batch(
    const EpipolarGeometry& g, const IntensityImage& I0, const IntensityImage& I1,
    const std::vector<PixelCoord>& pixels, const std::vector<std::optional<DepthPrior>>& priors,
    const SearchConfig& cfg = {}) {
  const int n = static_cast<int>(pixels.size());
  std::vector<double> px(2 * n), pr(2 * n, 0.0);
  std::vector<uint8_t> has(n, 0);
  for (int k = 0; k < n; ++k) {
    px[2 * k] = pixels[k].x;
    px[2 * k + 1] = pixels[k].y;
    if (k < static_cast<int>(priors.size()) && priors[k]) {
      has[k] = 1;
      pr[2 * k] = priors[k]->depth;
      pr[2 * k + 1] = priors[k]->sigma;
    }
  }
  std::vector<int32_t> st(n);
  std::vector<EpipolarObservation> obs(n);
  const dfuse_epigeom cg = g.c_abi();
  const dfuse_search_cfg cc = cfg.c_abi();
  // the images' device copies are shared by every call and thread while
  // their generations are unchanged (one upload per image version)
  device::check(dfuse_search_depth_gen(device::ctx(), &cg, I0.raster().data(), I0.generation(),
                                       I1.raster().data(), I1.generation(), n, px.data(),
                                       pr.data(), has.data(), &cc, st.data(),
                                       reinterpret_cast<dfuse_obs*>(obs.data()), nullptr, nullptr),
                "search_depth");
  std::vector<EpipolarResult> out(n);
  for (int k = 0; k < n; ++k) {
    out[k].status = static_cast<EpipolarStatus>(st[k]);
    if (out[k].ok()) out[k].obs = obs[k];
  }
  return out;
}

inline EpipolarResult search_depth(const EpipolarGeometry& g, const IntensityImage& I0,
                                   const IntensityImage& I1, const PixelCoord& x,
                                   std::optional<DepthPrior> prior, const SearchConfig& cfg = {}) {
  return search_depth_batch(g, I0, I1, {x}, {prior}, cfg)[0];
}

inline EpipolarResult search_depth(const IntensityImage& I0, const IntensityImage& I1,
                                   const PixelCoord& x, std::optional<DepthPrior> prior,
                                   const Pose& T0, const Pose& T1, const CameraIntrinsics& K,
                                   const SearchConfig& cfg = {}) {
  return search_depth(make_epipolar_geometry(T0, T1, K), I0, I1, x, prior, cfg);
}

inline constexpr double kOutlierGateSigmas = 5.0;

inline SemiDenseMap update_semidense(SemiDenseMap map,
                                     const std::vector<EpipolarObservation>& observations) {
  int32_t count = map.inlier_count;
  device::check(dfuse_update_semidense(
                    device::ctx(), map.depth.width(), map.depth.height(), map.depth.data(),
                    map.variance.data(), map.valid.data(), &count,
                    static_cast<int>(observations.size()),
                    reinterpret_cast<const dfuse_obs*>(observations.data())),
                "update_semidense");
  map.inlier_count = count;
  return map;
}

inline bool should_create_keyframe(const Pose& T_kf, const Pose& T_cur, double median_depth,
                                   const SemiDenseMap& map, const KeyframePolicy& policy) {
  if (median_depth <= 0.0) throw Error(Err::NonPositiveDepth, "median depth");
  const double trans = compose(T_kf.inverse(), T_cur).translation.norm();
  return trans / median_depth > policy.lambda_trans || map.inlier_count < policy.lambda_inliers;
}

}  // namespace dfuse
