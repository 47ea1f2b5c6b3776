// dfuse/session.hpp -- the device-resident keyframe (replaces the hot part of
// proj/include/dfuse/pipeline.hpp: make_keyframe 125-153, from prediction
// planes or from a DFPRED file (load_predictions + focal_adjust on the
// device), and process_frame 194-228 for tracked frames; the retirement test
// should_create_keyframe (215-218) with the median predicted depth cached on
// the device).
//
//   dfuse::DeviceKeyframe kf(K, I0, predictions, cfg.texture_threshold);
//   auto r = kf.process_frame(kf_pose, frame_pose, frame.intensity,
//                             cfg.search, cfg.robust, cfg.mode);
//   // r.observations, r.optimize_status (CgDivergence -> state unchanged,
//   // exactly like run_sequence's skipped solve, pipeline.hpp:328-331)
//   FusionState st = kf.fusion();  SemiDenseMap m = kf.semidense();
#pragma once

#include <fstream>
#include <iterator>
#include <string>
#include <vector>

#include "dfuse/fusion.hpp"
#include "dfuse/semidense.hpp"

namespace dfuse {

struct FrameOutcome {
  int observations = 0;
  int inlier_count = 0;
  int stereo_frames = 0;
  int optimize_status = 0;  // 0, or (int)Err + 1 of the error optimize threw
  float stereo_ms = 0.f;
  float optimise_ms = 0.f;
  dfuse_solver_stats stats{};
};

class DeviceKeyframe {
 public:
  DeviceKeyframe(const CameraIntrinsics& K, const IntensityImage& I0, const PredictionSet& pred,
                 double texture_threshold)
      : K_(K) {
    const dfuse_intrinsics k = K.c_abi();
    const double* planes[6] = {pred.log_depth.data(), pred.log_depth_var.data(),
                               pred.grad_x.data(),    pred.grad_x_var.data(),
                               pred.grad_y.data(),    pred.grad_y_var.data()};
    device::check(dfuse_kf_create(device::ctx(), &k, I0.raster().data(), planes,
                                  texture_threshold, &kf_),
                  "make_keyframe");
  }
  // make_keyframe with cfg.predictions_dir set (pipeline.hpp:133-147): the
  // DFPRED file at `dfpred_path` is read here and validated, widened and
  // focal-adjusted to K.fx on the device
  DeviceKeyframe(const CameraIntrinsics& K, const IntensityImage& I0,
                 const std::string& dfpred_path, double texture_threshold)
      : K_(K) {
    std::ifstream in(dfpred_path, std::ios::binary);
    if (!in) throw Error(Err::MissingFile, dfpred_path);  // predictions.hpp:70-71
    const std::vector<char> bytes((std::istreambuf_iterator<char>(in)),
                                  std::istreambuf_iterator<char>());
    const dfuse_intrinsics k = K.c_abi();
    device::check(dfuse_kf_create_dfpred(device::ctx(), &k, I0.raster().data(), bytes.data(),
                                         bytes.size(), texture_threshold, &kf_),
                  dfpred_path.c_str());
  }
  ~DeviceKeyframe() { dfuse_kf_destroy(kf_); }

  // detail::median_predicted_depth (pipeline.hpp:94-99), once per keyframe
  double median_depth() const {
    double m = 0.0;
    device::check(dfuse_kf_median_depth(kf_, &m), "median_predicted_depth");
    return m;
  }

  // process_frame's retirement test (pipeline.hpp:215-218) for the frame at
  // `frame_pose`, after its process_frame call
  bool should_create_keyframe(const Pose& keyframe_pose, const Pose& frame_pose,
                              const KeyframePolicy& policy = {}) const {
    SemiDenseMap m;
    int32_t count = 0;
    device::check(dfuse_kf_download(kf_, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                                    &count, nullptr),
                  "download");
    m.inlier_count = count;
    return dfuse::should_create_keyframe(keyframe_pose, frame_pose, median_depth(), m, policy);
  }
  DeviceKeyframe(const DeviceKeyframe&) = delete;
  DeviceKeyframe& operator=(const DeviceKeyframe&) = delete;

  FrameOutcome process_frame(const EpipolarGeometry& g, const IntensityImage& I1,
                             const SearchConfig& search, const RobustConfig& robust,
                             FusionMode mode) {
    const dfuse_epigeom cg = g.c_abi();
    const dfuse_search_cfg sc = search.c_abi();
    const dfuse_robust_cfg rc = robust.c_abi();
    dfuse_frame_result r;
    device::check(dfuse_kf_process_frame(kf_, &cg, I1.raster().data(), &sc, &rc,
                                         detail::mode_of(mode), &r),
                  "process_frame");
    return {r.observations, r.inlier_count, r.stereo_frames, r.optimize_status, r.stereo_ms,
            r.optimise_ms, r.stats};
  }

  FrameOutcome process_frame(const Pose& keyframe_pose, const Pose& frame_pose,
                             const IntensityImage& I1, const SearchConfig& search,
                             const RobustConfig& robust, FusionMode mode) {
    return process_frame(make_epipolar_geometry(keyframe_pose, frame_pose, K_), I1, search,
                         robust, mode);
  }

  // Pipelined submission of a host frame (dfuse_kf_process_frame_host_async):
  // returns at once; the frame is copied in while the previous one computes,
  // and log_depth_out (width*height doubles, or null) receives this frame's
  // fused log-depth while the next one computes. Use pinned buffers
  // (cudaHostAlloc) for the copies to overlap; both must stay untouched until
  // finish(), which waits and returns the last submitted frame's outcome.
  void submit_frame(const EpipolarGeometry& g, const float* I1, const SearchConfig& search,
                    const RobustConfig& robust, FusionMode mode, double* log_depth_out) {
    const dfuse_epigeom cg = g.c_abi();
    const dfuse_search_cfg sc = search.c_abi();
    const dfuse_robust_cfg rc = robust.c_abi();
    device::check(dfuse_kf_process_frame_host_async(kf_, &cg, I1, &sc, &rc,
                                                    detail::mode_of(mode), log_depth_out),
                  "submit_frame");
  }

  FrameOutcome finish() {
    dfuse_frame_result r;
    device::check(dfuse_kf_last_result(kf_, &r), "finish");
    return {r.observations, r.inlier_count, r.stereo_frames, r.optimize_status, r.stereo_ms,
            r.optimise_ms, r.stats};
  }

  FusionState fusion() const {
    FusionState st{Raster<double>(K_.width, K_.height, 0.0), 1.0, 0};
    int32_t it = 0;
    device::check(dfuse_kf_download(kf_, st.log_depth.data(), &st.scale, &it, nullptr, nullptr,
                                    nullptr, nullptr, nullptr),
                  "download");
    st.iteration = it;
    return st;
  }

  SemiDenseMap semidense() const {
    SemiDenseMap m = SemiDenseMap::empty(K_.width, K_.height);
    int32_t count = 0;
    device::check(dfuse_kf_download(kf_, nullptr, nullptr, nullptr, m.depth.data(),
                                    m.variance.data(), m.valid.data(), &count, nullptr),
                  "download");
    m.inlier_count = count;
    return m;
  }

  Mask texture() const {
    Mask m(K_.width, K_.height, 0);
    device::check(dfuse_kf_download(kf_, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                                    nullptr, m.data()),
                  "download");
    return m;
  }

  void reset() { device::check(dfuse_kf_reset(kf_), "reset"); }

 private:
  CameraIntrinsics K_;
  dfuse_keyframe* kf_ = nullptr;
};

}  // namespace dfuse
