// Compile check of dfuse::gpu::stereo_scan against stand-ins with the shape of
// the reference's Keyframe / Frame / PipelineConfig (pipeline.hpp:25-33,
// datasets.hpp:49-55, config.hpp:20-48) -- the one-line switch INTEGRATION.md
// shows for pipeline.hpp's stereo_scan. Built (not run) by tests/test_cpp_dropin.py.
#include "dfuse/stereo_scan.hpp"

namespace ref_shape {
struct Frame {
  double timestamp = 0.0;
  dfuse::IntensityImage intensity;
  dfuse::Pose pose;
};
struct Keyframe {
  int id = 0;
  Frame frame;
  dfuse::Mask texture;
  dfuse::SemiDenseMap semidense;
  int stereo_frames = 0;
};
struct PipelineConfig {
  dfuse::SearchConfig search;
  double texture_threshold = 0.02;
};
inline std::vector<dfuse::EpipolarObservation> stereo_scan(const Keyframe& kf, const Frame& frame,
                                                           const dfuse::CameraIntrinsics& camera,
                                                           const PipelineConfig& cfg) {
  return dfuse::gpu::stereo_scan(kf, frame, camera, cfg);
}
}  // namespace ref_shape

int main() {
  ref_shape::Keyframe kf;
  ref_shape::Frame f;
  ref_shape::PipelineConfig cfg;
  const dfuse::CameraIntrinsics K{100.0, 100.0, 15.5, 11.5, 32, 24};
  (void)&ref_shape::stereo_scan;
  (void)kf;
  (void)f;
  (void)cfg;
  (void)K;
  return 0;
}
