// dfuse/stereo_scan.hpp -- drop-in for stereo_scan, pipeline.hpp:157-190.
//
// The reference scans a frame with one search_depth call per masked pixel
// (an OpenMP loop over rows, pipeline.hpp:167-178). Here the whole scan is
// one kernel launch (dfuse_stereo_scan): every masked pixel is searched with
// its prior from the semi-dense map, and the OK observations come back in
// raster order -- the same vector, bit for bit.
//
// pipeline.hpp's own Keyframe / Frame / PipelineConfig live next to the
// dataset readers (OpenCV), which this repo does not redefine, so the
// keyframe-level entry point is a template over those types: a reference
// build switches its scan over by making the body of pipeline.hpp's
// stereo_scan `return dfuse::gpu::stereo_scan(kf, frame, camera, cfg);`
// (INTEGRATION.md).
#pragma once

#include <vector>

#include "dfuse/semidense.hpp"

namespace dfuse {

// stereo_scan on explicit inputs: geometry, keyframe image, tracked image,
// texture mask and the keyframe's semi-dense map (read only)
inline std::vector<EpipolarObservation> stereo_scan(const EpipolarGeometry& g,
                                                    const IntensityImage& I0,
                                                    const IntensityImage& I1, const Mask& texture,
                                                    const SemiDenseMap& map,
                                                    const SearchConfig& cfg = {}) {
  const int w = I0.width(), h = I0.height();
  require_same_size(I0.raster(), I1.raster(), "stereo_scan images");
  require_same_size(I0.raster(), texture, "stereo_scan mask");
  require_same_size(I0.raster(), map.depth, "stereo_scan semi-dense map");
  if (g.K.width != w || g.K.height != h)
    throw Error(Err::DimensionMismatch, "stereo_scan: camera does not match the images");
  std::vector<EpipolarObservation> obs(static_cast<std::size_t>(w) * h);
  int32_t n = 0;
  const dfuse_epigeom cg = g.c_abi();
  const dfuse_search_cfg cc = cfg.c_abi();
  device::check(dfuse_stereo_scan(device::ctx(), &cg, I0.raster().data(), I0.generation(),
                                  I1.raster().data(), I1.generation(), texture.data(),
                                  map.depth.data(), map.variance.data(), map.valid.data(), &cc,
                                  reinterpret_cast<dfuse_obs*>(obs.data()), &n),
                "stereo_scan");
  obs.resize(static_cast<std::size_t>(n));
  return obs;
}

namespace gpu {

// stereo_scan(kf, frame, camera, cfg) with the reference's signature
// (pipeline.hpp:157-190): KeyframeT has .frame.pose, .frame.intensity,
// .texture and .semidense; FrameT has .pose and .intensity; ConfigT has
// .search (pipeline.hpp:25-33, datasets.hpp:49-55, config.hpp:20-48)
template <class KeyframeT, class FrameT, class ConfigT>
std::vector<EpipolarObservation> stereo_scan(const KeyframeT& kf, const FrameT& frame,
                                             const CameraIntrinsics& camera,
                                             const ConfigT& cfg) {
  const EpipolarGeometry g = make_epipolar_geometry(kf.frame.pose, frame.pose, camera);
  if (g.t_10.norm() < 1e-12) return {};  // pipeline.hpp:160
  return dfuse::stereo_scan(g, kf.frame.intensity, frame.intensity, kf.texture, kf.semidense,
                            cfg.search);
}

}  // namespace gpu
}  // namespace dfuse
