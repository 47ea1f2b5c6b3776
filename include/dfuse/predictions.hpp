// dfuse/predictions.hpp -- drop-in for the solver input of
// proj/include/dfuse/predictions.hpp:18-29 (PredictionSet: six rasters of
// float32-exact doubles) and focal_adjust (148-157). DFPRED file I/O and the
// synthetic oracle are per-keyframe tooling outside the per-frame hot path
// and are not part of this drop-in yet.
#pragma once

#include <cmath>

#include "dfuse/raster.hpp"

namespace dfuse {

struct PredictionSet {
  Raster<double> log_depth;
  Raster<double> log_depth_var;
  Raster<double> grad_x;
  Raster<double> grad_x_var;
  Raster<double> grad_y;
  Raster<double> grad_y_var;
  double source_focal = 0.0;

  int width() const { return log_depth.width(); }
  int height() const { return log_depth.height(); }
};

// shift log-depths to a new focal length (gradients and variances are
// focal-invariant); once per keyframe, host side
inline PredictionSet focal_adjust(const PredictionSet& p, double test_focal) {
  if (!(test_focal > 0.0) || !(p.source_focal > 0.0))
    throw Error(Err::NonPositiveFocal, "focal_adjust requires positive focal lengths");
  PredictionSet out = p;
  if (test_focal == p.source_focal) return out;
  const double shift = std::log(test_focal / p.source_focal);
  for (std::size_t i = 0; i < out.log_depth.size(); ++i) out.log_depth[i] += shift;
  out.source_focal = test_focal;
  return out;
}

}  // namespace dfuse
