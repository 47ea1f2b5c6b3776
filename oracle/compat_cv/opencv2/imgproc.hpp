// TEST INFRASTRUCTURE ONLY (see core.hpp): nearest-neighbour resize is not
// exercised by the oracle; a shape-only placeholder keeps depth_io.hpp whole.
#pragma once
#include "opencv2/core.hpp"

namespace cv {
inline void resize(const Mat& src, Mat& dst, Size s, double, double, int) {
  Mat out(s.height, s.width, src.type());
  for (int y = 0; y < s.height; ++y)
    for (int x = 0; x < s.width; ++x)
      out.ptr<std::uint16_t>(y)[x] =
          src.ptr<std::uint16_t>(y * src.rows / s.height)[x * src.cols / s.width];
  dst = out;
}
}  // namespace cv
