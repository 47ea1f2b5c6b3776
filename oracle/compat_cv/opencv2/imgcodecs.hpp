// TEST INFRASTRUCTURE ONLY (see core.hpp)
#pragma once
#include "opencv2/core.hpp"

namespace cv {
inline bool imwrite(const std::string& path, const Mat& m) {
  image_store()[path] = m;
  return true;
}
inline Mat imread(const std::string& path, int) {
  auto it = image_store().find(path);
  return it == image_store().end() ? Mat() : it->second;
}
}  // namespace cv
