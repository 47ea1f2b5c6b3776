// TEST INFRASTRUCTURE ONLY: an in-memory stand-in for the few OpenCV names
// proj/include/dfuse/depth_io.hpp uses, so that the reference's eval.hpp /
// depth_io.hpp compile into oracle/_ref without OpenCV. imwrite keeps the
// 16-bit raster in a process-wide map instead of encoding a PNG; imread
// returns it. Only save_depth_png's quantisation is exercised through it.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

#define CV_16UC1 2

namespace cv {

enum { IMREAD_UNCHANGED = -1, INTER_NEAREST = 0 };

struct Size {
  int width, height;
  Size(int w, int h) : width(w), height(h) {}
};

struct Mat {
  int rows = 0, cols = 0, t = -1;
  std::shared_ptr<std::vector<std::uint16_t>> buf;
  Mat() = default;
  Mat(int r, int c, int type)
      : rows(r), cols(c), t(type),
        buf(std::make_shared<std::vector<std::uint16_t>>((std::size_t)r * c, 0)) {}
  template <class T>
  T* ptr(int y) {
    return reinterpret_cast<T*>(buf->data() + (std::size_t)y * cols);
  }
  template <class T>
  const T* ptr(int y) const {
    return reinterpret_cast<const T*>(buf->data() + (std::size_t)y * cols);
  }
  bool empty() const { return !buf || rows * cols == 0; }
  int type() const { return t; }
};

inline std::map<std::string, Mat>& image_store() {
  static std::map<std::string, Mat> s;
  return s;
}

}  // namespace cv
