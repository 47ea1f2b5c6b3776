// dfuse/errors.hpp -- drop-in for the reference's error convention
// (proj/include/dfuse/errors.hpp:8-88): one exception type carrying an Err
// code. The enumerator order is the C-ABI's error numbering minus one
// (include/dfuse_cuda.h), so codes cross the boundary unchanged.
#pragma once

#include <stdexcept>
#include <string>

#include "../dfuse_cuda.h"

namespace dfuse {

enum class Err {
  NonPositiveDepth,
  BehindCamera,
  OutOfBounds,
  DegenerateBaseline,
  NoMinimum,
  ZeroBaselineStep,
  DegenerateJacobian,
  BorderPixel,
  BadMagic,
  DimensionMismatch,
  NonPositiveVariance,
  TruncatedFile,
  NonPositiveFocal,
  NonPositiveGroundTruth,
  MissingFile,
  MalformedLine,
  NonUnitQuaternion,
  BadImageFormat,
  NonPositiveScale,
  CgDivergence,
  NoSemiDenseSupport,
  NoValidGroundTruth,
  MismatchedKeyframeSets,
  IoError,
  UnknownKey,
  TypeError,
  InvalidArgument,
};

inline const char* err_name(Err e) { return dfuse_err_name(static_cast<int>(e) + 1); }

class Error : public std::runtime_error {
 public:
  Error(Err code, const std::string& detail)
      : std::runtime_error(std::string(err_name(code)) + ": " + detail), code_(code) {}
  Err code() const { return code_; }

 private:
  Err code_;
};

// CUDA runtime failures are not reference errors; they surface as this type
// (there is no CPU fallback to hide them).
class DeviceError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

}  // namespace dfuse
