// dfuse/device.hpp -- the CUDA context behind the drop-in headers.
//
// The reference API has no context argument, so the drop-in functions run on
// a per-thread default context (device DFUSE_DEVICE, default 0). Errors from
// the C-ABI are rethrown as dfuse::Error with the reference's Err code;
// CUDA failures (no sm_100 device, launch errors) as dfuse::DeviceError.
// There is no CPU fallback.
#pragma once

#include <cstdlib>
#include <string>

#include "../dfuse_cuda.h"
#include "dfuse/errors.hpp"

namespace dfuse::device {

class Context {
 public:
  explicit Context(int device) {
    if (dfuse_ctx_create(device, &ctx_) != DFUSE_OK || !ctx_)
      throw DeviceError("dfuse: no usable sm_100 CUDA device " + std::to_string(device));
  }
  ~Context() { dfuse_ctx_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  dfuse_ctx* get() const { return ctx_; }

 private:
  dfuse_ctx* ctx_ = nullptr;
};

inline dfuse_ctx* ctx() {
  static thread_local Context c([] {
    const char* d = std::getenv("DFUSE_DEVICE");
    return d ? std::atoi(d) : 0;
  }());
  return c.get();
}

inline void check(int rc, const char* what) {
  if (rc == DFUSE_OK) return;
  const std::string msg = std::string(what) + ": " + dfuse_last_error(ctx());
  if (rc >= 1 && rc <= static_cast<int>(Err::InvalidArgument) + 1)
    throw Error(static_cast<Err>(rc - 1), msg);
  throw DeviceError(msg);
}

}  // namespace dfuse::device
