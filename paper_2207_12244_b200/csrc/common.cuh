// common.cuh -- shared device/host helpers of libdfuse_cuda.so (sm_100a).
//
// All FP64 code in this library is compiled with -fmad=false (see
// csrc/Makefile): the reference builds for baseline x86-64 without FMA, and
// the stereo search must reproduce its roundings bit for bit (SURVEY.md
// Appendix B, H1). IEEE division and sqrt are the CUDA defaults
// (-prec-div/-prec-sqrt true) and are kept.
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include <string>

#include "../../include/dfuse_cuda.h"

namespace dfuse_cuda {

// ---------------------------------------------------------------------------
// context
struct Buffer {
  void* ptr = nullptr;
  size_t bytes = 0;
};

}  // namespace dfuse_cuda

struct dfuse_ctx {
  int device = 0;
  int num_sms = 0;
  int solver_ctas = 0;  // 0 = auto (one per SM)
  int diag_repeat = 0, diag_sweep = 0;  // DFUSE_PCG_REPEAT=n[,1] (diagnostics)
  int force_streaming = 0;  // 1: never use the SM-resident PCG
  int trace = 0;            // DFUSE_TRACE=1: print per-phase PCG cycle counts
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[4] = {};
  std::string last_error;
  int64_t launches = 0;
  // grow-only scratch buffers keyed by slot
  dfuse_cuda::Buffer scratch[32];
  // pinned host staging for small results
  void* host_small = nullptr;
  // texture objects over tracked frames (stereo.cu frame_texture)
  struct TexEntry {
    const void* ptr = nullptr;
    int w = 0, h = 0;
    unsigned long long tex = 0;
  };
  TexEntry tex_cache[16];
  int tex_next = 0;
  int stereo_tex = 1;         // dfuse_ctx_set_stereo_texture
  int64_t tex_launches = 0;   // scan launches through the texture gather
  // per-device launch facts, filled on first use (kernel attributes and
  // occupancy are per device, so they live in the context, not in statics)
  int stereo_occ = 0;             // resident k_stereo CTAs per SM
  int fusion_occ = 0;             // resident k_fusion CTAs per SM
  size_t tex_base_align = 0, tex_pitch_align = 0;
  int pred_fp32 = 1;  // sessions keep float-exact prediction planes as fp32 (dfuse_ctx_set_fp32_predictions)
};

namespace dfuse_cuda {

// scratch slots
enum Slot {
  S_IMG0, S_IMG1, S_MASK, S_SEMI_D, S_SEMI_V, S_SEMI_VALID, S_STATUS, S_BEST, S_NSTEPS, S_OBS,
  S_LIST, S_COUNTERS, S_PRED, S_LD, S_FUSION_WS, S_PARTIALS, S_BARRIER, S_CONTROL, S_PX,
  S_PRIOR, S_HASPRIOR, S_TMP0, S_TMP1, S_TMP2, S_TMP3, S_TMP4, S_QUEUE, S_QCOUNT, S_NUM
};

void* scratch(dfuse_ctx* ctx, int slot, size_t bytes);  // throws CudaFailure

struct CudaFailure {
  cudaError_t err;
  const char* what;
};

#define DF_CUDA(call)                                   \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) throw dfuse_cuda::CudaFailure{e_, #call}; \
  } while (0)

// Reference error: (int)Err + 1 with a message
struct RefError {
  int code;
  std::string msg;
};

// launch bookkeeping: every kernel launch goes through this so the context
// can report how many of OUR kernels ran (bench "gpu_launches").
#define DF_LAUNCHED(ctx)                  \
  do {                                    \
    DF_CUDA(cudaGetLastError());          \
    (ctx)->launches++;                    \
  } while (0)

// ---------------------------------------------------------------------------
// device helpers shared by the stereo and fusion kernels

// glibc hypot (what std::hypot resolves to in the reference build,
// semidense.hpp:312): Borges' corrected hypot, non-FMA kernel, as in glibc
// >= 2.35 sysdeps/ieee754/dbl-64/e_hypot.c. Bit-identical to this image's
// libm (checked by tests/test_oracle_pin.py on the oracle's copy).
__device__ __forceinline__ double glibc_hypot_kernel(double ax, double ay) {
  double t1, t2;
  double h = sqrt(ax * ax + ay * ay);
  if (h <= 2.0 * ay) {
    const double delta = h - ay;
    t1 = ax * (2.0 * delta - ax);
    t2 = (delta - 2.0 * (ax - ay)) * delta;
  } else {
    const double delta = h - ax;
    t1 = 2.0 * delta * (ax - 2.0 * ay);
    t2 = (4.0 * delta - ay) * ay + delta * delta;
  }
  h -= (t1 + t2) / (2.0 * h);
  return h;
}

__device__ __forceinline__ double glibc_hypot(double x, double y) {
  if (!isfinite(x) || !isfinite(y)) {
    if (isinf(x) || isinf(y)) return CUDART_INF;
    return x + y;
  }
  x = fabs(x);
  y = fabs(y);
  const double ax = x < y ? y : x;
  const double ay = x < y ? x : y;
  if (ax > 0x1p+511) {
    if (ay <= ax * 0x1p-54) return ax + ay;
    return glibc_hypot_kernel(ax * 0x1p-600, ay * 0x1p-600) / 0x1p-600;
  }
  if (ay < 0x1p-511) {
    if (ax >= ay / 0x1p-54) return ax + ay;
    return glibc_hypot_kernel(ax / 0x1p-600, ay / 0x1p-600) * 0x1p-600;
  }
  if (ay <= ax * 0x1p-54) return ax + ay;
  return glibc_hypot_kernel(ax, ay);
}

// device wall clock in ns (diagnostics: DFUSE_TRACE)
__device__ __forceinline__ long long df_now() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// deterministic warp sum: fixed butterfly order, identical on every lane
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = v + __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ int warp_sum_int(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace dfuse_cuda
