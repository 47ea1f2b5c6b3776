// eval.cu -- device scoring of a fused depth raster: pct_within_10 and
// median_abs_rel (eval.hpp:34-68) as finalize_keyframe computes them
// (pipeline.hpp:232-247), and export_depth_image's 16-bit quantisation
// (eval.hpp:221-226 -> depth_io.hpp:51-63; the PNG encoding stays with the
// caller). HBM-bound streaming passes plus one exact device selection.
//
//   k_score   one pass over the raster: ratio |est - gt| / gt for the pixels
//             where both are defined (+inf elsewhere, so they sort last),
//             and three integer counts (valid gt, evaluated, within 10%)
//             reduced per warp and added with one atomic per warp (integer:
//             order-independent, bit-exact).
//   median    cub radix sort of the P ratios; the answer is the element at
//             n_evaluated / 2, exactly what nth_element returns.
#include <cub/device/device_radix_sort.cuh>
#include <string>

#include "common.cuh"
#include "eval.cuh"

namespace dfuse_cuda {

constexpr double kWithin = 0.10 + 1e-12;  // eval.hpp:29

__global__ void k_score(long P, const double* __restrict__ est, const double* __restrict__ ld,
                        const uint8_t* __restrict__ est_valid, const double* __restrict__ gt,
                        const uint8_t* __restrict__ gt_valid, double* __restrict__ ratio,
                        unsigned long long* __restrict__ counts) {
  unsigned long long n_gt = 0, n_ev = 0, n_ok = 0;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < P;
       i += (long)gridDim.x * blockDim.x) {
    double r = CUDART_INF;
    if (gt_valid[i]) {
      ++n_gt;
      if (!est_valid || est_valid[i]) {
        const double e = est ? est[i] : exp(ld[i]);  // pipeline.hpp:235
        const double g = gt[i];
        r = fabs(e - g) / g;
        ++n_ev;
        if (r <= kWithin) ++n_ok;  // eval.hpp:43
      }
    }
    ratio[i] = r;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    n_gt += __shfl_xor_sync(0xffffffffu, n_gt, o);
    n_ev += __shfl_xor_sync(0xffffffffu, n_ev, o);
    n_ok += __shfl_xor_sync(0xffffffffu, n_ok, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(counts, n_gt);
    atomicAdd(counts + 1, n_ev);
    atomicAdd(counts + 2, n_ok);
  }
}

__global__ void k_export_u16(long P, const double* __restrict__ ld, double scale,
                             uint16_t* __restrict__ out) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < P;
       i += (long)gridDim.x * blockDim.x) {
    double s = round(exp(ld[i]) * scale);  // depth_io.hpp:61-62
    s = s < 0.0 ? 0.0 : (s > 65535.0 ? 65535.0 : s);
    out[i] = (uint16_t)s;
  }
}

static int stream_grid(dfuse_ctx* ctx, long P) {
  long b = (P + 255) / 256;
  if (b > 8L * ctx->num_sms) b = 8L * ctx->num_sms;
  return (int)(b > 0 ? b : 1);
}

void score_device(dfuse_ctx* ctx, long P, const double* est, const double* log_depth,
                  const uint8_t* est_valid, const double* gt, const uint8_t* gt_valid,
                  dfuse_keyframe_score* out) {
  double* ratio = (double*)scratch(ctx, S_TMP0, 2 * sizeof(double) * P + 64);
  double* sorted = ratio + P;
  unsigned long long* counts = (unsigned long long*)(sorted + P);
  DF_CUDA(cudaMemsetAsync(counts, 0, 3 * sizeof(unsigned long long), ctx->stream));
  k_score<<<stream_grid(ctx, P), 256, 0, ctx->stream>>>(P, est, log_depth, est_valid, gt,
                                                        gt_valid, ratio, counts);
  DF_LAUNCHED(ctx);
  size_t temp = 0;
  DF_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, temp, ratio, sorted, (int)P, 0, 64,
                                         ctx->stream));
  void* tmp = scratch(ctx, S_TMP1, temp);
  DF_CUDA(cub::DeviceRadixSort::SortKeys(tmp, temp, ratio, sorted, (int)P, 0, 64, ctx->stream));
  DF_LAUNCHED(ctx);
  unsigned long long h[3];
  DF_CUDA(cudaMemcpyAsync(h, counts, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
  DF_CUDA(cudaStreamSynchronize(ctx->stream));
  if (h[0] == 0)  // eval.hpp:45
    throw RefError{DFUSE_E_NO_VALID_GROUND_TRUTH, "empty ground-truth mask"};
  double med = 0.0;  // eval.hpp:63
  if (h[1] > 0) {
    DF_CUDA(cudaMemcpyAsync(&med, sorted + h[1] / 2, sizeof med, cudaMemcpyDeviceToHost,
                            ctx->stream));
    DF_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  out->pct_within_10 = 100.0 * (double)h[2] / (double)h[0];
  out->n_evaluated = (int32_t)h[0];  // finalize_keyframe: the valid-gt count, pipeline.hpp:237-246
  out->median_abs_rel = med;
}

void export_u16_device(dfuse_ctx* ctx, long P, const double* log_depth, double depth_scale,
                       uint16_t* out_dev) {
  k_export_u16<<<stream_grid(ctx, P), 256, 0, ctx->stream>>>(P, log_depth, depth_scale, out_dev);
  DF_LAUNCHED(ctx);
}

}  // namespace dfuse_cuda

using namespace dfuse_cuda;

extern "C" int dfuse_score_depth(dfuse_ctx* ctx, int width, int height, const double* est,
                                 const uint8_t* est_valid, const double* gt_metres,
                                 const uint8_t* gt_valid, dfuse_keyframe_score* out) {
  if (!ctx) return DFUSE_E_INVALID_ARGUMENT;
  try {
    DF_CUDA(cudaSetDevice(ctx->device));
    if (!est || !gt_metres || !gt_valid || !out)
      throw RefError{DFUSE_E_INVALID_ARGUMENT, "null pointer"};
    if (width <= 0 || height <= 0)
      throw RefError{DFUSE_E_DIMENSION_MISMATCH, "estimate vs ground truth"};
    const long P = (long)width * height;
    char* d = (char*)scratch(ctx, S_TMP2, 2 * sizeof(double) * P + 2 * P + 512);
    double* d_est = (double*)d;
    double* d_gt = d_est + P;
    uint8_t* d_gv = (uint8_t*)(d_gt + P);
    uint8_t* d_ev = est_valid ? d_gv + P : nullptr;
    DF_CUDA(cudaMemcpyAsync(d_est, est, sizeof(double) * P, cudaMemcpyHostToDevice, ctx->stream));
    DF_CUDA(cudaMemcpyAsync(d_gt, gt_metres, sizeof(double) * P, cudaMemcpyHostToDevice,
                            ctx->stream));
    DF_CUDA(cudaMemcpyAsync(d_gv, gt_valid, P, cudaMemcpyHostToDevice, ctx->stream));
    if (d_ev) DF_CUDA(cudaMemcpyAsync(d_ev, est_valid, P, cudaMemcpyHostToDevice, ctx->stream));
    score_device(ctx, P, d_est, nullptr, d_ev, d_gt, d_gv, out);
    ctx->last_error.clear();
    return DFUSE_OK;
  } catch (const RefError& e) {
    ctx->last_error = e.msg;
    return e.code;
  } catch (const CudaFailure& e) {
    ctx->last_error = std::string("CUDA: ") + cudaGetErrorString(e.err) + " in " + e.what;
    return DFUSE_E_CUDA;
  }
}
