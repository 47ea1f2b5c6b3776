// eval.cuh -- device scoring of a fused depth raster (eval.hpp:34-68,
// 221-226; pipeline.hpp:232-247), used by the C-ABI in eval.cu and by the
// keyframe session (session.cu)
#pragma once

#include "common.cuh"

namespace dfuse_cuda {

// est: metres (device), or null with log_depth set: est = exp(log_depth).
// est_valid may be null. Returns NoValidGroundTruth (as RefError) when the
// ground-truth mask is empty.
void score_device(dfuse_ctx* ctx, long P, const double* est, const double* log_depth,
                  const uint8_t* est_valid, const double* gt, const uint8_t* gt_valid,
                  dfuse_keyframe_score* out);

void export_u16_device(dfuse_ctx* ctx, long P, const double* log_depth, double depth_scale,
                       uint16_t* out_dev);

}  // namespace dfuse_cuda
