// fusion_launch.cuh -- definition of launch_fusion_t (fusion_part_*.cu only)
#pragma once
#include <stdio.h>

#include <mutex>

#include "fusion_impl.cuh"

namespace dfuse_cuda {

constexpr size_t kMaxDynSmem = 227 * 1024;
constexpr int kMaxDevices = 64;

template <int PPT, int VAR>
void launch_fusion_t(dfuse_ctx* ctx, FusionArgs& a, int grid) {
  size_t smem = 0;
  if (PPT > 0) {
    smem = pcg_tile_smem(PPT, a.tw_max, a.th_max);
    // The attribute belongs to the (device, function) pair, shared by every
    // context and thread on the device: one process-wide table per device,
    // raised (never lowered) under a lock, to the largest tile launched so
    // far.
    static std::mutex mu;
    static size_t set[kMaxDevices] = {};
    if (ctx->device < 0 || ctx->device >= kMaxDevices)
      throw CudaFailure{cudaErrorInvalidDevice, "k_fusion attribute table"};
    std::lock_guard<std::mutex> lk(mu);
    if (smem > set[ctx->device]) {
      DF_CUDA(cudaFuncSetAttribute((const void*)k_fusion<PPT, VAR>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      set[ctx->device] = smem;
    }
  }
  void* args[] = {&a};
  const cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_fusion<PPT, VAR>, dim3(grid),
                                                    dim3(FT), args, smem, ctx->stream);
  if (e != cudaSuccess) {  // say why (occupancy of this instantiation at this smem)
    cudaGetLastError();
    int occ = -1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_fusion<PPT, VAR>, FT, smem);
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, (const void*)k_fusion<PPT, VAR>);
    fprintf(stderr,
            "dfuse: k_fusion<%d,%d> launch failed (%s): grid %d, dynamic smem %zu (attribute "
            "%d), static smem %zu, regs %d, blocks/SM %d\n",
            PPT, VAR, cudaGetErrorString(e), grid, smem, fa.maxDynamicSharedSizeBytes,
            fa.sharedSizeBytes, fa.numRegs, occ);
    throw CudaFailure{e, "cudaLaunchCooperativeKernel(k_fusion)"};
  }
}

}  // namespace dfuse_cuda
