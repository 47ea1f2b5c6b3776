// fusion_launch.cuh -- definition of launch_fusion_t (fusion_part_*.cu only)
#pragma once
#include "fusion_impl.cuh"

namespace dfuse_cuda {

constexpr size_t kMaxDynSmem = 227 * 1024;

template <int PPT, int VAR>
void launch_fusion_t(dfuse_ctx* ctx, FusionArgs& a, int grid) {
  size_t smem = 0;
  if (PPT > 0) {
    smem = pcg_tile_smem(PPT, a.tw_max, a.th_max);
    size_t& configured = ctx->fusion_smem_set[PPT * 4 + VAR];  // per context = per device
    if (smem > configured) {
      DF_CUDA(cudaFuncSetAttribute((const void*)k_fusion<PPT, VAR>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      configured = smem;
    }
  }
  void* args[] = {&a};
  DF_CUDA(cudaLaunchCooperativeKernel((const void*)k_fusion<PPT, VAR>, dim3(grid), dim3(FT), args,
                                      smem, ctx->stream));
}

}  // namespace dfuse_cuda
