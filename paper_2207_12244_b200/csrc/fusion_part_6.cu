// fusion_part_6.cu -- k_fusion instantiations <6, 0> (see fusion_impl.cuh)
#include "fusion_launch.cuh"

namespace dfuse_cuda {
template void launch_fusion_t<6, 0>(dfuse_ctx*, FusionArgs&, int);
}  // namespace dfuse_cuda
