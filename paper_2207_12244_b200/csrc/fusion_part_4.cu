// fusion_part_4.cu -- k_fusion instantiations <4, 0>, <4, 1>, <4, 2> (see fusion_impl.cuh)
#define DFUSE_RESIDENT_TU  // resident-PCG kernels: kResidentFT threads per CTA
#include "fusion_launch.cuh"

namespace dfuse_cuda {
template void launch_fusion_t<4, 0>(dfuse_ctx*, FusionArgs&, int);
template void launch_fusion_t<4, 1>(dfuse_ctx*, FusionArgs&, int);
template void launch_fusion_t<4, 2>(dfuse_ctx*, FusionArgs&, int);
}  // namespace dfuse_cuda
