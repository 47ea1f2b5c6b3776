// fusion_part_6.cu -- k_fusion instantiations <DFUSE_PPT_HI (6), 0/1/2> (see fusion_impl.cuh)
#define DFUSE_RESIDENT_TU  // resident-PCG kernels: kResidentFT threads per CTA
#include "fusion_launch.cuh"

namespace dfuse_cuda {
template void launch_fusion_t<DFUSE_PPT_HI, 0>(dfuse_ctx*, FusionArgs&, int);
template void launch_fusion_t<DFUSE_PPT_HI, 1>(dfuse_ctx*, FusionArgs&, int);
template void launch_fusion_t<DFUSE_PPT_HI, 2>(dfuse_ctx*, FusionArgs&, int);
}  // namespace dfuse_cuda
