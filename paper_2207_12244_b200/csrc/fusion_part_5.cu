// fusion_part_5.cu -- k_fusion instantiations <5, 0>, <5, 1>, <5, 2> (see fusion_impl.cuh)
#define DFUSE_RESIDENT_TU  // resident-PCG kernels: kResidentFT threads per CTA
#include "fusion_launch.cuh"

namespace dfuse_cuda {
template void launch_fusion_t<5, 0>(dfuse_ctx*, FusionArgs&, int);
template void launch_fusion_t<5, 1>(dfuse_ctx*, FusionArgs&, int);
template void launch_fusion_t<5, 2>(dfuse_ctx*, FusionArgs&, int);
}  // namespace dfuse_cuda
