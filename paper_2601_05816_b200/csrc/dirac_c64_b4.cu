// c64 hopping-kernel instantiations, rhs counts [4, 6] (separate unit: parallel build)
#define B200WD_HOP_ENTRY_DEF
#include "dirac_kernels.cuh"

namespace b200wd {
template void hop_entry<float, 2, 4>(const HopParams&, cudaStream_t);
template void hop_entry<float, 2, 6>(const HopParams&, cudaStream_t);
}  // namespace b200wd
