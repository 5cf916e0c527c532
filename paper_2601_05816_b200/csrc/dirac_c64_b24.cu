// c64 hopping-kernel instantiations, rhs counts [24, 32] (separate unit: parallel build)
#define B200WD_HOP_ENTRY_DEF
#include "dirac_kernels.cuh"

namespace b200wd {
template void hop_entry<float, 2, 24>(const HopParams&, cudaStream_t);
template void hop_entry<float, 2, 32>(const HopParams&, cudaStream_t);
}  // namespace b200wd
