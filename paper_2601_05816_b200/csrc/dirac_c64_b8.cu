// c64 hopping-kernel instantiations, rhs counts [8, 12] (separate unit: parallel build)
#define B200WD_HOP_ENTRY_DEF
#include "dirac_kernels.cuh"

namespace b200wd {
template void hop_entry<float, 2, 8>(const HopParams&, cudaStream_t);
template void hop_entry<float, 2, 12>(const HopParams&, cudaStream_t);
}  // namespace b200wd
