// c128 hopping-kernel instantiations, rhs counts [0, 1, 2, 3] (separate unit: parallel build)
#define B200WD_HOP_ENTRY_DEF
#include "dirac_kernels.cuh"

namespace b200wd {
template void hop_entry<double, 1, 0>(const HopParams&, cudaStream_t);
template void hop_entry<double, 1, 1>(const HopParams&, cudaStream_t);
template void hop_entry<double, 1, 2>(const HopParams&, cudaStream_t);
template void hop_entry<double, 1, 3>(const HopParams&, cudaStream_t);
}  // namespace b200wd
