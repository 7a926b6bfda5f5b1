// direct_q8.cu -- `direct` kernels with 8 column groups of 8 pixels per tile row
// (explicit instantiations of direct_impl.cuh; compiled in parallel with the other shapes).
#include "direct_impl.cuh"

namespace ai3 {
template cudaError_t launch_direct_qg<8, 8, 8>(const DirectArgs& a, cudaStream_t st);
template cudaError_t launch_direct_qg<8, 8, 7>(const DirectArgs& a, cudaStream_t st);
template cudaError_t launch_direct_qg<8, 4, 8>(const DirectArgs& a, cudaStream_t st);
template cudaError_t launch_direct_qg<8, 4, 7>(const DirectArgs& a, cudaStream_t st);
}  // namespace ai3
