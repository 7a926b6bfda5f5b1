// direct_q4.cu -- `direct` kernels with 4 column groups of 8 pixels per tile row
// (explicit instantiations of direct_impl.cuh; compiled in parallel with the other shapes).
#include "direct_impl.cuh"

namespace ai3 {
template cudaError_t launch_direct_qg<4, 8, 8>(const DirectArgs& a, cudaStream_t st);
template cudaError_t launch_direct_qg<4, 8, 7>(const DirectArgs& a, cudaStream_t st);
template cudaError_t launch_direct_qg<4, 4, 8>(const DirectArgs& a, cudaStream_t st);
template cudaError_t launch_direct_qg<4, 4, 7>(const DirectArgs& a, cudaStream_t st);
}  // namespace ai3
