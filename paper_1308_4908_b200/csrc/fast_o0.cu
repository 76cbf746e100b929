// fast_o0.cu -- the order-0 fast tile kernels and exact path (launch_all<0>),
// a separate translation unit so the library's kernels compile in parallel.
#include "launch.cuh"

namespace hdrlpa {
template int launch_all<0>(const DevParams &, const DevParams &, const TapParam &, int, int, int,
                            cudaStream_t);
}  // namespace hdrlpa
