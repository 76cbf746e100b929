// fast_o2.cu -- the order-2 fast tile kernels and exact path (launch_all<2>),
// a separate translation unit so the library's kernels compile in parallel.
#include "launch.cuh"

namespace hdrlpa {
template int launch_all<2>(const DevParams &, const DevParams &, const TapParam &, int, int, int,
                            cudaStream_t);
}  // namespace hdrlpa
