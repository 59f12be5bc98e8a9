// inst_poccd_16.cu — explicit instantiation(s) of the poccd.cuh launcher (see dispatch.cu)
#include "poccd.cuh"

namespace hjcd {
template cudaError_t launch_poccd_t<16, false>(const DevRobot&, const DevCfg&, const float*, int, const float*, float*, float*, float*, float*, int32_t*, TraceOut, uint32_t*, cudaStream_t);
}  // namespace hjcd
