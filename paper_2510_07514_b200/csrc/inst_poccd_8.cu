// inst_poccd_8.cu — explicit instantiation(s) of the poccd.cuh launcher (see dispatch.cu)
#include "poccd.cuh"

namespace hjcd {
template cudaError_t launch_poccd_t<8, true>(const DevRobot&, const DevCfg&, const float*, int, const float*, float*, float*, float*, float*, int32_t*, TraceOut, uint32_t*, cudaStream_t);
template cudaError_t launch_poccd_t<8, false>(const DevRobot&, const DevCfg&, const float*, int, const float*, float*, float*, float*, float*, int32_t*, TraceOut, uint32_t*, cudaStream_t);
}  // namespace hjcd
