// inst_poccd_7.cu — explicit instantiation(s) of the poccd.cuh launcher (see dispatch.cu)
#include "poccd.cuh"

namespace hjcd {
template cudaError_t launch_poccd_t<7, true>(const DevRobot&, const DevCfg&, const float*, int, const float*, float*, float*, float*, float*, int32_t*, TraceOut, uint32_t*, cudaStream_t);
}  // namespace hjcd
