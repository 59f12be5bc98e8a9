// inst_poccd_18.cu — explicit instantiation of the PO-CCD launcher, exact n = 18 (PAPER Table II DoF; see dispatch.cu)
#include "poccd.cuh"

namespace hjcd {
template cudaError_t launch_poccd_t<18, true>(const DevRobot&, const DevCfg&, const float*, int, const float*, float*, float*, float*, float*, int32_t*, TraceOut, uint32_t*, cudaStream_t);
}  // namespace hjcd
