// inst_poccd2_7.cu — explicit instantiation of the packed PO-CCD launcher (K17; see dispatch.cu)
#include "poccd_x2.cuh"

namespace hjcd {
template cudaError_t launch_poccd_x2_t<7, true>(const DevRobot&, const DevCfg&, const float*, int, float*, float*, float*, float*, int32_t*, TraceOut, uint32_t*, cudaStream_t);
}  // namespace hjcd
