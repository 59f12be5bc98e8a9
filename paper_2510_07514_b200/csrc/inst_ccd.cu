// inst_ccd.cu — explicit instantiations of the classic-CCD launcher (see dispatch.cu)
#include "ccd.cuh"

namespace hjcd {
template cudaError_t launch_ccd_t<7, true>(const DevRobot&, const DevCfg&, const float*, int, const float*, float*,
                                           float*, int32_t*, cudaStream_t);
template cudaError_t launch_ccd_t<8, false>(const DevRobot&, const DevCfg&, const float*, int, const float*, float*,
                                            float*, int32_t*, cudaStream_t);
template cudaError_t launch_ccd_t<16, false>(const DevRobot&, const DevCfg&, const float*, int, const float*, float*,
                                             float*, int32_t*, cudaStream_t);
template cudaError_t launch_ccd_t<32, false>(const DevRobot&, const DevCfg&, const float*, int, const float*, float*,
                                             float*, int32_t*, cudaStream_t);
}  // namespace hjcd
