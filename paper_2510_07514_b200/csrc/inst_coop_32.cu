// inst_coop_32.cu — explicit instantiation(s) of the pjik_coop.cuh launcher (see dispatch.cu)
#include "pjik_coop.cuh"

namespace hjcd {
template cudaError_t launch_coop_t<32, false>(const DevRobot&, const DevCfg&, const float*, int, const float*, float*, float*, float*, int32_t*, int32_t*, cudaStream_t);
}  // namespace hjcd
