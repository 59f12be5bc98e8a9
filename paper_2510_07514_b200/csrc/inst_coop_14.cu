// inst_coop_14.cu — explicit instantiation(s) of the cooperative PJ-IK launcher, float (see dispatch.cu)
#include "pjik_coop.cuh"

namespace hjcd {
template cudaError_t launch_coop_t<float, 14, true>(const DevRobotT<float>&, const DevCfg&, const float*, int, const float*, float*, float*, float*, int32_t*, int32_t*, cudaStream_t, const StageLink&);
}  // namespace hjcd
