// inst_coop_18.cu — explicit instantiation of the cooperative PJ-IK launcher, float, exact n = 18 (see dispatch.cu)
#include "pjik_coop.cuh"

namespace hjcd {
template cudaError_t launch_coop_t<float, 18, true>(const DevRobotT<float>&, const DevCfg&, const float*, int, const float*, float*, float*, float*, int32_t*, int32_t*, cudaStream_t, const StageLink&);
}  // namespace hjcd
