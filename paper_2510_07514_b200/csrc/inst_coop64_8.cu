// inst_coop64_8.cu — explicit instantiation(s) of the cooperative PJ-IK launcher, double (see dispatch.cu)
#include "pjik_coop.cuh"

namespace hjcd {
template cudaError_t launch_coop_t<double, 8, true>(const DevRobotT<double>&, const DevCfg&, const float*, int, const float*, double*, double*, double*, int32_t*, int32_t*, cudaStream_t, const StageLink&);
template cudaError_t launch_coop_t<double, 8, false>(const DevRobotT<double>&, const DevCfg&, const float*, int, const float*, double*, double*, double*, int32_t*, int32_t*, cudaStream_t, const StageLink&);
}  // namespace hjcd
