// Explicit instantiations: twisted single-series kernels, d = 3 (see whit_launch.cuh).
#define WHIT_LAUNCH_DEFS
#include "whit_launch.cuh"
namespace whit_detail {
#define WHIT_INST(IO, PD)                                                                  \
  template whit_status launch_tw<3, IO, PD, false, false>(const whit::Params&, cudaStream_t); \
  template whit_status launch_tw<3, IO, PD, true, false>(const whit::Params&, cudaStream_t);  \
  template whit_status launch_tw<3, IO, PD, false, true>(const whit::Params&, cudaStream_t);  \
  template whit_status launch_tw<3, IO, PD, true, true>(const whit::Params&, cudaStream_t);
WHIT_INST(float, true)
WHIT_INST(float, false)
WHIT_INST(double, true)
WHIT_INST(double, false)
}  // namespace whit_detail
