// Explicit instantiations: single-series daily-grid kernels, d = 3, double I/O (see whit_launch.cuh).
#define WHIT_LAUNCH_DEFS
#include "whit_launch.cuh"
namespace whit_detail {
#define WHIT_INST(PD)                                                                        \
  template whit_status launch<3, double, PD, false, false, false>(const whit::Params&, cudaStream_t); \
  template whit_status launch<3, double, PD, true, false, false>(const whit::Params&, cudaStream_t);  \
  template whit_status launch<3, double, PD, false, true, false>(const whit::Params&, cudaStream_t);  \
  template whit_status launch<3, double, PD, false, false, true>(const whit::Params&, cudaStream_t);  \
  template whit_status launch<3, double, PD, true, false, true>(const whit::Params&, cudaStream_t);
WHIT_INST(true)
WHIT_INST(false)
}  // namespace whit_detail
