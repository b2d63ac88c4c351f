// Explicit instantiations: single-series irregular-grid kernels (see whit_launch.cuh).
#define WHIT_LAUNCH_DEFS
#include "whit_launch.cuh"
namespace whit_detail {
#define WHIT_INST(D, IO, PD)                                                                  \
  template whit_status launch_irr<D, IO, PD, false>(const whit::Params&, cudaStream_t); \
  template whit_status launch_irr<D, IO, PD, true>(const whit::Params&, cudaStream_t);
#define WHIT_INST_D(D) WHIT_INST(D, float, true) WHIT_INST(D, float, false) WHIT_INST(D, double, true) WHIT_INST(D, double, false)
WHIT_INST_D(1)
WHIT_INST_D(2)
WHIT_INST_D(3)
}  // namespace whit_detail
