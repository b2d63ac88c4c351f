// Explicit instantiations: posterior-variance kernels (see whit_launch.cuh).
#define WHIT_LAUNCH_DEFS
#include "whit_launch.cuh"
namespace whit_detail {
#define WHIT_INST(D)                                                                     \
  template whit_status launch_var<D, float, true>(const whit::Params&, cudaStream_t);   \
  template whit_status launch_var<D, float, false>(const whit::Params&, cudaStream_t);  \
  template whit_status launch_var<D, double, true>(const whit::Params&, cudaStream_t);  \
  template whit_status launch_var<D, double, false>(const whit::Params&, cudaStream_t);
WHIT_INST(1)
WHIT_INST(2)
WHIT_INST(3)
}  // namespace whit_detail
