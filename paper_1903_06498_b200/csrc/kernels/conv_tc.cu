#include "../kernels.hpp"
namespace sb {
const char* conv_tc_unsupported(const ConvPlan&) { return "not built"; }
cudaError_t launch_conv_tc(const ConvPlan&, const ConvArgs&, cudaStream_t, int) { return cudaErrorNotSupported; }
}  // namespace sb
