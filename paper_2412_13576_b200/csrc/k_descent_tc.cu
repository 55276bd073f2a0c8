// tcgen05 descent kernel (placeholder until the tensor-core path lands).
#include "kernels.h"
namespace maple {
bool descent_tc_supported(int, int) { return false; }
cudaError_t launch_descent_tc(const DescentParams&, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace maple
