// batched.cu — K8 (multi-RHS) placeholder; filled in below.
#include "kernels.cuh"
namespace alnnls {
cudaError_t launch_batched(const BatchArgs&, int, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace alnnls
