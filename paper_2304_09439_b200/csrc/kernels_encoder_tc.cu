// kernels_encoder_tc.cu — placeholder until the tcgen05 encoder lands.
#include <cuda_runtime.h>
#include "internal.h"
namespace locc {
cudaError_t launch_encoder_tc(const DevParams&, const Batch&, int, cudaStream_t) { return cudaErrorNotSupported; }
size_t encoder_tc_smem_bytes() { return 0; }
}  // namespace locc
