#include "common.cuh"
namespace mac {
bool amend_mma_supported(const MacDecodeParams&) { return false; }
cudaError_t launch_amend_mma_bf16(const MacDecodeParams&, cudaStream_t) { return cudaErrorNotSupported; }
}
