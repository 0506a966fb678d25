#include "common.cuh"
namespace mac {
bool match_fast_supported(const MacDecodeParams&) { return false; }
cudaError_t launch_match_bf16_d128(const MacDecodeParams&, cudaStream_t) { return cudaErrorNotSupported; }
}
