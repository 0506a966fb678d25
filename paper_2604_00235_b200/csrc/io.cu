// Step I/O over the host link without the copy engines: a kernel that moves a step's
// inputs from pinned host memory to the device, or its output back (narrowing f32 to
// bf16 on the way), by loading / storing the pinned buffer through its device alias
// (UVA zero-copy).  For the ~0.3-0.4 MB per step of a decode step this costs less than a
// cudaMemcpyAsync pair (tools/zerocopy_probe.cu: 18 vs 30 us for both legs on B200 /
// PCIe 5 x16) and folds the output narrowing into the transfer.  Used by StepGraph.
#include <stdint.h>

#include "common.cuh"

namespace mac {
namespace {

__global__ void __launch_bounds__(256) io_copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                      size_t n16) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// 8 floats -> 8 bf16 (one 16-byte store) per thread-iteration
__global__ void __launch_bounds__(256) io_narrow_kernel(const float4* __restrict__ src, uint4* __restrict__ dst,
                                                        size_t n8) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n8; i += (size_t)gridDim.x * blockDim.x) {
    const float4 a = src[2 * i], b = src[2 * i + 1];
    __nv_bfloat162 r[4] = {__floats2bfloat162_rn(a.x, a.y), __floats2bfloat162_rn(a.z, a.w),
                           __floats2bfloat162_rn(b.x, b.y), __floats2bfloat162_rn(b.z, b.w)};
    dst[i] = *reinterpret_cast<const uint4*>(r);
  }
}

}  // namespace
}  // namespace mac

using namespace mac;

extern "C" {

int mac_host_alias(void* host, void** device_alias) {
  if (!host || !device_alias) return MAC_ERR_NULL;
  return (int)cudaHostGetDevicePointer(device_alias, host, 0);
}

int mac_io_copy(const void* src, int32_t src_dtype, void* dst, int32_t dst_dtype, size_t n_elems, void* stream) {
  if (!src || !dst) return MAC_ERR_NULL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uintptr_t al = reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst);
  if (al & 15) return MAC_ERR_SHAPE;
  const int grid = 296;  // 2 CTAs per SM: enough loads in flight to cover the host link's latency
  if (src_dtype == dst_dtype) {
    const size_t esz = src_dtype == MAC_DT_F64 ? 8 : (src_dtype == MAC_DT_F32 ? 4 : 2);
    if ((n_elems * esz) & 15) return MAC_ERR_SHAPE;
    if (n_elems == 0) return 0;
    io_copy_kernel<<<grid, 256, 0, st>>>(static_cast<const uint4*>(src), static_cast<uint4*>(dst), n_elems * esz / 16);
    return (int)cudaGetLastError();
  }
  if (src_dtype == MAC_DT_F32 && dst_dtype == MAC_DT_BF16) {
    if (n_elems & 7) return MAC_ERR_SHAPE;
    if (n_elems == 0) return 0;
    io_narrow_kernel<<<grid, 256, 0, st>>>(static_cast<const float4*>(src), static_cast<uint4*>(dst), n_elems / 8);
    return (int)cudaGetLastError();
  }
  return MAC_ERR_DTYPE;
}

}  // extern "C"
