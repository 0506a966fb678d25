// K3 — complete, standalone kernel: one warp per (request, q head), 4 heads
// per CTA (the per-head logic is complete.cuh).  Used by the generic path and
// by the stage-wise API; the bf16 fast path runs it fused in the amend tail.
#include "complete.cuh"

namespace mac {

template <int MODE>
__global__ void __launch_bounds__(128) complete_kernel(MacDecodeParams p, int full_mode) {
  // programmatic dependent launch: the grid is set up while the amend kernel drains
  TL_MARK(p, TL_COMPLETE_IN);
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  TL_MARK(p, TL_COMPLETE_WAITED);
  const int bh = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (bh < p.batch * p.n_q_heads) complete_head<MODE>(p, bh, full_mode);
#ifdef MAC_TIMELINE
  __syncthreads();
#endif
  TL_MARK(p, TL_COMPLETE_OUT);
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // work list consumed: list length and amend claim counter
    unsigned int* ctr = ws_ptr<unsigned int>(p, workspace_layout(p).ctr_off);
    ctr[0] = 0u;
    ctr[1] = 0u;
  }
}

template <int MODE>
cudaError_t launch_complete(const MacDecodeParams& p, cudaStream_t st, int full_mode) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((p.batch * p.n_q_heads + 3) / 4);
  cfg.blockDim = dim3(128);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, complete_kernel<MODE>, p, full_mode);
}

template cudaError_t launch_complete<MAC_MODE_F32>(const MacDecodeParams&, cudaStream_t, int);
template cudaError_t launch_complete<MAC_MODE_BF16>(const MacDecodeParams&, cudaStream_t, int);
template cudaError_t launch_complete<MAC_MODE_F64>(const MacDecodeParams&, cudaStream_t, int);

}  // namespace mac
