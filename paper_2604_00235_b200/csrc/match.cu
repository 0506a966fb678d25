// K1 — nearest-neighbour match of the pre-RoPE query against the W-entry ring.
//
// Reference: matching.py:141-175 (match_query) and engine.py:449-459 (gates).
//   live ring rows      positions max(1, m-W) .. m-1, slot (pos-1) % W
//   delta_max filter    m - pos <= delta_max           (matching.py:160-164)
//   post-RoPE ablation  candidate rotated by (pos-m)*omega (matching.py:165-168)
//   distance            ||q - c||^2 (the reference expands it in f64 and clamps
//                       at 0; the direct form is non-negative by construction)
//   decision            argmin, exact ties -> larger position (matching.py:171-173),
//                       hit iff best < thr^2 strictly (matching.py:174)
//   gates               break-even (engine.py:57-63,453-455), refresh (:456-459)
//
// The ring is [B, Hq, W, d] so one (request, head) scan is a contiguous W*d
// stream.  Generic kernel: one CTA per (request, head), one warp per ring row,
// lanes across the head dim; the bf16 d=128 fast path lives in match_fast.cu.
#include "common.cuh"

namespace mac {

template <typename D>
__device__ __forceinline__ bool better(D d, int pos, D bd, int bpos) {
  return d < bd || (d == bd && pos > bpos);
}

template <int MODE>
__global__ void __launch_bounds__(256) match_generic_kernel(MacDecodeParams p, const int32_t* __restrict__ mpos) {
  using kv_t = typename Traits<MODE>::kv_t;
  using dist_t = typename Traits<MODE>::dist_t;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  dist_t* qs = reinterpret_cast<dist_t*>(smem_raw);                   // [d]
  __shared__ dist_t wbest[32];
  __shared__ int wpos[32];

  const int bh = blockIdx.x;
  const int b = bh / p.n_q_heads;
  const int d = p.head_dim, W = p.window, half = d / 2;
  const int m = mpos[b];
  for (int k = threadIdx.x; k < d; k += blockDim.x) qs[k] = (dist_t)load_in(p.q_pre, (int64_t)bh * d + k, p.in_dtype);
  __syncthreads();

  int first = m - W;
  if (first < 1) first = 1;
  if (p.delta_max > 0 && m - p.delta_max > first) first = m - p.delta_max;
  const int last = m - 1;
  const int n_scan = last >= first ? last - first + 1 : 0;

  const kv_t* ring = static_cast<const kv_t*>(p.ring_q) + (int64_t)bh * W * d;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  dist_t best = (dist_t)CUDART_INF;
  int bpos = -1;
  for (int pos = last - warp; pos >= first; pos -= nwarps) {
    const kv_t* c = ring + (int64_t)((pos - 1) % W) * d;
    dist_t acc = 0;
    if (p.match_space == MAC_MATCH_PRE_ROPE) {
      for (int k = lane; k < d; k += 32) {
        dist_t e = qs[k] - (dist_t)to_f64(c[k]);
        acc += e * e;
      }
    } else {
      // rotate the candidate into the query's frame: R(pos - m) (matching.py:129-138,165-168)
      for (int j = lane; j < half; j += 32) {
        double s, co;
        sincos((double)(pos - m) * p.rope_freqs[j], &s, &co);
        double c0 = to_f64(c[2 * j]), c1 = to_f64(c[2 * j + 1]);
        dist_t e0 = qs[2 * j] - (dist_t)(c0 * co - c1 * s);
        dist_t e1 = qs[2 * j + 1] - (dist_t)(c0 * s + c1 * co);
        acc += e0 * e0 + e1 * e1;
      }
    }
    acc = warp_sum(acc);
    if (better(acc, pos, best, bpos)) { best = acc; bpos = pos; }
  }
  if (lane == 0) { wbest[warp] = best; wpos[warp] = bpos; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < nwarps; ++w)
      if (better(wbest[w], wpos[w], best, bpos)) { best = wbest[w]; bpos = wpos[w]; }
    decide_head(p, bh, m, n_scan, bpos > 0, (double)best, bpos);
  }
}

template <int MODE>
cudaError_t launch_match_generic(const MacDecodeParams& p, cudaStream_t st) {
  Workspace w = workspace_layout(p);
  const int32_t* mpos = reinterpret_cast<const int32_t*>(static_cast<char*>(p.workspace) + w.mpos_off);
  size_t smem = sizeof(typename Traits<MODE>::dist_t) * (size_t)p.head_dim;
  match_generic_kernel<MODE><<<p.batch * p.n_q_heads, 256, smem, st>>>(p, mpos);
  return cudaGetLastError();
}

template cudaError_t launch_match_generic<MAC_MODE_F32>(const MacDecodeParams&, cudaStream_t);
template cudaError_t launch_match_generic<MAC_MODE_BF16>(const MacDecodeParams&, cudaStream_t);
template cudaError_t launch_match_generic<MAC_MODE_F64>(const MacDecodeParams&, cudaStream_t);

}  // namespace mac
