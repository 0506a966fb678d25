// K1 fast path — bf16 ring, d = 128, pre-RoPE matching.
//
// Same rule as match.cu (matching.py:141-175; engine.py:449-459), laid out for
// HBM streaming: each (request, head) ring scan (W x 256 B contiguous) is split
// over ceil(W / 256) CTAs of 256 threads.  A half-warp owns one ring row per
// load: every lane streams 16 B (8 dims) with a cache-streaming 128-bit load,
// 16 loads in flight per thread; Sum (q - c)^2 is accumulated in fp32 and
// reduced with 4 xor-shuffles.  CTAs combine with one 64-bit atomicMax of the
// complemented key (dist_bits << 32 | ~pos): the max of ~key is the min
// distance, ties to the larger position (matching.py:171-173).  The last CTA
// of a (request, head) — found with a per-row arrival counter — applies the
// threshold and the gates, writes the decision and resets key and counter to
// zero for the next step (graph-replay safe, no host memset).
#include "common.cuh"

namespace mac {

namespace {
constexpr int kThreads = 256;
constexpr int kRowsPerCta = 256;           // ring rows per CTA
constexpr int kIters = kRowsPerCta / 16;   // 8 warps x 2 rows per load instruction

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

__device__ __forceinline__ float dist8(const float* q, uint4 c) {
  float acc = 0.f;
  uint32_t w[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float lo = __uint_as_float(w[i] << 16);
    float hi = __uint_as_float(w[i] & 0xffff0000u);
    float e0 = q[2 * i] - lo, e1 = q[2 * i + 1] - hi;
    acc = fmaf(e0, e0, acc);
    acc = fmaf(e1, e1, acc);
  }
  return acc;
}
}  // namespace

__global__ void __launch_bounds__(kThreads) match_bf16_d128_kernel(MacDecodeParams p,
                                                                   const int32_t* __restrict__ mpos,
                                                                   unsigned long long* __restrict__ keys,
                                                                   unsigned int* __restrict__ arrivals, int nsplit) {
  const int bh = blockIdx.x / nsplit, split = blockIdx.x % nsplit;
  const int b = bh / p.n_q_heads;
  const int W = p.window;
  const int m = mpos[b];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, sub = lane & 15, half = lane >> 4;

  float q[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) q[i] = (float)load_in(p.q_pre, (int64_t)bh * 128 + sub * 8 + i, p.in_dtype);

  int first = m - W;
  if (first < 1) first = 1;
  if (p.delta_max > 0 && m - p.delta_max > first) first = m - p.delta_max;
  const int last = m - 1;
  const int n_scan = last >= first ? last - first + 1 : 0;

  const uint4* ring = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(p.ring_q) +
                                                     (int64_t)bh * W * 128);
  const int row0 = split * kRowsPerCta;
  float best = CUDART_INF_F;
  int bpos = -1;
  uint4 v[kIters];
#pragma unroll
  for (int k = 0; k < kIters; ++k) {
    int slot = row0 + k * 16 + warp * 2 + half;
    v[k] = slot < W ? ld_stream(ring + (int64_t)slot * 16 + sub) : make_uint4(0, 0, 0, 0);
  }
#pragma unroll
  for (int k = 0; k < kIters; ++k) {
    int slot = row0 + k * 16 + warp * 2 + half;
    float d = dist8(q, v[k]);
    d += __shfl_xor_sync(0xffffffffu, d, 8);
    d += __shfl_xor_sync(0xffffffffu, d, 4);
    d += __shfl_xor_sync(0xffffffffu, d, 2);
    d += __shfl_xor_sync(0xffffffffu, d, 1);
    // position held by this slot: the latest pos <= last with (pos - 1) % W == slot
    int pos = last - ((last - 1 - slot) % W + W) % W;
    bool live = slot < W && last >= 1 && pos >= first;
    if (live && (d < best || (d == best && pos > bpos))) { best = d; bpos = pos; }
  }
  // reduce (best, bpos) over the block
  unsigned long long key = 0ull;  // complemented packed key; 0 = nothing
  if (bpos >= 0) key = ~(((unsigned long long)__float_as_uint(best) << 32) | (unsigned long long)(0xffffffffu - (unsigned)bpos));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
    key = other > key ? other : key;
  }
  __shared__ unsigned long long wkey[kThreads / 32];
  __shared__ bool is_last;
  if (lane == 0) wkey[warp] = key;
  __syncthreads();
  if (tid == 0) {
    unsigned long long k2 = wkey[0];
    for (int w = 1; w < kThreads / 32; ++w) k2 = wkey[w] > k2 ? wkey[w] : k2;
    if (k2) atomicMax(keys + bh, k2);
    __threadfence();
    unsigned prev = atomicAdd(arrivals + bh, 1u);
    is_last = (prev == (unsigned)nsplit - 1);
  }
  __syncthreads();
  if (!is_last || tid != 0) return;
  __threadfence();
  unsigned long long k3 = atomicExch(keys + bh, 0ull);
  arrivals[bh] = 0u;
  float bdist = CUDART_INF_F;
  int pp_best = -1;
  if (k3) {
    unsigned long long raw = ~k3;
    bdist = __uint_as_float((unsigned)(raw >> 32));
    pp_best = (int)(0xffffffffu - (unsigned)(raw & 0xffffffffull));
  }
  const bool hit = n_scan > 0 && pp_best > 0 && (double)bdist < p.thr_sq;
  const int pp = hit ? pp_best : -1;
  bool use = hit;
  if (use && p.roi_gate && !((double)pp * p.roi_b_kv >= (double)W * p.roi_b_q + (double)p.band * p.roi_b_kv))
    use = false;
  if (p.refresh_every > 0 && m % p.refresh_every == 0) use = false;
  if (p.force_miss) use = false;
  p.match_hit[bh] = hit;
  p.match_pos[bh] = pp;
  p.match_dist[bh] = n_scan > 0 ? (double)bdist : CUDART_INF;
  p.match_scanned[bh] = n_scan;
  p.use_hit[bh] = use;
}

bool match_fast_supported(const MacDecodeParams& p) {
  return p.storage == MAC_MODE_BF16 && p.head_dim == 128 && p.match_space == MAC_MATCH_PRE_ROPE;
}

cudaError_t launch_match_bf16_d128(const MacDecodeParams& p, cudaStream_t st) {
  Workspace w = workspace_layout(p);
  char* ws = static_cast<char*>(p.workspace);
  const int nsplit = (p.window + kRowsPerCta - 1) / kRowsPerCta;
  match_bf16_d128_kernel<<<p.batch * p.n_q_heads * nsplit, kThreads, 0, st>>>(
      p, reinterpret_cast<const int32_t*>(ws + w.mpos_off), reinterpret_cast<unsigned long long*>(ws + w.mkey_off),
      reinterpret_cast<unsigned int*>(ws + w.marr_off), nsplit);
  return cudaGetLastError();
}

}  // namespace mac
