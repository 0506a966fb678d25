// K0 + K1 fast path ("front" kernel) — bf16 storage, d = 128, pre-RoPE matching.
//
// One launch does the step's KV append with in-kernel RoPE (engine.py:434-437,
// attention.py:212-232; same math as append.cu) and the ring match
// (matching.py:141-175; engine.py:449-459; same rule as match.cu), and its
// epilogue plans the amend work (decide_head -> plan_group, common.cuh).
//
// Match layout: the query ring [B, Hq, W, 128] bf16 is one contiguous stream
// of 256 B rows.  A CTA of 256 threads owns 128 consecutive ring rows of one
// (request, head) (32 KiB); a half-warp owns one row per load, every lane
// streams 16 B (8 dims) with a cache-streaming 128-bit load, all 8 loads in
// flight before any math.  The kernel keeps <= 48 registers so 5 CTAs (40 warps) sit
// on an SM: on B200 a short (<= 300 MB) read stream is paced by thread-level
// parallelism, not by per-warp pipelining (tools/stream_probe.cu).
// Sum (q - c)^2 is accumulated in fp32 and reduced with 4 xor-shuffles.  CTAs
// publish (best, pos) with one 64-bit atomicMax of the complemented key
// (dist_bits << 32 | ~pos): max ~key = min distance, ties to the larger
// position (matching.py:171-173).  The CTA completing the per-(request, head)
// arrival count decides the head (decide_head) and resets key and counter to
// zero for the next step (graph-replay safe).  The step's KV appends (one
// warp per (request, kv head)) ride in the same launch.
#include <stdlib.h>

#include "front.cuh"

namespace mac {

namespace {
constexpr int kThreads = 256;

__device__ __forceinline__ float dist8(const float* q, uint4 c) {
  float acc = 0.f;
  const uint32_t w[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float lo = __uint_as_float(w[i] << 16);
    const float hi = __uint_as_float(w[i] & 0xffff0000u);
    const float e0 = q[2 * i] - lo, e1 = q[2 * i + 1] - hi;
    acc = fmaf(e0, e0, acc);
    acc = fmaf(e1, e1, acc);
  }
  return acc;
}

}  // namespace

template <int kRowsPerCta, int kMinBlocks>
__global__ void __launch_bounds__(kThreads, kMinBlocks) front_bf16_d128_kernel(MacDecodeParams p, int n_match,
                                                                               int do_append, int rotate_only,
                                                                               int plan) {
  constexpr int kLoads = kRowsPerCta / 16;  // per thread: 8 warps x 2 rows per load instruction
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // the first n_append CTAs append (one warp per (request, kv head)); they are
  // scheduled first so their latency hides under the ring stream
  const int n_append = do_append ? (p.batch * p.n_kv_heads + kThreads / 32 - 1) / (kThreads / 32) : 0;
  if ((int)blockIdx.x < n_append) {
    const int i = blockIdx.x * (kThreads / 32) + warp;
    if (i < p.batch * p.n_kv_heads) append_warp(p, i, rotate_only, plan);
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    return;
  }
  const int W = p.window;
  const int nsplit = (W + kRowsPerCta - 1) / kRowsPerCta;
  const int bh = (blockIdx.x - n_append) / nsplit, split = (blockIdx.x - n_append) % nsplit;
  const int b = bh / p.n_q_heads;
  const int m = p.seq_lens[b] + 1;
  const int sub = lane & 15, half = lane >> 4;
  const uint4* ring = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(p.ring_q) + (int64_t)bh * W * 128);
  const int row0 = split * kRowsPerCta;
  uint4 v[kLoads];
#pragma unroll
  for (int k = 0; k < kLoads; ++k) {
    const int slot = row0 + k * 16 + warp * 2 + half;
    v[k] = slot < W ? ld_stream(ring + (int64_t)slot * 16 + sub) : make_uint4(0, 0, 0, 0);
  }
  float q[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) q[i] = (float)load_in(p.q_pre, (int64_t)bh * 128 + sub * 8 + i, p.in_dtype);
  int first = m - W;
  if (first < 1) first = 1;
  if (p.delta_max > 0 && m - p.delta_max > first) first = m - p.delta_max;
  const int last = m - 1;
  const int n_scan = last >= first ? last - first + 1 : 0;
  const int cur_slot = last >= 1 ? (last - 1) % W : 0;  // slot of the newest ring entry
  float best = CUDART_INF_F;
  int bpos = -1;
#pragma unroll
  for (int k = 0; k < kLoads; ++k) {
    const int slot = row0 + k * 16 + warp * 2 + half;
    float d = dist8(q, v[k]);
    d += __shfl_xor_sync(0xffffffffu, d, 8);
    d += __shfl_xor_sync(0xffffffffu, d, 4);
    d += __shfl_xor_sync(0xffffffffu, d, 2);
    d += __shfl_xor_sync(0xffffffffu, d, 1);
    // latest position held by the slot: slots after the newest one hold the previous lap
    const int pos = last - cur_slot + slot - (slot > cur_slot ? W : 0);
    const bool live = slot < W && last >= 1 && pos >= first;
    if (live && (d < best || (d == best && pos > bpos))) { best = d; bpos = pos; }
  }
  unsigned long long key = 0ull;  // complemented packed key; 0 = nothing
  if (bpos > 0)
    key = ~(((unsigned long long)__float_as_uint(best) << 32) | (unsigned long long)(0xffffffffu - (unsigned)bpos));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
    key = other > key ? other : key;
  }
  __shared__ unsigned long long wkey[kThreads / 32];
  if (lane == 0) wkey[warp] = key;
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (tid != 0) return;
  for (int w = 1; w < kThreads / 32; ++w) key = wkey[w] > key ? wkey[w] : key;
  publish_and_decide(p, bh, m, n_scan, nsplit, key);
}

bool match_fast_supported(const MacDecodeParams& p) {
  return p.storage == MAC_MODE_BF16 && p.head_dim == 128 && p.head_dim_v == 128 && p.match_space == MAC_MATCH_PRE_ROPE;
}
bool front_fast_supported(const MacDecodeParams& p) {
  return p.storage == MAC_MODE_BF16 && p.head_dim == 128 && p.head_dim_v == 128;
}

// MAC_FRONT_VARIANT (development knob): (ring rows per CTA, min CTAs per SM) = (128,5) default,
// (64,8), (256,3).  Measured alternatives that lost on C3 (persistent tensor-core, persistent
// CUDA-core, f32x2 "lean", DSMEM-cluster argmin, one fused step kernel) are on branch
// exp/fused-step; numbers in DESIGN.md §4.
struct FrontVariant {
  void (*fn)(MacDecodeParams, int, int, int, int);
  int rows;
};
static const FrontVariant kFrontVariants[] = {
    {front_bf16_d128_kernel<128, 5>, 128}, {front_bf16_d128_kernel<64, 8>, 64},
    {front_bf16_d128_kernel<256, 3>, 256},
};

// append CTAs first (8 warps, one (request, kv head) each), then the match CTAs
cudaError_t launch_front_bf16(const MacDecodeParams& p, cudaStream_t st, bool do_match, bool do_append,
                              int rotate_only, int plan) {
  static int vi = -1;
  if (vi < 0) {
    const char* env = getenv("MAC_FRONT_VARIANT");
    vi = env ? atoi(env) : 0;
    if (vi < 0 || vi >= (int)(sizeof(kFrontVariants) / sizeof(kFrontVariants[0]))) vi = 0;
  }
  const FrontVariant& v = kFrontVariants[vi];
  const int n_match = do_match ? p.batch * p.n_q_heads * ((p.window + v.rows - 1) / v.rows) : 0;
  const int n_append = do_append ? (p.batch * p.n_kv_heads + 7) / 8 : 0;
  if (n_match + n_append == 0) return cudaSuccess;
  v.fn<<<n_match + n_append, kThreads, 0, st>>>(p, n_match, do_append ? 1 : 0, rotate_only, plan);
  return cudaGetLastError();
}

}  // namespace mac
