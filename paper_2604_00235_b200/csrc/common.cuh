// Shared device helpers for the MAC-Attention decode kernels (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "macattn.h"

namespace mac {

// ---------------------------------------------------------------------------
// storage-mode traits: K/V cache + query ring dtype, summary dtype, math dtype
// ---------------------------------------------------------------------------
template <int MODE> struct Traits;
template <> struct Traits<MAC_MODE_F32> {
  using kv_t = float;    // kvstore.py:113-115 f32 rounding
  using sum_t = float;   // engine.py:397-399 prefix.astype(f32)
  using acc_t = float;   // in-kernel accumulation
  using dist_t = double; // match distances (reference: f64)
};
template <> struct Traits<MAC_MODE_BF16> {
  using kv_t = __nv_bfloat16;
  using sum_t = float;
  using acc_t = float;
  using dist_t = float;
};
template <> struct Traits<MAC_MODE_F64> {
  using kv_t = double;
  using sum_t = double;
  using acc_t = double;
  using dist_t = double;
};

// ---------------------------------------------------------------------------
// conversions (round-to-nearest-even everywhere, like numpy astype)
// ---------------------------------------------------------------------------
template <typename T> __device__ __forceinline__ double to_f64(T x) { return (double)x; }
template <> __device__ __forceinline__ double to_f64<__nv_bfloat16>(__nv_bfloat16 x) {
  return (double)__bfloat162float(x);
}
template <typename T> __device__ __forceinline__ float to_f32(T x) { return (float)x; }
template <> __device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 x) {
  return __bfloat162float(x);
}
template <typename A, typename T> __device__ __forceinline__ A to_acc(T x) {
  return (A)to_f64(x);
}
template <> __device__ __forceinline__ float to_acc<float, float>(float x) { return x; }
template <> __device__ __forceinline__ float to_acc<float, __nv_bfloat16>(__nv_bfloat16 x) {
  return __bfloat162float(x);
}

template <typename T> __device__ __forceinline__ T from_f64(double x);
template <> __device__ __forceinline__ double from_f64<double>(double x) { return x; }
template <> __device__ __forceinline__ float from_f64<float>(double x) { return __double2float_rn(x); }
template <> __device__ __forceinline__ __nv_bfloat16 from_f64<__nv_bfloat16>(double x) {
  // double -> f32 -> bf16 is a double rounding; inputs that reach this path are
  // either f32-exact (bf16 mode inputs) or rounded once more by design.
  return __float2bfloat16_rn(__double2float_rn(x));
}

// element load from an input tensor of runtime dtype (MAC_DT_*)
__device__ __forceinline__ double load_in(const void* p, int64_t i, int dt) {
  if (dt == MAC_DT_F32) return (double)static_cast<const float*>(p)[i];
  if (dt == MAC_DT_BF16) return (double)__bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]);
  return static_cast<const double*>(p)[i];
}

// ---------------------------------------------------------------------------
// math helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ float fexp(float x) { return __expf(x); }
__device__ __forceinline__ double fexp(double x) { return exp(x); }
__device__ __forceinline__ float flog(float x) { return __logf(x); }
__device__ __forceinline__ double flog(double x) { return log(x); }

template <typename T> __device__ __forceinline__ T neg_inf();
template <> __device__ __forceinline__ float neg_inf<float>() { return -CUDART_INF_F; }
template <> __device__ __forceinline__ double neg_inf<double>() { return -CUDART_INF; }

// np.logaddexp: max + log1p(exp(-|a-b|)); either side -inf is the identity
__device__ __forceinline__ double logaddexp(double a, double b) {
  if (a == -CUDART_INF) return b;
  if (b == -CUDART_INF) return a;
  double mx = a > b ? a : b, mn = a > b ? b : a;
  return mx + log1p(exp(mn - mx));
}

template <typename T> __device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <typename T> __device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ---------------------------------------------------------------------------
// step geometry shared by amend and complete (must agree bit for bit)
// ---------------------------------------------------------------------------
// first token a head reads: hit -> max(1, p - r + 1), miss -> 1 (engine.py:466,485)
__device__ __forceinline__ int head_lo(int use, int p, int r) {
  if (!use) return 1;
  int lo = p - r + 1;
  return lo < 1 ? 1 : lo;
}

struct Chunking {
  int n;    // number of splits
  int len;  // tokens per split (last may be shorter)
};
// split [lo, m] (span tokens) into at most max_chunks pieces of >= min_chunk tokens,
// lengths rounded up to a multiple of 16
__host__ __device__ __forceinline__ Chunking chunking(int span, int max_chunks, int min_chunk) {
  Chunking c;
  if (span <= 0) { c.n = 0; c.len = 0; return c; }
  int n = (span + min_chunk - 1) / min_chunk;
  if (n > max_chunks) n = max_chunks;
  if (n < 1) n = 1;
  int len = (span + n - 1) / n;
  len = (len + 15) & ~15;
  c.len = len;
  c.n = (span + len - 1) / len;
  return c;
}

// first token of a group's split grid: max(lo_g, first local token) rounded down
// to a 16-token boundary in shard-local coordinates, so every 16-token sub-tile
// lies inside one KV page (page_size % 16 == 0).  Tokens below a head's own
// lo_h are masked by the kernels, so the rounding never changes a result.
__host__ __device__ __forceinline__ int grid_start(int lo_g, int kv_offset) {
  int local = lo_g - kv_offset;
  if (local < 1) local = 1;
  local = ((local - 1) & ~15) + 1;
  return local + kv_offset;
}

// physical row of token t (1-based, local to this KV shard) in a paged cache
__device__ __forceinline__ int64_t kv_row(const int32_t* __restrict__ page_table, int pages_per_seq,
                                          int b, int t, int page_size, int n_kv, int kvh) {
  int idx = t - 1;
  int page = page_table[(int64_t)b * pages_per_seq + idx / page_size];
  return ((int64_t)page * n_kv + kvh) * page_size + (idx % page_size);
}

// workspace layout (bytes, 256-aligned sections)
// mkey/marr (match keys and arrival counters) must start zeroed: the engine
// clears the workspace once at allocation and the match kernel re-zeroes them.
struct Workspace {
  size_t mkey_off, marr_off, mpos_off, qrot_off, part_off, total;
};
__host__ __device__ __forceinline__ size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }
__host__ __forceinline__ Workspace workspace_layout(const MacDecodeParams& p) {
  size_t acc = p.storage == MAC_MODE_F64 ? 8 : 4;
  Workspace w;
  const size_t rows = (size_t)p.batch * p.n_q_heads;
  w.mkey_off = 0;
  w.marr_off = align256(w.mkey_off + sizeof(unsigned long long) * rows);
  w.mpos_off = align256(w.marr_off + sizeof(unsigned int) * rows);
  w.qrot_off = align256(w.mpos_off + sizeof(int32_t) * (size_t)p.batch);
  w.part_off = align256(w.qrot_off + acc * (size_t)p.batch * p.n_q_heads * p.head_dim);
  size_t part = acc * (size_t)p.batch * p.n_q_heads * p.max_chunks * 2 * (p.head_dim_v + 1);
  w.total = align256(w.part_off + part);
  return w;
}

}  // namespace mac
