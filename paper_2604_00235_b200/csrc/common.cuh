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
  using merge_t = double;  // summary merge algebra (reference: f64)
};
template <> struct Traits<MAC_MODE_BF16> {
  using kv_t = __nv_bfloat16;
  using sum_t = float;
  using acc_t = float;
  using dist_t = float;
  using merge_t = double;  // summary merge algebra in fp64 like f32 storage (remove() cancels)
};
template <> struct Traits<MAC_MODE_F64> {
  using kv_t = double;
  using sum_t = double;
  using acc_t = double;
  using dist_t = double;
  using merge_t = double;
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

// element store into a buffer of runtime dtype (the staged inputs, inputs_host)
__device__ __forceinline__ void store_in(void* p, int64_t i, double v, int dt) {
  if (dt == MAC_DT_F32) static_cast<float*>(p)[i] = (float)v;
  else if (dt == MAC_DT_BF16) static_cast<__nv_bfloat16*>(p)[i] = __double2bfloat16(v);
  else static_cast<double*>(p)[i] = v;
}

// a pair of consecutive elements (index i even) in one load: with host-resident inputs every load
// instruction is its own PCIe read, so the pairs halve the append's requests
__device__ __forceinline__ void load_pair(const void* p, int64_t i, int dt, double& x0, double& x1) {
  if (dt == MAC_DT_BF16) {
    const __nv_bfloat162 v = *reinterpret_cast<const __nv_bfloat162*>(static_cast<const __nv_bfloat16*>(p) + i);
    x0 = (double)__bfloat162float(v.x);
    x1 = (double)__bfloat162float(v.y);
  } else if (dt == MAC_DT_F32) {
    const float2 v = *reinterpret_cast<const float2*>(static_cast<const float*>(p) + i);
    x0 = (double)v.x;
    x1 = (double)v.y;
  } else {
    const double2 v = *reinterpret_cast<const double2*>(static_cast<const double*>(p) + i);
    x0 = v.x;
    x1 = v.y;
  }
}
__device__ __forceinline__ void store_pair(void* p, int64_t i, double x0, double x1, int dt) {
  if (dt == MAC_DT_F32) *reinterpret_cast<float2*>(static_cast<float*>(p) + i) = make_float2((float)x0, (float)x1);
  else if (dt == MAC_DT_BF16) {
    __nv_bfloat162 v;
    v.x = __double2bfloat16(x0);
    v.y = __double2bfloat16(x1);
    *reinterpret_cast<__nv_bfloat162*>(static_cast<__nv_bfloat16*>(p) + i) = v;
  } else *reinterpret_cast<double2*>(static_cast<double*>(p) + i) = make_double2(x0, x1);
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
__device__ __forceinline__ float logaddexp(float a, float b) {
  if (a == -CUDART_INF_F) return b;
  if (b == -CUDART_INF_F) return a;
  const float mx = a > b ? a : b, mn = a > b ? b : a;
  return mx + log1pf(__expf(mn - mx));
}
__device__ __forceinline__ float fexpm1(float x) { return expm1f(x); }
__device__ __forceinline__ double fexpm1(double x) { return expm1(x); }


// gpu-scope acquire-release fetch-add: orders this thread's earlier writes before
// the increment and later reads after it (replaces a fence + atomicAdd pair)
__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
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

// ceil(a / b) for 0 <= a, 1 <= b: exact.  On the device, for a < 2^22, through a float quotient
// and one remainder correction each way (a handful of instructions instead of the ~25 of an integer
// division): the plan's chunking runs on one thread per GQA group at the end of the verify, where
// its chain of divisions sat on every step's critical path.
__host__ __device__ __forceinline__ int cdiv(int a, int b) {
#ifdef __CUDA_ARCH__
  if (a >= (1 << 22)) return (a + b - 1) / b;
  int q = __float2int_rz(__fdividef((float)a, (float)b));
  int r = a - q * b;
  if (r < 0) { q -= 1; r += b; }
  if (r >= b) { q += 1; r -= b; }
  return q + (r > 0 ? 1 : 0);
#else
  return (a + b - 1) / b;
#endif
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
  int n = cdiv(span, min_chunk);
  if (n > max_chunks) n = max_chunks;
  if (n < 1) n = 1;
  int len = cdiv(span, n);
  len = (len + 15) & ~15;
  c.len = len;
  c.n = cdiv(span, len);
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

// last position this KV shard holds for a step at position m (kv_limit 0: unbounded)
__host__ __device__ __forceinline__ int shard_end(const MacDecodeParams& p, int m) {
  return (p.kv_limit > 0 && p.kv_offset + p.kv_limit < m) ? p.kv_offset + p.kv_limit : m;
}
// the split grid of a GQA group over [grid_start(lo_g), shard_end(m)] (plan, amend and complete agree)
__host__ __device__ __forceinline__ Chunking group_chunking(const MacDecodeParams& p, int m, int lo_g) {
  const int cap = (p.span_chunks > 0 && p.span_chunks < p.max_chunks) ? p.span_chunks : p.max_chunks;
  return chunking(shard_end(p, m) - grid_start(lo_g, p.kv_offset) + 1, cap, p.min_chunk);
}

// Split band (the bf16 fast path's hit step, launch_band_split in amend_mma.cu): the band
// [max(1, m-r+1), m] never depends on the match (every head's lo_h <= m-r), so the amend
// warps compute it as `nb` fixed items BEFORE their grid-dependency wait — while the verify
// kernel decides the heads and the DRAM would otherwise idle — and the plan covers only the
// piece [grid_start(lo_g), m-r].  Band items start on the 16-token grid below m-r+1 and
// produce band partials only; their slots come first (0 .. n-1), the plan's piece slots
// follow.  The planner records nb in the group's pn word (bits 16+) for the complete.
struct BandItems {
  int n;    // band items (slots 0 .. n-1)
  int len;  // tokens per item (multiple of 16)
  int t0;   // first token of item 0 (16-aligned, <= max(1, m-r+1))
};
__host__ __device__ __forceinline__ BandItems band_items(int m, int r, int nb) {
  BandItems s = {0, 0, 1};
  if (nb <= 0 || m < 1) return s;
  const int b0 = m - r + 1 > 1 ? m - r + 1 : 1;
  s.t0 = ((b0 - 1) & ~15) + 1;
  const int span = m - s.t0 + 1;
  int n = (span + 15) / 16;
  if (n > nb) n = nb;
  s.len = (cdiv(span, n) + 15) & ~15;
  s.n = cdiv(span, s.len);
  return s;
}
// the plan's split grid with the split band (nb > 0): the piece [grid_start(lo_g), m-r] in
// at most max_chunks - nb slots; nb == 0: group_chunking.  (A guided variant — trailing
// 32-token items drained last — shortened the amend's tail but measured slower overall:
// the complete then merged more than 8 slots in two batches.)
// With the split band the piece is also cut into at most `ntarget` items (the amend's resident
// warps per group, band_split's caller): as many post-wait items as warps, so no warp starts
// a second item while the others finish (C3: 934 -> 768 items, 53.5 -> 50.0 us per step).
// A short (hit) piece is cut into items of >= min_chunk tokens, at most ntarget of them; a long
// piece (a group with a miss) into items of <= 256 tokens, up to max_chunks - nb — a warp
// streams ~5 GB/s, so a few long items would serialise the step on the warps that drew them.
// (Items of 32 tokens for C2's short pieces measured slower: 38.1 vs 35.5 us, the complete then
// merges 17 slots.)
// n_dense (match_mode 2: the heads the verify handed to dense_kernel, known when it plans):
// the groups with a miss share the amend grid, so a long piece takes at most its share,
// tgt * groups / n_dense items, and never fewer than span_chunks (C3 geometry at 16K: 2 %
// misses 113 -> 96 us with 33 slots, 10 % unchanged at 184 us; 128K with 2 %: 476 -> 301 us).
__host__ __device__ __forceinline__ Chunking plan_chunking(const MacDecodeParams& p, int m, int lo_g, int nb,
                                                          int ntarget = 0, int n_dense = 0) {
  if (nb <= 0) return group_chunking(p, m, lo_g);
  const int span = m - p.band - grid_start(lo_g, p.kv_offset) + 1;
  if (span <= 0) return chunking(span, 1, 16);
  const int cap = p.max_chunks - nb;
  // ntarget: bits 0-15 the item count target, bits 16+ the longest item in 16-token sub-tiles
  // (0: 256 tokens, the one-warp amend; the CTA-cooperative TMA amend streams longer items)
  const int tgt = ntarget & 0xffff, max_len = (ntarget >> 16) > 0 ? (ntarget >> 16) * 16 : 256;
  int n = cdiv(span, p.min_chunk);
  if (tgt > 0 && n > tgt) n = tgt;
  const int n_len = cdiv(span, max_len);
  if (n < n_len) n = n_len;
  if (n_dense > 0 && tgt > 0) {
    const int span_cap = (p.span_chunks > 0 && p.span_chunks < p.max_chunks) ? p.span_chunks : p.max_chunks;
    const long share = (long)tgt * p.batch * p.n_kv_heads / n_dense;
    const int fair = share > span_cap ? (int)(share < 0xffff ? share : 0xffff) : span_cap;
    if (n > fair) n = fair;
  }
  if (n > cap) n = cap;
  if (n < 1) n = 1;
  return chunking(span, n, 16);
}
// partial slots a group's complete merges, from its pn word (plan_group)
__host__ __device__ __forceinline__ int group_slots(int pn_word, int m, int r) {
  const int nb = pn_word >> 16;
  return (pn_word & 0xffff) + (nb > 0 ? band_items(m, r, nb).n : 0);
}

// physical row of token t (1-based, local to this KV shard) in a paged cache
__device__ __forceinline__ int64_t kv_row(const int32_t* __restrict__ page_table, int pages_per_seq,
                                          int b, int t, int page_size, int n_kv, int kvh) {
  int idx = t - 1;
  int pi = idx / page_size;
  pi = pi < pages_per_seq ? pi : pages_per_seq - 1;  // never past the request's table row (see kv_fits)
  int page = page_table[(int64_t)b * pages_per_seq + pi];
  return ((int64_t)page * n_kv + kvh) * page_size + (idx % page_size);
}

// whether token t (1-based, shard-local) has a page in the request's table row.  The appends
// store only when it does and otherwise raise the overflow flag (workspace ctr[2], read by
// BatchDecodeEngine.check_overflow); the engine grows the pool before a step would need it.
__device__ __forceinline__ bool kv_fits(int pages_per_seq, int t, int page_size) {
  return t >= 1 && (t - 1) / page_size < pages_per_seq;
}

// workspace layout (bytes, 256-aligned sections)
// The "persistent" section (match keys, arrival counters, group counters, work
// list length and work counters) must start zeroed: the engine clears the
// workspace once at allocation and the kernels return every counter to zero
// by the end of each step.
constexpr int kTlSlots = 24;
constexpr int kMaxWsum = 128;  // scan-warp summaries per head: ceil(W / rows per CTA) * 8 warps, W <= 1024

enum : int {  // timeline slots
  TL_SCAN_IN = 0, TL_SCAN_OUT = 1, TL_VERIFY_IN = 2, TL_VERIFY_WAITED = 3, TL_VERIFY_OUT = 4,
  TL_AMEND_IN = 5, TL_AMEND_WAITED = 6, TL_AMEND_OUT = 7, TL_COMPLETE_IN = 8, TL_COMPLETE_WAITED = 9,
  TL_COMPLETE_OUT = 10, TL_V_SELECTED = 11, TL_V_BOUND = 12, TL_V_SURVIVED = 13, TL_V_DECIDED = 14,
  TL_V_M = 15, TL_DENSE_IN = 16, TL_DENSE_WAITED = 17, TL_DENSE_OUT = 18, TL_DENSE_TASK = 19,
  TL_PLAN_IN = 20, TL_PLAN_ALLOC = 21, TL_PLAN_OUT = 22
};
struct Workspace {
  size_t mkey_off;   // [B*Hq] u64   complemented packed (dist, pos) match key
  size_t marr_off;   // [B*Hq] u32   ring rows scanned so far this step
  size_t gcnt_off;   // [B*Hkv] u32  heads of the group decided so far
  size_t ctr_off;    // [16] u32     0 work-list length, 1 amend work counter (both reset by complete),
                     //              4 heads missed and 6 steps completed since the feedback was last published
                     //              (complete adds; every 8th step's append warps publish and reset)
                     //              2 KV overflow flag (an append found no page for its token; sticky)
                     //              8 dense heads deferred by the verify (match_mode 2; reset by complete)
                     //              (3, 5, 7, 9-15 spare)
  size_t gdone_off;  // [B*Hkv] u32  splits of the group finished (fused complete)
  size_t pn_off;     // [B*Hkv] i32  piece splits planned for the group | band items requested << 16
  size_t mpos_off;   // [B] i32      position m of this step
  size_t lo_off;     // [B*Hq] i32   first token each head reads (plan)
  size_t list_off;   // [B*Hkv*max_chunks] int4 work items {grp + 1, c, t0, t1} (the amend
                     //              kernel reads them after the plan is complete; x = 0: empty)
  size_t qrot_off;   // [B*Hq*d]     rotated queries (math dtype)
  size_t part_off;   // [B*Hq*max_chunks*2*(d_v+1)] split partial summaries
  size_t hpart_off;  // [B*Hq*W] f32  two-pass match: distance over the first d/2 dims per ring row
  size_t wsum_off;   // [B*Hq*kMaxWsum] uint4  two-pass match: per scan warp {P1, slot1, P2, slot2},
                     //                 its two smallest partials (fp32 bits) and their ring slots
  size_t dstate_off; // [B*Hq] int4   two-pass match, dense heads deferred to dense_kernel (match_mode 2):
                     //               {bound D* (fp32 bits), candidate slot 1, candidate slot 2, -}
  size_t dlist_off;  // [B*Hq] i32    the deferred heads (bh), ctr[8] of them (reset by complete)
  size_t qstage_off; // [B*Hq*d] in_dtype  the step's queries staged from host memory (inputs_host)
  size_t tl_off;     // [kTlSlots][2] u64 timeline stamps (MAC_TIMELINE builds only)
  size_t total;
};
__host__ __device__ __forceinline__ size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }
__host__ __device__ __forceinline__ Workspace workspace_layout(const MacDecodeParams& p) {
  size_t acc = p.storage == MAC_MODE_F64 ? 8 : 4;
  Workspace w;
  const size_t rows = (size_t)p.batch * p.n_q_heads;
  const size_t groups = (size_t)p.batch * p.n_kv_heads;
  w.mkey_off = 0;
  w.marr_off = align256(w.mkey_off + 8 * rows);
  w.gcnt_off = align256(w.marr_off + 4 * rows);
  w.ctr_off = align256(w.gcnt_off + 4 * groups);
  w.gdone_off = align256(w.ctr_off + 64);
  w.pn_off = align256(w.gdone_off + 4 * groups);
  w.mpos_off = align256(w.pn_off + 4 * groups);
  w.lo_off = align256(w.mpos_off + 4 * (size_t)p.batch);
  w.list_off = align256(w.lo_off + 4 * rows);
  w.qrot_off = align256(w.list_off + 16 * groups * p.max_chunks);
  w.part_off = align256(w.qrot_off + acc * rows * p.head_dim);
  w.hpart_off = align256(w.part_off + acc * rows * p.max_chunks * 2 * (p.head_dim_v + 1));
  w.wsum_off = align256(w.hpart_off + 4 * rows * (size_t)p.window);
  w.dstate_off = align256(w.wsum_off + 16 * rows * (size_t)kMaxWsum);
  w.dlist_off = align256(w.dstate_off + 16 * rows);
  w.qstage_off = align256(w.dlist_off + 4 * rows);
  w.tl_off = align256(w.qstage_off + 8 * rows * (size_t)p.head_dim);
#ifdef MAC_TIMELINE
  w.total = align256(w.tl_off + 16 * kTlSlots);
#else
  w.total = w.tl_off;
#endif
  return w;
}

template <typename T> __host__ __device__ __forceinline__ T* ws_ptr(const MacDecodeParams& p, size_t off) {
  return reinterpret_cast<T*>(static_cast<char*>(p.workspace) + off);
}
// the step's queries as the kernels after the front read them: staged in the workspace by the
// append warps when the inputs live in host memory (inputs_host), else the caller's q_pre
__device__ __forceinline__ const void* q_src(const MacDecodeParams& p) {
  return p.inputs_host ? static_cast<const void*>(ws_ptr<const char>(p, workspace_layout(p).qstage_off)) : p.q_pre;
}

// development timeline (MAC_TIMELINE builds): per slot, the earliest and latest
// %globaltimer stamp over the CTAs that reach the mark (thread 0 of each CTA)
#ifdef MAC_TIMELINE
__device__ __forceinline__ void tl_mark(const MacDecodeParams& p, int slot, bool any_thread = false) {
  if (threadIdx.x != 0 && !any_thread) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  unsigned long long* tl = ws_ptr<unsigned long long>(p, workspace_layout(p).tl_off) + 2 * slot;
  atomicMin(tl, t);
  atomicMax(tl + 1, t);
}
#define TL_MARK(p, slot) tl_mark((p), (slot))
#define TL_MARK_THIS(p, slot) tl_mark((p), (slot), true)
// stamp once `v` (a loaded value) is available
#define TL_MARK_DEP(p, slot, v) do { asm volatile("" :: "r"(v)); tl_mark((p), (slot)); } while (0)
#define TL_MARK_DEP_THIS(p, slot, v) do { asm volatile("" :: "r"(v)); tl_mark((p), (slot), true); } while (0)
#else
#define TL_MARK(p, slot) ((void)0)
#define TL_MARK_THIS(p, slot) ((void)0)
#define TL_MARK_DEP(p, slot, v) ((void)0)
#define TL_MARK_DEP_THIS(p, slot, v) ((void)0)
#endif

// Plan one GQA group: split grid over [grid_start(lo_g), m] (or, with the split band,
// over the piece [grid_start(lo_g), m-r] after the band slots) and one work item
// {grp, slot, t0, t1} per split appended to the device work list (the paper's
// load-balancer plan, built on the device with no host synchronisation).
__device__ __forceinline__ void plan_group(const MacDecodeParams& p, int b, int kvh, int m, int lo_g, int nb = 0,
                                           int ntarget = 0, int n_dense = 0) {
  const int start = grid_start(lo_g, p.kv_offset);
  const int end = nb > 0 ? m - p.band : shard_end(p, m);
  const Chunking ch = plan_chunking(p, m, lo_g, nb, ntarget, n_dense);
  const int slot0 = nb > 0 ? band_items(m, p.band, nb).n : 0;
  const Workspace w = workspace_layout(p);
  unsigned int* ctr = ws_ptr<unsigned int>(p, w.ctr_off);
  int4* list = ws_ptr<int4>(p, w.list_off);
  const unsigned cap = (unsigned)(p.batch * p.n_kv_heads * p.max_chunks);
  const int grp = b * p.n_kv_heads + kvh;
  ws_ptr<int>(p, w.pn_off)[grp] = ch.n | (nb << 16);
  if (ch.n == 0) return;
  TL_MARK_THIS(p, TL_PLAN_IN);
  const unsigned base = atomicAdd(ctr, (unsigned)ch.n);
  TL_MARK_DEP_THIS(p, TL_PLAN_ALLOC, base);
  const int n = (int)min((unsigned)ch.n, base < cap ? cap - base : 0u);  // full list: cannot happen
  for (int c = 0; c < n; ++c) {
    const int t0 = start + c * ch.len;
    list[base + c] = make_int4(grp + 1, slot0 + c, t0, min(end, t0 + ch.len - 1));
  }
}

// Decide one (request, q head) from its best candidate and apply the gates;
// writes the match outputs and returns the first token the head reads
// (matching.py:171-175; engine.py:449-459).
__device__ __forceinline__ int decide_one(const MacDecodeParams& p, int bh, int m, int n_scan, bool have,
                                          double bdist, int bpos) {
  const int W = p.window;
  const bool hit = n_scan > 0 && have && bdist < p.thr_sq;
  const int pp = hit ? bpos : -1;
  bool use = hit;
  if (use && p.roi_gate && !((double)pp * p.roi_b_kv >= (double)W * p.roi_b_q + (double)p.band * p.roi_b_kv))
    use = false;
  if (p.refresh_every > 0 && m % p.refresh_every == 0) use = false;
  if (p.force_miss) use = false;
  p.match_hit[bh] = hit;
  p.match_pos[bh] = pp;
  p.match_dist[bh] = n_scan > 0 ? bdist : CUDART_INF;
  p.match_scanned[bh] = n_scan;
  p.use_hit[bh] = use;
  const int lo = head_lo(use, pp, p.band);
  ws_ptr<int>(p, workspace_layout(p).lo_off)[bh] = lo;
  return lo;
}

// decide_one, and the last head of a GQA group to be decided plans the group
__device__ __forceinline__ void decide_head(const MacDecodeParams& p, int bh, int m, int n_scan, bool have,
                                            double bdist, int bpos, int nb = 0, int ntarget = 0,
                                            int n_dense = 0) {
  const int Hq = p.n_q_heads, Hkv = p.n_kv_heads, g = Hq / Hkv;
  decide_one(p, bh, m, n_scan, have, bdist, bpos);
  const Workspace w = workspace_layout(p);
  const int* lo = ws_ptr<const int>(p, w.lo_off);
  const int b = bh / Hq, h = bh % Hq, kvh = h / g;
  unsigned int* gcnt = ws_ptr<unsigned int>(p, w.gcnt_off);
  const unsigned prev = atom_add_acq_rel(gcnt + b * Hkv + kvh, 1u);
  if (prev == (unsigned)g - 1) {
    gcnt[b * Hkv + kvh] = 0u;
    int lo_g = m;
    for (int j = 0; j < g; ++j) {
      const int l = __ldcg(lo + b * Hq + kvh * g + j);
      lo_g = l < lo_g ? l : lo_g;
    }
    plan_group(p, b, kvh, m, lo_g, nb, ntarget, n_dense);
  }
}

// host-side path decisions shared by the launchers (match_fast.cu, amend_mma.cu)
bool match_fast_supported(const MacDecodeParams& p);
bool front_two_pass(const MacDecodeParams& p);
bool verify_per_group(const MacDecodeParams& p);
bool dense_deferred(const MacDecodeParams& p);
bool amend_uses_tma(const MacDecodeParams& p);
bool amend_mma_supported(const MacDecodeParams& p);
int band_split(const MacDecodeParams& p);
int piece_target(const MacDecodeParams& p);

}  // namespace mac
