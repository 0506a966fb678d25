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

template <int kRowsPerCta, int kMinBlocks, bool HOST = true>
__global__ void __launch_bounds__(kThreads, kMinBlocks) front_bf16_d128_kernel(MacDecodeParams p, int n_match,
                                                                               int do_append, int rotate_only,
                                                                               int plan, int /*unused*/) {
  constexpr int kLoads = kRowsPerCta / 16;  // per thread: 8 warps x 2 rows per load instruction
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // the first n_append CTAs append (one warp per (request, kv head)); they are
  // scheduled first so their latency hides under the ring stream
  const int n_append = do_append ? (p.batch * p.n_kv_heads + kThreads / 32 - 1) / (kThreads / 32) : 0;
  if ((int)blockIdx.x < n_append) {
    const int i = blockIdx.x * (kThreads / 32) + warp;
    if (i < p.batch * p.n_kv_heads) append_warp<HOST>(p, i, rotate_only, plan);
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

// packed fp32 pairs (Blackwell FFMA2): two lanes of fp32 math per instruction
__device__ __forceinline__ unsigned long long f2_fma(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ unsigned long long f2_pack(float lo, float hi) {
  return (unsigned long long)__float_as_uint(lo) | ((unsigned long long)__float_as_uint(hi) << 32);
}
// sum over 8 dims of (q - c)^2, the bf16 row chunk c against the query pairs q2: per element
// pair one FFMA2 for q - c (exactly rounded, c * -1 + q) and one for the square-accumulate
__device__ __forceinline__ float dist8_f2(const unsigned long long* q2, uint4 c) {
  const unsigned long long neg1 = f2_pack(-1.f, -1.f);
  unsigned long long acc = 0ull;
  const uint32_t w[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const unsigned long long cc = f2_pack(__uint_as_float(w[i] << 16), __uint_as_float(w[i] & 0xffff0000u));
    const unsigned long long e = f2_fma(cc, neg1, q2[i]);
    acc = f2_fma(e, e, acc);
  }
  return __uint_as_float((unsigned)acc) + __uint_as_float((unsigned)(acc >> 32));
}

// ---------------------------------------------------------------------------
// Two-pass match (default for the bf16 d=128 decode step).
//
// Pass 1 (front_half_kernel) reads only the first d/2 = 64 dims of every ring
// row (128 of its 256 bytes; 32-byte sectors, so the other half is never
// fetched) and stores the partial distance P(r) = sum_{k<64} (q_k - c_k)^2 of
// every row: a pure stream, no cross-CTA reduction, no atomics.
// Pass 2 (verify_kernel, one CTA per (request, head), programmatic dependent
// launch) takes the row with the smallest P, completes its distance with its
// second half into a bound D* >= min_r D(r), keeps the rows with P(r) <= D*
// — every other row has D(r) = P(r) + S(r) >= P(r) > D* >= min D, with S(r) >= 0
// a sum of squares, so it can neither be the argmin nor tie it — completes
// their distances, takes the exact argmin (ties -> larger position,
// matching.py:171-173) and decides the head (decide_head).  On the hit path
// the survivors are the few near-repeats, so the match reads about half the
// ring bytes; when nearly every row survives (a fresh query, all distances
// ~2d) pass 2 reads the second halves of all rows — the one-pass bytes.  The
// distance is the one-pass kernel's fp32 sum of squares split in two sums.
// PLANAR (kQDims = MAC_PLANAR_DIMS = 8): the rows are read from ring_qp, 16 contiguous bytes
// per row (a contiguous 16 KiB stream per head at W = 1024) instead of strided prefixes of ring_q.
template <int kRowsPerCta, int kMinBlocks, int kQDims, bool PLANAR = false, bool HOST = true>
__global__ void __launch_bounds__(kThreads, kMinBlocks) front_half_kernel(MacDecodeParams p, int n_match,
                                                                          int do_append, int rotate_only, int plan,
                                                                          int /*unused*/) {
  constexpr int LPR = kQDims / 8;                    // lanes per row (16 B = 8 dims each)
  constexpr int RPW = 32 / LPR;                      // rows per warp-load
  constexpr int kLoads = kRowsPerCta / (8 * RPW);    // loads per lane
  static_assert(kLoads >= LPR && kLoads % LPR == 0 && (LPR == 8 || LPR == 4 || LPR == 2 || LPR == 1), "reduce-scatter layout");
  constexpr int NF = kLoads / LPR;                   // rows each lane ends up holding
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n_append = do_append ? (p.batch * p.n_kv_heads + kThreads / 32 - 1) / (kThreads / 32) : 0;
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  TL_MARK(p, TL_SCAN_IN);
  if ((int)blockIdx.x < n_append) {
    const int i = blockIdx.x * (kThreads / 32) + warp;
    if (i < p.batch * p.n_kv_heads) append_warp<HOST>(p, i, rotate_only, plan);
    return;
  }
  const int W = p.window;
  const int nsplit = (W + kRowsPerCta - 1) / kRowsPerCta;
  const int bh = (blockIdx.x - n_append) / nsplit, split = (blockIdx.x - n_append) % nsplit;
  const int b = bh / p.n_q_heads;
  const int m = p.seq_lens[b] + 1;
  const int sub = lane % LPR, quad = lane / LPR;
  static_assert(!PLANAR || kQDims == MAC_PLANAR_DIMS, "ring_qp holds MAC_PLANAR_DIMS dims");
  constexpr int kRowU4 = PLANAR ? kQDims / 8 : 16;  // uint4 per row of the source
  const uint4* ring = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(PLANAR ? p.ring_qp : p.ring_q) +
                                                     (int64_t)bh * W * (kRowU4 * 8));
  const int row0 = split * kRowsPerCta;
  uint4 v[kLoads];
#pragma unroll
  for (int k = 0; k < kLoads; ++k) {
    const int slot = row0 + k * 8 * RPW + warp * RPW + quad;
    v[k] = slot < W ? ld_stream(ring + (int64_t)slot * kRowU4 + sub) : make_uint4(0, 0, 0, 0);
  }
  unsigned long long q2[4];  // this lane's 8 query dims, as fp32 pairs
#pragma unroll
  for (int i = 0; i < 4; ++i)
    q2[i] = f2_pack((float)load_in(p.q_pre, (int64_t)bh * 128 + sub * 8 + 2 * i, p.in_dtype),
                    (float)load_in(p.q_pre, (int64_t)bh * 128 + sub * 8 + 2 * i + 1, p.in_dtype));
  int first = m - W;
  if (first < 1) first = 1;
  if (p.delta_max > 0 && m - p.delta_max > first) first = m - p.delta_max;
  const int last = m - 1;
  const int cur_slot = last >= 1 ? (last - 1) % W : 0;
  float* hpart = ws_ptr<float>(p, workspace_layout(p).hpart_off) + (int64_t)bh * W;
  float part[kLoads];
#pragma unroll
  for (int k = 0; k < kLoads; ++k) part[k] = dist8_f2(q2, v[k]);
  // reduce-scatter over the row's LPR lanes: each xor round halves the values a lane keeps;
  // afterwards lane `sub` holds the partials of rows kbase + i, i < NF
  int kbase = 0;
#pragma unroll
  for (int o = LPR / 2, n = kLoads; o > 0; o >>= 1) {
    const bool up = sub & o;
#pragma unroll
    for (int i = 0; i < n / 2; ++i) {
      const float send = up ? part[i] : part[i + n / 2];
      const float keep = up ? part[i + n / 2] : part[i];
      part[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
    kbase += up ? n / 2 : 0;
    n >>= 1;
  }
  // hpart and this warp's summary for pass 2: its two smallest partials (non-negative fp32,
  // so they order as unsigned bits; dead rows are +inf) and their slots
  unsigned a1 = 0x7f800000u, a2 = 0x7f800000u;
  int t1 = 0, t2 = 0;
#pragma unroll
  for (int i = 0; i < NF; ++i) {
    const int slot = row0 + (kbase + i) * 8 * RPW + warp * RPW + quad;
    const int pos = last - cur_slot + slot - (slot > cur_slot ? W : 0);
    const bool live = slot < W && last >= 1 && pos >= first;
    const float pv = live ? part[i] : CUDART_INF_F;
    if (slot < W) hpart[slot] = pv;
    const unsigned bits = __float_as_uint(pv);
    if (bits < a1) { a2 = a1; t2 = t1; a1 = bits; t1 = slot; }
    else if (bits < a2) { a2 = bits; t2 = slot; }
  }
  const unsigned w1 = __reduce_min_sync(0xffffffffu, a1);
  const int l1 = __ffs(__ballot_sync(0xffffffffu, a1 == w1)) - 1;
  const unsigned mine2 = lane == l1 ? a2 : a1;
  const unsigned w2 = __reduce_min_sync(0xffffffffu, mine2);
  const int l2 = __ffs(__ballot_sync(0xffffffffu, mine2 == w2)) - 1;
  const int s1 = __shfl_sync(0xffffffffu, t1, l1);
  const int s2 = __shfl_sync(0xffffffffu, lane == l1 ? t2 : t1, l2);
  if (lane == 0) {
    uint4* wsum = ws_ptr<uint4>(p, workspace_layout(p).wsum_off) + (int64_t)bh * kMaxWsum;
    wsum[split * (kThreads / 32) + warp] = make_uint4(w1, (unsigned)s1, w2, (unsigned)s2);
  }
  TL_MARK(p, TL_SCAN_OUT);
}

// Pass 2: one warp per head (a CTA per GQA group, or a CTA per head with PER_HEAD).
//   1. one load round: the head's scan-warp summaries (each scan warp's two smallest
//      partials and their slots), the remaining query dims, seq_lens;
//   2. candidates = the head's two smallest partials; their full distances (the remaining
//      dims of two ring rows) give the bound D* >= min D;
//   3. a scan warp's rows can hold a survivor (P <= D*, not a candidate) only if its
//      second-smallest partial is <= D*, or its smallest is and is not a candidate; only
//      those warps' partials are read and their survivors completed (usually none on the
//      hit path, all of them for a fresh query);
//   4. exact argmin (ties -> larger position, matching.py:171-173), decide; the group is
//      planned by its CTA (or by its last-decided head with PER_HEAD).
// rows: ring rows per scan CTA of the launched scan variant; kQDims: dims its pass covered.
template <bool PER_HEAD, int kQDims>
__global__ void __launch_bounds__(256) verify_kernel(MacDecodeParams p, int rows, int nb, int ntarget, int defer,
                                                     int n_append, int clustered) {
  constexpr int SPR = kQDims / 8, RPW = 32 / SPR;  // the scan's lanes per row, rows per warp-load
  constexpr int NR = (128 - kQDims) / 8;           // remaining 16-byte chunks per row
  constexpr int LR = NR <= 8 ? 8 : 16;             // lanes per row here (NR of them load)
  constexpr int G = 32 / LR;                       // rows per warp-round
  TL_MARK(p, TL_VERIFY_IN);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int Hq = p.n_q_heads, Hkv = p.n_kv_heads, g = Hq / Hkv, W = p.window;
  // (compiled into the per-head verify only — the only layout that takes the append: in the
  // per-group kernel its code alone raised the verify to 128 registers and a stack frame,
  // +1.2 us to the first loads after the wait and +6 us to the last plan at C3)
  if (PER_HEAD && (int)blockIdx.x < n_append) {
    // The step's KV append + query rotation, one warp per (request, kv head), in CTAs of their
    // own at the head of the verify grid: it does not depend on the scan, and in the scan grid
    // its chain of dependent loads made that grid — and so every decision — end ~4.4 us after
    // the last scan CTA at C2.  Here it runs beside the scan and the decisions.  The amend
    // reads its output: its band items (before their grid-dependency wait) only once every
    // verify CTA has triggered — these after all their warps appended and fenced — and its
    // piece items after this whole grid.
    const int i = blockIdx.x * (blockDim.x >> 5) + warp;
    if (i < p.batch * Hkv) append_warp<false>(p, i, 0, 0);  // (never with inputs_host)
    __threadfence();
    __syncthreads();
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    return;
  }
  const int blk = blockIdx.x - n_append;
  const int grp = PER_HEAD ? blk / g : blk;
  const int hl = PER_HEAD ? blk % g : warp;
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  TL_MARK(p, TL_VERIFY_WAITED);
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  const int b = grp / Hkv, kvh = grp % Hkv;
  const int bh = b * Hq + kvh * g + hl;
  const int nsum = ((W + rows - 1) / rows) * (kThreads / 32);  // scan warps of this head
  const int wrows = rows / 8;                                  // rows per scan warp
  const float* hpart = ws_ptr<const float>(p, workspace_layout(p).hpart_off) + (int64_t)bh * W;
  const uint4* wsum = ws_ptr<const uint4>(p, workspace_layout(p).wsum_off) + (int64_t)bh * kMaxWsum;
  const uint4* ring = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(p.ring_q) + (int64_t)bh * W * 128);
  const int ci = lane % LR, gi = lane / LR;  // chunk of the row, row group
  const bool cload = ci < NR;
  constexpr int kSumPerLane = kMaxWsum / 32;
  uint4 sm[kSumPerLane];
#pragma unroll
  for (int i = 0; i < kSumPerLane; ++i) {
    const int j = lane + 32 * i;
    sm[i] = j < nsum ? __ldcg(wsum + j) : make_uint4(0x7f800000u, 0u, 0x7f800000u, 0u);
  }
  float qh[8];  // the query dims of this lane's chunk (kQDims + 8 ci ..)
#pragma unroll
  for (int i = 0; i < 8; ++i)
    // (with append CTAs in this grid the inputs are device-resident: q_src(p) is p.q_pre)
    qh[i] = cload ? (float)load_in(q_src(p), (int64_t)bh * 128 + kQDims + ci * 8 + i, p.in_dtype) : 0.f;
  const int m = p.seq_lens[b] + 1;
  TL_MARK_DEP(p, TL_V_M, m);
  auto rest = [&](int slot) -> float {  // sum over the remaining dims of row `slot`, this row group
    float e = (slot >= 0 && cload) ? dist8(qh, ld_stream(ring + (int64_t)slot * 16 + SPR + ci)) : 0.f;
#pragma unroll
    for (int o = LR / 2; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
    return e;
  };
  // 1. the head's two smallest partials: this lane's best two of its summaries, then the warp's
  unsigned a1 = 0x7f800000u, a2 = 0x7f800000u, t1 = 0u, t2 = 0u;
#pragma unroll
  for (int i = 0; i < kSumPerLane; ++i) {
    if (sm[i].x < a1) { a2 = a1; t2 = t1; a1 = sm[i].x; t1 = sm[i].y; }
    else if (sm[i].x < a2) { a2 = sm[i].x; t2 = sm[i].y; }
    if (sm[i].z < a2) { a2 = sm[i].z; t2 = sm[i].w; }
  }
  const unsigned w1 = __reduce_min_sync(0xffffffffu, a1);
  const int lane1 = __ffs(__ballot_sync(0xffffffffu, a1 == w1)) - 1;
  const unsigned mine2 = lane == lane1 ? a2 : a1;
  const unsigned w2 = __reduce_min_sync(0xffffffffu, mine2);
  const int lane2 = __ffs(__ballot_sync(0xffffffffu, mine2 == w2)) - 1;
  const int cs1 = w1 < 0x7f800000u ? (int)__shfl_sync(0xffffffffu, t1, lane1) : -1;
  const unsigned ts2 = __shfl_sync(0xffffffffu, lane == lane1 ? t2 : t1, lane2);
  const int cs2 = w2 < 0x7f800000u ? (int)ts2 : -1;
  // step geometry (needs m)
  int first = m - W;
  if (first < 1) first = 1;
  if (p.delta_max > 0 && m - p.delta_max > first) first = m - p.delta_max;
  const int last = m - 1;
  const int n_scan = last >= first ? last - first + 1 : 0;
  const int cur_slot = last >= 1 ? (last - 1) % W : 0;
  auto pos_of = [&](int slot) { return last - cur_slot + slot - (slot > cur_slot ? W : 0); };
  auto key_of = [&](float d, int slot) {
    return ~(((unsigned long long)__float_as_uint(d) << 32) | (unsigned long long)(0xffffffffu - (unsigned)pos_of(slot)));
  };
  TL_MARK(p, TL_V_SELECTED);
  // 2. candidates' full distances: row group 0 candidate 1, row group 1 candidate 2
  const int cslot = gi == 0 ? cs1 : (gi == 1 ? cs2 : -1);
  const float cpart = __uint_as_float(gi == 0 ? w1 : w2);
  const float d2 = rest(cslot);
  const float cfull = cslot >= 0 ? cpart + d2 : CUDART_INF_F;
  unsigned long long key = (cslot >= 0 && ci == 0 && gi < 2) ? key_of(cfull, cslot) : 0ull;
  const float D = fminf(__shfl_sync(0xffffffffu, cfull, 0), __shfl_sync(0xffffffffu, cfull, LR));
  TL_MARK(p, TL_V_BOUND);
  // 3. scan warps that can hold a survivor (exact test per row inside)
  const unsigned Dbits = __float_as_uint(D);
  unsigned need = 0u;  // bit i: summary lane + 32 i
  if (D != CUDART_INF_F) {
#pragma unroll
    for (int i = 0; i < kSumPerLane; ++i) {
      const bool c1 = (int)sm[i].y == cs1 || (int)sm[i].y == cs2;
      const bool n = sm[i].z <= Dbits || (sm[i].x <= Dbits && !c1);
      need |= n ? (1u << i) : 0u;
    }
  }
  // Dense mode: when half the scan warps can hold a survivor (a query with no near-repeat:
  // every row survives pass 1), walk every ring row in order, 32 per iteration with all their
  // loads in flight, instead of the sparse walk's chain of round trips per flagged warp (C3
  // geometry, 4K context, every head missing: 433 -> 394 us per step).  Same survivor test,
  // same keys: the result is identical.  (Helper warps per head halve it again but double the
  // verify CTAs' registers, which evicts the amend's band items from the SMs during the verify:
  // +2.3 us on the all-hit C3 step.)
  const int n_need = (int)__reduce_add_sync(0xffffffffu, (unsigned)__popc(need));
  bool deferred = false;
  if (!PER_HEAD && defer && 2 * n_need >= nsum) {
    // match_mode 2: hand the dense walk to dense_kernel, which spreads it over the whole GPU
    // (a warp per 32-row chunk); this head's candidates seed its key, and its group is planned
    // by whichever dense chunk decides the group's last head
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
      key = other > key ? other : key;
    }
    if (lane == 0) {
      const Workspace ws = workspace_layout(p);
      if (key) atomicMax(ws_ptr<unsigned long long>(p, ws.mkey_off) + bh, key);
      ws_ptr<int4>(p, ws.dstate_off)[bh] = make_int4((int)Dbits, cs1, cs2, 0);
      const unsigned i = atomicAdd(ws_ptr<unsigned int>(p, ws.ctr_off) + 8, 1u);
      ws_ptr<int>(p, ws.dlist_off)[i] = bh;
    }
    deferred = true;
    need = 0u;
  } else if (2 * n_need >= nsum) {
    constexpr int RK = 32 / G;  // rows per lane group per iteration
#pragma unroll 1
    for (int base = 0; base < W; base += 32) {
      const float pr = base + lane < W ? hpart[base + lane] : CUDART_INF_F;
      uint4 rv[RK];
#pragma unroll
      for (int k = 0; k < RK; ++k) {
        const int slot = base + gi + G * k;
        rv[k] = (slot < W && cload) ? ld_stream(ring + (int64_t)slot * 16 + SPR + ci) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int k = 0; k < RK; ++k) {
        float e = cload ? dist8(qh, rv[k]) : 0.f;
#pragma unroll
        for (int o = LR / 2; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
        const int slot = base + gi + G * k;
        const float prs = __shfl_sync(0xffffffffu, pr, gi + G * k);
        if (slot < W && ci == 0 && prs <= D && prs != CUDART_INF_F && slot != cs1 && slot != cs2) {
          const unsigned long long k2 = key_of(prs + e, slot);
          key = k2 > key ? k2 : key;
        }
      }
    }
    need = 0u;  // the sparse walk has nothing left
  }
#pragma unroll 1
  for (int i = 0; i < kSumPerLane; ++i) {
    unsigned warps_i = __ballot_sync(0xffffffffu, (need >> i) & 1u);
#pragma unroll 1
    while (warps_i) {
      const int j = 32 * i + __ffs(warps_i) - 1;  // scan warp j = split * 8 + w
      warps_i &= warps_i - 1;
      // its rows: split * rows + k * 8 RPW + w * RPW + q (k < loads, q < RPW), row index l = k RPW + q
      const int jsplit = j / (kThreads / 32), jw = j % (kThreads / 32);
      auto slot_of = [&](int l) { return jsplit * rows + (l / RPW) * 8 * RPW + jw * RPW + (l % RPW); };
#pragma unroll 1
      for (int l0 = 0; l0 < wrows; l0 += 32) {
        const int my = slot_of(l0 + lane);
        const bool mine_ok = l0 + lane < wrows && my < W;
        const float pr = mine_ok ? hpart[my] : CUDART_INF_F;
        const bool surv = pr <= D && pr != CUDART_INF_F && my != cs1 && my != cs2;
        const unsigned mask = __ballot_sync(0xffffffffu, surv);
        // row group gi takes survivors gi, gi + G, gi + 2G, ... of these 32 rows, 8 per round
#pragma unroll 1
        for (int r0 = 0; r0 < __popc(mask); r0 += 8 * G) {
          int li[8];
          uint4 rv[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            li[k] = -1;
            int n = r0 + gi + G * k;  // the n-th set bit of mask
            unsigned mm = mask;
            for (; n > 0 && mm; --n) mm &= mm - 1;
            if (mm) li[k] = __ffs(mm) - 1;
            rv[k] = (li[k] >= 0 && cload) ? ld_stream(ring + (int64_t)slot_of(l0 + li[k]) * 16 + SPR + ci)
                                          : make_uint4(0, 0, 0, 0);
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            float e = cload ? dist8(qh, rv[k]) : 0.f;
#pragma unroll
            for (int o = LR / 2; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
            const float prs = __shfl_sync(0xffffffffu, pr, li[k] >= 0 ? li[k] : 0);
            if (li[k] >= 0 && ci == 0) {
              const unsigned long long k2 = key_of(prs + e, slot_of(l0 + li[k]));
              key = k2 > key ? k2 : key;
            }
          }
        }
      }
    }
  }
  TL_MARK(p, TL_V_SURVIVED);
  // 4. exact argmin, decision; the group's plan
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
    key = other > key ? other : key;
  }
  double bd = CUDART_INF;
  int bpos = -1;
  if (key) {
    const unsigned long long raw = ~key;
    bd = (double)__uint_as_float((unsigned)(raw >> 32));
    bpos = (int)(0xffffffffu - (unsigned)(raw & 0xffffffffull));
  }
  if (PER_HEAD) {
    if (!clustered) {
      if (lane == 0) decide_head(p, bh, m, n_scan, bpos > 0, bd, bpos, nb, ntarget);  // the group's last head plans it
      TL_MARK(p, TL_VERIFY_OUT);
      return;
    }
    // The group's g head CTAs are one thread-block cluster (launch_verify): each head's first
    // token goes into the leader CTA's shared memory (DSMEM) and one cluster barrier replaces
    // decide_head's chain through L2 (release fence, group-counter atomic, the lo loads of the
    // last arriver); the leader (cluster rank 0 = head 0 of the group) plans the group.
    __shared__ int s_lo[8];
    int lo = 0;
    if (lane == 0) lo = decide_one(p, bh, m, n_scan, bpos > 0, bd, bpos);
    if (lane == 0) {
      const uint32_t la = (uint32_t)__cvta_generic_to_shared(&s_lo[hl]);
      uint32_t ra;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(ra) : "r"(la), "r"(0));
      asm volatile("st.shared::cluster.u32 [%0], %1;\n" ::"r"(ra), "r"(lo) : "memory");
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    TL_MARK(p, TL_V_DECIDED);
    if (hl == 0 && lane == 0) {
      int lo_g = m;
      for (int j = 0; j < g; ++j) lo_g = s_lo[j] < lo_g ? s_lo[j] : lo_g;
      plan_group(p, b, kvh, m, lo_g, nb, ntarget);
    }
    TL_MARK(p, TL_VERIFY_OUT);
    return;
  }
  __shared__ int slo[8];
  if (lane == 0 && !deferred) slo[hl] = decide_one(p, bh, m, n_scan, bpos > 0, bd, bpos);
  const int n_def = __syncthreads_count(lane == 0 && deferred);
  TL_MARK(p, TL_V_DECIDED);
  if (threadIdx.x == 0) {  // (the amend reads the plan after this grid completes: no fence needed)
    if (n_def == 0) {
      int lo_g = m;
      for (int j = 0; j < g; ++j) lo_g = slo[j] < lo_g ? slo[j] : lo_g;
      plan_group(p, b, kvh, m, lo_g, nb, ntarget);
    } else {  // the decided heads count toward the group; dense_kernel's deciders plan it
      __threadfence();
      atom_add_acq_rel(ws_ptr<unsigned int>(p, workspace_layout(p).gcnt_off) + grp, (unsigned)(g - n_def));
    }
  }
  TL_MARK(p, TL_VERIFY_OUT);
}

// match_mode 2, after the verify: the full distances of every ring row of the heads the verify
// deferred (a query with no near-repeat makes every row survive pass 1), one warp per 128-row
// chunk over the whole GPU instead of one warp walking 1024 rows — the same survivor test and the
// same fp32 sums as the verify's walk (P(row) + the remaining 128 - MAC_PLANAR_DIMS dims, reduced over 16 lanes), so
// the argmin is the one the verify would have found.  Chunks publish their best key with an
// atomic max; the chunk completing a head decides it (finish_decide -> decide_head) and the last
// head of a group plans the group.
// 32 rows per warp: one load round per task.  (128-row tasks — four dependent rounds of
// shuffle-reduced distances — took 20 us each: at 2 % misses only ~1 task warp per SM, so
// nothing hid their latency; C3 geometry at 16K, r02 timeline.)
constexpr int kDenseRows = 32;
template <int kQDims>
__global__ void __launch_bounds__(256) dense_kernel(MacDecodeParams p, int nb, int ntarget) {
  constexpr int rows = kDenseRows;
  constexpr int SPR = kQDims / 8;
  constexpr int NR = (128 - kQDims) / 8;
  constexpr int LR = NR <= 8 ? 8 : 16;
  constexpr int G = 32 / LR;
  constexpr int RK = 32 / G;
  TL_MARK(p, TL_DENSE_IN);
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  TL_MARK(p, TL_DENSE_WAITED);
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const Workspace ws = workspace_layout(p);
  const int n_dense = (int)__ldcg(ws_ptr<const unsigned int>(p, ws.ctr_off) + 8);
  const int W = p.window, nch = (W + rows - 1) / rows;
  const int ci = lane % LR, gi = lane / LR;
  const bool cload = ci < NR;
  for (int task = blockIdx.x * (blockDim.x >> 5) + warp; task < n_dense * nch; task += gridDim.x * (blockDim.x >> 5)) {
    if (lane == 0) TL_MARK_THIS(p, TL_DENSE_TASK);
    const int bh = __ldcg(ws_ptr<const int>(p, ws.dlist_off) + task / nch);
    const int chunk = task % nch;
    const int4 st = __ldcg(ws_ptr<const int4>(p, ws.dstate_off) + bh);
    const float D = __uint_as_float((unsigned)st.x);
    const int cs1 = st.y, cs2 = st.z;
    const int b = bh / p.n_q_heads;
    const int m = p.seq_lens[b] + 1;
    int first = m - W;
    if (first < 1) first = 1;
    if (p.delta_max > 0 && m - p.delta_max > first) first = m - p.delta_max;
    const int last = m - 1;
    const int n_scan = last >= first ? last - first + 1 : 0;
    const int cur_slot = last >= 1 ? (last - 1) % W : 0;
    const float* hpart = ws_ptr<const float>(p, ws.hpart_off) + (int64_t)bh * W;
    const uint4* ring = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(p.ring_q) + (int64_t)bh * W * 128);
    float qh[8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      qh[i] = cload ? (float)load_in(q_src(p), (int64_t)bh * 128 + kQDims + ci * 8 + i, p.in_dtype) : 0.f;
    unsigned long long key = 0ull;
    const int r0 = chunk * rows, r1 = min(W, r0 + rows);
#pragma unroll 1
    for (int base = r0; base < r1; base += 32) {
      const float pr = base + lane < r1 ? __ldcg(hpart + base + lane) : CUDART_INF_F;
      uint4 rv[RK];
#pragma unroll
      for (int k = 0; k < RK; ++k) {
        const int slot = base + gi + G * k;
        rv[k] = (slot < r1 && cload) ? ld_stream(ring + (int64_t)slot * 16 + SPR + ci) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int k = 0; k < RK; ++k) {
        float e = cload ? dist8(qh, rv[k]) : 0.f;
#pragma unroll
        for (int o = LR / 2; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
        const int slot = base + gi + G * k;
        const float prs = __shfl_sync(0xffffffffu, pr, gi + G * k);
        if (slot < r1 && ci == 0 && prs <= D && prs != CUDART_INF_F && slot != cs1 && slot != cs2) {
          const int pos = last - cur_slot + slot - (slot > cur_slot ? W : 0);
          const unsigned long long k2 =
              ~(((unsigned long long)__float_as_uint(prs + e) << 32) | (unsigned long long)(0xffffffffu - (unsigned)pos));
          key = k2 > key ? k2 : key;
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
      key = other > key ? other : key;
    }
    if (lane == 0 && publish_key(p, bh, key) == (unsigned)nch - 1) {
      const unsigned long long k3 = atomicExch(ws_ptr<unsigned long long>(p, ws.mkey_off) + bh, 0ull);
      ws_ptr<unsigned int>(p, ws.marr_off)[bh] = 0u;
      double bd = CUDART_INF;
      int bp = -1;
      if (k3) {
        const unsigned long long raw = ~k3;
        bd = (double)__uint_as_float((unsigned)(raw >> 32));
        bp = (int)(0xffffffffu - (unsigned)(raw & 0xffffffffull));
      }
      decide_head(p, bh, m, n_scan, bp > 0, bd, bp, nb, ntarget, n_dense);
    }
    if (lane == 0) TL_MARK_THIS(p, TL_DENSE_OUT);
  }
}

cudaError_t launch_dense(const MacDecodeParams& p, cudaStream_t st, int qdims) {
  cudaLaunchConfig_t cfg = {};
  // 4 CTAs per SM (C3 geometry at 16K: 10 % misses 197 us vs 200 at 2 and 208 at 1; 2 % the
  // same 96 us at all three; profiles/r02/miss_regime/dense_grid_ab.jsonl)
  int per_sm = 4;
#ifdef MAC_DEV_KNOBS
  if (const char* env = getenv("MAC_DENSE_CTAS")) per_sm = atoi(env) > 0 ? atoi(env) : 1;
#endif
  cfg.gridDim = dim3(148 * per_sm);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const int nb = band_split(p);
  const int nt = nb > 0 ? piece_target(p) : 0;
  if (qdims == 8) return cudaLaunchKernelEx(&cfg, dense_kernel<8>, p, nb, nt);
  if (qdims == 16) return cudaLaunchKernelEx(&cfg, dense_kernel<16>, p, nb, nt);
  if (qdims == 32) return cudaLaunchKernelEx(&cfg, dense_kernel<32>, p, nb, nt);
  return cudaLaunchKernelEx(&cfg, dense_kernel<64>, p, nb, nt);
}

cudaError_t launch_verify(const MacDecodeParams& p, cudaStream_t st, bool per_head, int rows, int qdims,
                          bool append) {
  cudaLaunchConfig_t cfg = {};
  const int g = p.n_q_heads / p.n_kv_heads;
  const int warps = per_head ? 1 : g;
  // per-head verify: a GQA group's head CTAs form one cluster (exchange through DSMEM, see
  // verify_kernel); the append CTAs ahead of them are padded to whole clusters
  const int clustered = per_head && g > 1 && g <= 8 ? 1 : 0;
  int n_append = append ? (p.batch * p.n_kv_heads + warps - 1) / warps : 0;
  if (clustered) n_append = (n_append + g - 1) / g * g;
  cfg.gridDim = dim3(n_append + (per_head ? p.batch * p.n_q_heads : p.batch * p.n_kv_heads));
  cfg.blockDim = dim3(32 * warps);
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = clustered ? g : 1;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = clustered ? 2 : 1;
  const int nb = band_split(p);  // the amend computes the band before its wait (amend_mma.cu)
  const int nt = nb > 0 ? piece_target(p) : 0;
  const int defer = dense_deferred(p) ? 1 : 0;
  if (qdims == 8)
    return per_head ? cudaLaunchKernelEx(&cfg, verify_kernel<true, 8>, p, rows, nb, nt, defer, n_append, clustered)
                    : cudaLaunchKernelEx(&cfg, verify_kernel<false, 8>, p, rows, nb, nt, defer, n_append, clustered);
  if (qdims == 16)
    return per_head ? cudaLaunchKernelEx(&cfg, verify_kernel<true, 16>, p, rows, nb, nt, defer, n_append, clustered)
                    : cudaLaunchKernelEx(&cfg, verify_kernel<false, 16>, p, rows, nb, nt, defer, n_append, clustered);
  if (qdims == 32)
    return per_head ? cudaLaunchKernelEx(&cfg, verify_kernel<true, 32>, p, rows, nb, nt, defer, n_append, clustered)
                    : cudaLaunchKernelEx(&cfg, verify_kernel<false, 32>, p, rows, nb, nt, defer, n_append, clustered);
  return per_head ? cudaLaunchKernelEx(&cfg, verify_kernel<true, 64>, p, rows, nb, nt, defer, n_append, clustered)
                  : cudaLaunchKernelEx(&cfg, verify_kernel<false, 64>, p, rows, nb, nt, defer, n_append, clustered);
}

bool match_fast_supported(const MacDecodeParams& p) {
  return p.storage == MAC_MODE_BF16 && p.head_dim == 128 && p.head_dim_v == 128 && p.match_space == MAC_MATCH_PRE_ROPE;
}
bool front_fast_supported(const MacDecodeParams& p) {
  return p.storage == MAC_MODE_BF16 && p.head_dim == 128 && p.head_dim_v == 128;
}

// Front variants: two-pass match (ring rows per CTA, min CTAs per SM, first-pass dims) =
// (512, 4, 8) reading ring_qp when given (the product; 16 dims: C3 +1.8 us, r02 session 3), and the one-pass stream (128, 5).
// Development builds (-DMAC_DEV_KNOBS) add the measured alternatives, selected with
// MAC_FRONT_VARIANT: 2-3 one-pass (64, 8), (256, 3); 4-7 two-pass (256, 4, 64), (256, 4, 32),
// (512, 4, 32), (1024, 4, 8), 8: (512, 4, 16) from ring_q.  C3 step (us): 59.8 (0), 67.8 (4); the (256,6) and (512,3)
// shapes scanned 3.5 and 0.8 us slower than (0); (1024,4,16) scans 2 us faster but its verify
// (twice the rows per scan-warp summary) takes 1.3 us longer: step 50.4 vs 49.0, C2 34.6 vs
// 33.7 (r02, same box).  Round-1 alternatives that lost on C3
// (persistent tensor-core and CUDA-core scans, a DSMEM-cluster argmin, one fused step kernel)
// were measured and not kept; their numbers are in profiles/r01/SUMMARY.md.
using FrontFn = void (*)(MacDecodeParams, int, int, int, int, int);
struct FrontVariant {
  FrontFn fn;
  int rows;
  bool two_pass;  // front_half_kernel + verify_kernel
  int qdims;      // dims of the first pass (two-pass)
  FrontFn fn_planar;  // reads ring_qp when it is given
  FrontFn fn_dev, fn_planar_dev;  // the same without the host-input staging (inputs_host == 0)
};
static const FrontVariant kFrontVariants[] = {
    {front_half_kernel<512, 4, 8>, 512, true, 8, front_half_kernel<512, 4, 8, true>,
     front_half_kernel<512, 4, 8, false, false>, front_half_kernel<512, 4, 8, true, false>},
    {front_bf16_d128_kernel<128, 5>, 128, false, 0, nullptr, front_bf16_d128_kernel<128, 5, false>, nullptr},
#ifdef MAC_DEV_KNOBS
    {front_bf16_d128_kernel<64, 8>, 64, false, 0, nullptr},
    {front_bf16_d128_kernel<256, 3>, 256, false, 0, nullptr},
    {front_half_kernel<256, 4, 64>, 256, true, 64, nullptr},
    {front_half_kernel<256, 4, 32>, 256, true, 32, nullptr},
    {front_half_kernel<512, 4, 32>, 512, true, 32, nullptr},
    {front_half_kernel<1024, 4, 8>, 1024, true, 8, front_half_kernel<1024, 4, 8, true>},
    {front_half_kernel<512, 4, 16>, 512, true, 16, nullptr},  // 16 first-pass dims (strided ring_q reads)
#endif
};

// append CTAs first (8 warps, one (request, kv head) each), then the match CTAs
// passes: bit 0 = the scan (append, rows), bit 1 = the verify kernel (two-pass mode only)
static int front_variant() {
#ifdef MAC_DEV_KNOBS
  static int vi = -1;
  if (vi < 0) {
    const char* env = getenv("MAC_FRONT_VARIANT");
    vi = env ? atoi(env) : 0;
    if (vi < 0 || vi >= (int)(sizeof(kFrontVariants) / sizeof(kFrontVariants[0]))) vi = 0;
  }
  return vi;
#else
  return 0;
#endif
}
bool verify_per_group(const MacDecodeParams& p) {
#ifdef MAC_DEV_KNOBS
  static int forced = -2;
  if (forced == -2) {
    const char* env = getenv("MAC_VERIFY_PER_GROUP");
    forced = env ? atoi(env) : -1;
  }
  if (forced >= 0) return forced == 1 && p.n_q_heads / p.n_kv_heads <= 8;
#endif
  return p.batch * p.n_kv_heads >= 148 && p.n_q_heads / p.n_kv_heads <= 8;
}
// match_mode 2 (expected misses): the per-group verify defers dense heads to dense_kernel
bool dense_deferred(const MacDecodeParams& p) { return p.match_mode == 2 && verify_per_group(p); }
// whether a match launch of the fast front runs the two-pass scan + verify kernels: enough heads
// to fill the SMs, and a ring of 512..1024 rows — on smaller rings the one-pass scan reads little
// more and a head whose query has no near-repeat (every row survives pass 1) costs the verify a
// chain of round trips (C5 sweep, batch 16, W = 256: 111 us per step two-pass vs 44 one-pass)
bool front_two_pass(const MacDecodeParams& p) {
  return p.match_mode != 1 && match_fast_supported(p) && kFrontVariants[front_variant()].two_pass &&
         (verify_per_group(p) || p.batch * p.n_q_heads >= 148) && p.window >= 512 && p.window <= 1024;
}

cudaError_t launch_front_bf16(const MacDecodeParams& p, cudaStream_t st, bool do_match, bool do_append,
                              int rotate_only, int plan, int passes) {
  const FrontVariant& v = kFrontVariants[front_variant()];
  // the two-pass front covers the match stage only: append-only launches use the one-pass kernel,
  // and so does a batch with fewer heads than SMs (one long request): too little verify parallelism
  // verify: a CTA per GQA group when groups fill the SMs, a CTA per head when only heads do
  const bool per_group = verify_per_group(p);
  const bool per_head = !per_group && p.batch * p.n_q_heads >= 148;
  const bool two_pass = do_match && front_two_pass(p);
  const FrontVariant& u = (v.two_pass && !two_pass) ? kFrontVariants[1] : v;
  // with a verify CTA per head (fewer GQA groups than SMs: C2) a whole two-pass step runs the
  // append in CTAs of its own at the head of the verify grid (verify_kernel), so the scan grid —
  // which the decisions wait on — is the scan alone: C2 34.2 -> 31.9 us.  With a CTA per group
  // (C3) the scan is long enough to hide the append and the extra verify CTAs cost 2 us, and with
  // host-resident inputs the append's PCIe reads would sit on the decisions' path (C3 e2e +9 us)
  // (r02 A/B, profiles/r02/ab_append.sh).
  bool app_in_verify = two_pass && per_head && !p.inputs_host && do_append && passes == 3 && !rotate_only && !plan;
#ifdef MAC_DEV_KNOBS
  {
    static int knob = -1;  // MAC_APPEND_IN_VERIFY=0: append CTAs stay in the scan grid
    if (knob < 0) {
      const char* env = getenv("MAC_APPEND_IN_VERIFY");
      knob = env ? atoi(env) : 1;
    }
    app_in_verify = app_in_verify && knob != 0;
  }
#endif
  const bool app_in_front = do_append && !app_in_verify;
  const int n_match = do_match ? p.batch * p.n_q_heads * ((p.window + u.rows - 1) / u.rows) : 0;
  const int n_append = app_in_front ? (p.batch * p.n_kv_heads + 7) / 8 : 0;
  if (n_match + n_append == 0 && !app_in_verify) return cudaSuccess;
  if (passes & 1) {
    const bool planar = do_match && u.fn_planar && p.ring_qp;
    FrontFn fn = planar ? u.fn_planar : u.fn;
    if (!p.inputs_host) fn = planar ? (u.fn_planar_dev ? u.fn_planar_dev : fn) : (u.fn_dev ? u.fn_dev : fn);
    fn<<<n_match + n_append, kThreads, 0, st>>>(p, n_match, app_in_front ? 1 : 0, rotate_only, plan, 0);
    const cudaError_t e = cudaGetLastError();
    if (e) return e;
  }
  if ((passes & 2) && u.two_pass && do_match) {
    const cudaError_t e = launch_verify(p, st, per_head, u.rows, u.qdims, app_in_verify);
    if (e || !dense_deferred(p)) return e;
    return launch_dense(p, st, u.qdims);
  }
  return cudaSuccess;
}

}  // namespace mac
