// Shared pieces of the front (append + match + plan) kernels: the per-(request,
// kv head) append warp and the cross-CTA argmin publication.
#pragma once

#include "common.cuh"

namespace mac {

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// append + RoPE for one (request, kv head) by one warp; optionally plan the group as "all heads miss".
// Every input load (seq_lens, the step's k / v / q rows, the RoPE frequencies) is issued before
// any of them is used, so the warp pays two dependent memory round trips (those loads, then the
// page-table entry of position m) — it runs beside a DRAM-saturating scan, where each round trip
// costs ~1.5-2 us (C2: the dependent-load version ended the front grid 4.5 us after the scan).
__device__ __forceinline__ void append_warp(const MacDecodeParams& p, int idx, int rotate_only, int plan) {
  const int lane = threadIdx.x & 31;
  const int b = idx / p.n_kv_heads, kvh = idx % p.n_kv_heads;
  const int g = p.n_q_heads / p.n_kv_heads;
  const Workspace w = workspace_layout(p);
  __nv_bfloat16* kc = static_cast<__nv_bfloat16*>(p.k_cache);
  __nv_bfloat16* vc = static_cast<__nv_bfloat16*>(p.v_cache);
  float* qrot = ws_ptr<float>(p, w.qrot_off);
  // ---- round trip 1: everything that does not depend on m ----
  const int m = p.seq_lens[b] + (rotate_only ? 0 : 1);
  const int dt = p.in_dtype;
  const int64_t kbase = ((int64_t)b * p.n_kv_heads + kvh) * 128;
  double fr[2], kx[2][2], vx[4];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int j = lane + 32 * u;
    fr[u] = p.rope_freqs[j];
    kx[u][0] = rotate_only ? 0.0 : load_in(p.k_pre, kbase + 2 * j, dt);
    kx[u][1] = rotate_only ? 0.0 : load_in(p.k_pre, kbase + 2 * j + 1, dt);
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) vx[e] = rotate_only ? 0.0 : load_in(p.v_in, kbase + lane + 32 * e, dt);
  constexpr int kMaxG = 4;  // query heads held in registers per pass (more: further passes)
  float qx[kMaxG][2][2];
  auto load_q = [&](int h0) {
#pragma unroll
    for (int t = 0; t < kMaxG; ++t)
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int64_t qi = ((int64_t)b * p.n_q_heads + kvh * g + h0 + t) * 128 + 2 * (lane + 32 * u);
        qx[t][u][0] = h0 + t < g ? (float)load_in(p.q_pre, qi, dt) : 0.f;
        qx[t][u][1] = h0 + t < g ? (float)load_in(p.q_pre, qi + 1, dt) : 0.f;
      }
  };
  load_q(0);
  if (lane == 0) ws_ptr<int>(p, w.mpos_off)[b] = m;  // every group's warp (same value)
  // every 8th token: the misses counted since the last publication (complete.cu) -> host.  Not
  // every step: a kernel that stores to host memory pays for the flush when it ends (~1 us).
  // With several layers per token every layer's complete counts into the same counters and only
  // the first layer stepped at that token publishes (>= 8 steps counted since the last one).
  if (idx == 0 && lane == 0 && p.feedback && (m & 7) == 0 && ws_ptr<unsigned>(p, w.ctr_off)[6] >= 8u) {
    unsigned* ctr = ws_ptr<unsigned>(p, w.ctr_off);
    p.feedback[0] = (int)ctr[4];
    p.feedback[1] = (int)ctr[6] * p.batch * p.n_q_heads;
    ctr[4] = 0u;
    ctr[6] = 0u;
  }
  // ---- round trip 2: the page of position m ----
  const int t_local = m - p.kv_offset;
  bool store = !rotate_only && t_local >= 1 && (p.kv_limit <= 0 || t_local <= p.kv_limit);
  if (store && !kv_fits(p.pages_per_seq, t_local, p.page_size)) {
    store = false;
    if (lane == 0) atomicOr(ws_ptr<unsigned>(p, w.ctr_off) + 2, 1u);
  }
  int64_t row = 0;
  if (store) row = kv_row(p.page_table, p.pages_per_seq, b, t_local, p.page_size, p.n_kv_heads, kvh);
  double sn[2], cs[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) sincos((double)m * fr[u], &sn[u], &cs[u]);
  // rotated queries (fp64 angles, fp32 storage) need no page: stored first
  for (int h0 = 0; h0 < g; h0 += kMaxG) {
    if (h0 > 0) load_q(h0);
#pragma unroll
    for (int t = 0; t < kMaxG; ++t) {
      if (h0 + t >= g) break;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int64_t qi = ((int64_t)b * p.n_q_heads + kvh * g + h0 + t) * 128 + 2 * (lane + 32 * u);
        const double x0 = qx[t][u][0], x1 = qx[t][u][1];
        reinterpret_cast<float2*>(qrot + qi)[0] =
            make_float2((float)(x0 * cs[u] - x1 * sn[u]), (float)(x0 * sn[u] + x1 * cs[u]));
      }
    }
  }
  if (store) {
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int j = lane + 32 * u;
      __nv_bfloat162 kk;
      kk.x = from_f64<__nv_bfloat16>(kx[u][0] * cs[u] - kx[u][1] * sn[u]);
      kk.y = from_f64<__nv_bfloat16>(kx[u][0] * sn[u] + kx[u][1] * cs[u]);
      reinterpret_cast<__nv_bfloat162*>(kc + row * 128)[j] = kk;
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) vc[row * 128 + lane + 32 * e] = from_f64<__nv_bfloat16>(vx[e]);
  }
  if (plan && lane == 0) {
    int* lo = ws_ptr<int>(p, w.lo_off);
    for (int hl = 0; hl < g; ++hl) lo[b * p.n_q_heads + kvh * g + hl] = 1;
    plan_group(p, b, kvh, m, 1);
  }
}

// Publication of one worker's best candidate (complemented packed key
// ~(dist_bits << 32 | ~pos), 0 = nothing) for its (request, head), in two
// halves so a streaming worker need not wait for the round trip: publish_key
// returns the previous arrival count (consume it later); the worker that
// brought the count to nsplit runs finish_decide, which decides the head
// (decide_head) and returns key and counter to zero for the next step
// (graph-replay safe).  Single thread.
__device__ __forceinline__ unsigned publish_key(const MacDecodeParams& p, int bh, unsigned long long key) {
  const Workspace ws = workspace_layout(p);
  if (key) atomicMax(ws_ptr<unsigned long long>(p, ws.mkey_off) + bh, key);
  return atom_add_acq_rel(ws_ptr<unsigned int>(p, ws.marr_off) + bh, 1u);
}

__device__ __forceinline__ void finish_decide(const MacDecodeParams& p, int bh, int m, int n_scan) {
  const Workspace ws = workspace_layout(p);
  const unsigned long long k3 = atomicExch(ws_ptr<unsigned long long>(p, ws.mkey_off) + bh, 0ull);
  ws_ptr<unsigned int>(p, ws.marr_off)[bh] = 0u;
  double bd = CUDART_INF;
  int bp = -1;
  if (k3) {
    const unsigned long long raw = ~k3;
    bd = (double)__uint_as_float((unsigned)(raw >> 32));
    bp = (int)(0xffffffffu - (unsigned)(raw & 0xffffffffull));
  }
  decide_head(p, bh, m, n_scan, bp > 0, bd, bp);
}

__device__ __forceinline__ void publish_and_decide(const MacDecodeParams& p, int bh, int m, int n_scan, int nsplit,
                                                   unsigned long long key) {
  if (publish_key(p, bh, key) == (unsigned)nsplit - 1) finish_decide(p, bh, m, n_scan);
}

}  // namespace mac
