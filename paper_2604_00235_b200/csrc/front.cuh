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

// append + RoPE for one (request, kv head) by one warp; optionally plan the group as "all heads miss"
// HOST: compiled with the staging of host-resident inputs (inputs_host) and with pair / 8-byte
// loads of q, k, v (each load instruction is a PCIe read there: C3 e2e 65.6 -> 63.7 us); the
// kernels the device-input steps launch leave both out (they raised the scan kernel from 56 to
// 61-64 registers: +0.4 us on the device step)
template <bool HOST = true>
__device__ __forceinline__ void append_warp(const MacDecodeParams& p, int idx, int rotate_only, int plan) {
  const int lane = threadIdx.x & 31;
  const int b = idx / p.n_kv_heads, kvh = idx % p.n_kv_heads;
  const int g = p.n_q_heads / p.n_kv_heads;
  const Workspace w = workspace_layout(p);
  const int m = p.seq_lens[b] + (rotate_only ? 0 : 1);
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
  const int t_local = m - p.kv_offset;
  bool store = !rotate_only && t_local >= 1 && (p.kv_limit <= 0 || t_local <= p.kv_limit);
  if (store && !kv_fits(p.pages_per_seq, t_local, p.page_size)) {
    store = false;
    if (lane == 0) atomicOr(ws_ptr<unsigned>(p, w.ctr_off) + 2, 1u);
  }
  int64_t row = 0;
  if (store) row = kv_row(p.page_table, p.pages_per_seq, b, t_local, p.page_size, p.n_kv_heads, kvh);
  __nv_bfloat16* kc = static_cast<__nv_bfloat16*>(p.k_cache);
  __nv_bfloat16* vc = static_cast<__nv_bfloat16*>(p.v_cache);
  float* qrot = ws_ptr<float>(p, w.qrot_off);
  void* qstage = ws_ptr<void>(p, w.qstage_off);
  // bf16 / f32 inputs (exact in fp32 registers): each head's query pair used to be loaded after
  // the previous head's store — a memory round trip per head, which made the append warps, not
  // the scan, end the front kernel (C2: the verify waited 6.7 us past the last scan CTA)
  const bool batch = p.in_dtype != MAC_DT_F64;
  for (int j = lane; j < 64; j += 32) {
    double s, c;
    sincos((double)m * p.rope_freqs[j], &s, &c);
    if (store) {
      const int64_t ki = ((int64_t)b * p.n_kv_heads + kvh) * 128 + 2 * j;
      double x0, x1;
      if (HOST) load_pair(p.k_pre, ki, p.in_dtype, x0, x1);
      else x0 = load_in(p.k_pre, ki, p.in_dtype), x1 = load_in(p.k_pre, ki + 1, p.in_dtype);
      __nv_bfloat162 kk;
      kk.x = from_f64<__nv_bfloat16>(x0 * c - x1 * s);
      kk.y = from_f64<__nv_bfloat16>(x0 * s + x1 * c);
      reinterpret_cast<__nv_bfloat162*>(kc + row * 128)[j] = kk;
    }
    if (batch) {  // four heads' query pairs in flight together, then their stores
      for (int h0 = 0; h0 < g; h0 += 4) {
        float xa[4], xb[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int64_t qi = ((int64_t)b * p.n_q_heads + kvh * g + h0 + t) * 128 + 2 * j;
          if (HOST) {
            double d0 = 0.0, d1 = 0.0;
            if (h0 + t < g) load_pair(p.q_pre, qi, p.in_dtype, d0, d1);
            xa[t] = (float)d0;
            xb[t] = (float)d1;
          } else {
            xa[t] = h0 + t < g ? (float)load_in(p.q_pre, qi, p.in_dtype) : 0.f;
            xb[t] = h0 + t < g ? (float)load_in(p.q_pre, qi + 1, p.in_dtype) : 0.f;
          }
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          if (h0 + t >= g) break;
          const int64_t qi = ((int64_t)b * p.n_q_heads + kvh * g + h0 + t) * 128 + 2 * j;
          const double x0 = xa[t], x1 = xb[t];
          reinterpret_cast<float2*>(qrot + qi)[0] = make_float2((float)(x0 * c - x1 * s), (float)(x0 * s + x1 * c));
          if (HOST && p.inputs_host)  // host-resident inputs: stage the raw query for the later kernels
            store_pair(qstage, qi, x0, x1, p.in_dtype);
        }
      }
    } else {
      for (int hl = 0; hl < g; ++hl) {
        const int64_t qi = ((int64_t)b * p.n_q_heads + kvh * g + hl) * 128 + 2 * j;
        double x0, x1;
        if (HOST) load_pair(p.q_pre, qi, p.in_dtype, x0, x1);
        else x0 = load_in(p.q_pre, qi, p.in_dtype), x1 = load_in(p.q_pre, qi + 1, p.in_dtype);
        reinterpret_cast<float2*>(qrot + qi)[0] = make_float2((float)(x0 * c - x1 * s), (float)(x0 * s + x1 * c));
        if (HOST && p.inputs_host) store_pair(qstage, qi, x0, x1, p.in_dtype);
      }
    }
  }
  if (store && !HOST) {
    for (int e = lane; e < 128; e += 32)
      vc[row * 128 + e] =
          from_f64<__nv_bfloat16>(load_in(p.v_in, ((int64_t)b * p.n_kv_heads + kvh) * 128 + e, p.in_dtype));
  } else if (store) {  // host inputs: four consecutive values a lane (two pair loads, one 8-byte store)
    const int64_t vi = ((int64_t)b * p.n_kv_heads + kvh) * 128 + 4 * lane;
    double v0, v1, v2, v3;
    load_pair(p.v_in, vi, p.in_dtype, v0, v1);
    load_pair(p.v_in, vi + 2, p.in_dtype, v2, v3);
    __nv_bfloat162 lo, hi;
    lo.x = from_f64<__nv_bfloat16>(v0);
    lo.y = from_f64<__nv_bfloat16>(v1);
    hi.x = from_f64<__nv_bfloat16>(v2);
    hi.y = from_f64<__nv_bfloat16>(v3);
    uint2 w;
    w.x = *reinterpret_cast<uint32_t*>(&lo);
    w.y = *reinterpret_cast<uint32_t*>(&hi);
    *reinterpret_cast<uint2*>(vc + row * 128 + 4 * lane) = w;
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
