// K0 + K1 fast path ("front" kernel) — bf16 storage, d = 128, pre-RoPE matching.
//
// One launch does the step's KV append with in-kernel RoPE (engine.py:434-437,
// attention.py:212-232; same math as append.cu) and the ring match
// (matching.py:141-175; engine.py:449-459; same rule as match.cu), and its
// epilogue plans the amend work (decide_head -> plan_group, common.cuh).
//
// Match layout: the query ring [B, Hq, W, 128] bf16 is streamed as units of
// 64 rows (16 KiB).  A persistent CTA owns a contiguous run of units; one
// producer thread moves each unit into shared memory with a TMA bulk copy
// (cp.async.bulk ... mbarrier::complete_tx) through a 6-stage ring, and 8
// consumer warps compute Sum (q - c)^2 in fp32 (a half-warp per row, 16 B per
// lane, 4 xor-shuffles).  Each warp folds its rows into (best, pos) per
// (request, head) and publishes it with one 64-bit atomicMax of the
// complemented key (dist_bits << 32 | ~pos): max ~key = min distance, ties to
// the larger position (matching.py:171-173).  Rows scanned are counted per
// (request, head); the warp that completes the count decides the head and
// resets the key/counter to zero for the next step (graph-replay safe).
#include "common.cuh"

namespace mac {

namespace {
constexpr int kConsumerWarps = 8;
constexpr int kThreads = (kConsumerWarps + 1) * 32;
constexpr int kUnitRows = 64;
constexpr int kUnitBytes = kUnitRows * 256;
constexpr int kStages = 6;
constexpr int kSmem = kStages * kUnitBytes + 2 * kStages * 8 + 16;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, unsigned bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

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

// append + RoPE for one (request, kv head); optionally plan the group as "all heads miss"
__device__ void append_block(const MacDecodeParams& p, int idx, int rotate_only, int plan) {
  const int b = idx / p.n_kv_heads, kvh = idx % p.n_kv_heads;
  const int g = p.n_q_heads / p.n_kv_heads;
  const Workspace w = workspace_layout(p);
  const int m = p.seq_lens[b] + (rotate_only ? 0 : 1);
  if (kvh == 0 && threadIdx.x == 0) ws_ptr<int>(p, w.mpos_off)[b] = m;
  const int t_local = m - p.kv_offset;
  const bool store = !rotate_only && t_local >= 1;
  int64_t row = 0;
  if (store) row = kv_row(p.page_table, p.pages_per_seq, b, t_local, p.page_size, p.n_kv_heads, kvh);
  __nv_bfloat16* kc = static_cast<__nv_bfloat16*>(p.k_cache);
  __nv_bfloat16* vc = static_cast<__nv_bfloat16*>(p.v_cache);
  float* qrot = ws_ptr<float>(p, w.qrot_off);
  const int j = threadIdx.x;
  if (j < 64) {
    double s, c;
    sincos((double)m * p.rope_freqs[j], &s, &c);
    if (store) {
      const int64_t ki = ((int64_t)b * p.n_kv_heads + kvh) * 128 + 2 * j;
      const double x0 = load_in(p.k_pre, ki, p.in_dtype), x1 = load_in(p.k_pre, ki + 1, p.in_dtype);
      __nv_bfloat162 kk;
      kk.x = from_f64<__nv_bfloat16>(x0 * c - x1 * s);
      kk.y = from_f64<__nv_bfloat16>(x0 * s + x1 * c);
      reinterpret_cast<__nv_bfloat162*>(kc + row * 128)[j] = kk;
    }
    for (int hl = 0; hl < g; ++hl) {
      const int64_t qi = ((int64_t)b * p.n_q_heads + kvh * g + hl) * 128 + 2 * j;
      const double x0 = load_in(p.q_pre, qi, p.in_dtype), x1 = load_in(p.q_pre, qi + 1, p.in_dtype);
      reinterpret_cast<float2*>(qrot + qi)[0] = make_float2((float)(x0 * c - x1 * s), (float)(x0 * s + x1 * c));
    }
  } else if (store && j < 64 + 128) {
    const int e = j - 64;
    vc[row * 128 + e] = from_f64<__nv_bfloat16>(load_in(p.v_in, ((int64_t)b * p.n_kv_heads + kvh) * 128 + e,
                                                         p.in_dtype));
  }
  if (plan && threadIdx.x == 0) {
    int* lo = ws_ptr<int>(p, w.lo_off);
    for (int hl = 0; hl < g; ++hl) lo[b * p.n_q_heads + kvh * g + hl] = 1;
    plan_group(p, b, kvh, m, 1);
  }
}
}  // namespace

__global__ void __launch_bounds__(kThreads, 2) front_bf16_d128_kernel(MacDecodeParams p, int n_match_ctas,
                                                                      int do_append, int rotate_only, int plan) {
  if ((int)blockIdx.x >= n_match_ctas) {
    if (do_append) append_block(p, blockIdx.x - n_match_ctas, rotate_only, plan);
    return;
  }
  extern __shared__ __align__(128) unsigned char smem[];
  const uint32_t sbase = smem_u32(smem);
  const uint32_t full0 = sbase + kStages * kUnitBytes, empty0 = full0 + kStages * 8;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int W = p.window, Hq = p.n_q_heads;
  const int upb = (W + kUnitRows - 1) / kUnitRows;  // units per (request, head)
  const long units = (long)p.batch * Hq * upb;
  const long u_begin = units * blockIdx.x / n_match_ctas, u_end = units * (blockIdx.x + 1) / n_match_ctas;
  const Workspace ws = workspace_layout(p);
  unsigned long long* keys = ws_ptr<unsigned long long>(p, ws.mkey_off);
  unsigned int* rows_seen = ws_ptr<unsigned int>(p, ws.marr_off);

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    // ---------------- producer: one elected thread issues the bulk copies ----------------
    if (lane == 0) {
      const char* ring = static_cast<const char*>(p.ring_q);
      long k = 0;
      for (long u = u_begin; u < u_end; ++u, ++k) {
        const int s = (int)(k % kStages);
        if (k >= kStages) mbar_wait(empty0 + 8 * s, (unsigned)(((k / kStages) - 1) & 1));
        const long bh = u / upb;
        const int ub = (int)(u % upb);
        const int rows = min(kUnitRows, W - ub * kUnitRows);
        const unsigned bytes = (unsigned)rows * 256u;
        mbar_expect_tx(full0 + 8 * s, bytes);
        bulk_g2s(sbase + s * kUnitBytes, ring + ((bh * W + (long)ub * kUnitRows) * 256), bytes, full0 + 8 * s);
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const int sub = lane & 15, half = lane >> 4;
  long cur = -1;
  int m = 0, first = 1, last = 0, n_scan = 0;
  unsigned my_rows = 0;
  float q[8];
  float best = CUDART_INF_F;
  int bpos = -1;

  auto flush = [&]() {
    // warp-reduce (best, bpos): both half-warps hold their own candidate
    unsigned long long key = 0ull;
    if (bpos > 0)
      key = ~(((unsigned long long)__float_as_uint(best) << 32) | (unsigned long long)(0xffffffffu - (unsigned)bpos));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
      key = other > key ? other : key;
    }
    if (lane == 0) {
      if (key) atomicMax(keys + cur, key);
      __threadfence();
      const unsigned prev = atomicAdd(rows_seen + cur, my_rows);
      if (prev + my_rows == (unsigned)W) {  // every ring row of this head scanned: decide
        __threadfence();
        const unsigned long long k3 = atomicExch(keys + cur, 0ull);
        rows_seen[cur] = 0u;
        double bd = CUDART_INF;
        int bp = -1;
        if (k3) {
          const unsigned long long raw = ~k3;
          bd = (double)__uint_as_float((unsigned)(raw >> 32));
          bp = (int)(0xffffffffu - (unsigned)(raw & 0xffffffffull));
        }
        decide_head(p, (int)cur, m, n_scan, bp > 0, bd, bp);
      }
    }
  };

  long k = 0;
  for (long u = u_begin; u < u_end; ++u, ++k) {
    const int s = (int)(k % kStages);
    const long bh = u / upb;
    const int ub = (int)(u % upb);
    if (bh != cur) {
      if (cur >= 0) flush();
      cur = bh;
      const int b = (int)(bh / Hq);
      m = p.seq_lens[b] + 1;
      first = m - W;
      if (first < 1) first = 1;
      if (p.delta_max > 0 && m - p.delta_max > first) first = m - p.delta_max;
      last = m - 1;
      n_scan = last >= first ? last - first + 1 : 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) q[i] = (float)load_in(p.q_pre, bh * 128 + sub * 8 + i, p.in_dtype);
      best = CUDART_INF_F;
      bpos = -1;
      my_rows = 0;
    }
    const int rows = min(kUnitRows, W - ub * kUnitRows);
    mbar_wait(full0 + 8 * s, (unsigned)((k / kStages) & 1));
    const unsigned char* st = smem + s * kUnitBytes;
#pragma unroll
    for (int it = 0; it < kUnitRows / (2 * kConsumerWarps); ++it) {
      const int r = warp * (kUnitRows / kConsumerWarps) + it * 2 + half;
      float d = 0.f;
      if (r < rows) d = dist8(q, *reinterpret_cast<const uint4*>(st + r * 256 + sub * 16));
      d += __shfl_xor_sync(0xffffffffu, d, 8);
      d += __shfl_xor_sync(0xffffffffu, d, 4);
      d += __shfl_xor_sync(0xffffffffu, d, 2);
      d += __shfl_xor_sync(0xffffffffu, d, 1);
      const int slot = ub * kUnitRows + r;
      const int pos = last - ((last - 1 - slot) % W + W) % W;  // latest position held by the slot
      const bool live = r < rows && last >= 1 && pos >= first;
      if (live && (d < best || (d == best && pos > bpos))) { best = d; bpos = pos; }
    }
    const int mine = rows - warp * (kUnitRows / kConsumerWarps);
    my_rows += mine <= 0 ? 0 : (mine > kUnitRows / kConsumerWarps ? kUnitRows / kConsumerWarps : mine);
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8 * s);
  }
  if (cur >= 0) flush();
}

bool match_fast_supported(const MacDecodeParams& p) {
  return p.storage == MAC_MODE_BF16 && p.head_dim == 128 && p.head_dim_v == 128 && p.match_space == MAC_MATCH_PRE_ROPE;
}
bool front_fast_supported(const MacDecodeParams& p) {
  return p.storage == MAC_MODE_BF16 && p.head_dim == 128 && p.head_dim_v == 128;
}

// match: persistent CTAs over the ring; append: B*Hkv extra CTAs in the same launch
cudaError_t launch_front_bf16(const MacDecodeParams& p, cudaStream_t st, bool do_match, bool do_append,
                              int rotate_only, int plan) {
  static int sms = 0;
  if (!sms) {
    cudaError_t e = cudaFuncSetAttribute(front_bf16_d128_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (e != cudaSuccess) return e;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int n_match = 0;
  if (do_match) {
    const long units = (long)p.batch * p.n_q_heads * ((p.window + kUnitRows - 1) / kUnitRows);
    n_match = (int)(units < 2L * sms ? units : 2L * sms);
  }
  const int n_append = do_append ? p.batch * p.n_kv_heads : 0;
  if (n_match + n_append == 0) return cudaSuccess;
  front_bf16_d128_kernel<<<n_match + n_append, kThreads, kSmem, st>>>(p, n_match, do_append ? 1 : 0, rotate_only,
                                                                      plan);
  return cudaGetLastError();
}

}  // namespace mac
