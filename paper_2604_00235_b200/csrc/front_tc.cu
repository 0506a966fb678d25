// K0 + K1, persistent tensor-core form ("front_tc") — bf16 storage, d = 128.
//
// Same contract as front_bf16_d128_kernel (match_fast.cu): the step's KV
// appends with in-kernel RoPE (engine.py:434-437, attention.py:212-232), the
// ring match (matching.py:141-175) with its gates (engine.py:449-459), and the
// device plan of the amend work (decide_head -> plan_group, common.cuh).
//
// Why a different shape.  The match is a GEMV of one query against W ring
// rows.  On CUDA cores it is issue-bound at full HBM rate (r01 ncu: 79 %
// issue-active, 4.5 TB/s); one-shot CTAs also leave each SM idle between a
// CTA's last load and the next CTA's first.  Here the grid is persistent,
// one warp per CTA (≈6 per SM, the amend kernel's shape), and every warp
// streams a sequence of match items — (request, head, 128-row segment),
// 32 KiB each — through an 8-slot cp.async ring in shared memory (32 KiB in
// flight per warp, one item of prefetch), so loads never stop between items.
//
// Distances on the tensor cores (mma.sync.m16n8k16, bf16 in, fp32 accumulate):
//   dist = ||q||^2 + ||c||^2 - 2 q.c, clamped at 0 — the reference's own
//   expansion (matching.py:169-170).
//   q.c      A = 16 ring rows (ldmatrix from the XOR-swizzled tile), B column
//            0 = bf16 hi part of q, column 1 = lo part (q - hi): exact products,
//            no query rounding even for f32 inputs.
//   ||c||^2  B = the tile's own rows (rows 0-7: {a0, a2}, rows 8-15: {a1, a3});
//            the diagonal of the 16 x 8 products is the squared norm.
// Per 4 KiB tile a warp issues 8 cp.async + 8 ldmatrix + 24 HMMA per lane.
// Ties go to the larger position through the packed key ~(dist_bits<<32|~pos)
// (matching.py:171-173), combined across warps with atomicMax
// (publish_and_decide, front.cuh).
#include <stdlib.h>

#include "front.cuh"

namespace mac {

namespace {
constexpr int kTiles = 8;                 // 16-row tiles per match item (128 ring rows)
constexpr int kTileBytes = 16 * 256;      // 16 rows x 128 dims x bf16
constexpr int kQBytes = 128 * 8;          // one query, raw input bytes (up to f64)
constexpr int kSmem = kTiles * kTileBytes + 2 * kQBytes + 16;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// 16-byte async copy; src_bytes = 0 zero-fills the destination
__device__ __forceinline__ void cp16(uint32_t s, const void* g, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(g), "r"(src_bytes));
}
__device__ __forceinline__ void cp4(uint32_t s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(g));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N> __device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t swz(int r, int c) { return (uint32_t)(r * 256 + ((c ^ (r & 7)) << 4)); }
__device__ __forceinline__ uint32_t pack2(float lo_elem, float hi_elem) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo_elem, hi_elem);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float q_elem(const unsigned char* qs, int i, int dt) {
  if (dt == MAC_DT_BF16) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(qs)[i]);
  if (dt == MAC_DT_F32) return reinterpret_cast<const float*>(qs)[i];
  return (float)reinterpret_cast<const double*>(qs)[i];
}
}  // namespace

__global__ void __launch_bounds__(32, 6) front_tc_kernel(MacDecodeParams p, int do_match, int do_append,
                                                          int rotate_only, int plan, int n_items, int items_per_head) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x;
  const int n_app = do_append ? p.batch * p.n_kv_heads : 0;
  for (int i = blockIdx.x; i < n_app; i += gridDim.x) append_warp(p, i, rotate_only, plan);
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  const Workspace ws = workspace_layout(p);
  unsigned int* ctr = ws_ptr<unsigned int>(p, ws.ctr_off);
  if (do_match) {
    const int W = p.window, Hq = p.n_q_heads;
    const int dt = p.in_dtype;
    const int esz = dt == MAC_DT_BF16 ? 2 : (dt == MAC_DT_F32 ? 4 : 8);
    const uint32_t sm = smem_u32(smem);
    const uint32_t qsm = sm + kTiles * kTileBytes;           // 2 query buffers
    const uint32_t msm = qsm + 2 * kQBytes;                  // 2 seq_lens words
    const unsigned char* ring = static_cast<const unsigned char*>(p.ring_q);
    // first item: static for warps that did not append; later items: claimed
    const int n_static = (int)gridDim.x - (n_app < (int)gridDim.x ? n_app : (int)gridDim.x);
    // claims return lane 0's raw ticket; broadcast (and so wait for) it only when needed
    auto claim = [&]() -> unsigned { return lane == 0 ? atomicAdd(ctr + 3, 1u) : 0u; };
    auto ticket = [&](unsigned raw) -> int { return (int)__shfl_sync(0xffffffffu, raw, 0) + n_static; };
    // issue tile `tile` of `item` into slot `tile` (+ the item's query and seq_len with tile 0)
    auto issue = [&](int item, int tile, int qbuf) {
      if (item < n_items) {
        const int bh = item / items_per_head, seg = item % items_per_head;
        const int row0 = seg * (kTiles * 16) + tile * 16;
        const unsigned char* base = ring + ((int64_t)bh * W) * 256;
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) {
          const int ci = lane + 32 * rr, r = ci >> 4, c = ci & 15;
          const bool ok = row0 + r < W;
          cp16(sm + tile * kTileBytes + swz(r, c), base + (ok ? ((int64_t)(row0 + r) * 256 + c * 16) : 0), ok ? 16 : 0);
        }
        if (tile == 0) {
          const unsigned char* qg = static_cast<const unsigned char*>(p.q_pre) + (int64_t)bh * 128 * esz;
          for (int o = lane * 16; o < 128 * esz; o += 32 * 16) cp16(qsm + qbuf * kQBytes + o, qg + o, 16);
          if (lane == 0) cp4(msm + 4 * qbuf, p.seq_lens + bh / Hq);
        }
      }
      cp_commit();
    };
    const int g = lane >> 2, t = lane & 3, mi = lane >> 3, ii = lane & 7;
    const int arow = ii + 8 * (mi & 1), achunk = mi >> 1;
    const int nsrc = 4 * g + (g >> 1);  // lane holding the squared norms of rows g and g+8
    int cur = (int)blockIdx.x >= n_app ? (int)blockIdx.x - n_app : ticket(claim());
    const unsigned nxt_raw = claim();
    for (int tile = 0; tile < kTiles; ++tile) issue(cur, tile, 0);
    int nxt = ticket(nxt_raw);
    int seq = 0;
    // the previous item's publication, checked one item later (lane 0)
    unsigned pend_old = 0u;
    int pend_bh = -1, pend_m = 0, pend_scan = 0;
    while (cur < n_items) {
      const unsigned nxt2_raw = claim();  // needed one item from now
      const int bh = cur / items_per_head, seg = cur % items_per_head;
      uint32_t bq[8][2];
      float qn = 0.f;
      int m = 0, first = 0, last = 0, cur_slot = 0, n_scan = 0;
      float best = CUDART_INF_F;
      int bpos = -1;
      for (int tile = 0; tile < kTiles; ++tile) {
        cp_wait<kTiles - 1>();
        __syncwarp();
        if (tile == 0) {
          const unsigned char* qs = smem + kTiles * kTileBytes + (seq & 1) * kQBytes;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float x = q_elem(qs, lane * 4 + i, dt);
            qn = fmaf(x, x, qn);
          }
          qn = warp_sum(qn);
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            float x[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int e = ks * 16 + (i >> 1) * 8 + 2 * t + (i & 1);
              const float v = g < 2 ? q_elem(qs, e, dt) : 0.f;
              const float hi = __bfloat162float(__float2bfloat16_rn(v));
              x[i] = g == 0 ? hi : v - hi;  // column 0: hi, column 1: lo, columns 2-7: zero
            }
            bq[ks][0] = pack2(x[0], x[1]);
            bq[ks][1] = pack2(x[2], x[3]);
          }
          m = reinterpret_cast<const int*>(smem + kTiles * kTileBytes + 2 * kQBytes)[seq & 1] + 1;
          first = m - W;
          if (first < 1) first = 1;
          if (p.delta_max > 0 && m - p.delta_max > first) first = m - p.delta_max;
          last = m - 1;
          n_scan = last >= first ? last - first + 1 : 0;
          cur_slot = last >= 1 ? (last - 1) % W : 0;
        }
        float dq[4] = {0.f, 0.f, 0.f, 0.f}, n0[4] = {0.f, 0.f, 0.f, 0.f}, n1[4] = {0.f, 0.f, 0.f, 0.f};
        const uint32_t tb = sm + tile * kTileBytes;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          uint32_t a[4];
          ldsm_x4(tb + swz(arow, 2 * ks + achunk), a[0], a[1], a[2], a[3]);
          mma16816(dq, a, bq[ks][0], bq[ks][1]);
          mma16816(n0, a, a[0], a[2]);
          mma16816(n1, a, a[1], a[3]);
        }
        const float c0 = __shfl_sync(0xffffffffu, (g & 1) ? n0[1] : n0[0], nsrc);
        const float c1 = __shfl_sync(0xffffffffu, (g & 1) ? n1[3] : n1[2], nsrc);
        if (t == 0) {
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int slot = seg * (kTiles * 16) + tile * 16 + hh * 8 + g;
            const float dot = hh ? dq[2] + dq[3] : dq[0] + dq[1];
            float d = qn + (hh ? c1 : c0) - 2.f * dot;
            d = d > 0.f ? d : 0.f;
            const int pos = last - cur_slot + slot - (slot > cur_slot ? W : 0);
            const bool live = slot < W && last >= 1 && pos >= first;
            if (live && (d < best || (d == best && pos > bpos))) { best = d; bpos = pos; }
          }
        }
        __syncwarp();
        issue(nxt, tile, (seq + 1) & 1);
        if (tile == 3 && pend_bh >= 0) {
          if (lane == 0 && pend_old == (unsigned)items_per_head - 1) finish_decide(p, pend_bh, pend_m, pend_scan);
          pend_bh = -1;
          __syncwarp();
        }
      }
      unsigned long long key = 0ull;
      if (bpos > 0)
        key = ~(((unsigned long long)__float_as_uint(best) << 32) | (unsigned long long)(0xffffffffu - (unsigned)bpos));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
        key = other > key ? other : key;
      }
      if (lane == 0) pend_old = publish_key(p, bh, key);
      pend_bh = bh;
      pend_m = m;
      pend_scan = n_scan;
      cur = nxt;
      nxt = ticket(nxt2_raw);
      ++seq;
    }
    if (pend_bh >= 0 && lane == 0 && pend_old == (unsigned)items_per_head - 1)
      finish_decide(p, pend_bh, pend_m, pend_scan);
    cp_wait<0>();
  }
  // last warp out returns the item counter to zero for the next step
  if (lane == 0) {
    __threadfence();
    if (atomicAdd(ctr + 4, 1u) == gridDim.x - 1) {
      ctr[3] = 0u;
      ctr[4] = 0u;
    }
  }
}

cudaError_t launch_front_tc(const MacDecodeParams& p, cudaStream_t st, bool do_match, bool do_append, int rotate_only,
                            int plan) {
  static int grid_full = 0;
  if (!grid_full) {
    cudaError_t e = cudaFuncSetAttribute(front_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, front_tc_kernel, 32, kSmem);
    grid_full = sms * (per_sm < 1 ? 1 : per_sm);
  }
  const int items_per_head = (p.window + kTiles * 16 - 1) / (kTiles * 16);
  const int n_items = do_match ? p.batch * p.n_q_heads * items_per_head : 0;
  const int n_app = do_append ? p.batch * p.n_kv_heads : 0;
  int grid = grid_full;
  const int want = n_items + n_app;
  if (want < grid) grid = want < 1 ? 1 : want;
  front_tc_kernel<<<grid, 32, kSmem, st>>>(p, do_match ? 1 : 0, do_append ? 1 : 0, rotate_only, plan, n_items,
                                          items_per_head);
  return cudaGetLastError();
}

}  // namespace mac
