// Prefill ring construction on the 5th-generation tensor cores (tcgen05 / TMEM / TMA): the same
// contract as ring_build.cu (the ring entries of the last n positions of a cached prompt,
// slot (t-1) mod W <- (q_t, AS[1, t-r] under R_t q_t); engine.py:374-402, 484-499) computed as a
// flash-attention pass with a causal lag of r.
//
// CTA = (request, kv head, block of 256/g positions -> two 128-row query tiles of positions x g
// heads, key chunk).  The two tiles share every K/V tile and ping-pong on the tensor core: while
// one tile's softmax runs, the other tile's MMAs do.  Warp roles (320 threads):
//   warps 0-3 / 4-7  tile 0 / tile 1, one thread per row (TMEM lane 32 (w % 4) + lane): rotate
//              the query (fp64 angles), pre-scale it by log2(e)/sqrt(d), split it hi/lo into the
//              tile's two bf16 A operands (shared memory); per 64-key tile read the S row from
//              TMEM, online softmax in the log2 domain (lazy rescale: the reference max moves
//              only by > 8; O is then rescaled in TMEM), write P hi/lo as packed bf16 into the
//              same TMEM columns the S row came from; epilogue O / Z and lse -> ring slot
//   warp 8     one elected thread issues the UMMAs: S_t = Q_hi K^T + Q_lo K^T (A and B K-major
//              in shared memory, M = 128, N = 64, double-buffered per tile) and
//              O_t += P_hi V + P_lo V (A = P from TMEM, B = V MN-major in shared memory, N = 128);
//              tcgen05.commit signals S ready / O updated / K/V stage free
//   warp 9     TMA producer: each 64-key tile is 4 pages x 2 dim halves of K and of V (2D tensor
//              maps over the paged cache, SWIZZLE_128B = the UMMA canonical layout), 3 stages
// TMEM per tile: S/P buffers at columns 256 t + {0, 64}, O at 256 t + 128 (all 512 columns).
// The hi/lo splits keep the logits and P exact to fp32 (the parity the decode kernels hold, see
// amend_mma.cuh).  Descriptor and TMEM layouts: umma.cuh, validated against a host GEMM by
// tools/umma_probe.cu (including the TMEM A operand).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "umma.cuh"

namespace mac {

bool encode_cache_map(CUtensorMap* m, const void* ptr);  // amend_tma.cu

namespace {
using namespace umma;
constexpr int TC_THREADS = 320;            // 8 softmax warps (two tiles), the UMMA issuer, the TMA producer
constexpr int TC_NS = 3;                   // K/V stages
constexpr int TC_TILE = 64;                // keys per tile
constexpr int Q_TILE = 65536;              // one query tile: hi 32 KB + lo 32 KB (2 atoms x 128 rows x 128 B each)
constexpr int OFF_Q = 0, OFF_KV = 2 * Q_TILE;
constexpr int KV_STAGE = 32768;            // K 16 KB (2 atoms x 64 keys x 128 B) + V 16 KB
constexpr int OFF_BAR = OFF_KV + TC_NS * KV_STAGE;
constexpr int TC_SMEM = OFF_BAR + 256 + 1024;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

__device__ __forceinline__ uint32_t kmaj_off(int r, int k, int R) {
  return (uint32_t)((k >> 6) * R * 128 + r * 128 + ((((k & 63) >> 3) ^ (r & 7)) << 4) + (k & 7) * 2);
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}
// packed fp32 pairs (sm_100 FADD2) and the three-input max (FMNMX3): the softmax rows run at
// about 30 % fewer instructions for the same roundings.  (Measured: C3 ring 125.9 vs 125.4 ms,
// C2 7.8 vs 8.0 ms — the kernel is not issue-bound; ncu: tensor pipe ~50 % active, r02.)
__device__ __forceinline__ unsigned long long f2pack(float lo, float hi) {
  return ((unsigned long long)__float_as_uint(hi) << 32) | __float_as_uint(lo);
}
__device__ __forceinline__ unsigned long long add2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ float f2lo(unsigned long long v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float f2hi(unsigned long long v) { return __uint_as_float((uint32_t)(v >> 32)); }
__device__ __forceinline__ float max3f(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ void tma2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
}  // namespace

__global__ void __launch_bounds__(TC_THREADS, 1)
    ring_build_tc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                         MacDecodeParams p, MacRingBuildParams a) {
  extern __shared__ unsigned char smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  unsigned char* sm = smem_raw + (base - raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int Hkv = p.n_kv_heads, Hq = p.n_q_heads, g = Hq / Hkv, r = p.band, ps = p.page_size, W = p.window;
  const int pb_rows = 256 / g;  // positions per CTA (two tiles of 128 / g)
  const int n_pb = (a.n_rows + pb_rows - 1) / pb_rows;
  int item = blockIdx.x;
  const int ch = item % a.n_chunks;
  item /= a.n_chunks;
  const int pb = item % n_pb;
  item /= n_pb;
  const int kvh = item % Hkv, b = item / Hkv;
  const int n = p.seq_lens[b];
  const int first = n - a.n_rows + 1;
  const int i0 = pb * pb_rows;
  const int i_last = min(a.n_rows, i0 + pb_rows) - 1;
  const int kmax = first + i_last - r;
  const int span = kmax >= 1 ? (kmax + TC_TILE - 1) / TC_TILE : 0;
  const int per = (span + a.n_chunks - 1) / a.n_chunks;
  const int tile0 = ch * per, nt = max(0, min(span, tile0 + per) - tile0);
  const int k0 = 1 + tile0 * TC_TILE, k1 = min(kmax, (tile0 + per) * TC_TILE);

  const uint32_t bar = base + OFF_BAR;
  // full[NS] empty[NS] sfull[2 tiles][2 bufs] odone[2] pfull[2] qfull[2]
  const uint32_t b_full = bar, b_empty = bar + 8 * TC_NS, b_sfull = bar + 16 * TC_NS, b_odone = b_sfull + 32,
                 b_pfull = b_odone + 16, b_qfull = b_pfull + 16;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + OFF_BAR + 160);
  if (tid == 0) {
    for (int i = 0; i < TC_NS; ++i) {
      mbar_init(b_full + 8 * i, 1);
      mbar_init(b_empty + 8 * i, 1);
    }
    for (int i = 0; i < 4; ++i) mbar_init(b_sfull + 8 * i, 1);
    for (int t = 0; t < 2; ++t) {
      mbar_init(b_odone + 8 * t, 1);
      mbar_init(b_pfull + 8 * t, 128);
      mbar_init(b_qfull + 8 * t, 128);
    }
    fence_mbar_init();
  }
  if (warp == 8) tmem_alloc(smem_u32(tmem_slot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = *tmem_slot;

  if (warp == 9) {
    // ------------------------------------------------------------------ TMA producer
    for (int j = 0; j < nt; ++j) {
      const int st = j % TC_NS;
      int row = 0;  // lane s < 4: the cache row of sub-tile s (16 keys inside one page)
      if (lane < 4) {
        const int tok = k0 + j * TC_TILE + lane * 16;
        const int pg = p.page_table[(int64_t)b * p.pages_per_seq + min((tok - 1) / ps, p.pages_per_seq - 1)];
        row = (pg * Hkv + kvh) * ps + ((tok - 1) % ps);
      }
      const int r0 = __shfl_sync(0xffffffffu, row, 0), r1 = __shfl_sync(0xffffffffu, row, 1);
      const int r2 = __shfl_sync(0xffffffffu, row, 2), r3 = __shfl_sync(0xffffffffu, row, 3);
      if (lane == 0) {
        mbar_wait_parity(b_empty + 8 * st, ((j / TC_NS) & 1) ^ 1);
        const uint32_t fb = b_full + 8 * st;
        mbar_expect_tx(fb, KV_STAGE);
        const uint32_t ks = base + OFF_KV + st * KV_STAGE, vs = ks + 16384;
        const int rows[4] = {r0, r1, r2, r3};
#pragma unroll
        for (int s = 0; s < 4; ++s)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            tma2d(ks + h * 8192 + s * 2048, &tmK, h * 64, rows[s], fb);
            tma2d(vs + h * 8192 + s * 2048, &tmV, h * 64, rows[s], fb);
          }
      }
    }
  } else if (warp == 8) {
    // ------------------------------------------------------------------ UMMA issuer
    if (lane == 0 && nt > 0) {
      const uint32_t idS = instr_desc_bf16(128, TC_TILE, false, false);
      const uint32_t idO = instr_desc_bf16(128, 128, false, true);
      auto issue_s = [&](int t, int j) {  // S_t(j) into buffer j % 2 of tile t
        const uint32_t qhi = base + OFF_Q + t * Q_TILE, qlo = qhi + 32768;
        const uint32_t ks = base + OFF_KV + (j % TC_NS) * KV_STAGE;
        const uint32_t d = tm + (uint32_t)(256 * t + (j & 1) * TC_TILE);
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {  // 8 k-steps of the hi operand, then 8 of the lo operand
          const int ks8 = kk & 7;
          const uint32_t aoff = (ks8 >> 2) * 16384 + (ks8 & 3) * 32, boff = (ks8 >> 2) * 8192 + (ks8 & 3) * 32;
          mma_bf16(d, sdesc_kmajor_sw128((kk < 8 ? qhi : qlo) + aoff), sdesc_kmajor_sw128(ks + boff), idS, kk > 0);
        }
        mma_commit(b_sfull + 8 * (2 * t + (j & 1)));
      };
      auto issue_pv = [&](int t, int j) {  // O_t += P_t(j) . V(j), P hi/lo from TMEM buffer j % 2
        mbar_wait_parity(b_pfull + 8 * t, j & 1);
        tc_fence_after();
        const uint32_t vs = base + OFF_KV + (j % TC_NS) * KV_STAGE + 16384;
        const uint32_t pa = tm + (uint32_t)(256 * t + (j & 1) * TC_TILE);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // P_hi (columns 0..31) then P_lo (32..63), 8 columns per 16 keys
          const int k4 = kk & 3;
          mma_bf16_ta(tm + (uint32_t)(256 * t + 128), pa + (uint32_t)((kk >> 2) * 32 + k4 * 8),
                      sdesc_mnmajor_sw128(vs + k4 * 2048, 8192), idO, j > 0 || kk > 0);
        }
        mma_commit(b_odone + 8 * t);
      };
      mbar_wait_parity(b_qfull, 0);
      mbar_wait_parity(b_qfull + 8, 0);
      tc_fence_after();
      for (int j = 0; j <= nt; ++j) {
        if (j < nt) {
          mbar_wait_parity(b_full + 8 * (j % TC_NS), (j / TC_NS) & 1);
          tc_fence_after();
          issue_s(0, j);
          issue_s(1, j);
        }
        if (j > 0) {
          issue_pv(0, j - 1);
          issue_pv(1, j - 1);
          mma_commit(b_empty + 8 * ((j - 1) % TC_NS));
        }
      }
    }
  } else {
    // ------------------------------------------------------------------ softmax rows
    const int t = warp >> 2;                 // query tile
    const int rho = (warp & 3) * 32 + lane;  // row of the tile = TMEM lane
    const int pi = t * (128 / g) + rho / g, hl = rho % g;
    const int ri = i0 + pi;
    const bool rvalid = ri < a.n_rows;
    const int pos = first + ri;
    const int head = kvh * g + hl;
    const int hi_row = rvalid ? pos - r : 0;
    const float scale2 = (float)(1.0 / sqrt(128.0)) * kLog2e;
    {  // the query row: rotated at pos (fp64 angles), scaled into the log2 domain, split hi/lo
      const int64_t qb = ((int64_t)(b * a.n_rows + (rvalid ? ri : 0)) * Hq + head) * 128;
      unsigned char* qh = sm + OFF_Q + t * Q_TILE;
      unsigned char* ql = qh + 32768;
      for (int c = 0; c < 16; ++c) {  // 16-byte chunk c: dims 8c .. 8c+7
        uint32_t h4[4], l4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = 4 * c + u;  // rotation pair (2j, 2j+1)
          float e0 = 0.f, e1 = 0.f;
          if (rvalid) {
            double sn, cs;
            sincos((double)pos * p.rope_freqs[j], &sn, &cs);
            const double x0 = load_in(p.q_pre, qb + 2 * j, p.in_dtype), x1 = load_in(p.q_pre, qb + 2 * j + 1, p.in_dtype);
            e0 = (float)(x0 * cs - x1 * sn) * scale2;
            e1 = (float)(x0 * sn + x1 * cs) * scale2;
          }
          h4[u] = pack2(e0, e1);
          l4[u] = pack2(e0 - __uint_as_float(h4[u] << 16), e1 - __uint_as_float(h4[u] & 0xffff0000u));
        }
        const uint32_t off = kmaj_off(rho, 8 * c, 128);
        *reinterpret_cast<uint4*>(qh + off) = make_uint4(h4[0], h4[1], h4[2], h4[3]);
        *reinterpret_cast<uint4*>(ql + off) = make_uint4(l4[0], l4[1], l4[2], l4[3]);
      }
      fence_proxy_async_smem();
      mbar_arrive(b_qfull + 8 * t);
    }
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t tcol = (uint32_t)(256 * t);
    const int hi_mask = min(hi_row, k1);
    float M = -CUDART_INF_F, Z = 0.f;
    int odone_seen = 0;  // O-update phases of this tile waited for (in order: parity waits stay exact)
    auto wait_odone = [&](int upto) {  // PV_t(0 .. upto-1) complete
      for (; odone_seen < upto; ++odone_seen) mbar_wait_parity(b_odone + 8 * t, odone_seen & 1);
      tc_fence_after();
    };
    for (int j = 0; j < nt; ++j) {
      mbar_wait_parity(b_sfull + 8 * (2 * t + (j & 1)), (j >> 1) & 1);
      tc_fence_after();
      const uint32_t sa = tm + lane_base + tcol + (uint32_t)((j & 1) * TC_TILE);
      float l[64];
      {
        uint32_t v[32];
        tmem_ld32(sa, v);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 32; ++c) l[c] = __uint_as_float(v[c]);
        tmem_ld32(sa + 32, v);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 32; ++c) l[32 + c] = __uint_as_float(v[c]);
      }
      const int kt = k0 + j * TC_TILE;
      if (kt + TC_TILE - 1 > hi_mask) {  // a tile reaching past this row's last key: mask
#pragma unroll
        for (int c = 0; c < 64; ++c) l[c] = (kt + c <= hi_mask) ? l[c] : -CUDART_INF_F;
      }
      float mx;
      {  // three-input max tree: 64 -> 22 -> 8 -> 3 -> 1
        float m22[22];
#pragma unroll
        for (int c = 0; c < 21; ++c) m22[c] = max3f(l[3 * c], l[3 * c + 1], l[3 * c + 2]);
        m22[21] = l[63];
        float m8[8];
#pragma unroll
        for (int c = 0; c < 7; ++c) m8[c] = max3f(m22[3 * c], m22[3 * c + 1], m22[3 * c + 2]);
        m8[7] = m22[21];
        mx = max3f(max3f(m8[0], m8[1], m8[2]), max3f(m8[3], m8[4], m8[5]), fmaxf(m8[6], m8[7]));
      }
      const float Mn = (M == -CUDART_INF_F || mx > M + 8.f) ? fmaxf(M, mx) : M;
      const float alpha = (M == -CUDART_INF_F || Mn == M) ? 1.f : exp2f(M - Mn);
      float zs;
      {
        const float nm = (Mn == -CUDART_INF_F) ? 0.f : -Mn;  // a fully masked row: exp2(-inf) = 0
        const unsigned long long nm2 = f2pack(nm, nm);
        unsigned long long z4[4] = {0ull, 0ull, 0ull, 0ull};  // the pairs (c & 7) = (0,1) (2,3) (4,5) (6,7)
#pragma unroll
        for (int c = 0; c < 64; c += 2) {
          const unsigned long long x = add2(f2pack(l[c], l[c + 1]), nm2);
          l[c] = exp2f(f2lo(x));
          l[c + 1] = exp2f(f2hi(x));
          z4[(c & 7) >> 1] = add2(z4[(c & 7) >> 1], f2pack(l[c], l[c + 1]));
        }
        zs = ((f2lo(z4[0]) + f2hi(z4[0])) + (f2lo(z4[1]) + f2hi(z4[1]))) +
             ((f2lo(z4[2]) + f2hi(z4[2])) + (f2lo(z4[3]) + f2hi(z4[3])));
      }
      Z = Z * alpha + zs;
      if (__any_sync(0xffffffffu, alpha != 1.f)) {  // O row *= alpha once PV(j-1) has landed
        wait_odone(j);
        uint32_t v[32];
#pragma unroll
        for (int c = 0; c < 128; c += 32) {
          const uint32_t oa = tm + lane_base + tcol + 128 + c;
          tmem_ld32(oa, v);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = __float_as_uint(__uint_as_float(v[e]) * alpha);
          tmem_st32(oa, v);
        }
      }
      M = Mn;
      {  // P hi (columns 0..31) and lo (32..63), two bf16 per column, over the S row just read
        uint32_t ph[32], pl[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const float x0 = l[2 * c], x1 = l[2 * c + 1];
          ph[c] = pack2(x0, x1);
          // lo = x - hi for both halves in one FADD2 (hi negated through its sign bits)
          const unsigned long long nh = f2pack(__uint_as_float((ph[c] << 16) ^ 0x80000000u),
                                               __uint_as_float((ph[c] & 0xffff0000u) ^ 0x80000000u));
          const unsigned long long lo = add2(f2pack(x0, x1), nh);
          pl[c] = pack2(f2lo(lo), f2hi(lo));
        }
        tmem_st32(sa, ph);
        tmem_st32(sa + 32, pl);
      }
      tmem_wait_st();
      // P(j) may be published only once PV(j-1) consumed P(j-1): the issuer then already waited
      // for phase j-1 of this barrier, so it can never observe two of its phases at once (a
      // parity wait cannot tell them apart).  PV(j-1) was issued ~one softmax ago: rarely a wait.
      if (j > 0) wait_odone(j);
      tc_fence_before();
      mbar_arrive(b_pfull + 8 * t);
    }
    // epilogue: this row's normalised (acc, lse), 32 TMEM columns at a time
    if (nt > 0) wait_odone(nt);
    const float inv = Z > 0.f ? 1.f / Z : 0.f;
    const float lse = Z > 0.f ? M * kLn2 + logf(Z) : -CUDART_INF_F;
    const int slot = rvalid ? (pos - 1) % W : 0;
    float* dst = nullptr;
    if (rvalid) {
      if (a.n_chunks == 1) {
        dst = static_cast<float*>(p.ring_acc) + (((int64_t)b * Hq + head) * W + slot) * 128;
        static_cast<float*>(p.ring_lse)[((int64_t)b * Hq + head) * W + slot] = lse;
      } else {
        dst = static_cast<float*>(a.part) + ((((int64_t)b * a.n_rows + ri) * Hq + head) * a.n_chunks + ch) * 129;
        dst[128] = lse;
      }
    }
#pragma unroll 1
    for (int c = 0; c < 128; c += 32) {
      uint32_t v[32];
      if (nt > 0) {
        tmem_ld32(tm + lane_base + tcol + 128 + c, v);  // warp-collective: every lane takes part
        tmem_wait_ld();
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = 0u;
      }
      if (rvalid) {
#pragma unroll
        for (int e = 0; e < 32; e += 4) {
          const float4 v4 = make_float4(__uint_as_float(v[e]) * inv, __uint_as_float(v[e + 1]) * inv,
                                        __uint_as_float(v[e + 2]) * inv, __uint_as_float(v[e + 3]) * inv);
          if (a.n_chunks == 1) *reinterpret_cast<float4*>(dst + c + e) = v4;
          else { dst[c + e] = v4.x; dst[c + e + 1] = v4.y; dst[c + e + 2] = v4.z; dst[c + e + 3] = v4.w; }
        }
      }
    }
    if (rvalid && ch == 0) {  // the ring's query row (pre-RoPE, bf16 like the decode write-back)
      const int64_t qb = ((int64_t)(b * a.n_rows + ri) * Hq + head) * 128;
      __nv_bfloat16* rq = static_cast<__nv_bfloat16*>(p.ring_q) + (((int64_t)b * Hq + head) * W + slot) * 128;
      for (int e = 0; e < 128; ++e) rq[e] = from_f64<__nv_bfloat16>(load_in(p.q_pre, qb + e, p.in_dtype));
      if (p.ring_qp) {
        __nv_bfloat16* rp =
            static_cast<__nv_bfloat16*>(p.ring_qp) + (((int64_t)b * Hq + head) * W + slot) * MAC_PLANAR_DIMS;
        for (int e = 0; e < MAC_PLANAR_DIMS; ++e) rp[e] = from_f64<__nv_bfloat16>(load_in(p.q_pre, qb + e, p.in_dtype));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 8) tmem_dealloc(tm, 512);
}

bool ring_build_tc_supported(const MacDecodeParams& p) {
  const int g = p.n_q_heads / p.n_kv_heads;
  return p.storage == MAC_MODE_BF16 && p.head_dim == 128 && p.head_dim_v == 128 && g >= 1 && 128 % g == 0 &&
         g <= 8 && p.page_size % 16 == 0 && p.kv_offset == 0 && p.kv_limit == 0 &&
         (reinterpret_cast<uintptr_t>(p.k_cache) & 15) == 0 && (reinterpret_cast<uintptr_t>(p.v_cache) & 15) == 0;
}

cudaError_t launch_ring_build_tc(const MacDecodeParams& p, const MacRingBuildParams& a, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(ring_build_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  CUtensorMap mK, mV;
  if (!encode_cache_map(&mK, p.k_cache) || !encode_cache_map(&mV, p.v_cache)) return cudaErrorInvalidValue;
  const int g = p.n_q_heads / p.n_kv_heads;
  const long n_pb = (a.n_rows + 256 / g - 1) / (256 / g);
  const long items = (long)p.batch * p.n_kv_heads * n_pb * a.n_chunks;
  if (items > 0x7fffffffL) return cudaErrorInvalidValue;
  ring_build_tc_kernel<<<(unsigned)items, TC_THREADS, TC_SMEM, st>>>(mK, mV, p, a);
  return cudaGetLastError();
}

}  // namespace mac
