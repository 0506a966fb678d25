// Prefill ring construction in GEMM form — bf16 K/V, d = d_v = 128,
// GQA group g dividing 8, tensor cores.
//
// After a prompt's K/V is in the paged cache, the ring must hold, for each of the last
// positions t, the pre-RoPE query q_t and the prefix summary AS[1, t - r] under R_t q_t —
// exactly what t forced-miss decode steps leave (rectify_append, engine.py:374-402, with the
// miss path's prefix, engine.py:484-499).  Those are n_rows causal attention rows with a lag
// of r, all over the same keys: a real (rows x keys) contraction, so instead of n_rows decode
// steps (each streaming the whole cache) one pass streams every key tile ONCE per block of
// query rows and feeds it to all of them through shared memory — the chunked-GEMM form of
// oracle_outputs (engine.py:542-572).
//
// Work item = (request b, kv head, block of NW * 8/g positions, key chunk).  A CTA of NW warps
// streams the chunk's K/V in 32-token stages (two 16-token page sub-tiles) with cp.async into
// a 4-stage XOR-swizzled ring shared by all warps; each warp owns 8 query rows (8/g positions
// x g heads) and runs the decode amend's per-warp math on every stage (amend_mma.cuh: Q split
// hi/lo into rows h and 8+h of the m16n8k16 A tile, fp32 logits, log2-domain online softmax,
// P split hi/lo for P V), masking each row to keys <= t - r.  A single chunk writes the ring
// slot directly; several chunks write f32 partials merged by ring_merge_kernel.  The query
// rows are rotated in-kernel with fp64 angles, like the append (front.cuh).
#include "amend_mma.cuh"

namespace mac {

namespace {
constexpr int RB_NW = 8;                        // warps per CTA
constexpr int RB_ST = 4;                        // 32-token stages in the ring
constexpr int RB_STAGE = 4 * TILE_BYTES;        // K0, V0, K1, V1 sub-tiles (16 KiB)
constexpr int RB_SMEM = RB_ST * RB_STAGE;       // 64 KiB

__device__ __forceinline__ void cp_async16_zfill(uint32_t s, const void* g, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(g), "r"(valid ? 16 : 0));
}
}  // namespace

__global__ void __launch_bounds__(RB_NW * 32, 1) ring_build_kernel(MacDecodeParams p, MacRingBuildParams a) {
  extern __shared__ __align__(128) unsigned char smem[];
  const uint32_t sm = smem_u32(smem);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int Hkv = p.n_kv_heads, Hq = p.n_q_heads, g = Hq / Hkv, r = p.band, ps = p.page_size, W = p.window;
  const int qpw = 8 / g;                 // positions per warp
  const int pb_rows = RB_NW * qpw;       // positions per CTA
  const int n_pb = (a.n_rows + pb_rows - 1) / pb_rows;
  int item = blockIdx.x;
  const int ch = item % a.n_chunks;
  item /= a.n_chunks;
  const int pb = item % n_pb;
  item /= n_pb;
  const int kvh = item % Hkv, b = item / Hkv;
  const int n = p.seq_lens[b];           // tokens stored; rows are positions n - n_rows + 1 .. n
  const int first = n - a.n_rows + 1;
  const int i0 = pb * pb_rows;                          // first row index of the block
  const int i_last = min(a.n_rows, i0 + pb_rows) - 1;
  const int kmax = first + i_last - r;                  // keys any row of the block reads: [1, kmax]
  // this chunk's keys: 32-token aligned split of [1, kmax]
  const int span32 = kmax >= 1 ? (kmax + 31) / 32 : 0;
  const int per = (span32 + a.n_chunks - 1) / a.n_chunks;
  const int k0 = 1 + ch * per * 32, k1 = min(kmax, (ch + 1) * per * 32);
  const int nst = k1 >= k0 ? (k1 - k0) / 32 + 1 : 0;

  // this lane's query row: rho = lane >> 2 -> (position pi, head hl)
  const int row = lane >> 2, q4 = lane & 3;
  const int pi = row / g, hl = row % g;
  const int ri = i0 + warp * qpw + pi;                  // row index in [0, n_rows)
  const bool rvalid = ri < a.n_rows;
  const int t = first + ri;                              // its position
  const int head = kvh * g + hl;
  const int hi_row = rvalid ? t - r : 0;                 // keys <= t - r
  const __nv_bfloat16* kc = static_cast<const __nv_bfloat16*>(p.k_cache);
  const __nv_bfloat16* vc = static_cast<const __nv_bfloat16*>(p.v_cache);

  // CTA-wide stage copy: 1024 16-byte chunks (K0, V0, K1, V1 x 16 rows x 16 chunks), 4 per thread
  auto issue = [&](int s, int buf) {
    const uint32_t base = sm + buf * RB_STAGE;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int q = tid + u * RB_NW * 32;       // 0..1023
      const int tile = q >> 8, rr = (q >> 4) & 15, cc = q & 15;
      const int sub = tile >> 1;                // sub-tile 0 / 1
      const int tok = k0 + s * 32 + sub * 16;   // first token of the sub-tile (16-aligned, 1-based)
      const bool ok = tok <= k1;
      const int pg = p.page_table[(int64_t)b * p.pages_per_seq + min((max(tok, 1) - 1) / ps, p.pages_per_seq - 1)];
      const int64_t grow = ((int64_t)pg * Hkv + kvh) * ps + ((max(tok, 1) - 1) % ps) + rr;
      const __nv_bfloat16* src = (tile & 1) ? vc : kc;
      const uint32_t dst = base + tile * TILE_BYTES + swz(rr, cc);
      cp_async16_zfill(dst, src + grow * 128 + cc * 8, ok);
    }
  };
#pragma unroll
  for (int s = 0; s < RB_ST - 1; ++s) {
    if (s < nst) issue(s, s);
    cp_commit();
  }

  // Q fragments of this lane's row (rotated at t, fp64 angles), hi rows 0..7, lo rows 8..15
  uint32_t qa[8][4];
  {
    const int64_t qb = ((int64_t)(b * a.n_rows + (rvalid ? ri : 0)) * Hq + head) * 128;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      float v4[4];
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {  // pairs j = ks*8 + q4 and ks*8 + q4 + 4 (dims k0, k0+8)
        const int j = ks * 8 + q4 + 4 * hh;
        float e0 = 0.f, e1 = 0.f;
        if (rvalid) {
          double sn, cs;
          sincos((double)t * p.rope_freqs[j], &sn, &cs);
          const double x0 = load_in(p.q_pre, qb + 2 * j, p.in_dtype), x1 = load_in(p.q_pre, qb + 2 * j + 1, p.in_dtype);
          e0 = (float)(x0 * cs - x1 * sn);
          e1 = (float)(x0 * sn + x1 * cs);
        }
        v4[2 * hh] = e0;
        v4[2 * hh + 1] = e1;
      }
      float h0, l0, h1, l1, h8, l8, h9, l9;
      split_bf16(v4[0], h0, l0); split_bf16(v4[1], h1, l1);
      split_bf16(v4[2], h8, l8); split_bf16(v4[3], h9, l9);
      qa[ks][0] = pack_bf16(h0, h1);
      qa[ks][1] = pack_bf16(l0, l1);
      qa[ks][2] = pack_bf16(h8, h9);
      qa[ks][3] = pack_bf16(l8, l9);
    }
  }
  const float scale2 = (float)(1.0 / sqrt(128.0)) * LOG2E;
  State S;
  S.reset();
  const int hi_mask = min(hi_row, k1);
  for (int s = 0; s < nst; ++s) {
    cp_wait<RB_ST - 2>();
    __syncthreads();  // stage s landed for every thread; stage s-1's buffer is free
    if (s + RB_ST - 1 < nst) issue(s + RB_ST - 1, (s + RB_ST - 1) % RB_ST);
    cp_commit();
    const uint32_t base = sm + (s % RB_ST) * RB_STAGE;
    const uint32_t ks0 = base, vs0 = base + TILE_BYTES, ks1 = base + 2 * TILE_BYTES, vs1 = base + 3 * TILE_BYTES;
    const int ts = k0 + s * 32;
    if (!__any_sync(0xffffffffu, ts <= hi_mask)) continue;  // no row of this warp reads the stage
    float sc[4][2][4];
    {
      const int mi = lane >> 3, ii = lane & 7;
      const int trow = ((mi >> 1) << 3) + ii;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        uint32_t b0, b1, b2, b3, c0, c1, c2, c3;
        ldsm_x4(ks0 + swz(trow, 2 * ks + (mi & 1)), b0, b1, b2, b3);
        ldsm_x4(ks1 + swz(trow, 2 * ks + (mi & 1)), c0, c1, c2, c3);
        if (ks < 2) {
          mma16816_z(sc[0][ks & 1], qa[ks], b0, b1);
          mma16816_z(sc[1][ks & 1], qa[ks], b2, b3);
          mma16816_z(sc[2][ks & 1], qa[ks], c0, c1);
          mma16816_z(sc[3][ks & 1], qa[ks], c2, c3);
        } else {
          mma16816(sc[0][ks & 1], qa[ks], b0, b1);
          mma16816(sc[1][ks & 1], qa[ks], b2, b3);
          mma16816(sc[2][ks & 1], qa[ks], c0, c1);
          mma16816(sc[3][ks & 1], qa[ks], c2, c3);
        }
      }
    }
    float l[8];
    int tok[8];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      l[2 * nt] = ((sc[nt][0][0] + sc[nt][1][0]) + (sc[nt][0][2] + sc[nt][1][2])) * scale2;
      l[2 * nt + 1] = ((sc[nt][0][1] + sc[nt][1][1]) + (sc[nt][0][3] + sc[nt][1][3])) * scale2;
      tok[2 * nt] = ts + nt * 8 + q4 * 2;
      tok[2 * nt + 1] = ts + nt * 8 + q4 * 2 + 1;
    }
    softmax_pv<true>(S, l, tok, 1, hi_mask, vs0, vs1, lane);
  }
  cp_wait<0>();

  // epilogue: this row's normalised (acc, lse) -> ring slot (one chunk) or the chunk partial
  float Z = S.Z;
  Z += __shfl_xor_sync(0xffffffffu, Z, 1);
  Z += __shfl_xor_sync(0xffffffffu, Z, 2);
  if (!rvalid) return;
  const float inv = Z > 0.f ? 1.f / Z : 0.f;
  const float lse = Z > 0.f ? S.M * LN2 + logf(Z) : -CUDART_INF_F;
  const int slot = (t - 1) % W;
  float* dst;
  if (a.n_chunks == 1) {
    dst = static_cast<float*>(p.ring_acc) + (((int64_t)b * Hq + head) * W + slot) * 128;
    if (q4 == 0) static_cast<float*>(p.ring_lse)[((int64_t)b * Hq + head) * W + slot] = lse;
  } else {
    dst = static_cast<float*>(a.part) + ((((int64_t)b * a.n_rows + ri) * Hq + head) * a.n_chunks + ch) * 129;
    if (q4 == 0) dst[128] = lse;
  }
#pragma unroll
  for (int nt = 0; nt < 16; ++nt) {
    const float2 v = make_float2((S.o[nt][0] + S.o[nt][2]) * inv, (S.o[nt][1] + S.o[nt][3]) * inv);
    if (a.n_chunks == 1) *reinterpret_cast<float2*>(dst + nt * 8 + q4 * 2) = v;
    else { dst[nt * 8 + q4 * 2] = v.x; dst[nt * 8 + q4 * 2 + 1] = v.y; }
  }
  // the ring's query row (pre-RoPE, stored as bf16 exactly like the decode step's write-back)
  if (ch == 0) {
    const int64_t qb = ((int64_t)(b * a.n_rows + ri) * Hq + head) * 128;
    __nv_bfloat16* rq = static_cast<__nv_bfloat16*>(p.ring_q) + (((int64_t)b * Hq + head) * W + slot) * 128;
    for (int e = q4; e < 128; e += 4) rq[e] = from_f64<__nv_bfloat16>(load_in(p.q_pre, qb + e, p.in_dtype));
    if (p.ring_qp) {
      __nv_bfloat16* rp =
          static_cast<__nv_bfloat16*>(p.ring_qp) + (((int64_t)b * Hq + head) * W + slot) * MAC_PLANAR_DIMS;
      for (int e = q4; e < MAC_PLANAR_DIMS; e += 4) rp[e] = from_f64<__nv_bfloat16>(load_in(p.q_pre, qb + e, p.in_dtype));
    }
  }
}

// chunk partials of one (request, row, head) -> its ring slot (log-domain merge in f32)
__global__ void ring_merge_kernel(MacDecodeParams p, MacRingBuildParams a) {
  const int idx = blockIdx.x;  // (b * n_rows + ri) * Hq + head
  const int Hq = p.n_q_heads, W = p.window;
  const int head = idx % Hq, bri = idx / Hq, ri = bri % a.n_rows, b = bri / a.n_rows;
  const int t = p.seq_lens[b] - a.n_rows + 1 + ri;
  const float* part = static_cast<const float*>(a.part) + (int64_t)idx * a.n_chunks * 129;
  float M = -CUDART_INF_F;
  for (int c = 0; c < a.n_chunks; ++c) M = fmaxf(M, part[c * 129 + 128]);
  float Z = 0.f;
  if (M != -CUDART_INF_F)
    for (int c = 0; c < a.n_chunks; ++c) {
      const float l = part[c * 129 + 128];
      if (l != -CUDART_INF_F) Z += __expf(l - M);
    }
  const float L = Z > 0.f ? M + __logf(Z) : -CUDART_INF_F;
  const int slot = (t - 1) % W;
  float* acc = static_cast<float*>(p.ring_acc) + (((int64_t)b * Hq + head) * W + slot) * 128;
  for (int e = threadIdx.x; e < 128; e += blockDim.x) {
    float v = 0.f;
    if (L != -CUDART_INF_F)
      for (int c = 0; c < a.n_chunks; ++c) {
        const float l = part[c * 129 + 128];
        if (l != -CUDART_INF_F) v += part[c * 129 + e] * __expf(l - L);
      }
    acc[e] = v;
  }
  if (threadIdx.x == 0) static_cast<float*>(p.ring_lse)[((int64_t)b * Hq + head) * W + slot] = L;
}

bool ring_build_supported(const MacDecodeParams& p) {
  const int g = p.n_q_heads / p.n_kv_heads;
  return p.storage == MAC_MODE_BF16 && p.head_dim == 128 && p.head_dim_v == 128 && g >= 1 && 8 % g == 0 &&
         p.page_size % 16 == 0 && p.kv_offset == 0 && p.kv_limit == 0;
}

bool ring_build_tc_supported(const MacDecodeParams& p);
cudaError_t launch_ring_build_tc(const MacDecodeParams& p, const MacRingBuildParams& a, cudaStream_t st);

// the tcgen05 kernel (ring_build_tc.cu) where it applies, else this file's mma.sync kernel;
// use_tc < 0: by support, 0 / 1: forced (tests compare the two)
cudaError_t launch_ring_build(const MacDecodeParams& p, const MacRingBuildParams& a, cudaStream_t st, int use_tc) {
  const bool tc = use_tc < 0 ? ring_build_tc_supported(p) : (use_tc > 0 && ring_build_tc_supported(p));
  if (tc) {
    cudaError_t e = launch_ring_build_tc(p, a, st);
    if (e != cudaSuccess || a.n_chunks == 1) return e;
    ring_merge_kernel<<<p.batch * a.n_rows * p.n_q_heads, 128, 0, st>>>(p, a);
    return cudaGetLastError();
  }
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(ring_build_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, RB_SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int g = p.n_q_heads / p.n_kv_heads;
  const int pb_rows = RB_NW * (8 / g);
  const long n_pb = (a.n_rows + pb_rows - 1) / pb_rows;
  const long items = (long)p.batch * p.n_kv_heads * n_pb * a.n_chunks;
  if (items > 0x7fffffffL) return cudaErrorInvalidValue;
  ring_build_kernel<<<(unsigned)items, RB_NW * 32, RB_SMEM, st>>>(p, a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || a.n_chunks == 1) return e;
  ring_merge_kernel<<<p.batch * a.n_rows * p.n_q_heads, 128, 0, st>>>(p, a);
  return cudaGetLastError();
}

}  // namespace mac
