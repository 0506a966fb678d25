// K2 fast path — bf16 K/V, d = d_v = 128, GQA group g <= 8, tensor cores.
//
// Same contract as amend.cu (engine.py:464-470, 484-493; attention.py:75-116):
// for each (request, kv head, split) item, two partial summaries per head —
// piece (t <= m-r) and band (t > m-r) — over the group's span, masking each
// head below its own lo_h.
//
// Mapping onto mma.sync.m16n8k16 (bf16 in, fp32 accumulate):
//   S = Q K^T   A = Q as 16 rows: row h = hi(q_h), row 8+h = lo(q_h) with
//               q = hi + lo both bf16 (q_rot is fp32; the split keeps ~16
//               mantissa bits, so logits carry no bf16 query rounding); B = K^T
//               straight from the K tile (ldmatrix, non-transposed).  The
//               thread owning row h also owns row 8+h, so logit = c0 + c2.
//   O += P V    A = P from the same accumulator registers (flash-attention-2
//               register reuse), again split hi/lo into rows h and 8+h;
//               B = V via ldmatrix.trans.  O[h] = row h + row 8+h at the end.
// The g <= 8 real rows of the 16-row tile are exactly the hi/lo pairs, so the
// precision trick costs no extra MMAs.
//
// Each warp owns whole 16-token sub-tiles (one KV page for page_size % 16 == 0),
// streams K and V with 16-byte cp.async into an XOR-swizzled 3-stage ring
// (conflict-free ldmatrix), and keeps its own online-softmax state; the 4
// warps merge through shared memory once per (item, set).  The grid is
// persistent over split-major items (see amend.cu).
#include "common.cuh"

namespace mac {

namespace {
constexpr int NW = 4;                 // warps per CTA
constexpr int ST = 3;                 // cp.async stages per warp
constexpr int TILE_BYTES = 16 * 256;  // 16 tokens x 128 dims x bf16
constexpr int WARP_SMEM = ST * 2 * TILE_BYTES;
constexpr int SMEM = NW * WARP_SMEM;  // 96 KiB
constexpr float LOG2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(uint32_t s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(g));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N> __device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo_elem, float hi_elem) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo_elem, hi_elem);  // .x = lo_elem (low 16 bits)
  return *reinterpret_cast<uint32_t*>(&v);
}
// split x = hi + lo, both bf16
__device__ __forceinline__ void split_bf16(float x, float& hi, float& lo) {
  hi = __bfloat162float(__float2bfloat16_rn(x));
  lo = x - hi;
}
// byte offset of 16-byte chunk `c` (0..15) of row `r` in a swizzled 16 x 256 B tile
__device__ __forceinline__ uint32_t swz(int r, int c) { return (uint32_t)(r * 256 + ((c ^ (r & 7)) << 4)); }

struct SetState {
  float o[16][4];
  float M;  // running max (log2 domain), same for the 4 threads of a row
  float Z;  // this thread's partial sum
};
}  // namespace

bool amend_mma_supported(const MacDecodeParams& p) {
  const int g = p.n_q_heads / p.n_kv_heads;
  return p.storage == MAC_MODE_BF16 && p.head_dim == 128 && p.head_dim_v == 128 && g >= 1 && g <= 8 &&
         p.page_size % 16 == 0;
}

__global__ void __launch_bounds__(NW * 32, 2) amend_mma_kernel(MacDecodeParams p, const int32_t* __restrict__ mpos,
                                                              const float* __restrict__ qrot, float* __restrict__ part) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int Hkv = p.n_kv_heads, Hq = p.n_q_heads, g = Hq / Hkv, r = p.band, ps = p.page_size;
  const int G = p.batch * Hkv;
  const long total = (long)G * p.max_chunks;
  const float scale2 = (float)(1.0 / sqrt(128.0)) * LOG2E;
  const int row = lane >> 2;        // head owned by this thread (rows row and row + 8)
  const int q4 = lane & 3;
  unsigned char* wsm = smem + warp * WARP_SMEM;
  const uint32_t wsm_u = smem_u32(wsm);
  const __nv_bfloat16* kc = static_cast<const __nv_bfloat16*>(p.k_cache);
  const __nv_bfloat16* vc = static_cast<const __nv_bfloat16*>(p.v_cache);
  float* mrg = reinterpret_cast<float*>(smem);  // [NW][g][130] merge buffer, aliases the tiles

  for (long vi = blockIdx.x; vi < total; vi += gridDim.x) {
    const int c = (int)(vi / G), grp = (int)(vi % G);
    const int b = grp / Hkv, kvh = grp % Hkv;
    const int m = mpos[b];
    int lo_g = m;
    for (int j = 0; j < g; ++j) {
      int bh = b * Hq + kvh * g + j;
      int u = p.force_miss ? 0 : p.use_hit[bh];
      int lo = head_lo(u, u ? p.match_pos[bh] : 0, r);
      lo_g = lo < lo_g ? lo : lo_g;
    }
    const int start = grid_start(lo_g, p.kv_offset);
    const Chunking ch = chunking(m - start + 1, p.max_chunks, p.min_chunk);
    if (c >= ch.n) continue;
    const int t0 = start + c * ch.len;
    const int t1 = min(m, t0 + ch.len - 1);
    const int cpos = m - r;

    // per-thread head geometry
    int lo_h = 1 << 30;
    if (row < g) {
      int bh = b * Hq + kvh * g + row;
      int u = p.force_miss ? 0 : p.use_hit[bh];
      lo_h = head_lo(u, u ? p.match_pos[bh] : 0, r);
    }
    // Q fragments (hi rows 0..7, lo rows 8..15), 8 k-steps
    uint32_t qa[8][4];
    {
      const float* qr = qrot + ((int64_t)b * Hq + kvh * g + (row < g ? row : 0)) * 128;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const int k0 = ks * 16 + q4 * 2;
        float x0 = 0.f, x1 = 0.f, x8 = 0.f, x9 = 0.f;
        if (row < g) { x0 = qr[k0]; x1 = qr[k0 + 1]; x8 = qr[k0 + 8]; x9 = qr[k0 + 9]; }
        float h0, l0, h1, l1, h8, l8, h9, l9;
        split_bf16(x0, h0, l0); split_bf16(x1, h1, l1); split_bf16(x8, h8, l8); split_bf16(x9, h9, l9);
        qa[ks][0] = pack_bf16(h0, h1);
        qa[ks][1] = pack_bf16(l0, l1);
        qa[ks][2] = pack_bf16(h8, h9);
        qa[ks][3] = pack_bf16(l8, l9);
      }
    }

    for (int set = 0; set < 2; ++set) {
      const int ra = set == 0 ? t0 : max(t0, cpos + 1);
      const int rb = set == 0 ? min(t1, cpos) : t1;
      SetState S;
#pragma unroll
      for (int nt = 0; nt < 16; ++nt) S.o[nt][0] = S.o[nt][1] = S.o[nt][2] = S.o[nt][3] = 0.f;
      S.M = -CUDART_INF_F;
      S.Z = 0.f;
      const int lo_thr = max(lo_h, ra);
      if (ra <= rb) {
        const int ja = (ra - t0) >> 4, jb = (rb - t0) >> 4;
        const int n_my = (jb - ja - warp) >= 0 ? (jb - ja - warp) / NW + 1 : 0;
        auto issue = [&](int i, int stage) {
          const int ts = t0 + ((ja + warp + i * NW) << 4);
          const int local = ts - p.kv_offset;
          const int page = p.page_table[(int64_t)b * p.pages_per_seq + (local - 1) / ps];
          const int64_t row0 = ((int64_t)page * Hkv + kvh) * ps + ((local - 1) % ps);
          const char* kg = reinterpret_cast<const char*>(kc + row0 * 128);
          const char* vg = reinterpret_cast<const char*>(vc + row0 * 128);
          const uint32_t ks_ = wsm_u + stage * 2 * TILE_BYTES, vs_ = ks_ + TILE_BYTES;
#pragma unroll
          for (int rr = 0; rr < 8; ++rr) {
            const int ci = lane + 32 * rr, trow = ci >> 4, col = ci & 15;
            cp_async16(ks_ + swz(trow, col), kg + trow * 256 + col * 16);
            cp_async16(vs_ + swz(trow, col), vg + trow * 256 + col * 16);
          }
        };
#pragma unroll
        for (int i = 0; i < ST; ++i) {
          if (i < n_my) issue(i, i);
          cp_commit();
        }
        for (int i = 0; i < n_my; ++i) {
          const int stage = i % ST;
          cp_wait<ST - 1>();
          __syncwarp();
          const int ts = t0 + ((ja + warp + i * NW) << 4);
          const uint32_t ks_ = wsm_u + stage * 2 * TILE_BYTES, vs_ = ks_ + TILE_BYTES;
          // ---- S = Q K^T over 16 tokens (2 n-tiles) ----
          float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
          {
            const int mi = lane >> 3, ii = lane & 7;
            const int trow = ((mi >> 1) << 3) + ii;  // n-tile (mi>>1), token ii
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
              uint32_t b0, b1, b2, b3;
              ldsm_x4(ks_ + swz(trow, 2 * ks + (mi & 1)), b0, b1, b2, b3);
              mma16816(s0, qa[ks], b0, b1);
              mma16816(s1, qa[ks], b2, b3);
            }
          }
          // ---- online softmax (log2 domain) for head `row` over this thread's 4 tokens ----
          float l[4] = {(s0[0] + s0[2]) * scale2, (s0[1] + s0[3]) * scale2, (s1[0] + s1[2]) * scale2,
                        (s1[1] + s1[3]) * scale2};
          const int tok[4] = {ts + q4 * 2, ts + q4 * 2 + 1, ts + 8 + q4 * 2, ts + 9 + q4 * 2};
          float mx = -CUDART_INF_F;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const bool ok = tok[e] >= lo_thr && tok[e] <= rb;
            l[e] = ok ? l[e] : -CUDART_INF_F;
            mx = fmaxf(mx, l[e]);
          }
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
          const float Mn = fmaxf(S.M, mx);
          float pv[4];
          float alpha = 1.f;
          if (Mn == -CUDART_INF_F) {
            pv[0] = pv[1] = pv[2] = pv[3] = 0.f;
          } else {
            alpha = exp2f(S.M - Mn);  // S.M = -inf -> 0
#pragma unroll
            for (int e = 0; e < 4; ++e) pv[e] = exp2f(l[e] - Mn);
          }
          S.M = Mn;
          S.Z = S.Z * alpha + (pv[0] + pv[1] + pv[2] + pv[3]);
#pragma unroll
          for (int nt = 0; nt < 16; ++nt) {
            S.o[nt][0] *= alpha; S.o[nt][1] *= alpha; S.o[nt][2] *= alpha; S.o[nt][3] *= alpha;
          }
          float h0, lo0, h1, lo1, h2, lo2, h3, lo3;
          split_bf16(pv[0], h0, lo0); split_bf16(pv[1], h1, lo1);
          split_bf16(pv[2], h2, lo2); split_bf16(pv[3], h3, lo3);
          const uint32_t pa[4] = {pack_bf16(h0, h1), pack_bf16(lo0, lo1), pack_bf16(h2, h3), pack_bf16(lo2, lo3)};
          // ---- O += P V ----
          {
            const int mi = lane >> 3, ii = lane & 7;
            const int trow = ((mi & 1) << 3) + ii;  // token row
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              uint32_t b0, b1, b2, b3;
              ldsm_x4_t(vs_ + swz(trow, 2 * j + (mi >> 1)), b0, b1, b2, b3);
              mma16816(S.o[2 * j], pa, b0, b1);
              mma16816(S.o[2 * j + 1], pa, b2, b3);
            }
          }
          __syncwarp();
          if (i + ST < n_my) issue(i + ST, stage);
          cp_commit();
        }
        cp_wait<0>();
      }
      // ---- merge the 4 warps' states through shared memory ----
      float Zr = S.Z;
      Zr += __shfl_xor_sync(0xffffffffu, Zr, 1);
      Zr += __shfl_xor_sync(0xffffffffu, Zr, 2);
      __syncthreads();  // every warp done with its tiles: the merge buffer may alias them
      if (row < g) {
        float* wb = mrg + (warp * g + row) * 130;
#pragma unroll
        for (int nt = 0; nt < 16; ++nt) {
          wb[nt * 8 + q4 * 2] = S.o[nt][0] + S.o[nt][2];
          wb[nt * 8 + q4 * 2 + 1] = S.o[nt][1] + S.o[nt][3];
        }
        if (q4 == 0) { wb[128] = S.M; wb[129] = Zr; }
      }
      __syncthreads();
      float* out = part + ((int64_t)(grp * p.max_chunks + c) * g) * 2 * 129;
      for (int i = tid; i < g * 129; i += NW * 32) {
        const int h = i / 129, e = i % 129;
        float Ms = -CUDART_INF_F;
#pragma unroll
        for (int w = 0; w < NW; ++w) Ms = fmaxf(Ms, mrg[(w * g + h) * 130 + 128]);
        float Zs = 0.f, acc = 0.f;
        if (Ms != -CUDART_INF_F) {
#pragma unroll
          for (int w = 0; w < NW; ++w) {
            const float* wb = mrg + (w * g + h) * 130;
            const float f = wb[128] == -CUDART_INF_F ? 0.f : exp2f(wb[128] - Ms);
            Zs += wb[129] * f;
            if (e < 128) acc += wb[e] * f;
          }
        }
        float val;
        if (e < 128) val = Zs > 0.f ? acc / Zs : 0.f;
        else val = Zs > 0.f ? Ms * LN2 + logf(Zs) : -CUDART_INF_F;
        out[(h * 2 + set) * 129 + e] = val;
      }
      __syncthreads();  // merge buffer consumed before the next set's tiles land
    }
  }
}

cudaError_t launch_amend_mma_bf16(const MacDecodeParams& p, cudaStream_t st) {
  static int blocks_per_sm = 0, sms = 0;
  if (!blocks_per_sm) {
    cudaError_t e = cudaFuncSetAttribute(amend_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, amend_mma_kernel, NW * 32, SMEM);
    if (blocks_per_sm < 1) blocks_per_sm = 1;
  }
  Workspace w = workspace_layout(p);
  char* ws = static_cast<char*>(p.workspace);
  const long total = (long)p.batch * p.n_kv_heads * p.max_chunks;
  long grid = (long)sms * blocks_per_sm;
  if (grid > total) grid = total;
  amend_mma_kernel<<<(int)grid, NW * 32, SMEM, st>>>(p, reinterpret_cast<const int32_t*>(ws + w.mpos_off),
                                                     reinterpret_cast<const float*>(ws + w.qrot_off),
                                                     reinterpret_cast<float*>(ws + w.part_off));
  return cudaGetLastError();
}

}  // namespace mac
