// K2 fast path (the per-item math shared by the amend kernels of amend_mma.cu) —
// bf16 K/V, d = d_v = 128, GQA group g <= 8, tensor cores.
//
// Same contract as amend.cu (engine.py:464-470, 484-493; attention.py:75-116):
// for each work item {grp, c, t0, t1} of the device plan (common.cuh
// plan_group) emit two partial summaries per head of the group — piece
// (t <= m-r) and band (t > m-r) — masking each head below its own lo_h.
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
// Scheduling: one warp per CTA, persistent; warps pull items from the plan
// with an atomic counter (dynamic load balance across heterogeneous spans,
// the paper's K2 balancing).  A warp streams its item in
// 16-token sub-tiles (one KV page for page_size % 16 == 0) with 16-byte
// cp.async into an XOR-swizzled 4-stage ring (conflict-free ldmatrix) and
// consumes them two at a time: a 32-token step keeps 8 independent QK
// accumulator chains and 32 PV MMAs in flight, which is what a warp needs to
// cover tensor-core and shuffle latency at ~7 warps per SM (measured with
// %globaltimer traces: 16-token steps left warps compute-latency bound).
// The piece -> band switch happens in-stream: the piece partial is written
// out and the online-softmax state reset without draining the pipeline.
#pragma once

#include <type_traits>

#include "complete.cuh"

namespace mac {

namespace {
constexpr int TILE_BYTES = 16 * 256;  // 16 tokens x 128 dims x bf16
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
// the same MMA with a zero accumulator (no register zeroing before the first k-step)
__device__ __forceinline__ void mma16816_z(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%10,%10,%10,%10};\n"
      : "=f"(c[0]), "=f"(c[1]), "=f"(c[2]), "=f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "f"(0.f));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo_elem, float hi_elem) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo_elem, hi_elem);  // .x = lo_elem (low 16 bits)
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ void split_bf16(float x, float& hi, float& lo) {
  hi = __bfloat162float(__float2bfloat16_rn(x));
  lo = x - hi;
}
// byte offset of 16-byte chunk `c` (0..15) of row `r` in a swizzled 16 x 256 B tile
__device__ __forceinline__ uint32_t swz(int r, int c) { return (uint32_t)(r * 256 + ((c ^ (r & 7)) << 4)); }
// the same tile as the TMA engine writes it with CU_TENSOR_MAP_SWIZZLE_128B and 64-dim boxes
// (amend_tma.cu): two 16 x 128 B halves (dims 0..63, 64..127), the 16-byte chunk index XORed
// with the row's low 3 bits inside each 128 B row (tile base 1024-byte aligned)
__device__ __forceinline__ uint32_t swz128(int r, int c) {
  return (uint32_t)(((c >> 3) << 11) + (r << 7) + (((c & 7) ^ (r & 7)) << 4));
}
template <bool SW128> __device__ __forceinline__ uint32_t tile_off(int r, int c) {
  return SW128 ? swz128(r, c) : swz(r, c);
}

struct State {
  float o[16][4];
  float M;  // running max (log2 domain), shared by the 4 lanes of a row
  float Z;  // this lane's partial sum
  __device__ __forceinline__ void reset() {
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f;
    M = -CUDART_INF_F;
    Z = 0.f;
  }
};

// fold one 32-token step (two 16-token sub-tiles; this lane: 8 tokens of head `row`)
// into the online-softmax state and accumulate P V.  vs1 == 0: second sub-tile absent.
template <bool HAS1, bool SW128 = false>
__device__ __forceinline__ void softmax_pv(State& S, const float* l_in, const int* tok, int lo, int hi,
                                           uint32_t vs0, uint32_t vs1, int lane) {
  float l[8];
  float mx = -CUDART_INF_F;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    l[e] = (tok[e] >= lo && tok[e] <= hi) ? l_in[e] : -CUDART_INF_F;
    mx = fmaxf(mx, l[e]);
  }
  mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
  mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
  // Lazy rescaling: the reference max M moves only when a logit exceeds it by more than
  // 8 (log2 domain), so exp2(l - M) <= 256 stays exact in fp32 and in the bf16 hi/lo
  // split, and the 64-multiply rescale of O runs only on those rare moves (never on the
  // first tokens: O is still zero).  Z and O always share the same M, so acc = O / Z and
  // lse = M ln2 + ln Z are unchanged.
  const bool bump = mx > S.M + 8.f;
  const float Mn = bump ? mx : S.M;
  float pv[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  float alpha = 1.f;
  if (Mn != -CUDART_INF_F) {
    alpha = bump ? exp2f(S.M - Mn) : 1.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) pv[e] = exp2f(l[e] - Mn);
  }
  const bool rescale = bump && S.M != -CUDART_INF_F;
  S.M = Mn;
  S.Z = S.Z * alpha + (((pv[0] + pv[1]) + (pv[2] + pv[3])) + ((pv[4] + pv[5]) + (pv[6] + pv[7])));
  if (__any_sync(0xffffffffu, rescale)) {
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) {
      S.o[nt][0] *= alpha; S.o[nt][1] *= alpha; S.o[nt][2] *= alpha; S.o[nt][3] *= alpha;
    }
  }
  uint32_t pa[2][4];
#pragma unroll
  for (int kk = 0; kk < 2; ++kk) {
    float h0, lo0, h1, lo1, h2, lo2, h3, lo3;
    split_bf16(pv[4 * kk + 0], h0, lo0); split_bf16(pv[4 * kk + 1], h1, lo1);
    split_bf16(pv[4 * kk + 2], h2, lo2); split_bf16(pv[4 * kk + 3], h3, lo3);
    pa[kk][0] = pack_bf16(h0, h1);
    pa[kk][1] = pack_bf16(lo0, lo1);
    pa[kk][2] = pack_bf16(h2, h3);
    pa[kk][3] = pack_bf16(lo2, lo3);
  }
  const int mi = lane >> 3, ii = lane & 7;
  const int trow = ((mi & 1) << 3) + ii;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    uint32_t b0, b1, b2, b3;
    ldsm_x4_t(vs0 + tile_off<SW128>(trow, 2 * j + (mi >> 1)), b0, b1, b2, b3);
    mma16816(S.o[2 * j], pa[0], b0, b1);
    mma16816(S.o[2 * j + 1], pa[0], b2, b3);
    if (HAS1) {  // compile-time: no predicated ldmatrix (which costs a WARPSYNC + NOP each)
      uint32_t c0, c1, c2, c3;
      ldsm_x4_t(vs1 + tile_off<SW128>(trow, 2 * j + (mi >> 1)), c0, c1, c2, c3);
      mma16816(S.o[2 * j], pa[1], c0, c1);
      mma16816(S.o[2 * j + 1], pa[1], c2, c3);
    }
  }
}

// normalised partial (acc = O / Z, lse) of head `row` -> out[row][set]
__device__ __forceinline__ void write_partial(const State& S, float* out, int set, int row, int q4, int g) {
  float Z = S.Z;
  Z += __shfl_xor_sync(0xffffffffu, Z, 1);
  Z += __shfl_xor_sync(0xffffffffu, Z, 2);
  if (row >= g) return;
  float* o = out + (row * 2 + set) * 129;
  const float inv = Z > 0.f ? 1.f / Z : 0.f;
#pragma unroll
  for (int nt = 0; nt < 16; ++nt) {
    o[nt * 8 + q4 * 2] = (S.o[nt][0] + S.o[nt][2]) * inv;  // rows of 129 floats: scalar stores
    o[nt * 8 + q4 * 2 + 1] = (S.o[nt][1] + S.o[nt][3]) * inv;
  }
  if (q4 == 0) o[128] = Z > 0.f ? S.M * LN2 + logf(Z) : -CUDART_INF_F;
}
}  // namespace

// One work item {grp, c, t0, t1} of the device plan: stream the group's K/V
// rows [t0, t1] and write the piece and band partials of each of its g heads.
// on_issued() runs once the first KV stages are in flight (the caller's
// prefetch of its next work item hides under them).  BAND: a split-band item
// (common.cuh band_items), run before the plan exists — band partial only, no
// per-head lower bound (every head's band is [max(1, m-r+1), m]).
template <int ST, bool BAND, typename OnIssued>
__device__ __forceinline__ void amend_mma_item(const MacDecodeParams& p, int4 it, uint32_t sm, OnIssued on_issued) {
  const int lane = threadIdx.x & 31;
  const int Hkv = p.n_kv_heads, Hq = p.n_q_heads, g = Hq / Hkv, r = p.band, ps = p.page_size;
  const float scale2 = (float)(1.0 / sqrt(128.0)) * LOG2E;
  const int row = lane >> 2, q4 = lane & 3;
  const Workspace w = workspace_layout(p);
  const int* plan_lo = ws_ptr<const int>(p, w.lo_off);
  const int* mpos = ws_ptr<const int>(p, w.mpos_off);
  const float* qrot = ws_ptr<const float>(p, w.qrot_off);
  float* part = ws_ptr<float>(p, w.part_off);
  const __nv_bfloat16* kc = static_cast<const __nv_bfloat16*>(p.k_cache);
  const __nv_bfloat16* vc = static_cast<const __nv_bfloat16*>(p.v_cache);
  const int grp = (int)__reduce_max_sync(0xffffffffu, (unsigned)it.x);
  const int c = (int)__reduce_max_sync(0xffffffffu, (unsigned)it.y);
  const int t0 = (int)__reduce_max_sync(0xffffffffu, (unsigned)it.z);
  const int t1 = (int)__reduce_max_sync(0xffffffffu, (unsigned)it.w);
  const int b = grp / Hkv, kvh = grp % Hkv;
  const int nsub = ((t1 - t0) >> 4) + 1;
  // page rows of the item's sub-tiles, 32 at a time (lane j holds sub-tile 32*blk + j),
  // fetched one block ahead so the cp.async issue never waits on the page table
  auto rows_of = [&](int blk) -> long long {
    const int j = blk * 32 + lane;
    if (j >= nsub) return 0;
    const int local = t0 + (j << 4) - p.kv_offset;
    const int page = p.page_table[(int64_t)b * p.pages_per_seq + min((local - 1) / ps, p.pages_per_seq - 1)];
    return ((long long)page * Hkv + kvh) * ps + ((local - 1) % ps);
  };
  long long rows_cur = rows_of(0), rows_nxt = nsub > 32 ? rows_of(1) : 0;
  int blk_cur = 0;
  // this lane's 16-byte chunk of each of the 8 copy rounds: tile row 2*rr + (lane >> 4),
  // column lane & 15; the XOR swizzle repeats every 4 rounds (rows 8 apart), so four
  // offsets cover all eight (+2048 bytes for rounds 4-7), global offsets are linear
  const int chi = lane >> 4, ccol = lane & 15;
  uint32_t soff[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) soff[i] = swz(2 * i + chi, ccol);
  const int goff = chi * 256 + ccol * 16;
  auto issue = [&](int j, int stage) {
    if ((j >> 5) != blk_cur) {
      blk_cur = j >> 5;
      rows_cur = rows_nxt;
      rows_nxt = rows_of(blk_cur + 1);
    }
    const long long row0 = __shfl_sync(0xffffffffu, rows_cur, j & 31);
    const char* kg = reinterpret_cast<const char*>(kc + row0 * 128);
    const char* vg = reinterpret_cast<const char*>(vc + row0 * 128);
    const uint32_t ks_ = sm + stage * 2 * TILE_BYTES, vs_ = ks_ + TILE_BYTES;
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) {
      const uint32_t so = soff[rr & 3] + (rr >= 4 ? 2048u : 0u);
      cp_async16(ks_ + so, kg + goff + rr * 512);
      cp_async16(vs_ + so, vg + goff + rr * 512);
    }
  };
  // KV streams first; the query fragments and head bounds load underneath
#pragma unroll
  for (int i = 0; i < ST; ++i) {
    if (i < nsub) issue(i, i);
    cp_commit();
  }
  on_issued();
  const int m = (int)__reduce_max_sync(0xffffffffu, (unsigned)__ldcg(mpos + b));
  const int cpos = m - r;
  const int lo_h = row < g ? (BAND ? 1 : __ldcg(plan_lo + b * Hq + kvh * g + row)) : (1 << 30);
  // Q fragments (hi rows 0..7, lo rows 8..15), 8 k-steps
  uint32_t qa[8][4];
  {
    const float* qr = qrot + ((int64_t)b * Hq + kvh * g + (row < g ? row : 0)) * 128;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const int k0 = ks * 16 + q4 * 2;
      float2 x01 = make_float2(0.f, 0.f), x89 = make_float2(0.f, 0.f);
      if (row < g) {
        x01 = __ldcg(reinterpret_cast<const float2*>(qr + k0));
        x89 = __ldcg(reinterpret_cast<const float2*>(qr + k0 + 8));
      }
      float h0, l0, h1, l1, h8, l8, h9, l9;
      split_bf16(x01.x, h0, l0); split_bf16(x01.y, h1, l1);
      split_bf16(x89.x, h8, l8); split_bf16(x89.y, h9, l9);
      qa[ks][0] = pack_bf16(h0, h1);
      qa[ks][1] = pack_bf16(l0, l1);
      qa[ks][2] = pack_bf16(h8, h9);
      qa[ks][3] = pack_bf16(l8, l9);
    }
  }
  float* out = part + ((int64_t)(grp * p.max_chunks + c) * g) * 2 * 129;
  State S;
  S.reset();
  bool in_band = false;
  const int lo_piece = max(lo_h, t0), hi_piece = BAND ? t0 - 1 : min(t1, cpos);
  const int lo_band = max(lo_h, max(t0, cpos + 1));
  // 32-token steps: sub-tiles 2jp and 2jp+1 (stages (2jp) % ST and (2jp+1) % ST)
  // 32-token steps over sub-tile pairs (2jp, 2jp+1); an odd tail sub-tile gets a half step.
  // HAS1 is a template constant so the second sub-tile's ldmatrix is never predicated.
  auto step = [&](int jp, auto has1_tag) {
    constexpr bool HAS1 = decltype(has1_tag)::value;
    const int j0 = 2 * jp;
    cp_wait<ST - 2>();
    __syncwarp();
    const int ts = t0 + (jp << 5);
    const uint32_t ks0 = sm + (j0 % ST) * 2 * TILE_BYTES, vs0 = ks0 + TILE_BYTES;
    const uint32_t ks1 = sm + ((j0 + 1) % ST) * 2 * TILE_BYTES, vs1 = ks1 + TILE_BYTES;
    // S = Q K^T for 4 n-tiles (32 tokens); even/odd k-steps accumulate separately,
    // k-steps 0 and 1 start the two chains with a zero accumulator
    float s[4][2][4];
    {
      const int mi = lane >> 3, ii = lane & 7;
      const int trow = ((mi >> 1) << 3) + ii;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4(ks0 + swz(trow, 2 * ks + (mi & 1)), b0, b1, b2, b3);
        if (ks < 2) {
          mma16816_z(s[0][ks & 1], qa[ks], b0, b1);
          mma16816_z(s[1][ks & 1], qa[ks], b2, b3);
        } else {
          mma16816(s[0][ks & 1], qa[ks], b0, b1);
          mma16816(s[1][ks & 1], qa[ks], b2, b3);
        }
        if (HAS1) {
          uint32_t c0, c1, c2, c3;
          ldsm_x4(ks1 + swz(trow, 2 * ks + (mi & 1)), c0, c1, c2, c3);
          if (ks < 2) {
            mma16816_z(s[2][ks & 1], qa[ks], c0, c1);
            mma16816_z(s[3][ks & 1], qa[ks], c2, c3);
          } else {
            mma16816(s[2][ks & 1], qa[ks], c0, c1);
            mma16816(s[3][ks & 1], qa[ks], c2, c3);
          }
        }
      }
    }
    float l[8];
    int tok[8];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      if (!HAS1 && nt >= 2) {
        l[2 * nt] = l[2 * nt + 1] = -CUDART_INF_F;
      } else {
        l[2 * nt] = ((s[nt][0][0] + s[nt][1][0]) + (s[nt][0][2] + s[nt][1][2])) * scale2;
        l[2 * nt + 1] = ((s[nt][0][1] + s[nt][1][1]) + (s[nt][0][3] + s[nt][1][3])) * scale2;
      }
      tok[2 * nt] = ts + nt * 8 + q4 * 2;
      tok[2 * nt + 1] = ts + nt * 8 + q4 * 2 + 1;
    }
    const int hi_band = HAS1 ? t1 : min(t1, ts + 15);
    // (the step's branches are warp-uniform; saying so through a vote lets ptxas drop the
    // WARPSYNC it otherwise puts before every ldmatrix under them)
    if (__any_sync(0xffffffffu, ts <= hi_piece))
      softmax_pv<HAS1>(S, l, tok, lo_piece, HAS1 ? hi_piece : min(hi_piece, ts + 15), vs0, vs1, lane);
    if (__any_sync(0xffffffffu, ts + 31 > cpos && max(ts, cpos + 1) <= t1)) {
      if (!in_band) {
        write_partial(S, out, 0, row, q4, g);
        S.reset();
        in_band = true;
      }
      softmax_pv<HAS1>(S, l, tok, lo_band, hi_band, vs0, vs1, lane);
    }
    __syncwarp();
    if (j0 + ST < nsub) issue(j0 + ST, j0 % ST);
    cp_commit();
    if (j0 + 1 + ST < nsub) issue(j0 + 1 + ST, (j0 + 1) % ST);
    cp_commit();
  };
  const int npair = nsub >> 1;
  for (int jp = 0; jp < npair; ++jp) step(jp, std::true_type{});
  if (nsub & 1) step(npair, std::false_type{});
  cp_wait<0>();
  if (!in_band) {
    write_partial(S, out, 0, row, q4, g);
    S.reset();
  }
  write_partial(S, out, 1, row, q4, g);
}

}  // namespace mac
