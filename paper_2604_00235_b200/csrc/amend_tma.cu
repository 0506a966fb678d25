// K2 on the Blackwell copy engine: the bf16 d = 128 amend of the decode step's hit path, fed
// by TMA tensor loads (cp.async.bulk.tensor, SASS UTMALDG) through an mbarrier ring.
//
// Same contract and per-token math as amend_mma.cuh (engine.py:464-470, 484-493;
// attention.py:75-116): for each work item {grp, c, t0, t1} of the device plan
// (common.cuh plan_group / band_items) emit the piece (t <= m-r) and band (t > m-r)
// partial summaries of each of the group's g heads, masking each head below its own lo_h.
//
// What changes is who moves the bytes and how many warps share an item:
//   * one producer warp per CTA claims items and streams their K/V pages into a ring of
//     TA_NS 32-token stages (16 KiB: two 16-token K sub-tiles, two V sub-tiles) with 2D
//     tensor-map loads — 64-dim boxes of 16 rows, SWIZZLE_128B so the consumers' ldmatrix
//     is conflict-free (swz128 in amend_mma.cuh), L2 evict-first (the KV stream is read once
//     and must not push the split partials the complete kernel reads out of L2);
//   * TA_NC consumer warps split every item's stages round-robin, each with its own
//     online-softmax state, and merge their (piece, band) partials through shared memory at
//     the end of the item.  A 600-token item streams ~TA_NC times faster than on one warp,
//     which is what shortens the amend's tail (round 1: one warp per item, items finishing
//     over a 10 us spread) — and the bytes in flight per SM are the ring's, not the
//     registers'.
// The producer runs ahead across item boundaries (descriptor slots TA_ND deep), so the ring
// stays full while the consumers merge.
//
// Split band (common.cuh band_items): the producer first streams the CTA's static band items,
// which need only what the front kernel wrote, then waits on the grid dependency (the verify
// kernel's plan) and claims piece items from the device work list one at a time.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdio.h>
#include <stdlib.h>

#include "amend_mma.cuh"

namespace mac {

namespace {
constexpr int TA_STAGE = 4 * TILE_BYTES;      // K sub-tiles 0, 1 then V sub-tiles 0, 1
constexpr int TA_ND = 4;                      // item descriptor slots
constexpr int TA_PART = 8 * 2 * 129;          // one consumer's partials: [head][set][acc..., lse]
// Ring geometry per variant: NC consumer warps, NS 32-token stages.  NS must be a multiple of NC:
// consumers take an item's stages round-robin, so a stage slot is then always refilled for the
// consumer that drained it, which is what keeps every waiter within one phase of the slot's
// full barrier (a parity wait cannot tell phase L from L-2: with NS = 5, NC = 3 a consumer could
// pass the wait for lap L while lap L-1's TMA was still landing — the intermittent hang/fault
// measured in round 2).
template <int NC, int NS> struct TmaRing {
  static_assert(NS % NC == 0, "NS must be a multiple of NC");
  static constexpr int THREADS = 32 * (NC + 1);  // + one producer warp
  static constexpr int OFF_SCRATCH = NS * TA_STAGE;
  static constexpr int OFF_DESC = OFF_SCRATCH + NC * TA_PART * 4;
  static constexpr int OFF_BAR = OFF_DESC + TA_ND * 32;
  static constexpr int SMEM = OFF_BAR + 8 * (2 * NS + 2 * TA_ND) + 1024;  // + 1024-byte alignment
};

__device__ __forceinline__ void mbar_init(uint32_t a, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, unsigned tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar), "l"(policy)
      : "memory");
}
template <int NC> __device__ __forceinline__ void consumers_sync() {  // the NC consumer warps (named barrier 1)
  asm volatile("bar.sync 1, %0;" ::"n"(NC * 32) : "memory");
}
}  // namespace

template <int TA_NC, int TA_NS, int MINB>
__global__ void __launch_bounds__(TmaRing<TA_NC, TA_NS>::THREADS, MINB)
    amend_tma_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                     MacDecodeParams p, int nb) {
  using R = TmaRing<TA_NC, TA_NS>;
  constexpr int OFF_SCRATCH = R::OFF_SCRATCH, OFF_DESC = R::OFF_DESC, OFF_BAR = R::OFF_BAR;
  extern __shared__ unsigned char smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  unsigned char* smem = smem_raw + (base - raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t bar_full = base + OFF_BAR, bar_empty = bar_full + 8 * TA_NS;
  const uint32_t bar_dfull = bar_empty + 8 * TA_NS, bar_dempty = bar_dfull + 8 * TA_ND;
  int4* desc = reinterpret_cast<int4*>(smem + OFF_DESC);  // [slot][2]: {grp, c, t0, t1}, {stage0, nst, band, 0}
  float* scratch = reinterpret_cast<float*>(smem + OFF_SCRATCH);
  if (threadIdx.x == 0) {
    for (int i = 0; i < TA_NS; ++i) {
      mbar_init(bar_full + 8 * i, 1);
      mbar_init(bar_empty + 8 * i, 1);
    }
    for (int i = 0; i < TA_ND; ++i) {
      mbar_init(bar_dfull + 8 * i, 1);
      mbar_init(bar_dempty + 8 * i, TA_NC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  TL_MARK(p, TL_AMEND_IN);
  const int Hkv = p.n_kv_heads, Hq = p.n_q_heads, g = Hq / Hkv, r = p.band, ps = p.page_size;
  const Workspace w = workspace_layout(p);
  const int* mpos = ws_ptr<const int>(p, w.mpos_off);

  if (warp == TA_NC) {
    // ------------------------------------------------------------------ producer
    uint64_t policy;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
    int gstage = 0, ditem = 0;
    auto put = [&](int grp, int c, int t0, int t1, int band) {
      const int b = grp / Hkv, kvh = grp % Hkv;
      const int nsub = ((t1 - t0) >> 4) + 1, nst = (nsub + 1) >> 1;
      const int ds = ditem % TA_ND;
      if (lane == 0) {
        mbar_wait(bar_dempty + 8 * ds, ((ditem / TA_ND) & 1) ^ 1);
        desc[2 * ds] = make_int4(grp, c, t0, t1);
        desc[2 * ds + 1] = make_int4(gstage, nst, band, 0);
        mbar_arrive(bar_dfull + 8 * ds);
      }
      ++ditem;
      for (int blk = 0; blk * 32 < nsub; ++blk) {
        // lane j: the first cache row of sub-tile 32 blk + j (16 tokens inside one page)
        int row = 0;
        const int j = blk * 32 + lane;
        if (j < nsub) {
          const int local = t0 + (j << 4) - p.kv_offset;
          const int page = __ldg(p.page_table + (int64_t)b * p.pages_per_seq + min((local - 1) / ps, p.pages_per_seq - 1));
          row = (page * Hkv + kvh) * ps + ((local - 1) % ps);
        }
        const int nin = min(32, nsub - blk * 32);
        for (int jj = 0; jj < nin; jj += 2) {
          const int r0 = __shfl_sync(0xffffffffu, row, jj);
          const int r1 = __shfl_sync(0xffffffffu, row, (jj + 1) & 31);
          const bool has1 = jj + 1 < nin;
          if (lane == 0) {
            const int st = gstage % TA_NS;
            mbar_wait(bar_empty + 8 * st, ((gstage / TA_NS) & 1) ^ 1);
            const uint32_t fb = bar_full + 8 * st;
            mbar_expect_tx(fb, has1 ? TA_STAGE : TA_STAGE / 2);
            const uint32_t sb = base + st * TA_STAGE;
            tma_load(sb, &tmK, 0, r0, fb, policy);
            tma_load(sb + 2048, &tmK, 64, r0, fb, policy);
            tma_load(sb + 2 * TILE_BYTES, &tmV, 0, r0, fb, policy);
            tma_load(sb + 2 * TILE_BYTES + 2048, &tmV, 64, r0, fb, policy);
            if (has1) {
              tma_load(sb + TILE_BYTES, &tmK, 0, r1, fb, policy);
              tma_load(sb + TILE_BYTES + 2048, &tmK, 64, r1, fb, policy);
              tma_load(sb + 3 * TILE_BYTES, &tmV, 0, r1, fb, policy);
              tma_load(sb + 3 * TILE_BYTES + 2048, &tmV, 64, r1, fb, policy);
            }
          }
          ++gstage;
        }
      }
    };
    if (nb > 0) {  // static split-band items: need only what the front kernel wrote
      const int G = p.batch * Hkv;
      for (int i = blockIdx.x; i < G * nb; i += gridDim.x) {
        const int grp = i / nb, c = i - grp * nb;
        const int m = __ldcg(mpos + grp / Hkv);
        const BandItems bi = band_items(m, r, nb);
        if (c >= bi.n) continue;
        const int t0 = bi.t0 + c * bi.len;
        put(grp, c, t0, min(m, t0 + bi.len - 1), 1);
      }
    }
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    TL_MARK(p, TL_AMEND_WAITED);
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    unsigned int* ctr = ws_ptr<unsigned int>(p, w.ctr_off);
    const int4* list = ws_ptr<const int4>(p, w.list_off);
    const unsigned n_items = __ldcg(ctr);
    for (;;) {
      unsigned next = 0;
      if (lane == 0) next = atomicAdd(ctr + 1, 1u);
      next = __shfl_sync(0xffffffffu, next, 0);
      if (next >= n_items) break;
      const int4 it = __ldcg(list + next);
      put(it.x - 1, it.y, it.z, it.w, 0);
    }
    if (lane == 0) {  // end of work
      const int ds = ditem % TA_ND;
      mbar_wait(bar_dempty + 8 * ds, ((ditem / TA_ND) & 1) ^ 1);
      desc[2 * ds + 1] = make_int4(0, -1, 0, 0);
      mbar_arrive(bar_dfull + 8 * ds);
    }
    return;
  }

  // -------------------------------------------------------------------- consumers
  const int cw = warp;
  const int row = lane >> 2, q4 = lane & 3;
  const float scale2 = (float)(1.0 / sqrt(128.0)) * LOG2E;
  const int* plan_lo = ws_ptr<const int>(p, w.lo_off);
  const float* qrot = ws_ptr<const float>(p, w.qrot_off);
  float* part = ws_ptr<float>(p, w.part_off);
  float* scr = scratch + cw * TA_PART;
  bool waited = false;
  for (int ditem = 0;; ++ditem) {
    const int ds = ditem % TA_ND;
    mbar_wait(bar_dfull + 8 * ds, (ditem / TA_ND) & 1);
    const int4 it = desc[2 * ds];
    const int4 meta = desc[2 * ds + 1];
    const int nst = (int)__reduce_max_sync(0xffffffffu, (unsigned)(meta.y + 1)) - 1;
    if (nst < 0) break;
    const bool BAND = meta.z != 0;
    if (!BAND && !waited) {  // piece items read the verify kernel's plan
      asm volatile("griddepcontrol.wait;\n" ::: "memory");
      waited = true;
    }
    const int grp = (int)__reduce_max_sync(0xffffffffu, (unsigned)it.x);
    const int c = (int)__reduce_max_sync(0xffffffffu, (unsigned)it.y);
    const int t0 = (int)__reduce_max_sync(0xffffffffu, (unsigned)it.z);
    const int t1 = (int)__reduce_max_sync(0xffffffffu, (unsigned)it.w);
    const int stage0 = (int)__reduce_max_sync(0xffffffffu, (unsigned)meta.x);
    const int b = grp / Hkv, kvh = grp % Hkv;
    const int nsub = ((t1 - t0) >> 4) + 1;
    const int m = (int)__reduce_max_sync(0xffffffffu, (unsigned)__ldcg(mpos + b));
    const int cpos = m - r;
    const int lo_h = row < g ? (BAND ? 1 : __ldcg(plan_lo + b * Hq + kvh * g + row)) : (1 << 30);
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
    State S;
    S.reset();
    bool in_band = false;
    const int lo_piece = max(lo_h, t0), hi_piece = BAND ? t0 - 1 : min(t1, cpos);
    const int lo_band = max(lo_h, max(t0, cpos + 1));
    auto step = [&](int sidx, uint32_t sb, auto has1_tag) {
      constexpr bool HAS1 = decltype(has1_tag)::value;
      const int ts = t0 + (sidx << 5);
      const uint32_t ks0 = sb, ks1 = sb + TILE_BYTES, vs0 = sb + 2 * TILE_BYTES, vs1 = sb + 3 * TILE_BYTES;
      float s[4][2][4];
      {
        const int mi = lane >> 3, ii = lane & 7;
        const int trow = ((mi >> 1) << 3) + ii;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          uint32_t b0, b1, b2, b3;
          ldsm_x4(ks0 + swz128(trow, 2 * ks + (mi & 1)), b0, b1, b2, b3);
          if (ks < 2) {
            mma16816_z(s[0][ks & 1], qa[ks], b0, b1);
            mma16816_z(s[1][ks & 1], qa[ks], b2, b3);
          } else {
            mma16816(s[0][ks & 1], qa[ks], b0, b1);
            mma16816(s[1][ks & 1], qa[ks], b2, b3);
          }
          if (HAS1) {
            uint32_t c0, c1, c2, c3;
            ldsm_x4(ks1 + swz128(trow, 2 * ks + (mi & 1)), c0, c1, c2, c3);
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
      if (__any_sync(0xffffffffu, ts <= hi_piece))
        softmax_pv<HAS1, true>(S, l, tok, lo_piece, HAS1 ? hi_piece : min(hi_piece, ts + 15), vs0, vs1, lane);
      if (__any_sync(0xffffffffu, ts + 31 > cpos && max(ts, cpos + 1) <= t1)) {
        if (!in_band) {
          write_partial(S, scr, 0, row, q4, g);
          S.reset();
          in_band = true;
        }
        softmax_pv<HAS1, true>(S, l, tok, lo_band, hi_band, vs0, vs1, lane);
      }
    };
    for (int sidx = cw; sidx < nst; sidx += TA_NC) {
      const int gs = stage0 + sidx;
      const int st = gs % TA_NS;
      mbar_wait(bar_full + 8 * st, (gs / TA_NS) & 1);
      const uint32_t sb = base + st * TA_STAGE;
      if (2 * sidx + 1 < nsub) step(sidx, sb, std::true_type{});
      else step(sidx, sb, std::false_type{});
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_empty + 8 * st);
    }
    if (!in_band) {
      write_partial(S, scr, 0, row, q4, g);
      S.reset();
    }
    write_partial(S, scr, 1, row, q4, g);
    consumers_sync<TA_NC>();
    // merge the TA_NC consumers' partials of each (head, set) and store the item's slot
    float* out = part + ((int64_t)(grp * p.max_chunks + c) * g) * 2 * 129;
    for (int hs = cw; hs < 2 * g; hs += TA_NC) {
      float lw[TA_NC], L = -CUDART_INF_F;
#pragma unroll
      for (int k = 0; k < TA_NC; ++k) {
        lw[k] = scratch[k * TA_PART + hs * 129 + 128];
        L = fmaxf(L, lw[k]);
      }
      float wk[TA_NC], Z = 0.f;
#pragma unroll
      for (int k = 0; k < TA_NC; ++k) {
        wk[k] = lw[k] == -CUDART_INF_F ? 0.f : __expf(lw[k] - L);
        Z += wk[k];
      }
      const float iz = Z > 0.f ? 1.f / Z : 0.f;
#pragma unroll
      for (int e4 = 0; e4 < 4; ++e4) {
        const int e = lane + 32 * e4;
        float a = 0.f;
#pragma unroll
        for (int k = 0; k < TA_NC; ++k) a += scratch[k * TA_PART + hs * 129 + e] * wk[k];
        out[hs * 129 + e] = a * iz;
      }
      if (lane == 0) out[hs * 129 + 128] = Z > 0.f ? L + __logf(Z) : -CUDART_INF_F;
    }
    consumers_sync<TA_NC>();  // scratch free for the next item
    if (lane == 0) mbar_arrive(bar_dempty + 8 * ds);
  }
  if (!waited) asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  TL_MARK(p, TL_AMEND_OUT);
  // the work counters are returned to zero by the complete kernel (after this grid)
}

// ---------------------------------------------------------------------------------- host
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

// a [rows, 128] bf16 view of a paged cache ([num_pages, Hkv, page_size, 128]: one row per
// (page, kv head, slot)), 64 x 16 boxes, 128-byte swizzle.  The row count only bounds the
// coordinates (every coordinate the kernel issues lies inside the caller's allocation).
bool encode_cache_map(CUtensorMap* m, const void* ptr) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  const cuuint64_t dims[2] = {128, (cuuint64_t)1 << 31};
  const cuuint64_t strides[1] = {256};
  const cuuint32_t box[2] = {64, 16};
  const cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// variants (consumers, stages, CTAs per SM); development builds select 2-4 with MAC_AMEND_TMA
struct TmaVariant {
  void (*fn)(const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap, MacDecodeParams, int);
  int threads, smem;
};
static const TmaVariant kTma[] = {
    // 2 consumers, 4 stages, 2 CTAs per SM (same box, dev A/B vs 3 / 3 / 2: C2 34.3 vs 34.6 us;
    // C3 geometry at 16K in dense mode, 0.5 / 2 / 10 % misses: 71.5 / 87.5 / 180 vs 74 / 92 / 194)
    {amend_tma_kernel<2, 4, 2>, TmaRing<2, 4>::THREADS, TmaRing<2, 4>::SMEM},
#ifdef MAC_DEV_KNOBS
    {amend_tma_kernel<6, 6, 1>, TmaRing<6, 6>::THREADS, TmaRing<6, 6>::SMEM},  // MAC_AMEND_TMA=2
    {amend_tma_kernel<2, 2, 4>, TmaRing<2, 2>::THREADS, TmaRing<2, 2>::SMEM},  // MAC_AMEND_TMA=3 (38.3 at C2)
    {amend_tma_kernel<3, 3, 2>, TmaRing<3, 3>::THREADS, TmaRing<3, 3>::SMEM},  // MAC_AMEND_TMA=4 (round 2's first)
#endif
};
static int tma_variant() {
#ifdef MAC_DEV_KNOBS
  static int v = -1;
  if (v < 0) {
    const char* env = getenv("MAC_AMEND_TMA");
    v = env ? (atoi(env) == 2 ? 1 : atoi(env) == 3 ? 2 : atoi(env) == 4 ? 3 : 0) : 0;
  }
  return v;
#else
  return 0;
#endif
}

// CTAs of the persistent grid (occupancy x SMs); sets the shared-memory attribute on first use
int amend_tma_grid(cudaError_t* err) {
  static int grid = 0;
  if (!grid) {
    const TmaVariant& tv = kTma[tma_variant()];
    cudaError_t e = cudaFuncSetAttribute(tv.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, tv.smem);
    if (e != cudaSuccess) {
      if (err) *err = e;
      return 0;
    }
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tv.fn, tv.threads, tv.smem);
    grid = sms * (per_sm < 1 ? 1 : per_sm);
  }
  return grid;
}

bool amend_tma_supported(const MacDecodeParams& p) {
  return amend_mma_supported(p) && tensor_map_encoder() != nullptr &&
         (reinterpret_cast<uintptr_t>(p.k_cache) & 15) == 0 && (reinterpret_cast<uintptr_t>(p.v_cache) & 15) == 0;
}

cudaError_t launch_amend_tma(const MacDecodeParams& p, cudaStream_t st, int nb) {
  cudaError_t err = cudaSuccess;
  const int gfull = amend_tma_grid(&err);
  if (err != cudaSuccess) return err;
  // tensor maps of this layer's caches (encoded on the host; kept while the pointers repeat)
  static const void* lastK = nullptr;
  static const void* lastV = nullptr;
  static CUtensorMap mK, mV;
  if (p.k_cache != lastK || p.v_cache != lastV) {
    if (!encode_cache_map(&mK, p.k_cache) || !encode_cache_map(&mV, p.v_cache)) return cudaErrorInvalidValue;
    lastK = p.k_cache;
    lastV = p.v_cache;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(gfull);
  const TmaVariant& tv = kTma[tma_variant()];
  cfg.blockDim = dim3(tv.threads);
  cfg.dynamicSmemBytes = tv.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, tv.fn, mK, mV, p, nb);
}

}  // namespace mac
