// K2 on the 5th-generation tensor cores: the bf16 d = 128 amend of the decode step with
// tcgen05 MMAs (accumulators in TMEM) fed by TMA, for GQA groups of g = 1, 2, 4 or 8 heads.
//
// Same contract and per-token math as amend_mma.cuh / amend_tma.cu (engine.py:464-470,
// 484-493; attention.py:75-116): for each work item {grp, c, t0, t1} of the device plan
// (common.cuh plan_group / band_items) emit the piece (t <= m-r) and band (t > m-r) partial
// summaries of each of the group's g heads, masking each head below its own lo_h.
//
// Why: the mma.sync amends (one-warp and TMA-fed) reach ~0.5 of HBM bandwidth — a decode
// group has only g = 4 query rows, so a 16-row mma.sync tile is 3/4 idle and the warps' issue
// slots (ldmatrix, 32 MMAs per 16 tokens, softmax) run out before the bytes do.  Here the
// token axis is the MMA's M dimension instead, so the tensor core does the whole contraction
// of a 64-token block in 12 instructions of one thread:
//   S^T[t, n] = K[t, :] . Qc[n, :]      M = 128 (the 64 tokens of the block; rows 64..127 are
//                                       don't-care), N = 8 / 16: the g heads' queries split
//                                       hi + lo into bf16 (fp32-exact logits: logit = col h +
//                                       col g+h), pre-scaled by log2(e) / sqrt(d); K = 128 dims
//   O^T[d, n] = V[:, d] . P^T[:, n]     M = 128 dims (V read MN-major straight from the TMA
//                                       tile), N = 4g: P hi / lo for the piece and the band
//                                       sets as separate columns, so an item that straddles
//                                       m - r needs no second pass; K = the block's tokens
// Both operands of S^T and the V operand are the K/V tiles exactly as TMA lands them (64-dim
// SWIZZLE_128B boxes of 16 rows), validated by tools/umma_probe2.cu.
//
// Warp roles (192 threads, 2 CTAs per SM, persistent over the work list like amend_tma.cu):
//   warp 0    TMA producer: claims items (the static split-band items first, then the plan's
//             items after the grid-dependency wait), streams each item's pages in 64-token
//             blocks into a ring of TC_NS stages (K and V, 32 KiB), posts item descriptors;
//   warp 1    MMA issuer: writes each item's Qc (hi / lo, scaled) into shared memory, issues
//             S^T of block j+1 before P V of block j (S and O double-buffered in TMEM, P in
//             shared memory), and frees a stage when its P V completes;
//   warps 2-5 softmax + epilogue (TMEM lane i = token i for S, dim i for O): online softmax
//             with the lazy rescale of amend_mma.cuh (the running max moves only when a logit
//             exceeds it by > 8 in log2, decided by one barrier vote per block), P hi / lo into
//             shared memory, then O of the previous block folded into per-dim registers; at the
//             item's end the token-sums are reduced and the partials written.
//
// Measured (r02, profiles/r02/SUMMARY.md "tcgen05 amend"): parity-green on the whole GPU suite
// with every cooperative amend routed here, but SLOWER than the product amends — C3 hit step
// amend 46 us vs 27 (one-warp mma.sync) and 33 (TMA-fed mma.sync); C2 38.5 vs 34 us.  The
// tensor work was never the bound: per-CTA role counters (MAC_TIMELINE) show each 64-token
// block costing ~3 us of serial softmax-warp latency (TMEM load, vote barrier, P stores +
// proxy fence, MMA-commit round trips) with only two such pipelines per SM, while the C3 plan
// is ~1000 items of ~170 tokens.  (The one-warp mma.sync amend streams long spans at 7.2 TB/s —
// full attention — so its C3 gap to the roofline is item latency, not MMA issue.)  Compiled in
// development builds only (MAC_AMEND_TC=1 with MAC_AMEND_TMA=1).
#include <cuda.h>
#include <stdio.h>
#include <stdlib.h>

#include "amend_mma.cuh"
#include "umma.cuh"

#ifdef MAC_DEV_KNOBS  // development builds only (see the header: measured slower than the product amends)
namespace mac {

bool amend_tma_supported(const MacDecodeParams& p);
bool encode_cache_map(CUtensorMap* m, const void* ptr);

namespace {
constexpr int TC_BT = 64;                   // tokens per block
constexpr int TC_NS = 3;                    // K/V stages
constexpr int TC_KV = TC_BT * 256;          // one block's K (or V): two 64-dim atoms of 64 rows x 128 B
constexpr int TC_STAGE = 2 * TC_KV;         // K then V: 32 KiB
constexpr int TC_ND = 4;                    // item descriptor slots
constexpr int TC_THREADS = 192;

template <int G> struct TcGeom {
  static constexpr int NSQ = 2 * G <= 8 ? 8 : 16;          // S^T columns (hi, lo per head; padded)
  static constexpr int NO = 4 * G <= 8 ? 8 : 4 * G;         // O^T columns: (piece, band) x (hi, lo) x g
  static constexpr int QB = NSQ * 256;                      // Qc: two 64-dim atoms of NSQ rows x 128 B
  static constexpr int PB = (NO * 128 + 1023) & ~1023;      // P^T: one 64-token atom of NO rows x 128 B
  static constexpr int OFF_Q = TC_NS * TC_STAGE;
  static constexpr int OFF_P = OFF_Q + 2 * QB;
  static constexpr int OFF_RED = OFF_P + 2 * PB;            // [4 warps][2g] floats
  static constexpr int OFF_ACT = OFF_RED + 4 * 16 * 4;      // [2] sets of each P buffer's block
  static constexpr int OFF_DESC = OFF_ACT + 16;
  // g >= 4: P V per active set (N = 2g >= 8): a block entirely in the piece or the band computes
  // and multiplies one set only
  static constexpr bool SPLIT_SETS = G >= 4;
  static constexpr int OFF_BAR = OFF_DESC + TC_ND * 32;
  static constexpr int N_BAR = 2 * TC_NS + 2 * TC_ND + 12;
  static constexpr int OFF_TMEM = OFF_BAR + 8 * N_BAR;
  static constexpr int SMEM = OFF_TMEM + 16 + 1024;         // + 1024-byte alignment of the base
};
// TMEM columns: S^T buffers at 0 / 16, O^T buffers at 32 / 64
constexpr uint32_t TC_TMEM_COLS = 128;

__device__ __forceinline__ void tc_tma_load(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void sm_bar(int id) { asm volatile("bar.sync %0, 128;" ::"r"(id) : "memory"); }
__device__ __forceinline__ bool sm_bar_or(int id, bool v) {
  int r;
  asm volatile(
      "{\n"
      ".reg .pred p, q;\n"
      "setp.ne.s32 p, %1, 0;\n"
      "bar.red.or.pred q, %2, 128, p;\n"
      "selp.s32 %0, 1, 0, q;\n"
      "}\n"
      : "=r"(r)
      : "r"(v ? 1 : 0), "r"(id)
      : "memory");
  return r != 0;
}
// (row n, element k) of a K-major SW128 operand with R rows, 64-element atoms R*128 bytes apart
__device__ __forceinline__ uint32_t kmaj(int n, int k, int R) {
  return (uint32_t)((k >> 6) * R * 128 + n * 128 + ((((k & 63) >> 3) ^ (n & 7)) << 4) + (k & 7) * 2);
}
template <int N> __device__ __forceinline__ void tmem_ld_n(uint32_t taddr, uint32_t (&v)[N]) {
  if constexpr (N == 8) umma::tmem_ld8(taddr, v);
  else if constexpr (N == 16) umma::tmem_ld16(taddr, v);
  else umma::tmem_ld32(taddr, v);
}
}  // namespace

#ifdef MAC_TIMELINE
// development builds: per CTA {start ns, end ns, softmax cycles waiting S, waiting O, at item
// starts, producer cycles waiting for a stage, MMA cycles waiting for data, items}
__device__ unsigned long long g_tc_trace[1024 * 16];
#define TC_CLK(v) const long long v = clock64()
#define TC_ADD(i, v) (tr[i] += (unsigned long long)(clock64() - (v)))
#else
#define TC_CLK(v) ((void)0)
#define TC_ADD(i, v) ((void)0)
#endif

template <int G>
__global__ void __launch_bounds__(TC_THREADS, 2)
    amend_tc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                    MacDecodeParams p, int nb) {
  using Q = TcGeom<G>;
  constexpr int NSQ = Q::NSQ, NO = Q::NO;
  extern __shared__ unsigned char smem_raw[];
  const uint32_t raw = umma::smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  unsigned char* smem = smem_raw + (base - raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // barriers
  const uint32_t b_full = base + Q::OFF_BAR, b_empty = b_full + 8 * TC_NS;
  const uint32_t b_dfull = b_empty + 8 * TC_NS, b_dempty = b_dfull + 8 * TC_ND;
  const uint32_t b_sfull = b_dempty + 8 * TC_ND, b_sfree = b_sfull + 16, b_pfull = b_sfree + 16;
  const uint32_t b_ofull = b_pfull + 16, b_ofree = b_ofull + 16, b_qfree = b_ofree + 16;
  int4* desc = reinterpret_cast<int4*>(smem + Q::OFF_DESC);  // [slot][2]: {grp, c, t0, t1}, {gblk0, nblk, band, 0}
  float* red = reinterpret_cast<float*>(smem + Q::OFF_RED);
  int* act_s = reinterpret_cast<int*>(smem + Q::OFF_ACT);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + Q::OFF_TMEM);
  if (threadIdx.x == 0) {
    for (int i = 0; i < TC_NS; ++i) {
      umma::mbar_init(b_full + 8 * i, 1);
      umma::mbar_init(b_empty + 8 * i, 1);
    }
    for (int i = 0; i < TC_ND; ++i) {
      umma::mbar_init(b_dfull + 8 * i, 1);
      umma::mbar_init(b_dempty + 8 * i, 2);
    }
    for (int i = 0; i < 2; ++i) {
      umma::mbar_init(b_sfull + 8 * i, 1);
      umma::mbar_init(b_sfree + 8 * i, 4);
      umma::mbar_init(b_pfull + 8 * i, 4);
      umma::mbar_init(b_ofull + 8 * i, 1);
      umma::mbar_init(b_ofree + 8 * i, 4);
      umma::mbar_init(b_qfree + 8 * i, 1);
    }
    umma::fence_mbar_init();
  }
  // the Qc pad rows (2g .. NSQ-1) stay zero
  for (int i = threadIdx.x; i < 2 * Q::QB / 4; i += TC_THREADS) reinterpret_cast<uint32_t*>(smem + Q::OFF_Q)[i] = 0u;
  umma::fence_proxy_async_smem();
  if (warp == 1) umma::tmem_alloc(umma::smem_u32(tmem_slot), TC_TMEM_COLS);
  umma::tc_fence_before();
  __syncthreads();
  umma::tc_fence_after();
  const uint32_t tm = *tmem_slot;
  TL_MARK(p, TL_AMEND_IN);
#ifdef MAC_TIMELINE
  unsigned long long tr[16] = {};
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr[0]));
#endif
  const int Hkv = p.n_kv_heads, Hq = p.n_q_heads, r = p.band, ps = p.page_size;
  const Workspace w = workspace_layout(p);
  const int* mpos = ws_ptr<const int>(p, w.mpos_off);

  if (warp == 0) {
    // ------------------------------------------------------------------ producer
    uint64_t policy;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
    int gblk = 0, ditem = 0;
    auto put = [&](int grp, int c, int t0, int t1, int band) {
      const int b = grp / Hkv, kvh = grp % Hkv;
      const int nsub = ((t1 - t0) >> 4) + 1, nblk = (nsub + 3) >> 2;
      const int ds = ditem % TC_ND;
      if (lane == 0) {
        umma::mbar_wait_parity(b_dempty + 8 * ds, ((ditem / TC_ND) & 1) ^ 1);
        desc[2 * ds] = make_int4(grp, c, t0, t1);
        desc[2 * ds + 1] = make_int4(gblk, nblk, band, 0);
        umma::mbar_arrive(b_dfull + 8 * ds);
      }
      ++ditem;
      for (int blk = 0; blk < nblk; ++blk) {
        const int nin = min(4, nsub - 4 * blk);
        int row = 0;
        if (lane < nin) {
          const int local = t0 + 64 * blk + 16 * lane - p.kv_offset;
          const int page = __ldg(p.page_table + (int64_t)b * p.pages_per_seq + min((local - 1) / ps, p.pages_per_seq - 1));
          row = (page * Hkv + kvh) * ps + ((local - 1) % ps);
        }
        int rr[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) rr[j] = __shfl_sync(0xffffffffu, row, j);
        if (lane == 0) {
          const int st = gblk % TC_NS;
          TC_CLK(c0);
          umma::mbar_wait_parity(b_empty + 8 * st, ((gblk / TC_NS) & 1) ^ 1);
          TC_ADD(5, c0);
          const uint32_t fb = b_full + 8 * st, sb = base + st * TC_STAGE;
          umma::mbar_expect_tx(fb, (unsigned)nin * 4 * 2048);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (j < nin) {
              tc_tma_load(sb + j * 2048, &tmK, 0, rr[j], fb, policy);
              tc_tma_load(sb + TC_KV / 2 + j * 2048, &tmK, 64, rr[j], fb, policy);
              tc_tma_load(sb + TC_KV + j * 2048, &tmV, 0, rr[j], fb, policy);
              tc_tma_load(sb + TC_KV + TC_KV / 2 + j * 2048, &tmV, 64, rr[j], fb, policy);
            }
          }
        }
        ++gblk;
      }
    };
    if (nb > 0) {  // static split-band items: need only what the front kernel wrote
      const int Gn = p.batch * Hkv;
      for (int i = blockIdx.x; i < Gn * nb; i += gridDim.x) {
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
      const int ds = ditem % TC_ND;
      umma::mbar_wait_parity(b_dempty + 8 * ds, ((ditem / TC_ND) & 1) ^ 1);
      desc[2 * ds + 1] = make_int4(0, -1, 0, 0);
      umma::mbar_arrive(b_dfull + 8 * ds);
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    const float scale2 = (float)(1.0 / sqrt(128.0)) * LOG2E;
    const float* qrot = ws_ptr<const float>(p, w.qrot_off);
    constexpr uint32_t idS = umma::instr_desc_bf16(128, NSQ, false, false);
    constexpr uint32_t idO = umma::instr_desc_bf16(128, NO, true, false);
    constexpr uint32_t idO2 = umma::instr_desc_bf16(128, 2 * G < 8 ? 8 : 2 * G, true, false);  // one set
    // Event loop of one thread (lane 0; the warp only helps write Qc): S^T of the next block
    // needs its stage and a free S buffer, P V of a block needs its P and a free O buffer, and
    // whichever is ready first is issued — so a stage is released as soon as its P is, not
    // behind the next block's TMA (up to two blocks between their S^T and their P V).
    int gb = 0;
    int pv_head = 0, pv_tail = 0;  // queued P V blocks [pv_head, pv_tail): gb of each is its index
    int pv_st[2], pv_nk[2];
    auto try_pv = [&]() {  // lane 0 only
      if (pv_head == pv_tail) return;
      const int buf = pv_head & 1, u = pv_head >> 1;
      if (!umma::mbar_test_parity(b_pfull + 8 * buf, u & 1) || !umma::mbar_test_parity(b_ofree + 8 * buf, (u & 1) ^ 1))
        return;
      umma::tc_fence_after();
      const int st = pv_st[buf];
      const uint32_t vb = base + st * TC_STAGE + TC_KV;
      const uint32_t pbuf = base + Q::OFF_P + buf * Q::PB;
      if constexpr (Q::SPLIT_SETS) {
        const int act = act_s[buf];
#pragma unroll
        for (int s = 0; s < 2; ++s)
          if ((act >> s) & 1)
            for (int ks = 0; ks < pv_nk[buf]; ++ks)
              umma::mma_bf16(tm + 32 + 32 * buf + s * 2 * G, umma::sdesc_mnmajor_sw128(vb + ks * 2048, TC_KV / 2),
                             umma::sdesc_kmajor_sw128(pbuf + s * 2 * G * 128 + ks * 32), idO2, ks > 0);
      } else {
        for (int ks = 0; ks < pv_nk[buf]; ++ks)
          umma::mma_bf16(tm + 32 + 32 * buf, umma::sdesc_mnmajor_sw128(vb + ks * 2048, TC_KV / 2),
                         umma::sdesc_kmajor_sw128(pbuf + ks * 32), idO, ks > 0);
      }
      umma::mma_commit(b_ofull + 8 * buf);
      umma::mma_commit(b_empty + 8 * st);
      ++pv_head;
    };
    auto wait_for = [&](uint32_t bar, unsigned parity) {  // lane 0: spin, issuing ready P V meanwhile
      while (!umma::mbar_test_parity(bar, parity)) try_pv();
    };
    for (int ditem = 0;; ++ditem) {
      const int ds = ditem % TC_ND;
      if (lane == 0) wait_for(b_dfull + 8 * ds, (ditem / TC_ND) & 1);
      __syncwarp();
      const int4 it = desc[2 * ds];
      const int4 meta = desc[2 * ds + 1];
      __syncwarp();
      if (lane == 0) umma::mbar_arrive(b_dempty + 8 * ds);
      if (meta.y < 0) break;
      const int grp = it.x, t0 = it.z, t1 = it.w, gblk0 = meta.x, nblk = meta.y;
      const int b = grp / Hkv, kvh = grp % Hkv;
      const int nsub = ((t1 - t0) >> 4) + 1;
      // this item's Qc (buffer ditem & 1, free once the S^T MMAs of item ditem - 2 completed)
      const int qb = ditem & 1;
      float4 x[G];
#pragma unroll
      for (int h = 0; h < G; ++h)
        x[h] = __ldcg(reinterpret_cast<const float4*>(qrot + ((int64_t)b * Hq + kvh * G + h) * 128) + lane);
      if (lane == 0) wait_for(b_qfree + 8 * qb, ((ditem >> 1) & 1) ^ 1);
      __syncwarp();
      unsigned char* sq = smem + Q::OFF_Q + qb * Q::QB;
#pragma unroll
      for (int h = 0; h < G; ++h) {
        const float xs[4] = {x[h].x * scale2, x[h].y * scale2, x[h].z * scale2, x[h].w * scale2};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float hi, lo;
          split_bf16(xs[e], hi, lo);
          *reinterpret_cast<__nv_bfloat16*>(sq + kmaj(h, 4 * lane + e, NSQ)) = __float2bfloat16_rn(hi);
          *reinterpret_cast<__nv_bfloat16*>(sq + kmaj(G + h, 4 * lane + e, NSQ)) = __float2bfloat16_rn(lo);
        }
      }
      umma::fence_proxy_async_smem();
      __syncwarp();
      const uint32_t qaddr = base + Q::OFF_Q + qb * Q::QB;
      if (lane == 0) {
        for (int blk = 0; blk < nblk; ++blk, ++gb) {
          const int gblk = gblk0 + blk, st = gblk % TC_NS, buf = gb & 1, u = gb >> 1;
          TC_CLK(c0);
          wait_for(b_full + 8 * st, (gblk / TC_NS) & 1);
          TC_ADD(6, c0);
          wait_for(b_sfree + 8 * buf, (u & 1) ^ 1);
          while (pv_tail - pv_head >= 2) try_pv();  // block gb-2 still queued: its P is on the way
          umma::tc_fence_after();
          const uint32_t kb = base + st * TC_STAGE;
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)
            umma::mma_bf16(tm + 16 * buf, umma::sdesc_kmajor_sw128(kb + (ks >> 2) * (TC_KV / 2) + (ks & 3) * 32),
                           umma::sdesc_kmajor_sw128(qaddr + (ks >> 2) * (NSQ * 128) + (ks & 3) * 32), idS, ks > 0);
          umma::mma_commit(b_sfull + 8 * buf);
          if (blk == nblk - 1) umma::mma_commit(b_qfree + 8 * qb);
          pv_st[buf] = st;
          pv_nk[buf] = min(4, nsub - 4 * blk);
          ++pv_tail;
          try_pv();
        }
      }
      gb = __shfl_sync(0xffffffffu, gb, 0);
    }
    if (lane == 0)
      while (pv_head != pv_tail) try_pv();
  } else {
    // ------------------------------------------------------- softmax + epilogue (128 threads)
    const int q = warp & 3;                // TMEM lane quadrant of this warp
    const int L = 32 * q + lane;           // token row (S^T) / dim (O^T)
    const uint32_t tl = tm + ((uint32_t)(32 * q) << 16);
    const int* plan_lo = ws_ptr<const int>(p, w.lo_off);
    float* part = ws_ptr<float>(p, w.part_off);
    const bool tok_thread = L < TC_BT;
    int gb = 0;
    for (int ditem = 0;; ++ditem) {
      const int ds = ditem % TC_ND;
      TC_CLK(ci);
      umma::mbar_wait_parity(b_dfull + 8 * ds, (ditem / TC_ND) & 1);
      const int4 it = desc[2 * ds];
      const int4 meta = desc[2 * ds + 1];
      sm_bar(1);  // every softmax thread holds the descriptor before the slot is released
      if (threadIdx.x == 64) umma::mbar_arrive(b_dempty + 8 * ds);
      if (meta.y < 0) break;
      const int grp = it.x, c = it.y, t0 = it.z, t1 = it.w, nblk = meta.y;
      const bool BAND = meta.z != 0;
      const int b = grp / Hkv, kvh = grp % Hkv;
      const int m = __ldcg(mpos + b), cpos = m - r;
      int lo_p[G], lo_b[G];
      const int hi_p = BAND ? t0 - 1 : min(t1, cpos), hi_b = t1;
#pragma unroll
      for (int h = 0; h < G; ++h) {
        const int lo_h = BAND ? 1 : __ldcg(plan_lo + b * Hq + kvh * G + h);
        lo_p[h] = max(lo_h, t0);
        lo_b[h] = max(lo_h, max(t0, cpos + 1));
      }
      TC_ADD(4, ci);
#ifdef MAC_TIMELINE
      tr[7]++;
#endif
      float M[2 * G], Z[2 * G], acc[2 * G], a_pend[2 * G];  // index 2h + set
#pragma unroll
      for (int i = 0; i < 2 * G; ++i) {
        M[i] = -CUDART_INF_F;
        Z[i] = 0.f;
        acc[i] = 0.f;
        a_pend[i] = 1.f;
      }
      int act_pend = 3;
      auto epilogue = [&](int eb, int eact) {  // fold block eb's O^T (this thread's dim) into acc
        const int buf = eb & 1, u = eb >> 1;
        TC_CLK(c0);
        umma::mbar_wait_parity(b_ofull + 8 * buf, u & 1);
        TC_ADD(3, c0);
        umma::tc_fence_after();
        uint32_t ov[NO];
        tmem_ld_n<NO>(tl + 32 + 32 * buf, ov);
        umma::tmem_wait_ld();
        umma::tc_fence_before();
        __syncwarp();
        if (lane == 0) umma::mbar_arrive(b_ofree + 8 * buf);
#pragma unroll
        for (int h = 0; h < G; ++h)
#pragma unroll
          for (int s = 0; s < 2; ++s) {
            if (!((eact >> s) & 1)) continue;  // (that set's columns were not written by this block)
            const float o = __uint_as_float(ov[s * 2 * G + h]) + __uint_as_float(ov[s * 2 * G + G + h]);
            acc[2 * h + s] = acc[2 * h + s] * a_pend[2 * h + s] + o;
          }
      };
      for (int blk = 0; blk < nblk; ++blk, ++gb) {
        const int buf = gb & 1, u = gb >> 1;
        TC_CLK(c0);
        umma::mbar_wait_parity(b_sfull + 8 * buf, u & 1);
        TC_ADD(2, c0);
        umma::tc_fence_after();
        uint32_t sv[NSQ];
        tmem_ld_n<NSQ>(tl + 16 * buf, sv);
        umma::tmem_wait_ld();
        umma::tc_fence_before();
        __syncwarp();
        if (lane == 0) umma::mbar_arrive(b_sfree + 8 * buf);
        TC_CLK(c1);
        const int t = t0 + 64 * blk + L;
        // the sets this block touches (uniform): piece tokens <= hi_p, band tokens > cpos
        const int bt0 = t0 + 64 * blk, bt1 = min(t1, bt0 + 63);
        const int act = Q::SPLIT_SETS ? ((bt0 <= hi_p ? 1 : 0) | (bt1 > cpos && bt0 <= hi_b ? 2 : 0)) : 3;
        float lg[2 * G];
        bool ok[2 * G];
        bool exceed = false;
#pragma unroll
        for (int h = 0; h < G; ++h) {
          const float x = __uint_as_float(sv[h]) + __uint_as_float(sv[G + h]);
          ok[2 * h] = (act & 1) && tok_thread && t >= lo_p[h] && t <= hi_p;
          ok[2 * h + 1] = (act & 2) && tok_thread && t >= lo_b[h] && t <= hi_b;
          lg[2 * h] = lg[2 * h + 1] = x;
          exceed |= (ok[2 * h] && x > M[2 * h] + 8.f) || (ok[2 * h + 1] && x > M[2 * h + 1] + 8.f);
        }
        float a_cur[2 * G];
#pragma unroll
        for (int i = 0; i < 2 * G; ++i) a_cur[i] = 1.f;
        TC_ADD(8, c1);
        TC_CLK(c2);
        const bool any_exceed = sm_bar_or(2, exceed);
        TC_ADD(9, c2);
        TC_CLK(c3);
        if (any_exceed) {
          // block max per (head, set) over the 128 threads; the running max moves where a logit
          // exceeds it by more than 8 (lazy rescale: exp2(l - M) <= 256 stays exact)
#pragma unroll
          for (int i = 0; i < 2 * G; ++i) {
            float v = ok[i] ? lg[i] : -CUDART_INF_F;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
            if (lane == 0) red[q * 2 * G + i] = v;
          }
          sm_bar(1);
#pragma unroll
          for (int i = 0; i < 2 * G; ++i) {
            const float bm = fmaxf(fmaxf(red[i], red[2 * G + i]), fmaxf(red[4 * G + i], red[6 * G + i]));
            if (bm > M[i] + 8.f) {
              a_cur[i] = M[i] == -CUDART_INF_F ? 1.f : exp2f(M[i] - bm);
              M[i] = bm;
              Z[i] *= a_cur[i];
            }
          }
          sm_bar(1);  // red is rewritten only after every thread read it
        }
        TC_ADD(10, c3);
        TC_CLK(c4);
        // P^T (buffer gb & 1: its previous P V completed — that block's epilogue waited on it)
        unsigned char* sp = smem + Q::OFF_P + buf * Q::PB;
#pragma unroll
        for (int h = 0; h < G; ++h)
#pragma unroll
          for (int s = 0; s < 2; ++s) {
            if (!((act >> s) & 1)) continue;
            const int i = 2 * h + s;
            const float pv = ok[i] ? exp2f(lg[i] - M[i]) : 0.f;
            Z[i] += pv;
            if (tok_thread) {
              float hi, lo;
              split_bf16(pv, hi, lo);
              *reinterpret_cast<__nv_bfloat16*>(sp + kmaj(s * 2 * G + h, L, NO)) = __float2bfloat16_rn(hi);
              *reinterpret_cast<__nv_bfloat16*>(sp + kmaj(s * 2 * G + G + h, L, NO)) = __float2bfloat16_rn(lo);
            }
          }
        if (threadIdx.x == 64) act_s[buf] = act;
        umma::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) umma::mbar_arrive(b_pfull + 8 * buf);
        TC_ADD(11, c4);
#ifdef MAC_TIMELINE
        tr[12]++;
#endif
        if (blk > 0) epilogue(gb - 1, act_pend);
#pragma unroll
        for (int i = 0; i < 2 * G; ++i) a_pend[i] = a_cur[i];
        act_pend = act;
      }
      epilogue(gb - 1, act_pend);
      TC_CLK(c5);
      // token sums over the 128 threads, then this thread's dim of every (head, set) partial
#pragma unroll
      for (int i = 0; i < 2 * G; ++i) {
        float v = Z[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) red[q * 2 * G + i] = v;
      }
      sm_bar(1);
      float* out = part + ((int64_t)(grp * p.max_chunks + c) * G) * 2 * 129;
#pragma unroll
      for (int i = 0; i < 2 * G; ++i) {
        const float Zt = (red[i] + red[2 * G + i]) + (red[4 * G + i] + red[6 * G + i]);
        out[i * 129 + L] = Zt > 0.f ? acc[i] / Zt : 0.f;
        if (L == 0) out[i * 129 + 128] = Zt > 0.f ? M[i] * LN2 + logf(Zt) : -CUDART_INF_F;
      }
      sm_bar(1);
      TC_ADD(13, c5);
    }
  }
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  umma::tc_fence_before();
  __syncthreads();
  if (warp == 1) umma::tmem_dealloc(tm, TC_TMEM_COLS);
  TL_MARK(p, TL_AMEND_OUT);
#ifdef MAC_TIMELINE
  // producer lane 0 (5), MMA lane 0 (6), softmax thread 64 (2, 3, 4, 7) hold their fields
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr[1]));
  if (blockIdx.x < 1024) {
    unsigned long long* o = g_tc_trace + blockIdx.x * 16;
    if (threadIdx.x == 0) { o[0] = tr[0]; o[1] = tr[1]; o[5] = tr[5]; }
    if (threadIdx.x == 32) o[6] = tr[6];
    if (threadIdx.x == 64) { o[2] = tr[2]; o[3] = tr[3]; o[4] = tr[4]; o[7] = tr[7]; for (int i = 8; i < 16; ++i) o[i] = tr[i]; }
  }
#endif
}

#ifdef MAC_TIMELINE
extern "C" int mac_timeline_amend_tc(void* host_out, int n) {
  return (int)cudaMemcpyFromSymbol(host_out, g_tc_trace, (size_t)n * 16 * sizeof(unsigned long long));
}
#endif

// ---------------------------------------------------------------------------------- host
template <int G> static int tc_grid(cudaError_t* err) {
  static int grid = 0;
  if (!grid) {
    cudaError_t e = cudaFuncSetAttribute(amend_tc_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcGeom<G>::SMEM);
    // the whole unified L1 as shared memory, so two CTAs (2 x ~108 KB at g = 4) fit per SM
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(amend_tc_kernel<G>, cudaFuncAttributePreferredSharedMemoryCarveout,
                               cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) {
      if (err) *err = e;
      return 0;
    }
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, amend_tc_kernel<G>, TC_THREADS, TcGeom<G>::SMEM);
    // (the occupancy query answers 1 for the ~108 KB of g = 4 although two CTAs fit the SM's
    // 228 KB — ncu reports a shared-memory limit of 2 — so the grid is sized from the budget)
    int smem_sm = 0;
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    if (per_sm < 2 && 2 * (TcGeom<G>::SMEM + 1024) <= smem_sm) per_sm = 2;
    grid = sms * (per_sm < 1 ? 1 : per_sm);
#ifdef MAC_DEV_KNOBS
    if (getenv("MAC_TC_DEBUG")) {
      cudaFuncAttributes fa;
      cudaFuncGetAttributes(&fa, amend_tc_kernel<G>);
      fprintf(stderr, "amend_tc<%d>: per_sm %d grid %d smem dyn %d static %zu regs %d maxdyn %d\n", G, per_sm, grid,
              TcGeom<G>::SMEM, fa.sharedSizeBytes, fa.numRegs, fa.maxDynamicSharedSizeBytes);
    }
#endif
  }
  return grid;
}

bool amend_tc_supported(const MacDecodeParams& p) {
  const int g = p.n_q_heads / p.n_kv_heads;
  return amend_tma_supported(p) && (g == 1 || g == 2 || g == 4 || g == 8);
}

int amend_tc_grid(const MacDecodeParams& p, cudaError_t* err) {
  switch (p.n_q_heads / p.n_kv_heads) {
    case 1: return tc_grid<1>(err);
    case 2: return tc_grid<2>(err);
    case 4: return tc_grid<4>(err);
    default: return tc_grid<8>(err);
  }
}

cudaError_t launch_amend_tc(const MacDecodeParams& p, cudaStream_t st, int nb) {
  cudaError_t err = cudaSuccess;
  const int g = p.n_q_heads / p.n_kv_heads;
  const int grid = amend_tc_grid(p, &err);
  if (err != cudaSuccess) return err;
  static const void* lastK = nullptr;
  static const void* lastV = nullptr;
  static CUtensorMap mK, mV;
  if (p.k_cache != lastK || p.v_cache != lastV) {
    if (!encode_cache_map(&mK, p.k_cache) || !encode_cache_map(&mV, p.v_cache)) return cudaErrorInvalidValue;
    lastK = p.k_cache;
    lastV = p.v_cache;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(TC_THREADS);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  switch (g) {
    case 1: cfg.dynamicSmemBytes = TcGeom<1>::SMEM; return cudaLaunchKernelEx(&cfg, amend_tc_kernel<1>, mK, mV, p, nb);
    case 2: cfg.dynamicSmemBytes = TcGeom<2>::SMEM; return cudaLaunchKernelEx(&cfg, amend_tc_kernel<2>, mK, mV, p, nb);
    case 4: cfg.dynamicSmemBytes = TcGeom<4>::SMEM; return cudaLaunchKernelEx(&cfg, amend_tc_kernel<4>, mK, mV, p, nb);
    default: cfg.dynamicSmemBytes = TcGeom<8>::SMEM; return cudaLaunchKernelEx(&cfg, amend_tc_kernel<8>, mK, mV, p, nb);
  }
}

}  // namespace mac
#endif  // MAC_DEV_KNOBS
