// Per-head "complete" (K3): merge cached(p) (+) piece (+) band, emit the
// output, write the ring entry back (the paper's rectify-append).  Shared by
// the standalone complete kernel (complete.cu) and the tail of the fused
// tensor-core amend kernel (amend_mma.cu).
//
// Reference: engine.py:468-479 (prefix = merge(cached, piece1); full =
// merge(prefix, band); out = finalize(full)), engine.py:486-499 (miss),
// engine.py:474-478,494-498 (optional remove() downdate with its
// cancellation guard, attention.py:138-172), engine.py:501 (band mass rho),
// engine.py:374-402 (ring slot (m-1) % W <- storage-rounded q_pre and the
// prefix summary over [1, max(0, m-r)]).  merge is attention.py:119-135
// (np.logaddexp; the empty summary, lse = -inf, is the identity and is
// returned bit-for-bit).
#pragma once

#include "common.cuh"

namespace mac {

constexpr int kElems = 4;   // d_v elements per lane per pass (d_v <= 128 in one pass)
constexpr int kSplits = 8;  // splits whose partials are loaded in one batch

// Modes of complete_head:
enum : int {
  COMPLETE_RING = 0,    // decode step: merge, output, rho, ring write-back, seq_lens advance
  COMPLETE_FULL = 1,    // full-attention decode: merge and output only
  COMPLETE_EXPORT = 2,  // KV shard: this shard's (piece, band) summaries -> shard_out
  COMPLETE_SHARDS = 3   // KV-sharded step: partials are the gathered shard_parts; as COMPLETE_RING
};

// One warp per (request, q head), 4 heads per CTA.  The merge is latency-bound,
// so memory is touched in two hops: (A) the step's scalars, (B) every partial,
// the cached ring summary and the query row, all issued before any use; the
// algebra then runs from registers.
template <int MODE>
__device__ __forceinline__ void complete_head(const MacDecodeParams& p, int bh, int mode) {
  using kv_t = typename Traits<MODE>::kv_t;
  using A = typename Traits<MODE>::acc_t;
  using S = typename Traits<MODE>::sum_t;
  using D = typename Traits<MODE>::merge_t;  // merge algebra: fp64
  using M = A;
  const int lane = threadIdx.x & 31;
  const Workspace wsl = workspace_layout(p);
  const int32_t* mpos = ws_ptr<const int32_t>(p, wsl.mpos_off);
  const A* part = ws_ptr<const A>(p, wsl.part_off);
  const int b = bh / p.n_q_heads, h = bh % p.n_q_heads;
  const int Hkv = p.n_kv_heads, g = p.n_q_heads / Hkv, kvh = h / g, hl = h % g;
  const int d = p.head_dim, dv = p.head_dim_v, W = p.window, r = p.band, dvp = dv + 1;
  const int* plan_lo = ws_ptr<const int>(p, wsl.lo_off);
  const D NINF = neg_inf<D>();
  const bool full_mode = mode == COMPLETE_FULL || mode == COMPLETE_EXPORT;  // no ring traffic

  // ---- hop A: scalars of this step ----
  const int m = mpos[b];
  const int use = p.force_miss ? 0 : p.use_hit[bh];
  const int pp_raw = p.force_miss ? -1 : p.match_pos[bh];
  const int lo = plan_lo[bh];
  int lo_g = 1 << 30;
  for (int j = lane; j < g; j += 32) lo_g = min(lo_g, plan_lo[b * p.n_q_heads + kvh * g + j]);
  double qv[kElems];  // exact input values  // this lane's slice of the pre-RoPE query (ring write-back)
  if (!full_mode) {
#pragma unroll
    for (int k = 0; k < kElems; ++k) {
      const int e = lane + 32 * k;
      qv[k] = e < d ? load_in(p.q_pre, (int64_t)bh * d + e, p.in_dtype) : 0.0;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lo_g = min(lo_g, __shfl_xor_sync(0xffffffffu, lo_g, o));
  lo_g = min(lo_g, m);
  const int pp = use ? pp_raw : -1;
  Chunking ch = group_chunking(p, m, lo_g);
  const int cpos = m - r;
  const int grp = b * Hkv + kvh;
  {  // the split band's slots come before the plan's (common.cuh band_items)
    const int pnw = __ldcg(ws_ptr<const int>(p, workspace_layout(p).pn_off) + grp);
    if (pnw >> 16) ch.n = group_slots(pnw, m, r);
  }
  const A* pbase = part + ((int64_t)grp * p.max_chunks * g + hl) * 2 * dvp;
  int64_t cstride = (int64_t)g * 2 * dvp;
  if (mode == COMPLETE_SHARDS) {  // one (piece, band) pair per shard, rank order
    pbase = static_cast<const A*>(p.shard_parts) + (int64_t)bh * 2 * dvp;
    cstride = (int64_t)p.batch * p.n_q_heads * 2 * dvp;
    ch.n = p.n_shards;
  }
  const S* racc = static_cast<const S*>(p.ring_acc);
  const S* rlse = static_cast<const S*>(p.ring_lse);
  const int64_t cslot = use ? (int64_t)bh * W + (pp - 1) % W : 0;

  // ---- hop B: cached summary + split lse values ----
  const D La = (use && mode != COMPLETE_EXPORT) ? (D)rlse[cslot] : NINF;
  A lse_p[kSplits], lse_b[kSplits];
#pragma unroll
  for (int i = 0; i < kSplits; ++i) {
    const bool ok = i < ch.n;
    lse_p[i] = ok ? __ldcg(pbase + (int64_t)i * cstride + dv) : neg_inf<A>();
    lse_b[i] = ok ? __ldcg(pbase + (int64_t)i * cstride + dvp + dv) : neg_inf<A>();
  }
  // log-sum-exp over all splits (splits beyond kSplits: strided loop, rare)
  D mp = NINF, mb = NINF;
#pragma unroll
  for (int i = 0; i < kSplits; ++i) { mp = fmax(mp, (D)lse_p[i]); mb = fmax(mb, (D)lse_b[i]); }
  for (int c = kSplits + lane; c < ch.n; c += 32) {
    mp = fmax(mp, (D)__ldcg(pbase + (int64_t)c * cstride + dv));
    mb = fmax(mb, (D)__ldcg(pbase + (int64_t)c * cstride + dvp + dv));
  }
  if (ch.n > kSplits) { mp = warp_max(mp); mb = warp_max(mb); }
  D sp = 0.0, sb = 0.0;
#pragma unroll
  for (int i = 0; i < kSplits; ++i) {
    if (mp != NINF && (D)lse_p[i] != NINF) sp += fexp((D)lse_p[i] - mp);
    if (mb != NINF && (D)lse_b[i] != NINF) sb += fexp((D)lse_b[i] - mb);
  }
  if (ch.n > kSplits) {
    D sp2 = 0.0, sb2 = 0.0;
    for (int c = kSplits + lane; c < ch.n; c += 32) {
      const D l1 = (D)__ldcg(pbase + (int64_t)c * cstride + dv);
      const D l2 = (D)__ldcg(pbase + (int64_t)c * cstride + dvp + dv);
      if (l1 != NINF) sp2 += fexp(l1 - mp);
      if (l2 != NINF) sb2 += fexp(l2 - mb);
    }
    sp += warp_sum(sp2);
    sb += warp_sum(sb2);
  }
  const D Lp = mp == NINF ? NINF : mp + flog(sp);  // piece
  const D Lb = mb == NINF ? NINF : mb + flog(sb);  // band

  // prefix = cached (+) piece, full = prefix (+) band (attention.py:119-135)
  const D Lpre = logaddexp(La, Lp);
  const D Lfull = logaddexp(Lpre, Lb);
  const D wa = La == NINF ? (D)0 : fexp(La - Lpre);
  const D wp = Lp == NINF ? (D)0 : fexp(Lp - Lpre);
  const D wpre = Lpre == NINF ? (D)0 : fexp(Lpre - Lfull);
  const D wb = Lb == NINF ? (D)0 : fexp(Lb - Lfull);

  // token counts (for remove() and rho): band = [max(lo, cpos+1), m]
  const int bstart = lo > cpos + 1 ? lo : cpos + 1;
  const int bcount = m - bstart + 1 > 0 ? m - bstart + 1 : 0;
  const int pcount = m - bcount;

  // optional downdate prefix = remove(full, band) (engine.py:474-478, 494-498)
  int do_remove = 0, fell_back = 0;
  D Lrem = NINF, wr_full = 0, wr_band = 0;
  if (!full_mode && p.downdate == MAC_DOWNDATE_REMOVE && bcount > 0 && (use || pcount > 0)) {
    if (bcount == m) {
      if (Lb == Lfull) { do_remove = 1; Lrem = NINF; }  // whole == band: empty prefix
      else fell_back = 1;
    } else {
      const D diff = Lfull - Lb;
      if (diff < p.eps_cancel) fell_back = 1;  // CancellationError (or mass exceeded) -> keep split
      else {
        do_remove = 1;
        Lrem = Lb + flog(fexpm1(diff));
        wr_full = fexp(Lfull - Lrem);
        wr_band = fexp(Lb - Lrem);
      }
    }
  }

  S* out = static_cast<S*>(p.out);
  kv_t* rq = static_cast<kv_t*>(p.ring_q);
  S* racc_w = static_cast<S*>(p.ring_acc);
  const int64_t wslot = (int64_t)bh * W + (m - 1) % W;
  for (int e0 = 0; e0 < dv; e0 += 32 * kElems) {
    // ---- hop B (vectors): cached acc and every split's acc slice, all in flight together ----
    D aacc[kElems];
#pragma unroll
    for (int k = 0; k < kElems; ++k) {
      const int e = e0 + lane + 32 * k;
      aacc[k] = (use && mode != COMPLETE_EXPORT && e < dv) ? (D)racc[cslot * dv + e] : (D)0;
    }
    M pacc[kElems] = {0, 0, 0, 0}, bacc[kElems] = {0, 0, 0, 0};
    const M Lpm = (M)Lp, Lbm = (M)Lb;
    for (int cb = 0; cb < ch.n; cb += kSplits) {
      A xp[kSplits][kElems], xb[kSplits][kElems];
      M wpc[kSplits], wbc[kSplits];
#pragma unroll
      for (int i = 0; i < kSplits; ++i) {
        const int c = cb + i;
        const bool ok = c < ch.n;
        const A* row = pbase + (int64_t)c * cstride;
#pragma unroll
        for (int k = 0; k < kElems; ++k) {
          const int e = e0 + lane + 32 * k;
          xp[i][k] = (ok && e < dv) ? __ldcg(row + e) : (A)0;
          xb[i][k] = (ok && e < dv) ? __ldcg(row + dvp + e) : (A)0;
        }
        const M l1 = cb == 0 ? (M)lse_p[i] : (ok ? (M)__ldcg(row + dv) : neg_inf<M>());
        const M l2 = cb == 0 ? (M)lse_b[i] : (ok ? (M)__ldcg(row + dvp + dv) : neg_inf<M>());
        wpc[i] = (l1 == neg_inf<M>() || Lp == NINF) ? (M)0 : fexp(l1 - Lpm);
        wbc[i] = (l2 == neg_inf<M>() || Lb == NINF) ? (M)0 : fexp(l2 - Lbm);
      }
#pragma unroll
      for (int i = 0; i < kSplits; ++i)
#pragma unroll
        for (int k = 0; k < kElems; ++k) {
          pacc[k] += (M)xp[i][k] * wpc[i];
          bacc[k] += (M)xb[i][k] * wbc[i];
        }
    }
#pragma unroll
    for (int k = 0; k < kElems; ++k) {
      const int e = e0 + lane + 32 * k;
      if (e >= dv) continue;
      // merge keeps an empty side's partner bit-exact (weight exp(0) == 1)
      const D pk = (D)pacc[k], bk = (D)bacc[k];
      if (mode == COMPLETE_EXPORT) {
        S* so = static_cast<S*>(p.shard_out) + (int64_t)bh * 2 * dvp;
        so[e] = (S)pk;
        so[dvp + e] = (S)bk;
        continue;
      }
      const D pre = (La == NINF) ? pk : (Lp == NINF ? aacc[k] : aacc[k] * wa + pk * wp);
      const D full = (Lpre == NINF) ? bk : (Lb == NINF ? pre : pre * wpre + bk * wb);
      out[(int64_t)bh * dv + e] = (S)full;
      if (!full_mode) {
        if (p.cached_acc) static_cast<S*>(p.cached_acc)[(int64_t)bh * dv + e] = (S)aacc[k];
        D ring_v = pre;
        if (do_remove) ring_v = (Lrem == NINF) ? (D)0 : full * wr_full - bk * wr_band;
        racc_w[wslot * dv + e] = (S)ring_v;
      }
    }
  }
  if (!full_mode) {  // every lane read its cached slice above, before this slot can be overwritten
    __syncwarp();
#pragma unroll
    for (int k = 0; k < kElems; ++k) {
      const int e = lane + 32 * k;
      if (e < d) rq[wslot * d + e] = from_f64<kv_t>(qv[k]);
    }
    if (MODE == MAC_MODE_BF16 && d == 128 && p.ring_qp && lane < MAC_PLANAR_DIMS)  // the scan's planar copy
      static_cast<kv_t*>(p.ring_qp)[wslot * MAC_PLANAR_DIMS + lane] = from_f64<kv_t>(qv[0]);
    for (int e = lane + 32 * kElems; e < d; e += 32)  // d > 128
      rq[wslot * d + e] = from_f64<kv_t>(load_in(p.q_pre, (int64_t)bh * d + e, p.in_dtype));
  }
  if (mode == COMPLETE_EXPORT) {
    if (lane == 0) {
      S* so = static_cast<S*>(p.shard_out) + (int64_t)bh * 2 * dvp;
      so[dv] = (S)Lp;
      so[dvp + dv] = (S)Lb;
    }
    return;
  }
  if (lane == 0) {
    static_cast<S*>(p.full_lse)[bh] = (S)Lfull;
    if (!full_mode) {
      const D lse_store = do_remove ? Lrem : Lpre;
      static_cast<S*>(p.ring_lse)[wslot] = (S)lse_store;
      static_cast<S*>(p.band_mass)[bh] = (S)(bcount > 0 ? fexp(Lb - Lfull) : (D)0);
      if (p.cached_lse) static_cast<S*>(p.cached_lse)[bh] = (S)La;
      if (p.fallbacks) p.fallbacks[bh] = fell_back;
    }
    if (h == 0) p.seq_lens[b] = m;
  }
}

}  // namespace mac
