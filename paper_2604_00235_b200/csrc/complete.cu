// K3 — complete, standalone kernel: one warp per (request, q head), 4 heads
// per CTA (the per-head logic is complete.cuh), and its lean bf16 d = 128 form for
// the decode step (complete_bf16_kernel).
#include "complete.cuh"

namespace mac {

template <int MODE>
__global__ void __launch_bounds__(128) complete_kernel(MacDecodeParams p, int full_mode) {
  // programmatic dependent launch: the grid is set up while the amend kernel drains
  TL_MARK(p, TL_COMPLETE_IN);
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  TL_MARK(p, TL_COMPLETE_WAITED);
  const int bh = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (bh < p.batch * p.n_q_heads) complete_head<MODE>(p, bh, full_mode);
#ifdef MAC_TIMELINE
  __syncthreads();
#endif
  TL_MARK(p, TL_COMPLETE_OUT);
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // work list consumed: list length and amend claim counter
    unsigned int* ctr = ws_ptr<unsigned int>(p, workspace_layout(p).ctr_off);
    ctr[0] = 0u;
    ctr[1] = 0u;
    ctr[8] = 0u;
  }
}

// The decode step's complete on the bf16 d = d_v = 128 path: complete_head's algebra
// (engine.py:468-502, attention.py:119-135, rectify_append engine.py:374-402) in a lean
// register budget, with two memory hops instead of three: (A) the step's scalars and the
// query row, (B) the cached ring summary and the first 8 splits' partials (lse and acc
// together).  Splits beyond 8 (long miss spans) merge online in further batches of 8.
__global__ void __launch_bounds__(128) complete_bf16_kernel(MacDecodeParams p) {
  TL_MARK(p, TL_COMPLETE_IN);
  const int lane = threadIdx.x & 31;
  const int bh = blockIdx.x * 4 + (threadIdx.x >> 5);
  const Workspace wsl = workspace_layout(p);
  const bool live = bh < p.batch * p.n_q_heads;
  // Everything before the grid-dependency wait was written by kernels that finished before
  // this grid could launch (the front and verify kernels; earlier steps for the ring), so
  // hop A and the cached ring summary load while the amend kernel drains (L2 loads: nothing
  // stale in L1).  Only the amend's partials are read after the wait.
  if (!live) {
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      unsigned int* ctr = ws_ptr<unsigned int>(p, wsl.ctr_off);
      ctr[0] = 0u;
      ctr[1] = 0u;
      ctr[8] = 0u;
    }
  }
  if (live) {
    const float NINF = -CUDART_INF_F;
    const int b = bh / p.n_q_heads, h = bh % p.n_q_heads;
    const int Hkv = p.n_kv_heads, g = p.n_q_heads / Hkv, kvh = h / g, hl = h % g;
    const int W = p.window, r = p.band;
    // ---- hop A ----
    const int m = __ldcg(ws_ptr<const int32_t>(p, wsl.mpos_off) + b);
    const int use = p.force_miss ? 0 : __ldcg(p.use_hit + bh);
    const int pp = __ldcg(p.match_pos + bh);
    const int* plan_lo = ws_ptr<const int>(p, wsl.lo_off);
    const int lo = __ldcg(plan_lo + bh);
    int lo_g = lane < g ? __ldcg(plan_lo + b * p.n_q_heads + kvh * g + lane) : (1 << 30);
    double qv[4];
#pragma unroll
    const void* qs = q_src(p);
    for (int k = 0; k < 4; ++k) qv[k] = load_in(qs, (int64_t)bh * 128 + lane + 32 * k, p.in_dtype);
    lo_g = min(lo_g, __shfl_xor_sync(0xffffffffu, lo_g, 1));
    lo_g = min(lo_g, __shfl_xor_sync(0xffffffffu, lo_g, 2));
    lo_g = min(lo_g, __shfl_xor_sync(0xffffffffu, lo_g, 4));
    lo_g = min(lo_g, __shfl_xor_sync(0xffffffffu, lo_g, 8));
    lo_g = min(lo_g, __shfl_xor_sync(0xffffffffu, lo_g, 16));
    lo_g = min(lo_g, m);
    const int grp = b * Hkv + kvh;
    // partial slots: the plan's split grid, after the split band's slots when the plan says so
    const int pnw = __ldcg(ws_ptr<const int>(p, wsl.pn_off) + grp);
    const int nsl = (pnw >> 16) ? group_slots(pnw, m, r) : group_chunking(p, m, lo_g).n;
    const int cpos = m - r;
    const float* pbase = ws_ptr<const float>(p, wsl.part_off) + ((int64_t)grp * p.max_chunks * g + hl) * 2 * 129;
    const int64_t cstride = (int64_t)g * 2 * 129;
    const float* racc = static_cast<const float*>(p.ring_acc);
    const float* rlse = static_cast<const float*>(p.ring_lse);
    const int64_t cslot = use ? (int64_t)bh * W + (pp - 1) % W : 0;
    // ---- hop B: cached summary, then the splits in batches of 8 (online log-sum-exp) ----
    const float La = use ? __ldcg(rlse + cslot) : NINF;
    float aacc[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) aacc[k] = use ? __ldcg(racc + cslot * 128 + lane + 32 * k) : 0.f;
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    TL_MARK(p, TL_COMPLETE_WAITED);
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // work list consumed: list length and amend claim counter
      unsigned int* ctr = ws_ptr<unsigned int>(p, wsl.ctr_off);
      ctr[0] = 0u;
      ctr[1] = 0u;
      ctr[8] = 0u;
    }
    float Mp = NINF, Sp = 0.f, Mb = NINF, Sb = 0.f, ap[4] = {0.f, 0.f, 0.f, 0.f}, ab[4] = {0.f, 0.f, 0.f, 0.f};
    for (int cb = 0; cb < nsl; cb += 8) {
      float lp[8], lb[8], xp[8][4], xb[8][4];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const bool ok = cb + i < nsl;
        const float* row = pbase + (int64_t)(cb + i) * cstride;
        lp[i] = ok ? __ldcg(row + 128) : NINF;
        lb[i] = ok ? __ldcg(row + 129 + 128) : NINF;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          xp[i][k] = ok ? __ldcg(row + lane + 32 * k) : 0.f;
          xb[i][k] = ok ? __ldcg(row + 129 + lane + 32 * k) : 0.f;
        }
      }
      float np = Mp, nb = Mb;
#pragma unroll
      for (int i = 0; i < 8; ++i) { np = fmaxf(np, lp[i]); nb = fmaxf(nb, lb[i]); }
      if (np != NINF) {
        const float sc = Mp == NINF ? 0.f : fexp(Mp - np);
        Sp *= sc;
#pragma unroll
        for (int k = 0; k < 4; ++k) ap[k] *= sc;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float wgt = lp[i] == NINF ? 0.f : fexp(lp[i] - np);
          Sp += wgt;
#pragma unroll
          for (int k = 0; k < 4; ++k) ap[k] += wgt * xp[i][k];
        }
        Mp = np;
      }
      if (nb != NINF) {
        const float sc = Mb == NINF ? 0.f : fexp(Mb - nb);
        Sb *= sc;
#pragma unroll
        for (int k = 0; k < 4; ++k) ab[k] *= sc;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float wgt = lb[i] == NINF ? 0.f : fexp(lb[i] - nb);
          Sb += wgt;
#pragma unroll
          for (int k = 0; k < 4; ++k) ab[k] += wgt * xb[i][k];
        }
        Mb = nb;
      }
    }
    const float Lp = Mp == NINF ? NINF : Mp + flog(Sp);  // piece
    const float Lb = Mb == NINF ? NINF : Mb + flog(Sb);  // band
    const float ip = Sp > 0.f ? 1.f / Sp : 0.f, ib = Sb > 0.f ? 1.f / Sb : 0.f;
    // the summary algebra: fp32 for the split prefix (as the partials), fp64 with the remove()
    // downdate, whose cancellation fp32 would amplify into the stored prefix (as f32 storage)
    float* out = static_cast<float*>(p.out);
    float* racc_w = static_cast<float*>(p.ring_acc);
    __nv_bfloat16* rq = static_cast<__nv_bfloat16*>(p.ring_q);
    const int64_t wslot = (int64_t)bh * W + (m - 1) % W;
    // token counts (remove() and rho): band = [max(lo, cpos+1), m]
    const int bstart = lo > cpos + 1 ? lo : cpos + 1;
    const int bcount = m - bstart + 1 > 0 ? m - bstart + 1 : 0;
    const int pcount = m - bcount;
    auto finish = [&](auto zero) {
      using T = decltype(zero);
      const T TINF = -(T)CUDART_INF;
      const T dLa = La, dLp = Lp, dLb = Lb;
      // prefix = cached (+) piece, full = prefix (+) band (attention.py:119-135)
      const T Lpre = logaddexp(dLa, dLp);
      const T Lfull = logaddexp(Lpre, dLb);
      const T wa = dLa == TINF ? zero : fexp(dLa - Lpre);
      const T wp = dLp == TINF ? zero : fexp(dLp - Lpre);
      const T wpre = Lpre == TINF ? zero : fexp(Lpre - Lfull);
      const T wb = dLb == TINF ? zero : fexp(dLb - Lfull);
      // optional downdate prefix = remove(full, band) (engine.py:474-478, 494-498)
      int do_remove = 0, fell_back = 0;
      T Lrem = TINF, wr_full = zero, wr_band = zero;
      if (p.downdate == MAC_DOWNDATE_REMOVE && bcount > 0 && (use || pcount > 0)) {
        if (bcount == m) {
          if (dLb == Lfull) { do_remove = 1; Lrem = TINF; }
          else fell_back = 1;
        } else {
          const T diff = Lfull - dLb;
          if (diff < (T)p.eps_cancel) fell_back = 1;
          else {
            do_remove = 1;
            Lrem = dLb + flog(fexpm1(diff));
            wr_full = fexp(Lfull - Lrem);
            wr_band = fexp(dLb - Lrem);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int e = lane + 32 * k;
        const T pk = ap[k] * ip, bk = ab[k] * ib;  // merge keeps an empty side's partner exact
        const T pre = (dLa == TINF) ? pk : (dLp == TINF ? (T)aacc[k] : aacc[k] * wa + pk * wp);
        const T full = (Lpre == TINF) ? bk : (dLb == TINF ? pre : pre * wpre + bk * wb);
        out[(int64_t)bh * 128 + e] = (float)full;
        if (p.out_bf16) static_cast<__nv_bfloat16*>(p.out_bf16)[(int64_t)bh * 128 + e] = __float2bfloat16_rn((float)full);
        if (p.cached_acc) static_cast<float*>(p.cached_acc)[(int64_t)bh * 128 + e] = aacc[k];
        racc_w[wslot * 128 + e] = (float)(do_remove ? ((Lrem == TINF) ? zero : full * wr_full - bk * wr_band) : pre);
      }
      if (lane == 0) {
        static_cast<float*>(p.full_lse)[bh] = (float)Lfull;
        static_cast<float*>(p.ring_lse)[wslot] = (float)(do_remove ? Lrem : Lpre);
        static_cast<float*>(p.band_mass)[bh] = bcount > 0 ? (float)fexp(dLb - Lfull) : 0.f;
        if (p.fallbacks) p.fallbacks[bh] = fell_back;
      }
    };
    if (p.downdate == MAC_DOWNDATE_REMOVE) finish(0.0);
    else finish(0.f);
    __syncwarp();  // every lane read its cached slice above, before this slot can be overwritten
#pragma unroll
    for (int k = 0; k < 4; ++k) rq[wslot * 128 + lane + 32 * k] = from_f64<__nv_bfloat16>(qv[k]);
    if (p.ring_qp && lane < MAC_PLANAR_DIMS)  // the scan's planar copy of dims 0..P-1
      static_cast<__nv_bfloat16*>(p.ring_qp)[wslot * MAC_PLANAR_DIMS + lane] = from_f64<__nv_bfloat16>(qv[0]);
    if (lane == 0) {
      if (p.cached_lse) static_cast<float*>(p.cached_lse)[bh] = La;
      if (h == 0) p.seq_lens[b] = m;
    }
  }
  // heads whose raw match missed this step (the case that makes the two-pass verify walk the
  // ring; gate-forced misses do not), counted fire-and-forget (RED); a forced-miss step (prefill,
  // force_miss) is not counted at all.  A later step's append warps publish the count to
  // `feedback` (front.cuh).
  if (p.feedback && !p.force_miss) {
    if (live && lane == 0 && !__ldcg(p.match_hit + bh)) atomicAdd(ws_ptr<unsigned>(p, wsl.ctr_off) + 4, 1u);
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(ws_ptr<unsigned>(p, wsl.ctr_off) + 6, 1u);
  }
#ifdef MAC_TIMELINE
  __syncthreads();
#endif
  TL_MARK(p, TL_COMPLETE_OUT);
}

template <int MODE>
cudaError_t launch_complete(const MacDecodeParams& p, cudaStream_t st, int full_mode) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((p.batch * p.n_q_heads + 3) / 4);
  cfg.blockDim = dim3(128);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (MODE == MAC_MODE_BF16 && full_mode == COMPLETE_RING && p.head_dim == 128 && p.head_dim_v == 128)
    return cudaLaunchKernelEx(&cfg, complete_bf16_kernel, p);
  return cudaLaunchKernelEx(&cfg, complete_kernel<MODE>, p, full_mode);
}

template cudaError_t launch_complete<MAC_MODE_F32>(const MacDecodeParams&, cudaStream_t, int);
template cudaError_t launch_complete<MAC_MODE_BF16>(const MacDecodeParams&, cudaStream_t, int);
template cudaError_t launch_complete<MAC_MODE_F64>(const MacDecodeParams&, cudaStream_t, int);

}  // namespace mac
