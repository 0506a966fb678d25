// Diagnostics beside the decode step: device-side decision
// statistics and the offline stored-prefix mass-bound check.
//
// step_stats_kernel — DecodeMetrics.record_hit / record_miss (engine.py:188-205)
//   and the GQA group span (engine.py:66-77 group_kv_span, used at :525-528),
//   accumulated on the device per q head and per kv head over the batch, so a
//   serving loop reads acceptance / skip ratio / kv fraction / mean gap / mean
//   band mass per (layer, head) without copying decisions to the host each step.
//   One warp per (request, kv group); lanes are the group's q heads.
//
// mass_bound_kernel — mass_bound_check (engine.py:246-281): for a hit at p,
//   compare the drift of the reused non-band prefix, lhs = ||(a_p - a_m)[:cut] V||,
//   with its first-order bound rhs = expm1(dl) (1 - rho) E_ap[||v||], both
//   softmaxes taken over [1, p], cut = max(0, p - band).  Offline (fp64, one CTA
//   per item, two passes over the item's keys: maxima + drift, then the sums).
#include "common.cuh"

namespace mac {

__device__ __forceinline__ int warp_min(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <int MODE>
__global__ void __launch_bounds__(256) step_stats_kernel(MacDecodeParams p, double* __restrict__ hs,
                                                         double* __restrict__ gs) {
  using S = typename Traits<MODE>::sum_t;
  const int lane = threadIdx.x & 31;
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int Hkv = p.n_kv_heads, Hq = p.n_q_heads, g = Hq / Hkv, r = p.band;
  if (w >= p.batch * Hkv) return;
  const int b = w / Hkv, kvh = w % Hkv;
  const int m = p.seq_lens[b];  // the step advanced seq_lens to its position m
  int floor_g = 1 << 30;
  for (int hl = lane; hl < g; hl += 32) {
    const int h = kvh * g + hl, bh = b * Hq + h;
    const int hit = p.match_hit[bh], use = p.use_hit[bh], pos = p.match_pos[bh];
    double* s = hs + (int64_t)h * MAC_STAT_COUNT;
    atomicAdd(s + MAC_STAT_STEPS, 1.0);
    atomicAdd(s + MAC_STAT_KV_FULL, (double)m);
    atomicAdd(s + MAC_STAT_CANDIDATES, (double)p.match_scanned[bh]);
    atomicAdd(s + MAC_STAT_RHO_SUM, (double)static_cast<const S*>(p.band_mass)[bh]);
    if (use) {
      const int skipped = pos - r > 0 ? pos - r : 0;
      atomicAdd(s + MAC_STAT_HITS, 1.0);
      atomicAdd(s + MAC_STAT_SKIP_SUM, (double)skipped / (double)m);
      atomicAdd(s + MAC_STAT_KV_READ, (double)(m - skipped));
      atomicAdd(s + MAC_STAT_GAP_SUM, (double)(m - pos));
    } else {
      atomicAdd(s + MAC_STAT_KV_READ, (double)m);
    }
    if (hit && !use) atomicAdd(s + MAC_STAT_FORCED, 1.0);
    if (p.fallbacks && p.fallbacks[bh]) atomicAdd(s + MAC_STAT_FALLBACKS, 1.0);
    // group_kv_span: the raw match decides the floor (misses contribute 0)
    floor_g = min(floor_g, hit ? (pos - r > 0 ? pos - r : 0) : 0);
  }
  floor_g = warp_min(floor_g);
  if (lane == 0) {
    atomicAdd(gs + (int64_t)kvh * MAC_GSTAT_COUNT + MAC_GSTAT_KV_TOKENS, (double)(m - floor_g));
    atomicAdd(gs + (int64_t)kvh * MAC_GSTAT_COUNT + MAC_GSTAT_KV_TOTAL, (double)m);
  }
}

template <int MODE>
cudaError_t launch_step_stats(const MacDecodeParams& p, double* hs, double* gs, cudaStream_t st) {
  const int warps = p.batch * p.n_kv_heads;
  step_stats_kernel<MODE><<<(warps + 7) / 8, 256, 0, st>>>(p, hs, gs);
  return cudaGetLastError();
}

template cudaError_t launch_step_stats<MAC_MODE_F32>(const MacDecodeParams&, double*, double*, cudaStream_t);
template cudaError_t launch_step_stats<MAC_MODE_BF16>(const MacDecodeParams&, double*, double*, cudaStream_t);
template cudaError_t launch_step_stats<MAC_MODE_F64>(const MacDecodeParams&, double*, double*, cudaStream_t);

// ---------------------------------------------------------------------------
// mass_bound_check (engine.py:246-281)
// ---------------------------------------------------------------------------

constexpr int kMbWarps = 8;
constexpr int kMbMaxE = 8;  // d, d_v <= 256: up to 8 elements per lane

__device__ __forceinline__ double block_reduce(double v, double* sh, bool is_max) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = is_max ? warp_max(v) : warp_sum(v);
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = sh[0];
  for (int i = 1; i < kMbWarps; ++i) t = is_max ? fmax(t, sh[i]) : t + sh[i];
  return t;
}

template <int MODE>
__global__ void __launch_bounds__(kMbWarps * 32) mass_bound_kernel(MacDecodeParams p, MacMassBoundParams mb) {
  using kv_t = typename Traits<MODE>::kv_t;
  __shared__ double sh_red[kMbWarps];
  __shared__ double sh_acc[kMbWarps][2][kMbMaxE * 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int it = blockIdx.x;
  const int b = mb.item_req[it], kvh = mb.item_kv_head[it], pos_m = mb.item_m[it], pp = mb.item_p[it];
  const int d = p.head_dim, dv = p.head_dim_v, Hkv = p.n_kv_heads;
  const int cut = pp - mb.band > 0 ? pp - mb.band : 0;
  double* out = mb.out + 2 * (int64_t)it;
  if (cut == 0) {  // the band covers [1, p]: vacuous (engine.py:272-273)
    if (threadIdx.x == 0) { out[0] = 0.0; out[1] = 0.0; }
    return;
  }
  // the two queries, post-RoPE in fp64 (engine.py:482: q_p rotated at p, q_m at m)
  double qm[kMbMaxE], qp[kMbMaxE];
#pragma unroll
  for (int k = 0; k < kMbMaxE; ++k) {
    const int e = lane + 32 * k;
    qm[k] = 0.0;
    qp[k] = 0.0;
    if (e >= d) continue;
    const double* xm = mb.q_m + (int64_t)it * d;
    const double* xp = mb.q_p + (int64_t)it * d;
    if (mb.rotate) {
      const int j = e >> 1;
      double sm, cm, sp, cp;
      sincos((double)pos_m * p.rope_freqs[j], &sm, &cm);
      sincos((double)pp * p.rope_freqs[j], &sp, &cp);
      if (e & 1) {
        qm[k] = xm[e - 1] * sm + xm[e] * cm;
        qp[k] = xp[e - 1] * sp + xp[e] * cp;
      } else {
        qm[k] = xm[e] * cm - xm[e + 1] * sm;
        qp[k] = xp[e] * cp - xp[e + 1] * sp;
      }
    } else {
      qm[k] = xm[e];
      qp[k] = xp[e];
    }
  }
  const double scale = 1.0 / sqrt((double)d);
  const kv_t* kc = static_cast<const kv_t*>(p.k_cache);
  const kv_t* vc = static_cast<const kv_t*>(p.v_cache);
  auto logits = [&](int t, double& lp, double& lm) {  // t is 1-based
    const int64_t row = kv_row(p.page_table, p.pages_per_seq, b, t, p.page_size, Hkv, kvh);
    double ap = 0.0, am = 0.0;
#pragma unroll
    for (int k = 0; k < kMbMaxE; ++k) {
      const int e = lane + 32 * k;
      if (e < d) {
        const double kk = to_f64(kc[row * d + e]);
        ap += kk * qp[k];
        am += kk * qm[k];
      }
    }
    lp = warp_sum(ap) * scale;
    lm = warp_sum(am) * scale;
  };

  // pass 1: softmax maxima over [1, p] and the logit drift over the prefix [1, cut]
  double mxp = -INFINITY, mxm = -INFINITY, dl = 0.0;
  for (int t = 1 + wid; t <= pp; t += kMbWarps) {
    double lp, lm;
    logits(t, lp, lm);
    mxp = fmax(mxp, lp);
    mxm = fmax(mxm, lm);
    if (t <= cut) dl = fmax(dl, fabs(lm - lp));
  }
  mxp = block_reduce(mxp, sh_red, true);
  mxm = block_reduce(mxm, sh_red, true);
  dl = block_reduce(dl, sh_red, true);

  // pass 2: partition functions, band share, E[||v||] and the two prefix value sums
  double zp = 0.0, zm = 0.0, zband = 0.0, zpre = 0.0, evs = 0.0;
  double accp[kMbMaxE], accm[kMbMaxE];
#pragma unroll
  for (int k = 0; k < kMbMaxE; ++k) { accp[k] = 0.0; accm[k] = 0.0; }
  for (int t = 1 + wid; t <= pp; t += kMbWarps) {
    double lp, lm;
    logits(t, lp, lm);
    const double ep = exp(lp - mxp), em = exp(lm - mxm);
    zp += ep;
    zm += em;
    if (t > cut) { zband += ep; continue; }
    zpre += ep;
    const int64_t row = kv_row(p.page_table, p.pages_per_seq, b, t, p.page_size, Hkv, kvh);
    double nv = 0.0;
#pragma unroll
    for (int k = 0; k < kMbMaxE; ++k) {
      const int e = lane + 32 * k;
      if (e < dv) {
        const double vv = to_f64(vc[row * dv + e]);
        nv += vv * vv;
        accp[k] += ep * vv;
        accm[k] += em * vv;
      }
    }
    evs += ep * sqrt(warp_sum(nv));
  }
  // lanes carry identical scalar sums (warp-uniform); reduce them once per warp
  if (lane != 0) { zp = zm = zband = zpre = evs = 0.0; }
  zp = block_reduce(zp, sh_red, false);
  zm = block_reduce(zm, sh_red, false);
  zband = block_reduce(zband, sh_red, false);
  zpre = block_reduce(zpre, sh_red, false);
  evs = block_reduce(evs, sh_red, false);
#pragma unroll
  for (int k = 0; k < kMbMaxE; ++k) {
    sh_acc[wid][0][lane + 32 * k] = accp[k];
    sh_acc[wid][1][lane + 32 * k] = accm[k];
  }
  __syncthreads();
  double diff2 = 0.0;
  for (int e = threadIdx.x; e < dv; e += blockDim.x) {
    double sp = 0.0, sm = 0.0;
    for (int w = 0; w < kMbWarps; ++w) { sp += sh_acc[w][0][e]; sm += sh_acc[w][1][e]; }
    const double dlt = sp / zp - sm / zm;
    diff2 += dlt * dlt;
  }
  diff2 = block_reduce(diff2, sh_red, false);
  if (threadIdx.x == 0) {
    const double rho = zband / zp;
    const double prefix_mass = zpre / zp;
    const double ev = prefix_mass > 0.0 ? (evs / zp) / prefix_mass : 0.0;
    out[0] = sqrt(diff2);
    out[1] = expm1(dl) * (1.0 - rho) * ev;
  }
}

template <int MODE>
cudaError_t launch_mass_bound(const MacDecodeParams& p, const MacMassBoundParams& mb, cudaStream_t st) {
  mass_bound_kernel<MODE><<<mb.n_items, kMbWarps * 32, 0, st>>>(p, mb);
  return cudaGetLastError();
}

template cudaError_t launch_mass_bound<MAC_MODE_F32>(const MacDecodeParams&, const MacMassBoundParams&, cudaStream_t);
template cudaError_t launch_mass_bound<MAC_MODE_BF16>(const MacDecodeParams&, const MacMassBoundParams&, cudaStream_t);
template cudaError_t launch_mass_bound<MAC_MODE_F64>(const MacDecodeParams&, const MacMassBoundParams&, cudaStream_t);

}  // namespace mac
