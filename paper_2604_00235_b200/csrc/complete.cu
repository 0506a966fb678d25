// K3 — complete: merge cached(p) (+) piece (+) band, emit the output, and write
// the ring entry back (the paper's "rectify-append").
//
// Reference: engine.py:468-479 (prefix = merge(cached, piece1); full =
// merge(prefix, band); out = finalize(full)), engine.py:486-499 (miss),
// engine.py:474-478,494-498 (optional remove() downdate with its
// cancellation guard, attention.py:138-172), engine.py:501 (band mass rho),
// engine.py:374-402 (ring slot (m-1) % W <- storage-rounded q_pre and the
// prefix summary over [1, max(0, m-r)]).  merge is attention.py:119-135
// (np.logaddexp; the empty summary, lse = -inf, is the identity and is
// returned bit-for-bit).
//
// One CTA per (request, q head); threads across d_v.  Scalars (lse values,
// weights) are evaluated in fp64, vectors in fp64 then rounded once.
#include "common.cuh"

namespace mac {

// block-wide max / sum over 128 threads
__device__ __forceinline__ double block_reduce(double v, bool is_max, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double x = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmax(v, x) : v + x;
  }
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  v = red[0];
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) v = is_max ? fmax(v, red[w]) : v + red[w];
  return v;
}

// merge n split partials of one set: lse into L, per-split weights exp(l_c - L) into wts
template <typename A>
__device__ __forceinline__ double merge_weights(const A* base, int n, int stride, double* wts, double* red) {
  double mx = -CUDART_INF;
  for (int c = threadIdx.x; c < n; c += blockDim.x) mx = fmax(mx, (double)base[(int64_t)c * stride]);
  mx = block_reduce(mx, true, red);
  if (mx == -CUDART_INF) {
    for (int c = threadIdx.x; c < n; c += blockDim.x) wts[c] = 0.0;
    return mx;
  }
  double sum = 0.0;
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    const double l = (double)base[(int64_t)c * stride];
    sum += l == -CUDART_INF ? 0.0 : exp(l - mx);
  }
  sum = block_reduce(sum, false, red);
  const double L = mx + log(sum);
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    const double l = (double)base[(int64_t)c * stride];
    wts[c] = l == -CUDART_INF ? 0.0 : exp(l - L);
  }
  return L;
}

template <int MODE>
__global__ void __launch_bounds__(128) complete_kernel(MacDecodeParams p, const int32_t* __restrict__ mpos,
                                                       const typename Traits<MODE>::acc_t* __restrict__ part,
                                                       int full_mode) {
  using kv_t = typename Traits<MODE>::kv_t;
  using A = typename Traits<MODE>::acc_t;
  using S = typename Traits<MODE>::sum_t;
  extern __shared__ double wsm[];  // [2][max_chunks] split weights
  __shared__ double red[32];
  const int bh = blockIdx.x;
  const int b = bh / p.n_q_heads, h = bh % p.n_q_heads;
  const int Hkv = p.n_kv_heads, g = p.n_q_heads / Hkv, kvh = h / g, hl = h % g;
  const int d = p.head_dim, dv = p.head_dim_v, W = p.window, r = p.band, dvp = dv + 1;
  const int m = mpos[b];
  const int* plan_lo = ws_ptr<const int>(p, workspace_layout(p).lo_off);

  int lo_g = m;
  for (int j = 0; j < g; ++j) {
    const int l = plan_lo[b * p.n_q_heads + kvh * g + j];
    lo_g = l < lo_g ? l : lo_g;
  }
  const int lo_first = grid_start(lo_g, p.kv_offset);
  const Chunking ch = chunking(m - lo_first + 1, p.max_chunks, p.min_chunk);
  const int use = p.force_miss ? 0 : p.use_hit[bh];
  const int pp = use ? p.match_pos[bh] : -1;
  const int lo = plan_lo[bh];
  const int cpos = m - r;

  // partial slots of this head: (grp, c, hl, set) -> stride between splits
  const int grp = b * Hkv + kvh;
  const A* pbase = part + ((int64_t)grp * p.max_chunks * g + hl) * 2 * dvp;
  const int cstride = g * 2 * dvp;
  double* wp_s = wsm;
  double* wb_s = wsm + p.max_chunks;
  const double Lp = merge_weights(pbase + dv, ch.n, cstride, wp_s, red);         // piece
  const double Lb = merge_weights(pbase + dvp + dv, ch.n, cstride, wb_s, red);   // band
  __syncthreads();

  // cached summary at p (covers [1, max(0, p-r)]); empty on a miss
  const S* racc = static_cast<const S*>(p.ring_acc);
  const S* rlse = static_cast<const S*>(p.ring_lse);
  double La = -CUDART_INF;
  int64_t cslot = 0;
  if (use) {
    cslot = (int64_t)bh * W + (pp - 1) % W;
    La = (double)rlse[cslot];
  }
  // prefix = cached (+) piece, full = prefix (+) band (attention.py:119-135)
  const double Lpre = logaddexp(La, Lp);
  const double Lfull = logaddexp(Lpre, Lb);
  const double wa = La == -CUDART_INF ? 0.0 : exp(La - Lpre);
  const double wp = Lp == -CUDART_INF ? 0.0 : exp(Lp - Lpre);
  const double wpre = Lpre == -CUDART_INF ? 0.0 : exp(Lpre - Lfull);
  const double wb = Lb == -CUDART_INF ? 0.0 : exp(Lb - Lfull);

  // token counts (for remove() and rho): band = [max(lo, cpos+1), m]
  int bstart = lo > cpos + 1 ? lo : cpos + 1;
  const int bcount = m - bstart + 1 > 0 ? m - bstart + 1 : 0;
  const int pcount = m - bcount;

  // optional downdate prefix = remove(full, band) (engine.py:474-478, 494-498)
  int do_remove = 0, fell_back = 0;
  double Lrem = -CUDART_INF, wr_full = 0.0, wr_band = 0.0;
  if (!full_mode && p.downdate == MAC_DOWNDATE_REMOVE && bcount > 0 && (use || pcount > 0)) {
    if (bcount == m) {
      if (Lb == Lfull) { do_remove = 1; Lrem = -CUDART_INF; }  // whole == band: empty prefix
      else fell_back = 1;
    } else {
      double diff = Lfull - Lb;
      if (diff < p.eps_cancel) fell_back = 1;  // CancellationError (or mass exceeded) -> keep split
      else {
        do_remove = 1;
        Lrem = Lb + log(expm1(diff));
        wr_full = exp(Lfull - Lrem);
        wr_band = exp(Lb - Lrem);
      }
    }
  }

  S* out = static_cast<S*>(p.out);
  kv_t* rq = static_cast<kv_t*>(p.ring_q);
  S* racc_w = static_cast<S*>(p.ring_acc);
  const int64_t wslot = (int64_t)bh * W + (m - 1) % W;
  for (int e = threadIdx.x; e < dv; e += blockDim.x) {
    double pacc = 0.0, bacc = 0.0;
    for (int c = 0; c < ch.n; ++c) {
      const A* pc = pbase + (int64_t)c * cstride;
      const double fp = wp_s[c], fb = wb_s[c];
      if (fp != 0.0) pacc += (double)pc[e] * fp;
      if (fb != 0.0) bacc += (double)pc[dvp + e] * fb;
    }
    double aacc = use ? (double)racc[cslot * dv + e] : 0.0;
    // merge keeps an empty side's partner bit-exact (weight exp(0) == 1)
    double pre = (La == -CUDART_INF) ? pacc : (Lp == -CUDART_INF ? aacc : aacc * wa + pacc * wp);
    double full = (Lpre == -CUDART_INF) ? bacc : (Lb == -CUDART_INF ? pre : pre * wpre + bacc * wb);
    out[(int64_t)bh * dv + e] = (S)full;
    if (!full_mode) {
      if (p.cached_acc) static_cast<S*>(p.cached_acc)[(int64_t)bh * dv + e] = (S)aacc;
      double ring_v = pre;
      if (do_remove) ring_v = (Lrem == -CUDART_INF) ? 0.0 : full * wr_full - bacc * wr_band;
      racc_w[wslot * dv + e] = (S)ring_v;
    }
  }
  __syncthreads();  // cached summary fully read before the same slot may be overwritten
  if (!full_mode) {
    for (int k = threadIdx.x; k < d; k += blockDim.x)
      rq[wslot * d + k] = from_f64<kv_t>(load_in(p.q_pre, (int64_t)bh * d + k, p.in_dtype));
  }
  if (threadIdx.x == 0) {
    static_cast<S*>(p.full_lse)[bh] = (S)Lfull;
    if (!full_mode) {
      double lse_store = do_remove ? Lrem : Lpre;
      static_cast<S*>(p.ring_lse)[wslot] = (S)lse_store;
      static_cast<S*>(p.band_mass)[bh] = (S)(bcount > 0 ? exp(Lb - Lfull) : 0.0);
      if (p.cached_lse) static_cast<S*>(p.cached_lse)[bh] = (S)La;
      if (p.fallbacks) p.fallbacks[bh] = fell_back;
    }
    if (h == 0) p.seq_lens[b] = m;
    if (bh == 0) ws_ptr<unsigned int>(p, workspace_layout(p).ctr_off)[0] = 0u;  // work list consumed
  }
}

template <int MODE>
cudaError_t launch_complete(const MacDecodeParams& p, cudaStream_t st, int full_mode) {
  Workspace w = workspace_layout(p);
  char* ws = static_cast<char*>(p.workspace);
  complete_kernel<MODE><<<p.batch * p.n_q_heads, 128, 2 * sizeof(double) * p.max_chunks, st>>>(
      p, reinterpret_cast<const int32_t*>(ws + w.mpos_off),
      reinterpret_cast<const typename Traits<MODE>::acc_t*>(ws + w.part_off), full_mode);
  return cudaGetLastError();
}

template cudaError_t launch_complete<MAC_MODE_F32>(const MacDecodeParams&, cudaStream_t, int);
template cudaError_t launch_complete<MAC_MODE_BF16>(const MacDecodeParams&, cudaStream_t, int);
template cudaError_t launch_complete<MAC_MODE_F64>(const MacDecodeParams&, cudaStream_t, int);

}  // namespace mac
