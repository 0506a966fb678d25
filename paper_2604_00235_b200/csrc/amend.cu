// K2 — amend: split-KV partial summaries over [lo, m], cut at m - r.
//
// Reference: engine.py:464-470 (hit: read [lo, m], lo = max(1, p-r+1), two
// summaries split at m-r via _attend_span :404-408) and engine.py:484-493
// (miss: [1, m], prefix/band split at m-r).  summarize() is attention.py:75-116
// (online softmax, logits scaled by 1/sqrt(d)).
//
// GQA: one work item is (request, kv head, split).  It streams the group's
// KV rows [lo_g, m] (lo_g = min over the group's heads, engine.py:66-77) once
// and evaluates all g heads against them, masking tokens below each head's
// own lo_h.  Every item emits two partials per head: "piece" (t <= m-r) and
// "band" (t > m-r).  Splits are planned on the device from the match output
// (no host sync); the grid is persistent over (split, group) slots, ordered
// split-major so the few live splits of the hit path are dense at the front.
//
// This file holds the generic CUDA-core kernel (any d, d_v, dtype); the
// bf16 d=128 tensor-core kernel is amend_mma.cu.
#include "common.cuh"

namespace mac {

template <int MODE>
__global__ void __launch_bounds__(128) amend_generic_kernel(MacDecodeParams p, const int32_t* __restrict__ mpos,
                                                            const typename Traits<MODE>::acc_t* __restrict__ qrot,
                                                            typename Traits<MODE>::acc_t* __restrict__ part, int TT) {
  using kv_t = typename Traits<MODE>::kv_t;
  using A = typename Traits<MODE>::acc_t;
  const int d = p.head_dim, dv = p.head_dim_v;
  const int Hkv = p.n_kv_heads, g = p.n_q_heads / Hkv, r = p.band;
  const int dp = d + 1, dvp = dv + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  A* Ks = reinterpret_cast<A*>(smem_raw);       // [TT][d+1]
  A* Vs = Ks + (size_t)TT * dp;                  // [TT][dv+1]
  A* S = Vs + (size_t)TT * dvp;                  // [g][TT] logits -> weights
  A* Q = S + (size_t)g * TT;                     // [g][d]
  A* Acc = Q + (size_t)g * d;                    // [2][g][dv]
  A* Mx = Acc + (size_t)2 * g * dv;              // [2][g]
  A* Zs = Mx + 2 * g;                            // [2][g]
  A* Al = Zs + 2 * g;                            // [2][g]
  int* lo_h = reinterpret_cast<int*>(Al + 2 * g); // [g]

  const A scale = (A)(1.0 / sqrt((double)d));
  const int G = p.batch * Hkv;
  const long total = (long)G * p.max_chunks;
  const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, warp = tid >> 5, nwarps = nthr >> 5;
  const kv_t* kc = static_cast<const kv_t*>(p.k_cache);
  const kv_t* vc = static_cast<const kv_t*>(p.v_cache);

  for (long v = blockIdx.x; v < total; v += gridDim.x) {
    const int c = (int)(v / G), grp = (int)(v % G);
    const int b = grp / Hkv, kvh = grp % Hkv;
    const int m = mpos[b];
    // group span [lo_g, m] (every thread computes it; tiny)
    int lo_g = m;
    for (int hl = 0; hl < g; ++hl) {
      int bh = b * p.n_q_heads + kvh * g + hl;
      int use = p.force_miss ? 0 : p.use_hit[bh];
      int lo = head_lo(use, use ? p.match_pos[bh] : 0, r);
      if (lo < lo_g) lo_g = lo;
    }
    const int lo_first = grid_start(lo_g, p.kv_offset);  // shard-local floor
    const Chunking ch = group_chunking(p, m, lo_g);
    if (c >= ch.n) continue;  // block-uniform
    const int t0 = lo_first + c * ch.len;
    const int t1 = min(shard_end(p, m), t0 + ch.len - 1);
    const int cpos = m - r;

    __syncthreads();  // previous item finished with shared memory
    for (int i = tid; i < g * d; i += nthr) {
      int hl = i / d, k = i % d;
      Q[i] = qrot[((int64_t)b * p.n_q_heads + kvh * g + hl) * d + k];
    }
    for (int i = tid; i < 2 * g * dv; i += nthr) Acc[i] = (A)0;
    if (tid < 2 * g) { Mx[tid] = neg_inf<A>(); Zs[tid] = (A)0; }
    if (tid < g) {
      int bh = b * p.n_q_heads + kvh * g + tid;
      int use = p.force_miss ? 0 : p.use_hit[bh];
      lo_h[tid] = head_lo(use, use ? p.match_pos[bh] : 0, r);
    }

    for (int ts = t0; ts <= t1; ts += TT) {
      const int nt = min(TT, t1 - ts + 1);
      __syncthreads();
      for (int i = tid; i < nt * d; i += nthr) {
        int tt = i / d, k = i % d;
        int64_t row = kv_row(p.page_table, p.pages_per_seq, b, ts + tt - p.kv_offset, p.page_size, Hkv, kvh);
        Ks[tt * dp + k] = to_acc<A>(kc[row * d + k]);
      }
      for (int i = tid; i < nt * dv; i += nthr) {
        int tt = i / dv, k = i % dv;
        int64_t row = kv_row(p.page_table, p.pages_per_seq, b, ts + tt - p.kv_offset, p.page_size, Hkv, kvh);
        Vs[tt * dvp + k] = to_acc<A>(vc[row * dv + k]);
      }
      __syncthreads();
      for (int i = tid; i < g * TT; i += nthr) {
        int hl = i / TT, tt = i % TT;
        int t = ts + tt;
        A l = neg_inf<A>();
        if (tt < nt && t >= lo_h[hl]) {
          A s = 0;
          const A* kr = Ks + tt * dp;
          const A* qr = Q + hl * d;
          for (int k = 0; k < d; ++k) s += qr[k] * kr[k];
          l = s * scale;
        }
        S[hl * TT + tt] = l;
      }
      __syncthreads();
      int split = cpos - ts + 1;  // tokens [0, split) are piece, [split, nt) band
      split = split < 0 ? 0 : (split > nt ? nt : split);
      // One warp per (set, head): the piece set reads and rewrites S[hl][0, split), the band set
      // S[hl][split, nt) — disjoint elements of the same row, so no barrier is needed between the
      // max pass and the exp pass (compute-sanitizer racecheck reports these as potential WAR
      // hazards on the shared row; profiles/r02/SUMMARY.md).
      for (int pr = warp; pr < 2 * g; pr += nwarps) {
        const int set = pr / g, hl = pr % g;
        const int a = set == 0 ? 0 : split, e = set == 0 ? split : nt;
        A mx = neg_inf<A>();
        for (int tt = a + lane; tt < e; tt += 32) mx = fmax(mx, S[hl * TT + tt]);
        mx = warp_max(mx);
        const A Mold = Mx[pr];
        const A Mnew = fmax(Mold, mx);
        A sum = 0;
        if (Mnew == neg_inf<A>()) {
          for (int tt = a + lane; tt < e; tt += 32) S[hl * TT + tt] = (A)0;
        } else {
          for (int tt = a + lane; tt < e; tt += 32) {
            A w = fexp(S[hl * TT + tt] - Mnew);
            S[hl * TT + tt] = w;
            sum += w;
          }
        }
        sum = warp_sum(sum);
        if (lane == 0) {
          A alpha = (Mold == neg_inf<A>()) ? (A)0 : fexp(Mold - Mnew);
          if (Mnew == neg_inf<A>()) alpha = (A)1;
          Al[pr] = alpha;
          Zs[pr] = Zs[pr] * alpha + sum;
          Mx[pr] = Mnew;
        }
      }
      __syncthreads();
      for (int i = tid; i < g * dv; i += nthr) {
        const int hl = i / dv, e = i % dv;
        A ap = Acc[i] * Al[hl];
        for (int tt = 0; tt < split; ++tt) ap += S[hl * TT + tt] * Vs[tt * dvp + e];
        Acc[i] = ap;
        A ab = Acc[g * dv + i] * Al[g + hl];
        for (int tt = split; tt < nt; ++tt) ab += S[hl * TT + tt] * Vs[tt * dvp + e];
        Acc[g * dv + i] = ab;
      }
    }
    __syncthreads();
    // partials: [(grp, c, hl, set)] x (dv acc normalised, lse)
    A* out = part + ((int64_t)(grp * p.max_chunks + c) * g) * 2 * dvp;
    for (int i = tid; i < 2 * g * dvp; i += nthr) {
      const int hl = i / (2 * dvp), rem = i % (2 * dvp), set = rem / dvp, e = rem % dvp;
      const int pr = set * g + hl;
      const A z = Zs[pr];
      A val;
      if (e < dv) val = z > (A)0 ? Acc[set * g * dv + hl * dv + e] / z : (A)0;
      else val = z > (A)0 ? Mx[pr] + flog(z) : neg_inf<A>();
      out[i] = val;
    }
  }
}

static inline size_t amend_generic_smem(int TT, int d, int dv, int g, size_t asz) {
  return asz * ((size_t)TT * (d + 1) + (size_t)TT * (dv + 1) + (size_t)g * TT + (size_t)g * d + 2ull * g * dv +
                6ull * g) + sizeof(int) * g + 16;
}

template <int MODE>
cudaError_t launch_amend_generic(const MacDecodeParams& p, cudaStream_t st) {
  using A = typename Traits<MODE>::acc_t;
  Workspace w = workspace_layout(p);
  char* ws = static_cast<char*>(p.workspace);
  const int g = p.n_q_heads / p.n_kv_heads;
  int TT = 64;
  while (TT > 8 && amend_generic_smem(TT, p.head_dim, p.head_dim_v, g, sizeof(A)) > 200 * 1024) TT /= 2;
  size_t smem = amend_generic_smem(TT, p.head_dim, p.head_dim_v, g, sizeof(A));
  cudaError_t e = cudaFuncSetAttribute(amend_generic_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  long total = (long)p.batch * p.n_kv_heads * p.max_chunks;
  int grid = (int)(total < 148 * 16 ? total : 148 * 16);
  amend_generic_kernel<MODE><<<grid, 128, smem, st>>>(p, reinterpret_cast<const int32_t*>(ws + w.mpos_off),
                                                      reinterpret_cast<const A*>(ws + w.qrot_off),
                                                      reinterpret_cast<A*>(ws + w.part_off), TT);
  return cudaGetLastError();
}

template cudaError_t launch_amend_generic<MAC_MODE_F32>(const MacDecodeParams&, cudaStream_t);
template cudaError_t launch_amend_generic<MAC_MODE_BF16>(const MacDecodeParams&, cudaStream_t);
template cudaError_t launch_amend_generic<MAC_MODE_F64>(const MacDecodeParams&, cudaStream_t);

}  // namespace mac
